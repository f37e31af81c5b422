"""Multi-GPU peer-memory plumbing on one B200.

* The CUDA-IPC mapping the fused transposes rely on, between two real processes: each
  process allocates a buffer inside torch's caching allocator (so the pointer is an offset
  into a larger cudaMalloc block, as the bound workspace is), exports the record
  cssar_bind_workspace all-gathers, opens the peer's record, writes a pattern into the peer's
  buffer with a kernel ending in a system-scope fence, and -- after a host-side (gloo)
  barrier, no kernel waits on another process -- checks its own buffer holds the peer's
  pattern.  (Two NCCL ranks cannot share one GPU, and kernels of two processes that spin on
  each other are not allowed on one GPU; the flag barrier's protocol is tested below.)
* The flag barrier that orders the fused sweeps on real ranks: every emulated rank's
  barrier in ONE cooperative launch (co-resident blocks), many rounds, epochs and slots in
  the ranks' real workspaces; then a full emulated solve still matches one GPU bitwise.
"""
import os
import socket

import numpy as np
import pytest

from tests._common import need_gpu

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu():
    need_gpu()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _ipc_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1302_3120_b200 import cssar
        torch.cuda.set_device(0)
        n = 1 << 20
        pad = torch.empty(4096 + 1000 * rank, dtype=torch.uint8, device="cuda")   # offset inside a block
        buf = torch.zeros(n, dtype=torch.int32, device="cuda")
        rec = cssar.ipc_export(buf)
        recs = [None] * world
        dist.all_gather_object(recs, rec)
        peer = (rank + 1) % world
        base, ptr = cssar.ipc_open(recs[peer])
        pattern = 0x5A000000 | (rank << 8) | 0x11
        cssar.peer_store(ptr, pattern, n)
        torch.cuda.synchronize()
        dist.barrier()                       # every process's stores are complete
        src = (rank - 1) % world
        want = (np.uint32(0x5A000000 | (src << 8) | 0x11) ^ np.arange(n, dtype=np.uint32)).view(np.int32)
        got = buf.cpu().numpy()
        ok = bool(np.array_equal(got, want))
        dist.barrier()
        cssar.ipc_close(base)
        del pad
        q.put((rank, ok, None))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


def test_ipc_mapping_between_two_processes():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res


@pytest.mark.parametrize("world", [2, 4, 8, 16])
def test_flag_barrier_protocol_group(world):
    from paper_1302_3120_b200 import Group
    from inputs.configs import SarParams
    p = SarParams(n_az=2048, n_rg=2048)
    g = Group(p, world)
    g.debug_barrier(1000)
    g.debug_barrier(3)          # fresh epochs after a reset of the slots


def test_peer_transpose_flag_group_bitwise():
    """The emulation group with the fused (peer-store) transposes equals one GPU bitwise (the
    flag only gates real NCCL ranks; the group path is the same kernels)."""
    from tests.test_gpu_multi import _group_run, _single_run
    from tests._common import problem
    prob = problem("c1")
    Xg, lg = _group_run(prob, 4, 10)
    Xs, ls = _single_run(prob, 10)
    assert np.array_equal(Xg.view(np.float32), Xs.view(np.float32))
    assert [e["sigma"] for e in lg] == [e["sigma"] for e in ls]
