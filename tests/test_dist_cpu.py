"""world_size-2 `gloo` tests (CPU) of the multi-GPU host logic (include/cssar.h
world > 1): the slab block algebra of the all-to-all transposes, the blocked row-slab index
the range kernel uses (RgArgs::blk), the sweep schedule with global Doppler rows, and the
exact k-rule select over rank-reduced histograms.  The CUDA path itself runs the same
schedule on one device in tests/test_gpu_multi.py (bitwise equal to one GPU); here real
collectives run between two processes and the per-axis arithmetic comes from the oracle.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _a2a(send_blocks):
    """all-to-all of equal blocks: send_blocks [P][...] -> recv [P][...] (block p from rank p)."""
    x = torch.from_numpy(np.ascontiguousarray(send_blocks))
    if torch.is_complex(x):
        x = torch.view_as_real(x)
    y = torch.empty_like(x)
    dist.all_to_all_single(y, x)
    y = y.numpy()
    if np.iscomplexobj(send_blocks):
        y = y[..., 0] + 1j * y[..., 1]
    return y


def to_col(rowslab, P):
    """row slab [nrow][n_rg] -> column slab [n_az][ncol] (send blocks [q][nrow][ncol])."""
    nrow, n_rg = rowslab.shape
    ncol = n_rg // P
    send = rowslab.reshape(nrow, P, ncol).transpose(1, 0, 2)
    return _a2a(send).reshape(P * nrow, ncol)


def to_row_blocked(colslab, P):
    """column slab [n_az][ncol] -> blocked row slab [P][nrow][ncol] (what libcssar's range
    kernel reads); the column slab itself is the send buffer (block q = rank q's lines)."""
    n_az, ncol = colslab.shape
    return _a2a(colslab.reshape(P, n_az // P, ncol))


def _worker(rank, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from inputs.configs import SarParams
        from oracle import csa
        P = WORLD
        p = SarParams(n_az=256, n_rg=256)
        op = csa.CSAOperator(p)
        rng = np.random.default_rng(5)
        X = rng.standard_normal((p.n_az, p.n_rg)) + 1j * rng.standard_normal((p.n_az, p.n_rg))
        nrow, ncol = p.n_az // P, p.n_rg // P
        lo, hi = rank * nrow, (rank + 1) * nrow
        out = {}

        # 1. transposes: row slab -> column slab is the global column block
        col = to_col(X[lo:hi], P)
        out["col_ok"] = bool(np.array_equal(col, X[:, rank * ncol:(rank + 1) * ncol]))
        # 2. blocked row slab and the range kernel's index (j >> log_w) * blk + r * w + (j & (w-1))
        blk = to_row_blocked(col, P)
        flat = blk.reshape(-1)
        log_w = int(np.log2(ncol))
        j = np.arange(p.n_rg)
        r = np.arange(nrow)[:, None]
        idx = (j >> log_w) * (nrow * ncol) + r * ncol + (j & (ncol - 1))
        out["blocked_ok"] = bool(np.array_equal(flat[idx], X[lo:hi]))

        # 3. the ITA operator schedule on slabs: G = F_eta^-1 o (range G body on row slabs,
        #    global Doppler rows) o F_eta on column slabs, two transposes in between
        U = csa.fft_az(col)                                          # S1 on the column slab
        V = to_row_blocked(U, P).transpose(1, 0, 2).reshape(nrow, p.n_rg)
        full = np.zeros((p.n_az, p.n_rg), dtype=np.complex128)
        full[lo:hi] = V
        V = op.range_segment(full, conj=True)[lo:hi]                 # S2 on rows lo..hi
        Gc = csa.fft_az(to_col(V, P), inverse=True)                  # S3's inverse transform
        allc = [torch.zeros(p.n_az, ncol, 2, dtype=torch.float64) for _ in range(P)]
        dist.all_gather(allc, torch.view_as_real(torch.from_numpy(np.ascontiguousarray(Gc))))
        G = np.concatenate([c[..., 0].numpy() + 1j * c[..., 1].numpy() for c in allc], axis=1)
        ref = op.G(X)
        out["G_err"] = float(np.linalg.norm(G - ref) / np.linalg.norm(ref))

        # 4. exact (k+1)-th largest |b|^2 pattern from rank-reduced histograms: top 11 bits,
        #    then two 10-bit levels (libcssar's split select), ties and zeros included
        b = (rng.standard_normal((p.n_az, p.n_rg)) + 1j * rng.standard_normal((p.n_az, p.n_rg))).astype(np.complex64)
        b.reshape(-1)[:300] = b.reshape(-1)[300:600]
        b.reshape(-1)[1000:3000] = 0
        re, im = b.real.astype(np.float32), b.imag.astype(np.float32)
        u_all = ((re * re) + (im * im)).astype(np.float32).view(np.uint32).reshape(-1)
        u = u_all.reshape(p.n_az, p.n_rg)[lo:hi].reshape(-1)           # this rank's patterns
        sel = {}
        for k in (1, 77, 4096, u_all.size - 2):
            def reduced(counts):
                t = torch.from_numpy(counts.astype(np.int64))
                dist.all_reduce(t)
                return t.numpy()

            def pick(counts, rank_k):
                above = np.concatenate([np.cumsum(counts[::-1])[::-1][1:], [0]])   # # in higher bins
                bbin = int(np.nonzero((above <= rank_k) & (rank_k < above + counts))[0][0])
                return bbin, rank_k - int(above[bbin]), int(above[bbin])

            h = reduced(np.bincount(u >> 20, minlength=2048))
            B, rk, abv = pick(h, k)
            prefix = B
            for sh in (10, 0):
                m = (u >> (sh + 10)) == prefix
                h = reduced(np.bincount((u[m] >> sh) & 1023, minlength=1024))
                d, rk, a2 = pick(h, rk)
                prefix = (prefix << 10) | d
                abv += a2
            srt = np.sort(u_all)[::-1]
            sel[k] = (int(prefix) == int(srt[k]), abv == int(np.count_nonzero(u_all > srt[k])))
        out["select"] = sel
        results[rank] = out
    finally:
        dist.destroy_process_group()


def test_slab_schedule_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        results = mgr.dict()
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, port, results)) for r in range(WORLD)]
        for pr in procs:
            pr.start()
        for pr in procs:
            pr.join(timeout=240)
        assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
        res = dict(results)
    assert sorted(res) == list(range(WORLD))
    for r, out in res.items():
        assert out["col_ok"] and out["blocked_ok"], (r, out)
        assert out["G_err"] <= 1e-12, (r, out["G_err"])
        for k, (val_ok, above_ok) in out["select"].items():
            assert val_ok and above_ok, (r, k)


def test_sparse_x_fold_identity():
    """The sparse-X' decomposition (api.cu sx_s1, sparse.cu): with N = P m and n = m n1 + n2,
    F_p[n2] = sum_{n = n2 mod m} w_N^{p n} x[n] and the m-point DFT of F_p gives bins p + P k2
    of the N-point DFT, for every rank p (numpy, fp64)."""
    import numpy as np
    rng = np.random.default_rng(7)
    N, P, cols = 256, 8, 5
    m = N // P
    x = np.zeros((N, cols), complex)
    idx = rng.choice(N * cols, 40, replace=False)
    x.reshape(-1)[idx] = rng.standard_normal(40) + 1j * rng.standard_normal(40)
    ref = np.fft.fft(x, axis=0)
    n = np.arange(N)
    for p in range(P):
        F = np.zeros((m, cols), complex)
        np.add.at(F, n % m, np.exp(-2j * np.pi * p * n / N)[:, None] * x)
        assert np.abs(np.fft.fft(F, axis=0) - ref[p::P]).max() < 1e-10
