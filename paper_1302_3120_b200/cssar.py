"""Thin ctypes binding of libcssar (include/cssar.h): argument marshalling only.

Every step of the hot path runs in the CUDA library; PyTorch supplies device memory and
streams.  There is no CPU fallback: if libcssar.so is missing or the GPU is absent, the
calls raise.
"""
import ctypes
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcssar.so")

CSSAR_THR_SOFT, CSSAR_THR_HALF, CSSAR_THR_HARD, CSSAR_THR_TWOTHIRDS = 1, 2, 3, 4
THR_CODES = {"soft": 1, "half": 2, "hard": 3, "twothirds": 4}
CSSAR_RULE_KSPARSE, CSSAR_RULE_FIXED_LAMBDA = 1, 2

ERRORS = {
    -1: "CSSAR_ERR_INVALID_PARAMS", -2: "CSSAR_ERR_UNSUPPORTED_SIZE", -3: "CSSAR_ERR_BAD_K",
    -4: "CSSAR_ERR_BAD_MU", -5: "CSSAR_ERR_ALIGNMENT", -6: "CSSAR_ERR_NONFINITE", -7: "CSSAR_ERR_CUDA",
    -8: "CSSAR_ERR_WORKSPACE", -9: "CSSAR_ERR_NCCL", -10: "CSSAR_ERR_BAD_PLAN",
}

# every symbol include/cssar.h declares
SYMBOLS = [
    "cssar_plan_create", "cssar_plan_destroy", "cssar_workspace_size", "cssar_bind_workspace",
    "cssar_forward", "cssar_adjoint", "cssar_image", "cssar_ita_iterate", "cssar_pack_mask",
    "cssar_error_string", "cssar_debug_range_sweep", "cssar_debug_az_fft", "cssar_debug_select",
    "cssar_debug_fallbacks", "cssar_stage_times", "cssar_nccl_unique_id", "cssar_group_create",
    "cssar_group_destroy", "cssar_group_workspace_size", "cssar_group_bind_workspace", "cssar_group_ita_iterate",
    "cssar_ita_iters_done", "cssar_plan_set_pulse", "cssar_group_operator", "cssar_ita_status",
    "cssar_debug_ipc_export", "cssar_debug_ipc_open", "cssar_debug_ipc_close", "cssar_debug_peer_store",
    "cssar_group_debug_barrier", "cssar_debug_plan_create_nccl", "cssar_debug_graph_info",
    "cssar_group_debug_graph_info",
]
CSSAR_FLAG_PROFILE_STAGES = 1
CSSAR_FLAG_ADAPTIVE_MU = 2
CSSAR_FLAG_SPARSE_X = 4
CSSAR_FLAG_PEER_TRANSPOSE = 8
CSSAR_FLAG_SPARSE_STATE = 16
CSSAR_FLAG_FUSE_LAMBDA = 32
STAGES = ("S1_az_head", "S2_rg_G", "S3_az_resid", "S4_rg_M", "S5_az_tail", "S6_select")


class CssarError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"{what}: {ERRORS.get(code, code)} ({code})")
        self.code = code


class SarParamsC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("fc", "Kr", "Tr", "Fr", "prf", "Vr", "R_ref", "squint")] + \
               [("n_az", ctypes.c_int64), ("n_rg", ctypes.c_int64), ("op", ctypes.c_int32)]


OP_CODES = {"csa": 1, "rda": 2}   # cssar_op (include/cssar.h): the approximated observation pair


class ItaParamsC(ctypes.Structure):
    _fields_ = [("thr", ctypes.c_int32), ("rule", ctypes.c_int32), ("k", ctypes.c_int64),
                ("lam", ctypes.c_double), ("mu", ctypes.c_double), ("iters", ctypes.c_int32),
                ("flags", ctypes.c_int32), ("tol", ctypes.c_double)]


class IterLogC(ctypes.Structure):
    _fields_ = [("sigma", ctypes.c_float), ("lam", ctypes.c_float), ("support", ctypes.c_int64),
                ("resid2", ctypes.c_double), ("mu", ctypes.c_float), ("gap", ctypes.c_float),
                ("gap_exact", ctypes.c_int32)]


_lib = None


def load_library(path=None):
    """Load libcssar.so (raises if it was not built: there is no fallback).  CSSAR_LIB may
    point at a tuning variant of the same library (tools/variants.py)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("CSSAR_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} not built; run __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    P, V, I, I64, U32P = ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.POINTER(ctypes.c_uint32)
    lib.cssar_plan_create.argtypes = [ctypes.POINTER(P), ctypes.POINTER(SarParamsC), I, I, V, V]
    lib.cssar_plan_destroy.argtypes = [P]
    lib.cssar_workspace_size.argtypes = [P, ctypes.POINTER(ctypes.c_size_t)]
    lib.cssar_bind_workspace.argtypes = [P, V, ctypes.c_size_t]
    for f in ("cssar_forward", "cssar_adjoint", "cssar_image"):
        getattr(lib, f).argtypes = [P, V, V, V, V]
    lib.cssar_ita_iterate.argtypes = [P, V, V, ctypes.POINTER(ItaParamsC), V, ctypes.POINTER(IterLogC), V]
    lib.cssar_pack_mask.argtypes = [V, V, I64, I64, V]
    lib.cssar_error_string.argtypes = [I]
    lib.cssar_error_string.restype = ctypes.c_char_p
    lib.cssar_debug_range_sweep.argtypes = [P, V, I, V]
    lib.cssar_debug_az_fft.argtypes = [P, V, V, I, V]
    lib.cssar_debug_select.argtypes = [P, V, I64, U32P, ctypes.POINTER(ctypes.c_int64), V]
    lib.cssar_debug_fallbacks.argtypes = [P, ctypes.POINTER(ctypes.c_int32), V]
    lib.cssar_debug_graph_info.argtypes = [P, ctypes.POINTER(ctypes.c_int32)]
    lib.cssar_group_debug_graph_info.argtypes = [P, ctypes.POINTER(ctypes.c_int32)]
    lib.cssar_stage_times.argtypes = [P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int32)]
    lib.cssar_nccl_unique_id.argtypes = [V]
    lib.cssar_group_create.argtypes = [ctypes.POINTER(P), ctypes.POINTER(SarParamsC), I, V]
    lib.cssar_group_destroy.argtypes = [P]
    lib.cssar_group_workspace_size.argtypes = [P, ctypes.POINTER(ctypes.c_size_t)]
    lib.cssar_ita_iters_done.argtypes = [P, ctypes.POINTER(ctypes.c_int32)]
    lib.cssar_ita_status.argtypes = [P]
    lib.cssar_debug_ipc_export.argtypes = [V, V]
    lib.cssar_debug_ipc_open.argtypes = [V, ctypes.POINTER(V), ctypes.POINTER(V)]
    lib.cssar_debug_ipc_close.argtypes = [V]
    lib.cssar_debug_peer_store.argtypes = [V, ctypes.c_uint32, I64, V]
    lib.cssar_group_debug_barrier.argtypes = [P, ctypes.c_int32, V]
    lib.cssar_debug_plan_create_nccl.argtypes = [ctypes.POINTER(P), ctypes.POINTER(SarParamsC), V]
    lib.cssar_plan_set_pulse.argtypes = [P, V, I64]
    lib.cssar_group_operator.argtypes = [P, I, ctypes.POINTER(V), ctypes.POINTER(V), ctypes.POINTER(V), V]
    lib.cssar_group_bind_workspace.argtypes = [P, I, V, ctypes.c_size_t]
    lib.cssar_group_ita_iterate.argtypes = [P, ctypes.POINTER(V), ctypes.POINTER(V), ctypes.POINTER(ItaParamsC),
                                            ctypes.POINTER(V), ctypes.POINTER(IterLogC), V]
    for s in SYMBOLS:
        if s != "cssar_error_string":
            getattr(lib, s).restype = I
    _lib = lib
    return lib


def _check(code, what):
    if code != 0:
        raise CssarError(code, what)


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _ptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("libcssar takes device tensors")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _params_c(p, op="csa"):
    return SarParamsC(p.fc, p.Kr, p.Tr, p.Fr, p.prf, p.Vr, p.R_ref, p.squint, int(p.n_az), int(p.n_rg),
                      OP_CODES[op])


def write_log_csv(entries, path):
    """Per-iteration solver report (SPEC "SolverReport", CSV export S:L394): one row
    per X update with sigma_i, lambda_i, mu_i, support size and ||Theta(Y - G X_i)||^2."""
    import csv
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["iter", "sigma", "lambda", "mu", "support", "resid2"])
        for i, e in enumerate(entries):
            w.writerow([i, repr(float(e["sigma"])), repr(float(e["lam"])), repr(float(e["mu"])), int(e["support"]),
                        repr(float(e["resid2"]))])


def nccl_unique_id():
    """A fresh 128-byte ncclUniqueId (bytes) for Plan(world > 1)."""
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    _check(lib.cssar_nccl_unique_id(buf), "cssar_nccl_unique_id")
    return buf.raw


def ipc_export(t):
    """80-byte CUDA-IPC record of a device tensor's storage (cssar_debug_ipc_export)."""
    lib = load_library()
    buf = ctypes.create_string_buffer(80)
    _check(lib.cssar_debug_ipc_export(_ptr(t), buf), "cssar_debug_ipc_export")
    return bytes(buf.raw)


def ipc_open(rec):
    """Map a peer process's record: returns (base, ptr) device addresses (ints)."""
    lib = load_library()
    base, ptr = ctypes.c_void_p(), ctypes.c_void_p()
    _check(lib.cssar_debug_ipc_open(ctypes.create_string_buffer(rec, 80), ctypes.byref(base), ctypes.byref(ptr)),
           "cssar_debug_ipc_open")
    return base.value, ptr.value


def ipc_close(base):
    _check(load_library().cssar_debug_ipc_close(ctypes.c_void_p(base)), "cssar_debug_ipc_close")


def peer_store(ptr, pattern, n_words, stream=None):
    _check(load_library().cssar_debug_peer_store(ctypes.c_void_p(ptr), pattern, n_words, _stream(stream)),
           "cssar_debug_peer_store")


def slab_rows(n_az, world, rank):
    """Azimuth lines [lo, hi) of rank's row slab."""
    h = int(n_az) // int(world)
    return rank * h, (rank + 1) * h


def pack_mask(mask_u8, stream=None):
    """uint8/bool (n_az, n_rg) device tensor -> bit-packed int32 tensor (n_az, n_rg/32)."""
    lib = load_library()
    m = mask_u8.to(torch.uint8).contiguous()
    rows, cols = m.shape
    bits = torch.empty((rows, cols // 32), dtype=torch.int32, device=m.device)
    _check(lib.cssar_pack_mask(_ptr(m), _ptr(bits), rows, cols, _stream(stream)), "cssar_pack_mask")
    return bits


class Plan:
    """cssar_plan: SAR parameters -> phase-coefficient table; operator calls and ITA."""

    def __init__(self, params, stream=None, workspace=True, world=1, rank=0, unique_id=None, op="csa"):
        """world > 1: this process is `rank` of a slab-partitioned plan; its
        arrays are row slabs of n_az/world azimuth lines; unique_id = the 128-byte NCCL id
        (nccl_unique_id() on one rank, shared by the caller, e.g. dist.broadcast_object_list).
        op: "csa" (north star) or "rda" (NEXT-2, the paper's CSRDA pair, eq. 14-18).
        world == 1 with a unique_id: a one-rank NCCL plan that runs the slab path (a test of the
        NCCL plumbing on one GPU, cssar_debug_plan_create_nccl)."""
        self.lib = load_library()
        self.params = params
        self.op = op
        self.world, self.rank = int(world), int(rank)
        self.shape = (int(params.n_az) // self.world, int(params.n_rg))
        h = ctypes.c_void_p()
        pc = _params_c(params, op)
        uid = None
        if self.world > 1 or unique_id is not None:
            if unique_id is None or len(unique_id) != 128:
                raise ValueError("world > 1 needs the 128-byte NCCL unique id")
            uid = ctypes.create_string_buffer(bytes(unique_id), 128)
        if self.world == 1 and uid is not None:     # one-rank NCCL plan on the slab path (test hook)
            _check(self.lib.cssar_debug_plan_create_nccl(ctypes.byref(h), ctypes.byref(pc), uid),
                   "cssar_debug_plan_create_nccl")
        else:
            _check(self.lib.cssar_plan_create(ctypes.byref(h), ctypes.byref(pc), self.world, self.rank, uid,
                                              _stream(stream)), "cssar_plan_create")
        self.h = h
        self.ws = None
        if workspace:
            self.bind_workspace()

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.cssar_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def workspace_size(self):
        n = ctypes.c_size_t()
        _check(self.lib.cssar_workspace_size(self.h, ctypes.byref(n)), "cssar_workspace_size")
        return n.value

    def bind_workspace(self, ws=None):
        nbytes = self.workspace_size()
        if ws is None:
            ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        _check(self.lib.cssar_bind_workspace(self.h, _ptr(ws), ws.numel()), "cssar_bind_workspace")
        self.ws = ws

    def _out(self, out):
        return torch.empty(self.shape, dtype=torch.complex64, device="cuda") if out is None else out

    def forward(self, X, mask_bits=None, out=None, stream=None):
        """A X = Theta o G(X)."""
        out = self._out(out)
        _check(self.lib.cssar_forward(self.h, _ptr(X), _ptr(mask_bits), _ptr(out), _stream(stream)), "cssar_forward")
        return out

    def adjoint(self, R, mask_bits=None, out=None, stream=None):
        """A^H R = M(Theta o R)."""
        out = self._out(out)
        _check(self.lib.cssar_adjoint(self.h, _ptr(R), _ptr(mask_bits), _ptr(out), _stream(stream)), "cssar_adjoint")
        return out

    def image(self, Y, mask_bits=None, out=None, stream=None):
        """Matched-filter (CSA) image M(Theta o Y), eq. 10."""
        out = self._out(out)
        _check(self.lib.cssar_image(self.h, _ptr(Y), _ptr(mask_bits), _ptr(out), _stream(stream)), "cssar_image")
        return out

    def ita_iterate(self, Y, mask_bits, *, thr="soft", rule="k", k=0, lam=0.0, mu=1.0, iters=1, X=None,
                    log=False, profile_stages=False, stream=None, tol=0.0, sparse=False, peer=False, check=True,
                    sparse_state=False, fuse_lambda=False):
        """Algorithm 1: X <- E(X + mu M(Theta o (Y - G X))) `iters` times, in place on X.
        mu="adaptive": the eq. 27 step rule (CSSAR_FLAG_ADAPTIVE_MU).  tol > 0: stop after the
        first update with ||X_(i+1) - X_i|| <= tol ||X_i|| (self.iters_done = updates performed).
        fuse_lambda=True fuses S5 with the next S1 under the fixed-lambda rule (CSSAR_FLAG_FUSE_LAMBDA).
        sparse_state=True requests the sparse-state list schedule (world 1, NEXT-3; see
        include/cssar.h CSSAR_FLAG_SPARSE_STATE).
        world > 1: peer=True requests the fused peer-memory transposes (CSSAR_FLAG_PEER_TRANSPOSE),
        sparse=True additionally the sparse-X' first sweep.
        check=True waits for the solve and raises CssarError(CSSAR_ERR_NONFINITE) if a NaN/Inf
        entered the iterate (cssar_ita_status); check=False returns without synchronising."""
        if X is None:
            X = torch.zeros(self.shape, dtype=torch.complex64, device="cuda")
        adaptive = isinstance(mu, str)
        if adaptive and mu != "adaptive":
            raise ValueError("mu must be a positive number or 'adaptive'")
        prm = ItaParamsC(THR_CODES[thr],
                         CSSAR_RULE_KSPARSE if rule == "k" else CSSAR_RULE_FIXED_LAMBDA,
                         int(k), float(lam), 1.0 if adaptive else float(mu), int(iters),
                         (CSSAR_FLAG_PROFILE_STAGES if profile_stages else 0) |
                         (CSSAR_FLAG_ADAPTIVE_MU if adaptive else 0) | (CSSAR_FLAG_SPARSE_X if sparse else 0) |
                         (CSSAR_FLAG_PEER_TRANSPOSE if peer else 0) | (CSSAR_FLAG_SPARSE_STATE if sparse_state else 0) |
                         (CSSAR_FLAG_FUSE_LAMBDA if fuse_lambda else 0),
                         float(tol))
        logbuf = (IterLogC * max(1, iters))() if log else None
        rc = self.lib.cssar_ita_iterate(self.h, _ptr(Y), _ptr(mask_bits), ctypes.byref(prm), _ptr(X),
                                        logbuf if log else None, _stream(stream))
        _check(rc, "cssar_ita_iterate")
        if check:
            _check(self.lib.cssar_ita_status(self.h), "cssar_ita_status")
        done = ctypes.c_int32()
        _check(self.lib.cssar_ita_iters_done(self.h, ctypes.byref(done)), "cssar_ita_iters_done")
        self.iters_done = done.value
        if log:
            entries = [dict(sigma=e.sigma, lam=e.lam, support=int(e.support), resid2=e.resid2, mu=e.mu,
                            gap=e.gap, gap_exact=bool(e.gap_exact))
                       for e in list(logbuf)[:self.iters_done]]
            return X, entries
        return X

    def status(self):
        """Wait for the last ita_iterate and raise on a non-finite iterate (cssar_ita_status)."""
        _check(self.lib.cssar_ita_status(self.h), "cssar_ita_status")

    def set_pulse(self, pulse=None):
        """RDA plans: recorded transmitted pulse (complex samples at (m - (L-1)/2)/F_r) as the range
        filter; None restores the chirp P_tau."""
        if pulse is None:
            _check(self.lib.cssar_plan_set_pulse(self.h, None, 0), "cssar_plan_set_pulse")
            return
        import numpy as np
        buf = np.ascontiguousarray(np.asarray(pulse, dtype=np.complex64))
        _check(self.lib.cssar_plan_set_pulse(self.h, buf.ctypes.data_as(ctypes.c_void_p), buf.size),
               "cssar_plan_set_pulse")

    def stage_times(self):
        """Per-step device milliseconds (summed) of the last profile_stages run, and its iterations."""
        ms = (ctypes.c_double * 6)()
        it = ctypes.c_int32()
        _check(self.lib.cssar_stage_times(self.h, ms, ctypes.byref(it)), "cssar_stage_times")
        return dict(zip(STAGES, list(ms))), it.value

    def solve_host(self, Y_host, mask_bits_host, out_host=None, stream=None, **ita_kw):
        """End-to-end user call: host (pinned) Y and mask -> device -> ITA -> host X."""
        Y = Y_host.to("cuda", non_blocking=True)
        mb = None if mask_bits_host is None else mask_bits_host.to("cuda", non_blocking=True)
        X = torch.zeros(self.shape, dtype=torch.complex64, device="cuda")
        self.ita_iterate(Y, mb, X=X, stream=stream, **ita_kw)
        if out_host is None:
            out_host = torch.empty(self.shape, dtype=torch.complex64, pin_memory=True)
        out_host.copy_(X, non_blocking=True)
        return out_host

    # ---- test hooks
    def debug_range_sweep(self, U, gbody, stream=None):
        _check(self.lib.cssar_debug_range_sweep(self.h, _ptr(U), int(gbody), _stream(stream)), "range_sweep")
        return U

    def debug_az_fft(self, inp, out=None, dir=-1, stream=None):
        out = self._out(out)
        _check(self.lib.cssar_debug_az_fft(self.h, _ptr(inp), _ptr(out), int(dir), _stream(stream)), "az_fft")
        return out

    def debug_select(self, b, k, stream=None):
        s2 = ctypes.c_uint32()
        above = ctypes.c_int64()
        _check(self.lib.cssar_debug_select(self.h, _ptr(b), int(k), ctypes.byref(s2), ctypes.byref(above),
                                           _stream(stream)), "select")
        return s2.value, above.value

    def debug_fallbacks(self, stream=None):
        v = ctypes.c_int32()
        _check(self.lib.cssar_debug_fallbacks(self.h, ctypes.byref(v), _stream(stream)), "fallbacks")
        return v.value

    def debug_graph_info(self):
        """1 when the cached multi-GPU iteration graph gates the select's fallback round with a
        conditional node (cssar_debug_graph_info)."""
        v = ctypes.c_int32()
        _check(self.lib.cssar_debug_graph_info(self.h, ctypes.byref(v)), "cssar_debug_graph_info")
        return v.value


def _itaprm(thr, rule, k, lam, mu, iters, profile_stages=False):
    return ItaParamsC(THR_CODES[thr],
                      CSSAR_RULE_KSPARSE if rule == "k" else CSSAR_RULE_FIXED_LAMBDA,
                      int(k), float(lam), float(mu), int(iters),
                      CSSAR_FLAG_PROFILE_STAGES if profile_stages else 0)


class Group:
    """cssar_group: `world` rank plans emulated on the current device — the multi-GPU
    schedule (slab partition, transposes, reduced select) with device-copy exchanges."""

    def __init__(self, params, world, stream=None, op="csa"):
        self.lib = load_library()
        self.params = params
        self.op = op
        self.world = int(world)
        self.shape = (int(params.n_az) // self.world, int(params.n_rg))
        h = ctypes.c_void_p()
        pc = _params_c(params, op)
        _check(self.lib.cssar_group_create(ctypes.byref(h), ctypes.byref(pc), self.world, _stream(stream)),
               "cssar_group_create")
        self.h = h
        n = ctypes.c_size_t()
        _check(self.lib.cssar_group_workspace_size(self.h, ctypes.byref(n)), "cssar_group_workspace_size")
        self.ws = []
        for r in range(self.world):
            ws = torch.empty(n.value, dtype=torch.uint8, device="cuda")
            _check(self.lib.cssar_group_bind_workspace(self.h, r, _ptr(ws), ws.numel()), "cssar_group_bind_workspace")
            self.ws.append(ws)

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.cssar_group_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def debug_graph_info(self):
        """1 when the cached iteration graph gates the fallback round with a conditional node."""
        v = ctypes.c_int32()
        _check(self.lib.cssar_group_debug_graph_info(self.h, ctypes.byref(v)), "cssar_group_debug_graph_info")
        return v.value

    def debug_barrier(self, rounds, stream=None):
        """`rounds` flag-barrier rounds over all ranks in one cooperative launch."""
        _check(self.lib.cssar_group_debug_barrier(self.h, int(rounds), _stream(stream)), "cssar_group_debug_barrier")

    def _operator(self, forward, ins, mask_bits, outs, stream):
        W = self.world
        arr = ctypes.c_void_p * W
        if outs is None:
            outs = [torch.empty(self.shape, dtype=torch.complex64, device="cuda") for _ in range(W)]
        ms = arr(*([_ptr(m) for m in mask_bits] if mask_bits is not None else [None] * W))
        _check(self.lib.cssar_group_operator(self.h, int(forward), arr(*[_ptr(x) for x in ins]), ms,
                                             arr(*[_ptr(y) for y in outs]), _stream(stream)), "cssar_group_operator")
        return outs

    def forward(self, Xs, mask_bits=None, outs=None, stream=None):
        """Row slabs of Theta o G(X) (cssar_forward on world ranks)."""
        return self._operator(True, Xs, mask_bits, outs, stream)

    def adjoint(self, Rs, mask_bits=None, outs=None, stream=None):
        """Row slabs of M(Theta o R) (cssar_adjoint / cssar_image on world ranks)."""
        return self._operator(False, Rs, mask_bits, outs, stream)

    def ita_iterate(self, Ys, mask_bits, Xs, *, thr="soft", rule="k", k=0, lam=0.0, mu=1.0, iters=1, log=False,
                    stream=None, sparse=False):
        """Ys, Xs: lists of row-slab tensors (rank order); mask_bits: list or None.
        sparse=True: the sparse-X' schedule (CSSAR_FLAG_SPARSE_X)."""
        W = self.world
        arr = ctypes.c_void_p * W
        ys = arr(*[_ptr(y) for y in Ys])
        ms = arr(*([_ptr(m) for m in mask_bits] if mask_bits is not None else [None] * W))
        xs = arr(*[_ptr(x) for x in Xs])
        prm = _itaprm(thr, rule, k, lam, mu, iters)
        if sparse:
            prm.flags |= CSSAR_FLAG_SPARSE_X
        logbuf = (IterLogC * max(1, iters))() if log else None
        _check(self.lib.cssar_group_ita_iterate(self.h, ys, ms, ctypes.byref(prm), xs, logbuf if log else None,
                                                _stream(stream)), "cssar_group_ita_iterate")
        if log:
            return [dict(sigma=e.sigma, lam=e.lam, support=int(e.support), resid2=e.resid2, mu=e.mu,
                         gap=e.gap, gap_exact=bool(e.gap_exact))
                    for e in list(logbuf)[:iters]]
        return None
