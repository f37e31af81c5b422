"""Batched-scene mode (NEXT-3): many independent small scenes solved concurrently.

A scene of a few hundred pixels per side fills only a handful of CTAs per sweep, so one
solve leaves the B200 mostly idle.  BatchRunner keeps `slots` plans, each with its own CUDA
stream, workspace and device buffers, and issues the scenes round-robin: every slot's
iteration graph runs concurrently with the others'.  Marshalling only — every step is the
plans' own kernels (cssar_ita_iterate on the slot's stream).
"""
import torch

from .cssar import Plan, _check, _ptr, _stream


class BatchRunner:
    def __init__(self, params, slots=16, op="csa"):
        self.params = params
        self.shape = (int(params.n_az), int(params.n_rg))
        self.streams = [torch.cuda.Stream() for _ in range(slots)]
        self.plans = [Plan(params, op=op, stream=s) for s in self.streams]
        self.Y = [torch.empty(self.shape, dtype=torch.complex64, device="cuda") for _ in range(slots)]
        self.M = [torch.empty((self.shape[0], self.shape[1] // 32), dtype=torch.int32, device="cuda")
                  for _ in range(slots)]
        self.X = [torch.empty(self.shape, dtype=torch.complex64, device="cuda") for _ in range(slots)]

    def run(self, Ys, masks_u8, **ita_kw):
        """Ys: complex64 (n_az, n_rg) tensors (host or device); masks_u8: uint8/bool tensors of the
        same shape.  Returns the reconstructions as a list of host complex64 tensors."""
        out = [None] * len(Ys)
        pending = []
        for i, (Y, m) in enumerate(zip(Ys, masks_u8)):
            q = i % len(self.plans)
            if len(pending) == len(self.plans):       # slot q is reused: collect its last scene
                self._collect(pending.pop(0), out)
            s = self.streams[q]
            with torch.cuda.stream(s):
                self.Y[q].copy_(Y, non_blocking=True)
                mu8 = m.to("cuda", non_blocking=True).to(torch.uint8).contiguous()
                _check(self.plans[q].lib.cssar_pack_mask(_ptr(mu8), _ptr(self.M[q]), self.shape[0], self.shape[1],
                                                         _stream(s)), "cssar_pack_mask")
                self.X[q].zero_()
                self.plans[q].ita_iterate(self.Y[q], self.M[q], X=self.X[q], stream=s, **ita_kw)
                host = torch.empty(self.shape, dtype=torch.complex64, pin_memory=True)
                host.copy_(self.X[q], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s)
            pending.append((i, host, ev))
        while pending:
            self._collect(pending.pop(0), out)
        return out

    @staticmethod
    def _collect(item, out):
        i, host, ev = item
        ev.synchronize()
        out[i] = host
