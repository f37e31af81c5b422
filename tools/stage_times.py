"""Per-step device times of the ITA loop on a random problem of any grid (tuning aid):
    python tools/stage_times.py N_AZ N_RG [iters [op]]      (GPU box; honours CSSAR_LIB)"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from inputs.configs import SarParams  # noqa: E402
from paper_1302_3120_b200 import Plan, pack_mask  # noqa: E402


def main():
    n_az, n_rg = int(sys.argv[1]), int(sys.argv[2])
    iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    g = torch.Generator(device="cuda").manual_seed(1)
    Y = torch.randn((n_az, n_rg), dtype=torch.complex64, device="cuda", generator=g)
    mask = torch.rand((n_az, n_rg), device="cuda", generator=g) < 0.5
    Y = torch.where(mask, Y, torch.zeros_like(Y))
    mb = pack_mask(mask)
    op = sys.argv[4] if len(sys.argv) > 4 else "csa"
    pl = Plan(SarParams(n_az=n_az, n_rg=n_rg), op=op)
    k = n_az * n_rg // 100
    X = torch.zeros_like(Y)
    pl.ita_iterate(Y, mb, X=X, k=k, iters=3, check=False)
    pl.ita_iterate(Y, mb, X=X, k=k, iters=iters, profile_stages=True, check=False)
    st, it = pl.stage_times()
    print(json.dumps({"grid": [n_az, n_rg], "op": op, **{kk: round(v / it, 4) for kk, v in st.items()}}))


if __name__ == "__main__":
    main()
