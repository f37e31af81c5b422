"""End-to-end use of the library on a seeded synthetic scene (GPU box):

    python examples/reconstruct.py [c2|c3|...] [--op csa|rda] [--iters N] [--tol T] [--csv log.csv]

Builds a plan from the config's SAR parameters, simulates the sub-sampled echo with the
library's own forward operator (Y = Theta o (G X_true + noise)), reconstructs with
Algorithm 1 (k-sparsity rule) and reports the per-iteration log, the recovered fraction of
the scene's support and the device time.
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs import configs, synth  # noqa: E402
from paper_1302_3120_b200 import Plan, pack_mask  # noqa: E402
from paper_1302_3120_b200.cssar import write_log_csv  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="c2")
    ap.add_argument("--op", default="csa", choices=["csa", "rda"])
    ap.add_argument("--iters", type=int, default=None)
    ap.add_argument("--tol", type=float, default=0.0)
    ap.add_argument("--csv", default=None)
    args = ap.parse_args()
    cfg = configs.get(args.config)
    p = cfg.params
    plan = Plan(p, op=args.op)
    sc = synth.make_scene(cfg)
    X_true = torch.zeros((p.n_az, p.n_rg), dtype=torch.complex64, device="cuda")
    X_true.view(-1)[torch.from_numpy(sc.idx).cuda()] = torch.from_numpy(sc.val.astype(np.complex64)).cuda()
    mask = torch.from_numpy(synth.make_mask(cfg)).cuda()
    mb = pack_mask(mask.to(torch.uint8))
    Yc = plan.forward(X_true, None)
    s2 = (Yc.abs() ** 2)[mask].mean() / 10.0 ** (cfg.snr_db / 10.0)
    noise = torch.from_numpy(synth.noise_unit(cfg, dtype=np.complex64)).cuda()
    Y = torch.where(mask, Yc + torch.sqrt(s2) * noise, torch.zeros_like(Yc)).contiguous()
    del Yc, noise
    iters = args.iters or cfg.iters
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    X, log = plan.ita_iterate(Y, mb, thr=cfg.thr, rule=cfg.rule, k=cfg.k, lam=cfg.lam, mu=cfg.mu, iters=iters,
                              tol=args.tol, log=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    found = torch.zeros(p.n_az * p.n_rg, dtype=torch.bool, device="cuda")
    found[X.view(-1).abs() > 0] = True
    hit = found[torch.from_numpy(sc.idx).cuda()].float().mean().item()
    rel = ((X - X_true).abs().pow(2).sum() / X_true.abs().pow(2).sum()).sqrt().item()
    for i in (0, len(log) // 2, len(log) - 1):
        e = log[i]
        print(f"iter {i:4d}: sigma {e['sigma']:.4g}  support {e['support']}  ||r||^2 {e['resid2']:.5g}")
    print(f"{args.config} ({p.n_az}x{p.n_rg}, {args.op}): {plan.iters_done} iterations in {ms:.1f} ms "
          f"({ms / max(plan.iters_done, 1):.3f} ms/it); truth support recovered {100 * hit:.1f}%, "
          f"relative error {rel:.3f}")
    if args.csv:
        write_log_csv(log, args.csv)


if __name__ == "__main__":
    main()
