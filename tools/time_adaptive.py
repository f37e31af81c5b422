"""ms per ITA iteration on c3 with the fixed and the adaptive (eq. 27) step (GPU box)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from inputs import configs  # noqa: E402
from paper_1302_3120_b200 import Plan  # noqa: E402
cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else "c3")
pl = Plan(cfg.params)
Y, mb, mask, sc = bench.make_problem_gpu(cfg, pl)
for mu in (1.0, "adaptive"):
    X = torch.zeros_like(Y)
    pl.ita_iterate(Y, mb, k=cfg.k, mu=mu, iters=5, X=X)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    X, log = pl.ita_iterate(Y, mb, k=cfg.k, mu=mu, iters=30, X=X, log=True)
    e1.record(); torch.cuda.synchronize()
    print(mu, "ms/it", round(e0.elapsed_time(e1) / 30, 3), "mu_i", [round(e["mu"], 4) for e in log[:3]], "resid2",
          f"{log[-1]['resid2']:.5g}")
