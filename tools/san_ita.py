"""Small ITA run for compute-sanitizer (one tool per call): python tools/san_ita.py [c1] [iters]"""
import sys
import torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from inputs import configs  # noqa: E402
from paper_1302_3120_b200 import Plan, pack_mask  # noqa: E402
cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else "c1")
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
p = cfg.params
pl = Plan(p)
g = torch.Generator(device="cuda").manual_seed(44)
m = (torch.rand((p.n_az, p.n_rg), device="cuda", generator=g) < 0.5)
mb = pack_mask(m.to(torch.uint8))
Y = torch.randn((p.n_az, p.n_rg), dtype=torch.complex64, device="cuda", generator=g)
Y = torch.where(m, Y, torch.zeros_like(Y))
X = pl.ita_iterate(Y, mb, rule="lambda", lam=1.0, iters=iters)
Xb = pl.ita_iterate(Y, mb, rule="lambda", lam=1.0, iters=1, X=pl.ita_iterate(Y, mb, rule="lambda", lam=1.0, iters=1))
torch.cuda.synchronize()
print("done", torch.equal(X.view(torch.float32), Xb.view(torch.float32)))
