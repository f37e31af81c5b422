#!/usr/bin/env python
"""Benchmark of the ITA hot path (one step = one ITA iteration S1..S6 over the whole scene).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl cssar|reference]

Workload: BASELINE.json configs[3] (c3), the configuration the metric's 1/2/4/8-GPU runs are
quoted on: 8192 x 8192 complex64, 1% Rayleigh clutter + 500 bright targets, 60% azimuth-line
mask, 15 dB, soft threshold, k-rule k = 671589, mu = 1.  (c4, 32768 x 16384, also fits one
B200; it is measured in the line's "c4" object.)  Synthetic inputs from inputs/ (seeded), echo
Y = Theta o (G(X_true) + noise) generated with the library's own forward operator (P:L47
inverse-focusing simulation); arrays are 512 MiB each, larger than L2 (126 MB), so no L2
flush is needed between steps.

Prints ONE JSON line (rank 0).  value = complex samples * iterations / s of the scene.
N > 1 (torchrun): the SAME c3 scene slab-partitioned over the ranks by azimuth lines
(NCCL all-to-all transposes between the sweeps by default; --peer-transpose
fuses them into the sweeps as CUDA-IPC peer-memory stores and adds the sparse-X' first sweep;
reduced exact select, its fallback round a conditional graph node) -> "scaling": "strong";
the time is the max over ranks.  The line also carries a "library_chain" object: the same
iteration composed from torch.fft (cuFFT) + torch ops on this GPU (timing context).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_SAMPLE = {  # algorithmic HBM bytes per sample per launch
    "S1_az_head": 16.0, "S2_rg_G": 16.0, "S3_az_resid": 24.125, "S4_rg_M": 16.0, "S5_az_tail": 24.0,
    "S6_select": 0.0,
}
ITER_BYTES_PER_SAMPLE = 96.125     # k-rule, SURVEY.md 8(a)
# BASELINE.json's metric; `value` is its complex samples*iter/s part (it_per_s rides along)
METRIC = "ITA iterations/sec and complex samples\u00b7iter/s vs HBM roofline, 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default="c3")
    ap.add_argument("--op", default="csa", choices=["csa", "rda"],
                    help="approximated observation pair (rda: NEXT-2, the paper's CSRDA; not the north star)")
    ap.add_argument("--impl", default="cssar", choices=["cssar", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--no-c4", action="store_true", help="skip the c4 (32768 x 16384) object")
    ap.add_argument("--no-library", action="store_true", help="skip the torch.fft library-chain comparator")
    ap.add_argument("--no-sparse-state", action="store_true", help="skip the sparse-state (NEXT-3) object")
    ap.add_argument("--peer-transpose", action="store_true",
                    help="N > 1: fused peer-memory transposes and the sparse-X' sweep (not yet validated on >1 GPU)")
    ap.add_argument("--slab", action="store_true",
                    help="diagnostic: at N = 1 run the multi-rank slab path over a one-rank NCCL communicator "
                         "(transposes to itself) instead of the single-GPU schedule")
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms while running."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "100", "-i", str(self.index)],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        rows = [r.split(",") for r in out.strip().splitlines() if r.strip()]
        rows = [[c.strip() for c in r] for r in rows if len(r) >= 8]
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = max(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        loaded = [s for s in sm if s > 0.5 * mx] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())}


def make_problem_gpu(cfg, plan, seed_offset=0):
    """Seeded c-config inputs on the device; echo via the library's forward operator."""
    import dataclasses
    import numpy as np
    import torch
    from inputs import synth
    from paper_1302_3120_b200 import pack_mask
    if seed_offset:
        cfg = dataclasses.replace(cfg, seed=cfg.seed + 1000 * seed_offset)
    p = cfg.params
    sc = synth.make_scene(cfg)
    X = torch.zeros((p.n_az, p.n_rg), dtype=torch.complex64, device="cuda")
    X.view(-1)[torch.from_numpy(sc.idx).cuda()] = torch.from_numpy(sc.val.astype(np.complex64)).cuda()
    mask = torch.from_numpy(synth.make_mask(cfg)).cuda()
    mb = pack_mask(mask.to(torch.uint8))
    Yc = plan.forward(X, None)
    sig = (Yc.abs() ** 2)[mask].mean()
    s2 = sig / 10.0 ** (cfg.snr_db / 10.0)
    noise = torch.from_numpy(synth.noise_unit(cfg, dtype=np.complex64)).cuda()
    Y = torch.where(mask, Yc + torch.sqrt(s2) * noise, torch.zeros_like(Yc))
    del Yc, noise, X
    torch.cuda.synchronize()
    return Y.contiguous(), mb, mask, sc


def timed_iters(plan, Y, mb, X, iters, **kw):
    """Device time (CUDA events on the current stream) of one ita_iterate call of `iters`."""
    import torch
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    plan.ita_iterate(Y, mb, X=X, iters=iters, check=False, **kw)
    e1.record(stream)
    torch.cuda.synchronize()
    plan.status()
    return e0.elapsed_time(e1)


def stage_profile(plan, Y, mb, X, iters, **kw):
    plan.ita_iterate(Y, mb, X=X, iters=iters, profile_stages=True, **kw)
    st_ms, it_meas = plan.stage_times()
    return {k: v / it_meas for k, v in st_ms.items()}


def measure_c4(args, peak, peak_kind):
    """BASELINE.json configs[4] (c4, 32768 x 16384, Fr = 120 MHz, 0.5% clutter, 50% mask,
    k = 2684355, 50 iterations) on one GPU: graph-replayed iterations, per-step stage times,
    the iteration's HBM roofline, and an end-to-end solve through the public API."""
    import torch
    from inputs import configs
    from paper_1302_3120_b200 import Plan
    from paper_1302_3120_b200.cssar import STAGES
    cfg = configs.get("c4")
    p = cfg.params
    n = p.n_az * p.n_rg
    plan = Plan(p)
    Y, mb, mask, sc = make_problem_gpu(cfg, plan)
    del mask
    X = torch.zeros_like(Y)
    kw = dict(thr=cfg.thr, rule=cfg.rule, k=cfg.k, lam=cfg.lam, mu=cfg.mu)
    plan.ita_iterate(Y, mb, X=X, iters=3, **kw)
    steps = 10
    ms = timed_iters(plan, Y, mb, X, steps, **kw)
    it_s = steps / (ms * 1e-3)
    stages = stage_profile(plan, Y, mb, X, 5, **kw)
    dom = max((s for s in STAGES if s != "S6_select"), key=lambda s: stages[s])
    dom_ach = BYTES_PER_SAMPLE[dom] * n / (stages[dom] * 1e-3) / 1e9
    iter_ach = ITER_BYTES_PER_SAMPLE * n * it_s / 1e9
    tf = os.path.join(ROOT, "profiles", "traffic_c4.json")
    traffic = json.load(open(tf)).get(dom) if os.path.exists(tf) else None
    out = {"workload": f"c4: {p.n_az}x{p.n_rg} complex64, Fr {p.Fr / 1e6:.0f} MHz, {cfg.scene} scene, {cfg.mask} "
                       f"mask {cfg.rate}, SNR {cfg.snr_db} dB, soft threshold, k = {cfg.k}",
           "value": n * it_s, "unit": "samples*it/s", "ms_per_step": ms / steps, "it_per_s": it_s, "steps": steps,
           "stages_ms": stages,
           "roofline": {"bound": "hbm", "kernel": dom, "achieved": dom_ach, "peak": peak, "unit": "GB/s",
                        "frac": dom_ach / peak, "traffic": traffic, "peak_kind": peak_kind,
                        "algorithmic_bytes_per_launch": BYTES_PER_SAMPLE[dom] * n, "avg_launch_ms": stages[dom]},
           "iteration_roofline": {"bound": "hbm", "achieved": iter_ach, "peak": peak, "unit": "GB/s",
                                  "frac": iter_ach / peak, "bytes_per_sample": ITER_BYTES_PER_SAMPLE},
           "select_fallbacks": plan.debug_fallbacks()}
    if not args.no_e2e:
        Yh = Y.cpu().pin_memory()
        mbh = mb.cpu().pin_memory()
        del Y, X
        torch.cuda.empty_cache()
        Xh = torch.empty_like(Yh).pin_memory()
        plan.solve_host(Yh, mbh, out_host=Xh, iters=2, **kw)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        plan.solve_host(Yh, mbh, out_host=Xh, iters=cfg.iters, **kw)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        out["e2e"] = {"value": n * cfg.iters / dt, "unit": "samples*it/s",
                      "h2d_bytes_per_step": (Yh.numel() * 8 + mbh.numel() * 4) / cfg.iters,
                      "d2h_bytes_per_step": Xh.numel() * 8 / cfg.iters, "solve_iters": cfg.iters}
    del plan
    torch.cuda.empty_cache()
    return out


def launches(steps, rule, slab, cond, fallbacks, peer):
    """libcssar kernel launches in the timed ita_iterate call (init + finalize = 2).  World 1:
    S1..S5 + sel_coarse, fb_hist, fb_find, fb_collect, sel_fine (the fallback kernels exit early
    when not needed) = 10 per iteration (k-rule), S1..S5 + the lambda step = 6 (fixed lambda).
    Slab path: the sweeps + sel_coarse, three fine-level kernels and, when the iteration graph
    gates the fallback round with a conditional node (cond), a set-condition kernel plus the
    three fallback kernels only in the iterations that fell back; + 4 flag barriers with peer
    transposes (the sparse-X' S1 adds its compact + fold kernels from iteration 1 on)."""
    if not slab:
        return steps * (10 if rule == "k" else 6) + 2
    per = 5 + (4 + (1 if cond else 3) if rule == "k" else 1) + (4 if peer else 0) + (2 if peer and rule == "k" else 0)
    return steps * per + (3 * fallbacks if cond and rule == "k" else 0) + 2


def library_chain(Y, mask, k, mu, steps=10, warm=3):
    """SURVEY 8(d) "library chain" comparator (context, not the product and not a parity path):
    the same ITA iteration composed from torch.fft (cuFFT) and torch elementwise / topk ops in
    complex64 on this GPU -- E_sigma (soft), F_eta, Phi3*, F_tau, Phi2*, F_tau^-1, Phi1*, F_eta^-1,
    r = Theta(Y - g), the M chain, b = X + mu D, sigma = (k+1)-th largest |b| by torch.topk.  The
    phase screens are seeded unit phasors of the operator's shape: every multiply, FFT and select
    the chain performs is the one the operator needs, so the time is that of the composition."""
    import math
    import torch
    n_az, n_rg = Y.shape
    g = torch.Generator(device="cuda").manual_seed(1302)

    def phasor():
        return torch.polar(torch.ones(n_az, n_rg, device="cuda"),
                           2 * math.pi * torch.rand(n_az, n_rg, device="cuda", generator=g))
    P1, P2, P3 = phasor(), phasor(), phasor()
    P1c, P2c, P3c = P1.conj().resolve_conj(), P2.conj().resolve_conj(), P3.conj().resolve_conj()
    maskf = mask.to(torch.float32)
    fft, ifft = torch.fft.fft, torch.fft.ifft

    def step(b, sigma):
        mag = b.abs()
        X = b * torch.clamp(1 - sigma / mag.clamp_min(1e-30), min=0)                  # E_sigma(b)
        U = fft(X, dim=0, norm="ortho").mul_(P3c)
        U = fft(U, dim=1, norm="ortho").mul_(P2c)
        U = ifft(U, dim=1, norm="ortho").mul_(P1c)
        r = (Y - ifft(U, dim=0, norm="ortho")).mul_(maskf)                            # Theta(Y - G X)
        V = fft(r, dim=0, norm="ortho").mul_(P1)
        V = fft(V, dim=1, norm="ortho").mul_(P2)
        V = ifft(V, dim=1, norm="ortho").mul_(P3)
        b = X.add_(ifft(V, dim=0, norm="ortho"), alpha=mu)                             # X + mu M(r)
        sigma = torch.topk(b.abs().view(-1), k + 1, sorted=False).values.min()
        return b, sigma

    b = Y.clone()
    sigma = torch.zeros((), device="cuda")
    for _ in range(warm):
        b, sigma = step(b, sigma)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(steps):
        b, sigma = step(b, sigma)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    del P1, P2, P3, P1c, P2c, P3c, maskf, b
    torch.cuda.empty_cache()
    return {"ms_per_step": ms, "it_per_s": 1e3 / ms, "value": n_az * n_rg * 1e3 / ms, "unit": "samples*it/s",
            "steps": steps, "note": "the iteration composed from torch.fft (cuFFT) + torch elementwise / topk "
            "ops, complex64, same grid and k; timing context only (seeded unit phase screens, not a parity path)"}


def cpu_baseline(cfg_name, n_az, n_rg, iters):
    """The fp64 oracle (as it stands) timed on this host on a bounded sample of the workload."""
    import dataclasses
    import numpy as np
    from inputs import configs, synth
    from oracle import csa, echo, ita
    base = configs.get(cfg_name)
    cfg = configs.with_grid(base, n_az, n_rg)
    sc = synth.make_scene(cfg)
    cfg = dataclasses.replace(cfg, k=int(sc.idx.size))
    op = csa.CSAOperator(cfg.params)
    prob = synth.make_problem(cfg, lambda s, c: echo.inverse_csa_echo(op, s.dense()))
    Y = prob.Y.astype(np.complex128)
    ita.ita(op, Y, prob.mask, thr=cfg.thr, rule=cfg.rule, k=cfg.k, mu=cfg.mu, iters=1)   # warm (phase screens)
    t0 = time.perf_counter()
    ita.ita(op, Y, prob.mask, thr=cfg.thr, rule=cfg.rule, k=cfg.k, mu=cfg.mu, iters=iters)
    dt = time.perf_counter() - t0
    return dict(value=n_az * n_rg * iters / dt, unit="samples*it/s", cores=len(os.sched_getaffinity(0)),
                kind="oracle", seconds=dt,
                sample=f"{cfg_name} recipe on a {n_az}x{n_rg} grid (k = {cfg.k}), {iters} ITA iteration(s), "
                       f"fp64 numpy/scipy.fft (workers = all cores)")


def run_reference(args):
    """--impl reference: the oracle on the host cores, each step one ITA iteration on a bounded
    sample of the workload (c3 recipe on a 1024 x 2048 grid)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import dataclasses
    import numpy as np
    from inputs import configs, synth
    from oracle import csa, echo, ita
    n_az, n_rg = 1024, 2048
    cfg = configs.with_grid(configs.get(args.config), n_az, n_rg)
    sc = synth.make_scene(cfg)
    cfg = dataclasses.replace(cfg, k=int(sc.idx.size))
    op = csa.CSAOperator(cfg.params)
    prob = synth.make_problem(cfg, lambda s, c: echo.inverse_csa_echo(op, s.dense()))
    Y = prob.Y.astype(np.complex128)
    X = np.zeros_like(Y)
    for _ in range(args.warmup):
        X = ita.ita(op, Y, prob.mask, thr=cfg.thr, rule=cfg.rule, k=cfg.k, mu=cfg.mu, iters=1, X0=X)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        X = ita.ita(op, Y, prob.mask, thr=cfg.thr, rule=cfg.rule, k=cfg.k, mu=cfg.mu, iters=1, X0=X)
    dt = time.perf_counter() - t0
    value = n_az * n_rg * args.steps / dt
    cores = len(os.sched_getaffinity(0))
    sample = f"{args.config} recipe on a {n_az}x{n_rg} grid (k = {cfg.k}), one ITA iteration per step"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples*it/s",
        "n_gpus": args.gpus, "device": "host cpu (the oracle)", "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: bounded sample of the recipe on {n_az}x{n_rg} (k = {cfg.k})",
                   "n_az": n_az, "n_rg": n_rg, "k": cfg.k, "iters_per_step": 1},
        "cpu_baseline": {"value": value, "unit": "samples*it/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "samples*it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


_JSON_OUT = None


def emit(line):
    """The ONE JSON line on the process's original stdout."""
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    global _JSON_OUT
    # keep stdout for the JSON line alone: anything else written to fd 1 (NCCL's version
    # banner, library chatter) goes to stderr
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch
    import torch.distributed as dist
    from inputs import configs
    from paper_1302_3120_b200 import Plan
    from paper_1302_3120_b200.cssar import STAGES

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = configs.get(args.config)
    p = cfg.params
    n = p.n_az * p.n_rg
    plan = Plan(p, op=args.op)
    Y, mb, mask, sc = make_problem_gpu(cfg, plan)
    X = torch.zeros_like(Y)
    kw = dict(thr=cfg.thr, rule=cfg.rule, k=cfg.k, lam=cfg.lam, mu=cfg.mu)
    slab = world > 1 or args.slab
    if slab and args.peer_transpose:
        # fused peer-memory transposes + sparse-X' first sweep (CSSAR_FLAG_PEER_TRANSPOSE |
        # CSSAR_FLAG_SPARSE_X); default: NCCL all-to-all transposes (validated path)
        kw["peer"] = True
        kw["sparse"] = True
    if slab:
        # strong scaling: ONE scene slab-partitioned by azimuth lines; NCCL
        # all-to-all transposes inside libcssar, communicator from a broadcast unique id
        from paper_1302_3120_b200 import nccl_unique_id, slab_rows
        uid = [nccl_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(uid, src=0)
        lo, hi = slab_rows(p.n_az, world, rank)
        Y = Y[lo:hi].contiguous()
        mb = mb[lo:hi].contiguous()
        X = torch.zeros_like(Y)
        del plan
        torch.cuda.synchronize()
        plan = Plan(p, world=world, rank=rank, unique_id=uid[0], op=args.op)
    sampler = ClockSampler(local)
    sampler.start()
    plan.ita_iterate(Y, mb, X=X, iters=args.warmup, **kw)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    plan.ita_iterate(Y, mb, X=X, iters=args.steps, check=False, **kw)
    e1.record(stream)
    torch.cuda.synchronize()
    plan.status()                              # non-finite iterate -> CssarError
    fallbacks_timed = plan.debug_fallbacks()
    ms = e0.elapsed_time(e1)
    clocks = sampler.stop()
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = n * args.steps / (ms * 1e-3)       # global samples (one scene over all ranks)
    it_s = args.steps / (ms * 1e-3)
    peak, peak_kind = peaks()

    # per-step breakdown (CUDA events on the launch stream inside the library)
    stages = None
    roof = None
    if not args.no_profile and not slab:
        kp = max(3, min(args.steps, 30))
        plan.ita_iterate(Y, mb, X=X, iters=kp, profile_stages=True, **kw)
        st_ms, it_meas = plan.stage_times()
        stages = {k: v / it_meas for k, v in st_ms.items()}
        dom = max((s for s in STAGES if s != "S6_select"), key=lambda s: stages[s])
        tb = BYTES_PER_SAMPLE[dom] * n
        achieved = tb / (stages[dom] * 1e-3) / 1e9
        traffic = None
        tf = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
        if os.path.exists(tf):
            traffic = json.load(open(tf)).get(dom)
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                "algorithmic_bytes_per_launch": tb, "avg_launch_ms": stages[dom]}

    iter_ach = ITER_BYTES_PER_SAMPLE * n * it_s / 1e9
    line = {
        "metric": METRIC,
        "value": value, "unit": "samples*it/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "it_per_s": it_s, "higher_is_better": True,
        "scaling": "weak" if world == 1 else "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.config}{'' if args.op == 'csa' else ' [RDA pair]'}: {p.n_az}x{p.n_rg} complex64, {cfg.scene} scene, {cfg.mask} mask "
                               f"{cfg.rate}, SNR {cfg.snr_db} dB, {cfg.thr} threshold, k = {cfg.k}, mu = {cfg.mu}",
                   "n_az": p.n_az, "n_rg": p.n_rg, "k": cfg.k, "l2": "inputs larger than L2 (512 MiB arrays)",
                   "parallelism": "single" if not slab else
                   f"slab{world} (azimuth-line row slabs; " + ("transposes fused into the sweeps as peer-memory "
                   "stores, sparse-X' S1" if args.peer_transpose else "NCCL all-to-all transposes") +
                   "; rank-reduced select" + ("; one-rank NCCL diagnostic)" if world == 1 else ")")},
        "roofline": roof,
        "iteration_roofline": {"bound": "hbm", "achieved": iter_ach, "peak": peak * world, "unit": "GB/s",
                               "frac": iter_ach / (peak * world), "bytes_per_sample": ITER_BYTES_PER_SAMPLE,
                               "note": "aggregate over ranks; excludes NVLink transpose bytes" if world > 1 else None},
        "stages_ms": stages,
        "gpu_launches": launches(args.steps, cfg.rule, slab, plan.debug_graph_info() if slab else 0,
                                 fallbacks_timed, args.peer_transpose),
        "select_fallbacks": plan.debug_fallbacks(),
        "clocks": clocks,
    }

    if not args.no_e2e:
        # end to end through the public API: pinned host Y + mask -> device -> full solve -> host X
        # (world > 1: every rank its row slabs, collective solve, time = max over ranks)
        Yh = Y.cpu().pin_memory()
        mbh = mb.cpu().pin_memory()
        Xh = torch.empty_like(Yh).pin_memory()
        iters = cfg.iters
        plan.solve_host(Yh, mbh, out_host=Xh, iters=iters, **kw)      # warm (graph capture for new X)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        plan.solve_host(Yh, mbh, out_host=Xh, iters=iters, **kw)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([dt], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        h2d = (Yh.numel() * 8 + mbh.numel() * 4) * world
        d2h = Xh.numel() * 8 * world
        line["e2e"] = {"value": n * iters / dt, "unit": "samples*it/s", "h2d_bytes_per_step": h2d / iters,
                       "d2h_bytes_per_step": d2h / iters, "solve_iters": iters,
                       "note": "one full reconstruction (config iteration count) per call; copies once per solve"}
    if not slab and not args.no_sparse_state and cfg.rule == "k":
        # NEXT-3 sparse-state schedule (CSSAR_FLAG_SPARSE_STATE) on the same workload: 72.125
        # algorithmic HBM B/sample instead of 96.125 (the dense b traffic of S1 and S5 removed)
        plan.ita_iterate(Y, mb, X=X, iters=max(3, args.warmup), sparse_state=True, **kw)
        ms_ss = timed_iters(plan, Y, mb, X, args.steps, sparse_state=True, **kw)
        st_ss = stage_profile(plan, Y, mb, X, 10, sparse_state=True, **kw)
        it_ss = args.steps / (ms_ss * 1e-3)
        line["sparse_state"] = {"ms_per_step": ms_ss / args.steps, "it_per_s": it_ss, "value": n * it_ss,
                                "unit": "samples*it/s", "bytes_per_sample": 72.125,
                                "iteration_achieved_GBps": 72.125 * n * it_ss / 1e9, "stages_ms": st_ss,
                                "note": "opt-in schedule; bitwise the dense schedule's results"}
    if not slab and not args.no_library and cfg.rule == "k" and cfg.thr == "soft":
        line["library_chain"] = library_chain(Y, mask, cfg.k, cfg.mu)
    del mask
    if not slab and not args.no_c4 and args.config == "c3":
        del Y, X
        torch.cuda.empty_cache()
        line["c4"] = measure_c4(args, peak, peak_kind)
    if rank == 0 and not slab and not args.no_cpu_baseline:
        # the oracle on the full c3 grid (one ITA iteration; ~10-30 s of host work)
        line["cpu_baseline"] = cpu_baseline(args.config, p.n_az, p.n_rg, 1)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        emit(line)
    return 0


if __name__ == "__main__":
    sys.exit(main())
