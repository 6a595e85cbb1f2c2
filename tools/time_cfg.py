"""Median device time (CUDA events around mpdp_run, L2 flushed) of named configs,
optionally under environment overrides.  Usage:
  python tools/time_cfg.py star-25 clique-18 [--env MPDP_DEBUG_STAR_RUN=2,4,8] [--reps 20]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import workload as W  # noqa: E402
from paper_2202_13511_b200 import mpdp  # noqa: E402

args = sys.argv[1:]
reps, env, seeds = 20, None, [0]
if "--reps" in args:
    i = args.index("--reps"); reps = int(args[i + 1]); del args[i:i + 2]
if "--seeds" in args:
    i = args.index("--seeds"); seeds = list(range(int(args[i + 1]))); del args[i:i + 2]
if "--env" in args:
    i = args.index("--env"); env = args[i + 1]; del args[i:i + 2]
variants = [None]
if env:
    k, vs = env.split("=")
    variants = [(k, v) for v in vs.split(",")]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ctx = mpdp.Context(device=0, workspace_bytes=8 << 30)
for name, seed in [(a, sd) for a in args for sd in seeds]:
    topo, n = name.rsplit("-", 1)
    g = W.generate(topo, int(n), seed)
    for var in variants:
        if var:
            os.environ[var[0]] = var[1]
        for _ in range(3):
            ctx.mpdp_optimize(g)
        ts = []
        for _ in range(reps):
            ctx.mpdp_stage(g)
            flush.fill_(1)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ctx.stream)
            ctx.mpdp_run()
            e1.record(ctx.stream)
            r = ctx.mpdp_fetch()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        import ctypes as C
        st, dn = (C.c_double * 64)(), (C.c_double * 64)()
        nn = ctx.L.mpdp_debug_level_span(ctx.h, st, dn, 64)
        lv = f"init {dn[0]:.0f} start {st[0]:.0f} " + " ".join(f"{k}:{st[k]:.0f}-{dn[k]:.0f}" for k in range(2, nn))
        print(f"{name:12s} s{seed} {str(var or ''):26s} {ms:8.4f} ms kernel(ev) {r.eval_ms:.4f}  min {min(ts):.4f}  {r.pairs_evaluated / ms / 1e6:8.2f} Gpairs/s"
              f"  levels(us): {lv}", flush=True)
        if var:
            del os.environ[var[0]]
