"""Run W warm-up queries then one query of a workload (for ncu launch lists /
captures).  Usage: python tools/profile_one.py star-25 [warmup]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workload as W  # noqa: E402
from paper_2202_13511_b200 import mpdp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "star-25"
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 1
topo, n = name.rsplit("-", 1)
g = W.generate(topo, int(n), 0)
with mpdp.Context(device=0, workspace_bytes=6 << 30) as ctx:
    for _ in range(warm):
        ctx.mpdp_optimize(g)
    r = ctx.mpdp_optimize(g)
    print(name, "cost", r.cost, "pairs", r.pairs_evaluated, "probes", r.probes, "ms", r.time_ms,
          "launches", r.gpu_launches, file=sys.stderr)
