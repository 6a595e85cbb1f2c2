"""Per-level device time of the fused kernel.  Usage: python tools/level_times.py star-10 [...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workload as W  # noqa: E402
from paper_2202_13511_b200 import mpdp  # noqa: E402

with mpdp.Context(device=0, workspace_bytes=4 << 30) as ctx:
    for name in sys.argv[1:]:
        topo, n = name.rsplit("-", 1)
        g = W.generate(topo, int(n), 0)
        for _ in range(3):
            r = ctx.mpdp_optimize(g)
        print(f"{name}: total {r.time_ms:.3f} ms, levels sum {sum(r.level_ms):.3f} ms")
        for k in range(2, g.n + 1):
            print(f"   k={k:2d} {r.level_ms[k]*1e3:8.1f} us  csg {r.level_csg[k]:9d}  pairs {r.level_pairs[k]:10d}")
