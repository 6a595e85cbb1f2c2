"""Fixed per-query cost outside the level loop.  Usage: python tools/overhead.py star-10 clique-14 ...
Prints: events around the whole query (k_init + kernel + result D2H), the
whole-query kernel alone, the sum of its level phases, and host wall time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workload as W  # noqa: E402
from paper_2202_13511_b200 import mpdp  # noqa: E402

with mpdp.Context(device=0, workspace_bytes=4 << 30) as ctx:
    for name in sys.argv[1:]:
        topo, n = name.rsplit("-", 1)
        g = W.generate(topo, int(n), 0)
        for _ in range(5):
            r = ctx.mpdp_optimize(g)
        rows = []
        for _ in range(10):
            t = time.perf_counter()
            r = ctx.mpdp_optimize(g)
            wall = (time.perf_counter() - t) * 1e3
            rows.append((r.time_ms, r.eval_ms, sum(r.level_ms), wall))
        rows.sort()
        q, kern, lv, wall = rows[len(rows) // 2]
        print(f"{name:14s} query {q*1e3:8.1f} us  kernel {kern*1e3:8.1f} us  levels {lv*1e3:8.1f} us  "
              f"outside-levels {(kern-lv)*1e3:6.1f} us  outside-kernel {(q-kern)*1e3:6.1f} us  host wall {wall*1e3:8.1f} us")
