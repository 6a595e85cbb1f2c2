"""Dataflow kernel timing breakdown per CTA (MPDP_DEBUG_DF_STATS).
Usage: MPDP_DEBUG_DF_STATS=1 python tools/df_stats.py star-25 clique-18"""
import ctypes as C
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MPDP_DEBUG_DF_STATS", "1")
import workload as W  # noqa: E402
from paper_2202_13511_b200 import mpdp  # noqa: E402

ctx = mpdp.Context(device=0, workspace_bytes=8 << 30)
for name in sys.argv[1:]:
    topo, n = name.rsplit("-", 1)
    g = W.generate(topo, int(n), 0)
    for _ in range(3):
        r = ctx.mpdp_optimize(g)
    buf = (C.c_uint64 * (8 * 2048))()
    nw = ctx.L.mpdp_debug_df_stats(ctx.h, buf, 8 * 2048)
    rows = [buf[i:i + 8] for i in range(0, nw, 8) if buf[i + 2]]
    col = lambda j: [x[j] / 1e3 for x in rows]   # noqa: E731
    print(f"{name}: {len(rows)} CTAs, kernel {r.eval_ms:.3f} ms")
    for j, nm in enumerate(["ctl wait slot us", "ctl wait dep us", "ctl loop us", "chunks (x1e3)",
                            "warp0 wait take us", "warp0 loop us"]):
        v = col(j)
        print(f"   {nm:22s} mean {statistics.mean(v):9.2f}  min {min(v):9.2f}  max {max(v):9.2f}")
