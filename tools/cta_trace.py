"""Per-level, per-CTA phase times of the fused kernel (needs a -DMPDP_TRACE
build via MPDP_LIBRARY): enumeration, queueing and evaluation time summed over
the CTA's tiles, and the barrier arrival spread.
Usage: MPDP_LIBRARY=tools/dbg/libmpdp_trace.so python tools/cta_trace.py star-25"""
import ctypes as C
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workload as W  # noqa: E402
from paper_2202_13511_b200 import mpdp  # noqa: E402

L = mpdp.load_library()
L.mpdp_debug_cta_trace.restype = C.c_int
L.mpdp_debug_cta_trace.argtypes = [C.POINTER(C.c_uint64), C.c_int]
L.mpdp_debug_cta_trace_clear.restype = None
NMAX, CMAX, SL = 57, 1024, 8
with mpdp.Context(device=0, workspace_bytes=6 << 30) as ctx:
    for name in sys.argv[1:]:
        topo, n = name.rsplit("-", 1)
        g = W.generate(topo, int(n), 0)
        for _ in range(2):
            ctx.mpdp_optimize(g)
        L.mpdp_debug_cta_trace_clear()
        r = ctx.mpdp_optimize(g)
        buf = (C.c_uint64 * (NMAX * CMAX * SL))()
        assert L.mpdp_debug_cta_trace(buf, NMAX * CMAX * SL) == CMAX
        print(f"{name}: {r.time_ms:.3f} ms")
        print("   k  level_us  spread_us  idle   busy_ctas  slowest: tiles enum_us queue_us eval_us   median busy: tiles enum queue eval   small: sets max_us")
        prev, idle_tot = None, 0.0
        for k in range(2, g.n + 1):
            rec = []
            for b in range(CMAX):
                o = (k * CMAX + b) * SL
                if buf[o + 5]:
                    rec.append((buf[o + 5], b, buf[o], buf[o + 1] / 1e3, buf[o + 2] / 1e3, buf[o + 3] / 1e3, buf[o + 4],
                                buf[o + 6] / 1e3, buf[o + 7]))
            if not rec:
                continue
            arr = [x[0] for x in rec]
            t0 = min(x[2] for x in rec) if prev is None else prev
            mx = max(rec)
            busy = [x for x in rec if x[6] > 0]
            idle = sum(mx[0] - a for a in arr) / len(arr)
            idle_tot += idle
            med = sorted(busy, key=lambda x: x[5])[len(busy) // 2] if busy else None
            ms = f"{med[6]:5d} {med[3]:5.1f} {med[4]:5.1f} {med[5]:6.1f}" if med else ""
            print(f"  {k:2d} {(mx[0] - t0) / 1e3:9.1f} {(mx[0] - min(arr)) / 1e3:10.1f} {idle / 1e3:6.1f} {len(busy):9d}"
                  f"   cta {mx[1]:4d}: {mx[6]:3d} {mx[3]:7.1f} {mx[4]:8.1f} {mx[5]:7.1f}   {ms:28s}"
                  f"   {rec[0][8]:7d} {max(x[7] for x in rec):6.1f}")
            prev = mx[0]
        print(f"  mean CTA idle at barriers: {idle_tot / 1e3:.1f} us")
