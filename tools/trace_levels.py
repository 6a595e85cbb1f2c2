"""Phase trace of block 0 of the fused kernel (needs a -DMPDP_TRACE build via
MPDP_LIBRARY).  Usage: MPDP_LIBRARY=tools/dbg/libmpdp_trace.so python tools/trace_levels.py star-10"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workload as W  # noqa: E402
from paper_2202_13511_b200 import mpdp  # noqa: E402

PH = ["start", "ticket", "enum", "queued", "evald", "counted", "barrier", "heavy"]  # (k_dp_small: start, enum, -, listed, evald)
L = mpdp.load_library()
L.mpdp_debug_trace.restype = C.c_int
L.mpdp_debug_trace.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.c_int]
with mpdp.Context(device=0, workspace_bytes=4 << 30, flags=int(os.environ.get("MPDP_FLAGS", "0"))) as ctx:
    for name in sys.argv[1:]:
        topo, n = name.rsplit("-", 1)
        g = W.generate(topo, int(n), 0)
        for _ in range(3):
            r = ctx.mpdp_optimize(g)
        buf = (C.c_uint64 * 512)()
        m = L.mpdp_debug_trace(ctx.h, buf, 512)
        print(f"{name}: {r.time_ms:.3f} ms, {m} trace points")
        prev = None
        line = []
        for x in buf[:m]:
            t, k, ph = x >> 8, (x >> 3) & 31, x & 7
            if ph == 0 and line:
                print("  " + " ".join(line))
                line = []
            line.append(f"k{k}:{PH[ph]}+{0 if prev is None else (t - prev) / 1000:.2f}")
            prev = t
        print("  " + " ".join(line))
