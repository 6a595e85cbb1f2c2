"""Host cost of one query through the public API, split by call: mpdp_stage
(validation, layout, staging, H2D enqueue), mpdp_run (kernel enqueue),
mpdp_fetch (wait + D2H + result), and the binding's marshalling.
Usage: python tools/host_split.py star-10 star-25"""
import os
import statistics
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
            ctx.mpdp_optimize(g)
        rows = []
        for _ in range(30):
            t0 = time.perf_counter()
            ga = mpdp.GraphArgs(g)
            t1 = time.perf_counter()
            ctx._check(ctx.L.mpdp_stage(ctx.h, ga.ref()))
            t2 = time.perf_counter()
            ctx._check(ctx.L.mpdp_run(ctx.h))
            t3 = time.perf_counter()
            rb = mpdp.ResultBuf(g.n)
            ctx._check(ctx.L.mpdp_fetch(ctx.h, rb.ref()))
            r = rb.to_result()
            t4 = time.perf_counter()
            t5 = time.perf_counter()
            r2 = ctx.mpdp_optimize(g)
            t6 = time.perf_counter()
            rows.append(((t1 - t0) * 1e6, (t2 - t1) * 1e6, (t3 - t2) * 1e6, (t4 - t3) * 1e6, r.time_ms * 1e3,
                         (t6 - t5) * 1e6))
        med = [statistics.median(x[i] for x in rows) for i in range(6)]
        print(f"{name:12s} marshal {med[0]:6.1f} us  stage {med[1]:6.1f} us  run {med[2]:6.1f} us  "
              f"fetch {med[3]:7.1f} us (device query {med[4]:7.1f} us)  mpdp_optimize wall {med[5]:7.1f} us")
