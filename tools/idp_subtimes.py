"""Where IDP2's time goes at BASELINE config 5: every recorded inner
sub-problem re-timed alone (device time, L2 flushed), with its shape (hub
degree), csg count, pairs and the kernel that ran it (memo_kind).
Usage: python tools/idp_subtimes.py [n] [k] [seed]"""
import collections
import ctypes as C
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch  # noqa: E402
import workload as W  # noqa: E402
from paper_2202_13511_b200 import mpdp  # noqa: E402
from test_gpu_heuristics import subproblems  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 25
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 0
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
with mpdp.Context(device=0, workspace_bytes=4 << 30, flags=mpdp.FLAG_RECORD_SUBPROBLEMS) as rctx:
    rctx.mpdp_optimize(W.snowflake(n, seed), algo="IDP2_MPDP", k=k)
    subs = subproblems(rctx)
tot = collections.Counter()
with mpdp.Context(device=0, workspace_bytes=4 << 30) as ctx:
    for i, (q, _) in enumerate(subs):
        for _ in range(2):
            ctx.mpdp_optimize(q)
        ts = []
        for _ in range(5):
            ctx.mpdp_stage(q)
            flush.fill_(1)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ctx.stream)
            ctx.mpdp_run()
            e1.record(ctx.stream)
            r = ctx.mpdp_fetch()
            ts.append(e0.elapsed_time(e1))
        deg = collections.Counter()
        for u, v in q.edges:
            deg[u] += 1
            deg[v] += 1
        hub = max(deg.values()) if deg else 0
        ms = statistics.median(ts)
        tot[r.memo_kind] += ms
        print(f"{i:3d} n={q.n:2d} hubdeg={hub:2d} csg={r.csg_count:9d} pairs={r.pairs_evaluated:10d} "
              f"memo_kind={r.memo_kind} {ms:7.3f} ms  {r.pairs_evaluated / ms / 1e6:7.1f} G pairs/s", flush=True)
print("device ms by memo_kind:", dict(tot), "total", sum(tot.values()))
