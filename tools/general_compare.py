"""General graphs: device time of MPDP vs the DPSUB-enumeration ablation, with
connectivity by memo probes (reading R20, default) or by BFS
(MPDP_DEBUG_BFS_CONN=1).  Usage: python tools/general_compare.py random-18 random-20 [--reps 5]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import workload as W  # noqa: E402
from paper_2202_13511_b200 import mpdp  # noqa: E402

args = sys.argv[1:]
reps = 5
if "--reps" in args:
    i = args.index("--reps"); reps = int(args[i + 1]); del args[i:i + 2]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ctxs = {"mpdp": mpdp.Context(device=0, workspace_bytes=8 << 30),
        "dpsub": mpdp.Context(device=0, workspace_bytes=8 << 30, flags=mpdp.FLAG_DPSUB_ENUM)}
print(f"{'config':12s} {'variant':6s} {'conn':4s} {'ms':>9s} {'pairs':>12s} {'ccp':>11s} {'Gpairs/s':>9s}")
for name in args:
    topo, n = name.rsplit("-", 1)
    g = W.generate(topo, int(n), 0)
    for conn in ("memo", "bfs"):
        if conn == "bfs":
            os.environ["MPDP_DEBUG_BFS_CONN"] = "1"
        else:
            os.environ.pop("MPDP_DEBUG_BFS_CONN", None)
        for var, ctx in ctxs.items():
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
            print(f"{name:12s} {var:6s} {conn:4s} {ms:9.3f} {r.pairs_evaluated:12d} {r.ccp_pairs:11d} "
                  f"{r.pairs_evaluated / ms / 1e6:9.2f}  cost={r.cost!r}", flush=True)
os.environ.pop("MPDP_DEBUG_BFS_CONN", None)
