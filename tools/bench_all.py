"""Device-time breakdown of every BASELINE config (CUDA events, warm, L2 flushed
between queries).  Usage: python tools/bench_all.py [reps] [--hash]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import workload as W  # noqa: E402
from paper_2202_13511_b200 import mpdp  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 10
base = mpdp.FLAG_HASH_MEMO if "--hash" in sys.argv else 0
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
configs = ["star-10", "snowflake-20", "star-25", "clique-18", "chain-25", "cycle-20", "random-20"]
ctx = mpdp.Context(device=0, workspace_bytes=8 << 30, flags=base)                     # graph replay
pctx = mpdp.Context(device=0, workspace_bytes=8 << 30, flags=base | mpdp.FLAG_PROFILE_KERNELS)
if True:
    print(f"{'config':14s} {'ms':>8s} {'direct':>8s} {'enum':>8s} {'eval':>8s} {'pairs':>12s} {'Gpairs/s':>9s} launches")
    for name in configs:
        topo, n = name.rsplit("-", 1)
        g = W.generate(topo, int(n), 0)
        for _ in range(3):
            ctx.mpdp_optimize(g)
        ts, te, tv, td = [], [], [], []
        for _ in range(3):
            pctx.mpdp_optimize(g)
        for _ in range(reps):
            flush.fill_(1)
            torch.cuda.synchronize()
            r = pctx.mpdp_optimize(g)
            te.append(r.enum_ms)
            tv.append(r.eval_ms)
            td.append(r.time_ms)
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
        print(f"{name:14s} {ms:8.3f} {statistics.median(td):8.3f} {statistics.median(te):8.3f} {statistics.median(tv):8.3f} "
              f"{r.pairs_evaluated:12d} {r.pairs_evaluated / ms / 1e6:9.2f} {r.gpu_launches}")
