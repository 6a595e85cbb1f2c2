"""Device time of star queries through the fused peer exchange, W ranks
emulated on one GPU (CTA groups of one launch), vs the single-GPU kernel.
Usage: python tools/xr_time.py star-25 [--reps 10]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import workload as W  # noqa: E402
from paper_2202_13511_b200 import mpdp  # noqa: E402

args = sys.argv[1:]
reps = 10
if "--reps" in args:
    i = args.index("--reps"); reps = int(args[i + 1]); del args[i:i + 2]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name in args or ["star-25", "clique-18"]:
    topo, n = name.rsplit("-", 1)
    g = W.generate(topo, int(n), 0)
    for world in (1, 2, 4, 8):
        flags = 0 if world == 1 else mpdp.FLAG_SIMULATE_WORLD | mpdp.FLAG_FUSED_EXCHANGE
        with mpdp.Context(device=0, workspace_bytes=(8 << 30), world=world, flags=flags) as ctx:
            r0 = ctx.mpdp_optimize(g)
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
            assert r.cost == r0.cost and r.tree() == r0.tree()
            print(f"{name:10s} ranks {world}: {statistics.median(ts):8.3f} ms  (min {min(ts):.3f})  "
                  f"pairs {r.pairs_evaluated}  launches {r.gpu_launches}", flush=True)
