"""Enhancement ablations on one B200, device time per query
(CUDA events via time_ms, warm, median of reps):
  * MPDP (whole-query kernel)          -- the product path
  * per-level kernels (MPDP_FLAG_NO_FUSED): separate enumerate / evaluate /
    extract launches per level (the paper's phase structure)
  * DPSUB enumeration (MPDP_FLAG_DPSUB_ENUM): every connected set evaluates all
    2^(|S|-1)-1 splits with CCP checks (Alg. generic_dpsub)
  * no-ccc (MPDP_FLAG_NO_CCC): no Collaborative Context Collection
  * rank-memo (MPDP_FLAG_RANK_MEMO): colex-rank memo instead of the bitmask one
    on cliques / general graphs
  * no-small (MPDP_FLAG_NO_SMALL): small / thin tree queries on the multi-CTA
    list kernel instead of the single-CTA kernels
  * no-star (MPDP_FLAG_NO_STAR): star queries on the general tree kernel
Usage: python tools/ablation.py [reps] [config ...]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workload as W  # noqa: E402
from paper_2202_13511_b200 import mpdp  # noqa: E402

args = [a for a in sys.argv[1:]]
reps = int(args.pop(0)) if args and args[0].isdigit() else 5
configs = args or ["star-10", "star-20", "star-25", "snowflake-20", "chain-25", "clique-14", "clique-18", "cycle-16",
                   "random-18"]
modes = [("mpdp", 0), ("per-level", mpdp.FLAG_NO_FUSED), ("dpsub", mpdp.FLAG_DPSUB_ENUM),
         ("no-ccc", mpdp.FLAG_NO_CCC), ("rank-memo", mpdp.FLAG_RANK_MEMO), ("no-small", mpdp.FLAG_NO_SMALL),
         ("no-star", mpdp.FLAG_NO_STAR)]
ctxs = {m: mpdp.Context(device=0, workspace_bytes=8 << 30, flags=f) for m, f in modes}
print(f"{'config':13s} {'mode':10s} {'ms':>10s} {'pairs_evaluated':>16s} {'ccp_pairs':>12s} {'pairs/ccp':>10s} {'time/mpdp':>9s}")
for name in configs:
    topo, n = name.rsplit("-", 1)
    g = W.generate(topo, int(n), 0)
    base = None
    for m, _ in modes:
        c = ctxs[m]
        r = c.mpdp_optimize(g)
        ts = []
        for _ in range(reps if m != "dpsub" else max(1, reps // 5)):
            ts.append(c.mpdp_optimize(g).time_ms)
        ms = statistics.median(ts)
        base = base or ms
        print(f"{name:13s} {m:10s} {ms:10.3f} {r.pairs_evaluated:16d} {r.ccp_pairs:12d} "
              f"{r.pairs_evaluated / max(1, r.ccp_pairs):10.2f} {ms / base:9.2f}", flush=True)
