"""Randomised parity sweep across contexts with different flags (hash memo, rank
memo, per-level kernels, no single-CTA / star kernels, no CCC, simulated 2-rank
world) interleaved in one process, plus batches.  python tools/sweep_flags.py"""
import os, sys, random
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import workload as W
from oracle import pyoracle as O
from paper_2202_13511_b200 import mpdp
from test_gpu_parity import check
rng = random.Random(11)
F = mpdp
ctxs = [mpdp.Context(device=0, workspace_bytes=2 << 30, flags=f) for f in
        (0, F.FLAG_HASH_MEMO, F.FLAG_RANK_MEMO, F.FLAG_NO_FUSED, F.FLAG_NO_SMALL | F.FLAG_NO_STAR, F.FLAG_NO_CCC)]
ctxs.append(mpdp.Context(device=0, workspace_bytes=2 << 30, world=2, flags=F.FLAG_SIMULATE_WORLD))
ctxs.append(mpdp.Context(device=0, workspace_bytes=2 << 30, world=3,
                         flags=F.FLAG_SIMULATE_WORLD | F.FLAG_FUSED_EXCHANGE))   # fused peer exchange
bad = 0
batch = []
for i in range(200):
    topo = rng.choice(["star", "snowflake", "chain", "cycle", "clique", "random"])
    hi = {"clique": 14, "random": 14, "cycle": 16, "star": 20, "snowflake": 20, "chain": 22}[topo]
    g = W.generate(topo, rng.randint(2 if topo in ("star", "chain", "snowflake") else 3, hi), 9000 + i)
    o = O.optimize(g)
    c = rng.choice(ctxs)
    try:
        check(c.mpdp_optimize(g), o, g)
    except Exception as e:
        bad += 1
        print("MISMATCH", g.name, ctxs.index(c), e)
    batch.append((g, o))
    if len(batch) == 16:
        try:
            for (g2, o2), r in zip(batch, ctxs[0].mpdp_optimize_batch([b[0] for b in batch])):
                check(r, o2, g2)
        except Exception as e:
            bad += 1
            print("BATCH MISMATCH", e)
        batch = []
print("flag sweep done, mismatches:", bad)
