"""Randomised parity sweep (300 seeded graphs of every topology, plus a simulated
3-rank sharded context every 5th graph) against the oracle.  Run on a GPU box:
python tools/sweep_big.py"""
import os, sys, random
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import workload as W
from oracle import pyoracle as O
from paper_2202_13511_b200 import mpdp
from test_gpu_parity import check
rng = random.Random(7)
bad = 0
with mpdp.Context(device=0, workspace_bytes=4 << 30) as ctx, \
     mpdp.Context(device=0, workspace_bytes=2 << 30, world=3, flags=mpdp.FLAG_SIMULATE_WORLD | mpdp.FLAG_SHARD_ALL_LEVELS) as sh:
    for i in range(300):
        topo = rng.choice(["star", "snowflake", "chain", "cycle", "clique", "random"])
        hi = {"clique": 15, "random": 15, "cycle": 18, "star": 21, "snowflake": 22, "chain": 24}[topo]
        g = W.generate(topo, rng.randint(2 if topo in ("star", "chain", "snowflake") else 3, hi), 5000 + i)
        if rng.random() < 0.3:
            g.leaf_cost = [float(rng.choice([0, 1, 7, 1000])) for _ in range(g.n)]
        o = O.optimize(g)
        print("case", i, g.name, g.n, len(g.edges), flush=True)
        try:
            check(ctx.mpdp_optimize(g), o, g)
            if i % 5 == 0:
                check(sh.mpdp_optimize(g), o, g)
        except Exception as e:
            bad += 1
            print("MISMATCH", g.name, g.n, e)
print("sweep done, mismatches:", bad)
