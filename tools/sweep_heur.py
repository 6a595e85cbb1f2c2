"""IDP2 / UnionDP on the GPU vs the same drivers with the oracle as the inner
solver (mpdp_heuristic_optimize) on seeded mid-size queries: plans must be
identical.  python tools/sweep_heur.py"""
import ctypes as C, os, sys, random
sys.setrecursionlimit(100000)
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import workload as W
from paper_2202_13511_b200 import mpdp
from test_heuristics_cpu import run as cpu_run
rng = random.Random(5)
bad = 0
with mpdp.Context(device=0, workspace_bytes=4 << 30) as ctx:
    for i in range(12):
        n, k = rng.randint(60, 400), rng.choice([6, 8, 10, 12, 16])
        topo = rng.choice(["snowflake", "snowflake", "star", "chain"])
        g = W.generate(topo, n, 700 + i)
        for algo in ("IDP2_MPDP", "UNIONDP_MPDP"):
            r = ctx.mpdp_optimize(g, algo=algo, k=k)
            o, _ = cpu_run(g, algo, k)
            same = r.cost == o.cost and r.tree() == o.tree()
            if not same:
                bad += 1
            print(g.name, algo, k, "same" if same else "DIFF", r.cost, o.cost, flush=True)
print("heuristic sweep mismatches:", bad)
