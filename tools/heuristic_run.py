"""BASELINE config 5: IDP2 / UnionDP with the GPU MPDP inner DP on 1000-relation
snowflakes.  Usage: python tools/heuristic_run.py [n] [k] [seeds] [--verify]"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workload as W  # noqa: E402
from paper_2202_13511_b200 import mpdp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 25
seeds = int(sys.argv[3]) if len(sys.argv) > 3 else 1
verify = "--verify" in sys.argv
L = mpdp.load_library()
with mpdp.Context(device=0, workspace_bytes=4 << 30, flags=mpdp.FLAG_RECORD_SUBPROBLEMS) as ctx:
    for seed in range(seeds):
        g = W.snowflake(n, seed)
        goo = ctx.mpdp_optimize(g, algo="IDP2_MPDP", k=2)
        for algo, t_part in (("IDP2_MPDP", 0), ("UNIONDP_MPDP", 0), ("UNIONDP_MPDP", 15)):
            run = (lambda: ctx.mpdp_optimize(g, algo=algo, k=k)) if t_part == 0 else \
                (lambda: ctx.mpdp_optimize_uniondp(g, k=k, t=t_part))
            run()                                        # warm
            t = time.perf_counter()
            r = run()
            dt = time.perf_counter() - t
            nsub = L.mpdp_subproblem_count(ctx.h)
            sizes = []
            for i in range(nsub):
                sg = mpdp.mpdp_query_graph()
                L.mpdp_subproblem_get(ctx.h, i, C.byref(sg), None)
                sizes.append(sg.n)
            print(f"seed {seed} {algo:13s} n={n} k={k} t={t_part or k}: {dt*1e3:8.1f} ms, cost {r.cost:.6g} "
                  f"(GOO {goo.cost:.6g}, ratio {r.cost/goo.cost if goo.cost else float('nan'):.4f}), "
                  f"inner calls {r.inner_calls}, max sub n {max(sizes)}, pairs {r.pairs_evaluated}", flush=True)
