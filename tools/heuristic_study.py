"""plan quality of the heuristics under C_out (P:1103-1140 Tables
1-2, the k-sweep of P:1231) on the GPU: GOO (IDP2 with k = 2, nothing
re-optimised), IDP2 (k = 5..25) and UnionDP (k = 25 with partition threshold
t = 15 or 25) on 100 seeded snowflake and star queries of 30-1000 relations
(the workload generator, PK-FK selectivities).  Cost is normalised to
the best plan any of them found for the query; reported as geometric means,
wins and mean optimisation time per (topology, n).  Relative ordering only:
the paper's numbers come from a PostgreSQL-like cost model and real data.

A second part repeats GOO / IDP2(25) / UnionDP on queries whose selectivities
are NOT PK-FK (cards log-uniform in [1, 100], a plain predicate factor
10^U(-2,0) per edge) and on 22-relation snowflakes against the exact optimum
(oracle), as evidence for why UnionDP trails under PK-FK + C_out.

Usage (GPU box): python tools/heuristic_study.py > profiles/r02_heuristic_quality.txt"""
import math
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workload as W  # noqa: E402
from paper_2202_13511_b200 import mpdp  # noqa: E402

ALGOS = [("GOO", "IDP2_MPDP", 2, 0)] + [(f"IDP2({k})", "IDP2_MPDP", k, 0) for k in (5, 10, 15, 20, 25)] + \
        [("UnionDP(25,t=15)", "UNIONDP_MPDP", 25, 15), ("UnionDP(25,t=25)", "UNIONDP_MPDP", 25, 25)]


def run(ctx, g, algo, k, t):
    t0 = time.perf_counter()
    r = ctx.mpdp_optimize_uniondp(g, k=k, t=t) if algo == "UNIONDP_MPDP" else ctx.mpdp_optimize(g, algo=algo, k=k)
    return r.cost, time.perf_counter() - t0


def plain(g, seed):
    """Same topology, NOT PK-FK: cardinalities log-uniform in [1, 100] and a
    plain predicate factor 10^U(-2,0) per edge, independent of the endpoints
    (with the generator's cards the final join's card(V) ~ 10^(2.5 n) would
    dominate every plan's C_out and all plans would tie)."""
    rng = np.random.default_rng(10_000 + seed)
    return W.QueryGraph(g.n, [float(10 ** rng.uniform(0, 2)) for _ in range(g.n)], list(g.edges),
                        [float(10 ** rng.uniform(-2, 0)) for _ in g.edges], name=g.name + "-plain")


def table(ctx, groups, algos, label):
    print(f"\n== {label}")
    print("   (normalised cost = cost / best cost found by any listed algorithm for the query; geo = geometric "
          "mean over the queries, max = worst query, wins = queries where it found the best plan)")
    for (topo, n), gs in groups:
        rows = {name: ([], [], 0) for name, *_ in algos}
        for g in gs:
            res = {name: run(ctx, g, a, k, t) for name, a, k, t in algos}
            best = min(c for c, _ in res.values())
            for name in res:
                c, dt = res[name]
                norm, times, wins = rows[name]
                norm.append(c / best if best > 0 else 1.0)
                times.append(dt)
                rows[name] = (norm, times, wins + (c == best))
        print(f"-- {topo}, n = {n}, {len(gs)} queries")
        for name, (norm, times, wins) in rows.items():
            geo = math.exp(statistics.mean(math.log(x) for x in norm))
            print(f"   {name:18s} geo {geo:12.4g}  max {max(norm):12.4g}  wins {wins:3d}/{len(gs)}  "
                  f"time {1e3 * statistics.mean(times):8.2f} ms")
        sys.stdout.flush()


def main():
    only_evidence = "--evidence" in sys.argv
    with mpdp.Context(device=0, workspace_bytes=6 << 30) as ctx:
        # part 1: 100 PK-FK queries (snowflake 52, star 48)
        groups = []
        for topo, sizes, seeds in (("snowflake", (30, 100, 300, 1000), 13), ("star", (30, 100, 300, 1000), 12)):
            for n in sizes:
                groups.append(((topo, n), [W.generate(topo, n, s) for s in range(seeds)]))
        assert sum(len(gs) for _, gs in groups) == 100
        if not only_evidence:
            table(ctx, groups, ALGOS, "PK-FK selectivities (workload generator), 100 queries")
        # part 2: evidence -- plain predicate factors instead of PK-FK
        sub = [a for a in ALGOS if a[0] in ("GOO", "IDP2(10)", "IDP2(25)", "UnionDP(25,t=15)", "UnionDP(25,t=25)")]
        g2 = [(("snowflake", n), [plain(W.generate("snowflake", n, s), s) for s in range(10)]) for n in (30, 100, 300)]
        table(ctx, g2, sub, "not PK-FK: cards 10^U(0,2), plain predicate factors 10^U(-2,0), snowflakes, 30 queries")
        # part 3: against the exact optimum (22 relations, oracle = exact MPDP on the GPU here)
        print("\n== 22-relation snowflakes against the exact optimum (MPDP), cost / optimum")
        small = [("GOO", "IDP2_MPDP", 2, 0), ("IDP2(8)", "IDP2_MPDP", 8, 0), ("UnionDP(8,t=8)", "UNIONDP_MPDP", 8, 8)]
        for model in ("pkfk", "plain"):
            ratios = {name: [] for name, *_ in small}
            for s in range(10):
                g = W.generate("snowflake", 22, s)
                if model == "plain":
                    g = plain(g, s)
                opt = ctx.mpdp_optimize(g).cost
                for name, a, k, t in small:
                    ratios[name].append(run(ctx, g, a, k, t)[0] / opt)
            print(f"-- {model}: " + "  ".join(
                f"{name} geo {math.exp(statistics.mean(math.log(x) for x in v)):.4g} max {max(v):.4g}"
                for name, v in ratios.items()))


if __name__ == "__main__":
    main()
