"""IDP2 / UnionDP driver logic on CPU: the exported
mpdp_heuristic_optimize with the ORACLE plugged in as the inner exact solver
(test-only; the product path mpdp_optimize always uses the GPU MPDP).

Checks: n <= k reduces to the exact optimum; plans are valid cross-product-free
trees over every relation exactly once; the reported cost equals the cost
recomputed with the documented recurrence; inner sub-problems respect the
bound k and are connected; IDP2 never ends above its GOO start (k = 2 is GOO);
UnionDP / IDP2 finish 1000-relation snowflakes (BASELINE config 5 shape).
"""
import ctypes as C

import pytest

from oracle import pyoracle as O
import workload as W

REL = 1e-9


def _lib():
    from paper_2202_13511_b200 import build, mpdp
    build.build()
    L = mpdp.load_library()
    return L, mpdp


SOLVER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p)


class Oracle:
    """Inner solver callback: decode the sub-problem, solve with the oracle."""

    def __init__(self, mpdp, k):
        self.mpdp = mpdp
        self.k = k
        self.subs = []
        self.cb = SOLVER(self._solve)

    def _solve(self, user, gp, rp):
        mp = self.mpdp
        g = C.cast(gp, C.POINTER(mp.mpdp_query_graph)).contents
        r = C.cast(rp, C.POINTER(mp.mpdp_result)).contents
        n, m = g.n, g.n_edges
        edges = [(g.edges[2 * i], g.edges[2 * i + 1]) for i in range(m)]
        q = W.QueryGraph(n, [g.cardinalities[i] for i in range(n)], edges, [g.selectivities[i] for i in range(m)],
                         leaf_cost=[g.leaf_costs[i] for i in range(n)] if g.leaf_costs else None)
        self.subs.append(q)
        o = O.optimize(q)
        for i, nd in enumerate(o.nodes):
            x = r.nodes[i]
            x.left, x.right, x.relation, x.set = nd.left, nd.right, nd.relation, nd.set
            x.cardinality, x.cost = nd.card, nd.cost
        r.n_nodes = len(o.nodes)
        r.cost = o.cost
        r.pairs_evaluated, r.ccp_pairs, r.csg_count = o.pairs_evaluated, o.ccp_pairs, o.csg_count
        return 0


def run(g, algo, k):
    L, mp = _lib()
    L.mpdp_heuristic_optimize.restype = C.c_int
    L.mpdp_heuristic_optimize.argtypes = [C.POINTER(mp.mpdp_query_graph), C.c_int, C.c_uint32, SOLVER,
                                          C.c_void_p, C.POINTER(mp.mpdp_result)]
    solver = Oracle(mp, k)
    ga, rb = mp.GraphArgs(g), mp.ResultBuf(g.n)
    st = L.mpdp_heuristic_optimize(ga.ref(), mp.ALGOS[algo], k, solver.cb, None, rb.ref())
    assert st == 0, L.mpdp_last_error(None)
    return rb.to_result(), solver.subs


def recompute(g, res):
    """Cost of the returned tree by the documented recurrence; validates the tree."""
    nodes = res.nodes
    adj = {}
    for i, (u, v) in enumerate(g.edges):
        adj.setdefault(u, []).append((v, i))
        adj.setdefault(v, []).append((u, i))
    rels, card, cost = {}, {}, {}
    for i, nd in enumerate(nodes):
        if nd.relation >= 0:
            rels[i] = {nd.relation}
            card[i] = g.card[nd.relation]
            cost[i] = g.leaf_cost[nd.relation] if g.leaf_cost else 0.0
            continue
        assert nd.left < i and nd.right < i
        Lr, Rr = rels[nd.left], rels[nd.right]
        assert not (Lr & Rr)
        cross = sorted(e for r in Lr for (u, e) in adj.get(r, []) if u in Rr)
        assert cross, "cross product"
        c = card[nd.left] * card[nd.right]
        for e in cross:
            c = c * g.sel[e]
        rels[i] = Lr | Rr
        card[i] = c
        cost[i] = (cost[nd.left] + cost[nd.right]) + c
        assert nd.cost == cost[i] and nd.cardinality == c
    root = len(nodes) - 1
    assert rels[root] == set(range(g.n)) and len(nodes) == 2 * g.n - 1
    assert sum(1 for nd in nodes if nd.relation >= 0) == g.n
    return cost[root]


@pytest.mark.parametrize("algo", ["IDP2_MPDP", "UNIONDP_MPDP"])
@pytest.mark.parametrize("topo,n", [("snowflake", 9), ("star", 8), ("random", 10), ("clique", 7)])
def test_small_query_is_exact(algo, topo, n):
    """n <= k: one inner DP over everything = the exact optimum (Alg. uniondp lines 1-4)."""
    g = W.generate(topo, n, 3)
    res, subs = run(g, algo, 12)
    o = O.optimize(g)
    assert abs(res.cost - o.cost) <= REL * o.cost
    assert recompute(g, res) == res.cost


@pytest.mark.parametrize("algo", ["IDP2_MPDP", "UNIONDP_MPDP"])
@pytest.mark.parametrize("topo,n,k,seed", [("snowflake", 30, 8, 0), ("snowflake", 40, 10, 1),
                                           ("star", 30, 8, 2), ("random", 24, 6, 3), ("chain", 40, 7, 4)])
def test_plans_valid_and_bounded(algo, topo, n, k, seed):
    g = W.generate(topo, n, seed)
    res, subs = run(g, algo, k)
    assert recompute(g, res) == res.cost
    assert res.inner_calls == len(subs) >= 1
    for q in subs:
        assert 2 <= q.n <= k
        assert O.connected(q, (1 << q.n) - 1)
    assert res.pairs_evaluated == sum(O.optimize(q).pairs_evaluated for q in subs)


@pytest.mark.parametrize("seed", range(4))
def test_idp2_improves_on_goo(seed):
    g = W.snowflake(35, seed)
    goo, _ = run(g, "IDP2_MPDP", 2)          # k = 2: nothing to re-optimise = the GOO plan
    for k in (5, 10):
        res, _ = run(g, "IDP2_MPDP", k)
        assert res.cost <= goo.cost * (1 + REL)
    exact_small = W.snowflake(12, seed)
    res, _ = run(exact_small, "IDP2_MPDP", 2)
    assert res.cost >= O.optimize(exact_small).cost * (1 - REL)   # GOO never beats the optimum


@pytest.mark.parametrize("algo", ["IDP2_MPDP", "UNIONDP_MPDP"])
def test_thousand_relation_snowflake(algo):
    g = W.snowflake(1000, 0)
    res, subs = run(g, algo, 10)
    assert recompute(g, res) == res.cost
    assert all(q.n <= 10 for q in subs)


def test_invalid_k_rejected():
    L, mp = _lib()
    g = W.snowflake(20, 0)
    with pytest.raises(AssertionError):
        run(g, "UNIONDP_MPDP", 1)


def run_t(g, algo, k, t):
    L, mp = _lib()
    L.mpdp_heuristic_optimize_t.restype = C.c_int
    L.mpdp_heuristic_optimize_t.argtypes = [C.POINTER(mp.mpdp_query_graph), C.c_int, C.c_uint32, C.c_uint32,
                                            SOLVER, C.c_void_p, C.POINTER(mp.mpdp_result)]
    solver = Oracle(mp, k)
    ga, rb = mp.GraphArgs(g), mp.ResultBuf(g.n)
    st = L.mpdp_heuristic_optimize_t(ga.ref(), mp.ALGOS[algo], k, t, solver.cb, None, rb.ref())
    return st, rb.to_result() if st == 0 else None, solver.subs


@pytest.mark.parametrize("n,k,t,seed", [(60, 12, 6, 0), (120, 15, 8, 1), (300, 14, 14, 2)])
def test_uniondp_partition_threshold(n, k, t, seed):
    """UnionDP's upper threshold t: every partition of a
    recursion level has at most t relations; only the final exact DP may hold up
    to k composites; t = k is the algorithm as listed (= mpdp_heuristic_optimize)."""
    g = W.snowflake(n, seed)
    st, res, subs = run_t(g, "UNIONDP_MPDP", k, t)
    assert st == 0
    assert recompute(g, res) == res.cost
    assert all(q.n <= t for q in subs[:-1]) and subs[-1].n <= k
    if t == k:
        ref, _ = run(g, "UNIONDP_MPDP", k)
        assert ref.cost == res.cost and ref.tree() == res.tree()


def test_uniondp_threshold_rejected():
    g = W.snowflake(30, 0)
    for algo, k, t in [("UNIONDP_MPDP", 10, 11), ("UNIONDP_MPDP", 10, 1), ("IDP2_MPDP", 10, 5)]:
        st, _, _ = run_t(g, algo, k, t)
        assert st == 1                        # MPDP_ERR_INVALID_ARGUMENT
