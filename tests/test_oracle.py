"""Pins for the CPU oracle (oracle/), all `-m "not gpu"`.

Every check below pins the oracle to something other than itself: a value the
paper prints (tests/golden/, cited), a closed form, an exhaustive enumeration
written independently here, or an invariant the paper proves.
§"Oracle pins".
"""
import itertools
import math
import random

import pytest

from conftest import labels_to_mask, read_golden
from oracle import pyoracle as O
import workload as W


def edges_from_golden(s):
    return [tuple(int(x) for x in e.split("-")) for e in s.split()]


def graph_from_labels(n, edge_labels, card=None, sel=None):
    edges = sorted((min(a, b) - 1, max(a, b) - 1) for a, b in edge_labels)
    return W.QueryGraph(n, card or [10.0] * n, edges, sel or [0.5] * len(edges))


# --------------------------------------------------------------------------
# Independent brute-force helpers (plain Python, written from P:181-187)
# --------------------------------------------------------------------------
def py_connected(adj, S):
    if S == 0:
        return False
    seen, todo = 0, S & -S
    while todo:
        v = (todo & -todo).bit_length() - 1
        todo &= todo - 1
        if seen >> v & 1:
            continue
        seen |= 1 << v
        todo |= adj[v] & S & ~seen
    return seen == S


def py_ccp_count(g):
    """Unordered CCP pairs by testing every pair of disjoint non-empty subsets."""
    adj, n = g.adjacency(), g.n
    total = 0
    for S in range(1, 1 << n):
        if not py_connected(adj, S):
            continue
        A = (S - 1) & S
        while A:
            B = S & ~A
            if A < B and py_connected(adj, A) and py_connected(adj, B) and \
                    any(adj[v] & B for v in range(n) if A >> v & 1):
                total += 1
            A = (A - 1) & S
    return total


# --------------------------------------------------------------------------
# Paper worked examples
# --------------------------------------------------------------------------
def test_fig5_blocks_cut_vertices_grow():
    gold = read_golden("fig5_blocks.txt")
    g = graph_from_labels(9, edges_from_golden(gold["edges"]))
    full = (1 << 9) - 1
    want = sorted(labels_to_mask(b) for b in gold["blocks"].split("|"))
    assert sorted(O.blocks(g, full)) == want
    cut = {int(x) - 1 for x in gold["cut_vertices"].split()}
    cut_by_blocks = {v for v in range(9) if sum(b >> v & 1 for b in want) > 1}
    assert cut_by_blocks == cut
    for v in range(9):     # a cut vertex disconnects the graph when removed
        assert (not O.connected(g, full & ~(1 << v))) == (v in cut)
    kv = dict(x.split("=") for x in gold["grow"].split())
    assert O.grow(g, labels_to_mask(kv["source"]), labels_to_mask(kv["restriction"])) == \
        labels_to_mask(kv["result"])
    # removing edge (1,4) does not split the graph
    assert O.connected(g, full)
    # 512 subsets for DPSUB vs 32 ordered block splits for MPDP (16 unordered, R3)
    assert 2 ** 9 == int(gold["dpsub_subsets_full_set"])
    assert 2 * O.mpdp_pairs(g, full) == int(gold["mpdp_ordered_block_splits_full_set"])


def test_fig5_block_cut_chain():
    gold = read_golden("fig5_blocks.txt")
    g = graph_from_labels(9, edges_from_golden(gold["edges"]))
    items = [x.strip() for x in gold["block_cut_chain"].split("|")]
    blocks = set(O.blocks(g, (1 << 9) - 1))
    for i, it in enumerate(items):
        if i % 2 == 0:
            assert labels_to_mask(it) in blocks
        else:  # cut vertex shared by its two neighbouring blocks
            c = labels_to_mask(it)
            assert labels_to_mask(items[i - 1]) & labels_to_mask(items[i + 1]) == c


def test_fig3_ccp_examples():
    gold = read_golden("fig3_tree.txt")
    g = graph_from_labels(8, edges_from_golden(gold["edges"]))
    a, b = gold["not_ccp"].split("|")
    assert not O.is_ccp(g, labels_to_mask(a), labels_to_mask(b))
    a, b = gold["ccp"].split("|")
    assert O.is_ccp(g, labels_to_mask(a), labels_to_mask(b))
    kv = dict(x.split("=") for x in gold["tree_pairs"].split())
    S = labels_to_mask(kv["set"])
    assert O.mpdp_pairs(g, S) == int(kv["count"])
    # the same count by brute force over all unordered splits of S
    adj = g.adjacency()
    splits = [A for A in range(1, S) if A & ~S == 0 and A < (S & ~A)
              and O.is_ccp(g, A, S & ~A)]
    assert len(splits) == int(kv["count"])


def test_paper_counter_ratios():
    gold = read_golden("paper_counters.txt")
    # P:319 "around 2805" at star-25: sum_{connected S, |S|>=2} 2^|S| / unordered CCP
    kv = dict(x.split("=") for x in gold["star_dpsub_over_ccp"].split())
    n = int(kv["n"])
    lc, lp = O.counters(W.star(n, 0))
    dpsub = sum(lc[k] * 2 ** k for k in range(2, n + 1))
    ccp = sum(lp)                               # = ccp on trees (Lemma 8)
    assert ccp == (n - 1) * 2 ** (n - 2)
    assert math.floor(dpsub / ccp) == int(kv["value"])
    # P:1071 "12024x fewer Join-Pairs at 20 relations" vs DPSIZE
    kv = dict(x.split("=") for x in gold["star_dpsize_over_mpdp"].split())
    n = int(kv["n"])
    lc, lp = O.counters(W.star(n, 0))
    dpsize = sum(lc[l] * lc[s - l] for s in range(2, n + 1) for l in range(1, s))
    assert math.floor(dpsize / (2 * sum(lp))) == int(kv["value"])


# --------------------------------------------------------------------------
# Closed forms (tests/golden/closed_forms.txt)
# --------------------------------------------------------------------------
CLOSED = {
    "chain": (lambda n: n * (n + 1) // 2, lambda n: (n ** 3 - n) // 6),
    "star": (lambda n: 2 ** (n - 1) + n - 1, lambda n: (n - 1) * 2 ** (n - 2)),
    "clique": (lambda n: 2 ** n - 1, lambda n: (3 ** n - 2 ** (n + 1) + 1) // 2),
    "cycle": (lambda n: n * n - n + 1, lambda n: (n ** 3 - 2 * n * n + n) // 2),
}


@pytest.mark.parametrize("topo", sorted(CLOSED))
@pytest.mark.parametrize("n", [3, 4, 5, 7, 9, 12])
def test_closed_form_counts(topo, n):
    g = W.generate(topo, n, seed=n)
    r = O.optimize_definition(g)
    csg, ccp = CLOSED[topo]
    assert r.csg_count == csg(n)
    assert r.ccp_pairs == ccp(n)
    r1 = O.optimize_dpccp(g)
    assert (r1.csg_count, r1.ccp_pairs) == (csg(n), ccp(n))
    lc, lp = O.counters(g)
    assert sum(lc) == csg(n)
    if topo != "cycle":            # Lemma 8: trees and cliques waste nothing
        assert r.pairs_evaluated == r.ccp_pairs
    else:                          # the whole cycle is one non-complete block
        assert r.pairs_evaluated == r.ccp_pairs + (2 ** (n - 1) - 1) - n * (n - 1) // 2


@pytest.mark.parametrize("topo,n", [("star", 25), ("clique", 18), ("chain", 25)])
def test_closed_form_counts_full_size(topo, n):
    lc, lp = O.counters(W.generate(topo, n, 0))
    csg, ccp = CLOSED[topo]
    assert sum(lc) == csg(n)
    assert sum(lp) == ccp(n)       # Lemma 8: MPDP pairs == CCP on trees / cliques


def test_ccp_count_bruteforce_random():
    for seed in range(8):
        g = W.random_connected(8, seed, extra=0.35)
        assert O.optimize_definition(g).ccp_pairs == py_ccp_count(g)


# --------------------------------------------------------------------------
# Optimum: brute force over every join tree (n <= 7)
# --------------------------------------------------------------------------
def catalan(m):
    return math.comb(2 * m, m) // (m + 1)


@pytest.mark.parametrize("n", [2, 3, 4, 5, 6, 7])
def test_tree_counts(n):
    _, t = O.bruteforce(W.chain(n, 1))
    assert t == 2 ** (n - 1) * catalan(n - 1)
    _, t = O.bruteforce(W.star(n, 1))
    assert t == 2 ** (n - 1) * math.factorial(n - 1)
    _, t = O.bruteforce(W.clique(n, 1))
    assert t == math.factorial(2 * n - 2) // math.factorial(n - 1)


@pytest.mark.parametrize("seed", range(12))
def test_bruteforce_equals_dp_exactly(seed):
    rng = random.Random(seed)
    for topo in ["star", "chain", "cycle", "clique", "snowflake", "random"]:
        n = rng.randint(3, 7) if topo != "cycle" else rng.randint(3, 7)
        g = W.generate(topo, n, seed)
        best, _ = O.bruteforce(g)
        r = O.optimize_definition(g)
        assert r.cost == best          # bit-exact: rounding is monotone (R8)
        assert O.optimize_dpccp(g).cost == best


def test_hand_computed_chain3():
    # cards 8, 4, 2; sel(0,1) = 1/2, sel(1,2) = 1/4 (all exact in binary)
    g = W.QueryGraph(3, [8.0, 4.0, 2.0], [(0, 1), (1, 2)], [0.5, 0.25])
    r = O.optimize_definition(g)
    # card{0,1} = 16, card{1,2} = 2, card{0,1,2} = 8:  (0 join (1 join 2)) costs 2 + 8 = 10
    assert r.cost == 10.0
    assert O.tree_of(r.nodes) == (0, (1, 2))
    assert r.nodes[-1].card == 8.0


def test_leaf_costs_enter_cost():
    g = W.QueryGraph(2, [8.0, 4.0], [(0, 1)], [0.5], leaf_cost=[3.0, 5.0])
    r = O.optimize_definition(g)
    assert r.cost == (3.0 + 5.0) + 16.0


# --------------------------------------------------------------------------
# The three optimisers agree on plan, cost and counters
# --------------------------------------------------------------------------
@pytest.mark.parametrize("seed", range(30))
def test_definition_dpccp_dpsize_agree(seed):
    rng = random.Random(1000 + seed)
    topo = ["random", "random", "snowflake", "star", "cycle", "clique", "chain"][seed % 7]
    n = rng.randint(2, 12) if topo != "cycle" else rng.randint(3, 12)
    g = W.generate(topo, n, seed)
    a, b, c = O.optimize_definition(g), O.optimize_dpccp(g), O.optimize_dpsize(g)
    for r in (b, c):
        assert r.cost == a.cost
        assert O.tree_of(r.nodes) == O.tree_of(a.nodes)
        assert (r.csg_count, r.ccp_pairs, r.pairs_evaluated) == \
            (a.csg_count, a.ccp_pairs, a.pairs_evaluated)
        assert r.level_csg == a.level_csg and r.level_ccp == a.level_ccp


def test_random_numbering_dpccp_order():
    # DPccp's emission order must be a valid DP order for any vertex numbering;
    # the oracle checks it at run time (status 8 on violation).
    for seed in range(40):
        g = W.random_connected(11, seed, extra=0.25, shuffle=True)
        a, b = O.optimize_definition(g), O.optimize_dpccp(g)
        assert O.tree_of(a.nodes) == O.tree_of(b.nodes) and a.cost == b.cost


def test_plan_invariants():
    for seed in range(10):
        g = W.random_connected(10, seed, extra=0.3)
        r = O.optimize_definition(g)
        adj = g.adjacency()
        for nd in r.nodes:
            if nd.relation >= 0:
                continue
            L, R = r.nodes[nd.left].set, r.nodes[nd.right].set
            assert L & R == 0 and L | R == nd.set and L < R            # tie-break R7
            assert O.is_ccp(g, L, R)
            assert nd.cost == (r.nodes[nd.left].cost + r.nodes[nd.right].cost) + O.card(g, nd.set)
        assert len(r.nodes) == 2 * g.n - 1


# --------------------------------------------------------------------------
# Cardinality: closed-form products on power-of-two inputs
# --------------------------------------------------------------------------
def test_card_closed_form():
    rng = random.Random(5)
    n = 12
    ec = [rng.randint(0, 20) for _ in range(n)]
    g = W.random_connected(n, 3, extra=0.4)
    es = [rng.randint(1, 6) for _ in g.edges]
    g.card = [2.0 ** e for e in ec]
    g.sel = [2.0 ** -e for e in es]
    adj = g.adjacency()
    for S in [rng.randrange(1, 1 << n) for _ in range(300)]:
        expo = sum(ec[v] for v in range(n) if S >> v & 1)
        expo -= sum(es[i] for i, (u, v) in enumerate(g.edges) if S >> u & 1 and S >> v & 1)
        assert O.card(g, S) == 2.0 ** expo


def test_card_spec_examples():
    g = W.QueryGraph(3, [10.0, 10.0, 10.0], [(0, 1), (0, 2), (1, 2)], [0.1, 0.1, 0.1])
    assert abs(O.card(g, 0b111) - 1.0) < 1e-15          # SPEC S:192 triangle
    g = W.QueryGraph(2, [1000.0, 500.0], [(0, 1)], [0.001])
    assert abs(O.card(g, 0b11) - 500.0) < 1e-12


# --------------------------------------------------------------------------
# Unranking (reading R10)
# --------------------------------------------------------------------------
def test_unrank_colex():
    assert O.unrank_colex(4, 2, 0) == 0b0011
    assert O.unrank_colex(4, 2, 5) == 0b1100
    for n in range(1, 11):
        for k in range(0, n + 1):
            want = sorted(sum(1 << x for x in c) for c in itertools.combinations(range(n), k))
            got = [O.unrank_colex(n, k, r) for r in range(math.comb(n, k))]
            assert got == want


# --------------------------------------------------------------------------
# Edge cases
# --------------------------------------------------------------------------
def test_edge_cases():
    g1 = W.QueryGraph(1, [42.0], [], [])
    r = O.optimize_definition(g1)
    assert r.cost == 0.0 and r.csg_count == 1 and r.ccp_pairs == 0 and len(r.nodes) == 1
    g2 = W.QueryGraph(2, [4.0, 8.0], [(0, 1)], [0.25])
    r = O.optimize_dpccp(g2)
    assert r.cost == 8.0 and O.tree_of(r.nodes) == (0, 1)
    gd = W.QueryGraph(3, [1.0, 2.0, 3.0], [(0, 1)], [0.5])
    for f in (O.optimize_definition, O.optimize_dpccp, O.optimize_dpsize):
        with pytest.raises(O.OracleError) as e:
            f(gd)
        assert e.value.code == 2
    bad = W.QueryGraph(2, [4.0, 8.0], [(0, 1)], [0.0])
    with pytest.raises(O.OracleError):
        O.optimize_dpccp(bad)
