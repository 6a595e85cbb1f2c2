"""GPU parity: the CUDA path through the C ABI vs the CPU oracle.

The bar (BASELINE.json north_star): bit-exact connected-set,
join-pair and per-level counts and the identical plan tree under the tie-break
R7; optimal cost within relative 1e-9 (bit equality is expected under
R5/R6/R7 and asserted as well)."""
import random

import pytest

from oracle import pyoracle as O
import workload as W

pytestmark = pytest.mark.gpu

REL = 1e-9


@pytest.fixture(scope="module")
def ctx():
    from paper_2202_13511_b200 import mpdp
    with mpdp.Context(device=0, workspace_bytes=3 << 30) as c:
        yield c


@pytest.fixture(scope="module")
def big_ctx():
    from paper_2202_13511_b200 import mpdp
    with mpdp.Context(device=0, workspace_bytes=12 << 30) as c:
        yield c


@pytest.fixture(scope="module")
def wide_ctx():
    from paper_2202_13511_b200 import mpdp
    with mpdp.Context(device=0, workspace_bytes=1 << 30, flags=mpdp.FLAG_FORCE_WIDE_MASKS) as c:
        yield c


def check(r, o, g, exact=True):
    assert abs(r.cost - o.cost) <= REL * abs(o.cost), (g.name, r.cost, o.cost)
    if exact:
        assert r.cost == o.cost, (g.name, r.cost.hex(), o.cost.hex())
    assert r.csg_count == o.csg_count, g.name
    assert r.ccp_pairs == o.ccp_pairs, g.name
    assert r.pairs_evaluated == o.pairs_evaluated, g.name
    assert r.level_csg == o.level_csg, g.name
    assert r.level_ccp == o.level_ccp, g.name
    assert r.level_pairs == o.level_pairs, g.name
    assert r.tree() == O.tree_of(o.nodes), g.name
    assert len(r.nodes) == 2 * g.n - 1
    for a, b in zip(r.nodes, o.nodes):
        assert (a.left, a.right, a.relation, a.set) == (b.left, b.right, b.relation, b.set)
        assert a.cardinality == b.card and a.cost == b.cost
    assert r.gpu_launches >= 1


SMALL = [(t, n, s) for t in ["star", "snowflake", "chain", "clique", "cycle", "random"]
         for n in ([2, 3, 5, 8, 11, 14] if t != "cycle" else [3, 5, 8, 11, 14]) for s in range(2)]


@pytest.mark.parametrize("topo,n,seed", SMALL)
def test_small_parity(ctx, topo, n, seed):
    g = W.generate(topo, n, seed)
    check(ctx.mpdp_optimize(g), O.optimize(g), g)


@pytest.mark.parametrize("seed", range(40))
def test_random_cyclic_parity(ctx, seed):
    rng = random.Random(seed)
    n = rng.randint(4, 15)
    g = W.random_connected(n, seed, extra=rng.choice([0.1, 0.25, 0.5, 0.8]))
    check(ctx.mpdp_optimize(g), O.optimize(g), g)


# multi-tile levels with ragged tails, heavy (cross-warp) sets, blocks with checks
MEDIUM = [("star", 18, 0), ("snowflake", 20, 1), ("chain", 22, 2), ("clique", 14, 3),
          ("cycle", 17, 4), ("random", 16, 5), ("random", 17, 6), ("clique", 16, 7)]


@pytest.mark.parametrize("topo,n,seed", MEDIUM)
def test_medium_parity(ctx, topo, n, seed):
    g = W.generate(topo, n, seed)
    check(ctx.mpdp_optimize(g), O.optimize(g), g)


# BASELINE.json configurations at full size (configs 1-4), in the bench launch path
FULL = [("star", 10, 0), ("snowflake", 20, 0), ("snowflake", 20, 1), ("star", 25, 0), ("clique", 18, 0)]


@pytest.mark.parametrize("topo,n,seed", FULL)
def test_full_size_parity(ctx, topo, n, seed):
    g = W.generate(topo, n, seed)
    ctx.mpdp_stage(g)                   # the launch sequence bench.py times
    ctx.mpdp_run()
    r = ctx.mpdp_fetch()
    check(r, O.optimize_dpccp(g), g)


@pytest.mark.parametrize("topo,n,seed", [("snowflake", 24, 2), ("snowflake", 28, 3), ("chain", 28, 4)])
def test_large_sparse_tree_parity(big_ctx, topo, n, seed):
    """Sparse trees beyond the BASELINE sizes: the list kernel generates most
    levels from the previous level's sets (expand_to_list with G lanes per set,
    or the evaluation walk's emit_children for levels with more sets than half
    the grid's threads) instead of scanning C(n, k+1) ranks."""
    g = W.generate(topo, n, seed)
    check(big_ctx.mpdp_optimize(g), O.optimize_dpccp(g), g)


@pytest.mark.parametrize("topo,n,seed", [("star", 9, 0), ("clique", 10, 1), ("cycle", 12, 2),
                                         ("random", 13, 3), ("snowflake", 15, 4)])
def test_wide_mask_kernels(wide_ctx, topo, n, seed):
    g = W.generate(topo, n, seed)
    check(wide_ctx.mpdp_optimize(g), O.optimize(g), g)


def test_wide_beyond_32_chain_closed_form(ctx):
    n = 34                              # 64-bit masks for real (2^34 ranks)
    g = W.chain(n, 0)
    r = ctx.mpdp_optimize(g)
    assert r.csg_count == n * (n + 1) // 2
    assert r.ccp_pairs == (n ** 3 - n) // 6 == r.pairs_evaluated
    # the plan is a valid CP-free tree whose recomputed cost is the reported one
    for nd in r.nodes:
        if nd.relation < 0:
            L, R = r.nodes[nd.left], r.nodes[nd.right]
            assert L.set & R.set == 0 and L.set | R.set == nd.set and L.set < R.set
            assert nd.cost == (L.cost + R.cost) + O.card(g, nd.set)


def test_edge_cases(ctx):
    from paper_2202_13511_b200 import mpdp
    g1 = W.QueryGraph(1, [42.0], [], [])
    r = ctx.mpdp_optimize(g1)
    assert r.cost == 0.0 and r.csg_count == 1 and r.ccp_pairs == 0 and r.tree() == 0
    g2 = W.QueryGraph(2, [4.0, 8.0], [(0, 1)], [0.25], leaf_cost=[1.0, 2.0])
    r = ctx.mpdp_optimize(g2)
    assert r.cost == (1.0 + 2.0) + 8.0 and r.tree() == (0, 1)
    gd = W.QueryGraph(3, [1.0, 2.0, 3.0], [(0, 1)], [0.5])
    with pytest.raises(mpdp.MPDPError) as e:
        ctx.mpdp_optimize(gd)
    assert e.value.status == mpdp.ERR_DISCONNECTED
    for bad in [W.QueryGraph(2, [4.0, 8.0], [(0, 1)], [0.0]),
                W.QueryGraph(2, [4.0, -8.0], [(0, 1)], [0.5]),
                W.QueryGraph(2, [4.0, float("inf")], [(0, 1)], [0.5]),
                W.QueryGraph(2, [4.0, 8.0], [(1, 0)], [0.5]),
                W.QueryGraph(3, [4.0, 8.0, 1.0], [(0, 1), (0, 1), (1, 2)], [0.5, 0.5, 0.5])]:
        with pytest.raises(mpdp.MPDPError) as e:
            ctx.mpdp_optimize(bad)
        assert e.value.status == mpdp.ERR_INVALID_ARGUMENT
    with pytest.raises(mpdp.MPDPError) as e:
        ctx.mpdp_optimize(W.star(5, 0), algo="DPSIZE_REF")
    assert e.value.status == mpdp.ERR_UNSUPPORTED
    # the context stays usable after errors
    g = W.star(8, 3)
    check(ctx.mpdp_optimize(g), O.optimize(g), g)


def test_leaf_costs_parity(ctx):
    for seed in range(6):
        g = W.random_connected(10, seed, extra=0.3)
        rng = random.Random(seed)
        g.leaf_cost = [rng.choice([0.0, 1.0, 1e3, 12345.678]) for _ in range(g.n)]
        check(ctx.mpdp_optimize(g), O.optimize(g), g)


def test_repeated_queries_reuse_memo(ctx):
    # memo tags: stale slots of earlier queries must read as empty
    gs = [W.star(12, 0), W.clique(8, 1), W.star(12, 0), W.snowflake(13, 2), W.clique(8, 1)]
    for g in gs:
        check(ctx.mpdp_optimize(g), O.optimize(g), g)


def test_determinism(ctx):
    g = W.random_connected(15, 9, extra=0.3)
    a, b = ctx.mpdp_optimize(g), ctx.mpdp_optimize(g)
    assert a.tree() == b.tree() and a.cost == b.cost and a.level_ccp == b.level_ccp


def test_load_factor_variants():
    from paper_2202_13511_b200 import mpdp
    g = W.clique(12, 4)
    o = O.optimize(g)
    for lf in (0.25, 0.75, 0.9):
        with mpdp.Context(device=0, workspace_bytes=256 << 20, load_factor=lf,
                          flags=mpdp.FLAG_HASH_MEMO) as c:
            check(c.mpdp_optimize(g), o, g)


@pytest.fixture(scope="module")
def hash_ctx():
    from paper_2202_13511_b200 import mpdp
    with mpdp.Context(device=0, workspace_bytes=2 << 30, flags=mpdp.FLAG_HASH_MEMO) as c:
        yield c


@pytest.mark.parametrize("topo,n,seed", [("star", 14, 0), ("clique", 12, 1), ("cycle", 13, 2),
                                         ("random", 14, 3), ("snowflake", 17, 4), ("star", 20, 5),
                                         ("clique", 15, 6)])
def test_hash_memo_ablation_parity(hash_ctx, topo, n, seed):
    """The Murmur3 open-addressing memo (MPDP_FLAG_HASH_MEMO) gives the same results."""
    g = W.generate(topo, n, seed)
    check(hash_ctx.mpdp_optimize(g), O.optimize(g), g)


@pytest.mark.parametrize("topo,n,seed", [("clique", 12, 1), ("cycle", 16, 2), ("random", 15, 3),
                                         ("clique", 16, 7), ("random", 16, 8)])
def test_memo_layouts_agree(ctx, topo, n, seed):
    """Clique / general queries use the bitmask-indexed memo (memo_kind 2) by
    default; the colex-rank layout (MPDP_FLAG_RANK_MEMO) gives the same results."""
    from paper_2202_13511_b200 import mpdp
    g = W.generate(topo, n, seed)
    o = O.optimize(g)
    r = ctx.mpdp_optimize(g)
    assert r.memo_kind == 2, r.memo_kind
    check(r, o, g)
    with mpdp.Context(device=0, workspace_bytes=1 << 30, flags=mpdp.FLAG_RANK_MEMO) as c:
        r2 = c.mpdp_optimize(g)
        assert r2.memo_kind == 1
        check(r2, o, g)
    assert ctx.mpdp_optimize(W.snowflake(20, seed)).memo_kind == 1     # (n > 13) trees keep the colex layout


@pytest.mark.parametrize("topo,n,seed", [("star", 2, 0), ("chain", 3, 1), ("star", 10, 0), ("snowflake", 13, 2),
                                         ("chain", 13, 3), ("snowflake", 9, 4), ("star", 13, 10), ("chain", 2, 5)])
def test_small_kernel_parity(ctx, topo, n, seed):
    """Tree queries with n <= 13 run on the single-CTA shared-memory kernel
    (memo_kind 3); the multi-CTA path (MPDP_FLAG_NO_SMALL) and the oracle agree."""
    from paper_2202_13511_b200 import mpdp
    g = W.generate(topo, n, seed)
    o = O.optimize(g)
    r = ctx.mpdp_optimize(g)
    assert r.memo_kind == 3, (g.name, r.memo_kind)
    assert r.gpu_launches == 1
    check(r, o, g)
    with mpdp.Context(device=0, workspace_bytes=256 << 20, flags=mpdp.FLAG_NO_SMALL) as c:
        r2 = c.mpdp_optimize(g)
        assert r2.memo_kind != 3
        check(r2, o, g)


@pytest.mark.parametrize("topo,n,seed", [("chain", 14, 0), ("chain", 20, 1), ("chain", 25, 3), ("chain", 26, 4)])
def test_tree1_kernel_parity(ctx, topo, n, seed):
    """Sparse tree queries whose levels fit the single-CTA list kernel
    (k_dp_tree1: one launch, global colex-rank memo) agree with the oracle and
    with the multi-CTA list kernel (MPDP_FLAG_NO_SMALL)."""
    from paper_2202_13511_b200 import mpdp
    g = W.generate(topo, n, seed)
    o = O.optimize(g)
    r = ctx.mpdp_optimize(g)
    assert (r.memo_kind, r.gpu_launches) == (1, 1), g.name
    check(r, o, g)
    with mpdp.Context(device=0, workspace_bytes=2 << 30, flags=mpdp.FLAG_NO_SMALL) as c:
        r2 = c.mpdp_optimize(g)
        assert r2.gpu_launches >= 2                 # multi-CTA kernels
        check(r2, o, g)


@pytest.mark.parametrize("topo,n,seed", [("random", 14, 0), ("random", 16, 1), ("cycle", 17, 2)])
def test_ccc_ablation_parity(ctx, topo, n, seed):
    """Collaborative Context Collection (default) and lane-contiguous candidate
    chunks (MPDP_FLAG_NO_CCC) give the oracle's results on general graphs."""
    from paper_2202_13511_b200 import mpdp
    g = W.generate(topo, n, seed)
    o = O.optimize(g)
    check(ctx.mpdp_optimize(g), o, g)
    with mpdp.Context(device=0, workspace_bytes=1 << 30, flags=mpdp.FLAG_NO_CCC) as c:
        check(c.mpdp_optimize(g), o, g)


@pytest.mark.parametrize("n,seed,hub", [(14, 0, 0), (17, 1, 0), (20, 2, 0), (16, 3, 15), (18, 4, 7)])
def test_star_kernel_parity(ctx, n, seed, hub):
    """Star queries (n >= 14) run on k_dp_star (memo_kind 4), also with the hub
    not at vertex 0 (relabelled stars) and with composite leaf costs; the general
    tree kernel (MPDP_FLAG_NO_STAR) and the oracle agree."""
    from paper_2202_13511_b200 import mpdp
    g = W.star(n, seed)
    if hub:
        perm = list(range(n))
        perm[0], perm[hub] = perm[hub], perm[0]          # swap vertex 0 and `hub`
        card = [0.0] * n
        for v in range(n):
            card[perm[v]] = g.card[v]
        edges = [(min(perm[a], perm[b]), max(perm[a], perm[b])) for a, b in g.edges]
        g = W.QueryGraph(n, card, edges, list(g.sel), name=f"star-{n}-hub{hub}")
    if seed % 2:
        g.leaf_cost = [float((7 * i) % 5) for i in range(n)]
    o = O.optimize(g)
    r = ctx.mpdp_optimize(g)
    assert r.memo_kind == 4, r.memo_kind
    check(r, o, g)
    with mpdp.Context(device=0, workspace_bytes=1 << 30, flags=mpdp.FLAG_NO_STAR) as c:
        r2 = c.mpdp_optimize(g)
        assert r2.memo_kind == 1
        check(r2, o, g)


def test_optimize_batch(ctx):
    """mpdp_optimize_batch: small tree queries share one launch (one CTA
    each), the others run one by one; every result equals the oracle's and the
    single-query call's."""
    gs = [W.generate(t, n, s) for s, (t, n) in enumerate(
        [("star", 2), ("chain", 3), ("star", 10), ("snowflake", 13), ("chain", 13), ("snowflake", 9),
         ("clique", 8), ("star", 16), ("cycle", 9), ("snowflake", 12), ("star", 13)])]
    gs[5].leaf_cost = [float(i % 3) for i in range(gs[5].n)]
    rs = ctx.mpdp_optimize_batch(gs)
    assert len(rs) == len(gs)
    for g, r in zip(gs, rs):
        o = O.optimize(g)
        check(r, o, g)
        r1 = ctx.mpdp_optimize(g)
        assert r.tree() == r1.tree() and r.cost == r1.cost
        tree = len(g.edges) == g.n - 1
        clique = g.n >= 3 and len(g.edges) == g.n * (g.n - 1) // 2
        # the single-CTA kernel: trees with n <= 13, and general graphs with
        # n <= 10 or at most 4 independent cycles (memo-probe connectivity)
        sparse_general = not tree and not clique and (g.n <= 10 or len(g.edges) + 1 <= g.n + 4)
        assert (r.memo_kind == 3) == (g.n <= 13 and (tree or sparse_general)), (g.name, r.memo_kind)
        # mid-size trees whose levels fit the kernel's shared-memory lists
        assert (r.memo_kind == 5) == (tree and 14 <= g.n <= 32 and max(o.level_csg) <= 6144), (g.name, r.memo_kind)
    assert ctx.mpdp_optimize_batch([]) == []


def test_optimize_batch_128bit_memo(ctx):
    """Mid-size tree sub-problems (14 <= n <= 32) of one batch share ONE memo
    keyed by 128-bit {sub-problem, mask} (memo_kind 5); every result equals the
    oracle's, also with composite leaf costs, across repeated batches (stale
    slots of earlier batches are reused through the epoch) and with the same
    graph twice in one batch (same masks, different sub-problem keys)."""
    rng = random.Random(128)
    gs = []
    for i in range(24):
        topo = rng.choice(["snowflake", "chain", "star"])
        g = W.generate(topo, rng.randint(14, 22 if topo != "star" else 15), 500 + i)   # (star-15: 3432 sets per level at most)
        if rng.random() < 0.5:
            g.leaf_cost = [float(rng.choice([0, 3, 250, 1e4])) for _ in range(g.n)]
        gs.append(g)
    gs.append(gs[0])
    oracle = [O.optimize(g) for g in gs]
    for rep in range(3):
        rs = ctx.mpdp_optimize_batch(gs if rep != 1 else gs[::-1])
        for g, o, r in zip(gs if rep != 1 else gs[::-1], oracle if rep != 1 else oracle[::-1], rs):
            assert r.memo_kind == 5, (g.name, r.memo_kind)
            check(r, o, g)


def test_small_kernel_leaf_costs_and_dpsub():
    """Composite leaves (non-zero leaf costs) on the small kernel; the
    DPSUB-enumeration ablation (general-graph kernels) agrees on the cost."""
    from paper_2202_13511_b200 import mpdp
    g = W.generate("snowflake", 12, 3)
    g.leaf_cost = [float(10 * (i % 4)) + 0.5 for i in range(g.n)]
    with mpdp.Context(device=0, workspace_bytes=256 << 20) as c:
        check(c.mpdp_optimize(g), O.optimize(g), g)
    with mpdp.Context(device=0, workspace_bytes=256 << 20, flags=mpdp.FLAG_DPSUB_ENUM) as c:
        r = c.mpdp_optimize(g)
        o = O.optimize(g)
        assert r.cost == o.cost


def test_alternating_memo_kinds(ctx, hash_ctx):
    # interleave both memo layouts and widths on one device
    for g in [W.star(12, 1), W.clique(9, 2), W.random_connected(13, 3), W.star(11, 4), W.cycle(12, 5)]:
        o = O.optimize(g)
        check(ctx.mpdp_optimize(g), o, g)
        check(hash_ctx.mpdp_optimize(g), o, g)


def test_graph_and_direct_paths_agree():
    """The cached CUDA-graph replay, the direct launch path and the timeout
    (per-level synchronising) path produce identical results."""
    from paper_2202_13511_b200 import mpdp
    gs = [W.star(16, 2), W.clique(13, 3), W.random_connected(14, 4, extra=0.3)]
    outs = []
    for flags, tmo in [(0, 0.0), (mpdp.FLAG_NO_GRAPH, 0.0), (0, 60000.0)]:
        with mpdp.Context(device=0, workspace_bytes=512 << 20, flags=flags, timeout_ms=tmo) as c:
            outs.append([c.mpdp_optimize(g) for g in gs] + [c.mpdp_optimize(g) for g in gs])
    for g, o in zip(gs + gs, zip(*outs)):
        ref = O.optimize(g)
        for r in o:
            check(r, ref, g)


@pytest.mark.parametrize("topo,n,seed", [("star", 12, 0), ("clique", 13, 1), ("cycle", 14, 2),
                                         ("random", 15, 3), ("snowflake", 18, 4), ("chain", 16, 5)])
def test_fused_and_per_level_kernels_agree(topo, n, seed):
    """The single cooperative kernel (default) and the per-level kernels
    (MPDP_FLAG_NO_FUSED) both match the oracle."""
    from paper_2202_13511_b200 import mpdp
    g = W.generate(topo, n, seed)
    o = O.optimize(g)
    for flags in (mpdp.FLAG_NO_SMALL, mpdp.FLAG_NO_FUSED):
        with mpdp.Context(device=0, workspace_bytes=512 << 20, flags=flags) as c:
            r = c.mpdp_optimize(g)
            check(r, o, g)
            if flags == mpdp.FLAG_NO_SMALL:
                # the whole-query kernel, after k_init unless the previous
                # launch was a (self-resetting) dataflow kernel
                assert r.gpu_launches in (1, 2)


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("topo,n,seed", [("star", 12, 0), ("clique", 13, 1), ("cycle", 13, 2),
                                         ("random", 14, 3), ("snowflake", 16, 4), ("star", 17, 5)])
def test_sharded_world_all_levels(world, topo, n, seed):
    """The multi-GPU sharded level loop (per-level colex-rank shares + in-place
    segment exchange + counter reduction), with `world` ranks simulated as memo
    replicas on one device and EVERY level sharded (shares down to empty)."""
    from paper_2202_13511_b200 import mpdp
    g = W.generate(topo, n, seed)
    with mpdp.Context(device=0, workspace_bytes=1 << 30, world=world,
                      flags=mpdp.FLAG_SIMULATE_WORLD | mpdp.FLAG_SHARD_ALL_LEVELS) as c:
        check(c.mpdp_optimize(g), O.optimize(g), g)


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_world_default_threshold(world):
    from paper_2202_13511_b200 import mpdp
    for g in (W.star(20, 1), W.clique(15, 2)):
        o = O.optimize_dpccp(g)
        with mpdp.Context(device=0, workspace_bytes=2 << 30, world=world, flags=mpdp.FLAG_SIMULATE_WORLD) as c:
            r = c.mpdp_optimize(g)
            check(r, o, g)


@pytest.fixture(scope="module")
def dpsub_ctx():
    from paper_2202_13511_b200 import mpdp
    with mpdp.Context(device=0, workspace_bytes=2 << 30, flags=mpdp.FLAG_DPSUB_ENUM) as c:
        yield c


@pytest.mark.parametrize("topo,n,seed", [("star", 9, 0), ("snowflake", 12, 1), ("chain", 10, 2), ("cycle", 9, 3),
                                         ("clique", 8, 4), ("random", 11, 5), ("star", 2, 0), ("clique", 3, 1)])
def test_dpsub_enumeration_ablation(dpsub_ctx, topo, n, seed):
    """MPDP_FLAG_DPSUB_ENUM (NEXT-3 ablation, Alg. generic_dpsub):
    same plan, cost and CCP pairs as MPDP; evaluated pairs = sum over connected
    S of 2^(|S|-1) - 1 (unordered, reading R3), from the oracle's csg levels."""
    g = W.generate(topo, n, seed)
    r, o = dpsub_ctx.mpdp_optimize(g), O.optimize(g)
    assert r.cost == o.cost and r.tree() == O.tree_of(o.nodes)
    assert r.csg_count == o.csg_count and r.ccp_pairs == o.ccp_pairs and r.level_ccp == o.level_ccp
    want = [c * ((1 << (k - 1)) - 1) if k >= 2 else 0 for k, c in enumerate(o.level_csg)]
    assert r.level_pairs == want
    assert r.pairs_evaluated == sum(want)


def test_dpsub_star_closed_form(dpsub_ctx):
    """Star-20 under DPSUB enumeration: sum_j C(19,j)(2^j - 1) = 3^19 - 2^19
    evaluated pairs against MPDP's 19 * 2^18 (P:319's ratio, unordered)."""
    g = W.star(20, 0)
    r = dpsub_ctx.mpdp_optimize(g)
    assert r.pairs_evaluated == 3 ** 19 - 2 ** 19
    assert r.ccp_pairs == 19 * 2 ** 18


def test_randomized_sweep_all_paths(ctx):
    """Seeded sweep over topologies and sizes that hit every single-GPU kernel
    (single-CTA small / tree1, star, list, clique, general) and the batch entry
    point; every result equals the oracle's."""
    import random
    from paper_2202_13511_b200 import mpdp
    rng = random.Random(2202)
    gs = []
    for i in range(48):
        topo = rng.choice(["star", "snowflake", "chain", "cycle", "clique", "random"])
        hi = {"clique": 13, "random": 13, "cycle": 16, "star": 19, "snowflake": 19, "chain": 22}[topo]
        g = W.generate(topo, rng.randint(2 if topo in ("star", "chain", "snowflake") else 3, hi), 1000 + i)
        if topo == "star" and g.n >= 3 and rng.random() < 0.5:        # hub moved off vertex 0
            h = rng.randrange(g.n)
            perm = list(range(g.n))
            perm[0], perm[h] = perm[h], perm[0]
            card = [0.0] * g.n
            for v in range(g.n):
                card[perm[v]] = g.card[v]
            edges = [(min(perm[a], perm[b]), max(perm[a], perm[b])) for a, b in g.edges]
            g = W.QueryGraph(g.n, card, edges, list(g.sel), name=f"{g.name}-hub{h}")
        if rng.random() < 0.3:
            g.leaf_cost = [float(rng.choice([0, 1, 7, 1000])) for _ in range(g.n)]
        gs.append(g)
    oracle = [O.optimize(g) for g in gs]
    for g, o in zip(gs, oracle):
        check(ctx.mpdp_optimize(g), o, g)
    for g, o, r in zip(gs, oracle, ctx.mpdp_optimize_batch(gs)):
        check(r, o, g)
    with mpdp.Context(device=0, workspace_bytes=1 << 30, flags=mpdp.FLAG_NO_SMALL | mpdp.FLAG_NO_STAR) as c:
        for g, o in zip(gs[:16], oracle[:16]):
            check(c.mpdp_optimize(g), o, g)


def test_contexts_share_kernel_attributes(ctx):
    """Kernel attributes (dynamic shared memory limits) are process-wide: a
    sharded context running a small query must not lower the limit another
    context's larger query launches with (regression: cooperative launch
    'invalid argument' after a simulated-world run of a smaller n)."""
    from paper_2202_13511_b200 import mpdp
    small, big = W.snowflake(14, 3), W.snowflake(22, 4)
    ob = O.optimize(big)
    with mpdp.Context(device=0, workspace_bytes=1 << 30, world=2,
                      flags=mpdp.FLAG_SIMULATE_WORLD | mpdp.FLAG_SHARD_ALL_LEVELS) as sh:
        check(ctx.mpdp_optimize(big), ob, big)
        check(sh.mpdp_optimize(small), O.optimize(small), small)
        check(ctx.mpdp_optimize(big), ob, big)


def test_batch_invalidates_staged_query(ctx):
    """a batch between mpdp_stage and mpdp_run used to
    leave the context's per-query fields (star hub, largest tree level) from
    the batch's last small query, so mpdp_run could route the staged query into
    the wrong kernel.  A batch now restores them and invalidates the staged
    query: mpdp_run fails loudly until the next mpdp_stage, and a restage
    gives the oracle's result."""
    from paper_2202_13511_b200 import mpdp
    big = W.snowflake(18, 5)                  # a non-star tree with n >= 14
    ctx.mpdp_stage(big)
    ctx.mpdp_optimize_batch([W.chain(3, 0), W.star(6, 1)])
    with pytest.raises(mpdp.MPDPError) as e:
        ctx.mpdp_run()
    assert e.value.status == mpdp.ERR_INVALID_ARGUMENT
    ctx.mpdp_stage(big)
    ctx.mpdp_run()
    check(ctx.mpdp_fetch(), O.optimize(big), big)


def _structured(name, n, edges, seed):
    """A fixed topology with the recipe's numbers (cards log-uniform, factors)."""
    import numpy as np
    rng = np.random.default_rng(seed)
    card = [float(x) for x in 10.0 ** rng.uniform(1.0, 6.0, size=n)]
    edges = sorted({(min(a, b), max(a, b)) for a, b in edges})
    sel = [float(x) for x in 10.0 ** rng.uniform(-1.0, 0.0, size=len(edges))]
    return W.QueryGraph(n, card, edges, sel, name=name)


def _sun(k, pend):
    """A k-cycle whose every vertex carries `pend` pendant vertices: its large
    connected sets have many blocks (the cycle plus one bridge per pendant)."""
    edges = [(i, (i + 1) % k) for i in range(k)]
    v = k
    for i in range(k):
        for _ in range(pend):
            edges.append((i, v))
            v += 1
    return v, edges


def _cut_triangle():
    """A triangle of cut vertices (a block made only of cut vertices) whose
    corners carry pendant paths and a chorded square."""
    edges = [(0, 1), (1, 2), (0, 2),                  # the triangle
             (0, 3), (3, 4), (1, 5), (5, 6), (2, 7),  # pendant paths
             (7, 8), (8, 9), (9, 10), (10, 7), (7, 9)]   # a chorded square at vertex 7
    return 11, edges


@pytest.mark.parametrize("shape", ["sun6x2", "sun5x3", "sun8x1", "sun7x2", "cut_triangle", "barbell"])
def test_block_structures_parity(ctx, shape):
    """Readings R20/R21 on shapes the random graphs rarely produce: sets with
    more blocks than the heavy list caches (kHeavyBlk = 8, the Find-Blocks
    fallback), blocks made only of cut vertices (found from an edge), bridges
    (small blocks evaluated lane-parallel) and hanging parts of several cut
    vertices of one block."""
    if shape.startswith("sun"):
        k, p = (int(x) for x in shape[3:].split("x"))
        n, edges = _sun(k, p)
    elif shape == "cut_triangle":
        n, edges = _cut_triangle()
    else:                                          # two 5-cliques joined by a 3-path
        edges = [(a, b) for a in range(5) for b in range(a + 1, 5)]
        edges += [(a + 8, b + 8) for a in range(5) for b in range(a + 1, 5)]
        edges += [(4, 5), (5, 6), (6, 7), (7, 8)]
        n = 13
    g = _structured(shape, n, edges, 11)
    r = ctx.mpdp_optimize(g)
    check(r, O.optimize(g), g)
    from paper_2202_13511_b200 import mpdp
    with mpdp.Context(device=0, workspace_bytes=1 << 30, flags=mpdp.FLAG_DPSUB_ENUM) as c:   # (ablation)
        r2 = c.mpdp_optimize(g)
        assert r2.cost == r.cost and r2.tree() == r.tree() and r2.ccp_pairs == r.ccp_pairs
