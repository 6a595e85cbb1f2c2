"""The fused peer exchange of the star and clique kernels (MPDP_FLAG_FUSED_EXCHANGE,
SURVEY §8(e)): W ranks, each with a full memo replica, store
every chunk's costs into every replica and count it in every replica's
dataflow counters; emulated on one GPU as the CTA groups of one cooperative
launch (the guide's rule for ranks that wait on one another).  Every replica
must extract the oracle's plan with the oracle's counters (the library checks
that the W replicas agree bit for bit)."""
import pytest

from oracle import pyoracle as O
import workload as W
from test_gpu_parity import check

pytestmark = pytest.mark.gpu


def relabel(g, hub):
    n = g.n
    perm = list(range(n))
    perm[0], perm[hub] = perm[hub], perm[0]
    card = [0.0] * n
    for v in range(n):
        card[perm[v]] = g.card[v]
    edges = [(min(perm[a], perm[b]), max(perm[a], perm[b])) for a, b in g.edges]
    return W.QueryGraph(n, card, edges, list(g.sel), name=f"{g.name}-hub{hub}")


@pytest.fixture(scope="module", params=[2, 3, 4, 8])
def xr_ctx(request):
    from paper_2202_13511_b200 import mpdp
    with mpdp.Context(device=0, workspace_bytes=4 << 30, world=request.param,
                      flags=mpdp.FLAG_SIMULATE_WORLD | mpdp.FLAG_FUSED_EXCHANGE) as c:
        yield c


@pytest.mark.parametrize("n,seed,hub,leaf", [(3, 0, 0, False), (5, 1, 2, True), (9, 2, 0, False),
                                             (14, 3, 13, False), (17, 4, 0, True), (20, 5, 7, False)])
def test_fused_exchange_star(xr_ctx, n, seed, hub, leaf):
    g = W.star(n, seed)
    if hub:
        g = relabel(g, hub)
    if leaf:
        g.leaf_cost = [float((3 * i) % 7) for i in range(n)]
    r = xr_ctx.mpdp_optimize(g)
    assert r.memo_kind == 4
    check(r, O.optimize(g), g)


def test_fused_exchange_repeated_and_mixed(xr_ctx):
    """Queries back to back (the per-query start barrier and the self-reset
    of every replica's dataflow state), with non-star queries in between
    (they keep the NCCL-style sharded path)."""
    for i, g in enumerate([W.star(16, 7), W.snowflake(12, 1), W.star(16, 7), W.clique(9, 2), W.star(13, 3)]):
        check(xr_ctx.mpdp_optimize(g), O.optimize(g), g)


def test_fused_exchange_star25_full_size():
    """BASELINE config 3 (star-25) with 8 emulated ranks: every replica holds
    the full 2^24-set memo, plan and counters equal the oracle's."""
    from paper_2202_13511_b200 import mpdp
    g = W.star(25, 0)
    with mpdp.Context(device=0, workspace_bytes=8 << 30, world=8,
                      flags=mpdp.FLAG_SIMULATE_WORLD | mpdp.FLAG_FUSED_EXCHANGE) as c:
        r = c.mpdp_optimize(g)
    check(r, O.optimize(g), g)


def test_fused_exchange_needs_peers_across_gpus():
    """A real multi-GPU context must map its peers before a fused-exchange
    query; the record call refuses simulated worlds."""
    from paper_2202_13511_b200 import mpdp
    with mpdp.Context(device=0, workspace_bytes=1 << 30, world=2,
                      flags=mpdp.FLAG_SIMULATE_WORLD | mpdp.FLAG_FUSED_EXCHANGE) as c:
        with pytest.raises(mpdp.MPDPError) as e:
            c.peer_record()
        assert e.value.status == mpdp.ERR_INVALID_ARGUMENT


@pytest.mark.parametrize("n,seed,leaf", [(3, 0, False), (5, 1, True), (9, 2, False), (12, 3, True), (14, 4, False)])
def test_fused_exchange_clique(xr_ctx, n, seed, leaf):
    """Cliques through k_dp_clique_df with the fused exchange: every set
    written into every rank's bitmask-memo replica, counted in every replica."""
    g = W.clique(n, seed)
    if leaf:
        g.leaf_cost = [float((5 * i) % 3) for i in range(n)]
    r = xr_ctx.mpdp_optimize(g)
    assert r.memo_kind == 2
    check(r, O.optimize(g), g)


def test_fused_exchange_clique18_full_size():
    """BASELINE config 4 (clique-18) with 4 emulated ranks."""
    from paper_2202_13511_b200 import mpdp
    g = W.clique(18, 0)
    with mpdp.Context(device=0, workspace_bytes=4 << 30, world=4,
                      flags=mpdp.FLAG_SIMULATE_WORLD | mpdp.FLAG_FUSED_EXCHANGE) as c:
        r = c.mpdp_optimize(g)
    check(r, O.optimize(g), g)
