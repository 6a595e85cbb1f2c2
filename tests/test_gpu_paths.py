"""GPU tests of the round-2 paths: the device deadline of the single-launch
kernels (P:1003's time limit), the real NCCL exchange on one GPU (a 1-rank
communicator, every level sharded), counted join pairs against the closed
forms of Lemma 8, and general graphs at the BASELINE size n = 20."""
import os
import subprocess
import sys

import pytest

from oracle import pyoracle as O
import workload as W
from test_gpu_parity import check

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("topo,n", [("star", 25), ("clique", 18)])
def test_device_timeout_fires_and_context_recovers(topo, n):
    """timeout_ms is checked on the device inside the single-launch kernels
    (k_dp_star: every chunk and dependency wait; k_dp_clique: every level
    barrier).  A deadline far below the query's time returns MPDP_ERR_TIMEOUT;
    the same context then solves queries exactly again."""
    from paper_2202_13511_b200 import mpdp
    g = W.generate(topo, n, 0)
    with mpdp.Context(device=0, workspace_bytes=6 << 30, timeout_ms=0.05) as c:
        with pytest.raises(mpdp.MPDPError) as e:
            c.mpdp_optimize(g)
        assert e.value.status == mpdp.ERR_TIMEOUT
        small = W.generate(topo, 12 if topo == "clique" else 14, 1)
        with pytest.raises(mpdp.MPDPError) as e2:       # still over 50 us
            c.mpdp_optimize(W.generate(topo, n, 1))
        assert e2.value.status == mpdp.ERR_TIMEOUT
    with mpdp.Context(device=0, workspace_bytes=6 << 30, timeout_ms=60000.0) as c:
        r = c.mpdp_optimize(g)
        assert r.memo_kind == (4 if topo == "star" else 2)      # the fast kernel ran, not a fallback
        check(r, O.optimize_dpccp(g), g)
        check(c.mpdp_optimize(small), O.optimize(small), small)


def test_closed_form_counts_full_size():
    """The star and clique kernels count the pairs they evaluate; at full size
    the counts equal Lemma 8's closed forms (trees / cliques: every evaluated
    pair is a ccp): star (n-1) 2^(n-2), clique (3^n - 2^(n+1) + 1) / 2."""
    from paper_2202_13511_b200 import mpdp
    with mpdp.Context(device=0, workspace_bytes=6 << 30) as c:
        for n in (20, 25):
            r = c.mpdp_optimize(W.star(n, 3))
            assert r.memo_kind == 4
            assert r.pairs_evaluated == r.ccp_pairs == (n - 1) * 2 ** (n - 2)
            assert r.csg_count == 2 ** (n - 1) + n - 1
            assert r.level_pairs[2:] == [(k - 1) * __import__("math").comb(n - 1, k - 1) for k in range(2, n + 1)]
        for n in (16, 18):
            r = c.mpdp_optimize(W.clique(n, 3))
            assert r.memo_kind == 2
            assert r.pairs_evaluated == r.ccp_pairs == (3 ** n - 2 ** (n + 1) + 1) // 2
            assert r.csg_count == 2 ** n - 1


@pytest.mark.parametrize("topo,n,seed", [("star", 14, 0), ("clique", 11, 1), ("cycle", 13, 2),
                                         ("random", 12, 3), ("snowflake", 16, 4), ("chain", 15, 5),
                                         ("star", 20, 6)])
def test_nccl_self_communicator(topo, n, seed):
    """MPDP_FLAG_NCCL_SELF: a real 1-rank NCCL communicator; every level goes
    through the sharded level loop with the in-place ncclAllGather exchange and
    the final ncclAllReduce of the counters.  Results equal the oracle's."""
    from paper_2202_13511_b200 import mpdp
    g = W.generate(topo, n, seed)
    with mpdp.Context(device=0, workspace_bytes=1 << 30, flags=mpdp.FLAG_NCCL_SELF) as c:
        r = c.mpdp_optimize(g)
        check(r, O.optimize(g), g)
        assert r.gpu_launches >= n            # one launch per level + extraction (+ k_init)


def test_nccl_self_log_shows_collectives():
    """The NCCL path really executes: a child process with NCCL_DEBUG=INFO
    (subsystems INIT and COLL) logs the communicator init and the AllGather /
    AllReduce calls of one sharded query."""
    code = ("import sys; sys.path.insert(0, %r)\n"
            "import workload as W\n"
            "from paper_2202_13511_b200 import mpdp\n"
            "with mpdp.Context(device=0, workspace_bytes=1 << 30, flags=mpdp.FLAG_NCCL_SELF) as c:\n"
            "    r = c.mpdp_optimize(W.star(12, 0))\n"
            "    print('COST', r.cost)\n" % ROOT)
    env = dict(os.environ, NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT,COLL")
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
    log = p.stdout + p.stderr
    assert p.returncode == 0, log[-2000:]
    assert "COST" in log
    assert "Init COMPLETE" in log or "init.cc" in log, log[-2000:]
    assert "AllGather" in log and "AllReduce" in log, log[-2000:]


@pytest.mark.parametrize("topo,n,seed,extra", [("cycle", 20, 0, None), ("random", 20, 0, None),
                                               ("random", 20, 7, 0.15), ("random", 19, 11, 0.4)])
def test_general_graphs_full_size(topo, n, seed, extra):
    """General graphs (block decomposition, Find-Blocks, CCP checks) at the
    BASELINE size n = 20 through k_dp_fused<GENERAL, MEMO_MASK>: random-20 s0 is
    the bench_all instance (1.33 G evaluated pairs, 467 M ccp)."""
    from paper_2202_13511_b200 import mpdp
    g = W.generate(topo, n, seed) if extra is None else W.random_connected(n, seed, extra=extra)
    with mpdp.Context(device=0, workspace_bytes=4 << 30) as c:
        check(c.mpdp_optimize(g), O.optimize_dpccp(g), g)


def test_nccl_self_batch_and_heuristics():
    """Multi-GPU batch (MPDP_FLAG_NCCL_SELF: a real 1-rank communicator): the
    independent queries go through the distributed path (per-rank share on the
    single-GPU kernels, results allgathered over NCCL); UnionDP / IDP2 on such
    a context give the single-GPU context's plans."""
    from paper_2202_13511_b200 import mpdp
    gs = [W.generate(t, n, 40 + i) for i, (t, n) in enumerate(
        [("star", 9), ("snowflake", 16), ("chain", 20), ("clique", 9), ("cycle", 12), ("star", 15)])]
    g = W.snowflake(200, 3)
    with mpdp.Context(device=0, workspace_bytes=1 << 30) as one:
        ref = [one.mpdp_optimize_uniondp(g, k=20, t=12), one.mpdp_optimize(g, algo="IDP2_MPDP", k=12)]
    with mpdp.Context(device=0, workspace_bytes=1 << 30, flags=mpdp.FLAG_NCCL_SELF) as c:
        for q, r in zip(gs, c.mpdp_optimize_batch(gs)):
            o = O.optimize(q)
            assert r.cost == o.cost and r.tree() == O.tree_of(o.nodes)
            assert (r.csg_count, r.ccp_pairs, r.pairs_evaluated) == (o.csg_count, o.ccp_pairs, o.pairs_evaluated)
        got = [c.mpdp_optimize_uniondp(g, k=20, t=12), c.mpdp_optimize(g, algo="IDP2_MPDP", k=12)]
    for a, b in zip(ref, got):
        assert a.cost == b.cost and a.tree() == b.tree() and a.pairs_evaluated == b.pairs_evaluated


@pytest.mark.parametrize("n,seed", [(16, 0), (18, 1), (20, 2), (22, 3), (24, 4), (26, 5), (20, 6)])
def test_cluster_tree_kernel(n, seed):
    """Sparse trees with 513..6144 sets per level run on one thread-block
    cluster (k_dp_tree_cluster: cluster barrier between levels, one global
    reservation per CTA for the next level list); results equal the oracle's
    and the multi-CTA list kernel's (MPDP_FLAG_NO_SMALL), with and without
    composite leaf costs."""
    from paper_2202_13511_b200 import mpdp
    g = W.snowflake(n, seed)
    if seed % 2:
        g.leaf_cost = [float((5 * i) % 7) for i in range(g.n)]
    o = O.optimize(g)
    with mpdp.Context(device=0, workspace_bytes=2 << 30) as c:
        r = c.mpdp_optimize(g)
        if 512 < max(o.level_csg) <= 6144:               # the cluster kernel's range: one launch
            assert r.gpu_launches == 1 and r.memo_kind == 1
        check(r, o, g)
        check(c.mpdp_optimize(g), o, g)                  # repeated: counters and lists reset
    with mpdp.Context(device=0, workspace_bytes=2 << 30, flags=mpdp.FLAG_NO_SMALL) as c:
        check(c.mpdp_optimize(g), o, g)
