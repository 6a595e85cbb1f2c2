"""Seeded synthetic join graphs with the shapes of the paper's workloads.

Topologies follow PAPER.md §7.2.1 (lines 1055-1058): star ("a single fact
relation to which other dimension relations join"), snowflake ("The maximum
depth we use is 4"), clique ("all relations have joins to all other
relations"); chain/cycle are the textbook shapes the paper mentions at P:1061.
The number recipe is DESIGN.md §"Input recipe":

* cardinalities log-uniform in [10, 1e6]                      (card = 10**U(1,6))
* tree edges are PK-FK with a random predicate factor         (sel = 10**U(-1,0) / card(child))
  "child" = the endpoint farther from the root ("We only consider
  primary key - foreign key joins ... we generate queries with selections")
* clique edges and non-tree edges of random graphs             (sel = 10**U(-1,0))

Draw order (part of the contract): cards (n draws), then topology draws,
then one predicate factor per edge in edge-list order.  Everything is plain
Python floats, serialised with repr() so JSON round trips are bit exact.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np


@dataclass
class QueryGraph:
    n: int
    card: List[float]
    edges: List[Tuple[int, int]]          # u < v, no duplicates
    sel: List[float]                      # one per edge, in (0, 1]
    leaf_cost: Optional[List[float]] = None
    name: str = ""
    meta: dict = field(default_factory=dict)

    @property
    def n_edges(self) -> int:
        return len(self.edges)

    def adjacency(self) -> List[int]:
        adj = [0] * self.n
        for u, v in self.edges:
            adj[u] |= 1 << v
            adj[v] |= 1 << u
        return adj


def _cards(rng, n):
    return [float(x) for x in 10.0 ** rng.uniform(1.0, 6.0, size=n)]


def _factors(rng, m):
    return [float(x) for x in 10.0 ** rng.uniform(-1.0, 0.0, size=m)]


def _pkfk(card, edges, child, f):
    # sel = f / card(child); child is the key side (farther from the root)
    return [f[i] / card[child[i]] for i in range(len(edges))]


def star(n: int, seed: int = 0) -> QueryGraph:
    """Hub = relation 0, edges (0, i) ("single fact relation")."""
    rng = np.random.default_rng(seed)
    card = _cards(rng, n)
    edges = [(0, i) for i in range(1, n)]
    f = _factors(rng, len(edges))
    sel = _pkfk(card, edges, [v for _, v in edges], f)
    return QueryGraph(n, card, edges, sel, name=f"star-{n}-s{seed}")


def snowflake(n: int, seed: int = 0, max_depth: int = 4) -> QueryGraph:
    """Node v >= 1 attaches to a uniformly random earlier node of depth < max_depth
    ("The maximum depth we use is 4")."""
    rng = np.random.default_rng(seed)
    card = _cards(rng, n)
    depth = [0] * n
    edges, child = [], []
    for v in range(1, n):
        cands = [u for u in range(v) if depth[u] < max_depth]
        u = cands[int(rng.integers(0, len(cands)))]
        depth[v] = depth[u] + 1
        edges.append((u, v))
        child.append(v)
    f = _factors(rng, len(edges))
    sel = _pkfk(card, edges, child, f)
    return QueryGraph(n, card, edges, sel, name=f"snowflake-{n}-s{seed}",
                      meta={"depth": depth})


def chain(n: int, seed: int = 0) -> QueryGraph:
    rng = np.random.default_rng(seed)
    card = _cards(rng, n)
    edges = [(i, i + 1) for i in range(n - 1)]
    f = _factors(rng, len(edges))
    sel = _pkfk(card, edges, [v for _, v in edges], f)
    return QueryGraph(n, card, edges, sel, name=f"chain-{n}-s{seed}")


def cycle(n: int, seed: int = 0) -> QueryGraph:
    assert n >= 3
    rng = np.random.default_rng(seed)
    card = _cards(rng, n)
    edges = [(i, i + 1) for i in range(n - 1)] + [(0, n - 1)]
    f = _factors(rng, len(edges))
    sel = _pkfk(card, edges, [v for _, v in edges], f)   # closing edge's child = n-1
    return QueryGraph(n, card, edges, sel, name=f"cycle-{n}-s{seed}")


def clique(n: int, seed: int = 0) -> QueryGraph:
    rng = np.random.default_rng(seed)
    card = _cards(rng, n)
    edges = [(u, v) for u in range(n) for v in range(u + 1, n)]
    sel = _factors(rng, len(edges))
    return QueryGraph(n, card, edges, sel, name=f"clique-{n}-s{seed}")


def random_connected(n: int, seed: int = 0, extra: float = 0.3,
                     shuffle: bool = True) -> QueryGraph:
    """Random spanning tree (PK-FK edges) plus each remaining pair with
    probability `extra` (plain predicate factor).  With shuffle=True the vertex
    numbering is a random permutation, so nothing depends on BFS numbering."""
    rng = np.random.default_rng(seed)
    card = _cards(rng, n)
    parent = [-1] + [int(rng.integers(0, v)) for v in range(1, n)]
    perm = list(range(n))
    if shuffle:
        perm = [int(x) for x in rng.permutation(n)]
    tree = set()
    child_of = {}
    for v in range(1, n):
        a, b = perm[parent[v]], perm[v]
        e = (min(a, b), max(a, b))
        tree.add(e)
        child_of[e] = b
    coins = rng.uniform(0.0, 1.0, size=n * (n - 1) // 2)
    edges = []
    ci = 0
    for u in range(n):
        for v in range(u + 1, n):
            if (u, v) in tree or coins[ci] < extra:
                edges.append((u, v))
            ci += 1
    f = _factors(rng, len(edges))
    sel = []
    for i, e in enumerate(edges):
        sel.append(f[i] / card[child_of[e]] if e in child_of else f[i])
    return QueryGraph(n, card, edges, sel, name=f"random-{n}-s{seed}")


def _fixture(n_labels, edge_list, name):
    # paper labels 1..n -> vertex ids 0..n-1; unit cards/sels (primitives only)
    edges = sorted((min(a, b) - 1, max(a, b) - 1) for a, b in edge_list)
    return QueryGraph(n_labels, [10.0] * n_labels, edges, [0.5] * len(edges), name=name)


def fig5_fixture() -> QueryGraph:
    """9-relation graph of fig:ex-join-graph; edge list from SPEC.md:154."""
    return _fixture(9, [(1, 2), (2, 3), (3, 4), (1, 4), (4, 5), (5, 9), (6, 7), (7, 8),
                        (8, 9), (6, 9)], "fig5")


def fig3_fixture() -> QueryGraph:
    """8-relation tree of fig:tree; edge list from SPEC.md:155."""
    return _fixture(8, [(1, 2), (2, 3), (2, 4), (4, 5), (5, 6), (6, 7), (6, 8)], "fig3")


_TOPOS = {"star": star, "snowflake": snowflake, "chain": chain, "cycle": cycle,
          "clique": clique, "random": random_connected}


def generate(topology: str, n: int, seed: int = 0) -> QueryGraph:
    return _TOPOS[topology](n, seed)


def to_json(g: QueryGraph) -> str:
    """SPEC.md:541-544 format (+ optional leaf_costs)."""
    d = {"relations": [{"name": f"R{i}", "cardinality": c, "selectivity": 1.0}
                       for i, c in enumerate(g.card)],
         "edges": [{"left": u, "right": v, "selectivity": s}
                   for (u, v), s in zip(g.edges, g.sel)]}
    if g.leaf_cost is not None:
        d["leaf_costs"] = list(g.leaf_cost)
    return json.dumps(d)


def from_json(text: str) -> QueryGraph:
    d = json.loads(text)
    card = [float(r["cardinality"]) * float(r.get("selectivity", 1.0)) for r in d["relations"]]
    edges = [(int(e["left"]), int(e["right"])) for e in d["edges"]]
    sel = [float(e["selectivity"]) for e in d["edges"]]
    lc = d.get("leaf_costs")
    return QueryGraph(len(card), card, edges, sel,
                      leaf_cost=[float(x) for x in lc] if lc is not None else None)
