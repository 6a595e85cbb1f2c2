"""ctypes wrapper around oracle/liboracle.so.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  The product package
(paper_2202_13511_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from typing import List, Optional

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(HERE, "oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-fPIC", "-shared",
                               "-ffp-contract=off", "-o", LIB_PATH, src, "-lm"])
    return LIB_PATH


class _Graph(C.Structure):
    _fields_ = [("n", C.c_uint32), ("card", C.POINTER(C.c_double)),
                ("n_edges", C.c_uint32), ("edges", C.POINTER(C.c_uint32)),
                ("sel", C.POINTER(C.c_double)), ("leaf_cost", C.POINTER(C.c_double))]


class _Node(C.Structure):
    _fields_ = [("left", C.c_int32), ("right", C.c_int32), ("relation", C.c_int32),
                ("set", C.c_uint64), ("card", C.c_double), ("cost", C.c_double)]


class _Result(C.Structure):
    _fields_ = [("nodes", C.POINTER(_Node)), ("capacity", C.c_uint32),
                ("n_nodes", C.c_uint32), ("cost", C.c_double),
                ("csg_count", C.c_uint64), ("ccp_pairs", C.c_uint64),
                ("pairs_evaluated", C.c_uint64),
                ("level_csg", C.POINTER(C.c_uint64)), ("level_ccp", C.POINTER(C.c_uint64)),
                ("level_pairs", C.POINTER(C.c_uint64)), ("dpsize_checks", C.c_uint64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        G = C.POINTER(_Graph)
        u64, i32, dbl = C.c_uint64, C.c_int, C.c_double
        for name, res, args in [
            ("oracle_neighbours", u64, [G, u64]),
            ("oracle_grow", u64, [G, u64, u64]),
            ("oracle_connected", i32, [G, u64]),
            ("oracle_is_ccp", i32, [G, u64, u64]),
            ("oracle_card", dbl, [G, u64]),
            ("oracle_blocks", i32, [G, u64, C.POINTER(u64), i32]),
            ("oracle_mpdp_pairs", u64, [G, u64]),
            ("oracle_unrank_colex", u64, [C.c_uint32, C.c_uint32, u64]),
            ("oracle_optimize_definition", i32, [G, C.POINTER(_Result)]),
            ("oracle_optimize_dpccp", i32, [G, C.POINTER(_Result)]),
            ("oracle_optimize_dpsize", i32, [G, C.POINTER(_Result)]),
            ("oracle_bruteforce", i32, [G, C.POINTER(dbl), C.POINTER(u64)]),
            ("oracle_counters", i32, [G, C.POINTER(u64), C.POINTER(u64)]),
        ]:
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"{what}: oracle status {code}")
        self.code = code


@dataclass
class PlanNode:
    left: int
    right: int
    relation: int
    set: int
    card: float
    cost: float


@dataclass
class OracleResult:
    cost: float
    nodes: List[PlanNode]
    csg_count: int
    ccp_pairs: int
    pairs_evaluated: int
    level_csg: List[int]
    level_ccp: List[int]
    level_pairs: List[int]
    dpsize_checks: int = 0


class _Marshal:
    """Keeps ctypes buffers alive for the duration of a call."""

    def __init__(self, g):
        n = g.n
        self.card = (C.c_double * n)(*g.card)
        m = len(g.edges)
        flat = [x for e in g.edges for x in e]
        self.edges = (C.c_uint32 * max(1, 2 * m))(*flat)
        self.sel = (C.c_double * max(1, m))(*g.sel)
        self.leaf = (C.c_double * n)(*g.leaf_cost) if g.leaf_cost is not None else None
        self.g = _Graph(n, self.card, m, self.edges, self.sel,
                        self.leaf if self.leaf is not None else None)

    @property
    def ptr(self):
        return C.byref(self.g)


def _run(fn_name: str, g) -> OracleResult:
    L = lib()
    mg = _Marshal(g)
    n = g.n
    nodes = (_Node * (2 * n - 1))()
    lc, lp, lx = (C.c_uint64 * (n + 1))(), (C.c_uint64 * (n + 1))(), (C.c_uint64 * (n + 1))()
    res = _Result(nodes, 2 * n - 1, 0, 0.0, 0, 0, 0, lc, lx, lp, 0)
    st = getattr(L, fn_name)(mg.ptr, C.byref(res))
    if st != 0:
        raise OracleError(st, fn_name)
    out = [PlanNode(x.left, x.right, x.relation, x.set, x.card, x.cost)
           for x in nodes[:res.n_nodes]]
    return OracleResult(res.cost, out, res.csg_count, res.ccp_pairs, res.pairs_evaluated,
                        list(lc), list(lx), list(lp), res.dpsize_checks)


def optimize_definition(g) -> OracleResult:
    return _run("oracle_optimize_definition", g)


def optimize_dpccp(g) -> OracleResult:
    return _run("oracle_optimize_dpccp", g)


def optimize_dpsize(g) -> OracleResult:
    return _run("oracle_optimize_dpsize", g)


def optimize(g) -> OracleResult:
    """The oracle used for parity: the plain definition up to n = 16, DPccp
    above (pinned equal to the definition on every size both can run)."""
    return optimize_definition(g) if g.n <= 16 else optimize_dpccp(g)


def bruteforce(g):
    L = lib()
    mg = _Marshal(g)
    c, t = C.c_double(), C.c_uint64()
    st = L.oracle_bruteforce(mg.ptr, C.byref(c), C.byref(t))
    if st != 0:
        raise OracleError(st, "oracle_bruteforce")
    return c.value, t.value


def counters(g):
    L = lib()
    mg = _Marshal(g)
    lc, lp = (C.c_uint64 * (g.n + 1))(), (C.c_uint64 * (g.n + 1))()
    st = L.oracle_counters(mg.ptr, lc, lp)
    if st != 0:
        raise OracleError(st, "oracle_counters")
    return list(lc), list(lp)


def grow(g, source: int, restriction: int) -> int:
    return lib().oracle_grow(_Marshal(g).ptr, source, restriction)


def connected(g, S: int) -> bool:
    return bool(lib().oracle_connected(_Marshal(g).ptr, S))


def is_ccp(g, S1: int, S2: int) -> bool:
    return bool(lib().oracle_is_ccp(_Marshal(g).ptr, S1, S2))


def card(g, S: int) -> float:
    return lib().oracle_card(_Marshal(g).ptr, S)


def blocks(g, S: int) -> List[int]:
    buf = (C.c_uint64 * 64)()
    nb = lib().oracle_blocks(_Marshal(g).ptr, S, buf, 64)
    return list(buf[:nb])


def mpdp_pairs(g, S: int) -> int:
    return lib().oracle_mpdp_pairs(_Marshal(g).ptr, S)


def neighbours(g, S: int) -> int:
    return lib().oracle_neighbours(_Marshal(g).ptr, S)


def unrank_colex(n: int, k: int, r: int) -> int:
    return lib().oracle_unrank_colex(n, k, r)


def tree_of(nodes: List[PlanNode]) -> Optional[tuple]:
    """Canonical nested-tuple form of a post-order plan (root last)."""
    if not nodes:
        return None

    def rec(i):
        x = nodes[i]
        if x.relation >= 0:
            return x.relation
        return (rec(x.left), rec(x.right))
    return rec(len(nodes) - 1)
