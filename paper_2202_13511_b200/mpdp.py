"""Thin ctypes binding of include/mpdp.h (argument marshalling only).

Every step of the DP runs in the CUDA kernels of libmpdp.so; there is no CPU
path.  If the shared library is missing or no CUDA device is present, the
calls raise instead of falling back.  PyTorch is used for plumbing only: the
workspace is a torch CUDA tensor and the context runs on torch's current
stream.
"""
from __future__ import annotations

import array
import ctypes as C
import itertools
import os
from dataclasses import dataclass, field
from typing import List, Optional

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MPDP_LIBRARY", os.path.join(HERE, "libmpdp.so"))

# mpdp_status
OK, ERR_INVALID_ARGUMENT, ERR_DISCONNECTED, ERR_CAPACITY, ERR_TIMEOUT, ERR_OOM, \
    ERR_CUDA, ERR_NCCL, ERR_INTERNAL, ERR_UNSUPPORTED = range(10)
# mpdp_algo
ALGOS = {"DPSIZE_REF": 0, "MPDP": 1, "IDP2_MPDP": 2, "UNIONDP_MPDP": 3}


class mpdp_query_graph(C.Structure):
    _fields_ = [("n", C.c_uint32), ("cardinalities", C.POINTER(C.c_double)),
                ("n_edges", C.c_uint32), ("edges", C.POINTER(C.c_uint32)),
                ("selectivities", C.POINTER(C.c_double)),
                ("leaf_costs", C.POINTER(C.c_double))]


class mpdp_plan_node(C.Structure):
    _fields_ = [("left", C.c_int32), ("right", C.c_int32), ("relation", C.c_int32),
                ("reserved", C.c_uint32), ("set", C.c_uint64),
                ("cardinality", C.c_double), ("cost", C.c_double)]


class mpdp_result(C.Structure):
    _fields_ = [("nodes", C.POINTER(mpdp_plan_node)), ("capacity", C.c_uint32),
                ("n_nodes", C.c_uint32), ("root", C.c_uint32), ("gpu_launches", C.c_uint32),
                ("cost", C.c_double), ("pairs_evaluated", C.c_uint64),
                ("ccp_pairs", C.c_uint64), ("csg_count", C.c_uint64),
                ("level_csg", C.POINTER(C.c_uint64)), ("level_ccp", C.POINTER(C.c_uint64)),
                ("level_pairs", C.POINTER(C.c_uint64)), ("time_ms", C.c_double),
                ("probes", C.c_uint64), ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
                ("enum_ms", C.c_double), ("eval_ms", C.c_double),
                ("enum_launches", C.c_uint32), ("eval_launches", C.c_uint32),
                ("memo_kind", C.c_uint32), ("inner_calls", C.c_uint32),
                ("level_ms", C.POINTER(C.c_double))]


class mpdp_ctx_config(C.Structure):
    _fields_ = [("device", C.c_int), ("rank", C.c_int), ("world", C.c_int),
                ("nccl_unique_id", C.c_void_p), ("cuda_stream", C.c_void_p),
                ("mem_budget_bytes", C.c_uint64), ("timeout_ms", C.c_double),
                ("workspace", C.c_void_p), ("workspace_bytes", C.c_uint64),
                ("flags", C.c_uint32), ("load_factor", C.c_double)]

FLAG_FORCE_WIDE_MASKS = 1
FLAG_PROFILE_KERNELS = 2
FLAG_HASH_MEMO = 4
FLAG_NO_GRAPH = 8
FLAG_NO_FUSED = 16
FLAG_SIMULATE_WORLD = 32
FLAG_SHARD_ALL_LEVELS = 64
FLAG_RECORD_SUBPROBLEMS = 128
FLAG_DPSUB_ENUM = 256
FLAG_RANK_MEMO = 512
FLAG_NO_SMALL = 1024
FLAG_NO_CCC = 2048
FLAG_NO_STAR = 4096
FLAG_NCCL_SELF = 8192
FLAG_FUSED_EXCHANGE = 16384
PEER_RECORD_BYTES = 72


EXPORTS = ["mpdp_ctx_create", "mpdp_ctx_destroy", "mpdp_optimize", "mpdp_optimize_batch", "mpdp_stage",
           "mpdp_run", "mpdp_fetch", "mpdp_last_error", "mpdp_status_string", "mpdp_abi_version",
           "mpdp_nccl_get_unique_id", "mpdp_share", "mpdp_debug_trace", "mpdp_subproblem_count",
           "mpdp_subproblem_get", "mpdp_heuristic_optimize", "mpdp_debug_level_span",
           "mpdp_debug_df_stats", "mpdp_heuristic_optimize_t", "mpdp_optimize_uniondp",
           "mpdp_ctx_peer_record", "mpdp_ctx_open_peers"]

_lib = None


def load_library(path: str = LIB_PATH):
    """Load libmpdp.so (raises OSError if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise OSError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(path)
    P = C.c_void_p
    sig = {
        "mpdp_ctx_create": (C.c_int, [C.POINTER(mpdp_ctx_config), C.POINTER(P)]),
        "mpdp_ctx_destroy": (C.c_int, [P]),
        "mpdp_optimize": (C.c_int, [P, C.POINTER(mpdp_query_graph), C.c_int, C.c_uint32,
                                    C.POINTER(mpdp_result)]),
        "mpdp_optimize_batch": (C.c_int, [P, C.POINTER(mpdp_query_graph), C.c_uint32, C.POINTER(mpdp_result)]),
        "mpdp_stage": (C.c_int, [P, C.POINTER(mpdp_query_graph)]),
        "mpdp_run": (C.c_int, [P]),
        "mpdp_fetch": (C.c_int, [P, C.POINTER(mpdp_result)]),
        "mpdp_last_error": (C.c_char_p, [P]),
        "mpdp_status_string": (C.c_char_p, [C.c_int]),
        "mpdp_abi_version": (C.c_int, []),
        "mpdp_nccl_get_unique_id": (C.c_int, [P]),
        "mpdp_share": (None, [C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_uint64),
                              C.POINTER(C.c_uint64)]),
        "mpdp_debug_level_span": (C.c_int, [P, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int]),
        "mpdp_debug_df_stats": (C.c_int, [P, C.POINTER(C.c_uint64), C.c_int]),
        "mpdp_optimize_uniondp": (C.c_int, [P, C.POINTER(mpdp_query_graph), C.c_uint32, C.c_uint32,
                                            C.POINTER(mpdp_result)]),
        "mpdp_ctx_peer_record": (C.c_int, [P, P]),
        "mpdp_ctx_open_peers": (C.c_int, [P, P]),
    }
    for name, (res, args) in sig.items():
        if not hasattr(L, name):           # an older build (A/B timing via MPDP_LIBRARY)
            continue
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


class MPDPError(RuntimeError):
    def __init__(self, status: int, msg: str):
        name = load_library().mpdp_status_string(status).decode()
        super().__init__(f"{name}: {msg}")
        self.status = status


@dataclass
class PlanNode:
    left: int
    right: int
    relation: int
    set: int
    cardinality: float
    cost: float


class Result:
    """One optimisation result (mpdp_result).  The plan nodes are converted
    from the C array on first access (`nodes`): building 2n-1 Python objects
    per call was most of the binding's per-query cost."""
    _FIELDS = ("cost", "pairs_evaluated", "ccp_pairs", "csg_count", "level_csg", "level_ccp", "level_pairs",
               "time_ms", "gpu_launches", "probes", "h2d_bytes", "d2h_bytes", "enum_ms", "eval_ms",
               "enum_launches", "eval_launches", "memo_kind", "level_ms", "inner_calls")

    def __init__(self, cost, nodes, pairs_evaluated, ccp_pairs, csg_count, level_csg, level_ccp, level_pairs,
                 time_ms, gpu_launches, probes=0, h2d_bytes=0, d2h_bytes=0, enum_ms=0.0, eval_ms=0.0,
                 enum_launches=0, eval_launches=0, memo_kind=0, level_ms=None, inner_calls=0):
        self.cost, self.pairs_evaluated, self.ccp_pairs, self.csg_count = cost, pairs_evaluated, ccp_pairs, csg_count
        self._lv = [level_csg, level_ccp, level_pairs]   # lists, or ctypes arrays converted lazily
        self.time_ms, self.gpu_launches, self.probes = time_ms, gpu_launches, probes
        self.h2d_bytes, self.d2h_bytes, self.enum_ms, self.eval_ms = h2d_bytes, d2h_bytes, enum_ms, eval_ms
        self.enum_launches, self.eval_launches, self.memo_kind = enum_launches, eval_launches, memo_kind
        self._lv.append(level_ms if level_ms is not None else [])
        self.inner_calls = inner_calls
        self._nodes = nodes                # a list, or (ctypes node array, count) converted lazily

    @property
    def nodes(self) -> List[PlanNode]:
        if isinstance(self._nodes, tuple):
            arr, cnt = self._nodes
            self._nodes = [PlanNode(x.left, x.right, x.relation, x.set, x.cardinality, x.cost) for x in arr[:cnt]]
        return self._nodes

    @nodes.setter
    def nodes(self, v):
        self._nodes = v

    def _level(self, i):
        x = self._lv[i]
        if x is not None and not isinstance(x, list):
            x = self._lv[i] = list(x)
        return x

    level_csg = property(lambda self: self._level(0), lambda self, v: self._lv.__setitem__(0, v))
    level_ccp = property(lambda self: self._level(1), lambda self, v: self._lv.__setitem__(1, v))
    level_pairs = property(lambda self: self._level(2), lambda self, v: self._lv.__setitem__(2, v))
    level_ms = property(lambda self: self._level(3), lambda self, v: self._lv.__setitem__(3, v))

    def __repr__(self):
        return "Result(" + ", ".join(f"{f}={getattr(self, f)!r}" for f in ("cost", "pairs_evaluated", "csg_count",
                                                                          "memo_kind", "time_ms")) + ")"

    def tree(self):
        """Nested tuples: leaves are relation ids, internal nodes (left, right)."""
        def rec(i):
            x = self.nodes[i]
            return x.relation if x.relation >= 0 else (rec(x.left), rec(x.right))
        return rec(len(self.nodes) - 1) if self.nodes else None


class GraphArgs:
    """Marshals a workload.QueryGraph-like object (n, card, edges, sel, leaf_cost)."""

    def __init__(self, g):
        # array.array buffers (C-speed conversion of the Python lists), viewed
        # as ctypes arrays without a copy
        n, m = g.n, len(g.edges)
        self._a = [array.array("d", g.card), array.array("I", itertools.chain.from_iterable(g.edges) if m else (0, 0)),
                   array.array("d", g.sel if m else (0.0,))]
        self.card = (C.c_double * n).from_buffer(self._a[0])
        self.edges = (C.c_uint32 * max(1, 2 * m)).from_buffer(self._a[1])
        self.sel = (C.c_double * max(1, m)).from_buffer(self._a[2])
        lc = getattr(g, "leaf_cost", None)
        self.leaf = None
        if lc is not None:
            self._a.append(array.array("d", lc))
            self.leaf = (C.c_double * n).from_buffer(self._a[3])
        self.s = mpdp_query_graph(n, self.card, m, self.edges, self.sel, self.leaf)
        self.n = n

    def ref(self):
        return C.byref(self.s)


class ResultBuf:
    def __init__(self, n: int):
        self.n = n
        self.nodes = (mpdp_plan_node * (2 * n - 1))()
        self.lc = (C.c_uint64 * (n + 1))()
        self.lx = (C.c_uint64 * (n + 1))()
        self.lp = (C.c_uint64 * (n + 1))()
        self.s = mpdp_result(self.nodes, 2 * n - 1)
        self.lt = (C.c_double * (n + 1))()
        self.s.level_csg, self.s.level_ccp, self.s.level_pairs = self.lc, self.lx, self.lp
        self.s.level_ms = self.lt

    def ref(self):
        return C.byref(self.s)

    def to_result(self) -> Result:
        r = self.s
        nodes = (self.nodes, r.n_nodes)   # converted on first access (Result.nodes)
        return Result(r.cost, nodes, r.pairs_evaluated, r.ccp_pairs, r.csg_count,
                      self.lc, self.lx, self.lp, r.time_ms, r.gpu_launches,
                      r.probes, r.h2d_bytes, r.d2h_bytes, r.enum_ms, r.eval_ms,
                      r.enum_launches, r.eval_launches, r.memo_kind, self.lt, r.inner_calls)


class Context:
    """One mpdp_ctx on one GPU.  The workspace is a torch uint8 CUDA tensor
    (torch = device-memory plumbing); the context runs on torch's current stream."""

    def __init__(self, device: int = 0, workspace_bytes: int = 4 << 30, timeout_ms: float = 0.0,
                 use_torch: bool = True, stream: Optional[int] = None, flags: int = 0,
                 load_factor: float = 0.0, rank: int = 0, world: int = 1,
                 nccl_unique_id: Optional[bytes] = None):
        L = load_library()
        self._ws = None
        self.stream = None
        ws_ptr, stream_ptr = None, stream
        # the fused peer exchange across GPUs maps the workspace of every rank
        # through CUDA IPC, which needs a library-allocated workspace
        peers = world > 1 and (flags & FLAG_FUSED_EXCHANGE) and not (flags & FLAG_SIMULATE_WORLD)
        if use_torch:
            import torch
            if not torch.cuda.is_available():
                raise MPDPError(ERR_CUDA, "no CUDA device (this library has no CPU path)")
            torch.cuda.set_device(device)
            if not peers:
                self._ws = torch.empty(workspace_bytes, dtype=torch.uint8, device=f"cuda:{device}")
                torch.cuda.synchronize(device)
                ws_ptr = self._ws.data_ptr()
            if stream_ptr is None:
                # a dedicated torch stream (the legacy default stream's handle is 0,
                # which the C ABI reads as "create your own")
                self.stream = torch.cuda.Stream(device=device)
                stream_ptr = self.stream.cuda_stream
        self._uid = (C.c_char * 128).from_buffer_copy(nccl_unique_id) if nccl_unique_id else None
        cfg = mpdp_ctx_config(device, rank, world, C.cast(self._uid, C.c_void_p) if self._uid else None,
                              stream_ptr, workspace_bytes, timeout_ms,
                              ws_ptr, workspace_bytes if ws_ptr else 0, flags, load_factor)
        h = C.c_void_p()
        st = L.mpdp_ctx_create(C.byref(cfg), C.byref(h))
        if st != OK:
            raise MPDPError(st, L.mpdp_last_error(None).decode())
        self.h = h
        self.L = L
        if peers:
            self.connect_peers()

    def peer_record(self) -> bytes:
        """This rank's MPDP_PEER_RECORD_BYTES record (IPC handle + workspace size)."""
        buf = (C.c_char * PEER_RECORD_BYTES)()
        self._check(self.L.mpdp_ctx_peer_record(self.h, C.cast(buf, C.c_void_p)))
        return bytes(buf)

    def open_peers(self, records: List[bytes]):
        """Map the other ranks' workspaces (records in rank order)."""
        blob = b"".join(records)
        buf = (C.c_char * len(blob)).from_buffer_copy(blob)
        self._check(self.L.mpdp_ctx_open_peers(self.h, C.cast(buf, C.c_void_p)))

    def connect_peers(self, group=None):
        """Exchange the peer records over torch.distributed (host plumbing) and
        open the peers."""
        self.open_peers(gather_peer_records(self.peer_record(), group))

    def _check(self, st):
        if st != OK:
            raise MPDPError(st, self.L.mpdp_last_error(self.h).decode())

    def mpdp_optimize(self, g, algo: str = "MPDP", k: int = 0) -> Result:
        ga, rb = GraphArgs(g), ResultBuf(g.n)
        self._check(self.L.mpdp_optimize(self.h, ga.ref(), ALGOS[algo], k, rb.ref()))
        return rb.to_result()

    optimize = mpdp_optimize

    def mpdp_optimize_uniondp(self, g, k: int = 25, t: int = 0) -> Result:
        """UnionDP with partition threshold t (0 = k)."""
        ga, rb = GraphArgs(g), ResultBuf(g.n)
        self._check(self.L.mpdp_optimize_uniondp(self.h, ga.ref(), k, t, rb.ref()))
        return rb.to_result()

    def mpdp_optimize_batch(self, graphs) -> List[Result]:
        """mpdp_optimize(MPDP) of independent queries; small tree queries share
        one launch (one CTA each)."""
        gas = [GraphArgs(g) for g in graphs]
        rbs = [ResultBuf(g.n) for g in graphs]
        ga_arr = (mpdp_query_graph * max(1, len(gas)))(*[a.s for a in gas])
        rb_arr = (mpdp_result * max(1, len(rbs)))(*[b.s for b in rbs])
        self._check(self.L.mpdp_optimize_batch(self.h, ga_arr, len(gas), rb_arr))
        out = []
        for i, b in enumerate(rbs):
            C.memmove(C.byref(b.s), C.byref(rb_arr[i]), C.sizeof(mpdp_result))
            out.append(b.to_result())
        return out

    def mpdp_stage(self, g):
        self._ga = GraphArgs(g)
        self._check(self.L.mpdp_stage(self.h, self._ga.ref()))

    def mpdp_run(self):
        self._check(self.L.mpdp_run(self.h))

    def mpdp_fetch(self) -> Result:
        rb = ResultBuf(self._ga.n)
        self._check(self.L.mpdp_fetch(self.h, rb.ref()))
        return rb.to_result()

    def close(self):
        if getattr(self, "h", None):
            self.L.mpdp_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def gather_peer_records(record: bytes, group=None) -> List[bytes]:
    """All ranks' peer records in rank order (torch.distributed object
    allgather: any backend, e.g. gloo on the host)."""
    import torch.distributed as dist
    out: List[Optional[bytes]] = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(record), group=group)
    for r in out:
        if not isinstance(r, (bytes, bytearray)) or len(r) != PEER_RECORD_BYTES:
            raise MPDPError(ERR_INVALID_ARGUMENT, "malformed peer record")
    return [bytes(r) for r in out]


def mpdp_nccl_get_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it, the caller broadcasts it)."""
    buf = (C.c_char * 128)()
    L = load_library()
    st = L.mpdp_nccl_get_unique_id(C.cast(buf, C.c_void_p))
    if st != OK:
        raise MPDPError(st, L.mpdp_last_error(None).decode())
    return bytes(buf)


def mpdp_share(total: int, rank: int, world: int):
    lo, hi = C.c_uint64(), C.c_uint64()
    load_library().mpdp_share(total, rank, world, C.byref(lo), C.byref(hi))
    return lo.value, hi.value
