"""Host logic of the sharded (multi-GPU) level loop, exercised by 2 processes
over torch.distributed/gloo on CPU:

* rank 0 creates the NCCL unique id through the C ABI and broadcasts it;
* every level's colex-rank space is split by mpdp_share into equal contiguous
  segments that cover it exactly once across ranks;
* the in-place allgather of equal segments over the padded per-level dense
  memo layout (dense_off[k] = sum_j<k (C(n,j) + W)) rebuilds on every rank
  exactly the array a single rank would hold.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, shard_min, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2202_13511_b200 import build, mpdp
        mpdp.load_library()
        # ---- NCCL unique id bootstrap (the same call bench.py makes)
        uid = torch.zeros(128, dtype=torch.uint8)
        have = torch.zeros(1, dtype=torch.int32)
        if rank == 0:
            try:
                uid = torch.tensor(list(mpdp.mpdp_nccl_get_unique_id()), dtype=torch.uint8)
                have[0] = 1
            except Exception:
                have[0] = 0
        dist.broadcast(have, 0)
        dist.broadcast(uid, 0)
        # ---- shares and the padded layout
        off, layout = 0, {}
        for k in range(2, n + 1):
            C = math.comb(n, k)
            layout[k] = (off, C)
            off += C + world
        full = np.full(off, -1.0)
        mine = np.full(off, -1.0)
        shares = []
        for k in range(2, n + 1):
            o, C = layout[k]
            sharded = C >= shard_min
            lo, hi = mpdp.mpdp_share(C, rank, world) if sharded else (0, C)
            shares.append((k, lo, hi, sharded))
            idx = np.arange(C)
            full[o:o + C] = k * 1e6 + idx                     # what one rank alone would hold
            mine[o + lo:o + hi] = k * 1e6 + np.arange(lo, hi)  # what this rank computes
            if sharded:                                     # in-place allgather of equal segments
                seg = (C + world - 1) // world
                t = torch.from_numpy(mine[o + rank * seg:o + (rank + 1) * seg].copy())
                parts = [torch.empty(seg, dtype=torch.float64) for _ in range(world)]
                dist.all_gather(parts, t)
                mine[o:o + world * seg] = torch.cat(parts).numpy()
        ok_arrays = bool(np.array_equal(np.concatenate([mine[o:o + C] for o, C in layout.values()]),
                                        np.concatenate([full[o:o + C] for o, C in layout.values()])))
        q.put((rank, bool(have[0]), bytes(uid.tolist()), shares, ok_arrays))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,world,shard_min", [(25, 2, 1 << 14), (13, 2, 0), (9, 3, 0)])
def test_sharded_host_logic_gloo(n, world, shard_min):
    from paper_2202_13511_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, shard_min, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    res.sort()
    uids = {r[2] for r in res}
    assert len(uids) == 1                                   # everyone got rank 0's id
    if res[0][1]:
        assert any(b != 0 for b in res[0][2])
    for _, _, _, _, ok in res:
        assert ok                                           # every replica complete after the exchange
    per_level = {}
    for _, _, _, shares, _ in res:
        for k, lo, hi, sharded in shares:
            per_level.setdefault(k, []).append((lo, hi, sharded))
    for k, parts in per_level.items():
        C = math.comb(n, k)
        if parts[0][2]:
            parts.sort()
            assert parts[0][0] == 0 and parts[-1][1] == C
            for a, b in zip(parts, parts[1:]):
                assert a[1] == b[0]                         # contiguous, disjoint
        else:
            assert all(lo == 0 and hi == C for lo, hi, _ in parts)   # redundant small level


def _peer_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2202_13511_b200 import mpdp
        # a stand-in record (the real one holds this rank's CUDA IPC handle and
        # workspace size, mpdp_ctx_peer_record): 64 handle bytes + the size
        rec = bytes([rank + 1] * 64) + (1 << 30).to_bytes(8, "little")
        recs = mpdp.gather_peer_records(rec)
        bad = None
        try:
            mpdp.gather_peer_records(b"short")
        except mpdp.MPDPError as e:
            bad = e.status
        q.put((rank, recs, bad))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_fused_exchange_peer_records_gloo(world):
    """Host logic of the fused peer exchange (MPDP_FLAG_FUSED_EXCHANGE across
    GPUs): every rank gathers every rank's peer record, in rank order, before
    mpdp_ctx_open_peers maps the peers' workspaces; malformed records are
    rejected on every rank."""
    from paper_2202_13511_b200 import mpdp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    want = [bytes([r + 1] * 64) + (1 << 30).to_bytes(8, "little") for r in range(world)]
    for rank, recs, bad in res:
        assert recs == want
        assert all(len(r) == mpdp.PEER_RECORD_BYTES for r in recs)
        assert bad == mpdp.ERR_INVALID_ARGUMENT
