#!/usr/bin/env python3
"""Benchmark: exact MPDP join-order optimisation on B200 (BASELINE.json metric:
"exact join-order optimization time (ms) and join pairs/s at 1/2/4/8 B200").

One step = one exact optimisation of one synthetic query of the bench workload
(default star-25, BASELINE config 3 -- the configuration the metric's 1/2/4/8-GPU
scaling is quoted on), seeds cycling 0..2.  `value` = join pairs evaluated per
second (unordered, reading R3) with the query already staged in HBM, timed with
CUDA events on the context's stream around the whole level loop; `e2e` = the
same metric through mpdp_optimize() with host buffers (H2D of the graph, D2H of
the plan inside the timed region).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload star-25]
                    [--impl reference]

--impl reference times the CPU oracle (DPccp, oracle/) as it stands on the
host, one bounded query per step.  Multi-GPU (N > 1, torchrun): every rank
works on the same query; each level's colex ranks are split across ranks and
the new memo segments are allgathered in place over NCCL after the level
(DESIGN.md §8).  value = pairs of the optimised queries / max-over-ranks device
time (strong scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workload as W  # noqa: E402

METRIC = "exact join-order optimisation: join pairs evaluated/s (MPDP)"
UNIT = "pairs/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="star-25")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--seeds", type=int, default=3)
    return ap.parse_args()


def workload_graphs(name, nseeds, seed_offset=0):
    topo, n = name.rsplit("-", 1)
    return [W.generate(topo, int(n), seed_offset + s) for s in range(nseeds)]


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ------------------------------------------------------------------ oracle legs
def oracle_step(g):
    from oracle import pyoracle as O
    t = time.perf_counter()
    r = O.optimize_dpccp(g)
    dt = time.perf_counter() - t
    return r, dt


def cpu_baseline(graph):
    """The oracle as it stands (single-threaded DPccp), one full query."""
    r, dt = oracle_step(graph)
    return {"value": r.pairs_evaluated / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"1 full {graph.name} query, DPccp (oracle/oracle.c), {dt:.2f} s on 1 host core",
            "seconds": dt}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    topo, n = args.workload.rsplit("-", 1)
    n = int(n)
    # bound the whole run to a few minutes: shrink the instance until one step fits
    budget = 150.0 / max(1, args.steps + args.warmup)
    probe_n = min(n, 20)
    _, dt = oracle_step(W.generate(topo, probe_n, 0))
    est = dt
    m = probe_n
    while m < n and est * (2.2 if topo != "clique" else 3.0) <= budget:
        m += 1
        est *= (2.2 if topo != "clique" else 3.0)
    graphs = [W.generate(topo, m, s) for s in range(args.seeds)]
    for i in range(args.warmup):
        oracle_step(graphs[i % len(graphs)])
    times, pairs = [], 0
    for i in range(args.steps):
        r, dt = oracle_step(graphs[i % len(graphs)])
        times.append(dt)
        pairs += r.pairs_evaluated
    tot = sum(times)
    val = pairs / tot
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{topo}-{m}", "requested_workload": args.workload,
                       "seeds": args.seeds, "oracle": "DPccp"},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"{args.steps} x {topo}-{m} queries (bounded from {args.workload})"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm
def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2202_13511_b200 import mpdp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    graphs = workload_graphs(args.workload, args.seeds)           # every rank: the same queries
    topo_is_tree = args.workload.rsplit("-", 1)[0] in ("star", "snowflake", "chain")
    n = graphs[0].n
    ws = 6 << 30 if n >= 24 else 2 << 30
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)    # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    if world > 1:
        # sharded multi-GPU mode: one communicator per process, the same query on
        # every rank, each level's colex ranks split across ranks
        uid = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            uid.copy_(torch.tensor(list(mpdp.mpdp_nccl_get_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        ctx = mpdp.Context(device=local, workspace_bytes=ws, rank=rank, world=world,
                           nccl_unique_id=bytes(uid.cpu().tolist()))
    else:
        ctx = mpdp.Context(device=local, workspace_bytes=ws)      # production path: fused kernel
    stream = ctx.stream                       # the stream every library kernel runs on
    # ---- warm-up
    for i in range(args.warmup):
        ctx.mpdp_optimize(graphs[i % len(graphs)])
    # ---- timed device-resident steps: query staged, time the level loop
    step_ms, pairs_total, probes_total, launches, sets_total = [], 0, 0, 0, 0
    kernel_ms, kernel_launches = 0.0, 0
    barrier()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            g = graphs[i % len(graphs)]
            ctx.mpdp_stage(g)
            flush.fill_(i & 0xff)                     # flush L2 between steps (untimed)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctx.mpdp_run()
            e1.record(stream)
            r = ctx.mpdp_fetch()
            memo_kind = r.memo_kind
            step_ms.append(e0.elapsed_time(e1))
            pairs_total += r.pairs_evaluated
            probes_total += r.probes
            sets_total += r.csg_count - g.n
            launches += r.gpu_launches
            kernel_ms += r.eval_ms                    # CUDA events around the level-loop kernel
            kernel_launches += r.eval_launches
        barrier()
    total_ms = sum(step_ms)
    if world > 1:                             # max over ranks; the ranks share each query
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    pairs_all = float(pairs_total)            # pairs of the queries the job optimised
    value = pairs_all / (total_ms / 1e3)

    # ---- e2e: public API with host buffers, H2D + D2H inside the timed region
    e2e_times, e2e_pairs, h2d, d2h = [], 0, 0, 0
    barrier()
    for i in range(args.steps):
        g = graphs[i % len(graphs)]
        flush.fill_(i & 0xff)
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = ctx.mpdp_optimize(g)
        e2e_times.append(time.perf_counter() - t)
        e2e_pairs += r.pairs_evaluated
        h2d, d2h = r.h2d_bytes, r.d2h_bytes
    barrier()
    e2e_s = sum(e2e_times)
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = e2e_pairs / e2e_s

    # ---- roofline of the dominant kernel: the whole-query level-loop kernel
    # (one launch per query does unrank, filter, compaction, evaluate, min and
    # memo scatter for every level; k_dp_list for tree queries, k_dp_fused
    # otherwise).  DESIGN.md §6: perfect-hash memo = 8 B cost per probe + per
    # connected set 16 B level-list write + read (the compaction of P:889) and
    # 8 B cost + 4 B left insert; open-addressing memo = 16 B slot per probe,
    # per set list write + read + 16 B slot + left.
    msz = 4 if n <= 32 else 8
    if memo_kind == 4:                        # star: no level lists; card(S \ max) read + cost/card/left write
        alg_bytes = 8 * probes_total + sets_total * (8 + 8 + 8 + 4)
    elif memo_kind in (1, 2, 3):              # colex-rank or bitmask-indexed arrays: same bytes
        alg_bytes = 8 * probes_total + sets_total * (16 + 8 + 4)
    else:
        alg_bytes = 16 * probes_total + sets_total * (2 * msz + 16 + msz)
    kernel_name = {4: "k_dp_star (star queries: closed-form level indexing, one launch per query)",
                   3: "k_dp_small (single CTA, shared-memory memo)"}.get(memo_kind) or (
        "k_dp_list (tree queries: whole level loop, one launch per query)" if topo_is_tree
        else "k_dp_fused / k_dp_clique (whole level loop, one launch per query)")
    peak, peak_kind = measured_peaks()
    kern_s = kernel_ms / 1e3
    achieved = alg_bytes / kern_s / 1e9 if kern_s > 0 else 0.0
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tfile):
        traffic = json.load(open(tfile)).get(args.workload)
    roof = {"bound": "hbm",
            "kernel": kernel_name,
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic.get("dram_bytes_per_launch") if traffic else None,
            "traffic_source": traffic.get("source") if traffic else None,
            "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)",
            "memo": {1: "perfect-hash (colex rank)", 2: "bitmask-indexed (MEMO_MASK)",
                     3: "shared-memory bitmask memo (single CTA)",
                     4: "star memo (leaf-set colex rank, C(n-1,k-1) per level)"}.get(
                memo_kind, "murmur3 open addressing"),
            "algorithmic_bytes_per_launch": alg_bytes / max(1, kernel_launches),
            "avg_launch_ms": kernel_ms / max(1, kernel_launches),
            "share_of_step": kernel_ms / max(1e-9, sum(step_ms))}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": args.workload, "seeds": args.seeds,
                       "pairs_per_query": pairs_total / args.steps,
                       "l2": "flushed between steps (256 MiB write)",
                       "parallelism": f"level-sharded x{world} (NCCL allgather per level)" if world > 1 else "single-gpu",
                       "opt_time_ms_median": statistics.median(step_ms)},
            "clocks": clk.summary(), "roofline": roof,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": 1e3 * e2e_s / args.steps},
            "gpu_launches": launches}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(graphs[0])
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
