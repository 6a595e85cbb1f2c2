"""Key metrics + hottest SASS lines of an ncu --set full report.
Usage: python tools/ncu_summary.py report.ncu-rep [top_n]"""
import csv
import io
import subprocess
import sys

KEEP = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "L2 Cache Throughput", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Theoretical Occupancy", "Achieved Occupancy", "Executed Instructions",
        "Avg. Active Threads Per Warp", "Warp Cycles Per Issued Instruction", "Grid Size", "Block Size"]


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main(rep, top=25):
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    h = rows[0]
    seen = set()
    for x in rows[1:]:
        name, unit, val = x[h.index("Metric Name")], x[h.index("Metric Unit")], x[h.index("Metric Value")]
        if name in KEEP and name not in seen:
            seen.add(name)
            print(f"  {name:38s} {val:>16s} {unit}")
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    if len(raw) > 2:
        hh, units, vals = raw[0], raw[1], raw[2]
        for m in ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
                  "sm__inst_executed_pipe_alu.sum", "sm__inst_executed_pipe_fma.sum",
                  "sm__inst_executed_pipe_lsu.sum", "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct"]:
            if m in hh:
                i = hh.index(m)
                print(f"  {m:38s} {vals[i]:>16s} {units[i]}")
    src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    hs = src[1]
    data = src[2:]
    ia, isrc = hs.index("Address"), hs.index("Source")
    iss, iex = hs.index("Warp Stall Sampling (All Samples)"), hs.index("Instructions Executed")
    ith = hs.index("Avg. Threads Executed")
    tot = sum(int(r[iss]) for r in data)
    print(f"  stall samples {tot}, warp instructions {sum(int(r[iex]) for r in data)}")
    for r in sorted(data, key=lambda r: -int(r[iss]))[:top]:
        print(f"   {r[ia][-5:]} {int(r[iss]):7d} {int(r[iex]):11d} {r[ith]:>5s}  {r[isrc][:84]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
