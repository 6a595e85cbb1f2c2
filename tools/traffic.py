"""DRAM traffic of the whole-query kernel per config -> profiles/traffic.json.
Runs (under gpurun) ncu with dram__bytes_{read,write}.sum on the 2nd query of
tools/profile_one.py for each config and records the per-launch bytes.
Usage: python tools/traffic.py [round_tag] star-25 clique-18 ..."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
DIR = os.environ.get("TRAFFIC_DIR", os.path.join(ROOT, "profiles"))   # gpurun: a gpurun_out/ subdirectory
os.makedirs(DIR, exist_ok=True)
out = os.path.join(DIR, "traffic.json")
if not os.path.exists(out) and os.path.exists(os.path.join(ROOT, "profiles", "traffic.json")):
    out_init = os.path.join(ROOT, "profiles", "traffic.json")
else:
    out_init = out
data = json.load(open(out_init)) if os.path.exists(out_init) else {}
for cfg in sys.argv[2:]:
    csvp = os.path.join(DIR, f"{tag}_traffic_{cfg}.csv")
    cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
           "smsp__inst_executed.sum,lts__t_sectors_srcunit_tex_op_read.sum",
           "--clock-control", "none", "-k", "regex:k_dp_", "--csv", "--log-file", csvp,
           sys.executable, os.path.join(ROOT, "tools", "profile_one.py"), cfg, "1"]
    subprocess.run(cmd, check=True, capture_output=True)
    text = "\n".join(x for x in open(csvp).read().splitlines() if x.startswith('"'))
    rows = list(csv.reader(io.StringIO(text)))
    hdr = None
    per = {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        d = dict(zip(hdr, r))
        per.setdefault(d["ID"], {"name": d["Kernel Name"]})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    last = per[max(per, key=int)]               # the measured (2nd) query's kernel
    rd, wr = last.get("dram__bytes_read.sum", 0.0), last.get("dram__bytes_write.sum", 0.0)
    data[cfg] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                 "warp_inst": last.get("smsp__inst_executed.sum"),
                 "l2_read_sectors_from_l1": last.get("lts__t_sectors_srcunit_tex_op_read.sum"),
                 "kernel_ns_ncu": last.get("gpu__time_duration.sum"), "kernel": last["name"][:60],
                 "source": f"profiles/{tag}_traffic_{cfg}.csv: ncu --metrics dram__bytes_read.sum,"
                           f"dram__bytes_write.sum,smsp__inst_executed.sum (2nd query, "
                           f"{last['name'].split('<')[0]})"}
    print(cfg, data[cfg])
json.dump(data, open(out, "w"), indent=1)
