"""Per-CUDA-source-line summary of an ncu report (stall samples by reason,
instructions).  Usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, f, hdr = [], None, None
tot = {}
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if r[0] == "Function Name" or hdr is None or r[2] != "-":
        continue
    try:
        ln = int(r[0])
        samp, ins = int(r[4]), int(r[7])
    except ValueError:
        continue
    st = {}
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                v = int(r[i])
            except ValueError:
                continue
            if v:
                st[h[6:]] = v
                tot[h[6:]] = tot.get(h[6:], 0) + v
    if samp or ins:
        rows.append((samp, ins, f, ln, r[1].strip()[:70], st))
ts = sum(x[0] for x in rows) or 1
ti = sum(x[1] for x in rows) or 1
print(f"total stall samples {ts}, warp instructions {ti}")
print("by reason:", ", ".join(f"{k} {100 * v / ts:.1f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1])[:8]))
for samp, ins, f, ln, src, st in sorted(rows, reverse=True)[:top]:
    rs = " ".join(f"{k}:{v}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:3])
    print(f"{100 * samp / ts:5.1f}% {100 * ins / ti:5.1f}%i {f}:{ln:<4d} {src:70s} | {rs}")
