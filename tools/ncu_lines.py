"""Per-source-line stall samples / instructions of an .ncu-rep (cuda,sass correlated view).

    python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv
import subprocess
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname, agg, hdr = "?", {}, None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 8 or r[2] != "-" or not r[0].isdigit():
        continue
    samp = float(r[4] or 0)
    inst = float(r[7] or 0)
    stalls = {hdr[i]: float(r[i] or 0) for i in range(len(hdr)) if hdr[i].startswith("stall_") and "Not" not in hdr[i]}
    agg[(fname, int(r[0]))] = (samp, inst, r[1][:70], stalls)
tot = sum(v[0] for v in agg.values()) or 1
toti = sum(v[1] for v in agg.values()) or 1
for (f, ln), (s, i, src, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    best = sorted(st.items(), key=lambda kv: -kv[1])[:2]
    print(f"{f}:{ln:5d} {s / tot * 100:5.1f}% samp {i / toti * 100:5.1f}% inst  {src:70s} "
          + " ".join(f"{k[6:]}={v / max(s, 1) * 100:.0f}%" for k, v in best))
