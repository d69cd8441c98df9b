"""Warp-stall summary of one kernel capture (run here, no GPU needed):

    python tools/ncu_stalls.py gpurun_out/TAG/prof_lloyd.ncu-rep [N]

Prints the kernel's sampled stall reasons and the N SASS instructions with the most samples
(a barrier stall lands on the instruction after its BAR.SYNC), from ncu's raw and source pages.
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12


def page(*args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


raw = page("--page", "raw")
hdr, vals = raw[0], raw[2] if len(raw) > 2 else raw[1]
stalls = {h.split("stalled_")[1]: float(v.replace(",", "")) for h, v in zip(hdr, vals)
          if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued") and v}
tot = sum(stalls.values())
for h, v in zip(hdr, vals):
    if h in ("gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active"):
        print(f"{h:60s} {v}")
print(f"sampled warp stalls: {tot:.0f}")
for k, v in sorted(stalls.items(), key=lambda x: -x[1]):
    if v > 0.005 * tot:
        print(f"  {k:24s} {v:8.0f}  {100 * v / tot:5.1f}%")
src = page("--page", "source", "--print-source", "sass")
shdr, data = src[1], src[2:]
ix = {h: i for i, h in enumerate(shdr)}
col = ix["Warp Stall Sampling (All Samples)"]
keys = [k for k in shdr if k.startswith("stall_") and "Not Issued" not in k]
rows = []
for n, r in enumerate(data):
    s = int(r[col] or 0)
    prev = data[n - 1][ix["Source"]].strip() if n else ""
    br = sorted(((k[6:], int(r[ix[k]] or 0)) for k in keys if int(r[ix[k]] or 0)), key=lambda x: -x[1])[:2]
    rows.append((s, n, r[ix["Source"]].strip(), prev, r[ix["Instructions Executed"]], br))
print(f"top {top} SASS instructions by samples (#index, instruction, previous instruction, executions):")
for s, n, ins, prev, ex, br in sorted(rows, reverse=True)[:top]:
    print(f"  {100 * s / tot:5.1f}% #{n:5d} {ins[:44]:44s} after {prev[:34]:34s} ex={ex} {br}")
