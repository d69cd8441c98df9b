"""Copy one gpu_session.sh run into profiles/<round>/ (default r2): ncu summaries, per-launch DRAM traffic, the launch
list summary and the bench JSON lines.

    python tools/refresh_profiles.py TAG [ROUND]      (reads gpurun_out/TAG/)
"""

import collections
import csv
import json
import re
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
tag = sys.argv[1]
src = ROOT / "gpurun_out" / tag
dst = ROOT / "profiles" / (sys.argv[2] if len(sys.argv) > 2 else "r2")
dst.mkdir(parents=True, exist_ok=True)
if not (dst / "traffic.json").exists():
    shutil.copy(ROOT / "profiles" / "r1" / "traffic.json", dst / "traffic.json")
CAPTURES = {"lloyd": "lloyd", "score_trees": "score_trees", "dedup_insert": "dedup_insert",
            "kmeanspp_init": "init_kernel"}
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

traffic = json.loads((dst / "traffic.json").read_text())
for key, cap in CAPTURES.items():
    rep = src / f"prof_{cap}.ncu-rep"
    if not rep.exists():
        continue
    text = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"), str(rep)],
                          capture_output=True, text=True).stdout
    (dst / f"prof_{cap}.txt").write_text(text)

    def val(name):
        m = re.search(name + r"\s+([\d.]+)\s+(\w+)", text)
        return float(m.group(1)) * UNITS[m.group(2)]

    traffic["kernels"][key] = {"dram_bytes_per_launch": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
                               "capture": f"{tag}/prof_{cap}"}
(dst / "traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")

launches = src / "launches.csv"
if launches.exists():
    rows = list(csv.reader(line for line in open(launches) if not line.startswith("==")))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "ns": 1, "us": 1e3, "ms": 1e6}
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
    tot = sum(v for _, v in agg.values())
    with open(dst / "launches_summary.txt", "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised); "
                f"bench.py --steps 2 --warmup 1 --no-wall95 --no-extra-configs (capture {tag})\n# kernel, launches, total ns, share\n")
        for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{k:60s} {c:6d} {v:14.1f} {100 * v / tot:6.2f}%\n")
    for old in dst.glob("launches_bench_*.csv"):
        old.unlink()
    shutil.copy(launches, dst / f"launches_bench_{tag}.csv")

for name, out in (("bench.json", "bench"), ("bench_ref.json", "bench_ref"), ("bench_rl.json", "bench_rl")):
    if (src / name).exists():
        for old in dst.glob(f"{out}_{dst.name}*.json"):
            old.unlink()
        shutil.copy(src / name, dst / f"{out}_{tag}.json")
print(f"profiles/{dst.name} refreshed from", src)
