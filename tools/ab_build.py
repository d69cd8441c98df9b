"""Build an A/B variant of the engine: copy csrc/, apply textual replacements, link build/ab/<name>.so.

    python tools/ab_build.py NAME 'old=>new' ['old2=>new2' ...]     (run with KT_LIB_PATH=build/ab/NAME.so)
"""
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1905_12799_b200 import build as b  # noqa: E402

name = sys.argv[1]
work = Path("/tmp/ab_" + name)
shutil.rmtree(work, ignore_errors=True)
shutil.copytree(ROOT / "paper_1905_12799_b200" / "csrc", work / "paper_1905_12799_b200" / "csrc")
shutil.copytree(ROOT / "include", work / "include")
for rep in sys.argv[2:]:
    old, new = rep.split("=>")
    hit = False
    for f in (work / "paper_1905_12799_b200" / "csrc").iterdir():
        t = f.read_text()
        if old in t:
            f.write_text(t.replace(old, new))
            hit = True
    assert hit, f"pattern not found: {old}"
out = ROOT / "build" / "ab"
out.mkdir(parents=True, exist_ok=True)
objs = []
procs = []
for src in sorted((work / "paper_1905_12799_b200" / "csrc").glob("*.cu")):
    obj = work / (src.stem + ".o")
    objs.append(obj)
    procs.append(subprocess.Popen([b._nvcc(), *b.ARCH, *b.FLAGS, "-c", str(src), "-o", str(obj)]))
assert all(p.wait() == 0 for p in procs)
subprocess.run([b._nvcc(), *b.ARCH, "-shared", "-o", str(out / f"{name}.so"), *map(str, objs), "-lcudart_static",
                "-lrt", "-ldl", "-lpthread"], check=True)
print(out / f"{name}.so")
