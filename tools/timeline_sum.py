"""Summarise a KT_LLOYD_TIMELINE probe log: per-phase totals of the last repetition."""
import re
import sys

import numpy as np

L = [l for l in open(sys.argv[1]) if l.startswith("[lloyd] pass")]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 98
v = np.array([list(map(float, re.findall(r"([\d.]+) us", l))) for l in L[-n:]])
print("phases:", L[-1].split(":",1)[1].strip())
print("sum (us):", v.sum(0).round(0), "total", v.sum().round(0))
print("first 25:", v[:25].sum(0).round(0), " rest:", v[25:].sum(0).round(0))
print(v[[0, 1, 2, 5, 10, 20, 30, 50, 80]])
