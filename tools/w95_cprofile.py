"""cProfile of bench.py's wall-to-95% tuning loop (5 landscapes, after one warm tune): python tools/w95_cprofile.py"""
import cProfile
import pstats
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import paper_1905_12799_b200 as kt  # noqa: E402
from paper_1905_12799_b200 import tune  # noqa: E402
from paper_1905_12799_b200.landscape import landscape_from_dict  # noqa: E402

fx = bench.w95_fixture()
space = kt.space_from_dict(fx["space"])
eng = kt.engine(0)
lands = [landscape_from_dict(doc, space) for doc in fx["landscapes"]]
fstars = [1.0 / kt.best_runtime(land)[0] for land in lands]
tune.tune_rows(space, lands[0], bench.W95_STRATEGY, 100, 1, engine=eng)


def run():
    for land, fs in zip(lands, fstars):
        tune.tune_rows(space, land, bench.W95_STRATEGY, bench.W95_BUDGET, bench.W95_SEED, engine=eng,
                       stop_fitness=0.95 * fs)


pr = cProfile.Profile()
pr.enable()
run()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(35)
