"""Parity of the CUDA path against the reference (golden vectors) and the CPU oracle.

Bit-exact for integer/index work and for the float64 paths whose rounding the
engine reproduces (tree scores, k-means centroids/loss, SA); runtimes within
1e-12 relative (CUDA exp vs glibc exp, <= 1 ulp; north star allows 1e-5).
"""

import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU containers
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1905_12799_b200 as kt  # noqa: E402
from golden_io import GOLDEN, cases, meta, npz  # noqa: E402
from oracle import landscape as oland  # noqa: E402
from oracle import sa as osa  # noqa: E402
from oracle import sampler as osamp  # noqa: E402
from oracle import trees as otrees  # noqa: E402
from paper_1905_12799_b200 import space as sp  # noqa: E402

MODELS = json.loads((GOLDEN / "models.json").read_text())
LANDS = json.loads((GOLDEN / "landscapes.json").read_text())


def space_of(values, name="grid"):
    return kt.DesignSpace(name, tuple(kt.KnobDef(f"k{i}", tuple(v)) for i, v in enumerate(values)))


def dev_rows(idx):
    return torch.from_numpy(sp.pack(np.asarray(idx)).view(np.int64)).cuda()


@pytest.fixture(scope="module", autouse=True)
def _engine_loaded():
    kt.engine(0)


# ------------------------------------------------------------------ K2 trees
@pytest.mark.parametrize("name", sorted(MODELS))
def test_predict_bit_exact_vs_reference(name):
    m = MODELS[name]
    space = space_of(m["values"])
    model = kt.CostModel.from_dict(m["model"])
    g = npz("predict")
    got = kt.predict_rows(model, space, dev_rows(g[f"{name}/idx"])).cpu().numpy()
    assert np.array_equal(got, g[f"{name}/scores"])


def test_predict_dropin_signature_and_errors():
    m = MODELS["bowl_g10"]
    space = space_of(m["values"])
    model = kt.CostModel.from_dict(m["model"])
    configs = [kt.Configuration((1, 2, 3)), kt.Configuration((9, 0, 4))]
    want = otrees.predict_features(m["model"], otrees.featurize_rows(m["values"], [[1, 2, 3], [9, 0, 4]]))
    assert np.array_equal(kt.predict(model, space, configs), want)
    assert kt.predict(model, space, []).shape == (0,)
    with pytest.raises(kt.errors.DimensionMismatchError):
        kt.predict(kt.CostModel.sentinel(2), space, configs)
    with pytest.raises(kt.errors.SpaceValidationError):
        kt.predict(model, space, [kt.Configuration((10, 0, 0))])


@pytest.mark.parametrize("n_rows", [1, 2, 3, 255, 256, 257, 100_003, 1 << 20])
def test_predict_random_sizes_vs_oracle(n_rows):
    m = MODELS["s2_resnet18"]
    space = space_of(m["values"])
    model = kt.CostModel.from_dict(m["model"])
    rng = np.random.default_rng(n_rows)
    idx = rng.integers(0, np.array(space.cardinalities), size=(n_rows, 8))
    got = kt.predict_rows(model, space, dev_rows(idx)).cpu().numpy()
    check = slice(None) if n_rows <= 200_000 else slice(0, n_rows, 97)  # oracle cost bound
    want = otrees.predict_features(m["model"], otrees.featurize_rows(m["values"], idx[check]))
    assert np.array_equal(got[check], want)


# ------------------------------------------------------------------ K3 landscape
@pytest.mark.parametrize("name", sorted(LANDS))
def test_landscape_vs_reference(name):
    d = LANDS[name]
    space = space_of(d["values"])
    land = kt.landscape.landscape_from_dict(d["landscape"], space)
    g = npz("landscape")
    got = kt.runtimes_rows(land, dev_rows(g[f"{name}/idx"])).cpu().numpy()
    want = g[f"{name}/runtime"]
    assert np.array_equal(got, want)  # bit-exact: glibc's exp restated on the device


BEST = json.loads((GOLDEN / "best.json").read_text())


@pytest.mark.parametrize("case", BEST, ids=lambda c: c["name"])
def test_landscape_best_vs_reference_enumeration(case):
    """kt_landscape_best == the reference's _enumerated_oracle (cli.py:77-90) on byte and bit-field
    row layouts; sampled runtimes bit-exact (tests/golden/make_best.py)."""
    space = kt.space_from_dict(case["space"])
    land = kt.landscape.landscape_from_dict(case["landscape"], space)
    best, arg = kt.best_runtime(land)
    assert float(best).hex() == case["best_runtime"]
    assert list(arg) == case["best_indices"]
    idx = np.array(case["sample_idx"])
    rows = torch.from_numpy(sp.pack(idx, np.array(space.cardinalities)).view(np.int64)).cuda()
    got = kt.runtimes_rows(land, rows).cpu().numpy()
    assert [float(x).hex() for x in got] == case["sample_runtime"]


def test_landscape_runtimes_random_vs_oracle():
    """200K random S2 configurations against the oracle (math.exp): bit-exact."""
    m = MODELS["s2_resnet18"]
    space = space_of(m["values"])
    land = kt.SyntheticLandscape(seed=77, space=space, centers=((10, 5, 70, 3, 1, 0, 2, 1), (80, 40, 2, 6, 0, 1, 0, 0)),
                                 depths=(0.6, 0.3), radii=(9.5, 31.25), noise_rel=0.02)
    rng = np.random.default_rng(12)
    idx = rng.integers(0, np.array(space.cardinalities), size=(200_000, 8))
    got = kt.runtimes_rows(land, dev_rows(idx)).cpu().numpy()
    doc = {"seed": 77, "centers": [list(c) for c in land.centers], "depths": list(land.depths),
           "radii": list(land.radii), "base_runtime": 1.0, "noise_rel": 0.02}
    want = oland.synthetic_runtimes(doc, idx)
    assert np.array_equal(got, want)


def test_landscape_hash_noise_bit_pattern():
    """With depth term 0 the runtime is base*(1+noise*u): exposes the blake2b word exactly."""
    space = space_of([list(range(200))] * 8)
    land = kt.SyntheticLandscape(seed=12345, space=space, centers=((0,) * 8,), depths=(0.5,), radii=(1e-3,),
                                 noise_rel=0.5)
    rng = np.random.default_rng(3)
    idx = rng.integers(0, 200, size=(2000, 8))
    idx[:, 0] = np.maximum(idx[:, 0], 1)  # away from the center: exp underflows to 0 exactly
    got = kt.runtimes_rows(land, dev_rows(idx)).cpu().numpy()
    want = np.array([1.0 * (1.0 + 0.5 * oland.hash_unit(12345, r)) for r in idx.tolist()])
    assert np.array_equal(got, want)


# ------------------------------------------------------------------ K7/K8 k-means
@pytest.mark.parametrize("name", cases("kmeans", "points"))
def test_kmeans_vs_reference(name):
    g = npz("kmeans")
    k, seed = (int(x) for x in g[f"{name}/meta"])
    res = kt.kmeans(g[f"{name}/points"], k, seed)
    assert np.array_equal(res.centroids, g[f"{name}/centroids"])
    assert np.array_equal(res.assignment, g[f"{name}/assignment"])
    assert np.array_equal(np.array(res.loss_history), g[f"{name}/history"])


@pytest.mark.parametrize("seed", range(6))
def test_kmeans_random_lattice_vs_oracle(seed):
    rng = np.random.default_rng(100 + seed)
    m = int(rng.integers(20, 3000))
    n = int(rng.integers(1, 9))
    pts = np.unique(rng.integers(0, int(rng.integers(3, 60)), size=(m, n)), axis=0)
    pts = pts[rng.permutation(len(pts))].astype(np.float64)
    k = int(min(len(pts), rng.integers(1, 40)))
    res = kt.kmeans(pts, k, seed)
    want = osamp.kmeans(pts, k, seed)
    assert np.array_equal(res.centroids, want["centroids"])
    assert np.array_equal(res.assignment, want["assignment"])
    assert res.loss_history == want["history"]


def test_kmeans_errors():
    with pytest.raises(ValueError, match="out of range"):
        kt.kmeans(np.array([[0.0], [1.0], [1.0]]), 3, 0)
    with pytest.raises(ValueError, match="out of range"):
        kt.kmeans(np.array([[0.0], [1.0]]), 0, 0)


@pytest.mark.parametrize("name", cases("knee", "points"))
def test_knee_vs_reference(name):
    g = npz("knee")
    res, scanned = kt.knee_scan(g[f"{name}/points"], int(g[f"{name}/seed"][0]))
    assert np.array_equal(np.array(scanned, dtype=np.float64), g[f"{name}/scanned"])
    assert np.array_equal(res.centroids, g[f"{name}/centroids"])
    assert np.array_equal(res.assignment, g[f"{name}/assignment"])


# ------------------------------------------------------------------ adaptive sample
@pytest.mark.parametrize("name", sorted(meta("adaptive")))
def test_adaptive_sample_vs_reference(name):
    g = npz("adaptive")
    md = meta("adaptive")[name]
    space = space_of([list(range(c)) for c in md["cards"]])
    idx = g[f"{name}/idx"]
    traj = kt.Trajectory(dev_rows(idx), torch.zeros(len(idx), dtype=torch.float64, device="cuda"), n_knobs=len(md["cards"]))
    visited = kt.VisitedSet([kt.Configuration(tuple(r)) for r in g[f"{name}/visited"].tolist()])
    batch = kt.adaptive_sample(traj, visited, space, md["seed"])
    assert [c.indices for c in batch] == [tuple(r) for r in g[f"{name}/batch"].tolist()]
    assert kt.mode_config(traj, space).indices == tuple(g[f"{name}/mode"].tolist())


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_adaptive_sample_uniform_s2_vs_oracle(seed):
    m = MODELS["s2_resnet18"]
    space = space_of(m["values"])
    rng = np.random.default_rng(seed)
    n_rows = [2000, 9000, 20000, 40000][seed]
    idx = rng.integers(0, np.array(space.cardinalities), size=(n_rows, 8))
    idx = np.vstack([idx, idx[: n_rows // 10]])  # duplicates
    visited = {tuple(r) for r in idx[rng.integers(0, len(idx), size=50)].tolist()}
    vis_rows = sp.pack(np.array(sorted(visited)))
    got = kt.adaptive_sample_rows(dev_rows(idx), vis_rows, space, seed=seed + 11)
    want = osamp.adaptive_sample(idx, visited, space.cardinalities, seed + 11)
    assert [tuple(r) for r in sp.unpack(got, 8).tolist()] == want


@pytest.mark.parametrize("mode", ["stream", "tile64", "gather", "init_chunked", "pack5", "grid", "cluster8", "blocks7",
                                  "blocks7_miss", "cluster1"])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_lloyd_variants_vs_oracle(mode, seed, monkeypatch):
    """Both Lloyd kernels (streaming, and resident with many queue tiles per block) and both k-means++
    kernels (resident, chunked) agree with the oracle; small point sets also through the cooperative
    grid (grid: no cluster), an 8-block cluster, and a 7-block cooperative grid.  The 7-block grid
    (>= 1,536 points per block from 20K candidates on) and the one-block cluster run the speculative
    scan at small sizes, blocks7_miss with a zero guard (almost every pass drops its queue)."""
    if mode == "blocks7_miss":
        monkeypatch.setenv("KT_LLOYD_SPEC_FACTOR", "0")
        mode = "blocks7"
    if mode == "cluster1":
        monkeypatch.setenv("KT_LLOYD_CLUSTER", "1")
    elif mode == "grid":
        monkeypatch.setenv("KT_LLOYD_CLUSTER", "0")
    elif mode == "cluster8":
        monkeypatch.setenv("KT_LLOYD_CLUSTER", "8")
    elif mode == "blocks7":
        monkeypatch.setenv("KT_LLOYD_CLUSTER", "0")
        monkeypatch.setenv("KT_LLOYD_BLOCKS", "7")
    elif mode == "init_chunked":
        monkeypatch.setenv("KT_INIT_MODE", "chunked")
    elif mode == "stream":
        monkeypatch.setenv("KT_LLOYD_MODE", "stream")
    elif mode == "gather":
        monkeypatch.setenv("KT_LLOYD_ROWS", "global")
    elif mode == "pack5":
        monkeypatch.setenv("KT_LLOYD_PACK5", "1")
    else:
        monkeypatch.setenv("KT_LLOYD_TILE", "64")
    test_kmeans_random_lattice_vs_oracle(seed)
    test_adaptive_sample_uniform_s2_vs_oracle(seed + 1)


LARGE = json.loads((GOLDEN / "large.json").read_text())


LLOYD_MODES = {"resident": {}, "stream": {"KT_LLOYD_MODE": "stream"}, "tile64": {"KT_LLOYD_TILE": "64"},
               "gather": {"KT_LLOYD_ROWS": "global"}, "init_chunked": {"KT_INIT_MODE": "chunked"},
               "pack5": {"KT_LLOYD_PACK5": "1"},
               # speculative scan (blocks of >= 1536 points): guard 0 -> almost every pass rescans,
               # guard 16 -> every speculative queue is used, with many extra (exact) evaluations
               "spec_miss": {"KT_LLOYD_SPEC_FACTOR": "0"}, "spec_wide": {"KT_LLOYD_SPEC_FACTOR": "16"}}


@pytest.mark.parametrize("mode", sorted(LLOYD_MODES))
@pytest.mark.parametrize("name", sorted(LARGE))
def test_knee_large_vs_oracle_golden(name, mode, monkeypatch):
    """131K / 262K candidates (config C3 size): knee curve, centroids, assignment and batch bit-exact."""
    import hashlib

    for k, v in LLOYD_MODES[mode].items():
        monkeypatch.setenv(k, v)
    g = LARGE[name]
    space = space_of(MODELS["s2_resnet18"]["values"])
    cards = np.array(space.cardinalities)
    idx = np.random.default_rng(g["cand_seed"]).integers(0, cards, size=(g["n"], cards.size))
    uniq = osamp.distinct_rows(idx)
    assert len(uniq) == g["m"]
    res, curve = kt.knee_scan(uniq.astype(np.float64), g["seed"])
    assert [[k, float(x).hex()] for k, x in curve] == g["curve"]
    assert [[float(x).hex() for x in c] for c in res.centroids] == g["centroids"]
    asg = np.asarray(res.assignment, dtype=np.int64)
    assert hashlib.sha256(asg.tobytes()).hexdigest() == g["assignment_sha256"]
    got = kt.adaptive_sample_rows(dev_rows(idx), np.zeros(0, dtype=np.uint64), space, seed=g["seed"])
    assert sp.unpack(got, 8).tolist() == g["batch"]


def test_adaptive_sample_1m_candidates_properties():
    """North-star size: 1,048,576 uniform S2 candidates — dedup count, batch contract, knee k."""
    m = MODELS["s2_resnet18"]
    space = space_of(m["values"])
    rng = np.random.default_rng(2026)
    idx = rng.integers(0, np.array(space.cardinalities), size=(1 << 20, 8))
    rows = dev_rows(idx)
    visited = {tuple(r) for r in idx[:100].tolist()}
    info = kt._lib.SampleInfo()
    got = kt.adaptive_sample_rows(rows, sp.pack(np.array(sorted(visited))), space, seed=99, info=info)
    assert info.n_distinct == len(np.unique(sp.pack(idx)))
    batch = [tuple(r) for r in sp.unpack(got, 8).tolist()]
    assert 1 <= len(batch) < 64 and len(set(batch)) == len(batch)
    assert not (set(batch) & visited)
    assert 8 <= info.chosen_k <= 63
    losses = [info.scanned_loss[i] for i in range(info.n_scanned)]
    for a, b in zip(losses, losses[1:-1]):
        assert 1.1 * b <= a  # every non-final k passed the knee test
    if info.n_scanned >= 2:
        assert 1.1 * losses[-1] > losses[-2] or info.chosen_k == 63


# ------------------------------------------------------------------ K10 SA
@pytest.mark.parametrize("launch", ["fused", "unfused"])
@pytest.mark.parametrize("name", sorted(meta("sa")))
def test_sa_vs_reference(name, launch, monkeypatch):
    """fused: the warp kernel scores the starts and derives T0 itself (<= 1024 chains);
    unfused: score_trees + pairwise sums + temperature launches (KT_SA_UNFUSED)."""
    if launch == "unfused":
        monkeypatch.setenv("KT_SA_UNFUSED", "1")
    g = npz("sa")
    md = meta("sa")[name]
    mm = MODELS[md["model"]]
    space = space_of(mm["values"])
    model = kt.CostModel.from_dict(mm["model"])
    params = kt.SAParams(chains=md["chains"], steps_per_round=md["steps"],
                         initial_temperature=md["initial_temperature"], cooling=md["cooling"])
    starts = [kt.Configuration(tuple(r)) for r in g[f"{name}/starts"].tolist()]
    tr = kt.run_sa_round(params, model, space, starts, md["seed"])
    assert np.array_equal(tr.index_matrix(), g[f"{name}/idx"])
    assert np.array_equal(tr.scores(), g[f"{name}/scores"])
    assert tr.step_indices == tuple(g[f"{name}/steps"].tolist())


@pytest.mark.parametrize("chains,unfused", [(1024, False), (1024, True), (1500, False), (64, False)])
def test_sa_large_vs_oracle(chains, unfused, monkeypatch):
    if unfused:
        monkeypatch.setenv("KT_SA_UNFUSED", "1")
    mm = MODELS["s2_resnet18"]
    space = space_of(mm["values"])
    model = kt.CostModel.from_dict(mm["model"])
    rng = np.random.default_rng(8)
    idx = rng.integers(0, np.array(space.cardinalities), size=(1000, 8))
    tr = kt.run_sa_round(kt.SAParams(chains=chains, steps_per_round=40), model, space,
                         [kt.Configuration(tuple(r)) for r in idx.tolist()], seed=2**40 + 3)
    o_idx, o_sc, o_st = osa.run_sa_round(mm["model"], mm["values"], idx, 2**40 + 3, chains=chains, steps=40)
    assert np.array_equal(tr.index_matrix(), o_idx)
    assert np.array_equal(tr.scores(), o_sc)
    assert np.array_equal(np.array(tr.step_indices), o_st)


def test_sa_errors():
    mm = MODELS["bowl_g10"]
    space = space_of(mm["values"])
    model = kt.CostModel.from_dict(mm["model"])
    with pytest.raises(ValueError):
        kt.run_sa_round(kt.SAParams(), model, space, [], 0)
    with pytest.raises(ValueError, match="chains"):
        kt.SAParams(chains=0)


BENCH_G = json.loads((GOLDEN / "bench_golden.json").read_text())


def _bench_case(name, mode, monkeypatch):
    import hashlib

    for k, v in LLOYD_MODES[mode].items():
        monkeypatch.setenv(k, v)
    g = BENCH_G[name]
    space = space_of(MODELS["s2_resnet18"]["values"])
    cards = np.array(space.cardinalities)
    idx = np.random.default_rng(g["cand_seed"]).integers(0, cards, size=(g["n"], cards.size))
    rows = dev_rows(idx)
    info = kt._lib.SampleInfo()
    got = kt.adaptive_sample_rows(rows, np.zeros(0, dtype=np.uint64), space, seed=g["seed"], info=info)
    assert info.n_distinct == g["m"]
    assert [[info.scanned_k[i], float(info.scanned_loss[i]).hex()] for i in range(info.n_scanned)] == g["curve"]
    assert sp.unpack(got, 8).tolist() == g["batch"]
    vinfo = kt._lib.SampleInfo()
    got_v = kt.adaptive_sample_rows(rows, sp.pack(np.array(g["visited"])), space, seed=g["seed"], info=vinfo)
    assert sp.unpack(got_v, 8).tolist() == g["batch_visited"]
    assert bool(vinfo.used_mode) == (g["mode"] is not None)
    uniq = osamp.distinct_rows(idx)
    res, curve = kt.knee_scan(uniq.astype(np.float64), g["seed"])
    assert [[k, float(x).hex()] for k, x in curve] == g["curve"]
    assert [[float(x).hex() for x in c] for c in res.centroids] == g["centroids"]
    asg = np.asarray(res.assignment, dtype=np.int64)
    assert hashlib.sha256(asg.tobytes()).hexdigest() == g["assignment_sha256"]


@pytest.mark.parametrize("mode", ["resident", "tile64", "pack5", "spec_miss", "spec_wide"])
def test_bench_headline_config_bit_exact(mode, monkeypatch):
    """bench.py's exact headline step (1,048,576 uniform S2 candidates, candidate seed 0, seed 1000):
    distinct count, knee curve, centroids, assignment, batch with and without the bench's visited set
    (mode vote) bit-exact vs the oracle (tests/golden/make_bench_golden.py)."""
    _bench_case("s2", mode, monkeypatch)


def test_c5_4m_candidates_streaming_bit_exact(monkeypatch):
    """configs[4]'s large end: 4,194,304 candidates (~4M distinct points, streaming Lloyd kernel)."""
    if "c5" not in BENCH_G:
        pytest.skip("c5 golden not generated (tests/golden/make_bench_golden.py c5)")
    _bench_case("c5", "resident", monkeypatch)
