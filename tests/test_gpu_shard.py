"""Sharded k-means on the GPU (kt_lloyd_* C-ABI + shard.py driver).

* world size 1 over a real NCCL process group: ``adaptive_sample_sharded`` equals the
  single-GPU ``adaptive_sample_rows`` and the oracle;
* 2 / 3 / 4 shards of one task on the same GPU, one thread per shard with an
  in-process all-reduce: the knee scan (curve, centroids) and the empty-cluster reseed
  are bit-exact against the CPU oracle — the protocol the gloo tests (test_shard.py)
  check with a numpy backend, here with the CUDA kernels.
"""

from __future__ import annotations

import json
import os
import socket
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU containers
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1905_12799_b200 as kt  # noqa: E402
from golden_io import GOLDEN  # noqa: E402
from oracle import sampler as osamp  # noqa: E402
from paper_1905_12799_b200 import _lib, shard  # noqa: E402
from paper_1905_12799_b200 import space as sp  # noqa: E402

MODELS = json.loads((GOLDEN / "models.json").read_text())


def space_of(values):
    return kt.DesignSpace("grid", tuple(kt.KnobDef(f"k{i}", tuple(v)) for i, v in enumerate(values)))


def dev_rows(idx, cards=None):
    return torch.from_numpy(sp.pack(np.asarray(idx), cards).view(np.int64)).cuda()


class ThreadComm:
    """In-process stand-in for a process group: one thread per shard."""

    def __init__(self, world):
        self.world = world
        self.bar = threading.Barrier(world)
        self.slots = [None] * world

    def view(self, rank):
        outer = self

        class _C:
            def __init__(self):
                self.rank, self.world = rank, outer.world

            def all_reduce_sum(self, t):
                torch.cuda.synchronize()
                outer.slots[rank] = t.clone()
                outer.bar.wait()
                total = sum(outer.slots)
                outer.bar.wait()
                t.copy_(total)
                torch.cuda.synchronize()

            def all_gather_f64(self, vals):
                outer.slots[rank] = np.asarray(vals, dtype=np.float64).copy()
                outer.bar.wait()
                out = np.stack(outer.slots)
                outer.bar.wait()
                return out

        return _C()


class Locked:
    """Serialise engine calls of concurrent shard threads (one engine, shared scratch)."""

    lock = threading.Lock()

    def __init__(self, inner):
        self.inner = inner
        self.ks = inner.ks

    def __getattr__(self, name):
        fn = getattr(self.inner, name)

        def call(*a):
            with Locked.lock:
                out = fn(*a)
                torch.cuda.synchronize()
                return out

        return call


def run_shards(world, job):
    comm = ThreadComm(world)
    out, errs = [None] * world, []

    def body(r):
        try:
            out[r] = job(r, comm.view(r))
        except Exception as ex:  # pragma: no cover
            errs.append(ex)
            comm.bar.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return out


def rows_to_float(rows, n, cards=None):
    return sp.unpack(np.asarray(rows, dtype=np.uint64), n, cards).astype(np.float64)


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("seed", [1, 2])
def test_gpu_sharded_knee_scan_vs_oracle(world, seed):
    rng = np.random.default_rng(seed)
    idx = osamp.distinct_rows(rng.integers(0, 40, size=(6000, 8)))
    pts = idx.astype(np.float64)
    want, curve = osamp.knee_scan(pts, seed)
    cards = np.full(8, 40, dtype=np.int32)
    eng = kt.engine(0)
    distinct = dev_rows(idx)
    host_rows = sp.pack(idx)
    ps = shard.point_shards(len(idx), world)

    def init_fn(k):
        out = np.zeros(k, dtype=np.uint64)
        with Locked.lock:
            _lib.call("kt_kmeanspp_rows", eng.handle, _lib.ptr(distinct), len(idx), 8,
                      _lib.as_ptr(cards, _lib.C.c_int32), seed, k, _lib.as_ptr(out, _lib.C.c_uint64))
        return out

    def job(rank, comm):
        lo, hi = ps.ranges[rank]
        res, scanned = shard.knee_scan_sharded(
            lambda ks, init: Locked(shard.GpuLloydShard(eng, distinct[lo:hi], 8, cards, ks, init)), comm, ps,
            host_rows, 8, lambda r: rows_to_float(r, 8), init_fn)
        return res, scanned

    for res, scanned in run_shards(world, job):
        assert [(k, float(x).hex()) for k, x in scanned] == [(k, float(x).hex()) for k, x in curve]
        assert np.array_equal(res.centroids, want["centroids"])


@pytest.mark.parametrize("world", [1, 2, 3])
def test_gpu_sharded_reseed_vs_oracle(world):
    from test_shard import lloyd_from_init

    rng = np.random.default_rng(11)
    idx = osamp.distinct_rows(rng.integers(0, 30, size=(2500, 4)))
    pts = idx.astype(np.float64)
    init = np.vstack([idx[:5], idx[:3]])  # centroids 5..7 duplicate 0..2 -> empty clusters
    cent, asg, hist = lloyd_from_init(pts, init.astype(np.float64))
    cards = np.full(4, 30, dtype=np.int32)
    eng = kt.engine(0)
    distinct = dev_rows(idx, cards)
    host_rows = sp.pack(idx, cards)
    ps = shard.point_shards(len(idx), world)
    init_rows = sp.pack(init, cards)

    def job(rank, comm):
        lo, hi = ps.ranges[rank]
        be = shard.GpuLloydShard(eng, distinct[lo:hi], 4, cards, [8], init_rows)
        res = shard.lloyd_runs(Locked(be), comm, ps, host_rows, 4, lambda r: rows_to_float(r, 4, cards))
        with Locked.lock:
            return res[0], be.assignment(0)

    outs = run_shards(world, job)
    assert np.array_equal(np.concatenate([a for _, a in outs]), asg)
    for res, _ in outs:
        assert np.array_equal(res.centroids, cent)
        assert res.loss == hist[-1] and res.passes == len(hist)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_adaptive_sample_sharded_world1_nccl():
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        space = space_of(MODELS["s2_resnet18"]["values"])
        cards = np.array(space.cardinalities)
        idx = np.random.default_rng(5).integers(0, cards, size=(40_000, 8))
        idx = np.vstack([idx, idx[:3000]])
        rows = dev_rows(idx)
        visited = sp.pack(idx[:20])
        eng = kt.engine()
        eng.set_timing(True)
        eng.kernel_stats(reset=True)
        got = shard.adaptive_sample_sharded(rows, visited, space, seed=17)
        stats = eng.kernel_stats(reset=True)
        eng.set_timing(False)
        # the device-driven loop ran: pass -> ncclAllReduce -> apply on the engine stream
        assert "lloyd_apply_dev" in stats and shard.NativeComm.for_group(eng) is not None
        ref = kt.adaptive_sample_rows(rows, visited, space, seed=17)
        assert got.tolist() == np.asarray(ref).tolist()
        want = osamp.adaptive_sample(idx, {tuple(r) for r in idx[:20].tolist()}, cards.tolist(), 17)
        assert [tuple(r) for r in sp.unpack(got, 8).tolist()] == want
    finally:
        dist.destroy_process_group()


# ------------------------------------------------------------------ sharded PPO search round
@pytest.mark.parametrize("world", [2, 3])
def test_gpu_sharded_search_round_vs_oracle(world):
    """Episodes split over `world` shards (one engine + thread each): the concatenated
    trajectory equals the oracle's bit for bit, the agent replicas stay identical, and the
    update is within the TF32 tier of the unsharded float64 reference."""
    from test_gpu_rl import LR, MODELS as RL_MODELS, assert_update_close, oracle_from, space_of as rl_space

    from oracle import agent as oagent
    from paper_1905_12799_b200.agent import PARAM_KEYS, _flat

    mm = RL_MODELS["table1"]
    space = rl_space(mm["values"])
    model = kt.CostModel.from_dict(mm["model"])
    hyper = kt.AgentHyperparams(episodes_per_round=1536)
    E = 1536
    replicas = [kt.init_agent(space, hyper, seed=21) for _ in range(world)]
    ref = oracle_from(replicas[0])
    before = _flat(replicas[0].params)
    starts = np.random.default_rng(4).integers(0, np.array(space.cardinalities), size=(E, 8))
    o_idx, o_sc, o_st = oagent.search_round(ref, mm["model"], mm["values"], starts, hyper.to_dict())
    engines = [kt.engine(0)] + [_lib.Engine(0) for _ in range(world - 1)]
    comm = ThreadComm(world)

    def job(rank, view):
        lo, hi = shard.shard_range(E, rank, world)
        rows = torch.from_numpy(kt.pack(starts[lo:hi]).view(np.int64)).cuda()
        r, s, st = kt.run_search_rows(replicas[rank], model, space, rows, engine=engines[rank],
                                      all_reduce=view.all_reduce_sum, episode_offset=lo)
        torch.cuda.synchronize()
        return r.cpu().numpy(), s.cpu().numpy(), st.cpu().numpy()

    outs = [None] * world
    errs = []

    def body(r):
        try:
            outs[r] = job(r, comm.view(r))
        except Exception as ex:  # pragma: no cover
            errs.append(ex)
            comm.bar.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    rows = np.concatenate([o[0] for o in outs])
    assert np.array_equal(kt.unpack(rows.view(np.uint64), 8), o_idx)
    assert np.array_equal(np.concatenate([o[1] for o in outs]), o_sc)
    assert np.array_equal(np.concatenate([o[2] for o in outs]), o_st)
    p0 = _flat(replicas[0].params)
    for a in replicas[1:]:
        assert np.array_equal(_flat(a.params), p0)  # every rank applied the same Adam step
        assert a.adam.t == replicas[0].adam.t
    want = np.concatenate([ref["params"][k].ravel() for k in PARAM_KEYS])
    assert_update_close(before, p0, want, replicas[0].params, 8)
    assert LR > 0


def test_sharded_search_round_world1_nccl_equals_unsharded():
    import torch.distributed as dist

    mm = MODELS["table1"]
    space = space_of(mm["values"])
    model = kt.CostModel.from_dict(mm["model"])
    hyper = kt.AgentHyperparams(episodes_per_round=512)
    a1, a2 = kt.init_agent(space, hyper, seed=3), kt.init_agent(space, hyper, seed=3)
    starts = np.random.default_rng(9).integers(0, np.array(space.cardinalities), size=(512, 8))
    rows = torch.from_numpy(kt.pack(starts).view(np.int64)).cuda()
    r1, s1, t1 = kt.run_search_rows(a1, model, space, rows)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        def no_torch_collectives(*_a, **_k):  # the native kt_comm path must carry every exchange
            raise AssertionError("torch.distributed all_reduce used on the sharded PPO path")

        orig = shard.Comm.all_reduce_sum
        shard.Comm.all_reduce_sum = no_torch_collectives
        try:
            r2, s2, t2 = shard.run_search_rows_sharded(a2, model, space, rows, episode_offset=0)
        finally:
            shard.Comm.all_reduce_sum = orig
    finally:
        dist.destroy_process_group()
    assert torch.equal(r1, r2) and torch.equal(s1, s2) and torch.equal(t1, t2)
    from paper_1905_12799_b200.agent import _flat

    assert np.array_equal(_flat(a1.params), _flat(a2.params))


@pytest.mark.parametrize("batch", [1, 3, 8])
def test_device_driven_reseed_world1_nccl(batch, monkeypatch):
    """kt_lloyd_run (pass -> ncclAllReduce -> apply enqueued `batch` rounds ahead, device-side
    iteration counter and freeze flag) through an empty-cluster reseed: bit-exact vs the
    oracle's Lloyd from the same init (sampler.py:94-116)."""
    import torch.distributed as dist

    from test_shard import lloyd_from_init

    rng = np.random.default_rng(11)
    idx = osamp.distinct_rows(rng.integers(0, 30, size=(2500, 4)))
    pts = idx.astype(np.float64)
    init = np.vstack([idx[:5], idx[:3]])  # centroids 5..7 duplicate 0..2 -> empty clusters
    cent, asg, hist = lloyd_from_init(pts, init.astype(np.float64))
    cards = np.full(4, 30, dtype=np.int32)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        eng = kt.engine(0)
        distinct = dev_rows(idx, cards)
        ps = shard.point_shards(len(idx), 1)
        be = shard.GpuLloydShard(eng, distinct, 4, cards, [8], sp.pack(init, cards))
        orig_run = be.run
        monkeypatch.setattr(be, "run", lambda native: orig_run(native, batch))
        comm = shard.Comm(None, device="cuda:0")
        comm.native = shard.NativeComm.for_group(eng)
        assert comm.native is not None
        eng.set_timing(True)
        eng.kernel_stats(reset=True)
        res = shard.lloyd_runs(be, comm, ps, sp.pack(idx, cards), 4, lambda r: rows_to_float(r, 4, cards))
        stats = eng.kernel_stats(reset=True)
        eng.set_timing(False)
        assert "lloyd_apply_dev" in stats
        assert np.array_equal(be.assignment(0), asg)
        assert np.array_equal(res[0].centroids, cent)
        assert res[0].loss == hist[-1] and res[0].passes == len(hist)
    finally:
        dist.destroy_process_group()
