"""Multi-GPU sharding protocol (paper_1905_12799_b200/shard.py) on CPU.

* placement / shard ranges / numpy pairwise-tree leaves (bit-exact loss combination);
* the sharded Lloyd loop and knee scan driven over torch.distributed **gloo, world
  size 2 (and 4)**, with a numpy Lloyd backend standing in for the CUDA one
  (``GpuLloydShard``; same protocol, covered on the GPU by test_gpu_shard.py).
  Results must equal the single-process oracle bit for bit.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import socket

import numpy as np
import pytest
import torch

from oracle import sampler as osamp
from paper_1905_12799_b200 import shard

# ------------------------------------------------------------------ pure host logic


def test_place_tasks_resnet18_on_8_gpus():
    pl = shard.place_tasks(12, 8)
    work = [sum(1.0 / s[2] for s in p.shards) for p in pl]
    assert work == [1.5] * 8
    tasks = {}
    for p in pl:
        for t, i, n, group in p.shards:
            tasks.setdefault(t, []).append((i, n, group, p.rank))
    assert sorted(tasks) == list(range(12))
    for t, parts in tasks.items():
        n = parts[0][1]
        assert sorted(i for i, *_ in parts) == list(range(n))
        assert all(p[3] in p[2] for p in parts)


@pytest.mark.parametrize("n_tasks,world", [(5, 1), (5, 2), (5, 8), (12, 8), (8, 8), (3, 8), (0, 4)])
def test_place_tasks_covers_every_task_once(n_tasks, world):
    pl = shard.place_tasks(n_tasks, world)
    seen = {}
    for p in pl:
        for t, i, n, group in p.shards:
            seen.setdefault(t, set()).add(i)
            assert p.rank in group and len(group) == n
    assert set(seen) == set(range(n_tasks))
    assert all(v == set(range(len(v))) for v in seen.values())
    work = [sum(1.0 / s[2] for s in p.shards) for p in pl]
    assert max(work) - min(work) <= 1.0 + 1e-9


def test_shard_range_partitions_in_order():
    for count in (0, 1, 7, 1000, 1 << 20):
        for n in (1, 2, 3, 8):
            r = [shard.shard_range(count, i, n) for i in range(n)]
            assert r[0][0] == 0 and r[-1][1] == count
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))


@pytest.mark.parametrize("m", [300, 1000, 4097, 65_536, 262_144 + 13, 1_042_523])
@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_tree_leaves_reproduce_numpy_sum(m, world):
    ps = shard.point_shards(m, world)
    if ps is None:
        assert m < 2 ** np.ceil(np.log2(world)) * 129
        return
    x = np.random.default_rng(m + world).random(m) * 1e6
    leaf_sums = [np.sum(x[lo:hi]) for lo, hi in ps.leaves]
    assert shard.combine_leaves(leaf_sums) == np.sum(x)  # bit-exact, numpy's own pairwise order
    assert ps.leaves[0][0] == 0 and ps.leaves[-1][1] == m
    # every rank owns a contiguous, non-empty run of leaves in rank order
    for r in range(world):
        lo, hi = ps.ranges[r]
        assert hi > lo
        b = ps.local_leaf_bounds(r)
        assert b[0] == 0 and b[-1] == hi - lo
    assert list(ps.owner) == sorted(ps.owner)


def test_point_shards_too_small():
    assert shard.point_shards(200, 2) is not None  # 200 > 128 splits once
    assert shard.point_shards(128, 2) is None
    assert shard.point_shards(500, 8) is None


# ------------------------------------------------------------------ numpy backend (test stand-in for the GPU)
class NumpyLloydShard:
    """Same protocol as shard.GpuLloydShard; Lloyd semantics of sampler.py:91-116."""

    def __init__(self, pts_shard: np.ndarray, ks, init: np.ndarray):
        self.p = np.asarray(pts_shard, dtype=np.float64)
        self.m, self.n = self.p.shape
        self.ks = list(ks)
        self.K = sum(self.ks)
        self.off = np.concatenate([[0], np.cumsum(self.ks)]).astype(int)
        self.cur = [np.array(init[:k], dtype=np.float64) for k in self.ks]  # centroids for the next pass
        self.used = [c.copy() for c in self.cur]
        self.asg = [np.full(self.m, -1, dtype=np.int64) for _ in self.ks]
        self.own = [np.zeros(self.m) for _ in self.ks]
        self.S = np.zeros((self.K, 9), dtype=np.int64)
        self.state = [5] * len(self.ks)
        self.it = 0
        self.iters = [0] * len(self.ks)

    def local_pass(self):
        ext = np.zeros(self.K * 9 + len(self.ks), dtype=np.int64)
        for r, k in enumerate(self.ks):
            if self.state[r] not in shard.ACTIVE_STATES:
                continue
            if self.state[r] == 0:
                S = self.S[self.off[r]:self.off[r + 1]]
                self.cur[r] = S[:, : self.n].astype(np.float64) / S[:, 8:9].astype(np.float64)
            c = self.cur[r]
            self.used[r] = c.copy()
            d = np.empty((self.m, k))
            for j in range(k):
                d[:, j] = osamp._sq_dist(self.p, c[j])
            fresh = d.argmin(axis=1)
            self.own[r] = d[np.arange(self.m), fresh]
            old = self.asg[r]
            delta = np.zeros((k, 9), dtype=np.int64)
            pi = self.p.astype(np.int64)
            for j in range(k):
                delta[j, : self.n] += pi[fresh == j].sum(axis=0)
                delta[j, 8] += int((fresh == j).sum())
                delta[j, : self.n] -= pi[old == j].sum(axis=0)
                delta[j, 8] -= int((old == j).sum())
            ext[self.off[r] * 9:self.off[r + 1] * 9] = delta.reshape(-1)
            ext[self.K * 9 + r] = int(np.any(fresh != old))
            self.asg[r] = fresh
        return torch.from_numpy(ext)

    def apply(self, ext):
        e = ext.numpy()
        self.S += e[: self.K * 9].reshape(self.K, 9)
        for r, k in enumerate(self.ks):
            if self.state[r] not in shard.ACTIVE_STATES:
                continue
            counts = self.S[self.off[r]:self.off[r + 1], 8]
            if e[self.K * 9 + r] == 0:
                st = shard.CONVERGED
            elif self.it == 99:
                st = shard.MAXED
            elif (counts == 0).any():
                st = shard.NEEDS_RESEED
            else:
                st = 0
            if st != 0:
                self.iters[r] = self.it
            self.state[r] = st
        self.it += 1
        passes = [self.it if s in shard.ACTIVE_STATES else self.iters[r] + 1 for r, s in enumerate(self.state)]
        return list(self.state), passes

    def sums(self):
        return self.S.copy()

    def farthest(self, run, blocked_local):
        if self.m == 0:
            return -1.0, -1
        order = np.argsort(-self.own[run], kind="stable")
        bl = set(int(b) for b in blocked_local)
        for i in order:
            if int(i) not in bl:
                return float(self.own[run][i]), int(i)
        return -1.0, -1

    def set_centroids(self, run, cent):
        self.cur[run] = np.array(cent, dtype=np.float64)
        self.state[run] = 1

    def centroids(self, run):
        return self.used[run].copy()

    def leaf_losses(self, run, bounds):
        return np.array([np.sum(self.own[run][a:b]) for a, b in zip(bounds[:-1], bounds[1:])])


def lloyd_from_init(pts, init, max_iters=100):
    """oracle.kmeans' loop (sampler.py:91-116) started from given centroids."""
    m, k = pts.shape[0], init.shape[0]
    centroids = init.astype(np.float64).copy()
    assignment = np.full(m, -1, dtype=np.int64)
    history = []
    for it in range(max_iters):
        dist = np.empty((m, k))
        for j in range(k):
            dist[:, j] = osamp._sq_dist(pts, centroids[j])
        fresh = dist.argmin(axis=1)
        own = dist[np.arange(m), fresh]
        history.append(float(own.sum()))
        if np.array_equal(fresh, assignment):
            break
        assignment = fresh
        if it == max_iters - 1:
            break
        counts = np.bincount(assignment, minlength=k)
        for j in np.flatnonzero(counts):
            centroids[j] = pts[assignment == j].mean(axis=0)
        empty = np.flatnonzero(counts == 0)
        if empty.size:
            far = np.argsort(-own, kind="stable")
            used, cur = set(), 0
            for j in empty:
                while int(far[cur]) in used:
                    cur += 1
                used.add(int(far[cur]))
                centroids[int(j)] = pts[int(far[cur])]
    return centroids, assignment, history


# ------------------------------------------------------------------ gloo workers
def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, job, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, job(rank, world)))
    except Exception as ex:  # pragma: no cover - surfaced by the parent
        q.put((rank, ex))
    finally:
        dist.destroy_process_group()


def run_group(job, world):
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, job, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r, v in out.items():
        if isinstance(v, Exception):
            raise v
    return [out[r] for r in range(world)]


def _points(seed, m, n=8, hi=40):
    rng = np.random.default_rng(seed)
    pts = osamp.distinct_rows(rng.integers(0, hi, size=(m, n))).astype(np.float64)
    return pts


class _KneeJob:
    def __init__(self, pts, seed):
        self.pts, self.seed = pts, seed

    def __call__(self, rank, world):
        comm = shard.Comm()
        ps = shard.point_shards(len(self.pts), world)
        lo, hi = ps.ranges[rank]

        def init_fn(k):
            return osamp.plus_plus_init(self.pts, k, osamp.seeded_generator(self.seed))

        res, scanned = shard.knee_scan_sharded(
            lambda ks, init: NumpyLloydShard(self.pts[lo:hi], ks, init), comm, ps, self.pts, self.pts.shape[1],
            lambda rows: np.asarray(rows, dtype=np.float64), init_fn)
        return res.k, res.centroids, res.loss, scanned


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("seed", [0, 3])
def test_sharded_knee_scan_matches_oracle(world, seed):
    pts = _points(seed, 3000 if world == 2 else 5000)
    want, curve = osamp.knee_scan(pts, seed)
    outs = run_group(_KneeJob(pts, seed), world)
    for k, cent, loss, scanned in outs:
        assert [(kk, float(l).hex()) for kk, l in scanned] == [(kk, float(l).hex()) for kk, l in curve]
        assert np.array_equal(cent, want["centroids"])
        assert loss == want["loss"]


class _ReseedJob:
    """Coinciding initial centroids force empty clusters -> the distributed reseed path."""

    def __init__(self, pts, init):
        self.pts, self.init = pts, init

    def __call__(self, rank, world):
        comm = shard.Comm()
        ps = shard.point_shards(len(self.pts), world)
        lo, hi = ps.ranges[rank]
        backend = NumpyLloydShard(self.pts[lo:hi], [len(self.init)], self.init)
        res = shard.lloyd_runs(backend, comm, ps, self.pts, self.pts.shape[1], lambda r: np.asarray(r, float))
        return res[0].centroids, res[0].loss, res[0].passes, backend.asg[0]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_lloyd_reseed_matches_oracle(world):
    pts = _points(11, 2500, n=4, hi=30)
    init = np.vstack([pts[:5], pts[:3]])  # centroids 5..7 duplicate 0..2 -> empty after pass 1
    cent, asg, hist = lloyd_from_init(pts, init)
    outs = run_group(_ReseedJob(pts, init), world)
    ps = shard.point_shards(len(pts), world)
    got_asg = np.concatenate([o[3] for o in outs])
    for c, loss, passes, _ in outs:
        assert np.array_equal(c, cent)
        assert loss == hist[-1]
        assert passes == len(hist)
    assert np.array_equal(got_asg, asg)
    assert ps is not None


def test_assemble_batch_matches_oracle_rules():
    from paper_1905_12799_b200 import space as sp

    cards = [5, 6, 7]
    cent = np.array([[0.5, 1.49, 6.7], [4.6, 5.5, -0.2], [0.4, 1.2, 6.6], [2.0, 2.0, 2.0]])
    mode = [2, 2, 2]
    visited = sp.pack(np.array([[4, 5, 0]]), cards)
    got = [tuple(r) for r in sp.unpack(shard.assemble_batch(cent, mode, visited, cards), 3, cards).tolist()]
    want, seen, vis = [], set(), {(4, 5, 0)}
    for c in cent:  # sampler.py:200-215
        cand = osamp.round_centroid(c, cards)
        if cand in vis:
            cand = tuple(mode)
            if cand in vis:
                continue
        if cand in seen:
            continue
        seen.add(cand)
        want.append(cand)
    assert got == want and (2, 2, 2) in got and len(got) == 3


def _native_comm_job(rank, world):
    class _Eng:  # stands in for an engine: for_group must decide before touching it
        pass

    return shard.NativeComm.for_group(_Eng()) is None and shard.Comm().native is None


def test_native_comm_only_on_nccl_groups():
    """gloo groups (these CPU tests) keep the torch.distributed path: NativeComm.for_group
    returns None there and Comm carries no native communicator."""
    assert run_group(_native_comm_job, 2) == [True, True]
