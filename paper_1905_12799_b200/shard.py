"""Multi-GPU sharding of the search step.

One process per GPU (torch.distributed; NCCL over NVLink on the B200 box, gloo in
the CPU tests).  What is partitioned, and the only exchanges:

* **Tasks** (`place_tasks`): whole tuning tasks go round-robin to ranks; tasks left
  over when ``n_tasks % world != 0`` are split into candidate shards over groups of
  ranks, so 12 ResNet-18 tasks on 8 GPUs cost 1.5 task-steps per GPU, not 2.
* **Candidates of one task**: contiguous, episode-major shards.  Scoring (K2/K3) and
  rollouts need no communication.  First-occurrence dedup (sampler.py:187-192) is
  global, so the candidate rows are all-gathered (8 B per candidate) and every rank
  dedups / votes the mode / runs k-means++ on the identical list.
* **k-means points**: the distinct list is cut at the nodes of numpy's pairwise-sum
  tree (`tree_leaves`), ``ceil(log2 G)`` levels deep, and each rank runs Lloyd on
  its contiguous leaves.  Per pass ONE all-reduce (SUM) of an int64 buffer — the
  [K][9] cluster coordinate/count deltas and the per-run changed counts — gives
  every rank the same exact sums, hence the same decisions and centroids
  (sampler.py:91-116).  Losses are numpy pairwise sums per leaf, all-gathered and
  combined in tree order, so ``L_k`` — and the knee decision
  ``1.1 * L_k > L_{k-1}`` — are bit-identical to the single-GPU result.
* **Empty-cluster reseed** (sampler.py:108-115): each rank proposes its farthest
  unblocked point; an all-gather picks the global maximum (ties -> lowest index).

The pass loop is written against a small backend protocol (`LloydShard`); the
product backend is `GpuLloydShard` (kt_lloyd_* C-ABI, CUDA kernels).  The CPU
tests drive the same loop with a numpy backend under gloo, world size 2.
"""

from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from . import space as sp

PW_BLOCKSIZE = 128  # numpy pairwise_sum leaf size (numpy/_core/src/umath/loops_utils.h.src)
KNEE_K_MIN, KNEE_K_MAX, KNEE_CONSTANT = 8, 63, 1.1
ACTIVE_STATES = (0, 1, 5)
CONVERGED, MAXED, NEEDS_RESEED = 2, 3, 4


# ------------------------------------------------------------------ placement
@dataclass(frozen=True)
class Placement:
    """Work of one rank: ``shards`` = [(task, shard_index, n_shards, group_ranks)]."""

    rank: int
    shards: tuple


def place_tasks(n_tasks: int, world: int) -> list[Placement]:
    """Whole tasks round-robin, then the remainder split evenly into candidate shards.

    Every rank gets ``n_tasks / world`` task-steps of work when the remainder tasks
    divide the ranks (C4: 12 tasks / 8 GPUs -> 1 whole task + half of a shared one).
    """
    if n_tasks < 0 or world < 1:
        raise ValueError("n_tasks >= 0 and world >= 1 required")
    per = {r: [] for r in range(world)}
    whole = (n_tasks // world) * world
    for t in range(whole):
        per[t % world].append((t, 0, 1, (t % world,)))
    rest = n_tasks - whole
    if rest:
        # remainder task i is shared by a contiguous group of ranks
        bounds = [round(i * world / rest) for i in range(rest + 1)]
        for i in range(rest):
            group = tuple(range(bounds[i], bounds[i + 1]))
            for s, r in enumerate(group):
                per[r].append((whole + i, s, len(group), group))
    return [Placement(r, tuple(per[r])) for r in range(world)]


def shard_range(count: int, index: int, n_shards: int) -> tuple[int, int]:
    """Contiguous candidate shard ``index`` of ``n_shards`` (episode-major order preserved)."""
    return count * index // n_shards, count * (index + 1) // n_shards


# ------------------------------------------------------------------ numpy pairwise tree
def pairwise_split(n: int) -> int:
    """numpy's split point of a pairwise_sum node of n > 128 elements."""
    n2 = n // 2
    return n2 - n2 % 8


def tree_leaves(m: int, depth: int) -> list[tuple[int, int]] | None:
    """The 2**depth nodes at ``depth`` of numpy's pairwise tree over m elements, left
    to right; None if some node on the way has <= 128 elements (it would not split)."""
    nodes = [(0, m)]
    for _ in range(depth):
        nxt = []
        for lo, hi in nodes:
            if hi - lo <= PW_BLOCKSIZE:
                return None
            mid = lo + pairwise_split(hi - lo)
            nxt += [(lo, mid), (mid, hi)]
        nodes = nxt
    return nodes


def combine_leaves(vals) -> float:
    """Sum leaf values the way numpy combines the subtrees: ((v0 + v1) + (v2 + v3)) + ..."""
    v = [float(x) for x in vals]
    while len(v) > 1:
        v = [v[i] + v[i + 1] for i in range(0, len(v), 2)]
    return v[0]


@dataclass(frozen=True)
class PointShards:
    """Tree-aligned split of m distinct points over G ranks."""

    m: int
    leaves: tuple      # all leaves (lo, hi), tree order
    owner: tuple       # owner rank of each leaf
    ranges: tuple      # per rank: (lo, hi) point range (empty when the rank owns no leaf)

    def local_leaf_bounds(self, rank: int) -> np.ndarray:
        lo = self.ranges[rank][0]
        mine = [lf for lf, o in zip(self.leaves, self.owner) if o == rank]
        return np.array([mine[0][0] - lo] + [hi - lo for _, hi in mine], dtype=np.int64)


def point_shards(m: int, world: int) -> PointShards | None:
    """None when m is too small to split (every rank then runs the whole problem)."""
    if world == 1:
        return PointShards(m, ((0, m),), (0,), ((0, m),))
    depth = math.ceil(math.log2(world))
    leaves = tree_leaves(m, depth)
    if leaves is None:
        return None
    L = len(leaves)
    owner = tuple(min(world - 1, (i * world) // L) for i in range(L))
    ranges = []
    for r in range(world):
        mine = [lf for lf, o in zip(leaves, owner) if o == r]
        ranges.append((mine[0][0], mine[-1][1]) if mine else (0, 0))
    return PointShards(m, tuple(leaves), owner, tuple(ranges))


# ------------------------------------------------------------------ collectives
class Comm:
    """torch.distributed on one process group; ``run`` orders device work on a stream."""

    def __init__(self, group=None, device=None, stream_scope=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = device
        self.scope = stream_scope
        self.native = None  # NativeComm when the group is an NCCL group (set by the GPU entry points)

    def all_reduce_sum(self, t) -> None:
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)

    def all_gather_f64(self, vals) -> np.ndarray:
        """[world, len(vals)] float64 (values travel as int64 bit patterns: exact)."""
        import torch

        a = np.ascontiguousarray(np.asarray(vals, dtype=np.float64)).view(np.int64)
        t = torch.from_numpy(a.copy()).to(self.device or "cpu")
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return np.stack([o.cpu().numpy() for o in out]).view(np.float64)

    def all_gather_rows(self, rows):
        """Concatenate every rank's int64 tensor (variable lengths) in rank order."""
        import torch

        n = torch.tensor([rows.numel()], dtype=torch.int64, device=rows.device)
        ns = [torch.empty_like(n) for _ in range(self.world)]
        self.dist.all_gather(ns, n, group=self.group)
        sizes = [int(x.item()) for x in ns]
        cap = max(sizes)
        buf = torch.zeros(cap, dtype=torch.int64, device=rows.device)
        buf[: rows.numel()] = rows
        outs = [torch.empty_like(buf) for _ in range(self.world)]
        self.dist.all_gather(outs, buf, group=self.group)
        return torch.cat([o[:s] for o, s in zip(outs, sizes)])


class NativeComm:
    """kt_comm: an NCCL communicator of the engine library over the ranks of ``group`` (the
    unique id is broadcast over the torch process group).  Its all-reduces run on the engine
    stream inside the library: kt_lloyd_run's per-pass k-means exchange and, as a kt_collective
    callback, the PPO statistics / gradient all-reduce — no Python per exchange."""

    _cache: dict = {}

    def __init__(self, eng, group=None):
        import torch.distributed as dist

        self.eng = eng
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        uid = np.zeros(128, dtype=np.uint8)
        if self.rank == 0:
            _lib.call("kt_comm_unique_id", _lib.as_ptr(uid, C.c_uint8))
        obj = [uid.tobytes()]
        src = dist.get_global_rank(group, 0) if group is not None else 0
        dist.broadcast_object_list(obj, src=src, group=group)
        uid = np.frombuffer(obj[0], dtype=np.uint8).copy()
        h = _lib.P()
        _lib.call("kt_comm_create", eng.handle, _lib.as_ptr(uid, C.c_uint8), self.rank, self.world, C.byref(h))
        self.handle = h

    @classmethod
    def for_group(cls, eng, group=None):
        """One communicator per (engine, group) for the life of the process, or None when the
        group is not an NCCL group (gloo / CPU tests keep the torch.distributed path)."""
        import torch.distributed as dist

        if dist.get_backend(group) != "nccl" or os.environ.get("KT_NATIVE_COMM", "1") == "0":
            return None
        key = (id(eng), id(group), dist.get_rank(group), dist.get_world_size(group))
        if key not in cls._cache:
            cls._cache[key] = cls(eng, group)
        return cls._cache[key]

    def collective(self, episode_offset: int):
        """kt_collective whose callback is kt_comm_all_reduce_f64 itself (a C function)."""
        fn = C.cast(_lib.load().kt_comm_all_reduce_f64, C.c_void_p).value
        return _lib.Collective(_lib.ALL_REDUCE_F64(fn), self.handle, int(episode_offset))


# ------------------------------------------------------------------ GPU backend
class GpuLloydShard:
    """kt_lloyd_*: Lloyd passes of one rank's point shard on its GPU."""

    def __init__(self, eng, shard_rows_dev, n_knobs: int, cards, ks, init_rows: np.ndarray):
        import torch

        self.eng = eng
        self.rows = shard_rows_dev  # keep alive
        self.n = n_knobs
        self.ks = list(ks)
        self.cards = np.ascontiguousarray(cards, dtype=np.int32)
        h = _lib.P()
        kk = np.array(self.ks, dtype=np.int32)
        init = np.ascontiguousarray(init_rows, dtype=np.uint64)
        _lib.call("kt_lloyd_create", eng.handle, _lib.ptr(shard_rows_dev), int(shard_rows_dev.numel()), n_knobs,
                  _lib.as_ptr(self.cards, C.c_int32), len(self.ks), _lib.as_ptr(kk, C.c_int32),
                  _lib.as_ptr(init, C.c_uint64), C.byref(h))
        self.h = h
        self.K = int(sum(self.ks))
        self.ext = torch.zeros(self.K * 9 + len(self.ks), dtype=torch.int64, device=f"cuda:{eng.device}")
        self.m = int(shard_rows_dev.numel())

    def __del__(self):
        try:
            _lib.load().kt_lloyd_destroy(self.h)
        except Exception:
            pass

    def local_pass(self):
        _lib.call("kt_lloyd_pass", self.eng.handle, self.h, _lib.ptr(self.ext))
        return self.ext

    def run(self, native: "NativeComm", batch: int = 8):
        """Device-driven passes (kt_lloyd_run) until convergence or a reseed."""
        st = np.zeros(len(self.ks), dtype=np.int32)
        ps = np.zeros(len(self.ks), dtype=np.int32)
        reseed = C.c_int32(0)
        _lib.call("kt_lloyd_run", self.eng.handle, self.h, native.handle if native is not None else None, int(batch),
                  _lib.as_ptr(st, C.c_int32), _lib.as_ptr(ps, C.c_int32), C.byref(reseed))
        return st.tolist(), ps.tolist()

    def apply(self, ext):
        st = np.zeros(len(self.ks), dtype=np.int32)
        ps = np.zeros(len(self.ks), dtype=np.int32)
        _lib.call("kt_lloyd_apply", self.eng.handle, self.h, _lib.ptr(ext), _lib.as_ptr(st, C.c_int32),
                  _lib.as_ptr(ps, C.c_int32))
        return st.tolist(), ps.tolist()

    def sums(self) -> np.ndarray:
        out = np.zeros((self.K, 9), dtype=np.int64)
        _lib.call("kt_lloyd_sums", self.eng.handle, self.h, _lib.as_ptr(out, C.c_int64))
        return out

    def farthest(self, run: int, blocked_local) -> tuple[float, int]:
        b = np.ascontiguousarray(blocked_local, dtype=np.int64)
        d2, idx = C.c_double(0), C.c_int64(-1)
        if self.m == 0:
            return -1.0, -1
        _lib.call("kt_lloyd_farthest", self.eng.handle, self.h, run, _lib.as_ptr(b, C.c_int64), len(b),
                  C.byref(d2), C.byref(idx))
        return float(d2.value), int(idx.value)

    def set_centroids(self, run: int, cent: np.ndarray) -> None:
        c = np.ascontiguousarray(cent, dtype=np.float64)
        _lib.call("kt_lloyd_set_centroids", self.eng.handle, self.h, run, _lib.as_ptr(c, C.c_double))

    def centroids(self, run: int) -> np.ndarray:
        out = np.zeros((self.ks[run], self.n), dtype=np.float64)
        _lib.call("kt_lloyd_centroids", self.eng.handle, self.h, run, _lib.as_ptr(out, C.c_double))
        return out

    def assignment(self, run: int) -> np.ndarray:
        out = np.zeros(self.m, dtype=np.int64)
        _lib.call("kt_lloyd_assignment", self.eng.handle, self.h, run, _lib.as_ptr(out, C.c_int64))
        return out

    def leaf_losses(self, run: int, bounds: np.ndarray) -> np.ndarray:
        b = np.ascontiguousarray(bounds, dtype=np.int64)
        out = np.zeros(len(b) - 1, dtype=np.float64)
        _lib.call("kt_lloyd_leaf_losses", self.eng.handle, self.h, run, _lib.as_ptr(b, C.c_int64), len(b) - 1,
                  _lib.as_ptr(out, C.c_double))
        return out


# ------------------------------------------------------------------ the sharded Lloyd loop
@dataclass
class RunResult:
    k: int
    loss: float
    passes: int
    centroids: np.ndarray


def lloyd_runs(backend, comm: Comm, shards: PointShards, full_rows_host: np.ndarray, n_knobs: int, fmt_get,
               scope=None) -> list[RunResult]:
    """Run every k of ``backend`` to convergence; identical results on every rank.

    ``full_rows_host``: the distinct points (replicated), for reseeding at a chosen
    global index; ``fmt_get(rows) -> (len, n)`` unpacks rows to coordinates.
    """
    import contextlib

    scope = scope or contextlib.nullcontext
    rank = comm.rank
    lo, hi = shards.ranges[rank]
    ks = backend.ks
    offs = np.concatenate([[0], np.cumsum(ks)]).astype(int)
    states = [1] * len(ks)
    passes = [0] * len(ks)
    native = getattr(comm, "native", None)
    while any(s in ACTIVE_STATES for s in states):
        with scope():
            if native is not None and hasattr(backend, "run"):
                states, passes = backend.run(native)  # passes + NCCL exchange on the device
            else:
                ext = backend.local_pass()
                comm.all_reduce_sum(ext)
                states, passes = backend.apply(ext)
        if NEEDS_RESEED in states:
            S = backend.sums()
            for r, st in enumerate(states):
                if st != NEEDS_RESEED:
                    continue
                sums = S[offs[r]:offs[r + 1]]
                cent = np.zeros((ks[r], n_knobs), dtype=np.float64)
                blocked: list[int] = []
                for j in range(ks[r]):
                    if sums[j, 8] > 0:
                        cent[j] = sums[j, :n_knobs].astype(np.float64) / float(sums[j, 8])
                for j in range(ks[r]):
                    if sums[j, 8] > 0:
                        continue
                    local_blocked = [g - lo for g in blocked if lo <= g < hi]
                    d2, idx = backend.farthest(r, local_blocked)
                    cand = comm.all_gather_f64([d2, float(lo + idx) if idx >= 0 else -1.0])
                    best_v, best_i = -1.0, -1
                    for v, i in cand:
                        i = int(i)
                        if i >= 0 and (best_i < 0 or v > best_v or (v == best_v and i < best_i)):
                            best_v, best_i = v, i
                    if best_i < 0:
                        raise RuntimeError("no point left to reseed an empty cluster")
                    blocked.append(best_i)
                    cent[j] = fmt_get(full_rows_host[best_i:best_i + 1])[0]
                backend.set_centroids(r, cent)
                states[r] = 1
    bounds = shards.local_leaf_bounds(rank) if hi > lo else None
    out = []
    for r, k in enumerate(ks):
        mine = backend.leaf_losses(r, bounds) if bounds is not None else np.zeros(0)
        gathered = comm.all_gather_f64(np.pad(mine, (0, 2 - len(mine)), constant_values=np.nan))
        leaf_vals = []
        per_rank = {q: [v for v in gathered[q] if not np.isnan(v)] for q in range(comm.world)}
        cursor = {q: 0 for q in range(comm.world)}
        for o in shards.owner:
            leaf_vals.append(per_rank[o][cursor[o]])
            cursor[o] += 1
        out.append(RunResult(k, combine_leaves(leaf_vals), passes[r], backend.centroids(r)))
    return out


def next_batch(k0: int, upper: int, rnd: int) -> list[int]:
    """Speculative k batches of the knee scan (same widths as the engine: 2, 2, 4, 8, ...)."""
    widths = (2, 2, 4, 8)
    want = widths[rnd] if rnd < 4 else 8
    ks, total = [], 0
    for k in range(k0, upper + 1):
        if len(ks) >= want or total + k > 256:
            break
        ks.append(k)
        total += k
    return ks


def knee_scan_sharded(make_backend, comm: Comm, shards: PointShards, full_rows_host: np.ndarray, n_knobs: int,
                      fmt_get, init_rows_fn, knee_constant: float = KNEE_CONSTANT, k_max: int = KNEE_K_MAX,
                      scope=None):
    """knee_scan (sampler.py:125-148) over sharded points -> (chosen RunResult, [(k, L_k)])."""
    upper = min(k_max, shards.m)
    if upper < KNEE_K_MIN:
        raise ValueError("knee scan needs at least 8 distinct points")
    init = init_rows_fn(upper)  # k-means++ rows, init(k) is a prefix of init(k+1)
    previous = math.inf
    scanned = []
    k0, rnd = KNEE_K_MIN, 0
    while k0 <= upper:
        ks = next_batch(k0, upper, rnd)
        res = lloyd_runs(make_backend(ks, init[: max(ks)]), comm, shards, full_rows_host, n_knobs, fmt_get, scope)
        for r, rr in enumerate(res):
            scanned.append((rr.k, rr.loss))
            if knee_constant * rr.loss > previous:
                return rr, scanned
            previous = rr.loss
        if ks[-1] >= upper:
            return res[-1], scanned
        k0, rnd = ks[-1] + 1, rnd + 1
    raise RuntimeError("knee scan ended without a result")


# ------------------------------------------------------------------ drop-in (GPU)
def adaptive_sample_sharded(rows_local, visited, space, seed: int, group=None,
                            knee_constant: float = KNEE_CONSTANT):
    """adaptive_sample (sampler.py:173-215) for one task whose candidates are sharded
    over the ranks of ``group`` (contiguous, rank order = trajectory order).

    Returns the batch rows (np.uint64), identical on every rank of the group.
    """
    import torch

    from . import sampler as samp

    eng = _lib.engine()
    comm = Comm(group, device=f"cuda:{eng.device}")
    comm.native = NativeComm.for_group(eng, group)
    cards = np.ascontiguousarray(sp.check_engine_space(space), dtype=np.int32)
    n = cards.size
    with eng.scope():
        all_rows = comm.all_gather_rows(rows_local.view(torch.int64).reshape(-1))
    count = int(all_rows.numel())
    distinct = torch.empty_like(all_rows)
    nd = C.c_int64(0)
    with eng.scope():
        _lib.call("kt_dedup", eng.handle, _lib.ptr(all_rows), count, _lib.ptr(distinct), C.byref(nd))
    m = int(nd.value)
    distinct = distinct[:m]
    host_distinct = distinct.cpu().numpy().view(np.uint64)
    vis = visited if isinstance(visited, np.ndarray) else samp.visited_rows(visited, cards)
    vis = np.ascontiguousarray(vis, dtype=np.uint64)
    if m <= KNEE_K_MIN:
        vset = set(vis.tolist())
        return np.array([r for r in host_distinct.tolist() if r not in vset], dtype=np.uint64)
    shards = point_shards(m, comm.world)
    if shards is None:  # too few points to split: every rank runs the single-GPU path
        return samp.adaptive_sample_rows(all_rows, vis, space, seed, knee_constant)
    lo, hi = shards.ranges[comm.rank]

    def fmt_get(rows):
        return sp.unpack(np.asarray(rows, dtype=np.uint64), n, space.cardinalities).astype(np.float64)

    def init_rows_fn(k):
        out = np.zeros(k, dtype=np.uint64)
        with eng.scope():
            _lib.call("kt_kmeanspp_rows", eng.handle, _lib.ptr(distinct), m, n, _lib.as_ptr(cards, C.c_int32),
                      int(seed) & (2**64 - 1), k, _lib.as_ptr(out, C.c_uint64))
        return out

    def make_backend(ks, init):
        return GpuLloydShard(eng, distinct[lo:hi], n, cards, ks, init)

    chosen, _ = knee_scan_sharded(make_backend, comm, shards, host_distinct, n, fmt_get, init_rows_fn,
                                  knee_constant, scope=eng.scope)
    mode = np.zeros(n, dtype=np.int32)
    with eng.scope():
        _lib.call("kt_mode_vote", eng.handle, _lib.ptr(all_rows), count, n, _lib.as_ptr(cards, C.c_int32),
                  _lib.as_ptr(mode, C.c_int32))
    return assemble_batch(chosen.centroids, mode, vis, space.cardinalities)


def assemble_batch(centroids: np.ndarray, mode, visited_rows: np.ndarray, cards) -> np.ndarray:
    """Batch assembly (sampler.py:200-215): round each centroid; a visited one becomes the
    mode (dropped if the mode is visited too); duplicates dropped; centroid order kept."""
    vset = set(np.asarray(visited_rows, dtype=np.uint64).tolist())
    n = len(cards)
    mode_row = int(sp.pack(np.asarray(mode, dtype=np.int64).reshape(1, n), cards)[0])
    out, taken = [], set()
    for c in np.asarray(centroids, dtype=np.float64):
        idx = np.minimum(np.maximum(np.floor(c + 0.5), 0), np.asarray(cards) - 1).astype(np.int64)
        row = int(sp.pack(idx.reshape(1, n), cards)[0])
        if row in vset:
            row = mode_row
            if row in vset:
                continue
        if row in taken:
            continue
        taken.add(row)
        out.append(row)
    return np.array(out, dtype=np.uint64)


# ------------------------------------------------------------------ sharded search round (GPU)
def run_search_rows_sharded(agent, model, space, start_rows_local, episode_offset: int, group=None, engine=None,
                            info=None):
    """run_search_round (agent.py:267-366) with the round's episodes sharded over ``group``.

    This rank runs episodes [episode_offset, episode_offset + len(start_rows_local)) —
    rollouts and scoring need no communication — and the PPO update all-reduces the
    reward / advantage statistics and the float64 gradients of every epoch (19,289
    values for 8 knobs), so every rank applies the same Adam step and the agent
    replicas stay identical.  Returns this shard's (rows, scores, steps).
    """
    from .agent import run_search_rows

    eng = engine if engine is not None else _lib.engine()
    native = NativeComm.for_group(eng, group)
    if native is not None:  # statistics and gradients all-reduced by NCCL inside the library
        return run_search_rows(agent, model, space, start_rows_local, engine=eng, info=info,
                               collective=native.collective(episode_offset), episode_offset=episode_offset)
    comm = Comm(group)
    return run_search_rows(agent, model, space, start_rows_local, engine=eng, info=info,
                           all_reduce=comm.all_reduce_sum, episode_offset=episode_offset)
