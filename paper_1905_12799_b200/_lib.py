"""ctypes binding of libknobtuner_b200.so (include/knobtuner_b200.h).

There is no CPU fallback: if the library or a CUDA device is missing, every
engine call raises ``EngineUnavailable`` (a RuntimeError) with the reason.
"""

from __future__ import annotations

import contextlib
import os
import ctypes as C
import re
import threading
from pathlib import Path

from . import errors

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["KT_LIB_PATH"]) if os.environ.get("KT_LIB_PATH") else PKG / "lib" / "libknobtuner_b200.so"
HEADER = PKG.parent / "include" / "knobtuner_b200.h"

KT_OK, KT_ERR_VALUE, KT_ERR_DIMENSION, KT_ERR_SPACE, KT_ERR_UNSUPPORTED = 0, 1, 2, 3, 4

P = C.c_void_p
i32, i64, u64, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double
pi32, pi64, pu64, pf64, pu32 = (C.POINTER(t) for t in (C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_uint32))


class EngineUnavailable(RuntimeError):
    """The CUDA engine library or device is not available (no CPU fallback exists)."""


class SampleInfo(C.Structure):
    _fields_ = [
        ("n_distinct", C.c_int64),
        ("chosen_k", C.c_int32),
        ("n_scanned", C.c_int32),
        ("scanned_k", C.c_int32 * 56),
        ("scanned_loss", C.c_double * 56),
        ("lloyd_passes", C.c_int32),
        ("used_mode", C.c_int32),
        ("lloyd_launches", C.c_int32),
        ("lloyd_bytes", C.c_int64),
    ]


class RoundInfo(C.Structure):
    _fields_ = [("steps", C.c_int64), ("entries", C.c_int64), ("guarded", C.c_int64),
                ("policy_loss", C.c_double), ("value_loss", C.c_double), ("entropy", C.c_double),
                ("total", C.c_double), ("guard_tau", C.c_double)]


class PPOHyper(C.Structure):
    _fields_ = [("adam_step_size", C.c_double), ("discount", C.c_double), ("gae_parameter", C.c_double),
                ("clip", C.c_double), ("value_coef", C.c_double), ("entropy_coef", C.c_double),
                ("epochs", C.c_int32), ("max_steps", C.c_int32)]


# name -> (restype, argtypes); every entry must exist in the header and the .so
ALL_REDUCE_F64 = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64)


class Collective(C.Structure):
    """kt_collective: in-place SUM of device doubles over the ranks + this shard's episode offset."""

    _fields_ = [("all_reduce_sum_f64", ALL_REDUCE_F64), ("user", C.c_void_p), ("episode_offset", C.c_int64)]


class _DeviceArray:
    """Zero-copy view of raw device memory for torch.as_tensor (__cuda_array_interface__ v2)."""

    def __init__(self, ptr: int, count: int, typestr: str = "<f8"):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 2}


def device_tensor(ptr: int, count: int, device: int, typestr: str = "<f8"):
    import torch

    return torch.as_tensor(_DeviceArray(ptr, count, typestr), device=f"cuda:{device}")


SIGNATURES = {
    "kt_last_error": (C.c_char_p, []),
    "kt_version": (C.c_char_p, []),
    "kt_row_layout": (C.c_int, [pi32, C.c_int, pi32, pi32]),
    "kt_engine_create": (C.c_int, [C.c_int, C.POINTER(P)]),
    "kt_engine_destroy": (C.c_int, [P]),
    "kt_engine_set_stream": (C.c_int, [P, P]),
    "kt_engine_synchronize": (C.c_int, [P]),
    "kt_engine_order": (C.c_int, [P, P, C.c_int]),
    "kt_engine_launch_count": (C.c_int64, [P]),
    "kt_engine_set_timing": (C.c_int, [P, C.c_int]),
    "kt_engine_kernel_stats": (C.c_int, [P, C.c_int, C.c_char_p, pi64, pf64, pi32, C.c_int]),
    "kt_pcg64_draw": (C.c_int, [pu32, C.c_int, pu32, C.c_int, C.c_int, u64, i64, P]),
    "kt_forest_create": (C.c_int, [P, C.c_int, pi32, pf64, C.c_int, C.c_int, pi32, pi32, pf64, pi32, pi32, pf64,
                                   f64, C.POINTER(P)]),
    "kt_forest_destroy": (C.c_int, [P]),
    "kt_forest_depth": (C.c_int, [P]),
    "kt_score_trees": (C.c_int, [P, P, P, i64, P]),
    "kt_landscape_create": (C.c_int, [P, C.c_int, pi32, C.c_int, pi32, pf64, pf64, f64, f64, C.c_char_p, C.POINTER(P)]),
    "kt_landscape_destroy": (C.c_int, [P]),
    "kt_score_landscape": (C.c_int, [P, P, P, i64, P]),
    "kt_landscape_best": (C.c_int, [P, P, pi32, pf64, pi64]),
    "kt_top_unvisited": (C.c_int, [P, P, P, i64, pu64, i64, C.c_int, pu64, pi32]),
    "kt_dedup": (C.c_int, [P, P, i64, P, pi64]),
    "kt_mode_vote": (C.c_int, [P, P, i64, C.c_int, pi32, pi32]),
    "kt_kmeans": (C.c_int, [P, P, i64, C.c_int, pi32, C.c_int, u64, pf64, pi64, pf64, pf64, pi32]),
    "kt_knee_scan": (C.c_int, [P, P, i64, C.c_int, pi32, u64, f64, C.c_int, pi32, pf64, pi32, pf64, pi64]),
    "kt_adaptive_sample": (C.c_int, [P, P, i64, C.c_int, pi32, pu64, i64, u64, f64, pu64, pi32,
                                     C.POINTER(SampleInfo)]),
    "kt_lloyd_create": (C.c_int, [P, P, i64, C.c_int, pi32, C.c_int, pi32, pu64, C.POINTER(P)]),
    "kt_lloyd_destroy": (C.c_int, [P]),
    "kt_lloyd_clusters": (C.c_int, [P, pi32]),
    "kt_lloyd_pass": (C.c_int, [P, P, P]),
    "kt_lloyd_apply": (C.c_int, [P, P, P, pi32, pi32]),
    "kt_lloyd_sums": (C.c_int, [P, P, pi64]),
    "kt_lloyd_run": (C.c_int, [P, P, P, C.c_int, pi32, pi32, pi32]),
    "kt_comm_unique_id": (C.c_int, [P]),
    "kt_comm_create": (C.c_int, [P, P, C.c_int, C.c_int, C.POINTER(P)]),
    "kt_comm_destroy": (C.c_int, [P]),
    "kt_comm_all_reduce_f64": (C.c_int, [P, P, i64]),
    "kt_comm_all_reduce_i64": (C.c_int, [P, P, i64]),
    "kt_lloyd_farthest": (C.c_int, [P, P, C.c_int, pi64, C.c_int, pf64, pi64]),
    "kt_lloyd_set_centroids": (C.c_int, [P, P, C.c_int, pf64]),
    "kt_lloyd_centroids": (C.c_int, [P, P, C.c_int, pf64]),
    "kt_lloyd_assignment": (C.c_int, [P, P, C.c_int, pi64]),
    "kt_lloyd_leaf_losses": (C.c_int, [P, P, C.c_int, pi64, C.c_int, pf64]),
    "kt_gae": (C.c_int, [P, P, P, P, C.c_int32, f64, f64, P]),
    "kt_fit_trees": (C.c_int, [pf64, pf64, i64, C.c_int, C.c_int, C.c_int, f64, pi32, pf64, pi32, pi32, pf64, i64,
                               pi32, pf64]),
    "kt_fit_trees_device": (C.c_int, [P, pf64, pf64, i64, C.c_int, C.c_int, C.c_int, f64, pi32, pf64, pi32, pi32,
                                      pf64, i64, pi32, pf64]),
    "kt_step_best": (C.c_int, [P, P, P, i64, C.c_int, pf64, pi32]),
    "kt_pca_moments": (C.c_int, [P, P, i64, C.c_int, pi32, pi64, pi64]),
    "kt_pca_project": (C.c_int, [P, P, i64, C.c_int, pi32, pf64, pf64, pf64, P, P]),
    "kt_kmeanspp_rows": (C.c_int, [P, P, i64, C.c_int, pi32, u64, C.c_int, pu64]),
    "kt_agent_create": (C.c_int, [P, C.c_int, C.c_int, C.c_int, pf64, pf64, pf64, i64, C.POINTER(P)]),
    "kt_agent_destroy": (C.c_int, [P]),
    "kt_agent_get_state": (C.c_int, [P, P, pf64, pf64, pf64, pi64]),
    "kt_search_round": (C.c_int, [P, P, P, P, i32, pi32, C.c_int, pu32, C.c_int, i64, C.POINTER(PPOHyper), P, P, P,
                                  pi64, C.POINTER(RoundInfo), P, P]),
    "kt_search_round_ex": (C.c_int, [P, P, P, P, i32, pi32, C.c_int, pu32, C.c_int, i64, C.POINTER(PPOHyper), P, P, P,
                                  pi64, C.POINTER(RoundInfo), P, P, C.POINTER(Collective)]),
    "kt_gemm_f32": (C.c_int, [P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, P, C.c_int, P, C.c_int, P, C.c_int]),
    "kt_sa_chains": (C.c_int, [P, P, P, i32, i32, i32, pi32, C.c_int, pu32, C.c_int, C.c_int, f64, f64, P, P, P,
                               pi64]),
}

_lock = threading.Lock()
_lib = None
_load_error: str | None = None
_engines: dict[int, "Engine"] = {}


def header_symbols() -> list[str]:
    """Function names declared by include/knobtuner_b200.h."""
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(kt_[a-z0-9_]+)\s*\(", text)))


def load(path: Path | None = None):
    """Load the shared library (no GPU needed).  Raises EngineUnavailable if absent."""
    global _lib, _load_error
    with _lock:
        if _lib is not None:
            return _lib
        p = Path(path) if path else LIB_PATH
        if not p.exists():
            _load_error = f"{p} not built (run __graft_entry__.build() or python -m paper_1905_12799_b200.build)"
            raise EngineUnavailable(_load_error)
        lib = C.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def raise_for(code: int) -> None:
    if code == KT_OK:
        return
    msg = (_lib.kt_last_error() or b"").decode("utf-8", "replace")
    if code == KT_ERR_VALUE:
        raise ValueError(msg)
    if code == KT_ERR_DIMENSION:
        raise errors.DimensionMismatchError(msg)
    if code == KT_ERR_SPACE:
        raise errors.SpaceValidationError(msg)
    if code == KT_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(f"knobtuner_b200 engine error {code}: {msg}")


def call(name: str, *args) -> None:
    raise_for(getattr(load(), name)(*args))


class Engine:
    """One per CUDA device; wraps kt_engine (stream + workspace)."""

    def __init__(self, device: int):
        import torch

        lib = load()
        h = P()
        raise_for(lib.kt_engine_create(int(device), C.byref(h)))
        self.handle = h
        self.device = int(device)
        # all engine work is ordered on one torch-visible stream
        self.stream = torch.cuda.Stream(device=self.device)
        raise_for(lib.kt_engine_set_stream(h, P(self.stream.cuda_stream)))
        self._lib = lib
        self._raw = int(self.stream.cuda_stream)
        self._ids = (self.stream.stream_id, self.stream.device_index, self.stream.device_type)

    @contextlib.contextmanager
    def scope(self):
        """Run a block on the engine stream, ordered after/before the caller's stream.

        Lean on purpose (it brackets every engine call): the ordering is one event record + wait
        each way inside the library, and the current-stream switch uses torch's raw accessors —
        the torch.cuda.stream / wait_stream Python layers cost ~50 us per call."""
        import torch

        tc = torch._C
        prev_dev = tc._cuda_getDevice()
        if prev_dev != self.device:
            tc._cuda_setDevice(self.device)
        caller_raw = tc._cuda_getCurrentRawStream(self.device)
        prev = tc._cuda_getCurrentStream(self.device)  # (stream_id, device_index, device_type)
        lib = self._lib
        same = caller_raw == self._raw
        if not same:
            raise_for(lib.kt_engine_order(self.handle, P(caller_raw), 0))
            tc._cuda_setStream(*self._ids)
        try:
            yield self
        finally:
            if not same:
                tc._cuda_setStream(*prev)
                raise_for(lib.kt_engine_order(self.handle, P(caller_raw), 1))
            if prev_dev != self.device:
                tc._cuda_setDevice(prev_dev)

    @property
    def launches(self) -> int:
        return int(load().kt_engine_launch_count(self.handle))

    def synchronize(self) -> None:
        call("kt_engine_synchronize", self.handle)

    def set_timing(self, enabled: bool) -> None:
        call("kt_engine_set_timing", self.handle, int(bool(enabled)))

    def kernel_stats(self, reset: bool = True) -> dict[str, tuple[int, float]]:
        """{kernel name: (launches, total ms)} recorded while timing was on."""
        cap = 64
        names = C.create_string_buffer(cap * 32)
        counts = (C.c_int64 * cap)()
        ms = (C.c_double * cap)()
        n = C.c_int32(0)
        call("kt_engine_kernel_stats", self.handle, cap, names, counts, ms, C.byref(n), int(reset))
        out = {}
        for i in range(n.value):
            name = names.raw[i * 32:(i + 1) * 32].split(b"\0", 1)[0].decode()
            out[name] = (int(counts[i]), float(ms[i]))
        return out

    def set_stream(self, stream) -> None:
        """Order the engine's work on ``stream`` (a torch.cuda.Stream) instead of its own."""
        import torch

        stream = stream if stream is not None else torch.cuda.Stream(device=self.device)
        call("kt_engine_set_stream", self.handle, P(stream.cuda_stream))
        self.stream = stream
        self._raw = int(stream.cuda_stream)
        self._ids = (stream.stream_id, stream.device_index, stream.device_type)


def engine(device: int | None = None) -> Engine:
    """The engine for ``device`` (default: torch's current CUDA device)."""
    import torch

    if not torch.cuda.is_available():
        raise EngineUnavailable("no CUDA device visible; the B200 engine has no CPU fallback")
    dev = torch.cuda.current_device() if device is None else int(device)
    with _lock:
        e = _engines.get(dev)
    if e is None:
        e = Engine(dev)
        with _lock:
            _engines[dev] = e
    return e


def ptr(t) -> P:
    """Raw device/host pointer of a torch tensor or numpy array."""
    if hasattr(t, "data_ptr"):
        return P(t.data_ptr())
    return P(t.ctypes.data)


def as_ptr(arr, ctype):
    return arr.ctypes.data_as(C.POINTER(ctype))
