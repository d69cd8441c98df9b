"""Design-space data model and the engine's packed row layout.

Mirrors the reference's lattice types (knobtuner/space.py:27-90) closely
enough to be interchangeable: every public function here accepts either these
classes or the reference's own objects (duck typing on ``.knobs``,
``.cardinalities``, ``.indices``).

Engine layout: a configuration is one ``uint64`` *row*.  Spaces of up to 8
knobs with at most 255 settings each use byte i for knob i's index; spaces with
wider knobs (AlexNet's tile_f has 480 settings) pack minimal-width bit fields,
knob i in bits [shift_i, shift_i + width_i), at most 63 bits in all
(``row_layout``; the C side's ``row_fmt`` applies the same rule).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import errors

MAX_KNOBS = 8
MAX_CARD = 255           # byte layout limit
MAX_WIDE_CARD = 65535    # bit-field layout limit
MAX_ROW_BITS = 63


@dataclass(frozen=True)
class KnobDef:
    name: str
    values: tuple[int, ...]

    def __post_init__(self) -> None:
        object.__setattr__(self, "values", tuple(int(v) for v in self.values))
        if not self.name:
            raise errors.SpaceValidationError("knob name must be non-empty")
        if not self.values:
            raise errors.SpaceValidationError(f"knob {self.name!r}: values list is empty")
        if any(b <= a for a, b in zip(self.values, self.values[1:])):
            raise errors.SpaceValidationError(f"knob {self.name!r}: values not strictly increasing")


@dataclass(frozen=True)
class DesignSpace:
    name: str
    knobs: tuple[KnobDef, ...]

    @property
    def n_knobs(self) -> int:
        return len(self.knobs)

    @property
    def cardinalities(self) -> tuple[int, ...]:
        return tuple(len(k.values) for k in self.knobs)

    @property
    def total_cardinality(self) -> int:
        return math.prod(self.cardinalities)


@dataclass(frozen=True)
class Configuration:
    indices: tuple[int, ...]

    def __post_init__(self) -> None:
        object.__setattr__(self, "indices", tuple(int(i) for i in self.indices))
        if any(i < 0 for i in self.indices):
            raise ValueError(f"indices must be non-negative, got {self.indices}")

    def __len__(self) -> int:
        return len(self.indices)


def space_from_dict(obj: dict) -> DesignSpace:
    """Space document (reference JSON schema, space.py:107-129) -> DesignSpace."""
    return DesignSpace(name=obj["name"], knobs=tuple(KnobDef(k["name"], tuple(k["values"])) for k in obj["knobs"]))


def grid(*cards: int) -> DesignSpace:
    """Integer-valued test space, as the reference tests build it."""
    return DesignSpace("grid", tuple(KnobDef(f"k{i}", tuple(range(c))) for i, c in enumerate(cards)))


# ------------------------------------------------------------- duck access
def cardinalities(space) -> np.ndarray:
    return np.asarray(tuple(space.cardinalities), dtype=np.int32)


def knob_values(space) -> list[list[int]]:
    return [list(k.values) for k in space.knobs]


def knob_names(space) -> list[str]:
    return [k.name for k in space.knobs]


def row_layout(cards) -> tuple[np.ndarray, np.ndarray]:
    """(shifts, widths) of each knob's field in a row; bytes when every card <= 255."""
    cards = np.asarray(cards, dtype=np.int64).reshape(-1)
    n = cards.size
    if not 1 <= n <= MAX_KNOBS:
        raise NotImplementedError(f"engine rows hold 1..{MAX_KNOBS} knobs; got {n}")
    if cards.max() <= MAX_CARD:
        return np.arange(n, dtype=np.int64) * 8, np.full(n, 8, dtype=np.int64)
    if cards.max() > MAX_WIDE_CARD:
        raise NotImplementedError(f"engine rows hold knob cardinalities <= {MAX_WIDE_CARD}; got {int(cards.max())}")
    widths = np.array([max(1, int(c - 1).bit_length()) for c in cards], dtype=np.int64)
    shifts = np.concatenate([[0], np.cumsum(widths)[:-1]]).astype(np.int64)
    if int(widths.sum()) > MAX_ROW_BITS:
        raise NotImplementedError(f"the space's knob indices need {int(widths.sum())} bits; rows hold {MAX_ROW_BITS}")
    return shifts, widths


def check_engine_space(space) -> np.ndarray:
    """Cardinalities as int32, or NotImplementedError if outside the row layout."""
    cards = cardinalities(space)
    try:
        row_layout(cards)
    except NotImplementedError as ex:
        raise NotImplementedError(f"space {space.name!r}: {ex}") from None
    return cards


# ------------------------------------------------------------- packing
def pack(idx, cards=None) -> np.ndarray:
    """(N, n) index matrix -> (N,) uint64 rows (byte i = knob i, or the bit fields
    of ``row_layout(cards)`` when a knob has more than 255 settings)."""
    idx = np.asarray(idx)
    if idx.ndim == 1:
        idx = idx[None, :]
    N, n = idx.shape
    if n > MAX_KNOBS:
        raise NotImplementedError(f"engine rows hold at most {MAX_KNOBS} knobs")
    if cards is None or int(np.max(cards)) <= MAX_CARD:
        b = np.zeros((N, 8), dtype=np.uint8)
        b[:, :n] = idx.astype(np.uint8)
        return b.view("<u8").reshape(N)
    shifts, _ = row_layout(cards)
    rows = np.zeros(N, dtype=np.uint64)
    for k in range(n):
        rows |= idx[:, k].astype(np.uint64) << np.uint64(shifts[k])
    return rows


def unpack(rows, n: int, cards=None) -> np.ndarray:
    """(N,) uint64 rows -> (N, n) int64 index matrix."""
    r = np.ascontiguousarray(np.asarray(rows).astype("<u8", copy=False).view(np.uint64))
    if cards is None or int(np.max(cards)) <= MAX_CARD:
        return r.view(np.uint8).reshape(-1, 8)[:, :n].astype(np.int64)
    shifts, widths = row_layout(cards)
    out = np.empty((r.size, n), dtype=np.int64)
    for k in range(n):
        out[:, k] = ((r >> np.uint64(shifts[k])) & np.uint64((1 << int(widths[k])) - 1)).astype(np.int64)
    return out


def validate_index_matrix(space, idx: np.ndarray) -> None:
    """Vectorised validate_config (space.py:151-158): same exception types and messages."""
    idx = np.asarray(idx)
    n = len(space.knobs)
    if idx.ndim != 2 or idx.shape[1] != n:
        width = idx.shape[1] if idx.ndim == 2 else (idx.shape[0] if idx.ndim == 1 else 0)
        raise errors.DimensionMismatchError(
            f"configuration has {width} indices, space {space.name!r} has {n} knobs")
    if idx.size == 0:
        return
    cards = cardinalities(space)
    bad = (idx < 0) | (idx >= cards[None, :])
    if bad.any():
        r, c = np.argwhere(bad)[0]
        raise errors.SpaceValidationError(
            f"knob {space.knobs[c].name!r}: index {int(idx[r, c])} out of range [0, {int(cards[c])})")


def index_matrix(space, configs) -> np.ndarray:
    """Configurations (any objects with ``.indices``) -> validated (N, n) int64 matrix."""
    n = len(space.knobs)
    rows = [c.indices for c in configs]
    if not rows:
        return np.empty((0, n), dtype=np.int64)
    for r in rows:
        if len(r) != n:
            raise errors.DimensionMismatchError(
                f"configuration has {len(r)} indices, space {space.name!r} has {n} knobs")
    idx = np.array(rows, dtype=np.int64)
    validate_index_matrix(space, idx)
    return idx


def rows_from_configs(space, configs) -> np.ndarray:
    return pack(index_matrix(space, configs), cardinalities(space))


def configs_from_rows(rows, n: int, cls=Configuration, cards=None) -> list:
    return [cls(tuple(r)) for r in unpack(rows, n, cards).tolist()]
