"""Synthetic tuning-task spaces of the shapes the benchmark configs name.

The reference ships two small spaces (``pkg/spaces/bench_grid4d.json``,
``pkg/spaces/conv_gpu_table1.json``) and says only that AlexNet / VGG-16 /
ResNet-18 have 5 / 9 / 12 tuning tasks.  The benchmark
needs AutoTVM-cardinality conv spaces, built here from layer shapes with the
paper's Table-1 knob names:

* ``tile_f``/``tile_y``/``tile_x``: ordered 4-way factorisations of the output
  channels / height / width (AutoTVM ``define_split(num_outputs=4)``);
* ``tile_rc``/``tile_ry``/``tile_rx``: 2-way factorisations of the reduction axes;
* ``auto_unroll_max_step`` in {0, 512, 1500}, ``unroll_explicit`` in {0, 1}.

Split knobs take ordinal values 0..card-1 (the factor tuples themselves are not
needed by the surrogate, which only sees log2(1 + value)).  The ResNet-18
3x3 64->64 56x56 layer gives cardinalities (84, 80, 80, 7, 2, 2, 3, 2) =
90,316,800 configurations — survey space "S2".
"""

from __future__ import annotations

from dataclasses import dataclass


def _factorize(n: int) -> dict[int, int]:
    out: dict[int, int] = {}
    p = 2
    while p * p <= n:
        while n % p == 0:
            out[p] = out.get(p, 0) + 1
            n //= p
        p += 1
    if n > 1:
        out[n] = out.get(n, 0) + 1
    return out


def split_count(n: int, parts: int) -> int:
    """Number of ordered factorisations of n into ``parts`` positive factors."""
    from math import comb

    total = 1
    for exp in _factorize(n).values():
        total *= comb(exp + parts - 1, parts - 1)
    return total


@dataclass(frozen=True)
class ConvLayer:
    name: str
    in_ch: int
    out_ch: int
    out_hw: int
    kernel: int

    def knobs(self) -> list[tuple[str, list[int]]]:
        def ordinal(card: int) -> list[int]:
            return list(range(card))

        return [
            ("tile_f", ordinal(split_count(self.out_ch, 4))),
            ("tile_y", ordinal(split_count(self.out_hw, 4))),
            ("tile_x", ordinal(split_count(self.out_hw, 4))),
            ("tile_rc", ordinal(split_count(self.in_ch, 2))),
            ("tile_ry", ordinal(split_count(self.kernel, 2))),
            ("tile_rx", ordinal(split_count(self.kernel, 2))),
            ("auto_unroll_max_step", [0, 512, 1500]),
            ("unroll_explicit", [0, 1]),
        ]

    def space_dict(self) -> dict:
        """Space document in the reference's JSON schema (space.py:107-129)."""
        return {"name": self.name, "knobs": [{"name": k, "values": v} for k, v in self.knobs()]}


@dataclass(frozen=True)
class DenseLayer:
    name: str
    in_features: int
    out_features: int

    def knobs(self) -> list[tuple[str, list[int]]]:
        return [
            ("tile_x", list(range(split_count(self.out_features, 2)))),
            ("tile_k", list(range(split_count(self.in_features, 2)))),
            ("auto_unroll_max_step", [0, 512, 1500]),
            ("unroll_explicit", [0, 1]),
        ]

    def space_dict(self) -> dict:
        return {"name": self.name, "knobs": [{"name": k, "values": v} for k, v in self.knobs()]}


RESNET18_TASKS = (
    ConvLayer("resnet18.c1_7x7_3x64_112", 3, 64, 112, 7),
    ConvLayer("resnet18.c2_3x3_64x64_56", 64, 64, 56, 3),
    ConvLayer("resnet18.c3_1x1_64x128_28", 64, 128, 28, 1),
    ConvLayer("resnet18.c4_3x3_64x128_28", 64, 128, 28, 3),
    ConvLayer("resnet18.c5_3x3_128x128_28", 128, 128, 28, 3),
    ConvLayer("resnet18.c6_1x1_128x256_14", 128, 256, 14, 1),
    ConvLayer("resnet18.c7_3x3_128x256_14", 128, 256, 14, 3),
    ConvLayer("resnet18.c8_3x3_256x256_14", 256, 256, 14, 3),
    ConvLayer("resnet18.c9_1x1_256x512_7", 256, 512, 7, 1),
    ConvLayer("resnet18.c10_3x3_256x512_7", 256, 512, 7, 3),
    ConvLayer("resnet18.c11_3x3_512x512_7", 512, 512, 7, 3),
    DenseLayer("resnet18.dense_512x1000", 512, 1000),
)

# AlexNet's 5 conv layers (configs[1]); conv3-conv5 have tile_f cardinality 480 / 165,
# beyond one byte per knob, so their rows use the variable-width layout (space.row_layout).
ALEXNET_TASKS = (
    ConvLayer("alexnet.c1_11x11_3x96_55", 3, 96, 55, 11),
    ConvLayer("alexnet.c2_5x5_96x256_27", 96, 256, 27, 5),
    ConvLayer("alexnet.c3_3x3_256x384_13", 256, 384, 13, 3),
    ConvLayer("alexnet.c4_3x3_384x384_13", 384, 384, 13, 3),
    ConvLayer("alexnet.c5_3x3_384x256_13", 384, 256, 13, 3),
)

VGG16_TASKS = (
    ConvLayer("vgg16.c1_3x3_3x64_224", 3, 64, 224, 3),
    ConvLayer("vgg16.c2_3x3_64x64_224", 64, 64, 224, 3),
    ConvLayer("vgg16.c3_3x3_64x128_112", 64, 128, 112, 3),
    ConvLayer("vgg16.c4_3x3_128x128_112", 128, 128, 112, 3),
    ConvLayer("vgg16.c5_3x3_128x256_56", 128, 256, 56, 3),
    ConvLayer("vgg16.c6_3x3_256x256_56", 256, 256, 56, 3),
    ConvLayer("vgg16.c7_3x3_256x512_28", 256, 512, 28, 3),
    ConvLayer("vgg16.c8_3x3_512x512_28", 512, 512, 28, 3),
    ConvLayer("vgg16.c9_3x3_512x512_14", 512, 512, 14, 3),
)

# The S2 headline space.
RESNET18_S2 = RESNET18_TASKS[1]
