"""Bundled spaces and definitions.

``stencil3d_space`` / ``stencil3d_definition`` / ``vector_add_definition``
reproduce the reference presets (pkg/src/kltune/presets.py:15-89): the paper's
Table 2 space — 5*5*5 * 3^3 * 2^6 * 6 * 6 = 7,776,000 raw points, optional
``block_x * block_y * block_z <= 1024`` — and the tile-aware 3-D grid rule.
Their fingerprints (hence kernel keys) equal the reference's.

The real MicroHH kernels (``advec_u`` / ``diff_uvw`` in fp32 and fp64) live in
``paper_2303_12374_b200.stencils.definitions``: same Table 2 parameters plus
the B200 staging knobs, with CUDA bodies.
"""

from __future__ import annotations

from .kerneldef import KernelBuilder, KernelDefinition
from .space import ConfigSpace, TunableParam

__all__ = [
    "BLOCK_LIMIT_RESTRICTION", "UNRAVEL_ORDERS", "table2_params", "stencil3d_space", "stencil3d_definition",
    "vector_add_definition",
]

BLOCK_LIMIT_RESTRICTION = "block_x * block_y * block_z <= 1024"
UNRAVEL_ORDERS = ("XYZ", "XZY", "YXZ", "YZX", "ZXY", "ZYX")

_GRID3D_DECL = """\
template<int TILE_TOTAL>
__global__ void grid3d(float *out, const float *in, int nx, int ny, int nz);
"""

_VECTOR_ADD_DECL = """\
template<int block_size>
__global__ void vector_add(float *c, const float *a, const float *b, int n);
"""


def table2_params() -> list[TunableParam]:
    """The paper's Table 2 knobs in declaration order."""
    knobs = [
        TunableParam("block_x", (16, 32, 64, 128, 256), 256),
        TunableParam("block_y", (1, 2, 4, 8, 16), 1),
        TunableParam("block_z", (1, 2, 4, 8, 16), 1),
    ]
    knobs += [TunableParam(f"tile_{a}", (1, 2, 4), 1) for a in "xyz"]
    knobs += [TunableParam(f"unroll_{a}", (True, False), False) for a in "xyz"]
    knobs += [TunableParam(f"contiguous_{a}", (True, False), False) for a in "xyz"]
    knobs.append(TunableParam("unravel", UNRAVEL_ORDERS, "XYZ"))
    knobs.append(TunableParam("min_blocks", (1, 2, 3, 4, 5, 6), 1))
    return knobs


def stencil3d_space(block_limit: bool = True) -> ConfigSpace:
    return ConfigSpace(table2_params(), [BLOCK_LIMIT_RESTRICTION] if block_limit else [])


def stencil3d_definition(block_limit: bool = True) -> KernelDefinition:
    return KernelDefinition(
        "grid3d",
        stencil3d_space(block_limit),
        source_text=_GRID3D_DECL,
        problem_size=("arg2", "arg3", "arg4"),
        block=("block_x", "block_y", "block_z"),
        grid=tuple(f"ceil_div(problem_{a}, block_{a} * tile_{a})" for a in "xyz"),
        defines=[("TILE_TOTAL", "tile_x * tile_y * tile_z")],
        template_args=("tile_x * tile_y * tile_z",),
        flags=("-std=c++17",),
    )


def vector_add_definition() -> KernelDefinition:
    kb = KernelBuilder("vector_add", source_text=_VECTOR_ADD_DECL)
    bs = kb.tune("block_size", [32, 64, 128, 256, 1024], default=128)
    return kb.problem_size("arg3").template_args(bs).block(bs).build()
