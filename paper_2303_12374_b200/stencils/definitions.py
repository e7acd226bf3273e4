"""KernelDefinitions of the MicroHH stencils on the reference API.

Each kernel is defined once per precision so the precision reaches the
wisdom key (the reference ``kernel_key`` hashes only the space,
so the name must carry it): ``advec_u_fp32``, ``advec_u_fp64``,
``diff_uvw_fp32`` … for the hot path (``KERNELS``), the fused
``diff_uvw_rk3`` (``FUSED_KERNELS``: the base kernel's source compiled with a
-D switch, same space) and the §8f family (``FAMILY_KERNELS``).

Space = the paper's Table 2 (presets.table2_params, 7,776,000 raw points) plus
three B200 knobs:

``staging``  "DIRECT" (the paper's kernel) | "ZMARCH" (register/shared-memory
             z-marching column) | "TMA" (z-march fed by cp.async.bulk.tensor
             into an mbarrier ring; column tiles; packed fp32 pairs);
``zchunk``   planes marched per block (8..128); 1 under DIRECT, so
             ``block_z * tile_z * zchunk`` is the z extent of a block in every
             family and one grid formula serves the whole space;
``depth``    TMA prefetch depth (planes in flight beyond the ones read).

Restrictions: ``block_x*block_y*block_z <= 1024`` (Table 2 limit); knobs
without meaning in a family pinned (no duplicate binaries); the TMA rings fit
the 227 KB opt-in shared memory for the precision (exact byte expressions,
so fp32 and fp64 spaces differ) and TMA boxes stay <= 256 elements.  The
advection family (advec_v/w/s) and diff_c / evisc_smag have DIRECT + TMA
spaces of the same shape; rk3_uvw is DIRECT only.

Launch geometry: a 1-D list of blocks (the paper's "thread blocks are launched
as a one-dimensional list ... each thread unravels its 1D block identifier",
PAPER.md:425-431) of ``nbx*nby*nbz`` blocks; shared memory is derived per
configuration.  ``KL_JJ``/``KL_KK`` specialise the row/plane pitch from the
launch's scalar arguments.
"""

from __future__ import annotations

import re
from functools import lru_cache
from pathlib import Path

from ..kerneldef import KernelDefinition
from ..presets import BLOCK_LIMIT_RESTRICTION, table2_params
from ..space import ConfigSpace, TunableParam

__all__ = [
    "KERNELS", "PRECISIONS", "stencil_space", "advec_u_definition", "diff_uvw_definition", "definition_for",
    "assemble_source", "ARG_LAYOUT", "family_space", "FAMILY_PINS", "FAMILY_KERNELS", "ALL_KERNELS",
]

_HERE = Path(__file__).resolve().parent
PRECISIONS = {"fp32": "float", "fp64": "double"}
KERNELS = ("advec_u", "diff_uvw")
#: the rest of the MicroHH stencil family: DIRECT staging
FAMILY_KERNELS = ("advec_v", "advec_w", "advec_s", "diff_c", "evisc_smag", "rk3_uvw")
#: family kernels that also have a TMA-staged flux-form variant (advec_family_tma.cuh)
ADV_FAMILY = ("advec_v", "advec_w", "advec_s")
#: family kernels with a TMA z-march over 1-halo planes: (halo'd inputs, RMW output, ring slots - depth)
#: — diff_c: kl_plane_tma.cuh (planes k-1..k+1 per step); evisc_smag: evisc_smag_tma.cuh (planes k, k+1)
PLANE_FAMILY = {"diff_c": (2, 1, 3), "evisc_smag": (3, 0, 2)}
#: hot-path kernels with a fused epilogue: same space and
#: staging families as their base kernel, compiled with a -D switch
FUSED_KERNELS = {"diff_uvw_rk3": ("diff_uvw", "KL_RK3"),
                 # z-slab halo fused into the TMA staging: planes outside the
                 # slab are read from the neighbours' fields (diff_uvw.cu /
                 # advec_u.cu KL_PEER)
                 "diff_uvw_peer": ("diff_uvw", "KL_PEER"),
                 "advec_u_peer": ("advec_u", "KL_PEER"),
                 # both: the RK3 substep of a multi-GPU time loop (slab.SlabDriver.rk3_substep)
                 "diff_uvw_rk3_peer": ("diff_uvw", "KL_RK3 KL_PEER")}
ALL_KERNELS = KERNELS + tuple(FUSED_KERNELS) + FAMILY_KERNELS


def base_kernel(kernel: str) -> str:
    """The kernel whose source, space and shared-memory layout ``kernel`` uses."""
    return FUSED_KERNELS[kernel][0] if kernel in FUSED_KERNELS else kernel

STAGING_VALUES = ("DIRECT", "ZMARCH", "TMA")
#: ``xshare`` (evisc_smag TMA, tile_x == 1): lane 31 of each warp evaluates
#: only the west-face edges of the next column and every lane takes its east
#: edges from its right neighbour by shuffle — 31 output columns per warp
#: (evisc_smag_tma.cuh KL_XSHARE)
XSHARE_KERNELS = ("evisc_smag",)
#: ``ysplit`` (advec_u TMA): 0 = blocks of block_y*tile_y rows; k > 0 = the y
#: extent cut into near-equal runs of at most block_y*tile_y rows, as many as
#: make nbx*nby*nbz ~ k blocks per SM of the B200's 148 (a grid of whole
#: waves whatever jtot / rows-per-block is; advec_u_tma.cuh KL_YBAL)
YSPLIT_KERNELS = ("advec_u",)
YSPLIT_VALUES = (0, 1, 2)
B200_SMS = 148
DEPTH_VALUES = (0, 1, 2, 3)
ZCHUNK_VALUES = (1, 8, 16, 32, 64, 128)

#: argument positions of each kernel's MicroHH-style signature
ARG_LAYOUT = {
    "advec_u": {
        "buffers": [("ut", "output"), ("u", "input"), ("v", "input"), ("w", "input"),
                    ("rhoref", "input"), ("rhorefh", "input"), ("dzi", "input")],
        "scalars": ["dxi", "dyi", "jj", "kk", "istart", "jstart", "kstart", "iend", "jend", "kend"],
    },
    "diff_uvw": {
        "buffers": [("ut", "output"), ("vt", "output"), ("wt", "output"), ("evisc", "input"), ("u", "input"),
                    ("v", "input"), ("w", "input"), ("dzi", "input"), ("dzhi", "input"), ("rhoref", "input"),
                    ("rhorefh", "input")],
        "scalars": ["dxi", "dyi", "jj", "kk", "istart", "jstart", "kstart", "iend", "jend", "kend"],
    },
    "advec_v": {
        "buffers": [("vt", "output"), ("u", "input"), ("v", "input"), ("w", "input"),
                    ("rhoref", "input"), ("rhorefh", "input"), ("dzi", "input")],
        "scalars": ["dxi", "dyi", "jj", "kk", "istart", "jstart", "kstart", "iend", "jend", "kend"],
    },
    "advec_w": {
        "buffers": [("wt", "output"), ("u", "input"), ("v", "input"), ("w", "input"),
                    ("rhoref", "input"), ("rhorefh", "input"), ("dzhi", "input")],
        "scalars": ["dxi", "dyi", "jj", "kk", "istart", "jstart", "kstart", "iend", "jend", "kend"],
    },
    "advec_s": {
        "buffers": [("st", "output"), ("s", "input"), ("u", "input"), ("v", "input"), ("w", "input"),
                    ("rhoref", "input"), ("rhorefh", "input"), ("dzi", "input")],
        "scalars": ["dxi", "dyi", "jj", "kk", "istart", "jstart", "kstart", "iend", "jend", "kend"],
    },
    "diff_c": {
        "buffers": [("st", "output"), ("s", "input"), ("evisc", "input"), ("dzi", "input"), ("dzhi", "input"),
                    ("rhoref", "input"), ("rhorefh", "input")],
        "scalars": ["dxi", "dyi", "tpri", "jj", "kk", "istart", "jstart", "kstart", "iend", "jend", "kend"],
    },
    "evisc_smag": {
        "buffers": [("evisc", "output"), ("u", "input"), ("v", "input"), ("w", "input"), ("dzi", "input"),
                    ("dzhi", "input")],
        "scalars": ["dxi", "dyi", "cs", "jj", "kk", "istart", "jstart", "kstart", "iend", "jend", "kend"],
    },
    "diff_uvw_rk3": {
        "buffers": [("ut", "output"), ("vt", "output"), ("wt", "output"), ("evisc", "input"), ("u", "input"),
                    ("v", "input"), ("w", "input"), ("dzi", "input"), ("dzhi", "input"), ("rhoref", "input"),
                    ("rhorefh", "input"), ("u_next", "output"), ("v_next", "output"), ("w_next", "output")],
        "scalars": ["dxi", "dyi", "rk_a", "rk_bdt", "jj", "kk", "istart", "jstart", "kstart", "iend", "jend",
                    "kend"],
    },
    "advec_u_peer": {
        "buffers": [("ut", "output"), ("u", "input"), ("v", "input"), ("w", "input"),
                    ("rhoref", "input"), ("rhorefh", "input"), ("dzi", "input"), ("u_lo", "input"),
                    ("w_lo", "input"), ("u_hi", "input"), ("w_hi", "input")],
        "scalars": ["dxi", "dyi", "peer_klo", "peer_khi", "peer_shift_lo", "peer_shift_hi", "jj", "kk", "istart",
                    "jstart", "kstart", "iend", "jend", "kend"],
    },
    "diff_uvw_peer": {
        "buffers": [("ut", "output"), ("vt", "output"), ("wt", "output"), ("evisc", "input"), ("u", "input"),
                    ("v", "input"), ("w", "input"), ("dzi", "input"), ("dzhi", "input"), ("rhoref", "input"),
                    ("rhorefh", "input"), ("evisc_lo", "input"), ("u_lo", "input"), ("v_lo", "input"),
                    ("w_lo", "input"), ("evisc_hi", "input"), ("u_hi", "input"), ("v_hi", "input"),
                    ("w_hi", "input")],
        "scalars": ["dxi", "dyi", "peer_klo", "peer_khi", "peer_shift_lo", "peer_shift_hi", "jj", "kk", "istart",
                    "jstart", "kstart", "iend", "jend", "kend"],
    },
    "diff_uvw_rk3_peer": {
        "buffers": [("ut", "output"), ("vt", "output"), ("wt", "output"), ("evisc", "input"), ("u", "input"),
                    ("v", "input"), ("w", "input"), ("dzi", "input"), ("dzhi", "input"), ("rhoref", "input"),
                    ("rhorefh", "input"), ("u_next", "output"), ("v_next", "output"), ("w_next", "output"),
                    ("evisc_lo", "input"), ("u_lo", "input"), ("v_lo", "input"), ("w_lo", "input"),
                    ("evisc_hi", "input"), ("u_hi", "input"), ("v_hi", "input"), ("w_hi", "input")],
        "scalars": ["dxi", "dyi", "rk_a", "rk_bdt", "peer_klo", "peer_khi", "peer_shift_lo", "peer_shift_hi", "jj",
                    "kk", "istart", "jstart", "kstart", "iend", "jend", "kend"],
    },
    "rk3_uvw": {
        "buffers": [("ut", "output"), ("vt", "output"), ("wt", "output"), ("u", "output"), ("v", "output"),
                    ("w", "output")],
        "scalars": ["rk_a", "rk_bdt", "jj", "kk", "istart", "jstart", "kstart", "iend", "jend", "kend"],
    },
}


def _pos(kernel: str, name: str) -> int:
    layout = ARG_LAYOUT[kernel]
    names = [b for b, _ in layout["buffers"]] + layout["scalars"]
    return names.index(name)


_INCLUDE = re.compile(r'^\s*#\s*include\s+"([^"]+)"\s*$', re.M)


def _inline(path: Path, depth: int = 0) -> str:
    """Textually inline local ``#include "x"`` (headers carry include guards, so
    every occurrence is inlined and the preprocessor picks the live ones)."""
    if depth > 8:
        raise RecursionError(f"include nesting too deep at {path.name}")
    text = path.read_text(encoding="utf-8")

    def repl(m: re.Match) -> str:
        name = m.group(1)
        return f"// ---- begin {name} ----\n{_inline(_HERE / name, depth + 1)}\n// ---- end {name} ----"

    return _INCLUDE.sub(repl, text)


def _strip_comments(text: str) -> str:
    """Remove // and /* */ comments outside string/char literals, keeping
    every newline (line numbers of the assembled source are unchanged) and
    dropping trailing blanks.  The assembled source is embedded in every
    capture's metadata, which the .klcap format caps at 64 KiB
    (reference capture.py:37); the commented sources stay in stencils/."""
    out, i, n = [], 0, len(text)
    quote = None
    while i < n:
        ch = text[i]
        if quote:
            out.append(ch)
            if ch == "\\" and i + 1 < n:
                out.append(text[i + 1])
                i += 2
                continue
            if ch == quote:
                quote = None
            i += 1
        elif ch in "\"'":
            quote = ch
            out.append(ch)
            i += 1
        elif text.startswith("//", i):
            j = text.find("\n", i)
            i = n if j < 0 else j
        elif text.startswith("/*", i):
            j = text.find("*/", i + 2)
            j = n if j < 0 else j + 2
            out.append("\n" * text.count("\n", i, j))
            i = j
        else:
            out.append(ch)
            i += 1
    return "\n".join(line.rstrip() for line in "".join(out).split("\n"))


@lru_cache(maxsize=None)
def assemble_source(kernel: str, precision: str) -> str:
    """Self-contained NVRTC source: precision/entry prelude + inlined headers
    (comments stripped, see ``_strip_comments``)."""
    if kernel not in ALL_KERNELS or precision not in PRECISIONS:
        raise ValueError(f"unknown kernel/precision {kernel}/{precision}")
    prelude = (
        f"// {kernel} ({precision}) — B200 Kernel Launcher stencil, runtime-compiled by NVRTC\n"
        f"#define KL_REAL {PRECISIONS[precision]}\n"
        f"#define KL_ENTRY {kernel}_{precision}\n"
        "#define DIRECT 0\n#define ZMARCH 1\n#define TMA 2\n"
    )
    if kernel in FUSED_KERNELS:
        prelude += "".join(f"#define {name} 1\n" for name in FUSED_KERNELS[kernel][1].split())
    return prelude + _strip_comments(_inline(_HERE / f"{base_kernel(kernel)}.cu"))


#: ZMARCH shared-memory plane budget per kernel, in halo'd cells per plane
#: (keeps fp64 staging <= ~96 KB so at least two blocks fit per SM).
_ZMARCH_PLANE_LIMIT = {
    "advec_u": "(block_x + 6) * (block_y * tile_y + 6) <= 6144",
    "diff_uvw": "(block_x + 2) * (block_y * tile_y + 2) <= 1024",
}
#: opt-in shared memory per block on B200 (cudaDevAttrMaxSharedMemoryPerBlockOptin,
#: 227 KB); the executor re-checks the live device's value before launching
SMEM_OPTIN_BYTES = 232448
#: TMA box extents are <= 256 elements; the smem ring must fit the opt-in limit
_TMA_LIMIT = {
    "diff_uvw": ['staging != "TMA" || (block_x * tile_x <= 128 && {SMEM_TMA} <= ' + str(SMEM_OPTIN_BYTES) + ")"],
    "advec_u": ['staging != "TMA" || (block_x * tile_x <= 128 && {SMEM_TMA} <= ' + str(SMEM_OPTIN_BYTES) + ")"],
}
#: knobs the ZMARCH/TMA variants of each kernel fix (pinned to their defaults)
_ZMARCH_PINNED = {
    # a contiguous y strip; one column per thread, or (TMA) tile_x consecutive columns
    "advec_u": '!unroll_x && !unroll_y && !contiguous_y && '
               '((tile_x == 1 && !contiguous_x) || (staging == "TMA" && tile_x > 1 && contiguous_x))',
    # a contiguous strip of tile_y rows (flux reuse along y); one column per
    # thread, or (TMA) tile_x consecutive columns (x-face reuse)
    "diff_uvw": '!unroll_x && !unroll_y && !contiguous_y && '
                '((tile_x == 1 && !contiguous_x) || (staging == "TMA" && tile_x > 1 && contiguous_x))',
}


@lru_cache(maxsize=None)
def stencil_space(kernel: str = "advec_u", precision: str = "fp32") -> ConfigSpace:
    """The kernel's space: Table 2 x the B200 knobs, restricted per precision
    (shared-memory limits depend on the element size, so the fp32 and fp64
    spaces — and their fingerprints — may differ)."""
    kernel = base_kernel(kernel)
    size = 4 if precision == "fp32" else 8
    if kernel in ADV_FAMILY:
        # DIRECT (Table 2) or TMA flux-form with column pairs (tile_x in {2, 4})
        params = table2_params() + [
            TunableParam("staging", ("DIRECT", "TMA"), "DIRECT"),
            TunableParam("zchunk", ZCHUNK_VALUES, 1),
            TunableParam("depth", DEPTH_VALUES, 0),
        ]
        return ConfigSpace(params, [
            BLOCK_LIMIT_RESTRICTION,
            'staging != "DIRECT" || (zchunk == 1 && depth == 0)',
            'staging != "TMA" || (zchunk > 1 && depth > 0 && block_z == 1 && tile_z == 1 && !unroll_x && '
            '!unroll_y && !unroll_z && !contiguous_y && !contiguous_z && contiguous_x && tile_x >= 2 && '
            'block_x * block_y >= 32 && block_x * tile_x <= 128 && '
            + _adv_family_smem(kernel).format(S=size) + f" <= {SMEM_OPTIN_BYTES})",
        ])
    if kernel in PLANE_FAMILY:
        # DIRECT (Table 2) or the TMA plane z-march (tile_x consecutive columns)
        params = table2_params() + [
            TunableParam("staging", ("DIRECT", "TMA"), "DIRECT"),
            TunableParam("zchunk", ZCHUNK_VALUES, 1),
            TunableParam("depth", DEPTH_VALUES, 0),
        ]
        restrictions = [
            BLOCK_LIMIT_RESTRICTION,
            'staging != "DIRECT" || (zchunk == 1 && depth == 0)',
            'staging != "TMA" || (zchunk > 1 && depth > 0 && block_z == 1 && tile_z == 1 && !unroll_x && '
            '!unroll_y && !unroll_z && !contiguous_y && !contiguous_z && '
            '((tile_x == 1 && !contiguous_x) || (tile_x > 1 && contiguous_x)) && '
            'block_x * block_y >= 32 && block_x * tile_x <= 128 && '
            + _plane_family_smem(kernel).format(S=size) + f" <= {SMEM_OPTIN_BYTES})",
        ]
        if kernel in XSHARE_KERNELS:
            params.append(TunableParam("xshare", (0, 1), 0))
            restrictions.append('xshare == 0 || (staging == "TMA" && tile_x == 1 && block_x >= 32)')
        return ConfigSpace(params, restrictions)
    if kernel in FAMILY_KERNELS:
        # DIRECT staging only: the B200 knobs are pinned, the Table-2 space is the search space
        params = table2_params() + [TunableParam("staging", ("DIRECT",), "DIRECT"),
                                    TunableParam("zchunk", (1,), 1), TunableParam("depth", (0,), 0)]
        return ConfigSpace(params, [BLOCK_LIMIT_RESTRICTION])
    params = table2_params() + [
        TunableParam("staging", STAGING_VALUES, "DIRECT"),
        TunableParam("zchunk", ZCHUNK_VALUES, 1),
        TunableParam("depth", DEPTH_VALUES, 0),
    ]
    if kernel in YSPLIT_KERNELS:
        params.append(TunableParam("ysplit", YSPLIT_VALUES, 0))
    restrictions = [
        BLOCK_LIMIT_RESTRICTION,
        'staging != "DIRECT" || zchunk == 1',
        'staging == "DIRECT" || (zchunk > 1 && block_z == 1 && tile_z == 1 && !unroll_z && !contiguous_z)',
        # TMA prefetch depth only exists for TMA staging
        '(staging == "TMA" && depth > 0) || (staging != "TMA" && depth == 0)',
        # a marching block must hold at least one warp of columns
        'staging == "DIRECT" || block_x * block_y >= 32',
        # register-resident tiles: the tile loops are always unrolled when marching
        f'staging == "DIRECT" || ({_ZMARCH_PINNED[kernel]})',
        # (diff_uvw's TMA ring is bounded by its own shared-memory restriction below)
        (f'staging != "ZMARCH" || ({_ZMARCH_PLANE_LIMIT[kernel]})' if kernel == "diff_uvw" else
         f'staging == "DIRECT" || ({_ZMARCH_PLANE_LIMIT[kernel]})'),
    ] + [r.replace("{SMEM_TMA}", _SMEM_TMA[kernel].format(S=size)) for r in _TMA_LIMIT.get(kernel, [])]
    if kernel in YSPLIT_KERNELS:
        restrictions.append('ysplit == 0 || staging == "TMA"')
    return ConfigSpace(params, restrictions)


#: per staging family, the knobs it fixes (value lists narrowed to one value)
_MARCH_PINS = {"block_z": 1, "tile_z": 1, "unroll_x": False, "unroll_y": False, "unroll_z": False,
               "contiguous_z": False}
FAMILY_PINS = {
    "DIRECT": {"staging": "DIRECT", "zchunk": 1, "depth": 0},
    "ZMARCH": dict(_MARCH_PINS, staging="ZMARCH", depth=0),
    "TMA": dict(_MARCH_PINS, staging="TMA"),
}
_FAMILY_EXTRA = {
    (kernel, fam): {"tile_x": 1, "contiguous_x": False, "contiguous_y": False}
    for kernel in ("diff_uvw", "advec_u") for fam in ("ZMARCH", "TMA")
}
# tile_x in {1, 2, 4} (consecutive columns)
_FAMILY_EXTRA["advec_u", "TMA"] = {"contiguous_y": False}
_FAMILY_EXTRA["diff_uvw", "TMA"] = {"contiguous_y": False}
for _k in ADV_FAMILY + tuple(PLANE_FAMILY):
    _FAMILY_EXTRA[_k, "TMA"] = {"contiguous_y": False}


def family_space(kernel: str, family: str, precision: str = "fp32") -> ConfigSpace:
    """The kernel's space with the family's fixed knobs narrowed to one value.

    Every point is valid in (and measured as) the full ``stencil_space`` — the
    narrowing only makes rejection sampling efficient: ZMARCH points are ~1e-4
    of the full product, so unrestricted random search would almost never
    reach them.  Tuning runs one session per family and keeps the best in the
    kernel's wisdom file (keep-best append, wisdom.py:151-178).
    """
    full = stencil_space(kernel, precision)
    pins = dict(FAMILY_PINS[family], **_FAMILY_EXTRA.get((base_kernel(kernel), family), {}))
    params = [TunableParam(p.name, (pins[p.name],), pins[p.name]) if p.name in pins else p for p in full.params]
    return ConfigSpace(params, full.restrictions)


_SMEM = {
    # ZMARCH shared-memory bytes (see *_zmarch.cuh): advec_u double-buffers one
    # 3-halo plane of u; diff_uvw keeps a 3-slot ring of 1-halo planes of 4 fields.
    "advec_u": "(2 * (block_x + 6) * (block_y * tile_y + 6)) * {S}",
    "diff_uvw": "(12 * (block_x + 2) * (block_y * tile_y + 2)) * {S}",
}


# TMA rings: 128 B alignment slack + 128 B of mbarriers + ring slots of 128-B
# aligned field-planes (diff_uvw: depth+2 slots x (4 halo'd + 3 tendency)
# fields; advec_u: depth+4 slots of u (3-halo; plane k+3 feeds the z-window)
# and depth+2 slots of v, w, ut); box width = columns + halo plus up to one
# 16-byte chunk of alignment slack, rounded to 16 B.
_BW = "(ceil_div(({X} + {H}) * {S} + 16 - {S}, 16) * 16 / {S})"
_ADVEC_BOX = "ceil_div(" + _BW + " * (block_y * tile_y + {R}) * {S}, 128) * 128"
_SMEM_TMA = {
    # plus the chunk's 5 per-plane z factors
    # halo'd box kXT + 2 kE wide (kE = 16 / S), tendency box kXT wide (rounded to 16 B)
    "diff_uvw": "(256 + (depth + 2) * (4 * ceil_div(ceil_div(block_x * tile_x * {S} + 32, 16) * 16"
                " * (block_y * tile_y + 2), 128) * 128 + 3 * ceil_div(ceil_div(block_x * tile_x * {S}, 16) * 16"
                " * (block_y * tile_y), 128) * 128) + 5 * zchunk * {S})",
    # advec_u boxes start at column i0-4: u (x halo 4+4, y halo 3+3), v (4 + 1 row), w (4), ut (0)
    # plus the chunk's z factors (2 per plane)
    # in two rings: u in depth+4 slots, v/w/ut in depth+2 slots (advec_u_tma.cuh)
    "advec_u": "(256 + (depth + 4) * " + _ADVEC_BOX.format(X="block_x * tile_x", H=8, R=6, S="{S}") +
    " + (depth + 2) * (" + " + ".join(
        _ADVEC_BOX.format(X="block_x * tile_x", H=h, R=r, S="{S}") for h, r in ((4, 1), (4, 0), (0, 0))) +
    ") + 2 * zchunk * {S})",
}


def _adv_family_smem(kernel: str) -> str:
    """Shared-memory bytes of the family TMA advection (advec_family_tma.cuh):
    128 B alignment slack + 128 B of mbarriers, the phi ring (depth+4 slots of
    the 3-halo box) and the velocity/tendency ring (depth+2 slots of boxes A
    (u, x faces), B (w), C (v), T (tendency) by staggering), the chunk's z
    factors."""
    xt, r = "block_x * tile_x", "block_y * tile_y"

    def width(cols):
        return f"ceil_div(({cols}) * {{S}} + 16 - {{S}}, 16) * 16"

    def box(cols, rows):
        return f"ceil_div({width(cols)} * ({rows}), 128) * 128"

    phi = box(f"{xt} + 8", f"{r} + 6")
    a_rows = f"{r} + 1" if kernel == "advec_v" else r
    parts = [box(f"{xt} + 1", a_rows)]
    if kernel != "advec_w":  # B: w
        parts.append(box(xt, f"{r} + 1" if kernel == "advec_v" else r))
    if kernel != "advec_v":  # C: v
        parts.append(box(xt, f"{r} + 1"))
    parts.append(box(xt, r))  # T
    return f"(256 + (depth + 4) * {phi} + (depth + 2) * ({' + '.join(parts)}) + 2 * zchunk * {{S}})"


def _plane_family_smem(kernel: str) -> str:
    """Shared-memory bytes of the TMA plane z-marches (kl_plane_tma.cuh,
    evisc_smag_tma.cuh): 128 B alignment slack + 128 B of mbarriers and
    depth+3 (depth+2) slots of the halo'd input boxes (columns i0-1 ..
    i0+XT, rows j0-1 .. j0+R) plus, for a read-modify-write output, its box."""
    nh, has_t, extra = PLANE_FAMILY[kernel]
    xt, r = "block_x * tile_x", "block_y * tile_y"
    halo = f"ceil_div(ceil_div(({xt} + 2) * {{S}} + 16 - {{S}}, 16) * 16 * ({r} + 2), 128) * 128"
    tend = f"ceil_div(ceil_div({xt} * {{S}} + 16 - {{S}}, 16) * 16 * ({r}), 128) * 128"
    slot = f"{nh} * {halo}" + (f" + {tend}" if has_t else "")
    return f"(256 + (depth + {extra}) * ({slot}))"


def _definition(kernel: str, precision: str) -> KernelDefinition:
    space = stencil_space(kernel, precision)
    bk = base_kernel(kernel)  # fused variants take their base kernel's knobs and grid
    p = lambda n: f"arg{_pos(kernel, n)}"  # noqa: E731
    size = 4 if precision == "fp32" else 8
    # z extent of one block: block_z*tile_z under DIRECT (zchunk pinned to 1),
    # zchunk under ZMARCH (block_z = tile_z = 1 pinned) -> one formula for both.
    grid_x = (
        "ceil_div(problem_x, block_x * tile_x) * ceil_div(problem_y, block_y * tile_y) * "
        "ceil_div(problem_z, block_z * tile_z * zchunk)"
    )
    if bk in XSHARE_KERNELS:
        grid_x = grid_x.replace("ceil_div(problem_x, block_x * tile_x)",
                                "ceil_div(problem_x, block_x * tile_x - xshare * (block_x / 32))")
    if bk in YSPLIT_KERNELS:
        nbxz = "(ceil_div(problem_x, block_x * tile_x) * ceil_div(problem_z, block_z * tile_z * zchunk))"
        # at least the natural count (<= block_y*tile_y rows per run), at most
        # problem_y runs (every run holds a row)
        grid_x = (f"{nbxz} * max(ceil_div(problem_y, block_y * tile_y), "
                  f"min(ysplit, 1) * min(problem_y, ({B200_SMS} * ysplit) / {nbxz}))")
    defines = [
        ("BLOCK_X", "block_x"), ("BLOCK_Y", "block_y"), ("BLOCK_Z", "block_z"),
        ("TILE_X", "tile_x"), ("TILE_Y", "tile_y"), ("TILE_Z", "tile_z"),
        ("UNROLL_X", "unroll_x"), ("UNROLL_Y", "unroll_y"), ("UNROLL_Z", "unroll_z"),
        ("CONTIG_X", "contiguous_x"), ("CONTIG_Y", "contiguous_y"), ("CONTIG_Z", "contiguous_z"),
        ("UNRAVEL", "unravel"), ("MIN_BLOCKS", "min_blocks"),
        ("STAGING", "staging"), ("ZCHUNK", "zchunk"), ("DEPTH", "depth"),
        ("KL_JJ", p("jj")), ("KL_KK", p("kk")),
    ] + ([("KL_YBAL", "ysplit")] if bk in YSPLIT_KERNELS else []) + (
        [("KL_XSHARE", "xshare")] if bk in XSHARE_KERNELS else [])
    return KernelDefinition(
        f"{kernel}_{precision}",
        space,
        source_text=assemble_source(kernel, precision),
        problem_size=(f"{p('iend')} - {p('istart')}", f"{p('jend')} - {p('jstart')}", f"{p('kend')} - {p('kstart')}"),
        block=("block_x", "block_y", "block_z"),
        grid=(grid_x, 1, 1),
        shared_mem=(f"min(depth, 1) * {_adv_family_smem(kernel).format(S=size)}" if kernel in ADV_FAMILY else
                    f"min(depth, 1) * {_plane_family_smem(kernel).format(S=size)}" if kernel in PLANE_FAMILY else
                    "0" if kernel in FAMILY_KERNELS else
                    f"min(zchunk - 1, 1) * ((1 - min(depth, 1)) * {_SMEM[base_kernel(kernel)].format(S=size)}"
                    f" + min(depth, 1) * {_SMEM_TMA[base_kernel(kernel)].format(S=size)})"),
        defines=defines,
        flags=("-std=c++17",),
    )


def definition_for(kernel: str, precision: str) -> KernelDefinition:
    return _cached_definition(kernel, precision)


@lru_cache(maxsize=None)
def _cached_definition(kernel: str, precision: str) -> KernelDefinition:
    return _definition(kernel, precision)


def advec_u_definition(precision: str = "fp32") -> KernelDefinition:
    return definition_for("advec_u", precision)


def diff_uvw_definition(precision: str = "fp32") -> KernelDefinition:
    return definition_for("diff_uvw", precision)
