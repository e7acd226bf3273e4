"""Size-matched floors for a small stencil launch (config 2: advec_u fp32 256^3).

Timed exactly like the bench suite (klb_time_launches: memset flush of 2x L2,
then event / launch / event per rep, median):
  * ``empty``      — an empty kernel with the record's grid / block / shared
                     memory: the event + launch + block-dispatch overhead;
  * ``stream4r1w`` — ut += u + v + w over the interior cells (float4, rows
                     of the same padded fields): the record's algorithmic
                     bytes (4 reads + 1 write per cell) with no halo, one-shot
                     grid and grid-stride variants;
  * the wisdom-selected record itself (WisdomKernel.bind, same method);
  * a D2D copy of the same byte count (events around cuMemcpyDtoDAsync).
GPU only.
"""

from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

SRC = r'''
extern "C" __global__ void empty_k(int dummy) {
  extern __shared__ unsigned char smem[];
  if (dummy == 12345) smem[threadIdx.x] = 0;
}
extern "C" __global__ void flush_k(unsigned* buf, unsigned long long n, unsigned seed) {
  extern __shared__ unsigned char smem[];
  if (seed == 0xFFFFFFFFu) smem[threadIdx.x] = 0;
  for (unsigned long long t = blockIdx.x * 256ull + threadIdx.x; t < n / 16; t += gridDim.x * 256ull)
    reinterpret_cast<uint4*>(buf)[t] = make_uint4(seed, seed + 1, seed + 2, t);
}
// the stencil's traversal without its ring: a block of 64 threads owns a
// 64 x 8 column tile (thread tile 4 x 2) and marches ZC planes, each thread
// reading its cells of u, v, w, ut with float4 loads and writing ut
extern "C" __global__ void __launch_bounds__(64) march4(float* __restrict__ ut, const float* __restrict__ u,
    const float* __restrict__ v, const float* __restrict__ w, int jj, int kk, int istart, int jstart, int kstart,
    int itot, int jtot, int ktot, int zc) {
  const int nbx = itot / 64, nby = jtot / 8;
  const int b = blockIdx.x, bx = b % nbx, by = (b / nbx) % nby, bz = b / (nbx * nby);
  const int i = istart + bx * 64 + (threadIdx.x % 16) * 4, j = jstart + by * 8 + (threadIdx.x / 16) * 2;
  const int k0 = kstart + bz * zc;
#pragma unroll 2
  for (int k = k0; k < k0 + zc; ++k) {
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const long long o = i + static_cast<long long>(j + t) * jj + static_cast<long long>(k) * kk;
      const float4 a = __ldcs(reinterpret_cast<const float4*>(u + o));
      const float4 bb = __ldcs(reinterpret_cast<const float4*>(v + o));
      const float4 c = __ldcs(reinterpret_cast<const float4*>(w + o));
      float4 d = *reinterpret_cast<const float4*>(ut + o);
      d.x += a.x + bb.x + c.x; d.y += a.y + bb.y + c.y; d.z += a.z + bb.z + c.z; d.w += a.w + bb.w + c.w;
      __stcs(reinterpret_cast<float4*>(ut + o), d);
    }
  }
}
extern "C" __global__ void __launch_bounds__(256) stream4(float* __restrict__ ut, const float* __restrict__ u,
    const float* __restrict__ v, const float* __restrict__ w, int jj, int kk, int istart, int jstart, int kstart,
    int itot, int jtot, int ktot) {
  const int q = itot / 4;
  const long long n = static_cast<long long>(q) * jtot * ktot;
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i4 = static_cast<int>(t % q);
    const long long r = t / q;
    const int j = static_cast<int>(r % jtot), k = static_cast<int>(r / jtot);
    const long long o = istart + 4 * i4 + static_cast<long long>(jstart + j) * jj + static_cast<long long>(kstart + k) * kk;
    const float4 a = __ldcs(reinterpret_cast<const float4*>(u + o));
    const float4 b = __ldcs(reinterpret_cast<const float4*>(v + o));
    const float4 c = __ldcs(reinterpret_cast<const float4*>(w + o));
    float4 d = *reinterpret_cast<const float4*>(ut + o);
    d.x += a.x + b.x + c.x; d.y += a.y + b.y + c.y; d.z += a.z + b.z + c.z; d.w += a.w + b.w + c.w;
    __stcs(reinterpret_cast<float4*>(ut + o), d);
  }
}
'''


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", default="256,256,256")
    ap.add_argument("--kernel", default="advec_u")
    ap.add_argument("--reps", type=int, default=15)
    a = ap.parse_args(argv)

    from paper_2303_12374_b200.capture import CapturePolicy, ScalarArg
    from paper_2303_12374_b200.cuda import DeviceArray, DeviceBuffer, Event, NvrtcCompiler, open_device
    from paper_2303_12374_b200.cuda._abi import check, lib
    from paper_2303_12374_b200.dispatch import WisdomKernel
    from paper_2303_12374_b200.kerneldef import CompileRequest, LaunchGeometry
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import StencilProblem

    ctx = open_device(0)
    grid = tuple(int(x) for x in a.grid.split(","))
    lay = GridLayout(*grid, "fp32")
    prob = StencilProblem(a.kernel, lay, ctx)
    comp = NvrtcCompiler(ctx)
    flush = ctx.flush_buffer()
    alg = prob.algorithmic_bytes
    res = {"grid": list(grid), "algorithmic_bytes": alg}

    def row(secs):
        t = statistics.median(secs)
        return {"us": round(t * 1e6, 2), "alg_gbs": round(alg / t / 1e9, 1)}

    wk = WisdomKernel(prob.definition, comp, wisdom_dir=ROOT / "wisdom", capture_policy=CapturePolicy())
    handle, config, kind = wk.resolve(ctx.ident, prob.definition.derive_problem_size(prob.scalar_env()),
                                      prob.scalar_env())
    entry = next(iter(wk._cache.values()))
    geom = wk._geometry(entry, prob.definition.derive_problem_size(prob.scalar_env()), prob.scalar_env())
    res["record"] = dict(row(handle.time_launches(geom, prob.args(), 3, a.reps, flush=flush)),
                         config=config, match_kind=kind, grid_blocks=list(geom.grid), block=list(geom.block),
                         smem=geom.shared_mem_bytes)

    empty = comp.compile(CompileRequest(SRC, "empty_k", (), ("-std=c++17",)), ctx.ident)
    empty.load()
    eg = LaunchGeometry(geom.block, geom.grid, geom.shared_mem_bytes)
    res["empty_same_geometry"] = row(empty.time_launches(eg, [ScalarArg(0, "i32", 0)], 3, a.reps, flush=flush))

    st = comp.compile(CompileRequest(SRC, "stream4", (), ("-std=c++17",)), ctx.ident)
    st.load()
    ut, u, v, w = (prob.field_ptr(n) for n in ("ut", "u", "v", "w"))
    n = lay.alloc_bytes // 4
    sargs = [DeviceBuffer(0, "output", "f32", ut, n), DeviceBuffer(1, "input", "f32", u, n),
             DeviceBuffer(2, "input", "f32", v, n), DeviceBuffer(3, "input", "f32", w, n)]
    for pos, val in enumerate((lay.jj, lay.kk, lay.igc, lay.jgc, lay.kgc, grid[0], grid[1], grid[2]), start=4):
        sargs.append(ScalarArg(pos, "i32", val))
    items = grid[0] // 4 * grid[1] * grid[2]
    for label, blocks in (("oneshot", (items + 255) // 256), ("gridstride_148x8", 148 * 8),
                          ("gridstride_148x4", 148 * 4), ("gridstride_148x16", 148 * 16)):
        g = LaunchGeometry((256, 1, 1), (blocks, 1, 1), 0)
        res[f"stream4r1w_{label}"] = row(st.time_launches(g, sargs, 3, a.reps, flush=flush))

    mk = comp.compile(CompileRequest(SRC, "march4", (), ("-std=c++17",)), ctx.ident)
    mk.load()
    for zc in (256, 64, 32, 16, 8, 4):
        margs = sargs + [ScalarArg(12, "i32", zc)]
        nblk = (grid[0] // 64) * (grid[1] // 8) * (grid[2] // zc)
        res[f"march4_64x8_zchunk{zc}_{nblk}blocks"] = row(
            mk.time_launches(LaunchGeometry((64, 1, 1), (nblk, 1, 1), 0), margs, 3, a.reps, flush=flush))

    # shared-memory carveout: the empty kernel with no dynamic shared memory,
    # and the empty kernel / the record after a flush done by a kernel that
    # itself requests the record's shared memory (no carveout switch at the
    # timed launch, as inside a time loop of TMA stencils)
    s = ctx.stream
    eg0 = LaunchGeometry(geom.block, geom.grid, 0)
    res["empty_no_smem"] = row(empty.time_launches(eg0, [ScalarArg(0, "i32", 0)], 3, a.reps, flush=flush))
    fk = comp.compile(CompileRequest(SRC, "flush_k", (), ("-std=c++17",)), ctx.ident)
    fk.load()
    fgeom = LaunchGeometry((256, 1, 1), (148 * 4, 1, 1), geom.shared_mem_bytes)
    fargs = [DeviceBuffer(0, "output", "u32", flush.ptr, flush.nbytes // 4), ScalarArg(1, "u64", flush.nbytes),
             ScalarArg(2, "u32", 0)]
    run_flush = fk.bound(fgeom, fargs, stream=s)
    run_rec = handle.bound(geom, prob.args(), stream=s)
    run_empty = empty.bound(eg, [ScalarArg(0, "i32", 0)], stream=s)

    def after_kernel_flush(run):
        ts = []
        for i in range(a.reps + 3):
            run_flush()
            e0, e1 = Event(), Event()
            e0.record(s)
            run()
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_ms(e1) * 1e-3)
        return ts[3:]

    res["empty_after_smem_flush_kernel"] = row(after_kernel_flush(run_empty))
    res["record_after_smem_flush_kernel"] = row(after_kernel_flush(run_rec))
    res["record_again_after_memset"] = row(handle.time_launches(geom, prob.args(), 3, a.reps, flush=flush))

    src, dst = DeviceArray(alg // 2), DeviceArray(alg // 2)
    ts = []
    for i in range(a.reps + 3):
        check(lib().klb_memset_d8(flush.ptr, i & 0xFF, flush.nbytes, s.handle))
        e0, e1 = Event(), Event()
        e0.record(s)
        check(lib().klb_memcpy_dtod(dst.ptr, src.ptr, alg // 2, s.handle))
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_ms(e1) * 1e-3)
    res["d2d_copy_same_bytes"] = row(ts[3:])
    print(json.dumps(res))
    prob.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
