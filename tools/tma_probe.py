"""Minimal TMA probe: copy a 3-D box into shared memory via the kl_tma.cuh helpers, write it back."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2303_12374_b200.capture import ScalarArg  # noqa: E402
from paper_2303_12374_b200.cuda import DeviceArray, DeviceBuffer, NvrtcCompiler, open_device  # noqa: E402
from paper_2303_12374_b200.kerneldef import CompileRequest, LaunchGeometry  # noqa: E402

SRC = (ROOT / "paper_2303_12374_b200/stencils/kl_tma.cuh").read_text() + r'''
extern "C" __device__ const int kl_tma_spec[1 + 5] = {1, 0, 2, 3, 16, 4};
struct __align__(64) KlTmaParams { TmaDesc map[1]; };
extern "C" __global__ void probe(const float* src, float* dst, int jj, int kk, int x, int y, int z,
                                 const __grid_constant__ KlTmaParams tma) {
  __shared__ __align__(128) float tile[4 * 16];
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) { kl::mbar_init(&bar, 1); kl::mbar_init_fence(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    kl::mbar_expect_tx(&bar, 4 * 16 * 4);
    kl::tma_load_3d(tile, &tma.map[0], &bar, x + kl::tma_xoff(src), y, z);
  }
  kl::mbar_wait(&bar, 0);
  for (int t = threadIdx.x; t < 64; t += blockDim.x) dst[t] = tile[t];
}
'''


def main():
    ctx = open_device(0)
    comp = NvrtcCompiler(ctx)
    exe = comp.compile(CompileRequest(SRC, "probe", (), ("-std=c++17",)), ctx.ident)
    exe.load()
    print("tma spec", exe.tma_spec)
    jj, jc, kc = 32, 8, 4
    kk = jj * jc
    host = np.arange(kk * kc + 64, dtype=np.float32)
    lead = 1  # make the kernel pointer 4 bytes past a 16-byte boundary, like the grid layout
    src = DeviceArray(host.nbytes + 64)
    src.upload(host, offset_bytes=0)
    out = DeviceArray(64 * 4)
    ptr = src.ptr + lead * 4
    args = [DeviceBuffer(0, "input", "f32", ptr, kk * kc), DeviceBuffer(1, "output", "f32", out.ptr, 64),
            ScalarArg(2, "i32", jj), ScalarArg(3, "i32", kk), ScalarArg(4, "i32", 3), ScalarArg(5, "i32", 2),
            ScalarArg(6, "i32", 1)]
    exe.launch(LaunchGeometry((32, 1, 1), (1, 1, 1)), args, timed=True)
    got = out.download_array(np.float32)
    view = host[lead:lead + kk * kc].reshape(kc, jc, jj)
    want = view[1, 2:6, 3:19].ravel()
    print("match", np.array_equal(got, want))
    print(got[:8], want[:8])


if __name__ == "__main__":
    main()
