/* A plain-C client of libklb200.so (include/klb200.h): no Python, no torch.
 * Compiles a kernel with NVRTC for sm_100a, loads it, captures `reps`
 * launches on a stream as one CUDA graph, replays it and checks the result
 * exactly.  tests/test_c_abi_client.py builds it with gcc; without a GPU it
 * must fail cleanly at klb_init (exit code 3), with one it prints "c-abi ok".
 *
 *   gcc -std=c11 -I include tests/c_abi_client.c -L paper_2303_12374_b200 -lklb200 -o c_abi_client
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "klb200.h"

static const char* SRC =
    "extern \"C\" __global__ void axpy(float* y, const float* x, float a, int n) {\n"
    "  int i = blockIdx.x * blockDim.x + threadIdx.x;\n"
    "  if (i < n) y[i] += a * x[i];\n"
    "}\n";

#define CHECK(call)                                                           \
  do {                                                                        \
    if ((call) != 0) {                                                        \
      fprintf(stderr, "%s failed: %s\n", #call, klb_last_error());            \
      return 1;                                                               \
    }                                                                         \
  } while (0)

int main(void) {
  klb_device_info info;
  if (klb_init(0, &info) != 0) {
    printf("no device: %s\n", klb_last_error());
    return 3;
  }
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17"};
  void* image = NULL;
  size_t image_size = 0;
  char *lowered = NULL, *log = NULL;
  if (klb_compile(SRC, "axpy.cu", "axpy", opts, 2, &image, &image_size, &lowered, &log) != 0) {
    fprintf(stderr, "compile failed: %s\n", log ? log : klb_last_error());
    return 1;
  }
  klb_module mod;
  klb_function fn;
  CHECK(klb_module_load(image, &mod));
  CHECK(klb_module_function(mod, lowered, &fn));

  enum { N = 1 << 20, REPS = 8 };
  float* hx = (float*)malloc(N * sizeof(float));
  float* hy = (float*)malloc(N * sizeof(float));
  for (int i = 0; i < N; ++i) {
    hx[i] = (float)(i % 64);  /* small integers: every sum below is exact */
    hy[i] = (float)(i % 7);
  }
  uint64_t dx, dy;
  klb_stream s;
  klb_graph g;
  CHECK(klb_mem_alloc(N * sizeof(float), &dx));
  CHECK(klb_mem_alloc(N * sizeof(float), &dy));
  CHECK(klb_stream_create(&s, 0));
  CHECK(klb_memcpy_htod(dx, hx, N * sizeof(float), s));
  CHECK(klb_memcpy_htod(dy, hy, N * sizeof(float), s));

  float a = 2.0f;
  int n = N;
  void* params[] = {&dy, &dx, &a, &n};
  const unsigned grid[3] = {(N + 255) / 256, 1, 1}, block[3] = {256, 1, 1};
  CHECK(klb_stream_begin_capture(s));
  for (int r = 0; r < REPS; ++r) CHECK(klb_launch(fn, grid, block, 0, s, params));
  CHECK(klb_stream_end_capture(s, &g));
  CHECK(klb_graph_launch(g, s));
  CHECK(klb_memcpy_dtoh(hy, dy, N * sizeof(float), s));
  CHECK(klb_stream_synchronize(s));

  int bad = 0;
  for (int i = 0; i < N; ++i)
    if (hy[i] != (float)(i % 7) + REPS * a * (float)(i % 64)) ++bad;
  CHECK(klb_graph_destroy(g));
  CHECK(klb_stream_destroy(s));
  CHECK(klb_mem_free(dx));
  CHECK(klb_mem_free(dy));
  CHECK(klb_module_unload(mod));
  klb_free(image);
  klb_free(lowered);
  klb_free(log);
  free(hx);
  free(hy);
  if (bad) {
    printf("c-abi mismatch: %d of %d\n", bad, N);
    return 2;
  }
  printf("c-abi ok (%s, %d graph-replayed launches)\n", info.name, REPS);
  return 0;
}
