/*
 * abi_smoke.c — libs2.so driven from plain C (no Python, no torch): the C ABI of
 * include/s2.h is usable on its own, as a reference-side FFI would bind it.
 *
 * Checks the known-answer values of SURVEY.md Appendix B, which come from the live
 * reference (sketchgrad/core.py:27-38 mix64, sketch.py:86-128 CountSketchTable):
 *   CountSketchTable(3, 8, seed=0, dim=16), insert {1: 1.0, 5: -2.0, 9: 0.5}
 *     row 0 = [0, 3, 0, 0, 0, 0, 0, 0.5]
 *     row 1 = [-2, -0.5, 0, 0, 0, 0, -1, 0]
 *     row 2 = [0, 0, 0, -1, 0, 0, -0.5, 0]
 *     query([1, 5, 9]) = [1, -2, 0.5]
 * through s2_compress (mask = g != 0) and s2_decode (workers = 1), plus the error path.
 *
 *   gcc -std=c99 -Iinclude -I/usr/local/cuda/include tests/c/abi_smoke.c \
 *       -Lpaper_2110_02140_b200 -ls2 -L/usr/local/cuda/lib64 -lcudart -o abi_smoke
 *
 * Exit 0 and "abi_smoke ok" on success; with --no-gpu only the host entry points run.
 */
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include "s2.h"

static int fails = 0;
#define CHECK(cond, ...)                 \
  do {                                   \
    if (!(cond)) {                       \
      fprintf(stderr, "FAIL: " __VA_ARGS__); \
      fprintf(stderr, "\n");             \
      ++fails;                           \
    }                                    \
  } while (0)

static int host_checks(void) {
  CHECK(s2_mix64(0) == 0ull, "mix64(0)");
  CHECK(s2_mix64(1) == 0x5692161d100b05e5ull, "mix64(1)");
  const uint64_t parts[2] = {0, 0};
  CHECK(s2_derive_seed(parts, 2) == 0xa8871e3718ca0053ull, "derive_seed(0, 0)");
  s2_plan* bad = NULL;
  const int rc = s2_plan_create(16, 16, 0, 8, 0, 0, &bad);
  CHECK(rc == S2_EINVAL, "rows = 0 must be S2_EINVAL, got %d", rc);
  CHECK(s2_last_error() != NULL && strlen(s2_last_error()) > 0, "s2_last_error after a failure");
  return fails;
}

static int gpu_checks(void) {
  const int64_t dim = 16;
  const int rows = 3, cols = 8;
  float g[16] = {0};
  g[1] = 1.0f;
  g[5] = -2.0f;
  g[9] = 0.5f;
  const float want[3][8] = {{0, 3, 0, 0, 0, 0, 0, 0.5f}, {-2, -0.5f, 0, 0, 0, 0, -1, 0}, {0, 0, 0, -1, 0, 0, -0.5f, 0}};

  s2_plan* plan = NULL;
  CHECK(s2_plan_create(dim, dim, rows, cols, 0, 0, &plan) == S2_OK, "plan: %s", s2_last_error());
  if (!plan) return fails;
  const int64_t words = s2_plan_bitmap_words(plan);
  CHECK(words == 1, "bitmap words %lld", (long long)words);

  float *dg = NULL, *dtable = NULL, *dout = NULL;
  uint32_t* dbitmap = NULL;
  uint64_t* dcnt = NULL;
  cudaMalloc((void**)&dg, sizeof g);
  cudaMalloc((void**)&dtable, sizeof(float) * rows * cols);
  cudaMalloc((void**)&dout, sizeof g);
  cudaMalloc((void**)&dbitmap, sizeof(uint32_t) * 4);
  cudaMalloc((void**)&dcnt, sizeof(uint64_t) * S2_NUM_COUNTERS);
  cudaMemcpy(dg, g, sizeof g, cudaMemcpyHostToDevice);

  CHECK(s2_compress(plan, dg, dbitmap, dtable, S2_MASK_NONZERO, dcnt, NULL) == S2_OK, "compress: %s", s2_last_error());
  CHECK(s2_decode(plan, dbitmap, dtable, 1, dout, NULL) == S2_OK, "decode: %s", s2_last_error());
  CHECK(cudaDeviceSynchronize() == cudaSuccess, "sync");

  float table[3][8], out[16];
  uint32_t word = 0;
  uint64_t cnt[S2_NUM_COUNTERS];
  cudaMemcpy(table, dtable, sizeof table, cudaMemcpyDeviceToHost);
  cudaMemcpy(out, dout, sizeof out, cudaMemcpyDeviceToHost);
  cudaMemcpy(&word, dbitmap, sizeof word, cudaMemcpyDeviceToHost);
  cudaMemcpy(cnt, dcnt, sizeof cnt, cudaMemcpyDeviceToHost);

  CHECK(word == ((1u << 1) | (1u << 5) | (1u << 9)), "bitmap word %#x", word);
  CHECK(cnt[S2_CNT_NNZ] == 3, "nnz counter %llu", (unsigned long long)cnt[S2_CNT_NNZ]);
  CHECK(cnt[S2_CNT_NONFINITE] == 0, "non-finite flag");
  for (int j = 0; j < rows; ++j)
    for (int c = 0; c < cols; ++c) CHECK(table[j][c] == want[j][c], "table[%d][%d] = %g, want %g", j, c, table[j][c], want[j][c]);
  for (int i = 0; i < 16; ++i) CHECK(out[i] == g[i], "out[%d] = %g, want %g", i, out[i], g[i]);

  /* NaN is reported through the counters, not by a crash (core.py:157-158) */
  g[3] = 0.0f / 0.0f;
  cudaMemcpy(dg, g, sizeof g, cudaMemcpyHostToDevice);
  CHECK(s2_compress(plan, dg, dbitmap, dtable, S2_MASK_NONZERO, dcnt, NULL) == S2_OK, "compress(NaN)");
  cudaMemcpy(cnt, dcnt, sizeof cnt, cudaMemcpyDeviceToHost);
  CHECK(cnt[S2_CNT_NONFINITE] != 0, "NaN must raise the non-finite flag");

  cudaFree(dg);
  cudaFree(dtable);
  cudaFree(dout);
  cudaFree(dbitmap);
  cudaFree(dcnt);
  s2_plan_destroy(plan);
  return fails;
}

int main(int argc, char** argv) {
  host_checks();
  if (!(argc > 1 && strcmp(argv[1], "--no-gpu") == 0)) gpu_checks();
  if (fails) {
    fprintf(stderr, "abi_smoke: %d failure(s)\n", fails);
    return 1;
  }
  printf("abi_smoke ok\n");
  return 0;
}
