/*
 * c_api_demo.c -- libhist256 from plain C, no Python and no torch: the C ABI of
 * include/hist256.h as a non-Python host (or a cgo / JNI / FFI binding) would use it.
 *
 *   1. a 64 MiB + 12 B host stream, cut into three word-aligned segments;
 *   2. hs_histogram_batched on a device copy (NAIVE), with a workspace;
 *   3. hs_binning_pattern + hs_degeneracy on the host counts, then ADAPTIVE;
 *   4. hs_histogram_host straight from the pageable host buffer (blocking).
 * Every result is compared with a host count. Prints "c_api_demo ok" and exits 0.
 *
 * build (examples/Makefile):
 *   gcc -O2 -std=c11 -I include -I /usr/local/cuda/include examples/c_api_demo.c \
 *       -L paper_1011_0235_b200/_lib -lhist256 -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,'$ORIGIN/../paper_1011_0235_b200/_lib' -o examples/c_api_demo
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "hist256.h"

#define NSEG 3

static int check(int rc, const char* where) {
  if (rc != HS_OK) {
    fprintf(stderr, "%s: %s (%d)\n", where, hs_strerror(rc), rc);
    exit(1);
  }
  return rc;
}

static void cuda_check(cudaError_t e, const char* where) {
  if (e != cudaSuccess) {
    fprintf(stderr, "%s: %s\n", where, cudaGetErrorString(e));
    exit(1);
  }
}

static int same(const uint64_t* a, const uint64_t* b, size_t n) { return memcmp(a, b, n * sizeof(uint64_t)) == 0; }

int main(void) {
  const size_t n = (64u << 20) + 12;
  uint8_t* h = (uint8_t*)malloc(n);
  uint64_t x = 0x1011023512345678ull;
  for (size_t i = 0; i < n; ++i) {  /* xorshift bytes, skewed towards 128 */
    x ^= x << 13;
    x ^= x >> 7;
    x ^= x << 17;
    h[i] = (uint8_t)(((x & 0xff) + ((x >> 8) & 0xff)) >> 1);
  }
  const uint64_t begin[NSEG] = {0, 4, 1u << 20};
  const uint64_t end[NSEG] = {4, 1u << 20, n};
  static uint64_t want[NSEG][HS_BINS], got[NSEG][HS_BINS], total[HS_BINS];
  for (int s = 0; s < NSEG; ++s)
    for (uint64_t i = begin[s]; i < end[s]; ++i) ++want[s][h[i]];
  for (int b = 0; b < HS_BINS; ++b) total[b] = want[0][b] + want[1][b] + want[2][b];

  uint8_t* d = NULL;
  uint64_t* d_out = NULL;
  void* d_ws = NULL;
  uint8_t* d_stage = NULL;
  const size_t ws = hs_workspace_bytes(NSEG);
  cuda_check(cudaMalloc((void**)&d, n), "cudaMalloc data");
  cuda_check(cudaMalloc((void**)&d_out, sizeof(got)), "cudaMalloc out");
  cuda_check(cudaMalloc(&d_ws, ws), "cudaMalloc workspace");
  cuda_check(cudaMemset(d_ws, 0, ws), "zero workspace");  /* once; calls leave its slots zero */
  cuda_check(cudaMemcpy(d, h, n, cudaMemcpyHostToDevice), "H2D");

  /* 2. NAIVE over three segments: one launch, counts written by the last CTA of each */
  check(hs_histogram_batched(d, begin, end, NSEG, HS_KIND_NAIVE, HS_IMPL_AUTO, NULL, NULL, 0, 0, d_out, d_ws, ws,
                             NULL),
        "hs_histogram_batched NAIVE");
  cuda_check(cudaMemcpy(got, d_out, sizeof(got), cudaMemcpyDeviceToHost), "D2H");
  if (!same(&got[0][0], &want[0][0], NSEG * HS_BINS)) return fprintf(stderr, "NAIVE mismatch\n"), 1;

  /* 3. the reference's control plane on the host, then ADAPTIVE with that pattern */
  int64_t offset[HS_BINS], count[HS_BINS];
  double share = 0.0;
  int argmax = -1;
  uint64_t pixels = 0;
  check(hs_binning_pattern(total, 960, 8, offset, count), "hs_binning_pattern");
  check(hs_degeneracy(total, &share, &argmax, &pixels), "hs_degeneracy");
  memset(got, 0, sizeof(got));
  check(hs_histogram_batched(d, begin, end, NSEG, HS_KIND_ADAPTIVE | (share < 0.999 ? HS_KIND_FLAG_SPREAD : 0),
                             HS_IMPL_AUTO, offset, count, 960, 8, d_out, d_ws, ws, NULL),
        "hs_histogram_batched ADAPTIVE");
  cuda_check(cudaMemcpy(got, d_out, sizeof(got), cudaMemcpyDeviceToHost), "D2H");
  if (!same(&got[0][0], &want[0][0], NSEG * HS_BINS)) return fprintf(stderr, "ADAPTIVE mismatch\n"), 1;

  /* 4. blocking call straight from host memory: copy in, launch, counts out, wait */
  const uint8_t* chunks[NSEG] = {h + begin[0], h + begin[1], h + begin[2]};
  uint64_t sizes[NSEG];
  size_t stage_bytes = 0;
  for (int s = 0; s < NSEG; ++s) {
    sizes[s] = end[s] - begin[s];
    stage_bytes += (sizes[s] + 15) & ~(size_t)15;
  }
  cuda_check(cudaMalloc((void**)&d_stage, stage_bytes), "cudaMalloc stage");
  memset(got, 0, sizeof(got));
  check(hs_histogram_host(chunks, sizes, NSEG, HS_KIND_NAIVE, HS_IMPL_AUTO, NULL, NULL, 0, 0, d_stage, stage_bytes,
                          d_out, &got[0][0], d_ws, ws, NULL),
        "hs_histogram_host");
  if (!same(&got[0][0], &want[0][0], NSEG * HS_BINS)) return fprintf(stderr, "host-entry mismatch\n"), 1;

  printf("c_api_demo ok: %llu pixels, max-bin share %.4f at bin %d\n", (unsigned long long)pixels, share, argmax);
  cudaFree(d);
  cudaFree(d_out);
  cudaFree(d_ws);
  cudaFree(d_stage);
  free(h);
  return 0;
}
