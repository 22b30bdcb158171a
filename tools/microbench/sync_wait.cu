// How should the blocking entries wait? Latency of one 1 MiB histogram call (the C1
// per-image path) through libhist256.so, counts written by the kernel into page-locked
// host memory, waited for by:
//   sync   hs_histogram_sync (launch + cudaStreamSynchronize)
//   query  hs_histogram_batched + spin on cudaStreamQuery
//   event  hs_histogram_batched + cudaEventRecord + spin on cudaEventQuery
//   flag   hs_histogram_batched + a 1-thread kernel that stores a sequence word into mapped
//          host memory after it (stream order), host spins on the word
// plus the floors: an empty kernel + cudaStreamSynchronize, and the async launch alone.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o sw sync_wait.cu -I../../include
//        -L../../paper_1011_0235_b200/_lib -lhist256 -Xlinker -rpath=$PWD/../../paper_1011_0235_b200/_lib
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#include "hist256.h"

__global__ void k_empty() {}
__global__ void k_flag(volatile uint32_t* f, uint32_t v) { *f = v; }

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  const size_t n = 1 << 20;
  uint8_t* d;
  cudaMalloc(&d, n);
  cudaMemset(d, 7, n);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const size_t wsn = hs_workspace_bytes(1);
  void* ws;
  cudaMalloc(&ws, wsn);
  cudaMemset(ws, 0, wsn);
  uint64_t *h_out, *d_out;
  cudaHostAlloc(&h_out, 256 * 8, cudaHostAllocMapped);
  cudaMalloc(&d_out, 256 * 8);
  uint64_t* m_out;
  cudaHostGetDevicePointer(&m_out, h_out, 0);
  uint32_t* h_flag;
  cudaHostAlloc(&h_flag, 64, cudaHostAllocMapped);
  uint32_t* m_flag;
  cudaHostGetDevicePointer(&m_flag, h_flag, 0);
  *h_flag = 0;
  cudaEvent_t ev;
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  cudaDeviceSynchronize();
  const uint64_t b = 0, e = n;
  const int reps = 3000;
  uint32_t seq = 0;
  for (int mode = 0; mode < 6; ++mode) {
    for (int round = 0; round < 2; ++round) {
      std::vector<double> t(reps);
      for (int r = 0; r < reps; ++r) {
        const double t0 = now_us();
        int rc = 0;
        if (mode == 0) {
          rc = hs_histogram_sync(d, &b, &e, 1, HS_KIND_NAIVE, HS_IMPL_AUTO, nullptr, nullptr, 0, 0, d_out, h_out, ws,
                                 wsn, st);
        } else if (mode <= 3) {
          rc = hs_histogram_batched(d, &b, &e, 1, HS_KIND_NAIVE, HS_IMPL_AUTO, nullptr, nullptr, 0, 0, m_out, ws, wsn,
                                    st);
          if (mode == 1) {
            while (cudaStreamQuery(st) == cudaErrorNotReady) {}
          } else if (mode == 2) {
            cudaEventRecord(ev, st);
            while (cudaEventQuery(ev) == cudaErrorNotReady) {}
          } else {
            ++seq;
            k_flag<<<1, 1, 0, st>>>(m_flag, seq);
            while (*(volatile uint32_t*)h_flag != seq) {}
          }
        } else if (mode == 4) {
          k_empty<<<1, 32, 0, st>>>();
          cudaStreamSynchronize(st);
        } else {
          rc = hs_histogram_batched(d, &b, &e, 1, HS_KIND_NAIVE, HS_IMPL_AUTO, nullptr, nullptr, 0, 0, m_out, ws, wsn,
                                    st);
          t[r] = now_us() - t0;
          cudaStreamSynchronize(st);
          continue;
        }
        t[r] = now_us() - t0;
        if (rc) { printf("rc %d\n", rc); return 1; }
      }
      cudaStreamSynchronize(st);
      if (h_out[7] != n) { printf("bad count %llu\n", (unsigned long long)h_out[7]); return 1; }
      std::sort(t.begin(), t.end());
      static const char* names[] = {"sync (hs_histogram_sync)", "batched + cudaStreamQuery spin",
                                    "batched + event query spin", "batched + flag kernel + host spin",
                                    "empty kernel + stream sync", "batched launch only (async)"};
      if (round) printf("%-36s median %6.2f us  p10 %6.2f  p90 %6.2f\n", names[mode], t[reps / 2], t[reps / 10],
                        t[reps * 9 / 10]);
    }
  }
  return 0;
}
