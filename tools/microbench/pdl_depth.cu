// How many programmatically dependent launches can be resident at once on one stream?
// A chain of K kernels, each G CTAs of 1024 threads, launched back to back with
// programmatic stream serialization. Every CTA triggers its dependents at entry, then
// spins S us; mode 1 adds griddepcontrol.wait at the end (as a rotating k_lane call's
// output store does). Each kernel stamps its first CTA's start and its last CTA's end
// (globaltimer); the per-kernel start times show how deep the chain runs ahead.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 pdl_depth.cu -o pd && ./pd
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(1024, 2) k_chain(int idx, int spin_ns, int wait_end, unsigned long long* stamps) {
  if (threadIdx.x == 0) atomicMin(&stamps[2 * idx], now());
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const unsigned long long t0 = now();
  while (now() - t0 < (unsigned long long)spin_ns) { }
  if (wait_end) asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&stamps[2 * idx + 1], now());
}

int main(int argc, char** argv) {
  const int K = 16;
  unsigned long long* d;
  cudaMalloc(&d, 2 * K * sizeof(unsigned long long));
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const int grids[] = {4, 32, 64, 148};
  const int spins[] = {2000, 10000};
  for (int wait_end = 0; wait_end < 2; ++wait_end)
    for (int g : grids)
      for (int s : spins) {
        for (int rep = 0; rep < 2; ++rep) {
          unsigned long long init[2 * K];
          for (int k = 0; k < K; ++k) init[2 * k] = ~0ull, init[2 * k + 1] = 0;
          cudaMemcpy(d, init, sizeof(init), cudaMemcpyHostToDevice);
          cudaDeviceSynchronize();
          for (int k = 0; k < K; ++k) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(g);
            cfg.blockDim = dim3(1024);
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, k_chain, k, s, wait_end, d);
          }
          cudaStreamSynchronize(st);
          unsigned long long h[2 * K];
          cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
          if (rep == 0) continue;  // warm
          const unsigned long long t0 = h[0];
          double total = (h[2 * K - 1] - t0) / 1e3;
          // max number of kernels whose [start, end] intervals overlap any instant
          int depth = 0;
          for (int a = 0; a < K; ++a) {
            int c = 0;
            for (int b = 0; b < K; ++b)
              if (h[2 * b] <= h[2 * a] && h[2 * b + 1] > h[2 * a]) ++c;
            if (c > depth) depth = c;
          }
          printf("wait_end=%d grid=%3d spin=%5.1f us: %2d kernels in %7.2f us (%.2f us/kernel), max resident %d; starts:",
                 wait_end, g, s / 1e3, K, total, total / K, depth);
          for (int k = 0; k < 8; ++k) printf(" %.1f", (h[2 * k] - t0) / 1e3);
          printf("\n");
        }
      }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
