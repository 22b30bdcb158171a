// Which threads of a CTA must execute griddepcontrol.launch_dependents before a
// programmatically dependent launch may start? Kernel A (PDL primary) triggers with one
// of several patterns, then spins for ~50 us; kernel B (launched with programmatic
// stream serialization) stamps its start. B's start relative to A's start tells when
// A counted as triggered.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 pdl_trigger.cu -o pt && ./pt
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void k_a(int mode, unsigned long long* stamps) {
  if (threadIdx.x == 0 && blockIdx.x == 0) stamps[0] = now();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  bool trig = false;
  switch (mode) {
    case 0: trig = false; break;                                   // never (implicit at exit)
    case 1: trig = threadIdx.x == 0; break;                        // thread 0 only
    case 2: trig = lane == 0; break;                               // lane 0 of every warp
    case 3: trig = true; break;                                    // every thread
    case 4: trig = warp == 0; break;                               // all threads of warp 0
    case 5: trig = threadIdx.x != 0; break;                        // all but thread 0
  }
  if (trig) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const unsigned long long t0 = now();
  while (now() - t0 < 50000) { }
  if (threadIdx.x == 0 && blockIdx.x == 0) stamps[1] = now();
}

__global__ void k_b(unsigned long long* stamps) {
  if (threadIdx.x == 0 && blockIdx.x == 0) stamps[2] = now();
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  cudaStream_t s;
  cudaStreamCreate(&s);
  const char* names[] = {"none (exit)", "thread 0 only", "lane 0 of each warp", "all threads",
                         "warp 0 only", "all but thread 0"};
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode < 6; ++mode) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at0[1];
      at0[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at0[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.gridDim = dim3(getenv("PT_GRID") ? atoi(getenv("PT_GRID")) : 148);
      cfg.blockDim = dim3(1024);
      cfg.stream = s;
      cfg.attrs = at0;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, k_a, mode, d);  // the primary itself PDL-launched, as k_lane is
      cfg.gridDim = dim3(1);
      cfg.blockDim = dim3(32);
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, k_b, d);
      unsigned long long h[3];
      cudaMemcpyAsync(h, d, 24, cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      printf("%-22s B starts %7.2f us after A's start (A runs %6.2f us)\n", names[mode], (h[2] - h[0]) / 1e3,
             (h[1] - h[0]) / 1e3);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
