// Sustained power: 5 s each of (a) a streaming read kernel (LDG.128 + xor, the copy
// roofline's read side) and (b) the lane-banked shared-atomic histogram, back to back
// on 1 GiB. Run with nvidia-smi sampling power and SM clock alongside.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pm power_mix.cu
#include <cstdio>
#include <cstdint>
#include <chrono>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

__global__ void __launch_bounds__(1024, 2) k_read(const uint4* in, size_t nvec, unsigned* out) {
  uint32_t x = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nvec; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = ldg_stream(in + i);
    x ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (x == 0x12345678u) out[0] = x;
}

__global__ void __launch_bounds__(1024, 2) k_hist(const uint4* in, size_t nvec, unsigned long long* out) {
  __shared__ uint32_t h[256 * 32];
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const uint32_t tb = (uint32_t)__cvta_generic_to_shared(h) + (threadIdx.x & 31) * 4;
  auto w = [&](uint32_t x) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(tb + (__byte_perm(x, 0, 0x4440 | q) << 7)));
  };
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nvec; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = ldg_stream(in + i);
    w(v.x); w(v.y); w(v.z); w(v.w);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 256; b += blockDim.x) {
    unsigned long long s = 0;
    for (int l = 0; l < 32; ++l) s += h[b * 32 + ((l + b) & 31)];
    atomicAdd(out + b, s);
  }
}

__global__ void fill_random(uint64_t* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t z = (i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    p[i] = z ^ (z >> 31);
  }
}

int main(int argc, char** argv) {
  const double secs = argc > 1 ? atof(argv[1]) : 5.0;
  size_t n = (size_t)1 << 30;
  uint8_t* d; cudaMalloc(&d, n);
  if (argc > 2 && argv[2][0] == 'r') fill_random<<<1184, 256>>>((uint64_t*)d, n / 8);
  else cudaMemset(d, 0x5a, n);
  cudaDeviceSynchronize();
  unsigned long long* out; cudaMalloc(&out, 4096);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int which = 0; which < 2; ++which) {
    auto t0 = std::chrono::steady_clock::now();
    int it = 0;
    while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < secs) {
      cudaEventRecord(a);
      for (int r = 0; r < 20; ++r) {
        if (which == 0) k_read<<<sms * 2, 1024>>>((const uint4*)d, n / 16, (unsigned*)out);
        else k_hist<<<sms * 2, 1024>>>((const uint4*)d, n / 16, out);
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double t = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (it++ % 10 == 0) printf("%s t=%.2fs %.1f us/launch %.1f GB/s\n", which ? "hist" : "read", t, ms / 20 * 1e3, n / (ms / 20 * 1e6));
      fflush(stdout);
    }
    cudaDeviceSynchronize();
    if (which == 0) {  // cool down between phases
      auto t1 = std::chrono::steady_clock::now();
      while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count() < 3.0) {}
    }
  }
  return 0;
}
