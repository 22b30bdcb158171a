// Lane-banked histogram (k_lane's core: U=2 double-buffered LDG.128, PRMT + ATOMS per
// byte, 2 x 1024-thread CTAs per SM) under two CTA->address mappings: one contiguous
// range per CTA vs grid-stride batches (all CTAs inside one G x 32 KB window).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sh stride_hist.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void red_inc(uint32_t a) { asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(a)); }

template <bool STRIDE>
__global__ void __launch_bounds__(1024, 2) k(const uint4* __restrict__ in, size_t nvec, unsigned long long* out) {
  __shared__ __align__(16) uint32_t h[256 * 32];
  for (int i = threadIdx.x; i < 256 * 32; i += 1024) h[i] = 0;
  __syncthreads();
  const uint32_t tb = (uint32_t)__cvta_generic_to_shared(h) + (threadIdx.x & 31) * 4;
  auto word = [&](uint32_t w) {
#pragma unroll
    for (int q = 0; q < 4; ++q) red_inc(tb + (__byte_perm(w, 0, 0x4440 | q) << 7));
  };
  auto vec = [&](const uint4& v) { word(v.x); word(v.y); word(v.z); word(v.w); };
  constexpr size_t B = 2 * 1024;  // vectors per batch (U=2 x 1024 threads)
  const size_t nb = nvec / B;     // batches (inputs are batch multiples here)
  size_t j, step, nmine;
  if (STRIDE) { j = blockIdx.x; step = gridDim.x; nmine = (nb > j) ? (nb - j + step - 1) / step : 0; }
  else { const size_t per = nb / gridDim.x; j = per * blockIdx.x; step = 1; nmine = per; }
  const uint4* q = in + j * B + threadIdx.x;
  const size_t sv = step * B;
  uint4 A0, A1, B0, B1;
  if (nmine) { A0 = ldg_stream(q); A1 = ldg_stream(q + 1024); }
  for (size_t t = 0; t < nmine; t += 2) {
    const bool more = t + 1 < nmine;
    if (more) { B0 = ldg_stream(q + sv); B1 = ldg_stream(q + sv + 1024); }
    vec(A0); vec(A1);
    if (!more) break;
    if (t + 2 < nmine) { A0 = ldg_stream(q + 2 * sv); A1 = ldg_stream(q + 2 * sv + 1024); }
    vec(B0); vec(B1);
    q += 2 * sv;
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 256; b += 1024) {
    unsigned long long s = 0;
    for (int l = 0; l < 32; ++l) s += h[b * 32 + ((l + b) & 31)];
    atomicAdd(out + b, s);
  }
}

__global__ void fill(uint64_t* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t z = (i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    p[i] = z ^ (z >> 31);
  }
}

int main() {
  size_t maxn = (size_t)64 << 30;
  uint8_t* d;
  if (cudaMalloc(&d, maxn) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  fill<<<1184, 256>>>((uint64_t*)d, maxn / 8);
  unsigned long long* o; cudaMalloc(&o, 4096);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int G = 296;
  for (size_t gib : {1, 4, 16, 64}) {
    // a multiple of G batches so both mappings cover the same bytes
    size_t nb = (gib << 30) / (2 * 1024 * 16);
    nb = nb / G * G;
    size_t nvec = nb * 2 * 1024;
    for (int mode = 0; mode < 2; ++mode) {
      float tot = 0; int cnt = 0;
      std::vector<unsigned long long> hst(256);
      for (int r = 0; r < 6; ++r) {
        cudaMemset(o, 0, 2048);
        cudaEventRecord(a);
        for (int rep = 0; rep < 5; ++rep) {
          if (mode == 0) k<false><<<G, 1024>>>((const uint4*)d, nvec, o);
          else k<true><<<G, 1024>>>((const uint4*)d, nvec, o);
        }
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (r > 0) { tot += ms / 5; ++cnt; }
        if (r == 0) cudaMemcpy(hst.data(), o, 2048, cudaMemcpyDeviceToHost);
      }
      unsigned long long s = 0; for (auto x : hst) s += x;
      float ms = tot / cnt;
      printf("%3zu GiB %-14s %8.3f ms/launch %7.1f GB/s  total %s\n", gib, mode ? "grid-stride" : "per-CTA range",
             ms, nvec * 16.0 / (ms * 1e6), s == 5 * nvec * 16 ? "ok" : "BAD");
    }
  }
  return 0;
}
