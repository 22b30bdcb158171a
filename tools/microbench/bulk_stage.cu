// Does staging the input through shared memory with the bulk-copy engine (TMA-class
// cp.async.bulk + mbarrier) beat k_lane's register double buffer? Same lane-banked
// counting (PRMT + ATOMS per byte, 2 x 1024-thread CTAs per SM); the staged variant
// adds one LDS.128 per 16 bytes and a barrier per stage.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bs bulk_stage.cu
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
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
  return r;
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile("{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
               " @!p bra WAIT_%=;\n}" ::"r"(bar), "r"(parity) : "memory");
}

template <int S>
__global__ void __launch_bounds__(1024, 2) k_bulk(const uint8_t* __restrict__ in, size_t nbytes, unsigned long long* out) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint32_t* h = reinterpret_cast<uint32_t*>(smem);                 // 32 KB counters
  const uint32_t hbase = (uint32_t)__cvta_generic_to_shared(h);
  const uint32_t sbase = hbase + 32768;                               // S stages of 16 KB
  __shared__ __align__(8) uint64_t bars[S];
  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(bars);
  for (int i = threadIdx.x; i < 256 * 32; i += 1024) h[i] = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(bar0 + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t tb = hbase + (threadIdx.x & 31) * 4;
  constexpr uint32_t kStage = 16384;
  const size_t per = nbytes / gridDim.x;  // multiple of kStage here
  const uint8_t* base = in + per * blockIdx.x;
  const uint32_t nst = uint32_t(per / kStage);
  if (threadIdx.x == 0)
    for (uint32_t s = 0; s < S && s < nst; ++s) {
      mbar_expect_tx(bar0 + 8 * s, kStage);
      bulk_g2s(sbase + s * kStage, base + size_t(s) * kStage, kStage, bar0 + 8 * s);
    }
  for (uint32_t k = 0; k < nst; ++k) {
    const uint32_t s = k % S;
    mbar_wait(bar0 + 8 * s, (k / S) & 1);
    const uint4 v = lds128(sbase + s * kStage + threadIdx.x * 16);
    __syncthreads();  // everyone has read stage s: refill it
    if (threadIdx.x == 0 && k + S < nst) {
      mbar_expect_tx(bar0 + 8 * s, kStage);
      bulk_g2s(sbase + s * kStage, base + size_t(k + S) * kStage, kStage, bar0 + 8 * s);
    }
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) red_inc(tb + (__byte_perm(w[j], 0, 0x4440 | q) << 7));
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 256; b += 1024) {
    unsigned long long t = 0;
    for (int l = 0; l < 32; ++l) t += h[b * 32 + ((l + b) & 31)];
    atomicAdd(out + b, t);
  }
}

__global__ void __launch_bounds__(1024, 2) k_reg(const uint8_t* __restrict__ in, size_t nbytes, unsigned long long* out) {
  __shared__ __align__(16) uint32_t h[256 * 32];
  for (int i = threadIdx.x; i < 256 * 32; i += 1024) h[i] = 0;
  __syncthreads();
  const uint32_t tb = (uint32_t)__cvta_generic_to_shared(h) + (threadIdx.x & 31) * 4;
  auto vec = [&](const uint4& v) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) red_inc(tb + (__byte_perm(w[j], 0, 0x4440 | q) << 7));
  };
  const size_t per = nbytes / gridDim.x / 16;
  const uint4* p = reinterpret_cast<const uint4*>(in) + per * blockIdx.x + threadIdx.x;
  const size_t nb = per / 2048;
  uint4 A0 = ldg_stream(p), A1 = ldg_stream(p + 1024), B0, B1;
  for (size_t t = 0; t < nb; t += 2) {
    if (t + 1 < nb) { B0 = ldg_stream(p + 2048); B1 = ldg_stream(p + 3072); }
    vec(A0); vec(A1);
    if (t + 1 >= nb) break;
    if (t + 2 < nb) { A0 = ldg_stream(p + 4096); A1 = ldg_stream(p + 5120); }
    vec(B0); vec(B1);
    p += 4096;
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 256; b += 1024) {
    unsigned long long t = 0;
    for (int l = 0; l < 32; ++l) t += h[b * 32 + ((l + b) & 31)];
    atomicAdd(out + b, t);
  }
}

__global__ void fill(uint64_t* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t z = (i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    p[i] = z ^ (z >> 31);
  }
}

template <class F>
void time_it(const char* name, F launch, unsigned long long* o, size_t n) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9;
  std::vector<unsigned long long> hst(256);
  for (int r = 0; r < 6; ++r) {
    cudaMemset(o, 0, 2048);
    cudaEventRecord(a);
    for (int k = 0; k < 5; ++k) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (r && ms / 5 < best) best = ms / 5;
    if (r == 0) cudaMemcpy(hst.data(), o, 2048, cudaMemcpyDeviceToHost);
  }
  unsigned long long s = 0; for (auto x : hst) s += x;
  printf("%-28s %8.1f us  %7.1f GB/s  %s\n", name, best * 1e3, n / (best * 1e6), s == 5 * n ? "ok" : "BAD");
}

int main() {
  const int G = 296;
  size_t n = (size_t(1) << 30) / (G * 32768) * (G * 32768);  // a whole number of 32 KB batches per CTA
  uint8_t* d; cudaMalloc(&d, n);
  fill<<<1184, 256>>>((uint64_t*)d, n / 8);
  unsigned long long* o; cudaMalloc(&o, 4096);
  cudaFuncSetAttribute(k_bulk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 + 2 * 16384);
  cudaFuncSetAttribute(k_bulk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 + 4 * 16384);
  time_it("register double buffer", [&] { k_reg<<<G, 1024>>>(d, n, o); }, o, n);
  time_it("bulk copy, 2 x 16 KB stages", [&] { k_bulk<2><<<G, 1024, 32768 + 2 * 16384>>>(d, n, o); }, o, n);
  time_it("bulk copy, 4 x 16 KB stages", [&] { k_bulk<4><<<G, 1024, 32768 + 4 * 16384>>>(d, n, o); }, o, n);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("CUDA error %s\n", cudaGetErrorString(e));
  return 0;
}
