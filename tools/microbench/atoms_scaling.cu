// Does lane-private shared-atomic throughput scale with warps per SM?
// Counts (byte & (NB-1)) into lane-private u32 columns (NB*32*4 bytes per warp) with
// W warps per CTA, one CTA per SM, identical per-byte instruction stream (PRMT+IMAD+ATOMS).
// Not a histogram of the data when NB < 256 -- a throughput probe only.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o as atoms_scaling.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void inc(uint32_t a) { asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(a)); }
__device__ __forceinline__ void add_ret(uint32_t a, uint32_t& sink) {
  uint32_t o; asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(o) : "r"(a)); sink ^= o;
}

template <int NB, int MODE, int U, int TH>  // MODE 0: red, 1: atom with return, 2: lds+sts (no atomic, wrong under aliasing: probe only)
__global__ void __launch_bounds__(TH, 1) k(const uint4* __restrict__ in, size_t nvec, unsigned* sink) {
  extern __shared__ __align__(16) uint8_t sm[];
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm);
  const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (uint32_t i = threadIdx.x; i < nw * NB * 32; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  __syncthreads();
  const uint32_t tb = sb + warp * NB * 128 + lane * 4;
  const uint32_t mask = NB - 1;
  size_t per = (nvec + gridDim.x - 1) / gridDim.x;
  size_t beg = blockIdx.x * per, end = min(nvec, beg + per);
  const size_t batch = (size_t)U * blockDim.x;
  size_t nfull = (end - beg) / batch;
  uint4 A[U], B[U];
  uint32_t x = 0;
  auto word = [&](uint32_t w) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t a = tb + ((__byte_perm(w, 0, 0x4440 | q) & mask) << 7);
      if (MODE == 0) inc(a);
      else if (MODE == 1) add_ret(a, x);
      else { uint32_t v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a)); asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v + 1)); }
    }
  };
  auto vec = [&](const uint4& v) { word(v.x); word(v.y); word(v.z); word(v.w); };
  const uint4* vp = in + beg;
  if (nfull) {
#pragma unroll
    for (int u = 0; u < U; ++u) A[u] = ldg_stream(vp + u * blockDim.x + threadIdx.x);
  }
  for (size_t j = 0; j < nfull; j += 2) {
    if (threadIdx.x == 0 && (j + 3) * batch * 16 < (end - beg) * 16)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(vp + (j + 3) * batch), "r"((uint32_t)(2 * batch * 16)) : "memory");
    if (j + 1 < nfull) {
#pragma unroll
      for (int u = 0; u < U; ++u) B[u] = ldg_stream(vp + (j + 1) * batch + u * blockDim.x + threadIdx.x);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) vec(A[u]);
    if (j + 1 >= nfull) break;
    if (j + 2 < nfull) {
#pragma unroll
      for (int u = 0; u < U; ++u) A[u] = ldg_stream(vp + (j + 2) * batch + u * blockDim.x + threadIdx.x);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) vec(B[u]);
  }
  __syncthreads();
  uint32_t s = x;
  for (uint32_t i = threadIdx.x; i < nw * NB * 32; i += blockDim.x) s += reinterpret_cast<uint32_t*>(sm)[i];
  atomicAdd(sink, s);
}

template <int NB, int MODE, int U, int TH>
int run(const uint4* d, size_t n, unsigned* sink, int sms, int warps, const char* tag) {
  size_t smem = (size_t)warps * NB * 128;
  CK(cudaFuncSetAttribute(k<NB, MODE, U, TH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  std::vector<float> t;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int r = 0; r < 8; ++r) {
    cudaMemset(sink, 0, 4);
    cudaEventRecord(a);
    k<NB, MODE, U, TH><<<sms, warps * 32, smem>>>(d, n / 16, sink);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (r >= 3) t.push_back(ms);
  }
  unsigned h; cudaMemcpy(&h, sink, 4, cudaMemcpyDeviceToHost);
  std::sort(t.begin(), t.end());
  printf("%-10s U=%2d NB=%3d warps=%2d smem=%6zu  %.3f ms  %7.1f GB/s  (sum %s)\n", tag, U, NB, warps, smem, t[2], n / (t[2] * 1e6),
         (MODE == 2) ? "n/a" : (h == (unsigned)n ? "ok" : "BAD"));
  return 0;
}

__global__ void fill(uint8_t* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n / 8; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t z = (i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; z ^= z >> 31;
    reinterpret_cast<uint64_t*>(p)[i] = z;
  }
}

int main() {
  size_t n = (size_t)1 << 30;
  uint8_t* d; CK(cudaMalloc(&d, n));
  unsigned* sink; CK(cudaMalloc(&sink, 4));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  fill<<<sms * 8, 256>>>(d, n);
  CK(cudaDeviceSynchronize());
  const uint4* in = reinterpret_cast<const uint4*>(d);
  run<256, 0, 8, 224>(in, n, sink, sms, 7, "red");
  run<256, 0, 4, 224>(in, n, sink, sms, 7, "red");
  run<256, 0, 4, 192>(in, n, sink, sms, 6, "red");
  run<256, 0, 4, 128>(in, n, sink, sms, 4, "red");
  run<128, 0, 4, 448>(in, n, sink, sms, 14, "red");
  run<128, 0, 4, 256>(in, n, sink, sms, 8, "red");
  run<64, 0, 4, 896>(in, n, sink, sms, 28, "red");
  run<64, 0, 4, 512>(in, n, sink, sms, 16, "red");
  run<64, 0, 2, 896>(in, n, sink, sms, 28, "red");
  run<32, 0, 2, 1024>(in, n, sink, sms, 32, "red");
  run<256, 1, 4, 224>(in, n, sink, sms, 7, "atom_ret");
  run<128, 1, 4, 448>(in, n, sink, sms, 14, "atom_ret");
  run<256, 2, 4, 224>(in, n, sink, sms, 7, "lds_sts");
  run<128, 2, 4, 448>(in, n, sink, sms, 14, "lds_sts");
  run<64, 2, 4, 896>(in, n, sink, sms, 28, "lds_sts");
  return 0;
}
