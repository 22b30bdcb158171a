// Lane-banked u32 counters SHARED by all warps of a CTA: word bin*32 + lane.
// Every lane of one ATOMS hits its own bank (conflict-free); warps of the CTA share
// the 32 KB array through the atomicity of ATOMS. Footprint per CTA is fixed, so
// occupancy is free to grow. Measures CTA shape vs throughput.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o slb shared_lanebank.cu
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
__device__ __forceinline__ void red_inc(uint32_t a) { asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(a)); }

template <int U, int TH, int COPIES>
__global__ void __launch_bounds__(TH) k(const uint4* __restrict__ in, size_t nvec, unsigned long long* out) {
  // COPIES lane-banked arrays per CTA; warp w uses copy w % COPIES
  __shared__ __align__(16) uint32_t h[COPIES * 256 * 32];
  for (int i = threadIdx.x; i < COPIES * 256 * 32; i += TH) h[i] = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t tb = (uint32_t)__cvta_generic_to_shared(h) + (warp % COPIES) * 32768 + lane * 4;
  size_t per = (nvec + gridDim.x - 1) / gridDim.x;
  size_t beg = blockIdx.x * per, end = min(nvec, beg + per);
  const size_t batch = (size_t)U * TH;
  const size_t nfull = (end - beg) / batch;
  uint4 A[U], B[U];
  auto word = [&](uint32_t w) {
#pragma unroll
    for (int q = 0; q < 4; ++q) red_inc(tb + (__byte_perm(w, 0, 0x4440 | q) << 7));
  };
  auto vec = [&](const uint4& v) { word(v.x); word(v.y); word(v.z); word(v.w); };
  const uint4* vp = in + beg;
  if (nfull) {
#pragma unroll
    for (int u = 0; u < U; ++u) A[u] = ldg_stream(vp + u * TH + threadIdx.x);
  }
  for (size_t j = 0; j < nfull; j += 2) {
    if (j + 1 < nfull) {
#pragma unroll
      for (int u = 0; u < U; ++u) B[u] = ldg_stream(vp + (j + 1) * batch + u * TH + threadIdx.x);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) vec(A[u]);
    if (j + 1 >= nfull) break;
    if (j + 2 < nfull) {
#pragma unroll
      for (int u = 0; u < U; ++u) A[u] = ldg_stream(vp + (j + 2) * batch + u * TH + threadIdx.x);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) vec(B[u]);
  }
  for (size_t i = beg + nfull * batch + threadIdx.x; i < end; i += TH) vec(ldg_stream(in + i));
  asm volatile("" ::: "memory");
  __syncthreads();
  for (int b = threadIdx.x; b < 256; b += TH) {
    unsigned long long s = 0;
    for (int c = 0; c < COPIES; ++c)
      for (int l = 0; l < 32; ++l) s += h[c * 8192 + b * 32 + ((l + b) & 31)];
    if (s) atomicAdd(out + b, s);
  }
}

template <int U, int TH, int COPIES>
int run(const uint4* d, size_t n, unsigned long long* out, int grid, const std::vector<unsigned long long>& ref,
        const char* tag) {
  std::vector<float> t;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  bool ok = true;
  for (int r = 0; r < 8; ++r) {
    cudaMemset(out, 0, 2048);
    cudaEventRecord(a);
    k<U, TH, COPIES><<<grid, TH>>>(d, n / 16, out);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    CK(cudaGetLastError());
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (r >= 3) t.push_back(ms);
    if (r == 0) {
      std::vector<unsigned long long> h(256);
      cudaMemcpy(h.data(), out, 2048, cudaMemcpyDeviceToHost);
      ok = h == ref;
    }
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k<U, TH, COPIES>, TH, 0);
  std::sort(t.begin(), t.end());
  printf("%-10s U=%d threads=%4d copies=%d grid=%5d occ=%d (warps/SM %2d)  %.3f ms  %7.1f GB/s  %s\n", tag, U, TH,
         COPIES, grid, occ, occ * TH / 32, t[2], n / (t[2] * 1e6), ok ? "exact" : "MISMATCH");
  return 0;
}

__global__ void fill(uint8_t* p, size_t n, int kind) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n / 8; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t z = (i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; z ^= z >> 31;
    uint64_t v = z;
    if (kind == 1) v = 0x7f7f7f7f7f7f7f7full;
    if (kind == 2) v = (z & 0x0707070707070707ull) + 0x7c7c7c7c7c7c7c7cull;
    reinterpret_cast<uint64_t*>(p)[i] = v;
  }
}

int main() {
  size_t n = (size_t)1 << 30;
  uint8_t* d; CK(cudaMalloc(&d, n));
  unsigned long long* out; CK(cudaMalloc(&out, 2048));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  std::vector<uint8_t> hbuf(n);
  const char* names[] = {"uniform", "const127", "narrow8"};
  for (int kind = 0; kind < 3; ++kind) {
    fill<<<sms * 8, 256>>>(d, n, kind);
    CK(cudaDeviceSynchronize());
    cudaMemcpy(hbuf.data(), d, n, cudaMemcpyDeviceToHost);
    std::vector<unsigned long long> ref(256, 0);
    for (size_t i = 0; i < n; ++i) ref[hbuf[i]]++;
    const uint4* in = reinterpret_cast<const uint4*>(d);
    run<4, 512, 1>(in, n, out, sms * 4, ref, names[kind]);

    run<8, 256, 1>(in, n, out, sms * 6, ref, names[kind]);
    run<4, 256, 1>(in, n, out, sms * 8, ref, names[kind]);
    run<2, 1024, 1>(in, n, out, sms * 2, ref, names[kind]);
    run<8, 512, 1>(in, n, out, sms * 4, ref, names[kind]);
    run<4, 384, 1>(in, n, out, sms * 4, ref, names[kind]);
    run<6, 384, 1>(in, n, out, sms * 4, ref, names[kind]);
  }
  return 0;
}
