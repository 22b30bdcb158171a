// Does streaming input into shared memory with the bulk-copy engine (TMA class,
// cp.async.bulk) take shared-atomic throughput away, the way LDG write-back does?
// k_lane is bound by the L1 data pipe: 16 atomic wavefronts + 4 load write-back cycles
// per 512 B per warp (profiles/r2_l1_pipe_floor.md). If bulk fills into shared memory
// did not compete with ATOMS, a TMA -> smem -> tcgen05.cp -> TMEM -> tcgen05.ld route
// could feed the counters without the write-back cycles. Kernels (2 CTAs x 1024 threads
// per SM, the 32 KB lane-banked counter array of k_lane, a 4 x 16 KB bulk ring):
//   mode 0  warps 0-30: ATOMS on synthetic bytes (PRMT + IMAD + ATOMS); warp 31 idle
//   mode 1  the same, while warp 31 lane 0 streams HBM into the ring with cp.async.bulk
//           (16 KB per copy, mbarrier complete_tx), nobody reading the ring
//   mode 2  mode 1's bulk stream alone (warps 0-30 idle): the fill rate by itself
// Reported: warp-ATOMS per SM clock and the bulk bytes/s.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o ta tma_atoms.cu -lnvidia-ml
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include <nvml.h>

constexpr int kStages = 4;
constexpr uint32_t kStageBytes = 16384;

__device__ __forceinline__ void sh_inc(uint32_t a) { asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(a)); }
__device__ __forceinline__ uint32_t byte_of(uint32_t w, int k) { return __byte_perm(w, 0u, 0x4440u | k); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok) : "r"(bar), "r"(phase) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar) : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(1024, 2) k_probe(const uint8_t* in, size_t bytes_per_cta, int iters,
                                                   unsigned long long* cyc, unsigned long long* tma_bytes,
                                                   unsigned* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint32_t* h = reinterpret_cast<uint32_t*>(smem);  // 32 KB counters
  const uint32_t ring = (uint32_t)__cvta_generic_to_shared(smem + 32768);
  __shared__ __align__(8) unsigned long long bars[kStages];
  __shared__ volatile int stop;
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) h[i] = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init((uint32_t)__cvta_generic_to_shared(&bars[s]), 1);
    stop = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  const unsigned long long t0 = clock64();
  if (warp == 31) {
    if (MODE != 0 && (threadIdx.x & 31) == 0) {
      // stream this CTA's range through the ring until the atom warps are done (mode 1)
      // or for the whole range (mode 2); nobody reads the data
      const uint8_t* src = in + size_t(blockIdx.x) * bytes_per_cta;
      const size_t n = bytes_per_cta / kStageBytes;
      unsigned long long moved = 0;
      uint32_t phase[kStages] = {0, 0, 0, 0};
      for (int s = 0; s < kStages && s < (int)n; ++s) {
        const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[s]);
        mbar_expect_tx(bar, kStageBytes);
        bulk_g2s(ring + s * kStageBytes, src + size_t(s) * kStageBytes, kStageBytes, bar);
      }
      int last = -1;
      for (size_t k = kStages; ; ++k) {
        const int s = int(k % kStages);
        const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[s]);
        int spin = 0;
        while (!mbar_try_wait(bar, phase[s]) && ++spin < (1 << 26)) { }
        if (spin >= (1 << 26)) { moved = 0; last = s; break; }  // a copy never landed: report 0
        phase[s] ^= 1;
        moved += kStageBytes;
        if ((MODE == 1 && stop) || (MODE == 2 && k >= n)) { last = s; break; }
        mbar_expect_tx(bar, kStageBytes);
        bulk_g2s(ring + s * kStageBytes, src + size_t(k % n) * kStageBytes, kStageBytes, bar);
      }
      // drain the copies still in flight (every stage but the one just consumed)
      for (int s = 0; s < kStages; ++s) {
        if (s == last) continue;
        const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[s]);
        for (int spin = 0; spin < (1 << 24) && !mbar_try_wait(bar, phase[s]); ++spin) { }
      }
      atomicAdd(tma_bytes, moved);
    }
  } else if (MODE != 2) {
    const uint32_t tb = (uint32_t)__cvta_generic_to_shared(h) + (threadIdx.x & 31) * 4;
    uint32_t w = threadIdx.x * 0x9E3779B9u + blockIdx.x * 0x85EBCA6Bu;
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        sh_inc(tb + (byte_of(w, k & 3) << 7));
        if ((k & 3) == 3) w += 0x6F4F2A1Bu;
      }
    }
  }
  // the atom warps (0-30, named barrier 1) tell the streaming lane to stop; then all wait
  if (warp != 31) {
    asm volatile("bar.sync 1, %0;" ::"r"(992) : "memory");
    if (threadIdx.x == 0) {
      stop = 1;
      atomicAdd(cyc, clock64() - t0);
    }
  }
  __syncthreads();
  if (h[threadIdx.x] == 0xFFFFFFFFu) sink[0] = 1;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = 2 * sms;
  const size_t per_cta = 16ull << 20;  // 16 MiB per CTA, 4.6 GiB total
  uint8_t* in;
  cudaMalloc(&in, per_cta * grid);
  cudaMemset(in, 7, per_cta * grid);
  unsigned long long *cyc, *tb;
  unsigned* sink;
  cudaMalloc(&cyc, 8); cudaMalloc(&tb, 8); cudaMalloc(&sink, 4);
  const int smem = 32768 + kStages * kStageBytes;
  cudaFuncSetAttribute(k_probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  nvmlInit();
  nvmlDevice_t dev;
  nvmlDeviceGetHandleByIndex(0, &dev);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4000;
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(cyc, 0, 8); cudaMemset(tb, 0, 8);
      cudaEventRecord(e0);
      if (mode == 0) k_probe<0><<<grid, 1024, smem>>>(in, per_cta, iters, cyc, tb, sink);
      if (mode == 1) k_probe<1><<<grid, 1024, smem>>>(in, per_cta, iters, cyc, tb, sink);
      if (mode == 2) k_probe<2><<<grid, 1024, smem>>>(in, per_cta, iters, cyc, tb, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaError_t err = cudaGetLastError();
      if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); return 1; }
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long bytes = 0; cudaMemcpy(&bytes, tb, 8, cudaMemcpyDeviceToHost);
      unsigned clk = 0; nvmlDeviceGetClockInfo(dev, NVML_CLOCK_SM, &clk);
      const double atoms = mode == 2 ? 0.0 : double(grid) * 31 * iters * 16;  // warp-ATOMS
      printf("mode %d rep %d: %.3f ms, %.3f warp-ATOMS per SM clock (%u MHz), bulk %.0f GB/s\n", mode, rep, ms,
             atoms / (ms * 1e-3) / sms / (clk * 1e6), clk, bytes / (ms * 1e-3) / 1e9);
    }
  }
  return 0;
}
