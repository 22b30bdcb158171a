// atoms_form.cu (derived from atoms_rate.cu): k_lane's loop with the increment as
// ATOMS.POPC.INC (red.shared.add with an immediate 1, what k_lane compiles to) vs a plain
// ATOMS.ADD of a register holding 1: rate cold and under the power cap, clock and power.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o af atoms_form.cu -lnvidia-ml
// Original header follows.
// Conflict-free shared-atomic rate at 64 warps/SM: is k_lane's
// ~0.76 warp-ATOMS per clock per SM the atomic pipe's ceiling, or a gap?
// Kernels (1024 threads x 2 CTAs per SM, the 32 KB lane-banked counter array of k_lane):
//   atoms_only   ATOMS.POPC.INC per byte of a register word that changes by one IADD per
//                4 bytes: PRMT + IMAD + ATOMS per byte, no global loads at all
//   atoms_lds    the same addresses, LDS instead of ATOMS (the MIO pipe without atomics)
//   k_lane_like  k_lane's inner loop over 1 GiB of HBM (LDG.128 + 16 x (PRMT+IMAD+ATOMS))
// Each reports warp-ATOMS per SM per clock (rate / 148 / NVML SM clock) and the
// bytes/s-equivalent (16 B per 16 ATOMS); run for ~3 s each with NVML sampling SM clock and power alongside.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o ar atoms_rate.cu -lnvidia-ml
#include <cstdio>
#include <cstdint>
#include <chrono>
#include <thread>
#include <atomic>
#include <vector>
#include <cuda_runtime.h>
#include <nvml.h>

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void sh_inc(uint32_t a) { asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(a)); }
__device__ __forceinline__ uint32_t sh_ld(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t byte_of(uint32_t w, int k) { return __byte_perm(w, 0u, 0x4440u | k); }

template <int MODE>
__global__ void __launch_bounds__(1024, 2) k_synth(int iters, unsigned long long* cyc, unsigned* sink) {
  __shared__ __align__(16) uint32_t h[256 * 32];
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const uint32_t tb = (uint32_t)__cvta_generic_to_shared(h) + (threadIdx.x & 31) * 4;
  uint32_t w = threadIdx.x * 0x9E3779B9u + blockIdx.x * 0x85EBCA6Bu, acc = 0;
  const unsigned long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {  // 16 bytes per "vector", as k_lane
      const uint32_t a = tb + (byte_of(w, k & 3) << 7);
      if (MODE == 0) sh_inc(a); else acc += sh_ld(a);
      if ((k & 3) == 3) w += 0x6F4F2A1Bu;
    }
  }
  const unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(cyc, t1 - t0);
  if (acc == 0x1234567u) sink[0] = acc + h[threadIdx.x];
}

template <int FORM>
__global__ void __launch_bounds__(1024, 2) k_lane_like(const uint4* in, size_t nvec, unsigned long long* cyc,
                                                       unsigned* sink, unsigned one) {
  __shared__ __align__(16) uint32_t h[256 * 32];
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const uint32_t tb = (uint32_t)__cvta_generic_to_shared(h) + (threadIdx.x & 31) * 4;
  const unsigned long long t0 = clock64();
  const size_t per = (nvec / gridDim.x) / 4096 * 4096, v0 = per * blockIdx.x;  // whole rounds of 4 vectors/thread
  const uint4* p = in + v0 + threadIdx.x;
  const size_t n = per / blockDim.x;  // vectors per thread, a multiple of 4
  uint4 A[2], B[2];
  A[0] = ldg_stream(p); A[1] = ldg_stream(p + 1024);
  auto inc = [&](uint32_t a) {
    if (FORM == 0) sh_inc(a);
    else asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(one));
  };
  auto word = [&](uint32_t x) {
    inc(tb + (byte_of(x, 0) << 7)); inc(tb + (byte_of(x, 1) << 7));
    inc(tb + (byte_of(x, 2) << 7)); inc(tb + (byte_of(x, 3) << 7));
  };
  auto vec = [&](const uint4& v) { word(v.x); word(v.y); word(v.z); word(v.w); };
  for (size_t j = 0; j + 4 <= n; j += 4) {
    B[0] = ldg_stream(p + 2048); B[1] = ldg_stream(p + 3072);
    vec(A[0]); vec(A[1]);
    if (j + 4 < n) { A[0] = ldg_stream(p + 4096); A[1] = ldg_stream(p + 5120); }
    vec(B[0]); vec(B[1]);
    p += 4096;
  }
  const unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(cyc, t1 - t0);
  if (h[threadIdx.x] == 0xFFFFFFFFu) sink[0] = 1;
}

struct Sampler {
  std::atomic<bool> stop{false};
  std::vector<unsigned> mhz, mw;
  std::thread th;
  nvmlDevice_t dev;
  void start() {
    nvmlInit();
    nvmlDeviceGetHandleByIndex(0, &dev);
    th = std::thread([this] {
      while (!stop) {
        unsigned c = 0, p = 0;
        nvmlDeviceGetClockInfo(dev, NVML_CLOCK_SM, &c);
        nvmlDeviceGetPowerUsage(dev, &p);
        mhz.push_back(c); mw.push_back(p);
        std::this_thread::sleep_for(std::chrono::milliseconds(10));
      }
    });
  }
  void finish(const char* name) {
    stop = true; th.join();
    size_t n = mhz.size(), a = n / 3;  // the last two thirds: settled under the cap
    double c = 0, p = 0;
    for (size_t i = a; i < n; ++i) { c += mhz[i]; p += mw[i]; }
    printf("  %-12s settled SM clock %.0f MHz, power %.0f W (%zu samples)\n", name, c / (n - a), p / (n - a) / 1000.0, n - a);
  }
};

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = 1ull << 30, nvec = bytes / 16;
  uint4* in;
  cudaMalloc(&in, bytes);
  // random bytes (splitmix-like) so the histogram sees uniform data
  std::vector<uint64_t> hbuf(bytes / 8);
  uint64_t z = 1;
  for (auto& x : hbuf) { z += 0x9E3779B97F4A7C15ull; uint64_t q = z; q = (q ^ (q >> 30)) * 0xBF58476D1CE4E5B9ull; q = (q ^ (q >> 27)) * 0x94D049BB133111EBull; x = q ^ (q >> 31); }
  cudaMemcpy(in, hbuf.data(), bytes, cudaMemcpyHostToDevice);
  unsigned long long* cyc; unsigned* sink;
  cudaMalloc(&cyc, 8); cudaMalloc(&sink, 4);
  const int grid = 2 * sms;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch, double instr_per_launch, double bytes_per_launch) {
    for (int w = 0; w < 3; ++w) launch();
    cudaDeviceSynchronize();
    // cold: 20 launches right after idle
    std::this_thread::sleep_for(std::chrono::milliseconds(1000));
    cudaMemset(cyc, 0, 8);
    cudaEventRecord(e0);
    for (int r = 0; r < 20; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    unsigned clk = 0;
    { nvmlDevice_t d; nvmlInit(); nvmlDeviceGetHandleByIndex(0, &d); nvmlDeviceGetClockInfo(d, NVML_CLOCK_SM, &clk); }
    const double per_s = instr_per_launch / (ms / 20 * 1e-3);
    printf("%-12s cold: %.3f ms/launch, %.3f warp-ATOMS per SM clock (at %u MHz), %.0f GB/s-equivalent\n", name,
           ms / 20, per_s / sms / (clk * 1e6), clk, bytes_per_launch / (ms / 20 * 1e-3) / 1e9);
    // sustained: ~3 s with NVML sampling
    Sampler s; s.start();
    cudaMemset(cyc, 0, 8);
    int n = 0;
    auto t0 = std::chrono::steady_clock::now();
    cudaEventRecord(e0);
    while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < 3.0) {
      for (int r = 0; r < 20; ++r) launch();
      n += 20;
      cudaStreamSynchronize(0);
    }
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    s.finish(name);
    double mhz = 0;
    for (size_t i = s.mhz.size() / 3; i < s.mhz.size(); ++i) mhz += s.mhz[i];
    mhz /= double(s.mhz.size() - s.mhz.size() / 3);
    printf("  %-12s sustained: %.3f ms/launch, %.3f warp-ATOMS per SM clock, %.0f GB/s-equivalent\n", name,
           ms / n, instr_per_launch / (ms / n * 1e-3) / sms / (mhz * 1e6), bytes_per_launch / (ms / n * 1e-3) / 1e9);
  };
  const int iters = 2048;
  // per launch: grid*32 warps * iters * 16 ATOMS
  const double synth_instr = double(grid) * 32 * iters * 16, synth_bytes = double(grid) * 1024 * iters * 16;
  const double kb = double((nvec / grid) / 4096 * 4096) * grid * 16;  // bytes the kernel reads
  for (int round = 0; round < 2; ++round) {
    run("popc_inc", [&] { k_lane_like<0><<<grid, 1024>>>(in, nvec, cyc, sink, 1u); }, kb / 32, kb);
    run("atoms_add", [&] { k_lane_like<1><<<grid, 1024>>>(in, nvec, cyc, sink, 1u); }, kb / 32, kb);
  }
  return 0;
}
