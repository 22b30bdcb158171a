// libhist256 host side: the CPU control plane around the kernels, native so the
// pattern/policy step stays far below a chunk's device time (the reference's
// Python apportionment costs 310-820 us per call, SURVEY.md §7 hard part 3).
//
//   hs_binning_pattern  <- compute_binning_pattern / uniform_pattern (pattern.py:85-133)
//   hs_degeneracy       <- degeneracy (policy.py:39-46)
//   hs_generate_host    <- _fill_uniform/_fill_normal/_fill_mixture + generate (datagen.py:92-178)
//
// Floating point follows the reference operation by operation; this file is built
// with -ffp-contract=off so no multiply-add is fused (numpy and numba do not fuse).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>
#if defined(__x86_64__)
#include <immintrin.h>
#endif

#include "../../include/hist256.h"

namespace {

// Python's int / int true division is correctly rounded; so is IEEE division of two
// exactly representable doubles. For operands >= 2^53 fall back to long double
// (64-bit mantissa) which is exact in the conversion and only risks a double
// rounding in the last bit (totals beyond 9e15 pixels).
double int_div(uint64_t a, uint64_t b) {
  if ((a >> 53) == 0 && (b >> 53) == 0) return double(a) / double(b);
  return double((long double)a / (long double)b);
}

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr double kUnit = 1.0 / 9007199254740992.0;  // 2^-53

inline uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <class F>
void parallel_for(uint64_t n, int threads, F&& f) {
  if (threads <= 1 || n < (1ull << 20)) { f(0, n); return; }
  const uint64_t t = std::min<uint64_t>(uint64_t(threads), n >> 16);
  std::vector<std::thread> pool;
  pool.reserve(t);
  for (uint64_t i = 0; i < t; ++i) {
    uint64_t a = n * i / t, b = n * (i + 1) / t;
    a &= ~uint64_t(7); b = (i + 1 == t) ? n : (b & ~uint64_t(7));
    pool.emplace_back([&f, a, b] { f(a, b); });
  }
  for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

int hs_binning_pattern(const uint64_t* prior, int64_t total_slots, int64_t cap, int64_t* offset,
                       int64_t* count) {
  if (!prior || !offset || !count) return HS_ERR_INVALID_ARG;
  // _check_slot_range (pattern.py:70-76)
  if (cap < 1) return HS_ERR_SLOT_RANGE;
  if (!(256 <= total_slots && total_slots <= 256 * cap)) return HS_ERR_SLOT_RANGE;
  const int64_t extras = total_slots - 256;
  uint64_t total = 0;  // Histogram256.total(): uint64 sum (wraps like numpy)
  for (int b = 0; b < 256; ++b) total += prior[b];
  double ideal[256];
  if (total == 0) {
    const double share = double(extras) / 256.0;  // extras / BINS
    for (int b = 0; b < 256; ++b) ideal[b] = share;
  } else {
    const double r = int_div(uint64_t(extras), total);  // extras / total
    for (int b = 0; b < 256; ++b) ideal[b] = double(prior[b]) * r;
  }
  double floors[256];
  int64_t granted_sum = 0;
  for (int b = 0; b < 256; ++b) {
    floors[b] = std::floor(ideal[b]);
    const double g = std::min(floors[b], double(cap - 1));
    const int64_t gi = int64_t(g);
    count[b] = 1 + gi;
    granted_sum += gi;
  }
  int64_t remaining = extras - granted_sum;
  if (remaining > 0) {
    double frac[256];
    int order[256];
    for (int b = 0; b < 256; ++b) { frac[b] = ideal[b] - floors[b]; order[b] = b; }
    // sorted(range(BINS), key=lambda b: (-frac[b], b))
    std::sort(order, order + 256, [&](int a, int b) {
      const double fa = -frac[a], fb = -frac[b];
      if (fa < fb) return true;
      if (fb < fa) return false;
      return a < b;
    });
    std::vector<int> pool;
    for (int i = 0; i < 256; ++i) if (count[order[i]] < cap) pool.push_back(order[i]);
    while (remaining > 0) {
      bool progressed = false;
      for (int b : pool) {
        if (count[b] < cap) {
          ++count[b];
          --remaining;
          progressed = true;
          if (remaining == 0) break;
        }
      }
      if (!progressed) return HS_ERR_SLOT_RANGE;  // unreachable while total_slots <= 256*cap
      std::vector<int> next;
      for (int b : pool) if (count[b] < cap) next.push_back(b);
      pool.swap(next);
    }
  }
  offset[0] = 0;
  for (int b = 1; b < 256; ++b) offset[b] = offset[b - 1] + count[b - 1];
  return HS_OK;
}

int hs_degeneracy(const uint64_t* counts, double* frac, int* argmax, uint64_t* total_out) {
  if (!counts || !frac || !argmax || !total_out) return HS_ERR_INVALID_ARG;
  uint64_t total = 0;
  for (int b = 0; b < 256; ++b) total += counts[b];
  *total_out = total;
  if (total == 0) { *frac = 0.0; *argmax = 0; return HS_OK; }
  int am = 0;
  for (int b = 1; b < 256; ++b) if (counts[b] > counts[am]) am = b;  // np.argmax: first max
  *argmax = am;
  *frac = int_div(counts[am], total);
  return HS_OK;
}

// numpy's pairwise float64 sum (numpy 2.x pairwise_sum, PW_BLOCKSIZE 128): blocks of at
// most 128 elements are summed with 8 interleaved accumulators combined as
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)); longer runs split at a multiple of 8 below n/2.
static double pairwise_sum(const double* a, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r += a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return pairwise_sum(a, n2) + pairwise_sum(a + n2, n - n2);
}

int hs_divergence(const uint64_t* a, const uint64_t* b, double* out) {
  if (!a || !b || !out) return HS_ERR_INVALID_ARG;
  uint64_t ta = 0, tb = 0;
  for (int k = 0; k < 256; ++k) {
    ta += a[k];
    tb += b[k];
  }
  if (ta == 0 || tb == 0) return HS_ERR_INVALID_ARG;
  const double da = double(ta), db = double(tb);
  double d[256];
  for (int k = 0; k < 256; ++k) d[k] = std::fabs(double(a[k]) / da - double(b[k]) / db);
  *out = 0.5 * pairwise_sum(d, 256);
  return HS_OK;
}

int hs_copy_streaming(void* dst, const void* src, uint64_t n, int threads) {
  if (n == 0) return HS_OK;
  if (!dst || !src) return HS_ERR_INVALID_ARG;
  uint8_t* const d0 = static_cast<uint8_t*>(dst);
  const uint8_t* const s0 = static_cast<const uint8_t*>(src);
  parallel_for(n, threads, [d0, s0](uint64_t a, uint64_t b) {
    uint8_t* d = d0 + a;
    const uint8_t* s = s0 + a;
    uint64_t m = b - a;
#if defined(__x86_64__)
    // head up to a 16-B aligned destination, then 64 B per step with streaming stores
    // (movntdq: the lines go to memory without being left dirty in the CPU caches), tail
    const uint64_t head = std::min<uint64_t>(m, (16 - (reinterpret_cast<uintptr_t>(d) & 15)) & 15);
    std::memcpy(d, s, head);
    d += head;
    s += head;
    m -= head;
    for (; m >= 64; m -= 64, d += 64, s += 64) {
      const __m128i x0 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s));
      const __m128i x1 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 16));
      const __m128i x2 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 32));
      const __m128i x3 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 48));
      _mm_stream_si128(reinterpret_cast<__m128i*>(d), x0);
      _mm_stream_si128(reinterpret_cast<__m128i*>(d + 16), x1);
      _mm_stream_si128(reinterpret_cast<__m128i*>(d + 32), x2);
      _mm_stream_si128(reinterpret_cast<__m128i*>(d + 48), x3);
    }
    std::memcpy(d, s, m);
    _mm_sfence();  // the streamed lines are in memory before the caller hands them to a DMA
#else
    std::memcpy(d, s, m);
#endif
  });
  return HS_OK;
}

int hs_generate_host(int kind, uint64_t seed, int value, double mean, double sigma, double degeneracy,
                     uint8_t* out, uint64_t n, int threads) {
  if (n == 0) return HS_OK;
  if (!out) return HS_ERR_INVALID_ARG;
  switch (kind) {
    case HS_GEN_CONSTANT:
      if (value < 0 || value > 255) return HS_ERR_INVALID_ARG;
      std::memset(out, value, n);
      return HS_OK;
    case HS_GEN_SEQUENTIAL:
      parallel_for(n, threads, [&](uint64_t a, uint64_t b) {
        for (uint64_t i = a; i < b; ++i) out[i] = uint8_t(i & 0xff);
      });
      return HS_OK;
    case HS_GEN_UNIFORM:
      // output k = mix(seed + (k+1)*GOLDEN), 8 pixels per output, LSB first
      parallel_for(n, threads, [&](uint64_t a, uint64_t b) {
        for (uint64_t i = a; i < b;) {
          const uint64_t z = mix(seed + ((i >> 3) + 1) * kGolden);
          for (int k = int(i & 7); k < 8 && i < b; ++k, ++i) out[i] = uint8_t(z >> (8 * k));
        }
      });
      return HS_OK;
    case HS_GEN_NORMAL:
      if (!(sigma > 0)) return HS_ERR_INVALID_ARG;
      parallel_for(n, threads, [&](uint64_t a, uint64_t b) {
        uint64_t state = seed + (a * 12) * kGolden;
        for (uint64_t i = a; i < b; ++i) {
          double total = 0.0;
          for (int j = 0; j < 12; ++j) {
            state += kGolden;
            total += double(mix(state) >> 11) * kUnit;
          }
          double val = std::floor(mean + sigma * (total - 6.0) + 0.5);
          if (val < 0.0) val = 0.0;
          else if (val > 255.0) val = 255.0;
          out[i] = uint8_t(val);
        }
      });
      return HS_OK;
    case HS_GEN_MIXTURE: {
      if (!(degeneracy >= 0.0 && degeneracy <= 1.0) || value < 0 || value > 255) return HS_ERR_INVALID_ARG;
      if (degeneracy == 1.0) { std::memset(out, value, n); return HS_OK; }  // generate(): constant path
      uint64_t state = seed;
      for (uint64_t i = 0; i < n; ++i) {
        state += kGolden;
        const double unit = double(mix(state) >> 11) * kUnit;
        if (unit < degeneracy) {
          out[i] = uint8_t(value);
        } else {
          state += kGolden;
          out[i] = uint8_t(mix(state) & 0xff);
        }
      }
      return HS_OK;
    }
    default:
      return HS_ERR_INVALID_ARG;
  }
}

}  // extern "C"
