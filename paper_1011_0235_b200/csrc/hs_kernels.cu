// libhist256 device side: sm_100a kernels for the 256-bin byte histogram of
// arXiv 1011.0235 and the C ABI that launches them (include/hist256.h).
//
// Reference behaviour being replaced (all paths /root/reference/pkg/src/histostream):
//   _naive_worker     kernels.py:97-130   -> k_lane (HS_IMPL_LANE) / k_warp (HS_IMPL_WARP)
//   _adaptive_worker  kernels.py:133-168  -> k_lane<HOT> (HS_IMPL_LANE) / k_subbin (HS_IMPL_SUBBIN)
//   reduce_subbins    kernels.py:410-418  -> fused flush epilogues below
//   merge_all         core.py:152-156     -> u64 RED into a workspace row per segment, moved to d_out by
//                                            the segment's last CTA (integer adds commute: exact)
//   batch_histograms  stream.py:260-316   -> one launch per <= kMaxSeg segments and <= 1 GiB
//   _adaptive_worker_traced / _u16        -> k_group_slots (reference group/lane mapping)
//   _stage_*_worker   kernels.py:212-264  -> k_genealogy (production skeleton)
//   _fill_*           datagen.py:98-133   -> k_gen_*
//
// Design notes (numbers in DESIGN.md §4, tools/microbench/hist_variants.cu):
//   * Input bytes are read once with 16-B streaming loads (LDG.128, L1::no_allocate),
//     register double-buffered so a batch is in flight while the previous one is counted.
//   * HS_IMPL_LANE keeps one u32 counter column per lane: counter (lane, bin) is shared
//     word bin*32 + lane of ONE 32 KB array used by all 32 warps of the CTA, so every
//     lane of an ATOMS hits its own bank (conflict-free for any input, including fully
//     degenerate data) and occupancy is unconstrained (2 CTAs = 64 warps per SM).
//   * Blackwell merges same-address lanes of one shared atomic, so the contention the
//     paper's AHist relieves (all lanes on one bin) is cheap here; what costs is distinct
//     addresses in one bank. ADAPTIVE therefore keeps the lane-banked core; for a prior
//     dominated by one value it counts that hot bin's all-hot 16-byte vectors in a
//     register (no shared-memory traffic at all on degenerate input).
//   * Launches are chained with programmatic dependent launch (griddepcontrol): a launch
//     streams while the previous one's tail drains. Output is ticketed (one kernel per
//     launch, no memset) through a workspace slot: large calls use the serial slot and
//     wait for their predecessor before their first RED; small single-launch calls take
//     rotating slots, so only their output store waits (WsHeader).
//   * CTA ranges are whole 4 KiB units of the launch's concatenated range; full-grid
//     launches over several segments weight the split so that a CTA crossing a segment
//     boundary (and paying a flush there) gets less data.
//   * The blocking entries (hs_histogram_sync / hs_histogram_host) size the grid for
//     latency and let the kernel write the counts into a page-locked h_out.
#include <cuda_runtime.h>
#include <cstdint>
#ifdef HS_CHECK_SPLIT
#include <cstdio>
#endif
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <vector>

#include "../../include/hist256.h"

namespace {

constexpr int kMaxSeg = 256;         // segments per launch (SegParams ~6.5 KB: large kernel params)
constexpr int kMaxSegEngine = 64;    // per hs_stream_step batch (the fold stages it in shared memory)
constexpr size_t kTicketBytes = 1024;  // per call slot: kMaxSeg u32 tickets
// Ticketed workspace = [header][kCallSlots rotating slots + 1 serial slot, each tickets +
// accumulator rows]: see WsHeader.
#ifndef HS_CALL_SLOTS
#define HS_CALL_SLOTS HS_WS_SLOTS
#endif
constexpr int kCallSlots = HS_CALL_SLOTS;
static_assert(kCallSlots >= 1 && kCallSlots <= 31, "warp 0's lanes 1..K probe the slots");
constexpr size_t kWsHeadBytes = HS_WS_HEAD_BYTES;
// Every rotating call adds exactly kArrive to the header's call counter (claim_and_probe_warp0);
// grids must stay below it.
constexpr unsigned long long kArrive = 4096;
constexpr uint64_t kBigCap = 1ull << 30;  // u32 per-warp counters: far from wrapping
// CTA ranges are whole multiples of 4 KiB of the launch's concatenated range: with
// ranges cut at word granularity (1 GiB over 296 CTAs = 3,627,504 bytes each) a warp's
// 512-byte vector load straddles five 128-byte lines instead of four, and a 1 GiB
// launch took 162 us instead of 157 us (tools/size_sweep.py)
constexpr uint64_t kSplitWords = 1024;

constexpr int kMaxSplitGrid = 320;  // weighted split table size (>= 2 CTAs x 148 SMs)

struct SegParams {
  uint64_t begin[kMaxSeg];       // device byte offset of segment s
  uint64_t vstart[kMaxSeg + 1];  // virtual (concatenated) start of segment s
  int nseg;
  int out_base;                  // index of segment 0 of this launch in d_out
  int acc_base;                  // its workspace accumulator row / ticket index
  // segments that continue in the next launch of the same call (bit s): their CTAs
  // only RED into the accumulator row; the launch holding a segment's end finalizes it
  uint32_t open_mask[kMaxSeg / 32];
  // balanced split of the concatenated range over the grid in kSplitWords units,
  // precomputed on the host (no 64-bit division on the device): CTA b owns q units,
  // plus one if b < r; the last unit may be partial
  uint64_t q, r;
  // Cost-weighted split (split_cost > 0, k_lane launches over several segments): a CTA
  // whose range crosses a segment boundary flushes its counters there (barrier, drain
  // of the load pipeline, 256 global REDs), so such a CTA is given split_cost fewer
  // units. Cost(u) = u + split_cost * (boundaries before unit u); CTA b starts at the
  // first unit whose cost reaches floor(b * Cost(units) / grid) = cq*b + cr*b/grid,
  // tabulated on the host in cta_unit (the fields above it describe the split).
  uint32_t split_cost;
  uint32_t lead_empty;           // boundaries s >= 1 at virtual offset 0 (not counted)
  uint64_t units;                // kSplitWords units of the launch
  uint64_t cq;
  uint32_t cr;
  uint32_t ctas_after_first[kMaxSeg];  // CTAs with work in segment s, minus one
  uint32_t cta_unit[kMaxSplitGrid + 1];  // weighted split: first unit of CTA b (host-computed)
  // HS_KIND_FLAG_MERGE: every segment counts into ONE output row (merge_all of the
  // per-slice histograms, core.py:152-156, formed in the epilogue): a CTA flushes once
  // whatever the segment boundaries in its range, and only the call's last launch
  // (merge_final) takes tickets -- merge_ctas + 1 of its CTAs have work.
  int merge;
  int merge_final;
  uint32_t merge_ctas;
};

// output / accumulator row of launch-local segment s
__host__ __device__ __forceinline__ int seg_row(const SegParams& sp, int s) { return sp.merge ? 0 : s; }

// Cost of the first u units under the weighted split (host: the table is built at launch)
inline uint64_t split_cost_at(const SegParams& sp, uint64_t u) {
  const uint64_t x = u * (4 * kSplitWords);
  int lo = 1, hi = sp.nseg;  // first s in [1, nseg) with vstart[s] >= x
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (sp.vstart[mid] < x) lo = mid + 1; else hi = mid;
  }
  const uint32_t before = uint32_t(lo - 1);
  const uint32_t nb = before > sp.lead_empty ? before - sp.lead_empty : 0u;
  return u + uint64_t(sp.split_cost) * nb;
}

#ifdef HS_CHECK_SPLIT
// First unit of CTA b (b == grid: the end) under the weighted split, by binary search:
// the definition split_table() is checked against in HS_CHECK_SPLIT builds
inline uint64_t split_unit_of(const SegParams& sp, uint32_t b, uint32_t grid) {
  const uint64_t t = sp.cq * b + (uint64_t(sp.cr) * b) / grid;
  uint64_t lo = 0, hi = sp.units;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (split_cost_at(sp, mid) < t) lo = mid + 1; else hi = mid;
  }
  return lo;
}
#endif

struct PatternParams {
  uint32_t entry[256];           // offset | count << 16   (sub-bin kernels)
  int32_t total_slots;
  int32_t hot_bin;               // ADAPTIVE hot bin (argmax count, lowest bin on ties)
  int32_t hot_unique;            // exactly one bin holds the maximal count: a dominant value
};

// ------------------------------------------------------------------ primitives
__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ void sh_inc(uint32_t addr) {
  asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr));
}

__device__ __forceinline__ void sh_add(uint32_t addr, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v));
}

__device__ __forceinline__ uint32_t sh_ld(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ void sh_st(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v));
}

__device__ __forceinline__ void sh_st4(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w));
}

__device__ __forceinline__ void compiler_fence() { asm volatile("" ::: "memory"); }

// Programmatic dependent launch (no-ops unless launched with the PDL attribute):
// let the next kernel on the stream start filling SMs as this one's CTAs retire, and
// wait for the previous kernel to finish before touching memory it may still use.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Instrumented builds only (-DHS_TRACE, tools/trace_lane.py): thread 0 of each k_lane
// CTA stamps %globaltimer at fixed points of its life; compiled out otherwise.
#ifdef HS_TRACE
__device__ unsigned long long hs_trace_buf[1024][16];
#define HS_STAMP(slot)                                                                          \
  do {                                                                                          \
    if (threadIdx.x == 0 && blockIdx.x < 1024 && (slot) < 16) {                                 \
      unsigned long long t_;                                                                    \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                    \
      hs_trace_buf[blockIdx.x][(slot)] = t_;                                                    \
    }                                                                                           \
  } while (0)
#define HS_FSTAMP(slot)                                                                         \
  do {                                                                                          \
    if (threadIdx.x == 0) {                                                                     \
      unsigned long long t_;                                                                    \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                    \
      hs_trace_buf[1023][(slot)] = t_;                                                          \
    }                                                                                           \
  } while (0)
#else
#define HS_STAMP(slot) do { } while (0)
#define HS_FSTAMP(slot) do { } while (0)
#endif

// byte k of w, zero-extended (PRMT)
__device__ __forceinline__ uint32_t byte_of(uint32_t w, int k) { return __byte_perm(w, 0u, 0x4440u | k); }

// ------------------------------------------------------------------ segment walk
// Block b owns the word-aligned virtual range [vb, ve) of the concatenated segments:
// The same split with the host's q, r (SegParams launches)
__device__ __forceinline__ void block_range(const SegParams& sp, uint64_t& vb, uint64_t& ve) {
  const uint64_t b = blockIdx.x, total = sp.vstart[sp.nseg];
  uint64_t u0, u1;
  if (sp.split_cost) {
    u0 = sp.cta_unit[b];
    u1 = sp.cta_unit[b + 1];
  } else {
    u0 = sp.q * b + min(b, sp.r);
    u1 = u0 + sp.q + (b < sp.r ? 1 : 0);
  }
  vb = min(total, 4 * kSplitWords * u0);
  ve = min(total, 4 * kSplitWords * u1);
}

// Walks the pieces (segment index, device byte range) of the block's range and calls
// body(seg, p0, p1) for each non-empty piece; body must end with a block-wide flush.
template <uint64_t kCap, class Body>
__device__ __forceinline__ void for_each_piece(const SegParams& sp, Body&& body) {
  uint64_t vb, ve;
  block_range(sp, vb, ve);
  if (vb >= ve) return;
  int s = 0;
  while (s < sp.nseg && sp.vstart[s + 1] <= vb) ++s;
  uint64_t v = vb;
  for (; s < sp.nseg && v < ve; ++s) {
    const uint64_t s0 = sp.vstart[s], s1 = sp.vstart[s + 1];
    if (s1 <= v) continue;
    const uint64_t hi = min(ve, s1);
    // sub-pieces of <= kCap bytes per CTA keep every narrow counter from wrapping
    for (uint64_t a = v; a < hi;) {
      const uint64_t b = (hi - a > kCap) ? a + kCap : hi;
      body(s, sp.begin[s] + (a - s0), sp.begin[s] + (b - s0));
      a = b;
    }
    v = hi;
  }
}

// Streams the device byte range [p0, p1) (word aligned) through count_word(uint32)
// and count_vec(uint4): unaligned head/tail words, then 16-B vectors in register
// double-buffered batches of U vectors per thread.
template <int U, int PF, class WordFn, class VecFn, class BatchFn>
__device__ __forceinline__ void stream_range(const uint8_t* __restrict__ data, uint64_t p0, uint64_t p1,
                                             WordFn&& count_word, VecFn&& count_vec, BatchFn&& count_batch) {
  const uint32_t T = blockDim.x, tid = threadIdx.x;
  // 16-B alignment is decided on absolute addresses (data itself is only word aligned)
  const uint64_t base = reinterpret_cast<uintptr_t>(data);
  const uint64_t a0 = min(p1, ((base + p0 + 15) & ~uint64_t(15)) - base);
  const uint64_t a1 = max(a0, ((base + p1) & ~uint64_t(15)) - base);
  for (uint64_t i = p0 + 4ull * tid; i < a0; i += 4ull * T)
    count_word(*reinterpret_cast<const uint32_t*>(data + i));
  for (uint64_t i = a1 + 4ull * tid; i < p1; i += 4ull * T)
    count_word(*reinterpret_cast<const uint32_t*>(data + i));
  const uint4* __restrict__ vp = reinterpret_cast<const uint4*>(data + a0);
  const uint64_t nv = (a1 - a0) >> 4;
  const uint64_t batch = (uint64_t)U * T;
  const uint64_t nfull = nv / batch;
  // Bulk L2 prefetch PF batches ahead: with one CTA of 7 warps per SM the register
  // double buffer alone keeps too few bytes in flight to cover HBM latency; the
  // prefetched lines turn the LDG.128s into L2 hits. Issued by one thread, no
  // registers or shared memory involved.
  const uint64_t vbytes = nv << 4, bbytes = batch << 4;
  auto prefetch = [&](uint64_t j) {
    const uint64_t off = j * bbytes;
    if (tid == 0 && PF > 0 && off < vbytes) {
      const uint32_t len = uint32_t(min(bbytes, vbytes - off));
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(data + a0 + off), "r"(len) : "memory");
    }
  };
#pragma unroll 1
  for (int j = 1; j <= PF; ++j) prefetch(j);
  uint4 A[U], B[U];
  if (nfull > 0) {
#pragma unroll
    for (int u = 0; u < U; ++u) A[u] = ldg_stream(vp + u * T + tid);
  }
  for (uint64_t j = 0; j < nfull; j += 2) {
    prefetch(j + 1 + PF);
    prefetch(j + 2 + PF);
    if (j + 1 < nfull) {
      const uint4* q = vp + (j + 1) * batch + tid;
#pragma unroll
      for (int u = 0; u < U; ++u) B[u] = ldg_stream(q + u * T);
    }
    count_batch(A);
    if (j + 1 >= nfull) break;
    if (j + 2 < nfull) {
      const uint4* q = vp + (j + 2) * batch + tid;
#pragma unroll
      for (int u = 0; u < U; ++u) A[u] = ldg_stream(q + u * T);
    }
    count_batch(B);
  }
  for (uint64_t i = nfull * batch + tid; i < nv; i += T) count_vec(ldg_stream(vp + i));
}

// count_batch adapter for kernels without a batch-level decision
template <int U, class VecFn>
struct EachVec {
  VecFn& f;
  __device__ __forceinline__ void operator()(const uint4 (&v)[U]) const {
#pragma unroll
    for (int u = 0; u < U; ++u) f(v[u]);
  }
};
template <int U, class VecFn>
__device__ __forceinline__ EachVec<U, VecFn> each_vec(VecFn& f) { return EachVec<U, VecFn>{f}; }

// ================================================================== HS_IMPL_LANE
// Lane-banked u32 counters shared by every warp of the CTA: counter (lane, bin) is
// shared word bin*32 + lane of one 32 KB array. Within one warp-wide atomic each lane
// hits its own bank (conflict-free for ANY data, fully degenerate included); across
// warps the array is shared through the atomicity of ATOMS. Because the footprint per
// CTA is fixed at 32 KB, occupancy is free: 2 CTAs x 32 warps = 64 warps per SM keep
// the loads and the shared-atomic pipe busy (tools/microbench/shared_lanebank.cu).
// Per byte: PRMT (extract) + IMAD (address) + ATOMS.POPC.INC.
// A column (lane) adds at most piece/32 per flush; pieces are capped at 1 GiB per CTA.
// Plain form: threads per CTA and resident CTAs per SM. Measured alternatives at the
// same 64 warps/SM (tools/size_sweep.py, 1 GiB launches, before the 4 KiB-aligned
// split): 672 x 3 -> 171 us, 512 x 4 -> 184 us, against 162 us here; each CTA brings
// its own 32 KB counter array, and more arrays per SM slow the shared atomics (as did
// two arrays per CTA).
#ifndef HS_LANE_THREADS
#define HS_LANE_THREADS 1024
#define HS_LANE_BLOCKS 2
#endif
constexpr int kLaneThreads = HS_LANE_THREADS;
constexpr int kLaneBlocks = HS_LANE_BLOCKS;
constexpr int kLaneHotThreads = 768;
static_assert(kMaxSeg <= kLaneHotThreads && kMaxSeg <= kLaneThreads, "one ticket-taking thread per segment");
constexpr int kLaneMinBlocks = 2;  // HOT form
constexpr uint32_t kLaneArrayBytes = 256 * 32 * 4;

// Ticketed output (single launch, no memset): CTAs RED their counts for launch-local
// segment s into an accumulator row acc[s] of a workspace slot (zero between calls);
// after a fence each CTA takes a ticket, and the last CTA to finish segment s takes the
// row with atomicExch(.., 0) (reading and re-zeroing it), stores out[s] and resets the
// ticket. Tail work is O(256) whatever the number of CTAs.
//
// Two ways a call gets its slot (the workspace header, WsHeader):
//  * serial (large or multi-launch calls): the slot after the rotating ones; every CTA
//    waits for the previous launch on the stream to complete (griddepcontrol.wait)
//    before its first RED, so calls -- and the launches of one call -- use it in turn.
//  * rotating (single-launch calls up to kRotateMaxBytes): consecutive such calls take
//    slots 0, 1, .., K-1, 0, .. Each CTA arrives on the call counter before it lets the
//    next launch in, so the counter orders the calls; a call's CTAs RED into their slot
//    once every earlier call on it has drained it (drained[slot] == the call's epoch),
//    and the call's last finalization releases it (drained[slot] = epoch + 1) -- before
//    waiting for the predecessor. Only the CTAs that store the output wait for the
//    previous launch (the output is what a call shares with it); the rest of the call
//    streams, flushes and exits while earlier calls drain. A small call's time is then
//    one completion latency, not its predecessor's whole tail: 1 MiB chained calls 4.3 ->
//    2.3 us. For larger launches the arrival (an atomic round trip before the trigger) on
//    the launch-to-launch path costs more than the overlap gains (48 MiB: 8.7 -> 10.3 us),
//    so they stay serial (profiles/r2_call_slots.txt).
//    Deadlock-free: a launch starts only after every CTA of the launch before it has
//    arrived, so when a CTA spins on its slot, all CTAs of earlier calls are resident or
//    done, and an earlier call's release waits on nothing later.
struct WsHeader {  // one 128-byte line per field: the arrivals do not contend with the probes
  unsigned long long calls;            // kArrive per rotating call
  unsigned long long pad0[15];
  unsigned int drained[kCallSlots];    // calls that have released slot j
  unsigned int pad1[32 - kCallSlots];
  unsigned int finalized[kCallSlots];  // finalizations of the current call on slot j
  unsigned int pad2[32 - kCallSlots];
};
static_assert(sizeof(WsHeader) <= kWsHeadBytes, "workspace header");

struct Tickets {
  WsHeader* hdr;       // nullptr: untracked output (memset + RED into d_out)
  uint8_t* slots;      // slot j at slots + j * slot_bytes: [tickets][rows]; j = kCallSlots: serial
  uint32_t slot_bytes;
  uint32_t rotate;     // this call takes a rotating slot (one launch)
  uint32_t nfinal;     // segment finalizations of the call (rotating: releases the slot)
};

// The slot a CTA counts into
struct SlotView {
  unsigned int* ticket;
  unsigned long long* acc;
  uint32_t slot, epoch, probe;  // probe: drained[slot] as read after the claim
};

__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void set_slot(const Tickets& tk, uint32_t slot, SlotView& sv) {
  sv.slot = slot;
  uint8_t* base = tk.slots + size_t(slot) * tk.slot_bytes;
  sv.ticket = reinterpret_cast<unsigned int*>(base);
  sv.acc = reinterpret_cast<unsigned long long*>(base + kTicketBytes);
}

// warp 0 of every CTA of a rotating call, before it triggers. Lane 0 arrives on the call
// counter (CTA 0 adds kArrive - grid + 1, the others 1, so the counter moves by kArrive
// per call and the value returned to any CTA of the call, over kArrive, is the call's
// number n, which names its slot and epoch) while lanes 1..K read (acquire)
// every slot's drained word, so the probe's round trip overlaps the arrival's instead of
// following it (tools/trace_lane.py: wait return -> loop begin 1.4 us, two round trips).
// Reading drained[] before the claim is returned is sound: the word only reaches the
// call's epoch through the release of the slot's previous user, never beyond it before
// this call releases it, so probe == epoch still means "released" (await_slot), and an
// older value only sends await_slot to its acquire loop. lane 0 then lets the next
// launch in; the first flush looks at sv.probe.
__device__ __forceinline__ void claim_and_probe_warp0(const Tickets& tk, SlotView& sv) {
  const uint32_t lane = threadIdx.x & 31;
  unsigned long long n = 0;
  if (lane == 0) n = atomicAdd(&tk.hdr->calls, blockIdx.x == 0 ? kArrive - gridDim.x + 1 : 1ull);
  // lanes 1..K acquire drained[lane - 1] (issued behind the arrival, not ordered before it:
  // an acquire orders only its own thread's later accesses, and lane 0 is not among them)
  const unsigned int d =
      (lane >= 1 && lane <= uint32_t(kCallSlots)) ? ld_acquire_u32(&tk.hdr->drained[lane - 1]) : 0u;
  n = __shfl_sync(0xffffffffu, n, 0) / kArrive;
  const uint32_t slot = uint32_t(n % kCallSlots);
  const unsigned int probe = __shfl_sync(0xffffffffu, d, slot + 1);
  if (lane == 0) {
    set_slot(tk, slot, sv);
    sv.epoch = uint32_t(n / kCallSlots);
    pdl_launch_dependents();
    sv.probe = probe;
  }
}

// thread 0, before the CTA's first RED into a rotating slot: every earlier call on the
// slot has released it (the prologue's acquire saw the release store -- the barrier
// before the flush carries that to every thread's REDs -- or the acquire loop does)
__device__ __forceinline__ void await_slot(const Tickets& tk, SlotView& sv) {
  if (sv.probe == sv.epoch) return;  // acquired in the prologue (claim_and_probe_warp0)
  while (ld_acquire_u32(&tk.hdr->drained[sv.slot]) != sv.epoch) __nanosleep(64);
  sv.probe = sv.epoch;
}

// Adds the CTA's counters into dst[256] (the output row, or the segment's accumulator
// row of a ticketed launch) and re-zeroes them unless this was the CTA's last piece:
// 4 threads per bin, each summing 8 of the bin's 32 lane words (staggered: conflict
// free), shuffle-combined. No fence here: the fence and the tickets are taken once per
// CTA at the end (lane_tickets), after all of its flushes.
__device__ __forceinline__ void lane_flush(uint32_t sbase, unsigned long long* __restrict__ dst, bool rezero,
                                           bool wait_pred) {
  compiler_fence();
  __syncthreads();
  if (wait_pred) pdl_wait();  // the previous launch may still own the rows (see k_lane)
  for (uint32_t t = threadIdx.x; t < 1024; t += blockDim.x) {
    const uint32_t b = t >> 2, sub = t & 3;
    uint32_t v = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t a = sbase + b * 128 + (((sub * 8 + i + b) & 31) << 2);
      v += sh_ld(a);
      if (rezero) sh_st(a, 0);  // not after the CTA's last piece
    }
    unsigned long long tot = v;
    tot += __shfl_xor_sync(0xffffffffu, tot, 1);
    tot += __shfl_xor_sync(0xffffffffu, tot, 2);
    if (sub == 0 && tot) atomicAdd(dst + b, tot);
  }
  compiler_fence();
  __syncthreads();
}

// The rotating call's last finalization releases its slot
__device__ __forceinline__ void release_slot(const Tickets& tk, const SlotView& sv, int m) {
  if (threadIdx.x != 0) return;
  // (the caller's barrier orders the CTA's drains before thread 0; the fence makes the
  // release cover them at GPU scope)
  __threadfence();
  if (unsigned(m) == tk.nfinal) {  // the call's only finalizing CTA
    st_release_u32(&tk.hdr->drained[sv.slot], sv.epoch + 1);
    return;
  }
  if (atomicAdd(&tk.hdr->finalized[sv.slot], unsigned(m)) + unsigned(m) == tk.nfinal) {
    tk.hdr->finalized[sv.slot] = 0;
    __threadfence();
    st_release_u32(&tk.hdr->drained[sv.slot], sv.epoch + 1);
  }
}

// End of a ticketed CTA that flushed segments [s_first, s_last] into their accumulator
// rows: one fence, then a ticket per segment; the last CTA of a segment takes the row
// with atomicExch(.., 0) (reading and re-zeroing it) and stores the output row. Tickets
// are atomicInc with the segment's last ticket as the wrap limit, so the last CTA's
// ticket returns the counter to zero by itself: no reset store for the slot's release
// fence to wait on, and the slot's rows and tickets are zero again when the call ends.
// stage: the CTA's 32 KB counter array, free after its last flush (16 rows of u64[256])
constexpr int kStageRows = 16;
__device__ __forceinline__ void lane_tickets(const Tickets& tk, const SlotView& sv, const SegParams& sp, int s_first,
                                          int s_last, unsigned long long* __restrict__ out, uint32_t* stage_words) {
  __shared__ int last_seg[kMaxSeg];
  __shared__ int n_last;
  if (sp.merge && !sp.merge_final) return;  // a later launch of the call finalizes the row
  if (threadIdx.x == 0) n_last = 0;
  __threadfence();
  __syncthreads();
  // one ticket per segment, taken by thread (s - s_first) so that a CTA spanning several
  // segments pays one round trip, not one per segment; a thread that draws a segment's
  // last ticket fences (acquire: the other CTAs' REDs) before the barrier carries it to
  // every thread
  if (sp.merge) {
    if (threadIdx.x == 0 && atomicInc(sv.ticket + sp.acc_base, sp.merge_ctas) == sp.merge_ctas) {
      __threadfence();
      last_seg[0] = 0;
      n_last = 1;
    }
  } else if (s_first + int(threadIdx.x) <= s_last) {
    const int s = s_first + int(threadIdx.x);
    if (sp.vstart[s + 1] != sp.vstart[s] &&                 // empty: no CTA owns it
        !((sp.open_mask[s >> 5] >> (s & 31)) & 1) &&        // open: finalized by a later launch
        atomicInc(sv.ticket + sp.acc_base + s, sp.ctas_after_first[s]) == sp.ctas_after_first[s]) {
      __threadfence();
      last_seg[atomicAdd(&n_last, 1)] = s;
    }
  }
  __syncthreads();
  const int m = n_last;
  if (!m) return;
  // The output is what this call shares with its predecessor on the stream (the same
  // buffer, or one the predecessor reads): it is stored only once that one is complete
  // (griddepcontrol.wait; serial calls have waited before their first RED). A rotating
  // slot is drained and released before that wait, so later calls can take it meanwhile.
  if (tk.rotate && m <= kStageRows) {
    unsigned long long* stage = reinterpret_cast<unsigned long long*>(stage_words);
    for (int k = 0; k < m; ++k) {
      const int s = last_seg[k];
      for (uint32_t b = threadIdx.x; b < 256; b += blockDim.x)
        stage[k * 256 + b] = atomicExch(sv.acc + size_t(sp.acc_base + s) * 256 + b, 0ull);
    }
    __syncthreads();
    release_slot(tk, sv, m);
    pdl_wait();
    for (int k = 0; k < m; ++k)
      for (uint32_t b = threadIdx.x; b < 256; b += blockDim.x)
        out[size_t(sp.out_base + last_seg[k]) * 256 + b] = stage[k * 256 + b];
    return;
  }
  pdl_wait();
  for (int k = 0; k < m; ++k) {
    const int s = last_seg[k];
    for (uint32_t b = threadIdx.x; b < 256; b += blockDim.x)
      out[size_t(sp.out_base + s) * 256 + b] = atomicExch(sv.acc + size_t(sp.acc_base + s) * 256 + b, 0ull);
  }
  if (tk.rotate) {
    __syncthreads();
    release_slot(tk, sv, m);
  }
}

// The streaming loop of one piece, written lean for the 32-register budget of 64
// resident warps: the < U*T-vector remainder is counted first, so nothing but the
// running 16-B pointer, a countdown and the column base is live across the main
// double-buffered loop; compile-time stride.
template <int U, bool HOT, int TH, class Hook>
__device__ __forceinline__ uint32_t lane_loop(const uint8_t* __restrict__ data, uint64_t a0, uint64_t a1,
                                              uint32_t tb, uint32_t hot4, Hook&& hook) {
  constexpr uint32_t T = TH;
  const uint32_t tid = threadIdx.x;
  uint32_t hotcnt = 0;
  auto word = [&](uint32_t w) {
    sh_inc(tb + (byte_of(w, 0) << 7));
    sh_inc(tb + (byte_of(w, 1) << 7));
    sh_inc(tb + (byte_of(w, 2) << 7));
    sh_inc(tb + (byte_of(w, 3) << 7));
  };
  auto vec = [&](const uint4& v) {
    if (HOT) {  // a 16-B vector made only of the hot bin is counted in a register
      const uint32_t d = (v.x ^ hot4) | (v.y ^ hot4) | (v.z ^ hot4) | (v.w ^ hot4);
      if (d == 0) { hotcnt += 16; return; }
    }
    word(v.x); word(v.y); word(v.z); word(v.w);
  };
  const uint32_t nv = uint32_t((a1 - a0) >> 4);  // pieces are < 2^36 bytes
  uint32_t nfull = nv / (U * T);
  {
    const uint4* __restrict__ r = reinterpret_cast<const uint4*>(data + a0);
    for (uint32_t i = nfull * U * T + tid; i < nv; i += T) vec(ldg_stream(r + i));
  }
  const uint4* __restrict__ q = reinterpret_cast<const uint4*>(data + a0) + tid;
  uint4 A[U], B[U];
  if (nfull > 0) {
#pragma unroll
    for (int u = 0; u < U; ++u) A[u] = ldg_stream(q + u * T);
  }
  hook();  // (the CTA's first piece: its start protocol, while the first loads are in flight)
  // invariant at the loop head: A holds batch 0 of the nfull batches left at q
  while (nfull >= 2) {
#pragma unroll
    for (int u = 0; u < U; ++u) B[u] = ldg_stream(q + (U + u) * T);
#pragma unroll
    for (int u = 0; u < U; ++u) vec(A[u]);
    if (nfull > 2) {
#pragma unroll
      for (int u = 0; u < U; ++u) A[u] = ldg_stream(q + (2 * U + u) * T);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) vec(B[u]);
    q += 2 * U * T;
    nfull -= 2;
  }
  if (nfull == 1) {
#pragma unroll
    for (int u = 0; u < U; ++u) vec(A[u]);
  }
  return hotcnt;
}

// One piece [p0, p1): unaligned head/tail words, then the 16-B body. HOT (ADAPTIVE)
// tests every vector against the CPU pattern's hot bin and adds the register count of
// hot bytes to the thread's column at the end.
// Everything in k_lane is inlined: with no calls there is no ABI stack frame, and
// ptxas keeps the global-memory descriptor in a uniform register (the noinline form
// re-moved it with 4 R2UR per load pair). tests/test_native_abi.py checks the SASS of
// the streaming loop (tools/loopcheck.py): no local-memory traffic, no R2UR.
// (Tried and rejected: verifying the hot bin on a per-CTA sample and switching between
// the checked and the plain loop at run time -- both loops in one function exceed the
// 32-register budget of 64 resident warps and the plain loop spills.)
template <int U, bool HOT, int TH, class Hook>
__device__ __forceinline__ uint32_t lane_piece(const uint8_t* __restrict__ data, uint64_t p0, uint64_t p1,
                                            uint32_t tb, uint32_t hot4, Hook&& hook) {
  const uint32_t tid = threadIdx.x;
  auto word = [&](uint32_t w) {
    sh_inc(tb + (byte_of(w, 0) << 7));
    sh_inc(tb + (byte_of(w, 1) << 7));
    sh_inc(tb + (byte_of(w, 2) << 7));
    sh_inc(tb + (byte_of(w, 3) << 7));
  };
  const uint64_t base = reinterpret_cast<uintptr_t>(data);
  const uint64_t a0 = min(p1, ((base + p0 + 15) & ~uint64_t(15)) - base);
  const uint64_t a1 = max(a0, ((base + p1) & ~uint64_t(15)) - base);
  if (p0 + 4ull * tid < a0) word(*reinterpret_cast<const uint32_t*>(data + p0 + 4ull * tid));
  if (a1 + 4ull * tid < p1) word(*reinterpret_cast<const uint32_t*>(data + a1 + 4ull * tid));
  const uint32_t hotcnt = lane_loop<U, HOT, TH>(data, a0, a1, tb, hot4, hook);
  if (HOT && hotcnt) sh_add(tb + ((hot4 & 0xffu) << 7), hotcnt);
  return 0;
}

// HOT (ADAPTIVE): register path for the hot bin `hot_bin`.
// wait_first: the first launch of a public call, whose stream predecessor may be the
// kernel that wrote the input: wait for it (griddepcontrol.wait: complete and flushed)
// before the first load. The next launch is still allowed to become resident early;
// if it too waits first, it waits for us, hence transitively for our producer.
// Chained launches (later launches of the same call, hs_stream_step, or a caller's
// HS_KIND_FLAG_CHAINED) stream before their predecessor -- a libhist256 kernel, which
// never writes the input -- has finished, and wait only before their first write.
template <int U, bool HOT, int TH = kLaneThreads, int MB = kLaneBlocks>
__global__ void __launch_bounds__(TH, MB)
    k_lane(const uint8_t* __restrict__ data, const __grid_constant__ SegParams sp, int hot_bin,
           unsigned long long* __restrict__ out, Tickets tk, int wait_first) {
  __shared__ __align__(16) uint32_t counters[256 * 32];
  // The CTA's pieces (segment, byte range) are listed in shared memory first, so no
  // segment-walk state is live across the streaming loop (it would take registers the
  // loop needs at 64 resident warps).
  __shared__ uint64_t pc_p0[kMaxSeg], pc_p1[kMaxSeg];
  __shared__ int pc_seg[kMaxSeg];
  __shared__ int pc_n;
  __shared__ SlotView sv;
  HS_STAMP(0);
  // A call's first launch waits for its stream predecessor before loading (round 2 A/B,
  // profiles/r2_first_launch_ab.txt: waiting first, then letting the next launch in, was
  // the fastest safe order). A rotating call's CTAs let the next launch in only after
  // arriving on the workspace's call counter (claim_and_probe_warp0), which orders the calls' slots.
  if (wait_first) pdl_wait();
  const bool ticketed = tk.hdr != nullptr;
  const bool rotating = ticketed && tk.rotate;
  // A CTA counts as triggered once any of its threads has executed launch_dependents
  // (tools/microbench/pdl_trigger.cu). Every thread triggering at entry lets the next
  // launch in soonest (in the microbenchmark a lone thread's trigger took ~2 us longer to
  // take effect); a rotating call's CTAs trigger from thread 0 only, after its arrival
  // is back, so that every CTA of the call arrives before any CTA of the next one.
  if (!rotating) pdl_launch_dependents();
  if (rotating && threadIdx.x < 32) claim_and_probe_warp0(tk, sv);
  if (threadIdx.x == 0) {
    if (ticketed && !rotating) set_slot(tk, kCallSlots, sv);
    int n = 0;
    for_each_piece<~0ull>(sp, [&](int s, uint64_t p0, uint64_t p1) {
      pc_p0[n] = p0;
      pc_p1[n] = p1;
      pc_seg[n] = s;
      ++n;
    });
    pc_n = n;
  }
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(counters);
  for (uint32_t i = threadIdx.x; i < kLaneArrayBytes / 16; i += blockDim.x) sh_st4(sbase + i * 16, make_uint4(0, 0, 0, 0));
  __syncthreads();
  const uint32_t tb = sbase + (threadIdx.x & 31) * 4;  // column base: bank == lane
  const uint32_t hot = uint32_t(hot_bin) & 0xff;
  if (ticketed && blockIdx.x == 0 && !sp.merge) {
    // ticketed launches have no memset: CTA 0 zeroes the empty segments' outputs
    bool any_empty = false;
    for (int s = 0; s < sp.nseg; ++s) any_empty |= sp.vstart[s + 1] == sp.vstart[s];
    if (any_empty) {
      pdl_wait();
      for (int s = 0; s < sp.nseg; ++s)
        if (sp.vstart[s + 1] == sp.vstart[s])
          for (uint32_t b = threadIdx.x; b < 256; b += blockDim.x) out[size_t(sp.out_base + s) * 256 + b] = 0;
    }
  }
  auto no_hook = []() {};
  // u32 columns: a column adds at most (CTA bytes)/32 <= 2^32, so one flush per
  // (CTA, segment) suffices -- required by the ticketed output
  const uint32_t hot4 = hot * 0x01010101u;
  HS_STAMP(1);
  for (int i = 0; i < pc_n; ++i) {
    lane_piece<U, HOT, TH>(data, pc_p0[i], pc_p1[i], tb, hot4, no_hook);
    HS_STAMP(2 + 2 * i);
    if (sp.merge && i + 1 < pc_n) continue;  // merged output: one flush per CTA
    const int r = seg_row(sp, pc_seg[i]);
    // a rotating call counts into its slot once the slot is free; a serial one once the
    // previous launch on the stream is complete (and so, transitively, every earlier one)
    if (rotating && threadIdx.x == 0) await_slot(tk, sv);  // lane_flush's barrier publishes it
    lane_flush(sbase, ticketed ? sv.acc + size_t(sp.acc_base + r) * 256 : out + size_t(sp.out_base + r) * 256,
               i + 1 < pc_n, ticketed && !rotating);
    HS_STAMP(3 + 2 * i);
  }
  if (ticketed && pc_n > 0) lane_tickets(tk, sv, sp, pc_seg[0], pc_seg[pc_n - 1], out, counters);
  HS_STAMP(15);
}

// ================================================================== HS_IMPL_WARP
// per-warp shared u32[256] (SDK / paper NVHist). 8 warps per block.
constexpr int kWarpThreads = 256;

template <int U, int PF>
__global__ void __launch_bounds__(kWarpThreads)
    k_warp(const uint8_t* __restrict__ data, const __grid_constant__ SegParams sp,
           unsigned long long* __restrict__ out) {
  __shared__ __align__(16) uint32_t hist[8 * 256];
  for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const uint32_t hb = (uint32_t)__cvta_generic_to_shared(hist) + (threadIdx.x >> 5) * 1024;
  auto word = [&](uint32_t w) {
    sh_inc(hb + (byte_of(w, 0) << 2));
    sh_inc(hb + (byte_of(w, 1) << 2));
    sh_inc(hb + (byte_of(w, 2) << 2));
    sh_inc(hb + (byte_of(w, 3) << 2));
  };
  auto vec = [&](const uint4& v) { word(v.x); word(v.y); word(v.z); word(v.w); };
  for_each_piece<kBigCap>(sp, [&](int s, uint64_t p0, uint64_t p1) {
    stream_range<U, PF>(data, p0, p1, word, vec, each_vec<U>(vec));
    compiler_fence();
    __syncthreads();
    const int b = threadIdx.x;
    unsigned long long tot = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) { tot += hist[w * 256 + b]; hist[w * 256 + b] = 0; }
    if (tot) atomicAdd(out + size_t(sp.out_base + seg_row(sp, s)) * 256 + b, tot);
    __syncthreads();
  });
}

// ================================================================== HS_IMPL_SUBBIN
// The paper's AHist: per-warp S-slot array; lane L adds byte b into slot
// offset[b] + L % count[b] (kernels.py:149-150). The CPU pattern is expanded into a
// lane-banked LUT slot_of[b*32 + lane] (32 KB) so the per-byte lookup is conflict-free;
// the slot atomics themselves see the pattern's bank spread.
constexpr int kSubThreads = 256;

template <int U, int PF>
__global__ void __launch_bounds__(kSubThreads)
    k_subbin(const uint8_t* __restrict__ data, const __grid_constant__ SegParams sp,
             const __grid_constant__ PatternParams pp, unsigned long long* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t* lut = reinterpret_cast<uint32_t*>(smem);            // 256*32 words
  uint32_t* slots = lut + 256 * 32;                             // 8 warps x S
  const int S = pp.total_slots;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) {
    const uint32_t b = i >> 5, l = i & 31, e = pp.entry[b];
    const uint32_t off = e & 0xffff, cnt = e >> 16;
    lut[i] = (off + l % cnt) * 4;
  }
  for (int i = threadIdx.x; i < 8 * S; i += blockDim.x) slots[i] = 0;
  __syncthreads();
  const uint32_t lb = (uint32_t)__cvta_generic_to_shared(lut) + lane * 4;
  const uint32_t wb = (uint32_t)__cvta_generic_to_shared(slots) + warp * S * 4;
  auto word = [&](uint32_t w) {
    sh_inc(wb + sh_ld(lb + (byte_of(w, 0) << 7)));
    sh_inc(wb + sh_ld(lb + (byte_of(w, 1) << 7)));
    sh_inc(wb + sh_ld(lb + (byte_of(w, 2) << 7)));
    sh_inc(wb + sh_ld(lb + (byte_of(w, 3) << 7)));
  };
  auto vec = [&](const uint4& v) { word(v.x); word(v.y); word(v.z); word(v.w); };
  for_each_piece<kBigCap>(sp, [&](int s, uint64_t p0, uint64_t p1) {
    stream_range<U, PF>(data, p0, p1, word, vec, each_vec<U>(vec));
    compiler_fence();
    __syncthreads();
    // reduce_subbins fused: bin b = sum of its count[b] slots over the 8 warps
    const int b = threadIdx.x;
    const uint32_t e = pp.entry[b], off = e & 0xffff, cnt = e >> 16;
    unsigned long long tot = 0;
    for (int w = 0; w < 8; ++w)
      for (uint32_t j = 0; j < cnt; ++j) tot += slots[w * S + off + j];
    __syncthreads();
    for (int i = threadIdx.x; i < 8 * S; i += blockDim.x) slots[i] = 0;
    if (tot) atomicAdd(out + size_t(sp.out_base + seg_row(sp, s)) * 256 + b, tot);
    __syncthreads();
  });
}

// ================================================================== compat slots
// Reference group/lane mapping, one thread per word; global 64-bit atomics.
__global__ void k_group_slots(const uint32_t* __restrict__ words, uint64_t n_words, int group_size,
                              int group_count, const __grid_constant__ PatternParams pp, int mode,
                              unsigned long long* __restrict__ out) {
  const uint64_t base = n_words / group_count;
  const int S = pp.total_slots;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_words;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t g = base ? min(i / base, uint64_t(group_count - 1)) : uint64_t(group_count - 1);
    const uint64_t start = g * base;
    const uint32_t lane = uint32_t((i - start) % uint64_t(group_size));
    const uint32_t w = words[i];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t b = (w >> (8 * k)) & 0xff;
      const uint32_t e = pp.entry[b], off = e & 0xffff, cnt = e >> 16;
      const uint32_t slot = off + lane % cnt;
      size_t idx = mode == 1 ? (g * group_size + lane) * S + slot : g * S + slot;
      atomicAdd(out + idx, 1ull);
    }
  }
}

__global__ void k_wrap16(const unsigned long long* __restrict__ in, uint16_t* __restrict__ out, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (uint16_t)(in[i] & 0xffff);
}

// ================================================================== ablation (genealogy)
// The paper's Table 1 (run_ablation, kernels.py:212-264, :421-496): cumulative stages on
// the PRODUCTION skeleton -- k_lane's 1024-thread CTAs, two per SM, 16-B streaming loads
// in 4 KiB-aligned CTA ranges -- with shared memory only from the stage that needs it:
//   COPY_ONLY         read every word, XOR checksum                   (no shared memory)
//   COPY_INIT         + zero the 32 KB lane-banked counter array       (32 KB)
//   PATTERN_LOAD      + per pixel, read the pattern's entry for its bin from a lane-banked
//                       table (offset[b] + count[b], the reference's per-pixel load) (64 KB)
//   SUBHIST_NOREDUCE  + per pixel, increment the (bin, lane) sub-counter -- on the B200
//                       a bin's sub-bins are its 32 lane columns
//   FULL              + reduce the 32 columns per bin and merge into d_out (u64 RED)
// Sinks: COPY_* the XOR of every 32-bit word, PATTERN_LOAD the XOR over pixels of
// offset[b] + count[b] -- both the reference's values; SUBHIST/FULL the number of
// increments (the host turns it into the reference's per-group form).
template <int U, int TH, class WordFn, class VecFn>
__device__ __forceinline__ void gen_piece(const uint8_t* __restrict__ data, uint64_t p0, uint64_t p1,
                                          WordFn&& word, VecFn&& vec) {
  constexpr uint32_t T = TH;
  const uint32_t tid = threadIdx.x;
  const uint64_t base = reinterpret_cast<uintptr_t>(data);
  const uint64_t a0 = min(p1, ((base + p0 + 15) & ~uint64_t(15)) - base);
  const uint64_t a1 = max(a0, ((base + p1) & ~uint64_t(15)) - base);
  if (p0 + 4ull * tid < a0) word(*reinterpret_cast<const uint32_t*>(data + p0 + 4ull * tid));
  if (a1 + 4ull * tid < p1) word(*reinterpret_cast<const uint32_t*>(data + a1 + 4ull * tid));
  const uint32_t nv = uint32_t((a1 - a0) >> 4);
  uint32_t nfull = nv / (U * T);
  {
    const uint4* __restrict__ r = reinterpret_cast<const uint4*>(data + a0);
    for (uint32_t i = nfull * U * T + tid; i < nv; i += T) vec(ldg_stream(r + i));
  }
  const uint4* __restrict__ q = reinterpret_cast<const uint4*>(data + a0) + tid;
  uint4 A[U], B[U];
  if (nfull > 0) {
#pragma unroll
    for (int u = 0; u < U; ++u) A[u] = ldg_stream(q + u * T);
  }
  while (nfull >= 2) {
#pragma unroll
    for (int u = 0; u < U; ++u) B[u] = ldg_stream(q + (U + u) * T);
#pragma unroll
    for (int u = 0; u < U; ++u) vec(A[u]);
    if (nfull > 2) {
#pragma unroll
      for (int u = 0; u < U; ++u) A[u] = ldg_stream(q + (2 * U + u) * T);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) vec(B[u]);
    q += 2 * U * T;
    nfull -= 2;
  }
  if (nfull == 1) {
#pragma unroll
    for (int u = 0; u < U; ++u) vec(A[u]);
  }
}

template <int STAGE>
__global__ void __launch_bounds__(kLaneThreads, kLaneBlocks)
    k_genealogy(const uint8_t* __restrict__ data, uint64_t n_bytes, uint64_t q, uint64_t r,
                const __grid_constant__ PatternParams pp, unsigned long long* __restrict__ sink,
                unsigned long long* __restrict__ out) {
  extern __shared__ __align__(16) uint32_t gsm[];
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t cbase = (uint32_t)__cvta_generic_to_shared(gsm);  // counters [256][32]
  const uint32_t tbase = cbase + kLaneArrayBytes;                    // table    [256][32]
  if (STAGE >= HS_STAGE_COPY_INIT)
    for (uint32_t i = threadIdx.x; i < kLaneArrayBytes / 16; i += blockDim.x) sh_st4(cbase + i * 16, make_uint4(0, 0, 0, 0));
  if (STAGE >= HS_STAGE_PATTERN_LOAD)
    for (uint32_t i = threadIdx.x; i < 256 * 32; i += blockDim.x) {
      const uint32_t e = pp.entry[i >> 5];
      sh_st(tbase + i * 4, (e & 0xffffu) + (e >> 16));
    }
  if (STAGE >= HS_STAGE_COPY_INIT) __syncthreads();
  const uint32_t col = lane * 4;
  uint32_t x = 0;
  auto word = [&](uint32_t w) {
    if (STAGE <= HS_STAGE_COPY_INIT) {
      x ^= w;
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t off = (byte_of(w, k) << 7) + col;
        x ^= sh_ld(tbase + off);
        if (STAGE >= HS_STAGE_SUBHIST_NOREDUCE) sh_inc(cbase + off);
      }
    }
  };
  auto vec = [&](const uint4& v) { word(v.x); word(v.y); word(v.z); word(v.w); };
  // the CTA's whole 4 KiB units (q, r from the host: no 64-bit division on the device)
  const uint64_t b = blockIdx.x;
  const uint64_t u0 = q * b + min(b, r), u1 = u0 + q + (b < r ? 1 : 0);
  const uint64_t vb = min(n_bytes, 4 * kSplitWords * u0), ve = min(n_bytes, 4 * kSplitWords * u1);
  // the copy stages finish a vector in one LOP3 per word, so ptxas would hoist the loads
  // of both buffers and spill at U = 2 under the 32-register budget: one vector per buffer
  constexpr int U = STAGE <= HS_STAGE_COPY_INIT ? 1 : 2;
  if (vb < ve) gen_piece<U, kLaneThreads>(data, vb, ve, word, vec);
  if (STAGE <= HS_STAGE_PATTERN_LOAD) {
    // XOR is order independent: the reference's checksum whatever the schedule
    for (int o = 16; o; o >>= 1) x ^= __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0 && x) atomicXor(sink, (unsigned long long)x);
    return;
  }
  asm volatile("" ::"r"(x));  // the table loads stay part of the measured work
  compiler_fence();
  __syncthreads();
  if (STAGE == HS_STAGE_SUBHIST_NOREDUCE) {
    // sink += every sub-counter of the CTA (the reference: sum of every slot, :462-463)
    unsigned long long t = 0;
    for (uint32_t i = threadIdx.x; i < 256 * 32; i += blockDim.x) t += sh_ld(cbase + i * 4);
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0 && t) atomicAdd(sink, t);
    return;
  }
  lane_flush(cbase, out, false, false);  // FULL: reduce_subbins + merge (u64 RED per bin)
  if (threadIdx.x == 0 && vb < ve) atomicAdd(sink, (unsigned long long)(ve - vb));
}

// ================================================================== device stream engine
// Device-resident accumulator, moving window and switch policy (stream.py:62-116,
// :390-425; policy.py:39-64) so lag-1 kernel switching needs no host round trip.
// State (caller-allocated, hs_stream_state_bytes): header | acc[256] | win[256] | ring[W][256].
struct DevStreamHeader {
  uint32_t kind;   // kernel kind decided for the next iteration (logged by the next fold)
  uint32_t hot;    // hot bin for ADAPTIVE: argmax of the window (lowest bin on ties)
  uint32_t head;   // ring head
  uint32_t count;  // ring entries
  uint32_t error;  // 1: NegativeCount (stream.py:96-97), 2: empty totals
  uint32_t pad0[3];
  unsigned long long chunks_seen;
  unsigned long long t_reset_ns;  // %globaltimer when hs_stream_reset ran
  double decided_degeneracy;      // window degeneracy at the last decision (the host's
                                  // lagged choice of the register path reads it)
  unsigned long long pad1;
};
static_assert(sizeof(DevStreamHeader) == 64, "header size");

// numpy's float64 add.reduce over a contiguous array (pairwise, 8 accumulators, blocks
// of 128): reproduces np.abs(pa - pb).sum() bit for bit (numpy 2.3, checked on 20k cases)
__device__ double np_pairwise_sum(const double* a, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, a[i]);
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(np_pairwise_sum(a, n2), np_pairwise_sum(a + n2, n - n2));
}

// numpy's pairwise sum of exactly 256 doubles, in parallel: 256 = 128 + 128, and each
// 128-block is 8 running accumulators over 16 elements, combined ((0+1)+(2+3))+((4+5)+(6+7)).
// Threads 0..15 run the 16 accumulators (same order of adds, so the same bits as
// np_pairwise_sum(d, 256)); thread 0 combines. Returns the sum in thread 0.
__device__ double np_pairwise_sum256(const double* d, double* acc16) {
  const int t = threadIdx.x;
  if (t < 16) {
    const double* blk = d + (t >> 3) * 128;
    const int j = t & 7;
    double r = blk[j];
    for (int i = 8; i < 128; i += 8) r = __dadd_rn(r, blk[i + j]);
    acc16[t] = r;
  }
  __syncthreads();
  double res = 0.0;
  if (t == 0) {
    double h[2];
    for (int k = 0; k < 2; ++k) {
      const double* r = acc16 + 8 * k;
      h[k] = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                       __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    }
    res = __dadd_rn(h[0], h[1]);
  }
  return res;
}

// exact u64 sums and first maximum (value, lowest index) over bins 0..255 (threads 0..255)
struct FoldRed { unsigned long long ta, tb, mx; uint32_t am; };
__device__ FoldRed fold_reduce(unsigned long long a, unsigned long long w, uint32_t b) {
  // bins 0..255 live in warps 0..7; the block's other warps only join the barrier
  __shared__ unsigned long long r_ta[8], r_tb[8], r_mx[8];
  __shared__ uint32_t r_am[8];
  unsigned long long ta = a, tb = w, mx = w;
  uint32_t am = b;
  for (int o = 16; o > 0; o >>= 1) {
    ta += __shfl_xor_sync(0xffffffffu, ta, o);
    tb += __shfl_xor_sync(0xffffffffu, tb, o);
    const unsigned long long m2 = __shfl_xor_sync(0xffffffffu, mx, o);
    const uint32_t a2 = __shfl_xor_sync(0xffffffffu, am, o);
    if (m2 > mx || (m2 == mx && a2 < am)) { mx = m2; am = a2; }
  }
  const int wid = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0 && wid < 8) { r_ta[wid] = ta; r_tb[wid] = tb; r_mx[wid] = mx; r_am[wid] = am; }
  __syncthreads();
  FoldRed r{0, 0, r_mx[0], r_am[0]};
  for (int k = 0; k < 8; ++k) {
    r.ta += r_ta[k];
    r.tb += r_tb[k];
    if (r_mx[k] > r.mx || (r_mx[k] == r.mx && r_am[k] < r.am)) { r.mx = r_mx[k]; r.am = r_am[k]; }
  }
  return r;
}

// One CTA of 256 threads, latency-bound (one launch per iteration): all threads first
// stage the batch's chunk histograms into shared memory with independent 16-B loads
// (and the ring too for windows below kFoldSmallWin); then thread b < 256 folds bin b
// (stream.py:_StreamState.post: accumulator, window push/evict, NegativeCount check in
// push order) with every input loaded independently, kFoldBatch pushes per round.
constexpr int kFoldThreads = 256;  // one thread per bin; small enough to share an SM
                                   // with a histogram CTA of the next iteration
constexpr int kFoldBatch = 8;      // pushes whose inputs are loaded per round (registers)
constexpr int kFoldSmallWin = 16;  // windows below this keep the ring in shared memory
constexpr size_t kFoldSmem = size_t(kMaxSegEngine) * 256 * 8 + size_t(kFoldSmallWin - 1) * 256 * 8;

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// hs_stream_reset: zero the state and stamp the device clock
__global__ void k_stream_reset(unsigned long long* __restrict__ state, size_t words) {
  constexpr size_t kStamp = offsetof(DevStreamHeader, t_reset_ns) / 8;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < words; i += size_t(gridDim.x) * blockDim.x)
    state[i] = i == kStamp ? globaltimer_ns() : 0ull;
}

__global__ void __maxnreg__(128)
    k_stream_fold(const unsigned long long* __restrict__ hist, int nseg, uint8_t* __restrict__ state, int window,
                  double threshold, int decide, int iteration, double* __restrict__ deg_log,
                  double* __restrict__ div_log, int32_t* __restrict__ kind_log,
                  unsigned long long* __restrict__ ns_log) {
  DevStreamHeader* hd = reinterpret_cast<DevStreamHeader*>(state);
  unsigned long long* acc = reinterpret_cast<unsigned long long*>(state + sizeof(DevStreamHeader));
  unsigned long long* win = acc + 256;
  unsigned long long* ring = win + 256;
  extern __shared__ __align__(16) unsigned long long fold_smem[];
  unsigned long long* sh = fold_smem;                        // [nseg][256] chunk histograms
  unsigned long long* sring = fold_smem + size_t(nseg) * 256;  // [window][256] when small
  __shared__ double d[256];
  __shared__ double acc16[16];
  const uint32_t t = threadIdx.x, b = t;
  HS_FSTAMP(0);
  pdl_launch_dependents();  // the next histogram launch may start streaming meanwhile
  pdl_wait();               // the histogram launch before us must be complete
  HS_FSTAMP(1);
  const bool small = window < kFoldSmallWin;
  {
    const uint4* src = reinterpret_cast<const uint4*>(hist);
    uint4* dst = reinterpret_cast<uint4*>(sh);
    const int nv = nseg * 128;  // 16-B vectors, 16 per thread in flight per round
    constexpr int kV = 16;
    for (int i0 = 0; i0 < nv; i0 += kV * kFoldThreads) {
      uint4 v[kV];
#pragma unroll
      for (int k = 0; k < kV; ++k)
        if (i0 + t + k * kFoldThreads < nv) v[k] = __ldcg(src + i0 + t + k * kFoldThreads);
#pragma unroll
      for (int k = 0; k < kV; ++k)
        if (i0 + t + k * kFoldThreads < nv) dst[i0 + t + k * kFoldThreads] = v[k];
    }
    if (small) {
      const uint4* rs = reinterpret_cast<const uint4*>(ring);
      uint4* rd = reinterpret_cast<uint4*>(sring);
      for (int i = t; i < window * 128; i += kFoldThreads) rd[i] = __ldcg(rs + i);
    }
  }
  uint32_t head = hd->head, count = hd->count;
  unsigned long long a = acc[b], w = win[b];
  bool neg = false;
  __syncthreads();
  HS_FSTAMP(6);
  if (b < 256) {
    // The pushes as a queue: entries E = (ring, oldest first: count0 of them) followed by
    // the batch's h_0..h_{n-1}. Push k evicts E[count0 + k - W] once count0 + k >= W;
    // that entry is a ring slot when its index is below count0 and h_{idx-count0}
    // (already in shared memory) otherwise. Every evicted value is therefore known up
    // front and loaded independently; only the running window sum (for the
    // NegativeCount check, in push order) is a serial chain, of register adds.
    const unsigned long long* rg = small ? sring : ring;
    const int W = window, c0 = int(count), n = nseg;
    const int k_ev = max(0, W - c0);  // first evicting push
    for (int j0 = 0; j0 < n; j0 += kFoldBatch) {
      unsigned long long hv[kFoldBatch], ov[kFoldBatch];
#pragma unroll
      for (int k = 0; k < kFoldBatch; ++k) {
        const int j = j0 + k;
        if (j < n) {
          hv[k] = sh[j * 256 + b];
          if (j >= k_ev) {
            const int idx = c0 + j - W;  // evicted entry of E
            if (idx < c0) {
              int slot = int(head) + idx;
              if (slot >= W) slot -= W;
              ov[k] = rg[size_t(slot) * 256 + b];
            } else {
              ov[k] = sh[(idx - c0) * 256 + b];
            }
          }
        }
      }
#pragma unroll
      for (int k = 0; k < kFoldBatch; ++k) {
        const int j = j0 + k;
        if (j >= n) break;
        a += hv[k];
        w += hv[k];
        if (j >= k_ev) {
          neg |= w < ov[k];
          w -= ov[k];
        }
      }
    }
    // ring after the batch: push k sits in slot (head + count0 + k) mod W, and only
    // the last W pushes survive, so each slot is written once
    unsigned long long* rw = small ? sring : ring;
    {
      const int j0 = max(0, n - W);
      int slot = int((uint32_t(head) + uint32_t(c0) + uint32_t(j0)) % uint32_t(W));  // once
      for (int j = j0; j < n; ++j) {
        rw[size_t(slot) * 256 + b] = sh[j * 256 + b];
        slot = slot + 1 == W ? 0 : slot + 1;
      }
    }
    const int ev = max(0, c0 + n - W);
    head = uint32_t((uint32_t(head) + uint32_t(ev)) % uint32_t(W));
    count = uint32_t(min(W, c0 + n));
    acc[b] = a;
    win[b] = w;
  }
  HS_FSTAMP(7);
  __syncthreads();
  if (small) {
    const uint4* rs = reinterpret_cast<const uint4*>(sring);
    uint4* rd = reinterpret_cast<uint4*>(ring);
    for (int i = t; i < window * 128; i += kFoldThreads) rd[i] = rs[i];
  }
  HS_FSTAMP(2);
  const FoldRed r = fold_reduce(a, w, b);
  const bool err = __syncthreads_or(neg);
  HS_FSTAMP(3);
  if (b == 0) {
    const double frac = r.tb ? __ddiv_rn((double)r.mx, (double)r.tb) : 0.0;
    deg_log[iteration] = frac;
    kind_log[iteration] = int32_t(hd->kind);
    if (decide) {  // decision for the next iteration (lag 1)
      hd->kind = frac >= threshold ? HS_KIND_ADAPTIVE : HS_KIND_NAIVE;
      hd->hot = r.am;
      hd->decided_degeneracy = frac;
    }
    hd->head = head;
    hd->count = count;
    hd->chunks_seen += uint64_t(nseg);
    if (err) hd->error |= 1u;
    if (r.ta == 0 || r.tb == 0) hd->error |= 2u;
  }
  if (b < 256) {
    const double pa = r.ta ? __ddiv_rn((double)a, (double)r.ta) : 0.0;
    const double pb = r.tb ? __ddiv_rn((double)w, (double)r.tb) : 0.0;
    d[b] = fabs(__dadd_rn(pa, -pb));
  }
  HS_FSTAMP(4);
  __syncthreads();
  const double tv = np_pairwise_sum256(d, acc16);
  if (b == 0) {
    div_log[iteration] = __dmul_rn(0.5, tv);
    if (ns_log) ns_log[iteration] = globaltimer_ns();
  }
  HS_FSTAMP(5);
}


// ------------------------------------------------------------------ block engine
// Several iterations per launch chain (hs_stream_block): the histograms of all their
// chunks in ONE histogram call, then the per-iteration fold of every iteration at once.
// The fold is exact integer algebra over the sequence E = (ring, oldest first) ++ (the
// block's chunk histograms h_0..h_{m-1}): with prefix sums PE[k] = sum of E[0..k),
//   window after iteration i = PE[c0 + c_i] - PE[max(0, c0 + c_i - W)]
//   acc after iteration i    = acc_prev + PE[c0 + c_i] - PE[c0]
// (c0 = ring entries before the block, c_i = chunks up to and including iteration i),
// the same integers the reference's incremental push/evict gives (stream.py:141-178).
// Every entry is a device-made histogram (non-negative), so the window never goes
// negative (the NegativeCount guard of the per-step fold has nothing to catch here).
//   k_block_scan    local inclusive prefix of E in tiles of kScanTile rows + tile totals
//   k_block_fold    one CTA per iteration: window, acc, degeneracy, divergence -> logs
//   k_block_commit  one CTA: kind log and lag-1 decisions in order, acc/window/ring/head
constexpr int kScanTile = 16;
constexpr int kBlockMaxIter = 256;
constexpr int kBlockMaxChunks = kMaxSeg;

struct BlockMap {                 // per-block layout, host-computed
  int n_iter, m, c0_unused;
  int first_iteration;
  int end_chunk[kBlockMaxIter];   // c_i: chunks of iterations 0..i of the block
};

__device__ __forceinline__ const unsigned long long* e_row(const unsigned long long* ring, int W, uint32_t head,
                                                           int c0, const unsigned long long* hist, int k) {
  if (k < c0) {
    int slot = int(head) + k;
    if (slot >= W) slot -= W;
    return ring + size_t(slot) * 256;
  }
  return hist + size_t(k - c0) * 256;
}

// grid = ceil((W + m) / kScanTile) CTAs x 256 threads (bin b = thread). Each CTA scans
// its tile of rows; the last CTA to finish (ticket) turns the tile totals into their
// exclusive prefix in place, so PE[k] = local[k-1] + tile_pre[(k-1) / kScanTile].
__global__ void __launch_bounds__(256) k_block_scan(const unsigned long long* __restrict__ hist, int m,
                                                    const uint8_t* __restrict__ state, int W,
                                                    unsigned long long* __restrict__ local,
                                                    unsigned long long* __restrict__ tile_tot,
                                                    unsigned int* __restrict__ ticket) {
  __shared__ bool last;
  pdl_launch_dependents();
  pdl_wait();  // the block's histogram launch is complete
  const DevStreamHeader* hd = reinterpret_cast<const DevStreamHeader*>(state);
  const unsigned long long* ring = reinterpret_cast<const unsigned long long*>(state + sizeof(DevStreamHeader)) + 512;
  const int c0 = int(hd->count), R = c0 + m, b = threadIdx.x;
  const uint32_t head = hd->head;
  const int k0 = blockIdx.x * kScanTile;
  unsigned long long v[kScanTile];
#pragma unroll
  for (int j = 0; j < kScanTile; ++j) v[j] = (k0 + j < R) ? __ldcg(e_row(ring, W, head, c0, hist, k0 + j) + b) : 0ull;
  unsigned long long s = 0;
#pragma unroll
  for (int j = 0; j < kScanTile; ++j) {
    s += v[j];
    if (k0 + j < R) local[size_t(k0 + j) * 256 + b] = s;  // inclusive: E[k0..k0+j]
  }
  tile_tot[size_t(blockIdx.x) * 256 + b] = s;
  __threadfence();
  __syncthreads();
  if (b == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int T = gridDim.x;
  unsigned long long run = 0;
  for (int j0 = 0; j0 < T; j0 += 8) {  // 8 independent loads in flight per round
    unsigned long long t[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) t[j] = j0 + j < T ? __ldcg(tile_tot + size_t(j0 + j) * 256 + b) : 0ull;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j0 + j < T) {
        tile_tot[size_t(j0 + j) * 256 + b] = run;  // exclusive prefix
        run += t[j];
      }
  }
  if (b == 0) *ticket = 0;  // zero again for the next block
}

// PE[k] (sum of E[0..k)) for bin b from the tile scan
__device__ __forceinline__ unsigned long long pe_at(const unsigned long long* local, const unsigned long long* tile_pre,
                                                    int k, int b) {
  if (k <= 0) return 0ull;
  const int last = k - 1;
  return __ldcg(local + size_t(last) * 256 + b) + __ldcg(tile_pre + size_t(last / kScanTile) * 256 + b);
}

// one CTA (256 threads) per iteration of the block
__global__ void __launch_bounds__(256) k_block_fold(const __grid_constant__ BlockMap bm, uint8_t* __restrict__ state,
                                                    int W, const unsigned long long* __restrict__ local,
                                                    const unsigned long long* __restrict__ tile_tot,
                                                    double* __restrict__ deg_log, double* __restrict__ div_log,
                                                    uint32_t* __restrict__ argmax_out) {
  __shared__ double d[256];
  __shared__ double acc16[16];
  pdl_launch_dependents();
  pdl_wait();
  DevStreamHeader* hd = reinterpret_cast<DevStreamHeader*>(state);
  const unsigned long long* acc_prev = reinterpret_cast<const unsigned long long*>(state + sizeof(DevStreamHeader));
  const int i = blockIdx.x, b = threadIdx.x;
  const int c0 = int(hd->count), ci = c0 + bm.end_chunk[i];
  const int lo = max(0, ci - W);
  const unsigned long long pci = pe_at(local, tile_tot, ci, b);
  const unsigned long long w = pci - pe_at(local, tile_tot, lo, b);
  const unsigned long long a = acc_prev[b] + (pci - pe_at(local, tile_tot, c0, b));
  const FoldRed r = fold_reduce(a, w, b);
  const double frac = r.tb ? __ddiv_rn((double)r.mx, (double)r.tb) : 0.0;
  const double pa = r.ta ? __ddiv_rn((double)a, (double)r.ta) : 0.0;
  const double pb = r.tb ? __ddiv_rn((double)w, (double)r.tb) : 0.0;
  d[b] = fabs(__dadd_rn(pa, -pb));
  __syncthreads();
  const double tv = np_pairwise_sum256(d, acc16);
  if (b == 0) {
    const int it = bm.first_iteration + i;
    deg_log[it] = frac;
    div_log[it] = __dmul_rn(0.5, tv);
    argmax_out[i] = r.am;
    if (r.ta == 0 || r.tb == 0) atomicOr(&hd->error, 2u);
  }
}

// one CTA: the decisions in iteration order and the state after the block
__global__ void __launch_bounds__(256) k_block_commit(const __grid_constant__ BlockMap bm,
                                                      const unsigned long long* __restrict__ hist,
                                                      uint8_t* __restrict__ state, int W, double threshold,
                                                      int recompute_every, const unsigned long long* __restrict__ local,
                                                      const unsigned long long* __restrict__ tile_tot,
                                                      const double* __restrict__ deg_log,
                                                      const uint32_t* __restrict__ argmax_in,
                                                      int32_t* __restrict__ kind_log,
                                                      unsigned long long* __restrict__ ns_log,
                                                      unsigned long long* __restrict__ decision) {
  pdl_launch_dependents();  // the next block's histogram does not touch the state
  pdl_wait();  // every iteration's fold is done (and with it the histogram and the scan)
  DevStreamHeader* hd = reinterpret_cast<DevStreamHeader*>(state);
  unsigned long long* acc = reinterpret_cast<unsigned long long*>(state + sizeof(DevStreamHeader));
  unsigned long long* win = acc + 256;
  unsigned long long* ring = win + 256;
  const int b = threadIdx.x, m = bm.m;
  const int c0 = int(hd->count);
  const uint32_t head = hd->head;
  const int R = c0 + m;
  // acc and window after the block's last iteration
  const unsigned long long pR = pe_at(local, tile_tot, R, b);
  acc[b] += pR - pe_at(local, tile_tot, c0, b);
  win[b] = pR - pe_at(local, tile_tot, max(0, R - W), b);
  // ring: push k of the block sits in slot (head + c0 + k) mod W; only the last W survive
  {
    // 16 loads in flight per thread before their stores: one at a time, the copy of up to
    // W rows was a chain of L2 round trips (77 us of a 256-chunk block's commit in ncu)
    constexpr int kBatch = 16;
    const int j0 = max(0, m - W);
    int slot = int((uint32_t(head) + uint32_t(c0) + uint32_t(j0)) % uint32_t(W));
    for (int j = j0; j < m; j += kBatch) {
      unsigned long long v[kBatch];
#pragma unroll
      for (int u = 0; u < kBatch; ++u)
        if (j + u < m) v[u] = __ldcg(hist + size_t(j + u) * 256 + b);
#pragma unroll
      for (int u = 0; u < kBatch; ++u)
        if (j + u < m) {
          ring[size_t(slot) * 256 + b] = v[u];
          slot = slot + 1 == W ? 0 : slot + 1;
        }
    }
  }
  __shared__ double s_deg[kBlockMaxIter];
  __shared__ uint32_t s_am[kBlockMaxIter];
  __shared__ int32_t s_kind[kBlockMaxIter];
  __shared__ unsigned long long s_now;
  for (int i = b; i < bm.n_iter; i += blockDim.x) {  // independent loads, then a serial pass in smem
    s_deg[i] = __ldcg(deg_log + bm.first_iteration + i);
    s_am[i] = argmax_in[i];
  }
  __syncthreads();
  if (b == 0) {
    uint32_t kind = hd->kind, hot = hd->hot;
    double dd = hd->decided_degeneracy;
    s_now = globaltimer_ns();
    for (int i = 0; i < bm.n_iter; ++i) {
      const int it = bm.first_iteration + i;
      s_kind[i] = int32_t(kind);
      if (((it + 1) % recompute_every) == 0) {  // decision for the next iteration (lag 1)
        const double frac = s_deg[i];
        kind = frac >= threshold ? HS_KIND_ADAPTIVE : HS_KIND_NAIVE;
        hot = s_am[i];
        dd = frac;
      }
    }
    hd->kind = kind;
    hd->hot = hot;
    hd->decided_degeneracy = dd;
    if (decision) {  // the decision in force after this block, for the host (mapped memory)
      volatile unsigned long long* dv = decision;
      dv[1] = (unsigned long long)kind | ((unsigned long long)hot << 32);
      dv[2] = __double_as_longlong(dd);
      __threadfence_system();
      dv[0] = (unsigned long long)(bm.first_iteration + bm.n_iter);  // written last: the block's stamp
    }
    const int ev = max(0, R - W);
    hd->head = uint32_t((uint32_t(head) + uint32_t(ev)) % uint32_t(W));
    hd->count = uint32_t(min(W, R));
    hd->chunks_seen += uint64_t(m);
  }
  __syncthreads();
  for (int i = b; i < bm.n_iter; i += blockDim.x) {
    kind_log[bm.first_iteration + i] = s_kind[i];
    if (ns_log) ns_log[bm.first_iteration + i] = s_now;
  }
}

// ================================================================== generators
__host__ __device__ __forceinline__ uint64_t sm64_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

// uniform: pixel i is byte (i & 7) of splitmix output (i >> 3) (datagen.py:98-112)
__global__ void k_gen_uniform(uint64_t seed, uint64_t first, uint8_t* __restrict__ out, uint64_t n) {
  const uint64_t k0 = first >> 3, k1 = (first + n + 7) >> 3;
  for (uint64_t k = k0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < k1;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t z = sm64_mix(seed + (k + 1) * kGolden);
    const uint64_t p = k * 8;
    if (p >= first && p + 8 <= first + n && ((p - first) & 7) == 0 &&
        ((reinterpret_cast<uintptr_t>(out + (p - first)) & 7) == 0)) {
      *reinterpret_cast<uint64_t*>(out + (p - first)) = z;
    } else {
      for (int j = 0; j < 8; ++j) {
        const uint64_t q = p + j;
        if (q >= first && q < first + n) out[q - first] = uint8_t(z >> (8 * j));
      }
    }
  }
}

// normal: Irwin-Hall of 12 units, floor(mean + sigma*z + 0.5) clamped (datagen.py:115-133);
// explicit _rn intrinsics keep nvcc from contracting into FMA (numba does not).
__global__ void k_gen_normal(uint64_t seed, double mean, double sigma, uint64_t first,
                             uint8_t* __restrict__ out, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t pix = first + i;
    uint64_t st = seed + (pix * 12) * kGolden;
    double total = 0.0;
#pragma unroll
    for (int j = 0; j < 12; ++j) {
      st += kGolden;
      total = __dadd_rn(total, __dmul_rn((double)(sm64_mix(st) >> 11), 1.0 / 9007199254740992.0));
    }
    double val = floor(__dadd_rn(__dadd_rn(mean, __dmul_rn(sigma, __dadd_rn(total, -6.0))), 0.5));
    val = val < 0.0 ? 0.0 : (val > 255.0 ? 255.0 : val);
    out[i] = (uint8_t)val;
  }
}

__global__ void k_gen_sequential(uint64_t first, uint8_t* __restrict__ out, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = uint8_t((first + i) & 0xff);
}

// ================================================================== host helpers
inline int fold(cudaError_t e) { return e == cudaSuccess ? HS_OK : HS_ERR_CUDA_BASE - int(e); }

struct DevInfo { int sms = 0; int smem_optin = 0; int l2 = 0; };

int dev_info(DevInfo& di) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fold(e);
  // cached per device (attribute queries are cheap but not free)
  static thread_local int cached_dev = -1;
  static thread_local DevInfo cached;
  if (cached_dev == dev) { di = cached; return HS_OK; }
  if ((e = cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return fold(e);
  if ((e = cudaDeviceGetAttribute(&di.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev)) != cudaSuccess) return fold(e);
  if ((e = cudaDeviceGetAttribute(&di.l2, cudaDevAttrL2CacheSize, dev)) != cudaSuccess) return fold(e);
  cached_dev = dev;
  cached = di;
  return HS_OK;
}

int validate(const int64_t* off, const int64_t* cnt, int64_t S, int64_t cap) {
  if (!off || !cnt) return HS_ERR_PATTERN_SHAPE;
  for (int b = 0; b < 256; ++b) if (cnt[b] < 1) return HS_ERR_PATTERN_COUNT_LOW;
  for (int b = 0; b < 256; ++b) if (cnt[b] > cap) return HS_ERR_PATTERN_COUNT_HIGH;
  int64_t sum = 0;
  for (int b = 0; b < 256; ++b) sum += cnt[b];
  if (sum != S) return HS_ERR_PATTERN_TOTAL;
  if (off[0] != 0) return HS_ERR_PATTERN_OFFSETS;
  for (int b = 1; b < 256; ++b) if (off[b] != off[b - 1] + cnt[b - 1]) return HS_ERR_PATTERN_OFFSETS;
  return HS_OK;
}

// entries: the sub-bin kernels' packed (offset | count << 16) table is needed; it
// limits total_slots to 16 bits. The lane kernels use only the hot bin, so any legal
// pattern (total_slots up to 256 * cap, pattern.py:70-76) is accepted there.
int make_pattern(const int64_t* off, const int64_t* cnt, int64_t S, int64_t cap, PatternParams& pp,
                 bool entries = true) {
  int st = validate(off, cnt, S, cap);
  if (st != HS_OK) return st;
  if (entries && S > 65535) return HS_ERR_UNSUPPORTED;
  int64_t best = -1;
  int nbest = 0;
  pp.hot_bin = 0;
  for (int b = 0; b < 256; ++b) {
    const int64_t c = cnt[b] > 0xffff ? 0xffff : cnt[b];
    pp.entry[b] = uint32_t(off[b]) | (uint32_t(c) << 16);
    if (cnt[b] > best) { best = cnt[b]; pp.hot_bin = b; nbest = 1; }
    else if (cnt[b] == best) ++nbest;
  }
  // The apportionment gives a dominant value the unique widest run; a spread prior
  // (normal, uniform) ties many bins at the cap or leaves all below it.
  pp.hot_unique = nbest == 1 && best > 1;
  pp.total_slots = int32_t(S);
  return HS_OK;
}

template <class K>
int set_smem(K kernel, size_t bytes) {
  if (bytes <= 48 * 1024) return HS_OK;
  return fold(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
}

// set_smem once per device (the attribute belongs to the current device's context):
// `done` is a per-kernel bitmask of devices already configured
template <class K>
int set_smem_once(K kernel, size_t bytes, std::atomic<uint64_t>& done) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return set_smem(kernel, bytes);
  const uint64_t bit = 1ull << dev;
  if (done.load(std::memory_order_acquire) & bit) return HS_OK;
  const int rc = set_smem(kernel, bytes);
  if (rc == HS_OK) done.fetch_or(bit, std::memory_order_acq_rel);
  return rc;
}

// CTA index owning word w of the balanced split of tw words over g CTAs
uint32_t cta_of_word(uint64_t w, uint64_t tw, uint64_t g) {
  const uint64_t units = (tw + kSplitWords - 1) / kSplitWords, u = w / kSplitWords;
  const uint64_t q = units / g, r = units % g;
  if (u < r * (q + 1)) return uint32_t(u / (q + 1));
  return uint32_t(r + (u - r * (q + 1)) / q);
}

// Units a segment boundary inside a CTA's range costs that CTA (the weighted split of
// k_lane launches over several segments). 0 = plain split. Per 1 GiB launch
// (tools/split_cost_ab.py, profiles/r1_split_cost_ab.txt), plain -> 32: 16 x 64 MiB
// 158.7 -> 157.0 us, 64 x 16 MiB 158.7 -> 158.3, 64 random sizes 161.2 -> 158.8; one
// segment 156.7. The split is a host-computed table in the launch parameters: computing
// it on the device (binary searches by thread 0 before the first load) cost 2 us.
// Launches with several boundaries per CTA lose with it (256 x 1 MiB, 128 CTAs:
// 49.6 -> 55.7 us), so it applies to full-grid launches with >= 2 CTAs per segment.
#ifndef HS_SPLIT_COST
#define HS_SPLIT_COST 32
#endif
constexpr uint32_t kLaneSplitCost = HS_SPLIT_COST;

// The weighted split's table in one pass: CTA targets rise with b, so the first unit
// whose cost reaches each target is found by walking units and boundaries forward
// (O(grid + nseg); split_unit_of's binary searches were ~30 us per launch on the host).
// Boundary s counts from unit vstart[s] / unit_bytes + 1 on (Cost counts vstart < u*unit).
void split_table(const SegParams& sp, uint32_t g, uint32_t* ub) {
  const uint64_t unit_bytes = 4 * kSplitWords, d = sp.split_cost;
  int k = 1 + int(sp.lead_empty);
  uint64_t u = 0, nb = 0;
  for (uint32_t b = 0; b <= g; ++b) {
    const uint64_t t = sp.cq * b + (uint64_t(sp.cr) * b) / g;
    for (;;) {
      const uint64_t jump = k < sp.nseg ? sp.vstart[k] / unit_bytes + 1 : ~0ull;
      const uint64_t need = t > d * nb ? t - d * nb : 0;
      const uint64_t cand = std::max(u, need);
      if (cand < jump) {
        u = cand;
        break;
      }
      u = jump;  // no unit before the boundary reaches t: cross it
      ++nb;
      ++k;
    }
    ub[b] = uint32_t(u);
  }
}

// fills the grid split of sp (q, r or the weighted split, and the per-segment CTA
// counts the tickets use)
void split_grid(SegParams& sp, int grid, uint32_t split_cost = 0) {
  const uint64_t tw = sp.vstart[sp.nseg] >> 2, g = uint64_t(grid);
  const uint64_t units = (tw + kSplitWords - 1) / kSplitWords;
  sp.q = units / g;
  sp.r = units % g;
  sp.units = units;
  // plain split: CTA b has work iff it owns a unit (the last unit may be partial)
  sp.merge_ctas = uint32_t(std::max<uint64_t>(1, std::min(g, units)) - 1);
  if (sp.merge) split_cost = 0;  // no flush at segment boundaries: nothing to weigh
  sp.split_cost = sp.nseg > 1 && grid <= kMaxSplitGrid ? split_cost : 0;
  sp.lead_empty = 0;
  for (int s = 1; s < sp.nseg && sp.vstart[s] == 0; ++s) ++sp.lead_empty;
  if (sp.split_cost) {
    const uint64_t total_cost = split_cost_at(sp, units);
    sp.cq = total_cost / g;
    sp.cr = uint32_t(total_cost % g);
    uint32_t* ub = sp.cta_unit;  // units of one launch (<= 1 GiB) fit 32 bits
    split_table(sp, uint32_t(g), ub);
#ifdef HS_CHECK_SPLIT
    for (uint32_t b = 0; b <= uint32_t(g); ++b)
      if (ub[b] != split_unit_of(sp, b, uint32_t(g))) {
        fprintf(stderr, "[hs] split table mismatch at CTA %u\n", b);
        abort();
      }
#endif
    // CTAs with a non-empty range that meets segment s (units [first, last] of its words)
    uint32_t b = 0;
    for (int s = 0; s < sp.nseg; ++s) {
      sp.ctas_after_first[s] = 0;
      if (sp.vstart[s + 1] <= sp.vstart[s]) continue;
      const uint64_t uf = (sp.vstart[s] >> 2) / kSplitWords, ul = ((sp.vstart[s + 1] >> 2) - 1) / kSplitWords;
      while (ub[b + 1] <= uf) ++b;  // first CTA whose range reaches unit uf (ranges are monotone)
      uint32_t n = 0;
      for (uint32_t c = b; c < uint32_t(g) && ub[c] <= ul; ++c) n += ub[c + 1] > ub[c];
      sp.ctas_after_first[s] = n - 1;
    }
    return;
  }
  for (int s = 0; s < sp.nseg; ++s) {
    sp.ctas_after_first[s] = 0;
    if (sp.vstart[s + 1] > sp.vstart[s])
      sp.ctas_after_first[s] = cta_of_word((sp.vstart[s + 1] >> 2) - 1, tw, g) - cta_of_word(sp.vstart[s] >> 2, tw, g);
  }
}

// CTAs for a k_lane launch over v bytes (capped later by the resident slots). Each CTA
// pays a fixed start (zero 32 KB of counters) and end (flush, tickets), so mid-size
// launches run faster on fewer, longer CTAs; from ~384 MiB on every resident slot is
// used. Per-launch times (tools/size_sweep.py, graph-replayed, aligned CTA ranges):
//   16 MiB: 64 CTAs 5.6 us (>= 64 KiB per CTA, 256 CTAs: 7.7 us)
//   64 MiB: 128 CTAs 12.7 us (14.7 us);  1 GiB: 296 CTAs 154 us (256 CTAs: 159 us)
// The blocking entries (hs_histogram_sync / hs_histogram_host) wait for the one launch,
// so there the grid is sized for latency instead: >= 16 KiB per CTA below 48 MiB. On a
// 1024x1024 image that is 64 CTAs instead of 4: 28 -> 18 us per blocking call, while
// graph-replayed back-to-back launches lose 3% (tools/c1_breakdown.py).
// Back-to-back small calls (rotating call slots) run faster on more, shorter CTAs: per
// call, 1 MiB with 4 CTAs 2.38 us, 8 CTAs 2.03, 32 CTAs 1.85; 2 MiB 2.42 -> 2.0 us with
// 32 CTAs; from 6 MiB on 256 KiB per CTA stays best (8 MiB with 64 CTAs: 2.95 -> 3.46 us;
// tools/diag/late_wait_ab.py, profiles/r2_call_slots.txt). So <= 1 / 2 / 4 MiB calls get
// 32 / 64 / 128 KiB per CTA.
uint64_t lane_grid_for(uint64_t v, bool latency = false) {
  if (!latency && v <= (4ull << 20)) {
    const int s = v <= (1ull << 20) ? 15 : v <= (2ull << 20) ? 16 : 17;
    return std::max<uint64_t>(1, (v + (1ull << s) - 1) >> s);
  }
  // above 8 MiB, 512 KiB per CTA (up to 64): 10 MiB 3.52 -> 3.31 us, 12 MiB 3.89 -> 3.62,
  // 24 MiB 5.89 -> 5.72; 16 and 32-48 MiB unchanged
  const int shift = latency ? 14 : (v > (8ull << 20) ? 19 : 18);
  if (v <= (48ull << 20)) return std::max<uint64_t>(1, std::min<uint64_t>(64, (v + (1ull << shift) - 1) >> shift));
  if (v <= (384ull << 20)) return 128;
  return ~0ull;  // every resident slot
}

// one launch over the <= kMaxSeg (pieces of) segments prepared in sp
int launch_batch(const uint8_t* d_data, SegParams& sp, int kind, int impl, const PatternParams* pp,
                 unsigned long long* d_out, cudaStream_t st, const DevInfo& di, const Tickets& tk,
                 int reserve_slots, bool latency, bool wait_first) {
  const uint64_t v = sp.vstart[sp.nseg];
  if (v == 0) return HS_OK;
  cudaError_t e = cudaSuccess;
  if (impl == HS_IMPL_LANE) {
    // A call that waits for its predecessor before loading cannot overlap it, so its
    // grid is sized for its own latency: >= 64 KiB per CTA but at least min(64, v/16 KiB)
    // CTAs, up to every resident slot. Back-to-back waiting calls (profiles/
    // r2_call_slots.txt): 1 MiB 11.8 -> 8.5 us, 16 MiB 19.1 (32 CTAs) -> 12.4 us (256),
    // 48 MiB 23.0 -> 15.3, 256 MiB 51.1 -> 46.3 us against the throughput grid.
    const uint64_t want =
        (wait_first && !latency && v <= (384ull << 20))
            ? std::max<uint64_t>((v + (1ull << 16) - 1) >> 16, std::min<uint64_t>(64, (v + (1ull << 14) - 1) >> 14))
            : lane_grid_for(v, latency);
    // reserve_slots CTA slots are left free (the device stream engine's fold CTA takes
    // one while the next histogram streams, instead of delaying one of its CTAs)
    const bool hot = kind == HS_KIND_ADAPTIVE && pp != nullptr && pp->hot_unique;
    const int per_sm = hot ? kLaneMinBlocks : kLaneBlocks;
    const int grid = int(std::max<uint64_t>(
        1, std::min<uint64_t>(want, uint64_t(di.sms) * per_sm - uint64_t(reserve_slots))));
    // weighted split only for full-grid launches with at least two CTAs per segment:
    // with several boundaries per CTA, or one CTA per SM, it measured slower
    // (256 x 1 MiB: 49.6 -> 55.7 us)
    const bool weighted = want == ~0ull && 2 * sp.nseg <= grid && !sp.merge;
    split_grid(sp, grid, weighted ? kLaneSplitCost : 0);
    const int hb = pp ? pp->hot_bin : 0;
    // ADAPTIVE runs the register path for the pattern's hot bin only when the pattern
    // marks a dominant value (unique widest sub-bin run, and no HS_KIND_FLAG_SPREAD
    // from the caller). The HOT form uses 768-thread CTAs (40 registers): at 1024
    // threads its loop spills under the 32-register budget.
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    // PDL overlaps a launch's ramp with the previous launch's tail (in the device
    // stream engine: with the previous iteration's one-CTA fold)
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (tk.hdr != nullptr && uint64_t(grid) >= kArrive) return HS_ERR_UNSUPPORTED;
    if (hot) {
      cfg.blockDim = dim3(kLaneHotThreads);
      e = cudaLaunchKernelEx(&cfg, k_lane<2, true, kLaneHotThreads, kLaneMinBlocks>, d_data, sp, hb, d_out, tk,
                             int(wait_first));
    } else {
      cfg.blockDim = dim3(kLaneThreads);
      e = cudaLaunchKernelEx(&cfg, k_lane<2, false>, d_data, sp, hb, d_out, tk, int(wait_first));
    }
    if (e != cudaSuccess) return fold(e);
  } else if (impl == HS_IMPL_WARP) {
    const uint64_t want = (v + (32ull << 10) - 1) / (32ull << 10);
    const int grid = int(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(di.sms) * 8)));
    split_grid(sp, grid);
    k_warp<4, 0><<<grid, kWarpThreads, 0, st>>>(d_data, sp, d_out);
  } else if (impl == HS_IMPL_SUBBIN) {
    if (!pp) return HS_ERR_INVALID_ARG;
    const size_t smem = (256 * 32 + 8 * size_t(pp->total_slots)) * 4;
    if (smem > (size_t)di.smem_optin) return HS_ERR_UNSUPPORTED;
    int rc = set_smem(k_subbin<4, 0>, smem);
    if (rc != HS_OK) return rc;
    const uint64_t want = (v + (64ull << 10) - 1) / (64ull << 10);
    const int per_sm = std::max(1, int(di.smem_optin / (smem + 1024)));
    const int grid = int(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(di.sms) * per_sm)));
    split_grid(sp, grid);
    k_subbin<4, 0><<<grid, kSubThreads, smem, st>>>(d_data, sp, *pp, d_out);
  } else {
    return HS_ERR_INVALID_ARG;
  }
  e = cudaGetLastError();
  return fold(e);
}

// Segments [s0, s0 + ns) as launches of at most kLaunchBytes each. A single launch over
// many GiB lets the two CTAs of an SM drift apart (the exits of a 16 GiB launch spread
// from 57% to 100% of its time; tools/trace_lane.py), and the SM idles once its faster
// CTA is done. Consecutive <= 1 GiB launches with programmatic dependent launch refill
// those slots with the next launch's CTAs: one 16 GiB call 5.93 -> 6.57 TB/s, measured
// from a settled power state (the board's power cap otherwise confounds long runs;
// DESIGN.md §5). A segment cut by a launch boundary accumulates in
// its workspace row (or, without a workspace, in d_out after the memset) and is
// finalized by the launch that holds its end.
constexpr uint64_t kLaunchBytes = 1ull << 30;  // a word multiple, so every cut is word aligned

int launch_segments(const uint8_t* d_data, const uint64_t* h_begin, const uint64_t* h_end, int s0, int ns,
                    int kind, int impl, const PatternParams* pp, unsigned long long* d_out, cudaStream_t st,
                    const DevInfo& di, Tickets& tk, int reserve_slots, bool latency, bool& wait_first,
                    bool merge = false, bool final_group = true) {
  uint64_t vs[kMaxSeg + 1];
  vs[0] = 0;
  for (int i = 0; i < ns; ++i) vs[i + 1] = vs[i] + (h_end[s0 + i] - h_begin[s0 + i]);
  const uint64_t total = vs[ns];
  if (total == 0) return HS_OK;
  for (uint64_t v0 = 0; v0 < total; v0 += kLaunchBytes) {
    const uint64_t v1 = std::min(total, v0 + kLaunchBytes);
    const bool last = v1 == total;
    SegParams sp;
    sp.nseg = 0;
    for (auto& w : sp.open_mask) w = 0;
    sp.acc_base = -1;
    sp.merge = merge;
    sp.merge_final = merge && final_group && last;
    for (int i = 0; i < ns; ++i) {
      // a non-empty segment joins every launch it intersects; an empty one the launch
      // holding its position (the last launch for positions at the very end)
      const bool empty = vs[i + 1] == vs[i];
      const bool in = empty ? (vs[i] >= v0 && (vs[i] < v1 || last)) : (vs[i] < v1 && vs[i + 1] > v0);
      if (!in) continue;
      if (sp.acc_base < 0) sp.acc_base = i;  // members are consecutive indices
      const uint64_t a = std::max(vs[i], v0), b = std::min(vs[i + 1], v1);
      const int k = sp.nseg++;
      sp.begin[k] = h_begin[s0 + i] + (empty ? 0 : a - vs[i]);
      sp.vstart[k] = (empty ? std::min(vs[i], v1) : a) - v0;
      sp.vstart[k + 1] = (empty ? std::min(vs[i], v1) : b) - v0;
      if (vs[i + 1] > v1) sp.open_mask[k >> 5] |= 1u << (k & 31);
    }
    sp.out_base = s0 + sp.acc_base;
    if (merge) sp.out_base = sp.acc_base = 0;  // one row for the whole call
    int rc = launch_batch(d_data, sp, kind, impl, pp, d_out, st, di, tk, reserve_slots, latency, wait_first);
    if (rc != HS_OK) return rc;
    wait_first = false;  // the rest of the call chains behind our own launches
  }
  return HS_OK;
}


}  // namespace

// ================================================================== C ABI
extern "C" {

int hs_abi_version(void) { return HS_ABI_VERSION; }

const char* hs_strerror(int status) {
  switch (status) {
    case HS_OK: return "ok";
    case HS_ERR_INVALID_ARG: return "invalid argument";
    case HS_ERR_PATTERN_SHAPE: return "pattern arrays must have 256 entries";
    case HS_ERR_PATTERN_COUNT_LOW: return "count below 1";
    case HS_ERR_PATTERN_COUNT_HIGH: return "count above cap";
    case HS_ERR_PATTERN_TOTAL: return "slot total mismatch";
    case HS_ERR_PATTERN_OFFSETS: return "offsets not contiguous";
    case HS_ERR_SLOT_RANGE: return "total_slots outside [256, 256 * cap]";
    case HS_ERR_WORKSPACE: return "workspace too small";
    case HS_ERR_UNSUPPORTED: return "configuration not supported on this device";
    case HS_ERR_ALIGNMENT: return "segment bounds must be multiples of 4 bytes";
    case HS_ERR_NO_DEVICE: return "no CUDA device";
    default: break;
  }
  if (status <= HS_ERR_CUDA_BASE) return cudaGetErrorString(cudaError_t(HS_ERR_CUDA_BASE - status));
  return "unknown status";
}

int hs_device_query(int device, int* sm_count, int* smem_optin, int* l2_bytes) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) return HS_ERR_NO_DEVICE;
  if (device < 0 || device >= n) return HS_ERR_INVALID_ARG;
  if (sm_count && (e = cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, device)) != cudaSuccess) return fold(e);
  if (smem_optin && (e = cudaDeviceGetAttribute(smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device)) != cudaSuccess) return fold(e);
  if (l2_bytes && (e = cudaDeviceGetAttribute(l2_bytes, cudaDevAttrL2CacheSize, device)) != cudaSuccess) return fold(e);
  return HS_OK;
}

int hs_validate_pattern(const int64_t* h_offset, const int64_t* h_count, int64_t total_slots, int64_t cap) {
  return validate(h_offset, h_count, total_slots, cap);
}

// [header: call counter, drained[K], finalized[K]] then K call slots of [tickets: kMaxSeg
// u32 = 1 KB][accumulators: one 256 x u64 row per segment of a launch]; zero it once
// after allocating -- every call leaves its slot's tickets and rows zero again (the
// header's counters advance). A workspace sized for n segments lets launches take up to
// n (<= kMaxSeg) segments.
constexpr size_t slot_bytes_for(int nseg) { return kTicketBytes + size_t(nseg) * 256 * sizeof(uint64_t); }
constexpr size_t ws_bytes_for(int nseg) { return kWsHeadBytes + (kCallSlots + 1) * slot_bytes_for(nseg); }
constexpr size_t kWorkspaceBytes = ws_bytes_for(kMaxSegEngine);  // the minimum accepted
size_t hs_workspace_bytes(int nseg) {
  return nseg < 0 ? 0 : ws_bytes_for(std::max(kMaxSegEngine, std::min(nseg, kMaxSeg)));
}

}  // extern "C"

namespace {
// Ticket view of a caller workspace of ws_bytes (rows per slot: the launch group size)
Tickets tickets_of(void* d_ws, size_t ws_bytes, int& rows) {
  Tickets tk{};
  const size_t per = (ws_bytes - kWsHeadBytes) / (kCallSlots + 1);
  rows = int(std::min<size_t>(kMaxSeg, (per - kTicketBytes) / (256 * sizeof(uint64_t))));
  tk.hdr = reinterpret_cast<WsHeader*>(d_ws);
  tk.slots = reinterpret_cast<uint8_t*>(d_ws) + kWsHeadBytes;
  tk.slot_bytes = uint32_t(slot_bytes_for(rows));
  tk.rotate = 0;
  tk.nfinal = 0;
  return tk;
}

// A call over segments [s0, s0 + ns) of `total` bytes takes a rotating slot when it is one
// launch of at most kRotateMaxBytes (see WsHeader); it then needs its finalization count.
#ifndef HS_ROTATE_MAX_MIB
#define HS_ROTATE_MAX_MIB 16
#endif
constexpr uint64_t kRotateMaxBytes = uint64_t(HS_ROTATE_MAX_MIB) << 20;
void plan_call(Tickets& tk, const uint64_t* h_begin, const uint64_t* h_end, int s0, int ns, bool merge) {
  if (tk.hdr == nullptr) return;
  uint64_t total = 0;
  uint32_t n = 0;
  for (int i = s0; i < s0 + ns; ++i) {
    total += h_end[i] - h_begin[i];
    n += h_end[i] > h_begin[i];
  }
  tk.rotate = total > 0 && total <= kRotateMaxBytes;
  tk.nfinal = merge ? 1 : n;
}

int histogram_batched(const uint8_t* d_data, const uint64_t* h_begin, const uint64_t* h_end, int nseg, int kind,
                      int impl, const int64_t* h_offset, const int64_t* h_count, int64_t total_slots, int64_t cap,
                      uint64_t* d_out, void* d_ws, size_t ws_bytes, void* stream, bool latency) {
  if (nseg < 0 || (nseg > 0 && (!h_begin || !h_end || !d_out))) return HS_ERR_INVALID_ARG;
  const bool spread = (kind & HS_KIND_FLAG_SPREAD) != 0;
  bool wait_first = (kind & HS_KIND_FLAG_CHAINED) == 0;
  const bool merge = (kind & HS_KIND_FLAG_MERGE) != 0;
  kind &= ~(HS_KIND_FLAG_SPREAD | HS_KIND_FLAG_CHAINED | HS_KIND_FLAG_MERGE);
  if (kind != HS_KIND_NAIVE && kind != HS_KIND_ADAPTIVE) return HS_ERR_INVALID_ARG;
  if (impl < HS_IMPL_AUTO || impl > HS_IMPL_SUBBIN) return HS_ERR_INVALID_ARG;
  PatternParams pp;
  const bool have_pattern = h_offset && h_count;
  if (kind == HS_KIND_ADAPTIVE && !have_pattern) return HS_ERR_INVALID_ARG;
  if (impl == HS_IMPL_SUBBIN && !have_pattern) return HS_ERR_INVALID_ARG;
  if (have_pattern) {
    int rc = make_pattern(h_offset, h_count, total_slots, cap, pp, impl == HS_IMPL_SUBBIN);
    if (rc != HS_OK) return rc;
    if (spread) pp.hot_unique = 0;  // caller's hint: no dominant value in the prior
  }
  uint64_t total = 0;
  for (int s = 0; s < nseg; ++s) {
    if (h_end[s] < h_begin[s]) return HS_ERR_INVALID_ARG;
    if ((h_begin[s] & 3) || (h_end[s] & 3)) return HS_ERR_ALIGNMENT;
    total += h_end[s] - h_begin[s];
  }
  if (total > 0 && !d_data) return HS_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(d_data) & 3) return HS_ERR_ALIGNMENT;
  if (nseg == 0) return HS_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  DevInfo di;
  int rc = dev_info(di);
  if (rc != HS_OK) return rc;
  if (impl == HS_IMPL_AUTO) impl = HS_IMPL_LANE;
  // LANE with a workspace: one launch per group of segments the workspace has rows for
  // (<= kMaxSeg), output written in-kernel; otherwise memset + RED, kMaxSeg per launch
  Tickets tk{};
  int group = kMaxSeg;
  if (impl == HS_IMPL_LANE && d_ws != nullptr && ws_bytes >= kWorkspaceBytes && total > 0) {
    if (reinterpret_cast<uintptr_t>(d_ws) & 15) return HS_ERR_ALIGNMENT;
    tk = tickets_of(d_ws, ws_bytes, group);
    if (merge) group = kMaxSeg;  // one accumulator row whatever the segment count
    // a merged call over several groups finalizes once, in its last group: serial. So
    // are the blocking entries (latency): the host waits for each call, so there is no
    // next call to overlap and the arrival would only add its round trip.
    if (merge && nseg <= group && !latency && !wait_first) plan_call(tk, h_begin, h_end, 0, nseg, true);
  } else {
    cudaError_t e = cudaMemsetAsync(d_out, 0, size_t(merge ? 1 : nseg) * 256 * sizeof(uint64_t), st);
    if (e != cudaSuccess) return fold(e);
  }
  if (total == 0) {
    if (merge && tk.hdr != nullptr) return fold(cudaMemsetAsync(d_out, 0, 256 * sizeof(uint64_t), st));
    return HS_OK;
  }
  // merged calls: the last group holding bytes finalizes the row
  int last_busy = 0;
  for (int s = 0; s < nseg; ++s) if (h_end[s] > h_begin[s]) last_busy = s;
  for (int s0 = 0; s0 < nseg; s0 += group) {
    const int ns = std::min(group, nseg - s0);
    bool empty = true;
    for (int i = 0; i < ns; ++i) empty = empty && h_end[s0 + i] == h_begin[s0 + i];
    if (empty && merge) continue;
    if (empty && tk.hdr != nullptr) {
      cudaError_t e = cudaMemsetAsync(d_out + size_t(s0) * 256, 0, size_t(ns) * 256 * sizeof(uint64_t), st);
      if (e != cudaSuccess) return fold(e);
      continue;
    }
    // each group is a call of its own. A call that waits for its predecessor before
    // loading (the default) gains nothing from a rotating slot -- the predecessor is
    // complete before any of its CTAs counts -- and would only add the arrival's round
    // trip, so it keeps the serial slot, as the blocking entries do.
    if (!merge && !latency && !wait_first) plan_call(tk, h_begin, h_end, s0, ns, false);
    rc = launch_segments(d_data, h_begin, h_end, s0, ns, kind, impl, have_pattern ? &pp : nullptr,
                         reinterpret_cast<unsigned long long*>(d_out), st, di, tk, 0, latency, wait_first, merge,
                         last_busy < s0 + ns);
    if (rc != HS_OK) return rc;
  }
  return HS_OK;
}
}  // namespace

extern "C" {

int hs_histogram_batched(const uint8_t* d_data, const uint64_t* h_begin, const uint64_t* h_end, int nseg,
                         int kind, int impl, const int64_t* h_offset, const int64_t* h_count,
                         int64_t total_slots, int64_t cap, uint64_t* d_out, void* d_ws, size_t ws_bytes,
                         void* stream) {
  return histogram_batched(d_data, h_begin, h_end, nseg, kind, impl, h_offset, h_count, total_slots, cap, d_out,
                           d_ws, ws_bytes, stream, false);
}

}  // extern "C"

namespace {
// Device view of a page-locked h_out, or nullptr. The blocking entries let the kernel
// write the counts straight into page-locked host memory (one PCIe write of 2 KiB per
// segment from the segment's last CTA) instead of a D2H copy after it: only on the
// ticketed path, whose output is plain stores (the memset + RED path would put
// atomics on host memory).
uint64_t* mapped_host_out(uint64_t* h_out, int impl, void* d_ws, size_t ws_bytes) {
#ifndef HS_NO_DIRECT_HOST_OUT
  if ((impl != HS_IMPL_AUTO && impl != HS_IMPL_LANE) || !d_ws || ws_bytes < kWorkspaceBytes) return nullptr;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, h_out) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (a.type != cudaMemoryTypeHost || a.devicePointer == nullptr) return nullptr;
  return reinterpret_cast<uint64_t*>(a.devicePointer);
#else
  (void)h_out; (void)impl; (void)d_ws; (void)ws_bytes;
  return nullptr;
#endif
}
}  // namespace

extern "C" {

int hs_histogram_sync(const uint8_t* d_data, const uint64_t* h_begin, const uint64_t* h_end, int nseg,
                      int kind, int impl, const int64_t* h_offset, const int64_t* h_count,
                      int64_t total_slots, int64_t cap, uint64_t* d_out, uint64_t* h_out,
                      void* d_ws, size_t ws_bytes, void* stream) {
  if (nseg > 0 && !h_out) return HS_ERR_INVALID_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (uint64_t* m = nseg > 0 ? mapped_host_out(h_out, impl, d_ws, ws_bytes) : nullptr) {
    int rc = histogram_batched(d_data, h_begin, h_end, nseg, kind, impl, h_offset, h_count, total_slots, cap, m,
                               d_ws, ws_bytes, stream, true);
    return rc != HS_OK ? rc : fold(cudaStreamSynchronize(st));
  }
  int rc = histogram_batched(d_data, h_begin, h_end, nseg, kind, impl, h_offset, h_count, total_slots, cap, d_out,
                             d_ws, ws_bytes, stream, true);
  if (rc != HS_OK || nseg == 0) return rc;
  const size_t rows = (kind & HS_KIND_FLAG_MERGE) ? 1 : size_t(nseg);
  cudaError_t e = cudaMemcpyAsync(h_out, d_out, rows * 256 * sizeof(uint64_t), cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return fold(e);
  return fold(cudaStreamSynchronize(st));
}

int hs_histogram_host(const uint8_t* const* h_chunks, const uint64_t* h_sizes, int nseg, int kind, int impl,
                      const int64_t* h_offset, const int64_t* h_count, int64_t total_slots, int64_t cap,
                      uint8_t* d_stage, size_t stage_bytes, uint64_t* d_out, uint64_t* h_out,
                      void* d_ws, size_t ws_bytes, void* stream) {
  if (nseg < 0 || (nseg > 0 && (!h_chunks || !h_sizes || !d_out || !h_out))) return HS_ERR_INVALID_ARG;
  if (nseg == 0) return HS_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  std::vector<uint64_t> begin(nseg), end(nseg);
  uint64_t off = 0;
  for (int s = 0; s < nseg; ++s) {
    if (h_sizes[s] & 3) return HS_ERR_ALIGNMENT;
    begin[s] = off;
    end[s] = off + h_sizes[s];
    off += (h_sizes[s] + 15) & ~uint64_t(15);
  }
  if (off > 0 && (!d_stage || stage_bytes < off)) return HS_ERR_WORKSPACE;
  for (int s = 0; s < nseg; ++s) {
    if (h_sizes[s] == 0) continue;
    if (!h_chunks[s]) return HS_ERR_INVALID_ARG;
    cudaError_t e = cudaMemcpyAsync(d_stage + begin[s], h_chunks[s], h_sizes[s], cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return fold(e);
  }
  if (uint64_t* m = mapped_host_out(h_out, impl, d_ws, ws_bytes)) {
    int rc = histogram_batched(d_stage, begin.data(), end.data(), nseg, kind, impl, h_offset, h_count,
                               total_slots, cap, m, d_ws, ws_bytes, stream, true);
    return rc != HS_OK ? rc : fold(cudaStreamSynchronize(st));
  }
  int rc = histogram_batched(d_stage, begin.data(), end.data(), nseg, kind, impl, h_offset, h_count, total_slots,
                             cap, d_out, d_ws, ws_bytes, stream, true);
  if (rc != HS_OK) return rc;
  const size_t rows = (kind & HS_KIND_FLAG_MERGE) ? 1 : size_t(nseg);
  cudaError_t e = cudaMemcpyAsync(h_out, d_out, rows * 256 * sizeof(uint64_t), cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return fold(e);
  return fold(cudaStreamSynchronize(st));
}

int hs_histogram(const uint8_t* d_data, uint64_t n_bytes, int kind, int impl, const int64_t* h_offset,
                 const int64_t* h_count, int64_t total_slots, int64_t cap, uint64_t* d_out, void* d_ws,
                 size_t ws_bytes, void* stream) {
  const uint64_t b = 0, e = n_bytes;
  return hs_histogram_batched(d_data, &b, &e, 1, kind, impl, h_offset, h_count, total_slots, cap, d_out,
                              d_ws, ws_bytes, stream);
}

size_t hs_group_slots_ws_bytes(int group_size, int group_count, int64_t total_slots, int mode) {
  if (group_size < 1 || group_count < 1 || total_slots < 1 || mode < 0 || mode > 2) return 0;
  // mode 2 only: exact totals in u64 before the 16-bit wrap
  return mode == 2 ? size_t(group_count) * size_t(total_slots) * sizeof(uint64_t) : 0;
}

int hs_group_slots(const uint8_t* d_data, uint64_t n_bytes, int group_size, int group_count,
                   const int64_t* h_offset, const int64_t* h_count, int64_t total_slots, int64_t cap,
                   int mode, void* d_out, void* d_ws, size_t ws_bytes, void* stream) {
  if (group_size < 1 || group_count < 1 || mode < 0 || mode > 2 || !d_out) return HS_ERR_INVALID_ARG;
  if (n_bytes & 3) return HS_ERR_ALIGNMENT;
  if (n_bytes && !d_data) return HS_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(d_data) & 3) return HS_ERR_ALIGNMENT;
  PatternParams pp;
  int rc = make_pattern(h_offset, h_count, total_slots, cap, pp);
  if (rc != HS_OK) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const uint64_t S = uint64_t(total_slots);
  const uint64_t n_out = mode == 1 ? uint64_t(group_count) * group_size * S : uint64_t(group_count) * S;
  unsigned long long* acc = nullptr;
  cudaError_t e;
  if (mode == 2) {
    // exact 64-bit totals in the caller's workspace, then wrapped to 16 bits
    if (!d_ws || ws_bytes < n_out * 8) return HS_ERR_WORKSPACE;
    acc = reinterpret_cast<unsigned long long*>(d_ws);
  } else {
    acc = reinterpret_cast<unsigned long long*>(d_out);
  }
  e = cudaMemsetAsync(acc, 0, n_out * 8, st);
  if (e != cudaSuccess) return fold(e);
  const uint64_t nw = n_bytes / 4;
  if (nw) {
    const int grid = int(std::min<uint64_t>((nw + 255) / 256, 4096));
    k_group_slots<<<grid, 256, 0, st>>>(reinterpret_cast<const uint32_t*>(d_data), nw, group_size, group_count,
                                        pp, mode == 1 ? 1 : 0, acc);
    if ((e = cudaGetLastError()) != cudaSuccess) return fold(e);
  }
  if (mode == 2) {
    const int grid = int(std::min<uint64_t>((n_out + 255) / 256, 4096));
    k_wrap16<<<grid, 256, 0, st>>>(acc, reinterpret_cast<uint16_t*>(d_out), n_out);
    if ((e = cudaGetLastError()) != cudaSuccess) return fold(e);
  }
  return HS_OK;
}

int hs_ablation_stage(const uint8_t* d_data, uint64_t n_bytes, int stage, const int64_t* h_offset,
                      const int64_t* h_count, int64_t total_slots, int64_t cap, uint64_t* d_sink,
                      uint64_t* d_out256, void* d_ws, size_t ws_bytes, void* stream) {
  (void)d_ws; (void)ws_bytes;
  if (stage < HS_STAGE_COPY_ONLY || stage > HS_STAGE_FULL || !d_sink) return HS_ERR_INVALID_ARG;
  if (stage == HS_STAGE_FULL && !d_out256) return HS_ERR_INVALID_ARG;
  if ((n_bytes & 3) || (reinterpret_cast<uintptr_t>(d_data) & 3)) return HS_ERR_ALIGNMENT;
  PatternParams pp;
  int rc = make_pattern(h_offset, h_count, total_slots, cap, pp);
  if (rc != HS_OK) return rc;
  DevInfo di;
  if ((rc = dev_info(di)) != HS_OK) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(d_sink, 0, 8, st);
  if (e != cudaSuccess) return fold(e);
  if (d_out256 && (e = cudaMemsetAsync(d_out256, 0, 2048, st)) != cudaSuccess) return fold(e);
  if (n_bytes == 0) return HS_OK;
  // shared memory only from the stage that uses it (none for the copy baseline)
  const size_t smem = stage == HS_STAGE_COPY_ONLY ? 0 : stage == HS_STAGE_COPY_INIT ? kLaneArrayBytes
                                                                                     : 2 * size_t(kLaneArrayBytes);
  const int grid = int(std::max<uint64_t>(1, std::min<uint64_t>(lane_grid_for(n_bytes), uint64_t(di.sms) * kLaneBlocks)));
  const uint64_t units = ((n_bytes >> 2) + kSplitWords - 1) / kSplitWords;
  const uint64_t q = units / uint64_t(grid), r = units % uint64_t(grid);
  auto* sk = reinterpret_cast<unsigned long long*>(d_sink);
  auto* ot = reinterpret_cast<unsigned long long*>(d_out256);
  static std::atomic<uint64_t> set2{0}, set3{0}, set4{0};
  switch (stage) {
    case HS_STAGE_COPY_ONLY:
      k_genealogy<HS_STAGE_COPY_ONLY><<<grid, kLaneThreads, 0, st>>>(d_data, n_bytes, q, r, pp, sk, ot);
      break;
    case HS_STAGE_COPY_INIT:
      k_genealogy<HS_STAGE_COPY_INIT><<<grid, kLaneThreads, smem, st>>>(d_data, n_bytes, q, r, pp, sk, ot);
      break;
    case HS_STAGE_PATTERN_LOAD:
      if ((rc = set_smem_once(k_genealogy<HS_STAGE_PATTERN_LOAD>, smem, set2)) != HS_OK) return rc;
      k_genealogy<HS_STAGE_PATTERN_LOAD><<<grid, kLaneThreads, smem, st>>>(d_data, n_bytes, q, r, pp, sk, ot);
      break;
    case HS_STAGE_SUBHIST_NOREDUCE:
      if ((rc = set_smem_once(k_genealogy<HS_STAGE_SUBHIST_NOREDUCE>, smem, set3)) != HS_OK) return rc;
      k_genealogy<HS_STAGE_SUBHIST_NOREDUCE><<<grid, kLaneThreads, smem, st>>>(d_data, n_bytes, q, r, pp, sk, ot);
      break;
    default:
      if ((rc = set_smem_once(k_genealogy<HS_STAGE_FULL>, smem, set4)) != HS_OK) return rc;
      k_genealogy<HS_STAGE_FULL><<<grid, kLaneThreads, smem, st>>>(d_data, n_bytes, q, r, pp, sk, ot);
      break;
  }
  return fold(cudaGetLastError());
}

size_t hs_stream_state_bytes(int window_size) {
  if (window_size < 1) return 0;
  return sizeof(DevStreamHeader) + size_t(2 + window_size) * 256 * sizeof(uint64_t);
}

int hs_stream_reset(void* d_state, int window_size, void* stream) {
  if (!d_state || window_size < 1) return HS_ERR_INVALID_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (reinterpret_cast<uintptr_t>(d_state) & 15) return HS_ERR_ALIGNMENT;
  // zero state (kind NAIVE, hot 0, empty window) + the device clock at reset
  k_stream_reset<<<16, 256, 0, st>>>(reinterpret_cast<unsigned long long*>(d_state),
                                     hs_stream_state_bytes(window_size) / 8);
  return fold(cudaGetLastError());
}

int hs_stream_step(const uint8_t* d_data, const uint64_t* h_begin, const uint64_t* h_end, int nseg,
                   void* d_state, int window_size, double threshold, int recompute_every, int iteration,
                   uint64_t* d_out, double* d_deg_log, double* d_div_log, int32_t* d_kind_log,
                   uint64_t* d_ns_log, void* d_ws, size_t ws_bytes, void* stream) {
  if (!d_state || window_size < 1 || nseg < 1 || nseg > kMaxSegEngine || recompute_every < 1 || iteration < 0 ||
      !d_out || !d_deg_log || !d_div_log || !d_kind_log || !h_begin || !h_end)
    return HS_ERR_INVALID_ARG;
  if (!(threshold > 0.0 && threshold < 1.0)) return HS_ERR_INVALID_ARG;
  if (!d_ws || ws_bytes < kWorkspaceBytes) return HS_ERR_WORKSPACE;
  uint64_t total = 0;
  for (int s = 0; s < nseg; ++s) {
    if (h_end[s] < h_begin[s]) return HS_ERR_INVALID_ARG;
    if ((h_begin[s] & 3) || (h_end[s] & 3)) return HS_ERR_ALIGNMENT;
    total += h_end[s] - h_begin[s];
  }
  if (reinterpret_cast<uintptr_t>(d_data) & 3) return HS_ERR_ALIGNMENT;
  // the fold moves the chunk histograms and the ring with 16-B loads
  if ((reinterpret_cast<uintptr_t>(d_out) | reinterpret_cast<uintptr_t>(d_state)) & 15) return HS_ERR_ALIGNMENT;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  DevInfo di;
  int rc = dev_info(di);
  if (rc != HS_OK) return rc;
  if (reinterpret_cast<uintptr_t>(d_ws) & 15) return HS_ERR_ALIGNMENT;
  int rows = 0;
  Tickets tk = tickets_of(d_ws, ws_bytes, rows);
  plan_call(tk, h_begin, h_end, 0, nseg, false);
  tk.rotate = tk.nfinal > 0 && total <= kLaunchBytes;  // followed by the fold, as hs_stream_block
  bool empty = total == 0;
  if (empty) {
    cudaError_t e = cudaMemsetAsync(d_out, 0, size_t(nseg) * 256 * sizeof(uint64_t), st);
    if (e != cudaSuccess) return fold(e);
  } else {
    // The histogram does not wait for the previous fold's decision: both kinds count
    // exactly the same, so the lane kernel runs for either and streams while the fold
    // (one CTA) finishes on the side; the decided kind is what the log records.
    // chained: the step's stream predecessor is the previous step's fold or
    // hs_stream_reset (the batch must be complete before that was issued; see hist256.h)
    bool wait_first = false;
    rc = launch_segments(d_data, h_begin, h_end, 0, nseg, HS_KIND_NAIVE, HS_IMPL_LANE, nullptr,
                         reinterpret_cast<unsigned long long*>(d_out), st, di, tk, /*reserve_slots=*/1, false,
                         wait_first);
    if (rc != HS_OK) return rc;
  }
  // pattern and kernel refresh for iteration+1 when (iteration+1) % every == 0 (stream.py:407-414)
  const int decide = ((iteration + 1) % recompute_every) == 0;
  static std::atomic<uint64_t> fold_smem_set{0};
  if ((rc = set_smem_once(k_stream_fold, kFoldSmem, fold_smem_set)) != HS_OK) return rc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(kFoldThreads);
  cfg.dynamicSmemBytes = size_t(nseg) * 256 * 8 + (window_size < kFoldSmallWin ? size_t(window_size) * 256 * 8 : 0);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_stream_fold, reinterpret_cast<const unsigned long long*>(d_out), nseg,
                                     reinterpret_cast<uint8_t*>(d_state), window_size, threshold, decide, iteration,
                                     d_deg_log, d_div_log, d_kind_log,
                                     reinterpret_cast<unsigned long long*>(d_ns_log));
  if (e != cudaSuccess) return fold(e);
  return fold(cudaGetLastError());
}

// workspace of hs_stream_block: [scan ticket][argmax u32 x kBlockMaxIter][histogram
// tickets + rows (hs_workspace_bytes(256))][local prefix (W + max_chunks) x 256 u64]
// [tile totals -> their exclusive prefix]; zeroed once, every block leaves its tickets zero
constexpr size_t kBlockHead = 16 + kBlockMaxIter * 4;  // scan ticket (16 B), argmax u32 per iteration
size_t hs_stream_block_ws_bytes(int window_size, int max_chunks) {
  if (window_size < 1 || max_chunks < 1 || max_chunks > kBlockMaxChunks) return 0;
  const size_t rows = size_t(window_size) + size_t(max_chunks);
  const size_t tiles = (rows + kScanTile - 1) / kScanTile;
  return kBlockHead + ws_bytes_for(kMaxSeg) + rows * 256 * 8 + tiles * 256 * 8;
}

int hs_stream_block(const uint8_t* d_data, const uint64_t* h_begin, const uint64_t* h_end, int nseg,
                    const int32_t* h_iter_chunks, int n_iter, void* d_state, int window_size, double threshold,
                    int recompute_every, int first_iteration, int hot_bin, uint64_t* d_out, double* d_deg_log,
                    double* d_div_log, int32_t* d_kind_log, uint64_t* d_ns_log, uint64_t* h_decision,
                    void* d_ws, size_t ws_bytes, void* stream) {
  if (!d_state || window_size < 1 || nseg < 1 || nseg > kBlockMaxChunks || n_iter < 1 || n_iter > kBlockMaxIter ||
      recompute_every < 1 || first_iteration < 0 || !d_out || !d_deg_log || !d_div_log || !d_kind_log || !h_begin ||
      !h_end || !h_iter_chunks || hot_bin > 255)
    return HS_ERR_INVALID_ARG;
  if (!(threshold > 0.0 && threshold < 1.0)) return HS_ERR_INVALID_ARG;
  const size_t need = hs_stream_block_ws_bytes(window_size, nseg);
  if (!d_ws || ws_bytes < need) return HS_ERR_WORKSPACE;
  BlockMap bm;
  bm.n_iter = n_iter;
  bm.m = nseg;
  bm.c0_unused = 0;
  bm.first_iteration = first_iteration;
  int c = 0;
  for (int i = 0; i < n_iter; ++i) {
    if (h_iter_chunks[i] < 0) return HS_ERR_INVALID_ARG;
    c += h_iter_chunks[i];
    bm.end_chunk[i] = c;
  }
  if (c != nseg) return HS_ERR_INVALID_ARG;
  uint64_t total = 0;
  for (int s = 0; s < nseg; ++s) {
    if (h_end[s] < h_begin[s]) return HS_ERR_INVALID_ARG;
    if ((h_begin[s] & 3) || (h_end[s] & 3)) return HS_ERR_ALIGNMENT;
    total += h_end[s] - h_begin[s];
  }
  if (reinterpret_cast<uintptr_t>(d_data) & 3) return HS_ERR_ALIGNMENT;
  if ((reinterpret_cast<uintptr_t>(d_out) | reinterpret_cast<uintptr_t>(d_state) |
       reinterpret_cast<uintptr_t>(d_ws)) & 15)
    return HS_ERR_ALIGNMENT;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  DevInfo di;
  int rc = dev_info(di);
  if (rc != HS_OK) return rc;
  unsigned long long* dec = nullptr;
  if (h_decision) {  // page-locked host memory, written by the commit kernel
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, h_decision) != cudaSuccess || a.type != cudaMemoryTypeHost ||
        a.devicePointer == nullptr) {
      cudaGetLastError();
      return HS_ERR_INVALID_ARG;
    }
    dec = reinterpret_cast<unsigned long long*>(a.devicePointer);
  }
  uint8_t* ws = reinterpret_cast<uint8_t*>(d_ws);
  unsigned int* scan_ticket = reinterpret_cast<unsigned int*>(ws);
  uint32_t* argmax = reinterpret_cast<uint32_t*>(ws + 16);
  uint8_t* hist_ws = ws + kBlockHead;
  const size_t rows = size_t(window_size) + size_t(nseg);
  unsigned long long* local = reinterpret_cast<unsigned long long*>(hist_ws + ws_bytes_for(kMaxSeg));
  unsigned long long* tile_tot = local + rows * 256;
  if (total == 0) {
    cudaError_t e = cudaMemsetAsync(d_out, 0, size_t(nseg) * 256 * sizeof(uint64_t), st);
    if (e != cudaSuccess) return fold(e);
  } else {
    // One histogram call for the whole block, chained behind the previous block's commit
    // (input contract as hs_stream_step). hot_bin >= 0: the register path for that bin
    // (the host's lagged view of the device's ADAPTIVE decision); counts are identical.
    int rows = 0;
    Tickets tk = tickets_of(hist_ws, ws_bytes_for(kMaxSeg), rows);
    plan_call(tk, h_begin, h_end, 0, nseg, false);
    // Every single-launch block rotates, whatever its size: the histogram's successor
    // here is the fold chain, not another histogram, and in the serial slot each of its
    // CTAs would wait at its flush for the previous block's commit (and so for that
    // block's whole fold). 1 MiB batch-1 iterations, 256 MiB blocks, host ahead:
    // 2.55 -> 2.85-2.95 TB/s (tools/diag/c3_only.py).
    tk.rotate = tk.nfinal > 0 && total <= kLaunchBytes;
    PatternParams pp{};
    pp.hot_bin = hot_bin >= 0 ? hot_bin : 0;
    pp.hot_unique = hot_bin >= 0;
    pp.total_slots = 256;
    bool wait_first = false;
    rc = launch_segments(d_data, h_begin, h_end, 0, nseg, hot_bin >= 0 ? HS_KIND_ADAPTIVE : HS_KIND_NAIVE,
                         HS_IMPL_LANE, &pp, reinterpret_cast<unsigned long long*>(d_out), st, di, tk, 0, false,
                         wait_first);
    if (rc != HS_OK) return rc;
  }
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const auto* hist = reinterpret_cast<const unsigned long long*>(d_out);
  cfg.gridDim = dim3(unsigned((rows + kScanTile - 1) / kScanTile));
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_block_scan, hist, nseg, reinterpret_cast<const uint8_t*>(d_state),
                                     window_size, local, tile_tot, scan_ticket);
  if (e != cudaSuccess) return fold(e);
  cfg.gridDim = dim3(unsigned(n_iter));
  e = cudaLaunchKernelEx(&cfg, k_block_fold, bm, reinterpret_cast<uint8_t*>(d_state), window_size,
                         (const unsigned long long*)local, (const unsigned long long*)tile_tot, d_deg_log, d_div_log,
                         argmax);
  if (e != cudaSuccess) return fold(e);
  cfg.gridDim = dim3(1);
  e = cudaLaunchKernelEx(&cfg, k_block_commit, bm, hist, reinterpret_cast<uint8_t*>(d_state), window_size, threshold,
                         recompute_every, (const unsigned long long*)local, (const unsigned long long*)tile_tot,
                         (const double*)d_deg_log, (const uint32_t*)argmax, d_kind_log,
                         reinterpret_cast<unsigned long long*>(d_ns_log), dec);
  if (e != cudaSuccess) return fold(e);
  return fold(cudaGetLastError());
}

int hs_generate_device(int kind, uint64_t seed, int value, double mean, double sigma, uint64_t first,
                       uint8_t* d_out, uint64_t n, void* stream) {
  if (n == 0) return HS_OK;
  if (!d_out) return HS_ERR_INVALID_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  DevInfo di;
  int rc = dev_info(di);
  if (rc != HS_OK) return rc;
  const int grid = di.sms * 8;
  switch (kind) {
    case HS_GEN_UNIFORM: k_gen_uniform<<<grid, 256, 0, st>>>(seed, first, d_out, n); break;
    case HS_GEN_SEQUENTIAL: k_gen_sequential<<<grid, 256, 0, st>>>(first, d_out, n); break;
    case HS_GEN_CONSTANT:
      if (value < 0 || value > 255) return HS_ERR_INVALID_ARG;
      return fold(cudaMemsetAsync(d_out, value, n, st));
    case HS_GEN_NORMAL:
      if (!(sigma > 0)) return HS_ERR_INVALID_ARG;
      k_gen_normal<<<grid, 256, 0, st>>>(seed, mean, sigma, first, d_out, n);
      break;
    default: return HS_ERR_INVALID_ARG;  // mixture consumes a data-dependent draw count: host only
  }
  return fold(cudaGetLastError());
}

}  // extern "C"

#ifdef HS_TRACE
extern "C" int hs_trace_read(void* host, size_t bytes) {
  if (bytes > sizeof(hs_trace_buf)) bytes = sizeof(hs_trace_buf);
  return cudaMemcpyFromSymbol(host, hs_trace_buf, bytes) == cudaSuccess ? 0 : -1;
}
extern "C" int hs_trace_clear() {
  void* p = nullptr;
  if (cudaGetSymbolAddress(&p, hs_trace_buf) != cudaSuccess) return -1;
  return cudaMemset(p, 0, sizeof(hs_trace_buf)) == cudaSuccess ? 0 : -1;
}
#endif
