/*
 * hist256.h — C ABI of libhist256.so, the B200 (sm_100a) 256-bin byte-histogram
 * engine behind the `paper_1011_0235_b200` drop-in for the reference package
 * `histostream` (arXiv 1011.0235, /root/reference/pkg/src/histostream).
 *
 * The reference has no FFI: its hot path is a pair of Numba workers that mutate a
 * caller-owned zeroed output in place (kernels.py:97-98, :133-134) and are driven
 * from Python threads. Each entry point below replaces one of those seams; the
 * Python host layer (paper_1011_0235_b200/kernels.py, stream.py) binds them with
 * ctypes exactly as INTEGRATION.md shows for a maintainer of the reference.
 *
 * Conventions
 *   - plain pointers and sizes only; `d_` = device pointer, `h_` = host pointer.
 *   - `stream` is a cudaStream_t passed as void* (0 = legacy default stream).
 *   - every call is asynchronous on `stream` unless its name ends in `_sync`,
 *     holds no global mutable state and never allocates device memory: callers
 *     own outputs and workspace (query sizes with hs_workspace_bytes).
 *   - return 0 (HS_OK) or a negative status; hs_strerror() names it. CUDA errors
 *     are folded in as HS_ERR_CUDA_BASE - cudaError_t.
 *   - histogram outputs are uint64[256] per histogram (core.py:70-94); pattern
 *     arrays are the reference's int64 offset/count[256] (pattern.py:42-67).
 */
#ifndef HIST256_H
#define HIST256_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HS_BINS 256
#define HS_ABI_VERSION 1

/* ---- status codes ------------------------------------------------------- */
#define HS_OK 0
#define HS_ERR_INVALID_ARG -1          /* null pointer, bad size, bad enum       */
#define HS_ERR_PATTERN_SHAPE -2        /* pattern.py:141-142 "256 entries"       */
#define HS_ERR_PATTERN_COUNT_LOW -3    /* pattern.py:143-144 "count below 1"     */
#define HS_ERR_PATTERN_COUNT_HIGH -4   /* pattern.py:145-146 "count above cap"   */
#define HS_ERR_PATTERN_TOTAL -5        /* pattern.py:147-148 "slot total mismatch" */
#define HS_ERR_PATTERN_OFFSETS -6      /* pattern.py:149-150 "offsets not contiguous" */
#define HS_ERR_SLOT_RANGE -7           /* pattern.py:70-76 SlotCountOutOfRange   */
#define HS_ERR_WORKSPACE -8            /* workspace smaller than hs_workspace_bytes */
#define HS_ERR_UNSUPPORTED -9          /* e.g. slot array larger than shared memory */
#define HS_ERR_ALIGNMENT -10           /* segment bounds not multiples of 4 bytes */
#define HS_ERR_NO_DEVICE -11
#define HS_ERR_CUDA_BASE -1000         /* HS_ERR_CUDA_BASE - (int)cudaError_t    */

/* ---- kernel kinds (kernels.py:42-52 KernelKind) ------------------------- */
#define HS_KIND_NAIVE 0      /* NVHist analogue, kernels.py:336-346 */
#define HS_KIND_ADAPTIVE 1   /* AHist analogue,  kernels.py:349-384 */
/* OR-ed into kind with HS_KIND_ADAPTIVE: the caller knows the pattern's prior is not
 * dominated by one value (max-bin share below ~0.999), so the register path for the hot
 * bin would not pay and the plain lane core runs. Counts are identical either way. */
#define HS_KIND_FLAG_SPREAD 0x100
/* OR-ed into kind: the caller guarantees that the kernel preceding this call on the
 * stream is a libhist256 launch (for instance the previous call over the same resident
 * input) and that the input was complete before that launch started (written before
 * a stream synchronisation, or before an earlier call that has completed). The call's
 * first launch may then start streaming before its predecessor finishes (programmatic
 * dependent launch). Without it the first launch waits for its predecessor -- complete
 * and its writes visible -- before its first load, so input written by ANY preceding
 * kernel, including producers that trigger their dependents early, is read complete.
 * With a workspace, a chained single-launch call of <= 16 MiB also takes the next
 * rotating workspace slot, so back-to-back small calls overlap (1 MiB: ~1.75 us each);
 * calls without the flag use the serial slot (~6.5 us each back to back at 1 MiB). */
#define HS_KIND_FLAG_CHAINED 0x200
/* OR-ed into kind: merge every segment into ONE histogram, d_out = uint64[256] = the
 * sum over all nseg segments (merge_all of the per-slice histograms, core.py:152-156),
 * formed in the kernel epilogue: CTAs do not flush at segment boundaries, and with a
 * workspace one ticket per CTA finalizes the row. A rank's partial for the multi-GPU
 * path (one call over its shard, then one allreduce of 256 counts). */
#define HS_KIND_FLAG_MERGE 0x400

/* ---- device strategies behind a kind --------------------- */
#define HS_IMPL_AUTO 0       /* library picks by kind and size                     */
#define HS_IMPL_LANE 1       /* lane-private u32 sub-histograms, bank == lane      */
#define HS_IMPL_WARP 2       /* per-warp shared u32[256] (paper/SDK NVHist)        */
#define HS_IMPL_SUBBIN 3     /* per-warp S-slot sub-bins, lane % count (paper AHist) */

/* ---- ablation stages (kernels.py:54-60 ABLATION_STAGES) ----------------- */
#define HS_STAGE_COPY_ONLY 0
#define HS_STAGE_COPY_INIT 1
#define HS_STAGE_PATTERN_LOAD 2
#define HS_STAGE_SUBHIST_NOREDUCE 3
#define HS_STAGE_FULL 4

int hs_abi_version(void);
const char* hs_strerror(int status);

/* Number of SMs, opt-in shared memory per block and L2 bytes of `device`. */
int hs_device_query(int device, int* sm_count, int* smem_optin, int* l2_bytes);

/* Pattern check in the reference's order (validate_pattern, pattern.py:136-149).
 * Returns HS_OK or the HS_ERR_PATTERN_* code of the first violated invariant. */
int hs_validate_pattern(const int64_t* h_offset, const int64_t* h_count,
                        int64_t total_slots, int64_t cap);

/* Device workspace of hs_histogram_batched / hs_stream_step: a HS_WS_HEAD_BYTES header
 * (a u64 call counter, u32 drained[HS_WS_SLOTS], u32 finalized[HS_WS_SLOTS]) and
 * HS_WS_SLOTS call slots, each 1 KB of tickets plus one 2 KB accumulator row per segment
 * of a launch, for launches of up to nseg segments (clamped to [64, 256]). Consecutive
 * calls count into consecutive slots, so only the CTAs that store a call's output wait
 * for the previous call on the stream. A workspace sized for n segments makes the call
 * launch groups of n segments; hs_stream_step needs at least hs_workspace_bytes(64).
 * Zero it once; calls leave every slot zero again and advance the header's counters.
 * 16-byte aligned. */
#define HS_WS_HEAD_BYTES 384
#define HS_WS_SLOTS 4
size_t hs_workspace_bytes(int nseg);

/*
 * Batched 256-bin histograms over `nseg` word-aligned byte ranges of one device
 * buffer: d_out[s*256 + b] = #{ i in [h_begin[s], h_end[s]) : d_data[i] == b }.
 * Replaces batch_histograms (stream.py:260-316), which drives _naive_worker
 * (kernels.py:97-130) / _adaptive_worker (kernels.py:133-168) per slice and
 * merges group partials (core.py:152-156). One launch for the whole batch.
 *   kind     HS_KIND_NAIVE or HS_KIND_ADAPTIVE (ADAPTIVE requires the pattern),
 *            optionally | HS_KIND_FLAG_SPREAD
 *   impl     HS_IMPL_* (HS_IMPL_AUTO for production)
 *   h_offset/h_count: the CPU binning pattern (pattern.py:94-133), may be NULL
 *            for NAIVE; validated before launch (kernels.py:363).
 *   d_out    uint64[nseg*256] (uint64[256] with HS_KIND_FLAG_MERGE), overwritten.
 *   d_ws     optional workspace of hs_workspace_bytes() bytes, zeroed once by the caller:
 *            the call is then ONE kernel launch per <= 256 segments and 1 GiB (CTAs RED into
 *            workspace rows; the last CTA per segment stores d_out and re-zeroes its row).
 *            Without it a memset of d_out precedes the launch. Calls sharing a workspace
 *            must be stream-ordered.
 * Byte offsets must be multiples of 4 (PackedChunk words, core.py:38-67).
 */
int hs_histogram_batched(const uint8_t* d_data, const uint64_t* h_begin, const uint64_t* h_end,
                         int nseg, int kind, int impl,
                         const int64_t* h_offset, const int64_t* h_count,
                         int64_t total_slots, int64_t cap,
                         uint64_t* d_out, void* d_ws, size_t ws_bytes, void* stream);

/* hs_histogram_batched, then the counts into h_out[nseg][256] and a wait for the stream:
 * the synchronous API path for device-resident chunks in one call. Blocking.
 * The launch grid is sized for latency (>= 16 KiB per CTA) rather than for
 * back-to-back throughput. When h_out is page-locked (cudaHostAlloc, torch
 * pin_memory, cudaHostRegister) and the call is ticketed (HS_IMPL_AUTO/LANE with
 * d_ws), each segment's last CTA writes its counts straight into h_out and d_out is
 * not written; otherwise the counts go to d_out and are copied to h_out. */
int hs_histogram_sync(const uint8_t* d_data, const uint64_t* h_begin, const uint64_t* h_end, int nseg,
                      int kind, int impl, const int64_t* h_offset, const int64_t* h_count,
                      int64_t total_slots, int64_t cap, uint64_t* d_out, uint64_t* h_out,
                      void* d_ws, size_t ws_bytes, void* stream);

/* Synchronous convenience for host-resident chunks (the one-call naive_histogram /
 * adaptive_histogram / batch_histograms path of the reference API, kernels.py:336-384,
 * stream.py:260-316): copies the nseg host chunks (h_chunks[s], h_sizes[s] bytes, any
 * host memory) into d_stage at 16-byte aligned offsets, runs hs_histogram_batched with
 * d_ws, copies d_out[nseg][256] into h_out and waits for the stream. Everything else as
 * hs_histogram_batched. d_stage must hold the chunks rounded up to 16 bytes each
 * (HS_ERR_WORKSPACE otherwise). One call instead of a copy, a launch and a readback
 * issued from Python: a 1 MiB image costs about half. Blocking. Grid and h_out as
 * hs_histogram_sync (a page-locked h_out is written by the kernel directly). */
int hs_histogram_host(const uint8_t* const* h_chunks, const uint64_t* h_sizes, int nseg, int kind, int impl,
                      const int64_t* h_offset, const int64_t* h_count, int64_t total_slots, int64_t cap,
                      uint8_t* d_stage, size_t stage_bytes, uint64_t* d_out, uint64_t* h_out,
                      void* d_ws, size_t ws_bytes, void* stream);

/* Single histogram: hs_histogram_batched with one segment [0, n_bytes).
 * Replaces naive_histogram (kernels.py:336-346) and adaptive_histogram
 * (kernels.py:349-384); `compute_histogram` (kernels.py:499-512) is the kind switch. */
int hs_histogram(const uint8_t* d_data, uint64_t n_bytes, int kind, int impl,
                 const int64_t* h_offset, const int64_t* h_count,
                 int64_t total_slots, int64_t cap,
                 uint64_t* d_out, void* d_ws, size_t ws_bytes, void* stream);

/*
 * Reference-mapping slot totals (compat path for return_slots / narrow_counters /
 * adaptive_lane_touches, kernels.py:349-407). Words are split with group_ranges
 * (kernels.py:311-316); word i of group g runs on lane (i - start_g) % group_size and
 * hits slot offset[b] + lane % count[b] (kernels.py:149-150).
 *   mode 0: d_out uint64[group_count][total_slots]          (slot_counts)
 *   mode 1: d_out uint64[group_count][group_size][total_slots] (lane_touch)
 *   mode 2: d_out uint16[group_count][total_slots], each slot wrapped mod 2^16
 *           (_adaptive_worker_u16, kernels.py:267-303)
 * d_out is overwritten. Mode 2 needs a device workspace of hs_group_slots_ws_bytes()
 * bytes (exact totals before the wrap; contents on entry do not matter); modes 0/1 need
 * none (d_ws may be NULL). Intended for test-scale inputs (global atomics). */
size_t hs_group_slots_ws_bytes(int group_size, int group_count, int64_t total_slots, int mode);
int hs_group_slots(const uint8_t* d_data, uint64_t n_bytes, int group_size, int group_count,
                   const int64_t* h_offset, const int64_t* h_count, int64_t total_slots,
                   int64_t cap, int mode, void* d_out, void* d_ws, size_t ws_bytes, void* stream);

/* Genealogy ablation stage (run_ablation, kernels.py:421-496) on the sub-bin kernel
 * skeleton. d_sink: uint64[1] checksum; d_out256 receives the histogram for
 * HS_STAGE_FULL (may be NULL otherwise). */
int hs_ablation_stage(const uint8_t* d_data, uint64_t n_bytes, int stage,
                      const int64_t* h_offset, const int64_t* h_count,
                      int64_t total_slots, int64_t cap,
                      uint64_t* d_sink, uint64_t* d_out256, void* d_ws, size_t ws_bytes,
                      void* stream);

/* ---- device-resident stream engine ----------------------------------------
 * The accumulator, moving window and NVHist/AHist switch of the stream driver
 * (stream.py:62-116, :390-425; policy.py:39-64) kept on the device, so lag-1 kernel
 * switching runs at device speed with no host round trip.
 * State is caller-allocated (hs_stream_state_bytes) and zeroed by hs_stream_reset,
 * which also stamps the device clock (%globaltimer, ns) at byte offset 32 + 8.
 * Error word: uint32 at byte offset 16 of the state, sticky, read once after the last
 * step -- bit 0 = window count went negative (stream.py NegativeCount), bit 1 = empty
 * histogram in divergence (policy.py EmptyHistogram). */
size_t hs_stream_state_bytes(int window_size);
int hs_stream_reset(void* d_state, int window_size, void* stream);

/* One iteration: histograms of the batch's nseg (<= 64) segments into d_out[nseg][256],
 * Input contract: the histogram launch is chained behind the previous step's fold (or
 * hs_stream_reset) with programmatic dependent launch and reads the batch before that
 * predecessor has finished, so the batch's bytes must be complete before the previous
 * step was issued (produced ahead, or ordered before the stream's previous step).
 * then the fold: acc += each chunk, window push/evict (error bit on NegativeCount),
 * d_kind_log[iteration] = kind the previous fold decided, d_deg_log[iteration] = window
 * degeneracy,
 * d_div_log[iteration] = total-variation(acc, window) in numpy's summation order, and
 * -- when (iteration+1) % recompute_every == 0 -- the decision for the next iteration:
 * ADAPTIVE iff degeneracy >= threshold (policy.py:49-53), hot bin = window argmax.
 * Both kinds count exactly alike on this device, so the histogram does not wait for the
 * decision: it streams while the previous fold finishes, and steps chain with
 * programmatic dependent launch. d_ns_log (may be NULL): device clock (ns) when the
 * iteration's fold finished -- per-iteration time without events between launches.
 * Requires a workspace of hs_workspace_bytes(); d_state and d_out 16-byte aligned.
 * Asynchronous; no host sync. */
int hs_stream_step(const uint8_t* d_data, const uint64_t* h_begin, const uint64_t* h_end, int nseg,
                   void* d_state, int window_size, double threshold, int recompute_every, int iteration,
                   uint64_t* d_out, double* d_deg_log, double* d_div_log, int32_t* d_kind_log,
                   uint64_t* d_ns_log, void* d_ws, size_t ws_bytes, void* stream);

/* Several iterations per call: the block engine behind run_device_stream. The nseg
 * (<= 256) chunk segments of n_iter (<= 256) consecutive iterations -- iteration i owns
 * the next h_iter_chunks[i] segments -- are counted in ONE histogram call into
 * d_out[nseg][256], then three small kernels fold every iteration exactly as n_iter
 * successive hs_stream_step folds would (same state, same logs at
 * [first_iteration, first_iteration + n_iter), bit for bit): window and accumulator per
 * iteration from prefix sums over (ring ++ block chunks), degeneracy/decision/divergence
 * per iteration in parallel, then the lag-1 decisions in order and the new state.
 * hot_bin >= 0 runs the histogram's register path for that bin (the caller's lagged
 * view of the ADAPTIVE decision, state header: kind at byte 0, hot bin at byte 4, the
 * deciding degeneracy as a double at byte 48); -1 the plain core -- counts are
 * identical. d_ns_log: every iteration of the block gets the commit's device clock.
 * h_decision (may be NULL): page-locked host uint64[3] the commit kernel writes after
 * the block -- [1] kind | hot << 32, [2] the deciding degeneracy (double bits), then
 * [0] = first_iteration + n_iter (written last, after a system fence): the host reads
 * the device's latest decision without an event or copy.
 * Workspace: hs_stream_block_ws_bytes(window_size, nseg) bytes, 16-byte aligned, zeroed
 * once by the caller (every call leaves its tickets zero again). Input contract as
 * hs_stream_step (the histogram is chained behind the previous block's commit). */
size_t hs_stream_block_ws_bytes(int window_size, int max_chunks);
int hs_stream_block(const uint8_t* d_data, const uint64_t* h_begin, const uint64_t* h_end, int nseg,
                    const int32_t* h_iter_chunks, int n_iter, void* d_state, int window_size, double threshold,
                    int recompute_every, int first_iteration, int hot_bin, uint64_t* d_out, double* d_deg_log,
                    double* d_div_log, int32_t* d_kind_log, uint64_t* d_ns_log, uint64_t* h_decision,
                    void* d_ws, size_t ws_bytes, void* stream);

/* ---- host-side control plane (native replacements of pattern.py / policy.py) */

/* compute_binning_pattern (pattern.py:94-133) / uniform_pattern (pattern.py:85-91 when
 * the prior is all zero): floor-1, cap, largest-remainder apportionment in float64.
 * Bit-identical to the reference for totals below 2^53. */
int hs_binning_pattern(const uint64_t* h_prior, int64_t total_slots, int64_t cap,
                       int64_t* h_offset, int64_t* h_count);

/* degeneracy (policy.py:39-46): max-bin share, lowest bin on ties, 0 for empty. */
int hs_degeneracy(const uint64_t* h_counts, double* max_bin_fraction, int* argmax_bin,
                  uint64_t* total);

/* divergence (policy.py:56-64): half the L1 distance of the two normalised histograms,
 * summed in numpy's pairwise order, so the value is the reference's bit for bit.
 * HS_ERR_INVALID_ARG when either histogram is empty (the reference's EmptyHistogram). */
int hs_divergence(const uint64_t* h_a, const uint64_t* h_b, double* out);

/* Host staging helper (no reference counterpart; the reference has no device): copy n
 * bytes from pageable memory into page-locked memory with streaming stores, leaving no
 * dirty lines in the CPU caches, so the DMA that reads the destination next reads DRAM
 * at the link's rate instead of snooping them. Copies of >= 1 MiB are split over up to
 * `threads` host threads (one thread copies ~15 GB/s, a quarter of the PCIe link). */
int hs_copy_streaming(void* dst, const void* src, uint64_t n, int threads);

/* ---- seeded generators (datagen.py:92-155; splitmix64, byte-exact) ------ */
#define HS_GEN_UNIFORM 0
#define HS_GEN_SEQUENTIAL 1
#define HS_GEN_CONSTANT 2
#define HS_GEN_NORMAL 3
#define HS_GEN_MIXTURE 4

/* Host generator: writes n pixels to h_out (uses up to `threads` host threads for
 * the counter-based kinds; mixture is sequential). */
int hs_generate_host(int kind, uint64_t seed, int value, double mean, double sigma,
                     double degeneracy, uint8_t* h_out, uint64_t n, int threads);

/* Device generator (uniform / sequential / constant / normal) for stream positions
 * [first, first+n) of the pixel sequence `generate` would produce: d_out[i] is
 * pixel first+i. Used for >=16 GiB device-resident inputs and sharded streams. */
int hs_generate_device(int kind, uint64_t seed, int value, double mean, double sigma,
                       uint64_t first, uint8_t* d_out, uint64_t n, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HIST256_H */
