/*
 * ORACLE — test infrastructure only. CPU restatement of the reference's histogram
 * workers (/root/reference/pkg/src/histostream/kernels.py). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load this library; the product path (paper_1011_0235_b200) never does.
 *
 * Pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py) and the reference tests' known answers
 * (tests/test_oracle.py).
 *
 *   or_histogram          reference_histogram  kernels.py:330-333 (np.bincount of the bytes)
 *   or_group_ranges       group_ranges         kernels.py:311-316
 *   or_naive_worker       _naive_worker        kernels.py:97-130  (tag arbitration loop)
 *   or_adaptive_worker    _adaptive_worker     kernels.py:133-168 (+ lane_touch: _traced :171-209,
 *                                               16-bit wrap: _adaptive_worker_u16 :267-303)
 *   or_naive_histogram    naive_histogram      kernels.py:336-346 (group threads + merge_all)
 *   or_adaptive_histogram adaptive_histogram   kernels.py:349-384 (slots per group, reduce_subbins)
 *   or_fill_*             _fill_uniform/_fill_normal/_fill_mixture datagen.py:98-155
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off -pthread).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define BINS 256

/* kernels.py:330-333 — serial count of every pixel (pixel 4i+k is byte k of word i,
 * so the byte stream in memory order is the pixel stream, core.py:1-6). */
void or_histogram(const uint8_t* p, uint64_t n, uint64_t* out) {
  uint64_t c[BINS];
  memset(c, 0, sizeof c);
  for (uint64_t i = 0; i < n; ++i) c[p[i]]++;
  memcpy(out, c, sizeof c);
}

/* kernels.py:311-316 — equal word ranges, remainder to the last group. */
void or_group_ranges(int64_t word_count, int64_t group_count, int64_t* starts, int64_t* stops) {
  const int64_t base = word_count / group_count;
  for (int64_t g = 0; g + 1 < group_count; ++g) { starts[g] = g * base; stops[g] = (g + 1) * base; }
  starts[group_count - 1] = (group_count - 1) * base;
  stops[group_count - 1] = word_count;
}

/* One step of the lockstep group: lanes [0, active) hold words[base + lane]; for each of
 * the 4 packed pixels the arbitration loop commits same-counter lanes one per round,
 * the last pending lane in index order winning each round (kernels.py:105-130). The
 * loop is restated faithfully because its executed work is what the reference's CPU
 * timing measures; its result equals one increment per lane. */
static void step_naive(const uint32_t* lane_words, int64_t active, uint64_t* counters, int64_t* tags,
                       int64_t* slots, int64_t* pend, int64_t* nxt) {
  for (int k = 0; k < 4; ++k) {
    const int shift = 8 * k;
    for (int64_t lane = 0; lane < active; ++lane) {
      slots[lane] = (lane_words[lane] >> shift) & 0xFF;
      pend[lane] = lane;
    }
    int64_t npend = active;
    while (npend > 0) {
      for (int64_t i = 0; i < npend; ++i) tags[slots[pend[i]]] = pend[i];
      int64_t nnext = 0;
      for (int64_t i = 0; i < npend; ++i) {
        const int64_t lane = pend[i];
        const int64_t s = slots[lane];
        if (tags[s] == lane) counters[s] += 1;
        else nxt[nnext++] = lane;
      }
      for (int64_t i = 0; i < nnext; ++i) pend[i] = nxt[i];
      npend = nnext;
    }
  }
}

/* kernels.py:97-130 */
void or_naive_worker(const uint32_t* words, int64_t start, int64_t stop, int64_t group_size,
                     uint64_t* counters) {
  int64_t tags[BINS];
  for (int b = 0; b < BINS; ++b) tags[b] = -1;
  int64_t* slots = (int64_t*)malloc(sizeof(int64_t) * group_size * 3);
  int64_t* pend = slots + group_size;
  int64_t* nxt = pend + group_size;
  uint32_t* lane_words = (uint32_t*)malloc(sizeof(uint32_t) * group_size);
  for (int64_t base = start; base < stop; base += group_size) {
    const int64_t active = (stop - base) < group_size ? (stop - base) : group_size;
    for (int64_t lane = 0; lane < active; ++lane) lane_words[lane] = words[base + lane];
    step_naive(lane_words, active, counters, tags, slots, pend, nxt);
  }
  free(lane_words);
  free(slots);
}

/* kernels.py:133-168 (+ :171-209 when lane_touch != NULL, + :267-303 when narrow != 0).
 * slot_counts: uint64[total_slots] (narrow: values wrap modulo 2^16 like the u16 array);
 * lane_touch: uint64[group_size][total_slots] or NULL. */
void or_adaptive_worker(const uint32_t* words, int64_t start, int64_t stop, int64_t group_size,
                        const int64_t* offset, const int64_t* count, int64_t total_slots,
                        uint64_t* slot_counts, uint64_t* lane_touch, int narrow) {
  int64_t* tags = (int64_t*)malloc(sizeof(int64_t) * total_slots);
  for (int64_t s = 0; s < total_slots; ++s) tags[s] = -1;
  int64_t* slots = (int64_t*)malloc(sizeof(int64_t) * group_size * 3);
  int64_t* pend = slots + group_size;
  int64_t* nxt = pend + group_size;
  uint32_t* lane_words = (uint32_t*)malloc(sizeof(uint32_t) * group_size);
  for (int64_t base = start; base < stop; base += group_size) {
    const int64_t active = (stop - base) < group_size ? (stop - base) : group_size;
    for (int64_t lane = 0; lane < active; ++lane) lane_words[lane] = words[base + lane];
    for (int k = 0; k < 4; ++k) {
      const int shift = 8 * k;
      for (int64_t lane = 0; lane < active; ++lane) {
        const uint32_t b = (lane_words[lane] >> shift) & 0xFF;
        slots[lane] = offset[b] + lane % count[b];
        pend[lane] = lane;
      }
      int64_t npend = active;
      while (npend > 0) {
        for (int64_t i = 0; i < npend; ++i) tags[slots[pend[i]]] = pend[i];
        int64_t nnext = 0;
        for (int64_t i = 0; i < npend; ++i) {
          const int64_t lane = pend[i];
          const int64_t s = slots[lane];
          if (tags[s] == lane) {
            slot_counts[s] = narrow ? ((slot_counts[s] + 1) & 0xFFFF) : slot_counts[s] + 1;
            if (lane_touch) lane_touch[lane * total_slots + s] += 1;
          } else {
            nxt[nnext++] = lane;
          }
        }
        for (int64_t i = 0; i < nnext; ++i) pend[i] = nxt[i];
        npend = nnext;
      }
    }
  }
  free(lane_words);
  free(slots);
  free(tags);
}

/* ---- group-thread drivers (kernels.py:319-327 _run_group_threads) ----------- */
typedef struct {
  const uint32_t* words;
  int64_t start, stop, group_size;
  const int64_t* offset;
  const int64_t* count;
  int64_t total_slots;
  uint64_t* out;
  uint64_t* touch;
  int narrow, adaptive;
} job_t;

static void* run_job(void* arg) {
  job_t* j = (job_t*)arg;
  if (j->adaptive)
    or_adaptive_worker(j->words, j->start, j->stop, j->group_size, j->offset, j->count, j->total_slots,
                       j->out, j->touch, j->narrow);
  else
    or_naive_worker(j->words, j->start, j->stop, j->group_size, j->out);
  return NULL;
}

static void run_groups(job_t* jobs, int64_t g) {
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * g);
  for (int64_t i = 0; i < g; ++i) pthread_create(&th[i], NULL, run_job, &jobs[i]);
  for (int64_t i = 0; i < g; ++i) pthread_join(th[i], NULL);
  free(th);
}

/* kernels.py:336-346; per_group (may be NULL): uint64[group_count][256] partials.
 * Returns 0, or 1 if merging overflowed 64 bits (core.py:146-148 CountOverflow). */
int or_naive_histogram(const uint32_t* words, int64_t n_words, int64_t group_size, int64_t group_count,
                       uint64_t* out, uint64_t* per_group) {
  int64_t* st = (int64_t*)malloc(sizeof(int64_t) * group_count * 2);
  int64_t* sp = st + group_count;
  or_group_ranges(n_words, group_count, st, sp);
  uint64_t* part = (uint64_t*)calloc((size_t)group_count * BINS, sizeof(uint64_t));
  job_t* jobs = (job_t*)calloc((size_t)group_count, sizeof(job_t));
  for (int64_t g = 0; g < group_count; ++g) {
    jobs[g].words = words; jobs[g].start = st[g]; jobs[g].stop = sp[g]; jobs[g].group_size = group_size;
    jobs[g].out = part + g * BINS; jobs[g].adaptive = 0;
  }
  run_groups(jobs, group_count);
  int overflow = 0;
  for (int b = 0; b < BINS; ++b) {
    uint64_t s = 0;
    for (int64_t g = 0; g < group_count; ++g) {
      const uint64_t t = s + part[g * BINS + b];
      if (t < s) overflow = 1;
      s = t;
    }
    out[b] = s;
  }
  if (per_group) memcpy(per_group, part, sizeof(uint64_t) * group_count * BINS);
  free(jobs); free(part); free(st);
  return overflow;
}

/* kernels.py:349-384 (and adaptive_lane_touches :387-407 when touch != NULL).
 * slots_out: uint64[group_count][total_slots] (may be NULL); touch: uint64[G][gs][S] or NULL.
 * Result = merge_all(reduce_subbins(slots_g)) (kernels.py:376, :410-418). */
void or_adaptive_histogram(const uint32_t* words, int64_t n_words, int64_t group_size, int64_t group_count,
                           const int64_t* offset, const int64_t* count, int64_t total_slots, int narrow,
                           uint64_t* out, uint64_t* slots_out, uint64_t* touch) {
  int64_t* st = (int64_t*)malloc(sizeof(int64_t) * group_count * 2);
  int64_t* sp = st + group_count;
  or_group_ranges(n_words, group_count, st, sp);
  uint64_t* slots = (uint64_t*)calloc((size_t)group_count * total_slots, sizeof(uint64_t));
  job_t* jobs = (job_t*)calloc((size_t)group_count, sizeof(job_t));
  for (int64_t g = 0; g < group_count; ++g) {
    jobs[g].words = words; jobs[g].start = st[g]; jobs[g].stop = sp[g]; jobs[g].group_size = group_size;
    jobs[g].offset = offset; jobs[g].count = count; jobs[g].total_slots = total_slots;
    jobs[g].out = slots + g * total_slots; jobs[g].adaptive = 1; jobs[g].narrow = narrow;
    jobs[g].touch = touch ? touch + g * group_size * total_slots : NULL;
  }
  run_groups(jobs, group_count);
  memset(out, 0, sizeof(uint64_t) * BINS);
  for (int64_t g = 0; g < group_count; ++g)
    for (int b = 0; b < BINS; ++b)
      for (int64_t j = 0; j < count[b]; ++j) out[b] += slots[g * total_slots + offset[b] + j];
  if (slots_out) memcpy(slots_out, slots, sizeof(uint64_t) * group_count * total_slots);
  free(jobs); free(slots); free(st);
}

/* ---- splitmix64 generators (datagen.py:6-29, :98-155) ---------------------- */
static uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
#define GOLDEN 0x9E3779B97F4A7C15ull
#define UNIT (1.0 / 9007199254740992.0)

void or_fill_uniform(uint8_t* out, uint64_t n, uint64_t seed) {
  uint64_t state = seed, i = 0;
  while (i < n) {
    state += GOLDEN;
    const uint64_t z = mix(state);
    for (int k = 0; k < 8 && i < n; ++k) out[i++] = (uint8_t)((z >> (8 * k)) & 0xFF);
  }
}

void or_fill_normal(uint8_t* out, uint64_t n, uint64_t seed, double mean, double sigma) {
  uint64_t state = seed;
  for (uint64_t i = 0; i < n; ++i) {
    double total = 0.0;
    for (int j = 0; j < 12; ++j) {
      state += GOLDEN;
      total += (double)(mix(state) >> 11) * UNIT;
    }
    double val = floor(mean + sigma * (total - 6.0) + 0.5);
    if (val < 0.0) val = 0.0;
    else if (val > 255.0) val = 255.0;
    out[i] = (uint8_t)val;
  }
}

void or_fill_mixture(uint8_t* out, uint64_t n, uint64_t seed, double degeneracy, int value) {
  uint64_t state = seed;
  for (uint64_t i = 0; i < n; ++i) {
    state += GOLDEN;
    const double unit = (double)(mix(state) >> 11) * UNIT;
    if (unit < degeneracy) {
      out[i] = (uint8_t)value;
    } else {
      state += GOLDEN;
      out[i] = (uint8_t)(mix(state) & 0xFF);
    }
  }
}
