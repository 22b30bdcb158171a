// Host-only check of the weighted CTA split (no GPU needed): random segment layouts
// through split_grid() of hs_kernels.cu, built with HS_CHECK_SPLIT so the one-pass
// table is compared with the binary-search definition at every CTA; then the table is
// checked to partition the units monotonically and the per-segment ticket targets are
// recomputed by brute force. Prints "split_check ok" and exits 0.
#define HS_CHECK_SPLIT
#include "../../paper_1011_0235_b200/csrc/hs_kernels.cu"

#include <cstdio>
#include <random>

int main() {
  std::mt19937_64 rng(1011);
  long checked = 0;
  for (int trial = 0; trial < 20000; ++trial) {
    SegParams sp;
    sp.nseg = 1 + int(rng() % kMaxSeg);
    const uint64_t total = 4 * (1 + rng() % ((1ull << 30) / 4));
    std::vector<uint64_t> cut(sp.nseg + 1);
    cut[0] = 0;
    cut[sp.nseg] = total;
    for (int s = 1; s < sp.nseg; ++s) cut[s] = 4 * (rng() % (total / 4 + 1));
    std::sort(cut.begin(), cut.end());
    if (rng() % 4 == 0)  // runs of empty segments, leading ones included
      for (int s = 1; s < sp.nseg && s < 1 + int(rng() % 8); ++s) cut[s] = cut[0];
    for (int s = 0; s <= sp.nseg; ++s) sp.vstart[s] = cut[s];
    const int grid = 1 + int(rng() % kMaxSplitGrid);
    const uint32_t cost = uint32_t(rng() % 64);
    split_grid(sp, grid, cost);  // aborts on a table mismatch (HS_CHECK_SPLIT)
    if (!sp.split_cost) continue;
    const uint64_t units = sp.units;
    if (sp.cta_unit[0] != 0 || sp.cta_unit[grid] != units) return printf("ends wrong\n"), 1;
    for (int b = 0; b < grid; ++b)
      if (sp.cta_unit[b] > sp.cta_unit[b + 1]) return printf("not monotone\n"), 1;
    for (int s = 0; s < sp.nseg; ++s) {
      if (sp.vstart[s + 1] <= sp.vstart[s]) continue;
      uint32_t n = 0;  // CTAs whose byte range meets the segment
      for (int b = 0; b < grid; ++b) {
        const uint64_t vb = std::min<uint64_t>(total, 4096ull * sp.cta_unit[b]);
        const uint64_t ve = std::min<uint64_t>(total, 4096ull * sp.cta_unit[b + 1]);
        n += vb < ve && vb < sp.vstart[s + 1] && ve > sp.vstart[s];
      }
      if (sp.ctas_after_first[s] != n - 1) return printf("ticket target wrong (trial %d seg %d)\n", trial, s), 1;
    }
    ++checked;
  }
  printf("split_check ok: %ld weighted layouts\n", checked);
  return 0;
}
