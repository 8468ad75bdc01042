// Per-unit device cost of an all-pairs alignment vs N = max(n_a, n_b), for
// the multi-GPU split (cfgsim_allpairs_split; the Python mirror
// distributed.split_units parses this table).  Microseconds of one B200 per
// unit (1 / throughput), measured by tools/calibrate_split.py: allpairs_range
// over whole rows of each N's row group of the c5 corpus (a row's partners
// are all smaller graphs, the mix the triangle has).  Piecewise linear in N
// between the samples, clamped at the ends.  Only ratios matter for the
// split; the tiers show: two-stage (N <= 64) amortises the per-graph
// sequences over a row, the per-pair kernels above 64 cost ~linear in N.
#pragma once

namespace cfgsim {

// clang-format off
// COST_TABLE_BEGIN
static const int kCostN[] = {16, 32, 33, 48, 64, 65, 72, 80, 96, 112, 128, 129, 144, 160, 176, 192, 208, 224, 240, 256, 257, 288, 320, 352, 384, 416, 448, 480, 512};
static const double kCostUs[] = {0.023, 0.023, 0.05, 0.055, 0.07, 1.13, 1.235, 1.345, 2.39, 2.89, 3.16, 2.35, 2.31, 2.57, 2.82, 2.98, 3.45, 3.7, 3.98, 3.95, 5.99, 6.51, 7.36, 8.21, 9.31, 10.17, 11.13, 12.56, 13.41};
// COST_TABLE_END
// clang-format on

inline double unit_cost_us(int N) {
  constexpr int n = (int)(sizeof(kCostN) / sizeof(kCostN[0]));
  if (N <= kCostN[0]) return kCostUs[0];
  for (int i = 1; i < n; i++)
    if (N <= kCostN[i]) {
      const double t = (double)(N - kCostN[i - 1]) / (double)(kCostN[i] - kCostN[i - 1]);
      return kCostUs[i - 1] + t * (kCostUs[i] - kCostUs[i - 1]);
    }
  return kCostUs[n - 1];
}

}  // namespace cfgsim
