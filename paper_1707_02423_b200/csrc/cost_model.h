// Per-unit device cost of an all-pairs alignment vs N = max(n_a, n_b), for
// the multi-GPU split (cfgsim_allpairs_split; the Python mirror
// distributed.split_units parses this table).  Microseconds of one B200 per
// unit (1 / throughput), measured by tools/calibrate_split.py: allpairs_range
// over whole row groups of each N of the c5 corpus (a row's partners are all
// smaller graphs, the mix the triangle has; whole groups, so the large-N
// history mode applies as in the real run; gpurun_out/r2y).  N <= 64: the
// two-stage path's per-unit cost from a C2 step's per-group kernel times
// (the c5 corpus has too few small-N units to time it).  Piecewise linear in N
// between the samples, clamped at the ends.  Only ratios matter for the
// split; the tiers show: two-stage (N <= 64) amortises the per-graph
// sequences over a row, the per-pair kernels above 64 cost ~linear in N.
#pragma once

namespace cfgsim {

// clang-format off
// COST_TABLE_BEGIN
static const int kCostN[] = {16, 32, 33, 48, 64, 65, 72, 88, 96, 97, 112, 120, 128, 129, 136, 160, 184, 192, 208, 232, 256, 257, 280, 304, 328, 352, 376, 384, 400, 424, 448, 472, 496, 512};
static const double kCostUs[] = {0.023, 0.023, 0.05, 0.055, 0.07, 1.37, 1.43, 1.52, 2.54, 2.16, 1.13, 1.33, 1.22, 1.48, 1.74, 1.75, 2.08, 2.17, 2.67, 2.9, 3.02, 4.27, 4.67, 5.08, 5.8, 6.25, 7.24, 7.18, 7.99, 8.64, 9.05, 9.75, 10.57, 10.28};
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
