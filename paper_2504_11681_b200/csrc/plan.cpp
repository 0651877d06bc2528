// Host-side FFT plan analysis: prune masks and the canonical op / twiddle
// budgets of the reference's radix-2 Stockham plan (fnofuse/fft.py:97-182).
// These budgets are the canonical flop count of the layer (SURVEY.md §8d,
// pipeline.py:369-416 layer_op_stats) used for GFLOP/s and the roofline.
#include <stdint.h>
#include <string.h>

#include <vector>

extern "C" int tfno_plan_counts(int n, int direction, int keep, int src_len, int64_t* op_budget,
                                int64_t* twiddle_budget, int64_t* full_ops, uint8_t* masks) {
  (void)direction;  // the DAG does not depend on the sign of the exponent
  if (n < 1 || (n & (n - 1))) return 2;
  if (keep < 1 || keep > n || src_len < 1 || src_len > n) return 2;
  int ns = 0;
  while ((1 << ns) < n) ++ns;
  // backward pass: stage outputs some retained bin depends on (fft.py:131-144)
  std::vector<std::vector<uint8_t>> needed(ns);
  std::vector<uint8_t> need(n, 0), prev(n);
  for (int i = 0; i < keep; ++i) need[i] = 1;
  for (int j = ns - 1; j >= 0; --j) {
    const int s = 1 << j, m = n >> (j + 1);
    needed[j] = need;
    std::fill(prev.begin(), prev.end(), 0);
    for (int p = 0; p < m; ++p)
      for (int q = 0; q < s; ++q) {
        // outputs q + s*(2p + r), r in {0,1}, both read slots q+s*p and q+s*(p+m)
        if (need[q + s * (2 * p)] || need[q + s * (2 * p + 1)]) {
          prev[q + s * p] = 1;
          prev[q + s * (p + m)] = 1;
        }
      }
    need.swap(prev);
  }
  // forward pass: possibly-nonzero stage outputs (fft.py:146-161)
  std::vector<uint8_t> nz(n, 0), out(n);
  for (int i = 0; i < src_len; ++i) nz[i] = 1;
  int64_t budget = 0, tw = 0;
  for (int j = 0; j < ns; ++j) {
    const int s = 1 << j, m = n >> (j + 1);
    for (int p = 0; p < m; ++p)
      for (int q = 0; q < s; ++q) {
        uint8_t a = nz[q + s * p], b = nz[q + s * (p + m)];
        uint8_t o = a | b;
        out[q + s * (2 * p)] = o;
        out[q + s * (2 * p + 1)] = o;
        // masks, budgets (fft.py:163-182)
        uint8_t e0 = needed[j][q + s * (2 * p)] & o, e1 = needed[j][q + s * (2 * p + 1)] & o;
        budget += e0 + e1;
        if ((e0 | e1) && b && q >= 1) ++tw;
        if (masks) {
          masks[(size_t)j * n + q + s * (2 * p)] = e0;
          masks[(size_t)j * n + q + s * (2 * p + 1)] = e1;
        }
      }
    nz.swap(out);
  }
  if (op_budget) *op_budget = budget;
  if (twiddle_budget) *twiddle_budget = tw;
  if (full_ops) *full_ops = (int64_t)n * ns;
  return 0;
}
