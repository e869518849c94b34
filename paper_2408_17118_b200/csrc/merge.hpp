// Global selection decision over per-rank cluster records (reading A6, DESIGN.md §2/§5).
// __host__ __device__: the same source runs in the device accept kernel (product path) and
// in the host-only ABI function oica_merge_records (CPU unit tests of the multi-rank logic).
#pragma once
#include <math.h>
#include <stdint.h>

#include "../../include/oica.h"

#ifndef __CUDACC__
#define OICA_HD
#else
#define OICA_HD __host__ __device__
#endif

namespace oica {

struct MergeOut {
  int32_t winner;        // index of the record that supplies q (or -1)
  int64_t merged_size;   // sum of sizes of the winner's group
  uint8_t near_tie;
};

// records[r].w is w + r*N.  group[] is scratch of length n.  raw: no grouping (OICA_RAW_ARGMAX).
OICA_HD inline MergeOut merge_records(const oica_cluster_record* rec, const double* w, int32_t n,
                                      int32_t N, int32_t* group, bool raw, double delta,
                                      double near_rel) {
  MergeOut out{-1, 0, 0};
  // 1. group records on the same fixed point: 1 - |w_a . w_b| <= delta (first matching root).
  for (int a = 0; a < n; ++a) {
    group[a] = -1;
    if (!rec[a].valid) continue;
    group[a] = a;
    if (raw) continue;
    for (int b = 0; b < a; ++b) {
      if (!rec[b].valid || group[b] != b) continue;
      double dot = 0.0;
      for (int j = 0; j < N; ++j) dot += w[(int64_t)a * N + j] * w[(int64_t)b * N + j];
      if (1.0 - fabs(dot) <= delta) { group[a] = b; break; }
    }
  }
  // 2. per root: key = max upsilon of members, q-record = member of minimum q, size = sum.
  int best = -1, second = -1;
  double best_key = -INFINITY, second_key = -INFINITY;
  int64_t best_q = INT64_MAX;
  for (int r = 0; r < n; ++r) {
    if (group[r] != r) continue;
    double key = -INFINITY;
    int64_t qmin = INT64_MAX;
    for (int a = r; a < n; ++a) {
      if (group[a] != r) continue;
      if (rec[a].upsilon > key) key = rec[a].upsilon;
      if (rec[a].q < qmin) qmin = rec[a].q;
    }
    if (key > best_key || (key == best_key && qmin < best_q)) {
      second = best; second_key = best_key;
      best = r; best_key = key; best_q = qmin;
    } else if (key > second_key) {
      second = r; second_key = key;
    }
  }
  if (best < 0 || !(best_key > -INFINITY)) return out;
  int64_t size = 0;
  int win = -1;
  for (int a = best; a < n; ++a) {
    if (group[a] != best) continue;
    size += rec[a].size;
    if (win < 0 || rec[a].q < rec[win].q) win = a;
  }
  out.winner = win;
  out.merged_size = size;
  out.near_tie = (second >= 0 && best_key - second_key <= near_rel * fabs(best_key)) ? 1 : 0;
  return out;
}

}  // namespace oica
