// Box -> rank (GPU) assignment: the C++ side of DistributionMapping's
// builders (reference: /root/reference/pkg/src/amrkit/distribution.py).
//
//   morton keys  distribution.py:70-90   box centre (lo + hi) // 2 (floor),
//                shifted by the layout's minimal-box lo; bit k of axis d ->
//                key bit k*D + d (axis 0 least significant), 63/D bits per axis
//   SFC split    distribution.py:97-131  boxes in (key, index) order cut into
//                nranks contiguous runs, each grown while it stays within
//                1e-12 of the remaining average cost; every rank below the box
//                count keeps at least one box, the last rank takes the rest
//   knapsack     distribution.py:134-148 longest processing time first: costs
//                descending (ties: lower index), each to the least-loaded rank
//                (ties: lower rank)
//
// The caller passes the total cost it summed (numpy's pairwise sum in the
// Python wrapper) so the split thresholds are the reference's bits.
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <queue>
#include <vector>

#include "amrb_internal.h"

namespace {

int64_t floor_half(int64_t x) { return x >= 0 ? x / 2 : -((-x + 1) / 2); }

// shifted coordinates must lie in [0, 2^bits); 1-D keys use 63 bits
bool in_key_range(int64_t c, int bits) { return c >= 0 && (bits >= 63 || c < ((int64_t)1 << bits)); }

// Morton keys of the box centres; false if a shifted coordinate is out of range
bool centre_keys(int dim, int n, const int32_t* lohi, std::vector<uint64_t>& keys, int64_t* bad_coord) {
  std::vector<int64_t> origin(dim, 0);
  for (int d = 0; d < dim; ++d) {
    int64_t m = lohi[d];
    for (int b = 1; b < n; ++b) m = std::min<int64_t>(m, lohi[(int64_t)b * 2 * dim + d]);
    origin[d] = m;
  }
  const int bits = 63 / dim;
  keys.assign(n, 0);
  for (int b = 0; b < n; ++b) {
    const int32_t* box = lohi + (int64_t)b * 2 * dim;
    uint64_t key = 0;
    for (int d = 0; d < dim; ++d) {
      const int64_t centre = floor_half((int64_t)box[d] + box[dim + d]);
      const int64_t c = centre - origin[d];
      if (!in_key_range(c, bits)) {
        if (bad_coord) *bad_coord = centre;
        return false;
      }
      for (int k = 0; k < bits && (c >> k); ++k)
        if ((c >> k) & 1) key |= (uint64_t)1 << (k * dim + d);
    }
    keys[b] = key;
  }
  return true;
}

}  // namespace

using amrb::Error;
using amrb::guarded;

extern "C" int amrb_morton_key(int dim, const int32_t* point, const int32_t* origin, uint64_t* key) {
  return guarded([&] {
    if (dim < 1 || dim > 3 || !point || !origin || !key) throw Error(AMRB_EINVAL, "amrb_morton_key: bad arguments");
    const int bits = 63 / dim;
    uint64_t k = 0;
    for (int d = 0; d < dim; ++d) {
      const int64_t c = (int64_t)point[d] - origin[d];
      if (!in_key_range(c, bits))
        throw Error(AMRB_EINVAL, "coordinate " + std::to_string(point[d]) + " out of key range (needs 0 <= shifted < 2^" +
                                     std::to_string(bits) + ")");
      for (int b = 0; b < bits && (c >> b); ++b)
        if ((c >> b) & 1) k |= (uint64_t)1 << (b * dim + d);
    }
    *key = k;
  });
}

extern "C" int amrb_sfc_distribute(int dim, int n, const int32_t* lohi, const double* cost, double total,
                                   int nranks, int32_t* owner) {
  return guarded([&] {
    if (dim < 1 || dim > 3 || n < 0 || nranks < 1 || (n && (!lohi || !cost || !owner)))
      throw Error(AMRB_EINVAL, "amrb_sfc_distribute: bad arguments");
    if (n == 0) return;
    std::vector<uint64_t> keys;
    int64_t bad = 0;
    if (!centre_keys(dim, n, lohi, keys, &bad))
      throw Error(AMRB_EINVAL, "coordinate " + std::to_string(bad) + " out of key range");
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int a, int b) { return keys[a] != keys[b] ? keys[a] < keys[b] : a < b; });
    int pos = 0;
    double done = 0.0;
    for (int r = 0; r < nranks; ++r) {
      const int ranks_left = nranks - r;
      const int limit = (n - pos) - (ranks_left - 1);
      const double goal = (total - done) / ranks_left;
      int take = 0;
      double run = 0.0;
      for (; take < limit; ++take) {
        const double c = cost[order[pos + take]];
        if (take > 0 && run + c > goal + 1e-12) break;
        run += c;
      }
      if (r == nranks - 1) take = n - pos;
      for (int x = 0; x < take; ++x) owner[order[pos + x]] = r;
      pos += take;
      done += run;
    }
  });
}

extern "C" int amrb_knapsack_distribute(int n, const double* cost, int nranks, int32_t* owner) {
  return guarded([&] {
    if (n < 0 || nranks < 1 || (n && (!cost || !owner))) throw Error(AMRB_EINVAL, "amrb_knapsack_distribute: bad arguments");
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
    using Slot = std::pair<double, int>;  // (load, rank): smallest first, ties to the lower rank
    std::priority_queue<Slot, std::vector<Slot>, std::greater<Slot>> ranks;
    for (int r = 0; r < nranks; ++r) ranks.emplace(0.0, r);
    for (int i : order) {
      Slot s = ranks.top();
      ranks.pop();
      owner[i] = s.second;
      ranks.emplace(s.first + cost[i], s.second);
    }
  });
}
