// Ghost-push tables (amrb_push_*): FillBoundary fused into the kernel that
// produces a field.  The records are exactly the fill plan's
// (fabarray.py:262-277 / plan.cpp), restricted to sources this rank owns; each
// becomes (source region, destination rank, destination element offset and
// strides).  A producer kernel stores every valid cell it writes also to the
// ghost cells those records map it to -- locally, or over NVLink into the
// owner's symmetric allocation -- so the consumer needs no copy program, only
// (multi-GPU) a device barrier.
#include <algorithm>
#include <cstring>
#include <memory>

#include "device.h"

namespace amrb {
namespace {

int cls_lo(int c, int n, int g) { return c == 0 ? 0 : (c == 1 ? g : n - g); }
int cls_hi(int c, int n, int g) { return c == 0 ? g - 1 : (c == 1 ? n - g - 1 : n - 1); }

}  // namespace
}  // namespace amrb

extern "C" int amrb_push_create(const amrb_level* lv_, int nrec, const int32_t* rec11, const int64_t* fabtab,
                                int nboxes, const int32_t* owner, int my_rank, int nranks, int width,
                                amrb_push** out) {
  using namespace amrb;
  return guarded([&] {
    if (!lv_ || !out || nrec < 0 || (nrec && !rec11) || !fabtab || !owner || width < 1 || nranks < 1 ||
        nranks > kMaxPeers || my_rank < 0 || my_rank >= nranks)
      throw Error(AMRB_EINVAL, "amrb_push_create: bad arguments");
    const Level& lv = *reinterpret_cast<const Level*>(lv_);
    if (lv.nboxes != nboxes) throw Error(AMRB_EINVAL, "amrb_push_create: box count differs from the level");
    const int g = width;
    auto P = std::make_unique<Push>();
    P->g = g;
    P->nboxes = nboxes;
    P->nranks = nranks;
    P->my_rank = my_rank;
    P->hbox.assign(nboxes, PushBox{});
    std::vector<std::vector<int>> lists((size_t)nboxes * 9);
    for (int b = 0; b < nboxes; ++b) {
      PushBox& pb = P->hbox[b];
      std::memcpy(pb.n, lv.geo[b].n, sizeof pb.n);
      if (owner[b] == my_rank)
        for (int d = 0; d < 3; ++d)
          if (lv.geo[b].n[d] < 2 * g) throw Error(AMRB_ENOTSUP, "amrb_push_create: box thinner than 2 x width");
    }
    auto ft = [&](int b, int w) { return fabtab[(int64_t)b * AMRB_FABTAB_W + w]; };
    for (int q = 0; q < nrec; ++q) {
      const int32_t* r = rec11 + (int64_t)q * 11;
      const int s = r[0], d = r[1];
      if (s < 0 || s >= nboxes || d < 0 || d >= nboxes) throw Error(AMRB_EINVAL, "amrb_push_create: bad record");
      if (owner[s] != my_rank) continue;
      const BoxGeom& gs = lv.geo[s];
      PushRec pr{};
      for (int x = 0; x < 3; ++x) {
        pr.lo[x] = r[2 + x] - gs.lo[x];
        pr.hi[x] = r[5 + x] - gs.lo[x];
      }
      pr.peer = owner[d];
      pr.s0 = ft(d, 2);
      pr.s1 = ft(d, 3);
      pr.off = ft(d, 0) + (int64_t)(gs.lo[0] + r[8] - ft(d, 4)) * pr.s0 + (int64_t)(gs.lo[1] + r[9] - ft(d, 5)) * pr.s1 +
               (gs.lo[2] + r[10] - ft(d, 6));
      if (pr.s0 != ft(s, 2)) throw Error(AMRB_ENOTSUP, "amrb_push_create: destination plane stride differs");
      const int idx = (int)P->hrec.size();
      P->hrec.push_back(pr);
      for (int ci = 0; ci < 3; ++ci)
        for (int cj = 0; cj < 3; ++cj) {
          const int a0 = cls_lo(ci, gs.n[0], g), a1 = cls_hi(ci, gs.n[0], g);
          const int b0 = cls_lo(cj, gs.n[1], g), b1 = cls_hi(cj, gs.n[1], g);
          if (a0 > a1 || b0 > b1) continue;
          if (pr.hi[0] < a0 || pr.lo[0] > a1 || pr.hi[1] < b0 || pr.lo[1] > b1) continue;
          lists[(size_t)s * 9 + 3 * ci + cj].push_back(idx);
        }
    }
    for (int b = 0; b < nboxes; ++b) {
      PushBox& pb = P->hbox[b];
      for (int c = 0; c < 9; ++c) {
        const auto& l = lists[(size_t)b * 9 + c];
        pb.off[c] = (int)P->hcand.size();
        pb.cnt[c] = (int)l.size();
        P->hcand.insert(P->hcand.end(), l.begin(), l.end());
      }
      if (owner[b] != my_rank) continue;
      // interior planes: producers precompute per-cell destination deltas, so
      // every record touching them must span all interior planes and no cell
      // may have more than three destinations there (two faces + edge)
      const int n0 = pb.n[0], n1 = pb.n[1], n2 = pb.n[2];
      for (int cj = 0; cj < 3; ++cj) {
        const auto& l = lists[(size_t)b * 9 + 3 + cj];
        for (int q : l) {
          const PushRec& pr = P->hrec[q];
          if (pr.lo[0] > g || pr.hi[0] < n0 - g - 1)
            throw Error(AMRB_ENOTSUP, "amrb_push_create: record covers part of the interior planes");
        }
        const int j0 = cls_lo(cj, n1, g), j1 = cls_hi(cj, n1, g);
        for (int j = j0; j <= j1; ++j)
          for (int k = 0; k < n2; ++k) {
            int cover = 0;
            for (int q : l) {
              const PushRec& pr = P->hrec[q];
              cover += j >= pr.lo[1] && j <= pr.hi[1] && k >= pr.lo[2] && k <= pr.hi[2];
            }
            if (cover > 3) throw Error(AMRB_ENOTSUP, "amrb_push_create: more than three destinations per cell");
          }
      }
    }
    P->box.upload(P->hbox);
    P->rec.upload(P->hrec);
    if (P->hcand.empty()) P->hcand.push_back(0);
    P->cand.upload(P->hcand);
    *out = reinterpret_cast<amrb_push*>(P.release());
  });
}

extern "C" int amrb_push_destroy(amrb_push* p) {
  delete reinterpret_cast<amrb::Push*>(p);
  return AMRB_OK;
}
