// Communication-plan builders: the C++ twin of the reference's record builders.
//
//   fill  : _build_fill            /root/reference/pkg/src/amrkit/fabarray.py:262-277
//   copy  : _build_copy            fabarray.py:291-302
//           build_plan_copy_grown  coarse_fine.py:201-220
//   sum   : build_plan_sum_boundary fabarray.py:305-318 (transpose of fill)
//
// Records are sorted by (dst, dst_box.lo, src, shift) exactly as CommPlan does
// (fabarray.py:182-197), so the table is field-for-field the reference's.
// The spatial hash is a dense bin grid at the largest box extent (the
// reference's BoxHash, boxarray.py:216-278); a 4096-box 512^3 fill plan builds
// in milliseconds instead of the reference's ~20 s.
#include <algorithm>
#include <array>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "amrb_internal.h"

namespace amrb {

namespace {

struct IBox {
  int lo[3];
  int hi[3];
  bool empty() const { return hi[0] < lo[0] || hi[1] < lo[1] || hi[2] < lo[2]; }
};

// D-dim boxes are embedded in 3-D at axes (3-D .. 2); padding axes are [0,0].
IBox load_box(int dim, const int32_t* lohi) {
  IBox b;
  int pad = 3 - dim;
  for (int a = 0; a < 3; ++a) {
    b.lo[a] = 0;
    b.hi[a] = 0;
  }
  for (int d = 0; d < dim; ++d) {
    b.lo[pad + d] = lohi[d];
    b.hi[pad + d] = lohi[dim + d];
  }
  return b;
}

IBox meet(const IBox& a, const IBox& b) {
  IBox r;
  for (int x = 0; x < 3; ++x) {
    r.lo[x] = std::max(a.lo[x], b.lo[x]);
    r.hi[x] = std::min(a.hi[x], b.hi[x]);
  }
  return r;
}

IBox moved(const IBox& a, const int s[3], int sign) {
  IBox r = a;
  for (int x = 0; x < 3; ++x) {
    r.lo[x] += sign * s[x];
    r.hi[x] += sign * s[x];
  }
  return r;
}

IBox grown(const IBox& a, int dim, int g) {
  IBox r = a;
  for (int x = 3 - dim; x < 3; ++x) {
    r.lo[x] -= g;
    r.hi[x] += g;
  }
  return r;
}

// a minus core (core non-empty, inside a): slabs along axis 0 first, lo then hi
// -- the reference box_diff order (index_space.py:320-345).
void slabs(const IBox& a, const IBox& core, int dim, std::vector<IBox>& out) {
  int lo[3], hi[3];
  std::memcpy(lo, a.lo, sizeof lo);
  std::memcpy(hi, a.hi, sizeof hi);
  for (int x = 3 - dim; x < 3; ++x) {
    if (lo[x] < core.lo[x]) {
      IBox p;
      std::memcpy(p.lo, lo, sizeof lo);
      std::memcpy(p.hi, hi, sizeof hi);
      p.hi[x] = core.lo[x] - 1;
      out.push_back(p);
      lo[x] = core.lo[x];
    }
    if (hi[x] > core.hi[x]) {
      IBox p;
      std::memcpy(p.lo, lo, sizeof lo);
      std::memcpy(p.hi, hi, sizeof hi);
      p.lo[x] = core.hi[x] + 1;
      out.push_back(p);
      hi[x] = core.hi[x];
    }
  }
}

// Dense bin grid over a box list, bin size = largest extent per axis.
class BinGrid {
 public:
  explicit BinGrid(const std::vector<IBox>& boxes) : boxes_(boxes) {
    for (int x = 0; x < 3; ++x) {
      size_[x] = 1;
      org_[x] = boxes.empty() ? 0 : boxes[0].lo[x];
      int top = org_[x];
      for (const IBox& b : boxes) {
        size_[x] = std::max(size_[x], b.hi[x] - b.lo[x] + 1);
        org_[x] = std::min(org_[x], b.lo[x]);
        top = std::max(top, b.hi[x]);
      }
      n_[x] = (top - org_[x]) / size_[x] + 1;
    }
    start_.assign((size_t)n_[0] * n_[1] * n_[2] + 1, 0);
    // two-pass CSR fill
    std::vector<int> cnt(start_.size(), 0);
    for (int pass = 0; pass < 2; ++pass) {
      std::fill(cnt.begin(), cnt.end(), 0);
      for (int i = 0; i < (int)boxes.size(); ++i) {
        int klo[3], khi[3];
        keys(boxes[i], klo, khi);
        for (int a = klo[0]; a <= khi[0]; ++a)
          for (int b = klo[1]; b <= khi[1]; ++b)
            for (int c = klo[2]; c <= khi[2]; ++c) {
              size_t bin = ((size_t)a * n_[1] + b) * n_[2] + c;
              if (pass == 0)
                cnt[bin]++;
              else
                items_[start_[bin] + cnt[bin]++] = i;
            }
      }
      if (pass == 0) {
        for (size_t k = 0; k + 1 < start_.size(); ++k) start_[k + 1] = start_[k] + cnt[k];
        items_.resize(start_.back());
      }
    }
    seen_.assign(boxes.size(), -1);
  }

  // (index, overlap) for members meeting q; candidate order is irrelevant
  // because records are sorted afterwards.
  template <class F>
  void query(const IBox& q, F&& fn) {
    if (q.empty() || boxes_.empty()) return;
    ++stamp_;
    int klo[3], khi[3];
    keys(q, klo, khi);
    for (int x = 0; x < 3; ++x) {
      klo[x] = std::max(klo[x], 0);
      khi[x] = std::min(khi[x], n_[x] - 1);
      if (klo[x] > khi[x]) return;
    }
    for (int a = klo[0]; a <= khi[0]; ++a)
      for (int b = klo[1]; b <= khi[1]; ++b)
        for (int c = klo[2]; c <= khi[2]; ++c) {
          size_t bin = ((size_t)a * n_[1] + b) * n_[2] + c;
          for (int k = start_[bin]; k < start_[bin + 1]; ++k) {
            int i = items_[k];
            if (seen_[i] == stamp_) continue;
            seen_[i] = stamp_;
            IBox ov = meet(boxes_[i], q);
            if (!ov.empty()) fn(i, ov);
          }
        }
  }

 private:
  static int fdiv(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }
  void keys(const IBox& q, int klo[3], int khi[3]) const {
    for (int x = 0; x < 3; ++x) {
      klo[x] = fdiv(q.lo[x] - org_[x], size_[x]);
      khi[x] = fdiv(q.hi[x] - org_[x], size_[x]);
    }
  }
  const std::vector<IBox>& boxes_;
  int size_[3], org_[3], n_[3];
  std::vector<int> start_, items_;
  std::vector<int> seen_;
  int stamp_ = 0;
};

std::vector<IBox> load_boxes(int dim, int n, const int32_t* lohi) {
  std::vector<IBox> v((size_t)n);
  for (int i = 0; i < n; ++i) v[i] = load_box(dim, lohi + (size_t)i * 2 * dim);
  return v;
}

// _periodic_shifts (fabarray.py:235-243); the order is irrelevant after the
// record sort, but the zero shift is kept first like the reference.
std::vector<std::array<int, 3>> periodic_shifts(int dim, const IBox& dom, const uint8_t* periodic) {
  std::vector<std::array<int, 3>> out;
  int pad = 3 - dim;
  int choice[3][3], nc[3];
  for (int x = 0; x < 3; ++x) {
    nc[x] = 1;
    choice[x][0] = 0;
    if (x >= pad && periodic && periodic[x - pad]) {
      int e = dom.hi[x] - dom.lo[x] + 1;
      nc[x] = 3;
      choice[x][1] = -e;
      choice[x][2] = e;
    }
  }
  for (int a = 0; a < nc[0]; ++a)
    for (int b = 0; b < nc[1]; ++b)
      for (int c = 0; c < nc[2]; ++c) out.push_back({choice[0][a], choice[1][b], choice[2][c]});
  return out;
}

void sort_records(std::vector<Record>& recs) {
  std::sort(recs.begin(), recs.end(), [](const Record& p, const Record& q) {
    if (p.dst != q.dst) return p.dst < q.dst;
    for (int x = 0; x < 3; ++x) {
      int a = p.lo[x] + p.shift[x], b = q.lo[x] + q.shift[x];
      if (a != b) return a < b;
    }
    if (p.src != q.src) return p.src < q.src;
    for (int x = 0; x < 3; ++x)
      if (p.shift[x] != q.shift[x]) return p.shift[x] < q.shift[x];
    return false;
  });
}

Record make_record(int src, int dst, const IBox& ov, const std::array<int, 3>& s) {
  Record r;
  r.src = src;
  r.dst = dst;
  for (int x = 0; x < 3; ++x) {
    r.lo[x] = ov.lo[x];
    r.hi[x] = ov.hi[x];
    r.shift[x] = s[x];
  }
  return r;
}

std::vector<Record> build_fill(int dim, const std::vector<IBox>& boxes, int ngrow, const IBox& dom,
                               const uint8_t* periodic) {
  int pad = 3 - dim;
  for (int d = 0; d < dim; ++d) {
    int e = dom.hi[pad + d] - dom.lo[pad + d] + 1;
    if (periodic && periodic[d] && ngrow > e)
      throw Error(AMRB_EINVAL, "ghost width exceeds domain extent in a periodic dimension");
  }
  auto shifts = periodic_shifts(dim, dom, periodic);
  BinGrid grid(boxes);
  std::vector<Record> recs;
  std::vector<IBox> pieces;
  for (int j = 0; j < (int)boxes.size(); ++j) {
    const IBox& v = boxes[j];
    pieces.clear();
    if (ngrow > 0) slabs(grown(v, dim, ngrow), v, dim, pieces);
    for (const IBox& piece : pieces)
      for (const auto& s : shifts) {
        bool zero = s[0] == 0 && s[1] == 0 && s[2] == 0;
        grid.query(moved(piece, s.data(), -1), [&](int i, const IBox& ov) {
          if (i == j && zero) return;
          recs.push_back(make_record(i, j, ov, s));
        });
      }
  }
  sort_records(recs);
  return recs;
}

IBox load_domain(int dim, const int32_t* d) { return load_box(dim, d); }

}  // namespace

int64_t Plan::cells() const {
  int64_t n = 0;
  for (const Record& r : recs) n += r.cells();
  return n;
}

}  // namespace amrb

using amrb::Error;
using amrb::Plan;

extern "C" int amrb_plan_fill_create(int dim, int nboxes, const int32_t* lohi, int ngrow,
                                     const int32_t* domain_lohi, const uint8_t* periodic,
                                     amrb_plan** out) {
  return amrb::guarded([&] {
    if (dim < 1 || dim > 3 || nboxes < 0 || ngrow < 0 || !out || (nboxes && !lohi) || !domain_lohi)
      throw Error(AMRB_EINVAL, "amrb_plan_fill_create: bad arguments");
    auto boxes = amrb::load_boxes(dim, nboxes, lohi);
    auto* p = new Plan;
    p->dim = dim;
    p->recs = amrb::build_fill(dim, boxes, ngrow, amrb::load_domain(dim, domain_lohi), periodic);
    *out = reinterpret_cast<amrb_plan*>(p);
  });
}

extern "C" int amrb_plan_sum_create(int dim, int nboxes, const int32_t* lohi, int ngrow,
                                    const int32_t* domain_lohi, const uint8_t* periodic,
                                    amrb_plan** out) {
  return amrb::guarded([&] {
    if (dim < 1 || dim > 3 || nboxes < 0 || ngrow < 0 || !out || (nboxes && !lohi) || !domain_lohi)
      throw Error(AMRB_EINVAL, "amrb_plan_sum_create: bad arguments");
    auto boxes = amrb::load_boxes(dim, nboxes, lohi);
    auto fill = amrb::build_fill(dim, boxes, ngrow, amrb::load_domain(dim, domain_lohi), periodic);
    auto* p = new Plan;
    p->dim = dim;
    p->recs.reserve(fill.size());
    for (const auto& r : fill) {
      amrb::Record t;
      t.src = r.dst;
      t.dst = r.src;
      for (int x = 0; x < 3; ++x) {
        t.lo[x] = r.lo[x] + r.shift[x];
        t.hi[x] = r.hi[x] + r.shift[x];
        t.shift[x] = -r.shift[x];
      }
      p->recs.push_back(t);
    }
    amrb::sort_records(p->recs);
    *out = reinterpret_cast<amrb_plan*>(p);
  });
}

extern "C" int amrb_plan_copy_create(int dim, int ndst, const int32_t* dst_lohi, int nsrc,
                                     const int32_t* src_lohi, int dst_ngrow,
                                     const int32_t* domain_lohi, const uint8_t* periodic,
                                     amrb_plan** out) {
  return amrb::guarded([&] {
    if (dim < 1 || dim > 3 || ndst < 0 || nsrc < 0 || dst_ngrow < 0 || !out)
      throw Error(AMRB_EINVAL, "amrb_plan_copy_create: bad arguments");
    auto dst = amrb::load_boxes(dim, ndst, dst_lohi);
    auto src = amrb::load_boxes(dim, nsrc, src_lohi);
    std::vector<std::array<int, 3>> shifts;
    if (domain_lohi)
      shifts = amrb::periodic_shifts(dim, amrb::load_domain(dim, domain_lohi), periodic);
    else
      shifts.push_back({0, 0, 0});
    auto* p = new Plan;
    p->dim = dim;
    if (nsrc > 0) {
      amrb::BinGrid grid(src);
      for (int j = 0; j < ndst; ++j) {
        amrb::IBox target = amrb::grown(dst[j], dim, dst_ngrow);
        for (const auto& s : shifts)
          grid.query(amrb::moved(target, s.data(), -1), [&](int i, const amrb::IBox& ov) {
            p->recs.push_back(amrb::make_record(i, j, ov, s));
          });
      }
    }
    amrb::sort_records(p->recs);
    *out = reinterpret_cast<amrb_plan*>(p);
  });
}

extern "C" int amrb_plan_size(const amrb_plan* p, int64_t* nrecords, int64_t* ncells) {
  return amrb::guarded([&] {
    if (!p) throw Error(AMRB_EINVAL, "null plan");
    const Plan* q = reinterpret_cast<const Plan*>(p);
    if (nrecords) *nrecords = (int64_t)q->recs.size();
    if (ncells) *ncells = q->cells();
  });
}

extern "C" int amrb_plan_records(const amrb_plan* p, int32_t* out) {
  return amrb::guarded([&] {
    if (!p || !out) throw Error(AMRB_EINVAL, "null argument");
    const Plan* q = reinterpret_cast<const Plan*>(p);
    for (const auto& r : q->recs) {
      *out++ = r.src;
      *out++ = r.dst;
      for (int x = 0; x < 3; ++x) *out++ = r.lo[x];
      for (int x = 0; x < 3; ++x) *out++ = r.hi[x];
      for (int x = 0; x < 3; ++x) *out++ = r.shift[x];
    }
  });
}

extern "C" int amrb_plan_destroy(amrb_plan* p) {
  delete reinterpret_cast<Plan*>(p);
  return AMRB_OK;
}
