// Device helpers shared by the stencil translation units.
//
// Operand order of the 7-point operator and the GSRB relaxation is the
// oracle's (oracle/mlmg_ref.py); with --fmad=false every product and sum is
// rounded separately, so kernels match numpy bit for bit.
#pragma once

#include "device.h"

namespace amrb {

struct Coef {
  double dh0, dh1, dh2, rgamma;  // rgamma = 1 / (-2 (dh0 + dh1 + dh2))
};

inline Coef make_coef(const double dh[3]) {
  Coef c;
  c.dh0 = dh[0];
  c.dh1 = dh[1];
  c.dh2 = dh[2];
  c.rgamma = 1.0 / (-2.0 * ((dh[0] + dh[1]) + dh[2]));
  return c;
}

// ((dh0*((xm - 2c) + xp) + dh1*((ym - 2c) + yp)) + dh2*((zm - 2c) + zp))
__device__ __forceinline__ double lap7(double c, double xm, double xp, double ym, double yp, double zm,
                                       double zp, const Coef& k) {
  const double c2 = 2.0 * c;
  const double tx = k.dh0 * ((xm - c2) + xp);
  const double ty = k.dh1 * ((ym - c2) + yp);
  const double tz = k.dh2 * ((zm - c2) + zp);
  return (tx + ty) + tz;
}

__device__ __forceinline__ double relax(double c, double rhs, double lap, double rgamma) {
  return c + (rhs - lap) * rgamma;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

// Ghost push helpers (see PushRec in device.h).
__device__ __forceinline__ int push_cls(int x, int n, int g) { return x < g ? 0 : (x >= n - g ? 2 : 1); }

// Store v (box-local cell (i, j, k) of box b) into every destination ghost
// cell whose record covers it.  Out of line: only rows/planes within g of a
// box face take this path.
// Returns true when it stored to another rank (the caller then issues one
// system-scope fence before it exits, so the consumer's barrier orders it).
template <bool INL = false>
static __device__ __forceinline__ bool push_cell_t(const PushDev* pd, int b, int i, int j, int k, double v) {
  const PushBox& B = pd->box[b];
  const int cls = 3 * push_cls(i, B.n[0], pd->g) + push_cls(j, B.n[1], pd->g);
  const int o = B.off[cls], n = B.cnt[cls];
  bool remote = false;
  for (int q = 0; q < n; ++q) {
    const PushRec& r = pd->rec[pd->cand[o + q]];
    if (i < r.lo[0] || i > r.hi[0] || j < r.lo[1] || j > r.hi[1] || k < r.lo[2] || k > r.hi[2]) continue;
    pd->base[r.peer][r.off + (int64_t)i * r.s0 + (int64_t)j * r.s1 + k] = v;
    remote |= r.peer != pd->my_rank;
  }
  return remote;
}
static __device__ __noinline__ bool push_cell(const PushDev* pd, int b, int i, int j, int k, double v) {
  return push_cell_t(pd, b, i, j, k, v);
}

// Destinations of cell (j, k) of box b in the box's interior planes (all
// planes at least g from the i faces), as element deltas from the cell's own
// address in the producer's output (view V at out_base): at most kPushMid
// records (j face, k face, j-k edge) cover such a cell; 0 = none.
// push_create guarantees interior records span every interior plane and the
// destination plane stride equals V's, so the deltas do not depend on the plane.
constexpr int kPushMid = 3;
__device__ __forceinline__ void push_deltas_mid(const PushDev& pd, int b, int j, int k, const FabView& V,
                                                const double* out_base, int64_t (&d)[kPushMid], bool& remote) {
#pragma unroll
  for (int x = 0; x < kPushMid; ++x) d[x] = 0;
  const PushBox& B = pd.box[b];
  const int c = 3 + push_cls(j, B.n[1], pd.g);
  const int o = B.off[c], n = B.cnt[c];
  int m = 0;
  for (int q = 0; q < n; ++q) {
    const PushRec& r = pd.rec[pd.cand[o + q]];
    if (j < r.lo[1] || j > r.hi[1] || k < r.lo[2] || k > r.hi[2]) continue;
    const int64_t dd = ((int64_t)pd.base[r.peer] - (int64_t)out_base) / 8 + r.off + (int64_t)j * r.s1 -
                       V.off - (int64_t)j * V.s1;
#pragma unroll
    for (int x = 0; x < kPushMid; ++x)
      if (m == x) d[x] = dd;
    ++m;
    remote |= r.peer != pd.my_rank;
  }
}

// Launchers implemented in sweep.cu (TMA path).  Return false when the level's
// storage is not uniform enough for a tensor map (caller falls back).
bool launch_sweep_tma(Level& lv, const Field& a, const double* a_base, const Field& b, double* b_base,
                      const Field& r, const double* r_base, const Coef& cf, const int fixed_lo[3],
                      const int fixed_hi[3], bool fixed, cudaStream_t st, const PushDev* push = nullptr);
// gsrb_stream.cu: mode 0 plain, 1 fused prolongation (clv / c / c_base),
// 2 plain + max |rhs - L(a)| into *norm (u64 bit pattern, caller zeroes it)
bool launch_sweep_stream(int mode, Level& lv, const Field& a, const double* a_base, const Field& b, double* b_base,
                         const Field& r, const double* r_base, const Coef& cf, const int flo[3], const int fhi[3],
                         cudaStream_t st, const Level* clv, const Field* c, const double* c_base,
                         unsigned long long* norm);
bool launch_sweep_prolong_tma(Level& lv, const Field& a, const double* a_base, const Field& b, double* b_base,
                              const Field& r, const double* r_base, const Coef& cf, const Level& clv, const Field& c,
                              const double* c_base, cudaStream_t st);

}  // namespace amrb
