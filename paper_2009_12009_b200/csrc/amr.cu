// Inter-level AMR operators and the two-level advection step on device
// (SURVEY.md 8(f)4): fill_patch's time blend and interpolation
// (coarse_fine.py:46-99,231-309), the flux register (:317-472) and the upwind
// flux / update kernels of the subcycled advection driver (advect.py:24-47).
//
// Every kernel reproduces the reference's numpy evaluation order (the library
// is compiled with --fmad=false), so results are bit-identical:
//   * upwind flux   F = u * phi(upwind cell)
//   * update        v -= dtdx[d] * (F[hi] - F[lo]) for d = 0 .. dim-1 in turn
//   * blend         (1 - w) * old + w * new
//   * linear interp v = c; v = v + slope_d * off_d for d in turn, slope_d the
//                   minmod of (c - lo, hi - c), off = (m + 0.5) / r - 0.5
//   * register      crse_add: reg - scale * F; fine_add: reg + scale * avg,
//                   avg of the 2 (2-D) or 4 (3-D) fine faces in numpy's
//                   reshape-mean order; reflux: crse + (sign dt/dx) * reg,
//                   contributions in patch order.
// Work is enumerated as a flat index over all resident boxes (per-box prefix
// counts; each thread binary-searches its box).
#include <cmath>

#include "device.h"

namespace amrb {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ int find_box(const int64_t* prefix, int nb, int64_t g) {
  int lo = 0, hi = nb - 1;  // last b with prefix[b] <= g
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (prefix[mid] <= g)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

struct Ext3 {
  int n[3];
};

// Upwind face fluxes along 3-D axis `ax` (a real dimension): face f of the
// box's (ncomp, n + e_ax) face array gets u * phi(f - 1) if u >= 0 else u * phi(f)
// (advect.py:24-36, `src` slices of the ghosted array).
__global__ void __launch_bounds__(kThreads)
    k_adv_flux(const int64_t* __restrict__ prefix, const int* __restrict__ boxes, int nb, const BoxGeom* __restrict__ geo,
               const FabView* __restrict__ pv, const double* __restrict__ phi, const int64_t* __restrict__ foff,
               double* __restrict__ flux, int ncomp, int ax, double u) {
  pdl_entry();
  const int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (g >= prefix[nb]) return;
  const int q = find_box(prefix, nb, g);
  const int b = boxes[q];
  const BoxGeom G = geo[b];
  int e[3] = {G.n[0], G.n[1], G.n[2]};
  e[ax] += 1;
  int64_t t = g - prefix[q];
  const int k = (int)(t % e[2]);
  t /= e[2];
  const int j = (int)(t % e[1]);
  t /= e[1];
  const int i = (int)(t % e[0]);
  const int c = (int)(t / e[0]);
  int x[3] = {i, j, k};
  if (u >= 0.0) x[ax] -= 1;
  const FabView P = pv[b];
  const double v = phi[P.off + c * P.cs + (int64_t)x[0] * P.s0 + (int64_t)x[1] * P.s1 + x[2]];
  flux[foff[b] + g - prefix[q]] = u * v;
}

struct Faces {
  const double* f[3];
  const int64_t* off[3];
};

// phi -= dtdx[d] * (F_d[i + e_d] - F_d[i]) for each real dimension d in turn
// (advect.py:39-47).
__global__ void __launch_bounds__(kThreads)
    k_adv_update(const int64_t* __restrict__ prefix, const int* __restrict__ boxes, int nb,
                 const BoxGeom* __restrict__ geo, const FabView* __restrict__ pv, double* __restrict__ phi,
                 const __grid_constant__ Faces F, int ncomp, int dim, double dt0, double dt1, double dt2) {
  pdl_entry();
  const int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (g >= prefix[nb]) return;
  const int q = find_box(prefix, nb, g);
  const int b = boxes[q];
  const BoxGeom G = geo[b];
  int64_t t = g - prefix[q];
  const int k = (int)(t % G.n[2]);
  t /= G.n[2];
  const int j = (int)(t % G.n[1]);
  t /= G.n[1];
  const int i = (int)(t % G.n[0]);
  const int c = (int)(t / G.n[0]);
  const FabView P = pv[b];
  double* p = phi + P.off + c * P.cs + (int64_t)i * P.s0 + (int64_t)j * P.s1 + k;
  double v = *p;
  const int pad = 3 - dim;
  const double dts[3] = {dt0, dt1, dt2};
  for (int d = 0; d < dim; ++d) {
    const int ax = pad + d;
    int e[3] = {G.n[0], G.n[1], G.n[2]};
    e[ax] += 1;
    int x[3] = {i, j, k};
    const int64_t lo = (((int64_t)c * e[0] + x[0]) * e[1] + x[1]) * e[2] + x[2];
    x[ax] += 1;
    const int64_t hi = (((int64_t)c * e[0] + x[0]) * e[1] + x[1]) * e[2] + x[2];
    const double* fd = F.f[d] + F.off[d][b];
    v = v - dts[d] * (fd[hi] - fd[lo]);
  }
  *p = v;
}

// out = a * x + b * y over valid cells (fill_patch's time blend, coarse_fine.py:267-273).
__global__ void __launch_bounds__(kThreads)
    k_axpby(const int64_t* __restrict__ prefix, const int* __restrict__ boxes, int nb, const BoxGeom* __restrict__ geo,
            const FabView* __restrict__ ov, double* __restrict__ out, double a, const FabView* __restrict__ xv,
            const double* __restrict__ x, double bcoef, const FabView* __restrict__ yv, const double* __restrict__ y) {
  pdl_entry();
  const int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (g >= prefix[nb]) return;
  const int q = find_box(prefix, nb, g);
  const int b = boxes[q];
  const BoxGeom G = geo[b];
  int64_t t = g - prefix[q];
  const int k = (int)(t % G.n[2]);
  t /= G.n[2];
  const int j = (int)(t % G.n[1]);
  t /= G.n[1];
  const int i = (int)(t % G.n[0]);
  const int c = (int)(t / G.n[0]);
  auto at = [&](const FabView& V) { return V.off + c * V.cs + (int64_t)i * V.s0 + (int64_t)j * V.s1 + k; };
  const FabView O = ov[b], X = xv[b], Y = yv[b];
  out[at(O)] = a * x[at(X)] + bcoef * y[at(Y)];
}

__device__ __forceinline__ double minmod_slope(double c, double lo, double hi) {
  const double dl = c - lo, dr = hi - c;
  if (dl > 0.0 && dr > 0.0) return fmin(dl, dr);
  if (dl < 0.0 && dr < 0.0) return fmax(dl, dr);
  return 0.0;
}

__device__ __forceinline__ int floordiv(int a, int r) { return a >= 0 ? a / r : -((-a + r - 1) / r); }

// Interpolation of every cell of each fine box's GROWN box from the coarse
// stage (box j = coarsen(fine box j) grown by gc): pc or minmod-limited
// linear (interp_block, coarse_fine.py:60-99).
__global__ void __launch_bounds__(kThreads)
    k_interp(const int64_t* __restrict__ prefix, const int* __restrict__ boxes, int nb, const BoxGeom* __restrict__ fgeo,
             int3 fng, const FabView* __restrict__ fv, double* __restrict__ fine, const BoxGeom* __restrict__ cgeo,
             const FabView* __restrict__ cv, const double* __restrict__ crse, int ncomp, int dim, int r0, int r1,
             int r2, int linear) {
  pdl_entry();
  const int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (g >= prefix[nb]) return;
  const int q = find_box(prefix, nb, g);
  const int b = boxes[q];
  const BoxGeom G = fgeo[b];
  const int pad = 3 - dim;
  const int ng[3] = {fng.x, fng.y, fng.z};
  const int e0 = G.n[0] + 2 * ng[0], e1 = G.n[1] + 2 * ng[1], e2 = G.n[2] + 2 * ng[2];
  int64_t t = g - prefix[q];
  const int k = (int)(t % e2);
  t /= e2;
  const int j = (int)(t % e1);
  t /= e1;
  const int i = (int)(t % e0);
  const int c = (int)(t / e0);
  const int X[3] = {G.lo[0] - ng[0] + i, G.lo[1] - ng[1] + j, G.lo[2] - ng[2] + k};
  const int r[3] = {r0, r1, r2};
  int Pc[3];
  for (int a = 0; a < 3; ++a) Pc[a] = floordiv(X[a], r[a]);
  const BoxGeom C = cgeo[b];
  const FabView V = cv[b];
  auto cat = [&](int p0, int p1, int p2) {
    return crse[V.off + c * V.cs + (int64_t)(p0 - C.lo[0]) * V.s0 + (int64_t)(p1 - C.lo[1]) * V.s1 + (p2 - C.lo[2])];
  };
  const double core = cat(Pc[0], Pc[1], Pc[2]);
  double v = core;
  if (linear) {
    for (int d = 0; d < dim; ++d) {
      const int a = pad + d;
      int lo[3] = {Pc[0], Pc[1], Pc[2]}, hi[3] = {Pc[0], Pc[1], Pc[2]};
      lo[a] -= 1;
      hi[a] += 1;
      const double s = minmod_slope(core, cat(lo[0], lo[1], lo[2]), cat(hi[0], hi[1], hi[2]));
      const int m = X[a] - Pc[a] * r[a];
      const double off = ((double)m + 0.5) / (double)r[a] - 0.5;
      v = v + s * off;
    }
  }
  const FabView Fv = fv[b];
  fine[Fv.off + c * Fv.cs + (int64_t)(X[0] - G.lo[0]) * Fv.s0 + (int64_t)(X[1] - G.lo[1]) * Fv.s1 +
       (X[2] - G.lo[2])] = v;
}

// count NaNs in per-box regions (box-local valid coords, may reach into ghosts)
__global__ void __launch_bounds__(kThreads)
    k_nan_count(const int64_t* __restrict__ prefix, const int* __restrict__ boxes, int nb,
                const int* __restrict__ region, const FabView* __restrict__ fv, const double* __restrict__ x, int ncomp,
                unsigned long long* __restrict__ count) {
  pdl_entry();
  const int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (g >= prefix[nb]) return;
  const int q = find_box(prefix, nb, g);
  const int b = boxes[q];
  const int* R = region + 6 * q;
  const int e0 = R[3] - R[0] + 1, e1 = R[4] - R[1] + 1, e2 = R[5] - R[2] + 1;
  int64_t t = g - prefix[q];
  const int k = (int)(t % e2);
  t /= e2;
  const int j = (int)(t % e1);
  t /= e1;
  const int i = (int)(t % e0);
  const int c = (int)(t / e0);
  const FabView V = fv[b];
  const double v = x[V.off + c * V.cs + (int64_t)(R[0] + i) * V.s0 + (int64_t)(R[1] + j) * V.s1 + R[2] + k];
  if (v != v) atomicAdd(count, 1ull);
}

// register <- register - scale * F[src] (crse_add: one contribution per face)
__global__ void __launch_bounds__(kThreads)
    k_fr_crse(const int64_t* __restrict__ pairs, int64_t n, double* __restrict__ reg, const double* __restrict__ F,
              double scale) {
  pdl_entry();
  const int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (g >= n) return;
  const int64_t d = pairs[2 * g], s = pairs[2 * g + 1];
  reg[d] = reg[d] - scale * F[s];
}

// register <- register + scale * avg(fine faces) (fine_add).  nsrc = 2 (2-D):
// (a0 + a1) / 2; nsrc = 4 (3-D): ((a00 + a01) + (a10 + a11)) / 4, or
// (((a00 + a01) + a10) + a11) / 4 when numpy coalesces the two reduced axes
// (seq = 1: the coarse plane has one face along its last axis).
__global__ void __launch_bounds__(kThreads)
    k_fr_fine(const int64_t* __restrict__ idx, int64_t n, int nsrc, int seq, double* __restrict__ reg,
              const double* __restrict__ F, double scale) {
  pdl_entry();
  const int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (g >= n) return;
  const int64_t* e = idx + g * (1 + nsrc);
  double avg;
  if (nsrc == 1) {
    avg = F[e[1]];
  } else if (nsrc == 2) {
    avg = (F[e[1]] + F[e[2]]) / 2.0;
  } else {
    const double a00 = F[e[1]], a01 = F[e[2]], a10 = F[e[3]], a11 = F[e[4]];
    avg = (seq ? (((a00 + a01) + a10) + a11) : ((a00 + a01) + (a10 + a11))) / 4.0;
  }
  reg[e[0]] = reg[e[0]] + scale * avg;
}

// crse[target] += coef * reg[src] over each target's contributions in patch
// order (reflux, coarse_fine.py:428-472); CSR by target.
__global__ void __launch_bounds__(kThreads)
    k_fr_reflux(const int64_t* __restrict__ tgt, const int64_t* __restrict__ start, int64_t n,
                const int64_t* __restrict__ src, const double* __restrict__ coef, double* __restrict__ crse,
                const double* __restrict__ reg) {
  pdl_entry();
  const int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (g >= n) return;
  double v = crse[tgt[g]];
  for (int64_t e = start[g]; e < start[g + 1]; ++e) v = v + coef[e] * reg[src[e]];
  crse[tgt[g]] = v;
}

unsigned grid_of(int64_t n) { return (unsigned)std::max<int64_t>(1, (n + kThreads - 1) / kThreads); }

}  // namespace
}  // namespace amrb

using amrb::BoxGeom;
using amrb::FabView;
using amrb::Field;
using amrb::Level;

namespace {
const Level& LV(const amrb_level* p) {
  if (!p) throw amrb::Error(AMRB_EINVAL, "null level");
  return *reinterpret_cast<const Level*>(p);
}
const Field& FD(const amrb_field* p) {
  if (!p) throw amrb::Error(AMRB_EINVAL, "null field");
  return *reinterpret_cast<const Field*>(p);
}
}  // namespace

// Work lists come from the Python layer (amr.py): prefix = int64[nb+1] prefix
// of per-box work items over the resident boxes `boxes` (int32[nb]).
extern "C" int amrb_adv_flux(const amrb_level* lv, const amrb_field* phi_f, const double* phi, const int64_t* prefix,
                             const int32_t* boxes, int nb, int64_t total, const int64_t* face_off, double* flux,
                             int ncomp, int axis3, double u, void* stream) {
  return amrb::guarded([&] {
    if (nb < 1 || total < 1) return;
    amrb::launch_k(amrb::k_adv_flux, amrb::grid_of(total), amrb::kThreads, 0, (cudaStream_t)stream,
        prefix, boxes, nb, LV(lv).dgeo.p, FD(phi_f).dev.p, phi, face_off, flux, ncomp, axis3, u);
    amrb::check_launch("k_adv_flux");
  });
}

extern "C" int amrb_adv_update(const amrb_level* lv, const amrb_field* phi_f, double* phi, const int64_t* prefix,
                               const int32_t* boxes, int nb, int64_t total, const double* const* flux,
                               const int64_t* const* face_off, int ncomp, int dim, const double dtdx[3],
                               void* stream) {
  return amrb::guarded([&] {
    if (nb < 1 || total < 1) return;
    amrb::Faces F{};
    for (int d = 0; d < dim; ++d) {
      F.f[d] = flux[d];
      F.off[d] = face_off[d];
    }
    amrb::launch_k(amrb::k_adv_update, amrb::grid_of(total), amrb::kThreads, 0, (cudaStream_t)stream,
        prefix, boxes, nb, LV(lv).dgeo.p, FD(phi_f).dev.p, phi, F, ncomp, dim, dtdx[0], dtdx[1], dtdx[2]);
    amrb::check_launch("k_adv_update");
  });
}

extern "C" int amrb_axpby(const amrb_level* lv, const int64_t* prefix, const int32_t* boxes, int nb, int64_t total,
                          const amrb_field* out_f, double* out, double a, const amrb_field* x_f, const double* x,
                          double b, const amrb_field* y_f, const double* y, void* stream) {
  return amrb::guarded([&] {
    if (nb < 1 || total < 1) return;
    amrb::launch_k(amrb::k_axpby, amrb::grid_of(total), amrb::kThreads, 0, (cudaStream_t)stream,
        prefix, boxes, nb, LV(lv).dgeo.p, FD(out_f).dev.p, out, a, FD(x_f).dev.p, x, b, FD(y_f).dev.p, y);
    amrb::check_launch("k_axpby");
  });
}

extern "C" int amrb_interp(const amrb_level* fine_lv, const amrb_field* fine_f, double* fine,
                           const amrb_level* crse_lv, const amrb_field* crse_f, const double* crse,
                           const int64_t* prefix, const int32_t* boxes, int nb, int64_t total, int ncomp, int dim,
                           const int32_t ratio[3], int linear, void* stream) {
  return amrb::guarded([&] {
    if (nb < 1 || total < 1) return;
    const Field& ff = FD(fine_f);
    amrb::launch_k(amrb::k_interp, amrb::grid_of(total), amrb::kThreads, 0, (cudaStream_t)stream,
        prefix, boxes, nb, LV(fine_lv).dgeo.p, make_int3(ff.ng3[0], ff.ng3[1], ff.ng3[2]), ff.dev.p, fine,
        LV(crse_lv).dgeo.p, FD(crse_f).dev.p, crse, ncomp, dim, ratio[0], ratio[1], ratio[2], linear);
    amrb::check_launch("k_interp");
  });
}

extern "C" int amrb_nan_count(const amrb_field* f, const double* x, const int64_t* prefix, const int32_t* boxes,
                              int nb, int64_t total, const int32_t* region, int ncomp, unsigned long long* dev_count,
                              void* stream) {
  return amrb::guarded([&] {
    if (nb < 1 || total < 1) return;
    amrb::launch_k(amrb::k_nan_count, amrb::grid_of(total), amrb::kThreads, 0, (cudaStream_t)stream,
        prefix, boxes, nb, region, FD(f).dev.p, x, ncomp, dev_count);
    amrb::check_launch("k_nan_count");
  });
}

extern "C" int amrb_fr_crse(const int64_t* pairs, int64_t n, double* reg, const double* flux, double scale,
                            void* stream) {
  return amrb::guarded([&] {
    if (n < 1) return;
    amrb::launch_k(amrb::k_fr_crse, amrb::grid_of(n), amrb::kThreads, 0, (cudaStream_t)stream, pairs, n, reg, flux, scale);
    amrb::check_launch("k_fr_crse");
  });
}

extern "C" int amrb_fr_fine(const int64_t* idx, int64_t n, int nsrc, int seq, double* reg, const double* flux,
                            double scale, void* stream) {
  return amrb::guarded([&] {
    if (n < 1) return;
    if (nsrc != 1 && nsrc != 2 && nsrc != 4) throw amrb::Error(AMRB_EINVAL, "amrb_fr_fine: nsrc must be 1, 2 or 4");
    amrb::launch_k(amrb::k_fr_fine, amrb::grid_of(n), amrb::kThreads, 0, (cudaStream_t)stream, idx, n, nsrc, seq, reg, flux,
                                                                                   scale);
    amrb::check_launch("k_fr_fine");
  });
}

extern "C" int amrb_fr_reflux(const int64_t* tgt, const int64_t* start, int64_t n, const int64_t* src,
                              const double* coef, double* crse, const double* reg, void* stream) {
  return amrb::guarded([&] {
    if (n < 1) return;
    amrb::launch_k(amrb::k_fr_reflux, amrb::grid_of(n), amrb::kThreads, 0, (cudaStream_t)stream, tgt, start, n, src, coef, crse,
                                                                                     reg);
    amrb::check_launch("k_fr_reflux");
  });
}
