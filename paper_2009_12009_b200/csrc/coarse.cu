// Coarse tail of the MLMG V-cycle in one CTA.
//
// Below the box-local levels the hierarchy is a chain of single-box periodic
// levels (the agglomerated domain, 16^3 .. 4^3 for the configs here).  Each of
// them is a few KB, so launching fill + sweep kernels for them is pure launch
// latency (the bottom alone was 64 launches per V-cycle).  This kernel keeps
// every tail level in shared memory and runs the whole sub-cycle -- nu1
// sweeps, residual + restriction, the bottom sweeps, pc prolongation + nu2
// sweeps -- with __syncthreads between phases.
//
// Exactness: the periodic ghost fill of a single box is a copy of the wrapped
// valid cell (only the 6 faces are filled: the 7-point operator reads nothing
// else), and every update uses the shared lap7 / relax / avg8 expressions,
// so results are bit-identical to the oracle's fill / red / fill / black
// sequence (oracle/mlmg_ref.py) and to the device multi-kernel path.
#include <cooperative_groups.h>

#include <cstdlib>
#include <cstring>
#include <algorithm>

#include "stencil_common.cuh"

namespace amrb {

namespace {

constexpr int kMaxTail = 8;
constexpr int kTailThreads = 1024;

struct TailLevel {
  int n[3];
  int lo_par;        // (lo0 + lo1 + lo2) & 1
  int phi_off;       // doubles, into smem: (n0+2)(n1+2)(n2+2) with one ghost layer
  int rhs_off;       // doubles: n0 n1 n2
  Coef cf;
};

struct TailArgs {
  int nlev;
  TailLevel lv[kMaxTail];
  int nu1, nu2, nbottom;
  int warp_from;  // first level small enough for one warp
  const double* rhs;  // level 0 rhs (valid lo cell)
  int64_t rs0, rs1;
  double* phi;        // level 0 phi (valid lo cell)
  int64_t ps0, ps1;
};

__device__ __forceinline__ double avg8t(const double* v) {
  return ((((v[0] + v[1]) + (v[2] + v[3])) + (v[4] + v[5])) + (v[6] + v[7])) * 0.125;
}

__global__ void __launch_bounds__(kTailThreads, 1) k_coarse_tail(TailArgs a) {
  pdl_entry();
  extern __shared__ __align__(16) double sm[];
  // Levels >= a.warp_from are tiny (<= 512 cells): warp 0 runs their whole
  // sub-cycle with __syncwarp while the other warps wait at one barrier.
  bool wmode = false;
  int t = threadIdx.x, nt = kTailThreads;
  auto sync = [&]() {
    if (wmode)
      __syncwarp();
    else
      __syncthreads();
  };

  auto P = [&](const TailLevel& L) { return sm + L.phi_off; };
  auto Rr = [&](const TailLevel& L) { return sm + L.rhs_off; };
  auto pidx = [](const TailLevel& L, int i, int j, int k) {
    return ((i + 1) * (L.n[1] + 2) + (j + 1)) * (L.n[2] + 2) + (k + 1);
  };
  auto ridx = [](const TailLevel& L, int i, int j, int k) { return (i * L.n[1] + j) * L.n[2] + k; };

  auto fill_faces = [&](const TailLevel& L) {
    double* p = P(L);
    const int n0 = L.n[0], n1 = L.n[1], n2 = L.n[2];
    const int f0 = n1 * n2, f1 = n0 * n2, f2 = n0 * n1;
    const int tot = 2 * (f0 + f1 + f2);
    for (int e = t; e < tot; e += nt) {
      int x = e;
      if (x < 2 * f0) {
        const int side = x / f0;
        x -= side * f0;
        const int j = x / n2, k = x - j * n2;
        p[pidx(L, side ? n0 : -1, j, k)] = p[pidx(L, side ? 0 : n0 - 1, j, k)];
        continue;
      }
      x -= 2 * f0;
      if (x < 2 * f1) {
        const int side = x / f1;
        x -= side * f1;
        const int i = x / n2, k = x - i * n2;
        p[pidx(L, i, side ? n1 : -1, k)] = p[pidx(L, i, side ? 0 : n1 - 1, k)];
        continue;
      }
      x -= 2 * f1;
      const int side = x / f2;
      x -= side * f2;
      const int i = x / n1, j = x - i * n1;
      p[pidx(L, i, j, side ? n2 : -1)] = p[pidx(L, i, j, side ? 0 : n2 - 1)];
    }
  };
  auto color = [&](const TailLevel& L, int c) {
    double* p = P(L);
    const double* r = Rr(L);
    const int n0 = L.n[0], n1 = L.n[1], n2 = L.n[2];
    const int sj = n2 + 2, si = (n1 + 2) * sj;
    const int h = (n2 + 1) / 2;
    const int np = n0 * n1 * h;
    for (int e = t; e < np; e += nt) {
      const int ij = e / h, kp = e - ij * h;
      const int i = ij / n1, j = ij - i * n1;
      const int k = 2 * kp + ((L.lo_par + i + j + c) & 1);
      if (k >= n2) continue;
      const int o = pidx(L, i, j, k);
      const double v = p[o];
      const double lap = lap7(v, p[o - si], p[o + si], p[o - sj], p[o + sj], p[o - 1], p[o + 1], L.cf);
      p[o] = relax(v, r[ridx(L, i, j, k)], lap, L.cf.rgamma);
    }
  };
  auto smooth = [&](const TailLevel& L, int n) {
    for (int s = 0; s < n; ++s)
      for (int c = 0; c < 2; ++c) {
        fill_faces(L);
        sync();
        color(L, c);
        sync();
      }
  };
  auto zero_phi = [&](const TailLevel& L) {
    double* p = P(L);
    const int tot = (L.n[0] + 2) * (L.n[1] + 2) * (L.n[2] + 2);
    for (int e = t; e < tot; e += nt) p[e] = 0.0;
  };
  auto restrict_resid = [&](const TailLevel& L, const TailLevel& C) {
    const double* p = P(L);
    const double* r = Rr(L);
    double* rc = Rr(C);
    const int sj = L.n[2] + 2, si = (L.n[1] + 2) * sj;
    const int tot = C.n[0] * C.n[1] * C.n[2];
    for (int e = t; e < tot; e += nt) {
      const int IJ = e / C.n[2], K = e - IJ * C.n[2];
      const int I = IJ / C.n[1], J = IJ - I * C.n[1];
      double v[8];
#pragma unroll
      for (int di = 0; di < 2; ++di)
#pragma unroll
        for (int dj = 0; dj < 2; ++dj)
#pragma unroll
          for (int dk = 0; dk < 2; ++dk) {
            const int i = 2 * I + di, j = 2 * J + dj, k = 2 * K + dk;
            const int o = pidx(L, i, j, k);
            const double c0 = p[o];
            v[di * 4 + dj * 2 + dk] =
                r[ridx(L, i, j, k)] - lap7(c0, p[o - si], p[o + si], p[o - sj], p[o + sj], p[o - 1], p[o + 1], L.cf);
          }
      rc[e] = avg8t(v);
    }
  };
  auto prolong_add = [&](const TailLevel& L, const TailLevel& C) {
    double* p = P(L);
    const double* pc = P(C);
    const int tot = L.n[0] * L.n[1] * L.n[2];
    for (int e = t; e < tot; e += nt) {
      const int ij = e / L.n[2], k = e - ij * L.n[2];
      const int i = ij / L.n[1], j = ij - i * L.n[1];
      const int o = pidx(L, i, j, k);
      p[o] = p[o] + pc[pidx(C, i >> 1, j >> 1, k >> 1)];
    }
  };
  // down-sweep of levels [l0, nl): level l0's rhs is ready
  auto down = [&](int l0, int nl) {
    for (int l = l0; l < nl; ++l) {
      const TailLevel& L = a.lv[l];
      zero_phi(L);
      sync();
      if (l == a.nlev - 1) {
        smooth(L, a.nbottom);
        return;
      }
      smooth(L, a.nu1);
      fill_faces(L);
      sync();
      restrict_resid(L, a.lv[l + 1]);
      sync();
    }
  };
  auto up = [&](int from, int to) {  // levels from .. to (descending), each prolonged from the next
    for (int l = from; l >= to; --l) {
      prolong_add(a.lv[l], a.lv[l + 1]);
      sync();
      smooth(a.lv[l], a.nu2);
    }
  };

  {  // load level-0 rhs
    const TailLevel& L = a.lv[0];
    double* r = Rr(L);
    const int tot = L.n[0] * L.n[1] * L.n[2];
    for (int e = t; e < tot; e += nt) {
      const int ij = e / L.n[2], k = e - ij * L.n[2];
      const int i = ij / L.n[1], j = ij - i * L.n[1];
      r[e] = a.rhs[i * a.rs0 + j * a.rs1 + k];
    }
  }
  __syncthreads();
  const int wf = a.warp_from;  // first tiny level (nlev if none)
  down(0, wf);
  if (wf < a.nlev) {
    __syncthreads();
    if (threadIdx.x < 32) {
      wmode = true;
      nt = 32;
      down(wf, a.nlev);
      up(a.nlev - 2, wf);
      wmode = false;
      nt = kTailThreads;
    }
    __syncthreads();
  }
  up(min(wf, a.nlev - 1) - 1, 0);
  __syncthreads();
  {  // store level-0 phi (valid)
    const TailLevel& L = a.lv[0];
    const double* p = P(L);
    const int tot = L.n[0] * L.n[1] * L.n[2];
    for (int e = t; e < tot; e += nt) {
      const int ij = e / L.n[2], k = e - ij * L.n[2];
      const int i = ij / L.n[1], j = ij - i * L.n[1];
      a.phi[i * a.ps0 + j * a.ps1 + k] = p[pidx(L, i, j, k)];
    }
  }
}


// ---------------------------------------------------------------------------
// Power-of-two cubic tails (16^3 .. 4^3 in the configs): no ghost cells at
// all -- the periodic neighbour of (i-1) is ((i-1) & (n-1)), which reads the
// very value a ghost fill would have copied, so the result is unchanged while
// every fill phase (and its barrier) disappears.  Each level runs with just
// enough threads (one per cell of a colour, capped at the block) and syncs on
// a named barrier sized to them (one warp: __syncwarp).
// ---------------------------------------------------------------------------
// GIO: level-0 rhs comes from / phi goes to global memory (false: both stay
// in shared memory, the cluster kernel below owns them).  base: first TailArgs
// level this body runs (its level 0).
template <int LOG0, bool GIO>
__device__ __forceinline__ void tail_p2_body(const TailArgs& a, double* sm, int base) {
  const int tid = threadIdx.x;
  // level l: n = 1 << (LOG0 - l); phi and rhs dense n^3 at smem offsets
  auto cells = [](int l) { return 1 << (3 * (LOG0 - l)); };
  auto nact = [&](int l) { return min(kTailThreads, max(32, cells(l) / 2)); };
  auto lsync = [&](int l) {
    const int na = nact(l);
    if (na == 32)
      __syncwarp();
    else if (na == kTailThreads)
      __syncthreads();
    else
      asm volatile("bar.sync 1, %0;\n" ::"r"(na) : "memory");
  };
  auto PHI = [&](int l) { return sm + a.lv[base + l].phi_off; };
  auto RHS = [&](int l) { return sm + a.lv[base + l].rhs_off; };

  auto color = [&](int l, int c) {
    const int s = LOG0 - l, n = 1 << s, m = n - 1;
    double* p = PHI(l);
    const double* r = RHS(l);
    const Coef cf = a.lv[base + l].cf;
    const int lp = a.lv[base + l].lo_par;
    const int np = cells(l) / 2;
    for (int e = tid; e < np; e += nact(l)) {
      const int kp = e & ((n >> 1) - 1), ij = e >> (s - 1);
      const int j = ij & m, i = ij >> s;
      const int k = 2 * kp + ((lp + i + j + c) & 1);
      const int o = (i << (2 * s)) | (j << s) | k;
      const double v = p[o];
      const double lap = lap7(v, p[(((i - 1) & m) << (2 * s)) | (j << s) | k], p[(((i + 1) & m) << (2 * s)) | (j << s) | k],
                              p[(i << (2 * s)) | (((j - 1) & m) << s) | k], p[(i << (2 * s)) | (((j + 1) & m) << s) | k],
                              p[(i << (2 * s)) | (j << s) | ((k - 1) & m)], p[(i << (2 * s)) | (j << s) | ((k + 1) & m)], cf);
      p[o] = relax(v, r[o], lap, cf.rgamma);
    }
  };
  auto smooth = [&](int l, int nsw) {
    for (int q = 0; q < nsw; ++q) {
      color(l, 0);
      lsync(l);
      color(l, 1);
      lsync(l);
    }
  };
  auto restrict_resid = [&](int l) {  // rhs_{l+1} = avg8(rhs_l - L phi_l)
    const int s = LOG0 - l, m = (1 << s) - 1, cs = s - 1;
    const double* p = PHI(l);
    const double* r = RHS(l);
    double* rc = RHS(l + 1);
    const Coef cf = a.lv[base + l].cf;
    for (int e = tid; e < cells(l + 1); e += nact(l)) {
      const int K = e & ((1 << cs) - 1), J = (e >> cs) & ((1 << cs) - 1), I = e >> (2 * cs);
      double v[8];
#pragma unroll
      for (int di = 0; di < 2; ++di)
#pragma unroll
        for (int dj = 0; dj < 2; ++dj)
#pragma unroll
          for (int dk = 0; dk < 2; ++dk) {
            const int i = 2 * I + di, j = 2 * J + dj, k = 2 * K + dk;
            const int o = (i << (2 * s)) | (j << s) | k;
            const double c0 = p[o];
            v[di * 4 + dj * 2 + dk] =
                r[o] - lap7(c0, p[(((i - 1) & m) << (2 * s)) | (j << s) | k], p[(((i + 1) & m) << (2 * s)) | (j << s) | k],
                            p[(i << (2 * s)) | (((j - 1) & m) << s) | k], p[(i << (2 * s)) | (((j + 1) & m) << s) | k],
                            p[(i << (2 * s)) | (j << s) | ((k - 1) & m)], p[(i << (2 * s)) | (j << s) | ((k + 1) & m)], cf);
          }
      rc[e] = avg8t(v);
    }
  };
  auto prolong_add = [&](int l) {  // phi_l += phi_{l+1}(parent)
    const int s = LOG0 - l, cs = s - 1;
    double* p = PHI(l);
    const double* pc = PHI(l + 1);
    for (int e = tid; e < cells(l); e += nact(l)) {
      const int k = e & ((1 << s) - 1), j = (e >> s) & ((1 << s) - 1), i = e >> (2 * s);
      p[e] = p[e] + pc[((i >> 1) << (2 * cs)) | ((j >> 1) << cs) | (k >> 1)];
    }
  };
  auto zero = [&](int l) {
    double* p = PHI(l);
    for (int e = tid; e < cells(l); e += nact(l)) p[e] = 0.0;
  };

  if (GIO) {  // level-0 rhs from global
    const int s = LOG0, n = 1 << s;
    double* r = RHS(0);
    for (int e = tid; e < cells(0); e += kTailThreads) {
      const int k = e & (n - 1), j = (e >> s) & (n - 1), i = e >> (2 * s);
      r[e] = a.rhs[i * a.rs0 + j * a.rs1 + k];
    }
  }
  __syncthreads();
  const int L = a.nlev - base;
  for (int l = 0; l < L; ++l) {
    if (tid < nact(l)) {
      zero(l);
      lsync(l);
      if (l == L - 1) {
        smooth(l, a.nbottom);
      } else {
        smooth(l, a.nu1);
        restrict_resid(l);
      }
    }
    __syncthreads();
  }
  for (int l = L - 2; l >= 0; --l) {
    if (tid < nact(l)) {
      prolong_add(l);
      lsync(l);
      smooth(l, a.nu2);
    }
    __syncthreads();
  }
  if (GIO) {  // level-0 phi to global
    const int s = LOG0, n = 1 << s;
    const double* p = PHI(0);
    for (int e = tid; e < cells(0); e += kTailThreads) {
      const int k = e & (n - 1), j = (e >> s) & (n - 1), i = e >> (2 * s);
      a.phi[i * a.ps0 + j * a.ps1 + k] = p[e];
    }
  }
}

template <int LOG0>
__global__ void __launch_bounds__(kTailThreads, 1) k_coarse_tail_p2(TailArgs a) {
  pdl_entry();
  extern __shared__ __align__(16) double sm[];
  tail_p2_body<LOG0, true>(a, sm, 0);
}

// Power-of-two but not cubic tails (the multi-GPU weak-scaling domains give
// 32x16x16 .. 8x4x4 at 2 GPUs, 32x32x16 .. at 4): the same masked periodic
// indexing with one shift per axis (every extent >= 2 and halving per level).
// Replaces the generic fill-based k_coarse_tail there (103 us -> ~30 us).
// GIO / base as for tail_p2_body.
template <bool GIO>
__device__ __forceinline__ void tail_p2x_body(const TailArgs& a, double* sm, int base) {
  const int tid = threadIdx.x;
  auto sh = [&](int l, int x) { return __ffs(a.lv[base + l].n[x]) - 1; };
  auto cells = [&](int l) { return 1 << (sh(l, 0) + sh(l, 1) + sh(l, 2)); };
  auto nact = [&](int l) { return min(kTailThreads, max(32, cells(l) / 2)); };
  auto lsync = [&](int l) {
    const int na = nact(l);
    if (na == 32)
      __syncwarp();
    else if (na == kTailThreads)
      __syncthreads();
    else
      asm volatile("bar.sync 1, %0;\n" ::"r"(na) : "memory");
  };
  auto PHI = [&](int l) { return sm + a.lv[base + l].phi_off; };
  auto RHS = [&](int l) { return sm + a.lv[base + l].rhs_off; };
  // masked periodic 7-point Laplacian at (i, j, k) of a level with shifts s1, s2
  // and masks m0, m1, m2
  auto lapm = [&](const double* p, int i, int j, int k, int s1, int s2, int m0, int m1, int m2, const Coef& cf) {
    const int si = s1 + s2;
    return lap7(p[(i << si) | (j << s2) | k], p[(((i - 1) & m0) << si) | (j << s2) | k],
                p[(((i + 1) & m0) << si) | (j << s2) | k], p[(i << si) | (((j - 1) & m1) << s2) | k],
                p[(i << si) | (((j + 1) & m1) << s2) | k], p[(i << si) | (j << s2) | ((k - 1) & m2)],
                p[(i << si) | (j << s2) | ((k + 1) & m2)], cf);
  };

  auto color = [&](int l, int c) {
    const int s1 = sh(l, 1), s2 = sh(l, 2);
    const int m0 = a.lv[base + l].n[0] - 1, m1 = a.lv[base + l].n[1] - 1, m2 = a.lv[base + l].n[2] - 1;
    double* p = PHI(l);
    const double* r = RHS(l);
    const Coef cf = a.lv[base + l].cf;
    const int lp = a.lv[base + l].lo_par;
    const int np = cells(l) / 2;
    for (int e = tid; e < np; e += nact(l)) {
      const int kp = e & ((1 << (s2 - 1)) - 1), ij = e >> (s2 - 1);
      const int j = ij & m1, i = ij >> s1;
      const int k = 2 * kp + ((lp + i + j + c) & 1);
      const int o = (i << (s1 + s2)) | (j << s2) | k;
      const double v = p[o];
      const double lap = lapm(p, i, j, k, s1, s2, m0, m1, m2, cf);
      p[o] = relax(v, r[o], lap, cf.rgamma);
    }
  };
  auto smooth = [&](int l, int nsw) {
    for (int q = 0; q < nsw; ++q) {
      color(l, 0);
      lsync(l);
      color(l, 1);
      lsync(l);
    }
  };
  auto restrict_resid = [&](int l) {  // rhs_{l+1} = avg8(rhs_l - L phi_l)
    const int s1 = sh(l, 1), s2 = sh(l, 2), c1 = s1 - 1, c2 = s2 - 1;
    const int m0 = a.lv[base + l].n[0] - 1, m1 = a.lv[base + l].n[1] - 1, m2 = a.lv[base + l].n[2] - 1;
    const double* p = PHI(l);
    const double* r = RHS(l);
    double* rc = RHS(l + 1);
    const Coef cf = a.lv[base + l].cf;
    for (int e = tid; e < cells(l + 1); e += nact(l)) {
      const int K = e & ((1 << c2) - 1), J = (e >> c2) & ((1 << c1) - 1), I = e >> (c1 + c2);
      double v[8];
#pragma unroll
      for (int di = 0; di < 2; ++di)
#pragma unroll
        for (int dj = 0; dj < 2; ++dj)
#pragma unroll
          for (int dk = 0; dk < 2; ++dk) {
            const int i = 2 * I + di, j = 2 * J + dj, k = 2 * K + dk;
            const int o = (i << (s1 + s2)) | (j << s2) | k;
            v[di * 4 + dj * 2 + dk] = r[o] - lapm(p, i, j, k, s1, s2, m0, m1, m2, cf);
          }
      rc[e] = avg8t(v);
    }
  };
  auto prolong_add = [&](int l) {  // phi_l += phi_{l+1}(parent)
    const int s1 = sh(l, 1), s2 = sh(l, 2), c1 = s1 - 1, c2 = s2 - 1;
    double* p = PHI(l);
    const double* pc = PHI(l + 1);
    for (int e = tid; e < cells(l); e += nact(l)) {
      const int k = e & ((1 << s2) - 1), j = (e >> s2) & ((1 << s1) - 1), i = e >> (s1 + s2);
      p[e] = p[e] + pc[((i >> 1) << (c1 + c2)) | ((j >> 1) << c2) | (k >> 1)];
    }
  };
  auto zero = [&](int l) {
    double* p = PHI(l);
    for (int e = tid; e < cells(l); e += nact(l)) p[e] = 0.0;
  };

  if (GIO) {
    const int s1 = sh(0, 1), s2 = sh(0, 2);
    double* r = RHS(0);
    for (int e = tid; e < cells(0); e += kTailThreads) {
      const int k = e & ((1 << s2) - 1), j = (e >> s2) & ((1 << s1) - 1), i = e >> (s1 + s2);
      r[e] = a.rhs[i * a.rs0 + j * a.rs1 + k];
    }
  }
  __syncthreads();
  const int L = a.nlev - base;
  for (int l = 0; l < L; ++l) {
    if (tid < nact(l)) {
      zero(l);
      lsync(l);
      if (l == L - 1) {
        smooth(l, a.nbottom);
      } else {
        smooth(l, a.nu1);
        restrict_resid(l);
      }
    }
    __syncthreads();
  }
  for (int l = L - 2; l >= 0; --l) {
    if (tid < nact(l)) {
      prolong_add(l);
      lsync(l);
      smooth(l, a.nu2);
    }
    __syncthreads();
  }
  if (GIO) {
    const int s1 = sh(0, 1), s2 = sh(0, 2);
    const double* p = PHI(0);
    for (int e = tid; e < cells(0); e += kTailThreads) {
      const int k = e & ((1 << s2) - 1), j = (e >> s2) & ((1 << s1) - 1), i = e >> (s1 + s2);
      a.phi[i * a.ps0 + j * a.ps1 + k] = p[e];
    }
  }
}

__global__ void __launch_bounds__(kTailThreads, 1) k_coarse_tail_p2x(TailArgs a) {
  pdl_entry();
  extern __shared__ __align__(16) double sm[];
  tail_p2x_body<true>(a, sm, 0);
}

// ---------------------------------------------------------------------------
// 32^3 top level + 16^3 .. tail in ONE cluster of 8 CTAs.  The 32^3 level
// (phi + rhs = 512 KB) does not fit one CTA, but it does fit a cluster: CTA r
// holds planes [4r, 4r+4) of phi and rhs in its shared memory and reads the
// two neighbouring planes (4r-1, 4r+4, periodic) from its cluster peers'
// shared memory (DSMEM); cluster barriers separate the colours.  The
// restriction writes the 16^3 rhs straight into CTA 0's shared memory, CTA 0
// runs the power-of-two tail body on it, and every CTA prolongs from CTA 0's
// 16^3 phi.  The 32^3 phi leaves with its width-1 periodic ghost layer
// written, so the next finer level's fused prolongation sweep needs no fill.
// This replaces 16 launches per V-cycle (fills, sweeps, residual-restrict,
// gather copies, prolongation at 32^3) with one.  Same lap7 / relax / avg8
// operand order as every other path: bit-identical results.
// ---------------------------------------------------------------------------
constexpr int kClCtas = 8;
constexpr int kClN = 32;                  // top-level extent along i
constexpr int kClPl = kClN / kClCtas;     // planes per CTA

// The top level may also be 32 x n1 x n2 with n1, n2 powers of two <= 32 (the
// multi-GPU weak-scaling chains 32x16x16 .. and 32x32x16 ..): planes are
// n1 x n2, indexed with shifts s1, s2; CTA 0 then runs the non-cubic chain
// body (tail_p2x_body) on the levels below.
// CUBIC: 32^3 top level with compile-time plane shifts (the default path).
template <bool CUBIC>
__global__ void __cluster_dims__(kClCtas, 1, 1) __launch_bounds__(kTailThreads, 1)
    k_coarse_tail_cl(TailArgs a, int slab_off, int cubic) {
  pdl_entry();
  extern __shared__ __align__(16) double sm[];
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int r = (int)cl.block_rank();
  const int tid = threadIdx.x;
  const TailLevel& L = a.lv[0];
  const int s1 = CUBIC ? 5 : __ffs(L.n[1]) - 1, s2 = CUBIC ? 5 : __ffs(L.n[2]) - 1, si = s1 + s2;
  const int m1 = (1 << s1) - 1, m2 = (1 << s2) - 1;
  const int c1 = s1 - 1, c2 = s2 - 1;  // next level's shifts
  const int plane = 1 << si, slab = kClPl << si;
  double* p = sm + slab_off;  // phi [kClPl][n1][n2]
  double* rh = p + slab;      // rhs, same shape
  const double* pm = cl.map_shared_rank(p, (r + kClCtas - 1) % kClCtas) + (kClPl - 1) * plane;  // plane 4r-1
  const double* pp = cl.map_shared_rank(p, (r + 1) % kClCtas);                                   // plane 4r+4
  const Coef cf = L.cf;
  const int i0 = kClPl * r;

  for (int e = tid; e < slab; e += kTailThreads) {
    const int k = e & m2, j = (e >> s2) & m1, li = e >> si;
    rh[e] = a.rhs[(int64_t)(i0 + li) * a.rs0 + (int64_t)j * a.rs1 + k];
    p[e] = 0.0;
  }
  cl.sync();

  auto at = [&](int li, int j, int k) { return p[(li << si) | (j << s2) | k]; };
  auto color = [&](int c) {
    for (int e = tid; e < slab / 2; e += kTailThreads) {
      const int kp = e & ((1 << c2) - 1), j = (e >> c2) & m1, li = e >> (si - 1);
      const int k = 2 * kp + ((L.lo_par + i0 + li + j + c) & 1);
      const int jk = (j << s2) | k;
      const int o = (li << si) | jk;
      const double v = p[o];
      const double xm = li > 0 ? p[o - plane] : pm[jk];
      const double xp = li < kClPl - 1 ? p[o + plane] : pp[jk];
      const double lap = lap7(v, xm, xp, at(li, (j - 1) & m1, k), at(li, (j + 1) & m1, k), at(li, j, (k - 1) & m2),
                              at(li, j, (k + 1) & m2), cf);
      p[o] = relax(v, rh[o], lap, cf.rgamma);
    }
  };
  auto smooth = [&](int nsw) {
    for (int q = 0; q < nsw; ++q) {
      color(0);
      cl.sync();
      color(1);
      cl.sync();
    }
  };

  smooth(a.nu1);
  {  // rhs_c = avg8(rhs - L phi), coarse planes [2r, 2r+2), into CTA 0
    double* rc = cl.map_shared_rank(sm + a.lv[1].rhs_off, 0);
    for (int e = tid; e < slab / 8; e += kTailThreads) {
      const int K = e & ((1 << c2) - 1), J = (e >> c2) & ((1 << c1) - 1), dI = e >> (c1 + c2);
      double v[8];
#pragma unroll
      for (int di = 0; di < 2; ++di)
#pragma unroll
        for (int dj = 0; dj < 2; ++dj)
#pragma unroll
          for (int dk = 0; dk < 2; ++dk) {
            const int li = 2 * dI + di, j = 2 * J + dj, k = 2 * K + dk;
            const int jk = (j << s2) | k;
            const int o = (li << si) | jk;
            const double xm = li > 0 ? p[o - plane] : pm[jk];
            const double xp = li < kClPl - 1 ? p[o + plane] : pp[jk];
            v[di * 4 + dj * 2 + dk] = rh[o] - lap7(p[o], xm, xp, at(li, (j - 1) & m1, k), at(li, (j + 1) & m1, k),
                                                   at(li, j, (k - 1) & m2), at(li, j, (k + 1) & m2), cf);
          }
      rc[((i0 / 2 + dI) << (c1 + c2)) | (J << c2) | K] = avg8t(v);
    }
  }
  cl.sync();
  if (r == 0) {
    if (CUBIC || cubic)
      tail_p2_body<4, false>(a, sm, 1);
    else
      tail_p2x_body<false>(a, sm, 1);
  }
  cl.sync();
  {  // phi += phi_c(parent), from CTA 0
    const double* pc = cl.map_shared_rank(sm + a.lv[1].phi_off, 0);
    for (int e = tid; e < slab; e += kTailThreads) {
      const int k = e & m2, j = (e >> s2) & m1, li = e >> si;
      p[e] = p[e] + pc[(((i0 + li) >> 1) << (c1 + c2)) | ((j >> 1) << c2) | (k >> 1)];
    }
  }
  cl.sync();
  smooth(a.nu2);
  // valid cells + the width-1 periodic ghost layer (the full grown box, as a
  // width-1 FillBoundary of a single periodic box writes it)
  const int E1 = m1 + 3, E2 = m2 + 3;
  for (int e = tid; e < kClPl * E1 * E2; e += kTailThreads) {
    const int kk = e % E2, jj = (e / E2) % E1, li = e / (E1 * E2);
    const int j = jj - 1, k = kk - 1;
    const double v = at(li, j & m1, k & m2);
    const int64_t jko = (int64_t)j * a.ps1 + k;
    a.phi[(int64_t)(i0 + li) * a.ps0 + jko] = v;
    if (i0 + li == 0) a.phi[(int64_t)kClN * a.ps0 + jko] = v;
    if (i0 + li == kClN - 1) a.phi[-a.ps0 + jko] = v;
  }
}

// ---------------------------------------------------------------------------
// One small single-box periodic level's half of the V-cycle in ONE grid-
// synchronised launch (cooperative: every CTA resident, grid.sync() between
// phases).  Down: zero phi, nu1 in-place GSRB sweeps (red, sync, black,
// sync), rhs_c = avg8(rhs - L phi) into the next coarser level.  Up: phi +=
// phi_c(parent), nu2 sweeps, then the width-1 periodic ghost layer.  The
// periodic neighbour is read by index wrap (the cell a ghost fill would have
// copied), so no fill kernels run; the level stays in L2 (64^3: 2 MB phi).
// Replaces per sweep a fill + a sweep launch (~15 us of launch-latency-bound
// work at 64^3) with two grid barriers.  Same lap7 / relax / avg8 operand
// order: bit-identical to the multi-kernel path and the oracle.
// ---------------------------------------------------------------------------
struct GridLevelArgs {
  int n0, n1, n2, lo_par, nsw, up;
  int l1, l2;  // log2(n1), log2(n2) when powers of two, else -1 (index math by shifts)
  Coef cf;
  double* phi;  // valid lo cell
  int ps0, ps1;  // 32-bit strides: these levels are small (checked on the host)
  const double* rhs;
  int rs0, rs1;
  double* c;  // down: coarse rhs (written); up: coarse phi (read); valid lo cell
  int cs0, cs1;
};

// e -> (e / n, e % n): shifts when n = 2^l
__device__ __forceinline__ void divmod(int e, int n, int l, int& q, int& r) {
  if (l >= 0) {
    q = e >> l;
    r = e & (n - 1);
  } else {
    q = e / n;
    r = e - q * n;
  }
}

// One single-box periodic level's half V-cycle, cooperative: every phase is a
// grid-stride loop, phases separated by grid.sync.  The level (<= 2^20 cells)
// lives in L2, so a phase is bound by gather latency: each thread works on
// kU cells at once with all their loads issued before any arithmetic.
constexpr int kU = 4;

__global__ void __launch_bounds__(512, 1) k_level_grid(GridLevelArgs a) {
  pdl_entry();
  namespace cg = cooperative_groups;
  cg::grid_group g = cg::this_grid();
  const int nt = (int)gridDim.x * blockDim.x;
  const int t0 = (int)blockIdx.x * blockDim.x + threadIdx.x;
  const int n0 = a.n0, n1 = a.n1, n2 = a.n2, h = n2 >> 1;
  const int lh = a.l2 > 0 ? a.l2 - 1 : -1;
  const int ncell = (int)n0 * n1 * n2;
  double* const p = a.phi;
  auto P = [&](int i, int j, int k) -> double& { return p[i * a.ps0 + j * a.ps1 + k]; };
  // the 7-point operator at (i, j, k) with periodic wrap; operands first
  struct Nb {
    double c, xm, xp, ym, yp, zm, zp;
  };
  auto load = [&](int i, int j, int k) {
    const int im = i ? i - 1 : n0 - 1, ip = i + 1 < n0 ? i + 1 : 0;
    const int jm = j ? j - 1 : n1 - 1, jp = j + 1 < n1 ? j + 1 : 0;
    const int km = k ? k - 1 : n2 - 1, kp = k + 1 < n2 ? k + 1 : 0;
    return Nb{P(i, j, k), P(im, j, k), P(ip, j, k), P(i, jm, k), P(i, jp, k), P(i, j, km), P(i, j, kp)};
  };
  auto lapn = [&](const Nb& n) { return lap7(n.c, n.xm, n.xp, n.ym, n.yp, n.zm, n.zp, a.cf); };
  auto cell = [&](int e, int& i, int& j, int& k) {
    int ij;
    divmod(e, n2, a.l2, ij, k);
    divmod(ij, n1, a.l1, i, j);
  };
  auto color = [&](int c) {
    for (int e0 = t0; e0 < ncell / 2; e0 += kU * nt) {
      Nb nb[kU];
      double rh[kU];
      int off[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int e = min(e0 + u * nt, ncell / 2 - 1);  // clamped duplicates are not stored
        int kq, ij, i, j;
        divmod(e, h, lh, ij, kq);
        divmod(ij, n1, a.l1, i, j);
        const int k = 2 * kq + ((a.lo_par + i + j + c) & 1);
        nb[u] = load(i, j, k);
        rh[u] = a.rhs[i * a.rs0 + j * a.rs1 + k];
        off[u] = i * a.ps0 + j * a.ps1 + k;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (e0 + u * nt < ncell / 2) p[off[u]] = relax(nb[u].c, rh[u], lapn(nb[u]), a.cf.rgamma);
    }
  };
  auto smooth = [&](int first) {
    for (int q = first; q < a.nsw; ++q) {
      color(0);
      g.sync();
      color(1);
      g.sync();
    }
  };
  if (!a.up) {
    // the correction starts from zero: the first red half-sweep sees only
    // zeros around its cells, so it is fused with the zeroing pass -- the same
    // operations on the same (zero) operands, one pass and one grid sync less
    for (int e = t0; e < ncell; e += nt) {
      int i, j, k;
      cell(e, i, j, k);
      const bool red = (k & 1) == ((a.lo_par + i + j) & 1);
      P(i, j, k) = red && a.nsw > 0 ? relax(0.0, a.rhs[i * a.rs0 + j * a.rs1 + k],
                                            lap7(0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, a.cf), a.cf.rgamma)
                                     : 0.0;
    }
    if (a.nsw > 0) {
      g.sync();
      color(1);
      g.sync();
      smooth(1);
    } else {
      g.sync();
    }
    const int c0 = n0 >> 1, c1 = n1 >> 1, c2 = n2 >> 1;
    const int lc1 = a.l1 > 0 ? a.l1 - 1 : -1, lc2 = a.l2 > 0 ? a.l2 - 1 : -1;
    for (int e = t0; e < ncell / 8; e += nt) {
      int K, IJ, I, J;
      divmod(e, c2, lc2, IJ, K);
      divmod(IJ, c1, lc1, I, J);
      Nb nb[8];
      double rh[8];
#pragma unroll
      for (int di = 0; di < 2; ++di)
#pragma unroll
        for (int dj = 0; dj < 2; ++dj)
#pragma unroll
          for (int dk = 0; dk < 2; ++dk) {
            const int i = 2 * I + di, j = 2 * J + dj, k = 2 * K + dk;
            nb[di * 4 + dj * 2 + dk] = load(i, j, k);
            rh[di * 4 + dj * 2 + dk] = a.rhs[i * a.rs0 + j * a.rs1 + k];
          }
      double v[8];
#pragma unroll
      for (int x = 0; x < 8; ++x) v[x] = rh[x] - lapn(nb[x]);
      a.c[I * a.cs0 + J * a.cs1 + K] = avg8t(v);
    }
    (void)c0;
    return;
  }
  for (int e = t0; e < ncell; e += nt) {
    int i, j, k;
    cell(e, i, j, k);
    P(i, j, k) = P(i, j, k) + a.c[(i >> 1) * a.cs0 + (j >> 1) * a.cs1 + (k >> 1)];
  }
  g.sync();
  smooth(0);
  // width-1 ghost layer of the grown box (valid cells are final)
  const int E1 = n1 + 2, E2 = n2 + 2, ng = (int)(n0 + 2) * E1 * E2;
  for (int e = t0; e < ng; e += nt) {
    const int kk = (int)(e % E2) - 1;
    const int q = e / E2;
    const int jj = (int)(q % E1) - 1, ii = (int)(q / E1) - 1;
    if (ii >= 0 && ii < n0 && jj >= 0 && jj < n1 && kk >= 0 && kk < n2) continue;
    const int i = ii < 0 ? n0 - 1 : ii >= n0 ? 0 : ii;
    const int j = jj < 0 ? n1 - 1 : jj >= n1 ? 0 : jj;
    const int k = kk < 0 ? n2 - 1 : kk >= n2 ? 0 : kk;
    p[ii * a.ps0 + jj * a.ps1 + kk] = P(i, j, k);
  }
}

}  // namespace
}  // namespace amrb

using namespace amrb;

extern "C" int amrb_coarse_tail(int nlev, const int32_t* lohi, const double* dh, const amrb_field* rhs,
                                const double* rhs_base, amrb_field* phi, double* phi_base, int nu1, int nu2,
                                int nbottom, int cluster, int32_t* ghosts_written, void* stream) {
  return guarded([&] {
    if (cluster < 0 || cluster > 2) throw Error(AMRB_EINVAL, "amrb_coarse_tail: cluster must be 0, 1 or 2");
    if (ghosts_written) *ghosts_written = 0;
    if (nlev < 1 || nlev > kMaxTail || !lohi || !dh || !rhs || !phi)
      throw Error(AMRB_EINVAL, "amrb_coarse_tail: bad arguments");
    const Field& fr = *reinterpret_cast<const Field*>(rhs);
    const Field& fp = *reinterpret_cast<const Field*>(phi);
    if (fr.host.size() != 1 || fp.host.size() != 1) throw Error(AMRB_EINVAL, "coarse tail needs single-box fields");
    TailArgs a;
    std::memset(&a, 0, sizeof a);
    a.nlev = nlev;
    int off = 0;
    for (int l = 0; l < nlev; ++l) {
      TailLevel& L = a.lv[l];
      int par = 0;
      for (int x = 0; x < 3; ++x) {
        L.n[x] = lohi[6 * l + 3 + x] - lohi[6 * l + x] + 1;
        par += lohi[6 * l + x];
        if (L.n[x] < 1) throw Error(AMRB_EINVAL, "empty tail level");
        if (l + 1 < nlev && L.n[x] % 2) throw Error(AMRB_EINVAL, "tail level not coarsenable");
      }
      L.lo_par = par & 1;
      L.phi_off = off;
      off += (L.n[0] + 2) * (L.n[1] + 2) * (L.n[2] + 2);
      L.rhs_off = off;
      off += L.n[0] * L.n[1] * L.n[2];
      L.cf = make_coef(dh + 3 * l);
      if (l > 0)
        for (int x = 0; x < 3; ++x)
          if (a.lv[l - 1].n[x] != 2 * L.n[x]) throw Error(AMRB_EINVAL, "tail levels must halve");
    }
    const size_t bytes = (size_t)off * sizeof(double);
    const FabView& vr = fr.host[0];
    const FabView& vp = fp.host[0];
    a.warp_from = nlev;
    for (int l = 0; l < nlev; ++l)
      if (a.lv[l].n[0] * a.lv[l].n[1] * a.lv[l].n[2] <= 512) {
        a.warp_from = l;
        break;
      }
    a.nu1 = nu1;
    a.nu2 = nu2;
    a.nbottom = nbottom;
    a.rhs = rhs_base + vr.off;
    a.rs0 = vr.s0;
    a.rs1 = vr.s1;
    a.phi = phi_base + vp.off;
    a.ps0 = vp.s0;
    a.ps1 = vp.s1;
    // power-of-two cubic chain (each level >= 4 per side except possibly the
    // bottom, which must be >= 2): dense layout, masked periodic indexing
    const int n0 = a.lv[0].n[0];
    // 32 x n1 x n2 top level (n1, n2 powers of two <= 32) halving per level
    // down to extents >= 2: the top level on a cluster, the chain below in CTA 0
    // (cluster = 0 keeps the one-CTA kernels, for A/B runs).  Default (1):
    // cubic chains only -- the non-cubic top levels (cluster = 2) are
    // bit-identical but measured slower than k_coarse_tail_p2x (C4 weak
    // scaling, 2 GPUs 10.18 -> 10.35 ms, 4 GPUs 10.99 -> 11.02 ms)
    const int cl_mode = cluster;
    bool cl = cl_mode != 0 && n0 == kClN && nlev >= 2 && fp.ng3[0] >= 1 && fp.ng3[1] >= 1 && fp.ng3[2] >= 1;
    for (int l = 0; l < nlev && cl; ++l)
      for (int x = 0; x < 3; ++x) {
        const int e = a.lv[l].n[x];
        cl = cl && e >= 2 && e <= kClN && (e & (e - 1)) == 0 && (l == 0 || a.lv[l - 1].n[x] == 2 * e);
      }
    if (cl && cl_mode < 2)
      for (int l = 0; l < nlev && cl; ++l) cl = a.lv[l].n[1] == a.lv[l].n[0] && a.lv[l].n[2] == a.lv[l].n[0];
    if (cl) {
      bool cubic = true;
      int o2 = 0;
      for (int l = 1; l < nlev; ++l) {
        const int c = a.lv[l].n[0] * a.lv[l].n[1] * a.lv[l].n[2];
        cubic = cubic && a.lv[l].n[0] == a.lv[l].n[1] && a.lv[l].n[1] == a.lv[l].n[2];
        a.lv[l].phi_off = o2;
        o2 += c;
        a.lv[l].rhs_off = o2;
        o2 += c;
      }
      cubic = cubic && a.lv[1].n[0] == 16;  // tail_p2_body<4>: a 16^3 .. chain
      const int slab_off = (o2 + 15) & ~15;
      const int slab = kClPl * a.lv[0].n[1] * a.lv[0].n[2];
      const size_t b2 = (size_t)(slab_off + 2 * slab) * sizeof(double);
      if (b2 <= 227 * 1024) {
        const bool top_cubic = a.lv[0].n[1] == kClN && a.lv[0].n[2] == kClN;
        auto kern = top_cubic && cubic ? k_coarse_tail_cl<true> : k_coarse_tail_cl<false>;
        AMRB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        launch_k(kern, kClCtas, kTailThreads, b2, (cudaStream_t)stream, a, slab_off, cubic ? 1 : 0);
        check_launch("k_coarse_tail_cl");
        if (ghosts_written) *ghosts_written = 1;  // the cluster kernel leaves the top phi's width-1 ghosts current
        return;
      }
    }
    bool p2 = n0 >= 2 && n0 <= 16 && (n0 & (n0 - 1)) == 0 && (n0 >> (nlev - 1)) >= 2;
    for (int l = 0; l < nlev && p2; ++l)
      p2 = a.lv[l].n[0] == (n0 >> l) && a.lv[l].n[1] == (n0 >> l) && a.lv[l].n[2] == (n0 >> l);
    if (p2) {
      int o2 = 0;
      for (int l = 0; l < nlev; ++l) {
        const int c = (n0 >> l) * (n0 >> l) * (n0 >> l);
        a.lv[l].phi_off = o2;
        o2 += c;
        a.lv[l].rhs_off = o2;
        o2 += c;
      }
      const size_t b2 = (size_t)o2 * sizeof(double);
      auto kern = n0 == 16 ? k_coarse_tail_p2<4> : n0 == 8 ? k_coarse_tail_p2<3> : n0 == 4 ? k_coarse_tail_p2<2>
                                                                                            : k_coarse_tail_p2<1>;
      AMRB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b2));
      launch_k(kern, 1, kTailThreads, b2, (cudaStream_t)stream, a);
      check_launch("k_coarse_tail_p2");
      return;
    }
    if (bytes > 227 * 1024) throw Error(AMRB_EINVAL, "coarse tail does not fit in shared memory");
    // power-of-two per axis, not cubic: same dense masked layout
    bool p2x = true;
    for (int l = 0; l < nlev && p2x; ++l)
      for (int x = 0; x < 3; ++x) {
        const int e = a.lv[l].n[x];
        p2x = p2x && e >= 2 && (e & (e - 1)) == 0 && (l == 0 || a.lv[l - 1].n[x] == 2 * e);
      }
    if (p2x) {
      TailArgs b = a;  // dense layout; a keeps the ghosted one for the generic kernel
      int o2 = 0;
      for (int l = 0; l < nlev; ++l) {
        const int c = b.lv[l].n[0] * b.lv[l].n[1] * b.lv[l].n[2];
        b.lv[l].phi_off = o2;
        o2 += c;
        b.lv[l].rhs_off = o2;
        o2 += c;
      }
      const size_t b2 = (size_t)o2 * sizeof(double);
      if (b2 <= 227 * 1024) {
        AMRB_CUDA(cudaFuncSetAttribute(k_coarse_tail_p2x, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b2));
        launch_k(k_coarse_tail_p2x, 1, kTailThreads, b2, (cudaStream_t)stream, b);
        check_launch("k_coarse_tail_p2x");
        return;
      }
    }
    static bool configured = false;
    if (!configured) {
      AMRB_CUDA(cudaFuncSetAttribute(k_coarse_tail, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      configured = true;
    }
    a.warp_from = nlev;  // block mode throughout (measured faster than one warp)
    launch_k(k_coarse_tail, 1, kTailThreads, bytes, (cudaStream_t)stream, a);
    check_launch("k_coarse_tail");
  });
}

extern "C" int amrb_level_grid(int up, const int32_t* lohi, const double* dh, const amrb_field* rhs,
                               const double* rhs_base, amrb_field* phi, double* phi_base, const amrb_field* crse,
                               double* crse_base, int nsweeps, void* stream) {
  return guarded([&] {
    if (!lohi || !dh || !rhs || !phi || !crse || nsweeps < 0) throw Error(AMRB_EINVAL, "amrb_level_grid: bad arguments");
    const Field& fr = *reinterpret_cast<const Field*>(rhs);
    const Field& fp = *reinterpret_cast<const Field*>(phi);
    const Field& fc = *reinterpret_cast<const Field*>(crse);
    if (fr.host.size() != 1 || fp.host.size() != 1 || fc.host.size() != 1)
      throw Error(AMRB_EINVAL, "amrb_level_grid needs single-box fields");
    GridLevelArgs a;
    std::memset(&a, 0, sizeof a);
    int par = 0, n[3];
    for (int x = 0; x < 3; ++x) {
      n[x] = lohi[3 + x] - lohi[x] + 1;
      par += lohi[x];
      if (n[x] < 2 || n[x] % 2) throw Error(AMRB_EINVAL, "amrb_level_grid: extents must be even");
      if (up && fp.ng3[x] < 1) throw Error(AMRB_EINVAL, "amrb_level_grid: phi needs a ghost layer");
    }
    a.n0 = n[0];
    a.n1 = n[1];
    a.n2 = n[2];
    a.lo_par = par & 1;
    a.nsw = nsweeps;
    a.up = up;
    a.cf = make_coef(dh);
    const FabView &vr = fr.host[0], &vp = fp.host[0], &vc = fc.host[0];
    const int64_t span = (int64_t)(n[0] + 2) * vp.s0 + (int64_t)(n[0] + 2) * vr.s0 + (int64_t)(n[0] / 2 + 2) * vc.s0;
    if (span >= (int64_t)1 << 30) throw Error(AMRB_EINVAL, "amrb_level_grid: level too large");
    a.phi = phi_base + vp.off;
    a.ps0 = vp.s0;
    a.ps1 = vp.s1;
    a.rhs = rhs_base + vr.off;
    a.rs0 = vr.s0;
    a.rs1 = vr.s1;
    a.c = crse_base + vc.off;
    a.cs0 = vc.s0;
    a.cs1 = vc.s1;
    auto lg = [](int n) {
      int l = 0;
      while ((1 << l) < n) ++l;
      return (1 << l) == n ? l : -1;
    };
    a.l1 = lg(n[1]);
    a.l2 = lg(n[2]);
    static int max_per_sm = 0;
    if (!max_per_sm) {
      AMRB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&max_per_sm, k_level_grid, 512, 0));
      max_per_sm = max_per_sm < 1 ? 1 : max_per_sm > 2 ? 2 : max_per_sm;
    }
    int per_sm = max_per_sm;
    if (const int64_t want = option("grid_per_sm"))  // CTAs per SM (grid.sync cost vs threads), A/B runs
      per_sm = std::max(1, std::min(per_sm, (int)want));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(num_sms() * per_sm);
    cfg.blockDim = dim3(512);
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    AMRB_CUDA(cudaLaunchKernelEx(&cfg, k_level_grid, a));
    check_launch("k_level_grid");
  });
}
