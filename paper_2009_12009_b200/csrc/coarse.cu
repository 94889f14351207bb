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
#include <cstring>

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
  const double* rhs;  // level 0 rhs (valid lo cell)
  int64_t rs0, rs1;
  double* phi;        // level 0 phi (valid lo cell)
  int64_t ps0, ps1;
};

__device__ __forceinline__ double avg8t(const double* v) {
  return ((((v[0] + v[1]) + (v[2] + v[3])) + (v[4] + v[5])) + (v[6] + v[7])) * 0.125;
}

__global__ void __launch_bounds__(kTailThreads, 1) k_coarse_tail(TailArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x;

  auto P = [&](const TailLevel& L) { return sm + L.phi_off; };
  auto Rr = [&](const TailLevel& L) { return sm + L.rhs_off; };
  // phi index of valid cell (i, j, k): one ghost layer
  auto pidx = [](const TailLevel& L, int i, int j, int k) {
    return ((i + 1) * (L.n[1] + 2) + (j + 1)) * (L.n[2] + 2) + (k + 1);
  };
  auto ridx = [](const TailLevel& L, int i, int j, int k) { return (i * L.n[1] + j) * L.n[2] + k; };

  auto fill_faces = [&](const TailLevel& L) {
    double* p = P(L);
    const int n0 = L.n[0], n1 = L.n[1], n2 = L.n[2];
    const int f0 = n1 * n2, f1 = n0 * n2, f2 = n0 * n1;
    const int tot = 2 * (f0 + f1 + f2);
    for (int e = tid; e < tot; e += kTailThreads) {
      int x = e, axis, side;
      if (x < 2 * f0) {
        axis = 0;
        side = x / f0;
        x -= side * f0;
        const int j = x / n2, k = x - j * n2;
        const int i = side ? n0 : -1, si = side ? 0 : n0 - 1;
        p[pidx(L, i, j, k)] = p[pidx(L, si, j, k)];
        continue;
      }
      x -= 2 * f0;
      if (x < 2 * f1) {
        axis = 1;
        side = x / f1;
        x -= side * f1;
        const int i = x / n2, k = x - i * n2;
        const int j = side ? n1 : -1, sj = side ? 0 : n1 - 1;
        p[pidx(L, i, j, k)] = p[pidx(L, i, sj, k)];
        continue;
      }
      x -= 2 * f1;
      axis = 2;
      side = x / f2;
      x -= side * f2;
      const int i = x / n1, j = x - i * n1;
      const int k = side ? n2 : -1, sk = side ? 0 : n2 - 1;
      p[pidx(L, i, j, k)] = p[pidx(L, i, j, sk)];
      (void)axis;
    }
  };
  auto color = [&](const TailLevel& L, int c) {
    double* p = P(L);
    const double* r = Rr(L);
    const int n0 = L.n[0], n1 = L.n[1], n2 = L.n[2];
    const int sj = n2 + 2, si = (n1 + 2) * sj;
    const int np = n0 * n1 * ((n2 + 1) / 2);
    const int h = (n2 + 1) / 2;
    for (int e = tid; e < np; e += kTailThreads) {
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
        __syncthreads();
        color(L, c);
        __syncthreads();
      }
  };
  auto zero_phi = [&](const TailLevel& L) {
    double* p = P(L);
    const int tot = (L.n[0] + 2) * (L.n[1] + 2) * (L.n[2] + 2);
    for (int e = tid; e < tot; e += kTailThreads) p[e] = 0.0;
  };

  // load level-0 rhs
  {
    const TailLevel& L = a.lv[0];
    double* r = Rr(L);
    const int tot = L.n[0] * L.n[1] * L.n[2];
    for (int e = tid; e < tot; e += kTailThreads) {
      const int ij = e / L.n[2], k = e - ij * L.n[2];
      const int i = ij / L.n[1], j = ij - i * L.n[1];
      r[e] = a.rhs[i * a.rs0 + j * a.rs1 + k];
    }
  }
  // down
  for (int l = 0; l < a.nlev; ++l) {
    const TailLevel& L = a.lv[l];
    zero_phi(L);
    __syncthreads();
    if (l == a.nlev - 1) {
      smooth(L, a.nbottom);
      break;
    }
    smooth(L, a.nu1);
    fill_faces(L);
    __syncthreads();
    // residual + restriction into level l+1's rhs
    const TailLevel& C = a.lv[l + 1];
    {
      const double* p = P(L);
      const double* r = Rr(L);
      double* rc = Rr(C);
      const int sj = L.n[2] + 2, si = (L.n[1] + 2) * sj;
      const int tot = C.n[0] * C.n[1] * C.n[2];
      for (int e = tid; e < tot; e += kTailThreads) {
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
    }
    __syncthreads();
  }
  // up
  for (int l = a.nlev - 2; l >= 0; --l) {
    const TailLevel& L = a.lv[l];
    const TailLevel& C = a.lv[l + 1];
    double* p = P(L);
    const double* pc = P(C);
    const int tot = L.n[0] * L.n[1] * L.n[2];
    for (int e = tid; e < tot; e += kTailThreads) {
      const int ij = e / L.n[2], k = e - ij * L.n[2];
      const int i = ij / L.n[1], j = ij - i * L.n[1];
      const int o = pidx(L, i, j, k);
      p[o] = p[o] + pc[pidx(C, i >> 1, j >> 1, k >> 1)];
    }
    __syncthreads();
    smooth(L, a.nu2);
  }
  // store level-0 phi (valid)
  {
    const TailLevel& L = a.lv[0];
    const double* p = P(L);
    const int tot = L.n[0] * L.n[1] * L.n[2];
    for (int e = tid; e < tot; e += kTailThreads) {
      const int ij = e / L.n[2], k = e - ij * L.n[2];
      const int i = ij / L.n[1], j = ij - i * L.n[1];
      a.phi[i * a.ps0 + j * a.ps1 + k] = p[pidx(L, i, j, k)];
    }
  }
}

}  // namespace
}  // namespace amrb

using namespace amrb;

extern "C" int amrb_coarse_tail(int nlev, const int32_t* lohi, const double* dh, const amrb_field* rhs,
                                const double* rhs_base, amrb_field* phi, double* phi_base, int nu1, int nu2,
                                int nbottom, void* stream) {
  return guarded([&] {
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
    if (bytes > 227 * 1024) throw Error(AMRB_EINVAL, "coarse tail does not fit in shared memory");
    const FabView& vr = fr.host[0];
    const FabView& vp = fp.host[0];
    a.nu1 = nu1;
    a.nu2 = nu2;
    a.nbottom = nbottom;
    a.rhs = rhs_base + vr.off;
    a.rs0 = vr.s0;
    a.rs1 = vr.s1;
    a.phi = phi_base + vp.off;
    a.ps0 = vp.s0;
    a.ps1 = vp.s1;
    static bool configured = false;
    if (!configured) {
      AMRB_CUDA(cudaFuncSetAttribute(k_coarse_tail, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      configured = true;
    }
    k_coarse_tail<<<1, kTailThreads, bytes, (cudaStream_t)stream>>>(a);
    check_launch("k_coarse_tail");
  });
}
