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

// gsrb_stream.cu: mode 0 plain, 1 fused prolongation (clv / c / c_base),
// 2 plain + max |rhs - L(a)| into *norm (u64 bit pattern, caller zeroes it)
bool launch_resid_restrict_stream(Level& lv, const Field& phi, const double* phi_base, const Field& rhs,
                                  const double* rhs_base, const Field& crse, double* crse_base, const Coef& cf,
                                  cudaStream_t st);
// in-kernel ghost pull of the input (modes 0 and 2): table + device barrier
struct StreamPull {
  const long long* tab;  // 27 per box (ghosts.pull_table)
  uint32_t* pads[kMaxPeers];
  uint32_t* epoch;
  int rank = 0, nranks = 1;
};
bool launch_sweep_stream(int mode, Level& lv, const Field& a, const double* a_base, const Field& b, double* b_base,
                         const Field& r, const double* r_base, const Coef& cf, const int flo[3], const int fhi[3],
                         cudaStream_t st, const Level* clv, const Field* c, const double* c_base,
                         unsigned long long* norm, const long long* push = nullptr,
                         const StreamPull* pull = nullptr);


}  // namespace amrb
