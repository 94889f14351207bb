// Fused GSRB sweep, TMA path (sm_100a).
//
// Same algorithm and bit-exact result as k_gsrb_sweep / k_gsrb_sweep3
// (stencil.cu): out of place A -> B, red of the ghost ring recomputed
// locally, black relaxed and streamed out.  What is different:
//
//  * planes of A (phi, grown by 2 in j, k) and of rhs (grown by 1) arrive by
//    TMA -- one cp.async.bulk.tensor per plane per operand, issued by one
//    thread, completion on a per-slot mbarrier -- so the load path costs no
//    per-element instructions and no registers;
//  * red(p+2) and black(p) are independent (red reads only black cells, which
//    no phase ever writes back to shared memory; black reads only red cells),
//    so one step runs both in a single phase with ONE __syncthreads:
//        wait(phi p+3, rhs p+2); barrier; TMA(phi p+3+D, rhs p+2+D);
//        black(p) -> global;  red(p+2) -> shared
//  * warp roles are uniform: warp w relaxes red ring row w+1 (one k-pair per
//    lane, TK = 64), warps w < TJ also relax + store black row w+2, and the
//    two extra warps relax the ring columns k0-1 / k0+TK.
//  * persistent CTAs march balanced contiguous ranges of (column, plane)
//    steps, like k_gsrb_sweep3.
//
// Slot rotation (relative to the segment's first plane): phi has D+5 slots,
// rhs D+3.  At step p the TMA for phi(p+3+D) reuses the slot of phi(p-2) and
// rhs(p+2+D) the slot of rhs(p-1); their last readers ran in step p-1, before
// the step-p barrier.  All threads fence.proxy.async after their shared
// stores so the async-proxy TMA writes are ordered after them.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <climits>
#include <cstring>
#include <map>
#include <mutex>

#include "stencil_common.cuh"

namespace amrb {

namespace {

struct Sweep4Args {
  const int4* cols;  // (box, j0, k0, first plane-step of the column)
  const FabView* fa;  // bulk mode: phi-in and rhs views (source addresses)
  const FabView* fr;
  const double* a;
  const double* rhs;
  const int* slot;   // per box: index of its block in the allocation
  int ncols;
  long long total;
  const BoxGeom* geo;
  const FabView* fb;
  double* b;
  Coef cf;
  int a_kc, a_jc, a_ic;  // tensor-map coordinate offsets: phi plane ip, rows from j0-2, cols from k0-2
  int r_kc, r_jc, r_ic;  // rhs: rows from j0-1, cols from k0-2
  int fixed_lo[3], fixed_hi[3];
  PushDev push;  // k_gsrb_sweep5<..., PUSH>: fill b's ghosts as planes are written
  int c_kc, c_jc, c_ic;  // k_gsrb_sweep5<..., PROL>: coarse tensor-map offsets (tile from (j0/2-1, k0/2-1))
  int rpf;               // k_gsrb_sweep5: rhs plane prefetch distance into L2 (0: off)
  int q_kc, q_jc, q_ic;  // rhs tensor-map offsets (prefetch box from (j0-1, k0-1), even start column)
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_inval(uint64_t* bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity));
}
__device__ __forceinline__ void tma_load4(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                          int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5}], [%6];\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tma_prefetch4(const CUtensorMap* map, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];\n" ::"l"(map), "r"(c0),
               "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

constexpr int kTK = 64;

// BULK: a tile spans whole rows of its box (TK == box k-extent), so a plane's
// rows j0-2 .. j0+TJ+1 are one contiguous chunk of memory: one 1-D
// cp.async.bulk copy per plane, smem rows keep the storage pitch PP = 72 and
// smem col CO + c holds cell k0-2+c.  Otherwise a 4-D tensor-map TMA box of
// PP = TK+4 columns (CO = 0).
template <int TJ, int TK, int D, bool BULK>
struct Sweep4Layout {
  static constexpr int PP = BULK ? TK + 8 : TK + 4;  // smem row pitch (doubles)
  static constexpr int CO = BULK ? 2 : 0;
  static constexpr int PJ = TJ + 4;   // phi rows j0-2 .. j0+TJ+1
  static constexpr int RJ = TJ + 2;   // rhs rows j0-1 .. j0+TJ
  static constexpr int NPHI = D + 5, NRHS = D + 3;
  static constexpr int PBYTES = PJ * PP * 8;
  static constexpr int RBYTES = RJ * PP * 8;
  static constexpr int PSTRIDE = (PBYTES + 127) / 128 * 128;
  static constexpr int RSTRIDE = (RBYTES + 127) / 128 * 128;
  static constexpr int BAR_OFF = NPHI * PSTRIDE + NRHS * RSTRIDE;
  static constexpr int BYTES = BAR_OFF + 8 * (NPHI + NRHS);
  static constexpr int NW = TJ + 2;  // warps
};

template <int TJ, int TK, int D, int MINB, bool FIXED, bool BULK>
__global__ void __launch_bounds__(32 * (TJ + 2), MINB)
    k_gsrb_sweep4(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmR, Sweep4Args args) {
  pdl_entry();
  using LY = Sweep4Layout<TJ, TK, D, BULK>;
  constexpr int PK = LY::PP;
  constexpr int CO = LY::CO;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + LY::BAR_OFF);
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const Coef cf = args.cf;
  auto phi_slot = [&](int rel) { return reinterpret_cast<double*>(smem_raw + (rel % LY::NPHI) * LY::PSTRIDE); };
  auto rhs_slot = [&](int rel) {
    return reinterpret_cast<double*>(smem_raw + LY::NPHI * LY::PSTRIDE + (rel % LY::NRHS) * LY::RSTRIDE);
  };

  const long long G = gridDim.x;
  long long s = args.total * blockIdx.x / G;
  const long long e = args.total * (blockIdx.x + 1) / G;
  if (s >= e) return;
  int col = 0;
  {
    int lo = 0, hi = args.ncols - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (args.cols[mid].w <= s)
        lo = mid;
      else
        hi = mid - 1;
    }
    col = lo;
  }
  bool first_segment = true;
  while (s < e) {
    const int4 cd = args.cols[col];
    const BoxGeom g = args.geo[cd.x];
    const FabView B = args.fb[cd.x];
    const FabView AV = BULK ? args.fa[cd.x] : B;
    const FabView RV = BULK ? args.fr[cd.x] : B;
    const int slot = args.slot[cd.x];
    const int j0 = cd.y, k0 = cd.z;
    const int i0 = (int)(s - cd.w);
    const int i1 = (int)min((long long)g.n[0], e - cd.w);
    s += i1 - i0;
    ++col;
    const int jk0 = g.lo[1] + j0 + g.lo[2] + k0;
    const int pbase = i0 - 2;  // relative index origin of phi planes
    const int rbase = i0 - 1;  // and of rhs planes

    // (re)arm the barriers: every load of the previous segment was waited on
    __syncthreads();
    if (tid == 0) {
      for (int x = 0; x < LY::NPHI + LY::NRHS; ++x) {
        if (!first_segment) mbar_inval(&bars[x]);
        mbar_init(&bars[x], 1);
      }
      fence_barrier_init();
    }
    first_segment = false;
    __syncthreads();

    auto issue_phi = [&](int ip) {
      const int rel = ip - pbase;
      uint64_t* bar = &bars[rel % LY::NPHI];
      mbar_expect_tx(bar, LY::PBYTES);
      if (BULK)
        bulk_load(phi_slot(rel), args.a + AV.off + (int64_t)ip * AV.s0 + (int64_t)(j0 - 2) * AV.s1 + (k0 - 2 - CO),
                  LY::PBYTES, bar);
      else
        tma_load4(phi_slot(rel), &tmA, bar, k0 + args.a_kc, j0 + args.a_jc, ip + args.a_ic, slot);
    };
    auto issue_rhs = [&](int ip) {
      const int rel = ip - rbase;
      uint64_t* bar = &bars[LY::NPHI + rel % LY::NRHS];
      mbar_expect_tx(bar, LY::RBYTES);
      if (BULK)
        bulk_load(rhs_slot(rel), args.rhs + RV.off + (int64_t)ip * RV.s0 + (int64_t)(j0 - 1) * RV.s1 + (k0 - 2 - CO),
                  LY::RBYTES, bar);
      else
        tma_load4(rhs_slot(rel), &tmR, bar, k0 + args.r_kc, j0 + args.r_jc, ip + args.r_ic, slot);
    };
    auto wait_phi = [&](int ip) {
      const int rel = ip - pbase;
      mbar_wait(&bars[rel % LY::NPHI], (rel / LY::NPHI) & 1);
    };
    auto wait_rhs = [&](int ip) {
      const int rel = ip - rbase;
      mbar_wait(&bars[LY::NPHI + rel % LY::NRHS], (rel / LY::NRHS) & 1);
    };
    auto is_fixed = [&](int gi, int r, int c) {
      const int gj = g.lo[1] + j0 - 2 + r, gk = g.lo[2] + k0 - 2 + c;
      return gi < args.fixed_lo[0] || gi > args.fixed_hi[0] || gj < args.fixed_lo[1] || gj > args.fixed_hi[1] ||
             gk < args.fixed_lo[2] || gk > args.fixed_hi[2];
    };
    // relax smem cell o (row r, col c) of plane ip; rhs row r-1, same col
    auto relax_at = [&](const double* P, const double* Pm, const double* Pp, const double* Rh, int o) {
      const double v = P[o];
      const double lap = lap7(v, Pm[o], Pp[o], P[o - PK], P[o + PK], P[o - 1], P[o + 1], cf);
      return relax(v, Rh[o - PK], lap, cf.rgamma);
    };
    // red of plane ip (its smem parity base bp): ring row w+1 (pair = lane), or a ring column
    auto red = [&](int ip) {
      double* P = phi_slot(ip - pbase);
      const double* Pm = phi_slot(ip - 1 - pbase);
      const double* Pp = phi_slot(ip + 1 - pbase);
      const double* Rh = rhs_slot(ip - rbase);
      const int gi = g.lo[0] + ip;
      const int bp = (gi + jk0) & 1;  // smem cell (r, c) has parity (bp + r + c) & 1; red is even
      if (lane < TK / 2) {
        const int r = warp + 1;
        const int c = 2 * lane + 2 + ((bp + r) & 1);
        if (!(FIXED && is_fixed(gi, r, c))) {
          const int o = r * PK + CO + c;
          P[o] = relax_at(P, Pm, Pp, Rh, o);
        }
      }
      if (warp >= TJ && lane < TJ + 2) {
        const int r = lane + 1;
        const int c = warp == TJ ? 1 : TK + 2;
        if (((bp + r + c) & 1) == 0 && !(FIXED && is_fixed(gi, r, c))) {
          const int o = r * PK + CO + c;
          P[o] = relax_at(P, Pm, Pp, Rh, o);
        }
      }
    };
    // One step, bank-conflict free: black(p) and red(p+2) occupy complementary
    // columns of a row (planes p and p+2 have the same parity pattern), so
    // warp w takes row r = w+1 with lane -> consecutive column c; a lane whose
    // cell is black in plane p relaxes it there, the others relax their red
    // cell of plane p+2.  Consecutive lanes read consecutive doubles (from two
    // slots 128-byte aligned apart): 2 wavefronts per LDS.64.  Every lane of
    // rows 2..TJ+1 then streams plane p's value of its column (new black, or the
    // final red read back from shared) with one coalesced STG.64.
    auto step = [&](int p, bool do_red) {
      const int r = warp + 1;
      const bool row_black = r >= 2 && r <= TJ + 1;
      const int gi = g.lo[0] + p;
      const int bp = (gi + jk0) & 1;  // same for plane p+2
      const double* S0 = phi_slot(p - pbase);       // plane p
      double* S2 = phi_slot(p + 2 - pbase);         // plane p+2
      const double* Sm = phi_slot(p - 1 - pbase);   // p-1
      const double* S1 = phi_slot(p + 1 - pbase);   // p+1
      const double* S3 = phi_slot(p + 3 - pbase);   // p+3
      const double* R0 = rhs_slot(p - rbase);
      const double* R2 = rhs_slot(p + 2 - rbase);
      double* out = args.b + B.off + (int64_t)p * B.s0 + (int64_t)(j0 + warp - 1) * B.s1 + k0 - 2;
#pragma unroll
      for (int h = 0; h < (TK + 31) / 32; ++h) {
        if (TK < 32 && lane >= TK) break;
        const int c = 2 + lane + 32 * h;
        const bool black = ((bp + r + c) & 1) != 0;  // cell (r, c) is black in planes p, p+2
        const double* P = black ? S0 : S2;
        const double* Pm = black ? Sm : S1;
        const double* Pp = black ? S1 : S3;
        const double* Rh = black ? R0 : R2;
        const int o = r * PK + CO + c;
        const bool act = black ? row_black : do_red;
        double v = P[o];
        if (act && !(FIXED && is_fixed(black ? gi : gi + 2, r, c))) v = relax_at(P, Pm, Pp, Rh, o);
        if (!black && act) S2[o] = v;
        if (row_black) out[c] = black ? v : S0[o];
      }
      // ring columns k0-1 / k0+TK of plane p+2 (red only)
      if (do_red && lane < 2) {
        const int c = lane ? TK + 2 : 1;
        if (((bp + r + c) & 1) == 0 && !(FIXED && is_fixed(gi + 2, r, c))) {
          const int o = r * PK + CO + c;
          S2[o] = relax_at(S2, S1, S3, R2, o);
        }
      }
    };

    // prologue: phi i0-2 .. i0+2+D, rhs i0-1 .. i0+1+D (clipped to what the segment needs)
    if (tid == 0) {
      for (int ip = i0 - 2; ip <= min(i0 + 2 + D, i1 + 1); ++ip) issue_phi(ip);
      for (int ip = i0 - 1; ip <= min(i0 + 1 + D, i1); ++ip) issue_rhs(ip);
    }
    for (int ip = i0 - 2; ip <= i0 + 2; ++ip) wait_phi(ip);
    for (int ip = i0 - 1; ip <= i0 + 1; ++ip) wait_rhs(ip);
    red(i0 - 1);
    red(i0);
    red(i0 + 1);
    fence_proxy_async();
    for (int p = i0; p < i1; ++p) {
      const bool do_red = p + 2 <= i1;
      if (do_red) {
        wait_phi(p + 3);
        wait_rhs(p + 2);
      }
      __syncthreads();
      if (tid == 0) {
        if (p + 3 + D <= i1 + 1) issue_phi(p + 3 + D);
        if (p + 2 + D <= i1) issue_rhs(p + 2 + D);
      }
      step(p, do_red);
      fence_proxy_async();
    }
  }
}

// ---------------------------------------------------------------------------
// k_gsrb_sweep5: same schedule and result as k_gsrb_sweep4, re-balanced for
// the B200 (ncu of sweep4: issue-bound at ~227 warp-instructions per warp-step,
// every relaxation a serial LDS -> 9-deep DADD chain, one plane of phi in
// flight, barrier waits on the one warp that also issued TMA and relaxed ring
// columns).
//
//  * only phi goes through shared memory (TMA ring of D+5 plane tiles); rhs,
//    read once per cell per sweep, is loaded by each lane straight into
//    registers two steps ahead (ld.global.nc);
//  * the step body is branch-free: all shared loads first, both of a lane's
//    relaxations computed unconditionally and selected, so their DADD chains
//    interleave;
//  * warp roles balance the per-step latency at <= 2 chains per warp:
//      warp 0          red cells of the two ring rows (j0-1, j0+TJ), one per lane,
//      warps 1..TJ     tile row j0+w-1: black(p) or red(p+2) per lane, streams plane p out,
//      warp TJ+1       red cells of the two ring columns (k0-1, k0+TK), and issues the TMA;
//  * ring-slot indices, mbarrier phases and pointers advance incrementally.
// ---------------------------------------------------------------------------
template <int TJ, int TK, int D>
struct Sweep5Layout {
  // smem row = TMA box width: cols k0-2 .. k0+TK+3 (two spare columns keep the
  // ring-column warp's every-other-row accesses off a single bank pair)
  static constexpr int PK = TK + 6;
  static constexpr int PJ = TJ + 4;
  static constexpr int NPHI = D + 5;
  static constexpr int PBYTES = PJ * PK * 8;
  static constexpr int PSTRIDE = (PBYTES + 127) / 128 * 128;
  static constexpr int BAR_OFF = NPHI * PSTRIDE;
  static constexpr int BYTES = BAR_OFF + 8 * NPHI;
  static constexpr int NW = TJ + 2;
  static constexpr int NH = (TK + 31) / 32;
  // PUSH: per (warp, destination slot 0..3NH-1, lane) element delta of the lane's
  // interior-plane ghost destinations
  static constexpr int PDEL_OFF = BYTES;
  static constexpr int BYTES_PUSH = PDEL_OFF + NW * 3 * NH * 32 * 8;  // + NW flag words
  // PROL: ring of NC coarse plane tiles, rows (j0-2)/2 .. (j0+TJ+1)/2, cols
  // (k0-2)/2 - kshift .. : a TMA box must start on a 16-byte boundary in its
  // inner dimension, so the tile starts at the even tensor column at or below
  // (k0-2)/2 (kshift = 0 or 1) and is TK/2 + 4 wide
  // NC = 5: a segment prologue issues fine planes i0-2 .. i0+5, i.e. up to five
  // coarse planes (odd i0); in steady state <= 2 are needed at once
  static constexpr int CJ = TJ / 2 + 2, CK = TK / 2 + 4, NC = 5;
  static constexpr int CBYTES = CJ * CK * 8;
  static constexpr int CSTRIDE = (CBYTES + 127) / 128 * 128;
  static constexpr int C_OFF = (BYTES + 127) / 128 * 128;
  static constexpr int BYTES_PROL = C_OFF + NC * CSTRIDE;
};

template <int TJ, int TK, int D, int MINB, bool FIXED, bool PUSH, bool PROL = false>
__global__ void __launch_bounds__(32 * (TJ + 2), MINB)
    k_gsrb_sweep5(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmC,
                  const __grid_constant__ CUtensorMap tmR, const __grid_constant__ Sweep4Args args) {
  pdl_entry();
  using LY = Sweep5Layout<TJ, TK, D>;
  constexpr int PK = LY::PK, NPHI = LY::NPHI, NH = LY::NH, NW = LY::NW;
  static_assert(TJ % 2 == 0 && TJ + 2 <= 32, "ring-column warp holds one cell per lane");
  static_assert(!PROL || (!FIXED && !PUSH && D >= 3), "PROL: periodic levels, corrects plane p+4 in step p");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + LY::BAR_OFF);
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  constexpr int ROLE_RROW = 0, ROLE_ROW = 1, ROLE_RCOL = 2;
  const int role = warp == 0 ? ROLE_RROW : (warp == NW - 1 ? ROLE_RCOL : ROLE_ROW);
  const int producer = 32 * (NW - 1);  // lane 0 of the ring-column warp
  const Coef cf = args.cf;
  auto slot = [&](int idx) { return reinterpret_cast<double*>(smem_raw + idx * LY::PSTRIDE); };
  auto wrap = [](int x) { return x >= NPHI ? x - NPHI : x; };
  auto cslot = [&](int idx) { return reinterpret_cast<double*>(smem_raw + LY::C_OFF + idx * LY::CSTRIDE); };

  const long long G = gridDim.x;
  long long s = args.total * blockIdx.x / G;
  const long long e = args.total * (blockIdx.x + 1) / G;
  if (s >= e) return;
  int col = 0;
  {
    int lo = 0, hi = args.ncols - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (args.cols[mid].w <= s)
        lo = mid;
      else
        hi = mid - 1;
    }
    col = lo;
  }
  bool remote = false;  // this thread stored ghosts on another rank
  bool first_segment = true;
  while (s < e) {
    const int4 cd = args.cols[col];
    const BoxGeom g = args.geo[cd.x];
    const FabView B = args.fb[cd.x];
    const FabView RV = args.fr[cd.x];
    const int bslot = args.slot[cd.x];
    const int j0 = cd.y, k0 = cd.z;
    const int i0 = (int)(s - cd.w);
    const int i1 = (int)min((long long)g.n[0], e - cd.w);
    s += i1 - i0;
    ++col;
    const int jk0 = g.lo[1] + j0 + g.lo[2] + k0;
    // smem cell (row, c) of plane ip is red iff ((g.lo[0] + ip + jk0 + row + c) & 1) == 0
    const int par0 = (g.lo[0] + i0 + jk0) & 1;  // parity base of plane i0
    const int cbase = (i0 - 2) >> 1;            // PROL: coarse plane of ring slot 0
    const int qkx = (k0 + args.q_kc) & ~1;      // rhs prefetch box: even start column
    const int ckx = (k0 >> 1) + args.c_kc;      // PROL: tensor column of coarse cell (k0-2)/2
    const int cshift = ckx & 1;                 //       the tile starts cshift columns before it

    __syncthreads();
    if (tid == producer) {
      for (int x = 0; x < NPHI; ++x) {
        if (!first_segment) mbar_inval(&bars[x]);
        mbar_init(&bars[x], 1);
      }
      fence_barrier_init();
    }
    first_segment = false;
    __syncthreads();

    // plane ip lives in slot (ip - i0 + 2) % NPHI
    // PROL: the first fine plane of each coarse plane also brings that coarse
    // tile, on the same mbarrier (coarse plane ip>>1 lives in coarse slot
    // ((ip>>1) - cbase) % NC; the coarse plane of slot x is rewritten only by
    // the TMA issued with fine plane 2((ip>>1) + NC), six steps after its last reader)
    auto issue = [&](int ip, int idx) {
      const bool cl = PROL && (ip == i0 - 2 || (ip & 1) == 0);
      mbar_expect_tx(&bars[idx], LY::PBYTES + (cl ? LY::CBYTES : 0));
      tma_load4(slot(idx), &tmA, &bars[idx], k0 + args.a_kc, j0 + args.a_jc, ip + args.a_ic, bslot);
      if (cl)
        tma_load4(cslot(((ip >> 1) - cbase) % LY::NC), &tmC, &bars[idx], ckx - cshift, (j0 >> 1) + args.c_jc,
                  (ip >> 1) + args.c_ic, bslot);
    };
    // PROL: plane tile P (plane ip) += coarse parent, rows 0..TJ+3, cols 0..TK+3 --
    // the same single addition as k_prolong, so the sweep sees exactly the
    // prolongated field and its (periodic) ghosts.  Warp w corrects row w.
    auto correct = [&](double* P, int ip) {
      const double* Cc = cslot(((ip >> 1) - cbase) % LY::NC);
      auto row = [&](int rr) {
        double* Pr = P + rr * PK;
        const double* Cr = Cc + (rr >> 1) * LY::CK + cshift;
#pragma unroll
        for (int h = 0; h < (TK + 4 + 31) / 32; ++h) {
          const int c = lane + 32 * h;
          if (c < TK + 4) Pr[c] = Pr[c] + Cr[c >> 1];
        }
      };
      row(warp);
      // rows TJ+2, TJ+3: one cell per thread, on the highest thread ids (the
      // ring-column warp relaxes the fewest cells).  Measured: 8.80-8.84 ms C3
      // solve vs 8.88 with both extra rows on the two ring warps; 16-byte
      // pair loads/stores measured no faster (8.85-8.86).
      constexpr int NT = 32 * NW, NX = 2 * (TK + 4);
      static_assert(NX <= NT, "two extra rows fit one pass");
      const int x = NT - 1 - tid;
      if (x < NX) {
        const int rr = NW + x / (TK + 4), c = x % (TK + 4);
        P[rr * PK + c] = P[rr * PK + c] + Cc[(rr >> 1) * LY::CK + (c >> 1) + cshift];
      }
    };
    if (tid == producer)
      for (int ip = i0 - 2; ip <= min(i0 + 2 + D, i1 + 1); ++ip) issue(ip, ip - i0 + 2);

    auto is_fixed = [&](int gi, int rw, int c) {
      const int gj = g.lo[1] + j0 - 2 + rw, gk = g.lo[2] + k0 - 2 + c;
      return gi < args.fixed_lo[0] || gi > args.fixed_hi[0] || gj < args.fixed_lo[1] || gj > args.fixed_hi[1] ||
             gk < args.fixed_lo[2] || gk > args.fixed_hi[2];
    };
    auto relax_at = [&](const double* P, const double* Pm, const double* Pp, double rh, int o) {
      const double v = P[o];
      const double lap = lap7(v, Pm[o], Pp[o], P[o - PK], P[o + PK], P[o - 1], P[o + 1], cf);
      return relax(v, rh, lap, cf.rgamma);
    };
    const double* rbase = args.rhs + RV.off + (int64_t)(j0 - 2) * RV.s1 + (k0 - 2);  // smem (0, 0) of plane 0
    const int64_t rs0 = RV.s0, rs1 = RV.s1;

    for (int ip = i0 - 2; ip <= i0 + 2; ++ip) mbar_wait(&bars[ip - i0 + 2], 0);
    if constexpr (PROL) {  // planes i0-2 .. i0+3 corrected before anything reads them
      if (i0 + 3 <= i1 + 1) mbar_wait(&bars[5], 0);
      for (int ip = i0 - 2; ip <= min(i0 + 3, i1 + 1); ++ip) correct(slot(ip - i0 + 2), ip);
      __syncthreads();
    }
    // prologue: red of planes i0-1, i0, i0+1 over rows 1..TJ+2, cols 1..TK+2
    // (independent: red reads only black cells).  Red cells only, loads first.
    {
      constexpr int RW = TJ + 2, HC = (TK + 2) / 2;  // red cells per ring-row
      constexpr int NCELL = 3 * RW * HC;
      constexpr int NIT = (NCELL + 32 * NW - 1) / (32 * NW);
      double rh[NIT];
      int oo[NIT], pl[NIT];
      bool ok[NIT];
#pragma unroll
      for (int it = 0; it < NIT; ++it) {
        const int x = tid + it * 32 * NW;
        ok[it] = x < NCELL;
        const int xx = ok[it] ? x : 0;
        pl[it] = xx / (RW * HC);
        const int rem = xx - pl[it] * RW * HC;
        const int rw = 1 + rem / HC;
        const int ip = i0 - 1 + pl[it];
        const int c = 1 + ((par0 + pl[it] + 1 + rw + 1) & 1) + 2 * (rem % HC);  // red column
        oo[it] = rw * PK + c;
        if (FIXED && is_fixed(g.lo[0] + ip, rw, c)) ok[it] = false;
        rh[it] = ok[it] ? __ldg(rbase + (int64_t)ip * rs0 + (int64_t)rw * rs1 + c) : 0.0;
      }
#pragma unroll
      for (int it = 0; it < NIT; ++it) {
        double* P = slot(pl[it] + 1);
        const double v = relax_at(P, slot(pl[it]), slot(pl[it] + 2), rh[it], oo[it]);
        if (ok[it]) P[oo[it]] = v;
      }
    }
    fence_proxy_async();

    // ---- per-role geometry -------------------------------------------------
    // ROLE_ROW: row r = warp+1, column c = 2 + lane + 32h; cell black in plane p
    //           iff ((par0 + (p - i0) + r + lane) & 1) == 1 (same colour in p+2).
    // ROLE_RROW: red cell m = lane + 32h of the ring rows (m < TK/2: row 1, else
    //           row TJ+2), column 2 + 2 idx + parity; plane p+2.
    // ROLE_RCOL: red cell m = lane of the ring columns (m < (TJ+2)/2: col 1, else
    //           col TK+2), row 1 + 2 idx + parity; plane p+2.
    const int r = warp + 1;
    const int lk = TK >= 32 ? lane : (lane & (TK - 1));  // idle lanes alias a valid column
    int rrow[NH], ridx[NH];
    bool rok[NH];
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      const int m = lane + 32 * h;
      rok[h] = m < TK;
      const int mm = rok[h] ? m : 0;
      rrow[h] = mm < TK / 2 ? 1 : TJ + 2;
      ridx[h] = mm < TK / 2 ? mm : mm - TK / 2;
    }
    const bool cok = lane < TJ + 2;
    const int cm = cok ? lane : 0;
    const int ccol = cm < (TJ + 2) / 2 ? 1 : TK + 2;
    const int cidx = cm < (TJ + 2) / 2 ? cm : cm - (TJ + 2) / 2;
    // smem offset of the role's cell h in plane q (q relative to i0: colour flips with q)
    auto cell_off = [&](int q, int h) {
      if (role == ROLE_ROW) return r * PK + 2 + lk + 32 * h;
      if (role == ROLE_RROW) return rrow[h] * PK + 2 + ((par0 + q + rrow[h]) & 1) + 2 * ridx[h];
      return (1 + ((par0 + q + ccol + 1) & 1) + 2 * cidx) * PK + ccol;
    };

    // rhs of the cells step p relaxes, straight to registers.  load_rhs runs for
    // p = i0, i0+1, ... in order: a running plane pointer plus, per cell, two
    // element offsets selected by a parity bit that flips every call (row
    // lanes: black(p) / red(p+2); ring lanes: the red cell of plane p+2)
    const double* rptr;
    int co0[NH], co1[NH];  // ring lanes: smem offset of the red cell in plane p+2, by parity of p - i0
    int rsel;
    if (role == ROLE_ROW) {
      rptr = rbase + (int64_t)i0 * rs0 + (int64_t)r * rs1 + 2 + lk;
      rsel = ((par0 + r + lane) & 1) != 0 ? 0 : 1;  // 0: black(p)
#pragma unroll
      for (int h = 0; h < NH; ++h) co0[h] = co1[h] = 0;
    } else {
      rptr = rbase + (int64_t)(i0 + 2) * rs0;
      rsel = 0;
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        co0[h] = cell_off(2, h);
        co1[h] = cell_off(3, h);
      }
    }
    auto load_rhs = [&](int p, double (&rv)[NH]) {
      if (role == ROLE_ROW) {
        const bool need = (TK >= 32 || lane < TK) && (rsel == 0 ? p < i1 : p + 2 <= i1);
        const double* rp = rptr + (rsel ? 2 * rs0 : 0);
#pragma unroll
        for (int h = 0; h < NH; ++h) rv[h] = need ? __ldg(rp + 32 * h) : 0.0;
      } else {
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          const bool need = p + 2 <= i1 && (role == ROLE_RROW ? rok[h] : (h == 0 && cok));
          const int o = rsel ? co1[h] : co0[h];
          const int rw = o / PK;
          rv[h] = need ? __ldg(rptr + ((int64_t)rw * rs1 + (o - rw * PK))) : 0.0;
        }
      }
      rptr += rs0;
      rsel ^= 1;
    };

    // rhs one step ahead; a lane's colour is the same in steps p and p+2, so a
    // red lane streams out at step p the red(p) it computed at step p-2 (vpA /
    // vpB by step parity; the first two come from the prologue, in shared)
    double rv[NH], vpA[NH], vpB[NH];
    load_rhs(i0, rv);
    // slots of planes p-1 .. p+3 (rotated each step); nidx = slot of plane p+4
    double *sm_ = slot(1), *s0_ = slot(2), *s1_ = slot(3), *s2_ = slot(4), *s3_ = slot(5);
    int nidx = 6 % NPHI;
    constexpr int W0 = PROL ? 6 : 5;    // slot of plane p+3 (PROL: p+4) (awaited)
    int widx = W0 % NPHI;
    unsigned wph = (W0 / NPHI) & 1;
    int iidx = 0;                       // slot of plane p+3+D (issued)
    double* out = args.b + B.off + (int64_t)i0 * B.s0 + (int64_t)(j0 - 2 + r) * B.s1 + (k0 + lk);
    const int64_t bs0 = B.s0;
    // ghost push (PUSH): in interior planes each lane cell has at most two
    // destinations, fixed element deltas from its output address (computed
    // here, kept in shared memory); the first/last g planes take push_cell.
    // shared: [warp][slot 0..3NH-1][lane] deltas, then one flag word per warp
    auto pdel = [&]() {
      return reinterpret_cast<int64_t*>(smem_raw + LY::PDEL_OFF) + warp * 3 * NH * 32 + lane;
    };
    if (PUSH && role == ROLE_ROW) {
      bool any = false;
      int64_t* pd = pdel();
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        int64_t d[kPushMid] = {0, 0, 0};
        if (TK >= 32 || lane < TK) push_deltas_mid(args.push, cd.x, j0 - 2 + r, k0 + lk + 32 * h, B, args.b, d, remote);
#pragma unroll
        for (int x = 0; x < kPushMid; ++x) pd[(3 * h + x) * 32] = d[x];
        any |= d[0] != 0;
      }
      any = __any_sync(0xffffffffu, any);
      if (lane == 0) reinterpret_cast<int*>(smem_raw + LY::BYTES_PUSH)[warp] = any ? 1 : 0;
      __syncwarp();
    }

    auto step = [&](int p, double (&vp)[NH]) {
      const int q = p - i0;
      const bool do_red = p + 2 <= i1;
      if (PROL ? p + 4 <= i1 + 1 : do_red) mbar_wait(&bars[widx], wph);
      widx = wrap(widx + 1);
      wph ^= widx == 0 ? 1u : 0u;
      __syncthreads();
      if (tid == producer && p + 3 + D <= i1 + 1) issue(p + 3 + D, iidx);
      // rhs plane x is first read by load_rhs at the end of step x-3: warm L2
      // with plane p + rpf (no registers; the per-lane loads then hit L2)
      if (tid == producer && args.rpf && p + args.rpf < i1 + 2)
        tma_prefetch4(&tmR, qkx, j0 + args.q_jc, p + args.rpf + args.q_ic, bslot);
      iidx = wrap(iidx + 1);
      const double* Sm = sm_;
      const double* S0 = s0_;
      const double* S1 = s1_;
      double* S2 = s2_;
      const double* S3 = s3_;
      sm_ = s0_;
      s0_ = s1_;
      s1_ = s2_;
      s2_ = s3_;
      s3_ = slot(nidx);
      nidx = wrap(nidx + 1);
      if (role == ROLE_ROW) {
        const bool blk = ((par0 + q + r + lane) & 1) != 0;
        const double* P = blk ? S0 : S2;
        const double* Pm = blk ? Sm : S1;
        const double* Pp = blk ? S1 : S3;
        const bool lane_ok = TK >= 32 || lane < TK;
        const bool act = lane_ok && (blk || do_red);
        // all shared loads first (red(p+2) writes only red cells of S2, which no
        // lane reads in this step except as its own centre value)
        double c[NH], xm[NH], xp[NH], ym[NH], yp[NH], zm[NH], zp[NH];
        // red lanes stream out red(p): computed two steps ago, in vp -- or, in
        // the push variant (register-bound), read back from shared
        if (PUSH || q < 2) {
#pragma unroll
          for (int h = 0; h < NH; ++h) vp[h] = S0[r * PK + 2 + lk + 32 * h];
        }
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          const int o = r * PK + 2 + lk + 32 * h;
          c[h] = P[o];
          xm[h] = Pm[o];
          xp[h] = Pp[o];
          ym[h] = P[o - PK];
          yp[h] = P[o + PK];
          zm[h] = P[o - 1];
          zp[h] = P[o + 1];
        }
        const int gi = g.lo[0] + (blk ? p : p + 2);
        double v[NH];
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          const double nv = relax(c[h], rv[h], lap7(c[h], xm[h], xp[h], ym[h], yp[h], zm[h], zp[h], cf), cf.rgamma);
          const bool a = act && !(FIXED && is_fixed(gi, r, 2 + lk + 32 * h));
          v[h] = a ? nv : c[h];
          if (a && !blk) S2[r * PK + 2 + lk + 32 * h] = v[h];
        }
        double ov[NH];
#pragma unroll
        for (int h = 0; h < NH; ++h) ov[h] = blk ? v[h] : vp[h];
        if (lane_ok) {
#pragma unroll
          for (int h = 0; h < NH; ++h) out[32 * h] = ov[h];
        }
        if (PUSH) {
          if (push_cls(p, g.n[0], args.push.g) == 1) {
            if (reinterpret_cast<const int*>(smem_raw + LY::BYTES_PUSH)[warp]) {
              const int64_t* pd = pdel();
#pragma unroll
              for (int h = 0; h < NH; ++h)
#pragma unroll
                for (int x = 0; x < kPushMid; ++x) {
                  const int64_t dx = pd[(3 * h + x) * 32];
                  if (dx != 0) out[32 * h + dx] = ov[h];
                }
            }
          } else if (lane_ok) {
            const int4 cc = args.cols[col - 1];  // this segment's column
#pragma unroll
            for (int h = 0; h < NH; ++h)
              remote |= push_cell_t(&args.push, cc.x, p, cc.y - 2 + r, cc.z + lk + 32 * h, ov[h]);
          }
        }
        if (!PUSH) {
#pragma unroll
          for (int h = 0; h < NH; ++h) vp[h] = v[h];
        }
      } else if (do_red) {
        // ring rows / ring columns: red(p+2) only
        double nv[NH];
        int o[NH];
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          o[h] = (q & 1) ? co1[h] : co0[h];
          nv[h] = relax_at(S2, S1, S3, rv[h], o[h]);
        }
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          bool a = role == ROLE_RROW ? rok[h] : (h == 0 && cok);
          if (FIXED && a) {
            const int rw = o[h] / PK, cc = o[h] - rw * PK;
            a = !is_fixed(g.lo[0] + p + 2, rw, cc);
          }
          if (a) S2[o[h]] = nv[h];
        }
      }
      if constexpr (PROL) {  // s3_ is plane p+4's slot now; first read in step p+1
        if (p + 4 <= i1 + 1) correct(s3_, p + 4);
      }
      out += bs0;
      load_rhs(p + 1, rv);
      if (q & 1) fence_proxy_async();
    };
    for (int p = i0; p < i1; p += 2) {
      step(p, vpA);
      if (p + 1 < i1) step(p + 1, vpB);
    }
    fence_proxy_async();
  }
  if (PUSH && remote) __threadfence_system();  // remote ghost stores before the consumer's barrier
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// Describe one FabArray's storage as a 4-D tensor (k, j, i, block) when every
// resident box has the same grown shape and blocks are equally spaced.
struct TmaDesc {
  bool ok = false;
  int64_t base;  // element offset of tensor element (0, 0, 0, 0) (16-byte aligned)
  int64_t pitch, rows, planes, stride;
  int f, g;      // k index of the grown box's first cell = f
  std::vector<int> slot;  // per box
};

TmaDesc describe(const Level& lv, const Field& f) {
  TmaDesc d;
  const int g = f.ngrow;
  if (f.ng3[0] != g || f.ng3[1] != g || f.ng3[2] != g) return d;
  d.g = g;
  int first = -1, second = -1;
  for (int b = 0; b < lv.nboxes; ++b)
    if (lv.resident[b]) {
      if (first < 0)
        first = b;
      else if (second < 0)
        second = b;
    }
  if (first < 0) return d;
  const BoxGeom& g0 = lv.geo[first];
  const FabView& v0 = f.host[first];
  auto grown = [&](const FabView& v) { return v.off - g * v.s0 - g * v.s1 - g; };
  const int64_t og = grown(v0);
  d.f = (int)(og & 1);  // shift the tensor origin back to a 16-byte boundary
  d.base = og - d.f;
  d.pitch = v0.s1;
  d.rows = v0.s0 / v0.s1;
  d.planes = g0.n[0] + 2 * g;
  if (d.f + g0.n[2] + 2 * g > d.pitch) return d;
  d.stride = second >= 0 ? grown(f.host[second]) - og : d.planes * v0.s0;
  if (d.stride <= 0 || d.stride % 2) return d;
  d.slot.assign(lv.nboxes, 0);
  int k = 0;
  for (int b = 0; b < lv.nboxes; ++b) {
    if (!lv.resident[b]) continue;
    const BoxGeom& gb = lv.geo[b];
    const FabView& v = f.host[b];
    if (gb.n[0] != g0.n[0] || gb.n[1] != g0.n[1] || gb.n[2] != g0.n[2] || v.s0 != v0.s0 || v.s1 != v0.s1)
      return d;
    if (grown(v) != og + (int64_t)k * d.stride) return d;
    d.slot[b] = k++;
  }
  d.ok = true;
  return d;
}

bool make_map(CUtensorMap* map, const double* base, const TmaDesc& d, int nblocks, int box_rows, int box_cols) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t gdim[4] = {(cuuint64_t)d.pitch, (cuuint64_t)d.rows, (cuuint64_t)d.planes, (cuuint64_t)nblocks};
  cuuint64_t gstride[3] = {(cuuint64_t)d.pitch * 8, (cuuint64_t)(d.pitch * d.rows) * 8, (cuuint64_t)d.stride * 8};
  cuuint32_t box[4] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base + d.base), gdim, gstride, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int TJ, int TK, int D, int MINB, bool BULK>
bool launch4(Level& lv, const Field& a, const double* a_base, const Field& b, double* b_base, const Field& r,
             const double* r_base, const Coef& cf, const int fixed_lo[3], const int fixed_hi[3], bool fixed,
             cudaStream_t st) {
  using LY = Sweep4Layout<TJ, TK, D, BULK>;
  for (auto& gg : lv.geo)
    if (gg.n[1] % TJ || gg.n[2] % TK || (BULK && gg.n[2] != TK)) return false;
  if (a.ngrow < 2 || r.ngrow < 1) return false;
  CUtensorMap ma, mr;
  std::memset(&ma, 0, sizeof ma);
  std::memset(&mr, 0, sizeof mr);
  Sweep4Args args;
  std::memset(&args, 0, sizeof args);
  if (BULK) {
    // every resident box: smem pitch == storage pitch, valid k=0 at row index CO+2
    for (int bx = 0; bx < lv.nboxes; ++bx) {
      if (!lv.resident[bx]) continue;
      const FabView& va = a.host[bx];
      const FabView& vr = r.host[bx];
      if (va.s1 != LY::PP || vr.s1 != LY::PP || va.off % 4 || vr.off % 4) return false;
      if (a.ng3[2] + (4 - a.ng3[2] % 4) % 4 != LY::CO + 2 || r.ng3[2] + (4 - r.ng3[2] % 4) % 4 != LY::CO + 2)
        return false;
    }
  } else {
    TmaDesc da = describe(lv, a), dr = describe(lv, r);
    if (!da.ok || !dr.ok) return false;
    if (da.slot != lv.slot || dr.slot != lv.slot) return false;
    int nres = 0;
    for (auto x : lv.resident) nres += x ? 1 : 0;
    if (!make_map(&ma, a_base, da, nres, LY::PJ, LY::PP)) return false;
    if (!make_map(&mr, r_base, dr, nres, LY::RJ, LY::PP)) return false;
    args.a_kc = -2 + da.g + da.f;
    args.a_jc = -2 + da.g;
    args.a_ic = da.g;
    args.r_kc = -2 + dr.g + dr.f;
    args.r_jc = -1 + dr.g;
    args.r_ic = dr.g;
  }
  const auto& cols = lv.columns(TJ, TK);
  if (cols.host.empty()) return true;
  args.cols = cols.dev.p;
  args.fa = a.dev.p;
  args.fr = r.dev.p;
  args.a = a_base;
  args.rhs = r_base;
  args.slot = lv.dslot.p;
  args.ncols = (int)cols.host.size();
  args.total = cols.total;
  args.geo = lv.dgeo.p;
  args.fb = b.dev.p;
  args.b = b_base;
  args.cf = cf;
  for (int x = 0; x < 3; ++x) {
    args.fixed_lo[x] = fixed_lo[x];
    args.fixed_hi[x] = fixed_hi[x];
  }
  auto kern = fixed ? k_gsrb_sweep4<TJ, TK, D, MINB, true, BULK> : k_gsrb_sweep4<TJ, TK, D, MINB, false, BULK>;
  static int per_sm[2] = {0, 0};
  if (!per_sm[fixed]) {
    AMRB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, LY::BYTES));
    AMRB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[fixed], kern, 32 * LY::NW, LY::BYTES));
    per_sm[fixed] = std::max(per_sm[fixed], 1);
  }
  const long long slots = (long long)per_sm[fixed] * num_sms();
  const long long ncol = (long long)cols.host.size();
  long long grid;
  // balanced persistent split: every CTA marches ~total/G plane-steps.  Big
  // levels: one CTA slot each.  Small levels: segments of >= 2 planes so the
  // level still spreads over the chip (their data lives in L2 anyway).
  grid = std::min<long long>(slots, std::max<long long>(ncol, cols.total / 2));
  launch_k(kern, (unsigned)std::max<long long>(grid, 1), 32 * LY::NW, LY::BYTES, st, ma, mr, args);
  check_launch("k_gsrb_sweep4");
  return true;
}

// rhs tensor map for the L2 prefetch of k_gsrb_sweep5 (box TJ+2 rows x TK+4
// columns from (j0-1, even column <= k0-1)); rpf = 0 when it cannot be made.
// Distance in planes: AMRB_RHS_PREFETCH (plain sweep, default 0) and
// AMRB_RHS_PREFETCH_PROL (fused prolongation sweep, default 3).  Measured on
// the C3 solve (bench.py): PROL 3 -> 8.84 to 8.67 ms (2: no gain, 5: same as
// 3); on the plain fine-level sweep 3 costs 3 us per launch (104.5 -> 107.5),
// 2 is neutral, so it stays off there.
template <int TJ, int TK>
void rhs_prefetch_map(const Level& lv, const Field& r, const double* r_base, int nres, CUtensorMap* mq,
                      Sweep4Args& args, bool prol) {
  static const int dist_plain = getenv("AMRB_RHS_PREFETCH") ? atoi(getenv("AMRB_RHS_PREFETCH")) : 0;
  static const int dist_prol = getenv("AMRB_RHS_PREFETCH_PROL") ? atoi(getenv("AMRB_RHS_PREFETCH_PROL")) : 3;
  const int dist = prol ? dist_prol : dist_plain;
  std::memset(mq, 0, sizeof *mq);
  args.rpf = 0;
  if (dist <= 0) return;
  TmaDesc dr = describe(lv, r);
  if (!dr.ok || dr.slot != lv.slot) return;
  if (!make_map(mq, r_base, dr, nres, TJ + 2, TK + 4)) return;
  args.q_kc = -1 + dr.g + dr.f;
  args.q_jc = -1 + dr.g;
  args.q_ic = dr.g;
  args.rpf = dist;
}

template <int TJ, int TK, int D, int MINB>
bool launch5(Level& lv, const Field& a, const double* a_base, const Field& b, double* b_base, const Field& r,
             const double* r_base, const Coef& cf, const int fixed_lo[3], const int fixed_hi[3], bool fixed,
             cudaStream_t st, const PushDev* push) {
  using LY = Sweep5Layout<TJ, TK, D>;
  for (auto& gg : lv.geo)
    if (gg.n[1] % TJ || gg.n[2] % TK) return false;
  if (a.ngrow < 2 || r.ngrow < 1) return false;
  CUtensorMap ma;
  std::memset(&ma, 0, sizeof ma);
  Sweep4Args args;
  std::memset(&args, 0, sizeof args);
  TmaDesc da = describe(lv, a);
  if (!da.ok || da.slot != lv.slot) return false;
  int nres = 0;
  for (auto x : lv.resident) nres += x ? 1 : 0;
  if (!make_map(&ma, a_base, da, nres, LY::PJ, LY::PK)) return false;
  args.a_kc = -2 + da.g + da.f;
  args.a_jc = -2 + da.g;
  args.a_ic = da.g;
  const auto& cols = lv.columns(TJ, TK);
  if (cols.host.empty()) return true;
  args.cols = cols.dev.p;
  args.fa = a.dev.p;
  args.fr = r.dev.p;
  args.a = a_base;
  args.rhs = r_base;
  args.slot = lv.dslot.p;
  args.ncols = (int)cols.host.size();
  args.total = cols.total;
  args.geo = lv.dgeo.p;
  args.fb = b.dev.p;
  args.b = b_base;
  args.cf = cf;
  for (int x = 0; x < 3; ++x) {
    args.fixed_lo[x] = fixed_lo[x];
    args.fixed_hi[x] = fixed_hi[x];
  }
  if (push) args.push = *push;
  CUtensorMap mq;
  rhs_prefetch_map<TJ, TK>(lv, r, r_base, nres, &mq, args, false);
  const int kv = (fixed ? 1 : 0) + (push ? 2 : 0);
  auto kern = kv == 0   ? k_gsrb_sweep5<TJ, TK, D, MINB, false, false>
              : kv == 1 ? k_gsrb_sweep5<TJ, TK, D, MINB, true, false>
              : kv == 2 ? k_gsrb_sweep5<TJ, TK, D, MINB, false, true>
                        : k_gsrb_sweep5<TJ, TK, D, MINB, true, true>;
  const int bytes = push ? LY::BYTES_PUSH + 4 * LY::NW : LY::BYTES;
  static int per_sm[4] = {0, 0, 0, 0};
  if (!per_sm[kv]) {
    AMRB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    AMRB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[kv], kern, 32 * LY::NW, bytes));
    per_sm[kv] = std::max(per_sm[kv], 1);
  }
  const long long slots = (long long)per_sm[kv] * num_sms();
  const long long ncol = (long long)cols.host.size();
  // balanced contiguous (column, plane) ranges; aligning ranges across columns
  // (grid = ncol * (slots / ncol)) cut L2 misses but measured no faster
  static const int min_steps = getenv("AMRB_SWEEP_MINSTEPS") ? atoi(getenv("AMRB_SWEEP_MINSTEPS")) : 2;
  const long long grid = std::min<long long>(slots, std::max<long long>(ncol, cols.total / min_steps));
  launch_k(kern, (unsigned)std::max<long long>(grid, 1), 32 * LY::NW, bytes, st, ma, ma, mq, args);
  check_launch("k_gsrb_sweep5");
  return true;
}

// Fused prolongation + first post-smoothing sweep: B = sweep(A + P(C)), where
// P(C) is the piecewise-constant parent value of the coarse field C on the
// box-local coarsening of A's level (A's ghosts filled to 2, C's to 1,
// periodic).  Bit-identical to prolong_add; fill_boundary(A, 2); sweep.
template <int TJ, int TK>
bool launch5p(Level& lv, const Field& a, const double* a_base, const Field& b, double* b_base, const Field& r,
              const double* r_base, const Coef& cf, const Level& clv, const Field& c, const double* c_base,
              cudaStream_t st) {
  constexpr int D = 3;
  using LY = Sweep5Layout<TJ, TK, D>;
  for (auto& gg : lv.geo)
    if (gg.n[1] % TJ || gg.n[2] % TK) return false;
  if (a.ngrow < 2 || r.ngrow < 1 || c.ngrow < 1) return false;
  TmaDesc da = describe(lv, a), dc = describe(clv, c);
  if (!da.ok || da.slot != lv.slot || !dc.ok || dc.slot != da.slot) return false;
  int nres = 0;
  for (auto x : lv.resident) nres += x ? 1 : 0;
  CUtensorMap ma, mc;
  std::memset(&ma, 0, sizeof ma);
  std::memset(&mc, 0, sizeof mc);
  if (!make_map(&ma, a_base, da, nres, LY::PJ, LY::PK)) return false;
  if (!make_map(&mc, c_base, dc, nres, LY::CJ, LY::CK)) return false;
  Sweep4Args args;
  std::memset(&args, 0, sizeof args);
  args.a_kc = -2 + da.g + da.f;
  args.a_jc = -2 + da.g;
  args.a_ic = da.g;
  args.c_kc = -1 + dc.g + dc.f;
  args.c_jc = -1 + dc.g;
  args.c_ic = dc.g;
  const auto& cols = lv.columns(TJ, TK);
  if (cols.host.empty()) return true;
  args.cols = cols.dev.p;
  args.fa = a.dev.p;
  args.fr = r.dev.p;
  args.a = a_base;
  args.rhs = r_base;
  args.slot = lv.dslot.p;
  args.ncols = (int)cols.host.size();
  args.total = cols.total;
  args.geo = lv.dgeo.p;
  args.fb = b.dev.p;
  args.b = b_base;
  args.cf = cf;
  CUtensorMap mq;
  rhs_prefetch_map<TJ, TK>(lv, r, r_base, nres, &mq, args, true);
  auto kern = k_gsrb_sweep5<TJ, TK, D, 2, false, false, true>;
  static int per_sm = 0;
  if (!per_sm) {
    AMRB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, LY::BYTES_PROL));
    AMRB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * LY::NW, LY::BYTES_PROL));
    per_sm = std::max(per_sm, 1);
  }
  const long long slots = (long long)per_sm * num_sms();
  const long long ncol = (long long)cols.host.size();
  const long long grid = std::min<long long>(slots, std::max<long long>(ncol, cols.total / 2));
  launch_k(kern, (unsigned)std::max<long long>(grid, 1), 32 * LY::NW, LY::BYTES_PROL, st, ma, mc, mq, args);
  check_launch("k_gsrb_sweep5<PROL>");
  return true;
}

}  // namespace

bool launch_sweep_prolong_tma(Level& lv, const Field& a, const double* a_base, const Field& b, double* b_base,
                              const Field& r, const double* r_base, const Coef& cf, const Level& clv, const Field& c,
                              const double* c_base, cudaStream_t st) {
  int minj = 1 << 30;
  for (auto& g : lv.geo) minj = std::min(minj, g.n[1]);
  if (minj < 32) return false;
  if (launch5p<16, 64>(lv, a, a_base, b, b_base, r, r_base, cf, clv, c, c_base, st)) return true;
  if (launch5p<16, 32>(lv, a, a_base, b, b_base, r, r_base, cf, clv, c, c_base, st)) return true;
  return false;
}

bool launch_sweep_tma(Level& lv, const Field& a, const double* a_base, const Field& b, double* b_base,
                      const Field& r, const double* r_base, const Coef& cf, const int fixed_lo[3],
                      const int fixed_hi[3], bool fixed, cudaStream_t st, const PushDev* push) {
  // Tile: TK = widest of 64/32/16 dividing every box's k-extent.  C3 fine level
  // (64 boxes of 64^3): k_gsrb_sweep5 104.5 us, k_gsrb_sweep4 114.6 us; see
  // DESIGN.md for the variants measured.
  int mink = 1 << 30, minj = 1 << 30;
  for (auto& g : lv.geo) {
    mink = std::min(mink, g.n[2]);
    minj = std::min(minj, g.n[1]);
  }
  // 16-row tiles (boxes >= 32 in j): k_gsrb_sweep5, D = 2, two CTAs/SM.  8-row
  // tiles (small, L2-resident levels): k_gsrb_sweep4, which measured faster there.
  // AMRB_SWEEP_IMPL=4 forces k_gsrb_sweep4 everywhere (A/B runs).
  static const int impl = getenv("AMRB_SWEEP_IMPL") ? atoi(getenv("AMRB_SWEEP_IMPL")) : 5;
#define AMRB_TRY4(TJ, TK) \
  if (launch4<TJ, TK, 1, 1, false>(lv, a, a_base, b, b_base, r, r_base, cf, fixed_lo, fixed_hi, fixed, st)) return true;
#define AMRB_TRY5(TJ, TK) \
  if (launch5<TJ, TK, 2, 2>(lv, a, a_base, b, b_base, r, r_base, cf, fixed_lo, fixed_hi, fixed, st, push)) return true;
  if (push) {  // only k_gsrb_sweep5 pushes ghosts
    if (minj < 32) return false;
    AMRB_TRY5(16, 64)
    AMRB_TRY5(16, 32)
    return false;
  }
  static const int tk_force = getenv("AMRB_SWEEP_TK") ? atoi(getenv("AMRB_SWEEP_TK")) : 0;
  if (tk_force == 32 && minj >= 32 && impl != 4) {
    AMRB_TRY5(16, 32)
  }

  // Large levels (every box a multiple of 128 in k, >= ~200 plane-steps per
  // CTA slot): 8 x 128 tiles, four cells per lane, amortize the per-step
  // overhead (512^3 in 128^3 boxes: 773.6 -> 708.5 us).  On the C3 fine level
  // (one 256^3 box, ~55 steps per CTA) they measured 107.5 vs 104.6 us.
  {
    long long cells = 0;
    bool k128 = true;
    for (int bx = 0; bx < lv.nboxes; ++bx) {
      if (!lv.resident[bx]) continue;
      const auto& gg = lv.geo[bx];
      cells += (long long)gg.n[0] * gg.n[1] * gg.n[2];
      k128 = k128 && gg.n[2] % 128 == 0 && gg.n[1] % 8 == 0;
    }
    const bool big = cells / 1024 >= 200LL * 2 * num_sms();
    if (impl != 4 && k128 && (big || tk_force == 128) && tk_force != 64 && !push)
      if (launch5<8, 128, 2, 2>(lv, a, a_base, b, b_base, r, r_base, cf, fixed_lo, fixed_hi, fixed, st, push))
        return true;
  }
  // AMRB_SWEEP5_MINCELLS: levels with fewer cells take the k_gsrb_sweep4 tiles (A/B runs)
  static const long long min5 = getenv("AMRB_SWEEP5_MINCELLS") ? atoll(getenv("AMRB_SWEEP5_MINCELLS")) : 0;
  long long lcells = 0;
  for (int bx = 0; bx < lv.nboxes; ++bx)
    if (lv.resident[bx]) lcells += (long long)lv.geo[bx].n[0] * lv.geo[bx].n[1] * lv.geo[bx].n[2];
  if (minj >= 32 && lcells >= min5) {
    if (impl == 4) {
      if (minj >= 64) {
        AMRB_TRY4(16, 64)
        AMRB_TRY4(16, 32)
      }
    } else {
      AMRB_TRY5(16, 64)
      AMRB_TRY5(16, 32)
    }
  }
  AMRB_TRY4(8, 64)
  AMRB_TRY4(8, 32)
  AMRB_TRY4(8, 16)
#undef AMRB_TRY4
#undef AMRB_TRY5
  (void)mink;
  return false;
}

}  // namespace amrb
