// k_gsrb_stream: the fused red+black GSRB sweep, register-streamed (sm_100a).
//
// Same result as the oracle's "fill; red; fill; black" (oracle/mlmg_ref.py
// gsrb_color), bit for bit, written out of place A -> B.  The
// design goal is a kernel bound by HBM, not by the SM:
//
//  * Work unit: a tile column TJ x TK of one box streamed along i over a
//    SEGMENT of planes.  One CTA per (column, segment), all resident at once
//    (one wave), and neighbouring segments stream in opposite directions, so
//    every halo a CTA loads -- the j/k ring of its tile and the two planes past
//    each segment end -- is loaded by its neighbour at about the same time and
//    comes out of L2, not HBM.
//  * Phi (tile + 2-cell halo) and rhs (tile + 1-cell ring) planes arrive by TMA
//    into a ring of D+3 shared slots (one mbarrier per slot, one elected
//    producer).
//  * Each lane owns a k-PAIR (16-byte vectors: LDS.128 / STG.128) in RW rows of
//    the tile ("strip") and keeps that column's values for planes p-1 .. p+2 in
//    registers.  With the i-neighbours and the in-strip j-neighbours in
//    registers, a relaxation reads ~1.5 values from shared memory instead of 7.
//  * Skew 1: step p relaxes red(p+1) then black(p) in the same column.  red(p+1)
//    needs only OLD black values; black(p) needs red(p +- 1) -- both the lane's
//    own -- and the red of plane p's j/k neighbours, stored to shared memory in
//    step p-1.  So a step has ONE __syncthreads: phase A (arrival, red(p+1),
//    residual) | barrier | phase B (publish red(p+1), black(p), store plane p).
//  * Ring warp(s): the red cells of the tile's ghost ring (rows j0-1, j0+TJ and
//    columns k0-1, k0+TK) are recomputed from the halo exactly as the owning
//    tile computes them, so "fill; red; fill; black" needs no fill in between.
//
// Modes: 0 plain sweep; 1 PROL: B = sweep(A + pc(C)) -- every arriving plane
// gets its coarse parent added (the single addition of k_prolong) before
// anything reads it, so the prolongation's read+write pass and its fill
// disappear; 2 NORM: also max |rhs - L(A)| over the valid cells of A (the
// residual of the sweep's INPUT, computed from the same registers), atomically
// max-ed into a u64 (non-negative doubles order like their bit patterns).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "tma.cuh"
#include "peer.cuh"

namespace amrb {

// ---------------------------------------------------------------------------
// tensor maps (shared with the other TMA kernels)
// ---------------------------------------------------------------------------
namespace {
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
}  // namespace

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
    if (gb.n[0] != g0.n[0] || gb.n[1] != g0.n[1] || gb.n[2] != g0.n[2] || v.s0 != v0.s0 || v.s1 != v0.s1) return d;
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

namespace {

constexpr int kModePlain = 0, kModeProl = 1, kModeNorm = 2;

struct StreamArgs {
  const int* seg;  // 8 ints per CTA: box, j0, k0, i0, i1, dir, -, -  (box-local valid coords)
  const BoxGeom* geo;
  const FabView* fb;  // output views
  double* b;
  int64_t b_elems;  // size of the output allocation (checked builds)
  unsigned int* dcheck;  // checked builds: {failures, line}
  const int* slot;  // per box: block index in the tensor maps
  Coef cf;
  int a_kc, a_jc, a_ic;  // tensor coordinate of phi cell (i, j0-2, k0-2) = (i + a_ic, j0 + a_jc, k0 + a_kc)
  int r_kc, r_jc, r_ic;  // rhs (i, j0-1, k0-2)
  int c_kc, c_jc, c_ic;  // coarse (i>>1, j0/2-1, k0/2-1) before the even-column shift
  int flo[3], fhi[3];    // cells outside [flo, fhi] (global) are never relaxed
  unsigned long long* norm;  // kModeNorm
  // ghost push (ghosts.py): per box 27 destination base addresses (0: none);
  // the ghost copy of output cell (i, j, k) of box b toward direction
  // (dx, dy, dz) is at push[27 b + 9 (dx+1) + 3 (dy+1) + (dz+1)] + i s0 + j s1 + k
  const long long* push;
  int push_fence;
  // in-kernel ghost pull (ghosts.pull_table): per box 27 source addresses (0:
  // none; bit 0 set: the source box is on another GPU); the INPUT's ghost cell
  // (i, j, k) (box-local, inside direction d's width-2 slab) is copied from
  // (pull[27 b + d] & ~1) + i s0 + j s1 + k (elements, the input's strides)
  // before the CTA's first TMA load -- the copy-program fill disappears.  The
  // CTAs whose footprint reaches a remote slab (and CTA 0) first wait for
  // every peer to reach this launch: k_copy's fused device barrier, same pads
  // and epoch (comm.cu).
  const long long* pull;
  double* a;          // the input's allocation (ghost destinations)
  const FabView* fa;  // the input's views
  uint32_t* pads[kMaxPeers];
  uint32_t* epoch;
  int rank, nranks;
  Fault fault;
};

constexpr int r128(int x) { return (x + 127) / 128 * 128; }

template <int TJ, int TK, int D, int MODE>
struct StreamLayout {
  static constexpr int NS = D + 3;       // ring slots
  static constexpr int PK = TK + 4;      // smem row pitch: cols k0-2 .. k0+TK+1
  static constexpr int PJ = TJ + 4;      // phi rows j0-2 .. j0+TJ+1
  static constexpr int RJ = TJ + 2;      // rhs rows j0-1 .. j0+TJ
  static constexpr int CJ = TJ / 2 + 2;  // PROL coarse rows j0/2-1 .. j0/2+TJ/2
  static constexpr int CK = TK / 2 + 4;  // PROL coarse cols from the even column at or below k0/2-1
  static constexpr int PB = PJ * PK * 8, RB = RJ * PK * 8, CB = CJ * CK * 8;
  static constexpr int ROFF = r128(PB);
  static constexpr int COFF = ROFF + r128(RB);
  static constexpr int SLOT = COFF + (MODE == kModeProl ? r128(CB) : 0);
  static constexpr int BAR = NS * SLOT;
  static constexpr int PTAB = BAR + 8 * NS;  // PUSH / PULL: this box's 27 table entries
  static constexpr int BYTES = PTAB + 8 * 27;
  // lanes per tile row: 32 k-pairs per warp for TK >= 64 (WK warps across k),
  // else TK/2 lanes per row and RPW = 32 / LK row groups per warp
  static constexpr int WK = TK >= 64 ? TK / 64 : 1;
  static constexpr int LK = TK >= 64 ? 32 : TK / 2;
  static constexpr int RPW = 32 / LK;
};

template <int TJ, int TK, int RW>
__host__ __device__ constexpr int stream_warps() {
  return (TJ / (RW * (TK >= 64 ? 1 : 64 / TK)) + 1) * (TK >= 64 ? TK / 64 : 1);
}

__device__ __forceinline__ double2 lds2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void sts2(double* p, double x, double y) { *reinterpret_cast<double2*>(p) = make_double2(x, y); }

// x / d for 0 <= x < 2^22 through a float reciprocal (off by at most one,
// corrected): the pull's index math without the ~20-instruction integer
// division chain per cell
__device__ __forceinline__ int quick_div(int x, int d, float rcp) {
  int q = __float2int_rz(__int2float_rz(x) * rcp);
  const int r = x - q * d;
  q += (r >= d) - (r < 0);
  return q;
}

// In-kernel ghost pull of one CTA's input footprint (planes fi0..fi1, rows
// fj0..fj1, cols fk0..fk1, box-local; see StreamArgs::pull).  Every CTA whose
// footprint holds a ghost cell copies that cell itself, so a CTA's TMA only
// ever reads ghost values it (or a neighbour, with the same value) wrote.
template <int NT>
__device__ __forceinline__ void pull_ghosts(const StreamArgs& args, long long* tab, int box, const BoxGeom& g, int fi0,
                                            int fi1, int fj0, int fj1, int fk0, int fk1) {
  const int tid = threadIdx.x;
  if (tid < 27) tab[tid] = args.pull[27 * box + tid];
  __syncthreads();
  const int flo[3] = {fi0, fj0, fk0}, fhi[3] = {fi1, fj1, fk1};
  // the footprint's part of direction d's ghost slab (width 2)
  auto part = [&](int d, int lo[3], int hi[3]) {
    const int dd[3] = {d / 9 - 1, (d / 3) % 3 - 1, d % 3 - 1};
    bool any = true;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      const int slo = dd[ax] < 0 ? -2 : (dd[ax] > 0 ? g.n[ax] : 0);
      const int shi = dd[ax] < 0 ? -1 : (dd[ax] > 0 ? g.n[ax] + 1 : g.n[ax] - 1);
      lo[ax] = max(flo[ax], slo);
      hi[ax] = min(fhi[ax], shi);
      any &= lo[ax] <= hi[ax];
    }
    return any;
  };
  if (args.nranks > 1) {
    const uint32_t ep = *reinterpret_cast<volatile uint32_t*>(args.epoch) + 1;
    if (tid < 32) {
      bool wait = blockIdx.x == 0;
      int lo[3], hi[3];
      for (int d = 0; d < 27 && !wait; ++d)
        if (d != 13 && (tab[d] & 1)) wait = part(d, lo, hi);
      const int p = tid;
      if (p < args.nranks && p != args.rank) {
        if (blockIdx.x == 0) signal_store(args.pads[p] + args.rank, ep);
        if (wait) peer_wait(args.pads[args.rank] + p, ep, args.rank, p, args.fault);
      }
      // every CTA has read the old epoch once all have taken a ticket
      if (tid == 0 && atomicAdd(args.epoch + 1, 1u) == gridDim.x - 1) {
        args.epoch[0] = ep;
        args.epoch[1] = 0;
      }
    }
    __syncthreads();
  }
  const FabView A = args.fa[box];
  double* dst = args.a + A.off;
  for (int d = 0; d < 27; ++d) {
    const long long e = tab[d];
    int lo[3], hi[3];
    if (d == 13 || !e || !part(d, lo, hi)) continue;
    const int e1 = hi[1] - lo[1] + 1, e2 = hi[2] - lo[2] + 1;
    const int total = (hi[0] - lo[0] + 1) * e1 * e2;
    const float r1 = 1.0f / (float)e1, r2 = 1.0f / (float)e2;
    const double* src = reinterpret_cast<const double*>(e & ~1ll);
    constexpr int U = 16;  // loads in flight per thread (NVLink latency)
    for (int base = 0; base < total; base += U * NT) {
      double v[U];
      int64_t o[U];  // box-local offsets: negative for the low ghost slabs
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int x = base + u * NT + tid;
        if (x < total) {
          const int r = quick_div(x, e2, r2), i = quick_div(r, e1, r1);
          const int k = x - r * e2, j = r - i * e1;
          o[u] = (int64_t)(lo[0] + i) * A.s0 + (int64_t)(lo[1] + j) * A.s1 + (lo[2] + k);
          v[u] = src[o[u]];
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (base + u * NT + tid < total) dst[o[u]] = v[u];
    }
  }
  // generic-proxy stores before this CTA's TMA (async proxy) reads of them
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}

// XCH: 0 = plain, 1 = ghost push (args.push), 2 = ghost pull (args.pull)
template <int TJ, int TK, int RW, int D, int MODE, int MINB, int XCH>
__global__ void __launch_bounds__(32 * stream_warps<TJ, TK, RW>(), MINB)
    k_gsrb_stream(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmR,
                  const __grid_constant__ CUtensorMap tmC, const __grid_constant__ StreamArgs args) {
  pdl_entry();
#define AMRB_DCHECK(cond) AMRB_DCHECK_AT(args.dcheck, cond)
  using LY = StreamLayout<TJ, TK, D, MODE>;
  constexpr int WK = LY::WK, LK = LY::LK, RPW = LY::RPW, NS = LY::NS, PK = LY::PK, CK = LY::CK;
  constexpr int NSW = TJ / (RW * RPW) * WK;  // strip warps (then WK ring warps)
  constexpr bool PROL = MODE == kModeProl, NORM = MODE == kModeNorm;
  constexpr bool PUSH = XCH == 1, PULL = XCH == 2;
  static_assert((TK % 64 == 0 || TK == 32) && TJ % (RW * RPW) == 0 && RW % 2 == 0 && TJ + 2 <= 32, "tile shape");
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + LY::BAR);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int producer = 32 * NSW;  // lane 0 of ring warp 0
  const Coef cf = args.cf;

  const int* sg = args.seg + 8 * blockIdx.x;
  const int box = sg[0], j0 = sg[1], k0 = sg[2], i0 = sg[3], i1 = sg[4], dir = sg[5];
  const int L = i1 - i0;
  const int istart = dir > 0 ? i0 : i1 - 1;  // box-local plane of stream position 0
  const BoxGeom g = args.geo[box];
  AMRB_DCHECK(0 <= i0 && i0 < i1 && i1 <= g.n[0] && (dir == 1 || dir == -1));
  AMRB_DCHECK(0 <= j0 && j0 + TJ <= g.n[1] && 0 <= k0 && k0 + TK <= g.n[2]);
  const int bslot = args.slot[box];
  const int gj0 = g.lo[1] + j0, gk0 = g.lo[2] + k0;
  const int cshift = ((k0 >> 1) + args.c_kc) & 1;

  auto plane = [&](int q) { return istart + dir * q; };
  auto slot_base = [&](int q) { return sm + ((q + 2) % NS) * LY::SLOT; };  // phi position q (q >= -2)
  auto phi_s = [&](int q) { return reinterpret_cast<double*>(slot_base(q)); };
  auto rhs_s = [&](int q) { return reinterpret_cast<const double*>(slot_base(q + 1) + LY::ROFF); };  // rides with phi q+1
  auto crs_s = [&](int q) { return reinterpret_cast<const double*>(slot_base(q) + LY::COFF); };
  auto wait_pos = [&](int q) {
    AMRB_DCHECK(q >= -2 && q <= L + 1);
    mbar_wait(&bars[(q + 2) % NS], (unsigned)(((q + 2) / NS) & 1));
  };
  auto issue = [&](int q) {  // phi position q, rhs position q-1 (from q = 0), coarse parent plane
    AMRB_DCHECK(q >= -2 && q <= L + 1);
    uint64_t* bar = &bars[(q + 2) % NS];
    const bool wr = q >= 0;
    mbar_expect_tx(bar, LY::PB + (wr ? LY::RB : 0) + (PROL ? LY::CB : 0));
    const int ip = plane(q);
    tma_load4(slot_base(q), &tmA, bar, k0 + args.a_kc, j0 + args.a_jc, ip + args.a_ic, bslot);
    if (wr) tma_load4(slot_base(q) + LY::ROFF, &tmR, bar, k0 + args.r_kc, j0 + args.r_jc, plane(q - 1) + args.r_ic, bslot);
    if (PROL)
      tma_load4(slot_base(q) + LY::COFF, &tmC, bar, (k0 >> 1) + args.c_kc - cshift, (j0 >> 1) + args.c_jc,
                (ip >> 1) + args.c_ic, bslot);
  };

  // never-relaxed (fixed) ring cells: the tile's ring outside the domain
  auto plane_ok = [&](int q) {
    const int gi = g.lo[0] + plane(q);
    return gi >= args.flo[0] && gi <= args.fhi[0];
  };
  const bool top_ok = gj0 - 1 >= args.flo[1], bot_ok = gj0 + TJ <= args.fhi[1];
  const bool lft_ok = gk0 - 1 >= args.flo[2], rgt_ok = gk0 + TK <= args.fhi[2];

  if (tid == producer) {
    for (int x = 0; x < NS; ++x) mbar_init(&bars[x], 1);
    fence_barrier_init();
  }
  if (PUSH && tid < 27) reinterpret_cast<long long*>(sm + LY::PTAB)[tid] = args.push[27 * box + tid];
  if (PULL) pull_ghosts<32 * stream_warps<TJ, TK, RW>()>(args, reinterpret_cast<long long*>(sm + LY::PTAB), box, g,
                                                         i0 - 2, i1 + 1, j0 - 2, j0 + TJ + 1, k0 - 2, k0 + TK + 1);
  __syncthreads();
  if (tid == producer)
    for (int q = -2; q <= min(NS - 3, L + 1); ++q) issue(q);

  // ---- roles ---------------------------------------------------------------
  const bool strip = warp < NSW;
  const int wk = strip ? warp % WK : warp - NSW;
  const int rg = lane / LK;              // row group of the lane (RPW > 1: narrow tiles)
  const int m = LK * wk + lane % LK;     // k-pair index in the tile
  const int c0 = 2 + 2 * m;              // smem column of the pair's first cell
  const int r0 = 2 + (strip ? ((warp / WK) * RPW + rg) * RW : 0);  // strip: first smem row

  // strip state (row x = smem row r0 + x): pairs of planes p, p+1, p+2
  double a0[RW][2], a1[RW][2], a2[RW][2], am[RW], rs[RW], ao[RW];
  // ring-row state (h = 0: row 1, h = 1: row TJ+2)
  double g0[2][2], g1[2][2], g2[2][2];
  unsigned long long nmax = 0;  // NORM: max |r| as bit pattern (NaN sorts above +inf)

  double* out = nullptr;
  int64_t ostep = 0;
  if (strip) {
    const FabView B = args.fb[box];
    out = args.b + B.off + (int64_t)istart * B.s0 + (int64_t)(j0 + r0 - 2) * B.s1 + (k0 + 2 * m);
    ostep = dir * B.s0;
    AMRB_DCHECK(r0 >= 2 && r0 + RW <= TJ + 2 && c0 >= 2 && c0 + 1 <= TK + 1);
  }
  const int64_t orow = strip ? args.fb[box].s1 : 0;
  bool pushed = false;
  // Ghost push of the plane just written (strip rows of this lane): a cell
  // within 2 of a box face also goes to the neighbour(s) across it; the
  // destination of each nonempty subset of its near faces is one entry of the
  // box's table (staged in shared memory).  A lane's column fixes its row and
  // column classes for the whole segment, so warps away from the box's j / k
  // edges only push the first and last two planes of the box.
  const long long* ptab = reinterpret_cast<const long long*>(sm + LY::PTAB);
  const int kk_ = k0 + 2 * m;
  const int ck_ = kk_ < 2 ? 0 : (kk_ >= g.n[2] - 2 ? 2 : 1);
  int cjs = 0;  // 2 bits per strip row: the row's class
#pragma unroll
  for (int x = 0; x < RW; ++x) {
    const int jj = j0 + r0 - 2 + x;
    cjs |= (jj < 2 ? 0 : (jj >= g.n[1] - 2 ? 2 : 1)) << (2 * x);
  }
  const bool jk_edge = PUSH && strip && __any_sync(0xffffffffu, ck_ != 1 || cjs != 0x55555555 >> (32 - 2 * RW));
  auto push_plane = [&](int ip) {
    const int ci = ip < 2 ? 0 : (ip >= g.n[0] - 2 ? 2 : 1);
    if (ci == 1 && !jk_edge) return;  // warp-uniform
    const int64_t pbase = (int64_t)ip * ostep * dir + kk_;
#pragma unroll
    for (int x = 0; x < RW; ++x) {
      const int cj = (cjs >> (2 * x)) & 3;
      const int64_t rel = pbase + (int64_t)(j0 + r0 - 2 + x) * orow;
      const double2 v = make_double2(a0[x][0], a0[x][1]);
      auto put = [&](int a, int b, int c) {
        const long long dst = ptab[a * 9 + b * 3 + c];
        if (dst) {
          *reinterpret_cast<double2*>(reinterpret_cast<double*>(dst) + rel) = v;
          pushed = true;
        }
      };
      if (cj != 1) put(1, cj, 1);
      if (ck_ != 1) put(1, 1, ck_);
      if (cj != 1 && ck_ != 1) put(1, cj, ck_);
      if (ci != 1) {
        put(ci, 1, 1);
        if (cj != 1) put(ci, cj, 1);
        if (ck_ != 1) put(ci, 1, ck_);
        if (cj != 1 && ck_ != 1) put(ci, cj, ck_);
      }
    }
  };
  // PROL: a plane tile holds the fine values BEFORE the prolongation; every
  // read of a not-yet-relaxed value adds its coarse parent on the fly (the
  // single addition of k_prolong, so the bits equal prolong-then-sweep).
  // Relaxed values written back to shared memory already include it.
  auto parent = [&](int q, int off) {  // smem offset off = r * PK + c of plane position q
    const int r = off / PK, c = off - r * PK;
    return crs_s(q)[(r >> 1) * CK + (c >> 1) + cshift];
  };
  auto old = [&](const double* S, int q, int off) { return PROL ? S[off] + parent(q, off) : S[off]; };
  // arrival of plane position q: own pairs to registers
  auto arrive_strip = [&](int q, double (&dst)[RW][2]) {
    const double* S = phi_s(q);
#pragma unroll
    for (int x = 0; x < RW; ++x) {
      const double2 v = lds2(S + (r0 + x) * PK + c0);
      const double cp = PROL ? parent(q, (r0 + x) * PK + c0) : 0.0;  // one parent per pair
      dst[x][0] = PROL ? v.x + cp : v.x;
      dst[x][1] = PROL ? v.y + cp : v.y;
    }
  };
  auto arrive_ring = [&](int q, double (&dst)[2][2]) {
    const double* S = phi_s(q);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const double2 v = lds2(S + (h ? TJ + 2 : 1) * PK + c0);
      const double cp = PROL ? parent(q, (h ? TJ + 2 : 1) * PK + c0) : 0.0;
      dst[h][0] = PROL ? v.x + cp : v.x;
      dst[h][1] = PROL ? v.y + cp : v.y;
    }
  };

  // prologue: positions -2, -1
  wait_pos(-2);
  wait_pos(-1);
  if (strip) {
    arrive_strip(-2, a0);
    arrive_strip(-1, a1);
#pragma unroll
    for (int x = 0; x < RW; ++x) am[x] = rs[x] = ao[x] = 0.0;
  } else {
    arrive_ring(-2, g0);
    arrive_ring(-1, g1);
  }
  __syncthreads();

  // One step per role; PHI = the pair element relaxed in strip row 0
  // (b = (PHI + x) & 1); UP: the stream runs toward +i.  lap7's operand order
  // is fixed (i-1 before i+1), so the stream neighbours go in plane order.
  // Strip and ring warps run separate loops (their register state never
  // overlaps) that meet at the same __syncthreads once per step.
  auto strip_step = [&](auto phi_tag, auto up_tag, int p) {
    constexpr int PHI = decltype(phi_tag)::value;
    constexpr bool UP = decltype(up_tag)::value;
    auto lapi = [&](double c, double prev, double next, double ym, double yp, double zm, double zp) {
      return UP ? lap7(c, prev, next, ym, yp, zm, zp, cf) : lap7(c, next, prev, ym, yp, zm, zp, cf);
    };
    wait_pos(p + 2);
    const double* S0 = phi_s(p);
    double* S1 = phi_s(p + 1);
    const double* R1 = rhs_s(p + 1);
    const bool red_on = (p + 1 >= 0 && p + 1 < L) || plane_ok(p + 1);
    double nr[RW], rsn[RW];
    arrive_strip(p + 2, a2);
    // ---- phase A: red(p+1) in column (r, c0 + b); NORM: residual of plane p+1
#pragma unroll
    for (int x = 0; x < RW; ++x) {
      const int b = (PHI + x) & 1;  // compile-time after unrolling
      const int row = (r0 + x) * PK;
      const double c = a1[x][b];
      const double ym = x > 0 ? a1[x > 0 ? x - 1 : 0][b] : old(S1, p + 1, row - PK + c0 + b);
      const double yp = x < RW - 1 ? a1[x < RW - 1 ? x + 1 : 0][b] : old(S1, p + 1, row + PK + c0 + b);
      const double kn = old(S1, p + 1, b ? row + c0 + 2 : row + c0 - 1);  // the neighbour pair's cell
      const double zm = b ? a1[x][0] : kn;
      const double zp = b ? kn : a1[x][1];
      const double2 rr = lds2(R1 + row - PK + c0);
      const double rb = b ? rr.y : rr.x;
      rsn[x] = b ? rr.x : rr.y;
      const double d = rb - lapi(c, a0[x][b], a2[x][b], ym, yp, zm, zp);
      nr[x] = c + d * cf.rgamma;
      if (NORM && p + 1 >= 0 && p + 1 < L) {
        // the other cell of the pair (black in plane p+1), old values only
        const int o = 1 - b;
        const double ym2 = x > 0 ? a1[x > 0 ? x - 1 : 0][o] : S1[row - PK + c0 + o];
        const double yp2 = x < RW - 1 ? a1[x < RW - 1 ? x + 1 : 0][o] : S1[row + PK + c0 + o];
        const double kn2 = o ? S1[row + c0 + 2] : S1[row + c0 - 1];
        const double zm2 = o ? a1[x][0] : kn2;
        const double zp2 = o ? kn2 : a1[x][1];
        const double d2 = rsn[x] - lapi(a1[x][o], ao[x], a2[x][o], ym2, yp2, zm2, zp2);
        nmax = max(nmax, max((unsigned long long)__double_as_longlong(fabs(d)),
                             (unsigned long long)__double_as_longlong(fabs(d2))));
      }
    }
    __syncthreads();
    // ---- phase B: publish red(p+1); black(p); plane p out
#pragma unroll
    for (int x = 0; x < RW; ++x) {
      const int b = (PHI + x) & 1;
      if (red_on) S1[(r0 + x) * PK + c0 + b] = nr[x];
    }
    if (p >= 0) {
#pragma unroll
      for (int x = 0; x < RW; ++x) {
        const int b = (PHI + x) & 1;
        const int row = (r0 + x) * PK;
        const double c = a0[x][b];
        const double ym = x > 0 ? a0[x > 0 ? x - 1 : 0][b] : S0[row - PK + c0 + b];
        const double yp = x < RW - 1 ? a0[x < RW - 1 ? x + 1 : 0][b] : S0[row + PK + c0 + b];
        const double kn = b ? S0[row + c0 + 2] : S0[row + c0 - 1];
        const double zm = b ? a0[x][0] : kn;
        const double zp = b ? kn : a0[x][1];
        const double xp = red_on ? nr[x] : a1[x][b];
        a0[x][b] = relax(c, rs[x], lapi(c, am[x], xp, ym, yp, zm, zp), cf.rgamma);
      }
#pragma unroll
      for (int x = 0; x < RW; ++x) {
        AMRB_DCHECK(out + x * orow >= args.b && out + x * orow + 2 <= args.b + args.b_elems &&
                    ((reinterpret_cast<uintptr_t>(out + x * orow) & 15) == 0));
        *reinterpret_cast<double2*>(out + x * orow) = make_double2(a0[x][0], a0[x][1]);
      }
      out += ostep;
      if (PUSH) push_plane(plane(p));
    }
#pragma unroll
    for (int x = 0; x < RW; ++x) {
      const int b = (PHI + x) & 1;
      am[x] = a0[x][1 - b];
      ao[x] = a1[x][b];
      a0[x][0] = a1[x][0];
      a0[x][1] = a1[x][1];
      if (red_on) a0[x][b] = nr[x];
      a1[x][0] = a2[x][0];
      a1[x][1] = a2[x][1];
      rs[x] = rsn[x];
    }
    if (p + 1 + NS <= L + 1) fence_proxy_async();  // our shared stores before a later TMA into the slot
  };

  auto ring_step = [&](auto phi_tag, auto up_tag, int p) {
    constexpr int PHI = decltype(phi_tag)::value;
    constexpr bool UP = decltype(up_tag)::value;
    auto lapi = [&](double c, double prev, double next, double ym, double yp, double zm, double zp) {
      return UP ? lap7(c, prev, next, ym, yp, zm, zp, cf) : lap7(c, next, prev, ym, yp, zm, zp, cf);
    };
    wait_pos(p + 2);
    const double* S0 = phi_s(p);
    double* S1 = phi_s(p + 1);
    const double* S2 = phi_s(p + 2);
    const double* R1 = rhs_s(p + 1);
    const bool red_on = (p + 1 >= 0 && p + 1 < L) || plane_ok(p + 1);
    double rv[2], rc = 0.0;  // ring rows / ring column red(p+1)
    int rco = 0;             // ring column cell offset
    bool rcok = false;
    arrive_ring(p + 2, g2);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (RPW > 1 && h != rg) continue;  // narrow tiles: one ring row per row group
      const int b = h ? PHI : 1 - PHI;
      const int row = (h ? TJ + 2 : 1) * PK;
      const double kn = old(S1, p + 1, b ? row + c0 + 2 : row + c0 - 1);
      const double zm = b ? g1[h][0] : kn;
      const double zp = b ? kn : g1[h][1];
      const double c = g1[h][b];
      const double rb = R1[row - PK + c0 + b];
      rv[h] = relax(c, rb, lapi(c, g0[h][b], g2[h][b], old(S1, p + 1, row - PK + c0 + b), old(S1, p + 1, row + PK + c0 + b),
                                zm, zp),
                    cf.rgamma);
    }
    if (wk == 0 && lane < TJ + 2) {
      constexpr int HALF = (TJ + 2) / 2;
      const int side = lane >= HALF;
      const int idx = lane - side * HALF;
      const int cc = side ? TK + 2 : 1;
      const int rr = 1 + 2 * idx + (side ? 1 - PHI : PHI);
      rco = rr * PK + cc;
      AMRB_DCHECK(rr >= 1 && rr <= TJ + 2 && rco - PK >= 0 && rco + PK < LY::PJ * PK);
      const double c = old(S1, p + 1, rco);
      rc = relax(c, R1[rco - PK], lapi(c, old(S0, p, rco), old(S2, p + 2, rco), old(S1, p + 1, rco - PK),
                                       old(S1, p + 1, rco + PK), old(S1, p + 1, rco - 1), old(S1, p + 1, rco + 1)),
                 cf.rgamma);
      rcok = (side ? rgt_ok : lft_ok) && (rr != 1 || top_ok) && (rr != TJ + 2 || bot_ok);
    }
    __syncthreads();
    if (tid == producer && p >= -1 && p - 1 + NS <= L + 1) issue(p - 1 + NS);
    if (red_on) {
      if (top_ok && (RPW == 1 || rg == 0)) S1[1 * PK + c0 + (1 - PHI)] = rv[0];
      if (bot_ok && (RPW == 1 || rg == 1)) S1[(TJ + 2) * PK + c0 + PHI] = rv[1];
      if (rcok) S1[rco] = rc;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      g0[h][0] = g1[h][0];
      g0[h][1] = g1[h][1];
      g1[h][0] = g2[h][0];
      g1[h][1] = g2[h][1];
    }
    if (p + 1 + NS <= L + 1) fence_proxy_async();
  };

  // PHI of stream position p: b of strip row 0 = 1 - ((i + j0 + k0) & 1), global
  auto run = [&](auto up_tag, auto& stepfn) {
    using I0 = std::integral_constant<int, 0>;
    using I1 = std::integral_constant<int, 1>;
    int p = -2;
    const int par = (g.lo[0] + plane(-2) + gj0 + gk0) & 1;  // PHI flips every step
    if (par == 0) {
      stepfn(I1{}, up_tag, p);
      ++p;
    }
    for (; p + 1 < L; p += 2) {
      stepfn(I0{}, up_tag, p);
      stepfn(I1{}, up_tag, p + 1);
    }
    if (p < L) stepfn(I0{}, up_tag, p);
  };
  if (strip) {
    if (dir > 0)
      run(std::true_type{}, strip_step);
    else
      run(std::false_type{}, strip_step);
  } else {
    if (dir > 0)
      run(std::true_type{}, ring_step);
    else
      run(std::false_type{}, ring_step);
  }

#undef AMRB_DCHECK
  // Pushes to peers before the consumer's device barrier: the barrier is
  // signalled by a LATER kernel on this stream, and a kernel completes only
  // once its stores (NVLink ones included) are acknowledged, so no fence is
  // needed here; a system-scope fence would also wait behind in-flight PCIe
  // copies.  (Library option "push_fence" = 1 restores it, for A/B runs.)
  if (PUSH && pushed && args.push_fence) __threadfence_system();
  if (NORM) {
    for (int o = 16; o; o >>= 1) nmax = max(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
    if (strip && lane == 0 && nmax) atomicMax(args.norm, nmax);
  }
}

// ---------------------------------------------------------------------------
// k_resid_restrict_stream: crse = average_down(rhs - L(phi)) (coarse_fine.py:
// 136-163 applied to the residual, the V-cycle's down-leg transfer), streamed
// like the sweep: phi (+ halo) and rhs plane tiles by TMA, each lane owning a
// k-pair of RW rows and its column's planes q-1 .. q+1 in registers, j/k
// neighbours from shared memory (read only: nothing is written back), one
// barrier per plane for the ring.  A k-pair x row-pair x plane-pair is one
// coarse cell: the pair sums of plane 2I are kept until plane 2I+1 arrives and
// the eight residuals are summed in numpy's reshape-mean order
// ((((c000+c001) + (c010+c011)) + (c100+c101)) + (c110+c111)) * 0.125 (avg8 in
// stencil.cu).  Segments start on even planes; a downward segment meets the
// odd plane of a pair first and keeps its pair sums instead.
// ---------------------------------------------------------------------------
struct RRArgs {
  const int* seg;
  const BoxGeom* geo;
  const FabView* fc;  // coarse views (box-local coarsening of the fine boxes)
  double* crse;
  const int* slot;
  Coef cf;
  int a_kc, a_jc, a_ic, r_kc, r_jc, r_ic;
};

template <int TJ, int TK, int RW, int D>
__global__ void __launch_bounds__(32 * (TJ / (RW * (TK >= 64 ? 1 : 64 / TK))) * (TK >= 64 ? TK / 64 : 1))
    k_resid_restrict_stream(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmR,
                            const __grid_constant__ RRArgs args) {
  pdl_entry();
  using LY = StreamLayout<TJ, TK, D, kModePlain>;
  constexpr int WK = LY::WK, LK = LY::LK, RPW = LY::RPW, NS = LY::NS, PK = LY::PK;
  static_assert(RW % 2 == 0, "row pairs");
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + LY::BAR);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Coef cf = args.cf;
  const int* sg = args.seg + 8 * blockIdx.x;
  const int box = sg[0], j0 = sg[1], k0 = sg[2], i0 = sg[3], i1 = sg[4], dir = sg[5];
  const int L = i1 - i0;
  const int istart = dir > 0 ? i0 : i1 - 1;
  const int bslot = args.slot[box];
  auto plane = [&](int q) { return istart + dir * q; };
  // phi position q in slot (q + 1) % NS (q >= -1); rhs position q rides with phi q+1
  auto slot_base = [&](int q) { return sm + ((q + 1) % NS) * LY::SLOT; };
  auto phi_s = [&](int q) { return reinterpret_cast<const double*>(slot_base(q)); };
  auto rhs_s = [&](int q) { return reinterpret_cast<const double*>(slot_base(q + 1) + LY::ROFF); };
  auto wait_pos = [&](int q) { mbar_wait(&bars[(q + 1) % NS], (unsigned)(((q + 1) / NS) & 1)); };
  auto issue = [&](int q) {  // phi position q (q = -1 .. L), rhs position q-1 (from q = 1)
    uint64_t* bar = &bars[(q + 1) % NS];
    const bool wr = q >= 1;
    mbar_expect_tx(bar, LY::PB + (wr ? LY::RB : 0));
    tma_load4(slot_base(q), &tmA, bar, k0 + args.a_kc, j0 + args.a_jc, plane(q) + args.a_ic, bslot);
    if (wr) tma_load4(slot_base(q) + LY::ROFF, &tmR, bar, k0 + args.r_kc, j0 + args.r_jc, plane(q - 1) + args.r_ic, bslot);
  };
  if (tid == 0) {
    for (int x = 0; x < NS; ++x) mbar_init(&bars[x], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int q = -1; q <= min(NS - 2, L); ++q) issue(q);

  const int wk = warp % WK;
  const int rg = lane / LK;
  const int m = LK * wk + lane % LK;
  const int c0 = 2 + 2 * m;
  const int r0 = 2 + ((warp / WK) * RPW + rg) * RW;
  const FabView Cv = args.fc[box];
  // coarse row of strip row pair x/2, coarse column of the pair
  double* cout = args.crse + Cv.off + (int64_t)((j0 + r0 - 2) >> 1) * Cv.s1 + ((k0 + 2 * m) >> 1);
  double a0[RW][2], a1[RW][2], a2[RW][2], keep[RW / 2][2];
  auto arrive = [&](int q, double (&dst)[RW][2]) {
    const double* S = phi_s(q);
#pragma unroll
    for (int x = 0; x < RW; ++x) {
      const double2 v = lds2(S + (r0 + x) * PK + c0);
      dst[x][0] = v.x;
      dst[x][1] = v.y;
    }
  };
  wait_pos(-1);
  wait_pos(0);
  arrive(-1, a0);
  arrive(0, a1);
  auto step = [&](auto up_tag, int q) {
    constexpr bool UP = decltype(up_tag)::value;
    wait_pos(q + 1);
    arrive(q + 1, a2);
    const double* S = phi_s(q);
    const double* R = rhs_s(q);
    double r[RW][2];
#pragma unroll
    for (int x = 0; x < RW; ++x) {
      const int row = (r0 + x) * PK;
      const double2 rh = lds2(R + row - PK + c0);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double c = a1[x][e];
        const double prev = a0[x][e], next = a2[x][e];
        const double ym = x > 0 ? a1[x > 0 ? x - 1 : 0][e] : S[row - PK + c0 + e];
        const double yp = x < RW - 1 ? a1[x < RW - 1 ? x + 1 : 0][e] : S[row + PK + c0 + e];
        const double zm = e ? a1[x][0] : S[row + c0 - 1];
        const double zp = e ? S[row + c0 + 2] : a1[x][1];
        const double lap = UP ? lap7(c, prev, next, ym, yp, zm, zp, cf) : lap7(c, next, prev, ym, yp, zm, zp, cf);
        r[x][e] = (e ? rh.y : rh.x) - lap;
      }
    }
    const int ip = plane(q);
    const bool first = UP ? (ip & 1) == 0 : (ip & 1) == 1;  // first plane of its pair in stream order
#pragma unroll
    for (int h = 0; h < RW / 2; ++h) {
      const double pr = r[2 * h][0] + r[2 * h][1];          // pair sum, row 2h
      const double qr = r[2 * h + 1][0] + r[2 * h + 1][1];  // pair sum, row 2h+1
      if (first) {
        keep[h][0] = pr;
        keep[h][1] = qr;
      } else {
        // even plane's (P0, Q0), odd plane's (P1, Q1): ((P0 + Q0) + P1) + Q1
        const double s = UP ? ((keep[h][0] + keep[h][1]) + pr) + qr : ((pr + qr) + keep[h][0]) + keep[h][1];
        cout[(int64_t)(ip >> 1) * Cv.s0 + (int64_t)h * Cv.s1] = s * 0.125;
      }
    }
#pragma unroll
    for (int x = 0; x < RW; ++x) {
      a0[x][0] = a1[x][0];
      a0[x][1] = a1[x][1];
      a1[x][0] = a2[x][0];
      a1[x][1] = a2[x][1];
    }
    __syncthreads();  // everyone is done with phi q-1's slot (and rhs q-1)
    if (tid == 0 && q + NS - 1 <= L) issue(q + NS - 1);
  };
  if (dir > 0)
    for (int q = 0; q < L; ++q) step(std::true_type{}, q);
  else
    for (int q = 0; q < L; ++q) step(std::false_type{}, q);
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
// (column, segment) work items: every resident box cut into TJ x TK columns,
// each column into nseg near-equal plane ranges; odd segments stream downward.
// Cached on the Level.
const SegTable& seg_table(Level& lv, int tj, int tk, int nseg, bool alternate, bool even = false) {
  auto key = std::make_tuple(tj * (even ? -1 : 1), tk, alternate ? nseg : -nseg);
  auto it = lv.segtabs.find(key);
  if (it != lv.segtabs.end()) return *it->second;
  auto* t = new SegTable;
  for (int b = 0; b < lv.nboxes; ++b) {
    if (!lv.resident[b]) continue;
    const BoxGeom& gb = lv.geo[b];
    const int ns = std::max(1, std::min(nseg, gb.n[0] / 4));
    for (int j = 0; j < gb.n[1]; j += tj)
      for (int k = 0; k < gb.n[2]; k += tk)
        for (int s = 0; s < ns; ++s) {
          int a = (int)((long long)gb.n[0] * s / ns), e = (int)((long long)gb.n[0] * (s + 1) / ns);
          if (even) {  // plane pairs stay inside one segment
            a &= ~1;
            e = s + 1 == ns ? gb.n[0] : (e & ~1);
          }
          if (e <= a) continue;
          const int v[8] = {b, j, k, a, e, (alternate && (s & 1)) ? -1 : 1, 0, 0};
          t->host.insert(t->host.end(), v, v + 8);
          ++t->n;
        }
  }
  t->dev.upload(t->host);
  lv.segtabs[key] = t;
  return *t;
}

template <int TJ, int TK, int RW, int D, int MODE, int MINB, int XCH>
bool launch_stream(Level& lv, const Field& a, const double* a_base, const Field& b, double* b_base, const Field& r,
                   const double* r_base, const Coef& cf, const int flo[3], const int fhi[3], cudaStream_t st,
                   const Level* clv, const Field* c, const double* c_base, unsigned long long* norm,
                   const long long* push, const StreamPull* pull) {
  using LY = StreamLayout<TJ, TK, D, MODE>;
  constexpr int NW = stream_warps<TJ, TK, RW>();
  int nres = 0;
  for (int bx = 0; bx < lv.nboxes; ++bx) {
    if (!lv.resident[bx]) continue;
    ++nres;
    const BoxGeom& gg = lv.geo[bx];
    if (gg.n[1] % TJ || gg.n[2] % TK || gg.n[0] < 2) return false;
  }
  if (a.ngrow < 2 || r.ngrow < 1) return false;
  if (nres == 0) return true;
  TmaDesc da = describe(lv, a), dr = describe(lv, r);
  if (!da.ok || !dr.ok || da.slot != lv.slot || dr.slot != lv.slot) return false;
  CUtensorMap ma, mr, mc;
  std::memset(&ma, 0, sizeof ma);
  std::memset(&mr, 0, sizeof mr);
  std::memset(&mc, 0, sizeof mc);
  if (!make_map(&ma, a_base, da, nres, LY::PJ, LY::PK)) return false;
  if (!make_map(&mr, r_base, dr, nres, LY::RJ, LY::PK)) return false;
  StreamArgs args;
  std::memset(&args, 0, sizeof args);
  args.a_kc = -2 + da.g + da.f;
  args.a_jc = -2 + da.g;
  args.a_ic = da.g;
  args.r_kc = -2 + dr.g + dr.f;
  args.r_jc = -1 + dr.g;
  args.r_ic = dr.g;
  if (MODE == kModeProl) {
    if (!clv || !c || c->ngrow < 1) return false;
    TmaDesc dc = describe(*clv, *c);
    if (!dc.ok || dc.slot != da.slot) return false;
    if (!make_map(&mc, c_base, dc, nres, LY::CJ, LY::CK)) return false;
    args.c_kc = -1 + dc.g + dc.f;
    args.c_jc = -1 + dc.g;
    args.c_ic = dc.g;
  } else {
    mc = ma;
  }
  auto kern = k_gsrb_stream<TJ, TK, RW, D, MODE, MINB, XCH>;
  static int per_sm = 0;
  if (!per_sm) {
    AMRB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, LY::BYTES));
    AMRB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    AMRB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * NW, LY::BYTES));
    per_sm = std::max(per_sm, 1);
  }
  long long ncols = 0;
  for (int bx = 0; bx < lv.nboxes; ++bx)
    if (lv.resident[bx]) ncols += (long long)(lv.geo[bx].n[1] / TJ) * (lv.geo[bx].n[2] / TK);
  const long long slots = (long long)per_sm * num_sms();
  int nseg = (int)std::max<long long>(1, slots / ncols);
  if (const int64_t want = option("stream_segments")) nseg = (int)want;  // A/B runs
  const SegTable& t = seg_table(lv, TJ, TK, nseg, option("stream_alternate") != 0);
  args.seg = t.dev.p;
  args.geo = lv.dgeo.p;
  args.fb = b.dev.p;
  args.b = b_base;
  {
    int64_t hi = 0;  // one past the last element any resident box of b touches
    for (int bx = 0; bx < lv.nboxes; ++bx)
      if (lv.resident[bx]) {
        const FabView& v = b.host[bx];
        const BoxGeom& gg = lv.geo[bx];
        hi = std::max<int64_t>(hi, v.off + (int64_t)(gg.n[0] + b.ng3[0]) * v.s0 + (int64_t)(gg.n[1] + b.ng3[1]) * v.s1 +
                                       gg.n[2] + b.ng3[2] + 1);
      }
    args.b_elems = hi;
  }
  args.slot = lv.dslot.p;
  args.dcheck = AMRB_CHECKED ? debug_check_words() : nullptr;
  args.cf = cf;
  for (int x = 0; x < 3; ++x) {
    args.flo[x] = flo[x];
    args.fhi[x] = fhi[x];
  }
  args.norm = norm;
  args.push = push;
  args.push_fence = (int)option("push_fence");
  if (XCH == 2) {
    args.pull = pull->tab;
    args.a = const_cast<double*>(a_base);
    args.fa = a.dev.p;
    for (int x = 0; x < pull->nranks; ++x) args.pads[x] = pull->pads[x];
    args.epoch = pull->epoch;
    args.rank = pull->rank;
    args.nranks = pull->nranks;
    args.fault = pull->nranks > 1 ? current_fault() : Fault{};
  }
  launch_k(kern, (unsigned)t.n, 32 * NW, LY::BYTES, st, ma, mr, mc, args);
  check_launch("k_gsrb_stream");
  return true;
}


template <int TJ, int TK, int RW, int D>
bool launch_rr_stream(Level& lv, const Field& phi, const double* phi_base, const Field& rhs, const double* rhs_base,
                      const Field& crse, double* crse_base, const Coef& cf, cudaStream_t st) {
  using LY = StreamLayout<TJ, TK, D, kModePlain>;
  constexpr int NW = TJ / (RW * LY::RPW) * LY::WK;
  int nres = 0;
  for (int bx = 0; bx < lv.nboxes; ++bx) {
    if (!lv.resident[bx]) continue;
    ++nres;
    const BoxGeom& gg = lv.geo[bx];
    if (gg.n[1] % TJ || gg.n[2] % TK || gg.n[0] % 2 || gg.lo[0] % 2 || gg.lo[1] % 2 || gg.lo[2] % 2) return false;
  }
  if (phi.ngrow < 2 || rhs.ngrow < 1) return false;
  if (nres == 0) return true;
  TmaDesc da = describe(lv, phi), dr = describe(lv, rhs);
  if (!da.ok || !dr.ok || da.slot != lv.slot || dr.slot != lv.slot) return false;
  CUtensorMap ma, mr;
  std::memset(&ma, 0, sizeof ma);
  std::memset(&mr, 0, sizeof mr);
  if (!make_map(&ma, phi_base, da, nres, LY::PJ, LY::PK)) return false;
  if (!make_map(&mr, rhs_base, dr, nres, LY::RJ, LY::PK)) return false;
  RRArgs args;
  std::memset(&args, 0, sizeof args);
  args.a_kc = -2 + da.g + da.f;
  args.a_jc = -2 + da.g;
  args.a_ic = da.g;
  args.r_kc = -2 + dr.g + dr.f;
  args.r_jc = -1 + dr.g;
  args.r_ic = dr.g;
  auto kern = k_resid_restrict_stream<TJ, TK, RW, D>;
  static int per_sm = 0;
  if (!per_sm) {
    AMRB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, LY::BYTES));
    AMRB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    AMRB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * NW, LY::BYTES));
    per_sm = std::max(per_sm, 1);
  }
  long long ncols = 0;
  for (int bx = 0; bx < lv.nboxes; ++bx)
    if (lv.resident[bx]) ncols += (long long)(lv.geo[bx].n[1] / TJ) * (lv.geo[bx].n[2] / TK);
  const int nseg = (int)std::max<long long>(1, (long long)per_sm * num_sms() / ncols);
  const SegTable& t = seg_table(lv, TJ, TK, nseg, option("stream_alternate") != 0, true);
  args.seg = t.dev.p;
  args.geo = lv.dgeo.p;
  args.fc = crse.dev.p;
  args.crse = crse_base;
  args.slot = lv.dslot.p;
  args.cf = cf;
  launch_k(kern, (unsigned)t.n, 32 * NW, LY::BYTES, st, ma, mr, args);
  check_launch("k_resid_restrict_stream");
  return true;
}

}  // namespace

// crse (on the box-local coarsening of phi's level) = average_down(rhs - L(phi));
// false (nothing launched) where the layout does not take the streaming kernel
bool launch_resid_restrict_stream(Level& lv, const Field& phi, const double* phi_base, const Field& rhs,
                                  const double* rhs_base, const Field& crse, double* crse_base, const Coef& cf,
                                  cudaStream_t st) {
  return launch_rr_stream<16, 64, 4, 2>(lv, phi, phi_base, rhs, rhs_base, crse, crse_base, cf, st) ||
         launch_rr_stream<16, 32, 4, 2>(lv, phi, phi_base, rhs, rhs_base, crse, crse_base, cf, st);
}

namespace {
}  // namespace

unsigned int* debug_check_words() {
  static unsigned int* words = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    AMRB_CUDA(cudaMalloc(&words, 2 * sizeof(unsigned int)));
    AMRB_CUDA(cudaMemset(words, 0, 2 * sizeof(unsigned int)));
  });
  return words;
}

// mode 0: plain, 1: PROL (clv/c/c_base), 2: NORM (norm)
template <int TJ, int TK, int RW, int D, int M, int B>
bool dispatch_stream(Level& lv, const Field& a, const double* a_base, const Field& b, double* b_base, const Field& r,
                     const double* r_base, const Coef& cf, const int flo[3], const int fhi[3], cudaStream_t st,
                     const Level* clv, const Field* c, const double* c_base, unsigned long long* norm,
                     const long long* push, const StreamPull* pull) {
  if (push)
    return launch_stream<TJ, TK, RW, D, M, B, 1>(lv, a, a_base, b, b_base, r, r_base, cf, flo, fhi, st, clv, c, c_base,
                                                 norm, push, pull);
  if (pull) {
    if constexpr (M == kModeProl) {
      return false;  // the up-leg input's ghosts come from the restriction's fill
    } else {
      return launch_stream<TJ, TK, RW, D, M, B, 2>(lv, a, a_base, b, b_base, r, r_base, cf, flo, fhi, st, clv, c,
                                                   c_base, norm, push, pull);
    }
  }
  return launch_stream<TJ, TK, RW, D, M, B, 0>(lv, a, a_base, b, b_base, r, r_base, cf, flo, fhi, st, clv, c, c_base,
                                               norm, push, pull);
}

bool launch_sweep_stream(int mode, Level& lv, const Field& a, const double* a_base, const Field& b, double* b_base,
                         const Field& r, const double* r_base, const Coef& cf, const int flo[3], const int fhi[3],
                         cudaStream_t st, const Level* clv, const Field* c, const double* c_base,
                         unsigned long long* norm, const long long* push, const StreamPull* pull) {
#define AMRB_STREAM(TJ, TK, RW, D, M, B)                                                                            \
  dispatch_stream<TJ, TK, RW, D, M, B>(lv, a, a_base, b, b_base, r, r_base, cf, flo, fhi, st, clv, c, c_base, norm, \
                                       push, pull)
  // variants (library option "stream_config" forces one; measured on the C3 fine
  // level, tools/mb_stream.py): 1 = 16x64 tiles, 4-row strips (the fastest plain
  // sweep); 2 = 16x64, 2-row strips (two CTAs/SM even with the ghost push);
  // 4 = 16x128, 4-row (the fastest fused prolongation); 6 = 16x32 (two rows
  // per warp, 32-wide boxes)
#define AMRB_STREAM_CFG(M, CFG)                  \
  switch (CFG) {                                 \
    case 1:                                      \
      return AMRB_STREAM(16, 64, 4, 2, M, 1);    \
    case 2:                                      \
      return AMRB_STREAM(16, 64, 2, 2, M, 2);    \
    case 4:                                      \
      return AMRB_STREAM(16, 128, 4, 2, M, 1);   \
    case 6:                                      \
      return AMRB_STREAM(16, 32, 4, 2, M, 4);    \
  }                                              \
  return false;
  auto run = [&](int cfg) -> bool {
    switch (mode) {
      case kModePlain:
        AMRB_STREAM_CFG(kModePlain, cfg)
      case kModeProl:
        AMRB_STREAM_CFG(kModeProl, cfg)
      case kModeNorm:
        AMRB_STREAM_CFG(kModeNorm, cfg)
    }
    return false;
  };
  if (const int64_t forced = option("stream_config")) return run((int)forced);
  // defaults per mode (with / without ghost push), then narrower tiles when a
  // box does not divide
  static const int prefs[2][3][4] = {{{1, 2, 6, 0}, {4, 1, 6, 0}, {2, 1, 6, 0}},
                                     {{2, 1, 6, 0}, {4, 2, 6, 0}, {2, 1, 6, 0}}};
  for (int cfg : prefs[push ? 1 : 0][mode])
    if (cfg && run(cfg)) return true;
  return false;
#undef AMRB_STREAM_CFG

#undef AMRB_STREAM
  return false;
}

}  // namespace amrb

extern "C" int amrb_debug_checks(int64_t* failures, int64_t* line, int reset) {
  return amrb::guarded([&] {
    if (!failures || !line) throw amrb::Error(AMRB_EINVAL, "amrb_debug_checks: null argument");
    unsigned int w[2] = {0, 0};
    if (AMRB_CHECKED) AMRB_CUDA(cudaMemcpy(w, amrb::debug_check_words(), sizeof w, cudaMemcpyDeviceToHost));
    *failures = AMRB_CHECKED ? (int64_t)w[0] : -1;
    *line = (int64_t)w[1];
    if (AMRB_CHECKED && reset) AMRB_CUDA(cudaMemset(amrb::debug_check_words(), 0, sizeof w));
  });
}
