// Box-loop kernels of the MLMG hot path (sm_100a, fp64, HBM-bound).
//
// The reference runs these as Python loops over boxes with numpy slicing
// (advect.py:143-178 is its ParallelFor pattern; average_down coarse_fine.py:
// 136-163; interp_to_fine "pc" :166-185; reduce fabarray.py:409-440).  The
// Laplacian / GSRB / residual have no reference code; their definitions are
// the oracle's (oracle/mlmg_ref.py) and every kernel reproduces its operand
// order exactly (the library is compiled with --fmad=false), so results are
// bit-identical, not merely within tolerance.
//
// Work decomposition: a level's valid region is cut into tiles
// (box, i0, j0, k0); one CTA per tile; threadIdx.x runs along k (unit
// stride), threadIdx.y along j, and each thread marches along i.
#include <atomic>
#include <cfloat>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>

#include "stencil_common.cuh"

namespace amrb {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

namespace {
std::atomic<long long> g_launches{0};
}
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
// Library options (amrb_set_option): explicit, process-wide, no environment.
namespace {
std::mutex g_opt_mu;
std::map<std::string, int64_t>& options() {
  static std::map<std::string, int64_t> o = {{"pdl", 2}, {"sweep_kernel", 0}, {"grid_per_sm", 0}, {"stream_segments", 0}, {"stream_alternate", 1},
                                               {"stream_config", 0}, {"push_fence", 0},
                                               {"peer_timeout_ms", 30000}};
  return o;
}
}  // namespace
int64_t option(const char* name) {
  std::lock_guard<std::mutex> lk(g_opt_mu);
  auto it = options().find(name);
  return it == options().end() ? 0 : it->second;
}
int pdl_mode() { return (int)option("pdl"); }

const TileTable& Level::tiles(int ti, int tj, int tk) {
  auto key = std::make_tuple(ti, tj, tk);
  auto it = tables.find(key);
  if (it != tables.end()) return *it->second;
  auto* t = new TileTable;
  t->ti = ti;
  t->tj = tj;
  t->tk = tk;
  for (int b = 0; b < nboxes; ++b) {
    if (!resident[b]) continue;
    const BoxGeom& g = geo[b];
    for (int i = 0; i < g.n[0]; i += ti)
      for (int j = 0; j < g.n[1]; j += tj)
        for (int k = 0; k < g.n[2]; k += tk) t->host.push_back(make_int4(b, i, j, k));
  }
  t->dev.upload(t->host);
  tables[key] = t;
  return *t;
}

const TileTable& Level::columns(int tj, int tk) {
  auto key = std::make_tuple(-1, tj, tk);
  auto it = tables.find(key);
  if (it != tables.end()) return *it->second;
  auto* t = new TileTable;
  t->ti = -1;
  t->tj = tj;
  t->tk = tk;
  long long acc = 0;
  for (int b = 0; b < nboxes; ++b) {
    if (!resident[b]) continue;
    const BoxGeom& g = geo[b];
    for (int j = 0; j < g.n[1]; j += tj)
      for (int k = 0; k < g.n[2]; k += tk) {
        t->host.push_back(make_int4(b, j, k, (int)acc));
        acc += g.n[0];
      }
  }
  t->total = acc;
  t->dev.upload(t->host);
  tables[key] = t;
  return *t;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    AMRB_CUDA(cudaGetDevice(&dev));
    AMRB_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

bool Level::all_even() const {
  for (int b = 0; b < nboxes; ++b)
    for (int x = 0; x < 3; ++x)
      if (geo[b].n[x] % 2) return false;
  return true;
}

namespace {

template <class T>
__device__ __forceinline__ T ldg(const T* p) {
  return __ldg(p);
}

// ---------------------------------------------------------------------------
// Simple tiles: TI x 8 x 32, block (32, 8); thread = one k, one j, march i.
// ---------------------------------------------------------------------------
constexpr int kTI = 8, kTJ = 8, kTK = 32;

enum class Op { kLap, kResid };

template <Op op>
__global__ void __launch_bounds__(256)
    k_stencil(const int4* __restrict__ tiles, int ti, const BoxGeom* __restrict__ geo, const FabView* __restrict__ fo,
              double* __restrict__ out, const FabView* __restrict__ fr, const double* __restrict__ rhs,
              const FabView* __restrict__ fp, const double* __restrict__ phi, Coef cf) {
  pdl_entry();
  const int4 t = tiles[blockIdx.x];
  const BoxGeom g = geo[t.x];
  const int j = t.z + threadIdx.y, k = t.w + threadIdx.x;
  if (j >= g.n[1] || k >= g.n[2]) return;
  const FabView P = fp[t.x], O = fo[t.x];
  const double* p = phi + P.off + (int64_t)j * P.s1 + k;
  double* o = out + O.off + (int64_t)j * O.s1 + k;
  const double* r = nullptr;
  int64_t rs0 = 0;
  if (op == Op::kResid) {
    const FabView R = fr[t.x];
    r = rhs + R.off + (int64_t)j * R.s1 + k;
    rs0 = R.s0;
  }
  const int iend = min(t.y + ti, g.n[0]);
  int i = t.y;
  double xm = ldg(p + (int64_t)(i - 1) * P.s0);
  double c = ldg(p + (int64_t)i * P.s0);
  for (; i < iend; ++i) {
    const double* pc = p + (int64_t)i * P.s0;
    const double xp = ldg(pc + P.s0);
    const double lap = lap7(c, xm, xp, ldg(pc - P.s1), ldg(pc + P.s1), ldg(pc - 1), ldg(pc + 1), cf);
    double v = lap;
    if (op == Op::kResid) v = ldg(r + (int64_t)i * rs0) - lap;
    o[(int64_t)i * O.s0] = v;
    xm = c;
    c = xp;
  }
}

// ---------------------------------------------------------------------------
// One GSRB colour, in place.  Tile TI x 8 x 64; thread = a k-pair (exactly one
// cell of the pair has the colour), so no lane idles on parity.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
    k_gsrb_color(const int4* __restrict__ tiles, int ti, const BoxGeom* __restrict__ geo, const FabView* __restrict__ fp,
                 double* __restrict__ phi, const FabView* __restrict__ fr, const double* __restrict__ rhs,
                 Coef cf, int color) {
  pdl_entry();
  const int4 t = tiles[blockIdx.x];
  const BoxGeom g = geo[t.x];
  const int j = t.z + threadIdx.y;
  const int kp = t.w + 2 * threadIdx.x;
  if (j >= g.n[1] || kp >= g.n[2]) return;
  const FabView P = fp[t.x], R = fr[t.x];
  const int iend = min(t.y + ti, g.n[0]);
  for (int i = t.y; i < iend; ++i) {
    // global parity of (i, j, kp): pick the member of the pair with the colour
    const int par = (g.lo[0] + i + g.lo[1] + j + g.lo[2] + kp + color) & 1;
    const int k = kp + par;
    if (k >= g.n[2]) continue;
    double* pc = phi + P.off + (int64_t)i * P.s0 + (int64_t)j * P.s1 + k;
    const double c = *pc;
    const double lap = lap7(c, pc[-P.s0], pc[P.s0], pc[-P.s1], pc[P.s1], pc[-1], pc[1], cf);
    const double b = rhs[R.off + (int64_t)i * R.s0 + (int64_t)j * R.s1 + k];
    *pc = relax(c, b, lap, cf.rgamma);
  }
}

// ---------------------------------------------------------------------------
// Fused red+black sweep, out of place (A -> B), marching along i.
//
// A CTA owns a TJ x TK column of one box over i in [i0, i0 + CI).  It keeps
// four planes of A (grown by 2 in j and k) and two planes of rhs (grown by 1)
// in shared memory.  At step p it relaxes the red cells of plane p+1 over the
// tile grown by one ring (reading only black, i.e. old, values), then the
// black cells of plane p over the tile (reading the new red values), then
// streams plane p to B and prefetches plane p+3 / rhs p+2 with cp.async.
// Because A is never written, neighbouring tiles and boxes read consistent
// old values; the red update of ring cells is recomputed from the same
// operands as its owner computes it, hence bit-identical to "fill; red; fill;
// black" with a width-1 fill in between.  Cells outside the domain in a
// non-periodic direction are never relaxed (they hold boundary values).
// ---------------------------------------------------------------------------
struct SweepArgs {
  const int4* tiles;
  const BoxGeom* geo;
  const FabView* fa;  // phi in (ngrow >= 2)
  const FabView* fb;  // phi out
  const FabView* fr;  // rhs (ngrow >= 1)
  const double* a;
  double* b;
  const double* rhs;
  Coef cf;
  int ci;
  int fixed_lo[3], fixed_hi[3];  // cells outside [lo, hi] (global) are not relaxed
};

template <int TJ, int TK>
struct SweepSmem {
  static constexpr int PJ = TJ + 4, PK = TK + 4;  // phi plane (grown by 2)
  static constexpr int RJ = TJ + 2;               // rhs plane rows (grown by 1), PK cols
  double phi[4][PJ][PK];
  double rhs[2][RJ][PK];
};

template <int TJ, int TK>
__device__ __forceinline__ void load_phi_plane(SweepSmem<TJ, TK>& sm, int slot, const double* a,
                                               const FabView& A, int i, int j0, int jn, int k0, int kn) {
  // rows j0-2 .. j0+jn+1, 16-byte chunks covering k0-2 .. k0+kn+1
  const int rows = jn + 4, chunks = (kn + 4 + 1) / 2;
  const double* base = a + A.off + (int64_t)i * A.s0 + (int64_t)(j0 - 2) * A.s1 + (k0 - 2);
  for (int e = threadIdx.x + threadIdx.y * blockDim.x; e < rows * chunks; e += blockDim.x * blockDim.y) {
    const int r = e / chunks, q = e - r * chunks;
    cp_async16(&sm.phi[slot][r][2 * q], base + (int64_t)r * A.s1 + 2 * q);
  }
}

template <int TJ, int TK>
__device__ __forceinline__ void load_rhs_plane(SweepSmem<TJ, TK>& sm, int slot, const double* rhs,
                                               const FabView& R, int i, int j0, int jn, int k0, int kn) {
  const int rows = jn + 2, chunks = (kn + 4 + 1) / 2;
  const double* base = rhs + R.off + (int64_t)i * R.s0 + (int64_t)(j0 - 1) * R.s1 + (k0 - 2);
  for (int e = threadIdx.x + threadIdx.y * blockDim.x; e < rows * chunks; e += blockDim.x * blockDim.y) {
    const int r = e / chunks, q = e - r * chunks;
    cp_async16(&sm.rhs[slot][r][2 * q], base + (int64_t)r * R.s1 + 2 * q);
  }
}

template <int TJ, int TK>
__global__ void __launch_bounds__(256, 2) k_gsrb_sweep(SweepArgs args) {
  pdl_entry();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<SweepSmem<TJ, TK>*>(smem_raw);
  const int4 t = args.tiles[blockIdx.x];
  const BoxGeom g = args.geo[t.x];
  const FabView A = args.fa[t.x], B = args.fb[t.x], R = args.fr[t.x];
  const Coef cf = args.cf;
  const int i0 = t.y, j0 = t.z, k0 = t.w;
  const int i1 = min(i0 + args.ci, g.n[0]);
  const int jn = min(TJ, g.n[1] - j0), kn = min(TK, g.n[2] - k0);
  const int nthreads = blockDim.x * blockDim.y;
  const int tid = threadIdx.x + threadIdx.y * blockDim.x;

  auto slot = [&](int plane) { return (plane - i0 + 8) & 3; };
  auto rslot = [&](int plane) { return (plane - i0 + 8) & 1; };

  // red relaxation of plane ip over the ring-grown tile
  auto red = [&](int ip) {
    const int s = slot(ip), sm1 = slot(ip - 1), sp1 = slot(ip + 1), rs = rslot(ip);
    const int gi = g.lo[0] + ip;
    const bool ifix = gi < args.fixed_lo[0] || gi > args.fixed_hi[0];
    const int rows = jn + 2, pairs = (kn + 2) / 2;
    for (int e = tid; e < rows * pairs; e += nthreads) {
      const int rr = e / pairs, q = e - rr * pairs;
      const int j = j0 - 1 + rr;
      const int kb = k0 - 1 + 2 * q;
      const int par = (gi + g.lo[1] + j + g.lo[2] + kb) & 1;  // red: even
      const int k = kb + par;
      const int gj = g.lo[1] + j, gk = g.lo[2] + k;
      if (ifix || gj < args.fixed_lo[1] || gj > args.fixed_hi[1] || gk < args.fixed_lo[2] ||
          gk > args.fixed_hi[2])
        continue;
      const int r = rr + 1, c = k - k0 + 2;
      const double v = sm.phi[s][r][c];
      const double lap = lap7(v, sm.phi[sm1][r][c], sm.phi[sp1][r][c], sm.phi[s][r - 1][c],
                              sm.phi[s][r + 1][c], sm.phi[s][r][c - 1], sm.phi[s][r][c + 1], cf);
      sm.phi[s][r][c] = relax(v, sm.rhs[rs][rr][c], lap, cf.rgamma);
    }
  };
  auto black = [&](int ip) {
    const int s = slot(ip), sm1 = slot(ip - 1), sp1 = slot(ip + 1), rs = rslot(ip);
    const int gi = g.lo[0] + ip;
    const bool ifix = gi < args.fixed_lo[0] || gi > args.fixed_hi[0];
    const int pairs = kn / 2;
    for (int e = tid; e < jn * pairs; e += nthreads) {
      const int jj = e / pairs, q = e - jj * pairs;
      const int j = j0 + jj;
      const int kb = k0 + 2 * q;
      const int par = (gi + g.lo[1] + j + g.lo[2] + kb + 1) & 1;  // black: odd
      const int k = kb + par;
      const int gj = g.lo[1] + j, gk = g.lo[2] + k;
      if (ifix || gj < args.fixed_lo[1] || gj > args.fixed_hi[1] || gk < args.fixed_lo[2] ||
          gk > args.fixed_hi[2])
        continue;
      const int r = jj + 2, c = k - k0 + 2;
      const double v = sm.phi[s][r][c];
      const double lap = lap7(v, sm.phi[sm1][r][c], sm.phi[sp1][r][c], sm.phi[s][r - 1][c],
                              sm.phi[s][r + 1][c], sm.phi[s][r][c - 1], sm.phi[s][r][c + 1], cf);
      sm.phi[s][r][c] = relax(v, sm.rhs[rs][jj + 1][c], lap, cf.rgamma);
    }
  };
  auto store = [&](int ip) {
    const int s = slot(ip);
    const int pairs = kn / 2;
    double* base = args.b + B.off + (int64_t)ip * B.s0 + (int64_t)j0 * B.s1 + k0;
    for (int e = tid; e < jn * pairs; e += nthreads) {
      const int jj = e / pairs, q = e - jj * pairs;
      const double2 v = make_double2(sm.phi[s][jj + 2][2 * q + 2], sm.phi[s][jj + 2][2 * q + 3]);
      *reinterpret_cast<double2*>(base + (int64_t)jj * B.s1 + 2 * q) = v;
    }
  };

  // prologue: planes i0-2 .. i0+1 of phi, i0-1 .. i0 of rhs
  for (int ip = i0 - 2; ip <= i0 + 1; ++ip) load_phi_plane(sm, slot(ip), args.a, A, ip, j0, jn, k0, kn);
  for (int ip = i0 - 1; ip <= i0; ++ip) load_rhs_plane(sm, rslot(ip), args.rhs, R, ip, j0, jn, k0, kn);
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  // red of planes i0-1 and i0 (independent: red reads only black cells)
  red(i0 - 1);
  red(i0);
  __syncthreads();
  load_phi_plane(sm, slot(i0 + 2), args.a, A, i0 + 2, j0, jn, k0, kn);
  load_rhs_plane(sm, rslot(i0 + 1), args.rhs, R, i0 + 1, j0, jn, k0, kn);
  cp_async_commit();
  for (int p = i0; p < i1; ++p) {
    cp_async_wait_all();
    __syncthreads();
    red(p + 1);
    __syncthreads();
    black(p);
    __syncthreads();
    // plane p is final; slot of p-1 and rhs slot of p are free
    if (p + 3 <= i1 + 1) load_phi_plane(sm, slot(p + 3), args.a, A, p + 3, j0, jn, k0, kn);
    if (p + 2 <= i1) load_rhs_plane(sm, rslot(p + 2), args.rhs, R, p + 2, j0, jn, k0, kn);
    cp_async_commit();
    store(p);
  }
  cp_async_wait_all();
}

// ---------------------------------------------------------------------------
// Fused sweep, full-tile fast path (every box a multiple of TJ x TK in j, k).
//
// Persistent and balanced: the level's (box, j0, k0) columns are laid end to
// end as one sequence of plane-steps; CTA b of G marches the contiguous range
// [T*b/G, T*(b+1)/G), restarting its pipeline only where it crosses into the
// next column.  Per step p:
//   wait(phi p+2, rhs p+1); barrier; prefetch phi(p+4), rhs(p+3) (cp.async);
//   red(p+1) over the ring-grown tile; barrier; black(p) + stream plane p out.
// Shared planes are stored parity-split: cell (r, c) lives at [r][c & 1][c >> 1],
// so the red (or black) cells of a row and their k-neighbours are unit-stride
// across lanes (no bank conflicts).  phi slots rotate mod 6, rhs mod 4:
// phi(p+4) overwrites phi(p-2) and rhs(p+3) overwrites rhs(p-1), whose last
// readers (black(p-1)) finish before the barrier that opens step p.
// ---------------------------------------------------------------------------
template <int TJ, int TK>
struct Sweep3Smem {
  static constexpr int PJ = TJ + 4, RJ = TJ + 2, H = TK / 2 + 2;  // H: cells per parity half-row
  double phi[6][PJ][2][H];
  double rhs[4][RJ][2][H];
};

struct Sweep3Args {
  const int4* cols;  // (box, j0, k0, first plane-step of the column)
  int ncols;
  long long total;  // plane-steps over all columns
  const BoxGeom* geo;
  const FabView* fa;
  const FabView* fb;
  const FabView* fr;
  const double* a;
  double* b;
  const double* rhs;
  Coef cf;
  int fixed_lo[3], fixed_hi[3];
};

template <int TJ, int TK, bool FIXED>
__global__ void __launch_bounds__(256, 2) k_gsrb_sweep3(Sweep3Args args) {
  pdl_entry();
  using SM = Sweep3Smem<TJ, TK>;
  constexpr int NT = 256;
  constexpr int PK = TK + 4;        // cells per smem row (k0-2 .. k0+TK+1)
  constexpr int H = SM::H;          // cells per parity half-row
  constexpr int ROW = 2 * H;        // doubles per smem row
  constexpr int PSLOT = SM::PJ * ROW;
  constexpr int RSLOT = SM::RJ * ROW;
  constexpr int LPR = TK / 2;       // lanes per row (one k-pair each)
  constexpr int RPP = NT / LPR;     // rows per pass
  constexpr int NCP = (PK + 31) / 32;  // copies per lane per row
  static_assert(NT % LPR == 0, "tile width");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);
  double* const phi_s = &sm.phi[0][0][0][0];
  double* const rhs_s = &sm.rhs[0][0][0][0];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int q = tid % LPR;          // pair index inside a row
  const int rsub = tid / LPR;       // row inside a pass
  const Coef cf = args.cf;
  // per-lane split-parity smem offsets of the row elements this lane copies
  int soff[NCP];
#pragma unroll
  for (int u = 0; u < NCP; ++u) {
    const int c = lane + 32 * u;
    soff[u] = (c & 1) * H + (c >> 1);
  }

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
  while (s < e) {
    const int4 cd = args.cols[col];
    const BoxGeom g = args.geo[cd.x];
    const FabView A = args.fa[cd.x], B = args.fb[cd.x], R = args.fr[cd.x];
    const int j0 = cd.y, k0 = cd.z;
    const int i0 = (int)(s - cd.w);
    const int i1 = (int)min((long long)g.n[0], e - cd.w);
    s += i1 - i0;
    ++col;
    const int jk0 = g.lo[1] + j0 + g.lo[2] + k0;
    const double* abase = args.a + A.off + (int64_t)(j0 - 2) * A.s1 + (k0 - 2);
    const double* rbase = args.rhs + R.off + (int64_t)(j0 - 1) * R.s1 + (k0 - 2);
    double* obase = args.b + B.off + (int64_t)j0 * B.s1 + k0 + 2 * q;

    auto phi_slot = [&](int ip) { return phi_s + ((ip + 12) % 6) * PSLOT; };
    auto rhs_slot = [&](int ip) { return rhs_s + ((ip + 12) & 3) * RSLOT; };
    auto load_rows = [&](double* dst, const double* src, int64_t s1, int nrows) {
      for (int r = warp; r < nrows; r += NT / 32) {
        const double* gs = src + (int64_t)r * s1 + lane;
        double* sd = dst + r * ROW;
#pragma unroll
        for (int u = 0; u < NCP; ++u)
          if (lane + 32 * u < PK) cp_async8(sd + soff[u], gs + 32 * u);
      }
    };
    auto load_phi = [&](int ip) { load_rows(phi_slot(ip), abase + (int64_t)ip * A.s0, A.s1, SM::PJ); };
    auto load_rhs = [&](int ip) { load_rows(rhs_slot(ip), rbase + (int64_t)ip * R.s0, R.s1, SM::RJ); };
    auto is_fixed = [&](int gi, int r, int c) {
      const int gj = g.lo[1] + j0 - 2 + r, gk = g.lo[2] + k0 - 2 + c;
      return gi < args.fixed_lo[0] || gi > args.fixed_hi[0] || gj < args.fixed_lo[1] || gj > args.fixed_hi[1] ||
             gk < args.fixed_lo[2] || gk > args.fixed_hi[2];
    };
    // relax the cell at smem offset o (its half known through kl: the offset of
    // its k-1 neighbour; k+1 is kl + 1).  rhs row = phi row - 1.
    auto relax_at = [&](const double* P, const double* Pm, const double* Pp, const double* Rh, int o, int kl) {
      const double v = P[o];
      const double lap = lap7(v, Pm[o], Pp[o], P[o - ROW], P[o + ROW], P[kl], P[kl + 1], cf);
      return relax(v, Rh[o - ROW], lap, cf.rgamma);
    };
    auto red = [&](int ip) {
      double* P = phi_slot(ip);
      const double* Pm = phi_slot(ip - 1);
      const double* Pp = phi_slot(ip + 1);
      const double* Rh = rhs_slot(ip);
      const int gi = g.lo[0] + ip;
      const int bp = (gi + jk0) & 1;  // parity of smem cell (r, c) = (bp + r + c) & 1
      // interior pairs: cols 2q+2, 2q+3 (half x = q+1); red member off = (bp + r) & 1
#pragma unroll
      for (int m = 0; m < (TJ + 2 + RPP - 1) / RPP; ++m) {
        const int r = 1 + rsub + m * RPP;  // ring rows 1 .. TJ+2
        if ((TJ + 2) % RPP != 0 && r > TJ + 2) break;
        const int off = (bp + r) & 1;
        if (FIXED && is_fixed(gi, r, 2 * q + 2 + off)) continue;
        const int o = r * ROW + off * H + q + 1;
        const int kl = off ? o - H : o + H - 1;
        P[o] = relax_at(P, Pm, Pp, Rh, o, kl);
      }
      // ring columns c = 1 (k0-1) and c = TK+2 (k0+TK)
      if (tid < 2 * (TJ + 2)) {
        const int r = 1 + (tid >> 1);
        const int c = (tid & 1) ? TK + 2 : 1;
        if (((bp + r + c) & 1) == 0 && !(FIXED && is_fixed(gi, r, c))) {
          const int o = r * ROW + (c & 1) * H + (c >> 1);
          const int kl = r * ROW + ((c - 1) & 1) * H + ((c - 1) >> 1);
          P[o] = relax_at(P, Pm, Pp, Rh, o, kl);
        }
      }
    };
    auto black_store = [&](int ip) {
      const double* P = phi_slot(ip);
      const double* Pm = phi_slot(ip - 1);
      const double* Pp = phi_slot(ip + 1);
      const double* Rh = rhs_slot(ip);
      const int gi = g.lo[0] + ip;
      const int bp = (gi + jk0) & 1;
      double* out = obase + (int64_t)ip * B.s0;
#pragma unroll
      for (int m = 0; m < (TJ + RPP - 1) / RPP; ++m) {
        const int r = 2 + rsub + m * RPP;  // rows 2 .. TJ+1
        if (TJ % RPP != 0 && r > TJ + 1) break;
        const int off = ((bp + r) & 1) ^ 1;  // black member of the pair
        const int o = r * ROW + off * H + q + 1;
        const int kl = off ? o - H : o + H - 1;
        double bv = P[o];
        if (!(FIXED && is_fixed(gi, r, 2 * q + 2 + off))) bv = relax_at(P, Pm, Pp, Rh, o, kl);
        const double rv = off ? P[o - H] : P[o + H];
        const double2 w = off ? make_double2(rv, bv) : make_double2(bv, rv);
        *reinterpret_cast<double2*>(out + (int64_t)(r - 2) * B.s1) = w;
      }
    };

    // prologue for this column segment
    __syncthreads();  // previous segment's smem readers are done
    for (int ip = i0 - 2; ip <= i0 + 2; ++ip) load_phi(ip);
    for (int ip = i0 - 1; ip <= i0 + 1; ++ip) load_rhs(ip);
    cp_async_commit();
    if (i0 + 3 <= i1 + 1) load_phi(i0 + 3);
    if (i0 + 2 <= i1) load_rhs(i0 + 2);
    cp_async_commit();
    asm volatile("cp.async.wait_group 1;\n" ::);
    __syncthreads();
    red(i0 - 1);
    red(i0);
    for (int p = i0; p < i1; ++p) {
      asm volatile("cp.async.wait_group 1;\n" ::);
      __syncthreads();
      if (p + 4 <= i1 + 1) load_phi(p + 4);
      if (p + 3 <= i1) load_rhs(p + 3);
      cp_async_commit();
      red(p + 1);
      __syncthreads();
      black_store(p);
    }
    cp_async_wait_all();
  }
}

// ---------------------------------------------------------------------------
// Restriction (ratio 2, box-local coarsened layout) and fused residual-restrict.
// Tile over coarse boxes: 8 x 8 x 32 coarse cells.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double avg8(double c000, double c001, double c010, double c011, double c100,
                                       double c101, double c110, double c111) {
  // numpy reshape(...).mean(axis=(2,4,6)) order (verified bit-for-bit)
  return ((((c000 + c001) + (c010 + c011)) + (c100 + c101)) + (c110 + c111)) * 0.125;
}

// Generic restriction with per-axis ratio in {1, 2}.  Sum order = numpy's
// reshape-mean: pair the last-axis children, then accumulate the pairs
// sequentially in lexicographic order of the outer child offsets (verified
// bit-for-bit against numpy 2.3 in 1-D, 2-D and 3-D).  mode 1 = injection
// (child at offset 0, coarse_fine.py:150-154).
__global__ void __launch_bounds__(256)
    k_restrict(const int4* __restrict__ tiles, int ti, const BoxGeom* __restrict__ cgeo, const FabView* __restrict__ fc,
               double* __restrict__ crse, const FabView* __restrict__ ff, const double* __restrict__ fine,
               int ncomp, int3 rr, int mode, double inv) {
  pdl_entry();
  const int4 t = tiles[blockIdx.x];
  const BoxGeom g = cgeo[t.x];
  const int j = t.z + threadIdx.y, k = t.w + threadIdx.x;
  if (j >= g.n[1] || k >= g.n[2]) return;
  const FabView C = fc[t.x], F = ff[t.x];
  const int iend = min(t.y + ti, g.n[0]);
  for (int n = 0; n < ncomp; ++n)
    for (int i = t.y; i < iend; ++i) {
      const double* f0 = fine + F.off + n * F.cs + (int64_t)(rr.x * i) * F.s0 + (int64_t)(rr.y * j) * F.s1 + rr.z * k;
      double acc;
      if (mode == 1) {
        acc = f0[0];
      } else {
        acc = 0.0;
        bool first = true;
        for (int a = 0; a < rr.x; ++a)
          for (int b = 0; b < rr.y; ++b) {
            const double* f = f0 + (int64_t)a * F.s0 + (int64_t)b * F.s1;
            const double p = rr.z == 2 ? f[0] + f[1] : f[0];
            acc = first ? p : acc + p;
            first = false;
          }
        acc = acc * inv;
      }
      crse[C.off + n * C.cs + (int64_t)i * C.s0 + (int64_t)j * C.s1 + k] = acc;
    }
}

__device__ __forceinline__ double resid_at(const double* p, int64_t s0, int64_t s1, double b, const Coef& cf) {
  const double c = *p;
  return b - lap7(c, p[-s0], p[s0], p[-s1], p[s1], p[-1], p[1], cf);
}

__global__ void __launch_bounds__(256)
    k_resid_restrict(const int4* __restrict__ tiles, int ti, const BoxGeom* __restrict__ cgeo,
                     const FabView* __restrict__ fc, double* __restrict__ crse, const FabView* __restrict__ fr,
                     const double* __restrict__ rhs, const FabView* __restrict__ fp,
                     const double* __restrict__ phi, Coef cf) {
  pdl_entry();
  const int4 t = tiles[blockIdx.x];
  const BoxGeom g = cgeo[t.x];
  const int j = t.z + threadIdx.y, k = t.w + threadIdx.x;
  if (j >= g.n[1] || k >= g.n[2]) return;
  const FabView C = fc[t.x], R = fr[t.x], P = fp[t.x];
  const int iend = min(t.y + ti, g.n[0]);
  for (int i = t.y; i < iend; ++i) {
    double v[8];
#pragma unroll
    for (int di = 0; di < 2; ++di)
#pragma unroll
      for (int dj = 0; dj < 2; ++dj)
#pragma unroll
        for (int dk = 0; dk < 2; ++dk) {
          const int fi = 2 * i + di, fj = 2 * j + dj, fk = 2 * k + dk;
          const double* p = phi + P.off + (int64_t)fi * P.s0 + (int64_t)fj * P.s1 + fk;
          const double b = rhs[R.off + (int64_t)fi * R.s0 + (int64_t)fj * R.s1 + fk];
          v[di * 4 + dj * 2 + dk] = resid_at(p, P.s0, P.s1, b, cf);
        }
    crse[C.off + (int64_t)i * C.s0 + (int64_t)j * C.s1 + k] = avg8(v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7]);
  }
}

// Prolongation (pc), optionally added: fine(c) (+)= crse(c / 2).  Planes go
// four at a time with every load issued before the first store (four fine
// reads in flight per thread instead of one).
__global__ void __launch_bounds__(256)
    k_prolong(const int4* __restrict__ tiles, int ti, const BoxGeom* __restrict__ fgeo, const FabView* __restrict__ ff,
              double* __restrict__ fine, const FabView* __restrict__ fc, const double* __restrict__ crse,
              int ncomp, int add, int3 sh) {
  pdl_entry();
  const int4 t = tiles[blockIdx.x];
  const BoxGeom g = fgeo[t.x];
  const int j = t.z + threadIdx.y, k = t.w + threadIdx.x;
  if (j >= g.n[1] || k >= g.n[2]) return;
  const FabView F = ff[t.x], C = fc[t.x];
  const int iend = min(t.y + ti, g.n[0]);
  // coarse local index: floor((lo + x)/2) - floor(lo/2); lo is even on coarsenable layouts
  for (int n = 0; n < ncomp; ++n) {
    const double* cb = crse + C.off + n * C.cs + (int64_t)(j >> sh.y) * C.s1 + (k >> sh.z);
    double* fb = fine + F.off + n * F.cs + (int64_t)j * F.s1 + k;
    int i = t.y;
    for (; i + 4 <= iend; i += 4) {
      double c[4], f[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        c[u] = ldg(cb + (int64_t)((i + u) >> sh.x) * C.s0);
        f[u] = add ? fb[(int64_t)(i + u) * F.s0] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) fb[(int64_t)(i + u) * F.s0] = add ? f[u] + c[u] : c[u];
    }
    for (; i < iend; ++i) {
      const double c = ldg(cb + (int64_t)(i >> sh.x) * C.s0);
      double* f = fb + (int64_t)i * F.s0;
      *f = add ? *f + c : c;
    }
  }
}


// ---------------------------------------------------------------------------
// Reductions: per-tile partial (fixed tree), then one ordered final pass.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double combine(int kind, double a, double b) {
  switch (kind) {
    case 0:
      return a + b;
    case 1:
      return fmin(a, b);
    default:
      return fmax(a, b);
  }
}

__device__ __forceinline__ double identity(int kind) {
  return kind == 0 ? 0.0 : kind == 1 ? DBL_MAX * 2.0 : -DBL_MAX * 2.0;
}

__device__ double block_combine(int kind, double v, double* scratch) {
  for (int o = 16; o > 0; o >>= 1) v = combine(kind, v, __shfl_down_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, warp = (threadIdx.x + threadIdx.y * blockDim.x) >> 5;
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  const int nw = (blockDim.x * blockDim.y) >> 5;
  if (warp == 0) {
    v = lane < nw ? scratch[lane] : identity(kind);
    for (int o = 16; o > 0; o >>= 1) v = combine(kind, v, __shfl_down_sync(0xffffffffu, v, o));
  }
  return v;
}

__global__ void __launch_bounds__(256)
    k_reduce_tiles(const int4* __restrict__ tiles, int ti, const BoxGeom* __restrict__ geo, const FabView* __restrict__ fx,
                   const double* __restrict__ x, int comp, int kind, double* __restrict__ partial) {
  pdl_entry();
  __shared__ double scratch[32];
  const int4 t = tiles[blockIdx.x];
  const BoxGeom g = geo[t.x];
  const int j = t.z + threadIdx.y, k = t.w + threadIdx.x;
  const int rkind = kind == 3 ? 2 : kind;
  double acc = identity(rkind);
  if (j < g.n[1] && k < g.n[2]) {
    const FabView X = fx[t.x];
    const int iend = min(t.y + ti, g.n[0]);
    for (int i = t.y; i < iend; ++i) {
      double v = x[X.off + comp * X.cs + (int64_t)i * X.s0 + (int64_t)j * X.s1 + k];
      if (kind == 3) v = fabs(v);
      acc = combine(rkind, acc, v);
    }
  }
  acc = block_combine(rkind, acc, scratch);
  if (threadIdx.x == 0 && threadIdx.y == 0) partial[blockIdx.x] = acc;
}

// Residual inf-norm without materialising r: per-tile max |rhs - L(phi)|,
// then the ordered final pass of k_reduce_final (max is order-independent).
__global__ void __launch_bounds__(256)
    k_resid_norm(const int4* __restrict__ tiles, int ti, const BoxGeom* __restrict__ geo, const FabView* __restrict__ fr,
                 const double* __restrict__ rhs, const FabView* __restrict__ fp, const double* __restrict__ phi,
                 Coef cf, double* __restrict__ partial) {
  pdl_entry();
  __shared__ double scratch[32];
  const int4 t = tiles[blockIdx.x];
  const BoxGeom g = geo[t.x];
  const int j = t.z + threadIdx.y, k = t.w + threadIdx.x;
  double acc = 0.0;
  if (j < g.n[1] && k < g.n[2]) {
    const FabView P = fp[t.x], R = fr[t.x];
    const double* p = phi + P.off + (int64_t)j * P.s1 + k;
    const double* r = rhs + R.off + (int64_t)j * R.s1 + k;
    const int iend = min(t.y + ti, g.n[0]);
    int i = t.y;
    double xm = ldg(p + (int64_t)(i - 1) * P.s0);
    double c = ldg(p + (int64_t)i * P.s0);
    for (; i < iend; ++i) {
      const double* pc = p + (int64_t)i * P.s0;
      const double xp = ldg(pc + P.s0);
      const double lap = lap7(c, xm, xp, ldg(pc - P.s1), ldg(pc + P.s1), ldg(pc - 1), ldg(pc + 1), cf);
      acc = fmax(acc, fabs(ldg(r + (int64_t)i * R.s0) - lap));
      xm = c;
      c = xp;
    }
  }
  acc = block_combine(2, acc, scratch);
  if (threadIdx.x == 0 && threadIdx.y == 0) partial[blockIdx.x] = acc;
}

__global__ void __launch_bounds__(1024) k_reduce_final(const double* __restrict__ partial, int n, int kind,
                                                       double* __restrict__ out) {
  pdl_entry();
  __shared__ double scratch[32];
  const int rkind = kind == 3 ? 2 : kind;
  double acc = identity(rkind);
  for (int e = threadIdx.x; e < n; e += blockDim.x) acc = combine(rkind, acc, partial[e]);
  acc = block_combine(rkind, acc, scratch);
  if (threadIdx.x == 0) *out = acc;
}

// ---------------------------------------------------------------------------
// Physical-domain ghost cells (apply_domain_boundary, amr_core.py:111-146):
// one launch per (axis, side) in the reference's order, over every box whose
// grown box pokes out of the domain on that side.
// ---------------------------------------------------------------------------
__global__ void k_domain_bc(const BoxGeom* __restrict__ geo, const FabView* __restrict__ fv, double* __restrict__ x,
                            int nboxes, int3 ng, int ncomp, int axis, int side, int dlo, int dhi, int cond,
                            double value) {
  pdl_entry();
  const int b = blockIdx.y;
  if (b >= nboxes) return;
  const BoxGeom g = geo[b];
  const FabView F = fv[b];
  const int gw[3] = {ng.x, ng.y, ng.z};
  int glo[3], gn[3];
  for (int a = 0; a < 3; ++a) {
    glo[a] = g.lo[a] - gw[a];
    gn[a] = g.n[a] + 2 * gw[a];
  }
  int width, first, edge;
  if (side == 0) {
    width = dlo - glo[axis];
    first = glo[axis];
    edge = dlo;
  } else {
    width = glo[axis] + gn[axis] - 1 - dhi;
    first = dhi + 1;
    edge = dhi;
  }
  if (width <= 0) return;
  int ext[3] = {gn[0], gn[1], gn[2]};
  ext[axis] = width;
  const int64_t cells = (int64_t)ext[0] * ext[1] * ext[2];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < cells * ncomp;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(e / cells);
    int64_t r = e - (int64_t)n * cells;
    int c[3];
    c[2] = (int)(r % ext[2]);
    r /= ext[2];
    c[1] = (int)(r % ext[1]);
    c[0] = (int)(r / ext[1]);
    int gidx[3] = {glo[0] + c[0], glo[1] + c[1], glo[2] + c[2]};
    gidx[axis] = first + c[axis];
    auto addr = [&](const int* q) {
      return F.off + n * F.cs + (int64_t)(q[0] - g.lo[0]) * F.s0 + (int64_t)(q[1] - g.lo[1]) * F.s1 +
             (q[2] - g.lo[2]);
    };
    double v = value;
    if (cond == 2) {
      int src[3] = {gidx[0], gidx[1], gidx[2]};
      src[axis] = edge;
      v = x[addr(src)];
    } else if (cond == 3) {  // value * the cell mirrored across the face
      int src[3] = {gidx[0], gidx[1], gidx[2]};
      src[axis] = side == 0 ? 2 * dlo - 1 - gidx[axis] : 2 * dhi + 1 - gidx[axis];
      v = value * x[addr(src)];
    }
    x[addr(gidx)] = v;
  }
}

// setval (fabarray.py:119-122 / Fab.setval :58-65) over every resident box:
// components [c0, c1), the valid box grown by `grow` cells per axis.
__global__ void k_setval(const BoxGeom* __restrict__ geo, const FabView* __restrict__ fv, double* __restrict__ x,
                         int nboxes, int box, int3 grow, int c0, int c1, double value, int ghosts_only) {
  pdl_entry();
  const int b = box >= 0 ? box : blockIdx.y;
  if (b >= nboxes) return;
  const BoxGeom g = geo[b];
  const FabView F = fv[b];
  const int e0 = g.n[0] + 2 * grow.x, e1 = g.n[1] + 2 * grow.y, e2 = g.n[2] + 2 * grow.z;
  const int64_t plane = (int64_t)e1 * e2, cells = (int64_t)e0 * plane;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < cells * (c1 - c0);
       t += (int64_t)gridDim.x * blockDim.x) {
    const int c = c0 + (int)(t / cells);
    int64_t r = t - (int64_t)(c - c0) * cells;
    const int i = (int)(r / plane) - grow.x;
    r -= (int64_t)(i + grow.x) * plane;
    const int j = (int)(r / e2) - grow.y;
    const int k = (int)(r - (int64_t)(j + grow.y) * e2) - grow.z;
    if (ghosts_only && i >= 0 && i < g.n[0] && j >= 0 && j < g.n[1] && k >= 0 && k < g.n[2]) continue;
    x[F.off + (int64_t)c * F.cs + (int64_t)i * F.s0 + (int64_t)j * F.s1 + k] = value;
  }
}

__global__ void k_fill(double* __restrict__ x, int64_t n, double value) {
  pdl_entry();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    x[t] = value;
}

const Level& L(const amrb_level* p) {
  if (!p) throw Error(AMRB_EINVAL, "null level");
  return *reinterpret_cast<const Level*>(p);
}
Level& Lm(const amrb_level* p) { return const_cast<Level&>(L(p)); }
const Field& F(const amrb_field* p) {
  if (!p) throw Error(AMRB_EINVAL, "null field");
  return *reinterpret_cast<const Field*>(p);
}

void need_ghost(const Field& f, int g, const char* what) {
  if (f.ngrow < g) throw Error(AMRB_EINVAL, std::string(what) + ": needs ghost width >= " + std::to_string(g));
}

void need_same_level(const Field& f, const Level& lv, const char* what) {
  if (f.lv != &lv) throw Error(AMRB_EINVAL, std::string(what) + ": field bound to another level");
}

}  // namespace
}  // namespace amrb

using namespace amrb;

extern "C" const char* amrb_last_error(void) { return amrb::g_last_error.c_str(); }
extern "C" int amrb_version(void) { return 1; }
extern "C" int amrb_set_option(const char* name, int64_t value) {
  return amrb::guarded([&] {
    if (!name) throw amrb::Error(AMRB_EINVAL, "set_option: null name");
    std::lock_guard<std::mutex> lk(amrb::g_opt_mu);
    auto it = amrb::options().find(name);
    if (it == amrb::options().end()) throw amrb::Error(AMRB_EINVAL, std::string("unknown option ") + name);
    it->second = value;
  });
}
extern "C" int amrb_get_option(const char* name, int64_t* value) {
  return amrb::guarded([&] {
    if (!name || !value) throw amrb::Error(AMRB_EINVAL, "get_option: null argument");
    std::lock_guard<std::mutex> lk(amrb::g_opt_mu);
    auto it = amrb::options().find(name);
    if (it == amrb::options().end()) throw amrb::Error(AMRB_EINVAL, std::string("unknown option ") + name);
    *value = it->second;
  });
}
extern "C" int64_t amrb_launch_count(void) { return (int64_t)amrb::g_launches.load(); }

namespace amrb {
namespace {
__global__ void k_store_host(const double* __restrict__ src, double* dst, int64_t n) {
  pdl_entry();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
  // (no system fence: the stores are visible to the host once the kernel has
  // completed and the host synchronised with the stream)
}
}  // namespace
}  // namespace amrb

// Small device -> pinned-host transfers by a kernel (UVA stores), so they do
// not queue behind bulk copies on the copy engines.
extern "C" int amrb_store_host(const double* src, double* host_dst, int64_t n, void* stream) {
  return amrb::guarded([&] {
    if (n < 0 || (n && (!src || !host_dst))) throw amrb::Error(AMRB_EINVAL, "amrb_store_host: bad arguments");
    if (!n) return;
    amrb::launch_k(amrb::k_store_host, 1, 32, 0, (cudaStream_t)stream, src, host_dst, n);
    amrb::check_launch("k_store_host");
  });
}

extern "C" int amrb_fill(double* ptr, int64_t n, double value, void* stream) {
  return amrb::guarded([&] {
    if (n < 0 || (n && !ptr)) throw amrb::Error(AMRB_EINVAL, "amrb_fill: bad arguments");
    if (!n) return;
    const long long blocks = std::min<long long>((n + 255) / 256, 8LL * amrb::num_sms());
    amrb::launch_k(amrb::k_fill, (unsigned)blocks, 256, 0, (cudaStream_t)stream, ptr, n, value);
    amrb::check_launch("k_fill");
  });
}

extern "C" int amrb_setval(const amrb_level* lv_, amrb_field* f, double* base, int box, int comp0, int comp1,
                           int ghosts, double value, void* stream) {
  return amrb::guarded([&] {
    const amrb::Level& lv = amrb::L(lv_);
    const amrb::Field& fld = amrb::F(f);
    amrb::need_same_level(fld, lv, "setval");
    if (comp0 < 0 || comp1 < comp0) throw amrb::Error(AMRB_EINVAL, "setval: bad component range");
    if (box >= lv.nboxes || (box >= 0 && !lv.resident[box])) throw amrb::Error(AMRB_EINVAL, "setval: box not resident");
    if (lv.nboxes == 0 || comp1 == comp0) return;
    if (ghosts < 0 || ghosts > 2) throw amrb::Error(AMRB_EINVAL, "setval: ghosts must be 0, 1 or 2");
    const int3 gw = ghosts ? make_int3(fld.ng3[0], fld.ng3[1], fld.ng3[2]) : make_int3(0, 0, 0);
    amrb::launch_k(amrb::k_setval, dim3(box >= 0 ? 64 : 16, box >= 0 ? 1 : lv.nboxes), 256, 0, (cudaStream_t)stream,
                   lv.dgeo.p, fld.dev.p, base, lv.nboxes, box, gw, comp0, comp1, value, ghosts == 2 ? 1 : 0);
    amrb::check_launch("k_setval");
  });
}

namespace amrb {
namespace {
// FillBoundary of a single periodic box (the box is the whole domain): every
// ghost cell within w of the box is a copy of the valid cell its periodic
// image names -- the records fabarray.py:254-277 builds for this layout, as
// one kernel without a record table.  Warps take whole grown rows (rows of
// the ghost planes, ghost rows of the valid planes), threads the 2w ghost
// cells at the two ends of each valid row (16-byte pairs when w = 2).
__device__ __forceinline__ int wrap_idx(int x, int n) { return x < 0 ? x + n : (x >= n ? x - n : x); }

__global__ void __launch_bounds__(256) k_wrap_fill(double* base, FabView v, int n0, int n1, int n2, int w, int ncomp,
                                                   int blocks_a, int pairs) {
  pdl_entry();
  const int rows_a = 2 * w * (n1 + 2 * w) + n0 * 2 * w;
  const int segs = (n2 + 2 * w + 31) / 32;  // 32-cell segments per grown row: one per warp
  if ((int)blockIdx.x < blocks_a) {
    const int item = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    const int ra = item / segs;
    if (ra >= rows_a) return;
    const int k = (item - ra * segs) * 32 + lane - w;
    int ip, j;
    const int ga = 2 * w * (n1 + 2 * w);
    if (ra < ga) {
      const int pl = ra / (n1 + 2 * w);
      ip = pl < w ? pl - w : n0 + (pl - w);
      j = ra - pl * (n1 + 2 * w) - w;
    } else {
      const int r2 = ra - ga;
      ip = r2 / (2 * w);
      const int t = r2 - ip * 2 * w;
      j = t < w ? t - w : n1 + (t - w);
    }
    const int64_t drow = v.off + (int64_t)ip * v.s0 + (int64_t)j * v.s1;
    const int64_t srow = v.off + (int64_t)wrap_idx(ip, n0) * v.s0 + (int64_t)wrap_idx(j, n1) * v.s1;
    if (k < n2 + w)
      for (int c = 0; c < ncomp; ++c) base[drow + c * v.cs + k] = base[srow + c * v.cs + wrap_idx(k, n2)];
    return;
  }
  const int rb = (blockIdx.x - blocks_a) * 256 + threadIdx.x;
  if (rb >= n0 * n1) return;
  const int ip = rb / n1, j = rb - ip * n1;
  const int64_t row = v.off + (int64_t)ip * v.s0 + (int64_t)j * v.s1;
  for (int c = 0; c < ncomp; ++c) {
    double* r = base + row + c * v.cs;
    if (pairs) {  // w = 2: cols -2, -1 <- n2-2, n2-1 and n2, n2+1 <- 0, 1
      const double2 lo = *reinterpret_cast<const double2*>(r + n2 - 2);
      const double2 hi = *reinterpret_cast<const double2*>(r);
      *reinterpret_cast<double2*>(r - 2) = lo;
      *reinterpret_cast<double2*>(r + n2) = hi;
    } else {
      for (int k = 1; k <= w; ++k) {
        r[-k] = r[n2 - k];
        r[n2 + k - 1] = r[k - 1];
      }
    }
  }
}
}  // namespace
}  // namespace amrb

extern "C" int amrb_fill_wrap(const amrb_level* lv_, amrb_field* f, double* base, int ncomp, int width,
                              void* stream) {
  return amrb::guarded([&] {
    const amrb::Level& lv = amrb::L(lv_);
    const amrb::Field& fld = amrb::F(f);
    amrb::need_same_level(fld, lv, "fill_wrap");
    if (lv.nboxes != 1 || !lv.resident[0]) throw amrb::Error(AMRB_ENOTSUP, "fill_wrap: one resident box only");
    const amrb::BoxGeom& g = lv.geo[0];
    if (ncomp < 1) throw amrb::Error(AMRB_EINVAL, "fill_wrap: ncomp < 1");
    if (width < 1) return;
    for (int a = 0; a < 3; ++a)
      if (fld.ng3[a] < width || g.n[a] < width) throw amrb::Error(AMRB_ENOTSUP, "fill_wrap: ghost width exceeds box");
    const amrb::FabView v = fld.host[0];
    const int n0 = g.n[0], n1 = g.n[1], n2 = g.n[2];
    const int rows_a = 2 * width * (n1 + 2 * width) + n0 * 2 * width;
    const long long items_a = (long long)rows_a * ((n2 + 2 * width + 31) / 32);
    const int blocks_a = (int)((items_a + 7) / 8);
    const long long rows_b = (long long)n0 * n1;
    const int blocks_b = (int)((rows_b + 255) / 256);
    const bool even = !(v.off & 1) && !(v.s0 & 1) && !(v.s1 & 1) && !(v.cs & 1) && !(n2 & 1);
    const int pairs = width == 2 && even && !(reinterpret_cast<uintptr_t>(base) & 15);
    amrb::launch_k(amrb::k_wrap_fill, blocks_a + blocks_b, 256, 0, (cudaStream_t)stream, base, v, n0, n1, n2, width,
                   ncomp, blocks_a, pairs);
    amrb::check_launch("k_wrap_fill");
  });
}

extern "C" int amrb_zero(double* ptr, int64_t n, void* stream) {
  return amrb::guarded([&] {
    if (n < 0 || (n && !ptr)) throw amrb::Error(AMRB_EINVAL, "amrb_zero: bad arguments");
    if (n) AMRB_CUDA(cudaMemsetAsync(ptr, 0, (size_t)n * sizeof(double), (cudaStream_t)stream));
  });
}

extern "C" int amrb_level_create(int nboxes, const int32_t* boxes, const uint8_t* resident, amrb_level** out) {
  return guarded([&] {
    if (nboxes < 0 || (nboxes && !boxes) || !out) throw Error(AMRB_EINVAL, "amrb_level_create: bad arguments");
    auto lv = std::make_unique<Level>();
    lv->nboxes = nboxes;
    lv->geo.resize(nboxes);
    lv->resident.assign(nboxes, 1);
    for (int b = 0; b < nboxes; ++b) {
      for (int a = 0; a < 3; ++a) {
        lv->geo[b].lo[a] = boxes[6 * b + a];
        lv->geo[b].n[a] = boxes[6 * b + 3 + a] - boxes[6 * b + a] + 1;
        if (lv->geo[b].n[a] < 1) throw Error(AMRB_EINVAL, "empty box in level");
      }
      if (resident) lv->resident[b] = resident[b];
    }
    lv->dgeo.upload(lv->geo);
    lv->slot.assign(nboxes, 0);
    for (int b = 0, k = 0; b < nboxes; ++b)
      if (lv->resident[b]) lv->slot[b] = k++;
    lv->dslot.upload(lv->slot);
    *out = reinterpret_cast<amrb_level*>(lv.release());
  });
}

extern "C" int amrb_level_destroy(amrb_level* lv) {
  delete reinterpret_cast<Level*>(lv);
  return AMRB_OK;
}

extern "C" int amrb_field_create(const amrb_level* lv_, const int64_t* fabtab, int ngrow, amrb_field** out) {
  return guarded([&] {
    const Level& lv = L(lv_);
    if (!fabtab || !out || ngrow < 0) throw Error(AMRB_EINVAL, "amrb_field_create: bad arguments");
    auto f = std::make_unique<Field>();
    f->lv = &lv;
    f->ngrow = ngrow;
    f->host.resize(lv.nboxes);
    for (int b = 0; b < lv.nboxes; ++b) {
      const int64_t* t = fabtab + (int64_t)b * AMRB_FABTAB_W;
      FabView v;
      v.cs = t[1];
      v.s0 = t[2];
      v.s1 = t[3];
      // offset of the valid lo cell = grown lo offset + ngrow in each axis
      v.off = t[0] + (lv.geo[b].lo[0] - t[4]) * v.s0 + (lv.geo[b].lo[1] - t[5]) * v.s1 + (lv.geo[b].lo[2] - t[6]);
      f->host[b] = v;
      if (b == 0)
        for (int a = 0; a < 3; ++a) f->ng3[a] = (int)(lv.geo[b].lo[a] - t[4 + a]);
    }
    f->dev.upload(f->host);
    *out = reinterpret_cast<amrb_field*>(f.release());
  });
}

extern "C" int amrb_field_destroy(amrb_field* f) {
  delete reinterpret_cast<Field*>(f);
  return AMRB_OK;
}

namespace {
template <class K, class... Args>
void launch_tiles(const TileTable& tt, K kernel, cudaStream_t st, dim3 block, Args... args) {
  if (tt.host.empty()) return;
  launch_k(kernel, (unsigned)tt.host.size(), block, 0, st, tt.dev.p, tt.ti, args...);
}

// Tile depth along i: 8 planes per CTA (register reuse along i) on levels big
// enough to fill the chip several times over, 1 plane on small levels so the
// latency-bound work spreads over more CTAs.
int pick_ti(const Level& lv, int tj, int tk) {
  long long tiles8 = 0;
  for (int b = 0; b < lv.nboxes; ++b) {
    if (!lv.resident[b]) continue;
    const BoxGeom& g = lv.geo[b];
    tiles8 += (long long)((g.n[0] + 7) / 8) * ((g.n[1] + tj - 1) / tj) * ((g.n[2] + tk - 1) / tk);
  }
  return tiles8 >= 4LL * num_sms() ? 8 : 1;
}
}  // namespace

extern "C" int amrb_lap_apply(const amrb_level* lv_, amrb_field* out, double* out_base, const amrb_field* phi,
                              const double* phi_base, const double dh[3], void* stream) {
  return guarded([&] {
    Level& lv = Lm(lv_);
    need_ghost(F(phi), 1, "lap_apply");
    need_same_level(F(out), lv, "lap_apply");
    need_same_level(F(phi), lv, "lap_apply");
    const auto& tt = lv.tiles(pick_ti(lv, kTJ, kTK), kTJ, kTK);
    launch_tiles(tt, k_stencil<Op::kLap>, (cudaStream_t)stream, dim3(32, 8), lv.dgeo.p, F(out).dev.p, out_base,
                 (const FabView*)nullptr, (const double*)nullptr, F(phi).dev.p, phi_base, make_coef(dh));
    check_launch("k_stencil<lap>");
  });
}

extern "C" int amrb_residual(const amrb_level* lv_, amrb_field* r, double* r_base, const amrb_field* rhs,
                             const double* rhs_base, const amrb_field* phi, const double* phi_base,
                             const double dh[3], void* stream) {
  return guarded([&] {
    Level& lv = Lm(lv_);
    need_ghost(F(phi), 1, "residual");
    for (auto* f : {r, (amrb_field*)rhs, (amrb_field*)phi}) need_same_level(F(f), lv, "residual");
    const auto& tt = lv.tiles(pick_ti(lv, kTJ, kTK), kTJ, kTK);
    launch_tiles(tt, k_stencil<Op::kResid>, (cudaStream_t)stream, dim3(32, 8), lv.dgeo.p, F(r).dev.p, r_base,
                 F(rhs).dev.p, rhs_base, F(phi).dev.p, phi_base, make_coef(dh));
    check_launch("k_stencil<resid>");
  });
}

extern "C" int amrb_gsrb_color(const amrb_level* lv_, amrb_field* phi, double* phi_base, const amrb_field* rhs,
                               const double* rhs_base, const double dh[3], int color, void* stream) {
  return guarded([&] {
    Level& lv = Lm(lv_);
    need_ghost(F(phi), 1, "gsrb_color");
    need_same_level(F(phi), lv, "gsrb_color");
    need_same_level(F(rhs), lv, "gsrb_color");
    if (color != 0 && color != 1) throw Error(AMRB_EINVAL, "color must be 0 or 1");
    const auto& tt = lv.tiles(pick_ti(lv, kTJ, 2 * kTK), kTJ, 2 * kTK);
    launch_tiles(tt, k_gsrb_color, (cudaStream_t)stream, dim3(32, 8), lv.dgeo.p, F(phi).dev.p, phi_base,
                 F(rhs).dev.p, rhs_base, make_coef(dh), color);
    check_launch("k_gsrb_color");
  });
}

namespace {
constexpr int kSweepCI = 16;

template <int TJ, int TK>
void launch_sweep(Level& lv, const Field& a, const double* a_base, const Field& b, double* b_base, const Field& r,
                  const double* r_base, const Coef& cf, const int fixed_lo[3], const int fixed_hi[3],
                  cudaStream_t st) {
  const auto& tt = lv.tiles(kSweepCI, TJ, TK);
  if (tt.host.empty()) return;
  SweepArgs args;
  args.tiles = tt.dev.p;
  args.geo = lv.dgeo.p;
  args.fa = a.dev.p;
  args.fb = b.dev.p;
  args.fr = r.dev.p;
  args.a = a_base;
  args.b = b_base;
  args.rhs = r_base;
  args.cf = cf;
  args.ci = kSweepCI;
  for (int x = 0; x < 3; ++x) {
    args.fixed_lo[x] = fixed_lo[x];
    args.fixed_hi[x] = fixed_hi[x];
  }
  const size_t smem = sizeof(SweepSmem<TJ, TK>);
  static bool configured = false;
  if (!configured) {
    AMRB_CUDA(cudaFuncSetAttribute(k_gsrb_sweep<TJ, TK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = true;
  }
  launch_k(k_gsrb_sweep<TJ, TK>, (unsigned)tt.host.size(), dim3(32, 8), smem, st, args);
  check_launch("k_gsrb_sweep");
}
template <int TJ, int TK>
void launch_sweep_full(Level& lv, const Field& a, const double* a_base, const Field& b, double* b_base,
                       const Field& r, const double* r_base, const Coef& cf, const int fixed_lo[3],
                       const int fixed_hi[3], bool fixed, cudaStream_t st) {
  const auto& cols = lv.columns(TJ, TK);
  if (cols.host.empty()) return;
  Sweep3Args args;
  args.cols = cols.dev.p;
  args.ncols = (int)cols.host.size();
  args.total = cols.total;
  args.geo = lv.dgeo.p;
  args.fa = a.dev.p;
  args.fb = b.dev.p;
  args.fr = r.dev.p;
  args.a = a_base;
  args.b = b_base;
  args.rhs = r_base;
  args.cf = cf;
  for (int x = 0; x < 3; ++x) {
    args.fixed_lo[x] = fixed_lo[x];
    args.fixed_hi[x] = fixed_hi[x];
  }
  const size_t smem = sizeof(Sweep3Smem<TJ, TK>);
  auto kern = fixed ? k_gsrb_sweep3<TJ, TK, true> : k_gsrb_sweep3<TJ, TK, false>;
  static int per_sm[2] = {0, 0};
  if (!per_sm[fixed]) {
    AMRB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    AMRB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[fixed], kern, 256, smem));
    per_sm[fixed] = std::max(per_sm[fixed], 1);
  }
  // enough CTAs to fill the chip, but >= 16 planes (or a whole column) each
  long long want = std::max<long long>((long long)cols.host.size(), cols.total / 16);
  long long grid = std::min<long long>((long long)per_sm[fixed] * num_sms(), want);
  launch_k(kern, (unsigned)std::max<long long>(grid, 1), 256, smem, st, args);
  check_launch("k_gsrb_sweep3");
}
}  // namespace

extern "C" int amrb_gsrb_sweep(const amrb_level* lv_, const amrb_field* a, const double* a_base, amrb_field* b,
                                  double* b_base, const amrb_field* rhs, const double* rhs_base, const double dh[3],
                                  const int32_t* fixed_lohi, const uint64_t* push, void* stream) {
  return guarded([&] {
    Level& lv = Lm(lv_);
    need_ghost(F(a), 2, "gsrb_sweep (phi in)");
    need_ghost(F(rhs), 1, "gsrb_sweep (rhs)");
    for (auto* f : {a, (const amrb_field*)b, rhs}) need_same_level(F(f), lv, "gsrb_sweep");
    if (!lv.all_even()) throw Error(AMRB_EINVAL, "gsrb_sweep needs even box extents");
    int flo[3] = {-(1 << 30), -(1 << 30), -(1 << 30)}, fhi[3] = {1 << 30, 1 << 30, 1 << 30};
    if (fixed_lohi)
      for (int x = 0; x < 3; ++x) {
        flo[x] = fixed_lohi[x];
        fhi[x] = fixed_lohi[3 + x];
      }
    // full-tile fast path when every box is a multiple of the tile
    int minj = 1 << 30, mink = 1 << 30, maxk = 0;
    for (auto& g : lv.geo) {
      minj = std::min(minj, g.n[1]);
      mink = std::min(mink, g.n[2]);
      maxk = std::max(maxk, g.n[2]);
    }
    auto divides = [&](int tj, int tk) {
      for (auto& g : lv.geo)
        if (g.n[1] % tj || g.n[2] % tk) return false;
      return true;
    };
    const bool fixed = fixed_lohi != nullptr;
    cudaStream_t st = (cudaStream_t)stream;
    const Coef cf = make_coef(dh);
    const long long* ptab = reinterpret_cast<const long long*>(push);
    if (ptab) need_ghost(F(b), 2, "gsrb_sweep (pushed phi out)");
    if (option("sweep_kernel") == 0 &&
        launch_sweep_stream(0, lv, F(a), a_base, F(b), b_base, F(rhs), rhs_base, cf, flo, fhi, st, nullptr, nullptr,
                            nullptr, nullptr, ptab))
      return;
    if (ptab) throw Error(AMRB_ENOTSUP, "gsrb_sweep: ghost push needs the k_gsrb_stream path");
    if (divides(16, 64))
      launch_sweep_full<16, 64>(lv, F(a), a_base, F(b), b_base, F(rhs), rhs_base, cf, flo, fhi, fixed, st);
    else if (divides(16, 32))
      launch_sweep_full<16, 32>(lv, F(a), a_base, F(b), b_base, F(rhs), rhs_base, cf, flo, fhi, fixed, st);
    else if (divides(16, 16))
      launch_sweep_full<16, 16>(lv, F(a), a_base, F(b), b_base, F(rhs), rhs_base, cf, flo, fhi, fixed, st);
    else if (divides(8, 8))
      launch_sweep_full<8, 8>(lv, F(a), a_base, F(b), b_base, F(rhs), rhs_base, cf, flo, fhi, fixed, st);
    else if (divides(4, 4))
      launch_sweep_full<4, 4>(lv, F(a), a_base, F(b), b_base, F(rhs), rhs_base, cf, flo, fhi, fixed, st);
    else if (maxk >= 64)
      launch_sweep<16, 64>(lv, F(a), a_base, F(b), b_base, F(rhs), rhs_base, cf, flo, fhi, st);
    else
      launch_sweep<16, 32>(lv, F(a), a_base, F(b), b_base, F(rhs), rhs_base, cf, flo, fhi, st);
    (void)minj;
    (void)mink;
  });
}

extern "C" int amrb_gsrb_sweep_norm(const amrb_level* lv_, const amrb_field* a, const double* a_base, amrb_field* b,
                                    double* b_base, const amrb_field* rhs, const double* rhs_base, const double dh[3],
                                    const int32_t* fixed_lohi, uint64_t* norm, const uint64_t* push, void* stream) {
  return guarded([&] {
    Level& lv = Lm(lv_);
    need_ghost(F(a), 2, "gsrb_sweep_norm (phi in)");
    need_ghost(F(rhs), 1, "gsrb_sweep_norm (rhs)");
    for (auto* f : {a, (const amrb_field*)b, rhs}) need_same_level(F(f), lv, "gsrb_sweep_norm");
    if (!norm) throw Error(AMRB_EINVAL, "gsrb_sweep_norm: null norm");
    if (push) need_ghost(F(b), 2, "gsrb_sweep_norm (pushed phi out)");
    if (!lv.all_even()) throw Error(AMRB_EINVAL, "gsrb_sweep needs even box extents");
    int flo[3] = {-(1 << 30), -(1 << 30), -(1 << 30)}, fhi[3] = {1 << 30, 1 << 30, 1 << 30};
    if (fixed_lohi)
      for (int x = 0; x < 3; ++x) {
        flo[x] = fixed_lohi[x];
        fhi[x] = fixed_lohi[3 + x];
      }
    if (option("sweep_kernel") != 0 ||
        !launch_sweep_stream(2, lv, F(a), a_base, F(b), b_base, F(rhs), rhs_base, make_coef(dh), flo, fhi,
                             (cudaStream_t)stream, nullptr, nullptr, nullptr,
                             reinterpret_cast<unsigned long long*>(norm), reinterpret_cast<const long long*>(push)))
      throw Error(AMRB_ENOTSUP, "gsrb_sweep_norm: level does not take the k_gsrb_stream path");
  });
}

extern "C" int amrb_gsrb_sweep_pull(const amrb_level* lv_, const amrb_field* a, double* a_base, amrb_field* b,
                                    double* b_base, const amrb_field* rhs, const double* rhs_base, const double dh[3],
                                    const uint64_t* pull, const uint64_t* pad_ptrs, int rank, int nranks,
                                    uint32_t* epoch, uint64_t* norm, void* stream) {
  return guarded([&] {
    Level& lv = Lm(lv_);
    need_ghost(F(a), 2, "gsrb_sweep_pull (phi in)");
    need_ghost(F(rhs), 1, "gsrb_sweep_pull (rhs)");
    for (auto* f : {a, (const amrb_field*)b, rhs}) need_same_level(F(f), lv, "gsrb_sweep_pull");
    if (!pull) throw Error(AMRB_EINVAL, "gsrb_sweep_pull: null pull table");
    if (nranks < 1 || nranks > kMaxPeers || rank < 0 || rank >= nranks || (nranks > 1 && (!pad_ptrs || !epoch)))
      throw Error(AMRB_EINVAL, "gsrb_sweep_pull: bad peer arguments");
    if (!lv.all_even()) throw Error(AMRB_EINVAL, "gsrb_sweep needs even box extents");
    StreamPull pl;
    pl.tab = reinterpret_cast<const long long*>(pull);
    pl.rank = rank;
    pl.nranks = nranks;
    pl.epoch = epoch;
    for (int r = 0; r < nranks && pad_ptrs; ++r) pl.pads[r] = reinterpret_cast<uint32_t*>(pad_ptrs[r]);
    const int flo[3] = {-(1 << 30), -(1 << 30), -(1 << 30)}, fhi[3] = {1 << 30, 1 << 30, 1 << 30};
    if (option("sweep_kernel") != 0 ||
        !launch_sweep_stream(norm ? 2 : 0, lv, F(a), a_base, F(b), b_base, F(rhs), rhs_base, make_coef(dh), flo, fhi,
                             (cudaStream_t)stream, nullptr, nullptr, nullptr,
                             reinterpret_cast<unsigned long long*>(norm), nullptr, &pl))
      throw Error(AMRB_ENOTSUP, "gsrb_sweep_pull: level does not take the k_gsrb_stream path");
  });
}

extern "C" int amrb_gsrb_sweep_prolong(const amrb_level* lv_, const amrb_field* a, const double* a_base,
                                          amrb_field* b, double* b_base, const amrb_field* rhs, const double* rhs_base,
                                          const double dh[3], const amrb_level* clv_, const amrb_field* c,
                                          const double* c_base, const uint64_t* push, void* stream) {
  return guarded([&] {
    Level& lv = Lm(lv_);
    const Level& clv = L(clv_);
    need_ghost(F(a), 2, "gsrb_sweep_prolong (phi in)");
    need_ghost(F(rhs), 1, "gsrb_sweep_prolong (rhs)");
    need_ghost(F(c), 1, "gsrb_sweep_prolong (coarse)");
    for (auto* f : {a, (const amrb_field*)b, rhs}) need_same_level(F(f), lv, "gsrb_sweep_prolong");
    need_same_level(F(c), clv, "gsrb_sweep_prolong (coarse)");
    if (!lv.all_even()) throw Error(AMRB_EINVAL, "gsrb_sweep_prolong needs even box extents");
    // coarse box b must be the box-local coarsening (ratio 2) of fine box b
    if (clv.nboxes != lv.nboxes) throw Error(AMRB_EINVAL, "gsrb_sweep_prolong: box counts differ");
    for (int x = 0; x < lv.nboxes; ++x) {
      if (clv.resident[x] != lv.resident[x]) throw Error(AMRB_EINVAL, "gsrb_sweep_prolong: residency differs");
      for (int d = 0; d < 3; ++d)
        if (lv.geo[x].lo[d] % 2 || clv.geo[x].lo[d] * 2 != lv.geo[x].lo[d] || clv.geo[x].n[d] * 2 != lv.geo[x].n[d])
          throw Error(AMRB_EINVAL, "gsrb_sweep_prolong: coarse box is not the coarsened fine box");
    }
    const int flo[3] = {-(1 << 30), -(1 << 30), -(1 << 30)}, fhi[3] = {1 << 30, 1 << 30, 1 << 30};
    if (option("sweep_kernel") != 0 ||
        !launch_sweep_stream(1, lv, F(a), a_base, F(b), b_base, F(rhs), rhs_base, make_coef(dh), flo, fhi,
                             (cudaStream_t)stream, &clv, &F(c), c_base, nullptr,
                             reinterpret_cast<const long long*>(push)))
      throw Error(AMRB_ENOTSUP, "gsrb_sweep_prolong: level does not take the k_gsrb_stream path");
  });
}

namespace {
int3 ratio3(const int32_t* ratio) {
  int3 r = make_int3(2, 2, 2);
  if (ratio) r = make_int3(ratio[0], ratio[1], ratio[2]);
  if ((r.x != 1 && r.x != 2) || (r.y != 1 && r.y != 2) || (r.z != 1 && r.z != 2))
    throw Error(AMRB_EINVAL, "device restriction/prolongation supports ratio 1 or 2 per axis");
  return r;
}
}  // namespace

extern "C" int amrb_restrict(const amrb_level* clv_, amrb_field* crse, double* crse_base, const amrb_field* fine,
                             const double* fine_base, int ncomp, const int32_t* ratio, int mode, void* stream) {
  return guarded([&] {
    Level& lv = Lm(clv_);
    need_same_level(F(crse), lv, "restrict");
    const int3 r = ratio3(ratio);
    if (mode != 0 && mode != 1) throw Error(AMRB_EINVAL, "restrict mode must be 0 (average) or 1 (injection)");
    const auto& tt = lv.tiles(pick_ti(lv, kTJ, kTK), kTJ, kTK);
    launch_tiles(tt, k_restrict, (cudaStream_t)stream, dim3(32, 8), lv.dgeo.p, F(crse).dev.p, crse_base,
                 F(fine).dev.p, fine_base, ncomp, r, mode, 1.0 / (r.x * r.y * r.z));
    check_launch("k_restrict");
  });
}

extern "C" int amrb_residual_restrict(const amrb_level* clv_, amrb_field* crse, double* crse_base,
                                      const amrb_field* rhs, const double* rhs_base, const amrb_field* phi,
                                      const double* phi_base, const double dh[3], void* stream) {
  return guarded([&] {
    Level& lv = Lm(clv_);
    need_same_level(F(crse), lv, "residual_restrict");
    need_ghost(F(phi), 1, "residual_restrict");
    const Field& fphi = F(phi);
    if (option("sweep_kernel") == 0 && fphi.lv &&
        launch_resid_restrict_stream(const_cast<Level&>(*fphi.lv), fphi, phi_base, F(rhs), rhs_base, F(crse), crse_base,
                                     make_coef(dh), (cudaStream_t)stream))
      return;
    const auto& tt = lv.tiles(pick_ti(lv, kTJ, kTK), kTJ, kTK);
    launch_tiles(tt, k_resid_restrict, (cudaStream_t)stream, dim3(32, 8), lv.dgeo.p, F(crse).dev.p, crse_base,
                 F(rhs).dev.p, rhs_base, F(phi).dev.p, phi_base, make_coef(dh));
    check_launch("k_resid_restrict");
  });
}

extern "C" int amrb_prolong(const amrb_level* flv_, amrb_field* fine, double* fine_base, const amrb_field* crse,
                            const double* crse_base, int ncomp, const int32_t* ratio, int add, void* stream) {
  return guarded([&] {
    Level& lv = Lm(flv_);
    need_same_level(F(fine), lv, "prolong");
    const int3 r = ratio3(ratio);
    const int3 sh = make_int3(r.x == 2, r.y == 2, r.z == 2);
    const auto& tt = lv.tiles(pick_ti(lv, kTJ, kTK), kTJ, kTK);
    launch_tiles(tt, k_prolong, (cudaStream_t)stream, dim3(32, 8), lv.dgeo.p, F(fine).dev.p, fine_base,
                 F(crse).dev.p, crse_base, ncomp, add, sh);
    check_launch("k_prolong");
  });
}


extern "C" int amrb_residual_norm(const amrb_level* lv_, const amrb_field* rhs, const double* rhs_base,
                                  const amrb_field* phi, const double* phi_base, const double dh[3], double* dev_out,
                                  void* stream) {
  return guarded([&] {
    Level& lv = Lm(lv_);
    need_ghost(F(phi), 1, "residual_norm");
    need_same_level(F(rhs), lv, "residual_norm");
    need_same_level(F(phi), lv, "residual_norm");
    const auto& tt = lv.tiles(pick_ti(lv, kTJ, kTK), kTJ, kTK);
    const int n = (int)tt.host.size();
    if (lv.partials.n < (size_t)std::max(n, 1)) lv.partials.alloc(std::max(n, 1));
    cudaStream_t st = (cudaStream_t)stream;
    if (n) {
      launch_tiles(tt, k_resid_norm, st, dim3(32, 8), lv.dgeo.p, F(rhs).dev.p, rhs_base, F(phi).dev.p, phi_base,
                   make_coef(dh), lv.partials.p);
      check_launch("k_resid_norm");
    }
    launch_k(k_reduce_final, 1, 1024, 0, st, lv.partials.p, n, 3, dev_out);
    check_launch("k_reduce_final");
  });
}

extern "C" int amrb_reduce(const amrb_level* lv_, const amrb_field* x, const double* x_base, int comp, int kind,
                           double* dev_out, void* stream) {
  return guarded([&] {
    Level& lv = Lm(lv_);
    if (kind < 0 || kind > 3) throw Error(AMRB_EINVAL, "unknown reduction kind");
    need_same_level(F(x), lv, "reduce");
    const auto& tt = lv.tiles(pick_ti(lv, kTJ, kTK), kTJ, kTK);
    const int n = (int)tt.host.size();
    if (lv.partials.n < (size_t)std::max(n, 1)) lv.partials.alloc(std::max(n, 1));
    cudaStream_t st = (cudaStream_t)stream;
    if (n) {
      launch_tiles(tt, k_reduce_tiles, st, dim3(32, 8), lv.dgeo.p, F(x).dev.p, x_base, comp, kind, lv.partials.p);
      check_launch("k_reduce_tiles");
    }
    launch_k(k_reduce_final, 1, 1024, 0, st, lv.partials.p, n, kind, dev_out);
    check_launch("k_reduce");
  });
}

extern "C" int amrb_domain_bc(const amrb_level* lv_, amrb_field* f, double* base, int ncomp, const int32_t* domain,
                              const int32_t* bc, double value, void* stream) {
  return guarded([&] {
    Level& lv = Lm(lv_);
    const Field& fld = F(f);
    need_same_level(fld, lv, "domain_bc");
    if (!domain || !bc) throw Error(AMRB_EINVAL, "domain_bc: null argument");
    if (fld.ngrow == 0 || lv.nboxes == 0) return;
    for (int axis = 0; axis < 3; ++axis)
      for (int side = 0; side < 2; ++side) {
        const int cond = bc[2 * axis + side];
        if (cond == 0) continue;
        dim3 grid(64, lv.nboxes);
        launch_k(k_domain_bc, grid, 256, 0, (cudaStream_t)stream, lv.dgeo.p, fld.dev.p, base, lv.nboxes,
                                                           make_int3(fld.ng3[0], fld.ng3[1], fld.ng3[2]), ncomp,
                                                           axis, side, domain[axis], domain[3 + axis], cond, value);
        check_launch("k_domain_bc");
      }
  });
}
