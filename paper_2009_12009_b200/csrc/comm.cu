// Copy programs: a CommPlan bound to concrete device storage, plus the NCCL
// plumbing.  Replaces the reference's two-phase executor
// (/root/reference/pkg/src/amrkit/fabarray.py:326-361) and its in-process
// Transport (transport.py:27-58).
//
// Execution of one program:
//   1. pack   : records whose source is here and destination is remote are
//               gathered into the send buffer, one contiguous segment per
//               destination rank (C-order (ncomp, e0, e1, e2) record slices in
//               plan order -- byte-identical to the reference's message).
//   2. NCCL   : one ncclSend / ncclRecv per ordered peer pair inside a group.
//   3. apply  : records whose destination is here, in waves.  Copy programs
//               have two waves (local records, then records fed from the
//               receive buffer); add programs (sum_boundary) put records that
//               touch the same cells in successive waves so every cell sees its
//               contributions in plan order, which keeps sums bit-identical to
//               the reference for any rank count.
//
// The kernel walks a flat index space over all records of a wave (see k_copy
// for how records map to CTAs).
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>

#include "device.h"
#include "peer.cuh"

namespace amrb {

unsigned long long* g_fault_box = nullptr;  // amrb_set_fault_mailbox
unsigned long long* g_fault_dev = nullptr;

Fault current_fault() {
  Fault f;
  f.box = g_fault_box;
  f.dev = g_fault_box ? g_fault_dev : nullptr;
  const int64_t ms = option("peer_timeout_ms");
  f.timeout_ns = ms > 0 ? (unsigned long long)ms * 1000000ull : 0ull;
  return f;
}

namespace {

constexpr int kCopyThreads = 256;
constexpr int kCopyItems = 4;
constexpr int kChunk = kCopyThreads * kCopyItems;

struct DevRec {
  int64_t src;    // element offset of the first source cell (comp 0)
  int64_t dst;    // element offset of the first destination cell (comp 0)
  int64_t begin;  // first flat index of this record in its wave
  int64_t ss0, ss1, scs;
  int64_t ds0, ds1, dcs;
  int32_t e0, e1, e2;
  int32_t from_buf;  // 1: source is the receive/staging buffer
  int32_t src_peer = -1;  // >= 0: source lives in that peer's storage (p2p mode)
  int32_t vec = 0;  // 1: moved as 16-byte pairs (even row length, even offsets and strides; large records)
};

struct PeerPtrs {
  const double* p[kMaxPeers];
};

// Device barrier fused into a p2p copy launch (see k_copy): pads[r] = rank r's
// signal pad, epoch = {this rank's barrier epoch, CTA completion ticket}.


struct SyncArgs {
  uint32_t* pads[kMaxPeers];
  uint32_t* epoch;
  int rank, nranks, on;
  Fault fault;
};

struct Wave {
  std::vector<DevRec> host;
  std::vector<int2> blocks;  // (record, first flat index inside the record)
  DevArray<DevRec> recs;
  DevArray<int2> dblocks;
  int64_t total = 0;
};

// Blocks: a record of >= kSmall flat indices gets one CTA per chunk of kChunk
// (no search); runs of consecutive small records (edges and corners: 1-64
// cells each) are packed into shared CTAs of up to kChunk indices / kPackMax
// records, and each thread binary-searches the packed records' offsets (staged
// in shared memory).  Every thread issues all of its loads before its stores
// so remote (NVLink) and local latencies overlap.
constexpr int kSmall = kChunk / 4;
constexpr int kPackMax = 256;

// (comp, i, j, k) of flat index loc of a record, as source / destination
// element offsets.  A record holds < 2^31 cells per component, so after the
// component split the index arithmetic is unsigned 32-bit (the 64-bit
// division runs only for multi-component records).
__device__ __forceinline__ void rec_cell(const DevRec& r, int64_t loc, int64_t cells, int ncomp, int64_t& so,
                                         int64_t& dofs) {
  int c = 0;
  unsigned t = (unsigned)loc;
  if (ncomp > 1) {
    c = (int)(loc / cells);
    t = (unsigned)(loc - (int64_t)c * cells);
  }
  const unsigned e2 = (unsigned)r.e2, e1 = (unsigned)r.e1;
  const unsigned row = t / e2;
  const unsigned k = t - row * e2;
  const unsigned i = row / e1;
  const unsigned j = row - i * e1;
  so = r.src + c * r.scs + (int64_t)i * r.ss0 + (int64_t)j * r.ss1 + k;
  dofs = r.dst + c * r.dcs + (int64_t)i * r.ds0 + (int64_t)j * r.ds1 + k;
}

// rec_cell for a vec record: loc indexes cell PAIRS (comp, i, j, k/2)
__device__ __forceinline__ void rec_pair(const DevRec& r, int64_t loc, int64_t units, int ncomp, int64_t& so,
                                         int64_t& dofs) {
  int c = 0;
  unsigned t = (unsigned)loc;
  if (ncomp > 1) {
    c = (int)(loc / units);
    t = (unsigned)(loc - (int64_t)c * units);
  }
  const unsigned e2h = (unsigned)r.e2 >> 1, e1 = (unsigned)r.e1;
  const unsigned row = t / e2h;
  const unsigned k = 2 * (t - row * e2h);
  const unsigned i = row / e1;
  const unsigned j = row - i * e1;
  so = r.src + c * r.scs + (int64_t)i * r.ss0 + (int64_t)j * r.ss1 + k;
  dofs = r.dst + c * r.dcs + (int64_t)i * r.ds0 + (int64_t)j * r.ds1 + k;
}

// With sy.on (p2p fills) the launch also is the cross-rank barrier that used to
// precede it: CTA 0 publishes this rank's next epoch in every peer's pad; CTA 0
// and every CTA that reads a peer's storage wait until all peers published
// it (their previous kernels -- the producers of the data pulled here -- are
// complete); CTAs with local sources start at once.  The last CTA to finish
// advances the epoch.  CTA 0 always waits, so this launch also orders every
// peer's earlier pulls from this rank before whatever follows it here.
template <bool kAdd>
__global__ void __launch_bounds__(kCopyThreads)
    k_copy(const DevRec* __restrict__ recs, const int2* __restrict__ blocks, int ncomp, int aligned,
           const double* __restrict__ src, const double* __restrict__ buf, double* __restrict__ dst,
           const __grid_constant__ PeerPtrs peers, const __grid_constant__ SyncArgs sy) {
  amrb::pdl_entry();
  const int2 bl = blocks[blockIdx.x];
  uint32_t ep = 0;
  if (sy.on) {
    // warp 0: lane p publishes to / polls peer p concurrently (one NVLink
    // round trip whatever the peer count)
    ep = *reinterpret_cast<volatile uint32_t*>(sy.epoch) + 1;
    if (threadIdx.x < 32) {
      const int p = threadIdx.x;
      bool wait = blockIdx.x == 0;
      if (bl.x >= 0) {
        wait |= recs[bl.x].src_peer >= 0 && recs[bl.x].src_peer != sy.rank;
      } else {
        for (int q = 0; q < bl.y && !wait; ++q) wait |= recs[-bl.x - 1 + q].src_peer != sy.rank;
      }
      if (p < sy.nranks && p != sy.rank) {
        if (blockIdx.x == 0) signal_store(sy.pads[p] + sy.rank, ep);
        if (wait) peer_wait(sy.pads[sy.rank] + p, ep, sy.rank, p, sy.fault);
      }
    }
    __syncthreads();
  }
  double v[kCopyItems];
  int64_t dofs[kCopyItems];
  bool paired = false;
  if (bl.x >= 0 && recs[bl.x].vec) {  // one large record moved as 16-byte pairs
    paired = true;
    const DevRec r = recs[bl.x];
    const int64_t units = (int64_t)r.e0 * r.e1 * (r.e2 >> 1);
    const int64_t end = min(units * ncomp, (int64_t)bl.y + kChunk);
    const double* s = r.from_buf ? buf : (r.src_peer >= 0 ? peers.p[r.src_peer] : src);
    double2 w2[kCopyItems];
#pragma unroll
    for (int u = 0; u < kCopyItems; ++u) {
      const int64_t loc = (int64_t)bl.y + u * kCopyThreads + threadIdx.x;
      dofs[u] = -1;
      if (loc < end) {
        int64_t so, dof;
        rec_pair(r, loc, units, ncomp, so, dof);
        dofs[u] = dof;
        if (aligned) {
          w2[u] = *reinterpret_cast<const double2*>(s + so);
        } else {  // a base pointer off 16 bytes: same pairs, scalar accesses
          w2[u].x = s[so];
          w2[u].y = s[so + 1];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kCopyItems; ++u) {
      if (dofs[u] < 0) continue;
      double* q = dst + dofs[u];
      double2 o = w2[u];
      if (kAdd) {
        o.x = q[0] + o.x;
        o.y = q[1] + o.y;
      }
      if (aligned) {
        *reinterpret_cast<double2*>(q) = o;
      } else {
        q[0] = o.x;
        q[1] = o.y;
      }
    }
  } else if (bl.x >= 0) {  // one large record, chunk starting at flat index bl.y
    const DevRec r = recs[bl.x];
    const int64_t cells = (int64_t)r.e0 * r.e1 * r.e2;
    const int64_t end = min(cells * ncomp, (int64_t)bl.y + kChunk);
    const double* s = r.from_buf ? buf : (r.src_peer >= 0 ? peers.p[r.src_peer] : src);
#pragma unroll
    for (int u = 0; u < kCopyItems; ++u) {
      const int64_t loc = (int64_t)bl.y + u * kCopyThreads + threadIdx.x;
      dofs[u] = -1;
      if (loc < end) {
        int64_t so, dof;
        rec_cell(r, loc, cells, ncomp, so, dof);
        dofs[u] = dof;
        v[u] = s[so];
      }
    }
  } else {  // records -bl.x-1 .. -bl.x-1+bl.y-1, packed
    __shared__ int64_t beg[kPackMax + 1];
    const int r0 = -bl.x - 1, cnt = bl.y;
    const int64_t base = recs[r0].begin;
    for (int q = threadIdx.x; q < cnt; q += kCopyThreads) beg[q] = recs[r0 + q].begin - base;
    if (threadIdx.x == 0) {
      const DevRec& last = recs[r0 + cnt - 1];
      beg[cnt] = last.begin - base + (int64_t)last.e0 * last.e1 * last.e2 * ncomp;
    }
    __syncthreads();
    const int64_t total = beg[cnt];
#pragma unroll
    for (int u = 0; u < kCopyItems; ++u) {
      const int64_t loc = (int64_t)u * kCopyThreads + threadIdx.x;
      dofs[u] = -1;
      if (loc < total) {
        int lo = 0, hi = cnt - 1;  // last q with beg[q] <= loc
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (beg[mid] <= loc)
            lo = mid;
          else
            hi = mid - 1;
        }
        const DevRec& r = recs[r0 + lo];
        const int64_t cells = (int64_t)r.e0 * r.e1 * r.e2;
        const double* s = r.from_buf ? buf : (r.src_peer >= 0 ? peers.p[r.src_peer] : src);
        int64_t so, dof;
        rec_cell(r, loc - beg[lo], cells, ncomp, so, dof);
        dofs[u] = dof;
        v[u] = s[so];
      }
    }
  }
#pragma unroll
  for (int u = 0; u < kCopyItems && !paired; ++u) {
    if (dofs[u] < 0) continue;
    if (kAdd)
      dst[dofs[u]] = dst[dofs[u]] + v[u];
    else
      dst[dofs[u]] = v[u];
  }
  if (sy.on && threadIdx.x == 0 && atomicAdd(sy.epoch + 1, 1u) == gridDim.x - 1) {
    sy.epoch[0] = ep;  // every CTA has read the old epoch by now
    sy.epoch[1] = 0;
  }
}

struct Peer {
  int rank;
  int64_t off, count;  // elements
};

}  // namespace

struct Prog {
  int ncomp = 1;
  int op = 0;
  int sim = 1;
  int my_rank = 0;
  Wave pack;                // source fab -> send buffer
  std::vector<Wave*> apply;  // destination fab <- source fab / receive buffer
  int local_waves = 0;      // copy programs: apply[0] is local-only
  std::vector<Peer> sends, recvs;
  int64_t send_elems = 0, recv_elems = 0;
  std::vector<int64_t> pair_table;  // src, dst, off, count
  int64_t local_records = 0;
  ~Prog() {
    for (auto* w : apply) delete w;
  }
};

namespace {

struct Tab {
  const int64_t* t;
  int64_t at(int box, int w) const { return t[(int64_t)box * AMRB_FABTAB_W + w]; }
};

// Element offset of cell `lo` (3-D) in box `b` of a fab table, comp 0.
int64_t cell_offset(const Tab& tab, int b, const int lo[3]) {
  return tab.at(b, 0) + (lo[0] - tab.at(b, 4)) * tab.at(b, 2) + (lo[1] - tab.at(b, 5)) * tab.at(b, 3) +
         (lo[2] - tab.at(b, 6));
}

void prepare_wave(Wave& w, int ncomp) {
  w.total = 0;
  w.blocks.clear();
  int pack0 = -1, packn = 0;  // open run of small records
  int64_t packc = 0;
  auto close_pack = [&] {
    if (packn) w.blocks.push_back(make_int2(-pack0 - 1, packn));
    pack0 = -1;
    packn = 0;
    packc = 0;
  };
  for (size_t i = 0; i < w.host.size(); ++i) {
    DevRec& r = w.host[i];
    const int64_t n = (int64_t)r.e0 * r.e1 * r.e2 * ncomp;
    r.begin = w.total;
    w.total += n;
    if (n >= kSmall) {
      close_pack();  // packs hold consecutive records only
      // 16-byte pairs when every row starts 16-byte aligned on both sides
      // (allocations are 256-byte aligned; offsets and strides in elements)
      auto even = [](int64_t x) { return (x & 1) == 0; };
      r.vec = even(r.e2) && even(r.src) && even(r.dst) && even(r.ss0) && even(r.ss1) && even(r.ds0) &&
              even(r.ds1) && (ncomp == 1 || (even(r.scs) && even(r.dcs)));
      const int64_t units = r.vec ? n / 2 : n;
      for (int64_t o = 0; o < units; o += kChunk) w.blocks.push_back(make_int2((int)i, (int)o));
      continue;
    }
    if (packn && (packc + n > kChunk || packn == kPackMax)) close_pack();
    if (!packn) pack0 = (int)i;
    ++packn;
    packc += n;
  }
  close_pack();
  w.recs.upload(w.host);
  w.dblocks.upload(w.blocks);
}

bool run_wave(const Wave& w, int ncomp, bool add, const double* src, const double* buf, double* dst,
              cudaStream_t st, const PeerPtrs& peers = PeerPtrs{}, const SyncArgs& sy = SyncArgs{}) {
  if (w.blocks.empty()) return false;
  const unsigned nb = (unsigned)w.blocks.size();
  // 16-byte accesses for the pair records need every base 16-byte aligned
  uintptr_t bases = reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(buf) |
                    reinterpret_cast<uintptr_t>(dst);
  for (int r = 0; r < kMaxPeers; ++r) bases |= reinterpret_cast<uintptr_t>(peers.p[r]);
  const int aligned = (bases & 15) == 0;
  if (add)
    launch_k(k_copy<true>, nb, kCopyThreads, 0, st, w.recs.p, w.dblocks.p, ncomp, aligned, src, buf, dst, peers, sy);
  else
    launch_k(k_copy<false>, nb, kCopyThreads, 0, st, w.recs.p, w.dblocks.p, ncomp, aligned, src, buf, dst, peers, sy);
  check_launch("k_copy");
  return true;
}

bool overlaps(const Record& a, const Record& b) {
  for (int x = 0; x < 3; ++x) {
    int alo = a.lo[x] + a.shift[x], ahi = a.hi[x] + a.shift[x];
    int blo = b.lo[x] + b.shift[x], bhi = b.hi[x] + b.shift[x];
    if (ahi < blo || bhi < alo) return false;
  }
  return true;
}

}  // namespace
}  // namespace amrb

using amrb::Error;

extern "C" int amrb_prog_create(const amrb_plan* plan_, int ncomp, const int64_t* src_fabtab, int nsrc,
                                const int32_t* src_owner, const int64_t* dst_fabtab, int ndst,
                                const int32_t* dst_owner, int nranks, int my_rank, int mode, int op,
                                amrb_prog** out) {
  return amrb::guarded([&] {
    using namespace amrb;
    if (!plan_ || !out || ncomp < 1 || nranks < 1 || my_rank < 0 || my_rank >= nranks || op < 0 || op > 2 ||
        (op == 2 && mode != 3) ||
        mode < 0 || mode > 3 || (mode == 3 && nranks > kMaxPeers))
      throw Error(AMRB_EINVAL, "amrb_prog_create: bad arguments");
    const int sim_ranks = mode == 1;
    const bool local_only = mode == 2;
    const bool p2p = mode == 3;  // src_fabtab = each box's layout in its OWNER's storage
    // op 2: copy only the records whose source is resident here (p2p: the
    // local half of a fill whose remote half the producing kernel pushed)
    const bool local_src = op == 2;
    if (local_src) op = 0;
    const Plan& plan = *reinterpret_cast<const Plan*>(plan_);
    Tab st{src_fabtab}, dt{dst_fabtab};
    auto* g = new Prog;
    std::unique_ptr<Prog> guard(g);
    g->ncomp = ncomp;
    g->op = op;
    g->sim = sim_ranks;
    g->my_rank = my_rank;

    const auto& recs = plan.recs;
    const int64_t n = (int64_t)recs.size();
    std::vector<int> sr(n), dr(n);
    for (int64_t r = 0; r < n; ++r) {
      if (recs[r].src < 0 || recs[r].src >= nsrc || recs[r].dst < 0 || recs[r].dst >= ndst)
        throw Error(AMRB_EINVAL, "plan record box index out of range for the given layouts");
      sr[r] = src_owner ? src_owner[recs[r].src] : 0;
      dr[r] = dst_owner ? dst_owner[recs[r].dst] : 0;
      if (sr[r] < 0 || sr[r] >= nranks || dr[r] < 0 || dr[r] >= nranks)
        throw Error(AMRB_EINVAL, "owner rank out of range");
      if (local_only && !(sr[r] == my_rank && dr[r] == my_rank)) sr[r] = dr[r] = -1;  // dropped
      if (local_src && sr[r] != my_rank) sr[r] = dr[r] = -1;
    }
    // ---- message segments: ordered (src, dst) pairs, plan order inside ------
    // buffer offset of each remote record (elements)
    std::vector<int64_t> buf_off(n, -1);
    {
      std::map<std::pair<int, int>, std::vector<int64_t>> pairs;
      for (int64_t r = 0; r < n; ++r)
        if (!p2p && sr[r] >= 0 && sr[r] != dr[r] && (sim_ranks || sr[r] == my_rank || dr[r] == my_rank))
          pairs[{sr[r], dr[r]}].push_back(r);
      // sim: one staging buffer holding every pair; dist: separate send/recv
      int64_t soff = 0, roff = 0;
      for (auto& kv : pairs) {
        int s = kv.first.first, d = kv.first.second;
        int64_t cnt = 0;
        for (int64_t r : kv.second) cnt += recs[r].cells() * ncomp;
        if (sim_ranks) {
          int64_t o = soff;
          for (int64_t r : kv.second) {
            buf_off[r] = o;
            o += recs[r].cells() * ncomp;
          }
          g->pair_table.insert(g->pair_table.end(), {s, d, soff, cnt});
          soff += cnt;
        } else if (s == my_rank) {
          int64_t o = soff;
          for (int64_t r : kv.second) {
            buf_off[r] = o;
            o += recs[r].cells() * ncomp;
          }
          g->sends.push_back({d, soff, cnt});
          g->pair_table.insert(g->pair_table.end(), {s, d, soff, cnt});
          soff += cnt;
        } else {  // d == my_rank
          int64_t o = roff;
          for (int64_t r : kv.second) {
            buf_off[r] = o;
            o += recs[r].cells() * ncomp;
          }
          g->recvs.push_back({s, roff, cnt});
          roff += cnt;
        }
      }
      g->send_elems = soff;
      g->recv_elems = sim_ranks ? soff : roff;
    }
    auto fab_side = [&](const Tab& t, int box, const int lo[3], int64_t& off, int64_t& s0, int64_t& s1,
                        int64_t& cs) {
      if (!t.at(box, 7)) throw Error(AMRB_EINVAL, "record touches a box that is not resident here");
      off = cell_offset(t, box, lo);
      s0 = t.at(box, 2);
      s1 = t.at(box, 3);
      cs = t.at(box, 1);
    };
    auto buf_side = [&](int64_t r, int64_t& off, int64_t& s0, int64_t& s1, int64_t& cs) {
      const Record& q = recs[r];
      int e1 = q.hi[1] - q.lo[1] + 1, e2 = q.hi[2] - q.lo[2] + 1;
      off = buf_off[r];
      s1 = e2;
      s0 = (int64_t)e1 * e2;
      cs = q.cells();
    };
    // ---- pack ---------------------------------------------------------------
    for (int64_t r = 0; r < n && !p2p; ++r) {
      if (sr[r] == dr[r] || buf_off[r] < 0) continue;
      if (!sim_ranks && sr[r] != my_rank) continue;
      const Record& q = recs[r];
      DevRec d{};
      d.e0 = q.hi[0] - q.lo[0] + 1;
      d.e1 = q.hi[1] - q.lo[1] + 1;
      d.e2 = q.hi[2] - q.lo[2] + 1;
      fab_side(st, q.src, q.lo, d.src, d.ss0, d.ss1, d.scs);
      buf_side(r, d.dst, d.ds0, d.ds1, d.dcs);
      g->pack.host.push_back(d);
    }
    // ---- apply ---------------------------------------------------------------
    std::vector<int64_t> mine;
    for (int64_t r = 0; r < n; ++r)
      if (sr[r] >= 0 && (sim_ranks || dr[r] == my_rank)) mine.push_back(r);
    auto make_apply = [&](int64_t r) {
      const Record& q = recs[r];
      DevRec d{};
      d.e0 = q.hi[0] - q.lo[0] + 1;
      d.e1 = q.hi[1] - q.lo[1] + 1;
      d.e2 = q.hi[2] - q.lo[2] + 1;
      int dlo[3] = {q.lo[0] + q.shift[0], q.lo[1] + q.shift[1], q.lo[2] + q.shift[2]};
      fab_side(dt, q.dst, dlo, d.dst, d.ds0, d.ds1, d.dcs);
      d.src_peer = -1;
      if (sr[r] == dr[r]) {
        fab_side(st, q.src, q.lo, d.src, d.ss0, d.ss1, d.scs);
        d.from_buf = 0;
      } else if (p2p) {
        // the global table holds the owner's layout for every box
        fab_side(st, q.src, q.lo, d.src, d.ss0, d.ss1, d.scs);
        d.from_buf = 0;
        d.src_peer = sr[r];
      } else {
        buf_side(r, d.src, d.ss0, d.ss1, d.scs);
        d.from_buf = 1;
      }
      return d;
    };
    if (op == 0 && p2p) {
      // one wave: a copy's records never share a destination cell, and in
      // the pull model nothing waits for a receive buffer -- the CTAs reading
      // a peer wait for the fused barrier while the local ones run (k_copy).
      // Peer records first, so their CTAs are scheduled (and start waiting)
      // first.
      auto* w = new Wave;
      g->apply.push_back(w);
      for (int pass = 0; pass < 2; ++pass)
        for (int64_t r : mine)
          if ((sr[r] == dr[r]) == (pass == 1)) w->host.push_back(make_apply(r));
      for (int64_t r : mine)
        if (sr[r] == dr[r]) g->local_records++;
      g->local_waves = 0;
    } else if (op == 0) {
      auto* local = new Wave;
      auto* remote = new Wave;
      g->apply.push_back(local);
      g->apply.push_back(remote);
      for (int64_t r : mine) {
        (sr[r] == dr[r] ? local : remote)->host.push_back(make_apply(r));
        if (sr[r] == dr[r]) g->local_records++;
      }
      g->local_waves = 1;
    } else {
      // wave(r) = 1 + max wave of earlier records into the same box that overlap
      std::map<int, std::vector<std::pair<int64_t, int>>> by_dst;
      int nw = 0;
      std::vector<int> wave_of(mine.size());
      for (size_t m = 0; m < mine.size(); ++m) {
        int64_t r = mine[m];
        int w = 0;
        for (auto& pr : by_dst[recs[r].dst])
          if (overlaps(recs[pr.first], recs[r])) w = std::max(w, pr.second + 1);
        by_dst[recs[r].dst].push_back({r, w});
        wave_of[m] = w;
        nw = std::max(nw, w + 1);
        if (sr[r] == dr[r]) g->local_records++;
      }
      for (int w = 0; w < nw; ++w) g->apply.push_back(new Wave);
      for (size_t m = 0; m < mine.size(); ++m) g->apply[wave_of[m]]->host.push_back(make_apply(mine[m]));
      g->local_waves = 0;
    }
    prepare_wave(g->pack, ncomp);
    for (auto* w : g->apply) prepare_wave(*w, ncomp);
    *out = reinterpret_cast<amrb_prog*>(guard.release());
  });
}

extern "C" int amrb_prog_info(const amrb_prog* g_, int64_t* send_elems, int64_t* recv_elems, int64_t* npairs,
                              int64_t* local_records) {
  return amrb::guarded([&] {
    if (!g_) throw Error(AMRB_EINVAL, "null program");
    auto* g = reinterpret_cast<const amrb::Prog*>(g_);
    if (send_elems) *send_elems = g->send_elems;
    if (recv_elems) *recv_elems = g->recv_elems;
    if (npairs) *npairs = (int64_t)g->pair_table.size() / 4;
    if (local_records) *local_records = g->local_records;
  });
}

extern "C" int amrb_prog_pairs(const amrb_prog* g_, int64_t* out) {
  return amrb::guarded([&] {
    if (!g_ || !out) throw Error(AMRB_EINVAL, "null argument");
    auto* g = reinterpret_cast<const amrb::Prog*>(g_);
    std::memcpy(out, g->pair_table.data(), g->pair_table.size() * sizeof(int64_t));
  });
}

extern "C" int amrb_prog_run(amrb_prog* g_, const double* src_base, double* dst_base, double* sendbuf,
                             double* recvbuf, void* nccl_comm, void* stream) {
  return amrb::guarded([&] {
    using namespace amrb;
    if (!g_) throw Error(AMRB_EINVAL, "null program");
    auto* g = reinterpret_cast<Prog*>(g_);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if ((g->send_elems && !sendbuf) || (g->recv_elems && !g->sim && !recvbuf))
      throw Error(AMRB_EINVAL, "missing staging buffer");
    const double* rbuf = g->sim ? sendbuf : recvbuf;
    run_wave(g->pack, g->ncomp, false, src_base, nullptr, sendbuf, st);
    if (!g->sim && (!g->sends.empty() || !g->recvs.empty())) {
      if (!nccl_comm) throw Error(AMRB_ENCCL, "remote records but no NCCL communicator");
      ncclComm_t comm = reinterpret_cast<ncclComm_t>(nccl_comm);
      auto nc = [](ncclResult_t r, const char* what) {
        if (r != ncclSuccess) throw Error(AMRB_ENCCL, std::string(what) + ": " + ncclGetErrorString(r));
      };
      nc(ncclGroupStart(), "ncclGroupStart");
      for (const auto& p : g->sends)
        nc(ncclSend(sendbuf + p.off, (size_t)p.count, ncclFloat64, p.rank, comm, st), "ncclSend");
      for (const auto& p : g->recvs)
        nc(ncclRecv(recvbuf + p.off, (size_t)p.count, ncclFloat64, p.rank, comm, st), "ncclRecv");
      nc(ncclGroupEnd(), "ncclGroupEnd");
    }
    for (auto* w : g->apply) run_wave(*w, g->ncomp, g->op == 1, src_base, rbuf, dst_base, st);
  });
}

extern "C" int amrb_prog_destroy(amrb_prog* g) {
  delete reinterpret_cast<amrb::Prog*>(g);
  return AMRB_OK;
}


extern "C" int amrb_peer_barrier(const uint64_t* pad_ptrs, int rank, int nranks, uint32_t* epoch, void* stream);

extern "C" int amrb_prog_run_p2p_sync(amrb_prog* g_, const double* src_base, double* dst_base,
                                      const uint64_t* peer_bases, int npeers, const uint64_t* pad_ptrs, int rank,
                                      uint32_t* epoch, void* stream) {
  int status = amrb::guarded([&] {
    using namespace amrb;
    if (!g_ || npeers < 1 || npeers > kMaxPeers || !peer_bases || !pad_ptrs || rank < 0 || rank >= npeers || !epoch)
      throw Error(AMRB_EINVAL, "amrb_prog_run_p2p_sync: bad arguments");
    auto* g = reinterpret_cast<Prog*>(g_);
    PeerPtrs peers{};
    SyncArgs sy{};
    for (int r = 0; r < npeers; ++r) {
      peers.p[r] = reinterpret_cast<const double*>(peer_bases[r]);
      sy.pads[r] = reinterpret_cast<uint32_t*>(pad_ptrs[r]);
    }
    sy.epoch = epoch;
    sy.rank = rank;
    sy.nranks = npeers;
    sy.on = 1;
    sy.fault = current_fault();
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    bool synced = false;
    for (auto* w : g->apply) {
      if (run_wave(*w, g->ncomp, g->op == 1, src_base, nullptr, dst_base, st, peers, synced ? SyncArgs{} : sy))
        synced = true;
    }
    // nothing to copy here: the peers still wait for this rank's epoch
    if (!synced && amrb_peer_barrier(pad_ptrs, rank, npeers, epoch, stream) != AMRB_OK)
      throw Error(AMRB_ECUDA, "amrb_prog_run_p2p_sync: barrier launch failed");
  });
  return status;
}

extern "C" int amrb_prog_run_p2p(amrb_prog* g_, const double* src_base, double* dst_base, const uint64_t* peer_bases,
                                 int npeers, void* stream) {
  return amrb::guarded([&] {
    using namespace amrb;
    if (!g_ || npeers < 1 || npeers > kMaxPeers || !peer_bases) throw Error(AMRB_EINVAL, "amrb_prog_run_p2p: bad arguments");
    auto* g = reinterpret_cast<Prog*>(g_);
    PeerPtrs peers{};
    for (int r = 0; r < npeers; ++r) peers.p[r] = reinterpret_cast<const double*>(peer_bases[r]);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    for (auto* w : g->apply) run_wave(*w, g->ncomp, g->op == 1, src_base, nullptr, dst_base, st, peers);
  });
}

namespace {
struct PadPtrs {
  uint32_t* p[amrb::kMaxPeers];
};

// Device-side barrier over NVLink: bump a device epoch counter, publish it in
// every peer's signal pad (slot = my rank), wait until every peer published it
// in mine.  The epoch lives in device memory, so a captured graph replays
// correctly; the wrap-safe compare allows 2^31 outstanding epochs.
__global__ void k_peer_barrier(uint32_t* my_pad, PadPtrs pads, int rank, int nranks, uint32_t* epoch,
                               amrb::Fault fault) {
  amrb::pdl_entry();
  // one warp; lane p publishes to and polls peer p concurrently
  const int p = threadIdx.x;
  const uint32_t e = *reinterpret_cast<volatile uint32_t*>(epoch) + 1;
  __syncwarp();
  if (p < nranks && p != rank) {
    amrb::signal_store(pads.p[p] + rank, e);
    amrb::peer_wait(my_pad + p, e, rank, p, fault);
  }
  __syncwarp();
  if (p == 0) *epoch = e;
}
}  // namespace

extern "C" int amrb_set_fault_mailbox(void* pinned_host) {
  return amrb::guarded([&] {
    if (pinned_host && !amrb::g_fault_dev) {
      void* d = nullptr;
      AMRB_CUDA(cudaMalloc(&d, sizeof(unsigned long long)));
      AMRB_CUDA(cudaMemset(d, 0, sizeof(unsigned long long)));
      AMRB_CUDA(cudaDeviceSynchronize());
      amrb::g_fault_dev = reinterpret_cast<unsigned long long*>(d);
    }
    amrb::g_fault_box = reinterpret_cast<unsigned long long*>(pinned_host);
  });
}

extern "C" int amrb_peer_barrier(const uint64_t* pad_ptrs, int rank, int nranks, uint32_t* epoch, void* stream) {
  return amrb::guarded([&] {
    using namespace amrb;
    if (!pad_ptrs || nranks < 1 || nranks > kMaxPeers || rank < 0 || rank >= nranks || !epoch)
      throw Error(AMRB_EINVAL, "amrb_peer_barrier: bad arguments");
    PadPtrs pads{};
    for (int r = 0; r < nranks; ++r) pads.p[r] = reinterpret_cast<uint32_t*>(pad_ptrs[r]);
    launch_k(k_peer_barrier, 1, 32, 0, reinterpret_cast<cudaStream_t>(stream), pads.p[rank], pads, rank, nranks, epoch,
             current_fault());
    check_launch("k_peer_barrier");
  });
}


using amrb::PeerPtrs;
namespace {
// Max-all-reduce of one double over NVLink, as tagged words (no flag, no
// fence on the data): rank r stores its value into slot r of every peer's
// symmetric buffer as two 64-bit words (epoch << 32 | low half, epoch << 32 |
// high half) -- each store single-copy atomic -- and each rank polls its own
// slots until both words of every peer carry this epoch.  Arriving there also
// means every peer finished the kernels before this one (the gpu-scope fence
// before the stores orders them), so the call doubles as the device barrier.
__global__ void k_peer_allmax(PadPtrs pads, amrb::Fault fault, int rank, int nranks, uint32_t* epoch, double* val,
                              unsigned long long* my_slots, PeerPtrs peer_slots) {
  amrb::pdl_entry();
  (void)pads;
  // one warp; lane p serves peer p (stores, poll) concurrently
  const int p = threadIdx.x;
  const double v = *val;
  const uint32_t e = *reinterpret_cast<volatile uint32_t*>(epoch) + 1;
  const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
  const unsigned long long tag = (unsigned long long)e << 32;
  double got = v;
  __syncwarp();
  if (p < nranks && p != rank) {
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(const_cast<double*>(peer_slots.p[p])) + 2 * rank;
    asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;\n" ::"l"(dst), "l"(tag | (bits & 0xffffffffull)) : "memory");
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;\n" ::"l"(dst + 1), "l"(tag | (bits >> 32)) : "memory");
    const unsigned long long* src = my_slots + 2 * p;
    const unsigned long long t0 = amrb::global_ns();
    bool dead = amrb::faulted(fault);
    for (unsigned it = 0; !dead; ++it) {
      unsigned long long lo, hi;
      asm volatile("ld.relaxed.sys.global.u64 %0, [%1];\n" : "=l"(lo) : "l"(src) : "memory");
      asm volatile("ld.relaxed.sys.global.u64 %0, [%1];\n" : "=l"(hi) : "l"(src + 1) : "memory");
      if ((uint32_t)(lo >> 32) == e && (uint32_t)(hi >> 32) == e) {
        got = __longlong_as_double((long long)((hi << 32) | (lo & 0xffffffffull)));
        break;
      }
      if ((it & 255) == 255 && fault.timeout_ns && amrb::global_ns() - t0 > fault.timeout_ns) {
        amrb::record_fault(fault, rank, p, e);
        dead = true;
      }
    }
    asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
  }
  // max over lanes on the bit patterns: the operands are norms (>= 0), which
  // order like their bits, and a NaN (above +inf) on any rank wins -- a
  // diverged rank cannot look converged
  unsigned long long gb = (unsigned long long)__double_as_longlong(got);
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long x = __shfl_xor_sync(0xffffffffu, gb, o);
    gb = x > gb ? x : gb;
  }
  if (p == 0) {
    *epoch = e;
    *val = __longlong_as_double((long long)gb);
  }
}
}  // namespace

extern "C" int amrb_peer_allmax(const uint64_t* pad_ptrs, const uint64_t* slot_ptrs, int rank, int nranks,
                                uint32_t* epoch, double* val, void* stream) {
  return amrb::guarded([&] {
    using namespace amrb;
    if (!pad_ptrs || !slot_ptrs || nranks < 1 || nranks > kMaxPeers || rank < 0 || rank >= nranks || !epoch || !val)
      throw Error(AMRB_EINVAL, "amrb_peer_allmax: bad arguments");
    PadPtrs pads{};
    PeerPtrs slots{};
    for (int r = 0; r < nranks; ++r) {
      pads.p[r] = reinterpret_cast<uint32_t*>(pad_ptrs[r]);
      slots.p[r] = reinterpret_cast<const double*>(slot_ptrs[r]);
    }
    launch_k(k_peer_allmax, 1, 32, 0, reinterpret_cast<cudaStream_t>(stream), pads, current_fault(), rank, nranks,
             epoch, val, reinterpret_cast<unsigned long long*>(const_cast<double*>(slots.p[rank])), slots);
    check_launch("k_peer_allmax");
  });
}

// ----------------------------------------------------------------------------
// NCCL plumbing
// ----------------------------------------------------------------------------
namespace {
void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Error(AMRB_ENCCL, std::string(what) + ": " + ncclGetErrorString(r));
}
}  // namespace

extern "C" int amrb_nccl_unique_id(uint8_t* out128) {
  return amrb::guarded([&] {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    nccl_check(ncclGetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out128, &id, 128);
  });
}

extern "C" int amrb_nccl_comm_create(const uint8_t* id128, int nranks, int rank, void** comm) {
  return amrb::guarded([&] {
    ncclUniqueId id;
    std::memcpy(&id, id128, 128);
    ncclComm_t c;
    nccl_check(ncclCommInitRank(&c, nranks, id, rank), "ncclCommInitRank");
    *comm = c;
  });
}

extern "C" int amrb_nccl_comm_destroy(void* comm) {
  return amrb::guarded([&] {
    if (comm) nccl_check(ncclCommDestroy(reinterpret_cast<ncclComm_t>(comm)), "ncclCommDestroy");
  });
}

extern "C" int amrb_nccl_allreduce(double* buf, int64_t n, int op, void* comm, void* stream) {
  return amrb::guarded([&] {
    ncclRedOp_t o = op == 0 ? ncclSum : op == 1 ? ncclMin : ncclMax;
    nccl_check(ncclAllReduce(buf, buf, (size_t)n, ncclFloat64, o, reinterpret_cast<ncclComm_t>(comm),
                             reinterpret_cast<cudaStream_t>(stream)),
               "ncclAllReduce");
  });
}

extern "C" int amrb_nccl_allgather(const double* send, double* recv, int64_t n, void* comm, void* stream) {
  return amrb::guarded([&] {
    nccl_check(ncclAllGather(send, recv, (size_t)n, ncclFloat64, reinterpret_cast<ncclComm_t>(comm),
                             reinterpret_cast<cudaStream_t>(stream)),
               "ncclAllGather");
  });
}
