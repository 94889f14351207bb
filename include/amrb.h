/*
 * amrb.h -- C ABI of libamrb.so, the B200 (sm_100a) MultiFab / FillBoundary /
 * MLMG hot path.
 *
 * The reference (/root/reference/pkg, package `amrkit`) is pure Python and has
 * no FFI; its drop-in surface is the module API.  Each entry point below names
 * the reference function whose work it takes over; the Python layer in
 * paper_2009_12009_b200/ keeps the reference's signatures and calls these
 * through ctypes.
 *
 * Conventions
 *   - every call returns AMRB_OK (0) or a negative status; amrb_last_error()
 *     gives a thread-local message.  The Python wrapper maps AMRB_EINVAL to
 *     ValueError, AMRB_ENCCL to TransportError(src, dst, why) and AMRB_ECUDA to
 *     RuntimeError.
 *   - plain pointers and sizes only; device buffers are owned by the caller
 *     (PyTorch).  Plans and programs own their host/device descriptor tables.
 *   - `stream` is a cudaStream_t passed as void*; every device call is
 *     asynchronous on it.  `nccl_comm` is an ncclComm_t passed as void*.
 *   - All boxes are described in 3-D: a D-dimensional box's axis d maps to
 *     axis (3 - D + d); padding axes have lo = hi = 0.  Storage is C-order
 *     (comp, i, j, k) with k unit-stride, like the reference's Fab
 *     (fabarray.py:33-38), but every k-row is padded so valid rows start on a
 *     32-byte sector.
 *
 * Fab table ("fabtab"): int64[nboxes][AMRB_FABTAB_W] describing one
 * FabArray's storage on one device:
 *     [0] element offset of the grown box's lo cell, comp 0
 *     [1] comp stride   [2] axis-0 stride   [3] axis-1 stride  (axis-2 stride 1)
 *     [4..6] grown-box lo (3-D padded)
 *     [7] 1 if the box is resident on this device, else 0
 */
#ifndef AMRB_H
#define AMRB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AMRB_OK 0
#define AMRB_EINVAL (-1)
#define AMRB_ECUDA (-2)
#define AMRB_ENCCL (-3)
#define AMRB_ENOMEM (-4)
#define AMRB_ENOTSUP (-5) /* valid request this fast path does not cover (caller falls back) */

#define AMRB_FABTAB_W 8
#define AMRB_REC_W 11 /* src, dst, src_lo[3], src_hi[3], shift[3] (3-D padded) */

const char* amrb_last_error(void);
int amrb_version(void);
/* Kernel launches issued so far by this process (host-side count; launches
 * replayed from a captured CUDA graph are not included). */
int64_t amrb_launch_count(void);
/* Device-side solve loop (csrc/graph.cu): a CUDA graph whose WHILE node
 * repeats a captured body until its control kernel says stop.  Between
 * amrb_loop_begin and amrb_loop_end every launch on `stream` is captured into
 * the body; the body must end with amrb_loop_control, which appends *norm to
 * the state block's history, zeroes *norm, counts the iteration and
 * continues while !(norm <= rtol * *r0) and iters < max_iter (the oracle's
 * stopping test, oracle/mlmg_ref.py OracleMLMG.solve).  state: DEVICE memory
 * {double rtol; int32 max_iter; int32 iters; double r0; double
 * hist[capacity]}; amrb_loop_reset fills rtol / max_iter / r0 and zeroes
 * iters (a kernel, on the launch stream) before amrb_loop_launch; afterwards
 * move it to the host (amrb_store_host) and read iters / hist.  Nothing in
 * the loop touches host memory, so it does not wait behind bulk PCIe copies
 * running on other streams. */
typedef struct amrb_loop amrb_loop;
int amrb_loop_begin(void* stream, amrb_loop** out);
int amrb_loop_reset(void* state, double rtol, int max_iter, const double* r0, void* stream);
int amrb_loop_control(amrb_loop* loop, double* norm, const double* r0, void* state, int capacity,
                      void* stream);
int amrb_loop_end(amrb_loop* loop);
int amrb_loop_launch(amrb_loop* loop, void* stream);
int amrb_loop_destroy(amrb_loop* loop);

/* Checked builds (make CHECKED=1 -> libamrb_checked.so): number of failed
 * device-side invariant checks since the last reset and the source line of
 * the first; *failures = -1 in the normal build. */
int amrb_debug_checks(int64_t* failures, int64_t* line, int reset);

/* Library options: process-wide, set explicitly by the caller (the library
 * reads no environment variables).  Names and defaults:
 *   "pdl"          2  programmatic dependent launch: 0 off, 1 always, 2 eager
 *                     launches only (not inside stream capture)
 *   "sweep_kernel" 0  fused GSRB sweep: 0 k_gsrb_stream wherever the layout
 *                     allows it, 1 the previous TMA kernels (A/B runs)
 *   "grid_per_sm"  0  CTAs per SM of the grid-synchronised level kernel
 *                     (0: the occupancy maximum)
 *   "stream_segments"  0  plane segments per tile column of k_gsrb_stream
 *                     (0: enough for one wave of CTAs)
 *   "stream_alternate" 1  odd segments stream downward (L2 halo sharing)
 *   "stream_config"    0  k_gsrb_stream tile / strip / depth variant (A/B runs)
 *   "peer_timeout_ms" 30000  bound on every device-side wait for a peer
 *                     (NVLink signal pads); 0 waits forever
 *   "push_fence"   0  1: a ghost-pushing sweep ends with a system-scope
 *                     fence (A/B runs; the consumer's barrier is signalled
 *                     by a later kernel, after this one's stores completed)
 * AMRB_EINVAL for an unknown name. */
int amrb_set_option(const char* name, int64_t value);
int amrb_get_option(const char* name, int64_t* value);
/* ptr[0..n) = value (one kernel). */
int amrb_fill(double* ptr, int64_t n, double value, void* stream);
/* Zero n doubles (cudaMemsetAsync on `stream`; a memset node in a graph). */
int amrb_zero(double* ptr, int64_t n, void* stream);
/* host_dst[0..n) <- src (device) by a kernel storing through UVA into pinned
 * host memory: small results reach the host without a copy-engine transfer
 * (which would queue behind bulk copies).  Synchronize the stream to read. */
int amrb_store_host(const double* src, double* host_dst, int64_t n, void* stream);

/* ------------------------------------------------------------------------ */
/* Box -> rank assignment (host; distribution.py:19-148).  lohi = int32     */
/* [n][2*dim] (lo then hi per box).                                          */
/* ------------------------------------------------------------------------ */
/* morton_key: bit k of axis d of (point - origin) -> key bit k*dim + d. */
int amrb_morton_key(int dim, const int32_t* point, const int32_t* origin, uint64_t* key);
/* sfc_distribute (distribution.py:97-131): box centres (lo+hi)//2 in Morton
 * order, contiguous runs of ~equal cost; `total` = the caller's sum of cost. */
int amrb_sfc_distribute(int dim, int n, const int32_t* lohi, const double* cost, double total,
                        int nranks, int32_t* owner);
/* knapsack_distribute (distribution.py:134-148): longest processing time. */
int amrb_knapsack_distribute(int n, const double* cost, int nranks, int32_t* owner);

/* ------------------------------------------------------------------------ */
/* Communication plans (host).  Records are CopyRecord(src, dst, src_box,    */
/* dst_box = src_box + shift, shift) sorted by (dst, dst_box.lo, src, shift) */
/* -- the reference's CommPlan order (fabarray.py:169-197).                  */
/* ------------------------------------------------------------------------ */
typedef struct amrb_plan amrb_plan;

/* C++ twin of _build_fill (fabarray.py:262-277) incl. _periodic_shifts
 * (:235-243), box_diff slabs (index_space.py:320-345) and the BoxHash query
 * (boxarray.py:169-180, 216-278).  lohi: nboxes x 2*dim (lo then hi). */
int amrb_plan_fill_create(int dim, int nboxes, const int32_t* lohi, int ngrow,
                          const int32_t* domain_lohi, const uint8_t* periodic,
                          amrb_plan** out);

/* _build_copy (fabarray.py:291-302) when dst_ngrow == 0, and
 * build_plan_copy_grown (coarse_fine.py:201-220) otherwise.  domain_lohi may be
 * NULL (no periodic images). */
int amrb_plan_copy_create(int dim, int ndst, const int32_t* dst_lohi, int nsrc,
                          const int32_t* src_lohi, int dst_ngrow,
                          const int32_t* domain_lohi, const uint8_t* periodic,
                          amrb_plan** out);

/* Transpose of the fill plan (build_plan_sum_boundary, fabarray.py:305-318). */
int amrb_plan_sum_create(int dim, int nboxes, const int32_t* lohi, int ngrow,
                         const int32_t* domain_lohi, const uint8_t* periodic,
                         amrb_plan** out);

/* Number of records and total cells (one component). */
int amrb_plan_size(const amrb_plan* p, int64_t* nrecords, int64_t* ncells);
/* Export records: out = int32[nrecords][AMRB_REC_W] (parity checks). */
int amrb_plan_records(const amrb_plan* p, int32_t* out);
int amrb_plan_destroy(amrb_plan* p);

/* ------------------------------------------------------------------------ */
/* Copy programs (device): a plan bound to concrete storage.  Replaces the   */
/* two-phase executor _execute_plan (fabarray.py:326-361).                   */
/* mode 1 (sim): every rank's boxes live on this device (the reference's    */
/*     simulated ranks); remote records are packed into one staging buffer,  */
/*     one segment per ordered (src,dst) rank pair, and unpacked from it.    */
/* mode 0 (nccl): one process per GPU; this device is rank `my_rank`.        */
/*     Remote records ride one NCCL send/recv per ordered peer pair.         */
/* mode 2 (local): keep only records with src and dst owned by my_rank      */
/*     (copies between a distributed FabArray and a per-rank replica).      */
/* mode 3 (p2p): records with dst here; remote sources are read directly     */
/*     from the owner's storage over NVLink (src_fabtab = every box's layout */
/*     in its owner's allocation; see amrb_prog_run_p2p).                   */
/* op: 0 = dst = src (fill / parallel_copy), 1 = dst += src (sum_boundary;   */
/*     overlapping records are applied in plan order, in waves);            */
/*     2 = copy only the records whose SOURCE box is resident here (mode 3   */
/*     only: the local half of a fill whose remote half the producing sweep  */
/*     pushed over NVLink; run it with amrb_prog_run_p2p_sync, whose fused   */
/*     barrier then orders the peers' pushes before the consumer).           */
/* Message payloads are C-order (ncomp, e0, e1, e2) record slices           */
/* concatenated in plan order -- the reference's message layout (:341-347). */
/* ------------------------------------------------------------------------ */
typedef struct amrb_prog amrb_prog;

int amrb_prog_create(const amrb_plan* plan, int ncomp,
                     const int64_t* src_fabtab, int nsrc, const int32_t* src_owner,
                     const int64_t* dst_fabtab, int ndst, const int32_t* dst_owner,
                     int nranks, int my_rank, int mode, int op,
                     amrb_prog** out);
/* Elements of staging needed: send (and recv, which is the same buffer in
 * sim mode).  Per-pair message table: int64[npairs][4] = src_rank, dst_rank,
 * element offset, element count, in (src,dst) order. */
int amrb_prog_info(const amrb_prog* g, int64_t* send_elems, int64_t* recv_elems,
                   int64_t* npairs, int64_t* local_records);
int amrb_prog_pairs(const amrb_prog* g, int64_t* out);
int amrb_prog_run(amrb_prog* g, const double* src_base, double* dst_base,
                  double* sendbuf, double* recvbuf, void* nccl_comm, void* stream);
int amrb_prog_destroy(amrb_prog* g);
/* Run a mode-3 program: peer_bases[r] = rank r's storage base, mapped into
 * this process (symmetric memory).  Callers frame it with amrb_peer_barrier. */
int amrb_prog_run_p2p(amrb_prog* g, const double* src_base, double* dst_base,
                      const uint64_t* peer_bases, int npeers, void* stream);
/* amrb_peer_barrier + amrb_prog_run_p2p in one launch: the copy kernel's CTA
 * 0 publishes this rank's epoch, CTAs reading peer storage (and CTA 0) wait
 * for every peer's; local-source CTAs start at once.  epoch = uint32[2]
 * (epoch, completion ticket), shared with amrb_peer_barrier. */
int amrb_prog_run_p2p_sync(amrb_prog* g, const double* src_base, double* dst_base,
                           const uint64_t* peer_bases, int npeers, const uint64_t* pad_ptrs,
                           int rank, uint32_t* epoch, void* stream);
/* Device-side barrier across ranks over NVLink signal pads: pad_ptrs[r] =
 * rank r's pad (>= nranks uint32 slots), epoch = this rank's device counter. */
/* Failure detection: pinned host memory of 4 uint64 {code, rank, peer, epoch}
 * the device-side peer waits report into (code 1: a peer did not arrive within
 * the "peer_timeout_ms" option; later waits then return at once -- the
 * waits poll a device-memory twin of the code, never the host block).  The
 * caller zeroes it, and after synchronising raises TransportError(rank, peer)
 * when code != 0 (comm.py Transport.check_faults).  NULL disables reporting. */
int amrb_set_fault_mailbox(void* pinned_host);
int amrb_peer_barrier(const uint64_t* pad_ptrs, int rank, int nranks, uint32_t* epoch,
                      void* stream);
/* In-place max over ranks of one device double >= 0 over NVLink (one launch,
 * also a device barrier; NaN on any rank wins): slot_ptrs[r] = rank r's
 * symmetric buffer of >= 2 * nranks uint64 words, zeroed before first use
 * (epoch-tagged value halves; pad_ptrs is unused, kept for the signature).
 * Cross-GPU signalling uses gpu-scope fences only (see comm.cu): no
 * system-scope fence that would wait behind in-flight PCIe copies. */
int amrb_peer_allmax(const uint64_t* pad_ptrs, const uint64_t* slot_ptrs, int rank,
                     int nranks, uint32_t* epoch, double* val, void* stream);

/* ------------------------------------------------------------------------ */
/* Level descriptors for the ParallelFor box loop (advect.py:143-178 is the  */
/* reference's per-box loop pattern).  A level = one BoxArray on one device: */
/* per-box valid lo / extents (3-D padded) and, per operand, the fab table.  */
/* ------------------------------------------------------------------------ */
typedef struct amrb_level amrb_level;

/* boxes: int32[nboxes][6] valid lo, hi (3-D padded); resident: uint8[nboxes]
 * (1 = box on this device).  Builds the device tile tables. */
int amrb_level_create(int nboxes, const int32_t* boxes, const uint8_t* resident,
                      amrb_level** out);
int amrb_level_destroy(amrb_level* lv);

/* A bound operand: fab table for one FabArray on a level. */
typedef struct amrb_field amrb_field;
int amrb_field_create(const amrb_level* lv, const int64_t* fabtab, int ngrow,
                      amrb_field** out);
int amrb_field_destroy(amrb_field* f);

/* out = L(phi) on valid cells, 7-point, ((phi[-1] - 2 phi) + phi[+1]) * dh
 * per axis, summed x, y, z left to right.  phi ghosts (width 1) must be
 * filled.  dh = 1/dx^2 per axis. */
int amrb_lap_apply(const amrb_level* lv, amrb_field* out, double* out_base,
                   const amrb_field* phi, const double* phi_base,
                   const double dh[3], void* stream);

/* r = rhs - L(phi). */
int amrb_residual(const amrb_level* lv, amrb_field* r, double* r_base,
                  const amrb_field* rhs, const double* rhs_base,
                  const amrb_field* phi, const double* phi_base,
                  const double dh[3], void* stream);

/* One GSRB colour: cells with (i+j+k+color) % 2 == 0 (global indices) get
 * phi += (rhs - L(phi)) * rgamma, rgamma = 1 / (-2 (dh0+dh1+dh2)). */
int amrb_gsrb_color(const amrb_level* lv, amrb_field* phi, double* phi_base,
                    const amrb_field* rhs, const double* rhs_base,
                    const double dh[3], int color, void* stream);

/* One fused red+black sweep, out of place: b = GSRB(a) (bit-identical to
 * colour 0 then colour 1 in place with a width-1 fill in between).  Needs the
 * ghosts of `a` filled to width 2 and of `rhs` to width 1; the red update of
 * the first ghost ring is recomputed locally, so no second exchange is needed.
 * fixed_lohi (nullable) = int32[6] global lo, hi: cells outside it in any axis
 * are never relaxed (non-periodic physical boundaries).
 * push (nullable): a DEVICE table of int64 addresses, 27 per box (ghosts.py):
 * every output cell within 2 of a box face is also stored through it into
 * the ghost cells FillBoundary(b, 2) would copy it to -- on this GPU or, via
 * NVLink-mapped symmetric memory, a peer -- so b's width-2 ghosts are current
 * when the kernel ends (a peer's: after a device barrier).  With push the
 * call is AMRB_ENOTSUP (nothing launched) unless the level takes the
 * k_gsrb_stream path. */
int amrb_gsrb_sweep(const amrb_level* lv, const amrb_field* a, const double* a_base,
                    amrb_field* b, double* b_base, const amrb_field* rhs,
                    const double* rhs_base, const double dh[3],
                    const int32_t* fixed_lohi, const uint64_t* push, void* stream);

/* amrb_gsrb_sweep that also reduces the residual of its INPUT:
 * *norm = max(*norm, max over valid cells of |rhs - L(a)|), stored as the
 * uint64 bit pattern of a non-negative double (the caller zeroes *norm; a NaN
 * residual propagates).  Same result as amrb_residual_norm(a) followed by
 * amrb_gsrb_sweep, in one pass over a and rhs.  AMRB_ENOTSUP (nothing
 * launched) when the level does not take the k_gsrb_stream path. */
int amrb_gsrb_sweep_norm(const amrb_level* lv, const amrb_field* a, const double* a_base,
                         amrb_field* b, double* b_base, const amrb_field* rhs,
                         const double* rhs_base, const double dh[3],
                         const int32_t* fixed_lohi, uint64_t* norm, const uint64_t* push,
                         void* stream);

/* amrb_gsrb_sweep (norm == NULL) / amrb_gsrb_sweep_norm with FillBoundary
 * fused in: every CTA first copies the width-2 ghost cells of its input
 * footprint through `pull` (27 entries per box, ghosts.pull_table: the source
 * address of ghost cell (0, 0, 0) of each direction's slab, bit 0 set when the
 * source box is on another GPU; 0 = not filled, e.g. a non-periodic side), so
 * a's ghosts need not be current and are current afterwards.  nranks > 1: the
 * launch is also the device barrier of amrb_prog_run_p2p_sync (same pads and
 * epoch): CTA 0 publishes, the CTAs that read another GPU's cells (and CTA 0)
 * wait for every peer -- the rest start at once.  Periodic levels only (no
 * fixed cells). */
int amrb_gsrb_sweep_pull(const amrb_level* lv, const amrb_field* a, double* a_base,
                         amrb_field* b, double* b_base, const amrb_field* rhs,
                         const double* rhs_base, const double dh[3], const uint64_t* pull,
                         const uint64_t* pad_ptrs, int rank, int nranks, uint32_t* epoch,
                         uint64_t* norm, void* stream);

/* Prolongation fused into the first post-smoothing sweep of the V-cycle up-leg:
 * b = GSRB(a + P(c)), P = piecewise-constant interpolation of the coarse
 * correction c (interp_to_fine(..., "pc"), coarse_fine.py:166-185, then
 * phi_f += tmp).  c lives on the box-local coarsening (ratio 2) of a's level;
 * ghosts of a filled to 2, of rhs and c to 1; periodic (no fixed cells).
 * Bit-identical to amrb_prolong(add) + fill_boundary(a, 2) + amrb_gsrb_sweep;
 * `a` itself is left unchanged.  AMRB_ENOTSUP when the level does not take the
 * k_gsrb_sweep5 path (nothing launched). */
int amrb_gsrb_sweep_prolong(const amrb_level* lv, const amrb_field* a, const double* a_base,
                            amrb_field* b, double* b_base, const amrb_field* rhs,
                            const double* rhs_base, const double dh[3],
                            const amrb_level* clv, const amrb_field* c, const double* c_base,
                            const uint64_t* push, void* stream);



/* average_down (coarse_fine.py:136-163) on the box-local coarsened layout
 * (crse box b = fine box b coarsened).  ratio = int32[3] per 3-D axis, each 1
 * or 2 (NULL = 2,2,2).  mode 0 "average": crse = mean of the children summed
 * in numpy's reshape-mean order, e.g. in 3-D ((((c000+c001)+(c010+c011))
 * +(c100+c101))+(c110+c111))/8; mode 1 "injection": the child at offset 0. */
int amrb_restrict(const amrb_level* crse_lv, amrb_field* crse, double* crse_base,
                  const amrb_field* fine, const double* fine_base, int ncomp,
                  const int32_t* ratio, int mode, void* stream);

/* Fused residual + restriction (3-D, ratio 2): crse = average_down of
 * (rhs - L(phi)), bit-identical to residual then amrb_restrict. */
int amrb_residual_restrict(const amrb_level* crse_lv, amrb_field* crse,
                           double* crse_base, const amrb_field* rhs,
                           const double* rhs_base, const amrb_field* phi,
                           const double* phi_base, const double dh[3],
                           void* stream);

/* interp_to_fine "pc" (coarse_fine.py:166-185, interp_block :60-72),
 * optionally followed by an add: fine(c) (+)= crse(c / ratio), crse on the
 * box-local coarsened layout.  add = 0 is plain pc interpolation. */
int amrb_prolong(const amrb_level* fine_lv, amrb_field* fine, double* fine_base,
                 const amrb_field* crse, const double* crse_base, int ncomp,
                 const int32_t* ratio, int add, void* stream);



/* ------------------------------------------------------------------------ */
/* Inter-level AMR operators + two-level advection.  Work     */
/* lists: prefix = int64[nb+1] prefix of per-box work items over the        */
/* resident boxes `boxes` (int32[nb]); total = prefix[nb].  All results are  */
/* bit-identical to the reference's numpy (see csrc/amr.cu).                */
/* ------------------------------------------------------------------------ */
/* Upwind face fluxes (advect.py:24-36) along 3-D axis axis3: face array of
 * box b at flux + face_off[b], layout (ncomp, n + e_axis) C order; phi needs
 * one filled ghost layer. */
int amrb_adv_flux(const amrb_level* lv, const amrb_field* phi_f, const double* phi,
                  const int64_t* prefix, const int32_t* boxes, int nb, int64_t total,
                  const int64_t* face_off, double* flux, int ncomp, int axis3, double u,
                  void* stream);
/* phi -= dtdx[d] * (F_d[hi] - F_d[lo]) for d = 0..dim-1 (advect.py:39-47);
 * flux[d] / face_off[d] = device pointers of dimension d's face arrays. */
int amrb_adv_update(const amrb_level* lv, const amrb_field* phi_f, double* phi,
                    const int64_t* prefix, const int32_t* boxes, int nb, int64_t total,
                    const double* const* flux, const int64_t* const* face_off, int ncomp,
                    int dim, const double dtdx[3], void* stream);
/* out = a*x + b*y on valid cells (fill_patch time blend, coarse_fine.py:267-273). */
int amrb_axpby(const amrb_level* lv, const int64_t* prefix, const int32_t* boxes, int nb,
               int64_t total, const amrb_field* out_f, double* out, double a,
               const amrb_field* x_f, const double* x, double b, const amrb_field* y_f,
               const double* y, void* stream);
/* fine (every cell of each box's grown box) <- interpolation of crse (box b =
 * coarsen(fine box b) with enough ghosts), pc (linear = 0) or minmod-limited
 * linear (interp_block, coarse_fine.py:60-99). */
int amrb_interp(const amrb_level* fine_lv, const amrb_field* fine_f, double* fine,
                const amrb_level* crse_lv, const amrb_field* crse_f, const double* crse,
                const int64_t* prefix, const int32_t* boxes, int nb, int64_t total, int ncomp,
                int dim, const int32_t ratio[3], int linear, void* stream);
/* *dev_count += NaNs in region (int32[nb][6] box-local lo, hi) of each box. */
int amrb_nan_count(const amrb_field* f, const double* x, const int64_t* prefix,
                   const int32_t* boxes, int nb, int64_t total, const int32_t* region,
                   int ncomp, unsigned long long* dev_count, void* stream);
/* FluxRegister (coarse_fine.py:317-472).  crse_add: reg[p0] -= scale*F[p1]
 * per (p0, p1) pair; fine_add: reg[e0] += scale * avg(F[e1..e_nsrc]) in
 * numpy's reshape-mean order (seq = 1: sequential 4-term sum); reflux:
 * crse[tgt[t]] += coef[e] * reg[src[e]], e in start[t] .. start[t+1]-1. */
int amrb_fr_crse(const int64_t* pairs, int64_t n, double* reg, const double* flux,
                 double scale, void* stream);
int amrb_fr_fine(const int64_t* idx, int64_t n, int nsrc, int seq, double* reg,
                 const double* flux, double scale, void* stream);
int amrb_fr_reflux(const int64_t* tgt, const int64_t* start, int64_t n, const int64_t* src,
                   const double* coef, double* crse, const double* reg, void* stream);

/* ||rhs - L(phi)||_inf over this device's valid cells, without writing the
 * residual (phi ghosts width 1 filled).  Result (one double) to dev_out. */
int amrb_residual_norm(const amrb_level* lv, const amrb_field* rhs,
                       const double* rhs_base, const amrb_field* phi,
                       const double* phi_base, const double dh[3], double* dev_out,
                       void* stream);

/* Coarse tail of the V-cycle in ONE CTA (all levels in shared memory):
 * nlev single-box periodic levels, each half the previous; lohi = int32
 * [nlev][6] (3-D padded), dh = double[nlev][3].  Reads level-0 rhs (valid) from
 * `rhs`, runs zero/nu1 sweeps/residual-restrict down to the bottom (nbottom
 * sweeps), pc-prolong + nu2 sweeps back up, and writes level-0 phi (valid).
 * Bit-identical to the per-level kernels / oracle.  cluster: 0 one-CTA kernels
 * only, 1 an 8-CTA cluster kernel (which also runs a 32^3 top level) for cubic
 * power-of-two chains, 2 also for 32 x n1 x n2 chains.  *ghosts_written
 * (nullable) = the ghost width of level-0 phi the launched kernel left current
 * (1 for the cluster kernel, else 0). */
int amrb_coarse_tail(int nlev, const int32_t* lohi, const double* dh,
                     const amrb_field* rhs, const double* rhs_base, amrb_field* phi,
                     double* phi_base, int nu1, int nu2, int nbottom, int cluster,
                     int32_t* ghosts_written, void* stream);

/* One single-box periodic MLMG level's half V-cycle in one grid-synchronised
 * (cooperative) launch -- the per-level steps of the reference-semantics
 * V-cycle (oracle/mlmg_ref.py) for a level small enough
 * to be launch-latency bound.  up == 0: zero phi, nsweeps in-place GSRB
 * sweeps, then crse (the next coarser level's rhs, valid cells) =
 * avg8(rhs - L phi).  up == 1: phi += crse(parent) (crse = coarser phi, valid
 * cells read), nsweeps sweeps, then phi's width-1 periodic ghost layer.
 * lohi: the level's box (6 ints), dh: 1/h^2 per axis.  Extents must be even.
 * Bit-identical to fill + amrb_gsrb_sweep / amrb_residual_restrict /
 * amrb_prolong. */
int amrb_level_grid(int up, const int32_t* lohi, const double* dh, const amrb_field* rhs,
                    const double* rhs_base, amrb_field* phi, double* phi_base, const amrb_field* crse,
                    double* crse_base, int nsweeps, void* stream);

/* reduce (fabarray.py:409-440) over valid cells of one component on this
 * device: kind 0 sum, 1 min, 2 max, 3 max|x| (inf-norm).  Deterministic:
 * fixed-shape per-tile partials then one ordered pass.  Result (one double)
 * is written to dev_out. */
int amrb_reduce(const amrb_level* lv, const amrb_field* x, const double* x_base,
                int comp, int kind, double* dev_out, void* stream);

/* FillBoundary (fabarray.py:364) of a level that is ONE periodic box equal to
 * its domain: every ghost cell within `width` is copied from its periodic
 * image, as the fill plan's records would (same bits), in one launch without
 * a record table.  AMRB_ENOTSUP unless the level has exactly one resident box
 * and width <= both the field's ghost width and the box extent on each axis
 * (3-D).  ncomp = the field's component count. */
int amrb_fill_wrap(const amrb_level* lv, amrb_field* f, double* base, int ncomp, int width,
                   void* stream);
/* setval (fabarray.py:119-122, Fab.setval :58-65): components [comp0, comp1)
 * of box `box` (-1: every resident box) = value: ghosts 0 the valid cells,
 * 1 the grown box, 2 the ghost cells only. */
int amrb_setval(const amrb_level* lv, amrb_field* f, double* base, int box, int comp0, int comp1,
                int ghosts, double value, void* stream);

/* Fill ghost cells outside the physical domain (apply_domain_boundary,
 * amr_core.py:111-146).  bc: int32[3][2] per (axis, side) 0 periodic/skip,
 * 1 external (value), 2 extrap, 3 reflect: value * the cell mirrored across
 * the face (the MLMG coarse-level homogeneous Dirichlet ghosts,
 * oracle/mlmg_ref.py reflect_ghosts).  One pass per (axis, side) in that
 * order.  domain: int32[6] lo, hi (3-D padded). */
int amrb_domain_bc(const amrb_level* lv, amrb_field* f, double* base, int ncomp,
                   const int32_t* domain, const int32_t* bc, double value,
                   void* stream);

/* ------------------------------------------------------------------------ */
/* NCCL plumbing (multi-GPU).  The unique id is exchanged by the caller      */
/* (torch.distributed); the communicator is owned by the Transport.          */
/* ------------------------------------------------------------------------ */
int amrb_nccl_unique_id(uint8_t* out128);
int amrb_nccl_comm_create(const uint8_t* id128, int nranks, int rank, void** comm);
int amrb_nccl_comm_destroy(void* comm);
/* In-place all-reduce of n doubles: op 0 sum, 1 min, 2 max. */
int amrb_nccl_allreduce(double* buf, int64_t n, int op, void* comm, void* stream);
/* All-gather: each rank contributes n doubles. */
int amrb_nccl_allgather(const double* send, double* recv, int64_t n, void* comm,
                        void* stream);

#ifdef __cplusplus
}
#endif
#endif /* AMRB_H */
