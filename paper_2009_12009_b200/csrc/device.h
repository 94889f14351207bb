// Device-side descriptors shared by the kernel translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "amrb_internal.h"

namespace amrb {

#define AMRB_CUDA(call)                                                              \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess)                                                           \
      throw ::amrb::Error(AMRB_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// Host-side tally of kernel launches issued by the library (graph replays are
// not seen here; callers multiply captured launches by replays).
void count_launch();

inline void check_launch(const char* what) {
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error(AMRB_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Programmatic dependent launch.  Every library kernel begins with pdl_entry():
// griddepcontrol.wait returns once the preceding grid in the stream has
// completed and its writes are visible (a no-op for a normally launched grid),
// then launch_dependents lets the next grid be scheduled onto the SMs this one
// leaves free -- only after ALL of this grid's CTAs have started, so a waiting
// dependent never takes a slot from it.  The wait comes before any early
// return, so completion stays transitive along the stream.  launch_k() adds
// the programmatic-serialization attribute to EAGER launches only (AMRB_PDL=2,
// the default): measured on the C3 bench, eager PDL takes 0.14 ms off the
// end-to-end step (10.49 -> 10.35 ms), while programmatic edges inside the
// captured V-cycle graph cost 0.1 ms per solve (9.05 -> 9.16 ms).
// AMRB_PDL=0: off, 1: everywhere.
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
int pdl_mode();
int64_t option(const char* name);  // amrb_set_option registry (stencil.cu)
template <class... KArgs, class... Args>
void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  const int mode = pdl_mode();
  bool on = mode == 1;
  if (mode == 2) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    on = cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone;
  }
  cfg.numAttrs = on ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Checked builds (make CHECKED=1 -> _lib/libamrb_checked.so): device-side
// invariant checks in the concurrency-heavy kernels.  A failed check counts
// into a device word and records its line (amrb_debug_checks reads them);
// compute-sanitizer is closed on this GPU pool, so these are the sanitizer.
#ifndef AMRB_CHECKED
#define AMRB_CHECKED 0
#endif
// `box` = unsigned int[2] in device memory: {failures, first failing line}
#define AMRB_DCHECK_AT(box, cond)                                   \
  do {                                                              \
    if (AMRB_CHECKED && !(cond) && (box)) {                         \
      if (atomicAdd((box), 1u) == 0u) (box)[1] = (unsigned)__LINE__; \
    }                                                               \
  } while (0)
unsigned int* debug_check_words();  // device words of the checked build (gsrb_stream.cu)

// Valid box of one grid, 3-D padded, global index space.
struct BoxGeom {
  int lo[3];
  int n[3];
};

// Storage of one box of one FabArray: element offset of the VALID lo cell
// (comp 0) and strides.  Axis-2 stride is 1.
struct FabView {
  int64_t off;
  int64_t s0, s1, cs;
};

// Unique device allocation helper.
template <class T>
struct DevArray {
  T* p = nullptr;
  size_t n = 0;
  DevArray() = default;
  DevArray(const DevArray&) = delete;
  DevArray& operator=(const DevArray&) = delete;
  ~DevArray() {
    if (p) cudaFree(p);
  }
  void upload(const std::vector<T>& h) {
    if (p) cudaFree(p);
    p = nullptr;
    n = h.size();
    if (n == 0) return;
    AMRB_CUDA(cudaMalloc(&p, n * sizeof(T)));
    AMRB_CUDA(cudaMemcpy(p, h.data(), n * sizeof(T), cudaMemcpyHostToDevice));
  }
  void alloc(size_t count) {
    if (p) cudaFree(p);
    p = nullptr;
    n = count;
    if (n) AMRB_CUDA(cudaMalloc(&p, n * sizeof(T)));
  }
};

// Tiles of the valid region: (box, i0, j0, k0) in box-local valid coords.
struct TileTable {
  int ti, tj, tk;
  long long total = 0;  // column tables: plane-steps over all columns
  std::vector<int4> host;
  DevArray<int4> dev;
};

// Streaming-sweep work items, 8 ints each (gsrb_stream.cu seg_table)
struct SegTable {
  std::vector<int> host;
  DevArray<int> dev;
  int n = 0;
};

struct Level {
  int nboxes = 0;
  std::vector<BoxGeom> geo;
  std::vector<uint8_t> resident;
  DevArray<BoxGeom> dgeo;
  std::map<std::tuple<int, int, int>, TileTable*> tables;
  std::map<std::tuple<int, int, int>, SegTable*> segtabs;
  DevArray<double> partials;  // reduction scratch
  // block index of each resident box inside a FabArray allocation (resident order)
  std::vector<int> slot;
  DevArray<int> dslot;
  ~Level() {
    for (auto& kv : tables) delete kv.second;
    for (auto& kv : segtabs) delete kv.second;
  }
  const TileTable& tiles(int ti, int tj, int tk);
  // (box, j0, k0, first plane-step) per TJ x TK column of the valid region
  const TileTable& columns(int tj, int tk);
  bool all_even() const;
};

struct Field {
  const Level* lv = nullptr;
  int ngrow = 0;
  int ng3[3] = {0, 0, 0};  // ghost width per 3-D axis (0 on padding axes)
  std::vector<FabView> host;
  DevArray<FabView> dev;
};

int num_sms();

constexpr int kMaxPeers = 8;

}  // namespace amrb
