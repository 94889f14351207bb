// Device-side solve loop: a CUDA graph with a conditional WHILE node.
//
// The MLMG solve (paper_2009_12009_b200/mlmg.py) captures ONE iteration --
// the V-cycle and the residual norm that decides whether to go on -- into the
// body of a WHILE node; the body ends with k_loop_control, which appends the
// norm to the residual history, counts the iteration and sets the node's
// condition to "not converged and under max_iter".  A whole solve is then one
// graph launch and one host synchronisation, instead of a replay + stream sync
// + host test per cycle.  The stopping test is the oracle's
// (oracle/mlmg_ref.py OracleMLMG.solve): stop once norm <= rtol * r0,
// evaluated in the same fp64 operations.
//
// The loop state lives in DEVICE memory: k_loop_reset writes it from kernel
// arguments before a launch and the caller moves it to the host once after
// (amrb_store_host).  Nothing inside the loop touches host memory -- a kernel
// store to pinned memory, or a system-scope fence, waits behind whatever bulk
// PCIe copies are in flight on other streams (measured 2 -> 70 us per store
// with the e2e pipeline's copies running, tools/mb_interfere.py).
#include <cuda_runtime.h>

#include "device.h"

namespace amrb {

namespace {

struct LoopState {
  double rtol;
  int32_t max_iter;
  int32_t iters;
  double r0;
  double hist[1];  // [capacity]
};

__global__ void k_loop_reset(LoopState* st, double rtol, int max_iter, const double* r0) {
  st->rtol = rtol;
  st->max_iter = max_iter;
  st->iters = 0;
  st->r0 = *r0;
}

__global__ void k_loop_control(cudaGraphConditionalHandle h, double* norm, const double* r0, LoopState* st,
                               int capacity) {
  pdl_entry();
  const double rn = *norm;
  int it = st->iters;
  if (it < capacity) st->hist[it] = rn;
  st->iters = ++it;
  *norm = 0.0;  // the next iteration's norm accumulates from zero
  const bool done = rn <= st->rtol * *r0 || it >= st->max_iter;
  cudaGraphSetConditional(h, done ? 0u : 1u);
}

}  // namespace

struct Loop {
  cudaGraph_t graph = nullptr;
  cudaGraph_t body = nullptr;  // owned by graph
  cudaGraphExec_t exec = nullptr;
  cudaGraphConditionalHandle handle = 0;
  cudaStream_t capture = nullptr;
  bool capturing = false;
  ~Loop() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
  }
};

}  // namespace amrb

using amrb::Error;
using amrb::guarded;
using amrb::Loop;

extern "C" int amrb_loop_begin(void* stream, amrb_loop** out) {
  return guarded([&] {
    if (!out || !stream) throw Error(AMRB_EINVAL, "amrb_loop_begin: null argument");
    auto* L = new Loop;
    try {
      AMRB_CUDA(cudaGraphCreate(&L->graph, 0));
      AMRB_CUDA(cudaGraphConditionalHandleCreate(&L->handle, L->graph, 1, cudaGraphCondAssignDefault));
      cudaGraphNodeParams p = {};
      p.type = cudaGraphNodeTypeConditional;
      p.conditional.handle = L->handle;
      p.conditional.type = cudaGraphCondTypeWhile;
      p.conditional.size = 1;
      cudaGraphNode_t node;
      AMRB_CUDA(cudaGraphAddNode(&node, L->graph, nullptr, 0, &p));
      L->body = p.conditional.phGraph_out[0];
      L->capture = reinterpret_cast<cudaStream_t>(stream);
      AMRB_CUDA(cudaStreamBeginCaptureToGraph(L->capture, L->body, nullptr, nullptr, 0,
                                              cudaStreamCaptureModeRelaxed));
      L->capturing = true;
    } catch (...) {
      delete L;
      throw;
    }
    *out = reinterpret_cast<amrb_loop*>(L);
  });
}

extern "C" int amrb_loop_reset(void* state, double rtol, int max_iter, const double* r0, void* stream) {
  return guarded([&] {
    if (!state || !r0 || max_iter < 0) throw Error(AMRB_EINVAL, "amrb_loop_reset: bad arguments");
    amrb::launch_k(amrb::k_loop_reset, 1, 1, 0, reinterpret_cast<cudaStream_t>(stream),
                   reinterpret_cast<amrb::LoopState*>(state), rtol, max_iter, r0);
    amrb::check_launch("k_loop_reset");
  });
}

extern "C" int amrb_loop_control(amrb_loop* loop, double* norm, const double* r0, void* state, int capacity,
                                 void* stream) {
  return guarded([&] {
    Loop* L = reinterpret_cast<Loop*>(loop);
    if (!L || !norm || !r0 || !state || capacity < 1) throw Error(AMRB_EINVAL, "amrb_loop_control: bad arguments");
    if (!L->capturing || reinterpret_cast<cudaStream_t>(stream) != L->capture)
      throw Error(AMRB_EINVAL, "amrb_loop_control: not inside this loop's capture");
    amrb::launch_k(amrb::k_loop_control, 1, 1, 0, L->capture, L->handle, norm, r0,
                   reinterpret_cast<amrb::LoopState*>(state), capacity);
    amrb::check_launch("k_loop_control");
  });
}

extern "C" int amrb_loop_end(amrb_loop* loop) {
  return guarded([&] {
    Loop* L = reinterpret_cast<Loop*>(loop);
    if (!L || !L->capturing) throw Error(AMRB_EINVAL, "amrb_loop_end: no capture in progress");
    cudaGraph_t g = nullptr;
    L->capturing = false;
    AMRB_CUDA(cudaStreamEndCapture(L->capture, &g));
    AMRB_CUDA(cudaGraphInstantiate(&L->exec, L->graph, 0));
  });
}

extern "C" int amrb_loop_launch(amrb_loop* loop, void* stream) {
  return guarded([&] {
    Loop* L = reinterpret_cast<Loop*>(loop);
    if (!L || !L->exec) throw Error(AMRB_EINVAL, "amrb_loop_launch: loop not instantiated");
    AMRB_CUDA(cudaGraphLaunch(L->exec, reinterpret_cast<cudaStream_t>(stream)));
  });
}

extern "C" int amrb_loop_destroy(amrb_loop* loop) {
  return guarded([&] {
    Loop* L = reinterpret_cast<Loop*>(loop);
    if (L && L->capturing) {
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(L->capture, &g);
      cudaGetLastError();
    }
    delete L;
  });
}
