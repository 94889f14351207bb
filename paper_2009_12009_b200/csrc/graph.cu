// Device-side solve loop: a CUDA graph with a conditional WHILE node.
//
// The MLMG solve (paper_2009_12009_b200/mlmg.py) captures ONE iteration --
// the V-cycle and the residual norm that decides whether to go on -- into the
// body of a WHILE node; the body ends with k_loop_control, which appends the
// norm to the residual history (pinned host memory), counts the iteration and
// sets the node's condition to "not converged and under max_iter".  A whole
// solve is then one graph launch and one host synchronisation, instead of a
// replay + stream sync + host test per cycle.  The stopping test is the
// oracle's (oracle/mlmg_ref.py OracleMLMG.solve): stop once
// norm <= rtol * r0, evaluated in the same fp64 operations.
#include <cuda_runtime.h>

#include "device.h"

namespace amrb {

namespace {

// Pinned host block shared with the control kernel (UVA): the host writes
// rtol / max_iter / iters = 0 before each launch and reads iters / hist after.
struct LoopHost {
  double rtol;
  int32_t max_iter;
  int32_t iters;
  double hist[1];  // [capacity]
};

__global__ void k_loop_control(cudaGraphConditionalHandle h, double* norm, const double* r0, LoopHost* host,
                               int capacity) {
  pdl_entry();
  const double rn = *norm;
  int it = host->iters;
  if (it < capacity) host->hist[it] = rn;
  host->iters = ++it;
  *norm = 0.0;  // the next iteration's norm accumulates from zero
  const bool done = rn <= host->rtol * *r0 || it >= host->max_iter;
  __threadfence_system();
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

extern "C" int amrb_loop_control(amrb_loop* loop, double* norm, const double* r0, void* host_block, int capacity,
                                 void* stream) {
  return guarded([&] {
    Loop* L = reinterpret_cast<Loop*>(loop);
    if (!L || !norm || !r0 || !host_block || capacity < 1) throw Error(AMRB_EINVAL, "amrb_loop_control: bad arguments");
    if (!L->capturing || reinterpret_cast<cudaStream_t>(stream) != L->capture)
      throw Error(AMRB_EINVAL, "amrb_loop_control: not inside this loop's capture");
    amrb::launch_k(amrb::k_loop_control, 1, 1, 0, L->capture, L->handle, norm, r0,
                   reinterpret_cast<amrb::LoopHost*>(host_block), capacity);
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
