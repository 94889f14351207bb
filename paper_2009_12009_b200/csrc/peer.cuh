// Cross-GPU signalling helpers shared by the copy programs (comm.cu) and the
// streaming sweep's in-kernel ghost pull (gsrb_stream.cu).
#pragma once
#include <cstdint>

namespace amrb {

// Failure detection for the NVLink signalling (transport.py:20-24,37-38: a
// failed message raises TransportError(src, dst, why)).  Every device-side
// wait for a peer is bounded: after `timeout_ns` of %globaltimer the waiting
// lane records (code, waiting rank, missing peer, epoch) in the fault mailbox
// -- pinned host memory the Transport registered -- and gives up; once a fault
// is recorded every later wait returns at once, so a dead peer costs one
// timeout, not one per barrier.  The host raises TransportError from the
// mailbox after its next synchronisation (Transport.check_faults).
struct Fault {
  unsigned long long* box;  // [0] code (0 none, 1 peer wait timed out), [1] rank, [2] peer, [3] epoch
  unsigned long long* dev;  // device twin of box[0]: what the waits poll (never host memory, see signal_store)
  unsigned long long timeout_ns;
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Cross-GPU signals.  Every exchange here is a PULL: what a peer reads after
// a signal lives in the signalling GPU's own HBM, written by earlier kernels,
// and the owner's L2 serves the peer's NVLink loads -- so a gpu-scope release
// fence orders it before the signal store, and the waiting side needs a
// gpu-scope acquire fence after it sees the signal.  No system-scope fence:
// fence.sc.sys / MEMBAR.SYS also drains this GPU's outstanding PCIe traffic,
// and with bulk host copies in flight on side streams (the e2e pipeline) one
// barrier measured 200 us instead of 6 (tools/mb_interfere.py, 4 GPUs).
__device__ __forceinline__ void signal_store(uint32_t* slot, uint32_t v) {
  asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;\n" ::"l"(slot), "r"(v) : "memory");
}

__device__ __forceinline__ void record_fault(const Fault& f, int rank, int peer, uint32_t target) {
  if (f.dev && atomicCAS(f.dev, 0ull, 1ull) == 0ull && f.box) {
    f.box[1] = (unsigned long long)rank;
    f.box[2] = (unsigned long long)peer;
    f.box[3] = (unsigned long long)target;
    __threadfence_system();  // failure path only
    f.box[0] = 1ull;
  }
}

__device__ __forceinline__ bool faulted(const Fault& f) {
  return f.dev && *reinterpret_cast<volatile unsigned long long*>(f.dev) != 0;
}

// spin until *pad (wrap-safe) reaches `target`; false (and a fault recorded) on timeout
__device__ __forceinline__ bool peer_wait(const uint32_t* pad, uint32_t target, int rank, int peer, const Fault& f) {
  if (faulted(f)) return false;
  const unsigned long long t0 = global_ns();
  for (unsigned it = 0;; ++it) {
    uint32_t x;
    asm volatile("ld.relaxed.sys.global.u32 %0, [%1];\n" : "=r"(x) : "l"(pad) : "memory");
    if ((int32_t)(x - target) >= 0) {
      asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
      return true;
    }
    if ((it & 255) == 255 && f.timeout_ns && global_ns() - t0 > f.timeout_ns) {
      record_fault(f, rank, peer, target);
      return false;
    }
  }
}


Fault current_fault();  // host: the mailbox + the "peer_timeout_ms" option (comm.cu)

}  // namespace amrb
