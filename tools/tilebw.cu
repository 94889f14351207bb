// Microbenchmark: stream (ROWS x 68)-double plane tiles of a big padded array into
// shared memory with a STAGES-deep ring, no compute.  Three load mechanisms.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

constexpr int PK = 68;

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// array: [planes][rows_total][pitch] ; tile (rows x 68) at (plane, j0, k0)
struct Args {
  const double* a;
  int pitch, rows_total, planes, ntj, ntk, rows;
  long long tiles_per_col;  // planes
  double* sink;
};

template <int STAGES>
__global__ void __launch_bounds__(256) k_ldg(Args g) {
  extern __shared__ __align__(128) double sm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ncol = g.ntj * g.ntk;
  double acc = 0;
  for (int col = blockIdx.x; col < ncol; col += gridDim.x) {
    const int tj = col / g.ntk, tk = col % g.ntk;
    for (int p = 0; p < g.planes; ++p) {
      double* dst = sm + (p % STAGES) * g.rows * PK;
      const double* src = g.a + ((long long)p * g.rows_total + tj * 16) * g.pitch + tk * 64;
      for (int r = warp; r < g.rows; r += 8) {
        const double2* s2 = reinterpret_cast<const double2*>(src + (long long)r * g.pitch);
        double2 v = __ldcg(s2 + lane);
        double2 w = lane < 2 ? __ldcg(s2 + 32 + lane) : make_double2(0, 0);
        reinterpret_cast<double2*>(dst + r * PK)[lane] = v;
        if (lane < 2) reinterpret_cast<double2*>(dst + r * PK)[32 + lane] = w;
      }
      if ((p % STAGES) == STAGES - 1) {
        __syncthreads();
        acc += sm[tid];
      }
    }
  }
  if (acc == 12345.678) g.sink[0] = acc;
}

template <int STAGES>
__global__ void __launch_bounds__(256) k_cpasync(Args g) {
  extern __shared__ __align__(128) double sm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ncol = g.ntj * g.ntk;
  double acc = 0;
  for (int col = blockIdx.x; col < ncol; col += gridDim.x) {
    const int tj = col / g.ntk, tk = col % g.ntk;
    for (int p = 0; p < g.planes; ++p) {
      double* dst = sm + (p % STAGES) * g.rows * PK;
      const double* src = g.a + ((long long)p * g.rows_total + tj * 16) * g.pitch + tk * 64;
      for (int r = warp; r < g.rows; r += 8) {
        const double* s = src + (long long)r * g.pitch;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(su32(dst + r * PK + 2 * lane)), "l"(s + 2 * lane));
        if (lane < 2)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(su32(dst + r * PK + 64 + 2 * lane)), "l"(s + 64 + 2 * lane));
      }
      asm volatile("cp.async.commit_group;\n" ::);
      asm volatile("cp.async.wait_group %0;\n" ::"n"(STAGES - 1));
      if ((p % STAGES) == STAGES - 1) {
        __syncthreads();
        acc += sm[tid];
      }
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
  }
  if (acc == 12345.678) g.sink[0] = acc;
}

template <int STAGES>
__global__ void __launch_bounds__(256) k_tma(const __grid_constant__ CUtensorMap tm, Args g) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bars[STAGES];
  const int tid = threadIdx.x;
  const int ncol = g.ntj * g.ntk;
  const int bytes = g.rows * PK * 8;
  const int stride = (bytes + 127) / 128 * 128 / 8;
  if (tid == 0)
    for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bars[s])));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  double acc = 0;
  long long issued = 0, waited = 0;
  auto issue = [&](int col, int p) {
    const int tj = col / g.ntk, tk = col % g.ntk;
    const int s = issued % STAGES;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&bars[s])), "r"(bytes));
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
            su32(sm + s * stride)),
        "l"(&tm), "r"(tk * 64), "r"(tj * 16), "r"(p), "r"(su32(&bars[s]))
        : "memory");
    ++issued;
  };
  // flatten (col, plane) sequence for this CTA
  long long total = 0;
  for (int col = blockIdx.x; col < ncol; col += gridDim.x) total += g.planes;
  auto colof = [&](long long q, int& col, int& p) {
    col = blockIdx.x + (int)(q / g.planes) * gridDim.x;
    p = (int)(q % g.planes);
  };
  if (tid == 0)
    for (long long q = 0; q < STAGES - 1 && q < total; ++q) {
      int c, p;
      colof(q, c, p);
      issue(c, p);
    }
  for (long long q = 0; q < total; ++q) {
    if (tid == 0 && q + STAGES - 1 < total) {
      int c, p;
      colof(q + STAGES - 1, c, p);
      issue(c, p);
    }
    const int s = waited % STAGES;
    const unsigned par = (waited / STAGES) & 1;
    asm volatile(
        "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(
            su32(&bars[s])),
        "r"(par));
    ++waited;
    acc += sm[s * stride + tid];
    __syncthreads();
  }
  if (acc == 12345.678) g.sink[0] = acc;
}

extern "C" int run_tilebw(int mode, int stages, int rows, int ctas_per_sm, float* out_us) {
  // 256 planes x 260 rows x 264 pitch doubles ~ 140 MB
  const int planes = 128, rows_total = 1028, pitch = 264;
  size_t n = (size_t)planes * rows_total * pitch;
  double* a;
  cudaMalloc(&a, n * 8);
  cudaMemset(a, 0, n * 8);
  double* sink;
  cudaMalloc(&sink, 8);
  Args g{a, pitch, rows_total, planes, 64, 4, rows, planes, sink};
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int grid = sms * ctas_per_sm;
  if (grid > 256) grid = 256;  // 256 columns
  size_t smem = (size_t)stages * ((rows * PK * 8 + 127) / 128 * 128);
  CUtensorMap tm;
  if (mode == 2) {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    auto fn = (PFN_cuTensorMapEncodeTiled_v12000)fp;
    cuuint64_t gd[3] = {(cuuint64_t)pitch, (cuuint64_t)rows_total, (cuuint64_t)planes};
    cuuint64_t gs[2] = {(cuuint64_t)pitch * 8, (cuuint64_t)pitch * rows_total * 8};
    cuuint32_t box[3] = {PK, (cuuint32_t)rows, 1}, es[3] = {1, 1, 1};
    fn(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, a, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  auto launch = [&]() {
    if (mode == 0) {
      if (stages == 2) k_ldg<2><<<grid, 256, smem>>>(g);
      else k_ldg<4><<<grid, 256, smem>>>(g);
    } else if (mode == 1) {
      if (stages == 2) k_cpasync<2><<<grid, 256, smem>>>(g);
      else k_cpasync<4><<<grid, 256, smem>>>(g);
    } else {
      if (stages == 2) k_tma<2><<<grid, 256, smem>>>(tm, g);
      else if (stages == 4) k_tma<4><<<grid, 256, smem>>>(tm, g);
      else k_tma<8><<<grid, 256, smem>>>(tm, g);
    }
  };
  cudaFuncSetAttribute(k_ldg<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  cudaFuncSetAttribute(k_ldg<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  cudaFuncSetAttribute(k_cpasync<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  cudaFuncSetAttribute(k_cpasync<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  cudaFuncSetAttribute(k_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  cudaFuncSetAttribute(k_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  cudaFuncSetAttribute(k_tma<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  for (int i = 0; i < 3; ++i) launch();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 10; ++i) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  *out_us = ms * 100.0f;
  cudaError_t err = cudaGetLastError();
  cudaFree(a);
  cudaFree(sink);
  return (int)err;
}
