#include <cuda_runtime.h>
#include <cstdint>
// A, B: 64 boxes, each [E0][E1][pitch] doubles at box stride; copy valid (64x64x64) rows.
extern "C" __global__ void rowcopy(const double* __restrict__ A, double* __restrict__ B, long long bstride, int pitch,
                                   int E1, int g, int front, int n, int nboxes, int rows_per_warp, int scatter) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  long long nrows = (long long)nboxes * n * n;
  for (long long rr = (long long)warp * rows_per_warp; rr < nrows; rr += (long long)gridDim.x * blockDim.x / 32 * rows_per_warp) {
    for (int q = 0; q < rows_per_warp && rr + q < nrows; ++q) {
      long long row = rr + q;
      int b, rem;
      if (scatter) { b = row % nboxes; rem = row / nboxes; } else { b = row / (n * n); rem = row % (n * n); }
      int i = rem / n, j = rem % n;
      long long off = b * bstride + (long long)(i + g) * E1 * pitch + (long long)(j + g) * pitch + front + g;
      const double2* s = reinterpret_cast<const double2*>(A + off);
      double2* d = reinterpret_cast<double2*>(B + off);
      d[lane] = __ldg(s + lane);
    }
  }
}
extern "C" __global__ void flatcopy(const double2* __restrict__ A, double2* __restrict__ B, long long n2) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x) B[i] = __ldg(A + i);
}
extern "C" void launch_rowcopy(const double* A, double* B, long long bstride, int pitch, int E1, int g, int front, int n, int nboxes, int rpw, int grid, int block, cudaStream_t s, int scatter) {
  rowcopy<<<grid, block, 0, s>>>(A, B, bstride, pitch, E1, g, front, n, nboxes, rpw, scatter);
}
extern "C" void launch_flat(const double* A, double* B, long long n, int grid, int block, cudaStream_t s) {
  flatcopy<<<grid, block, 0, s>>>((const double2*)A, (double2*)B, n / 2);
}
