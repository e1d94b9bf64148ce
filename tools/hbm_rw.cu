// Read-only, write-only and copy HBM bandwidth on one B200 (streaming 16-byte
// accesses, grid = 4 x 148 x 8 CTAs of 256 threads, best of 5).  Pass A of the
// RHS is write-heavy (25 GB written, 6 GB read per C5 launch): its memory
// floor is set by the write bandwidth, not the copy figure.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rd(const double2* __restrict__ a, size_t n, double* out) {
  double s = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const double2 v = __ldcs(a + i);
    s += v.x + v.y;
  }
  if (s == 12345.678) out[0] = s;
}
__global__ void wr(double2* a, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(a + i, make_double2((double)i, 1.0));
}
__global__ void cp(const double2* __restrict__ a, double2* b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(b + i, __ldcs(a + i));
}

int main() {
  const size_t bytes = (size_t)16 << 30, n = bytes / 16;
  double2 *a, *b;
  double* o;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMalloc(&o, 8);
  cudaMemset(a, 0, bytes);
  cudaMemset(b, 0, bytes);
  const int grid = 148 * 8 * 4;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int k = 0; k < 3; ++k) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      if (k == 0) rd<<<grid, 256>>>(a, n, o);
      if (k == 1) wr<<<grid, 256>>>(a, n);
      if (k == 2) cp<<<grid, 256>>>(a, b, n / 2);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    const double moved = (k == 2) ? (double)bytes : (double)bytes;  // copy: n/2 elements read + written
    printf("%-6s %.1f GB/s (%s)\n", k == 0 ? "read" : k == 1 ? "write" : "copy", moved / (best * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
