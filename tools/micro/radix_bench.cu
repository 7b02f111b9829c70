// Microbenchmark: cycles per block-wide radix sort (2 passes) of n keys, as used by k_heavy_numeric.
#include <cstdio>
#include "../../paper_2501_07056_b200/csrc/heavy_rows.cuh"
using namespace mg;
__global__ void __launch_bounds__(kNT, 1) bench(int n, int iters, unsigned long long* out) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint16_t* key0 = reinterpret_cast<uint16_t*>(smem);
  uint16_t* key1 = key0 + kCap + kCap / 8;
  uint16_t* pay0 = key1 + kCap;
  uint16_t* pay1 = pay0 + kCap + kCap / 8;
  uint32_t* hist = reinterpret_cast<uint32_t*>(pay1 + kCap);
  uint32_t* scratch = hist + kRadix * kNW;
  unsigned long long t0 = 0, acc = 0;
  for (int it = 0; it < iters; ++it) {
    for (int q = threadIdx.x; q < n; q += kNT) { key0[pad_k(q)] = (uint16_t)((q * 2654435761u + it) % 8191u); pay0[pad_k(q)] = q; }
    __syncthreads();
    t0 = clock64();
    radix_pass<true>(key0, pay0, key1, pay1, n, 0, 7, hist, scratch);
    radix_pass<false>(key1, pay1, key0, pay0, n, 7, 6, hist, scratch);
    acc += clock64() - t0;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = acc / iters;
}
__global__ void __launch_bounds__(kNT, 1) bench_sync(int iters, unsigned long long* out) {
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = (clock64() - t0) / iters;
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 1024 * 8);
  size_t sm = 100 * 1024;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  for (int n : {512, 1024, 2048, 4096, 8192}) {
    for (int grid : {1, 148}) {
      bench<<<grid, kNT, sm>>>(n, 200, d);
      unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("n=%5d grid=%3d: %llu cycles per 2-pass sort (%.2f cyc/elem)\n", n, grid, h, (double)h / n);
    }
  }
  bench_sync<<<148, kNT>>>(10000, d);
  unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("__syncthreads (512 thr): %llu cycles\n", h);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
