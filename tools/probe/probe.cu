// Microarchitecture probe for design decisions (L2-hit bandwidth, smem atomics, match_any).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__global__ void rd(const int4* __restrict__ p, size_t n_vec, size_t iters, int4* out) {
  int4 acc = make_int4(0,0,0,0);
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t it = 0; it < iters; ++it)
    for (size_t i = tid; i < n_vec; i += stride) {
      int4 v = __ldcg(p + i);
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  if (acc.x == 0x12345 && acc.y == 7) out[0] = acc;
}
__global__ void copyk(const int4* __restrict__ p, int4* __restrict__ q, size_t n_vec) {
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = tid; i < n_vec; i += stride) q[i] = __ldcs(p + i);
}
// random 4B gathers from a buffer of given size (sector-granularity test)
__global__ void gather4(const uint32_t* __restrict__ p, uint32_t mask, size_t n, uint32_t* out) {
  uint32_t acc = 0;
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  uint32_t h = (uint32_t)tid * 2654435761u;
  for (size_t i = tid; i < n; i += stride) {
    h = h * 1664525u + 1013904223u;
    acc += __ldcg(p + (h & mask));
  }
  if (acc == 0xdeadbeef) out[0] = acc;
}
template <int MODE>
__global__ void smem_k(int iters, uint32_t* out) {
  extern __shared__ uint32_t s[];
  const int W = 49152; // 192KB / 4
  for (int i = threadIdx.x; i < W; i += blockDim.x) s[i] = 0;
  __syncthreads();
  uint32_t h = threadIdx.x * 2654435761u + blockIdx.x;
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    h = h * 1664525u + 1013904223u;
    uint32_t idx = (h >> 8) % W;
    if (MODE == 0) s[idx] = h;                         // plain store
    else if (MODE == 1) atomicOr(&s[idx], 1u << (h & 31));  // smem atomic or
    else if (MODE == 2) atomicAdd(&s[idx], 1u);        // smem atomic add
    else if (MODE == 3) { unsigned m = __match_any_sync(0xffffffffu, idx >> 6); acc += m; s[idx] = h; }
    else if (MODE == 4) { ((unsigned char*)s)[idx * 4 + (h & 3)] = 1; }
    else if (MODE == 5) { double* d = (double*)s; d[idx >> 1] += 1.0; }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[h % W] + acc;
}
int main() {
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, 0));
  printf("dev %s SMs %d l2 %d smemOptin %zu smemPerSM %zu clock %d memclk %d busw %d\n", pr.name, pr.multiProcessorCount,
         pr.l2CacheSize, pr.sharedMemPerBlockOptin, pr.sharedMemPerMultiprocessor, pr.clockRate, pr.memoryClockRate, pr.memoryBusWidth);
  int nsm = pr.multiProcessorCount;
  size_t big = (size_t)4 << 30;
  int4 *p, *q; CK(cudaMalloc(&p, big)); CK(cudaMalloc(&q, big)); CK(cudaMemset(p, 1, big));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  // HBM read
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a); rd<<<nsm * 8, 512>>>(p, big / 16, 1, q); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("HBM read 4GiB: %.1f GB/s\n", big / ms / 1e6);
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a); copyk<<<nsm * 8, 512>>>(p, q, big / 16); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("HBM copy 4GiB: %.1f GB/s (r+w)\n", 2 * big / ms / 1e6);
  }
  // L2-resident reads for sizes
  size_t sizes[] = {8u << 20, 32u << 20, 64u << 20, 96u << 20};
  for (size_t sz : sizes) {
    int iters = (int)((16ull << 30) / sz);
    rd<<<nsm * 8, 512>>>(p, sz / 16, 2, q); cudaDeviceSynchronize();
    cudaEventRecord(a); rd<<<nsm * 8, 512>>>(p, sz / 16, iters, q); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("L2 read footprint %zu MB: %.1f GB/s\n", sz >> 20, (double)sz * iters / ms / 1e6);
  }
  // random 4B gathers
  uint32_t fp[] = {(1u << 20) - 1, (1u << 24) - 1, (1u << 28) - 1};  // 4MB, 64MB, 1GB footprints
  for (uint32_t m : fp) {
    size_t n = (size_t)1 << 30;
    gather4<<<nsm * 8, 512>>>((uint32_t*)p, m, n / 16, (uint32_t*)q); cudaDeviceSynchronize();
    cudaEventRecord(a); gather4<<<nsm * 8, 512>>>((uint32_t*)p, m, n, (uint32_t*)q); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("random 4B gather footprint %u MB: %.2f Gops/s\n", (m + 1) >> 18, n / ms / 1e6);
  }
  const char* names[] = {"STS.32", "ATOMS.OR", "ATOMS.ADD", "MATCH+STS", "STS.U8", "DADD smem rmw"};
  uint32_t* o; CK(cudaMalloc(&o, 4096 * 4));
  auto run = [&](auto kern, int mode) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608);
    int iters = 4096;
    kern<<<nsm, 1024, 196608>>>(iters, o); cudaDeviceSynchronize();
    cudaEventRecord(a); kern<<<nsm * 4, 1024, 196608>>>(iters, o); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    double ops = (double)nsm * 4 * 1024 * iters;
    printf("smem %-14s: %.1f Gops/s  (%.2f ops/clk/SM at %d MHz)\n", names[mode], ops / ms / 1e6, ops / (ms * 1e-3) / nsm / (pr.clockRate * 1e3), pr.clockRate / 1000);
  };
  run(smem_k<0>, 0); run(smem_k<1>, 1); run(smem_k<2>, 2); run(smem_k<3>, 3); run(smem_k<4>, 4); run(smem_k<5>, 5);
  CK(cudaGetLastError());
  return 0;
}
