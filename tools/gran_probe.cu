// DRAM bytes per random 8-byte gather from a 1 GB table, by load flavour.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
__device__ __forceinline__ uint32_t h32(uint32_t x){x^=x>>16;x*=0x7feb352du;x^=x>>15;x*=0x846ca68bu;x^=x>>16;return x;}
template <int V>
__global__ void k(const double* t, uint32_t mask, int iters, double* sink) {
  uint32_t s = h32(blockIdx.x * blockDim.x + threadIdx.x);
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    s = s * 1664525u + 1013904223u;
    const double* p = t + ((s >> 3) & mask);
    double v;
    if (V == 0) v = __ldg(p);
    else if (V == 1) v = __ldcg(p);
    else if (V == 2) asm volatile("ld.global.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    else if (V == 3) asm volatile("ld.global.cg.L2::64B.f64 %0, [%1];" : "=d"(v) : "l"(p));
    else if (V == 4) asm volatile("ld.volatile.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
    else if (V == 5) asm volatile("ld.global.cv.f64 %0, [%1];" : "=d"(v) : "l"(p));
    else if (V == 6) asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
    else if (V == 7) asm volatile("ld.global.nc.L1::no_allocate.L2::64B.f64 %0, [%1];" : "=d"(v) : "l"(p));
    else if (V == 8) asm volatile("ld.global.ca.L2::64B.f64 %0, [%1];" : "=d"(v) : "l"(p));
    else asm volatile("ld.global.cg.L2::256B.f64 %0, [%1];" : "=d"(v) : "l"(p));
    acc += v;
  }
  if (acc == 1.5) sink[0] = acc;
}
int main() {
  size_t n = (1u << 30) / 8; double* t; double* sink;
  cudaMalloc(&t, n * 8); cudaMemset(t, 0, n * 8); cudaMalloc(&sink, 64);
  const int blocks = 148 * 8, threads = 256, iters = 64;
  float ms; cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
#define RUN(V) k<V><<<blocks, threads>>>(t, (uint32_t)(n - 1), iters, sink); cudaEventRecord(a); k<V><<<blocks, threads>>>(t, (uint32_t)(n - 1), iters, sink); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); printf("variant %d: %.3f ms, %.1f Gload/s\n", V, ms, (double)blocks*threads*iters/ms/1e6);
  RUN(0) RUN(3) RUN(4) RUN(5) RUN(6) RUN(7) RUN(8) RUN(9)
  printf("loads per launch %d\n", blocks*threads*iters);
  return 0;
}
