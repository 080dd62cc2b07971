// Microbenchmark: issue throughput of packed FFMA2 (fma.rn.f32x2, sm_100a) vs scalar FFMA.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t f2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r;
}
template <int N>
__global__ void k2(uint64_t* out, uint64_t a, uint64_t b) {
  uint64_t x[8];
  for (int i = 0; i < 8; ++i) x[i] = a + threadIdx.x + i;
  for (int it = 0; it < N; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = f2(x[i], b, x[i]);
  uint64_t s = 0; for (int i = 0; i < 8; ++i) s ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int N>
__global__ void k1(float* out, float a, float b) {
  float x[16];
  for (int i = 0; i < 16; ++i) x[i] = a + threadIdx.x + i;
  for (int it = 0; it < N; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %0;" : "+f"(x[i]) : "f"(b));
  float s = 0; for (int i = 0; i < 16; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  const int blocks = 148 * 8, threads = 256; const int N = 4096;
  uint64_t* o2; float* o1;
  cudaMalloc(&o2, blocks * threads * 8); cudaMalloc(&o1, blocks * threads * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); k1<N><<<blocks, threads>>>(o1, 1.0f, 0.999f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float t1; cudaEventElapsedTime(&t1, e0, e1);
    cudaEventRecord(e0); k2<N><<<blocks, threads>>>(o2, 0x3f8000003f800000ull, 0x3f7fbe773f7fbe77ull); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float t2; cudaEventElapsedTime(&t2, e0, e1);
    double n1 = (double)blocks * threads * N * 16, n2 = (double)blocks * threads * N * 8;  // instructions (thread level)
    printf("FFMA : %.3f ms, %.1f Tinst/s (thread), %.1f TFLOP/s\n", t1, n1 / t1 / 1e9, 2 * n1 / t1 / 1e9);
    printf("FFMA2: %.3f ms, %.1f Tinst/s (thread), %.1f TFLOP/s\n", t2, n2 / t2 / 1e9, 4 * n2 / t2 / 1e9);
  }
  return 0;
}
