// Isolate: mbarrier alone (V=0), mbarrier + 1D bulk copy (V=1), + expect_tx only (V=2)
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
template <int V>
__global__ void k(const float* src, float* out) {
  __shared__ __align__(128) float buf[256];
  __shared__ __align__(8) unsigned long long bar;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (V == 0) {
      asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(b) : "memory");
    } else {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(V == 1 ? 1024 : 0) : "memory");
      if (V == 1)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"((uint32_t)__cvta_generic_to_shared(buf)), "l"(src), "r"(1024), "r"(b) : "memory");
    }
  }
  uint32_t ph = 0;
  asm volatile("{\n .reg .pred P;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra W_%=;\n}"
               ::"r"(b), "r"(ph) : "memory");
  for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = buf[i];
}
int main() {
  float *s, *o;
  cudaMalloc(&s, 4096); cudaMalloc(&o, 4096);
  cudaMemset(s, 0, 4096);
  int v = getenv("V") ? atoi(getenv("V")) : 0;
  if (v == 0) k<0><<<1, 128>>>(s, o); else if (v == 1) k<1><<<1, 128>>>(s, o); else k<2><<<1, 128>>>(s, o);
  printf("V=%d %s\n", v, cudaGetErrorString(cudaDeviceSynchronize()));
}
