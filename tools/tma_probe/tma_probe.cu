// Minimal TMA (cp.async.bulk.tensor 2D) probe: one box from a device array into shared memory,
// tensor map in global memory (variant 0) or as a __grid_constant__ kernel parameter (variant 1).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void probe_global(const CUtensorMap* map, float* out, int x, int y, int W, int H) {
  __shared__ __align__(128) float buf[64 * 64];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)),
                 "r"((uint32_t)(W * H * 4)) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"((uint32_t)__cvta_generic_to_shared(buf)), "l"((uint64_t)map), "r"(x), "r"(y),
                 "r"((uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
  }
  asm volatile("{\n .reg .pred P;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n @!P bra W_%=;\n}"
               ::"r"((uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
  for (int i = threadIdx.x; i < W * H; i += blockDim.x) out[i] = buf[i];
}

template <int V>
__global__ void probe_var(const __grid_constant__ CUtensorMap map, float* out, int x, int y, int W, int H) {
  __shared__ __align__(128) float buf[64 * 64];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    if (V & 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (V & 2) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)),
                 "r"((uint32_t)(W * H * 4)) : "memory");
    if (V & 4)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"((uint32_t)__cvta_generic_to_shared(buf)), "l"((uint64_t)&map), "r"(x), "r"(y),
                 "r"((uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"((uint32_t)__cvta_generic_to_shared(buf)), "l"((uint64_t)&map), "r"(x), "r"(y),
                 "r"((uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
  }
  uint32_t ph = 0;
  asm volatile("{\n .reg .pred P;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra W_%=;\n}"
               ::"r"((uint32_t)__cvta_generic_to_shared(&bar)), "r"(ph) : "memory");
  for (int i = threadIdx.x; i < W * H; i += blockDim.x) out[i] = buf[i];
}

__global__ void probe_param(const __grid_constant__ CUtensorMap map, float* out, int x, int y, int W, int H) {
  __shared__ __align__(128) float buf[64 * 64];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)),
                 "r"((uint32_t)(W * H * 4)) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"((uint32_t)__cvta_generic_to_shared(buf)), "l"((uint64_t)&map), "r"(x), "r"(y),
                 "r"((uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
  }
  asm volatile("{\n .reg .pred P;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n @!P bra W_%=;\n}"
               ::"r"((uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
  for (int i = threadIdx.x; i < W * H; i += blockDim.x) out[i] = buf[i];
}

int main() {
  const int pitch = 256, rows = 64, W = 16, H = 15, x = 5, y = 7;
  std::vector<float> h(pitch * rows);
  for (int i = 0; i < pitch * rows; ++i) h[i] = (float)i;
  float *d, *o;
  cudaMalloc(&d, h.size() * 4);
  cudaMalloc(&o, W * H * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {pitch, rows}, str[1] = {pitch * 4};
  int bh = getenv("BH") ? atoi(getenv("BH")) : H;
  cuuint32_t box[2] = {W, (cuuint32_t)bh}, es[2] = {1, 1};
  if (getenv("DIRECT")) enc = (PFN_cuTensorMapEncodeTiled_v12000)cuTensorMapEncodeTiled;
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, getenv("NOPROMO") ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("desc:"); for (int i = 0; i < 16; ++i) printf(" %016llx", (unsigned long long)((unsigned long long*)&tm)[i]); printf("\n");
  printf("encode %d (entry %d)\n", (int)r, (int)q);
  {
    int v = 0;
    if (getenv("V")) v = atoi(getenv("V"));
    cudaMemset(o, 0, W * H * 4);
    switch (v) {
      case 0: probe_var<0><<<1, 128>>>(tm, o, x, y, W, H); break;
      case 1: probe_var<1><<<1, 128>>>(tm, o, x, y, W, H); break;
      case 2: probe_var<2><<<1, 128>>>(tm, o, x, y, W, H); break;
      case 4: probe_var<4><<<1, 128>>>(tm, o, x, y, W, H); break;
      case 8: {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(1); cfg.blockDim = dim3(128);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        printf("launch %s\n", cudaGetErrorString(cudaLaunchKernelEx(&cfg, probe_var<4>, tm, o, x, y, W, H)));
        break;
      }
      case 5: probe_var<5><<<1, 128>>>(tm, o, x, y, W, H); break;
      case 6: probe_var<6><<<1, 128>>>(tm, o, x, y, W, H); break;
    }
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> ho(W * H);
    cudaMemcpy(ho.data(), o, ho.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int vv = 0; vv < H; ++vv)
      for (int u = 0; u < W; ++u) bad += ho[vv * W + u] != h[(y + vv) * pitch + x + u];
    printf("V=%d: %s, mismatches %d\n", v, cudaGetErrorString(e), bad);
    return 0;
  }
  for (int variant = 1; variant >= 0; --variant) {
    cudaMemset(o, 0, W * H * 4);
    if (variant == 0) {
      CUtensorMap* dm;
      cudaMalloc(&dm, sizeof tm);
      cudaMemcpy(dm, &tm, sizeof tm, cudaMemcpyHostToDevice);
      probe_global<<<1, 128>>>(dm, o, x, y, W, H);
    } else {
      probe_param<<<1, 128>>>(tm, o, x, y, W, H);
    }
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> ho(W * H);
    cudaMemcpy(ho.data(), o, ho.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int v = 0; v < H; ++v)
      for (int u = 0; u < W; ++u) bad += ho[v * W + u] != h[(y + v) * pitch + x + u];
    printf("variant %s: %s, mismatches %d\n", variant ? "param" : "global", cudaGetErrorString(e), bad);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
