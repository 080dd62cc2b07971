// Layout probe for the K-step sweep (K1 / §5): the production sweepk_kernel (this file
// includes fdtd_kernels.cu) on a config-4-sized fp32 grid (32768^2, K = 4, energy on, 4 warps per
// CTA, 256-row chunks), once with separate row-major arrays (8 allocations) and once with the
// tile-interleaved pools (fields ex|ey|hz per buffer, materials mea|msb; TILE = 64 columns).
// Same work, same arithmetic; only the addresses differ.  Prints ms per 4-step pass (CUDA events).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include
//        -I paper_1609_07114_b200/csrc -o /tmp/slp tools/sweep_layout_probe.cu
#include "../paper_1609_07114_b200/csrc/fdtd_kernels.cu"

#include <cstdio>
#include <vector>
#include <algorithm>
#include <cstdlib>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

__global__ void fill(float* a, size_t n, float base, float amp, uint32_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ seed;
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
    a[i] = base + amp * ((h & 0xffff) / 65536.f - 0.5f);
  }
}

int main(int argc, char** argv) {
  const int64_t nx = getenv("SLP_N") ? atoi(getenv("SLP_N")) : 32768, rows = nx, pitch = nx + 64;
  const bool k8 = getenv("SLP_K8") != nullptr;  // experiment: 8 steps per pass (V = 2, 4 halo lanes)
  const int row0 = k8 ? 16 : 8, nrows_alloc = (int)rows + row0 + 12;
  const int reps = argc > 1 ? atoi(argv[1]) : 10;
  const size_t tail = 32 * 1024 / 4;
  const size_t na1 = (size_t)nrows_alloc * pitch + tail;  // one row-major array
  std::vector<float*> bufs;
  auto alloc = [&](size_t n, float base, float amp) -> float* {
    float* p = nullptr;
    if (cudaMalloc(&p, n * sizeof(float)) != cudaSuccess) { printf("alloc failed\n"); exit(1); }
    fill<<<4096, 256>>>(p, n, base, amp, (uint32_t)bufs.size() * 7919u);
    bufs.push_back(p);
    return p;
  };
  // material terms: mea = eps0 eps_r / (2 dt) ~ 20, msb = sigma / 4 ~ 0.01; fields ~ 1e-3
  const double dt = 1e-12, dx = 1e-3;
  fdtd::SweepParams<float> base{};
  base.nx = nx; base.rows = (int)rows; base.row0 = row0; base.pitch = pitch;
  base.chunk = getenv("SLP_CHUNK") ? atoi(getenv("SLP_CHUNK")) : 256;
  const int warps = getenv("SLP_WARPS") ? atoi(getenv("SLP_WARPS")) : 4;
  base.chx = (float)(dt / (4e-7 * M_PI * dx)); base.chy = base.chx;
  base.src_row = -1; base.src_row_end = -1; base.src_col = -1;
  int64_t* d_step; CK(cudaMalloc(&d_step, 16)); CK(cudaMemset(d_step, 0, 16));
  base.step = d_step; base.src_meta = d_step;
  double* part; const int64_t npart = 4 * 256 * 1024; CK(cudaMalloc(&part, npart * 8 * 4));
  base.partials = getenv("SLP_NOENERGY") ? nullptr : part; base.pstride = npart;
  base.cap = 1;
  base.idx = (float)(1 / dx); base.idy = base.idx; base.wxy = (float)(dx * dx);
  base.wh = (float)(4e-7 * M_PI * dx * dx / dt);
  cudaStream_t st; CK(cudaStreamCreate(&st));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  auto launch = [&](const fdtd::SweepParams<float>& p) {
    if (!k8) {
      fdtd::launch_sweep<float>(p, 4, warps, st, 0, -1);
      return;
    }
    const int nch = (p.rows + p.chunk - 1) / p.chunk;
    const int64_t nvec = (p.nx + 1) / 2, nw = (nvec + 23) / 24;
    dim3 grid((unsigned)((nw + warps - 1) / warps), nch);
    const size_t smem = (size_t)warps * 8 * fdtd::NCOEF * 32 * 2 * sizeof(float);
    cudaFuncSetAttribute(fdtd::sweepk_kernel<float, 8, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    fdtd::sweepk_kernel<float, 8, 2, true><<<grid, 32 * warps, smem, st>>>(p);
  };
  auto timeit = [&](fdtd::SweepParams<float> p, const char* name) {
    for (int w = 0; w < 3; ++w) {
      launch(p);
      std::swap(p.ex0, *(const float**)&p.ex1); std::swap(p.ey0, *(const float**)&p.ey1);
      std::swap(p.hz0, *(const float**)&p.hz1);
    }
    cudaStreamSynchronize(st);
    float best = 1e9, sum = 0;
    std::vector<float> all;
    for (int r = 0; r < reps; ++r) {
      cudaEventRecord(e0, st);
      launch(p);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      best = std::min(best, ms); sum += ms; all.push_back(ms);
      std::swap(p.ex0, *(const float**)&p.ex1); std::swap(p.ey0, *(const float**)&p.ey1);
      std::swap(p.hz0, *(const float**)&p.hz1);
    }
    const cudaError_t e = cudaGetLastError();
    std::vector<float> srt = all;
    std::sort(srt.begin(), srt.end());
    printf("%-34s best %.3f ms  median %.3f  mean %.3f ms per 4-step pass  (%s)  %.1f G cell-steps/s\n", name, best,
           srt[reps / 2], sum / reps, cudaGetErrorString(e), (k8 ? 8.0 : 4.0) * nx * rows / (best * 1e-3) / 1e9);
    if (getenv("SLP_ALL")) {
      for (float v : all) printf(" %.2f", v);
      printf("\n");
    }
  };
  {  // separate arrays
    fdtd::SweepParams<float> p = base;
    p.naf = p.nam = 1;
    const float fa = getenv("SLP_ZERO") ? 0.f : 1e-3f;  // SLP_ZERO: all-zero fields (data-dependent power)
    p.ex0 = alloc(na1, 0.f, fa); p.ey0 = alloc(na1, 0.f, fa); p.hz0 = alloc(na1, 0.f, fa);
    p.ex1 = alloc(na1, 0.f, fa); p.ey1 = alloc(na1, 0.f, fa); p.hz1 = alloc(na1, 0.f, fa);
    p.mea = alloc(na1, 20.f, 10.f); p.msb = alloc(na1, 0.01f, 0.01f);
    p.alloc_elems_f = p.alloc_elems_m = (int64_t)na1;
    CK(cudaDeviceSynchronize());
    timeit(p, "separate row-major arrays");
    for (float* b : bufs) cudaFree(b);
    bufs.clear();
  }
  if (getenv("SLP_POOL")) {  // pools
    fdtd::SweepParams<float> p = base;
    p.naf = 3; p.nam = 2;
    const size_t nf = (size_t)nrows_alloc * pitch * 3 + tail, nm = (size_t)nrows_alloc * pitch * 2 + tail;
    float* f0 = alloc(nf, 0.f, 1e-3f); float* f1 = alloc(nf, 0.f, 1e-3f);
    float* m = alloc(nm, 20.f, 10.f);
    fill<<<4096, 256>>>(m, nm, 20.f, 10.f, 1u);
    // msb entries: every second tile of the material pool
    p.ex0 = f0; p.ey0 = f0 + fdtd::TILE; p.hz0 = f0 + 2 * fdtd::TILE;
    p.ex1 = f1; p.ey1 = f1 + fdtd::TILE; p.hz1 = f1 + 2 * fdtd::TILE;
    p.mea = m; p.msb = m + fdtd::TILE;
    p.alloc_elems_f = (int64_t)nf; p.alloc_elems_m = (int64_t)nm;
    CK(cudaDeviceSynchronize());
    timeit(p, "tile-interleaved pools (3 + 2)");
    for (float* b : bufs) cudaFree(b);
    bufs.clear();
  }
  return 0;
}
