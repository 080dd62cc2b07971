// Memory-pattern probe for the K-step sweep (K1): the same per-warp row walk (5 input
// arrays read, 3 output arrays written per row, register prefetch of row j+1 and an L2 prefetch
// of row j+1+PFD) with trivial arithmetic, to separate the HBM ceiling of that access pattern
// from the sweep's compute.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sp stream_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int V> struct Vec;
template <> struct Vec<2> { using t = float2; };
template <> struct Vec<4> { using t = float4; };

__device__ __forceinline__ void pf(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
__device__ __forceinline__ float2 ld(const float* p) { return __ldg(reinterpret_cast<const float2*>(p)); }

template <int V, int PFD>
__global__ void __launch_bounds__(256, 2) walk(const float* a0, const float* a1, const float* a2, const float* a3,
                                              const float* a4, float* o0, float* o1, float* o2, uint32_t P,
                                              int rows, int chunk, int nout) {
  using VT = typename Vec<V>::t;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  const uint32_t c = ((blockIdx.x * wpc + warp) * nout + lane) * V;
  const int r0 = blockIdx.y * chunk + 8, r1 = min(r0 + chunk, rows + 8);
  VT x0, x1, x2, x3, x4;
  auto L = [&](int j) {
    const uint32_t o = (uint32_t)j * P + c;
    x0 = __ldg(reinterpret_cast<const VT*>(a0 + o)); x1 = __ldg(reinterpret_cast<const VT*>(a1 + o));
    x2 = __ldg(reinterpret_cast<const VT*>(a2 + o)); x3 = __ldg(reinterpret_cast<const VT*>(a3 + o));
    x4 = __ldg(reinterpret_cast<const VT*>(a4 + o));
  };
  L(r0 - 4);
  for (int j = r0 - 4; j < r1; ++j) {
    VT y0 = x0, y1 = x1, y2 = x2, y3 = x3, y4 = x4;
    if (j + 1 < r1) L(j + 1);
    if (PFD > 0 && j + 1 + PFD < r1) {
      const uint32_t o = (uint32_t)(j + 1 + PFD) * P + c;
      pf(a0 + o); pf(a1 + o); pf(a2 + o); pf(a3 + o); pf(a4 + o);
    }
    if (j >= r0 && lane >= (V == 2 ? 2 : 1) && lane < (V == 2 ? 30 : 31)) {
      const uint32_t o = (uint32_t)(j - 3) * P + c;
      VT s;
      s.x = y0.x + y1.x * y3.x; s.y = y0.y + y1.y * y3.y;
      *reinterpret_cast<VT*>(o0 + o) = s;
      s.x = y2.x * y4.x; s.y = y2.y - y4.y;
      *reinterpret_cast<VT*>(o1 + o) = s;
      s.x = y1.x + y2.x; s.y = y3.y + y0.y;
      *reinterpret_cast<VT*>(o2 + o) = s;
    }
  }
}

// tile-interleaved layout: per row, tiles of TW columns; a tile holds the NA arrays' TW-column
// segments back to back (in pool: ex, ey, hz, ma, ms; out pool: ex, ey, hz)
template <int PFD, int TW>
__global__ void __launch_bounds__(256, 2) walk_il(const float* in, float* out, uint32_t ntile, int rows, int chunk,
                                                 int nout) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  const uint32_t c = ((blockIdx.x * wpc + warp) * nout + lane) * 2;
  const uint32_t t = c / TW, w = c % TW;
  const int r0 = blockIdx.y * chunk + 8, r1 = min(r0 + chunk, rows + 8);
  float2 x0, x1, x2, x3, x4;
  auto base_in = [&](int j) { return ((uint32_t)j * ntile + t) * (5 * TW) + w; };
  auto L = [&](int j) {
    const float* p = in + base_in(j);
    x0 = ld(p); x1 = ld(p + TW); x2 = ld(p + 2 * TW); x3 = ld(p + 3 * TW); x4 = ld(p + 4 * TW);
  };
  L(r0 - 4);
  for (int j = r0 - 4; j < r1; ++j) {
    float2 y0 = x0, y1 = x1, y2 = x2, y3 = x3, y4 = x4;
    if (j + 1 < r1) L(j + 1);
    if (PFD > 0 && j + 1 + PFD < r1) {
      const float* p = in + base_in(j + 1 + PFD);
      pf(p); pf(p + TW); pf(p + 2 * TW); pf(p + 3 * TW); pf(p + 4 * TW);
    }
    if (j >= r0 && lane >= 2 && lane < 30) {
      float* q = out + ((uint32_t)(j - 3) * ntile + t) * (3 * TW) + w;
      float2 s;
      s.x = y0.x + y1.x * y3.x; s.y = y0.y + y1.y * y3.y;
      *reinterpret_cast<float2*>(q) = s;
      s.x = y2.x * y4.x; s.y = y2.y - y4.y;
      *reinterpret_cast<float2*>(q + TW) = s;
      s.x = y1.x + y2.x; s.y = y3.y + y0.y;
      *reinterpret_cast<float2*>(q + 2 * TW) = s;
    }
  }
}

// block-major ("strip") layout: each array stored as [block][row][BW] with BW = the stored width of
// one warp strip (28 lanes x 2 = 56 columns), so a warp walking its rows reads one contiguous stream
// per array (lanes 2..29) plus two 8-byte pieces of each neighbour block (its halo lanes).  R rows
// per block (ny + 16 padded); block -1 and nblk exist (zero) so that the halo lanes of the edge
// warps load unconditionally.
template <int PFD>
__global__ void __launch_bounds__(256, 2) walk_blk(const float* a0, const float* a1, const float* a2, const float* a3,
                                                  const float* a4, float* o0, float* o1, float* o2, uint32_t R,
                                                  int rows, int chunk) {
  constexpr int BW = 56;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  const int blk = blockIdx.x * wpc + warp + 1;  // +1: block -1 is the front pad
  const int bl = blk + (lane < 2 ? -1 : lane >= 30 ? 1 : 0);
  const int off = lane < 2 ? 52 + 2 * lane : lane >= 30 ? 2 * (lane - 30) : 2 * (lane - 2);
  const uint32_t c = (uint32_t)bl * R * BW + off;  // element of row 0
  const uint32_t cs = (uint32_t)blk * R * BW + 2 * (lane - 2);
  const int r0 = blockIdx.y * chunk + 8, r1 = min(r0 + chunk, rows + 8);
  float2 x0, x1, x2, x3, x4;
  auto L = [&](int j) {
    const uint32_t o = (uint32_t)j * BW + c;
    x0 = ld(a0 + o); x1 = ld(a1 + o); x2 = ld(a2 + o); x3 = ld(a3 + o); x4 = ld(a4 + o);
  };
  L(r0 - 4);
  for (int j = r0 - 4; j < r1; ++j) {
    float2 y0 = x0, y1 = x1, y2 = x2, y3 = x3, y4 = x4;
    if (j + 1 < r1) L(j + 1);
    if (PFD > 0 && j + 1 + PFD < r1) {
      const uint32_t o = (uint32_t)(j + 1 + PFD) * BW + c;
      pf(a0 + o); pf(a1 + o); pf(a2 + o); pf(a3 + o); pf(a4 + o);
    }
    if (j >= r0 && lane >= 2 && lane < 30) {
      const uint32_t o = (uint32_t)(j - 3) * BW + cs;
      float2 s;
      s.x = y0.x + y1.x * y3.x; s.y = y0.y + y1.y * y3.y;
      *reinterpret_cast<float2*>(o0 + o) = s;
      s.x = y2.x * y4.x; s.y = y2.y - y4.y;
      *reinterpret_cast<float2*>(o1 + o) = s;
      s.x = y1.x + y2.x; s.y = y3.y + y0.y;
      *reinterpret_cast<float2*>(o2 + o) = s;
    }
  }
}

__global__ void copyk(const float4* a, float4* b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
  const int nx = 32768, ny = 32768, P = nx + 64;
  const size_t n = (size_t)P * (ny + 16);
  float* buf[8];
  for (int i = 0; i < 8; ++i) {
    if (cudaMalloc(&buf[i], n * 4) != cudaSuccess) { printf("oom\n"); return 1; }
    cudaMemset(buf[i], 0, n * 4);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto time = [&](auto&& f, const char* name, double bytes) {
    for (int w = 0; w < 3; ++w) f();
    cudaEventRecord(e0);
    for (int it = 0; it < 10; ++it) f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 10;
    cudaError_t err = cudaGetLastError();
    printf("%-28s %8.3f ms  %7.1f GB/s %s\n", name, ms, bytes / ms / 1e6, err ? cudaGetErrorString(err) : "");
  };
  const double bytes = 32.0 * nx * (double)ny;
  for (int chunk : {256}) {
    for (int wpc : {4}) {
      const int nout = 28;
      dim3 g((nx / 2 + nout * wpc - 1) / (nout * wpc), ny / chunk);
      char nm[64];
      snprintf(nm, 64, "walk V2 pfd1 ch%d w%d", chunk, wpc);
      time([&] { walk<2, 1><<<g, wpc * 32>>>(buf[0], buf[1], buf[2], buf[3], buf[4], buf[5], buf[6], buf[7], P, ny, chunk, nout); }, nm, bytes);
      snprintf(nm, 64, "walk V2 pfd0 ch%d w%d", chunk, wpc);
      time([&] { walk<2, 0><<<g, wpc * 32>>>(buf[0], buf[1], buf[2], buf[3], buf[4], buf[5], buf[6], buf[7], P, ny, chunk, nout); }, nm, bytes);
      snprintf(nm, 64, "walk V2 pfd2 ch%d w%d", chunk, wpc);
      time([&] { walk<2, 2><<<g, wpc * 32>>>(buf[0], buf[1], buf[2], buf[3], buf[4], buf[5], buf[6], buf[7], P, ny, chunk, nout); }, nm, bytes);
    }
  }
  {
    const int nout = 28, wpc = 4, chunk = 256;
    dim3 g((nx / 2 + nout * wpc - 1) / (nout * wpc), ny / chunk);
    const uint32_t nt64 = (P + 63) / 64, nt256 = (P + 255) / 256, nt1k = (P + 1023) / 1024;
    float *pin, *pout;
    const size_t nil = (size_t)(ny + 16) * nt1k * 1024;
    if (cudaMalloc(&pin, nil * 5 * 4) != cudaSuccess || cudaMalloc(&pout, nil * 3 * 4) != cudaSuccess) { printf("oom\n"); return 1; }
    cudaMemset(pin, 0, nil * 20); cudaMemset(pout, 0, nil * 12);
    time([&] { walk_il<1, 64><<<g, wpc * 32>>>(pin, pout, nt64, ny, chunk, nout); }, "il64 pfd1", bytes);
    time([&] { walk_il<2, 64><<<g, wpc * 32>>>(pin, pout, nt64, ny, chunk, nout); }, "il64 pfd2", bytes);
    time([&] { walk_il<1, 256><<<g, wpc * 32>>>(pin, pout, nt256, ny, chunk, nout); }, "il256 pfd1", bytes);
    time([&] { walk_il<2, 256><<<g, wpc * 32>>>(pin, pout, nt256, ny, chunk, nout); }, "il256 pfd2", bytes);
    time([&] { walk_il<0, 256><<<g, wpc * 32>>>(pin, pout, nt256, ny, chunk, nout); }, "il256 pfd0", bytes);
    time([&] { walk_il<2, 1024><<<g, wpc * 32>>>(pin, pout, nt1k, ny, chunk, nout); }, "il1k pfd2", bytes);
    for (int pfd = 3; pfd <= 4; ++pfd) {
      dim3 g2((nx / 2 + nout * wpc - 1) / (nout * wpc), ny / chunk);
      if (pfd == 3) time([&] { walk<2, 3><<<g2, wpc * 32>>>(buf[0], buf[1], buf[2], buf[3], buf[4], buf[5], buf[6], buf[7], P, ny, chunk, nout); }, "walk V2 pfd3 ch256 w4", bytes);
      else time([&] { walk<2, 4><<<g2, wpc * 32>>>(buf[0], buf[1], buf[2], buf[3], buf[4], buf[5], buf[6], buf[7], P, ny, chunk, nout); }, "walk V2 pfd4 ch256 w4", bytes);
    }
  }
  {
    const int nout = 30, wpc = 4, chunk = 256;  // V = 4: 16-byte vectors, one halo lane per side
    dim3 g((nx / 4 + nout * wpc - 1) / (nout * wpc), ny / chunk);
    time([&] { walk<4, 1><<<g, wpc * 32>>>(buf[0], buf[1], buf[2], buf[3], buf[4], buf[5], buf[6], buf[7], P, ny, chunk, nout); }, "walk V4 pfd1 ch256 w4", bytes);
    time([&] { walk<4, 0><<<g, wpc * 32>>>(buf[0], buf[1], buf[2], buf[3], buf[4], buf[5], buf[6], buf[7], P, ny, chunk, nout); }, "walk V4 pfd0 ch256 w4", bytes);
    time([&] { walk<4, 2><<<g, wpc * 32>>>(buf[0], buf[1], buf[2], buf[3], buf[4], buf[5], buf[6], buf[7], P, ny, chunk, nout); }, "walk V4 pfd2 ch256 w4", bytes);
  }
  {  // block-major layout (walk_blk): 32768 / 56 = 586 blocks (+2 pad), R = ny + 16 rows each
    const int wpc = 4;
    const uint32_t R = ny + 16, nblk = (nx + 55) / 56;
    const size_t nb = (size_t)(nblk + 8) * R * 56;  // the grid rounds the blocks up to whole CTAs
    float* bb[8];
    for (int i = 0; i < 8; ++i) {
      if (cudaMalloc(&bb[i], nb * 4) != cudaSuccess) { printf("oom\n"); return 1; }
      cudaMemset(bb[i], 0, nb * 4);
    }
    for (int chunk : {256, 512, 2048}) {
      dim3 g((nblk + wpc - 1) / wpc, ny / chunk);
      char nm[64];
      snprintf(nm, 64, "blk56 pfd1 ch%d w4", chunk);
      time([&] { walk_blk<1><<<g, wpc * 32>>>(bb[0], bb[1], bb[2], bb[3], bb[4], bb[5], bb[6], bb[7], R, ny, chunk); }, nm, bytes);
      snprintf(nm, 64, "blk56 pfd2 ch%d w4", chunk);
      time([&] { walk_blk<2><<<g, wpc * 32>>>(bb[0], bb[1], bb[2], bb[3], bb[4], bb[5], bb[6], bb[7], R, ny, chunk); }, nm, bytes);
      snprintf(nm, 64, "blk56 pfd0 ch%d w4", chunk);
      time([&] { walk_blk<0><<<g, wpc * 32>>>(bb[0], bb[1], bb[2], bb[3], bb[4], bb[5], bb[6], bb[7], R, ny, chunk); }, nm, bytes);
    }
    for (int i = 0; i < 8; ++i) cudaFree(bb[i]);
  }
  time([&] { copyk<<<148 * 8, 512>>>((const float4*)buf[0], (float4*)buf[5], n / 4); }, "copy (1 in 1 out)", 8.0 * n);
  return 0;
}
