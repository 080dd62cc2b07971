// CUDA kernels of the hot path (sm_100a).  See DESIGN.md for the derivations.
//
//  K1 sweep_kernel : one pass over the grid per time step.  For every owned cell row it
//                    computes Hz^{n+1/2} (eq:updateH), adds the soft
//                    source, then the E^{n+1} of that row's x- and y-directed edges
//                    (eq:updateEx L209-214 and its Ey analogue L223) from the new Hz of
//                    this row and the row below (kept in registers).  16-byte vector
//                    loads, one warp per 32x16-byte column strip, rows walked upward by
//                    each CTA over a chunk; ping-pong buffers so no CTA ever reads a value
//                    another CTA writes in the same launch.  Edge masks (PEC, ROM holes,
//                    ROM interfaces) are encoded in the coefficients (ca = 1, cb = 0).
//  K3 post_kernel  : per ROM instance (one CTA each) the factored eq:connExplicit update
//                    (gather h, y; reduced matvecs; Schur solve; scatter y^{n+1});
//                    one CTA records the probes; the last CTA to finish reduces the
//                    energy partials in a fixed order and advances the step counter.
#include "fdtd_kernels.cuh"

#include <cstdio>

namespace fdtd {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr double MU0 = 4.0e-7 * 3.14159265358979323846;
constexpr double C0 = 299792458.0;
constexpr double EPS0 = 1.0 / (MU0 * C0 * C0);
constexpr int64_t IDX_MASK = (int64_t(1) << 62) - 1;

template <typename T> struct VT;
template <> struct VT<float> { static constexpr int N = 4; };
template <> struct VT<double> { static constexpr int N = 2; };

__device__ __forceinline__ void ldv(const float* p, float (&v)[4]) {
  const float4 x = __ldg(reinterpret_cast<const float4*>(p));
  v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
}
__device__ __forceinline__ void ldv(const double* p, double (&v)[2]) {
  const double2 x = __ldg(reinterpret_cast<const double2*>(p));
  v[0] = x.x; v[1] = x.y;
}
__device__ __forceinline__ void stv(float* p, const float (&v)[4]) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
__device__ __forceinline__ void stv(double* p, const double (&v)[2]) {
  *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
}
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }

// eq:updateH divided by dx dy mu / dt:  Hz' = Hz + chy (Ex_{j+1} - Ex_j) - chx (Ey_{i+1} - Ey_i).
// Explicit fused operations pin the rounding, so the redundant recomputations at warp and
// chunk edges are bit-identical to the owner's value (needed for 1-GPU == N-GPU fields).
template <typename T>
__device__ __forceinline__ T hupd(T hz, T exn, T exc, T eyr, T eyl, T chy, T chx) {
  return fma_rn(-chx, eyr - eyl, fma_rn(chy, exn - exc, hz));
}

// Reciprocal of an edge's (eps/dt + sigma/2): fp32 uses the single-instruction MUFU
// approximation (max relative error ~2^-23, deterministic); fp64 the correctly rounded one.
__device__ __forceinline__ float rcp_rn(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ double rcp_rn(double x) { return __drcp_rn(x); }

// E half-step of one edge from the two adjacent cells' material terms (eq:updateEx divided by
// its left-hand coefficient):  E' = [(a - s) E + dH / l] / (a + s),  a = eps/dt, s = sigma/2 of
// the edge (arithmetic means, R2), l = the dual length.  An edge next to a cell with a < 0
// (ROM hole, PEC wall, padding) keeps its value (PEC edges stay 0; interface edges are
// written by the ROM kernel).
template <typename T>
__device__ __forceinline__ T eupd(T e, T dh_over_l, T a0, T s0, T a1, T s1, bool& live, T& a) {
  a = a0 + a1;
  const T s = s0 + s1;
  live = (a0 >= T(0)) & (a1 >= T(0));
  const T r = rcp_rn(a + s);
  const T v = mul_rn(r, fma_rn(a - s, e, dh_over_l));
  return live ? v : e;
}

// Cells outside the live grid (ROM hole, ghost row below the grid, padding) keep their Hz.
template <typename T>
__device__ __forceinline__ T hmask(T mea_cell, T hold, T hnew) {
  return mea_cell < T(0) ? hold : hnew;
}

template <typename T, bool ENERGY>
__global__ void __launch_bounds__(256) sweep_kernel(const SweepParams<T> p) {
  constexpr int V = VT<T>::N;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int wpc = blockDim.x >> 5;
  const int colv = (blockIdx.x * wpc + warp) * 32 + lane;
  const bool act = colv < p.ncolv;
  const int64_t c = (int64_t)colv * V;
  const int cy = p.chunk0 + blockIdx.y;  // row chunk
  const int r0 = p.row0 + cy * p.chunk;
  const int r1 = min(r0 + p.chunk, p.row0 + p.rows);
  const int64_t P = p.pitch;

  T src = T(0);
  if (p.src_row >= 0) {
    const int64_t k = *p.step - p.src_t0;
    if (k >= 0 && k < p.src_n) src = (T)p.src_samples[k];
  }

  // carried between rows: Ex^n of edge row j, Hz^{n+1/2} of cell row j-1, materials of row j-1
  T exc[V], hzp[V], mpa[V], mps[V], exn[V], eyv[V], hzv[V], ma[V], ms[V];
  T excl = T(0);
  // ---- prologue: row r0-1 (recomputed; the ghost row when r0 == 1)
  {
    const int64_t rj = (int64_t)(r0 - 1) * P;
    T exl[V];
#pragma unroll
    for (int k = 0; k < V; ++k) exl[k] = exn[k] = eyv[k] = hzv[k] = mpa[k] = mps[k] = T(0);
    if (act) {
      ldv(p.ex0 + rj + c, exl);
      ldv(p.ex0 + rj + P + c, exn);
      ldv(p.ey0 + rj + c, eyv);
      ldv(p.hz0 + rj + c, hzv);
      ldv(p.mea + rj + c, mpa);
      ldv(p.msb + rj + c, mps);
    }
    T eyr = __shfl_down_sync(FULL, eyv[0], 1);
    if (lane == 31) eyr = (act && colv + 1 < p.ncolv) ? __ldg(p.ey0 + rj + c + V) : T(0);
#pragma unroll
    for (int k = 0; k < V; ++k)
      hzp[k] = hmask(mpa[k], hzv[k], hupd(hzv[k], exn[k], exl[k], k + 1 < V ? eyv[k + 1] : eyr, eyv[k], p.chy, p.chx));
    if (r0 - 1 == p.src_row) {
#pragma unroll
      for (int k = 0; k < V; ++k)
        if (c + k == p.src_col) hzp[k] += src;
    }
#pragma unroll
    for (int k = 0; k < V; ++k) exc[k] = exn[k];
    if (lane == 0 && act && c > 0) excl = __ldg(p.ex0 + rj + P + c - 1);
  }

  double eacc = 0.0;
  for (int j = r0; j < r1; ++j) {
    const int64_t rj = (int64_t)j * P;
    const int64_t rn = rj + P;
#pragma unroll
    for (int k = 0; k < V; ++k) exn[k] = eyv[k] = hzv[k] = ma[k] = ms[k] = T(0);
    if (act) {
      ldv(p.ex0 + rn + c, exn);
      ldv(p.ey0 + rj + c, eyv);
      ldv(p.hz0 + rj + c, hzv);
      ldv(p.mea + rj + c, ma);
      ldv(p.msb + rj + c, ms);
    }
    T lhz = T(0), lexn = T(0), ley = T(0), lma = T(-1), lms = T(0);
    if (lane == 0 && act && c > 0) {
      lhz = __ldg(p.hz0 + rj + c - 1);
      lexn = __ldg(p.ex0 + rn + c - 1);
      ley = __ldg(p.ey0 + rj + c - 1);
      lma = __ldg(p.mea + rj + c - 1);
      lms = __ldg(p.msb + rj + c - 1);
    }
    T eyr = __shfl_down_sync(FULL, eyv[0], 1);
    if (lane == 31) eyr = (act && colv + 1 < p.ncolv) ? __ldg(p.ey0 + rj + c + V) : T(0);
    T hzn[V];
#pragma unroll
    for (int k = 0; k < V; ++k)
      hzn[k] = hmask(ma[k], hzv[k], hupd(hzv[k], exn[k], exc[k], k + 1 < V ? eyv[k + 1] : eyr, eyv[k], p.chy, p.chx));
    if (j == p.src_row) {  // S2: soft source after the H half-step
#pragma unroll
      for (int k = 0; k < V; ++k)
        if (c + k == p.src_col) hzn[k] += src;
    }
    T hl = __shfl_up_sync(FULL, hzn[V - 1], 1);
    T la = __shfl_up_sync(FULL, ma[V - 1], 1);
    T ls = __shfl_up_sync(FULL, ms[V - 1], 1);
    if (lane == 0) {
      if (c > 0) {
        hl = hmask(lma, lhz, hupd(lhz, lexn, excl, eyv[0], ley, p.chy, p.chx));
        if (j == p.src_row && c - 1 == p.src_col) hl += src;
      } else {
        hl = T(0);  // Ey column 0 is the PEC wall (lma = -1 keeps it at 0)
      }
      la = lma;
      ls = lms;
      excl = lexn;
    }
    T exo[V], eyo[V];
    T e = T(0);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      bool lx, ly;
      T ax, ay;
      // Ex edge (row j, column c+k): cells (c+k, j-1) and (c+k, j)
      exo[k] = eupd(exc[k], mul_rn(p.idy, hzn[k] - hzp[k]), mpa[k], mps[k], ma[k], ms[k], lx, ax);
      // Ey edge (row j, column c+k): cells (c+k-1, j) and (c+k, j)
      const T hleft = k ? hzn[k - 1] : hl;
      eyo[k] = eupd(eyv[k], -mul_rn(p.idx, hzn[k] - hleft), k ? ma[k - 1] : la, k ? ms[k - 1] : ls, ma[k], ms[k],
                    ly, ay);
      if (ENERGY) {  // S3: (1/dt)[C E^2 + mu A H^{n-1/2} H^{n+1/2}], C/dt = dx dy a
        e += p.wxy * ((lx ? ax * exc[k] * exc[k] : T(0)) + (ly ? ay * eyv[k] * eyv[k] : T(0)));
        e += p.wh * hzv[k] * hzn[k];
      }
    }
    if (act) {
      stv(p.hz1 + rj + c, hzn);
      stv(p.ex1 + rj + c, exo);
      stv(p.ey1 + rj + c, eyo);
    }
    if (ENERGY) eacc += (double)e;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      exc[k] = exn[k];
      hzp[k] = hzn[k];
      mpa[k] = ma[k];
      mps[k] = ms[k];
    }
  }
  if (ENERGY) {
    __shared__ double red[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) eacc += __shfl_down_sync(FULL, eacc, o);
    if (lane == 0) red[warp] = eacc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < wpc; ++w) s += red[w];
      p.partials[(int64_t)cy * gridDim.x + blockIdx.x] = s;
    }
  }
}

// K1b: two time steps per pass.  At row j the warp advances
// step n on row j and step n+1 on row j-1 entirely in registers, so each field and material
// byte crosses HBM once per two steps.  Lanes 0 and 31 are redundant halo lanes (their
// leftmost / rightmost values may be wrong after the first step, which only they use); lanes
// 1..30 store.  Interface edges are treated as frozen (masked) in both steps; the fix-up
// kernel (post2) repairs the cells and edges next to every ROM instance.
template <typename T, bool ENERGY>
__global__ void __maxnreg__(96) sweep2_kernel(const SweepParams<T> p) {
  constexpr int V = VT<T>::N;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int wpc = blockDim.x >> 5;
  const int colv = (blockIdx.x * wpc + warp) * 30 + lane - 1;
  const bool act = colv >= 0 && colv < p.ncolv;
  const bool out = act && lane >= 1 && lane <= 30;
  const int64_t c = (int64_t)colv * V;
  const int cy = p.chunk0 + blockIdx.y;  // row chunk
  const int r0 = p.row0 + cy * p.chunk;
  const int r1 = min(r0 + p.chunk, p.row0 + p.rows);
  const int64_t P = p.pitch;

  T g0 = T(0), g1 = T(0);
  if (p.src_row >= 0) {
    const int64_t k = *p.step - p.src_t0;
    if (k >= 0 && k < p.src_n) g0 = (T)p.src_samples[k];
    if (k + 1 >= 0 && k + 1 < p.src_n) g1 = (T)p.src_samples[k + 1];
  }
  auto load_row = [&](const T* a, int row, T (&v)[V], T fill) {
#pragma unroll
    for (int k = 0; k < V; ++k) v[k] = fill;
    if (act && row >= 0) ldv(a + (int64_t)row * P + c, v);
  };

  T exc[V], h1p[V], ma1[V], ms1[V], ma2[V], ms2[V], e1c[V], y1c[V], h2p[V];
  // ---- prologue: step n on rows r0-2 (Hz only) and r0-1 (Hz, Ex, Ey)
  {
    T hA[V], exA[V], eyA[V], hB[V], exB[V], eyB[V], exC[V];
    load_row(p.hz0, r0 - 2, hA, T(0));
    load_row(p.ex0, r0 - 2, exA, T(0));
    load_row(p.ey0, r0 - 2, eyA, T(0));
    load_row(p.mea, r0 - 2, ma2, T(-1));
    load_row(p.msb, r0 - 2, ms2, T(0));
    load_row(p.hz0, r0 - 1, hB, T(0));
    load_row(p.ex0, r0 - 1, exB, T(0));
    load_row(p.ey0, r0 - 1, eyB, T(0));
    load_row(p.mea, r0 - 1, ma1, T(-1));
    load_row(p.msb, r0 - 1, ms1, T(0));
    load_row(p.ex0, r0, exC, T(0));
    T rA = __shfl_down_sync(FULL, eyA[0], 1);
    T rB = __shfl_down_sync(FULL, eyB[0], 1);
    T h1a[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
      h1a[k] = hmask(ma2[k], hA[k], hupd(hA[k], exB[k], exA[k], k + 1 < V ? eyA[k + 1] : rA, eyA[k], p.chy, p.chx));
      h1p[k] = hmask(ma1[k], hB[k], hupd(hB[k], exC[k], exB[k], k + 1 < V ? eyB[k + 1] : rB, eyB[k], p.chy, p.chx));
    }
    if (r0 - 2 == p.src_row) {
#pragma unroll
      for (int k = 0; k < V; ++k)
        if (c + k == p.src_col) h1a[k] += g0;
    }
    if (r0 - 1 == p.src_row) {
#pragma unroll
      for (int k = 0; k < V; ++k)
        if (c + k == p.src_col) h1p[k] += g0;
    }
    const T hl = __shfl_up_sync(FULL, h1p[V - 1], 1);
    const T la = __shfl_up_sync(FULL, ma1[V - 1], 1);
    const T ls = __shfl_up_sync(FULL, ms1[V - 1], 1);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      bool l;
      T a;
      e1c[k] = eupd(exB[k], mul_rn(p.idy, h1p[k] - h1a[k]), ma2[k], ms2[k], ma1[k], ms1[k], l, a);
      const T left = k ? h1p[k - 1] : hl;
      y1c[k] = eupd(eyB[k], -mul_rn(p.idx, h1p[k] - left), k ? ma1[k - 1] : la, k ? ms1[k - 1] : ls, ma1[k], ms1[k],
                    l, a);
      exc[k] = exC[k];
      h2p[k] = T(0);
    }
  }

  double eacc0 = 0.0, eacc1 = 0.0;
  // software pipeline: the loads of row j+1 are in flight while row j computes
  T nexn[V], neyv[V], nhzv[V], nma[V], nms[V];
  load_row(p.ex0, r0 + 1, nexn, T(0));
  load_row(p.ey0, r0, neyv, T(0));
  load_row(p.hz0, r0, nhzv, T(0));
  load_row(p.mea, r0, nma, T(-1));
  load_row(p.msb, r0, nms, T(0));
  for (int j = r0; j <= r1; ++j) {
    T exn[V], eyv[V], hzv[V], ma[V], ms[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
      exn[k] = nexn[k]; eyv[k] = neyv[k]; hzv[k] = nhzv[k]; ma[k] = nma[k]; ms[k] = nms[k];
    }
    if (j < r1) {
      load_row(p.ex0, j + 2, nexn, T(0));
      load_row(p.ey0, j + 1, neyv, T(0));
      load_row(p.hz0, j + 1, nhzv, T(0));
      load_row(p.mea, j + 1, nma, T(-1));
      load_row(p.msb, j + 1, nms, T(0));
    }
    // ---- step n on row j
    const T eyr = __shfl_down_sync(FULL, eyv[0], 1);
    T h1[V];
#pragma unroll
    for (int k = 0; k < V; ++k)
      h1[k] = hmask(ma[k], hzv[k], hupd(hzv[k], exn[k], exc[k], k + 1 < V ? eyv[k + 1] : eyr, eyv[k], p.chy, p.chx));
    if (j == p.src_row) {
#pragma unroll
      for (int k = 0; k < V; ++k)
        if (c + k == p.src_col) h1[k] += g0;
    }
    const T hl = __shfl_up_sync(FULL, h1[V - 1], 1);
    const T la = __shfl_up_sync(FULL, ma[V - 1], 1);
    const T ls = __shfl_up_sync(FULL, ms[V - 1], 1);
    T e1[V], y1[V];
    T en = T(0);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      bool lx, ly;
      T ax, ay;
      e1[k] = eupd(exc[k], mul_rn(p.idy, h1[k] - h1p[k]), ma1[k], ms1[k], ma[k], ms[k], lx, ax);
      const T left = k ? h1[k - 1] : hl;
      y1[k] = eupd(eyv[k], -mul_rn(p.idx, h1[k] - left), k ? ma[k - 1] : la, k ? ms[k - 1] : ls, ma[k], ms[k], ly, ay);
      if (ENERGY) {
        en += p.wxy * ((lx ? ax * exc[k] * exc[k] : T(0)) + (ly ? ay * eyv[k] * eyv[k] : T(0)));
        en += p.wh * hzv[k] * h1[k];
      }
    }
    if (ENERGY && out && j < r1) eacc0 += (double)en;
    // ---- step n+1 on row j-1
    const T y1r = __shfl_down_sync(FULL, y1c[0], 1);
    T h2[V];
#pragma unroll
    for (int k = 0; k < V; ++k)
      h2[k] = hmask(ma1[k], h1p[k], hupd(h1p[k], e1[k], e1c[k], k + 1 < V ? y1c[k + 1] : y1r, y1c[k], p.chy, p.chx));
    if (j - 1 == p.src_row) {
#pragma unroll
      for (int k = 0; k < V; ++k)
        if (c + k == p.src_col) h2[k] += g1;
    }
    const T hl2 = __shfl_up_sync(FULL, h2[V - 1], 1);
    const T la1 = __shfl_up_sync(FULL, ma1[V - 1], 1);
    const T ls1 = __shfl_up_sync(FULL, ms1[V - 1], 1);
    T e2[V], y2[V];
    T en1 = T(0);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      bool lx, ly;
      T ax, ay;
      e2[k] = eupd(e1c[k], mul_rn(p.idy, h2[k] - h2p[k]), ma2[k], ms2[k], ma1[k], ms1[k], lx, ax);
      const T left = k ? h2[k - 1] : hl2;
      y2[k] = eupd(y1c[k], -mul_rn(p.idx, h2[k] - left), k ? ma1[k - 1] : la1, k ? ms1[k - 1] : ls1, ma1[k], ms1[k],
                   ly, ay);
      if (ENERGY) {
        en1 += p.wxy * ((lx ? ax * e1c[k] * e1c[k] : T(0)) + (ly ? ay * y1c[k] * y1c[k] : T(0)));
        en1 += p.wh * h1p[k] * h2[k];
      }
    }
    if (out && j > r0) {
      const int64_t rs = (int64_t)(j - 1) * P + c;
      stv(p.hz1 + rs, h2);
      stv(p.ex1 + rs, e2);
      stv(p.ey1 + rs, y2);
      if (ENERGY) eacc1 += (double)en1;
    }
#pragma unroll
    for (int k = 0; k < V; ++k) {
      ma2[k] = ma1[k]; ms2[k] = ms1[k];
      ma1[k] = ma[k]; ms1[k] = ms[k];
      exc[k] = exn[k];
      h2p[k] = h2[k];
      h1p[k] = h1[k];
      e1c[k] = e1[k];
      y1c[k] = y1[k];
    }
  }
  if (ENERGY) {
    __shared__ double red0[32], red1[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      eacc0 += __shfl_down_sync(FULL, eacc0, o);
      eacc1 += __shfl_down_sync(FULL, eacc1, o);
    }
    if (lane == 0) { red0[warp] = eacc0; red1[warp] = eacc1; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double s0 = 0.0, s1 = 0.0;
      for (int w = 0; w < wpc; ++w) { s0 += red0[w]; s1 += red1[w]; }
      const int64_t b = (int64_t)cy * gridDim.x + blockIdx.x;
      p.partials[b] = s0;
      p.partials2[b] = s1;
    }
  }
}

// block-wide fixed-order sum of doubles (deterministic)
__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(FULL, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
  return s;  // valid in thread 0
}

// Y[i][b] += alpha * sum_c A[c*m + i] X[c][b] for i < m, b < B.  A is a shared model operator
// (column-major, L2-resident: one coalesced 128-byte row of A per warp and column, reused for the
// IPI instances of a thread's item); X, Y in shared memory with row stride B.
template <typename T, int IPI>
__device__ __forceinline__ void bgemm_ipi(const T* __restrict__ A, int m, int k, const T* X, T* Y, int B, T alpha) {
  const int G = B / IPI;
  for (int it = threadIdx.x; it < m * G; it += blockDim.x) {
    const int i = it % m, g = (it / m) * IPI;
    T acc[IPI];
#pragma unroll
    for (int u = 0; u < IPI; ++u) acc[u] = T(0);
#pragma unroll 16
    for (int c = 0; c < k; ++c) {
      const T a = __ldg(A + (int64_t)c * m + i);
      const T* x = X + c * B + g;
#pragma unroll
      for (int u = 0; u < IPI; ++u) acc[u] = fma_rn(a, x[u], acc[u]);
    }
    T* y = Y + i * B + g;
#pragma unroll
    for (int u = 0; u < IPI; ++u) y[u] = fma_rn(alpha, acc[u], y[u]);
  }
}

template <typename T>
__device__ __forceinline__ void bgemm(const T* A, int m, int k, const T* X, T* Y, int B, T alpha) {
  if (m * (B / 4) >= (int)blockDim.x) bgemm_ipi<T, 4>(A, m, k, X, Y, B, alpha);
  else if (m * (B / 2) >= (int)blockDim.x) bgemm_ipi<T, 2>(A, m, k, X, Y, B, alpha);
  else bgemm_ipi<T, 1>(A, m, k, X, Y, B, alpha);
}

// Shared-memory vectors of a batch (row stride B, NV rows each):
//   sx = [E~; H~] (q1 + q2), sy = y (nY), sh = h (nY), so = M1 x (q2 + q1 + nY),
//   st = t (nY), sU = U (nY), so2 = [E~; y] (q1 + nY)
template <typename T>
struct RomVec {
  T *sx, *sy, *sh, *so, *st, *sU, *so2;
  __device__ RomVec(T* sv, int64_t S) : sx(sv), sy(sv + S), sh(sv + 2 * S), so(sv + 3 * S), st(sv + 4 * S),
                                         sU(sv + 5 * S), so2(sv + 6 * S) {}
};

// One ROM step for a batch of nb (<= B) instances of one model (eq:connExplicit, K3).
// On entry sx (x~^n), sy (y^n), sh (h = Hz^{n+1/2} of the outside cells) hold the batch's vectors
// (zero padding for b >= nb).  On exit sx holds x~^{n+1} and sy holds y^{n+1}; with ENERGY the ROM
// part of W^n (coarse half cells + x~^T R~ x~) of instance b is in eout[b].
template <typename T, bool ENERGY>
__device__ void rom_step(const PostParams<T>& p, const RomModelDev& m, int first, int nb, T* sv, double* eout) {
  const int nY = m.nY, q1 = m.q1, q2 = m.q2, nx = q1 + q2, m1 = q2 + q1 + nY, m2 = q1 + nY;
  const int B = p.batch;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t S = (int64_t)p.nthreads_vec * B;
  RomVec<T> v(sv, S);
  const T* mp = p.mpool;
  for (int64_t k = tid; k < S; k += nt) { v.so[k] = T(0); v.so2[k] = T(0); }
  __syncthreads();
  if (ENERGY) {  // x~^T Rt x~ + sum D_l D_l' eps/dt y^2
    bgemm<T>(mp + m.off_Rt, nx, nx, v.sx, v.so, B, T(1));
    __syncthreads();
    const int lane = tid & 31, w = tid >> 5, nw = nt >> 5;
    for (int b = w; b < nb; b += nw) {
      const int64_t po = p.port_off[first + b];
      double acc = 0.0;
      for (int i = lane; i < nY; i += 32) acc += p.ehalf[po + i] * (double)v.sy[i * B + b] * (double)v.sy[i * B + b];
      for (int i = lane; i < nx; i += 32) acc += (double)v.sx[i * B + b] * (double)v.so[i * B + b];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(FULL, acc, o);
      if (lane == 0) eout[b] = acc;
    }
    __syncthreads();
    for (int64_t k = tid; k < S; k += nt) v.so[k] = T(0);
    __syncthreads();
  }
  // [H~^{n+1}; E*; -L~^T E*] = M1 x~^n
  bgemm<T>(mp + m.off_M1, m1, nx, v.sx, v.so, B, T(1));
  __syncthreads();
  // t = (a_y/c_y) y + (D_l G/c_y) h - L~^T E*
  for (int it = tid; it < nY * nb; it += nt) {
    const int i = it % nY, b = it / nY;
    const int64_t po = p.port_off[first + b];
    v.st[i * B + b] = v.so[(q2 + q1 + i) * B + b] +
                      fma_rn(p.cyg[po + i], v.sh[i * B + b], mul_rn(p.cya[po + i], v.sy[i * B + b]));
  }
  __syncthreads();
  // U = S_k t (per-instance Schur inverse, streamed from HBM); [E*; -L~^T E*] as the base of M2 U
  for (int it = tid; it < nY * nb; it += nt) {
    const int i = it % nY, b = it / nY;
    const T* Sk = p.Sk + p.Sk_off[first + b] + i;
    T a = T(0);
#pragma unroll 16
    for (int c = 0; c < nY; ++c) a = fma_rn(__ldg(Sk + (int64_t)c * nY), v.st[c * B + b], a);
    v.sU[i * B + b] = a;
  }
  for (int64_t k = tid; k < (int64_t)m2 * B; k += nt) {
    const int64_t r = k / B;
    v.so2[k] = r < q1 ? v.so[(q2 + r) * B + k % B] : -v.so[(q2 + r) * B + k % B];
  }
  __syncthreads();
  // [E~^{n+1}; y^{n+1}] = [E*; L~^T E*] + M2 U
  bgemm<T>(mp + m.off_M2, m2, nY, v.sU, v.so2, B, T(1));
  __syncthreads();
  for (int64_t k = tid; k < (int64_t)nx * B; k += nt) {
    const int64_t r = k / B;
    v.sx[k] = r < q1 ? v.so2[k] : v.so[(r - q1) * B + k % B];  // E~ from so2, H~ from so rows 0..q2
  }
  for (int64_t k = tid; k < (int64_t)nY * B; k += nt) v.sy[k] = v.so2[(int64_t)q1 * B + k];
  __syncthreads();
}

template <typename T>
__device__ __forceinline__ T* rom_end(const PostParams<T>& p, T* sv) {
  return sv + 7 * (int64_t)p.nthreads_vec * p.batch;  // first free element after the ROM vectors
}

template <typename T>
__device__ void load_rom_state(const PostParams<T>& p, const RomModelDev& m, int first, int nb, T* sv) {
  const int B = p.batch;
  T* sx = sv;
  const int nx = m.q1 + m.q2;
  for (int it = threadIdx.x; it < nx * nb; it += blockDim.x) {
    const int i = it % nx, b = it / nx;
    sx[i * B + b] = p.state[p.state_off[first + b] + i];
  }
}

template <typename T>
__device__ void store_rom(const PostParams<T>& p, const RomModelDev& m, int first, int nb, const T* sv, T* ex,
                          T* ey) {
  const int B = p.batch;
  const int64_t S = (int64_t)p.nthreads_vec * B;
  const T* sx = sv;
  const T* sy = sv + S;
  for (int it = threadIdx.x; it < m.nY * nb; it += blockDim.x) {  // S6: scatter y^{n+1}
    const int i = it % m.nY, b = it / m.nY;
    const int64_t e = p.port_edge[p.port_off[first + b] + i];
    if (e >> 62) ey[e & IDX_MASK] = sy[i * B + b];
    else ex[e & IDX_MASK] = sy[i * B + b];
  }
  const int nx = m.q1 + m.q2;
  for (int it = threadIdx.x; it < nx * nb; it += blockDim.x) {
    const int i = it % nx, b = it / nx;
    p.state[p.state_off[first + b] + i] = sx[i * B + b];
  }
}

// One-step post kernel body for one batch: gather, ROM step, scatter.
template <typename T, bool ENERGY>
__device__ void rom_batch(const PostParams<T>& p, int bi, T* sv) {
  const int model = p.batch_tab[3 * bi], first = p.batch_tab[3 * bi + 1], nb = p.batch_tab[3 * bi + 2];
  const RomModelDev m = p.models[model];
  const int B = p.batch;
  const int64_t S = (int64_t)p.nthreads_vec * B;
  for (int64_t k = threadIdx.x; k < 7 * S; k += blockDim.x) sv[k] = T(0);
  __syncthreads();
  T* sy = sv + S;
  T* sh = sv + 2 * S;
  // S4: gather y^n (interface edges, copied old->new by the sweep), h = Hz^{n+1/2} outside, state
  for (int it = threadIdx.x; it < m.nY * nb; it += blockDim.x) {
    const int i = it % m.nY, b = it / m.nY;
    const int64_t po = p.port_off[first + b];
    const int64_t e = p.port_edge[po + i];
    sy[i * B + b] = (e >> 62) ? p.ey1[e & IDX_MASK] : p.ex1[e & IDX_MASK];
    sh[i * B + b] = p.hz1[p.port_h[po + i]];
  }
  load_rom_state(p, m, first, nb, sv);
  __syncthreads();
  rom_step<T, ENERGY>(p, m, first, nb, sv, p.rom_partials + first);
  store_rom(p, m, first, nb, sv, p.ex1, p.ey1);
}

// Two-step fix-up for one batch (K3b).  sweep2 advanced every cell two steps with the
// interface edges frozen at y^n; here, per instance, step n is recomputed in the region
// [i0-2, i0+bx+2) x [j0-2, j0+by+2) from the input buffer (bit-identical to the sweep's own
// arithmetic), the ROM takes step n (y^{n+1}), the outside cells' Hz^{n+3/2} and their
// non-interface edges' E^{n+2} are recomputed with the correct y^{n+1}, the ROM takes step n+1
// (y^{n+2}), and the corrected values are written over the sweep's output.  The energy of
// step n+1 is corrected by mu A/dt H^{n+1/2} (H_correct - H_sweep) on the outside cells.
template <typename T, bool ENERGY>
__device__ void rom_batch2(const PostParams<T>& p, int bi, T* sv, T g0, T g1, double* sdelta) {
  const int model = p.batch_tab[3 * bi], first = p.batch_tab[3 * bi + 1], nb = p.batch_tab[3 * bi + 2];
  const RomModelDev m = p.models[model];
  const int B = p.batch, nY = m.nY;
  const int64_t S = (int64_t)p.nthreads_vec * B;
  const int tid = threadIdx.x, nt = blockDim.x;
  T* reg = rom_end(p, sv);
  const int64_t P = p.pitch;
  for (int64_t k = tid; k < 7 * S; k += nt) sv[k] = T(0);
  if (tid < B) sdelta[tid] = 0.0;  // B <= 64
  T* sy = sv + S;
  T* sh = sv + 2 * S;
  // region geometry of slot b
  auto geo = [&](int b, int& i0, int& j0, int& bx, int& by) {
    const int32_t* r = p.rects + 4 * (int64_t)(first + b);
    i0 = r[0]; j0 = r[1]; bx = r[2]; by = r[3];
  };
  // layout of one region: H1, H2, MA, MS [Hr][Wr]; EX [Hr+1][Wr]; EY [Hr][Wr+1]
  auto arrays = [&](int b, int bx, int by, T*& H1, T*& H2, T*& MA, T*& MS, T*& EX, T*& EY) {
    const int Wr = bx + 4, Hr = by + 4;
    H1 = reg + (int64_t)b * p.region_stride;
    H2 = H1 + Hr * Wr;
    MA = H2 + Hr * Wr;
    MS = MA + Hr * Wr;
    EX = MS + Hr * Wr;
    EY = EX + (Hr + 1) * Wr;
  };
  auto goff = [&](int gi, int gj) { return ((int64_t)gj - p.row_begin + p.row0) * P + gi; };
  const bool src_on = p.src_row >= 0;
  const int64_t src_off = src_on ? (int64_t)p.src_row * P + p.src_col : -1;
  // ---- R1: load the region (materials, E^n, the sweep's Hz^{n+3/2} into H2)
  for (int b = 0; b < nb; ++b) {
    int i0, j0, bx, by;
    geo(b, i0, j0, bx, by);
    T *H1, *H2, *MA, *MS, *EX, *EY;
    arrays(b, bx, by, H1, H2, MA, MS, EX, EY);
    const int Wr = bx + 4, Hr = by + 4;
    for (int t = tid; t < Hr * Wr; t += nt) {
      const int u = t % Wr, v = t / Wr;
      const int64_t o = goff(i0 - 2 + u, j0 - 2 + v);
      MA[t] = p.mea[o];
      MS[t] = p.msb[o];
      H2[t] = p.hz1[o];
    }
    for (int t = tid; t < (Hr + 1) * Wr; t += nt) EX[t] = p.ex0[goff(i0 - 2 + t % Wr, j0 - 2 + t / Wr)];
    for (int t = tid; t < Hr * (Wr + 1); t += nt) EY[t] = p.ey0[goff(i0 - 2 + t % (Wr + 1), j0 - 2 + t / (Wr + 1))];
  }
  load_rom_state(p, m, first, nb, sv);
  __syncthreads();
  // ---- R2: Hz^{n+1/2} on the region (same arithmetic as the sweep)
  for (int b = 0; b < nb; ++b) {
    int i0, j0, bx, by;
    geo(b, i0, j0, bx, by);
    T *H1, *H2, *MA, *MS, *EX, *EY;
    arrays(b, bx, by, H1, H2, MA, MS, EX, EY);
    const int Wr = bx + 4, Hr = by + 4;
    for (int t = tid; t < Hr * Wr; t += nt) {
      const int u = t % Wr, v = t / Wr;
      const int64_t o = goff(i0 - 2 + u, j0 - 2 + v);
      const T hz = p.hz0[o];
      T h = hmask(MA[t], hz, hupd(hz, EX[(v + 1) * Wr + u], EX[v * Wr + u], EY[v * (Wr + 1) + u + 1],
                                  EY[v * (Wr + 1) + u], p.chy, p.chx));
      if (o == src_off) h += g0;
      H1[t] = h;
    }
  }
  __syncthreads();
  // ---- R3: E^{n+1} on the region's interior edges (in place); gather y^n and h^{n+1/2}
  for (int b = 0; b < nb; ++b) {
    int i0, j0, bx, by;
    geo(b, i0, j0, bx, by);
    T *H1, *H2, *MA, *MS, *EX, *EY;
    arrays(b, bx, by, H1, H2, MA, MS, EX, EY);
    const int Wr = bx + 4, Hr = by + 4;
    bool l;
    T a;
    for (int t = tid; t < (Hr - 1) * Wr; t += nt) {  // Ex edge rows v = 1 .. Hr-1
      const int u = t % Wr, v = t / Wr + 1;
      const int cb = v * Wr + u, ca = cb - Wr;
      EX[v * Wr + u] = eupd(EX[v * Wr + u], mul_rn(p.idy, H1[cb] - H1[ca]), MA[ca], MS[ca], MA[cb], MS[cb], l, a);
    }
    for (int t = tid; t < Hr * (Wr - 1); t += nt) {  // Ey edge columns u = 1 .. Wr-1
      const int u = t % (Wr - 1) + 1, v = t / (Wr - 1);
      const int cb = v * Wr + u, ca = cb - 1;
      EY[v * (Wr + 1) + u] =
          eupd(EY[v * (Wr + 1) + u], -mul_rn(p.idx, H1[cb] - H1[ca]), MA[ca], MS[ca], MA[cb], MS[cb], l, a);
    }
    for (int i = tid; i < nY; i += nt) {
      int eidx, hidx;  // interface edge (EX or EY index) and outside cell, region coordinates
      bool isy;
      if (i < bx) { isy = false; eidx = 2 * Wr + 2 + i; hidx = 1 * Wr + 2 + i; }
      else if (i < 2 * bx) { isy = false; eidx = (2 + by) * Wr + 2 + (i - bx); hidx = (2 + by) * Wr + 2 + (i - bx); }
      else if (i < 2 * bx + by) { isy = true; eidx = (2 + i - 2 * bx) * (Wr + 1) + 2; hidx = (2 + i - 2 * bx) * Wr + 1; }
      else { isy = true; eidx = (2 + i - 2 * bx - by) * (Wr + 1) + 2 + bx; hidx = (2 + i - 2 * bx - by) * Wr + 2 + bx; }
      sy[i * B + b] = isy ? EY[eidx] : EX[eidx];  // y^n (interface edges are frozen copies)
      sh[i * B + b] = H1[hidx];
    }
  }
  __syncthreads();
  // ---- ROM step n: y^{n+1}, x~^{n+1}; ROM energy of W^n
  rom_step<T, ENERGY>(p, m, first, nb, sv, p.rom_partials + first);
  // ---- R4: y^{n+1} into the interface edges; Hz^{n+3/2} of the outside cells
  for (int b = 0; b < nb; ++b) {
    int i0, j0, bx, by;
    geo(b, i0, j0, bx, by);
    T *H1, *H2, *MA, *MS, *EX, *EY;
    arrays(b, bx, by, H1, H2, MA, MS, EX, EY);
    const int Wr = bx + 4;
    for (int i = tid; i < nY; i += nt) {
      if (i < bx) EX[2 * Wr + 2 + i] = sy[i * B + b];
      else if (i < 2 * bx) EX[(2 + by) * Wr + 2 + (i - bx)] = sy[i * B + b];
      else if (i < 2 * bx + by) EY[(2 + i - 2 * bx) * (Wr + 1) + 2] = sy[i * B + b];
      else EY[(2 + i - 2 * bx - by) * (Wr + 1) + 2 + bx] = sy[i * B + b];
    }
  }
  __syncthreads();
  auto port_cell = [&](int i, int bx, int by, int& u, int& v) {  // outside cell of port i
    if (i < bx) { u = 2 + i; v = 1; }
    else if (i < 2 * bx) { u = 2 + i - bx; v = 2 + by; }
    else if (i < 2 * bx + by) { u = 1; v = 2 + i - 2 * bx; }
    else { u = 2 + bx; v = 2 + i - 2 * bx - by; }
  };
  for (int b = 0; b < nb; ++b) {  // corrected Hz^{n+3/2} of the outside cells -> sh
    int i0, j0, bx, by;
    geo(b, i0, j0, bx, by);
    T *H1, *H2, *MA, *MS, *EX, *EY;
    arrays(b, bx, by, H1, H2, MA, MS, EX, EY);
    const int Wr = bx + 4;
    for (int i = tid; i < nY; i += nt) {
      int u, v;
      port_cell(i, bx, by, u, v);
      const int t = v * Wr + u;
      T h = hmask(MA[t], H1[t], hupd(H1[t], EX[(v + 1) * Wr + u], EX[v * Wr + u], EY[v * (Wr + 1) + u + 1],
                                     EY[v * (Wr + 1) + u], p.chy, p.chx));
      if (goff(i0 - 2 + u, j0 - 2 + v) == src_off) h += g1;
      sh[i * B + b] = h;
    }
  }
  __syncthreads();
  {  // energy correction of W^{n+1} (fixed order: one warp per instance), then H2 <- corrected
    const int lane = tid & 31, w = tid >> 5, nw = nt >> 5;
    for (int b = w; b < nb; b += nw) {
      int i0, j0, bx, by;
      geo(b, i0, j0, bx, by);
      T *H1, *H2, *MA, *MS, *EX, *EY;
      arrays(b, bx, by, H1, H2, MA, MS, EX, EY);
      double d = 0.0;
      for (int i = lane; i < nY; i += 32) {
        int u, v;
        port_cell(i, bx, by, u, v);
        const int t = v * (bx + 4) + u;
        d += (double)(p.wh * H1[t] * sh[i * B + b]) - (double)(p.wh * H1[t] * H2[t]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) d += __shfl_down_sync(FULL, d, o);
      if (lane == 0) sdelta[b] = d;
    }
  }
  __syncthreads();
  for (int b = 0; b < nb; ++b) {
    int i0, j0, bx, by;
    geo(b, i0, j0, bx, by);
    T *H1, *H2, *MA, *MS, *EX, *EY;
    arrays(b, bx, by, H1, H2, MA, MS, EX, EY);
    for (int i = tid; i < nY; i += nt) {
      int u, v;
      port_cell(i, bx, by, u, v);
      H2[v * (bx + 4) + u] = sh[i * B + b];
    }
  }
  __syncthreads();
  // ---- ROM step n+1: y^{n+2}, x~^{n+2}; ROM energy of W^{n+1}
  rom_step<T, ENERGY>(p, m, first, nb, sv, p.rom_partials2 + first);
  // ---- R5: E^{n+2} of the outside cells' non-interface edges, the outside cells' Hz, y^{n+2}
  for (int b = 0; b < nb; ++b) {
    int i0, j0, bx, by;
    geo(b, i0, j0, bx, by);
    T *H1, *H2, *MA, *MS, *EX, *EY;
    arrays(b, bx, by, H1, H2, MA, MS, EX, EY);
    const int Wr = bx + 4, Hr = by + 4;
    auto hole = [&](int u, int v) { return u >= 2 && u < 2 + bx && v >= 2 && v < 2 + by; };
    auto outside = [&](int u, int v) {
      return ((v == 1 || v == 2 + by) && u >= 2 && u < 2 + bx) || ((u == 1 || u == 2 + bx) && v >= 2 && v < 2 + by);
    };
    bool l;
    T a;
    for (int t = tid; t < (Hr - 1) * Wr; t += nt) {
      const int u = t % Wr, v = t / Wr + 1;
      if (!(outside(u, v - 1) || outside(u, v)) || hole(u, v - 1) || hole(u, v)) continue;
      const int cb = v * Wr + u, ca = cb - Wr;
      p.ex1[goff(i0 - 2 + u, j0 - 2 + v)] =
          eupd(EX[v * Wr + u], mul_rn(p.idy, H2[cb] - H2[ca]), MA[ca], MS[ca], MA[cb], MS[cb], l, a);
    }
    for (int t = tid; t < Hr * (Wr - 1); t += nt) {
      const int u = t % (Wr - 1) + 1, v = t / (Wr - 1);
      if (!(outside(u - 1, v) || outside(u, v)) || hole(u - 1, v) || hole(u, v)) continue;
      const int cb = v * Wr + u, ca = cb - 1;
      p.ey1[goff(i0 - 2 + u, j0 - 2 + v)] =
          eupd(EY[v * (Wr + 1) + u], -mul_rn(p.idx, H2[cb] - H2[ca]), MA[ca], MS[ca], MA[cb], MS[cb], l, a);
    }
    for (int i = tid; i < nY; i += nt) {
      int u, v;
      port_cell(i, bx, by, u, v);
      p.hz1[goff(i0 - 2 + u, j0 - 2 + v)] = H2[v * Wr + u];
    }
  }
  store_rom(p, m, first, nb, sv, p.ex1, p.ey1);
  __syncthreads();
  if (ENERGY && tid < nb) p.rom_partials2[first + tid] += sdelta[tid];
}

template <typename T, bool ENERGY>
__global__ void __launch_bounds__(256) post2_kernel(const PostParams<T> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double red[32];
  __shared__ double sdelta[64];
  __shared__ bool last;
  T* sv = reinterpret_cast<T*>(smem_raw);
  const int b = blockIdx.x;
  const int64_t step = *p.step;
  T g0 = T(0), g1 = T(0);
  if (p.src_row >= 0) {
    const int64_t k = step - p.src_t0;
    if (k >= 0 && k < p.src_n) g0 = (T)p.src_samples[k];
    if (k + 1 >= 0 && k + 1 < p.src_n) g1 = (T)p.src_samples[k + 1];
  }
  if (b < p.n_batch) {
    rom_batch2<T, ENERGY>(p, b, sv, g0, g1, sdelta);
  } else {  // probes: Hz^{n+1/2} recomputed from the input buffer, Hz^{n+3/2} from the output
    const int64_t P = p.pitch;
    const int64_t src_off = p.src_row >= 0 ? (int64_t)p.src_row * P + p.src_col : -1;
    for (int k = threadIdx.x; k < p.n_probe; k += blockDim.x) {
      const int64_t o = p.probe_idx[k];
      const T hz = p.hz0[o];
      T h = hmask(p.mea[o], hz, hupd(hz, p.ex0[o + P], p.ex0[o], p.ey0[o + 1], p.ey0[o], p.chy, p.chx));
      if (o == src_off) h += g0;
      p.probe_ring[(int64_t)k * p.cap + step % p.cap] = h;
      p.probe_ring[(int64_t)k * p.cap + (step + 1) % p.cap] = p.hz1[o];
    }
  }
  if (ENERGY) {
    const int per = (p.n_sweep_partials + gridDim.x - 1) / gridDim.x;
    const int k0 = b * per, k1 = min(p.n_sweep_partials, k0 + per);
    double v0 = 0.0, v1 = 0.0;
    for (int k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
      v0 += __ldcg(p.sweep_partials + k);
      v1 += __ldcg(p.sweep_partials2 + k);
    }
    __syncthreads();
    if (b < p.n_batch) {
      const int first = p.batch_tab[3 * b + 1], nb = p.batch_tab[3 * b + 2];
      for (int k = threadIdx.x; k < nb; k += blockDim.x) {
        v0 += p.rom_partials[first + k];
        v1 += p.rom_partials2[first + k];
      }
    }
    const double t0 = block_sum(v0, red);
    const double t1 = block_sum(v1, red);
    if (threadIdx.x == 0) {
      p.level1[b] = t0;
      p.level1b[b] = t1;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned t = atomicAdd(p.done, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (ENERGY) {
    double s0 = 0.0, s1 = 0.0;
    for (int k = threadIdx.x; k < (int)gridDim.x; k += blockDim.x) {
      s0 += __ldcg(p.level1 + k);
      s1 += __ldcg(p.level1b + k);
    }
    const double t0 = block_sum(s0, red);
    const double t1 = block_sum(s1, red);
    if (threadIdx.x == 0) {
      p.energy_ring[step % p.cap] = t0;
      p.energy_ring[(step + 1) % p.cap] = t1;
    }
  }
  if (threadIdx.x == 0) {
    *p.done = 0u;
    *p.step = step + 2;
  }
}

template <typename T, bool ENERGY>
__global__ void __launch_bounds__(256) post_kernel(const PostParams<T> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double red[32];
  __shared__ bool last;
  T* sv = reinterpret_cast<T*>(smem_raw);
  const int b = blockIdx.x;
  const int64_t step = *p.step;
  if (b < p.n_batch) {
    rom_batch<T, ENERGY>(p, b, sv);
  } else {
    for (int k = threadIdx.x; k < p.n_probe; k += blockDim.x)
      p.probe_ring[(int64_t)k * p.cap + step % p.cap] = p.hz1[p.probe_idx[k]];
  }
  if (ENERGY) {
    // level 1 (every CTA, fixed slice): sweep partials [b*per, (b+1)*per) + this batch's ROM energies
    const int per = (p.n_sweep_partials + gridDim.x - 1) / gridDim.x;
    const int k0 = b * per, k1 = min(p.n_sweep_partials, k0 + per);
    double v = 0.0;
    for (int k = k0 + threadIdx.x; k < k1; k += blockDim.x) v += __ldcg(p.sweep_partials + k);
    __syncthreads();  // rom_partials of this batch written (rom_batch ends with barriers)
    if (b < p.n_batch) {
      const int first = p.batch_tab[3 * b + 1], nb = p.batch_tab[3 * b + 2];
      for (int k = threadIdx.x; k < nb; k += blockDim.x) v += p.rom_partials[first + k];
    }
    const double tot = block_sum(v, red);
    if (threadIdx.x == 0) p.level1[b] = tot;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned t = atomicAdd(p.done, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (ENERGY) {  // level 2: fixed-order sum of the per-CTA values (deterministic)
    double s = 0.0;
    for (int k = threadIdx.x; k < (int)gridDim.x; k += blockDim.x) s += __ldcg(p.level1 + k);
    const double tot = block_sum(s, red);
    if (threadIdx.x == 0) p.energy_ring[step % p.cap] = tot;
  }
  if (threadIdx.x == 0) {
    *p.done = 0u;
    *p.step = step + 1;
  }
}

// ---------------------------------------------------------------- setup kernels
template <typename T, typename M>
__global__ void material_kernel(const M* eps_r, const M* sigma, int64_t mat_row0, int64_t mat_row_end, int64_t nx,
                                int64_t ny, int64_t row_begin, int row0, int nrows_alloc, int64_t pitch, double dt,
                                T* mea, T* msb) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int jl = blockIdx.y;  // every local row, ghost rows included
  if (i >= pitch || jl >= nrows_alloc) return;
  const int64_t g = row_begin + jl - row0;
  const int64_t o = (int64_t)jl * pitch + i;
  if (g < 0 || g >= ny || i >= nx || g < mat_row0 || g >= mat_row_end) {
    mea[o] = T(-1);  // outside the grid / not provided: walls and padding (edges next to it stay put)
    msb[o] = T(0);
    return;
  }
  const int64_t k = (g - mat_row0) * nx + i;
  mea[o] = (T)(EPS0 * (double)eps_r[k] / (2.0 * dt));  // half of eps/dt: edge a = mea_a + mea_b
  msb[o] = (T)((double)sigma[k] / 4.0);                 // quarter of sigma: edge s = sigma_edge / 2
}

template <typename M>
__global__ void gather_mat_kernel(const M* eps_r, const M* sigma, int64_t nx, int64_t mat_row0,
                                  const int64_t* cells, int64_t n, double* oe, double* os) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t gj = cells[k] / nx, gi = cells[k] % nx;
  oe[k] = (double)eps_r[(gj - mat_row0) * nx + gi];
  os[k] = (double)sigma[(gj - mat_row0) * nx + gi];
}

template <typename T>
__global__ void mask_kernel(T* mea, T* f0, T* f1, T* f2, T* f3, T* f4, T* f5, int64_t pitch, const int32_t* rects,
                            int64_t row_begin, int row0, bool zero_iface) {
  const int32_t* r = rects + 4 * (int64_t)blockIdx.x;
  const int i0 = r[0], bx = r[2], by = r[3];
  const int64_t jl0 = (int64_t)r[1] - row_begin + row0;  // local row of the block's bottom cells
  T* ex[2] = {f0, f3};
  T* ey[2] = {f1, f4};
  T* hz[2] = {f2, f5};
  // Ex edges rows jl0 .. jl0+by (interface at both ends), columns i0 .. i0+bx-1
  for (int t = threadIdx.x; t < (by + 1) * bx; t += blockDim.x) {
    const int dj = t / bx, di = t % bx;
    const int64_t o = (jl0 + dj) * pitch + i0 + di;
    if (!(dj == 0 || dj == by) || zero_iface)
      for (int q = 0; q < 2; ++q) ex[q][o] = T(0);
  }
  // Ey edges rows jl0 .. jl0+by-1, columns i0 .. i0+bx
  for (int t = threadIdx.x; t < by * (bx + 1); t += blockDim.x) {
    const int dj = t / (bx + 1), di = t % (bx + 1);
    const int64_t o = (jl0 + dj) * pitch + i0 + di;
    if (!(di == 0 || di == bx) || zero_iface)
      for (int q = 0; q < 2; ++q) ey[q][o] = T(0);
  }
  // hole cells: zero fields; mark the material so every edge touching the block keeps its value
  for (int t = threadIdx.x; t < by * bx; t += blockDim.x) {
    const int64_t o = (jl0 + t / bx) * pitch + i0 + t % bx;
    for (int q = 0; q < 2; ++q) hz[q][o] = T(0);
    if (mea) mea[o] = T(-1);
  }
}

template <typename M>
__global__ void min2_kernel(const M* a, const M* b, int64_t n, double* out) {
  double ma = INFINITY, mb = INFINITY;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    ma = fmin(ma, (double)a[k]);
    mb = fmin(mb, (double)b[k]);
  }
  __shared__ double ra[32], rb[32];
  for (int o = 16; o > 0; o >>= 1) {
    ma = fmin(ma, __shfl_down_sync(FULL, ma, o));
    mb = fmin(mb, __shfl_down_sync(FULL, mb, o));
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { ra[w] = ma; rb[w] = mb; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) { ma = fmin(ma, ra[k]); mb = fmin(mb, rb[k]); }
    out[2 * blockIdx.x] = fmin(ma, ra[0]);
    out[2 * blockIdx.x + 1] = fmin(mb, rb[0]);
  }
}

}  // namespace

template <typename M>
void launch_min2(const M* a, const M* b, int64_t n, double* out, int nblocks, cudaStream_t s) {
  min2_kernel<M><<<nblocks, 256, 0, s>>>(a, b, n, out);
}
template void launch_min2<float>(const float*, const float*, int64_t, double*, int, cudaStream_t);
template void launch_min2<double>(const double*, const double*, int64_t, double*, int, cudaStream_t);

template <typename T>
void launch_sweep(const SweepParams<T>& p, int warps_per_cta, cudaStream_t s, int chunk_begin, int chunk_count) {
  const int per_cta = 32 * warps_per_cta;
  const int nch = (p.rows + p.chunk - 1) / p.chunk;
  if (chunk_count < 0) chunk_count = nch - chunk_begin;
  if (chunk_count <= 0) return;
  SweepParams<T> q = p;
  q.chunk0 = chunk_begin;
  dim3 grid((p.ncolv + per_cta - 1) / per_cta, chunk_count);
  if (p.partials) sweep_kernel<T, true><<<grid, per_cta, 0, s>>>(q);
  else sweep_kernel<T, false><<<grid, per_cta, 0, s>>>(q);
}

template <typename T>
void launch_sweep2(const SweepParams<T>& p, int warps_per_cta, cudaStream_t s, int chunk_begin, int chunk_count) {
  const int nch = (p.rows + p.chunk - 1) / p.chunk;
  if (chunk_count < 0) chunk_count = nch - chunk_begin;
  if (chunk_count <= 0) return;
  SweepParams<T> q = p;
  q.chunk0 = chunk_begin;
  dim3 grid(sweep2_ctas_x(p.ncolv, warps_per_cta), chunk_count);
  if (p.partials) sweep2_kernel<T, true><<<grid, 32 * warps_per_cta, 0, s>>>(q);
  else sweep2_kernel<T, false><<<grid, 32 * warps_per_cta, 0, s>>>(q);
}

size_t post_smem_bytes(size_t es, int nvec, int batch) { return es * (size_t)7 * nvec * batch; }
size_t post2_smem_bytes(size_t es, int nvec, int batch, int region_stride) {
  return post_smem_bytes(es, nvec, batch) + es * (size_t)batch * region_stride;
}

template <typename T>
void launch_post2(const PostParams<T>& p, bool energy, cudaStream_t s) {
  const size_t smem = post2_smem_bytes(sizeof(T), p.nthreads_vec, p.batch, p.region_stride);
  if (energy) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(post2_kernel<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    post2_kernel<T, true><<<p.n_batch + 1, p.block, smem, s>>>(p);
  } else {
    if (smem > 48 * 1024) cudaFuncSetAttribute(post2_kernel<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    post2_kernel<T, false><<<p.n_batch + 1, p.block, smem, s>>>(p);
  }
}

template <typename T>
void launch_post(const PostParams<T>& p, bool energy, cudaStream_t s) {
  const size_t smem = post_smem_bytes(sizeof(T), p.nthreads_vec, p.batch);
  if (energy) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(post_kernel<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    post_kernel<T, true><<<p.n_batch + 1, p.block, smem, s>>>(p);
  } else {
    if (smem > 48 * 1024) cudaFuncSetAttribute(post_kernel<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    post_kernel<T, false><<<p.n_batch + 1, p.block, smem, s>>>(p);
  }
}

template <typename T, typename M>
void launch_materials(const M* eps_r, const M* sigma, int64_t mat_row0, int64_t mat_row_end, int64_t nx, int64_t ny,
                      int64_t row_begin, int row0, int nrows_alloc, int64_t pitch, double dt, T* mea, T* msb,
                      cudaStream_t s) {
  dim3 grid((unsigned)((pitch + 255) / 256), nrows_alloc);
  material_kernel<T, M><<<grid, 256, 0, s>>>(eps_r, sigma, mat_row0, mat_row_end, nx, ny, row_begin, row0,
                                             nrows_alloc, pitch, dt, mea, msb);
}

template <typename M>
void launch_gather_materials(const M* eps_r, const M* sigma, int64_t nx, int64_t mat_row0,
                             const int64_t* cells, int64_t n, double* oe, double* os, cudaStream_t s) {
  if (n <= 0) return;
  gather_mat_kernel<M><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(eps_r, sigma, nx, mat_row0, cells, n, oe, os);
}

template <typename T>
void launch_mask(T* mea, T* f[6], int64_t pitch, const int32_t* rects, int64_t n_rect, int64_t row_begin, int row0,
                 bool zero_iface, cudaStream_t s) {
  if (n_rect <= 0) return;
  mask_kernel<T><<<(unsigned)n_rect, 256, 0, s>>>(mea, f[0], f[1], f[2], f[3], f[4], f[5], pitch, rects, row_begin,
                                                   row0, zero_iface);
}

#define INST(T)                                                                                     \
  template void launch_sweep<T>(const SweepParams<T>&, int, cudaStream_t, int, int);              \
  template void launch_sweep2<T>(const SweepParams<T>&, int, cudaStream_t, int, int);             \
  template void launch_post<T>(const PostParams<T>&, bool, cudaStream_t);                        \
  template void launch_post2<T>(const PostParams<T>&, bool, cudaStream_t);                       \
  template void launch_materials<T, float>(const float*, const float*, int64_t, int64_t, int64_t, int64_t, \
                                           int64_t, int, int, int64_t, double, T*, T*, cudaStream_t);     \
  template void launch_materials<T, double>(const double*, const double*, int64_t, int64_t, int64_t,      \
                                            int64_t, int64_t, int, int, int64_t, double, T*, T*,          \
                                            cudaStream_t);                                                \
  template void launch_mask<T>(T*, T* [6], int64_t, const int32_t*, int64_t, int64_t, int, bool, cudaStream_t);
INST(float)
INST(double)
template void launch_gather_materials<float>(const float*, const float*, int64_t, int64_t,
                                             const int64_t*, int64_t, double*, double*, cudaStream_t);
template void launch_gather_materials<double>(const double*, const double*, int64_t, int64_t,
                                              const int64_t*, int64_t, double*, double*, cudaStream_t);

}  // namespace fdtd
