// Kernels of the hot path.  One pass advances K time steps:
//  K1 sweepk_kernel  : the fused Yee sweep -- per stage-0 row, the K steps of the wavefront in
//                      registers (H half-step eq:updateH L267-273, soft source, probes, storage-
//                      function partials, E half-step eq:updateEx L209-214 and its Ey analogue
//                      L223), packed fp32x2 arithmetic, a per-warp shared-memory ring of the rows'
//                      edge coefficients, ping-pong buffers (no CTA reads a value another CTA
//                      writes in the same launch).  Edge masks (PEC, ROM holes, interfaces) are
//                      encoded in the coefficients (ca = 1, cb = 0).
//  K3 postk_kernel   : per batch of ROM instances, the K steps recomputed on each instance's
//                      region with the factored eq:connExplicit update between H and E (gather,
//                      batched reduced GEMMs, Schur solve, scatter), written back on the zone.
//  pml_kernel        : the CPML band fix-up on both x-ends (NEXT-2).
//  finalize_kernel   : fixed-order energy sum of the pass and the device step counter.
#include "fdtd_kernels.cuh"

#include <algorithm>
#include <climits>
#include <type_traits>
#include <cstdio>

#include <cooperative_groups.h>

namespace fdtd {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr double MU0 = 4.0e-7 * 3.14159265358979323846;
constexpr double C0 = 299792458.0;
constexpr double EPS0 = 1.0 / (MU0 * C0 * C0);
constexpr int64_t IDX_MASK = (int64_t(1) << 62) - 1;


__device__ __forceinline__ void ldv(const float* p, float (&v)[4]) {
  const float4 x = __ldg(reinterpret_cast<const float4*>(p));
  v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
}
__device__ __forceinline__ void ldv(const float* p, float (&v)[2]) {
  const float2 x = __ldg(reinterpret_cast<const float2*>(p));
  v[0] = x.x; v[1] = x.y;
}
__device__ __forceinline__ void stv(float* p, const float (&v)[2]) {
  *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
}
[[maybe_unused]] __device__ __forceinline__ void ldv_s(const float* p, float (&v)[2]) {
  const float2 x = *reinterpret_cast<const float2*>(p);
  v[0] = x.x; v[1] = x.y;
}
__device__ __forceinline__ void stv_s(float* p, const float (&v)[2]) { stv(p, v); }
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
__device__ __forceinline__ void ldv_s(const float* p, float (&v)[4]) {
  const float4 x = *reinterpret_cast<const float4*>(p);
  v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
}
__device__ __forceinline__ void ldv_s(const double* p, double (&v)[2]) {
  const double2 x = *reinterpret_cast<const double2*>(p);
  v[0] = x.x; v[1] = x.y;
}
__device__ __forceinline__ void stv_s(float* p, const float (&v)[4]) { stv(p, v); }
__device__ __forceinline__ void stv_s(double* p, const double (&v)[2]) { stv(p, v); }
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }

// Packed fp32 pairs (sm_100a FADD2 / FMUL2 / FFMA2: two lanes of work per issue slot).  Each
// element is rounded exactly as the scalar fadd / fmul / fma of the same operands, so packed and
// scalar code paths (sweep vs fix-up) stay bit-identical.
struct F2 {
  float x, y;
};
__device__ __forceinline__ F2 sub2(F2 a, F2 b) {
  F2 r;
  asm("{.reg .b64 ra, rb, rd;\n mov.b64 ra, {%2,%3};\n mov.b64 rb, {%4,%5};\n sub.rn.f32x2 rd, ra, rb;\n"
      " mov.b64 {%0,%1}, rd;}" : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ F2 mul2(F2 a, F2 b) {
  F2 r;
  asm("{.reg .b64 ra, rb, rd;\n mov.b64 ra, {%2,%3};\n mov.b64 rb, {%4,%5};\n mul.rn.f32x2 rd, ra, rb;\n"
      " mov.b64 {%0,%1}, rd;}" : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ F2 fma2(F2 a, F2 b, F2 c) {
  F2 r;
  asm("{.reg .b64 ra, rb, rc, rd;\n mov.b64 ra, {%2,%3};\n mov.b64 rb, {%4,%5};\n mov.b64 rc, {%6,%7};\n"
      " fma.rn.f32x2 rd, ra, rb, rc;\n mov.b64 {%0,%1}, rd;}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}

// one element global -> shared, asynchronously (LDGSTS); completed by cp.async.wait_all
template <typename T>
__device__ __forceinline__ void cp_async_el(T* dst, const T* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src),
               "n"(sizeof(T)) : "memory");
}

#ifndef FDTD_REG_RING  // sweep: coefficient ring of K rows in registers (1) or shared memory (0)
#define FDTD_REG_RING 0
#endif
#ifndef FDTD_EXP  // sweep diagnostics (tools/sweep_layout_probe.cu only): 1 no ring loads, 4 no stores
#define FDTD_EXP 0
#endif
#ifndef FDTD_PFD
#define FDTD_PFD 1  // sweep: row distance of the L2 prefetch beyond the register-prefetched row (measured best)
#endif
constexpr int PFD = FDTD_PFD;
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

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

// Coefficients of one edge of eq:updateEx (and its Ey analogue) divided by its left-hand
// coefficient, from the two adjacent cells' material terms (arithmetic means, R2):
//   E' = ca E + cb dH,  ca = (a - s)/(a + s) = 1 - 2s/(a + s),  cb = il/(a + s),
// a = eps/dt, s = sigma/2 of the edge, il = 1/dy (Ex, dH = H - H_below) or -1/dx (Ey,
// dH = H - H_left).  An edge next to a cell with a < 0 (ROM hole, PEC wall, padding) is dead:
// ca = 1, cb = 0 keeps its value exactly (PEC edges stay 0; interface edges belong to the ROM).
// The sign bit of s0 / s1 marks fix-up zone cells and is ignored here.
template <typename T>
__device__ __forceinline__ void edge_coef(T a0, T s0, T a1, T s1, T il, T& ca, T& cb, T& a, bool& live) {
  a = a0 + a1;
  const T s = fabs(s0) + fabs(s1);
  live = (a0 >= T(0)) & (a1 >= T(0));
  // r = 0 on a dead edge makes ca = 1 and cb = 0 (the edge keeps its value) with one select
  const T r = live ? rcp_rn(a + s) : T(0);
  // ca = 1 - 2 s r: exactly 1 on lossless edges whatever the rounding of r (an approximate
  // reciprocal only perturbs the small loss term and the curl gain, so a lossless grid stays
  // lossless instead of decaying by ~1 ulp per step)
  ca = fma_rn(T(-2) * s, r, T(1));
  cb = mul_rn(r, il);
}

template <typename T>
__device__ __forceinline__ T eupd(T e, T ca, T cb, T dh) {
  return fma_rn(ca, e, mul_rn(cb, dh));
}

// Storage-function partial (eq:R, R17) of one cell at the start of a step, accumulated into acc:
// (1/dt)[C E^2 of the cell's bottom Ex and left Ey edge + mu A H^{n-1/2} H^{n+1/2}] with the
// weights wx, wy = dx dy a of live edges (C/dt = dx dy eps/dt), hw = mu0 dx dy / dt.
template <typename T>
__device__ __forceinline__ T cell_energy(T acc, T ex, T ey, T h0, T h1, T wx, T wy, T hw) {
  return fma_rn(mul_rn(hw, h0), h1, fma_rn(mul_rn(wy, ey), ey, fma_rn(mul_rn(wx, ex), ex, acc)));
}

// Per-cell coefficient set of one row of a warp strip (K1): the cell's bottom Ex edge
// (cax, cbx), left Ey edge (cay, cby) and the energy weights of those edges (wx, wy; 0 if dead or a
// zone cell).  The cell's own flags ride in the sign bits of the weights, which are otherwise
// non-negative: wx = -0 on a dead cell (hole, wall, padding: its Hz is kept), wy = -0 on a fix-up
// zone cell (the fix-up adds its energy); the Hz weight mu0 dx dy/dt applies when neither is set
// (cell_hw).  Six vectors per row: built once per pass at stage 0, reused by stages 1..K-1.
template <typename T, int V>
struct RowCoef {
  T cax[V], cbx[V], cay[V], cby[V], wx[V], wy[V];
};
constexpr int NCOEF = 6;
template <typename T>
__device__ __forceinline__ bool cell_dead(T wx) { return signbit(wx); }
template <typename T>
__device__ __forceinline__ T cell_hw(T wx, T wy, T wh) { return (signbit(wx) | signbit(wy)) ? T(0) : wh; }
#ifndef FDTD_EACC2  // with FDTD_EFAST: per-stage packed fp32 pair accumulators (no per-row pair sum)
#define FDTD_EACC2 0  // measured: +3.6 % per pass (one spill, 128-register cap)
#endif
#ifndef FDTD_EFAST  // sweep energy: cheaper Hz weight and fp32 row sums flushed to fp64 every 16 rows
#define FDTD_EFAST 1  // round 2 measured -2.5 % per sweep pass (cold and power-capped, tools/sweep_layout_probe.cu)
#endif
// The Hz weight of the sweep's packed energy term without a select: wh, or 0 on a zone cell (wy = -0).
// A dead cell (hole, wall, padding) keeps Hz = 0, so its weight does not matter: wh * 0 * 0 = 0.
__device__ __forceinline__ F2 cell_hw2(float wy0, float wy1, float hwh) {
  return fma2(F2{copysignf(1.f, wy0), copysignf(1.f, wy1)}, F2{hwh, hwh}, F2{hwh, hwh});  // hwh = wh / 2
}

template <typename T, int V>
__device__ __forceinline__ void row_coef(const T (&ma)[V], const T (&ms)[V], const T (&mb)[V], const T (&sb)[V],
                                         T idx, T idy, T wxy, T wh, RowCoef<T, V>& cf) {
  const T la = __shfl_up_sync(FULL, ma[V - 1], 1);
  const T ls = __shfl_up_sync(FULL, ms[V - 1], 1);
#pragma unroll
  for (int k = 0; k < V; ++k) {
    bool lx, ly;
    T ax, ay;
    edge_coef(mb[k], sb[k], ma[k], ms[k], idy, cf.cax[k], cf.cbx[k], ax, lx);
    edge_coef(k ? ma[k - 1] : la, k ? ms[k - 1] : ls, ma[k], ms[k], -idx, cf.cay[k], cf.cby[k], ay, ly);
    const bool z = signbit(ms[k]);
    cf.wx[k] = (lx && !z) ? mul_rn(wxy, ax) : (ma[k] < T(0) ? T(-0.0) : T(0));  // a dead cell has no live edge
    cf.wy[k] = (ly && !z) ? mul_rn(wxy, ay) : (z ? T(-0.0) : T(0));
    (void)wh;
  }
}

// Coefficient sources for yee_row: registers (stage 0 just built them) or the warp's shared-memory
// ring (stages 1..K-1), read lazily so that only the vectors in use occupy registers.
template <typename T, int V>
struct CoefRegs {
  const RowCoef<T, V>& c;
  __device__ __forceinline__ void ex(T (&a)[V], T (&b)[V]) const {
    for (int k = 0; k < V; ++k) { a[k] = c.cax[k]; b[k] = c.cbx[k]; }
  }
  __device__ __forceinline__ void ey(T (&a)[V], T (&b)[V]) const {
    for (int k = 0; k < V; ++k) { a[k] = c.cay[k]; b[k] = c.cby[k]; }
  }
  __device__ __forceinline__ void w(T (&a)[V], T (&b)[V]) const {
    for (int k = 0; k < V; ++k) { a[k] = c.wx[k]; b[k] = c.wy[k]; }
  }
};
#ifndef FDTD_RING128  // fp32 pairs: the ring holds (a, b) vector pairs as one 16-byte LDS / STS each
#define FDTD_RING128 1
#endif
template <typename T, int V>
__host__ __device__ constexpr bool ring_packed() { return FDTD_RING128 && sizeof(T) == 4 && V == 2; }
template <typename T, int V>
struct CoefRing {
  const T* b;  // this lane's slot: component i at b + i * 32 * V (packed: pair i/2 at b + (i/2) * 64 * V)
  __device__ __forceinline__ void ld2(int i, T (&a)[V], T (&c)[V]) const {
    if constexpr (ring_packed<T, V>()) {
      const float4 t = *reinterpret_cast<const float4*>(b + i * 32 * V);
      a[0] = t.x; a[1] = t.y; c[0] = t.z; c[1] = t.w;
    } else {
      ldv_s(b + i * 32 * V, a);
      ldv_s(b + (i + 1) * 32 * V, c);
    }
  }
  __device__ __forceinline__ void ex(T (&a)[V], T (&c)[V]) const { ld2(0, a, c); }
  __device__ __forceinline__ void ey(T (&a)[V], T (&c)[V]) const { ld2(2, a, c); }
  __device__ __forceinline__ void w(T (&a)[V], T (&c)[V]) const { ld2(4, a, c); }
};

// One Yee step on one row r of a warp's column strip (K1): Hz^{new} of row r from
// (Ex edge rows r and r+1, Ey and Hz of row r), the soft source, then Ex of edge row r and Ey of
// row r from Hz^{new} of rows r and r-1 (hb).  Column neighbours come from warp shuffles (the
// outermost lanes of a strip get wrong outermost values; they are redundant halo lanes).  All
// lanes call it.  Returns the row's storage-function partial of W at the step's start (zone cells
// excluded).
template <typename T, int V, bool ENERGY, typename CS>
__device__ __forceinline__ T yee_row(const T (&exb)[V], const T (&ext)[V], const T (&ey)[V], const T (&hz)[V],
                                     const T (&hb)[V], const CS& cs, const SweepParams<T>& p, T gsrc,
                                     bool srow, int src_k, T (&hn)[V], T (&exo)[V], T (&eyo)[V]) {
  const T eyr = __shfl_down_sync(FULL, ey[0], 1);
  T wx[V], wy[V];  // energy weights, with the dead / zone flags in their sign bits
  cs.w(wx, wy);
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const T hu = hupd(hz[k], ext[k], exb[k], k + 1 < V ? ey[k + 1] : eyr, ey[k], p.chy, p.chx);
    hn[k] = cell_dead(wx[k]) ? hz[k] : hu;  // dead cells keep their Hz
  }
  if (srow) {  // S2: soft source after the H half-step (this lane holds the source column)
#pragma unroll
    for (int k = 0; k < V; ++k)
      if (k == src_k) hn[k] += gsrc;
  }
  const T hl = __shfl_up_sync(FULL, hn[V - 1], 1);
  {
    T ca[V], cb[V];
    cs.ex(ca, cb);
#pragma unroll
    for (int k = 0; k < V; ++k) exo[k] = eupd(exb[k], ca[k], cb[k], hn[k] - hb[k]);
  }
  {
    T ca[V], cb[V];
    cs.ey(ca, cb);
#pragma unroll
    for (int k = 0; k < V; ++k) eyo[k] = eupd(ey[k], ca[k], cb[k], hn[k] - (k ? hn[k - 1] : hl));
  }
  T en = T(0);
  if (ENERGY) {
#pragma unroll
    for (int k = 0; k < V; ++k)
      en = cell_energy(en, exb[k], ey[k], hz[k], hn[k], wx[k], wy[k], cell_hw(wx[k], wy[k], p.wh));
  }
  return en;
}

// yee_row for fp32 with the column pairs of a lane in packed FADD2 / FMUL2 / FFMA2 (the same
// per-element operations as the generic version, in the same order).
// ACC: the storage-function terms go straight into the caller's packed accumulator (when `own`)
// and 0 is returned.
template <int V, bool ENERGY, typename CS, bool ACC = false>
__device__ __forceinline__ float yee_row_f2(const float (&exb)[V], const float (&ext)[V], const float (&ey)[V],
                                            const float (&hz)[V], const float (&hb)[V], const CS& cs,
                                            const SweepParams<float>& p, float gsrc, bool srow, int src_k,
                                            float (&hn)[V], float (&exo)[V], float (&eyo)[V],
                                            F2* acc_out = nullptr, bool own = true) {
  static_assert(V % 2 == 0, "pairs");
  const float eyr = __shfl_down_sync(FULL, ey[0], 1);
  float wx[V], wy[V];  // energy weights, with the dead / zone flags in their sign bits
  cs.w(wx, wy);
  const F2 chy{p.chy, p.chy}, mchx{-p.chx, -p.chx};
#pragma unroll
  for (int k = 0; k < V; k += 2) {
    const F2 dex = sub2(F2{ext[k], ext[k + 1]}, F2{exb[k], exb[k + 1]});
    const F2 dey = sub2(F2{ey[k + 1], k + 2 < V ? ey[k + 2] : eyr}, F2{ey[k], ey[k + 1]});
    const F2 hu = fma2(mchx, dey, fma2(chy, dex, F2{hz[k], hz[k + 1]}));
    hn[k] = cell_dead(wx[k]) ? hz[k] : hu.x;  // dead cells keep their Hz
    hn[k + 1] = cell_dead(wx[k + 1]) ? hz[k + 1] : hu.y;
  }
  if (srow) {  // S2: soft source after the H half-step (this lane holds the source column)
#pragma unroll
    for (int k = 0; k < V; ++k)
      if (k == src_k) hn[k] += gsrc;
  }
  const float hl = __shfl_up_sync(FULL, hn[V - 1], 1);
  {
    float ca[V], cb[V];
    cs.ex(ca, cb);
#pragma unroll
    for (int k = 0; k < V; k += 2) {
      const F2 t = mul2(F2{cb[k], cb[k + 1]}, sub2(F2{hn[k], hn[k + 1]}, F2{hb[k], hb[k + 1]}));
      const F2 e = fma2(F2{ca[k], ca[k + 1]}, F2{exb[k], exb[k + 1]}, t);
      exo[k] = e.x; exo[k + 1] = e.y;
    }
  }
  {
    float ca[V], cb[V];
    cs.ey(ca, cb);
#pragma unroll
    for (int k = 0; k < V; k += 2) {
      const F2 t = mul2(F2{cb[k], cb[k + 1]}, sub2(F2{hn[k], hn[k + 1]}, F2{k ? hn[k - 1] : hl, hn[k]}));
      const F2 e = fma2(F2{ca[k], ca[k + 1]}, F2{ey[k], ey[k + 1]}, t);
      eyo[k] = e.x; eyo[k + 1] = e.y;
    }
  }
  float en = 0.f;
  if (ENERGY && (!ACC || own)) {
    F2 acc{0.f, 0.f};
    if constexpr (ACC) acc = *acc_out;
#pragma unroll
    for (int k = 0; k < V; k += 2) {
      const F2 ex2{exb[k], exb[k + 1]}, ey2{ey[k], ey[k + 1]};
#if FDTD_EFAST
      const F2 hw = cell_hw2(wy[k], wy[k + 1], 0.5f * p.wh);
#else
      const F2 hw{cell_hw(wx[k], wy[k], p.wh), cell_hw(wx[k + 1], wy[k + 1], p.wh)};
#endif
      acc = fma2(mul2(F2{wx[k], wx[k + 1]}, ex2), ex2, acc);
      acc = fma2(mul2(F2{wy[k], wy[k + 1]}, ey2), ey2, acc);
      acc = fma2(mul2(hw, F2{hz[k], hz[k + 1]}), F2{hn[k], hn[k + 1]}, acc);
    }
    if constexpr (ACC)
      *acc_out = acc;
    else
      en = acc.x + acc.y;
  }
  return en;
}

// energy accumulators of the sweep: fp64, fp32 row sums (FDTD_EFAST), or packed fp32 pairs
__device__ __forceinline__ double ea_value(double a) { return a; }
__device__ __forceinline__ double ea_value(float a) { return (double)a; }
[[maybe_unused]] __device__ __forceinline__ double ea_value(F2 a) { return (double)a.x + (double)a.y; }
__device__ __forceinline__ void ea_zero(double& a) { a = 0.0; }
__device__ __forceinline__ void ea_zero(float& a) { a = 0.f; }
[[maybe_unused]] __device__ __forceinline__ void ea_zero(F2& a) { a = F2{0.f, 0.f}; }

// S3 probes: record Hz^{n+s+1/2} of the probes in row r owned by this lane (sorted per row).
// Out of line: only the few row chunks holding a probe row take this path.
template <typename T, int V>
struct VecV {
  T v[V];
};
template <typename T, int V>
__device__ __forceinline__ void record_probes_v(const SweepParams<T>& p, int r, VecV<T, V> h, int64_t slot, int64_t c) {
  if (!p.probe_rows) return;
  const int2 pr = __ldg(p.probe_rows + r);
  for (int i = 0; i < pr.y; ++i) {
    const int2 e = __ldg(p.probe_list + pr.x + i);
    const int64_t d = (int64_t)e.x - c;
    if (d >= 0 && d < V) {
      T v = h.v[0];
#pragma unroll
      for (int k = 1; k < V; ++k)
        if (d == k) v = h.v[k];
      FCHK(e.y >= 0 && slot >= 0 && slot < p.cap);
      p.probe_ring[(int64_t)e.y * p.cap + slot] = v;
    }
  }
}
template <typename T, int V>
__device__ __forceinline__ void record_probes(const SweepParams<T>& p, int r, const T (&h)[V], int64_t slot, int64_t c) {
  VecV<T, V> hv;
#pragma unroll
  for (int k = 0; k < V; ++k) hv.v[k] = h[k];
  record_probes_v<T, V>(p, r, hv, slot, c);
}

// per-warp shared-memory ring of K rows of coefficient sets (lane-private 16-byte vectors)
template <typename T, int V>
__device__ __forceinline__ void ring_store(T* ring, int slot, const RowCoef<T, V>& cf) {  // ring: this lane's base
  T* b = ring + slot * (NCOEF * 32 * V);
  if constexpr (ring_packed<T, V>()) {
    *reinterpret_cast<float4*>(b) = make_float4(cf.cax[0], cf.cax[1], cf.cbx[0], cf.cbx[1]);
    *reinterpret_cast<float4*>(b + 2 * 32 * V) = make_float4(cf.cay[0], cf.cay[1], cf.cby[0], cf.cby[1]);
    *reinterpret_cast<float4*>(b + 4 * 32 * V) = make_float4(cf.wx[0], cf.wx[1], cf.wy[0], cf.wy[1]);
    return;
  }
  stv_s(b + 0 * 32 * V, cf.cax); stv_s(b + 1 * 32 * V, cf.cbx); stv_s(b + 2 * 32 * V, cf.cay);
  stv_s(b + 3 * 32 * V, cf.cby); stv_s(b + 4 * 32 * V, cf.wx); stv_s(b + 5 * 32 * V, cf.wy);
}
template <typename T, int V>
__device__ __forceinline__ void ring_load(const T* ring, int slot, RowCoef<T, V>& cf) {
  const T* b = ring + slot * (NCOEF * 32 * V);
  ldv_s(b + 0 * 32 * V, cf.cax); ldv_s(b + 1 * 32 * V, cf.cbx); ldv_s(b + 2 * 32 * V, cf.cay);
  ldv_s(b + 3 * 32 * V, cf.cby); ldv_s(b + 4 * 32 * V, cf.wx); ldv_s(b + 5 * 32 * V, cf.wy);
}

// Row data of one stage-0 row j (loaded from HBM): Ex of edge row j+1, Ey / Hz / materials of row j
template <typename T, int V>
struct RowIn {
  T ext[V], ey[V], hz[V], ma[V], ms[V];
};
// Outputs of every stage at one stage-0 row j: stage s's Hz^{n+s+1/2}, Ex^{n+s+1}, Ey^{n+s+1} of row j-s
template <typename T, int V, int K>
struct StageOut {
  T h[K][V], x[K][V], y[K][V];
};

template <typename T, int V, int K>
struct SweepCtx {
  uint32_t c;       // this lane's first column
  uint32_t cf, Pf;  // its element offset in a row of the field pool and that pool's row pitch
  uint32_t cm, Pm;  // the same in the material pool: every pool holds < 2^32 elements
                    // (fdtd_create), so offsets stay 32-bit and each address is one wide
                    // multiply-add on the pool's base pointer (the pools' arrays sit TILE apart)
  T* ring;
  int lane, r0, r1, src_r, src_r1, src_k;  // source rows [src_r, src_r1) in this lane's column src_k
  bool out;
  int64_t step;
  T g[K];
  int64_t slot[K];  // probe-ring slot of each stage's step
};

// One stage-0 row j of the K-step sweep: X holds row j's data, Y row j-1's (and receives row
// j+1's once stage 0 is done), A the stage outputs of row j-1, B receives those of row j.
// Naming the two buffers statically (the caller alternates them) keeps every carried value in
// place: no register moves.
// fp32: packed pairs; fp64: the generic scalar row
template <typename T, int V, bool ENERGY, typename CS, typename EA>
__device__ __forceinline__ void yee_any(const T (&exb)[V], const T (&ext)[V], const T (&ey)[V], const T (&hz)[V],
                                        const T (&hb)[V], const CS& cs, const SweepParams<T>& p, T gsrc, bool srow,
                                        int src_k, T (&hn)[V], T (&exo)[V], T (&eyo)[V], EA& acc, bool own) {
  if constexpr (std::is_same<EA, F2>::value) {
    yee_row_f2<V, ENERGY, CS, true>(exb, ext, ey, hz, hb, cs, p, gsrc, srow, src_k, hn, exo, eyo, &acc, own);
  } else {
    T en;
    if constexpr (sizeof(T) == 4 && V % 2 == 0)
      en = yee_row_f2<V, ENERGY>(exb, ext, ey, hz, hb, cs, p, gsrc, srow, src_k, hn, exo, eyo);
    else
      en = yee_row<T, V, ENERGY>(exb, ext, ey, hz, hb, cs, p, gsrc, srow, src_k, hn, exo, eyo);
    if (ENERGY && own) acc += (EA)en;
  }
}

template <typename T, int V, int K, bool ENERGY, bool CHK, int T0, typename EA>
__device__ __forceinline__ void sweep_row(const SweepParams<T>& p, const SweepCtx<T, V, K>& x, int j, int je,
                                          const RowIn<T, V>& X, RowIn<T, V>& Y, const StageOut<T, V, K>& A,
                                          StageOut<T, V, K>& B, EA (&eacc)[K], RowCoef<T, V> (&rc)[K]) {
  // T0 = (j - jb) mod the loop's unroll: the coefficient set of row j - s lives in rc[(T0 - s) mod K]
  // (registers, statically named; FDTD_REG_RING) or in the shared-memory ring
  // CHK: some stage rows may lie outside the chunk [r0, r1) (energy, probes and stores skip them)
  // and the probe table is consulted; without CHK every stage row is the chunk's own, probe-free.
  {  // ---- stage 0: step n on row j (builds the row's coefficients and parks them in the ring)
#if FDTD_REG_RING
    RowCoef<T, V>& cf = rc[T0 & (K - 1)];
    row_coef<T, V>(X.ma, X.ms, Y.ma, Y.ms, p.idx, p.idy, p.wxy, p.wh, cf);
#else
#if FDTD_EXP & 1
    RowCoef<T, V>& cf = rc[0];
    row_coef<T, V>(X.ma, X.ms, Y.ma, Y.ms, p.idx, p.idy, p.wxy, p.wh, cf);
#else
    RowCoef<T, V> cf;
    row_coef<T, V>(X.ma, X.ms, Y.ma, Y.ms, p.idx, p.idy, p.wxy, p.wh, cf);
    if (K > 1) ring_store<T, V>(x.ring, j & (K - 1), cf);
#endif
#endif
    const bool own = !CHK || (j >= x.r0 && j < x.r1);
    yee_any<T, V, ENERGY>(Y.ext, X.ext, X.ey, X.hz, A.h[0], CoefRegs<T, V>{cf}, p, x.g[0],
                          CHK && j >= x.src_r && j < x.src_r1, x.src_k, B.h[0], B.x[0], B.y[0], eacc[0], own);
    if (CHK && own && x.out) record_probes<T, V>(p, j, B.h[0], x.slot[0], (int32_t)x.c);
  }
  if (j + 1 < je) {  // row j+1 into the buffer of row j-1 (consumed above)
    const uint32_t o = (uint32_t)(j + 1) * x.Pf + x.cf, om = (uint32_t)(j + 1) * x.Pm + x.cm;
    FCHK((int64_t)o + x.Pf + 2 * TILE + V <= p.alloc_elems_f && (int64_t)om + TILE + V <= p.alloc_elems_m);
    ldv(p.ex0 + (o + x.Pf), Y.ext);
    ldv(p.ey0 + o, Y.ey);
    ldv(p.hz0 + o, Y.hz);
    ldv(p.mea + om, Y.ma);
    ldv(p.msb + om, Y.ms);
  }
  if (PFD > 0 && j + 1 + PFD < je) {  // pull row j+1+PFD into L2 (no registers held)
    const uint32_t o = (uint32_t)(j + 1 + PFD) * x.Pf + x.cf, om = (uint32_t)(j + 1 + PFD) * x.Pm + x.cm;
    prefetch_l2(p.ex0 + (o + x.Pf));
    prefetch_l2(p.ey0 + o);
    prefetch_l2(p.hz0 + o);
    prefetch_l2(p.mea + om);
    prefetch_l2(p.msb + om);
  }
  // ---- stage s: step n+s on row j-s, from stage s-1's outputs of rows j-s (A) and j-s+1 (B)
#pragma unroll
  for (int s = 1; s < K; ++s) {
    const int r = j - s;
#if FDTD_REG_RING
    const CoefRegs<T, V> cr{rc[(T0 - s) & (K - 1)]};
#elif FDTD_EXP & 1  // diagnostic: no ring loads (wrong coefficients)
    const CoefRegs<T, V> cr{rc[0]};
#else
    const CoefRing<T, V> cr{x.ring + (r & (K - 1)) * (NCOEF * 32 * V)};
#endif
    const bool own = !CHK || (r >= x.r0 && r < x.r1);
    yee_any<T, V, ENERGY>(A.x[s - 1], B.x[s - 1], A.y[s - 1], A.h[s - 1], A.h[s], cr, p, x.g[s],
                          CHK && r >= x.src_r && r < x.src_r1, x.src_k, B.h[s], B.x[s], B.y[s], eacc[s], own);
    if (CHK && own && x.out) record_probes<T, V>(p, r, B.h[s], x.slot[s], (int32_t)x.c);
  }
  // stage K-1's outputs are the fields at step n+K of row j-K+1
  const int rs = j - (K - 1);
  if (!(FDTD_EXP & 4) && x.out && (!CHK || (rs >= x.r0 && rs < x.r1))) {
    const uint32_t o = (uint32_t)rs * x.Pf + x.cf;
    FCHK(rs >= p.row0 && rs < p.row0 + p.rows && x.c + V <= p.pitch);  // stores stay in the owned rows
    stv(p.hz1 + o, B.h[K - 1]);
    stv(p.ex1 + o, B.x[K - 1]);
    stv(p.ey1 + o, B.y[K - 1]);
  }
}

// K1: K time steps per pass (temporal blocking).  At stage-0 row j a warp advances step n on row
// j, step n+1 on row j-1, ..., step n+K-1 on row j-K+1, entirely in registers, so every field and
// material byte crosses HBM once per K steps (32/K B per cell-step in fp32).  Lanes 0 and 31 are
// redundant halo lanes (a 16-byte vector holds V >= K columns, so after K steps only they carry
// wrong values); lanes 1..30 store.  A row chunk starts K rows early (recomputed, never stored).
// Stage 0 builds the row's edge coefficients once (row_coef) and parks them in a per-warp
// shared-memory ring of K rows, where stages 1..K-1 find them.  Interface edges are dead (frozen)
// in every step; the fix-up kernel repairs the zone around every ROM instance.  The arrays are
// padded so that every lane loads unconditionally.
#ifndef FDTD_SWEEP_THREADS  // at most 8 warps per CTA (fdtd_set_tuning)
#define FDTD_SWEEP_THREADS 256
#endif
#if FDTD_REG_RING && !defined(FDTD_SWEEP_MAXNREG)  // register ring: per-thread register cap
#define FDTD_SWEEP_MAXNREG 168
#endif
#ifndef FDTD_SWEEP_MINB  // 2 x 256 threads: <= 128 registers, 16 resident warps per SM
#define FDTD_SWEEP_MINB (FDTD_REG_RING ? 1 : 2)
#endif
template <typename T, int K, int V, bool ENERGY, int UR = 2>
#if defined(FDTD_SWEEP_MAXNREG)
__global__ void __maxnreg__(FDTD_SWEEP_MAXNREG) sweepk_kernel(
#else
__global__ void __launch_bounds__(FDTD_SWEEP_THREADS, FDTD_SWEEP_MINB) sweepk_kernel(
#endif
    const SweepParams<T> p) {
  constexpr int HL = (K + V - 1) / V;  // halo lanes at each end of a warp (sweep_halo)
  constexpr int NOUT = 32 - 2 * HL;    // storing lanes per warp
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SweepCtx<T, V, K> x;
  x.lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int wpc = blockDim.x >> 5;
  x.ring = reinterpret_cast<T*>(smem_raw) + (int64_t)warp * K * NCOEF * 32 * V + x.lane * V * (ring_packed<T, V>() ? 2 : 1);
  const int64_t colv = (int64_t)(blockIdx.x * wpc + warp) * NOUT + x.lane - HL;
  x.out = colv >= 0 && colv < (p.nx + V - 1) / V && x.lane >= HL && x.lane < 32 - HL;
  const int64_t c = (int64_t)colv * V;
  const int cy = p.chunk0 + blockIdx.y;  // row chunk
  x.r0 = p.row0 + cy * p.chunk;
  x.r1 = min(x.r0 + p.chunk, p.row0 + p.rows);
  x.c = (uint32_t)c;
  // pool offsets (c >= -V: row offsets >= one pitch keep every element offset non-negative)
  x.Pf = (uint32_t)(p.pitch * p.naf);
  x.Pm = (uint32_t)(p.pitch * p.nam);
  x.cf = (uint32_t)pool_off(c, p.naf);
  x.cm = (uint32_t)pool_off(c, p.nam);

  const bool src_lane = p.src_row >= 0 && p.src_col >= c && p.src_col < c + V;
  x.src_k = src_lane ? (int)(p.src_col - c) : -1;
  x.src_r = src_lane ? p.src_row : INT_MIN;
  x.src_r1 = src_lane ? p.src_row_end : INT_MIN;
  x.step = *p.step;
#pragma unroll
  for (int s = 0; s < K; ++s) {
    x.g[s] = T(0);
    if (p.src_row >= 0) {
      const int64_t k = x.step + s - p.src_meta[0];
      if (k >= 0 && k < p.src_meta[1]) x.g[s] = (T)p.src_samples[k];
    }
    x.slot[s] = (x.step + s) % p.cap;
  }
  const int jb = x.r0 - K, je = x.r1 + K - 1;  // stage-0 rows [jb, je); jb - 1 >= 0 (ROW0 = 2 KMAX)
  RowIn<T, V> R0, R1;  // rows jb-1 (only Ex of edge row jb and the materials are used) and jb
  {
    const uint32_t o = (uint32_t)(jb - 1) * x.Pf + x.cf, om = (uint32_t)(jb - 1) * x.Pm + x.cm;
    FCHK(jb - 1 >= 0 && (int64_t)o + 2 * x.Pf + 2 * TILE + V <= p.alloc_elems_f &&
         (int64_t)om + x.Pm + TILE + V <= p.alloc_elems_m);
    ldv(p.ex0 + (o + x.Pf), R0.ext);
    ldv(p.mea + om, R0.ma);
    ldv(p.msb + om, R0.ms);
    const uint32_t o1 = o + x.Pf, om1 = om + x.Pm;
    ldv(p.ex0 + (o1 + x.Pf), R1.ext);
    ldv(p.ey0 + o1, R1.ey);
    ldv(p.hz0 + o1, R1.hz);
    ldv(p.mea + om1, R1.ma);
    ldv(p.msb + om1, R1.ms);
  }
  StageOut<T, V, K> O0, O1;
#pragma unroll
  for (int s = 0; s < K; ++s)
#pragma unroll
    for (int k = 0; k < V; ++k) O0.h[s][k] = O0.x[s][k] = O0.y[s][k] = T(0);
  // energy partials: per stage, the rows' sums in EA (fp32 with FDTD_EFAST, flushed into the fp64
  // dacc every 16 rows) -- fp64 over the chunk
  // (packed fp32 pairs, FDTD_EACC2, on the packed row path)
  using EA = typename std::conditional<
      FDTD_EFAST && sizeof(T) == 4,
      typename std::conditional<FDTD_EACC2 && V % 2 == 0, F2, float>::type, double>::type;
  EA eacc[K];
  double dacc[K];
#pragma unroll
  for (int s = 0; s < K; ++s) {
    ea_zero(eacc[s]);
    dacc[s] = 0.0;
  }
  // does this warp's strip hold a probe in the chunk's rows?  (scanned once per warp)
  bool warp_probes = false;
  if (p.probe_rows) {
    const int64_t c_lo = (colv - x.lane + HL) * V, c_hi = c_lo + (int64_t)NOUT * V;  // stored columns
    for (int r = x.r0 + x.lane; r < x.r1; r += 32) {
      const int2 pr = __ldg(p.probe_rows + r);
      for (int i = 0; i < pr.y; ++i) {
        const int col = __ldg(p.probe_list + pr.x + i).x;
        warp_probes |= col >= c_lo && col < c_hi;
      }
    }
    warp_probes = __any_sync(FULL, warp_probes);
  }
  // the soft source (S2) is applied only by the generic row body: a warp whose strip (halo lanes
  // included) holds the source column takes it for the whole chunk
  const bool warp_source = __any_sync(FULL, x.src_k >= 0) && p.src_row_end > jb - K && p.src_row < je;
  // rows [jb, jm): the first stages' rows precede the chunk; [jm, jend): every stage row is the
  // chunk's own (the fast body, unless the chunk holds a probe row); [jend, je): the last rows.
  // Pairs of rows keep the ping-pong parity; the generic body checks rows at run time.
  // Groups of U rows keep the ping-pong parity and (register ring) the static coefficient slots.
  // UR = 4 (K = 4 fp32 on chunks of >= 256 rows, sweepk_launch): one rotation of the ping-pong
  // registers per four rows instead of two (-4.6 % instructions in the fast loop; at 64-row chunks
  // the longer generic head and tail lose)
  constexpr int U = (FDTD_REG_RING && K > 2) ? K : (UR == 4 ? 4 : 2);
  RowCoef<T, V> rc[K];
#if FDTD_REG_RING
#pragma unroll
  for (int s = 0; s < K; ++s)
#pragma unroll
    for (int k = 0; k < V; ++k)
      rc[s].cax[k] = rc[s].cbx[k] = rc[s].cay[k] = rc[s].cby[k] = rc[s].wx[k] = rc[s].wy[k] = T(0);
#endif
  const int jm = min(jb + ((x.r0 + K - jb + U - 1) / U) * U, je);
  const int jend = (warp_probes || warp_source) ? jm : jm + (max(x.r1 - jm, 0) / U) * U;
  for (int j = jb; j < je; j += U) {
    if (j >= jm && j < jend) {
      sweep_row<T, V, K, ENERGY, false, 0>(p, x, j, je, R1, R0, O0, O1, eacc, rc);
      sweep_row<T, V, K, ENERGY, false, 1>(p, x, j + 1, je, R0, R1, O1, O0, eacc, rc);
      if constexpr (U == 4) {
        sweep_row<T, V, K, ENERGY, false, 2>(p, x, j + 2, je, R1, R0, O0, O1, eacc, rc);
        sweep_row<T, V, K, ENERGY, false, 3>(p, x, j + 3, je, R0, R1, O1, O0, eacc, rc);
      }
    } else {
      sweep_row<T, V, K, ENERGY, true, 0>(p, x, j, je, R1, R0, O0, O1, eacc, rc);
      if (j + 1 < je) sweep_row<T, V, K, ENERGY, true, 1>(p, x, j + 1, je, R0, R1, O1, O0, eacc, rc);
      if constexpr (U == 4) {
        if (j + 2 < je) sweep_row<T, V, K, ENERGY, true, 2>(p, x, j + 2, je, R1, R0, O0, O1, eacc, rc);
        if (j + 3 < je) sweep_row<T, V, K, ENERGY, true, 3>(p, x, j + 3, je, R0, R1, O1, O0, eacc, rc);
      }
    }
    if (ENERGY && !std::is_same<EA, double>::value && ((j - jb) & 15) == 16 - U) {
#pragma unroll
      for (int s = 0; s < K; ++s) {
        dacc[s] += ea_value(eacc[s]);
        ea_zero(eacc[s]);
      }
    }
  }
#pragma unroll
#pragma unroll
  for (int s = 0; s < K; ++s) dacc[s] = x.out ? dacc[s] + ea_value(eacc[s]) : 0.0;
  if (ENERGY) {
    __shared__ double red[K][32];
#pragma unroll
    for (int s = 0; s < K; ++s) {
      double v = dacc[s];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(FULL, v, o);
      if (x.lane == 0) red[s][warp] = v;
    }
    __syncthreads();
    if (threadIdx.x < K) {
      double t = 0.0;
      for (int w = 0; w < wpc; ++w) t += red[threadIdx.x][w];
      p.partials[threadIdx.x * p.pstride + (int64_t)cy * gridDim.x + blockIdx.x] = t;
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

// ---- tensor-core path of the batched reduced GEMMs: FP64 DMMA (mma.sync.m8n8k4.f64), for fp32
// and fp64 states alike.  A (a shared model operator) is kept in fp64 in the pool, pre-tiled in
// the A-fragment order of the m8n8k4 MMA (fdtd_api.cpp push_tiles): per 8 x 4 tile lane l holds
// A[l / 4][l % 4] -- one coalesced 8-byte load per lane and tile (an fp32 copy would halve the L2
// bytes but its per-element widening cost more than it saved: measured).  The batch's vectors X
// (k x B, row stride B; the B instances are the MMA's N = 8 columns) are widened to fp64:
// products and sums are fp64 and only the result is rounded to the state precision (fp32 states
// get a more accurate ROM update than fp32 FMAs would give).  Each output column depends on that
// column only, so a batch's composition never changes an instance's values.
// FDTD_PHASES=1 (a tuning build, tools/phase_times.py): thread 0 of each fix-up CTA stamps
// clock64() at every phase barrier into g_phase (read back with fdtd_debug_phases)
#ifndef FDTD_PHASES
#define FDTD_PHASES 0
#endif
#if FDTD_PHASES
__device__ long long g_phase[4096][72];
__device__ __forceinline__ int& ph_counter() {
  __shared__ int ph;
  return ph;
}
#define PHASE()                                                                                      \
  do {                                                                                               \
    if (threadIdx.x == 0 && blockIdx.x < 4096 && ph_counter() < 72) g_phase[blockIdx.x][ph_counter()++] = clock64(); \
  } while (0)
#else
#define PHASE() \
  do {          \
  } while (0)
#endif
#ifndef FDTD_TPW  // dmma_gemm: row tiles per warp sharing a B fragment; A tiles in flight
#define FDTD_TPW 3
#endif
#ifndef FDTD_UNR
#define FDTD_UNR 4
#endif
#ifndef FDTD_SCHUR16  // Schur solve: 16 loads in flight per thread
#define FDTD_SCHUR16 1
#endif
#ifndef FDTD_REGION_LDG  // region loads: register-staged loads (1) or per-element cp.async (0)
#define FDTD_REGION_LDG 0
#endif
#ifndef FDTD_M2PRE  // M2's operator tiles loaded into registers before the Schur phase
#define FDTD_M2PRE 0  // measured: M2 4 k instead of 6 k cycles, but M1 loses its registers (16 k instead of 10 k)
#endif
#ifndef FDTD_FUSE  // fix-up: five barrier phases per step (M1 beside the H half-step, E beside the gather)
#define FDTD_FUSE 1
#endif
#ifndef FDTD_FUSE2  // whole-grid path: t formed in the gather, the ROM energy in the Schur phase (4 barriers)
#define FDTD_FUSE2 1
#endif
#ifndef BIG_TILES  // large-model path: row tiles of [M1; R~] per CTA processed together in phase 1
#define BIG_TILES 3
#endif
#ifndef FDTD_SKPF  // prefetch the batch's Schur inverses into L2 at the batch start
#define FDTD_SKPF 1
#endif
__device__ __forceinline__ void mma_f64(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// Y = A X for rows [0, m): epi(r, c, v) receives element (r, c) in fp64.  A tiled as above with
// mtiles x ktiles tiles of 8 x 4 (m <= 8 mtiles, k <= 4 ktiles, zero-padded); X in shared memory.
// A warp owns up to TPW row tiles (w, w + nw, ...) of one 8-column tile and walks k once: each
// B fragment is loaded and widened once for all of them, and the next UNR A tiles are in flight
// while the current ones multiply.
template <typename TA, typename T, typename Epi>
__device__ __forceinline__ void dmma_gemm(const TA* __restrict__ At, int mtiles, int ktiles, int m, int k,
                                          const T* X, int B, Epi epi) {
  constexpr int TPW = FDTD_TPW, UNR = FDTD_UNR;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int ntiles = (B + 7) >> 3;
  const int groups = (mtiles + nw * TPW - 1) / (nw * TPW);  // passes over the row tiles
  for (int job = warp; job < groups * nw * ntiles; job += nw) {
    const int grp = job / (nw * ntiles), rem = job % (nw * ntiles);
    const int nt = rem / nw, w = rem % nw;
    const int mt0 = grp * nw * TPW + w;  // this warp's tiles: mt0 + j nw, j < TPW
    const int col = nt * 8 + g;          // this lane's B-fragment column (instance slot)
    const bool cl = col < B;
    double d[TPW][2];
    const TA* ap[TPW];
    bool on[TPW];
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      d[j][0] = d[j][1] = 0.0;
      on[j] = mt0 + j * nw < mtiles;
      ap[j] = At + (int64_t)(on[j] ? mt0 + j * nw : 0) * ktiles * 32 + lane;
    }
    if (!on[0]) continue;
    double a[2][TPW][UNR];
    auto load = [&](int buf, int kt0) {
#pragma unroll
      for (int u = 0; u < UNR; ++u)
#pragma unroll
        for (int j = 0; j < TPW; ++j)
          a[buf][j][u] = (on[j] && kt0 + u < ktiles) ? __ldg(ap[j] + (kt0 + u) * 32) : 0.0;
    };
    load(0, 0);
    for (int kt0 = 0; kt0 < ktiles; kt0 += 2 * UNR) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int kb = kt0 + h * UNR;
        if (kb >= ktiles) break;
        load(h ^ 1, kb + UNR);  // the next UNR tiles in flight
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const int kk = (kb + u) * 4 + t;
          const double b = (cl && kk < k) ? (double)X[kk * B + col] : 0.0;
#pragma unroll
          for (int j = 0; j < TPW; ++j) mma_f64(d[j], a[h][j][u], b);
        }
      }
    }
    const int c0 = nt * 8 + 2 * t;
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      const int r = (mt0 + j * nw) * 8 + g;
      if (on[j] && r < m) {
        if (c0 < B) epi(r, c0, d[j][0]);
        if (c0 + 1 < B) epi(r, c0 + 1, d[j][1]);
      }
    }
  }
}

// Shared-memory vectors of a batch (row stride B, NV rows each):
//   sx = [E~; H~] (q1 + q2), sy = y (nY), sh = h (nY), so = [M1; R~] x (q2 + q1 + nY + q1 + q2, two
//   slots), st = t (nY), sU = U (nY)
constexpr int NROMVEC = 7;  // vector slots of one batch (stride S = (q1 + q2 + nY) x B each)
// the slot stride, rounded up to 4 elements so that the fp64 constants after the slots stay aligned
__host__ __device__ inline int64_t vec_stride(int nvec, int B) { return ((int64_t)nvec * B + 3) / 4 * 4; }
template <typename T>
struct RomVec {
  T *sx, *sy, *sh, *so, *st, *sU;
  __device__ RomVec(T* sv, int64_t S) : sx(sv), sy(sv + S), sh(sv + 2 * S), so(sv + 3 * S), st(sv + 5 * S),
                                         sU(sv + 6 * S) {}
};
// Per-pass constants of a batch, staged in shared memory once per pass (after the vectors):
// eh = D_l D_l' eps / dt (fp64, storage function), cya, cyg = the t coefficients, per (port, slot)
// (nYB = nY x B entries each); then zw, the per-warp zone-energy partials ([slot][ZWARPS] fp64).
constexpr int ZWARPS = 32;
template <typename T>
struct RomConst {
  double* eh; T* cya; T* cyg; double* zw;
  __device__ RomConst(T* sv, int64_t S, int64_t nYB)
      : eh(reinterpret_cast<double*>(sv + NROMVEC * S)),
        cya(sv + NROMVEC * S + nYB * (int64_t)(sizeof(double) / sizeof(T))),
        cyg(sv + NROMVEC * S + nYB * (int64_t)(sizeof(double) / sizeof(T)) + nYB),
        zw(reinterpret_cast<double*>(sv + NROMVEC * S + nYB * (int64_t)(sizeof(double) / sizeof(T)) + 2 * nYB)) {}
};
template <typename T>
__device__ __forceinline__ T* rom_end(T* sv, int64_t S, int64_t nYB, int B) {
  // first free element after the ROM vectors, the per-pass constants and the zone partials
  return sv + NROMVEC * S + nYB * (int64_t)(sizeof(double) / sizeof(T)) + 2 * nYB +
         (int64_t)B * ZWARPS * (int64_t)(sizeof(double) / sizeof(T));
}

// One ROM step for a batch of nb (<= B) instances of one model (eq:connExplicit, K3).
// On entry sx (x~^n), sy (y^n), sh (h = Hz^{n+1/2} of the outside cells) hold the batch's vectors
// (zero padding for b >= nb).  On exit sx holds x~^{n+1} and sy holds y^{n+1}; with ENERGY the ROM
// part of W^n (coarse half cells + x~^T R~ x~) of instance b is in eout[b].  Four phases: M1 GEMM |
// energy + t | Schur solve | M2 GEMM with the base added in its epilogue (fp32: tensor cores).
template <typename T, bool ENERGY>
__device__ void rom_step(const PostParams<T>& p, const RomModelDev& m, const int32_t* mem, int nb, int B, int64_t S,
                         T* sv, double* ep) {
  const int nY = m.nY, q1 = m.q1, q2 = m.q2, nx = q1 + q2, m1 = q2 + q1 + nY, m2 = q1 + nY;
  const int tid = threadIdx.x, nt = blockDim.x;
  RomVec<T> v(sv, S);
  const RomConst<T> rc(sv, S, (int64_t)nY * B);
  // [H~^{n+1}; E*; -L~^T E*] = M1 x~^n, and with ENERGY also R~ x~^n (R~ is stored after M1 as
  // q1 + q2 further rows of the same operator: one GEMM phase); so is overwritten
  {
    T* so = v.so;
    dmma_gemm(p.mpool + m.off_M1t, ENERGY ? m.mt1 : (m1 + 7) / 8, m.kt1, ENERGY ? m1 + nx : m1, nx, v.sx, B,
              [&](int r, int c, double x) { so[r * B + c] = (T)x; });
  }
  __syncthreads();
  PHASE();
  if (ENERGY) {  // x~^T R~ x~ + sum D_l D_l' eps/dt y^2 (storage function, R17); one warp per instance
    const int lane = tid & 31, w = tid >> 5, nw = nt >> 5;
    for (int b = w; b < nb; b += nw) {
      double acc = 0.0;
      for (int i = lane; i < nY; i += 32) {
        const double y = (double)v.sy[i * B + b];
        acc += rc.eh[i * B + b] * y * y;
      }
      for (int i = lane; i < nx; i += 32) acc += (double)v.sx[i * B + b] * (double)v.so[(m1 + i) * B + b];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(FULL, acc, o);
      if (lane == 0) ep[mem[b]] = acc;
    }
  }
  // t = (a_y/c_y) y + (D_l G/c_y) h - L~^T E*
  for (int it = tid; it < nY * nb; it += nt) {
    const int i = it % nY, b = it / nY;
    const int k = i * B + b;
    v.st[k] = v.so[(q2 + q1 + i) * B + b] + fma_rn(rc.cyg[k], v.sh[k], mul_rn(rc.cya[k], v.sy[k]));
  }
  __syncthreads();
  PHASE();
  // M2's operator tiles, when every warp holds at most one of at most 16 k-tiles: loaded now, in
  // flight during the Schur phase (the M2 phase then waits on no L2 round trip)
  const int lane = tid & 31, warp = tid >> 5, nwarp = nt >> 5;
  const bool pre2 = FDTD_M2PRE && m.mt2 <= nwarp && m.kt2 <= 16 && B <= 8;
  double a2[16];
  if (pre2) {
    const double* ap = p.mpool + m.off_M2t + (int64_t)(warp < m.mt2 ? warp : 0) * m.kt2 * 32 + lane;
#pragma unroll
    for (int k = 0; k < 16; ++k) a2[k] = (k < m.kt2 && warp < m.mt2) ? __ldg(ap + k * 32) : 0.0;
  }
  // U = S_k t (per-instance Schur inverse, L2-resident after the prefetch at the batch start)
  for (int it = tid; it < nY * nb; it += nt) {
    const int i = it % nY, b = it / nY;
    const T* Sk = p.Sk + p.Sk_off[mem[b]] + i;
    T a[4] = {T(0), T(0), T(0), T(0)};  // four interleaved partial sums: a quarter of the FMA chain
    int c = 0;
    for (; FDTD_SCHUR16 && c + 15 < nY; c += 16) {  // 16 loads in flight, then their FMAs
      T sk[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) sk[u] = __ldg(Sk + (int64_t)(c + u) * nY);
#pragma unroll
      for (int u = 0; u < 16; ++u) a[u & 3] = fma_rn(sk[u], v.st[(c + u) * B + b], a[u & 3]);
    }
    for (; c + 3 < nY; c += 4)
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] = fma_rn(__ldg(Sk + (int64_t)(c + u) * nY), v.st[(c + u) * B + b], a[u]);
    for (; c < nY; ++c) a[0] = fma_rn(__ldg(Sk + (int64_t)c * nY), v.st[c * B + b], a[0]);
    v.sU[i * B + b] = (a[0] + a[1]) + (a[2] + a[3]);
  }
  __syncthreads();
  PHASE();
  // [E~^{n+1}; y^{n+1}] = [E*; L~^T E*] + M2 U (the base added in fp64 in the epilogue; literal:
  // y' = the U rows themselves), and H~^{n+1} = so rows 0 .. q2 copied beside it
  {
    T* sx = v.sx;
    T* sy = v.sy;
    const T* so = v.so;
    const bool lit = m.literal != 0;
    auto epi = [&](int r, int c, double x) {
      if (r < q1) sx[r * B + c] = (T)((double)so[(q2 + r) * B + c] + x);
      else sy[(r - q1) * B + c] = (T)((lit ? 0.0 : -(double)so[(q2 + r) * B + c]) + x);
    };
    if (pre2) {
      if (warp < m.mt2) {  // the same DMMA sequence as dmma_gemm's, from the preloaded tiles
        const int g = lane >> 2, t4 = lane & 3;
        double d[2] = {0.0, 0.0};
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (k < m.kt2) {
            const int kk = k * 4 + t4;
            mma_f64(d, a2[k], (g < B && kk < nY) ? (double)v.sU[kk * B + g] : 0.0);
          }
        const int r = warp * 8 + g, c0 = 2 * t4;
        if (r < m2) {
          if (c0 < B) epi(r, c0, d[0]);
          if (c0 + 1 < B) epi(r, c0 + 1, d[1]);
        }
      }
    } else {
      dmma_gemm(p.mpool + m.off_M2t, m.mt2, m.kt2, m2, nY, v.sU, B, epi);
    }
    for (int64_t k = tid; k < (int64_t)q2 * B; k += nt) sx[(int64_t)q1 * B + k] = so[k];
  }
  __syncthreads();
  PHASE();
}

// The same ROM step split into the phases the fused fix-up step schedules beside its region work
// (FDTD_FUSE, K3): rom_m1 (M1 GEMM; needs x~ only), rom_t (energy + t; needs the gathered y
// and h), rom_schur (U = S_k t), rom_m2 (M2 GEMM, the base added in its epilogue, which also hands
// each y^{n+1} to scat(port, slot, y) -- the scatter into the region's interface edge -- and H~
// copied).  The caller puts a barrier between consecutive phases.
template <typename T, bool ENERGY>
__device__ __forceinline__ void rom_m1(const PostParams<T>& p, const RomModelDev& m, int B, int64_t S, T* sv) {
  const int nY = m.nY, q1 = m.q1, q2 = m.q2, nx = q1 + q2, m1 = q2 + q1 + nY;
  RomVec<T> v(sv, S);
  T* so = v.so;
  dmma_gemm(p.mpool + m.off_M1t, ENERGY ? m.mt1 : (m1 + 7) / 8, m.kt1, ENERGY ? m1 + nx : m1, nx, v.sx, B,
            [&](int r, int c, double x) { so[r * B + c] = (T)x; });
}
template <typename T, bool ENERGY>
__device__ __forceinline__ void rom_t(const RomModelDev& m, const int32_t* mem, int nb, int B, int64_t S, T* sv,
                                      double* ep) {
  const int nY = m.nY, q1 = m.q1, q2 = m.q2, nx = q1 + q2, m1 = q2 + q1 + nY;
  const int tid = threadIdx.x, nt = blockDim.x;
  RomVec<T> v(sv, S);
  const RomConst<T> rc(sv, S, (int64_t)nY * B);
  if (ENERGY) {  // x~^T R~ x~ + sum D_l D_l' eps/dt y^2 (storage function, R17); one warp per instance
    const int lane = tid & 31, w = tid >> 5, nw = nt >> 5;
    for (int b = w; b < nb; b += nw) {
      double acc = 0.0;
      for (int i = lane; i < nY; i += 32) {
        const double y = (double)v.sy[i * B + b];
        acc += rc.eh[i * B + b] * y * y;
      }
      for (int i = lane; i < nx; i += 32) acc += (double)v.sx[i * B + b] * (double)v.so[(m1 + i) * B + b];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(FULL, acc, o);
      if (lane == 0) ep[mem[b]] = acc;
    }
  }
  for (int it = tid; it < nY * nb; it += nt) {  // t = (a_y/c_y) y + (D_l G/c_y) h - L~^T E*
    const int i = it % nY, b = it / nY;
    const int k = i * B + b;
    v.st[k] = v.so[(q2 + q1 + i) * B + b] + fma_rn(rc.cyg[k], v.sh[k], mul_rn(rc.cya[k], v.sy[k]));
  }
}
// The storage-function part of rom_t alone (FDTD_FUSE2: t is formed by the gather), one warp per
// instance; plus z(b) (the zone energy of the member's region, or 0) added by its lane 0 -- the
// same two fp64 additions rom_t and the zone add make.
template <typename T, bool ENERGY, typename Z>
__device__ __forceinline__ void rom_energy(const RomModelDev& m, const int32_t* mem, int nb, int B, int64_t S, T* sv,
                                           double* ep, Z z) {
  if (!ENERGY) return;
  const int nY = m.nY, q1 = m.q1, q2 = m.q2, nx = q1 + q2, m1 = q2 + q1 + nY;
  const int tid = threadIdx.x, nt = blockDim.x;
  RomVec<T> v(sv, S);
  const RomConst<T> rc(sv, S, (int64_t)nY * B);
  const int lane = tid & 31, w = tid >> 5, nw = nt >> 5;
  for (int b = w; b < nb; b += nw) {
    double acc = 0.0;
    for (int i = lane; i < nY; i += 32) {
      const double y = (double)v.sy[i * B + b];
      acc += rc.eh[i * B + b] * y * y;
    }
    for (int i = lane; i < nx; i += 32) acc += (double)v.sx[i * B + b] * (double)v.so[(m1 + i) * B + b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(FULL, acc, o);
    if (lane == 0) {
      ep[mem[b]] = acc;
      ep[mem[b]] += z(b);
    }
  }
}

template <typename T>
__device__ __forceinline__ void rom_schur(const PostParams<T>& p, const RomModelDev& m, const int32_t* mem, int nb,
                                          int B, int64_t S, T* sv) {
  const int nY = m.nY;
  const int tid = threadIdx.x, nt = blockDim.x;
  RomVec<T> v(sv, S);
  for (int it = tid; it < nY * nb; it += nt) {  // U = S_k t (as in rom_step)
    const int i = it % nY, b = it / nY;
    const T* Sk = p.Sk + p.Sk_off[mem[b]] + i;
    T a[4] = {T(0), T(0), T(0), T(0)};
    int c = 0;
    for (; c + 15 < nY; c += 16) {
      T sk[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) sk[u] = __ldg(Sk + (int64_t)(c + u) * nY);
#pragma unroll
      for (int u = 0; u < 16; ++u) a[u & 3] = fma_rn(sk[u], v.st[(c + u) * B + b], a[u & 3]);
    }
    for (; c + 3 < nY; c += 4)
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] = fma_rn(__ldg(Sk + (int64_t)(c + u) * nY), v.st[(c + u) * B + b], a[u]);
    for (; c < nY; ++c) a[0] = fma_rn(__ldg(Sk + (int64_t)c * nY), v.st[c * B + b], a[0]);
    v.sU[i * B + b] = (a[0] + a[1]) + (a[2] + a[3]);
  }
}
template <typename T, typename Scat>
__device__ __forceinline__ void rom_m2(const PostParams<T>& p, const RomModelDev& m, int nb, int B, int64_t S, T* sv,
                                       Scat scat) {
  const int nY = m.nY, q1 = m.q1, q2 = m.q2, m2 = q1 + nY;
  const int tid = threadIdx.x, nt = blockDim.x;
  RomVec<T> v(sv, S);
  T* sx = v.sx;
  T* sy = v.sy;
  const T* so = v.so;
  const bool lit = m.literal != 0;
  auto epi = [&](int r, int c, double x) {
    if (r < q1) {
      sx[r * B + c] = (T)((double)so[(q2 + r) * B + c] + x);
    } else {
      const T y = (T)((lit ? 0.0 : -(double)so[(q2 + r) * B + c]) + x);
      sy[(r - q1) * B + c] = y;
      if (c < nb) scat(r - q1, c, y);
    }
  };
  dmma_gemm(p.mpool + m.off_M2t, m.mt2, m.kt2, m2, nY, v.sU, B, epi);
  for (int64_t k = tid; k < (int64_t)q2 * B; k += nt) sx[(int64_t)q1 * B + k] = so[k];
}

// ---- the large-model path (one instance at a time on the whole GPU; fdtd_api.cpp "big" models):
// a cooperative grid of one CTA per SM evaluates the ROM step of one instance, CTA 0 doing the
// region work of fixup_batch.  Scratch in global memory (p.big): x~ in two buffers X0 / X1 (the
// pass input stays in p.state until the pass ends), SO = [M1; R~] x~ (m1 + q1 + q2 rows), YH = the
// gathered y and h (nY each).  Two grid barriers per step:
//   phase 1: SO = [M1; R~] x~ -- every 8-row tile on one CTA (CTAs 1.. when there are several),
//            split over its warps along k (fixed-order sum of the warps' partials); CTA 0 publishes y, h;
//   phase 2: t and U = S_k t (every CTA, redundantly), E~' = E* + (M2 U) rows on CTAs 1..,
//            y' rows and the storage-function term on CTA 0, H~' copied;
// CTA 0 then scatters y' and takes the E half-step while the others start the next step's M1.
template <typename T>
struct BigScratch {
  T *X0, *X1, *SO, *YH;
  __device__ BigScratch(T* big, const RomModelDev& m) {
    const int nx = m.q1 + m.q2, m1 = m.q2 + m.q1 + m.nY;
    X0 = big; X1 = big + nx; SO = big + 2 * nx; YH = SO + m1 + nx;
  }
};

template <typename T, bool ENERGY>
__device__ void rom_step_big(const PostParams<T>& p, const RomModelDev& m, const int32_t* mem, int s, T* sv,
                             int64_t S, double* ep, double* part) {
  const int first = mem[0];
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int nY = m.nY, q1 = m.q1, q2 = m.q2, nx = q1 + q2, m1 = q2 + q1 + nY, m2 = q1 + nY;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int G = gridDim.x, cta = blockIdx.x;
  const bool rg = cta == 0;
  const int G1 = G > 1 ? G - 1 : 1, c1 = G > 1 ? cta - 1 : 0;  // CTA 0 keeps to its region when G > 1
  const bool worker = G == 1 || cta > 0;
  const BigScratch<T> bsc(p.big, m);
  const T* xin = s == 0 ? p.state + p.state_off[first] : ((s - 1) & 1 ? bsc.X1 : bsc.X0);
  T* xout = (s & 1) ? bsc.X1 : bsc.X0;
  RomVec<T> v(sv, S);
  const double* mp = p.mpool;
  // ---- phase 1: SO = [M1; R~] x~ (with ENERGY all m1 + nx rows)
  const int rows1 = ENERGY ? m1 + nx : m1, mt1 = (rows1 + 7) / 8, kt1 = m.kt1;
  if (worker) {
    // the CTA's row tiles (c1, c1 + G1, ...) BT at a time: warp w takes k-tiles [ka, kb) of every one
    // of them (each tile's DMMA chain and the fixed-order sum over the warps as one tile alone), so
    // BT x 8 A-tile loads are in flight per warp instead of 8
    constexpr int BT = BIG_TILES;
    const int kpw = (kt1 + nw - 1) / nw;
    const int ka = warp * kpw, kb = min(ka + kpw, kt1);
    for (int tile0 = c1; tile0 < mt1; tile0 += BT * G1) {
      const double* ap[BT];
      bool on[BT];
      double d[BT][2];
#pragma unroll
      for (int j = 0; j < BT; ++j) {
        const int tile = tile0 + j * G1;
        on[j] = tile < mt1;
        ap[j] = mp + m.off_M1t + (int64_t)(on[j] ? tile : 0) * kt1 * 32 + lane;
        d[j][0] = d[j][1] = 0.0;
      }
      int kt = ka;
      for (; kt + 8 <= kb; kt += 8) {
        double a[BT][8], b[8];
#pragma unroll
        for (int j = 0; j < BT; ++j)
#pragma unroll
          for (int u = 0; u < 8; ++u) a[j][u] = on[j] ? (double)__ldg(ap[j] + (kt + u) * 32) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int kk = (kt + u) * 4 + t4;
          b[u] = (g == 0 && kk < nx) ? (double)xin[kk] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < BT; ++j)
#pragma unroll
          for (int u = 0; u < 8; ++u) mma_f64(d[j], a[j][u], b[u]);
      }
      for (; kt < kb; ++kt) {
        const int kk = kt * 4 + t4;
        const double b = (g == 0 && kk < nx) ? (double)xin[kk] : 0.0;
#pragma unroll
        for (int j = 0; j < BT; ++j)
          if (on[j]) mma_f64(d[j], (double)__ldg(ap[j] + kt * 32), b);
      }
#pragma unroll
      for (int j = 0; j < BT; ++j)
        if (t4 == 0) part[(warp * BT + j) * 8 + g] = d[j][0];  // column 0 (the instance) of rows tile*8 + g
      __syncthreads();
      if (tid < 8 * BT) {
        const int j = tid / 8, r8 = tid % 8;
        double acc = 0.0;
        for (int w = 0; w < nw; ++w) acc += part[(w * BT + j) * 8 + r8];
        const int r = (tile0 + j * G1) * 8 + r8;
        if (tile0 + j * G1 < mt1 && r < rows1) bsc.SO[r] = (T)acc;
      }
      __syncthreads();
    }
  }
  if (rg)
    for (int i = tid; i < nY; i += nt) {
      bsc.YH[i] = v.sy[i];
      bsc.YH[nY + i] = v.sh[i];
    }
  PHASE();
  grid.sync();
  PHASE();
  // ---- phase 2
  const RomConst<T> rc(sv, S, (int64_t)nY);
  // storage function of the instance on the last CTA (it holds no M2 tile; CTA 0 is busiest): every
  // warp sums a slice of x~^T R~ x~ (global scratch: all loads in flight), the fixed-order sum of
  // the warps follows the Schur phase's barriers
  const bool ecta = G > 1 ? cta == G - 1 : true;
  if (ENERGY && ecta) {
    double acc = 0.0;
    if (warp == 0) {
      const int64_t po = p.port_off[first];
      for (int i = lane; i < nY; i += 32) {
        const double y = (double)bsc.YH[i];
        acc += p.ehalf[po + i] * y * y;
      }
    }
    const int per = (nx + nw - 1) / nw, i0 = warp * per, i1 = min(nx, i0 + per);
    for (int i = i0 + lane; i < i1; i += 32) acc += (double)xin[i] * (double)bsc.SO[m1 + i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(FULL, acc, o);
    if (lane == 0) part[warp] = acc;
  }
  {  // t and U = S_k t, in every CTA
    const int64_t po = p.port_off[first];
    for (int i = tid; i < nY; i += nt)
      v.st[i] = bsc.SO[q2 + q1 + i] + fma_rn(p.cyg[po + i], bsc.YH[nY + i], mul_rn(p.cya[po + i], bsc.YH[i]));
    __syncthreads();
    // U = S_k t: warp w sums the columns [w cw, (w + 1) cw) for every row (lanes along the rows:
    // coalesced column loads, all in flight at once), the warps' partials then in a fixed order
    // (partials in the unused `so` slots of the vector area: 2 S elements)
    const int pw = max(1, min(nw, (int)((2 * S * (int64_t)sizeof(T)) / (8 * (int64_t)nY))));
    const int cw = (nY + pw - 1) / pw;
    double* sp = reinterpret_cast<double*>(v.so);
    if (warp < pw) {
      const T* Sk = p.Sk + p.Sk_off[first];
      const int c0 = warp * cw, c1e = min(nY, c0 + cw);
      for (int i = lane; i < nY; i += 32) {
        T a[4] = {T(0), T(0), T(0), T(0)};
        int c = c0;
        for (; c + 3 < c1e; c += 4)
#pragma unroll
          for (int u = 0; u < 4; ++u) a[u] = fma_rn(__ldg(Sk + (int64_t)(c + u) * nY + i), v.st[c + u], a[u]);
        for (; c < c1e; ++c) a[0] = fma_rn(__ldg(Sk + (int64_t)c * nY + i), v.st[c], a[0]);
        sp[warp * nY + i] = (double)((a[0] + a[1]) + (a[2] + a[3]));
      }
    }
    __syncthreads();
    for (int i = tid; i < nY; i += nt) {
      double u = 0.0;
      for (int w = 0; w < pw; ++w) u += sp[w * nY + i];
      v.sU[i] = (T)u;
    }
    __syncthreads();
    if (ENERGY && ecta && tid == 0) {  // (part holds the energy warps' sums; reused after the grid barriers)
      double e = 0.0;
      for (int w = 0; w < nw; ++w) e += part[w];
      ep[first] = e;
    }
    PHASE();
  }
  // [E~'; y'] = [E*; L~^T E*] + M2 U: the tiles holding y rows on CTA 0 (it scatters y'), the others
  // one warp each on CTAs 1..
  const int mt2 = m.mt2, kt2 = m.kt2, ty = q1 / 8;  // tiles >= ty hold y rows
  const bool lit = m.literal != 0;
  auto m2_tile = [&](int tile) {
    const double* ap = mp + m.off_M2t + (int64_t)tile * kt2 * 32 + lane;
    double d[2] = {0.0, 0.0};
    int kt = 0;
    for (; kt + 8 <= kt2; kt += 8) {  // eight A tiles in flight, then their MMAs (the same order)
      double a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = (double)__ldg(ap + (kt + u) * 32);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int kk = (kt + u) * 4 + t4;
        mma_f64(d, a[u], (g == 0 && kk < nY) ? (double)v.sU[kk] : 0.0);
      }
    }
    for (; kt < kt2; ++kt) {
      const int kk = kt * 4 + t4;
      mma_f64(d, (double)__ldg(ap + kt * 32), (g == 0 && kk < nY) ? (double)v.sU[kk] : 0.0);
    }
    const int r = tile * 8 + g;
    if (t4 == 0 && r < m2) {
      if (r < q1) xout[r] = (T)((double)bsc.SO[q2 + r] + d[0]);
      else v.sy[r - q1] = (T)((lit ? 0.0 : -(double)bsc.SO[q2 + r]) + d[0]);
    }
  };
  if (rg) {
    __syncthreads();  // the energy above read sy
    for (int tile = ty + warp; tile < mt2; tile += nw) m2_tile(tile);
  }
  if (worker)
    for (int tile = c1 * nw + warp; tile < ty; tile += G1 * nw) m2_tile(tile);
  if (worker)
    for (int r = c1 * nt + tid; r < q2; r += G1 * nt) xout[q1 + r] = bsc.SO[r];
  PHASE();
  grid.sync();
}

template <typename T>
__device__ void load_rom_state(const PostParams<T>& p, const RomModelDev& m, const int32_t* mem, int nb, int B, T* sv) {
  T* sx = sv;
  const int nx = m.q1 + m.q2;
  for (int it = threadIdx.x; it < nx * nb; it += blockDim.x) {
    const int i = it % nx, b = it / nx;
    sx[i * B + b] = p.state[p.state_off[mem[b]] + i];
  }
}

template <typename T>
__device__ void store_rom(const PostParams<T>& p, const RomModelDev& m, const int32_t* mem, int nb, int B, int64_t S,
                          const T* sv, T* ex, T* ey) {
  const T* sx = sv;
  const T* sy = sv + S;
  for (int it = threadIdx.x; it < m.nY * nb; it += blockDim.x) {  // S6: scatter y^{n+1}
    const int i = it % m.nY, b = it / m.nY;
    const int64_t e = p.port_edge[p.port_off[mem[b]] + i];
    FCHK((e & IDX_MASK) >= (int64_t)p.row0 * p.pitch && (e & IDX_MASK) < (int64_t)(p.row0 + p.rows) * p.pitch);
    if (e >> 62) ey[e & IDX_MASK] = sy[i * B + b];
    else ex[e & IDX_MASK] = sy[i * B + b];
  }
  const int nx = m.q1 + m.q2;
  bool bad = false;
  for (int it = threadIdx.x; it < nx * nb; it += blockDim.x) {
    const int i = it % nx, b = it / nx;
    const T v = sx[i * B + b];
    bad |= !isfinite(v);
    p.state[p.state_off[mem[b]] + i] = v;
  }
  if (bad) *p.flag = 1;  // non-finite sentinel (a ROM blow-up reaches the state first)
}

// K3: the K-step fix-up of one batch (instances of one model).  The sweep advanced every cell K
// steps with the interface edges frozen at y^n; here, per instance, the K steps are recomputed
// on the region [i0-M, i0+bx+M) x [j0-M, j0+by+M), M = Kz + K - 1, from the pass's input buffer
// with the sweep's own arithmetic (yee_row's device functions), and between the H and E half
// steps the ROM takes its step (S4 gather, S5 eq:connExplicit, S6 scatter).  Values in the
// region go wrong from its border inwards by one cell per step, so after K steps every cell
// within Kz of the block is exact.  Written back: the zone cells (block + Kz - 1 rings, + one
// more column / row on the right / top, holes excluded) with their bottom Ex and left Ey edges;
// y^{n+K}; the ROM state.  Their energy (which the sweep skipped) and the zone probes are
// recorded here for every step of the pass.
// (b, v, u) walked over nb instances x a ch x cw cell window [v0, v0 + ch) x [u0, u0 + cw), thread
// tid first, nt apart, advanced incrementally (no division per cell).  All instances of a batch
// share one model, hence one region shape: the batch's regions are one flat index space.
struct Flat {
  int u, v, b, du, dv, db, u0, cw, v0, ch;
  __device__ __forceinline__ Flat(int tid, int nt, int u0_, int cw_, int v0_, int ch_)
      : u0(u0_), cw(cw_), v0(v0_), ch(ch_) {
    const int per = cw * ch;
    b = tid / per;
    const int r = tid % per;
    v = v0 + r / cw;
    u = u0 + r % cw;
    db = nt / per;
    const int rr = nt % per;
    dv = rr / cw;
    du = rr % cw;
  }
  __device__ __forceinline__ void next() {
    u += du;
    v += dv;
    b += db;
    if (u >= u0 + cw) { u -= cw; ++v; }
    if (v >= v0 + ch) { v -= ch; ++b; }
  }
};

// per-region / per-member constants of a batch (static shared memory of the fix-up kernels)
constexpr int MAXB = 64;  // largest batch (FDTD_ROM_BATCH; a cluster's members)
struct BatchShared {
  int64_t gi0[MAXB], gj0[MAXB];        // global cell (column, row) of region cell (0, 0)
  int64_t gbase[MAXB];                 // its device element offset
  int su[MAXB], sv0[MAXB], sv1[MAXB];  // the source cells in region coordinates (su = -1: none)
  int rr[MAXB], bu[MAXB], bv[MAXB];    // member b: its region, its block's lower-left cell there
  double zsum[MAXB];                   // zone energy per region
};

// K3: the K-step fix-up of one batch (instances of one model).  The sweep advanced every cell K
// steps with the interface edges frozen at y^n; here the K steps are recomputed on each region
// from the pass's input buffer with the sweep's own arithmetic (yee_row's device functions), and
// between the H and E half steps every member's ROM takes its step (S4 gather, S5
// eq:connExplicit, S6 scatter).  A batch's regions are either one per member (kind 0:
// [i0-M, i0+bx+M) x [j0-M, j0+by+M), M = Kz + K - 1) or one shared by all members (kind 1: a
// cluster of instances closer than the pass depth allows; the region is their bounding box + M,
// DESIGN.md "Pass depth").  Values in a region go wrong from its border inwards by one cell per
// step, so after K steps every cell within Kz of the blocks is exact.  Written back: the zone of
// each region (block or bounding box + Kz - 1 rings, + one more column / row on the right / top,
// holes excluded) with the cells' bottom Ex and left Ey edges; y^{n+K}; the ROM states.  The
// zones' energy (which the sweep skipped) and the zone probes are recorded here for every step of
// the pass.  Cells outside the grid (walls) load as dead cells with zero fields.  Every region
// phase runs over the whole batch at once.
// WHOLE (wholegrid_kernel, K3c): the batch is every instance of the grid around one
// region that is the whole grid plus a one-cell ring of dead wall cells, so nothing in it goes
// wrong at its border: nsteps steps run back to back (no cone), every cell is a zone cell (energy,
// probes from p.wprobe, write-back of every cell and edge), and each step's W^n goes straight to
// the energy ring.
template <typename T, int K, bool ENERGY, bool BIG = false, bool WHOLE = false>
__device__ void fixup_batch(const PostParams<T>& p, int bi, T* sv, const T (&g)[K], int64_t step, BatchShared& bs,
                            double* part = nullptr, int64_t nsteps = K) {
  const int* bt = p.batch_tab + BATCH_FIELDS * bi;  // (model, member offset, count, slots B, region stride, kind)
  const int model = bt[0], nb = bt[2], B = bt[3], rstride = bt[4], kind = bt[5];
  const int32_t* mem = p.batch_inst + bt[1];
  const RomModelDev m = p.models[model];
  const int nY = m.nY;
  const int64_t S = vec_stride(m.q1 + m.q2 + nY, B);  // vector stride of this batch's layout
  const int tid = threadIdx.x, nt = blockDim.x;
  // BIG (one instance on the whole cooperative grid): only CTA 0 holds the region; the others take
  // part in the ROM step only (nr = nreg = 0 empties every region loop of theirs)
  const bool rg = !BIG || blockIdx.x == 0;
  const int nr = rg ? nb : 0;
  const int nreg = rg ? (kind ? 1 : nb) : 0;
  const int64_t nYB = (int64_t)nY * B;
  T* reg = rom_end(sv, S, nYB, B);
  const RomConst<T> rc(sv, S, nYB);
  const int Kz = p.Kz, M = WHOLE ? 1 : Kz + K - 1;
  const int64_t P = p.pitch;
  // the members' blocks (one model: bx x by); the region's block: a member's, or the cluster's box
  const int bx = p.rects[4 * (int64_t)mem[0] + 2], by = p.rects[4 * (int64_t)mem[0] + 3];
  const int rbx = kind ? p.batch_rect[4 * bi + 2] : bx, rby = kind ? p.batch_rect[4 * bi + 3] : by;
  const int Wr = rbx + 2 * M, Hr = rby + 2 * M, W1 = Wr + 1, n = Hr * Wr;
  int zu0 = 0, zu1 = 0, zv0 = 0, zv1 = 0;
  if (WHOLE) {  // every cell of the grid
    zu0 = M; zu1 = M + rbx; zv0 = M; zv1 = M + rby;
  } else if (Kz >= 2) {  // zone rectangle in region coordinates
    zu0 = M - (Kz - 1); zu1 = M + rbx + Kz; zv0 = M - (Kz - 1); zv1 = M + rby + Kz;
  }
  const int zw = zu1 - zu0, nz = zw * (zv1 - zv0);
  auto H = [&](int r) { return reg + (int64_t)r * rstride; };
  auto MA = [&](int r) { return reg + (int64_t)r * rstride + n; };
  auto MS = [&](int r) { return reg + (int64_t)r * rstride + 2 * n; };
  auto EX = [&](int r) { return reg + (int64_t)r * rstride + 3 * n; };
  auto EY = [&](int r) { return reg + (int64_t)r * rstride + 4 * n + Wr; };
  auto ZE = [&](int r) { return reg + (int64_t)r * rstride + 4 * n + Wr + Hr * W1; };
  FCHK(4 * n + Wr + Hr * W1 + nz <= rstride &&
       (size_t)((char*)(reg + (int64_t)(kind ? 1 : B) * rstride) - (char*)sv) <= (BIG ? p.big_smem_bytes : p.smem_bytes));
  for (int64_t k = tid; rg && k < NROMVEC * S; k += nt) sv[k] = T(0);
  for (int r = tid; r < nreg; r += nt) {
    const int32_t* q = kind ? p.batch_rect + 4 * bi : p.rects + 4 * (int64_t)mem[r];
    const int64_t i0 = (int64_t)q[0] - M, j0 = (int64_t)q[1] - M;  // global cell of region cell (0, 0)
    const int64_t lr0 = j0 - p.row_begin + p.row0;                  // its local row
    bs.gi0[r] = i0;
    bs.gj0[r] = j0;
    bs.gbase[r] = lr0 * P + i0;
    FCHK(lr0 >= 0 || j0 < 0);  // region rows below the slab only where the grid ends
    const int64_t cu = p.src_col - i0;
    const bool hit = p.src_row >= 0 && cu >= 0 && cu < Wr;
    bs.su[r] = hit ? (int)cu : -1;
    bs.sv0[r] = hit ? (int)max(p.src_row - lr0, (int64_t)0) : 0;
    bs.sv1[r] = hit ? (int)min(p.src_row_end - lr0, (int64_t)Hr) : 0;
  }
  for (int b = tid; b < nr; b += nt) {  // members: region and block position
    const int32_t* q = p.rects + 4 * (int64_t)mem[b];
    const int32_t* o = kind ? p.batch_rect + 4 * bi : q;
    bs.rr[b] = kind ? 0 : b;
    bs.bu[b] = q[0] - o[0] + M;
    bs.bv[b] = q[1] - o[1] + M;
  }
  __syncthreads();  // the zero padding lands before load_rom_state fills the live slots
  PHASE();
  T* sy = sv + S;
  T* sh = sv + 2 * S;
  // ---- load the regions: materials and the fields at step n (asynchronous element copies, all in
  // flight at once: the region rows are not 16-byte aligned).  Outside the grid: dead cells (the
  // PEC walls), zero fields.
  const int64_t NX = p.nx, NY = p.ny;
#if FDTD_REGION_LDG
  // loads into registers, RU cells at a time per thread (all in flight), then the stores
  constexpr int RU = 4;
  for (Flat f(tid, nt, 0, Wr, 0, Hr); f.b < nreg;) {
    int64_t o[RU];
    int tt[RU], rr[RU];
    bool in[RU];
#pragma unroll
    for (int k = 0; k < RU; ++k) {
      in[k] = false;
      rr[k] = -1;
      if (f.b < nreg) {
        const int64_t gi = bs.gi0[f.b] + f.u, gj = bs.gj0[f.b] + f.v;
        in[k] = gi >= 0 && gi < NX && gj >= 0 && gj < NY;
        o[k] = bs.gbase[f.b] + (int64_t)f.v * P + f.u;
        tt[k] = f.v * Wr + f.u;
        rr[k] = f.b;
        f.next();
      }
    }
    T a[RU], b[RU], h[RU];
#pragma unroll
    for (int k = 0; k < RU; ++k)
      if (in[k]) { a[k] = __ldg(p.mea + o[k]); b[k] = __ldg(p.msb + o[k]); h[k] = __ldg(p.hz0 + o[k]); }
      else { a[k] = T(-1); b[k] = T(0); h[k] = T(0); }
#pragma unroll
    for (int k = 0; k < RU; ++k)
      if (rr[k] >= 0) { MA(rr[k])[tt[k]] = a[k]; MS(rr[k])[tt[k]] = b[k]; H(rr[k])[tt[k]] = h[k]; }
  }
  for (int e = 0; e < 2; ++e) {  // Ex edge rows (Hr + 1 rows x Wr), Ey edge columns (Hr rows x Wr + 1)
    const int cw = e ? W1 : Wr, chh = e ? Hr : Hr + 1, pw = e ? W1 : Wr;
    const T* src = e ? p.ey0 : p.ex0;
    for (Flat f(tid, nt, 0, cw, 0, chh); f.b < nreg;) {
      int64_t o[2 * RU];
      int tt[2 * RU], rr[2 * RU];
      bool in[2 * RU];
#pragma unroll
      for (int k = 0; k < 2 * RU; ++k) {
        in[k] = false;
        rr[k] = -1;
        if (f.b < nreg) {
          const int64_t gi = bs.gi0[f.b] + f.u, gj = bs.gj0[f.b] + f.v;
          in[k] = e ? (gi >= 0 && gi <= NX && gj >= 0 && gj < NY) : (gi >= 0 && gi < NX && gj >= 0 && gj <= NY);
          o[k] = bs.gbase[f.b] + (int64_t)f.v * P + f.u;
          tt[k] = f.v * pw + f.u;
          rr[k] = f.b;
          f.next();
        }
      }
      T x[2 * RU];
#pragma unroll
      for (int k = 0; k < 2 * RU; ++k) x[k] = in[k] ? __ldg(src + o[k]) : T(0);
#pragma unroll
      for (int k = 0; k < 2 * RU; ++k)
        if (rr[k] >= 0) (e ? EY(rr[k]) : EX(rr[k]))[tt[k]] = x[k];
    }
  }
#else
  for (Flat f(tid, nt, 0, Wr, 0, Hr); f.b < nreg; f.next()) {
    const int t = f.v * Wr + f.u;
    const int64_t gi = bs.gi0[f.b] + f.u, gj = bs.gj0[f.b] + f.v;
    if (gi >= 0 && gi < NX && gj >= 0 && gj < NY) {
      const int64_t o = bs.gbase[f.b] + (int64_t)f.v * P + f.u;
      FCHK(o >= 0 && o < p.alloc_elems);
      cp_async_el(MA(f.b) + t, p.mea + o);
      cp_async_el(MS(f.b) + t, p.msb + o);
      cp_async_el(H(f.b) + t, p.hz0 + o);
    } else {
      MA(f.b)[t] = T(-1);
      MS(f.b)[t] = T(0);
      H(f.b)[t] = T(0);
    }
  }
  for (Flat f(tid, nt, 0, Wr, 0, Hr + 1); f.b < nreg; f.next()) {  // Ex edge rows
    const int64_t gi = bs.gi0[f.b] + f.u, gj = bs.gj0[f.b] + f.v;
    if (gi >= 0 && gi < NX && gj >= 0 && gj <= NY) cp_async_el(EX(f.b) + f.v * Wr + f.u, p.ex0 + bs.gbase[f.b] + (int64_t)f.v * P + f.u);
    else EX(f.b)[f.v * Wr + f.u] = T(0);
  }
  for (Flat f(tid, nt, 0, W1, 0, Hr); f.b < nreg; f.next()) {  // Ey edge columns
    const int64_t gi = bs.gi0[f.b] + f.u, gj = bs.gj0[f.b] + f.v;
    if (gi >= 0 && gi <= NX && gj >= 0 && gj < NY) cp_async_el(EY(f.b) + f.v * W1 + f.u, p.ey0 + bs.gbase[f.b] + (int64_t)f.v * P + f.u);
    else EY(f.b)[f.v * W1 + f.u] = T(0);
  }
#endif
  PHASE();
  if (!BIG) load_rom_state(p, m, mem, nb, B, sv);  // (BIG: the ROM step reads x~ from global memory)
  PHASE();
  for (int it = tid; FDTD_SKPF && it < nr * ((nY * nY + 31) / 32); it += nt) {  // the batch's Schur inverses into L2
    const int b = it % nr, l = it / nr;
    prefetch_l2(p.Sk + p.Sk_off[mem[b]] + l * 32);
  }
  for (int it = tid; it < nY * nr; it += nt) {  // per-pass constants of the batch's ports (RomConst)
    const int i = it % nY, b = it / nY;
    const int64_t po = p.port_off[mem[b]] + i;
    rc.eh[i * B + b] = p.ehalf[po];
    rc.cya[i * B + b] = p.cya[po];
    rc.cyg[i * B + b] = p.cyg[po];
  }
  PHASE();
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  PHASE();
  // WHOLE with p.whole_coef: every edge's (ca, cb) and energy weight, built once for all the steps
  // (edge_coef, the functions the per-step code calls; cb == 0 exactly on a dead edge)
  T *CAX = nullptr, *CBX = nullptr, *WXC = nullptr, *CAY = nullptr, *CBY = nullptr, *WYC = nullptr;
  if (WHOLE && p.whole_coef) {
    const int nex = (Hr + 1) * Wr, ney = Hr * W1;
    CAX = reg + (int64_t)rstride;
    CBX = CAX + nex;
    WXC = CBX + nex;
    CAY = WXC + nex;
    CBY = CAY + ney;
    WYC = CBY + ney;
    const T* ma = MA(0);
    const T* ms = MS(0);
    for (int k = tid; k < nex; k += nt) {  // Ex edge rows 1 .. Hr-1 (rows 0 and Hr: dead borders)
      const int v = k / Wr;
      T ca = T(1), cb = T(0), a = T(0);
      bool l = false;
      if (v >= 1 && v < Hr) edge_coef(ma[k - Wr], ms[k - Wr], ma[k], ms[k], p.idy, ca, cb, a, l);
      CAX[k] = ca; CBX[k] = l ? cb : T(0); WXC[k] = l ? mul_rn(p.wxy, a) : T(0);
    }
    for (int k = tid; k < ney; k += nt) {  // Ey edge columns 1 .. Wr-1
      const int v = k / W1, u = k % W1;
      T ca = T(1), cb = T(0), a = T(0);
      bool l = false;
      if (u >= 1 && u < Wr) edge_coef(ma[v * Wr + u - 1], ms[v * Wr + u - 1], ma[v * Wr + u], ms[v * Wr + u], -p.idx, ca, cb, a, l);
      CAY[k] = ca; CBY[k] = l ? cb : T(0); WYC[k] = l ? mul_rn(p.wxy, a) : T(0);
    }
    __syncthreads();
  }
  // Values go wrong from the region's border inwards one cell per step, so step s only updates the
  // cone that is still exact: cells [s, Wr - s) x [s, Hr - s) (edges one further in across their
  // normal); the zone, the ROM's gather cells and the write-back all lie inside the last cone.
  // the step's region pieces (K3)
  auto gsrc = [&](int s) -> T {  // soft-source sample of step n+s
    if constexpr (WHOLE) {
      const int64_t k = step + s - p.src_meta[0];
      return (p.src_row >= 0 && k >= 0 && k < p.src_meta[1]) ? (T)p.src_samples[k] : T(0);
    } else {
      return g[s];
    }
  };
  // H half-step (+ source, + the zone cells' storage-function terms of W^{n+s}) on the cone of step s
  auto h_half = [&](int s) {
    const int sc = WHOLE ? 0 : s;  // (the whole grid has no cone)
    const int cw = Wr - 2 * sc, ch = Hr - 2 * sc;
    for (Flat f(tid, nt, sc, cw, sc, ch); f.b < nreg; f.next()) {
      const int u = f.u, v = f.v, r = f.b;
      const T* ex = EX(r);
      const T* ey = EY(r);
      const T* ma = MA(r);
      T* hz = H(r);
      const int t = v * Wr + u;
      const T h0 = hz[t];
      const T hu = hupd(h0, ex[t + Wr], ex[t], ey[v * W1 + u + 1], ey[v * W1 + u], p.chy, p.chx);
      T h = ma[t] < T(0) ? h0 : hu;  // dead cells keep their Hz (as in yee_row)
      if (u == bs.su[r] && v >= bs.sv0[r] && v < bs.sv1[r]) h += gsrc(s);
      if (ENERGY && u >= zu0 && u < zu1 && v >= zv0 && v < zv1) {
        // the zone cell's full storage-function term (row_coef's weights without the zone mask)
        T wx, wy;
        if (WHOLE && WXC) {
          wx = WXC[t];
          wy = WYC[v * W1 + u];
        } else {
          const T* ms = MS(r);
          bool lx, ly;
          T ax, ay, ca, cb;
          edge_coef(ma[t - Wr], ms[t - Wr], ma[t], ms[t], p.idy, ca, cb, ax, lx);
          edge_coef(ma[t - 1], ms[t - 1], ma[t], ms[t], -p.idx, ca, cb, ay, ly);
          wx = lx ? mul_rn(p.wxy, ax) : T(0);
          wy = ly ? mul_rn(p.wxy, ay) : T(0);
        }
        const T hw = ma[t] < T(0) ? T(0) : p.wh;
        ZE(r)[(v - zv0) * zw + u - zu0] = cell_energy(T(0), ex[t], ey[v * W1 + u], h0, h, wx, wy, hw);
      }
      hz[t] = h;
    }
  };
  // zone probes; S4 gather of y^{n+s} (interface edges) and h = Hz^{n+s+1/2} (outside cells); the
  // regions' zone energies (fixed order, one warp per region)
  auto gather = [&](int s, bool with_t) {
    if constexpr (WHOLE) {  // every probe of the grid
      for (int z = tid; z < p.n_wprobe; z += nt) {
        const int u = p.wprobe[3 * z] + M, v = p.wprobe[3 * z + 1] + M;
        p.probe_ring[(int64_t)p.wprobe[3 * z + 2] * p.cap + (step + s) % p.cap] = H(0)[v * Wr + u];
      }
    }
    for (int b = 0; !WHOLE && b < nr; ++b) {
      const int z0 = p.zp_off[mem[b]], z1 = p.zp_off[mem[b] + 1];
      if (z0 == z1) continue;
      const int r = bs.rr[b];
      for (int z = z0 + tid; z < z1; z += nt) {
        const int u = (int)(p.zp[3 * z] - bs.gi0[r]), v = (int)(p.zp[3 * z + 1] - bs.gj0[r]);
        FCHK(u >= 0 && u < Wr && v >= 0 && v < Hr && p.zp[3 * z + 2] < p.n_probe);
        p.probe_ring[(int64_t)p.zp[3 * z + 2] * p.cap + (step + s) % p.cap] = H(r)[v * Wr + u];
      }
    }
    for (int it = tid; it < nY * nr; it += nt) {
      const int i = it % nY, b = it / nY;
      const int r = bs.rr[b], U0 = bs.bu[b], V0 = bs.bv[b];
      const T* ex = EX(r);
      const T* ey = EY(r);
      const T* hz = H(r);
      T y, h;
      if (i < bx) {  // S side: Ex edge row V0, outside cell row V0-1
        y = ex[V0 * Wr + U0 + i]; h = hz[(V0 - 1) * Wr + U0 + i];
      } else if (i < 2 * bx) {  // N side: Ex edge row V0+by, outside cell row V0+by
        y = ex[(V0 + by) * Wr + U0 + i - bx]; h = hz[(V0 + by) * Wr + U0 + i - bx];
      } else if (i < 2 * bx + by) {  // W side: Ey edge column U0, outside cell column U0-1
        const int v = V0 + i - 2 * bx;
        y = ey[v * W1 + U0]; h = hz[v * Wr + U0 - 1];
      } else {  // E side: Ey edge column U0+bx, outside cell column U0+bx
        const int v = V0 + i - 2 * bx - by;
        y = ey[v * W1 + U0 + bx]; h = hz[v * Wr + U0 + bx];
      }
      sy[i * B + b] = y;
      sh[i * B + b] = h;
      if (with_t) {  // t = (a_y/c_y) y + (D_l G/c_y) h - L~^T E*, as rom_t forms it (M1 ran in the H phase)
        const int k = i * B + b;
        sv[5 * S + k] = sv[3 * S + (m.q2 + m.q1 + i) * B + b] + fma_rn(rc.cyg[k], h, mul_rn(rc.cya[k], y));
      }
    }
    if (ENERGY && WHOLE) {  // one region: every warp sums a fixed slice (per-warp partials in zsum)
      const int lane = tid & 31, w = tid >> 5, nw = nt >> 5;
      const int per = (nz + nw - 1) / nw;
      const int i0 = w * per, i1 = min(nz, i0 + per);
      const T* ze = ZE(0);
      double acc = 0.0;
      for (int i = i0 + lane; i < i1; i += 32) acc += (double)ze[i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(FULL, acc, o);
      if (lane == 0) bs.zsum[w] = acc;
    } else if (ENERGY) {
      const int lane = tid & 31, w = tid >> 5, nw = nt >> 5;
      for (int r = w; r < nreg; r += nw) {
        const T* ze = ZE(r);
        double acc = 0.0;
        for (int i = lane; i < nz; i += 32) acc += (double)ze[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(FULL, acc, o);
        if (lane == 0) bs.zsum[r] = acc;
      }
    }
  };
  // S6: y into member b's interface edge i
  auto scatter1 = [&](int i, int b, T y) {
    const int r = bs.rr[b], U0 = bs.bu[b], V0 = bs.bv[b];
    T* ex = EX(r);
    T* ey = EY(r);
    if (i < bx) ex[V0 * Wr + U0 + i] = y;
    else if (i < 2 * bx) ex[(V0 + by) * Wr + U0 + i - bx] = y;
    else if (i < 2 * bx + by) ey[(V0 + i - 2 * bx) * W1 + U0] = y;
    else ey[(V0 + i - 2 * bx - by) * W1 + U0 + bx] = y;
  };
  // E half-step on the regions' live edges (dead edges -- interface, PEC, hole -- keep their value:
  // they are skipped, so the scatter and the update never touch the same edge)
  auto e_half = [&](int s) {
    const int sc = WHOLE ? 0 : s;
    const int cw = Wr - 2 * sc, ch = Hr - 2 * sc;
    if (WHOLE && CBX) {  // precomputed coefficients (the same values; cb == 0 on dead edges)
      const T* hz = H(0);
      T* ex = EX(0);
      T* ey = EY(0);
      for (Flat f(tid, nt, 0, Wr, 1, Hr - 1); f.b < nreg; f.next()) {
        const int t = f.v * Wr + f.u;
        const T cb = CBX[t];
        if (cb != T(0)) ex[t] = eupd(ex[t], CAX[t], cb, hz[t] - hz[t - Wr]);
      }
      for (Flat f(tid, nt, 1, Wr - 1, 0, Hr); f.b < nreg; f.next()) {
        const int c = f.v * Wr + f.u, e = f.v * W1 + f.u;
        const T cb = CBY[e];
        if (cb != T(0)) ey[e] = eupd(ey[e], CAY[e], cb, hz[c] - hz[c - 1]);
      }
      return;
    }
    for (Flat f(tid, nt, sc, cw, sc + 1, ch - 1); f.b < nreg; f.next()) {  // Ex edge rows s+1 .. Hr-s-1,
      const int t = f.v * Wr + f.u;                                         // columns s .. Wr-s-1
      const T* ma = MA(f.b);
      const T* ms = MS(f.b);
      const T* hz = H(f.b);
      T* ex = EX(f.b);
      bool l;
      T a, ca, cb;
      edge_coef(ma[t - Wr], ms[t - Wr], ma[t], ms[t], p.idy, ca, cb, a, l);
      if (l) ex[t] = eupd(ex[t], ca, cb, hz[t] - hz[t - Wr]);
    }
    for (Flat f(tid, nt, sc + 1, cw - 1, sc, ch); f.b < nreg; f.next()) {  // Ey edge columns s+1 .. Wr-s-1,
      const int c = f.v * Wr + f.u;                                         // rows s .. Hr-s-1
      const T* ma = MA(f.b);
      const T* ms = MS(f.b);
      const T* hz = H(f.b);
      T* ey = EY(f.b);
      bool l;
      T a, ca, cb;
      edge_coef(ma[c - 1], ms[c - 1], ma[c], ms[c], -p.idx, ca, cb, a, l);
      if (l) ey[f.v * W1 + f.u] = eupd(ey[f.v * W1 + f.u], ca, cb, hz[c] - hz[c - 1]);
    }
  };
#pragma unroll 1
  for (int s = 0; s < (WHOLE ? nsteps : K); ++s) {
    double* ep = p.rom_partials + (int64_t)(WHOLE ? 0 : s) * p.n_inst;
    if constexpr ((FDTD_FUSE || WHOLE) && !BIG) {
      // five barrier phases per step instead of seven: the M1 GEMM needs x~ only, so it shares the
      // H half-step's phase; the live-edge E half-step needs neither y nor the ROM, so it shares the
      // gather's; the scatter rides in the M2 epilogue
      h_half(s);
      rom_m1<T, ENERGY>(p, m, B, S, sv);
      __syncthreads();
      PHASE();
      gather(s, FDTD_FUSE2 != 0 && WHOLE);
      e_half(s);
      __syncthreads();
      PHASE();
      if constexpr (FDTD_FUSE2 != 0 && WHOLE) {
        // four barrier phases per step: t was formed by the gather, so the storage-function terms
        // (one warp per instance, the zone energy added by the same lane) share the Schur phase.
        // Whole grid only: cfg1 7.5 instead of 8.15 us per step; on the batched fix-up the energy
        // warps lengthen the Schur phase more than the saved barrier gains (0.432 vs 0.419 ms)
        rom_energy<T, ENERGY>(m, mem, nb, B, S, sv, ep, [&](int b) {
          return (!WHOLE && (kind == 0 || b == 0)) ? bs.zsum[bs.rr[b]] : 0.0;
        });
        rom_schur<T>(p, m, mem, nb, B, S, sv);
        __syncthreads();
        PHASE();
        if (WHOLE && ENERGY && tid == 0) {  // W^{n+s}: the grid's cells (zsum) and every ROM, fixed order
          double tot = 0.0;
          for (int w = 0; w < (nt >> 5); ++w) tot += bs.zsum[w];
          for (int b = 0; b < nb; ++b) tot += ep[mem[b]];
          p.energy_ring[(step + s) % p.cap] = tot;
          if (!isfinite(tot)) *p.flag = 1;
        }
        rom_m2<T>(p, m, nb, B, S, sv, scatter1);
        __syncthreads();
        PHASE();
        continue;
      }
      rom_t<T, ENERGY>(m, mem, nb, B, S, sv, ep);
      __syncthreads();
      PHASE();
      // (after the barrier: rom_t's warps have written ep)
      if (ENERGY && !WHOLE && tid < nr && (kind == 0 || tid == 0)) ep[mem[tid]] += bs.zsum[bs.rr[tid]];
      if (WHOLE && ENERGY && tid == 0) {  // W^{n+s}: the grid's cells (zsum) and every ROM, fixed order
        double tot = 0.0;
        for (int w = 0; w < (nt >> 5); ++w) tot += bs.zsum[w];
        for (int b = 0; b < nb; ++b) tot += ep[mem[b]];
        p.energy_ring[(step + s) % p.cap] = tot;
        if (!isfinite(tot)) *p.flag = 1;
      }
      rom_schur<T>(p, m, mem, nb, B, S, sv);
      __syncthreads();
      PHASE();
      rom_m2<T>(p, m, nb, B, S, sv, scatter1);
      __syncthreads();
      PHASE();
      continue;
    }
    h_half(s);
    __syncthreads();
    PHASE();
    gather(s, false);
    __syncthreads();
    PHASE();
    // ---- S5: ROM step n+s -> y^{n+s+1}, x~^{n+s+1}; ROM energy of W^{n+s} (+ the zone energy of
    // the member's region on its first member)
    if constexpr (BIG) rom_step_big<T, ENERGY>(p, m, mem, s, sv, S, ep, part);
    else rom_step<T, ENERGY>(p, m, mem, nb, B, S, sv, ep);
    if (ENERGY && tid < nr && (kind == 0 || tid == 0)) ep[mem[tid]] += bs.zsum[bs.rr[tid]];
    // ---- S6: y^{n+s+1} into the regions' interface edges, and in the same phase the E half-step
    for (int it = tid; it < nY * nr; it += nt) {
      const int i = it % nY, b = it / nY;
      scatter1(i, b, sy[i * B + b]);
    }
    e_half(s);
    __syncthreads();
    PHASE();
  }
  // ---- write back the zones: Hz of the live zone cells, their bottom Ex and left Ey edges
  if constexpr (WHOLE) {  // every cell of the grid with its bottom Ex and left Ey edge (dead ones
                          // included; the top and east wall edges never change), a finiteness check
    bool bad = false;
    for (Flat f(tid, nt, M, rbx, M, rby); f.b < nreg; f.next()) {
      const int t = f.v * Wr + f.u;
      const int64_t o = bs.gbase[f.b] + (int64_t)f.v * P + f.u;
      FCHK(o >= (int64_t)p.row0 * p.pitch && o < (int64_t)(p.row0 + p.rows) * p.pitch);  // owned rows only
      const T h = H(f.b)[t];
      bad |= !isfinite((double)h);
      p.hz1[o] = h;
      p.ex1[o] = EX(f.b)[t];
      p.ey1[o] = EY(f.b)[f.v * W1 + f.u];
    }
    if (__syncthreads_or(bad) && tid == 0) *p.flag = 1;
  } else if (nz > 0)
    for (Flat f(tid, nt, zu0, zw, zv0, zv1 - zv0); f.b < nreg; f.next()) {
      const int t = f.v * Wr + f.u;
      if (!(MA(f.b)[t] >= T(0))) continue;
      const int64_t o = bs.gbase[f.b] + (int64_t)f.v * P + f.u;
      FCHK(o >= (int64_t)p.row0 * p.pitch && o < (int64_t)(p.row0 + p.rows) * p.pitch);  // owned rows only
      p.hz1[o] = H(f.b)[t];
      p.ex1[o] = EX(f.b)[t];
      p.ey1[o] = EY(f.b)[f.v * W1 + f.u];
    }
  if constexpr (BIG) {  // the final x~ from the scratch into the slot store_rom reads
    if (!rg) return;
    const BigScratch<T> bsc(p.big, m);
    const T* xf = ((K - 1) & 1) ? bsc.X1 : bsc.X0;
    for (int i = tid; i < m.q1 + m.q2; i += nt) sv[i] = xf[i];
    __syncthreads();
    PHASE();
  }
  store_rom(p, m, mem, nb, B, S, sv, p.ex1, p.ey1);
}

#ifndef FDTD_PERSIST  // fix-up: one CTA per SM walking the batches (b, b + grid, ...), the next batch's
#define FDTD_PERSIST 0    // regions pulled into L2 while the current one runs
#endif
// the rows of batch b's regions (materials and the pass's input fields) into L2 (prefetch hints;
// rows outside this slab's allocated rows are skipped)
template <typename T, int K>
__device__ void prefetch_regions(const PostParams<T>& p, int b) {
  const int* bt = p.batch_tab + BATCH_FIELDS * b;
  const int nb = bt[2], kind = bt[5];
  const int32_t* mem = p.batch_inst + bt[1];
  const int M = p.Kz + K - 1, nreg = kind ? 1 : nb;
  const int32_t* q0 = p.rects + 4 * (int64_t)mem[0];
  const int bw = kind ? p.batch_rect[4 * b + 2] : q0[2], bh = kind ? p.batch_rect[4 * b + 3] : q0[3];
  const int Wr = bw + 2 * M + 1, Hr = bh + 2 * M + 1, lines = (Wr + 31) / 32 + 1;  // 128-byte lines per row
  const int per = Hr * lines * 5;
  for (int it = threadIdx.x; it < nreg * per; it += blockDim.x) {
    const int r = it / per, rem = it % per, a = rem / (Hr * lines), v = (rem / lines) % Hr, l = rem % lines;
    const int32_t* q = kind ? p.batch_rect + 4 * b : p.rects + 4 * (int64_t)mem[r];
    const int64_t i0 = (int64_t)q[0] - M, lr = (int64_t)q[1] - M + v - p.row_begin + p.row0;
    if (lr < 0 || lr >= p.row0 + p.rows + K) continue;
    const int64_t c = max(i0, (int64_t)0) + 32 * l;
    if (c >= p.pitch) continue;
    const T* base = a == 0 ? p.mea : a == 1 ? p.msb : a == 2 ? p.hz0 : a == 3 ? p.ex0 : p.ey0;
    prefetch_l2(base + lr * p.pitch + c);
  }
}

template <typename T, int K, bool ENERGY>
__global__ void __launch_bounds__(512, 1) postk_kernel(const PostParams<T> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double red[32];
  __shared__ BatchShared bs;
  T* sv = reinterpret_cast<T*>(smem_raw);
#if FDTD_PHASES
  if (threadIdx.x == 0) ph_counter() = 0;
  PHASE();
#endif
  const int64_t step = *p.step;
  T g[K];
#pragma unroll
  for (int s = 0; s < K; ++s) {
    g[s] = T(0);
    if (p.src_row >= 0) {
      const int64_t k = step + s - p.src_meta[0];
      if (k >= 0 && k < p.src_meta[1]) g[s] = (T)p.src_samples[k];
    }
  }
  for (int b = blockIdx.x; b < (FDTD_PERSIST ? p.n_batch_reg : blockIdx.x + 1); b += gridDim.x) {
    if (b >= p.n_batch_reg) break;
    if (FDTD_PERSIST && b != (int)blockIdx.x) __syncthreads();  // the previous batch's readers are done
    if (FDTD_PERSIST && b + (int)gridDim.x < p.n_batch_reg) prefetch_regions<T, K>(p, b + gridDim.x);
    fixup_batch<T, K, ENERGY>(p, b, sv, g, step, bs);
    PHASE();
    if (ENERGY) {  // this batch's ROM + zone energies, one value per step (level 1)
      __syncthreads();  // rom_partials of this batch written (fixup_batch ends with barriers)
      const int32_t* mem = p.batch_inst + p.batch_tab[BATCH_FIELDS * b + 1];
      const int nb = p.batch_tab[BATCH_FIELDS * b + 2];
#pragma unroll 1
      for (int s = 0; s < K; ++s) {
        double v = 0.0;
        for (int k = threadIdx.x; k < nb; k += blockDim.x) v += p.rom_partials[(int64_t)s * p.n_inst + mem[k]];
        const double tot = block_sum(v, red);
        if (threadIdx.x == 0) p.level1[(int64_t)s * p.n_batch + b] = tot;
      }
    }
  }
}

// K3c: the whole grid and all its ROM instances in one CTA's shared memory for nsteps steps (small
// grids: config 1, the degenerate cases); one launch per fdtd_step call.  Advances the device step
// counter (no finalize kernel: the energy ring is written per step).
template <typename T, bool ENERGY>
__global__ void __launch_bounds__(512, 1) wholegrid_kernel(const PostParams<T> p, int64_t nsteps) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ BatchShared bs;
  T* sv = reinterpret_cast<T*>(smem_raw);
#if FDTD_PHASES
  if (threadIdx.x == 0) ph_counter() = 0;
#endif
  const int64_t step = *p.step;
  const T g[1] = {T(0)};
  fixup_batch<T, 1, ENERGY, false, true>(p, 0, sv, g, step, bs, nullptr, nsteps);
  __syncthreads();
  if (threadIdx.x == 0) *const_cast<int64_t*>(p.step) = step + nsteps;  // (the context's counter)
}

// The large-model fix-up (one instance at a time on a cooperative grid of one CTA per SM): the
// batches [n_batch_reg, n_batch), each a single instance of a model of order >= the big threshold.
template <typename T, int K, bool ENERGY>
__global__ void __launch_bounds__(512, 1) bigrom_kernel(const PostParams<T> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double red[32];
  __shared__ BatchShared bs;
  __shared__ double part[16 * 8 * BIG_TILES];  // phase-1 partials: [warp][tile][row]
  T* sv = reinterpret_cast<T*>(smem_raw);
#if FDTD_PHASES
  if (threadIdx.x == 0) ph_counter() = 0;
#endif
  const int64_t step = *p.step;
  T g[K];
#pragma unroll
  for (int s = 0; s < K; ++s) {
    g[s] = T(0);
    if (p.src_row >= 0) {
      const int64_t k = step + s - p.src_meta[0];
      if (k >= 0 && k < p.src_meta[1]) g[s] = (T)p.src_samples[k];
    }
  }
  for (int b = p.n_batch_reg; b < p.n_batch; ++b) {
    fixup_batch<T, K, ENERGY, true>(p, b, sv, g, step, bs, part);
    if (ENERGY && blockIdx.x == 0) {
      __syncthreads();
      const int first = p.batch_inst[p.batch_tab[BATCH_FIELDS * b + 1]];
#pragma unroll 1
      for (int s = 0; s < K; ++s) {
        const double tot = block_sum(threadIdx.x == 0 ? p.rom_partials[(int64_t)s * p.n_inst + first] : 0.0, red);
        if (threadIdx.x == 0) p.level1[(int64_t)s * p.n_batch + b] = tot;
      }
    }
    cooperative_groups::this_grid().sync();  // the scratch is reused by the next instance
  }
}

// End of a pass: W^{n+s} = fixed-order two-level sum of the sweep / band partials and the fix-up
// batches' values (deterministic), and the device step counter.
__global__ void __launch_bounds__(256) finalize_kernel(const FinParams p) {
  __shared__ double red[32];
  __shared__ bool last;
  const int b = blockIdx.x;
  const int64_t step = *p.step;
  if (p.energy) {
    const int64_t per = (p.n_sweep_partials + gridDim.x - 1) / gridDim.x;
    const int64_t k0 = b * per, k1 = min(p.n_sweep_partials, k0 + per);
    const int perr = (p.n_rom + gridDim.x - 1) / gridDim.x;
    const int r0 = b * perr, r1 = min(p.n_rom, r0 + perr);
#pragma unroll 1
    for (int s = 0; s < p.K; ++s) {
      double v = 0.0;
      for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) v += __ldcg(p.sweep_partials + s * p.pstride + k);
      for (int k = r0 + threadIdx.x; k < r1; k += blockDim.x) v += __ldcg(p.rom_level1 + (int64_t)s * p.n_rom + k);
      const double tot = block_sum(v, red);
      if (threadIdx.x == 0) p.level2[(int64_t)s * gridDim.x + b] = tot;
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
  bool bad = false;
  if (p.energy) {
#pragma unroll 1
    for (int s = 0; s < p.K; ++s) {
      double v = 0.0;
      for (int k = threadIdx.x; k < (int)gridDim.x; k += blockDim.x) v += __ldcg(p.level2 + (int64_t)s * gridDim.x + k);
      const double tot = block_sum(v, red);
      if (threadIdx.x == 0) {
        p.energy_ring[(step + s) % p.cap] = tot;
        bad |= !isfinite(tot);  // the storage function sums the square of every field value
      }
    }
  }
  // non-finite sentinel: NSAMPLE Hz cells of the pass's output on a fixed stride pattern (a blow-up
  // is a growing global mode; with the energy recorded every cell is covered above)
  for (int k = threadIdx.x; k < NSAMPLE && p.rows > 0; k += blockDim.x) {
    const int64_t r = p.row0 + (int64_t)(((uint64_t)k * 2654435761u + (uint64_t)step) % (uint64_t)p.rows);
    const int64_t col = (int64_t)(((uint64_t)k * 40503u + (uint64_t)step * 7u) % (uint64_t)p.nx);
    const int64_t o = r * p.pitch + col;
    const double v = p.es == 8 ? __ldcg((const double*)p.hz + o) : (double)__ldcg((const float*)p.hz + o);
    bad |= !isfinite(v);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) *p.flag = 1;
  if (threadIdx.x == 0) {
    *p.done = 0u;
    *p.step = step + p.K;
  }
}

// NEXT-2: CPML band fix-up.  Per CTA: one row chunk [r0, r1) of one side; region = columns
// [c0, c0 + WB), WB = w + Kz + K + 2, rows [r0 - K, r1 + K - 1) (+ one Ex edge row).  K steps with the
// sweep's device functions plus, in the layer, psi_hz = b psi_hz + a dEy/dx (Hz -= dt/mu0 psi_hz)
// and psi_ey = b psi_ey + a dHz/dx (the Ey curl term gains dx psi_ey).  Values go wrong from the
// region's border inwards one cell per step, so after K steps the write-back columns (the layer
// and Kz + 1 interior columns) of the chunk's rows are exact; the sweep's plain-Yee values there are
// overwritten.  Also: the storage-function terms of the write-back cells (their msb marks made the
// sweep skip them), the probes in them, and the layer's psi state.
template <typename T, int K, bool ENERGY>
__global__ void __launch_bounds__(256) pml_kernel(const PmlParams<T> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double red[32];
  const int side = blockIdx.y;
  // region: the write-back columns plus K + 1 (Kz > K on the shorter passes ending a step count)
  const int w = p.w, WW = w + p.Kz + 1, WB = WW + K + 1;
  const int64_t nx = p.nx, P = p.pitch;
  const int r0 = p.row0 + blockIdx.x * p.chunk, r1 = min(r0 + p.chunk, p.row0 + p.rows);
  const int R0 = r0 - K, Hr = (r1 - r0) + 2 * K - 1;  // region cell rows [R0, R0 + Hr)
  const int64_t c0 = side == 0 ? 0 : nx - WB;          // first region column
  const int64_t lay0 = side == 0 ? 0 : nx - w;         // first layer column
  const int64_t wb0 = side == 0 ? 0 : nx - WW, wb1 = side == 0 ? WW : nx;  // write-back columns
  const int tid = threadIdx.x, nt = blockDim.x;
  const int n = Hr * WB;
  T* H = reinterpret_cast<T*>(smem_raw);
  T* MA = H + n;
  T* MS = MA + n;
  T* PH = MS + n;              // psi_hz per region cell (0 outside the layer)
  T* EX = PH + n;              // (Hr + 1) x WB
  T* EY = EX + n + WB;         // Hr x (WB + 1)
  T* PE = EY + Hr * (WB + 1);  // psi_ey per region Ey edge
  const int W1 = WB + 1;
  const int64_t step = *p.step;
  auto off = [&](int u, int v) { return (int64_t)(R0 + v) * P + c0 + u; };
  FCHK(R0 >= 0 && off(WB, Hr + 1) < p.alloc_elems && c0 >= 0);
  auto hcol = [&](int64_t gi) { return side == 0 ? (int)gi : (int)(gi - lay0); };  // Hz layer index
  auto in_layer_h = [&](int64_t gi) { return side == 0 ? gi < w : gi >= lay0; };
  auto in_layer_e = [&](int64_t gi) { return side == 0 ? (gi >= 1 && gi <= w) : (gi >= lay0 && gi < nx); };
  auto ecol = [&](int64_t gi) { return side == 0 ? (int)gi : (int)(gi - lay0); };
  const T* bh = p.bh + side * w; const T* ah = p.ah + side * w;
  const T* be = p.be + side * (w + 1); const T* ae = p.ae + side * (w + 1);
  const T* psih = p.psih + (int64_t)side * p.psi_rows * w;
  const T* psie = p.psie + (int64_t)side * p.psi_rows * (w + 1);
  T* psih1 = p.psih1 + (int64_t)side * p.psi_rows * w;
  T* psie1 = p.psie1 + (int64_t)side * p.psi_rows * (w + 1);
  // ---- load the region (fields at step n, materials, psi)
  for (int t = tid; t < n; t += nt) {
    const int u = t % WB, v = t / WB;
    const int64_t o = off(u, v), gi = c0 + u;
    H[t] = p.hz0[o]; MA[t] = p.mea[o]; MS[t] = p.msb[o];
    PH[t] = in_layer_h(gi) ? psih[(int64_t)(R0 + v) * w + hcol(gi)] : T(0);
  }
  for (int t = tid; t < n + WB; t += nt) EX[t] = p.ex0[off(t % WB, t / WB)];
  for (int t = tid; t < Hr * W1; t += nt) {
    const int u = t % W1, v = t / W1;
    const int64_t gi = c0 + u;
    EY[t] = p.ey0[off(u, v)];
    PE[t] = in_layer_e(gi) ? psie[(int64_t)(R0 + v) * (w + 1) + ecol(gi)] : T(0);
  }
  __syncthreads();
  double eacc[K];
#pragma unroll
  for (int s = 0; s < K; ++s) eacc[s] = 0.0;
#pragma unroll 1
  for (int s = 0; s < K; ++s) {
    T gsrc = T(0);
    if (p.src_row >= 0) {
      const int64_t k = step + s - p.src_meta[0];
      if (k >= 0 && k < p.src_meta[1]) gsrc = (T)p.src_samples[k];
    }
    // ---- H half-step (+ CPML psi_hz, + source, + storage terms of the write-back cells)
    T ea = T(0);
    for (int t = tid; t < n; t += nt) {
      const int u = t % WB, v = t / WB;
      const int64_t gi = c0 + u;
      const T h0 = H[t];
      T h = hupd(h0, EX[t + WB], EX[t], EY[v * W1 + u + 1], EY[v * W1 + u], p.chy, p.chx);
      if (MA[t] < T(0)) {
        h = h0;  // dead cells keep their Hz
      } else if (in_layer_h(gi)) {
        const int hc = hcol(gi);
        const T ps = fma_rn(bh[hc], PH[t], mul_rn(ah[hc], mul_rn(p.idx, EY[v * W1 + u + 1] - EY[v * W1 + u])));
        PH[t] = ps;
        h = fma_rn(-p.cpsi, ps, h);
      }
      const int lr = R0 + v;
      if (p.src_row >= 0 && gi == p.src_col && lr >= p.src_row && lr < p.src_row_end) h += gsrc;
      if (ENERGY && gi >= wb0 && gi < wb1 && lr >= r0 && lr < r1) {  // v >= K >= 1 here
        bool lx, ly = false;
        T ax, ay = T(0), ca, cb;
        edge_coef(MA[t - WB], MS[t - WB], MA[t], MS[t], p.idy, ca, cb, ax, lx);
        if (u >= 1) edge_coef(MA[t - 1], MS[t - 1], MA[t], MS[t], -p.idx, ca, cb, ay, ly);  // u = 0: the x = 0 wall
        const T wx = lx ? mul_rn(p.wxy, ax) : T(0), wy = ly ? mul_rn(p.wxy, ay) : T(0);
        const T hw = MA[t] < T(0) ? T(0) : p.wh;
        ea = cell_energy(ea, EX[t], EY[v * W1 + u], h0, h, wx, wy, hw);
      }
      H[t] = h;
    }
    if (ENERGY) eacc[s] += (double)ea;
    __syncthreads();
    for (int k = tid; k < p.n_probe; k += nt) {  // probes in the write-back cells of the chunk
      const int64_t gi = p.probe_gi[k];
      const int lr = p.probe_lr[k];
      if (gi >= wb0 && gi < wb1 && lr >= r0 && lr < r1)
        p.probe_ring[(int64_t)k * p.cap + (step + s) % p.cap] = H[(lr - R0) * WB + (gi - c0)];
    }
    // ---- E half-step on the region's interior edges (+ CPML psi_ey on the layer's Ey edges)
    for (int t = WB + tid; t < n; t += nt) {  // Ex edge rows 1 .. Hr-1
      bool l;
      T a, ca, cb;
      edge_coef(MA[t - WB], MS[t - WB], MA[t], MS[t], p.idy, ca, cb, a, l);
      EX[t] = eupd(EX[t], ca, cb, H[t] - H[t - WB]);
    }
    for (int t = tid; t < Hr * (WB - 1); t += nt) {  // Ey edge columns 1 .. WB-1
      const int u = t % (WB - 1) + 1, v = t / (WB - 1);
      const int c = v * WB + u;
      const int64_t gi = c0 + u;
      bool l;
      T a, ca, cb;
      edge_coef(MA[c - 1], MS[c - 1], MA[c], MS[c], -p.idx, ca, cb, a, l);
      T dh = H[c] - H[c - 1];
      if (l && in_layer_e(gi)) {
        const int ec = ecol(gi);
        const T ps = fma_rn(be[ec], PE[v * W1 + u], mul_rn(ae[ec], mul_rn(p.idx, dh)));
        PE[v * W1 + u] = ps;
        dh = fma_rn(p.dxv, ps, dh);
      }
      EY[v * W1 + u] = eupd(EY[v * W1 + u], ca, cb, dh);
    }
    __syncthreads();
  }
  // ---- write back the chunk's write-back cells (Hz, bottom Ex, left Ey) and the layer's psi
  for (int t = tid; t < n; t += nt) {
    const int u = t % WB, v = t / WB;
    const int64_t gi = c0 + u;
    const int lr = R0 + v;
    if (gi < wb0 || gi >= wb1 || lr < r0 || lr >= r1) continue;
    const int64_t o = off(u, v);
    FCHK(lr >= p.row0 && lr < p.row0 + p.rows);
    p.hz1[o] = H[t];
    p.ex1[o] = EX[t];
    p.ey1[o] = EY[v * W1 + u];
    if (in_layer_h(gi)) psih1[(int64_t)lr * w + hcol(gi)] = PH[t];
    if (in_layer_e(gi)) psie1[(int64_t)lr * (w + 1) + ecol(gi)] = PE[v * W1 + u];
  }
  if (ENERGY) {
#pragma unroll 1
    for (int s = 0; s < K; ++s) {
      const double tot = block_sum(eacc[s], red);
      if (tid == 0) p.partials[s * p.pstride + p.poff + (int64_t)blockIdx.y * gridDim.x + blockIdx.x] = tot;
    }
  }
}

template <typename T>
__global__ void band_marks_kernel(T* msb, const T* mea, int64_t pitch, int64_t nx, int row0, int ncol, bool set) {
  const int r = row0 + blockIdx.x;
  for (int t = threadIdx.x; t < 2 * ncol; t += blockDim.x) {
    const int64_t gi = t < ncol ? t : nx - 2 * ncol + t;
    if (gi < 0 || gi >= nx) continue;
    const int64_t o = (int64_t)r * pitch + gi;
    if (mea[o] >= T(0)) msb[o] = set ? -fabs(msb[o]) : fabs(msb[o]);
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

// Seeded random state on the live cells and edges of the owned rows (fdtd_set_random_fields): each
// value a hash of (seed, array, global row, column) -- independent of the row-slab decomposition;
// dead cells and edges (PEC, holes, interface edges) keep their values.
__device__ __forceinline__ double hash_unit(uint64_t seed, uint64_t a, uint64_t j, uint64_t i) {
  uint64_t z = seed ^ (a << 60) ^ (j << 30) ^ i;
  z += 0x9e3779b97f4a7c15ull;  // splitmix64
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  z ^= z >> 31;
  return (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;  // [-1, 1)
}
template <typename T>
__global__ void random_fields_kernel(T* ex, T* ey, T* hz, const T* mea, int64_t pitch, int64_t nx, int row0,
                                     int64_t row_begin, uint64_t seed, double ae, double ah) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nx) return;
  const int64_t jl = row0 + blockIdx.y, gj = row_begin + blockIdx.y;
  const int64_t o = jl * pitch + i;
  if (!(mea[o] >= T(0))) return;
  hz[o] = (T)(ah * hash_unit(seed, 2, gj, i));
  if (mea[o - pitch] >= T(0)) ex[o] = (T)(ae * hash_unit(seed, 0, gj, i));
  if (mea[o - 1] >= T(0)) ey[o] = (T)(ae * hash_unit(seed, 1, gj, i));  // (column -1: padding, dead)
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

// Zone marks (K3): the sign bit of msb on every live cell of an instance's zone
// [i0-(Kz-1), i0+bx+Kz) x [j0-(Kz-1), j0+by+Kz) (Kz >= 2; empty for Kz = 1).
template <typename T>
__global__ void zone_kernel(T* msb, const T* mea, int64_t pitch, const int32_t* rects, int64_t row_begin, int row0,
                            int Kz, bool set) {
  if (Kz < 2) return;
  const int32_t* r = rects + 4 * (int64_t)blockIdx.x;
  const int u0 = r[0] - (Kz - 1), v0 = r[1] - (Kz - 1);
  const int w = r[2] + 2 * Kz - 1, h = r[3] + 2 * Kz - 1;
  for (int t = threadIdx.x; t < w * h; t += blockDim.x) {
    const int64_t o = ((int64_t)v0 + t / w - row_begin + row0) * pitch + u0 + t % w;
    if (mea[o] >= T(0)) msb[o] = set ? -fabs(msb[o]) : fabs(msb[o]);
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

#ifndef FDTD_SWEEP_U4_CHUNK  // rows per chunk from which the fp32 K = 4 sweep runs the four-row body
#define FDTD_SWEEP_U4_CHUNK 256
#endif
template <typename T, int K, int UR>
void sweepk_launch_u(const SweepParams<T>& q, dim3 grid, int threads, cudaStream_t s) {
  constexpr int V = (sizeof(T) == 4 && K < 4) ? 4 : 2;  // sweep_width
  const size_t smem = (K > 1 && !FDTD_REG_RING) ? (size_t)(threads / 32) * K * NCOEF * 32 * V * sizeof(T) : 0;
  if (q.partials) {
    if (smem > 32 * 1024)  // (static shared memory counts against the 48 KB default too)
      cudaFuncSetAttribute(sweepk_kernel<T, K, V, true, UR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    sweepk_kernel<T, K, V, true, UR><<<grid, threads, smem, s>>>(q);
  } else {
    if (smem > 32 * 1024)  // (static shared memory counts against the 48 KB default too)
      cudaFuncSetAttribute(sweepk_kernel<T, K, V, false, UR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    sweepk_kernel<T, K, V, false, UR><<<grid, threads, smem, s>>>(q);
  }
}
template <typename T, int K>
void sweepk_launch(const SweepParams<T>& q, dim3 grid, int threads, cudaStream_t s) {
  if constexpr (K == 4 && sizeof(T) == 4)
    if (q.chunk >= FDTD_SWEEP_U4_CHUNK) return sweepk_launch_u<T, K, 4>(q, grid, threads, s);
  sweepk_launch_u<T, K, 2>(q, grid, threads, s);
}

template <typename T>
void launch_sweep(const SweepParams<T>& p, int K, int warps_per_cta, cudaStream_t s, int chunk_begin,
                  int chunk_count) {
  const int nch = (p.rows + p.chunk - 1) / p.chunk;
  if (chunk_count < 0) chunk_count = nch - chunk_begin;
  if (chunk_count <= 0) return;
  SweepParams<T> q = p;
  q.chunk0 = chunk_begin;
  dim3 grid(sweep_ctas_x(p.nx, (int)sizeof(T), K, warps_per_cta), chunk_count);
  const int nt = 32 * warps_per_cta;
  if (K == 1) sweepk_launch<T, 1>(q, grid, nt, s);
  else if (K == 2) sweepk_launch<T, 2>(q, grid, nt, s);
  else if constexpr (sizeof(T) == 4) sweepk_launch<T, 4>(q, grid, nt, s);
}

size_t post_smem_bytes(size_t es, int nvec, int nY, int batch, int region_stride) {
  // ROM vectors, the per-pass port constants (fp64 eh + two T arrays), the zone partials, the regions
  return es * ((size_t)NROMVEC * vec_stride(nvec, batch) + (size_t)(8 / es + 2) * nY * batch +
               (size_t)batch * ZWARPS * (8 / es) + (size_t)batch * region_stride);
}

template <typename T, int K>
void postk_launch(const PostParams<T>& p, bool energy, cudaStream_t s) {
  const size_t smem = p.smem_bytes;
  int grid = p.n_batch_reg;
  if (FDTD_PERSIST) {  // one CTA per SM (the fix-up CTA fills an SM's registers)
    int nsm = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    grid = std::min(grid, nsm);
  }
  if (grid <= 0) return;
  if (energy) {
    if (smem > 32 * 1024)  // (static shared memory counts against the 48 KB default too)
      cudaFuncSetAttribute(postk_kernel<T, K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    postk_kernel<T, K, true><<<grid, p.block, smem, s>>>(p);
  } else {
    if (smem > 32 * 1024)  // (static shared memory counts against the 48 KB default too)
      cudaFuncSetAttribute(postk_kernel<T, K, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    postk_kernel<T, K, false><<<grid, p.block, smem, s>>>(p);
  }
}

#if FDTD_PHASES
void debug_phases(long long* out, int n) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_phase, sizeof(long long) * (size_t)std::min(n, 4096 * 72));
}
#endif

void launch_finalize(const FinParams& p, cudaStream_t s) { finalize_kernel<<<p.energy ? FIN_GRID : 1, 256, 0, s>>>(p); }

template <typename T, int K, bool ENERGY>
void bigrom_launch(const PostParams<T>& p, cudaStream_t s) {
  auto kern = bigrom_kernel<T, K, ENERGY>;
  const size_t smem = p.big_smem_bytes;
  if (smem > 32 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.big_grid);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, p);
}

template <typename T>
void launch_wholegrid(const PostParams<T>& p, int64_t nsteps, bool energy, cudaStream_t s) {
  if (nsteps <= 0) return;
  const size_t smem = p.smem_bytes;
  auto kern = energy ? wholegrid_kernel<T, true> : wholegrid_kernel<T, false>;
  if (smem > 32 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<1, p.block, smem, s>>>(p, nsteps);
}

template <typename T>
void launch_post_big(const PostParams<T>& p, int K, bool energy, cudaStream_t s) {
  if (p.n_batch <= p.n_batch_reg) return;
  if (K == 1) energy ? bigrom_launch<T, 1, true>(p, s) : bigrom_launch<T, 1, false>(p, s);
  else if (K == 2) energy ? bigrom_launch<T, 2, true>(p, s) : bigrom_launch<T, 2, false>(p, s);
  else if constexpr (sizeof(T) == 4) energy ? bigrom_launch<T, 4, true>(p, s) : bigrom_launch<T, 4, false>(p, s);
}

// co-resident CTAs of the large-model kernel (one per SM), 0 if it cannot be launched cooperatively
template <typename T>
int big_grid_size(size_t smem, int K) {
  int dev = 0, nsm = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  auto kern = K == 1 ? bigrom_kernel<T, 1, true> : bigrom_kernel<T, 2, true>;
  if constexpr (sizeof(T) == 4) if (K == 4) kern = bigrom_kernel<T, 4, true>;
  if (smem > 32 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 512, smem) != cudaSuccess || per < 1) return 0;
  return nsm;
}

template <typename T>
void launch_post(const PostParams<T>& p, int K, bool energy, cudaStream_t s) {
  if (p.n_batch <= 0) return;  // no ROM instances: nothing to fix up
  if (K == 1) postk_launch<T, 1>(p, energy, s);
  else if (K == 2) postk_launch<T, 2>(p, energy, s);
  else if constexpr (sizeof(T) == 4) postk_launch<T, 4>(p, energy, s);
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

template <typename T>
void launch_random_fields(T* ex, T* ey, T* hz, const T* mea, int64_t pitch, int64_t nx, int rows, int row0,
                          int64_t row_begin, uint64_t seed, double ae, double ah, cudaStream_t s) {
  if (rows <= 0 || nx <= 0) return;
  random_fields_kernel<T><<<dim3((unsigned)((nx + 255) / 256), rows), 256, 0, s>>>(ex, ey, hz, mea, pitch, nx, row0,
                                                                                  row_begin, seed, ae, ah);
}

template <typename T>
void launch_zone(T* msb, const T* mea, int64_t pitch, const int32_t* rects, int64_t n_rect, int64_t row_begin,
                 int row0, int Kz, bool set, cudaStream_t s) {
  if (n_rect <= 0 || Kz < 2) return;
  zone_kernel<T><<<(unsigned)n_rect, 256, 0, s>>>(msb, mea, pitch, rects, row_begin, row0, Kz, set);
}

template <typename T, int K>
void pml_launch(const PmlParams<T>& p, bool energy, cudaStream_t s) {
  const int WB = p.w + p.Kz + K + 2, Hr = p.chunk + 2 * K - 1;
  const size_t smem = sizeof(T) * ((size_t)5 * Hr * WB + WB + (size_t)2 * Hr * (WB + 1));
  dim3 grid((p.rows + p.chunk - 1) / p.chunk, 2);
  auto kern = energy ? pml_kernel<T, K, true> : pml_kernel<T, K, false>;
  if (smem > 32 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<grid, 256, smem, s>>>(p);
}

template <typename T>
void launch_pml(const PmlParams<T>& p, int K, bool energy, cudaStream_t s) {
  if (p.w <= 0 || p.rows <= 0) return;
  if (K == 1) pml_launch<T, 1>(p, energy, s);
  else if (K == 2) pml_launch<T, 2>(p, energy, s);
  else if constexpr (sizeof(T) == 4) pml_launch<T, 4>(p, energy, s);
}

template <typename T>
void launch_band_marks(T* msb, const T* mea, int64_t pitch, int64_t nx, int row0, int rows, int ncol, bool set,
                       cudaStream_t s) {
  if (rows <= 0 || ncol <= 0) return;
  band_marks_kernel<T><<<rows, 128, 0, s>>>(msb, mea, pitch, nx, row0, ncol, set);
}

#define INST(T)                                                                                     \
  template void launch_sweep<T>(const SweepParams<T>&, int, int, cudaStream_t, int, int);         \
  template void launch_post<T>(const PostParams<T>&, int, bool, cudaStream_t);                   \
  template void launch_post_big<T>(const PostParams<T>&, int, bool, cudaStream_t);               \
  template void launch_wholegrid<T>(const PostParams<T>&, int64_t, bool, cudaStream_t);          \
  template int big_grid_size<T>(size_t, int);                                                     \
  template void launch_materials<T, float>(const float*, const float*, int64_t, int64_t, int64_t, int64_t, \
                                           int64_t, int, int, int64_t, double, T*, T*, cudaStream_t);     \
  template void launch_materials<T, double>(const double*, const double*, int64_t, int64_t, int64_t,      \
                                            int64_t, int64_t, int, int, int64_t, double, T*, T*,          \
                                            cudaStream_t);                                                \
  template void launch_random_fields<T>(T*, T*, T*, const T*, int64_t, int64_t, int, int, int64_t, uint64_t, \
                                        double, double, cudaStream_t);                                     \
  template void launch_zone<T>(T*, const T*, int64_t, const int32_t*, int64_t, int64_t, int, int, bool,   \
                               cudaStream_t);                                                             \
  template void launch_pml<T>(const PmlParams<T>&, int, bool, cudaStream_t);                             \
  template void launch_band_marks<T>(T*, const T*, int64_t, int64_t, int, int, int, bool, cudaStream_t);  \
  template void launch_mask<T>(T*, T* [6], int64_t, const int32_t*, int64_t, int64_t, int, bool, cudaStream_t);
INST(float)
INST(double)
template void launch_gather_materials<float>(const float*, const float*, int64_t, int64_t,
                                             const int64_t*, int64_t, double*, double*, cudaStream_t);
template void launch_gather_materials<double>(const double*, const double*, int64_t, int64_t,
                                              const int64_t*, int64_t, double*, double*, cudaStream_t);

}  // namespace fdtd
