// GPU-side ROM construction, declared in include/fdtdrom_build.h.
//
// Steps (PAPER.md lines): fine assembly of the refined block with the exact collapse onto
// coarse-edge ports (Sec. II, eq:equalE, R9; or the literal nP-port
// set of NEXT-1) -> SPRIM block Arnoldi (L393-400, R10) with the shifted systems solved
// in H form (multigrid-preconditioned CG on the cell stencil) -> the E and H rows orthonormalised
// in Krylov order -> congruence (eq:R11_tilde .. eq:K_tilde, L431-447) -> optional CFL extension
// (eq:CFLgeneralized L741-745, R11) through one-sided Jacobi SVDs.
//
// Design: every O(n) or larger step runs in kernels of this file; the host only
// sequences them and takes the scalar decisions (Gram-Schmidt deflation, Jacobi convergence).  The
// fine operator is never formed as a matrix product: K is a CSR of the collapsed curl (r entries
// on port rows, 2 on interior rows; K^T 4 per cell), and the H-form Schur complement
// s0 R22 + K^T D^-1 K is a 5-point cell stencil plus one rank-1 block per port.  The CG runs one
// CTA per right-hand side for the whole iteration, the Jacobi SVD one CTA per column pair (a whole
// sweep per cooperative launch), the dense products in a tiled fp64 kernel.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "fdtdrom_build.h"

namespace {

namespace cg = cooperative_groups;

constexpr double PI = 3.14159265358979323846;
constexpr double MU0 = 4.0e-7 * PI;
constexpr double C0 = 299792458.0;
constexpr double EPS0 = 1.0 / (MU0 * C0 * C0);

thread_local std::string g_err;

fdtd_status failf(fdtd_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define CUCK(call)                                                                               \
  do {                                                                                           \
    cudaError_t e_ = (call);                                                                     \
    if (e_ != cudaSuccess) return failf(FDTD_E_CUDA, "%s: %s", #call, cudaGetErrorString(e_));   \
  } while (0)
#define STCK(call)                              \
  do {                                          \
    fdtd_status s_ = (call);                    \
    if (s_ != FDTD_OK) return s_;               \
  } while (0)

// ------------------------------------------------------------------------------------------
// geometry of the collapsed system (R9): ports first (S bx, N bx, W by, E by coarse
// edges), then the interior fine E nodes in fine order (Ex rows 1 .. Ny-1, then Ey columns
// 1 .. Nx-1 row by row); H cells row-major.
struct Geo {
  int bx, by, r, Nx, Ny, nY, nEc, nH;
  double fdx, fdy;
  __host__ __device__ int ex(int i, int j) const {  // collapsed index of fine Ex node (i, j)
    if (j == 0) return i / r;
    if (j == Ny) return bx + i / r;
    return nY + (j - 1) * Nx + i;
  }
  __host__ __device__ int ey(int i, int j) const {  // collapsed index of fine Ey node (i, j)
    if (i == 0) return 2 * bx + j / r;
    if (i == Nx) return 2 * bx + by + j / r;
    return nY + (Ny - 1) * Nx + j * (Nx - 1) + (i - 1);
  }
  __host__ __device__ int rowptr(int e) const { return e < nY ? e * r : nY * r + (e - nY) * 2; }
};

// E nodes: R11, F11 diagonals (eq:R11 = D_l D_l' D_eps, eq:F11 = D_l D_l' D_sigma / 2, summed over
// the r fine nodes of a port) and the collapsed K rows (eq:K: +dx^ H_above - dx^ H_below for Ex,
// -dy^ H_right + dy^ H_left for Ey, sign of eq:updateEymat).
__global__ void assemble_e_kernel(Geo g, const double* eps, const double* sig, double* r11, double* f11,
                                  int* col, double* val, double* Sc) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= g.nEc) return;
  const int Nx = g.Nx, Ny = g.Ny;
  double a = 0.0, f = 0.0;
  int p = g.rowptr(e);
  if (e < g.nY) {
    int side, k;
    if (e < g.bx) { side = 0; k = e; }
    else if (e < 2 * g.bx) { side = 1; k = e - g.bx; }
    else if (e < 2 * g.bx + g.by) { side = 2; k = e - 2 * g.bx; }
    else { side = 3; k = e - 2 * g.bx - g.by; }
    for (int t = k * g.r; t < (k + 1) * g.r; ++t) {
      if (side == 0) {  // S: Ex(t, 0), half dual length, the cell above
        a += g.fdx * (g.fdy / 2) * EPS0 * eps[t]; f += g.fdx * (g.fdy / 2) * sig[t] / 2;
        col[p] = t; val[p++] = +g.fdx;
      } else if (side == 1) {  // N: Ex(t, Ny), the cell below
        const int c = (Ny - 1) * Nx + t;
        a += g.fdx * (g.fdy / 2) * EPS0 * eps[c]; f += g.fdx * (g.fdy / 2) * sig[c] / 2;
        col[p] = c; val[p++] = -g.fdx;
      } else if (side == 2) {  // W: Ey(0, t), the cell to the right
        const int c = t * Nx;
        a += g.fdy * (g.fdx / 2) * EPS0 * eps[c]; f += g.fdy * (g.fdx / 2) * sig[c] / 2;
        col[p] = c; val[p++] = -g.fdy;
      } else {  // E: Ey(Nx, t), the cell to the left
        const int c = t * Nx + Nx - 1;
        a += g.fdy * (g.fdx / 2) * EPS0 * eps[c]; f += g.fdy * (g.fdx / 2) * sig[c] / 2;
        col[p] = c; val[p++] = +g.fdy;
      }
    }
    Sc[e] = side == 0 ? -g.fdx * g.r : side == 1 ? g.fdx * g.r : side == 2 ? g.fdy * g.r : -g.fdy * g.r;
  } else if (e - g.nY < (Ny - 1) * Nx) {  // interior Ex(i, j): mean of the cells below and above
    const int t = e - g.nY, j = t / Nx + 1, i = t % Nx;
    const double ea = 0.5 * (eps[(j - 1) * Nx + i] + eps[j * Nx + i]);
    const double sa = 0.5 * (sig[(j - 1) * Nx + i] + sig[j * Nx + i]);
    a = g.fdx * g.fdy * EPS0 * ea; f = g.fdx * g.fdy * sa / 2;
    col[p] = j * Nx + i; val[p++] = +g.fdx;
    col[p] = (j - 1) * Nx + i; val[p++] = -g.fdx;
  } else {  // interior Ey(i, j): mean of the cells left and right
    const int t = e - g.nY - (Ny - 1) * Nx, j = t / (Nx - 1), i = t % (Nx - 1) + 1;
    const double ea = 0.5 * (eps[j * Nx + i - 1] + eps[j * Nx + i]);
    const double sa = 0.5 * (sig[j * Nx + i - 1] + sig[j * Nx + i]);
    a = g.fdy * g.fdx * EPS0 * ea; f = g.fdy * g.fdx * sa / 2;
    col[p] = j * Nx + i; val[p++] = -g.fdy;
    col[p] = j * Nx + i - 1; val[p++] = +g.fdy;
  }
  r11[e] = a;
  f11[e] = f;
}

// H cells: R22 = D_A D_mu (mu = mu0, R3) and the 4 entries of K^T per cell.
__global__ void assemble_h_kernel(Geo g, double* r22, int* colT, double* valT) {
  const int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= g.nH) return;
  const int i = h % g.Nx, j = h / g.Nx;
  r22[h] = g.fdx * g.fdy * MU0;
  colT[4 * h + 0] = g.ex(i, j);     valT[4 * h + 0] = +g.fdx;
  colT[4 * h + 1] = g.ex(i, j + 1); valT[4 * h + 1] = -g.fdx;
  colT[4 * h + 2] = g.ey(i, j);     valT[4 * h + 2] = -g.fdy;
  colT[4 * h + 3] = g.ey(i + 1, j); valT[4 * h + 3] = +g.fdy;
}

// d = 2 F11 + s0 R11, dH = 1 / (s0 R22), minv = 1 / diag(S) (Jacobi preconditioner)
__global__ void schur_diag_kernel(Geo g, double s0, const double* r11, const double* f11, const double* r22,
                                  const int* col, const double* val, double* d, double* dH, double* minv) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < g.nH) dH[e] = 1.0 / (s0 * r22[e]);
  if (e >= g.nEc) return;
  const double de = 2.0 * f11[e] + s0 * r11[e];
  double s = de;
  for (int p = g.rowptr(e); p < g.rowptr(e + 1); ++p) s += val[p] * val[p] / (s0 * r22[col[p]]);
  d[e] = de;
  minv[e] = 1.0 / s;
}

// Y[:, c] = A[:, c] + K (w o X[:, c]) (nEc rows; w = nullptr: 1, A = nullptr: 0)
__global__ void k_apply_kernel(Geo g, const int* col, const double* val, const double* w, const double* X, int ldx,
                               const double* A, int lda, double* Y, int ldy, int ncol) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x, c = blockIdx.y;
  if (e >= g.nEc || c >= ncol) return;
  const double* x = X + (size_t)c * ldx;
  double s = A ? A[(size_t)c * lda + e] : 0.0;
  for (int p = g.rowptr(e); p < g.rowptr(e + 1); ++p) s += val[p] * (w ? w[col[p]] : 1.0) * x[col[p]];
  Y[(size_t)c * ldy + e] = s;
}

// xH = dH o (bH - K^T xE)
__global__ void h_recover_kernel(Geo g, const int* colT, const double* valT, const double* dH, const double* XE,
                                 int ldxe, const double* BH, int ldbh, double* XH, int ldxh, int ncol) {
  const int h = blockIdx.x * blockDim.x + threadIdx.x, c = blockIdx.y;
  if (h >= g.nH || c >= ncol) return;
  const double* x = XE + (size_t)c * ldxe;
  const double kt = valT[4 * h] * x[colT[4 * h]] + valT[4 * h + 1] * x[colT[4 * h + 1]] +
                    valT[4 * h + 2] * x[colT[4 * h + 2]] + valT[4 * h + 3] * x[colT[4 * h + 3]];
  XH[(size_t)c * ldxh + h] = dH[h] * ((BH ? BH[(size_t)c * ldbh + h] : 0.0) - kt);
}

template <int NT>
__device__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < NT / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

// Jacobi-preconditioned CG on S x = b, one CTA per right-hand side for the whole iteration
// (x, r, p, Ap in global memory: L2-resident for the block sizes of the configs).
struct CGArgs {
  Geo g;
  const int* col; const double* val; const int* colT; const double* valT;
  const double *d, *dH, *minv;
  const double* B; int ldb;  // right-hand sides (nEc x ncol)
  double* X; int ldx;        // solutions
  double *R, *P, *AP, *T;    // scratch: nEc (R, P, AP) / nH (T) per column
  double tol; int maxit;
  int* iters;                // per column (-1: not converged)
};
constexpr int CG_NT = 1024;
__global__ void __launch_bounds__(CG_NT) cg_kernel(CGArgs a) {
  __shared__ double red[32];
  const int c = blockIdx.x, n = a.g.nEc, nh = a.g.nH, tid = threadIdx.x;
  const double* b = a.B + (size_t)c * a.ldb;
  double* x = a.X + (size_t)c * a.ldx;
  double* r = a.R + (size_t)c * n;
  double* p = a.P + (size_t)c * n;
  double* ap = a.AP + (size_t)c * n;
  double* t = a.T + (size_t)c * nh;
  double bb = 0.0, rz = 0.0;
  for (int i = tid; i < n; i += CG_NT) {
    const double bi = b[i], zi = a.minv[i] * bi;
    x[i] = 0.0; r[i] = bi; p[i] = zi;
    bb += bi * bi; rz += bi * zi;
  }
  bb = block_sum<CG_NT>(bb, red);
  rz = block_sum<CG_NT>(rz, red);
  const double stop = a.tol * a.tol * bb;
  if (bb == 0.0) { if (tid == 0) a.iters[c] = 0; return; }
  int it = 0;
  for (; it < a.maxit; ++it) {
    for (int h = tid; h < nh; h += CG_NT)
      t[h] = a.dH[h] * (a.valT[4 * h] * p[a.colT[4 * h]] + a.valT[4 * h + 1] * p[a.colT[4 * h + 1]] +
                        a.valT[4 * h + 2] * p[a.colT[4 * h + 2]] + a.valT[4 * h + 3] * p[a.colT[4 * h + 3]]);
    __syncthreads();
    double pap = 0.0;
    for (int i = tid; i < n; i += CG_NT) {
      double s = a.d[i] * p[i];
      for (int q = a.g.rowptr(i); q < a.g.rowptr(i + 1); ++q) s += a.val[q] * t[a.col[q]];
      ap[i] = s;
      pap += p[i] * s;
    }
    pap = block_sum<CG_NT>(pap, red);
    const double alpha = rz / pap;
    double rr = 0.0, rzn = 0.0;
    for (int i = tid; i < n; i += CG_NT) {
      x[i] += alpha * p[i];
      const double ri = r[i] - alpha * ap[i];
      r[i] = ri;
      rr += ri * ri;
      rzn += ri * a.minv[i] * ri;
    }
    rr = block_sum<CG_NT>(rr, red);
    rzn = block_sum<CG_NT>(rzn, red);
    if (rr <= stop) { ++it; break; }
    const double beta = rzn / rz;
    rz = rzn;
    for (int i = tid; i < n; i += CG_NT) p[i] = a.minv[i] * r[i] + beta * p[i];
    __syncthreads();
  }
  if (tid == 0) a.iters[c] = it < a.maxit ? it : -1;
}

// ---- H-form shifted solves: eliminate E instead of H,
//   (s0 R22 + K^T D^-1 K) xH = bH - K^T D^-1 bE,   xE = D^-1 (bE + K xH),   D = 2 F11 + s0 R11.
// S_H is a 5-point stencil on the fine cells (one coupling per interior edge) plus one rank-1 block
// per port (the r cells along a coarse interface edge).  CG preconditioned by a geometric multigrid
// V-cycle (2 x 2 aggregation, Galerkin coarse stencils, symmetric red-black Gauss-Seidel) on the
// stencil with the port blocks' diagonal; one CTA per right-hand side for the whole iteration.
constexpr int MG_MAXLEV = 16;
struct MGLevel { int nx, ny; long off; };
struct MGArgs {
  Geo g;
  int nlev; MGLevel lev[MG_MAXLEV];
  const double *cc, *we, *wn;  // per level (pool offsets): diagonal, east and north couplings
  const float *fcc, *fwe, *fwn;  // the same in fp32: the V-cycle is a preconditioner, run in fp32
  const double* cS;            // level-0 exact stencil diagonal (no port terms)
  const double* pw;            // per port: v^2 / D_e (v = fdx for S/N ports, fdy for W/E)
  const double* B; int ldb;    // right-hand sides (nH x ncol)
  double* X; int ldx;          // solutions
  double* work; long wstride;  // per column: r, z, p, q (4 nH doubles), then the V-cycle's fp32
                               // x, b of every level (level 0 first)
  double* psum;                // per column: nY
  double tol; int maxit; int* iters;
};

// level-0 stencil: we(i,j) couples (i,j)-(i+1,j) through interior Ey(i+1,j); wn(i,j) couples
// (i,j)-(i,j+1) through interior Ex(i,j+1) (entries k_a k_b / D_e = -fdy^2/D, -fdx^2/D)
__global__ void hs_setup0_kernel(Geo g, double s0, const double* r22, const double* d, double* cS, double* cc,
                                 double* we, double* wn, double* pw) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < g.nY) pw[t] = (t < 2 * g.bx ? g.fdx * g.fdx : g.fdy * g.fdy) / d[t];
  if (t >= g.nH) return;
  const int i = t % g.Nx, j = t / g.Nx;
  we[t] = i < g.Nx - 1 ? -g.fdy * g.fdy / d[g.ey(i + 1, j)] : 0.0;
  wn[t] = j < g.Ny - 1 ? -g.fdx * g.fdx / d[g.ex(i, j + 1)] : 0.0;
}
__global__ void hs_setup0b_kernel(Geo g, double s0, const double* r22, const double* pw, double* cS, double* cc,
                                  const double* we, const double* wn) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= g.nH) return;
  const int i = t % g.Nx, j = t / g.Nx;
  double c = s0 * r22[t] - we[t] - wn[t];
  if (i > 0) c -= we[t - 1];
  if (j > 0) c -= wn[t - g.Nx];
  cS[t] = c;
  if (j == 0) c += pw[i / g.r];
  if (j == g.Ny - 1) c += pw[g.bx + i / g.r];
  if (i == 0) c += pw[2 * g.bx + j / g.r];
  if (i == g.Nx - 1) c += pw[2 * g.bx + g.by + j / g.r];
  cc[t] = c;
}
// Galerkin coarsening with piecewise-constant 2 x 2 aggregation: A_c = P^T A P
__global__ void hs_coarsen_kernel(MGLevel f, MGLevel c, const double* cc_f, const double* we_f, const double* wn_f,
                                  double* cc_c, double* we_c, double* wn_c) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= c.nx * c.ny) return;
  const int I = t % c.nx, J = t / c.nx;
  const int i0 = 2 * I, j0 = 2 * J, i1 = min(i0 + 1, f.nx - 1), j1 = min(j0 + 1, f.ny - 1);
  double dg = 0.0, e = 0.0, n = 0.0;
  for (int j = j0; j <= j1; ++j)
    for (int i = i0; i <= i1; ++i) {
      const int k = j * f.nx + i;
      dg += cc_f[k];
      if (i < i1) dg += 2.0 * we_f[k];  // internal horizontal coupling
      if (j < j1) dg += 2.0 * wn_f[k];  // internal vertical coupling
      if (i == i1 && I + 1 < c.nx) e += we_f[k];
      if (j == j1 && J + 1 < c.ny) n += wn_f[k];
    }
  cc_c[t] = dg;
  we_c[t] = e;
  wn_c[t] = n;
}

constexpr int MG_NT = 1024;
__device__ __forceinline__ void mg_smooth(const MGArgs& a, int l, float* x, const float* b, int color) {
  const MGLevel L = a.lev[l];
  const float *c = a.fcc + L.off, *we = a.fwe + L.off, *wn = a.fwn + L.off;
  const int nx = L.nx, n = L.nx * L.ny;
  // cells of one colour: (i + j) % 2 == color; thread t handles the t-th such cell
  const int half = (n + 1) / 2 + 1;
  for (int u = threadIdx.x; u < half; u += MG_NT) {
    // row-major walk over the colour: cell index k = 2u + ((row parity) ^ color) within its row
    const int k2 = 2 * u;
    int j = k2 / nx, i = k2 % nx;
    if (((i + j) & 1) != color) ++i;
    if (i >= nx) { i -= nx; ++j; }
    if (j >= L.ny) continue;
    const int k = j * nx + i;
    if (k >= n) continue;
    float s = b[k];
    if (i > 0) s -= we[k - 1] * x[k - 1];
    if (i < nx - 1) s -= we[k] * x[k + 1];
    if (j > 0) s -= wn[k - nx] * x[k - nx];
    if (j < L.ny - 1) s -= wn[k] * x[k + nx];
    x[k] = s / c[k];
  }
  __syncthreads();
}
__device__ __forceinline__ void mg_restrict(const MGArgs& a, int l, const float* x, const float* b, float* bc) {
  const MGLevel f = a.lev[l], c = a.lev[l + 1];
  const float *cc = a.fcc + f.off, *we = a.fwe + f.off, *wn = a.fwn + f.off;
  for (int t = threadIdx.x; t < c.nx * c.ny; t += MG_NT) {
    const int I = t % c.nx, J = t / c.nx;
    const int i0 = 2 * I, j0 = 2 * J, i1 = min(i0 + 1, f.nx - 1), j1 = min(j0 + 1, f.ny - 1);
    float s = 0.f;
    for (int j = j0; j <= j1; ++j)
      for (int i = i0; i <= i1; ++i) {
        const int k = j * f.nx + i;
        float r = b[k] - cc[k] * x[k];
        if (i > 0) r -= we[k - 1] * x[k - 1];
        if (i < f.nx - 1) r -= we[k] * x[k + 1];
        if (j > 0) r -= wn[k - f.nx] * x[k - f.nx];
        if (j < f.ny - 1) r -= wn[k] * x[k + f.nx];
        s += r;
      }
    bc[t] = s;
  }
  __syncthreads();
}
__device__ __forceinline__ void mg_prolong(const MGArgs& a, int l, float* x, const float* xc) {
  const MGLevel f = a.lev[l], c = a.lev[l + 1];
  for (int k = threadIdx.x; k < f.nx * f.ny; k += MG_NT) {
    const int i = k % f.nx, j = k / f.nx;
    x[k] += xc[(j / 2) * c.nx + i / 2];
  }
  __syncthreads();
}
// z = V-cycle(r) (fp32 inside, fp64 in and out): symmetric (pre: red-black, post: black-red;
// coarsest: symmetric sweep pairs)
__device__ void mg_vcycle(const MGArgs& a, double* wcol, double* z, const double* r) {
  constexpr int NU = 2, NCOARSE = 30;
  float* fb = reinterpret_cast<float*>(wcol + 4L * a.g.nH);
  auto xl = [&](int l) { return fb + 2 * a.lev[l].off; };
  auto bl = [&](int l) { return fb + 2 * a.lev[l].off + a.lev[l].nx * a.lev[l].ny; };
  for (int k = threadIdx.x; k < a.g.nH; k += MG_NT) bl(0)[k] = (float)r[k];
  for (int l = 0; l < a.nlev; ++l) {
    float* x = xl(l);
    for (int k = threadIdx.x; k < a.lev[l].nx * a.lev[l].ny; k += MG_NT) x[k] = 0.f;
    __syncthreads();
    if (l == a.nlev - 1) {
      for (int it = 0; it < NCOARSE; ++it) {
        mg_smooth(a, l, x, bl(l), 0); mg_smooth(a, l, x, bl(l), 1);
        mg_smooth(a, l, x, bl(l), 1); mg_smooth(a, l, x, bl(l), 0);
      }
      break;
    }
    for (int it = 0; it < NU; ++it) { mg_smooth(a, l, x, bl(l), 0); mg_smooth(a, l, x, bl(l), 1); }
    mg_restrict(a, l, x, bl(l), bl(l + 1));
  }
  for (int l = a.nlev - 2; l >= 0; --l) {
    mg_prolong(a, l, xl(l), xl(l + 1));
    for (int it = 0; it < NU; ++it) { mg_smooth(a, l, xl(l), bl(l), 1); mg_smooth(a, l, xl(l), bl(l), 0); }
  }
  for (int k = threadIdx.x; k < a.g.nH; k += MG_NT) z[k] = (double)xl(0)[k];
  __syncthreads();
}
__global__ void to_f32_kernel(const double* a, float* b, long n) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = (float)a[i];
}
// q = S_H p exactly (stencil with cS + the port rank-1 blocks)
__device__ __forceinline__ void hs_apply(const MGArgs& a, const double* p, double* q, double* ps) {
  const Geo& g = a.g;
  for (int e = threadIdx.x; e < g.nY; e += MG_NT) {
    double s = 0.0;
    for (int u = 0; u < g.r; ++u) {
      int cell;
      if (e < g.bx) cell = e * g.r + u;                                             // S: row 0
      else if (e < 2 * g.bx) cell = (g.Ny - 1) * g.Nx + (e - g.bx) * g.r + u;       // N: row Ny-1
      else if (e < 2 * g.bx + g.by) cell = ((e - 2 * g.bx) * g.r + u) * g.Nx;       // W: column 0
      else cell = ((e - 2 * g.bx - g.by) * g.r + u) * g.Nx + g.Nx - 1;              // E: column Nx-1
      s += p[cell];
    }
    ps[e] = a.pw[e] * s;
  }
  __syncthreads();
  const int nx = g.Nx;
  for (int k = threadIdx.x; k < g.nH; k += MG_NT) {
    const int i = k % nx, j = k / nx;
    double y = a.cS[k] * p[k];
    if (i > 0) y += a.we[k - 1] * p[k - 1];
    if (i < nx - 1) y += a.we[k] * p[k + 1];
    if (j > 0) y += a.wn[k - nx] * p[k - nx];
    if (j < g.Ny - 1) y += a.wn[k] * p[k + nx];
    if (j == 0) y += ps[i / g.r];
    if (j == g.Ny - 1) y += ps[g.bx + i / g.r];
    if (i == 0) y += ps[2 * g.bx + j / g.r];
    if (i == nx - 1) y += ps[2 * g.bx + g.by + j / g.r];
    q[k] = y;
  }
  __syncthreads();
}
__global__ void __launch_bounds__(MG_NT) mg_pcg_kernel(MGArgs a) {
  __shared__ double red[32];
  const int c = blockIdx.x, n = a.g.nH, tid = threadIdx.x;
  const double* b = a.B + (size_t)c * a.ldb;
  double* x = a.X + (size_t)c * a.ldx;
  double* wcol = a.work + (size_t)c * a.wstride;
  double *r = wcol, *z = wcol + n, *p = wcol + 2L * n, *q = wcol + 3L * n;
  double* ps = a.psum + (size_t)c * a.g.nY;
  double bb = 0.0;
  for (int i = tid; i < n; i += MG_NT) { x[i] = 0.0; r[i] = b[i]; bb += b[i] * b[i]; }
  bb = block_sum<MG_NT>(bb, red);
  if (bb == 0.0) { if (tid == 0) a.iters[c] = 0; return; }
  const double stop = a.tol * a.tol * bb;
  mg_vcycle(a, wcol, z, r);
  double rz = 0.0;
  for (int i = tid; i < n; i += MG_NT) { p[i] = z[i]; rz += r[i] * z[i]; }
  rz = block_sum<MG_NT>(rz, red);
  int it = 0;
  for (; it < a.maxit; ++it) {
    hs_apply(a, p, q, ps);
    double pq = 0.0;
    for (int i = tid; i < n; i += MG_NT) pq += p[i] * q[i];
    pq = block_sum<MG_NT>(pq, red);
    const double alpha = rz / pq;
    double rr = 0.0;
    for (int i = tid; i < n; i += MG_NT) {
      x[i] += alpha * p[i];
      r[i] -= alpha * q[i];
      rr += r[i] * r[i];
    }
    rr = block_sum<MG_NT>(rr, red);
    if (rr <= stop) { ++it; break; }
    mg_vcycle(a, wcol, z, r);
    double rzn = 0.0;
    for (int i = tid; i < n; i += MG_NT) rzn += r[i] * z[i];
    rzn = block_sum<MG_NT>(rzn, red);
    const double beta = rzn / rz;
    rz = rzn;
    for (int i = tid; i < n; i += MG_NT) p[i] = z[i] + beta * p[i];
    __syncthreads();
  }
  if (tid == 0) a.iters[c] = it < a.maxit ? it : -1;
}
// rhsH = bH - K^T D^-1 bE
__global__ void hs_rhs_kernel(Geo g, const int* colT, const double* valT, const double* d, const double* BE, int ldbe,
                              const double* BH, int ldbh, double* R, int ldr, int ncol) {
  const int h = blockIdx.x * blockDim.x + threadIdx.x, c = blockIdx.y;
  if (h >= g.nH || c >= ncol) return;
  const double* e = BE + (size_t)c * ldbe;
  double s = 0.0;
  for (int u = 0; u < 4; ++u) s += valT[4 * h + u] * e[colT[4 * h + u]] / d[colT[4 * h + u]];
  R[(size_t)c * ldr + h] = (BH ? BH[(size_t)c * ldbh + h] : 0.0) - s;
}
// xE = D^-1 (bE + K xH)
__global__ void hs_erec_kernel(Geo g, const int* col, const double* val, const double* d, const double* BE, int ldbe,
                               const double* XH, int ldxh, double* XE, int ldxe, int ncol) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x, c = blockIdx.y;
  if (e >= g.nEc || c >= ncol) return;
  const double* xh = XH + (size_t)c * ldxh;
  double s = BE[(size_t)c * ldbe + e];
  for (int p = g.rowptr(e); p < g.rowptr(e + 1); ++p) s += val[p] * xh[col[p]];
  XE[(size_t)c * ldxe + e] = s / d[e];
}

// ---- Gram-Schmidt in the C inner product (c = [R11; R22] diagonal)
// out[0] = sum c v^2 (one CTA; fixed order)
constexpr int RN_NT = 1024;
__global__ void __launch_bounds__(RN_NT) cnorm2_kernel(const double* c, const double* v, int n, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += RN_NT) s += (c ? c[i] : 1.0) * v[i] * v[i];
  s = block_sum<RN_NT>(s, red);
  if (threadIdx.x == 0) *out = s;
}
// h[k] = W[:, k]^T (c o v), one CTA per k
constexpr int GV_NT = 256;
__global__ void __launch_bounds__(GV_NT) wtcv_kernel(const double* W, int ldw, const double* c, const double* v,
                                                     int n, double* h) {
  __shared__ double red[32];
  const double* w = W + (size_t)blockIdx.x * ldw;
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += GV_NT) s += w[i] * (c ? c[i] : 1.0) * v[i];
  s = block_sum<GV_NT>(s, red);
  if (threadIdx.x == 0) h[blockIdx.x] = s;
}
// v -= W[:, :k] h
__global__ void v_minus_wh_kernel(const double* W, int ldw, const double* h, int k, double* v, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int j = 0; j < k; ++j) s += W[(size_t)j * ldw + i] * h[j];
  v[i] -= s;
}
// Two-level fixed-order versions for long vectors: slice partials, then one ordered sum.
constexpr int RED_SLICE = 8192;  // rows per partial
__global__ void __launch_bounds__(GV_NT) cnorm2_part_kernel(const double* c, const double* v, int n, double* part) {
  __shared__ double red[32];
  const int i0 = blockIdx.x * RED_SLICE, i1 = min(n, i0 + RED_SLICE);
  double s = 0.0;
  for (int i = i0 + threadIdx.x; i < i1; i += GV_NT) s += (c ? c[i] : 1.0) * v[i] * v[i];
  s = block_sum<GV_NT>(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}
// h_part[g * k + col] = slice g of W[:, col]^T (c o v)
__global__ void __launch_bounds__(GV_NT) wtcv_part_kernel(const double* W, int ldw, const double* c, const double* v,
                                                          int n, int k, double* part) {
  __shared__ double red[32];
  const int col = blockIdx.x, g = blockIdx.y;
  const int i0 = g * RED_SLICE, i1 = min(n, i0 + RED_SLICE);
  const double* w = W + (size_t)col * ldw;
  double s = 0.0;
  for (int i = i0 + threadIdx.x; i < i1; i += GV_NT) s += w[i] * (c ? c[i] : 1.0) * v[i];
  s = block_sum<GV_NT>(s, red);
  if (threadIdx.x == 0) part[(size_t)g * k + col] = s;
}
// out[j] = sum over g of part[g * m + j], in order (m outputs, ng slices)
__global__ void sum_parts_kernel(const double* part, int ng, int m, double* out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  double s = 0.0;
  for (int g = 0; g < ng; ++g) s += part[(size_t)g * m + j];
  out[j] = s;
}
__global__ void scale_copy_kernel(const double* v, double a, double* out, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = a * v[i];
}
// Out[:, t] = w o In[rows, idx[t]] (gather columns, optional row weights)
__global__ void gather_cols_kernel(const double* In, int ldi, const int* idx, const double* w, int rows, double* Out,
                                   int ldo, int ncol) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, t = blockIdx.y;
  if (i >= rows || t >= ncol) return;
  Out[(size_t)t * ldo + i] = (w ? w[i] : 1.0) * In[(size_t)idx[t] * ldi + i];
}

// ---- one-sided Jacobi SVD (Hestenes): one round of the round-robin pairing, one CTA per pair.
// Players 0 .. mp-1 (mp even); in round t player 0 is fixed and the others rotate.
constexpr int JB_NT = 256;
__device__ __forceinline__ void jacobi_pair(double* A, int lda, int rows, int m, double* V, int ldv, int vrows,
                                            int mp, int t, int pair, double tol, double floor2, int* rotated,
                                            double* red) {
  auto player = [&](int k) { return k == 0 ? 0 : (k - 1 + t) % (mp - 1) + 1; };
  int a = player(pair), b = player(mp - 1 - pair);
  if (a >= m || b >= m) return;  // uniform over the CTA
  if (a > b) { const int x = a; a = b; b = x; }
  double* ca = A + (size_t)a * lda;
  double* cb = A + (size_t)b * lda;
  double al = 0.0, be = 0.0, ga = 0.0;
  for (int i = threadIdx.x; i < rows; i += JB_NT) {
    const double x = ca[i], y = cb[i];
    al += x * x; be += y * y; ga += x * y;
  }
  al = block_sum<JB_NT>(al, red);
  be = block_sum<JB_NT>(be, red);
  ga = block_sum<JB_NT>(ga, red);
  // converged pair, or a column at rounding level of the largest (floor2 = (1e-15 s_max)^2): such
  // directions are below every rank tolerance used here and would rotate forever on noise
  if (ga == 0.0 || fabs(ga) <= tol * sqrt(al * be) || al < floor2 || be < floor2) return;
  const double zeta = (be - al) / (2.0 * ga);
  const double tt = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + hypot(1.0, zeta));
  const double cs = 1.0 / hypot(1.0, tt), sn = cs * tt;
  for (int i = threadIdx.x; i < rows; i += JB_NT) {
    const double x = ca[i], y = cb[i];
    ca[i] = cs * x - sn * y;
    cb[i] = sn * x + cs * y;
  }
  if (V) {
    double* va = V + (size_t)a * ldv;
    double* vb = V + (size_t)b * ldv;
    for (int i = threadIdx.x; i < vrows; i += JB_NT) {
      const double x = va[i], y = vb[i];
      va[i] = cs * x - sn * y;
      vb[i] = sn * x + cs * y;
    }
  }
  if (threadIdx.x == 0) atomicAdd(rotated, 1);
  __syncthreads();
}
__global__ void __launch_bounds__(JB_NT) jacobi_round_kernel(double* A, int lda, int rows, int m, double* V,
                                                             int ldv, int vrows, int mp, int t, double tol,
                                                             double floor2, int* rotated) {
  __shared__ double red[32];
  jacobi_pair(A, lda, rows, m, V, ldv, vrows, mp, t, blockIdx.x, tol, floor2, rotated, red);
}
// a whole sweep (mp - 1 rounds) in one cooperative launch: grid-wide barrier between rounds
__global__ void __launch_bounds__(JB_NT) jacobi_sweep_kernel(double* A, int lda, int rows, int m, double* V,
                                                             int ldv, int vrows, int mp, double tol, double floor2,
                                                             int* rotated) {
  __shared__ double red[32];
  cg::grid_group grid = cg::this_grid();
  for (int t = 0; t < mp - 1; ++t) {
    for (int pair = blockIdx.x; pair < mp / 2; pair += gridDim.x)
      jacobi_pair(A, lda, rows, m, V, ldv, vrows, mp, t, pair, tol, floor2, rotated, red);
    grid.sync();
  }
}
// norms of the columns
__global__ void __launch_bounds__(JB_NT) colnorm_kernel(const double* A, int lda, int rows, double* out) {
  __shared__ double red[32];
  const double* c = A + (size_t)blockIdx.x * lda;
  double s = 0.0;
  for (int i = threadIdx.x; i < rows; i += JB_NT) s += c[i] * c[i];
  s = block_sum<JB_NT>(s, red);
  if (threadIdx.x == 0) out[blockIdx.x] = sqrt(s);
}
// Out[:, t] = In[:, perm[t]] * scale[t]
__global__ void permute_scale_kernel(const double* In, int ldi, const int* perm, const double* scale, int rows,
                                     double* Out, int ldo, int ncol) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, t = blockIdx.y;
  if (i >= rows || t >= ncol) return;
  Out[(size_t)t * ldo + i] = In[(size_t)perm[t] * ldi + i] * (scale ? scale[t] : 1.0);
}
__global__ void identity_kernel(double* V, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n * n) V[i] = (i % n == i / n) ? 1.0 : 0.0;
}

// ---- dense fp64 C (M x N) = op(A) diag(w) op(B), column-major; 32 x 32 tiles, 256 threads.
constexpr int GT = 32;
template <bool TA, bool TB>
__global__ void __launch_bounds__(256) gemm_kernel(int M, int N, int K, const double* A, int lda, const double* w,
                                                   const double* B, int ldb, double* C, int ldc, int kchunk) {
  // blockIdx.z: a K range of kchunk (split-K); C then points at this split's partial matrix
  __shared__ double As[GT][GT + 1], Bs[GT][GT + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;  // 16 x 16 threads, 2 x 2 outputs each
  const int i0 = blockIdx.x * GT, j0 = blockIdx.y * GT;
  const int kb0 = blockIdx.z * kchunk, kb1 = min(K, kb0 + kchunk);
  C += (size_t)blockIdx.z * ldc * N;
  double acc[2][2] = {{0, 0}, {0, 0}};
  for (int k0 = kb0; k0 < kb1; k0 += GT) {
    for (int t = threadIdx.x; t < GT * GT; t += 256) {
      // the index that is contiguous in memory runs fastest across threads (coalesced tiles)
      const int ii = TA ? t / GT : t % GT, kk = TA ? t % GT : t / GT;  // As[kk][ii] = op(A)(i0+ii, k0+kk) w
      const int gi = i0 + ii, gk = k0 + kk;
      double av = 0.0;
      if (gi < M && gk < kb1) av = TA ? A[(size_t)gi * lda + gk] : A[(size_t)gk * lda + gi];
      if (w && gk < kb1) av *= w[gk];
      As[kk][ii] = av;
      const int jj = TB ? t % GT : t / GT, kb = TB ? t / GT : t % GT;  // Bs[kb][jj] = op(B)(k0+kb, j0+jj)
      const int gj = j0 + jj, gkb = k0 + kb;
      double bv = 0.0;
      if (gj < N && gkb < kb1) bv = TB ? B[(size_t)gkb * ldb + gj] : B[(size_t)gj * ldb + gkb];
      Bs[kb][jj] = bv;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < GT; ++kk) {
      const double a0 = As[kk][tx], a1 = As[kk][tx + 16];
      const double b0 = Bs[kk][ty], b1 = Bs[kk][ty + 16];
      acc[0][0] += a0 * b0; acc[1][0] += a1 * b0; acc[0][1] += a0 * b1; acc[1][1] += a1 * b1;
    }
    __syncthreads();
  }
  for (int u = 0; u < 2; ++u)
    for (int v = 0; v < 2; ++v) {
      const int gi = i0 + tx + 16 * u, gj = j0 + ty + 16 * v;
      if (gi < M && gj < N) C[(size_t)gj * ldc + gi] = acc[u][v];
    }
}
// C = sum over the splits of the partials, in split order (deterministic)
__global__ void sum_splits_kernel(const double* P, int splits, int M, int N, double* C, int ldc) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long)M * N) return;
  const int i = (int)(t % M), j = (int)(t / M);
  double s = 0.0;
  for (int z = 0; z < splits; ++z) s += P[((size_t)z * N + j) * M + i];
  C[(size_t)j * ldc + i] = s;
}

// ------------------------------------------------------------------------------------------
// host side
// Stream-ordered device memory of one build (zeroed), from the device's default memory pool, which
// keeps freed blocks for the next build (no cudaMalloc / cudaFree round trips per buffer).
struct Dev {
  cudaStream_t s = nullptr;
  std::vector<void*> owned;
  ~Dev() { for (void* p : owned) cudaFreeAsync(p, s); }
  template <typename T>
  T* alloc(size_t n) {
    void* p = nullptr;
    const size_t bytes = std::max<size_t>(n, 1) * sizeof(T);
    if (cudaMallocAsync(&p, bytes, s) != cudaSuccess) return nullptr;
    owned.push_back(p);
    cudaMemsetAsync(p, 0, bytes, s);
    return (T*)p;
  }
};
void keep_pool_memory() {
  static bool done = false;
  if (done) return;
  done = true;
  int dev = 0;
  cudaMemPool_t pool;
  cudaGetDevice(&dev);
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
}

struct Timer {
  cudaEvent_t a = nullptr, b = nullptr;
  double ms = 0.0;
  Timer() { cudaEventCreate(&a); cudaEventCreate(&b); }
  ~Timer() { cudaEventDestroy(a); cudaEventDestroy(b); }
  void start(cudaStream_t s) { cudaEventRecord(a, s); }
  void stop(cudaStream_t s) {
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float t = 0.f;
    cudaEventElapsedTime(&t, a, b);
    ms += t;
  }
};

struct PhaseLog {  // FDTD_ROM_VERBOSE: device-synchronised wall time of each construction phase
  bool on = getenv("FDTD_ROM_VERBOSE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(cudaStream_t s, const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto n = std::chrono::steady_clock::now();
    fprintf(stderr, "rom_build %-12s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

inline unsigned blocks(long n, int nt) { return (unsigned)((n + nt - 1) / nt); }

struct Builder {
  Geo g{};
  double s0 = 0.0, cg_tol = 1e-13;
  cudaStream_t s = nullptr;
  Dev dev;
  // assembled system
  double *r11 = nullptr, *f11 = nullptr, *r22 = nullptr, *Sc = nullptr, *cdiag = nullptr;
  int *col = nullptr, *colT = nullptr;
  double *val = nullptr, *valT = nullptr, *d = nullptr, *dH = nullptr, *minv = nullptr;
  // CG scratch for up to cg_cols columns
  int cg_cols = 0;
  double *cgR = nullptr, *cgP = nullptr, *cgAP = nullptr, *cgT = nullptr, *rhs = nullptr;
  int* cg_it = nullptr;
  int cg_it_max = 0, jac_sweeps_max = 0;
  double* scal = nullptr;  // device scalars
  Timer t_solve, t_orth, t_svd;

  int n() const { return g.nEc + g.nH; }

  // multigrid hierarchy of the H-form solve
  int nlev = 0;
  MGLevel lev[MG_MAXLEV];
  double *mcc = nullptr, *mwe = nullptr, *mwn = nullptr, *mcS = nullptr, *mpw = nullptr;
  float *fcc = nullptr, *fwe = nullptr, *fwn = nullptr;
  double *hrhs = nullptr, *hwork = nullptr, *hpsum = nullptr;
  int h_cols = 0;
  long wstride = 0;
  bool h_form = true;
  int coop_grid = 0;  // co-resident CTAs of the cooperative Jacobi sweep (0: one launch per round)

  void setup_coop() {
    int dev_id = 0, nsm = 0, per = 0, coop = 0;
    cudaGetDevice(&dev_id);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev_id);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev_id);
    if (coop && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, jacobi_sweep_kernel, JB_NT, 0) == cudaSuccess)
      coop_grid = per * nsm;
    const char* e = getenv("FDTD_ROM_JACOBI_ROUNDS");  // 1: one launch per round (comparison)
    if (e && e[0] == '1') coop_grid = 0;
  }

  fdtd_status setup_mg() {
    long off = 0;
    int nx = g.Nx, ny = g.Ny;
    nlev = 0;
    while (true) {
      lev[nlev] = MGLevel{nx, ny, off};
      off += (long)nx * ny;
      ++nlev;
      if ((long)nx * ny <= 64 || nlev == MG_MAXLEV) break;
      nx = (nx + 1) / 2;
      ny = (ny + 1) / 2;
    }
    mcc = dev.alloc<double>(off); mwe = dev.alloc<double>(off); mwn = dev.alloc<double>(off);
    mcS = dev.alloc<double>(g.nH); mpw = dev.alloc<double>(g.nY);
    if (!mcc || !mwe || !mwn || !mcS || !mpw) return failf(FDTD_E_NOMEM, "multigrid hierarchy");
    hs_setup0_kernel<<<blocks(std::max(g.nH, g.nY), 256), 256, 0, s>>>(g, s0, r22, d, mcS, mcc, mwe, mwn, mpw);
    hs_setup0b_kernel<<<blocks(g.nH, 256), 256, 0, s>>>(g, s0, r22, mpw, mcS, mcc, mwe, mwn);
    for (int l = 0; l + 1 < nlev; ++l) {
      const MGLevel f = lev[l], c = lev[l + 1];
      hs_coarsen_kernel<<<blocks((long)c.nx * c.ny, 256), 256, 0, s>>>(f, c, mcc + f.off, mwe + f.off, mwn + f.off,
                                                                      mcc + c.off, mwe + c.off, mwn + c.off);
    }
    fcc = dev.alloc<float>(off); fwe = dev.alloc<float>(off); fwn = dev.alloc<float>(off);
    if (!fcc || !fwe || !fwn) return failf(FDTD_E_NOMEM, "multigrid hierarchy");
    to_f32_kernel<<<blocks(off, 256), 256, 0, s>>>(mcc, fcc, off);
    to_f32_kernel<<<blocks(off, 256), 256, 0, s>>>(mwe, fwe, off);
    to_f32_kernel<<<blocks(off, 256), 256, 0, s>>>(mwn, fwn, off);
    wstride = 4L * g.nH + (2 * off + 1) / 2;  // + the fp32 x, b of every level (in doubles)
    CUCK(cudaGetLastError());
    return FDTD_OK;
  }

  fdtd_status ensure_h(int ncol) {
    if (ncol <= h_cols) return FDTD_OK;
    h_cols = ncol;
    hrhs = dev.alloc<double>((size_t)ncol * g.nH);
    hwork = dev.alloc<double>((size_t)ncol * wstride);
    hpsum = dev.alloc<double>((size_t)ncol * g.nY);
    if (!cg_it) cg_it = dev.alloc<int>(std::max(ncol, 256));
    if (!hrhs || !hwork || !hpsum || !cg_it) return failf(FDTD_E_NOMEM, "H-form scratch");
    return FDTD_OK;
  }

  // H-form: rhsH = bH - K^T D^-1 bE; multigrid-PCG on S_H; xE = D^-1 (bE + K xH)
  fdtd_status solve_h(const double* BE, int ldbe, const double* BH, int ldbh, int ncol, double* X) {
    STCK(ensure_h(ncol));
    if (ncol > 256) return failf(FDTD_E_ARG, "block of %d right-hand sides", ncol);
    t_solve.start(s);
    const dim3 ge(blocks(g.nEc, 256), ncol), gh(blocks(g.nH, 256), ncol);
    hs_rhs_kernel<<<gh, 256, 0, s>>>(g, colT, valT, d, BE, ldbe, BH, ldbh, hrhs, g.nH, ncol);
    MGArgs a{};
    a.g = g; a.nlev = nlev;
    for (int l = 0; l < nlev; ++l) a.lev[l] = lev[l];
    a.cc = mcc; a.we = mwe; a.wn = mwn; a.cS = mcS; a.pw = mpw;
    a.fcc = fcc; a.fwe = fwe; a.fwn = fwn;
    a.B = hrhs; a.ldb = g.nH; a.X = X + g.nEc; a.ldx = n();
    a.work = hwork; a.wstride = wstride; a.psum = hpsum;
    a.tol = cg_tol; a.maxit = 5000; a.iters = cg_it;
    mg_pcg_kernel<<<ncol, MG_NT, 0, s>>>(a);
    hs_erec_kernel<<<ge, 256, 0, s>>>(g, col, val, d, BE, ldbe, X + g.nEc, n(), X, n(), ncol);
    CUCK(cudaGetLastError());
    std::vector<int> it(ncol);
    CUCK(cudaMemcpyAsync(it.data(), cg_it, sizeof(int) * ncol, cudaMemcpyDeviceToHost, s));
    t_solve.stop(s);
    for (int k = 0; k < ncol; ++k) {
      if (it[k] < 0) return failf(FDTD_E_STATE, "multigrid PCG did not converge to %.1e (column %d)", cg_tol, k);
      cg_it_max = std::max(cg_it_max, it[k]);
    }
    return FDTD_OK;
  }

  fdtd_status ensure_cg(int ncol) {
    if (ncol <= cg_cols) return FDTD_OK;
    cg_cols = ncol;
    cgR = dev.alloc<double>((size_t)ncol * g.nEc);
    cgP = dev.alloc<double>((size_t)ncol * g.nEc);
    cgAP = dev.alloc<double>((size_t)ncol * g.nEc);
    cgT = dev.alloc<double>((size_t)ncol * g.nH);
    rhs = dev.alloc<double>((size_t)ncol * g.nEc);
    cg_it = dev.alloc<int>(ncol);
    if (!cgR || !cgP || !cgAP || !cgT || !rhs || !cg_it) return failf(FDTD_E_NOMEM, "CG scratch");
    return FDTD_OK;
  }

  // X (n x ncol, ld n) = (G + s0 C)^{-1} [BE; BH] with BE (nEc x ncol, ld ldbe), BH (nH x ncol, ld ldbh
  // or nullptr: 0): eliminate H (xH = dH o (bH - K^T xE)), CG on the Schur complement for xE.
  fdtd_status solve(const double* BE, int ldbe, const double* BH, int ldbh, int ncol, double* X) {
    if (ncol == 0) return FDTD_OK;
    if (h_form) return solve_h(BE, ldbe, BH, ldbh, ncol, X);
    STCK(ensure_cg(ncol));
    t_solve.start(s);
    const dim3 ge(blocks(g.nEc, 256), ncol), gh(blocks(g.nH, 256), ncol);
    if (BH) k_apply_kernel<<<ge, 256, 0, s>>>(g, col, val, dH, BH, ldbh, BE, ldbe, rhs, g.nEc, ncol);
    else CUCK(cudaMemcpy2DAsync(rhs, (size_t)g.nEc * 8, BE, (size_t)ldbe * 8, (size_t)g.nEc * 8, ncol,
                                cudaMemcpyDeviceToDevice, s));
    CGArgs a{g, col, val, colT, valT, d, dH, minv, rhs, g.nEc, X, n(), cgR, cgP, cgAP, cgT, cg_tol, 200000, cg_it};
    cg_kernel<<<ncol, CG_NT, 0, s>>>(a);
    h_recover_kernel<<<gh, 256, 0, s>>>(g, colT, valT, dH, X, n(), BH, ldbh, X + g.nEc, n(), ncol);
    CUCK(cudaGetLastError());
    std::vector<int> it(ncol);
    CUCK(cudaMemcpyAsync(it.data(), cg_it, sizeof(int) * ncol, cudaMemcpyDeviceToHost, s));
    t_solve.stop(s);
    for (int k = 0; k < ncol; ++k) {
      if (it[k] < 0) return failf(FDTD_E_STATE, "CG did not converge to %.1e (column %d)", cg_tol, k);
      cg_it_max = std::max(cg_it_max, it[k]);
    }
    return FDTD_OK;
  }

  // one-sided Jacobi SVD of A (rows x m, ld lda, overwritten by A V); V (m x m) accumulated if
  // non-null.  sig: column norms afterwards (unsorted).
  // Jacobi sweeps on A (rows x m, ld lda) until no pair rotates; V (m x m) accumulates the
  // rotations (initialised to I when init is set).
  fdtd_status jacobi_sweeps(double* A, int lda, int rows, int m, double* V, bool init, double tol = 0.0,
                             double floor_rel = 1e-15) {
    if (V && init) identity_kernel<<<blocks((long)m * m, 256), 256, 0, s>>>(V, m);
    const int mp = m + (m & 1);
    // converged when every pair is orthogonal to sqrt(m) eps relative (the dgesvj criterion)
    if (tol <= 0) tol = std::max(1e-15, std::sqrt((double)m) * 2.220446049250313e-16);
    int* rot = (int*)scal;
    double floor2 = 0.0;
    {
      double* nrm = dev.alloc<double>(m);
      if (!nrm) return failf(FDTD_E_NOMEM, "jacobi");
      colnorm_kernel<<<m, JB_NT, 0, s>>>(A, lda, rows, nrm);
      std::vector<double> h(m);
      CUCK(cudaMemcpyAsync(h.data(), nrm, sizeof(double) * m, cudaMemcpyDeviceToHost, s));
      CUCK(cudaStreamSynchronize(s));
      const double mx = *std::max_element(h.begin(), h.end());
      floor2 = (floor_rel * mx) * (floor_rel * mx);  // column norms only shrink below the largest
    }
    int sweeps = 0;
    for (; sweeps < 60; ++sweeps) {
      CUCK(cudaMemsetAsync(rot, 0, sizeof(int), s));
      if (coop_grid > 0 && mp > 2) {  // one launch per sweep
        int ldv = m, vrows = m;
        double* Vp = V;
        double tl = tol;
        int mm = m, mpp = mp, ld = lda, rw = rows;
        void* args[] = {&A, &ld, &rw, &mm, &Vp, &ldv, &vrows, &mpp, &tl, &floor2, &rot};
        CUCK(cudaLaunchCooperativeKernel((void*)jacobi_sweep_kernel, dim3(std::min(coop_grid, mp / 2)), dim3(JB_NT),
                                         args, 0, s));
      } else {
        for (int t = 0; t < mp - 1; ++t)
          jacobi_round_kernel<<<mp / 2, JB_NT, 0, s>>>(A, lda, rows, m, V, m, m, mp, t, tol, floor2, rot);
      }
      int h = 0;
      CUCK(cudaMemcpyAsync(&h, rot, sizeof(int), cudaMemcpyDeviceToHost, s));
      CUCK(cudaStreamSynchronize(s));
      if (h == 0) break;
    }
    jac_sweeps_max = std::max(jac_sweeps_max, sweeps + 1);
    if (getenv("FDTD_ROM_VERBOSE")) fprintf(stderr, "jacobi %d x %d: %d sweeps\n", rows, m, sweeps + 1);
    CUCK(cudaGetLastError());
    return FDTD_OK;
  }

  // one-sided Jacobi SVD of A (rows x m, ld lda, overwritten by A V = U S); V (m x m) returned if
  // non-null.  sig: column norms afterwards (unsorted).  Tall A is first rotated by the
  // eigenvectors of its Gram matrix A^T A (itself diagonalised by Jacobi), after which the
  // columns are orthogonal up to the Gram matrix's rounding and few sweeps remain.
  fdtd_status jacobi(double* A, int lda, int rows, int m, double* V, std::vector<double>& sig,
                     double floor_rel = 1e-15) {
    sig.assign(m, 0.0);
    if (m == 0) return FDTD_OK;
    t_svd.start(s);
    if (rows > m && m >= 16) {
      double* G = dev.alloc<double>((size_t)m * m);
      double* Vg = dev.alloc<double>((size_t)m * m);
      double* T = dev.alloc<double>((size_t)rows * m);
      if (!G || !Vg || !T) return failf(FDTD_E_NOMEM, "jacobi preconditioning");
      gemm<true, false>(m, m, rows, A, lda, nullptr, A, lda, G, m);
      STCK(jacobi_sweeps(G, m, m, m, Vg, true, 1e-10, 1e-12));  // a preconditioner: loose
      gemm<false, false>(rows, m, m, A, lda, nullptr, Vg, m, T, rows);
      CUCK(cudaMemcpy2DAsync(A, (size_t)lda * 8, T, (size_t)rows * 8, (size_t)rows * 8, m, cudaMemcpyDeviceToDevice,
                             s));
      if (V) CUCK(cudaMemcpyAsync(V, Vg, sizeof(double) * m * m, cudaMemcpyDeviceToDevice, s));
      STCK(jacobi_sweeps(A, lda, rows, m, V, false, 0.0, floor_rel));
    } else {
      STCK(jacobi_sweeps(A, lda, rows, m, V, true, 0.0, floor_rel));
    }
    double* nrm = dev.alloc<double>(m);
    if (!nrm) return failf(FDTD_E_NOMEM, "jacobi");
    colnorm_kernel<<<m, JB_NT, 0, s>>>(A, lda, rows, nrm);
    CUCK(cudaMemcpyAsync(sig.data(), nrm, sizeof(double) * m, cudaMemcpyDeviceToHost, s));
    t_svd.stop(s);
    CUCK(cudaGetLastError());
    return FDTD_OK;
  }

  // U (rows x k): orthonormal basis of span(A) (rows x m) built column by column in Krylov order
  // (classical Gram-Schmidt twice, Euclidean; a column is deflated when less than 1e-10 of its norm
  // remains) -- romgen._orth_ordered, R10
  fdtd_status orth(const double* A, int lda, int rows, int m, double* U, int ldu, int& k) {
    k = 0;
    double* v = dev.alloc<double>(rows);
    double* h = dev.alloc<double>(std::max(m, 1));
    if (!v || !h) return failf(FDTD_E_NOMEM, "orth");
    double* nrm = scal + 24;
    t_orth.start(s);
    for (int j = 0; j < m; ++j) {
      CUCK(cudaMemcpyAsync(v, A + (size_t)j * lda, sizeof(double) * rows, cudaMemcpyDeviceToDevice, s));
      STCK(cnorm2(nullptr, v, rows, nrm));
      for (int pass = 0; pass < 2 && k > 0; ++pass) {
        STCK(wtcv(U, ldu, nullptr, v, rows, k, h));
        v_minus_wh_kernel<<<blocks(rows, 256), 256, 0, s>>>(U, ldu, h, k, v, rows);
      }
      STCK(cnorm2(nullptr, v, rows, nrm + 1));
      double nn[2];
      CUCK(cudaMemcpyAsync(nn, nrm, sizeof nn, cudaMemcpyDeviceToHost, s));
      CUCK(cudaStreamSynchronize(s));
      const double n0 = std::sqrt(nn[0]), n1 = std::sqrt(nn[1]);
      if (n0 == 0.0 || n1 <= 1e-10 * n0) continue;
      scale_copy_kernel<<<blocks(rows, 256), 256, 0, s>>>(v, 1.0 / n1, U + (size_t)k * ldu, rows);
      ++k;
    }
    t_orth.stop(s);
    CUCK(cudaGetLastError());
    return FDTD_OK;
  }

  // C (M x N) = op(A) diag(w) op(B); a long K is split over enough CTAs to fill the GPU, the
  // partials summed in a fixed order
  double* gemm_part = nullptr;
  size_t gemm_cap = 0;
  template <bool TA, bool TB>
  void gemm(int M, int N, int K, const double* A, int lda, const double* w, const double* B, int ldb, double* C,
            int ldc) {
    const int tiles = (int)(blocks(M, GT) * blocks(N, GT));
    int splits = std::max(1, std::min((K + 4095) / 4096, 296 / std::max(tiles, 1)));
    if (splits > 1 && (size_t)splits * M * N > gemm_cap) {
      gemm_cap = (size_t)splits * M * N;
      gemm_part = dev.alloc<double>(gemm_cap);
      if (!gemm_part) splits = 1;
    }
    if (splits == 1) {
      gemm_kernel<TA, TB><<<dim3(blocks(M, GT), blocks(N, GT), 1), 256, 0, s>>>(M, N, K, A, lda, w, B, ldb, C, ldc, K);
      return;
    }
    const int kchunk = ((K + splits - 1) / splits + GT - 1) / GT * GT;
    splits = (K + kchunk - 1) / kchunk;
    gemm_kernel<TA, TB><<<dim3(blocks(M, GT), blocks(N, GT), splits), 256, 0, s>>>(M, N, K, A, lda, w, B, ldb,
                                                                                 gemm_part, M, kchunk);
    sum_splits_kernel<<<blocks((long)M * N, 256), 256, 0, s>>>(gemm_part, splits, M, N, C, ldc);
  }

  // ||v||_c^2 into out[0] and W[:, :k]^T (c o v) into h, single-CTA for short vectors, two-level
  // (slices of RED_SLICE rows, ordered sum) for long ones; deterministic either way
  double* red_part = nullptr;
  size_t red_cap = 0;
  fdtd_status red_buf(size_t n) {
    if (n <= red_cap) return FDTD_OK;
    red_cap = n;
    red_part = dev.alloc<double>(n);
    return red_part ? FDTD_OK : failf(FDTD_E_NOMEM, "reduction scratch");
  }
  fdtd_status cnorm2(const double* c, const double* v, int n, double* out) {
    const int ng = (n + RED_SLICE - 1) / RED_SLICE;
    if (ng <= 2) {
      cnorm2_kernel<<<1, RN_NT, 0, s>>>(c, v, n, out);
      return FDTD_OK;
    }
    STCK(red_buf(ng));
    cnorm2_part_kernel<<<ng, GV_NT, 0, s>>>(c, v, n, red_part);
    sum_parts_kernel<<<1, 32, 0, s>>>(red_part, ng, 1, out);
    return FDTD_OK;
  }
  fdtd_status wtcv(const double* W, int ldw, const double* c, const double* v, int n, int k, double* h) {
    const int ng = (n + RED_SLICE - 1) / RED_SLICE;
    if (ng <= 2) {
      wtcv_kernel<<<k, GV_NT, 0, s>>>(W, ldw, c, v, n, h);
      return FDTD_OK;
    }
    STCK(red_buf((size_t)ng * k));
    wtcv_part_kernel<<<dim3(k, ng), GV_NT, 0, s>>>(W, ldw, c, v, n, k, red_part);
    sum_parts_kernel<<<blocks(k, 128), 128, 0, s>>>(red_part, ng, k, h);
    return FDTD_OK;
  }

  // SPRIM basis from m Krylov vectors (romgen._sprim_basis_m): V1 (nEc x k1), V2 (nH x k2)
  fdtd_status sprim_m(int m, double* V1, int& k1, double* V2, int& k2, int& used) {
    const int N = n(), nY = g.nY;
    m = std::min(m, N);
    double* W = dev.alloc<double>((size_t)N * m);
    double* blk = dev.alloc<double>((size_t)N * std::max(nY, 1));
    double* v = dev.alloc<double>(N);
    double* h = dev.alloc<double>(std::max(m, 1));
    double* B0 = dev.alloc<double>((size_t)g.nEc * nY);
    if (!W || !blk || !v || !h || !B0) return failf(FDTD_E_NOMEM, "Arnoldi basis (%d x %d)", N, m);
    // B0[k, k] = S_c[k] (B_c = [diag(S_c); 0]); X0 = solve(B0, 0)
    {
      std::vector<double> sc(nY);
      CUCK(cudaMemcpyAsync(sc.data(), Sc, sizeof(double) * nY, cudaMemcpyDeviceToHost, s));
      CUCK(cudaStreamSynchronize(s));
      for (int k = 0; k < nY; ++k)
        CUCK(cudaMemcpyAsync(B0 + (size_t)k * g.nEc + k, &sc[k], sizeof(double), cudaMemcpyHostToDevice, s));
      CUCK(cudaStreamSynchronize(s));
    }
    PhaseLog lg;
    lg.mark(s, " B0");
    STCK(solve(B0, g.nEc, nullptr, 0, nY, blk));
    lg.mark(s, " X0 solve");
    int nb = nY, k = 0;
    double* nrm = scal + 16;
    std::vector<int> acc;
    while (k < m && nb > 0) {
      acc.clear();
      for (int c = 0; c < nb && k < m; ++c) {
        // add(v): CGS2 in the C inner product with deflation 1e-10 (romgen.add)
        t_orth.start(s);
        const double* src = blk + (size_t)c * N;
        STCK(cnorm2(cdiag, src, N, nrm));
        CUCK(cudaMemcpyAsync(v, src, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
        for (int pass = 0; pass < 2 && k > 0; ++pass) {
          STCK(wtcv(W, N, cdiag, v, N, k, h));
          v_minus_wh_kernel<<<blocks(N, 256), 256, 0, s>>>(W, N, h, k, v, N);
        }
        STCK(cnorm2(cdiag, v, N, nrm + 1));
        double nn[2];
        CUCK(cudaMemcpyAsync(nn, nrm, sizeof nn, cudaMemcpyDeviceToHost, s));
        t_orth.stop(s);
        const double n0 = std::sqrt(nn[0]), n1 = std::sqrt(nn[1]);
        if (n0 == 0.0 || n1 <= 1e-10 * n0) continue;
        scale_copy_kernel<<<blocks(N, 256), 256, 0, s>>>(v, 1.0 / n1, W + (size_t)k * N, N);
        acc.push_back(k);
        ++k;
      }
      lg.mark(s, " block GS");
      if (k >= m || acc.empty()) break;
      // next block: solve(R11 o W_E[:, acc], R22 o W_H[:, acc])
      nb = (int)acc.size();
      int* didx = dev.alloc<int>(nb);
      double* bE = dev.alloc<double>((size_t)g.nEc * nb);
      double* bH = dev.alloc<double>((size_t)g.nH * nb);
      if (nb > nY) blk = dev.alloc<double>((size_t)N * nb);
      if (!didx || !bE || !bH || !blk) return failf(FDTD_E_NOMEM, "Arnoldi block");
      CUCK(cudaMemcpyAsync(didx, acc.data(), sizeof(int) * nb, cudaMemcpyHostToDevice, s));
      gather_cols_kernel<<<dim3(blocks(g.nEc, 256), nb), 256, 0, s>>>(W, N, didx, r11, g.nEc, bE, g.nEc, nb);
      gather_cols_kernel<<<dim3(blocks(g.nH, 256), nb), 256, 0, s>>>(W + g.nEc, N, didx, r22, g.nH, bH, g.nH, nb);
      STCK(solve(bE, g.nEc, bH, g.nH, nb, blk));
      lg.mark(s, " block solve");
    }
    used = k;
    // V1, V2: the E and H rows of W orthonormalised in Krylov order
    STCK(orth(W, N, g.nEc, k, V1, g.nEc, k1));
    STCK(orth(W + g.nEc, N, g.nH, k, V2, g.nH, k2));
    lg.mark(s, " orth");
    return FDTD_OK;
  }
};

// symmetric positive definite A (m x m, device): H = A^{1/2}, I = A^{-1/2} via one-sided Jacobi
// (for SPD A the normalised columns of A V are the eigenvectors, the norms the eigenvalues)
fdtd_status spd_sqrt(Builder& b, const double* A, int m, double* H, double* I, const char* name) {
  double* W = b.dev.alloc<double>((size_t)m * m);
  double* U = b.dev.alloc<double>((size_t)m * m);
  double* w = b.dev.alloc<double>(m);
  if (!W || !U || !w) return failf(FDTD_E_NOMEM, "spd_sqrt");
  CUCK(cudaMemcpyAsync(W, A, sizeof(double) * m * m, cudaMemcpyDeviceToDevice, b.s));
  std::vector<double> sg;
  STCK(b.jacobi(W, m, m, m, nullptr, sg));
  std::vector<int> perm(m);
  std::iota(perm.begin(), perm.end(), 0);
  std::stable_sort(perm.begin(), perm.end(), [&](int x, int y) { return sg[x] > sg[y]; });
  if (!(sg[perm[m - 1]] > 1e-14 * sg[perm[0]]))
    return failf(FDTD_E_STATE, "%s is not positive definite (eigenvalue floor)", name);
  std::vector<double> sc(m), ws(m);
  for (int t = 0; t < m; ++t) sc[t] = 1.0 / sg[perm[t]];
  int* dperm = b.dev.alloc<int>(m);
  double* dsc = b.dev.alloc<double>(m);
  if (!dperm || !dsc) return failf(FDTD_E_NOMEM, "spd_sqrt");
  CUCK(cudaMemcpyAsync(dperm, perm.data(), sizeof(int) * m, cudaMemcpyHostToDevice, b.s));
  CUCK(cudaMemcpyAsync(dsc, sc.data(), sizeof(double) * m, cudaMemcpyHostToDevice, b.s));
  permute_scale_kernel<<<dim3(blocks(m, 256), m), 256, 0, b.s>>>(W, m, dperm, dsc, m, U, m, m);
  for (int t = 0; t < m; ++t) ws[t] = std::sqrt(sg[perm[t]]);
  CUCK(cudaMemcpyAsync(w, ws.data(), sizeof(double) * m, cudaMemcpyHostToDevice, b.s));
  b.gemm<false, true>(m, m, m, U, m, w, U, m, H, m);  // U diag(sqrt s) U^T
  for (int t = 0; t < m; ++t) ws[t] = 1.0 / std::sqrt(sg[perm[t]]);
  double* w2 = b.dev.alloc<double>(m);
  if (!w2) return failf(FDTD_E_NOMEM, "spd_sqrt");
  CUCK(cudaMemcpyAsync(w2, ws.data(), sizeof(double) * m, cudaMemcpyHostToDevice, b.s));
  b.gemm<false, true>(m, m, m, U, m, w2, U, m, I, m);
  CUCK(cudaGetLastError());
  return FDTD_OK;
}

fdtd_status build(const fdtd_rom_spec* sp, fdtd_rom_built* out) {
  if (!sp || !out || !sp->eps_r || !sp->sigma || sp->bx < 1 || sp->by < 1 || sp->r < 1 || sp->q < 2 ||
      !(sp->dx > 0) || !(sp->dy > 0) || !(sp->fmax > 0))
    return failf(FDTD_E_ARG, "invalid ROM spec");
  // the stream outlives the builder (its buffers are freed on it, then it is synchronised)
  struct StreamGuard {
    cudaStream_t s = nullptr;
    ~StreamGuard() { if (s) { cudaStreamSynchronize(s); cudaStreamDestroy(s); } }
  } sg;
  CUCK(cudaStreamCreateWithFlags(&sg.s, cudaStreamNonBlocking));
  keep_pool_memory();
  Builder b;
  b.s = sg.s;
  b.dev.s = sg.s;
  Geo& g = b.g;
  g.bx = sp->bx; g.by = sp->by; g.r = sp->r;
  g.Nx = g.bx * g.r; g.Ny = g.by * g.r;
  g.fdx = sp->dx / g.r; g.fdy = sp->dy / g.r;
  if (sp->literal) {  // NEXT-1 port set: every fine boundary node is a port (Geo's port math with
                      // Nx x Ny "coarse edges" of one fine node each)
    g.bx = g.Nx; g.by = g.Ny; g.r = 1;
  }
  g.nY = 2 * g.bx + 2 * g.by;
  g.nEc = g.nY + (g.Ny - 1) * g.Nx + g.Ny * (g.Nx - 1);
  g.nH = g.Nx * g.Ny;
  const size_t ncell = (size_t)g.Nx * g.Ny;
  for (size_t i = 0; i < ncell; ++i)
    if (!(sp->eps_r[i] > 0) || !std::isfinite(sp->eps_r[i]) || !std::isfinite(sp->sigma[i]) || sp->sigma[i] < 0)
      return failf(FDTD_E_ARG, "fine cell %zu: eps_r must be positive and finite, sigma finite and >= 0", i);
  b.s0 = PI * sp->fmax;
  b.cg_tol = sp->cg_tol > 0 ? sp->cg_tol : 1e-13;
  Timer t_all;
  t_all.start(b.s);
  const int nnz = g.nY * g.r + 2 * (g.nEc - g.nY);
  double* eps = b.dev.alloc<double>(ncell);
  double* sig = b.dev.alloc<double>(ncell);
  b.r11 = b.dev.alloc<double>(g.nEc); b.f11 = b.dev.alloc<double>(g.nEc); b.r22 = b.dev.alloc<double>(g.nH);
  b.Sc = b.dev.alloc<double>(g.nY); b.cdiag = b.dev.alloc<double>(g.nEc + g.nH);
  b.col = b.dev.alloc<int>(nnz); b.val = b.dev.alloc<double>(nnz);
  b.colT = b.dev.alloc<int>(4 * (size_t)g.nH); b.valT = b.dev.alloc<double>(4 * (size_t)g.nH);
  b.d = b.dev.alloc<double>(g.nEc); b.dH = b.dev.alloc<double>(g.nH); b.minv = b.dev.alloc<double>(g.nEc);
  b.scal = b.dev.alloc<double>(64);
  if (!eps || !sig || !b.r11 || !b.f11 || !b.r22 || !b.Sc || !b.cdiag || !b.col || !b.val || !b.colT || !b.valT ||
      !b.d || !b.dH || !b.minv || !b.scal)
    return failf(FDTD_E_NOMEM, "assembly buffers");
  CUCK(cudaMemcpyAsync(eps, sp->eps_r, sizeof(double) * ncell, cudaMemcpyHostToDevice, b.s));
  CUCK(cudaMemcpyAsync(sig, sp->sigma, sizeof(double) * ncell, cudaMemcpyHostToDevice, b.s));
  assemble_e_kernel<<<blocks(g.nEc, 256), 256, 0, b.s>>>(g, eps, sig, b.r11, b.f11, b.col, b.val, b.Sc);
  assemble_h_kernel<<<blocks(g.nH, 256), 256, 0, b.s>>>(g, b.r22, b.colT, b.valT);
  schur_diag_kernel<<<blocks(std::max(g.nEc, g.nH), 256), 256, 0, b.s>>>(g, b.s0, b.r11, b.f11, b.r22, b.col, b.val,
                                                                          b.d, b.dH, b.minv);
  {  // FDTD_ROM_SOLVER=e: the E-form (Jacobi-preconditioned CG on the E-node Schur complement)
    const char* sv = getenv("FDTD_ROM_SOLVER");
    b.h_form = !(sv && sv[0] == 'e');
  }
  PhaseLog plog;
  plog.mark(b.s, "assembly");
  if (b.h_form) STCK(b.setup_mg());
  plog.mark(b.s, "multigrid");
  b.setup_coop();
  CUCK(cudaMemcpyAsync(b.cdiag, b.r11, sizeof(double) * g.nEc, cudaMemcpyDeviceToDevice, b.s));
  CUCK(cudaMemcpyAsync(b.cdiag + g.nEc, b.r22, sizeof(double) * g.nH, cudaMemcpyDeviceToDevice, b.s));
  CUCK(cudaGetLastError());

  // SPRIM with q1 = ceil(q/2), q2 = floor(q/2); m grows until both parts reach their share
  // (romgen.sprim_basis)
  const int q1w = (sp->q + 1) / 2, q2w = sp->q / 2;
  double *V1 = nullptr, *V2 = nullptr;
  int m = q1w, k1 = 0, k2 = 0, used = 0;
  for (int rep = 0; rep < 8; ++rep) {
    const int mm = std::min(m, g.nEc + g.nH);
    V1 = b.dev.alloc<double>((size_t)g.nEc * mm);
    V2 = b.dev.alloc<double>((size_t)g.nH * mm);
    if (!V1 || !V2) return failf(FDTD_E_NOMEM, "basis");
    STCK(b.sprim_m(m, V1, k1, V2, k2, used));
    if ((k1 >= q1w && k2 >= q2w) || m >= g.nEc + g.nH) break;
    m = (int)(m + std::max({q1w - k1, q2w - k2, 1}) * 1.5);
  }
  int q1 = std::min(k1, q1w);
  const int q2 = std::min(k2, q2w);
  if (q1 < 1 || q2 < 1) return failf(FDTD_E_STATE, "empty basis (q1 %d, q2 %d)", q1, q2);
  if (sp->literal) {  // the E basis must span the nP port directions (A1 regular, R9):
                      // [P | V1] orthonormalised in order, the first nP + ceil(q/2) kept
    const int nP = g.nY, mc = nP + q1;
    double* PV = b.dev.alloc<double>((size_t)g.nEc * mc);
    double* VL = b.dev.alloc<double>((size_t)g.nEc * mc);
    if (!PV || !VL) return failf(FDTD_E_NOMEM, "literal basis");
    std::vector<double> one(1, 1.0);
    for (int k = 0; k < nP; ++k)
      CUCK(cudaMemcpyAsync(PV + (size_t)k * g.nEc + k, one.data(), sizeof(double), cudaMemcpyHostToDevice, b.s));
    CUCK(cudaMemcpy2DAsync(PV + (size_t)nP * g.nEc, (size_t)g.nEc * 8, V1, (size_t)g.nEc * 8, (size_t)g.nEc * 8, q1,
                           cudaMemcpyDeviceToDevice, b.s));
    int kl = 0;
    STCK(b.orth(PV, g.nEc, g.nEc, mc, VL, g.nEc, kl));
    V1 = VL;
    q1 = std::min(kl, nP + q1w);
  }

  plog.mark(b.s, "sprim");
  // congruence (eq:R11_tilde .. eq:K_tilde)
  double* R11 = b.dev.alloc<double>((size_t)q1 * q1);
  double* F11 = b.dev.alloc<double>((size_t)q1 * q1);
  double* R22 = b.dev.alloc<double>((size_t)q2 * q2);
  double* Kt = b.dev.alloc<double>((size_t)q1 * q2);
  double* KV2 = b.dev.alloc<double>((size_t)g.nEc * q2);
  if (!R11 || !F11 || !R22 || !Kt || !KV2) return failf(FDTD_E_NOMEM, "reduced matrices");
  b.gemm<true, false>(q1, q1, g.nEc, V1, g.nEc, b.r11, V1, g.nEc, R11, q1);
  b.gemm<true, false>(q1, q1, g.nEc, V1, g.nEc, b.f11, V1, g.nEc, F11, q1);
  b.gemm<true, false>(q2, q2, g.nH, V2, g.nH, b.r22, V2, g.nH, R22, q2);
  k_apply_kernel<<<dim3(blocks(g.nEc, 256), q2), 256, 0, b.s>>>(g, b.col, b.val, nullptr, V2, g.nH, nullptr, 0, KV2,
                                                                 g.nEc, q2);
  b.gemm<true, false>(q1, q2, g.nEc, V1, g.nEc, nullptr, KV2, g.nEc, Kt, q1);
  CUCK(cudaGetLastError());

  plog.mark(b.s, "congruence");
  // CFL: singular values of R11^-1/2 K R22^-1/2 (eq:CFLgeneralized), optional clip
  double *h1 = b.dev.alloc<double>((size_t)q1 * q1), *i1 = b.dev.alloc<double>((size_t)q1 * q1);
  double *h2 = b.dev.alloc<double>((size_t)q2 * q2), *i2 = b.dev.alloc<double>((size_t)q2 * q2);
  double *T1 = b.dev.alloc<double>((size_t)q1 * q2), *X = b.dev.alloc<double>((size_t)q1 * q2);
  double* Vx = b.dev.alloc<double>((size_t)q2 * q2);
  if (!h1 || !i1 || !h2 || !i2 || !T1 || !X || !Vx) return failf(FDTD_E_NOMEM, "CFL buffers");
  // symmetrise first (exact symmetry of the congruences, as romgen): A <- (A + A^T) / 2 on the host
  auto sym_host = [&](double* dA, int mdim, std::vector<double>& hA) -> fdtd_status {
    hA.resize((size_t)mdim * mdim);
    CUCK(cudaMemcpyAsync(hA.data(), dA, sizeof(double) * mdim * mdim, cudaMemcpyDeviceToHost, b.s));
    CUCK(cudaStreamSynchronize(b.s));
    for (int i = 0; i < mdim; ++i)
      for (int j = 0; j < i; ++j) {
        const double v = 0.5 * (hA[(size_t)i * mdim + j] + hA[(size_t)j * mdim + i]);
        hA[(size_t)i * mdim + j] = hA[(size_t)j * mdim + i] = v;
      }
    CUCK(cudaMemcpyAsync(dA, hA.data(), sizeof(double) * mdim * mdim, cudaMemcpyHostToDevice, b.s));
    CUCK(cudaStreamSynchronize(b.s));
    return FDTD_OK;
  };
  std::vector<double> hR11, hR22, hF11;
  STCK(sym_host(R11, q1, hR11));
  STCK(sym_host(R22, q2, hR22));
  STCK(sym_host(F11, q1, hF11));
  STCK(spd_sqrt(b, R11, q1, h1, i1, "R~11"));
  STCK(spd_sqrt(b, R22, q2, h2, i2, "R~22"));
  b.gemm<false, false>(q1, q2, q1, i1, q1, nullptr, Kt, q1, T1, q1);
  b.gemm<false, false>(q1, q2, q2, T1, q1, nullptr, i2, q2, X, q1);
  std::vector<double> sv;
  STCK(b.jacobi(X, q1, q1, q2, Vx, sv));  // X Vx = U S (columns of X now U S)
  std::vector<int> perm(q2);
  std::iota(perm.begin(), perm.end(), 0);
  std::stable_sort(perm.begin(), perm.end(), [&](int x, int y) { return sv[x] > sv[y]; });
  const double smax = sv[perm[0]];
  out->natural_dt_limit = smax > 0 ? 2.0 / smax : INFINITY;
  out->n_clipped = 0;
  if (sp->dt_target > 0) {
    const double cap = (2.0 / sp->dt_target) * (1.0 - 1e-6);
    int nclip = 0;
    for (double v : sv) nclip += v > cap;
    out->n_clipped = nclip;
    if (nclip) {
      // K~ = h1 U diag(min(s, cap)) Vx^T h2, with U S = X: scale column t of X by min(s_t, cap) / s_t
      std::vector<double> f(q2);
      for (int t = 0; t < q2; ++t) f[t] = sv[t] > 0 ? std::min(sv[t], cap) / sv[t] : 0.0;
      double* df = b.dev.alloc<double>(q2);
      int* id = b.dev.alloc<int>(q2);
      double* Y = b.dev.alloc<double>((size_t)q1 * q2);
      if (!df || !id || !Y) return failf(FDTD_E_NOMEM, "clip");
      std::vector<int> idn(q2);
      std::iota(idn.begin(), idn.end(), 0);
      CUCK(cudaMemcpyAsync(df, f.data(), sizeof(double) * q2, cudaMemcpyHostToDevice, b.s));
      CUCK(cudaMemcpyAsync(id, idn.data(), sizeof(int) * q2, cudaMemcpyHostToDevice, b.s));
      permute_scale_kernel<<<dim3(blocks(q1, 256), q2), 256, 0, b.s>>>(X, q1, id, df, q1, Y, q1, q2);
      b.gemm<false, true>(q1, q2, q2, Y, q1, nullptr, Vx, q2, T1, q1);  // U S' Vx^T
      b.gemm<false, false>(q1, q2, q1, h1, q1, nullptr, T1, q1, X, q1);
      b.gemm<false, false>(q1, q2, q2, X, q1, nullptr, h2, q2, Kt, q1);
      CUCK(cudaGetLastError());
    }
  }

  plog.mark(b.s, "cfl");
  // outputs (row-major)
  std::vector<double> hK((size_t)q1 * q2), hV1p((size_t)g.nY * q1);
  CUCK(cudaMemcpyAsync(hK.data(), Kt, sizeof(double) * q1 * q2, cudaMemcpyDeviceToHost, b.s));
  CUCK(cudaMemcpy2DAsync(hV1p.data(), (size_t)g.nY * 8, V1, (size_t)g.nEc * 8, (size_t)g.nY * 8, q1,
                         cudaMemcpyDeviceToHost, b.s));
  t_all.stop(b.s);
  for (int i = 0; i < q1; ++i)
    for (int j = 0; j < q1; ++j) {
      out->R11[(size_t)i * q1 + j] = hR11[(size_t)j * q1 + i];
      out->F11[(size_t)i * q1 + j] = hF11[(size_t)j * q1 + i];
    }
  for (int i = 0; i < q2; ++i)
    for (int j = 0; j < q2; ++j) out->R22[(size_t)i * q2 + j] = hR22[(size_t)j * q2 + i];
  for (int i = 0; i < q1; ++i)
    for (int j = 0; j < q2; ++j) out->K[(size_t)i * q2 + j] = hK[(size_t)j * q1 + i];
  for (int i = 0; i < q1; ++i)  // L~ = V1^T L_c = the port rows of V1, transposed: L[i][k] = V1[k][i]
    for (int k = 0; k < g.nY; ++k) out->L[(size_t)i * g.nY + k] = hV1p[(size_t)i * g.nY + k];
  out->q1 = q1; out->q2 = q2; out->nY = g.nY;
  out->krylov_vectors = used;
  out->cg_iterations_max = b.cg_it_max;
  out->jacobi_sweeps_max = b.jac_sweeps_max;
  out->ms_total = t_all.ms; out->ms_solve = b.t_solve.ms; out->ms_orth = b.t_orth.ms; out->ms_svd = b.t_svd.ms;
  return FDTD_OK;
}

}  // namespace

extern "C" fdtd_status fdtd_rom_build(const fdtd_rom_spec* spec, fdtd_rom_built* out) {
  g_err.clear();
  return build(spec, out);
}

extern "C" const char* fdtd_rom_build_last_error(void) { return g_err.c_str(); }
