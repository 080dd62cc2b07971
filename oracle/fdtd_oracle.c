/*
 * oracle/fdtd_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct fp64 CPU implementation of the hot path of
 * Zhang, Bekmambetova, Triverio, "A Stable FDTD Method with Embedded
 * Reduced-Order Models" (arXiv 1609.07114).  Only tests/, __graft_entry__.smoke()
 * and bench.py (cpu_baseline / --impl reference) may load this file.  It shares
 * no code, header, table or constant generator with the CUDA path
 * (paper_1609_07114_b200/), and the CUDA path never calls it.
 *
 * What it computes, in the paper's order (citations are PAPER.md lines):
 *   - coarse H half-step, eq:updateH (L267-273), at coarse resolution;
 *   - soft Hz source (excitation L838, L882; reading R15);
 *   - storage function W^n (paper silent; eq:R L323-330, reading R17);
 *   - per ROM: eq:sysform (L632-664) solved every step with an LU of A1
 *     (L674 "A sparse LU factorization can be performed on A1"), in the
 *     collapsed reading (R9: T -> I, 1/r -> 1);
 *   - coarse E half-step, eq:updateEx (L209-214) and its Ey analogue (L223),
 *     written with the coefficients exactly as printed (no ca/cb folding);
 *   - scatter of y^{n+1} into the interface edges (eq:yandxt L627-630).
 * Plus a direct subgridding reference (no matrices at all) used only to pin
 * the coupled ROM path at full order (DESIGN.md pin P-SUBGRID).
 *
 * Conventions (R1): cells (i,j) 0-based, i along x; arrays row-major
 * with j slow: Hz[ny][nx], Ex[ny+1][nx], Ey[ny][nx+1].  PEC outer walls.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define O_C0 299792458.0
#define O_MU0 (4.0e-7 * 3.14159265358979323846)
#define O_EPS0 (1.0 / (O_MU0 * O_C0 * O_C0))

/* edge / cell kinds */
enum { K_NORMAL = 0, K_PEC = 1, K_HOLE = 2, K_IFACE = 3 };

typedef struct {
  int i0, j0, bx, by, q1, q2, nY, q, nz;
  int r, nU, xoff;                 /* hanging variables: nU = nY (collapsed) or r nY (literal); xt at z[xoff] */
  double *R11, *R22, *F11, *K, *L; /* row-major copies, L is q1 x nU */
  double *A1;                      /* LU factors of A1 (nz x nz), row-major */
  int *piv;
  double *A2;                      /* dense nz x nz */
  double *z;                       /* [y (nY); U or u^ (nU); xt (q)], length nz */
  double *DlG;                     /* D_l G per port */
  double *eps_half;                /* D_l D_l' eps (coarse half cell) per port */
  int *port_is_ey;                 /* 0: Ex edge, 1: Ey edge */
  int *port_edge;                  /* flat index into Ex or Ey */
  int *port_h;                     /* flat index of outside coarse Hz */
} orom;

typedef struct {
  int nx, ny;
  double dx, dy, dt;
  double *eps_r, *sigma;  /* per coarse cell */
  double *Ex, *Ey, *Hz, *Hold;
  unsigned char *kx, *ky, *kc; /* kinds of Ex edges, Ey edges, Hz cells */
  int nrom;
  orom *roms;
  int src_i, src_j, src_j1;  /* soft Hz source on cells (src_i, src_j .. src_j1-1) */
  double *src;
  int64_t nsrc, src_t0;
  int nprobe;
  int *probe;  /* flat Hz index */
  int64_t n;   /* steps taken */
  /* direct subgridding regions (reference only, pin P-SUBGRID) */
  int nsub;
  struct osub_s *subs;
  /* CPML on the two x-ends (NEXT-2): width w cells each side; per column coefficients and the
   * auxiliary fields psi_hz (Hz cells) and psi_ey (Ey edges); 0 outside the layers */
  int pml_w;
  double *pml_bh, *pml_ah;   /* per Hz column i: b, a of the recursive convolution */
  double *pml_be, *pml_ae;   /* per Ey column i (nx + 1) */
  double *psi_hz, *psi_ey;
} osim;

/* A finely meshed region marched directly (no matrices): fine Yee cells of
 * size dx/r x dy/r inside the block, with the r fine boundary E nodes of each
 * coarse interface edge tied to that edge (eq:equalE, collapsed). */
typedef struct osub_s {
  int i0, j0, bx, by, r, Nx, Ny;
  double *eps_r, *sigma;       /* per fine cell [Ny][Nx] */
  double *Ex, *Ey, *Hz;        /* fine fields [(Ny+1)][Nx], [Ny][Nx+1], [Ny][Nx] */
} osub;

/* ------------------------------------------------------------------ */
/* dense LU with partial pivoting (plain Doolittle, row-major)          */
/* ------------------------------------------------------------------ */
static int lu_factor(double *A, int n, int *piv) {
  for (int k = 0; k < n; ++k) {
    int p = k;
    double best = fabs(A[(size_t)k * n + k]);
    for (int i = k + 1; i < n; ++i) {
      double v = fabs(A[(size_t)i * n + k]);
      if (v > best) { best = v; p = i; }
    }
    piv[k] = p;
    if (best == 0.0) return -1;
    if (p != k)
      for (int c = 0; c < n; ++c) {
        double t = A[(size_t)k * n + c];
        A[(size_t)k * n + c] = A[(size_t)p * n + c];
        A[(size_t)p * n + c] = t;
      }
    for (int i = k + 1; i < n; ++i) {
      double f = A[(size_t)i * n + k] / A[(size_t)k * n + k];
      A[(size_t)i * n + k] = f;
      for (int c = k + 1; c < n; ++c) A[(size_t)i * n + c] -= f * A[(size_t)k * n + c];
    }
  }
  return 0;
}

static void lu_solve(const double *LU, int n, const int *piv, double *b) {
  for (int k = 0; k < n; ++k)
    if (piv[k] != k) { double t = b[k]; b[k] = b[piv[k]]; b[piv[k]] = t; }
  for (int i = 0; i < n; ++i) {
    double s = b[i];
    for (int c = 0; c < i; ++c) s -= LU[(size_t)i * n + c] * b[c];
    b[i] = s;
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = b[i];
    for (int c = i + 1; c < n; ++c) s -= LU[(size_t)i * n + c] * b[c];
    b[i] = s / LU[(size_t)i * n + i];
  }
}

/* ------------------------------------------------------------------ */
/* indexing                                                            */
/* ------------------------------------------------------------------ */
#define HZ(s, i, j) ((s)->Hz[(size_t)(j) * (s)->nx + (i)])
#define EX(s, i, j) ((s)->Ex[(size_t)(j) * (s)->nx + (i)])
#define EY(s, i, j) ((s)->Ey[(size_t)(j) * ((s)->nx + 1) + (i)])
#define CELL(s, a, i, j) ((s)->a[(size_t)(j) * (s)->nx + (i)])

osim *osim_create(int nx, int ny, double dx, double dy, double dt, const double *eps_r,
                  const double *sigma) {
  if (nx < 1 || ny < 1 || !(dx > 0) || !(dy > 0) || !(dt > 0)) return NULL;
  osim *s = (osim *)calloc(1, sizeof(osim));
  s->nx = nx; s->ny = ny; s->dx = dx; s->dy = dy; s->dt = dt;
  size_t nc = (size_t)nx * ny, nex = (size_t)nx * (ny + 1), ney = (size_t)(nx + 1) * ny;
  s->eps_r = (double *)malloc(nc * sizeof(double));
  s->sigma = (double *)malloc(nc * sizeof(double));
  memcpy(s->eps_r, eps_r, nc * sizeof(double));
  memcpy(s->sigma, sigma, nc * sizeof(double));
  s->Ex = (double *)calloc(nex, sizeof(double));
  s->Ey = (double *)calloc(ney, sizeof(double));
  s->Hz = (double *)calloc(nc, sizeof(double));
  s->Hold = (double *)calloc(nc, sizeof(double));
  s->kx = (unsigned char *)calloc(nex, 1);
  s->ky = (unsigned char *)calloc(ney, 1);
  s->kc = (unsigned char *)calloc(nc, 1);
  /* PEC outer walls: tangential E on the boundary is zero (R1). */
  for (int i = 0; i < nx; ++i) { s->kx[i] = K_PEC; s->kx[(size_t)ny * nx + i] = K_PEC; }
  for (int j = 0; j < ny; ++j) {
    s->ky[(size_t)j * (nx + 1)] = K_PEC;
    s->ky[(size_t)j * (nx + 1) + nx] = K_PEC;
  }
  s->src_i = -1;
  return s;
}

/* ------------------------------------------------------------------ */
/* CPML (NEXT-2; Roden & Gedney's recursive-convolution PML, kappa = 1, */
/* alpha = 0) on the cells i < w and i >= nx - w, backed by the PEC     */
/* walls.  Depth d in [0, 1] from the layer's inner face; sigma(d) =    */
/* sigma_max d^m, sigma_max = (m + 1) ln(1/R0) / (2 eta0 w dx).  Per    */
/* step: b = exp(-sigma dt / eps0), a = b - 1;                          */
/*   psi_hz = b psi_hz + a (Ey_{i+1} - Ey_i)/dx,  Hz -= dt/mu0 psi_hz;  */
/*   psi_ey = b psi_ey + a (Hz_i - Hz_{i-1})/dx,                        */
/*   Ey: the curl term -(dHz/dx) becomes -(dHz/dx + psi_ey).            */
/* ------------------------------------------------------------------ */
static double pml_sigma(int w, int order, double r0, double dx, double d) {
  const double eta0 = sqrt(O_MU0 / O_EPS0);
  const double smax = (order + 1) * log(1.0 / r0) / (2.0 * eta0 * w * dx);
  return d <= 0.0 ? 0.0 : smax * pow(d, order);
}

int osim_set_pml(osim *s, int w, int order, double r0) {
  const int nx = s->nx;
  if (w < 0 || 2 * w > nx || order < 0 || !(r0 > 0 && r0 < 1)) return -1;
  free(s->pml_bh); free(s->pml_ah); free(s->pml_be); free(s->pml_ae); free(s->psi_hz); free(s->psi_ey);
  s->pml_w = w;
  s->pml_bh = (double *)calloc(nx, sizeof(double));
  s->pml_ah = (double *)calloc(nx, sizeof(double));
  s->pml_be = (double *)calloc(nx + 1, sizeof(double));
  s->pml_ae = (double *)calloc(nx + 1, sizeof(double));
  s->psi_hz = (double *)calloc((size_t)nx * s->ny, sizeof(double));
  s->psi_ey = (double *)calloc((size_t)(nx + 1) * s->ny, sizeof(double));
  for (int i = 0; i < nx; ++i) {  /* Hz at x = (i + 1/2) dx */
    double d = 0.0;
    if (i < w) d = (w - i - 0.5) / w;
    else if (i >= nx - w) d = (i + 0.5 - (nx - w)) / w;
    const double b = exp(-pml_sigma(w, order, r0, s->dx, d) * s->dt / O_EPS0);
    s->pml_bh[i] = b; s->pml_ah[i] = b - 1.0;
  }
  for (int i = 0; i <= nx; ++i) {  /* Ey at x = i dx */
    double d = 0.0;
    if (i < w) d = (double)(w - i) / w;
    else if (i > nx - w) d = (double)(i - (nx - w)) / w;
    const double b = exp(-pml_sigma(w, order, r0, s->dx, d) * s->dt / O_EPS0);
    s->pml_be[i] = b; s->pml_ae[i] = b - 1.0;
  }
  return 0;
}

/* CPML state accessors (row-slab tests exchange psi rows): psi_hz ny x nx, psi_ey ny x (nx + 1);
   returns -1 without layers.  State only, no arithmetic. */
int osim_get_psi(const osim *s, double *psi_hz, double *psi_ey) {
  if (s->pml_w <= 0) return -1;
  memcpy(psi_hz, s->psi_hz, sizeof(double) * (size_t)s->nx * s->ny);
  memcpy(psi_ey, s->psi_ey, sizeof(double) * (size_t)(s->nx + 1) * s->ny);
  return 0;
}
int osim_set_psi(osim *s, const double *psi_hz, const double *psi_ey) {
  if (s->pml_w <= 0) return -1;
  memcpy(s->psi_hz, psi_hz, sizeof(double) * (size_t)s->nx * s->ny);
  memcpy(s->psi_ey, psi_ey, sizeof(double) * (size_t)(s->nx + 1) * s->ny);
  return 0;
}

static int in_pml_col(const osim *s, int i) { return s->pml_w > 0 && (i < s->pml_w || i >= s->nx - s->pml_w); }

void osim_destroy(osim *s) {
  if (!s) return;
  for (int r = 0; r < s->nrom; ++r) {
    orom *m = &s->roms[r];
    free(m->R11); free(m->R22); free(m->F11); free(m->K); free(m->L);
    free(m->A1); free(m->piv); free(m->A2); free(m->z); free(m->DlG); free(m->eps_half);
    free(m->port_is_ey); free(m->port_edge); free(m->port_h);
  }
  free(s->roms);
  for (int r = 0; r < s->nsub; ++r) {
    osub *g = &s->subs[r];
    free(g->eps_r); free(g->sigma); free(g->Ex); free(g->Ey); free(g->Hz);
  }
  free(s->subs);
  free(s->eps_r); free(s->sigma); free(s->Ex); free(s->Ey); free(s->Hz); free(s->Hold);
  free(s->kx); free(s->ky); free(s->kc); free(s->src); free(s->probe);
  free(s->pml_bh); free(s->pml_ah); free(s->pml_be); free(s->pml_ae); free(s->psi_hz); free(s->psi_ey);
  free(s);
}

/* ------------------------------------------------------------------ */
/* Embedded ROM (collapsed reading of Sec. IV, R9)           */
/*                                                                     */
/* Ports, in order S (bx), N (bx), W (by), E (by):      */
/*   S k: Ex[j0][i0+k],    outside cell (i0+k, j0-1),  G = -1          */
/*   N k: Ex[j0+by][i0+k], outside cell (i0+k, j0+by), G = +1          */
/*   W k: Ey[j0+k][i0],    outside cell (i0-1, j0+k),  G = +1          */
/*   E k: Ey[j0+k][i0+bx], outside cell (i0+bx, j0+k), G = -1          */
/* eq:updateExboundary (L461-468): the coarse half cell outside the    */
/* block supplies eps, sigma; D_l = dx (Ex) / dy (Ey); D_l' = dy/2 or  */
/* dx/2 (L603).  G signs: DESIGN.md R5.                                */
/* ------------------------------------------------------------------ */
int osim_add_rom(osim *s, int i0, int j0, int bx, int by, int q1, int q2, const double *R11,
                 const double *R22, const double *F11, const double *K, const double *L, int r, int literal) {
  if (bx < 1 || by < 1 || q1 < 1 || q2 < 0 || r < 1) return -1;
  if (i0 < 1 || j0 < 1 || i0 + bx > s->nx - 1 || j0 + by > s->ny - 1) return -2;
  /* footprint + ring must not touch another block */
  for (int j = j0 - 1; j <= j0 + by; ++j)
    for (int i = i0 - 1; i <= i0 + bx; ++i)
      if (CELL(s, kc, i, j) != K_NORMAL) return -3;
  s->roms = (orom *)realloc(s->roms, (size_t)(s->nrom + 1) * sizeof(orom));
  orom *m = &s->roms[s->nrom];
  memset(m, 0, sizeof(*m));
  m->i0 = i0; m->j0 = j0; m->bx = bx; m->by = by; m->q1 = q1; m->q2 = q2;
  int nY = 2 * bx + 2 * by, q = q1 + q2;
  /* literal (the paper's own Sec. IV, NEXT-1): nU = r nY fine hanging variables u^ tied to the
   * coarse edges by T (eq:equalE: fine port k sits on coarse port k / r, the side order being
   * the same) and averaged by 1/r T^T (eq:averH).  Collapsed (R9): T -> I, 1/r -> 1. */
  int nU = literal ? r * nY : nY, nz = nY + nU + q;
  m->nY = nY; m->q = q; m->nz = nz; m->r = literal ? r : 1; m->nU = nU; m->xoff = nY + nU;
  const int X = nY + nU;
#define DUP(dst, src, cnt)                                      \
  do {                                                          \
    dst = (double *)malloc((size_t)(cnt) * sizeof(double) + 8); \
    memcpy(dst, src, (size_t)(cnt) * sizeof(double));           \
  } while (0)
  DUP(m->R11, R11, q1 * q1);
  DUP(m->R22, R22, q2 * q2);
  DUP(m->F11, F11, q1 * q1);
  DUP(m->K, K, q1 * q2);
  DUP(m->L, L, q1 * nU);
#undef DUP
  m->DlG = (double *)calloc(nY, sizeof(double));
  m->eps_half = (double *)calloc(nY, sizeof(double));
  m->port_is_ey = (int *)calloc(nY, sizeof(int));
  m->port_edge = (int *)calloc(nY, sizeof(int));
  m->port_h = (int *)calloc(nY, sizeof(int));
  double *c = (double *)calloc(nY, sizeof(double)), *a = (double *)calloc(nY, sizeof(double));
  const double dx = s->dx, dy = s->dy, dt = s->dt;
  const int nx = s->nx;
  for (int p = 0; p < nY; ++p) {
    int side, k, oi, oj, isey, edge;
    double Dl, Dlp, G;
    if (p < bx) { side = 0; k = p; }
    else if (p < 2 * bx) { side = 1; k = p - bx; }
    else if (p < 2 * bx + by) { side = 2; k = p - 2 * bx; }
    else { side = 3; k = p - 2 * bx - by; }
    switch (side) {
      case 0: oi = i0 + k; oj = j0 - 1; isey = 0; edge = j0 * nx + i0 + k; G = -1; break;
      case 1: oi = i0 + k; oj = j0 + by; isey = 0; edge = (j0 + by) * nx + i0 + k; G = +1; break;
      case 2: oi = i0 - 1; oj = j0 + k; isey = 1; edge = (j0 + k) * (nx + 1) + i0; G = +1; break;
      default: oi = i0 + bx; oj = j0 + k; isey = 1; edge = (j0 + k) * (nx + 1) + i0 + bx; G = -1; break;
    }
    Dl = isey ? dy : dx;
    Dlp = isey ? dx / 2 : dy / 2;
    double eps = O_EPS0 * CELL(s, eps_r, oi, oj), sig = CELL(s, sigma, oi, oj);
    c[p] = Dl * Dlp * (eps / dt + sig / 2);
    a[p] = Dl * Dlp * (eps / dt - sig / 2);
    m->DlG[p] = Dl * G;
    m->eps_half[p] = Dl * Dlp * eps;
    m->port_is_ey[p] = isey;
    m->port_edge[p] = edge;
    m->port_h[p] = oj * nx + oi;
  }
  /* A1 and A2 of eq:sysform (L649-664).
   * z = [y (nY); u (nU); xt (q)], xt = [E~ (q1); H~ (q2)].
   * R~ + F~ = [[R11/dt + F11, -K], [0, R22/dt]]       (eq:R, eq:F_f, L416-425)
   * R~ - F~ = [[R11/dt - F11, 0], [-K^T, R22/dt]]
   * B~ = L~ S, S = diag(-dx (S), +dx (N), +dy (W), -dy (E)) per coarse port (collapsed) or the
   * same divided by r per fine port (literal)  (eq:B, eq:cond3rom, eq:S) */
  const int rr = m->r;
  double *A1 = (double *)calloc((size_t)nz * nz, sizeof(double));
  double *A2 = (double *)calloc((size_t)nz * nz, sizeof(double));
#define A1_(r_, cc) A1[(size_t)(r_) * nz + (cc)]
#define A2_(r_, cc) A2[(size_t)(r_) * nz + (cc)]
  for (int p = 0; p < nY; ++p) {
    /* row block 1: D_l D_l'(D_eps/dt + D_sig/2) y' + (1/r) D_l G^T T^T u = ... (eq:updateEBC2) */
    A1_(p, p) = c[p];
    for (int k = p * rr; k < (p + 1) * rr; ++k) A1_(p, nY + k) = m->DlG[p] / rr;
    A2_(p, p) = a[p];
  }
  for (int k = 0; k < nU; ++k) {
    /* row block 2: T y' - L~^T xt' = 0 (eq:yandxt with transpose, R6) */
    A1_(nY + k, k / rr) = 1.0;
    for (int e = 0; e < q1; ++e) A1_(nY + k, X + e) = -L[(size_t)e * nU + k];
  }
  for (int e = 0; e < q1; ++e) {
    int row = X + e;
    for (int k = 0; k < nU; ++k) {
      const int p = k / rr;  /* coarse port of (fine) port k */
      double Sc = (p < bx) ? -dx : (p < 2 * bx) ? dx : (p < 2 * bx + by) ? dy : -dy;
      A1_(row, nY + k) = -L[(size_t)e * nU + k] * Sc / rr; /* -B~ */
    }
    for (int f = 0; f < q1; ++f) {
      A1_(row, X + f) = R11[(size_t)e * q1 + f] / dt + F11[(size_t)e * q1 + f];
      A2_(row, X + f) = R11[(size_t)e * q1 + f] / dt - F11[(size_t)e * q1 + f];
    }
    for (int h = 0; h < q2; ++h) A1_(row, X + q1 + h) = -K[(size_t)e * q2 + h];
  }
  for (int h = 0; h < q2; ++h) {
    int row = X + q1 + h;
    for (int g = 0; g < q2; ++g) {
      A1_(row, X + q1 + g) = R22[(size_t)h * q2 + g] / dt;
      A2_(row, X + q1 + g) = R22[(size_t)h * q2 + g] / dt;
    }
    for (int e = 0; e < q1; ++e) A2_(row, X + e) = -K[(size_t)e * q2 + h];
  }
#undef A1_
#undef A2_
  m->piv = (int *)malloc((size_t)nz * sizeof(int));
  if (lu_factor(A1, nz, m->piv) != 0) {
    free(A1); free(A2); free(c); free(a);
    return -4; /* singular A1 */
  }
  m->A1 = A1;
  m->A2 = A2;
  m->z = (double *)calloc(nz, sizeof(double));
  free(c); free(a);
  /* mark hole and interface (kinds) */
  for (int j = j0; j < j0 + by; ++j)
    for (int i = i0; i < i0 + bx; ++i) CELL(s, kc, i, j) = K_HOLE;
  for (int j = j0 + 1; j < j0 + by; ++j)
    for (int i = i0; i < i0 + bx; ++i) s->kx[(size_t)j * nx + i] = K_HOLE;
  for (int j = j0; j < j0 + by; ++j)
    for (int i = i0 + 1; i < i0 + bx; ++i) s->ky[(size_t)j * (nx + 1) + i] = K_HOLE;
  for (int p = 0; p < nY; ++p) {
    if (m->port_is_ey[p]) s->ky[m->port_edge[p]] = K_IFACE;
    else s->kx[m->port_edge[p]] = K_IFACE;
  }
  s->nrom++;
  return s->nrom - 1;
}

void osim_set_source_line(osim *s, int i, int j0, int j1, const double *samples, int64_t n, int64_t t0) {
  free(s->src);
  s->src = NULL;
  s->src_i = i; s->src_j = j0; s->src_j1 = j1; s->nsrc = n; s->src_t0 = t0;
  if (n > 0) {
    s->src = (double *)malloc((size_t)n * sizeof(double));
    memcpy(s->src, samples, (size_t)n * sizeof(double));
  }
}

void osim_set_source(osim *s, int i, int j, const double *samples, int64_t n, int64_t t0) {
  osim_set_source_line(s, i, j, j + 1, samples, n, t0);
}

void osim_set_probes(osim *s, const int *ij, int n) {
  free(s->probe);
  s->probe = (int *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int));
  s->nprobe = n;
  for (int p = 0; p < n; ++p) s->probe[p] = ij[2 * p + 1] * s->nx + ij[2 * p];
}

/* ------------------------------------------------------------------ */
/* one time step                                                       */
/* ------------------------------------------------------------------ */
/* Row loops may run on several host threads (OpenMP, rows are independent; results do not
 * depend on the thread count).  osim_set_threads(1) gives the plain single-threaded oracle. */
void osim_set_threads(int n) {
#ifdef _OPENMP
  omp_set_num_threads(n > 0 ? n : omp_get_num_procs());
#else
  (void)n;
#endif
}

int osim_get_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

static void coarse_h(osim *s) {
  /* eq:updateH (L267-273) at coarse resolution:
   * dx dy mu/dt H^{n+1/2} = dx dy mu/dt H^{n-1/2} - dx Ex_j + dx Ex_{j+1} + dy Ey_i - dy Ey_{i+1} */
  const int nx = s->nx, ny = s->ny;
  const double dx = s->dx, dy = s->dy, dt = s->dt, mu = O_MU0;
  memcpy(s->Hold, s->Hz, (size_t)nx * ny * sizeof(double));
#pragma omp parallel for schedule(static) if (ny >= 256)
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      if (CELL(s, kc, i, j) == K_HOLE) continue;
      double lhs = dx * dy * mu / dt;
      double rhs = lhs * HZ(s, i, j) - dx * EX(s, i, j) + dx * EX(s, i, j + 1) + dy * EY(s, i, j) -
                   dy * EY(s, i + 1, j);
      if (in_pml_col(s, i)) {  /* CPML: the x-derivative gains psi_hz */
        double *ps = &s->psi_hz[(size_t)j * nx + i];
        *ps = s->pml_bh[i] * *ps + s->pml_ah[i] * (EY(s, i + 1, j) - EY(s, i, j)) / dx;
        rhs -= dx * dy * *ps;
      }
      HZ(s, i, j) = rhs / lhs;
    }
}

static void coarse_e(osim *s) {
  /* eq:updateEx (L209-214): dx dy (eps/dt + sig/2) Ex^{n+1} = dx dy (eps/dt - sig/2) Ex^n
   *                           + dx Hz_{j+1/2} - dx Hz_{j-1/2};
   * eps, sig: arithmetic mean of the two adjacent cells (L215, R2).
   * Ey analogue (L223, sign from eq:updateEymat L239-252):
   *   dy dx (eps/dt + sig/2) Ey^{n+1} = dy dx (eps/dt - sig/2) Ey^n - dy (Hz_{i+1/2} - Hz_{i-1/2}). */
  const int nx = s->nx, ny = s->ny;
  const double dx = s->dx, dy = s->dy, dt = s->dt;
#pragma omp parallel for schedule(static) if (ny >= 256)
  for (int j = 1; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      if (s->kx[(size_t)j * nx + i] != K_NORMAL) continue;
      double eps = O_EPS0 * 0.5 * (CELL(s, eps_r, i, j - 1) + CELL(s, eps_r, i, j));
      double sig = 0.5 * (CELL(s, sigma, i, j - 1) + CELL(s, sigma, i, j));
      double lhs = dx * dy * (eps / dt + sig / 2);
      double rhs = dx * dy * (eps / dt - sig / 2) * EX(s, i, j) + dx * HZ(s, i, j) - dx * HZ(s, i, j - 1);
      EX(s, i, j) = rhs / lhs;
    }
#pragma omp parallel for schedule(static) if (ny >= 256)
  for (int j = 0; j < ny; ++j)
    for (int i = 1; i < nx; ++i) {
      if (s->ky[(size_t)j * (nx + 1) + i] != K_NORMAL) continue;
      double eps = O_EPS0 * 0.5 * (CELL(s, eps_r, i - 1, j) + CELL(s, eps_r, i, j));
      double sig = 0.5 * (CELL(s, sigma, i - 1, j) + CELL(s, sigma, i, j));
      double lhs = dy * dx * (eps / dt + sig / 2);
      double rhs = dy * dx * (eps / dt - sig / 2) * EY(s, i, j) - dy * HZ(s, i, j) + dy * HZ(s, i - 1, j);
      if (s->pml_w > 0 && (i <= s->pml_w || i >= nx - s->pml_w)) {  /* CPML psi_ey */
        double *ps = &s->psi_ey[(size_t)j * (nx + 1) + i];
        *ps = s->pml_be[i] * *ps + s->pml_ae[i] * (HZ(s, i, j) - HZ(s, i - 1, j)) / dx;
        rhs -= dy * dx * *ps;
      }
      EY(s, i, j) = rhs / lhs;
    }
}

/* storage function (R17):
 * W^n = (1/dt)[sum_e C_e (E_e^n)^2 + sum_c mu A H_c^{n-1/2} H_c^{n+1/2}] + sum_k xt_k^T R~ xt_k,
 * C_e = D_l D_l' eps (coarse half cell on interface edges), R~ of eq:R (L416-420). */
static double energy(const osim *s) {
  const int nx = s->nx, ny = s->ny;
  const double dx = s->dx, dy = s->dy, dt = s->dt;
  /* per-row partial sums (fixed order, so the value does not depend on the thread count) */
  double *row = (double *)calloc((size_t)ny + 1, sizeof(double));
#pragma omp parallel for schedule(static) if (ny >= 256)
  for (int j = 0; j <= ny; ++j) {
    double w = 0.0;
    if (j >= 1 && j < ny)
      for (int i = 0; i < nx; ++i) {
        if (s->kx[(size_t)j * nx + i] != K_NORMAL) continue;
        double eps = O_EPS0 * 0.5 * (CELL(s, eps_r, i, j - 1) + CELL(s, eps_r, i, j));
        w += dx * dy * eps * EX(s, i, j) * EX(s, i, j);
      }
    if (j < ny) {
      for (int i = 1; i < nx; ++i) {
        if (s->ky[(size_t)j * (nx + 1) + i] != K_NORMAL) continue;
        double eps = O_EPS0 * 0.5 * (CELL(s, eps_r, i - 1, j) + CELL(s, eps_r, i, j));
        w += dx * dy * eps * EY(s, i, j) * EY(s, i, j);
      }
      for (int i = 0; i < nx; ++i) {
        size_t c = (size_t)j * nx + i;
        if (s->kc[c] != K_HOLE) w += O_MU0 * dx * dy * s->Hold[c] * s->Hz[c];
      }
    }
    row[j] = w;
  }
  double w = 0.0;
  for (int j = 0; j <= ny; ++j) w += row[j];
  free(row);
  for (int r = 0; r < s->nrom; ++r) {
    const orom *m = &s->roms[r];
    for (int p = 0; p < m->nY; ++p) {
      double y = m->port_is_ey[p] ? s->Ey[m->port_edge[p]] : s->Ex[m->port_edge[p]];
      w += m->eps_half[p] * y * y;
    }
  }
  w /= dt;
  for (int r = 0; r < s->nrom; ++r) {
    const orom *m = &s->roms[r];
    const double *E = m->z + m->xoff, *H = E + m->q1;
    double e11 = 0, e22 = 0, ek = 0;
    for (int a = 0; a < m->q1; ++a)
      for (int b = 0; b < m->q1; ++b) e11 += E[a] * m->R11[(size_t)a * m->q1 + b] * E[b];
    for (int a = 0; a < m->q2; ++a)
      for (int b = 0; b < m->q2; ++b) e22 += H[a] * m->R22[(size_t)a * m->q2 + b] * H[b];
    for (int a = 0; a < m->q1; ++a)
      for (int b = 0; b < m->q2; ++b) ek += E[a] * m->K[(size_t)a * m->q2 + b] * H[b];
    /* xt^T R~ xt with R~ = [[R11/dt, -K/2], [-K^T/2, R22/dt]] */
    w += e11 / dt + e22 / dt - ek;
  }
  return w;
}

static void rom_step(osim *s, orom *m) {
  /* eq:sysform (L632-638): A1 z^{n+1} = A2 z^n + [D_l G^T H^{n+1/2}; 0; 0] */
  const int nz = m->nz, nY = m->nY;
  double *rhs = (double *)calloc(nz, sizeof(double));
  for (int p = 0; p < nY; ++p)  /* y^n from the interface edges */
    m->z[p] = m->port_is_ey[p] ? s->Ey[m->port_edge[p]] : s->Ex[m->port_edge[p]];
  for (int r = 0; r < nz; ++r) {
    double acc = 0.0;
    for (int c = 0; c < nz; ++c) acc += m->A2[(size_t)r * nz + c] * m->z[c];
    rhs[r] = acc;
  }
  for (int p = 0; p < nY; ++p) rhs[p] += m->DlG[p] * s->Hz[m->port_h[p]];
  lu_solve(m->A1, nz, m->piv, rhs);
  memcpy(m->z, rhs, (size_t)nz * sizeof(double));
  free(rhs);
}

/* ------------------------------------------------------------------ */
/* Direct subgridding reference (pin P-SUBGRID; no matrices).          */
/* Fine cells dx/r x dy/r (eq. (2)).  Fine interior updates:    */
/* eq:updateEx / eq:updateH with fine lengths.  Each coarse interface   */
/* edge is ONE node shared by the coarse half cell and the r fine half  */
/* cells behind it (eq:equalE); its row is the sum of the     */
/* coarse eq:updateExboundary and the r fine eq:updateExS rows, in      */
/* which the hanging terms cancel by eq:averH (L613-616):               */
/*   (c + sum_k c^_k) y' = (a + sum_k a^_k) y + D_l G h + sum_k (+-l^ H^_k) */
/* ------------------------------------------------------------------ */
#define FH(g, i, j) ((g)->Hz[(size_t)(j) * (g)->Nx + (i)])
#define FEX(g, i, j) ((g)->Ex[(size_t)(j) * (g)->Nx + (i)])
#define FEY(g, i, j) ((g)->Ey[(size_t)(j) * ((g)->Nx + 1) + (i)])
#define FC(g, a, i, j) ((g)->a[(size_t)(j) * (g)->Nx + (i)])

int osim_add_subgrid(osim *s, int i0, int j0, int bx, int by, int r, const double *fine_eps_r,
                     const double *fine_sigma) {
  if (bx < 1 || by < 1 || r < 1) return -1;
  if (i0 < 1 || j0 < 1 || i0 + bx > s->nx - 1 || j0 + by > s->ny - 1) return -2;
  for (int j = j0 - 1; j <= j0 + by; ++j)
    for (int i = i0 - 1; i <= i0 + bx; ++i)
      if (CELL(s, kc, i, j) != K_NORMAL) return -3;
  s->subs = (osub *)realloc(s->subs, (size_t)(s->nsub + 1) * sizeof(osub));
  osub *g = &s->subs[s->nsub];
  memset(g, 0, sizeof(*g));
  g->i0 = i0; g->j0 = j0; g->bx = bx; g->by = by; g->r = r;
  g->Nx = bx * r; g->Ny = by * r;
  size_t nf = (size_t)g->Nx * g->Ny;
  g->eps_r = (double *)malloc(nf * sizeof(double));
  g->sigma = (double *)malloc(nf * sizeof(double));
  memcpy(g->eps_r, fine_eps_r, nf * sizeof(double));
  memcpy(g->sigma, fine_sigma, nf * sizeof(double));
  g->Ex = (double *)calloc((size_t)g->Nx * (g->Ny + 1), sizeof(double));
  g->Ey = (double *)calloc((size_t)(g->Nx + 1) * g->Ny, sizeof(double));
  g->Hz = (double *)calloc(nf, sizeof(double));
  const int nx = s->nx;
  for (int j = j0; j < j0 + by; ++j)
    for (int i = i0; i < i0 + bx; ++i) CELL(s, kc, i, j) = K_HOLE;
  for (int j = j0 + 1; j < j0 + by; ++j)
    for (int i = i0; i < i0 + bx; ++i) s->kx[(size_t)j * nx + i] = K_HOLE;
  for (int j = j0; j < j0 + by; ++j)
    for (int i = i0 + 1; i < i0 + bx; ++i) s->ky[(size_t)j * (nx + 1) + i] = K_HOLE;
  for (int i = i0; i < i0 + bx; ++i) {
    s->kx[(size_t)j0 * nx + i] = K_IFACE;
    s->kx[(size_t)(j0 + by) * nx + i] = K_IFACE;
  }
  for (int j = j0; j < j0 + by; ++j) {
    s->ky[(size_t)j * (nx + 1) + i0] = K_IFACE;
    s->ky[(size_t)j * (nx + 1) + i0 + bx] = K_IFACE;
  }
  s->nsub++;
  return s->nsub - 1;
}

static void subgrid_step(osim *s, osub *g) {
  const int nx = s->nx, r = g->r, Nx = g->Nx, Ny = g->Ny, i0 = g->i0, j0 = g->j0;
  const int bx = g->bx, by = g->by;
  const double dx = s->dx, dy = s->dy, dt = s->dt, fdx = dx / r, fdy = dy / r;
  /* fine boundary E nodes take the value of their coarse edge (y^n) */
  for (int k = 0; k < Nx; ++k) {
    FEX(g, k, 0) = EX(s, i0 + k / r, j0);
    FEX(g, k, Ny) = EX(s, i0 + k / r, j0 + by);
  }
  for (int k = 0; k < Ny; ++k) {
    FEY(g, 0, k) = EY(s, i0, j0 + k / r);
    FEY(g, Nx, k) = EY(s, i0 + bx, j0 + k / r);
  }
  /* fine H: eq:updateH (L267-273) with fine lengths */
  for (int j = 0; j < Ny; ++j)
    for (int i = 0; i < Nx; ++i) {
      double lhs = fdx * fdy * O_MU0 / dt;
      double rhs = lhs * FH(g, i, j) - fdx * FEX(g, i, j) + fdx * FEX(g, i, j + 1) +
                   fdy * FEY(g, i, j) - fdy * FEY(g, i + 1, j);
      FH(g, i, j) = rhs / lhs;
    }
  /* interface rows: new coarse-edge values */
  double *ynew = (double *)malloc((size_t)(2 * bx + 2 * by) * sizeof(double));
  int p = 0;
  for (int side = 0; side < 4; ++side) {
    int nk = side < 2 ? bx : by;
    for (int k = 0; k < nk; ++k, ++p) {
      int oi, oj, fj = 0, fi = 0;
      double y, Dl, Dlp, G, fl, fmp;
      if (side == 0) { oi = i0 + k; oj = j0 - 1; y = EX(s, i0 + k, j0); G = -1; }
      else if (side == 1) { oi = i0 + k; oj = j0 + by; y = EX(s, i0 + k, j0 + by); G = +1; }
      else if (side == 2) { oi = i0 - 1; oj = j0 + k; y = EY(s, i0, j0 + k); G = +1; }
      else { oi = i0 + bx; oj = j0 + k; y = EY(s, i0 + bx, j0 + k); G = -1; }
      Dl = side < 2 ? dx : dy;
      Dlp = side < 2 ? dy / 2 : dx / 2;
      fl = side < 2 ? fdx : fdy;       /* fine primary edge length */
      fmp = side < 2 ? fdy / 2 : fdx / 2; /* fine half dual edge */
      double eps = O_EPS0 * CELL(s, eps_r, oi, oj), sig = CELL(s, sigma, oi, oj);
      double cap = Dl * Dlp * (eps / dt + sig / 2), keep = Dl * Dlp * (eps / dt - sig / 2);
      double drive = Dl * G * HZ(s, oi, oj);
      for (int m = 0; m < r; ++m) {
        double fe, fs, H, sgn;
        if (side == 0) { fi = k * r + m; fj = 0; H = FH(g, fi, 0); sgn = +1; }
        else if (side == 1) { fi = k * r + m; fj = Ny - 1; H = FH(g, fi, Ny - 1); sgn = -1; }
        else if (side == 2) { fi = 0; fj = k * r + m; H = FH(g, 0, fj); sgn = -1; }
        else { fi = Nx - 1; fj = k * r + m; H = FH(g, Nx - 1, fj); sgn = +1; }
        fe = O_EPS0 * FC(g, eps_r, fi, fj);
        fs = FC(g, sigma, fi, fj);
        cap += fl * fmp * (fe / dt + fs / 2);
        keep += fl * fmp * (fe / dt - fs / 2);
        drive += sgn * fl * H;
      }
      ynew[p] = (keep * y + drive) / cap;
    }
  }
  /* fine interior E: eq:updateEx / Ey analogue with fine lengths, mean of 2 fine cells */
  for (int j = 1; j < Ny; ++j)
    for (int i = 0; i < Nx; ++i) {
      double eps = O_EPS0 * 0.5 * (FC(g, eps_r, i, j - 1) + FC(g, eps_r, i, j));
      double sig = 0.5 * (FC(g, sigma, i, j - 1) + FC(g, sigma, i, j));
      double lhs = fdx * fdy * (eps / dt + sig / 2);
      FEX(g, i, j) = (fdx * fdy * (eps / dt - sig / 2) * FEX(g, i, j) + fdx * FH(g, i, j) -
                      fdx * FH(g, i, j - 1)) / lhs;
    }
  for (int j = 0; j < Ny; ++j)
    for (int i = 1; i < Nx; ++i) {
      double eps = O_EPS0 * 0.5 * (FC(g, eps_r, i - 1, j) + FC(g, eps_r, i, j));
      double sig = 0.5 * (FC(g, sigma, i - 1, j) + FC(g, sigma, i, j));
      double lhs = fdy * fdx * (eps / dt + sig / 2);
      FEY(g, i, j) = (fdy * fdx * (eps / dt - sig / 2) * FEY(g, i, j) - fdy * FH(g, i, j) +
                      fdy * FH(g, i - 1, j)) / lhs;
    }
  p = 0;
  for (int k = 0; k < bx; ++k) EX(s, i0 + k, j0) = ynew[p++];
  for (int k = 0; k < bx; ++k) EX(s, i0 + k, j0 + by) = ynew[p++];
  for (int k = 0; k < by; ++k) EY(s, i0, j0 + k) = ynew[p++];
  for (int k = 0; k < by; ++k) EY(s, i0 + bx, j0 + k) = ynew[p++];
  free(ynew);
  (void)nx;
}

/* probe_out: [nprobe][ldp] row-major, column (n - n_begin); energy_out: [nsteps] */
void osim_step(osim *s, int64_t nsteps, double *probe_out, int64_t ldp, double *energy_out) {
  for (int64_t t = 0; t < nsteps; ++t) {
    coarse_h(s);                                          /* S1 */
    if (s->src_i >= 0) {                                  /* S2 */
      int64_t k = s->n - s->src_t0;
      if (k >= 0 && k < s->nsrc)
        for (int j = s->src_j; j < s->src_j1; ++j) HZ(s, s->src_i, j) += s->src[k];
    }
    if (energy_out) energy_out[t] = energy(s);            /* S3: W^n */
    if (probe_out)
      for (int p = 0; p < s->nprobe; ++p) probe_out[(size_t)p * ldp + t] = s->Hz[s->probe[p]];
#pragma omp parallel for schedule(dynamic) if (s->nrom >= 8)
    for (int r = 0; r < s->nrom; ++r) rom_step(s, &s->roms[r]); /* S4-S5 (ROMs are independent) */
    for (int r = 0; r < s->nsub; ++r) subgrid_step(s, &s->subs[r]); /* reference only */
    coarse_e(s);                                          /* S7 */
    for (int r = 0; r < s->nrom; ++r) {                   /* S6 */
      orom *m = &s->roms[r];
      for (int p = 0; p < m->nY; ++p) {
        if (m->port_is_ey[p]) s->Ey[m->port_edge[p]] = m->z[p];
        else s->Ex[m->port_edge[p]] = m->z[p];
      }
    }
    s->n++;
  }
}

/* state access (NULL pointers skipped).  rom_state: per ROM xt (q1+q2). */
void osim_get_state(const osim *s, double *Ex, double *Ey, double *Hz, double *rom_state) {
  size_t nc = (size_t)s->nx * s->ny;
  if (Ex) memcpy(Ex, s->Ex, (size_t)s->nx * (s->ny + 1) * sizeof(double));
  if (Ey) memcpy(Ey, s->Ey, (size_t)(s->nx + 1) * s->ny * sizeof(double));
  if (Hz) memcpy(Hz, s->Hz, nc * sizeof(double));
  if (rom_state) {
    size_t off = 0;
    for (int r = 0; r < s->nrom; ++r) {
      const orom *m = &s->roms[r];
      memcpy(rom_state + off, m->z + m->xoff, (size_t)m->q * sizeof(double));
      off += m->q;
    }
  }
}

void osim_set_state(osim *s, const double *Ex, const double *Ey, const double *Hz,
                    const double *rom_state) {
  size_t nc = (size_t)s->nx * s->ny;
  if (Ex) memcpy(s->Ex, Ex, (size_t)s->nx * (s->ny + 1) * sizeof(double));
  if (Ey) memcpy(s->Ey, Ey, (size_t)(s->nx + 1) * s->ny * sizeof(double));
  if (Hz) memcpy(s->Hz, Hz, nc * sizeof(double));
  if (rom_state) {
    size_t off = 0;
    for (int r = 0; r < s->nrom; ++r) {
      orom *m = &s->roms[r];
      memcpy(m->z + m->xoff, rom_state + off, (size_t)m->q * sizeof(double));
      off += m->q;
    }
  }
}

int64_t osim_steps_taken(const osim *s) { return s->n; }
