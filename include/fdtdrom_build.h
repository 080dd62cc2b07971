/*
 * fdtdrom_build.h -- C ABI of the GPU-side ROM construction of
 * Zhang, Bekmambetova, Triverio, "A Stable FDTD Method with Embedded Reduced-Order Models"
 * (arXiv 1609.07114).  Implemented by paper_1609_07114_b200/libfdtdrom.so (CUDA, sm_100a).
 *
 * One call runs the whole construction of one embedded model on one GPU and returns the reduced
 * matrices that fdtd_add_rom (fdtdrom.h) consumes:
 *   1. fine assembly of the refined block (Sec. II, eq:sys1a/b L286-292 with eq:R, eq:F_f, eq:B,
 *      eq:L, eq:F11, eq:K L323-382; boundary nodes with half dual lengths, eq:updateExS L217-222)
 *      and the exact collapse onto coarse-edge ports (R9: eq:equalE L608-611 makes the r
 *      fine boundary E nodes of one coarse edge one degree of freedom);
 *   2. SPRIM (L393-400, R10): block Arnoldi on (G + s0 C)^{-1} C from (G + s0 C)^{-1} B
 *      with C = blkdiag(R11, R22), G = [[2 F11, -K], [K^T, 0]], real s0 = pi f_max, classical
 *      Gram-Schmidt run twice in the C inner product, deflation 1e-10; the shifted systems are
 *      solved through the E-node Schur complement diag(2 F11 + s0 R11) + K (s0 R22)^{-1} K^T with
 *      Jacobi-preconditioned conjugate gradients (one CTA per right-hand side);
 *   3. the E and H rows of the basis orthonormalised separately, column by column in Krylov order
 *      (classical Gram-Schmidt twice, deflation 1e-10), the first q1 / q2 directions kept:
 *      V = blkdiag(V1, V2) (eq:V L394-400);
 *   4. congruence eq:R11_tilde .. eq:K_tilde (L431-447): R~11 = V1^T R11 V1, R~22, F~11,
 *      K~ = V1^T K V2, L~ = V1^T L_c (the port rows of V1);
 *   5. optionally the CFL extension (eq:CFLgeneralized L741-745, R11/R12): the singular
 *      values of R~11^{-1/2} K~ R~22^{-1/2} (one-sided Jacobi SVD) are clipped at
 *      (2 / dt_target)(1 - 1e-6).
 * The same algorithm, step for step, is inputs/romgen.py (the CPU input generator); the two share
 * no code.  Both port forms: collapsed (R9) and the paper-literal nP-port set (NEXT-1).
 *
 * Ownership: host inputs are read before the call returns; outputs are written into caller
 * buffers sized for the requested order.  Device memory is allocated and freed inside the call
 * (cudaMalloc on the current device, work on one internal stream).
 * Errors: FDTD_E_ARG (bad sizes, q < 2, non-finite or non-positive eps_r), FDTD_E_STATE (a CG
 * solve did not converge, or R~11 / R~22 not positive definite), FDTD_E_CUDA, FDTD_E_NOMEM.
 */
#ifndef FDTDROM_BUILD_H
#define FDTDROM_BUILD_H

#include <stdint.h>

#include "fdtdrom.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t bx, by, r;     /* coarse block (cells) and refinement factor                         */
  double dx, dy;         /* coarse cell size (m); fine cells are dx / r x dy / r                */
  const double *eps_r;   /* host, (by r) x (bx r) fine cells, row-major (row j of y slow)      */
  const double *sigma;   /* host, same layout (S/m)                                            */
  int32_t q;             /* requested order: q1 = ceil(q / 2) E directions, q2 = floor(q / 2) */
  double fmax;           /* expansion point s0 = pi fmax (Hz)                                  */
  double dt_target;      /* > 0: clip at (2 / dt_target)(1 - 1e-6); <= 0: no clip             */
  double cg_tol;         /* relative residual of the shifted solves (<= 0: 1e-13)              */
  int32_t literal;       /* 1: the paper-literal nP-port form (NEXT-1): ports are the nP =
                          * 2 (bx + by) r fine boundary nodes (no collapse), the E basis is
                          * [port unit vectors | SPRIM directions] orthonormalised in order
                          * (q1 = nP + ceil(q/2)); output L is q1 x nP                        */
} fdtd_rom_spec;

typedef struct {
  /* outputs (row-major, host, caller-allocated for q1 = ceil(q/2) (literal: nP + ceil(q/2)),
   * q2 = floor(q/2) and nY = 2 bx + 2 by (literal: nP = r nY)): R11 q1 x q1, R22 q2 x q2,
   * F11 q1 x q1, K q1 x q2, L q1 x nY.  The built
   * orders are returned in q1 / q2 (smaller when the Krylov space is exhausted) and the arrays
   * are packed for those orders. */
  double *R11, *R22, *F11, *K, *L;
  int32_t q1, q2, nY;
  int32_t n_clipped;          /* singular values clipped by the CFL extension                  */
  double natural_dt_limit;    /* 2 / s_max(R~11^{-1/2} K~ R~22^{-1/2}) before the clip          */
  /* diagnostics */
  int32_t krylov_vectors;     /* m of the final Arnoldi run                                    */
  int32_t cg_iterations_max;  /* largest CG iteration count of any solve                       */
  int32_t jacobi_sweeps_max;  /* largest sweep count of any one-sided Jacobi SVD               */
  double ms_total, ms_solve, ms_orth, ms_svd;  /* device-timed phases                          */
} fdtd_rom_built;

/* Build one ROM on the current CUDA device (see the header comment for the steps). */
fdtd_status fdtd_rom_build(const fdtd_rom_spec *spec, fdtd_rom_built *out);

/* Text of the calling thread's last fdtd_rom_build failure ("" if none). */
const char *fdtd_rom_build_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* FDTDROM_BUILD_H */
