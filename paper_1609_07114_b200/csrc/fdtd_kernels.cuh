// Internal device-side declarations shared by fdtd_kernels.cu and fdtd_api.cpp.
// Not part of the public ABI (include/fdtdrom.h is).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

// FDTD_CHECK=1 (a separate checked build, tools/checked_run.py): device-side bounds checks on every
// global and region access of the hot kernels, trapping with a message -- the stand-in for
// compute-sanitizer, which is closed on the GPU pool.
#ifndef FDTD_CHECK
#define FDTD_CHECK 0
#endif
#if FDTD_CHECK
#include <cstdio>
#define FCHK(cond, ...)                                                                       \
  do {                                                                                        \
    if (!(cond)) {                                                                            \
      printf("FDTD_CHECK %s:%d block (%d,%d) thread %d: %s\n", __FILE__, __LINE__, blockIdx.x,  \
             blockIdx.y, threadIdx.x, #cond);                                                 \
      __trap();                                                                               \
    }                                                                                         \
  } while (0)
#else
#define FCHK(cond, ...) \
  do {                  \
  } while (0)
#endif

namespace fdtd {

// K-step sweep: K time steps per pass over the grid (temporal blocking; K = 1
// is the plain fused one-step sweep).  Each step is S1 (eq:updateH), S2 (source), S3 (probes,
// energy partials of the non-zone cells) and S7 (eq:updateEx / Ey analogue); ping-pong buffers.
// ROM interface edges are frozen for the whole pass; the fix-up kernel repairs the zone around
// every instance.
constexpr int KMAX = 4;  // deepest pass (ghost rows on each side of a slab)
// HBM layout: the arrays of a pool are tile-interleaved along each row: a row of a
// pool of `na` arrays is a sequence of column tiles, tile t holding columns [t TILE, (t+1) TILE)
// of array 0, then of array 1, ...  Element (row, col) of array a sits at
// row * na * pitch + pool_off(col, na) + a * TILE (na = 1: the plain row-major array).
constexpr int TILE = 64;
__host__ __device__ inline int64_t pool_off(int64_t col, int na) {
  const int64_t t = col >= 0 ? col / TILE : -((-col + TILE - 1) / TILE);  // floor
  return t * TILE * na + (col - t * TILE);
}
template <typename T>
struct SweepParams {
  const T* ex0; const T* ey0; const T* hz0;  // fields at step n (E^n, H^{n-1/2})
  T* ex1; T* ey1; T* hz1;                     // fields at step n+K (E^{n+K}, H^{n+K-1/2})
  // per cell: mea = eps0 eps_r / (2 dt) (< 0: hole / wall / dead), msb = sigma / 4 with the sign
  // bit set on fix-up zone cells (their energy is added by the fix-up kernel)
  const T* mea; const T* msb;
  int64_t pitch;   // columns per row (a multiple of TILE)
  int naf, nam;    // arrays per pool: fields (ex, ey, hz of one buffer) and materials (mea, msb);
                   // 1 = separate row-major arrays
  int64_t nx;      // grid columns (the sweep processes ceil(nx / W) lane vectors per row)
  int rows;        // owned cell rows: local rows row0 .. row0+rows-1
  int row0;        // local row of the first owned row (KMAX ghost rows below)
  int chunk;       // rows per CTA
  int chunk0;      // first row chunk of this launch (split launches overlap the halo exchange)
  T chx, chy;      // dt/(mu0 dx), dt/(mu0 dy)
  int src_row;     // local rows [src_row, src_row_end) of the soft (line) source at column src_col (-1: none)
  int src_row_end;
  int64_t src_col;
  // src_meta = {t0, n}: the samples cover steps [t0, t0 + n) (device memory, so a new sample
  // window does not invalidate a captured graph)
  const double* src_samples; const int64_t* src_meta;
  const int64_t* step;  // device step counter (value n during the pass starting at step n)
  double* partials;     // energy partial per CTA and step: partials[s * pstride + cta] (nullptr: off)
  int64_t pstride;
  const int2* probe_rows;  // per local row: (first, count) into probe_list (count 0: none)
  const int2* probe_list;  // (column, probe index), sorted by row then column
  T* probe_ring; int64_t cap;
  T idx, idy;           // 1/dx, 1/dy
  T wxy, wh;            // dx dy, mu0 dx dy / dt (energy weights)
  int64_t alloc_elems_f, alloc_elems_m;  // elements of a field / material pool incl. its tail (FDTD_CHECK)
};

// Fused per-model operators (column-major, in the model pool), with x = [E~; H~] (q1 + q2):
//   M1 ((q2 + q1 + nY) x (q1 + q2)) = [[Q1, I], [Aq', Kq], [-L~^T Aq', -L~^T Kq]],  Aq' = Aq + Kq Q1
//      -> [H~^{n+1}; E*; -L~^T E*] in one product (K3)
//   M2 ((q1 + nY) x nY) = [Bq; L~^T Bq]  -> [E~ - E*; y - L~^T E*] from U
//   Rt ((q1 + q2) x (q1 + q2)) = [[R~11/dt, -K~/2], [-K~^T/2, R~22/dt]]  (storage function)
// The fix-up's GEMMs run on the FP64 tensor cores (mma.sync.m8n8k4.f64, fdtd_kernels.cu
// dmma_gemm): [M1; R~] and M2 are kept in an fp64 pool, pre-tiled in the MMA's A-fragment order
// (mt x kt tiles of 8 x 4, one double per lane and tile).
struct RomModelDev {
  int nY, q1, q2;
  int literal;  // paper-literal coupling: U is y^{n+1} itself and M2 = [Z T; I] (K3)
  int64_t off_M1t, off_M2t;     // tiled operators in the pool
  int mt1, kt1, mt2, kt2;       // their tile counts: [M1; R~] (m1 + q1 + q2 rows), M2 (q1 + nY rows)
};

// Fix-up kernel: per ROM instance, the K steps of the pass are recomputed on
// the region [i0-M, i0+bx+M) x [j0-M, j0+by+M) (M = Kz + K - 1) from the pass's input buffer,
// with the ROM update (S4-S6, eq:connExplicit) between them; the zone cells (the ones the sweep
// may have got wrong and whose energy it skipped) are written back.  Also: zone probes and the
// per-batch ROM + zone energies (finalize_kernel sums them with the sweep's).
constexpr int BATCH_FIELDS = 6;  // batch table entry: model, member offset, count, slots, region stride, kind
template <typename T>
struct PostParams {
  int n_inst;
  int n_batch;                     // batches of <= batch instances of one model (level-1 energy slots)
  int n_batch_reg;                 // batches [0, n_batch_reg): postk_kernel; the rest are single
                                   // instances of large models (bigrom_kernel, cooperative)
  const int32_t* batch_tab;        // per batch: (model, member offset, count, slots B, region stride, kind)
  const int32_t* batch_inst;       // the batches' members (instance indices)
  const int32_t* batch_rect;       // per batch: the cluster's bounding box (i0, j0, w, h) (kind 1)
  const RomModelDev* models;
  const double* mpool;             // shared model operators (fp64), tiled for the DMMA GEMMs
  const T* Sk; const int64_t* Sk_off;        // per-instance Schur inverses (col-major nY x nY)
  const int64_t* port_off;                    // per-instance offset into port arrays
  const T* cya; const T* cyg;                 // a_y / c_y, D_l G / c_y per port
  const double* ehalf;                        // D_l D_l' eps / dt per port (energy)
  const int64_t* port_edge;                   // per port: (is_ey << 62) | element offset
  T* state; const int64_t* state_off;         // per instance [E~ (q1); H~ (q2)]
  T* ex1; T* ey1; T* hz1;                     // output buffer (the sweep's)
  const T* ex0; const T* ey0; const T* hz0;   // input buffer (state at step n)
  const T* mea; const T* msb;
  int64_t pitch, row_begin;
  int64_t nx, ny;                  // global grid (cells outside load as dead cells)
  int row0;                        // local row of global row row_begin
  int Kz;                          // zone depth of the material marks (>= K)
  const int32_t* rects;            // per instance (i0, j0, bx, by), global
  const int32_t* zp_off; const int32_t* zp;  // zone probes per instance: (gi, gj, probe index)
  T* probe_ring; int64_t cap;
  T chx, chy, idx, idy, wxy, wh;
  int src_row, src_row_end; int64_t src_col; const double* src_samples; const int64_t* src_meta;
  double* rom_partials;            // [s * n_inst + instance]: ROM + zone energy of step n+s
  double* level1;                  // [s * n_batch + batch]: the batch's sum of rom_partials
  const int64_t* step;             // step counter (value n during the pass; finalize advances it)
  int block;         // threads per CTA
  size_t smem_bytes; // dynamic shared memory of the launch (max over batches)
  int* flag;         // non-finite sentinel: set to 1 when a stored ROM state is not finite
  T* big;            // bigrom_kernel scratch (x~ twice, [M1; R~] x~, y and h of the largest model)
  size_t big_smem_bytes; int big_grid;
  int64_t alloc_elems; int rows, n_probe;  // FDTD_CHECK bounds: array elements, owned rows, probes
  // whole-grid mode (wholegrid_kernel): every probe (i, j, probe index) and the energy ring
  const int32_t* wprobe; int n_wprobe;
  double* energy_ring;
  int whole_coef;  // 1: every edge's coefficients precomputed in shared memory after the region
};

// End of a pass (finalize_kernel, after the sweep, the CPML bands and the fix-up): W^{n+s} as a
// fixed-order two-level sum of the sweep / band partials and the fix-up batches' values
// (deterministic), and the device step counter.  FIN_GRID CTAs (one when energy is off).
constexpr int FIN_GRID = 64;
struct FinParams {
  const double* sweep_partials; int64_t n_sweep_partials, pstride;  // [s * pstride + cta]
  const double* rom_level1; int n_rom;                              // [s * n_rom + batch]
  double* level2;                  // [s * FIN_GRID + cta]
  double* energy_ring; int64_t cap;
  int64_t* step; unsigned int* done;
  int K; bool energy;
  // non-finite sentinel (include/fdtdrom.h "Errors"): the last CTA sets *flag = 1 when an energy
  // value of the pass or one of NSAMPLE strided Hz cells of the pass's output is not finite
  const void* hz; int64_t pitch, nx; int row0, rows, es;
  int* flag;
};
constexpr int NSAMPLE = 256;
void launch_finalize(const FinParams& p, cudaStream_t s);

// CPML band fix-up (NEXT-2): the sweep advances the two x-end layers with the plain Yee update; per
// row chunk and side this kernel recomputes the K steps on the band [layer + Kz + K + 2 columns] x
// [chunk rows +- K] from the pass's input buffer with the CPML terms (Roden-Gedney, kappa 1, alpha 0)
// and writes back the layer plus Kz + 1 interior columns (the sweep skipped their energy: msb marks).
template <typename T>
struct PmlParams {
  const T* ex0; const T* ey0; const T* hz0;
  T* ex1; T* ey1; T* hz1;
  const T* mea; const T* msb;
  int64_t pitch, nx;
  int rows, row0, chunk;       // owned rows, local row of the first, rows per CTA
  int w, Kz;                   // layer width (cells); zone depth (write-back = w + Kz + 1 columns)
  const T* bh; const T* ah;    // per side [2][w]: Hz columns, index = distance into the layer
  const T* be; const T* ae;    // per side [2][w + 1]: Ey columns
  const T* psih; const T* psie;  // psi at step n: [2 sides][rows_alloc][w], [2 sides][rows_alloc][w + 1]
  T* psih1; T* psie1;            // psi at step n + K (ping-pong like the fields: CTAs read their
                                 // neighbours' ghost rows while they write their own)
  int64_t psi_rows;              // rows_alloc
  T chx, chy, idx, idy, wxy, wh, cpsi, dxv;  // cpsi = dt / mu0, dxv = dx
  int src_row, src_row_end; int64_t src_col; const double* src_samples; const int64_t* src_meta;
  const int64_t* step;
  int n_probe; const int64_t* probe_gi; const int32_t* probe_lr; T* probe_ring; int64_t cap;
  double* partials; int64_t pstride, poff;  // energy: partials[s * pstride + poff + cta]
  int64_t alloc_elems;                      // FDTD_CHECK bounds
};
template <typename T>
void launch_pml(const PmlParams<T>& p, int K, bool energy, cudaStream_t s);
inline int pml_ctas(int rows, int chunk) { return 2 * ((rows + chunk - 1) / chunk); }

template <typename T>
void launch_sweep(const SweepParams<T>& p, int K, int warps_per_cta, cudaStream_t s, int chunk_begin = 0,
                  int chunk_count = -1);
// Lane geometry of a K-step sweep: every lane holds W consecutive columns (one 8- or 16-byte
// vector per array); errors from a warp's outermost columns spread one column per step, so the
// HL = ceil(K / W) lanes at each end are redundant halo lanes and 32 - 2 HL lanes store.
inline int sweep_width(int elem_bytes, int K) { return elem_bytes == 4 ? (K >= 4 ? 2 : 4) : 2; }
inline int sweep_halo(int K, int W) { return (K + W - 1) / W; }
inline int sweep_ctas_x(int64_t nx, int elem_bytes, int K, int warps_per_cta) {
  const int W = sweep_width(elem_bytes, K), HL = sweep_halo(K, W);
  const int64_t nvec = (nx + W - 1) / W, nw = (nvec + 32 - 2 * HL - 1) / (32 - 2 * HL);
  return (int)((nw + warps_per_cta - 1) / warps_per_cta);
}
template <typename T>
void launch_post(const PostParams<T>& p, int K, bool energy, cudaStream_t s);
template <typename T>
void launch_post_big(const PostParams<T>& p, int K, bool energy, cudaStream_t s);
// K3c: the whole grid in one CTA for nsteps steps (p.n_batch == 1: one batch of every instance
// around the whole-grid region; p.smem_bytes its shared memory)
template <typename T>
void launch_wholegrid(const PostParams<T>& p, int64_t nsteps, bool energy, cudaStream_t s);
template <typename T>
int big_grid_size(size_t smem, int K);
// shared-memory bytes of the fix-up kernel for a given batch (host-side sizing)
size_t post_smem_bytes(size_t es, int nvec, int nY, int batch, int region_stride);
// elements of one instance region for zone depth Kz and pass depth K (<= Kz)
// H, MA, MS (Hr x Wr), EX ((Hr + 1) x Wr), EY (Hr x (Wr + 1)) and the zone energies (at most
// (bx + M) x (by + M): the zone of depth Kz spans bx + 2 Kz - 1 <= bx + M columns)
inline int region_elems(int bx, int by, int M) {
  const int Wr = bx + 2 * M, Hr = by + 2 * M;
  return 3 * Hr * Wr + (Hr + 1) * Wr + Hr * (Wr + 1) + (bx + M) * (by + M);
}

// setup kernels
template <typename T, typename M>
void launch_materials(const M* eps_r, const M* sigma, int64_t mat_row0, int64_t mat_row_end, int64_t nx, int64_t ny,
                      int64_t row_begin, int row0, int nrows_alloc, int64_t pitch, double dt, T* mea, T* msb,
                      cudaStream_t s);
template <typename M>
void launch_gather_materials(const M* eps_r, const M* sigma, int64_t nx, int64_t mat_row0,
                             const int64_t* cells /*global j*nx+i*/, int64_t n, double* out_eps,
                             double* out_sig, cudaStream_t s);
template <typename M>
void launch_min2(const M* a, const M* b, int64_t n, double* out /*2 per block*/, int nblocks, cudaStream_t s);
template <typename T>
void launch_random_fields(T* ex, T* ey, T* hz, const T* mea, int64_t pitch, int64_t nx, int rows, int row0,
                          int64_t row_begin, uint64_t seed, double ae, double ah, cudaStream_t s);
template <typename T>
void launch_mask(T* mea, T* fields[6], int64_t pitch, const int32_t* rects, int64_t n_rect, int64_t row_begin,
                 int row0, bool zero_iface, cudaStream_t s);
// sign bit of msb on the columns [0, ncol) and [nx - ncol, nx) of every owned row (PML bands)
template <typename T>
void launch_band_marks(T* msb, const T* mea, int64_t pitch, int64_t nx, int row0, int rows, int ncol, bool set,
                       cudaStream_t s);
// sign bit of msb on the zone cells of every instance (depth Kz; set or clear), holes excluded
template <typename T>
void launch_zone(T* msb, const T* mea, int64_t pitch, const int32_t* rects, int64_t n_rect, int64_t row_begin,
                 int row0, int Kz, bool set, cudaStream_t s);

#if FDTD_PHASES
void debug_phases(long long* out, int n);  // tuning builds: the fix-up's phase stamps
#endif

}  // namespace fdtd
