// Internal device-side declarations shared by fdtd_kernels.cu and fdtd_api.cpp.
// Not part of the public ABI (include/fdtdrom.h is).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fdtd {

// Fused single-pass H+E sweep: S1 (eq:updateH), S2 (source), S3 (energy
// partials) and S7 (eq:updateEx / Ey analogue) for one time step, ping-pong buffers.
template <typename T>
struct SweepParams {
  const T* ex0; const T* ey0; const T* hz0;  // fields at step n (E^n, H^{n-1/2})
  T* ex1; T* ey1; T* hz1;                     // fields at step n+1 (E^{n+1}, H^{n+1/2})
  const T* mea; const T* msb;  // per cell: eps0 eps_r / (2 dt) (< 0: hole / wall / dead) and sigma / 4
  int64_t pitch;   // elements per row (all arrays)
  int ncolv;       // vector columns processed (16-byte vectors)
  int rows;        // owned cell rows: local rows row0 .. row0+rows-1
  int row0;        // local row of the first owned row (ROW0 = 2: two ghost rows below)
  int chunk;       // rows per CTA
  int chunk0;      // first row chunk of this launch (split launches overlap the halo exchange)
  T chx, chy;      // dt/(mu0 dx), dt/(mu0 dy)
  int src_row;     // local row of the soft source (-1: none)
  int64_t src_col;
  const double* src_samples; int64_t src_n, src_t0;
  const int64_t* step;  // device step counter (value n during step n)
  double* partials;     // energy partial per CTA (nullptr: energy off)
  double* partials2;    // two-step sweep: partials of the second step
  T idx, idy;           // 1/dx, 1/dy
  T wxy, wh;            // dx dy, mu0 dx dy / dt (energy weights)
};

// Fused per-model operators (column-major, in the model pool), with x = [E~; H~] (q1 + q2):
//   M1 ((q2 + q1 + nY) x (q1 + q2)) = [[Q1, I], [Aq', Kq], [-L~^T Aq', -L~^T Kq]],  Aq' = Aq + Kq Q1
//      -> [H~^{n+1}; E*; -L~^T E*] in one product (K3)
//   M2 ((q1 + nY) x nY) = [Bq; L~^T Bq]  -> [E~ - E*; y - L~^T E*] from U
//   Rt ((q1 + q2) x (q1 + q2)) = [[R~11/dt, -K~/2], [-K~^T/2, R~22/dt]]  (storage function)
struct RomModelDev {
  int nY, q1, q2;
  int64_t off_M1, off_M2, off_Rt;
};

// Post kernel: S4-S6 per ROM instance, probe recording, deterministic
// energy finalisation and the device step counter.
template <typename T>
struct PostParams {
  int n_inst;
  int n_batch;                     // CTAs doing ROM work; batches of <= batch instances of one model
  int batch;                       // instances per batch (multiple of 4)
  const int32_t* batch_tab;        // per batch: (model, first instance, count)
  const int32_t* inst_model;
  const RomModelDev* models;
  const T* mpool;                  // shared model matrices (column-major)
  const T* Sk; const int64_t* Sk_off;        // per-instance Schur inverses (col-major nY x nY)
  const int64_t* port_off;                    // per-instance offset into port arrays
  const T* cya; const T* cyg;                 // a_y / c_y, D_l G / c_y per port
  const double* ehalf;                        // D_l D_l' eps / dt per port (energy)
  const int64_t* port_edge;                   // per port: (is_ey << 62) | element offset
  const int64_t* port_h;                      // per port: Hz element offset of the outside cell
  const int64_t* ring_idx; const int64_t* ring_off;  // hole-ring Hz cells per instance
  T* state; const int64_t* state_off;         // per instance [E~ (q1); H~ (q2)]
  T* ex1; T* ey1; T* hz1;
  int n_probe; const int64_t* probe_idx; T* probe_ring; int64_t cap;
  const double* sweep_partials; int n_sweep_partials; double* rom_partials; double* energy_ring;
  double* level1;                  // per post CTA energy partial (gridDim.x entries)
  int64_t* step; unsigned int* done;
  int nthreads_vec;  // max(q1 + q2 + nY) over models: shared-memory vector stride
  int block;         // threads per CTA
  // ---- two-step mode (post2): fix-up around every instance after sweep2 (K3b)
  const int32_t* rects;            // per instance (i0, j0, bx, by), global
  int64_t row_begin, pitch;
  int row0;                        // local row of global row row_begin
  const T* ex0; const T* ey0; const T* hz0;  // fields at step n (the sweep's input buffer)
  const T* mea; const T* msb;
  T chx, chy, idx, idy, wh;
  int src_row; int64_t src_col; const double* src_samples; int64_t src_n, src_t0;
  const double* sweep_partials2; double* rom_partials2; double* level1b;
  int region_stride;               // shared-memory elements per instance region
};

template <typename T>
void launch_sweep(const SweepParams<T>& p, int warps_per_cta, cudaStream_t s, int chunk_begin = 0,
                  int chunk_count = -1);
// two time steps per pass (temporal blocking; 30 output lanes per warp)
template <typename T>
void launch_sweep2(const SweepParams<T>& p, int warps_per_cta, cudaStream_t s, int chunk_begin = 0,
                   int chunk_count = -1);
inline int sweep2_ctas_x(int ncolv, int warps_per_cta) {
  const int nw = (ncolv + 29) / 30;
  return (nw + warps_per_cta - 1) / warps_per_cta;
}
template <typename T>
void launch_post(const PostParams<T>& p, bool energy, cudaStream_t s);
template <typename T>
void launch_post2(const PostParams<T>& p, bool energy, cudaStream_t s);
// shared-memory bytes of the two kernels for a given batch (host-side sizing)
size_t post_smem_bytes(size_t es, int nvec, int batch);
size_t post2_smem_bytes(size_t es, int nvec, int batch, int region_stride);

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
void launch_mask(T* mea, T* fields[6], int64_t pitch, const int32_t* rects, int64_t n_rect, int64_t row_begin,
                 int row0, bool zero_iface, cudaStream_t s);

}  // namespace fdtd
