// Host implementation of the C ABI declared in include/fdtdrom.h.
//
// Owns the device state of one row slab: ping-pong field buffers with ghost rows on each side,
// the per-cell material terms, the ROM operators, probe/energy record rings, and (for several
// ranks) an NCCL communicator used for the per-pass halo exchange of DESIGN.md "Multi-GPU".  All
// work is enqueued on one stream; fdtd_step replays a captured CUDA graph of two K-step passes
// when possible.
#include "fdtdrom.h"

#include <dlfcn.h>

#include <algorithm>
#include <array>
#include <functional>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "dense.hpp"
#include "fdtd_kernels.cuh"

namespace {

using fdtd::KMAX;
constexpr int ROW0 = 2 * KMAX;  // local row of the first owned row: the K-step sweep's first chunk
                                // reads K halo rows below it and stage rows down to r0 - 2K
constexpr int GHOST_UP = KMAX;  // ghost rows above the slab (Ex edge rows up to row_end + K - 1)
constexpr int PML_CHUNK = 32;   // rows per CTA of the CPML band fix-up
constexpr double MU0 = 4.0e-7 * 3.14159265358979323846;
constexpr double C0 = 299792458.0;
constexpr double EPS0 = 1.0 / (MU0 * C0 * C0);

// ---------------------------------------------------------------- NCCL (dlopen)
typedef struct { char internal[128]; } nccl_uid;
typedef void* nccl_comm;
struct Nccl {
  void* h = nullptr;
  int (*CommInitRank)(nccl_comm*, int, nccl_uid, int) = nullptr;
  int (*CommDestroy)(nccl_comm) = nullptr;
  int (*Send)(const void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  int (*GetUniqueId)(nccl_uid*) = nullptr;
  bool load(std::string& err) {
    if (h) return true;
    const char* env = getenv("FDTD_NCCL_LIB");
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the copy torch already loaded
    if (!h && env) h = dlopen(env, RTLD_NOW);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) { err = "cannot load libnccl.so.2"; return false; }
#define SYM(n) n = reinterpret_cast<decltype(n)>(dlsym(h, "nccl" #n)); if (!n) { err = "missing nccl" #n; return false; }
    SYM(CommInitRank) SYM(CommDestroy) SYM(Send) SYM(Recv) SYM(GroupStart) SYM(GroupEnd) SYM(AllReduce)
    SYM(GetErrorString) SYM(GetUniqueId)
#undef SYM
    return true;
  }
};
Nccl g_nccl;
constexpr int NCCL_I32 = 2, NCCL_F32 = 7, NCCL_F64 = 8, NCCL_SUM = 0, NCCL_MAX = 2, NCCL_MIN = 3;

struct ModelHost {
  int bx, by, nY, q1, q2;
  bool literal = false;
  // per-instance Schur base (nY x nY): collapsed L~^T C^-1 B~ (S_k = (P + diag(D_l G / c_y))^-1);
  // literal Psi = (1/r) D_l G T^T P_f^-1 T (S_k = (diag(c_y) + Psi)^-1)
  std::vector<double> P;
  fdtd::RomModelDev dev;
};

}  // namespace

struct fdtd_ctx {
  fdtd_grid_desc d{};
  int prec = 32;
  size_t es = 4;  // element size
  int V = 4;      // elements per 16-byte vector
  int rows = 0;   // owned rows
  int64_t nrows_alloc = 0, pitch = 0;  // rows + ROW0 + GHOST_UP
  int ncolv = 0;
  cudaStream_t stream = nullptr, cap_stream = nullptr;
  std::string err;
  // device buffers (element type T)
  void* f[2][3] = {{nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr}};  // [buf][ex,ey,hz]
  void* coef[2] = {nullptr, nullptr};  // per cell: mea = eps0 eps_r/(2 dt) (-1: hole/wall), msb = sigma/4
  void* mat_eps = nullptr;  // device copy of per-cell materials for rows [mrow0, row_end)
  void* mat_sig = nullptr;
  bool mat_f32 = false;
  int64_t mrow0 = 0, mrow_end = 0;
  int64_t* d_step = nullptr;
  unsigned* d_done = nullptr;
  double* d_partials = nullptr;   // [KMAX][n_partials] sweep energy partials
  double* d_level1 = nullptr;     // [KMAX][post grid]
  int n_partials = 0;
  int chunk = 64, warps = 4;
  // source
  double* d_src = nullptr;
  int64_t* d_src_meta = nullptr;  // {t0, n} of the sample window (device: graphs survive a new window)
  int64_t h_src_meta[2] = {0, 0};
  int64_t src_i = -1, src_j = -1, src_j1 = -1, src_cap = 0;  // cells (i, j .. j1-1)
  int* d_flag = nullptr;          // non-finite sentinel (sticky; read at the synchronous calls)
  // probes & energy rings
  int64_t cap = 65536;
  int n_probe = 0;
  std::vector<int64_t> probe_ij;   // global (i, j) per probe
  int2* d_probe_rows = nullptr;    // per local row: (first, count) into d_probe_list
  int2* d_probe_list = nullptr;    // (column, probe index), owned probes sorted by row, column
  void* d_probe_ring = nullptr;
  double* d_energy_ring = nullptr;
  bool energy_on = false;
  int64_t steps = 0, rd_probe = 0, rd_energy = 0;
  int cur = 0;  // buffer holding the current state (E^n, H^{n-1/2})
  // K-step passes (K1/K3): k_want requested, k_ok the deepest this rank can do,
  // kz the depth in use (agreed over ranks; the zone marks in msb are for kz)
  int k_want = 4, k_ok = 1, kz = 1, kz_marked = 1;
  bool kz_dirty = true;
  size_t post_smem = 0;  // dynamic shared memory of the fix-up launch
  int post_threads = 512;
  int32_t* d_rects = nullptr;
  std::vector<int32_t> zp_off, zp;  // zone probes per instance (gi, gj, probe index)
  // CPML on the two x-ends (NEXT-2): width, per-column coefficients, psi state, marked columns
  int pml_w = 0, pml_marked = 0;
  void *d_pml_bh = nullptr, *d_pml_ah = nullptr, *d_pml_be = nullptr, *d_pml_ae = nullptr;
  void *d_psih = nullptr, *d_psie = nullptr;
  int64_t* d_probe_gi = nullptr;
  int32_t* d_probe_lr = nullptr;
  int32_t* d_zp_off = nullptr;
  int32_t* d_zp = nullptr;
  // ROMs
  std::vector<ModelHost> models;
  std::vector<int32_t> inst_model, rects;  // rects: (i0, j0, bx, by) global
  std::vector<int64_t> port_off, port_edge, state_off, Sk_off;
  std::vector<double> cya, cyg, ehalf, Sk;  // fp64 host copies (converted on upload)
  std::vector<double> mpool;                // shared model operators tiled for the DMMA GEMMs (fp64)
  int nvec = 1;
  std::vector<int32_t> batch_tab;  // (model, member offset, count, slots B, region stride, kind)
  std::vector<int32_t> batch_inst, batch_rect;  // batch members; cluster boxes (kind 1)
  int32_t* d_batch_tab = nullptr;
  int32_t* d_batch_inst = nullptr;
  int32_t* d_batch_rect = nullptr;
  std::vector<int32_t> zone_marked;  // the zone boxes whose cells carry the msb marks (kz_marked deep)
  int32_t* d_zone_marked = nullptr;
  int n_clusters = 0;
  // whole-grid mode (K3c): the grid and every instance in one CTA, one launch per
  // fdtd_step call; its batch table (one kind-1 batch around the whole grid) and probe list
  bool whole = false;
  bool whole_coef = false;
  size_t whole_smem = 0;
  int32_t* d_wb_tab = nullptr;
  int32_t* d_wb_inst = nullptr;
  int32_t* d_wb_rect = nullptr;
  int32_t* d_wprobe = nullptr;
  int n_wprobe = 0;
  int post_grid = 1;
  int n_batch_reg = 0;           // regular fix-up batches; the rest are large-model instances
  void* d_big = nullptr;         // bigrom_kernel scratch
  size_t big_smem = 0;
  int big_grid = 0;
  // device ROM arrays
  void* d_mpool = nullptr; void* d_Sk = nullptr; void* d_cya = nullptr; void* d_cyg = nullptr;
  void* d_state = nullptr; double* d_ehalf = nullptr; double* d_rom_partials = nullptr;
  int64_t *d_port_off = nullptr, *d_port_edge = nullptr, *d_state_off = nullptr, *d_Sk_off = nullptr;
  int32_t* d_inst_model = nullptr;
  fdtd::RomModelDev* d_models = nullptr;
  int64_t state_len = 0;
  // graphs
  cudaGraphExec_t gexec = nullptr;
  bool graph_dirty = true;
  int graph_steps = 0;
  int64_t graph_launches = 0;
  int64_t graph_builds = 0;
  bool graph_broken = false;
  int64_t launches = 0;
  // profiling (event pairs around each launch)
  bool profiling = false;
  std::vector<cudaEvent_t> ev;
  size_t ev_used = 0;
  // multi-rank
  nccl_comm comm = nullptr;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_ready = nullptr, ev_halo = nullptr;
  double* d_level2 = nullptr;  // [KMAX][FIN_GRID]
  // row slabs: the slab-edge row chunks run on a side stream beside the interior chunks
  cudaStream_t edge_stream = nullptr;
  cudaEvent_t ev_edge_go = nullptr, ev_edge = nullptr;
  std::vector<void*> owned;  // every device allocation
};

namespace {

fdtd_status fail(fdtd_ctx* c, fdtd_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return s;
}

#define CK(call)                                                                             \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess) return fail(c, FDTD_E_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

#define NK(call)                                                                         \
  do {                                                                                   \
    int r_ = (call);                                                                     \
    if (r_ != 0) return fail(c, FDTD_E_NCCL, "%s: %s", #call, g_nccl.GetErrorString(r_)); \
  } while (0)

void* dalloc(fdtd_ctx* c, size_t bytes) {
  if (bytes == 0) bytes = 16;
  void* p = nullptr;
  if (c->d.alloc) {
    p = c->d.alloc(bytes, c->d.alloc_user);
  } else if (cudaMalloc(&p, bytes) != cudaSuccess) {
    p = nullptr;
  }
  if (p) {
    c->owned.push_back(p);
    if (cudaMemsetAsync(p, 0, bytes, c->stream) != cudaSuccess) return nullptr;
  }
  return p;
}

void dfree(fdtd_ctx* c, void* p) {
  if (!p) return;
  auto it = std::find(c->owned.begin(), c->owned.end(), p);
  if (it != c->owned.end()) c->owned.erase(it);
  if (c->d.free) c->d.free(p, c->d.alloc_user);
  else cudaFree(p);
}

template <typename X>
fdtd_status upload(fdtd_ctx* c, X** dst, const std::vector<X>& v) {
  if (*dst) { dfree(c, *dst); *dst = nullptr; }
  *dst = static_cast<X*>(dalloc(c, v.size() * sizeof(X)));
  if (!*dst) return fail(c, FDTD_E_NOMEM, "device allocation of %zu bytes failed", v.size() * sizeof(X));
  if (!v.empty()) CK(cudaMemcpyAsync(*dst, v.data(), v.size() * sizeof(X), cudaMemcpyHostToDevice, c->stream));
  return FDTD_OK;
}

// upload an fp64 host vector converted to the storage precision
fdtd_status upload_T(fdtd_ctx* c, void** dst, const std::vector<double>& v) {
  if (c->prec == 64) return upload(c, reinterpret_cast<double**>(dst), v);
  std::vector<float> f(v.begin(), v.end());
  return upload(c, reinterpret_cast<float**>(dst), f);
}

inline int64_t lrow(const fdtd_ctx* c, int64_t g) { return g - c->d.row_begin + ROW0; }
constexpr size_t ARRAY_TAIL = 32 * 1024;  // bytes past the last row of every field / material array
inline int64_t alloc_elems(const fdtd_ctx* c) { return c->nrows_alloc * c->pitch + (int64_t)(ARRAY_TAIL / c->es); }

template <typename T>
fdtd::SweepParams<T> sweep_params(fdtd_ctx* c, int q) {
  fdtd::SweepParams<T> p{};
  p.ex0 = (const T*)c->f[q][0]; p.ey0 = (const T*)c->f[q][1]; p.hz0 = (const T*)c->f[q][2];
  p.ex1 = (T*)c->f[1 - q][0]; p.ey1 = (T*)c->f[1 - q][1]; p.hz1 = (T*)c->f[1 - q][2];
  p.mea = (const T*)c->coef[0]; p.msb = (const T*)c->coef[1];
  p.pitch = c->pitch; p.nx = c->d.nx; p.rows = c->rows; p.chunk = c->chunk; p.row0 = ROW0;
  p.chx = (T)(c->d.dt / (MU0 * c->d.dx));
  p.chy = (T)(c->d.dt / (MU0 * c->d.dy));
  // source rows clipped to this slab +- KMAX (the chunks next to the slab edges recompute up to KMAX
  // ghost rows, adding the source as its owner does)
  const int64_t sj0 = std::max(c->src_j, c->d.row_begin - KMAX), sj1 = std::min(c->src_j1, c->d.row_end + KMAX);
  const bool src_here = c->d_src && sj0 < sj1;
  p.src_row = src_here ? (int)lrow(c, sj0) : -1;
  p.src_row_end = src_here ? (int)lrow(c, sj1) : -1;
  p.src_col = src_here ? c->src_i : -1;
  p.src_samples = c->d_src; p.src_meta = c->d_src_meta;
  p.step = c->d_step;
  p.partials = c->energy_on ? c->d_partials : nullptr;
  p.pstride = c->n_partials;
  p.probe_rows = c->d_probe_rows; p.probe_list = c->d_probe_list;
  p.probe_ring = (T*)c->d_probe_ring; p.cap = c->cap;
  p.idx = (T)(1.0 / c->d.dx); p.idy = (T)(1.0 / c->d.dy);
  p.wxy = (T)(c->d.dx * c->d.dy);
  p.wh = (T)(MU0 * c->d.dx * c->d.dy / c->d.dt);
  p.naf = p.nam = 1;
  p.alloc_elems_f = p.alloc_elems_m = alloc_elems(c);
  return p;
}

int sweep_gx(const fdtd_ctx* c, int K) { return fdtd::sweep_ctas_x(c->d.nx, (int)c->es, K, c->warps); }
int sweep_gx_max(const fdtd_ctx* c) {
  int g = 1;
  for (int K = 1; K <= KMAX; K *= 2) g = std::max(g, sweep_gx(c, K));
  return g;
}

template <typename T>
fdtd::PostParams<T> post_params(fdtd_ctx* c, int q) {
  fdtd::PostParams<T> p{};
  p.n_inst = (int)c->inst_model.size();
  p.models = c->d_models; p.mpool = (const double*)c->d_mpool;
  p.Sk = (const T*)c->d_Sk; p.Sk_off = c->d_Sk_off; p.port_off = c->d_port_off;
  p.cya = (const T*)c->d_cya; p.cyg = (const T*)c->d_cyg; p.ehalf = c->d_ehalf;
  p.port_edge = c->d_port_edge;
  p.state = (T*)c->d_state; p.state_off = c->d_state_off;
  p.ex1 = (T*)c->f[1 - q][0]; p.ey1 = (T*)c->f[1 - q][1]; p.hz1 = (T*)c->f[1 - q][2];
  p.ex0 = (const T*)c->f[q][0]; p.ey0 = (const T*)c->f[q][1]; p.hz0 = (const T*)c->f[q][2];
  p.mea = (const T*)c->coef[0]; p.msb = (const T*)c->coef[1];
  p.pitch = c->pitch; p.row_begin = c->d.row_begin; p.row0 = ROW0;
  p.Kz = c->kz;
  p.rects = c->d_rects;
  p.zp_off = c->d_zp_off; p.zp = c->d_zp;
  p.probe_ring = (T*)c->d_probe_ring; p.cap = c->cap;
  p.chx = (T)(c->d.dt / (MU0 * c->d.dx));
  p.chy = (T)(c->d.dt / (MU0 * c->d.dy));
  p.idx = (T)(1.0 / c->d.dx); p.idy = (T)(1.0 / c->d.dy);
  p.wxy = (T)(c->d.dx * c->d.dy);
  p.wh = (T)(MU0 * c->d.dx * c->d.dy / c->d.dt);
  // source rows clipped to this slab +- KMAX (the chunks next to the slab edges recompute up to KMAX
  // ghost rows, adding the source as its owner does)
  const int64_t sj0 = std::max(c->src_j, c->d.row_begin - KMAX), sj1 = std::min(c->src_j1, c->d.row_end + KMAX);
  const bool src_here = c->d_src && sj0 < sj1;
  p.src_row = src_here ? (int)lrow(c, sj0) : -1;
  p.src_row_end = src_here ? (int)lrow(c, sj1) : -1;
  p.src_col = src_here ? c->src_i : -1;
  p.src_samples = c->d_src; p.src_meta = c->d_src_meta;
  p.rom_partials = c->d_rom_partials;
  p.level1 = c->d_level1;
  p.step = c->d_step;
  p.n_batch = c->inst_model.empty() ? 0 : (int)(c->batch_tab.size() / fdtd::BATCH_FIELDS);
  p.n_batch_reg = c->inst_model.empty() ? 0 : c->n_batch_reg;
  p.big = (T*)c->d_big; p.big_smem_bytes = c->big_smem; p.big_grid = c->big_grid;
  p.batch_tab = c->d_batch_tab;
  p.batch_inst = c->d_batch_inst;
  p.batch_rect = c->d_batch_rect;
  p.nx = c->d.nx;
  p.ny = c->d.ny;
  p.block = c->post_threads;
  p.smem_bytes = c->post_smem;
  p.flag = c->d_flag;
  p.alloc_elems = alloc_elems(c); p.rows = c->rows; p.n_probe = c->n_probe;
  p.energy_ring = c->d_energy_ring;
  p.wprobe = c->d_wprobe; p.n_wprobe = c->n_wprobe;
  if (c->whole) {  // the whole-grid batch
    p.batch_tab = c->d_wb_tab; p.batch_inst = c->d_wb_inst; p.batch_rect = c->d_wb_rect;
    p.n_batch = p.n_batch_reg = 1;
    p.smem_bytes = c->whole_smem;
    p.whole_coef = c->whole_coef ? 1 : 0;
  }
  return p;
}

// CPML state buffer q (0/1) of psi_hz (e = 0: w columns per row) or psi_ey (e = 1: w + 1 columns),
// both sides: [buffer][side][row][column]
inline char* psi_base(const fdtd_ctx* c, int e, int q, int side) {
  const int64_t rw = e ? c->pml_w + 1 : c->pml_w;
  return (char*)(e ? c->d_psie : c->d_psih) + (size_t)((2 * q + side) * c->nrows_alloc * rw) * c->es;
}
template <typename T>
T* psi_buf(const fdtd_ctx* c, int e, int q) { return (T*)psi_base(c, e, q, 0); }

fdtd::FinParams fin_params(fdtd_ctx* c, int K, int q) {
  fdtd::FinParams f{};
  f.sweep_partials = c->d_partials;  // exactly the partials the matching sweep / band launches wrote
  f.n_sweep_partials = (int64_t)sweep_gx(c, K) * ((c->rows + c->chunk - 1) / c->chunk) +
                       (c->pml_w > 0 ? fdtd::pml_ctas(c->rows, PML_CHUNK) : 0);  // + the CPML band CTAs
  f.pstride = c->n_partials;
  f.rom_level1 = c->d_level1;
  f.n_rom = c->inst_model.empty() ? 0 : (int)(c->batch_tab.size() / fdtd::BATCH_FIELDS);
  f.level2 = c->d_level2;
  f.energy_ring = c->d_energy_ring; f.cap = c->cap;
  f.step = c->d_step; f.done = c->d_done;
  f.K = K; f.energy = c->energy_on;
  f.hz = c->f[1 - q][2]; f.pitch = c->pitch; f.nx = c->d.nx; f.row0 = ROW0; f.rows = c->rows; f.es = (int)c->es;
  f.flag = c->d_flag;
  return f;
}

template <typename T>
fdtd::PmlParams<T> pml_params(fdtd_ctx* c, int q) {
  fdtd::PmlParams<T> p{};
  p.ex0 = (const T*)c->f[q][0]; p.ey0 = (const T*)c->f[q][1]; p.hz0 = (const T*)c->f[q][2];
  p.ex1 = (T*)c->f[1 - q][0]; p.ey1 = (T*)c->f[1 - q][1]; p.hz1 = (T*)c->f[1 - q][2];
  p.mea = (const T*)c->coef[0]; p.msb = (const T*)c->coef[1];
  p.pitch = c->pitch; p.nx = c->d.nx; p.rows = c->rows; p.row0 = ROW0; p.chunk = PML_CHUNK;
  p.w = c->pml_w; p.Kz = c->kz;
  p.bh = (const T*)c->d_pml_bh; p.ah = (const T*)c->d_pml_ah; p.be = (const T*)c->d_pml_be; p.ae = (const T*)c->d_pml_ae;
  p.psih = psi_buf<T>(c, 0, q); p.psie = psi_buf<T>(c, 1, q);
  p.psih1 = psi_buf<T>(c, 0, 1 - q); p.psie1 = psi_buf<T>(c, 1, 1 - q);
  p.psi_rows = c->nrows_alloc;
  p.chx = (T)(c->d.dt / (MU0 * c->d.dx));
  p.chy = (T)(c->d.dt / (MU0 * c->d.dy));
  p.idx = (T)(1.0 / c->d.dx); p.idy = (T)(1.0 / c->d.dy);
  p.wxy = (T)(c->d.dx * c->d.dy);
  p.wh = (T)(MU0 * c->d.dx * c->d.dy / c->d.dt);
  p.cpsi = (T)(c->d.dt / MU0);
  p.dxv = (T)c->d.dx;
  const int64_t sj0 = std::max(c->src_j, c->d.row_begin - KMAX), sj1 = std::min(c->src_j1, c->d.row_end + KMAX);
  const bool src_here = c->d_src && sj0 < sj1;
  p.src_row = src_here ? (int)lrow(c, sj0) : -1;
  p.src_row_end = src_here ? (int)lrow(c, sj1) : -1;
  p.src_col = src_here ? c->src_i : -1;
  p.src_samples = c->d_src; p.src_meta = c->d_src_meta;
  p.step = c->d_step;
  p.n_probe = c->d_probe_gi ? c->n_probe : 0;
  p.probe_gi = c->d_probe_gi; p.probe_lr = c->d_probe_lr; p.probe_ring = (T*)c->d_probe_ring; p.cap = c->cap;
  p.partials = c->energy_on ? c->d_partials : nullptr;
  p.pstride = c->n_partials;
  p.alloc_elems = alloc_elems(c);
  return p;
}

// Halo plan of a K-step pass: rank g owns cell rows and Ex edge rows
// [row_begin, row_end).  Its sweep reads rows [row_begin - K, row_end + K): all three fields of
// the K rows below (the top K rows of rank g-1), Ex of the K edge rows above and Ey / Hz of the
// K-1 cell rows above (the bottom rows of rank g+1).  Rows are whole device rows (pitch
// elements); sends and receives are listed in the order both transports pair them.
// With CPML layers (NEXT-2) the psi rows travel with the field they belong to: psi_ey (a = 3, 4:
// left / right side) with Ey, psi_hz (a = 5, 6) with Hz.
struct HaloRow { int a; int64_t row; int peer; };
void halo_plan_rows(int nranks, int rank, int64_t rows, int depth, bool pml, std::vector<HaloRow>& sends,
                    std::vector<HaloRow>& recvs) {
  sends.clear();
  recvs.clear();
  const int up = rank + 1, dn = rank - 1;
  const int64_t top = ROW0 + rows;  // first row above the slab
  auto push = [&](std::vector<HaloRow>& v, int a, int64_t r, int peer) {
    v.push_back({a, r, peer});
    if (pml && a == 1) { v.push_back({3, r, peer}); v.push_back({4, r, peer}); }
    if (pml && a == 2) { v.push_back({5, r, peer}); v.push_back({6, r, peer}); }
  };
  auto down_list = [&](int64_t base, int peer, std::vector<HaloRow>& v) {  // rows the lower rank needs
    for (int64_t r = 0; r < depth; ++r) {
      push(v, 0, base + r, peer);
      if (r + 1 < depth) {
        push(v, 1, base + r, peer);
        push(v, 2, base + r, peer);
      }
    }
  };
  if (up < nranks) {
    for (int64_t r = top - depth; r < top; ++r)
      for (int a = 0; a < 3; ++a) push(sends, a, r, up);
    down_list(top, up, recvs);  // rows above the slab come from rank g+1's bottom rows
  }
  if (dn >= 0) {
    for (int64_t r = ROW0 - depth; r < ROW0; ++r)
      for (int a = 0; a < 3; ++a) push(recvs, a, r, dn);
    down_list(ROW0, dn, sends);
  }
}
void halo_plan(const fdtd_ctx* c, int depth, std::vector<HaloRow>& sends, std::vector<HaloRow>& recvs) {
  halo_plan_rows(c->d.nranks, c->d.rank, c->rows, depth, c->pml_w > 0, sends, recvs);
}

// device address and element count of halo row (a, r) of buffer q
inline char* dev_row(const fdtd_ctx* c, int q, int a, int64_t r) {
  if (a < 3) return (char*)c->f[q][a] + (size_t)r * c->pitch * c->es;
  const int e = a < 5 ? 1 : 0, side = (a - 3) & 1;
  const int64_t rw = e ? c->pml_w + 1 : c->pml_w;
  return psi_base(c, e, q, side) + (size_t)(r * rw) * c->es;
}
inline size_t row_elems(const fdtd_ctx* c, int a) {
  return a < 3 ? (size_t)c->pitch : (size_t)(a < 5 ? c->pml_w + 1 : c->pml_w);
}

fdtd_status halo_exchange(fdtd_ctx* c, int q, cudaStream_t s, int depth) {
  if (c->d.nranks <= 1 || (c->d.flags & FDTD_LOCAL_GROUP)) return FDTD_OK;
  const int dt = c->prec == 64 ? NCCL_F64 : NCCL_F32;
  std::vector<HaloRow> sends, recvs;
  halo_plan(c, depth, sends, recvs);
  NK(g_nccl.GroupStart());
  for (auto& x : sends) NK(g_nccl.Send(dev_row(c, q, x.a, x.row), row_elems(c, x.a), dt, x.peer, c->comm, s));
  for (auto& x : recvs) NK(g_nccl.Recv(dev_row(c, q, x.a, x.row), row_elems(c, x.a), dt, x.peer, c->comm, s));
  NK(g_nccl.GroupEnd());
  return FDTD_OK;
}

// Local transport for an in-process group: every receive pairs with the peer's sends to this
// rank in plan order (the same pairing NCCL applies).
fdtd_status halo_local(fdtd_ctx* const* g, int n, int k, int q, cudaStream_t s, int depth) {
  fdtd_ctx* c = g[k];
  std::vector<HaloRow> sends, recvs, psends, precvs;
  halo_plan(c, depth, sends, recvs);
  for (int peer = 0; peer < n; ++peer) {
    if (peer == k) continue;
    halo_plan(g[peer], depth, psends, precvs);
    std::vector<HaloRow> in, out;
    for (auto& x : recvs) if (x.peer == peer) in.push_back(x);
    for (auto& x : psends) if (x.peer == k) out.push_back(x);
    if (in.size() != out.size()) return fail(c, FDTD_E_STATE, "halo plans of ranks %d and %d do not pair", k, peer);
    for (size_t i = 0; i < in.size(); ++i) {
      if (in[i].a != out[i].a) return fail(c, FDTD_E_STATE, "halo plans of ranks %d and %d do not pair", k, peer);
      CK(cudaMemcpyAsync(dev_row(c, q, in[i].a, in[i].row), dev_row(g[peer], q, out[i].a, out[i].row),
                         row_elems(c, in[i].a) * c->es, cudaMemcpyDeviceToDevice, s));
    }
  }
  return FDTD_OK;
}

cudaEvent_t next_event(fdtd_ctx* c) {
  if (c->ev_used == c->ev.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->ev.push_back(e);
  }
  return c->ev[c->ev_used++];
}

// One pass of K time steps (K1 sweep q -> 1-q, then the K3 fix-up).  With several ranks the sweep
// is split: the interior row chunks (which read no ghost row) run on the compute stream while the
// NCCL halo exchange runs on a side stream; the chunks next to the slab edges follow once the
// ghost rows have arrived.
fdtd_status enqueue_pass(fdtd_ctx* c, int q, cudaStream_t s, int K) {
  const bool prof = c->profiling && s == c->stream;
  const int nch = (c->rows + c->chunk - 1) / c->chunk;
  // chunks [lo, hi) read only owned rows: a chunk reads rows [r0 - K, r1 + K)
  int lo = 0, hi = nch;
  while (lo < nch && lo * c->chunk - K < 0) ++lo;
  while (hi > lo && std::min((hi) * c->chunk, c->rows) + K > c->rows) --hi;
  const bool split = c->d.nranks > 1 && hi > lo;
  const bool nccl_overlap = split && c->comm && c->comm_stream;
  auto sweep_on = [&](int b, int n, cudaStream_t st) {
    if (n <= 0) return;
    if (c->prec == 64) fdtd::launch_sweep<double>(sweep_params<double>(c, q), K, c->warps, st, b, n);
    else fdtd::launch_sweep<float>(sweep_params<float>(c, q), K, c->warps, st, b, n);
    c->launches += 1;
  };
  auto sweep = [&](int b, int n) { sweep_on(b, n, s); };
  // the chunk rows next to the slab edges (one or two chunk rows: a fraction of a wave) run on a
  // side stream once their ghost rows are in, beside the interior launch, whose tail they fill
  // instead of idling the GPU after it
  auto edges_beside = [&](cudaEvent_t ready) -> fdtd_status {
    CK(cudaStreamWaitEvent(c->edge_stream, ready, 0));
    sweep_on(0, lo, c->edge_stream);
    sweep_on(hi, nch - hi, c->edge_stream);
    CK(cudaEventRecord(c->ev_edge, c->edge_stream));
    return FDTD_OK;
  };
  const bool has_fix = !c->inst_model.empty();
  auto post = [&](cudaStream_t st) {
    if (c->prec == 64) fdtd::launch_post<double>(post_params<double>(c, q), K, c->energy_on, st);
    else fdtd::launch_post<float>(post_params<float>(c, q), K, c->energy_on, st);
    c->launches += c->n_batch_reg > 0;
    if ((int)(c->batch_tab.size() / fdtd::BATCH_FIELDS) > c->n_batch_reg) {  // large models: the cooperative fix-up
      if (c->prec == 64) fdtd::launch_post_big<double>(post_params<double>(c, q), K, c->energy_on, st);
      else fdtd::launch_post_big<float>(post_params<float>(c, q), K, c->energy_on, st);
      c->launches += 1;
    }
  };
  cudaEvent_t e[3];
  if (prof) {
    for (auto& x : e) x = next_event(c);
    CK(cudaEventRecord(e[0], s));
  }
  if (nccl_overlap) {
    CK(cudaEventRecord(c->ev_ready, s));
    CK(cudaStreamWaitEvent(c->comm_stream, c->ev_ready, 0));
    fdtd_status st = halo_exchange(c, q, c->comm_stream, K);
    if (st != FDTD_OK) return st;
    CK(cudaEventRecord(c->ev_halo, c->comm_stream));
    sweep(lo, hi - lo);  // interior chunks: no ghost rows needed
    if (c->edge_stream) {
      fdtd_status st2 = edges_beside(c->ev_halo);
      if (st2 != FDTD_OK) return st2;
      CK(cudaStreamWaitEvent(s, c->ev_edge, 0));
      CK(cudaStreamWaitEvent(s, c->ev_halo, 0));  // join the comm stream too (graph capture)
    } else {
      CK(cudaStreamWaitEvent(s, c->ev_halo, 0));
      sweep(0, lo);
      sweep(hi, nch - hi);
    }
  } else {
    fdtd_status st = halo_exchange(c, q, s, K);
    if (st != FDTD_OK) return st;
    if (split) {  // local groups: same split launches (their halo copies precede on this stream)
      if (c->edge_stream) {
        CK(cudaEventRecord(c->ev_edge_go, s));
        sweep(lo, hi - lo);
        fdtd_status st2 = edges_beside(c->ev_edge_go);
        if (st2 != FDTD_OK) return st2;
        CK(cudaStreamWaitEvent(s, c->ev_edge, 0));
      } else {
        sweep(lo, hi - lo);
        sweep(0, lo);
        sweep(hi, nch - hi);
      }
    } else {
      sweep(0, nch);
    }
  }
  if (c->pml_w > 0) {  // NEXT-2: CPML bands (their energy partials follow the sweep's)
    const int64_t poff = (int64_t)sweep_gx(c, K) * nch;
    if (c->prec == 64) {
      auto pp = pml_params<double>(c, q);
      pp.poff = poff;
      fdtd::launch_pml<double>(pp, K, c->energy_on, s);
    } else {
      auto pp = pml_params<float>(c, q);
      pp.poff = poff;
      fdtd::launch_pml<float>(pp, K, c->energy_on, s);
    }
    c->launches += 1;
  }
  if (prof) CK(cudaEventRecord(e[1], s));
  if (has_fix) post(s);
  fdtd::launch_finalize(fin_params(c, K, q), s);  // energy of the K steps, step counter
  c->launches += 1;
  if (prof) CK(cudaEventRecord(e[2], s));
  return FDTD_OK;
}

void drop_graph(fdtd_ctx* c) {
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  c->gexec = nullptr;
  c->graph_dirty = true;
}

// Captures one "period" starting from buffer 0: two K-step passes (0 -> 1 -> 0).
fdtd_status build_graph(fdtd_ctx* c) {
  drop_graph(c);
  if (!c->cap_stream) CK(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal));
  const int64_t before = c->launches;
  fdtd_status st = enqueue_pass(c, 0, c->cap_stream, c->kz);
  if (st == FDTD_OK) st = enqueue_pass(c, 1, c->cap_stream, c->kz);
  c->graph_launches = c->launches - before;
  c->launches = before;
  cudaError_t e = cudaStreamEndCapture(c->cap_stream, &g);
  if (st != FDTD_OK) return st;
  if (e != cudaSuccess) return fail(c, FDTD_E_CUDA, "graph capture: %s", cudaGetErrorString(e));
  e = cudaGraphInstantiate(&c->gexec, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return fail(c, FDTD_E_CUDA, "graph instantiate: %s", cudaGetErrorString(e));
  c->graph_steps = 2 * c->kz;
  c->graph_dirty = false;
  c->graph_builds += 1;
  return FDTD_OK;
}

// Synchronous point: CUDA faults, then the non-finite sentinel (include/fdtdrom.h "Errors").
// collective: with NCCL ranks the sentinel is first max-reduced over ranks, so that every rank
// of a collective read (fdtd_probe, fdtd_energy) fails together instead of one rank leaving the
// records' all-reduce.
fdtd_status check_async(fdtd_ctx* c, bool collective = false) {
  if (collective && c->d.nranks > 1 && c->comm)
    NK(g_nccl.AllReduce(c->d_flag, c->d_flag, 1, NCCL_I32, NCCL_MAX, c->comm, c->stream));
  int flag = 0;
  CK(cudaMemcpyAsync(&flag, c->d_flag, sizeof flag, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaGetLastError());
  if (flag)
    return fail(c, FDTD_E_UNSTABLE, "non-finite field or ROM state detected (by step %lld): the scheme is unstable at "
                "dt = %g", (long long)c->steps, c->d.dt);
  return FDTD_OK;
}

template <typename M>
fdtd_status build_coefficients(fdtd_ctx* c) {
  const M* e = (const M*)c->mat_eps;
  const M* s = (const M*)c->mat_sig;
  if (c->prec == 64)
    fdtd::launch_materials<double, M>(e, s, c->mrow0, c->mrow_end, c->d.nx, c->d.ny, c->d.row_begin, ROW0, (int)c->nrows_alloc, c->pitch, c->d.dt,
                                      (double*)c->coef[0], (double*)c->coef[1], c->stream);
  else
    fdtd::launch_materials<float, M>(e, s, c->mrow0, c->mrow_end, c->d.nx, c->d.ny, c->d.row_begin, ROW0, (int)c->nrows_alloc, c->pitch, c->d.dt,
                                     (float*)c->coef[0], (float*)c->coef[1], c->stream);
  CK(cudaGetLastError());
  return FDTD_OK;
}

fdtd_status gather_materials(fdtd_ctx* c, const std::vector<int64_t>& cells, std::vector<double>& eps,
                             std::vector<double>& sig) {
  const int64_t n = (int64_t)cells.size();
  eps.assign(n, 0.0);
  sig.assign(n, 0.0);
  if (n == 0) return FDTD_OK;
  int64_t* dc = nullptr;
  fdtd_status st = upload(c, &dc, cells);
  if (st != FDTD_OK) return st;
  double* de = (double*)dalloc(c, n * sizeof(double));
  double* ds = (double*)dalloc(c, n * sizeof(double));
  if (!de || !ds) return fail(c, FDTD_E_NOMEM, "gather buffers");
  if (c->mat_f32)
    fdtd::launch_gather_materials<float>((const float*)c->mat_eps, (const float*)c->mat_sig, c->d.nx, c->mrow0, dc,
                                         n, de, ds, c->stream);
  else
    fdtd::launch_gather_materials<double>((const double*)c->mat_eps, (const double*)c->mat_sig, c->d.nx, c->mrow0,
                                          dc, n, de, ds, c->stream);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(eps.data(), de, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(sig.data(), ds, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  dfree(c, dc);
  dfree(c, de);
  dfree(c, ds);
  return FDTD_OK;
}

fdtd_status upload_roms(fdtd_ctx* c) {
  fdtd_status st;
  std::vector<fdtd::RomModelDev> md;
  for (auto& m : c->models) md.push_back(m.dev);
  if ((st = upload(c, reinterpret_cast<double**>(&c->d_mpool), c->mpool)) != FDTD_OK) return st;
  if ((st = upload(c, &c->d_models, md)) != FDTD_OK) return st;
  if ((st = upload(c, &c->d_rects, c->rects)) != FDTD_OK) return st;
  if ((st = upload_T(c, &c->d_Sk, c->Sk)) != FDTD_OK) return st;
  if ((st = upload(c, &c->d_Sk_off, c->Sk_off)) != FDTD_OK) return st;
  if ((st = upload(c, &c->d_port_off, c->port_off)) != FDTD_OK) return st;
  if ((st = upload_T(c, &c->d_cya, c->cya)) != FDTD_OK) return st;
  if ((st = upload_T(c, &c->d_cyg, c->cyg)) != FDTD_OK) return st;
  if ((st = upload(c, &c->d_ehalf, c->ehalf)) != FDTD_OK) return st;
  if ((st = upload(c, &c->d_port_edge, c->port_edge)) != FDTD_OK) return st;
  if ((st = upload(c, &c->d_state_off, c->state_off)) != FDTD_OK) return st;
  // ROM states start at zero (R26: x~0 = 0 with y0 = 0 on the freshly zeroed interface edges)
  std::vector<double> zero(c->state_len, 0.0);
  void* prev = c->d_state;
  c->d_state = nullptr;
  if ((st = upload_T(c, &c->d_state, zero)) != FDTD_OK) return st;
  if (prev) dfree(c, prev);
  std::vector<double> zp((size_t)KMAX * (c->inst_model.size() + 1), 0.0);
  if ((st = upload(c, &c->d_rom_partials, zp)) != FDTD_OK) return st;
  c->kz_dirty = true;
  return FDTD_OK;
}

// The fix-up regions of a K-step pass: instances whose (block + K)
// rectangles meet, directly or through others, share one region -- their bounding box plus the
// margin -- and are fixed up together by one CTA (a "cluster"); every other instance has its own.
// Two regions' (block + K) boxes never meet, so no fix-up needs another's ROM within the K steps.
struct PassRegion {
  int model = -1;
  bool mixed = false;            // members of different models (not supported: a shallower pass)
  std::vector<int> members;      // instance indices, ascending
  int64_t i0 = 0, j0 = 0, i1 = 0, j1 = 0;  // bounding box of the blocks [i0, i1) x [j0, j1)
};

std::vector<PassRegion> pass_regions_of(const std::vector<int32_t>& rects, const std::vector<int32_t>& inst_model,
                                        int K) {
  // Start from one region per instance and merge any two regions whose boxes, grown by K, meet --
  // with the merged (bounding) boxes, until no pair meets: then no region's box + 2K - 1 reaches
  // into another region, whatever the shape of a cluster.
  const int n = (int)inst_model.size();
  std::vector<PassRegion> cur(n);
  for (int i = 0; i < n; ++i) {
    PassRegion& g = cur[i];
    g.model = inst_model[i];
    g.members = {i};
    g.i0 = rects[4 * i]; g.j0 = rects[4 * i + 1];
    g.i1 = g.i0 + rects[4 * i + 2]; g.j1 = g.j0 + rects[4 * i + 3];
  }
  if (K < 2) return cur;
  for (bool merged = true; merged;) {
    merged = false;
    const int m = (int)cur.size();
    std::vector<int> ord(m), par(m);
    for (int i = 0; i < m; ++i) ord[i] = par[i] = i;
    std::function<int(int)> find = [&](int x) { return par[x] == x ? x : par[x] = find(par[x]); };
    std::sort(ord.begin(), ord.end(), [&](int a, int b) { return cur[a].i0 < cur[b].i0; });
    int64_t wmax = 0;
    for (const PassRegion& g : cur) wmax = std::max(wmax, g.i1 - g.i0);
    for (int a = 0; a < m; ++a)
      for (int b = a + 1; b < m && cur[ord[b]].i0 <= cur[ord[a]].i1 + wmax + 2 * K; ++b) {
        const PassRegion &A = cur[ord[a]], &Bq = cur[ord[b]];
        const bool ox = A.i0 - K < Bq.i1 + K && Bq.i0 - K < A.i1 + K;
        const bool oy = A.j0 - K < Bq.j1 + K && Bq.j0 - K < A.j1 + K;
        if (ox && oy && find(ord[a]) != find(ord[b])) {
          par[find(ord[a])] = find(ord[b]);
          merged = true;
        }
      }
    if (!merged) break;
    std::vector<PassRegion> next;
    std::vector<int> slot(m, -1);
    for (int i = 0; i < m; ++i) {  // in instance order of the first members
      const int r = find(i);
      if (slot[r] < 0) {
        slot[r] = (int)next.size();
        next.push_back(cur[i]);
        continue;
      }
      PassRegion& g = next[slot[r]];
      g.mixed |= cur[i].mixed || g.model != cur[i].model;
      g.i0 = std::min(g.i0, cur[i].i0); g.j0 = std::min(g.j0, cur[i].j0);
      g.i1 = std::max(g.i1, cur[i].i1); g.j1 = std::max(g.j1, cur[i].j1);
      g.members.insert(g.members.end(), cur[i].members.begin(), cur[i].members.end());
    }
    for (PassRegion& g : next) std::sort(g.members.begin(), g.members.end());
    cur.swap(next);
  }
  return cur;
}
std::vector<PassRegion> pass_regions(const fdtd_ctx* c, int K) { return pass_regions_of(c->rects, c->inst_model, K); }

// shared memory of one fix-up batch: B member slots of model m's vectors plus nreg regions of
// stride rs
size_t batch_smem(const fdtd_ctx* c, const ModelHost& m, int B, int nreg, int rs) {
  return fdtd::post_smem_bytes(c->es, m.q1 + m.q2 + m.nY, m.nY, B, 0) + (size_t)nreg * rs * c->es;
}
constexpr size_t FIX_BUDGET = 220 * 1024;  // one 512-thread fix-up CTA per SM
constexpr int MAX_CLUSTER = 64;            // fdtd_kernels.cu MAXB

// Can this rank run K-step passes (K3)?  Every fix-up region (block or cluster box +
// 2K-1 cells) must lie inside this slab's rows wherever a neighbouring slab continues the grid
// (beyond the PEC walls the region holds dead cells), a cluster must hold instances of one model
// only, and its batch must fit the fix-up's shared memory.
bool passes_valid(const fdtd_ctx* c, int K) {
  if (K > c->V) return false;  // a halo lane of V columns covers at most V steps of error spread
  const int64_t M = 2 * K - 1;
  if (c->pml_w > 0) {  // ROM rings 2K + 1 cells clear of the CPML layers: neither fix-up then sees the
                       // other's physics within the K steps (the band region may hold ROM edges it never
                       // updates, the ROM region no layer cell)
    const int64_t WB = c->pml_w + 2 * K + 2;
    if (2 * WB > c->d.nx) return false;
    for (size_t r = 0; r < c->rects.size(); r += 4)
      if (c->rects[r] - 1 < c->pml_w + 2 * K + 1 || c->rects[r] + c->rects[r + 2] + 1 > c->d.nx - c->pml_w - 2 * K - 1)
        return false;
  }
  if (K == 1) return true;
  for (const PassRegion& g : pass_regions(c, K)) {
    if (g.mixed || (int)g.members.size() > MAX_CLUSTER) return false;
    if ((g.j0 - M < c->d.row_begin && c->d.row_begin > 0) || (g.j1 + M > c->d.row_end && c->d.row_end < c->d.ny))
      return false;
    if (g.members.size() > 1) {
      const ModelHost& m = c->models[g.model];
      const int rs = (fdtd::region_elems((int)(g.i1 - g.i0), (int)(g.j1 - g.j0), (int)M) + 3) / 4 * 4;
      if (batch_smem(c, m, (int)g.members.size(), 1, rs) > FIX_BUDGET) return false;
    }
  }
  return true;
}

fdtd_status apply_passes(fdtd_ctx* c, int k);

// Append a row-major (rows x cols) operator to the fp64 pool in the A-fragment order of
// mma.sync.m8n8k4.f64 (fdtd_kernels.cu dmma_gemm): per 8 x 4 tile (row tile mt, column tile kt, kt
// fastest) lane l holds A[8 mt + l / 4][4 kt + l % 4]; zero padding outside rows x cols.
int64_t push_tiles(std::vector<double>& pool, const std::vector<double>& A, int rows, int cols, int& mt, int& kt) {
  while (pool.size() % 32) pool.push_back(0.0);  // 256-byte aligned tiles
  const int64_t off = (int64_t)pool.size();
  mt = (rows + 7) / 8;
  kt = (cols + 3) / 4;
  for (int a = 0; a < mt; ++a)
    for (int b = 0; b < kt; ++b)
      for (int l = 0; l < 32; ++l) {
        const int r = 8 * a + l / 4, cc = 4 * b + l % 4;
        pool.push_back(r < rows && cc < cols ? A[(size_t)r * cols + cc] : 0.0);
      }
  return off;
}

// Zone depth, zone marks, fix-up batches and zone probes for passes of depth kz (all ranks agree
// on kz: one NCCL min-reduction).  Runs at the first fdtd_step after a configuration change.
fdtd_status configure_passes(fdtd_ctx* c) {
  if (!c->kz_dirty) return FDTD_OK;
  int want = std::max(1, std::min(c->k_want, c->V));
  int k = want >= 4 ? 4 : want >= 2 ? 2 : 1;
  while (k > 1 && !passes_valid(c, k)) k /= 2;
  // the fix-up kernel's shared memory: regions of margin 2k-1 plus the ROM vectors of a batch
  auto stride_for = [&](int kk) {
    int rs = 4;
    for (auto& m : c->models) rs = std::max(rs, fdtd::region_elems(m.bx, m.by, 2 * kk - 1));
    return (rs + 3) / 4 * 4;
  };
  auto fits = [&](int b, int rs, size_t lim) { return fdtd::post_smem_bytes(c->es, c->nvec, c->nvec, b, rs) <= lim; };
  while (k > 1 && !fits(1, stride_for(k), 220 * 1024)) k /= 2;
  c->k_ok = k;
  if (c->d.nranks > 1 && c->comm) {  // collective min over ranks (all ranks reach this call together)
    int32_t* d = (int32_t*)dalloc(c, sizeof(int32_t));
    if (!d) return fail(c, FDTD_E_NOMEM, "agree");
    const int32_t mine = k;
    CK(cudaMemcpyAsync(d, &mine, sizeof mine, cudaMemcpyHostToDevice, c->stream));
    NK(g_nccl.AllReduce(d, d, 1, NCCL_I32, NCCL_MIN, c->comm, c->stream));
    int32_t all = 0;
    CK(cudaMemcpyAsync(&all, d, sizeof all, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    dfree(c, d);
    k = all;
  }
  return apply_passes(c, k);
}

fdtd_status apply_passes(fdtd_ctx* c, int k) {
  fdtd_status st;
  const std::vector<PassRegion> regs = pass_regions(c, k);
  // zone boxes (one per region: an instance's block or a cluster's bounding box)
  std::vector<int32_t> zr;
  for (const PassRegion& g : regs)
    zr.insert(zr.end(), {(int32_t)g.i0, (int32_t)g.j0, (int32_t)(g.i1 - g.i0), (int32_t)(g.j1 - g.j0)});
  // zone marks: clear those of the previous depth / regions, set those of the new ones
  if (c->kz_marked != k || c->zone_marked != zr) {
    int32_t* dz = nullptr;
    if ((st = upload(c, &dz, zr)) != FDTD_OK) return st;
    const int64_t n_old = (int64_t)c->zone_marked.size() / 4, n_new = (int64_t)zr.size() / 4;
    if (c->prec == 64) {
      fdtd::launch_zone<double>((double*)c->coef[1], (const double*)c->coef[0], c->pitch, c->d_zone_marked, n_old,
                                c->d.row_begin, ROW0, c->kz_marked, false, c->stream);
      fdtd::launch_zone<double>((double*)c->coef[1], (const double*)c->coef[0], c->pitch, dz, n_new, c->d.row_begin,
                                ROW0, k, true, c->stream);
    } else {
      fdtd::launch_zone<float>((float*)c->coef[1], (const float*)c->coef[0], c->pitch, c->d_zone_marked, n_old,
                               c->d.row_begin, ROW0, c->kz_marked, false, c->stream);
      fdtd::launch_zone<float>((float*)c->coef[1], (const float*)c->coef[0], c->pitch, dz, n_new, c->d.row_begin,
                               ROW0, k, true, c->stream);
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
    if (c->d_zone_marked) dfree(c, c->d_zone_marked);
    c->d_zone_marked = dz;
    c->zone_marked = zr;
  }
  c->kz_marked = k;
  c->kz = k;
  {  // CPML write-back columns (layer + k + 1): the sweep skips their storage-function terms
    const int want = c->pml_w > 0 ? c->pml_w + k + 1 : 0;
    if (c->pml_marked != want) {
      if (c->prec == 64) {
        fdtd::launch_band_marks<double>((double*)c->coef[1], (const double*)c->coef[0], c->pitch, c->d.nx, ROW0,
                                        c->rows, c->pml_marked, false, c->stream);
        fdtd::launch_band_marks<double>((double*)c->coef[1], (const double*)c->coef[0], c->pitch, c->d.nx, ROW0,
                                        c->rows, want, true, c->stream);
      } else {
        fdtd::launch_band_marks<float>((float*)c->coef[1], (const float*)c->coef[0], c->pitch, c->d.nx, ROW0,
                                       c->rows, c->pml_marked, false, c->stream);
        fdtd::launch_band_marks<float>((float*)c->coef[1], (const float*)c->coef[0], c->pitch, c->d.nx, ROW0,
                                       c->rows, want, true, c->stream);
      }
      CK(cudaGetLastError());
      c->pml_marked = want;
    }
  }
  // Fix-up batches (K3).  Instances with their own region are batched by model, up to 8
  // per CTA under one shared-memory budget (~220 KB: one 512-thread fix-up CTA per SM; 8 instances
  // fill the DMMA's N = 8; a row slab with few instances uses smaller batches so that the fix-up's
  // CTAs still fill one wave); a cluster is one batch of its members around their shared region;
  // the instances of large models (order >= FDTD_BIG_Q, default 512) take the cooperative
  // one-instance-at-a-time path (bigrom_kernel), decided by the model alone so that every slab
  // decomposition runs the same arithmetic.  Batch order: regular batches, then the large ones.
  {
    const int M = 2 * k - 1;
    // batch size: the fewest instances per CTA that still need no more waves of one-CTA-per-SM
    // fix-up CTAs than 8 per CTA would (the phases are latency-bound, so a wave costs about the same
    // whatever its batches hold; fewer instances per CTA shorten every phase): 4096 instances on
    // 148 SMs -> 7 (4 waves), a 512-instance slab -> 4 (one wave)
    const char* env = getenv("FDTD_ROM_BATCH");
    int Bauto = 8;
    {
      int nsm = 148, dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      const int64_t n = (int64_t)c->inst_model.size();
      auto waves = [&](int b) { return ((n + b - 1) / b + nsm - 1) / nsm; };
      while (Bauto > 1 && waves(Bauto - 1) == waves(8)) --Bauto;
    }
    const int Bmax = env ? std::max(1, std::min(64, atoi(env))) : Bauto;
    const char* benv = getenv("FDTD_BIG_Q");
    const int big_q = benv ? atoi(benv) : 512;
    const int nm = (int)c->models.size();
    std::vector<int> rs(nm), Bm(nm);
    std::vector<char> big(nm, 0);
    size_t big_smem = 0;
    int64_t big_elems = 0;
    for (int mi = 0; mi < nm; ++mi) {
      const ModelHost& m = c->models[mi];
      rs[mi] = (fdtd::region_elems(m.bx, m.by, M) + 3) / 4 * 4;
      const size_t per = batch_smem(c, m, 1, 1, rs[mi]);
      Bm[mi] = (int)std::max<size_t>(1, std::min<size_t>(Bmax, FIX_BUDGET / per));  // any B <= 8: N = 8, zero-padded
      if (big_q > 0 && m.q1 + m.q2 >= big_q) {
        big[mi] = 1;
        big_smem = std::max(big_smem, per);
        big_elems = std::max<int64_t>(big_elems, 3 * (m.q1 + m.q2) + (m.q2 + m.q1 + m.nY) + 2 * m.nY);
      }
    }
    c->big_grid = 0;
    if (big_elems > 0) {
      c->big_grid = c->prec == 64 ? fdtd::big_grid_size<double>(big_smem, k) : fdtd::big_grid_size<float>(big_smem, k);
      if (c->big_grid <= 0) std::fill(big.begin(), big.end(), 0);  // cannot launch cooperatively: batch path
    }
    for (int mi = 0; mi < nm; ++mi)
      if (big[mi]) Bm[mi] = 1;  // bigrom_kernel steps one instance at a time
    c->big_smem = big_smem;
    c->post_smem = 16;
    c->batch_tab.clear();
    c->batch_inst.clear();
    c->batch_rect.clear();
    auto add_batch = [&](int model, const std::vector<int>& mem, int B, int stride, int kind, const PassRegion* g) {
      c->batch_tab.insert(c->batch_tab.end(), {model, (int32_t)c->batch_inst.size(), (int32_t)mem.size(), B, stride, kind});
      c->batch_inst.insert(c->batch_inst.end(), mem.begin(), mem.end());
      if (g) c->batch_rect.insert(c->batch_rect.end(), {(int32_t)g->i0, (int32_t)g->j0, (int32_t)(g->i1 - g->i0),
                                                        (int32_t)(g->j1 - g->j0)});
      else c->batch_rect.insert(c->batch_rect.end(), {0, 0, 0, 0});
    };
    for (int pass = 0; pass < 2; ++pass) {
      // instances with their own region, grouped by model in instance order
      std::vector<int> cur;
      int cur_model = -1;
      auto flush = [&]() {
        if (cur.empty()) return;
        add_batch(cur_model, cur, Bm[cur_model], rs[cur_model], 0, nullptr);
        if (!pass) c->post_smem = std::max(c->post_smem, batch_smem(c, c->models[cur_model], Bm[cur_model],
                                                                     Bm[cur_model], rs[cur_model]));
        cur.clear();
      };
      for (const PassRegion& g : regs) {
        if (g.members.size() != 1 || big[g.model] != pass) continue;
        if (g.model != cur_model || (int)cur.size() == Bm[g.model]) {
          flush();
          cur_model = g.model;
        }
        cur.push_back(g.members[0]);
      }
      flush();
      if (pass == 0) {  // clusters: one batch per cluster around its shared region
        for (const PassRegion& g : regs) {
          if (g.members.size() < 2) continue;
          const int crs = (fdtd::region_elems((int)(g.i1 - g.i0), (int)(g.j1 - g.j0), M) + 3) / 4 * 4;
          add_batch(g.model, g.members, (int)g.members.size(), crs, 1, &g);
          c->post_smem = std::max(c->post_smem, batch_smem(c, c->models[g.model], (int)g.members.size(), 1, crs));
        }
        c->n_batch_reg = (int)(c->batch_tab.size() / fdtd::BATCH_FIELDS);
      }
    }
    c->n_clusters = 0;
    for (const PassRegion& g : regs) c->n_clusters += g.members.size() > 1;
    if (c->batch_tab.empty()) {
      c->batch_tab.assign(fdtd::BATCH_FIELDS, 0);
      c->batch_inst.assign(1, 0);
      c->batch_rect.assign(4, 0);
    }
    if ((st = upload(c, &c->d_batch_tab, c->batch_tab)) != FDTD_OK) return st;
    if ((st = upload(c, &c->d_batch_inst, c->batch_inst)) != FDTD_OK) return st;
    if ((st = upload(c, &c->d_batch_rect, c->batch_rect)) != FDTD_OK) return st;
    const int n = (int)c->inst_model.size();
    c->post_grid = n > 0 ? (int)(c->batch_tab.size() / fdtd::BATCH_FIELDS) : 1;
    std::vector<double> l1((size_t)KMAX * c->post_grid, 0.0);
    if ((st = upload(c, &c->d_level1, l1)) != FDTD_OK) return st;
    if (big_elems > 0 && c->big_grid > 0) {
      std::vector<double> z((size_t)big_elems, 0.0);
      if ((st = upload_T(c, &c->d_big, z)) != FDTD_OK) return st;
    }
  }
  // zone probes: the probes inside a region's zone (outside every hole) are recorded by its fix-up,
  // on the region's first member
  {
    const int n = (int)c->inst_model.size();
    std::vector<std::vector<int32_t>> per(n);
    if (k >= 2)
      for (const PassRegion& g : regs)
        for (int pr = 0; pr < c->n_probe; ++pr) {
          const int64_t pi = c->probe_ij[2 * pr], pj = c->probe_ij[2 * pr + 1];
          if (!(pi >= g.i0 - (k - 1) && pi < g.i1 + k && pj >= g.j0 - (k - 1) && pj < g.j1 + k)) continue;
          bool hole = false;
          for (int i : g.members) {
            const int64_t i0 = c->rects[4 * i], j0 = c->rects[4 * i + 1];
            hole |= pi >= i0 && pi < i0 + c->rects[4 * i + 2] && pj >= j0 && pj < j0 + c->rects[4 * i + 3];
          }
          if (!hole) per[g.members[0]].insert(per[g.members[0]].end(), {(int32_t)pi, (int32_t)pj, pr});
        }
    c->zp_off.assign(n + 1, 0);
    c->zp.clear();
    for (int i = 0; i < n; ++i) {
      c->zp_off[i] = (int32_t)(c->zp.size() / 3);
      c->zp.insert(c->zp.end(), per[i].begin(), per[i].end());
    }
    c->zp_off[n] = (int32_t)(c->zp.size() / 3);
    if (c->zp.empty()) c->zp.assign(3, 0);
    if ((st = upload(c, &c->d_zp_off, c->zp_off)) != FDTD_OK) return st;
    if ((st = upload(c, &c->d_zp, c->zp)) != FDTD_OK) return st;
  }
  // whole-grid mode: one rank, no CPML, at least one instance, every instance of one model that is
  // not on the large-model path, at most MAX_CLUSTER of them, and the grid + one ring of wall cells
  // with the batch's ROM vectors inside the fix-up's shared memory
  c->whole = false;
  {
    const int n = (int)c->inst_model.size();
    const char* wenv = getenv("FDTD_WHOLE");
    bool ok = c->d.nranks == 1 && !(c->d.flags & (FDTD_LOCAL_GROUP | FDTD_NO_WHOLE)) && c->pml_w == 0 && n >= 1 &&
              n <= MAX_CLUSTER && !(wenv && atoi(wenv) == 0) && c->d.nx <= 4096 && c->d.ny <= 4096;
    for (int i = 0; ok && i < n; ++i) ok = c->inst_model[i] == c->inst_model[0];
    if (ok) {
      const ModelHost& m = c->models[c->inst_model[0]];
      const char* benv = getenv("FDTD_BIG_Q");
      const int big_q = benv ? atoi(benv) : 512;
      ok = !(big_q > 0 && m.q1 + m.q2 >= big_q);
      const int rs = (fdtd::region_elems((int)c->d.nx, (int)c->d.ny, 1) + 3) / 4 * 4;
      const size_t smem = batch_smem(c, m, n, 1, rs);
      if (ok && smem <= FIX_BUDGET) {
        std::vector<int32_t> tab = {c->inst_model[0], 0, n, n, rs, 1}, inst(n), rect = {0, 0, (int32_t)c->d.nx,
                                                                                         (int32_t)c->d.ny};
        for (int i = 0; i < n; ++i) inst[i] = i;
        std::vector<int32_t> wp;
        for (int pr = 0; pr < c->n_probe; ++pr)
          wp.insert(wp.end(), {(int32_t)c->probe_ij[2 * pr], (int32_t)c->probe_ij[2 * pr + 1], pr});
        c->n_wprobe = c->n_probe;
        if (wp.empty()) wp.assign(3, 0);
        if ((st = upload(c, &c->d_wb_tab, tab)) != FDTD_OK) return st;
        if ((st = upload(c, &c->d_wb_inst, inst)) != FDTD_OK) return st;
        if ((st = upload(c, &c->d_wb_rect, rect)) != FDTD_OK) return st;
        if ((st = upload(c, &c->d_wprobe, wp)) != FDTD_OK) return st;
        // every edge's (ca, cb) and energy weight precomputed in shared memory, if they fit
        const int64_t Wr = c->d.nx + 2, Hr = c->d.ny + 2;
        const size_t coef = (size_t)(3 * (Hr + 1) * Wr + 3 * Hr * (Wr + 1)) * c->es;
        c->whole_coef = smem + coef <= FIX_BUDGET;
        c->whole_smem = smem + (c->whole_coef ? coef : 0);
        c->whole = true;
      }
    }
  }
  CK(cudaStreamSynchronize(c->stream));
  c->kz_dirty = false;
  drop_graph(c);
  return FDTD_OK;
}

}  // namespace

extern "C" {

const char* fdtd_status_string(fdtd_status s) {
  switch (s) {
    case FDTD_OK: return "ok";
    case FDTD_E_ARG: return "invalid argument";
    case FDTD_E_STATE: return "invalid state";
    case FDTD_E_PASSIVITY: return "reduced model not passive at dt";
    case FDTD_E_UNSTABLE: return "unstable";
    case FDTD_E_CUDA: return "CUDA error";
    case FDTD_E_NCCL: return "NCCL error";
    case FDTD_E_NOMEM: return "out of memory";
  }
  return "unknown";
}

const char* fdtd_last_error(const fdtd_ctx* c) { return c ? c->err.c_str() : "null context"; }

fdtd_status fdtd_create(const fdtd_grid_desc* desc, fdtd_ctx** out) {
  fdtd_ctx* c = nullptr;
  if (!desc || !out) return FDTD_E_ARG;
  *out = nullptr;
  const fdtd_grid_desc& d = *desc;
  if (d.nx < 1 || d.ny < 1 || !(d.dx > 0) || !(d.dy > 0) || !(d.dt > 0)) return FDTD_E_ARG;
  if (d.precision != 32 && d.precision != 64) return FDTD_E_ARG;
  if (!d.eps_r || !d.sigma) return FDTD_E_ARG;
  const int nranks = d.nranks <= 0 ? 1 : d.nranks;
  int64_t rb = d.row_begin, re = d.row_end;
  if (nranks == 1 && rb == 0 && re == 0) re = d.ny;
  if (rb < 0 || re > d.ny || re <= rb) return FDTD_E_ARG;
  if (re - rb > (int64_t)1 << 30) return FDTD_E_ARG;
  if (nranks > 1 && !d.nccl_id && !(d.flags & FDTD_LOCAL_GROUP)) return FDTD_E_ARG;
  // materials of rows [rb-KMAX, re+KMAX) (clipped to the grid): a K-step sweep computes up to K
  // ghost rows on each side of the slab
  const int64_t m0 = std::max<int64_t>(rb - KMAX, 0), m1 = std::min<int64_t>(re + KMAX, d.ny);
  if (d.materials_row0 > m0) return FDTD_E_ARG;

  c = new fdtd_ctx();
  c->d = d;
  c->d.nranks = nranks;
  c->d.row_begin = rb;
  c->d.row_end = re;
  c->prec = d.precision;
  c->es = d.precision == 64 ? 8 : 4;
  c->V = 16 / (int)c->es;
  c->rows = (int)(re - rb);
  c->nrows_alloc = c->rows + ROW0 + GHOST_UP;
  c->ncolv = (int)((d.nx + c->V - 1) / c->V);
  const int64_t align = 128 / (int64_t)c->es;
  // at least one column past the grid: the east PEC wall Ey[j][nx] (always 0) is read by the fix-up
  c->pitch = (std::max<int64_t>((int64_t)c->ncolv * c->V, d.nx + 1) + align - 1) / align * align;
  c->cap = d.record_capacity > 0 ? d.record_capacity : 65536;
  c->stream = (cudaStream_t)d.stream;
  if (cudaSetDevice(d.device) != cudaSuccess) {
    delete c;
    return FDTD_E_CUDA;
  }

  // eq.(1) with c_max from the smallest eps_r (host check needs the values; device arrays
  // are reduced on the host after a copy of the owned rows)
  const int64_t nmat = (m1 - m0) * d.nx;
  c->mrow_end = m1;
  const bool f32 = (d.flags & FDTD_MATERIALS_F32) != 0;
  const bool on_dev = (d.flags & FDTD_MATERIALS_ON_DEVICE) != 0;
  const size_t mes = f32 ? 4 : 8;
  const char* ebase = (const char*)d.eps_r + (size_t)(m0 - d.materials_row0) * d.nx * mes;
  const char* sbase = (const char*)d.sigma + (size_t)(m0 - d.materials_row0) * d.nx * mes;
  c->mat_f32 = f32;
  c->mrow0 = m0;
  c->mat_eps = dalloc(c, nmat * mes);
  c->mat_sig = dalloc(c, nmat * mes);
  if (!c->mat_eps || !c->mat_sig) {
    fdtd_destroy(c);
    return FDTD_E_NOMEM;
  }
  const cudaMemcpyKind kind = on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  if (cudaMemcpyAsync(c->mat_eps, ebase, nmat * mes, kind, c->stream) != cudaSuccess ||
      cudaMemcpyAsync(c->mat_sig, sbase, nmat * mes, kind, c->stream) != cudaSuccess) {
    fdtd_destroy(c);
    return FDTD_E_CUDA;
  }
  double emin = INFINITY, smin = INFINITY;
  {
    // min eps_r / sigma over the owned rows (+ ghost row), reduced on the device
    const int nb = 1024;
    double* dm = (double*)dalloc(c, 2 * nb * sizeof(double));
    if (!dm) { fdtd_destroy(c); return FDTD_E_NOMEM; }
    if (f32) fdtd::launch_min2<float>((const float*)c->mat_eps, (const float*)c->mat_sig, nmat, dm, nb, c->stream);
    else fdtd::launch_min2<double>((const double*)c->mat_eps, (const double*)c->mat_sig, nmat, dm, nb, c->stream);
    std::vector<double> hm(2 * nb);
    if (cudaMemcpyAsync(hm.data(), dm, hm.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
        cudaStreamSynchronize(c->stream) != cudaSuccess) {
      fdtd_destroy(c);
      return FDTD_E_CUDA;
    }
    for (int k = 0; k < nb; ++k) { emin = std::min(emin, hm[2 * k]); smin = std::min(smin, hm[2 * k + 1]); }
    dfree(c, dm);
  }
  // a row slab must hold the K rows a K-step pass sends to each neighbour (the halo plan sends
  // owned rows only)
  double short_slab = (nranks > 1 && c->rows < KMAX) ? 1.0 : 0.0;
  if (nranks > 1 && !(d.flags & FDTD_LOCAL_GROUP)) {
    // The checks below are collective (every rank takes the same decision): the communicator is
    // created first and the global min eps_r / sigma and the slab check are agreed over the ranks,
    // so no rank can return while its peers block in ncclCommInitRank or a later collective.
    if (!g_nccl.load(c->err)) { fdtd_destroy(c); return FDTD_E_NCCL; }
    nccl_uid id;
    memcpy(&id, d.nccl_id, sizeof id);
    if (g_nccl.CommInitRank(&c->comm, nranks, id, d.rank) != 0) { fdtd_destroy(c); return FDTD_E_NCCL; }
    double hv[3] = {emin, smin, -short_slab};
    double* dv = (double*)dalloc(c, sizeof hv);
    if (!dv || cudaMemcpyAsync(dv, hv, sizeof hv, cudaMemcpyHostToDevice, c->stream) != cudaSuccess ||
        g_nccl.AllReduce(dv, dv, 3, NCCL_F64, NCCL_MIN, c->comm, c->stream) != 0 ||
        cudaMemcpyAsync(hv, dv, sizeof hv, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
        cudaStreamSynchronize(c->stream) != cudaSuccess) {
      fdtd_destroy(c);
      return FDTD_E_NCCL;
    }
    dfree(c, dv);
    emin = hv[0];
    smin = hv[1];
    short_slab = -hv[2];
  }
  if (short_slab > 0) {
    fdtd_destroy(c);
    return FDTD_E_ARG;
  }
  if (!(emin > 0) || smin < 0) {
    fail(c, FDTD_E_ARG, "materials must have eps_r > 0 and sigma >= 0");
    fdtd_destroy(c);
    return FDTD_E_ARG;
  }
  const double cmax = C0 / std::sqrt(emin);
  const double eq1 = 1.0 / (cmax * std::sqrt(1.0 / (d.dx * d.dx) + 1.0 / (d.dy * d.dy)));
  if (d.dt > eq1 && !(d.flags & FDTD_ALLOW_DT_ABOVE_EQ1)) {
    fdtd_destroy(c);
    return FDTD_E_UNSTABLE;
  }

  // + a tail: the sweep's lanes past the last vector column load unconditionally (their values are
  // never stored), reaching up to 31 vectors beyond the last row of an array
  if ((double)c->nrows_alloc * (double)c->pitch >= 4294967296.0) {  // the sweep indexes rows with 32-bit offsets
    fail(c, FDTD_E_ARG, "a slab of %lld x %lld elements per array exceeds 2^32; use more row slabs",
         (long long)c->nrows_alloc, (long long)c->pitch);
    fdtd_destroy(c);
    return FDTD_E_ARG;
  }
  const size_t fbytes = (size_t)c->nrows_alloc * c->pitch * c->es + ARRAY_TAIL;
  for (int b = 0; b < 2; ++b)
    for (int a = 0; a < 3; ++a)
      if (!(c->f[b][a] = dalloc(c, fbytes))) { fdtd_destroy(c); return FDTD_E_NOMEM; }
  for (int a = 0; a < 2; ++a)
    if (!(c->coef[a] = dalloc(c, fbytes))) { fdtd_destroy(c); return FDTD_E_NOMEM; }
  c->d_step = (int64_t*)dalloc(c, sizeof(int64_t));
  c->d_flag = (int*)dalloc(c, sizeof(int));
  c->d_src_meta = (int64_t*)dalloc(c, 2 * sizeof(int64_t));
  c->d_done = (unsigned*)dalloc(c, sizeof(unsigned) * 4);
  c->d_energy_ring = (double*)dalloc(c, c->cap * sizeof(double));
  c->d_level1 = (double*)dalloc(c, KMAX * sizeof(double));
  c->d_level2 = (double*)dalloc(c, (size_t)KMAX * fdtd::FIN_GRID * sizeof(double));
  c->k_want = c->V;  // deepest pass the vector width allows (4 in fp32, 2 in fp64)
  if (const char* e = getenv("FDTD_K")) c->k_want = std::max(1, atoi(e));
  if (!c->d_step || !c->d_done || !c->d_energy_ring || !c->d_flag || !c->d_src_meta) {
    fdtd_destroy(c);
    return FDTD_E_NOMEM;
  }
  fdtd_status st = f32 ? build_coefficients<float>(c) : build_coefficients<double>(c);
  if (st != FDTD_OK) { fdtd_destroy(c); return st; }
  fdtd_set_tuning(c, 0, 0);
  if (nranks > 1 && !(d.flags & FDTD_LOCAL_GROUP)) {
    if (cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming) != cudaSuccess) {
      fdtd_destroy(c);
      return FDTD_E_CUDA;
    }
  }
  if (nranks > 1 && (cudaStreamCreateWithFlags(&c->edge_stream, cudaStreamNonBlocking) != cudaSuccess ||
                     cudaEventCreateWithFlags(&c->ev_edge_go, cudaEventDisableTiming) != cudaSuccess ||
                     cudaEventCreateWithFlags(&c->ev_edge, cudaEventDisableTiming) != cudaSuccess)) {
    fdtd_destroy(c);
    return FDTD_E_CUDA;
  }
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) { fdtd_destroy(c); return FDTD_E_CUDA; }
  *out = c;
  return FDTD_OK;
}

fdtd_status fdtd_set_tuning(fdtd_ctx* c, int32_t rows_per_cta, int32_t warps_per_cta) {
  if (!c) return FDTD_E_ARG;
  if (rows_per_cta < 0 || warps_per_cta < 0 || warps_per_cta > 8) return fail(c, FDTD_E_ARG, "bad tuning");
  // rows per CTA: the 2K - 1 stage rows recomputed at a chunk start against the tail of the last
  // wave; a row slab of a multi-GPU run does better with 128 than 64 below 8192 rows and with 256
  // from 8192 rows (config 4 on 4 slabs: 495 vs 482 G, on 8 slabs 128 beats 256: 453 vs 423 G;
  // profiles/r02g_slab_chunks.txt); 512 rows measured 1.3 % faster than 256 on 32768 rows
  // (tools/sweep_layout_probe.cu, round 2).
  // Small grids (< 2048 rows, too few CTAs for one wave): a pass is the latency of one CTA's row
  // chain, so short chunks of 2-warp CTAs spread it over >= ~600 CTAs (the Sec. VI-A cavity, 500^2
  // fp64: 43 -> 31 us per step with 4-row chunks)
  const bool slab = c->d.nranks > 1;
  c->chunk = rows_per_cta ? rows_per_cta
                          : (c->rows >= 32768 ? 512 : c->rows >= 16384 ? 256
                             : c->rows >= 2048 ? (slab ? (c->rows < 8192 ? 128 : 256) : 64) : 32);
  c->warps = warps_per_cta ? warps_per_cta : 4;
  if (!rows_per_cta && !warps_per_cta && c->rows < 2048) {
    c->warps = 2;
    int gx2 = 1;
    for (int K = 1; K <= KMAX; K *= 2) gx2 = std::max(gx2, sweep_gx(c, K));
    int ch = 32;
    while (ch > 4 && (int64_t)((c->rows + ch - 1) / ch) * gx2 < 600) ch /= 2;
    c->chunk = ch;
  }
  if (!rows_per_cta)
    if (const char* e = getenv("FDTD_CHUNK")) c->chunk = std::max(1, atoi(e));  // tuning experiments
  if (!warps_per_cta)
    if (const char* e = getenv("FDTD_WARPS")) c->warps = std::max(1, std::min(8, atoi(e)));
  if (const char* e = getenv("FDTD_POST_THREADS")) c->post_threads = std::max(64, std::min(512, atoi(e) / 32 * 32));
  const int gx = sweep_gx_max(c);
  const int gy = (c->rows + c->chunk - 1) / c->chunk;
  const int n = gx * gy + fdtd::pml_ctas(c->rows, PML_CHUNK);  // sweep CTAs + (possible) CPML band CTAs
  if (n > c->n_partials) {
    if (c->d_partials) dfree(c, c->d_partials);
    c->d_partials = (double*)dalloc(c, (size_t)KMAX * n * sizeof(double));
    if (!c->d_partials) return fail(c, FDTD_E_NOMEM, "partials");
    c->n_partials = n;
  }
  drop_graph(c);
  return FDTD_OK;
}

fdtd_status fdtd_add_rom(fdtd_ctx* c, const fdtd_rom_model* m, const int32_t* anchors, int64_t count,
                         int32_t* model_id) {
  if (!c || !m) return FDTD_E_ARG;
  if (m->bx < 1 || m->by < 1 || m->q1 < 1 || m->q2 < 1 || !m->R11 || !m->R22 || !m->F11 || !m->K || !m->L)
    return fail(c, FDTD_E_ARG, "bad model");
  if (count < 0 || (count > 0 && !anchors)) return fail(c, FDTD_E_ARG, "bad anchors");
  const int bx = m->bx, by = m->by, q1 = m->q1, q2 = m->q2, nY = 2 * bx + 2 * by, q = q1 + q2;
  const bool literal = m->literal != 0;
  const int rr = literal ? m->r : 1, nU = rr * nY;  // ports of L: nY coarse edges or r nY fine nodes
  if (literal && m->r < 1) return fail(c, FDTD_E_ARG, "literal model needs r >= 1");
  const double dt = c->d.dt, dx = c->d.dx, dy = c->d.dy;
  using fdtd::dense::Mat;
  namespace dense = fdtd::dense;
  Mat R11(m->R11, m->R11 + q1 * q1), R22(m->R22, m->R22 + q2 * q2), F11(m->F11, m->F11 + q1 * q1),
      K(m->K, m->K + q1 * q2), L(m->L, m->L + (size_t)q1 * nU);
  // eq:cond1rom: R~ = [[R11/dt, -K/2], [-K^T/2, R22/dt]] > 0 (Cholesky of the diagonally scaled matrix)
  {
    Mat R = dense::zeros(q, q);
    for (int i = 0; i < q1; ++i)
      for (int j = 0; j < q1; ++j) R[(size_t)i * q + j] = 0.5 * (R11[i * q1 + j] + R11[j * q1 + i]) / dt;
    for (int i = 0; i < q2; ++i)
      for (int j = 0; j < q2; ++j) R[(size_t)(q1 + i) * q + q1 + j] = 0.5 * (R22[i * q2 + j] + R22[j * q2 + i]) / dt;
    for (int i = 0; i < q1; ++i)
      for (int j = 0; j < q2; ++j) {
        R[(size_t)i * q + q1 + j] = -0.5 * K[i * q2 + j];
        R[(size_t)(q1 + j) * q + i] = -0.5 * K[i * q2 + j];
      }
    std::vector<double> s(q);
    for (int i = 0; i < q; ++i) {
      const double dg = R[(size_t)i * q + i];
      if (!(dg > 0)) return fail(c, FDTD_E_PASSIVITY, "R~ has a non-positive diagonal entry");
      s[i] = 1.0 / std::sqrt(dg);
    }
    for (int i = 0; i < q; ++i)
      for (int j = 0; j < q; ++j) R[(size_t)i * q + j] *= s[i] * s[j];
    if (!dense::cholesky_ok(R, q))
      return fail(c, FDTD_E_PASSIVITY, "eq:cond1rom fails: R~ is not positive definite at dt = %g", dt);
    // eq:cond2rom: F~ + F~^T >= 0 -> F11 + F11^T + 2 tol I must be positive definite
    Mat FF = dense::zeros(q1, q1);
    double fmax = 0.0;
    for (int i = 0; i < q1; ++i)
      for (int j = 0; j < q1; ++j) {
        FF[i * q1 + j] = F11[i * q1 + j] + F11[j * q1 + i];
        fmax = std::max(fmax, std::fabs(FF[i * q1 + j]));
      }
    if (fmax > 0) {
      for (int i = 0; i < q1; ++i) FF[i * q1 + i] += 2e-12 * fmax;
      if (!dense::cholesky_ok(FF, q1)) return fail(c, FDTD_E_PASSIVITY, "eq:cond2rom fails: F~ + F~^T not >= 0");
    }
  }
  // placement checks
  for (int64_t k = 0; k < count; ++k) {
    const int64_t i0 = anchors[2 * k], j0 = anchors[2 * k + 1];
    if (i0 < 1 || j0 < 1 || i0 + bx > c->d.nx - 1 || j0 + by > c->d.ny - 1)
      return fail(c, FDTD_E_ARG, "instance %lld: footprint + ring leaves the grid", (long long)k);
    if (j0 - 1 < c->d.row_begin || j0 + by > c->d.row_end - 1)
      return fail(c, FDTD_E_ARG, "instance %lld: footprint + ring straddles this rank's rows", (long long)k);
    if (c->pml_w > 0 && (i0 - 1 < c->pml_w + 3 || i0 + bx + 1 > c->d.nx - c->pml_w - 3))
      return fail(c, FDTD_E_ARG, "instance %lld lies within the CPML band", (long long)k);
  }
  {
    // ring-vs-footprint overlap: sort all rectangles by i0 and sweep
    struct Rc { int64_t i0, j0, bx, by; };
    std::vector<Rc> all;
    for (size_t r = 0; r < c->rects.size(); r += 4)
      all.push_back({c->rects[r], c->rects[r + 1], c->rects[r + 2], c->rects[r + 3]});
    for (int64_t k = 0; k < count; ++k) all.push_back({anchors[2 * k], anchors[2 * k + 1], bx, by});
    std::sort(all.begin(), all.end(), [](const Rc& a, const Rc& b) { return a.i0 < b.i0; });
    int64_t wmax = 0;
    for (auto& r : all) wmax = std::max(wmax, r.bx);
    for (size_t a = 0; a < all.size(); ++a)
      for (size_t b = a + 1; b < all.size() && all[b].i0 <= all[a].i0 + all[a].bx + wmax + 2; ++b) {
        const Rc &A = all[a], &B = all[b];
        // expanded A = [i0-1, i0+bx] vs footprint B = [i0, i0+bx-1] (and symmetric)
        const bool ox = A.i0 - 1 <= B.i0 + B.bx - 1 && B.i0 <= A.i0 + A.bx;
        const bool oy = A.j0 - 1 <= B.j0 + B.by - 1 && B.j0 <= A.j0 + A.by;
        const bool ox2 = B.i0 - 1 <= A.i0 + A.bx - 1 && A.i0 <= B.i0 + B.bx;
        const bool oy2 = B.j0 - 1 <= A.j0 + A.by - 1 && A.j0 <= B.j0 + B.by;
        if ((ox && oy) || (ox2 && oy2))
          return fail(c, FDTD_E_ARG, "instances at (%lld,%lld) and (%lld,%lld) overlap (footprint + ring)",
                      (long long)A.i0, (long long)A.j0, (long long)B.i0, (long long)B.j0);
      }
  }
  // ---- shared model operators (fp64), K3:
  // C = R11/dt + F11; Aq = C^-1 (R11/dt - F11); Kq = C^-1 K; Q1 = -dt R22^-1 K^T;
  // Bq = C^-1 L S_c; P = L^T Bq; Lt = L^T
  Mat Cm = dense::zeros(q1, q1), Cr = dense::zeros(q1, q1);
  for (int i = 0; i < q1 * q1; ++i) { Cm[i] = R11[i] / dt + F11[i]; Cr[i] = R11[i] / dt - F11[i]; }
  Mat Ci, R22i;
  if (!dense::inverse(Cm, q1, Ci) || !dense::inverse(R22, q2, R22i))
    return fail(c, FDTD_E_PASSIVITY, "singular R~11/dt + F~11 or R~22");
  std::vector<double> Sc(nY), DlGm(nY);
  for (int p = 0; p < nY; ++p) {
    Sc[p] = p < bx ? -dx : p < 2 * bx ? dx : p < 2 * bx + by ? dy : -dy;
    DlGm[p] = p < bx ? -dx : p < 2 * bx ? dx : p < 2 * bx + by ? dy : -dy;  // D_l G (R5): same numbers
  }
  // B~ = L~ S over the ports of L (S_f = S_c / r on the literal fine ports)
  Mat Be = dense::zeros(q1, nU);
  for (int i = 0; i < q1; ++i)
    for (int k = 0; k < nU; ++k) Be[(size_t)i * nU + k] = L[(size_t)i * nU + k] * Sc[k / rr] / rr;
  Mat Aq = dense::matmul(Ci, Cr, q1, q1, q1);
  Mat Kq = dense::matmul(Ci, K, q1, q1, q2);
  Mat Kt = dense::transpose(K, q1, q2);
  Mat Q1 = dense::matmul(R22i, Kt, q2, q2, q1);
  for (auto& v : Q1) v *= -dt;
  Mat Bq = dense::matmul(Ci, Be, q1, q1, nU);
  Mat Lt = dense::transpose(L, q1, nU);
  Mat P = dense::matmul(Lt, Bq, nU, q1, nU);
  ModelHost mh;
  mh.bx = bx; mh.by = by; mh.nY = nY; mh.q1 = q1; mh.q2 = q2; mh.literal = literal;
  // literal coupling (eq:sysform with T, 1/r; K3): with P_f = L~^T C^-1 B~ (nP x nP),
  //   u^ = P_f^-1 (T y' - L~^T E*),  (diag(c_y) + Psi) y' = a_y y + D_l G h + W1 E*,
  //   E~' = (I - Z L~^T) E* + Z T y',  Z = C^-1 B~ P_f^-1,  Psi = (1/r) D_l G T^T P_f^-1 T,
  //   W1 = (1/r) D_l G T^T P_f^-1 L~^T
  Mat Zl, Wl, Psi;
  if (literal) {
    Mat Pfi;
    if (!dense::inverse(P, nU, Pfi))
      return fail(c, FDTD_E_ARG, "literal coupling: A1 is singular (the ROM's E basis must span the %d port "
                  "directions; q1 = %d)", nU, q1);
    Zl = dense::matmul(Bq, Pfi, q1, nU, nU);
    Mat TtPfi = dense::zeros(nY, nU);  // (1/r) D_l G T^T P_f^-1
    for (int k = 0; k < nU; ++k)
      for (int j = 0; j < nU; ++j) TtPfi[(size_t)(k / rr) * nU + j] += DlGm[k / rr] / rr * Pfi[(size_t)k * nU + j];
    Psi = dense::zeros(nY, nY);
    for (int p = 0; p < nY; ++p)
      for (int j = 0; j < nU; ++j) Psi[(size_t)p * nY + j / rr] += TtPfi[(size_t)p * nU + j];
    Wl = dense::matmul(TtPfi, Lt, nY, nU, q1);
    mh.P = Psi;
  } else {
    mh.P = P;
  }
  Mat R11dt(R11), R22dt(R22);
  for (auto& v : R11dt) v /= dt;
  for (auto& v : R22dt) v /= dt;
  // fused operators (K3): x = [E~; H~]
  //   collapsed: M1 = [[Q1, I], [Aq', Kq], [-Lt Aq', -Lt Kq]] with Aq' = Aq + Kq Q1;  M2 = [Bq; Lt Bq]
  //   literal:   M1 = [[Q1, I], [(I - Z Lt)[Aq', Kq]], [W1 [Aq', Kq]]];             M2 = [Z T; I]
  const int nxs = q1 + q2, m1 = q2 + q1 + nY, m2 = q1 + nY;
  Mat Aqp = dense::matmul(Kq, Q1, q1, q2, q1);
  for (int i = 0; i < q1 * q1; ++i) Aqp[i] += Aq[i];
  Mat EA = Aqp, EK = Kq, TA, TK;  // E* rows and t rows of M1
  if (literal) {
    Mat ZL = dense::matmul(Zl, Lt, q1, nU, q1);  // Z L~^T
    for (int i = 0; i < q1; ++i)
      for (int j = 0; j < q1; ++j) ZL[(size_t)i * q1 + j] = (i == j ? 1.0 : 0.0) - ZL[(size_t)i * q1 + j];
    EA = dense::matmul(ZL, Aqp, q1, q1, q1);
    EK = dense::matmul(ZL, Kq, q1, q1, q2);
    TA = dense::matmul(Wl, Aqp, nY, q1, q1);
    TK = dense::matmul(Wl, Kq, nY, q1, q2);
  } else {
    TA = dense::matmul(Lt, Aqp, nY, q1, q1);
    TK = dense::matmul(Lt, Kq, nY, q1, q2);
    for (auto& v : TA) v = -v;
    for (auto& v : TK) v = -v;
  }
  Mat M1 = dense::zeros(m1, nxs);
  for (int i = 0; i < q2; ++i) {
    for (int j = 0; j < q1; ++j) M1[(size_t)i * nxs + j] = Q1[(size_t)i * q1 + j];
    M1[(size_t)i * nxs + q1 + i] = 1.0;
  }
  for (int i = 0; i < q1; ++i) {
    for (int j = 0; j < q1; ++j) M1[(size_t)(q2 + i) * nxs + j] = EA[(size_t)i * q1 + j];
    for (int j = 0; j < q2; ++j) M1[(size_t)(q2 + i) * nxs + q1 + j] = EK[(size_t)i * q2 + j];
  }
  for (int i = 0; i < nY; ++i) {
    for (int j = 0; j < q1; ++j) M1[(size_t)(q2 + q1 + i) * nxs + j] = TA[(size_t)i * q1 + j];
    for (int j = 0; j < q2; ++j) M1[(size_t)(q2 + q1 + i) * nxs + q1 + j] = TK[(size_t)i * q2 + j];
  }
  Mat M2 = dense::zeros(m2, nY);
  if (literal) {
    for (int i = 0; i < q1; ++i)
      for (int k = 0; k < nU; ++k) M2[(size_t)i * nY + k / rr] += Zl[(size_t)i * nU + k];  // Z T
    for (int i = 0; i < nY; ++i) M2[(size_t)(q1 + i) * nY + i] = 1.0;
  } else {
    for (int i = 0; i < q1; ++i)
      for (int j = 0; j < nY; ++j) M2[(size_t)i * nY + j] = Bq[(size_t)i * nY + j];
    for (int i = 0; i < nY; ++i)
      for (int j = 0; j < nY; ++j) M2[(size_t)(q1 + i) * nY + j] = P[(size_t)i * nY + j];
  }
  Mat Rt = dense::zeros(nxs, nxs);
  for (int i = 0; i < q1; ++i)
    for (int j = 0; j < q1; ++j) Rt[(size_t)i * nxs + j] = R11dt[(size_t)i * q1 + j];
  for (int i = 0; i < q2; ++i)
    for (int j = 0; j < q2; ++j) Rt[(size_t)(q1 + i) * nxs + q1 + j] = R22dt[(size_t)i * q2 + j];
  for (int i = 0; i < q1; ++i)
    for (int j = 0; j < q2; ++j) {
      Rt[(size_t)i * nxs + q1 + j] = -0.5 * K[(size_t)i * q2 + j];
      Rt[(size_t)(q1 + j) * nxs + i] = -0.5 * K[(size_t)i * q2 + j];
    }
  mh.dev.nY = nY; mh.dev.q1 = q1; mh.dev.q2 = q2; mh.dev.literal = literal ? 1 : 0;
  {  // [M1; R~] as one operator (the fix-up's first GEMM phase also yields R~ x~), and M2
    Mat M1R = dense::zeros(m1 + nxs, nxs);
    for (int i = 0; i < m1; ++i)
      for (int j = 0; j < nxs; ++j) M1R[(size_t)i * nxs + j] = M1[(size_t)i * nxs + j];
    for (int i = 0; i < nxs; ++i)
      for (int j = 0; j < nxs; ++j) M1R[(size_t)(m1 + i) * nxs + j] = Rt[(size_t)i * nxs + j];
    mh.dev.off_M1t = push_tiles(c->mpool, M1R, m1 + nxs, nxs, mh.dev.mt1, mh.dev.kt1);
    mh.dev.off_M2t = push_tiles(c->mpool, M2, m2, nY, mh.dev.mt2, mh.dev.kt2);
  }
  const int mid = (int)c->models.size();
  c->models.push_back(mh);
  c->nvec = std::max(c->nvec, q1 + q2 + nY);

  // ---- per instance: outside-cell materials -> c_y, a_y, Schur inverse S_k
  std::vector<int64_t> cells;
  auto outside = [&](int64_t i0, int64_t j0, int p, int64_t& oi, int64_t& oj) {
    if (p < bx) { oi = i0 + p; oj = j0 - 1; }
    else if (p < 2 * bx) { oi = i0 + p - bx; oj = j0 + by; }
    else if (p < 2 * bx + by) { oi = i0 - 1; oj = j0 + p - 2 * bx; }
    else { oi = i0 + bx; oj = j0 + p - 2 * bx - by; }
  };
  for (int64_t k = 0; k < count; ++k)
    for (int p = 0; p < nY; ++p) {
      int64_t oi, oj;
      outside(anchors[2 * k], anchors[2 * k + 1], p, oi, oj);
      cells.push_back(oj * c->d.nx + oi);
    }
  std::vector<double> oe, os;
  fdtd_status st = gather_materials(c, cells, oe, os);
  if (st != FDTD_OK) return st;
  const int64_t P_ = c->pitch;
  for (int64_t k = 0; k < count; ++k) {
    const int64_t i0 = anchors[2 * k], j0 = anchors[2 * k + 1];
    c->inst_model.push_back(mid);
    c->rects.insert(c->rects.end(), {(int32_t)i0, (int32_t)j0, bx, by});
    c->port_off.push_back((int64_t)c->port_edge.size());
    c->state_off.push_back(c->state_len);
    c->state_len += q;
    c->Sk_off.push_back((int64_t)c->Sk.size());
    Mat A = mh.P;
    for (int p = 0; p < nY; ++p) {
      const bool isey = p >= 2 * bx;
      const double Dl = isey ? dy : dx, Dlp = isey ? dx / 2 : dy / 2;
      const double G = (p < bx) ? -1.0 : (p < 2 * bx) ? 1.0 : (p < 2 * bx + by) ? 1.0 : -1.0;
      const double eps = EPS0 * oe[k * nY + p], sig = os[k * nY + p];
      const double cy = Dl * Dlp * (eps / dt + sig / 2), ay = Dl * Dlp * (eps / dt - sig / 2);
      if (literal) {  // (diag(c_y) + Psi) y' = a_y y + D_l G h + W1 E*
        A[(size_t)p * nY + p] += cy;
        c->cya.push_back(ay);
        c->cyg.push_back(Dl * G);
      } else {        // (P + diag(D_l G / c_y)) U = (a_y/c_y) y + (D_l G/c_y) h - L~^T E*
        A[(size_t)p * nY + p] += Dl * G / cy;
        c->cya.push_back(ay / cy);
        c->cyg.push_back(Dl * G / cy);
      }
      c->ehalf.push_back(Dl * Dlp * eps / dt);
      int64_t e;
      if (p < bx) e = lrow(c, j0) * P_ + i0 + p;
      else if (p < 2 * bx) e = lrow(c, j0 + by) * P_ + i0 + p - bx;
      else if (p < 2 * bx + by) e = (int64_t(1) << 62) | (lrow(c, j0 + p - 2 * bx) * P_ + i0);
      else e = (int64_t(1) << 62) | (lrow(c, j0 + p - 2 * bx - by) * P_ + i0 + bx);
      c->port_edge.push_back(e);
    }
    Mat S;
    if (!dense::inverse(A, nY, S)) return fail(c, FDTD_E_ARG, "singular interface Schur matrix");
    for (int j = 0; j < nY; ++j)  // column-major
      for (int i = 0; i < nY; ++i) c->Sk.push_back(S[(size_t)i * nY + j]);
  }
  // masks (coefficients + zeroed holes/interfaces in both buffers)
  std::vector<int32_t> nr(c->rects.end() - 4 * count, c->rects.end());
  int32_t* drect = nullptr;
  if ((st = upload(c, &drect, nr)) != FDTD_OK) return st;
  if (c->prec == 64) {
    double* fl[6] = {(double*)c->f[0][0], (double*)c->f[0][1], (double*)c->f[0][2],
                     (double*)c->f[1][0], (double*)c->f[1][1], (double*)c->f[1][2]};
    fdtd::launch_mask<double>((double*)c->coef[0], fl, P_, drect, count, c->d.row_begin, ROW0, true, c->stream);
  } else {
    float* fl[6] = {(float*)c->f[0][0], (float*)c->f[0][1], (float*)c->f[0][2],
                    (float*)c->f[1][0], (float*)c->f[1][1], (float*)c->f[1][2]};
    fdtd::launch_mask<float>((float*)c->coef[0], fl, P_, drect, count, c->d.row_begin, ROW0, true, c->stream);
  }
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(c->stream));
  dfree(c, drect);
  if ((st = upload_roms(c)) != FDTD_OK) return st;
  CK(cudaStreamSynchronize(c->stream));
  drop_graph(c);
  if (model_id) *model_id = mid;
  return FDTD_OK;
}

fdtd_status fdtd_set_source_line(fdtd_ctx* c, int64_t i, int64_t j0, int64_t j1, const double* samples, int64_t n,
                                 int64_t step0) {
  if (!c) return FDTD_E_ARG;
  if (i < 0 || i >= c->d.nx || j0 < 0 || j1 > c->d.ny || j1 <= j0 || n < 0 || (n > 0 && !samples))
    return fail(c, FDTD_E_ARG, "bad source");
  // The captured graph bakes the sample pointer and the source cells into its kernels, not the
  // window {t0, n}: a new window of at most src_cap samples on the same cells (the per-call
  // pattern of an end-to-end run) keeps the graph.
  bool regraph = !c->d_src || i != c->src_i || j0 != c->src_j || j1 != c->src_j1;
  if (!c->d_src || n > c->src_cap) {
    if (c->d_src) dfree(c, c->d_src);
    c->src_cap = std::max<int64_t>(n, 1);
    c->d_src = (double*)dalloc(c, c->src_cap * sizeof(double));
    if (!c->d_src) return fail(c, FDTD_E_NOMEM, "source");
    regraph = true;
  }
  if (n) CK(cudaMemcpyAsync(c->d_src, samples, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  c->h_src_meta[0] = step0;
  c->h_src_meta[1] = n;
  CK(cudaMemcpyAsync(c->d_src_meta, c->h_src_meta, sizeof c->h_src_meta, cudaMemcpyHostToDevice, c->stream));
  c->src_i = i;
  c->src_j = j0;
  c->src_j1 = j1;
  if (regraph) drop_graph(c);
  return FDTD_OK;
}

fdtd_status fdtd_set_source(fdtd_ctx* c, int64_t i, int64_t j, const double* samples, int64_t n, int64_t step0) {
  return fdtd_set_source_line(c, i, j, j + 1, samples, n, step0);
}

fdtd_status fdtd_set_probes(fdtd_ctx* c, const int64_t* ij, int32_t n) {
  if (!c || n < 0 || (n > 0 && !ij)) return FDTD_E_ARG;
  // S3: the sweep records the probes of its own rows (a per-row table); probes of other ranks are
  // never written here and contribute 0 to the cross-rank sum
  std::vector<std::array<int64_t, 3>> own;  // (local row, column, probe index)
  c->probe_ij.assign(ij, ij + 2 * (int64_t)n);
  for (int32_t k = 0; k < n; ++k) {
    const int64_t i = ij[2 * k], j = ij[2 * k + 1];
    if (i < 0 || i >= c->d.nx || j < 0 || j >= c->d.ny) return fail(c, FDTD_E_ARG, "probe %d outside grid", k);
    if (j >= c->d.row_begin && j < c->d.row_end) own.push_back({lrow(c, j), i, k});
  }
  std::sort(own.begin(), own.end());
  std::vector<int2> rows_tab((size_t)c->nrows_alloc, int2{0, 0}), list(std::max<size_t>(own.size(), 1), int2{0, 0});
  for (size_t t = 0; t < own.size(); ++t) {
    list[t] = int2{(int)own[t][1], (int)own[t][2]};
    int2& r = rows_tab[own[t][0]];
    if (r.y == 0) r.x = (int)t;
    r.y += 1;
  }
  fdtd_status st = upload(c, &c->d_probe_rows, rows_tab);
  if (st != FDTD_OK) return st;
  {  // column and local row of every probe (-1: another rank's) for the CPML band fix-up
    std::vector<int64_t> gi(std::max(n, 1), -1);
    std::vector<int32_t> lr(std::max(n, 1), -1);
    for (int32_t k = 0; k < n; ++k) {
      gi[k] = ij[2 * k];
      const int64_t j = ij[2 * k + 1];
      lr[k] = (j >= c->d.row_begin && j < c->d.row_end) ? (int32_t)lrow(c, j) : -1;
    }
    if ((st = upload(c, &c->d_probe_gi, gi)) != FDTD_OK) return st;
    if ((st = upload(c, &c->d_probe_lr, lr)) != FDTD_OK) return st;
  }
  if ((st = upload(c, &c->d_probe_list, list)) != FDTD_OK) return st;
  if (c->d_probe_ring) dfree(c, c->d_probe_ring);
  c->d_probe_ring = dalloc(c, (size_t)std::max(n, 1) * c->cap * c->es);
  if (!c->d_probe_ring) return fail(c, FDTD_E_NOMEM, "probe ring");
  c->n_probe = n;
  c->rd_probe = c->steps;
  c->kz_dirty = true;  // zone probes
  drop_graph(c);
  return FDTD_OK;
}

fdtd_status fdtd_record_energy(fdtd_ctx* c, int32_t on) {
  if (!c) return FDTD_E_ARG;
  if ((on != 0) != c->energy_on) {
    c->energy_on = on != 0;
    c->rd_energy = c->steps;
    drop_graph(c);
  }
  return FDTD_OK;
}

fdtd_status fdtd_step(fdtd_ctx* c, int64_t nsteps) {
  if (!c || nsteps < 0) return FDTD_E_ARG;
  int64_t oldest = c->steps + nsteps;
  if (c->n_probe > 0) oldest = std::min(oldest, c->rd_probe);
  if (c->energy_on) oldest = std::min(oldest, c->rd_energy);
  if (c->steps + nsteps - oldest > c->cap)
    return fail(c, FDTD_E_STATE, "unread records would exceed record_capacity (%lld)", (long long)c->cap);
  if (c->d.flags & FDTD_LOCAL_GROUP) return fail(c, FDTD_E_STATE, "members of a local group step with fdtd_step_group");
  // graphs also with NCCL ranks (the halo send/recv group and the split sweeps are captured with
  // the side streams forked and joined by events); a capture that fails falls back to eager passes
  const bool use_graph = !(c->d.flags & FDTD_NO_GRAPH) && !(c->d.flags & FDTD_LOCAL_GROUP) && !c->profiling &&
                         !c->graph_broken;
  fdtd_status st = configure_passes(c);
  if (st != FDTD_OK) return st;
  if (c->whole && nsteps > 0) {  // K3c: all the steps in one launch (buffer cur -> 1 - cur)
    if (c->prec == 64) fdtd::launch_wholegrid<double>(post_params<double>(c, c->cur), nsteps, c->energy_on, c->stream);
    else fdtd::launch_wholegrid<float>(post_params<float>(c, c->cur), nsteps, c->energy_on, c->stream);
    c->launches += 1;
    c->steps += nsteps;
    c->cur ^= 1;
    CK(cudaGetLastError());
    return FDTD_OK;
  }
  int64_t left = nsteps;
  while (left > 0) {
    const int per = 2 * c->kz;
    if (use_graph && c->cur == 0 && left >= per) {
      if (c->graph_dirty || !c->gexec || c->graph_steps != per) {
        if ((st = build_graph(c)) != FDTD_OK) {
          if (st != FDTD_E_CUDA) return st;
          c->graph_broken = true;  // e.g. a launch the runtime cannot capture: stay eager
          cudaGetLastError();
          drop_graph(c);
          continue;
        }
      }
      CK(cudaGraphLaunch(c->gexec, c->stream));
      c->launches += c->graph_launches;
      c->steps += per;
      left -= per;
      continue;
    }
    // passes of depth kz; a remainder with shallower passes (the zone marks stay those of kz)
    const int K = left >= c->kz ? c->kz : left >= 2 ? 2 : 1;
    if ((st = enqueue_pass(c, c->cur, c->stream, K)) != FDTD_OK) return st;
    c->steps += K;
    left -= K;
    c->cur ^= 1;
  }
  CK(cudaGetLastError());
  return FDTD_OK;
}

static fdtd_status read_ring(fdtd_ctx* c, const void* ring, int rows_, size_t es, int64_t from, int64_t to,
                             int dtype, void* host, int64_t ldh) {
  // copy ring entries for steps [from, to) of `rows_` rows (ring row stride cap) into host [rows_][ldh]
  const int64_t n = to - from;
  if (n <= 0 || rows_ <= 0) return FDTD_OK;
  void* tmp = dalloc(c, (size_t)rows_ * n * es);
  if (!tmp) return fail(c, FDTD_E_NOMEM, "record staging");
  int64_t done = 0;
  while (done < n) {
    const int64_t s = (from + done) % c->cap;
    const int64_t len = std::min(n - done, c->cap - s);
    CK(cudaMemcpy2DAsync((char*)tmp + done * es, n * es, (const char*)ring + s * es, c->cap * es, len * es, rows_,
                         cudaMemcpyDeviceToDevice, c->stream));
    done += len;
  }
  if (c->d.nranks > 1 && c->comm) NK(g_nccl.AllReduce(tmp, tmp, (size_t)rows_ * n, dtype, NCCL_SUM, c->comm, c->stream));
  CK(cudaMemcpy2DAsync(host, ldh * es, tmp, n * es, n * es, rows_, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  dfree(c, tmp);
  return FDTD_OK;
}

fdtd_status fdtd_probe(fdtd_ctx* c, double* out, int64_t cap_steps, int64_t* n_steps) {
  if (!c || !n_steps) return FDTD_E_ARG;
  fdtd_status st = check_async(c, true);
  if (st != FDTD_OK) return st;
  const int64_t n = c->steps - c->rd_probe;
  if (n > cap_steps) return fail(c, FDTD_E_ARG, "output holds %lld steps, %lld pending", (long long)cap_steps, (long long)n);
  *n_steps = n;
  if (c->n_probe == 0 || n == 0) { c->rd_probe = c->steps; return FDTD_OK; }
  if (!out) return FDTD_E_ARG;
  std::vector<char> h((size_t)c->n_probe * cap_steps * c->es);
  st = read_ring(c, c->d_probe_ring, c->n_probe, c->es, c->rd_probe, c->steps, c->prec == 64 ? NCCL_F64 : NCCL_F32,
                 h.data(), cap_steps);
  if (st != FDTD_OK) return st;
  for (int64_t p = 0; p < c->n_probe; ++p)
    for (int64_t k = 0; k < n; ++k)
      out[p * cap_steps + k] = c->prec == 64 ? ((double*)h.data())[p * cap_steps + k]
                                             : (double)((float*)h.data())[p * cap_steps + k];
  c->rd_probe = c->steps;
  return FDTD_OK;
}

fdtd_status fdtd_energy(fdtd_ctx* c, double* out, int64_t cap, int64_t* n_out) {
  if (!c || !n_out) return FDTD_E_ARG;
  fdtd_status st = check_async(c, true);
  if (st != FDTD_OK) return st;
  const int64_t n = c->energy_on ? c->steps - c->rd_energy : 0;
  if (n > cap) return fail(c, FDTD_E_ARG, "output holds %lld steps, %lld pending", (long long)cap, (long long)n);
  *n_out = n;
  if (n == 0) return FDTD_OK;
  if (!out) return FDTD_E_ARG;
  st = read_ring(c, c->d_energy_ring, 1, 8, c->rd_energy, c->steps, NCCL_F64, out, cap);
  if (st != FDTD_OK) return st;
  c->rd_energy = c->steps;
  return FDTD_OK;
}

static fdtd_status window_io(fdtd_ctx* c, int64_t i0, int64_t j0, int64_t w, int64_t h, double* Ex, double* Ey,
                             double* Hz, bool set) {
  if (!c || w < 0 || h < 0 || i0 < 0 || j0 < 0 || i0 + w > c->d.nx || j0 + h > c->d.ny)
    return fail(c, FDTD_E_ARG, "bad window");
  fdtd_status st = check_async(c);
  if (st != FDTD_OK) return st;
  const int q = c->cur;
  const int64_t rb = c->d.row_begin, re = c->d.row_end;
  const size_t es = c->es;
  // arrays: (ptr, ncols, global row range [g0, g1), device array, row range owned, col limit stored)
  struct A { double* p; int64_t cols; int64_t g0, g1; int a; };
  A arr[3] = {{Ex, w, j0, j0 + h + 1, 0}, {Ey, w + 1, j0, j0 + h, 1}, {Hz, w, j0, j0 + h, 2}};
  std::vector<char> stg;
  for (auto& x : arr) {
    if (!x.p) continue;
    const int64_t a0 = std::max(x.g0, rb), a1 = std::min(x.g1, re);
    if (a1 <= a0) continue;
    const int64_t nrow = a1 - a0;
    const int64_t cstore = std::min<int64_t>(x.cols, c->pitch - i0);  // columns stored on device
    if (cstore <= 0) continue;
    stg.assign((size_t)nrow * cstore * es, 0);
    char* dev = (char*)c->f[q][x.a] + ((size_t)lrow(c, a0) * c->pitch + i0) * es;
    if (!set) {
      CK(cudaMemcpy2DAsync(stg.data(), cstore * es, dev, c->pitch * es, cstore * es, nrow, cudaMemcpyDeviceToHost,
                           c->stream));
      CK(cudaStreamSynchronize(c->stream));
      for (int64_t r = 0; r < nrow; ++r)
        for (int64_t k = 0; k < x.cols; ++k) {
          double v = 0.0;
          if (k < cstore) v = c->prec == 64 ? ((double*)stg.data())[r * cstore + k] : ((float*)stg.data())[r * cstore + k];
          x.p[(a0 - x.g0 + r) * x.cols + k] = v;
        }
    } else {
      for (int64_t r = 0; r < nrow; ++r)
        for (int64_t k = 0; k < cstore; ++k) {
          const int64_t g = a0 + r, col = i0 + k;
          double v = x.p[(a0 - x.g0 + r) * x.cols + k];
          if (x.a == 0 && (g == 0 || g == c->d.ny)) v = 0.0;      // PEC Ex rows
          if (x.a == 1 && (col == 0 || col >= c->d.nx)) v = 0.0;  // PEC Ey columns
          if (x.a != 1 && col >= c->d.nx) v = 0.0;
          if (c->prec == 64) ((double*)stg.data())[r * cstore + k] = v;
          else ((float*)stg.data())[r * cstore + k] = (float)v;
        }
      CK(cudaMemcpy2DAsync(dev, c->pitch * es, stg.data(), cstore * es, cstore * es, nrow, cudaMemcpyHostToDevice,
                           c->stream));
      CK(cudaStreamSynchronize(c->stream));
    }
  }
  if (set && !c->inst_model.empty()) {  // keep ROM holes at zero (interface edges keep the given y)
    int32_t* drect = nullptr;
    if ((st = upload(c, &drect, c->rects)) != FDTD_OK) return st;
    const int64_t nr = (int64_t)c->rects.size() / 4;
    if (c->prec == 64) {
      double* fl[6] = {(double*)c->f[q][0], (double*)c->f[q][1], (double*)c->f[q][2],
                       (double*)c->f[q][0], (double*)c->f[q][1], (double*)c->f[q][2]};
      fdtd::launch_mask<double>(nullptr, fl, c->pitch, drect, nr, rb, ROW0, false, c->stream);
    } else {
      float* fl[6] = {(float*)c->f[q][0], (float*)c->f[q][1], (float*)c->f[q][2],
                      (float*)c->f[q][0], (float*)c->f[q][1], (float*)c->f[q][2]};
      fdtd::launch_mask<float>(nullptr, fl, c->pitch, drect, nr, rb, ROW0, false, c->stream);
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
    dfree(c, drect);
  }
  return FDTD_OK;
}

fdtd_status fdtd_get_window(fdtd_ctx* c, int64_t i0, int64_t j0, int64_t w, int64_t h, double* Ex, double* Ey,
                            double* Hz) {
  return window_io(c, i0, j0, w, h, Ex, Ey, Hz, false);
}

fdtd_status fdtd_set_window(fdtd_ctx* c, int64_t i0, int64_t j0, int64_t w, int64_t h, const double* Ex,
                            const double* Ey, const double* Hz) {
  return window_io(c, i0, j0, w, h, const_cast<double*>(Ex), const_cast<double*>(Ey), const_cast<double*>(Hz), true);
}

fdtd_status fdtd_set_random_fields(fdtd_ctx* c, uint64_t seed, double amplitude) {
  if (!c || !(amplitude >= 0.0)) return FDTD_E_ARG;
  fdtd_status st = check_async(c);
  if (st != FDTD_OK) return st;
  const int q = c->cur;
  const double ah = amplitude / (MU0 * C0);  // |H| ~ |E| / eta0
  if (c->prec == 64)
    fdtd::launch_random_fields<double>((double*)c->f[q][0], (double*)c->f[q][1], (double*)c->f[q][2],
                                       (const double*)c->coef[0], c->pitch, c->d.nx, c->rows, ROW0, c->d.row_begin,
                                       seed, amplitude, ah, c->stream);
  else
    fdtd::launch_random_fields<float>((float*)c->f[q][0], (float*)c->f[q][1], (float*)c->f[q][2],
                                      (const float*)c->coef[0], c->pitch, c->d.nx, c->rows, ROW0, c->d.row_begin,
                                      seed, amplitude, ah, c->stream);
  CK(cudaGetLastError());
  return FDTD_OK;
}

fdtd_status fdtd_get_rom_state(fdtd_ctx* c, double* out, int64_t cap, int64_t* n) {
  if (!c || !n) return FDTD_E_ARG;
  fdtd_status st = check_async(c);
  if (st != FDTD_OK) return st;
  *n = c->state_len;
  if (c->state_len == 0) return FDTD_OK;
  if (cap < c->state_len || !out) return fail(c, FDTD_E_ARG, "rom state buffer too small");
  std::vector<char> h(c->state_len * c->es);
  CK(cudaMemcpy(h.data(), c->d_state, h.size(), cudaMemcpyDeviceToHost));
  for (int64_t k = 0; k < c->state_len; ++k)
    out[k] = c->prec == 64 ? ((double*)h.data())[k] : (double)((float*)h.data())[k];
  return FDTD_OK;
}

fdtd_status fdtd_set_rom_state(fdtd_ctx* c, const double* in, int64_t n) {
  if (!c || n != c->state_len || (n > 0 && !in)) return fail(c, FDTD_E_ARG, "rom state length mismatch");
  fdtd_status st = check_async(c);
  if (st != FDTD_OK) return st;
  if (n == 0) return FDTD_OK;
  std::vector<double> v(in, in + n);
  if (c->prec == 64) {
    CK(cudaMemcpy(c->d_state, v.data(), n * 8, cudaMemcpyHostToDevice));
  } else {
    std::vector<float> f(v.begin(), v.end());
    CK(cudaMemcpy(c->d_state, f.data(), n * 4, cudaMemcpyHostToDevice));
  }
  return FDTD_OK;
}

fdtd_status fdtd_step_group(fdtd_ctx** g, int32_t n, int64_t nsteps) {
  if (!g || n < 1 || nsteps < 0) return FDTD_E_ARG;
  for (int k = 0; k < n; ++k) {
    fdtd_ctx* c = g[k];
    if (!c || c->d.rank != k || c->d.nranks != n || !(c->d.flags & FDTD_LOCAL_GROUP) || c->stream != g[0]->stream ||
        c->steps != g[0]->steps || c->cur != g[0]->cur || c->prec != g[0]->prec || c->pitch != g[0]->pitch)
      return c ? fail(c, FDTD_E_ARG, "context %d is not rank %d of a local group of %d on one stream", k, k, n)
               : FDTD_E_ARG;
    int64_t oldest = c->steps + nsteps;
    if (c->n_probe > 0) oldest = std::min(oldest, c->rd_probe);
    if (c->energy_on) oldest = std::min(oldest, c->rd_energy);
    if (c->steps + nsteps - oldest > c->cap) return fail(c, FDTD_E_STATE, "unread records would overflow");
  }
  cudaStream_t s = g[0]->stream;
  int k = KMAX;  // pass depth: the deepest every slab can do
  for (int r = 0; r < n; ++r) {
    fdtd_ctx* c = g[r];
    if (c->kz_dirty) {
      int want = std::max(1, std::min(c->k_want, c->V));
      int kk = want >= 4 ? 4 : want >= 2 ? 2 : 1;
      while (kk > 1 && !passes_valid(c, kk)) kk /= 2;
      c->k_ok = kk;
    } else {
      c->k_ok = c->kz;
    }
    k = std::min(k, c->k_ok);
  }
  for (int r = 0; r < n; ++r)
    if (g[r]->kz_dirty || g[r]->kz != k) {
      fdtd_status st = apply_passes(g[r], k);
      if (st != FDTD_OK) return st;
    }
  int64_t left = nsteps;
  while (left > 0) {
    const int K = left >= k ? k : left >= 2 ? 2 : 1;
    const int q = g[0]->cur;
    for (int r = 0; r < n; ++r) {
      fdtd_status st = halo_local(g, n, r, q, s, K);
      if (st != FDTD_OK) return st;
    }
    for (int r = 0; r < n; ++r) {
      fdtd_status st = enqueue_pass(g[r], q, s, K);
      if (st != FDTD_OK) return st;
      g[r]->steps += K;
      g[r]->cur ^= 1;
    }
    left -= K;
  }
  fdtd_ctx* c = g[0];
  CK(cudaGetLastError());
  return FDTD_OK;
}

fdtd_status fdtd_set_pml(fdtd_ctx* c, int32_t width, int32_t order, double r0) {
  if (!c) return FDTD_E_ARG;
  if (width < 0 || order < 0 || order > 8 || !(r0 > 0 && r0 < 1)) return fail(c, FDTD_E_ARG, "bad CPML parameters");
  if (2 * (width + 4) > c->d.nx) return fail(c, FDTD_E_ARG, "CPML layers of %d cells do not fit nx = %lld", width,
                                             (long long)c->d.nx);
  for (size_t r = 0; width > 0 && r < c->rects.size(); r += 4)  // rings 3 cells clear of the layers (K = 1)
    if (c->rects[r] - 1 < width + 3 || c->rects[r] + c->rects[r + 2] + 1 > c->d.nx - width - 3)
      return fail(c, FDTD_E_ARG, "a ROM instance lies within the CPML band");
  fdtd_status st;
  for (void** pp : {&c->d_pml_bh, &c->d_pml_ah, &c->d_pml_be, &c->d_pml_ae, &c->d_psih, &c->d_psie})
    if (*pp) { dfree(c, *pp); *pp = nullptr; }
  c->pml_w = width;
  if (width > 0) {
    // sigma(d) = sigma_max d^order, sigma_max = (order + 1) ln(1/R0) / (2 eta0 width dx); b = exp(-sigma dt / eps0),
    // a = b - 1 (kappa 1, alpha 0); d = depth from the layer's inner face, per column position
    const double eta0 = std::sqrt(MU0 / EPS0);
    const double smax = (order + 1) * std::log(1.0 / r0) / (2.0 * eta0 * width * c->d.dx);
    auto bcoef = [&](double d) { return std::exp(-(d > 0 ? smax * std::pow(d, order) : 0.0) * c->d.dt / EPS0); };
    const int64_t nx = c->d.nx;
    std::vector<double> bh(2 * width), ah(2 * width), be(2 * (width + 1)), ae(2 * (width + 1));
    for (int k = 0; k < width; ++k) {  // Hz columns: left i = k, right i = nx - width + k
      const double dl = (width - k - 0.5) / width, dr = (k + 0.5) / width;
      bh[k] = bcoef(dl); ah[k] = bh[k] - 1.0;
      bh[width + k] = bcoef(dr); ah[width + k] = bh[width + k] - 1.0;
    }
    for (int k = 0; k <= width; ++k) {  // Ey columns: left i = k, right i = nx - width + k
      const double dl = (double)(width - k) / width, dr = (double)k / width;
      be[k] = bcoef(dl); ae[k] = be[k] - 1.0;
      be[width + 1 + k] = bcoef(dr); ae[width + 1 + k] = be[width + 1 + k] - 1.0;
    }
    (void)nx;
    if ((st = upload_T(c, &c->d_pml_bh, bh)) != FDTD_OK) return st;
    if ((st = upload_T(c, &c->d_pml_ah, ah)) != FDTD_OK) return st;
    if ((st = upload_T(c, &c->d_pml_be, be)) != FDTD_OK) return st;
    if ((st = upload_T(c, &c->d_pml_ae, ae)) != FDTD_OK) return st;
    c->d_psih = dalloc(c, (size_t)4 * c->nrows_alloc * width * c->es);        // [buffer][side][row][col]
    c->d_psie = dalloc(c, (size_t)4 * c->nrows_alloc * (width + 1) * c->es);
    if (!c->d_psih || !c->d_psie) return fail(c, FDTD_E_NOMEM, "CPML state");
  }
  c->kz_dirty = true;
  drop_graph(c);
  CK(cudaStreamSynchronize(c->stream));
  return FDTD_OK;
}

fdtd_status fdtd_set_time_blocking(fdtd_ctx* c, int32_t steps_per_pass) {
  if (!c || (steps_per_pass != 1 && steps_per_pass != 2 && steps_per_pass != 4)) return FDTD_E_ARG;
  c->k_want = steps_per_pass;
  c->kz_dirty = true;
  drop_graph(c);
  return FDTD_OK;
}

fdtd_status fdtd_profile(fdtd_ctx* c, int32_t on) {
  if (!c) return FDTD_E_ARG;
  c->profiling = on != 0;
  c->ev_used = 0;
  return FDTD_OK;
}

fdtd_status fdtd_profile_read(fdtd_ctx* c, double* sweep_ms, double* post_ms, int64_t* n) {
  if (!c || !sweep_ms || !post_ms || !n) return FDTD_E_ARG;
  CK(cudaStreamSynchronize(c->stream));
  double a = 0.0, b = 0.0;
  for (size_t k = 0; k + 3 <= c->ev_used; k += 3) {
    float t1 = 0.f, t2 = 0.f;
    CK(cudaEventElapsedTime(&t1, c->ev[k], c->ev[k + 1]));
    CK(cudaEventElapsedTime(&t2, c->ev[k + 1], c->ev[k + 2]));
    a += t1;
    b += t2;
  }
  *sweep_ms = a;
  *post_ms = b;
  *n = (int64_t)(c->ev_used / 3);
  c->ev_used = 0;
  return FDTD_OK;
}

fdtd_status fdtd_sync(fdtd_ctx* c) {
  if (!c) return FDTD_E_ARG;
  return check_async(c, true);
}

fdtd_status fdtd_get_info(const fdtd_ctx* c, fdtd_info* o) {
  if (!c || !o) return FDTD_E_ARG;
  o->steps_taken = c->steps;
  o->n_instances = (int64_t)c->inst_model.size();
  o->kernel_launches = c->launches;
  o->pitch = c->pitch;
  o->sweep_ctas = c->n_partials;
  o->graphs = !(c->d.flags & FDTD_NO_GRAPH) && !(c->d.flags & FDTD_LOCAL_GROUP) && !c->graph_broken;
  o->precision = c->prec;
  o->steps_per_pass = c->kz;
  // read Ex, Ey, Hz, mea, msb and write Ex, Ey, Hz once per pass
  o->bytes_per_cell_step = 8.0 * (double)c->es / o->steps_per_pass;
  o->sweep_stream = (void*)c->stream;
  o->graph_builds = c->graph_builds;
  o->fixup_clusters = c->n_clusters;
  o->big_instances = (int32_t)(c->batch_tab.size() / fdtd::BATCH_FIELDS) - c->n_batch_reg;
  if (c->inst_model.empty()) o->big_instances = 0;
  o->whole_grid = c->whole ? 1 : 0;
  return FDTD_OK;
}

fdtd_status fdtd_nccl_unique_id(void* out128) {
  std::string err;
  if (!out128) return FDTD_E_ARG;
  if (!g_nccl.load(err)) return FDTD_E_NCCL;
  nccl_uid id;
  if (g_nccl.GetUniqueId(&id) != 0) return FDTD_E_NCCL;
  memcpy(out128, &id, sizeof id);
  return FDTD_OK;
}

fdtd_status fdtd_halo_plan(int32_t nranks, int32_t rank, int64_t row_begin, int64_t row_end, int32_t depth,
                           int32_t pml, int64_t* out, int32_t cap, int32_t* n) {
  if (!n || nranks < 1 || rank < 0 || rank >= nranks || row_end - row_begin < 1 || depth < 1 || depth > KMAX ||
      (nranks > 1 && row_end - row_begin < KMAX) || cap < 0 || (cap > 0 && !out))
    return FDTD_E_ARG;
  std::vector<HaloRow> sends, recvs;
  halo_plan_rows(nranks, rank, row_end - row_begin, depth, pml != 0, sends, recvs);
  *n = (int32_t)(sends.size() + recvs.size());
  if (*n > cap) return FDTD_E_ARG;
  int k = 0;
  for (int dir = 0; dir < 2; ++dir)
    for (const HaloRow& x : dir ? recvs : sends) {
      out[4 * k + 0] = dir;
      out[4 * k + 1] = x.a;
      out[4 * k + 2] = row_begin + x.row - ROW0;  // global row (cell row for Ey / Hz / psi, edge row for Ex)
      out[4 * k + 3] = x.peer;
      ++k;
    }
  return FDTD_OK;
}

#if FDTD_PHASES
int fdtd_debug_phases(long long* out, int n) {  // tuning builds only (tools/phase_times.py)
  fdtd::debug_phases(out, n);
  return 0;
}
#endif

fdtd_status fdtd_pass_regions(const int32_t* rects, const int32_t* models, int64_t n, int32_t depth, int32_t* region,
                              int32_t* boxes, int64_t* n_regions) {
  if (n < 0 || (n > 0 && (!rects || !models || !region)) || depth < 1 || depth > KMAX || !n_regions) return FDTD_E_ARG;
  std::vector<int32_t> r(rects, rects + 4 * n), m(models, models + n);
  const std::vector<PassRegion> regs = pass_regions_of(r, m, depth);
  *n_regions = (int64_t)regs.size();
  for (size_t g = 0; g < regs.size(); ++g) {
    for (int i : regs[g].members) region[i] = (int32_t)g;
    if (boxes) {
      boxes[5 * g + 0] = (int32_t)regs[g].i0;
      boxes[5 * g + 1] = (int32_t)regs[g].j0;
      boxes[5 * g + 2] = (int32_t)(regs[g].i1 - regs[g].i0);
      boxes[5 * g + 3] = (int32_t)(regs[g].j1 - regs[g].j0);
      boxes[5 * g + 4] = regs[g].mixed ? 1 : 0;
    }
  }
  return FDTD_OK;
}

void fdtd_destroy(fdtd_ctx* c) {
  if (!c) return;
  if (c->stream) cudaStreamSynchronize(c->stream);
  drop_graph(c);
  for (auto e : c->ev) cudaEventDestroy(e);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  if (c->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(c->comm);
  if (c->edge_stream) cudaStreamDestroy(c->edge_stream);
  if (c->ev_edge_go) cudaEventDestroy(c->ev_edge_go);
  if (c->ev_edge) cudaEventDestroy(c->ev_edge);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  if (c->ev_ready) cudaEventDestroy(c->ev_ready);
  if (c->ev_halo) cudaEventDestroy(c->ev_halo);
  std::vector<void*> all = c->owned;
  for (void* p : all) dfree(c, p);
  delete c;
}

}  // extern "C"
