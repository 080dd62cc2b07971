/*
 * fdtdrom.h -- C ABI of the B200 time-marching hot path of
 * Zhang, Bekmambetova, Triverio, "A Stable FDTD Method with Embedded
 * Reduced-Order Models" (arXiv 1609.07114).  Implemented by
 * paper_1609_07114_b200/libfdtdrom.so (CUDA, sm_100a).
 *
 * The calls follow the paper's problem statement: "the
 * proposed scheme consists of conventional FDTD equations to update the coarse
 * grid, and (eq:connExplicit) to update the reduced model state and the
 * interface.  If multiple reduced models are present, (eq:connExplicit) is
 * applied to each one of them."
 *
 * Grid conventions (R1): coarse cells (i, j), 0-based, i along x.
 * Hz at cell centres [ny][nx]; Ex on x-directed edges [ny+1][nx] (edge row j
 * lies at y = j dy); Ey on y-directed edges [ny][nx+1] (edge column i lies at
 * x = i dx).  All host arrays are row-major with j slow.  SI units.  PEC outer
 * walls: Ex rows 0 and ny and Ey columns 0 and nx are identically zero.
 *
 * Ownership: every host input is copied before the call returns; the caller
 * keeps its buffers.  The context owns its device memory (obtained through the
 * optional allocator, so the PyTorch caching allocator can back it).  The
 * stream and the NCCL unique id are borrowed.
 *
 * Errors: every call returns an fdtd_status; no exception crosses the ABI.
 * fdtd_last_error() gives the text of the last failure of that context.
 * fdtd_step only enqueues work; asynchronous faults (CUDA errors, the
 * non-finite sentinel) surface at the next synchronous call (fdtd_probe,
 * fdtd_energy, fdtd_get_window, fdtd_get_rom_state, fdtd_sync).  The
 * non-finite sentinel ("instability detected") is a device
 * flag set at the end of every pass when a recorded energy value W^n (which
 * sums the square of every field value and ROM state), one of 256 Hz cells
 * sampled on a fixed stride pattern of the pass's output, or a stored ROM state
 * is not finite; it is sticky and turns every later synchronous call into
 * FDTD_E_UNSTABLE.
 *
 * Threading: a context is single-threaded; several contexts may coexist.
 *
 * Several ranks (nranks > 1, one process per GPU over NCCL): fdtd_create,
 * fdtd_add_rom, fdtd_set_probes, fdtd_set_pml, fdtd_set_time_blocking,
 * fdtd_step, fdtd_probe, fdtd_energy and fdtd_sync are collective -- every rank
 * calls them, in the same order (fdtd_add_rom with count 0 on a rank that owns
 * none of a model's instances); their validity checks are agreed over the ranks
 * so that all ranks fail together.  The other calls are rank-local.
 */
#ifndef FDTDROM_H
#define FDTDROM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fdtd_ctx fdtd_ctx;

typedef enum {
  FDTD_OK = 0,
  FDTD_E_ARG = 1,       /* invalid argument, placement or state                       */
  FDTD_E_STATE = 2,     /* call not valid now (e.g. record buffer would overflow)     */
  FDTD_E_PASSIVITY = 3, /* ROM violates eq:cond1rom / eq:cond2rom at dt (L713-719)     */
  FDTD_E_UNSTABLE = 4,  /* dt above eq.(1) (L36-38) or non-finite fields detected      */
  FDTD_E_CUDA = 5,
  FDTD_E_NCCL = 6,
  FDTD_E_NOMEM = 7
} fdtd_status;

/* fdtd_grid_desc.flags */
#define FDTD_MATERIALS_ON_DEVICE 0x1u /* eps_r / sigma are device pointers            */
#define FDTD_MATERIALS_F32 0x2u       /* eps_r / sigma are float (else double)        */
#define FDTD_ALLOW_DT_ABOVE_EQ1 0x4u  /* skip the eq.(1) check (e.g. tests of blow-up) */
#define FDTD_NO_GRAPH 0x8u            /* never capture CUDA graphs in fdtd_step        */
#define FDTD_LOCAL_GROUP 0x10u        /* rank of an in-process slab group (no NCCL; see
                                         fdtd_step_group)                               */
#define FDTD_NO_WHOLE 0x20u           /* never use the whole-grid path (K3c): small
                                         grids then also take the sweep + fix-up passes */

typedef struct {
  int64_t nx, ny;          /* global coarse cells                                         */
  double dx, dy, dt;       /* cell sizes and time step, SI                                */
  int32_t precision;       /* 32 (fp32 state) or 64 (fp64 state)                          */
  uint32_t flags;          /* FDTD_* flags above                                          */
  /* Per-cell relative permittivity and conductivity (S/m), row-major [rows][nx].  The
   * pointer addresses global row `materials_row0`; it must cover the rows
   * [max(row_begin-4, 0), min(row_end+4, ny)) of the grid (the slab plus the ghost rows a
   * four-step pass recomputes).  Edge values are the arithmetic mean of
   * the two adjacent cells (R2).  mu = mu0 everywhere
   * (R3).  Host or device memory (FDTD_MATERIALS_ON_DEVICE), double or float
   * (FDTD_MATERIALS_F32). */
  const void *eps_r, *sigma;
  int64_t materials_row0;
  int32_t device;          /* CUDA device ordinal                                         */
  void *stream;            /* cudaStream_t work is ordered on (borrowed); NULL: legacy     */
  /* optional allocator (e.g. the PyTorch caching allocator); NULL: cudaMalloc/cudaFree  */
  void *(*alloc)(size_t bytes, void *user);
  void (*free)(void *ptr, void *user);
  void *alloc_user;
  /* row-slab decomposition: this rank owns coarse cell rows
   * [row_begin, row_end) and Ex edge rows [row_begin, row_end).  nranks == 1: the
   * whole grid (row_begin = 0, row_end = ny). */
  int32_t nranks, rank;
  const void *nccl_id;     /* 128-byte ncclUniqueId (same on every rank); NULL if nranks == 1 */
  int64_t row_begin, row_end;
  int64_t record_capacity; /* steps of probe / energy records kept on device (0: 65536)  */
} fdtd_grid_desc;

/* Create a context: validates the descriptor, builds the per-edge update
 * coefficients of eq:updateEx (L209-214) on the device, allocates the fields
 * (zero) and checks dt against eq.(1) (L36-38) with c_max = c0/sqrt(min eps_r).
 * FDTD_E_UNSTABLE if dt exceeds eq.(1) and FDTD_ALLOW_DT_ABOVE_EQ1 is not set.
 * Device materials (FDTD_MATERIALS_ON_DEVICE) must be ready on desc->stream (the copy is
 * ordered on that stream only).  With NCCL ranks the communicator is created first and the
 * global minimum eps_r / sigma (over all ranks' rows) decides the eq.(1) check on every rank;
 * FDTD_E_ARG (on every rank) if a slab holds fewer than 4 rows (the deepest pass sends 4 owned
 * rows to each neighbour). */
fdtd_status fdtd_create(const fdtd_grid_desc *desc, fdtd_ctx **out);

/* One reduced model, as emitted by the ROM generator (fp64, row-major, host):
 * R11 (q1 x q1), R22 (q2 x q2), F11 (q1 x q1), K (q1 x q2), L (q1 x nY) with
 * nY = 2 bx + 2 by ports ordered S (bx, left->right), N (bx), W (by,
 * bottom->top), E (by).  These are R~11, R~22, F~11, K~, L~ of eq:rom1a/b and
 * eq:R11_tilde..eq:K_tilde (L406-447) after the exact collapse onto coarse-edge
 * ports (R9); B~ = L~ S_c is implied with S_c = diag(-dx, +dx, +dy,
 * -dy) per side (eq:cond3rom L717, eq:S L698-707).  r is informational. */
typedef struct {
  int32_t bx, by, r, q1, q2;
  const double *R11, *R22, *F11, *K, *L;
  /* 0: collapsed ports (L is q1 x nY, R9).  1: the paper-literal coupling (NEXT-1):
   * L is q1 x nP with nP = r nY fine hanging variables in the same side order (fine port k on
   * coarse port k / r), B~ = L~ S_f with S_f = S_c / r, coupled by eq:sysform with T and 1/r
   * (eq:equalE, eq:averH L613-616); FDTD_E_ARG if that A1 is singular (the E basis
   * must span the nP port directions, which needs q1 >= nP). */
  int32_t literal;
} fdtd_rom_model;

/* Embed `count` instances of one model with lower-left coarse cells anchors[2k],
 * anchors[2k+1] (global (i0, j0)).  Each instance occupies cells [i0, i0+bx) x
 * [j0, j0+by); it is coupled through eq:updateExboundary (L461-468, coarse half
 * cell outside the block) and eq:connExplicit (L666-675), evaluated in an
 * equivalent factored form.
 * Checks: FDTD_E_PASSIVITY if R~(dt) is not positive definite (eq:cond1rom) or
 * F~11 + F~11^T has an eigenvalue below -1e-12 |F| (eq:cond2rom); FDTD_E_ARG if
 * a footprint plus its one-cell ring leaves this rank's rows, touches the PEC
 * wall, or overlaps another instance's footprint plus ring.  On success
 * *model_id receives the model's index. */
fdtd_status fdtd_add_rom(fdtd_ctx *c, const fdtd_rom_model *m, const int32_t *anchors,
                         int64_t count, int32_t *model_id);

/* Soft Hz source (R15): after the H half-step of step n,
 * Hz[j][i] += samples[n - step0] for step0 <= n < step0 + n_samples, else 0.
 * Replaces any previous source.  A cell outside this rank's rows is ignored. */
fdtd_status fdtd_set_source(fdtd_ctx *c, int64_t i, int64_t j, const double *samples,
                            int64_t n_samples, int64_t step0);

/* Soft Hz line source on the cells (i, j0 .. j1-1), every cell driven by the same samples (the
 * "line source" that excites the paper's waveguides, L882, L945; NEXT-2).  Replaces any previous
 * source.  fdtd_set_source(i, j) is the line (i, j .. j). */
fdtd_status fdtd_set_source_line(fdtd_ctx *c, int64_t i, int64_t j0, int64_t j1, const double *samples,
                                 int64_t n_samples, int64_t step0);

/* Probes: record Hz^{n+1/2} at cells ij[2p], ij[2p+1] after every step n (R16).  Replaces any
 * previous set; the record of a probe in another rank's rows reads 0 on this rank. */
fdtd_status fdtd_set_probes(fdtd_ctx *c, const int64_t *ij, int32_t n_probes);

/* Record the storage function W^n (R17) every step (1) or not (0). */
fdtd_status fdtd_record_energy(fdtd_ctx *c, int32_t on);

/* Enqueue `nsteps` time steps on the context's stream (asynchronous).  Each step:
 * H half-step (eq:updateH), source, probes and energy, per-ROM gather / reduced
 * update / scatter (eq:connExplicit), E half-step (eq:updateEx) -- S1..S8 of
 * DESIGN.md.  FDTD_E_STATE if the unread probe/energy records would exceed
 * record_capacity.  Large grids run K-step passes (sweep + ROM fix-up, CUDA graphs); a small
 * single-rank grid with a few instances of one model runs the whole call as one kernel launch
 * (fdtd_info.whole_grid; FDTD_NO_WHOLE opts out) -- the results are bit-identical either way. */
fdtd_status fdtd_step(fdtd_ctx *c, int64_t nsteps);

/* In-process slab group (testing the decomposition on one device): contexts created with
 * FDTD_LOCAL_GROUP, nranks = n, rank = k (k = 0..n-1, ctxs[k] has rank k), all on the same
 * stream.  Enqueues `nsteps` steps of every slab; before each step the halo rows move by
 * device copies following exactly the NCCL exchange plan of fdtd_step.  Probe and energy
 * records stay per slab (the caller sums them). */
fdtd_status fdtd_step_group(fdtd_ctx **ctxs, int32_t n, int64_t nsteps);

/* Read and consume the probe records of the steps taken since the last read:
 * out[p * cap_steps + k] (row-major [n_probes][cap_steps]), k = 0 .. *n_steps-1.
 * With several ranks, probes are summed over ranks (each cell lives on one rank).
 * Synchronous. */
fdtd_status fdtd_probe(fdtd_ctx *c, double *out, int64_t cap_steps, int64_t *n_steps);

/* Read and consume the energy records W^n of the steps since the last read
 * (fp64, summed over ranks).  Synchronous. */
fdtd_status fdtd_energy(fdtd_ctx *c, double *out, int64_t cap, int64_t *n);

/* Copy a window of the global fields to / from host fp64 arrays: Hz cells
 * [i0, i0+w) x [j0, j0+h) -> Hz[h][w]; Ex edges [i0, i0+w) x rows [j0, j0+h]
 * -> Ex[h+1][w]; Ey edges columns [i0, i0+w] x rows [j0, j0+h) -> Ey[h][w+1].
 * Only rows owned by this rank are transferred; NULL pointers are skipped.
 * fdtd_set_window also zeroes ROM hole cells/edges and keeps PEC walls zero.
 * Synchronous. */
fdtd_status fdtd_get_window(fdtd_ctx *c, int64_t i0, int64_t j0, int64_t w, int64_t h,
                            double *Ex, double *Ey, double *Hz);
fdtd_status fdtd_set_window(fdtd_ctx *c, int64_t i0, int64_t j0, int64_t w, int64_t h,
                            const double *Ex, const double *Ey, const double *Hz);

/* Seeded random initial fields on the device (R26, the random-init state of the tests
 * at any grid size): every live Hz cell and every live Ex / Ey edge of this rank's rows gets
 * amplitude * u (E) or amplitude / eta0 * u (H), u in [-1, 1) a hash of (seed, component, global
 * row, column) -- so every row-slab decomposition gets the same state.  Dead cells and edges (PEC
 * walls, ROM holes, interface edges) keep their values, so the state stays consistent with the ROM
 * states (y = L~^T E~).  Asynchronous on the stream; amplitude < 0: FDTD_E_ARG. */
fdtd_status fdtd_set_random_fields(fdtd_ctx *c, uint64_t seed, double amplitude);

/* ROM states x~ = [E~; H~] (q1 + q2 per instance, instances in the order they were
 * added on this rank), fp64.  Synchronous. */
fdtd_status fdtd_get_rom_state(fdtd_ctx *c, double *out, int64_t cap, int64_t *n);
fdtd_status fdtd_set_rom_state(fdtd_ctx *c, const double *in, int64_t n);

/* Block until all enqueued work finished; reports asynchronous faults. */
fdtd_status fdtd_sync(fdtd_ctx *c);

/* Introspection (host values; no synchronisation). */
typedef struct {
  int64_t steps_taken;         /* steps enqueued so far                                    */
  int64_t n_instances;         /* ROM instances on this rank                               */
  int64_t kernel_launches;     /* kernels launched by fdtd_step so far (graph nodes count)  */
  int64_t pitch;               /* elements per device row                                  */
  int64_t sweep_ctas;          /* CTAs of one fused-sweep launch                           */
  int32_t graphs;              /* 1 if fdtd_step replays CUDA graphs                       */
  int32_t precision;
  double bytes_per_cell_step;  /* HBM bytes of the sweep per cell-step as implemented       */
  int32_t steps_per_pass;      /* time steps per sweep pass in use (1, 2 or 4)              */
  void *sweep_stream;          /* cudaStream_t the kernels are launched on                 */
  int64_t graph_builds;        /* CUDA graphs captured so far (a new source window on the same
                                  cells, or a new probe/energy read, keeps the graph)          */
  int32_t fixup_clusters;      /* fix-up regions shared by several instances closer than the pass
                                  depth allows                        */
  int32_t big_instances;       /* instances on the cooperative large-model path                */
  int32_t whole_grid;          /* 1: fdtd_step runs the whole grid and its ROM instances in one
                                  CTA, one launch per call (single rank, no CPML, one model of
                                  fewer than 512 states, <= 64 instances, the grid and the batch
                                  in one CTA's shared memory; K3c)                   */
} fdtd_info;
fdtd_status fdtd_get_info(const fdtd_ctx *c, fdtd_info *out);

/* Kernel timing (for bench.py's roofline): while on, fdtd_step launches eagerly and brackets
 * every sweep and post launch with CUDA events on the context's stream.  fdtd_profile_read
 * synchronises and returns the summed device milliseconds and the launch count since the
 * last read. */
fdtd_status fdtd_profile(fdtd_ctx *c, int32_t on);
fdtd_status fdtd_profile_read(fdtd_ctx *c, double *sweep_ms, double *post_ms, int64_t *n_launches);

/* Time steps per sweep pass K: 1, 2 or 4 (temporal blocking with a per-instance fix-up,
 * DESIGN.md K1/K3; default: 4 in fp32, 2 in fp64 -- a 16-byte vector must hold K columns).
 * K-step passes are used when every ROM instance's fix-up region [i0-(2K-1), i0+bx+2K-1) x
 * [j0-(2K-1), j0+by+2K-1) lies inside the grid columns and this rank's rows, and no two
 * instances' [i0-K, i0+bx+K) x [j0-K, j0+by+K) rectangles meet -- on every rank (agreed
 * collectively at the first fdtd_step after a configuration change; the halo exchange is then K
 * rows deep); otherwise the deepest valid K below is used.  A step count that is not a multiple
 * of K ends with shallower passes.  Fields, ROM states and probes are bit-identical for every
 * K; the energy trace agrees up to summation order. */
fdtd_status fdtd_set_time_blocking(fdtd_ctx *c, int32_t steps_per_pass);

/* CPML absorbing layers (NEXT-2) of `width` cells at both x-ends (x < width dx and x > (nx - width) dx),
 * backed by the PEC walls, for the paper's PML-terminated waveguides (L882, L945): Roden-Gedney
 * recursive convolution with kappa = 1, alpha = 0, sigma(d) = sigma_max d^order with
 * sigma_max = (order + 1) ln(1/r0) / (2 eta0 width dx), d the depth from the layer's inner face;
 * b = exp(-sigma dt / eps0), a = b - 1; psi_hz = b psi_hz + a dEy/dx (Hz -= dt/mu0 psi_hz),
 * psi_ey = b psi_ey + a dHz/dx (Ey's curl term -dHz/dx becomes -(dHz/dx + psi_ey)).  width 0
 * removes the layers.  The layer cells stay in the storage function (their standard terms).
 * With row slabs every rank calls it with the same arguments; the psi rows of the ghost rows
 * travel with the halo exchange (psi_ey with Ey, psi_hz with Hz).  FDTD_E_ARG when
 * 2 (width + 4) > nx, or when a ROM instance's ring comes within 3 cells of a layer (K-step
 * passes need 2K + 1; shallower passes are used otherwise).  Resets the auxiliary state. */
fdtd_status fdtd_set_pml(fdtd_ctx *c, int32_t width, int32_t order, double r0);

/* Tuning knobs for the fused sweep (rows per CTA, warps per CTA); 0 keeps default. */
fdtd_status fdtd_set_tuning(fdtd_ctx *c, int32_t rows_per_cta, int32_t warps_per_cta);

/* Halo plan of one K-step pass (no paper counterpart -- the row-slab
 * decomposition of north_star (4)): the rows rank `rank` of `nranks` (owning global cell rows
 * and Ex edge rows [row_begin, row_end)) sends to and receives from its neighbours before a pass
 * of `depth` (1..4) steps, in the order both transports pair them.  Host-only (no context, no
 * device).  out[4k .. 4k+3] = {direction (0 send, 1 receive), array (0 Ex edge row, 1 Ey cell
 * row, 2 Hz cell row; with pml != 0 also 3 / 4 psi_ey of the left / right CPML layer and 5 / 6
 * psi_hz), global row, peer rank}; sends first, then receives; *n = number of entries.
 * FDTD_E_ARG on bad sizes, a slab shorter than 4 rows with nranks > 1, or cap < *n (then *n
 * still holds the count). */
fdtd_status fdtd_halo_plan(int32_t nranks, int32_t rank, int64_t row_begin, int64_t row_end, int32_t depth,
                           int32_t pml, int64_t *out, int32_t cap, int32_t *n);

/* Fix-up regions of a `depth`-step pass (the temporal blocking of
 * north_star (2), no paper counterpart): instances (rects[4k..4k+3] = i0, j0, bx, by; models[k] their
 * model) whose blocks grown by `depth` cells meet, directly or through others, share one region --
 * merged into their bounding box until no two regions' boxes grown by `depth` meet.  Host-only.
 * region[k] receives instance k's region index; boxes (optional, 5 per region) the region's
 * (i0, j0, width, height, mixed-models flag); *n_regions the count.  depth 1: one region per
 * instance. */
fdtd_status fdtd_pass_regions(const int32_t *rects, const int32_t *models, int64_t n, int32_t depth,
                              int32_t *region, int32_t *boxes, int64_t *n_regions);

/* Fill out[128] with a fresh ncclUniqueId (rank 0 calls it and broadcasts the bytes, e.g. with
 * torch.distributed.broadcast).  FDTD_E_NCCL if libnccl.so.2 cannot be loaded. */
fdtd_status fdtd_nccl_unique_id(void *out128);

const char *fdtd_last_error(const fdtd_ctx *c);
const char *fdtd_status_string(fdtd_status s);
void fdtd_destroy(fdtd_ctx *c);

#ifdef __cplusplus
}
#endif
#endif /* FDTDROM_H */
