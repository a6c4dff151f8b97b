/*
 * fdtd.h — C ABI of the B200 hot path of structure-preserving reduced FDTD
 * (X. Li, C. D. Sarris, P. Triverio, arXiv 1406.7042).
 *
 * One time step n -> n+1 advances the reduced hybrid recursion (paper Eq. (4)
 * for the coarse grid, Eq. (12) for each reduced block; PAPER.md P:109-112,
 * P:182-185) written as the leap-frog of P:211:
 *
 *   coarse E   E   <- E - cb * (K_inc H)                     rows of (3)
 *   interface  E_r <- E_r - c_r * (sum_k W_rk H_k + y_r)       coarse/fine coupling
 *   sources    E_u <- E_u - coef_u * J_u^{n+1/2}               B u^{n+1}
 *   reduced E  e~  <- e~ - G_e (K~' h~)                        Eq. (12)/(13)
 *   coarse H   H   <- H + ch * (K_inc^T E)                     rows of (3)
 *   reduced H  h~  <- h~ + G_h (K~'^T e~ + S_E^T E_if)         Eq. (12), coupling
 *   coupling   y   <- S_E h~                                   (used by the next step)
 *
 * K_inc is the +-1 incidence of the uniform coarse Yee grid (paper K = K_inc /
 * delta), so every coefficient (cb = dt/(eps delta), ch = dt/(mu delta),
 * c_r, G) is an inverse diagonal block of (R+F) (Eq. (5)) supplied by
 * the caller in fp64 (reading R8).  K~' is the stability-enforced
 * reduced curl matrix of §III-A.
 *
 * Conventions
 *  - "storage index": each field component c lives on the index box
 *    (i, j, k) in [0,nx]x[0,ny]x[0,nz] (2-D: [0,nx]x[0,ny]), flat index
 *    s = (k*(ny+1) + j)*(nx+1) + i; S = number of storage indices.
 *    Component c = 0..5 is Ex(i+1/2,j,k) Ey(i,j+1/2,k) Ez(i,j,k+1/2)
 *    Hx(i,j+1/2,k+1/2) Hy(i+1/2,j,k+1/2) Hz(i+1/2,j+1/2,k); 2-D uses
 *    Ez(i,j)=2, Hx(i,j+1/2)=3, Hy(i+1/2,j)=4.
 *  - "unknown id" = c*S + s.
 *  - Entries that are not unknowns (PEC walls: tangential E and normal H on
 *    the outer boundary; indices past the component's extent) are held at 0.
 *  - Arrays passed in are BORROWED for the duration of the call and deep
 *    copied; the handle owns all device memory.  Host state buffers use the
 *    layout [batch][S] (fp64).
 *  - Every function returns FDTD_OK or an error code; fdtd_last_error()
 *    returns a thread-local message.  Errors detected asynchronously on the
 *    device (divergence) are reported by the next synchronising call.
 *  - A handle is not thread-safe; several handles may coexist.
 */
#ifndef FDTD_H
#define FDTD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FDTD_VERSION 100

enum {
  FDTD_OK = 0,
  FDTD_EINVAL = 1,     /* invalid argument: bad sizes, shape mismatch ("invalid-grid") */
  FDTD_ESTAMP = 2,     /* source / probe / interface index outside the grid      */
  FDTD_ENOMEM = 3,     /* device or host allocation failed                               */
  FDTD_ECUDA = 4,      /* CUDA runtime error (message in fdtd_last_error)               */
  FDTD_ENOTSUP = 5,    /* unsupported combination (e.g. non-cubic cells, no sm_100 GPU) */
  FDTD_EDIVERGED = 6   /* non-finite or |x| > 1e100 detected              */
};

typedef struct fdtd_t fdtd_t;

/* Grid (P:36 cell sizes; configs use cubic cells). */
typedef struct fdtd_grid {
  int32_t dim;          /* 2 (Ez/Hx/Hy, the paper's TM) or 3                     */
  int32_t nx, ny, nz;   /* coarse cells; nz = 1 when dim == 2                     */
  double dx, dy, dz;    /* cell sizes [m]; this version requires dx == dy (== dz) */
  int32_t batch;        /* B >= 1 independent excitations sharing all matrices    */
  int32_t precision;    /* 32 (fp32 storage + FFMA, hi/lo coefficients) or 64     */
  double dt;            /* time step [s] (informational; coefficients carry it)  */
} fdtd_grid;

/* Per-unknown coefficients through a material table (owning-cell
 * rule S:73).  coef[m][c] for E components is cb (E -= cb * sum(+-H)), for H
 * components ch (H += ch * sum(+-E)); 0 marks an inert unknown (PEC, or a
 * coarse unknown inside a refined box).  if_mask[m] bit c marks that E
 * component c at this storage index is an explicit row (see fdtd_interface):
 * its update is computed from the row, not from the stencil. */
typedef struct fdtd_materials {
  int32_t n_mat;            /* 0: uniform_coef everywhere, mat_id ignored (<= 256)   */
  const uint8_t* mat_id;    /* [S] material id per storage index                       */
  const double* coef;       /* [n_mat][6] cb_x cb_y cb_z ch_x ch_y ch_z                */
  const uint8_t* if_mask;   /* [n_mat]                                                  */
  double uniform_coef[6];
  /* Lossy media (sigma_e, sigma_m > 0; Eq. (2a)/(2b) P:64-74 with the
   * conductivity terms of D_sigma, Eq. (5)): E <- ca E - cb (K_inc H),
   * H <- da H + ch (K_inc^T E) with ca = (eps/dt - sigma_e/2)/(eps/dt + sigma_e/2),
   * cb = 1/((eps/dt + sigma_e/2) delta), da / ch likewise with mu, sigma_m.
   * coef_a[m][c] = ca (E components) / da (H components); NULL = lossless (all 1).
   * Matched absorbers are graded sigma layers expressed this way.
   * Lossy problems run the 3-D tile stencil or the per-step 2-D kernel; reduced
   * blocks and interface rows stay lossless. */
  const double* coef_a;     /* [n_mat][6] or NULL                                       */
} fdtd_materials;

/* Interface rows: coarse E unknowns on the surface of a refined box
 * (reading R4).  Row r: E_r -= c[r]*(sum_k val[k] H[col[k]] + y_r),
 * y_r = S_E[local[r]] . h~[block[r]][inst[r]] of the previous half step. */
typedef struct fdtd_interface {
  int64_t n_rows;
  const int64_t* unknown;   /* [n_rows] E unknown ids                      */
  const double* c;          /* [n_rows] c_r = dt / D_eps,r (lumped)        */
  const int64_t* rowptr;    /* [n_rows+1] CSR row pointers                  */
  const int64_t* col;       /* [nnz] H unknown ids                          */
  const double* val;        /* [nnz] W_if entries (scaled units)            */
  const int32_t* block;     /* [n_rows] reduced block                       */
  const int32_t* inst;      /* [n_rows] instance of that block              */
  const int32_t* local;     /* [n_rows] row of the block's S_E              */
} fdtd_interface;

/* One reduced model (Eqs. (12)-(16)), possibly shared by several
 * congruent regions ("instances").  State per instance and batch member:
 * e~ (qe), h~ (qh).  G_e = dt * D~_eps^{-1} and G_h = dt * D~_mu^{-1} must be
 * diagonal (scalar when the basis is D-orthonormal, R5(vi)). */
typedef struct fdtd_reduced_block {
  int32_t qe, qh;           /* K~' is qe x qh (the paper's N~ x N~)        */
  int32_t n_inst;           /* instances sharing the model                  */
  int32_t n_if;             /* rows of S_E (interface rows per instance)    */
  const double* K;          /* [qe][qh] row-major, stability-enforced K~'  */
  const double* S_E;        /* [n_if][qh] row-major coupling K_cf V2_f     */
  const double* g_e;        /* [qe] or NULL -> g_e_scalar                   */
  const double* g_h;        /* [qh] or NULL -> g_h_scalar                   */
  double g_e_scalar, g_h_scalar;
} fdtd_reduced_block;

/* Sources J on coarse E unknowns (u^{n+1} = J^{n+1/2}, R2(i)):
 * E_u -= coef_u * wave[n][col_u][b].  Sources sharing a time signature (a
 * current sheet, a gap source) share a waveform column and carry their
 * spatial amplitude in coef. */
typedef struct fdtd_sources {
  int64_t n_src;
  const int64_t* unknown;   /* [n_src] E unknown ids                                  */
  const double* coef;       /* [n_src] E -= coef * J  (coef = amplitude * dt / eps)   */
  const int32_t* column;    /* [n_src] waveform column; NULL -> column s for source s */
  int64_t n_cols;           /* waveform columns (n_src when column == NULL)           */
  int64_t n_wave;           /* samples per column; J = 0 for steps >= n_wave           */
  const double* wave;       /* [n_wave][n_cols][batch] J^{n+1/2} for step n           */
} fdtd_sources;

/* Probes (Eq. (10) P:170-175 for fine-region reconstruction).  kind 0: sum of
 * weight * coarse unknown (all E or all H); kind 1 / 2: weight . e~ / h~ of
 * (block, inst) (a row of V1_f / V2_f).  E is sampled after the E half, H
 * after the H half. */
typedef struct fdtd_probes {
  int64_t n_probe;
  const int32_t* kind;      /* [n_probe]                                   */
  const int64_t* rowptr;    /* [n_probe+1] term pointers                   */
  const int64_t* index;     /* kind 0: unknown id; kind 1/2: vector index  */
  const double* weight;     /* [n_terms]                                   */
  const int32_t* block;     /* [n_probe] (kind 1/2)                        */
  const int32_t* inst;      /* [n_probe] (kind 1/2)                        */
} fdtd_probes;

/* Execution context.  stream: a cudaStream_t (NULL = legacy default stream).
 * alloc/free: optional device allocator (e.g. PyTorch's caching allocator);
 * NULL -> cudaMalloc/cudaFree. */
typedef struct fdtd_exec {
  void* stream;
  void* (*alloc)(size_t bytes, void* ctx);
  void (*free)(void* ptr, void* ctx);
  void* alloc_ctx;
  int32_t check_every;      /* divergence check period in steps; 0 = off (default 100 if < 0) */
  int32_t graph_steps;      /* steps per captured CUDA graph (0 = no graphs; default 32 if < 0) */
  int64_t probe_capacity;   /* device probe ring in steps (0 = default 65536)                 */
  int32_t reduced_form;     /* 0 auto, 1 fused update matrix, 2 leap-frog GEMVs  */
} fdtd_exec;

/* Validate, deep-copy and upload everything; zero initial state.
 * blocks may be NULL when n_blocks == 0; iface / src / probes may be NULL. */
int fdtd_create(const fdtd_grid* grid, const fdtd_materials* mat, const fdtd_interface* iface,
                const fdtd_reduced_block* blocks, int32_t n_blocks, const fdtd_sources* src,
                const fdtd_probes* probes, const fdtd_exec* exec, fdtd_t** out);

/* Enqueue n time steps on the handle's stream (asynchronous). */
int fdtd_step(fdtd_t* h, int64_t n);

/* Synchronise; copy the probe series recorded since the last call as
 * out[step][probe][batch] (fp64); *written = number of doubles written.
 * FDTD_EINVAL if cap is too small (nothing is consumed). */
int fdtd_probe(fdtd_t* h, double* out, int64_t cap, int64_t* written);

/* State access (synchronising).  which = 0..5: coarse component c, n = batch*S,
 * layout [batch][S]; which = 6 / 7: all reduced e~ / h~, layout
 * [block][inst][batch][q]; which = 8: the step counter n (n = 1; it indexes
 * the source waveforms, so a restored checkpoint sets it too).  In 3-D,
 * fdtd_set_state stores E entries that are not unknowns (E tangential to the
 * PEC walls, Eq. (3) with PEC elimination) as 0 whatever `in` holds. */
int fdtd_get_state(fdtd_t* h, int32_t which, double* out, int64_t n);
int fdtd_set_state(fdtd_t* h, int32_t which, const double* in, int64_t n);

/* Block until all enqueued work is done; reports asynchronous errors. */
int fdtd_sync(fdtd_t* h);

/* Number of device kernel launches enqueued so far (each graph replay counts
 * its kernel nodes). */
int64_t fdtd_launch_count(const fdtd_t* h);

/* Which kernel paths fdtd_step takes (bit mask, fixed at fdtd_create):
 *   1  persistent on-chip-resident 2-D kernel (one cooperative launch per
 *      fdtd_step call; 2-D, batch 1, fused single-column reduced blocks)
 *   2  TMA 3-D stencil (else the cp.async one, in 3-D)
 *   4  cluster-split GEMM kernel for fused reduced blocks (else warp-per-row)
 *   8  leap-frog GEMV path for at least one large reduced block
 *  16  the 3-D tile stencil (W elements per thread, NS-plane TMA ring; with bit 2)
 *  32  tensor-core (tcgen05, 3xTF32) GEMM for y = S_E h~ of a batched leap-frog block
 *  64  explicit rows of the next step evaluated inside the batched reduced GEMM (no pre-pass
 *      launch in steady state; FDTD_NO_ROWFUSE=1 turns it off)
 * Environment overrides (testing): FDTD_PERSIST=0, FDTD_NO_TMA,
 * FDTD_FUSED=gemv|gemm, FDTD_KCHUNK=<planes>, FDTD_STENCIL_OLD=1 (the
 * reference TMA stencils instead of the tile stencil), FDTD_TILE=<W>,<NS>, FDTD_NO_TC=1
 * (SIMT GEMM instead of the tensor-core one). */
int32_t fdtd_path(const fdtd_t* h);

/* Per-phase tracing.  fdtd_profile(h, 1) resets the accumulators and makes the
 * following fdtd_step calls launch eagerly with CUDA events around each
 * kernel group (read back every 64 steps, so the stream stays busy and the
 * spans are kernel durations rather than launch latencies); fdtd_profile(h, 0) returns to
 * graph launches.  fdtd_phase_times writes the accumulated device time [ms] of
 * the phases {coarse stencil incl. explicit E rows, reduced chain incl.
 * probes, grid-path reduced kernels (large blocks only)} into ms[0..2] and,
 * if n > 3, the number of profiled steps into ms[3]. */
int fdtd_profile(fdtd_t* h, int32_t enable);
int fdtd_phase_times(fdtd_t* h, double* ms, int32_t n);

/* Halo exchange of a slab decomposition along z: copy
 * z-plane k (0..nz) of coarse component `which` (0..5) between the state and a
 * caller-owned DEVICE buffer of (ny+1)(nx+1)*batch values of the run precision,
 * layout [ny+1][nx+1][batch], on the handle's stream (asynchronous; ordered
 * after the steps enqueued so far).  dir 0: state -> buffer, 1: buffer ->
 * state.  3-D only.  paper_1406_7042_b200/dist.py (SlabSim) drives it: each
 * rank owns a slab with one ghost cell layer per internal side and receives
 * the tangential H of that layer after every step. */
int fdtd_plane_device(fdtd_t* h, int32_t which, int32_t k, void* dev_buf, int32_t dir);

void fdtd_destroy(fdtd_t* h);
const char* fdtd_last_error(void);
int fdtd_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FDTD_H */
