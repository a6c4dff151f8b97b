/*
 * fdtd_rom.h — C ABI of the whole-domain reduced model, batched over
 * excitations (the paper's own runtime mode, PAPER.md
 * P:176-211 and the "Proposed" rows of Tables II-VI).
 *
 * The reduced system (12) with the block structure (13)
 * is advanced in the leap-frog order of P:211.  Lossless, with diagonal reduced
 * mass blocks (D~ = I for a D-orthonormal basis, R5(vi)), one step
 * n -> n+1 of batch member b is
 *
 *   e~ <- e~ - g_e o (K~' h~) + g_e o (B~_e amp[:, b]) wave[n][b]      Eq. (12), E rows
 *   p_e  = L_e e~                                                     Eq. (10)
 *   h~ <- h~ + g_h o (K~'^T e~)                                       Eq. (12), H rows
 *   p_h  = L_h h~
 *
 * g_e = dt / diag(D~_eps), g_h = dt / diag(D~_mu) (inverse diagonal blocks of
 * R~ + F~, Eq. (13)); K~' is the stability-enforced reduced curl of §III-A
 * (P:283-303); B~_e = V1^T B_E (Eq. (16)) holds the source sign;
 * u^{n+1} = J^{n+1/2} (R2(i)); L_e / L_h are rows of V1 / V2.
 * All arithmetic is fp64 (the paper's MATLAB precision; DESIGN.md §5.8 explains
 * why fp32 cannot hold the north-star tolerance for this recursion): the two
 * products per step run on the fp64 tensor cores (mma.sync m8n8k4 f64) with K~'
 * resident in the register file for the whole launch.
 *
 * Arrays passed in are host pointers, BORROWED for the call and deep copied.
 * Every function returns FDTD_OK (0) or an FDTD_E* code of fdtd.h; the message
 * is in fdtd_last_error().  A handle is not thread-safe.
 */
#ifndef FDTD_ROM_H
#define FDTD_ROM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rom_t rom_t;

/* The reduced model (Eqs. (13)-(16)). */
typedef struct rom_model {
  int32_t q_e, q_h;        /* K~' is q_e x q_h (1 <= q <= 256)                                */
  int32_t n_in;            /* columns of B~_e (current sources)                                */
  int32_t n_out_e, n_out_h;/* probe rows (<= 64 each)                                          */
  const double* K;         /* [q_e][q_h] row-major                                             */
  const double* g_e;       /* [q_e]                                                            */
  const double* g_h;       /* [q_h]                                                            */
  const double* B_e;       /* [q_e][n_in]                                                      */
  const double* L_e;       /* [n_out_e][q_e] (NULL when n_out_e == 0)                          */
  const double* L_h;       /* [n_out_h][q_h] (NULL when n_out_h == 0)                          */
} rom_model;

/* The batch: member b is driven by u^{n+1}[:, b] = amp[:, b] * wave[n][b]
 * (a spatial pattern times a time signature; u = 0 for n >= n_wave). */
typedef struct rom_excitation {
  int32_t batch;           /* independent excitations (>= 1)                                   */
  const double* amp;       /* [n_in][batch]                                                    */
  int64_t n_wave;
  const double* wave;      /* [n_wave][batch] J^{n+1/2} samples                                */
} rom_excitation;

/* Validate, deep-copy, upload; zero initial state.  stream: a
 * cudaStream_t (NULL = default stream).  cols_per_cluster: 0 = auto, else 8,
 * 16 or 32 batch columns per CTA cluster. */
int rom_create(const rom_model* model, const rom_excitation* exc, void* stream, int32_t cols_per_cluster,
               rom_t** out);

/* Enqueue n time steps (one persistent launch; asynchronous). */
int rom_step(rom_t* h, int64_t n);

/* Synchronise; copy the probe series recorded since the last call as
 * out[step][n_out_e + n_out_h][batch] (fp64).  FDTD_EINVAL if cap is too small. */
int rom_probe(rom_t* h, double* out, int64_t cap, int64_t* written);

/* State access (synchronising): which = 0: e~ as [batch][q_e]; 1: h~ as
 * [batch][q_h]; 2: the step counter (n = 1). */
int rom_get_state(rom_t* h, int32_t which, double* out, int64_t n);
int rom_set_state(rom_t* h, int32_t which, const double* in, int64_t n);

int rom_sync(rom_t* h);

/* Launch geometry chosen at create: info[0] = CTAs per cluster, [1] = batch
 * columns per cluster, [2] = clusters, [3] = threads per CTA, [4] = padded q,
 * [5] = registers per thread of the kernel, [6] = kernel launches so far. */
int rom_info(const rom_t* h, int64_t* info, int32_t n);

/* Measured throughput [TFLOP/s] of a register-only mma.sync m8n8k4 f64 loop on
 * every SM: the roofline denominator of the reduced update (bench.py). */
double rom_dmma_peak_tflops(void* stream);

void rom_destroy(rom_t* h);

#ifdef __cplusplus
}
#endif
#endif /* FDTD_ROM_H */
