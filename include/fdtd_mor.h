/*
 * fdtd_mor.h — C ABI of the offline reduction on the device (SURVEY §8(f)
 * NEXT-1; the paper's dominant 3-D cost and its stated future work, PAPER.md
 * P:354-393).
 *
 * The lossless fine-region system (R + F) x^{n+1} = (R - F) x^n + B u^{n+1}
 * (Eq. (4)-(6)) with diagonal masses is given by (De, Dm, K, dt):
 *
 *   R + F = [ De/dt    0    ]      R - F = [ De/dt   -K    ]
 *           [ -K^T    Dm/dt ]              [  0      Dm/dt ]
 *
 * so A(z) = z (R + F) - (R - F) (the shifted operator, P:358 with the sign of
 * DESIGN.md reading R5(i)) has the blocks of P:373-392
 *
 *   A11 = (z-1) De/dt,  A12 = K,  A21 = -z K^T,  A22 = (z-1) Dm/dt.
 *
 * mor_shifted_solve eliminates the diagonal A22 (block Schur):
 *
 *   (A11 + z K A22^-1 K^T) x1 = b1 - K A22^-1 b2,   x2 = A22^-1 (b2 + z K^T x1)
 *
 * and solves the Schur system matrix-free (two CSR products per application)
 * with CGS to a normalised residue ||r|| / ||rhs|| <= tol ("CGS ...
 * normalized residue of 1e-4" in 3-D), every right-hand side a column of one
 * batched iteration with its own scalars.  z = 0 is the back-substitution fast
 * path of P:371 (A11, A22 diagonal, no iteration).  Real z runs in real fp64,
 * complex z in complex fp64.
 *
 * mor_krylov_basis runs the multi-point block Arnoldi of P:169 / P:342 on the
 * device: per expansion point z_l (Eq. (19)) the blocks
 * A(z_l)^-1 B, A(z_l)^-1 (R+F) W, ... orthonormalised by classical block
 * Gram-Schmidt applied twice plus modified Gram-Schmidt inside the block with
 * deflation; the realified rows keep_e / keep_h of every accepted block feed the
 * V1 / V2 pools round-robin over the points until both hold q columns
 * (readings R5(iv), (v), (vii)).  All arithmetic is fp64.
 *
 * Arrays passed in are HOST pointers, BORROWED for the call and deep copied;
 * outputs are HOST pointers owned by the caller.  Vectors are stored one per
 * row: X[j][i] = component i of vector j.  Every function returns FDTD_OK (0)
 * or an FDTD_E* code of fdtd.h with the message in fdtd_last_error().  A handle
 * is not thread-safe.
 */
#ifndef FDTD_MOR_H
#define FDTD_MOR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mor_t mor_t;

/* The system to reduce: K is n_e x n_h in CSR (the curl of (3), of
 * the fine region or of the whole hybrid), De / Dm the diagonal masses
 * (eps / mu times the dual-to-primal ratios of the mesh; > 0). */
typedef struct mor_system {
  int64_t n_e, n_h;
  const int64_t* K_rowptr; /* [n_e + 1]                         */
  const int32_t* K_col;    /* [nnz], 0 <= col < n_h             */
  const double* K_val;     /* [nnz]                             */
  const double* De;        /* [n_e]                             */
  const double* Dm;        /* [n_h]                             */
  double dt;               /* > 0                               */
} mor_system;

/* Validate, upload, build K^T on the device side's behalf.  The handle works
 * on an internal stream (the CGS iterations replay a captured CUDA graph) and
 * every mor_* call returns synchronised; stream (a cudaStream_t, may be NULL)
 * is only synchronised here. */
int mor_create(const mor_system* sys, void* stream, mor_t** out);

/* A(z) x = b for nrhs columns.  b_re / b_im / x_re / x_im are
 * [nrhs][n_e + n_h] (E part first); b_im may be NULL (real right-hand side);
 * x_im may be NULL when z_im == 0 and b_im == NULL.  tol, max_iter: CGS
 * stopping rule (ignored for z = 0).  iters[nrhs] (iterations each column took)
 * and resid[nrhs] (final ||r|| / ||rhs|| of the Schur system from the
 * recursion) may be NULL.  Columns that do not reach tol in max_iter
 * iterations are returned as they are (FDTD_OK; check resid); a breakdown
 * (rho = 0 or sigma = 0) freezes the column and sets iters[j] = -iteration.
 * z = 1 is singular for the lossless system: FDTD_EINVAL. */
int mor_shifted_solve(mor_t* h, double z_re, double z_im, int32_t nrhs, const double* b_re, const double* b_im,
                      double tol, int32_t max_iter, double* x_re, double* x_im, int32_t* iters, double* resid);

/* The multi-point block Arnoldi request. */
typedef struct mor_basis_request {
  int32_t n_points;        /* expansion points (>= 1)                                         */
  const double* z_re;      /* [n_points]                                                      */
  const double* z_im;      /* [n_points]                                                      */
  int32_t n_b;             /* columns of the starting block B (1..64)                         */
  const double* B;         /* [n_b][n_e + n_h] real                                           */
  int64_t n_keep_e;        /* rows of the E part that form V1                                 */
  const int64_t* keep_e;   /* [n_keep_e] indices < n_e                                        */
  int64_t n_keep_h;
  const int64_t* keep_h;   /* [n_keep_h] indices < n_h                                        */
  int32_t q;               /* columns wanted in each of V1, V2                                */
  int32_t max_iter;        /* sweeps over the points (0 = 4 q)                                */
  double solve_tol;        /* CGS normalised residue (paper: 1e-4)                            */
  int32_t solve_max_iter;  /* CGS iteration cap                                               */
  double tol_krylov;       /* deflation threshold of the Krylov blocks (host prep: 1e-10)     */
  double tol_pool;         /* deflation threshold of the V1 / V2 pools (host prep: 1e-8)      */
  double window_bytes;     /* device bytes for the Krylov vectors of all points together;
                              beyond it only a sliding window of recent vectors is kept per
                              point for the re-orthogonalisation (0 = 64e9)                   */
} mor_basis_request;

/* V1 [q][n_keep_e], V2 [q][n_keep_h]: Euclidean-orthonormal rows spanning the
 * restricted Krylov blocks.  stats (may be NULL) receives up to n_stats values:
 * [0] sweeps, [1] shifted solves (columns), [2] CGS iterations in total,
 * [3] worst final normalised residue, [4] seconds in solves, [5] seconds in
 * orthogonalisation, [6] Krylov vectors kept, [7] 1 if the window slid.
 * FDTD_ENOTSUP-free: FDTD_EINVAL for bad sizes, FDTD_EDIVERGED if the basis
 * stalls before q columns. */
int mor_krylov_basis(mor_t* h, const mor_basis_request* req, double* V1, double* V2, double* stats,
                     int32_t n_stats);

/* Kernel launches enqueued through this handle so far. */
int64_t mor_launch_count(const mor_t* h);

void mor_destroy(mor_t* h);

#ifdef __cplusplus
}
#endif
#endif /* FDTD_MOR_H */
