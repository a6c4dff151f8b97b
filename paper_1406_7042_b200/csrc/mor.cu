// mor.cu — the offline reduction on the device (fdtd_mor.h; SURVEY §8(f) NEXT-1;
// PAPER.md P:354-393 shifted solves with the 2x2 block Schur elimination
// CGS / z = 0 fast path, P:169 / P:342 multi-point block Arnoldi).
//
// Everything is fp64 (real for real expansion points, complex otherwise).
// Vectors are stored one per row (X[j][i]), so that a set of right-hand sides,
// a Krylov block or the growing orthonormal basis are row ranges of one array:
//
//   spmm_kernel          y = post o (d o x + beta K t) for a block of columns:
//                        one thread per CSR row and column (<= 4 entries per
//                        row of a curl matrix; neighbouring rows read
//                        neighbouring columns, so the gathers coalesce)
//   dot_partial_kernel   per-column inner products, fixed chunks, fixed-order
//                        second stage inside the scalar kernels (deterministic)
//   cgs_*                the batched CGS recursion: every column carries its own
//                        rho / alpha / beta / residue and freezes when converged;
//                        4 iterations (52 launches) replay as one captured graph
//   gram_stream_kernel   G = V^H W of the block Gram-Schmidt (the block staged in
//                        shared memory, every warp streams its basis vectors
//                        through it: the basis read once), gs_update_kernel W -= V G
//
// The Arnoldi driver (host C++) mirrors the host preprocessing
// (prep/reduce.py krylov_basis) step for step; only scalars (norms, residues,
// active counts) cross the bus during the iteration.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/fdtd.h"
#include "../../include/fdtd_mor.h"

namespace fdtd {
int set_error(int code, const char* msg);     // fdtd_api.cu
}

struct mor_t {
  int64_t ne = 0, nh = 0, nnz = 0;
  double dt = 0;
  cudaStream_t st = nullptr;
  int64_t *rp = nullptr, *rpT = nullptr;
  int32_t *ci = nullptr, *ciT = nullptr;
  double *val = nullptr, *valT = nullptr, *De = nullptr, *Dm = nullptr, *invDe = nullptr, *invDm = nullptr;
  int64_t launches = 0;
};

namespace {

#define MCK(call)                                                                                  \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess) {                                                                       \
      char b_[512];                                                                                \
      snprintf(b_, sizeof(b_), "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
      return fdtd::set_error(e_ == cudaErrorMemoryAllocation ? FDTD_ENOMEM : FDTD_ECUDA, b_);      \
    }                                                                                              \
  } while (0)
#define MTRY(expr)                \
  do {                            \
    int rc_ = (expr);             \
    if (rc_ != FDTD_OK) return rc_; \
  } while (0)

int mfail(int code, const std::string& m) { return fdtd::set_error(code, m.c_str()); }

#define HD __host__ __device__ __forceinline__
using cd = double2;

HD double cmul(double a, double b) { return a * b; }
HD cd cmul(cd a, cd b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
HD double rmul(double s, double a) { return s * a; }
HD cd rmul(double s, cd a) { return make_double2(s * a.x, s * a.y); }
HD double cadd(double a, double b) { return a + b; }
HD cd cadd(cd a, cd b) { return make_double2(a.x + b.x, a.y + b.y); }
HD double csub(double a, double b) { return a - b; }
HD cd csub(cd a, cd b) { return make_double2(a.x - b.x, a.y - b.y); }
HD double cconj(double a) { return a; }
HD cd cconj(cd a) { return make_double2(a.x, -a.y); }
HD double cdiv(double a, double b) { return a / b; }
HD cd cdiv(cd a, cd b) {
  double d = b.x * b.x + b.y * b.y;
  return make_double2((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}
HD double creal(double a) { return a; }
HD double creal(cd a) { return a.x; }
HD double cimag(double) { return 0.0; }
HD double cimag(cd a) { return a.y; }
HD bool ciszero(double a) { return a == 0.0; }
HD bool ciszero(cd a) { return a.x == 0.0 && a.y == 0.0; }
HD bool cfinite(double a) { return isfinite(a); }
HD bool cfinite(cd a) { return isfinite(a.x) && isfinite(a.y); }
template <class T> HD T cmake(double re, double im);
template <> HD double cmake<double>(double re, double) { return re; }
template <> HD cd cmake<cd>(double re, double im) { return make_double2(re, im); }
// acc += a * b
HD void cfma(double& acc, double a, double b) { acc = fma(a, b, acc); }
HD void cfma(cd& acc, cd a, cd b) {
  acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
}

constexpr int TPB = 256;
constexpr int MAX_CH = 128;        // chunks of a reduction over the vector length

inline int chunks_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(MAX_CH, (n + 2047) / 2048)); }

// ------------------------------------------------------------------ elementwise / sparse
// y[j][r] = P(r) * ( X(r) + beta * sum_k val[k] t[j][col[k]] )
//   X(r) = dscal * dg[r] * x[j][r]   (x == nullptr: 0; dg == nullptr: dscal * x[j][r])
//   P(r) = pscal * post[r]            (post == nullptr: 1)
template <class T>
__global__ void spmm_kernel(int64_t nrows, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const double* __restrict__ val, const T* __restrict__ t, int64_t ldt, const T* x,
                            int64_t ldx, const double* __restrict__ dg, T dscal, T beta,
                            const double* __restrict__ post, T pscal, T* y, int64_t ldy) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  int j = blockIdx.y;
  const T* tj = t + (int64_t)j * ldt;
  T s = cmake<T>(0, 0);
  for (int64_t k = rp[r]; k < rp[r + 1]; ++k) s = cadd(s, rmul(val[k], tj[ci[k]]));
  T out = cmul(beta, s);
  if (x) {
    T xv = x[(int64_t)j * ldx + r];
    if (dg) xv = rmul(dg[r], xv);
    out = cadd(out, cmul(dscal, xv));
  }
  if (post) out = cmul(pscal, rmul(post[r], out));
  y[(int64_t)j * ldy + r] = out;
}

// y[j][i] = s * d[i] * x[j][i]   (d == nullptr: s * x)
template <class T>
__global__ void diag_mul_kernel(int64_t n, const double* __restrict__ d, T s, const T* x, int64_t ldx, T* y,
                                int64_t ldy) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int j = blockIdx.y;
  T v = x[(int64_t)j * ldx + i];
  if (d) v = rmul(d[i], v);
  y[(int64_t)j * ldy + i] = cmul(s, v);
}

template <class T>
__global__ void zero_kernel(int64_t n, T* y, int64_t ldy) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[(int64_t)blockIdx.y * ldy + i] = cmake<T>(0, 0);
}

template <class T>
__global__ void from_real_kernel(int64_t n, const double* re, const double* im, int64_t ldr, T* y, int64_t ldy) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int j = blockIdx.y;
  y[(int64_t)j * ldy + i] = cmake<T>(re[(int64_t)j * ldr + i], im ? im[(int64_t)j * ldr + i] : 0.0);
}

template <class T>
__global__ void to_real_kernel(int64_t n, const T* x, int64_t ldx, double* re, double* im, int64_t ldr) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int j = blockIdx.y;
  T v = x[(int64_t)j * ldx + i];
  re[(int64_t)j * ldr + i] = creal(v);
  if (im) im[(int64_t)j * ldr + i] = cimag(v);
}

// out[j][r] = Re W[j][off + keep[r]],  out[m + j][r] = Im W[j][off + keep[r]] (complex only)
template <class T>
__global__ void gather_real_kernel(int64_t nk, const int64_t* __restrict__ keep, int64_t off, const T* W, int64_t ldw,
                                   int m, double* out, int64_t ldo) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nk) return;
  int j = blockIdx.y;
  T v = W[(int64_t)j * ldw + off + keep[r]];
  out[(int64_t)j * ldo + r] = creal(v);
  if (sizeof(T) == sizeof(cd)) out[(int64_t)(m + j) * ldo + r] = cimag(v);
}

// ------------------------------------------------------------------ reductions
template <class T>
__device__ __forceinline__ T warp_sum(T v);
template <>
__device__ __forceinline__ double warp_sum<double>(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <>
__device__ __forceinline__ cd warp_sum<cd>(cd v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

// partial[j][c] = sum over chunk c of conj(a[j][i]) b[j][i]
template <class T>
__global__ void dot_partial_kernel(int64_t n, const T* a, int64_t lda, const T* b, int64_t ldb, T* partial, int nch,
                                   const int* active) {
  int j = blockIdx.y, c = blockIdx.x;
  if (active && !active[j]) return;
  int64_t per = (n + nch - 1) / nch, lo = c * per, hi = min(n, lo + per);
  const T* aj = a + (int64_t)j * lda;
  const T* bj = b + (int64_t)j * ldb;
  T s = cmake<T>(0, 0);
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) cfma(s, cconj(aj[i]), bj[i]);
  s = warp_sum(s);
  __shared__ T sm[TPB / 32];
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    T tsum = sm[0];
    for (int w = 1; w < TPB / 32; ++w) tsum = cadd(tsum, sm[w]);
    partial[(int64_t)j * nch + c] = tsum;
  }
}

template <class T>
__global__ void dot_finish_kernel(const T* partial, int nch, int m, T* out) {
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (j >= m) return;
  T s = cmake<T>(0, 0);
  for (int c = lane; c < nch; c += 32) s = cadd(s, partial[(int64_t)j * nch + c]);
  s = warp_sum(s);
  if (lane == 0) out[j] = s;
}

// ------------------------------------------------------------------ batched CGS
template <class T>
struct CgsScal {
  T *rho, *rho_old, *alpha, *beta;
  double *nb, *res;
  int *active, *iters, *n_active;
  int* it;          // the iteration about to run (device side, so that a captured graph replays)
};

template <class T>
__device__ __forceinline__ T sum_partials(const T* partial, int nch, int j) {
  T s = partial[(int64_t)j * nch];
  for (int c = 1; c < nch; ++c) s = cadd(s, partial[(int64_t)j * nch + c]);
  return s;
}

// ||rhs|| -> nb; columns with a zero right-hand side never start
template <class T>
__global__ void cgs_init_kernel(CgsScal<T> S, const T* partial, int nch, int m) {
  int j = threadIdx.x;
  if (j == 0) { *S.n_active = 0; *S.it = 1; }
  __syncthreads();
  if (j >= m) return;
  double nb = sqrt(creal(sum_partials(partial, nch, j)));
  S.nb[j] = nb;
  S.res[j] = nb > 0 ? 1.0 : 0.0;
  S.iters[j] = 0;
  S.rho_old[j] = cmake<T>(1, 0);
  bool act = nb > 0 && isfinite(nb);
  S.active[j] = act;
  if (act) atomicAdd(S.n_active, 1);
}

// rho = <rt, r>, beta = rho / rho_old
template <class T>
__global__ void cgs_s1_kernel(CgsScal<T> S, const T* partial, int nch, int m, int max_iter) {
  int j = threadIdx.x;
  const int it = *S.it;
  if (j >= m || !S.active[j]) return;
  if (it > max_iter) {                      // (a replayed graph past the cap: the column stays as it is)
    S.active[j] = 0;
    return;
  }
  T rho = sum_partials(partial, nch, j);
  if (ciszero(rho) || !cfinite(rho)) {     // breakdown
    S.active[j] = 0;
    S.iters[j] = -it;
    return;
  }
  S.rho[j] = rho;
  S.beta[j] = it > 1 ? cdiv(rho, S.rho_old[j]) : cmake<T>(0, 0);
}

// sigma = <rt, v>, alpha = rho / sigma
template <class T>
__global__ void cgs_s2_kernel(CgsScal<T> S, const T* partial, int nch, int m) {
  int j = threadIdx.x;
  const int it = *S.it;
  if (j >= m || !S.active[j]) return;
  T sigma = sum_partials(partial, nch, j);
  if (ciszero(sigma) || !cfinite(sigma)) {
    S.active[j] = 0;
    S.iters[j] = -it;
    return;
  }
  S.alpha[j] = cdiv(S.rho[j], sigma);
  S.rho_old[j] = S.rho[j];
}

// res = ||r|| / ||rhs||; converged columns freeze
template <class T>
__global__ void cgs_s3_kernel(CgsScal<T> S, const T* partial, int nch, int m, double tol) {
  int j = threadIdx.x;
  const int it = *S.it;
  __syncthreads();
  if (j == 0) { *S.n_active = 0; *S.it = it + 1; }
  __syncthreads();
  if (j >= m || !S.active[j]) return;
  double res = sqrt(creal(sum_partials(partial, nch, j))) / S.nb[j];
  S.res[j] = res;
  S.iters[j] = it;
  if (!(res > tol)) S.active[j] = 0;       // also stops on NaN
  else atomicAdd(S.n_active, 1);
}

// u = r + beta q;  p = u + beta (q + beta p)
template <class T>
__global__ void cgs_v1_kernel(int64_t n, CgsScal<T> S, const T* r, const T* q, T* u, T* p, int64_t ld, int64_t ldx) {
  int j = blockIdx.y;
  if (!S.active[j]) return;
  const int it = *S.it;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t o = (int64_t)j * ld + i;
  if (it == 1) {
    u[o] = r[o];
    p[o] = r[o];
    return;
  }
  T b = S.beta[j];
  T qv = q[o];
  T uv = cadd(r[o], cmul(b, qv));
  u[o] = uv;
  p[o] = cadd(uv, cmul(b, cadd(qv, cmul(b, p[o]))));
}

// q = u - alpha v;  uh = u + q;  x += alpha uh
template <class T>
__global__ void cgs_v2_kernel(int64_t n, CgsScal<T> S, const T* u, const T* v, T* q, T* uh, int64_t ld, T* x,
                              int64_t ldx) {
  int j = blockIdx.y;
  if (!S.active[j]) return;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t o = (int64_t)j * ld + i;
  T a = S.alpha[j];
  T uv = u[o];
  T qv = csub(uv, cmul(a, v[o]));
  q[o] = qv;
  T h = cadd(uv, qv);
  uh[o] = h;
  int64_t ox = (int64_t)j * ldx + i;
  x[ox] = cadd(x[ox], cmul(a, h));
}

// r -= alpha w
template <class T>
__global__ void cgs_v3_kernel(int64_t n, CgsScal<T> S, const T* w, T* r, int64_t ld) {
  int j = blockIdx.y;
  if (!S.active[j]) return;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t o = (int64_t)j * ld + i;
  r[o] = csub(r[o], cmul(S.alpha[j], w[o]));
}

// ------------------------------------------------------------------ block Gram-Schmidt
// partial[c][kk][mm] = sum over chunk c of conj(A[kk][i]) W[mm][i]
// One CTA per chunk of rows and group of MB block columns.  The chunk is walked
// in sub-chunks of GSUB rows: the W tile [MB][GSUB] is staged in shared memory
// once, then every warp streams its basis vectors (kk = warp, warp + 8, ...)
// through it -- GSUB / 32 independent coalesced loads per lane, MB accumulators,
// one warp reduction per vector and sub-chunk -- so the basis is read exactly
// once per Gram product and the block once.  The per-vector sums of a sub-chunk
// are added to partial[] by the same lanes in sub-chunk order (deterministic).
constexpr int GTPB = 384;          // threads of the Gram kernel (one CTA per SM: the W tile fills shared memory)
constexpr int GROWS = 3072;        // rows of the W tile: MB x GROWS words = 192 KB
template <class T, int MB, int KK>
__global__ void __launch_bounds__(GTPB, 1) gram_stream_kernel(int64_t n, const T* __restrict__ A, int64_t lda, int k,
                                                              const T* __restrict__ W, int64_t ldw, int m, T* partial,
                                                              int nch) {
  // KK basis vectors per warp pass share every shared-memory read of the W tile
  // (one vector per pass was bound by shared-memory bandwidth, MB words of W
  // per word of the basis: 2.2 TB/s), and the tile holds the CTA's whole chunk
  // whenever it fits, so a vector is reduced across the warp once per chunk
  extern __shared__ __align__(16) unsigned char gram_smem[];
  T (*Ws)[GROWS] = reinterpret_cast<T (*)[GROWS]>(gram_smem);
  const int c = blockIdx.x, m0 = blockIdx.y * MB;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t per = (n + nch - 1) / nch, lo = c * per, hi = min(n, lo + per);
  bool first = true;
  for (int64_t s0 = lo; s0 < hi || first; s0 += GROWS) {
    const int rows = (int)max((int64_t)0, min((int64_t)GROWS, hi - s0));
    const int rows32 = (rows + 31) & ~31;
    __syncthreads();
    for (int e = threadIdx.x; e < MB * rows32; e += GTPB) {
      const int b = e / rows32, i = e % rows32;
      Ws[b][i] = (m0 + b < m && i < rows) ? W[(int64_t)(m0 + b) * ldw + s0 + i] : cmake<T>(0, 0);
    }
    __syncthreads();
    for (int kk = warp * KK; kk < k; kk += (GTPB / 32) * KK) {
      const T* a[KK];
#pragma unroll
      for (int j = 0; j < KK; ++j) a[j] = A + (int64_t)min(kk + j, k - 1) * lda + s0;
      T acc[KK][MB];
#pragma unroll
      for (int j = 0; j < KK; ++j)
#pragma unroll
        for (int b = 0; b < MB; ++b) acc[j][b] = cmake<T>(0, 0);
#pragma unroll 4
      for (int o = lane; o < rows32; o += 32) {
        const bool in = o < rows;
        T av[KK], wv[MB];
#pragma unroll
        for (int j = 0; j < KK; ++j) av[j] = in ? cconj(a[j][o]) : cmake<T>(0, 0);
#pragma unroll
        for (int b = 0; b < MB; ++b) wv[b] = Ws[b][o];
#pragma unroll
        for (int j = 0; j < KK; ++j)
#pragma unroll
          for (int b = 0; b < MB; ++b) cfma(acc[j][b], av[j], wv[b]);
      }
#pragma unroll
      for (int j = 0; j < KK; ++j) {
        T mine = cmake<T>(0, 0);
#pragma unroll
        for (int b = 0; b < MB; ++b) {
          const T sum = warp_sum(acc[j][b]);
          if (lane == b) mine = sum;
        }
        if (lane < MB && m0 + lane < m && kk + j < k) {
          T* o = partial + ((int64_t)c * k + kk + j) * m + m0 + lane;
          *o = first ? mine : cadd(*o, mine);
        }
      }
    }
    first = false;
  }
}

// G[e] = sum over the chunks of partial[c][e]: one warp per element, lanes over
// the chunks, a fixed shuffle tree (deterministic)
template <class T>
__global__ void gram_finish_kernel(const T* partial, int nch, int64_t km, T* G) {
  const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (e >= km) return;
  T s = cmake<T>(0, 0);
  for (int c = lane; c < nch; c += 32) s = cadd(s, partial[(int64_t)c * km + e]);
  s = warp_sum(s);
  if (lane == 0) G[e] = s;
}

// W[mm][i] -= sum_kk A[kk][i] G[kk][mm]
template <class T, int MB>
__global__ void __launch_bounds__(TPB) gs_update_kernel(int64_t n, const T* __restrict__ A, int64_t lda, int k,
                                                        const T* __restrict__ G, int m, T* W, int64_t ldw) {
  constexpr int KTILE = 128;
  __shared__ T Gs[KTILE][MB];
  int64_t i = (int64_t)blockIdx.x * TPB + threadIdx.x;
  int m0 = blockIdx.y * MB;
  T acc[MB];
#pragma unroll
  for (int b = 0; b < MB; ++b) acc[b] = cmake<T>(0, 0);
  for (int kb = 0; kb < k; kb += KTILE) {
    int kn = min(KTILE, k - kb);
    __syncthreads();
    for (int e = threadIdx.x; e < kn * MB; e += TPB) {
      int a = e / MB, b = e % MB;
      Gs[a][b] = (m0 + b < m) ? G[(int64_t)(kb + a) * m + m0 + b] : cmake<T>(0, 0);
    }
    __syncthreads();
    if (i < n) {
      for (int a = 0; a < kn; ++a) {
        T av = A[(int64_t)(kb + a) * lda + i];
#pragma unroll
        for (int b = 0; b < MB; ++b) cfma(acc[b], av, Gs[a][b]);
      }
    }
  }
  if (i < n) {
#pragma unroll
    for (int b = 0; b < MB; ++b)
      if (m0 + b < m) {
        int64_t o = (int64_t)(m0 + b) * ldw + i;
        W[o] = csub(W[o], acc[b]);
      }
  }
}

// ------------------------------------------------------------------ host helpers
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { if (p) cudaFree(p); }
  cudaError_t alloc(size_t count) {
    if (p) cudaFree(p);
    p = nullptr;
    n = count;
    return cudaMalloc((void**)&p, std::max<size_t>(count, 1) * sizeof(T));
  }
};

inline dim3 grid1(int64_t n, int m) { return dim3((unsigned)((n + TPB - 1) / TPB), (unsigned)std::max(m, 1)); }

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

template <class T> struct GramTile;
template <> struct GramTile<double> { static constexpr int MB = 8, KK = 4; };     // W tile [MB][GROWS]: 192 KB either way
template <> struct GramTile<cd> { static constexpr int MB = 4, KK = 4; };
// chunks of the Gram product: ~3 CTAs per SM on long vectors (each CTA walks all the basis vectors of its rows)
// (one CTA per SM; chunks of at most GROWS rows up to 8 waves of CTAs, longer chunks beyond)
inline int gram_chunks(int64_t n) {
  int64_t c = std::max<int64_t>(1, (n + GROWS - 1) / GROWS);
  if (c > 148) c = (c + 147) / 148 * 148;            // whole waves of one CTA per SM
  return (int)std::min<int64_t>(1184, c);
}

// Growing orthonormal set (mirror of prep/reduce.py _Basis): block classical
// Gram-Schmidt twice against the set, then MGS (twice) inside the block with
// deflation of columns whose norm drops below tol x their original norm.
template <class T>
struct DBasis {
  mor_t* h = nullptr;
  int64_t n = 0;
  int cap = 0, k = 0, mmax = 0;
  double tol = 0;
  DevBuf<T> Vt, W, G, partial, dots;
  int nch = 1;

  int init(mor_t* h_, int64_t n_, int cap_, int mmax_, double tol_) {
    h = h_; n = n_; cap = cap_; mmax = mmax_; tol = tol_; k = 0;
    nch = gram_chunks(n);
    MCK(cudaFuncSetAttribute(gram_stream_kernel<T, GramTile<T>::MB, GramTile<T>::KK>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(GramTile<T>::MB * GROWS * sizeof(T))));
    MCK(Vt.alloc((size_t)cap * n));
    MCK(W.alloc((size_t)mmax * n));
    MCK(G.alloc((size_t)cap * mmax));
    MCK(partial.alloc((size_t)nch * cap * mmax + (size_t)nch * mmax));
    MCK(dots.alloc(mmax));
    return FDTD_OK;
  }

  // W[0:m] -= A^T (conj(A) W) for the k_ rows starting at A
  int project(const T* A, int k_, T* Wp, int m) {
    using GT = GramTile<T>;
    dim3 g1(nch, (m + GT::MB - 1) / GT::MB);
    gram_stream_kernel<T, GT::MB, GT::KK><<<g1, GTPB, GT::MB * GROWS * sizeof(T), h->st>>>(n, A, n, k_, Wp, n, m,
                                                                                          partial.p, nch);
    int64_t km = (int64_t)k_ * m;
    gram_finish_kernel<T><<<(unsigned)((km * 32 + TPB - 1) / TPB), TPB, 0, h->st>>>(partial.p, nch, km, G.p);
    dim3 g2((unsigned)((n + TPB - 1) / TPB), (m + GT::MB - 1) / GT::MB);
    gs_update_kernel<T, GT::MB><<<g2, TPB, 0, h->st>>>(n, A, n, k_, G.p, m, Wp, n);
    h->launches += 3;
    MCK(cudaGetLastError());
    return FDTD_OK;
  }

  int norms(const T* X, int64_t ldx, int m, std::vector<double>& out) {
    dot_partial_kernel<T><<<dim3(nch, m), TPB, 0, h->st>>>(n, X, ldx, X, ldx, partial.p, nch, nullptr);
    dot_finish_kernel<T><<<(m * 32 + 63) / 64, 64, 0, h->st>>>(partial.p, nch, m, dots.p);
    h->launches += 2;
    std::vector<T> tmp(m);
    MCK(cudaMemcpyAsync(tmp.data(), dots.p, m * sizeof(T), cudaMemcpyDeviceToHost, h->st));
    MCK(cudaStreamSynchronize(h->st));
    out.resize(m);
    for (int j = 0; j < m; ++j) out[j] = std::sqrt(std::max(0.0, creal(tmp[j])));
    return FDTD_OK;
  }

  // orthogonalise the m vectors X[j] (row stride ldx) against the set and append
  // the survivors; *first / *count: the accepted rows Vt[first .. first+count)
  int add(const T* X, int64_t ldx, int m, int limit, int* first, int* count) {
    limit = std::min(limit < 0 ? cap : limit, cap);
    *first = k;
    *count = 0;
    if (k >= limit || m == 0) return FDTD_OK;
    if (m > mmax) return mfail(FDTD_EINVAL, "mor: block wider than the basis scratch");
    std::vector<double> nrm0, nrm;
    MTRY(norms(X, ldx, m, nrm0));
    diag_mul_kernel<T><<<grid1(n, m), TPB, 0, h->st>>>(n, nullptr, cmake<T>(1, 0), X, ldx, W.p, n);     // W = X
    h->launches += 1;
    for (int pass = 0; pass < 2; ++pass)
      if (k) MTRY(project(Vt.p, k, W.p, m));
    int start = k;
    for (int j = 0; j < m; ++j) {
      if (k >= limit) break;
      T* w = W.p + (int64_t)j * n;
      for (int pass = 0; pass < 2; ++pass)
        if (k > start) MTRY(project(Vt.p + (int64_t)start * n, k - start, w, 1));
      MTRY(norms(w, n, 1, nrm));
      if (nrm0[j] > 0 && nrm[0] > tol * nrm0[j] && std::isfinite(nrm[0])) {
        diag_mul_kernel<T><<<grid1(n, 1), TPB, 0, h->st>>>(n, nullptr, cmake<T>(1.0 / nrm[0], 0), w, n,
                                                           Vt.p + (int64_t)k * n, n);
        h->launches += 1;
        ++k;
      }
    }
    *count = k - start;
    MCK(cudaGetLastError());
    return FDTD_OK;
  }

  // keep the last `keep` vectors (sliding window of the partial re-orthogonalisation)
  int slide(int keep) {
    if (keep >= k) return FDTD_OK;
    int src = k - keep;
    for (int r = 0; r < keep; ++r)    // ascending order: source rows are always ahead of the destination
      MCK(cudaMemcpyAsync(Vt.p + (int64_t)r * n, Vt.p + (int64_t)(src + r) * n, n * sizeof(T),
                          cudaMemcpyDeviceToDevice, h->st));
    k = keep;
    return FDTD_OK;
  }
};

// The shifted system A(z) of one expansion point with its CGS workspace.
template <class T>
struct Shifted {
  mor_t* h = nullptr;
  T z, a11s, ia22s;       // A11 = a11s De,  A22^-1 = ia22s / Dm
  bool zero = false;
  int mcap = 0, nch = 1;
  DevBuf<T> r, rt, p, q, u, v, uh, tH, partial, sc_T;
  DevBuf<double> sc_d;
  DevBuf<int> sc_i;
  CgsScal<T> S;
  // GIT iterations of the recursion captured once as a CUDA graph and replayed
  // (the iteration number lives on the device); re-captured when the solution
  // pointer, the block width or the stopping rule change
  static constexpr int GIT = 4;
  cudaGraphExec_t gexec = nullptr;
  const T* g_x = nullptr;
  int64_t g_ldx = 0;
  int g_m = 0, g_max = 0;
  double g_tol = 0;
  int* h_active = nullptr;                 // pinned
  int64_t total_iters = 0, total_cols = 0;
  double worst_res = 0;

  Shifted() = default;
  Shifted(const Shifted&) = delete;
  Shifted& operator=(const Shifted&) = delete;
  ~Shifted() {
    if (gexec) cudaGraphExecDestroy(gexec);
    if (h_active) cudaFreeHost(h_active);
  }

  int init(mor_t* h_, T z_, int mcap_) {
    h = h_; z = z_; mcap = mcap_;
    zero = ciszero(z);
    T zm1 = csub(z, cmake<T>(1, 0));
    if (ciszero(zm1)) return mfail(FDTD_EINVAL, "mor: z = 1 is singular for the lossless system (P:349)");
    a11s = rmul(1.0 / h->dt, zm1);
    ia22s = cdiv(cmake<T>(h->dt, 0), zm1);
    nch = chunks_for(h->ne);
    size_t ve = (size_t)mcap * h->ne;
    MCK(tH.alloc((size_t)mcap * h->nh));
    MCK(r.alloc(ve));
    if (!zero) {
      MCK(rt.alloc(ve)); MCK(p.alloc(ve)); MCK(q.alloc(ve)); MCK(u.alloc(ve)); MCK(v.alloc(ve)); MCK(uh.alloc(ve));
    }
    MCK(partial.alloc((size_t)mcap * nch));
    MCK(sc_T.alloc((size_t)4 * mcap));
    MCK(sc_d.alloc((size_t)2 * mcap));
    MCK(sc_i.alloc((size_t)2 * mcap + 2));
    MCK(cudaHostAlloc((void**)&h_active, sizeof(int), cudaHostAllocDefault));
    S.rho = sc_T.p; S.rho_old = sc_T.p + mcap; S.alpha = sc_T.p + 2 * mcap; S.beta = sc_T.p + 3 * mcap;
    S.nb = sc_d.p; S.res = sc_d.p + mcap;
    S.active = sc_i.p; S.iters = sc_i.p + mcap; S.n_active = sc_i.p + 2 * mcap; S.it = sc_i.p + 2 * mcap + 1;
    return FDTD_OK;
  }

  // y = (A11 + z K A22^-1 K^T) x for the active columns (inactive ones are skipped by their consumers)
  void schur_apply(const T* x, int64_t ldx, T* y, int64_t ldy, int m) {
    T one = cmake<T>(1, 0);
    spmm_kernel<T><<<grid1(h->nh, m), TPB, 0, h->st>>>(h->nh, h->rpT, h->ciT, h->valT, x, ldx, nullptr, 0, nullptr, one,
                                                      one, h->invDm, ia22s, tH.p, h->nh);
    spmm_kernel<T><<<grid1(h->ne, m), TPB, 0, h->st>>>(h->ne, h->rp, h->ci, h->val, tH.p, h->nh, x, ldx, h->De, a11s, z,
                                                      nullptr, one, y, ldy);
    h->launches += 2;
  }

  void dot(const T* a, int64_t lda, const T* b, int64_t ldb, int m, bool masked) {
    dot_partial_kernel<T><<<dim3(nch, m), TPB, 0, h->st>>>(h->ne, a, lda, b, ldb, partial.p, nch,
                                                          masked ? S.active : nullptr);
    h->launches += 1;
  }

  // b, x: [m][ne + nh] with row strides ldb, ldx (device).  iters / resid: host, may be null.
  int solve(const T* b, int64_t ldb, T* x, int64_t ldx, int m, double tol, int max_iter, int32_t* iters,
            double* resid) {
    if (m > mcap) return mfail(FDTD_EINVAL, "mor: more right-hand sides than the solver workspace");
    if (m == 0) return FDTD_OK;
    const int64_t ne = h->ne, nh = h->nh;
    T one = cmake<T>(1, 0), mone = cmake<T>(-1, 0);
    // rhs = b1 - K (A22^-1 b2)
    diag_mul_kernel<T><<<grid1(nh, m), TPB, 0, h->st>>>(nh, h->invDm, ia22s, b + ne, ldb, tH.p, nh);
    spmm_kernel<T><<<grid1(ne, m), TPB, 0, h->st>>>(ne, h->rp, h->ci, h->val, tH.p, nh, b, ldb, nullptr, one, mone,
                                                   nullptr, one, r.p, ne);
    h->launches += 2;
    if (zero) {
      // z = 0: A11 = -De/dt is diagonal, no iteration
      diag_mul_kernel<T><<<grid1(ne, m), TPB, 0, h->st>>>(ne, h->invDe, cdiv(one, a11s), r.p, ne, x, ldx);
      h->launches += 1;
      for (int j = 0; j < m; ++j) {
        if (iters) iters[j] = 0;
        if (resid) resid[j] = 0.0;
      }
    } else {
      MCK(cudaMemcpyAsync(rt.p, r.p, (size_t)m * ne * sizeof(T), cudaMemcpyDeviceToDevice, h->st));
      zero_kernel<T><<<grid1(ne, m), TPB, 0, h->st>>>(ne, x, ldx);
      h->launches += 1;
      dot(r.p, ne, r.p, ne, m, false);
      cgs_init_kernel<T><<<1, 64, 0, h->st>>>(S, partial.p, nch, m);
      h->launches += 1;
      // one iteration of the recursion (13 launches)
      auto iteration = [&]() {
        dot(rt.p, ne, r.p, ne, m, true);
        cgs_s1_kernel<T><<<1, 64, 0, h->st>>>(S, partial.p, nch, m, max_iter);
        cgs_v1_kernel<T><<<grid1(ne, m), TPB, 0, h->st>>>(ne, S, r.p, q.p, u.p, p.p, ne, ldx);
        schur_apply(p.p, ne, v.p, ne, m);
        dot(rt.p, ne, v.p, ne, m, true);
        cgs_s2_kernel<T><<<1, 64, 0, h->st>>>(S, partial.p, nch, m);
        cgs_v2_kernel<T><<<grid1(ne, m), TPB, 0, h->st>>>(ne, S, u.p, v.p, q.p, uh.p, ne, x, ldx);
        schur_apply(uh.p, ne, v.p, ne, m);         // w reuses v
        cgs_v3_kernel<T><<<grid1(ne, m), TPB, 0, h->st>>>(ne, S, v.p, r.p, ne);
        dot(r.p, ne, r.p, ne, m, true);
        cgs_s3_kernel<T><<<1, 64, 0, h->st>>>(S, partial.p, nch, m, tol);
        h->launches += 6;
      };
      if (!gexec || g_x != x || g_ldx != ldx || g_m != m || g_max != max_iter || g_tol != tol) {
        if (gexec) { cudaGraphExecDestroy(gexec); gexec = nullptr; }
        const int64_t l0 = h->launches;
        cudaGraph_t gr = nullptr;
        MCK(cudaStreamBeginCapture(h->st, cudaStreamCaptureModeThreadLocal));
        for (int i = 0; i < GIT; ++i) iteration();
        cudaError_t ce = cudaMemcpyAsync(h_active, S.n_active, sizeof(int), cudaMemcpyDeviceToHost, h->st);
        cudaError_t ce2 = cudaStreamEndCapture(h->st, &gr);
        h->launches = l0;                          // (capturing launches nothing)
        MCK(ce);
        MCK(ce2);
        MCK(cudaGraphInstantiate(&gexec, gr, 0));
        MCK(cudaGraphDestroy(gr));
        g_x = x; g_ldx = ldx; g_m = m; g_max = max_iter; g_tol = tol;
      }
      int n_active = m;
      for (int it = 0; it < max_iter && n_active > 0; it += GIT) {
        MCK(cudaGraphLaunch(gexec, h->st));
        h->launches += 13 * GIT;
        MCK(cudaStreamSynchronize(h->st));
        n_active = *h_active;
      }
      std::vector<int> hi(m);
      std::vector<double> hr(m);
      MCK(cudaMemcpyAsync(hi.data(), S.iters, m * sizeof(int), cudaMemcpyDeviceToHost, h->st));
      MCK(cudaMemcpyAsync(hr.data(), S.res, m * sizeof(double), cudaMemcpyDeviceToHost, h->st));
      MCK(cudaStreamSynchronize(h->st));
      for (int j = 0; j < m; ++j) {
        if (iters) iters[j] = hi[j];
        if (resid) resid[j] = hr[j];
        total_iters += std::abs(hi[j]);
        if (std::isfinite(hr[j])) worst_res = std::max(worst_res, hr[j]);
        else worst_res = INFINITY;
      }
    }
    total_cols += m;
    // x2 = A22^-1 (b2 + z K^T x1)
    spmm_kernel<T><<<grid1(nh, m), TPB, 0, h->st>>>(nh, h->rpT, h->ciT, h->valT, x, ldx, b + ne, ldb, nullptr, one, z,
                                                   h->invDm, ia22s, x + ne, ldx);
    h->launches += 1;
    MCK(cudaGetLastError());
    return FDTD_OK;
  }

  // b = (R + F) w:  b1 = (De/dt) wE,  b2 = (Dm/dt) wH - K^T wE
  int rf_apply(const T* w, int64_t ldw, T* b, int64_t ldb, int m) {
    const int64_t ne = h->ne, nh = h->nh;
    T idt = cmake<T>(1.0 / h->dt, 0);
    diag_mul_kernel<T><<<grid1(ne, m), TPB, 0, h->st>>>(ne, h->De, idt, w, ldw, b, ldb);
    spmm_kernel<T><<<grid1(nh, m), TPB, 0, h->st>>>(nh, h->rpT, h->ciT, h->valT, w, ldw, w + ne, ldw, h->Dm, idt,
                                                   cmake<T>(-1, 0), nullptr, cmake<T>(1, 0), b + ne, ldb);
    h->launches += 2;
    MCK(cudaGetLastError());
    return FDTD_OK;
  }
};

struct Pools {
  DBasis<double> P1, P2;
  DevBuf<int64_t> keep_e, keep_h;
  DevBuf<double> scratch;      // [2 n_b][max(n_keep_e, n_keep_h)]
  int64_t nke = 0, nkh = 0;
  int q = 0;
  bool full() const { return P1.k >= q && P2.k >= q; }
};

// One expansion point of the Arnoldi sweep.
struct PointBase {
  virtual ~PointBase() = default;
  virtual int start(const double* dB, int n_b, double tol, int maxit) = 0;
  virtual int sweep(Pools& P, double tol, int maxit, bool windowed, bool* progressed, bool* slid) = 0;
  virtual void stats(int64_t* cols, int64_t* iters, double* worst, int* kept) const = 0;
  double t_solve = 0, t_orth = 0;
};

template <class T>
struct Point : PointBase {
  mor_t* h;
  Shifted<T> A;
  DBasis<T> Q;
  DevBuf<T> nxt, rhs;       // [n_b][N]
  int n_nxt = 0;
  int64_t N;

  int init(mor_t* h_, T z, int n_b, int cap, double tol_krylov) {
    h = h_;
    N = h->ne + h->nh;
    MTRY(A.init(h, z, n_b));
    MTRY(Q.init(h, N, cap, n_b, tol_krylov));
    MCK(nxt.alloc((size_t)n_b * N));
    MCK(rhs.alloc((size_t)n_b * N));
    return FDTD_OK;
  }

  int start(const double* dB, int n_b, double tol, int maxit) override {
    double t0 = now_s();
    from_real_kernel<T><<<grid1(N, n_b), TPB, 0, h->st>>>(N, dB, nullptr, N, rhs.p, N);
    h->launches += 1;
    MTRY(A.solve(rhs.p, N, nxt.p, N, n_b, tol, maxit, nullptr, nullptr));
    n_nxt = n_b;
    MCK(cudaStreamSynchronize(h->st));
    t_solve += now_s() - t0;
    return FDTD_OK;
  }

  int sweep(Pools& P, double tol, int maxit, bool windowed, bool* progressed, bool* slid) override {
    if (windowed && Q.k + n_nxt > Q.cap) {
      MTRY(Q.slide(Q.cap / 2));
      *slid = true;
    }
    if (n_nxt == 0 || Q.k >= Q.cap) return FDTD_OK;
    double t0 = now_s();
    int first = 0, cnt = 0;
    MTRY(Q.add(nxt.p, N, n_nxt, -1, &first, &cnt));
    if (cnt == 0) {
      n_nxt = 0;
      MCK(cudaStreamSynchronize(h->st));
      t_orth += now_s() - t0;
      return FDTD_OK;
    }
    *progressed = true;
    const T* Wb = Q.Vt.p + (int64_t)first * N;
    const int mr = sizeof(T) == sizeof(cd) ? 2 * cnt : cnt;
    int f2, c2;
    gather_real_kernel<T><<<grid1(P.nke, cnt), TPB, 0, h->st>>>(P.nke, P.keep_e.p, 0, Wb, N, cnt, P.scratch.p, P.nke);
    h->launches += 1;
    MTRY(P.P1.add(P.scratch.p, P.nke, mr, P.q, &f2, &c2));
    gather_real_kernel<T><<<grid1(P.nkh, cnt), TPB, 0, h->st>>>(P.nkh, P.keep_h.p, h->ne, Wb, N, cnt, P.scratch.p,
                                                               P.nkh);
    h->launches += 1;
    MTRY(P.P2.add(P.scratch.p, P.nkh, mr, P.q, &f2, &c2));
    MCK(cudaStreamSynchronize(h->st));
    double t1 = now_s();
    t_orth += t1 - t0;
    if (P.full()) return FDTD_OK;
    // next block: A^-1 (R + F) W
    MTRY(A.rf_apply(Wb, N, rhs.p, N, cnt));
    MTRY(A.solve(rhs.p, N, nxt.p, N, cnt, tol, maxit, nullptr, nullptr));
    n_nxt = cnt;
    MCK(cudaStreamSynchronize(h->st));
    t_solve += now_s() - t1;
    return FDTD_OK;
  }

  void stats(int64_t* cols, int64_t* iters, double* worst, int* kept) const override {
    *cols = A.total_cols; *iters = A.total_iters; *worst = A.worst_res; *kept = Q.k;
  }
};

template <class T>
int upload(DevBuf<T>& d, const T* src, size_t n, cudaStream_t st) {
  MCK(d.alloc(n));
  if (n) MCK(cudaMemcpyAsync(d.p, src, n * sizeof(T), cudaMemcpyHostToDevice, st));
  return FDTD_OK;
}

template <class T>
int solve_host(mor_t* h, T z, int32_t nrhs, const double* b_re, const double* b_im, double tol, int32_t max_iter,
               double* x_re, double* x_im, int32_t* iters, double* resid) {
  const int64_t N = h->ne + h->nh;
  Shifted<T> A;
  MTRY(A.init(h, z, nrhs));
  DevBuf<double> dre, dim_, ore, oim;
  DevBuf<T> b, x;
  MTRY(upload(dre, b_re, (size_t)nrhs * N, h->st));
  if (b_im) MTRY(upload(dim_, b_im, (size_t)nrhs * N, h->st));
  MCK(b.alloc((size_t)nrhs * N));
  MCK(x.alloc((size_t)nrhs * N));
  from_real_kernel<T><<<grid1(N, nrhs), TPB, 0, h->st>>>(N, dre.p, b_im ? dim_.p : nullptr, N, b.p, N);
  h->launches += 1;
  MTRY(A.solve(b.p, N, x.p, N, nrhs, tol, max_iter, iters, resid));
  MCK(ore.alloc((size_t)nrhs * N));
  if (x_im) MCK(oim.alloc((size_t)nrhs * N));
  to_real_kernel<T><<<grid1(N, nrhs), TPB, 0, h->st>>>(N, x.p, N, ore.p, x_im ? oim.p : nullptr, N);
  h->launches += 1;
  MCK(cudaMemcpyAsync(x_re, ore.p, (size_t)nrhs * N * sizeof(double), cudaMemcpyDeviceToHost, h->st));
  if (x_im) MCK(cudaMemcpyAsync(x_im, oim.p, (size_t)nrhs * N * sizeof(double), cudaMemcpyDeviceToHost, h->st));
  MCK(cudaStreamSynchronize(h->st));
  return FDTD_OK;
}

}  // namespace

extern "C" {

int mor_create(const mor_system* sys, void* stream, mor_t** out) {
  if (!sys || !out) return mfail(FDTD_EINVAL, "mor_create: null argument");
  *out = nullptr;
  if (sys->n_e < 1 || sys->n_h < 1 || !(sys->dt > 0) || !sys->K_rowptr || !sys->De || !sys->Dm)
    return mfail(FDTD_EINVAL, "mor_create: bad sizes or null arrays");
  if (sys->n_e > INT32_MAX || sys->n_h > INT32_MAX) return mfail(FDTD_EINVAL, "mor_create: more than 2^31 unknowns");
  const int64_t ne = sys->n_e, nh = sys->n_h;
  const int64_t nnz = sys->K_rowptr[ne];
  if (sys->K_rowptr[0] != 0 || nnz < 0 || (nnz > 0 && (!sys->K_col || !sys->K_val)))
    return mfail(FDTD_EINVAL, "mor_create: bad CSR arrays");
  for (int64_t r = 0; r < ne; ++r)
    if (sys->K_rowptr[r + 1] < sys->K_rowptr[r]) return mfail(FDTD_EINVAL, "mor_create: row pointers decrease");
  for (int64_t k = 0; k < nnz; ++k)
    if (sys->K_col[k] < 0 || sys->K_col[k] >= nh) return mfail(FDTD_ESTAMP, "mor_create: column index outside K");
  for (int64_t i = 0; i < ne; ++i)
    if (!(sys->De[i] > 0) || !std::isfinite(sys->De[i])) return mfail(FDTD_EINVAL, "mor_create: De must be > 0");
  for (int64_t i = 0; i < nh; ++i)
    if (!(sys->Dm[i] > 0) || !std::isfinite(sys->Dm[i])) return mfail(FDTD_EINVAL, "mor_create: Dm must be > 0");
  int dev = 0;
  cudaDeviceProp prop;
  MCK(cudaGetDevice(&dev));
  MCK(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10) return mfail(FDTD_ENOTSUP, "mor_create: needs an sm_100 GPU");
  // K^T in CSR (counting sort; columns of each row of K^T ascend)
  std::vector<int64_t> rpT(nh + 1, 0);
  for (int64_t k = 0; k < nnz; ++k) rpT[sys->K_col[k] + 1]++;
  for (int64_t c = 0; c < nh; ++c) rpT[c + 1] += rpT[c];
  std::vector<int32_t> ciT(nnz);
  std::vector<double> valT(nnz);
  {
    std::vector<int64_t> pos(rpT.begin(), rpT.end() - 1);
    for (int64_t r = 0; r < ne; ++r)
      for (int64_t k = sys->K_rowptr[r]; k < sys->K_rowptr[r + 1]; ++k) {
        int64_t o = pos[sys->K_col[k]]++;
        ciT[o] = (int32_t)r;
        valT[o] = sys->K_val[k];
      }
  }
  std::vector<double> iDe(ne), iDm(nh);
  for (int64_t i = 0; i < ne; ++i) iDe[i] = 1.0 / sys->De[i];
  for (int64_t i = 0; i < nh; ++i) iDm[i] = 1.0 / sys->Dm[i];
  std::unique_ptr<mor_t, void (*)(mor_t*)> h(new mor_t, mor_destroy);
  h->ne = ne; h->nh = nh; h->nnz = nnz; h->dt = sys->dt;
  // an internal stream: the CGS iterations are captured into a CUDA graph, which
  // the legacy default stream cannot do.  Every mor_* call takes host buffers
  // and returns synchronised, so nothing is ordered against the caller's stream
  // beyond a synchronise of it here.
  if (stream) MCK(cudaStreamSynchronize((cudaStream_t)stream));
  MCK(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking));
  auto up = [&](auto** dst, const auto* src, size_t n) -> cudaError_t {
    cudaError_t e = cudaMalloc((void**)dst, std::max<size_t>(n, 1) * sizeof(**dst));
    if (e != cudaSuccess) return e;
    return n ? cudaMemcpyAsync(*dst, src, n * sizeof(**dst), cudaMemcpyHostToDevice, h->st) : cudaSuccess;
  };
  MCK(up(&h->rp, sys->K_rowptr, ne + 1));
  MCK(up(&h->ci, sys->K_col, nnz));
  MCK(up(&h->val, sys->K_val, nnz));
  MCK(up(&h->rpT, rpT.data(), nh + 1));
  MCK(up(&h->ciT, ciT.data(), nnz));
  MCK(up(&h->valT, valT.data(), nnz));
  MCK(up(&h->De, sys->De, ne));
  MCK(up(&h->Dm, sys->Dm, nh));
  MCK(up(&h->invDe, iDe.data(), ne));
  MCK(up(&h->invDm, iDm.data(), nh));
  MCK(cudaStreamSynchronize(h->st));
  *out = h.release();
  return FDTD_OK;
}

int mor_shifted_solve(mor_t* h, double z_re, double z_im, int32_t nrhs, const double* b_re, const double* b_im,
                      double tol, int32_t max_iter, double* x_re, double* x_im, int32_t* iters, double* resid) {
  if (!h || !b_re || !x_re) return mfail(FDTD_EINVAL, "mor_shifted_solve: null argument");
  if (nrhs < 1 || nrhs > 64) return mfail(FDTD_EINVAL, "mor_shifted_solve: nrhs must be 1..64");
  const bool cplx = z_im != 0.0 || b_im != nullptr;
  if (cplx && !x_im) return mfail(FDTD_EINVAL, "mor_shifted_solve: complex solve needs x_im");
  const bool zero = z_re == 0.0 && z_im == 0.0;
  if (!zero && (!(tol > 0) || max_iter < 1))
    return mfail(FDTD_EINVAL, "mor_shifted_solve: tol must be > 0 and max_iter >= 1");
  if (cplx) return solve_host<cd>(h, make_double2(z_re, z_im), nrhs, b_re, b_im, tol, max_iter, x_re, x_im, iters, resid);
  int rc = solve_host<double>(h, z_re, nrhs, b_re, nullptr, tol, max_iter, x_re, nullptr, iters, resid);
  if (rc == FDTD_OK && x_im) std::memset(x_im, 0, (size_t)nrhs * (h->ne + h->nh) * sizeof(double));
  return rc;
}

int mor_krylov_basis(mor_t* h, const mor_basis_request* req, double* V1, double* V2, double* stats, int32_t n_stats) {
  if (!h || !req || !V1 || !V2) return mfail(FDTD_EINVAL, "mor_krylov_basis: null argument");
  const int64_t ne = h->ne, nh = h->nh, N = ne + nh;
  if (req->n_points < 1 || !req->z_re || !req->z_im || req->n_b < 1 || req->n_b > 64 || !req->B || req->q < 1 ||
      req->n_keep_e < 1 || req->n_keep_h < 1 || !req->keep_e || !req->keep_h)
    return mfail(FDTD_EINVAL, "mor_krylov_basis: bad sizes or null arrays");
  if (req->q > req->n_keep_e || req->q > req->n_keep_h)
    return mfail(FDTD_EINVAL, "mor_krylov_basis: q exceeds the number of kept rows");
  for (int64_t i = 0; i < req->n_keep_e; ++i)
    if (req->keep_e[i] < 0 || req->keep_e[i] >= ne) return mfail(FDTD_ESTAMP, "mor_krylov_basis: keep_e outside the E part");
  for (int64_t i = 0; i < req->n_keep_h; ++i)
    if (req->keep_h[i] < 0 || req->keep_h[i] >= nh) return mfail(FDTD_ESTAMP, "mor_krylov_basis: keep_h outside the H part");
  bool any_iter = false;
  for (int p = 0; p < req->n_points; ++p) {
    if (req->z_re[p] == 1.0 && req->z_im[p] == 0.0) return mfail(FDTD_EINVAL, "mor_krylov_basis: z = 1 is singular (P:349)");
    any_iter |= (req->z_re[p] != 0.0 || req->z_im[p] != 0.0);
  }
  if (any_iter && (!(req->solve_tol > 0) || req->solve_max_iter < 1))
    return mfail(FDTD_EINVAL, "mor_krylov_basis: solve_tol must be > 0 and solve_max_iter >= 1");
  const int q = req->q, nb = req->n_b, npts = req->n_points;
  const int max_iter = req->max_iter > 0 ? req->max_iter : 4 * q;
  const double tol_k = req->tol_krylov > 0 ? req->tol_krylov : 1e-10;
  const double tol_p = req->tol_pool > 0 ? req->tol_pool : 1e-8;
  const double window = req->window_bytes > 0 ? req->window_bytes : 64e9;
  // capacity of each point's Krylov set, as in the host preprocessing
  int64_t cap = 2ll * max_iter * nb / npts + 4ll * nb;
  cap = std::min<int64_t>(cap, 4ll * q + 4ll * nb);
  bool windowed = false;
  double bytes = 0;
  for (int p = 0; p < npts; ++p) bytes += (double)N * cap * (req->z_im[p] != 0.0 ? 16 : 8);
  if (bytes > window) {
    double per_vec = 0;
    for (int p = 0; p < npts; ++p) per_vec += (double)N * (req->z_im[p] != 0.0 ? 16 : 8);
    cap = std::max<int64_t>(4ll * nb, (int64_t)(window / per_vec) / nb * nb);
    windowed = true;
  }
  Pools P;
  P.q = q; P.nke = req->n_keep_e; P.nkh = req->n_keep_h;
  MTRY(P.P1.init(h, P.nke, q, 2 * nb, tol_p));
  MTRY(P.P2.init(h, P.nkh, q, 2 * nb, tol_p));
  MTRY(upload(P.keep_e, req->keep_e, (size_t)P.nke, h->st));
  MTRY(upload(P.keep_h, req->keep_h, (size_t)P.nkh, h->st));
  MCK(P.scratch.alloc((size_t)2 * nb * std::max(P.nke, P.nkh)));
  DevBuf<double> dB;
  MTRY(upload(dB, req->B, (size_t)nb * N, h->st));
  std::vector<std::unique_ptr<PointBase>> pts;
  for (int p = 0; p < npts; ++p) {
    if (req->z_im[p] != 0.0) {
      auto pt = std::make_unique<Point<cd>>();
      MTRY(pt->init(h, make_double2(req->z_re[p], req->z_im[p]), nb, (int)cap, tol_k));
      pts.push_back(std::move(pt));
    } else {
      auto pt = std::make_unique<Point<double>>();
      MTRY(pt->init(h, req->z_re[p], nb, (int)cap, tol_k));
      pts.push_back(std::move(pt));
    }
    MTRY(pts.back()->start(dB.p, nb, req->solve_tol, req->solve_max_iter));
  }
  int it = 0;
  bool slid = false;
  while (!P.full() && it < max_iter) {
    bool progressed = false;
    for (auto& pt : pts) {
      MTRY(pt->sweep(P, req->solve_tol, req->solve_max_iter, windowed, &progressed, &slid));
      if (P.full()) break;
    }
    if (!progressed) break;
    ++it;
  }
  if (!P.full()) {
    char b[160];
    snprintf(b, sizeof(b), "mor_krylov_basis: basis stalled at %d / %d of %d columns", P.P1.k, P.P2.k, q);
    return mfail(FDTD_EDIVERGED, b);
  }
  MCK(cudaMemcpyAsync(V1, P.P1.Vt.p, (size_t)q * P.nke * sizeof(double), cudaMemcpyDeviceToHost, h->st));
  MCK(cudaMemcpyAsync(V2, P.P2.Vt.p, (size_t)q * P.nkh * sizeof(double), cudaMemcpyDeviceToHost, h->st));
  MCK(cudaStreamSynchronize(h->st));
  if (stats) {
    double s[8] = {(double)it, 0, 0, 0, 0, 0, 0, slid ? 1.0 : 0.0};
    for (auto& pt : pts) {
      int64_t c, i;
      double w;
      int kept;
      pt->stats(&c, &i, &w, &kept);
      s[1] += c; s[2] += i; s[3] = std::max(s[3], w); s[4] += pt->t_solve; s[5] += pt->t_orth; s[6] += kept;
    }
    for (int i = 0; i < n_stats && i < 8; ++i) stats[i] = s[i];
  }
  return FDTD_OK;
}

int64_t mor_launch_count(const mor_t* h) { return h ? h->launches : 0; }

void mor_destroy(mor_t* h) {
  if (!h) return;
  cudaFree(h->rp); cudaFree(h->rpT); cudaFree(h->ci); cudaFree(h->ciT); cudaFree(h->val); cudaFree(h->valT);
  cudaFree(h->De); cudaFree(h->Dm); cudaFree(h->invDe); cudaFree(h->invDm);
  if (h->st) cudaStreamDestroy(h->st);
  delete h;
}

}  // extern "C"
