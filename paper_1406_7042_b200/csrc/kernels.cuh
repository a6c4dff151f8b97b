// kernels.cuh — device kernels of the reduced-hybrid FDTD step (sm_100a).
//
// One time step n -> n+1 (DESIGN.md §1 rows a1-a7) is two launches:
//   stencil   fused coarse E->H pass over the grid (ping-pong buffers); the
//             explicit E rows (interface rows a3, source rows a1) are
//             evaluated in place by the thread that owns them           a1-a3, a5
//   reduced   the reduced chain of every small block as ONE GEMV with a
//             precomposed update matrix (a4, a6: e~, G gather, h~, y),
//             + probes, divergence check, device step counter            a7
// Large reduced blocks (S_E of hundreds of MB) run the leap-frog as
// grid-wide GEMV launches between the two (see fdtd_api.cu).
//
// Coarse fields live in "device storage": component arrays indexed
// ((k*(ny+1) + j)*px + i)*B + b with the batch b innermost and px >= nx+1.
// E^{n+1} = E^n + cb * curl(H)  ==  E^n - cb * (K_inc H)   (K_inc = -curl)
// H^{n+1} = H^n - ch * curl(E)  ==  H^n + ch * (K_inc^T E)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fdtd {


template <typename T> struct Coef;       // per-material coefficient, hi/lo for fp32 (R11)
template <> struct Coef<float> {
  float hi, lo;
  __device__ __forceinline__ float apply(float d) const { return fmaf(hi, d, lo * d); }
};
template <> struct Coef<double> {
  double hi, lo;
  __device__ __forceinline__ double apply(double d) const { return hi * d; }
};

constexpr int MAX_MAT = 256;

template <typename T>
struct MatTable {                 // lives in shared memory inside the stencil kernels
  Coef<T> c[MAX_MAT][6];
  uint8_t ifm[MAX_MAT];
};

struct Dims {
  int nx, ny, nz;                 // coarse cells
  int px;                         // x pitch (>= nx+1)
  int B;                          // batch
  int64_t plane;                  // (ny+1)*px  (storage indices per k-plane)
};

template <typename T>
struct Fields {                   // one parity of the coarse state, by component
  T* f[6];
};

__device__ __forceinline__ bool finite_small(double v) {
  return isfinite(v) && fabs(v) <= 1e100;
}

// ---------------------------------------------------------------------------
// explicit E rows (interface rows of reading R4 and source rows):
//   E1 = E0 - c (sum_k W_k H0[col_k] + y_r) - cs J[step]
// row_of[comp][storage offset] gives the row (dense int32 map, -1 elsewhere).
// ---------------------------------------------------------------------------
template <typename T>
struct RowsE {
  int64_t n_rows;
  const int32_t* row_of[3];    // per E component, [plane*nplanes] or null
  const Coef<T>* c;            // [n_rows]
  const int64_t* rowptr;       // [n_rows+1]
  const int32_t* h_comp;       // [nnz]
  const int64_t* h_off;        // [nnz]
  const T* w;                  // [nnz]
  const int64_t* y_off;        // [n_rows] offset into y (block base + local*N + inst*B), -1 none
  const int32_t* src;          // [n_rows] source index or -1
  const T* cs;                 // [n_rows] source coefficient
  const T* wave;               // [n_wave][n_src][B]
  int64_t n_wave, n_src;
  T* g_out;                    // interface rows publish E^{n+1} at G[y_off] (reduced-chain input)
  // list form (for the standalone rows kernel)
  const int32_t* e_comp;       // [n_rows]
  const int64_t* e_off;        // [n_rows]
};

template <typename T>
__device__ __forceinline__ T eval_row(const RowsE<T>& R, int r, int b, int B, T e0, const Fields<T>& H0,
                                      const T* __restrict__ y, int64_t step) {
  T acc = 0;
  for (int64_t k = R.rowptr[r]; k < R.rowptr[r + 1]; ++k)
    acc += R.w[k] * H0.f[R.h_comp[k]][R.h_off[k] * B + b];
  const int64_t yo = R.y_off[r];
  if (yo >= 0) acc += y[yo + b];
  T e = e0 - R.c[r].apply(acc);
  const int s = R.src[r];
  if (s >= 0 && step < R.n_wave) e -= R.cs[r] * R.wave[(step * R.n_src + s) * B + b];
  if (yo >= 0) R.g_out[yo + b] = e;        // identical value from every thread computing it
  return e;
}

// ---------------------------------------------------------------------------
// 2-D (Ez, Hx, Hy) fused E->H stencil.  Block (BX, BY) threads; each thread owns
// CY consecutive rows of one column (all its loads are issued before any
// compute: CY x 5 independent loads in flight per thread).  The block computes
// Ez^{n+1} on its BX/B x BY*CY footprint and updates Hx, Hy on the footprint
// minus its last column and row (overlapped tiling: the halo Ez is recomputed
// by the neighbouring block; the old buffers are read-only, race free).
// Ez += cb ((Hy(i) - Hy(i-1)) - (Hx(j) - Hx(j-1)))
// Hx -= ch (Ez(j+1) - Ez(j))        Hy += ch (Ez(i+1) - Ez(i))
// ---------------------------------------------------------------------------
template <typename T, bool UNIFORM, int CY>
__global__ void __launch_bounds__(256, 4)
stencil2d_rows_kernel(Dims d, Fields<T> F0, Fields<T> F1, const uint8_t* __restrict__ mat_id,
                      const Coef<T>* __restrict__ gtab, const uint8_t* __restrict__ gifm, int n_mat,
                      Coef<T> u0, Coef<T> u1, RowsE<T> R, const T* __restrict__ y,
                      const int64_t* __restrict__ d_step, int check_every,
                      unsigned long long* __restrict__ bad_step) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int BX = blockDim.x, BY = blockDim.y, B = d.B;
  const int tx = threadIdx.x, ty = threadIdx.y;
  T* sE = reinterpret_cast<T*>(smem_raw);                    // [BY*CY][BX]
  MatTable<T>* tab = reinterpret_cast<MatTable<T>*>(sE + BX * BY * CY);
  const T* __restrict__ Ez0 = F0.f[2];
  const T* __restrict__ Hx0 = F0.f[3];
  const T* __restrict__ Hy0 = F0.f[4];
  const int nx = d.nx, ny = d.ny;
  const int outx = BX / B - 1, outy = BY * CY - 1;
  const int i = blockIdx.x * outx + tx / B;
  const int b = tx % B;
  const int jb = blockIdx.y * outy + ty * CY;
  const int ii = min(i, nx);
  const int64_t sx = (i > 0) ? B : 0;
  const int64_t rs = (int64_t)d.px * B;
  const int64_t step = *d_step;
  // issue every load first
  T hx[CY], hy[CY], hyim[CY], ez0[CY];
  int m[CY];
  int64_t o[CY];
#pragma unroll
  for (int r = 0; r < CY; ++r) {
    const int jj = min(jb + r, ny);
    o[r] = ((int64_t)jj * d.px + ii) * B + b;
    hx[r] = Hx0[o[r]]; hy[r] = Hy0[o[r]]; hyim[r] = Hy0[o[r] - sx]; ez0[r] = Ez0[o[r]];
    m[r] = UNIFORM ? 0 : (int)mat_id[(int64_t)jj * d.px + ii];
  }
  const T hx_jm = (jb > 0) ? Hx0[o[0] - rs] : (T)0;
  if (!UNIFORM) {
    for (int q = ty * BX + tx; q < n_mat; q += BX * BY) {
      tab->c[q][2] = gtab[q * 6 + 2];
      tab->c[q][3] = gtab[q * 6 + 3];
      tab->c[q][4] = gtab[q * 6 + 4];
      tab->ifm[q] = gifm[q];
    }
  }
  __syncthreads();
  T ez[CY];
  const bool ci = (i > 0) && (i < nx);
#pragma unroll
  for (int r = 0; r < CY; ++r) {
    const int j = jb + r;
    const T hxm = (r == 0) ? hx_jm : hx[r - 1];
    const Coef<T> c = UNIFORM ? u0 : tab->c[m[r]][2];
    const T dd = (hy[r] - hyim[r]) - (hx[r] - hxm);
    ez[r] = (ci && j > 0 && j < ny) ? ez0[r] + c.apply(dd) : (T)0;
    if (!UNIFORM && (tab->ifm[m[r]] & 4) && i <= nx && j <= ny) {
      const int64_t so = (int64_t)min(j, ny) * d.px + ii;
      ez[r] = eval_row(R, R.row_of[2][so], b, B, ez0[r], F0, y, step);
    }
    sE[(ty * CY + r) * BX + tx] = ez[r];
  }
  __syncthreads();
  const bool colown = (i <= nx) && (tx / B < outx);
  const bool do_check = check_every > 0 && (step % check_every) == 0;
  bool bad = false;
#pragma unroll
  for (int r = 0; r < CY; ++r) {
    const int j = jb + r;
    if (!colown || j > ny || ty * CY + r >= outy) continue;
    const T ez_jp = (r + 1 < CY) ? ez[r + 1] : sE[((ty + 1) * CY) * BX + tx];
    const T ez_ip = sE[(ty * CY + r) * BX + tx + B];
    Coef<T> cx, cy;
    if (UNIFORM) { cx = u1; cy = u1; }
    else { cx = tab->c[m[r]][3]; cy = tab->c[m[r]][4]; }
    const T hx1 = (ci && j < ny) ? hx[r] - cx.apply(ez_jp - ez[r]) : hx[r];
    const T hy1 = (i < nx && j > 0 && j < ny) ? hy[r] + cy.apply(ez_ip - ez[r]) : hy[r];
    F1.f[2][o[r]] = ez[r]; F1.f[3][o[r]] = hx1; F1.f[4][o[r]] = hy1;
    if (do_check) bad |= !(finite_small(ez[r]) && finite_small(hx1) && finite_small(hy1));
  }
  if (bad) atomicMin(bad_step, (unsigned long long)step);
}

// ---------------------------------------------------------------------------
// 3-D fused E->H stencil.  Block (BX, BY) threads covers BX/B cells in x and
// BY cells in y; it computes E^{n+1} on the whole footprint and H^{n+3/2} on
// the footprint minus its last x cell and last y row (overlapped tiling), and
// marches z over [k0, k1).
// ---------------------------------------------------------------------------
template <typename T, bool UNIFORM>
__global__ void __launch_bounds__(1024)
stencil3d_kernel(Dims d, Fields<T> F0, Fields<T> F1, const uint8_t* __restrict__ mat_id,
                 const Coef<T>* __restrict__ gtab, const uint8_t* __restrict__ gifm, int n_mat,
                 Coef<T> u0, Coef<T> u1, RowsE<T> R, const T* __restrict__ y, int kchunk,
                 const int64_t* __restrict__ d_step, int check_every,
                 unsigned long long* __restrict__ bad_step) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int BX = blockDim.x, BY = blockDim.y, B = d.B;
  const int tx = threadIdx.x, ty = threadIdx.y;
  T* sE = reinterpret_cast<T*>(smem_raw);                       // [2][3][BY][BX]
  MatTable<T>* tab = reinterpret_cast<MatTable<T>*>(sE + 2 * 3 * BX * BY);
  if (!UNIFORM) {
    for (int m = ty * BX + tx; m < n_mat; m += BX * BY) {
      for (int c = 0; c < 6; ++c) tab->c[m][c] = gtab[m * 6 + c];
      tab->ifm[m] = gifm[m];
    }
  }
  const T* __restrict__ Ex0 = F0.f[0];
  const T* __restrict__ Ey0 = F0.f[1];
  const T* __restrict__ Ez0 = F0.f[2];
  const T* __restrict__ Hx0 = F0.f[3];
  const T* __restrict__ Hy0 = F0.f[4];
  const T* __restrict__ Hz0 = F0.f[5];
  const int cells_x = BX / B;
  const int outx = cells_x - 1, outy = BY - 1;
  const int i = blockIdx.x * outx + tx / B;
  const int b = tx % B;
  const int j = blockIdx.y * outy + ty;
  const int k0 = blockIdx.z * kchunk;
  const int k1 = min(k0 + kchunk, d.nz + 1);
  const bool inside = (i <= d.nx) && (j <= d.ny);
  const bool own = inside && (tx / B < outx) && (ty < outy);
  const int nx = d.nx, ny = d.ny, nz = d.nz;
  const int64_t sx = (i > 0) ? B : 0;
  const int64_t sy = (j > 0) ? (int64_t)d.px * B : 0;
  const int64_t sz = d.plane * B;
  const int ii = min(i, nx), jj = min(j, ny);
  const int64_t scol = (int64_t)jj * d.px + ii;
  const int64_t col = scol * B + b;
  const bool ax_ij = (i < nx) && (j > 0) && (j < ny);
  const bool ay_ij = (j < ny) && (i > 0) && (i < nx);
  const bool az_ij = (i > 0) && (i < nx) && (j > 0) && (j < ny);
  const bool hx_ij = (i > 0) && (i < nx) && (j < ny);
  const bool hy_ij = (j > 0) && (j < ny) && (i < nx);
  const bool hz_ij = (i < nx) && (j < ny);
  const int64_t step = *d_step;
  const bool do_check = check_every > 0 && (step % check_every) == 0;
  bool bad = false;
  __syncthreads();

  auto mat_of = [&](int k) -> int { return UNIFORM ? 0 : (int)mat_id[(int64_t)k * d.plane + scol]; };
  T hx_p = 0, hy_p = 0;
  auto compute_E = [&](int k, T& hx_c, T& hy_c, T& hz_c, T& ex, T& ey, T& ez) {
    const int64_t o = (int64_t)k * sz + col;
    hx_c = Hx0[o]; hy_c = Hy0[o]; hz_c = Hz0[o];
    const T hz_jm = Hz0[o - sy], hx_jm = Hx0[o - sy];
    const T hz_im = Hz0[o - sx], hy_im = Hy0[o - sx];
    const T ex0 = Ex0[o], ey0 = Ey0[o], ez0 = Ez0[o];
    const int m = mat_of(k);
    Coef<T> cx, cy, cz;
    uint8_t ifm = 0;
    if (UNIFORM) { cx = u0; cy = u0; cz = u0; }
    else { cx = tab->c[m][0]; cy = tab->c[m][1]; cz = tab->c[m][2]; ifm = tab->ifm[m]; }
    const bool kin = (k > 0) && (k < nz);
    const T dx_ = (hz_c - hz_jm) - (hy_c - hy_p);
    const T dy_ = (hx_c - hx_p) - (hz_c - hz_im);
    const T dz_ = (hy_c - hy_im) - (hx_c - hx_jm);
    ex = (ax_ij && kin) ? ex0 + cx.apply(dx_) : (T)0;
    ey = (ay_ij && kin) ? ey0 + cy.apply(dy_) : (T)0;
    ez = (az_ij && k < nz) ? ez0 + cz.apply(dz_) : (T)0;
    if (ifm) {   // explicit rows (interface / sources)
      const int64_t s = (int64_t)k * d.plane + scol;
      if (ifm & 1) ex = eval_row(R, R.row_of[0][s], b, B, ex0, F0, y, step);
      if (ifm & 2) ey = eval_row(R, R.row_of[1][s], b, B, ey0, F0, y, step);
      if (ifm & 4) ez = eval_row(R, R.row_of[2][s], b, B, ez0, F0, y, step);
    }
  };

  T* sEx[2] = {sE, sE + 3 * BX * BY};
  const int sidx = ty * BX + tx;
  T ex_p = 0, ey_p = 0, ez_p = 0;
  T hx_c = 0, hy_c = 0, hz_c = 0;
  if (inside) {
    if (k0 > 0) {
      const int64_t o = (int64_t)(k0 - 1) * sz + col;
      hx_p = Hx0[o]; hy_p = Hy0[o];
    }
    compute_E(k0, hx_c, hy_c, hz_c, ex_p, ey_p, ez_p);
  }
  {
    T* s = sEx[k0 & 1];
    s[sidx] = ex_p; s[BX * BY + sidx] = ey_p; s[2 * BX * BY + sidx] = ez_p;
  }
  if (own) {
    const int64_t o = (int64_t)k0 * sz + col;
    F1.f[0][o] = ex_p; F1.f[1][o] = ey_p; F1.f[2][o] = ez_p;
    if (do_check) bad |= !(finite_small(ex_p) && finite_small(ey_p) && finite_small(ez_p));
  }
  for (int k = k0; k < k1; ++k) {
    T ex_n = 0, ey_n = 0, ez_n = 0;
    const T hx_k = hx_c, hy_k = hy_c, hz_k = hz_c;
    hx_p = hx_c; hy_p = hy_c;
    if (inside && k + 1 <= nz) compute_E(k + 1, hx_c, hy_c, hz_c, ex_n, ey_n, ez_n);
    T* s1 = sEx[(k + 1) & 1];
    s1[sidx] = ex_n; s1[BX * BY + sidx] = ey_n; s1[2 * BX * BY + sidx] = ez_n;
    __syncthreads();
    if (own) {
      const T* s0 = sEx[k & 1];
      const T ey_ip = s0[BX * BY + sidx + B], ez_ip = s0[2 * BX * BY + sidx + B];
      const T ex_jp = s0[sidx + BX], ez_jp = s0[2 * BX * BY + sidx + BX];
      const int64_t o = (int64_t)k * sz + col;
      Coef<T> cx, cy, cz;
      if (UNIFORM) { cx = u1; cy = u1; cz = u1; }
      else { const int m = mat_of(k); cx = tab->c[m][3]; cy = tab->c[m][4]; cz = tab->c[m][5]; }
      const T dhx = (ez_jp - ez_p) - (ey_n - ey_p);
      const T dhy = (ex_n - ex_p) - (ez_ip - ez_p);
      const T dhz = (ey_ip - ey_p) - (ex_jp - ex_p);
      const T hx1 = (hx_ij && k < nz) ? hx_k - cx.apply(dhx) : hx_k;
      const T hy1 = (hy_ij && k < nz) ? hy_k - cy.apply(dhy) : hy_k;
      const T hz1 = (hz_ij && k > 0 && k < nz) ? hz_k - cz.apply(dhz) : hz_k;
      F1.f[3][o] = hx1; F1.f[4][o] = hy1; F1.f[5][o] = hz1;
      if (k + 1 < k1 && k + 1 <= nz) {
        const int64_t o1 = o + sz;
        F1.f[0][o1] = ex_n; F1.f[1][o1] = ey_n; F1.f[2][o1] = ez_n;
      }
      if (do_check) bad |= !(finite_small(hx1) && finite_small(hy1) && finite_small(hz1) &&
                             finite_small(ex_n) && finite_small(ey_n) && finite_small(ez_n));
    }
    ex_p = ex_n; ey_p = ey_n; ez_p = ez_n;
    __syncthreads();
  }
  if (bad) atomicMin(bad_step, (unsigned long long)step);
}

// ---------------------------------------------------------------------------
// reduced blocks.  Small blocks ("fused", see fdtd_api.cu): one GEMV with the
// precomposed update matrix M per step,
//   [h~' ; y' ; e~'' ; probe rows] = M [e~ ; G ; h~],
// spread over many CTAs (16 rows each); every CTA stages the input vector in
// shared memory ([N][C] so that lanes read consecutive columns).
// ---------------------------------------------------------------------------
template <typename T>
struct Probes {
  int n_probe;
  const int64_t* rowptr;
  const int32_t* src;           // [terms] 0..5 coarse comp, 6 = e~ buffer, 7 = h~ buffer
  const int64_t* off;           // [terms] coarse: storage offset; reduced: element index
  const T* w;
  const int32_t* owner;         // [n_probe] -1: sampled by CTA 0, -2: a row of a fused matrix
};

template <typename T>
struct FusedBlock {
  int qe, qh, n_if, N, R, C, Cp;   // Cp: padded row pitch (multiple of 32 * VEC)
  const T* M;                      // [R][Cp]
  int64_t e_off, h_off, y_off;
  int n_probe_rows;
  const int32_t* probe_id;
  const int32_t* probe_inst;
};

template <typename T>
struct FusedParams {
  const FusedBlock<T>* blocks;
  const int2* ctas;             // (block, first row)
  int n_ctas, B, rows_per_cta;
  const T* e_in; T* e_out;      // e~^{n+1} in, e~^{n+2} out
  const T* h_in; T* h_out;      // h~^{n+1/2} in, h~^{n+3/2} out
  T* y;
  const T* G;                   // E_if^{n+1} published by the stencil ([n_if][N] per block)
  const T* red_base[2];         // leapfrog-path e~ / h~ buffers (probe terms 6 / 7)
  Fields<T> F;                  // coarse fields after the step
  Probes<T> pr;
  T* ring;
  int64_t cap;
  int64_t* d_step;
  unsigned int* done;
  int check_every;
  unsigned long long* bad_step;
};

template <typename T> struct Vec;
template <> struct Vec<float> { using type = float4; static constexpr int n = 4; };
template <> struct Vec<double> { using type = double2; static constexpr int n = 2; };

template <typename T>
__device__ __forceinline__ T vdot(const typename Vec<T>::type& a, const typename Vec<T>::type& x);
template <>
__device__ __forceinline__ float vdot<float>(const float4& a, const float4& x) {
  return a.x * x.x + a.y * x.y + a.z * x.z + a.w * x.w;
}
template <>
__device__ __forceinline__ double vdot<double>(const double2& a, const double2& x) {
  return a.x * x.x + a.y * x.y;
}

template <typename T, int NB>
__global__ void __launch_bounds__(256)
reduced_fused_kernel(FusedParams<T> P) {
  using V = typename Vec<T>::type;
  constexpr int VN = Vec<T>::n;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* X = reinterpret_cast<T*>(smem_raw);
  const int64_t step = *P.d_step;
  const bool check = P.check_every > 0 && (step % P.check_every) == 0;
  bool bad = false;
  const int B = P.B;
  if ((int)blockIdx.x < P.n_ctas) {
    const int2 ct = P.ctas[blockIdx.x];
    const FusedBlock<T> FB = P.blocks[ct.x];
    const int C = FB.C, Cp = FB.Cp, N = FB.N, qe = FB.qe, qh = FB.qh, ni = FB.n_if;
    // stage X = [e~ ; G ; h~ ; 0-padding] as [N][Cp]
    for (int t = threadIdx.x; t < qe * N; t += blockDim.x) X[(t % N) * Cp + t / N] = P.e_in[FB.e_off + t];
    for (int t = threadIdx.x; t < ni * N; t += blockDim.x) X[(t % N) * Cp + qe + t / N] = P.G[FB.y_off + t];
    for (int t = threadIdx.x; t < qh * N; t += blockDim.x) X[(t % N) * Cp + qe + ni + t / N] = P.h_in[FB.h_off + t];
    for (int t = threadIdx.x; t < (Cp - C) * N; t += blockDim.x) X[(t % N) * Cp + C + t / N] = (T)0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    const int r1 = min(ct.y + P.rows_per_cta, FB.R);
    for (int r = ct.y + warp; r < r1; r += nwarp) {
      T acc[NB];
#pragma unroll
      for (int n = 0; n < NB; ++n) acc[n] = 0;
      const V* a = reinterpret_cast<const V*>(FB.M + (int64_t)r * Cp);
      const int nv = Cp / VN;
#pragma unroll 8
      for (int c = lane; c < nv; c += 32) {
        const V av = a[c];
#pragma unroll
        for (int n = 0; n < NB; ++n)
          if (n < N) acc[n] += vdot<T>(av, reinterpret_cast<const V*>(X + n * Cp)[c]);
      }
#pragma unroll
      for (int n = 0; n < NB; ++n) {
        T v = acc[n];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        acc[n] = v;
      }
      if (lane < N) {
        T v = 0;
#pragma unroll
        for (int n = 0; n < NB; ++n)
          if (n == lane) v = acc[n];
        if (r < qh) P.h_out[FB.h_off + (int64_t)r * N + lane] = v;
        else if (r < qh + ni) P.y[FB.y_off + (int64_t)(r - qh) * N + lane] = v;
        else if (r < qh + ni + qe) P.e_out[FB.e_off + (int64_t)(r - qh - ni) * N + lane] = v;
        else {
          const int q = r - qh - ni - qe;
          const int p = FB.probe_id[q], in = FB.probe_inst[q];
          if (lane >= in * B && lane < in * B + B)
            P.ring[(step % P.cap) * (int64_t)P.pr.n_probe * B + (int64_t)p * B + (lane - in * B)] = v;
        }
        if (check && !finite_small((double)v)) bad = true;
      }
    }
  }
  // coarse probes and leapfrog-path reduced probes
  if (blockIdx.x == 0) {
    for (int t = threadIdx.x; t < P.pr.n_probe * B; t += blockDim.x) {
      const int p = t / B, bb = t % B;
      if (P.pr.owner[p] != -1) continue;
      T acc = 0;
      for (int64_t k = P.pr.rowptr[p]; k < P.pr.rowptr[p + 1]; ++k) {
        const int s = P.pr.src[k];
        const T v = (s < 6) ? P.F.f[s][P.pr.off[k] * B + bb] : P.red_base[s - 6][P.pr.off[k] + bb];
        acc += P.pr.w[k] * v;
      }
      P.ring[(step % P.cap) * (int64_t)P.pr.n_probe * B + t] = acc;
    }
  }
  if (bad) atomicMin(P.bad_step, (unsigned long long)step);
  // the last CTA to finish advances the device step counter
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int prev = atomicAdd(P.done, 1u);
    if (prev == gridDim.x - 1) {
      *P.done = 0;
      __threadfence();
      *P.d_step = step + 1;
    }
  }
}

// out[r][n] = (accumulate ? out[r][n] : 0) + alpha g[r] sum_c A[r][c] X[c][n]
// for the rows of this warp set (warp w handles rows w, w + nw, ...)
template <typename T, int NB>
__device__ __forceinline__ void warp_rows(int rows, int cols, int N, const T* __restrict__ A,
                                          const T* __restrict__ X, T* __restrict__ out,
                                          const T* __restrict__ g, T alpha, bool accumulate,
                                          int w0, int nw, bool check, bool& bad) {
  const int lane = threadIdx.x & 31;
  for (int r = w0; r < rows; r += nw) {
    T acc[NB];
#pragma unroll
    for (int n = 0; n < NB; ++n) acc[n] = 0;
    const T* a = A + (int64_t)r * cols;
#pragma unroll 4
    for (int c = lane; c < cols; c += 32) {
      const T av = a[c];
      const T* x = X + (int64_t)c * N;
#pragma unroll
      for (int n = 0; n < NB; ++n)
        if (n < N) acc[n] += av * x[n];
    }
#pragma unroll
    for (int n = 0; n < NB; ++n) {
      T v = acc[n];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      acc[n] = v;
    }
    if (lane < N) {
      T v = 0;
#pragma unroll
      for (int n = 0; n < NB; ++n)
        if (n == lane) v = acc[n];
      const T gr = g ? g[r] : (T)1;
      T* o = out + (int64_t)r * N + lane;
      const T res = (accumulate ? *o : (T)0) + alpha * gr * v;
      *o = res;
      if (check && !finite_small((double)res)) bad = true;
    }
  }
}

// ---------------------------------------------------------------------------
// grid-wide path for large reduced blocks (S_E of 10^5 x 10^3 and beyond)
// ---------------------------------------------------------------------------
template <typename T, int NB>
__global__ void gemv_rows_kernel(int rows, int cols, int N, const T* __restrict__ A,
                                 const T* __restrict__ X, T* __restrict__ out,
                                 const T* __restrict__ g, T alpha, bool accumulate,
                                 const int64_t* __restrict__ d_step, int check_every,
                                 unsigned long long* bad_step) {
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  bool bad = false;
  const bool check = check_every > 0 && (*d_step % check_every) == 0;
  warp_rows<T, NB>(rows, cols, N, A, X, out, g, alpha, accumulate, w0, nw, check, bad);
  if (bad) atomicMin(bad_step, (unsigned long long)*d_step);
}

template <typename T>
__global__ void gather_kernel(int64_t n, int B, const int32_t* __restrict__ comp, const int64_t* __restrict__ off,
                              const int64_t* __restrict__ dst, Fields<T> F, T* __restrict__ G) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * B) return;
  const int64_t r = t / B;
  const int b = (int)(t % B);
  G[dst[r] + b] = F.f[comp[r]][off[r] * B + b];
}

}  // namespace fdtd
