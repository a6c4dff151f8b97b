// kernels.cuh — device kernels of the reduced-hybrid FDTD step (sm_100a).
//
// Step n -> n+1 (DESIGN.md §1 rows a1-a7), all on one stream:
//   rows_e     explicit E rows (interface rows + source rows)     a1, a3
//   gemv       reduced E half  e~ -= G_e K~' h~                  a4
//   stencil    fused coarse E->H pass (ping-pong buffers)        a2, a5
//   gather     E_if -> G                                         a6
//   gemv       h~ += G_h [K~'^T | S_E^T] [e~ ; G]                a6
//   gemv       y = S_E h~                                        a6 (for a3 of step n+1)
//   probes     sample + advance the device step counter          a7
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

__device__ __forceinline__ int64_t didx(const Dims& d, int i, int j, int k) {
  return ((int64_t)k * (d.ny + 1) + j) * d.px + i;
}

__device__ __forceinline__ bool finite_small(double v) {
  return isfinite(v) && fabs(v) <= 1e100;
}

// ---------------------------------------------------------------------------
// 3-D fused E->H stencil.  Block (BX, BY) threads covers BX/B cells in x and
// BY cells in y; it computes E^{n+1} on the whole footprint and H^{n+3/2} on
// the footprint minus its last x cell and last y row (overlapped tiling: the
// halo E is recomputed by the neighbouring block, H_old / E_old are read-only
// so this is race free).  Marches z over [k0, k1).
// ---------------------------------------------------------------------------
template <typename T, bool UNIFORM>
__global__ void __launch_bounds__(1024)
stencil3d_kernel(Dims d, const T* __restrict__ Ex0, const T* __restrict__ Ey0, const T* __restrict__ Ez0,
                 const T* __restrict__ Hx0, const T* __restrict__ Hy0, const T* __restrict__ Hz0,
                 T* __restrict__ Ex1, T* __restrict__ Ey1, T* __restrict__ Ez1,
                 T* __restrict__ Hx1, T* __restrict__ Hy1, T* __restrict__ Hz1,
                 const uint8_t* __restrict__ mat_id, const Coef<T>* __restrict__ gtab,
                 const uint8_t* __restrict__ gifm, int n_mat, Coef<T> u0, Coef<T> u1,
                 int kchunk, const int64_t* __restrict__ d_step, int check_every,
                 unsigned long long* __restrict__ bad_step) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int BX = blockDim.x, BY = blockDim.y, B = d.B;
  const int tx = threadIdx.x, ty = threadIdx.y;
  // shared: E^{n+1} of two planes (3 comps), then the material table
  T* sE = reinterpret_cast<T*>(smem_raw);                       // [2][3][BY][BX]
  MatTable<T>* tab = reinterpret_cast<MatTable<T>*>(sE + 2 * 3 * BX * BY);
  if (!UNIFORM) {
    for (int m = threadIdx.y * BX + tx; m < n_mat; m += BX * BY) {
      for (int c = 0; c < 6; ++c) tab->c[m][c] = gtab[m * 6 + c];
      tab->ifm[m] = gifm[m];
    }
  }
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
  // neighbour offsets (device element units), clamped at the low walls where
  // the partner only feeds an inert (PEC) unknown
  const int64_t sx = (i > 0) ? B : 0;
  const int64_t sy = (j > 0) ? (int64_t)d.px * B : 0;
  const int64_t sz = d.plane * B;
  const int ii = min(i, nx), jj = min(j, ny);
  const int64_t col = ((int64_t)jj * d.px + ii) * B + b;       // offset within a k-plane
  // activity masks (outer PEC walls and array extents, fdtd.h conventions)
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

  // material lookup
  auto mat_of = [&](int k) -> int { return UNIFORM ? 0 : (int)mat_id[(int64_t)k * d.plane + (int64_t)jj * d.px + ii]; };

  // H^{n+1/2} of the thread's own column at planes k-1 (prev) and k (cur)
  T hx_p = 0, hy_p = 0;
  // compute E^{n+1} at plane k (needs H planes k and k-1)
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
    if (ifm) {   // explicit rows (interface / sources): value already in the new buffer
      if (ifm & 1) ex = Ex1[o];
      if (ifm & 2) ey = Ey1[o];
      if (ifm & 4) ez = Ez1[o];
    }
  };

  T* sEx[2] = {sE, sE + 3 * BX * BY};
  const int sidx = ty * BX + tx;
  T ex_p = 0, ey_p = 0, ez_p = 0;           // E^{n+1} at plane k (own column)
  T hx_c = 0, hy_c = 0, hz_c = 0;
  if (inside) {
    if (k0 > 0) {                            // H of plane k0-1 for the first E compute
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
    Ex1[o] = ex_p; Ey1[o] = ey_p; Ez1[o] = ez_p;
    if (do_check) bad |= !(finite_small(ex_p) && finite_small(ey_p) && finite_small(ez_p));
  }
  for (int k = k0; k < k1; ++k) {
    // E^{n+1} at plane k+1 (own column); H(k) moves to "prev"
    T ex_n = 0, ey_n = 0, ez_n = 0;
    T hx_k = hx_c, hy_k = hy_c, hz_k = hz_c;      // H^{n+1/2} at plane k
    hx_p = hx_c; hy_p = hy_c;
    if (inside && k + 1 <= nz) compute_E(k + 1, hx_c, hy_c, hz_c, ex_n, ey_n, ez_n);
    T* s1 = sEx[(k + 1) & 1];
    s1[sidx] = ex_n; s1[BX * BY + sidx] = ey_n; s1[2 * BX * BY + sidx] = ez_n;
    __syncthreads();
    if (own) {
      const T* s0 = sEx[k & 1];
      // neighbours at plane k: (i+1, j) and (i, j+1)
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
      Hx1[o] = hx1; Hy1[o] = hy1; Hz1[o] = hz1;
      if (k + 1 < k1 && k + 1 <= nz) {
        const int64_t o1 = o + sz;
        Ex1[o1] = ex_n; Ey1[o1] = ey_n; Ez1[o1] = ez_n;
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
// 2-D (Ez, Hx, Hy) fused stencil: block of BX threads covers BX/B cells in x,
// marches y over [j0, j1).
// Ez += cb ((Hy(i) - Hy(i-1)) - (Hx(j) - Hx(j-1)))
// Hx -= ch (Ez(j+1) - Ez(j))        Hy += ch (Ez(i+1) - Ez(i))
// ---------------------------------------------------------------------------
template <typename T, bool UNIFORM>
__global__ void __launch_bounds__(1024)
stencil2d_kernel(Dims d, const T* __restrict__ Ez0, const T* __restrict__ Hx0, const T* __restrict__ Hy0,
                 T* __restrict__ Ez1, T* __restrict__ Hx1, T* __restrict__ Hy1,
                 const uint8_t* __restrict__ mat_id, const Coef<T>* __restrict__ gtab,
                 const uint8_t* __restrict__ gifm, int n_mat, Coef<T> u0, Coef<T> u1,
                 int jchunk, const int64_t* __restrict__ d_step, int check_every,
                 unsigned long long* __restrict__ bad_step) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int BX = blockDim.x, B = d.B, tx = threadIdx.x;
  T* sE = reinterpret_cast<T*>(smem_raw);                  // [2][BX]
  MatTable<T>* tab = reinterpret_cast<MatTable<T>*>(sE + 2 * BX);
  if (!UNIFORM) {
    for (int m = tx; m < n_mat; m += BX) {
      for (int c = 0; c < 6; ++c) tab->c[m][c] = gtab[m * 6 + c];
      tab->ifm[m] = gifm[m];
    }
  }
  const int outx = BX / B - 1;
  const int i = blockIdx.x * outx + tx / B;
  const int b = tx % B;
  const int j0 = blockIdx.y * jchunk;
  const int j1 = min(j0 + jchunk, d.ny + 1);
  const int nx = d.nx, ny = d.ny;
  const bool inside = i <= nx;
  const bool own = inside && (tx / B < outx);
  const int ii = min(i, nx);
  const int64_t sx = (i > 0) ? B : 0;
  const int64_t rowst = (int64_t)d.px * B;
  const int64_t step = *d_step;
  const bool do_check = check_every > 0 && (step % check_every) == 0;
  bool bad = false;
  __syncthreads();
  auto mat_of = [&](int j) -> int { return UNIFORM ? 0 : (int)mat_id[(int64_t)j * d.px + ii]; };
  const bool ez_i = (i > 0) && (i < nx);
  T hx_p = 0;                                    // Hx^{n+1/2}(i, j-1)
  auto compute_E = [&](int j, T& hx_c, T& hy_c) -> T {
    const int64_t o = (int64_t)j * rowst + (int64_t)ii * B + b;
    hx_c = Hx0[o]; hy_c = Hy0[o];
    const T hy_im = Hy0[o - sx];
    const T ez0 = Ez0[o];
    T ez;
    int m = mat_of(j);
    Coef<T> c = UNIFORM ? u0 : tab->c[m][2];
    const T dd = (hy_c - hy_im) - (hx_c - hx_p);
    ez = (ez_i && j > 0 && j < ny) ? ez0 + c.apply(dd) : (T)0;
    if (!UNIFORM && (tab->ifm[m] & 4)) ez = Ez1[o];
    return ez;
  };
  T hx_c = 0, hy_c = 0, ez_p = 0;
  if (inside) {
    if (j0 > 0) hx_p = Hx0[(int64_t)(j0 - 1) * rowst + (int64_t)ii * B + b];
    ez_p = compute_E(j0, hx_c, hy_c);
    if (own) {
      Ez1[(int64_t)j0 * rowst + (int64_t)ii * B + b] = ez_p;
      if (do_check) bad |= !finite_small(ez_p);
    }
  }
  for (int j = j0; j < j1; ++j) {
    const T hx_j = hx_c, hy_j = hy_c;
    hx_p = hx_c;
    T ez_n = 0;
    if (inside && j + 1 <= ny) ez_n = compute_E(j + 1, hx_c, hy_c);
    sE[(j & 1) * BX + tx] = ez_p;
    __syncthreads();
    if (own) {
      const int64_t o = (int64_t)j * rowst + (int64_t)ii * B + b;
      const T ez_ip = sE[(j & 1) * BX + tx + B];
      Coef<T> cx, cy;
      if (UNIFORM) { cx = u1; cy = u1; }
      else { const int m = mat_of(j); cx = tab->c[m][3]; cy = tab->c[m][4]; }
      const T hx1 = (i > 0 && i < nx && j < ny) ? hx_j - cx.apply(ez_n - ez_p) : hx_j;
      const T hy1 = (i < nx && j > 0 && j < ny) ? hy_j + cy.apply(ez_ip - ez_p) : hy_j;
      Hx1[o] = hx1; Hy1[o] = hy1;
      if (j + 1 < j1 && j + 1 <= ny) Ez1[o + rowst] = ez_n;
      if (do_check) bad |= !(finite_small(hx1) && finite_small(hy1) && finite_small(ez_n));
    }
    ez_p = ez_n;
    __syncthreads();
  }
  if (bad) atomicMin(bad_step, (unsigned long long)step);
}

// ---------------------------------------------------------------------------
// explicit E rows: E1[u] = E0[u] - c (sum_k W_k H0[col_k] + y) - cs J[step]
// one thread per (row, member)
// ---------------------------------------------------------------------------
template <typename T>
struct RowsE {
  int64_t n_rows;
  const int32_t* e_comp;       // [n_rows]
  const int64_t* e_off;        // [n_rows] storage offset (device index / B)
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
};

template <typename T>
__global__ void rows_e_kernel(RowsE<T> R, int B, const T* const* E0, T* const* E1, const T* const* H0,
                              const T* __restrict__ y, const int64_t* __restrict__ d_step) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= R.n_rows * B) return;
  const int64_t r = t / B;
  const int b = (int)(t % B);
  T acc = 0;
  for (int64_t k = R.rowptr[r]; k < R.rowptr[r + 1]; ++k)
    acc += R.w[k] * H0[R.h_comp[k]][R.h_off[k] * B + b];
  const int64_t yo = R.y_off[r];
  if (yo >= 0) acc += y[yo + b];
  const int ec = R.e_comp[r];
  const int64_t eo = R.e_off[r] * B + b;
  T e = E0[ec][eo] - R.c[r].apply(acc);
  const int s = R.src[r];
  const int64_t step = *d_step;
  if (s >= 0 && step < R.n_wave) e -= R.cs[r] * R.wave[(step * R.n_src + s) * B + b];
  E1[ec][eo] = e;
}

// ---------------------------------------------------------------------------
// small dense products for the reduced blocks:
//   out[r][n] = beta * out[r][n] + alpha * g[r] * sum_c A[r][c] X[c][n],  n < N
// one warp per row, A row-major (rows x cols), X [cols][N], N <= NB.
// ---------------------------------------------------------------------------
template <typename T, int NB>
__global__ void gemv_rows_kernel(int rows, int cols, int N, const T* __restrict__ A,
                                 const T* __restrict__ X, T* __restrict__ out,
                                 const T* __restrict__ g, T g_scalar, T alpha, T beta,
                                 const int64_t* __restrict__ d_step, int check_every, unsigned long long* bad_step) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  T acc[NB];
#pragma unroll
  for (int n = 0; n < NB; ++n) acc[n] = 0;
  const T* a = A + (int64_t)warp * cols;
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
    const T gr = g ? g[warp] : g_scalar;
    T* o = out + (int64_t)warp * N + lane;
    const T res = (beta == (T)0 ? (T)0 : beta * *o) + alpha * gr * v;
    *o = res;
    if (check_every > 0 && (*d_step % check_every) == 0 && !finite_small((double)res))
      atomicMin(bad_step, (unsigned long long)*d_step);
  }
}

// gather interface E values: G[l][inst*B + b] = E[comp][off*B + b]
template <typename T>
__global__ void gather_kernel(int64_t n, int B, const int32_t* __restrict__ comp, const int64_t* __restrict__ off,
                              const int64_t* __restrict__ dst, T* const* E, T* __restrict__ G) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * B) return;
  const int64_t r = t / B;
  const int b = (int)(t % B);
  G[dst[r] + b] = E[comp[r]][off[r] * B + b];
}

// probes: one block; ring[(step % cap)][p][b]; then step += 1
template <typename T>
struct Probes {
  int n_probe;
  const int64_t* rowptr;
  const int32_t* src;        // [terms] 0..5 coarse comp, 6 = e~ buffer, 7 = h~ buffer
  const int64_t* off;        // [terms] element offset (coarse: storage offset, reduced: base index)
  const int32_t* stride;     // [terms] multiplier for b (coarse: 1, reduced: 1)
  const T* w;
};

template <typename T>
__global__ void probe_kernel(Probes<T> P, int B, const T* const* F, const T* const* RED,
                             T* __restrict__ ring, int64_t cap, int64_t* d_step) {
  const int64_t step = *d_step;
  for (int t = threadIdx.x; t < P.n_probe * B; t += blockDim.x) {
    const int p = t / B, b = t % B;
    T acc = 0;
    for (int64_t k = P.rowptr[p]; k < P.rowptr[p + 1]; ++k) {
      const int s = P.src[k];
      const T v = (s < 6) ? F[s][P.off[k] * B + b] : RED[s - 6][P.off[k] + b];
      acc += P.w[k] * v;
    }
    ring[(step % cap) * (int64_t)P.n_probe * B + t] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) *d_step = step + 1;
}

}  // namespace fdtd
