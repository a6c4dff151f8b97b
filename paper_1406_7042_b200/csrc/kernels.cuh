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
#include <type_traits>
#include <cuda.h>
#include <cuda_runtime.h>

namespace fdtd {


template <typename T> struct Coef;       // per-material coefficient, hi/lo for fp32 (R11)
template <> struct Coef<float> {
  float hi, lo;
  __device__ __forceinline__ float apply(float d) const { return fmaf(hi, d, lo * d); }
  // e +- c d with the rounding sequence every stencil kernel uses (bitwise-equality tests)
  __device__ __forceinline__ float add(float e, float d) const { return e + fmaf(hi, d, lo * d); }
  __device__ __forceinline__ float sub(float e, float d) const { return e - fmaf(hi, d, lo * d); }
};
template <> struct Coef<double> {
  double hi, lo;
  __device__ __forceinline__ double apply(double d) const { return hi * d; }
  // fp64: one fused multiply-add (what the compiler's contraction makes of
  // e + hi * d in the reference kernels), spelled out so that restructured code
  // cannot round differently
  __device__ __forceinline__ double add(double e, double d) const { return __fma_rn(hi, d, e); }
  __device__ __forceinline__ double sub(double e, double d) const { return __fma_rn(-hi, d, e); }
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
  const int32_t* src;          // [n_rows] waveform column or -1
  const T* cs;                 // [n_rows] source coefficient (amplitude * dt / eps)
  const T* wave;               // [n_wave][n_src][B]   (n_src = number of waveform columns)
  int64_t n_wave, n_src;
  T* g_out;                    // interface rows publish E^{n+1} at G[y_off] (reduced-chain input)
  const T* a;                  // [n_rows] ca of the row's unknown (lossy media), null: lossless
  // list form (rows_prepass_kernel)
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
  T e = R.a ? fma(R.a[r], e0, -R.c[r].apply(acc)) : R.c[r].sub(e0, acc);
  const int s = R.src[r];
  if (s >= 0 && step < R.n_wave) e -= R.cs[r] * R.wave[(step * R.n_src + s) * B + b];
  if (yo >= 0) R.g_out[yo + b] = e;        // identical value from every thread computing it
  return e;
}

// Explicit rows ahead of the 3-D tile stencil: one thread per
// (row, batch member) evaluates the row from the old parity (the same CSR walk
// as in the reference stencils, so the value is theirs bit for bit), publishes
// it into G and stores E^{n+1} of the row's unknown into the NEW parity; the
// stencil thread that owns the unknown then reads that value back instead of
// walking the row itself (a chain of dependent global loads per row that made
// the tiles with interface rows the stragglers of the step).
template <typename T>
__global__ void __launch_bounds__(256)
rows_prepass_kernel(RowsE<T> R, int B, Fields<T> F0, Fields<T> F1, const T* __restrict__ y,
                    const int64_t* __restrict__ d_step) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= R.n_rows * B) return;
  const int r = (int)(t / B), b = (int)(t % B);
  const int64_t o = R.e_off[r] * B + b;
  const int c = R.e_comp[r];
  F1.f[c][o] = eval_row(R, r, b, B, F0.f[c][o], F0, y, *d_step);
}

// The same pre-pass on packed row records (every row has at most 4 H terms --
// all interface rows of the R4 construction and all source rows): one level of
// row-indexed loads (3 x 16 bytes of integers, the reals), then the field / y /
// waveform loads, instead of eval_row's chain of dependent CSR loads.  The
// arithmetic is eval_row's, term by term in CSR order.
struct RowPackI {          // 48 bytes
  int32_t e_comp, e_off, nterm, src;
  int32_t h_off[4];
  int32_t h_comp;          // 4 x 8 bits
  int32_t y_off;           // -1: none
  int32_t pad[2];
};
template <typename T>
struct RowPackR {          // 32 (fp32) / 64 (fp64) bytes
  T w[4];
  Coef<T> c;
  T cs;
  T a;                     // ca of the row's unknown (1 when lossless)
};

// One packed explicit row of member b: E^{n+1} from the old parity F0, the y
// value yv (ignored without a y term) and the step's source sample; stored
// into the new parity F1 and published to g_out.
template <typename T>
__device__ __forceinline__ void packed_row_eval(int r, int b, T yv, const RowPackI* __restrict__ RI,
                                                const RowPackR<T>* __restrict__ RR, int B, const Fields<T>& F0,
                                                const Fields<T>& F1, T* __restrict__ g_out,
                                                const T* __restrict__ wave, int64_t n_wave, int64_t n_src,
                                                int64_t step, int lossy) {
  const int4* pi = reinterpret_cast<const int4*>(RI + r);
  const int4 i0 = pi[0], i1 = pi[1], i2 = pi[2];
  const RowPackR<T> rr = RR[r];
  auto field = [&](int c) -> const T* {
    return c == 0 ? F0.f[0] : c == 1 ? F0.f[1] : c == 2 ? F0.f[2] : c == 3 ? F0.f[3] : c == 4 ? F0.f[4] : F0.f[5];
  };
  const int ec = i0.x, nt = i0.z, src = i0.w, yo = i2.y;
  const int64_t eo = (int64_t)i0.y * B + b;
  const int ho[4] = {i1.x, i1.y, i1.z, i1.w};
  const T e0 = field(ec)[eo];
  T h[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) h[k] = k < nt ? field((i2.x >> (8 * k)) & 0xff)[(int64_t)ho[k] * B + b] : (T)0;
  const bool has_src = src >= 0 && step < n_wave;
  const T wv = has_src ? wave[(step * n_src + src) * B + b] : (T)0;
  T acc = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (k < nt) acc += rr.w[k] * h[k];
  if (yo >= 0) acc += yv;
  T e = lossy ? fma(rr.a, e0, -rr.c.apply(acc)) : rr.c.sub(e0, acc);
  if (has_src) e -= rr.cs * wv;
  if (yo >= 0) g_out[yo + b] = e;
  T* o = ec == 0 ? F1.f[0] : ec == 1 ? F1.f[1] : F1.f[2];
  o[eo] = e;
}

template <typename T>
__global__ void __launch_bounds__(256)
rows_prepass_packed_kernel(int64_t n_rows, const RowPackI* __restrict__ RI, const RowPackR<T>* __restrict__ RR,
                           int B, Fields<T> F0, Fields<T> F1, const T* __restrict__ y, T* __restrict__ g_out,
                           const T* __restrict__ wave, int64_t n_wave, int64_t n_src,
                           const int64_t* __restrict__ d_step, int lossy) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_rows * B) return;
  const int r = (int)(t / B), b = (int)(t % B);
  const int yo = RI[r].y_off;
  const T yv = yo >= 0 ? y[yo + b] : (T)0;
  packed_row_eval<T>(r, b, yv, RI, RR, B, F0, F1, g_out, wave, n_wave, n_src, *d_step, lossy);
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
                      unsigned long long* __restrict__ bad_step, const T* __restrict__ taba) {
  // taba: [n_mat][6] ca / da of lossy media (null: lossless, the branch is never taken)
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
  // 32-bit element offsets (the host checks the 2-D state fits)
  const int sx = (i > 0) ? B : 0;
  const int rs = d.px * B;
  const int64_t step = *d_step;
  // issue every load first
  T hx[CY], hy[CY], hyim[CY], ez0[CY];
  int m[CY];
  const int o0 = (min(jb, ny) * d.px + ii) * B + b;
#pragma unroll
  for (int r = 0; r < CY; ++r) {
    const int o = (min(jb + r, ny) * d.px + ii) * B + b;
    hx[r] = Hx0[o]; hy[r] = Hy0[o]; hyim[r] = Hy0[o - sx]; ez0[r] = Ez0[o];
    m[r] = UNIFORM ? 0 : (int)mat_id[min(jb + r, ny) * d.px + ii];
  }
  const T hx_jm = (jb > 0) ? Hx0[o0 - rs] : (T)0;
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
    ez[r] = (ci && j > 0 && j < ny) ? ((!UNIFORM && taba) ? fma(__ldg(taba + m[r] * 6 + 2), ez0[r], c.apply(dd)) : c.add(ez0[r], dd))
                                    : (T)0;
    if (!UNIFORM && (tab->ifm[m[r]] & 4) && i <= nx && j <= ny)
      ez[r] = eval_row(R, R.row_of[2][min(j, ny) * d.px + ii], b, B, ez0[r], F0, y, step);
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
    T hx1, hy1;
    if (!UNIFORM && taba) {
      const T ax = __ldg(taba + m[r] * 6 + 3), ay = __ldg(taba + m[r] * 6 + 4);
      hx1 = (ci && j < ny) ? fma(ax, hx[r], -cx.apply(ez_jp - ez[r])) : hx[r];
      hy1 = (i < nx && j > 0 && j < ny) ? fma(ay, hy[r], cy.apply(ez_ip - ez[r])) : hy[r];
    } else {
      hx1 = (ci && j < ny) ? cx.sub(hx[r], ez_jp - ez[r]) : hx[r];
      hy1 = (i < nx && j > 0 && j < ny) ? cy.add(hy[r], ez_ip - ez[r]) : hy[r];
    }
    const int o = o0 + r * rs;
    F1.f[2][o] = ez[r]; F1.f[3][o] = hx1; F1.f[4][o] = hy1;
    if (do_check) bad |= !(finite_small(ez[r]) && finite_small(hx1) && finite_small(hy1));
  }
  if (bad) atomicMin(bad_step, (unsigned long long)step);
}

// ---------------------------------------------------------------------------
// 3-D fused E->H stencil with a cp.async (LDGSTS) z-plane pipeline.
// Block (BX, BY) threads covers BX/B cells in x and BY cells in y and marches
// z over [k0, k1).  Planes of H (with a -x / -y halo) and of E_old stream into
// an NS-stage shared-memory ring NS-1 planes ahead of use, so every thread
// keeps ~(NS-1) x 6 words of HBM traffic in flight without registers.  E^{n+1}
// is computed on the whole footprint (overlapped tiling) and H^{n+3/2} on the
// footprint minus its last x cell and last y row.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
template <typename T>
__device__ __forceinline__ void cp_async(T* dst, const T* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(smem_u32(dst)), "l"(src),
               "n"(sizeof(T)), "r"(valid ? (int)sizeof(T) : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
// 16-byte global -> shared copy; zero-fills when !valid
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 16 : 0));
}

template <typename T, bool UNIFORM, int NS>
__global__ void __launch_bounds__(256, 3)
stencil3d_pipe_kernel(Dims d, Fields<T> F0, Fields<T> F1, const uint8_t* __restrict__ mat_id,
                      const Coef<T>* __restrict__ gtab, const uint8_t* __restrict__ gifm, int n_mat,
                      Coef<T> u0, Coef<T> u1, RowsE<T> R, const T* __restrict__ y, int kchunk,
                      const int64_t* __restrict__ d_step, int check_every,
                      unsigned long long* __restrict__ bad_step) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int BX = blockDim.x, BY = blockDim.y, B = d.B;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int HW = BX + B, HH = BY + 1;                 // H plane with halo
  const int HP = HW * HH, EP = BX * BY;
  T* Hs = reinterpret_cast<T*>(smem_raw);            // [NS][3][HH][HW]
  T* Es = Hs + NS * 3 * HP;                          // [NS][3][BY][BX]
  T* En = Es + NS * 3 * EP;                          // [2][3][BY][BX]
  MatTable<T>* tab = reinterpret_cast<MatTable<T>*>(En + 2 * 3 * EP);
  if (!UNIFORM) {
    for (int m = ty * BX + tx; m < n_mat; m += BX * BY) {
      for (int c = 0; c < 6; ++c) tab->c[m][c] = gtab[m * 6 + c];
      tab->ifm[m] = gifm[m];
    }
  }
  const int nx = d.nx, ny = d.ny, nz = d.nz;
  const int outx = BX / B - 1, outy = BY - 1;
  const int i = blockIdx.x * outx + tx / B;
  const int b = tx % B;
  const int j = blockIdx.y * outy + ty;
  const int k0 = blockIdx.z * kchunk;
  const int k1 = min(k0 + kchunk, nz + 1);
  const int kend = min(k1, nz);                      // last E plane computed
  const bool inside = (i <= nx) && (j <= ny);
  const bool own = inside && (tx / B < outx) && (ty < outy);
  const int ii = min(i, nx), jj = min(j, ny);
  const int64_t scol = (int64_t)jj * d.px + ii;
  const int64_t col = scol * B + b;
  const int64_t sz = d.plane * B;
  const int xi = tx + B, yi = ty + 1;
  // halo sources: -y row (ty == 0) and -x column (tx < B)
  const bool hy_halo = (ty == 0), hx_halo = (tx < B);
  const int64_t col_jm = ((int64_t)max(j - 1, 0) * d.px + ii) * B + b;
  const int64_t col_im = ((int64_t)jj * d.px + max(i - 1, 0)) * B + b;
  const bool ok_jm = inside && j > 0, ok_im = inside && i > 0;
  const bool ax_ij = (i < nx) && (j > 0) && (j < ny);
  const bool ay_ij = (j < ny) && (i > 0) && (i < nx);
  const bool az_ij = (i > 0) && (i < nx) && (j > 0) && (j < ny);
  const bool hx_ij = (i > 0) && (i < nx) && (j < ny);
  const bool hy_ij = (j > 0) && (j < ny) && (i < nx);
  const bool hz_ij = (i < nx) && (j < ny);
  const int64_t step = *d_step;
  const bool do_check = check_every > 0 && (step % check_every) == 0;
  bool bad = false;

  auto issue = [&](int k) {
    const int st = k % NS;
    T* h = Hs + st * 3 * HP;
    T* e = Es + st * 3 * EP;
    const int64_t o = (int64_t)k * sz;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      cp_async(h + c * HP + yi * HW + xi, F0.f[3 + c] + o + col, inside);
      cp_async(e + c * EP + ty * BX + tx, F0.f[c] + o + col, inside);
    }
    if (hy_halo) {     // H at j-1: Hx and Hz are used
      cp_async(h + 0 * HP + 0 * HW + xi, F0.f[3] + o + col_jm, ok_jm);
      cp_async(h + 2 * HP + 0 * HW + xi, F0.f[5] + o + col_jm, ok_jm);
    }
    if (hx_halo) {     // H at i-1: Hy and Hz are used
      cp_async(h + 1 * HP + yi * HW + tx, F0.f[4] + o + col_im, ok_im);
      cp_async(h + 2 * HP + yi * HW + tx, F0.f[5] + o + col_im, ok_im);
    }
  };
  // prologue: planes k0 .. k0+NS-2 in flight; own H of plane k0-1 in registers
#pragma unroll
  for (int q = 0; q < NS - 1; ++q) {
    if (k0 + q <= kend) issue(k0 + q);
    cp_async_commit();
  }
  T hx_p = 0, hy_p = 0;
  if (inside && k0 > 0) {
    const int64_t o = (int64_t)(k0 - 1) * sz + col;
    hx_p = F0.f[3][o]; hy_p = F0.f[4][o];
  }
  __syncthreads();                                   // material table
  T hxk = 0, hyk = 0, hzk = 0;                       // H_old of the previous plane (own)
  T exk = 0, eyk = 0, ezk = 0;                       // E_new of the previous plane (own)
  int m_next = UNIFORM ? 0 : (int)__ldg(mat_id + (int64_t)k0 * d.plane + scol), m_prev = 0;
  for (int kk = k0; kk <= kend; ++kk) {
    if (kk + NS - 1 <= kend) issue(kk + NS - 1);
    cp_async_commit();
    cp_async_wait<NS - 1>();
    __syncthreads();
    const int st = kk % NS;
    const T* h = Hs + st * 3 * HP;
    const T* e = Es + st * 3 * EP;
    const T hx_c = h[0 * HP + yi * HW + xi], hy_c = h[1 * HP + yi * HW + xi], hz_c = h[2 * HP + yi * HW + xi];
    const T hz_jm = h[2 * HP + (yi - 1) * HW + xi], hx_jm = h[0 * HP + (yi - 1) * HW + xi];
    const T hz_im = h[2 * HP + yi * HW + xi - B], hy_im = h[1 * HP + yi * HW + xi - B];
    const T ex0 = e[0 * EP + ty * BX + tx], ey0 = e[1 * EP + ty * BX + tx], ez0 = e[2 * EP + ty * BX + tx];
    const int m = m_next;                                   // material of plane kk (prefetched)
    if (!UNIFORM && kk + 1 <= kend) m_next = (int)__ldg(mat_id + (int64_t)(kk + 1) * d.plane + scol);
    Coef<T> cx, cy, cz;
    uint8_t ifmk = 0;
    if (UNIFORM) { cx = u0; cy = u0; cz = u0; }
    else { cx = tab->c[m][0]; cy = tab->c[m][1]; cz = tab->c[m][2]; ifmk = tab->ifm[m]; }
    const bool kin = (kk > 0) && (kk < nz);
    T ex = (ax_ij && kin) ? cx.add(ex0, (hz_c - hz_jm) - (hy_c - hy_p)) : (T)0;
    T ey = (ay_ij && kin) ? cy.add(ey0, (hx_c - hx_p) - (hz_c - hz_im)) : (T)0;
    T ez = (az_ij && kk < nz) ? cz.add(ez0, (hy_c - hy_im) - (hx_c - hx_jm)) : (T)0;
    if (!UNIFORM && ifmk && inside) {
      const int64_t s = (int64_t)kk * d.plane + scol;
      if (ifmk & 1) ex = eval_row(R, R.row_of[0][s], b, B, ex0, F0, y, step);
      if (ifmk & 2) ey = eval_row(R, R.row_of[1][s], b, B, ey0, F0, y, step);
      if (ifmk & 4) ez = eval_row(R, R.row_of[2][s], b, B, ez0, F0, y, step);
    }
    T* en = En + (kk & 1) * 3 * EP;
    en[0 * EP + ty * BX + tx] = ex; en[1 * EP + ty * BX + tx] = ey; en[2 * EP + ty * BX + tx] = ez;
    if (own && kk < k1) {
      const int64_t o = (int64_t)kk * sz + col;
      F1.f[0][o] = ex; F1.f[1][o] = ey; F1.f[2][o] = ez;
      if (do_check) bad |= !(finite_small(ex) && finite_small(ey) && finite_small(ez));
    }
    __syncthreads();
    if (kk > k0 && own) {       // H^{n+3/2} of plane kk-1
      const T* e0 = En + ((kk - 1) & 1) * 3 * EP;
      const int q = ty * BX + tx;
      const T ey_ip = e0[1 * EP + q + B], ez_ip = e0[2 * EP + q + B];
      const T ex_jp = e0[0 * EP + q + BX], ez_jp = e0[2 * EP + q + BX];
      const int km = kk - 1;
      Coef<T> hx_, hy_, hz_;
      if (UNIFORM) { hx_ = u1; hy_ = u1; hz_ = u1; }
      else { hx_ = tab->c[m_prev][3]; hy_ = tab->c[m_prev][4]; hz_ = tab->c[m_prev][5]; }   // plane kk-1
      const T hx1 = (hx_ij && km < nz) ? hx_.sub(hxk, (ez_jp - ezk) - (ey - eyk)) : hxk;
      const T hy1 = (hy_ij && km < nz) ? hy_.sub(hyk, (ex - exk) - (ez_ip - ezk)) : hyk;
      const T hz1 = (hz_ij && km > 0 && km < nz) ? hz_.sub(hzk, (ey_ip - eyk) - (ex_jp - exk)) : hzk;
      const int64_t o = (int64_t)km * sz + col;
      F1.f[3][o] = hx1; F1.f[4][o] = hy1; F1.f[5][o] = hz1;
      if (do_check) bad |= !(finite_small(hx1) && finite_small(hy1) && finite_small(hz1));
    }
    hx_p = hx_c; hy_p = hy_c;
    hxk = hx_c; hyk = hy_c; hzk = hz_c;
    exk = ex; eyk = ey; ezk = ez;
    m_prev = m;
  }
  // last chunk: plane nz of H has no update (Hx, Hy absent, Hz normal to the
  // PEC wall); the new buffer still needs it
  if (k1 == nz + 1 && own) {
    const int64_t o = (int64_t)nz * sz + col;
    F1.f[3][o] = hxk; F1.f[4][o] = hyk; F1.f[5][o] = hzk;
  }
  cp_async_wait<0>();
  if (bad) atomicMin(bad_step, (unsigned long long)step);
}

// ---------------------------------------------------------------------------
// 3-D fused E->H stencil, TMA version.  Per z-plane one elected thread issues
// six cp.async.bulk.tensor tile loads (Hx, Hy, Hz with a -x/-y halo, Ex, Ey,
// Ez) into an NS-stage shared-memory ring, completing on one mbarrier per
// stage; the 256 threads only compute and store.  The tensor maps start one
// row and SX elements (16 bytes) before each field (a zeroed guard allocation
// and spare end-of-row columns), and the tile origins are multiples of 16
// bytes: box starts are then never negative and always 16-byte aligned (both
// raised illegal-instruction faults on this driver, tools/dbg/tma_probe*).
// The tail past nx / ny is zero-filled.  Same overlapped tiling and z-march
// as stencil3d_pipe_kernel, with the x overlap rounded up to the alignment.
// ---------------------------------------------------------------------------
struct TmaSet {
  CUtensorMap h[3];             // box (HBX, BY+1, 1), start (x0 - B, j0 - 1, k)
  CUtensorMap e[3];             // box (BX, BY, 1),    start (x0, j0, k)
};

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

template <typename T, bool UNIFORM, int NS>
__global__ void __launch_bounds__(256, 3)
stencil3d_tma_kernel(const __grid_constant__ TmaSet tm, int HBX, int SX, int outx, Dims d, Fields<T> F0, Fields<T> F1,
                     const uint8_t* __restrict__ mat_id, const Coef<T>* __restrict__ gtab,
                     const uint8_t* __restrict__ gifm, int n_mat, Coef<T> u0, Coef<T> u1, RowsE<T> R,
                     const T* __restrict__ y, int kchunk, const int64_t* __restrict__ d_step,
                     int check_every, unsigned long long* __restrict__ bad_step) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int BX = blockDim.x, BY = blockDim.y, B = d.B;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int HW = HBX, HH = BY + 1;
  // every TMA destination starts on a 128-byte boundary
  const int al = 128 / (int)sizeof(T);
  const int HP = (HW * HH + al - 1) / al * al, EP = (BX * BY + al - 1) / al * al;
  const unsigned base_u = smem_u32(smem_raw);
  unsigned char* smem_al = smem_raw + ((128u - (base_u & 127u)) & 127u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_al);                 // [NS]
  T* Hs = reinterpret_cast<T*>(smem_al + 128);                           // [NS][3][HH][HW]
  T* Es = Hs + NS * 3 * HP;                                               // [NS][3][BY][BX]
  // E^{n+1} planes: three buffers, because no CTA barrier separates iteration
  // kk's H update (reads plane kk-1, rows ty+1 written by another warp) from
  // iteration kk+1's stores -- only the mbarrier wait, which is per thread
  T* En = Es + NS * 3 * EP;                                               // [3][3][BY][BX]
  MatTable<T>* tab = reinterpret_cast<MatTable<T>*>(En + 3 * 3 * EP);
  const bool leader = (tx == 0 && ty == 0);
  if (leader) {
    for (int q = 0; q < NS; ++q) mbar_init(&bars[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (!UNIFORM) {
    for (int m = ty * BX + tx; m < n_mat; m += BX * BY) {
      for (int c = 0; c < 6; ++c) tab->c[m][c] = gtab[m * 6 + c];
      tab->ifm[m] = gifm[m];
    }
  }
  __syncthreads();
  const int nx = d.nx, ny = d.ny, nz = d.nz;
  const int outy = BY - 1;                  // outx: aligned so box origins are 16-byte aligned
  const int i0 = blockIdx.x * outx, j0 = blockIdx.y * outy;
  const int i = i0 + tx / B;
  const int b = tx % B;
  const int j = j0 + ty;
  const int k0 = blockIdx.z * kchunk;
  const int k1 = min(k0 + kchunk, nz + 1);
  const int kend = min(k1, nz);
  const bool inside = (i <= nx) && (j <= ny);
  const bool own = inside && (tx / B < outx) && (ty < outy);
  const int ii = min(i, nx), jj = min(j, ny);
  const int64_t scol = (int64_t)jj * d.px + ii;
  const int64_t col = scol * B + b;
  const int64_t sz = d.plane * B;
  const int xi = tx + SX, yi = ty + 1;      // H box starts SX elements before the tile
  const bool ax_ij = (i < nx) && (j > 0) && (j < ny);
  const bool ay_ij = (j < ny) && (i > 0) && (i < nx);
  const bool az_ij = (i > 0) && (i < nx) && (j > 0) && (j < ny);
  const bool hx_ij = (i > 0) && (i < nx) && (j < ny);
  const bool hy_ij = (j > 0) && (j < ny) && (i < nx);
  const bool hz_ij = (i < nx) && (j < ny);
  const int64_t step = *d_step;
  const bool do_check = check_every > 0 && (step % check_every) == 0;
  bool bad = false;
  // transaction bytes = the boxes actually delivered (not the padded slots)
  const unsigned stage_bytes = (unsigned)((3 * HW * HH + 3 * BX * BY) * sizeof(T));
  // the tensor maps are addressed in kernel-parameter space (__grid_constant__):
  // no lambda / local copy may be taken of them
#define FDTD_TMA_ISSUE(K)                                                              \
  do {                                                                                 \
    const int st_ = ((K) - k0) % NS;                                                   \
    T* h_ = Hs + st_ * 3 * HP;                                                         \
    T* e_ = Es + st_ * 3 * EP;                                                         \
    mbar_expect_tx(&bars[st_], stage_bytes);                                           \
    tma_load_3d(h_ + 0 * HP, &tm.h[0], i0 * B, j0, (K), &bars[st_]);                   \
    tma_load_3d(h_ + 1 * HP, &tm.h[1], i0 * B, j0, (K), &bars[st_]);                   \
    tma_load_3d(h_ + 2 * HP, &tm.h[2], i0 * B, j0, (K), &bars[st_]);                   \
    tma_load_3d(e_ + 0 * EP, &tm.e[0], i0 * B + SX, j0 + 1, (K), &bars[st_]);          \
    tma_load_3d(e_ + 1 * EP, &tm.e[1], i0 * B + SX, j0 + 1, (K), &bars[st_]);          \
    tma_load_3d(e_ + 2 * EP, &tm.e[2], i0 * B + SX, j0 + 1, (K), &bars[st_]);          \
  } while (0)
  if (leader) {
    for (int q = 0; q < NS - 1; ++q)
      if (k0 + q <= kend) FDTD_TMA_ISSUE(k0 + q);
  }
  T hx_p = 0, hy_p = 0;
  if (inside && k0 > 0) {
    const int64_t o = (int64_t)(k0 - 1) * sz + col;
    hx_p = F0.f[3][o]; hy_p = F0.f[4][o];
  }
  T hxk = 0, hyk = 0, hzk = 0;
  T exk = 0, eyk = 0, ezk = 0;
  int m_next = UNIFORM ? 0 : (int)__ldg(mat_id + (int64_t)k0 * d.plane + scol), m_prev = 0;
  for (int kk = k0; kk <= kend; ++kk) {
    if (leader && kk + NS - 1 <= kend) FDTD_TMA_ISSUE(kk + NS - 1);
    const int st = (kk - k0) % NS;
    mbar_wait(&bars[st], (unsigned)(((kk - k0) / NS) & 1));
    const T* h = Hs + st * 3 * HP;
    const T* e = Es + st * 3 * EP;
    const T hx_c = h[0 * HP + yi * HW + xi], hy_c = h[1 * HP + yi * HW + xi], hz_c = h[2 * HP + yi * HW + xi];
    const T hz_jm = h[2 * HP + (yi - 1) * HW + xi], hx_jm = h[0 * HP + (yi - 1) * HW + xi];
    const T hz_im = h[2 * HP + yi * HW + xi - B], hy_im = h[1 * HP + yi * HW + xi - B];
    const T ex0 = e[0 * EP + ty * BX + tx], ey0 = e[1 * EP + ty * BX + tx], ez0 = e[2 * EP + ty * BX + tx];
    const int m = m_next;                                   // material of plane kk (prefetched)
    if (!UNIFORM && kk + 1 <= kend) m_next = (int)__ldg(mat_id + (int64_t)(kk + 1) * d.plane + scol);
    Coef<T> cx, cy, cz;
    uint8_t ifmk = 0;
    if (UNIFORM) { cx = u0; cy = u0; cz = u0; }
    else { cx = tab->c[m][0]; cy = tab->c[m][1]; cz = tab->c[m][2]; ifmk = tab->ifm[m]; }
    const bool kin = (kk > 0) && (kk < nz);
    T ex = (ax_ij && kin) ? cx.add(ex0, (hz_c - hz_jm) - (hy_c - hy_p)) : (T)0;
    T ey = (ay_ij && kin) ? cy.add(ey0, (hx_c - hx_p) - (hz_c - hz_im)) : (T)0;
    T ez = (az_ij && kk < nz) ? cz.add(ez0, (hy_c - hy_im) - (hx_c - hx_jm)) : (T)0;
    if (!UNIFORM && ifmk && inside) {
      const int64_t s = (int64_t)kk * d.plane + scol;
      if (ifmk & 1) ex = eval_row(R, R.row_of[0][s], b, B, ex0, F0, y, step);
      if (ifmk & 2) ey = eval_row(R, R.row_of[1][s], b, B, ey0, F0, y, step);
      if (ifmk & 4) ez = eval_row(R, R.row_of[2][s], b, B, ez0, F0, y, step);
    }
    T* en = En + (kk % 3) * 3 * EP;
    en[0 * EP + ty * BX + tx] = ex; en[1 * EP + ty * BX + tx] = ey; en[2 * EP + ty * BX + tx] = ez;
    if (own && kk < k1) {
      const int64_t o = (int64_t)kk * sz + col;
      F1.f[0][o] = ex; F1.f[1][o] = ey; F1.f[2][o] = ez;
      if (do_check) bad |= !(finite_small(ex) && finite_small(ey) && finite_small(ez));
    }
    __syncthreads();            // En of plane kk complete; stage st free for reuse after this
    if (kk > k0 && own) {
      const T* e0 = En + ((kk + 2) % 3) * 3 * EP;   // plane kk-1
      const int q = ty * BX + tx;
      const T ey_ip = e0[1 * EP + q + B], ez_ip = e0[2 * EP + q + B];
      const T ex_jp = e0[0 * EP + q + BX], ez_jp = e0[2 * EP + q + BX];
      const int km = kk - 1;
      Coef<T> hx_, hy_, hz_;
      if (UNIFORM) { hx_ = u1; hy_ = u1; hz_ = u1; }
      else { hx_ = tab->c[m_prev][3]; hy_ = tab->c[m_prev][4]; hz_ = tab->c[m_prev][5]; }   // plane kk-1
      const T hx1 = (hx_ij && km < nz) ? hx_.sub(hxk, (ez_jp - ezk) - (ey - eyk)) : hxk;
      const T hy1 = (hy_ij && km < nz) ? hy_.sub(hyk, (ex - exk) - (ez_ip - ezk)) : hyk;
      const T hz1 = (hz_ij && km > 0 && km < nz) ? hz_.sub(hzk, (ey_ip - eyk) - (ex_jp - exk)) : hzk;
      const int64_t o = (int64_t)km * sz + col;
      F1.f[3][o] = hx1; F1.f[4][o] = hy1; F1.f[5][o] = hz1;
      if (do_check) bad |= !(finite_small(hx1) && finite_small(hy1) && finite_small(hz1));
    }
    hx_p = hx_c; hy_p = hy_c;
    hxk = hx_c; hyk = hy_c; hzk = hz_c;
    exk = ex; eyk = ey; ezk = ez;
    m_prev = m;
  }
  if (k1 == nz + 1 && own) {
    const int64_t o = (int64_t)nz * sz + col;
    F1.f[3][o] = hxk; F1.f[4][o] = hyk; F1.f[5][o] = hzk;
  }
  if (bad) atomicMin(bad_step, (unsigned long long)step);
#undef FDTD_TMA_ISSUE
}

// ---------------------------------------------------------------------------
// Batched 3-D stencil (B >= 2 members innermost): the TMA kernel with each
// thread owning W = 16 bytes of members of one cell (float4 / double2), so a
// 32-thread row covers 32*W elements = 32*W/B cells instead of 2 (B = 16,
// W = 4: 8 cells, x overlap 8/7 instead of 2/1).  Same plane march, ring,
// mbarriers, overlapped tiling and arithmetic (per member, in the same order)
// as stencil3d_tma_kernel.
// ---------------------------------------------------------------------------
template <typename T, int W>
struct LV {
  T v[W];
};
template <typename T, int W>
__device__ __forceinline__ LV<T, W> lv_ld(const T* p) {
  LV<T, W> r;
  if constexpr (sizeof(T) * W == 16) {
    using V = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
    const V x = *reinterpret_cast<const V*>(p);
    if constexpr (W == 4) { r.v[0] = x.x; r.v[1] = x.y; r.v[2] = x.z; r.v[3] = x.w; }
    else { r.v[0] = x.x; r.v[1] = x.y; }
  } else {
#pragma unroll
    for (int w = 0; w < W; ++w) r.v[w] = p[w];
  }
  return r;
}
template <typename T, int W>
__device__ __forceinline__ void lv_st(T* p, const LV<T, W>& r) {
  if constexpr (sizeof(T) * W == 16) {
    using V = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
    V x;
    if constexpr (W == 4) { x.x = r.v[0]; x.y = r.v[1]; x.z = r.v[2]; x.w = r.v[3]; }
    else { x.x = r.v[0]; x.y = r.v[1]; }
    *reinterpret_cast<V*>(p) = x;
  } else {
#pragma unroll
    for (int w = 0; w < W; ++w) p[w] = r.v[w];
  }
}

template <typename T, bool UNIFORM, int NS, int W>
__global__ void __launch_bounds__(256, 2)
stencil3d_tma_vec_kernel(const __grid_constant__ TmaSet tm, int HBX, int SX, int outx, Dims d, Fields<T> F0,
                         Fields<T> F1, const uint8_t* __restrict__ mat_id, const Coef<T>* __restrict__ gtab,
                         const uint8_t* __restrict__ gifm, int n_mat, Coef<T> u0, Coef<T> u1, RowsE<T> R,
                         const T* __restrict__ y, int kchunk, const int64_t* __restrict__ d_step,
                         int check_every, unsigned long long* __restrict__ bad_step) {
  using L = LV<T, W>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int BX = blockDim.x * W, BY = blockDim.y, B = d.B;   // BX: elements per tile row
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int HW = HBX, HH = BY + 1;
  const int al = 128 / (int)sizeof(T);
  const int HP = (HW * HH + al - 1) / al * al, EP = (BX * BY + al - 1) / al * al;
  const unsigned base_u = smem_u32(smem_raw);
  unsigned char* smem_al = smem_raw + ((128u - (base_u & 127u)) & 127u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_al);
  T* Hs = reinterpret_cast<T*>(smem_al + 128);
  T* Es = Hs + NS * 3 * HP;
  T* En = Es + NS * 3 * EP;                  // [3][3][BY][BX] (three buffers, see the scalar kernel)
  MatTable<T>* tab = reinterpret_cast<MatTable<T>*>(En + 3 * 3 * EP);
  const bool leader = (tx == 0 && ty == 0);
  if (leader) {
    for (int q = 0; q < NS; ++q) mbar_init(&bars[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (!UNIFORM) {
    for (int m = ty * blockDim.x + tx; m < n_mat; m += blockDim.x * BY) {
      for (int c = 0; c < 6; ++c) tab->c[m][c] = gtab[m * 6 + c];
      tab->ifm[m] = gifm[m];
    }
  }
  __syncthreads();
  const int nx = d.nx, ny = d.ny, nz = d.nz;
  const int outy = BY - 1;
  const int i0 = blockIdx.x * outx, j0 = blockIdx.y * outy;
  const int xe = tx * W;                     // first element of this thread in the tile row
  const int i = i0 + xe / B;
  const int b = xe % B;
  const int j = j0 + ty;
  const int k0 = blockIdx.z * kchunk;
  const int k1 = min(k0 + kchunk, nz + 1);
  const int kend = min(k1, nz);
  const bool inside = (i <= nx) && (j <= ny);
  const bool own = inside && (xe / B < outx) && (ty < outy);
  const int ii = min(i, nx), jj = min(j, ny);
  const int64_t scol = (int64_t)jj * d.px + ii;
  const int64_t col = scol * B + b;
  const int64_t sz = d.plane * B;
  const int xi = xe + SX, yi = ty + 1;
  const bool ax_ij = (i < nx) && (j > 0) && (j < ny);
  const bool ay_ij = (j < ny) && (i > 0) && (i < nx);
  const bool az_ij = (i > 0) && (i < nx) && (j > 0) && (j < ny);
  const bool hx_ij = (i > 0) && (i < nx) && (j < ny);
  const bool hy_ij = (j > 0) && (j < ny) && (i < nx);
  const bool hz_ij = (i < nx) && (j < ny);
  const int64_t step = *d_step;
  const bool do_check = check_every > 0 && (step % check_every) == 0;
  bool bad = false;
  const unsigned stage_bytes = (unsigned)((3 * HW * HH + 3 * BX * BY) * sizeof(T));
#define FDTD_TMA_ISSUE(K)                                                              \
  do {                                                                                 \
    const int st_ = ((K) - k0) % NS;                                                   \
    T* h_ = Hs + st_ * 3 * HP;                                                         \
    T* e_ = Es + st_ * 3 * EP;                                                         \
    mbar_expect_tx(&bars[st_], stage_bytes);                                           \
    tma_load_3d(h_ + 0 * HP, &tm.h[0], i0 * B, j0, (K), &bars[st_]);                   \
    tma_load_3d(h_ + 1 * HP, &tm.h[1], i0 * B, j0, (K), &bars[st_]);                   \
    tma_load_3d(h_ + 2 * HP, &tm.h[2], i0 * B, j0, (K), &bars[st_]);                   \
    tma_load_3d(e_ + 0 * EP, &tm.e[0], i0 * B + SX, j0 + 1, (K), &bars[st_]);          \
    tma_load_3d(e_ + 1 * EP, &tm.e[1], i0 * B + SX, j0 + 1, (K), &bars[st_]);          \
    tma_load_3d(e_ + 2 * EP, &tm.e[2], i0 * B + SX, j0 + 1, (K), &bars[st_]);          \
  } while (0)
  if (leader) {
    for (int q = 0; q < NS - 1; ++q)
      if (k0 + q <= kend) FDTD_TMA_ISSUE(k0 + q);
  }
  L hx_p{}, hy_p{};
  if (inside && k0 > 0) {
    const int64_t o = (int64_t)(k0 - 1) * sz + col;
    hx_p = lv_ld<T, W>(F0.f[3] + o); hy_p = lv_ld<T, W>(F0.f[4] + o);
  }
  L hxk{}, hyk{}, hzk{}, exk{}, eyk{}, ezk{};
  int m_next = UNIFORM ? 0 : (int)__ldg(mat_id + (int64_t)k0 * d.plane + scol), m_prev = 0;
  for (int kk = k0; kk <= kend; ++kk) {
    if (leader && kk + NS - 1 <= kend) FDTD_TMA_ISSUE(kk + NS - 1);
    const int st = (kk - k0) % NS;
    mbar_wait(&bars[st], (unsigned)(((kk - k0) / NS) & 1));
    const T* h = Hs + st * 3 * HP;
    const T* e = Es + st * 3 * EP;
    const L hx_c = lv_ld<T, W>(h + 0 * HP + yi * HW + xi), hy_c = lv_ld<T, W>(h + 1 * HP + yi * HW + xi);
    const L hz_c = lv_ld<T, W>(h + 2 * HP + yi * HW + xi);
    const L hz_jm = lv_ld<T, W>(h + 2 * HP + (yi - 1) * HW + xi), hx_jm = lv_ld<T, W>(h + 0 * HP + (yi - 1) * HW + xi);
    const L hz_im = lv_ld<T, W>(h + 2 * HP + yi * HW + xi - B), hy_im = lv_ld<T, W>(h + 1 * HP + yi * HW + xi - B);
    const L ex0 = lv_ld<T, W>(e + 0 * EP + ty * BX + xe), ey0 = lv_ld<T, W>(e + 1 * EP + ty * BX + xe);
    const L ez0 = lv_ld<T, W>(e + 2 * EP + ty * BX + xe);
    const int m = m_next;
    if (!UNIFORM && kk + 1 <= kend) m_next = (int)__ldg(mat_id + (int64_t)(kk + 1) * d.plane + scol);
    Coef<T> cx, cy, cz;
    uint8_t ifmk = 0;
    if (UNIFORM) { cx = u0; cy = u0; cz = u0; }
    else { cx = tab->c[m][0]; cy = tab->c[m][1]; cz = tab->c[m][2]; ifmk = tab->ifm[m]; }
    const bool kin = (kk > 0) && (kk < nz);
    L ex, ey, ez;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      ex.v[w] = (ax_ij && kin) ? cx.add(ex0.v[w], (hz_c.v[w] - hz_jm.v[w]) - (hy_c.v[w] - hy_p.v[w])) : (T)0;
      ey.v[w] = (ay_ij && kin) ? cy.add(ey0.v[w], (hx_c.v[w] - hx_p.v[w]) - (hz_c.v[w] - hz_im.v[w])) : (T)0;
      ez.v[w] = (az_ij && kk < nz) ? cz.add(ez0.v[w], (hy_c.v[w] - hy_im.v[w]) - (hx_c.v[w] - hx_jm.v[w])) : (T)0;
    }
    if (!UNIFORM && ifmk && inside) {
      const int64_t s = (int64_t)kk * d.plane + scol;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        if (ifmk & 1) ex.v[w] = eval_row(R, R.row_of[0][s], b + w, B, ex0.v[w], F0, y, step);
        if (ifmk & 2) ey.v[w] = eval_row(R, R.row_of[1][s], b + w, B, ey0.v[w], F0, y, step);
        if (ifmk & 4) ez.v[w] = eval_row(R, R.row_of[2][s], b + w, B, ez0.v[w], F0, y, step);
      }
    }
    T* en = En + (kk % 3) * 3 * EP;
    lv_st<T, W>(en + 0 * EP + ty * BX + xe, ex); lv_st<T, W>(en + 1 * EP + ty * BX + xe, ey);
    lv_st<T, W>(en + 2 * EP + ty * BX + xe, ez);
    if (own && kk < k1) {
      const int64_t o = (int64_t)kk * sz + col;
      lv_st<T, W>(F1.f[0] + o, ex); lv_st<T, W>(F1.f[1] + o, ey); lv_st<T, W>(F1.f[2] + o, ez);
      if (do_check)
#pragma unroll
        for (int w = 0; w < W; ++w) bad |= !(finite_small(ex.v[w]) && finite_small(ey.v[w]) && finite_small(ez.v[w]));
    }
    __syncthreads();
    if (kk > k0 && own) {
      const T* e0 = En + ((kk + 2) % 3) * 3 * EP;   // plane kk-1
      const int q = ty * BX + xe;
      const L ey_ip = lv_ld<T, W>(e0 + 1 * EP + q + B), ez_ip = lv_ld<T, W>(e0 + 2 * EP + q + B);
      const L ex_jp = lv_ld<T, W>(e0 + 0 * EP + q + BX), ez_jp = lv_ld<T, W>(e0 + 2 * EP + q + BX);
      const int km = kk - 1;
      Coef<T> hx_, hy_, hz_;
      if (UNIFORM) { hx_ = u1; hy_ = u1; hz_ = u1; }
      else { hx_ = tab->c[m_prev][3]; hy_ = tab->c[m_prev][4]; hz_ = tab->c[m_prev][5]; }
      L hx1, hy1, hz1;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        hx1.v[w] = (hx_ij && km < nz) ? hx_.sub(hxk.v[w], (ez_jp.v[w] - ezk.v[w]) - (ey.v[w] - eyk.v[w])) : hxk.v[w];
        hy1.v[w] = (hy_ij && km < nz) ? hy_.sub(hyk.v[w], (ex.v[w] - exk.v[w]) - (ez_ip.v[w] - ezk.v[w])) : hyk.v[w];
        hz1.v[w] = (hz_ij && km > 0 && km < nz) ? hz_.sub(hzk.v[w], (ey_ip.v[w] - eyk.v[w]) - (ex_jp.v[w] - exk.v[w]))
                                                 : hzk.v[w];
      }
      const int64_t o = (int64_t)km * sz + col;
      lv_st<T, W>(F1.f[3] + o, hx1); lv_st<T, W>(F1.f[4] + o, hy1); lv_st<T, W>(F1.f[5] + o, hz1);
      if (do_check)
#pragma unroll
        for (int w = 0; w < W; ++w) bad |= !(finite_small(hx1.v[w]) && finite_small(hy1.v[w]) && finite_small(hz1.v[w]));
    }
    hx_p = hx_c; hy_p = hy_c;
    hxk = hx_c; hyk = hy_c; hzk = hz_c;
    exk = ex; eyk = ey; ezk = ez;
    m_prev = m;
  }
  if (k1 == nz + 1 && own) {
    const int64_t o = (int64_t)nz * sz + col;
    lv_st<T, W>(F1.f[3] + o, hxk); lv_st<T, W>(F1.f[4] + o, hyk); lv_st<T, W>(F1.f[5] + o, hzk);
  }
  if (bad) atomicMin(bad_step, (unsigned long long)step);
#undef FDTD_TMA_ISSUE
}

// ---------------------------------------------------------------------------
// reduced blocks.  Small blocks ("fused", see fdtd_api.cu): one GEMV with the
// precomposed update matrix M per step,
//   [h~' ; y' ; e~'' ; probe rows] = M [e~ ; h~ ; G] (G columns last),
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
  const uint16_t* Ml;              // fp32 runs: [R][Cp] bf16 low parts, M = M + Ml to ~2^-33 (R14)
  const double* M64;               // fp32 runs: [R][Cp] fp64 copy (the batched GEMM kernel)
  int64_t e_off, h_off, y_off;
  int n_probe_rows;
  const int32_t* probe_id;
  const int32_t* probe_inst;
};

constexpr int kMaxFusedBlocks = 8;
template <typename T>
struct FusedParams {
  // block descriptors live in the kernel parameters (__grid_constant__): the
  // CTA -> (block, first row) map is arithmetic, no dependent global loads
  FusedBlock<T> fb[kMaxFusedBlocks];
  int tile0[kMaxFusedBlocks + 1];   // first tile (CTA / cluster) of each block
  int nfb;
  int n_ctas, B, rows_per_cta;
  int tail_mode;                // 0: probes + step counter here; 1: divergence flag only (split step, §5.6)
  // explicit rows of the NEXT step, evaluated by the thread that finalises their
  // y (reduced_gemm_kernel): no pre-pass launch in steady state
  int fuse_rows;                // 0: off
  int lossy_rows;
  const RowPackI* rp_i;
  const void* rp_r;             // RowPackR<T>
  const int32_t* y_row;         // [y elements / B] explicit row whose y term this is, -1: none
  const int32_t* src_rows;      // explicit rows without a y term (sources off the interface)
  int n_src_rows;
  Fields<T> Fn0;                // next step's old parity (this step's output) ...
  Fields<T> Fn1;                // ... and its new parity (this step's input buffers)
  T* g_next;                    // next step's G (the other parity's buffer)
  const T* wave;
  int64_t n_wave, n_wsrc;
  const T* e_in; T* e_out;      // e~^{n+1} in, e~^{n+2} out
  const T* h_in; T* h_out;      // h~^{n+1/2} in, h~^{n+3/2} out
  T* y;
  const T* G;                   // E_if^{n+1} published by the stencil ([n_if][N] per block)
  const T* red_base[2];         // leapfrog-path e~ / h~ buffers (probe terms 6 / 7)
  Fields<T> F;                  // coarse fields after the step
  Probes<T> pr;
  T* ring;
  int64_t cap;
  const int64_t* d_step;        // this step's counter slot
  int64_t* d_step_next;         // the other parity's slot: <- step + 1
  int check_every;
  unsigned long long* bad_step;
};

template <typename T>
__device__ __forceinline__ int2 fused_tile(const FusedParams<T>& P, int tile) {
  int b = 0;
#pragma unroll 1
  while (b + 1 < P.nfb && tile >= P.tile0[b + 1]) ++b;
  return make_int2(b, (tile - P.tile0[b]) * P.rows_per_cta);
}

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

// four bf16 (the low parts of a compensated fp32 matrix, R14) -> float4
__device__ __forceinline__ float4 bf16x4(uint2 u) {
  return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xffff0000u),
                     __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xffff0000u));
}

// (a + l) . x with a, l, x fp32: exact products summed in fp64, fixed order
// (the compensated fused update of fp32 runs, reading R14)
__device__ __forceinline__ double dot_hilo(const float4& a, const float4& l, const float4& x) {
  double s = (double)a.x * (double)x.x;
  s = fma((double)l.x, (double)x.x, s);
  s = fma((double)a.y, (double)x.y, s);
  s = fma((double)l.y, (double)x.y, s);
  s = fma((double)a.z, (double)x.z, s);
  s = fma((double)l.z, (double)x.z, s);
  s = fma((double)a.w, (double)x.w, s);
  s = fma((double)l.w, (double)x.w, s);
  return s;
}
__device__ __forceinline__ double dot_hilo_reg(const float4& a, const float4& l, const float* x) {
  return dot_hilo(a, l, make_float4(x[0], x[1], x[2], x[3]));
}

template <typename T>
__device__ __forceinline__ T vdot_reg(const typename Vec<T>::type& a, const T* x);
template <>
__device__ __forceinline__ float vdot_reg<float>(const float4& a, const float* x) {
  return a.x * x[0] + a.y * x[1] + a.z * x[2] + a.w * x[3];
}
template <>
__device__ __forceinline__ double vdot_reg<double>(const double2& a, const double* x) {
  return a.x * x[0] + a.y * x[1];
}
// load a word of CTA `rank`'s shared memory (same offset) through the cluster
template <typename T>
__device__ __forceinline__ T dsmem_load(unsigned local_addr, unsigned rank);
template <>
__device__ __forceinline__ float dsmem_load<float>(unsigned local_addr, unsigned rank) {
  unsigned remote;
  float v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(remote) : "r"(local_addr), "r"(rank));
  asm volatile("ld.shared::cluster.f32 %0, [%1];\n" : "=f"(v) : "r"(remote) : "memory");
  return v;
}
template <>
__device__ __forceinline__ double dsmem_load<double>(unsigned local_addr, unsigned rank) {
  unsigned remote;
  double v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(remote) : "r"(local_addr), "r"(rank));
  asm volatile("ld.shared::cluster.f64 %0, [%1];\n" : "=d"(v) : "r"(remote) : "memory");
  return v;
}

// coarse probes, leapfrog-path reduced probes, divergence flag and the device
// step counter (advanced by the last CTA to finish) -- shared by both fused
// reduced kernels
template <typename T>
__device__ __forceinline__ void fused_tail(const FusedParams<T>& P, int64_t step, bool bad) {
  const int B = P.B;
  if (P.tail_mode == 1) {               // probes and counter run in the tail launch after the stencil
    if (bad) atomicMin(P.bad_step, (unsigned long long)step);
    return;
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
  // the step counter lives in two slots by step parity: this kernel reads slot
  // p and publishes step + 1 in slot p^1, which only the next step reads (no
  // grid-wide completion counter needed)
  if (blockIdx.x == 0 && threadIdx.x == 0) *P.d_step_next = step + 1;
}

template <typename T, int NB>
__global__ void __launch_bounds__(256)
reduced_fused_kernel(const __grid_constant__ FusedParams<T> P) {
  using V = typename Vec<T>::type;
  constexpr int VN = Vec<T>::n;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* X = reinterpret_cast<T*>(smem_raw);
  // launched as a programmatic dependent of the stencil: wait for its results
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  const int64_t step = *P.d_step;
  const bool check = P.check_every > 0 && (step % P.check_every) == 0;
  bool bad = false;
  const int B = P.B;
  if ((int)blockIdx.x < P.n_ctas) {
    const int2 ct = fused_tile(P, (int)blockIdx.x);
    const FusedBlock<T>& FB = P.fb[ct.x];
    const int C = FB.C, Cp = FB.Cp, N = FB.N, qe = FB.qe, qh = FB.qh, ni = FB.n_if;
    // stage X = [e~ ; h~ ; G ; 0-padding] as [N][Cp]
    for (int t = threadIdx.x; t < qe * N; t += blockDim.x) X[(t % N) * Cp + t / N] = P.e_in[FB.e_off + t];
    for (int t = threadIdx.x; t < qh * N; t += blockDim.x) X[(t % N) * Cp + qe + t / N] = P.h_in[FB.h_off + t];
    for (int t = threadIdx.x; t < ni * N; t += blockDim.x) X[(t % N) * Cp + qe + qh + t / N] = P.G[FB.y_off + t];
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
      if constexpr (sizeof(T) == 4) {
        // compensated matrix, fp64 accumulation of exact fp32 products,
        // rounded once (reading R14)
        const uint2* al = reinterpret_cast<const uint2*>(FB.Ml + (int64_t)r * Cp);
        double acd[NB];
#pragma unroll
        for (int n = 0; n < NB; ++n) acd[n] = 0.0;
#pragma unroll 4
        for (int c = lane; c < nv; c += 32) {
          const float4 av = reinterpret_cast<const float4*>(a)[c];
          const float4 lv = bf16x4(al[c]);
#pragma unroll
          for (int n = 0; n < NB; ++n)
            if (n < N) acd[n] += dot_hilo(av, lv, reinterpret_cast<const float4*>(X + n * Cp)[c]);
        }
#pragma unroll
        for (int n = 0; n < NB; ++n) {
          double v = acd[n];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          acc[n] = (T)v;
        }
      } else {
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
  fused_tail(P, step, bad);
}

// ---------------------------------------------------------------------------
// Batched reduced blocks (N = instances x batch >= 4 columns): the same fused
// update [h~' ; y' ; e~'' ; probe rows] = M [e~ ; h~ ; G] as a register-tiled
// SIMT GEMM.  A cluster of KS CTAs shares one tile of TR rows: CTA `rank`
// contracts the K-slice [rank*Cp/KS, (rank+1)*Cp/KS) -- its slice of X staged
// in shared memory as [k][NP] (the natural [q][N] layout of the states: a
// straight copy, lanes read consecutive words) -- and the KS partial tiles are
// summed in a fixed order through distributed shared memory (deterministic).
// Lane = (row group, column n): M is read with 16-byte broadcast loads (every
// lane of a row group reads the same row), X with conflict-free 4-byte loads.
// ---------------------------------------------------------------------------
template <typename T, int NP, int RPW, int KS>
__global__ void __cluster_dims__(KS, 1, 1) __launch_bounds__(256)
reduced_gemm_kernel(const __grid_constant__ FusedParams<T> P) {
  // fp64 arithmetic for both precisions: fp32 runs read an fp64 copy of M
  // (M64, composed in fp64 and never rounded to fp32) and stage their fp32
  // states as fp64, so the update is rounded once (reading R14)
  constexpr int GPW = 32 / NP;                 // row groups per warp
  constexpr int TR = 8 * GPW * RPW;            // rows per tile
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* Ps = reinterpret_cast<double*>(smem_raw);   // [TR][NP] partial tile
  T* Xs = reinterpret_cast<T*>(Ps + TR * NP);         // [kc][NP] slice of [e~ ; h~ ; G] (run precision)
  const int64_t step = *P.d_step;
  const bool check = P.check_every > 0 && (step % P.check_every) == 0;
  bool bad = false;
  const int B = P.B;
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
  const int tile = blockIdx.x / KS;
  const bool active = tile < P.n_ctas;
  int2 ct = make_int2(0, 0);
  if (active) {
    ct = fused_tile(P, tile);
    const FusedBlock<T>& FB = P.fb[ct.x];
    const int N = FB.N, C = FB.C, qe = FB.qe, qh = FB.qh;
    const int kc = FB.Cp / KS, k_lo = (int)rank * kc;
    double* Ms = reinterpret_cast<double*>(Xs + kc * NP);   // [TR][kc + 2] slice of M (padded pitch)
    const int mp = kc + 2;
    const double* Msrc = (sizeof(T) == 4) ? FB.M64 : reinterpret_cast<const double*>(FB.M);
    // M slice: 16-byte cp.async (two doubles), all in flight at once
    for (int t = threadIdx.x; t < TR * (kc / 2); t += blockDim.x) {
      const int u = t / (kc / 2), v = t % (kc / 2);
      cp_async16(Ms + u * mp + v * 2, Msrc + (int64_t)(ct.y + u) * FB.Cp + k_lo + v * 2, true);
    }
    cp_async_commit();
    // M does not depend on the step; the states and G do: launched as a
    // programmatic dependent of the stencil, wait for it here
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    constexpr int VN = Vec<T>::n;
    if (N == NP && N % VN == 0) {
      // X slice, straight 16-byte copies (every k-row is N contiguous words)
      for (int t = threadIdx.x; t < kc * (NP / VN); t += blockDim.x) {
        const int kk = t / (NP / VN), n = (t % (NP / VN)) * VN, k = k_lo + kk;
        const T* src = P.e_in;                 // any valid address when zero-filled
        if (k < qe) src = P.e_in + FB.e_off + (int64_t)k * N + n;
        else if (k < qe + qh) src = P.h_in + FB.h_off + (int64_t)(k - qe) * N + n;
        else if (k < C) src = P.G + FB.y_off + (int64_t)(k - qe - qh) * N + n;
        cp_async16(Xs + kk * NP + n, src, k < C);
      }
    } else {
      for (int t0 = threadIdx.x; t0 < kc * NP; t0 += 8 * 256) {
        T v[8];
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          const int t = t0 + w * 256, kk = t / NP, n = t % NP, k = k_lo + kk;
          v[w] = 0;
          if (t < kc * NP && n < N && k < C) {
            if (k < qe) v[w] = P.e_in[FB.e_off + (int64_t)k * N + n];
            else if (k < qe + qh) v[w] = P.h_in[FB.h_off + (int64_t)(k - qe) * N + n];
            else v[w] = P.G[FB.y_off + (int64_t)(k - qe - qh) * N + n];
          }
        }
#pragma unroll
        for (int w = 0; w < 8; ++w)
          if (t0 + w * 256 < kc * NP) Xs[t0 + w * 256] = v[w];
      }
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int n = lane % NP, g = lane / NP;
    const int rl0 = (warp * GPW + g) * RPW;
    double acc[RPW];
#pragma unroll
    for (int u = 0; u < RPW; ++u) acc[u] = 0.0;
    const int nv = kc / 2;
#pragma unroll 4
    for (int kv = 0; kv < nv; ++kv) {
      const double x0 = (double)Xs[(2 * kv) * NP + n], x1 = (double)Xs[(2 * kv + 1) * NP + n];
#pragma unroll
      for (int u = 0; u < RPW; ++u) {
        const double2 m = *reinterpret_cast<const double2*>(Ms + (rl0 + u) * mp + 2 * kv);
        acc[u] = fma(m.x, x0, acc[u]);
        acc[u] = fma(m.y, x1, acc[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < RPW; ++u) Ps[(rl0 + u) * NP + n] = acc[u];
  }
  // all partial tiles of the cluster written
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  if (active) {
    const FusedBlock<T>& FB = P.fb[ct.x];
    const int N = FB.N, qe = FB.qe, qh = FB.qh, ni = FB.n_if;
    constexpr int RPR = TR / KS;               // rows reduced by this rank
    const unsigned ps_local = smem_u32(Ps);
    for (int t = threadIdx.x; t < RPR * NP; t += blockDim.x) {
      const int rl = (int)rank * RPR + t / NP, n = t % NP;
      const int r = ct.y + rl;
      double vs = 0;
#pragma unroll
      for (int q = 0; q < KS; ++q) vs += dsmem_load<double>(ps_local + (unsigned)((rl * NP + n) * sizeof(double)), (unsigned)q);
      const T v = (T)vs;
      if (r >= FB.R || n >= N) continue;
      if (r < qh) P.h_out[FB.h_off + (int64_t)r * N + n] = v;
      else if (r < qh + ni) {
        const int64_t yi = FB.y_off + (int64_t)(r - qh) * N + n;
        P.y[yi] = v;
        if (P.fuse_rows) {
          // this y element is final: its explicit row of the next step (the
          // stencil of this step has finished, so H^{n+1} and E^{n+1} are final;
          // the next step's new parity and G buffers are free)
          const int er = P.y_row[yi / B];
          if (er >= 0)
            packed_row_eval<T>(er, (int)(yi % B), v, P.rp_i, reinterpret_cast<const RowPackR<T>*>(P.rp_r), B, P.Fn0,
                               P.Fn1, P.g_next, P.wave, P.n_wave, P.n_wsrc, step + 1, P.lossy_rows);
        }
      } else if (r < qh + ni + qe) P.e_out[FB.e_off + (int64_t)(r - qh - ni) * N + n] = v;
      else {
        const int q = r - qh - ni - qe;
        const int p = FB.probe_id[q], in = FB.probe_inst[q];
        if (n >= in * B && n < in * B + B)
          P.ring[(step % P.cap) * (int64_t)P.pr.n_probe * B + (int64_t)p * B + (n - in * B)] = v;
      }
      if (check && !finite_small((double)v)) bad = true;
    }
  }
  if (P.fuse_rows) {
    // explicit rows without a y term (sources off the interface), spread over the grid
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)P.n_src_rows * P.B;
         t += (int64_t)gridDim.x * blockDim.x)
      packed_row_eval<T>(P.src_rows[t / P.B], (int)(t % P.B), (T)0, P.rp_i, reinterpret_cast<const RowPackR<T>*>(P.rp_r),
                         P.B, P.Fn0, P.Fn1, P.g_next, P.wave, P.n_wave, P.n_wsrc, step + 1, P.lossy_rows);
  }
  // no CTA leaves (releasing its shared memory) before every rank has read it
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  fused_tail(P, step, bad);
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

// ---------------------------------------------------------------------------
// leap-frog path for large reduced blocks (config 4: S_E = 65,024 x 1,024,
// N = 16 columns).  Two streaming kernels, HBM-bound on the matrix:
//  * rowblock_gemv: out[r][n] = (acc ? out : 0) + alpha g[r] sum_c A[r][c] X[c][n]
//    persistent CTAs; X staged once per CTA in shared memory as [N][K]; A rows
//    streamed with 16-byte loads (requires K % (32 * VEC) == 0 -> padded rows)
//  * colsum_gemv: out[c][n] += sum_r A[r][c] X[r][n] over a contiguous row chunk
//    per CTA (A row-major is read once, coalesced); partial sums in registers,
//    then one atomicAdd per (c, n) per CTA.
// ---------------------------------------------------------------------------
// (products and sums in fp64 for both precisions, one rounding of the output:
// the leap-frog increments are small differences of large sums, reading R14;
// OT = double keeps an intermediate sum unrounded)
template <typename T, int NB, typename OT = T>
__global__ void __launch_bounds__(256)
rowblock_gemv_kernel(int rows, int K, int Kp, int N, const T* __restrict__ A, const T* __restrict__ X,
                     OT* __restrict__ out, const T* __restrict__ g, T alpha, bool accumulate,
                     const int64_t* __restrict__ d_step, int check_every, unsigned long long* bad_step) {
  using V = typename Vec<T>::type;
  constexpr int VN = Vec<T>::n;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Xs = reinterpret_cast<T*>(smem_raw);                   // [N][Kp]
  for (int t = threadIdx.x; t < Kp * N; t += blockDim.x) {
    const int n = t / Kp, c = t % Kp;
    Xs[t] = (c < K) ? X[(int64_t)c * N + n] : (T)0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const bool check = check_every > 0 && (*d_step % check_every) == 0;
  bool bad = false;
  const int nv = Kp / VN;
  for (int r = w0; r < rows; r += nw) {
    double acc[NB];
#pragma unroll
    for (int n = 0; n < NB; ++n) acc[n] = 0;
    const V* a = reinterpret_cast<const V*>(A + (int64_t)r * Kp);
#pragma unroll 4
    for (int c = lane; c < nv; c += 32) {
      const V av = a[c];
      const T* ap = reinterpret_cast<const T*>(&av);
#pragma unroll
      for (int n = 0; n < NB; ++n)
        if (n < N) {
          const V xv = reinterpret_cast<const V*>(Xs + n * Kp)[c];
          const T* xp = reinterpret_cast<const T*>(&xv);
#pragma unroll
          for (int j = 0; j < VN; ++j) acc[n] = fma((double)ap[j], (double)xp[j], acc[n]);
        }
    }
#pragma unroll
    for (int n = 0; n < NB; ++n) {
      double v = acc[n];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      acc[n] = v;
    }
    if (lane < N) {
      double v = 0;
#pragma unroll
      for (int n = 0; n < NB; ++n)
        if (n == lane) v = acc[n];
      const double gr = g ? (double)g[r] : 1.0;
      OT* o = out + (int64_t)r * N + lane;
      const OT res = (OT)((accumulate ? (double)*o : 0.0) + (double)alpha * gr * v);
      *o = res;
      if (check && !finite_small((double)res)) bad = true;
    }
  }
  if (bad) atomicMin(bad_step, (unsigned long long)*d_step);
}

template <typename T, int NB, int CPT>
__global__ void __launch_bounds__(256)
colsum_gemv_kernel(int rows, int cols, int Kp, int N, const T* __restrict__ A, const T* __restrict__ X,
                   double* __restrict__ out) {
  // thread t owns columns c = c0 + t + 256 * u (u < CPT), c0 = 256 * CPT * blockIdx.y;
  // rows [r0, r1) of this CTA; fp64 products and sums (reading R14)
  const int c0 = 256 * CPT * blockIdx.y;
  const int chunk = (rows + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * chunk, r1 = min(rows, r0 + chunk);
  double acc[CPT][NB];
#pragma unroll
  for (int u = 0; u < CPT; ++u)
#pragma unroll
    for (int n = 0; n < NB; ++n) acc[u][n] = 0;
  for (int r = r0; r < r1; ++r) {
    double xv[NB];
#pragma unroll
    for (int n = 0; n < NB; ++n) xv[n] = (n < N) ? (double)X[(int64_t)r * N + n] : 0.0;
    const T* a = A + (int64_t)r * Kp;
#pragma unroll
    for (int u = 0; u < CPT; ++u) {
      const int c = c0 + threadIdx.x + 256 * u;
      const double av = (c < cols) ? (double)a[c] : 0.0;
#pragma unroll
      for (int n = 0; n < NB; ++n) acc[u][n] = fma(av, xv[n], acc[u][n]);
    }
  }
#pragma unroll
  for (int u = 0; u < CPT; ++u) {
    const int c = c0 + threadIdx.x + 256 * u;
    if (c >= cols) continue;
#pragma unroll
    for (int n = 0; n < NB; ++n)
      if (n < N) atomicAdd(out + (int64_t)c * N + n, acc[u][n]);
  }
}

// h~ += G_h * T   (T = K~'^T e~ + S_E^T G accumulated by the two kernels above)
template <typename T>
__global__ void axpy_diag_kernel(int rows, int N, const T* __restrict__ g, const double* __restrict__ Tv,
                                 T* __restrict__ h) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= rows * N) return;
  h[t] = (T)fma((double)g[t / N], Tv[t], (double)h[t]);
}

// ---------------------------------------------------------------------------
// Leap-frog path, fp32 tall-skinny GEMMs (config 4: S_E 65,024 x 1,024, N = 16).
// Register-tiled SIMT: every thread owns a 4 x 4 (rows x columns) tile of the
// output; operands staged in shared memory by 16-byte cp.async in a 3-stage
// ring; inner step = 8 LDS.128 for 64 FMA.  HBM-bound on A (each element read
// once per product), FMA work 2 R K N per product.
//
// gemm_nn: out[r][n] = (acc ? out[r][n] : 0) + alpha g[r] sum_k A[r][k] X[k][n]
//   A row-major with pitch Kp (multiple of 32), X [K][N] (N = 4 NQ) staged once
//   per CTA; each CTA owns a contiguous, balanced range of rows.
// ---------------------------------------------------------------------------
template <int NQ>
__global__ void __launch_bounds__(256, 1)
gemm_nn_f32_kernel(int rows, int K, int Kp, const float* __restrict__ A, const float* __restrict__ X,
                   float* __restrict__ out, const float* __restrict__ g, float alpha, bool accumulate,
                   const int64_t* __restrict__ d_step, int check_every, unsigned long long* bad_step) {
  constexpr int N = 4 * NQ;
  constexpr int RQ = 256 / NQ;                 // row quads per tile
  constexpr int TR = 4 * RQ;                   // rows per tile
  constexpr int KC = NQ >= 4 ? 32 : 16, KCP = KC + 4, NS = 3;
  extern __shared__ __align__(16) float smf[];
  float* Xs = smf;                             // [Kp][N]
  float* As = Xs + (size_t)Kp * N;             // [NS][TR][KCP]
  const int tid = threadIdx.x;
  const int cq = tid % NQ, rq = tid / NQ;
  for (int t = tid; t < Kp * NQ; t += 256) {
    const int k = t / NQ, c = (t % NQ) * 4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (k < K) v = *reinterpret_cast<const float4*>(X + (int64_t)k * N + c);
    *reinterpret_cast<float4*>(Xs + (int64_t)k * N + c) = v;
  }
  const int r_begin = (int)((int64_t)rows * blockIdx.x / gridDim.x);
  const int r_end = (int)((int64_t)rows * (blockIdx.x + 1) / gridDim.x);
  const int nkc = (K + KC - 1) / KC;
  const int ntile = (r_end - r_begin + TR - 1) / TR;
  const int total = ntile * nkc;
  const bool check = check_every > 0 && (*d_step % check_every) == 0;
  bool bad = false;
  auto issue = [&](int it) {
    if (it < total) {
      const int tile = it / nkc, kc = it % nkc;
      const int r0 = r_begin + tile * TR, k0 = kc * KC;
      float* dst = As + (size_t)(it % NS) * TR * KCP;
      for (int q = tid; q < TR * (KC / 4); q += 256) {
        const int rr = q / (KC / 4), c4 = (q % (KC / 4)) * 4;
        const int r = r0 + rr;
        const bool ok = r < r_end && k0 + c4 < Kp;
        cp_async16(dst + rr * KCP + c4, A + (int64_t)(ok ? r : r_begin) * Kp + (ok ? k0 + c4 : 0), ok);
      }
    }
    cp_async_commit();
  };
  issue(0);
  issue(1);
  float acc[4][4];
  for (int it = 0; it < total; ++it) {
    const int tile = it / nkc, kc = it % nkc;
    if (kc == 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[i][c] = 0.f;
    }
    issue(it + 2);
    cp_async_wait<2>();
    __syncthreads();
    const float* a = As + (size_t)(it % NS) * TR * KCP + (rq * 4) * KCP;
    const float* x = Xs + (int64_t)(kc * KC) * N + cq * 4;
#pragma unroll
    for (int kk = 0; kk < KC; kk += 4) {
      float4 a4[4], x4[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a4[i] = *reinterpret_cast<const float4*>(a + i * KCP + kk);
#pragma unroll
      for (int j = 0; j < 4; ++j) x4[j] = *reinterpret_cast<const float4*>(x + (kk + j) * N);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float av[4] = {a4[i].x, a4[i].y, a4[i].z, a4[i].w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[i][0] += av[j] * x4[j].x;
          acc[i][1] += av[j] * x4[j].y;
          acc[i][2] += av[j] * x4[j].z;
          acc[i][3] += av[j] * x4[j].w;
        }
      }
    }
    if (kc == nkc - 1) {
      const int r0 = r_begin + tile * TR + rq * 4;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = r0 + i;
        if (r >= r_end) continue;
        const float gr = g ? g[r] : 1.f;
        float4* o = reinterpret_cast<float4*>(out + (int64_t)r * N + cq * 4);
        float4 v = accumulate ? *o : make_float4(0.f, 0.f, 0.f, 0.f);
        v.x += alpha * gr * acc[i][0]; v.y += alpha * gr * acc[i][1];
        v.z += alpha * gr * acc[i][2]; v.w += alpha * gr * acc[i][3];
        *o = v;
        if (check) bad |= !(finite_small(v.x) && finite_small(v.y) && finite_small(v.z) && finite_small(v.w));
      }
    }
    __syncthreads();                           // stage it % NS is refilled by issue(it + 3)
  }
  cp_async_wait<0>();
  if (bad) atomicMin(bad_step, (unsigned long long)*d_step);
}

// gemm_tn partial: part[s][c][n] = sum_{r in split s} A[r][c] G[r][n]
//   grid (column tiles of TC = 4 * 256 / NQ columns, splits); the splits are
//   summed in a fixed order by reduce_axpy_f32_kernel (deterministic).
template <int NQ>
__global__ void __launch_bounds__(256, 2)
gemm_tn_f32_partial_kernel(int rows, int cols, int Kp, const float* __restrict__ A, const float* __restrict__ G,
                           double* __restrict__ part) {
  constexpr int N = 4 * NQ;
  constexpr int CQ = 256 / NQ;                 // column quads per tile
  constexpr int TC = 4 * CQ;
  constexpr int RC = 16, NS = 3;
  extern __shared__ __align__(16) float smf[];
  float* As = smf;                             // [NS][RC][TC]
  float* Gs = As + NS * RC * TC;               // [NS][RC][N]
  double* Ad = reinterpret_cast<double*>(Gs + NS * RC * N);   // the current chunk in fp64: [RC][TC]
  double* Gd = Ad + RC * TC;                                   // [RC][N]
  const int tid = threadIdx.x;
  const int nq = tid % NQ, cq = tid / NQ;
  const int c0 = blockIdx.x * TC;
  const int r_begin = (int)((int64_t)rows * blockIdx.y / gridDim.y);
  const int r_end = (int)((int64_t)rows * (blockIdx.y + 1) / gridDim.y);
  const int nch = (r_end - r_begin + RC - 1) / RC;
  auto issue = [&](int ch) {
    if (ch < nch) {
      const int r0 = r_begin + ch * RC;
      float* da = As + (size_t)(ch % NS) * RC * TC;
      float* dg = Gs + (size_t)(ch % NS) * RC * N;
      for (int q = tid; q < RC * (TC / 4); q += 256) {
        const int rr = q / (TC / 4), c4 = (q % (TC / 4)) * 4;
        const int r = r0 + rr;
        const bool ok = r < r_end && c0 + c4 < Kp;
        cp_async16(da + rr * TC + c4, A + (int64_t)(ok ? r : r_begin) * Kp + (ok ? c0 + c4 : 0), ok);
      }
      for (int q = tid; q < RC * NQ; q += 256) {
        const int rr = q / NQ, n4 = (q % NQ) * 4;
        const int r = r0 + rr;
        const bool ok = r < r_end;
        cp_async16(dg + rr * N + n4, G + (int64_t)(ok ? r : r_begin) * N + n4, ok);
      }
    }
    cp_async_commit();
  };
  issue(0);
  issue(1);
  // fp64 accumulation of the exact fp32 products (reading R14): the leap-frog
  // sums K~'^T e~ + S_E^T G cancel to a small h~ increment, so fp32 partial
  // sums alone lose ~1e-4 of it (measured, R14)
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[i][c] = 0.0;
  for (int ch = 0; ch < nch; ++ch) {
    issue(ch + 2);
    cp_async_wait<2>();
    __syncthreads();
    {
      // convert the chunk to fp64 once (each element once, not once per
      // thread that reads it)
      const float* a = As + (size_t)(ch % NS) * RC * TC;
      const float* gg = Gs + (size_t)(ch % NS) * RC * N;
      for (int q = tid; q < RC * TC / 4; q += 256) {
        const float4 v = reinterpret_cast<const float4*>(a)[q];
        reinterpret_cast<double2*>(Ad)[2 * q] = make_double2(v.x, v.y);
        reinterpret_cast<double2*>(Ad)[2 * q + 1] = make_double2(v.z, v.w);
      }
      for (int q = tid; q < RC * N; q += 256) Gd[q] = (double)gg[q];
    }
    __syncthreads();
    const double* a = Ad + cq * 4;
    const double* gg = Gd + nq * 4;
#pragma unroll 4
    for (int rr = 0; rr < RC; ++rr) {
      const double2 a01 = *reinterpret_cast<const double2*>(a + rr * TC);
      const double2 a23 = *reinterpret_cast<const double2*>(a + rr * TC + 2);
      const double2 g01 = *reinterpret_cast<const double2*>(gg + rr * N);
      const double2 g23 = *reinterpret_cast<const double2*>(gg + rr * N + 2);
      const double av[4] = {a01.x, a01.y, a23.x, a23.y};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[i][0] = fma(av[i], g01.x, acc[i][0]); acc[i][1] = fma(av[i], g01.y, acc[i][1]);
        acc[i][2] = fma(av[i], g23.x, acc[i][2]); acc[i][3] = fma(av[i], g23.y, acc[i][3]);
      }
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int c = c0 + cq * 4 + i;
    if (c >= cols) continue;
    double2* o = reinterpret_cast<double2*>(part + ((int64_t)blockIdx.y * cols + c) * N + nq * 4);
    o[0] = make_double2(acc[i][0], acc[i][1]);
    o[1] = make_double2(acc[i][2], acc[i][3]);
  }
}

// gemm_tn partial for N = 16 members and long contractions (config 4's S_E^T G:
// 65,024 rows): the same product as gemm_tn_f32_partial_kernel<4> with an
// 8 column x 8 member register tile per thread.  The 4 x 4 tile of the general
// kernel was bound by shared-memory traffic (ncu: fp64 pipe 38 % active, top
// stalls short_scoreboard / mio_throttle: 4 shared loads per 16 DFMA plus the
// fp32 -> fp64 conversion pass); here it is 8 loads per 64 DFMA.  One CTA per SM
// covers up to 1,024 columns: chunks of WRC = 8 rows, cp.async 3-stage ring of
// the fp32 chunk, converted once to fp64 in shared memory, fp64 accumulation of
// the exact products (R14).  Thread (cq, nq): columns {256 j + 2 cq, 256 j + 2 cq
// + 1 : j = 0..3} (so a warp's 16-byte loads are contiguous: no bank conflicts),
// members nq * 8 .. nq * 8 + 7.
constexpr int WRC = 8, WTC = 1024, WNS = 3;
constexpr int gemm_tn_wide_smem() {
  return WNS * WRC * WTC * 4 + WNS * WRC * 16 * 4 + WRC * WTC * 8 + WRC * 16 * 8;
}
// NG member groups per column octet: NG = 2 -> 8 members per thread, 256 threads; NG = 4 -> 4 members per
// thread, 512 threads (twice the warps to hide the shared-memory and DFMA latencies)
template <int NG>
__global__ void __launch_bounds__(128 * NG, 1)
gemm_tn_f32_wide_kernel(int rows, int cols, int Kp, const float* __restrict__ A, const float* __restrict__ G,
                        double* __restrict__ part) {
  constexpr int N = 16, NT = 128 * NG, MN = N / NG;      // threads, members per thread
  extern __shared__ __align__(16) float smw[];
  float* As = smw;                                   // [WNS][WRC][WTC]
  float* Gs = As + WNS * WRC * WTC;                  // [WNS][WRC][N]
  double* Ad = reinterpret_cast<double*>(Gs + WNS * WRC * N);   // [WRC][WTC]
  double* Gd = Ad + WRC * WTC;                       // [WRC][N]
  const int tid = threadIdx.x;
  const int nq = tid % NG, cq = tid / NG;
  const int c0 = blockIdx.x * WTC;
  const int r_begin = (int)((int64_t)rows * blockIdx.y / gridDim.y);
  const int r_end = (int)((int64_t)rows * (blockIdx.y + 1) / gridDim.y);
  const int nch = (r_end - r_begin + WRC - 1) / WRC;
  auto issue = [&](int ch) {
    if (ch < nch) {
      const int r0 = r_begin + ch * WRC;
      float* da = As + (size_t)(ch % WNS) * WRC * WTC;
      float* dg = Gs + (size_t)(ch % WNS) * WRC * N;
      for (int q = tid; q < WRC * (WTC / 4); q += NT) {
        const int rr = q / (WTC / 4), c4 = (q % (WTC / 4)) * 4;
        const int r = r0 + rr;
        const bool ok = r < r_end && c0 + c4 < Kp;
        cp_async16(da + rr * WTC + c4, A + (int64_t)(ok ? r : r_begin) * Kp + (ok ? c0 + c4 : 0), ok);
      }
      if (tid < WRC * (N / 4)) {
        const int rr = tid / (N / 4), n4 = (tid % (N / 4)) * 4;
        const int r = r0 + rr;
        const bool ok = r < r_end;
        cp_async16(dg + rr * N + n4, G + (int64_t)(ok ? r : r_begin) * N + n4, ok);
      }
    }
    cp_async_commit();
  };
  issue(0);
  issue(1);
  double acc[8][MN];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int c = 0; c < MN; ++c) acc[i][c] = 0.0;
  for (int ch = 0; ch < nch; ++ch) {
    issue(ch + 2);
    cp_async_wait<2>();
    __syncthreads();
    {
      const float2* a2 = reinterpret_cast<const float2*>(As + (size_t)(ch % WNS) * WRC * WTC);
      double2* d2 = reinterpret_cast<double2*>(Ad);
      for (int q = tid; q < WRC * WTC / 2; q += NT) {
        const float2 v = a2[q];
        d2[q] = make_double2((double)v.x, (double)v.y);
      }
      const float* gg = Gs + (size_t)(ch % WNS) * WRC * N;
      if (tid < WRC * N) Gd[tid] = (double)gg[tid];
    }
    __syncthreads();
    const double* a = Ad + cq * 2;
    const double* gq = Gd + nq * MN;
#pragma unroll 2
    for (int rr = 0; rr < WRC; ++rr) {
      double av[8], gv[MN];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double2 t = *reinterpret_cast<const double2*>(a + rr * WTC + j * 256);
        av[2 * j] = t.x; av[2 * j + 1] = t.y;
      }
#pragma unroll
      for (int j = 0; j < MN / 2; ++j) {
        const double2 t = *reinterpret_cast<const double2*>(gq + rr * N + 2 * j);
        gv[2 * j] = t.x; gv[2 * j + 1] = t.y;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int c = 0; c < MN; ++c) acc[i][c] = fma(av[i], gv[c], acc[i][c]);
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int c = c0 + (i >> 1) * 256 + cq * 2 + (i & 1);
    if (c >= cols) continue;
    double2* o = reinterpret_cast<double2*>(part + ((int64_t)blockIdx.y * cols + c) * N + nq * MN);
#pragma unroll
    for (int j = 0; j < MN / 2; ++j) o[j] = make_double2(acc[i][2 * j], acc[i][2 * j + 1]);
  }
}

// h[c][n] += g[c] (T[c][n] + sum_s part[s][c][n])   (splits in order; T optional)
// xs (optional, N = 16): the new h~ split for the tensor-core GEMM of
// tc_gemm.cuh -- per 32-row chunk of h~, [hi | lo] tiles of [16 n][32 k] in
// the 128-byte swizzled K-major layout, so one bulk copy per chunk lands them
// 256 threads = 32 outputs x 8 split groups: each thread sums a contiguous
// range of the splits, then the 8 group sums of an output are added in group
// order (fixed order, deterministic; 8x the memory-level parallelism of one
// thread per output walking all splits)
static __global__ void __launch_bounds__(256) reduce_axpy_f32_kernel(int cols, int N, int splits, const double* __restrict__ part,
                                       const float* __restrict__ Tv, const float* __restrict__ gh,
                                       float* __restrict__ h, float* __restrict__ xs) {
  __shared__ double gs[8][32];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int t = blockIdx.x * 32 + lane;
  const int s_lo = (int)((int64_t)splits * grp / 8), s_hi = (int)((int64_t)splits * (grp + 1) / 8);
  double acc = 0.0;
  if (t < cols * N) {
#pragma unroll 4
    for (int s2 = s_lo; s2 < s_hi; ++s2) acc += part[(int64_t)s2 * cols * N + t];
  }
  gs[grp][lane] = acc;
  __syncthreads();
  if (grp != 0 || t >= cols * N) return;
  double v = Tv ? (double)Tv[t] : 0.0;
#pragma unroll
  for (int g2 = 0; g2 < 8; ++g2) v += gs[g2][lane];
  // fp64 partials, one rounding of the new state (R14)
  const float hn = (float)fma((double)gh[t / N], v, (double)h[t]);
  h[t] = hn;
  if (xs) {
    const int k = t / N, n = t % N, ch = k >> 5, kk = k & 31;
    const int o = n * 32 + ((((kk >> 2) ^ (n & 7)) & 7) << 2) + (kk & 3);   // swizzled element offset
    const float hi = __uint_as_float(__float_as_uint(hn) & 0xFFFFE000u);
    xs[(int64_t)ch * 1024 + o] = hi;
    xs[(int64_t)ch * 1024 + 512 + o] = hn - hi;
  }
}

// fdtd_set_state for a coarse component: in [B][S] fp64 (storage order) ->
// the padded device layout ((k (ny+1) + j) px + i) B + b, rounded to T; with
// mask_e, 3-D E entries that are not unknowns are stored as 0 (fdtd.h)
template <typename T>
__global__ void state_scatter_kernel(const double* __restrict__ in, int64_t S, int B, int nx, int ny, int nz, int px,
                                     int dim, int comp, bool mask_e, T* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= S * B) return;
  const int b = (int)(t / S);
  const int64_t s = t % S;
  const int64_t i = s % (nx + 1);
  int64_t j, k;
  if (dim == 3) { j = (s / (nx + 1)) % (ny + 1); k = s / ((int64_t)(nx + 1) * (ny + 1)); }
  else { j = s / (nx + 1); k = 0; }
  bool keep = true;
  if (mask_e) {
    const bool xi = i > 0 && i < nx, yi = j > 0 && j < ny, zi = k > 0 && k < nz;
    keep = comp == 0 ? (i < nx && yi && zi) : comp == 1 ? (xi && j < ny && zi) : (xi && yi && k < nz);
  }
  out[((k * (ny + 1) + j) * px + i) * B + b] = keep ? (T)in[t] : (T)0;
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
