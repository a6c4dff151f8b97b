// stencil3d.cuh — the 3-D fused E->H Yee stencil (rows a1-a3, a5 of DESIGN.md
// §1), tile kernel of round 1b.
//
// One CTA = 32 x BY threads; a tile is a (row of 32*W elements) x BY rows
// footprint; the CTA is persistent and marches its balanced range of
// column-planes (TileSplit below).  Per z-plane one elected thread issues
// six TMA tile loads (H with a -x/-y halo, E^n) into an NS-stage ring that
// completes on mbarriers; the ring is refilled right after the plane's CTA
// barrier, so NS planes are in flight while one is computed.
//
// Each thread owns W consecutive elements of a tile row (16 or 8 bytes):
//   XV = true  (batch 1): W consecutive x cells.  The x-1 neighbour of its
//              first cell and the x+1 neighbour of its last cell are scalar
//              shared loads, the others are its own registers;
//   XV = false (batch B, B % W == 0): W batch members of one cell; x
//              neighbours are the vectors B elements away.
// E^{n+1} is computed on the whole footprint and H^{n+3/2} on the footprint
// minus its last x cell and last row (overlapped tiling; the halo E is
// recomputed by the neighbour, race free because old and new buffers differ).
//
// Per plane kk (one CTA barrier):
//   wait stage(kk); E^{n+1}(kk) from H(kk), H(kk-1) (registers), E^n(kk);
//   store E^{n+1}(kk) to En[kk&1] (shared) and to HBM;
//   H^{n+3/2}(kk-1) from E^{n+1}(kk) (registers), E^{n+1}(kk-1) (registers +
//   the x+1 / y+1 neighbours from En[(kk-1)&1]); store to HBM;
//   barrier; refill stage(kk) with plane kk+NS.
// Two En buffers suffice: all reads of En[(kk-1)&1] precede barrier kk, all
// writes of En[(kk+1)&1] follow it.
//
// The arithmetic of every update is the same expression, in the same order,
// as stencil3d_tma_kernel / stencil3d_pipe_kernel (bitwise-equal results,
// tests/test_gpu_configs.py).
#pragma once
#include "kernels.cuh"
#include "stencil3d_launch.h"   // TileSplit

namespace fdtd {

template <typename T, int W>
struct VecIO {
  static __device__ __forceinline__ LV<T, W> ld(const T* p) {
    LV<T, W> r;
    if constexpr (sizeof(T) * W == 16) {
      using V = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
      const V x = *reinterpret_cast<const V*>(p);
      if constexpr (W == 4) { r.v[0] = x.x; r.v[1] = x.y; r.v[2] = x.z; r.v[3] = x.w; }
      else { r.v[0] = x.x; r.v[1] = x.y; }
    } else if constexpr (sizeof(T) * W == 8 && W == 2) {
      const float2 x = *reinterpret_cast<const float2*>(p);
      r.v[0] = x.x; r.v[1] = x.y;
    } else {
#pragma unroll
      for (int w = 0; w < W; ++w) r.v[w] = p[w];
    }
    return r;
  }
  static __device__ __forceinline__ void st(T* p, const LV<T, W>& r) {
    if constexpr (sizeof(T) * W == 16) {
      using V = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
      V x;
      if constexpr (W == 4) { x.x = r.v[0]; x.y = r.v[1]; x.z = r.v[2]; x.w = r.v[3]; }
      else { x.x = r.v[0]; x.y = r.v[1]; }
      *reinterpret_cast<V*>(p) = x;
    } else if constexpr (sizeof(T) * W == 8 && W == 2) {
      *reinterpret_cast<float2*>(p) = make_float2(r.v[0], r.v[1]);
    } else {
#pragma unroll
      for (int w = 0; w < W; ++w) p[w] = r.v[w];
    }
  }
};

// padded (128-byte) plane sizes in elements; the host mirror is in stencil3d_launch.h
__host__ __device__ constexpr int tile_hp(int HBX, int BY, int esz) {
  return ((HBX * (BY + 1)) * esz + 127) / 128 * 128 / esz;
}
__host__ __device__ constexpr int tile_ep(int RX, int BY, int esz) {
  return ((RX * BY) * esz + 127) / 128 * 128 / esz;
}

constexpr int TILE_BY = 8;   // default tile rows (one warp per row)

// Persistent work split: the (x, y) tiles are "columns" of nz+1 planes, cut
// into z-chunks of S.kc planes; item = chunk * ncols + column (chunk-major, so
// the CTAs of one round work on neighbouring tiles of the same z band and
// share their halos in L2).  CTA c processes items c, c + G, c + 2G, ...
// An item [a, b) loads plane a-1 (H only: H(a-1) for the z-derivative of
// E(a); not for a = 0), planes a .. min(b, nz) (plane b only feeds H(b-1)),
// stores E on [a, b) and H on [a, b-1) (+ the copied-through top plane when
// b = nz+1).  The TMA ring runs across item boundaries without draining.
struct SegCursor {               // walks the load sequence of one CTA's items
  int item, col, a, b, kl, k;    // current item, its column and [a, b), last plane loaded, next plane
  bool done;
  __device__ __forceinline__ void set(const TileSplit& S, int it, int nz) {
    item = it;
    done = it >= S.nitems;
    if (done) return;
    col = S.column(it % S.ncols);
    a = (it / S.ncols) * S.kc;
    b = min(a + S.kc, S.nzp);
    kl = min(b, nz);
    k = a > 0 ? a - 1 : a;
  }
  __device__ __forceinline__ void next(const TileSplit& S, int nz) {
    if (++k > kl) set(S, item + (int)gridDim.x, nz);
  }
};

template <typename T, bool UNIFORM, int NS, int W, int MB, int MINB, int BY = TILE_BY, bool LOSSY = false>
__global__ void __launch_bounds__(32 * BY, MINB)
stencil3d_tile_kernel(const __grid_constant__ TmaSet tm, const TileSplit S, Dims d, Fields<T> F0,
                      Fields<T> F1, const uint8_t* __restrict__ mat_id, const Coef<T>* __restrict__ gtab,
                      const uint8_t* __restrict__ gifm, int n_mat, Coef<T> u0, Coef<T> u1, RowsE<T> R,
                      const T* __restrict__ y, const int64_t* __restrict__ d_step, int check_every,
                      unsigned long long* __restrict__ bad_step, const T* __restrict__ gtaba) {
  // LOSSY (table variant only): gtaba [n_mat][6] holds ca / da of Eq. (2a)/(2b) with
  // conductivities, E <- ca E + cb curl, H <- da H - ch curl (fdtd.h coef_a)
  // MB == 0: batch 1, W x cells per thread (XV); MB > 0: batch of MB members, W per thread
  constexpr bool XV = MB == 0;
  using L = LV<T, W>;
  using IO = VecIO<T, W>;
  constexpr int RX = 32 * W;                   // elements per tile row
  constexpr int B = XV ? 1 : MB;
  constexpr int SX = (16 / (int)sizeof(T)) > B ? (16 / (int)sizeof(T)) : B;
  constexpr int HW = RX + SX;                  // H box width (elements): SX halo elements + the tile
  constexpr int HP = tile_hp(HW, BY, (int)sizeof(T)), EP = tile_ep(RX, BY, (int)sizeof(T));
  constexpr int STG = 3 * (HP + EP);           // elements per ring stage
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // programmatic dependent launch: the step's reduced kernel may be scheduled
  // once every CTA of this grid has started (it then waits for our completion
  // with griddepcontrol.wait; no stencil CTA is still pending by then)
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const int tx = threadIdx.x, ty = threadIdx.y;
  const unsigned base_u = smem_u32(smem_raw);
  unsigned char* smem_al = smem_raw + ((128u - (base_u & 127u)) & 127u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_al);                 // [NS]
  T* Ring = reinterpret_cast<T*>(smem_al + 128);                         // [NS][H 3][E 3]
  T* En = Ring + NS * STG;                                                // [2][3][EP]
  Coef<T>* tabc = reinterpret_cast<Coef<T>*>(En + 2 * 3 * EP);           // [n_mat][6]
  uint8_t* tabf = reinterpret_cast<uint8_t*>(tabc + 6 * n_mat);           // [n_mat] explicit-row bits
  T* taba = reinterpret_cast<T*>(tabf + ((n_mat + 15) & ~15));            // [n_mat][6] (LOSSY)
  const bool leader = (tx == 0 && ty == 0);
  if (leader) {
    for (int q = 0; q < NS; ++q) mbar_init(&bars[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (!UNIFORM) {
    for (int m = ty * 32 + tx; m < n_mat; m += 32 * BY) {
      for (int c = 0; c < 6; ++c) tabc[m * 6 + c] = gtab[m * 6 + c];
      if (LOSSY)
        for (int c = 0; c < 6; ++c) taba[m * 6 + c] = gtaba[m * 6 + c];
      tabf[m] = gifm[m];
    }
  }
  __syncthreads();
  const int nx = d.nx, ny = d.ny, nz = d.nz;
  const unsigned stage_bytes = (unsigned)((3 * HW * (BY + 1) + 3 * RX * BY) * sizeof(T));
  // producer (leader thread): issues the load sequence NS planes ahead
  SegCursor pc;
  pc.set(S, blockIdx.x, nz);
  auto issue = [&](int st) {
    const int i0p = (pc.col % S.ntx) * S.outx, j0p = (pc.col / S.ntx) * S.outy;
    T* h_ = Ring + st * STG;
    T* e_ = h_ + 3 * HP;
    mbar_expect_tx(&bars[st], stage_bytes);
    tma_load_3d(h_ + 0 * HP, &tm.h[0], i0p * B, j0p, pc.k, &bars[st]);
    tma_load_3d(h_ + 1 * HP, &tm.h[1], i0p * B, j0p, pc.k, &bars[st]);
    tma_load_3d(h_ + 2 * HP, &tm.h[2], i0p * B, j0p, pc.k, &bars[st]);
    tma_load_3d(e_ + 0 * EP, &tm.e[0], i0p * B + SX, j0p + 1, pc.k, &bars[st]);
    tma_load_3d(e_ + 1 * EP, &tm.e[1], i0p * B + SX, j0p + 1, pc.k, &bars[st]);
    tma_load_3d(e_ + 2 * EP, &tm.e[2], i0p * B + SX, j0p + 1, pc.k, &bars[st]);
    pc.next(S, nz);
  };
  if (leader) {
    for (int q = 0; q < NS && !pc.done; ++q) issue(q);
  }
  const int xe = tx * W;                       // first element of this thread in the tile row
  const int ci = XV ? xe : xe / B;             // its (first) cell within the tile
  const int b = XV ? 0 : xe % B;
  const int hoff = (ty + 1) * HW + xe + SX;    // this thread's H element in a stage
  const int erow = ty * RX + xe;
  const int64_t sz = d.plane * B;
  const uint32_t sz32 = (uint32_t)sz;
  const int64_t step = *d_step;
  const bool do_check = check_every > 0 && (step % check_every) == 0;
  bool bad = false;
  int st = 0;
  unsigned phase = 0;
  unsigned ebuf = 0;                           // En buffer of the current plane
  for (int item = blockIdx.x; item < S.nitems; item += gridDim.x) {
    // ---- item start: this thread's cell in the column's tile
    const int col = S.column(item % S.ncols);
    const int a = (item / S.ncols) * S.kc, bseg = min(a + S.kc, S.nzp), kl = min(bseg, nz);
    const int i0 = (col % S.ntx) * S.outx, j0 = (col / S.ntx) * S.outy;
    const int i = i0 + ci, j = j0 + ty;
    const bool inside = (i <= nx) && (j <= ny);
    const bool own = inside && (ci < S.outx) && (ty < S.outy);
    // XV: clamp to a W-aligned cell so vector loads of the material row stay
    // aligned (i itself is W-aligned, so every inside thread keeps ii == i)
    const int ii = XV ? min(i, nx & ~(W - 1)) : min(i, nx), jj = min(j, ny);
    const int64_t scol = (int64_t)jj * d.px + ii;
    const int64_t colo = scol * B + b;
    // per-element masks of the unknowns in (x, y), as exact 0/1 multipliers of
    // the curl difference: d * 1 == d, so an unknown gets the reference
    // expression bit for bit; a masked entry gets x_old + c*(+-0) == x_old,
    // which is 0 for E (the state outside the unknowns is 0 and
    // fdtd_set_state stores it as 0) and the old value for H, as in the
    // reference kernels.  The z-wall planes are uniform fix-ups below.
    //   fa = [i<nx][0<j<ny] (Ex, Hy)   fb = [0<i<nx][j<ny] (Ey, Hx)
    //   fc = [0<i<nx][0<j<ny] (Ez)     fd = [i<nx][j<ny] (Hz)
    T fa[W], fb[W], fc[W], fd[W];
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const int iw = XV ? i + w : i;
      const bool x1 = iw < nx, x0 = (iw > 0) && x1, y1 = j < ny, y0 = (j > 0) && y1;
      fa[w] = (x1 && y0) ? (T)1 : (T)0;
      fb[w] = (x0 && y1) ? (T)1 : (T)0;
      fc[w] = (x0 && y0) ? (T)1 : (T)0;
      fd[w] = (x1 && y1) ? (T)1 : (T)0;
    }
    // H(kk-1) and E^{n+1}(kk-1) of this thread's elements, carried in registers
    L hxk{}, hyk{}, hzk{}, exk{}, eyk{}, ezk{};
    if (a > 0) {
      // lead plane a-1: only its H (own position) is used
      mbar_wait(&bars[st], phase);
      const T* h = Ring + st * STG + hoff;
      hxk = IO::ld(h + 0 * HP); hyk = IO::ld(h + 1 * HP); hzk = IO::ld(h + 2 * HP);
      __syncthreads();
      if (leader && !pc.done) issue(st);
      if (++st == NS) { st = 0; phase ^= 1u; }
    }
    // element offset of plane kk (E) in the output arrays; H(kk-1) is at oe - sz
    uint32_t oe = (uint32_t)((int64_t)a * sz + colo);
    // material ids (XV: W bytes packed), loaded 3 planes ahead of use
    uint32_t m_n1 = 0, m_n2 = 0, m_n3 = 0, m_cur = 0, m_prev = 0;
    auto load_mat = [&](int k) -> uint32_t {
      const uint8_t* p = mat_id + (int64_t)k * d.plane + scol;
      if constexpr (XV && W == 4) return *reinterpret_cast<const uint32_t*>(p);
      else if constexpr (XV && W == 2) return *reinterpret_cast<const uint16_t*>(p);
      else return (uint32_t)__ldg(p);
    };
    if (!UNIFORM) {
      m_n1 = load_mat(a);
      if (a + 1 <= kl) m_n2 = load_mat(a + 1);
      if (a + 2 <= kl) m_n3 = load_mat(a + 2);
    }
    for (int kk = a; kk <= kl; ++kk) {
      if (S.jitter) {
        const unsigned hsh = (unsigned)(blockIdx.x * 2654435761u) ^ (unsigned)(kk * 40503u) ^ (threadIdx.y * 97u);
        if ((threadIdx.x & 31) == 0) __nanosleep((hsh * 2246822519u >> 7) % (unsigned)S.jitter);
        __syncwarp();
      }
      mbar_wait(&bars[st], phase);
      const T* h = Ring + st * STG + hoff;
      const T* e = Ring + st * STG + 3 * HP + erow;
      const L hx_c = IO::ld(h + 0 * HP), hy_c = IO::ld(h + 1 * HP), hz_c = IO::ld(h + 2 * HP);
      const L hz_jm = IO::ld(h + 2 * HP - HW), hx_jm = IO::ld(h + 0 * HP - HW);
      L hz_im, hy_im;
      if constexpr (XV) {
        hz_im.v[0] = h[2 * HP - 1];
        hy_im.v[0] = h[1 * HP - 1];
#pragma unroll
        for (int w = 1; w < W; ++w) { hz_im.v[w] = hz_c.v[w - 1]; hy_im.v[w] = hy_c.v[w - 1]; }
      } else {
        hz_im = IO::ld(h + 2 * HP - B);
        hy_im = IO::ld(h + 1 * HP - B);
      }
      const L ex0 = IO::ld(e + 0 * EP), ey0 = IO::ld(e + 1 * EP), ez0 = IO::ld(e + 2 * EP);
      if (!UNIFORM) {
        m_prev = m_cur; m_cur = m_n1; m_n1 = m_n2; m_n2 = m_n3;
        if (kk + 3 <= kl) m_n3 = load_mat(kk + 3);
      }
      L ex, ey, ez;
      uint8_t ifm_any = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        Coef<T> cx, cy, cz;
        if (UNIFORM) { cx = u0; cy = u0; cz = u0; }
        else {
          const int m = XV ? (int)((m_cur >> (8 * w)) & 0xffu) : (int)m_cur;
          cx = tabc[m * 6 + 0]; cy = tabc[m * 6 + 1]; cz = tabc[m * 6 + 2];
          ifm_any |= tabf[m];
        }
        if constexpr (LOSSY && !UNIFORM) {
          const int ml = XV ? (int)((m_cur >> (8 * w)) & 0xffu) : (int)m_cur;
          ex.v[w] = fma(taba[ml * 6 + 0], ex0.v[w], cx.apply(((hz_c.v[w] - hz_jm.v[w]) - (hy_c.v[w] - hyk.v[w])) * fa[w]));
          ey.v[w] = fma(taba[ml * 6 + 1], ey0.v[w], cy.apply(((hx_c.v[w] - hxk.v[w]) - (hz_c.v[w] - hz_im.v[w])) * fb[w]));
          ez.v[w] = fma(taba[ml * 6 + 2], ez0.v[w], cz.apply(((hy_c.v[w] - hy_im.v[w]) - (hx_c.v[w] - hx_jm.v[w])) * fc[w]));
        } else {
        ex.v[w] = cx.add(ex0.v[w], ((hz_c.v[w] - hz_jm.v[w]) - (hy_c.v[w] - hyk.v[w])) * fa[w]);
        ey.v[w] = cy.add(ey0.v[w], ((hx_c.v[w] - hxk.v[w]) - (hz_c.v[w] - hz_im.v[w])) * fb[w]);
        ez.v[w] = cz.add(ez0.v[w], ((hy_c.v[w] - hy_im.v[w]) - (hx_c.v[w] - hx_jm.v[w])) * fc[w]);
        }
      }
      // z walls: tangential E on k = 0 and everything on k = nz are not unknowns
      if (kk == 0) {
#pragma unroll
        for (int w = 0; w < W; ++w) { ex.v[w] = (T)0; ey.v[w] = (T)0; }
      }
      if (kk == nz) {
#pragma unroll
        for (int w = 0; w < W; ++w) { ex.v[w] = (T)0; ey.v[w] = (T)0; ez.v[w] = (T)0; }
      }
      if (!UNIFORM && ifm_any && inside) {
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const int m = XV ? (int)((m_cur >> (8 * w)) & 0xffu) : (int)m_cur;
          const uint8_t f = tabf[m];
          if (!f || (XV && i + w > nx)) continue;
          // rows_prepass_kernel (kernels.cuh) evaluated every explicit row of this
          // step and stored its E^{n+1} into the new parity: read it back
          if (f & 1) ex.v[w] = F1.f[0][oe + w];
          if (f & 2) ey.v[w] = F1.f[1][oe + w];
          if (f & 4) ez.v[w] = F1.f[2][oe + w];
        }
      }
      T* en = En + ebuf * (3 * EP) + erow;
      IO::st(en + 0 * EP, ex); IO::st(en + 1 * EP, ey); IO::st(en + 2 * EP, ez);
      if (own && kk < bseg) {
        IO::st(F1.f[0] + oe, ex); IO::st(F1.f[1] + oe, ey); IO::st(F1.f[2] + oe, ez);
        if (do_check)
#pragma unroll
          for (int w = 0; w < W; ++w) bad |= !(finite_small(ex.v[w]) && finite_small(ey.v[w]) && finite_small(ez.v[w]));
      }
      if (kk > a && own) {
        // H^{n+3/2} of plane kk-1 (kk-1 < nz always)
        const T* ep = En + (ebuf ^ 1u) * (3 * EP) + erow;
        L ey_ip, ez_ip;
        if constexpr (XV) {
#pragma unroll
          for (int w = 0; w + 1 < W; ++w) { ey_ip.v[w] = eyk.v[w + 1]; ez_ip.v[w] = ezk.v[w + 1]; }
          ey_ip.v[W - 1] = ep[1 * EP + W];
          ez_ip.v[W - 1] = ep[2 * EP + W];
        } else {
          ey_ip = IO::ld(ep + 1 * EP + B);
          ez_ip = IO::ld(ep + 2 * EP + B);
        }
        const L ex_jp = IO::ld(ep + 0 * EP + RX), ez_jp = IO::ld(ep + 2 * EP + RX);
        const bool hz_on = kk - 1 > 0;         // Hz on k = 0 (normal to the bottom wall) is not updated
        L hx1, hy1, hz1;
#pragma unroll
        for (int w = 0; w < W; ++w) {
          Coef<T> hx_, hy_, hz_;
          if (UNIFORM) { hx_ = u1; hy_ = u1; hz_ = u1; }
          else {
            const int m = XV ? (int)((m_prev >> (8 * w)) & 0xffu) : (int)m_prev;
            hx_ = tabc[m * 6 + 3]; hy_ = tabc[m * 6 + 4]; hz_ = tabc[m * 6 + 5];
          }
          if constexpr (LOSSY && !UNIFORM) {
            // masked entries (fb / fa / fd = 0) are not unknowns: they keep their value
            const int ml = XV ? (int)((m_prev >> (8 * w)) & 0xffu) : (int)m_prev;
            hx1.v[w] = fb[w] != (T)0 ? fma(taba[ml * 6 + 3], hxk.v[w], -hx_.apply((ez_jp.v[w] - ezk.v[w]) - (ey.v[w] - eyk.v[w]))) : hxk.v[w];
            hy1.v[w] = fa[w] != (T)0 ? fma(taba[ml * 6 + 4], hyk.v[w], -hy_.apply((ex.v[w] - exk.v[w]) - (ez_ip.v[w] - ezk.v[w]))) : hyk.v[w];
            hz1.v[w] = (hz_on && fd[w] != (T)0) ? fma(taba[ml * 6 + 5], hzk.v[w], -hz_.apply((ey_ip.v[w] - eyk.v[w]) - (ex_jp.v[w] - exk.v[w]))) : hzk.v[w];
          } else {
          hx1.v[w] = hx_.sub(hxk.v[w], ((ez_jp.v[w] - ezk.v[w]) - (ey.v[w] - eyk.v[w])) * fb[w]);
          hy1.v[w] = hy_.sub(hyk.v[w], ((ex.v[w] - exk.v[w]) - (ez_ip.v[w] - ezk.v[w])) * fa[w]);
          hz1.v[w] = hz_on ? hz_.sub(hzk.v[w], ((ey_ip.v[w] - eyk.v[w]) - (ex_jp.v[w] - exk.v[w])) * fd[w])
                           : hzk.v[w];
          }
        }
        const uint32_t oh = oe - sz32;
        IO::st(F1.f[3] + oh, hx1); IO::st(F1.f[4] + oh, hy1); IO::st(F1.f[5] + oh, hz1);
        if (do_check)
#pragma unroll
          for (int w = 0; w < W; ++w) bad |= !(finite_small(hx1.v[w]) && finite_small(hy1.v[w]) && finite_small(hz1.v[w]));
      }
      __syncthreads();            // stage st and the other En buffer are free after this
      if (leader && !pc.done) issue(st);
      hxk = hx_c; hyk = hy_c; hzk = hz_c;
      exk = ex; eyk = ey; ezk = ez;
      oe += sz32;
      ebuf ^= 1u;
      if (++st == NS) { st = 0; phase ^= 1u; }
    }
    if (bseg == nz + 1 && own) {
      // the never-updated H plane k = nz (normal / tangential on the top wall) is copied through
      const uint32_t oh = oe - sz32;
      IO::st(F1.f[3] + oh, hxk); IO::st(F1.f[4] + oh, hyk); IO::st(F1.f[5] + oh, hzk);
    }
  }
  if (bad) atomicMin(bad_step, (unsigned long long)step);
}

}  // namespace fdtd
