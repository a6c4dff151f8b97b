// persist2d.cuh — persistent, on-chip-resident 2-D hybrid step (sm_100a).
//
// The whole time march of a 2-D problem (Ez, Hx, Hy coarse grid + fused
// single-column reduced blocks) in ONE cooperative launch.  Each CTA owns a
// TX x TY tile of the coarse grid and keeps its three fields in shared memory
// for the whole launch (config 2: 1025^2 x 3 fp32 = 12.6 MB spread over 289
// CTAs, 48 KB each) -- no per-step HBM/L2 round trip of the state (DESIGN.md
// §5.4).  Per step (paper eq. (4)/(12) order, rows a1-a7 of DESIGN.md §1):
//
//   E phase  Ez^{n+1} on the tile; the left column of Hy / bottom row of Hx it
//            needs come from the neighbours' published H halos of step n-1;
//            explicit rows (interface rows with the reduced coupling y = S_E
//            h~, source rows) are evaluated in place and interface rows
//            publish E_if^{n+1} into G.
//   H phase  Hx, Hy on the tile; the right column / top row of Ez come from
//            the neighbours' published E halos of step n.
//   reduced  every CTA keeps a few rows of the fused update matrix M
//            resident in shared memory and computes them once all interface
//            tiles published G: [h~' ; y' ; e~'' ; probe rows] = M [e~ ; h~ ; G].
//
// Synchronisation is point to point through monotonic per-tile flags (fE, fH:
// phases completed) and two counters (gready: interface tiles that published
// G, reddone: CTAs that finished their reduced rows); halos are double
// buffered by step parity, which makes every write-after-read safe (the
// argument is in DESIGN.md §5.4).  Cross-CTA data is read with ld.global.cg
// (L2, never a stale L1 line).  Every wait is bounded: after ~1 s of spinning
// the CTA raises `abort` and all CTAs leave; the host reports the error.
//
// The arithmetic of every update is the same expression, in the same order,
// as stencil2d_rows_kernel / eval_row / reduced_fused_kernel: the persistent
// and the per-step paths agree bit for bit (tests/test_gpu_parity.py).
#pragma once

namespace fdtd {

template <typename T>
struct P2Rows {                 // explicit rows grouped by tile (CSR over tiles)
  const int32_t* tile_ptr;      // [nT+1]
  const int32_t* li;            // local cell index jl * TX + il
  const Coef<T>* c;
  const int8_t* nterm;          // H terms (<= 4), in the problem's CSR order
  const int8_t* slot;           // [4]: 0 Hy(i,j) 1 Hy(i-1,j) 2 Hx(i,j) 3 Hx(i,j-1)
  const T* w;                   // [4]
  const int64_t* yo;            // y / G index, -1 none
  const int32_t* src;           // waveform column, -1 none
  const T* cs;
  const T* wave;                // [n_wave][n_cols]
  int64_t n_wave, n_cols;
  const int8_t* own;            // temporal blocking: 1 if the row's cell is in the tile's owned region
};

template <typename T>
struct P2Row {                  // one explicit row, cached in shared memory
  Coef<T> c;
  T w[4];
  T cs;
  int64_t yo;
  int32_t li, src;
  int8_t nterm, slot[4], own;
};

template <typename T>
struct P2Probes {               // coarse probes whose terms all lie in one tile
  const int32_t* tile_ptr;      // [nT+1] over probes
  const int32_t* pid;
  const int32_t* term_ptr;      // [np+1]
  const int32_t* term_li;
  const int8_t* term_comp;      // 0 Ez, 1 Hx, 2 Hy
  const T* term_w;
};

template <typename T>
struct Persist2D {
  int nx, ny, px, TX, TY, ntx, nty;
  const T* Fin[3];              // Ez, Hx, Hy at the start (storage layout, pitch px)
  T* Fout[3];
  const uint8_t* mat_id;        // padded storage-indexed material ids (or null: uniform)
  const Coef<T>* gtab;          // [n_mat][6]
  const uint8_t* gifm;
  int n_mat;
  Coef<T> u0, u1;
  P2Rows<T> R;
  P2Probes<T> PR;
  T* ezL; T* ezB; T* hyR; T* hxT;         // halos [2][nT][TY] / [2][nT][TX]
  unsigned* fE; unsigned* fH;             // [nT] phases completed
  unsigned* gready; unsigned* reddone; int* abort_flag;
  const uint8_t* tile_if;                 // tile has interface rows
  int n_if_tiles, n_red_ctas;
  // reduced (fused, N = 1)
  FusedBlock<T> fb[kMaxFusedBlocks];
  int row0[kMaxFusedBlocks + 1];          // first global row of each block
  int nfb, Rtot, rpc, Cmax;           // rpc: rows per reduced CTA (CTAs nT .. nT+n_red_ctas-1)
  T* eb[2]; T* hb[2]; T* y; T* G;
  const T* y_in;                // fp32: a copy of y taken before the launch, read at local step 0 (the
                                // reduced CTAs overwrite y during the launch; a temporal-blocking halo
                                // tile is on no chain that orders its step-0 read before that write)
  T* ring; int64_t cap; int n_probe;
  int64_t step0; int p0; int nsteps;
  int64_t* d_step_out;
  int check_every;
  int maxrows;                  // explicit rows of the fullest tile
  unsigned long long* bad_step;
  unsigned long long* dbg;      // optional phase timestamps (FDTD_P2DBG), [cta slot][step][8]
  int dbg_tile_if;              // which tile to trace besides tile 0
  // fp32: flag-in-data ("LL") exchange buffers, each word = (step tag << 32) | value bits,
  // double buffered by local step parity; they replace the per-tile flags and counters
  unsigned long long *lezL, *lezB, *lhyR, *lhxT;   // halos [2][nT][TY] / [2][nT][TX]
  unsigned long long *lG, *ly;                     // [2][y_size]
  unsigned long long *leb, *lhb;                   // [2][e_size] / [2][h_size]
  int64_t ysz, esz, hsz;
  int ymask;                    // G / y ring depth - 1 (1: double buffer; temporal blocking: >= K)
  // temporal blocking (persist2d_tb_tile): K-cell halos, exchanged every K steps
  int K;                        // 0: per-step exchange (persist2d_tile)
  unsigned long long* lband;    // [2][nT][4 sides][3 fields][K][T] tagged words
  unsigned sleep_ns;            // poll back-off of the temporal-blocking kernel
  unsigned jitter;              // race testing (FDTD_JITTER=ns): pseudo-random per-warp delays
};

// race testing: warp-level pseudo-random delay of 0..P.jitter ns at a phase point
#define P2_JITTER(P, salt)                                                                        \
  do {                                                                                            \
    if ((P).jitter) {                                                                             \
      const unsigned hsh_ = (blockIdx.x * 2654435761u) ^ ((unsigned)(salt) * 40503u) ^ ((threadIdx.x >> 5) * 97u); \
      if ((threadIdx.x & 31) == 0) __nanosleep((hsh_ * 2246822519u >> 7) % (P).jitter);           \
      __syncwarp();                                                                               \
    }                                                                                             \
  } while (0)

template <bool B> struct BoolC { static constexpr bool value = B; };

// LL words: a 64-bit relaxed store/load is single-copy atomic, so a reader that
// sees the expected tag also sees the value stored with it; no fence, no flag
__device__ __forceinline__ void ll_st(unsigned long long* p, float v, unsigned tag) {
  const unsigned long long w = ((unsigned long long)tag << 32) | (unsigned long long)__float_as_uint(v);
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;\n" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ unsigned long long ll_raw(const unsigned long long* p) {
  unsigned long long w;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];\n" : "=l"(w) : "l"(p) : "memory");
  return w;
}
// spin until the word carries `tag`; false on abort / timeout (~1 s of SM clock)
// (sleep_ns > 0: back off after 8 failed polls, leaving the issue slots to
// the co-resident CTA -- the temporal-blocking kernel)
__device__ __forceinline__ bool ll_ld(const unsigned long long* p, unsigned tag, float& v, int* abort_flag,
                                      unsigned sleep_ns = 0) {
  unsigned long long w = ll_raw(p);
  if ((unsigned)(w >> 32) != tag) {
    const long long t0 = clock64();
    unsigned it = 0;
    do {
      if (sleep_ns && it >= 8) __nanosleep(sleep_ns);
      w = ll_raw(p);
      if ((++it & 63u) == 0) {
        if (*reinterpret_cast<volatile int*>(abort_flag)) return false;
        if (clock64() - t0 > 2000000000LL) { atomicExch(abort_flag, 1); return false; }
      }
    } while ((unsigned)(w >> 32) != tag);
  }
  v = __uint_as_float((unsigned)w);
  return true;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define P2_STAMP(slot, k)                                                                    \
  do {                                                                                       \
    if (P.dbg && threadIdx.x == 0 && ls >= 100 && ls < 108)                                  \
      P.dbg[((slot) * 8 + (ls - 100)) * 8 + (k)] = gtimer();                                 \
  } while (0)

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// thread 0 spins until *flag >= target; false on abort / timeout (~1 s of
// SM clock).  No back-off: the flags are the step's critical path.
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ bool p2_wait(const unsigned* flag, unsigned target, int* abort_flag) {
  // relaxed polling (no L1 invalidation per poll), one acquire fence on success
  if (ld_relaxed_u32(flag) < target) {
    const long long t0 = clock64();
    unsigned it = 0;
    while (ld_relaxed_u32(flag) < target) {
      if ((++it & 63u) == 0) {
        if (*reinterpret_cast<volatile int*>(abort_flag)) return false;
        if (clock64() - t0 > 2000000000LL) { atomicExch(abort_flag, 1); return false; }
      }
    }
  }
  asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
  return true;
}

template <typename T>
__device__ void persist2d_tile(const Persist2D<T>& P, unsigned char* smem_raw, int& s_abort) {
  const int TX = P.TX, TY = P.TY, TT = TX * TY;
  const int nT = P.ntx * P.nty;
  const int t = blockIdx.x;
  const int tx_ = t % P.ntx, ty_ = t / P.ntx;
  const int i0 = tx_ * TX, j0 = ty_ * TY;
  const int left = tx_ > 0 ? t - 1 : -1, right = tx_ + 1 < P.ntx ? t + 1 : -1;
  const int bottom = ty_ > 0 ? t - P.ntx : -1, top = ty_ + 1 < P.nty ? t + P.ntx : -1;
  const int nx = P.nx, ny = P.ny, px = P.px;
  const bool uniform = (P.mat_id == nullptr);
  T* sEz = reinterpret_cast<T*>(smem_raw);
  T* sHx = sEz + TT;
  T* sHy = sHx + TT;
  T* hL = sHy + TT;                  // Hy(i0-1, j)
  T* hB = hL + TY;                   // Hx(i, j0-1)
  T* eR = hB + TX;                   // Ez(i0+TX, j)
  T* eT = eR + TY;                   // Ez(i, j0+TY)
  Coef<T>* cE = reinterpret_cast<Coef<T>*>(eT + TX);
  Coef<T>* cHx = cE + MAX_MAT;
  Coef<T>* cHy = cHx + MAX_MAT;
  uint8_t* ifm = reinterpret_cast<uint8_t*>(cHy + MAX_MAT);
  uint8_t* smat = ifm + MAX_MAT;     // [TT]
  T* yv = reinterpret_cast<T*>(smat + ((TT + 15) / 16) * 16);   // [max rows per tile] prefetched y (+ source)
  P2Row<T>* rs = reinterpret_cast<P2Row<T>*>(yv + ((2 * P.maxrows * (int)sizeof(T) + 15) / 16) * 16 / (int)sizeof(T));
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int lx = tid & 31, ly = tid >> 5, NLY = nthr >> 5;
  const bool pair = sizeof(T) == 4 && TX == 64;   // paired interior loops (fp32, 64-wide tiles)
  // the tile covers cells i < nx, j < ny: the last storage column / row (PEC
  // wall Ez = 0, H never updated) is constant and written back by CTA 0
  for (int jl = ly; jl < TY; jl += NLY)
    for (int il = lx; il < TX; il += 32) {
      const int i = i0 + il, j = j0 + jl;
      const int c = jl * TX + il;
      T ez = 0, hx = 0, hy = 0;
      uint8_t m = 0;
      if (i < nx && j < ny) {
        const int64_t o = (int64_t)j * px + i;
        ez = P.Fin[0][o]; hx = P.Fin[1][o]; hy = P.Fin[2][o];
        if (!uniform) m = P.mat_id[o];
      }
      sEz[c] = ez; sHx[c] = hx; sHy[c] = hy; smat[c] = m;
    }
  if (!uniform) {
    for (int q = tid; q < P.n_mat; q += nthr) {
      cE[q] = P.gtab[q * 6 + 2]; cHx[q] = P.gtab[q * 6 + 3]; cHy[q] = P.gtab[q * 6 + 4];
      ifm[q] = P.gifm[q];
    }
  }
  const int rows_lo = P.R.tile_ptr[t], rows_hi = P.R.tile_ptr[t + 1];
  // explicit-row cells exist only in tiles with rows (the others skip the check)
  const bool tile_rows = !uniform && rows_hi > rows_lo;
  for (int r = rows_lo + tid; r < rows_hi; r += nthr) {
    P2Row<T> x;
    x.c = P.R.c[r]; x.cs = P.R.cs[r]; x.yo = P.R.yo[r]; x.li = P.R.li[r]; x.src = P.R.src[r];
    x.nterm = P.R.nterm[r];
    for (int k = 0; k < 4; ++k) { x.w[k] = P.R.w[4 * r + k]; x.slot[k] = P.R.slot[4 * r + k]; }
    rs[r - rows_lo] = x;
  }
  __syncthreads();
  const bool has_if = P.tile_if[t] != 0;
  const int pr_lo = P.PR.tile_ptr[t], pr_hi = P.PR.tile_ptr[t + 1];
  bool bad = false;
  long long first_bad = -1;
  const int dslot = (t == 0) ? 0 : (t == P.dbg_tile_if ? 1 : -1);
  for (int ls = 0; ls < P.nsteps; ++ls) {
    const int64_t step = P.step0 + ls;
    const bool do_check = P.check_every > 0 && (step % P.check_every) == 0;
    if (dslot >= 0) P2_STAMP(dslot, 0);
    P2_JITTER(P, 3 * ls);
    // ------------------------------------------------------------- E phase
    // (a) interior cells need no halo: computed before waiting for neighbours
    auto e_cell = [&](int il, int jl) {
      const int i = i0 + il, j = j0 + jl;
      const int c = jl * TX + il;
      const int m = smat[c];
      if (tile_rows && (ifm[m] & 4)) return;               // explicit row below
      const T hy = sHy[c], hx = sHx[c];
      const T hyim = (il > 0) ? sHy[c - 1] : hL[jl];
      const T hxm = (jl > 0) ? sHx[c - TX] : hB[il];
      const Coef<T> cc = uniform ? P.u0 : cE[m];
      const T dd = (hy - hyim) - (hx - hxm);
      sEz[c] = (i > 0 && j > 0) ? cc.add(sEz[c], dd) : (T)0;
    };
    if (pair) {
      // 64-wide tiles: lane lx owns the cell pair (2 lx, 2 lx + 1) of a row, so
      // the x-1 neighbour of the second cell is the first cell's register and
      // the loads are 8-byte pairs (same expression per cell as e_cell)
      const int ia = 2 * lx;
      for (int jl = 1 + ly; jl < TY; jl += NLY) {
        if (j0 + jl >= ny) break;
        const int c = jl * TX + ia;
        const float2 hy2 = *reinterpret_cast<const float2*>(sHy + c);
        const float2 hx2 = *reinterpret_cast<const float2*>(sHx + c);
        const float2 hxm2 = *reinterpret_cast<const float2*>(sHx + c - TX);
        const float2 ez2 = *reinterpret_cast<const float2*>(sEz + c);
        const uint16_t m2 = *reinterpret_cast<const uint16_t*>(smat + c);
        const int ma = m2 & 0xff, mb = m2 >> 8;
        float e0 = ez2.x, e1 = ez2.y;
        if (ia > 0 && i0 + ia < nx && !(tile_rows && (ifm[ma] & 4))) {
          const Coef<T> cc = uniform ? P.u0 : cE[ma];
          const T dd = (hy2.x - sHy[c - 1]) - (hx2.x - hxm2.x);
          e0 = (j0 + jl > 0) ? cc.add(e0, dd) : (T)0;
        }
        if (i0 + ia + 1 < nx && !(tile_rows && (ifm[mb] & 4))) {
          const Coef<T> cc = uniform ? P.u0 : cE[mb];
          const T dd = (hy2.y - hy2.x) - (hx2.y - hxm2.y);
          e1 = (j0 + jl > 0) ? cc.add(e1, dd) : (T)0;
        }
        *reinterpret_cast<float2*>(sEz + c) = make_float2(e0, e1);
      }
    } else {
    for (int jl = 1 + ly; jl < TY; jl += NLY) {
      if (j0 + jl >= ny) break;
      for (int il = 1 + lx; il < TX; il += 32) {
        if (i0 + il >= nx) break;
        e_cell(il, jl);
      }
    }
    }
    if (dslot >= 0) P2_STAMP(dslot, 5);
    // (b) wait for the left / bottom H halos (and, on interface tiles, for the
    //     reduced update of the previous step), then fetch halos and y together
    constexpr bool LL = sizeof(T) == 4;
    // tags: local step + 1 (the LL buffers are zeroed before every launch, so 0 never matches)
    const unsigned tag_prev = (unsigned)ls, tag_cur = (unsigned)(ls + 1);
    if (LL && ls > 0) {
      // fp32: every fetching thread polls its own tagged words (no flags); the
      // left halo, the bottom halo and the y values go to disjoint threads so
      // all polls are in flight at once
      const int hb_ = (ls - 1) & 1;
      bool ok = true;
      for (int q = tid; q < TY + TX && ok; q += nthr) {
        float v = 0.f;
        if (q < TY) {
          if (left >= 0) ok = ll_ld(P.lhyR + ((int64_t)hb_ * nT + left) * TY + q, tag_prev, v, P.abort_flag);
          hL[q] = (T)v;
        } else {
          if (bottom >= 0) ok = ll_ld(P.lhxT + ((int64_t)hb_ * nT + bottom) * TX + (q - TY), tag_prev, v, P.abort_flag);
          hB[q - TY] = (T)v;
        }
      }
      const int nrw = rows_hi - rows_lo;
      const int r0 = (nthr - TY - TX) > 0 ? (TY + TX) : 0;   // y polls on the threads after the halo ones
      for (int r = (tid - r0 + nthr) % nthr; r < nrw && ok; r += nthr) {
        const int64_t yo = rs[r].yo;
        const int sc = rs[r].src;
        float v = 0.f;
        if (yo >= 0) ok = ll_ld(P.ly + (int64_t)((ls - 1) & P.ymask) * P.ysz + yo, tag_prev, v, P.abort_flag);
        yv[r] = (T)v;
        if (sc >= 0) yv[P.maxrows + r] = (step < P.R.n_wave) ? P.R.wave[step * P.R.n_cols + sc] : (T)0;
      }
      if (!ok) s_abort = 1;
      __syncthreads();
      if (s_abort) break;
      if (dslot >= 0) P2_STAMP(dslot, 1);
    } else {
    if (ls > 0) {
      if (tid == 0) {
        bool ok = true;
        if (left >= 0) ok = p2_wait(P.fH + left, (unsigned)ls, P.abort_flag);
        if (ok && bottom >= 0) ok = p2_wait(P.fH + bottom, (unsigned)ls, P.abort_flag);
        if (ok && has_if) ok = p2_wait(P.reddone, (unsigned)(P.n_red_ctas * ls), P.abort_flag);
        if (!ok) s_abort = 1;
      }
      __syncthreads();
      if (s_abort) break;
    }
    if (dslot >= 0) P2_STAMP(dslot, 1);
    {
      const int hb_ = (ls - 1) & 1;
      for (int jl = tid; jl < TY; jl += nthr) {
        T v = 0;
        if (left >= 0) v = (ls == 0) ? ((j0 + jl < ny) ? P.Fin[2][(int64_t)(j0 + jl) * px + i0 - 1] : (T)0)
                                     : __ldcg(P.hyR + ((int64_t)hb_ * nT + left) * TY + jl);
        hL[jl] = v;
      }
      for (int il = tid; il < TX; il += nthr) {
        T v = 0;
        if (bottom >= 0) v = (ls == 0) ? ((i0 + il < nx) ? P.Fin[1][(int64_t)(j0 - 1) * px + i0 + il] : (T)0)
                                       : __ldcg(P.hxT + ((int64_t)hb_ * nT + bottom) * TX + il);
        hB[il] = v;
      }
      for (int r = tid; r < rows_hi - rows_lo; r += nthr) {
        const int64_t yo = rs[r].yo;
        const int sc = rs[r].src;
        yv[r] = (yo >= 0) ? __ldcg((LL ? P.y_in : P.y) + yo) : (T)0;
        if (sc >= 0) yv[P.maxrows + r] = (step < P.R.n_wave) ? P.R.wave[step * P.R.n_cols + sc] : (T)0;
      }
    }
    }
    __syncthreads();
    // (c) first column and first row
    for (int q = tid; q < TX + TY - 1; q += nthr) {
      const int il = q < TX ? q : 0, jl = q < TX ? 0 : q - TX + 1;
      if (i0 + il >= nx || j0 + jl >= ny) continue;
      e_cell(il, jl);
    }
    // (d) explicit rows (eval_row: acc in the problem's order, then y, then source)
    for (int r = tid; r < rows_hi - rows_lo; r += nthr) {
      const P2Row<T>& x = rs[r];
      const int c = x.li;
      const int il = c % TX, jl = c / TX;
      T acc = 0;
      for (int k = 0; k < x.nterm; ++k) {
        const int sl = x.slot[k];
        T hv;
        if (sl == 0) hv = sHy[c];
        else if (sl == 1) hv = (il > 0) ? sHy[c - 1] : hL[jl];
        else if (sl == 2) hv = sHx[c];
        else hv = (jl > 0) ? sHx[c - TX] : hB[il];
        acc += x.w[k] * hv;
      }
      if (x.yo >= 0) acc += yv[r];
      T e = x.c.sub(sEz[c], acc);
      if (x.src >= 0 && step < P.R.n_wave) e -= x.cs * yv[P.maxrows + r];
      sEz[c] = e;
      if (x.yo >= 0) {
        if constexpr (LL) ll_st(P.lG + (int64_t)(ls & P.ymask) * P.ysz + x.yo, (float)e, tag_cur);
        else __stcg(P.G + x.yo, e);
      }
    }
    __syncthreads();
    if (dslot >= 0) P2_STAMP(dslot, 6);
    if constexpr (LL) {
      const int eb_ = ls & 1;
      for (int jl = tid; jl < TY; jl += nthr) ll_st(P.lezL + ((int64_t)eb_ * nT + t) * TY + jl, (float)sEz[jl * TX], tag_cur);
      for (int il = tid; il < TX; il += nthr) ll_st(P.lezB + ((int64_t)eb_ * nT + t) * TX + il, (float)sEz[il], tag_cur);
      if (dslot >= 0) P2_STAMP(dslot, 2);
    } else {
    {
      const int eb_ = ls & 1;
      for (int jl = tid; jl < TY; jl += nthr) __stcg(P.ezL + ((int64_t)eb_ * nT + t) * TY + jl, sEz[jl * TX]);
      for (int il = tid; il < TX; il += nthr) __stcg(P.ezB + ((int64_t)eb_ * nT + t) * TX + il, sEz[il]);
    }
    __syncthreads();
    if (dslot >= 0) P2_STAMP(dslot, 2);
    if (tid == 0) {
      __threadfence();
      st_release_u32(P.fE + t, (unsigned)(ls + 1));
      if (has_if) atomicAdd(P.gready, 1u);
    }
    }
    P2_JITTER(P, 3 * ls + 1);
    // ------------------------------------------------------------- H phase
    auto h_cell = [&](int il, int jl) {
      const int i = i0 + il;
      const int c = jl * TX + il;
      const T ez = sEz[c];
      const T ez_jp = (jl + 1 < TY) ? sEz[c + TX] : eT[il];
      const T ez_ip = (il + 1 < TX) ? sEz[c + 1] : eR[jl];
      Coef<T> cx, cy;
      if (uniform) { cx = P.u1; cy = P.u1; }
      else { const int m = smat[c]; cx = cHx[m]; cy = cHy[m]; }
      const T hx = sHx[c], hy = sHy[c];
      const T hx1 = (i > 0) ? cx.sub(hx, ez_jp - ez) : hx;
      const T hy1 = (j0 + jl > 0) ? cy.add(hy, ez_ip - ez) : hy;
      sHx[c] = hx1; sHy[c] = hy1;
      if (do_check && !(finite_small(ez) && finite_small(hx1) && finite_small(hy1))) bad = true;
    };
    // (a) interior: no E halo needed
    if (pair) {
      const int ia = 2 * lx;
      for (int jl = ly; jl < TY - 1; jl += NLY) {
        if (j0 + jl >= ny) break;
        const int c = jl * TX + ia;
        const float2 ez2 = *reinterpret_cast<const float2*>(sEz + c);
        const float2 ezj2 = *reinterpret_cast<const float2*>(sEz + c + TX);
        const float2 hx2 = *reinterpret_cast<const float2*>(sHx + c);
        const float2 hy2 = *reinterpret_cast<const float2*>(sHy + c);
        const uint16_t m2 = *reinterpret_cast<const uint16_t*>(smat + c);
        float hx0 = hx2.x, hy0 = hy2.x, hx1 = hx2.y, hy1 = hy2.y;
        const bool jin = j0 + jl > 0;
        if (i0 + ia < nx) {
          Coef<T> cx, cy;
          if (uniform) { cx = P.u1; cy = P.u1; }
          else { const int m = m2 & 0xff; cx = cHx[m]; cy = cHy[m]; }
          hx0 = (i0 + ia > 0) ? cx.sub(hx2.x, ezj2.x - ez2.x) : hx2.x;
          hy0 = jin ? cy.add(hy2.x, ez2.y - ez2.x) : hy2.x;
          if (do_check && !(finite_small(ez2.x) && finite_small(hx0) && finite_small(hy0))) bad = true;
        }
        if (ia + 1 < TX - 1 && i0 + ia + 1 < nx) {
          Coef<T> cx, cy;
          if (uniform) { cx = P.u1; cy = P.u1; }
          else { const int m = m2 >> 8; cx = cHx[m]; cy = cHy[m]; }
          hx1 = cx.sub(hx2.y, ezj2.y - ez2.y);
          hy1 = jin ? cy.add(hy2.y, sEz[c + 2] - ez2.y) : hy2.y;
          if (do_check && !(finite_small(ez2.y) && finite_small(hx1) && finite_small(hy1))) bad = true;
        }
        *reinterpret_cast<float2*>(sHx + c) = make_float2(hx0, hx1);
        *reinterpret_cast<float2*>(sHy + c) = make_float2(hy0, hy1);
      }
    } else {
    for (int jl = ly; jl < TY - 1; jl += NLY) {
      if (j0 + jl >= ny) break;
      for (int il = lx; il < TX - 1; il += 32) {
        if (i0 + il >= nx) break;
        h_cell(il, jl);
      }
    }
    }
    // (b) right / top E halos
    if constexpr (LL) {
      const int eb_ = ls & 1;
      bool ok = true;
      for (int q = tid; q < TY + TX && ok; q += nthr) {
        float v = 0.f;
        if (q < TY) {
          if (right >= 0) ok = ll_ld(P.lezL + ((int64_t)eb_ * nT + right) * TY + q, tag_cur, v, P.abort_flag);
          eR[q] = (T)v;
        } else {
          if (top >= 0) ok = ll_ld(P.lezB + ((int64_t)eb_ * nT + top) * TX + (q - TY), tag_cur, v, P.abort_flag);
          eT[q - TY] = (T)v;
        }
      }
      if (!ok) s_abort = 1;
      __syncthreads();
      if (s_abort) break;
      if (dslot >= 0) P2_STAMP(dslot, 3);
    } else {
    if (tid == 0) {
      bool ok = true;
      if (right >= 0) ok = p2_wait(P.fE + right, (unsigned)(ls + 1), P.abort_flag);
      if (ok && top >= 0) ok = p2_wait(P.fE + top, (unsigned)(ls + 1), P.abort_flag);
      if (!ok) s_abort = 1;
    }
    __syncthreads();
    if (s_abort) break;
    if (dslot >= 0) P2_STAMP(dslot, 3);
    {
      const int eb_ = ls & 1;
      for (int jl = tid; jl < TY; jl += nthr)
        eR[jl] = (right >= 0) ? __ldcg(P.ezL + ((int64_t)eb_ * nT + right) * TY + jl) : (T)0;
      for (int il = tid; il < TX; il += nthr)
        eT[il] = (top >= 0) ? __ldcg(P.ezB + ((int64_t)eb_ * nT + top) * TX + il) : (T)0;
    }
    __syncthreads();
    }
    // (c) last column and last row
    for (int q = tid; q < TX + TY - 1; q += nthr) {
      const int il = q < TX ? q : TX - 1, jl = q < TX ? TY - 1 : q - TX;
      if (i0 + il >= nx || j0 + jl >= ny) continue;
      h_cell(il, jl);
    }
    if (bad && first_bad < 0) first_bad = step;
    __syncthreads();
    {
      const int hb_ = ls & 1;
      if constexpr (LL) {
        for (int jl = tid; jl < TY; jl += nthr)
          ll_st(P.lhyR + ((int64_t)hb_ * nT + t) * TY + jl, (float)sHy[jl * TX + TX - 1], tag_cur);
        for (int il = tid; il < TX; il += nthr)
          ll_st(P.lhxT + ((int64_t)hb_ * nT + t) * TX + il, (float)sHx[(TY - 1) * TX + il], tag_cur);
      } else {
        for (int jl = tid; jl < TY; jl += nthr) __stcg(P.hyR + ((int64_t)hb_ * nT + t) * TY + jl, sHy[jl * TX + TX - 1]);
        for (int il = tid; il < TX; il += nthr) __stcg(P.hxT + ((int64_t)hb_ * nT + t) * TX + il, sHx[(TY - 1) * TX + il]);
      }
    }
    // coarse probes owned by this tile (fields after the step)
    for (int q = pr_lo + tid; q < pr_hi; q += nthr) {
      T acc = 0;
      for (int k = P.PR.term_ptr[q]; k < P.PR.term_ptr[q + 1]; ++k) {
        const int c = P.PR.term_li[k], cp = P.PR.term_comp[k];
        const T v = cp == 0 ? sEz[c] : (cp == 1 ? sHx[c] : sHy[c]);
        acc += P.PR.term_w[k] * v;
      }
      P.ring[(step % P.cap) * (int64_t)P.n_probe + P.PR.pid[q]] = acc;
    }
    // fp32 tiles without probes need no barrier here: the next E phase writes
    // only sEz, which nothing after the previous barrier reads (the probe
    // loop would; the flag path needs every halo store before thread 0's release)
    if (!LL || pr_hi > pr_lo) __syncthreads();
    if (dslot >= 0) P2_STAMP(dslot, 4);
    if (!LL && tid == 0) { __threadfence(); st_release_u32(P.fH + t, (unsigned)(ls + 1)); }
  }
  __syncthreads();
  if (!s_abort) {
    for (int jl = ly; jl < TY; jl += NLY)
      for (int il = lx; il < TX; il += 32) {
        const int i = i0 + il, j = j0 + jl;
        if (i >= nx || j >= ny) continue;
        const int64_t o = (int64_t)j * px + i;
        const int c = jl * TX + il;
        P.Fout[0][o] = sEz[c]; P.Fout[1][o] = sHx[c]; P.Fout[2][o] = sHy[c];
      }
    if (t == 0) {
      // constant last column i = nx and row j = ny: Ez = 0 (wall) once stepped, H unchanged
      for (int q = tid; q < (ny + 1) + nx; q += nthr) {
        const int i = q <= ny ? nx : q - (ny + 1), j = q <= ny ? q : ny;
        const int64_t o = (int64_t)j * px + i;
        P.Fout[0][o] = P.nsteps > 0 ? (T)0 : P.Fin[0][o];
        P.Fout[1][o] = P.Fin[1][o]; P.Fout[2][o] = P.Fin[2][o];
      }
      if (tid == 0) *P.d_step_out = P.step0 + P.nsteps;
    }
  }
  if (first_bad >= 0) atomicMin(P.bad_step, (unsigned long long)first_bad);
}

// dedicated reduced CTAs: rows [r_lo, r_hi) of the fused update matrices,
// resident in shared memory for the whole launch
template <typename T>
__device__ void persist2d_reduced(const Persist2D<T>& P, unsigned char* smem_raw, int& s_abort) {
  using V = typename Vec<T>::type;
  constexpr int VN = Vec<T>::n;
  const int rc = blockIdx.x - P.ntx * P.nty;
  T* Xs = reinterpret_cast<T*>(smem_raw);       // [Cmax]
  T* Ms = Xs + P.Cmax;                          // [rpc][Cmax]
  T* Ps = Ms + (size_t)P.rpc * P.Cmax;          // [rpc][32] per-lane partial sums (fp64 runs)
  double* Pd = reinterpret_cast<double*>(Ps + (size_t)P.rpc * 32 + 2);  // fp32 runs: [rpc][32] fp64 partials
  Pd = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(Pd) + 15) & ~(uintptr_t)15);
  uint16_t* Mls = reinterpret_cast<uint16_t*>(Pd + (size_t)P.rpc * 32);   // fp32: [rpc][Cmax] bf16 (R14)
  constexpr bool LO = sizeof(T) == 4;
  const int tid = threadIdx.x, nthr = blockDim.x, lx = tid & 31;
  const int r_lo = min(rc * P.rpc, P.Rtot), r_hi = min(r_lo + P.rpc, P.Rtot);
  for (int g = r_lo; g < r_hi; ++g) {
    int b = 0;
    while (b + 1 < P.nfb && g >= P.row0[b + 1]) ++b;
    const FusedBlock<T>& FB = P.fb[b];
    const T* src = FB.M + (int64_t)(g - P.row0[b]) * FB.Cp;
    for (int c = tid; c < P.Cmax; c += nthr) Ms[(g - r_lo) * P.Cmax + c] = (c < FB.Cp) ? src[c] : (T)0;
    if constexpr (LO) {
      const uint16_t* sl = FB.Ml + (int64_t)(g - P.row0[b]) * FB.Cp;
      for (int c = tid; c < P.Cmax; c += nthr) Mls[(g - r_lo) * P.Cmax + c] = (c < FB.Cp) ? sl[c] : (uint16_t)0;
    }
  }
  __syncthreads();
  long long first_bad = -1;
  for (int ls = 0; ls < P.nsteps; ++ls) {
    const int64_t step = P.step0 + ls;
    const int p = (P.p0 + ls) & 1;
    const bool do_check = P.check_every > 0 && (step % P.check_every) == 0;
    if (rc == 0) P2_STAMP(2, 0);
    P2_JITTER(P, 3 * ls + 2);
    constexpr bool LL = sizeof(T) == 4;
    const unsigned tag_prev = (unsigned)ls, tag_cur = (unsigned)(ls + 1);
    // inputs e~, h~ of this step: every reduced CTA finished the previous one
    // (fp32: the tagged copies are polled word by word below)
    if (!LL) {
      if (tid == 0 && ls > 0 && !p2_wait(P.reddone, (unsigned)(P.n_red_ctas * ls), P.abort_flag)) s_abort = 1;
      __syncthreads();
      if (s_abort) break;
    }
    int g = r_lo;
    bool waited = false;
    while (g < r_hi) {
      int b = 0;
      while (b + 1 < P.nfb && g >= P.row0[b + 1]) ++b;
      const FusedBlock<T>& FB = P.fb[b];
      const int g_end = min(r_hi, P.row0[b + 1]);
      const int qe = FB.qe, ni = FB.n_if, qh = FB.qh, C = FB.C;
      const T* e_in = P.eb[p];
      const T* h_in = P.hb[p];
      const int nv = FB.Cp / VN;
      const int nv_eh = (qe + qh) / VN;            // vectors wholly in the e~, h~ columns
      const int warp = tid >> 5, nw = nthr >> 5;
      // (1) e~, h~ (+ zero padding): the previous reduced step's outputs (fp32:
      //     tagged copies, or the plain state at ls == 0); no wait on G
      {
        const int pl = (ls - 1) & 1;
        bool ok = true;
        for (int c = tid; c < FB.Cp && ok; c += nthr) {
          if (c >= qe + qh && c < C) continue;
          float v = 0.f;
          T tv = 0;
          if (c < qe) {
            if (LL && ls > 0) ok = ll_ld(P.leb + (int64_t)pl * P.esz + FB.e_off + c, tag_prev, v, P.abort_flag, P.sleep_ns), tv = (T)v;
            else tv = __ldcg(e_in + FB.e_off + c);
          } else if (c < qe + qh) {
            if (LL && ls > 0) ok = ll_ld(P.lhb + (int64_t)pl * P.hsz + FB.h_off + (c - qe), tag_prev, v, P.abort_flag, P.sleep_ns), tv = (T)v;
            else tv = __ldcg(h_in + FB.h_off + (c - qe));
          }
          Xs[c] = tv;
        }
        if (!ok) s_abort = 1;
      }
      __syncthreads();
      if (s_abort) break;
      // (2) the e~, h~ part of every row: per-lane partial sums in the same
      //     order as one pass over all columns (the G columns are last)
      for (int gg = g + warp; gg < g_end; gg += nw) {
        const V* a = reinterpret_cast<const V*>(Ms + (gg - r_lo) * P.Cmax);
        if constexpr (LO) {
          const uint2* al = reinterpret_cast<const uint2*>(Mls + (gg - r_lo) * P.Cmax);
          double acd = 0.0;
          for (int cc = lx; cc < nv_eh; cc += 32)
            acd += dot_hilo(reinterpret_cast<const float4*>(a)[cc], bf16x4(al[cc]), reinterpret_cast<const float4*>(Xs)[cc]);
          Pd[(gg - r_lo) * 32 + lx] = acd;
        } else {
          T acc = 0;
          for (int cc = lx; cc < nv_eh; cc += 32) acc += vdot<T>(a[cc], reinterpret_cast<const V*>(Xs)[cc]);
          Ps[(gg - r_lo) * 32 + lx] = acc;
        }
      }
      if (!waited && rc == 0) P2_STAMP(2, 1);
      // (3) G of this step
      if (LL) {
        bool ok = true;
        for (int c = qe + qh + tid; c < C && ok; c += nthr) {
          float v = 0.f;
          ok = ll_ld(P.lG + (int64_t)(ls & P.ymask) * P.ysz + FB.y_off + (c - qe - qh), tag_cur, v, P.abort_flag, P.sleep_ns);
          Xs[c] = (T)v;
        }
        if (!ok) s_abort = 1;
        __syncthreads();
        if (s_abort) break;
      } else {
        if (!waited) {
          if (tid == 0 && !p2_wait(P.gready, (unsigned)(P.n_if_tiles * (ls + 1)), P.abort_flag)) s_abort = 1;
          __syncthreads();
          if (s_abort) break;
        }
        for (int c = qe + qh + tid; c < C; c += nthr) Xs[c] = __ldcg(P.G + FB.y_off + (c - qe - qh));
        __syncthreads();
      }
      if (!waited && rc == 0) P2_STAMP(2, 2);
      waited = true;
      // (4) the rest of every row, reduction, outputs
      for (int gg = g + warp; gg < g_end; gg += nw) {
        const int r = gg - P.row0[b];
        const V* a = reinterpret_cast<const V*>(Ms + (gg - r_lo) * P.Cmax);
        int cc0 = lx;
        while (cc0 < nv_eh) cc0 += 32;
        T acc;
        if constexpr (LO) {
          // compensated matrix, fp64 accumulation of exact fp32 products,
          // rounded once (reading R14)
          const uint2* al = reinterpret_cast<const uint2*>(Mls + (gg - r_lo) * P.Cmax);
          double acd = Pd[(gg - r_lo) * 32 + lx];
#pragma unroll 4
          for (int cc = cc0; cc < nv; cc += 32)
            acd += dot_hilo(reinterpret_cast<const float4*>(a)[cc], bf16x4(al[cc]), reinterpret_cast<const float4*>(Xs)[cc]);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) acd += __shfl_xor_sync(0xffffffffu, acd, o);
          acc = (T)acd;
        } else {
          acc = Ps[(gg - r_lo) * 32 + lx];
#pragma unroll 4
          for (int cc = cc0; cc < nv; cc += 32) acc += vdot<T>(a[cc], reinterpret_cast<const V*>(Xs)[cc]);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        }
        if (lx == 0) {
          const int pc = ls & 1;
          if (r < qh) {
            __stcg(P.hb[p ^ 1] + FB.h_off + r, acc);
            if constexpr (LL) ll_st(P.lhb + (int64_t)pc * P.hsz + FB.h_off + r, (float)acc, tag_cur);
          } else if (r < qh + ni) {
            __stcg(P.y + FB.y_off + (r - qh), acc);
            if constexpr (LL) ll_st(P.ly + (int64_t)(ls & P.ymask) * P.ysz + FB.y_off + (r - qh), (float)acc, tag_cur);
          } else if (r < qh + ni + qe) {
            __stcg(P.eb[p ^ 1] + FB.e_off + (r - qh - ni), acc);
            if constexpr (LL) ll_st(P.leb + (int64_t)pc * P.esz + FB.e_off + (r - qh - ni), (float)acc, tag_cur);
          }
          else {
            const int q = r - qh - ni - qe;
            P.ring[(step % P.cap) * (int64_t)P.n_probe + FB.probe_id[q]] = acc;
          }
          if (do_check && !finite_small((double)acc) && first_bad < 0) first_bad = step;
        }
      }
      __syncthreads();
      g = g_end;
    }
    if (s_abort) break;
    if (rc == 0) P2_STAMP(2, 3);
    if (!LL && tid == 0) { __threadfence(); atomicAdd(P.reddone, 1u); }
  }
  if (first_bad >= 0) atomicMin(P.bad_step, (unsigned long long)first_bad);
}


// ---------------------------------------------------------------------------
// Temporal blocking.  Each tile keeps its TT x TT owned
// cells plus a K-cell halo on every side in shared memory (EX = TT + 2K per
// axis) and advances K steps between two halo exchanges.  Every sub-step
// updates E on extended rows / columns 1..EX-1 and H on 0..EX-2 (all cells
// whose stencil lies inside the extended tile); the values that are exact
// shrink by one cell per half-step from the outside, so after K sub-steps the
// owned region is exact -- every value produced bit for bit as the per-step
// kernels do (same expression, same inputs) -- and the rest of the halo holds
// finite junk until the next exchange overwrites it.  Then every tile
// publishes four K-wide bands of its owned region (tagged LL words, double
// buffered by block parity) and reads its neighbours' bands (edges, corners)
// into its halo.  The interface rows still couple to the reduced CTAs every
// step (G out, y in): a tile evaluates every explicit row of its extended
// region (halo rows redundantly) but only the owner publishes G.  y and G live
// in rings of depth ymask + 1 >= 2 (K + 1): a halo holder may lag the owner by
// up to K steps (one block), the bound that keeps every y slot alive until it
// is read.  fp32 only (the LL words carry 32-bit values); cells in pairs
// (8-byte shared loads), compile-time tile shape.
// ---------------------------------------------------------------------------

// poll n tagged words at once: issue every load, then spin only on the words
// that do not yet carry `tag` (the exchange costs one L2 round trip, not n)
template <int NMAX>
__device__ __forceinline__ bool ll_ld_batch(const unsigned long long* const* p, int n, unsigned tag, float* v,
                                            int* abort_flag, unsigned sleep_ns) {
  unsigned long long w[NMAX];
#pragma unroll
  for (int k = 0; k < NMAX; ++k)
    if (k < n) w[k] = ll_raw(p[k]);
  bool ok = true;
#pragma unroll
  for (int k = 0; k < NMAX; ++k) {
    if (k >= n) continue;
    if ((unsigned)(w[k] >> 32) != tag) {
      float x = 0.f;
      ok = ok && ll_ld(p[k], tag, x, abort_flag, sleep_ns);
      v[k] = x;
    } else {
      v[k] = __uint_as_float((unsigned)w[k]);
    }
  }
  return ok;
}

template <typename T, int TT, int K>
__device__ void persist2d_tb_tile(const Persist2D<T>& P, unsigned char* smem_raw, int& s_abort) {
  static_assert(sizeof(T) == 4, "temporal blocking uses the fp32 LL exchange");
  constexpr int EX = TT + 2 * K, EE = EX * EX;
  constexpr int NPR = EX / 2;                       // cell pairs per extended row
  constexpr int NTHR = 512;
  constexpr int BAND = 3 * K * TT;                  // words per published side
  static_assert(EX % 2 == 0, "pairs");
  const int nT = P.ntx * P.nty;
  const int t = blockIdx.x;
  const int tx_ = t % P.ntx, ty_ = t / P.ntx;
  const int gx0 = tx_ * TT - K, gy0 = ty_ * TT - K;   // global cell of extended (0, 0)
  const int nx = P.nx, ny = P.ny, px = P.px;
  const bool uniform = (P.mat_id == nullptr);
  // every extended cell strictly inside the domain (no wall, no outside cell):
  // the loops need no per-cell domain masks
  const bool inner = gx0 >= 1 && gy0 >= 1 && gx0 + EX <= nx && gy0 + EX <= ny;
  T* sEz = reinterpret_cast<T*>(smem_raw);
  T* sHx = sEz + EE;
  T* sHy = sHx + EE;
  Coef<T>* cE = reinterpret_cast<Coef<T>*>(sHy + EE);
  Coef<T>* cHx = cE + MAX_MAT;
  Coef<T>* cHy = cHx + MAX_MAT;
  uint8_t* ifm = reinterpret_cast<uint8_t*>(cHy + MAX_MAT);
  uint8_t* smat = ifm + MAX_MAT;     // [EE]
  P2Row<T>* rs = reinterpret_cast<P2Row<T>*>(smat + ((EE + 15) / 16) * 16);
  const int tid = threadIdx.x;
  for (int c = tid; c < EE; c += NTHR) {
    const int x = c % EX, y = c / EX;
    const int gi = gx0 + x, gj = gy0 + y;
    T ez = 0, hx = 0, hy = 0;
    uint8_t m = 0;
    if (gi >= 0 && gj >= 0 && gi < nx && gj < ny) {
      const int64_t o = (int64_t)gj * px + gi;
      ez = P.Fin[0][o]; hx = P.Fin[1][o]; hy = P.Fin[2][o];
      if (!uniform) m = P.mat_id[o];
    }
    sEz[c] = ez; sHx[c] = hx; sHy[c] = hy; smat[c] = m;
  }
  if (!uniform) {
    for (int q = tid; q < P.n_mat; q += NTHR) {
      cE[q] = P.gtab[q * 6 + 2]; cHx[q] = P.gtab[q * 6 + 3]; cHy[q] = P.gtab[q * 6 + 4];
      ifm[q] = P.gifm[q];
    }
  }
  // one material on the whole extended tile (most tiles): coefficients from
  // registers, no per-cell table lookups
  __shared__ int s_mmin, s_mmax;
  if (tid == 0) { s_mmin = 255; s_mmax = 0; }
  __syncthreads();
  if (!uniform) {
    int lo_ = 255, hi_ = 0;
    for (int c = tid; c < EE; c += NTHR) { const int m = smat[c]; lo_ = min(lo_, m); hi_ = max(hi_, m); }
    atomicMin(&s_mmin, lo_);
    atomicMax(&s_mmax, hi_);
  }
  const int rows_lo = P.R.tile_ptr[t], rows_hi = P.R.tile_ptr[t + 1];
  const int nrw = rows_hi - rows_lo;
  const bool tile_rows = !uniform && nrw > 0;
  for (int r = rows_lo + tid; r < rows_hi; r += NTHR) {
    P2Row<T> x;
    x.c = P.R.c[r]; x.cs = P.R.cs[r]; x.yo = P.R.yo[r]; x.li = P.R.li[r]; x.src = P.R.src[r];
    x.nterm = P.R.nterm[r]; x.own = P.R.own[r];
    for (int k = 0; k < 4; ++k) { x.w[k] = P.R.w[4 * r + k]; x.slot[k] = P.R.slot[4 * r + k]; }
    rs[r - rows_lo] = x;
  }
  __syncthreads();
  const int pr_lo = P.PR.tile_ptr[t], pr_hi = P.PR.tile_ptr[t + 1];
  const bool hl = tx_ > 0, hr = tx_ + 1 < P.ntx, hb = ty_ > 0, ht = ty_ + 1 < P.nty;
  long long first_bad = -1;
  int ls = 0, blk = 0;
  bool aborted = false;
  const int dslot = (t == 0) ? 0 : (t == P.dbg_tile_if ? 1 : -1);
  // mono: one material (uniform problems included); its coefficients in registers
  const bool mono = uniform || (s_mmin == s_mmax && !tile_rows);
  const int m0 = uniform ? 0 : s_mmin;
  const Coef<T> ce0 = uniform ? P.u0 : cE[m0], cx0 = uniform ? P.u1 : cHx[m0], cy0 = uniform ? P.u1 : cHy[m0];
  constexpr int DY = NTHR / NPR, DP = NTHR % NPR;     // pair-index stride as (rows, pairs)
  while (ls < P.nsteps && !aborted) {
    const int nb = min(K, P.nsteps - ls);
    if (dslot >= 0) P2_STAMP(dslot, 5);
    if (blk > 0) {
      // ---- halo in: the neighbours' owned bands at the end of block blk-1
      //      (edges K x TT, corners K x K, three fields)
      const unsigned tag = (unsigned)blk;
      const unsigned long long* src = P.lband + (size_t)((blk - 1) & 1) * nT * 4 * BAND;
      constexpr int N_EDGE = 4 * BAND, N_ALL = N_EDGE + 4 * 3 * K * K;
      constexpr int PER = (N_ALL + NTHR - 1) / NTHR;
      const unsigned long long* ptr[PER];
      T* dst[PER];
      int n = 0;
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int q = tid + k * NTHR;
        if (q >= N_ALL) continue;
        int nbr = -1, side = 0, f, kk, u, x, y;
        if (q < N_EDGE) {
          const int e = q / BAND, rem = q % BAND;
          f = rem / (K * TT); kk = (rem / TT) % K; u = rem % TT;
          if (e == 0) { if (hl) nbr = t - 1; side = 1; x = kk; y = K + u; }
          else if (e == 1) { if (hr) nbr = t + 1; side = 0; x = K + TT + kk; y = K + u; }
          else if (e == 2) { if (hb) nbr = t - P.ntx; side = 3; x = K + u; y = kk; }
          else { if (ht) nbr = t + P.ntx; side = 2; x = K + u; y = K + TT + kk; }
        } else {
          const int qq = q - N_EDGE;
          const int e = qq / (3 * K * K), rem = qq % (3 * K * K);
          f = rem / (K * K); kk = (rem / K) % K; const int v2 = rem % K;
          // a corner K x K block sits in the diagonal neighbour's left / right band
          if (e == 0) { if (hl && hb) nbr = t - P.ntx - 1; side = 1; x = kk; y = v2; u = TT - K + v2; }
          else if (e == 1) { if (hr && hb) nbr = t - P.ntx + 1; side = 0; x = K + TT + kk; y = v2; u = TT - K + v2; }
          else if (e == 2) { if (hl && ht) nbr = t + P.ntx - 1; side = 1; x = kk; y = K + TT + v2; u = v2; }
          else { if (hr && ht) nbr = t + P.ntx + 1; side = 0; x = K + TT + kk; y = K + TT + v2; u = v2; }
        }
        if (nbr < 0) continue;
        ptr[n] = src + ((size_t)nbr * 4 + side) * BAND + ((size_t)f * K + kk) * TT + u;
        dst[n] = (f == 0 ? sEz : (f == 1 ? sHx : sHy)) + y * EX + x;
        ++n;
      }
      float v[PER];
      const bool ok = ll_ld_batch<PER>(ptr, n, tag, v, P.abort_flag, P.sleep_ns);
#pragma unroll
      for (int k = 0; k < PER; ++k)
        if (k < n) *dst[k] = (T)v[k];
      if (!ok) s_abort = 1;
      __syncthreads();
      if (s_abort) { aborted = true; break; }
    }
    for (int s = 1; s <= nb; ++s, ++ls) {
      const int64_t step = P.step0 + ls;
      const bool do_check = P.check_every > 0 && (step % P.check_every) == 0;
      const unsigned tag_prev = (unsigned)ls, tag_cur = (unsigned)(ls + 1);
      if (dslot >= 0) P2_STAMP(dslot, 0);
      P2_JITTER(P, 3 * ls);
      // ---- E on extended rows 1..EX-1, cell pairs (x, x+1); explicit-row
      //      cells (and x = 0) keep their value here
      auto e_pass = [&](auto MONO) {
        constexpr bool MN = decltype(MONO)::value;
        int y = 1 + tid / NPR, pp = tid % NPR;
        for (; y < EX; y += DY) {
          const int x = 2 * pp;
          const int c = y * EX + x;
          const float2 hy2 = *reinterpret_cast<const float2*>(sHy + c);
          const float2 hx2 = *reinterpret_cast<const float2*>(sHx + c);
          const float2 hxm2 = *reinterpret_cast<const float2*>(sHx + c - EX);
          const float2 ez2 = *reinterpret_cast<const float2*>(sEz + c);
          float e0 = ez2.x, e1 = ez2.y;
          int ma = 0, mb = 0;
          if (!MN) { const uint16_t m2 = *reinterpret_cast<const uint16_t*>(smat + c); ma = m2 & 0xff; mb = m2 >> 8; }
          bool ua = x > 0, ub = true;                 // update cell a / b
          bool za = false, zb = false;                // wall: E = 0
          if (!inner) {
            const int gi = gx0 + x, gj = gy0 + y;
            const bool rowin = gj >= 0 && gj < ny;
            ua = ua && rowin && gi >= 0 && gi < nx;
            ub = rowin && gi + 1 >= 0 && gi + 1 < nx;
            za = gi <= 0 || gj <= 0;
            zb = gi + 1 <= 0 || gj <= 0;
          }
          if (!MN && tile_rows) { ua = ua && !(ifm[ma] & 4); ub = ub && !(ifm[mb] & 4); }
          if (ua) {
            const Coef<T> cc = MN ? ce0 : cE[ma];
            const T dd = (hy2.x - sHy[c - 1]) - (hx2.x - hxm2.x);
            e0 = za ? (T)0 : cc.add(e0, dd);
          }
          if (ub) {
            const Coef<T> cc = MN ? ce0 : cE[mb];
            const T dd = (hy2.y - hy2.x) - (hx2.y - hxm2.y);
            e1 = zb ? (T)0 : cc.add(e1, dd);
          }
          *reinterpret_cast<float2*>(sEz + c) = make_float2(e0, e1);
          pp += DP;
          if (pp >= NPR) { pp -= NPR; ++y; }
        }
      };
      if (mono) e_pass(BoolC<true>{}); else e_pass(BoolC<false>{});
      // the pair stores above write an explicit-row cell's OLD value back: the
      // rows below must start after every warp's pass (found by the jitter
      // test, tests/test_gpu_races.py)
      if (nrw > 0) __syncthreads();
      if (dslot >= 0) P2_STAMP(dslot, 1);
      // ---- explicit rows (eval_row order: terms, y, source); only the owner
      //      publishes E_if into G
      bool ok = true;
      for (int r = tid; r < nrw && ok; r += NTHR) {
        const P2Row<T>& xr = rs[r];
        const int c = xr.li;
        if (c % EX == 0 || c < EX) continue;        // stencil outside the extended tile
        T yvv = 0;
        if (xr.yo >= 0) {
          if (ls == 0) yvv = __ldcg(P.y_in + xr.yo);
          else {
            float v = 0.f;
            ok = ll_ld(P.ly + (int64_t)((ls - 1) & P.ymask) * P.ysz + xr.yo, tag_prev, v, P.abort_flag, P.sleep_ns);
            yvv = (T)v;
          }
        }
        T acc = 0;
        for (int k = 0; k < xr.nterm; ++k) {
          const int sl = xr.slot[k];
          const T hv = sl == 0 ? sHy[c] : (sl == 1 ? sHy[c - 1] : (sl == 2 ? sHx[c] : sHx[c - EX]));
          acc += xr.w[k] * hv;
        }
        if (xr.yo >= 0) acc += yvv;
        T e = xr.c.sub(sEz[c], acc);
        if (xr.src >= 0 && step < P.R.n_wave) e -= xr.cs * P.R.wave[step * P.R.n_cols + xr.src];
        sEz[c] = e;
        if (xr.own && xr.yo >= 0) ll_st(P.lG + (int64_t)(ls & P.ymask) * P.ysz + xr.yo, (float)e, tag_cur);
      }
      if (dslot >= 0) P2_STAMP(dslot, 2);
      if (!ok) s_abort = 1;
      __syncthreads();
      if (s_abort) { aborted = true; break; }
      if (dslot >= 0) P2_STAMP(dslot, 3);
      // ---- H on extended rows 0..EX-2 (the pair's second cell needs x+2 < EX)
      bool bad = false;
      auto h_pass = [&](auto MONO) {
        constexpr bool MN = decltype(MONO)::value;
        int y = tid / NPR, pp = tid % NPR;
        for (; y < EX - 1; y += DY) {
          const int x = 2 * pp;
          const int c = y * EX + x;
          const float2 ez2 = *reinterpret_cast<const float2*>(sEz + c);
          const float2 ezj2 = *reinterpret_cast<const float2*>(sEz + c + EX);
          const float2 hx2 = *reinterpret_cast<const float2*>(sHx + c);
          const float2 hy2 = *reinterpret_cast<const float2*>(sHy + c);
          float hx0 = hx2.x, hy0 = hy2.x, hx1 = hx2.y, hy1 = hy2.y;
          int ma = 0, mb = 0;
          if (!MN) { const uint16_t m2 = *reinterpret_cast<const uint16_t*>(smat + c); ma = m2 & 0xff; mb = m2 >> 8; }
          const bool lastp = x + 2 >= EX;
          bool ua = true, ub = !lastp, xa = true, xb = true, ya = true, yb = true;
          if (!inner) {
            const int gi = gx0 + x, gj = gy0 + y;
            const bool rowin = gj >= 0 && gj < ny;
            ua = rowin && gi >= 0 && gi < nx;
            ub = ub && rowin && gi + 1 >= 0 && gi + 1 < nx;
            xa = gi > 0; xb = gi + 1 > 0;
            ya = gj > 0; yb = ya;
          }
          if (ua) {
            const Coef<T> cx = MN ? cx0 : cHx[ma], cy = MN ? cy0 : cHy[ma];
            hx0 = xa ? cx.sub(hx2.x, ezj2.x - ez2.x) : hx2.x;
            hy0 = ya ? cy.add(hy2.x, ez2.y - ez2.x) : hy2.x;
          }
          if (ub) {
            const Coef<T> cx = MN ? cx0 : cHx[mb], cy = MN ? cy0 : cHy[mb];
            hx1 = xb ? cx.sub(hx2.y, ezj2.y - ez2.y) : hx2.y;
            hy1 = yb ? cy.add(hy2.y, sEz[c + 2] - ez2.y) : hy2.y;
          }
          *reinterpret_cast<float2*>(sHx + c) = make_float2(hx0, hx1);
          *reinterpret_cast<float2*>(sHy + c) = make_float2(hy0, hy1);
          if (do_check && y >= K && y < K + TT && x >= K && x < K + TT) {
            if (ua && !(finite_small(ez2.x) && finite_small(hx0) && finite_small(hy0))) bad = true;
            if (ub && !(finite_small(ez2.y) && finite_small(hx1) && finite_small(hy1))) bad = true;
          }
          pp += DP;
          if (pp >= NPR) { pp -= NPR; ++y; }
        }
      };
      if (mono) h_pass(BoolC<true>{}); else h_pass(BoolC<false>{});
      if (bad && first_bad < 0) first_bad = step;
      __syncthreads();
      if (dslot >= 0) P2_STAMP(dslot, 4);
      if (pr_hi > pr_lo) {
        for (int q = pr_lo + tid; q < pr_hi; q += NTHR) {
          T acc = 0;
          for (int k = P.PR.term_ptr[q]; k < P.PR.term_ptr[q + 1]; ++k) {
            const int c = P.PR.term_li[k], cp = P.PR.term_comp[k];
            const T v = cp == 0 ? sEz[c] : (cp == 1 ? sHx[c] : sHy[c]);
            acc += P.PR.term_w[k] * v;
          }
          P.ring[(step % P.cap) * (int64_t)P.n_probe + P.PR.pid[q]] = acc;
        }
        __syncthreads();
      }
    }
    if (aborted) break;
    // ---- halo out: the owned bands at the end of this block (none after the last)
    if (ls < P.nsteps) {
      const unsigned tag = (unsigned)(blk + 1);
      unsigned long long* dst = P.lband + (size_t)(blk & 1) * nT * 4 * BAND + (size_t)t * 4 * BAND;
      for (int q = tid; q < 4 * BAND; q += NTHR) {
        const int side = q / BAND, rem = q % BAND;
        const int f = rem / (K * TT), kk = (rem / TT) % K, u = rem % TT;
        int x, y;
        if (side == 0) { x = K + kk; y = K + u; }                 // owned columns 0..K-1
        else if (side == 1) { x = TT + kk; y = K + u; }           // owned columns TT-K..TT-1
        else if (side == 2) { x = K + u; y = K + kk; }            // owned rows 0..K-1
        else { x = K + u; y = TT + kk; }                          // owned rows TT-K..TT-1
        const T* srcf = f == 0 ? sEz : (f == 1 ? sHx : sHy);
        ll_st(dst + q, (float)srcf[y * EX + x], tag);
      }
    }
    ++blk;
  }
  __syncthreads();
  if (!s_abort) {
    for (int c = tid; c < TT * TT; c += NTHR) {
      const int x = c % TT, y = c / TT;
      const int i = tx_ * TT + x, j = ty_ * TT + y;
      if (i >= nx || j >= ny) continue;
      const int64_t o = (int64_t)j * px + i;
      const int e = (y + K) * EX + x + K;
      P.Fout[0][o] = sEz[e]; P.Fout[1][o] = sHx[e]; P.Fout[2][o] = sHy[e];
    }
    if (t == 0) {
      for (int q = tid; q < (ny + 1) + nx; q += NTHR) {
        const int i = q <= ny ? nx : q - (ny + 1), j = q <= ny ? q : ny;
        const int64_t o = (int64_t)j * px + i;
        P.Fout[0][o] = P.nsteps > 0 ? (T)0 : P.Fin[0][o];
        P.Fout[1][o] = P.Fin[1][o]; P.Fout[2][o] = P.Fin[2][o];
      }
      if (tid == 0) *P.d_step_out = P.step0 + P.nsteps;
    }
  }
  if (first_bad >= 0) atomicMin(P.bad_step, (unsigned long long)first_bad);
}

// TBK > 0: temporal blocking with TBT x TBT tiles and K = TBK (fp32)
template <typename T, int TBT = 0, int TBK = 0>
__global__ void __launch_bounds__(512, 2)
persist2d_kernel(const __grid_constant__ Persist2D<T> P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_abort;
  if (threadIdx.x == 0) s_abort = 0;
  __syncthreads();
  if ((int)blockIdx.x < P.ntx * P.nty) {
    if constexpr (TBK > 0) persist2d_tb_tile<T, TBT, TBK>(P, smem_raw, s_abort);
    else persist2d_tile<T>(P, smem_raw, s_abort);
  } else {
    persist2d_reduced<T>(P, smem_raw, s_abort);
  }
}

}  // namespace fdtd
