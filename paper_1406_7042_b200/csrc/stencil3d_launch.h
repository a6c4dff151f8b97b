// stencil3d_launch.h — host interface of the 3-D tile stencil (stencil3d.cu).
#pragma once
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace fdtd {

struct TileCfg {
  int W = 2;          // elements per thread (16 or 8 bytes)
  int NS = 4;         // TMA ring stages (planes in flight)
  int BY = 8;         // tile rows (one warp per row; TILE_BY)
  int MB = 0;         // 0: W x cells per thread (batch 1); > 0: batch of MB members, W per thread
};

template <typename T>
bool tile_supported(const TileCfg& c);
template <typename T>
cudaError_t tile_prepare(const TileCfg& c, size_t smem);
struct TileSplit {
  int ntx, outx, outy, nzp;      // tiles in x, tile pitch in cells (x, y), nz + 1
  int ncols, kc, nitems;         // tiles, planes per z-chunk, items = tiles * chunks
  // optional column subset: the launch covers columns colperm[col0 .. col0 +
  // ncols) (the interface columns or the rest); null: all
  const int* colperm = nullptr;
  int col0 = 0;
  // race testing (FDTD_JITTER=ns): every warp sleeps a pseudo-random 0..jitter
  // ns before each plane, shaking the warp / TMA interleaving; results must
  // stay bitwise identical (tests/test_gpu_races.py)
  int jitter = 0;
  __host__ __device__ __forceinline__ int column(int c) const { return colperm ? colperm[col0 + c] : c; }
};

template <typename T>
cudaError_t tile_launch(const TileCfg& c, bool uniform, int grid, size_t smem, cudaStream_t st, const TmaSet& tm,
                        const TileSplit& split, Dims d, Fields<T> F0, Fields<T> F1, const uint8_t* mat_id,
                        const Coef<T>* tab, const uint8_t* ifm, int n_mat, Coef<T> u0, Coef<T> u1, RowsE<T> rows,
                        const T* y, const int64_t* ds, int check_every, unsigned long long* bad,
                        const T* taba = nullptr);    // taba: [n_mat][6] ca / da (lossy media), null: lossless
template <typename T>
int tile_blocks_per_sm(const TileCfg& c, bool uniform, size_t smem);

// shared-memory bytes of one CTA (the layout of stencil3d_tile_kernel)
inline size_t tile_hp_elems(int HBX, int BY, int esz) { return ((size_t)HBX * (BY + 1) * esz + 127) / 128 * 128 / esz; }
inline size_t tile_ep_elems(int RX, int BY, int esz) { return ((size_t)RX * BY * esz + 127) / 128 * 128 / esz; }
inline size_t tile_smem_bytes(const TileCfg& c, int HBX, int esz, size_t tabsz) {
  const int RX = 32 * c.W;
  return 256 + (size_t)esz * ((size_t)c.NS * 3 * (tile_hp_elems(HBX, c.BY, esz) + tile_ep_elems(RX, c.BY, esz)) +
                              2 * 3 * tile_ep_elems(RX, c.BY, esz)) + tabsz;
}

}  // namespace fdtd
