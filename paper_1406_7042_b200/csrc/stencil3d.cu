// stencil3d.cu — instantiations and launcher of the 3-D tile stencil
// (stencil3d.cuh), a separate translation unit so it compiles in parallel with
// fdtd_api.cu.
#include "stencil3d.cuh"
#include "stencil3d_launch.h"

namespace fdtd {

namespace {

template <typename T, int NS, int W, int MB, int MINB, int BY = TILE_BY>
struct TileKernels {
  static constexpr auto uni = &stencil3d_tile_kernel<T, true, NS, W, MB, MINB, BY>;
  static constexpr auto mat = &stencil3d_tile_kernel<T, false, NS, W, MB, MINB, BY>;
  static constexpr auto lossy = &stencil3d_tile_kernel<T, false, NS, W, MB, MINB, BY, true>;
};

template <typename T, typename F>
bool tile_dispatch(const TileCfg& c, F&& f) {
  // the instantiated variants: B == 1 tiles of 32*W x cells, batched tiles of W members
  if (c.BY == 16) {
    // 16-row tiles (512 threads): 15 of 16 rows owned instead of 7 of 8
    if constexpr (sizeof(T) == 4) {
      if (c.MB == 0 && c.W == 2 && c.NS == 4) { f(TileKernels<T, 4, 2, 0, 1, 16>{}); return true; }
      if (c.MB == 16 && c.W == 4 && c.NS == 3) { f(TileKernels<T, 3, 4, 16, 1, 16>{}); return true; }
    } else {
      if (c.MB == 0 && c.W == 1 && c.NS == 4) { f(TileKernels<T, 4, 1, 0, 1, 16>{}); return true; }
    }
    return false;
  }
  if (c.BY != TILE_BY) return false;
  if constexpr (sizeof(T) == 4) {
    if (c.MB == 0 && c.W == 2 && c.NS == 4) { f(TileKernels<T, 4, 2, 0, 3>{}); return true; }
    if (c.MB == 0 && c.W == 2 && c.NS == 6) { f(TileKernels<T, 6, 2, 0, 2>{}); return true; }
    if (c.MB == 0 && c.W == 4 && c.NS == 3) { f(TileKernels<T, 3, 4, 0, 2>{}); return true; }
    if (c.MB == 0 && c.W == 1 && c.NS == 6) { f(TileKernels<T, 6, 1, 0, 3>{}); return true; }
    if (c.MB == 16 && c.W == 4 && c.NS == 3) { f(TileKernels<T, 3, 4, 16, 2>{}); return true; }
  } else {
    if (c.MB == 0 && c.W == 2 && c.NS == 3) { f(TileKernels<T, 3, 2, 0, 2>{}); return true; }
    if (c.MB == 0 && c.W == 1 && c.NS == 6) { f(TileKernels<T, 6, 1, 0, 2>{}); return true; }
    if (c.MB == 16 && c.W == 2 && c.NS == 3) { f(TileKernels<T, 3, 2, 16, 2>{}); return true; }
  }
  return false;
}

}  // namespace

template <typename T>
bool tile_supported(const TileCfg& c) {
  return tile_dispatch<T>(c, [](auto) {});
}

template <typename T>
cudaError_t tile_prepare(const TileCfg& c, size_t smem) {
  cudaError_t err = cudaErrorInvalidValue;
  // the attribute is per function, not per handle: several handles with different
  // table sizes coexist (slab decomposition), so always allow the device maximum
  int dev = 0, optin = 0;
  if (cudaGetDevice(&dev) == cudaSuccess &&
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) == cudaSuccess && (size_t)optin > smem)
    smem = (size_t)optin;
  tile_dispatch<T>(c, [&](auto K) {
    err = cudaFuncSetAttribute(K.uni, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err == cudaSuccess) err = cudaFuncSetAttribute(K.mat, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err == cudaSuccess) err = cudaFuncSetAttribute(K.lossy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  return err;
}

template <typename T>
cudaError_t tile_launch(const TileCfg& c, bool uniform, int grid, size_t smem, cudaStream_t st, const TmaSet& tm,
                        const TileSplit& split, Dims d, Fields<T> F0, Fields<T> F1, const uint8_t* mat_id,
                        const Coef<T>* tab, const uint8_t* ifm, int n_mat, Coef<T> u0, Coef<T> u1, RowsE<T> rows,
                        const T* y, const int64_t* ds, int check_every, unsigned long long* bad, const T* taba) {
  cudaError_t err = cudaErrorInvalidValue;
  tile_dispatch<T>(c, [&](auto K) {
    const auto fn = uniform ? K.uni : (taba ? K.lossy : K.mat);
    fn<<<grid, dim3(32, c.BY), smem, st>>>(tm, split, d, F0, F1, mat_id, tab, ifm, n_mat, u0, u1, rows, y, ds,
                                          check_every, bad, taba);
    err = cudaGetLastError();
  });
  return err;
}

template <typename T>
int tile_blocks_per_sm(const TileCfg& c, bool uniform, size_t smem) {
  int nb = 0;
  tile_dispatch<T>(c, [&](auto K) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, uniform ? K.uni : K.mat, 32 * c.BY, smem) != cudaSuccess)
      nb = 0;
  });
  return nb;
}

#define FDTD_TILE_INST(T)                                                                                        \
  template bool tile_supported<T>(const TileCfg&);                                                               \
  template cudaError_t tile_prepare<T>(const TileCfg&, size_t);                                                  \
  template cudaError_t tile_launch<T>(const TileCfg&, bool, int, size_t, cudaStream_t, const TmaSet&,              \
                                      const TileSplit&, Dims, Fields<T>, Fields<T>, const uint8_t*, const Coef<T>*, \
                                      const uint8_t*, int, Coef<T>, Coef<T>, RowsE<T>, const T*, const int64_t*,  \
                                      int, unsigned long long*, const T*);                                                 \
  template int tile_blocks_per_sm<T>(const TileCfg&, bool, size_t);
FDTD_TILE_INST(float)
FDTD_TILE_INST(double)

}  // namespace fdtd
