// fdtd_api.cu — the C ABI of include/fdtd.h: validation, upload, step
// orchestration (eager launches or captured CUDA graphs), probes, state.
//
// Reduced blocks run in one of two forms:
//  * fused   (small blocks): the three leap-frog half-updates of a step,
//            h~' = h~ + G_h(K~'^T e~ + S_E^T G), y' = S_E h~', e~'' = e~' - G_e K~' h~'
//            are composed on the host (fp64) into one update matrix applied by a
//            single GEMV phase per step (identical in exact arithmetic);
//  * leapfrog (large blocks, S_E of 10^5 rows): grid-wide GEMV launches in the
//            paper's order.
#include "../../include/fdtd.h"
#include "kernels.cuh"
#include "persist2d.cuh"
#include "stencil3d_launch.h"
#include "tc_gemm.cuh"

#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

}  // namespace
namespace fdtd {
// the thread-local message of fdtd_last_error(), for the other translation units (rom.cu)
int set_error(int code, const char* msg) { return fail(code, "%s", msg); }
}  // namespace fdtd
namespace {


// cudaFuncAttributeMaxDynamicSharedMemorySize is per function, not per handle:
// handles with different shared-memory needs coexist (slab decomposition, the
// tests), so a function's limit only ever grows.
template <typename F>
cudaError_t raise_smem_limit(F fn, int bytes) {
  static std::map<const void*, int> seen;
  int& cur = seen[(const void*)fn];
  if (bytes <= cur) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) cur = bytes;
  return e;
}

#define CK(call)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return fail(FDTD_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                             \
  } while (0)

template <typename T>
fdtd::Coef<T> make_coef(double c);
template <>
fdtd::Coef<float> make_coef<float>(double c) {
  fdtd::Coef<float> r;
  r.hi = (float)c;
  r.lo = (float)(c - (double)r.hi);   // hi/lo split of the fp64 coefficient (R11, F12)
  return r;
}
template <>
fdtd::Coef<double> make_coef<double>(double c) {
  fdtd::Coef<double> r;
  r.hi = c;
  r.lo = 0.0;
  return r;
}

}  // namespace

// ---------------------------------------------------------------------------
struct fdtd_t {
  virtual ~fdtd_t() {}
  virtual int step(int64_t n) = 0;
  virtual int probe(double* out, int64_t cap, int64_t* written) = 0;
  virtual int get_state(int which, double* out, int64_t n) = 0;
  virtual int set_state(int which, const double* in, int64_t n) = 0;
  virtual int sync() = 0;
  virtual int set_profile(int on) = 0;
  virtual int phase_times(double* ms, int n) = 0;
  virtual int plane_io(int which, int k, void* buf, int dir) = 0;
  int64_t launches = 0;
  int32_t path_bits = 0;
};

namespace {

struct DevMem {
  void* (*alloc)(size_t, void*) = nullptr;
  void (*free_)(void*, void*) = nullptr;
  void* ctx = nullptr;
  std::vector<void*> owned;
  // FDTD_GUARD=1 (debugging): every buffer sits between two 64 KB guard zones
  // filled with 0xA5; check() (called by fdtd_sync) reports the first buffer whose
  // guards a kernel has written -- out-of-bounds stores next to a buffer, which
  // the serial step order can hide (a later kernel rewrites the victim)
  static constexpr size_t GUARD = 64 * 1024;
  bool guard = getenv("FDTD_GUARD") != nullptr;
  // the fill byte: FDTD_GUARD=1 -> 0xA5 (a tiny finite float); FDTD_GUARD=255 -> 0xFF (NaN in fp32 and fp64: an
  // out-of-bounds READ that reaches the arithmetic then poisons the fields and trips the divergence check)
  int pat = (getenv("FDTD_GUARD") && atoi(getenv("FDTD_GUARD")) > 1) ? (atoi(getenv("FDTD_GUARD")) & 0xff) : 0xA5;
  std::vector<size_t> sizes;
  ~DevMem() {
    for (void* p : owned) {
      if (free_) free_(p, ctx);
      else cudaFree(p);
    }
  }
  void* get(size_t bytes) {
    if (bytes == 0) bytes = 16;
    const size_t total = guard ? ((bytes + 255) / 256 * 256 + 2 * GUARD) : bytes;
    void* p = nullptr;
    if (alloc) p = alloc(total, ctx);
    else if (cudaMalloc(&p, total) != cudaSuccess) p = nullptr;
    if (!p) return nullptr;
    owned.push_back(p);
    sizes.push_back(bytes);
    if (!guard) return p;
    cudaMemset(p, pat, GUARD);
    cudaMemset((char*)p + total - GUARD - ((bytes + 255) / 256 * 256 - bytes), pat,
               GUARD + ((bytes + 255) / 256 * 256 - bytes));
    return (char*)p + GUARD;
  }
  // index of the first buffer with a damaged guard (-1: none); *where: byte offset relative to the buffer start
  int check(long long* where) const {
    if (!guard) return -1;
    std::vector<unsigned char> h;
    for (size_t b = 0; b < owned.size(); ++b) {
      const size_t bytes = sizes[b], pad = (bytes + 255) / 256 * 256;
      const size_t tail = GUARD + (pad - bytes);
      h.resize(GUARD + tail);
      cudaMemcpy(h.data(), owned[b], GUARD, cudaMemcpyDeviceToHost);
      cudaMemcpy(h.data() + GUARD, (char*)owned[b] + GUARD + bytes, tail, cudaMemcpyDeviceToHost);
      for (size_t i = 0; i < GUARD; ++i)
        if (h[i] != (unsigned char)pat) { *where = (long long)i - (long long)GUARD; return (int)b; }
      for (size_t i = 0; i < tail; ++i)
        if (h[GUARD + i] != (unsigned char)pat) { *where = (long long)(bytes + i); return (int)b; }
    }
    return -1;
  }
};

// per reduced model
template <typename T>
struct BlockDev {
  int qe = 0, qh = 0, n_inst = 0, n_if = 0, N = 0;
  bool fused = false;
  // host fp64 copies (for the prologue and the fused matrix)
  std::vector<double> K, SE, ge, gh;
  // unpadded matrices (fused blocks: prologue GEMVs) and padded-row copies
  // (leap-frog blocks: 16-byte vector loads)
  T *K_d = nullptr, *KT_d = nullptr, *SE_d = nullptr, *SET_d = nullptr, *ge_d = nullptr, *gh_d = nullptr;
  T *Kp_d = nullptr, *KTp_d = nullptr, *SEp_d = nullptr;
  double* Tv_d = nullptr;                      // K~'^T e~ + S_E^T G, unrounded (R14)
  double* part_d = nullptr;                    // [ks + splits][qh][N] K~'^T e~ and S_E^T G partial sums (fp32 GEMM path, fp64)
  double* parte_d = nullptr;                   // [ks][qe][N] K~' h~ partial sums
  T* gen_d = nullptr;                          // -g_e (the e~ update as an axpy)
  int ks = 0;                                  // row splits of the K~' products
  bool tc = false;                             // y = S_E h~ on the tensor cores (tc_gemm.cuh, 3xTF32, N = 16)
  CUtensorMap se_map;                          // TMA map of SEp_d: [n_if][Kph] fp32, 32 x 128 boxes, 128-byte swizzle
  float* xs_d = nullptr;                       // h~ split for the tensor cores: [ceil(qh/32)][hi 512 | lo 512]
  int splits = 0;                              // > 0: tall-skinny fp32 GEMM kernels for the S_E products
  bool wide = false;                           // S_E^T G on gemm_tn_f32_wide_kernel (N = 16)
  int wide_ng = 2;                             // its member groups per column octet (2: 256 threads, measured 143 us on
                                               // config 4; 4: 512 threads, 147 us; FDTD_WIDE_NG)
  int Kph = 0, Kpe = 0;                        // padded row pitches (multiples of 32 * VEC)
  // state offsets (elements) in the concatenated buffers
  int64_t e_off = 0, h_off = 0, y_off = 0;     // e/h buffers [q][N], y / G [n_if][N]
  // fused path
  T* M_d = nullptr;                            // [R_M][C_M]
  int R_M = 0, C_M = 0;
  std::vector<int> probe_rows;                 // global probe ids realised as rows of M
};

template <typename T>
struct Impl : public fdtd_t {
  // grid
  int dim = 3, nx = 0, ny = 0, nz = 0, B = 1, px = 0;
  int64_t S = 0;          // storage indices per component (unpadded)
  int64_t plane = 0;      // (ny+1)*px
  int64_t nplanes = 0;    // nz+1 (3-D) or 1 (2-D)
  int64_t elems = 0;      // device elements per component (plane*nplanes*B)
  cudaStream_t stream = nullptr;
  DevMem mem;
  T* F[2][6] = {{nullptr}};
  // materials
  bool uniform = true;
  int n_mat = 0;
  uint8_t* mat_id = nullptr;
  fdtd::Coef<T>* tab = nullptr;
  uint8_t* ifm = nullptr;
  T* tab_a = nullptr;                 // [n_mat][6] ca / da of lossy media (fdtd.h coef_a), null: lossless
  bool lossy = false;
  fdtd::Coef<T> u0{}, u1{};
  // explicit rows
  fdtd::RowsE<T> rows{};
  // reduced blocks
  std::vector<BlockDev<T>> blocks;
  bool any_fused = false, any_leap = false;
  T* eb[2] = {nullptr, nullptr};      // e~ (fused: [state, ahead] by parity; leapfrog: eb[0])
  T* hb[2] = {nullptr, nullptr};      // h~ (fused: by parity; leapfrog: hb[0])
  T* y_all = nullptr;
  T* g_all = nullptr;                 // gathered interface E (leapfrog path)
  int64_t e_size = 0, h_size = 0, y_size = 0;
  // gather lists: per block, (comp, storage offset, dst index in [n_if][N])
  int64_t n_gather = 0;
  int32_t* g_comp = nullptr;
  int64_t* g_off = nullptr;
  int64_t* g_dst = nullptr;
  // fused kernel work decomposition
  std::vector<fdtd::FusedBlock<T>> fblocks;   // descriptors (copied into the kernel parameters)
  std::vector<int> tile0;                     // first tile of each fused block
  int n_ctas = 0, NBsel = 1, max_cols = 0, rows_per_cta = 8;
  bool fused_gemm = false;
  int NPsel = 32;
  static constexpr int GEMM_KS = 4;
  int gks = GEMM_KS;            // cluster K-split of the fused GEMM (N = 32: 8 by default, FDTD_GEMM_KS = 2 | 4 | 8)
  // rows per thread of the GEMM kernel: 64-row tiles for NP <= 16, 32 for NP = 32
  static constexpr int gemm_rpw(int np) { return np == 32 ? 2 : np / 4; }
  int64_t step_offset = 0;            // device step = host step + offset (set_state(8))
  size_t fused_smem = 0;
  // probes
  fdtd::Probes<T> pr{};
  int n_probe = 0;
  T* ring = nullptr;
  int64_t cap = 65536;
  std::vector<double> host_probes;
  int64_t drained_to = 0;
  // control
  int64_t* d_step = nullptr;
  unsigned long long* d_bad = nullptr;
  unsigned int* d_done = nullptr;
  int64_t host_step = 0;
  int check_every = 100;
  int graph_steps = 32;
  cudaGraphExec_t graph = nullptr;
  int64_t graph_kernels = 0;
  T* staging = nullptr;
  size_t staging_bytes = 0;
  double* d_in64 = nullptr;          // device copy of a set_state input (fp64)
  int64_t d_in64_n = 0;
  int kchunk_max = 32;         // z-planes per CTA of the 3-D stencils (upper bound)
  // z-chunk: at most kchunk_max planes, at least ~2 waves of CTAs (148 SMs x 3
  // resident), chunks balanced (config 5: 41 planes -> 3 x 14, not 32 + 9)
  int zchunk(int gxy) const {
    int nch = std::max((nz + 1 + kchunk_max - 1) / kchunk_max, (2 * 148 * 3 + gxy - 1) / gxy);
    nch = std::max(1, std::min(nch, (nz + 1 + 7) / 8));
    return (nz + 1 + nch - 1) / nch;
  }
  int reduced_form = 0;
  // TMA descriptors of the 3-D stencil (per parity of the OLD buffers)
  bool use_tma = false;
  fdtd::TmaSet tma[2];
  int tBX = 32, tBY = 8, tHBX = 36, tSX = 4, tOUTX = 28;
  int tW = 1;                   // members per thread in the TMA stencil (16 bytes when the batch allows)
  bool use_tile = false;        // the tile stencil (stencil3d.cuh) is the 3-D path
  fdtd::TileCfg tcfg;
  fdtd::TileSplit tsplit;
  int tc_grid = 148;            // CTAs of the tensor-core skinny GEMM (one per SM, persistent over row tiles)
  bool use_pdl = false;         // the fused reduced kernel as a programmatic dependent launch (FDTD_PDL=1;
                                // measured: config 5 -2 %, config 3 +0.2 %)
  int tile_grid = 0;
  size_t tile_smem = 0;
  static constexpr int kW = 16 / (int)sizeof(T);
  int64_t guard = 0;                  // elements allocated before each field (TMA halo base)
  // per-phase tracing
  static constexpr int NPHASE = 3;       // stencil (+ explicit rows), reduced (+ probes), leapfrog GEMVs
  bool prof = false;
  // event sets of up to NPOOL profiled steps are read back together, so the
  // stream stays busy and the spans are kernel durations, not launch latencies
  static constexpr int NPOOL = 64;
  std::vector<cudaEvent_t> ev;         // [NPOOL][2 * NPHASE]
  int prof_pending = 0;
  // split step: the stencil items of the columns that hold
  // interface rows run first, the reduced update runs on a second stream
  // beside the rest of the stencil
  // explicit rows fused into the reduced GEMM: the thread of
  // reduced_gemm_kernel that finalises a y element evaluates that element's
  // explicit row of the NEXT step, so the pre-pass launch disappears in steady
  // state.  rows_ahead: the rows of the step about to run are already evaluated
  // (false after create / set_state / fdtd_plane_device writes / a profiled step)
  bool fuse_rows = false, rows_ahead = false;
  T* g_alt = nullptr;                  // G of the other step parity (the reduced kernel reads one, writes the next)
  int32_t* y_row_d = nullptr;          // [y_size / B] explicit row of each y element (-1: none)
  int32_t* src_rows_d = nullptr;       // explicit rows without a y term
  int n_src_rows = 0;
  bool split = false;
  int n_ifc = 0;                       // interface columns (first in colperm)
  int* colperm_d = nullptr;
  fdtd::RowPackI* rowpack_i = nullptr;      // packed explicit rows (rows_prepass_packed_kernel), null: generic
  void* rowpack_r = nullptr;
  std::vector<std::pair<int, int>> split_rows;     // (i, j) of the explicit rows that read y
  cudaStream_t st2 = nullptr;
  cudaEvent_t evA = nullptr, evR = nullptr;
  double phase_ms[NPHASE] = {0};
  int64_t phase_n[NPHASE] = {0};

  ~Impl() override {
    if (graph) cudaGraphExecDestroy(graph);
    if (staging) cudaFreeHost(staging);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
  }
  int flush_profile() {
    if (prof_pending == 0) return FDTD_OK;
    CK(cudaEventSynchronize(ev[(size_t)(prof_pending - 1) * 2 * NPHASE + 3]));
    for (int q = 0; q < prof_pending; ++q)
      for (int ph = 0; ph < NPHASE; ++ph) {
        if (ph == 2 && !any_leap) continue;
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, ev[(size_t)q * 2 * NPHASE + 2 * ph], ev[(size_t)q * 2 * NPHASE + 2 * ph + 1]));
        phase_ms[ph] += ms;
        phase_n[ph] += 1;
      }
    prof_pending = 0;
    return FDTD_OK;
  }
  int set_profile(int on) override {
    if (on && ev.empty()) {
      ev.assign((size_t)NPOOL * 2 * NPHASE, nullptr);
      for (auto& e : ev) CK(cudaEventCreate(&e));
    }
    int e = flush_profile();
    if (e) return e;
    prof = on != 0;
    for (int i = 0; i < NPHASE; ++i) { phase_ms[i] = 0; phase_n[i] = 0; }
    return FDTD_OK;
  }
  // one z-plane of a coarse component <-> a contiguous device buffer [ny+1][nx+1][B]
  // (halo exchange of the slab decomposition, fdtd.h fdtd_plane_device)
  int plane_io(int which, int k, void* buf, int dir) override {
    if (dim != 3) return fail(FDTD_ENOTSUP, "fdtd_plane_device: 3-D problems only");
    if (which < 0 || which > 5 || k < 0 || k > nz || !buf || (dir != 0 && dir != 1))
      return fail(FDTD_EINVAL, "fdtd_plane_device: bad component / plane / buffer / direction");
    T* f = F[(int)(host_step & 1)][which] + (int64_t)k * plane * B;
    const size_t w = (size_t)(nx + 1) * B * sizeof(T), pitch = (size_t)px * B * sizeof(T);
    if (dir == 0) CK(cudaMemcpy2DAsync(buf, w, f, pitch, w, (size_t)(ny + 1), cudaMemcpyDeviceToDevice, stream));
    else {
      CK(cudaMemcpy2DAsync(f, pitch, buf, w, w, (size_t)(ny + 1), cudaMemcpyDeviceToDevice, stream));
      rows_ahead = false;
    }
    return FDTD_OK;
  }
  int phase_times(double* ms, int n) override {
    int e = flush_profile();
    if (e) return e;
    for (int i = 0; i < n && i < NPHASE; ++i) ms[i] = phase_n[i] ? phase_ms[i] : 0.0;
    for (int i = NPHASE; i < n; ++i) ms[i] = 0.0;
    if (n > NPHASE) ms[NPHASE] = (double)phase_n[0];
    return FDTD_OK;
  }

  template <typename U>
  U* dalloc(int64_t count) {
    return reinterpret_cast<U*>(mem.get(sizeof(U) * (size_t)count));
  }
  template <typename V>
  int upload(void* dst, const std::vector<V>& v) {
    if (!v.empty()) CK(cudaMemcpy(dst, v.data(), sizeof(V) * v.size(), cudaMemcpyHostToDevice));
    return FDTD_OK;
  }

  int64_t dev_off(int64_t s) const {   // storage index -> device storage offset (before *B)
    int64_t i = s % (nx + 1), j, k;
    if (dim == 3) {
      j = (s / (nx + 1)) % (ny + 1);
      k = s / ((int64_t)(nx + 1) * (ny + 1));
    } else {
      j = s / (nx + 1);
      k = 0;
    }
    return (k * (ny + 1) + j) * px + i;
  }

  bool is_e(int c) const { return dim == 3 ? (c >= 0 && c <= 2) : c == 2; }
  bool is_h(int c) const { return dim == 3 ? (c >= 3 && c <= 5) : (c == 3 || c == 4); }

  // reduced-state pointers for host access: a fused block keeps
  // e~ one step ahead, so after s steps e~^s = eb[(s+1)&1], e~^{s+1} = eb[s&1],
  // h~^{s+1/2} = hb[s&1]; a leap-frog block updates eb[0] / hb[0] in place.
  T* e_state(const BlockDev<T>& D, int64_t s) const { return (D.fused ? eb[(s + 1) & 1] : eb[0]) + D.e_off; }
  T* e_ahead(const BlockDev<T>& D, int64_t s) const { return eb[s & 1] + D.e_off; }
  T* h_state(const BlockDev<T>& D, int64_t s) const { return (D.fused ? hb[s & 1] : hb[0]) + D.h_off; }

  int create(const fdtd_grid* g, const fdtd_materials* mat, const fdtd_interface* itf,
             const fdtd_reduced_block* bl, int n_blocks, const fdtd_sources* src,
             const fdtd_probes* probes, const fdtd_exec* ex);
  // ---- persistent 2-D path (persist2d.cuh) ----
  struct XRow { int comp; int64_t s; double c; std::vector<std::pair<int64_t, double>> w; int64_t y; int src_col; double cs; };
  std::vector<XRow> xrows;                          // explicit rows (host copy)
  std::vector<int32_t> hpr_src, hpr_owner;          // coarse probes (host copy)
  std::vector<int64_t> hpr_off, hpr_rp;
  std::vector<double> hpr_w;
  bool persist = false;
  int p_maxrows = 0;
  int p_K = 0, p_D = 2;                             // temporal blocking: halo depth K, y / G ring depth D
  const void* p_kfn = nullptr;                      // the persist2d_kernel instantiation launched
  T* p_yin = nullptr;                               // y before the launch (persist2d.cuh, fp32)
  static const void* p2_kernel(int TX, int K) {
    if constexpr (sizeof(T) == 4) {
      if (TX == 64 && K == 4) return (const void*)fdtd::persist2d_kernel<T, 64, 4>;
      if (TX == 64 && K == 2) return (const void*)fdtd::persist2d_kernel<T, 64, 2>;
      if (TX == 32 && K == 4) return (const void*)fdtd::persist2d_kernel<T, 32, 4>;
      if (TX == 32 && K == 2) return (const void*)fdtd::persist2d_kernel<T, 32, 2>;
    }
    return (const void*)fdtd::persist2d_kernel<T>;
  }
  int pTX = 0, pTY = 0, pntx = 0, pnty = 0, p_nif_tiles = 0, p_nred = 0, p_Rtot = 0, p_rpc = 0, p_Cmax = 0;
  int p_row0[fdtd::kMaxFusedBlocks + 1] = {};
  size_t p_smem = 0;
  fdtd::P2Rows<T> p_rows{};
  fdtd::P2Probes<T> p_probes{};
  T *p_ezL = nullptr, *p_ezB = nullptr, *p_hyR = nullptr, *p_hxT = nullptr;
  unsigned* p_flags = nullptr;                      // fE[nT] fH[nT] gready reddone abort
  unsigned long long* p_ll = nullptr;               // fp32 flag-in-data exchange buffers (persist2d.cuh)
  size_t p_ll_words = 0;
  uint8_t* p_tile_if = nullptr;
  int setup_persist();
  int launch_persist(int64_t n, int64_t* count);
  int build_fused(const fdtd_probes* probes);
  int prepass(int p, cudaStream_t st);
  // G of the step of parity p: one buffer, or two with fused rows (the reduced
  // kernel reads this step's while it writes the next step's)
  T* g_of(int p) const { return (fuse_rows && p) ? g_alt : g_all; }
  int prologue(cudaStream_t st);
  int launch_step(int parity, cudaStream_t st, int64_t* count, bool profile = false);
  int step(int64_t n) override;
  int drain();
  int probe(double* out, int64_t cap, int64_t* written) override;
  int get_state(int which, double* out, int64_t n) override;
  int set_state(int which, const double* in, int64_t n) override;
  int sync() override;
  int check_async();
};

template <typename T>
static int launch_gemv(int rows, int cols, int N, const T* A, const T* X, T* out, const T* g, T alpha,
                       bool accumulate, const int64_t* d_step, int check_every, unsigned long long* bad,
                       cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return 0;
  const int threads = 256;
  const int blocks = std::min((rows * 32 + threads - 1) / threads, 148 * 16);
#define FDTD_GEMV(NB) fdtd::gemv_rows_kernel<T, NB><<<blocks, threads, 0, st>>>(rows, cols, N, A, X, out, g, alpha, accumulate, d_step, check_every, bad)
  if (N <= 1) FDTD_GEMV(1);
  else if (N <= 4) FDTD_GEMV(4);
  else if (N <= 16) FDTD_GEMV(16);
  else if (N <= 32) FDTD_GEMV(32);
  else return -1;
#undef FDTD_GEMV
  return 1;
}

template <typename T, typename OT>
static int launch_rowblock(int rows, int K, int Kp, int N, const T* A, const T* X, OT* out, const T* g, T alpha,
                           bool acc, const int64_t* d_step, int check_every, unsigned long long* bad,
                           cudaStream_t st) {
  if (rows <= 0) return 0;
  const size_t sm = (size_t)Kp * N * sizeof(T);
  const int blocks = std::min((rows + 7) / 8, 148 * 2);
#define FDTD_RB(NB) fdtd::rowblock_gemv_kernel<T, NB, OT><<<blocks, 256, sm, st>>>(rows, K, Kp, N, A, X, out, g, alpha, acc, d_step, check_every, bad)
  if (N <= 1) FDTD_RB(1);
  else if (N <= 4) FDTD_RB(4);
  else if (N <= 16) FDTD_RB(16);
  else FDTD_RB(32);
#undef FDTD_RB
  return 1;
}

template <typename T>
static int launch_colsum(int rows, int cols, int Kp, int N, const T* A, const T* X, double* out, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return 0;
  const int cpt = std::min((cols + 255) / 256, 4);
  const int ytiles = (cols + 256 * cpt - 1) / (256 * cpt);
  const dim3 blocks(std::max(1, std::min(rows, 148 * 4 / ytiles)), ytiles);
#define FDTD_CS(NB, CPT) fdtd::colsum_gemv_kernel<T, NB, CPT><<<blocks, 256, 0, st>>>(rows, cols, Kp, N, A, X, out)
  if (N <= 4) { if (cpt <= 1) FDTD_CS(4, 1); else if (cpt <= 2) FDTD_CS(4, 2); else FDTD_CS(4, 4); }
  else if (N <= 16) { if (cpt <= 1) FDTD_CS(16, 1); else if (cpt <= 2) FDTD_CS(16, 2); else FDTD_CS(16, 4); }
  else { if (cpt <= 1) FDTD_CS(32, 1); else if (cpt <= 2) FDTD_CS(32, 2); else FDTD_CS(32, 4); }
#undef FDTD_CS
  return 1;
}

static int gemm_nn_smem(int NQ, int Kp) {
  const int TR = 4 * 256 / NQ, KC = NQ >= 4 ? 32 : 16;
  return (int)(sizeof(float) * ((size_t)Kp * 4 * NQ + 3 * (size_t)TR * (KC + 4)));
}
static int gemm_tn_smem(int NQ) {
  const int TC = 4 * 256 / NQ;
  return (int)(sizeof(float) * 3 * 16 * ((size_t)TC + 4 * NQ) + sizeof(double) * 16 * ((size_t)TC + 4 * NQ));
}
// y = S_E h~ (rows = n_if) and S_E^T G partials for the fp32 GEMM path
static int launch_gemm_nn(int rows, int K, int Kp, int N, const float* A, const float* X, float* out, const float* g,
                          float alpha, bool acc, const int64_t* d_step, int check_every, unsigned long long* bad,
                          cudaStream_t st) {
  const int NQ = N / 4;
  const int grid = std::min(148, std::max(1, rows / 64));
  const int sm = gemm_nn_smem(NQ, Kp);
#define FDTD_GNN(Q) fdtd::gemm_nn_f32_kernel<Q><<<grid, 256, sm, st>>>(rows, K, Kp, A, X, out, g, alpha, acc, d_step, check_every, bad)
  if (NQ == 2) FDTD_GNN(2); else if (NQ == 4) FDTD_GNN(4); else FDTD_GNN(8);
#undef FDTD_GNN
  return 1;
}
static int launch_gemm_tn(int rows, int cols, int Kp, int N, int splits, const float* A, const float* G, double* part,
                          cudaStream_t st) {
  const int NQ = N / 4, TC = 4 * 256 / NQ;
  const dim3 grid((cols + TC - 1) / TC, splits);
  const int sm = gemm_tn_smem(NQ);
#define FDTD_GTN(Q) fdtd::gemm_tn_f32_partial_kernel<Q><<<grid, 256, sm, st>>>(rows, cols, Kp, A, G, part)
  if (NQ == 2) FDTD_GTN(2); else if (NQ == 4) FDTD_GTN(4); else FDTD_GTN(8);
#undef FDTD_GTN
  return 1;
}
template <typename T>
int Impl<T>::create(const fdtd_grid* g, const fdtd_materials* mat, const fdtd_interface* itf,
                    const fdtd_reduced_block* bl, int n_blocks, const fdtd_sources* src,
                    const fdtd_probes* probes, const fdtd_exec* ex) {
  dim = g->dim;
  nx = g->nx; ny = g->ny; nz = (dim == 3) ? g->nz : 0;
  B = g->batch;
  if (ex) {
    stream = reinterpret_cast<cudaStream_t>(ex->stream);
    mem.alloc = ex->alloc; mem.free_ = ex->free; mem.ctx = ex->alloc_ctx;
    check_every = ex->check_every < 0 ? 100 : ex->check_every;
    graph_steps = ex->graph_steps < 0 ? 32 : ex->graph_steps;
    if (graph_steps % 2) graph_steps += 1;
    if (ex->probe_capacity > 0) cap = ex->probe_capacity;
    reduced_form = ex->reduced_form;
  }
  // x pitch: 128 B rows for B == 1; in 3-D keep >= SX spare elements at the end
  // of each row so the TMA tensor map can start SX elements before a row
  // (negative box coordinates are not used, see stencil3d_tma_kernel)
  tSX = std::max(B, 16 / (int)sizeof(T));
  if (B == 1) px = ((nx + 1 + (dim == 3 ? tSX : 0) + 31) / 32) * 32;
  else {
    px = nx + 1 + (dim == 3 ? (tSX + B - 1) / B : 0);
    while ((px * B * (int)sizeof(T)) % 16) ++px;
  }
  plane = (int64_t)(ny + 1) * px;
  nplanes = (dim == 3) ? (nz + 1) : 1;
  S = (int64_t)(nx + 1) * (ny + 1) * (dim == 3 ? (nz + 1) : 1);
  elems = plane * nplanes * B;
  const int ncomp_first = dim == 3 ? 0 : 2, ncomp_last = dim == 3 ? 5 : 4;

  // ---- fields (both parities), zero initial state ----
  guard = ((int64_t)px * B + tSX + 127) / 128 * 128;
  for (int p = 0; p < 2; ++p)
    for (int c = ncomp_first; c <= ncomp_last; ++c) {
      T* base = dalloc<T>(elems + guard);
      if (!base) return fail(FDTD_ENOMEM, "field allocation failed (%lld elements)", (long long)elems);
      CK(cudaMemsetAsync(base, 0, sizeof(T) * (elems + guard), stream));
      F[p][c] = base + guard;
    }

  // ---- TMA tensor maps for the 3-D stencil (B == 1 / aligned batches) ----
  if (dim == 3) {
    tBX = (B == 1) ? 32 : B * std::max(2, 32 / B);
    tBY = (B == 1) ? 8 : std::max(2, 256 / tBX);
    if (tBX * tBY > 256) tBY = 256 / tBX;
    if (B > 1 && B % kW == 0 && 32 * kW >= 2 * B && !getenv("FDTD_NO_VEC")) {
      // batched: each thread owns 16 bytes of members, 32 threads per row
      tW = kW; tBX = 32 * kW; tBY = 8;
    }
    // the tile stencil (default): batch 1 with W x cells per thread, or a
    // batch of 16 members with 16 bytes per thread; 32-bit element offsets
    {
      fdtd::TileCfg c;
      c.BY = 8;
      if (B == 1) {
        c.MB = 0; c.W = 2; c.NS = sizeof(T) == 4 ? 6 : 3;
        // short z extent (config 5: 41 planes): the kernel is bound by issue
        // latency, not bandwidth (time follows the executed-instruction count),
        // so the variant with three resident CTAs per SM (8-row tiles, 4-plane
        // ring, <= 85 registers) wins: measured 55 vs 64 us per step
        if (sizeof(T) == 4 && nz + 1 < 64) { c.W = 2; c.NS = 4; c.BY = 8; }
      }
      else { c.MB = B; c.W = kW; c.NS = 3; }
      if (const char* e = getenv("FDTD_TILE")) { c.BY = 8; sscanf(e, "%d,%d,%d", &c.W, &c.NS, &c.BY); }
      const int64_t span = (int64_t)px * B * (ny + 1) * (nz + 1) + (int64_t)px * B + 64;
      if (fdtd::tile_supported<T>(c) && span < ((int64_t)1 << 31) && !getenv("FDTD_STENCIL_OLD")) {
        use_tile = true; tcfg = c;
        tW = c.W; tBX = 32 * c.W; tBY = c.BY;
      }
    }
    const int vec = 16 / (int)sizeof(T);
    tHBX = tBX + tSX;                                  // H box: SX halo elements + the tile
    const int al = std::max(1, 16 / (B * (int)sizeof(T)));
    tOUTX = (tBX / B - 1) / al * al;                   // 16-byte aligned tile origins
    (void)vec;
    const bool aligned = (tBX * (int)sizeof(T)) % 16 == 0 && (px * B * (int)sizeof(T)) % 16 == 0 && tHBX <= 256 &&
                         (tSX * (int)sizeof(T)) % 16 == 0 && tOUTX >= 1 && tSX >= B;
    if (aligned) {
      PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
      cudaDriverEntryPointQueryResult qres;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault,
                                  &qres) == cudaSuccess && encode && qres == cudaDriverEntryPointSuccess) {
        use_tma = true;
        // base = field - one row - SX elements: tensor coordinate (x', y', z) is
        // storage (x' - SX, y' - 1, z); the halo at x = -1 / y = -1 maps to the
        // spare end-of-row columns / the guard (finite, and only ever selected away)
        const cuuint64_t gdim[3] = {(cuuint64_t)px * B, (cuuint64_t)ny + 2, (cuuint64_t)nz + 1};
        const cuuint64_t gstr[2] = {(cuuint64_t)px * B * sizeof(T), (cuuint64_t)px * B * (ny + 1) * sizeof(T)};
        const cuuint32_t boxH[3] = {(cuuint32_t)tHBX, (cuuint32_t)tBY + 1, 1};
        const cuuint32_t boxE[3] = {(cuuint32_t)tBX, (cuuint32_t)tBY, 1};
        const cuuint32_t es[3] = {1, 1, 1};
        const CUtensorMapDataType dt = sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
        for (int p = 0; p < 2 && use_tma; ++p)
          for (int c = 0; c < 3 && use_tma; ++c) {
            CUresult r1 = encode(&tma[p].h[c], dt, 3, F[p][3 + c] - (int64_t)px * B - tSX, gdim, gstr, boxH, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            CUresult r2 = encode(&tma[p].e[c], dt, 3, F[p][c] - (int64_t)px * B - tSX, gdim, gstr, boxE, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r1 != CUDA_SUCCESS || r2 != CUDA_SUCCESS) use_tma = false;
          }
      }
    }
    if (getenv("FDTD_NO_TMA")) use_tma = false;
    if (!use_tma) use_tile = false;
    if (getenv("FDTD_PDL")) use_pdl = true;
    if (const char* e = getenv("FDTD_KCHUNK")) kchunk_max = std::max(1, atoi(e));
  }

  // ---- materials ----
  std::vector<double> coef;           // [n_mat][6]
  std::vector<uint8_t> ifmask;
  std::vector<uint8_t> ids;           // storage-indexed (unpadded)
  uniform = (mat == nullptr || mat->n_mat == 0);
  if (!uniform) {
    if (mat->n_mat > 256 || !mat->mat_id || !mat->coef || !mat->if_mask)
      return fail(FDTD_EINVAL, "materials: n_mat must be <= 256 with mat_id/coef/if_mask given");
    n_mat = mat->n_mat;
    coef.assign(mat->coef, mat->coef + 6 * n_mat);
    ifmask.assign(mat->if_mask, mat->if_mask + n_mat);
    ids.assign(mat->mat_id, mat->mat_id + S);
    for (int64_t s = 0; s < S; ++s)
      if (ids[s] >= n_mat) return fail(FDTD_EINVAL, "mat_id[%lld] = %d >= n_mat", (long long)s, ids[s]);
  } else {
    const double* uc = mat ? mat->uniform_coef : nullptr;
    n_mat = 1;
    coef.assign(6, 0.0);
    if (uc) for (int c = 0; c < 6; ++c) coef[c] = uc[c];
    ifmask.assign(1, 0);
  }
  // lossy media: ca / da per material (fdtd.h coef_a); coefa stays in step with coef
  std::vector<double> coefa((size_t)n_mat * 6, 1.0);
  if (mat && mat->n_mat > 0 && mat->coef_a) {
    coefa.assign(mat->coef_a, mat->coef_a + 6 * (size_t)n_mat);
    for (double v : coefa) {
      if (!(v > -1.0 && v <= 1.0)) return fail(FDTD_EINVAL, "materials: coef_a must lie in (-1, 1]");
      lossy |= (v != 1.0);
    }
  }
  auto ensure_table = [&]() {
    if (uniform) { uniform = false; ids.assign(S, 0); }
  };
  auto mat_coef = [&](int64_t s, int c) -> double { return coef[(uniform ? 0 : ids[s]) * 6 + c]; };
  auto storage_ijk = [&](int64_t s, int& i, int& j, int& k) {
    i = (int)(s % (nx + 1));
    if (dim == 3) { j = (int)((s / (nx + 1)) % (ny + 1)); k = (int)(s / ((int64_t)(nx + 1) * (ny + 1))); }
    else { j = (int)(s / (nx + 1)); k = 0; }
  };
  auto sidx = [&](int i, int j, int k) -> int64_t {
    return dim == 3 ? ((int64_t)k * (ny + 1) + j) * (nx + 1) + i : (int64_t)j * (nx + 1) + i;
  };

  // ---- reduced blocks ----
  if (n_blocks < 0 || (n_blocks > 0 && !bl)) return fail(FDTD_EINVAL, "blocks: n_blocks/pointer mismatch");
  blocks.resize(n_blocks);
  for (int b = 0; b < n_blocks; ++b) {
    const fdtd_reduced_block& R = bl[b];
    BlockDev<T>& D = blocks[b];
    if (R.qe < 1 || R.qh < 1 || R.n_inst < 1 || R.n_if < 0 || !R.K || (R.n_if > 0 && !R.S_E))
      return fail(FDTD_EINVAL, "block %d: q < 1, n_inst < 1 or missing matrices", b);
    D.qe = R.qe; D.qh = R.qh; D.n_inst = R.n_inst; D.n_if = R.n_if; D.N = R.n_inst * B;
    if (D.N > 32) return fail(FDTD_ENOTSUP, "block %d: n_inst*batch = %d > 32 not supported", b, D.N);
    D.e_off = e_size; e_size += (int64_t)D.qe * D.N;
    D.h_off = h_size; h_size += (int64_t)D.qh * D.N;
    D.y_off = y_size; y_size += (int64_t)D.n_if * D.N;
    D.K.assign(R.K, R.K + (size_t)D.qe * D.qh);
    if (D.n_if) D.SE.assign(R.S_E, R.S_E + (size_t)D.n_if * D.qh);
    D.ge.resize(D.qe); D.gh.resize(D.qh);
    for (int r = 0; r < D.qe; ++r) D.ge[r] = R.g_e ? R.g_e[r] : R.g_e_scalar;
    for (int r = 0; r < D.qh; ++r) D.gh[r] = R.g_h ? R.g_h[r] : R.g_h_scalar;
    const int64_t RM = (int64_t)D.qh + D.n_if + D.qe, CM = (int64_t)D.qe + D.n_if + D.qh;
    D.fused = RM * CM <= (int64_t)6 * 1024 * 1024 && CM * D.N * (int64_t)sizeof(T) <= 160 * 1024;
    if (reduced_form == 1 && !D.fused) return fail(FDTD_ENOTSUP, "block %d too large for the fused form", b);
    if (reduced_form == 2) D.fused = false;
    any_fused |= D.fused;
    any_leap |= !D.fused;
    // leapfrog matrices (also used for the prologue gemv e~ -= G_e K~' h~)
    std::vector<T> K((size_t)D.qe * D.qh), KT((size_t)D.qh * D.qe), SE((size_t)D.n_if * D.qh),
        SET((size_t)D.qh * D.n_if), ge(D.qe), gh(D.qh);
    for (int r = 0; r < D.qe; ++r)
      for (int c = 0; c < D.qh; ++c) {
        K[(size_t)r * D.qh + c] = (T)D.K[(size_t)r * D.qh + c];
        KT[(size_t)c * D.qe + r] = (T)D.K[(size_t)r * D.qh + c];
      }
    for (int r = 0; r < D.n_if; ++r)
      for (int c = 0; c < D.qh; ++c) {
        SE[(size_t)r * D.qh + c] = (T)D.SE[(size_t)r * D.qh + c];
        SET[(size_t)c * D.n_if + r] = (T)D.SE[(size_t)r * D.qh + c];
      }
    for (int r = 0; r < D.qe; ++r) ge[r] = (T)D.ge[r];
    for (int r = 0; r < D.qh; ++r) gh[r] = (T)D.gh[r];
    D.ge_d = dalloc<T>(D.qe); D.gh_d = dalloc<T>(D.qh);
    if (!D.ge_d || !D.gh_d || upload(D.ge_d, ge) || upload(D.gh_d, gh)) return fail(FDTD_ENOMEM, "block %d allocation failed", b);
    if (D.fused) {
      D.K_d = dalloc<T>(K.size());
      D.SE_d = dalloc<T>(std::max<size_t>(SE.size(), 1));
      if (!D.K_d || !D.SE_d) return fail(FDTD_ENOMEM, "block %d allocation failed", b);
      if (upload(D.K_d, K) || upload(D.SE_d, SE)) return FDTD_ECUDA;
    } else {
      const int PADC = 32 * (16 / (int)sizeof(T));
      D.Kph = (D.qh + PADC - 1) / PADC * PADC;
      D.Kpe = (D.qe + PADC - 1) / PADC * PADC;
      std::vector<T> Kp((size_t)D.qe * D.Kph, (T)0), KTp((size_t)D.qh * D.Kpe, (T)0), SEp((size_t)D.n_if * D.Kph, (T)0);
      for (int r = 0; r < D.qe; ++r)
        for (int c = 0; c < D.qh; ++c) Kp[(size_t)r * D.Kph + c] = K[(size_t)r * D.qh + c];
      for (int r = 0; r < D.qh; ++r)
        for (int c = 0; c < D.qe; ++c) KTp[(size_t)r * D.Kpe + c] = KT[(size_t)r * D.qe + c];
      for (int r = 0; r < D.n_if; ++r)
        for (int c = 0; c < D.qh; ++c) SEp[(size_t)r * D.Kph + c] = SE[(size_t)r * D.qh + c];
      D.Kp_d = dalloc<T>(Kp.size()); D.KTp_d = dalloc<T>(KTp.size());
      D.SEp_d = dalloc<T>(std::max<size_t>(SEp.size(), 1)); D.Tv_d = dalloc<double>((size_t)D.qh * D.N);
      if (!D.Kp_d || !D.KTp_d || !D.SEp_d || !D.Tv_d) return fail(FDTD_ENOMEM, "block %d allocation failed", b);
      if (upload(D.Kp_d, Kp) || upload(D.KTp_d, KTp) || upload(D.SEp_d, SEp)) return FDTD_ECUDA;
      if (sizeof(T) == 4 && (D.N == 8 || D.N == 16 || D.N == 32) &&
          (D.n_if >= 148 * 64 || getenv("FDTD_FORCE_SKINNY")) && !getenv("FDTD_NO_SKINNY")) {
        const int TC = 4 * 256 / (D.N / 4);
        const int ctile = (D.qh + TC - 1) / TC;
        D.splits = std::max(1, std::min(2 * 148 / ctile, D.n_if / 64));
        // N = 16: the S_E^T G product on the 8 x 8 register-tile kernel, one CTA per SM
        // (FDTD_NO_WIDE=1: the general 4 x 4 kernel)
        if (D.N == 16 && D.qh % 2 == 0 && !getenv("FDTD_NO_WIDE")) {
          D.wide = true;
          D.splits = std::max(1, std::min(148 / ((D.qh + fdtd::WTC - 1) / fdtd::WTC), D.n_if / 64));
          CK(cudaFuncSetAttribute(fdtd::gemm_tn_f32_wide_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  fdtd::gemm_tn_wide_smem()));
          CK(cudaFuncSetAttribute(fdtd::gemm_tn_f32_wide_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  fdtd::gemm_tn_wide_smem()));
          if (const char* e = getenv("FDTD_WIDE_NG")) D.wide_ng = atoi(e) == 2 ? 2 : 4;
        }
        // the K~' products as split-K TN GEMMs on the stored transposes: 4 column
        // tiles x ks row splits fill the GPU (a 1024 x 1024 x 16 product is too
        // small for one CTA per row block)
        D.ks = std::max(1, std::min(32, std::min(D.qe, D.qh) / 16));
        if (const char* e = getenv("FDTD_KS")) D.ks = std::max(1, atoi(e));
        D.part_d = dalloc<double>((size_t)(D.ks + D.splits) * D.qh * D.N);
        D.parte_d = dalloc<double>((size_t)D.ks * D.qe * D.N);
        D.gen_d = dalloc<T>((size_t)D.qe);
        if (!D.part_d || !D.parte_d || !D.gen_d) return fail(FDTD_ENOMEM, "block %d: partial-sum workspace allocation failed", b);
        {
          std::vector<T> gen(D.qe);
          for (int r = 0; r < D.qe; ++r) gen[r] = -ge[r];
          if (upload(D.gen_d, gen)) return FDTD_ECUDA;
        }
        if (D.N == fdtd::tc::BN && !getenv("FDTD_NO_TC")) {
          PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
          cudaDriverEntryPointQueryResult qres;
          if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault,
                                      &qres) == cudaSuccess && encode && qres == cudaDriverEntryPointSuccess) {
            const cuuint64_t gdim[2] = {(cuuint64_t)D.Kph, (cuuint64_t)D.n_if};
            const cuuint64_t gstr[1] = {(cuuint64_t)D.Kph * sizeof(float)};
            const cuuint32_t box[2] = {(cuuint32_t)fdtd::tc::BK, (cuuint32_t)fdtd::tc::BM};
            const cuuint32_t es[2] = {1, 1};
            D.tc = encode(&D.se_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)D.SEp_d, gdim, gstr, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
            if (D.tc) {
              // zero rows beyond qh stay zero; the prologue / set_state fill the rest (tc_split_x)
              const size_t nxs = (size_t)((D.qh + 31) / 32) * 1024;
              D.xs_d = dalloc<float>(nxs);
              if (!D.xs_d) return fail(FDTD_ENOMEM, "block %d: tensor-core operand buffer allocation failed", b);
              CK(cudaMemsetAsync(D.xs_d, 0, nxs * sizeof(float), stream));
            }
          }
        }
      }
    }
  }
  for (int p = 0; p < 2; ++p) {
    eb[p] = dalloc<T>(std::max<int64_t>(e_size, 1));
    hb[p] = dalloc<T>(std::max<int64_t>(h_size, 1));
    CK(cudaMemsetAsync(eb[p], 0, sizeof(T) * std::max<int64_t>(e_size, 1), stream));
    CK(cudaMemsetAsync(hb[p], 0, sizeof(T) * std::max<int64_t>(h_size, 1), stream));
  }
  y_all = dalloc<T>(std::max<int64_t>(y_size, 1));
  g_all = dalloc<T>(std::max<int64_t>(y_size, 1));
  CK(cudaMemsetAsync(y_all, 0, sizeof(T) * std::max<int64_t>(y_size, 1), stream));
  CK(cudaMemsetAsync(g_all, 0, sizeof(T) * std::max<int64_t>(y_size, 1), stream));

  // ---- explicit rows: interface rows, then source rows on regular unknowns ----
  struct HRow { std::vector<std::pair<int64_t, double>> w; double c = 0; int64_t y = -1; int src = -1; double cs = 0; int comp = 0; int64_t s = 0; double a = 1.0; };
  std::vector<HRow> hrows;
  std::map<int64_t, int> row_of;      // E unknown id -> explicit row
  std::vector<int32_t> gcomp, gblk; std::vector<int64_t> goff, gdst;
  if (itf && itf->n_rows > 0) {
    if (!itf->unknown || !itf->c || !itf->rowptr || !itf->block || !itf->inst || !itf->local)
      return fail(FDTD_EINVAL, "interface: missing arrays");
    if (uniform) return fail(FDTD_EINVAL, "interface rows need a material table with if_mask bits");
    for (int64_t r = 0; r < itf->n_rows; ++r) {
      const int64_t u = itf->unknown[r];
      const int c = (int)(u / S);
      const int64_t s = u % S;
      if (u < 0 || !is_e(c)) return fail(FDTD_ESTAMP, "interface row %lld: %lld is not an E unknown", (long long)r, (long long)u);
      if (!((ifmask[ids[s]] >> c) & 1))
        return fail(FDTD_EINVAL, "interface row %lld: if_mask bit not set for its unknown", (long long)r);
      if (row_of.count(u)) return fail(FDTD_EINVAL, "interface row %lld duplicates an unknown", (long long)r);
      const int b = itf->block[r], in = itf->inst[r], l = itf->local[r];
      if (b < 0 || b >= n_blocks || in < 0 || in >= blocks[b].n_inst || l < 0 || l >= blocks[b].n_if)
        return fail(FDTD_EINVAL, "interface row %lld: block/inst/local out of range", (long long)r);
      HRow h;
      h.comp = c; h.s = s; h.c = itf->c[r];
      for (int64_t k = itf->rowptr[r]; k < itf->rowptr[r + 1]; ++k) {
        const int64_t hu = itf->col[k];
        if (hu < 0 || !is_h((int)(hu / S))) return fail(FDTD_ESTAMP, "interface row %lld: column %lld is not an H unknown", (long long)r, (long long)hu);
        h.w.push_back({hu, itf->val[k]});
      }
      const BlockDev<T>& D = blocks[b];
      h.y = D.y_off + (int64_t)l * D.N + (int64_t)in * B;
      row_of[u] = (int)hrows.size();
      hrows.push_back(h);
      split_rows.push_back({(int)(s % (nx + 1)), (int)((s / (nx + 1)) % (ny + 1))});
      gcomp.push_back(c); goff.push_back(dev_off(s)); gblk.push_back(b);
      gdst.push_back((int64_t)l * D.N + (int64_t)in * B);        // within the block's [n_if][N]
    }
  }
  // the converse: every E unknown whose material carries an if_mask bit must
  // be an interface row (the per-step and the persistent kernels skip such
  // cells in the regular update; without a row the cell would be frozen in
  // one path and updated in the other)
  if (!uniform) {
    bool any_bit = false;
    for (size_t m = 0; m < ifmask.size(); ++m) any_bit |= (ifmask[m] & 7) != 0;
    if (any_bit)
      for (int64_t s = 0; s < S; ++s) {
        const uint8_t bits = ifmask[ids[s]] & 7;
        if (!bits) continue;
        for (int c = 0; c < 3; ++c)
          if (((bits >> c) & 1) && is_e(c) && !row_of.count((int64_t)c * S + s))
            return fail(FDTD_EINVAL, "storage index %lld: if_mask bit %d set but no interface row", (long long)s, c);
      }
  }
  int64_t n_src = 0, n_wave = 0, n_cols = 0;
  std::vector<T> wave;
  std::vector<int32_t> wcol;
  if (src && src->n_src > 0) {
    n_src = src->n_src; n_wave = src->n_wave;
    n_cols = src->column ? src->n_cols : n_src;
    if (!src->unknown || !src->coef || (n_wave > 0 && !src->wave) || n_cols < 1)
      return fail(FDTD_EINVAL, "sources: missing arrays");
    wcol.resize(n_src);
    for (int64_t q = 0; q < n_src; ++q) {
      wcol[q] = src->column ? src->column[q] : (int32_t)q;
      if (wcol[q] < 0 || wcol[q] >= n_cols) return fail(FDTD_EINVAL, "source %lld: waveform column out of range", (long long)q);
    }
    wave.resize((size_t)(n_wave * n_cols * B));
    for (size_t q = 0; q < wave.size(); ++q) wave[q] = (T)src->wave[q];
    for (int64_t s_ = 0; s_ < n_src; ++s_) {
      const int64_t u = src->unknown[s_];
      const int c = (int)(u / S);
      const int64_t s = u % S;
      if (u < 0 || u >= 6 * S || !is_e(c)) return fail(FDTD_ESTAMP, "source %lld: %lld is not an E unknown", (long long)s_, (long long)u);
      auto it = row_of.find(u);
      if (it != row_of.end()) {
        if (hrows[it->second].src >= 0) return fail(FDTD_EINVAL, "two sources on one unknown");
        hrows[it->second].src = (int)s_; hrows[it->second].cs = src->coef[s_];
        continue;
      }
      const double cb = mat_coef(s, c);
      int i, j, k;
      storage_ijk(s, i, j, k);
      const bool wall = (dim == 3) ? ((c == 0 && (j == 0 || j == ny || k == 0 || k == nz || i >= nx)) ||
                                      (c == 1 && (i == 0 || i == nx || k == 0 || k == nz || j >= ny)) ||
                                      (c == 2 && (i == 0 || i == nx || j == 0 || j == ny || k >= nz)))
                                   : (i == 0 || i == nx || j == 0 || j == ny);
      if (cb == 0.0 || wall) return fail(FDTD_ESTAMP, "source %lld sits on an inert (PEC / hole) unknown", (long long)s_);
      HRow h;
      h.comp = c; h.s = s; h.c = cb; h.src = (int)s_; h.cs = src->coef[s_];
      h.a = coefa[(size_t)(uniform ? 0 : ids[s]) * 6 + c];
      // K_inc row (= -curl_H) of the regular stencil, fdtd.h conventions
      const int64_t Hx = 3 * S, Hy = 4 * S, Hz = 5 * S;
      if (c == 0) {
        h.w = {{Hz + sidx(i, j, k), -1.0}, {Hz + sidx(i, j - 1, k), 1.0}, {Hy + sidx(i, j, k), 1.0}, {Hy + sidx(i, j, k - 1), -1.0}};
      } else if (c == 1) {
        h.w = {{Hx + sidx(i, j, k), -1.0}, {Hx + sidx(i, j, k - 1), 1.0}, {Hz + sidx(i, j, k), 1.0}, {Hz + sidx(i - 1, j, k), -1.0}};
      } else {
        h.w = {{Hy + sidx(i, j, k), -1.0}, {Hy + sidx(i - 1, j, k), 1.0}, {Hx + sidx(i, j, k), 1.0}, {Hx + sidx(i, j - 1, k), -1.0}};
      }
      row_of[u] = (int)hrows.size();
      hrows.push_back(h);
      ensure_table();
      const int old = ids[s];
      std::vector<double> nc(coef.begin() + old * 6, coef.begin() + old * 6 + 6);
      if (coefa.size() < ifmask.size() * 6) coefa.resize(ifmask.size() * 6, 1.0);      // ensure_table may have added class 0
      std::vector<double> na(coefa.begin() + old * 6, coefa.begin() + old * 6 + 6);
      const uint8_t nm = (uint8_t)(ifmask[old] | (1u << c));
      int found = -1;
      for (int m = 0; m < (int)ifmask.size(); ++m)
        if (ifmask[m] == nm && std::equal(nc.begin(), nc.end(), coef.begin() + m * 6) &&
            std::equal(na.begin(), na.end(), coefa.begin() + m * 6)) { found = m; break; }
      if (found < 0) {
        if ((int)ifmask.size() >= 256) return fail(FDTD_ENOTSUP, "more than 256 material classes after marking source rows");
        found = (int)ifmask.size();
        coef.insert(coef.end(), nc.begin(), nc.end());
        coefa.insert(coefa.end(), na.begin(), na.end());
        ifmask.push_back(nm);
      }
      ids[s] = (uint8_t)found;
    }
  }
  n_mat = (int)ifmask.size();
  if (!uniform) {
    std::vector<uint8_t> padded((size_t)(plane * nplanes), 0);
    for (int64_t s = 0; s < S; ++s) padded[dev_off(s)] = ids[s];
    mat_id = dalloc<uint8_t>(padded.size());
    std::vector<fdtd::Coef<T>> tb((size_t)n_mat * 6);
    for (int m = 0; m < n_mat; ++m)
      for (int c = 0; c < 6; ++c) tb[(size_t)m * 6 + c] = make_coef<T>(coef[(size_t)m * 6 + c]);
    tab = dalloc<fdtd::Coef<T>>(tb.size());
    ifm = dalloc<uint8_t>(n_mat);
    if (!mat_id || !tab || !ifm) return fail(FDTD_ENOMEM, "material allocation failed");
    if (upload(mat_id, padded) || upload(tab, tb) || upload(ifm, ifmask)) return FDTD_ECUDA;
    if (lossy) {
      coefa.resize((size_t)n_mat * 6, 1.0);
      std::vector<T> ta(coefa.begin(), coefa.end());
      tab_a = dalloc<T>(ta.size());
      if (!tab_a || upload(tab_a, ta)) return fail(FDTD_ENOMEM, "material allocation failed");
    }
  } else {
    if (lossy) return fail(FDTD_EINVAL, "lossy media need a material table");
    u0 = make_coef<T>(coef[dim == 3 ? 0 : 2]);
    u1 = make_coef<T>(coef[3]);
    for (int c = 1; c < 3; ++c)
      if (dim == 3 && coef[c] != coef[0]) return fail(FDTD_ENOTSUP, "uniform mode needs equal cb for all E components");
    for (int c = 4; c < (dim == 3 ? 6 : 5); ++c)
      if (coef[c] != coef[3]) return fail(FDTD_ENOTSUP, "uniform mode needs equal ch for all H components");
  }
  for (const auto& h : hrows)
    xrows.push_back(XRow{h.comp, h.s, h.c, h.w, h.y, h.src >= 0 ? wcol[h.src] : -1, h.cs});
  // upload explicit rows
  {
    const int64_t nr = (int64_t)hrows.size();
    rows.n_rows = nr; rows.n_wave = n_wave; rows.n_src = n_cols;     // n_src: waveform columns
    std::vector<int32_t> ec(nr), hc, srcv(nr);
    std::vector<int64_t> eo(nr), rp(nr + 1, 0), ho, yo(nr);
    std::vector<fdtd::Coef<T>> cc(nr);
    std::vector<T> w, cs(nr), ra(nr);
    for (int64_t r = 0; r < nr; ++r) {
      const HRow& h = hrows[r];
      ec[r] = h.comp; eo[r] = dev_off(h.s); cc[r] = make_coef<T>(h.c);
      yo[r] = h.y; srcv[r] = h.src >= 0 ? wcol[h.src] : -1; cs[r] = (T)h.cs; ra[r] = (T)h.a;
      for (auto& pw : h.w) {
        hc.push_back((int)(pw.first / S)); ho.push_back(dev_off(pw.first % S)); w.push_back((T)pw.second);
      }
      rp[r + 1] = (int64_t)w.size();
    }
    int32_t* d_ec = dalloc<int32_t>(std::max<int64_t>(nr, 1));
    int64_t* d_eo = dalloc<int64_t>(std::max<int64_t>(nr, 1));
    fdtd::Coef<T>* d_c = dalloc<fdtd::Coef<T>>(std::max<int64_t>(nr, 1));
    int64_t* d_rp = dalloc<int64_t>(nr + 1);
    int32_t* d_hc = dalloc<int32_t>(std::max<size_t>(hc.size(), 1));
    int64_t* d_ho = dalloc<int64_t>(std::max<size_t>(ho.size(), 1));
    T* d_w = dalloc<T>(std::max<size_t>(w.size(), 1));
    int64_t* d_yo = dalloc<int64_t>(std::max<int64_t>(nr, 1));
    int32_t* d_src = dalloc<int32_t>(std::max<int64_t>(nr, 1));
    T* d_cs = dalloc<T>(std::max<int64_t>(nr, 1));
    T* d_wave = dalloc<T>(std::max<size_t>(wave.size(), 1));
    if (upload(d_ec, ec) || upload(d_eo, eo) || upload(d_c, cc) || upload(d_rp, rp) || upload(d_hc, hc) ||
        upload(d_ho, ho) || upload(d_w, w) || upload(d_yo, yo) || upload(d_src, srcv) || upload(d_cs, cs) ||
        upload(d_wave, wave))
      return FDTD_ECUDA;
    rows.e_comp = d_ec; rows.e_off = d_eo; rows.c = d_c; rows.rowptr = d_rp; rows.h_comp = d_hc;
    rows.h_off = d_ho; rows.w = d_w; rows.y_off = d_yo; rows.src = d_src; rows.cs = d_cs; rows.wave = d_wave;
    rows.g_out = g_all;
    rows.a = nullptr;
    if (lossy) {
      T* d_ra = dalloc<T>(std::max<int64_t>(nr, 1));
      if (!d_ra || upload(d_ra, ra)) return FDTD_ECUDA;
      rows.a = d_ra;
    }
    // packed records for the pre-pass of the 3-D tile stencil (<= 4 terms per row,
    // 32-bit offsets)
    if (dim == 3 && nr > 0 && !getenv("FDTD_NO_ROWPACK")) {
      bool ok = true;
      std::vector<fdtd::RowPackI> pi((size_t)nr);
      std::vector<fdtd::RowPackR<T>> pr((size_t)nr);
      for (int64_t r = 0; r < nr && ok; ++r) {
        const HRow& h = hrows[r];
        fdtd::RowPackI& a = pi[r];
        fdtd::RowPackR<T>& q = pr[r];
        memset(&a, 0, sizeof(a));
        memset(&q, 0, sizeof(q));
        if (h.w.size() > 4 || yo[r] >= ((int64_t)1 << 31) || eo[r] >= ((int64_t)1 << 31)) { ok = false; break; }
        a.e_comp = ec[r]; a.e_off = (int32_t)eo[r]; a.nterm = (int32_t)h.w.size(); a.src = srcv[r];
        a.y_off = (int32_t)yo[r];
        for (size_t k = 0; k < h.w.size(); ++k) {
          const int64_t off = ho[rp[r] + k];
          if (off >= ((int64_t)1 << 31)) { ok = false; break; }
          a.h_off[k] = (int32_t)off;
          a.h_comp |= (hc[rp[r] + k] & 0xff) << (8 * k);
          q.w[k] = w[rp[r] + k];
        }
        q.c = cc[r]; q.cs = cs[r]; q.a = ra[r];
      }
      if (ok) {
        rowpack_i = dalloc<fdtd::RowPackI>(nr);
        fdtd::RowPackR<T>* prd = dalloc<fdtd::RowPackR<T>>(nr);
        if (!rowpack_i || !prd || upload(rowpack_i, pi) || upload(prd, pr)) return FDTD_ECUDA;
        rowpack_r = prd;
        // inverse map y element -> explicit row (one row per y element and member block)
        bool inv_ok = (y_size % B) == 0;
        std::vector<int32_t> yrow((size_t)std::max<int64_t>(y_size / B, 1), -1), srows;
        for (int64_t r = 0; r < nr && inv_ok; ++r) {
          if (yo[r] < 0) { srows.push_back((int32_t)r); continue; }
          if (yo[r] % B != 0 || yo[r] / B >= (int64_t)yrow.size() || yrow[yo[r] / B] != -1) { inv_ok = false; break; }
          yrow[yo[r] / B] = (int32_t)r;
        }
        if (inv_ok) {
          y_row_d = dalloc<int32_t>(yrow.size());
          src_rows_d = dalloc<int32_t>(std::max<size_t>(srows.size(), 1));
          g_alt = dalloc<T>(std::max<int64_t>(y_size, 1));
          if (!y_row_d || !src_rows_d || !g_alt || upload(y_row_d, yrow) || upload(src_rows_d, srows)) return FDTD_ECUDA;
          CK(cudaMemsetAsync(g_alt, 0, sizeof(T) * std::max<int64_t>(y_size, 1), stream));
          n_src_rows = (int)srows.size();
        }
      }
    }
    for (int c = 0; c < 3; ++c) rows.row_of[c] = nullptr;
    for (int c = 0; c < 3; ++c) {
      bool any = false;
      for (int64_t r = 0; r < nr; ++r) any |= (ec[r] == c);
      if (!any) continue;
      std::vector<int32_t> mp((size_t)(plane * nplanes), -1);
      for (int64_t r = 0; r < nr; ++r)
        if (ec[r] == c) mp[eo[r]] = (int32_t)r;
      int32_t* d_mp = dalloc<int32_t>(mp.size());
      if (!d_mp) return fail(FDTD_ENOMEM, "row map allocation failed");
      if (upload(d_mp, mp)) return FDTD_ECUDA;
      rows.row_of[c] = d_mp;
    }
    // gather lists (ordered by block), destinations relative to each block's [n_if][N]
    std::vector<int32_t> gc2;
    std::vector<int64_t> go2, gd2;
    for (int b = 0; b < n_blocks; ++b) {
      blocks[b].probe_rows.clear();
      for (size_t q = 0; q < gcomp.size(); ++q)
        if (gblk[q] == b) { gc2.push_back(gcomp[q]); go2.push_back(goff[q]); gd2.push_back(blocks[b].y_off + gdst[q]); }
    }
    n_gather = (int64_t)gc2.size();
    g_comp = dalloc<int32_t>(std::max<int64_t>(n_gather, 1));
    g_off = dalloc<int64_t>(std::max<int64_t>(n_gather, 1));
    g_dst = dalloc<int64_t>(std::max<int64_t>(n_gather, 1));
    if (upload(g_comp, gc2) || upload(g_off, go2) || upload(g_dst, gd2)) return FDTD_ECUDA;
  }

  // ---- probes: coarse terms and leapfrog-path reduced terms; fused-path
  // reduced probes become rows of the fused update matrix ----
  {
    std::vector<int64_t> rp(1, 0), off;
    std::vector<int32_t> srcv, owner;
    std::vector<T> w;
    n_probe = probes ? (int)probes->n_probe : 0;
    for (int p = 0; p < n_probe; ++p) {
      const int kind = probes->kind[p];
      bool any_e = false, any_h = false, as_row = false;
      if (kind == 1 || kind == 2) {
        const int b = probes->block[p], in = probes->inst[p];
        if (b < 0 || b >= n_blocks || in < 0 || in >= blocks[b].n_inst) return fail(FDTD_EINVAL, "probe %d: bad block/inst", p);
        as_row = blocks[b].fused;
        if (as_row) blocks[b].probe_rows.push_back(p);
      } else if (kind != 0) {
        return fail(FDTD_EINVAL, "probe %d: unknown kind %d", p, kind);
      }
      for (int64_t k = probes->rowptr[p]; k < probes->rowptr[p + 1]; ++k) {
        const int64_t idx = probes->index[k];
        if (kind == 0) {
          const int c = (int)(idx / S);
          if (idx < 0 || idx >= 6 * S || !(is_e(c) || is_h(c))) return fail(FDTD_ESTAMP, "probe %d: bad unknown %lld", p, (long long)idx);
          any_e |= is_e(c); any_h |= is_h(c);
          srcv.push_back(c); off.push_back(dev_off(idx % S)); w.push_back((T)probes->weight[k]);
        } else {
          const BlockDev<T>& D = blocks[probes->block[p]];
          const int q = kind == 1 ? D.qe : D.qh;
          if (idx < 0 || idx >= q) return fail(FDTD_ESTAMP, "probe %d: reduced index out of range", p);
          if (!as_row) {
            srcv.push_back(kind == 1 ? 6 : 7);
            off.push_back((kind == 1 ? D.e_off : D.h_off) + idx * D.N + (int64_t)probes->inst[p] * B);
            w.push_back((T)probes->weight[k]);
          }
        }
      }
      if (any_e && any_h) return fail(FDTD_EINVAL, "probe %d mixes E and H unknowns", p);
      owner.push_back(as_row ? -2 : -1);      // -1: sampled by the reduced kernel's CTA 0
      rp.push_back((int64_t)w.size());
    }
    int64_t* d_rp = dalloc<int64_t>(rp.size());
    int32_t* d_src = dalloc<int32_t>(std::max<size_t>(srcv.size(), 1));
    int64_t* d_off = dalloc<int64_t>(std::max<size_t>(off.size(), 1));
    T* d_w = dalloc<T>(std::max<size_t>(w.size(), 1));
    int32_t* d_ow = dalloc<int32_t>(std::max<size_t>(owner.size(), 1));
    if (upload(d_rp, rp) || upload(d_src, srcv) || upload(d_off, off) || upload(d_w, w) || upload(d_ow, owner))
      return FDTD_ECUDA;
    pr.n_probe = n_probe; pr.rowptr = d_rp; pr.src = d_src; pr.off = d_off; pr.w = d_w; pr.owner = d_ow;
    hpr_src = srcv; hpr_owner = owner; hpr_off = off; hpr_rp = rp;
    for (auto v : w) hpr_w.push_back((double)v);
    ring = dalloc<T>(std::max<int64_t>(cap * n_probe * B, 1));
    if (!ring) return fail(FDTD_ENOMEM, "probe ring allocation failed");
  }
  if (any_fused) {
    int e = build_fused(probes);
    if (e) return e;
  }
  d_step = dalloc<int64_t>(2);     // step counter, one slot per step parity
  d_bad = dalloc<unsigned long long>(1);
  d_done = dalloc<unsigned int>(1);
  CK(cudaMemsetAsync(d_done, 0, sizeof(unsigned int), stream));
  CK(cudaMemsetAsync(d_step, 0, 2 * sizeof(int64_t), stream));
  CK(cudaMemsetAsync(d_bad, 0xff, sizeof(unsigned long long), stream));
  staging_bytes = sizeof(T) * (size_t)std::max<int64_t>(elems, std::max(e_size, h_size));
  CK(cudaMallocHost(&staging, staging_bytes));
  const size_t smem3 = (size_t)(3 * 3 * 300 + 3 * 3 * 256 + 2 * 3 * 256) * sizeof(T) * 2 + sizeof(fdtd::MatTable<T>);
  if (dim == 2 && elems >= ((int64_t)1 << 31)) return fail(FDTD_ENOTSUP, "2-D state too large for 32-bit offsets");
  CK(cudaFuncSetAttribute(fdtd::stencil3d_pipe_kernel<T, false, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3));
  CK(cudaFuncSetAttribute(fdtd::stencil3d_pipe_kernel<T, true, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3));
  CK(cudaFuncSetAttribute(fdtd::stencil3d_tma_kernel<T, false, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3 + 8192));
  CK(cudaFuncSetAttribute(fdtd::stencil3d_tma_kernel<T, true, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3 + 8192));
  if (lossy && dim == 3 && !use_tile)
    return fail(FDTD_ENOTSUP, "lossy media need the 3-D tile stencil (batch 1 or 16, TMA available)");
  if (use_tile) {
    const size_t ttab = uniform ? 0 : ((size_t)n_mat * (6 * sizeof(fdtd::Coef<T>) + 1) + 15) / 16 * 16 + 16 +
                                      (lossy ? (size_t)n_mat * 6 * sizeof(T) : 0);
    tile_smem = fdtd::tile_smem_bytes(tcfg, tHBX, (int)sizeof(T), ttab) + 128;
    if (tile_smem > 227 * 1024) return fail(FDTD_ENOTSUP, "tile stencil: %zu bytes of shared memory", tile_smem);
    CK(fdtd::tile_prepare<T>(tcfg, tile_smem));
    // persistent grid: every resident CTA slot, each a balanced range of column-planes
    const int outy = tBY - 1;
    tsplit.ntx = (nx + 1 + tOUTX - 1) / tOUTX;
    tsplit.outx = tOUTX; tsplit.outy = outy; tsplit.nzp = nz + 1;
    tsplit.jitter = getenv("FDTD_JITTER") ? std::max(0, atoi(getenv("FDTD_JITTER"))) : 0;
    tsplit.ncols = tsplit.ntx * ((ny + 1 + outy - 1) / outy);
    int sms = 148;
    {
      int dev = 0;
      if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int per_sm = std::max(1, fdtd::tile_blocks_per_sm<T>(tcfg, uniform, tile_smem));
    int G = per_sm * sms;
    if (const char* e = getenv("FDTD_TILE_GRID")) G = std::max(1, atoi(e));
    // z-chunking (one item per CTA, hardware scheduling; measured on B200,
    // DESIGN.md §5.3): chunks of at most 24 planes (fp32, batch 1) or 8 (fp64,
    // batched) and at least 4 items per resident CTA slot, but not below 8
    // planes (each item loads 1-2 extra planes)
    {
      const int nzp = nz + 1;
      const int kmax = (sizeof(T) == 4 && B == 1) ? 24 : 8;
      int nch = std::max((nzp + kmax - 1) / kmax, (int)((4LL * G + tsplit.ncols - 1) / tsplit.ncols));
      nch = std::max(1, std::min(nch, nzp / 8));
      // short z extents: one wave of co-resident CTAs (items <= resident slots)
      if (sizeof(T) == 4 && B == 1 && nzp < 64) nch = std::max(1, std::min(nch, G / std::max(1, tsplit.ncols)));
      int kc = (nzp + nch - 1) / nch;
      if (const char* e = getenv("FDTD_TILE_KC")) kc = std::max(1, atoi(e));
      tsplit.kc = kc;
      tsplit.nitems = tsplit.ncols * ((nzp + kc - 1) / kc);
    }
    // persistent (round-robin items over resident CTAs) only on request:
    // measured slower than one CTA per item
    if (!getenv("FDTD_TILE_GRID")) G = tsplit.nitems;
    tile_grid = std::min(tsplit.nitems, G);
    if (getenv("FDTD_VERBOSE"))
      fprintf(stderr, "fdtd: tile stencil W=%d NS=%d MB=%d smem=%zu per_sm=%d grid=%d items=%d (cols %d x kc %d)\n",
              tcfg.W, tcfg.NS, tcfg.MB, tile_smem, per_sm, tile_grid, tsplit.nitems, tsplit.ncols, tsplit.kc);
  }
  // (opt-in, FDTD_SPLIT=1: measured no gain on config 4 and a loss on config
  // 5, DESIGN.md §12 -- the second grid waits for SM slots the stencil holds)
  if (dim == 3 && use_tile && n_blocks > 0 && tile_grid == tsplit.nitems && getenv("FDTD_SPLIT") &&
      std::string(getenv("FDTD_SPLIT")) == "1") {
    // columns whose tile footprint (with a one-cell margin) holds an explicit
    // row that reads y: they evaluate the interface rows, so they run before
    // the reduced update; every other column runs beside it
    const int cells_x = (tcfg.MB > 0) ? tBX / B : tBX;           // cells per tile row
    std::vector<char> isif(tsplit.ncols, 0);
    const int nty_ = tsplit.ncols / tsplit.ntx;
    for (const auto& h : split_rows) {
      const int i = h.first, j = h.second;
      for (int ty_ = std::max(0, (j - 1 - tBY) / tsplit.outy); ty_ < nty_ && ty_ * tsplit.outy <= j + 1; ++ty_)
        for (int tx_ = std::max(0, (i - 1 - cells_x) / tsplit.outx); tx_ < tsplit.ntx && tx_ * tsplit.outx <= i + 1; ++tx_) {
          const int x0 = tx_ * tsplit.outx, y0 = ty_ * tsplit.outy;
          if (i >= x0 - 1 && i <= x0 + cells_x && j >= y0 - 1 && j <= y0 + tBY) isif[ty_ * tsplit.ntx + tx_] = 1;
        }
    }
    std::vector<int> perm;
    for (int c = 0; c < tsplit.ncols; ++c) if (isif[c]) perm.push_back(c);
    n_ifc = (int)perm.size();
    for (int c = 0; c < tsplit.ncols; ++c) if (!isif[c]) perm.push_back(c);
    if (n_ifc > 0 && n_ifc < tsplit.ncols) {
      colperm_d = dalloc<int>(perm.size());
      if (!colperm_d || upload(colperm_d, perm)) return fail(FDTD_ENOMEM, "split-step allocation failed");
      CK(cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&evA, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&evR, cudaEventDisableTiming));
      split = true;
    }
    if (getenv("FDTD_VERBOSE"))
      fprintf(stderr, "fdtd: split step %s: %d interface columns of %d\n", split ? "on" : "off", n_ifc, tsplit.ncols);
  }
  if (!use_tile) {                // the reference batched kernel (its tile shape when it is the path)
    const int smv = (int)(sizeof(T) * (3 * 3 * (size_t)(tHBX * (tBY + 1) + 32) + 6 * 3 * (size_t)(tBX * tBY + 32)) +
                          sizeof(fdtd::MatTable<T>) + 512);
    CK(cudaFuncSetAttribute(fdtd::stencil3d_tma_vec_kernel<T, false, 3, kW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            std::max(smv, 48 * 1024)));
    CK(cudaFuncSetAttribute(fdtd::stencil3d_tma_vec_kernel<T, true, 3, kW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            std::max(smv, 48 * 1024)));
  }
  CK(cudaFuncSetAttribute(fdtd::stencil2d_rows_kernel<T, false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3));
  CK(cudaFuncSetAttribute(fdtd::stencil2d_rows_kernel<T, true, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3));
  {
    const int big = 200 * 1024;
    CK(cudaFuncSetAttribute(fdtd::rowblock_gemv_kernel<T, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CK(cudaFuncSetAttribute(fdtd::rowblock_gemv_kernel<T, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CK(cudaFuncSetAttribute(fdtd::rowblock_gemv_kernel<T, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CK(cudaFuncSetAttribute(fdtd::rowblock_gemv_kernel<T, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CK(cudaFuncSetAttribute(fdtd::rowblock_gemv_kernel<T, 1, double>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CK(cudaFuncSetAttribute(fdtd::rowblock_gemv_kernel<T, 4, double>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CK(cudaFuncSetAttribute(fdtd::rowblock_gemv_kernel<T, 16, double>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CK(cudaFuncSetAttribute(fdtd::rowblock_gemv_kernel<T, 32, double>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    for (auto& D : blocks)
      if (!D.fused && (size_t)std::max(D.Kph, D.Kpe) * D.N * sizeof(T) > (size_t)big)
        return fail(FDTD_ENOTSUP, "reduced block too large for the staged leap-frog GEMV (q x N)");
    for (auto& D : blocks) {
      if (!D.tc) continue;
      CK(cudaFuncSetAttribute(fdtd::tc::tc_skinny_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              fdtd::tc::SMEM_BYTES));
      int dev = 0, sms = 148;
      if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      tc_grid = sms;
      if (const char* e = getenv("FDTD_TC_GRID")) tc_grid = std::max(1, atoi(e));
    }
    for (auto& D : blocks) {
      if (!D.splits) continue;
      const int NQ = D.N / 4;
      const int sn = gemm_nn_smem(NQ, D.Kph), stn = gemm_tn_smem(NQ);
      if (sn > 220 * 1024) { D.splits = 0; continue; }
      if (NQ == 2) {
        CK(cudaFuncSetAttribute(fdtd::gemm_nn_f32_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sn));
        CK(cudaFuncSetAttribute(fdtd::gemm_tn_f32_partial_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, stn));
      } else if (NQ == 4) {
        CK(cudaFuncSetAttribute(fdtd::gemm_nn_f32_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sn));
        CK(cudaFuncSetAttribute(fdtd::gemm_tn_f32_partial_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, stn));
      } else {
        CK(cudaFuncSetAttribute(fdtd::gemm_nn_f32_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, sn));
        CK(cudaFuncSetAttribute(fdtd::gemm_tn_f32_partial_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, stn));
      }
    }
  }
  if (fused_gemm && fused_smem > 48 * 1024) {
    CK(raise_smem_limit(fdtd::reduced_gemm_kernel<T, 4, gemm_rpw(4), GEMM_KS>, (int)fused_smem));
    CK(raise_smem_limit(fdtd::reduced_gemm_kernel<T, 8, gemm_rpw(8), GEMM_KS>, (int)fused_smem));
    CK(raise_smem_limit(fdtd::reduced_gemm_kernel<T, 16, gemm_rpw(16), GEMM_KS>, (int)fused_smem));
    CK(raise_smem_limit(fdtd::reduced_gemm_kernel<T, 32, gemm_rpw(32), GEMM_KS>, (int)fused_smem));
    CK(raise_smem_limit(fdtd::reduced_gemm_kernel<T, 32, gemm_rpw(32), 2>, (int)fused_smem));
    CK(raise_smem_limit(fdtd::reduced_gemm_kernel<T, 32, gemm_rpw(32), 8>, (int)fused_smem));
  }
  if (!fused_gemm && fused_smem > 48 * 1024) {
    CK(raise_smem_limit(fdtd::reduced_fused_kernel<T, 1>, (int)fused_smem));
    CK(raise_smem_limit(fdtd::reduced_fused_kernel<T, 4>, (int)fused_smem));
    CK(raise_smem_limit(fdtd::reduced_fused_kernel<T, 16>, (int)fused_smem));
    CK(raise_smem_limit(fdtd::reduced_fused_kernel<T, 32>, (int)fused_smem));
  }
  {
    int e = setup_persist();
    if (e) return e;
  }
  bool any_tc = false;
  for (auto& D : blocks) any_tc |= D.tc;
  // explicit rows fused into the reduced GEMM: 3-D tile path, every block in
  // reduced_gemm_kernel, packed rows with an inverse y map
  fuse_rows = dim == 3 && use_tile && !split && fused_gemm && !any_leap && any_fused && n_ctas > 0 && rowpack_i &&
              y_row_d && g_alt && !getenv("FDTD_NO_ROWFUSE");
  rows_ahead = false;
  path_bits = (persist ? 1 : 0) | (use_tma ? 2 : 0) | (fused_gemm ? 4 : 0) | (any_leap ? 8 : 0) | (use_tile ? 16 : 0) |
              (any_tc ? 32 : 0) | (fuse_rows ? 64 : 0);
  CK(cudaStreamSynchronize(stream));
  return FDTD_OK;
}

// Persistent 2-D path (persist2d.cuh): eligible when the problem is 2-D,
// single-member, every reduced block fused with one column, every explicit row
// references only the four H neighbours of its own cell, every coarse probe
// lies in one tile, and all tiles fit co-resident.  Otherwise the per-step
// kernels run (same results, bit for bit).
template <typename T>
int Impl<T>::setup_persist() {
  persist = false;
  auto why_not = [&](int code) {
    if (getenv("FDTD_VERBOSE")) fprintf(stderr, "fdtd: persistent 2-D path not used (reason %d)\n", code);
    return FDTD_OK;
  };
  if (const char* e = getenv("FDTD_PERSIST"))
    if (std::string(e) == "0") return why_not(1);
  if (dim != 2 || B != 1 || any_leap || lossy) return why_not(2);
  for (auto& D : blocks)
    if (!D.fused || D.N != 1) return why_not(3);
  for (size_t q = 0; q < hpr_owner.size(); ++q) {
    if (hpr_owner[q] != -1) continue;
    for (int64_t k = hpr_rp[q]; k < hpr_rp[q + 1]; ++k)
      if (hpr_src[k] < 2 || hpr_src[k] > 4) return why_not(4);
  }
  int dev = 0, nsm = 0, coop = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
  if (!coop) return why_not(5);
  // reduced rows
  int Rtot = 0, Cmax = 0, nfb = 0;
  for (size_t b = 0; b < fblocks.size(); ++b) {
    p_row0[b] = Rtot;
    const int RMp = fblocks[b].R;
    Rtot += RMp;
    Cmax = std::max(Cmax, fblocks[b].Cp);
    ++nfb;
  }
  p_row0[nfb] = Rtot;
  // tiles cover cells i < nx, j < ny (the last storage column / row is constant)
  const int TX = (nx <= 32) ? 32 : 64;
  const int ntx = (nx + TX - 1) / TX;
  // temporal blocking (persist2d_tb_tile, fp32): K-cell halos, square tiles
  // (off by default: measured slower than the per-step exchange on config 2,
  // the interface tiles stay bound to the per-step reduced
  // chain, so the blocks only add redundant halo work)
  int K = 0;
  if (const char* e = getenv("FDTD_P2K")) K = std::max(0, atoi(e));
  if (sizeof(T) != 4 || (K != 2 && K != 4)) K = 0;       // the instantiated shapes (p2_kernel)
  p_K = K;
  p_D = 2;
  if (K > 0) while (p_D < 2 * (K + 1)) p_D *= 2;      // y / G ring: a halo holder lags <= K steps
  // the tiles whose (extended) region holds cell (i, j): [lo, hi] per axis
  auto tile_span = [&](int i, int T_, int nt_, int& lo, int& hi) {
    if (K == 0) { lo = hi = i / T_; return; }
    lo = 0;
    while (lo * T_ + T_ + K <= i) ++lo;
    hi = std::min(nt_ - 1, (i + K) / T_);
  };
  int TY = 0, nty = 0, rpc = 0, nT = 0, nR = 0;
  size_t smem = 0;
  for (int cand : {64, 96, 128, 32}) {
    const int ty = K > 0 ? TX : ((ny <= 32) ? 32 : cand);
    if (K > 0 && cand != 64) continue;
    const int nt_y = (ny + ty - 1) / ty;
    const int nt = ntx * nt_y;
    int maxrows = 0;
    {
      std::vector<int> cnt(ntx * nt_y, 0);
      for (const auto& x : xrows) {
        const int i = (int)(x.s % (nx + 1)), j = (int)(x.s / (nx + 1));
        if (i >= nx || j >= ny) continue;
        int xl, xh, yl, yh;
        tile_span(i, TX, ntx, xl, xh);
        tile_span(j, ty, nt_y, yl, yh);
        for (int b = yl; b <= yh; ++b)
          for (int a = xl; a <= xh; ++a) maxrows = std::max(maxrows, ++cnt[b * ntx + a]);
      }
    }
    const size_t EXs = (size_t)TX + 2 * K;
    const size_t tile_sm = K > 0 ?
        sizeof(T) * 3 * EXs * EXs + 3 * fdtd::MAX_MAT * sizeof(fdtd::Coef<T>) + fdtd::MAX_MAT +
            (EXs * EXs + 15) / 16 * 16 + sizeof(fdtd::P2Row<T>) * (size_t)maxrows + 64 :
        sizeof(T) * ((size_t)3 * TX * ty + 2 * TX + 2 * ty) +
                           3 * fdtd::MAX_MAT * sizeof(fdtd::Coef<T>) + fdtd::MAX_MAT +
                           ((size_t)TX * ty + 15) / 16 * 16 + (2 * sizeof(T) * (size_t)maxrows + 15) / 16 * 16 +
                           sizeof(fdtd::P2Row<T>) * (size_t)maxrows + 64;
    if (tile_sm > 220 * 1024) continue;
    const void* kfn = p2_kernel(TX, K);
    const int nthr = 512;
    CK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tile_sm));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, nthr, tile_sm));
    const int capacity = per_sm * nsm;
    int nr = 0, r = 0;
    size_t sm = tile_sm;
    if (Rtot > 0) {
      nr = std::min(capacity - nt, std::max(1, (Rtot + 7) / 8));
      if (nr < 1) continue;
      r = (Rtot + nr - 1) / nr;
      // fp32 LL exchange: a reduced CTA whose rows of some block are ALL probe
      // rows is on no dependency chain (nothing waits for its outputs), so the
      // block's e~ / h~ owners could overwrite the tagged copies it still has
      // to read.  Choose the rows per CTA so that every CTA that holds probe
      // rows of a block also holds an h~ / y / e~ row of that block (whose
      // output the owners' next step waits for).
      auto probe_only = [&](int rr) {
        for (int a = 0; a < Rtot; a += rr) {
          const int bnd = std::min(Rtot, a + rr);
          for (int b = 0; b < nfb; ++b) {
            const int r0 = p_row0[b], r1 = p_row0[b + 1];
            const int s0 = std::max(a, r0), s1 = std::min(bnd, r1);
            if (s0 < s1 && s0 >= r0 + fblocks[b].qh + fblocks[b].n_if + fblocks[b].qe) return true;
          }
        }
        return false;
      };
      while (r < Rtot && probe_only(r)) ++r;
      if (probe_only(r)) continue;
      sm = std::max(tile_sm, sizeof(T) * ((size_t)(1 + r) * Cmax + (size_t)r * 32) + 64 +
                                 (sizeof(T) == 4 ? (size_t)r * 32 * 8 + 32 + (size_t)r * Cmax * 2 : 0));
      if (sm > 220 * 1024) continue;
      CK(raise_smem_limit(kfn, (int)sm));
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, nthr, sm));
      nr = (Rtot + r - 1) / r;
      if (per_sm * nsm < nt + nr) continue;
    }
    TY = ty; nty = nt_y; nT = nt; nR = nr; rpc = r; smem = sm; p_maxrows = maxrows; p_kfn = kfn;
    break;
  }
  if (TY == 0) return why_not(6);
  auto storage_ijk = [&](int64_t s_, int& i, int& j, int& k) {   // 2-D storage index
    i = (int)(s_ % (nx + 1)); j = (int)(s_ / (nx + 1)); k = 0;
  };
  // explicit rows -> tiles, with the H terms as local slots
  std::vector<std::vector<int>> by_tile(nT);
  std::vector<std::vector<int32_t>> li_tile(nT);     // per tile: the row's local index (extended with K > 0)
  std::vector<int32_t> li(xrows.size());
  std::vector<int8_t> nterm(xrows.size()), slot(4 * xrows.size(), 0);
  std::vector<T> wv(4 * xrows.size(), (T)0);
  for (size_t r = 0; r < xrows.size(); ++r) {
    const XRow& x = xrows[r];
    if (x.comp != 2 || x.w.size() > 4) return why_not(7);
    int i, j, k;
    storage_ijk(x.s, i, j, k);
    if (i >= nx || j >= ny) return why_not(11);
    for (size_t q = 0; q < x.w.size(); ++q) {
      const int hc = (int)(x.w[q].first / S);
      int hi, hj, hk;
      storage_ijk(x.w[q].first % S, hi, hj, hk);
      int sl = -1;
      if (hc == 4 && hi == i && hj == j) sl = 0;
      else if (hc == 4 && hi == i - 1 && hj == j) sl = 1;
      else if (hc == 3 && hi == i && hj == j) sl = 2;
      else if (hc == 3 && hi == i && hj == j - 1) sl = 3;
      if (sl < 0) return why_not(8);
      slot[4 * r + q] = (int8_t)sl;
      wv[4 * r + q] = (T)x.w[q].second;
    }
    nterm[r] = (int8_t)x.w.size();
    li[r] = (j % TY) * TX + (i % TX);
    if (K == 0) {
      by_tile[(j / TY) * ntx + (i / TX)].push_back((int)r);
      li_tile[(j / TY) * ntx + (i / TX)].push_back(li[r]);
    } else {
      int xl, xh, yl, yh;
      tile_span(i, TX, ntx, xl, xh);
      tile_span(j, TY, nty, yl, yh);
      const int EXi = TX + 2 * K;
      for (int b = yl; b <= yh; ++b)
        for (int a = xl; a <= xh; ++a) {
          by_tile[b * ntx + a].push_back((int)r);
          li_tile[b * ntx + a].push_back((j - (b * TY - K)) * EXi + (i - (a * TX - K)));
        }
    }
  }
  std::vector<int32_t> tptr(1, 0), rli, rsrc;
  std::vector<int8_t> rnt, rsl;
  std::vector<T> rw, rcs;
  std::vector<fdtd::Coef<T>> rc;
  std::vector<int64_t> ryo;
  std::vector<uint8_t> tif(nT, 0);
  int nif_tiles = 0;
  std::vector<int8_t> rown;
  for (int t = 0; t < nT; ++t) {
    for (size_t q = 0; q < by_tile[t].size(); ++q) {
      const int r = by_tile[t][q];
      const XRow& x = xrows[r];
      {
        const int i = (int)(x.s % (nx + 1)), j = (int)(x.s / (nx + 1));
        rown.push_back((int8_t)((j / TY) * ntx + (i / TX) == t));
      }
      rli.push_back(li_tile[t][q]); rnt.push_back(nterm[r]);
      for (int q = 0; q < 4; ++q) { rsl.push_back(slot[4 * r + q]); rw.push_back(wv[4 * r + q]); }
      rc.push_back(make_coef<T>(x.c)); ryo.push_back(x.y); rsrc.push_back(x.src_col); rcs.push_back((T)x.cs);
      if (x.y >= 0) tif[t] = 1;
    }
    tptr.push_back((int32_t)rli.size());
    nif_tiles += tif[t];
  }
  // coarse probes -> tiles
  std::vector<std::vector<int>> pb_tile(nT);
  for (size_t q = 0; q < hpr_owner.size(); ++q) {
    if (hpr_owner[q] != -1) continue;
    int tt = -1;
    for (int64_t k = hpr_rp[q]; k < hpr_rp[q + 1]; ++k) {
      const int i = (int)(hpr_off[k] % px), j = (int)(hpr_off[k] / px);
      if (i >= nx || j >= ny) return why_not(12);
      const int t = (j / TY) * ntx + (i / TX);
      if (tt >= 0 && t != tt) return why_not(9);
      tt = t;
    }
    if (tt >= 0) pb_tile[tt].push_back((int)q);
  }
  std::vector<int32_t> pptr(1, 0), ppid, ptp(1, 0), pli;
  std::vector<int8_t> pcomp;
  std::vector<T> pw;
  for (int t = 0; t < nT; ++t) {
    for (int q : pb_tile[t]) {
      ppid.push_back(q);
      for (int64_t k = hpr_rp[q]; k < hpr_rp[q + 1]; ++k) {
        const int i = (int)(hpr_off[k] % px), j = (int)(hpr_off[k] / px);
        pli.push_back(K > 0 ? ((j % TY) + K) * (TX + 2 * K) + (i % TX) + K : (j % TY) * TX + (i % TX));
        pcomp.push_back((int8_t)(hpr_src[k] - 2));
        pw.push_back((T)hpr_w[k]);
      }
      ptp.push_back((int32_t)pli.size());
    }
    pptr.push_back((int32_t)ppid.size());
  }
  // device copies
  auto up = [&](auto& vec, auto*& dptr) -> int {
    using E = typename std::remove_reference<decltype(vec)>::type::value_type;
    E* d = dalloc<E>(std::max<size_t>(vec.size(), 1));
    if (!d) return fail(FDTD_ENOMEM, "persistent-path allocation failed");
    if (!vec.empty() && upload(d, vec)) return FDTD_ECUDA;
    dptr = d;
    return FDTD_OK;
  };
  const int32_t *d_tptr, *d_li, *d_src, *d_pptr, *d_ppid, *d_ptp, *d_pli;
  const int8_t *d_nt, *d_sl, *d_pcomp, *d_own;
  const T *d_w, *d_cs, *d_pw;
  const fdtd::Coef<T>* d_c;
  const int64_t* d_yo;
  const uint8_t* d_tif;
  int e = FDTD_OK;
#define FDTD_UP(v, d) do { auto* tmp_ = (decltype(v.data()))nullptr; e = up(v, tmp_); if (e) return e; d = tmp_; } while (0)
  FDTD_UP(tptr, d_tptr); FDTD_UP(rli, d_li); FDTD_UP(rsrc, d_src); FDTD_UP(pptr, d_pptr); FDTD_UP(ppid, d_ppid);
  FDTD_UP(ptp, d_ptp); FDTD_UP(pli, d_pli); FDTD_UP(rnt, d_nt); FDTD_UP(rsl, d_sl); FDTD_UP(pcomp, d_pcomp);
  FDTD_UP(rw, d_w); FDTD_UP(rcs, d_cs); FDTD_UP(pw, d_pw); FDTD_UP(rc, d_c); FDTD_UP(ryo, d_yo); FDTD_UP(tif, d_tif);
  FDTD_UP(rown, d_own);
#undef FDTD_UP
  p_rows = fdtd::P2Rows<T>{d_tptr, d_li, d_c, d_nt, d_sl, d_w, d_yo, d_src, d_cs, rows.wave, rows.n_wave, rows.n_src,
                           d_own};
  p_probes = fdtd::P2Probes<T>{d_pptr, d_ppid, d_ptp, d_pli, d_pcomp, d_pw};
  p_tile_if = const_cast<uint8_t*>(d_tif);
  p_ezL = dalloc<T>((size_t)2 * nT * TY); p_hyR = dalloc<T>((size_t)2 * nT * TY);
  p_ezB = dalloc<T>((size_t)2 * nT * TX); p_hxT = dalloc<T>((size_t)2 * nT * TX);
  p_flags = dalloc<unsigned>((size_t)2 * nT + 3);
  if (sizeof(T) == 4) {
    p_ll_words = (size_t)2 * nT * (2 * TY + 2 * TX) + (size_t)2 * p_D * std::max<int64_t>(y_size, 1) +
                 2 * (size_t)(std::max<int64_t>(e_size, 1) + std::max<int64_t>(h_size, 1)) +
                 (size_t)2 * nT * 4 * 3 * K * TX;
    p_ll = dalloc<unsigned long long>(p_ll_words);
    if (!p_ll) return fail(FDTD_ENOMEM, "persistent-path allocation failed");
  }
  if (!p_ezL || !p_hyR || !p_ezB || !p_hxT || !p_flags) return fail(FDTD_ENOMEM, "persistent-path allocation failed");
  CK(cudaMemsetAsync(p_flags, 0, sizeof(unsigned) * (2 * nT + 3), stream));
  pTX = TX; pTY = TY; pntx = ntx; pnty = nty; p_rpc = rpc; p_Rtot = Rtot; p_Cmax = Cmax; p_smem = smem;
  p_nif_tiles = nif_tiles;
  p_nred = nR;
  persist = true;
  if (getenv("FDTD_VERBOSE")) {
    fprintf(stderr, "fdtd: persistent 2-D path: %d x %d tiles of %d x %d, %d reduced CTAs x %d rows, smem %zu, "
            "maxrows %d (P2Row %zu B), interface tiles %d, temporal blocking K %d (ring %d)\n", ntx, nty, TX, TY, nR,
            rpc, smem, p_maxrows, sizeof(fdtd::P2Row<T>), nif_tiles, p_K, p_D);
    for (int t = 0; t < nT; ++t)
      if (tptr[t + 1] > tptr[t]) fprintf(stderr, "  tile %d: rows %d..%d\n", t, tptr[t], tptr[t + 1]);
  }
  return FDTD_OK;
}

template <typename T>
int Impl<T>::launch_persist(int64_t n, int64_t* count) {
  const int nT = pntx * pnty;
  const int p0 = (int)(host_step & 1), p1 = (int)((host_step + n) & 1);
  fdtd::Persist2D<T> P{};
  P.nx = nx; P.ny = ny; P.px = px; P.TX = pTX; P.TY = pTY; P.ntx = pntx; P.nty = pnty;
  P.Fin[0] = F[p0][2]; P.Fin[1] = F[p0][3]; P.Fin[2] = F[p0][4];
  P.Fout[0] = F[p1][2]; P.Fout[1] = F[p1][3]; P.Fout[2] = F[p1][4];
  P.mat_id = uniform ? nullptr : mat_id;
  P.gtab = tab; P.gifm = ifm; P.n_mat = n_mat; P.u0 = u0; P.u1 = u1;
  P.R = p_rows; P.PR = p_probes;
  P.ezL = p_ezL; P.ezB = p_ezB; P.hyR = p_hyR; P.hxT = p_hxT;
  P.fE = p_flags; P.fH = p_flags + nT; P.gready = p_flags + 2 * nT; P.reddone = p_flags + 2 * nT + 1;
  P.abort_flag = reinterpret_cast<int*>(p_flags + 2 * nT + 2);
  P.tile_if = p_tile_if; P.n_if_tiles = p_nif_tiles; P.n_red_ctas = p_nred;
  for (size_t b = 0; b < fblocks.size(); ++b) P.fb[b] = fblocks[b];
  for (size_t b = 0; b <= fblocks.size(); ++b) P.row0[b] = p_row0[b];
  P.nfb = (int)fblocks.size(); P.Rtot = p_Rtot; P.rpc = p_rpc; P.Cmax = p_Cmax;
  P.eb[0] = eb[0]; P.eb[1] = eb[1]; P.hb[0] = hb[0]; P.hb[1] = hb[1]; P.y = y_all; P.G = g_all;
  P.y_in = y_all;
  if (p_ll && y_size > 0) {
    if (!p_yin) p_yin = dalloc<T>(y_size);
    if (!p_yin) return fail(FDTD_ENOMEM, "persistent-path allocation failed");
    CK(cudaMemcpyAsync(p_yin, y_all, sizeof(T) * y_size, cudaMemcpyDeviceToDevice, stream));
    P.y_in = p_yin;
  }
  P.ring = ring; P.cap = cap; P.n_probe = n_probe;
  P.step0 = host_step + step_offset; P.p0 = p0; P.nsteps = (int)n;
  P.d_step_out = d_step + p1;
  P.check_every = check_every; P.bad_step = d_bad; P.maxrows = p_maxrows;
  CK(cudaMemsetAsync(p_flags, 0, sizeof(unsigned) * (2 * nT + 3), stream));
  if (p_ll) {
    // tagged words carry the local step + 1: zero them so no stale word matches
    CK(cudaMemsetAsync(p_ll, 0, sizeof(unsigned long long) * p_ll_words, stream));
    unsigned long long* q = p_ll;
    P.lezL = q; q += (size_t)2 * nT * pTY;
    P.lhyR = q; q += (size_t)2 * nT * pTY;
    P.lezB = q; q += (size_t)2 * nT * pTX;
    P.lhxT = q; q += (size_t)2 * nT * pTX;
    P.ysz = std::max<int64_t>(y_size, 1); P.esz = std::max<int64_t>(e_size, 1); P.hsz = std::max<int64_t>(h_size, 1);
    P.lG = q; q += (size_t)p_D * P.ysz;
    P.ly = q; q += (size_t)p_D * P.ysz;
    P.leb = q; q += 2 * P.esz;
    P.lhb = q; q += 2 * P.hsz;
    P.lband = q;
  }
  P.K = p_K;
  P.ymask = p_D - 1;
  P.jitter = getenv("FDTD_JITTER") ? (unsigned)std::max(0, atoi(getenv("FDTD_JITTER"))) : 0u;
  P.sleep_ns = 0;
  if (p_K > 0) {
    static const unsigned sl = getenv("FDTD_P2SLEEP") ? (unsigned)atoi(getenv("FDTD_P2SLEEP")) : 0u;
    P.sleep_ns = sl;
  }
  static unsigned long long* dbg = nullptr;
  if (getenv("FDTD_P2DBG")) {
    if (!dbg) CK(cudaMalloc(&dbg, 3 * 8 * 8 * sizeof(unsigned long long)));
    CK(cudaMemset(dbg, 0, 3 * 8 * 8 * sizeof(unsigned long long)));
    P.dbg = dbg;
    int ti = 0;
    std::vector<uint8_t> tif(nT);
    CK(cudaMemcpy(tif.data(), p_tile_if, nT, cudaMemcpyDeviceToHost));
    for (int q = 0; q < nT; ++q) if (tif[q]) { ti = q; break; }
    P.dbg_tile_if = ti;
  }
  void* args[] = {&P};
  CK(cudaLaunchCooperativeKernel(p_kfn, dim3(nT + p_nred), dim3(512), args, p_smem,
                                 stream));
  *count += 1;
  if (P.dbg && n >= 108) {
    std::vector<unsigned long long> h(3 * 8 * 8);
    CK(cudaStreamSynchronize(stream));
    CK(cudaMemcpy(h.data(), P.dbg, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    const unsigned long long t0 = h[0];
    for (int sl = 0; sl < 3; ++sl) {
      fprintf(stderr, "slot %d (%s):\n", sl, sl == 0 ? "tile 0" : sl == 1 ? "interface tile" : "reduced CTA 0");
      for (int st = 0; st < 8; ++st) {
        fprintf(stderr, "  step %d:", 100 + st);
        for (int k = 0; k < 7; ++k) {
          const unsigned long long v = h[(sl * 8 + st) * 8 + k];
          fprintf(stderr, " %8.3f", v ? (double)(v - t0) * 1e-3 : -1.0);
        }
        fprintf(stderr, "\n");
      }
    }
  }
  return FDTD_OK;
}

// Compose each small block's step into one update matrix (host, fp64):
//   columns [e~ (qe) ; G (n_if) ; h~ (qh)],   A1 = G_h K^T,  A2 = G_h S_E^T
//   rows    h~'  = [ A1          , A2          , I     ]
//           y'   = [ S_E A1      , S_E A2      , S_E   ]
//           e~'' = [ I - G_e K A1, -G_e K A2   , -G_e K]
//           probe rows: E probe [v^T, 0, 0];  H probe v^T [A1, A2, I]
template <typename T>
int Impl<T>::build_fused(const fdtd_probes* probes) {
  std::vector<fdtd::FusedBlock<T>> fb;
  std::vector<int2> ctas;
  const int PADC = 32 * (16 / (int)sizeof(T));   // lanes x vector width
  int maxN = 1, maxCp = 0;
  for (auto& D : blocks)
    if (D.fused) {
      maxN = std::max(maxN, D.N);
      maxCp = std::max(maxCp, (D.qe + D.n_if + D.qh + PADC - 1) / PADC * PADC);
    }
  NPsel = maxN <= 4 ? 4 : maxN <= 8 ? 8 : maxN <= 16 ? 16 : 32;
  // batched blocks (N >= 4 columns) take the cluster-split SIMT GEMM kernel,
  // single-column ones the warp-per-row GEMV kernel (FDTD_FUSED=gemv|gemm
  // overrides); the GEMM kernel's shared memory must fit
  {
    const int TRg = 8 * (32 / NPsel) * gemm_rpw(NPsel);
    if (NPsel == 32) {
      gks = 8;                  // measured: config 5 53.2 (K-split 8) vs 52.2 (4) vs 50.8 (2) Gcell/s
      if (const char* e = getenv("FDTD_GEMM_KS")) { const int k = atoi(e); if (k == 2 || k == 4 || k == 8) gks = k; }
    }
    const size_t need = (size_t)(TRg * NPsel + TRg * (maxCp / gks + 2)) * sizeof(double) +
                        (size_t)maxCp / gks * NPsel * sizeof(T);
    fused_gemm = maxN >= 4;
    if (const char* e = getenv("FDTD_FUSED")) fused_gemm = std::string(e) == "gemm";
    if (need > 200 * 1024) fused_gemm = false;
  }
  const int ROWS = fused_gemm ? 8 * (32 / NPsel) * gemm_rpw(NPsel) : 8;   // rows per tile / CTA
  for (int b = 0; b < (int)blocks.size(); ++b) {
    BlockDev<T>& D = blocks[b];
    if (!D.fused) continue;
    const int qe = D.qe, qh = D.qh, ni = D.n_if;
    const int CM = qe + ni + qh;
    const int np = (int)D.probe_rows.size();
    const int RM = qh + ni + qe + np;
    std::vector<double> A1((size_t)qh * qe), A2((size_t)qh * ni);
    for (int r = 0; r < qh; ++r) {
      for (int c = 0; c < qe; ++c) A1[(size_t)r * qe + c] = D.gh[r] * D.K[(size_t)c * qh + r];
      for (int c = 0; c < ni; ++c) A2[(size_t)r * ni + c] = D.gh[r] * D.SE[(size_t)c * qh + r];
    }
    std::vector<double> M((size_t)RM * CM, 0.0);
    auto at = [&](int r, int c) -> double& { return M[(size_t)r * CM + c]; };
    // h~' rows
    for (int r = 0; r < qh; ++r) {
      for (int c = 0; c < qe; ++c) at(r, c) = A1[(size_t)r * qe + c];
      for (int c = 0; c < ni; ++c) at(r, qe + c) = A2[(size_t)r * ni + c];
      at(r, qe + ni + r) = 1.0;
    }
    // y' rows = S_E * (h~' rows)
    for (int l = 0; l < ni; ++l)
      for (int k = 0; k < qh; ++k) {
        const double s = D.SE[(size_t)l * qh + k];
        if (s == 0.0) continue;
        for (int c = 0; c < CM; ++c) at(qh + l, c) += s * at(k, c);
      }
    // e~'' rows = [I, 0, 0] - G_e K (h~' rows)
    for (int r = 0; r < qe; ++r) {
      const int rr = qh + ni + r;
      at(rr, r) = 1.0;
      for (int k = 0; k < qh; ++k) {
        const double s = D.ge[r] * D.K[(size_t)r * qh + k];
        if (s == 0.0) continue;
        for (int c = 0; c < CM; ++c) at(rr, c) -= s * at(k, c);
      }
    }
    // probe rows
    std::vector<int> prow_probe(np), prow_inst(np);
    for (int q = 0; q < np; ++q) {
      const int p = D.probe_rows[q];
      const int rr = qh + ni + qe + q;
      prow_probe[q] = p;
      prow_inst[q] = probes->inst[p];
      for (int64_t k = probes->rowptr[p]; k < probes->rowptr[p + 1]; ++k) {
        const int idx = (int)probes->index[k];
        const double wv = probes->weight[k];
        if (probes->kind[p] == 1) at(rr, idx) += wv;
        else for (int c = 0; c < CM; ++c) at(rr, c) += wv * at(idx, c);
      }
    }
    const int Cp = (CM + PADC - 1) / PADC * PADC;
    const int RMp = (RM + ROWS - 1) / ROWS * ROWS;      // zero rows up to a whole tile
    std::vector<T> Mt((size_t)RMp * Cp, (T)0);
    // device column order [e~ ; h~ ; G] (composition above in [e~ ; G ; h~]):
    // the G columns last, so a consumer can contract the e~, h~ part before
    // G arrives (persist2d.cuh) in the same per-lane order as one pass
    auto dcol = [&](int c) { return c < qe ? c : (c < qe + ni ? qe + qh + (c - qe) : qe + (c - qe - ni)); };
    for (int r = 0; r < RM; ++r)
      for (int c = 0; c < CM; ++c) Mt[(size_t)r * Cp + dcol(c)] = (T)M[(size_t)r * CM + c];
    D.M_d = dalloc<T>(Mt.size());
    if (!D.M_d || upload(D.M_d, Mt)) return fail(FDTD_ENOMEM, "fused matrix allocation failed");
    // fp32: the composed matrix is stored compensated, M = hi (fp32) + lo
    // (bf16 of the fp32 remainder), relative error ~2^-33 (reading R14): the
    // rounding of one fp32 M alone drifts the reduced state coherently
    // (config 2: 1.2e-4 after 20,000 steps against the fp64 oracle)
    uint16_t* Ml_d = nullptr;
    if (sizeof(T) == 4) {
      std::vector<uint16_t> Ml((size_t)RMp * Cp, 0);
      for (int r = 0; r < RM; ++r)
        for (int c = 0; c < CM; ++c) {
          const double m = M[(size_t)r * CM + c];
          const float rem = (float)(m - (double)(float)m);
          uint32_t u;
          std::memcpy(&u, &rem, 4);
          u += 0x7fffu + ((u >> 16) & 1u);                 // round to nearest even
          Ml[(size_t)r * Cp + dcol(c)] = (uint16_t)(u >> 16);
        }
      Ml_d = dalloc<uint16_t>(Ml.size());
      if (!Ml_d || upload(Ml_d, Ml)) return fail(FDTD_ENOMEM, "fused matrix allocation failed");
    }
    double* M64_d = nullptr;
    if (sizeof(T) == 4 && fused_gemm) {
      std::vector<double> M64((size_t)RMp * Cp, 0.0);
      for (int r = 0; r < RM; ++r)
        for (int c = 0; c < CM; ++c) M64[(size_t)r * Cp + dcol(c)] = M[(size_t)r * CM + c];
      M64_d = dalloc<double>(M64.size());
      if (!M64_d || upload(M64_d, M64)) return fail(FDTD_ENOMEM, "fused matrix allocation failed");
    }
    D.R_M = RM; D.C_M = CM;
    fdtd::FusedBlock<T> f{};
    f.qe = qe; f.qh = qh; f.n_if = ni; f.N = D.N; f.R = RM; f.C = CM; f.Cp = Cp; f.M = D.M_d; f.Ml = Ml_d; f.M64 = M64_d;
    f.e_off = D.e_off; f.h_off = D.h_off; f.y_off = D.y_off;
    f.n_probe_rows = np;
    int32_t* pp = dalloc<int32_t>(std::max(np, 1));
    int32_t* pi = dalloc<int32_t>(std::max(np, 1));
    if (upload(pp, prow_probe) || upload(pi, prow_inst)) return FDTD_ECUDA;
    f.probe_id = pp; f.probe_inst = pi;
    fb.push_back(f);
    for (int r0 = 0; r0 < RM; r0 += ROWS) ctas.push_back(make_int2((int)fb.size() - 1, r0));
    maxN = std::max(maxN, D.N);
    max_cols = std::max(max_cols, Cp);
  }
  rows_per_cta = ROWS;
  n_ctas = (int)ctas.size();
  NBsel = maxN <= 1 ? 1 : maxN <= 4 ? 4 : maxN <= 16 ? 16 : 32;
  fused_smem = fused_gemm ? (size_t)(ROWS * NPsel + ROWS * (max_cols / gks + 2)) * sizeof(double) +
                                (size_t)max_cols / gks * NPsel * sizeof(T)
                          : (size_t)max_cols * maxN * sizeof(T);
  if (fused_smem > 200 * 1024)
    return fail(FDTD_ENOTSUP, "fused reduced kernel needs %zu bytes of shared memory (> 200 KB)", fused_smem);
  if ((int)fb.size() > fdtd::kMaxFusedBlocks)
    return fail(FDTD_ENOTSUP, "more than %d fused reduced blocks (model classes)", fdtd::kMaxFusedBlocks);
  fblocks = fb;
  tile0.assign(1, 0);
  for (size_t b = 0; b < fb.size(); ++b) {
    int nt = 0;
    for (auto& c : ctas) nt += (c.x == (int)b);
    tile0.push_back(tile0.back() + nt);
  }
  return FDTD_OK;
}

// e~^{s+1} = e~^s - G_e K~' h~^{s+1/2} and y^s = S_E h~^{s+1/2} after the
// reduced state was (re)set: the fused step consumes e~ one step ahead.
template <typename T>
int Impl<T>::prologue(cudaStream_t st) {
  for (auto& D : blocks) {
    if (!D.fused) {
      if (D.n_if > 0)
        launch_rowblock<T>(D.n_if, D.qh, D.Kph, D.N, D.SEp_d, h_state(D, host_step), y_all + D.y_off,
                           (const T*)nullptr, (T)1, false, d_step, 0, d_bad, st);
      continue;
    }
    if (D.n_if > 0)
      launch_gemv<T>(D.n_if, D.qh, D.N, D.SE_d, h_state(D, host_step), y_all + D.y_off, (const T*)nullptr,
                     (T)1, false, d_step, 0, d_bad, st);
    CK(cudaMemcpyAsync(e_ahead(D, host_step), e_state(D, host_step), sizeof(T) * D.qe * D.N,
                       cudaMemcpyDeviceToDevice, st));
    launch_gemv<T>(D.qe, D.qh, D.N, D.K_d, h_state(D, host_step), e_ahead(D, host_step), D.ge_d,
                   (T)-1, true, d_step, 0, d_bad, st);
  }
  CK(cudaGetLastError());
  return FDTD_OK;
}

// The explicit rows of the step of parity p (rows_prepass_*_kernel): E^{n+1} of
// every interface / source row into the new parity, G published.
template <typename T>
int Impl<T>::prepass(int p, cudaStream_t st) {
  fdtd::Fields<T> F0, F1;
  for (int c = 0; c < 6; ++c) { F0.f[c] = F[p][c]; F1.f[c] = F[p ^ 1][c]; }
  const int64_t nt = rows.n_rows * B;
  if (rowpack_i)
    fdtd::rows_prepass_packed_kernel<T><<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(
        rows.n_rows, rowpack_i, (const fdtd::RowPackR<T>*)rowpack_r, B, F0, F1, y_all, g_of(p), rows.wave,
        rows.n_wave, rows.n_src, d_step + p, lossy ? 1 : 0);
  else
    fdtd::rows_prepass_kernel<T><<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(rows, B, F0, F1, y_all, d_step + p);
  CK(cudaGetLastError());
  return FDTD_OK;
}

template <typename T>
int Impl<T>::launch_step(int p, cudaStream_t st, int64_t* count, bool profile) {
  int64_t n = 0;
  const int64_t* ds = d_step + p;          // this step's counter slot (the fused kernel writes the other)
  auto mark = [&](int ph, int edge) {
    if (profile) cudaEventRecord(ev[(size_t)prof_pending * 2 * NPHASE + 2 * ph + edge], st);
  };
  fdtd::Fields<T> F0, F1;
  for (int c = 0; c < 6; ++c) { F0.f[c] = F[p][c]; F1.f[c] = F[p ^ 1][c]; }
  // a1-a3 + a5: fused coarse stencil with the explicit rows evaluated in place
  mark(0, 0);
  const size_t tabsz = uniform ? 0 : sizeof(fdtd::MatTable<T>);
  const fdtd::Dims dm{nx, ny, nz, px, B, plane};
  // split step (§5.6): interface columns (A) now, the reduced update on st2,
  // the other columns (B) beside it, then the probe / counter tail
  const bool sp = split && !profile;
  fdtd::TileSplit SA = tsplit, SB = tsplit;
  if (sp) {
    const int nch = tsplit.nitems / tsplit.ncols;
    SA.colperm = SB.colperm = colperm_d;
    SA.col0 = 0; SA.ncols = n_ifc; SA.nitems = n_ifc * nch;
    SB.col0 = n_ifc; SB.ncols = tsplit.ncols - n_ifc; SB.nitems = SB.ncols * nch;
  }
  const cudaStream_t rs = sp ? st2 : st;    // the reduced update's stream
  if (dim == 3 && use_tile && rows.n_rows > 0 && !(fuse_rows && rows_ahead)) {
    // explicit rows first: the tile stencil reads their E^{n+1} back from the new parity
    // (with fused rows only when the previous step's reduced kernel has not done it)
    int e = prepass(p, st);
    if (e) return e;
    ++n;
  }
  if (dim == 3 && use_tile && sp) {
    CK(fdtd::tile_launch<T>(tcfg, uniform, SA.nitems, tile_smem, st, tma[p], SA, dm, F0, F1, mat_id, tab,
                            ifm, n_mat, u0, u1, rows, y_all, ds, check_every, d_bad, lossy ? tab_a : nullptr));
    CK(cudaEventRecord(evA, st));
    CK(cudaStreamWaitEvent(st2, evA, 0));
  } else if (dim == 3 && use_tile) {
    CK(fdtd::tile_launch<T>(tcfg, uniform, tile_grid, tile_smem, st, tma[p], tsplit, dm, F0, F1, mat_id, tab,
                            ifm, n_mat, u0, u1, rows, y_all, ds, check_every, d_bad, lossy ? tab_a : nullptr));
  } else if (dim == 3 && use_tma) {
    constexpr int NS = 3;
    const int BX = tBX, BY = tBY;
    const int outx = tOUTX, outy = BY - 1;
    const int kchunk = zchunk(((nx + 1 + outx - 1) / outx) * ((ny + 1 + outy - 1) / outy));
    dim3 grid((nx + 1 + outx - 1) / outx, (ny + 1 + outy - 1) / outy, (nz + 1 + kchunk - 1) / kchunk);
    const int al = 128 / (int)sizeof(T);
    const size_t HPp = (size_t)(tHBX * (BY + 1) + al - 1) / al * al, EPp = (size_t)(BX * BY + al - 1) / al * al;
    const size_t sm = 256 + (NS * 3 * HPp + NS * 3 * EPp + 3 * 3 * EPp) * sizeof(T) + tabsz;
    if (tW > 1) {
      if (uniform)
        fdtd::stencil3d_tma_vec_kernel<T, true, NS, kW><<<grid, dim3(BX / kW, BY), sm, st>>>(
            tma[p], tHBX, tSX, tOUTX, dm, F0, F1, mat_id, tab, ifm, n_mat, u0, u1, rows, y_all, kchunk, ds, check_every, d_bad);
      else
        fdtd::stencil3d_tma_vec_kernel<T, false, NS, kW><<<grid, dim3(BX / kW, BY), sm, st>>>(
            tma[p], tHBX, tSX, tOUTX, dm, F0, F1, mat_id, tab, ifm, n_mat, u0, u1, rows, y_all, kchunk, ds, check_every, d_bad);
    } else if (uniform)
      fdtd::stencil3d_tma_kernel<T, true, NS><<<grid, dim3(BX, BY), sm, st>>>(
          tma[p], tHBX, tSX, tOUTX, dm, F0, F1, mat_id, tab, ifm, n_mat, u0, u1, rows, y_all, kchunk, ds, check_every, d_bad);
    else
      fdtd::stencil3d_tma_kernel<T, false, NS><<<grid, dim3(BX, BY), sm, st>>>(
          tma[p], tHBX, tSX, tOUTX, dm, F0, F1, mat_id, tab, ifm, n_mat, u0, u1, rows, y_all, kchunk, ds, check_every, d_bad);
  } else if (dim == 3) {
    constexpr int NS = 3;
    int BX, BY;
    if (B == 1) { BX = 32; BY = 8; }
    else { BX = B * std::max(2, 32 / B); BY = std::max(2, 256 / BX); if (BX * BY > 256) BY = 256 / BX; }
    const int outx = BX / B - 1, outy = BY - 1;
    const int kchunk = zchunk(((nx + 1 + outx - 1) / outx) * ((ny + 1 + outy - 1) / outy));
    dim3 grid((nx + 1 + outx - 1) / outx, (ny + 1 + outy - 1) / outy, (nz + 1 + kchunk - 1) / kchunk);
    const size_t sm = (size_t)(NS * 3 * (BX + B) * (BY + 1) + NS * 3 * BX * BY + 2 * 3 * BX * BY) * sizeof(T) + tabsz;
    if (uniform)
      fdtd::stencil3d_pipe_kernel<T, true, NS><<<grid, dim3(BX, BY), sm, st>>>(
          dm, F0, F1, mat_id, tab, ifm, n_mat, u0, u1, rows, y_all, kchunk, ds, check_every, d_bad);
    else
      fdtd::stencil3d_pipe_kernel<T, false, NS><<<grid, dim3(BX, BY), sm, st>>>(
          dm, F0, F1, mat_id, tab, ifm, n_mat, u0, u1, rows, y_all, kchunk, ds, check_every, d_bad);
  } else {
    constexpr int CY = 4;
    int BX = (B == 1) ? 32 : B * std::max(2, 32 / B), BY = 8;
    if (BX * BY > 256) BY = std::max(1, 256 / BX);
    const int outx = BX / B - 1, outy = BY * CY - 1;
    dim3 grid((nx + 1 + outx - 1) / outx, (ny + 1 + outy - 1) / outy, 1);
    const size_t sm = (size_t)BX * BY * CY * sizeof(T) + tabsz;
    if (uniform)
      fdtd::stencil2d_rows_kernel<T, true, CY><<<grid, dim3(BX, BY), sm, st>>>(
          dm, F0, F1, mat_id, tab, ifm, n_mat, u0, u1, rows, y_all, ds, check_every, d_bad, nullptr);
    else
      fdtd::stencil2d_rows_kernel<T, false, CY><<<grid, dim3(BX, BY), sm, st>>>(
          dm, F0, F1, mat_id, tab, ifm, n_mat, u0, u1, rows, y_all, ds, check_every, d_bad, lossy ? tab_a : nullptr);
  }
  ++n;
  mark(0, 1);
  // leapfrog path for large blocks (grid-wide GEMVs in the paper's order)
  if (any_leap) {
    mark(2, 0);
    for (auto& D : blocks) {
      if (D.fused) continue;
      T* e = eb[0] + D.e_off;
      T* h = hb[0] + D.h_off;
      if constexpr (sizeof(T) == 4) {
        if (D.splits > 0) {
          // a4: e~ -= G_e K~' h~  (split-K TN on K~'^T, then the axpy with -g_e)
          n += launch_gemm_tn(D.qh, D.qe, D.Kpe, D.N, D.ks, (const float*)D.KTp_d, (const float*)h,
                              D.parte_d, rs);
          fdtd::reduce_axpy_f32_kernel<<<(D.qe * D.N + 31) / 32, 256, 0, rs>>>(
              D.qe, D.N, D.ks, D.parte_d, nullptr, (const float*)D.gen_d, (float*)e, nullptr);
          ++n;
          // a6: h~ += G_h (K~'^T e~ + S_E^T G): both as split-K partials into one
          // buffer, summed in a fixed order; y = S_E h~ (tensor cores or SIMT)
          n += launch_gemm_tn(D.qe, D.qh, D.Kph, D.N, D.ks, (const float*)D.Kp_d, (const float*)e,
                              D.part_d, rs);
          if (D.wide) {
            const dim3 gw((D.qh + fdtd::WTC - 1) / fdtd::WTC, D.splits);
            if (D.wide_ng == 2)
              fdtd::gemm_tn_f32_wide_kernel<2><<<gw, 256, fdtd::gemm_tn_wide_smem(), rs>>>(
                  D.n_if, D.qh, D.Kph, (const float*)D.SEp_d, (const float*)(g_all + D.y_off),
                  D.part_d + (size_t)D.ks * D.qh * D.N);
            else
              fdtd::gemm_tn_f32_wide_kernel<4><<<gw, 512, fdtd::gemm_tn_wide_smem(), rs>>>(
                  D.n_if, D.qh, D.Kph, (const float*)D.SEp_d, (const float*)(g_all + D.y_off),
                  D.part_d + (size_t)D.ks * D.qh * D.N);
            ++n;
          } else {
            n += launch_gemm_tn(D.n_if, D.qh, D.Kph, D.N, D.splits, (const float*)D.SEp_d,
                                (const float*)(g_all + D.y_off), D.part_d + (size_t)D.ks * D.qh * D.N, rs);
          }
          fdtd::reduce_axpy_f32_kernel<<<(D.qh * D.N + 31) / 32, 256, 0, rs>>>(
              D.qh, D.N, D.ks + D.splits, D.part_d, nullptr, (const float*)D.gh_d, (float*)h,
              D.tc ? D.xs_d : nullptr);
          ++n;
          if (D.tc) {
            const int tiles = (D.n_if + fdtd::tc::BM - 1) / fdtd::tc::BM;
            fdtd::tc::tc_skinny_gemm_kernel<<<std::min(tiles, tc_grid), fdtd::tc::NTHREADS, fdtd::tc::SMEM_BYTES, rs>>>(
                D.se_map, D.n_if, D.qh, D.xs_d, (float*)(y_all + D.y_off), ds, check_every, d_bad);
            ++n;
          } else {
            n += launch_gemm_nn(D.n_if, D.qh, D.Kph, D.N, (const float*)D.SEp_d, (const float*)h,
                                (float*)(y_all + D.y_off), nullptr, 1.f, false, ds, check_every, d_bad, rs);
          }
          continue;
        }
      }
      // a4: e~ -= G_e K~' h~^{n+1/2}
      n += launch_rowblock<T>(D.qe, D.qh, D.Kph, D.N, D.Kp_d, h, e, D.ge_d, (T)-1, true, ds, check_every, d_bad, rs);
      // a6: T = K~'^T e~ + S_E^T G ; h~ += G_h T ; y = S_E h~
      n += launch_rowblock<T>(D.qh, D.qe, D.Kpe, D.N, D.KTp_d, e, D.Tv_d, (const T*)nullptr, (T)1, false, ds, 0,
                              d_bad, rs);
      if (D.n_if > 0) n += launch_colsum<T>(D.n_if, D.qh, D.Kph, D.N, D.SEp_d, g_all + D.y_off, D.Tv_d, rs);
      fdtd::axpy_diag_kernel<T><<<(D.qh * D.N + 255) / 256, 256, 0, rs>>>(D.qh, D.N, D.gh_d, D.Tv_d, h);
      ++n;
      if (D.n_if > 0)
        n += launch_rowblock<T>(D.n_if, D.qh, D.Kph, D.N, D.SEp_d, h, y_all + D.y_off, (const T*)nullptr, (T)1, false,
                                ds, check_every, d_bad, rs);
    }
    mark(2, 1);
  }
  // fused reduced blocks (one GEMV phase) + probes + step counter
  mark(1, 0);
  fdtd::FusedParams<T> P{};
  for (size_t b = 0; b < fblocks.size(); ++b) P.fb[b] = fblocks[b];
  for (size_t b = 0; b < tile0.size(); ++b) P.tile0[b] = tile0[b];
  P.nfb = (int)fblocks.size();
  P.n_ctas = n_ctas;
  P.B = B;
  P.e_in = eb[p]; P.e_out = eb[p ^ 1];
  P.h_in = hb[p]; P.h_out = hb[p ^ 1];
  P.y = y_all;
  P.G = g_of(p);
  P.fuse_rows = fuse_rows ? 1 : 0;
  if (fuse_rows) {
    P.lossy_rows = lossy ? 1 : 0;
    P.rp_i = rowpack_i; P.rp_r = rowpack_r; P.y_row = y_row_d; P.src_rows = src_rows_d; P.n_src_rows = n_src_rows;
    P.Fn0 = F1; P.Fn1 = F0;
    P.g_next = g_of(p ^ 1);
    P.wave = rows.wave; P.n_wave = rows.n_wave; P.n_wsrc = rows.n_src;
  }
  P.rows_per_cta = rows_per_cta;
  P.red_base[0] = eb[0];      // leap-frog blocks (fused blocks' probes are matrix rows)
  P.red_base[1] = hb[0];
  P.F = F1;
  P.pr = pr;
  P.ring = ring;
  P.cap = cap;
  P.d_step = d_step + p;
  P.d_step_next = d_step + (p ^ 1);
  P.check_every = check_every;
  P.bad_step = d_bad;
  const size_t sm = fused_smem;
  P.tail_mode = sp ? 1 : 0;
  // optional programmatic dependent launch (the kernels wait with
  // griddepcontrol.wait before reading anything the preceding kernel writes;
  // without the attribute the wait is a no-op)
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t lc = {};
  lc.blockDim = dim3(256);
  lc.dynamicSmemBytes = sm;
  lc.stream = rs;
  lc.attrs = (use_pdl && !sp) ? pdl : nullptr;
  lc.numAttrs = (use_pdl && !sp) ? 1 : 0;
  if (sp && n_ctas == 0) {
    // leap-frog blocks only: nothing fused to run on st2
  } else if (fused_gemm) {
    lc.gridDim = dim3((unsigned)(std::max(n_ctas, 1) * gks));
    switch (NPsel) {
      case 4: CK(cudaLaunchKernelEx(&lc, fdtd::reduced_gemm_kernel<T, 4, gemm_rpw(4), GEMM_KS>, P)); break;
      case 8: CK(cudaLaunchKernelEx(&lc, fdtd::reduced_gemm_kernel<T, 8, gemm_rpw(8), GEMM_KS>, P)); break;
      case 16: CK(cudaLaunchKernelEx(&lc, fdtd::reduced_gemm_kernel<T, 16, gemm_rpw(16), GEMM_KS>, P)); break;
      default:
        if (gks == 2) CK(cudaLaunchKernelEx(&lc, fdtd::reduced_gemm_kernel<T, 32, gemm_rpw(32), 2>, P));
        else if (gks == 8) CK(cudaLaunchKernelEx(&lc, fdtd::reduced_gemm_kernel<T, 32, gemm_rpw(32), 8>, P));
        else CK(cudaLaunchKernelEx(&lc, fdtd::reduced_gemm_kernel<T, 32, gemm_rpw(32), GEMM_KS>, P));
        break;
    }
  } else {
    lc.gridDim = dim3((unsigned)std::max(n_ctas, 1));
    switch (NBsel) {
      case 1: CK(cudaLaunchKernelEx(&lc, fdtd::reduced_fused_kernel<T, 1>, P)); break;
      case 4: CK(cudaLaunchKernelEx(&lc, fdtd::reduced_fused_kernel<T, 4>, P)); break;
      case 16: CK(cudaLaunchKernelEx(&lc, fdtd::reduced_fused_kernel<T, 16>, P)); break;
      default: CK(cudaLaunchKernelEx(&lc, fdtd::reduced_fused_kernel<T, 32>, P)); break;
    }
  }
  if (!(sp && n_ctas == 0)) ++n;
  if (sp) {
    CK(cudaEventRecord(evR, st2));
    CK(fdtd::tile_launch<T>(tcfg, uniform, SB.nitems, tile_smem, st, tma[p], SB, dm, F0, F1, mat_id, tab,
                            ifm, n_mat, u0, u1, rows, y_all, ds, check_every, d_bad, lossy ? tab_a : nullptr));
    CK(cudaStreamWaitEvent(st, evR, 0));
    // probes (coarse fields after the whole stencil) and the step counter
    fdtd::FusedParams<T> Q = P;
    Q.n_ctas = 0;
    Q.tail_mode = 0;
    fdtd::reduced_fused_kernel<T, 1><<<1, 256, 0, st>>>(Q);
    n += 2;
  }
  mark(1, 1);
  CK(cudaGetLastError());
  if (fuse_rows) rows_ahead = true;          // the reduced kernel evaluated the next step's rows
  if (profile && ++prof_pending == NPOOL) {
    int e = flush_profile();
    if (e) return e;
  }
  *count += n;
  return FDTD_OK;
}

template <typename T>
int Impl<T>::drain() {
  const int64_t from = drained_to, to = host_step;
  if (to <= from || n_probe == 0) { drained_to = to; return FDTD_OK; }
  CK(cudaStreamSynchronize(stream));
  const int64_t per = (int64_t)n_probe * B;
  std::vector<T> buf((size_t)((to - from) * per));
  int64_t done = 0;
  while (done < to - from) {
    const int64_t s = from + done + step_offset;
    const int64_t pos = s % cap;
    const int64_t len = std::min(cap - pos, (to - from) - done);
    CK(cudaMemcpy(buf.data() + done * per, ring + pos * per, sizeof(T) * len * per, cudaMemcpyDeviceToHost));
    done += len;
  }
  const size_t old = host_probes.size();
  host_probes.resize(old + buf.size());
  for (size_t q = 0; q < buf.size(); ++q) host_probes[old + q] = (double)buf[q];
  drained_to = to;
  return FDTD_OK;
}

template <typename T>
int Impl<T>::step(int64_t n) {
  if (n < 0) return fail(FDTD_EINVAL, "negative step count");
  while (n > 0) {
    if (n_probe > 0 && host_step - drained_to >= cap) {
      int e = drain();
      if (e) return e;
    }
    const int64_t room = n_probe > 0 ? cap - (host_step - drained_to) : n;
    const int64_t chunk = std::min(n, room);
    int64_t done = 0;
    if (persist && !prof && graph_steps > 0 && chunk > 0) {
      // one launch runs at most 2^30 steps (the kernel's step count and the
      // LL exchange tags are 32-bit)
      while (done < chunk) {
        const int64_t part = std::min<int64_t>(chunk - done, (int64_t)1 << 30);
        int e = launch_persist(part, &launches);
        if (e) return e;
        host_step += part;
        done += part;
      }
    }
    while (done < chunk) {
      const int64_t left = chunk - done;
      if (!prof && graph_steps > 0 && (host_step & 1) == 0 && left >= graph_steps) {
        if (fuse_rows && !rows_ahead) {
          // the captured steps carry no pre-pass: evaluate the first step's rows here
          int e = prepass((int)(host_step & 1), stream);
          if (e) return e;
          ++launches;
          rows_ahead = true;
        }
        if (!graph) {
          cudaStream_t cs;
          CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
          cudaGraph_t gr;
          CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
          int64_t cnt = 0;
          int e = FDTD_OK;
          for (int s = 0; s < graph_steps && e == FDTD_OK; ++s) e = launch_step(s & 1, cs, &cnt);
          cudaError_t ce = cudaStreamEndCapture(cs, &gr);
          if (e) { cudaStreamDestroy(cs); return e; }
          CK(ce);
          CK(cudaGraphInstantiate(&graph, gr, 0));
          CK(cudaGraphDestroy(gr));
          CK(cudaStreamDestroy(cs));
          graph_kernels = cnt;
        }
        CK(cudaGraphLaunch(graph, stream));
        launches += graph_kernels;
        host_step += graph_steps;
        done += graph_steps;
      } else {
        int e = launch_step((int)(host_step & 1), stream, &launches, prof);
        if (e) return e;
        host_step += 1;
        done += 1;
      }
    }
    n -= chunk;
  }
  return FDTD_OK;
}

template <typename T>
int Impl<T>::check_async() {
  unsigned long long bad = 0;
  if (persist) {
    int ab = 0;
    CK(cudaMemcpy(&ab, p_flags + 2 * pntx * pnty + 2, sizeof(ab), cudaMemcpyDeviceToHost));
    if (ab) return fail(FDTD_ECUDA, "persistent 2-D kernel: inter-CTA wait timed out (watchdog)");
  }
  CK(cudaMemcpy(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost));
  if (bad != std::numeric_limits<unsigned long long>::max())
    return fail(FDTD_EDIVERGED, "divergence (non-finite or |x| > 1e100) detected at step %llu", bad);
  return FDTD_OK;
}

template <typename T>
int Impl<T>::sync() {
  CK(cudaStreamSynchronize(stream));
  if (mem.guard) {
    long long where = 0;
    const int b = mem.check(&where);
    if (b >= 0)
      return fail(FDTD_ECUDA, "FDTD_GUARD: out-of-bounds write next to device buffer #%d (%zu bytes) at byte offset %lld",
                  b, mem.sizes[b], where);
  }
  return check_async();
}

template <typename T>
int Impl<T>::probe(double* out, int64_t capn, int64_t* written) {
  int e = drain();
  if (e) return e;
  const int64_t need = (int64_t)host_probes.size();
  if (written) *written = 0;
  if (need > capn) return fail(FDTD_EINVAL, "probe buffer too small: need %lld doubles", (long long)need);
  if (need) std::memcpy(out, host_probes.data(), sizeof(double) * need);
  if (written) *written = need;
  host_probes.clear();
  return check_async();
}

template <typename T>
int Impl<T>::get_state(int which, double* out, int64_t n) {
  CK(cudaStreamSynchronize(stream));
  const int p = (int)(host_step & 1);
  if (which >= 0 && which <= 5) {
    if (n != S * B) return fail(FDTD_EINVAL, "get_state: n must be batch*S = %lld", (long long)(S * B));
    if (!F[p][which]) { std::fill(out, out + n, 0.0); return FDTD_OK; }
    CK(cudaMemcpy(staging, F[p][which], sizeof(T) * elems, cudaMemcpyDeviceToHost));
    for (int64_t s = 0; s < S; ++s) {
      const int64_t o = dev_off(s) * B;
      for (int b = 0; b < B; ++b) out[(int64_t)b * S + s] = (double)staging[o + b];
    }
    return check_async();
  }
  if (which == 6 || which == 7) {
    int64_t tot = 0;
    for (auto& D : blocks) tot += (int64_t)(which == 6 ? D.qe : D.qh) * D.N;
    if (n != tot) return fail(FDTD_EINVAL, "get_state: n must be %lld", (long long)tot);
    int64_t o = 0;
    for (auto& D : blocks) {
      const int q = which == 6 ? D.qe : D.qh;
      const T* srcp = which == 6 ? e_state(D, host_step) : h_state(D, host_step);
      CK(cudaMemcpy(staging, srcp, sizeof(T) * q * D.N, cudaMemcpyDeviceToHost));
      for (int in = 0; in < D.n_inst; ++in)
        for (int b = 0; b < B; ++b)
          for (int c = 0; c < q; ++c) out[o++] = (double)staging[(int64_t)c * D.N + in * B + b];
    }
    return check_async();
  }
  if (which == 8) {
    if (n != 1) return fail(FDTD_EINVAL, "get_state(8): n must be 1");
    int64_t s = 0;
    CK(cudaMemcpy(&s, d_step + (host_step & 1), sizeof(s), cudaMemcpyDeviceToHost));
    out[0] = (double)s;
    return FDTD_OK;
  }
  return fail(FDTD_EINVAL, "get_state: bad 'which' %d", which);
}

template <typename T>
int Impl<T>::set_state(int which, const double* in, int64_t n) {
  CK(cudaStreamSynchronize(stream));
  rows_ahead = false;
  const int p = (int)(host_step & 1);
  if (which >= 0 && which <= 5) {
    if (n != S * B) return fail(FDTD_EINVAL, "set_state: n must be batch*S");
    if (!F[p][which]) return fail(FDTD_EINVAL, "set_state: component %d unused in 2-D", which);
    if (!getenv("FDTD_HOST_SET_STATE")) {
      // on the device: copy the fp64 array, then one scatter / round / mask kernel
      if (!d_in64) {                  // S * B is fixed per handle: allocated once (owned until destroy)
        d_in64 = dalloc<double>(S * B);
        d_in64_n = d_in64 ? S * B : 0;
      }
      if (d_in64) {
        CK(cudaMemsetAsync(F[p][which], 0, sizeof(T) * elems, stream));
        CK(cudaMemcpyAsync(d_in64, in, sizeof(double) * S * B, cudaMemcpyHostToDevice, stream));
        const int64_t tot = S * B;
        fdtd::state_scatter_kernel<T><<<(unsigned)((tot + 255) / 256), 256, 0, stream>>>(
            d_in64, S, B, nx, ny, nz, px, dim, which, dim == 3 && which <= 2, F[p][which]);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(stream));
        return FDTD_OK;
      }
    }
    std::fill(staging, staging + elems, (T)0);
    // 3-D E entries that are not unknowns (tangential E on the PEC walls) are
    // stored as 0: the stencil keeps their old value (stencil3d.cuh)
    const bool mask_e = dim == 3 && which <= 2;
    for (int64_t s = 0; s < S; ++s) {
      if (mask_e) {
        const int64_t i = s % (nx + 1), j = (s / (nx + 1)) % (ny + 1), k = s / ((int64_t)(nx + 1) * (ny + 1));
        const bool xi = i > 0 && i < nx, yi = j > 0 && j < ny, zi = k > 0 && k < nz;
        const bool unk = which == 0 ? (i < nx && yi && zi) : which == 1 ? (xi && j < ny && zi) : (xi && yi && k < nz);
        if (!unk) continue;
      }
      const int64_t o = dev_off(s) * B;
      for (int b = 0; b < B; ++b) staging[o + b] = (T)in[(int64_t)b * S + s];
    }
    CK(cudaMemcpy(F[p][which], staging, sizeof(T) * elems, cudaMemcpyHostToDevice));
    return FDTD_OK;
  }
  if (which == 6 || which == 7) {
    int64_t tot = 0;
    for (auto& D : blocks) tot += (int64_t)(which == 6 ? D.qe : D.qh) * D.N;
    if (n != tot) return fail(FDTD_EINVAL, "set_state: n must be %lld", (long long)tot);
    int64_t o = 0;
    for (auto& D : blocks) {
      const int q = which == 6 ? D.qe : D.qh;
      T* dst = which == 6 ? e_state(D, host_step) : h_state(D, host_step);
      for (int in_ = 0; in_ < D.n_inst; ++in_)
        for (int b = 0; b < B; ++b)
          for (int c = 0; c < q; ++c) staging[(int64_t)c * D.N + in_ * B + b] = (T)in[o++];
      CK(cudaMemcpy(dst, staging, sizeof(T) * q * D.N, cudaMemcpyHostToDevice));
    }
    int e = prologue(stream);
    if (e) return e;
    CK(cudaStreamSynchronize(stream));
    return FDTD_OK;
  }
  if (which == 8) {
    if (n != 1) return fail(FDTD_EINVAL, "set_state(8): n must be 1");
    int e = drain();
    if (e) return e;
    const int64_t v = (int64_t)in[0];
    if (v < 0) return fail(FDTD_EINVAL, "set_state(8): negative step");
    CK(cudaMemcpy(d_step + (host_step & 1), &v, sizeof(v), cudaMemcpyHostToDevice));
    step_offset = v - host_step;
    return FDTD_OK;
  }
  return fail(FDTD_EINVAL, "set_state: bad 'which' %d", which);
}

}  // namespace

// ---------------------------------------------------------------------------
extern "C" {

int fdtd_create(const fdtd_grid* g, const fdtd_materials* mat, const fdtd_interface* iface,
                const fdtd_reduced_block* blocks, int32_t n_blocks, const fdtd_sources* src,
                const fdtd_probes* probes, const fdtd_exec* exec, fdtd_t** out) {
  if (!g || !out) return fail(FDTD_EINVAL, "null grid or output handle");
  *out = nullptr;
  if (g->dim != 2 && g->dim != 3) return fail(FDTD_EINVAL, "invalid-grid: dim must be 2 or 3");
  if (g->nx < 1 || g->ny < 1 || (g->dim == 3 && g->nz < 1) || (g->dim == 2 && g->nz != 1))
    return fail(FDTD_EINVAL, "invalid-grid: cell counts");
  if (!(g->dx > 0) || !(g->dy > 0) || (g->dim == 3 && !(g->dz > 0)))
    return fail(FDTD_EINVAL, "invalid-grid: cell sizes must be > 0");
  if (g->dx != g->dy || (g->dim == 3 && g->dx != g->dz))
    return fail(FDTD_ENOTSUP, "this version requires cubic (square) cells");
  if (g->batch < 1 || g->batch > 512) return fail(FDTD_EINVAL, "batch must be in [1, 512]");
  if (g->precision != 32 && g->precision != 64) return fail(FDTD_EINVAL, "precision must be 32 or 64");
  int dev = 0;
  cudaDeviceProp prop;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaGetDeviceProperties(&prop, dev) != cudaSuccess)
    return fail(FDTD_ECUDA, "no CUDA device");
  if (prop.major != 10 || prop.minor != 0)
    return fail(FDTD_ENOTSUP, "libfdtd is built for sm_100a; device is sm_%d%d", prop.major, prop.minor);
  fdtd_t* h = nullptr;
  int e;
  if (g->precision == 32) {
    auto* p = new Impl<float>();
    e = p->create(g, mat, iface, blocks, n_blocks, src, probes, exec);
    h = p;
  } else {
    auto* p = new Impl<double>();
    e = p->create(g, mat, iface, blocks, n_blocks, src, probes, exec);
    h = p;
  }
  if (e != FDTD_OK) {
    delete h;
    return e;
  }
  *out = h;
  return FDTD_OK;
}

int fdtd_step(fdtd_t* h, int64_t n) { return h ? h->step(n) : fail(FDTD_EINVAL, "null handle"); }
int fdtd_probe(fdtd_t* h, double* out, int64_t cap, int64_t* written) {
  return h ? h->probe(out, cap, written) : fail(FDTD_EINVAL, "null handle");
}
int fdtd_get_state(fdtd_t* h, int32_t which, double* out, int64_t n) {
  return h ? h->get_state(which, out, n) : fail(FDTD_EINVAL, "null handle");
}
int fdtd_set_state(fdtd_t* h, int32_t which, const double* in, int64_t n) {
  return h ? h->set_state(which, in, n) : fail(FDTD_EINVAL, "null handle");
}
int fdtd_sync(fdtd_t* h) { return h ? h->sync() : fail(FDTD_EINVAL, "null handle"); }
int64_t fdtd_launch_count(const fdtd_t* h) { return h ? h->launches : 0; }
int32_t fdtd_path(const fdtd_t* h) { return h ? h->path_bits : 0; }
int fdtd_profile(fdtd_t* h, int32_t enable) { return h ? h->set_profile(enable) : fail(FDTD_EINVAL, "null handle"); }
int fdtd_phase_times(fdtd_t* h, double* ms, int32_t n) {
  return h ? h->phase_times(ms, n) : fail(FDTD_EINVAL, "null handle");
}
int fdtd_plane_device(fdtd_t* h, int32_t which, int32_t k, void* dev_buf, int32_t dir) {
  return h ? h->plane_io(which, k, dev_buf, dir) : fail(FDTD_EINVAL, "null handle");
}
void fdtd_destroy(fdtd_t* h) {
  if (h) {
    h->sync();
    delete h;
  }
}
const char* fdtd_last_error(void) { return g_err.c_str(); }
int fdtd_version(void) { return FDTD_VERSION; }

}  // extern "C"
