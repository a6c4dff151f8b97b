// rom.cu — whole-domain reduced model batched over excitations (fdtd_rom.h,
// SURVEY §8(f) NEXT-3; Eq. (12) P:182-185 in the leap-frog order of
// P:211).
//
// One persistent launch runs all the time steps of a rom_step call.  The batch
// columns are independent, so the grid is a set of thread-block clusters, each
// advancing NB = 8 NT columns on its own (no inter-cluster communication).
// Inside a cluster of C CTAs the rows of K~' (E update) and of K~'^T (H update)
// are cut into 8-row tiles; every warp owns ONE tile of ONE of the two matrices
// and keeps it in registers for the whole launch as the A fragments of the fp64
// tensor-core instruction mma.sync.m8n8k4 (KS = QP/4 doubles per thread).  The
// reduced states e~, h~ [QP][NB] live in the shared memory of every CTA of the
// cluster; a warp writes its 8 x NB slice of the new state into all C copies
// (distributed shared memory) and a cluster barrier separates the two halves:
//
//   E half   E-warps:  e~ <- e~ - g_e o (K~' h~) + f[:, b] wave[n][b]
//   barrier
//   H half   H-warps:  h~ <- h~ + g_h o (K~'^T e~);   probe warps: p_e = L_e e~
//   barrier                                   (next E half: probe warps p_h = L_h h~)
//
// Steady state touches HBM only for the waveform samples and the probe
// outputs; K~' is read once per launch.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/fdtd.h"
#include "../../include/fdtd_rom.h"

namespace fdtd {
int set_error(int code, const char* msg);     // fdtd_api.cu (thread-local message of fdtd_last_error)
}

namespace {

#define RCK(call)                                                                                  \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess) {                                                                       \
      char b_[512];                                                                                \
      snprintf(b_, sizeof(b_), "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
      return fdtd::set_error(FDTD_ECUDA, b_);                                                      \
    }                                                                                              \
  } while (0)

int rfail(int code, const std::string& m) { return fdtd::set_error(code, m.c_str()); }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t map_rank(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_v2(uint32_t a, double x, double y) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};\n" ::"r"(a), "d"(x), "d"(y) : "memory");
}
template <bool CLUSTER>
__device__ __forceinline__ void half_barrier() {
  if constexpr (CLUSTER) {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  } else {
    __syncthreads();
  }
}

struct RomParams {
  const double* Ae;      // [QP][QP] padded K~'   (row m, column k): E update A = K~'
  const double* Ah;      // [QP][QP] padded K~'^T
  const double* Ape;     // [8 tpe][QP] padded L_e
  const double* Aph;     // [8 tph][QP] padded L_h
  const double* ge;      // [QP] (0 on padding)
  const double* gh;      // [QP]
  const double* force;   // [QP][batch_p]  g_e o (B~_e amp)
  const double* wave;    // [n_wave][batch_p]
  double* e;             // [QP][batch_p]  state (read at launch, written back at the end)
  double* h;
  double* out;           // probe ring [cap_steps][n_out][batch]
  int64_t n_wave, step0, nsteps, out_step0;
  int batch, batch_p, n_out_e, n_out_h, te, tpe, tph;   // te: 8-row tiles per matrix per CTA
};

// threads per CTA the register file allows: 2 KS registers of A fragments, the
// accumulators, forcing and waveform values of NT column tiles, ~48 of overhead
__host__ __device__ constexpr int rom_maxt(int KS, int NT) {
  const int t = (65536 / (2 * KS + 12 * NT + 42)) / 32 * 32;
  return t > 1024 ? 1024 : t;
}

// KS: contraction length / 4 (QP = 4 KS); NT: 8-column tiles per cluster.
template <int KS, int NT, bool CLUSTER>
__global__ void __launch_bounds__(rom_maxt(KS, NT), 1) rom_persist_kernel(const RomParams P, const int C) {
  constexpr int QP = 4 * KS;
  constexpr int NB = 8 * NT;
  constexpr int NBP = NT == 1 ? 8 : NB + 8;       // row stride (doubles): 8 mod 16 -> conflict-free fragments
  extern __shared__ __align__(16) double sm[];
  double* se = sm;                  // [QP][NBP]
  double* sh = sm + QP * NBP;       // [QP][NBP]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = CLUSTER ? (int)(blockIdx.x % (unsigned)C) : 0;
  const int cl = CLUSTER ? (int)(blockIdx.x / (unsigned)C) : (int)blockIdx.x;
  const int col0 = cl * NB;                        // first batch column of this cluster
  const int gr = lane >> 2, gc = lane & 3;         // fragment coordinates
  // ---- role: E tile | H tile | probe-E tile | probe-H tile
  const int te = P.te;
  int role, tile;                                  // tile: 8-row tile index within the whole matrix
  if (warp < te) { role = 0; tile = rank * te + warp; }
  else if (warp < 2 * te) { role = 1; tile = rank * te + (warp - te); }
  else if (warp < 2 * te + P.tpe) { role = 2; tile = warp - 2 * te; }
  else { role = 3; tile = warp - 2 * te - P.tpe; }
  const bool probe_active = role >= 2 && rank == 0;
  // ---- A fragments: row = tile*8 + gr, columns 4 k + gc
  const double* A = role == 0 ? P.Ae : role == 1 ? P.Ah : role == 2 ? P.Ape : P.Aph;
  double a[KS];
  {
    const double* ar = A + (size_t)(tile * 8 + gr) * QP + gc;
#pragma unroll
    for (int k = 0; k < KS; ++k) a[k] = ar[4 * k];
  }
  const int m = tile * 8 + gr;                     // this thread's row of the C fragment
  const double g = role == 0 ? P.ge[m] : role == 1 ? P.gh[m] : 0.0;
  // forcing of this thread's elements (row m, columns col0 + 8 t + 2 gc + {0, 1})
  double f[NT][2];
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int j = 0; j < 2; ++j) f[t][j] = role == 0 ? P.force[(size_t)m * P.batch_p + col0 + 8 * t + 2 * gc + j] : 0.0;
  // ---- state into shared memory (every CTA of the cluster keeps a full copy)
  for (int i = threadIdx.x; i < QP * NB; i += blockDim.x) {
    const int r = i / NB, c = i % NB;
    se[r * NBP + c] = P.e[(size_t)r * P.batch_p + col0 + c];
    sh[r * NBP + c] = P.h[(size_t)r * P.batch_p + col0 + c];
  }
  half_barrier<CLUSTER>();
  const uint32_t se_a = smem_addr(se), sh_a = smem_addr(sh);
  const int n_out = P.n_out_e + P.n_out_h;

  // out[NT][2] (+)= A_tile . X[:, 8 t ..] with two accumulator sets (even / odd k)
  auto contract = [&](const double* X, double (&acc)[NT][2]) {
    double acc2[NT][2];
#pragma unroll
    for (int t = 0; t < NT; ++t) { acc[t][0] = acc[t][1] = 0.0; acc2[t][0] = acc2[t][1] = 0.0; }
    const double* xb = X + gc * NBP + gr;
#pragma unroll
    for (int k = 0; k < KS; k += 2) {
#pragma unroll
      for (int t = 0; t < NT; ++t) dmma(acc[t][0], acc[t][1], a[k], xb[(4 * k) * NBP + 8 * t]);
      if (k + 1 < KS) {
#pragma unroll
        for (int t = 0; t < NT; ++t) dmma(acc2[t][0], acc2[t][1], a[k + 1], xb[(4 * k + 4) * NBP + 8 * t]);
      }
    }
#pragma unroll
    for (int t = 0; t < NT; ++t) { acc[t][0] += acc2[t][0]; acc[t][1] += acc2[t][1]; }
  };
  auto publish = [&](uint32_t base, int t, double x, double y) {
    const uint32_t off = (uint32_t)((m * NBP + 8 * t + 2 * gc) * sizeof(double));
    if constexpr (CLUSTER) {
      for (int r = 0; r < C; ++r) st_cluster_v2(map_rank(base + off, (uint32_t)r), x, y);
    } else {
      asm volatile("st.shared.v2.f64 [%0], {%1, %2};\n" ::"r"(base + off), "d"(x), "d"(y) : "memory");
    }
  };
  auto emit = [&](int64_t s, int row, const double (&acc)[NT][2]) {
    // probe row `row` of step s, this thread's columns
    double* o = P.out + ((size_t)(P.out_step0 + s) * n_out + row) * P.batch;
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int b = col0 + 8 * t + 2 * gc + j;
        if (b < P.batch) o[b] = acc[t][j];
      }
  };

  for (int64_t s = 0; s < P.nsteps; ++s) {
    const int64_t n = P.step0 + s;
    // ---- E half (probe-H warps: p_h of the previous step beside it)
    if (role == 0 || (role == 3 && probe_active && s > 0)) {
      double w[NT][2];
#pragma unroll
      for (int t = 0; t < NT; ++t)
#pragma unroll
        for (int j = 0; j < 2; ++j)
          w[t][j] = (role == 0 && n < P.n_wave) ? P.wave[(size_t)n * P.batch_p + col0 + 8 * t + 2 * gc + j] : 0.0;
      double acc[NT][2];
      contract(sh, acc);
      if (role == 0) {
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const double2 old = *reinterpret_cast<const double2*>(se + m * NBP + 8 * t + 2 * gc);
          const double x = fma(f[t][0], w[t][0], fma(-g, acc[t][0], old.x));
          const double y = fma(f[t][1], w[t][1], fma(-g, acc[t][1], old.y));
          publish(se_a, t, x, y);
        }
      } else if (m < P.n_out_h) {
        emit(s - 1, P.n_out_e + m, acc);
      }
    }
    half_barrier<CLUSTER>();
    // ---- H half (probe-E warps: p_e of this step beside it)
    if (role == 1 || (role == 2 && probe_active)) {
      double acc[NT][2];
      contract(se, acc);
      if (role == 1) {
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const double2 old = *reinterpret_cast<const double2*>(sh + m * NBP + 8 * t + 2 * gc);
          publish(sh_a, t, fma(g, acc[t][0], old.x), fma(g, acc[t][1], old.y));
        }
      } else if (m < P.n_out_e) {
        emit(s, m, acc);
      }
    }
    half_barrier<CLUSTER>();
  }
  // p_h of the last step, then the state back to global memory (rank 0's copy)
  if (role == 3 && probe_active && P.nsteps > 0) {
    double acc[NT][2];
    contract(sh, acc);
    if (m < P.n_out_h) emit(P.nsteps - 1, P.n_out_e + m, acc);
  }
  if (rank == 0) {
    for (int i = threadIdx.x; i < QP * NB; i += blockDim.x) {
      const int r = i / NB, c = i % NB;
      P.e[(size_t)r * P.batch_p + col0 + c] = se[r * NBP + c];
      P.h[(size_t)r * P.batch_p + col0 + c] = sh[r * NBP + c];
    }
  }
  if constexpr (CLUSTER) half_barrier<true>();    // no CTA exits while a peer may still address its memory
}

// register-only DMMA loop: the measured fp64 tensor-core peak
__global__ void __launch_bounds__(512, 1) dmma_peak_kernel(double* out, int iters) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { acc[i][0] = 0.0; acc[i][1] = 0.0; }
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma(acc[i][0], acc[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int KS, int NT>
cudaError_t launch_variant(bool cluster, int C, int grid, int threads, size_t smem, cudaStream_t st,
                           const RomParams& P) {
  if (!cluster) {
    cudaFuncSetAttribute(rom_persist_kernel<KS, NT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    rom_persist_kernel<KS, NT, false><<<grid, threads, smem, st>>>(P, 1);
    return cudaGetLastError();
  }
  auto fn = rom_persist_kernel<KS, NT, true>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fn, P, C);
}

template <int KS, int NT>
int regs_variant(bool cluster) {
  cudaFuncAttributes fa;
  if (cluster) { if (cudaFuncGetAttributes(&fa, rom_persist_kernel<KS, NT, true>) != cudaSuccess) return -1; }
  else { if (cudaFuncGetAttributes(&fa, rom_persist_kernel<KS, NT, false>) != cudaSuccess) return -1; }
  return fa.numRegs;
}

#define ROM_FOR_KS(KSV, ...)            \
  switch (KSV) {                          \
    case 8:  { constexpr int KS = 8; __VA_ARGS__ } break;  \
    case 16: { constexpr int KS = 16; __VA_ARGS__ } break;  \
    case 20: { constexpr int KS = 20; __VA_ARGS__ } break;  \
    case 24: { constexpr int KS = 24; __VA_ARGS__ } break;  \
    case 32: { constexpr int KS = 32; __VA_ARGS__ } break;  \
    case 40: { constexpr int KS = 40; __VA_ARGS__ } break;  \
    case 48: { constexpr int KS = 48; __VA_ARGS__ } break;  \
    case 64: { constexpr int KS = 64; __VA_ARGS__ } break;  \
    default: break;                       \
  }
#define ROM_FOR_NT(NTV, ...)            \
  switch (NTV) {                          \
    case 1: { constexpr int NT = 1; __VA_ARGS__ } break;  \
    case 2: { constexpr int NT = 2; __VA_ARGS__ } break;  \
    case 4: { constexpr int NT = 4; __VA_ARGS__ } break;  \
    default: break;                       \
  }

}  // namespace

struct rom_t {
  int qe = 0, qh = 0, QP = 0, KS = 0, NT = 1, C = 1, te = 0, tpe = 0, tph = 0, threads = 0, clusters = 0, regs = 0;
  int batch = 0, batch_p = 0, n_out_e = 0, n_out_h = 0;
  int64_t n_wave = 0, step = 0, launches = 0;
  int64_t cap_steps = 0, rec0 = 0, rec = 0;       // probe ring: steps recorded since the last rom_probe
  size_t smem = 0;
  cudaStream_t st = nullptr;
  std::vector<void*> owned;
  double *Ae = nullptr, *Ah = nullptr, *Ape = nullptr, *Aph = nullptr, *ge = nullptr, *gh = nullptr, *force = nullptr,
         *wave = nullptr, *e = nullptr, *h = nullptr, *out = nullptr;
  ~rom_t() {
    for (void* p : owned) cudaFree(p);
  }
  double* up(const std::vector<double>& v) {
    double* d = nullptr;
    if (cudaMalloc(&d, std::max<size_t>(v.size(), 1) * sizeof(double)) != cudaSuccess) return nullptr;
    owned.push_back(d);
    if (!v.empty() && cudaMemcpyAsync(d, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice, st) != cudaSuccess)
      return nullptr;
    cudaStreamSynchronize(st);
    return d;
  }
};

extern "C" {

int rom_create(const rom_model* M, const rom_excitation* X, void* stream, int32_t cols_per_cluster, rom_t** out) {
  if (!M || !X || !out) return rfail(FDTD_EINVAL, "rom_create: null argument");
  *out = nullptr;
  if (M->q_e < 1 || M->q_h < 1 || M->q_e > 256 || M->q_h > 256) return rfail(FDTD_EINVAL, "rom_create: 1 <= q_e, q_h <= 256");
  if (!M->K || !M->g_e || !M->g_h) return rfail(FDTD_EINVAL, "rom_create: K, g_e, g_h are required");
  if (M->n_in < 0 || (M->n_in > 0 && (!M->B_e || !X->amp))) return rfail(FDTD_EINVAL, "rom_create: B_e / amp missing");
  if (M->n_out_e < 0 || M->n_out_h < 0 || M->n_out_e > 64 || M->n_out_h > 64 ||
      (M->n_out_e > 0 && !M->L_e) || (M->n_out_h > 0 && !M->L_h))
    return rfail(FDTD_EINVAL, "rom_create: 0 <= n_out <= 64 with L given");
  if (X->batch < 1) return rfail(FDTD_EINVAL, "rom_create: batch >= 1");
  if (X->n_wave < 0 || (X->n_wave > 0 && !X->wave)) return rfail(FDTD_EINVAL, "rom_create: wave missing");
  if (cols_per_cluster != 0 && cols_per_cluster != 8 && cols_per_cluster != 16 && cols_per_cluster != 32)
    return rfail(FDTD_EINVAL, "rom_create: cols_per_cluster must be 0, 8, 16 or 32");
  int dev = 0;
  cudaDeviceProp prop;
  RCK(cudaGetDevice(&dev));
  RCK(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10) return rfail(FDTD_ENOTSUP, "rom_create: needs an sm_100 GPU");
  std::unique_ptr<rom_t> R(new rom_t);
  R->st = (cudaStream_t)stream;
  R->qe = M->q_e; R->qh = M->q_h; R->batch = X->batch; R->n_out_e = M->n_out_e; R->n_out_h = M->n_out_h;
  R->n_wave = X->n_wave;
  const int q = std::max(M->q_e, M->q_h);
  // columns per cluster: 8 unless asked otherwise -- measured on B200 (order 80):
  // one CTA per 8 columns holds 62 % of the fp64 tensor-core peak once every SM
  // has one (further columns run as further waves of the persistent launch);
  // wider tiles need more registers per warp, hence clusters, and reached 37 %
  int NT = cols_per_cluster ? cols_per_cluster / 8 : 1;
  R->NT = NT;
  const int NB = 8 * NT;
  R->tpe = (M->n_out_e + 7) / 8; R->tph = (M->n_out_h + 7) / 8;
  // cluster size: the smallest C in {1, 2, 4, 8} whose CTA (2 te + probe warps)
  // fits 1024 threads and the register file at the kernel's register count
  bool found = false;
  for (int C : {1, 2, 4, 8}) {
    int QP = (q + 8 * C - 1) / (8 * C) * (8 * C);
    int KS = QP / 4;
    for (int ks : {8, 16, 20, 24, 32, 40, 48, 64}) if (ks >= KS) { KS = ks; break; }
    if (KS > 64) continue;
    QP = 4 * KS;
    if ((QP / 8) % C) continue;
    const int te = QP / 8 / C;
    const int warps = 2 * te + R->tpe + R->tph;
    int regs = -1;
    ROM_FOR_KS(KS, ROM_FOR_NT(NT, regs = regs_variant<KS, NT>(C > 1);))
    if (regs <= 0) continue;
    const int NBP = NT == 1 ? 8 : NB + 8;
    const size_t smem = (size_t)2 * QP * NBP * sizeof(double);
    if (warps * 32 > rom_maxt(KS, NT) || (int64_t)warps * 32 * ((regs + 7) / 8 * 8) > 65536 || smem > 200 * 1024) continue;
    R->C = C; R->QP = QP; R->KS = KS; R->te = te; R->threads = warps * 32; R->regs = regs; R->smem = smem;
    found = true;
    break;
  }
  if (!found) return rfail(FDTD_ENOTSUP, "rom_create: no launch geometry for q = " + std::to_string(q));
  R->clusters = (X->batch + NB - 1) / NB;
  R->batch_p = R->clusters * NB;
  const int QP = R->QP, bp = R->batch_p;
  // ---- padded operands (fp64, zero padding: padded rows / columns stay exactly 0)
  std::vector<double> Ae((size_t)QP * QP, 0.0), Ah((size_t)QP * QP, 0.0), ge(QP, 0.0), gh(QP, 0.0);
  for (int i = 0; i < M->q_e; ++i)
    for (int j = 0; j < M->q_h; ++j) {
      const double v = M->K[(size_t)i * M->q_h + j];
      Ae[(size_t)i * QP + j] = v;
      Ah[(size_t)j * QP + i] = v;
    }
  for (int i = 0; i < M->q_e; ++i) ge[i] = M->g_e[i];
  for (int j = 0; j < M->q_h; ++j) gh[j] = M->g_h[j];
  std::vector<double> Ape((size_t)std::max(1, 8 * R->tpe) * QP, 0.0), Aph((size_t)std::max(1, 8 * R->tph) * QP, 0.0);
  for (int p = 0; p < M->n_out_e; ++p)
    for (int i = 0; i < M->q_e; ++i) Ape[(size_t)p * QP + i] = M->L_e[(size_t)p * M->q_e + i];
  for (int p = 0; p < M->n_out_h; ++p)
    for (int j = 0; j < M->q_h; ++j) Aph[(size_t)p * QP + j] = M->L_h[(size_t)p * M->q_h + j];
  // forcing f = g_e o (B~_e amp): the spatial part of G_E B~ u (Eq. (12)), composed once in fp64
  std::vector<double> force((size_t)QP * bp, 0.0);
  for (int i = 0; i < M->q_e; ++i)
    for (int b = 0; b < X->batch; ++b) {
      double s = 0.0;
      for (int k = 0; k < M->n_in; ++k) s += M->B_e[(size_t)i * M->n_in + k] * X->amp[(size_t)k * X->batch + b];
      force[(size_t)i * bp + b] = M->g_e[i] * s;
    }
  std::vector<double> wave((size_t)std::max<int64_t>(X->n_wave, 1) * bp, 0.0);
  for (int64_t n = 0; n < X->n_wave; ++n)
    for (int b = 0; b < X->batch; ++b) wave[(size_t)n * bp + b] = X->wave[(size_t)n * X->batch + b];
  std::vector<double> zero((size_t)QP * bp, 0.0);
  R->Ae = R->up(Ae); R->Ah = R->up(Ah); R->Ape = R->up(Ape); R->Aph = R->up(Aph); R->ge = R->up(ge); R->gh = R->up(gh);
  R->force = R->up(force); R->wave = R->up(wave); R->e = R->up(zero); R->h = R->up(zero);
  if (!R->Ae || !R->Ah || !R->Ape || !R->Aph || !R->ge || !R->gh || !R->force || !R->wave || !R->e || !R->h)
    return rfail(FDTD_ENOMEM, "rom_create: device allocation failed");
  const int n_out = M->n_out_e + M->n_out_h;
  R->cap_steps = n_out ? std::max<int64_t>(1, ((int64_t)1 << 28) / ((int64_t)n_out * X->batch)) : 0;   // <= 2 GiB ring
  R->cap_steps = std::min<int64_t>(R->cap_steps, 1 << 20);
  if (n_out) {
    void* p = nullptr;
    if (cudaMalloc(&p, (size_t)R->cap_steps * n_out * X->batch * sizeof(double)) != cudaSuccess)
      return rfail(FDTD_ENOMEM, "rom_create: probe ring allocation failed");
    R->owned.push_back(p);
    R->out = (double*)p;
  }
  *out = R.release();
  return FDTD_OK;
}

int rom_step(rom_t* R, int64_t n) {
  if (!R || n < 0) return rfail(FDTD_EINVAL, "rom_step: bad arguments");
  const int n_out = R->n_out_e + R->n_out_h;
  while (n > 0) {
    int64_t chunk = std::min<int64_t>(n, (int64_t)1 << 30);
    if (n_out) {
      if (R->rec >= R->cap_steps)
        return rfail(FDTD_EINVAL, "rom_step: probe ring full (" + std::to_string(R->cap_steps) + " steps): call rom_probe");
      chunk = std::min(chunk, R->cap_steps - R->rec);
    }
    RomParams P;
    P.Ae = R->Ae; P.Ah = R->Ah; P.Ape = R->Ape; P.Aph = R->Aph; P.ge = R->ge; P.gh = R->gh; P.force = R->force;
    P.wave = R->wave; P.e = R->e; P.h = R->h; P.out = R->out;
    P.n_wave = R->n_wave; P.step0 = R->step; P.nsteps = chunk; P.out_step0 = R->rec;
    P.batch = R->batch; P.batch_p = R->batch_p; P.n_out_e = R->n_out_e; P.n_out_h = R->n_out_h;
    P.te = R->te; P.tpe = R->tpe; P.tph = R->tph;
    cudaError_t err = cudaErrorInvalidValue;
    const int KSv = R->KS, NTv = R->NT;
    ROM_FOR_KS(KSv, ROM_FOR_NT(NTv, err = launch_variant<KS, NT>(R->C > 1, R->C, R->clusters * R->C, R->threads, R->smem,
                                                                R->st, P);))
    if (err != cudaSuccess) return rfail(FDTD_ECUDA, std::string("rom_step: launch failed: ") + cudaGetErrorString(err));
    ++R->launches;
    R->step += chunk;
    if (n_out) R->rec += chunk;
    n -= chunk;
  }
  return FDTD_OK;
}

int rom_sync(rom_t* R) {
  if (!R) return rfail(FDTD_EINVAL, "rom_sync: null handle");
  RCK(cudaStreamSynchronize(R->st));
  return FDTD_OK;
}

int rom_probe(rom_t* R, double* out, int64_t cap, int64_t* written) {
  if (!R || !written) return rfail(FDTD_EINVAL, "rom_probe: null argument");
  const int64_t n_out = R->n_out_e + R->n_out_h;
  const int64_t need = R->rec * n_out * R->batch;
  if (cap < need || (need > 0 && !out)) return rfail(FDTD_EINVAL, "rom_probe: buffer too small");
  RCK(cudaStreamSynchronize(R->st));
  if (need) RCK(cudaMemcpy(out, R->out, (size_t)need * sizeof(double), cudaMemcpyDeviceToHost));
  *written = need;
  R->rec = 0;
  return FDTD_OK;
}

static int rom_state(rom_t* R, int which, double* buf, int64_t n, bool set) {
  if (!R || !buf) return rfail(FDTD_EINVAL, "rom state: null argument");
  RCK(cudaStreamSynchronize(R->st));
  if (which == 2) {
    if (n != 1) return rfail(FDTD_EINVAL, "rom state: n must be 1 for the step counter");
    if (set) R->step = (int64_t)buf[0]; else buf[0] = (double)R->step;
    return FDTD_OK;
  }
  if (which != 0 && which != 1) return rfail(FDTD_EINVAL, "rom state: which must be 0, 1 or 2");
  const int q = which == 0 ? R->qe : R->qh;
  if (n != (int64_t)q * R->batch) return rfail(FDTD_EINVAL, "rom state: n must be batch * q");
  double* d = which == 0 ? R->e : R->h;
  std::vector<double> tmp((size_t)R->QP * R->batch_p, 0.0);
  if (!set) {
    RCK(cudaMemcpy(tmp.data(), d, tmp.size() * sizeof(double), cudaMemcpyDeviceToHost));
    for (int b = 0; b < R->batch; ++b)
      for (int i = 0; i < q; ++i) buf[(size_t)b * q + i] = tmp[(size_t)i * R->batch_p + b];
  } else {
    for (int b = 0; b < R->batch; ++b)
      for (int i = 0; i < q; ++i) tmp[(size_t)i * R->batch_p + b] = buf[(size_t)b * q + i];
    RCK(cudaMemcpy(d, tmp.data(), tmp.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  return FDTD_OK;
}

int rom_get_state(rom_t* R, int32_t which, double* out, int64_t n) { return rom_state(R, which, out, n, false); }
int rom_set_state(rom_t* R, int32_t which, const double* in, int64_t n) {
  return rom_state(R, which, const_cast<double*>(in), n, true);
}

int rom_info(const rom_t* R, int64_t* info, int32_t n) {
  if (!R || !info) return rfail(FDTD_EINVAL, "rom_info: null argument");
  const int64_t v[7] = {R->C, 8 * R->NT, R->clusters, R->threads, R->QP, R->regs, R->launches};
  for (int i = 0; i < n && i < 7; ++i) info[i] = v[i];
  return FDTD_OK;
}

double rom_dmma_peak_tflops(void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1.0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* d = nullptr;
  if (cudaMalloc(&d, 8) != cudaSuccess) return -1.0;
  const int iters = 20000, threads = 512;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  dmma_peak_kernel<<<sms, threads, 0, st>>>(d, iters / 10);
  double best = 0.0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0, st);
    dmma_peak_kernel<<<sms, threads, 0, st>>>(d, iters);
    cudaEventRecord(e1, st);
    if (cudaEventSynchronize(e1) != cudaSuccess) { best = -1.0; break; }
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = (double)sms * (threads / 32) * (double)iters * 8 * 512.0;
    best = std::max(best, flops / (ms * 1e-3) / 1e12);
  }
  cudaEventDestroy(e0); cudaEventDestroy(e1);
  cudaFree(d);
  return best;
}

void rom_destroy(rom_t* R) {
  if (!R) return;
  cudaStreamSynchronize(R->st);
  delete R;
}

}  // extern "C"
