// tc_gemm.cuh — tall-skinny fp32 GEMM on the 5th-generation tensor cores
// (tcgen05, kind::tf32) with 3xTF32 error compensation, for the batched
// reduced-block products of the leap-frog path:
//
//   out[r][n] = sum_k A[r][k] X[k][n]     A: rows x Kp fp32 row-major (S_E, config 4:
//                                          65,024 x 1,024), X: K x 16 fp32 (h~, 16 members)
//
// Plain TF32 (10-bit mantissa) is not accurate enough for the fp32 parity bar
// (1e-4 relative after 10^4 steps); with a = a_hi + a_lo, x = x_hi + x_lo
// (a_hi = a with the 13 low mantissa bits cleared: exact in TF32) the product
// a_hi x_hi + a_hi x_lo + a_lo x_hi recovers ~fp32 accuracy (the dropped
// a_lo x_lo term is 2^-22 relative).
//
// CTA = 10 warps, persistent over 128-row tiles, K in chunks of 32 (one
// 128-byte swizzle atom per row):
//   warp 0     TMA producer: A chunk [128 rows][32] fp32, SWIZZLE_128B, and
//              the chunk's x_hi | x_lo (bulk copy) into an NSTG-stage ring
//              (full / empty mbarriers)
//   warp 1     TMEM allocation (two tile buffers x KSETS accumulator sets x 64
//              columns; k-step kk of a chunk accumulates into set kk % KSETS, so
//              consecutive UMMAs do not chain on one accumulator) and
//              MMA issue (one elected thread): per chunk 4 k-steps x 2
//              products of M=128, N=32, K=8 (B = [x_hi ; x_lo] stacked, so
//              a_hi [x_hi|x_lo] and a_lo [x_hi|x_lo]: the three needed terms in
//              two instructions); tcgen05.commit frees the stage
//   warps 2-5  split: A chunk in place -> a_hi, a_lo, then fence.proxy.async
//              and arrive on the stage's split barrier (x_hi, x_lo arrive
//              pre-split with the A chunk: one bulk copy from the [K/32][hi|lo]
//              buffer the h~ update writes, reduce_axpy_f32_kernel)
//   warps 6-9  epilogue: tcgen05.ld of the accumulators (warp w reads TMEM lanes
//              32 (w % 4) ..), out = a_hi x_hi + (a_hi x_lo + a_lo x_hi), fp32
//              stores of the 16 outputs of each row
// Every mbarrier wait is bounded (trap after 2^26 polls) so a protocol error
// fails the launch instead of hanging the GPU.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace fdtd {
namespace tc {

constexpr int BM = 128;          // rows per tile (UMMA M)
constexpr int BN = 16;           // columns (UMMA N, batch members)
constexpr int BK = 32;           // K per chunk: 32 fp32 = one 128-byte swizzle row
constexpr int NSTG = 5;          // ring stages
constexpr int KSETS = 1;         // accumulator sets (independent MMA chains; 4 measured no faster), summed in the epilogue
constexpr int TMEM_COLS = 2 * KSETS * 4 * BN;   // two tile buffers x KSETS x (32 + 32) columns
constexpr int A_BYTES = BM * BK * 4;            // 16 KB
constexpr int B_BYTES = BN * BK * 4;            // 2 KB
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;   // a_hi (in place) | a_lo | x_hi | x_lo
constexpr int NTHREADS = 320;
constexpr int SMEM_BYTES = NSTG * STAGE_BYTES + 1024 /* align */ + 256 /* barriers */;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(count));
}
__device__ __forceinline__ void bar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
// bounded wait: a protocol error traps (launch error) instead of hanging
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t phase) {
  uint32_t done = 0;
  for (uint32_t it = 0;; ++it) {
    asm volatile(
        "{\n.reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(su32(b)), "r"(phase)
        : "memory");
    if (done) return;
    if (it > (1u << 26)) asm volatile("trap;");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          su32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(su32(bar))
      : "memory");
}
// UMMA shared-memory descriptor: K-major, SWIZZLE_128B (8 rows x 128 B atoms,
// 1024 B between 8-row groups), Blackwell descriptor version 1
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);          // start address
  d |= (uint64_t)1u << 16;                           // leading byte offset (unused for SW128 K-major)
  d |= (uint64_t)(1024u >> 4) << 32;                 // stride byte offset
  d |= (uint64_t)1u << 46;                           // version
  d |= (uint64_t)2u << 61;                           // layout: SWIZZLE_128B
  return d;
}
// instruction descriptor: D f32, A/B tf32, both K-major, N = 32 (x_hi and x_lo
// stacked as the 32 rows of one B tile), M = 128
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)((2 * BN) >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(IDESC), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(b)) : "memory");
}

// byte offset of element (row, k) of a [rows][32] fp32 tile in the 128-byte
// swizzled layout TMA writes (16-byte chunk index XOR row % 8)
__device__ __forceinline__ uint32_t sw_off(int row, int k) {
  return (uint32_t)(row * 128 + ((((k >> 2) ^ (row & 7)) & 7) << 4) + ((k & 3) << 2));
}

__device__ __forceinline__ float tf32_hi(float a) { return __uint_as_float(__float_as_uint(a) & 0xFFFFE000u); }

__global__ void __launch_bounds__(NTHREADS, 1)
tc_skinny_gemm_kernel(const __grid_constant__ CUtensorMap amap, int rows, int K, const float* __restrict__ Xs,
                      float* __restrict__ out, const int64_t* __restrict__ d_step, int check_every,
                      unsigned long long* __restrict__ bad_step) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NSTG * STAGE_BYTES);   // [NSTG] TMA landed
  uint64_t* split = full + NSTG;                                           // [NSTG] operands split
  uint64_t* empty = split + NSTG;                                          // [NSTG] MMAs done with the stage
  uint64_t* accf = empty + NSTG;                                           // [2] accumulator ready
  uint64_t* acce = accf + 2;                                               // [2] accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acce + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = (rows + BM - 1) / BM;
  const int nk = (K + BK - 1) / BK;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTG; ++s) { bar_init(&full[s], 1); bar_init(&split[s], 128); bar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { bar_init(&accf[b], 1); bar_init(&acce[b], 128); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)), "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x)
        for (int c = 0; c < nk; ++c) {
          bar_wait(&empty[s], ph ^ 1u);
          bar_expect_tx(&full[s], A_BYTES + 2 * B_BYTES);
          tma_2d(smem + s * STAGE_BYTES, &amap, c * BK, t * BM, &full[s]);
          // x_hi | x_lo of this chunk, pre-split and pre-swizzled (reduce_axpy_f32_kernel)
          bulk_g2s(smem + s * STAGE_BYTES + 2 * A_BYTES, Xs + (int64_t)c * 1024, 2 * B_BYTES, &full[s]);
          if (++s == NSTG) { s = 0; ph ^= 1u; }
        }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    int s = 0;
    uint32_t ph = 0;
    int j = 0;                                          // local tile count (accumulator buffer j & 1)
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++j) {
      const int ab = j & 1;
      bar_wait(&acce[ab], ((j >> 1) & 1) ^ 1u);         // epilogue drained this accumulator
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t d = tmem + (uint32_t)(ab * KSETS * 4 * BN);
      for (int c = 0; c < nk; ++c) {
        bar_wait(&split[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        if (lane == 0) {
          const uint32_t base = su32(smem + s * STAGE_BYTES);
          // stage: a_hi | a_lo | x_hi | x_lo, the two x tiles contiguous = one 32-row B
          const uint32_t ahi = base, alo = base + A_BYTES, xhi = base + 2 * A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint32_t o = (uint32_t)kk * 32u;       // 8 tf32 = 32 bytes along the swizzled row
            const uint64_t dah = sw128_desc(ahi + o), dal = sw128_desc(alo + o);
            const uint64_t dx = sw128_desc(xhi + o);     // [x_hi ; x_lo]: 32 rows of B
            // D0 = a_hi [x_hi | x_lo], D1 = a_lo [x_hi | x_lo] (its x_lo half unused);
            // one accumulator set per k-step of the chunk: KSETS independent chains
            const uint32_t dk = d + (uint32_t)((kk % KSETS) * 4 * BN);
            mma_tf32(dk, dah, dx, (c > 0 || kk >= KSETS) ? 1u : 0u);
            mma_tf32(dk + 2 * BN, dal, dx, (c > 0 || kk >= KSETS) ? 1u : 0u);
          }
          mma_commit(&empty[s]);                         // stage free once these MMAs completed
          if (c == nk - 1) mma_commit(&accf[ab]);        // accumulator complete
        }
        __syncwarp();
        if (++s == NSTG) { s = 0; ph ^= 1u; }
      }
    }
  } else if (warp < 6) {
    // ---------------- split warps (128 threads)
    const int tid = threadIdx.x - 64;
    int s = 0;
    uint32_t ph = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x)
      for (int c = 0; c < nk; ++c) {
        bar_wait(&full[s], ph);
        unsigned char* st = smem + s * STAGE_BYTES;
        // A: 4096 floats as 1024 16-byte chunks, position preserving
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int ch = q * 128 + tid;
          float4 a = *reinterpret_cast<const float4*>(st + ch * 16);
          float4 hi = make_float4(tf32_hi(a.x), tf32_hi(a.y), tf32_hi(a.z), tf32_hi(a.w));
          float4 lo = make_float4(a.x - hi.x, a.y - hi.y, a.z - hi.z, a.w - hi.w);
          *reinterpret_cast<float4*>(st + ch * 16) = hi;
          *reinterpret_cast<float4*>(st + A_BYTES + ch * 16) = lo;
        }
        // generic-proxy smem writes -> visible to the tensor core (async proxy)
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        bar_arrive(&split[s]);
        if (++s == NSTG) { s = 0; ph ^= 1u; }
      }
  } else {
    // ---------------- epilogue warps (128 threads): warp w reads TMEM lanes 32 (w % 4) ..
    const int quarter = warp & 3;
    const bool check = check_every > 0 && (*d_step % check_every) == 0;
    bool bad = false;
    int j = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++j) {
      const int ab = j & 1;
      bar_wait(&accf[ab], (j >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      uint32_t v[16], u[16], z[16];
      float acc[16];
      const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(ab * KSETS * 4 * BN);
#define FDTD_TMEM_LD16(R, A)                                                                                       \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, " \
               "%14, %15}, [%16];\n"                                                                               \
               : "=r"(R[0]), "=r"(R[1]), "=r"(R[2]), "=r"(R[3]), "=r"(R[4]), "=r"(R[5]), "=r"(R[6]), "=r"(R[7]),   \
                 "=r"(R[8]), "=r"(R[9]), "=r"(R[10]), "=r"(R[11]), "=r"(R[12]), "=r"(R[13]), "=r"(R[14]),         \
                 "=r"(R[15])                                                                                       \
               : "r"(A))
#pragma unroll
      for (int ks = 0; ks < KSETS; ++ks) {
        const uint32_t a0 = taddr + (uint32_t)(ks * 4 * BN);
        FDTD_TMEM_LD16(v, a0);                   // a_hi x_hi
        FDTD_TMEM_LD16(u, a0 + BN);              // a_hi x_lo
        FDTD_TMEM_LD16(z, a0 + 2 * BN);          // a_lo x_hi
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float term = __uint_as_float(v[e]) + (__uint_as_float(u[e]) + __uint_as_float(z[e]));
          acc[e] = ks == 0 ? term : acc[e] + term;
        }
      }
#undef FDTD_TMEM_LD16
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      bar_arrive(&acce[ab]);
      const int r = t * BM + quarter * 32 + lane;
      if (r < rows) {
        float4* o = reinterpret_cast<float4*>(out + (int64_t)r * BN);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 w = make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
          o[q] = w;
          if (check) bad |= !(isfinite(w.x) && isfinite(w.y) && isfinite(w.z) && isfinite(w.w) &&
                              fabsf(w.x) <= 1e30f && fabsf(w.y) <= 1e30f && fabsf(w.z) <= 1e30f &&
                              fabsf(w.w) <= 1e30f);
        }
      }
    }
    if (bad) atomicMin(bad_step, (unsigned long long)*d_step);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TMEM_COLS));
}

}  // namespace tc
}  // namespace fdtd
