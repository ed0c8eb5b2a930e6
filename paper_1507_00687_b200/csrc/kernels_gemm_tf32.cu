// K2 (FP32, FMM_LEAF_3XTF32 / FMM_LEAF_TF32): batched leaf products on the 5th-generation
// tensor cores (tcgen05.mma kind::tf32, accumulators in TMEM, operands staged by TMA).
//
// 3xTF32: every FP32 operand x is split as x = hi + lo with hi = x rounded to
// TF32 (exact in 19 bits) and lo = x - hi (exact in FP32); the product is accumulated in FP32
// TMEM as lo_A.hi_B + hi_A.lo_B + hi_A.hi_B (small terms first).  A TF32-only leaf fails the
// FP32 parity tolerance at C5; 3xTF32 passes with a wide margin.
//
// Two kernels per leaf batch:
//   k_split_tf32  S (m x k) -> S_hi, S_lo (m x kp, K-major);  T (k x n) -> T_hi^T, T_lo^T
//                 (n x kp, K-major, transposed through shared memory), kp = k rounded up to 32
//                 with zero padding -- into a per-launch arena in the workspace;
//   k2_tf32       one CTA per 128 x 256 output tile: warp 0 = TMA producer (3-D tensor maps
//                 over the whole arena, 128-byte swizzle), warp 1 = MMA issuer (one thread,
//                 tcgen05.mma.cta_group::1.kind::tf32, M = 128, N = 256, K = 8 per instruction),
//                 warp 2 = TMEM allocator, warps 4-7 = epilogue (tcgen05.ld 32x32b -> registers
//                 -> global).  2-stage smem ring with full / empty mbarriers; tcgen05.commit
//                 releases a stage and finally signals the epilogue.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "fmm_internal.h"

namespace fmm {

namespace {

constexpr int TBM = 128, TBN = 256, TBK = 32, TSTAGES = 2;
constexpr int A_BYTES = TBM * TBK * 4;  // 16 KB
constexpr int B_BYTES = TBN * TBK * 4;  // 32 KB
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
constexpr int SMEM_BYTES = TSTAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr int TMEM_COLS = 256;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}

// UMMA shared-memory descriptor, K-major, 128-byte swizzle (8-row x 128-byte atoms, SBO = 1024)
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);  // start address [0,14)
  d |= (uint64_t)1 << 16;                    // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;          // stride byte offset [32,46)
  d |= (uint64_t)1 << 46;                    // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                    // layout: SWIZZLE_128B
  return d;
}

// instruction descriptor: D F32, A/B TF32, both K-major, N = TBN, M = TBM
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TBN >> 3) << 17) |
                           ((uint32_t)(TBM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(IDESC), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   bar)
               : "memory");
}

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t u = __float_as_uint(x);
  u = (u + 0x1000u) & 0xFFFFE000u;  // round to nearest (ties away) at 10 mantissa bits
  return __uint_as_float(u);
}

// x = hi + lo exactly: hi = x rounded to TF32, lo = x - hi (exact in FP32)
__device__ __forceinline__ void split2(float x, float& h, float& l) {
  h = tf32_hi(x);
  l = x - h;
}

// K-major UMMA descriptor for a BK-float-wide swizzled tile (BK = 32: SW128, BK = 16: SW64).
template <int BK>
__device__ __forceinline__ uint64_t desc_k(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((8 * BK * 4) >> 4) << 32;  // 8 rows x row bytes
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(BK == 32 ? 2 : 4) << 61;  // SWIZZLE_128B / SWIZZLE_64B
  return d;
}

template <int BK, int STAGES>
struct TCfg {
  static constexpr int A_B = TBM * BK * 4, B_B = TBN * BK * 4;
  static constexpr int STAGE = 2 * A_B + 2 * B_B;
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
  static_assert(SMEM <= 227 * 1024, "smem");
};

template <int BK, int STAGES>
__global__ void __launch_bounds__(256, 1)
    k2_tf32(const __grid_constant__ CUtensorMap ta_hi, const __grid_constant__ CUtensorMap ta_lo,
            const __grid_constant__ CUtensorMap tb_hi, const __grid_constant__ CUtensorMap tb_lo,
            const LeafNode* __restrict__ leaves, Bases bases, int64_t m, int64_t n, int64_t kp,
            int tiles_n, int passes) {
  using CF = TCfg<BK, STAGES>;
  constexpr int TSTAGES = STAGES, TBK = BK, A_BYTES = CF::A_B, B_BYTES = CF::B_B,
                STAGE_BYTES = CF::STAGE;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(smem + TSTAGES * STAGE_BYTES);
  // bars[0..S) full, [S..2S) empty, [2S] tmem_full; then the TMEM base address
  uint32_t* tmem_slot = (uint32_t*)(bars + 2 * TSTAGES + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int leaf = blockIdx.y;
  const int tm = blockIdx.x / tiles_n, tn = blockIdx.x % tiles_n;
  const int m0 = tm * TBM, n0 = tn * TBN;
  const int KT = (int)(kp / TBK);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < TSTAGES; ++s) {
      mbar_init(su32(&bars[s]), 1);
      mbar_init(su32(&bars[TSTAGES + s]), 1);
    }
    mbar_init(su32(&bars[2 * TSTAGES]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     su32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer ----
      for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % TSTAGES;
        const uint32_t ph = (uint32_t)(kt / TSTAGES) & 1u;
        mbar_wait(su32(&bars[TSTAGES + s]), ph ^ 1u);
        uint8_t* st = smem + s * STAGE_BYTES;
        const uint32_t full = su32(&bars[s]);
        const int kc = kt * TBK;
        if (passes == 3) {
          mbar_expect_tx(full, STAGE_BYTES);
          tma_load_3d(su32(st), &ta_hi, kc, m0, leaf, full);
          tma_load_3d(su32(st + A_BYTES), &ta_lo, kc, m0, leaf, full);
          tma_load_3d(su32(st + 2 * A_BYTES), &tb_hi, kc, n0, leaf, full);
          tma_load_3d(su32(st + 2 * A_BYTES + B_BYTES), &tb_lo, kc, n0, leaf, full);
        } else {
          mbar_expect_tx(full, A_BYTES + B_BYTES);
          tma_load_3d(su32(st), &ta_hi, kc, m0, leaf, full);
          tma_load_3d(su32(st + 2 * A_BYTES), &tb_hi, kc, n0, leaf, full);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- MMA issuer (single thread) ----
      for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % TSTAGES;
        const uint32_t ph = (uint32_t)(kt / TSTAGES) & 1u;
        mbar_wait(su32(&bars[s]), ph);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        uint8_t* st = smem + s * STAGE_BYTES;
        const uint64_t a_hi = desc_k<BK>(su32(st)), a_lo = desc_k<BK>(su32(st + A_BYTES));
        const uint64_t b_hi = desc_k<BK>(su32(st + 2 * A_BYTES));
        const uint64_t b_lo = desc_k<BK>(su32(st + 2 * A_BYTES + B_BYTES));
#pragma unroll
        for (int kk = 0; kk < TBK / 8; ++kk) {
          const uint64_t off = (uint64_t)((kk * 32) >> 4);  // 8 tf32 = 32 bytes along K
          const uint32_t first = (kt == 0 && kk == 0) ? 0u : 1u;
          if (passes == 3) {
            mma_tf32(tmem, a_lo + off, b_hi + off, first);
            mma_tf32(tmem, a_hi + off, b_lo + off, 1u);
            mma_tf32(tmem, a_hi + off, b_hi + off, 1u);
          } else {
            mma_tf32(tmem, a_hi + off, b_hi + off, first);
          }
        }
        mma_commit(su32(&bars[TSTAGES + s]));  // stage s free once these MMAs complete
      }
      mma_commit(su32(&bars[2 * TSTAGES]));    // accumulator complete
    }
  } else if (warp >= 4) {
    // ---- epilogue: TMEM -> registers -> global ----
    mbar_wait(su32(&bars[2 * TSTAGES]), 0u);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const LeafNode& lf = leaves[leaf];
    int64_t ldc;
    float* Cp = op_ptr<float>(bases, lf.c, ldc);
    const int q = warp & 3;
    const int64_t row = m0 + q * 32 + lane;
#pragma unroll 1
    for (int cb = 0; cb < TBN / 32; ++cb) {
      uint32_t v[32];
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(cb * 32);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
          "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
            "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
            "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
            "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
            "=r"(v[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      if (KT == 0) {
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = 0u;  // empty inner dimension: C = 0
      }
      if (row < m) {
        float* crow = Cp + row * ldc + n0 + cb * 32;
        const int64_t cbase = n0 + cb * 32;
        const bool vec = ((((uintptr_t)crow) & 15u) == 0) && (cbase + 32 <= n);
        if (vec) {
#pragma unroll
          for (int e = 0; e < 32; e += 4)
            *reinterpret_cast<float4*>(crow + e) =
                make_float4(__uint_as_float(v[e]), __uint_as_float(v[e + 1]),
                            __uint_as_float(v[e + 2]), __uint_as_float(v[e + 3]));
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (cbase + e < n) crow[e] = __uint_as_float(v[e]);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "r"(TMEM_COLS));
}

// K2F for the FP32 tensor-core leaves: one CTA per (128 x 256 output tile, parent node) runs the
// parent's nr leaf products in ascending r.  TMEM holds TWO 128 x 256 FP32 accumulators (512
// columns): the single MMA-issuing thread writes product r into buffer r & 1 while warps 4-7
// drain product r-1 from the other buffer and apply the parent's W-combination -- C_k = w*m for
// the first contribution, else C_k = C_k + w*m (FP32, round to nearest, plain load / store by
// the thread owning the row) -- K3's per-element sequence, bitwise, with M_r never written and
// the epilogue overlapped with the next product's MMAs.  Barriers: full / empty per smem stage
// (TMA <-> MMA, as in k2_tf32), acc_full / acc_empty per TMEM buffer (MMA <-> epilogue; the
// epilogue's 128 threads arrive on acc_empty).  Operands: the per-launch hi / lo arena of
// k_split_tf32 with leaf index parent * nr + r.
template <int BK, int STAGES>
__global__ void __launch_bounds__(256, 1)
    k2f_tf32(const __grid_constant__ CUtensorMap ta_hi, const __grid_constant__ CUtensorMap ta_lo,
             const __grid_constant__ CUtensorMap tb_hi, const __grid_constant__ CUtensorMap tb_lo,
             const FusedNode* __restrict__ nodes, const double* __restrict__ coef_all, Bases bases,
             int64_t m, int64_t n, int64_t kp, int tiles_n, int passes, int P, int Q, int R,
             int count, int chunk, int* __restrict__ turn) {
  using CF = TCfg<BK, STAGES>;
  constexpr int TSTAGES = STAGES, TBK = BK, A_BYTES = CF::A_B, B_BYTES = CF::B_B,
                STAGE_BYTES = CF::STAGE;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(smem + TSTAGES * STAGE_BYTES);
  // bars: [0,S) full, [S,2S) empty, [2S,2S+2) acc_full, [2S+2,2S+4) acc_empty; then TMEM base
  uint32_t* tmem_slot = (uint32_t*)(bars + 2 * TSTAGES + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // chain split (chunk < nr; turnstiles and dispatch-order tickets as in k2f_gemm_f64: the work
  // item (group, parent, tile), group-major, comes from an atomicAdd ticket taken at CTA start,
  // so the group a CTA waits for has always started).  chunk = 1 keeps the unfused kernel's
  // order (all CTAs of one product first: the L2 reuse of that leaf's panels) while the
  // epilogue still applies the W-combination in place.
  const int tiles = gridDim.x;
  int parent = blockIdx.y, grp = 0, tile = blockIdx.x;
  if (turn) {
    __shared__ int s_ticket;
    if (threadIdx.x == 0) s_ticket = atomicAdd(turn + (int64_t)count * tiles, 1);
    __syncthreads();
    const int tk = s_ticket, per_grp = count * tiles;
    grp = tk / per_grp;
    parent = (tk % per_grp) / tiles;
    tile = tk % tiles;
  }
  const FusedNode& nd = nodes[parent];
  const int r_begin = grp * chunk;
  const int r_end = min(nd.nr, r_begin + chunk);
  const int nr_all = nd.nr;
  const int tm = tile / tiles_n, tn = tile % tiles_n;
  const int m0 = tm * TBM, n0 = tn * TBN;
  const int KT = (int)(kp / TBK);

  if (warp == 0 && lane == 0) {
    for (int s2 = 0; s2 < TSTAGES; ++s2) {
      mbar_init(su32(&bars[s2]), 1);
      mbar_init(su32(&bars[TSTAGES + s2]), 1);
    }
    for (int b2 = 0; b2 < 2; ++b2) {
      mbar_init(su32(&bars[2 * TSTAGES + b2]), 1);        // acc_full: one tcgen05.commit
      mbar_init(su32(&bars[2 * TSTAGES + 2 + b2]), 128);  // acc_empty: the 128 epilogue threads
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     su32(tmem_slot)),
                 "r"(2 * TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer over all (product, k-tile) ----
      int it = 0;
      for (int ri = r_begin; ri < r_end; ++ri) {
        const int leaf = parent * nr_all + ri;
        for (int kt = 0; kt < KT; ++kt, ++it) {
          const int s2 = it % TSTAGES;
          const uint32_t ph = (uint32_t)(it / TSTAGES) & 1u;
          mbar_wait(su32(&bars[TSTAGES + s2]), ph ^ 1u);
          uint8_t* st = smem + s2 * STAGE_BYTES;
          const uint32_t full = su32(&bars[s2]);
          const int kc = kt * TBK;
          if (passes == 3) {
            mbar_expect_tx(full, STAGE_BYTES);
            tma_load_3d(su32(st), &ta_hi, kc, m0, leaf, full);
            tma_load_3d(su32(st + A_BYTES), &ta_lo, kc, m0, leaf, full);
            tma_load_3d(su32(st + 2 * A_BYTES), &tb_hi, kc, n0, leaf, full);
            tma_load_3d(su32(st + 2 * A_BYTES + B_BYTES), &tb_lo, kc, n0, leaf, full);
          } else {
            mbar_expect_tx(full, A_BYTES + B_BYTES);
            tma_load_3d(su32(st), &ta_hi, kc, m0, leaf, full);
            tma_load_3d(su32(st + 2 * A_BYTES), &tb_hi, kc, n0, leaf, full);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer ----
      int it = 0;
      for (int ri = r_begin; ri < r_end; ++ri) {
        const int j = ri - r_begin;
        const int buf = j & 1;
        if (j >= 2) {  // the epilogue has drained this buffer (product ri - 2)
          mbar_wait(su32(&bars[2 * TSTAGES + 2 + buf]), (uint32_t)((j / 2 - 1) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        }
        const uint32_t acc = tmem + (uint32_t)(buf * TMEM_COLS);
        for (int kt = 0; kt < KT; ++kt, ++it) {
          const int s2 = it % TSTAGES;
          const uint32_t ph = (uint32_t)(it / TSTAGES) & 1u;
          mbar_wait(su32(&bars[s2]), ph);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          uint8_t* st = smem + s2 * STAGE_BYTES;
          const uint64_t a_hi = desc_k<BK>(su32(st)), a_lo = desc_k<BK>(su32(st + A_BYTES));
          const uint64_t b_hi = desc_k<BK>(su32(st + 2 * A_BYTES));
          const uint64_t b_lo = desc_k<BK>(su32(st + 2 * A_BYTES + B_BYTES));
#pragma unroll
          for (int kk = 0; kk < TBK / 8; ++kk) {
            const uint64_t off = (uint64_t)((kk * 32) >> 4);
            const uint32_t first = (kt == 0 && kk == 0) ? 0u : 1u;
            if (passes == 3) {
              mma_tf32(acc, a_lo + off, b_hi + off, first);
              mma_tf32(acc, a_hi + off, b_lo + off, 1u);
              mma_tf32(acc, a_hi + off, b_hi + off, 1u);
            } else {
              mma_tf32(acc, a_hi + off, b_hi + off, first);
            }
          }
          mma_commit(su32(&bars[TSTAGES + s2]));
        }
        mma_commit(su32(&bars[2 * TSTAGES + buf]));  // product ri complete in buffer buf
      }
    }
  } else if (warp >= 4) {  // ---- epilogue: TMEM -> registers -> W-combination ----
    const int q = warp & 3;
    const int64_t row = m0 + q * 32 + lane;
    int64_t ldo;
    float* out = op_ptr<float>(bases, nd.out, ldo);
    int* my_turn = turn ? turn + (int64_t)parent * tiles + tile : nullptr;
    for (int ri = r_begin; ri < r_end; ++ri) {
      const int j = ri - r_begin;
      const int buf = j & 1;
      mbar_wait(su32(&bars[2 * TSTAGES + buf]), (uint32_t)((j / 2) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      if (j == 0 && grp > 0 && my_turn) {  // group grp-1 released this unit
        if (threadIdx.x == 128) {
          unsigned ns = 64;
          while (atomicAdd(my_turn, 0) < grp) {  // grp-1 holds an earlier ticket: it is running
            __nanosleep(ns);
            if (ns < 2048) ns *= 2;
          }
          __threadfence();
        }
        asm volatile("bar.sync 1, 128;\n" ::: "memory");
      }
      const uint32_t wmask = nd.wmask[ri], fmask = nd.first[ri];
      const int r = nd.rlist[ri];
#pragma unroll 1
      for (int cb = 0; cb < TBN / 32; ++cb) {
        uint32_t v[32];
        const uint32_t taddr =
            tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * TMEM_COLS + cb * 32);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
            "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
              "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
              "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
              "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
              "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        if (KT == 0) {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = 0u;
        }
        if (row >= m) continue;
        const int64_t cbase = n0 + cb * 32;
        for (int kk = 0; kk < P * Q; ++kk) {  // kk = ia*Q + jb (row-major C blocks)
          if (!((wmask >> kk) & 1u)) continue;
          const float w = (float)coef_all[nd.coef_off + kk * R + r];
          const bool first = (fmask >> kk) & 1u;
          float* crow = out + ((int64_t)(kk / Q) * m + row) * ldo + (int64_t)(kk % Q) * n + cbase;
          const bool vec = ((((uintptr_t)crow) & 15u) == 0) && (cbase + 32 <= n);
          if (vec) {
#pragma unroll
            for (int e = 0; e < 32; e += 4) {
              float4 c4;
              const float y0 = __fmul_rn(w, __uint_as_float(v[e])), y1 = __fmul_rn(w, __uint_as_float(v[e + 1]));
              const float y2 = __fmul_rn(w, __uint_as_float(v[e + 2])), y3 = __fmul_rn(w, __uint_as_float(v[e + 3]));
              if (first) {
                c4 = make_float4(y0, y1, y2, y3);
              } else {
                c4 = *reinterpret_cast<const float4*>(crow + e);
                c4.x = __fadd_rn(c4.x, y0); c4.y = __fadd_rn(c4.y, y1);
                c4.z = __fadd_rn(c4.z, y2); c4.w = __fadd_rn(c4.w, y3);
              }
              *reinterpret_cast<float4*>(crow + e) = c4;
            }
          } else {
            for (int e = 0; e < 32; ++e) {
              if (cbase + e >= n) break;
              const float y = __fmul_rn(w, __uint_as_float(v[e]));
              crow[e] = first ? y : __fadd_rn(crow[e], y);
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(&bars[2 * TSTAGES + 2 + buf]))
                   : "memory");
    }
    if (my_turn && r_end < nr_all) {  // hand the unit to group grp+1
      __threadfence();
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
      if (threadIdx.x == 128) atomicExch(my_turn, grp + 1);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "r"(2 * TMEM_COLS));
}

// S (m x k, via the leaf's a operand) -> hi, lo (m x kp); T (k x n) -> hi^T, lo^T (n x kp).
// grid: x = kp / 32, y = ceil(rows / 32), z = leaf; block 32 x 8.
__global__ void k_split_tf32(const LeafNode* __restrict__ leaves, Bases bases, int64_t m,
                             int64_t n, int64_t k, int64_t kp, float* __restrict__ a_hi,
                             float* __restrict__ a_lo, float* __restrict__ b_hi,
                             float* __restrict__ b_lo, int side) {
  __shared__ float tile[32][33];
  const LeafNode& lf = leaves[blockIdx.z];
  const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  if (side == 0) {  // A side: no transpose
    int64_t lda;
    const float* A = op_ptr<const float>(bases, lf.a, lda);
    const size_t base = (size_t)blockIdx.z * (size_t)(m * kp);
    for (int rr = ty; rr < 32; rr += 8) {
      const int64_t r = r0 + rr, c = c0 + tx;
      if (r >= m) continue;
      const float x = (c < k) ? A[r * lda + c] : 0.f;
      float h, l;
      split2(x, h, l);
      a_hi[base + r * kp + c] = h;
      a_lo[base + r * kp + c] = l;
    }
  } else {  // B side: T (k x n) -> (n x kp); tile rows = n index, cols = k index
    int64_t ldb;
    const float* B = op_ptr<const float>(bases, lf.b, ldb);
    const size_t base = (size_t)blockIdx.z * (size_t)(n * kp);
    for (int rr = ty; rr < 32; rr += 8) {  // read T[c0 + rr][r0 + tx]
      const int64_t kk = c0 + rr, nn = r0 + tx;
      tile[rr][tx] = (kk < k && nn < n) ? B[kk * ldb + nn] : 0.f;
    }
    __syncthreads();
    for (int rr = ty; rr < 32; rr += 8) {  // write out[r0 + rr][c0 + tx] = T[c0 + tx][r0 + rr]
      const int64_t nn = r0 + rr, kk = c0 + tx;
      if (nn >= n) continue;
      const float x = tile[tx][rr];
      float h, l;
      split2(x, h, l);
      b_hi[base + nn * kp + kk] = h;
      b_lo[base + nn * kp + kk] = l;
    }
  }
}

// Vectorised hi / lo split (same elementwise split2 as k_split_tf32, so bitwise the same arena):
// A side: 16-byte loads / stores, one float4 per thread, rows grid-strided.
// B side: 64 x 64 tiles of T (k x n) staged through shared memory, 16-byte loads along n and
// 16-byte stores along k of the transposed (n x kp) outputs.
// Requires: leaf operands 16-byte aligned with ld % 4 == 0, k % 4 == 0 (checked by the caller).
__global__ void k_split_a_vec(const LeafNode* __restrict__ leaves, Bases bases, int64_t m,
                              int64_t k, int64_t kp, float* __restrict__ a_hi,
                              float* __restrict__ a_lo) {
  const LeafNode& lf = leaves[blockIdx.z];
  int64_t lda;
  const float* A = op_ptr<const float>(bases, lf.a, lda);
  const size_t base = (size_t)blockIdx.z * (size_t)(m * kp);
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (c >= kp) return;
  for (int64_t r = blockIdx.y; r < m; r += gridDim.y) {
    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
    if (c < k) x = *reinterpret_cast<const float4*>(A + r * lda + c);
    float4 h, l;
    split2(x.x, h.x, l.x); split2(x.y, h.y, l.y); split2(x.z, h.z, l.z); split2(x.w, h.w, l.w);
    *reinterpret_cast<float4*>(a_hi + base + r * kp + c) = h;
    *reinterpret_cast<float4*>(a_lo + base + r * kp + c) = l;
  }
}

__global__ void __launch_bounds__(256) k_split_b_vec(const LeafNode* __restrict__ leaves, Bases bases,
                                                     int64_t n, int64_t k, int64_t kp,
                                                     float* __restrict__ b_hi, float* __restrict__ b_lo) {
  __shared__ float tile[64][65];
  const LeafNode& lf = leaves[blockIdx.z];
  int64_t ldb;
  const float* B = op_ptr<const float>(bases, lf.b, ldb);
  const size_t base = (size_t)blockIdx.z * (size_t)(n * kp);
  const int64_t k0 = (int64_t)blockIdx.x * 64, n0 = (int64_t)blockIdx.y * 64;
  const int tid = threadIdx.x;
#pragma unroll
  for (int q = 0; q < 4; ++q) {  // 64 rows (k) x 16 float4 (n)
    const int idx = tid + q * 256;
    const int rr = idx >> 4, cc = (idx & 15) * 4;
    const int64_t kk = k0 + rr, nn = n0 + cc;
    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
    if (kk < k) {
      if (nn + 3 < n) x = *reinterpret_cast<const float4*>(B + kk * ldb + nn);
      else {
        if (nn < n) x.x = B[kk * ldb + nn];
        if (nn + 1 < n) x.y = B[kk * ldb + nn + 1];
        if (nn + 2 < n) x.z = B[kk * ldb + nn + 2];
      }
    }
    tile[rr][cc] = x.x; tile[rr][cc + 1] = x.y; tile[rr][cc + 2] = x.z; tile[rr][cc + 3] = x.w;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 4; ++q) {  // 64 rows (n) x 16 float4 (k) of the transposed tile
    const int idx = tid + q * 256;
    const int rr = idx >> 4, cc = (idx & 15) * 4;
    const int64_t nn = n0 + rr, kk = k0 + cc;
    if (nn >= n || kk >= kp) continue;
    float4 h, l;
    split2(tile[cc][rr], h.x, l.x);
    split2(tile[cc + 1][rr], h.y, l.y);
    split2(tile[cc + 2][rr], h.z, l.z);
    split2(tile[cc + 3][rr], h.w, l.w);
    *reinterpret_cast<float4*>(b_hi + base + nn * kp + kk) = h;
    *reinterpret_cast<float4*>(b_lo + base + nn * kp + kk) = l;
  }
}

// Split launcher: vectorised kernels when every leaf operand allows 16-byte access.
void launch_split(const LeafNode* dev_leaves, const LeafNode* host_leaves, int count, const Bases& b,
                  int64_t m, int64_t n, int64_t k, int64_t kp, float* a_hi, float* a_lo, float* b_hi,
                  float* b_lo, cudaStream_t st) {
  bool vec = host_leaves != nullptr && k % 4 == 0 && n % 4 == 0;
  for (int i = 0; vec && i < count; ++i) {
    int64_t lda, ldb;
    const float* A = op_ptr<const float>(b, host_leaves[i].a, lda);
    const float* B = op_ptr<const float>(b, host_leaves[i].b, ldb);
    vec = !((((uintptr_t)A) & 15u) || (((uintptr_t)B) & 15u) || (lda & 3) || (ldb & 3));
  }
  if (vec) {
    k_split_a_vec<<<dim3((unsigned)((kp / 4 + 255) / 256), (unsigned)(m < 8192 ? m : 8192), (unsigned)count), 256, 0, st>>>(
        dev_leaves, b, m, k, kp, a_hi, a_lo);
    k_split_b_vec<<<dim3((unsigned)((kp + 63) / 64), (unsigned)((n + 63) / 64), (unsigned)count), 256, 0, st>>>(
        dev_leaves, b, n, k, kp, b_hi, b_lo);
    return;
  }
  dim3 blk(32, 8);
  k_split_tf32<<<dim3((unsigned)(kp / 32), (unsigned)((m + 31) / 32), (unsigned)count), blk, 0, st>>>(
      dev_leaves, b, m, n, k, kp, a_hi, a_lo, b_hi, b_lo, 0);
  k_split_tf32<<<dim3((unsigned)(kp / 32), (unsigned)((n + 31) / 32), (unsigned)count), blk, 0, st>>>(
      dev_leaves, b, m, n, k, kp, a_hi, a_lo, b_hi, b_lo, 1);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  });
  return fn;
}

bool make_map(CUtensorMap* map, float* base, int64_t kp, int64_t rows, int64_t leaves,
              int box_rows, int box_k = TBK) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)kp, (cuuint64_t)rows, (cuuint64_t)leaves};
  cuuint64_t strides[2] = {(cuuint64_t)(kp * 4), (cuuint64_t)(kp * rows * 4)};
  cuuint32_t box[3] = {(cuuint32_t)box_k, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE,
                  box_k == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace

size_t tf32_arena_floats(int64_t count, int64_t m, int64_t n, int64_t k) {
  const int64_t kp = (k + TBK - 1) / TBK * TBK;
  return (size_t)count * (size_t)(2 * m * kp + 2 * n * kp);
}

cudaError_t launch_gemm_tf32(const LeafNode* dev_leaves, int count, int64_t m, int64_t n,
                             int64_t k, const Bases& b, int passes, float* arena,
                             cudaStream_t st, const LeafNode* host_leaves) {
  if (count == 0 || m == 0 || n == 0) return cudaSuccess;
  if (!arena) return cudaErrorInvalidValue;
  const int64_t kp = (k + TBK - 1) / TBK * TBK;
  float* a_hi = arena;
  float* a_lo = a_hi + (size_t)count * m * kp;
  float* b_hi = a_lo + (size_t)count * m * kp;
  float* b_lo = b_hi + (size_t)count * n * kp;
  if (kp > 0) launch_split(dev_leaves, host_leaves, count, b, m, n, k, kp, a_hi, a_lo, b_hi, b_lo, st);
  static const int cfg = [] {
    const char* e = getenv("FMM_TF32_CFG");  // 0: BK 32 / 2 stages (default), 1: BK 16 / 4 stages
    return e ? atoi(e) : 0;
  }();
  const int bk = cfg == 0 ? 32 : 16;
  CUtensorMap ma_hi, ma_lo, mb_hi, mb_lo;
  const int64_t kpe = kp > 0 ? kp : TBK;
  if (!make_map(&ma_hi, a_hi, kpe, m, count, TBM, bk) || !make_map(&ma_lo, a_lo, kpe, m, count, TBM, bk) ||
      !make_map(&mb_hi, b_hi, kpe, n, count, TBN, bk) || !make_map(&mb_lo, b_lo, kpe, n, count, TBN, bk))
    return cudaErrorInvalidValue;
  const int tiles_m = (int)((m + TBM - 1) / TBM), tiles_n = (int)((n + TBN - 1) / TBN);
  const dim3 grid((unsigned)(tiles_m * tiles_n), (unsigned)count);
  cudaError_t e;
  if (cfg == 0) {
    using CF = TCfg<32, 2>;
    e = cudaFuncSetAttribute(k2_tf32<32, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM);
    if (e != cudaSuccess) return e;
    k2_tf32<32, 2><<<grid, 256, CF::SMEM, st>>>(ma_hi, ma_lo, mb_hi, mb_lo, dev_leaves, b, m, n, kp,
                                                 tiles_n, passes);
  } else {
    using CF = TCfg<16, 4>;
    e = cudaFuncSetAttribute(k2_tf32<16, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM);
    if (e != cudaSuccess) return e;
    k2_tf32<16, 4><<<grid, 256, CF::SMEM, st>>>(ma_hi, ma_lo, mb_hi, mb_lo, dev_leaves, b, m, n, kp,
                                                 tiles_n, passes);
  }
  return cudaGetLastError();
}

// Fused FP32 tensor-core leaves: split every (parent, product) leaf of the launch into the hi /
// lo arena (leaf index parent * nr + r), then k2f_tf32.
cudaError_t launch_gemm_tf32_fused(const FusedNode* dev_nodes, const LeafNode* dev_split_leaves,
                                   int count, int nr, int64_t m, int64_t n, int64_t k,
                                   const double* dev_coef, int P, int Q, int R, const Bases& b,
                                   int passes, float* arena, cudaStream_t st, int chunk, int* turn) {
  if (count == 0 || m == 0 || n == 0) return cudaSuccess;
  if (!arena) return cudaErrorInvalidValue;
  const int leaves = count * nr;
  const int64_t kp = (k + TBK - 1) / TBK * TBK;
  float* a_hi = arena;
  float* a_lo = a_hi + (size_t)leaves * m * kp;
  float* b_hi = a_lo + (size_t)leaves * m * kp;
  float* b_lo = b_hi + (size_t)leaves * n * kp;
  if (kp > 0) launch_split(dev_split_leaves, nullptr, leaves, b, m, n, k, kp, a_hi, a_lo, b_hi, b_lo, st);
  CUtensorMap ma_hi, ma_lo, mb_hi, mb_lo;
  const int64_t kpe = kp > 0 ? kp : TBK;
  if (!make_map(&ma_hi, a_hi, kpe, m, leaves, TBM, 32) || !make_map(&ma_lo, a_lo, kpe, m, leaves, TBM, 32) ||
      !make_map(&mb_hi, b_hi, kpe, n, leaves, TBN, 32) || !make_map(&mb_lo, b_lo, kpe, n, leaves, TBN, 32))
    return cudaErrorInvalidValue;
  const int tiles_m = (int)((m + TBM - 1) / TBM), tiles_n = (int)((n + TBN - 1) / TBN);
  using CF = TCfg<32, 2>;
  cudaError_t e = cudaFuncSetAttribute(k2f_tf32<32, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM);
  if (e != cudaSuccess) return e;
  if (chunk <= 0 || chunk >= nr || !turn) chunk = nr;
  const int groups = (nr + chunk - 1) / chunk;
  if (groups > 1) {
    e = cudaMemsetAsync(turn, 0, sizeof(int) * ((size_t)count * tiles_m * tiles_n + 1), st);
    if (e != cudaSuccess) return e;
  }
  k2f_tf32<32, 2><<<dim3((unsigned)(tiles_m * tiles_n), (unsigned)(count * groups)), 256, CF::SMEM, st>>>(
      ma_hi, ma_lo, mb_hi, mb_lo, dev_nodes, dev_coef, b, m, n, kp, tiles_n, passes, P, Q, R, count,
      chunk, groups > 1 ? turn : nullptr);
  return cudaGetLastError();
}

}  // namespace fmm
