// K2 (FP32, FMM_LEAF_3XTF32 / FMM_LEAF_TF32): batched leaf products on the 5th-generation
// tensor cores (tcgen05.mma kind::tf32, accumulators in TMEM, operands staged by TMA).
//
// 3xTF32: every FP32 operand x is split as x = hi + lo with hi = x rounded to
// TF32 (exact in 19 bits) and lo = x - hi (exact in FP32); the product is accumulated in FP32
// TMEM as lo_A.hi_B + hi_A.lo_B + hi_A.hi_B (small terms first).  A TF32-only leaf fails the
// FP32 parity tolerance at C5; 3xTF32 passes with a wide margin.
//
// Per leaf batch:
//   k_split_*     S (m x k) -> S_hi, S_lo (m x kp, K-major);  T (k x n) -> T_hi, T_lo (kp x np,
//                 as stored: the MMA reads B MN-major), kp / np = k / n rounded up to 32 with
//                 zero padding -- into a per-launch arena in the workspace.  Where the leaf
//                 level's S / T come from a two-level K1X2 pass and k, n are multiples of 32,
//                 that pass writes the arena itself (fmm_plan_set_leaf_split) and no split runs;
//   k2p_tf32      persistent (one CTA per SM, static round-robin over (leaf, 128 x 256 tile)
//                 items): warp 0 = TMA producer (3-D tensor maps over the arena: A 128-byte
//                 swizzle, B 128-byte swizzle with 32-byte atoms), warp 1 = MMA issuer (one
//                 thread, tcgen05.mma.cta_group::1.kind::tf32,
//                 M = 128, N = 256, K = 8), warp 2 = TMEM owner, 8 epilogue warps.  The K range is
//                 accumulated in chunks (default 128): the tensor core's FP32 adds truncate, so
//                 each chunk's TMEM accumulator is drained into register totals with
//                 round-to-nearest adds while the next chunk runs in the other TMEM buffer
//                 (round 1 accumulated all of K in TMEM: 22x the FP32 oracle's
//                 error against double-double at C5, now below it).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "fmm_internal.h"

namespace fmm {

namespace {

constexpr int TBM = 128, TBN = 256, TBK = 32, TSTAGES = 2;  // tile, k-tile, smem stages
constexpr int TMEM_COLS = 256;                                 // one 128 x 256 FP32 accumulator

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

// instruction descriptor: D F32, A / B TF32, A K-major, B MN-major (bit 16), N = TBN, M = TBM
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) |
                           ((uint32_t)(TBN >> 3) << 17) | ((uint32_t)(TBM >> 4) << 24);

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

// x = hi + lo exactly: hi = x rounded to TF32 (nearest, ties away), lo = x - hi (exact in FP32)
__device__ __forceinline__ void split2(float x, float& h, float& l) { tf32_split(x, h, l); }

// K-major UMMA descriptor for the A tile: rows of TBK = 32 floats (128 bytes), 128-byte swizzle
// (8-row x 128-byte atoms, SBO = 1024 bytes)
__device__ __forceinline__ uint64_t desc_k(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);  // start address
  d |= (uint64_t)1 << 16;                    // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;          // stride byte offset: next 8 rows
  d |= (uint64_t)1 << 46;                    // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                    // SWIZZLE_128B
  return d;
}

// MN-major UMMA descriptor for the B tile, stored as TBK k-rows of 128 bytes (32 n) per
// 32-column atom, atoms 128 * TBK bytes apart along n: the tf32 MN-major layout
// SWIZZLE_128B_BASE32B (32-byte chunks XOR-ed with the k-row index mod 4, what TMA's
// SWIZZLE_128B_ATOM_32B writes); LBO = the n-atom stride, SBO = 4 k-rows (512 bytes)
__device__ __forceinline__ uint64_t desc_mn(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)((128 * TBK) >> 4) << 16;  // leading byte offset: next 32-column atom
  d |= (uint64_t)(512 >> 4) << 32;         // stride byte offset: next 4 k-rows
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)1 << 61;                  // SWIZZLE_128B_BASE32B
  return d;
}

constexpr int A_BYTES = TBM * TBK * 4, B_BYTES = TBN * TBK * 4;  // 16 KB, 32 KB (hi or lo)
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
constexpr int SMEM_BYTES = TSTAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
static_assert(SMEM_BYTES <= 227 * 1024, "smem");
// 8 epilogue warps: two per TMEM lane quadrant, each owning ECOLS = 128 columns
constexpr int EPI_WARPS = 8, K2P_THREADS = 32 * (4 + EPI_WARPS), ECOLS = 1024 / EPI_WARPS;

// Persistent leaf-product kernel with chunked round-to-nearest accumulation.  Work items are the
// (leaf, 128 x 256 tile) pairs, leaf-major; CTA b runs items b, b + G, b + 2G, ... (G = grid =
// min(items, SMs), one CTA per SM).  Roles: warp 0 lane 0 = TMA producer over the flattened
// (item, k-tile) sequence through a STAGES-deep ring of hi / lo A and B stages; warp 1 lane 0 =
// the MMA issuer; warp 2 = TMEM owner (512 columns: two 128 x 256 FP32 chunk accumulators);
// warps 4 .. 11 = epilogue.  The K range of an item is cut into chunks of chunk_kt k-tiles; the
// tensor core accumulates one chunk into TMEM buffer (chunk# & 1) -- its FP32 adds truncate
// -- and the epilogue drains that buffer into per-thread register totals with
// round-to-nearest adds (tot = c_0, tot = tot + c_1, ...) while the MMAs of the next chunk run in
// the other buffer.  So the truncation error grows only within a chunk, and both the drain and
// an item's final stores overlap the next chunk's / item's MMAs.  Epilogue warp w owns TMEM lanes
// 32 (w % 4) .. +31 (tile rows) and columns ECOLS ((w - 4) / 4) .. +ECOLS-1.
// Item t -> (leaf, tile origin): leaf-major; inside a leaf, tiles run in groups of group_m tile
// rows, column-major within a group, so the ~one wave of co-resident CTAs shares group_m A panels
// and about SMs / group_m B panels (L2 reuse of the hi / lo operand panels).
__device__ __forceinline__ void item_coords(int t, int tiles, int tiles_m, int tiles_n, int group_m,
                                            int& leaf, int& m0, int& n0) {
  leaf = t / tiles;
  const int tt = t % tiles;
  const int per_group = group_m * tiles_n;
  const int g0 = (tt / per_group) * group_m;
  const int gsz = min(tiles_m - g0, group_m);
  const int w = tt % per_group;
  m0 = (g0 + w % gsz) * TBM;
  n0 = (w / gsz) * TBN;
}

__global__ void __launch_bounds__(K2P_THREADS, 1)
    k2p_tf32(const __grid_constant__ CUtensorMap ta_hi, const __grid_constant__ CUtensorMap ta_lo,
             const __grid_constant__ CUtensorMap tb_hi, const __grid_constant__ CUtensorMap tb_lo,
             const LeafNode* __restrict__ leaves, Bases bases, int64_t m, int64_t n, int64_t kp,
             int tiles_m, int tiles_n, int group_m, int total, int passes, int chunk_kt) {
  constexpr int BK = TBK, STAGES = TSTAGES;
  const int tiles = tiles_m * tiles_n;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(smem + STAGES * STAGE_BYTES);
  // bars: [0,S) full, [S,2S) empty, [2S,2S+2) acc_full, [2S+2,2S+4) acc_empty; then TMEM base
  uint32_t* tmem_slot = (uint32_t*)(bars + 2 * STAGES + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KT = (int)(kp / BK);
  const int nch = (KT + chunk_kt - 1) / chunk_kt;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(su32(&bars[s]), 1);
      mbar_init(su32(&bars[STAGES + s]), 1);
    }
    for (int b2 = 0; b2 < 2; ++b2) {
      mbar_init(su32(&bars[2 * STAGES + b2]), 1);                  // acc_full: tcgen05.commit
      mbar_init(su32(&bars[2 * STAGES + 2 + b2]), EPI_WARPS * 32);  // acc_empty: epilogue threads
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

  // B tile, MN-major: eight boxes of 32 n x BK k-rows, 128 * BK bytes apart
  auto load_b = [&](uint8_t* dst, const CUtensorMap* map, int kc, int n0, int leaf, uint32_t full) {
#pragma unroll
    for (int j = 0; j < TBN / 32; ++j) tma_load_3d(su32(dst + j * 128 * BK), map, n0 + 32 * j, kc, leaf, full);
  };
  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer ----
      int it = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        int leaf, m0, n0;
        item_coords(t, tiles, tiles_m, tiles_n, group_m, leaf, m0, n0);
        for (int kt = 0; kt < KT; ++kt, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (uint32_t)(it / STAGES) & 1u;
          mbar_wait(su32(&bars[STAGES + s]), ph ^ 1u);
          uint8_t* st = smem + s * STAGE_BYTES;
          const uint32_t full = su32(&bars[s]);
          const int kc = kt * BK;
          if (passes == 3) {
            mbar_expect_tx(full, STAGE_BYTES);
            tma_load_3d(su32(st), &ta_hi, kc, m0, leaf, full);
            tma_load_3d(su32(st + A_BYTES), &ta_lo, kc, m0, leaf, full);
            load_b(st + 2 * A_BYTES, &tb_hi, kc, n0, leaf, full);
            load_b(st + 2 * A_BYTES + B_BYTES, &tb_lo, kc, n0, leaf, full);
          } else {
            mbar_expect_tx(full, A_BYTES + B_BYTES);
            tma_load_3d(su32(st), &ta_hi, kc, m0, leaf, full);
            load_b(st + 2 * A_BYTES, &tb_hi, kc, n0, leaf, full);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer ----
      int it = 0, g = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        for (int c = 0; c < nch; ++c, ++g) {
          const int buf = g & 1;
          mbar_wait(su32(&bars[2 * STAGES + 2 + buf]), (uint32_t)((g >> 1) & 1) ^ 1u);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const uint32_t acc = tmem + (uint32_t)(buf * TMEM_COLS);
          const int kt0 = c * chunk_kt, kt1 = min(KT, kt0 + chunk_kt);
          for (int kt = kt0; kt < kt1; ++kt, ++it) {
            const int s = it % STAGES;
            mbar_wait(su32(&bars[s]), (uint32_t)(it / STAGES) & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            uint8_t* st = smem + s * STAGE_BYTES;
            const uint64_t a_hi = desc_k(su32(st)), a_lo = desc_k(su32(st + A_BYTES));
            const uint64_t b_hi = desc_mn(su32(st + 2 * A_BYTES));
            const uint64_t b_lo = desc_mn(su32(st + 2 * A_BYTES + B_BYTES));
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
              const uint64_t off = (uint64_t)((kk * 32) >> 4);        // A: 8 tf32 = 32 bytes along K
              const uint64_t offb = (uint64_t)((kk * 8 * 128) >> 4);  // B: 8 k-rows of 128 bytes
              const uint32_t first = (kt == kt0 && kk == 0) ? 0u : 1u;
              if (passes == 3) {  // small terms first
                mma_tf32(acc, a_lo + off, b_hi + offb, first);
                mma_tf32(acc, a_hi + off, b_lo + offb, 1u);
                mma_tf32(acc, a_hi + off, b_hi + offb, 1u);
              } else {
                mma_tf32(acc, a_hi + off, b_hi + offb, first);
              }
            }
            mma_commit(su32(&bars[STAGES + s]));  // stage s free once these MMAs complete
          }
          mma_commit(su32(&bars[2 * STAGES + buf]));  // chunk complete in buffer buf
        }
      }
    }
  } else if (warp >= 4) {  // ---- epilogue: chunk drains into RN register totals, then stores ----
    const int q = warp & 3, h = (warp - 4) >> 2;
    int g = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      int leaf, m0, n0;
      item_coords(t, tiles, tiles_m, tiles_n, group_m, leaf, m0, n0);
      float tot[ECOLS];
#pragma unroll
      for (int e = 0; e < ECOLS; ++e) tot[e] = 0.f;
      for (int c = 0; c < nch; ++c, ++g) {
        const int buf = g & 1;
        mbar_wait(su32(&bars[2 * STAGES + buf]), (uint32_t)((g >> 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t tbase =
            tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * TMEM_COLS + h * ECOLS);
#pragma unroll
        for (int cb = 0; cb < ECOLS / 16; ++cb) {  // x16 loads keep the totals in registers
          uint32_t v[16];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
              "%13,%14,%15}, [%16];\n"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
                "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
              : "r"(tbase + (uint32_t)(cb * 16)));
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
          if (c == 0) {
#pragma unroll
            for (int e = 0; e < 16; ++e) tot[cb * 16 + e] = __uint_as_float(v[e]);
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) tot[cb * 16 + e] = __fadd_rn(tot[cb * 16 + e], __uint_as_float(v[e]));
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(&bars[2 * STAGES + 2 + buf]))
                     : "memory");
      }
      const int64_t row = m0 + q * 32 + lane;
      if (row < m) {
        const LeafNode& lf = leaves[leaf];
        int64_t ldc;
        float* Cp = op_ptr<float>(bases, lf.c, ldc);
        const int64_t cbase = n0 + h * ECOLS;
        float* crow = Cp + row * ldc + cbase;
        if (((((uintptr_t)crow) & 15u) == 0) && (cbase + ECOLS <= n)) {
#pragma unroll
          for (int e = 0; e < ECOLS; e += 4)
            *reinterpret_cast<float4*>(crow + e) = make_float4(tot[e], tot[e + 1], tot[e + 2], tot[e + 3]);
        } else {
#pragma unroll
          for (int e = 0; e < ECOLS; ++e)
            if (cbase + e < n) crow[e] = tot[e];
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "r"(2 * TMEM_COLS));
}

// S (m x k, via the leaf's a operand) -> hi, lo (m x kp, zero columns k .. kp).
// grid: x = kp / 32, y = ceil(m / 32), z = leaf; block 32 x 8.
__global__ void k_split_a(const LeafNode* __restrict__ leaves, Bases bases, int64_t m, int64_t k,
                          int64_t kp, float* __restrict__ a_hi, float* __restrict__ a_lo) {
  const LeafNode& lf = leaves[blockIdx.z];
  const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
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
}

// Vectorised hi / lo split (the same elementwise split2, so bitwise the same arena): 16-byte loads
// / stores, one float4 per thread, rows grid-strided.  Requires leaf operands 16-byte aligned with
// ld % 4 == 0, k % 4 == 0, n % 4 == 0 (checked by the caller).
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

// B side for the MN-major B operand: T (k x n) -> hi, lo (kp x np, rows = k, np = n rounded up
// to 32, pad rows / columns zero): elementwise, no transpose.  grid: x = np / 4 / 256 chunks,
// y = row stride, z = leaf.
__global__ void k_split_bn_vec(const LeafNode* __restrict__ leaves, Bases bases, int64_t n, int64_t k,
                               int64_t kp, int64_t np, float* __restrict__ b_hi, float* __restrict__ b_lo) {
  const LeafNode& lf = leaves[blockIdx.z];
  int64_t ldb;
  const float* B = op_ptr<const float>(bases, lf.b, ldb);
  const size_t base = (size_t)blockIdx.z * (size_t)(kp * np);
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (c >= np) return;
  for (int64_t r = blockIdx.y; r < kp; r += gridDim.y) {
    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r < k && c < n) x = *reinterpret_cast<const float4*>(B + r * ldb + c);
    float4 h, l;
    split2(x.x, h.x, l.x); split2(x.y, h.y, l.y); split2(x.z, h.z, l.z); split2(x.w, h.w, l.w);
    *reinterpret_cast<float4*>(b_hi + base + r * np + c) = h;
    *reinterpret_cast<float4*>(b_lo + base + r * np + c) = l;
  }
}

__global__ void k_split_bn(const LeafNode* __restrict__ leaves, Bases bases, int64_t n, int64_t k,
                           int64_t kp, int64_t np, float* __restrict__ b_hi, float* __restrict__ b_lo) {
  const LeafNode& lf = leaves[blockIdx.z];
  int64_t ldb;
  const float* B = op_ptr<const float>(bases, lf.b, ldb);
  const size_t base = (size_t)blockIdx.z * (size_t)(kp * np);
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= np) return;
  for (int64_t r = blockIdx.y; r < kp; r += gridDim.y) {
    const float x = (r < k && c < n) ? B[r * ldb + c] : 0.f;
    float h, l;
    split2(x, h, l);
    b_hi[base + r * np + c] = h;
    b_lo[base + r * np + c] = l;
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
  const int64_t np = (n + 31) / 32 * 32;
  const unsigned ry = (unsigned)(kp < 8192 ? kp : 8192);
  if (vec) {
    k_split_a_vec<<<dim3((unsigned)((kp / 4 + 255) / 256), (unsigned)(m < 8192 ? m : 8192), (unsigned)count), 256, 0, st>>>(
        dev_leaves, b, m, k, kp, a_hi, a_lo);
    k_split_bn_vec<<<dim3((unsigned)((np / 4 + 255) / 256), ry, (unsigned)count), 256, 0, st>>>(
        dev_leaves, b, n, k, kp, np, b_hi, b_lo);
    return;
  }
  k_split_a<<<dim3((unsigned)(kp / 32), (unsigned)((m + 31) / 32), (unsigned)count), dim3(32, 8), 0, st>>>(
      dev_leaves, b, m, k, kp, a_hi, a_lo);
  k_split_bn<<<dim3((unsigned)((np + 255) / 256), ry, (unsigned)count), 256, 0, st>>>(
      dev_leaves, b, n, k, kp, np, b_hi, b_lo);
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

// K-major A: S hi / lo (m x kp per leaf), boxes of TBK k x box_rows rows, 128-byte swizzle
bool make_map(CUtensorMap* map, float* base, int64_t kp, int64_t rows, int64_t leaves, int box_rows) {
  constexpr int box_k = TBK;
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)kp, (cuuint64_t)rows, (cuuint64_t)leaves};
  cuuint64_t strides[2] = {(cuuint64_t)(kp * 4), (cuuint64_t)(kp * rows * 4)};
  cuuint32_t box[3] = {(cuuint32_t)box_k, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// MN-major B: T hi / lo (kp x np per leaf, rows = k), boxes of 32 n x box_k k-rows, 128-byte
// swizzle with 32-byte atoms (the UMMA SWIZZLE_128B_BASE32B layout)
bool make_map_mn(CUtensorMap* map, float* base, int64_t np, int64_t kp, int64_t leaves, int box_k) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)np, (cuuint64_t)kp, (cuuint64_t)leaves};
  cuuint64_t strides[2] = {(cuuint64_t)(np * 4), (cuuint64_t)(np * kp * 4)};
  cuuint32_t box[3] = {32, (cuuint32_t)box_k, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int num_sms() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

cudaError_t launch_k2p(float* a_hi, float* a_lo, float* b_hi, float* b_lo, const LeafNode* dev_leaves,
                       int count, int64_t m, int64_t n, int64_t kp, const Bases& b, int passes,
                       int chunk_k, cudaStream_t st) {
  CUtensorMap ma_hi, ma_lo, mb_hi, mb_lo;
  const int64_t kpe = kp > 0 ? kp : TBK;
  const int64_t np = (n + 31) / 32 * 32;
  if (!make_map(&ma_hi, a_hi, kpe, m, count, TBM) || !make_map(&ma_lo, a_lo, kpe, m, count, TBM) ||
      !make_map_mn(&mb_hi, b_hi, np, kpe, count, TBK) || !make_map_mn(&mb_lo, b_lo, np, kpe, count, TBK))
    return cudaErrorInvalidValue;
  const int tiles_m = (int)((m + TBM - 1) / TBM), tiles_n = (int)((n + TBN - 1) / TBN);
  const int tiles = tiles_m * tiles_n;
  const int64_t total = (int64_t)tiles * count;
  if (total > INT32_MAX) return cudaErrorInvalidValue;
  const int grid = (int)std::min<int64_t>(total, num_sms());
  const int chunk_kt = std::max(1, chunk_k / TBK);
  static const int group_m = [] {
    const char* e = getenv("FMM_TF32_GROUP_M");  // tile rows per rasterisation group
    const int v = e ? atoi(e) : 16;
    return v >= 1 ? v : 16;
  }();
  cudaError_t e = cudaFuncSetAttribute(k2p_tf32, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  k2p_tf32<<<grid, K2P_THREADS, SMEM_BYTES, st>>>(ma_hi, ma_lo, mb_hi, mb_lo, dev_leaves, b, m, n, kp,
                                                 tiles_m, tiles_n, group_m, (int)total, passes, chunk_kt);
  return cudaGetLastError();
}

}  // namespace

// hi / lo arena: A side m x kp (K-major), B side kp x np (MN-major, np = n rounded up to 32);
// kp = k rounded up to 32
size_t tf32_arena_floats(int64_t count, int64_t m, int64_t n, int64_t k) {
  const int64_t kp = (k + TBK - 1) / TBK * TBK, np = (n + 31) / 32 * 32;
  // k = 0: no operand is read, but the kernel's tensor maps still need a (tiny) valid base
  return std::max<size_t>((size_t)count * (size_t)(2 * m * kp + 2 * np * kp), 1024);
}

// Chunk length (k elements) of the round-to-nearest accumulation: FMM_TF32_CHUNK, default 128
// (the truncating TMEM adds then span at most 128 products per element).
int tf32_chunk_k() {
  static const int ck = [] {
    const char* e = getenv("FMM_TF32_CHUNK");
    const int v = e ? atoi(e) : 128;
    return v >= 16 ? v : 128;
  }();
  return ck;
}

cudaError_t launch_gemm_tf32(const LeafNode* dev_leaves, int count, int64_t m, int64_t n,
                             int64_t k, const Bases& b, int passes, float* arena,
                             cudaStream_t st, const LeafNode* host_leaves, bool presplit) {
  if (count == 0 || m == 0 || n == 0) return cudaSuccess;
  if (!arena) return cudaErrorInvalidValue;
  // presplit: the leaf level's K1X2 wrote the arena (k, n multiples of 32, B MN-major)
  if (presplit && (k % TBK != 0 || n % 32 != 0)) return cudaErrorInvalidValue;
  const int64_t kp = (k + TBK - 1) / TBK * TBK;
  float* a_hi = arena;
  float* a_lo = a_hi + (size_t)count * m * kp;
  float* b_hi = a_lo + (size_t)count * m * kp;
  float* b_lo = b_hi + (size_t)count * ((n + 31) / 32 * 32) * kp;
  if (kp > 0 && !presplit) launch_split(dev_leaves, host_leaves, count, b, m, n, k, kp, a_hi, a_lo, b_hi, b_lo, st);
  // round 2 measured a 4-stage BK = 16 ring (busier tensor pipe, lower clock under the power cap:
  // 296.8 vs 255.9 ms at C5 FP32), 16 epilogue warps (312.7 ms), a K-major B operand transposed by
  // the split (same speed, but no in-pass split) and a CTA-pair form (7 % slower): this single
  // configuration remains (profiles/r02_tf32_persistent.md)
  return launch_k2p(a_hi, a_lo, b_hi, b_lo, dev_leaves, count, m, n, kp, b, passes, tf32_chunk_k(), st);
}

}  // namespace fmm
