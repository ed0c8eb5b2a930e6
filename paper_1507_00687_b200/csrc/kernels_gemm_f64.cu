// K2 (FP64): batched leaf products M = S.T on the FP64 tensor path of sm_100a.
//
// sm_100a's tcgen05.mma has no f64 kind; FP64 tensor math is the warp-level DMMA
// (mma.sync .f64 -> SASS DMMA.8x8x4), measured at 36.9 TFLOP/s on this pool's B200s
// (profiles/r01_fp64_peak_microbench.txt; DFMA reaches 33.7).  Design:
//   * CTA tile BM x BN x BK, warps arranged WARPS_M x WARPS_N, warp tile WTM x WTN made of
//     (WTM/16) x (WTN/8) m16n8k4 fragments (4 fp64 accumulators each per thread);
//   * STAGES-deep cp.async (16-byte, L2-only .cg) pipeline global -> shared; shared rows padded
//     by 4 doubles (row pitch = 4 mod 16 doubles) so the 8-byte fragment loads of each
//     half-warp hit 16 distinct bank pairs (ncu: 0 shared-memory bank conflicts);
//   * batched over the leaves of a level by grid.y with per-leaf operand descriptors;
//     grouped rasterisation (8 tile-rows) inside a leaf for L2 reuse;
//   * ragged edges handled by zero-fill (src-size 0) loads and guarded stores; a scalar
//     (8-byte) load path serves operands whose ld / offsets are not 16-byte aligned.
// The leaf's k-order is the tensor core's (reading A4): not the oracle's
// sequential order, covered by the parity tolerance.
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "fmm_internal.h"

namespace fmm {

// Dynamic shared memory above 48 KB, and the largest shared-memory carve-out: without the
// carve-out hint the driver sized the 64 x 64 kernels' L1/shared split at 168 KB, which fits
// only 2 of their 74 KB CTAs per SM instead of 3 (ncu "Block Limit Shared Mem").
template <typename K>
static cudaError_t set_smem(K* kern, int bytes) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                             (int)cudaSharedmemCarveoutMaxShared);
  return e;
}

namespace {

constexpr int GROUP_M = 8;
__device__ int g_group_m_f = 8;  // K2F rasterisation group (FMM_K2F_GROUP_M, experiments)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void cp16(uint32_t dst, const void* src, bool valid) {
  int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(sz));
}
__device__ __forceinline__ void cp8(uint32_t dst, const void* src, bool valid) {
  int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma16n8k4(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

template <int BM_, int BN_, int BK_, int STAGES_, int WARPS_M_, int WARPS_N_, int MINB_ = 1,
          bool PIPE_ = false>
struct Cfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, STAGES = STAGES_, MINB = MINB_;
  // PIPE: fragments of the next k-slice (and of the next stage) are loaded into a second
  // register set while the current slice's DMMAs issue; the stage barrier sits before the last
  // slice of each stage instead of in front of the first.
  static constexpr bool PIPE = PIPE_;
  static constexpr int WARPS_M = WARPS_M_, WARPS_N = WARPS_N_;
  static constexpr int THREADS = WARPS_M * WARPS_N * 32;
  static constexpr int WTM = BM / WARPS_M, WTN = BN / WARPS_N;
  static constexpr int MI = WTM / 16, NI = WTN / 8;
  static constexpr int A_LD = BK + 4, B_LD = BN + 4;
  static constexpr int A_STAGE = BM * A_LD, B_STAGE = BK * B_LD;
  static constexpr int SMEM_BYTES = STAGES * (A_STAGE + B_STAGE) * 8;
  static_assert(A_LD % 16 == 4 && B_LD % 16 == 4, "pitch must be 4 mod 16 doubles");
  static_assert((BM * BK / 2) % THREADS == 0 && (BK * BN / 2) % THREADS == 0, "chunking");
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory");
};

template <typename C, bool VEC>
__device__ __forceinline__ void load_tiles(double* As, double* Bs, const double* A, int64_t lda,
                                           const double* B, int64_t ldb, int64_t m, int64_t n,
                                           int64_t k, int64_t m0, int64_t n0, int64_t k0,
                                           int tid) {
  if constexpr (VEC) {
    constexpr int ACH = C::BK / 2;  // 16-byte chunks per A-tile row
#pragma unroll
    for (int q = 0; q < C::BM * C::BK / 2 / C::THREADS; ++q) {
      int c = tid + q * C::THREADS;
      int row = c / ACH, cc = (c % ACH) * 2;
      int64_t gr = m0 + row, gc = k0 + cc;
      bool ok = gr < m && gc < k;
      cp16(smem_u32(As + row * C::A_LD + cc), ok ? A + gr * lda + gc : A, ok);
    }
    constexpr int BCH = C::BN / 2;
#pragma unroll
    for (int q = 0; q < C::BK * C::BN / 2 / C::THREADS; ++q) {
      int c = tid + q * C::THREADS;
      int row = c / BCH, cc = (c % BCH) * 2;
      int64_t gr = k0 + row, gc = n0 + cc;
      bool ok = gr < k && gc < n;
      cp16(smem_u32(Bs + row * C::B_LD + cc), ok ? B + gr * ldb + gc : B, ok);
    }
  } else {
#pragma unroll
    for (int q = 0; q < C::BM * C::BK / C::THREADS; ++q) {
      int c = tid + q * C::THREADS;
      int row = c / C::BK, cc = c % C::BK;
      int64_t gr = m0 + row, gc = k0 + cc;
      bool ok = gr < m && gc < k;
      cp8(smem_u32(As + row * C::A_LD + cc), ok ? A + gr * lda + gc : A, ok);
    }
#pragma unroll
    for (int q = 0; q < C::BK * C::BN / C::THREADS; ++q) {
      int c = tid + q * C::THREADS;
      int row = c / C::BN, cc = c % C::BN;
      int64_t gr = k0 + row, gc = n0 + cc;
      bool ok = gr < k && gc < n;
      cp8(smem_u32(Bs + row * C::B_LD + cc), ok ? B + gr * ldb + gc : B, ok);
    }
  }
}

template <typename C, bool VEC>
__global__ void __launch_bounds__(C::THREADS, C::MINB)
    k2_gemm_f64(const LeafNode* __restrict__ leaves, Bases bases, int64_t m, int64_t n,
                int64_t k, int tiles_m, int tiles_n) {
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + C::STAGES * C::A_STAGE;

  const LeafNode& lf = leaves[blockIdx.y];
  int64_t lda, ldb, ldc;
  const double* A = op_ptr<const double>(bases, lf.a, lda);
  const double* B = op_ptr<const double>(bases, lf.b, ldb);
  double* Cp = op_ptr<double>(bases, lf.c, ldc);

  // grouped rasterisation
  const int tile = blockIdx.x;
  const int per_group = GROUP_M * tiles_n;
  const int group = tile / per_group;
  const int first_m = group * GROUP_M;
  const int gsz = min(tiles_m - first_m, GROUP_M);
  const int tm = first_m + (tile % per_group) % gsz;
  const int tn = (tile % per_group) / gsz;
  const int64_t m0 = (int64_t)tm * C::BM, n0 = (int64_t)tn * C::BN;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp / C::WARPS_N, wn = warp % C::WARPS_N;
  const int g = lane >> 2, t = lane & 3;

  double acc[C::MI][C::NI][4];
#pragma unroll
  for (int i = 0; i < C::MI; ++i)
#pragma unroll
    for (int j = 0; j < C::NI; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;

  const int KT = (int)((k + C::BK - 1) / C::BK);
#pragma unroll
  for (int s = 0; s < C::STAGES - 1; ++s) {
    if (s < KT)
      load_tiles<C, VEC>(As + s * C::A_STAGE, Bs + s * C::B_STAGE, A, lda, B, ldb, m, n, k, m0, n0,
                         (int64_t)s * C::BK, tid);
    cp_commit();
  }

  if constexpr (!C::PIPE) {
    for (int kt = 0; kt < KT; ++kt) {
      cp_wait<C::STAGES - 2>();
      __syncthreads();
      {
        int nk = kt + C::STAGES - 1;
        if (nk < KT) {
          int slot = nk % C::STAGES;
          load_tiles<C, VEC>(As + slot * C::A_STAGE, Bs + slot * C::B_STAGE, A, lda, B, ldb, m, n, k,
                             m0, n0, (int64_t)nk * C::BK, tid);
        }
        cp_commit();
      }
      const int slot = kt % C::STAGES;
      const double* as = As + slot * C::A_STAGE + (wm * C::WTM + g) * C::A_LD + t;
      const double* bs = Bs + slot * C::B_STAGE + t * C::B_LD + wn * C::WTN + g;
  #pragma unroll
      for (int kk = 0; kk < C::BK; kk += 4) {
        double af[C::MI][2], bf[C::NI];
  #pragma unroll
        for (int i = 0; i < C::MI; ++i) {
          af[i][0] = as[(i * 16) * C::A_LD + kk];
          af[i][1] = as[(i * 16 + 8) * C::A_LD + kk];
        }
  #pragma unroll
        for (int j = 0; j < C::NI; ++j) bf[j] = bs[kk * C::B_LD + j * 8];
  #pragma unroll
        for (int i = 0; i < C::MI; ++i)
  #pragma unroll
          for (int j = 0; j < C::NI; ++j) dmma16n8k4(acc[i][j], af[i][0], af[i][1], bf[j]);
      }
    }
  } else {
    constexpr int KQ = C::BK / 4;
    static_assert(KQ % 2 == 0, "even number of k-slices per stage");
    double af[2][C::MI][2], bf[2][C::NI];
    const int a_off = (wm * C::WTM + g) * C::A_LD + t, b_off = t * C::B_LD + wn * C::WTN + g;
    auto load_frag = [&](int buf, int slot, int kk) {
      const double* as = As + slot * C::A_STAGE + a_off;
      const double* bs = Bs + slot * C::B_STAGE + b_off;
#pragma unroll
      for (int i = 0; i < C::MI; ++i) {
        af[buf][i][0] = as[(i * 16) * C::A_LD + kk];
        af[buf][i][1] = as[(i * 16 + 8) * C::A_LD + kk];
      }
#pragma unroll
      for (int j = 0; j < C::NI; ++j) bf[buf][j] = bs[kk * C::B_LD + j * 8];
    };
    cp_wait<C::STAGES - 2>();
    __syncthreads();
    {
      const int nk = C::STAGES - 1;
      if (nk < KT)
        load_tiles<C, VEC>(As + (nk % C::STAGES) * C::A_STAGE, Bs + (nk % C::STAGES) * C::B_STAGE,
                           A, lda, B, ldb, m, n, k, m0, n0, (int64_t)nk * C::BK, tid);
      cp_commit();
    }
    if (KT > 0) load_frag(0, 0, 0);
    for (int kt = 0; kt < KT; ++kt) {
      const int slot = kt % C::STAGES;
#pragma unroll
      for (int q = 0; q < KQ; ++q) {
        const int cur = q & 1;
        if (q == KQ - 1) {
          cp_wait<C::STAGES - 2>();
          __syncthreads();  // every warp is done reading `slot` (its last slice is in registers)
          const int nk = kt + C::STAGES;
          if (nk < KT)
            load_tiles<C, VEC>(As + (nk % C::STAGES) * C::A_STAGE, Bs + (nk % C::STAGES) * C::B_STAGE,
                               A, lda, B, ldb, m, n, k, m0, n0, (int64_t)nk * C::BK, tid);
          cp_commit();
          if (kt + 1 < KT) load_frag(cur ^ 1, (kt + 1) % C::STAGES, 0);
        } else {
          load_frag(cur ^ 1, slot, (q + 1) * 4);
        }
#pragma unroll
        for (int i = 0; i < C::MI; ++i)
#pragma unroll
          for (int j = 0; j < C::NI; ++j) dmma16n8k4(acc[i][j], af[cur][i][0], af[cur][i][1], bf[cur][j]);
      }
    }
  }
  cp_wait<0>();

  // epilogue: c0,c1 at (row g, cols 2t, 2t+1); c2,c3 at row g+8
#pragma unroll
  for (int i = 0; i < C::MI; ++i) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t row = m0 + wm * C::WTM + i * 16 + g + h * 8;
      if (row >= m) continue;
      double* crow = Cp + row * ldc;
#pragma unroll
      for (int j = 0; j < C::NI; ++j) {
        const int64_t col = n0 + wn * C::WTN + j * 8 + 2 * t;
        const double v0 = acc[i][j][2 * h], v1 = acc[i][j][2 * h + 1];
        if (VEC && col + 1 < n) {
          *reinterpret_cast<double2*>(crow + col) = make_double2(v0, v1);
        } else {
          if (col < n) crow[col] = v0;
          if (col + 1 < n) crow[col + 1] = v1;
        }
      }
    }
  }
}

// K2F: the leaf products r = rlist[0..nr) of one parent node (grid.y) at one output tile
// position (grid.x), in ascending order, with the parent's W-combination in the epilogue
// (FusedNode in fmm_internal.h).  The cp.async pipeline runs over the flattened (product,
// k-tile) sequence, so the next product's first stages are in flight while the epilogue of the
// previous one updates C_k.  Each thread owns the same fragment positions in every product,
// so the read-modify-write chain of an element of C_k stays in one thread, in ascending r:
//   c = w*m (first contribution)  |  c = c + w*m        (both rounded to nearest, no FMA)
// exactly K3's sequence (k3_combine / k_acc), with M_r never written to memory.
__device__ __forceinline__ void red_add(double* p, double v) {
  asm volatile("red.global.add.f64 [%0], %1;\n" ::"l"(p), "d"(v) : "memory");
}

template <typename C, bool VEC, bool RED, bool FLAT>
__global__ void __launch_bounds__(C::THREADS, C::MINB)
    k2f_gemm_f64(const FusedNode* __restrict__ nodes, const double* __restrict__ coef_all,
                 Bases bases, int64_t m, int64_t n, int64_t k, int tiles_m, int tiles_n, int P,
                 int Q, int R, int count, int chunk, int* __restrict__ turn) {
  static_assert(C::PIPE, "the fused kernel uses the PIPE mainloop");
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + C::STAGES * C::A_STAGE;
  // per-CTA product tables: the 64 x 64 configuration sizes them for 2x2 rules with R <= 8
  // (the host selects it only for those) so that 3 CTAs fit an SM's 228 KB of shared memory
  constexpr bool SMALL = C::BM * C::BN <= 64 * 64;
  constexpr int CAPR = SMALL ? 8 : kMaxR, CAPW = SMALL ? 4 * 8 : kMaxBlk * kMaxR;
  __shared__ const double* pa[CAPR];
  __shared__ const double* pb[CAPR];
  __shared__ int64_t la[CAPR], lb[CAPR];
  __shared__ uint32_t wm_s[CAPR], fm_s[CAPR];
  __shared__ int r_s[CAPR];
  __shared__ double wcf[CAPW];

  // product chain split (chunk < nr): grid.y = group * count + parent, groups dispatched in
  // order; group g runs products [g*chunk, (g+1)*chunk) of its unit after group g-1 released
  // the unit's turnstile (so every C_k element still sees ascending r)
  const int parent = blockIdx.y % count, grp = blockIdx.y / count;
  const FusedNode& nd = nodes[parent];
  const int nr_all = nd.nr;
  const int r_begin = grp * chunk;
  const int nr = min(nr_all, r_begin + chunk) - r_begin;  // products of this CTA
  const int tid = threadIdx.x;
  if (tid < nr) {
    const int q = r_begin + tid;
    int64_t l;
    pa[tid] = op_ptr<const double>(bases, nd.a[q], l);
    la[tid] = l;
    pb[tid] = op_ptr<const double>(bases, nd.b[q], l);
    lb[tid] = l;
    wm_s[tid] = nd.wmask[q];
    fm_s[tid] = nd.first[q];
    r_s[tid] = nd.rlist[q];
  }
  for (int t = tid; t < P * Q * R; t += C::THREADS) wcf[t] = coef_all[nd.coef_off + t];
  __syncthreads();

  const int tile = blockIdx.x;
  const int gm = g_group_m_f;
  const int per_group = gm * tiles_n;
  const int group = tile / per_group;
  const int first_m = group * gm;
  const int gsz = min(tiles_m - first_m, gm);
  const int tm = first_m + (tile % per_group) % gsz;
  const int tn = (tile % per_group) / gsz;
  const int64_t m0 = (int64_t)tm * C::BM, n0 = (int64_t)tn * C::BN;

  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp / C::WARPS_N, wn = warp % C::WARPS_N;
  const int g = lane >> 2, t = lane & 3;

  double acc[C::MI][C::NI][4];
#pragma unroll
  for (int i = 0; i < C::MI; ++i)
#pragma unroll
    for (int j = 0; j < C::NI; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;

  const int KT = max(1, (int)((k + C::BK - 1) / C::BK));  // k = 0: one zero-filled tile
  const int total = nr * KT;
  // FLAT (any KT): one load stream over the flattened (product, k-tile) sequence, advanced
  // incrementally.  !FLAT (KT >= STAGES): per-product loops whose operand pointers are loop
  // invariant (the hot loop is the unfused kernel's); only the last STAGES k-tiles of a product
  // load the next product's first tiles.
  int l_kt = 0, l_ri = 0;
  const double* lA = pa[0];
  const double* lB = pb[0];
  int64_t lla = la[0], llb = lb[0];
  auto load_next = [&](int slot) {
    load_tiles<C, VEC>(As + slot * C::A_STAGE, Bs + slot * C::B_STAGE, lA, lla, lB, llb, m, n, k,
                       m0, n0, (int64_t)l_kt * C::BK, tid);
    if (++l_kt == KT) {
      l_kt = 0;
      if (++l_ri < nr) {
        lA = pa[l_ri]; lB = pb[l_ri]; lla = la[l_ri]; llb = lb[l_ri];
      }
    }
  };
  int* my_turn = turn ? turn + (int64_t)parent * gridDim.x + blockIdx.x : nullptr;
  auto turn_wait = [&]() {  // before this CTA's first epilogue: group grp-1 is done with the unit
    if (grp == 0 || !my_turn) return;
    if (tid == 0) {
      unsigned ns = 64;
      long long spins = 0;
      while (atomicAdd(my_turn, 0) < grp) {
        __nanosleep(ns);
        if (ns < 2048) ns *= 2;
        if (++spins > (1ll << 24)) __trap();  // > ~30 s: fail loudly instead of hanging
      }
      __threadfence();
    }
    __syncthreads();
  };
  auto turn_release = [&]() {  // after the last epilogue: hand the unit to group grp+1
    if (!my_turn || r_begin + nr >= nr_all) return;
    __threadfence();
    __syncthreads();
    if (tid == 0) atomicExch(my_turn, grp + 1);
  };
  auto epilogue = [&](int ri) {
    const uint32_t wmask = wm_s[ri], fmask = fm_s[ri];
    const int r = r_s[ri];
    int64_t ldo;
    double* out = op_ptr<double>(bases, nd.out, ldo);
    for (int kk = 0; kk < P * Q; ++kk) {  // kk = ia*Q + jb (row-major C blocks)
      if (!((wmask >> kk) & 1u)) continue;
      const double w = wcf[kk * R + r];
      const bool first = (fmask >> kk) & 1u;
      double* ob = out + (int64_t)(kk / Q) * m * ldo + (int64_t)(kk % Q) * n;
      if (RED && !first) {
        // c = c + w*m as L2 reductions (RED.ADD.F64, round to nearest): no load round trip.
        // Only this thread updates these elements, and same-address operations of one thread
        // are applied in program order, so the per-element sequence is K3's.
#pragma unroll
        for (int i = 0; i < C::MI; ++i)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int64_t row = m0 + wm * C::WTM + i * 16 + g + h * 8;
            if (row >= m) continue;
#pragma unroll
            for (int j = 0; j < C::NI; ++j) {
              const int64_t col = n0 + wn * C::WTN + j * 8 + 2 * t;
              double* cp = ob + row * ldo + col;
              if (col < n) red_add(cp, __dmul_rn(w, acc[i][j][2 * h]));
              if (col + 1 < n) red_add(cp + 1, __dmul_rn(w, acc[i][j][2 * h + 1]));
            }
          }
        continue;
      }
#pragma unroll
      for (int i = 0; i < C::MI; ++i) {
        double2 old[2][C::NI];
        if (!first) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int64_t row = m0 + wm * C::WTM + i * 16 + g + h * 8;
#pragma unroll
            for (int j = 0; j < C::NI; ++j) {
              const int64_t col = n0 + wn * C::WTN + j * 8 + 2 * t;
              old[h][j] = make_double2(0.0, 0.0);
              if (row < m) {
                const double* cp = ob + row * ldo + col;
                if (VEC && col + 1 < n) old[h][j] = *reinterpret_cast<const double2*>(cp);
                else {
                  if (col < n) old[h][j].x = cp[0];
                  if (col + 1 < n) old[h][j].y = cp[1];
                }
              }
            }
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t row = m0 + wm * C::WTM + i * 16 + g + h * 8;
          if (row >= m) continue;
#pragma unroll
          for (int j = 0; j < C::NI; ++j) {
            const int64_t col = n0 + wn * C::WTN + j * 8 + 2 * t;
            double v0 = __dmul_rn(w, acc[i][j][2 * h]), v1 = __dmul_rn(w, acc[i][j][2 * h + 1]);
            if (!first) {
              v0 = __dadd_rn(old[h][j].x, v0);
              v1 = __dadd_rn(old[h][j].y, v1);
            }
            double* cp = ob + row * ldo + col;
            if (VEC && col + 1 < n) {
              *reinterpret_cast<double2*>(cp) = make_double2(v0, v1);
            } else {
              if (col < n) cp[0] = v0;
              if (col + 1 < n) cp[1] = v1;
            }
          }
        }
      }
    }
  };

  constexpr int KQ = C::BK / 4;
  static_assert(KQ % 2 == 0, "even number of k-slices per stage");
  double af[2][C::MI][2], bf[2][C::NI];
  const int a_off = (wm * C::WTM + g) * C::A_LD + t, b_off = t * C::B_LD + wn * C::WTN + g;
  auto load_frag = [&](int buf, int slot, int kk) {
    const double* as = As + slot * C::A_STAGE + a_off;
    const double* bs = Bs + slot * C::B_STAGE + b_off;
#pragma unroll
    for (int i = 0; i < C::MI; ++i) {
      af[buf][i][0] = as[(i * 16) * C::A_LD + kk];
      af[buf][i][1] = as[(i * 16 + 8) * C::A_LD + kk];
    }
#pragma unroll
    for (int j = 0; j < C::NI; ++j) bf[buf][j] = bs[kk * C::B_LD + j * 8];
  };
  auto zero_acc = [&]() {
#pragma unroll
    for (int i = 0; i < C::MI; ++i)
#pragma unroll
      for (int j = 0; j < C::NI; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;
  };
  // one k-tile (global index it, ring slot it % STAGES); `refill(slot)` issues the load of
  // k-tile it + STAGES into the slot just consumed
  auto ktile = [&](int it, auto&& refill) {
    const int slot = it % C::STAGES;
#pragma unroll
    for (int q = 0; q < KQ; ++q) {
      const int cur = q & 1;
      if (q == KQ - 1) {
        cp_wait<C::STAGES - 2>();
        __syncthreads();  // every warp is done reading `slot` (its last slice is in registers)
        refill(slot);
        cp_commit();
        if (it + 1 < total) load_frag(cur ^ 1, (it + 1) % C::STAGES, 0);
      } else {
        load_frag(cur ^ 1, slot, (q + 1) * 4);
      }
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int j = 0; j < C::NI; ++j) dmma16n8k4(acc[i][j], af[cur][i][0], af[cur][i][1], bf[cur][j]);
    }
  };

  if constexpr (FLAT) {
#pragma unroll
    for (int s = 0; s < C::STAGES - 1; ++s) {
      if (s < total) load_next(s);
      cp_commit();
    }
    cp_wait<C::STAGES - 2>();
    __syncthreads();
    if (C::STAGES - 1 < total) load_next((C::STAGES - 1) % C::STAGES);
    cp_commit();
    load_frag(0, 0, 0);
    int kt_in_r = 0, ri = 0;
    for (int it = 0; it < total; ++it) {
      ktile(it, [&](int slot) { if (it + C::STAGES < total) load_next(slot); });
      if (++kt_in_r == KT) {
        if (ri == 0) turn_wait();
        epilogue(ri);
        if (ri == nr - 1) turn_release();
        zero_acc();
        kt_in_r = 0;
        ++ri;
      }
    }
  } else {
    // KT >= STAGES: the prologue only touches product 0
    {
      const double* A = pa[0];
      const double* B = pb[0];
      const int64_t lda = la[0], ldb = lb[0];
#pragma unroll
      for (int s = 0; s < C::STAGES - 1; ++s) {
        load_tiles<C, VEC>(As + s * C::A_STAGE, Bs + s * C::B_STAGE, A, lda, B, ldb, m, n, k, m0,
                           n0, (int64_t)s * C::BK, tid);
        cp_commit();
      }
      cp_wait<C::STAGES - 2>();
      __syncthreads();
      load_tiles<C, VEC>(As + (C::STAGES - 1) * C::A_STAGE, Bs + (C::STAGES - 1) * C::B_STAGE, A,
                         lda, B, ldb, m, n, k, m0, n0, (int64_t)(C::STAGES - 1) * C::BK, tid);
      cp_commit();
    }
    load_frag(0, 0, 0);
    int it = 0;
    for (int ri = 0; ri < nr; ++ri) {
      const double* A = pa[ri];
      const double* B = pb[ri];
      const int64_t lda = la[ri], ldb = lb[ri];
      for (int kt = 0; kt < KT - C::STAGES; ++kt, ++it)
        ktile(it, [&](int slot) {
          load_tiles<C, VEC>(As + slot * C::A_STAGE, Bs + slot * C::B_STAGE, A, lda, B, ldb, m, n,
                             k, m0, n0, (int64_t)(kt + C::STAGES) * C::BK, tid);
        });
      // last STAGES k-tiles: prefetch the next product's first STAGES k-tiles
      const bool more = ri + 1 < nr;
      const double* An = more ? pa[ri + 1] : A;
      const double* Bn = more ? pb[ri + 1] : B;
      const int64_t ldan = more ? la[ri + 1] : lda, ldbn = more ? lb[ri + 1] : ldb;
      for (int j = 0; j < C::STAGES; ++j, ++it)
        ktile(it, [&](int slot) {
          if (more)
            load_tiles<C, VEC>(As + slot * C::A_STAGE, Bs + slot * C::B_STAGE, An, ldan, Bn, ldbn,
                               m, n, k, m0, n0, (int64_t)j * C::BK, tid);
        });
      if (ri == 0) turn_wait();
      epilogue(ri);
      if (ri == nr - 1) turn_release();
      zero_acc();
    }
  }
  cp_wait<0>();
}

// K2O: K2F with operand fusion.  A product's S_i = sa0 X + sa1 Y is not
// materialised by K1: the kernel loads the tiles of both parent blocks X, Y (cp.async into two
// slots of the stage) and, once the stage has landed, combines them in place in shared memory
// -- v = sa0*x (exact negation), v = v + sa1*y (one rounding): K1's sequential sum, bitwise --
// before the stage's fragments are read.  Same for T_i.  A stage holds two A and two B slots,
// so the pipeline has 3 stages (221 KB).  Products whose operand is a single +1 source skip the
// combine; products with wider sums use their materialised S / T as a single source.
template <typename C, bool VEC>
__device__ __forceinline__ void load_a_tile(double* As, const double* A, int64_t lda, int64_t m,
                                            int64_t k, int64_t m0, int64_t k0, int tid) {
  if constexpr (VEC) {
    constexpr int ACH = C::BK / 2;
#pragma unroll
    for (int q = 0; q < C::BM * C::BK / 2 / C::THREADS; ++q) {
      int c = tid + q * C::THREADS;
      int row = c / ACH, cc = (c % ACH) * 2;
      int64_t gr = m0 + row, gc = k0 + cc;
      bool ok = gr < m && gc < k;
      cp16(smem_u32(As + row * C::A_LD + cc), ok ? A + gr * lda + gc : A, ok);
    }
  } else {
#pragma unroll
    for (int q = 0; q < C::BM * C::BK / C::THREADS; ++q) {
      int c = tid + q * C::THREADS;
      int row = c / C::BK, cc = c % C::BK;
      int64_t gr = m0 + row, gc = k0 + cc;
      bool ok = gr < m && gc < k;
      cp8(smem_u32(As + row * C::A_LD + cc), ok ? A + gr * lda + gc : A, ok);
    }
  }
}
template <typename C, bool VEC>
__device__ __forceinline__ void load_b_tile(double* Bs, const double* B, int64_t ldb, int64_t n,
                                            int64_t k, int64_t n0, int64_t k0, int tid) {
  if constexpr (VEC) {
    constexpr int BCH = C::BN / 2;
#pragma unroll
    for (int q = 0; q < C::BK * C::BN / 2 / C::THREADS; ++q) {
      int c = tid + q * C::THREADS;
      int row = c / BCH, cc = (c % BCH) * 2;
      int64_t gr = k0 + row, gc = n0 + cc;
      bool ok = gr < k && gc < n;
      cp16(smem_u32(Bs + row * C::B_LD + cc), ok ? B + gr * ldb + gc : B, ok);
    }
  } else {
#pragma unroll
    for (int q = 0; q < C::BK * C::BN / C::THREADS; ++q) {
      int c = tid + q * C::THREADS;
      int row = c / C::BN, cc = c % C::BN;
      int64_t gr = k0 + row, gc = n0 + cc;
      bool ok = gr < k && gc < n;
      cp8(smem_u32(Bs + row * C::B_LD + cc), ok ? B + gr * ldb + gc : B, ok);
    }
  }
}

template <typename C, bool VEC>
__global__ void __launch_bounds__(C::THREADS, C::MINB)
    k2o_gemm_f64(const FusedNode* __restrict__ nodes, const double* __restrict__ coef_all,
                 Bases bases, int64_t m, int64_t n, int64_t k, int tiles_m, int tiles_n, int P,
                 int Q, int R) {
  static_assert(C::PIPE && C::STAGES == 3, "operand fusion: PIPE mainloop, 3 stages");
  constexpr int ASZ = 2 * C::A_STAGE, BSZ = 2 * C::B_STAGE;  // two source slots per stage
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + C::STAGES * ASZ;
  __shared__ const double* pa[kMaxR];
  __shared__ const double* pb[kMaxR];
  __shared__ const double* pa2[kMaxR];
  __shared__ const double* pb2[kMaxR];
  __shared__ int64_t la[kMaxR], lb[kMaxR], la2[kMaxR], lb2[kMaxR];
  __shared__ uint32_t wm_s[kMaxR], fm_s[kMaxR];
  __shared__ int r_s[kMaxR];
  __shared__ int8_t na_s[kMaxR], nb_s[kMaxR], sa_s[kMaxR][2], sb_s[kMaxR][2];
  __shared__ double wcf[kMaxBlk * kMaxR];

  const FusedNode& nd = nodes[blockIdx.y];
  const int nr = nd.nr;
  const int tid = threadIdx.x;
  if (tid < nr) {
    int64_t l;
    pa[tid] = op_ptr<const double>(bases, nd.a[tid], l);
    la[tid] = l;
    pb[tid] = op_ptr<const double>(bases, nd.b[tid], l);
    lb[tid] = l;
    na_s[tid] = (int8_t)nd.na[tid];
    nb_s[tid] = (int8_t)nd.nb[tid];
    sa_s[tid][0] = nd.sa[tid][0]; sa_s[tid][1] = nd.sa[tid][1];
    sb_s[tid][0] = nd.sb[tid][0]; sb_s[tid][1] = nd.sb[tid][1];
    pa2[tid] = nd.na[tid] == 2 ? op_ptr<const double>(bases, nd.a2[tid], l) : nullptr;
    la2[tid] = nd.na[tid] == 2 ? l : 0;
    pb2[tid] = nd.nb[tid] == 2 ? op_ptr<const double>(bases, nd.b2[tid], l) : nullptr;
    lb2[tid] = nd.nb[tid] == 2 ? l : 0;
    wm_s[tid] = nd.wmask[tid];
    fm_s[tid] = nd.first[tid];
    r_s[tid] = nd.rlist[tid];
  }
  for (int t = tid; t < P * Q * R; t += C::THREADS) wcf[t] = coef_all[nd.coef_off + t];
  __syncthreads();

  const int tile = blockIdx.x;
  const int per_group = GROUP_M * tiles_n;
  const int group = tile / per_group;
  const int first_m = group * GROUP_M;
  const int gsz = min(tiles_m - first_m, GROUP_M);
  const int tm = first_m + (tile % per_group) % gsz;
  const int tn = (tile % per_group) / gsz;
  const int64_t m0 = (int64_t)tm * C::BM, n0 = (int64_t)tn * C::BN;

  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp / C::WARPS_N, wn = warp % C::WARPS_N;
  const int g = lane >> 2, t = lane & 3;

  double acc[C::MI][C::NI][4];
  auto zero_acc = [&]() {
#pragma unroll
    for (int i = 0; i < C::MI; ++i)
#pragma unroll
      for (int j = 0; j < C::NI; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;
  };
  zero_acc();
  const int KT = (int)((k + C::BK - 1) / C::BK);  // >= STAGES (host-checked)
  const int total = nr * KT;

  // all source tiles of product ri at k-tile kt into stage `slot`
  auto load_stage = [&](int slot, int ri, int kt) {
    const int64_t k0 = (int64_t)kt * C::BK;
    load_a_tile<C, VEC>(As + slot * ASZ, pa[ri], la[ri], m, k, m0, k0, tid);
    if (na_s[ri] == 2) load_a_tile<C, VEC>(As + slot * ASZ + C::A_STAGE, pa2[ri], la2[ri], m, k, m0, k0, tid);
    load_b_tile<C, VEC>(Bs + slot * BSZ, pb[ri], lb[ri], n, k, n0, k0, tid);
    if (nb_s[ri] == 2) load_b_tile<C, VEC>(Bs + slot * BSZ + C::B_STAGE, pb2[ri], lb2[ri], n, k, n0, k0, tid);
  };
  // combine the sources of stage `slot` (product ri) in place: K1's sequential sum
  auto combine = [&](int slot, int ri) {
    const int na = na_s[ri], nbq = nb_s[ri];
    const double a0 = sa_s[ri][0], a1 = sa_s[ri][1], b0 = sb_s[ri][0], b1 = sb_s[ri][1];
    if (na == 2 || a0 < 0) {
      double* x = As + slot * ASZ;
      const double* y = x + C::A_STAGE;
#pragma unroll
      for (int q = 0; q < C::BM * C::BK / 2 / C::THREADS; ++q) {
        const int c = tid + q * C::THREADS;
        const int off = (c / (C::BK / 2)) * C::A_LD + (c % (C::BK / 2)) * 2;
        double2 v = *reinterpret_cast<double2*>(x + off);
        v.x = a0 < 0 ? -v.x : v.x;
        v.y = a0 < 0 ? -v.y : v.y;
        if (na == 2) {
          const double2 w = *reinterpret_cast<const double2*>(y + off);
          v.x = __dadd_rn(v.x, a1 < 0 ? -w.x : w.x);
          v.y = __dadd_rn(v.y, a1 < 0 ? -w.y : w.y);
        }
        *reinterpret_cast<double2*>(x + off) = v;
      }
    }
    if (nbq == 2 || b0 < 0) {
      double* x = Bs + slot * BSZ;
      const double* y = x + C::B_STAGE;
#pragma unroll
      for (int q = 0; q < C::BK * C::BN / 2 / C::THREADS; ++q) {
        const int c = tid + q * C::THREADS;
        const int off = (c / (C::BN / 2)) * C::B_LD + (c % (C::BN / 2)) * 2;
        double2 v = *reinterpret_cast<double2*>(x + off);
        v.x = b0 < 0 ? -v.x : v.x;
        v.y = b0 < 0 ? -v.y : v.y;
        if (nbq == 2) {
          const double2 w = *reinterpret_cast<const double2*>(y + off);
          v.x = __dadd_rn(v.x, b1 < 0 ? -w.x : w.x);
          v.y = __dadd_rn(v.y, b1 < 0 ? -w.y : w.y);
        }
        *reinterpret_cast<double2*>(x + off) = v;
      }
    }
  };
  auto needs_combine = [&](int ri) {
    return na_s[ri] == 2 || nb_s[ri] == 2 || sa_s[ri][0] < 0 || sb_s[ri][0] < 0;
  };

  auto epilogue = [&](int ri) {
    const uint32_t wmask = wm_s[ri], fmask = fm_s[ri];
    const int r = r_s[ri];
    int64_t ldo;
    double* out = op_ptr<double>(bases, nd.out, ldo);
    for (int kk = 0; kk < P * Q; ++kk) {
      if (!((wmask >> kk) & 1u)) continue;
      const double w = wcf[kk * R + r];
      const bool first = (fmask >> kk) & 1u;
      double* ob = out + (int64_t)(kk / Q) * m * ldo + (int64_t)(kk % Q) * n;
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t row = m0 + wm * C::WTM + i * 16 + g + h * 8;
          if (row >= m) continue;
#pragma unroll
          for (int j = 0; j < C::NI; ++j) {
            const int64_t col = n0 + wn * C::WTN + j * 8 + 2 * t;
            double* cp = ob + row * ldo + col;
            const double v0 = __dmul_rn(w, acc[i][j][2 * h]), v1 = __dmul_rn(w, acc[i][j][2 * h + 1]);
            if (first) {
              if (VEC && col + 1 < n) {
                *reinterpret_cast<double2*>(cp) = make_double2(v0, v1);
              } else {
                if (col < n) cp[0] = v0;
                if (col + 1 < n) cp[1] = v1;
              }
            } else {
              if (col < n) red_add(cp, v0);
              if (col + 1 < n) red_add(cp + 1, v1);
            }
          }
        }
    }
  };

  constexpr int KQ = C::BK / 4;
  double af[2][C::MI][2], bf[2][C::NI];
  const int a_off = (wm * C::WTM + g) * C::A_LD + t, b_off = t * C::B_LD + wn * C::WTN + g;
  auto load_frag = [&](int buf, int slot, int kk) {
    const double* as = As + slot * ASZ + a_off;
    const double* bs = Bs + slot * BSZ + b_off;
#pragma unroll
    for (int i = 0; i < C::MI; ++i) {
      af[buf][i][0] = as[(i * 16) * C::A_LD + kk];
      af[buf][i][1] = as[(i * 16 + 8) * C::A_LD + kk];
    }
#pragma unroll
    for (int j = 0; j < C::NI; ++j) bf[buf][j] = bs[kk * C::B_LD + j * 8];
  };
  // one k-tile: before the next stage's first fragments are read, its sources are combined
  auto ktile = [&](int it, auto&& refill) {
    const int slot = it % C::STAGES;
#pragma unroll
    for (int q = 0; q < KQ; ++q) {
      const int cur = q & 1;
      if (q == KQ - 1) {
        cp_wait<C::STAGES - 2>();
        __syncthreads();
        refill(slot);
        cp_commit();
        if (it + 1 < total) {
          const int rn = (it + 1) / KT;
          if (needs_combine(rn)) {
            combine((it + 1) % C::STAGES, rn);
            __syncthreads();
          }
          load_frag(cur ^ 1, (it + 1) % C::STAGES, 0);
        }
      } else {
        load_frag(cur ^ 1, slot, (q + 1) * 4);
      }
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int j = 0; j < C::NI; ++j) dmma16n8k4(acc[i][j], af[cur][i][0], af[cur][i][1], bf[cur][j]);
    }
  };

#pragma unroll
  for (int s = 0; s < C::STAGES - 1; ++s) {
    load_stage(s, 0, s);
    cp_commit();
  }
  cp_wait<C::STAGES - 2>();
  __syncthreads();
  load_stage(C::STAGES - 1, 0, C::STAGES - 1);
  cp_commit();
  if (needs_combine(0)) {
    combine(0, 0);
    __syncthreads();
  }
  load_frag(0, 0, 0);
  int it = 0;
  for (int ri = 0; ri < nr; ++ri) {
    for (int kt = 0; kt < KT - C::STAGES; ++kt, ++it)
      ktile(it, [&](int slot) { load_stage(slot, ri, kt + C::STAGES); });
    const bool more = ri + 1 < nr;
    for (int j = 0; j < C::STAGES; ++j, ++it)
      ktile(it, [&](int slot) {
        if (more) load_stage(slot, ri + 1, j);
      });
    epilogue(ri);
    zero_acc();
  }
  cp_wait<0>();
}

// K2P: the fused leaf products (K2F) as a persistent kernel (one CTA per SM) with dynamic
// work distribution.  A unit is (parent, 128x128 output tile) with NR products.  Work is one
// counter (atomicAdd) over [0, U_dp) data-parallel units -- a CTA runs all NR products of the
// unit with K2F's epilogue, and the active units stay a contiguous window, as in K2F's grid
// order (L2 reuse of the S_r / T_r panels) -- followed by [U_dp, U_dp + T_tail) stream-K
// product-tiles of the last U - U_dp units (U mod G plus one wave): each is one product into a
// scratch slot with a ready flag, and the CTA that computes product NR-1 of a unit (taken last)
// applies the unit's NR products from scratch in ascending r with the same epilogue -- every
// element of C_k still sees c = w*m, c = c + w*m in ascending r (bitwise K2F / K3).  The
// finisher only waits for tiles handed out before its own, which run on co-resident CTAs, so
// the kernel cannot deadlock with G <= #SMs; CTAs end within about one product of each other.
template <typename C, bool VEC>
__global__ void __launch_bounds__(C::THREADS, 1)
    k2p_gemm_f64(const FusedNode* __restrict__ nodes, const double* __restrict__ coef_all,
                 Bases bases, int64_t m, int64_t n, int64_t k, int tiles_m, int tiles_n, int P,
                 int Q, int R, int NR, int64_t U, int64_t U_dp, double* __restrict__ scratch,
                 int* __restrict__ flags, unsigned long long* __restrict__ counter) {
  static_assert(C::PIPE, "the fused kernel uses the PIPE mainloop");
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + C::STAGES * C::A_STAGE;
  __shared__ int64_t next_work;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp / C::WARPS_N, wn = warp % C::WARPS_N;
  const int g = lane >> 2, t = lane & 3;
  const int tiles = tiles_m * tiles_n;
  const int64_t T_tail = (U - U_dp) * NR;
  const int64_t W = U_dp + T_tail;  // work indices

  auto grab = [&]() {  // thread 0 only
    const int64_t x = (int64_t)atomicAdd(counter, 1ull);
    next_work = x < W ? x : -1;
  };
  // product j of work item w -> (unit, ri); number of products of w
  auto nprod = [&](int64_t w) { return w < U_dp ? NR : 1; };
  auto prod_of = [&](int64_t w, int j, int64_t& u, int& ri) {
    if (w < U_dp) { u = w; ri = j; }
    else { const int64_t q = w - U_dp; u = U_dp + q / NR; ri = (int)(q % NR); }
  };
  auto tile_coords = [&](int64_t u, int64_t& m0, int64_t& n0, const FusedNode*& nd) {
    nd = nodes + u / tiles;
    const int tile = (int)(u % tiles);
    const int per_group = GROUP_M * tiles_n;
    const int group = tile / per_group;
    const int first_m = group * GROUP_M;
    const int gsz = min(tiles_m - first_m, GROUP_M);
    m0 = (int64_t)(first_m + (tile % per_group) % gsz) * C::BM;
    n0 = (int64_t)((tile % per_group) / gsz) * C::BN;
  };
  // operands with the tile offset folded in: A + m0 lda, B + n0, remaining rows / cols
  struct Opnd {
    const double* A;
    const double* B;
    int64_t lda, ldb, mr, nr;
  };
  auto operands = [&](int64_t u, int ri) {
    Opnd o;
    int64_t m0, n0;
    const FusedNode* nd;
    tile_coords(u, m0, n0, nd);
    const double* a0 = op_ptr<const double>(bases, nd->a[ri], o.lda);
    const double* b0 = op_ptr<const double>(bases, nd->b[ri], o.ldb);
    o.A = a0 + m0 * o.lda;
    o.B = b0 + n0;
    o.mr = m - m0;
    o.nr = n - n0;
    return o;
  };

  double acc[C::MI][C::NI][4];
  auto zero_acc = [&]() {
#pragma unroll
    for (int i = 0; i < C::MI; ++i)
#pragma unroll
      for (int j = 0; j < C::NI; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;
  };

  // W-combination of product ri of node nd at tile (m0, n0) from acc (K2F's RED epilogue)
  auto epilogue = [&](const FusedNode* nd, int ri, int64_t m0, int64_t n0) {
    const uint32_t wmask = nd->wmask[ri], fmask = nd->first[ri];
    const int r = nd->rlist[ri];
    int64_t ldo;
    double* out = op_ptr<double>(bases, nd->out, ldo);
    for (int kk = 0; kk < P * Q; ++kk) {  // kk = ia*Q + jb (row-major C blocks)
      if (!((wmask >> kk) & 1u)) continue;
      const double w = coef_all[nd->coef_off + kk * R + r];
      const bool first = (fmask >> kk) & 1u;
      double* ob = out + (int64_t)(kk / Q) * m * ldo + (int64_t)(kk % Q) * n;
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t row = m0 + wm * C::WTM + i * 16 + g + h * 8;
          if (row >= m) continue;
#pragma unroll
          for (int j = 0; j < C::NI; ++j) {
            const int64_t col = n0 + wn * C::WTN + j * 8 + 2 * t;
            double* cp = ob + row * ldo + col;
            const double v0 = __dmul_rn(w, acc[i][j][2 * h]), v1 = __dmul_rn(w, acc[i][j][2 * h + 1]);
            if (first) {
              if (VEC && col + 1 < n) {
                *reinterpret_cast<double2*>(cp) = make_double2(v0, v1);
              } else {
                if (col < n) cp[0] = v0;
                if (col + 1 < n) cp[1] = v1;
              }
            } else {
              if (col < n) red_add(cp, v0);
              if (col + 1 < n) red_add(cp + 1, v1);
            }
          }
        }
    }
  };
  constexpr int NACC = C::MI * C::NI * 4;
  auto store_scratch = [&](int64_t slot) {  // layout [slot][acc index][thread]: coalesced
    double* sp = scratch + slot * NACC * C::THREADS + tid;
#pragma unroll
    for (int i = 0; i < C::MI; ++i)
#pragma unroll
      for (int j = 0; j < C::NI; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) sp[((i * C::NI + j) * 4 + e) * C::THREADS] = acc[i][j][e];
    __threadfence();
    __syncthreads();
    if (tid == 0) atomicExch(&flags[slot], 1);
  };
  auto load_scratch = [&](int64_t slot) {
    if (tid == 0) {
      unsigned ns = 32;
      long long spins = 0;
      while (atomicAdd(&flags[slot], 0) == 0) {
        __nanosleep(ns);
        if (ns < 1024) ns *= 2;
        if (++spins > (1ll << 25)) __trap();  // > ~30 s: fail loudly instead of hanging
      }
      __threadfence();
    }
    __syncthreads();
    const double* sp = scratch + slot * NACC * C::THREADS + tid;
#pragma unroll
    for (int i = 0; i < C::MI; ++i)
#pragma unroll
      for (int j = 0; j < C::NI; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[i][j][e] = __ldcg(sp + ((i * C::NI + j) * 4 + e) * C::THREADS);
  };

  const int KT = (int)((k + C::BK - 1) / C::BK);  // >= STAGES (host-checked)
  constexpr int KQ = C::BK / 4;
  static_assert(KQ % 2 == 0, "even number of k-slices per stage");
  double af[2][C::MI][2], bf[2][C::NI];
  const int a_off = (wm * C::WTM + g) * C::A_LD + t, b_off = t * C::B_LD + wn * C::WTN + g;
  auto load_frag = [&](int buf, int slot, int kk) {
    const double* as = As + slot * C::A_STAGE + a_off;
    const double* bs = Bs + slot * C::B_STAGE + b_off;
#pragma unroll
    for (int i = 0; i < C::MI; ++i) {
      af[buf][i][0] = as[(i * 16) * C::A_LD + kk];
      af[buf][i][1] = as[(i * 16 + 8) * C::A_LD + kk];
    }
#pragma unroll
    for (int j = 0; j < C::NI; ++j) bf[buf][j] = bs[kk * C::B_LD + j * 8];
  };
  // one k-tile; `refill(slot)` loads k-tile it + STAGES; `last` = no k-tile follows
  auto ktile = [&](int it, bool last, auto&& refill) {
    const int slot = it % C::STAGES;
#pragma unroll
    for (int q = 0; q < KQ; ++q) {
      const int cur = q & 1;
      if (q == KQ - 1) {
        cp_wait<C::STAGES - 2>();
        __syncthreads();
        refill(slot);
        cp_commit();
        if (!last) load_frag(cur ^ 1, (it + 1) % C::STAGES, 0);
      } else {
        load_frag(cur ^ 1, slot, (q + 1) * 4);
      }
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int j = 0; j < C::NI; ++j) dmma16n8k4(acc[i][j], af[cur][i][0], af[cur][i][1], bf[cur][j]);
    }
  };

  // ---- first work item ------------------------------------------------------------------
  if (tid == 0) grab();
  __syncthreads();
  int64_t w = next_work;
  if (w < 0) return;
  int j = 0;  // product index within w
  {
    int64_t u;
    int ri;
    prod_of(w, 0, u, ri);
    const Opnd o = operands(u, ri);
#pragma unroll
    for (int s = 0; s < C::STAGES - 1; ++s) {
      load_tiles<C, VEC>(As + s * C::A_STAGE, Bs + s * C::B_STAGE, o.A, o.lda, o.B, o.ldb, o.mr, o.nr,
                         k, 0, 0, (int64_t)s * C::BK, tid);
      cp_commit();
    }
    cp_wait<C::STAGES - 2>();
    __syncthreads();
    load_tiles<C, VEC>(As + (C::STAGES - 1) * C::A_STAGE, Bs + (C::STAGES - 1) * C::B_STAGE, o.A,
                       o.lda, o.B, o.ldb, o.mr, o.nr, k, 0, 0, (int64_t)(C::STAGES - 1) * C::BK, tid);
    cp_commit();
  }
  zero_acc();
  load_frag(0, 0, 0);
  int it = 0;
  while (true) {
    int64_t u;
    int ri;
    prod_of(w, j, u, ri);
    const bool last_of_item = j + 1 == nprod(w);
    if (last_of_item) {  // take the next work item now: its first tiles load during this product
      if (tid == 0) grab();
      __syncthreads();
    }
    const int64_t w_next = last_of_item ? next_work : w;
    const int j_next = last_of_item ? 0 : j + 1;
    const bool more = w_next >= 0;
    {
      const Opnd o = operands(u, ri);
      for (int kt = 0; kt < KT - C::STAGES; ++kt, ++it)
        ktile(it, false, [&](int slot) {
          load_tiles<C, VEC>(As + slot * C::A_STAGE, Bs + slot * C::B_STAGE, o.A, o.lda, o.B,
                             o.ldb, o.mr, o.nr, k, 0, 0, (int64_t)(kt + C::STAGES) * C::BK, tid);
        });
    }
    {
      int64_t un = u;
      int rn = ri;
      if (more) prod_of(w_next, j_next, un, rn);
      const Opnd on = operands(un, rn);
      for (int jj = 0; jj < C::STAGES; ++jj, ++it)
        ktile(it, !more && jj == C::STAGES - 1, [&](int slot) {
          if (more)
            load_tiles<C, VEC>(As + slot * C::A_STAGE, Bs + slot * C::B_STAGE, on.A, on.lda, on.B,
                               on.ldb, on.mr, on.nr, k, 0, 0, (int64_t)jj * C::BK, tid);
        });
    }
    if (w < U_dp) {
      const FusedNode* nd;
      int64_t m0, n0;
      tile_coords(u, m0, n0, nd);
      epilogue(nd, ri, m0, n0);
    } else {
      const int64_t q = w - U_dp;
      store_scratch(q);
      if (ri == NR - 1) {  // finisher: the unit's products in ascending r
        const FusedNode* nd;
        int64_t m0, n0;
        tile_coords(u, m0, n0, nd);
        for (int r2 = 0; r2 < NR; ++r2) {
          load_scratch(q - (NR - 1) + r2);
          epilogue(nd, r2, m0, n0);
        }
      }
    }
    zero_acc();
    if (!more) break;
    w = w_next;
    j = j_next;
  }
  cp_wait<0>();
}

void fused_group_m_init() {
  static bool once = false;
  if (once) return;
  once = true;
  if (const char* e = getenv("FMM_K2F_GROUP_M")) {
    const int v = atoi(e);
    if (v >= 1) cudaMemcpyToSymbol(g_group_m_f, &v, sizeof(int));
  }
}

template <typename C, bool VEC, bool RED>
cudaError_t launch_fused_kernel(const FusedNode* dev_nodes, int count, int64_t m, int64_t n,
                                int64_t k, const double* coef, int P, int Q, int R,
                                const Bases& b, cudaStream_t st, int nr, int chunk, int* turn) {
  const int tiles_m = (int)((m + C::BM - 1) / C::BM), tiles_n = (int)((n + C::BN - 1) / C::BN);
  fused_group_m_init();
  const int KT = (int)std::max<int64_t>(1, (k + C::BK - 1) / C::BK);
  if (chunk <= 0 || chunk >= nr || KT < C::STAGES || !turn) chunk = nr;  // no split
  const int groups = (nr + chunk - 1) / chunk;
  if (groups > 1) {
    cudaError_t e = cudaMemsetAsync(turn, 0, sizeof(int) * (size_t)count * tiles_m * tiles_n, st);
    if (e != cudaSuccess) return e;
  }
  dim3 grid((unsigned)(tiles_m * tiles_n), (unsigned)(count * groups));
  auto go = [&](auto kern) {
    cudaError_t e = set_smem(kern, C::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    kern<<<grid, C::THREADS, C::SMEM_BYTES, st>>>(dev_nodes, coef, b, m, n, k, tiles_m, tiles_n, P,
                                                  Q, R, count, chunk, groups > 1 ? turn : nullptr);
    return cudaGetLastError();
  };
  if (KT >= C::STAGES) return go(k2f_gemm_f64<C, VEC, RED, false>);
  return go(k2f_gemm_f64<C, VEC, RED, true>);
}

int fused_red() {
  static int v = [] {
    const char* e = getenv("FMM_K2F_RED");
    return e ? atoi(e) : 1;
  }();
  return v;
}

template <typename C>
cudaError_t launch_fused_cfg(const FusedNode* dev_nodes, int count, int64_t m, int64_t n,
                             int64_t k, const double* coef, int P, int Q, int R, const Bases& b,
                             bool vec, cudaStream_t st, int nr, int chunk, int* turn) {
  if (fused_red()) {
    return vec ? launch_fused_kernel<C, true, true>(dev_nodes, count, m, n, k, coef, P, Q, R, b, st, nr, chunk, turn)
               : launch_fused_kernel<C, false, true>(dev_nodes, count, m, n, k, coef, P, Q, R, b, st, nr, chunk, turn);
  }
  return vec ? launch_fused_kernel<C, true, false>(dev_nodes, count, m, n, k, coef, P, Q, R, b, st, nr, chunk, turn)
             : launch_fused_kernel<C, false, false>(dev_nodes, count, m, n, k, coef, P, Q, R, b, st, nr, chunk, turn);
}

template <typename C>
cudaError_t launch_cfg(const LeafNode* dev_leaves, int count, int64_t m, int64_t n, int64_t k,
                       const Bases& b, bool vec, cudaStream_t st) {
  const int tiles_m = (int)((m + C::BM - 1) / C::BM), tiles_n = (int)((n + C::BN - 1) / C::BN);
  dim3 grid((unsigned)(tiles_m * tiles_n), (unsigned)count);
  cudaError_t e;
  if (vec) {
    e = set_smem(k2_gemm_f64<C, true>, C::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    k2_gemm_f64<C, true><<<grid, C::THREADS, C::SMEM_BYTES, st>>>(dev_leaves, b, m, n, k, tiles_m,
                                                                 tiles_n);
  } else {
    e = set_smem(k2_gemm_f64<C, false>, C::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    k2_gemm_f64<C, false><<<grid, C::THREADS, C::SMEM_BYTES, st>>>(dev_leaves, b, m, n, k, tiles_m,
                                                                  tiles_n);
  }
  return cudaGetLastError();
}

// Variants (selected by env FMM_K2_VARIANT for experiments; default chosen from measurements,
// profiles/r01_k2_variants.txt).
using V1 = Cfg<128, 128, 16, 4, 2, 4>;  // 8 warps, 64 x 32 warp tiles
using V2 = Cfg<128, 128, 32, 3, 2, 4>;  // BK = 32
using V3 = Cfg<128, 128, 16, 4, 4, 4>;  // 16 warps, 32 x 32 warp tiles
using V4 = Cfg<128, 128, 32, 3, 4, 4>;  // 16 warps, BK = 32
using V5 = Cfg<64, 128, 16, 4, 2, 4, 2>;  // 8 warps, 32 x 32 warp tiles (2 CTAs / SM)
using V6 = Cfg<64, 128, 16, 3, 2, 4, 2>;
using V7 = Cfg<128, 64, 16, 3, 4, 2, 2>;
using V8 = Cfg<64, 128, 32, 2, 2, 4, 2>;
using V9 = Cfg<64, 64, 16, 4, 2, 2, 3>;   // 4 warps, 3 CTAs / SM
using V10 = Cfg<64, 256, 16, 3, 2, 8, 1>; // 16 warps, 32 x 32 warp tiles
using V11 = Cfg<64, 64, 16, 3, 2, 2, 4>;  // 4 warps, 4 CTAs / SM
using V12 = Cfg<64, 64, 32, 2, 2, 2, 3>;
using V13 = Cfg<64, 64, 16, 4, 2, 2, 3, true>;  // v9 + cross-stage fragment prefetch
using V14 = Cfg<64, 64, 32, 2, 2, 2, 3, true>;
using V15 = Cfg<64, 128, 16, 4, 2, 4, 2, true>;
using V16 = Cfg<128, 128, 16, 4, 2, 4, 1, true>;
using V17 = Cfg<128, 128, 32, 3, 2, 4, 1, true>;
using V18 = Cfg<128, 128, 16, 3, 2, 4, 1, true>;
using V20 = Cfg<128, 128, 16, 5, 2, 4, 1, true>;

int variant() {
  static int v = [] {
    const char* e = getenv("FMM_K2_VARIANT");
    return e ? atoi(e) : 16;
  }();
  return v;
}

}  // namespace

cudaError_t launch_gemm_f64(const LeafNode* dev_leaves, int count, int64_t m, int64_t n,
                            int64_t k, const Bases& b, bool vec, cudaStream_t st) {
  if (count == 0 || m == 0 || n == 0) return cudaSuccess;
  // small batches (fewer 128x128 tiles than two per SM, e.g. C1: 49 leaves of 128^2): 64x64
  // tiles at 3 CTAs per SM give 4x the CTAs (profiles/r01_k2_variants.md: V13 is within 1 % of
  // V16 on large problems)
  const int64_t t128 = ((m + 127) / 128) * ((n + 127) / 128) * (int64_t)count;
  if (!getenv("FMM_K2_VARIANT") && t128 < 2 * 148)
    return launch_cfg<V13>(dev_leaves, count, m, n, k, b, vec, st);
  switch (variant()) {
    case 2: return launch_cfg<V2>(dev_leaves, count, m, n, k, b, vec, st);
    case 3: return launch_cfg<V3>(dev_leaves, count, m, n, k, b, vec, st);
    case 4: return launch_cfg<V4>(dev_leaves, count, m, n, k, b, vec, st);
    case 5: return launch_cfg<V5>(dev_leaves, count, m, n, k, b, vec, st);
    case 6: return launch_cfg<V6>(dev_leaves, count, m, n, k, b, vec, st);
    case 7: return launch_cfg<V7>(dev_leaves, count, m, n, k, b, vec, st);
    case 8: return launch_cfg<V8>(dev_leaves, count, m, n, k, b, vec, st);
    case 9: return launch_cfg<V9>(dev_leaves, count, m, n, k, b, vec, st);
    case 10: return launch_cfg<V10>(dev_leaves, count, m, n, k, b, vec, st);
    case 11: return launch_cfg<V11>(dev_leaves, count, m, n, k, b, vec, st);
    case 12: return launch_cfg<V12>(dev_leaves, count, m, n, k, b, vec, st);
    case 13: return launch_cfg<V13>(dev_leaves, count, m, n, k, b, vec, st);
    case 14: return launch_cfg<V14>(dev_leaves, count, m, n, k, b, vec, st);
    case 15: return launch_cfg<V15>(dev_leaves, count, m, n, k, b, vec, st);
    case 16: return launch_cfg<V16>(dev_leaves, count, m, n, k, b, vec, st);
    case 17: return launch_cfg<V17>(dev_leaves, count, m, n, k, b, vec, st);
    case 18: return launch_cfg<V18>(dev_leaves, count, m, n, k, b, vec, st);
    case 20: return launch_cfg<V20>(dev_leaves, count, m, n, k, b, vec, st);
    case 1: return launch_cfg<V1>(dev_leaves, count, m, n, k, b, vec, st);
    default: return launch_cfg<V16>(dev_leaves, count, m, n, k, b, vec, st);
  }
}

cudaError_t launch_gemm_f64_persistent(const FusedNode* dev_nodes, int count, int64_t m, int64_t n,
                                       int64_t k, const double* dev_coef, int P, int Q, int R,
                                       int NR, int ctas, double* scratch, int* flags,
                                       const Bases& b, bool vec, cudaStream_t st) {
  using Cf = V16;
  if (count == 0 || m == 0 || n == 0) return cudaSuccess;
  const int tiles_m = (int)((m + Cf::BM - 1) / Cf::BM), tiles_n = (int)((n + Cf::BN - 1) / Cf::BN);
  const int64_t U = (int64_t)count * tiles_m * tiles_n;
  // stream-K tail: the last (U mod G) units plus one more wave when there is a full wave to spare
  int64_t tail_units = U % ctas;
  if (U - tail_units >= 2 * (int64_t)ctas) tail_units += ctas;
  if (tail_units > persistent_max_tail_units(ctas)) tail_units = U % ctas;
  const int64_t U_dp = U - tail_units;
  unsigned long long* counter = (unsigned long long*)(flags + (size_t)2 * ctas * NR);
  cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(int) * (size_t)2 * ctas * NR + 16, st);
  if (e != cudaSuccess) return e;
  auto go = [&](auto kern) {
    cudaError_t e2 = set_smem(kern, Cf::SMEM_BYTES);
    if (e2 != cudaSuccess) return e2;
    kern<<<ctas, Cf::THREADS, Cf::SMEM_BYTES, st>>>(dev_nodes, dev_coef, b, m, n, k, tiles_m, tiles_n,
                                                    P, Q, R, NR, U, U_dp, scratch, flags, counter);
    return cudaGetLastError();
  };
  return vec ? go(k2p_gemm_f64<Cf, true>) : go(k2p_gemm_f64<Cf, false>);
}

// scratch: one 128x128 tile per stream-K product-tile (at most 2 G units x NR) + flags + counter
int64_t persistent_max_tail_units(int ctas) { return 2 * (int64_t)ctas; }
size_t persistent_scratch_bytes(int ctas, int NR) {
  using Cf = V16;
  const size_t tiles = (size_t)persistent_max_tail_units(ctas) * NR;
  return tiles * (size_t)(Cf::BM * Cf::BN) * sizeof(double) + tiles * sizeof(int) + 512;
}

int persistent_min_kt() { return V16::STAGES; }

namespace {
int fused_variant() {
  static int v = [] {
    const char* e = getenv("FMM_K2F_VARIANT");
    return e ? atoi(e) : 16;
  }();
  return v;
}
}  // namespace

using VO = Cfg<128, 128, 16, 3, 2, 4, 1, true>;  // operand-fused K2O: 3 stages x (2 A + 2 B slots)

cudaError_t launch_gemm_f64_fused(const FusedNode* dev_nodes, int count, int64_t m, int64_t n,
                                  int64_t k, const double* dev_coef, int P, int Q, int R,
                                  const Bases& b, bool vec, cudaStream_t st, bool opf, int nr,
                                  int chunk, int* turn, int cfg) {
  if (count == 0 || m == 0 || n == 0) return cudaSuccess;
  if (opf) {
    const int tiles_m = (int)((m + VO::BM - 1) / VO::BM), tiles_n = (int)((n + VO::BN - 1) / VO::BN);
    constexpr int smem = VO::STAGES * 2 * (VO::A_STAGE + VO::B_STAGE) * 8;
    auto go = [&](auto kern) {
      cudaError_t e = set_smem(kern, smem);
      if (e != cudaSuccess) return e;
      kern<<<dim3((unsigned)(tiles_m * tiles_n), (unsigned)count), VO::THREADS, smem, st>>>(
          dev_nodes, dev_coef, b, m, n, k, tiles_m, tiles_n, P, Q, R);
      return cudaGetLastError();
    };
    return vec ? go(k2o_gemm_f64<VO, true>) : go(k2o_gemm_f64<VO, false>);
  }
  int v = getenv("FMM_K2F_VARIANT") ? fused_variant() : cfg;
  if (v == 13 && (R > 8 || P * Q > 4)) v = 16;  // v13's product tables hold 2x2 rules, R <= 8
  switch (v) {
    case 13: return launch_fused_cfg<V13>(dev_nodes, count, m, n, k, dev_coef, P, Q, R, b, vec, st, nr, chunk, turn);
    case 15: return launch_fused_cfg<V15>(dev_nodes, count, m, n, k, dev_coef, P, Q, R, b, vec, st, nr, chunk, turn);
    case 17: return launch_fused_cfg<V17>(dev_nodes, count, m, n, k, dev_coef, P, Q, R, b, vec, st, nr, chunk, turn);
    case 18: return launch_fused_cfg<V18>(dev_nodes, count, m, n, k, dev_coef, P, Q, R, b, vec, st, nr, chunk, turn);
    case 20: return launch_fused_cfg<V20>(dev_nodes, count, m, n, k, dev_coef, P, Q, R, b, vec, st, nr, chunk, turn);
    default: return launch_fused_cfg<V16>(dev_nodes, count, m, n, k, dev_coef, P, Q, R, b, vec, st, nr, chunk, turn);
  }
}

}  // namespace fmm
