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

#include "fmm_internal.h"
#include "gemm_f64_dev.cuh"

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

template <typename C, bool VEC, bool FLAT, bool UNITW>
__global__ void __launch_bounds__(C::THREADS, C::MINB)
    k2f_gemm_f64(const FusedNode* __restrict__ nodes, const double* __restrict__ coef_all,
                 Bases bases, int64_t m, int64_t n, int64_t k, int tiles_m, int tiles_n, int P,
                 int Q, int R, int count, uint32_t split, int* __restrict__ turn) {
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

  // Product chain split (`turn` non-null; byte g of `split` = end of group g's products): the
  // work item -- (group, parent, tile), group-major -- comes from a ticket taken with atomicAdd
  // when the CTA starts, not from blockIdx, so tickets follow the actual dispatch order.  Group
  // g runs products [end(g-1), end(g)) of its unit after group g-1 released the unit's
  // turnstile (so every C_k element still sees ascending r); group g-1 of the unit holds an
  // earlier ticket, i.e. its CTA is already running, so the wait always ends (no assumption on
  // the CTA dispatch order).  turn[0 .. count*tiles) are the turnstiles, turn[count*tiles] the
  // ticket counter (zeroed by the launcher).  A persistent form (CTAs looping over tickets, the
  // next one prefetched) measured slower at C2, C4 and C5 and was dropped.
  const int tid = threadIdx.x;
  const int tiles = tiles_m * tiles_n;
  __shared__ int s_ticket;
  int parent = blockIdx.y, grp = 0, tile = blockIdx.x;
  if (turn) {
    if (tid == 0) s_ticket = atomicAdd(turn + (int64_t)count * tiles, 1);
    __syncthreads();
    const int tk = s_ticket, per_grp = count * tiles;
    grp = tk / per_grp;
    parent = (tk % per_grp) / tiles;
    tile = tk % tiles;
  }
  const FusedNode& nd = nodes[parent];
  const int nr_all = nd.nr;
  const int r_begin = grp ? (int)((split >> (8 * (grp - 1))) & 0xffu) : 0;
  const int nr = (turn ? (int)((split >> (8 * grp)) & 0xffu) : nr_all) - r_begin;  // this CTA's
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
  int* my_turn = turn ? turn + (int64_t)parent * tiles + tile : nullptr;
  auto turn_wait = [&]() {  // before this CTA's first epilogue: group grp-1 is done with the unit
    if (grp == 0 || !my_turn) return;
    if (tid == 0) {
      unsigned ns = 64;
      while (atomicAdd(my_turn, 0) < grp) {  // grp-1 holds an earlier ticket: it is running
        __nanosleep(ns);
        if (ns < 2048) ns *= 2;
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
  // first contribution: c = w*m (plain store); later ones: c = c + w*m as L2 reductions
  // (RED.ADD.F64, round to nearest) with no load round trip.  Only this thread updates these
  // elements, and same-address operations of one thread are applied in program order, so the
  // per-element sequence is K3's.
  auto store_block = [&](double* ob, int64_t ldo, bool first, auto&& wmul) {
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
          const double v0 = wmul(acc[i][j][2 * h]), v1 = wmul(acc[i][j][2 * h + 1]);
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
      if constexpr (UNITW)  // every w is +-1: w*m is exact, a sign flip on the integer pipe
        store_block(ob, ldo, first, [&](double x) {
          return __longlong_as_double(__double_as_longlong(x) ^ (w < 0 ? INT64_MIN : 0));
        });
      else
        store_block(ob, ldo, first, [&](double x) { return __dmul_rn(w, x); });
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

template <typename C, bool VEC>
cudaError_t launch_fused_kernel(const FusedNode* dev_nodes, int count, int64_t m, int64_t n,
                                int64_t k, const double* coef, int P, int Q, int R,
                                const Bases& b, cudaStream_t st, int nr, uint32_t split, int* turn,
                                bool unitw) {
  const int tiles_m = (int)((m + C::BM - 1) / C::BM), tiles_n = (int)((n + C::BN - 1) / C::BN);
  const int KT = (int)std::max<int64_t>(1, (k + C::BK - 1) / C::BK);
  int groups = split_groups(split, nr);
  if (groups <= 0) return cudaErrorInvalidValue;
  if (KT < C::STAGES || !turn) groups = 1;  // no split
  if (groups > 1) {  // turnstiles + the ticket counter
    cudaError_t e = cudaMemsetAsync(turn, 0, sizeof(int) * ((size_t)count * tiles_m * tiles_n + 1), st);
    if (e != cudaSuccess) return e;
  }
  auto go = [&](auto kern) {
    cudaError_t e = set_smem(kern, C::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    const dim3 grid((unsigned)(tiles_m * tiles_n), (unsigned)(count * groups));
    kern<<<grid, C::THREADS, C::SMEM_BYTES, st>>>(dev_nodes, coef, b, m, n, k, tiles_m, tiles_n, P,
                                                  Q, R, count, split, groups > 1 ? turn : nullptr);
    return cudaGetLastError();
  };
  if (KT >= C::STAGES)
    return unitw ? go(k2f_gemm_f64<C, VEC, false, true>) : go(k2f_gemm_f64<C, VEC, false, false>);
  return unitw ? go(k2f_gemm_f64<C, VEC, true, true>) : go(k2f_gemm_f64<C, VEC, true, false>);
}

template <typename C>
cudaError_t launch_cfg(const LeafNode* dev_leaves, int count, int64_t m, int64_t n, int64_t k,
                       const Bases& b, bool vec, cudaStream_t st) {
  const int tiles_m = (int)((m + C::BM - 1) / C::BM), tiles_n = (int)((n + C::BN - 1) / C::BN);
  dim3 grid((unsigned)(tiles_m * tiles_n), (unsigned)count);
  auto go = [&](auto kern) {
    cudaError_t e = set_smem(kern, C::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    kern<<<grid, C::THREADS, C::SMEM_BYTES, st>>>(dev_leaves, b, m, n, k, tiles_m, tiles_n);
    return cudaGetLastError();
  };
  return vec ? go(k2_gemm_f64<C, true>) : go(k2_gemm_f64<C, false>);
}

// The two tile configurations kept from the round-1 sweep (profiles/r01_k2_variants.md,
// profiles/r01_fusion_variants.md): 128 x 128 x 16, 8 warps of 64 x 32, 4 stages, one CTA per
// SM (v16: large leaves), and 64 x 64 x 16, 4 warps of 32 x 32, 4 stages, 3 CTAs per SM (v13:
// small batches and short leaf inner dimensions); both with the cross-stage fragment prefetch.
using V13 = Cfg<64, 64, 16, 4, 2, 2, 3, true>;
using V16 = Cfg<128, 128, 16, 4, 2, 4, 1, true>;

}  // namespace

// Groups of a chain split `split` (byte g = end of group g's products, ascending, the last one
// = nr; 0 = no split) for chains of nr products: 1..4, or -1 when malformed.
int split_groups(uint32_t split, int nr) {
  if (split == 0) return 1;
  int prev = 0;
  for (int g = 0; g < 4; ++g) {
    const int e = (int)((split >> (8 * g)) & 0xffu);
    if (e <= prev || e > nr) return -1;
    if (e == nr) return (g + 1 < 4 && (split >> (8 * (g + 1))) != 0u) ? -1 : g + 1;
    prev = e;
  }
  return -1;
}

int k2f_tile_of(int cfg) { return cfg == 13 ? V13::BM : V16::BM; }

cudaError_t launch_gemm_f64(const LeafNode* dev_leaves, int count, int64_t m, int64_t n,
                            int64_t k, const Bases& b, bool vec, cudaStream_t st) {
  if (count == 0 || m == 0 || n == 0) return cudaSuccess;
  // small batches (fewer 128x128 tiles than two per SM, e.g. C1: 49 leaves of 128^2): 64x64
  // tiles at 3 CTAs per SM give 4x the CTAs (profiles/r01_k2_variants.md: V13 is within 1 % of
  // V16 on large problems)
  const int64_t t128 = ((m + 127) / 128) * ((n + 127) / 128) * (int64_t)count;
  if (t128 < 2 * 148) return launch_cfg<V13>(dev_leaves, count, m, n, k, b, vec, st);
  return launch_cfg<V16>(dev_leaves, count, m, n, k, b, vec, st);
}

cudaError_t launch_gemm_f64_fused(const FusedNode* dev_nodes, int count, int64_t m, int64_t n,
                                  int64_t k, const double* dev_coef, int P, int Q, int R,
                                  const Bases& b, bool vec, cudaStream_t st, int nr, uint32_t split,
                                  int* turn, int cfg, bool unitw) {
  if (count == 0 || m == 0 || n == 0) return cudaSuccess;
  if (cfg == 13 && (R > 8 || P * Q > 4)) return cudaErrorInvalidValue;  // v13's tables: 2x2, R <= 8
  if (cfg == 13)
    return vec ? launch_fused_kernel<V13, true>(dev_nodes, count, m, n, k, dev_coef, P, Q, R, b, st, nr, split, turn, unitw)
               : launch_fused_kernel<V13, false>(dev_nodes, count, m, n, k, dev_coef, P, Q, R, b, st, nr, split, turn, unitw);
  // the 128 x 128 kernel keeps the DMUL epilogue: its leaves are long (the epilogue is rare)
  // and the sign-flip variant's main loop schedules worse at 255 registers (C5 +0.9 %)
  return vec ? launch_fused_kernel<V16, true>(dev_nodes, count, m, n, k, dev_coef, P, Q, R, b, st, nr, split, turn, false)
             : launch_fused_kernel<V16, false>(dev_nodes, count, m, n, k, dev_coef, P, Q, R, b, st, nr, split, turn, false);
}

}  // namespace fmm
