// HBM-streaming kernels of the recursion (K1 and K3):
//   K1  S_r = sum_i u_ir A_i / T_r = sum_j v_jr B_j   for every node of a level, one pass
//   K3  C_k = sum_r w_kr M_r                          for every node of a level, one pass
//   ACC C_k = w_kr M_r  |  C_k = C_k + w_kr M_r         one top-level r (depth-first / sharded)
//   ZERO blocks of C with no contribution (sharded partial sums)
// Each thread owns one 16-byte vector position (i, j..j+VEC-1) of the sub-block and touches
// the same position in every input / output block, so each input element is read once and
// each output written once per launch (the algorithmic floor).  Sums run sequentially in
// ascending index order with explicit round-to-nearest intrinsics (no FMA contraction),
// exactly the order of PAPER.md's sequential summation model (eqn:seq_summation_error).
#include <algorithm>
#include <cstdlib>
#include <utility>

#include "fmm_internal.h"
#include "builtin_tables.h"
#include "lincomb_dev.cuh"

namespace fmm {

namespace {
// K1X2 launch: grid x = column chunks of kThreadsX2 vectors, y = row groups of RPB grandchild
// rows, z = node (S nodes use the U tables, T nodes the V tables).
template <typename T, int VEC, int RPB, int RA, int RB, bool SPLIT = false>
__global__ void __launch_bounds__(kThreadsX2) k1x2_lincomb(const K1x2Node* __restrict__ nodes,
                                                            Bases bases) {
  __shared__ T* optr[kMaxX2];
  const K1x2Node& nd = nodes[blockIdx.z];
  const int64_t rows = nd.rows, cols = nd.cols;
  if ((int64_t)blockIdx.y * RPB >= rows || (int64_t)blockIdx.x * kThreadsX2 * VEC >= cols) return;
  if (threadIdx.x < nd.nout) {
    int64_t ldo;
    optr[threadIdx.x] = op_ptr<T>(bases, nd.out[threadIdx.x], ldo);
  }
  int64_t ldi;
  const T* in = op_ptr<const T>(bases, nd.in, ldi);
  const int tv = nd.tv;
  __syncthreads();
  const int64_t jv = ((int64_t)blockIdx.x * kThreadsX2 + threadIdx.x) * VEC;
  if (jv >= cols) return;
  const int64_t i0 = (int64_t)blockIdx.y * RPB;
#pragma unroll 1
  for (int ii = 0; ii < RPB; ++ii) {
    const int64_t i = i0 + ii;
    if (i >= rows) break;
    if (tv) k1x2_row<T, VEC, RA, RB, 1, SPLIT>(in, ldi, rows, cols, i, jv, optr, nd.lo_off);
    else k1x2_row<T, VEC, RA, RB, 0, SPLIT>(in, ldi, rows, cols, i, jv, optr, nd.lo_off);
  }
}

// rows per CTA of the two-level passes (tools/bench_k1x2.py sweep: 1 fastest, 0.654 vs 0.688 ms
// with 4 at C2, 25.8 vs 26.7 ms at C5)
int k1x2_rpb() {
  static int v = [] {
    const char* e = getenv("FMM_K1X2_RPB");
    return e ? atoi(e) : 1;
  }();
  return v;
}
int k3x2_rpb() {
  static int v = [] {
    const char* e = getenv("FMM_K3X2_RPB");
    return e ? atoi(e) : 4;  // K3X2: 4 rows per CTA (C2 0.223 vs 0.248 ms with 1, C4 0.090 vs 0.103)
  }();
  return v;
}

template <typename T, int VEC, int RA, int RB, int RPB>
void k1x2_go_rpb(const Step& s, const K1x2Node* nd, const Bases& b, cudaStream_t st) {
  const int64_t cv = (s.cols + VEC - 1) / VEC;
  dim3 grid((unsigned)((cv + kThreadsX2 - 1) / kThreadsX2), (unsigned)((s.rows + RPB - 1) / RPB),
            (unsigned)s.count);
  if constexpr (sizeof(T) == 4) {
    if (s.tf32_split) {
      k1x2_lincomb<T, VEC, RPB, RA, RB, true><<<grid, kThreadsX2, 0, st>>>(nd, b);
      return;
    }
  }
  k1x2_lincomb<T, VEC, RPB, RA, RB><<<grid, kThreadsX2, 0, st>>>(nd, b);
}

template <typename T, int VEC, int RA, int RB>
void k1x2_go(const Step& s, const K1x2Node* nd, const Bases& b, cudaStream_t st) {
  if (k1x2_rpb() == 4) k1x2_go_rpb<T, VEC, RA, RB, 4>(s, nd, b, st);
  else k1x2_go_rpb<T, VEC, RA, RB, 1>(s, nd, b, st);
}

template <typename T, int VEC>
void k1x2_pick(const Step& s, const K1x2Node* nd, const Bases& b, cudaStream_t st) {
  switch (s.x2 - 1) {
    case 0: k1x2_go<T, VEC, 0, 0>(s, nd, b, st); break;
    case 1: k1x2_go<T, VEC, 0, 1>(s, nd, b, st); break;
    case 2: k1x2_go<T, VEC, 0, 2>(s, nd, b, st); break;
    case 3: k1x2_go<T, VEC, 1, 0>(s, nd, b, st); break;
    case 4: k1x2_go<T, VEC, 1, 1>(s, nd, b, st); break;
    case 5: k1x2_go<T, VEC, 1, 2>(s, nd, b, st); break;
    case 6: k1x2_go<T, VEC, 2, 0>(s, nd, b, st); break;
    case 7: k1x2_go<T, VEC, 2, 1>(s, nd, b, st); break;
    default: k1x2_go<T, VEC, 2, 2>(s, nd, b, st); break;
  }
}

// K3X2 launch: grid x = column chunks of kThreadsX2 vectors, y = row groups of RPB, z = node.
// US: the root's combination with the unscale folded in (ur / uc: d_A, d_B of the scaling run)
template <typename T, int VEC, int RPB, int RA, int RB, bool US = false>
__global__ void __launch_bounds__(kThreadsX2) k3x2_combine(const K3x2Node* __restrict__ nodes,
                                                            Bases bases, const double* ur,
                                                            const double* uc) {
  constexpr int NIN = builtin_R(RA) * builtin_R(RB);
  __shared__ const T* iptr[NIN];
  const K3x2Node& nd = nodes[blockIdx.z];
  const int64_t rows = nd.rows, cols = nd.cols;
  if ((int64_t)blockIdx.y * RPB >= rows || (int64_t)blockIdx.x * kThreadsX2 * VEC >= cols) return;
  if (threadIdx.x < NIN) {
    int64_t l;
    iptr[threadIdx.x] = op_ptr<const T>(bases, nd.in[threadIdx.x], l);
  }
  int64_t ldo;
  T* out = op_ptr<T>(bases, nd.out, ldo);
  __syncthreads();
  const int64_t jv = ((int64_t)blockIdx.x * kThreadsX2 + threadIdx.x) * VEC;
  if (jv >= cols) return;
  const int64_t i0 = (int64_t)blockIdx.y * RPB;
#pragma unroll 1
  for (int ii = 0; ii < RPB; ++ii) {
    const int64_t i = i0 + ii;
    if (i >= rows) break;
    if constexpr (US) k3x2_row<T, VEC, RA, RB, true>(iptr, out, ldo, rows, cols, i, jv, ur + nd.out.row0, uc + nd.out.col0);
    else k3x2_row<T, VEC, RA, RB>(iptr, out, ldo, rows, cols, i, jv);
  }
}

template <typename T, int VEC, int RA, int RB, int RPB>
void k3x2_go_rpb(const Step& s, const K3x2Node* nd, const Bases& b, cudaStream_t st, const ScaleIn* sc) {
  const int64_t cv = (s.cols + VEC - 1) / VEC;
  dim3 grid((unsigned)((cv + kThreadsX2 - 1) / kThreadsX2), (unsigned)((s.rows + RPB - 1) / RPB),
            (unsigned)s.count);
  if constexpr (sizeof(T) == 8) {
    if (s.unscale && sc && sc->ur) {
      k3x2_combine<T, VEC, RPB, RA, RB, true><<<grid, kThreadsX2, 0, st>>>(nd, b, sc->ur, sc->uc);
      return;
    }
  }
  k3x2_combine<T, VEC, RPB, RA, RB><<<grid, kThreadsX2, 0, st>>>(nd, b, nullptr, nullptr);
}

template <typename T, int VEC, int RA, int RB>
void k3x2_go(const Step& s, const K3x2Node* nd, const Bases& b, cudaStream_t st, const ScaleIn* sc) {
  if (k3x2_rpb() == 4) k3x2_go_rpb<T, VEC, RA, RB, 4>(s, nd, b, st, sc);
  else k3x2_go_rpb<T, VEC, RA, RB, 1>(s, nd, b, st, sc);
}

template <typename T, int VEC>
void k3x2_pick(const Step& s, const K3x2Node* nd, const Bases& b, cudaStream_t st, const ScaleIn* sc) {
  switch (s.x2 - 1) {
    case 0: k3x2_go<T, VEC, 0, 0>(s, nd, b, st, sc); break;
    case 1: k3x2_go<T, VEC, 0, 1>(s, nd, b, st, sc); break;
    case 2: k3x2_go<T, VEC, 0, 2>(s, nd, b, st, sc); break;
    case 3: k3x2_go<T, VEC, 1, 0>(s, nd, b, st, sc); break;
    case 4: k3x2_go<T, VEC, 1, 1>(s, nd, b, st, sc); break;
    case 5: k3x2_go<T, VEC, 1, 2>(s, nd, b, st, sc); break;
    case 6: k3x2_go<T, VEC, 2, 0>(s, nd, b, st, sc); break;
    case 7: k3x2_go<T, VEC, 2, 1>(s, nd, b, st, sc); break;
    default: k3x2_go<T, VEC, 2, 2>(s, nd, b, st, sc); break;
  }
}

// K3: node output (P*rows x Q*cols) with P = M0, Q = N0; k = ia*Q + jb (row-major).
template <typename T, int VEC, int MAXR, bool US = false>
__global__ void __launch_bounds__(kThreads) k3_combine(const K3Node* __restrict__ nodes,
                                                       const double* __restrict__ coef_all,
                                                       Bases bases, int64_t rows, int64_t cols,
                                                       int P, int Q, int R, const double* ur,
                                                       const double* uc) {
  __shared__ double cf[kMaxBlk * kMaxR];
  __shared__ const T* iptr[kMaxR];
  __shared__ int64_t ild[kMaxR];
  const K3Node& nd = nodes[blockIdx.z];
  const int nk = P * Q;
  for (int t = threadIdx.x; t < nk * R; t += blockDim.x) cf[t] = coef_all[nd.coef_off + t];
  if (threadIdx.x < R) {
    int64_t l;
    iptr[threadIdx.x] = op_ptr<const T>(bases, nd.in[threadIdx.x], l);
    ild[threadIdx.x] = l;
  }
  __syncthreads();
  const int64_t jv = ((int64_t)blockIdx.x * kThreads + threadIdx.x) * VEC;
  if (jv >= cols) return;
  int64_t ldo;
  T* out = op_ptr<T>(bases, nd.out, ldo);
  const int64_t i0 = (int64_t)blockIdx.y * kRowsPerBlock;
  for (int ii = 0; ii < kRowsPerBlock; ++ii) {
    const int64_t i = i0 + ii;
    if (i >= rows) break;
    Vec<T, VEC> m[MAXR];
#pragma unroll
    for (int r = 0; r < MAXR; ++r) {
      if (r < R) m[r] = ld_vec<T, VEC>(iptr[r] + i * ild[r] + jv);
    }
    for (int k = 0; k < nk; ++k) {
      Vec<T, VEC> acc;
      bool started = false;
#pragma unroll
      for (int r = 0; r < MAXR; ++r) {
        if (r >= R) break;
        const double w = cf[k * R + r];
        if (w == 0.0) continue;
        const T wt = (T)w;
#pragma unroll
        for (int e = 0; e < VEC; ++e)
          acc.v[e] = started ? add_rn<T>(acc.v[e], mul_rn<T>(wt, m[r].v[e])) : mul_rn<T>(wt, m[r].v[e]);
        started = true;
      }
      if (!started) {
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc.v[e] = (T)0;
      }
      const int ia = k / Q, jb = k % Q;
      if constexpr (US) {  // the unscale folded in (reading A9)
        const double a = ur[nd.out.row0 + ia * rows + i];
#pragma unroll
        for (int e = 0; e < VEC; ++e)
          acc.v[e] = (T)__dmul_rn(__dmul_rn(a, (double)acc.v[e]), uc[nd.out.col0 + jb * cols + jv + e]);
      }
      st_vec<T, VEC>(out + (ia * rows + i) * ldo + jb * cols + jv, acc);
    }
  }
}

template <typename T, int VEC>
__global__ void __launch_bounds__(kThreads) k_acc(const AccNode* __restrict__ nodes,
                                                  const double* __restrict__ coef_all,
                                                  Bases bases, int64_t rows, int64_t cols, int P,
                                                  int Q, int R) {
  const AccNode& nd = nodes[blockIdx.z];
  const int64_t jv = ((int64_t)blockIdx.x * kThreads + threadIdx.x) * VEC;
  if (jv >= cols) return;
  int64_t ldo, ldm;
  T* out = op_ptr<T>(bases, nd.out, ldo);
  const T* mp = op_ptr<const T>(bases, nd.in, ldm);
  const int64_t i0 = (int64_t)blockIdx.y * kRowsPerBlock;
  for (int ii = 0; ii < kRowsPerBlock; ++ii) {
    const int64_t i = i0 + ii;
    if (i >= rows) break;
    const Vec<T, VEC> m = ld_vec<T, VEC>(mp + i * ldm + jv);
    for (int k = 0; k < P * Q; ++k) {
      const double w = coef_all[nd.coef_off + k * R + nd.r];
      if (w == 0.0) continue;
      const T wt = (T)w;
      const int ia = k / Q, jb = k % Q;
      T* o = out + (ia * rows + i) * ldo + jb * cols + jv;
      Vec<T, VEC> acc;
      if ((nd.first_mask >> k) & 1u) {
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc.v[e] = mul_rn<T>(wt, m.v[e]);
      } else {
        acc = ld_vec<T, VEC>(o);
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc.v[e] = add_rn<T>(acc.v[e], mul_rn<T>(wt, m.v[e]));
      }
      st_vec<T, VEC>(o, acc);
    }
  }
}

template <typename T>
__global__ void k_zero(const ZeroNode* __restrict__ nodes, Bases bases, int64_t rows,
                       int64_t cols, int P, int Q) {
  const ZeroNode& nd = nodes[blockIdx.z];
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  int64_t ldo;
  T* out = op_ptr<T>(bases, nd.out, ldo);
  const int64_t i0 = (int64_t)blockIdx.y * kRowsPerBlock;
  for (int ii = 0; ii < kRowsPerBlock; ++ii) {
    const int64_t i = i0 + ii;
    if (i >= rows) break;
    for (int k = 0; k < P * Q; ++k)
      if ((nd.mask >> k) & 1u) out[((k / Q) * rows + i) * ldo + (k % Q) * cols + j] = (T)0;
  }
}

inline dim3 grid_for(const Step& s, int vec) {
  int64_t cv = (s.cols + vec - 1) / vec;
  return dim3((unsigned)((cv + kThreads - 1) / kThreads),
              (unsigned)((s.rows + kRowsPerBlock - 1) / kRowsPerBlock), (unsigned)s.count);
}

}  // namespace

namespace {
template <typename T, int VEC, int NBLK, int RPB, int RIF, bool SC = false>
void k1_go(const Step& s, const K1Node* nd, const double* dev_coef, const Bases& b, cudaStream_t st,
           const ScaleIn& sc = ScaleIn{}) {
  const int64_t cv = (s.cols + VEC - 1) / VEC;
  dim3 grid((unsigned)((cv + kThreads - 1) / kThreads), (unsigned)((s.rows + RPB - 1) / RPB),
            (unsigned)s.count);
  k1_lincomb<T, VEC, NBLK, RPB, RIF, SC><<<grid, kThreads, 0, st>>>(nd, dev_coef, b, s.rows, s.cols, s.P, s.Q, s.R, sc);
}

}  // namespace

// K1C: a one-level K1 pass whose nodes all use built-in rule RA (2x2 blocks): the output list
// and every +-1 code are compile-time constants (as in K1X2), so a row is 4 loads, the adds and
// the stores -- the run-time code interpretation of k1_lincomb is issue-bound once a node forms
// all 7 or 8 products (the scaled root: its trivial columns are scaled copies, not views).
// Outputs r outside the node's out_mask (views) are skipped.  SC: virtual scaling as in
// k1_lincomb.  Same per-element operation sequence as k1_lincomb: bitwise equal.
// first nonzero term of column r (block order b ascending)
__host__ __device__ constexpr bool k1c_first(int id, int tv, int b, int r) {
  for (int q = 0; q < b; ++q)
    if (builtin_coef(id, tv, q, r) != 0) return false;
  return true;
}

template <typename T, int VEC, int RA, int TV, bool SC>
__device__ __forceinline__ void k1c_row(const Vec<T, VEC> (&x)[4], T* const* optr, const int64_t* old,
                                        int64_t i, int64_t jv) {
  constexpr int R = builtin_R(RA);
  static_for<R>([&](auto r) {
    if (optr[r]) {
      Vec<T, VEC> acc;
      static_for<4>([&](auto b) {
        constexpr int c = builtin_coef(RA, TV, b, r);
        if constexpr (c != 0) {
          lc_fixed<c == 1 ? 1u : 2u>(acc, k1c_first(RA, TV, b, r), x[b]);
        }
      });
      st_vec<T, VEC>(optr[r] + i * old[r] + jv, acc);
    }
  });
}

template <typename T, int VEC, int RA, bool SC>
__global__ void __launch_bounds__(kThreads) k1c_lincomb(const K1Node* __restrict__ nodes, Bases bases,
                                                        ScaleIn sc) {
  constexpr int RPB = 8;
  constexpr int R = builtin_R(RA);
  __shared__ T* optr[kMaxR];
  __shared__ int64_t old[kMaxR];
  const K1Node& nd = nodes[blockIdx.z];
  const int64_t rows = nd.rows, cols = nd.cols;
  if ((int64_t)blockIdx.y * RPB >= rows || (int64_t)blockIdx.x * kThreads * VEC >= cols) return;
  if (threadIdx.x < R) {
    const int r = threadIdx.x;
    int64_t ldo = 0;
    optr[r] = ((nd.out_mask >> r) & 1u) ? op_ptr<T>(bases, nd.out[r], ldo) : nullptr;
    old[r] = ldo;
  }
  int64_t ldi;
  const T* in = op_ptr<const T>(bases, nd.in, ldi);
  __syncthreads();
  const int64_t jv = ((int64_t)blockIdx.x * kThreads + threadIdx.x) * VEC;
  if (jv >= cols) return;
  const int64_t i0 = (int64_t)blockIdx.y * RPB;
  const int side = nd.tv;
  bool vscale = false, fast = false;
  const int32_t* ers = nullptr;
  int ecv[4][VEC];
  double fcv[4][VEC];
  if constexpr (SC) {
    if (*sc.mode != 0) {  // the scaling run materialised A' / B'
      ldi = side ? sc.ldm[1] : sc.ldm[0];
      in = (const T*)(side ? sc.mat[1] : sc.mat[0]) + nd.in.row0 * ldi + nd.in.col0;
    } else {
      vscale = true;
      ers = (side ? sc.er[1] : sc.er[0]) + nd.in.row0;
      const int32_t* ecs = (side ? sc.ec[1] : sc.ec[0]) + nd.in.col0;
      const int* ex = sc.ext + 4 * side;
      fast = ex[0] >= -1022 && ex[1] <= 1023 && ex[2] >= -1022 && ex[3] <= 1023 &&
             ex[0] + ex[2] >= -1022 && ex[1] + ex[3] <= 1023;
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          ecv[b][e] = jv + e < cols ? ecs[(b / 2) * cols + jv + e] : 0;
          fcv[b][e] = fast ? __longlong_as_double((int64_t)(ecv[b][e] + 1023) << 52) : 1.0;
        }
    }
  }
#pragma unroll 1
  for (int ii = 0; ii < RPB; ii += 2) {
    Vec<T, VEC> x[2][4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t i = i0 + ii + h;
      if (i < rows) {
#pragma unroll
        for (int b = 0; b < 4; ++b)  // block b = p + 2 q (column-major)
          x[h][b] = ld_vec<T, VEC>(in + ((b % 2) * rows + i) * ldi + (b / 2) * cols + jv);
      }
    }
    if constexpr (SC) {
      if (vscale) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t i = i0 + ii + h;
          if (i >= rows) break;
          const int er[2] = {ers[i], ers[rows + i]};
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            if (fast) {
              const double fr = __longlong_as_double((int64_t)(er[b % 2] + 1023) << 52);
#pragma unroll
              for (int e = 0; e < VEC; ++e) x[h][b].v[e] = (T)__dmul_rn((double)x[h][b].v[e], __dmul_rn(fr, fcv[b][e]));
            } else {
#pragma unroll
              for (int e = 0; e < VEC; ++e) x[h][b].v[e] = (T)scale2((double)x[h][b].v[e], er[b % 2] + ecv[b][e]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t i = i0 + ii + h;
      if (i >= rows) break;
      if (side == 0) k1c_row<T, VEC, RA, 0, SC>(x[h], optr, old, i, jv);
      else k1c_row<T, VEC, RA, 1, SC>(x[h], optr, old, i, jv);
    }
  }
}

template <typename T, int VEC, int RA, bool SC>
void k1c_go(const Step& s, const K1Node* nd, const Bases& b, cudaStream_t st, const ScaleIn& sc) {
  const int64_t cv = (s.cols + VEC - 1) / VEC;
  dim3 grid((unsigned)((cv + kThreads - 1) / kThreads), (unsigned)((s.rows + 7) / 8), (unsigned)s.count);
  k1c_lincomb<T, VEC, RA, SC><<<grid, kThreads, 0, st>>>(nd, b, sc);
}

template <typename T, int VEC, bool SC>
void k1c_pick(const Step& s, const K1Node* nd, const Bases& b, cudaStream_t st, const ScaleIn& sc) {
  switch (s.x1 - 1) {
    case 0: k1c_go<T, VEC, 0, SC>(s, nd, b, st, sc); break;
    case 1: k1c_go<T, VEC, 1, SC>(s, nd, b, st, sc); break;
    default: k1c_go<T, VEC, 2, SC>(s, nd, b, st, sc); break;
  }
}

template <typename T>
cudaError_t launch_k1(const Step& s, const void* dev_nodes, const double* dev_coef,
                      const Bases& b, bool vec, cudaStream_t st, const ScaleIn* sc) {
  if (s.count == 0 || s.rows == 0 || s.cols == 0) return cudaSuccess;
  constexpr int V = 16 / sizeof(T);
  if (s.x1 && !s.x2) {  // nodes on one built-in 2x2 rule: compile-time specialised
    const K1Node* nd = (const K1Node*)dev_nodes;
    const bool scd = sc && s.scaled;
    if constexpr (sizeof(T) == 8) {
      if (scd) {
        if (vec) k1c_pick<T, V, true>(s, nd, b, st, *sc);
        else k1c_pick<T, 1, true>(s, nd, b, st, *sc);
        return cudaGetLastError();
      }
    }
    if (vec) k1c_pick<T, V, false>(s, nd, b, st, ScaleIn{});
    else k1c_pick<T, 1, false>(s, nd, b, st, ScaleIn{});
    return cudaGetLastError();
  }
  if (sc && s.scaled && !s.x2) {  // the root under virtual scaling (FP64 plans only)
    // 16 rows per block: the per-block setup (mode flag, column exponents) is a dependent
    // load chain, amortised over 4x the rows of the plain pass
    const K1Node* nd = (const K1Node*)dev_nodes;
    if (s.P * s.Q <= 4) {
      if (vec) k1_go<T, V, 4, 16, 2, true>(s, nd, dev_coef, b, st, *sc);
      else k1_go<T, 1, 4, 16, 2, true>(s, nd, dev_coef, b, st, *sc);
    } else {
      if (vec) k1_go<T, V, kMaxBlk, 4, 1, true>(s, nd, dev_coef, b, st, *sc);
      else k1_go<T, 1, kMaxBlk, 4, 1, true>(s, nd, dev_coef, b, st, *sc);
    }
    return cudaGetLastError();
  }
  if (s.x2) {
    if (vec) k1x2_pick<T, V>(s, (const K1x2Node*)dev_nodes, b, st);
    else k1x2_pick<T, 1>(s, (const K1x2Node*)dev_nodes, b, st);
    return cudaGetLastError();
  }
  const K1Node* nd = (const K1Node*)dev_nodes;
  // 4 rows per block, 2 in flight: 6.58 TB/s (tools/bench_passes.py, the fastest of the
  // round-1 rows-per-block sweep)
  if (s.P * s.Q <= 4) {
    if (vec) k1_go<T, V, 4, 4, 2>(s, nd, dev_coef, b, st);
    else k1_go<T, 1, 4, 4, 2>(s, nd, dev_coef, b, st);
  } else {
    if (vec) k1_go<T, V, kMaxBlk, 4, 1>(s, nd, dev_coef, b, st);
    else k1_go<T, 1, kMaxBlk, 4, 1>(s, nd, dev_coef, b, st);
  }
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_k3(const Step& s, const void* dev_nodes, const double* dev_coef,
                      const Bases& b, bool vec, cudaStream_t st, const ScaleIn* sc) {
  if (s.count == 0 || s.rows == 0 || s.cols == 0) return cudaSuccess;
  constexpr int V = 16 / sizeof(T);
  if (s.x2) {
    if (vec) k3x2_pick<T, V>(s, (const K3x2Node*)dev_nodes, b, st, sc);
    else k3x2_pick<T, 1>(s, (const K3x2Node*)dev_nodes, b, st, sc);
    return cudaGetLastError();
  }
  const K3Node* nd = (const K3Node*)dev_nodes;
  const bool us = sizeof(T) == 8 && s.unscale && sc && sc->ur;
  const double* ur = us ? sc->ur : nullptr;
  const double* uc = us ? sc->uc : nullptr;
#define FMM_K3(V_, MR_, US_) k3_combine<T, V_, MR_, US_><<<grid_for(s, V_), kThreads, 0, st>>>(nd, dev_coef, b, s.rows, s.cols, s.P, s.Q, s.R, ur, uc)
  if (s.R <= 8) {
    if (us) { if (vec) FMM_K3(V, 8, true); else FMM_K3(1, 8, true); }
    else { if (vec) FMM_K3(V, 8, false); else FMM_K3(1, 8, false); }
  } else {
    if (us) { if (vec) FMM_K3(V, kMaxR, true); else FMM_K3(1, kMaxR, true); }
    else { if (vec) FMM_K3(V, kMaxR, false); else FMM_K3(1, kMaxR, false); }
  }
#undef FMM_K3
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_acc(const Step& s, const void* dev_nodes, const double* dev_coef,
                       const Bases& b, bool vec, cudaStream_t st) {
  if (s.count == 0 || s.rows == 0 || s.cols == 0) return cudaSuccess;
  constexpr int V = 16 / sizeof(T);
  if (vec)
    k_acc<T, V><<<grid_for(s, V), kThreads, 0, st>>>((const AccNode*)dev_nodes, dev_coef, b,
                                                     s.rows, s.cols, s.P, s.Q, s.R);
  else
    k_acc<T, 1><<<grid_for(s, 1), kThreads, 0, st>>>((const AccNode*)dev_nodes, dev_coef, b,
                                                     s.rows, s.cols, s.P, s.Q, s.R);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_zero(const Step& s, const void* dev_nodes, const Bases& b, cudaStream_t st) {
  if (s.count == 0 || s.rows == 0 || s.cols == 0) return cudaSuccess;
  k_zero<T><<<grid_for(s, 1), kThreads, 0, st>>>((const ZeroNode*)dev_nodes, b, s.rows, s.cols,
                                                 s.P, s.Q);
  return cudaGetLastError();
}

namespace {
// One thread per VEC-vector of a C row: block k = ia * N0 + jb of the element, then the
// sequential sum over r ascending of w_kr M_r (first term initialises) -- ACC's order, so the
// result is bitwise the single-GPU C.  Peer pointers are UVA addresses of the other ranks'
// symmetric buffers (CUDA IPC), so the loads of non-local products travel over NVLink.
template <typename T, int VEC>
__global__ void __launch_bounds__(kThreads) k_p2p_combine(const T* const* __restrict__ peers, int P,
                                                          const double* __restrict__ coef, int R,
                                                          int nw, int N0, int64_t mb, int64_t nb,
                                                          T* C, int64_t ldc, int64_t row0,
                                                          int64_t row1) {
  __shared__ double w[kMaxBlk * kMaxR];
  __shared__ const T* src[kMaxR];
  for (int t = threadIdx.x; t < nw; t += blockDim.x) w[t] = coef[t];
  if (threadIdx.x < R) src[threadIdx.x] = peers[threadIdx.x % P] + (int64_t)(threadIdx.x / P) * mb * nb;
  __syncthreads();
  const int64_t j = ((int64_t)blockIdx.x * kThreads + threadIdx.x) * VEC;
  if (j >= (int64_t)N0 * nb) return;
  const int jb = (int)(j / nb);
  const int64_t jj = j % nb;
  for (int64_t i = row0 + blockIdx.y; i < row1; i += gridDim.y) {
    const int ia = (int)(i / mb);
    const int64_t ii = i % mb;
    const int k = ia * N0 + jb;
    Vec<T, VEC> acc;
    bool started = false;
    for (int r = 0; r < R; ++r) {
      const double wk = w[k * R + r];
      if (wk == 0.0) continue;
      const Vec<T, VEC> m = ld_vec<T, VEC>(src[r] + ii * nb + jj);
      const T wt = (T)wk;
#pragma unroll
      for (int e = 0; e < VEC; ++e)
        acc.v[e] = started ? add_rn<T>(acc.v[e], mul_rn<T>(wt, m.v[e])) : mul_rn<T>(wt, m.v[e]);
      started = true;
    }
    if (!started) {
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc.v[e] = (T)0;
    }
    st_vec<T, VEC>(C + i * ldc + j, acc);
  }
}

template <typename T>
__global__ void k_pad_copy(const T* __restrict__ src, int64_t rows, int64_t cols, int64_t lds,
                           T* __restrict__ dst, int64_t rows_p, int64_t cols_p, int64_t ldd) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols_p) return;
  for (int64_t i = blockIdx.y; i < rows_p; i += gridDim.y)
    dst[i * ldd + j] = (i < rows && j < cols) ? src[i * lds + j] : (T)0;
}
}  // namespace

template <typename T>
cudaError_t launch_pad_copy(const T* src, int64_t rows, int64_t cols, int64_t lds, T* dst,
                            int64_t rows_p, int64_t cols_p, int64_t ldd, cudaStream_t st) {
  if (rows_p == 0 || cols_p == 0) return cudaSuccess;
  dim3 grid((unsigned)((cols_p + kThreads - 1) / kThreads), (unsigned)std::min<int64_t>(rows_p, 65535));
  k_pad_copy<T><<<grid, kThreads, 0, st>>>(src, rows, cols, lds, dst, rows_p, cols_p, ldd);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_p2p_combine(const T* const* dev_peers, int P, const double* dev_coef, int coef_off,
                               int R, int M0, int N0, int64_t mb, int64_t nb, T* C, int64_t ldc,
                               int64_t row0, int64_t row1, bool vec, cudaStream_t st) {
  if (row1 <= row0 || nb == 0) return cudaSuccess;
  constexpr int V = 16 / sizeof(T);
  const int vv = vec ? V : 1;
  const int64_t cv = (N0 * nb + vv - 1) / vv;
  dim3 grid((unsigned)((cv + kThreads - 1) / kThreads), (unsigned)std::min<int64_t>(row1 - row0, 65535));
  if (vec)
    k_p2p_combine<T, V><<<grid, kThreads, 0, st>>>(dev_peers, P, dev_coef + coef_off, R, M0 * N0 * R, N0, mb, nb, C, ldc, row0, row1);
  else
    k_p2p_combine<T, 1><<<grid, kThreads, 0, st>>>(dev_peers, P, dev_coef + coef_off, R, M0 * N0 * R, N0, mb, nb, C, ldc, row0, row1);
  return cudaGetLastError();
}

template cudaError_t launch_p2p_combine<double>(const double* const*, int, const double*, int, int, int, int, int64_t, int64_t, double*, int64_t, int64_t, int64_t, bool, cudaStream_t);
template cudaError_t launch_p2p_combine<float>(const float* const*, int, const double*, int, int, int, int, int64_t, int64_t, float*, int64_t, int64_t, int64_t, bool, cudaStream_t);
template cudaError_t launch_pad_copy<double>(const double*, int64_t, int64_t, int64_t, double*, int64_t, int64_t, int64_t, cudaStream_t);
template cudaError_t launch_pad_copy<float>(const float*, int64_t, int64_t, int64_t, float*, int64_t, int64_t, int64_t, cudaStream_t);
template cudaError_t launch_k1<double>(const Step&, const void*, const double*, const Bases&, bool, cudaStream_t, const ScaleIn*);
template cudaError_t launch_k1<float>(const Step&, const void*, const double*, const Bases&, bool, cudaStream_t, const ScaleIn*);
template cudaError_t launch_k3<double>(const Step&, const void*, const double*, const Bases&, bool, cudaStream_t, const ScaleIn*);
template cudaError_t launch_k3<float>(const Step&, const void*, const double*, const Bases&, bool, cudaStream_t, const ScaleIn*);
template cudaError_t launch_acc<double>(const Step&, const void*, const double*, const Bases&, bool, cudaStream_t);
template cudaError_t launch_acc<float>(const Step&, const void*, const double*, const Bases&, bool, cudaStream_t);
template cudaError_t launch_zero<double>(const Step&, const void*, const Bases&, cudaStream_t);
template cudaError_t launch_zero<float>(const Step&, const void*, const Bases&, cudaStream_t);

}  // namespace fmm
