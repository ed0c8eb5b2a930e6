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

namespace fmm {

namespace {

template <typename T>
__device__ __forceinline__ T mul_rn(T a, T b);
template <>
__device__ __forceinline__ double mul_rn<double>(double a, double b) { return __dmul_rn(a, b); }
template <>
__device__ __forceinline__ float mul_rn<float>(float a, float b) { return __fmul_rn(a, b); }
template <typename T>
__device__ __forceinline__ T add_rn(T a, T b);
template <>
__device__ __forceinline__ double add_rn<double>(double a, double b) { return __dadd_rn(a, b); }
template <>
__device__ __forceinline__ float add_rn<float>(float a, float b) { return __fadd_rn(a, b); }

template <typename T, int VEC>
struct Vec {
  T v[VEC];
};

template <typename T, int VEC>
__device__ __forceinline__ Vec<T, VEC> ld_vec(const T* p) {
  Vec<T, VEC> r;
  if constexpr (VEC * sizeof(T) == 16) {
    if constexpr (sizeof(T) == 8) {
      double2 x = *reinterpret_cast<const double2*>(p);
      r.v[0] = x.x;
      r.v[1] = x.y;
    } else {
      float4 x = *reinterpret_cast<const float4*>(p);
      r.v[0] = x.x; r.v[1] = x.y; r.v[2] = x.z; r.v[3] = x.w;
    }
  } else {
#pragma unroll
    for (int e = 0; e < VEC; ++e) r.v[e] = p[e];
  }
  return r;
}

template <typename T, int VEC>
__device__ __forceinline__ void st_vec(T* p, const Vec<T, VEC>& r) {
  if constexpr (VEC * sizeof(T) == 16) {
    if constexpr (sizeof(T) == 8) {
      *reinterpret_cast<double2*>(p) = make_double2(r.v[0], r.v[1]);
    } else {
      *reinterpret_cast<float4*>(p) = make_float4(r.v[0], r.v[1], r.v[2], r.v[3]);
    }
  } else {
#pragma unroll
    for (int e = 0; e < VEC; ++e) p[e] = r.v[e];
  }
}

constexpr int kThreads = 256;  // threads per block (x: column vectors)
constexpr int kRowsPerBlock = 4;

// K1 grid: x = column chunks of kThreads vectors, y = row groups of RPB rows, z = node.
// NBLK: compile-time bound on the number of input sub-blocks (4 for 2x2 rules) so that the
// per-thread input registers stay small; RIF rows are loaded before any is combined, so each
// thread keeps up to RIF*NBLK 16-byte loads in flight.  The output list (which r, and per r a
// 2-bit code per input block: 0 absent, 1 +1, 2 -1, 3 general coefficient) is compiled on the
// host into the node descriptor (k1_compile); threads 0..nout-1 resolve the output pointers in
// parallel, so the per-block setup is one shared-memory round trip.  u*x with u = +-1 is exact,
// so adding +-x is bitwise the oracle's  s + u*x.
// x 2^e correctly rounded (virtual scaling: one multiplication by an exact power of two)
__device__ __forceinline__ double scale2(double x, int e) {
  if (e == 0) return x;
  if (e >= -1022 && e <= 1023) return __dmul_rn(x, __longlong_as_double((int64_t)(e + 1023) << 52));
  return ldexp(x, e);
}

// SC: the root's K1 under virtual scaling (ScaleIn): inputs are the original A / B scaled on
// load by 2^(er_i + ec_j) -- bitwise the materialised A' / B' -- or the materialised A' / B'.
template <typename T, int VEC, int NBLK, int RPB, int RIF, bool SC = false>
__global__ void __launch_bounds__(kThreads) k1_lincomb(const K1Node* __restrict__ nodes,
                                                       const double* __restrict__ coef_all,
                                                       Bases bases, int64_t rows, int64_t cols,
                                                       int P, int Q, int R, ScaleIn sc) {
  __shared__ T* optr[kMaxR];
  __shared__ int64_t old[kMaxR];
  __shared__ uint32_t code[kMaxR];
  __shared__ int rlist[kMaxR];
  const K1Node& nd = nodes[blockIdx.z];
  // per-node split (S and T nodes of a level share one launch; the grid covers the largest)
  P = nd.P;
  Q = nd.Q;
  rows = nd.rows;
  cols = nd.cols;
  if ((int64_t)blockIdx.y * RPB >= rows || (int64_t)blockIdx.x * kThreads * VEC >= cols) return;
  const int nblk = P * Q;
  const int nout = nd.nout;
  const uint32_t need = nd.need;
  if (threadIdx.x < nout) {
    const int r = nd.rlist[threadIdx.x];
    int64_t ldo;
    optr[threadIdx.x] = op_ptr<T>(bases, nd.out[r], ldo);
    old[threadIdx.x] = ldo;
    code[threadIdx.x] = nd.code[threadIdx.x];
    rlist[threadIdx.x] = r;
  }
  int64_t ldi;
  const T* in = op_ptr<const T>(bases, nd.in, ldi);
  __syncthreads();

  const int64_t jv = ((int64_t)blockIdx.x * kThreads + threadIdx.x) * VEC;
  if (jv >= cols) return;
  const int64_t i0 = (int64_t)blockIdx.y * RPB;
  // virtual scaling: the exponents of this thread's columns (fixed over its rows)
  const int side = nd.in.base == BASE_B ? 1 : 0;
  bool vscale = false;
  const int32_t* ers = nullptr;
  int ecv[NBLK][VEC];
  if constexpr (SC) {
    if (*sc.mode != 0) {  // the scaling run materialised A' / B'
      in = (const T*)(side ? sc.mat[1] : sc.mat[0]) + nd.in.row0 * (side ? sc.ldm[1] : sc.ldm[0]) + nd.in.col0;
      ldi = side ? sc.ldm[1] : sc.ldm[0];
    } else {
      vscale = true;
      ers = (side ? sc.er[1] : sc.er[0]) + nd.in.row0;
      const int32_t* ecs = (side ? sc.ec[1] : sc.ec[0]) + nd.in.col0;
#pragma unroll
      for (int b = 0; b < NBLK; ++b)
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          const int q = b / P;
          ecv[b][e] = (b < nblk && jv + e < cols) ? ecs[q * cols + jv + e] : 0;
        }
    }
  }
#pragma unroll 1
  for (int ii = 0; ii < RPB; ii += RIF) {
    Vec<T, VEC> x[RIF][NBLK];
#pragma unroll
    for (int h = 0; h < RIF; ++h) {
      const int64_t i = i0 + ii + h;
#pragma unroll
      for (int b = 0; b < NBLK; ++b) {
        if (b < nblk && ((need >> b) & 1u) && i < rows) {
          const int p = b % P, q = b / P;  // column-major block index
          x[h][b] = ld_vec<T, VEC>(in + (p * rows + i) * ldi + q * cols + jv);
          if constexpr (SC) {
            if (vscale) {
              const int er = ers[p * rows + i];
#pragma unroll
              for (int e = 0; e < VEC; ++e) x[h][b].v[e] = (T)scale2((double)x[h][b].v[e], er + ecv[b][e]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int h = 0; h < RIF; ++h) {
      const int64_t i = i0 + ii + h;
      if (i >= rows) break;
#pragma unroll 1
      for (int o = 0; o < nout; ++o) {
        const uint32_t c = code[o];
        Vec<T, VEC> acc;
        bool started = false;
#pragma unroll
        for (int b = 0; b < NBLK; ++b) {
          const uint32_t cb = (c >> (2 * b)) & 3u;
          if (cb == 0u) continue;
          if (cb == 3u) {  // general dyadic coefficient: s + u*x
            const T ut = (T)coef_all[nd.coef_off + b * R + rlist[o]];
#pragma unroll
            for (int e = 0; e < VEC; ++e)
              acc.v[e] = started ? add_rn<T>(acc.v[e], mul_rn<T>(ut, x[h][b].v[e])) : mul_rn<T>(ut, x[h][b].v[e]);
          } else if (cb == 1u) {
#pragma unroll
            for (int e = 0; e < VEC; ++e) acc.v[e] = started ? add_rn<T>(acc.v[e], x[h][b].v[e]) : x[h][b].v[e];
          } else {
#pragma unroll
            for (int e = 0; e < VEC; ++e) acc.v[e] = started ? add_rn<T>(acc.v[e], -x[h][b].v[e]) : -x[h][b].v[e];
          }
          started = true;
        }
        if (!started) {
#pragma unroll
          for (int e = 0; e < VEC; ++e) acc.v[e] = (T)0;
        }
        st_vec<T, VEC>(optr[o] + i * old[o] + jv, acc);
      }
    }
  }
}

// One term of a sequential linear combination s = u_0 x_0 (+ u_1 x_1 ...) in K1's order: code
// cb (1 +1, 2 -1, 3 general dyadic coefficient *u); the first term initialises.
template <typename T, int VEC>
__device__ __forceinline__ void lc_term(Vec<T, VEC>& acc, bool& started, uint32_t cb,
                                        const Vec<T, VEC>& x, const double* u) {
  if (cb == 0u) return;
  if (cb == 3u) {
    const T ut = (T)*u;
#pragma unroll
    for (int e = 0; e < VEC; ++e)
      acc.v[e] = started ? add_rn<T>(acc.v[e], mul_rn<T>(ut, x.v[e])) : mul_rn<T>(ut, x.v[e]);
  } else if (cb == 1u) {
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc.v[e] = started ? add_rn<T>(acc.v[e], x.v[e]) : x.v[e];
  } else {
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc.v[e] = started ? add_rn<T>(acc.v[e], -x.v[e]) : -x.v[e];
  }
  started = true;
}

constexpr int kThreadsX2 = 128;

// Compile-time output structure of a K1X2 rule pair (RA at level d, RB at level d+1, table TV).
template <int RA, int RB, int TV>
struct X2Pair {
  static constexpr int R1 = builtin_R(RA), R2 = builtin_R(RB);
  static constexpr bool formed(int r1, int r2) {
    return !(builtin_trivial(RA, TV, r1) && builtin_trivial(RB, TV, r2));
  }
  static constexpr bool need2(int r1, int b2) {  // S_{r1}[b2] used by a formed output
    for (int r2 = 0; r2 < R2; ++r2)
      if (formed(r1, r2) && builtin_coef(RB, TV, b2, r2) != 0) return true;
    return false;
  }
  static constexpr bool need(int b1, int b2) {  // input sub-block (b1, b2) read
    for (int r1 = 0; r1 < R1; ++r1)
      if (builtin_coef(RA, TV, b1, r1) != 0 && need2(r1, b2)) return true;
    return false;
  }
  static constexpr int nout() {
    int n = 0;
    for (int r1 = 0; r1 < R1; ++r1)
      for (int r2 = 0; r2 < R2; ++r2) n += formed(r1, r2);
    return n;
  }
  static constexpr uint32_t code(int id, int b, int r) {
    return builtin_coef(id, TV, b, r) == 1 ? 1u : builtin_coef(id, TV, b, r) == -1 ? 2u : 0u;
  }
  static constexpr bool first(int id, int b, int r) {  // first nonzero term of column r
    for (int q = 0; q < b; ++q)
      if (builtin_coef(id, TV, q, r) != 0) return false;
    return true;
  }
  static constexpr int oidx(int r1, int r2) {  // position in the r1-major list of formed outputs
    int n = 0;
    for (int a = 0; a < R1; ++a)
      for (int c = 0; c < R2; ++c) {
        if (a == r1 && c == r2) return n;
        n += formed(a, c);
      }
    return n;
  }
};

// Compile-time loop: f(std::integral_constant<int, 0>) ... f(integral_constant<int, N-1>), so
// the K1X2 structure predicates below are constant expressions (if constexpr), not run-time
// table lookups.
template <typename F, int... I>
__device__ __forceinline__ void static_for_impl(F&& f, std::integer_sequence<int, I...>) {
  (f(std::integral_constant<int, I>{}), ...);
}
template <int N, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  static_for_impl(f, std::make_integer_sequence<int, N>{});
}

// One term s (+)= u x of a sequential sum with a compile-time code (1: +1, 2: -1).
template <uint32_t CB, typename T, int VEC>
__device__ __forceinline__ void lc_fixed(Vec<T, VEC>& acc, bool first, const Vec<T, VEC>& x) {
#pragma unroll
  for (int e = 0; e < VEC; ++e) {
    const T v = CB == 1u ? x.v[e] : -x.v[e];
    acc.v[e] = first ? v : add_rn<T>(acc.v[e], v);
  }
}

// One grandchild row position of a K1X2 node: load the needed input elements once, then per r1
// form S_{r1}[i2] (level d) and every formed S_{r1 r2} (level d+1) from them, ascending
// block order in both sums (the one-level K1's order).  All codes are constants, so the body is
// only the loads, the adds and the stores.
template <typename T, int VEC, int RA, int RB, int TV>
__device__ __forceinline__ void k1x2_row(const T* __restrict__ in, int64_t ldi, int64_t rows,
                                         int64_t cols, int64_t i, int64_t jv, T* const* optr) {
  using X = X2Pair<RA, RB, TV>;
  Vec<T, VEC> x[4][4];  // x[i2][i1]
  static_for<4>([&](auto b1) {
    static_for<4>([&](auto b2) {
      if constexpr (X::need(b1, b2)) {
        constexpr int p1 = b1 % 2, q1 = b1 / 2, p2 = b2 % 2, q2 = b2 / 2;
        x[b2][b1] = ld_vec<T, VEC>(in + ((2 * p1 + p2) * rows + i) * ldi + (2 * q1 + q2) * cols + jv);
      }
    });
  });
  const int64_t off = i * cols + jv;
  static_for<X::R1>([&](auto r1) {
    Vec<T, VEC> y[4];
    static_for<4>([&](auto b2) {
      if constexpr (X::need2(r1, b2)) {
        static_for<4>([&](auto b1) {
          if constexpr (X::code(RA, b1, r1) != 0u)
            lc_fixed<X::code(RA, b1, r1)>(y[b2], X::first(RA, b1, r1), x[b2][b1]);
        });
      }
    });
    static_for<X::R2>([&](auto r2) {
      if constexpr (X::formed(r1, r2)) {
        Vec<T, VEC> acc;
        static_for<4>([&](auto b2) {
          if constexpr (X::code(RB, b2, r2) != 0u)
            lc_fixed<X::code(RB, b2, r2)>(acc, X::first(RB, b2, r2), y[b2]);
        });
        st_vec<T, VEC>(optr[X::oidx(r1, r2)] + off, acc);
      }
    });
  });
}

// K1X2 launch: grid x = column chunks of kThreadsX2 vectors, y = row groups of RPB grandchild
// rows, z = node (S nodes use the U tables, T nodes the V tables).
template <typename T, int VEC, int RPB, int RA, int RB>
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
    if (tv) k1x2_row<T, VEC, RA, RB, 1>(in, ldi, rows, cols, i, jv, optr);
    else k1x2_row<T, VEC, RA, RB, 0>(in, ldi, rows, cols, i, jv, optr);
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

// Compile-time structure of a K3X2 rule pair (RA at level d, RB at level d+1).
template <int RA, int RB>
struct W2Pair {
  static constexpr int R1 = builtin_R(RA), R2 = builtin_R(RB);
  static constexpr uint32_t code(int id, int k, int r) {
    return builtin_w(id, k, r) == 1 ? 1u : builtin_w(id, k, r) == -1 ? 2u : 0u;
  }
  static constexpr bool first(int id, int k, int r) {  // first nonzero term of row k
    for (int q = 0; q < r; ++q)
      if (builtin_w(id, k, q) != 0) return false;
    return true;
  }
  static constexpr bool used(int id, int r) {
    for (int k = 0; k < 4; ++k)
      if (builtin_w(id, k, r) != 0) return true;
    return false;
  }
};

// One grandchild row position of a K3X2 node: per r1 (ascending) form C_{r1}[k2] from the
// M_{r1 r2} (level d+1, ascending r2) and accumulate w1_{k1 r1} C_{r1}[k2] into the 16 outputs
// (level d); then store them.
template <typename T, int VEC, int RA, int RB>
__device__ __forceinline__ void k3x2_row(const T* const* iptr, T* __restrict__ out, int64_t ldo,
                                         int64_t rows, int64_t cols, int64_t i, int64_t jv) {
  using X = W2Pair<RA, RB>;
  const int64_t off = i * cols + jv;
  Vec<T, VEC> acc[4][4];  // [k1][k2]
  static_for<X::R1>([&](auto r1) {
    if constexpr (X::used(RA, r1)) {
      Vec<T, VEC> y[4];
      static_for<X::R2>([&](auto r2) {
        if constexpr (X::used(RB, r2)) {
          const Vec<T, VEC> m = ld_vec<T, VEC>(iptr[r1 * X::R2 + r2] + off);
          static_for<4>([&](auto k2) {
            if constexpr (X::code(RB, k2, r2) != 0u)
              lc_fixed<X::code(RB, k2, r2)>(y[k2], X::first(RB, k2, r2), m);
          });
        }
      });
      static_for<4>([&](auto k1) {
        if constexpr (X::code(RA, k1, r1) != 0u) {
          static_for<4>([&](auto k2) {
            lc_fixed<X::code(RA, k1, r1)>(acc[k1][k2], X::first(RA, k1, r1), y[k2]);
          });
        }
      });
    }
  });
  static_for<4>([&](auto k1) {
    static_for<4>([&](auto k2) {
      constexpr int ia = 2 * (k1 / 2) + k2 / 2, jb = 2 * (k1 % 2) + k2 % 2;
      st_vec<T, VEC>(out + (ia * rows + i) * ldo + jb * cols + jv, acc[k1][k2]);
    });
  });
}

// K3X2 launch: grid x = column chunks of kThreadsX2 vectors, y = row groups of RPB, z = node.
template <typename T, int VEC, int RPB, int RA, int RB>
__global__ void __launch_bounds__(kThreadsX2) k3x2_combine(const K3x2Node* __restrict__ nodes,
                                                            Bases bases) {
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
    k3x2_row<T, VEC, RA, RB>(iptr, out, ldo, rows, cols, i, jv);
  }
}

template <typename T, int VEC, int RA, int RB, int RPB>
void k3x2_go_rpb(const Step& s, const K3x2Node* nd, const Bases& b, cudaStream_t st) {
  const int64_t cv = (s.cols + VEC - 1) / VEC;
  dim3 grid((unsigned)((cv + kThreadsX2 - 1) / kThreadsX2), (unsigned)((s.rows + RPB - 1) / RPB),
            (unsigned)s.count);
  k3x2_combine<T, VEC, RPB, RA, RB><<<grid, kThreadsX2, 0, st>>>(nd, b);
}

template <typename T, int VEC, int RA, int RB>
void k3x2_go(const Step& s, const K3x2Node* nd, const Bases& b, cudaStream_t st) {
  if (k3x2_rpb() == 4) k3x2_go_rpb<T, VEC, RA, RB, 4>(s, nd, b, st);
  else k3x2_go_rpb<T, VEC, RA, RB, 1>(s, nd, b, st);
}

template <typename T, int VEC>
void k3x2_pick(const Step& s, const K3x2Node* nd, const Bases& b, cudaStream_t st) {
  switch (s.x2 - 1) {
    case 0: k3x2_go<T, VEC, 0, 0>(s, nd, b, st); break;
    case 1: k3x2_go<T, VEC, 0, 1>(s, nd, b, st); break;
    case 2: k3x2_go<T, VEC, 0, 2>(s, nd, b, st); break;
    case 3: k3x2_go<T, VEC, 1, 0>(s, nd, b, st); break;
    case 4: k3x2_go<T, VEC, 1, 1>(s, nd, b, st); break;
    case 5: k3x2_go<T, VEC, 1, 2>(s, nd, b, st); break;
    case 6: k3x2_go<T, VEC, 2, 0>(s, nd, b, st); break;
    case 7: k3x2_go<T, VEC, 2, 1>(s, nd, b, st); break;
    default: k3x2_go<T, VEC, 2, 2>(s, nd, b, st); break;
  }
}

// K3: node output (P*rows x Q*cols) with P = M0, Q = N0; k = ia*Q + jb (row-major).
template <typename T, int VEC, int MAXR>
__global__ void __launch_bounds__(kThreads) k3_combine(const K3Node* __restrict__ nodes,
                                                       const double* __restrict__ coef_all,
                                                       Bases bases, int64_t rows, int64_t cols,
                                                       int P, int Q, int R) {
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

template <typename T>
cudaError_t launch_k1(const Step& s, const void* dev_nodes, const double* dev_coef,
                      const Bases& b, bool vec, cudaStream_t st, const ScaleIn* sc) {
  if (s.count == 0 || s.rows == 0 || s.cols == 0) return cudaSuccess;
  constexpr int V = 16 / sizeof(T);
  if (sc && s.scaled && !s.x2) {  // the root under virtual scaling (FP64 plans only)
    const K1Node* nd = (const K1Node*)dev_nodes;
    if (s.P * s.Q <= 4) {
      if (vec) k1_go<T, V, 4, 4, 2, true>(s, nd, dev_coef, b, st, *sc);
      else k1_go<T, 1, 4, 4, 2, true>(s, nd, dev_coef, b, st, *sc);
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
                      const Bases& b, bool vec, cudaStream_t st) {
  if (s.count == 0 || s.rows == 0 || s.cols == 0) return cudaSuccess;
  constexpr int V = 16 / sizeof(T);
  if (s.x2) {
    if (vec) k3x2_pick<T, V>(s, (const K3x2Node*)dev_nodes, b, st);
    else k3x2_pick<T, 1>(s, (const K3x2Node*)dev_nodes, b, st);
    return cudaGetLastError();
  }
  const K3Node* nd = (const K3Node*)dev_nodes;
  if (s.R <= 8) {
    if (vec)
      k3_combine<T, V, 8><<<grid_for(s, V), kThreads, 0, st>>>(nd, dev_coef, b, s.rows, s.cols, s.P, s.Q, s.R);
    else
      k3_combine<T, 1, 8><<<grid_for(s, 1), kThreads, 0, st>>>(nd, dev_coef, b, s.rows, s.cols, s.P, s.Q, s.R);
  } else {
    if (vec)
      k3_combine<T, V, kMaxR><<<grid_for(s, V), kThreads, 0, st>>>(nd, dev_coef, b, s.rows, s.cols, s.P, s.Q, s.R);
    else
      k3_combine<T, 1, kMaxR><<<grid_for(s, 1), kThreads, 0, st>>>(nd, dev_coef, b, s.rows, s.cols, s.P, s.Q, s.R);
  }
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
template cudaError_t launch_k3<double>(const Step&, const void*, const double*, const Bases&, bool, cudaStream_t);
template cudaError_t launch_k3<float>(const Step&, const void*, const double*, const Bases&, bool, cudaStream_t);
template cudaError_t launch_acc<double>(const Step&, const void*, const double*, const Bases&, bool, cudaStream_t);
template cudaError_t launch_acc<float>(const Step&, const void*, const double*, const Bases&, bool, cudaStream_t);
template cudaError_t launch_zero<double>(const Step&, const void*, const Bases&, cudaStream_t);
template cudaError_t launch_zero<float>(const Step&, const void*, const Bases&, cudaStream_t);

}  // namespace fmm
