// Device-side building blocks of the HBM-streaming passes (K1 / K1X2 / K3X2), shared by
// kernels_lincomb.cu (one launch per pass) and kernels_small.cu (the single-launch small-plan
// kernel).  Included inside no namespace; everything lives in fmm::{anonymous}.
#pragma once
#include <cstdint>
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

// CG: an L2-only load (ld.global.cg) -- for data written earlier in the same kernel by other
// SMs (the single-launch small plan), which a non-coherent L1 line must not serve
template <typename T, int VEC, bool CG = false>
__device__ __forceinline__ Vec<T, VEC> ld_vec(const T* p) {
  Vec<T, VEC> r;
  if constexpr (CG) {
    if constexpr (VEC * sizeof(T) == 16 && sizeof(T) == 8) {
      const double2 x = __ldcg(reinterpret_cast<const double2*>(p));
      r.v[0] = x.x;
      r.v[1] = x.y;
    } else {
#pragma unroll
      for (int e = 0; e < VEC; ++e) r.v[e] = __ldcg(p + e);
    }
    return r;
  }
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
__device__ __noinline__ double scale2_wide(double x, int e) { return ldexp(x, e); }
__device__ __forceinline__ double scale2(double x, int e) {
  if (e == 0) return x;
  if (e >= -1022 && e <= 1023) return __dmul_rn(x, __longlong_as_double((int64_t)(e + 1023) << 52));
  return scale2_wide(x, e);
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
  bool vscale = false, fast = false;
  const int32_t* ers = nullptr;
  int ecv[NBLK][VEC];
  double fcv[NBLK][VEC];
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
      // fast path: every exponent and every row + column sum a normal power of two (the
      // scaling run's extremes), so x 2^(er + ec) = x * (2^er * 2^ec), one rounding
      const int* ex = sc.ext + 4 * side;  // min / max of er, min / max of ec
      fast = ex[0] >= -1022 && ex[1] <= 1023 && ex[2] >= -1022 && ex[3] <= 1023 &&
             ex[0] + ex[2] >= -1022 && ex[1] + ex[3] <= 1023;
#pragma unroll
      for (int b = 0; b < NBLK; ++b)
#pragma unroll
        for (int e = 0; e < VEC; ++e)
          fcv[b][e] = fast ? __longlong_as_double((int64_t)(ecv[b][e] + 1023) << 52) : 1.0;
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
        }
      }
    }
    if constexpr (SC) {  // all loads issued above; now apply the exponents
      if (vscale) {
#pragma unroll
        for (int h = 0; h < RIF; ++h) {
          const int64_t i = i0 + ii + h;
          if (i >= rows) break;
#pragma unroll
          for (int b = 0; b < NBLK; ++b) {
            if (b < nblk && ((need >> b) & 1u)) {
              const int erp = ers[(b % P) * rows + i];
              if (fast) {
                const double fr = __longlong_as_double((int64_t)(erp + 1023) << 52);
#pragma unroll
                for (int e = 0; e < VEC; ++e) x[h][b].v[e] = (T)__dmul_rn((double)x[h][b].v[e], __dmul_rn(fr, fcv[b][e]));
              } else {
#pragma unroll
                for (int e = 0; e < VEC; ++e) x[h][b].v[e] = (T)scale2((double)x[h][b].v[e], erp + ecv[b][e]);
              }
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
// SPLIT: every (r1, r2) is formed (the tensor-core FP32 leaves' operand arena holds views too).
template <int RA, int RB, int TV, bool SPLIT = false>
struct X2Pair {
  static constexpr int R1 = builtin_R(RA), R2 = builtin_R(RB);
  static constexpr bool formed(int r1, int r2) {
    return SPLIT || !(builtin_trivial(RA, TV, r1) && builtin_trivial(RB, TV, r2));
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
// SPLIT (FP32 only): each output is written as its TF32 hi / lo pair (tf32_split), hi at
// optr[idx] and lo lo_off elements further -- the leaf GEMM's operand arena.
template <typename T, int VEC, int RA, int RB, int TV, bool SPLIT = false>
__device__ __forceinline__ void k1x2_row(const T* __restrict__ in, int64_t ldi, int64_t rows,
                                         int64_t cols, int64_t i, int64_t jv, T* const* optr,
                                         int64_t lo_off = 0) {
  using X = X2Pair<RA, RB, TV, SPLIT>;
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
        if constexpr (SPLIT) {
          static_assert(sizeof(T) == 4, "the TF32 split is FP32-only");
          Vec<T, VEC> hi, lo;
#pragma unroll
          for (int e = 0; e < VEC; ++e) tf32_split(acc.v[e], hi.v[e], lo.v[e]);
          st_vec<T, VEC>(optr[X::oidx(r1, r2)] + off, hi);
          st_vec<T, VEC>(optr[X::oidx(r1, r2)] + lo_off + off, lo);
        } else {
          st_vec<T, VEC>(optr[X::oidx(r1, r2)] + off, acc);
        }
      }
    });
  });
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
template <typename T, int VEC, int RA, int RB, bool US = false, bool CG = false>
__device__ __forceinline__ void k3x2_row(const T* const* iptr, T* __restrict__ out, int64_t ldo,
                                         int64_t rows, int64_t cols, int64_t i, int64_t jv,
                                         const double* ur = nullptr, const double* uc = nullptr) {
  using X = W2Pair<RA, RB>;
  const int64_t off = i * cols + jv;
  Vec<T, VEC> acc[4][4];  // [k1][k2]
  static_for<X::R1>([&](auto r1) {
    if constexpr (X::used(RA, r1)) {
      Vec<T, VEC> y[4];
      static_for<X::R2>([&](auto r2) {
        if constexpr (X::used(RB, r2)) {
          const Vec<T, VEC> m = ld_vec<T, VEC, CG>(iptr[r1 * X::R2 + r2] + off);
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
      if constexpr (US) {  // the unscale C = (d_A,i C'_ij) d_B,j folded in (reading A9)
        const double a = ur[ia * rows + i];
#pragma unroll
        for (int e = 0; e < VEC; ++e)
          acc[k1][k2].v[e] = (T)__dmul_rn(__dmul_rn(a, (double)acc[k1][k2].v[e]), uc[jb * cols + jv + e]);
      }
      st_vec<T, VEC>(out + (ia * rows + i) * ldo + jb * cols + jv, acc[k1][k2]);
    });
  });
}

}  // namespace
}  // namespace fmm
