// K4: diagonal scaling (Section 6, Alg. 1-3) on device, FP64.
//
// One scaling step = one tiny factor kernel + one streaming pass per matrix.  The streaming
// pass applies the step's factors (a / r'_i, a * p_k, b / s'_j, b / p_k -- true divisions,
// DESIGN.md reading A9) and, in the same read, accumulates the row and column max-abs of the
// RESULT, which are exactly the reductions the next step needs; so every step reads and writes
// each matrix once.  Max-abs is combined across CTAs with atomicMax on the IEEE bit pattern
// (non-negative doubles order like their bit patterns): exact and order-free.
// The stopping test of Thm stopping-criterion, from the step after the first O
// step, runs on device; once it fires, later steps' passes exit immediately, so the
// host never synchronises inside Alg. 3.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <utility>

#include "fmm_internal.h"

namespace fmm {

// flags layout (int32): [0] done, [1] steps taken, [2] error kind (0 none; 1 zero row of A,
// 2 zero col of B, 3 zero col of A, 4 zero row of B), [3] error index, [4] skip current step
// [5] inexact: some factor of the current step has no exactly representable power-of-two
// reciprocal (the multiply pass then yields to the dividing pass)
// [8] mode of the one-kernel run (0 virtual, 1 materialised), [9] bad (the virtual form cannot
// reproduce the sequential roundings: switch to materialised), [10], [11] stop-test failure
// counters of even / odd steps, [12] A' / B' are stored in the materialised buffers
enum { F_DONE = 0, F_STEPS = 1, F_ERR = 2, F_ERRIDX = 3, F_SKIP = 4, F_INEXACT = 5, F_MODE = 8,
       F_BAD = 9, F_FAIL = 10, F_STORED = 12, F_COUNT = 16 };
enum ApplyMode { AP_NONE = 0, AP_ROW_DIV = 1, AP_COL_DIV = 2, AP_COL_MUL = 3 };

namespace {

__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

// Nearest power of two in log2 (reading A8): x = m 2^e, m in [0.5, 1);
// round down to 2^(e-1) iff m*m < 1/2, decided exactly with an error-free square.
__device__ __forceinline__ double pow2_round(double x) {
  int e;
  double m = frexp(x, &e);
  double h = __dmul_rn(m, m);
  double l = fma(m, m, -h);
  bool below = (h < 0.5) || (h == 0.5 && l < 0.0);
  return ldexp(1.0, below ? e - 1 : e);
}

constexpr int TX = 32, TY = 8;
constexpr int CPL = 4;         // columns per lane (two 16-byte accesses)
constexpr int TC = TX * CPL;   // 128-column strips
constexpr int RU = 2;          // rows in flight per warp

// x / f, correctly rounded.  When f is an exact power of two whose reciprocal is a normal
// double (pow2 factors, reading A7), x * (1/f) is the same real number rounded
// once, i.e. bitwise x / f, and avoids the FP64 division sequence.
struct Divisor {
  double f, inv;
  bool pow2;
  __device__ __forceinline__ explicit Divisor(double v) : f(v) {
    const int64_t bits = __double_as_longlong(v);
    const int ex = (int)((bits >> 52) & 0x7ff);
    pow2 = (bits & 0x000fffffffffffffLL) == 0 && ex >= 2 && ex <= 2045 && v > 0.0;
    inv = pow2 ? __longlong_as_double((int64_t)(2046 - ex) << 52) : 0.0;
  }
  __device__ __forceinline__ Divisor() : f(1.0), inv(1.0), pow2(true) {}
  __device__ __forceinline__ double div(double x) const { return pow2 ? __dmul_rn(x, inv) : __ddiv_rn(x, f); }
};

// dst = apply(src); row_max[i] = max_j |dst_ij|, col_max[j] = max_i |dst_ij| (atomic).
// dst may equal src (in place) or be null (reduce only).  Block (x, y) owns the 128-column strip
// x and the row chunk y; warp w handles rows w, w + TY, ... of the chunk, RU rows at a time
// (their loads issued together), lane l owns columns 2l, 2l+1 and 64+2l, 64+2l+1 (16-byte
// accesses when VEC, each warp instruction covering 512 contiguous bytes).  Column maxima stay
// in registers over the whole chunk: one shared-memory combine and one atomic per column per
// block at the end, no block barrier inside the stream.
template <int MODE, bool VEC>
__global__ void __launch_bounds__(TX* TY, 4)
    k_apply_reduce(const double* src, int64_t lds, double* dst, int64_t ldd,
                   int64_t rows, int64_t cols, int64_t chunk, const double* __restrict__ f,
                   double* __restrict__ row_max, double* __restrict__ col_max,
                   const int* __restrict__ flags, int only_if_inexact) {
  if (flags && (flags[F_SKIP] || (only_if_inexact && !flags[F_INEXACT]))) return;
  __shared__ double cm[TY][TC];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t cbase = (int64_t)blockIdx.x * TC + 2 * tx;
  const int64_t rbeg = (int64_t)blockIdx.y * chunk;
  const int64_t rend = rbeg + chunk < rows ? rbeg + chunk : rows;
  int64_t cidx[CPL];
  bool ok[CPL];
#pragma unroll
  for (int e = 0; e < CPL; ++e) {
    cidx[e] = cbase + (e / 2) * (2 * TX) + (e & 1);
    ok[e] = cidx[e] < cols;
  }
  Divisor fcol[CPL];
  double mcol[CPL];
#pragma unroll
  for (int e = 0; e < CPL; ++e) {
    mcol[e] = 1.0;
    if (MODE == AP_COL_DIV || MODE == AP_COL_MUL) {
      const double v = ok[e] ? f[cidx[e]] : 1.0;
      if (MODE == AP_COL_DIV) fcol[e] = Divisor(v);
      else mcol[e] = v;
    }
  }
  double cmax[CPL];
#pragma unroll
  for (int e = 0; e < CPL; ++e) cmax[e] = 0.0;
#pragma unroll 1
  for (int64_t rb = rbeg + ty; rb < rend; rb += TY * RU) {
    double x[RU][CPL];
    double frow[RU];
#pragma unroll
    for (int u = 0; u < RU; ++u) {
      const int64_t r = rb + u * TY;
#pragma unroll
      for (int e = 0; e < CPL; ++e) x[u][e] = 0.0;
      frow[u] = 1.0;
      if (r < rend) {
        if (MODE == AP_ROW_DIV) frow[u] = f[r];  // issued with the row's data loads
        const double* sp = src + r * lds;
#pragma unroll
        for (int h = 0; h < CPL / 2; ++h) {
          const int64_t c0 = cidx[2 * h];
          if (VEC && ok[2 * h + 1]) {
            const double2 v = *reinterpret_cast<const double2*>(sp + c0);
            x[u][2 * h] = v.x; x[u][2 * h + 1] = v.y;
          } else {
            if (ok[2 * h]) x[u][2 * h] = sp[c0];
            if (ok[2 * h + 1]) x[u][2 * h + 1] = sp[c0 + 1];
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < RU; ++u) {
      const int64_t r = rb + u * TY;
      if (r >= rend) continue;  // warp-uniform
      Divisor fr;
      if (MODE == AP_ROW_DIV) fr = Divisor(frow[u]);
      double rmax = 0.0;
#pragma unroll
      for (int e = 0; e < CPL; ++e) {
        double y = x[u][e];
        if (MODE == AP_ROW_DIV) y = fr.div(y);
        else if (MODE == AP_COL_DIV) y = fcol[e].div(y);
        else if (MODE == AP_COL_MUL) y = __dmul_rn(y, mcol[e]);
        x[u][e] = y;
        const double v = ok[e] ? fabs(y) : 0.0;
        rmax = fmax(rmax, v);
        cmax[e] = fmax(cmax[e], v);
      }
      if (dst) {
        double* dp = dst + r * ldd;
#pragma unroll
        for (int h = 0; h < CPL / 2; ++h) {
          const int64_t c0 = cidx[2 * h];
          if (VEC && ok[2 * h + 1]) {
            *reinterpret_cast<double2*>(dp + c0) = make_double2(x[u][2 * h], x[u][2 * h + 1]);
          } else {
            if (ok[2 * h]) dp[c0] = x[u][2 * h];
            if (ok[2 * h + 1]) dp[c0 + 1] = x[u][2 * h + 1];
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
      if (tx == 0 && row_max) atomic_max_nonneg(&row_max[r], rmax);
    }
  }
  if (col_max) {
#pragma unroll
    for (int e = 0; e < CPL; ++e) cm[ty][(e / 2) * (2 * TX) + 2 * tx + (e & 1)] = cmax[e];
    __syncthreads();
    for (int q = ty * TX + tx; q < TC; q += TX * TY) {
      double mx = 0.0;
#pragma unroll
      for (int y = 0; y < TY; ++y) mx = fmax(mx, cm[y][q]);
      const int64_t cc = (int64_t)blockIdx.x * TC + q;
      if (cc < cols) atomic_max_nonneg(&col_max[cc], mx);
    }
  }
}

// Multiply-only pass for power-of-two factors (pow2 = 1): the factor kernels store the exact
// reciprocals 1/r, 1/s, 1/p (a power of two's reciprocal is a power of two, exact whenever it
// is representable), so x / f = x * (1/f) bitwise and every apply is one multiplication.
// MODE: AP_NONE (reduce only), AP_ROW_MUL (x * g_i), AP_COL_MUL (x * g_j).  Same block / warp
// layout as k_apply_reduce with 8 columns per lane (256-column strips): half the per-element
// cost of the row-max shuffles, 8 16-byte loads in flight per lane.  `need_exact`: return
// unless every factor of this step had an exact reciprocal (flags[F_INEXACT] == 0).
constexpr int CPL8 = 8, TC8 = TX * CPL8, RU8 = 2;
enum { AP_ROW_MUL = 4 };

template <int MODE>
constexpr int mul_blocks_per_sm() { return MODE == AP_COL_MUL ? 2 : 3; }  // COL: 8 more factor registers

template <int MODE, bool VEC>
__global__ void __launch_bounds__(TX* TY, mul_blocks_per_sm<MODE>())
    k_apply_reduce_mul(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows,
                       int64_t cols, int64_t chunk, const double* __restrict__ g,
                       double* __restrict__ row_max, double* __restrict__ col_max,
                       const int* __restrict__ flags, int need_exact) {
  if (flags && (flags[F_SKIP] || (need_exact && flags[F_INEXACT]))) return;
  __shared__ double cm[TY][TC8];
  const int tx = threadIdx.x, ty = threadIdx.y;
  // lane columns: cbase + off(e), off(e) = (e / 2) * 64 + (e & 1); valid iff off(e) < lim
  const int64_t cbase = (int64_t)blockIdx.x * TC8 + 2 * tx;
  const int64_t lim = cols - cbase;
  const int64_t rbeg = (int64_t)blockIdx.y * chunk;
  const int64_t rend = rbeg + chunk < rows ? rbeg + chunk : rows;
  const bool full = lim >= (CPL8 / 2 - 1) * 2 * TX + 2;  // every lane column valid
  double gc[CPL8], cmax[CPL8];
#pragma unroll
  for (int e = 0; e < CPL8; ++e) {
    const int off = (e / 2) * (2 * TX) + (e & 1);
    gc[e] = (MODE == AP_COL_MUL && off < lim) ? g[cbase + off] : 1.0;
    cmax[e] = 0.0;
  }
#pragma unroll 1
  for (int64_t rb = rbeg + ty; rb < rend; rb += TY * RU8) {
    double x[RU8][CPL8];
    double gr[RU8];
#pragma unroll
    for (int u = 0; u < RU8; ++u) {
      const int64_t r = rb + u * TY;
      gr[u] = 1.0;
#pragma unroll
      for (int e = 0; e < CPL8; ++e) x[u][e] = 0.0;
      if (r < rend) {
        if (MODE == AP_ROW_MUL) gr[u] = g[r];
        const double* sp = src + r * lds + cbase;
#pragma unroll
        for (int h = 0; h < CPL8 / 2; ++h) {
          const int off = h * (2 * TX);
          if (VEC && (full || off + 1 < lim)) {
            const double2 v = *reinterpret_cast<const double2*>(sp + off);
            x[u][2 * h] = v.x; x[u][2 * h + 1] = v.y;
          } else {
            if (off < lim) x[u][2 * h] = sp[off];
            if (off + 1 < lim) x[u][2 * h + 1] = sp[off + 1];
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < RU8; ++u) {
      const int64_t r = rb + u * TY;
      if (r >= rend) continue;  // warp-uniform
      double rmax = 0.0;
#pragma unroll
      for (int e = 0; e < CPL8; ++e) {
        const int off = (e / 2) * (2 * TX) + (e & 1);
        double y = x[u][e];
        if (MODE == AP_ROW_MUL) y = __dmul_rn(y, gr[u]);
        else if (MODE == AP_COL_MUL) y = __dmul_rn(y, gc[e]);
        x[u][e] = y;
        const double v = (full || off < lim) ? fabs(y) : 0.0;
        rmax = fmax(rmax, v);
        cmax[e] = fmax(cmax[e], v);
      }
      if (dst) {
        double* dp = dst + r * ldd + cbase;
#pragma unroll
        for (int h = 0; h < CPL8 / 2; ++h) {
          const int off = h * (2 * TX);
          if (VEC && (full || off + 1 < lim)) {
            *reinterpret_cast<double2*>(dp + off) = make_double2(x[u][2 * h], x[u][2 * h + 1]);
          } else {
            if (off < lim) dp[off] = x[u][2 * h];
            if (off + 1 < lim) dp[off + 1] = x[u][2 * h + 1];
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
      if (tx == 0 && row_max) atomic_max_nonneg(&row_max[r], rmax);
    }
  }
  if (col_max) {
#pragma unroll
    for (int e = 0; e < CPL8; ++e) cm[ty][(e / 2) * (2 * TX) + 2 * tx + (e & 1)] = cmax[e];
    __syncthreads();
    for (int q = ty * TX + tx; q < TC8; q += TX * TY) {
      double mx = 0.0;
#pragma unroll
      for (int y = 0; y < TY; ++y) mx = fmax(mx, cm[y][q]);
      const int64_t cc = (int64_t)blockIdx.x * TC8 + q;
      if (cc < cols) atomic_max_nonneg(&col_max[cc], mx);
    }
  }
}

// exact reciprocal of a power-of-two factor (false if f is not a power of two whose reciprocal
// is representable; then the dividing pass runs)
__device__ __forceinline__ bool exact_recip(double f, double* inv) {
  const int64_t bits = __double_as_longlong(f);
  const int ex = (int)((bits >> 52) & 0x7ff);
  if ((bits & 0x000fffffffffffffLL) != 0 || ex < 1 || ex > 2045 || !(f > 0.0)) return false;
  *inv = __longlong_as_double((int64_t)(2046 - ex) << 52);
  return true;
}

__device__ bool block_all(bool v) { return __syncthreads_and(v ? 1 : 0) != 0; }

// O step factors (Alg. 3): r'_i = rowmaxA_i, s'_j = colmaxB_j; dA_i *= r'_i;
// dB_j = s'_j * dB_j; stop test r', s' >= (1+tau)^(-1/2) when `test`.
__global__ void k_factor_O(const double* __restrict__ rmA, const double* __restrict__ cmB,
                           int64_t M, int64_t N, int pow2, double* dA, double* dB, double* r_out,
                           double* s_out, double* r_inv, double* s_inv, int* flags, int test,
                           double lo_O, double* next_zero, int64_t next_len) {
  const bool skip = flags[F_DONE] != 0;
  __syncthreads();
  if (threadIdx.x == 0) { flags[F_SKIP] = skip ? 1 : 0; flags[F_INEXACT] = 0; }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < next_len; i += blockDim.x) next_zero[i] = 0.0;
  if (skip) return;
  bool ok = true;
  for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
    double r = rmA[i];
    if (!(r > 0.0)) {
      if (atomicCAS(&flags[F_ERR], 0, 1) == 0) flags[F_ERRIDX] = (int)i;
      r = __longlong_as_double(0x7ff8000000000000LL);  // NaN propagates to C
    } else if (pow2) {
      r = pow2_round(r);
    }
    r_out[i] = r;
    if (pow2 && !exact_recip(r, &r_inv[i])) flags[F_INEXACT] = 1;
    dA[i] = __dmul_rn(dA[i], r);
    ok = ok && (r >= lo_O);
  }
  for (int64_t j = threadIdx.x; j < N; j += blockDim.x) {
    double s = cmB[j];
    if (!(s > 0.0)) {
      if (atomicCAS(&flags[F_ERR], 0, 2) == 0) flags[F_ERRIDX] = (int)j;
      s = __longlong_as_double(0x7ff8000000000000LL);
    } else if (pow2) {
      s = pow2_round(s);
    }
    s_out[j] = s;
    if (pow2 && !exact_recip(s, &s_inv[j])) flags[F_INEXACT] = 1;
    dB[j] = __dmul_rn(s, dB[j]);
    ok = ok && (s >= lo_O);
  }
  const bool all = block_all(ok);
  if (threadIdx.x == 0) {
    flags[F_STEPS] += 1;
    if (test && all) flags[F_DONE] = 1;
  }
}

// I step factor (Alg. 3): p_k = sqrt(rowmaxB_k / colmaxA_k); dI_k *= p_k;
// stop test p_k in [(1+tau)^(-1/4), (1+tau)^(1/4)] when `test`.
__global__ void k_factor_I(const double* __restrict__ cmA, const double* __restrict__ rmB,
                           int64_t K, int pow2, double* dI, double* p_out, double* p_inv,
                           int* flags, int test, double lo_I, double hi_I, double* next_zero,
                           int64_t next_len) {
  const bool skip = flags[F_DONE] != 0;
  __syncthreads();
  if (threadIdx.x == 0) { flags[F_SKIP] = skip ? 1 : 0; flags[F_INEXACT] = 0; }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < next_len; i += blockDim.x) next_zero[i] = 0.0;
  if (skip) return;
  bool ok = true;
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
    const double a = cmA[k], b = rmB[k];
    double p;
    if (!(a > 0.0) || !(b > 0.0)) {
      if (atomicCAS(&flags[F_ERR], 0, !(a > 0.0) ? 3 : 4) == 0) flags[F_ERRIDX] = (int)k;
      p = __longlong_as_double(0x7ff8000000000000LL);
    } else {
      p = __dsqrt_rn(__ddiv_rn(b, a));
      if (pow2) p = pow2_round(p);
    }
    p_out[k] = p;
    if (pow2 && !exact_recip(p, &p_inv[k])) flags[F_INEXACT] = 1;
    dI[k] = __dmul_rn(dI[k], p);
    ok = ok && (p >= lo_I && p <= hi_I);
  }
  const bool all = block_all(ok);
  if (threadIdx.x == 0) {
    flags[F_STEPS] += 1;
    if (test && all) flags[F_DONE] = 1;
  }
}

__global__ void k_fill(double* p, int64_t n, double v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// C_ij = (dA_i C'_ij) dB_j (reading A9); VEC: two columns per thread, 16-byte accesses
template <bool VEC>
__global__ void k_unscale(double* C, int64_t ldc, int64_t M, int64_t N, const double* dA,
                          const double* dB) {
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * (VEC ? 2 : 1);
  if (j >= N) return;
  const bool two = VEC && j + 1 < N;
  const double s0 = dB[j], s1 = two ? dB[j + 1] : 0.0;
  for (int64_t i = blockIdx.y; i < M; i += gridDim.y) {
    double* c = C + i * ldc + j;
    const double a = dA[i];
    if (two) {
      const double2 v = *reinterpret_cast<const double2*>(c);
      *reinterpret_cast<double2*>(c) = make_double2(__dmul_rn(__dmul_rn(a, v.x), s0), __dmul_rn(__dmul_rn(a, v.y), s1));
    } else {
      *c = __dmul_rn(__dmul_rn(a, *c), s0);
    }
  }
}

}  // namespace

// ---------------------------------------------------------------------------------------------
// Host-side driver of one scaling run (Alg. 1 / 2 / O->I / I->O / 3).  `sw` is a device scratch
// of scale_ws_bytes(M, K, N).  Writes A' / B' (A_out / B_out), dA, dB, dI and flags.
// ---------------------------------------------------------------------------------------------
size_t scale_ws_bytes(int64_t M, int64_t K, int64_t N) {
  // 2 sets of maxima (rowA M, colA K, rowB K, colB N) + factor vectors (r M, s N, p K) + flags
  // (16 doubles) + exact reciprocals (r M, s N, p K) of power-of-two factors + the net
  // exponents of the virtual form (int32: rowA M, colA K, rowB K, colB N)
  return (size_t)(2 * (M + K + K + N) + 2 * (M + N + K) + 16) * sizeof(double) +
         (size_t)(M + K + K + N) * sizeof(int32_t) + 256;
}

struct ScaleWsView {
  double* mx[2];  // each: rowA (M) | colA (K) | rowB (K) | colB (N)
  double *r, *s, *p;
  double *ri, *si, *pi;
  int* flags;
  int32_t* ex;    // rowA (M) | colA (K) | rowB (K) | colB (N)
};

static ScaleWsView scale_ws_view(void* ws, int64_t M, int64_t K, int64_t N) {
  ScaleWsView v;
  double* w = (double*)ws;
  const int64_t set = M + K + K + N;
  v.mx[0] = w;
  v.mx[1] = w + set;
  v.r = w + 2 * set;
  v.s = v.r + M;
  v.p = v.s + N;
  v.ri = v.p + K;
  v.si = v.ri + M;
  v.pi = v.si + N;
  v.flags = (int*)(v.pi + K);
  v.ex = (int32_t*)(v.pi + K + 16);
  return v;
}

int* scale_flags_ptr(void* ws, int64_t M, int64_t K, int64_t N) {
  return scale_ws_view(ws, M, K, N).flags;
}

static void grid_dims(int64_t rows, int64_t cols, int tc, int ru, int per_sm, dim3* g, int64_t* chunk) {
  // column strips x row chunks: one wave of per_sm resident blocks per SM, chunks a multiple
  // of TY * ru rows
  const int64_t strips = (cols + tc - 1) / tc;
  int64_t nchunks = std::max<int64_t>(1, (148 * per_sm) / strips);
  int64_t ch = (rows + nchunks - 1) / nchunks;
  ch = (ch + TY * ru - 1) / (TY * ru) * (TY * ru);
  nchunks = (rows + ch - 1) / ch;
  *g = dim3((unsigned)strips, (unsigned)nchunks);
  *chunk = ch;
}

// one streaming pass: dst = apply(src) with the row / column max-abs of the result.
// mode AP_ROW_DIV / AP_COL_DIV divide by f; with pow2 factors (finv != null) the multiply pass
// by the exact reciprocals runs instead, and the dividing pass only if some reciprocal was
// inexact (both check flags on device).
static void apply_reduce(cudaStream_t st, int mode, const double* src, int64_t lds, double* dst,
                         int64_t ldd, int64_t rows, int64_t cols, const double* f,
                         const double* finv, double* row_max, double* col_max, const int* flags) {
  if (rows == 0 || cols == 0) return;
  const bool vec = ((uintptr_t)src % 16 == 0) && lds % 2 == 0 &&
                   (!dst || (((uintptr_t)dst % 16 == 0) && ldd % 2 == 0));
  dim3 blk(TX, TY);
  dim3 g;
  int64_t chunk;
  const bool mul = mode == AP_NONE || mode == AP_COL_MUL || finv != nullptr;
  if (mul) {
    const int mm = mode == AP_ROW_DIV ? AP_ROW_MUL : mode == AP_COL_DIV ? AP_COL_MUL : mode;
    const double* gv = (mode == AP_ROW_DIV || mode == AP_COL_DIV) ? finv : f;
    const int need_exact = (mode == AP_ROW_DIV || mode == AP_COL_DIV) ? 1 : 0;
    grid_dims(rows, cols, TC8, RU8, mm == AP_COL_MUL ? 2 : 3, &g, &chunk);
#define FMM_ARM(M, V) k_apply_reduce_mul<M, V><<<g, blk, 0, st>>>(src, lds, dst, ldd, rows, cols, chunk, gv, row_max, col_max, flags, need_exact)
    switch (mm) {
      case AP_ROW_MUL: if (vec) FMM_ARM(AP_ROW_MUL, true); else FMM_ARM(AP_ROW_MUL, false); break;
      case AP_COL_MUL: if (vec) FMM_ARM(AP_COL_MUL, true); else FMM_ARM(AP_COL_MUL, false); break;
      default: if (vec) FMM_ARM(AP_NONE, true); else FMM_ARM(AP_NONE, false); break;
    }
#undef FMM_ARM
    if (!need_exact) return;
  }
  // dividing pass (pow2 = 0, or the fallback when a reciprocal was inexact)
  const int only_if_inexact = mul ? 1 : 0;
  grid_dims(rows, cols, TC, RU, 4, &g, &chunk);
#define FMM_AR(M, V) k_apply_reduce<M, V><<<g, blk, 0, st>>>(src, lds, dst, ldd, rows, cols, chunk, f, row_max, col_max, flags, only_if_inexact)
  switch (mode) {
    case AP_ROW_DIV: if (vec) FMM_AR(AP_ROW_DIV, true); else FMM_AR(AP_ROW_DIV, false); break;
    case AP_COL_DIV: if (vec) FMM_AR(AP_COL_DIV, true); else FMM_AR(AP_COL_DIV, false); break;
    default: break;
  }
#undef FMM_AR
}

// steps: sequence of 'O'/'I' (length nsteps); test_from: index from which the stop test runs
// (-1: never).  A_out / B_out may alias? no: they are distinct buffers (ws).
cudaError_t run_scaling(int64_t M, int64_t K, int64_t N, const double* A, int64_t lda,
                        const double* B, int64_t ldb, double* A_out, int64_t lda_out,
                        double* B_out, int64_t ldb_out, double* dA, double* dB, double* dI,
                        const char* steps, int nsteps, bool first_O, double tau, int pow2,
                        void* sws, cudaStream_t st) {
  ScaleWsView v = scale_ws_view(sws, M, K, N);
  const int64_t set = M + K + K + N;
  cudaError_t e;
  if ((e = cudaMemsetAsync(v.mx[0], 0, sizeof(double) * set, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(v.flags, 0, sizeof(int) * F_COUNT, st)) != cudaSuccess) return e;
  k_fill<<<64, 256, 0, st>>>(dA, M, 1.0);
  k_fill<<<64, 256, 0, st>>>(dB, N, 1.0);
  k_fill<<<64, 256, 0, st>>>(dI, K, 1.0);
  // initial reductions of A, B
  {
    double* m = v.mx[0];
    apply_reduce(st, AP_NONE, A, lda, nullptr, 0, M, K, nullptr, nullptr, m, m + M, nullptr);
    apply_reduce(st, AP_NONE, B, ldb, nullptr, 0, K, N, nullptr, nullptr, m + M + K, m + M + 2 * K, nullptr);
  }
  const double lo_I = pow(1.0 + tau, -0.25), hi_I = pow(1.0 + tau, 0.25), lo_O = pow(1.0 + tau, -0.5);
  int t0 = -1;
  for (int t = 0; t < nsteps; ++t) {
    const bool isO = steps[t] == 'O';
    if (isO && t0 < 0) t0 = t;
    const int test = (tau >= 0.0 && t0 >= 0 && t > t0) ? 1 : 0;
    double* cur = v.mx[t & 1];
    double* nxt = v.mx[(t + 1) & 1];
    const double* srcA = t == 0 ? A : A_out;
    const double* srcB = t == 0 ? B : B_out;
    const int64_t lsa = t == 0 ? lda : lda_out, lsb = t == 0 ? ldb : ldb_out;
    if (isO) {
      k_factor_O<<<1, 1024, 0, st>>>(cur, cur + M + 2 * K, M, N, pow2, dA, dB, v.r, v.s, v.ri, v.si, v.flags,
                                     test, lo_O, nxt, set);
      apply_reduce(st, AP_ROW_DIV, srcA, lsa, A_out, lda_out, M, K, v.r, pow2 ? v.ri : nullptr, nxt, nxt + M, v.flags);
      apply_reduce(st, AP_COL_DIV, srcB, lsb, B_out, ldb_out, K, N, v.s, pow2 ? v.si : nullptr, nxt + M + K,
                   nxt + M + 2 * K, v.flags);
    } else {
      k_factor_I<<<1, 1024, 0, st>>>(cur + M, cur + M + K, K, pow2, dI, v.p, v.pi, v.flags, test, lo_I,
                                     hi_I, nxt, set);
      apply_reduce(st, AP_COL_MUL, srcA, lsa, A_out, lda_out, M, K, v.p, nullptr, nxt, nxt + M, v.flags);
      apply_reduce(st, AP_ROW_DIV, srcB, lsb, B_out, ldb_out, K, N, v.p, pow2 ? v.pi : nullptr, nxt + M + K,
                   nxt + M + 2 * K, v.flags);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  (void)first_O;
  return cudaGetLastError();
}


// =============================================================================================
// Alg. 1-3 in ONE cooperative kernel.  All steps of a scaling run -- the max
// reductions, the factor computations with the stopping test, the applications -- run in one
// persistent launch with grid-wide barriers: no one-block factor kernels, no early-exiting
// steps enqueued by the host.
//
// Virtual form (power-of-two factors, pow2 = 1): the scaled operands are never written.  With
// exact power-of-two factors every sequential application a' <- a' / r' (or a' * p) is exact
// as long as its result is representable, so after t steps a'_ij = a_ij 2^(eR_i + eC_j) with
// integer net exponents (eR: -sum log2 r' over the O steps, eC: +sum log2 p over the I steps;
// B: -sum log2 p, -sum log2 s').  Step t's reductions then read the ORIGINAL A and B and
// apply the exponents on the fly: one read per step instead of a read + write, and the plan's
// root K1 applies the final exponents while forming S_r / T_r (kernels_lincomb.cu), so A', B'
// never touch HBM.  Multiplying by an exact 2^e is correctly rounded, so the last application
// (its result may round) equals the sequential one bitwise.  Every intermediate value a later
// step divides again must be exact: each virtual pass checks that its values are normal (or
// zero) and finite, and every factor an exact power of two with a normal reciprocal; otherwise
// the run switches, on device, to the materialised form from that step on -- it writes the
// values after the step from the exact values before it with the round-1 arithmetic (a / r,
// a * p, b / p, b / s', reading A9), then continues one read + write per step.
// pow2 = 0 runs materialised throughout.  Factors, step counts and the scaled matrices are
// bitwise the oracle's in every branch (tests/test_gpu_scaling.py).
// =============================================================================================
namespace {

constexpr int CT = 256;               // threads per block: 8 warps x 32 lanes
constexpr int CCOL = 4;               // columns per lane: 2 x 16-byte accesses
constexpr int CSTRIP = 32 * CCOL;     // 128-column strips
constexpr int CRU = 4;                // rows in flight per warp

struct CoopArgs {
  const double* A; int64_t lda; const double* B; int64_t ldb;
  double* Aw; int64_t ldaw; double* Bw; int64_t ldbw;  // materialised A', B'
  int64_t M, K, N;
  double *dA, *dB, *dI;
  int32_t *exAr, *exAc, *exBr, *exBc;  // net exponents of the virtual form
  double* mx[2];                       // rowA (M) | colA (K) | rowB (K) | colB (N)
  double *fr, *fs, *fp;                // factors of the current step (r M, s N, p K)
  int* flags;
  int nsteps, first_O, pow2, materialise_end;
  double tau, lo_O, lo_I, hi_I;
  int64_t chunkA, chunkB;              // rows per tile
  int stripsA, stripsB, tilesA, tilesB;
};

// x 2^e, correctly rounded (one multiplication by an exact power of two when it is a normal
// double, else ldexp)
__device__ __forceinline__ double scale2(double x, int e) {
  if (e == 0) return x;
  if (e >= -1022 && e <= 1023) return __dmul_rn(x, __longlong_as_double((int64_t)(e + 1023) << 52));
  return ldexp(x, e);
}
__device__ __forceinline__ bool exact_value(double x, double v) {
  const double a = fabs(v);
  return (a >= 2.2250738585072014e-308 || x == 0.0) && a <= 1.7976931348623157e308;
}
__device__ __forceinline__ int log2_pow2(double f) {  // f an exact normal power of two
  return (int)((__double_as_longlong(f) >> 52) & 0x7ff) - 1023;
}

enum PassKind { PK_RAW = 0, PK_VIRTUAL = 1, PK_MAT = 2 };

// One matrix's part of a pass: tile `tile` of the (rows x cols) matrix.  PK_RAW: maxima of the
// source; PK_VIRTUAL: maxima of src_ij 2^(er_i + ec_j), with the exactness check (F_BAD);
// PK_MAT: v = (stored ? src_ij : src_ij 2^(er_i + ec_j) undone to the values before this
// step) then this step's factor (row: divide by frow_i; column: multiply (cmul) or divide by
// fcol_j), stored to dst, maxima of v.
struct MatPass {
  const double* src; int64_t lds;
  double* dst; int64_t ldd;
  int64_t rows, cols, chunk;
  int strips;
  const int32_t* er; const int32_t* ec;
  const double* frow; const double* fcol;  // this step's factor (null: none on that side)
  int cmul;                                // column factor multiplies (A at an I step)
  int undo;                                // PK_MAT from the original: exponents include this step
  double* rmax; double* cmax;
};

template <int KIND>
__device__ void mat_tile(const MatPass& q, int tile, int* flags, double (*cm)[CSTRIP]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int strip = tile % q.strips;
  const int64_t rbeg = (int64_t)(tile / q.strips) * q.chunk;
  const int64_t rend = min(rbeg + q.chunk, q.rows);
  const int64_t cbase = (int64_t)strip * CSTRIP + 2 * lane;
  const int64_t lim = q.cols - cbase;
  const bool vec = ((((uintptr_t)q.src) & 15u) == 0) && (q.lds % 2 == 0) &&
                   (KIND != PK_MAT || (((((uintptr_t)q.dst) & 15u) == 0) && (q.ldd % 2 == 0)));
  int ecl[CCOL];
  double fcl[CCOL], cmx[CCOL];
  bool bad = false;
#pragma unroll
  for (int e = 0; e < CCOL; ++e) {
    const int off = (e / 2) * 64 + (e & 1);
    const bool ok = off < lim;
    ecl[e] = (KIND != PK_RAW && q.ec && ok) ? q.ec[cbase + off] : 0;
    fcl[e] = (KIND == PK_MAT && q.fcol && ok) ? q.fcol[cbase + off] : 1.0;
    if (KIND == PK_MAT && q.undo && q.fcol) {  // exponents already hold this step's column factor
      double inv;
      if (exact_recip(fcl[e], &inv)) ecl[e] += q.cmul ? -log2_pow2(fcl[e]) : log2_pow2(fcl[e]);
    }
    cmx[e] = 0.0;
  }
  for (int64_t rb = rbeg + warp; rb < rend; rb += 8 * CRU) {
    double x[CRU][CCOL];
#pragma unroll
    for (int u = 0; u < CRU; ++u) {
      const int64_t r = rb + u * 8;
#pragma unroll
      for (int e = 0; e < CCOL; ++e) x[u][e] = 0.0;
      if (r < rend) {
        const double* sp = q.src + r * q.lds + cbase;
#pragma unroll
        for (int h = 0; h < CCOL / 2; ++h) {
          const int off = h * 64;
          if (vec && off + 1 < lim) {
            const double2 v = *reinterpret_cast<const double2*>(sp + off);
            x[u][2 * h] = v.x; x[u][2 * h + 1] = v.y;
          } else {
            if (off < lim) x[u][2 * h] = sp[off];
            if (off + 1 < lim) x[u][2 * h + 1] = sp[off + 1];
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < CRU; ++u) {
      const int64_t r = rb + u * 8;
      if (r >= rend) continue;  // warp-uniform
      int erow = (KIND != PK_RAW && q.er) ? q.er[r] : 0;
      Divisor fdr;
      if (KIND == PK_MAT && q.frow) {
        const double f = q.frow[r];
        fdr = Divisor(f);
        double inv;
        if (q.undo && exact_recip(f, &inv)) erow += log2_pow2(f);  // undo this step's row exponent
      }
      double rmx = 0.0;
#pragma unroll
      for (int e = 0; e < CCOL; ++e) {
        const int off = (e / 2) * 64 + (e & 1);
        double v = x[u][e];
        if (KIND == PK_VIRTUAL) {
          const double y = scale2(v, erow + ecl[e]);
          if (off < lim && !exact_value(v, y)) bad = true;
          v = y;
        } else if (KIND == PK_MAT) {
          if (q.undo) v = scale2(v, erow + ecl[e]);  // exact: the values before this step
          if (q.frow) v = fdr.div(v);
          if (q.fcol) v = q.cmul ? __dmul_rn(v, fcl[e]) : Divisor(fcl[e]).div(v);
        }
        x[u][e] = v;
        const double a = off < lim ? fabs(v) : 0.0;
        rmx = fmax(rmx, a);
        cmx[e] = fmax(cmx[e], a);
      }
      if (KIND == PK_MAT) {
        double* dp = q.dst + r * q.ldd + cbase;
#pragma unroll
        for (int h = 0; h < CCOL / 2; ++h) {
          const int off = h * 64;
          if (vec && off + 1 < lim) {
            *reinterpret_cast<double2*>(dp + off) = make_double2(x[u][2 * h], x[u][2 * h + 1]);
          } else {
            if (off < lim) dp[off] = x[u][2 * h];
            if (off + 1 < lim) dp[off + 1] = x[u][2 * h + 1];
          }
        }
      }
      if (q.rmax) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) rmx = fmax(rmx, __shfl_xor_sync(0xffffffffu, rmx, o));
        if (lane == 0) atomic_max_nonneg(&q.rmax[r], rmx);
      }
    }
  }
  if (KIND == PK_VIRTUAL && __any_sync(0xffffffffu, bad) && lane == 0) atomicExch(&flags[F_BAD], 1);
  if (q.cmax) {
#pragma unroll
    for (int e = 0; e < CCOL; ++e) cm[warp][(e / 2) * 64 + 2 * lane + (e & 1)] = cmx[e];
    __syncthreads();
    for (int c = threadIdx.x; c < CSTRIP; c += CT) {
      double m = 0.0;
#pragma unroll
      for (int y = 0; y < 8; ++y) m = fmax(m, cm[y][c]);
      const int64_t cc = (int64_t)strip * CSTRIP + c;
      if (cc < q.cols) atomic_max_nonneg(&q.cmax[cc], m);
    }
    __syncthreads();
  }
}

// grid barrier: every block of the cooperative launch arrives, then all proceed
__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int nblocks, unsigned int& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    ++gen;
    __threadfence();
    const unsigned int target = gen * nblocks;
    atomicAdd(bar, 1u);
    while (true) {
      const unsigned int v = *(volatile unsigned int*)bar;
      if (v >= target) break;
      __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(CT, 2) k_scale_coop(CoopArgs a, unsigned int* bar) {
  __shared__ double cm[8][CSTRIP];
  const unsigned int nb = gridDim.x;
  unsigned int gen = 0;
  int* flags = a.flags;
  const int64_t M = a.M, K = a.K, N = a.N;
  const int64_t gtid = (int64_t)blockIdx.x * CT + threadIdx.x, gstride = (int64_t)nb * CT;
  // ---- init: factors, exponents, maxima set 0 (the launcher zeroed flags and the barrier)
  for (int64_t i = gtid; i < M; i += gstride) { a.dA[i] = 1.0; a.exAr[i] = 0; }
  for (int64_t j = gtid; j < N; j += gstride) { a.dB[j] = 1.0; a.exBc[j] = 0; }
  for (int64_t k = gtid; k < K; k += gstride) { a.dI[k] = 1.0; a.exAc[k] = 0; a.exBr[k] = 0; }
  for (int64_t i = gtid; i < M + 2 * K + N; i += gstride) { a.mx[0][i] = 0.0; a.mx[1][i] = 0.0; }
  if (gtid == 0) flags[F_MODE] = a.pow2 ? 0 : 1;
  grid_barrier(bar, nb, gen);

  auto views = [&](int isO, int kind, double* m) {  // (A part, B part) of a pass
    MatPass pa{}, pb{};
    const bool stored = flags[F_STORED] != 0;
    pa.src = (kind == PK_MAT && stored) ? a.Aw : a.A; pa.lds = (kind == PK_MAT && stored) ? a.ldaw : a.lda;
    pb.src = (kind == PK_MAT && stored) ? a.Bw : a.B; pb.lds = (kind == PK_MAT && stored) ? a.ldbw : a.ldb;
    pa.dst = a.Aw; pa.ldd = a.ldaw; pb.dst = a.Bw; pb.ldd = a.ldbw;
    pa.rows = M; pa.cols = K; pa.chunk = a.chunkA; pa.strips = a.stripsA;
    pb.rows = K; pb.cols = N; pb.chunk = a.chunkB; pb.strips = a.stripsB;
    pa.er = a.exAr; pa.ec = a.exAc; pb.er = a.exBr; pb.ec = a.exBc;
    pa.undo = pb.undo = (kind == PK_MAT && !stored) ? 1 : 0;
    return std::make_pair(pa, pb);
  };
  // run one pass over A and B (tiles of A, then of B, grid-strided)
  auto run_pass = [&](int kind, MatPass& pa, MatPass& pb) {
    for (int t = blockIdx.x; t < a.tilesA + a.tilesB; t += nb) {
      if (t < a.tilesA) {
        if (kind == PK_RAW) mat_tile<PK_RAW>(pa, t, flags, cm);
        else if (kind == PK_VIRTUAL) mat_tile<PK_VIRTUAL>(pa, t, flags, cm);
        else mat_tile<PK_MAT>(pa, t, flags, cm);
      } else {
        if (kind == PK_RAW) mat_tile<PK_RAW>(pb, t - a.tilesA, flags, cm);
        else if (kind == PK_VIRTUAL) mat_tile<PK_VIRTUAL>(pb, t - a.tilesA, flags, cm);
        else mat_tile<PK_MAT>(pb, t - a.tilesA, flags, cm);
      }
    }
  };
  // the maxima a step of kind isO needs, into maxima set m
  auto set_max = [&](MatPass& pa, MatPass& pb, int isO, double* m) {
    pa.rmax = isO ? m : nullptr;              // rowA
    pa.cmax = isO ? nullptr : m + M;          // colA
    pb.rmax = isO ? nullptr : m + M + K;      // rowB
    pb.cmax = isO ? m + M + 2 * K : nullptr;  // colB
  };
  // this step's factors on the A / B passes of a materialised application
  auto set_factors = [&](MatPass& pa, MatPass& pb, int isO) {
    if (isO) { pa.frow = a.fr; pb.fcol = a.fs; }
    else { pa.fcol = a.fp; pa.cmul = 1; pb.frow = a.fp; }
  };
  const int64_t set = M + 2 * K + N;
  // ---- initial reductions (the original operands) for step 0
  {
    const int isO = a.first_O;
    auto pp = views(isO, PK_RAW, a.mx[0]);
    set_max(pp.first, pp.second, isO, a.mx[0]);
    run_pass(PK_RAW, pp.first, pp.second);
  }
  grid_barrier(bar, nb, gen);
  int t0 = -1;
  for (int t = 0; t < a.nsteps; ++t) {
    const int isO = (t % 2 == 0) == (a.first_O != 0);
    if (isO && t0 < 0) t0 = t;
    const int test = (a.tau >= 0.0 && t0 >= 0 && t > t0) ? 1 : 0;
    double* cur = a.mx[t & 1];
    double* nxt = a.mx[(t + 1) & 1];
    int* fail = &flags[F_FAIL + (t & 1)];
    // ---- factors of step t (Alg. 3) from the maxima in `cur`; zero `nxt`
    for (int64_t i = gtid; i < set; i += gstride) nxt[i] = 0.0;
    if (gtid == 0) flags[F_FAIL + ((t + 1) & 1)] = 0;
    bool ok = true, badf = false;
    if (isO) {
      for (int64_t i = gtid; i < M; i += gstride) {
        double r = cur[i];
        if (!(r > 0.0)) {
          if (atomicCAS(&flags[F_ERR], 0, 1) == 0) flags[F_ERRIDX] = (int)i;
          r = __longlong_as_double(0x7ff8000000000000LL);
        } else if (a.pow2) {
          r = pow2_round(r);
        }
        a.fr[i] = r;
        a.dA[i] = __dmul_rn(a.dA[i], r);
        double inv;
        if (a.pow2 && exact_recip(r, &inv)) a.exAr[i] -= log2_pow2(r);
        else badf = true;
        ok = ok && (r >= a.lo_O);
      }
      for (int64_t j = gtid; j < N; j += gstride) {
        double sv = cur[M + 2 * K + j];
        if (!(sv > 0.0)) {
          if (atomicCAS(&flags[F_ERR], 0, 2) == 0) flags[F_ERRIDX] = (int)j;
          sv = __longlong_as_double(0x7ff8000000000000LL);
        } else if (a.pow2) {
          sv = pow2_round(sv);
        }
        a.fs[j] = sv;
        a.dB[j] = __dmul_rn(sv, a.dB[j]);
        double inv;
        if (a.pow2 && exact_recip(sv, &inv)) a.exBc[j] -= log2_pow2(sv);
        else badf = true;
        ok = ok && (sv >= a.lo_O);
      }
    } else {
      for (int64_t k = gtid; k < K; k += gstride) {
        const double ca = cur[M + k], rb = cur[M + K + k];
        double pv;
        if (!(ca > 0.0) || !(rb > 0.0)) {
          if (atomicCAS(&flags[F_ERR], 0, !(ca > 0.0) ? 3 : 4) == 0) flags[F_ERRIDX] = (int)k;
          pv = __longlong_as_double(0x7ff8000000000000LL);
        } else {
          pv = __dsqrt_rn(__ddiv_rn(rb, ca));
          if (a.pow2) pv = pow2_round(pv);
        }
        a.fp[k] = pv;
        a.dI[k] = __dmul_rn(a.dI[k], pv);
        double inv;
        if (a.pow2 && exact_recip(pv, &inv)) {
          const int e = log2_pow2(pv);
          a.exAc[k] += e;
          a.exBr[k] -= e;
        } else {
          badf = true;
        }
        ok = ok && (pv >= a.lo_I && pv <= a.hi_I);
      }
    }
    if (__any_sync(0xffffffffu, !ok) && (threadIdx.x & 31) == 0) atomicAdd(fail, 1);
    if (__any_sync(0xffffffffu, badf) && (threadIdx.x & 31) == 0 && flags[F_MODE] == 0)
      atomicExch(&flags[F_BAD], 1);
    grid_barrier(bar, nb, gen);
    if (gtid == 0) flags[F_STEPS] += 1;
    const bool done = (test && *(volatile int*)fail == 0) || t == a.nsteps - 1;
    const bool need_next = !done;  // the values after this step feed another step
    // ---- application of step t
    if (*(volatile int*)&flags[F_MODE] == 0 && *(volatile int*)&flags[F_BAD]) {
      // a factor the virtual form cannot carry: materialise from the exact values before it
      auto pp = views(isO, PK_MAT, nxt);
      set_factors(pp.first, pp.second, isO);
      if (need_next) set_max(pp.first, pp.second, !isO, nxt);
      run_pass(PK_MAT, pp.first, pp.second);
      if (gtid == 0) { flags[F_MODE] = 1; flags[F_STORED] = 1; }
      grid_barrier(bar, nb, gen);
    } else if (*(volatile int*)&flags[F_MODE] == 0) {
      if (need_next) {  // virtual: the next step's reductions of the values after this step
        auto pp = views(!isO, PK_VIRTUAL, nxt);
        set_max(pp.first, pp.second, !isO, nxt);
        run_pass(PK_VIRTUAL, pp.first, pp.second);
        grid_barrier(bar, nb, gen);
        if (*(volatile int*)&flags[F_BAD]) {  // inexact intermediates: redo, materialised
          for (int64_t i = gtid; i < set; i += gstride) nxt[i] = 0.0;
          grid_barrier(bar, nb, gen);
          auto pm = views(isO, PK_MAT, nxt);
          set_factors(pm.first, pm.second, isO);
          set_max(pm.first, pm.second, !isO, nxt);
          run_pass(PK_MAT, pm.first, pm.second);
          if (gtid == 0) { flags[F_MODE] = 1; flags[F_STORED] = 1; }
          grid_barrier(bar, nb, gen);
        }
      } else if (a.materialise_end) {  // the caller needs A', B' in memory
        auto pp = views(isO, PK_MAT, nxt);
        set_factors(pp.first, pp.second, isO);
        run_pass(PK_MAT, pp.first, pp.second);
        if (gtid == 0) { flags[F_MODE] = 1; flags[F_STORED] = 1; }
        grid_barrier(bar, nb, gen);
      }
    } else {  // materialised: apply in place (from A, B at the first application)
      auto pp = views(isO, PK_MAT, nxt);
      set_factors(pp.first, pp.second, isO);
      if (need_next) set_max(pp.first, pp.second, !isO, nxt);
      run_pass(PK_MAT, pp.first, pp.second);
      if (gtid == 0) flags[F_STORED] = 1;
      grid_barrier(bar, nb, gen);
    }
    if (done) {
      if (gtid == 0 && t < a.nsteps - 1) flags[F_DONE] = 1;
      break;
    }
  }
}

}  // namespace

size_t coop_scale_ws_extra() { return 64; }  // the grid barrier word (+ padding)

// Launch Alg. 1-3 as one cooperative kernel.  Writes dA, dB, dI, the flags, and either the
// virtual form's exponents (flags[F_MODE] = 0 at the end: the plan's root K1 applies them) or
// A', B' into A_out / B_out (flags[F_STORED] = 1).  materialise_end = 1 forces A', B' into
// A_out / B_out.  `bar` = 4 bytes of device scratch for the grid barrier.
cudaError_t run_scaling_coop(int64_t M, int64_t K, int64_t N, const double* A, int64_t lda,
                             const double* B, int64_t ldb, double* A_out, int64_t lda_out,
                             double* B_out, int64_t ldb_out, double* dA, double* dB, double* dI,
                             int nsteps, bool first_O, double tau, int pow2, int materialise_end,
                             void* sws, unsigned int* bar, cudaStream_t st) {
  ScaleWsView v = scale_ws_view(sws, M, K, N);
  cudaError_t e;
  if ((e = cudaMemsetAsync(v.flags, 0, sizeof(int) * F_COUNT, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(bar, 0, sizeof(unsigned int), st)) != cudaSuccess) return e;
  static int blocks_per_sm = -1, sms = 0;
  if (blocks_per_sm < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_scale_coop, CT, 0);
    if (blocks_per_sm > 3) blocks_per_sm = 3;
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  const int nblocks = sms * blocks_per_sm;
  CoopArgs a{};
  a.A = A; a.lda = lda; a.B = B; a.ldb = ldb;
  a.Aw = A_out; a.ldaw = lda_out; a.Bw = B_out; a.ldbw = ldb_out;
  a.M = M; a.K = K; a.N = N;
  a.dA = dA; a.dB = dB; a.dI = dI;
  a.exAr = v.ex; a.exAc = v.ex + M; a.exBr = v.ex + M + K; a.exBc = v.ex + M + 2 * K;
  a.mx[0] = v.mx[0]; a.mx[1] = v.mx[1];
  a.fr = v.r; a.fs = v.s; a.fp = v.p;
  a.flags = v.flags;
  a.nsteps = nsteps; a.first_O = first_O ? 1 : 0; a.pow2 = pow2; a.materialise_end = materialise_end;
  a.tau = tau;
  a.lo_O = pow(1.0 + tau, -0.5); a.lo_I = pow(1.0 + tau, -0.25); a.hi_I = pow(1.0 + tau, 0.25);
  auto tiles = [&](int64_t rows, int64_t cols, int64_t* chunk, int* strips, int* ntiles) {
    *strips = (int)((cols + CSTRIP - 1) / CSTRIP);
    int64_t nchunks = std::max<int64_t>(1, nblocks / *strips);
    int64_t ch = (rows + nchunks - 1) / nchunks;
    ch = std::max<int64_t>(8 * CRU, (ch + 8 * CRU - 1) / (8 * CRU) * (8 * CRU));
    *chunk = ch;
    *ntiles = (int)(*strips * ((rows + ch - 1) / ch));
  };
  tiles(M, K, &a.chunkA, &a.stripsA, &a.tilesA);
  tiles(K, N, &a.chunkB, &a.stripsB, &a.tilesB);
  void* args[] = {&a, &bar};
  return cudaLaunchCooperativeKernel((const void*)k_scale_coop, dim3((unsigned)nblocks), dim3(CT), args, 0, st);
}

// Exponent vectors and mode flag of the virtual form (for the plan's root K1).
void scale_virtual_view(void* sws, int64_t M, int64_t K, int64_t N, const int32_t** exAr,
                        const int32_t** exAc, const int32_t** exBr, const int32_t** exBc,
                        const int** mode_flag) {
  ScaleWsView v = scale_ws_view(sws, M, K, N);
  *exAr = v.ex; *exAc = v.ex + M; *exBr = v.ex + M + K; *exBc = v.ex + M + 2 * K;
  *mode_flag = v.flags + F_MODE;
}

// Apply given factors: A' = (a_ik / dA_i) * d_k, B' = (b_kj / d_k) / dB_j (each operation
// correctly rounded; exact for power-of-two factors).  One streaming pass per matrix.
__global__ void k_scale_apply_rows_cols(const double* __restrict__ X, int64_t ldx, double* __restrict__ Y,
                                        int64_t ldy, int64_t rows, int64_t cols,
                                        const double* __restrict__ rdiv, const double* __restrict__ cmul,
                                        const double* __restrict__ cdiv) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  const double cm = cmul ? cmul[j] : 1.0, cd = cdiv ? cdiv[j] : 1.0;
  for (int64_t i = blockIdx.y; i < rows; i += gridDim.y) {
    double x = __ddiv_rn(X[i * ldx + j], rdiv[i]);
    if (cmul) x = __dmul_rn(x, cm);
    if (cdiv) x = __ddiv_rn(x, cd);
    Y[i * ldy + j] = x;
  }
}

cudaError_t launch_scale_apply(int64_t M, int64_t K, int64_t N, const double* A, int64_t lda,
                               const double* B, int64_t ldb, const double* dA, const double* d,
                               const double* dB, double* A_out, int64_t lda_out, double* B_out,
                               int64_t ldb_out, cudaStream_t st) {
  if (M > 0 && K > 0)
    k_scale_apply_rows_cols<<<dim3((unsigned)((K + 255) / 256), (unsigned)(M < 4096 ? M : 4096)), 256, 0, st>>>(
        A, lda, A_out, lda_out, M, K, dA, d, nullptr);
  if (K > 0 && N > 0)
    k_scale_apply_rows_cols<<<dim3((unsigned)((N + 255) / 256), (unsigned)(K < 4096 ? K : 4096)), 256, 0, st>>>(
        B, ldb, B_out, ldb_out, K, N, d, nullptr, dB);
  return cudaGetLastError();
}

cudaError_t launch_unscale(double* C, int64_t ldc, int64_t M, int64_t N, const double* dA,
                           const double* dB, cudaStream_t st) {
  if (M == 0 || N == 0) return cudaSuccess;
  const bool vec = ((uintptr_t)C % 16 == 0) && ldc % 2 == 0;
  const int64_t per = vec ? 2 : 1;
  dim3 grid((unsigned)((N + 256 * per - 1) / (256 * per)), (unsigned)(M < 2048 ? M : 2048));
  if (vec) k_unscale<true><<<grid, 256, 0, st>>>(C, ldc, M, N, dA, dB);
  else k_unscale<false><<<grid, 256, 0, st>>>(C, ldc, M, N, dA, dB);
  return cudaGetLastError();
}

}  // namespace fmm
