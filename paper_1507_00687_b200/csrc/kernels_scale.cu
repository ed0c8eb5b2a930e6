// K4: diagonal scaling (Section 6, Alg. 1-3) on device, FP64: the whole run -- every
// step's max-abs reductions, factors, stopping test and applications -- in ONE cooperative
// kernel (k_scale_coop, below), plus the unscale / given-factor apply building blocks.
// Max-abs is combined across CTAs with atomicMax on the IEEE bit pattern (non-negative
// doubles order like their bit patterns): exact and order-free.  The stopping test of Thm
// stopping-criterion, from the step after the first O step, runs on
// device; the host never synchronises inside Alg. 3.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <utility>
#include <vector>

#include <cooperative_groups.h>

#include "fmm_internal.h"

namespace fmm {

namespace cg = cooperative_groups;

// flags layout (int32): [0] done, [1] steps taken, [2] error kind (0 none; 1 zero row of A,
// 2 zero col of B, 3 zero col of A, 4 zero row of B), [3] error index,
// [8] mode of the one-kernel run (0 virtual, 1 materialised), [9] bad (the virtual form cannot
// reproduce the sequential roundings: switch to materialised), [10], [11] stop-test failure
// counters of even / odd steps, [12] A' / B' are stored in the materialised buffers
enum { F_DONE = 0, F_STEPS = 1, F_ERR = 2, F_ERRIDX = 3, F_MODE = 8,
       F_BAD = 9, F_FAIL = 10, F_STORED = 12, F_BADX = 13, F_EXT = 16, F_COUNT = 24 };
// [13] the fused A pass (row_fused_tma) found a value after the O step the virtual form cannot
// carry (it counts only if that step's I reductions are needed)
// [16 .. 23]: min / max of the final net exponents exAr, exAc, exBr, exBc (the root K1's
// fast path needs every row + column exponent sum to be a normal power of two)

namespace {

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

// exact reciprocal of a power-of-two factor (false if f is not a power of two whose reciprocal
// is representable; then the dividing pass runs)
__device__ __forceinline__ bool exact_recip(double f, double* inv) {
  const int64_t bits = __double_as_longlong(f);
  const int ex = (int)((bits >> 52) & 0x7ff);
  if ((bits & 0x000fffffffffffffLL) != 0 || ex < 1 || ex > 2045 || !(f > 0.0)) return false;
  *inv = __longlong_as_double((int64_t)(2046 - ex) << 52);
  return true;
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
  // 3 sets of maxima (rowA M, colA K, rowB K, colB N; step t reads set t mod 3, the fused
  // A pass before an O step also writes set t + 1) + factor vectors (r M, s N, p K) + flags
  // (16 doubles) + exact reciprocals (r M, s N, p K) of power-of-two factors + the net
  // exponents of the virtual form (int32: rowA M, colA K, rowB K, colB N)
  return (size_t)(3 * (M + K + K + N) + 2 * (M + N + K) + 16) * sizeof(double) +
         (size_t)(M + K + K + N) * sizeof(int32_t) + 256;
}

struct ScaleWsView {
  double* mx[3];  // each: rowA (M) | colA (K) | rowB (K) | colB (N)
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
  v.mx[2] = w + 2 * set;
  v.r = w + 3 * set;
  v.s = v.r + M;
  v.p = v.s + N;
  v.ri = v.p + K;
  v.si = v.ri + M;
  v.pi = v.si + N;
  v.flags = (int*)(v.pi + K);
  v.ex = (int32_t*)(v.pi + K + 16);
  return v;
}

// [mx[0], flags + F_COUNT): the maxima sets, factor vectors, reciprocals and flags (contiguous)
static void* ws_zero_begin(const ScaleWsView& v) { return v.mx[0]; }
static size_t ws_zero_bytes(const ScaleWsView& v) {
  return (size_t)((const char*)(v.flags + F_COUNT) - (const char*)v.mx[0]);
}

int* scale_flags_ptr(void* ws, int64_t M, int64_t K, int64_t N) {
  return scale_ws_view(ws, M, K, N).flags;
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
  double* mx[3];                       // rowA (M) | colA (K) | rowB (K) | colB (N)
  double *fr, *fs, *fp;                // factors of the current step (r M, s N, p K)
  int* flags;
  int nsteps, first_O, pow2, materialise_end;
  double tau, lo_O, lo_I, hi_I;
  int64_t chunkA, chunkB;              // rows per tile (materialised passes)
  int stripsA, stripsB, tilesA, tilesB;
  // reduction-only passes: row tiles (1024-column segments x row chunks) and column tiles
  // (256-column strips x row chunks), per matrix
  int64_t rrowsA, rrowsB, crowsA, crowsB;
  int rsegsA, rsegsB, rtilesA, rtilesB, cstripsA, cstripsB, ctilesA, ctilesB;
  // B's row tiles when they share a pass with A's column tiles (an unfused I-reduction pass)
  int64_t rrowsBp; int rsegsBp, rtilesBp;
  // the fused A pass before an O step (row_fused_tma): whole-row tiles of frowsA rows
  int fuseA, ftilesA;
  int l2hint;  // L2 eviction-priority hints on the fused schedule's bulk copies
  int64_t frowsA;
  unsigned long long* trace;  // FMM_SCALE_TRACE: %globaltimer after every grid barrier
};

// x 2^e, correctly rounded (one multiplication by an exact power of two when it is a normal
// double, else ldexp)
__device__ __noinline__ double scale2_wide(double x, int e) { return ldexp(x, e); }
__device__ __forceinline__ double scale2(double x, int e) {
  if (e == 0) return x;
  if (e >= -1022 && e <= 1023) return __dmul_rn(x, __longlong_as_double((int64_t)(e + 1023) << 52));
  return scale2_wide(x, e);
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
  int l2pol;                               // bulk-copy L2 policy: 0 normal, 1 evict_first, 2 evict_last
};

// The per-element work of the reductions runs on IEEE bit patterns: for non-negative doubles the
// unsigned order of the bits is the numeric order (so a max is an integer max, combined across
// blocks with atomicMax), and an exact power-of-two scaling of a normal value is an integer add
// on the exponent field.  A virtual value a 2^e is exact -- equal to what the sequential
// divisions store -- iff a = 0 or both a and a 2^e are normal (else F_BAD).
constexpr uint64_t kAbsMask = 0x7fffffffffffffffULL, kInfBits = 0x7ff0000000000000ULL;

__device__ __forceinline__ uint64_t abs_bits(double x) { return (uint64_t)__double_as_longlong(x) & kAbsMask; }

// max(m, y) for a running maximum m that is never NaN (it starts at 0 and only takes values that
// compared greater): exactly fmax(m, y) -- a NaN y is ignored -- in one compare and two selects;
// sm_100 has no FP64 min / max instruction and fmax's NaN handling costs twice that
__device__ __forceinline__ double max_nn(double m, double y) { return y > m ? y : m; }

template <int KIND>
__device__ __noinline__ void mat_tile(const MatPass& q, int tile, int* flags, unsigned long long (*cm)[CSTRIP]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int strip = tile % q.strips;
  const int64_t rbeg = (int64_t)(tile / q.strips) * q.chunk;
  const int64_t rend = min(rbeg + q.chunk, q.rows);
  const int64_t cbase = (int64_t)strip * CSTRIP + 2 * lane;
  const int64_t lim = q.cols - cbase;
  const bool vec = ((((uintptr_t)q.src) & 15u) == 0) && (q.lds % 2 == 0) &&
                   (KIND != PK_MAT || (((((uintptr_t)q.dst) & 15u) == 0) && (q.ldd % 2 == 0)));
  int ecl[CCOL];
  double fcl[CCOL];
  uint64_t cmx[CCOL];
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
    cmx[e] = 0;
  }
  for (int64_t rb = rbeg + warp; rb < rend; rb += 8 * CRU) {
    double x[CRU][CCOL];
    int erow[CRU];
    double frw[CRU];
#pragma unroll
    for (int u = 0; u < CRU; ++u) {
      const int64_t r = rb + u * 8;
#pragma unroll
      for (int e = 0; e < CCOL; ++e) x[u][e] = 0.0;
      erow[u] = 0;
      frw[u] = 1.0;
      if (r < rend) {
        if (KIND != PK_RAW && q.er) erow[u] = q.er[r];
        if (KIND == PK_MAT && q.frow) frw[u] = q.frow[r];
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
      uint64_t rmx = 0;
      if (KIND == PK_MAT) {
        Divisor fdr;
        int er = erow[u];
        if (q.frow) {
          fdr = Divisor(frw[u]);
          double inv;
          if (q.undo && exact_recip(frw[u], &inv)) er += log2_pow2(frw[u]);  // undo this step's row exponent
        }
        double* dp = q.dst + r * q.ldd + cbase;
#pragma unroll
        for (int e = 0; e < CCOL; ++e) {
          double v = x[u][e];
          if (q.undo) v = scale2(v, er + ecl[e]);  // exact: the values before this step
          if (q.frow) v = fdr.div(v);
          if (q.fcol) v = q.cmul ? __dmul_rn(v, fcl[e]) : Divisor(fcl[e]).div(v);
          x[u][e] = v;
        }
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
#pragma unroll
      for (int e = 0; e < CCOL; ++e) {
        const int off = (e / 2) * 64 + (e & 1);
        uint64_t m = abs_bits(x[u][e]);
        if (KIND == PK_VIRTUAL) {  // |a| 2^e on the exponent field, with the exactness check
          const int ex = (int)(m >> 52), ee = ex + erow[u] + ecl[e];
          const bool ok = m == 0 || ((unsigned)(ex - 1) < 2046u && (unsigned)(ee - 1) < 2046u);
          if (off < lim && !ok) bad = true;
          m = m == 0 ? 0 : m + ((uint64_t)(int64_t)(erow[u] + ecl[e]) << 52);
        }
        if (m > kInfBits || off >= lim) m = 0;  // NaN is ignored by the max (as fmax)
        rmx = rmx > m ? rmx : m;
        cmx[e] = cmx[e] > m ? cmx[e] : m;
      }
      if (q.rmax) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const uint64_t y = __shfl_xor_sync(0xffffffffu, rmx, o);
          rmx = rmx > y ? rmx : y;
        }
        if (lane == 0) atomicMax(reinterpret_cast<unsigned long long*>(&q.rmax[r]), (unsigned long long)rmx);
      }
    }
  }
  if (KIND == PK_VIRTUAL && __any_sync(0xffffffffu, bad) && lane == 0) atomicExch(&flags[F_BAD], 1);
  if (q.cmax) {
#pragma unroll
    for (int e = 0; e < CCOL; ++e) cm[warp][(e / 2) * 64 + 2 * lane + (e & 1)] = cmx[e];
    __syncthreads();
    for (int c = threadIdx.x; c < CSTRIP; c += CT) {
      unsigned long long m = 0;
#pragma unroll
      for (int y = 0; y < 8; ++y) m = m > cm[y][c] ? m : cm[y][c];
      const int64_t cc = (int64_t)strip * CSTRIP + c;
      if (cc < q.cols) atomicMax(reinterpret_cast<unsigned long long*>(&q.cmax[cc]), m);
    }
    __syncthreads();
  }
}


// ---- reduction-only passes (the original operands, and the virtual form's steps) ------------
// Row maxima: a tile is a 512-column segment of a row chunk; lane l keeps the 16 column
// factors 2^ec_j of its columns (j = 64 it + 2 l + {0, 1}) in registers, and each warp walks
// rows with 8 16-byte loads in flight per lane: per element one multiply, a max and a nonzero
// min.  Column maxima: a tile is a 256-column strip of a row chunk, lane l owns 8 columns over
// the chunk's rows (per element: the row factor's multiply, a max, a min); warps combine in
// shared memory at the end.  Virtual values are exact iff every y = |a| 2^(one exponent) and
// every v = y 2^(the other) is normal or zero: checked on each row's / column's min and max
// (scaling is monotone).  RAW (the original values): only a NaN / Inf check (the virtual form
// cannot carry them: the run then materialises).
constexpr int RSEG = 512;  // 32 lanes x 16 columns
constexpr double kDblMin = 2.2250738585072014e-308, kDblMax = 1.7976931348623157e308;
constexpr double kInf = __builtin_huge_val();

__device__ __forceinline__ double pow2_of(int e, bool* bad) {  // 2^e as a normal double
  if (e < -1022 || e > 1023) { *bad = true; return 1.0; }
  return __longlong_as_double((int64_t)(e + 1023) << 52);
}

template <bool RAW>
__device__ __noinline__ void row_tile(const MatPass& q, int tile, int* flags, int segs, int64_t rows_per) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int seg = tile % segs;
  const int64_t r0 = (int64_t)(tile / segs) * rows_per;
  const int64_t r1 = min(r0 + rows_per, q.rows);
  const int64_t c0 = (int64_t)seg * RSEG + 2 * lane;
  const int64_t lim = q.cols - c0;  // lane column offset o is valid iff o < lim
  bool bad = false;
  double fc[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const int o = (e / 2) * 64 + (e & 1);
    fc[e] = (!RAW && o < lim) ? pow2_of(q.ec[c0 + o], &bad) : 1.0;
  }
  const bool vec = ((((uintptr_t)q.src) & 15u) == 0) && (q.lds % 2 == 0);
  // software pipeline: the next row's 8 16-byte loads (and its exponent) are in flight while
  // this row is reduced
  auto load = [&](int64_t r, double (&x)[16], int& er) {
    const double* sp = q.src + r * q.lds + c0;
    er = 0;
#pragma unroll
    for (int e = 0; e < 16; ++e) x[e] = 0.0;
    if (r >= r1) return;
    if (!RAW) er = q.er[r];
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      if (vec && h * 64 + 1 < lim) {
        const double2 v = *reinterpret_cast<const double2*>(sp + h * 64);
        x[2 * h] = v.x; x[2 * h + 1] = v.y;
      } else {
        if (h * 64 < lim) x[2 * h] = sp[h * 64];
        if (h * 64 + 1 < lim) x[2 * h + 1] = sp[h * 64 + 1];
      }
    }
  };
  double x[16], xn[16];
  int er, ern;
  load(r0 + warp, x, er);
  for (int64_t r = r0 + warp; r < r1; r += 8) {
    load(r + 8, xn, ern);
    double mx = 0.0, mn = kInf;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const double y = __dmul_rn(fabs(x[e]), fc[e]);
      if (RAW) bad = bad || !(y <= kDblMax);  // NaN or Inf
      mx = fmax(mx, y);
      mn = fmin(mn, y > 0.0 ? y : kInf);
    }
    if (!RAW && mn != kInf && (mn < kDblMin || scale2(mn, er) < kDblMin)) bad = true;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) {
      const double v = RAW ? mx : scale2(mx, er);
      if (!RAW && !(v <= kDblMax)) bad = true;
      atomicMax(reinterpret_cast<unsigned long long*>(&q.rmax[r]), (unsigned long long)abs_bits(v));
    }
#pragma unroll
    for (int e = 0; e < 16; ++e) x[e] = xn[e];
    er = ern;
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicExch(&flags[F_BAD], 1);
}

template <bool RAW>
__device__ __noinline__ void col_tile(const MatPass& q, int tile, int* flags, int strips, int64_t rows_per,
                                      double (*cm)[256]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int strip = tile % strips;
  const int64_t r0 = (int64_t)(tile / strips) * rows_per;
  const int64_t r1 = min(r0 + rows_per, q.rows);
  const int64_t c0 = (int64_t)strip * 256 + 2 * lane;
  const int64_t lim = q.cols - c0;
  bool bad = false;
  bool okc[8];
  double cmx[8], cmn[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    okc[e] = (e / 2) * 64 + (e & 1) < lim;
    cmx[e] = 0.0;
    cmn[e] = kInf;
  }
  const bool vec = ((((uintptr_t)q.src) & 15u) == 0) && (q.lds % 2 == 0);
  // software pipeline: the next 2 rows' loads (and row exponents) in flight during this pair
  auto load = [&](int64_t rb, double (&x)[2][8], int (&er)[2]) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t r = rb + 8 * u;
      er[u] = 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) x[u][e] = 0.0;
      if (r < r1) {
        if (!RAW) er[u] = q.er[r];
        const double* sp = q.src + r * q.lds + c0;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          if (vec && okc[2 * h + 1]) {
            const double2 v = *reinterpret_cast<const double2*>(sp + h * 64);
            x[u][2 * h] = v.x; x[u][2 * h + 1] = v.y;
          } else {
            if (okc[2 * h]) x[u][2 * h] = sp[h * 64];
            if (okc[2 * h + 1]) x[u][2 * h + 1] = sp[h * 64 + 1];
          }
        }
      }
    }
  };
  double x[2][8], xn[2][8];
  int er[2], ern[2];
  load(r0 + warp, x, er);
  for (int64_t rb = r0 + warp; rb < r1; rb += 16) {
    load(rb + 16, xn, ern);
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const double fr = RAW ? 1.0 : pow2_of(er[u], &bad);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const double y = __dmul_rn(fabs(x[u][e]), fr);
        if (RAW) bad = bad || !(y <= kDblMax);
        cmx[e] = fmax(cmx[e], y);
        cmn[e] = fmin(cmn[e], y > 0.0 ? y : kInf);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      er[u] = ern[u];
#pragma unroll
      for (int e = 0; e < 8; ++e) x[u][e] = xn[u][e];
    }
  }
  // combine the 8 warps: maxima in cm, minima (virtual form only) checked per warp and column
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    cm[warp][(e / 2) * 64 + 2 * lane + (e & 1)] = cmx[e];
    if (!RAW && okc[e] && cmn[e] != kInf) {
      const int64_t c = c0 + (e / 2) * 64 + (e & 1);
      if (cmn[e] < kDblMin || scale2(cmn[e], q.ec[c]) < kDblMin) bad = true;
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < 256; c += CT) {
    double m = 0.0;
#pragma unroll
    for (int y = 0; y < 8; ++y) m = fmax(m, cm[y][c]);
    const int64_t cc = (int64_t)strip * 256 + c;
    if (cc < q.cols) {
      const double v = RAW ? m : scale2(m, q.ec[cc]);
      if (!RAW && !(v <= kDblMax)) bad = true;
      atomicMax(reinterpret_cast<unsigned long long*>(&q.cmax[cc]), (unsigned long long)abs_bits(v));
    }
  }
  __syncthreads();
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicExch(&flags[F_BAD], 1);
}


// ---- TMA-staged forms of row_tile / col_tile (the default when rows are 16-byte aligned) ----
// Each warp streams its rows through its own ring of CS = 3 stages of 4 KB in shared memory:
// lane 0 issues one bulk copy (cp.async.bulk, completion counted on the stage's mbarrier) per
// 4 KB row segment (row tiles) or two 2 KB segments (column tiles: rows r, r + 8), CS copies
// ahead of the lanes consuming them -- 12 KB in flight per warp, 192 KB per SM, independent of
// registers.  The tile's row exponents are staged in shared memory once per tile.
constexpr int CS = 3;                   // stages per warp
constexpr int CSTG = 512;               // doubles per stage (4 KB)
constexpr int kTmaRows = 1024;          // row-exponent staging capacity per tile
struct TmaSmem {
  double* stage;                        // [8 warps][CS][CSTG]
  uint64_t* bar;                        // [8 warps][CS]
  int32_t* er;                          // [kTmaRows]
  uint32_t* phase;                      // [8 warps]: per-stage parity bits
};

__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ double2 lds2(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
// smallest nonzero y with y and y 2^e both normal: max(2^-1022, 2^(-1022 - e)); +inf if none
__device__ __forceinline__ double under_thr(int e) {
  const int t = -1022 - e;
  if (t <= -1022) return kDblMin;
  if (t > 1023) return kInf;
  return __longlong_as_double((int64_t)(t + 1023) << 52);
}
// bulk copy global -> shared, completion counted on `bar`; pol: the L2 eviction priority of the
// lines it reads (0 normal, 1 evict_first: not read again soon, 2 evict_last: the next pass reads
// them again -- DESIGN.md §6.4)
__device__ __forceinline__ void bulk_g2s_tx(void* dst, const void* src, uint32_t bytes, uint64_t* bar, int pol = 0) {
  if (pol == 0) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(s_u32(dst)), "l"(src), "r"(bytes), "r"(s_u32(bar)) : "memory");
    return;
  }
  uint64_t cp;
  if (pol == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(cp));
  else asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(cp));
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n"
               ::"r"(s_u32(dst)), "l"(src), "r"(bytes), "r"(s_u32(bar)), "l"(cp) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, int pol = 0) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(s_u32(bar)), "r"(bytes) : "memory");
  bulk_g2s_tx(dst, src, bytes, bar, pol);
}
__device__ __forceinline__ void expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(s_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                 " selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(s_u32(bar)), "r"(parity) : "memory");
  } while (!done);
}
// stage the tile's row exponents (rows [r0, r1)) in shared memory, the caller having synchronised
// the block before (nobody reads the previous tile's exponents any more)
__device__ __forceinline__ void stage_er_nosync(const MatPass& q, int64_t r0, int64_t r1, int32_t* sh) {
  for (int64_t r = r0 + threadIdx.x; r < r1; r += CT) sh[r - r0] = q.er ? q.er[r] : 0;
  __syncthreads();
}

template <bool RAW>
__device__ __noinline__ void row_tile_tma(const MatPass& q, int tile, int* flags, int segs, int64_t rows_per,
                                          const TmaSmem& sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int seg = tile % segs;
  const int64_t r0 = (int64_t)(tile / segs) * rows_per;
  const int64_t r1 = min(r0 + rows_per, q.rows);
  const int64_t cs = (int64_t)seg * RSEG;  // segment start column
  const int64_t len = min((int64_t)RSEG, q.cols - cs);
  const int64_t lim = len - 2 * lane;
  double* buf = sm.stage + (size_t)warp * CS * CSTG;
  uint64_t* bar = sm.bar + warp * CS;
  const int64_t rw = r0 + warp;
  const int n = rw < r1 ? (int)((r1 - rw + 7) / 8) : 0;
  const uint32_t bytes = (uint32_t)(len * 8);
  // the ring's first stages are requested before the exponent loads, so their latencies overlap
  __syncthreads();  // every warp is done with the previous tile's ring and exponents
  if (lane == 0)
    for (int k = 0; k < CS && k < n; ++k) bulk_g2s(buf + k * CSTG, q.src + (rw + 8 * k) * q.lds + cs, bytes, bar + k, q.l2pol);
  if (!RAW) stage_er_nosync(q, r0, r1, sm.er);
  bool bad = false;
  double fc[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const int o = (e / 2) * 64 + (e & 1);
    fc[e] = (!RAW && o < lim) ? pow2_of(q.ec[cs + 2 * lane + o], &bad) : 1.0;
  }
  __syncwarp();
  uint32_t ph = sm.phase[warp];
  for (int k = 0; k < n; ++k) {
    const int st = k % CS;
    const int64_t r = rw + 8 * k;
    bar_wait(bar + st, (ph >> st) & 1u);
    ph ^= 1u << st;
#ifdef FMM_SCALE_EXP  // development: the data movement alone (results invalid)
    __syncwarp();
    if (lane == 0 && k + CS < n) bulk_g2s(buf + st * CSTG, q.src + (r + 8 * CS) * q.lds + cs, bytes, bar + st, q.l2pol);
    continue;
#endif
    double x[16];
    const uint32_t sp = s_u32(buf + st * CSTG + 2 * lane);
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      const double2 v = lds2(sp + h * 64 * 8);
      x[2 * h] = v.x; x[2 * h + 1] = v.y;
    }
    __syncwarp();
    if (lane == 0 && k + CS < n) bulk_g2s(buf + st * CSTG, q.src + (r + 8 * CS) * q.lds + cs, bytes, bar + st, q.l2pol);
    const int er = RAW ? 0 : sm.er[r - r0];
    const double thr = under_thr(er);
    double mx = 0.0;
    if (lim < 512) {  // ragged segment: columns past the end read as 0
#pragma unroll
      for (int e = 0; e < 16; ++e)
        if ((e / 2) * 64 + (e & 1) >= lim) x[e] = 0.0;
    }
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const double y = __dmul_rn(fabs(x[e]), fc[e]);
      if (RAW) bad |= !(y <= kDblMax);          // NaN or Inf
      else bad |= (y < thr) & (y > 0.0);        // y or y 2^er not normal
      mx = max_nn(mx, y);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max_nn(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) {
      const double v = RAW ? mx : scale2(mx, er);
      if (!RAW && !(v <= kDblMax)) bad = true;
      atomicMax(reinterpret_cast<unsigned long long*>(&q.rmax[r]), (unsigned long long)abs_bits(v));
    }
  }
  if (lane == 0) sm.phase[warp] = ph;
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicExch(&flags[F_BAD], 1);
}

template <bool RAW>
__device__ __noinline__ void col_tile_tma(const MatPass& q, int tile, int* flags, int strips, int64_t rows_per,
                                          const TmaSmem& sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int strip = tile % strips;
  const int64_t r0 = (int64_t)(tile / strips) * rows_per;
  const int64_t r1 = min(r0 + rows_per, q.rows);
  const int64_t cs = (int64_t)strip * 256;
  const int64_t len = min((int64_t)256, q.cols - cs);
  const int64_t lim = len - 2 * lane;
  double* buf = sm.stage + (size_t)warp * CS * CSTG;
  uint64_t* bar = sm.bar + warp * CS;
  const int64_t rw = r0 + warp;  // this warp's rows: rw + 8 j; a stage holds rows j, j + 1 of them
  const int nr = rw < r1 ? (int)((r1 - rw + 7) / 8) : 0;
  const int n = (nr + 1) / 2;
  const uint32_t bytes = (uint32_t)(len * 8);
  auto issue = [&](int k, int st) {
    const int64_t ra = rw + 16 * k, rb = ra + 8;
    const uint32_t tot = rb < r1 ? 2 * bytes : bytes;
    expect_tx(bar + st, tot);
    bulk_g2s_tx(buf + st * CSTG, q.src + ra * q.lds + cs, bytes, bar + st, q.l2pol);
    if (rb < r1) bulk_g2s_tx(buf + st * CSTG + 256, q.src + rb * q.lds + cs, bytes, bar + st, q.l2pol);
  };
  // the ring's first stages are requested before the exponent loads, so their latencies overlap
  __syncthreads();  // every warp is done with the previous tile's ring and exponents
  if (lane == 0)
    for (int k = 0; k < CS && k < n; ++k) issue(k, k);
  if (!RAW) stage_er_nosync(q, r0, r1, sm.er);
  bool bad = false;
  double cmx[8], cthr[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int o = (e / 2) * 64 + (e & 1);
    cmx[e] = 0.0;
    cthr[e] = (!RAW && o < lim) ? under_thr(q.ec[cs + 2 * lane + o]) : kDblMin;
  }
  __syncwarp();
  uint32_t ph = sm.phase[warp];
  for (int k = 0; k < n; ++k) {
    const int st = k % CS;
    bar_wait(bar + st, (ph >> st) & 1u);
    ph ^= 1u << st;
#ifdef FMM_SCALE_EXP
    __syncwarp();
    if (lane == 0 && k + CS < n) issue(k + CS, st);
    continue;
#endif
    double x[2][8];
    const int64_t ra = rw + 16 * k;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint32_t sp = s_u32(buf + st * CSTG + u * 256 + 2 * lane);
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const double2 v = lds2(sp + h * 64 * 8);
        x[u][2 * h] = v.x; x[u][2 * h + 1] = v.y;
      }
    }
    __syncwarp();
    if (lane == 0 && k + CS < n) issue(k + CS, st);
    if (lim < 256) {  // ragged strip: columns past the end read as 0
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if ((e / 2) * 64 + (e & 1) >= lim) x[u][e] = 0.0;
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t r = ra + 8 * u;
      if (r >= r1) continue;  // warp-uniform
      const double fr = RAW ? 1.0 : pow2_of(sm.er[r - r0], &bad);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const double y = __dmul_rn(fabs(x[u][e]), fr);
        if (RAW) bad |= !(y <= kDblMax);          // NaN or Inf
        else bad |= (y < cthr[e]) & (y > 0.0);    // y or y 2^ec not normal
        cmx[e] = max_nn(cmx[e], y);
      }
    }
  }
  if (lane == 0) sm.phase[warp] = ph;
  // combine the 8 warps (in the stage buffers, now free)
  __syncthreads();
  double (*cm)[256] = reinterpret_cast<double (*)[256]>(sm.stage);
#pragma unroll
  for (int e = 0; e < 8; ++e) cm[warp][(e / 2) * 64 + (e & 1) + 2 * lane] = cmx[e];
  __syncthreads();
  for (int c = threadIdx.x; c < 256; c += CT) {
    double m = 0.0;
#pragma unroll
    for (int y = 0; y < 8; ++y) m = max_nn(m, cm[y][c]);
    if (c < len) {
      const double v = RAW ? m : scale2(m, q.ec[cs + c]);
      if (!RAW && !(v <= kDblMax)) bad = true;
      atomicMax(reinterpret_cast<unsigned long long*>(&q.cmax[cs + c]), (unsigned long long)abs_bits(v));
    }
  }
  __syncthreads();
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicExch(&flags[F_BAD], 1);
}

// ---- the fused A pass before an O step ------------------------------------
// The O step's row factor r_i depends on row i of A alone, so a block that holds whole
// rows can finish the O reduction of a row, form r_i, and feed the row's values AFTER the step
// into the next (I) step's column maxima of A while the row is still on chip: one read
// of A serves two steps.  A tile is a chunk of whole rows (K <= 4096: warp w owns columns
// [512 w, 512 w + 512), 16 per lane in registers); the rows stream through a ring of CS row-size
// stages (32 KB each, the per-warp rings' memory) filled by one bulk copy per row.  Per row: the
// O row maximum exactly as row_tile_tma forms it (written to rowA), r_i as the factor phase will
// recompute it from that maximum (pow2_round; the factor phase stays the only writer of r, D_A
// and the exponents, so a redo leaves nothing half-applied), then z = y 2^(er_i - log2 r_i) with
// y = |a| 2^(ec) into the lane's column maxima, which go to the next step's colA with atomicMax
// at the end of the tile.  Exactness of z (y 2^e normal or zero, the exponent in range) is
// flagged in F_BADX, which only matters when the I step's reductions are needed; the row part
// flags F_BAD exactly as row_tile_tma does.  Virtual form only (pow2, nothing materialised).
constexpr int FRK = 4096;  // longest fused row (doubles): 8 warps x 512 columns
template <bool RAW>
__device__ __noinline__ void row_fused_tma(const MatPass& q, double* colmax_next, int tile, int* flags,
                                           int64_t rows_per, const TmaSmem& sm, uint64_t* fbar,
                                           uint32_t* fphase, double (*red)[8]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r0 = (int64_t)tile * rows_per;
  const int64_t r1 = min(r0 + rows_per, q.rows);
  const int n = r0 < r1 ? (int)(r1 - r0) : 0;
  const int64_t cw = (int64_t)warp * 512;
  const int64_t lim = q.cols - cw - 2 * lane;  // lane column offset o valid iff o < lim
  const uint32_t bytes = (uint32_t)(q.cols * 8);
  double* ring = sm.stage;  // CS stages of FRK doubles
  __syncthreads();  // every warp is done with the previous tile's ring, exponents and red
  if (threadIdx.x == 0)
    for (int k = 0; k < CS && k < n; ++k) bulk_g2s(ring + k * FRK, q.src + (r0 + k) * q.lds, bytes, fbar + k, q.l2pol);
  if (!RAW) stage_er_nosync(q, r0, r1, sm.er);
  bool bad = false, badx = false;
  double fc[16], cmx[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const int o = (e / 2) * 64 + (e & 1);
    fc[e] = (!RAW && o < lim) ? pow2_of(q.ec[cw + 2 * lane + o], &bad) : 1.0;
    cmx[e] = 0.0;
  }
  uint32_t ph = *fphase;
  for (int k = 0; k < n; ++k) {
    const int st = k % CS;
    const int64_t r = r0 + k;
    bar_wait(fbar + st, (ph >> st) & 1u);
    ph ^= 1u << st;
#ifdef FMM_SCALE_EXP
    __syncthreads();
    if (threadIdx.x == 0 && k + CS < n) bulk_g2s(ring + st * FRK, q.src + (r + CS) * q.lds, bytes, fbar + st, q.l2pol);
    continue;
#endif
    double y[16];
    const uint32_t sp = s_u32(ring + st * FRK + cw + 2 * lane);
    if (lim > 0) {
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        if (h * 64 < lim) {
          const double2 v = lds2(sp + h * 64 * 8);
          y[2 * h] = v.x; y[2 * h + 1] = v.y;
        } else {
          y[2 * h] = 0.0; y[2 * h + 1] = 0.0;
        }
      }
    } else {
#pragma unroll
      for (int e = 0; e < 16; ++e) y[e] = 0.0;
    }
    const int er = RAW ? 0 : sm.er[r - r0];
    const double thr = under_thr(er);
    double mx = 0.0;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      y[e] = __dmul_rn(fabs(y[e]), fc[e]);
      if (RAW) bad |= !(y[e] <= kDblMax);          // NaN or Inf
      else bad |= (y[e] < thr) & (y[e] > 0.0);     // y or y 2^er not normal
      mx = max_nn(mx, y[e]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max_nn(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) red[k & 1][warp] = mx;
    __syncthreads();  // row k's maxima are in red; every warp has its values out of the stage
    if (threadIdx.x == 0 && k + CS < n) bulk_g2s(ring + st * FRK, q.src + (r + CS) * q.lds, bytes, fbar + st, q.l2pol);
    double m = red[k & 1][0];
#pragma unroll
    for (int w = 1; w < 8; ++w) m = max_nn(m, red[k & 1][w]);
    const double v = RAW ? m : scale2(m, er);  // the O row maximum (row_tile_tma's value)
    if (!RAW && !(v <= kDblMax)) bad = true;
    if (threadIdx.x == 0) q.rmax[r] = __longlong_as_double((int64_t)abs_bits(v));
    // r_i as the factor phase forms it (reading A8), and the row's values after the step
    int ern = er;
    double rf = 0.0, inv;
    if (v > 0.0) rf = pow2_round(v);
    if (v > 0.0 && exact_recip(rf, &inv)) ern = er - log2_pow2(rf);
    else badx = true;
    const double pf = pow2_of(ern, &badx);
    const double thr2 = under_thr(ern);
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      badx |= (y[e] < thr2) & (y[e] > 0.0);      // z = y 2^ern not normal
      cmx[e] = max_nn(cmx[e], __dmul_rn(y[e], pf));
    }
  }
  if (threadIdx.x == 0) *fphase = ph;
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const int o = (e / 2) * 64 + (e & 1);
    if (o < lim && n > 0) {
      if (!(cmx[e] <= kDblMax)) badx = true;
      atomicMax(reinterpret_cast<unsigned long long*>(&colmax_next[cw + 2 * lane + o]),
                (unsigned long long)abs_bits(cmx[e]));
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicExch(&flags[F_BAD], 1);
  if (__any_sync(0xffffffffu, badx) && lane == 0) atomicExch(&flags[F_BADX], 1);
}

// dynamic shared memory of k_scale_coop: the TMA stage ring (also the warp-combine buffers and
// the fused pass's row ring), its mbarriers, the row exponents of a tile, the per-warp parities,
// the fused pass's row-ring mbarriers, parity word and per-warp row maxima
static_assert(CS * FRK <= 8 * CS * CSTG, "fused row ring fits the per-warp rings");
constexpr size_t kCoopSmem = (size_t)8 * CS * CSTG * sizeof(double) + 8 * CS * sizeof(uint64_t) +
                             kTmaRows * sizeof(int32_t) + 8 * sizeof(uint32_t) +
                             CS * sizeof(uint64_t) + 8 + 2 * 8 * sizeof(double) + 8 * sizeof(int);

__global__ void __launch_bounds__(CT, 2) k_scale_coop(CoopArgs a) {
  extern __shared__ __align__(128) uint8_t dsm[];
  TmaSmem tsm;
  tsm.stage = reinterpret_cast<double*>(dsm);
  tsm.bar = reinterpret_cast<uint64_t*>(dsm + (size_t)8 * CS * CSTG * sizeof(double));
  tsm.er = reinterpret_cast<int32_t*>(tsm.bar + 8 * CS);
  tsm.phase = reinterpret_cast<uint32_t*>(tsm.er + kTmaRows);
  uint64_t* fbar = reinterpret_cast<uint64_t*>(tsm.phase + 8);  // fused row ring: CS mbarriers
  uint32_t* fphase = reinterpret_cast<uint32_t*>(fbar + CS);
  double (*red)[8] = reinterpret_cast<double (*)[8]>(fphase + 2);
  int* shflags = reinterpret_cast<int*>(red + 2);  // the run's flags, as thread 0 read them
  if (threadIdx.x < 8 * CS) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(s_u32(tsm.bar + threadIdx.x)));
  if (threadIdx.x < CS) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(s_u32(fbar + threadIdx.x)));
  if (threadIdx.x < 8) tsm.phase[threadIdx.x] = 0;
  if (threadIdx.x == 0) *fphase = 0;
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  double (*cmd)[256] = reinterpret_cast<double (*)[256]>(dsm);
  unsigned long long (*cm)[CSTRIP] = reinterpret_cast<unsigned long long (*)[CSTRIP]>(dsm);
  const unsigned int nb = gridDim.x;
  // grid-wide barrier of the cooperative launch (orders global memory and invalidates L1, so
  // the factors / exponents / maxima written before it are what every block reads after it)
  cg::grid_group grid = cg::this_grid();
  int nmark = 0;
  auto gsync = [&]() {
    if (a.trace) {  // arrival per block (a.trace is uniform over the grid)
      __syncthreads();
      if (threadIdx.x == 0 && nmark < 63 && blockIdx.x < 512) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.trace[64 + nmark * 512 + blockIdx.x] = t;
      }
    }
    grid.sync();
    if (a.trace && nmark < 63) {
      ++nmark;  // every thread counts the barriers; block 0 records the release time
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.trace[nmark] = t;
      }
    }
  };
  if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[0] = t;
  }
  int* flags = a.flags;
  const int64_t M = a.M, K = a.K, N = a.N;
  const int64_t gtid = (int64_t)blockIdx.x * CT + threadIdx.x, gstride = (int64_t)nb * CT;
  // ---- init: factors and exponents (the launcher zeroed the three maxima sets and the flags).
  // No barrier: the first pass (raw values) reads none of these, and the first reads of them
  // come after that pass's barrier
  for (int64_t i = gtid; i < M; i += gstride) { a.dA[i] = 1.0; a.exAr[i] = 0; }
  for (int64_t j = gtid; j < N; j += gstride) { a.dB[j] = 1.0; a.exBc[j] = 0; }
  for (int64_t k = gtid; k < K; k += gstride) { a.dI[k] = 1.0; a.exAc[k] = 0; a.exBr[k] = 0; }
  if (gtid == 0) flags[F_MODE] = a.pow2 ? 0 : 1;
  if (gtid < 8) flags[F_EXT + gtid] = (gtid & 1) ? (-0x7fffffff - 1) : 0x7fffffff;

  // The run's control flags after a grid barrier: thread 0 of each block reads them once (one
  // round trip, one request per block instead of every warp's chain of dependent loads on the
  // same words) and the block reads its copy in shared memory.
  struct FlagView { int mode, bad, badx, stored, fail; };
  auto read_flags = [&](const int* failp) {
    __syncthreads();  // nobody still reads the previous copy
    if (threadIdx.x == 0) {
      const int m = *(volatile int*)&flags[F_MODE], b = *(volatile int*)&flags[F_BAD];
      const int bx = *(volatile int*)&flags[F_BADX], st = *(volatile int*)&flags[F_STORED];
      const int f = failp ? *(volatile const int*)failp : 0;
      shflags[0] = m; shflags[1] = b; shflags[2] = bx; shflags[3] = st; shflags[4] = f;
    }
    __syncthreads();
    return FlagView{shflags[0], shflags[1], shflags[2], shflags[3], shflags[4]};
  };
  int stored_now = 0;  // F_STORED as of the last read_flags
  auto views = [&](int isO, int kind, double* m) {  // (A part, B part) of a pass
    MatPass pa{}, pb{};
    const bool stored = stored_now != 0;
    pa.src = (kind == PK_MAT && stored) ? a.Aw : a.A; pa.lds = (kind == PK_MAT && stored) ? a.ldaw : a.lda;
    pb.src = (kind == PK_MAT && stored) ? a.Bw : a.B; pb.lds = (kind == PK_MAT && stored) ? a.ldbw : a.ldb;
    pa.dst = a.Aw; pa.ldd = a.ldaw; pb.dst = a.Bw; pb.ldd = a.ldbw;
    pa.rows = M; pa.cols = K; pa.chunk = a.chunkA; pa.strips = a.stripsA;
    pb.rows = K; pb.cols = N; pb.chunk = a.chunkB; pb.strips = a.stripsB;
    pa.er = a.exAr; pa.ec = a.exAc; pb.er = a.exBr; pb.ec = a.exBc;
    // the exponents carry the factors applied so far only in the virtual form (pow2); a first
    // materialised application from A, B undoes this step's exponent to get the values before it
    pa.undo = pb.undo = (kind == PK_MAT && !stored && a.pow2) ? 1 : 0;
    return std::make_pair(pa, pb);
  };
  // run one pass over A and B (tiles of A, then of B, grid-strided)
  int npass = 0;
  bool fusedQ = false;  // the pass just run was the fused A pass before an O step
  // amode (reduction passes): 0 A's reductions as set in pa; 1 no A part; 2 the fused A pass
  // before an O step (row maxima into pa.rmax, the values after the step's column maxima into
  // colA_next)
  auto run_pass = [&](int kind, MatPass& pa, MatPass& pb, int amode = 0, double* colA_next = nullptr) {
    if (kind != PK_MAT && a.l2hint) {  // a fused pass keeps B in L2 for the B-only pass after it
      pa.l2pol = amode == 2 ? 1 : 0;
      pb.l2pol = amode == 2 ? 2 : amode == 1 ? 1 : 0;
    }
    if (kind != PK_MAT) {  // reductions only: row or column tiles per matrix
      const int na = amode == 1 ? 0 : amode == 2 ? a.ftilesA : pa.rmax ? a.rtilesA : a.ctilesA;
      const bool pairedB = na > 0 && pb.rmax != nullptr;  // B rows alongside A columns
      const int nbt = pb.rmax ? (pairedB ? a.rtilesBp : a.rtilesB) : a.ctilesB;
      // alternate passes walk the tiles in reverse: a pass starts on the ~100 MB the previous
      // one read last, still in the 126 MB L2
      const bool rev = (npass++ & 1) != 0;
      for (int t0 = blockIdx.x; t0 < na + nbt; t0 += nb) {
        const int t = rev ? na + nbt - 1 - t0 : t0;
        const bool isA = t < na;
        const MatPass& q = isA ? pa : pb;
        const int tt = isA ? t : t - na;
        const int segs = isA ? a.rsegsA : pairedB ? a.rsegsBp : a.rsegsB;
        const int strips = isA ? a.cstripsA : a.cstripsB;
        const int64_t rr = isA ? a.rrowsA : pairedB ? a.rrowsBp : a.rrowsB, cr = isA ? a.crowsA : a.crowsB;
        // TMA staging needs 16-byte aligned rows (and whole 16-byte row segments)
        const bool tma = ((((uintptr_t)q.src) & 15u) == 0) && q.lds % 2 == 0 && q.cols % 2 == 0;
        if (isA && amode == 2) {
          if (kind == PK_RAW) row_fused_tma<true>(q, colA_next, tt, flags, a.frowsA, tsm, fbar, fphase, red);
          else row_fused_tma<false>(q, colA_next, tt, flags, a.frowsA, tsm, fbar, fphase, red);
        } else if (q.rmax) {
          if (tma && rr <= kTmaRows) {
            if (kind == PK_RAW) row_tile_tma<true>(q, tt, flags, segs, rr, tsm);
            else row_tile_tma<false>(q, tt, flags, segs, rr, tsm);
          } else {
            if (kind == PK_RAW) row_tile<true>(q, tt, flags, segs, rr);
            else row_tile<false>(q, tt, flags, segs, rr);
          }
        } else {
          if (tma && cr <= kTmaRows) {
            if (kind == PK_RAW) col_tile_tma<true>(q, tt, flags, strips, cr, tsm);
            else col_tile_tma<false>(q, tt, flags, strips, cr, tsm);
          } else {
            __syncthreads();  // cmd aliases the stage ring
            if (kind == PK_RAW) col_tile<true>(q, tt, flags, strips, cr, cmd);
            else col_tile<false>(q, tt, flags, strips, cr, cmd);
          }
        }
      }
      return;
    }
    for (int t = blockIdx.x; t < a.tilesA + a.tilesB; t += nb) {
      const bool isA = t < a.tilesA;
      const MatPass& q = isA ? pa : pb;
      const int tt = isA ? t : t - a.tilesA;
      if (kind == PK_RAW) mat_tile<PK_RAW>(q, tt, flags, cm);
      else if (kind == PK_VIRTUAL) mat_tile<PK_VIRTUAL>(q, tt, flags, cm);
      else mat_tile<PK_MAT>(q, tt, flags, cm);
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
    fusedQ = isO && a.fuseA && a.nsteps > 1;
    run_pass(PK_RAW, pp.first, pp.second, fusedQ ? 2 : 0, a.mx[1] + M);
  }
  gsync();
  int t0 = -1;
  for (int t = 0; t < a.nsteps; ++t) {
    const int isO = (t % 2 == 0) == (a.first_O != 0);
    if (isO && t0 < 0) t0 = t;
    const int test = (a.tau >= 0.0 && t0 >= 0 && t > t0) ? 1 : 0;
    double* cur = a.mx[t % 3];
    double* nxt = a.mx[(t + 1) % 3];
    double* nxt2 = a.mx[(t + 2) % 3];
    int* fail = &flags[F_FAIL + (t & 1)];
    // ---- factors of step t (Alg. 3) from the maxima in `cur`; zero the set step
    // t + 2 reads (nxt was zeroed at step t - 1: the fused A pass before an O step t + 1 writes
    // into it and into nxt2 during step t's application)
    for (int64_t i = gtid; i < set; i += gstride) nxt2[i] = 0.0;
    if (gtid == 0) flags[F_FAIL + ((t + 1) & 1)] = 0;
    bool ok = true, badf = false;
    // one element per thread over rows then columns (O) or k (I); every input is loaded before
    // the first store, so each element costs one L2 round trip, not three
    if (isO) {
      for (int64_t idx = gtid; idx < M + N; idx += gstride) {
        const bool row = idx < M;                 // r_i of A's row, else s'_j of B's column
        const int64_t i = row ? idx : idx - M;
        double f = row ? cur[i] : cur[M + 2 * K + i];
        const double dold = row ? a.dA[i] : a.dB[i];
        const int32_t eold = row ? a.exAr[i] : a.exBc[i];
        if (!(f > 0.0)) {
          if (atomicCAS(&flags[F_ERR], 0, row ? 1 : 2) == 0) flags[F_ERRIDX] = (int)i;
          f = __longlong_as_double(0x7ff8000000000000LL);
        } else if (a.pow2) {
          f = pow2_round(f);
        }
        double inv;
        const bool ex = a.pow2 && exact_recip(f, &inv);
        if (!ex) badf = true;
        if (row) {
          a.fr[i] = f;
          a.dA[i] = __dmul_rn(dold, f);           // D_A <- D_A r'
          if (ex) a.exAr[i] = eold - log2_pow2(f);
        } else {
          a.fs[i] = f;
          a.dB[i] = __dmul_rn(f, dold);           // D_B <- s' D_B
          if (ex) a.exBc[i] = eold - log2_pow2(f);
        }
        ok = ok && (f >= a.lo_O);
      }
    } else {
      for (int64_t k = gtid; k < K; k += gstride) {
        const double ca = cur[M + k], rb = cur[M + K + k];
        const double dold = a.dI[k];
        const int32_t eac = a.exAc[k], ebr = a.exBr[k];
        double pv;
        if (!(ca > 0.0) || !(rb > 0.0)) {
          if (atomicCAS(&flags[F_ERR], 0, !(ca > 0.0) ? 3 : 4) == 0) flags[F_ERRIDX] = (int)k;
          pv = __longlong_as_double(0x7ff8000000000000LL);
        } else {
          pv = __dsqrt_rn(__ddiv_rn(rb, ca));
          if (a.pow2) pv = pow2_round(pv);
        }
        a.fp[k] = pv;
        a.dI[k] = __dmul_rn(dold, pv);
        double inv;
        if (a.pow2 && exact_recip(pv, &inv)) {
          const int e = log2_pow2(pv);
          a.exAc[k] = eac + e;
          a.exBr[k] = ebr - e;
        } else {
          badf = true;
        }
        ok = ok && (pv >= a.lo_I && pv <= a.hi_I);
      }
    }
    // one atomic per block, not per warp: up to 256 warps would serialise on the same word
    // right before the barrier
    const int blk_fail = __syncthreads_or(!ok), blk_bad = __syncthreads_or(badf);
    if (threadIdx.x == 0) {
      if (blk_fail) atomicAdd(fail, 1);
      if (blk_bad && *(volatile int*)&flags[F_MODE] == 0) atomicExch(&flags[F_BAD], 1);
    }
    gsync();
    if (gtid == 0) flags[F_STEPS] += 1;
    const FlagView fv = read_flags(fail);
    stored_now = fv.stored;
    const bool done = (test && fv.fail == 0) || t == a.nsteps - 1;
    const bool need_next = !done;  // the values after this step feed another step
    // ---- application of step t
    const bool fusedT = fusedQ;  // step t's maxima came from a fused A pass (nxt holds colA)
    fusedQ = false;
    if (fv.mode == 0 && fv.bad) {
      // a factor the virtual form cannot carry: materialise from the exact values before it
      if (fusedT && need_next) {  // drop the fused pass's speculative colA
        for (int64_t i = gtid; i < set; i += gstride) nxt[i] = 0.0;
        gsync();
      }
      auto pp = views(isO, PK_MAT, nxt);
      set_factors(pp.first, pp.second, isO);
      if (need_next) set_max(pp.first, pp.second, !isO, nxt);
      run_pass(PK_MAT, pp.first, pp.second);
      if (gtid == 0) { flags[F_MODE] = 1; flags[F_STORED] = 1; }
      gsync();
    } else if (fv.mode == 0) {
      if (need_next) {  // virtual: the next step's reductions of the values after this step
        auto pp = views(!isO, PK_VIRTUAL, nxt);
        set_max(pp.first, pp.second, !isO, nxt);
        // after an I step whose next (O) step is not the last: the fused A pass (it also
        // forms step t + 2's colA); after an O step whose A side the fused pass did: B only
        const int amode = fusedT ? 1 : (!isO && a.fuseA && t + 1 < a.nsteps - 1) ? 2 : 0;
        run_pass(PK_VIRTUAL, pp.first, pp.second, amode, nxt2 + M);
        gsync();
        const FlagView fp = read_flags(nullptr);
        const bool redo = fp.bad || (fusedT && fp.badx);
        if (!redo && amode == 2) fusedQ = true;
        if (redo) {  // inexact intermediates: redo, materialised
          for (int64_t i = gtid; i < set; i += gstride) nxt[i] = 0.0;
          if (amode == 2) for (int64_t i = gtid; i < set; i += gstride) nxt2[i] = 0.0;
          gsync();
          auto pm = views(isO, PK_MAT, nxt);
          set_factors(pm.first, pm.second, isO);
          set_max(pm.first, pm.second, !isO, nxt);
          run_pass(PK_MAT, pm.first, pm.second);
          if (gtid == 0) { flags[F_MODE] = 1; flags[F_STORED] = 1; }
          gsync();
        }
      } else if (a.materialise_end) {  // the caller needs A', B' in memory
        auto pp = views(isO, PK_MAT, nxt);
        set_factors(pp.first, pp.second, isO);
        run_pass(PK_MAT, pp.first, pp.second);
        if (gtid == 0) { flags[F_MODE] = 1; flags[F_STORED] = 1; }
        gsync();
      }
    } else {  // materialised: apply in place (from A, B at the first application)
      auto pp = views(isO, PK_MAT, nxt);
      set_factors(pp.first, pp.second, isO);
      if (need_next) set_max(pp.first, pp.second, !isO, nxt);
      run_pass(PK_MAT, pp.first, pp.second);
      if (gtid == 0) flags[F_STORED] = 1;
      gsync();
    }
    if (done) {
      if (gtid == 0 && t < a.nsteps - 1) flags[F_DONE] = 1;
      break;
    }
  }
  // extremes of the final exponents (for the root K1's two-multiply fast path)
  {
    const int32_t* ex[4] = {a.exAr, a.exAc, a.exBr, a.exBc};
    const int64_t len[4] = {M, K, K, N};
#pragma unroll 1
    for (int v = 0; v < 4; ++v) {
      int lo = 0x7fffffff, hi = -0x7fffffff - 1;
      for (int64_t i = gtid; i < len[v]; i += gstride) { lo = min(lo, ex[v][i]); hi = max(hi, ex[v][i]); }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
      }
      if ((threadIdx.x & 31) == 0) {
        atomicMin(&flags[F_EXT + 2 * v], lo);
        atomicMax(&flags[F_EXT + 2 * v + 1], hi);
      }
    }
  }
}

}  // namespace

// Launch Alg. 1-3 as one cooperative kernel.  Writes dA, dB, dI, the flags, and either the
// virtual form's exponents (flags[F_MODE] = 0 at the end: the plan's root K1 applies them) or
// A', B' into A_out / B_out (flags[F_STORED] = 1).  materialise_end = 1 forces A', B' into
// A_out / B_out.  `bar` = 4 bytes of device scratch for the grid barrier.
cudaError_t run_scaling_coop(int64_t M, int64_t K, int64_t N, const double* A, int64_t lda,
                             const double* B, int64_t ldb, double* A_out, int64_t lda_out,
                             double* B_out, int64_t ldb_out, double* dA, double* dB, double* dI,
                             int nsteps, bool first_O, double tau, int pow2, int materialise_end,
                             void* sws, cudaStream_t st) {
  ScaleWsView v = scale_ws_view(sws, M, K, N);
  cudaError_t e;
  // one memset zeroes the three maxima sets (the first pass combines into sets 0 and 1 with
  // atomicMax from its first instruction on), the factor vectors and the flags
  if ((e = cudaMemsetAsync(ws_zero_begin(v), 0, ws_zero_bytes(v), st)) != cudaSuccess) return e;
  static int blocks_per_sm = -1, sms = 0;
  if (blocks_per_sm < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_scale_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCoopSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_scale_coop, CT, kCoopSmem);
    if (blocks_per_sm > 2) blocks_per_sm = 2;
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  const int nblocks = sms * blocks_per_sm;
  CoopArgs a{};
  a.A = A; a.lda = lda; a.B = B; a.ldb = ldb;
  a.Aw = A_out; a.ldaw = lda_out; a.Bw = B_out; a.ldbw = ldb_out;
  a.M = M; a.K = K; a.N = N;
  a.dA = dA; a.dB = dB; a.dI = dI;
  a.exAr = v.ex; a.exAc = v.ex + M; a.exBr = v.ex + M + K; a.exBc = v.ex + M + 2 * K;
  a.mx[0] = v.mx[0]; a.mx[1] = v.mx[1]; a.mx[2] = v.mx[2];
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
  // reduction-only passes: about one tile per block per matrix
  auto rtiles = [&](int64_t rows, int64_t cols, int64_t* rows_per, int* segs, int* ntiles, int tgt) {
    *segs = (int)((cols + RSEG - 1) / RSEG);
    int64_t nch = std::max<int64_t>(1, tgt / *segs);
    int64_t rp = (rows + nch - 1) / nch;
    rp = std::max<int64_t>(8, (rp + 7) / 8 * 8);
    *rows_per = rp;
    *ntiles = (int)(*segs * ((rows + rp - 1) / rp));
  };
  auto ctiles = [&](int64_t rows, int64_t cols, int64_t* rows_per, int* strips, int* ntiles, int tgt) {
    *strips = (int)((cols + 255) / 256);
    int64_t nch = std::max<int64_t>(1, tgt / *strips);
    int64_t rp = (rows + nch - 1) / nch;
    rp = std::max<int64_t>(16, (rp + 15) / 16 * 16);
    *rows_per = rp;
    *ntiles = (int)(*strips * ((rows + rp - 1) / rp));
  };
  // fused A pass: whole rows (K <= FRK, 16-byte aligned).  In the fused schedule the A and the
  // B column tiles of an O-reduction pass are sized for half the blocks each, so a block streams
  // one tile per pass (one ring fill and drain) instead of two half-size ones
  static const bool small_tiles = getenv("FMM_SCALE_BIG") && atoi(getenv("FMM_SCALE_BIG")) == 0;
  const bool fuse_shape = pow2 && M > 0 && K > 0 && K <= FRK && K % 2 == 0 && lda % 2 == 0 &&
                          ((uintptr_t)A & 15u) == 0;
  static const bool no_fuse = getenv("FMM_SCALE_FUSE") && atoi(getenv("FMM_SCALE_FUSE")) == 0;
  const int half = (fuse_shape && !no_fuse && !small_tiles) ? std::max(1, nblocks / 2) : nblocks;
  // (an O-reduction pass the schedule does not fuse -- one-step runs, the last step -- pairs A's
  // row tiles with the same B column tiles, so they are sized alike; B's row tiles run alone in
  // the B-only passes)
  // (the B column tiles get a share bfrac of the blocks and A's tiles exactly the blocks left:
  // a fused A tile streams more slowly per byte -- one CTA barrier per row -- so an even split
  // leaves the B blocks waiting at the pass's end; FMM_SCALE_TRACE=2 shows the arrivals)
  static const double bfrac = getenv("FMM_SCALE_BFRAC") ? atof(getenv("FMM_SCALE_BFRAC")) : 0.45;
  const int btgt = half < nblocks ? std::max(1, (int)(nblocks * bfrac)) : nblocks;
  ctiles(M, K, &a.crowsA, &a.cstripsA, &a.ctilesA, half);
  ctiles(K, N, &a.crowsB, &a.cstripsB, &a.ctilesB, btgt);
  const int atgt = half < nblocks ? std::max(1, nblocks - a.ctilesB) : nblocks;
  rtiles(M, K, &a.rrowsA, &a.rsegsA, &a.rtilesA, atgt);
  rtiles(K, N, &a.rrowsB, &a.rsegsB, &a.rtilesB, nblocks);
  rtiles(K, N, &a.rrowsBp, &a.rsegsBp, &a.rtilesBp, half < nblocks ? std::max(1, nblocks - a.ctilesA) : nblocks);
  a.frowsA = std::max<int64_t>(1, (M + atgt - 1) / atgt);
  a.ftilesA = M > 0 ? (int)((M + a.frowsA - 1) / a.frowsA) : 0;
  static const bool no_hint = getenv("FMM_SCALE_L2HINT") && atoi(getenv("FMM_SCALE_L2HINT")) == 0;
  a.l2hint = no_hint ? 0 : 1;
  a.fuseA = (!no_fuse && fuse_shape && a.frowsA <= kTmaRows) ? 1 : 0;
  static unsigned long long* trace = nullptr;
  static const bool tracing = getenv("FMM_SCALE_TRACE") != nullptr;
  a.trace = nullptr;
  if (tracing) {  // barrier timing (development; synchronises)
    if (!trace) cudaMalloc(&trace, (64 + 64 * 512) * sizeof(unsigned long long));
    cudaMemsetAsync(trace, 0, (64 + 64 * 512) * sizeof(unsigned long long), st);
    a.trace = trace;
  }
  void* args[] = {&a};
  e = cudaLaunchCooperativeKernel((const void*)k_scale_coop, dim3((unsigned)nblocks), dim3(CT), args,
                                  kCoopSmem, st);
  if (tracing && e == cudaSuccess) {
    std::vector<unsigned long long> h(64 + 64 * 512);
    cudaMemcpyAsync(h.data(), trace, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    fprintf(stderr, "[scale] barriers (us from start):");
    for (int i = 1; i < 64 && h[i]; ++i) fprintf(stderr, " %.1f", (h[i] - h[0]) * 1e-3);
    fprintf(stderr, "\n");
    if (atoi(getenv("FMM_SCALE_TRACE")) >= 2) {  // per-block arrival at each barrier
      const int nbk = std::min(nblocks, 512);
      for (int i = 0; i < 63 && h[i + 1]; ++i) {
        std::vector<double> v;
        double lo = 0, hi = 0;
        for (int b = 0; b < nbk; ++b) {
          const double x = (h[64 + i * 512 + b] - h[0]) * 1e-3;
          v.push_back(x);
          (b < nbk / 2 ? lo : hi) += x;
        }
        std::sort(v.begin(), v.end());
        fprintf(stderr, "[scale]  barrier %2d arrivals: min %.1f p10 %.1f p50 %.1f p90 %.1f max %.1f | "
                "mean blocks < %d: %.1f, >= : %.1f\n", i + 1, v[0], v[nbk / 10], v[nbk / 2],
                v[nbk * 9 / 10], v[nbk - 1], nbk / 2, lo / (nbk / 2), hi / (nbk - nbk / 2));
      }
    }
  }
  return e;
}

// Exponent vectors and mode flag of the virtual form (for the plan's root K1).
void scale_virtual_view(void* sws, int64_t M, int64_t K, int64_t N, const int32_t** exAr,
                        const int32_t** exAc, const int32_t** exBr, const int32_t** exBc,
                        const int** mode_flag, const int** ext) {
  ScaleWsView v = scale_ws_view(sws, M, K, N);
  *exAr = v.ex; *exAc = v.ex + M; *exBr = v.ex + M + K; *exBc = v.ex + M + 2 * K;
  *mode_flag = v.flags + F_MODE;
  *ext = v.flags + F_EXT;
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
