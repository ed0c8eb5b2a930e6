// Device-side building blocks of the FP64 DMMA leaf GEMM (tile configuration, cp.async
// staging, the m16n8k4 fragment MMA, the RED.ADD epilogue), shared by kernels_gemm_f64.cu and
// kernels_small.cu.  Everything lives in fmm::{anonymous}.
#pragma once
#include <cstdint>

#include "fmm_internal.h"

namespace fmm {
namespace {


constexpr int GROUP_M = 8;

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


__device__ __forceinline__ void red_add(double* p, double v) {
  asm volatile("red.global.add.f64 [%0], %1;\n" ::"l"(p), "d"(v) : "memory");
}

}  // namespace
}  // namespace fmm
