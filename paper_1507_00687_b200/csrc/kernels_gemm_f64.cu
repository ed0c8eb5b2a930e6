// K2 (FP64): batched leaf products M = S.T on the FP64 tensor path of sm_100a.
//
// sm_100a's tcgen05.mma has no f64 kind; FP64 tensor math is the warp-level DMMA
// (mma.sync .f64 -> SASS DMMA.8x8x4), measured at 36.9 TFLOP/s on this pool's B200s
// (profiles/r01_fp64_peak_microbench.txt; DFMA reaches 33.7).  Design:
//   * CTA tile 128 x 128 x 16, 8 warps (2 x 4), warp tile 64 x 32 = 4 x 4 m16n8k4 fragments,
//     64 fp64 accumulators per thread;
//   * 4-stage cp.async (16-byte, L2-only .cg) pipeline global -> shared; shared rows padded
//     (+4 doubles) so the 8-byte fragment loads of each half-warp hit 16 distinct bank pairs;
//   * batched over the leaves of a level by grid.y with per-leaf operand descriptors;
//     grouped rasterisation (8 tile-rows) inside a leaf for L2 reuse;
//   * ragged edges handled by zero-fill (src-size 0) loads and guarded stores; a scalar
//     (8-byte) load path serves operands whose ld / offsets are not 16-byte aligned.
// The leaf's k-order is the tensor core's (reading A4): not the oracle's
// sequential order, covered by the parity tolerance.
#include <cstdint>

#include "fmm_internal.h"

namespace fmm {

namespace {

constexpr int BM = 128, BN = 128, BK = 16, STAGES = 4, THREADS = 256;
constexpr int A_LD = BK + 4;  // 20 doubles per smem row of the A tile
constexpr int B_LD = BN + 4;  // 132 doubles per smem row of the B tile
constexpr int A_STAGE = BM * A_LD;
constexpr int B_STAGE = BK * B_LD;
constexpr int SMEM_BYTES = STAGES * (A_STAGE + B_STAGE) * 8;
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

template <bool VEC>
__device__ __forceinline__ void load_tiles(double* As, double* Bs, const double* A, int64_t lda,
                                           const double* B, int64_t ldb, int64_t m, int64_t n,
                                           int64_t k, int64_t m0, int64_t n0, int64_t k0,
                                           int tid) {
  if constexpr (VEC) {
    // A tile: 128 rows x 16 doubles = 1024 chunks of 16 B
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int c = tid + q * THREADS;
      int row = c >> 3, cc = (c & 7) * 2;
      int64_t gr = m0 + row, gc = k0 + cc;
      bool ok = gr < m && gc < k;
      const double* src = ok ? A + gr * lda + gc : A;
      cp16(smem_u32(As + row * A_LD + cc), src, ok);
    }
    // B tile: 16 rows x 128 doubles
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int c = tid + q * THREADS;
      int row = c >> 6, cc = (c & 63) * 2;
      int64_t gr = k0 + row, gc = n0 + cc;
      bool ok = gr < k && gc < n;
      const double* src = ok ? B + gr * ldb + gc : B;
      cp16(smem_u32(Bs + row * B_LD + cc), src, ok);
    }
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      int c = tid + q * THREADS;
      int row = c >> 4, cc = c & 15;
      int64_t gr = m0 + row, gc = k0 + cc;
      bool ok = gr < m && gc < k;
      cp8(smem_u32(As + row * A_LD + cc), ok ? A + gr * lda + gc : A, ok);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      int c = tid + q * THREADS;
      int row = c >> 7, cc = c & 127;
      int64_t gr = k0 + row, gc = n0 + cc;
      bool ok = gr < k && gc < n;
      cp8(smem_u32(Bs + row * B_LD + cc), ok ? B + gr * ldb + gc : B, ok);
    }
  }
}

template <bool VEC>
__global__ void __launch_bounds__(THREADS, 1)
    k2_gemm_f64(const LeafNode* __restrict__ leaves, Bases bases, int64_t m, int64_t n,
                int64_t k, int tiles_m, int tiles_n) {
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * A_STAGE;

  const LeafNode& lf = leaves[blockIdx.y];
  int64_t lda, ldb, ldc;
  const double* A = op_ptr<const double>(bases, lf.a, lda);
  const double* B = op_ptr<const double>(bases, lf.b, ldb);
  double* C = op_ptr<double>(bases, lf.c, ldc);

  // grouped rasterisation
  const int tile = blockIdx.x;
  const int per_group = GROUP_M * tiles_n;
  const int group = tile / per_group;
  const int first_m = group * GROUP_M;
  const int gsz = min(tiles_m - first_m, GROUP_M);
  const int tm = first_m + (tile % per_group) % gsz;
  const int tn = (tile % per_group) / gsz;
  const int64_t m0 = (int64_t)tm * BM, n0 = (int64_t)tn * BN;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 2, wn = warp & 3;  // 2 x 4 warps
  const int g = lane >> 2, t = lane & 3;

  double acc[4][4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;

  const int KT = (int)((k + BK - 1) / BK);
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_tiles<VEC>(As + s * A_STAGE, Bs + s * B_STAGE, A, lda, B, ldb, m, n, k, m0,
                                n0, (int64_t)s * BK, tid);
    cp_commit();
  }

  for (int kt = 0; kt < KT; ++kt) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    {
      int nk = kt + STAGES - 1;
      if (nk < KT) {
        int slot = nk % STAGES;
        load_tiles<VEC>(As + slot * A_STAGE, Bs + slot * B_STAGE, A, lda, B, ldb, m, n, k, m0,
                        n0, (int64_t)nk * BK, tid);
      }
      cp_commit();
    }
    const int slot = kt % STAGES;
    const double* as = As + slot * A_STAGE + (wm * 64 + g) * A_LD + t;
    const double* bs = Bs + slot * B_STAGE + t * B_LD + wn * 32 + g;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4][2], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        af[i][0] = as[(i * 16) * A_LD + kk];
        af[i][1] = as[(i * 16 + 8) * A_LD + kk];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = bs[kk * B_LD + j * 8];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma16n8k4(acc[i][j], af[i][0], af[i][1], bf[j]);
    }
  }
  cp_wait<0>();

  // epilogue: c0,c1 at (row g, cols 2t, 2t+1); c2,c3 at row g+8
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t row = m0 + wm * 64 + i * 16 + g + h * 8;
      if (row >= m) continue;
      double* crow = C + row * ldc;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t col = n0 + wn * 32 + j * 8 + 2 * t;
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

}  // namespace

cudaError_t launch_gemm_f64(const LeafNode* dev_leaves, int count, int64_t m, int64_t n,
                            int64_t k, const Bases& b, bool vec, cudaStream_t st) {
  if (count == 0 || m == 0 || n == 0) return cudaSuccess;
  const int tiles_m = (int)((m + BM - 1) / BM), tiles_n = (int)((n + BN - 1) / BN);
  dim3 grid((unsigned)(tiles_m * tiles_n), (unsigned)count);
  cudaError_t e;
  if (vec) {
    e = cudaFuncSetAttribute(k2_gemm_f64<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             SMEM_BYTES);
    if (e != cudaSuccess) return e;
    k2_gemm_f64<true><<<grid, THREADS, SMEM_BYTES, st>>>(dev_leaves, b, m, n, k, tiles_m, tiles_n);
  } else {
    e = cudaFuncSetAttribute(k2_gemm_f64<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             SMEM_BYTES);
    if (e != cudaSuccess) return e;
    k2_gemm_f64<false><<<grid, THREADS, SMEM_BYTES, st>>>(dev_leaves, b, m, n, k, tiles_m, tiles_n);
  }
  return cudaGetLastError();
}

}  // namespace fmm
