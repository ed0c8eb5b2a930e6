// K2 (FP32, FMM_LEAF_NATIVE): batched leaf products on the FP32 FMA pipe (SIMT).
// 128 x 128 x 8 CTA tile, 256 threads, 8 x 8 register-blocked outputs per thread, register-
// staged double-buffered shared-memory tiles.  This is the plain-FP32 leaf; the tensor-core
// leaves (TF32 / 3xTF32 on tcgen05) live in kernels_gemm_tf32.cu.
#include <cstdlib>

#include "fmm_internal.h"

namespace fmm {

cudaError_t launch_gemm_tf32(const LeafNode* dev_leaves, int count, int64_t m, int64_t n,
                             int64_t k, const Bases& b, int passes, float* arena,
                             cudaStream_t st, const LeafNode* host_leaves, bool presplit);
namespace {

constexpr int BM = 128, BN = 128, BK = 8, THREADS = 256;

__global__ void __launch_bounds__(THREADS)
    k2_gemm_f32_simt(const LeafNode* __restrict__ leaves, Bases bases, int64_t m, int64_t n,
                     int64_t k, int tiles_n) {
  __shared__ float As[2][BK][BM + 4];
  __shared__ float Bs[2][BK][BN + 4];
  const LeafNode& lf = leaves[blockIdx.y];
  int64_t lda, ldb, ldc;
  const float* A = op_ptr<const float>(bases, lf.a, lda);
  const float* B = op_ptr<const float>(bases, lf.b, ldb);
  float* C = op_ptr<float>(bases, lf.c, ldc);
  const int64_t m0 = (int64_t)(blockIdx.x / tiles_n) * BM;
  const int64_t n0 = (int64_t)(blockIdx.x % tiles_n) * BN;
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;  // 16 x 16 threads, each 8 x 8 outputs

  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  // loaders: A tile 128 x 8 -> each thread 4 elements (row = tid/2, cols (tid%2)*4 .. +3)
  //          B tile 8 x 128 -> each thread 4 elements (row = tid/32, cols (tid%32)*4 .. +3)
  const int ar = tid >> 1, ac = (tid & 1) * 4;
  const int br = tid >> 5, bc = (tid & 31) * 4;
  float ra[4], rb[4];
  auto gload = [&](int64_t k0) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      int64_t gr = m0 + ar, gc = k0 + ac + e;
      ra[e] = (gr < m && gc < k) ? A[gr * lda + gc] : 0.f;
      int64_t hr = k0 + br, hc = n0 + bc + e;
      rb[e] = (hr < k && hc < n) ? B[hr * ldb + hc] : 0.f;
    }
  };
  auto sstore = [&](int buf) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      As[buf][ac + e][ar] = ra[e];
      Bs[buf][br][bc + e] = rb[e];
    }
  };
  const int KT = (int)((k + BK - 1) / BK);
  if (KT > 0) {
    gload(0);
    sstore(0);
  }
  __syncthreads();
  for (int kt = 0; kt < KT; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < KT) gload((int64_t)(kt + 1) * BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[8], bv[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = As[buf][kk][ty * 4 + i];
        a[i + 4] = As[buf][kk][64 + ty * 4 + i];
        bv[i] = Bs[buf][kk][tx * 4 + i];
        bv[i + 4] = Bs[buf][kk][64 + tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], bv[j], acc[i][j]);
    }
    if (kt + 1 < KT) sstore(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t row = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
    if (row >= m) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t col = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (col < n) C[row * ldc + col] = acc[i][j];
    }
  }
}

}  // namespace

cudaError_t launch_gemm_f32(const LeafNode* dev_leaves, const LeafNode* host_leaves, int count,
                            int64_t m, int64_t n, int64_t k, const Bases& b, bool vec, int leaf,
                            float* arena, cudaStream_t st, bool presplit) {
  (void)vec;
  if (count == 0 || m == 0 || n == 0) return cudaSuccess;
  if (leaf == FMM_LEAF_TF32 || leaf == FMM_LEAF_3XTF32) {
    const int passes = leaf == FMM_LEAF_TF32 ? 1 : 3;
    return launch_gemm_tf32(dev_leaves, count, m, n, k, b, passes, arena, st, host_leaves, presplit);
  }
  const int tiles_m = (int)((m + BM - 1) / BM), tiles_n = (int)((n + BN - 1) / BN);
  dim3 grid((unsigned)(tiles_m * tiles_n), (unsigned)count);
  k2_gemm_f32_simt<<<grid, THREADS, 0, st>>>(dev_leaves, b, m, n, k, tiles_n);
  return cudaGetLastError();
}

}  // namespace fmm
