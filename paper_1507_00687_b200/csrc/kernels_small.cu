// Single-launch small plans: a two-level plan whose steps are one K1X2 pass
// (levels 0-1 of S / T formation), one batched leaf GEMM and one K3X2 pass (levels 1-0 of the
// W-combination) -- BASELINE config C1, S-W L = 2 at 512^3 -- runs as ONE cooperative kernel
// with the three phases separated by grid-wide barriers.  At this size every pass touches a few
// MB that live in L2, so three launches cost more than their work (round 1: 38 us per step for a
// 9 us pipeline roofline); one launch removes two launch / drain boundaries and lets the leaf
// phase use a finer decomposition than the stand-alone K2 (32 x 64 output tiles, 784 work items
// at C1, about one wave of 3 CTAs per SM).
//
// Arithmetic is unchanged, element by element: phase 1 runs k1x2_row (K1X2's sequential sums),
// phase 2 accumulates every leaf element over k ascending in groups of 4 with the same
// m16n8k4 DMMA chain as k2_gemm_f64 (any tile shape gives each element the same chain), and
// phase 3 runs k3x2_row.  So the result is bitwise the three-launch schedule's
// (tests/test_gpu_small.py).  Data produced inside the kernel is read with L2-only loads
// (cp.async.cg, ld.global.cg).
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include <cooperative_groups.h>

#include "fmm_internal.h"
#include "gemm_f64_dev.cuh"
#include "lincomb_dev.cuh"

namespace fmm {

namespace cg = cooperative_groups;

namespace {

using SCfg = Cfg<32, 64, 16, 4, 2, 2, 3, true>;  // 4 warps of 16 x 32, 4 stages, 3 CTAs / SM
constexpr int kSmallThreads = SCfg::THREADS;      // 128

struct SmallArgs {
  const K1x2Node* k1;
  int nk1;
  const LeafNode* lf;
  int nlf;
  int64_t m, n, k;
  int tiles_m, tiles_n;
  const K3x2Node* k3;
  int nk3;
  Bases b;
  unsigned long long* trace;  // FMM_SMALL_TRACE: %globaltimer at the phase boundaries (block 0)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}


// One 32 x 64 tile of M = S T (m x k by k x n), full k, the PIPE mainloop of k2_gemm_f64.
template <bool VEC>
__device__ __forceinline__ void leaf_tile(double* As, double* Bs, const double* A, int64_t lda,
                                          const double* B, int64_t ldb, double* Cp, int64_t ldc,
                                          int64_t m, int64_t n, int64_t k, int64_t m0, int64_t n0) {
  using C = SCfg;
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
  constexpr int KQ = C::BK / 4;
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
      load_tiles<C, VEC>(As + (nk % C::STAGES) * C::A_STAGE, Bs + (nk % C::STAGES) * C::B_STAGE, A,
                         lda, B, ldb, m, n, k, m0, n0, (int64_t)nk * C::BK, tid);
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
        __syncthreads();
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
  cp_wait<0>();
  __syncthreads();  // the next tile reuses the stages
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

template <int RA, int RB, bool VEC>
__global__ void __launch_bounds__(kSmallThreads, 3) k_small_plan(SmallArgs a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ double* optr[2][kMaxX2];
  constexpr int V = VEC ? 2 : 1;
  const unsigned int nb = gridDim.x;
  // grid-wide barrier of the cooperative launch (orders global memory and invalidates L1)
  cg::grid_group grid = cg::this_grid();
  // phases 1 and 3 are few, long items (a row position of a two-level pass): warps are striped
  // across the blocks first so the items spread over every SM
  const int64_t gt = ((int64_t)(threadIdx.x >> 5) * nb + blockIdx.x) * 32 + (threadIdx.x & 31);
  const int64_t gs = (int64_t)nb * kSmallThreads;
  if (a.trace && gt == 0) a.trace[0] = gtimer();
  // Descriptor prefetch: the operand pointers of this block's first leaf tile (phase 2) and the
  // input pointers of a single K3X2 node (phase 3) are resolved now, by warp 3 (which has no
  // phase-1 item at C1's sizes), so their dependent global loads overlap phase 1 instead of
  // starting after the barriers.
  __shared__ const double* s_pa;
  __shared__ const double* s_pb;
  __shared__ double* s_pc;
  __shared__ int64_t s_ld[3];
  __shared__ const double* s_k3in[kMaxX2];
  constexpr int NIN = builtin_R(RA) * builtin_R(RB);
  const int tiles = a.tiles_m * a.tiles_n;
  if ((threadIdx.x >> 5) == 3) {
    const int lane = threadIdx.x & 31;
    if (lane == 0 && (int)blockIdx.x < a.nlf * tiles) {
      const LeafNode& lf = a.lf[blockIdx.x / tiles];
      s_pa = op_ptr<const double>(a.b, lf.a, s_ld[0]);
      s_pb = op_ptr<const double>(a.b, lf.b, s_ld[1]);
      s_pc = op_ptr<double>(a.b, lf.c, s_ld[2]);
    }
    if (a.nk3 == 1)
      for (int q = lane; q < NIN; q += 32) {
        int64_t l;
        s_k3in[q] = op_ptr<const double>(a.b, a.k3[0].in[q], l);
      }
  }
  // ---- phase 1: S / T of levels 0 and 1 (K1X2), both nodes' items in one index space ------
  {
    for (int q = 0; q < a.nk1; ++q)
      if (threadIdx.x < a.k1[q].nout) {
        int64_t l;
        optr[q][threadIdx.x] = op_ptr<double>(a.b, a.k1[q].out[threadIdx.x], l);
      }
    __syncthreads();
    const int64_t n0 = a.nk1 > 0 ? a.k1[0].rows * (a.k1[0].cols / V) : 0;
    const int64_t n1 = a.nk1 > 1 ? a.k1[1].rows * (a.k1[1].cols / V) : 0;
    for (int64_t it = gt; it < n0 + n1; it += gs) {
      const int q = it < n0 ? 0 : 1;
      const K1x2Node& nd = a.k1[q];
      const int64_t cv = nd.cols / V, li = q ? it - n0 : it;
      const int64_t i = li / cv, jv = (li % cv) * V;
      int64_t ldi;
      const double* in = op_ptr<const double>(a.b, nd.in, ldi);
      if (nd.tv == 0) k1x2_row<double, V, RA, RB, 0>(in, ldi, nd.rows, nd.cols, i, jv, optr[q]);
      else k1x2_row<double, V, RA, RB, 1>(in, ldi, nd.rows, nd.cols, i, jv, optr[q]);
    }
  }
  if (a.trace && threadIdx.x == 0) atomicMax(&a.trace[1], gtimer());
  grid.sync();
  if (a.trace && gt == 0) a.trace[2] = gtimer();
  // ---- phase 2: every leaf product M = S T, 32 x 64 tiles ----------------------------------
  {
    double* As = smem;
    double* Bs = smem + SCfg::STAGES * SCfg::A_STAGE;
    for (int w = blockIdx.x; w < a.nlf * tiles; w += nb) {
      const int tile = w % tiles;
      int64_t lda, ldb, ldc;
      const double* A;
      const double* B;
      double* Cp;
      if (w == (int)blockIdx.x) {  // prefetched
        A = s_pa; B = s_pb; Cp = s_pc;
        lda = s_ld[0]; ldb = s_ld[1]; ldc = s_ld[2];
      } else {
        const LeafNode& lf = a.lf[w / tiles];
        A = op_ptr<const double>(a.b, lf.a, lda);
        B = op_ptr<const double>(a.b, lf.b, ldb);
        Cp = op_ptr<double>(a.b, lf.c, ldc);
      }
      leaf_tile<VEC>(As, Bs, A, lda, B, ldb, Cp, ldc, a.m, a.n, a.k,
                     (int64_t)(tile / a.tiles_n) * SCfg::BM, (int64_t)(tile % a.tiles_n) * SCfg::BN);
    }
  }
  if (a.trace && threadIdx.x == 0) atomicMax(&a.trace[3], gtimer());
  grid.sync();
  if (a.trace && gt == 0) a.trace[4] = gtimer();
  // ---- phase 3: the W-combination of levels 1 and 0 (K3X2) ---------------------------------
  for (int q = 0; q < a.nk3; ++q) {
    const K3x2Node& nd = a.k3[q];
    const double* const* iptr = a.nk3 == 1 ? s_k3in : optr[0];
    if (a.nk3 != 1) {
      __syncthreads();
      if (threadIdx.x < NIN) {
        int64_t l;
        optr[0][threadIdx.x] = op_ptr<double>(a.b, nd.in[threadIdx.x], l);
      }
      __syncthreads();
    }
    int64_t ldo;
    double* out = op_ptr<double>(a.b, nd.out, ldo);
    const int64_t cv = nd.cols / V;
    for (int64_t it = gt; it < nd.rows * cv; it += gs) {
      const int64_t i = it / cv, jv = (it % cv) * V;
      k3x2_row<double, V, RA, RB, false, true>(iptr, out, ldo, nd.rows, nd.cols, i, jv);
    }
  }
  if (a.trace) {
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(&a.trace[5], gtimer());
  }
}

template <int RA, int RB, bool VEC>
cudaError_t go_small(const SmallArgs& a, cudaStream_t st) {
  constexpr int smem = SCfg::SMEM_BYTES;
  auto kern = k_small_plan<RA, RB, VEC>;
  static int blocks = -1;
  if (blocks < 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                               (int)cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, kSmallThreads, smem);
    blocks = sms * std::max(1, std::min(per, 3));
  }
  cudaError_t e = cudaSuccess;
  SmallArgs args = a;
  static unsigned long long* trace = nullptr;
  static const bool tracing = getenv("FMM_SMALL_TRACE") != nullptr;
  if (tracing) {  // phase timing (development; synchronises)
    if (!trace) cudaMalloc(&trace, 8 * sizeof(unsigned long long));
    cudaMemsetAsync(trace, 0, 8 * sizeof(unsigned long long), st);
    args.trace = trace;
  }
  void* p[] = {&args};
  e = cudaLaunchCooperativeKernel((const void*)kern, dim3((unsigned)blocks), dim3(kSmallThreads), p,
                                  smem, st);
  if (tracing && e == cudaSuccess) {
    unsigned long long h[8];
    cudaMemcpyAsync(h, trace, sizeof h, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    fprintf(stderr, "[small] phase1 %.2f us (+barrier %.2f) phase2 %.2f us (+barrier %.2f) phase3 %.2f us\n",
            (h[1] - h[0]) * 1e-3, (h[2] - h[1]) * 1e-3, (h[3] - h[2]) * 1e-3, (h[4] - h[3]) * 1e-3,
            (h[5] - h[4]) * 1e-3);
  }
  return e;
}

}  // namespace

int small_tile_m() { return SCfg::BM; }
int small_tile_n() { return SCfg::BN; }

cudaError_t launch_small_plan(int pair, const K1x2Node* k1, int nk1, const LeafNode* lf, int nlf,
                              int64_t m, int64_t n, int64_t k, const K3x2Node* k3, int nk3,
                              const Bases& b, bool vec, cudaStream_t st) {
  SmallArgs a{};
  a.k1 = k1; a.nk1 = nk1; a.lf = lf; a.nlf = nlf; a.m = m; a.n = n; a.k = k;
  a.tiles_m = (int)((m + SCfg::BM - 1) / SCfg::BM);
  a.tiles_n = (int)((n + SCfg::BN - 1) / SCfg::BN);
  a.k3 = k3; a.nk3 = nk3; a.b = b;
#define FMM_SMALL(RA, RB) return vec ? go_small<RA, RB, true>(a, st) : go_small<RA, RB, false>(a, st)
  switch (pair - 1) {
    case 0: FMM_SMALL(0, 0);
    case 1: FMM_SMALL(0, 1);
    case 2: FMM_SMALL(0, 2);
    case 3: FMM_SMALL(1, 0);
    case 4: FMM_SMALL(1, 1);
    case 5: FMM_SMALL(1, 2);
    case 6: FMM_SMALL(2, 0);
    case 7: FMM_SMALL(2, 1);
    default: FMM_SMALL(2, 2);
  }
#undef FMM_SMALL
}

}  // namespace fmm
