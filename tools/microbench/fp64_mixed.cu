// Do DMMA (mma.sync f64) and DFMA share one FP64 pipe on sm_100a?  Warps of one CTA split into
// a DMMA group and a DFMA group running register-only loops concurrently; the combined FLOP/s
// against each alone answers it (a sum near one pipe's peak = shared; near the sum of both
// peaks = separate units).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_mixed fp64_mixed.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_mixed(double* out, int iters_mma, int iters_fma, int mma_warps) {
  const int warp = threadIdx.x >> 5;
  if (warp < mma_warps) {
    double a0 = 1.0 + threadIdx.x * 1e-9, a1 = 1.0 + threadIdx.x * 2e-9, b = 1.0 - threadIdx.x * 1e-9;
    double c[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0;
    for (int it = 0; it < iters_mma; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  } else {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double c[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = i;
    for (int it = 0; it < iters_fma; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i) c[i] = fma(a, c[i], b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += c[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  }
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  double* out;
  cudaMalloc(&out, (size_t)sms * 2 * 1024 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int warps = 16, grid = sms * 2;
  // flops per warp-iteration: DMMA 8 x m16n8k4 = 8 * 1024; DFMA 32 threads x 16 x 2 = 1024
  for (int mw : {16, 0, 8, 12, 4}) {
    for (int fma_scale : {1, 2, 4}) {
      const int im = 2048, jf = (mw == 16) ? 0 : 2048 * fma_scale;
      auto run = [&] { k_mixed<<<grid, warps * 32>>>(out, im, jf, mw); };
      run();
      cudaDeviceSynchronize();
      cudaEventRecord(e0);
      for (int r = 0; r < 10; ++r) run();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 10;
      const double fl_mma = (double)grid * mw * im * 8 * 1024.0;
      const double fl_fma = (double)grid * (warps - mw) * jf * 1024.0;
      printf("dmma warps %2d / dfma warps %2d (dfma iters x%d): %.3f ms  DMMA %.2f + DFMA %.2f = %.2f TFLOP/s\n",
             mw, warps - mw, fma_scale, ms, fl_mma / ms / 1e9, fl_fma / ms / 1e9,
             (fl_mma + fl_fma) / ms / 1e9);
      if (mw == 16) break;
    }
  }
  return 0;
}
