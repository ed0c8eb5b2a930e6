// FP64 pipe microbenchmark for B200 (sm_100a): DMMA (mma.sync f64 shapes) vs DFMA.
// Register-only loops with many independent accumulators; reports TFLOP/s.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int NACC>
__global__ void k_dmma_884(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
__global__ void k_dmma_16816(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + (threadIdx.x + i) * 1e-9;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - (threadIdx.x + i) * 1e-9;
  double c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
__global__ void k_dmma_1684(double* out, int iters) {
  double a0 = 1.0 + threadIdx.x * 1e-9, a1 = 1.0 + threadIdx.x * 2e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
__global__ void k_dfma(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
static float time_it(F launch, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch();
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("device %s SMs %d\n", p.name, p.multiProcessorCount);
  double* out; CK(cudaMalloc(&out, 148 * 64 * 1024 * sizeof(double)));
  const int sms = p.multiProcessorCount;
  for (int warps : {4, 8, 16}) {
    for (int ctas_per_sm : {1, 2}) {
      int grid = sms * ctas_per_sm, block = 32 * warps, iters = 4096;
      double nthr = (double)grid * block;
      float ms;
      ms = time_it([&] { k_dmma_884<8><<<grid, block>>>(out, iters); }, 5);
      printf("DMMA m8n8k4   acc=8  warps=%2d cta/sm=%d: %.2f TFLOP/s\n", warps, ctas_per_sm,
             nthr / 32 * iters * 8 * 512.0 / (ms * 1e-3) / 1e12);
      ms = time_it([&] { k_dmma_1684<8><<<grid, block>>>(out, iters); }, 5);
      printf("DMMA m16n8k4  acc=8  warps=%2d cta/sm=%d: %.2f TFLOP/s\n", warps, ctas_per_sm,
             nthr / 32 * iters * 8 * 1024.0 / (ms * 1e-3) / 1e12);
      ms = time_it([&] { k_dmma_16816<4><<<grid, block>>>(out, iters / 4); }, 5);
      printf("DMMA m16n8k16 acc=4  warps=%2d cta/sm=%d: %.2f TFLOP/s\n", warps, ctas_per_sm,
             nthr / 32 * (iters / 4) * 4 * 4096.0 / (ms * 1e-3) / 1e12);
      ms = time_it([&] { k_dfma<16><<<grid, block>>>(out, iters); }, 5);
      printf("DFMA          acc=16 warps=%2d cta/sm=%d: %.2f TFLOP/s\n", warps, ctas_per_sm,
             nthr * iters * 16 * 2.0 / (ms * 1e-3) / 1e12);
    }
  }
  // sustained: DMMA for ~4 s
  {
    int grid = sms * 2, block = 256, iters = 4096;
    double nthr = (double)grid * block;
    float ms = time_it([&] { k_dmma_1684<8><<<grid, block>>>(out, iters); }, 400);
    printf("sustained DMMA m16n8k4 (%d reps): %.2f TFLOP/s\n", 400, nthr / 32 * iters * 8 * 1024.0 / (ms * 1e-3) / 1e12);
    ms = time_it([&] { k_dfma<16><<<grid, block>>>(out, iters); }, 400);
    printf("sustained DFMA (%d reps): %.2f TFLOP/s\n", 400, nthr * iters * 16 * 2.0 / (ms * 1e-3) / 1e12);
  }
  CK(cudaGetLastError());
  return 0;
}
