// FP32 SIMT (FFMA) peak on this B200 -- context for the FP32 leaf's roofline (SURVEY §8(d):
// "also report the FP32 SIMT (FFMA) peak").  Register-only FMA chains, 16 independent per thread.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ffma_peak ffma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_ffma(float* out, int iters) {
  float a = 1.0f + threadIdx.x * 1e-7f, b = 1.0f - threadIdx.x * 1e-7f;
  float c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = (float)i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = fmaf(a, c[i], b);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  float* out;
  cudaMalloc(&out, (size_t)sms * 4 * 1024 * sizeof(float));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int ctas : {2, 4}) {
    const int grid = sms * ctas, block = 512, iters = 8192;
    k_ffma<<<grid, block>>>(out, iters);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) k_ffma<<<grid, block>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 10;
    const double fl = (double)grid * block * iters * 16 * 2.0;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("FFMA ctas/sm=%d: %.1f TFLOP/s (%.3f ms)\n", ctas, fl / ms / 1e9, ms);
  }
  return 0;
}
