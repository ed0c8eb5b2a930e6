// Read-stream microbenchmark (development evidence for DESIGN.md §6.4): max |x| over a 256 MB
// FP64 buffer (4096 rows of 8192 doubles, the C4 A + B size), L2 flushed before every launch,
// timed with CUDA events.  Variants:
//   ldg_full   : LDG.128 grid-stride, 1024 threads / SM (8 x 128-thread CTAs), 4 loads in flight
//   ldg_ours   : LDG.128, 2 x 256-thread CTAs / SM (the scaling kernel's occupancy), 8 in flight
//   warp_ring  : per-warp cp.async.bulk rings, CS x 4 KB (the scaling kernel's row / column tiles)
//   cta_ring   : one ring per CTA of CS row stages of RB KB, one bulk copy per stage (the fused pass)
// each after a dirty flush (512 MB memset: L2 write-backs compete) and a clean one (512 MB read)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o read_stream read_stream.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ unsigned long long g_max;

__device__ __forceinline__ void fold(double v) {
  double m = v;
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(&g_max, (unsigned long long)__double_as_longlong(m));
}

template <int U>
__global__ void ldg_stream(const double2* __restrict__ x, int64_t n2) {
  double m = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n2; i += U * stride) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = x[i + u * stride];
#pragma unroll
    for (int u = 0; u < U; ++u) m = fmax(m, fmax(fabs(v[u].x), fabs(v[u].y)));
  }
  for (; i < n2; i += stride) m = fmax(m, fmax(fabs(x[i].x), fabs(x[i].y)));
  fold(m);
}

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(s32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(s32(dst)), "l"(src), "r"(bytes), "r"(s32(bar)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t par) {
  uint32_t done = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(s32(bar)), "r"(par) : "memory");
  } while (!done);
}

// per-warp rings: the buffer as chunks of 4 KB; warp w of the grid takes chunks w, w + W, ...
template <int CS>
__global__ void warp_ring(const double* x, int64_t nchunks) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double* buf = reinterpret_cast<double*>(sm) + (size_t)warp * CS * 512;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + (size_t)nw * CS * 4096) + warp * CS;
  if (lane < CS) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(s32(bar + lane)));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncwarp();
  const int64_t gw = (int64_t)blockIdx.x * nw + warp, W = (int64_t)gridDim.x * nw;
  const int n = gw < nchunks ? (int)((nchunks - 1 - gw) / W + 1) : 0;
  if (lane == 0)
    for (int k = 0; k < CS && k < n; ++k) bulk(buf + k * 512, x + (gw + k * W) * 512, 4096, bar + k);
  double m = 0.0;
  uint32_t ph = 0;
  for (int k = 0; k < n; ++k) {
    const int st = k % CS;
    wait(bar + st, (ph >> st) & 1u);
    ph ^= 1u << st;
    const double* b = buf + st * 512;
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      const double2 v = *reinterpret_cast<const double2*>(b + h * 64 + 2 * lane);
      m = fmax(m, fmax(fabs(v.x), fabs(v.y)));
    }
    __syncwarp();
    if (lane == 0 && k + CS < n) bulk(buf + st * 512, x + (gw + (k + CS) * W) * 512, 4096, bar + st);
  }
  fold(m);
}

// per-warp rings over the scaling kernel's row tiles: the buffer as 4096 rows x 8 segments of
// 4 KB; tile = (row chunk, segment), CTA b takes tile b, warp w rows r0 + w + 8 k of it
template <int CS>
__global__ void warp_ring_rowtiles(const double* x, int rows, int segs, int rows_per) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double* buf = reinterpret_cast<double*>(sm) + (size_t)warp * CS * 512;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + (size_t)nw * CS * 4096) + warp * CS;
  if (lane < CS) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(s32(bar + lane)));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncwarp();
  const int seg = blockIdx.x % segs, r0 = (blockIdx.x / segs) * rows_per;
  const int r1 = min(r0 + rows_per, rows);
  const int rw = r0 + warp;
  const int n = rw < r1 ? (r1 - rw + nw - 1) / nw : 0;
  auto src = [&](int k) { return x + (size_t)(rw + nw * k) * segs * 512 + seg * 512; };
  if (lane == 0)
    for (int k = 0; k < CS && k < n; ++k) bulk(buf + k * 512, src(k), 4096, bar + k);
  double m = 0.0;
  uint32_t ph = 0;
  for (int k = 0; k < n; ++k) {
    const int st = k % CS;
    wait(bar + st, (ph >> st) & 1u);
    ph ^= 1u << st;
    const double* b = buf + st * 512;
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      const double2 v = *reinterpret_cast<const double2*>(b + h * 64 + 2 * lane);
      m = fmax(m, fmax(fabs(v.x), fabs(v.y)));
    }
    __syncwarp();
    if (lane == 0 && k + CS < n) bulk(buf + st * 512, src(k + CS), 4096, bar + st);
  }
  fold(m);
}

// CTA rings: the buffer as rows of RB bytes; CTA b takes rows b, b + G, ...
template <int CS>
__global__ void cta_ring(const double* x, int64_t nrows, int rb) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int rd = rb / 8;
  double* ring = reinterpret_cast<double*>(sm);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + (size_t)CS * rb);
  if (threadIdx.x < CS) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(s32(bar + threadIdx.x)));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  const int64_t G = gridDim.x;
  const int n = blockIdx.x < nrows ? (int)((nrows - 1 - blockIdx.x) / G + 1) : 0;
  if (threadIdx.x == 0)
    for (int k = 0; k < CS && k < n; ++k) bulk(ring + (size_t)k * rd, x + (blockIdx.x + k * G) * rd, rb, bar + k);
  double m = 0.0;
  uint32_t ph = 0;
  for (int k = 0; k < n; ++k) {
    const int st = k % CS;
    wait(bar + st, (ph >> st) & 1u);
    ph ^= 1u << st;
    const double* b = ring + (size_t)st * rd;
    for (int j = 2 * threadIdx.x; j < rd; j += 2 * blockDim.x) {
      const double2 v = *reinterpret_cast<const double2*>(b + j);
      m = fmax(m, fmax(fabs(v.x), fabs(v.y)));
    }
    __syncthreads();
    if (threadIdx.x == 0 && k + CS < n) bulk(ring + (size_t)st * rd, x + (blockIdx.x + (k + CS) * G) * rd, rb, bar + st);
  }
  fold(m);
}

int main() {
  const int64_t nd = (int64_t)4096 * 8192;  // 256 MB of doubles
  const size_t bytes = nd * 8;
  double* x;
  uint8_t* fl;
  CK(cudaMalloc(&x, bytes));
  CK(cudaMalloc(&fl, 512u << 20));
  CK(cudaMemset(x, 0x3f, bytes));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  bool clean = false;
  auto timeit = [&](const char* name, auto launch) {
    float best = 1e9, tot = 0;
    const int reps = 10;
    for (int r = 0; r < reps + 2; ++r) {
      if (clean) ldg_stream<4><<<sms * 8, 128>>>((const double2*)fl, (512 << 20) / 16);  // clean L2
      else cudaMemsetAsync(fl, r, 512u << 20);                                         // dirty L2
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 2) { tot += ms; best = ms < best ? ms : best; }
    }
    cudaError_t e = cudaGetLastError();
    printf("%s %-34s %7.1f us avg %7.1f us best  %6.0f GB/s avg  %s\n", clean ? "clean" : "dirty", name, tot / reps * 1e3, best * 1e3,
           bytes / (tot / reps) / 1e6, e == cudaSuccess ? "" : cudaGetErrorString(e));
    (void)0;
  };
  CK(cudaMemset(fl, 0, 512u << 20));
  for (int pass = 0; pass < 2; ++pass) {
  clean = pass == 1;
  timeit("ldg_full (8 x 128 thr / SM, U4)", [&] { ldg_stream<4><<<sms * 8, 128>>>((const double2*)x, nd / 2); });
  timeit("ldg_full (8 x 128 thr / SM, U8)", [&] { ldg_stream<8><<<sms * 8, 128>>>((const double2*)x, nd / 2); });
  timeit("ldg_ours (2 x 256 thr / SM, U8)", [&] { ldg_stream<8><<<sms * 2, 256>>>((const double2*)x, nd / 2); });
  timeit("ldg_ours (2 x 256 thr / SM, U16)", [&] { ldg_stream<16><<<sms * 2, 256>>>((const double2*)x, nd / 2); });
  {
    const int smem3 = 8 * 3 * 4096 + 8 * 3 * 8;
    cudaFuncSetAttribute(warp_ring<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem3);
    timeit("warp_ring CS3 (2 x 8 warps / SM)", [&] { warp_ring<3><<<sms * 2, 256, smem3>>>(x, nd / 512); });
    const int smem6 = 8 * 6 * 4096 + 8 * 6 * 8;
    cudaFuncSetAttribute(warp_ring<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem6);
    timeit("warp_ring CS6 (1 x 8 warps / SM)", [&] { warp_ring<6><<<sms, 256, smem6>>>(x, nd / 512); });
    const int smem3b = 4 * 3 * 4096 + 4 * 3 * 8;
    cudaFuncSetAttribute(warp_ring<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem3);
    timeit("warp_ring CS3 (4 x 4 warps / SM)", [&] { warp_ring<3><<<sms * 4, 128, smem3b>>>(x, nd / 512); });
  }
  {
    const int smem3 = 8 * 3 * 4096 + 8 * 3 * 8;
    cudaFuncSetAttribute(warp_ring_rowtiles<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem3);
    // 4096 rows x 8 segments: rows_per 112 -> 37 chunks x 8 = 296 tiles (the kernel's B row tiles)
    timeit("warp_ring row tiles (4 KB @ 32 KB)", [&] { warp_ring_rowtiles<3><<<37 * 8, 256, smem3>>>(x, 4096, 8, 112); });
  }
  for (int rb : {8192, 16384, 32768}) {
    const int smem = 3 * rb + 64;
    cudaFuncSetAttribute(cta_ring<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    char nm[64];
    snprintf(nm, sizeof nm, "cta_ring CS3 x %2d KB (2 / SM)", rb / 1024);
    timeit(nm, [&] { cta_ring<3><<<sms * 2, 256, smem>>>(x, nd * 8 / rb, rb); });
  }
  {
    const int rb = 16384, smem = 6 * rb + 64;
    cudaFuncSetAttribute(cta_ring<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    timeit("cta_ring CS6 x 16 KB (2 / SM)", [&] { cta_ring<6><<<sms * 2, 256, smem>>>(x, nd * 8 / rb, rb); });
  }
  }
  return 0;
}
