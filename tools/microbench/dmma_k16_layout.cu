// Fragment layout and rounding probe for mma.sync m16n8k16 .f64 (sm_90+ shape) against two
// candidate layouts; prints which one reproduces D = A B + C exactly on small-integer inputs,
// and whether a k16 instruction rounds like four chained m16n8k4 instructions.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/k16 dmma_k16_layout.cu && /tmp/k16
#include <cmath>
#include <cstdio>

__device__ void mma_k16(double* d, const double* a, const double* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11},"
      " {%12,%13,%14,%15}, {%0,%1,%2,%3};"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
        "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}
__device__ void mma_k4(double* d, double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a0), "d"(a1), "d"(b0));
}

// layout 1: a_{2j} = A[g][t + 4j], a_{2j+1} = A[g + 8][t + 4j]; b_j = B[t + 4j][g]
// layout 2: a0,a1 = A[g][t], A[g][t+4]?  (the f16-style interleave: a_{i}: row g + 8*((i>>1)&1),
//           col t + 4*(i&1) + 8*(i>>2)); b_j = B[t + 4*(j&1) + 8*(j>>1)][g]
__global__ void probe(const double* A, const double* B, double* D1, double* D2, double* D4) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a[8], b[4], d[4];
  for (int j = 0; j < 4; ++j) {
    a[2 * j] = A[g * 16 + t + 4 * j];
    a[2 * j + 1] = A[(g + 8) * 16 + t + 4 * j];
    b[j] = B[(t + 4 * j) * 8 + g];
  }
  for (int e = 0; e < 4; ++e) d[e] = 0.0;
  mma_k16(d, a, b);
  D1[g * 8 + 2 * t] = d[0]; D1[g * 8 + 2 * t + 1] = d[1];
  D1[(g + 8) * 8 + 2 * t] = d[2]; D1[(g + 8) * 8 + 2 * t + 1] = d[3];
  for (int i = 0; i < 8; ++i) a[i] = A[(g + 8 * ((i >> 1) & 1)) * 16 + t + 4 * (i & 1) + 8 * (i >> 2)];
  for (int j = 0; j < 4; ++j) b[j] = B[(t + 4 * (j & 1) + 8 * (j >> 1)) * 8 + g];
  for (int e = 0; e < 4; ++e) d[e] = 0.0;
  mma_k16(d, a, b);
  D2[g * 8 + 2 * t] = d[0]; D2[g * 8 + 2 * t + 1] = d[1];
  D2[(g + 8) * 8 + 2 * t] = d[2]; D2[(g + 8) * 8 + 2 * t + 1] = d[3];
  // four chained k4 (the existing kernels' sequence)
  for (int e = 0; e < 4; ++e) d[e] = 0.0;
  for (int j = 0; j < 4; ++j)
    mma_k4(d, A[g * 16 + t + 4 * j], A[(g + 8) * 16 + t + 4 * j], B[(t + 4 * j) * 8 + g]);
  D4[g * 8 + 2 * t] = d[0]; D4[g * 8 + 2 * t + 1] = d[1];
  D4[(g + 8) * 8 + 2 * t] = d[2]; D4[(g + 8) * 8 + 2 * t + 1] = d[3];
}

int main() {
  double hA[256], hB[128], ref[128], h1[128], h2[128], h4[128];
  double *A, *B, *D1, *D2, *D4;
  cudaMalloc(&A, sizeof hA); cudaMalloc(&B, sizeof hB);
  cudaMalloc(&D1, sizeof h1); cudaMalloc(&D2, sizeof h2); cudaMalloc(&D4, sizeof h4);
  // pass 1: small integers (exact in any order): identifies the layout
  for (int i = 0; i < 256; ++i) hA[i] = (double)((i * 7) % 13 - 6);
  for (int i = 0; i < 128; ++i) hB[i] = (double)((i * 5) % 11 - 5);
  for (int r = 0; r < 16; ++r)
    for (int c = 0; c < 8; ++c) {
      double s = 0;
      for (int k = 0; k < 16; ++k) s += hA[r * 16 + k] * hB[k * 8 + c];
      ref[r * 8 + c] = s;
    }
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  probe<<<1, 32>>>(A, B, D1, D2, D4);
  cudaMemcpy(h1, D1, sizeof h1, cudaMemcpyDeviceToHost);
  cudaMemcpy(h2, D2, sizeof h2, cudaMemcpyDeviceToHost);
  int bad1 = 0, bad2 = 0;
  for (int i = 0; i < 128; ++i) { bad1 += h1[i] != ref[i]; bad2 += h2[i] != ref[i]; }
  printf("integer inputs: layout1 mismatches %d, layout2 mismatches %d\n", bad1, bad2);
  // pass 2: random doubles: does k16 round like four chained k4?
  unsigned s = 12345;
  auto rnd = [&] { s = s * 1664525u + 1013904223u; return ((double)(s >> 8) / 16777216.0 - 0.5) * std::ldexp(1.0, (int)(s % 40) - 20); };
  int diff = 0, n = 0;
  for (int trial = 0; trial < 200; ++trial) {
    for (int i = 0; i < 256; ++i) hA[i] = rnd();
    for (int i = 0; i < 128; ++i) hB[i] = rnd();
    cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
    cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
    probe<<<1, 32>>>(A, B, D1, D2, D4);
    cudaMemcpy(h1, D1, sizeof h1, cudaMemcpyDeviceToHost);
    cudaMemcpy(h4, D4, sizeof h4, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 128; ++i) { diff += h1[i] != h4[i]; ++n; }
  }
  printf("random inputs: k16 (layout1) vs 4 x k4 chained: %d of %d elements differ\n", diff, n);
  return 0;
}
