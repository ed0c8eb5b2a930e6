// Compile-time U / V / W tables of the three built-in 2x2x2 rules, for the K1X2 / K3X2 kernels that are
// specialised per (level-d rule, level-(d+1) rule) pair (kernels_lincomb.cu).  Block index
// b = ia + 2 ja (column-major), product r in the paper's numbering: Strassen App. A
// (P:1971-1991), Strassen-Winograd (reading A2), classical r = 4 ia + 2 ja
// + jb.  These tables are only a dispatch key: the host (capi.cu, builtin_id) selects a
// specialised kernel for a plan level only if that level's rule tables (from rules.cpp) equal
// one of these entry for entry, so a mismatch here can only disable the specialisation.
#pragma once
#include <cstdint>

namespace fmm {

constexpr int kBuiltinNone = -1, kBuiltinStrassen = 0, kBuiltinWinograd = 1, kBuiltinClassical = 2;

__host__ __device__ constexpr int builtin_R(int id) { return id == kBuiltinClassical ? 8 : 7; }

// coefficient (numerator, denominator 1) of block b in column r of U (tv = 0) or V (tv = 1)
__host__ __device__ constexpr int builtin_coef(int id, int tv, int b, int r) {
  // Strassen: S = A11+A22, A21+A22, A11, A22, A11+A12, A21-A11, A12-A22
  //           T = B11+B22, B11, B12-B22, B21-B11, B22, B11+B12, B21+B22
  const int8_t su[4][7] = {{1, 0, 1, 0, 1, -1, 0}, {0, 1, 0, 0, 0, 1, 0}, {0, 0, 0, 0, 1, 0, 1},
                           {1, 1, 0, 1, 0, 0, -1}};
  const int8_t sv[4][7] = {{1, 1, 0, -1, 0, 1, 0}, {0, 0, 0, 1, 0, 0, 1}, {0, 0, 1, 0, 0, 1, 0},
                           {1, 0, -1, 0, 1, 0, 1}};
  // Strassen-Winograd: S = A11, A12, A11-A21+A12-A22, A22, A21+A22, A21+A22-A11, A11-A21
  //                    T = B11, B21, B22, B11-B21-B12+B22, B12-B11, B11-B12+B22, B22-B12
  const int8_t wu[4][7] = {{1, 0, 1, 0, 0, -1, 1}, {0, 0, -1, 0, 1, 1, -1}, {0, 1, 1, 0, 0, 0, 0},
                           {0, 0, -1, 1, 1, 1, 0}};
  const int8_t wv[4][7] = {{1, 0, 0, 1, -1, 1, 0}, {0, 1, 0, -1, 0, 0, 0}, {0, 0, 0, -1, 1, -1, -1},
                           {0, 0, 1, 1, 0, 1, 1}};
  if (id == kBuiltinClassical) {
    const int ia = r / 4, ja = (r / 2) % 2, jb = r % 2;
    return tv == 0 ? (b == ia + 2 * ja ? 1 : 0) : (b == ja + 2 * jb ? 1 : 0);
  }
  if (id == kBuiltinStrassen) return tv == 0 ? su[b][r] : sv[b][r];
  return tv == 0 ? wu[b][r] : wv[b][r];
}

// coefficient of product r in output block k = 2 ia + jb (row-major) of W
__host__ __device__ constexpr int builtin_w(int id, int k, int r) {
  // Strassen: C11 = M1+M4-M5+M7, C12 = M3+M5, C21 = M2+M4, C22 = M1-M2+M3+M6
  const int8_t sw[4][7] = {{1, 0, 0, 1, -1, 0, 1}, {0, 0, 1, 0, 1, 0, 0}, {0, 1, 0, 1, 0, 0, 0},
                           {1, -1, 1, 0, 0, 1, 0}};
  // Strassen-Winograd: C11 = M1+M2, C12 = M1+M3+M5+M6, C21 = M1-M4+M6+M7, C22 = M1+M5+M6+M7
  const int8_t ww[4][7] = {{1, 1, 0, 0, 0, 0, 0}, {1, 0, 1, 0, 1, 1, 0}, {1, 0, 0, -1, 0, 1, 1},
                           {1, 0, 0, 0, 1, 1, 1}};
  if (id == kBuiltinClassical) {
    const int ia = r / 4, jb = r % 2;
    return k == 2 * ia + jb ? 1 : 0;
  }
  return id == kBuiltinStrassen ? sw[k][r] : ww[k][r];
}

// column r is a single +1 (the product's operand is a view of one block)
__host__ __device__ constexpr bool builtin_trivial(int id, int tv, int r) {
  int nz = 0, one = 0;
  for (int b = 0; b < 4; ++b) {
    const int c = builtin_coef(id, tv, b, r);
    nz += c != 0;
    one += c == 1;
  }
  return nz == 1 && one == 1;
}

}  // namespace fmm
