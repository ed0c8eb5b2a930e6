// Bilinear base-case rules <U,V,W> (Eq. eqn:bilinear_alg): creation, the
// exact Brent check, and the built-in table.  Host-only C++.
//
// Built-ins are written here from their product formulas (a transcription independent of the
// test oracle's tables); the equality of the two is itself a test (tests/test_capi_host.py).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>

#include "fmm_internal.h"

namespace fmm {

namespace {

// A term like "+A11" / "-B21": block (row, col) 1-based.
struct Term {
  int sign, row, col;
};

std::vector<Term> parse_terms(const char* s) {
  std::vector<Term> t;
  int sign = +1;
  for (const char* p = s; *p;) {
    if (*p == '+') { sign = +1; ++p; continue; }
    if (*p == '-') { sign = -1; ++p; continue; }
    if (*p == 'A' || *p == 'B' || *p == 'C' || *p == 'M') {
      t.push_back({sign, p[1] - '0', p[2] - '0'});
      sign = +1;
      p += 3;
      continue;
    }
    ++p;
  }
  return t;
}

// 2x2x2 rule from R products "S_r * T_r" and four C_k combinations over products M1..M7
// ("Mxy" is parsed as product number 10x+y-1 -> we use "M1_" style: digit then '_').
RuleData rule222(const char* name, const std::vector<std::pair<const char*, const char*>>& prods,
                 const char* c11, const char* c12, const char* c21, const char* c22) {
  RuleData d;
  d.name = name;
  d.m0 = d.k0 = d.n0 = 2;
  d.R = (int)prods.size();
  d.U.assign(4 * d.R, 0);
  d.V.assign(4 * d.R, 0);
  d.W.assign(4 * d.R, 0);
  for (int r = 0; r < d.R; ++r) {
    for (const Term& t : parse_terms(prods[r].first))  // A(ia, ja): U row ia + 2 ja
      d.U[((t.row - 1) + 2 * (t.col - 1)) * d.R + r] += t.sign;
    for (const Term& t : parse_terms(prods[r].second))  // B(ja, jb): V row ja + 2 jb
      d.V[((t.row - 1) + 2 * (t.col - 1)) * d.R + r] += t.sign;
  }
  const char* cs[4] = {c11, c12, c21, c22};  // W row k = 2 ia + jb: C11, C12, C21, C22
  for (int k = 0; k < 4; ++k) {
    // "M3" -> product 3 (1-based); terms are written with a single digit after 'M' and a
    // dummy '_' so that parse_terms' 3-char token works.
    for (const Term& t : parse_terms(cs[k])) d.W[k * d.R + (t.row - 1)] += t.sign;
  }
  return d;
}

RuleData make_strassen() {
  // App. A read in the paper's product numbering.
  return rule222("strassen",
                 {{"+A11+A22", "+B11+B22"},
                  {"+A21+A22", "+B11"},
                  {"+A11", "+B12-B22"},
                  {"+A22", "+B21-B11"},
                  {"+A11+A12", "+B22"},
                  {"+A21-A11", "+B11+B12"},
                  {"+A12-A22", "+B21+B22"}},
                 "+M1_+M4_-M5_+M7_", "+M3_+M5_", "+M2_+M4_", "+M1_-M2_+M3_+M6_");
}

RuleData make_winograd() {
  // Strassen-Winograd (reading A2).
  return rule222("winograd",
                 {{"+A11", "+B11"},
                  {"+A12", "+B21"},
                  {"+A11-A21+A12-A22", "+B22"},
                  {"+A22", "+B11-B21-B12+B22"},
                  {"+A21+A22", "+B12-B11"},
                  {"+A21+A22-A11", "+B11-B12+B22"},
                  {"+A11-A21", "+B22-B12"}},
                 "+M1_+M2_", "+M1_+M3_+M5_+M6_", "+M1_-M4_+M6_+M7_", "+M1_+M5_+M6_+M7_");
}

RuleData make_classical() {
  RuleData d;
  d.name = "classical222";
  d.m0 = d.k0 = d.n0 = 2;
  d.R = 8;
  d.U.assign(32, 0);
  d.V.assign(32, 0);
  d.W.assign(32, 0);
  for (int ia = 0; ia < 2; ++ia)
    for (int ja = 0; ja < 2; ++ja)
      for (int jb = 0; jb < 2; ++jb) {
        int r = 4 * ia + 2 * ja + jb;
        d.U[(ia + 2 * ja) * 8 + r] = 1;
        d.V[(ja + 2 * jb) * 8 + r] = 1;
        d.W[(2 * ia + jb) * 8 + r] = 1;
      }
  return d;
}

RuleData make_dalberto() {
  // D'Alberto's variant: V~ = (swap (x) I2) V swaps B's block columns,
  // W~ = (I2 (x) swap) W swaps C's block columns (row conventions of P:108).
  RuleData s = make_strassen();
  RuleData d = s;
  d.name = "strassen_dalberto";
  for (int ja = 0; ja < 2; ++ja)
    for (int jb = 0; jb < 2; ++jb)
      for (int r = 0; r < d.R; ++r) d.V[(ja + 2 * jb) * d.R + r] = s.V[(ja + 2 * (1 - jb)) * d.R + r];
  for (int ia = 0; ia < 2; ++ia)
    for (int jb = 0; jb < 2; ++jb)
      for (int r = 0; r < d.R; ++r) d.W[(2 * ia + jb) * d.R + r] = s.W[(2 * ia + (1 - jb)) * d.R + r];
  return d;
}

}  // namespace

// Brent equations: for A-entry i = (ia,ja) (column-major), B-entry j = (ja',jb) (column-major),
// C-entry k = (ia',jb') (row-major): sum_r U_ir V_jr W_kr = [ja==ja'][ia==ia'][jb==jb'],
// scaled by 2^(3*log2den) to stay in integers.
int64_t brent_violations(const RuleData& d, int64_t* first_i, int64_t* first_j, int64_t* first_k) {
  int64_t bad = 0;
  const int64_t one = (int64_t)1 << (3 * d.log2den);
  for (int i = 0; i < d.m0 * d.k0; ++i) {
    int ia = i % d.m0, ja = i / d.m0;
    for (int j = 0; j < d.k0 * d.n0; ++j) {
      int ja2 = j % d.k0, jb = j / d.k0;
      for (int k = 0; k < d.m0 * d.n0; ++k) {
        int ia2 = k / d.n0, jb2 = k % d.n0;
        int64_t s = 0;
        for (int r = 0; r < d.R; ++r)
          s += (int64_t)d.U[(size_t)i * d.R + r] * d.V[(size_t)j * d.R + r] * d.W[(size_t)k * d.R + r];
        int64_t want = (ja == ja2 && ia == ia2 && jb == jb2) ? one : 0;
        if (s != want) {
          if (bad == 0 && first_i) { *first_i = i; *first_j = j; *first_k = k; }
          ++bad;
        }
      }
    }
  }
  return bad;
}

bool builtin_rule(const std::string& name, RuleData* out) {
  if (name == "classical222") *out = make_classical();
  else if (name == "strassen") *out = make_strassen();
  else if (name == "winograd") *out = make_winograd();
  else if (name == "strassen_dalberto") *out = make_dalberto();
  else return false;
  return true;
}

}  // namespace fmm

// ---------------------------------------------------------------------------------------------
// Stability analysis of rules and plans (Sec. 4).  Host-only, double
// arithmetic (exact here: the quantities are sums / products of small dyadic numbers).
// ---------------------------------------------------------------------------------------------
namespace fmm {

RuleQuantities rule_quantities(const RuleData& d) {
  RuleQuantities q;
  const double den = (double)(1 << d.log2den);
  const int nu = d.m0 * d.k0, nv = d.k0 * d.n0, nw = d.m0 * d.n0;
  q.alpha.assign(d.R, 0); q.beta.assign(d.R, 0); q.a.assign(d.R, 0); q.b.assign(d.R, 0);
  q.gamma.assign(nw, 0); q.q.assign(nw, 0); q.e.assign(nw, 0);
  q.nnz = 0;
  for (int r = 0; r < d.R; ++r) {
    for (int i = 0; i < nu; ++i) {  // eqn:abg, eqn:ab: nonzeros and 1-norms of U's column r
      const int32_t u = d.U[(size_t)i * d.R + r];
      if (u) { q.alpha[r] += 1; q.a[r] += std::fabs(u / den); ++q.nnz; }
    }
    for (int j = 0; j < nv; ++j) {
      const int32_t v = d.V[(size_t)j * d.R + r];
      if (v) { q.beta[r] += 1; q.b[r] += std::fabs(v / den); ++q.nnz; }
    }
  }
  q.Q = 0; q.E = 0;
  for (int k = 0; k < nw; ++k) {
    double mx = 0;
    for (int r = 0; r < d.R; ++r) {
      const int32_t w = d.W[(size_t)k * d.R + r];
      if (!w) continue;
      q.gamma[k] += 1;
      ++q.nnz;
      mx = std::max(mx, q.alpha[r] + q.beta[r]);
      q.e[k] += q.a[r] * q.b[r] * std::fabs(w / den);  // Def. stability (eqn:emax)
    }
    q.q[k] = q.gamma[k] + mx;  // Def. prefactor (eqn:qmax)
    q.Q = std::max(q.Q, q.q[k]);
    q.E = std::max(q.E, q.e[k]);
  }
  return q;
}

}  // namespace fmm

// ---------------------------------------------------------------------------------------------
// Rule transformations (App. A-C): cyclic rotations and transposition.  With the stated row
// conventions (U / V column-major, W row-major) the rotation [[W,U,V]] is literally a
// <n0,m0,k0> algorithm and [[V,W,U]] a <k0,n0,m0> one (the row numbers coincide: a row-major
// index of an m x n matrix is the column-major index of its transpose).
// Transposition C^T = B^T A^T gives <n0,k0,m0> = [[P V, P U, P W]] with vec-permutations:
//   U'[jb + n0*ja] = V[ja + k0*jb],  V'[ja + k0*ia] = U[ia + m0*ja],  W'[jb*m0 + ia] = W[ia*n0 + jb].
// ---------------------------------------------------------------------------------------------
namespace fmm {

bool transform_rule(const RuleData& d, int kind, RuleData* out) {
  RuleData o;
  o.R = d.R;
  o.log2den = d.log2den;
  const int R = d.R;
  if (kind == 1) {  // [[W, U, V]]: <n0, m0, k0>
    o.name = d.name + "_rot";
    o.m0 = d.n0; o.k0 = d.m0; o.n0 = d.k0;
    o.U = d.W; o.V = d.U; o.W = d.V;
  } else if (kind == 2) {  // [[V, W, U]]: <k0, n0, m0>
    o.name = d.name + "_rot2";
    o.m0 = d.k0; o.k0 = d.n0; o.n0 = d.m0;
    o.U = d.V; o.V = d.W; o.W = d.U;
  } else if (kind == 3) {  // transpose: <n0, k0, m0>
    o.name = d.name + "_T";
    o.m0 = d.n0; o.k0 = d.k0; o.n0 = d.m0;
    o.U.assign((size_t)d.n0 * d.k0 * R, 0);
    o.V.assign((size_t)d.k0 * d.m0 * R, 0);
    o.W.assign((size_t)d.m0 * d.n0 * R, 0);
    for (int ja = 0; ja < d.k0; ++ja)
      for (int jb = 0; jb < d.n0; ++jb)
        for (int r = 0; r < R; ++r)
          o.U[((size_t)jb + (size_t)d.n0 * ja) * R + r] = d.V[((size_t)ja + (size_t)d.k0 * jb) * R + r];
    for (int ia = 0; ia < d.m0; ++ia)
      for (int ja = 0; ja < d.k0; ++ja)
        for (int r = 0; r < R; ++r)
          o.V[((size_t)ja + (size_t)d.k0 * ia) * R + r] = d.U[((size_t)ia + (size_t)d.m0 * ja) * R + r];
    for (int ia = 0; ia < d.m0; ++ia)
      for (int jb = 0; jb < d.n0; ++jb)
        for (int r = 0; r < R; ++r)
          o.W[((size_t)jb * d.m0 + ia) * R + r] = d.W[((size_t)ia * d.n0 + jb) * R + r];
  } else {
    return false;
  }
  *out = o;
  return true;
}

}  // namespace fmm
