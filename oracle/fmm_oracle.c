/*
 * fmm_oracle.c -- CPU ORACLE for the recursive fast-matrix-multiplication hot path of
 * arXiv 1507.00687 (Ballard, Benson, Druinsky, Lipshitz, Schwartz, "Numerical stability of
 * fast matrix multiplication").  PAPER.md line numbers are cited as P:<line>.
 *
 * THIS IS TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product path (the CUDA library under
 * paper_1507_00687_b200/) never links, imports or calls anything here, and this file shares no
 * code, header, table or constant with it.
 *
 * Plain, slow, obviously-correct C99 + OpenMP.  Build with -O2 -fno-fast-math -ffp-contract=off
 * so every "a*b" and "a+b" below is one IEEE-rounded operation (the paper's model of arithmetic,
 * fl(op(a,b)) = op(a,b)(1+theta)).
 *
 * Contents
 *   orc_fmm_f64 / orc_fmm_f32   recursive <U,V,W> executor (Eq. eqn:recursive_alg)
 *   orc_node_st_* / orc_node_c_* one node's S_r/T_r linear combinations and C_k combination
 *   orc_ref_dd                  classical product in double-double (stand-in for the paper's
 *                               quadruple-precision reference)
 *   orc_scale_*                 outside / inside / repeated outside-inside scaling (Alg. 1-3,
 *                               P:740-759)
 *
 * Summation order (reading A3): every multi-term S, T, C sum is accumulated
 * sequentially in ascending index order -- S_r over i, T_r over j, C_k over r -- which is the
 * sequential-summation model the paper analyses (eqn:seq_summation_error).  The
 * first term initialises the sum.  The classical leaf accumulates k ascending from 0.0.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* A base-case rule <M0,K0,N0;R> with coefficient matrices U (M0K0 x R), V (K0N0 x R),
 * W (M0N0 x R), each stored row-major (row index first).  Row conventions follow P:108:
 * U/V rows are column-major indices of A/B entries, W rows are row-major indices of C. */
typedef struct {
  int m0, k0, n0, R;
  const double* U;
  const double* V;
  const double* W;
} orc_rule;

/* A recursion plan: L levels; the rule used at node [l, r1..r_{l-1}] is
 * rules[node_rule[level_off[l] + idx]] with idx the mixed-radix BFS index
 * idx = ((r1*R2 + r2)*R3 + ...), 0-based.  A stationary plan has one entry per level
 * repeated; a uniform non-stationary plan one rule per level; a non-uniform plan
 * any rule per node, with equal (M0,K0,N0,R) within a level. */
typedef struct {
  int L;
  const orc_rule* rules;
  const int* node_rule;
  const int64_t* level_off;
} orc_plan;

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------------------------------
 * Executor, written once as a macro over the working precision T (double or float).
 * ------------------------------------------------------------------------------------------ */
#define ORC_DEFINE_EXECUTOR(T, SUF)                                                            \
  /* Classical leaf: c_ij = sum_k a_ik b_kj, k ascending from 0.0, one rounding   \
   * per multiply and per add.  Vectorised across j only, so each c_ij keeps its order. */    \
  static void leaf_##SUF(int64_t m, int64_t k, int64_t n, const T* A, int64_t lda,            \
                         const T* B, int64_t ldb, T* C, int64_t ldc) {                         \
    const int64_t JB = 256;                                                                    \
    int64_t njb = (n + JB - 1) / JB;                                                           \
    _Pragma("omp parallel for schedule(dynamic) collapse(2) if(m * n * k > 65536)")           \
    for (int64_t i = 0; i < m; ++i) {                                                          \
      for (int64_t jb = 0; jb < njb; ++jb) {                                                   \
        int64_t j0 = jb * JB, j1 = j0 + JB < n ? j0 + JB : n;                                  \
        T* c = C + i * ldc;                                                                    \
        for (int64_t j = j0; j < j1; ++j) c[j] = (T)0;                                         \
        for (int64_t p = 0; p < k; ++p) {                                                      \
          T a = A[i * lda + p];                                                                \
          const T* b = B + p * ldb;                                                            \
          for (int64_t j = j0; j < j1; ++j) c[j] = c[j] + a * b[j];                            \
        }                                                                                      \
      }                                                                                        \
    }                                                                                          \
  }                                                                                            \
                                                                                               \
  /* dst = sum_t coef[t] * src[t], t ascending, first term initialises (Eq. bilinear_alg's    \
   * S_r / T_r / C_k sums).  coef*x is exact for the dyadic coefficients used       \
   * (+-1, +-1/2), so each step is exactly one rounding of the addition. */                    \
  static void lincomb_##SUF(int64_t rows, int64_t cols, int nt, const double* coef,           \
                            const T* const* src, const int64_t* lds, T* dst, int64_t ldd) {    \
    _Pragma("omp parallel for schedule(static) if(rows * cols > 65536)")                       \
    for (int64_t i = 0; i < rows; ++i) {                                                       \
      T* d = dst + i * ldd;                                                                    \
      if (nt == 0) {                                                                           \
        for (int64_t j = 0; j < cols; ++j) d[j] = (T)0;                                        \
        continue;                                                                              \
      }                                                                                        \
      {                                                                                        \
        const T* s = src[0] + i * lds[0];                                                      \
        T u = (T)coef[0];                                                                      \
        for (int64_t j = 0; j < cols; ++j) d[j] = u * s[j];                                    \
      }                                                                                        \
      for (int t = 1; t < nt; ++t) {                                                           \
        const T* s = src[t] + i * lds[t];                                                      \
        T u = (T)coef[t];                                                                      \
        for (int64_t j = 0; j < cols; ++j) d[j] = d[j] + u * s[j];                             \
      }                                                                                        \
    }                                                                                          \
  }                                                                                            \
                                                                                               \
  /* S_r = sum_i u_ir A_i (i ascending), with A_i the (ia, ja) block, i = ia + M0*ja          \
   * (column-major block index). */                                                     \
  static void form_S_##SUF(const orc_rule* ru, int r, int64_t mb, int64_t kb, const T* A,     \
                           int64_t lda, T* S, int64_t lds_) {                                  \
    const T* src[64];                                                                          \
    int64_t lds[64];                                                                           \
    double cf[64];                                                                             \
    int nt = 0;                                                                                \
    for (int i = 0; i < ru->m0 * ru->k0; ++i) {                                                \
      double u = ru->U[i * ru->R + r];                                                         \
      if (u == 0.0) continue;                                                                  \
      int ia = i % ru->m0, ja = i / ru->m0;                                                    \
      src[nt] = A + ia * mb * lda + ja * kb;                                                   \
      lds[nt] = lda;                                                                           \
      cf[nt] = u;                                                                              \
      ++nt;                                                                                    \
    }                                                                                          \
    lincomb_##SUF(mb, kb, nt, cf, src, lds, S, lds_);                                          \
  }                                                                                            \
                                                                                               \
  /* T_r = sum_j v_jr B_j (j ascending), B_j the (ja, jb) block, j = ja + K0*jb. */            \
  static void form_T_##SUF(const orc_rule* ru, int r, int64_t kb, int64_t nb, const T* B,     \
                           int64_t ldb, T* Tm, int64_t ldt) {                                  \
    const T* src[64];                                                                          \
    int64_t lds[64];                                                                           \
    double cf[64];                                                                             \
    int nt = 0;                                                                                \
    for (int j = 0; j < ru->k0 * ru->n0; ++j) {                                                \
      double v = ru->V[j * ru->R + r];                                                         \
      if (v == 0.0) continue;                                                                  \
      int ja = j % ru->k0, jb = j / ru->k0;                                                    \
      src[nt] = B + ja * kb * ldb + jb * nb;                                                   \
      lds[nt] = ldb;                                                                           \
      cf[nt] = v;                                                                              \
      ++nt;                                                                                    \
    }                                                                                          \
    lincomb_##SUF(kb, nb, nt, cf, src, lds, Tm, ldt);                                          \
  }                                                                                            \
                                                                                               \
  /* C_k <- w_kr M_r  (first contribution)  or  C_k <- C_k + w_kr M_r, for every k with       \
   * w_kr != 0; C_k is the (ia, jb) block, k = ia*N0 + jb (row-major). */               \
  static void accum_C_##SUF(const orc_rule* ru, int r, int64_t mb, int64_t nb, const T* Mr,   \
                            int64_t ldm, T* C, int64_t ldc, int* started) {                    \
    for (int k = 0; k < ru->m0 * ru->n0; ++k) {                                                \
      double w = ru->W[k * ru->R + r];                                                         \
      if (w == 0.0) continue;                                                                  \
      int ia = k / ru->n0, jb = k % ru->n0;                                                    \
      T* Ck = C + ia * mb * ldc + jb * nb;                                                     \
      T wt = (T)w;                                                                             \
      if (!started[k]) {                                                                       \
        _Pragma("omp parallel for schedule(static) if(mb * nb > 65536)")                       \
        for (int64_t i = 0; i < mb; ++i)                                                       \
          for (int64_t j = 0; j < nb; ++j) Ck[i * ldc + j] = wt * Mr[i * ldm + j];             \
        started[k] = 1;                                                                        \
      } else {                                                                                 \
        _Pragma("omp parallel for schedule(static) if(mb * nb > 65536)")                       \
        for (int64_t i = 0; i < mb; ++i)                                                       \
          for (int64_t j = 0; j < nb; ++j)                                                     \
            Ck[i * ldc + j] = Ck[i * ldc + j] + wt * Mr[i * ldm + j];                          \
      }                                                                                        \
    }                                                                                          \
  }                                                                                            \
                                                                                               \
  typedef struct {                                                                             \
    T *S, *Tm, *M;                                                                             \
  } scratch_##SUF;                                                                             \
                                                                                               \
  /* One recursive call of Eq. eqn:recursive_alg, depth-first over r. */          \
  static void mul_rec_##SUF(const orc_plan* p, int level, int64_t idx, int64_t m, int64_t k,  \
                            int64_t n, const T* A, int64_t lda, const T* B, int64_t ldb, T* C, \
                            int64_t ldc, scratch_##SUF* sc) {                                  \
    if (level == p->L) {                                                                       \
      leaf_##SUF(m, k, n, A, lda, B, ldb, C, ldc);                                             \
      return;                                                                                  \
    }                                                                                          \
    const orc_rule* ru = &p->rules[p->node_rule[p->level_off[level] + idx]];                   \
    int64_t mb = m / ru->m0, kb = k / ru->k0, nb = n / ru->n0;                                 \
    int started[64];                                                                           \
    for (int q = 0; q < ru->m0 * ru->n0; ++q) started[q] = 0;                                  \
    for (int r = 0; r < ru->R; ++r) {                                                          \
      form_S_##SUF(ru, r, mb, kb, A, lda, sc[level].S, kb);                                    \
      form_T_##SUF(ru, r, kb, nb, B, ldb, sc[level].Tm, nb);                                   \
      mul_rec_##SUF(p, level + 1, idx * ru->R + r, mb, kb, nb, sc[level].S, kb, sc[level].Tm,  \
                    nb, sc[level].M, nb, sc);                                                  \
      accum_C_##SUF(ru, r, mb, nb, sc[level].M, nb, C, ldc, started);                          \
    }                                                                                          \
    for (int q = 0; q < ru->m0 * ru->n0; ++q) {                                                \
      if (started[q]) continue; /* an all-zero W row: C_k = 0 */                              \
      int ia = q / ru->n0, jb = q % ru->n0;                                                    \
      T* Ck = C + ia * mb * ldc + jb * nb;                                                     \
      for (int64_t i = 0; i < mb; ++i)                                                         \
        for (int64_t j = 0; j < nb; ++j) Ck[i * ldc + j] = (T)0;                               \
    }                                                                                          \
  }                                                                                            \
                                                                                               \
  /* C = A*B by the plan.  M, K, N must be divisible by the products of the per-level M0, K0,  \
   * N0 (the caller pads).  Returns 0, or -1 on bad dims / allocation failure. */   \
  int orc_fmm_##SUF(const orc_plan* p, int64_t M, int64_t K, int64_t N, const T* A,           \
                    int64_t lda, const T* B, int64_t ldb, T* C, int64_t ldc) {                 \
    scratch_##SUF sc[32];                                                                      \
    int64_t m = M, k = K, n = N;                                                               \
    if (p->L < 0 || p->L > 31) return -1;                                                      \
    for (int l = 0; l < p->L; ++l) {                                                           \
      const orc_rule* ru = &p->rules[p->node_rule[p->level_off[l]]];                           \
      if (m % ru->m0 || k % ru->k0 || n % ru->n0) return -1;                                   \
      m /= ru->m0;                                                                             \
      k /= ru->k0;                                                                             \
      n /= ru->n0;                                                                             \
      sc[l].S = (T*)malloc(sizeof(T) * (size_t)(m * k > 0 ? m * k : 1));                       \
      sc[l].Tm = (T*)malloc(sizeof(T) * (size_t)(k * n > 0 ? k * n : 1));                      \
      sc[l].M = (T*)malloc(sizeof(T) * (size_t)(m * n > 0 ? m * n : 1));                       \
      if (!sc[l].S || !sc[l].Tm || !sc[l].M) return -1;                                        \
    }                                                                                          \
    mul_rec_##SUF(p, 0, 0, M, K, N, A, lda, B, ldb, C, ldc, sc);                               \
    for (int l = 0; l < p->L; ++l) {                                                           \
      free(sc[l].S);                                                                           \
      free(sc[l].Tm);                                                                          \
      free(sc[l].M);                                                                           \
    }                                                                                          \
    return 0;                                                                                  \
  }                                                                                            \
                                                                                               \
  /* One node's linear combinations: S[r] (mb x kb) and T[r] (kb x nb) for r = 0..R-1, each     \
   * stored contiguously at S + r*mb*kb, T + r*kb*nb.  Exposed for kernel-level tests. */       \
  void orc_node_st_##SUF(const orc_rule* ru, int64_t m, int64_t k, int64_t n, const T* A,      \
                         int64_t lda, const T* B, int64_t ldb, T* S, T* Tm) {                  \
    int64_t mb = m / ru->m0, kb = k / ru->k0, nb = n / ru->n0;                                 \
    for (int r = 0; r < ru->R; ++r) {                                                          \
      form_S_##SUF(ru, r, mb, kb, A, lda, S + r * mb * kb, kb);                                \
      form_T_##SUF(ru, r, kb, nb, B, ldb, Tm + r * kb * nb, nb);                               \
    }                                                                                          \
  }                                                                                            \
                                                                                               \
  /* One node's output combination C_k = sum_r w_kr M_r (r ascending) from R contiguous        \
   * M_r blocks (mb x nb) into C (m x n). */                                                    \
  void orc_node_c_##SUF(const orc_rule* ru, int64_t m, int64_t n, const T* Mr, T* C,           \
                        int64_t ldc) {                                                         \
    int64_t mb = m / ru->m0, nb = n / ru->n0;                                                  \
    int started[64];                                                                           \
    for (int q = 0; q < ru->m0 * ru->n0; ++q) started[q] = 0;                                  \
    for (int r = 0; r < ru->R; ++r) accum_C_##SUF(ru, r, mb, nb, Mr + r * mb * nb, nb, C, ldc, started); \
    for (int q = 0; q < ru->m0 * ru->n0; ++q) {                                                \
      if (started[q]) continue;                                                                \
      int ia = q / ru->n0, jb = q % ru->n0;                                                    \
      for (int64_t i = 0; i < mb; ++i)                                                         \
        for (int64_t j = 0; j < nb; ++j) C[(ia * mb + i) * ldc + jb * nb + j] = (T)0;          \
    }                                                                                          \
  }

ORC_DEFINE_EXECUTOR(double, f64)
ORC_DEFINE_EXECUTOR(float, f32)

/* ------------------------------------------------------------------------------------------
 * Double-double classical reference (substitute for the paper's quad precision, P:548,
 * P:1858-1859).  Per entry: the compensated dot product "Dot2" -- TwoProduct via fma,
 * TwoSum -- k ascending.  Result returned unevaluated as hi + lo.  The fma here is the
 * intended error-free transformation, not a contraction (it is written explicitly).
 * rows == NULL: all M rows; else the nrows listed rows (output row t <-> A row rows[t]).
 * ------------------------------------------------------------------------------------------ */
void orc_ref_dd(int64_t K, int64_t N, const double* A, int64_t lda, const double* B,
                int64_t ldb, const int64_t* rows, int64_t nrows, double* hi, double* lo,
                int64_t ldo) {
  const int64_t JB = 64;
  int64_t njb = (N + JB - 1) / JB;
#pragma omp parallel for schedule(dynamic) collapse(2)
  for (int64_t t = 0; t < nrows; ++t) {
    for (int64_t jb = 0; jb < njb; ++jb) {
      int64_t i = rows ? rows[t] : t;
      int64_t j0 = jb * JB, j1 = j0 + JB < N ? j0 + JB : N;
      double s[64], c[64];
      for (int64_t j = j0; j < j1; ++j) { s[j - j0] = 0.0; c[j - j0] = 0.0; }
      for (int64_t p = 0; p < K; ++p) {
        double a = A[i * lda + p];
        const double* b = B + p * ldb;
        for (int64_t j = j0; j < j1; ++j) {
          double h = a * b[j];
          double r = fma(a, b[j], -h);           /* TwoProduct: a*b = h + r exactly */
          double x = s[j - j0] + h;               /* TwoSum(s, h) = (x, q) */
          double z = x - s[j - j0];
          double q = (s[j - j0] - (x - z)) + (h - z);
          s[j - j0] = x;
          c[j - j0] = c[j - j0] + (q + r);
        }
      }
      for (int64_t j = j0; j < j1; ++j) {
        /* FastTwoSum renormalisation so that hi = fl(hi + lo). */
        double x = s[j - j0] + c[j - j0];
        double e = c[j - j0] - (x - s[j - j0]);
        hi[t * ldo + j] = x;
        lo[t * ldo + j] = e;
      }
    }
  }
}

/* ------------------------------------------------------------------------------------------
 * Diagonal scaling (Section 6).  All operate in double on caller-owned, modified-in-place
 * copies A (M x K, lda) and B (K x N, ldb).  Divisions are divisions ("D^{-1} A" in Alg. 1-3),
 * never reciprocal multiplies (reading A9).
 * Return value: 0 ok; otherwise -(1 + index) of the first all-zero row/column, with *which
 * set to 0 (row of A), 1 (column of B), 2 (column of A), 3 (row of B)  (P:757 proviso).
 * ------------------------------------------------------------------------------------------ */

/* Nearest power of two in log2 ("rounding the scaling matrix entries to the nearest
 * power of two"); reading A8.  x = m * 2^e with m in [0.5, 1); log2 x rounds down to
 * e-1 iff log2 m < -1/2 iff m*m < 1/2, decided exactly with an error-free square. */
double orc_pow2_round(double x) {
  int e;
  double m = frexp(x, &e);
  double h = m * m;
  double l = fma(m, m, -h);
  int below = (h < 0.5) || (h == 0.5 && l < 0.0);
  return ldexp(1.0, below ? e - 1 : e);
}

static void row_absmax(int64_t M, int64_t K, const double* A, int64_t lda, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < M; ++i) {
    double mx = 0.0;
    for (int64_t j = 0; j < K; ++j) {
      double v = fabs(A[i * lda + j]);
      if (v > mx) mx = v;
    }
    out[i] = mx;
  }
}

static void col_absmax(int64_t K, int64_t N, const double* B, int64_t ldb, double* out) {
  for (int64_t j = 0; j < N; ++j) out[j] = 0.0;
  for (int64_t i = 0; i < K; ++i)
    for (int64_t j = 0; j < N; ++j) {
      double v = fabs(B[i * ldb + j]);
      if (v > out[j]) out[j] = v;
    }
}

static int64_t first_zero(const double* v, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!(v[i] > 0.0)) return i;
  return -1;
}

/* O step of Alg. 3 == Alg. 1 lines 1-4: r'_i = max_k |a'_ik|,
 * s'_j = max_k |b'_kj|; a'_ik <- a'_ik / r'_i; b'_kj <- b'_kj / s'_j. */
int orc_step_O(int64_t M, int64_t K, int64_t N, double* A, int64_t lda, double* B, int64_t ldb,
               int pow2, double* rp, double* sp, int* which) {
  row_absmax(M, K, A, lda, rp);
  col_absmax(K, N, B, ldb, sp);
  int64_t z;
  if ((z = first_zero(rp, M)) >= 0) { *which = 0; return (int)-(1 + z); }
  if ((z = first_zero(sp, N)) >= 0) { *which = 1; return (int)-(1 + z); }
  if (pow2) {
    for (int64_t i = 0; i < M; ++i) rp[i] = orc_pow2_round(rp[i]);
    for (int64_t j = 0; j < N; ++j) sp[j] = orc_pow2_round(sp[j]);
  }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < M; ++i)
    for (int64_t k = 0; k < K; ++k) A[i * lda + k] = A[i * lda + k] / rp[i];
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < K; ++k)
    for (int64_t j = 0; j < N; ++j) B[k * ldb + j] = B[k * ldb + j] / sp[j];
  return 0;
}

/* I step of Alg. 3 == Alg. 2:
 * p_k = sqrt( max_j |b'_kj| / max_i |a'_ik| ) (division then sqrt, each correctly rounded);
 * a'_ik <- a'_ik * p_k; b'_kj <- b'_kj / p_k. */
int orc_step_I(int64_t M, int64_t K, int64_t N, double* A, int64_t lda, double* B, int64_t ldb,
               int pow2, double* p, int* which) {
  double* ca = (double*)malloc(sizeof(double) * (size_t)(K > 0 ? K : 1));
  double* rb = (double*)malloc(sizeof(double) * (size_t)(K > 0 ? K : 1));
  col_absmax(M, K, A, lda, ca);
  row_absmax(K, N, B, ldb, rb);
  int64_t z;
  if ((z = first_zero(ca, K)) >= 0) { *which = 2; free(ca); free(rb); return (int)-(1 + z); }
  if ((z = first_zero(rb, K)) >= 0) { *which = 3; free(ca); free(rb); return (int)-(1 + z); }
  for (int64_t k = 0; k < K; ++k) {
    double q = rb[k] / ca[k];
    p[k] = sqrt(q);
    if (pow2) p[k] = orc_pow2_round(p[k]);
  }
  free(ca);
  free(rb);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < M; ++i)
    for (int64_t k = 0; k < K; ++k) A[i * lda + k] = A[i * lda + k] * p[k];
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < K; ++k)
    for (int64_t j = 0; j < N; ++j) B[k * ldb + j] = B[k * ldb + j] / p[k];
  return 0;
}

/* Alg. 3 with the stopping criterion of Thm stopping-criterion,
 * tested from the step after the first O step on; tau < 0 disables the test
 * (fixed step count), tau = 0 stops only at an exact fixed point.  Steps alternate starting with
 * O if first_O else I; a step is one O or one I.
 *   dA (M), dB (N): cumulative outer factors, start at 1: dA_i <- dA_i * r'_i,
 *                   dB_j <- s'_j * dB_j.
 *   dI (K): cumulative inner factor prod_t p_k^{(t)} (reporting only; D cancels, eqn:scaling).
 *   trace_kind[t] = 'O' or 'I'; trace_normA/B[t] = ||A'||max, ||B'||max after step t;
 *   trace_w[t] = max |log factor| of step t  (Lemma convergence-wt's w^{(t)}).
 *   trace_dA (max_steps x M), trace_dB (max_steps x N): cumulative factors after each step
 *   (nullable).  Returns steps taken (>= 0) or the negative error code of a step. */
int orc_scale_repeated(int64_t M, int64_t K, int64_t N, double* A, int64_t lda, double* B,
                       int64_t ldb, int first_O, double tau, int max_steps, int pow2, double* dA,
                       double* dB, double* dI, char* trace_kind, double* trace_normA,
                       double* trace_normB, double* trace_w, double* trace_dA, double* trace_dB,
                       int* which) {
  double lo_I = pow(1.0 + tau, -0.25), hi_I = pow(1.0 + tau, 0.25);
  double lo_O = pow(1.0 + tau, -0.5);
  double* rp = (double*)malloc(sizeof(double) * (size_t)(M > 0 ? M : 1));
  double* sp = (double*)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
  double* p = (double*)malloc(sizeof(double) * (size_t)(K > 0 ? K : 1));
  for (int64_t i = 0; i < M; ++i) dA[i] = 1.0;
  for (int64_t j = 0; j < N; ++j) dB[j] = 1.0;
  for (int64_t k = 0; k < K; ++k) dI[k] = 1.0;
  int t0 = -1; /* index (0-based) of the first O step */
  int steps = 0, rc = 0;
  for (int t = 0; t < max_steps; ++t) {
    int isO = first_O ? (t % 2 == 0) : (t % 2 == 1);
    int stop = 0;
    double w = 0.0;
    if (isO) {
      if (t0 < 0) t0 = t;
      rc = orc_step_O(M, K, N, A, lda, B, ldb, pow2, rp, sp, which);
      if (rc) break;
      for (int64_t i = 0; i < M; ++i) dA[i] = dA[i] * rp[i];
      for (int64_t j = 0; j < N; ++j) dB[j] = sp[j] * dB[j];
      int ok = 1;
      for (int64_t i = 0; i < M; ++i) {
        if (!(rp[i] >= lo_O)) ok = 0;
        double lw = fabs(log(rp[i]));
        if (lw > w) w = lw;
      }
      for (int64_t j = 0; j < N; ++j) {
        if (!(sp[j] >= lo_O)) ok = 0;
        double lw = fabs(log(sp[j]));
        if (lw > w) w = lw;
      }
      stop = (tau >= 0.0) && (t > t0) && ok;
    } else {
      rc = orc_step_I(M, K, N, A, lda, B, ldb, pow2, p, which);
      if (rc) break;
      int ok = 1;
      for (int64_t k = 0; k < K; ++k) {
        dI[k] = dI[k] * p[k];
        if (!(p[k] >= lo_I && p[k] <= hi_I)) ok = 0;
        double lw = fabs(log(p[k]));
        if (lw > w) w = lw;
      }
      stop = (tau >= 0.0) && (t0 >= 0) && (t > t0) && ok;
    }
    steps = t + 1;
    if (trace_kind) trace_kind[t] = isO ? 'O' : 'I';
    if (trace_w) trace_w[t] = w;
    if (trace_normA) {
      double mx = 0.0;
      for (int64_t i = 0; i < M; ++i)
        for (int64_t k = 0; k < K; ++k) if (fabs(A[i * lda + k]) > mx) mx = fabs(A[i * lda + k]);
      trace_normA[t] = mx;
    }
    if (trace_normB) {
      double mx = 0.0;
      for (int64_t k = 0; k < K; ++k)
        for (int64_t j = 0; j < N; ++j) if (fabs(B[k * ldb + j]) > mx) mx = fabs(B[k * ldb + j]);
      trace_normB[t] = mx;
    }
    if (trace_dA) memcpy(trace_dA + (int64_t)t * M, dA, sizeof(double) * (size_t)M);
    if (trace_dB) memcpy(trace_dB + (int64_t)t * N, dB, sizeof(double) * (size_t)N);
    if (stop) break;
  }
  free(rp);
  free(sp);
  free(p);
  return rc ? rc : steps;
}

/* Alg. 1 line 6 / Alg. 3 last line: C <- D_A C' D_B, as c_ij = (dA_i*c'_ij)*dB_j. */
void orc_unscale(int64_t M, int64_t N, double* C, int64_t ldc, const double* dA,
                 const double* dB) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < M; ++i)
    for (int64_t j = 0; j < N; ++j) C[i * ldc + j] = (dA[i] * C[i * ldc + j]) * dB[j];
}
