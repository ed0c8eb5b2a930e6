// Internal declarations of libfmm_b200 (not part of the ABI; see include/fmm.h).
//
// Data model: every operand the kernels touch -- a block of the caller's A, B,
// C or a temporary in the workspace -- is described by an Op: element (i, j) lives at
//   base[b] + (row0 + i) * ld + col0 + j,   ld = (Op.ld >= 0 ? Op.ld : bases.ld[b]).
// Descriptors are built once per plan on the host and uploaded once; fmm_execute only passes
// the four base pointers and the caller's leading dimensions as kernel arguments.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/fmm.h"

namespace fmm {

constexpr int kMaxBlk = 16;  // max m0*k0, k0*n0, m0*n0 of a rule
constexpr int kMaxR = 32;    // max rank R of a rule

// BASE_SYM: this rank's symmetric (peer-readable) buffer of top-level products (comm mode 3)
enum BaseId : int32_t { BASE_A = 0, BASE_B = 1, BASE_C = 2, BASE_WS = 3, BASE_SYM = 4 };

struct Op {
  int32_t base;
  int32_t pad_;
  int64_t row0, col0, ld;  // ld < 0: use the base's ld
};

struct Bases {
  const void* p[5];
  int64_t ld[5];
};

// Virtual diagonal scaling (power-of-two factors): the root K1 reads the
// ORIGINAL A (side 0) / B (side 1) and forms S_r / T_r from a_ij 2^(er_i + ec_j), i.e. from A' /
// B' without either being written -- unless the one-kernel scaling run switched to its
// materialised form (*mode != 0), in which case it reads A' / B' from mat[side] (ld ldm[side]).
struct ScaleIn {
  const int32_t* er[2];
  const int32_t* ec[2];
  const double* mat[2];
  int64_t ldm[2];
  const int* mode;
  const int* ext;    // min / max of er[0], ec[0], er[1], ec[1] (8 ints): the two-multiply fast path
  const double* ur;  // d_A, d_B of the run: the root combination (K3 / K3X2 with Step.unscale)
  const double* uc;  // writes C = (d_A,i C'_ij) d_B,j directly
};

// Selects instead of b.p[o.base]: dynamic indexing of a by-value kernel parameter would force
// a local-memory copy of Bases.
template <typename T>
__host__ __device__ inline T* op_ptr(const Bases& b, const Op& o, int64_t& ld) {
  const int id = o.base;
  const void* base = id == 0 ? b.p[0] : id == 1 ? b.p[1] : id == 2 ? b.p[2] : id == 3 ? b.p[3] : b.p[4];
  const int64_t bld = id == 0 ? b.ld[0] : id == 1 ? b.ld[1] : id == 2 ? b.ld[2] : id == 3 ? b.ld[3] : b.ld[4];
  ld = o.ld >= 0 ? o.ld : bld;
  return (T*)base + o.row0 * ld + o.col0;
}

// ---- rules -----------------------------------------------------------------------------------
struct RuleData {
  std::string name;
  int m0 = 0, k0 = 0, n0 = 0, R = 0, log2den = 0;
  std::vector<int32_t> U, V, W;  // numerators, row-major (rows x R)
  double coef(const std::vector<int32_t>& X, int row, int r) const {
    return (double)X[(size_t)row * R + r] / (double)(1 << log2den);
  }
};

// Principal quantities of a rule (Sec. 4.1): alpha / beta (nonzeros of U / V
// columns), gamma (nonzeros of W rows), a / b (1-norms of U / V columns), q_k, Q, e_k, E, nnz.
struct RuleQuantities {
  std::vector<double> alpha, beta, gamma, a, b, q, e;
  double Q = 0, E = 0;
  int64_t nnz = 0;
};
RuleQuantities rule_quantities(const RuleData& d);

// ---- K1: linear combinations S_r = sum_i u_ir A_i (or T_r = sum_j v_jr B_j) -------------
// The input operand (rows*P x cols*Q) is split into P x Q sub-blocks of rows x cols; the
// sub-block index is column-major, blk = p + P*q.  coef points at the rule's table
// ((P*Q) x R row-major).  Outputs are written for the r in out_mask.
// The output list is compiled on the host (k1_compile): nout outputs r = rlist[o], each with
// a 2-bit code per input block (0 absent, 1 +1, 2 -1, 3 general coefficient from the table).
struct K1Node {
  Op in;
  int64_t rows, cols;  // sub-block dims of this node's split (S: mb x kb, T: kb x nb)
  int32_t P, Q;        // split P x Q (S: m0 x k0, T: k0 x n0)
  int32_t coef_off;  // offset (in doubles) of the table in the plan's coefficient buffer
  int32_t tv;        // 0: S (U table), 1: T (V table) -- for the compile-time K1 (Step.x1)
  uint32_t out_mask;
  int32_t nout;      // number of outputs written
  uint32_t need;     // bit b: input block b is read
  uint8_t rlist[kMaxR];
  uint32_t code[kMaxR];
  Op out[kMaxR];
};

// Host: fill nout / rlist / code / need of a K1 node from its rule table X ((nblk) x R
// numerators over 2^log2den, i.e. U or V) and the node's out_mask.
inline void k1_compile(K1Node& n, const RuleData& ru, const std::vector<int32_t>& X, int nblk) {
  n.nout = 0;
  n.need = 0;
  const int32_t one = 1 << ru.log2den;
  for (int r = 0; r < ru.R; ++r) {
    if (!((n.out_mask >> r) & 1u)) continue;
    uint32_t c = 0;
    for (int b = 0; b < nblk; ++b) {
      const int32_t u = X[(size_t)b * ru.R + r];
      if (u == 0) continue;
      n.need |= 1u << b;
      c |= (u == one ? 1u : u == -one ? 2u : 3u) << (2 * b);
    }
    n.rlist[n.nout] = (uint8_t)r;
    n.code[n.nout] = c;
    ++n.nout;
  }
}

// ---- K1X2: two recursion levels of S (or T) formation in one HBM pass -------------------
// A node of level d (rule 1: 2 x 2 blocks, table X1 = U or V, rank R1) whose children all use
// rule 2 (2 x 2, X2, R2).  The grandchild operands
//   S_{r1 r2} = sum_{i2} x2_{i2 r2} S_{r1}[i2],   S_{r1}[i2] = sum_{i1} x1_{i1 r1} A[i1][i2]
// (P:104-105 applied at level d, then at level d+1 to the blocks of S_{r1}) are evaluated per
// element in registers, in the order of the two one-level passes (so bitwise equal to them),
// without writing the level-(d+1) operands S_{r1}.  Input block i1 = p1 + 2 q1 (column-major,
// P:108), its sub-block i2 = p2 + 2 q2: rows (2 p1 + p2) rows + i, cols (2 q1 + q2) cols + j.
// The rule pair is a kernel template (built-in rules, builtin_tables.h), so the output list --
// every (r1, r2) except those whose columns are a single +1 at both levels (views), r1-major --
// is known at compile time; the descriptor carries only the output pointers.
constexpr int kMaxX2 = 64;  // max formed grandchildren of a node (R1 * R2)
struct K1x2Node {
  Op in;
  int64_t rows, cols;  // grandchild block dims (outputs are workspace blocks with ld = cols)
  int32_t tv;          // 0: S (U tables, A side), 1: T (V tables, B side)
  int32_t nout;        // formed grandchildren (checked against the kernel's list)
  // FP32 tensor-core leaves, split mode (lo_off > 0): EVERY (r1, r2) is formed (views too) and
  // written as its TF32 hi / lo pair -- hi at out[idx], lo lo_off elements further -- straight
  // into the leaf GEMM's operand arena
  int64_t lo_off;
  Op out[kMaxX2];
};

// ---- K3X2: two levels of the W-combination in one pass --------------------------------------
// For a node of level d (built-in rule 1, R1) whose children all use built-in rule 2 (R2):
//   C[k1][k2] = sum_{r1} w1_{k1 r1} C_{r1}[k2],   C_{r1}[k2] = sum_{r2} w2_{k2 r2} M_{r1 r2}
// (P:119 at levels d+1 and d), per element in registers in K3's order (ascending r, first term
// initialises), so bitwise equal to two K3 passes; the children's outputs C_{r1} are never
// written.  Output block k1 = 2 ia1 + jb1 (row-major), its sub-block k2 = 2 ia2 + jb2:
// rows (2 ia1 + ia2) rows + i, cols (2 jb1 + jb2) cols + j of the node output.
struct K3x2Node {
  Op out;
  int64_t rows, cols;  // grandchild block dims (inputs are workspace blocks with ld = cols)
  Op in[kMaxX2];       // M_{r1 r2}, index r1 * R2 + r2
};

// ---- K3: C_k = sum_r w_kr M_r into the node output (rows*M0 x cols*N0), k = ia*N0 + jb ----
struct K3Node {
  Op out;
  int32_t coef_off;  // W table ((M0*N0) x R)
  int32_t pad_;
  Op in[kMaxR];
};

// ---- ACC: C_k (+)= w_kr M_r for one r (depth-first top level / multi-GPU partial) ----------
struct AccNode {
  Op out;     // node output (M0*rows x N0*cols)
  Op in;      // M_r (rows x cols)
  int32_t coef_off;
  int32_t r;
  uint32_t first_mask;  // bit k: this is the first contribution to C_k (initialise)
  uint32_t pad_;
};

// ---- ZERO: zero the blocks k in mask of a node output --------------------------------------
struct ZeroNode {
  Op out;
  uint32_t mask;
  uint32_t pad_;
};

// ---- K2: leaf products M = S.T ---------------------------------------------------------------
struct LeafNode {
  Op a, b, c;
};

// ---- K2F: leaf products with the parent's W-combination fused into the epilogue ----------
// One CTA computes one output tile position of the leaf products r = rlist[0..nr) of a parent
// node in ascending order and, after each product, updates the parent's output blocks
//   C_k = w_kr M_r (first contribution, bit k of first[i]) | C_k = C_k + w_kr M_r,
// i.e. the K3 / ACC arithmetic in the same per-element order (bitwise identical), without
// writing M_r to memory.
struct FusedNode {
  Op out;            // parent output (M0*m x N0*n)
  int32_t coef_off;  // W table ((M0*N0) x R)
  int32_t nr;
  uint8_t rlist[kMaxR];
  uint32_t wmask[kMaxR];  // bit k: w_kr != 0
  uint32_t first[kMaxR];  // bit k: this product initialises C_k
  Op a[kMaxR], b[kMaxR];  // leaf operands S_r, T_r (index i, not r)
};

enum StepKind { STEP_K1 = 1, STEP_K2 = 2, STEP_K3 = 3, STEP_ACC = 4, STEP_ZERO = 5, STEP_K2F = 8,
                STEP_SMALL = 9 };

struct Step {
  int kind;
  int count;         // number of nodes in the launch
  int64_t dev_off;   // byte offset of the node array in the plan's device descriptor buffer
  int64_t rows, cols, inner;  // sub-block dims (K1/K3/ACC/ZERO) or m, n, k (K2)
  int P, Q, R;       // K1: split P x Q, rank R.  K3/ACC/ZERO: P = M0, Q = N0, R
  int64_t arena_off; // K2 FP32 tensor-core leaves: offset (elements) of the hi/lo arena in ws
  bool vec_ok;       // all ws offsets / dims allow 16-byte vectors (caller bases checked later)
  int nr = 0;        // K2F: products per node (uniform)
  int64_t dev_off2 = -1;  // K2F FP32: LeafNode list (parent-major) for the hi / lo split
  bool unitw = false;  // K2F: every W coefficient of the level is 0 or +-1 (sign-flip epilogue)
  int k2f_cfg = 16;  // K2F tile configuration (16: 128 x 128 / 1 CTA per SM, 13: 64 x 64 / 3)
  int chunk = 0;     // K2F FP32: products per CTA when a unit's chain is split (0: whole chain)
  uint32_t split = 0;  // K2F FP64: chain split, byte g = end of group g's products (0: none);
                     // both: turnstiles (one int per unit) + a ticket counter at ws offset
                     // turn_off (in elements of the plan's dtype)
  int64_t turn_off = -1;
  int x2 = 0;        // K1 / K3: 0 one level (K1Node / K3Node); else K1x2Node / K3x2Node with
                     // rule pair (x2 - 1) / 3, (x2 - 1) % 3 (builtin_tables.h ids)
  int scaled = 0;    // K1 of the root with virtual scaling (reads A / B through ScaleIn)
  int x1 = 0;        // one-level K1 whose nodes all use built-in rule x1 - 1 (2x2): the
                     // compile-time specialised kernel (k1c_lincomb)
  int unscale = 0;   // K3 / K3X2 of the root of a scaled plan: the unscale folded in
  // STEP_SMALL (kernels_small.cu): the K1X2 nodes (dev_off, count), the leaves (dev_off2,
  // count2, rows x cols x inner), the K3X2 nodes (dev_off3, count3), rule pair x2
  int count2 = 0, count3 = 0;
  int64_t dev_off3 = -1;
  int tf32_split = 0;  // K1 (x2): split mode (K1x2Node.lo_off); K2 FP32: the arena is already
                       // filled by that pass (no split kernel)
};

// ---- kernel launchers (kernels_*.cu) -----------------------------------------------------------
template <typename T>
cudaError_t launch_k1(const Step& s, const void* dev_nodes, const double* dev_coef,
                      const Bases& b, bool vec, cudaStream_t st, const ScaleIn* sc = nullptr);
template <typename T>
cudaError_t launch_k3(const Step& s, const void* dev_nodes, const double* dev_coef,
                      const Bases& b, bool vec, cudaStream_t st, const ScaleIn* sc = nullptr);
template <typename T>
cudaError_t launch_acc(const Step& s, const void* dev_nodes, const double* dev_coef,
                       const Bases& b, bool vec, cudaStream_t st);
template <typename T>
cudaError_t launch_zero(const Step& s, const void* dev_nodes, const Bases& b, cudaStream_t st);

// Comm mode 3 (fused NVLink combine): rows [row0, row1) of C (M x N, ldc; blocks k = ia*N0 + jb
// of mb x nb) = sum_r ascending w_kr M_r, M_r read from peers[r % P] + (r / P) * mb * nb
// (each rank's symmetric buffer holds its owned products, slot r / P, dense mb x nb).
template <typename T>
cudaError_t launch_p2p_combine(const T* const* dev_peers, int P, const double* dev_coef, int coef_off,
                               int R, int M0, int N0, int64_t mb, int64_t nb, T* C, int64_t ldc,
                               int64_t row0, int64_t row1, bool vec, cudaStream_t st);

// dst (rows_p x cols_p, ldd) = src (rows x cols, lds) zero-extended (rows <= rows_p, cols <=
// cols_p): the zero padding / cropping of non-divisible dims
template <typename T>
cudaError_t launch_pad_copy(const T* src, int64_t rows, int64_t cols, int64_t lds, T* dst,
                            int64_t rows_p, int64_t cols_p, int64_t ldd, cudaStream_t st);

cudaError_t launch_gemm_f64(const LeafNode* dev_leaves, int count, int64_t m, int64_t n,
                            int64_t k, const Bases& b, bool vec, cudaStream_t st);
cudaError_t launch_gemm_f64_fused(const FusedNode* dev_nodes, int count, int64_t m, int64_t n,
                                  int64_t k, const double* dev_coef, int P, int Q, int R,
                                  const Bases& b, bool vec, cudaStream_t st, int nr, uint32_t split,
                                  int* turn, int cfg, bool unitw);
// groups (1..4) of a K2F chain split for chains of nr products; -1 when malformed
int split_groups(uint32_t split, int nr);
// output tile edge (BM = BN) of K2F tile configuration cfg (13: 64, 16: 128)
int k2f_tile_of(int cfg);
// The single-launch small plan (K1X2 -> leaf products -> K3X2 in one cooperative kernel); its
// leaf-phase tile (small_tile_m x small_tile_n)
cudaError_t launch_small_plan(int pair, const K1x2Node* k1, int nk1, const LeafNode* lf, int nlf,
                              int64_t m, int64_t n, int64_t k, const K3x2Node* k3, int nk3,
                              const Bases& b, bool vec, cudaStream_t st);
int small_tile_m();
int small_tile_n();
cudaError_t launch_gemm_f32(const LeafNode* dev_leaves, const LeafNode* host_leaves, int count,
                            int64_t m, int64_t n, int64_t k, const Bases& b, bool vec, int leaf,
                            float* arena, cudaStream_t st, bool presplit = false);
// floats of workspace the tensor-core FP32 leaf needs for a batch (hi / lo operand arena)
size_t tf32_arena_floats(int64_t count, int64_t m, int64_t n, int64_t k);

// TF32 hi / lo split of an FP32 value: hi = x rounded to 10 mantissa bits (nearest, ties away),
// lo = x - hi (exact); the split every producer of the tensor-core leaf operands uses
#ifdef __CUDACC__
__device__ __forceinline__ void tf32_split(float x, float& h, float& l) {
  const uint32_t u = (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u;
  h = __uint_as_float(u);
  l = x - h;
}
#endif

// ---- error reporting ------------------------------------------------------------------------
void set_error(const std::string& msg);
fmm_status cuda_status(cudaError_t e, const char* where);

}  // namespace fmm

// The opaque ABI types.
struct fmm_rule {
  fmm::RuleData d;
};
