/*
 * fmm.h -- C ABI of the B200-native recursive fast-matrix-multiplication library
 * (libfmm_b200.so), implementing the hot path of arXiv 1507.00687 (Ballard, Benson, Druinsky,
 * Lipshitz, Schwartz, "Numerical stability of fast matrix multiplication").
 * Citations "P:<line>" are lines of the paper's text and the section / equation /
 * algorithm they fall in.
 *
 * General conventions
 *  - Every entry point is extern "C", takes plain pointers and sizes, and returns fmm_status
 *    (FMM_OK = 0).  No C++ exception crosses the ABI.  On failure, fmm_last_error() returns a
 *    thread-local message naming the offending argument / index / CUDA or NCCL error text.
 *  - Matrices are dense ROW-MAJOR with a leading dimension in elements (ld >= #columns).
 *    A is M x K, B is K x N, C is M x N: C = A.B.
 *  - Device pointers ("dev") must be CUDA device memory of the current device; "host" pointers
 *    are CPU memory.  The caller owns every buffer passed in (A, B, C, workspace, factor
 *    vectors); the library owns fmm_rule / fmm_plan objects and their small device tables.
 *  - Work is enqueued asynchronously on the given cudaStream_t (passed as void*; NULL = legacy
 *    default stream).  Argument errors are reported synchronously; device faults surface as
 *    FMM_E_CUDA at a later call or synchronisation.
 *  - Inputs A and B are never modified.  NaN/Inf propagate (no checks).
 *  - Dtype FMM_F64: double; FMM_F32: float.
 */
#ifndef FMM_B200_H
#define FMM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FMM_OK = 0,
  FMM_E_ARG = 1,          /* bad argument (null pointer, negative size, bad enum, ld < cols) */
  FMM_E_RULE = 2,         /* rule violates the Brent equations (not a bilinear algorithm)    */
  FMM_E_SHAPE = 3,        /* dims not divisible by the plan's base-case products, mismatch   */
  FMM_E_ALIGN = 4,        /* pointer / ld alignment requirement not met                      */
  FMM_E_PRECOND = 5,      /* scaling precondition: an all-zero row or column         */
  FMM_E_UNSUPPORTED = 6,  /* valid request this build does not implement                     */
  FMM_E_CUDA = 7,         /* CUDA runtime error                                              */
  FMM_E_NCCL = 8,         /* NCCL error / NCCL library not loadable                          */
  FMM_E_OOM = 9,          /* workspace too small / device allocation failed                  */
  FMM_E_NOT_CONVERGED = 10 /* reserved                                                        */
} fmm_status;

typedef enum { FMM_F64 = 0, FMM_F32 = 1 } fmm_dtype;

/* Leaf (base-case) classical multiplication kind.
 *  NATIVE : FP64 -> DMMA tensor-core mma (f64 in, f64 accumulate); FP32 -> FP32 FMA.
 *  TF32   : FP32 only, single-pass TF32 tensor core (reported variant; fails FP32 parity).
 *  3XTF32 : FP32 only, hi/lo split 3-pass TF32 tensor core (default for FP32). */
typedef enum { FMM_LEAF_NATIVE = 0, FMM_LEAF_TF32 = 1, FMM_LEAF_3XTF32 = 2 } fmm_leaf;

/* Diagonal scaling modes (Section 6): outside = Alg. 1, inside = Alg. 2
 * (P:862-868), out_in / in_out = one O step then one I step (or reverse), repeated = Alg. 3
 * with the Thm stopping-criterion test. */
typedef enum {
  FMM_SCALE_NONE = 0,
  FMM_SCALE_OUTSIDE = 1,
  FMM_SCALE_INSIDE = 2,
  FMM_SCALE_OUT_IN = 3,
  FMM_SCALE_IN_OUT = 4,
  FMM_SCALE_REPEATED = 5
} fmm_scale_mode;

typedef struct {
  int mode;            /* fmm_scale_mode */
  int first_step_is_O; /* repeated: 1 = start with an O step (Alg. 3 as printed), 0 = I step */
  double tau;          /* repeated: stopping tolerance tau; tau < 0 disables the test,
                          tau = 0 stops only at an exact fixed point */
  int max_steps;       /* repeated: cap on the number of O/I steps (>= 1)                    */
  int pow2;            /* 1: round every factor to the nearest power of two      */
} fmm_scaling;

typedef struct fmm_rule fmm_rule; /* opaque, immutable after creation, thread-safe to share */
typedef struct fmm_plan fmm_plan; /* opaque; execute() is re-entrant for distinct C / ws   */

/* ---------------------------------------------------------------------------------------
 * Rules <U,V,W> (Eq. eqn:bilinear_alg)
 * U is (m0*k0) x R, V is (k0*n0) x R, W is (m0*n0) x R, each ROW-MAJOR int32 numerators;
 * coefficient = numerator / 2^log2_den.  Row conventions: U/V rows index the entries of
 * the A/B base-case block in COLUMN-major order (i = ia + m0*ja, j = ja + k0*jb); W rows index
 * C in ROW-major order (k = ia*n0 + jb).  The Brent equations are checked exactly in int64 over
 * all (m0k0)(k0n0)(m0n0) triples; on violation returns FMM_E_RULE, *n_violations (nullable) is
 * the count and fmm_last_error() names the first violated (i,j,k).  Limits: m0*k0, k0*n0,
 * m0*n0 <= 16, R <= 32, |numerator| < 2^20, 0 <= log2_den <= 8.  `name` (nullable) is copied.
 * ------------------------------------------------------------------------------------- */
fmm_status fmm_rule_create(int m0, int k0, int n0, int R, const int32_t* U, const int32_t* V,
                           const int32_t* W, int log2_den, const char* name, fmm_rule** out,
                           int64_t* n_violations);

/* Built-in rules: "classical222" (<2,2,2;8>, product r = 4ia + 2ja + jb), "strassen" (App. A,
 * P:1971-1991, converted to the stated convention, A1), "winograd"
 * (Strassen-Winograd, coefficients in DESIGN.md A2), "strassen_dalberto"
 * (<U, (swap (x) I2)V, (I2 (x) swap)W>). */
fmm_status fmm_rule_builtin(const char* name, fmm_rule** out);

/* Rule transformations (App. A-C); the result is validated
 * (Brent) and returned as a new rule (caller destroys).  kind 1: cyclic rotation [[W,U,V]], a
 * <n0,m0,k0> algorithm; kind 2: [[V,W,U]], <k0,n0,m0>; kind 3: transposition (C^T = B^T A^T,
 * vec-permuted rows), <n0,k0,m0>.  Rotations and transposition keep R and nnz; Q / E of the
 * rotations are those of the rotated tables (App. A: Strassen's three rotations share Q and E). */
fmm_status fmm_rule_transform(const fmm_rule* rule, int kind, fmm_rule** out);

/* Copy out a rule's dims and tables (any output pointer may be NULL; U/V/W must hold the
 * full table when non-NULL). */
fmm_status fmm_rule_info(const fmm_rule* rule, int* m0, int* k0, int* n0, int* R, int32_t* U,
                         int32_t* V, int32_t* W, int* log2_den);
void fmm_rule_destroy(fmm_rule* rule);

/* ---------------------------------------------------------------------------------------
 * Plans (Sections 3.2-3.4)
 *  uniform = 1: nodes[l] is the rule of level l (l = 0 is the root, "level 1" in the paper's
 *               numbering); n_nodes == levels.  Stationary plans repeat one rule.
 *  uniform = 0: nodes lists one rule per internal node of the recursion tree in BFS order,
 *               node [l, r1..r_{l-1}] at index sum_{l'<l} prod R + ((r1 R2 + r2) R3 + ...)
 *               (0-based r), n_nodes = 1 + R1 + R1 R2 + ....  Rules within a
 *               level must share (m0,k0,n0,R).
 *  levels = 0 means the classical algorithm (the leaf) on the whole problem.
 *  M, K, N must be divisible by prod m0, prod k0, prod n0 (else FMM_E_SHAPE).
 *  leaf: fmm_leaf; FP64 requires NATIVE.  scaling (nullable = none): applied inside
 *  fmm_execute around the multiplication (C = D_A (A' B') D_B, eqn:scaling P:717-722).
 * The plan copies what it needs from the rules; rules may be destroyed afterwards.
 * ------------------------------------------------------------------------------------- */
fmm_status fmm_plan_create(const fmm_rule* const* nodes, int n_nodes, int levels, int uniform,
                           int64_t M, int64_t K, int64_t N, int dtype, int leaf,
                           const fmm_scaling* scaling, fmm_plan** out);
void fmm_plan_destroy(fmm_plan* plan);

/* Multi-GPU partition of the top-level subproblems: rank p of P computes only
 * the top-level products M_r with r = p (mod P) and writes into C the PARTIAL sum
 * C_k = sum_{owned r, ascending} w_kr M_r (blocks with no owned contribution are zeroed).
 * nranks = 1 restores the full computation.  Host-only; call before fmm_execute. */
fmm_status fmm_plan_set_partition(fmm_plan* plan, int rank, int nranks);

/* Schedule control (host-only): 0 = automatic (breadth-first unless its workspace exceeds
 * 24 GiB, then 3 on one rank if its workspace stays within 64 GiB, else 2), 1 = breadth-first
 * over all levels, 2 = depth-first over the top-level products (each subtree breadth-first,
 * top-level accumulation r ascending, per r), 3 = hybrid: the root's S_r / T_r of all r in one
 * pass, the subtrees one after another, the root's (and level 1's, as one K3X2 pass)
 * W-combination at the end (single rank; falls back to 2 above 64 GiB of workspace).  Results
 * are bitwise identical across schedules.  FMM_E_ARG outside 0..3; the environment variable
 * FMM_HYBRID=0 makes 0 choose 2 instead of 3. */
fmm_status fmm_plan_set_schedule(fmm_plan* plan, int schedule);

/* Epilogue fusion of the accumulation step (host-only; north star item 3, Eq.
 * eqn:recursive_alg P:116-125): the parents of the leaves compute C_k = sum_r w_kr M_r inside
 * the leaf-product kernel -- one CTA runs the R leaf products of a parent at one output tile
 * in ascending r and updates C_k after each (c = w*m first, then c = c + w*m), so M_r is never
 * written to memory and the result is bitwise identical to the unfused K2 + K3 path.
 * mode: 0 = off, 1 = on, 2 = automatic (default; on when parents x output tiles fill the GPU
 * several times, the units' product chains split over CTAs where that balances the waves).
 * FMM_E_ARG for other modes.  FP64 plans; FP32 tensor-core plans fuse only with mode 1.  The
 * environment variable FMM_FUSION (0/1/2) sets the default at fmm_plan_create. */
fmm_status fmm_plan_set_fusion(fmm_plan* plan, int mode);

/* S / T formation levels per pass (host-only; north star item 1, P:104-105 applied twice).
 * levels = 2 (default): where two consecutive recursion levels d, d+1 split 2x2-or-smaller
 * blocks with built-in rules (Strassen, Strassen-Winograd, classical: tables equal to the built-in
 * ones) and every child of a level-d node uses one rule, one K1X2 launch forms
 * the level-(d+2) operands S_{r1 r2} = sum_i2 u2_{i2 r2} (sum_i1 u1_{i1 r1} A[i1][i2]) directly
 * from the level-d operand, in registers, in the order of two one-level passes (bitwise
 * identical); the level-(d+1) S_{r1} / T_{r1} are never written (less HBM traffic and
 * workspace).  Levels pair from the bottom: (L-2, L-1), (L-4, L-3), ...  levels = 1: one K1 pass
 * per level.  FMM_E_ARG for other values.  The environment variable FMM_K1X2=0 sets 1 at
 * fmm_plan_create. */
fmm_status fmm_plan_set_k1_levels(fmm_plan* plan, int levels);

/* Where the FP32 tensor-core leaves' operands are split (host-only; FMM_F32 plans with leaf
 * FMM_LEAF_3XTF32 / FMM_LEAF_TF32; north star item 2, the leaf products M_r = S_r T_r of P:125).
 * The tensor-core leaf multiplies TF32 hi / lo parts (x = hi + lo, hi = x rounded to 10 mantissa
 * bits, lo = x - hi exact) read from an operand arena in the workspace.  in_pass = 1 (default):
 * where the leaf level's S / T are formed by a two-level K1X2 pass and the leaf k and n are
 * multiples of 32, that pass writes the hi / lo pairs of every leaf operand straight into the
 * arena (views included) -- no separate split pass, and the leaf-level S_r / T_r themselves are
 * never written.  in_pass = 0: the pass writes S_r / T_r and a split kernel fills the arena.
 * Both give bitwise the same C.  FMM_E_ARG for other values.  The environment variable
 * FMM_TF32_PRESPLIT=0 sets 0 at fmm_plan_create. */
fmm_status fmm_plan_set_leaf_split(fmm_plan* plan, int in_pass);

/* W-combination levels per pass (host-only; north star item 3, P:119 applied twice).
 * levels = 2 (default): where a level d and its children use built-in 2x2x2 rules (Strassen,
 * Strassen-Winograd, classical: U, V and W tables equal to the built-in ones), one K3X2 launch
 * computes C[k1][k2] = sum_r1 w1_{k1 r1} (sum_r2 w2_{k2 r2} M_{r1 r2}) from the level-(d+2)
 * products into the level-d outputs, in registers, in K3's order (bitwise identical to two
 * K3 passes); the level-(d+1) outputs are never written.  Levels pair from the bottom of the
 * unfused K3 levels.  levels = 1: one K3 pass per level.  FMM_E_ARG for other values.  The
 * environment variable FMM_K3X2=0 sets 1 at fmm_plan_create. */
fmm_status fmm_plan_set_k3_levels(fmm_plan* plan, int levels);

/* Host-only query: number of fused leaf-product launches (K2F) in the compiled schedule. */
fmm_status fmm_plan_fused_launches(const fmm_plan* plan, int64_t* n);

/* ---------------------------------------------------------------------------------------
 * Stability analysis (host-only; Section 4)
 * fmm_rule_quantities: nnz of U, V, W; Q = max_k q_k with q_k = gamma_k + max_r (alpha_r +
 *   beta_r) I(w_kr != 0) (Def. prefactor); E = max_k e_k with e_k = sum_r a_r b_r
 *   |w_kr| (Def. stability), a / b the 1-norms of U / V columns (eqn:ab).
 *   q, e (nullable) receive the m0*n0 vectors (k row-major).
 * fmm_plan_stability: for the plan's recursion tree, xi = max_k xi_k (the largest intermediate
 *   growth, simplified form P:455-463; = prod E for uniform plans) and delta = max_k delta_k
 *   (the largest accumulation error, including the leaf term K / prod K0).
 *   uniform_bound (nullable): the Thm non_stationary_analysis factor (K/prod K0 + sum Q)
 *   (K/prod K0) prod E for uniform plans, NaN for non-uniform ones.
 * fmm_choose_variants: a two-level non-uniform plan -- `root` at level 1 and, at each of its R
 *   children, one of the n_variants rules (same (m0,k0,n0,R), e.g. the Castrapel-Gustafson
 *   variants) -- minimising xi (P:465-475's D'Alberto / <3,2,3> examples do this by
 *   hand).  choice[r] (R entries) receives the variant index of child r; exhaustive search
 *   (lexicographically first minimum) when n_variants^R <= 2^24, else coordinate descent.
 * ------------------------------------------------------------------------------------- */
fmm_status fmm_rule_quantities(const fmm_rule* rule, int64_t* nnz, double* Q, double* E, double* q,
                               double* e);
fmm_status fmm_plan_stability(const fmm_plan* plan, double* xi, double* delta, double* uniform_bound);
fmm_status fmm_choose_variants(const fmm_rule* root, const fmm_rule* const* variants, int n_variants,
                               int32_t* choice, double* xi);

/* Finer multi-GPU sharding (host-only): the units of the partition are the paths
 * (r_1, ..., r_d) of the first d = depth levels of the recursion tree (BFS order; d = 1, the
 * default, is the top-level products), unit u going to rank u mod nranks.  A rank forms, depth-
 * first, only the S / T it needs on the way to its units and accumulates the partial
 * C = sum over its units of the W-weighted products (every level's W applied, r ascending);
 * the ranks' partials sum to A.B (linearity of Eq. eqn:recursive_alg).  With R = 7, d = 2
 * gives 49 units (98 / 94 / 88 % balance at 2 / 4 / 8 ranks), d = 3 gives 343 (99.7 % at 8).
 * 1 <= depth <= levels. */
fmm_status fmm_plan_set_shard_depth(fmm_plan* plan, int depth);

/* Unit order of the multi-GPU partition (host-only): order = 0 (default) round-robin, unit u on
 * rank u mod nranks; order = 1 contiguous blocks, rank p owning units
 * [ceil(p U / nranks), ceil((p + 1) U / nranks)) of the U units -- at shard depth >= 2 a rank's
 * units then share their upper-level paths, so it repeats fewer S / T formation passes on the
 * way down.  fmm_plan_owned reports the assignment.  FMM_E_ARG for other values;
 * FMM_E_UNSUPPORTED together with comm mode 3 (its symmetric buffers are laid out round-robin). */
fmm_status fmm_plan_set_shard_order(fmm_plan* plan, int order);

/* The multi-GPU exchange after the ranks' partial products (host-only; default 0):
 * 0 = ncclReduce(sum) onto rank 0 (C valid on rank 0);
 * 1 = ncclAllReduce(sum) (C valid on every rank);
 * 2 = ncclReduceScatter(sum), in place: rank r's C holds the finished rows
 *     [r M / P, (r + 1) M / P) (M divisible by P, else FMM_E_SHAPE) -- a distributed C at
 *     1 / P of the reduce's per-rank output traffic;
 * 3 = fused NVLink combine: each rank writes its owned top-level products
 *     M_r (r = rank mod P, shard depth 1) into its symmetric buffer (fmm_plan_sym_alloc), and
 *     after a device-side barrier (1-word ncclAllReduce) rank q computes rows
 *     [q M / P, (q + 1) M / P) of C = sum_r w_kr M_r (Eq. eqn:recursive_alg) with one
 *     kernel that loads the peers' products over NVLink (CUDA IPC, fmm_plan_set_peer_handles):
 *     the W-combination and the exchange in one pass, no partial C, and the same summation
 *     order as one GPU (bitwise the single-GPU rows).  A second barrier follows.  Needs no
 *     padding and no scaling (FMM_E_ARG at execute).  Mode 3 recompiles the plan (its schedule
 *     differs). */
fmm_status fmm_plan_set_comm_mode(fmm_plan* plan, int mode);

/* Comm mode 3 buffers.  fmm_plan_sym_bytes: size of this rank's symmetric buffer (ceil(R / P)
 * top-level products of lm[1] x ln[1], slot r / P, plus 256 bytes of barrier scratch).
 * fmm_plan_sym_alloc: cudaMalloc it on the current device (owned by the plan, freed with it)
 * and write its 64-byte CUDA IPC handle to `handle`.  fmm_plan_sym_ptr: its device address.
 * fmm_plan_set_peer_handles: `handles` = n = nranks consecutive 64-byte handles in rank order
 * (this rank's own is not opened); the plan opens the others (cudaIpcOpenMemHandle) and keeps
 * the UVA pointer table.  FMM_E_ARG / FMM_E_CUDA on failure. */
fmm_status fmm_plan_sym_bytes(const fmm_plan* plan, size_t* bytes);
fmm_status fmm_plan_sym_alloc(fmm_plan* plan, void* handle);
fmm_status fmm_plan_sym_ptr(const fmm_plan* plan, void** ptr);
fmm_status fmm_plan_set_peer_handles(fmm_plan* plan, const void* handles, int n);

/* Building block of comm mode 3 (tests, tools): rows [row0, row1) of C (ldc) =
 * sum_r w_kr M_r with M_r at peer_ptrs[r % n] + (r / n) * lm[1] * ln[1] (device pointers:
 * host array of n).  Enqueued on `stream`. */
fmm_status fmm_plan_p2p_combine(fmm_plan* plan, const void* const* peer_ptrs, int n, void* C,
                                int64_t ldc, int64_t row0, int64_t row1, void* stream);

/* Host-only query: owned[u] = 1 if shard unit u is computed by `rank`; *R receives the number
 * of units (the top-level rank R at shard depth 1). */
fmm_status fmm_plan_owned(const fmm_plan* plan, int rank, int nranks, int32_t* owned, int* R);

/* Device workspace (bytes) fmm_execute needs for this plan (and its current partition). */
fmm_status fmm_plan_workspace_bytes(const fmm_plan* plan, size_t* bytes);

/* Kernel launches one fmm_execute issues (for the benchmark's launch accounting). */
fmm_status fmm_plan_launch_count(const fmm_plan* plan, int64_t* launches);

/* Device timing of fmm_execute's launches, per step kind, with CUDA events recorded on the
 * launch stream around each launch (enable = 1) -- for the benchmark's roofline numbers.
 * fmm_plan_step_times returns the totals since the previous call and resets them:
 * ms[k] / launches[k] for k = 1 K1 (S/T formation), 2 K2 (leaf products), 3 K3 (C
 * combination), 4 ACC (top-level accumulation), 5 ZERO, 6 scaling, 7 NCCL reduce (arrays of 8;
 * entry 0 unused).  Synchronises on the recorded events. */
fmm_status fmm_plan_set_timing(fmm_plan* plan, int enable);
fmm_status fmm_plan_step_times(fmm_plan* plan, double* ms, int64_t* launches);

/* CUDA-graph replay (enable = 1): fmm_execute captures its launch sequence into a CUDA graph
 * the first time it sees a given (A, B, C, ws, lda, ldb, ldc) and replays the graph on later
 * calls with the same arguments -- for small, launch-bound problems.  Ignored while timing is
 * enabled or a communicator is attached. */
fmm_status fmm_plan_set_graph(fmm_plan* plan, int enable);

/* C = A.B by the plan (dev pointers).  A: M x K (lda), B: K x N (ldb), C: M x N (ldc),
 * overwritten.  ws: dev workspace of >= fmm_plan_workspace_bytes.  Requirements: A, B, C, ws
 * 16-byte aligned for the vectorised paths (otherwise a scalar path is used).  With a
 * partition (nranks > 1) C receives this rank's partial sum; with a communicator set
 * (fmm_plan_set_comm) the partials are summed onto rank 0's C by ncclReduce. */
fmm_status fmm_execute(const fmm_plan* plan, const void* A, int64_t lda, const void* B,
                       int64_t ldb, void* C, int64_t ldc, void* ws, size_t ws_bytes,
                       void* stream);

/* End-to-end variant with HOST buffers: A_host (M x K, lda), B_host (K x N, ldb) are copied to
 * the caller's device staging buffers A_dev / B_dev (dense, ld = K / N), the product is computed
 * into C_dev (dense, ld = N) and copied back to C_host (ldc).  All copies and kernels are
 * enqueued on `stream`; host buffers should be pinned (cudaHostAlloc / torch pin_memory) for
 * asynchronous copies.  The call returns without synchronising; C_host is valid after the
 * stream completes. */
fmm_status fmm_execute_host(const fmm_plan* plan, const void* A_host, int64_t lda,
                            const void* B_host, int64_t ldb, void* C_host, int64_t ldc,
                            void* A_dev, void* B_dev, void* C_dev, void* ws, size_t ws_bytes,
                            void* stream);

/* A stream of `count` independent products C_i = A_i.B_i with HOST buffers (serving-style
 * batch), each as fmm_execute_host, pipelined across problems: problem i is staged in device
 * buffer set i mod nbuf (A_devs / B_devs / C_devs: nbuf dense device buffers each, ld = K / N /
 * N) and its input copies wait only for the compute of problem i - nbuf (the last reader of that
 * set), so with nbuf = 2 they stream in while problem i - 1 computes, and problem i - 1's C
 * copy-out overlaps problem i's compute.  Compute runs on `stream` in order (one workspace).
 * A_hosts / B_hosts / C_hosts: arrays of count host pointers (pinned for asynchronous copies;
 * C_hosts may repeat a buffer -- its copies are ordered).  Plans outside the per-block copy
 * pipeline (L = 0, scaling, zero padding, communicator) copy whole operands on the copy streams
 * around fmm_execute (still overlapped across problems); nbuf = 1 runs the problems one after
 * another.
 * Returns without synchronising; every C_host is valid after the stream completes.  FMM_E_ARG
 * for null pointers, count < 0, nbuf < 1 or bad ld. */
fmm_status fmm_execute_host_batch(const fmm_plan* plan, int count, const void* const* A_hosts,
                                  int64_t lda, const void* const* B_hosts, int64_t ldb,
                                  void* const* C_hosts, int64_t ldc, void* const* A_devs,
                                  void* const* B_devs, void* const* C_devs, int nbuf, void* ws,
                                  size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------------
 * Building blocks (one recursion node; used by tests and tools)
 * ------------------------------------------------------------------------------------- */
/* All S_r = sum_i u_ir A_i (mb x kb each, stored contiguously at S + r*mb*kb) and
 * T_r = sum_j v_jr B_j (kb x nb, at T + r*kb*nb) of one node, i / j ascending (Eq.
 * eqn:bilinear_alg).  A: m x k (lda), B: k x n (ldb), dev pointers. */
fmm_status fmm_node_st(const fmm_rule* rule, int dtype, int64_t m, int64_t k, int64_t n,
                       const void* A, int64_t lda, const void* B, int64_t ldb, void* S, void* T,
                       void* stream);
/* C_k = sum_r w_kr M_r, r ascending, from R contiguous blocks Ms (mb x nb each) into
 * C (m x n, ldc). */
fmm_status fmm_node_c(const fmm_rule* rule, int dtype, int64_t m, int64_t n, const void* Ms,
                      void* C, int64_t ldc, void* stream);
/* Classical C = A.B (the leaf kernel alone): dev pointers, row-major. */
fmm_status fmm_gemm(int dtype, int leaf, int64_t M, int64_t K, int64_t N, const void* A,
                    int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc, void* stream);

/* ---------------------------------------------------------------------------------------
 * Diagonal scaling (Section 6), FP64 only.  All pointers dev.  The scaled matrices are written
 * to A_out (M x K, lda_out) / B_out (K x N, ldb_out); A and B are not modified.  Factors:
 * dA (M) and dB (N) are the cumulative outer factors D_A, D_B; d (K) the inner factor D.
 * Divisions are true divisions (D^{-1}A), sqrt and division correctly rounded.
 * An all-zero row / column returns FMM_E_PRECOND (this check synchronises the stream).
 * ------------------------------------------------------------------------------------- */
/* Alg. 1 lines 1-4: dA_i = max_j |a_ij|, dB_j = max_i |b_ij|, A' = D_A^{-1} A,
 * B' = B D_B^{-1}. */
fmm_status fmm_scale_outside(int dtype, int64_t M, int64_t K, int64_t N, const void* A,
                             int64_t lda, const void* B, int64_t ldb, void* A_out,
                             int64_t lda_out, void* B_out, int64_t ldb_out, void* dA, void* dB,
                             int pow2, void* stream);
/* Alg. 2 lines 1-3: d_k = sqrt(max_j |b_kj| / max_i |a_ik|), A' = A D,
 * B' = D^{-1} B. */
fmm_status fmm_scale_inside(int dtype, int64_t M, int64_t K, int64_t N, const void* A,
                            int64_t lda, const void* B, int64_t ldb, void* A_out,
                            int64_t lda_out, void* B_out, int64_t ldb_out, void* d, int pow2,
                            void* stream);
/* Alg. 3: alternating O / I steps per `cfg`, with the stopping test of Thm
 * stopping-criterion evaluated ON DEVICE from the step after the first O step.
 * dI (K) receives the cumulative inner factor (reporting only).  steps_dev: dev int32 that
 * receives the number of steps taken (no host synchronisation for the stop test).  ws: dev
 * scratch of fmm_scale_workspace_bytes(M, K, N). */
fmm_status fmm_scale_repeated(int dtype, int64_t M, int64_t K, int64_t N, const void* A,
                              int64_t lda, const void* B, int64_t ldb, const fmm_scaling* cfg,
                              void* A_out, int64_t lda_out, void* B_out, int64_t ldb_out,
                              void* dA, void* dB, void* dI, int32_t* steps_dev, void* ws,
                              size_t ws_bytes, void* stream);
fmm_status fmm_scale_workspace_bytes(int64_t M, int64_t K, int64_t N, size_t* bytes);
/* Apply given diagonal factors (eqn:scaling): A' = D_A^-1 A D, B' = D^-1 B D_B^-1,
 * computed as a'_ik = (a_ik / dA_i) * d_k and b'_kj = (b_kj / d_k) / dB_j (each operation
 * correctly rounded; exact for power-of-two factors, so applying the cumulative factors of
 * fmm_scale_repeated with pow2 = 1 reproduces its A', B' bitwise).  dA (M), d (K), dB (N): device
 * vectors; A_out / B_out: caller device buffers (may not alias A / B).  FP64 only. */
fmm_status fmm_scale_apply(int dtype, int64_t M, int64_t K, int64_t N, const void* A, int64_t lda,
                           const void* B, int64_t ldb, const void* dA, const void* d,
                           const void* dB, void* A_out, int64_t lda_out, void* B_out,
                           int64_t ldb_out, void* stream);

/* Alg. 1 line 6: C <- D_A C D_B in place, c_ij = (dA_i * c_ij) * dB_j. */
fmm_status fmm_unscale(int dtype, int64_t M, int64_t N, void* C, int64_t ldc, const void* dA,
                       const void* dB, void* stream);
/* After an fmm_execute with scaling: copy the last run's step count (host int) -- synchronises
 * the stream. */
fmm_status fmm_plan_last_scaling_steps(const fmm_plan* plan, void* ws, int* steps, void* stream);

/* ---------------------------------------------------------------------------------------
 * Multi-GPU (one process per GPU).  NCCL is loaded at run time (dlopen of libnccl.so.2, or
 * the path in env FMM_NCCL_LIB).  The 128-byte unique id is created on rank 0 and broadcast
 * by the caller (e.g. torch.distributed).
 * ------------------------------------------------------------------------------------- */
fmm_status fmm_comm_unique_id(void* out128);
/* ncclCommInitRank on the current device; attaches the communicator and partition
 * (rank, nranks) to the plan.  fmm_execute then ends with the exchange of
 * fmm_plan_set_comm_mode (default ncclReduce(sum, root 0) of C).  A one-rank communicator
 * (nranks = 1) issues the same collectives (a sum over one rank: C is unchanged, bitwise), so
 * the exchange runs -- and is testable -- on a single GPU.  FMM_E_NCCL if NCCL cannot be
 * loaded or the init fails. */
fmm_status fmm_plan_set_comm(fmm_plan* plan, const void* id128, int rank, int nranks);

/* Single-launch small plans (host-only; default on).  A two-level FP64 plan (no padding, no
 * scaling, one rank) that compiles to one two-level S / T pass, the batched leaf products and
 * one two-level W-combination pass, with at most 4 waves of 32 x 64 leaf tiles (BASELINE C1:
 * Strassen-Winograd L = 2 at 512^3), runs the three as phases of ONE cooperative kernel with
 * grid-wide barriers (launch latency dominates three launches at this size).  Results are
 * bitwise the three-launch schedule's.  enable = 0 keeps three launches. */
fmm_status fmm_plan_set_single_launch(fmm_plan* plan, int enable);

/* Virtual scaling (host-only; default on).  With power-of-two factors (fmm_scaling.pow2 = 1) the
 * whole scaling run (Alg. 1-3) is one cooperative kernel whose steps read the
 * ORIGINAL A and B with the factors applied on the fly (exact: multiplication by powers of two),
 * and the root's S / T formation applies the final factors while it reads A and B, so A' and
 * B' are never written (the paper's "delay updating actual matrix entries").  Results
 * are bitwise those of the materialised form (A', B' written, then the recursion), which the
 * kernel switches to on device whenever an intermediate would not be exact.  enable = 0 forces
 * the materialised form (same kernel, A', B' written at the end).  Plans without power-of-two
 * factors, with zero padding, FP32 or L = 0 always materialise. */
fmm_status fmm_plan_set_virtual_scaling(fmm_plan* plan, int enable);

/* Comm mode 3's barrier, injected (host-only).  fmm_execute calls fn(user, stream) twice per
 * call -- after this rank's products are enqueued, and after its combine -- instead of the
 * 1-word ncclAllReduce; fn must return only when every rank has enqueued up to the same point
 * and the stream's prior work is complete or ordered before any peer's later reads (e.g.
 * synchronise the stream, then a host barrier).  Nonzero return -> FMM_E_NCCL.  With fn set,
 * mode 3 needs no communicator: this is how two processes sharing one GPU test the CUDA-IPC
 * exchange.  fn = NULL restores the NCCL barrier.  Recompiles the plan when it switches mode 3
 * on or off. */
typedef int (*fmm_barrier_fn)(void* user, void* stream);
fmm_status fmm_plan_set_barrier(fmm_plan* plan, fmm_barrier_fn fn, void* user);

/* Thread-local text of the last error (never NULL). */
const char* fmm_last_error(void);
/* Library version string. */
const char* fmm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FMM_B200_H */
