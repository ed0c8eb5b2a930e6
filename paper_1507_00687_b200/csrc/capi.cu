// The C ABI (include/fmm.h): rules, plans (host schedule + device descriptors), execute,
// building blocks, scaling entry points, NCCL glue.
//
// Schedule.  A plan is compiled once into a list of launch Steps:
//   breadth-first:  K1(level 0) .. K1(level L-1), K2(all leaves), K3(level L-1) .. K3(level 0)
//   depth-first at the top level (when the breadth-first workspace is large, or sharded):
//     for each owned top-level r (ascending): K1(root, only column r) -> breadth-first over
//     the subtree r -> ACC (C_k (+)= w_kr M_r)  ...  then ZERO of blocks without contributions.
// Operands are Op descriptors; S_r (T_r) whose U (V) column is a single +1 are not copied: the
// child operand aliases the parent's block (rounding-neutral).  Descriptors are uploaded once.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <queue>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: named ranges for nsys / ncu --nvtx

#include "fmm_internal.h"
#include "builtin_tables.h"

namespace fmm {
int64_t brent_violations(const RuleData& d, int64_t* fi, int64_t* fj, int64_t* fk);
bool transform_rule(const RuleData& d, int kind, RuleData* out);
bool builtin_rule(const std::string& name, RuleData* out);
size_t scale_ws_bytes(int64_t M, int64_t K, int64_t N);
int* scale_flags_ptr(void* ws, int64_t M, int64_t K, int64_t N);
cudaError_t run_scaling_coop(int64_t M, int64_t K, int64_t N, const double* A, int64_t lda,
                             const double* B, int64_t ldb, double* A_out, int64_t lda_out,
                             double* B_out, int64_t ldb_out, double* dA, double* dB, double* dI,
                             int nsteps, bool first_O, double tau, int pow2, int materialise_end,
                             void* sws, cudaStream_t st);
void scale_virtual_view(void* sws, int64_t M, int64_t K, int64_t N, const int32_t** exAr,
                        const int32_t** exAc, const int32_t** exBr, const int32_t** exBc,
                        const int** mode_flag, const int** ext);
cudaError_t launch_unscale(double* C, int64_t ldc, int64_t M, int64_t N, const double* dA,
                           const double* dB, cudaStream_t st);
cudaError_t launch_scale_apply(int64_t M, int64_t K, int64_t N, const double* A, int64_t lda,
                               const double* B, int64_t ldb, const double* dA, const double* d,
                               const double* dB, double* A_out, int64_t lda_out, double* B_out,
                               int64_t ldb_out, cudaStream_t st);

static thread_local std::string g_err = "no error";
void set_error(const std::string& msg) { g_err = msg; }
fmm_status cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return FMM_OK;
  set_error(std::string(where) + ": " + cudaGetErrorString(e));
  if (e == cudaErrorMemoryAllocation) return FMM_E_OOM;
  if (e == cudaErrorNotSupported) return FMM_E_UNSUPPORTED;
  return FMM_E_CUDA;
}
}  // namespace fmm

using namespace fmm;

// ---------------------------------------------------------------------------------------------
// NCCL (dlopen'ed; types mirrored from nccl.h 2.x ABI)
// ---------------------------------------------------------------------------------------------
namespace {
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
enum { ncclSum_ = 0 };
enum { ncclFloat32_ = 7, ncclFloat64_ = 8 };

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*reduce)(const void*, void*, size_t, int, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allreduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*reduce_scatter)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
};

NcclApi* nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = getenv("FMM_NCCL_LIB");
    const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      if (!n) continue;
      api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (!api.h) return;
    api.getUniqueId = (decltype(api.getUniqueId))dlsym(api.h, "ncclGetUniqueId");
    api.commInitRank = (decltype(api.commInitRank))dlsym(api.h, "ncclCommInitRank");
    api.reduce = (decltype(api.reduce))dlsym(api.h, "ncclReduce");
    api.allreduce = (decltype(api.allreduce))dlsym(api.h, "ncclAllReduce");
    api.reduce_scatter = (decltype(api.reduce_scatter))dlsym(api.h, "ncclReduceScatter");
    api.commDestroy = (decltype(api.commDestroy))dlsym(api.h, "ncclCommDestroy");
    api.getErrorString = (decltype(api.getErrorString))dlsym(api.h, "ncclGetErrorString");
  });
  if (!api.h || !api.getUniqueId || !api.commInitRank || !api.reduce) return nullptr;
  return &api;
}
}  // namespace

// ---------------------------------------------------------------------------------------------
// Plan
// ---------------------------------------------------------------------------------------------
struct fmm_plan {
  int dtype = FMM_F64, leaf = FMM_LEAF_NATIVE, L = 0;
  int64_t M = 0, K = 0, N = 0;
  // zero padding: the recursion runs on Mp x Kp x Np, the smallest multiples of
  // prod m0, prod k0, prod n0; A, B are copied into zero-padded workspace buffers and C is
  // cropped back.  padded = false when the dims already divide.
  int64_t Mp = 0, Kp = 0, Np = 0;
  bool padded = false;
  size_t pad_bytes = 0;
  std::vector<RuleData> rules;              // distinct rules
  std::vector<std::vector<int>> node_rule;  // per level, rule index per node (BFS)
  std::vector<int64_t> lm, lk, ln;          // node dims at level l (l = 0..L)
  fmm_scaling scaling{FMM_SCALE_NONE, 1, 1.0, 20, 0};
  int rank = 0, nranks = 1;
  int schedule = 0;  // 0 auto, 1 breadth-first, 2 depth-first top level
  int fusion = 2;    // W-combination of the leaves' parents in the leaf GEMM epilogue: 0 off, 1 on, 2 auto
  int shard_depth = 1;  // multi-GPU: units = paths of the first shard_depth levels, round-robin
  bool shard_block = false;  // units to ranks in contiguous blocks (else round-robin u mod nranks)
  int comm_mode = 0;    // multi-GPU exchange: 0 reduce to rank 0, 1 all-reduce, 2 reduce-scatter
  bool split_chains = true;     // fused units' product chains split over CTAs (turnstiles)
  bool k1_two_level = true;     // S / T of two recursion levels formed in one pass (K1X2)
  bool tf32_presplit = true;    // FP32 tensor-core leaves: the leaf level's K1X2 writes the
                                // hi / lo operand arena (no separate split pass)
  bool k3_two_level = true;     // W-combination of two recursion levels in one pass (K3X2)
  // virtual scaling (compile_plan): power-of-two factors applied by the root K1 while it forms
  // S_r / T_r from the original A, B (the scaled A', B' are not written)
  bool virt_scale = false;
  bool virt_scale_enable = true;  // fmm_plan_set_virtual_scaling
  bool single_launch = true;      // fmm_plan_set_single_launch: small two-level plans as one kernel
  bool unscale_fused = false;     // the root K3 / K3X2 applies the unscale
  ncclComm_t comm = nullptr;
  // comm mode 3 barrier (fmm_plan_set_barrier): called instead of the 1-word NCCL all-reduce
  fmm_barrier_fn barrier_fn = nullptr;
  void* barrier_user = nullptr;
  // compiled schedule
  std::vector<Step> steps;
  std::vector<int> coef_U, coef_V, coef_W;  // per rule: offset in coef buffer (doubles)
  std::vector<double> coef_host;
  std::vector<uint8_t> desc_host;  // descriptor arena (host copy)
  // device copies, uploaded lazily on first use so that plans can be built without a GPU
  mutable std::mutex dev_mu;
  mutable double* dev_coef = nullptr;
  mutable void* dev_desc = nullptr;
  mutable int dev_id = -1;
  size_t desc_bytes = 0;
  size_t fmm_ws_bytes = 0;     // FMM temporaries
  size_t scale_bytes = 0;      // scaling region (A', B', factors, scratch), placed first
  bool dims_vec_ok = true;     // every level's column dims / offsets multiple of the vector
  int64_t launches = 0;
  // depth-first top level: steps [begin, end) of top-level product r (for host-copy overlap)
  struct RGroup {
    int r;
    size_t begin, end;
  };
  std::vector<RGroup> groups;
  mutable cudaStream_t copy_h2d = nullptr, copy_d2h = nullptr;
  mutable int copy_dev = -1;
  // breadth-first plans: a depth-first twin used by fmm_execute_host to overlap the copies
  mutable fmm_plan* df_twin = nullptr;
  // optional CUDA-graph replay of fmm_execute
  bool use_graph = false;
  struct GraphEntry {
    const void *A, *B, *C, *ws;
    int64_t lda, ldb, ldc;
    cudaGraphExec_t exec;
  };
  mutable std::vector<GraphEntry> graphs;
  // comm mode 3 is live: products go to the symmetric buffer and, with a communicator or an
  // injected barrier, the fused combine runs (a one-rank communicator / barrier exercises the
  // exchange on one GPU; several ranks without either are the virtual-rank building block)
  bool p2p_active() const {
    return comm_mode == 3 && L > 0 && shard_depth == 1 && (nranks > 1 || comm || barrier_fn);
  }
  mutable std::mutex gmu;
  // optional per-step timing (events recorded on the launch stream)
  bool timing = false;
  mutable std::mutex tmu;
  mutable std::vector<cudaEvent_t> ev_pool;
  mutable std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_used;
  // comm mode 3 (fused NVLink combine): this rank's symmetric buffer of owned top-level
  // products (library-allocated, exported by CUDA IPC) and every rank's buffer as a UVA pointer
  void* sym_own = nullptr;
  size_t sym_alloc_bytes = 0;
  std::vector<void*> peers;          // [nranks]; peers[rank] = sym_own, others IPC-opened
  std::vector<bool> peer_opened;
  void* dev_peers = nullptr;         // device copy of peers
  void* dev_tmp_peers = nullptr;     // fmm_plan_p2p_combine's pointer table
  ~fmm_plan();
};

fmm_plan::~fmm_plan() {
  delete df_twin;
  for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
  if (copy_h2d) cudaStreamDestroy(copy_h2d);
  if (copy_d2h) cudaStreamDestroy(copy_d2h);
  for (auto& u : ev_used) { cudaEventDestroy(u.second.first); cudaEventDestroy(u.second.second); }
  for (auto e : ev_pool) cudaEventDestroy(e);
  if (dev_coef) cudaFree(dev_coef);
  if (dev_desc) cudaFree(dev_desc);
  if (comm && nccl() && nccl()->commDestroy) nccl()->commDestroy(comm);
  for (size_t q = 0; q < peers.size(); ++q)
    if (q < peer_opened.size() && peer_opened[q] && peers[q]) cudaIpcCloseMemHandle(peers[q]);
  if (dev_peers) cudaFree(dev_peers);
  if (dev_tmp_peers) cudaFree(dev_tmp_peers);
  if (sym_own) cudaFree(sym_own);
}

namespace {

constexpr size_t kHybridMaxWs = (size_t)64 << 30;  // hybrid top-level schedule: workspace cap
constexpr int64_t kK2fSmallK = 1024;  // leaf inner dimension up to which K2F uses 64 x 64 tiles

int elem_size(int dtype) { return dtype == FMM_F64 ? 8 : 4; }

struct Builder {
  fmm_plan* p;
  std::vector<uint8_t> desc;  // host copy of the descriptor arena
  int64_t ws_elems = 0, ws_peak = 0;
  int64_t align_elems;

  explicit Builder(fmm_plan* pl) : p(pl) { align_elems = 256 / elem_size(pl->dtype); }

  int64_t ws_alloc(int64_t elems) {
    int64_t off = ws_elems;
    ws_elems += (elems + align_elems - 1) / align_elems * align_elems;
    ws_peak = std::max(ws_peak, ws_elems);
    return off;
  }
  template <typename T>
  int64_t push(const std::vector<T>& v) {
    size_t off = (desc.size() + 255) / 256 * 256;
    desc.resize(off + v.size() * sizeof(T));
    std::memcpy(desc.data() + off, v.data(), v.size() * sizeof(T));
    return (int64_t)off;
  }
  Op ws_op(int64_t off, int64_t ld) { return Op{BASE_WS, 0, 0, off, ld}; }
  static Op sub(const Op& o, int64_t r0, int64_t c0) {
    return Op{o.base, 0, o.row0 + r0, o.col0 + c0, o.ld};
  }

  // one node of the active set at level l
  struct Node {
    int64_t idx;  // BFS index within level
    Op a, b, c;
  };

  const RuleData& rule_at(int l, int64_t idx) { return p->rules[p->node_rule[l][idx]]; }

  static bool trivial_col(const RuleData& r, const std::vector<int32_t>& X, int rows, int col,
                          int* only_row) {
    int nz = 0, row = -1;
    for (int i = 0; i < rows; ++i)
      if (X[(size_t)i * r.R + col] != 0) { ++nz; row = i; }
    if (nz == 1 && X[(size_t)row * r.R + col] == (1 << r.log2den)) { *only_row = row; return true; }
    return false;
  }

  // K1 for the active nodes of level l (columns in `only_r` if >= 0); returns child nodes.
  std::vector<Node> emit_k1(int l, const std::vector<Node>& nodes, int only_r, bool alloc_c = true) {
    const int64_t mb = p->lm[l + 1], kb = p->lk[l + 1], nb = p->ln[l + 1];
    // virtual scaling: the root's children are scaled copies, never views of A / B
    const bool noalias = l == 0 && p->virt_scale;
    std::vector<K1Node> ks, kt;
    std::vector<Node> kids;
    for (const Node& nd : nodes) {
      const RuleData& ru = rule_at(l, nd.idx);
      K1Node s{};
      s.in = nd.a;
      s.rows = mb; s.cols = kb; s.P = ru.m0; s.Q = ru.k0; s.tv = 0;
      s.coef_off = p->coef_U[p->node_rule[l][nd.idx]];
      K1Node t{};
      t.in = nd.b;
      t.rows = kb; t.cols = nb; t.P = ru.k0; t.Q = ru.n0; t.tv = 1;
      t.coef_off = p->coef_V[p->node_rule[l][nd.idx]];
      for (int r = 0; r < ru.R; ++r) {
        if (only_r >= 0 && r != only_r) continue;
        Node ch;
        ch.idx = nd.idx * ru.R + r;
        int row;
        if (!noalias && trivial_col(ru, ru.U, ru.m0 * ru.k0, r, &row)) {
          ch.a = sub(nd.a, (row % ru.m0) * mb, (row / ru.m0) * kb);
        } else {
          ch.a = ws_op(ws_alloc(mb * kb), kb);
          s.out[r] = ch.a;
          s.out_mask |= 1u << r;
        }
        if (!noalias && trivial_col(ru, ru.V, ru.k0 * ru.n0, r, &row)) {
          ch.b = sub(nd.b, (row % ru.k0) * kb, (row / ru.k0) * nb);
        } else {
          ch.b = ws_op(ws_alloc(kb * nb), nb);
          t.out[r] = ch.b;
          t.out_mask |= 1u << r;
        }
        if (alloc_c) ch.c = ws_op(ws_alloc(mb * nb), nb);
        kids.push_back(ch);
      }
      k1_compile(s, ru, ru.U, ru.m0 * ru.k0);
      k1_compile(t, ru, ru.V, ru.k0 * ru.n0);
      if (s.out_mask) ks.push_back(s);
      if (t.out_mask) kt.push_back(t);
    }
    // every S_r and T_r of the level in one launch (per-node dims in the descriptors)
    const RuleData& r0 = rule_at(l, nodes[0].idx);
    std::vector<K1Node> all = ks;
    all.insert(all.end(), kt.begin(), kt.end());
    if (!all.empty()) {
      Step st{};
      st.kind = STEP_K1;
      st.count = (int)all.size();
      st.dev_off = push(all);
      st.rows = ks.empty() ? kb : kt.empty() ? mb : std::max(mb, kb);
      st.cols = ks.empty() ? nb : kt.empty() ? kb : std::max(kb, nb);
      const int blk = std::max(ks.empty() ? 0 : r0.m0 * r0.k0, kt.empty() ? 0 : r0.k0 * r0.n0);
      st.P = blk; st.Q = 1; st.R = r0.R;  // P * Q: max input sub-blocks of a node
      st.scaled = noalias ? 1 : 0;
      {  // every node on one built-in rule: the compile-time specialised kernel
        const int id = builtin_id(r0);
        bool same = id != kBuiltinNone;
        for (const Node& nd : nodes) same = same && p->node_rule[l][nd.idx] == p->node_rule[l][nodes[0].idx];
        st.x1 = same ? 1 + id : 0;
      }
      p->steps.push_back(st);
    }
    return kids;
  }

  // Built-in rule id of a rule (builtin_tables.h) if its U, V and W tables are exactly one of
  // them, else kBuiltinNone.
  static int builtin_id(const RuleData& r) {
    if (r.m0 != 2 || r.k0 != 2 || r.n0 != 2 || r.log2den != 0) return kBuiltinNone;
    for (int id = 0; id < 3; ++id) {
      if (builtin_R(id) != r.R) continue;
      bool eq = true;
      for (int b = 0; b < 4 && eq; ++b)
        for (int q = 0; q < r.R && eq; ++q)
          eq = r.U[(size_t)b * r.R + q] == builtin_coef(id, 0, b, q) &&
               r.V[(size_t)b * r.R + q] == builtin_coef(id, 1, b, q) &&
               r.W[(size_t)b * r.R + q] == builtin_w(id, b, q);
      if (eq) return id;
    }
    return kBuiltinNone;
  }

  // K1X2 rule pair (1 + 3 * id_d + id_{d+1}) of levels (d, d+1) for `nodes` (level d), or 0:
  // every node of level d and every child use one built-in rule per level.
  int k1x2_pair(int d, const std::vector<Node>& nodes) {
    if (d + 2 > p->L || nodes.empty()) return 0;
    const int rule1 = p->node_rule[d][nodes[0].idx];
    const int ra = builtin_id(p->rules[rule1]);
    if (ra == kBuiltinNone) return 0;
    const int R1 = p->rules[rule1].R;
    const int rule2 = p->node_rule[d + 1][nodes[0].idx * R1];
    const int rb = builtin_id(p->rules[rule2]);
    if (rb == kBuiltinNone) return 0;
    for (const Node& nd : nodes) {
      if (p->node_rule[d][nd.idx] != rule1) return 0;
      for (int r = 0; r < R1; ++r)
        if (p->node_rule[d + 1][nd.idx * R1 + r] != rule2) return 0;
    }
    return 1 + 3 * ra + rb;
  }

  // Levels d and d+1 of S / T formation in one K1X2 launch.  Returns the children (level d+1:
  // products M_{r1}, only c allocated -- their S / T are never formed) and the grandchildren
  // (level d+2, operands formed or views, c allocated if alloc_c), both in BFS order.  The
  // formed outputs are listed r1-major, r2 ascending: the kernel's compile-time order.
  // split: the grandchildren are the leaves of an FP32 tensor-core K2 step; every S / T of them
  // (views too) is written as its TF32 hi / lo pair straight into that step's operand arena
  // (allocated here, leaf index = BFS position; A side m x k K-major, B side k x n MN-major:
  // exactly the K1X2 output layout when k and n are multiples of 32), which emit_k2 picks up.
  std::pair<std::vector<Node>, std::vector<Node>> emit_k1x2(int d, const std::vector<Node>& nodes,
                                                            int pair, bool alloc_c, bool split = false) {
    const int ra = (pair - 1) / 3, rb = (pair - 1) % 3;
    const int64_t mb1 = p->lm[d + 1], kb1 = p->lk[d + 1], nb1 = p->ln[d + 1];
    const int64_t mb = p->lm[d + 2], kb = p->lk[d + 2], nb = p->ln[d + 2];
    const int R1 = builtin_R(ra), R2 = builtin_R(rb);
    std::vector<K1x2Node> ks, kt;
    std::vector<Node> kids, grand;
    const int64_t nleaves = (int64_t)nodes.size() * R1 * R2;
    int64_t arena = -1, slab_a = mb * kb, slab_b = kb * nb;
    if (split) {
      arena = ws_alloc((int64_t)tf32_arena_floats(nleaves, mb, nb, kb));
      pending_arena = arena;
      pending_leaves = nleaves;
    }
    int64_t leaf = 0;
    for (const Node& nd : nodes) {
      K1x2Node s{}, t{};
      s.in = nd.a; s.rows = mb; s.cols = kb; s.tv = 0;
      t.in = nd.b; t.rows = kb; t.cols = nb; t.tv = 1;
      if (split) {
        s.lo_off = nleaves * slab_a;
        t.lo_off = nleaves * slab_b;
        for (int r1 = 0; r1 < R1; ++r1) {
          Node ch;
          ch.idx = nd.idx * R1 + r1;
          ch.a = Op{}; ch.b = Op{};
          ch.c = ws_op(ws_alloc(mb1 * nb1), nb1);
          kids.push_back(ch);
          for (int r2 = 0; r2 < R2; ++r2, ++leaf) {
            Node g;
            g.idx = ch.idx * R2 + r2;
            g.a = ws_op(arena + leaf * slab_a, kb);                           // S hi (m x k)
            g.b = ws_op(arena + 2 * nleaves * slab_a + leaf * slab_b, nb);    // T hi (k x n)
            s.out[s.nout++] = g.a;
            t.out[t.nout++] = g.b;
            if (alloc_c) g.c = ws_op(ws_alloc(mb * nb), nb);
            grand.push_back(g);
          }
        }
        ks.push_back(s);
        kt.push_back(t);
        continue;
      }
      for (int r1 = 0; r1 < R1; ++r1) {
        Node ch;
        ch.idx = nd.idx * R1 + r1;
        ch.a = Op{}; ch.b = Op{};  // not formed
        ch.c = ws_op(ws_alloc(mb1 * nb1), nb1);
        kids.push_back(ch);
        for (int r2 = 0; r2 < R2; ++r2) {
          Node g;
          g.idx = ch.idx * R2 + r2;
          if (builtin_trivial(ra, 0, r1) && builtin_trivial(rb, 0, r2)) {  // a view of one block
            int b1 = 0, b2 = 0;
            while (builtin_coef(ra, 0, b1, r1) == 0) ++b1;
            while (builtin_coef(rb, 0, b2, r2) == 0) ++b2;
            g.a = sub(sub(nd.a, (b1 % 2) * mb1, (b1 / 2) * kb1), (b2 % 2) * mb, (b2 / 2) * kb);
          } else {
            g.a = ws_op(ws_alloc(mb * kb), kb);
            s.out[s.nout++] = g.a;
          }
          if (builtin_trivial(ra, 1, r1) && builtin_trivial(rb, 1, r2)) {
            int b1 = 0, b2 = 0;
            while (builtin_coef(ra, 1, b1, r1) == 0) ++b1;
            while (builtin_coef(rb, 1, b2, r2) == 0) ++b2;
            g.b = sub(sub(nd.b, (b1 % 2) * kb1, (b1 / 2) * nb1), (b2 % 2) * kb, (b2 / 2) * nb);
          } else {
            g.b = ws_op(ws_alloc(kb * nb), nb);
            t.out[t.nout++] = g.b;
          }
          if (alloc_c) g.c = ws_op(ws_alloc(mb * nb), nb);
          grand.push_back(g);
        }
      }
      if (s.nout) ks.push_back(s);
      if (t.nout) kt.push_back(t);
    }
    std::vector<K1x2Node> all = ks;
    all.insert(all.end(), kt.begin(), kt.end());
    if (!all.empty()) {
      Step st{};
      st.kind = STEP_K1;
      st.x2 = pair;
      st.count = (int)all.size();
      st.dev_off = push(all);
      st.rows = ks.empty() ? kb : kt.empty() ? mb : std::max(mb, kb);
      st.cols = ks.empty() ? nb : kt.empty() ? kb : std::max(kb, nb);
      st.P = 4; st.Q = 1; st.R = R1;
      st.tf32_split = split ? 1 : 0;
      p->steps.push_back(st);
    }
    return {kids, grand};
  }

  // FP32 tensor-core leaves of dims m x k x n can take their hi / lo operands from the leaf
  // level's K1X2 (emit_k1x2 split mode)
  bool presplit_ok() const {
    const int64_t m = p->lm[p->L], k = p->lk[p->L], n = p->ln[p->L];
    return p->dtype == FMM_F32 && p->leaf != FMM_LEAF_NATIVE && p->tf32_presplit &&
           m > 0 && k > 0 && n > 0 && k % 32 == 0 && n % 32 == 0;
  }
  int64_t pending_arena = -1, pending_leaves = 0;  // a K1X2 split-mode arena for the next K2

  void emit_k2(const std::vector<Node>& leaves) {
    std::vector<LeafNode> lf;
    for (const Node& n : leaves) lf.push_back(LeafNode{n.a, n.b, n.c});
    Step st{};
    st.kind = STEP_K2;
    st.count = (int)lf.size();
    st.dev_off = push(lf);
    st.rows = p->lm[p->L]; st.cols = p->ln[p->L]; st.inner = p->lk[p->L];
    st.arena_off = -1;
    if (p->dtype == FMM_F32 && p->leaf != FMM_LEAF_NATIVE) {
      if (pending_arena >= 0 && pending_leaves == (int64_t)lf.size()) {  // filled by the K1X2
        st.arena_off = pending_arena;
        st.tf32_split = 1;
      } else {
        st.arena_off = ws_alloc((int64_t)tf32_arena_floats(st.count, st.rows, st.cols, st.inner));
      }
    }
    pending_arena = -1;
    pending_leaves = 0;
    p->steps.push_back(st);
  }

  // Is the leaf-parent level fused (K2F) for `nparents` parents?  FP64 only.  A fused CTA runs
  // all R products of its parent's tile (or a chunk of them, chains split with turnstiles), so
  // the fused grid has up to R times fewer, longer CTAs than the unfused leaf GEMM; auto mode
  // fuses when that grid (parents x 128x128 output tiles of a leaf, one CTA per SM) fills the
  // 148 SMs in >= 4 waves at >= 90 % wave efficiency, or when a chain split brings the
  // simulated efficiency to >= 93 % (measured: profiles/r01_fusion_variants.md).

  // Simulated makespan (in product durations) of the fused grid when each unit's R-product
  // chain is split into consecutive groups of products, dispatched group-major onto kSMs
  // slots as they free up (the tickets), each item costing its products plus a pipeline fill of
  // STAGES / KT products; group g of a unit cannot finish before group g-1 of that unit.
  // `ends` = the groups' product ends (ascending, the last = R).
  static double fused_makespan(int64_t units, const std::vector<int>& ends, int KT, int kSMs) {
    const double fill = 4.0 / std::max(KT, 1);
    std::priority_queue<double, std::vector<double>, std::greater<double>> sm;
    for (int i = 0; i < kSMs; ++i) sm.push(0.0);
    std::vector<double> prev(units, 0.0);
    double span = 0;
    for (size_t g = 0; g < ends.size(); ++g) {
      const int np = ends[g] - (g ? ends[g - 1] : 0);
      for (int64_t u = 0; u < units; ++u) {
        const double start = sm.top();
        sm.pop();
        const double fin = std::max(start + np + fill, g ? prev[u] + 0.1 : 0.0);
        sm.push(fin);
        prev[u] = fin;
        span = std::max(span, fin);
      }
    }
    return span;
  }
  static uint32_t pack_split(const std::vector<int>& ends) {
    if (ends.size() <= 1) return 0u;
    uint32_t s = 0;
    for (size_t g = 0; g < ends.size(); ++g) s |= (uint32_t)ends[g] << (8 * g);
    return s;
  }
  // best chain split for a fused leaf level (0: none) among 2 and 3 groups (any cut points for
  // R <= 8, else near-equal groups); the simulated efficiency out
  static uint32_t best_split(int64_t units, int R, int KT, int slots, double* eff) {
    std::vector<int> best{R};
    double best_span = fused_makespan(units, best, KT, slots);
    if (KT >= 4 && units <= (1 << 16) && R <= 255) {
      std::vector<std::vector<int>> cand;
      if (R <= 8) {
        for (int a = 1; a < R; ++a) {
          cand.push_back({a, R});
          for (int b2 = a + 1; b2 < R; ++b2) cand.push_back({a, b2, R});
        }
      } else {
        cand.push_back({(R + 1) / 2, R});
        cand.push_back({(R + 2) / 3, 2 * ((R + 2) / 3), R});
      }
      for (const auto& c : cand) {
        const double sp = fused_makespan(units, c, KT, slots);
        // take a split the model rates >= 0.1 % faster (C3: 6 + 1 modelled 0.16 %, measured
        // 0.6 % faster than no split; profiles/r02_k2f_split_sweep.md)
        if (sp < best_span * 0.999) { best_span = sp; best = c; }
      }
    }
    if (eff) *eff = (double)units * R / ((double)slots * best_span);
    return pack_split(best);
  }

  // K2F tile configuration for this plan's leaves: the 64 x 64 tile kernel (v13, 3 CTAs per
  // SM, so one CTA's epilogue overlaps two others' mainloops) for short leaf inner dimensions,
  // the 128 x 128 kernel (v16, one CTA per SM) otherwise (profiles/r01_fusion_variants.md).
  int k2f_cfg() const {
    if (p->lk[p->L] > kK2fSmallK) return 16;
    for (int ri : p->node_rule[p->L - 1]) {  // v13 holds the tables of 2x2 rules with R <= 8
      const RuleData& r = p->rules[ri];
      if (r.R > 8 || r.m0 * r.n0 > 4) return 16;
    }
    return 13;
  }
  int k2f_tile() const { return k2f_tile_of(k2f_cfg()); }
  int k2f_slots() const { return k2f_cfg() == 13 ? 3 * 148 : 148;
  }

  bool fuse_leaves(int64_t nparents) const {
    // FP64 only: the FP32 tensor-core leaves keep their products in TMEM chunk buffers and
    // register totals (k2p_tf32) and are combined by K3 (a fused FP32 epilogue,
    // k2f_tf32, measured slower at C5 in round 1 -- 310 vs 287 ms -- and was removed in round 2)
    if (p->dtype != FMM_F64 || p->fusion == 0) return false;
    if (p->fusion == 1) return true;
    {  // chain splitting (turnstiles) smooths the wave quantisation of R-product units
      const int ts = k2f_tile();
      const int64_t tiles = ((p->lm[p->L] + ts - 1) / ts) * ((p->ln[p->L] + ts - 1) / ts);
      const int R = p->rules[p->node_rule[p->L - 1][0]].R;
      const int KT = (int)((p->lk[p->L] + 15) / 16);
      const int slots = k2f_slots();
      double eff = 0;
      if (p->split_chains && KT >= 4 && nparents * tiles >= slots && nparents * tiles * R >= 4 * slots) {
        best_split(nparents * tiles, R, KT, slots, &eff);
        if (eff >= 0.93) return true;
      }
    }
    constexpr int64_t kSMs = 148;
    const int64_t tiles = ((p->lm[p->L] + 127) / 128) * ((p->ln[p->L] + 127) / 128);
    const int64_t units = nparents * tiles;
    const int64_t waves = (units + kSMs - 1) / kSMs;
    return waves >= 4 && units * 10 >= waves * kSMs * 9;
  }

  // K2F over parents at level l with their leaf children `kids` (R per parent, in order; or
  // one child per parent, product `only_r`, when only_r >= 0).  `started` carries, per
  // parent, the C blocks already initialised (depth-first top level).
  void emit_k2f(int l, const std::vector<Node>& parents, const std::vector<Node>& kids, int only_r,
                uint32_t* started_ext) {
    std::vector<FusedNode> fz;
    size_t ci = 0;
    for (const Node& nd : parents) {
      const RuleData& ru = rule_at(l, nd.idx);
      FusedNode f{};
      f.out = nd.c;
      f.coef_off = p->coef_W[p->node_rule[l][nd.idx]];
      uint32_t started = started_ext ? *started_ext : 0u;
      for (int r = 0; r < ru.R; ++r) {
        if (only_r >= 0 && r != only_r) continue;
        const Node& ch = kids[ci++];
        uint32_t wm = 0;
        for (int k = 0; k < ru.m0 * ru.n0; ++k)
          if (ru.W[(size_t)k * ru.R + r] != 0) wm |= 1u << k;
        f.rlist[f.nr] = (uint8_t)r;
        f.wmask[f.nr] = wm;
        f.first[f.nr] = wm & ~started;
        f.a[f.nr] = ch.a;
        f.b[f.nr] = ch.b;
        started |= wm;
        ++f.nr;
      }
      if (started_ext) *started_ext = started;
      fz.push_back(f);
    }
    const RuleData& r0 = rule_at(l, parents[0].idx);
    Step st{};
    st.kind = STEP_K2F;
    st.count = (int)fz.size();
    st.dev_off = push(fz);
    st.rows = p->lm[p->L]; st.cols = p->ln[p->L]; st.inner = p->lk[p->L];
    st.P = r0.m0; st.Q = r0.n0; st.R = r0.R;
    st.nr = fz[0].nr;
    st.arena_off = -1;
    // chain split with per-unit turnstiles (breadth-first levels: every parent has all R products)
    st.k2f_cfg = k2f_cfg();
    st.unitw = true;
    for (const Node& nd : parents) {
      const RuleData& ru = rule_at(l, nd.idx);
      for (int kk = 0; kk < ru.m0 * ru.n0; ++kk)
        for (int r = 0; r < ru.R; ++r) {
          const double w = ru.coef(ru.W, kk, r);
          if (w != 0.0 && w != 1.0 && w != -1.0) st.unitw = false;
        }
    }
    if (p->split_chains && fz.size() > 0 && fz[0].nr == r0.R && (st.inner + 15) / 16 >= 4) {
      const int ts = k2f_tile();
      const int64_t tiles = ((st.rows + ts - 1) / ts) * ((st.cols + ts - 1) / ts);
      uint32_t sp = best_split((int64_t)st.count * tiles, r0.R, (int)((st.inner + 15) / 16),
                               k2f_slots(), nullptr);
      if (const char* e = getenv("FMM_K2F_SPLIT")) sp = (uint32_t)strtoul(e, nullptr, 0);  // tuning
      if (split_groups(sp, r0.R) > 1) {
        st.split = sp;
        st.turn_off = ws_alloc((st.count * tiles + 2) / 2);  // count*tiles + 1 ints, in 8-byte elements
      }
    }
    p->steps.push_back(st);
  }

  // The root's W-combination writes C once: a scaled plan folds its unscale in there
  // (C = (d_A,i C'_ij) d_B,j, the same two roundings as the separate pass).
  bool root_unscale(int l) const {
    return l == 0 && p->scaling.mode != FMM_SCALE_NONE && !p->padded && p->dtype == FMM_F64;
  }

  // K3 for nodes of level l whose children are `kids` (R per node, in order).
  void emit_k3(int l, const std::vector<Node>& nodes, const std::vector<Node>& kids) {
    std::vector<K3Node> k3;
    size_t ci = 0;
    for (const Node& nd : nodes) {
      const RuleData& ru = rule_at(l, nd.idx);
      K3Node kn{};
      kn.out = nd.c;
      kn.coef_off = p->coef_W[p->node_rule[l][nd.idx]];
      for (int r = 0; r < ru.R; ++r) kn.in[r] = kids[ci++].c;
      k3.push_back(kn);
    }
    const RuleData& r0 = rule_at(l, nodes[0].idx);
    Step st{};
    st.kind = STEP_K3;
    st.count = (int)k3.size();
    st.dev_off = push(k3);
    st.rows = p->lm[l + 1]; st.cols = p->ln[l + 1]; st.P = r0.m0; st.Q = r0.n0; st.R = r0.R;
    st.unscale = root_unscale(l) ? 1 : 0;
    p->steps.push_back(st);
  }

  // K3X2: levels d and d+1 of the W-combination in one pass, from the grandchildren's products
  // (level d+2 c blocks) straight into the level-d nodes' outputs.
  void emit_k3x2(int d, const std::vector<Node>& nodes, const std::vector<Node>& grand, int pair) {
    const int ra = (pair - 1) / 3, rb = (pair - 1) % 3;
    const int n = builtin_R(ra) * builtin_R(rb);
    std::vector<K3x2Node> k3;
    size_t gi = 0;
    for (const Node& nd : nodes) {
      K3x2Node kn{};
      kn.out = nd.c;
      kn.rows = p->lm[d + 2]; kn.cols = p->ln[d + 2];
      for (int q = 0; q < n; ++q) kn.in[q] = grand[gi++].c;
      k3.push_back(kn);
    }
    Step st{};
    st.kind = STEP_K3;
    st.x2 = pair;
    st.count = (int)k3.size();
    st.dev_off = push(k3);
    st.rows = p->lm[d + 2]; st.cols = p->ln[d + 2]; st.P = 2; st.Q = 2; st.R = builtin_R(ra);
    st.unscale = root_unscale(d) ? 1 : 0;
    p->steps.push_back(st);
  }

  // W-combination levels top .. l (bottom-up); two levels per pass (K3X2) paired from the
  // bottom where the rules allow.  lv[q] = the nodes of level l + q.
  void emit_k3_levels(int l, int top, const std::vector<std::vector<Node>>& lv, int stop = -1) {
    if (stop < l) stop = l;  // levels below `stop` are combined by the caller
    for (int d = top; d >= stop;) {
      const int pr = p->k3_two_level && d - 1 >= stop ? k1x2_pair(d - 1, lv[d - 1 - l]) : 0;
      if (pr) {
        emit_k3x2(d - 1, lv[d - 1 - l], lv[d + 1 - l], pr);
        d -= 2;
      } else {
        emit_k3(d, lv[d - l], lv[d - l + 1]);
        d -= 1;
      }
    }
  }

  // breadth-first over the subtree(s) rooted at `nodes` (level l), outputs into nodes' c.
  // kid_c: if given, the outputs of the level-(l+1) nodes (persistent blocks of the caller);
  // k3_stop: W-combination levels below it are left to the caller.  Returns the level-(l+1)
  // nodes.
  std::vector<Node> breadth_first(int l, const std::vector<Node>& nodes,
                                  const std::vector<Op>* kid_c = nullptr, int k3_stop = -1) {
    std::vector<std::vector<Node>> lv{nodes};
    int64_t npar = (int64_t)nodes.size();  // parents of the leaves (R uniform per level)
    for (int d = l; d < p->L - 1; ++d) npar *= p->rules[p->node_rule[d][0]].R;
    const bool fuse = fuse_leaves(npar);
    // two levels per K1 pass (K1X2), paired from the bottom: (L-2, L-1), (L-4, L-3), ...
    std::vector<bool> pair_at(p->L + 1, false);
    for (int e = p->L - 2; e >= l; e -= 2) pair_at[e] = !(e == 0 && p->virt_scale);  // scaled root: one level
    for (int d = l; d < p->L;) {
      const int pr = pair_at[d] && p->k1_two_level ? k1x2_pair(d, lv.back()) : 0;
      if (pr) {
        auto kg = emit_k1x2(d, lv.back(), pr, !(d + 2 == p->L && fuse),
                            d + 2 == p->L && !fuse && presplit_ok());
        lv.push_back(kg.first);
        lv.push_back(kg.second);
        d += 2;
      } else {
        const bool last = d == p->L - 1;
        lv.push_back(emit_k1(d, lv.back(), -1, !(last && fuse)));
        d += 1;
      }
      if (kid_c && lv.size() == (pr ? 3u : 2u))  // the first pass created level l + 1
        for (size_t i = 0; i < lv[1].size(); ++i) lv[1][i].c = (*kid_c)[i];
    }
    int top = p->L - 1;
    if (fuse) {
      emit_k2f(p->L - 1, lv[p->L - 1 - l], lv.back(), -1, nullptr);
      --top;
    } else {
      emit_k2(lv.back());
    }
    emit_k3_levels(l, top, lv, k3_stop);
    return lv[1];
  }

  void build() {
    Node root{0, Op{BASE_A, 0, 0, 0, -1}, Op{BASE_B, 0, 0, 0, -1}, Op{BASE_C, 0, 0, 0, -1}};
    if (p->L == 0) {
      if (p->rank == 0) {
        emit_k2({root});
      } else {  // nothing owned: zero C
        std::vector<ZeroNode> z{ZeroNode{root.c, 1u, 0}};
        Step st{};
        st.kind = STEP_ZERO; st.count = 1; st.dev_off = push(z);
        st.rows = p->lm[0]; st.cols = p->ln[0]; st.P = 1; st.Q = 1; st.R = 1;
        p->steps.push_back(st);
      }
      return;
    }
    // breadth-first workspace estimate
    int64_t bf = 0, nodes = 1;
    for (int l = 0; l < p->L; ++l) {
      nodes *= p->rules[p->node_rule[l][0]].R;
      bf += nodes * (p->lm[l + 1] * p->lk[l + 1] + p->lk[l + 1] * p->ln[l + 1] +
                     p->lm[l + 1] * p->ln[l + 1]);
    }
    const int64_t bf_bytes = bf * elem_size(p->dtype);
    const bool split = p->schedule >= 2 || p->nranks > 1 || p2p_mode() ||
                       (p->schedule == 0 && bf_bytes > (int64_t)24 << 30);
    if (!split) {
      breadth_first(0, {root});
      try_single_launch();
      return;
    }
    if ((p->schedule == 3 || (p->schedule == 0 && hybrid_on())) && p->nranks == 1 && !p2p_mode() &&
        p->L >= 2) {
      const size_t s0 = p->steps.size(), d0 = desc.size();
      hybrid(root);
      if (ws_peak * elem_size(p->dtype) <= kHybridMaxWs) return;
      p->steps.resize(s0);  // too much workspace: per-r depth-first instead
      desc.resize(d0);
      ws_elems = ws_peak = 0;
    }
    depth_first(0, root, 0);
  }

  bool p2p_mode() const { return p->p2p_active(); }

  // A two-level plan compiled to K1X2 -> K2 -> K3X2 whose leaf phase is at most a few waves of
  // 32 x 64 tiles (C1: 784 tiles) runs as one cooperative kernel (kernels_small.cu): the three
  // launches are launch-bound at this size.  Bitwise the three-launch schedule.
  void try_single_launch() {
    if (!p->single_launch || p->dtype != FMM_F64 || p->L != 2 || p->padded ||
        p->scaling.mode != FMM_SCALE_NONE || p->nranks != 1 || p->steps.size() != 3)
      return;
    const Step s1 = p->steps[0], s2 = p->steps[1], s3 = p->steps[2];
    if (s1.kind != STEP_K1 || !s1.x2 || s1.count > 2 || s2.kind != STEP_K2 || s3.kind != STEP_K3 ||
        s3.x2 != s1.x2)
      return;
    const int64_t tiles = ((s2.rows + small_tile_m() - 1) / small_tile_m()) *
                          ((s2.cols + small_tile_n() - 1) / small_tile_n());
    if ((int64_t)s2.count * tiles > 4 * 3 * 148) return;
    Step st{};
    st.kind = STEP_SMALL;
    st.x2 = s1.x2;
    st.dev_off = s1.dev_off; st.count = s1.count;
    st.dev_off2 = s2.dev_off; st.count2 = s2.count;
    st.rows = s2.rows; st.cols = s2.cols; st.inner = s2.inner;
    st.dev_off3 = s3.dev_off; st.count3 = s3.count;
    p->steps.assign(1, st);
  }

  static bool hybrid_on() {
    const char* e = getenv("FMM_HYBRID");
    return !e || atoi(e) != 0;
  }

  // Single-rank plans too large for breadth-first (C5): the root's S_r / T_r for every r in one
  // K1 pass (A and B read once, instead of once per r), then each top-level subtree's levels
  // 1 .. L-1 one after another (their scratch workspace reused across r), then the root's
  // W-combination -- together with level 1's, as one K3X2 pass from the level-2 products, where
  // the rules pair -- at the end, instead of a per-r ACC read-modify-write of C.  The
  // summation order of every C element is unchanged (ascending r at each level): bitwise the
  // per-r depth-first schedule.  No top-level groups: fmm_execute_host uses the depth-first twin.
  void hybrid(const Node& root) {
    const RuleData& ru = rule_at(0, 0);
    // K3X2 (0, 1) reads the level-2 outputs, so level 1 must not be the leaf parents' level
    // (whose W-combination the leaf kernel may fuse into the level-1 outputs): L >= 3.  Only
    // when the leaf parents' combination is fused into the leaf kernel: otherwise each subtree
    // ends with a K3 pass anyway, and making it the two-level K3X2 (1, 2) into the level-1
    // output, with a one-level K3 at the root, moves fewer bytes (C5 FP32: -11 GB per step) and
    // keeps R instead of R^2 outputs -- the same sums in the same order, bitwise.
    int64_t npar = 1;  // leaf parents per subtree
    for (int d = 1; d < p->L - 1; ++d) npar *= p->rules[p->node_rule[d][0]].R;
    const int pair = p->k3_two_level && p->L >= 3 && fuse_leaves(npar) ? k1x2_pair(0, {root}) : 0;
    std::vector<Node> kids = emit_k1(0, {root}, -1, /*alloc_c=*/pair == 0);
    std::vector<Op> c2;  // persistent level-2 outputs (pair): the K3X2 inputs
    int R2 = 0;
    if (pair) {
      R2 = builtin_R((pair - 1) % 3);
      for (int q = 0; q < ru.R * R2; ++q) c2.push_back(ws_op(ws_alloc(p->lm[2] * p->ln[2]), p->ln[2]));
    }
    const int64_t mark = ws_elems;
    std::vector<Node> level2;
    for (int r = 0; r < ru.R; ++r) {
      ws_elems = mark;  // subtrees run one after another on one stream
      if (pair) {
        std::vector<Op> kc(c2.begin() + (size_t)r * R2, c2.begin() + (size_t)(r + 1) * R2);
        std::vector<Node> l2 = breadth_first(1, {kids[r]}, &kc, 2);
        level2.insert(level2.end(), l2.begin(), l2.end());
      } else {
        breadth_first(1, {kids[r]});
      }
    }
    if (pair) emit_k3x2(0, {root}, level2, pair);
    else emit_k3(0, {root}, kids);
  }

  // Number of shard units below one node of level l (product of the ranks of levels l ..
  // shard_depth - 1); units are the paths (r_1, ..., r_d) of the first d = shard_depth levels
  // in BFS order, unit u belongs to rank u mod nranks.
  int64_t unit_span(int l) const {
    int64_t s = 1;
    for (int q = l; q < p->shard_depth; ++q) s *= p->rules[p->node_rule[q][0]].R;
    return s;
  }
  bool owns_subtree(int level, int64_t unit_prefix) const {
    if (p->nranks == 1) return true;
    const int64_t span = unit_span(level);  // units below this node
    const int64_t u0 = unit_prefix * span;
    if (p->shard_block) {  // rank p owns units [ceil(p U / P), ceil((p + 1) U / P))
      const int64_t U = unit_span(0), P = p->nranks;
      const int64_t lo = ((int64_t)p->rank * U + P - 1) / P, hi = ((int64_t)(p->rank + 1) * U + P - 1) / P;
      return u0 < hi && u0 + span > lo;
    }
    if (span >= p->nranks) return true;
    for (int64_t u = u0; u < u0 + span; ++u)
      if (u % p->nranks == p->rank) return true;
    return false;
  }

  // Does this rank own every unit below a node of `level` (unit_prefix as in owns_subtree)?
  // Then the subtree runs breadth-first like a unit: one S / T pass for all its products, the
  // leaf parents fused over whole R-product chains (bitwise the unit-by-unit schedule).
  bool owns_all(int level, int64_t unit_prefix) const {
    if (p->nranks == 1) return true;
    const int64_t span = unit_span(level);
    if (span == 1) return owns_subtree(level, unit_prefix);
    if (!p->shard_block) return false;  // round-robin spreads every subtree over the ranks
    const int64_t U = unit_span(0), P = p->nranks, u0 = unit_prefix * span;
    const int64_t lo = ((int64_t)p->rank * U + P - 1) / P, hi = ((int64_t)(p->rank + 1) * U + P - 1) / P;
    return u0 >= lo && u0 + span <= hi;
  }

  // Depth-first over the products r of `node` (level l), accumulating C_k (+)= w_kr M_r into
  // node.c in ascending r; recursion continues depth-first down to the shard depth, then each
  // owned subtree runs breadth-first.  Children's workspace is reused across r (one stream).
  void depth_first(int l, const Node& node, int64_t unit_prefix) {
    const RuleData& ru = rule_at(l, node.idx);
    uint32_t started = 0;
    const int64_t mark = ws_elems;
    const bool leaf_next = l + 1 == p->L;
    for (int r = 0; r < ru.R; ++r) {
      const int64_t unit = unit_prefix * ru.R + r;
      if (!owns_subtree(l + 1, unit)) continue;
      ws_elems = mark;  // subtrees run one after another on one stream: reuse the workspace
      const size_t g0 = p->steps.size();
      // comm mode 3: the top-level product M_r goes to this rank's symmetric buffer (slot
      // r / nranks) for the fused NVLink combine; no ACC into a partial C
      const bool p2p = l == 0 && p2p_mode();
      const bool fuse1 = leaf_next && !p2p && fuse_leaves(1);
      std::vector<Node> kid = emit_k1(l, {node}, r, !fuse1 && !p2p);
      if (p2p) {
        kid[0].c = Op{BASE_SYM, 0, (int64_t)(r / p->nranks) * p->lm[1], 0, p->ln[1]};
        if (leaf_next) emit_k2(kid);
        else breadth_first(1, kid);
      } else if (fuse1) {
        emit_k2f(l, {node}, kid, r, &started);
      } else {
        if (leaf_next) emit_k2(kid);
        else if (l + 1 < p->shard_depth && p->nranks > 1 && !owns_all(l + 1, unit))
          depth_first(l + 1, kid[0], unit);
        else breadth_first(l + 1, kid);
        AccNode a{};
        a.out = node.c;
        a.in = kid[0].c;
        a.coef_off = p->coef_W[p->node_rule[l][node.idx]];
        a.r = r;
        for (int k = 0; k < ru.m0 * ru.n0; ++k)
          if (ru.W[(size_t)k * ru.R + r] != 0 && !((started >> k) & 1u)) {
            a.first_mask |= 1u << k;
            started |= 1u << k;
          }
        Step st{};
        st.kind = STEP_ACC; st.count = 1; st.dev_off = push(std::vector<AccNode>{a});
        st.rows = p->lm[l + 1]; st.cols = p->ln[l + 1]; st.P = ru.m0; st.Q = ru.n0; st.R = ru.R;
        p->steps.push_back(st);
      }
      if (l == 0) p->groups.push_back({r, g0, p->steps.size()});
    }
    const uint32_t all = (ru.m0 * ru.n0 >= 32) ? 0xffffffffu : ((1u << (ru.m0 * ru.n0)) - 1u);
    if ((started & all) != all && !(l == 0 && p2p_mode())) {
      std::vector<ZeroNode> z{ZeroNode{node.c, all & ~started, 0}};
      Step st{};
      st.kind = STEP_ZERO; st.count = 1; st.dev_off = push(z);
      st.rows = p->lm[l + 1]; st.cols = p->ln[l + 1]; st.P = ru.m0; st.Q = ru.n0; st.R = ru.R;
      p->steps.push_back(st);
    }
  }
};

void scaling_steps(const fmm_scaling& sc, std::string* steps, double* tau);

fmm_status compile_plan(fmm_plan* p) {
  {
    std::lock_guard<std::mutex> g(p->gmu);
    for (auto& ge : p->graphs) cudaGraphExecDestroy(ge.exec);
    p->graphs.clear();
  }
  p->steps.clear();
  p->groups.clear();
  {
    std::lock_guard<std::mutex> g(p->dev_mu);
    if (p->dev_desc) { cudaFree(p->dev_desc); p->dev_desc = nullptr; }
    p->dev_id = -1;
    delete p->df_twin;  // the twin copies the plan's settings: rebuilt on next use
    p->df_twin = nullptr;
  }
  // virtual scaling needs the root to be a K1 pass over the caller's A, B: FP64 power-of-two
  // factors, no zero padding, at least one recursion level
  p->virt_scale = p->scaling.mode != FMM_SCALE_NONE && p->scaling.pow2 && !p->padded &&
                  p->dtype == FMM_F64 && p->L >= 1 && p->virt_scale_enable;
  Builder b(p);
  b.build();
  p->fmm_ws_bytes = (size_t)b.ws_peak * elem_size(p->dtype);
  p->pad_bytes = 0;
  if (p->padded) {
    auto al = [](size_t x) { return (x + 255) / 256 * 256; };
    const size_t es = (size_t)elem_size(p->dtype);
    p->pad_bytes = al((size_t)p->Mp * p->Kp * es) + al((size_t)p->Kp * p->Np * es) +
                   al((size_t)p->Mp * p->Np * es);
  }
  p->desc_bytes = b.desc.size();
  p->launches = (int64_t)p->steps.size();
  p->unscale_fused = false;
  for (const Step& st : p->steps) p->unscale_fused = p->unscale_fused || st.unscale;
  if (p->scaling.mode != FMM_SCALE_NONE) {
    const size_t vec = (size_t)(p->M + p->N + p->K) * 8;
    const size_t mats = ((size_t)p->M * p->K + (size_t)p->K * p->N) * 8;
    p->scale_bytes = (mats + vec + scale_ws_bytes(p->M, p->K, p->N) + 4096 + 255) / 256 * 256;
    std::string stp;
    double tau;
    scaling_steps(p->scaling, &stp, &tau);
    p->launches += 1 + (p->unscale_fused ? 0 : 1);  // the one-kernel scaling run (+ unscale)
  } else {
    p->scale_bytes = 0;
  }
  if (p->comm && !p->p2p_active()) p->launches += 1;
  if (p->padded) p->launches += 3;  // pad A, pad B, crop C
  // vector-path feasibility of all plan-internal dims (caller lds / pointers checked at run)
  const int vec = 16 / elem_size(p->dtype);
  p->dims_vec_ok = true;
  for (int l = 0; l <= p->L; ++l)
    if (p->lk[l] % vec || p->ln[l] % vec) p->dims_vec_ok = false;
  p->desc_host = std::move(b.desc);
  return FMM_OK;
}

bool check_rule_dims(const RuleData& d) {
  return d.m0 > 0 && d.k0 > 0 && d.n0 > 0 && d.R > 0 && d.m0 * d.k0 <= kMaxBlk &&
         d.k0 * d.n0 <= kMaxBlk && d.m0 * d.n0 <= kMaxBlk && d.R <= kMaxR;
}

}  // namespace

// ---------------------------------------------------------------------------------------------
namespace {
static bool aligned16(const void* q) { return ((uintptr_t)q & 15u) == 0; }

// Upload coefficient tables and descriptors to the current device (once per plan / device).
static fmm_status ensure_device(const fmm_plan* p) {
  std::lock_guard<std::mutex> g(p->dev_mu);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice");
  if (p->dev_id == dev && (p->dev_coef || p->coef_host.empty()) && (p->dev_desc || p->desc_host.empty()))
    return FMM_OK;
  if (p->dev_id != -1 && p->dev_id != dev) {  // captured graphs hold the old tables' pointers
    std::lock_guard<std::mutex> gg(p->gmu);
    for (auto& ge : p->graphs) cudaGraphExecDestroy(ge.exec);
    p->graphs.clear();
  }
  if (p->dev_coef) { cudaFree(p->dev_coef); p->dev_coef = nullptr; }
  if (p->dev_desc) { cudaFree(p->dev_desc); p->dev_desc = nullptr; }
  if (!p->coef_host.empty()) {
    e = cudaMalloc((void**)&p->dev_coef, p->coef_host.size() * sizeof(double));
    if (e == cudaSuccess)
      e = cudaMemcpy(p->dev_coef, p->coef_host.data(), p->coef_host.size() * sizeof(double), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_status(e, "plan coefficient upload");
  }
  if (!p->desc_host.empty()) {
    e = cudaMalloc(&p->dev_desc, p->desc_host.size());
    if (e == cudaSuccess)
      e = cudaMemcpy(p->dev_desc, p->desc_host.data(), p->desc_host.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_status(e, "plan descriptor upload");
  }
  p->dev_id = dev;
  return FMM_OK;
}

static cudaEvent_t ev_get(const fmm_plan* p) {
  if (!p->ev_pool.empty()) {
    cudaEvent_t e = p->ev_pool.back();
    p->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// Record a timing bracket around a launch of kind `kind` (no-op unless timing is enabled).
struct TimedLaunch {
  const fmm_plan* p;
  int kind;
  cudaStream_t st;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  TimedLaunch(const fmm_plan* pl, int k, cudaStream_t s) : p(pl), kind(k), st(s) {
    if (!p->timing) return;
    std::lock_guard<std::mutex> g(p->tmu);
    e0 = ev_get(p);
    e1 = ev_get(p);
    cudaEventRecord(e0, st);
  }
  ~TimedLaunch() {
    if (!e0) return;
    cudaEventRecord(e1, st);
    std::lock_guard<std::mutex> g(p->tmu);
    p->ev_used.push_back({kind, {e0, e1}});
  }
};

// Launch one step (or one node-chunk of it: grid.y / grid.z carry the node count, limited to
// 65535, so steps with more nodes -- deep recursions, 7^6 = 117649 leaves -- run in chunks).
// `c0` = first node of the chunk: descriptor arrays, the FP32 split list and the turnstiles
// are offset accordingly; the FP32 hi / lo arena is reused by consecutive chunks.
template <typename T>
static cudaError_t launch_step(const fmm_plan* p, const Step& s, int64_t c0, const Bases& b,
                               bool vec, cudaStream_t st, const ScaleIn* sc) {
  size_t node_bytes = 0;
  switch (s.kind) {
    case STEP_K1: node_bytes = s.x2 ? sizeof(K1x2Node) : sizeof(K1Node); break;
    case STEP_K3: node_bytes = s.x2 ? sizeof(K3x2Node) : sizeof(K3Node); break;
    case STEP_ACC: node_bytes = sizeof(AccNode); break;
    case STEP_ZERO: node_bytes = sizeof(ZeroNode); break;
    case STEP_K2: node_bytes = sizeof(LeafNode); break;
    case STEP_K2F: node_bytes = sizeof(FusedNode); break;
    case STEP_SMALL: node_bytes = sizeof(K1x2Node); break;
  }
  const void* nd = (const uint8_t*)p->dev_desc + s.dev_off + c0 * node_bytes;
  const int ts = k2f_tile_of(s.k2f_cfg);
  const int64_t tiles_f = ((s.rows + ts - 1) / ts) * ((s.cols + ts - 1) / ts);
  switch (s.kind) {
    case STEP_SMALL: {
      const uint8_t* d = (const uint8_t*)p->dev_desc;
      return launch_small_plan(s.x2, (const K1x2Node*)(d + s.dev_off), s.count,
                               (const LeafNode*)(d + s.dev_off2), s.count2, s.rows, s.cols, s.inner,
                               (const K3x2Node*)(d + s.dev_off3), s.count3, b, vec, st);
    }
    case STEP_K1: return launch_k1<T>(s, nd, p->dev_coef, b, vec, st, sc);
    case STEP_K3: return launch_k3<T>(s, nd, p->dev_coef, b, vec, st, sc);
    case STEP_ACC: return launch_acc<T>(s, nd, p->dev_coef, b, vec, st);
    case STEP_ZERO: return launch_zero<T>(s, nd, b, st);
    case STEP_K2F:
      return launch_gemm_f64_fused(
          (const FusedNode*)nd, s.count, s.rows, s.cols, s.inner, p->dev_coef, s.P, s.Q, s.R, b, vec,
          st, s.nr, s.split,
          s.turn_off >= 0 ? (int*)((double*)b.p[BASE_WS] + s.turn_off) + c0 * tiles_f : nullptr,
          s.k2f_cfg, s.unitw);
    case STEP_K2:
      if (p->dtype == FMM_F64)
        return launch_gemm_f64((const LeafNode*)nd, s.count, s.rows, s.cols, s.inner, b, vec, st);
      return launch_gemm_f32((const LeafNode*)nd,
                             (const LeafNode*)(p->desc_host.data() + s.dev_off) + c0, s.count,
                             s.rows, s.cols, s.inner, b, vec, p->leaf,
                             s.arena_off >= 0 ? (float*)b.p[BASE_WS] + s.arena_off : nullptr, st,
                             s.tf32_split != 0);
  }
  return cudaSuccess;
}

// Host-side NVTX range (enqueue span of a launch / phase) for profiler timelines.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

static const char* step_name(const Step& s) {
  switch (s.kind) {
    case STEP_K1: return s.x2 ? "fmm.K1X2" : "fmm.K1";
    case STEP_K2: return "fmm.K2";
    case STEP_K3: return s.x2 ? "fmm.K3X2" : "fmm.K3";
    case STEP_ACC: return "fmm.ACC";
    case STEP_ZERO: return "fmm.ZERO";
    case STEP_K2F: return "fmm.K2F";
    case STEP_SMALL: return "fmm.SMALL";
  }
  return "fmm.step";
}

template <typename T>
static fmm_status run_steps(const fmm_plan* p, const Bases& b, bool vec, cudaStream_t st,
                            size_t i0 = 0, size_t i1 = (size_t)-1, const ScaleIn* sc = nullptr) {
  constexpr int64_t kMaxNodes = 32768;  // per launch (grid.y / grid.z <= 65535)
  if (i1 > p->steps.size()) i1 = p->steps.size();
  for (size_t si = i0; si < i1; ++si) {
    const Step& s = p->steps[si];
    NvtxRange nv(step_name(s));
    TimedLaunch tl(p, (s.kind == STEP_K2F || s.kind == STEP_SMALL) ? STEP_K2 : s.kind, st);
    cudaError_t e = cudaSuccess;
    int64_t maxn = kMaxNodes;
    if (s.kind == STEP_K2F && s.chunk > 0 && s.nr > s.chunk)  // grid.y = groups x nodes
      maxn = std::min<int64_t>(maxn, 65535 / ((s.nr + s.chunk - 1) / s.chunk));
    if (s.kind == STEP_K2F && s.split)
      maxn = std::min<int64_t>(maxn, 65535 / std::max(1, split_groups(s.split, s.nr)));
    for (int64_t c0 = 0; c0 < s.count && e == cudaSuccess; c0 += maxn) {
      Step sub = s;
      sub.count = (int)std::min<int64_t>(maxn, s.count - c0);
      e = launch_step<T>(p, sub, c0, b, vec, st, sc);
    }
    if (e != cudaSuccess) return cuda_status(e, "fmm_execute launch");
  }
  return FMM_OK;
}

void scaling_steps(const fmm_scaling& sc, std::string* steps, double* tau) {
  switch (sc.mode) {
    case FMM_SCALE_OUTSIDE: *steps = "O"; *tau = -1; break;
    case FMM_SCALE_INSIDE: *steps = "I"; *tau = -1; break;
    case FMM_SCALE_OUT_IN: *steps = "OI"; *tau = -1; break;
    case FMM_SCALE_IN_OUT: *steps = "IO"; *tau = -1; break;
    case FMM_SCALE_REPEATED: {
      steps->clear();
      for (int t = 0; t < sc.max_steps; ++t)
        steps->push_back(((t % 2 == 0) == (sc.first_step_is_O != 0)) ? 'O' : 'I');
      *tau = sc.tau;
      break;
    }
    default: steps->clear(); *tau = 0;
  }
}


static fmm_status scale_common(int64_t M, int64_t K, int64_t N, const void* A, int64_t lda,
                               const void* B, int64_t ldb, void* A_out, int64_t lda_out,
                               void* B_out, int64_t ldb_out, void* dA, void* dB, void* dI,
                               const std::string& steps, double tau, int pow2,
                               int32_t* steps_dev, void* ws, cudaStream_t st, bool sync_check) {
  if (!A || !B || !A_out || !B_out || M <= 0 || K <= 0 || N <= 0 || lda < K || ldb < N ||
      lda_out < K || ldb_out < N) {
    set_error("fmm_scale: bad argument");
    return FMM_E_ARG;
  }
  void* own = nullptr;
  cudaError_t e = cudaSuccess;
  double *tdA = (double*)dA, *tdB = (double*)dB, *tdI = (double*)dI;
  // layout: [scale workspace | 256 B | factor vectors the caller omitted]
  size_t need = scale_ws_bytes(M, K, N) + 256 + (size_t)(M + N + K) * 8 + 1024;
  if (!ws) {
    e = cudaMallocAsync(&own, need, st);
    if (e != cudaSuccess) return cuda_status(e, "fmm_scale alloc");
  }
  uint8_t* w = (uint8_t*)(ws ? ws : own);
  w = (uint8_t*)(((uintptr_t)w + 255) & ~(uintptr_t)255);
  uint8_t* extra = w + (scale_ws_bytes(M, K, N) + 255) / 256 * 256 + 256;
  if (!tdA) { tdA = (double*)extra; }
  if (!tdB) { tdB = (double*)extra + M; }
  if (!tdI) { tdI = (double*)extra + M + N; }
  e = run_scaling_coop(M, K, N, (const double*)A, lda, (const double*)B, ldb, (double*)A_out, lda_out,
                       (double*)B_out, ldb_out, tdA, tdB, tdI, (int)steps.size(), steps[0] == 'O', tau,
                       pow2, /*materialise_end=*/1, w, st);
  int* flags = scale_flags_ptr(w, M, K, N);
  if (e == cudaSuccess && steps_dev)
    e = cudaMemcpyAsync(steps_dev, flags + 1, sizeof(int32_t), cudaMemcpyDeviceToDevice, st);
  fmm_status status = FMM_OK;
  if (e == cudaSuccess && sync_check) {
    int hf[8];
    e = cudaMemcpyAsync(hf, flags, sizeof hf, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e == cudaSuccess && hf[2]) {
      static const char* what[] = {"", "row of A", "column of B", "column of A", "row of B"};
      set_error(std::string("scaling precondition: all-zero ") + what[hf[2] & 7] + " at index " + std::to_string(hf[3]));
      status = FMM_E_PRECOND;
    }
  }
  if (own) cudaFreeAsync(own, st);
  if (e != cudaSuccess) return cuda_status(e, "fmm_scale");
  return status;
}

}  // namespace

extern "C" {

const char* fmm_last_error(void) { return g_err.c_str(); }
const char* fmm_version(void) { return "fmm_b200 0.1 (sm_100a)"; }

fmm_status fmm_rule_create(int m0, int k0, int n0, int R, const int32_t* U, const int32_t* V,
                           const int32_t* W, int log2_den, const char* name, fmm_rule** out,
                           int64_t* n_violations) {
  if (!U || !V || !W || !out) { set_error("fmm_rule_create: null pointer"); return FMM_E_ARG; }
  if (log2_den < 0 || log2_den > 8) { set_error("fmm_rule_create: log2_den out of [0, 8]"); return FMM_E_ARG; }
  RuleData d;
  d.name = name ? name : "custom";
  d.m0 = m0; d.k0 = k0; d.n0 = n0; d.R = R; d.log2den = log2_den;
  if (!check_rule_dims(d)) { set_error("fmm_rule_create: dims out of range (m0k0,k0n0,m0n0 <= 16, R <= 32)"); return FMM_E_ARG; }
  d.U.assign(U, U + (size_t)m0 * k0 * R);
  d.V.assign(V, V + (size_t)k0 * n0 * R);
  d.W.assign(W, W + (size_t)m0 * n0 * R);
  for (auto* X : {&d.U, &d.V, &d.W})
    for (int32_t x : *X)
      if (x <= -(1 << 20) || x >= (1 << 20)) { set_error("fmm_rule_create: |numerator| >= 2^20"); return FMM_E_ARG; }
  int64_t fi = -1, fj = -1, fk = -1;
  int64_t nv = brent_violations(d, &fi, &fj, &fk);
  if (n_violations) *n_violations = nv;
  if (nv) {
    char buf[200];
    snprintf(buf, sizeof buf, "fmm_rule_create: %lld Brent violations; first at (i=%lld, j=%lld, k=%lld)",
             (long long)nv, (long long)fi, (long long)fj, (long long)fk);
    set_error(buf);
    return FMM_E_RULE;
  }
  *out = new fmm_rule{d};
  return FMM_OK;
}

fmm_status fmm_rule_builtin(const char* name, fmm_rule** out) {
  if (!name || !out) { set_error("fmm_rule_builtin: null pointer"); return FMM_E_ARG; }
  RuleData d;
  if (!builtin_rule(name, &d)) { set_error(std::string("unknown builtin rule: ") + name); return FMM_E_ARG; }
  if (brent_violations(d, nullptr, nullptr, nullptr) != 0) { set_error("builtin rule fails Brent"); return FMM_E_RULE; }
  *out = new fmm_rule{d};
  return FMM_OK;
}

fmm_status fmm_rule_info(const fmm_rule* r, int* m0, int* k0, int* n0, int* R, int32_t* U,
                         int32_t* V, int32_t* W, int* log2_den) {
  if (!r) { set_error("fmm_rule_info: null rule"); return FMM_E_ARG; }
  if (m0) *m0 = r->d.m0;
  if (k0) *k0 = r->d.k0;
  if (n0) *n0 = r->d.n0;
  if (R) *R = r->d.R;
  if (log2_den) *log2_den = r->d.log2den;
  if (U) std::copy(r->d.U.begin(), r->d.U.end(), U);
  if (V) std::copy(r->d.V.begin(), r->d.V.end(), V);
  if (W) std::copy(r->d.W.begin(), r->d.W.end(), W);
  return FMM_OK;
}

void fmm_rule_destroy(fmm_rule* r) { delete r; }

fmm_status fmm_rule_transform(const fmm_rule* r, int kind, fmm_rule** out) {
  if (!r || !out) { set_error("fmm_rule_transform: null"); return FMM_E_ARG; }
  RuleData d;
  if (!transform_rule(r->d, kind, &d)) { set_error("fmm_rule_transform: kind must be 1, 2 or 3"); return FMM_E_ARG; }
  if (!check_rule_dims(d)) { set_error("fmm_rule_transform: result dims out of range"); return FMM_E_ARG; }
  int64_t fi = -1, fj = -1, fk = -1;
  if (brent_violations(d, &fi, &fj, &fk) != 0) {
    set_error("fmm_rule_transform: result violates the Brent equations");
    return FMM_E_RULE;
  }
  *out = new fmm_rule{d};
  return FMM_OK;
}

fmm_status fmm_plan_create(const fmm_rule* const* nodes, int n_nodes, int levels, int uniform,
                           int64_t M, int64_t K, int64_t N, int dtype, int leaf,
                           const fmm_scaling* scaling, fmm_plan** out) {
  if (!out || levels < 0 || levels > 16 || M < 0 || K < 0 || N < 0 || (levels > 0 && !nodes)) {
    set_error("fmm_plan_create: bad argument");
    return FMM_E_ARG;
  }
  if (dtype != FMM_F64 && dtype != FMM_F32) { set_error("fmm_plan_create: bad dtype"); return FMM_E_ARG; }
  if (leaf < FMM_LEAF_NATIVE || leaf > FMM_LEAF_3XTF32 || (dtype == FMM_F64 && leaf != FMM_LEAF_NATIVE)) {
    set_error("fmm_plan_create: leaf kind not valid for dtype (FP64 requires NATIVE)");
    return FMM_E_ARG;
  }
  auto p = new fmm_plan();
  p->dtype = dtype; p->leaf = leaf; p->L = levels; p->M = M; p->K = K; p->N = N;
  if (const char* ce = getenv("FMM_SPLIT")) p->split_chains = atoi(ce) != 0;
  if (const char* xe = getenv("FMM_K1X2")) p->k1_two_level = atoi(xe) != 0;
  if (const char* xe = getenv("FMM_TF32_PRESPLIT")) p->tf32_presplit = atoi(xe) != 0;
  if (const char* xe = getenv("FMM_K3X2")) p->k3_two_level = atoi(xe) != 0;
  if (const char* fe = getenv("FMM_FUSION")) {
    const int f = atoi(fe);
    if (f >= 0 && f <= 2) p->fusion = f;
  }
  if (scaling) {
    if (scaling->mode < FMM_SCALE_NONE || scaling->mode > FMM_SCALE_REPEATED ||
        (scaling->mode == FMM_SCALE_REPEATED && scaling->max_steps < 1)) {
      delete p; set_error("fmm_plan_create: bad scaling config"); return FMM_E_ARG;
    }
    if (scaling->mode != FMM_SCALE_NONE && dtype != FMM_F64) {
      delete p; set_error("fmm_plan_create: scaling is implemented for FP64"); return FMM_E_UNSUPPORTED;
    }
    p->scaling = *scaling;
  }
  // expected node counts
  int64_t count = 1, total = 0;
  std::vector<int64_t> per_level;
  auto find_rule = [&](const fmm_rule* r) {
    for (size_t i = 0; i < p->rules.size(); ++i)
      if (p->rules[i].name == r->d.name && p->rules[i].U == r->d.U && p->rules[i].V == r->d.V &&
          p->rules[i].W == r->d.W && p->rules[i].log2den == r->d.log2den)
        return (int)i;
    p->rules.push_back(r->d);
    return (int)p->rules.size() - 1;
  };
  int64_t idx = 0;
  for (int l = 0; l < levels; ++l) {
    std::vector<int> nr;
    if (uniform) {
      if (l >= n_nodes || !nodes[l]) { delete p; set_error("fmm_plan_create: uniform needs one rule per level"); return FMM_E_ARG; }
      nr.assign((size_t)count, find_rule(nodes[l]));
    } else {
      if (idx + count > n_nodes) { delete p; set_error("fmm_plan_create: too few nodes for a non-uniform tree"); return FMM_E_ARG; }
      for (int64_t q = 0; q < count; ++q) {
        if (!nodes[idx + q]) { delete p; set_error("fmm_plan_create: null node rule"); return FMM_E_ARG; }
        nr.push_back(find_rule(nodes[idx + q]));
      }
      idx += count;
    }
    const RuleData& r0 = p->rules[nr[0]];
    for (int q : nr) {
      const RuleData& rq = p->rules[q];
      if (rq.m0 != r0.m0 || rq.k0 != r0.k0 || rq.n0 != r0.n0 || rq.R != r0.R) {
        delete p; set_error("fmm_plan_create: rules within a level must share (m0,k0,n0,R) (P:146)"); return FMM_E_ARG;
      }
    }
    p->node_rule.push_back(nr);
    total += count;
    count *= r0.R;
    if (count > (1 << 22)) { delete p; set_error("fmm_plan_create: recursion tree too large"); return FMM_E_ARG; }
  }
  if (!uniform && idx != n_nodes && levels > 0) { delete p; set_error("fmm_plan_create: node count mismatch"); return FMM_E_ARG; }
  (void)total;
  // pad_dims: smallest multiples of prod m0, prod k0, prod n0
  int64_t pm = 1, pk = 1, pn = 1;
  for (int l = 0; l < levels; ++l) {
    const RuleData& r = p->rules[p->node_rule[l][0]];
    pm *= r.m0; pk *= r.k0; pn *= r.n0;
  }
  p->Mp = (M + pm - 1) / pm * pm;
  p->Kp = (K + pk - 1) / pk * pk;
  p->Np = (N + pn - 1) / pn * pn;
  p->padded = p->Mp != M || p->Kp != K || p->Np != N;
  p->lm.push_back(p->Mp); p->lk.push_back(p->Kp); p->ln.push_back(p->Np);
  for (int l = 0; l < levels; ++l) {
    const RuleData& r = p->rules[p->node_rule[l][0]];
    p->lm.push_back(p->lm[l] / r.m0); p->lk.push_back(p->lk[l] / r.k0); p->ln.push_back(p->ln[l] / r.n0);
  }
  // coefficient tables
  for (const RuleData& r : p->rules) {
    p->coef_U.push_back((int)p->coef_host.size());
    for (int i = 0; i < r.m0 * r.k0; ++i) for (int q = 0; q < r.R; ++q) p->coef_host.push_back(r.coef(r.U, i, q));
    p->coef_V.push_back((int)p->coef_host.size());
    for (int j = 0; j < r.k0 * r.n0; ++j) for (int q = 0; q < r.R; ++q) p->coef_host.push_back(r.coef(r.V, j, q));
    p->coef_W.push_back((int)p->coef_host.size());
    for (int k = 0; k < r.m0 * r.n0; ++k) for (int q = 0; q < r.R; ++q) p->coef_host.push_back(r.coef(r.W, k, q));
  }
  fmm_status s = compile_plan(p);
  if (s != FMM_OK) { delete p; return s; }
  *out = p;
  return FMM_OK;
}

void fmm_plan_destroy(fmm_plan* p) { delete p; }

fmm_status fmm_plan_set_partition(fmm_plan* p, int rank, int nranks) {
  if (!p || nranks < 1 || rank < 0 || rank >= nranks) { set_error("fmm_plan_set_partition: bad rank/nranks"); return FMM_E_ARG; }
  p->rank = rank;
  p->nranks = nranks;
  return compile_plan(p);
}

fmm_status fmm_plan_set_schedule(fmm_plan* p, int schedule) {
  if (!p || schedule < 0 || schedule > 3) { set_error("fmm_plan_set_schedule: bad args"); return FMM_E_ARG; }
  p->schedule = schedule;
  return compile_plan(p);
}

fmm_status fmm_plan_set_fusion(fmm_plan* p, int mode) {
  if (!p || mode < 0 || mode > 2) { set_error("fmm_plan_set_fusion: mode must be 0, 1 or 2"); return FMM_E_ARG; }
  p->fusion = mode;
  return compile_plan(p);
}

fmm_status fmm_plan_set_k1_levels(fmm_plan* p, int levels) {
  if (!p || levels < 1 || levels > 2) { set_error("fmm_plan_set_k1_levels: levels must be 1 or 2"); return FMM_E_ARG; }
  p->k1_two_level = levels == 2;
  return compile_plan(p);
}

fmm_status fmm_plan_set_leaf_split(fmm_plan* p, int in_pass) {
  if (!p || in_pass < 0 || in_pass > 1) { set_error("fmm_plan_set_leaf_split: mode must be 0 or 1"); return FMM_E_ARG; }
  p->tf32_presplit = in_pass == 1;
  return compile_plan(p);
}

fmm_status fmm_plan_set_k3_levels(fmm_plan* p, int levels) {
  if (!p || levels < 1 || levels > 2) { set_error("fmm_plan_set_k3_levels: levels must be 1 or 2"); return FMM_E_ARG; }
  p->k3_two_level = levels == 2;
  return compile_plan(p);
}

fmm_status fmm_plan_fused_launches(const fmm_plan* p, int64_t* n) {
  if (!p || !n) { set_error("fmm_plan_fused_launches: null"); return FMM_E_ARG; }
  *n = 0;
  for (const Step& s : p->steps) *n += s.kind == STEP_K2F;
  return FMM_OK;
}

fmm_status fmm_plan_set_comm_mode(fmm_plan* p, int mode) {
  if (!p || mode < 0 || mode > 3) { set_error("fmm_plan_set_comm_mode: mode must be 0, 1, 2 or 3"); return FMM_E_ARG; }
  if (mode == 3 && p->shard_block) {
    set_error("fmm_plan_set_comm_mode: the fused NVLink combine (mode 3) needs round-robin units");
    return FMM_E_UNSUPPORTED;
  }
  const bool recompile = (mode == 3) != (p->comm_mode == 3);  // mode 3 changes the schedule
  p->comm_mode = mode;
  return recompile ? compile_plan(p) : FMM_OK;
}

static size_t sym_bytes_of(const fmm_plan* p) {
  if (p->L == 0 || p->nranks < 1) return 0;
  const int R = p->rules[p->node_rule[0][0]].R;
  const int64_t slots = (R + p->nranks - 1) / p->nranks;
  return (size_t)slots * p->lm[1] * p->ln[1] * elem_size(p->dtype) + 256;  // + barrier scratch
}

fmm_status fmm_plan_sym_bytes(const fmm_plan* p, size_t* bytes) {
  if (!p || !bytes) { set_error("fmm_plan_sym_bytes: null"); return FMM_E_ARG; }
  *bytes = sym_bytes_of(p);
  return FMM_OK;
}

fmm_status fmm_plan_sym_alloc(fmm_plan* p, void* handle) {
  if (!p || !handle) { set_error("fmm_plan_sym_alloc: null"); return FMM_E_ARG; }
  const size_t need = sym_bytes_of(p);
  if (need == 0) { set_error("fmm_plan_sym_alloc: no top-level products"); return FMM_E_ARG; }
  cudaError_t e = cudaSuccess;
  if (!p->sym_own || p->sym_alloc_bytes < need) {
    if (p->sym_own) cudaFree(p->sym_own);
    p->sym_own = nullptr;
    e = cudaMalloc(&p->sym_own, need);  // its own allocation: the IPC handle maps exactly it
    if (e != cudaSuccess) return cuda_status(e, "fmm_plan_sym_alloc");
    p->sym_alloc_bytes = need;
  }
  cudaIpcMemHandle_t h;
  e = cudaIpcGetMemHandle(&h, p->sym_own);
  if (e != cudaSuccess) return cuda_status(e, "fmm_plan_sym_alloc (IPC handle)");
  std::memcpy(handle, &h, sizeof h);
  return FMM_OK;
}

fmm_status fmm_plan_sym_ptr(const fmm_plan* p, void** ptr) {
  if (!p || !ptr) { set_error("fmm_plan_sym_ptr: null"); return FMM_E_ARG; }
  *ptr = p->sym_own;
  return FMM_OK;
}

static fmm_status upload_peers(const std::vector<void*>& ptrs, void** dev) {
  if (!*dev) {
    cudaError_t e = cudaMalloc(dev, sizeof(void*) * 64);
    if (e != cudaSuccess) return cuda_status(e, "peer table");
  }
  if (ptrs.size() > 64) { set_error("more than 64 ranks"); return FMM_E_ARG; }
  return cuda_status(cudaMemcpy(*dev, ptrs.data(), sizeof(void*) * ptrs.size(), cudaMemcpyHostToDevice),
                     "peer table");
}

fmm_status fmm_plan_set_peer_handles(fmm_plan* p, const void* handles, int n) {
  if (!p || !handles || n != p->nranks || n < 1) { set_error("fmm_plan_set_peer_handles: bad args (n must equal nranks)"); return FMM_E_ARG; }
  if (!p->sym_own) { set_error("fmm_plan_set_peer_handles: call fmm_plan_sym_alloc first"); return FMM_E_ARG; }
  for (size_t q = 0; q < p->peers.size(); ++q)
    if (q < p->peer_opened.size() && p->peer_opened[q] && p->peers[q]) cudaIpcCloseMemHandle(p->peers[q]);
  p->peers.assign(n, nullptr);
  p->peer_opened.assign(n, false);
  for (int q = 0; q < n; ++q) {
    if (q == p->rank) { p->peers[q] = p->sym_own; continue; }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, (const uint8_t*)handles + (size_t)q * sizeof h, sizeof h);
    cudaError_t e = cudaIpcOpenMemHandle(&p->peers[q], h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_status(e, "fmm_plan_set_peer_handles (cudaIpcOpenMemHandle)");
    p->peer_opened[q] = true;
  }
  return upload_peers(p->peers, &p->dev_peers);
}

}  // extern "C"

template <typename T>
static fmm_status p2p_combine(const fmm_plan* p, const void* dev_table, int n, void* C, int64_t ldc,
                              int64_t row0, int64_t row1, cudaStream_t st) {
  const RuleData& ru = p->rules[p->node_rule[0][0]];
  const int vecn = 16 / (int)sizeof(T);
  const bool vec = p->dims_vec_ok && aligned16(C) && ldc % vecn == 0;
  NvtxRange nv("fmm.p2p_combine");
  TimedLaunch tl(p, 7, st);
  return cuda_status(launch_p2p_combine<T>((const T* const*)dev_table, n, p->dev_coef,
                                           p->coef_W[p->node_rule[0][0]], ru.R, ru.m0, ru.n0,
                                           p->lm[1], p->ln[1], (T*)C, ldc, row0, row1, vec, st),
                     "p2p combine");
}

extern "C" {

fmm_status fmm_plan_p2p_combine(fmm_plan* p, const void* const* peer_ptrs, int n, void* C,
                                int64_t ldc, int64_t row0, int64_t row1, void* stream) {
  if (!p || !peer_ptrs || !C || n < 1 || p->L == 0 || ldc < p->N || row0 < 0 || row1 > p->M || row0 > row1) {
    set_error("fmm_plan_p2p_combine: bad args");
    return FMM_E_ARG;
  }
  if (p->padded || p->scaling.mode != FMM_SCALE_NONE) { set_error("fmm_plan_p2p_combine: not for padded or scaled plans"); return FMM_E_ARG; }
  fmm_status fs = ensure_device(p);
  if (fs != FMM_OK) return fs;
  std::vector<void*> v(n);
  for (int q = 0; q < n; ++q) v[q] = const_cast<void*>(peer_ptrs[q]);
  if ((fs = upload_peers(v, &p->dev_tmp_peers)) != FMM_OK) return fs;
  return p->dtype == FMM_F64 ? p2p_combine<double>(p, p->dev_tmp_peers, n, C, ldc, row0, row1, (cudaStream_t)stream)
                             : p2p_combine<float>(p, p->dev_tmp_peers, n, C, ldc, row0, row1, (cudaStream_t)stream);
}

fmm_status fmm_plan_set_shard_depth(fmm_plan* p, int depth) {
  if (!p || depth < 1 || (p->L > 0 && depth > p->L)) { set_error("fmm_plan_set_shard_depth: depth must be in [1, L]"); return FMM_E_ARG; }
  int64_t units = 1;
  for (int l = 0; l < depth && l < p->L; ++l) units *= p->rules[p->node_rule[l][0]].R;
  if (units > (1 << 20)) { set_error("fmm_plan_set_shard_depth: too many units"); return FMM_E_ARG; }
  p->shard_depth = depth;
  return compile_plan(p);
}

fmm_status fmm_plan_set_shard_order(fmm_plan* p, int order) {
  if (!p || order < 0 || order > 1) { set_error("fmm_plan_set_shard_order: order must be 0 or 1"); return FMM_E_ARG; }
  if (order == 1 && p->comm_mode == 3) {
    set_error("fmm_plan_set_shard_order: the fused NVLink combine (comm mode 3) needs round-robin units");
    return FMM_E_UNSUPPORTED;
  }
  p->shard_block = order == 1;
  return compile_plan(p);
}

fmm_status fmm_plan_owned(const fmm_plan* p, int rank, int nranks, int32_t* owned, int* R) {
  if (!p || nranks < 1 || rank < 0 || rank >= nranks) { set_error("fmm_plan_owned: bad args"); return FMM_E_ARG; }
  int64_t units = 1;
  for (int l = 0; l < p->shard_depth && l < p->L; ++l) units *= p->rules[p->node_rule[l][0]].R;
  if (R) *R = (int)units;
  if (owned)
    for (int64_t u = 0; u < units; ++u)
      owned[u] = (p->L > 0 ? (p->shard_block ? (u * nranks / units == rank) : (u % nranks == rank))
                           : (rank == 0)) ? 1 : 0;
  return FMM_OK;
}

fmm_status fmm_plan_workspace_bytes(const fmm_plan* p, size_t* bytes) {
  if (!p || !bytes) { set_error("fmm_plan_workspace_bytes: null"); return FMM_E_ARG; }
  *bytes = p->scale_bytes + p->pad_bytes + p->fmm_ws_bytes + 256;
  return FMM_OK;
}

fmm_status fmm_plan_launch_count(const fmm_plan* p, int64_t* launches) {
  if (!p || !launches) { set_error("fmm_plan_launch_count: null"); return FMM_E_ARG; }
  *launches = p->launches;
  return FMM_OK;
}

static fmm_status execute_impl(const fmm_plan* p, const void* A, int64_t lda, const void* B,
                               int64_t ldb, void* C, int64_t ldc, void* ws, size_t ws_bytes,
                               void* stream);

fmm_status fmm_plan_set_graph(fmm_plan* p, int enable) {
  if (!p) { set_error("fmm_plan_set_graph: null"); return FMM_E_ARG; }
  p->use_graph = enable != 0;
  return FMM_OK;
}

fmm_status fmm_execute(const fmm_plan* p, const void* A, int64_t lda, const void* B, int64_t ldb,
                       void* C, int64_t ldc, void* ws, size_t ws_bytes, void* stream) {
  NvtxRange nv("fmm_execute");
  if (!p || !p->use_graph || p->timing || p->comm || p->barrier_fn)
    return execute_impl(p, A, lda, B, ldb, C, ldc, ws, ws_bytes, stream);
  cudaStream_t st = (cudaStream_t)stream;
  {
    std::lock_guard<std::mutex> g(p->gmu);
    for (const auto& ge : p->graphs)
      if (ge.A == A && ge.B == B && ge.C == C && ge.ws == ws && ge.lda == lda && ge.ldb == ldb && ge.ldc == ldc)
        return cuda_status(cudaGraphLaunch(ge.exec, st), "fmm_execute graph launch");
  }
  {
    fmm_status es = ensure_device(p);  // uploads are not capturable
    if (es != FMM_OK) return es;
  }
  cudaStream_t cap = st;
  bool own = false;
  if (cap == nullptr) {  // the legacy stream cannot be captured: capture on a private stream
    if (cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) != cudaSuccess) return FMM_E_CUDA;
    own = true;
  }
  cudaError_t e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) { if (own) cudaStreamDestroy(cap); return cuda_status(e, "graph capture"); }
  fmm_status s = execute_impl(p, A, lda, B, ldb, C, ldc, ws, ws_bytes, cap);
  cudaGraph_t graph = nullptr;
  e = cudaStreamEndCapture(cap, &graph);
  if (own) cudaStreamDestroy(cap);
  if (s != FMM_OK) { if (graph) cudaGraphDestroy(graph); return s; }
  if (e != cudaSuccess) return cuda_status(e, "graph capture end");
  cudaGraphExec_t exec = nullptr;
  e = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return cuda_status(e, "graph instantiate");
  {
    std::lock_guard<std::mutex> g(p->gmu);
    p->graphs.push_back({A, B, C, ws, lda, ldb, ldc, exec});
  }
  return cuda_status(cudaGraphLaunch(exec, st), "fmm_execute graph launch");
}

static fmm_status execute_impl(const fmm_plan* p, const void* A, int64_t lda, const void* B,
                               int64_t ldb, void* C, int64_t ldc, void* ws, size_t ws_bytes,
                               void* stream) {
  if (!p) { set_error("fmm_execute: null plan"); return FMM_E_ARG; }
  const bool empty = p->M == 0 || p->N == 0;
  if (!empty && (!A && p->K > 0)) { set_error("fmm_execute: null A"); return FMM_E_ARG; }
  if (!empty && (!B && p->K > 0)) { set_error("fmm_execute: null B"); return FMM_E_ARG; }
  if (!empty && !C) { set_error("fmm_execute: null C"); return FMM_E_ARG; }
  if (lda < std::max<int64_t>(p->K, 1) || ldb < std::max<int64_t>(p->N, 1) || ldc < std::max<int64_t>(p->N, 1)) {
    set_error("fmm_execute: leading dimension smaller than the row length");
    return FMM_E_ARG;
  }
  size_t need = 0;
  fmm_plan_workspace_bytes(p, &need);
  if (ws_bytes < need || (need > 256 && !ws)) {
    set_error("fmm_execute: workspace too small (need " + std::to_string(need) + " bytes)");
    return FMM_E_OOM;
  }
  if (empty) return FMM_OK;
  {
    fmm_status es = ensure_device(p);
    if (es != FMM_OK) return es;
  }
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* wsb = (uint8_t*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  Bases b{};
  b.p[BASE_A] = A; b.p[BASE_B] = B; b.p[BASE_C] = C;
  b.p[BASE_WS] = wsb + p->scale_bytes + p->pad_bytes;
  b.ld[BASE_A] = lda; b.ld[BASE_B] = ldb; b.ld[BASE_C] = ldc; b.ld[BASE_WS] = 0;
  b.p[BASE_SYM] = p->sym_own; b.ld[BASE_SYM] = p->L > 0 ? p->ln[1] : 0;
  const bool p2p = p->p2p_active();
  if (p2p) {
    if (p->shard_depth != 1 || p->padded || p->scaling.mode != FMM_SCALE_NONE) {
      set_error("fmm_execute: comm mode 3 needs shard depth 1, no padding and no scaling");
      return FMM_E_ARG;
    }
    if (!p->sym_own) { set_error("fmm_execute: comm mode 3 needs fmm_plan_sym_alloc"); return FMM_E_ARG; }
  }
  double *dA = nullptr, *dB = nullptr;
  ScaleIn sin{};
  const ScaleIn* sinp = nullptr;
  if (p->scaling.mode != FMM_SCALE_NONE) {
    double* Ap = (double*)wsb;
    double* Bp = Ap + p->M * p->K;
    dA = Bp + p->K * p->N;
    dB = dA + p->M;
    double* dI = dB + p->N;
    void* sws = (void*)(((uintptr_t)(dI + p->K) + 255) & ~(uintptr_t)255);
    std::string steps;
    double tau;
    scaling_steps(p->scaling, &steps, &tau);
    NvtxRange nv("fmm.scale");
    TimedLaunch tl(p, 6, st);
    // Alg. 1-3 in one cooperative kernel; with virtual scaling the root K1 reads A, B and the
    // exponents (or A', B' if the run had to materialise them), else A', B' are written
    cudaError_t e = run_scaling_coop(p->M, p->K, p->N, (const double*)A, lda, (const double*)B, ldb,
                                     Ap, p->K, Bp, p->N, dA, dB, dI, (int)steps.size(), steps[0] == 'O',
                                     tau, p->scaling.pow2, p->virt_scale ? 0 : 1, sws, st);
    if (e != cudaSuccess) return cuda_status(e, "fmm_execute scaling");
    sin.ur = dA;
    sin.uc = dB;
    sinp = &sin;
    if (p->virt_scale) {
      const int32_t *ear, *eac, *ebr, *ebc;
      const int *mode, *ext;
      scale_virtual_view(sws, p->M, p->K, p->N, &ear, &eac, &ebr, &ebc, &mode, &ext);
      sin.ext = ext;
      sin.er[0] = ear; sin.ec[0] = eac; sin.er[1] = ebr; sin.ec[1] = ebc;
      sin.mat[0] = Ap; sin.mat[1] = Bp; sin.ldm[0] = p->K; sin.ldm[1] = p->N;
      sin.mode = mode;
    } else {
      b.p[BASE_A] = Ap; b.p[BASE_B] = Bp;
      b.ld[BASE_A] = p->K; b.ld[BASE_B] = p->N;
    }
  }
  if (p->padded) {  // zero-padded copies of A, B; the recursion writes a padded C
    const size_t es = (size_t)elem_size(p->dtype);
    auto al = [](size_t x) { return (x + 255) / 256 * 256; };
    uint8_t* pa = wsb + p->scale_bytes;
    uint8_t* pb = pa + al((size_t)p->Mp * p->Kp * es);
    uint8_t* pc = pb + al((size_t)p->Kp * p->Np * es);
    TimedLaunch tl(p, STEP_K1, st);
    cudaError_t e = p->dtype == FMM_F64
        ? launch_pad_copy<double>((const double*)b.p[BASE_A], p->M, p->K, b.ld[BASE_A], (double*)pa, p->Mp, p->Kp, p->Kp, st)
        : launch_pad_copy<float>((const float*)b.p[BASE_A], p->M, p->K, b.ld[BASE_A], (float*)pa, p->Mp, p->Kp, p->Kp, st);
    if (e == cudaSuccess)
      e = p->dtype == FMM_F64
          ? launch_pad_copy<double>((const double*)b.p[BASE_B], p->K, p->N, b.ld[BASE_B], (double*)pb, p->Kp, p->Np, p->Np, st)
          : launch_pad_copy<float>((const float*)b.p[BASE_B], p->K, p->N, b.ld[BASE_B], (float*)pb, p->Kp, p->Np, p->Np, st);
    if (e != cudaSuccess) return cuda_status(e, "fmm_execute pad");
    b.p[BASE_A] = pa; b.p[BASE_B] = pb; b.p[BASE_C] = pc;
    b.ld[BASE_A] = p->Kp; b.ld[BASE_B] = p->Np; b.ld[BASE_C] = p->Np;
  }
  const int vecn = 16 / elem_size(p->dtype);
  const bool vec = p->dims_vec_ok && aligned16(b.p[BASE_A]) && aligned16(b.p[BASE_B]) &&
                   aligned16(b.p[BASE_C]) && aligned16(b.p[BASE_WS]) && b.ld[BASE_A] % vecn == 0 &&
                   b.ld[BASE_B] % vecn == 0 && b.ld[BASE_C] % vecn == 0;
  fmm_status s = p->dtype == FMM_F64 ? run_steps<double>(p, b, vec, st, 0, (size_t)-1, sinp)
                                      : run_steps<float>(p, b, vec, st, 0, (size_t)-1, sinp);
  if (s != FMM_OK) return s;
  if (p->padded) {  // crop
    TimedLaunch tl(p, STEP_K3, st);
    cudaError_t e = p->dtype == FMM_F64
        ? launch_pad_copy<double>((const double*)b.p[BASE_C], p->M, p->N, p->Np, (double*)C, p->M, p->N, ldc, st)
        : launch_pad_copy<float>((const float*)b.p[BASE_C], p->M, p->N, p->Np, (float*)C, p->M, p->N, ldc, st);
    if (e != cudaSuccess) return cuda_status(e, "fmm_execute crop");
  }
  if (p->scaling.mode != FMM_SCALE_NONE && !p->unscale_fused) {
    NvtxRange nv("fmm.scale");
    TimedLaunch tl(p, 6, st);
    cudaError_t e = launch_unscale((double*)C, ldc, p->M, p->N, dA, dB, st);
    if (e != cudaSuccess) return cuda_status(e, "fmm_execute unscale");
  }
  if (p2p && (p->comm || p->barrier_fn)) {
    // every rank's owned M_r is in its symmetric buffer once all ranks pass this point; a 1-word
    // all-reduce orders the streams (device-side barrier; or the injected barrier), then rank q
    // computes rows [q M/P, (q+1) M/P) of C reading the products over NVLink, then a second
    // barrier keeps the next call from overwriting products a peer is still reading
    if (p->peers.size() != (size_t)p->nranks || !p->dev_peers) { set_error("fmm_execute: comm mode 3 needs fmm_plan_set_peer_handles"); return FMM_E_ARG; }
    NcclApi* api = p->barrier_fn ? nullptr : nccl();
    if (!p->barrier_fn && (!api || !api->allreduce)) { set_error("NCCL not loadable"); return FMM_E_NCCL; }
    float* bar = (float*)((uint8_t*)p->sym_own + sym_bytes_of(p) - 256);
    auto barrier = [&](float* word) -> fmm_status {
      NvtxRange nv("fmm.p2p_barrier");
      if (p->barrier_fn) {
        if (p->barrier_fn(p->barrier_user, (void*)st) != 0) { set_error("fmm_execute: injected barrier failed"); return FMM_E_NCCL; }
        return FMM_OK;
      }
      ncclResult_t r = api->allreduce(word, word, 1, ncclFloat32_, ncclSum_, p->comm, st);
      if (r != 0) { set_error(std::string("ncclAllReduce (barrier): ") + (api->getErrorString ? api->getErrorString(r) : "?")); return FMM_E_NCCL; }
      return FMM_OK;
    };
    fmm_status cs = barrier(bar);
    if (cs != FMM_OK) return cs;
    const int64_t row0 = p->M * p->rank / p->nranks, row1 = p->M * (p->rank + 1) / p->nranks;
    cs = p->dtype == FMM_F64 ? p2p_combine<double>(p, p->dev_peers, p->nranks, C, ldc, row0, row1, st)
                             : p2p_combine<float>(p, p->dev_peers, p->nranks, C, ldc, row0, row1, st);
    if (cs != FMM_OK) return cs;
    return barrier(bar + 1);
  }
  if (p->comm && !p2p) {  // a one-rank communicator issues the collective too (identity)
    NcclApi* api = nccl();
    if (!api) { set_error("NCCL not loadable"); return FMM_E_NCCL; }
    if (ldc != p->N) { set_error("fmm_execute: multi-GPU reduce needs ldc == N"); return FMM_E_ARG; }
    NvtxRange nv("fmm.nccl");
    TimedLaunch tl(p, 7, st);
    const int dt = p->dtype == FMM_F64 ? ncclFloat64_ : ncclFloat32_;
    const size_t total = (size_t)(p->M * p->N);
    ncclResult_t r = 0;
    const char* what = "ncclReduce";
    if (p->comm_mode == 1) {  // every rank gets C
      what = "ncclAllReduce";
      r = api->allreduce ? api->allreduce(C, C, total, dt, ncclSum_, p->comm, st) : 1;
    } else if (p->comm_mode == 2) {  // rank r gets rows [r M/P, (r+1) M/P) of C, in place
      what = "ncclReduceScatter";
      if (p->M % p->nranks) { set_error("fmm_execute: reduce-scatter needs M divisible by the ranks"); return FMM_E_SHAPE; }
      const size_t cnt = total / (size_t)p->nranks;
      const size_t es = (size_t)elem_size(p->dtype);
      r = api->reduce_scatter ? api->reduce_scatter(C, (uint8_t*)C + (size_t)p->rank * cnt * es, cnt, dt, ncclSum_, p->comm, st) : 1;
    } else {  // C on rank 0
      r = api->reduce(C, C, total, dt, ncclSum_, 0, p->comm, st);
    }
    if (r != 0) { set_error(std::string(what) + ": " + (api->getErrorString ? api->getErrorString(r) : "?")); return FMM_E_NCCL; }
  }
  return FMM_OK;
}

fmm_status fmm_plan_set_single_launch(fmm_plan* p, int enable) {
  if (!p) { set_error("fmm_plan_set_single_launch: null plan"); return FMM_E_ARG; }
  p->single_launch = enable != 0;
  return compile_plan(p);
}

fmm_status fmm_plan_set_virtual_scaling(fmm_plan* p, int enable) {
  if (!p) { set_error("fmm_plan_set_virtual_scaling: null plan"); return FMM_E_ARG; }
  p->virt_scale_enable = enable != 0;
  return compile_plan(p);
}

fmm_status fmm_plan_set_barrier(fmm_plan* p, fmm_barrier_fn fn, void* user) {
  if (!p) { set_error("fmm_plan_set_barrier: null plan"); return FMM_E_ARG; }
  const bool recompile = (fn != nullptr) != (p->barrier_fn != nullptr);
  p->barrier_fn = fn;
  p->barrier_user = user;
  return recompile ? compile_plan(p) : FMM_OK;
}

fmm_status fmm_plan_set_timing(fmm_plan* p, int enable) {
  if (!p) { set_error("fmm_plan_set_timing: null"); return FMM_E_ARG; }
  p->timing = enable != 0;
  return FMM_OK;
}

fmm_status fmm_plan_step_times(fmm_plan* p, double* ms, int64_t* launches) {
  if (!p || !ms || !launches) { set_error("fmm_plan_step_times: null"); return FMM_E_ARG; }
  for (int k = 0; k < 8; ++k) { ms[k] = 0; launches[k] = 0; }
  std::lock_guard<std::mutex> g(p->tmu);
  cudaError_t err = cudaSuccess;
  for (auto& u : p->ev_used) {
    cudaError_t e = cudaEventSynchronize(u.second.second);
    float t = 0;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&t, u.second.first, u.second.second);
    if (e != cudaSuccess && err == cudaSuccess) err = e;
    const int k = u.first & 7;
    ms[k] += t;
    launches[k] += 1;
    p->ev_pool.push_back(u.second.first);
    p->ev_pool.push_back(u.second.second);
  }
  p->ev_used.clear();
  return cuda_status(err, "fmm_plan_step_times");
}

// Host-buffer execution with the copies overlapped with the compute (depth-first plans): the
// top-level blocks of A and B are copied H2D on a copy stream in order of first use, each
// top-level product r waits only for the blocks its K1 reads, and every block C_k is copied
// D2H as soon as its last contribution (the last r with w_kr != 0) has been accumulated.
// The plan's two copy streams (host-to-device, device-to-host) on the current device.
static fmm_status ensure_copy_streams(const fmm_plan* p) {
  std::lock_guard<std::mutex> g(p->dev_mu);
  int dev = 0;
  cudaGetDevice(&dev);
  if (p->copy_dev != dev) {
    if (p->copy_h2d) cudaStreamDestroy(p->copy_h2d);
    if (p->copy_d2h) cudaStreamDestroy(p->copy_d2h);
    cudaError_t e = cudaStreamCreateWithFlags(&p->copy_h2d, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->copy_d2h, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_status(e, "fmm_execute_host streams");
    p->copy_dev = dev;
  }
  return FMM_OK;
}

// gate: if non-null, the copies into A_dev / B_dev wait for this event instead of for all
// earlier work on st (fmm_execute_host_batch: the compute that last read this buffer set).
// join: st waits for the C_host copies at the end.  done_out: if non-null, receives an event
// recorded after the last C_host copy (the caller destroys it).
static fmm_status execute_host_pipelined(const fmm_plan* p, const void* A_host, int64_t lda,
                                         const void* B_host, int64_t ldb, void* C_host,
                                         int64_t ldc, void* A_dev, void* B_dev, void* C_dev,
                                         void* ws, size_t ws_bytes, cudaStream_t st,
                                         cudaEvent_t gate = nullptr, bool join = true,
                                         cudaEvent_t* done_out = nullptr,
                                         const fmm_plan* streams_of = nullptr) {
  // the copy streams belong to the caller's plan (a depth-first twin shares its parent's), so
  // the copies of consecutive calls stay ordered whichever schedule runs the compute
  const fmm_plan* so = streams_of ? streams_of : p;
  fmm_status fs = ensure_device(p);
  if (fs != FMM_OK) return fs;
  size_t need = 0;
  fmm_plan_workspace_bytes(p, &need);
  if (ws_bytes < need || !ws) { set_error("fmm_execute_host: workspace too small"); return FMM_E_OOM; }
  cudaError_t e = cudaSuccess;
  if ((fs = ensure_copy_streams(so)) != FMM_OK) return fs;
  const RuleData& ru = p->rules[p->node_rule[0][0]];
  const size_t es = (size_t)elem_size(p->dtype);
  const int64_t mb = p->lm[1], kb = p->lk[1], nb = p->ln[1];
  const int nA = ru.m0 * ru.k0, nB = ru.k0 * ru.n0, nC = ru.m0 * ru.n0;
  std::vector<cudaEvent_t> evs;
  auto mkev = [&](cudaEvent_t* ev) {
    cudaError_t r = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    if (r == cudaSuccess) evs.push_back(*ev);
    return r;
  };
  cudaEvent_t entry = gate;
  if (!entry) {
    if ((e = mkev(&entry)) != cudaSuccess) return cuda_status(e, "event");
    cudaEventRecord(entry, st);  // device buffers may still be in use by earlier work on st
  }
  cudaStreamWaitEvent(so->copy_h2d, entry, 0);
  std::vector<cudaEvent_t> evA(nA, nullptr), evB(nB, nullptr);
  auto copyA = [&](int i) {
    const int ia = i % ru.m0, ja = i / ru.m0;  // column-major block index
    cudaMemcpy2DAsync((char*)A_dev + ((ia * mb) * p->K + ja * kb) * es, p->K * es,
                      (const char*)A_host + ((ia * mb) * lda + ja * kb) * es, lda * es, kb * es, mb,
                      cudaMemcpyHostToDevice, so->copy_h2d);
    mkev(&evA[i]);
    cudaEventRecord(evA[i], so->copy_h2d);
  };
  auto copyB = [&](int j) {
    const int ja = j % ru.k0, jb = j / ru.k0;
    cudaMemcpy2DAsync((char*)B_dev + ((ja * kb) * p->N + jb * nb) * es, p->N * es,
                      (const char*)B_host + ((ja * kb) * ldb + jb * nb) * es, ldb * es, nb * es, kb,
                      cudaMemcpyHostToDevice, so->copy_h2d);
    mkev(&evB[j]);
    cudaEventRecord(evB[j], so->copy_h2d);
  };
  for (const auto& g : p->groups) {
    for (int i = 0; i < nA; ++i)
      if (ru.U[(size_t)i * ru.R + g.r] != 0 && !evA[i]) copyA(i);
    for (int j = 0; j < nB; ++j)
      if (ru.V[(size_t)j * ru.R + g.r] != 0 && !evB[j]) copyB(j);
  }
  for (int i = 0; i < nA; ++i) if (!evA[i]) copyA(i);
  for (int j = 0; j < nB; ++j) if (!evB[j]) copyB(j);
  // last group contributing to each C block
  std::vector<int> last(nC, -1);
  for (size_t gi = 0; gi < p->groups.size(); ++gi)
    for (int k = 0; k < nC; ++k)
      if (ru.W[(size_t)k * ru.R + p->groups[gi].r] != 0) last[k] = (int)gi;
  uint8_t* wsb = (uint8_t*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  Bases b{};
  b.p[BASE_A] = A_dev; b.p[BASE_B] = B_dev; b.p[BASE_C] = C_dev; b.p[BASE_WS] = wsb + p->scale_bytes;
  b.ld[BASE_A] = p->K; b.ld[BASE_B] = p->N; b.ld[BASE_C] = p->N; b.ld[BASE_WS] = 0;
  const int vecn = 16 / elem_size(p->dtype);
  const bool vec = p->dims_vec_ok && aligned16(A_dev) && aligned16(B_dev) && aligned16(C_dev) &&
                   aligned16(b.p[BASE_WS]) && p->K % vecn == 0 && p->N % vecn == 0;
  std::vector<bool> copied(nC, false);
  auto copyC = [&](int k) {
    cudaEvent_t ev;
    mkev(&ev);
    cudaEventRecord(ev, st);
    cudaStreamWaitEvent(so->copy_d2h, ev, 0);
    const int ia = k / ru.n0, jb = k % ru.n0;  // row-major block index
    cudaMemcpy2DAsync((char*)C_host + ((ia * mb) * ldc + jb * nb) * es, ldc * es,
                      (const char*)C_dev + ((ia * mb) * p->N + jb * nb) * es, p->N * es, nb * es, mb,
                      cudaMemcpyDeviceToHost, so->copy_d2h);
    copied[k] = true;
  };
  for (size_t gi = 0; gi < p->groups.size(); ++gi) {
    const auto& g = p->groups[gi];
    for (int i = 0; i < nA; ++i)
      if (ru.U[(size_t)i * ru.R + g.r] != 0) cudaStreamWaitEvent(st, evA[i], 0);
    for (int j = 0; j < nB; ++j)
      if (ru.V[(size_t)j * ru.R + g.r] != 0) cudaStreamWaitEvent(st, evB[j], 0);
    fs = p->dtype == FMM_F64 ? run_steps<double>(p, b, vec, st, g.begin, g.end)
                             : run_steps<float>(p, b, vec, st, g.begin, g.end);
    if (fs != FMM_OK) return fs;
    for (int k = 0; k < nC; ++k)
      if (last[k] == (int)gi) copyC(k);
  }
  const size_t tail0 = p->groups.empty() ? 0 : p->groups.back().end;
  if (tail0 < p->steps.size()) {
    for (int i = 0; i < nA; ++i) cudaStreamWaitEvent(st, evA[i], 0);
    for (int j = 0; j < nB; ++j) cudaStreamWaitEvent(st, evB[j], 0);
    fs = p->dtype == FMM_F64 ? run_steps<double>(p, b, vec, st, tail0) : run_steps<float>(p, b, vec, st, tail0);
    if (fs != FMM_OK) return fs;
  }
  for (int k = 0; k < nC; ++k)
    if (!copied[k]) copyC(k);
  cudaEvent_t done;
  if (done_out) {
    if ((e = cudaEventCreateWithFlags(&done, cudaEventDisableTiming)) != cudaSuccess)
      return cuda_status(e, "event");
    *done_out = done;
  } else {
    mkev(&done);
  }
  cudaEventRecord(done, so->copy_d2h);
  if (join) cudaStreamWaitEvent(st, done, 0);  // stream completion => C_host valid
  e = cudaGetLastError();
  for (cudaEvent_t ev : evs) cudaEventDestroy(ev);  // deferred until the events complete
  return cuda_status(e, "fmm_execute_host");
}

// The depth-first twin of a breadth-first plan (same rules, dims, dtype; bitwise-identical
// results), built on first use.
static const fmm_plan* depth_first_twin(const fmm_plan* p) {
  std::lock_guard<std::mutex> g(p->dev_mu);
  if (!p->df_twin) {
    fmm_plan* t = new fmm_plan();
    t->dtype = p->dtype; t->leaf = p->leaf; t->L = p->L; t->M = p->M; t->K = p->K; t->N = p->N;
    t->Mp = p->Mp; t->Kp = p->Kp; t->Np = p->Np; t->padded = p->padded;
    t->rules = p->rules; t->node_rule = p->node_rule; t->lm = p->lm; t->lk = p->lk; t->ln = p->ln;
    t->scaling = p->scaling; t->coef_U = p->coef_U; t->coef_V = p->coef_V; t->coef_W = p->coef_W;
    t->coef_host = p->coef_host; t->schedule = 2; t->fusion = p->fusion; t->shard_depth = p->shard_depth; t->shard_block = p->shard_block;
    t->split_chains = p->split_chains;
    t->k1_two_level = p->k1_two_level;
    t->tf32_presplit = p->tf32_presplit;
    t->k3_two_level = p->k3_two_level;
    if (compile_plan(t) != FMM_OK) { delete t; return nullptr; }
    p->df_twin = t;
  }
  return p->df_twin;
}

// The plan whose top-level groups drive the host-copy pipeline (the plan itself if depth-first
// at the top, else its depth-first twin), or null where the pipeline does not apply.
static const fmm_plan* host_pipeline_plan(const fmm_plan* p, const void* ws, size_t ws_bytes) {
  if (!(p->L > 0 && p->scaling.mode == FMM_SCALE_NONE && !p->comm && !p->padded && p->M > 0 &&
        p->N > 0 && p->K > 0))
    return nullptr;
  // a partitioned plan runs its own (depth-first) schedule; with no owned product it has no
  // groups and fmm_execute's zeroing of C is the whole job -- never the full-product twin
  if (p->nranks > 1 && p->groups.empty()) return nullptr;
  const fmm_plan* q = p->groups.empty() ? depth_first_twin(p) : p;
  size_t need = 0;
  if (q) fmm_plan_workspace_bytes(q, &need);
  return q && !q->groups.empty() && ws && ws_bytes >= need ? q : nullptr;
}

fmm_status fmm_execute_host(const fmm_plan* p, const void* A_host, int64_t lda,
                            const void* B_host, int64_t ldb, void* C_host, int64_t ldc,
                            void* A_dev, void* B_dev, void* C_dev, void* ws, size_t ws_bytes,
                            void* stream) {
  if (!p || !A_host || !B_host || !C_host || !A_dev || !B_dev || !C_dev) {
    set_error("fmm_execute_host: null pointer");
    return FMM_E_ARG;
  }
  if (lda < p->K || ldb < p->N || ldc < p->N) { set_error("fmm_execute_host: bad ld"); return FMM_E_ARG; }
  cudaStream_t st = (cudaStream_t)stream;
  if (const fmm_plan* q = host_pipeline_plan(p, ws, ws_bytes))
    return execute_host_pipelined(q, A_host, lda, B_host, ldb, C_host, ldc, A_dev, B_dev, C_dev,
                                  ws, ws_bytes, st, nullptr, true, nullptr, p);
  const size_t es = (size_t)elem_size(p->dtype);
  cudaError_t e = cudaMemcpy2DAsync(A_dev, p->K * es, A_host, lda * es, p->K * es, p->M, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess)
    e = cudaMemcpy2DAsync(B_dev, p->N * es, B_host, ldb * es, p->N * es, p->K, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_status(e, "fmm_execute_host H2D");
  fmm_status s = fmm_execute(p, A_dev, p->K, B_dev, p->N, C_dev, p->N, ws, ws_bytes, stream);
  if (s != FMM_OK) return s;
  e = cudaMemcpy2DAsync(C_host, ldc * es, C_dev, p->N * es, p->N * es, p->M, cudaMemcpyDeviceToHost, st);
  return cuda_status(e, "fmm_execute_host D2H");
}

fmm_status fmm_execute_host_batch(const fmm_plan* p, int count, const void* const* A_hosts,
                                  int64_t lda, const void* const* B_hosts, int64_t ldb,
                                  void* const* C_hosts, int64_t ldc, void* const* A_devs,
                                  void* const* B_devs, void* const* C_devs, int nbuf, void* ws,
                                  size_t ws_bytes, void* stream) {
  if (!p || count < 0 || nbuf < 1 || !A_hosts || !B_hosts || !C_hosts || !A_devs || !B_devs || !C_devs) {
    set_error("fmm_execute_host_batch: bad arguments");
    return FMM_E_ARG;
  }
  for (int i = 0; i < count; ++i)
    if (!A_hosts[i] || !B_hosts[i] || !C_hosts[i]) { set_error("fmm_execute_host_batch: null host pointer"); return FMM_E_ARG; }
  for (int s = 0; s < nbuf; ++s)
    if (!A_devs[s] || !B_devs[s] || !C_devs[s]) { set_error("fmm_execute_host_batch: null device pointer"); return FMM_E_ARG; }
  if (lda < p->K || ldb < p->N || ldc < p->N) { set_error("fmm_execute_host_batch: bad ld"); return FMM_E_ARG; }
  cudaStream_t st = (cudaStream_t)stream;
  const fmm_plan* q = host_pipeline_plan(p, ws, ws_bytes);
  if (nbuf == 1) {  // no cross-problem overlap: one problem after the other
    for (int i = 0; i < count; ++i) {
      const int s = i % nbuf;
      fmm_status fs = fmm_execute_host(p, A_hosts[i], lda, B_hosts[i], ldb, C_hosts[i], ldc,
                                       A_devs[s], B_devs[s], C_devs[s], ws, ws_bytes, stream);
      if (fs != FMM_OK) return fs;
    }
    return FMM_OK;
  }
  // Problem i uses buffer set i mod nbuf.  Its input copies wait only for the compute of problem
  // i - nbuf (the last reader of that set), so they stream in while problem i - 1 computes; its
  // compute waits for problem i - nbuf's C copy-out (the same C buffer).  One compute stream, so
  // the workspace is reused safely.
  std::vector<cudaEvent_t> cdone(count, nullptr), ddone(count, nullptr);
  cudaEvent_t entry = nullptr;
  cudaError_t e = cudaEventCreateWithFlags(&entry, cudaEventDisableTiming);
  if (e != cudaSuccess) return cuda_status(e, "fmm_execute_host_batch event");
  cudaEventRecord(entry, st);
  fmm_status fs = FMM_OK;
  for (int i = 0; i < count && fs == FMM_OK; ++i) {
    const int s = i % nbuf;
    if (i >= nbuf) cudaStreamWaitEvent(st, ddone[i - nbuf], 0);
    cudaEvent_t gate = i >= nbuf ? cdone[i - nbuf] : entry;
    // Per-block copies (the depth-first groups) matter only at the edges of the stream -- the
    // first problem's inputs and the last one's output are not hidden behind a neighbour's
    // compute.  In between, whole-operand copies around the plan's own schedule (for C5 the
    // hybrid one, 18 ms per product faster than the depth-first twin) hide just as well.
    const bool edge = i == 0 || i == count - 1 || q == p;
    if (q && edge) {
      fs = execute_host_pipelined(q, A_hosts[i], lda, B_hosts[i], ldb, C_hosts[i], ldc, A_devs[s],
                                  B_devs[s], C_devs[s], ws, ws_bytes, st, gate, false, &ddone[i], p);
    } else {  // whole-operand copies on the copy streams around an ordinary fmm_execute
      fs = ensure_copy_streams(p);
      const size_t es = (size_t)elem_size(p->dtype);
      cudaEvent_t in = nullptr, out = nullptr;
      if (fs == FMM_OK && ((e = cudaEventCreateWithFlags(&in, cudaEventDisableTiming)) != cudaSuccess ||
                           (e = cudaEventCreateWithFlags(&out, cudaEventDisableTiming)) != cudaSuccess ||
                           (e = cudaEventCreateWithFlags(&ddone[i], cudaEventDisableTiming)) != cudaSuccess))
        fs = cuda_status(e, "fmm_execute_host_batch event");
      if (fs == FMM_OK) {
        cudaStreamWaitEvent(p->copy_h2d, gate, 0);
        cudaMemcpy2DAsync(A_devs[s], p->K * es, A_hosts[i], lda * es, p->K * es, p->M, cudaMemcpyHostToDevice, p->copy_h2d);
        cudaMemcpy2DAsync(B_devs[s], p->N * es, B_hosts[i], ldb * es, p->N * es, p->K, cudaMemcpyHostToDevice, p->copy_h2d);
        cudaEventRecord(in, p->copy_h2d);
        cudaStreamWaitEvent(st, in, 0);
        fs = fmm_execute(p, A_devs[s], p->K, B_devs[s], p->N, C_devs[s], p->N, ws, ws_bytes, stream);
      }
      if (fs == FMM_OK) {
        cudaEventRecord(out, st);
        cudaStreamWaitEvent(p->copy_d2h, out, 0);
        cudaMemcpy2DAsync(C_hosts[i], ldc * es, C_devs[s], p->N * es, p->N * es, p->M, cudaMemcpyDeviceToHost, p->copy_d2h);
        cudaEventRecord(ddone[i], p->copy_d2h);
      }
      if (in) cudaEventDestroy(in);
      if (out) cudaEventDestroy(out);
    }
    if (fs != FMM_OK) break;
    if ((e = cudaEventCreateWithFlags(&cdone[i], cudaEventDisableTiming)) != cudaSuccess) {
      fs = cuda_status(e, "fmm_execute_host_batch event");
      break;
    }
    cudaEventRecord(cdone[i], st);
  }
  for (int i = 0; i < count; ++i)
    if (ddone[i]) cudaStreamWaitEvent(st, ddone[i], 0);  // stream completion => all C_host valid
  for (int i = 0; i < count; ++i) {
    if (cdone[i]) cudaEventDestroy(cdone[i]);
    if (ddone[i]) cudaEventDestroy(ddone[i]);
  }
  cudaEventDestroy(entry);
  if (fs != FMM_OK) return fs;
  return cuda_status(cudaGetLastError(), "fmm_execute_host_batch");
}

fmm_status fmm_plan_last_scaling_steps(const fmm_plan* p, void* ws, int* steps, void* stream) {
  if (!p || !ws || !steps) { set_error("fmm_plan_last_scaling_steps: null"); return FMM_E_ARG; }
  if (p->scaling.mode == FMM_SCALE_NONE) { *steps = 0; return FMM_OK; }
  uint8_t* wsb = (uint8_t*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  double* dI = (double*)wsb + p->M * p->K + p->K * p->N + p->M + p->N;
  void* sws = (void*)(((uintptr_t)(dI + p->K) + 255) & ~(uintptr_t)255);
  int flags[8];
  cudaError_t e = cudaMemcpyAsync(flags, scale_flags_ptr(sws, p->M, p->K, p->N), sizeof flags,
                                  cudaMemcpyDeviceToHost, (cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_status(e, "fmm_plan_last_scaling_steps");
  *steps = flags[1];
  if (flags[2]) {
    static const char* what[] = {"", "row of A", "column of B", "column of A", "row of B"};
    set_error(std::string("scaling precondition: all-zero ") + what[flags[2] & 7] + " at index " + std::to_string(flags[3]));
    return FMM_E_PRECOND;
  }
  return FMM_OK;
}

// ---- building blocks ----------------------------------------------------------------------------

fmm_status fmm_node_st(const fmm_rule* rule, int dtype, int64_t m, int64_t k, int64_t n,
                       const void* A, int64_t lda, const void* B, int64_t ldb, void* S, void* T,
                       void* stream) {
  if (!rule || !A || !B || !S || !T) { set_error("fmm_node_st: null"); return FMM_E_ARG; }
  const RuleData& r = rule->d;
  if (m % r.m0 || k % r.k0 || n % r.n0) { set_error("fmm_node_st: dims not divisible"); return FMM_E_SHAPE; }
  // build K1 descriptors directly (no plan schedule needed): ws base = S for U, T for V
  std::vector<double> coef;
  for (int i = 0; i < r.m0 * r.k0; ++i) for (int q = 0; q < r.R; ++q) coef.push_back(r.coef(r.U, i, q));
  const int offV = (int)coef.size();
  for (int j = 0; j < r.k0 * r.n0; ++j) for (int q = 0; q < r.R; ++q) coef.push_back(r.coef(r.V, j, q));
  const int64_t mb = m / r.m0, kb = k / r.k0, nb = n / r.n0;
  K1Node ks{}, kt{};
  ks.in = Op{BASE_A, 0, 0, 0, -1};
  kt.in = Op{BASE_B, 0, 0, 0, -1};
  ks.rows = m / r.m0; ks.cols = k / r.k0; ks.P = r.m0; ks.Q = r.k0;
  kt.rows = k / r.k0; kt.cols = n / r.n0; kt.P = r.k0; kt.Q = r.n0;
  ks.coef_off = 0;
  kt.coef_off = offV;
  for (int q = 0; q < r.R; ++q) {
    ks.out[q] = Op{BASE_C, 0, 0, q * mb * kb, kb};
    kt.out[q] = Op{BASE_WS, 0, 0, q * kb * nb, nb};
  }
  ks.out_mask = kt.out_mask = (r.R >= 32) ? 0xffffffffu : ((1u << r.R) - 1u);
  k1_compile(ks, r, r.U, r.m0 * r.k0);
  k1_compile(kt, r, r.V, r.k0 * r.n0);
  cudaStream_t st = (cudaStream_t)stream;
  void* dmem = nullptr;
  size_t bytes = coef.size() * 8 + 2 * sizeof(K1Node) + 512;
  cudaError_t e = cudaMallocAsync(&dmem, bytes, st);
  if (e != cudaSuccess) return cuda_status(e, "fmm_node_st alloc");
  uint8_t* d8 = (uint8_t*)dmem;
  double* dcoef = (double*)d8;
  K1Node* dn = (K1Node*)(d8 + ((coef.size() * 8 + 255) / 256 * 256));
  std::vector<uint8_t> host(bytes, 0);
  std::memcpy(host.data(), coef.data(), coef.size() * 8);
  std::memcpy(host.data() + ((uint8_t*)dn - d8), &ks, sizeof ks);
  std::memcpy(host.data() + ((uint8_t*)dn - d8) + sizeof ks, &kt, sizeof kt);
  e = cudaMemcpyAsync(dmem, host.data(), bytes, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // host buffer lifetime
  Bases b{};
  b.p[BASE_A] = A; b.p[BASE_B] = B; b.p[BASE_C] = S; b.p[BASE_WS] = T;
  b.ld[BASE_A] = lda; b.ld[BASE_B] = ldb;
  const int vecn = 16 / elem_size(dtype);
  const bool vec = aligned16(A) && aligned16(B) && aligned16(S) && aligned16(T) && lda % vecn == 0 &&
                   ldb % vecn == 0 && kb % vecn == 0 && nb % vecn == 0;
  Step s1{};
  s1.kind = STEP_K1; s1.count = 1; s1.rows = mb; s1.cols = kb; s1.P = r.m0 * r.k0; s1.Q = 1; s1.R = r.R;
  Step s2 = s1;
  s2.rows = kb; s2.cols = nb; s2.P = r.k0 * r.n0;
  if (e == cudaSuccess) {
    e = dtype == FMM_F64 ? launch_k1<double>(s1, dn, dcoef, b, vec, st) : launch_k1<float>(s1, dn, dcoef, b, vec, st);
  }
  if (e == cudaSuccess) {
    e = dtype == FMM_F64 ? launch_k1<double>(s2, dn + 1, dcoef, b, vec, st) : launch_k1<float>(s2, dn + 1, dcoef, b, vec, st);
  }
  cudaError_t e2 = cudaFreeAsync(dmem, st);
  if (e == cudaSuccess) e = e2;
  return cuda_status(e, "fmm_node_st");
}

fmm_status fmm_node_c(const fmm_rule* rule, int dtype, int64_t m, int64_t n, const void* Ms,
                      void* C, int64_t ldc, void* stream) {
  if (!rule || !Ms || !C) { set_error("fmm_node_c: null"); return FMM_E_ARG; }
  const RuleData& r = rule->d;
  if (m % r.m0 || n % r.n0) { set_error("fmm_node_c: dims not divisible"); return FMM_E_SHAPE; }
  const int64_t mb = m / r.m0, nb = n / r.n0;
  std::vector<double> coef;
  for (int k = 0; k < r.m0 * r.n0; ++k) for (int q = 0; q < r.R; ++q) coef.push_back(r.coef(r.W, k, q));
  K3Node kn{};
  kn.out = Op{BASE_C, 0, 0, 0, -1};
  kn.coef_off = 0;
  for (int q = 0; q < r.R; ++q) kn.in[q] = Op{BASE_WS, 0, 0, q * mb * nb, nb};
  cudaStream_t st = (cudaStream_t)stream;
  void* dmem = nullptr;
  size_t off = (coef.size() * 8 + 255) / 256 * 256;
  size_t bytes = off + sizeof kn;
  cudaError_t e = cudaMallocAsync(&dmem, bytes, st);
  if (e != cudaSuccess) return cuda_status(e, "fmm_node_c alloc");
  std::vector<uint8_t> host(bytes, 0);
  std::memcpy(host.data(), coef.data(), coef.size() * 8);
  std::memcpy(host.data() + off, &kn, sizeof kn);
  e = cudaMemcpyAsync(dmem, host.data(), bytes, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  Bases b{};
  b.p[BASE_C] = C; b.p[BASE_WS] = Ms; b.ld[BASE_C] = ldc;
  const int vecn = 16 / elem_size(dtype);
  const bool vec = aligned16(C) && aligned16(Ms) && ldc % vecn == 0 && nb % vecn == 0;
  Step s{};
  s.kind = STEP_K3; s.count = 1; s.rows = mb; s.cols = nb; s.P = r.m0; s.Q = r.n0; s.R = r.R;
  if (e == cudaSuccess)
    e = dtype == FMM_F64 ? launch_k3<double>(s, (uint8_t*)dmem + off, (double*)dmem, b, vec, st)
                         : launch_k3<float>(s, (uint8_t*)dmem + off, (double*)dmem, b, vec, st);
  cudaError_t e2 = cudaFreeAsync(dmem, st);
  if (e == cudaSuccess) e = e2;
  return cuda_status(e, "fmm_node_c");
}

fmm_status fmm_gemm(int dtype, int leaf, int64_t M, int64_t K, int64_t N, const void* A,
                    int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc, void* stream) {
  if ((M && N && !C) || lda < std::max<int64_t>(K, 1) || ldb < std::max<int64_t>(N, 1) || ldc < std::max<int64_t>(N, 1)) {
    set_error("fmm_gemm: bad argument"); return FMM_E_ARG;
  }
  if (dtype == FMM_F64 && leaf != FMM_LEAF_NATIVE) { set_error("fmm_gemm: FP64 requires NATIVE leaf"); return FMM_E_ARG; }
  if (M == 0 || N == 0) return FMM_OK;
  cudaStream_t st = (cudaStream_t)stream;
  LeafNode lf{Op{BASE_A, 0, 0, 0, -1}, Op{BASE_B, 0, 0, 0, -1}, Op{BASE_C, 0, 0, 0, -1}};
  void* dmem = nullptr;
  const size_t arena = (dtype == FMM_F32 && leaf != FMM_LEAF_NATIVE) ? tf32_arena_floats(1, M, N, K) * 4 : 0;
  cudaError_t e = cudaMallocAsync(&dmem, 256 + arena, st);
  if (e != cudaSuccess) return cuda_status(e, "fmm_gemm alloc");
  e = cudaMemcpyAsync(dmem, &lf, sizeof lf, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  Bases b{};
  b.p[BASE_A] = A; b.p[BASE_B] = B; b.p[BASE_C] = C;
  b.ld[BASE_A] = lda; b.ld[BASE_B] = ldb; b.ld[BASE_C] = ldc;
  const int vecn = 16 / elem_size(dtype);
  const bool vec = aligned16(A) && aligned16(B) && aligned16(C) && lda % vecn == 0 && ldb % vecn == 0 &&
                   ldc % vecn == 0 && K % vecn == 0 && N % vecn == 0;
  if (e == cudaSuccess)
    e = dtype == FMM_F64 ? launch_gemm_f64((const LeafNode*)dmem, 1, M, N, K, b, vec, st)
                         : launch_gemm_f32((const LeafNode*)dmem, &lf, 1, M, N, K, b, vec, leaf,
                                           arena ? (float*)((uint8_t*)dmem + 256) : nullptr, st);
  cudaError_t e2 = cudaFreeAsync(dmem, st);
  if (e == cudaSuccess) e = e2;
  return cuda_status(e, "fmm_gemm");
}

// ---- scaling entry points ---------------------------------------------------------------------

fmm_status fmm_scale_workspace_bytes(int64_t M, int64_t K, int64_t N, size_t* bytes) {
  if (!bytes) return FMM_E_ARG;
  *bytes = scale_ws_bytes(M, K, N) + 1024;  // + alignment + the grid-barrier word
  return FMM_OK;
}

fmm_status fmm_scale_outside(int dtype, int64_t M, int64_t K, int64_t N, const void* A,
                             int64_t lda, const void* B, int64_t ldb, void* A_out,
                             int64_t lda_out, void* B_out, int64_t ldb_out, void* dA, void* dB,
                             int pow2, void* stream) {
  if (dtype != FMM_F64) { set_error("scaling: FP64 only"); return FMM_E_UNSUPPORTED; }
  if (!dA || !dB) { set_error("fmm_scale_outside: null factor vector"); return FMM_E_ARG; }
  return scale_common(M, K, N, A, lda, B, ldb, A_out, lda_out, B_out, ldb_out, dA, dB, nullptr,
                      "O", -1.0, pow2, nullptr, nullptr, (cudaStream_t)stream, true);
}

fmm_status fmm_scale_inside(int dtype, int64_t M, int64_t K, int64_t N, const void* A,
                            int64_t lda, const void* B, int64_t ldb, void* A_out,
                            int64_t lda_out, void* B_out, int64_t ldb_out, void* d, int pow2,
                            void* stream) {
  if (dtype != FMM_F64) { set_error("scaling: FP64 only"); return FMM_E_UNSUPPORTED; }
  if (!d) { set_error("fmm_scale_inside: null factor vector"); return FMM_E_ARG; }
  return scale_common(M, K, N, A, lda, B, ldb, A_out, lda_out, B_out, ldb_out, nullptr, nullptr,
                      d, "I", -1.0, pow2, nullptr, nullptr, (cudaStream_t)stream, true);
}

fmm_status fmm_scale_repeated(int dtype, int64_t M, int64_t K, int64_t N, const void* A,
                              int64_t lda, const void* B, int64_t ldb, const fmm_scaling* cfg,
                              void* A_out, int64_t lda_out, void* B_out, int64_t ldb_out,
                              void* dA, void* dB, void* dI, int32_t* steps_dev, void* ws,
                              size_t ws_bytes, void* stream) {
  if (dtype != FMM_F64) { set_error("scaling: FP64 only"); return FMM_E_UNSUPPORTED; }
  if (!cfg || cfg->max_steps < 1 || !dA || !dB || !dI) { set_error("fmm_scale_repeated: bad config / null factor"); return FMM_E_ARG; }
  size_t need;
  fmm_scale_workspace_bytes(M, K, N, &need);
  if (ws && ws_bytes < need) { set_error("fmm_scale_repeated: workspace too small"); return FMM_E_OOM; }
  std::string steps;
  double tau;
  fmm_scaling c = *cfg;
  c.mode = FMM_SCALE_REPEATED;
  scaling_steps(c, &steps, &tau);
  return scale_common(M, K, N, A, lda, B, ldb, A_out, lda_out, B_out, ldb_out, dA, dB, dI, steps,
                      tau, cfg->pow2, steps_dev, ws, (cudaStream_t)stream, false);
}

fmm_status fmm_scale_apply(int dtype, int64_t M, int64_t K, int64_t N, const void* A, int64_t lda,
                           const void* B, int64_t ldb, const void* dA, const void* d,
                           const void* dB, void* A_out, int64_t lda_out, void* B_out,
                           int64_t ldb_out, void* stream) {
  if (dtype != FMM_F64) { set_error("scaling: FP64 only"); return FMM_E_UNSUPPORTED; }
  if (!A || !B || !dA || !d || !dB || !A_out || !B_out || M < 0 || K < 0 || N < 0 || lda < K ||
      ldb < N || lda_out < K || ldb_out < N) {
    set_error("fmm_scale_apply: bad argument");
    return FMM_E_ARG;
  }
  return cuda_status(launch_scale_apply(M, K, N, (const double*)A, lda, (const double*)B, ldb,
                                        (const double*)dA, (const double*)d, (const double*)dB,
                                        (double*)A_out, lda_out, (double*)B_out, ldb_out,
                                        (cudaStream_t)stream), "fmm_scale_apply");
}

fmm_status fmm_unscale(int dtype, int64_t M, int64_t N, void* C, int64_t ldc, const void* dA,
                       const void* dB, void* stream) {
  if (dtype != FMM_F64) { set_error("scaling: FP64 only"); return FMM_E_UNSUPPORTED; }
  if (!C || !dA || !dB || ldc < N) { set_error("fmm_unscale: bad argument"); return FMM_E_ARG; }
  return cuda_status(launch_unscale((double*)C, ldc, M, N, (const double*)dA, (const double*)dB,
                                    (cudaStream_t)stream), "fmm_unscale");
}

// ---- stability analysis (Sec. 4) -----------------------------------

fmm_status fmm_rule_quantities(const fmm_rule* r, int64_t* nnz, double* Q, double* E, double* q,
                               double* e) {
  if (!r) { set_error("fmm_rule_quantities: null rule"); return FMM_E_ARG; }
  RuleQuantities x = rule_quantities(r->d);
  if (nnz) *nnz = x.nnz;
  if (Q) *Q = x.Q;
  if (E) *E = x.E;
  if (q) std::copy(x.q.begin(), x.q.end(), q);
  if (e) std::copy(x.e.begin(), x.e.end(), e);
  return FMM_OK;
}

namespace {
// xi_k over the flattened k = (k_l, ..., k_L) of the subtree rooted at node idx of level l
// (simplified form): sum_r |w_{k_l r}| a_r b_r * child_r[rest]
std::vector<double> xi_vec(const fmm_plan* p, int l, int64_t idx) {
  const RuleData& ru = p->rules[p->node_rule[l][idx]];
  const RuleQuantities q = rule_quantities(ru);
  const double den = (double)(1 << ru.log2den);
  const int nw = ru.m0 * ru.n0;
  if (l == p->L - 1) {
    std::vector<double> v(nw, 0.0);
    for (int k = 0; k < nw; ++k)
      for (int r = 0; r < ru.R; ++r) v[k] += std::fabs(ru.W[(size_t)k * ru.R + r] / den) * q.a[r] * q.b[r];
    return v;
  }
  std::vector<double> out;
  std::vector<std::vector<double>> child(ru.R);
  for (int r = 0; r < ru.R; ++r) child[r] = xi_vec(p, l + 1, idx * ru.R + r);
  const size_t rest = child[0].size();
  out.assign((size_t)nw * rest, 0.0);
  for (int k = 0; k < nw; ++k)
    for (int r = 0; r < ru.R; ++r) {
      const double c = std::fabs(ru.W[(size_t)k * ru.R + r] / den) * q.a[r] * q.b[r];
      if (c == 0) continue;
      for (size_t t = 0; t < rest; ++t) out[(size_t)k * rest + t] += c * child[r][t];
    }
  return out;
}

// delta^{[l, r_1..r_{l-1}]}_k over the flattened k = (k_l, ..., k_L); chi carries
// sum of alpha + beta along the path from the root (the S_r / T_r additions at the leaves).
std::vector<double> delta_vec(const fmm_plan* p, int l, int64_t idx, double chi) {
  const RuleData& ru = p->rules[p->node_rule[l][idx]];
  const RuleQuantities q = rule_quantities(ru);
  const int nw = ru.m0 * ru.n0;
  if (l == p->L - 1) {
    std::vector<double> v(nw, 0.0);
    for (int k = 0; k < nw; ++k) {
      double mx = 0;
      for (int r = 0; r < ru.R; ++r)
        if (ru.W[(size_t)k * ru.R + r] != 0) mx = std::max(mx, chi + q.alpha[r] + q.beta[r]);
      v[k] = q.gamma[k] + mx;
    }
    return v;
  }
  std::vector<std::vector<double>> child(ru.R);
  for (int r = 0; r < ru.R; ++r) child[r] = delta_vec(p, l + 1, idx * ru.R + r, chi + q.alpha[r] + q.beta[r]);
  const size_t rest = child[0].size();
  std::vector<double> out((size_t)nw * rest, 0.0);
  for (int k = 0; k < nw; ++k)
    for (size_t t = 0; t < rest; ++t) {
      double mx = 0;
      for (int r = 0; r < ru.R; ++r)
        if (ru.W[(size_t)k * ru.R + r] != 0) mx = std::max(mx, child[r][t]);
      out[(size_t)k * rest + t] = q.gamma[k] + mx;
    }
  return out;
}
}  // namespace

fmm_status fmm_plan_stability(const fmm_plan* p, double* xi, double* delta, double* uniform_bound) {
  if (!p) { set_error("fmm_plan_stability: null plan"); return FMM_E_ARG; }
  const double kl = (double)p->lk[p->L];  // K / prod K0 (padded K)
  double x = 1.0, d = kl * 1.0;
  if (p->L > 0) {
    std::vector<double> xv = xi_vec(p, 0, 0);
    x = *std::max_element(xv.begin(), xv.end());
    std::vector<double> dv = delta_vec(p, 0, 0, 0.0);
    d = kl + *std::max_element(dv.begin(), dv.end());
  }
  if (xi) *xi = x;
  if (delta) *delta = d;
  if (uniform_bound) {  // Thm non_stationary_analysis, uniform plans only
    bool uniform = true;
    double sq = 0, pe = 1;
    for (int l = 0; l < p->L; ++l) {
      for (int r : p->node_rule[l]) uniform = uniform && r == p->node_rule[l][0];
      const RuleQuantities q = rule_quantities(p->rules[p->node_rule[l][0]]);
      sq += q.Q;
      pe *= q.E;
    }
    *uniform_bound = uniform ? (kl + sq) * kl * pe : std::nan("");
  }
  return FMM_OK;
}

fmm_status fmm_choose_variants(const fmm_rule* root, const fmm_rule* const* variants, int n_variants,
                               int32_t* choice, double* xi_out) {
  if (!root || !variants || n_variants < 1 || !choice) { set_error("fmm_choose_variants: bad args"); return FMM_E_ARG; }
  const RuleData& rr = root->d;
  for (int v = 0; v < n_variants; ++v) {
    const RuleData& vd = variants[v]->d;
    if (vd.m0 != rr.m0 || vd.k0 != rr.k0 || vd.n0 != rr.n0 || vd.R != rr.R) {
      set_error("fmm_choose_variants: variants must share the root's (m0,k0,n0,R) (P:146)");
      return FMM_E_ARG;
    }
  }
  // two-level xi_k = sum_{r1} c_{k1 r1} e^{[2, r1]}_{k2}, c = |w| a b of the root
  const RuleQuantities qr = rule_quantities(rr);
  const double den = (double)(1 << rr.log2den);
  const int nw = rr.m0 * rr.n0, R = rr.R;
  std::vector<std::vector<double>> ev(n_variants);
  for (int v = 0; v < n_variants; ++v) ev[v] = rule_quantities(variants[v]->d).e;
  std::vector<double> c((size_t)nw * R);
  for (int k = 0; k < nw; ++k)
    for (int r = 0; r < R; ++r) c[(size_t)k * R + r] = std::fabs(rr.W[(size_t)k * R + r] / den) * qr.a[r] * qr.b[r];
  auto xi_of = [&](const std::vector<int>& ch) {
    double best = 0;
    for (int k1 = 0; k1 < nw; ++k1)
      for (int k2 = 0; k2 < nw; ++k2) {
        double s = 0;
        for (int r = 0; r < R; ++r) s += c[(size_t)k1 * R + r] * ev[ch[r]][k2];
        best = std::max(best, s);
      }
    return best;
  };
  std::vector<int> ch(R, 0), best_ch(R, 0);
  double best = xi_of(ch);
  double combos = std::pow((double)n_variants, (double)R);
  if (combos <= (double)(1 << 24)) {  // exhaustive, lexicographic (first minimum wins)
    for (int64_t id = 1; id < (int64_t)combos; ++id) {
      int64_t x = id;
      for (int r = R - 1; r >= 0; --r) { ch[r] = (int)(x % n_variants); x /= n_variants; }
      const double v = xi_of(ch);
      if (v < best) { best = v; best_ch = ch; }
    }
  } else {  // coordinate descent from all-variant-0 until no single change improves
    bool improved = true;
    ch = best_ch;
    while (improved) {
      improved = false;
      for (int r = 0; r < R; ++r)
        for (int v = 0; v < n_variants; ++v) {
          std::vector<int> t = ch;
          t[r] = v;
          const double x = xi_of(t);
          if (x < best) { best = x; ch = t; improved = true; }
        }
    }
    best_ch = ch;
  }
  for (int r = 0; r < R; ++r) choice[r] = best_ch[r];
  if (xi_out) *xi_out = best;
  return FMM_OK;
}

// ---- NCCL ----------------------------------------------------------------------------------------

fmm_status fmm_comm_unique_id(void* out128) {
  if (!out128) { set_error("fmm_comm_unique_id: null"); return FMM_E_ARG; }
  NcclApi* api = nccl();
  if (!api) { set_error("NCCL library not loadable (set FMM_NCCL_LIB)"); return FMM_E_NCCL; }
  ncclUniqueId id;
  ncclResult_t r = api->getUniqueId(&id);
  if (r != 0) { set_error("ncclGetUniqueId failed"); return FMM_E_NCCL; }
  std::memcpy(out128, &id, sizeof id);
  return FMM_OK;
}

fmm_status fmm_plan_set_comm(fmm_plan* p, const void* id128, int rank, int nranks) {
  if (!p || !id128 || nranks < 1 || rank < 0 || rank >= nranks) { set_error("fmm_plan_set_comm: bad args"); return FMM_E_ARG; }
  NcclApi* api = nccl();
  if (!api) { set_error("NCCL library not loadable (set FMM_NCCL_LIB)"); return FMM_E_NCCL; }
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  ncclComm_t c = nullptr;
  ncclResult_t r = api->commInitRank(&c, nranks, id, rank);
  if (r != 0) { set_error(std::string("ncclCommInitRank: ") + (api->getErrorString ? api->getErrorString(r) : "?")); return FMM_E_NCCL; }
  if (p->comm && api->commDestroy) api->commDestroy(p->comm);
  p->comm = c;
  p->rank = rank;
  p->nranks = nranks;
  return compile_plan(p);
}

}  // extern "C"
