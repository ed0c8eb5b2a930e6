"""The multi-GPU exchange, executed on the one GPU a test box has (
the coupling C_k = sum_r w_kr M_r of Eq. eqn:recursive_alg).

* A one-rank NCCL communicator really issues each collective of comm modes 0-2 (ncclReduce,
  ncclAllReduce, in-place ncclReduceScatter) and mode 3's two 1-word ncclAllReduce barriers
  through the dlopen'ed NCCL: the result is bitwise the no-communicator run (a sum over one
  rank), and the call fails loudly if a mirrored ABI type or enum were wrong.
* Two processes sharing the GPU run comm mode 3 end to end over CUDA IPC: symmetric buffers
  (fmm_plan_sym_alloc), handles exchanged through torch.distributed (gloo), opened with
  fmm_plan_set_peer_handles, the fused combine reading the other process's products, with the
  barrier injected (fmm_plan_set_barrier: stream synchronise + gloo barrier).  Each rank's rows
  are bitwise the single-GPU rows and within the parity tolerance of the oracle.
* Sharded partial sums (shard depth 1-3, 2 / 4 / 8 virtual ranks) against partial sums the
  oracle computes from its own building blocks (node_st, fmm, node_c with the unowned products
  zero): within the parity tolerance, and bitwise when the leaf inner dimension is 1."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import fmm_inputs as fi
import oracle
from oracle import rules as R
from oracle.rules import Plan as OPlan

pytestmark = pytest.mark.gpu

TOL64, TOL32 = 1e-13, 5e-5


@pytest.fixture(scope="module")
def fb():
    import paper_1507_00687_b200 as fb
    assert torch.cuda.is_available()
    return fb


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def exe(p, A, B):
    C = p.execute(dev(A), dev(B))
    torch.cuda.synchronize()
    return C.cpu().numpy()


def parity(Cg, Co, A, B):
    return oracle.parity_metric(Cg, Co, np.abs(A).max(), np.abs(B).max(), A.shape[1])


# ---- one-rank NCCL communicator ----------------------------------------------------------------

@pytest.mark.parametrize("mode", ["reduce", "allreduce", "reduce_scatter", "p2p"])
@pytest.mark.parametrize("names,dtype", [(("winograd",) * 2, "f64"), (("strassen",) * 3, "f64"),
                                         (("winograd",) * 2, "f32")])
def test_one_rank_communicator_issues_collectives(fb, mode, names, dtype):
    M, K, N = 512, 384, 256
    npdt = np.float64 if dtype == "f64" else np.float32
    A, B = fi.random_pair(M, K, N, seed=77, dtype=npdt)
    rules = [fb.Rule.builtin(n) for n in names]
    leaf = fb.fmm.LEAF_NATIVE if dtype == "f64" else fb.fmm.LEAF_3XTF32
    ref = exe(fb.Plan(rules, M, K, N, dtype=dtype, leaf=leaf), A, B)
    p = fb.Plan(rules, M, K, N, dtype=dtype, leaf=leaf)
    p.set_comm(fb.comm_unique_id(), 0, 1)
    if mode != "reduce":
        p.set_comm_mode(mode)
    if mode == "p2p":
        p.set_peer_handles([p.sym_alloc()])
        # the products of all 7 top-level r live in this rank's symmetric buffer
        assert p.sym_bytes() == 7 * (M // 2) * (N // 2) * A.itemsize + 256
    for _ in range(2):  # repeated calls reuse the communicator and the barrier words
        C = exe(p, A, B)
        assert np.array_equal(C, ref)
    Co = oracle.fmm(A, B, OPlan.uniform([R.builtin(n) for n in names]))
    assert parity(C, Co, A, B) <= (TOL64 if dtype == "f64" else TOL32)


def test_one_rank_communicator_scaled_and_padded(fb):
    # the reduce after the unscale / crop steps of a scaled, padded plan
    A, B = fi.draw("skew", 250, 130, 66, 3)
    w = fb.Rule.builtin("winograd")
    sc = {"mode": "repeated", "pow2": 1}
    ref = exe(fb.Plan([w, w], 250, 130, 66, scaling=sc), A, B)
    p = fb.Plan([w, w], 250, 130, 66, scaling=sc)
    p.set_comm(fb.comm_unique_id(), 0, 1)
    assert np.array_equal(exe(p, A, B), ref)


@pytest.mark.parametrize("mode", ["outside", "repeated"])
@pytest.mark.parametrize("nranks,depth,order", [(2, 1, "cyclic"), (3, 2, "block"), (4, 3, "block")])
def test_scaled_partitions_sum_to_scaled_product(fb, mode, nranks, depth, order):
    # multi-GPU partitions of a scaled plan: every rank runs the scaling (Alg. 1 / 3)
    # on the whole A, B, forms its units from the scaled operands and unscales its partial
    # (C = D_A C' D_B is linear in C'), so the partials sum to the one-rank scaled product --
    # within the rounding of the different summation order (componentwise: the C4 magnitudes
    # make the normalised metric vacuous)
    A, B = fi.draw("skew", 256, 256, 256, 3)
    w = fb.Rule.builtin("winograd")
    sc = {"mode": mode, "pow2": 1}
    ref = exe(fb.Plan([w, w, w], 256, 256, 256, scaling=sc), A, B)
    tot = np.zeros_like(ref)
    for rank in range(nranks):
        p = fb.Plan([w, w, w], 256, 256, 256, scaling=sc)
        p.set_shard_depth(depth)
        p.set_shard_order(order)
        p.set_partition(rank, nranks)
        tot += exe(p, A, B)
    absab = np.abs(A) @ np.abs(B)
    assert np.all(np.abs(tot - ref) <= 1e-12 * absab + 1e-300)


# ---- two processes on one GPU: comm mode 3 over CUDA IPC ------------------------------------------

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, world, port, names, dims, dtype, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_1507_00687_b200 as fb
        M, K, N = dims
        npdt = np.float64 if dtype == "f64" else np.float32
        A, B = fi.random_pair(M, K, N, seed=91, dtype=npdt)
        leaf = fb.fmm.LEAF_NATIVE if dtype == "f64" else fb.fmm.LEAF_3XTF32
        p = fb.Plan([fb.Rule.builtin(n) for n in names], M, K, N, dtype=dtype, leaf=leaf)
        p.set_partition(rank, world)
        p.set_comm_mode("p2p")

        def barrier(_stream):
            torch.cuda.synchronize()
            dist.barrier()

        p.set_barrier(barrier)
        handles = [None] * world
        dist.all_gather_object(handles, p.sym_alloc())
        p.set_peer_handles(handles)
        r0, r1 = M * rank // world, M * (rank + 1) // world
        outs = []
        for _ in range(2):  # twice: the second call overwrites the products after the barrier
            C = p.execute(dev(A), dev(B))
            torch.cuda.synchronize()
            outs.append(C[r0:r1].cpu().numpy())
        out_q.put((rank, outs[0], outs[1]))
        dist.barrier()  # peers' mappings stay valid until everyone has read
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,names,dtype", [(2, ("winograd",) * 2, "f64"),
                                               (2, ("strassen",) * 3, "f64"),
                                               (3, ("winograd",) * 2, "f64"),
                                               (2, ("winograd",) * 2, "f32")])
def test_p2p_mode_two_processes_ipc(fb, world, names, dtype):
    M, K, N = 2 ** len(names) * 60, 2 ** len(names) * 40, 2 ** len(names) * 36
    npdt = np.float64 if dtype == "f64" else np.float32
    A, B = fi.random_pair(M, K, N, seed=91, dtype=npdt)
    leaf = fb.fmm.LEAF_NATIVE if dtype == "f64" else fb.fmm.LEAF_3XTF32
    ref = exe(fb.Plan([fb.Rule.builtin(n) for n in names], M, K, N, dtype=dtype, leaf=leaf), A, B)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, names, (M, K, N), dtype, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    got = {}
    for _ in range(world):
        rank, c1, c2 = q.get(timeout=600)
        got[rank] = (c1, c2)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    Co = oracle.fmm(A, B, OPlan.uniform([R.builtin(n) for n in names]))
    for rank in range(world):
        r0, r1 = M * rank // world, M * (rank + 1) // world
        for c in got[rank]:
            assert np.array_equal(c, ref[r0:r1])  # bitwise the single-GPU rows (ascending r)
            assert parity(c, Co[r0:r1], A, B) <= (TOL64 if dtype == "f64" else TOL32)


# ---- sharded partial sums against oracle partials -------------------------------------------------

def oracle_partial(rules, A, B, depth, owned):
    """The partial C of a rank owning the depth-`depth` units `owned` (paths (r_1..r_d) in BFS
    order, u = r_1 R^{d-1} + ... + r_d): at every level the oracle's S / T formation
    (node_st), the owned subtrees' products by the oracle executor (fmm), and the oracle's
    W-combination (node_c, r ascending) with the products of unowned subtrees set to zero --
    0 + x = x, so the first owned contribution initialises C_k as on the GPU."""
    owned = set(owned)

    def rec(l, X, Y, prefix):
        rule = rules[l]
        S, T = oracle.node_st(rule, X, Y)
        mb, nb = X.shape[0] // rule.m0, Y.shape[1] // rule.n0
        Ms = np.zeros((rule.R, mb, nb), X.dtype)
        hit = False
        for r in range(rule.R):
            u = prefix * rule.R + r
            if l + 1 == depth:
                if u in owned:
                    Ms[r] = oracle.fmm(S[r], T[r], OPlan.uniform(rules[l + 1:]))
                    hit = True
            else:
                sub = rec(l + 1, S[r], T[r], u)
                if sub is not None:
                    Ms[r] = sub
                    hit = True
        return oracle.node_c(rule, Ms) if hit else None

    C = rec(0, A, B, 0)
    return np.zeros((A.shape[0], B.shape[1]), A.dtype) if C is None else C


@pytest.mark.parametrize("depth,nranks,order", [(1, 2, "cyclic"), (1, 4, "cyclic"), (2, 2, "cyclic"),
                                               (2, 4, "cyclic"), (2, 8, "cyclic"), (3, 8, "cyclic"),
                                               (2, 2, "block"), (3, 4, "block"), (3, 8, "block")])
@pytest.mark.parametrize("K", [8, 256])  # K = 8: leaf inner dimension 1 (bitwise)
def test_shard_partials_match_oracle_partials(fb, depth, nranks, order, K):
    M, N = 256, 192
    A, B = fi.random_pair(M, K, N, seed=40 + depth)
    names = ("winograd",) * 3
    orules = [R.builtin(n) for n in names]
    for rank in range(nranks):
        p = fb.Plan([fb.Rule.builtin(n) for n in names], M, K, N)
        p.set_shard_depth(depth)
        p.set_shard_order(order)
        p.set_partition(rank, nranks)
        owned = p.owned(rank, nranks)
        part = exe(p, A, B)
        Co = oracle_partial(orules, A, B, depth, owned)
        if K == 8:
            assert np.array_equal(part, Co)
        else:
            assert parity(part, Co, A, B) <= TOL64


def test_rank_without_products_returns_zero_host_path(fb):
    # R = 7 products over 8 ranks: rank 7 owns nothing; fmm_execute_host must return the zero
    # partial, not the full product of a single-rank twin (round-1 advisor finding)
    M = K = N = 256
    A, B = fi.random_pair(M, K, N, seed=5)
    w = fb.Rule.builtin("winograd")
    p = fb.Plan([w, w], M, K, N)
    p.set_partition(7, 8)
    Ah, Bh = torch.from_numpy(A).pin_memory(), torch.from_numpy(B).pin_memory()
    Ch = torch.full((M, N), float("nan"), dtype=torch.float64).pin_memory()
    Ad, Bd = dev(A), dev(B)
    Cd = torch.empty((M, N), dtype=torch.float64, device="cuda")
    p.execute_host(Ah, Bh, Ch, Ad, Bd, Cd)
    torch.cuda.synchronize()
    assert np.all(Ch.numpy() == 0)
    # and a plan reconfigured after its host path ran recompiles its twin (no stale schedule)
    q = fb.Plan([w, w], M, K, N)
    q.set_schedule("breadth")
    q.execute_host(Ah, Bh, Ch, Ad, Bd, Cd)
    torch.cuda.synchronize()
    full = Ch.numpy().copy()
    q.set_partition(0, 2)
    q.execute_host(Ah, Bh, Ch, Ad, Bd, Cd)
    torch.cuda.synchronize()
    assert np.array_equal(Ch.numpy(), exe(q, A, B))
    assert not np.array_equal(Ch.numpy(), full)
