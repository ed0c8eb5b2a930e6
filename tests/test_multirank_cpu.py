"""Multi-rank host logic on CPU (gloo, world size 2): the library's top-level partition
(fmm_plan_owned) assigns every top-level product to exactly one rank, and the
per-rank partial sums C^(p) = sum_{owned r} w_kr M_r (computed here with oracle building blocks)
summed across ranks by a collective equal the full product within the parity tolerance."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import fmm_inputs as fi


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _partial_oracle(rank, nranks, owned, A, B):
    import oracle
    from oracle import rules as R
    w = R.winograd()
    S, T = oracle.node_st(w, A, B)
    sub = R.Plan.stationary(w, 1)
    mb, nb = A.shape[0] // 2, B.shape[1] // 2
    Wf = w.as_float()[2]
    C = np.zeros((A.shape[0], B.shape[1]))
    started = [False] * 4
    for r in owned:
        Mr = oracle.fmm(S[r], T[r], sub)
        for k in range(4):
            if Wf[k, r] == 0:
                continue
            ia, jb = divmod(k, 2)
            blk = C[ia * mb:(ia + 1) * mb, jb * nb:(jb + 1) * nb]
            blk[...] = Wf[k, r] * Mr if not started[k] else blk + Wf[k, r] * Mr
            started[k] = True
    return C


def _combine(rule, blocks_by_r, mb, nb):
    """C = sum_r w_kr M_r over the given {r: M_r} in ascending r (oracle-side arithmetic)."""
    Wf = rule.as_float()[2]
    C = np.zeros((2 * mb, 2 * nb))
    started = [False] * 4
    for r in sorted(blocks_by_r):
        for k in range(4):
            if Wf[k, r] == 0:
                continue
            ia, jb = divmod(k, 2)
            blk = C[ia * mb:(ia + 1) * mb, jb * nb:(jb + 1) * nb]
            blk[...] = Wf[k, r] * blocks_by_r[r] if not started[k] else blk + Wf[k, r] * blocks_by_r[r]
            started[k] = True
    return C


def _partial_oracle_depth2(owned_units, A, B):
    """Partial C of a rank owning the depth-2 units u = 7 r1 + r2 of a 2-level S-W plan."""
    import oracle
    from oracle import rules as R
    w = R.winograd()
    leaf = R.Plan([])
    S1, T1 = oracle.node_st(w, A, B)
    m1 = {}
    for r1 in range(7):
        mine = [u % 7 for u in owned_units if u // 7 == r1]
        if not mine:
            continue
        S2, T2 = oracle.node_st(w, S1[r1], T1[r1])
        m2 = {r2: oracle.fmm(S2[r2], T2[r2], leaf) for r2 in mine}
        m1[r1] = _combine(w, m2, A.shape[0] // 4, B.shape[1] // 4)
    return _combine(w, m1, A.shape[0] // 2, B.shape[1] // 2)


def _worker_depth2(rank, world, port, out_q, order="cyclic"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1507_00687_b200 as fb
    w = fb.Rule.builtin("winograd")
    plan = fb.Plan([w, w], 128, 128, 128)
    plan.set_shard_depth(2)
    plan.set_shard_order(order)
    owned = plan.owned(rank, world)
    A, B = fi.random_pair(128, 128, 128, seed=22)
    part = torch.from_numpy(_partial_oracle_depth2(owned, A, B))
    dist.all_reduce(part)
    counts = torch.zeros(49, dtype=torch.int64)
    counts[owned] = 1
    dist.all_reduce(counts)
    if rank == 0:
        out_q.put((part.numpy(), counts.numpy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("order", ["cyclic", "block"])
def test_two_rank_depth2_units_and_reduce(order):
    # finer sharding (fmm_plan_set_shard_depth(2)): 49 units, every one owned once (round-robin
    # or in contiguous blocks); the ranks' partial sums reduced by a collective equal the full
    # product within the parity tolerance
    import oracle
    from oracle import rules as R
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_depth2, args=(r, 2, port, q, order)) for r in range(2)]
    for p in procs:
        p.start()
    total, counts = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert counts.tolist() == [1] * 49
    A, B = fi.random_pair(128, 128, 128, seed=22)
    full = oracle.fmm(A, B, R.Plan.stationary(R.winograd(), 2))
    assert oracle.parity_metric(total, full, np.abs(A).max(), np.abs(B).max(), 128) <= 1e-13


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1507_00687_b200 as fb
    w = fb.Rule.builtin("winograd")
    plan = fb.Plan([w, w], 128, 128, 128)
    owned = plan.owned(rank, world)
    A, B = fi.random_pair(128, 128, 128, seed=21)
    part = torch.from_numpy(_partial_oracle(rank, world, owned, A, B))
    dist.all_reduce(part)  # the exchange step (NCCL reduce on GPUs)
    counts = torch.zeros(7, dtype=torch.int64)
    counts[owned] = 1
    dist.all_reduce(counts)
    if rank == 0:
        out_q.put((part.numpy(), counts.numpy(), owned))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_partition_and_reduce(world):
    import oracle
    from oracle import rules as R
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    total, counts, owned0 = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert counts.tolist() == [1] * 7  # every top-level product exactly once
    assert owned0 == [0, 2, 4, 6]
    A, B = fi.random_pair(128, 128, 128, seed=21)
    full = oracle.fmm(A, B, R.Plan.stationary(R.winograd(), 2))
    assert oracle.parity_metric(total, full, np.abs(A).max(), np.abs(B).max(), 128) <= 1e-13


def _worker_rs(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1507_00687_b200 as fb
    w = fb.Rule.builtin("winograd")
    plan = fb.Plan([w, w], 128, 128, 128)
    plan.set_comm_mode("reduce_scatter")  # host-only setting; the exchange below mirrors it
    owned = plan.owned(rank, world)
    A, B = fi.random_pair(128, 128, 128, seed=21)
    part = torch.from_numpy(_partial_oracle(rank, world, owned, A, B))
    rows = 128 // world
    mine = torch.empty((rows, 128), dtype=part.dtype)
    dist.reduce_scatter_tensor(mine, part)  # rank r receives rows [r M/P, (r+1) M/P)
    out_q.put((rank, mine.numpy()))
    dist.destroy_process_group()


def test_two_rank_reduce_scatter_rows():
    # comm mode 2 (fmm_plan_set_comm_mode): the ranks' partials reduce-scattered by rows give
    # the product's row blocks (within the parity tolerance of the full oracle product)
    import oracle
    from oracle import rules as R
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_rs, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A, B = fi.random_pair(128, 128, 128, seed=21)
    full = oracle.fmm(A, B, R.Plan.stationary(R.winograd(), 2))
    C = np.vstack([got[0], got[1]])
    assert oracle.parity_metric(C, full, np.abs(A).max(), np.abs(B).max(), 128) <= 1e-13


@pytest.mark.parametrize("depth,nranks", [(1, 2), (2, 3), (2, 8), (3, 4), (3, 8), (3, 7)])
def test_block_unit_order(depth, nranks):
    # fmm_plan_set_shard_order(1): rank p owns the contiguous units
    # [ceil(p U / P), ceil((p + 1) U / P)) -- every unit exactly once, block sizes within one
    import paper_1507_00687_b200 as fb
    w = fb.Rule.builtin("winograd")
    plan = fb.Plan([w, w, w], 64, 64, 64)
    plan.set_shard_depth(depth)
    plan.set_shard_order("block")
    U = 7 ** depth
    seen = []
    for p in range(nranks):
        own = plan.owned(p, nranks)
        lo, hi = -(-p * U // nranks), -(-(p + 1) * U // nranks)
        assert own == list(range(lo, hi))
        seen += own
    assert seen == list(range(U))
    sizes = [len(plan.owned(p, nranks)) for p in range(nranks)]
    assert max(sizes) - min(sizes) <= 1
    with pytest.raises(fb.fmm.FmmError):  # the fused NVLink combine lays buffers out round-robin
        plan.set_comm_mode("p2p")
