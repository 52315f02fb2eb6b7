"""SURVEY.md §4 'virtual ranks' for every sharded evaluator (§8e): each
shard's slab is computed on one GPU by the sharded code path of
paper_2510_17505_b200.distributed, the slabs are assembled, and the result
must equal the unsharded evaluator bit for bit for world = 1, 2, 3, 4, 8
(every output row has exactly one owner and keeps its summation order).
The multi-process collective itself is covered by tests/test_distributed.py
(gloo, world 2/3)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

WORLDS = [1, 2, 3, 4, 8]


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_17505_b200 as P
    P.lib()
    return P


def bf16_dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(torch.bfloat16).cuda()


@pytest.mark.parametrize("kind", ["int", "real"])
@pytest.mark.parametrize("world", WORLDS)
def test_blockgroupcoo_block_row_shards(P, ixo, world, kind):
    """K4 balances slots across CTAs, so a block-row that crosses a CTA
    boundary is summed from per-CTA partials in a fixed order: bit-identical
    for a given launch, and across shard counts to fp32 rounding (exactly
    for integer-valued data)."""
    from paper_2510_17505_b200.distributed import shard_plan, spmm_blockgroupcoo_slab
    rng = ixo.Rng(31)
    k = ixo.INT if kind == "int" else ixo.REAL
    a = ixo.synth_block_sparse_matrix(rng, 16 * 90, 16 * 70, 16, 16, 0.15, k)
    b = ixo.synth_dense(rng, (70, 16, 256), k)
    fmt = P.dense_to_blockgroupcoo(bf16_dev(a), 16, 16, 0)
    B = bf16_dev(b)
    full = torch.zeros((90, 16, 256), device="cuda")
    P.spmm_blockgroupcoo(fmt.AM, fmt.AK, fmt.AV, B, full, flags=2)
    again = torch.zeros_like(full)
    P.spmm_blockgroupcoo(fmt.AM, fmt.AK, fmt.AV, B, again, flags=2)
    assert torch.equal(again, full)  # run-to-run deterministic
    shards = shard_plan(fmt.AM.cpu().numpy(), 90, world)
    assert shards[0].r0 == 0 and shards[-1].r1 == 90
    out = torch.full_like(full, float("nan"))
    for s in shards:
        out[s.r0:s.r1] = spmm_blockgroupcoo_slab(fmt, B, s)
    if kind == "int":
        assert torch.equal(out, full)
    else:
        torch.testing.assert_close(out, full, rtol=1e-6, atol=1e-5)


@pytest.mark.parametrize("world", WORLDS)
def test_conv_point_block_shards_bit_identical(P, world):
    from paper_2510_17505_b200.distributed import conv_shard_plan, point_blocks
    g = np.random.default_rng(5)
    pts = np.unique(g.integers(0, 24, (6000, 3)), axis=0).astype(np.int32)
    n = len(pts)
    mo, mi, mz = P.kernel_map(torch.from_numpy(pts).cuda())
    ones = torch.ones(mo.numel(), device="cuda")
    gt = P.group_coo_tensor([n, n, 27], [mo, mi, mz], ones, 2, 16, canonical=True)
    In = bf16_dev(g.standard_normal((n, 64)))
    W = bf16_dev(g.standard_normal((27, 64, 64)) * 0.1)
    full = torch.zeros((n, 64), device="cuda")
    P.ConvPlan(gt.group_coord, gt.member_coords[0], gt.member_coords[1], gt.values, n, 27,
               n).run(In, W, full, accumulate=False)
    out = torch.full_like(full, float("nan"))
    for s in point_blocks(n, world):
        plan = conv_shard_plan(mo, mi, mz, n, s, 16)
        local = torch.empty((s.r1 - s.r0, 64), device="cuda")
        plan.run(In, W, local, accumulate=False)
        out[s.r0:s.r1] = local
    assert torch.equal(out, full)


@pytest.mark.parametrize("world", WORLDS)
def test_tp_edge_shards_bit_identical(P, ixo, world):
    from paper_2510_17505_b200.distributed import edge_blocks
    t = ixo.cg_table(3)
    coords = [torch.from_numpy(np.ascontiguousarray(c, np.int32)).cuda()
              for c in (t["i"], t["j"], t["k"], t["l"])]
    nl = len(t["paths"])
    gt = P.group_coo_tensor([16, 16, 16, nl], coords,
                            torch.from_numpy(t["v"].astype(np.float32)).cuda(), 3, 4)
    plan = P.TpPlan(gt.group_coord, gt.member_coords[0], gt.member_coords[1],
                    gt.member_coords[2], gt.values, 16, 16, 16, nl)
    g = np.random.default_rng(9)
    Bt = 300
    X = bf16_dev(g.standard_normal((Bt, 16, 64)))
    Y = bf16_dev(g.standard_normal((Bt, 16)))
    W = bf16_dev(g.standard_normal((nl, 64, 64)) * 0.1)
    full = torch.zeros((Bt, 16, 64), device="cuda")
    plan.run(X, Y, W, full, accumulate=False)
    out = torch.full_like(full, float("nan"))
    for s in edge_blocks(Bt, world):
        if s.r1 > s.r0:
            local = torch.empty((s.r1 - s.r0, 16, 64), device="cuda")
            plan.run(X[s.r0:s.r1], Y[s.r0:s.r1], W, local, accumulate=False)
            out[s.r0:s.r1] = local
    assert torch.equal(out, full)


def _two_rank_worker(rank, world, port, q):
    import os
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [os.path.dirname(here), here]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2510_17505_b200 as P
        from paper_2510_17505_b200 import distributed as D
        from oracle import ixo
        torch.cuda.set_device(0)
        res = {}
        # GroupCOO row shards through SlabGather
        rng = ixo.Rng(41)
        a = ixo.synth_sparse_matrix(rng, 2500, 1800, 0.01)
        b = ixo.synth_dense(rng, (1800, 64))
        fmt = P.dense_to_groupcoo(torch.from_numpy(a.astype(np.float32)).cuda(), g=0)
        B = torch.from_numpy(b.astype(np.float32)).cuda()
        sh = D.shard_plan(fmt.AM.cpu().numpy(), 2500, world)
        s = sh[rank]
        sg = D.SlabGather(sh, rank, (64,), torch.float32, "cuda")
        sg.local.zero_()
        D.spmm_groupcoo_into(fmt.AM[s.g0:s.g1], fmt.AK[s.g0:s.g1], fmt.AV[s.g0:s.g1],
                             fmt.group_size, B, s, sg.local)
        res["groupcoo"] = sg().cpu().numpy()
        # BlockGroupCOO block-row shards
        a = ixo.synth_block_sparse_matrix(rng, 16 * 40, 16 * 30, 16, 16, 0.2)
        b = ixo.synth_dense(rng, (30, 16, 128))
        f16 = P.dense_to_blockgroupcoo(bf16_dev(a), 16, 16, 0)
        B16 = bf16_dev(b)
        res["bgcoo"] = D.sharded_spmm_blockgroupcoo(
            f16, B16, D.shard_plan(f16.AM.cpu().numpy(), 40, world), rank).cpu().numpy()
        # conv point blocks
        g = np.random.default_rng(2)
        pts = np.unique(g.integers(0, 14, (2000, 3)), axis=0).astype(np.int32)
        n = len(pts)
        mo, mi, mz = P.kernel_map(torch.from_numpy(pts).cuda())
        In, W = bf16_dev(g.standard_normal((n, 64))), bf16_dev(g.standard_normal((27, 64, 64)))
        blocks = D.point_blocks(n, world)
        plan = D.conv_shard_plan(mo, mi, mz, n, blocks[rank], 16)
        res["conv"] = D.sharded_conv(plan, In, W, blocks, rank).cpu().numpy()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_two_processes_share_gpu_sharded_gather(P, ixo):
    """Two real ranks (gloo, both on cuda:0) run the sharded evaluators and
    gather; every rank's result equals the single-call evaluator bit for bit."""
    import socket

    import torch.multiprocessing as mp
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_two_rank_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = ixo.Rng(41)
    a = ixo.synth_sparse_matrix(rng, 2500, 1800, 0.01)
    b = ixo.synth_dense(rng, (1800, 64))
    fmt = P.dense_to_groupcoo(torch.from_numpy(a.astype(np.float32)).cuda(), g=0)
    full = torch.zeros((2500, 64), device="cuda")
    P.spmm_groupcoo(fmt.AM, fmt.AK, fmt.AV, torch.from_numpy(b.astype(np.float32)).cuda(), full)
    a = ixo.synth_block_sparse_matrix(rng, 16 * 40, 16 * 30, 16, 16, 0.2)
    b = ixo.synth_dense(rng, (30, 16, 128))
    f16 = P.dense_to_blockgroupcoo(bf16_dev(a), 16, 16, 0)
    full16 = torch.zeros((40, 16, 128), device="cuda")
    P.spmm_blockgroupcoo(f16.AM, f16.AK, f16.AV, bf16_dev(b), full16)
    g = np.random.default_rng(2)
    pts = np.unique(g.integers(0, 14, (2000, 3)), axis=0).astype(np.int32)
    n = len(pts)
    mo, mi, mz = P.kernel_map(torch.from_numpy(pts).cuda())
    In, W = bf16_dev(g.standard_normal((n, 64))), bf16_dev(g.standard_normal((27, 64, 64)))
    gt = P.group_coo_tensor([n, n, 27], [mo, mi, mz], torch.ones(mo.numel(), device="cuda"), 2,
                            16, canonical=True)
    conv = torch.zeros((n, 64), device="cuda")
    P.ConvPlan(gt.group_coord, gt.member_coords[0], gt.member_coords[1], gt.values, n, 27,
               n).run(In, W, conv, accumulate=False)
    for rank, res in results:
        np.testing.assert_array_equal(res["groupcoo"], full.cpu().numpy())
        np.testing.assert_array_equal(res["bgcoo"], full16.cpu().numpy())
        np.testing.assert_array_equal(res["conv"], conv.cpu().numpy())


def test_more_ranks_than_rows_empty_shards(P, ixo):
    """world > output rows / voxels / edges: the empty shards build and
    evaluate without error and the assembled outputs still equal one call."""
    from paper_2510_17505_b200.distributed import (conv_shard_plan, edge_blocks, point_blocks,
                                                   shard_plan, spmm_blockgroupcoo_slab,
                                                   spmm_groupcoo_slab)
    world = 8
    rng = ixo.Rng(5)
    a = ixo.synth_sparse_matrix(rng, 3, 40, 0.3)
    b = ixo.synth_dense(rng, (40, 16))
    fmt = P.dense_to_groupcoo(torch.from_numpy(a.astype(np.float32)).cuda(), g=0)
    B = torch.from_numpy(b.astype(np.float32)).cuda()
    full = torch.zeros((3, 16), device="cuda")
    P.spmm_groupcoo(fmt.AM, fmt.AK, fmt.AV, B, full)
    shards = shard_plan(fmt.AM.cpu().numpy(), 3, world)
    assert sum(s.r1 - s.r0 for s in shards) == 3
    out = torch.cat([spmm_groupcoo_slab(fmt, B, s) for s in shards])
    assert torch.equal(out, full)

    a16 = ixo.synth_block_sparse_matrix(rng, 32, 64, 16, 16, 0.5)
    b16 = ixo.synth_dense(rng, (4, 16, 128))
    f16 = P.dense_to_blockgroupcoo(bf16_dev(a16), 16, 16, 0)
    full16 = torch.zeros((2, 16, 128), device="cuda")
    P.spmm_blockgroupcoo(f16.AM, f16.AK, f16.AV, bf16_dev(b16), full16)
    sh16 = shard_plan(f16.AM.cpu().numpy(), 2, world)
    out16 = torch.cat([spmm_blockgroupcoo_slab(f16, bf16_dev(b16), s) for s in sh16])
    assert torch.equal(out16, full16)

    pts = np.array([[0, 0, 0], [0, 0, 1], [5, 5, 5]], np.int32)
    mo, mi, mz = P.kernel_map(torch.from_numpy(pts).cuda())
    g = np.random.default_rng(1)
    In, W = bf16_dev(g.standard_normal((3, 64))), bf16_dev(g.standard_normal((27, 64, 64)))
    gt = P.group_coo_tensor([3, 3, 27], [mo, mi, mz], torch.ones(mo.numel(), device="cuda"), 2, 4,
                            canonical=True)
    fullc = torch.zeros((3, 64), device="cuda")
    P.ConvPlan(gt.group_coord, gt.member_coords[0], gt.member_coords[1], gt.values, 3, 27,
               3).run(In, W, fullc, accumulate=False)
    parts = []
    for s in point_blocks(3, world):
        plan = conv_shard_plan(mo, mi, mz, 3, s, 4)
        local = torch.zeros((s.r1 - s.r0, 64), device="cuda")
        if s.r1 > s.r0:
            plan.run(In, W, local, accumulate=False)
        parts.append(local)
    assert torch.equal(torch.cat(parts), fullc)

    blocks = edge_blocks(5, world)
    assert [s.r1 - s.r0 for s in blocks].count(0) == 3 and blocks[-1].r1 == 5


# ------------------------------------------- native (C-ABI) sharded path
@pytest.mark.parametrize("world", WORLDS)
@pytest.mark.parametrize("nchunks", [1, 3])
def test_native_groupcoo_shards_bit_identical(P, ixo, world, nchunks):
    """ixb_spmm_groupcoo_sharded: each virtual rank writes its chunks straight
    into the full output (no collective); the assembled C equals the
    unsharded K3 bit for bit, empty rows included."""
    from paper_2510_17505_b200 import distributed as D
    rng = ixo.Rng(17)
    a = ixo.synth_sparse_matrix(rng, 700, 300, 0.05)
    a[[0, 5, 6, 699]] = 0  # empty rows at the edges and between shards
    b = ixo.synth_dense(rng, (300, 64))
    fmt = P.dense_to_groupcoo(torch.from_numpy(a.astype(np.float32)).cuda(), g=4)
    B = torch.from_numpy(b.astype(np.float32)).cuda()
    full = torch.empty((700, 64), device="cuda")
    P.spmm_groupcoo(fmt.AM, fmt.AK, fmt.AV, B, full, accumulate=False, flags=2)
    out = torch.full_like(full, float("nan"))
    for r in range(world):
        plan = D.ShardPlan(fmt.AM, 700, world, r, nchunks)
        D.spmm_groupcoo_sharded(plan, fmt, B, out, comm=None, flags=2 | D.SHARD_NO_COMM)
    assert torch.equal(out, full)
    plan = D.ShardPlan(fmt.AM, 700, world, 0, nchunks)
    rows = [plan.chunk(q, c)[2:] for q in range(world) for c in range(nchunks)]
    assert rows[0][0] == 0 and rows[-1][1] == 700
    assert all(x[1] == y[0] for x, y in zip(rows, rows[1:]))  # a partition of the rows


@pytest.mark.parametrize("world", [1, 3, 8])
def test_native_blockgroupcoo_and_conv_shards(P, ixo, world):
    """K4 block-row chunks (exact on integer data) and K6 point-block tile
    chunks (bit-identical) through the native sharded entries."""
    from paper_2510_17505_b200 import distributed as D
    rng = ixo.Rng(23)
    a = ixo.synth_block_sparse_matrix(rng, 16 * 60, 16 * 40, 16, 16, 0.2, ixo.INT)
    b = ixo.synth_dense(rng, (40, 16, 256), ixo.INT)
    fmt = P.dense_to_blockgroupcoo(bf16_dev(a), 16, 16, 0)
    B = bf16_dev(b)
    full = torch.zeros((60, 16, 256), device="cuda")
    P.spmm_blockgroupcoo(fmt.AM, fmt.AK, fmt.AV, B, full, flags=2)
    out = torch.full_like(full, float("nan"))
    for r in range(world):
        plan = D.ShardPlan(fmt.AM, 60, world, r, 2)
        D.spmm_blockgroupcoo_sharded(plan, fmt, B, out, flags=2 | D.SHARD_NO_COMM)
    assert torch.equal(out, full)

    g = np.random.default_rng(5)
    pts = np.unique(g.integers(0, 24, (6000, 3)), axis=0).astype(np.int32)
    n = len(pts)
    mo, mi, mz = P.kernel_map(torch.from_numpy(pts).cuda())
    ones = torch.ones(mo.numel(), device="cuda")
    gt = P.group_coo_tensor([n, n, 27], [mo, mi, mz], ones, 2, 16, canonical=True)
    In = bf16_dev(g.standard_normal((n, 64)))
    W = bf16_dev(g.standard_normal((27, 64, 64)) * 0.1)
    ref = torch.zeros((n, 64), device="cuda")
    P.ConvPlan(gt.group_coord, gt.member_coords[0], gt.member_coords[1], gt.values, n, 27,
               n).run(In, W, ref, accumulate=False)
    out = torch.full_like(ref, float("nan"))
    for r, s in enumerate(D.point_blocks(n, world)):
        local = D.conv_shard_plan(mo, mi, mz, n, s, 16) if s.r1 > s.r0 else None
        D.conv_sharded(local, In, W, out, world, r, nchunks=3, flags=D.SHARD_NO_COMM)
    assert torch.equal(out, ref)


def test_native_sharded_with_nccl_comm(P, ixo):
    """The full native path with a real (1-rank) NCCL communicator: chunk
    evaluation, in-place broadcasts on the side stream, and the join back
    onto the caller's stream — also inside a captured CUDA graph."""
    from paper_2510_17505_b200 import distributed as D
    rng = ixo.Rng(3)
    a = ixo.synth_sparse_matrix(rng, 500, 200, 0.05)
    b = ixo.synth_dense(rng, (200, 128))
    fmt = P.dense_to_groupcoo(torch.from_numpy(a.astype(np.float32)).cuda(), g=0)
    B = torch.from_numpy(b.astype(np.float32)).cuda()
    full = torch.empty((500, 128), device="cuda")
    P.spmm_groupcoo(fmt.AM, fmt.AK, fmt.AV, B, full, accumulate=False, flags=2)
    comm = D.Comm(1, 0)
    plan = D.ShardPlan(fmt.AM, 500, 1, 0, 4)
    out = torch.full_like(full, float("nan"))
    D.spmm_groupcoo_sharded(plan, fmt, B, out, comm=comm)
    torch.cuda.synchronize()
    assert torch.equal(out, full)
    out.fill_(float("nan"))
    D.spmm_groupcoo_sharded(plan, fmt, B, out, comm=comm, flags=2 | D.SHARD_COMM_ONLY)
    torch.cuda.synchronize()
    assert torch.isnan(out).all()  # gather only: nothing computed
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, capture_error_mode="thread_local"):
        D.spmm_groupcoo_sharded(plan, fmt, B, out, comm=comm, flags=1 | 2)  # async index check
    out.fill_(float("nan"))
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, full)


def test_native_comm_broadcast_one_rank(P):
    from paper_2510_17505_b200 import distributed as D
    comm = D.Comm(1, 0)
    t = torch.arange(1000, dtype=torch.float32, device="cuda")
    comm.broadcast(t)
    torch.cuda.synchronize()
    assert torch.equal(t, torch.arange(1000, dtype=torch.float32, device="cuda"))
