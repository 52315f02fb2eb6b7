"""Multi-rank host logic on CPU (gloo, world sizes 2 and 3): shard planning at
row boundaries and the output all-gather. Each rank evaluates its shard with
the C oracle; the gathered result must equal the single-rank result
bit-for-bit (per-row summation order is unchanged by sharding)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
EXPR = "C[AM[p],n] += AV[p,q] * B[AK[p,q],n]"


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _make(seed, rows=97, cols=60, density=0.08, N=7, kind=0, g=3):
    sys.path[:0] = [ROOT, HERE]
    from oracle import ixo
    rng = ixo.Rng(seed)
    a = ixo.synth_sparse_matrix(rng, rows, cols, density, kind)
    a[10:20] = 0  # empty rows, possibly at a cut
    a[-4:] = 0
    b = ixo.synth_dense(rng, (cols, N), kind)
    r, c, v = ixo.dense_to_coo(a)
    gc = ixo.coo_to_groupcoo(rows, cols, r, c, v, 0, g)
    return gc, b


def _worker(rank, world, port, seed, q):
    sys.path[:0] = [ROOT, HERE]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import ixo
        from paper_2510_17505_b200.distributed import gather_rows, shard_plan
        gc, b = _make(seed)
        rows, N = 97, b.shape[1]
        shards = shard_plan(gc["AM"].astype(np.int32), rows, world)
        s = shards[rank]
        # this rank's shard, evaluated by the oracle into its slab (rows rebased)
        t = {"AM": gc["AM"][s.g0:s.g1] - s.r0, "AK": gc["AK"][s.g0:s.g1],
             "AV": gc["AV"][s.g0:s.g1], "B": b}
        slab = ixo.einsum(EXPR, t, "C", np.zeros((s.r1 - s.r0, N))) if s.g1 > s.g0 else \
            np.zeros((s.r1 - s.r0, N))
        full = gather_rows(torch.from_numpy(slab), shards, rank)
        q.put((rank, full.numpy(), [(x.g0, x.g1, x.r0, x.r1) for x in shards]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_groupcoo_gather_bit_identical(ixo, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 5, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    gc, b = _make(5)
    want = ixo.einsum(EXPR, {"AM": gc["AM"], "AK": gc["AK"], "AV": gc["AV"], "B": b}, "C",
                      np.zeros((97, b.shape[1])))
    for rank, full, shards in results:
        np.testing.assert_array_equal(full, want)  # bit-identical to one rank
        # shards tile the groups and the rows, cuts only at row changes
        assert shards[0][0] == 0 and shards[-1][1] == gc["AM"].size
        assert shards[0][2] == 0 and shards[-1][3] == 97
        for (g0, g1, r0, r1), (h0, h1, s0, s1) in zip(shards, shards[1:]):
            assert g1 == h0 and r1 == s0
            if 0 < h0 < gc["AM"].size:
                assert gc["AM"][h0] != gc["AM"][h0 - 1]
        for g0, g1, r0, r1 in shards:
            if g1 > g0:
                assert r0 <= gc["AM"][g0] and gc["AM"][g1 - 1] < r1


def test_shard_plan_edge_cases():
    sys.path[:0] = [ROOT, HERE]
    from paper_2510_17505_b200.distributed import shard_plan
    # one long row: every rank but one gets nothing, rows still tile
    am = np.zeros(50, np.int32)
    sh = shard_plan(am, 4, 3)
    assert [(s.g0, s.g1) for s in sh][0] == (0, 50) or sh[-1].g1 == 50
    assert sh[0].r0 == 0 and sh[-1].r1 == 4
    assert sum(s.g1 - s.g0 for s in sh) == 50
    # empty format
    sh = shard_plan(np.zeros(0, np.int32), 5, 2)
    assert sh[-1].r1 == 5 and all(s.g0 == s.g1 for s in sh)


CONV = "Out[MAPX[p,q],m] += MAPV[p,q] * In[MAPY[p,q],c] * Weight[MAPZ[p],c,m]"
TP = "Z[b,CGI[p,q],w] += CGV[p,q] * X[b,CGJ[p,q],u] * Y[b,CGK[p,q]] * W[CGL[p],u,w]"


def _conv_case(seed):
    sys.path[:0] = [ROOT, HERE]
    from oracle import ixo
    g = np.random.default_rng(seed)
    pts = np.unique(g.integers(0, 7, (120, 3)), axis=0).astype(np.int32)
    mo, mi, mz = ixo.kernel_map(pts)
    n = len(pts)
    In = g.integers(-3, 4, (n, 5)).astype(np.float64)
    W = g.integers(-2, 3, (27, 5, 4)).astype(np.float64)
    return n, mo, mi, mz, In, W


def _conv_eval(ixo, n_out, mo, mi, mz, In, W):
    gt = ixo.group_coo_tensor([n_out, In.shape[0], 27], np.stack([mo, mi, mz]),
                              np.ones(len(mo)), 2, 4)
    t = {"MAPZ": gt["group_coord"], "MAPX": gt["member_coords"][0],
         "MAPY": gt["member_coords"][1], "MAPV": gt["values"], "In": In, "Weight": W}
    return ixo.einsum(CONV, t, "Out", np.zeros((n_out, W.shape[2])))


def _tp_case(seed):
    sys.path[:0] = [ROOT, HERE]
    from oracle import ixo
    t = ixo.cg_table(2)
    nl = len(t["paths"])
    gt = ixo.group_coo_tensor([9, 9, 9, nl], np.stack([t["i"], t["j"], t["k"], t["l"]]),
                              t["v"], 3, 4)
    g = np.random.default_rng(seed)
    B = 23
    X, Y = g.standard_normal((B, 9, 6)), g.standard_normal((B, 9))
    W = g.standard_normal((nl, 6, 5))
    cg = {"CGL": gt["group_coord"], "CGI": gt["member_coords"][0],
          "CGJ": gt["member_coords"][1], "CGK": gt["member_coords"][2], "CGV": gt["values"]}
    return cg, X, Y, W


def _worker_conv_tp(rank, world, port, q):
    sys.path[:0] = [ROOT, HERE]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import ixo
        from paper_2510_17505_b200.distributed import (edge_blocks, gather_rows, point_blocks,
                                                       shard_map)
        n, mo, mi, mz, In, W = _conv_case(3)
        s = point_blocks(n, world)[rank]
        lo, li, lz = shard_map(mo, mi, mz, s)  # In is replicated: input indices stay global
        slab = _conv_eval(ixo, s.r1 - s.r0, lo, li, lz, In, W)
        conv = gather_rows(torch.from_numpy(slab), point_blocks(n, world), rank).numpy()
        cg, X, Y, Wt = _tp_case(4)
        e = edge_blocks(X.shape[0], world)[rank]
        t = dict(cg, X=X[e.r0:e.r1], Y=Y[e.r0:e.r1], W=Wt)
        z = ixo.einsum(TP, t, "Z", np.zeros((e.r1 - e.r0, 9, 5)))
        tp = gather_rows(torch.from_numpy(z), edge_blocks(X.shape[0], world), rank).numpy()
        q.put((rank, conv, tp))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_conv_and_tp_gather_bit_identical(ixo, world):
    """Point-block conv shards (map filtered by output voxel)
    and edge-range TP shards, each gathered over gloo, equal one rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_conv_tp, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n, mo, mi, mz, In, W = _conv_case(3)
    want_conv = _conv_eval(ixo, n, mo, mi, mz, In, W)
    cg, X, Y, Wt = _tp_case(4)
    want_tp = ixo.einsum(TP, dict(cg, X=X, Y=Y, W=Wt), "Z", np.zeros((X.shape[0], 9, 5)))
    for rank, conv, tp in results:
        np.testing.assert_array_equal(conv, want_conv)
        np.testing.assert_array_equal(tp, want_tp)


def test_shard_map_keeps_canonical_order():
    sys.path[:0] = [ROOT, HERE]
    from oracle import ixo
    from paper_2510_17505_b200.distributed import point_blocks, shard_map
    n, mo, mi, mz, _, _ = _conv_case(8)
    got = []
    for s in point_blocks(n, 4):
        lo, li, lz = shard_map(mo, mi, mz, s)
        key = lz.astype(np.int64) * n + lo
        assert np.all(np.diff(key) > 0)  # (offset, out) order survives the filter
        got.append(len(lo))
    assert sum(got) == len(mo)
