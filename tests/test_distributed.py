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
