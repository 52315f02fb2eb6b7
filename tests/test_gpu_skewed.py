"""K3 on skewed (power-law) rows: rows longer than the split threshold
(8192 slots) are cut into fixed pieces from the row start, shared out over
a device work queue and summed in piece order. Checks:
fp64 oracle within the fp32 tolerance, exact integer results, run-to-run
determinism, bit-identity across shard counts (pieces depend only on the
row), `+=`, and a power-law MatrixMarket file through the reference's
ingestion path (matrix_market.cpp:30-159) -> coo_to_groupcoo -> K3."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL_F32 = 1e-5


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_17505_b200 as P
    P.lib()
    return P


def power_law(rows, cols, seed, integer=False, heavy=(0, 7, 8, 1500)):
    """Row lengths ~ Zipf, plus a few rows with 20k-45k nonzeros."""
    g = np.random.default_rng(seed)
    lens = np.minimum(g.zipf(1.6, rows), cols // 4)
    for i, r in enumerate(heavy):
        lens[r] = 20000 + 8333 * i
    r = np.repeat(np.arange(rows), lens)
    c = np.concatenate([np.sort(g.choice(cols, n, replace=False)) for n in lens])
    if integer:
        v = g.integers(1, 5, len(r)) * g.choice([-1, 1], len(r))
    else:
        v = g.uniform(0.125, 1.0, len(r)) * g.choice([-1, 1], len(r))
    return r.astype(np.int32), c.astype(np.int32), v.astype(np.float32)


def dense_ref(rows, cols, r, c, v, b):
    out = np.zeros((rows, b.shape[1]))
    np.add.at(out, r, v.astype(np.float64)[:, None] * b.astype(np.float64)[c])
    return out


@pytest.mark.parametrize("g", [1, 8])
def test_long_rows_vs_fp64_and_deterministic(P, g):
    rows, cols, N = 3000, 60000, 64
    r, c, v = power_law(rows, cols, 3)
    b = np.random.default_rng(4).uniform(-1, 1, (cols, N)).astype(np.float32)
    fmt = P.coo_to_groupcoo(rows, cols, torch.from_numpy(r).cuda(), torch.from_numpy(c).cuda(),
                            torch.from_numpy(v).cuda(), 0, g, canonical=True)
    B = torch.from_numpy(b).cuda()
    C1 = torch.empty((rows, N), device="cuda")
    P.spmm_groupcoo(fmt.AM, fmt.AK, fmt.AV, B, C1, accumulate=False)
    want = dense_ref(rows, cols, r, c, v, b)
    err = np.abs(C1.double().cpu().numpy() - want).max() / np.abs(want).max()
    assert err <= TOL_F32
    for _ in range(3):  # pieces may land on any warp: the bits may not change
        C2 = torch.full_like(C1, 7.0)
        P.spmm_groupcoo(fmt.AM, fmt.AK, fmt.AV, B, C2, accumulate=False)
        assert torch.equal(C1, C2)
    C3 = torch.ones_like(C1)
    P.spmm_groupcoo(fmt.AM, fmt.AK, fmt.AV, B, C3, accumulate=True)
    torch.testing.assert_close(C3, C1 + 1, rtol=1e-6, atol=1e-5)


def test_long_rows_exact_and_shard_invariant(P):
    from paper_2510_17505_b200 import distributed as D
    rows, cols, N = 2000, 50000, 128
    r, c, v = power_law(rows, cols, 5, integer=True, heavy=(3, 4, 1999))
    b = np.random.default_rng(6).integers(-4, 5, (cols, N)).astype(np.float32)
    fmt = P.coo_to_groupcoo(rows, cols, torch.from_numpy(r).cuda(), torch.from_numpy(c).cuda(),
                            torch.from_numpy(v).cuda(), 0, 4, canonical=True)
    B = torch.from_numpy(b).cuda()
    C = torch.empty((rows, N), device="cuda")
    P.spmm_groupcoo(fmt.AM, fmt.AK, fmt.AV, B, C, accumulate=False)
    want = dense_ref(rows, cols, r, c, v, b)
    np.testing.assert_array_equal(C.double().cpu().numpy(), want)
    # real values: any shard count gives the same bits (row-relative pieces)
    vr = np.random.default_rng(7).uniform(-1, 1, len(r)).astype(np.float32)
    fr = P.coo_to_groupcoo(rows, cols, torch.from_numpy(r).cuda(), torch.from_numpy(c).cuda(),
                           torch.from_numpy(vr).cuda(), 0, 4, canonical=True)
    Bf = torch.from_numpy(np.random.default_rng(8).uniform(-1, 1, (cols, N)).astype(np.float32)).cuda()
    full = torch.empty((rows, N), device="cuda")
    P.spmm_groupcoo(fr.AM, fr.AK, fr.AV, Bf, full, accumulate=False)
    for world in (2, 3, 8):
        out = torch.full_like(full, float("nan"))
        for q in range(world):
            plan = D.ShardPlan(fr.AM, rows, world, q, 2)
            D.spmm_groupcoo_sharded(plan, fr, Bf, out, flags=2 | D.SHARD_NO_COMM)
        assert torch.equal(out, full)


def test_power_law_matrix_market(P, tmp_path):
    rows, cols, N = 4000, 40000, 96
    r, c, v = power_law(rows, cols, 9, heavy=(10, 3999))
    path = os.path.join(tmp_path, "powerlaw.mtx")
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real general\n")
        f.write(f"{rows} {cols} {len(r)}\n")
        for i in np.random.default_rng(1).permutation(len(r)):  # unsorted entries
            f.write(f"{r[i] + 1} {c[i] + 1} {float(v[i])!r}\n")
    coo = P.load_matrix_market(path, torch.float32)
    fmt = P.coo_to_groupcoo(rows, cols, coo.row, coo.col, coo.values, 0, 0)
    b = np.random.default_rng(2).uniform(-1, 1, (cols, N)).astype(np.float32)
    C = torch.empty((rows, N), device="cuda")
    P.spmm_groupcoo(fmt.AM, fmt.AK, fmt.AV, torch.from_numpy(b).cuda(), C, accumulate=False)
    want = dense_ref(rows, cols, r, c, v, b)
    err = np.abs(C.double().cpu().numpy() - want).max() / np.abs(want).max()
    assert err <= TOL_F32
