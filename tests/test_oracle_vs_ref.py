"""Pins the C oracle restatement (oracle/ixo.c) against the unmodified
reference compiled in place (oracle/_ref). CPU only."""
import numpy as np
import pytest

import instances

KINDS = [1, 0]  # int64, real64


def test_rng_stream_bit_exact(ixo, ref):
    for seed in (0, 1, 2, 99, 2**63 + 5):
        a, b = ixo.Rng(seed), ref.Rng(seed)
        assert [a.next() for _ in range(2000)] == [b.next() for _ in range(2000)]
        for lo, hi in ((1, 4), (0, 0), (0, 16383), (-5, 5), (0, 2**40)):
            assert [a.uniform_int(lo, hi) for _ in range(50)] == \
                   [b.uniform_int(lo, hi) for _ in range(50)]


@pytest.mark.parametrize("kind", KINDS)
def test_synth_bit_exact(ixo, ref, kind):
    for seed in range(5):
        a, b = ixo.Rng(seed), ref.Rng(seed)
        np.testing.assert_array_equal(ixo.synth_dense(a, (7, 5), kind), ref.synth_dense(b, (7, 5), kind))
        np.testing.assert_array_equal(ixo.synth_sparse_matrix(a, 33, 21, 0.17, kind),
                                      ref.synth_sparse_matrix(b, 33, 21, 0.17, kind))
        np.testing.assert_array_equal(ixo.synth_block_sparse_matrix(a, 30, 21, 4, 5, 0.3, kind),
                                      ref.synth_block_sparse_matrix(b, 30, 21, 4, 5, 0.3, kind))
        cx, vx = ixo.synth_coo_tensor(a, (6, 5, 4, 3), 70, kind)
        cy, vy = ref.synth_coo_tensor(b, (6, 5, 4, 3), 70, kind)
        np.testing.assert_array_equal(cx, cy)
        np.testing.assert_array_equal(vx, vy)
        # capacity clamp (synth.cpp:83)
        cx, _ = ixo.synth_coo_tensor(a, (2, 3), 100, kind)
        cy, _ = ref.synth_coo_tensor(b, (2, 3), 100, kind)
        np.testing.assert_array_equal(cx, cy)


def _random_coo(rng, n_rows, n_cols, nnz, dup=True):
    r = rng.integers(0, n_rows, nnz)
    c = rng.integers(0, n_cols, nnz)
    if not dup:
        flat = np.unique(r * n_cols + c)
        rng.shuffle(flat)
        r, c = flat // n_cols, flat % n_cols
    return r.astype(np.int64), c.astype(np.int64)


@pytest.mark.parametrize("group_dim", [0, 1])
def test_coo_to_groupcoo_bit_exact(ixo, ref, group_dim):
    g_np = np.random.default_rng(3)
    for it in range(40):
        rows, cols = int(g_np.integers(1, 20)), int(g_np.integers(1, 20))
        nnz = int(g_np.integers(0, 60))
        r, c = _random_coo(g_np, rows, cols, nnz, dup=bool(it % 2))
        v = g_np.standard_normal(len(r))
        for g in (1, 2, 3, 5, 8):
            a = ixo.coo_to_groupcoo(rows, cols, r, c, v, group_dim, g)
            b = ref.coo_to_groupcoo(rows, cols, r, c, v, group_dim, g)
            for k in ("AM", "AK", "AV", "mask"):
                np.testing.assert_array_equal(a[k], b[k], err_msg=f"{k} it={it} g={g}")


@pytest.mark.parametrize("kind", KINDS)
def test_dense_builders_bit_exact(ixo, ref, kind):
    for seed in range(12):
        rng = ixo.Rng(seed)
        rows, cols = rng.uniform_int(1, 23), rng.uniform_int(1, 23)
        a = ixo.synth_sparse_matrix(rng, rows, cols, 0.2, kind)
        for x, y in zip(ixo.dense_to_coo(a), ref.dense_to_coo(a)):
            np.testing.assert_array_equal(x, y)
        for bm, bk, g, gd in ((2, 2, 1, 0), (4, 4, 2, 0), (3, 5, 3, 1), (16, 16, 8, 0), (1, 7, 2, 1)):
            x = ixo.dense_to_blockgroupcoo(a, bm, bk, g, gd)
            y = ref.dense_to_blockgroupcoo(a, bm, bk, g, gd)
            for k in ("AM", "AK", "AV", "mask"):
                np.testing.assert_array_equal(x[k], y[k], err_msg=f"{k} seed={seed} {bm}x{bk}")


def test_group_coo_tensor_bit_exact(ixo, ref):
    g_np = np.random.default_rng(9)
    for it in range(30):
        rank = int(g_np.integers(2, 5))
        shape = [int(x) for x in g_np.integers(1, 7, rank)]
        nnz = int(g_np.integers(0, 50))
        coords = np.stack([g_np.integers(0, s, nnz) for s in shape]).astype(np.int64)
        vals = g_np.integers(-4, 5, nnz).astype(np.int64)
        for gd in range(rank):
            for g in (1, 2, 4):
                a = ixo.group_coo_tensor(shape, coords, vals, gd, g)
                b = ref.group_coo_tensor(shape, coords, vals, gd, g)
                for k in ("group_coord", "member_coords", "values", "mask"):
                    np.testing.assert_array_equal(a[k], b[k], err_msg=f"{k} it={it}")


def test_tuner_matches(ixo, ref):
    g_np = np.random.default_rng(5)
    profiles = [np.zeros(5, np.int64), np.array([3, 1, 1, 2]), np.array([0, 9, 0, 0, 1])]
    profiles += [g_np.integers(0, m, n) for m in (2, 10, 60) for n in (1, 7, 100)]
    for occ in profiles:
        occ = np.asarray(occ, np.int64)
        for ce in (False, True):
            t = ref.tune(occ, ce)
            assert ixo.select(occ, ce) == t["chosen"]
            assert ixo.g_star(occ, ce) == pytest.approx(t["gstar"], rel=0, abs=0)
            assert ixo.candidate_group_sizes(occ, ce) == [c for c, _ in t["candidates"]]
            assert ixo.brute_force_optimal(occ) == t["brute"]
        for g in range(1, 9):
            assert ixo.cost_exact(occ, g) == ref.cost_exact(occ, g)


@pytest.mark.parametrize("name", list(instances.EXPR))
def test_instances_and_einsum_match_reference(ixo, ref, name):
    """acceptance.cpp criterion 1, restated: identical instances from both
    backends; C oracle == reference oracle (int64 bit-exact, real64 bit-exact)."""
    for i in range(30):
        kind = 1 if i < 20 else 0
        seed = 1000 + i
        ta, expr, on, out = instances.make(ixo, name, kind, seed)
        tb, _, _, _ = instances.make(ref, name, kind, seed)
        assert sorted(ta) == sorted(tb)
        for k in ta:
            np.testing.assert_array_equal(ta[k], tb[k], err_msg=f"{name} {k} seed={seed}")
        mine = ixo.einsum(expr, ta, on, out)
        theirs, _ = ref.run(tb, expr, on, out, "oracle")
        np.testing.assert_array_equal(mine, theirs)
        plan, _ = ref.run(tb, expr, on, out, "plan")
        if kind == 1:
            np.testing.assert_array_equal(plan, mine)
        else:
            assert ixo.max_rel_error(plan, mine) <= 1e-10


def test_einsum_semantics_and_errors(ixo, ref):
    t = {"A": np.array([10, 20], np.int64), "B": np.array([1, 1], np.int64)}
    primed = np.array([5, 5], np.int64)
    np.testing.assert_array_equal(ixo.einsum("C[i] += A[i] * B[i]", t, "C", primed), [15, 25])
    np.testing.assert_array_equal(ixo.einsum("C[i] = A[i] * B[i]", t, "C", primed), [10, 20])
    bad = {"AV": np.array([2], np.int64), "AM": np.array([0], np.int64),
           "AK": np.array([5], np.int64), "B": np.array([[1, 2], [3, 4]], np.int64)}
    expr = "C[AM[p],n] += AV[p] * B[AK[p],n]"
    out = np.zeros((2, 2), np.int64)
    with pytest.raises(ixo.OracleError) as e1:
        ixo.einsum(expr, bad, "C", out)
    with pytest.raises(ref.RefError) as e2:
        ref.run(bad, expr, "C", out, "oracle")
    assert e1.value.code == e2.value.code == 6
    assert str(e1.value) == str(e2.value)
    with pytest.raises(ixo.OracleError) as e3:
        ixo.einsum("C[i] = A[i", t, "C", primed)
    with pytest.raises(ref.RefError) as e4:
        ref.run(t, "C[i] = A[i", "C", primed, "oracle")
    assert e3.value.code == e4.value.code == 2
    assert str(e3.value) == str(e4.value)


def test_metric_helpers_match(ixo, ref):
    g_np = np.random.default_rng(1)
    a = g_np.standard_normal((5, 7))
    b = a + 1e-7 * g_np.standard_normal((5, 7))
    assert ixo.max_rel_error(a, b) == ref.max_rel_error(a, b)
    assert ixo.tensor_hash(a) == ref.tensor_hash(a)
    i = g_np.integers(-9, 9, (3, 4)).astype(np.int64)
    assert ixo.tensor_hash(i) == ref.tensor_hash(i)
