"""Pins the C oracle against the reference unit tests' known answers
(tests/test_formats.cpp, test_plan.cpp, test_tuner.cpp). CPU only; does not
need the compiled reference, so it also runs on the GPU box."""
import math

import numpy as np
import pytest

from instances import occ3112_matrix

FIG = np.array([3, 1, 1, 2], np.int64)


def test_fig4_dense_to_coo(ixo):  # test_formats.cpp:14-29
    r, c, v = ixo.dense_to_coo(occ3112_matrix())
    assert r.tolist() == [0, 0, 0, 1, 2, 3, 3]
    assert c.tolist() == [0, 1, 3, 1, 2, 0, 3]
    assert ixo.dense_to_coo(np.zeros((3, 3)))[0].size == 0
    r, c, v = ixo.dense_to_coo(np.eye(3))
    assert r.tolist() == [0, 1, 2] and c.tolist() == [0, 1, 2] and v.tolist() == [1, 1, 1]


def test_fig4_occupancy(ixo):  # test_formats.cpp:54-64
    r, c, _ = ixo.dense_to_coo(occ3112_matrix())
    assert ixo.occupancy(r, 4).tolist() == [3, 1, 1, 2]
    assert ixo.occupancy(c, 4).tolist() == [2, 2, 1, 2]


def _fig_groupcoo(ixo, g, gd=0):
    r, c, v = ixo.dense_to_coo(occ3112_matrix())
    return ixo.coo_to_groupcoo(4, 4, r, c, v, gd, g), (r, c, v)


def test_fig4_g2_five_groups_three_pads(ixo):  # test_formats.cpp:66-83
    gc, _ = _fig_groupcoo(ixo, 2)
    assert gc["AM"].size == 5
    assert gc["AV"].shape == (5, 2)
    mask = gc["mask"].ravel()
    assert (mask == 0).sum() == 3 and mask.sum() == 7
    ak, av = gc["AK"].ravel(), gc["AV"].ravel()
    for s in range(10):
        if not mask[s]:
            assert av[s] == 0.0 and ak[s] == ak[s - 1]
        assert 0 <= ak[s] < 4
    assert gc["AM"].tolist() == [0, 0, 1, 2, 3]
    assert gc["AK"].tolist() == [[0, 1], [3, 3], [1, 1], [2, 2], [0, 3]]


def test_fig4_g1_is_coo_and_g3_is_ell(ixo):  # test_formats.cpp:85-105
    gc, (r, c, v) = _fig_groupcoo(ixo, 1)
    assert gc["AM"].tolist() == r.tolist() and gc["AK"].ravel().tolist() == c.tolist()
    assert (gc["mask"] == 0).sum() == 0
    gc3, _ = _fig_groupcoo(ixo, 3)
    assert gc3["AM"].size == 4 and (gc3["mask"] == 0).sum() == 5
    assert len(set(gc3["AM"].tolist())) == 4  # is_ell


def test_group_count_and_bytes(ixo):  # test_formats.cpp:133-150
    for g, groups in ((1, 7), (2, 5), (3, 4)):
        gc, _ = _fig_groupcoo(ixo, g)
        assert gc["AM"].size == groups == sum(math.ceil(o / g) for o in FIG)
    gc, _ = _fig_groupcoo(ixo, 2)
    assert 8 * (gc["AM"].size + gc["AK"].size + gc["AV"].size) == 200  # format_nbytes
    assert gc["mask"].size == 10                                        # mask_nbytes
    assert 8 * 3 * 7 == 168                                             # COO bytes


def test_groupcoo_roundtrip_random(ixo):  # test_formats.cpp:107-131
    rng = ixo.Rng(23)
    for it in range(30):
        t = ixo.synth_sparse_matrix(rng, 12, 9, 0.25)
        r, c, v = ixo.dense_to_coo(t)
        gd = it % 2
        occ = ixo.occupancy(r if gd == 0 else c, 12 if gd == 0 else 9)
        for g in range(1, max(int(occ.max()), 1) + 1):
            gc = ixo.coo_to_groupcoo(12, 9, r, c, v, gd, g)
            m = gc["mask"].astype(bool)
            back = np.zeros((12, 9))
            gco = np.repeat(gc["AM"], g)[m.ravel()]
            mco = gc["AK"].ravel()[m.ravel()]
            rows, cols = (gco, mco) if gd == 0 else (mco, gco)
            np.add.at(back, (rows, cols), gc["AV"].ravel()[m.ravel()])
            np.testing.assert_array_equal(back, t)
            assert gc["AM"].size == sum(-(-o // g) for o in occ)


def test_block_cases(ixo):  # test_formats.cpp:171-205
    t = np.zeros((4, 4))
    t[0, 0], t[1, 1] = 1.0, 2.0
    b = ixo.dense_to_blockgroupcoo(t, 2, 2, 1)
    assert b["AM"].size == 1 and b["AV"].shape == (1, 1, 2, 2)
    rng = ixo.Rng(5)
    d = ixo.synth_dense(rng, (4, 4))
    b = ixo.dense_to_blockgroupcoo(d, 2, 2, 2)
    assert b["mask"].sum() == 4 and b["AM"].size == 2
    b = ixo.dense_to_blockgroupcoo(ixo.synth_dense(ixo.Rng(6), (4, 4)), 4, 4, 1)
    assert b["AM"].size == 1 and b["AV"].size == 16
    s = ixo.synth_sparse_matrix(ixo.Rng(7), 5, 6, 0.5)
    b = ixo.dense_to_blockgroupcoo(s, 4, 4, 2)
    back = np.zeros((8, 8))
    for p in range(b["AM"].size):
        for q in range(2):
            if b["mask"][p, q]:
                br, bc = b["AM"][p], b["AK"][p, q]
                back[br * 4:br * 4 + 4, bc * 4:bc * 4 + 4] = b["AV"][p, q]
    np.testing.assert_array_equal(back[:5, :6], s)


def test_invalid_parameters(ixo):  # test_formats.cpp:277-282
    r, c, v = ixo.dense_to_coo(occ3112_matrix())
    with pytest.raises(ixo.OracleError):
        ixo.coo_to_groupcoo(4, 4, r, c, v, 0, 0)
    with pytest.raises(ixo.OracleError):
        ixo.coo_to_groupcoo(4, 4, r, c, v, 2, 1)
    with pytest.raises(ixo.OracleError):
        ixo.dense_to_blockgroupcoo(occ3112_matrix(), 0, 2, 1)


def test_padding_inert_vs_naive_matmul(ixo):  # test_formats.cpp:207-228
    rng = ixo.Rng(37)
    for it in range(10):
        a = ixo.synth_sparse_matrix(rng, 10, 8, 0.3, 1)
        b = ixo.synth_dense(rng, (8, 5), 1)
        expect = a @ b
        r, c, v = ixo.dense_to_coo(a)
        mo = max(int(ixo.occupancy(r, 10).max()), 1)
        for g in range(1, mo + 2):
            gc = ixo.coo_to_groupcoo(10, 8, r, c, v, 0, g)
            t = {"AV": gc["AV"], "AM": gc["AM"], "AK": gc["AK"], "B": b}
            got = ixo.einsum("C[AM[p],n] += AV[p,q] * B[AK[p,q],n]", t, "C",
                             np.zeros((10, 5), np.int64))
            np.testing.assert_array_equal(got, expect)


def test_plan_kats(ixo):  # test_plan.cpp:77-118
    t = {"AV": np.array([2], np.int64), "AM": np.array([0], np.int64),
         "AK": np.array([1], np.int64), "B": np.array([[1, 2], [3, 4]], np.int64)}
    e = "C[AM[p],n] += AV[p] * B[AK[p],n]"
    assert ixo.einsum(e, t, "C", np.zeros((2, 2), np.int64)).ravel().tolist() == [6, 8, 0, 0]
    t2 = {"AV": np.array([1, 1], np.int64), "AM": np.array([0, 0], np.int64),
          "AK": np.array([0, 1], np.int64), "B": np.array([[1, 2], [3, 4]], np.int64)}
    assert ixo.einsum(e, t2, "C", np.zeros((2, 2), np.int64)).ravel()[:2].tolist() == [4, 6]
    bad = dict(t)
    bad["AK"] = np.array([5], np.int64)
    with pytest.raises(ixo.OracleError) as ei:
        ixo.einsum(e, bad, "C", np.zeros((2, 2), np.int64))
    msg = str(ei.value)
    assert ei.value.code == 6 and "AK" in msg and "5" in msg and "B" in msg and "2" in msg


def test_groupcoo_spmm_vs_naive_real(ixo):  # test_plan.cpp:166-182
    rng = ixo.Rng(61)
    a = occ3112_matrix()
    b = ixo.synth_dense(rng, (4, 3))
    r, c, v = ixo.dense_to_coo(a)
    for g in (1, 2, 3):
        gc = ixo.coo_to_groupcoo(4, 4, r, c, v, 0, g)
        got = ixo.einsum("C[AM[p],n] += AV[p,q] * B[AK[p,q],n]",
                         {"AV": gc["AV"], "AM": gc["AM"], "AK": gc["AK"], "B": b}, "C",
                         np.zeros((4, 3)))
        assert ixo.max_rel_error(a @ b, got) <= 1e-12


def test_tuner_kats(ixo):  # test_tuner.cpp
    assert [ixo.cost_exact(FIG, g) for g in (1, 2, 3)] == [14, 15, 16]
    we = np.array([3, 0, 1, 0, 1, 2], np.int64)
    assert [ixo.cost_exact(we, g) for g in (1, 2, 3)] == [14, 15, 16]
    assert ixo.cost_relaxed(FIG, 1.0) == pytest.approx(22.0)
    assert ixo.cost_relaxed(FIG, 2.0) == pytest.approx(22.5)
    assert ixo.g_star(FIG) == pytest.approx(math.sqrt(7 / 4), rel=1e-12)
    p = np.array([4, 0, 2, 0], np.int64)
    assert ixo.g_star(p, False) == pytest.approx(math.sqrt(3))
    assert ixo.g_star(p, True) == pytest.approx(math.sqrt(1.5))
    assert ixo.cost_relaxed(p, 2.0, False) == pytest.approx(15)
    assert ixo.cost_relaxed(p, 2.0, True) == pytest.approx(21)
    C = ixo.candidate_group_sizes
    assert C(FIG) == [1, 2]
    assert C(np.array([4] * 4)) == [2]
    assert C(np.array([16, 16])) == [4]
    assert C(np.array([16, 1, 1])) == [2, 4]
    assert C(np.array([16])) == [4]
    assert C(np.array([10000])) == [64, 128]
    assert C(np.array([12] * 16)) == [2, 4]
    assert C(np.array([0])) == [1]
    assert ixo.brute_force_optimal(FIG) == (1, 14)
    assert ixo.brute_force_optimal(np.array([8] * 4)) == (8, 36)
    assert ixo.brute_force_optimal(np.array([0, 0])) is None
    assert ixo.select(FIG) == 1
    assert ixo.select(np.zeros(3, np.int64)) == 1


def test_kernel_map_bruteforce(ixo):
    """Reference-absent KAT: kernel map == brute force over all pairs."""
    g = np.random.default_rng(0)
    pts = np.unique(g.integers(0, 6, (80, 3)), axis=0).astype(np.int32)
    mo, mi, mz = ixo.kernel_map(pts)
    want = []
    for z in range(27):
        d = np.array([z // 9 - 1, (z // 3) % 3 - 1, z % 3 - 1])
        for i in range(len(pts)):
            for j in range(len(pts)):
                if (pts[j] == pts[i] + d).all():
                    want.append((z, i, j))
    got = sorted(zip(mz.tolist(), mo.tolist(), mi.tolist()))
    assert got == sorted(want)
    assert list(zip(mz.tolist(), mo.tolist())) == sorted(zip(mz.tolist(), mo.tolist()))


def test_cg_table_counts_and_orthogonality(ixo):
    """Reference-absent KAT: real-basis CG for l_max=3 — 23 parity-allowed
    paths and, per path, orthonormal coupling columns."""
    t = ixo.cg_table(3)
    assert len(t["paths"]) == 23
    for p, (l1, l2, l3) in enumerate(t["paths"]):
        sel = t["l"] == p
        M = np.zeros((2 * l3 + 1, (2 * l1 + 1) * (2 * l2 + 1)))
        M[t["i"][sel] - l3 * l3, (t["j"][sel] - l1 * l1) * (2 * l2 + 1) + (t["k"][sel] - l2 * l2)] \
            = t["v"][sel]
        np.testing.assert_allclose(M @ M.T, np.eye(2 * l3 + 1), atol=1e-12)
