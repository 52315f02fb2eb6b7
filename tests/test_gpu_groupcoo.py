"""GPU parity of K1 (GroupCOO builders + tuner) and K3 (GroupCOO SpMM)
against the C oracle. Integer-valued inputs (±{1..4}, synth.cpp:10-15) are
exact in fp32, so those runs must be bit-exact; real-valued inputs are
rounded to fp32 first and compared with max_rel_error <= 1e-5
(denominator max(|x|,|y|,1), tensor.cpp:124-136)."""
import numpy as np
import pytest

import instances

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

EXPR = "C[AM[p],n] += AV[p,q] * B[AK[p,q],n]"
TOL_F32 = 1e-5


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_17505_b200 as P
    P.lib()
    return P


def dev(x, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(x))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def f32(x):
    return np.asarray(x, np.float64).astype(np.float32).astype(np.float64)


# ------------------------------------------------------------------ builders
@pytest.mark.parametrize("kind", [0, 1])
def test_dense_to_coo_bit_exact(P, ixo, kind):
    rng = ixo.Rng(11)
    for rows, cols, d in ((1, 1, 1.0), (9, 7, 0.3), (33, 130, 0.1), (64, 64, 0.0), (5, 1000, 0.01),
                          (6, 5000, 0.002), (3, 40001, 0.0003)):  # multi-segment rows
        a = ixo.synth_sparse_matrix(rng, rows, cols, d, kind)
        r, c, v = P.dense_to_coo(dev(a, torch.float32))
        wr, wc, wv = ixo.dense_to_coo(a)
        np.testing.assert_array_equal(r.cpu().numpy(), wr)
        np.testing.assert_array_equal(c.cpu().numpy(), wc)
        np.testing.assert_array_equal(v.cpu().numpy().astype(np.float64), f32(wv))


@pytest.mark.parametrize("group_dim", [0, 1])
def test_dense_groupcoo_bit_exact(P, ixo, group_dim):
    rng = ixo.Rng(5)
    for rows, cols, d in ((4, 4, 0.5), (17, 29, 0.2), (100, 64, 0.05), (3, 3, 0.0), (40, 1, 0.7),
                          (7, 5000, 0.001), (2, 40000, 0.0002)):  # rows of several segments
        a = ixo.synth_sparse_matrix(rng, rows, cols, d)
        a32 = f32(a)
        r, c, v = ixo.dense_to_coo(a32)
        for g in (1, 2, 3, 8, 0):
            got = P.dense_to_groupcoo(dev(a32, torch.float32), g=g, group_dim=group_dim)
            gg = got.group_size
            if g == 0:
                occ = ixo.occupancy(r if group_dim == 0 else c, rows if group_dim == 0 else cols)
                assert gg == ixo.select(occ)
            want = ixo.coo_to_groupcoo(rows, cols, r, c, v, group_dim, gg)
            for k in ("AM", "AK", "AV", "mask"):
                x = getattr(got, k).cpu().numpy()
                np.testing.assert_array_equal(x.astype(want[k].dtype), want[k],
                                              err_msg=f"{k} {rows}x{cols} g={g}")


def test_coo_to_groupcoo_unsorted_with_duplicates(P, ixo):
    g_np = np.random.default_rng(7)
    for it in range(12):
        rows, cols = int(g_np.integers(1, 40)), int(g_np.integers(1, 40))
        n = int(g_np.integers(0, 300))
        r = g_np.integers(0, rows, n).astype(np.int64)
        c = g_np.integers(0, cols, n).astype(np.int64)
        v = f32(g_np.standard_normal(n))
        for gd in (0, 1):
            for g in (1, 4, 16):
                got = P.coo_to_groupcoo(rows, cols, dev(r, torch.int32), dev(c, torch.int32),
                                        dev(v, torch.float32), gd, g)
                want = ixo.coo_to_groupcoo(rows, cols, r, c, v, gd, g)
                for k in ("AM", "AK", "AV", "mask"):
                    x = getattr(got, k).cpu().numpy()
                    np.testing.assert_array_equal(x.astype(want[k].dtype), want[k])


def test_coo_to_groupcoo_canonical_fast_path(P, ixo):
    rng = ixo.Rng(3)
    a = ixo.synth_sparse_matrix(rng, 300, 200, 0.05)
    r, c, v = ixo.dense_to_coo(a)
    got = P.coo_to_groupcoo(300, 200, dev(r, torch.int32), dev(c, torch.int32),
                            dev(v, torch.float32), 0, 4, canonical=True)
    want = ixo.coo_to_groupcoo(300, 200, r, c, v, 0, 4)
    np.testing.assert_array_equal(got.AK.cpu().numpy(), want["AK"])
    np.testing.assert_array_equal(got.AM.cpu().numpy(), want["AM"])


@pytest.mark.parametrize("rows", [9000, 70000])
def test_dense_groupcoo_tall_profiles(P, ixo, rows):
    """Row profiles longer than one scan tile (8192 rows) and longer than the
    single-CTA scan (65536 rows, cub path): group offsets and AM bit-exact."""
    rng = ixo.Rng(rows)
    a = f32(ixo.synth_sparse_matrix(rng, rows, 12, 0.3))
    r, c, v = ixo.dense_to_coo(a)
    for g in (3, 0):
        got = P.dense_to_groupcoo(dev(a, torch.float32), g=g)
        want = ixo.coo_to_groupcoo(rows, 12, r, c, v, 0, got.group_size)
        for k in ("AM", "AK", "AV", "mask"):
            np.testing.assert_array_equal(getattr(got, k).cpu().numpy().astype(want[k].dtype),
                                          want[k], err_msg=f"{k} rows={rows} g={g}")


def test_tuner_matches_oracle(P, ixo):
    g_np = np.random.default_rng(2)
    for it in range(20):
        extent = int(g_np.integers(1, 300))
        n = int(g_np.integers(0, 3000))
        coord = np.sort(g_np.integers(0, extent, n) ** 1).astype(np.int64)
        occ = ixo.occupancy(coord, extent)
        for ce in (False, True):
            g, gs = P.tune_group_size(dev(coord, torch.int32), extent, ce)
            assert g == ixo.select(occ, ce)
            assert gs == ixo.g_star(occ, ce)


def test_invalid_builder_parameters(P, ixo):
    a = dev(np.eye(4), torch.float32)
    r, c, v = P.dense_to_coo(a)
    with pytest.raises(P.ShapeError):
        P.coo_to_groupcoo(4, 4, r, c, v, 2, 1)
    with pytest.raises(P.ShapeError):
        P.dense_to_blockgroupcoo(a, 0, 2, 1)
    with pytest.raises(P.ShapeError):
        P.dense_to_groupcoo(a, g=-1)


# ------------------------------------------------------------------- SpMM
def run_spmm(P, t, out, accumulate=True, flags=0):
    G, g = t["AV"].shape
    C = dev(out, torch.float32)
    P.spmm_groupcoo(dev(t["AM"], torch.int32), dev(t["AK"], torch.int32),
                    dev(t["AV"], torch.float32), dev(t["B"], torch.float32), C,
                    accumulate=accumulate, flags=flags)
    return C.cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("kind", [1, 0])
def test_spmm_instances_vs_oracle(P, ixo, kind):
    """acceptance.cpp make_groupcoo_spmm instances (200 int + 40 real there)."""
    for i in range(60 if kind == 1 else 30):
        t, expr, on, out = instances.make(ixo, "groupcoo_spmm", kind, 1000 + i)
        if kind == 0:
            t = {k: (f32(x) if x.dtype == np.float64 else x) for k, x in t.items()}
        want = ixo.einsum(expr, t, on, out)
        for flags in (0, 2):
            got = run_spmm(P, t, out, flags=flags)
            if kind == 1:
                np.testing.assert_array_equal(got.astype(np.int64), want)
            else:
                assert ixo.max_rel_error(want, got) <= TOL_F32


@pytest.mark.parametrize("N", [1, 3, 5, 8, 100, 128, 130, 256, 384, 512, 700])
def test_spmm_ragged_widths(P, ixo, N):
    rng = ixo.Rng(N)
    a = ixo.synth_sparse_matrix(rng, 70, 50, 0.15, 1)
    b = ixo.synth_dense(rng, (50, N), 1)
    r, c, v = ixo.dense_to_coo(a)
    for g in (1, 3, 8, 40):
        gc = ixo.coo_to_groupcoo(70, 50, r, c, v, 0, g)
        t = {"AM": gc["AM"], "AK": gc["AK"], "AV": gc["AV"], "B": b}
        got = run_spmm(P, t, np.zeros((70, N)), flags=2)
        np.testing.assert_array_equal(got.astype(np.int64), a @ b)


def test_spmm_assign_vs_accumulate(P, ixo):
    rng = ixo.Rng(4)
    a = ixo.synth_sparse_matrix(rng, 60, 30, 0.1, 1)
    a[10:20] = 0  # empty rows inside, before and after segments
    a[:3] = 0
    a[-5:] = 0
    b = ixo.synth_dense(rng, (30, 16), 1)
    r, c, v = ixo.dense_to_coo(a)
    gc = ixo.coo_to_groupcoo(60, 30, r, c, v, 0, 4)
    t = {"AM": gc["AM"], "AK": gc["AK"], "AV": gc["AV"], "B": b}
    primed = ixo.synth_dense(rng, (60, 16), 1)
    got_acc = run_spmm(P, t, primed, accumulate=True, flags=2)
    np.testing.assert_array_equal(got_acc.astype(np.int64), primed + a @ b)
    got_set = run_spmm(P, t, primed, accumulate=False, flags=2)
    np.testing.assert_array_equal(got_set.astype(np.int64), a @ b)


def test_spmm_unsorted_groups_and_collisions(P, ixo):
    """Arbitrary AM (collisions, any order): the stable-permutation path."""
    g_np = np.random.default_rng(1)
    for it in range(10):
        G, g, K, N, M = 200, 3, 40, 24, 30
        t = {"AM": g_np.integers(0, M, G).astype(np.int64),
             "AK": g_np.integers(0, K, (G, g)).astype(np.int64),
             "AV": g_np.integers(-4, 5, (G, g)).astype(np.int64),
             "B": g_np.integers(-4, 5, (K, N)).astype(np.int64)}
        out = np.zeros((M, N), np.int64)
        want = ixo.einsum(EXPR, t, "C", out)
        got = run_spmm(P, t, out, flags=0)
        np.testing.assert_array_equal(got.astype(np.int64), want)
        got = run_spmm(P, t, out, accumulate=False, flags=0)
        np.testing.assert_array_equal(got.astype(np.int64), want)


def test_spmm_empty_and_degenerate(P, ixo):
    t = {"AM": np.zeros(0, np.int64), "AK": np.zeros((0, 4), np.int64),
         "AV": np.zeros((0, 4)), "B": np.ones((5, 8))}
    primed = np.full((3, 8), 7.0)
    np.testing.assert_array_equal(run_spmm(P, t, primed, True), primed)
    np.testing.assert_array_equal(run_spmm(P, t, primed, False), np.zeros((3, 8)))


def test_spmm_index_range_errors_like_reference(P, ixo):
    b = np.array([[1, 2], [3, 4]], np.float64)
    t = {"AV": np.array([[2.0]]), "AM": np.array([0]), "AK": np.array([[5]]), "B": b}
    with pytest.raises(P.IndexRangeError) as e:
        run_spmm(P, t, np.zeros((2, 2)))
    want = ("index tensor AK value 5 at position [0] out of range for dim 0 of B (extent 2)")
    assert str(e.value) == want
    assert e.value.code == 6
    # gather errors win over scatter errors; first flat position wins
    t = {"AV": np.ones((3, 2)), "AM": np.array([0, 9, 9]),
         "AK": np.array([[0, 1], [1, 1], [7, -1]]), "B": b}
    with pytest.raises(P.IndexRangeError) as e:
        run_spmm(P, t, np.zeros((2, 2)), flags=2)
    assert "AK value 7 at position [4]" in str(e.value)
    t["AK"] = np.array([[0, 1], [1, 1], [1, 0]])
    with pytest.raises(P.IndexRangeError) as e:
        run_spmm(P, t, np.zeros((2, 2)), flags=2)
    assert str(e.value) == ("index tensor AM value 9 at position [1] out of range for dim 0 "
                            "of C (extent 2)")
    # the library stays usable after an error
    t["AM"] = np.array([0, 1, 1])
    run_spmm(P, t, np.zeros((2, 2)), flags=2)


def test_spmm_deterministic(P, ixo):
    rng = ixo.Rng(9)
    a = f32(ixo.synth_sparse_matrix(rng, 2000, 1500, 0.02))
    b = f32(ixo.synth_dense(rng, (1500, 128)))
    fmt = P.dense_to_groupcoo(dev(a, torch.float32), g=0)
    B = dev(b, torch.float32)
    outs = []
    for _ in range(3):
        C = torch.zeros((2000, 128), device="cuda")
        P.spmm_groupcoo(fmt.AM, fmt.AK, fmt.AV, B, C, flags=2)
        outs.append(C.cpu().numpy())
    assert all(np.array_equal(outs[0], o) for o in outs)


def test_cfg1_full_size_vs_oracle(P, ixo):
    """BASELINE configs[0]: 4096x4096 at 1%, N=128, seed 1 (materialize order:
    dense B first, then A — driver.cpp:169-186)."""
    rng = ixo.Rng(1)
    b = f32(ixo.synth_dense(rng, (4096, 128)))
    a = f32(ixo.synth_sparse_matrix(rng, 4096, 4096, 0.01))
    fmt = P.dense_to_groupcoo(dev(a, torch.float32), g=0)
    r, c, v = ixo.dense_to_coo(a)
    assert fmt.group_size == ixo.select(ixo.occupancy(r, 4096)) == 8
    want_fmt = ixo.coo_to_groupcoo(4096, 4096, r, c, v, 0, 8)
    np.testing.assert_array_equal(fmt.AM.cpu().numpy(), want_fmt["AM"])
    np.testing.assert_array_equal(fmt.AK.cpu().numpy(), want_fmt["AK"])
    C = torch.zeros((4096, 128), device="cuda")
    P.spmm_groupcoo(fmt.AM, fmt.AK, fmt.AV, dev(b, torch.float32), C, flags=2)
    t = {"AM": want_fmt["AM"], "AK": want_fmt["AK"], "AV": want_fmt["AV"], "B": b}
    want = ixo.einsum(EXPR, t, "C", np.zeros((4096, 128)))
    assert ixo.max_rel_error(want, C.cpu().numpy().astype(np.float64)) <= TOL_F32


def test_execute_mode_b200_matches_reference_oracle(P, ixo):
    from paper_2510_17505_b200 import execute_mode
    for i in range(10):
        t, expr, on, out = instances.make(ixo, "groupcoo_spmm", 1, 2000 + i)
        want = ixo.einsum(expr, t, on, out)
        mo = execute_mode("b200", expr, t, on, out)
        np.testing.assert_array_equal(mo.result.astype(np.int64), want)
        G, g = t["AV"].shape
        assert mo.counters == {"gathers": G * g, "scatters": G,
                               "atomic_updates": G * t["B"].shape[1]}
        t, expr, on, out = instances.make(ixo, "coo_spmm", 1, 3000 + i)
        mo = execute_mode("b200", expr, t, on, out)
        np.testing.assert_array_equal(mo.result.astype(np.int64), ixo.einsum(expr, t, on, out))


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_virtual_rank_shards_bit_identical(P, ixo, world):
    """SURVEY.md §4 'virtual ranks': every shard's slab computed on one GPU by
    the sharded code path, assembled, equals the unsharded result bit-for-bit."""
    from paper_2510_17505_b200.distributed import shard_plan, spmm_groupcoo_slab
    rng = ixo.Rng(21)
    a = f32(ixo.synth_sparse_matrix(rng, 3000, 2000, 0.01))
    b = f32(ixo.synth_dense(rng, (2000, 128)))
    fmt = P.dense_to_groupcoo(dev(a, torch.float32), g=0)
    B = dev(b, torch.float32)
    full = torch.zeros((3000, 128), device="cuda")
    P.spmm_groupcoo(fmt.AM, fmt.AK, fmt.AV, B, full, flags=2)
    shards = shard_plan(fmt.AM.cpu().numpy(), 3000, world)
    out = torch.empty_like(full)
    for s in shards:
        out[s.r0:s.r1] = spmm_groupcoo_slab(fmt, B, s)
    assert torch.equal(out, full)


@pytest.mark.parametrize("N", [128, 256])
@pytest.mark.parametrize("accumulate", [False, True])
def test_dense_rows_bit_exact(P, ixo, N, accumulate):
    """Long rows (>= 1024 slots per row on average, the cfg3 d = 0.30 regime):
    integer-valued data match the oracle exactly, for `=` and `+=`, with
    empty rows."""
    rng = ixo.Rng(17)
    M, K = 70, 2100
    a = ixo.synth_sparse_matrix(rng, M, K, 0.6, ixo.INT)
    a[5] = 0
    a[40:43] = 0
    b = ixo.synth_dense(rng, (K, N), ixo.INT)
    fmt = P.dense_to_groupcoo(torch.from_numpy(a).float().cuda(), g=8)
    assert fmt.AK.numel() >= 1024 * M
    c0 = ixo.synth_dense(rng, (M, N), ixo.INT)
    C = torch.from_numpy(c0).float().cuda() if accumulate else torch.zeros((M, N), device="cuda")
    P.spmm_groupcoo(fmt.AM, fmt.AK, fmt.AV, torch.from_numpy(b).float().cuda(), C,
                    accumulate=accumulate)
    r, c, v = ixo.dense_to_coo(a)
    want_f = ixo.coo_to_groupcoo(M, K, r, c, v, 0, 8)
    expr = "C[AM[p],n] += AV[p,q] * B[AK[p,q],n]"
    want = ixo.einsum(expr if accumulate else expr.replace("+=", "="),
                      {"AM": want_f["AM"], "AK": want_f["AK"], "AV": want_f["AV"], "B": b}, "C",
                      c0.astype(np.int64) if accumulate else np.zeros((M, N), np.int64))
    np.testing.assert_array_equal(C.cpu().numpy().astype(np.int64), want)


def test_dense_rows_fp32_column_invariance_and_unsorted_members(P, ixo):
    """fp32 long rows (~1200 terms): N = 256 and N = 192 on the same columns
    give the same bits (per-element summation order does not depend on N);
    the result and that of a hand-built format whose AK is not ascending
    within a row match the fp64 oracle within the fp32 tolerance 1e-5
    (compensated accumulation; plain fp32 sums drift to ~3e-5 here)."""
    rng = ixo.Rng(23)
    M, K, N = 40, 1500, 256
    a = ixo.synth_sparse_matrix(rng, M, K, 0.8)
    b = ixo.synth_dense(rng, (K, N))
    A = torch.from_numpy(a.astype(np.float32)).cuda()
    B = torch.from_numpy(b.astype(np.float32)).cuda()
    fmt = P.dense_to_groupcoo(A, g=16)
    assert fmt.AK.numel() >= 1024 * M
    C = torch.zeros((M, N), device="cuda")
    P.spmm_groupcoo(fmt.AM, fmt.AK, fmt.AV, B, C)
    want = a.astype(np.float32).astype(np.float64) @ b.astype(np.float32).astype(np.float64)
    assert ixo.max_rel_error(want, C.double().cpu().numpy()) <= 1e-5
    C192 = torch.zeros((M, 192), device="cuda")
    P.spmm_groupcoo(fmt.AM, fmt.AK, fmt.AV, B[:, :192].contiguous(), C192)
    assert torch.equal(C[:, :192], C192)
    # reverse the member order of every group: rows stay grouped, AK descends
    AK = fmt.AK.flip(1).contiguous()
    AV = fmt.AV.flip(1).contiguous()
    C2 = torch.zeros((M, N), device="cuda")
    P.spmm_groupcoo(fmt.AM, AK, AV, B, C2)
    t = {"AM": fmt.AM.cpu().numpy().astype(np.int64), "AK": AK.cpu().numpy().astype(np.int64),
         "AV": AV.double().cpu().numpy(), "B": b.astype(np.float32).astype(np.float64)}
    want2 = ixo.einsum("C[AM[p],n] += AV[p,q] * B[AK[p,q],n]", t, "C", np.zeros((M, N)))
    assert ixo.max_rel_error(want2, C2.double().cpu().numpy()) <= 1e-5


def test_cfg3_length_rows_within_fp32_tolerance(P, ixo):
    """Rows as long as cfg3 d = 0.30 (~4900 terms, K = 16384) stay within the
    fp32 tolerance 1e-5 of the fp64 oracle (plain fp32 accumulation: ~1e-4)."""
    rng = ixo.Rng(23)
    M, K, N = 24, 16384, 256
    a = ixo.synth_sparse_matrix(rng, M, K, 0.3).astype(np.float32)
    b = ixo.synth_dense(rng, (K, N)).astype(np.float32)
    fmt = P.dense_to_groupcoo(torch.from_numpy(a).cuda(), g=0)
    C = torch.zeros((M, N), device="cuda")
    P.spmm_groupcoo(fmt.AM, fmt.AK, fmt.AV, torch.from_numpy(b).cuda(), C)
    want = a.astype(np.float64) @ b.astype(np.float64)
    assert ixo.max_rel_error(want, C.double().cpu().numpy()) <= 1e-5


def test_groupcoo_helpers_match_reference_semantics(P, ixo):
    """real_count / pad_count, is_ell, ell_view and groupcoo_to_coo on the
    device (formats.cpp:105-113, 176-208): the round trip returns the
    canonical COO bit for bit, for both group dims and every g up to the
    maximum occupancy (test_formats.cpp:107-131's check, on the device)."""
    rng = ixo.Rng(23)
    for it in range(12):
        t = ixo.synth_sparse_matrix(rng, 40, 33, 0.2)
        r, c, v = ixo.dense_to_coo(t)
        gd = it % 2
        occ = ixo.occupancy(r if gd == 0 else c, 40 if gd == 0 else 33)
        rd = torch.from_numpy(r.astype(np.int32)).cuda()
        cd = torch.from_numpy(c.astype(np.int32)).cuda()
        vd = torch.from_numpy(v).float().cuda()
        ell = P.ell_view(40, 33, rd, cd, vd, gd, canonical=True)
        assert ell.group_size == max(int(occ.max()), 1) and P.is_ell(ell)
        want = ixo.coo_to_groupcoo(40, 33, r, c, v, gd, ell.group_size)
        np.testing.assert_array_equal(ell.AM.cpu().numpy(), want["AM"])
        for g in sorted({1, 2, 3, max(int(occ.max()), 1)}):
            fmt = P.coo_to_groupcoo(40, 33, rd, cd, vd, gd, g, canonical=True)
            w = ixo.coo_to_groupcoo(40, 33, r, c, v, gd, g)
            real = int(w["mask"].sum())
            assert P.real_count(fmt) == real == r.size
            assert P.pad_count(fmt) == w["mask"].size - real
            am = w["AM"]
            assert P.is_ell(fmt) == bool(np.all(am[1:] != am[:-1]))
            rr, cc, vv = P.groupcoo_to_coo(fmt)
            np.testing.assert_array_equal(rr.cpu().numpy(), r)
            np.testing.assert_array_equal(cc.cpu().numpy(), c)
            np.testing.assert_array_equal(vv.cpu().numpy(), v.astype(np.float32))
    # empty format
    e = P.coo_to_groupcoo(4, 4, torch.empty(0, dtype=torch.int32).cuda(),
                          torch.empty(0, dtype=torch.int32).cuda(),
                          torch.empty(0).cuda(), 0, 2, canonical=True)
    assert P.real_count(e) == 0 and P.is_ell(e)
    assert all(x is None or x.numel() == 0 for x in P.groupcoo_to_coo(e))
