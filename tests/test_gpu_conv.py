"""GPU parity of K5 (kernel map), rank-n grouping and K6 (grouped sparse
conv: tcgen05 implicit-GEMM path and the CSR fallback) against the C oracle.
bf16 In/Weight with fp32 accumulation: tolerance 1e-2 (max_rel_error);
integer-valued inputs must match bit-for-bit."""
import numpy as np
import pytest

import instances

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

EXPR = "Out[MAPX[p,q],m] += MAPV[p,q] * In[MAPY[p,q],c] * Weight[MAPZ[p],c,m]"
TOL_BF16 = 1e-2


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_17505_b200 as P
    P.lib()
    return P


def bf16_round(x):
    return torch.from_numpy(np.asarray(x, np.float64)).to(torch.bfloat16).double().numpy()


def cuda(x, dtype):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dtype).cuda()


def random_voxels(seed, n, extent):
    g = np.random.default_rng(seed)
    pts = np.unique(g.integers(-extent, extent, (n, 3)), axis=0)
    g.shuffle(pts)  # arbitrary voxel order: the map is in terms of indices
    return pts.astype(np.int32)


def test_kernel_map_bit_exact(P, ixo):
    from paper_2510_17505_b200 import synth as S
    cases = [random_voxels(0, 400, 6), random_voxels(1, 3000, 12), random_voxels(2, 50, 100),
             S.synth_voxel_shells(5000).numpy(), np.zeros((0, 3), np.int32),
             np.array([[5, -7, 3]], np.int32),
             # flat and thin boxes (the occupancy-bitmap count pass's column edges)
             np.array([[x, y, 0] for x in range(-3, 20) for y in range(9)], np.int32),
             np.array([[2, 1, z] for z in range(-40, 40, 1)], np.int32),
             random_voxels(3, 2000, 9)[:, [2, 0, 1]]]
    for pts in cases:
        mo, mi, mz = P.kernel_map(cuda(pts, torch.int32))
        wo, wi, wz = ixo.kernel_map(pts)
        np.testing.assert_array_equal(mo.cpu().numpy(), wo)
        np.testing.assert_array_equal(mi.cpu().numpy(), wi)
        np.testing.assert_array_equal(mz.cpu().numpy(), wz)


def test_kernel_map_rejects_duplicates(P):
    pts = np.array([[0, 0, 0], [1, 0, 0], [0, 0, 0]], np.int32)
    with pytest.raises(P.ShapeError):
        P.kernel_map(cuda(pts, torch.int32))


def test_group_coo_tensor_bit_exact(P, ixo):
    g_np = np.random.default_rng(3)
    for it in range(25):
        rank = int(g_np.integers(2, 5))
        shape = [int(x) for x in g_np.integers(1, 9, rank)]
        nnz = int(g_np.integers(0, 200))
        coords = np.stack([g_np.integers(0, s, nnz) for s in shape]).astype(np.int64)
        vals = g_np.integers(-4, 5, nnz).astype(np.float64)
        for gd in range(rank):
            for g in (1, 3, 8):
                got = P.group_coo_tensor(shape, [cuda(c, torch.int32) for c in coords],
                                         cuda(vals, torch.float32), gd, g)
                want = ixo.group_coo_tensor(shape, coords, vals, gd, g)
                np.testing.assert_array_equal(got.group_coord.cpu().numpy(), want["group_coord"])
                for m in range(rank - 1):
                    np.testing.assert_array_equal(got.member_coords[m].cpu().numpy(),
                                                  want["member_coords"][m])
                np.testing.assert_array_equal(got.values.double().cpu().numpy(), want["values"])
                np.testing.assert_array_equal(got.mask.cpu().numpy(), want["mask"])


def test_group_coo_tensor_canonical_small_extent(P, ixo):
    """canonical=True over small group extents: runs indexed by value (the
    histogram fast path), values absent from the input, and a coordinate
    out of range (falls back to the general run finder)."""
    g_np = np.random.default_rng(4)
    for it in range(12):
        rank = int(g_np.integers(2, 4))
        shape = [int(x) for x in g_np.integers(2, 12, rank)]
        nnz = int(g_np.integers(1, 300))
        gd = int(g_np.integers(0, rank))
        coords = np.stack([g_np.integers(0, s, nnz) for s in shape]).astype(np.int64)
        coords[gd] = np.where(coords[gd] % 3 == 1, 0, coords[gd])  # gaps in the group values
        # canonical order: group dim, then the other dims ascending
        keys = [coords[d] for d in reversed([d for d in range(rank) if d != gd])] + [coords[gd]]
        coords = coords[:, np.lexsort(keys)]
        vals = g_np.integers(-4, 5, nnz).astype(np.float64)
        for g in (1, 4):
            got = P.group_coo_tensor(shape, [cuda(c, torch.int32) for c in coords],
                                     cuda(vals, torch.float32), gd, g, canonical=True)
            want = ixo.group_coo_tensor(shape, coords, vals, gd, g)
            np.testing.assert_array_equal(got.group_coord.cpu().numpy(), want["group_coord"])
            for m in range(rank - 1):
                np.testing.assert_array_equal(got.member_coords[m].cpu().numpy(),
                                              want["member_coords"][m])
            np.testing.assert_array_equal(got.values.double().cpu().numpy(), want["values"])
            np.testing.assert_array_equal(got.mask.cpu().numpy(), want["mask"])
    # a group coordinate beyond the declared extent: same result as canonical=False
    coords = np.array([[0, 0, 2, 5], [1, 2, 0, 1]], np.int64)
    vals = np.array([1.0, 2.0, 3.0, 4.0])
    a = P.group_coo_tensor([3, 3], [cuda(c, torch.int32) for c in coords],
                           cuda(vals, torch.float32), 0, 2, canonical=True)
    b = P.group_coo_tensor([3, 3], [cuda(c, torch.int32) for c in coords],
                           cuda(vals, torch.float32), 0, 2)
    np.testing.assert_array_equal(a.group_coord.cpu().numpy(), b.group_coord.cpu().numpy())
    np.testing.assert_array_equal(a.values.cpu().numpy(), b.values.cpu().numpy())


def build_grouped_map(P, ixo, pts, g):
    """Device kernel map -> device group_coo_tensor(·, 2, g); checked vs oracle."""
    n = len(pts)
    mo, mi, mz = P.kernel_map(cuda(pts, torch.int32))
    ones = torch.ones(mo.numel(), dtype=torch.float32, device="cuda")
    gt = P.group_coo_tensor([n, n, 27], [mo, mi, mz], ones, 2, g, canonical=True)
    wo, wi, wz = ixo.kernel_map(pts)
    want = ixo.group_coo_tensor([n, n, 27], np.stack([wo, wi, wz]), np.ones(len(wo)), 2, g)
    np.testing.assert_array_equal(gt.group_coord.cpu().numpy(), want["group_coord"])
    np.testing.assert_array_equal(gt.member_coords[0].cpu().numpy(), want["member_coords"][0])
    np.testing.assert_array_equal(gt.member_coords[1].cpu().numpy(), want["member_coords"][1])
    np.testing.assert_array_equal(gt.values.double().cpu().numpy(), want["values"])
    return gt, want


def run_conv(P, t, n_in, n_out, n_off, accumulate=True, out=None, plan=False):
    Cin = t["In"].shape[1]
    Cout = t["Weight"].shape[2]
    Out = cuda(out if out is not None else np.zeros((n_out, Cout)), torch.float32)
    MAPX, MAPY, MAPZ = (cuda(t[k], torch.int32) for k in ("MAPX", "MAPY", "MAPZ"))
    MAPV = cuda(t["MAPV"], torch.float32)
    if MAPX.dim() == 1:
        MAPX, MAPY, MAPV = MAPX.reshape(-1, 1), MAPY.reshape(-1, 1), MAPV.reshape(-1, 1)
    In, W = cuda(t["In"], torch.bfloat16), cuda(t["Weight"], torch.bfloat16)
    if plan:
        cp = P.ConvPlan(MAPZ, MAPX, MAPY, MAPV, n_in, n_off, n_out)
        cp.run(In, W, Out, accumulate=accumulate)
    else:
        P.conv_grouped(MAPZ, MAPX, MAPY, MAPV, In, W, Out, accumulate=accumulate)
    return Out.double().cpu().numpy()


@pytest.mark.parametrize("name", ["grouped_sparse_conv", "sparse_conv"])
@pytest.mark.parametrize("kind", [1, 0])
def test_conv_acceptance_instances(P, ixo, name, kind):
    """acceptance.cpp make_sparse_conv (random maps with collisions): CSR path."""
    for i in range(30 if kind else 15):
        t, expr, on, out = instances.make(ixo, name, kind, 1000 + i)
        if kind == 0:
            t = {k: (bf16_round(v) if k in ("In", "Weight") else v) for k, v in t.items()}
        want = ixo.einsum(expr, t, on, out)
        got = run_conv(P, t, t["In"].shape[0], out.shape[0], t["Weight"].shape[0])
        if kind:
            np.testing.assert_array_equal(got.astype(np.int64), want)
        else:
            assert ixo.max_rel_error(want, got) <= TOL_BF16


@pytest.mark.parametrize("g", [1, 16, 0])
def test_conv_tcgen05_submanifold_int_bit_exact(P, ixo, g):
    from paper_2510_17505_b200 import synth as S
    pts = S.synth_voxel_shells(700).numpy()
    n = len(pts)
    gsz = g if g else 32
    gt, want = build_grouped_map(P, ixo, pts, gsz)
    rng = ixo.Rng(7)
    In = ixo.synth_dense(rng, (n, 64), 1)
    W = ixo.synth_dense(rng, (27, 64, 64), 1)
    t = {"MAPZ": want["group_coord"], "MAPX": want["member_coords"][0],
         "MAPY": want["member_coords"][1], "MAPV": want["values"].astype(np.int64), "In": In,
         "Weight": W}
    ref = ixo.einsum(EXPR, t, "Out", np.zeros((n, 64), np.int64))
    got = run_conv(P, {**t, "MAPV": want["values"]}, n, n, 27)
    np.testing.assert_array_equal(got.astype(np.int64), ref)
    got = run_conv(P, {**t, "MAPV": want["values"]}, n, n, 27, plan=True)
    np.testing.assert_array_equal(got.astype(np.int64), ref)


def test_conv_tcgen05_real_values_and_semantics(P, ixo):
    pts = random_voxels(5, 900, 7)
    n = len(pts)
    gt, want = build_grouped_map(P, ixo, pts, 8)
    rng = ixo.Rng(9)
    In = bf16_round(ixo.synth_dense(rng, (n, 64)))
    W = bf16_round(ixo.synth_dense(rng, (27, 64, 64)))
    MAPV = want["values"] * 0.5  # non-unit values: scaled in fp32, rounded to bf16
    t = {"MAPZ": want["group_coord"], "MAPX": want["member_coords"][0],
         "MAPY": want["member_coords"][1], "MAPV": MAPV, "In": In, "Weight": W}
    primed = ixo.synth_dense(rng, (n, 64))
    ref = ixo.einsum(EXPR, t, "Out", primed)
    got = run_conv(P, t, n, n, 27, accumulate=True, out=primed)
    assert ixo.max_rel_error(ref, got) <= TOL_BF16
    ref0 = ixo.einsum(EXPR.replace("+=", "="), t, "Out", primed)
    got0 = run_conv(P, t, n, n, 27, accumulate=False, out=primed)
    assert ixo.max_rel_error(ref0, got0) <= TOL_BF16


def test_conv_index_errors(P, ixo):
    pts = random_voxels(1, 200, 4)
    n = len(pts)
    gt, want = build_grouped_map(P, ixo, pts, 4)
    t = {"MAPZ": want["group_coord"], "MAPX": want["member_coords"][0].copy(),
         "MAPY": want["member_coords"][1].copy(), "MAPV": want["values"],
         "In": np.ones((n, 64)), "Weight": np.ones((27, 64, 64))}
    t["MAPY"].flat[5] = n + 3
    t["MAPX"].flat[2] = -1
    with pytest.raises(P.IndexRangeError) as e:
        run_conv(P, t, n, n, 27)
    assert str(e.value) == (f"index tensor MAPY value {n + 3} at position [5] out of range for "
                            f"dim 0 of In (extent {n})")
    t["MAPY"] = want["member_coords"][1]
    with pytest.raises(P.IndexRangeError) as e:
        run_conv(P, t, n, n, 27)
    assert "index tensor MAPX value -1 at position [2]" in str(e.value)


@pytest.mark.parametrize("nchunks", [1, 2, 5])
def test_conv_plan_run_host_matches_device(P, nchunks):
    """Host-buffer form (output-tile chunks started as their input rows land)
    equals the device call bit for bit, for `=` and `+=`."""
    g = np.random.default_rng(4)
    pts = np.unique(g.integers(0, 20, (3000, 3)), axis=0).astype(np.int32)
    order = np.lexsort((pts[:, 2], pts[:, 1], pts[:, 0]))  # sorted voxels: local windows
    pts = pts[order]
    n = len(pts)
    mo, mi, mz = P.kernel_map(torch.from_numpy(pts).cuda())
    gt = P.group_coo_tensor([n, n, 27], [mo, mi, mz], torch.ones(mo.numel(), device="cuda"), 2,
                            16, canonical=True)
    plan = P.ConvPlan(gt.group_coord, gt.member_coords[0], gt.member_coords[1], gt.values, n, 27,
                      n)
    In = torch.from_numpy(g.standard_normal((n, 64))).to(torch.bfloat16)
    W = torch.from_numpy(g.standard_normal((27, 64, 64)) * 0.1).to(torch.bfloat16).cuda()
    O0 = torch.from_numpy(g.standard_normal((n, 64))).float()
    for acc in (False, True):
        Od = O0.cuda() if acc else torch.zeros((n, 64), device="cuda")
        plan.run(In.cuda(), W, Od, accumulate=acc)
        Oh = O0.clone().pin_memory() if acc else torch.zeros((n, 64)).pin_memory()
        plan.run_host(In.pin_memory(), W, Oh, accumulate=acc, nchunks=nchunks)
        assert torch.equal(Oh, Od.cpu())


def test_conv_plan_run_host_non_unit_map(P):
    """Maps with MAPV != 1 take the host form's copy-all / run / copy-back
    branch; it equals the device call bit for bit."""
    g = np.random.default_rng(6)
    pts = np.unique(g.integers(0, 12, (900, 3)), axis=0).astype(np.int32)
    n = len(pts)
    mo, mi, mz = P.kernel_map(torch.from_numpy(pts).cuda())
    vals = torch.from_numpy(g.uniform(0.5, 1.5, mo.numel())).float().cuda()
    gt = P.group_coo_tensor([n, n, 27], [mo, mi, mz], vals, 2, 8, canonical=True)
    plan = P.ConvPlan(gt.group_coord, gt.member_coords[0], gt.member_coords[1], gt.values, n, 27,
                      n)
    In = torch.from_numpy(g.standard_normal((n, 64))).to(torch.bfloat16)
    W = torch.from_numpy(g.standard_normal((27, 64, 64)) * 0.1).to(torch.bfloat16).cuda()
    Od = torch.zeros((n, 64), device="cuda")
    plan.run(In.cuda(), W, Od, accumulate=False)
    Oh = torch.zeros((n, 64)).pin_memory()
    plan.run_host(In.pin_memory(), W, Oh, accumulate=False, nchunks=4)
    assert torch.equal(Oh, Od.cpu())
