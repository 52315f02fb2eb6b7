"""Parity at BASELINE's full sizes (cfg3 d = 0.30, cfg4, cfg5), built exactly
as bench.py builds them. The oracle (or a torch fp64 reference for these
floating-point kernels) checks slabs and subsets, and size-independent
identities check the whole output:
- row-sum: sum_n C[m, n] = A[m, :] . (sum_n B[:, n]);
- conv: sum_x Out[x, :] = sum_z (sum of In rows paired at offset z) . W[z].
Tolerances: fp32 1e-5 (compensated GroupCOO sums), bf16 inputs 1e-2; an
identity over a sum of terms is held to that tolerance relative to the sum of
the terms' magnitudes (its own value can cancel)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_17505_b200 as P
    P.lib()
    return P


def rel(want, got):
    return ((got - want).abs() / torch.maximum(want.abs(), torch.ones_like(want))).max().item()


def rel_to(want, got, scale):
    """max |got - want| / max(scale, 1): identities over sums of terms"""
    return ((got - want).abs() / torch.maximum(scale, torch.ones_like(scale))).max().item()


@pytest.mark.parametrize("density", [0.30, 0.20, 0.10, 0.05, 0.02])
def test_cfg3_full_size(P, density):
    """16384^2 at every BASELINE density (d = 0.30: 80.5 M nonzeros, ~4900 per
    row), N = 256, tuner-chosen g: rows 0..31 and 16352..16383 against fp64,
    every row through the row-sum identity."""
    from paper_2510_17505_b200 import synth as S
    rng = S.Rng(1)
    B = S.synth_dense(rng, (16384, 256), S.REAL, torch.float32).cuda()
    A = S.synth_sparse_matrix(rng, 16384, 16384, density, S.REAL, torch.float32).cuda()
    fmt = P.dense_to_groupcoo(A, g=0)
    C = torch.empty((16384, 256), device="cuda")
    P.spmm_groupcoo(fmt.AM, fmt.AK, fmt.AV, B, C, accumulate=False)
    for r0 in (0, 16352):
        want = A[r0:r0 + 32].double() @ B.double()
        assert rel(want, C[r0:r0 + 32].double()) <= 1e-5
    want_rs = A.double() @ B.double().sum(dim=1)
    C64 = C.double()
    assert rel_to(want_rs, C64.sum(dim=1), C64.abs().sum(dim=1)) <= 1e-5


def test_cfg5_kernel_map_full_size_bit_exact(P, ixo):
    """The 1 M-voxel kernel map (9.1 M pairs) and its grouping by offset are
    bit-identical to the C oracle (kernel map: brute-force-pinned restatement;
    grouping: reference group_coo_tensor restatement)."""
    from paper_2510_17505_b200 import synth as S
    coords = S.synth_voxel_shells(1_000_000)
    n = coords.shape[0]
    mo, mi, mz = P.kernel_map(coords.cuda())
    wo, wi, wz = ixo.kernel_map(coords.numpy().astype(np.int32))
    np.testing.assert_array_equal(mo.cpu().numpy(), wo)
    np.testing.assert_array_equal(mi.cpu().numpy(), wi)
    np.testing.assert_array_equal(mz.cpu().numpy(), wz)
    g, _ = P.tune_group_size(mz, 27)
    ones = torch.ones(mo.numel(), device="cuda")
    gt = P.group_coo_tensor([n, n, 27], [mo, mi, mz], ones, 2, g, canonical=True)
    want = ixo.group_coo_tensor([n, n, 27], np.stack([wo, wi, wz]).astype(np.int64),
                                np.ones(len(wo)), 2, g)
    np.testing.assert_array_equal(gt.group_coord.cpu().numpy(), want["group_coord"])
    np.testing.assert_array_equal(gt.member_coords[0].cpu().numpy(), want["member_coords"][0])
    np.testing.assert_array_equal(gt.member_coords[1].cpu().numpy(), want["member_coords"][1])
    np.testing.assert_array_equal(gt.values.cpu().numpy(), want["values"])


def test_cfg5_full_size(P):
    """1 M voxels (sphere shells), 64 -> 64 channels: 2000 random output
    voxels against a torch fp64 gather reference, the whole output through
    the per-offset sum identity."""
    from paper_2510_17505_b200 import synth as S
    coords = S.synth_voxel_shells(1_000_000).cuda()
    n = coords.shape[0]
    mo, mi, mz = P.kernel_map(coords)
    g, _ = P.tune_group_size(mz, 27)
    ones = torch.ones(mo.numel(), device="cuda")
    gt = P.group_coo_tensor([n, n, 27], [mo, mi, mz], ones, 2, g, canonical=True)
    plan = P.ConvPlan(gt.group_coord, gt.member_coords[0], gt.member_coords[1], gt.values, n, 27,
                      n)
    rng = S.Rng(1)
    In = S.synth_dense(rng, (n, 64), S.REAL, torch.bfloat16).cuda()
    Wt = S.synth_dense(rng, (27, 64, 64), S.REAL, torch.bfloat16).cuda()
    Out = torch.empty((n, 64), device="cuda")
    plan.run(In, Wt, Out, accumulate=False)
    In64, W64 = In.double(), Wt.double()
    # subset: Out[x] = sum over pairs (x, y, z) of In[y] @ W[z]
    pick = torch.from_numpy(np.random.default_rng(0).choice(n, 2000, replace=False)).cuda()
    sel = torch.isin(mo, pick)
    want = torch.zeros((n, 64), dtype=torch.float64, device="cuda")
    contrib = torch.einsum("pc,pcm->pm", In64[mi[sel].long()], W64[mz[sel].long()])
    want.index_add_(0, mo[sel].long(), contrib)
    assert rel(want[pick], Out.double()[pick]) <= 1e-2
    # whole output: sum_x Out[x] = sum_z (sum of paired In rows at z) @ W[z]
    S_z = torch.zeros((27, 64), dtype=torch.float64, device="cuda")
    S_z.index_add_(0, mz.long(), In64[mi.long()])
    want_total = torch.einsum("zc,zcm->m", S_z, W64)
    O64 = Out.double()
    assert rel_to(want_total, O64.sum(dim=0), O64.abs().sum(dim=0)) <= 1e-2


def test_cfg4_full_size(P, ixo):
    """1 M edges, l_max 3, shared W: edges at the start, middle and end of the
    batch (first, interior and last tiles) against the oracle."""
    from paper_2510_17505_b200 import synth as S
    Bt = 1_000_000
    rng = S.Rng(1)
    X = S.synth_dense(rng, (Bt, 16, 64), S.REAL, torch.bfloat16).cuda()
    Y = S.synth_dense(rng, (Bt, 16), S.REAL, torch.bfloat16).cuda()
    cg = S.cg_table(3)
    nl = cg["npaths"]
    W = S.synth_dense(rng, (nl, 64, 64), S.REAL, torch.bfloat16).cuda()
    l = cg["l"].cuda()
    g, _ = P.tune_group_size(l, nl)
    gt = P.group_coo_tensor([16, 16, 16, nl], [cg["i"].cuda(), cg["j"].cuda(), cg["k"].cuda(), l],
                            cg["v"].cuda(), 3, g)
    plan = P.TpPlan(gt.group_coord, *gt.member_coords, gt.values, 16, 16, 16, nl)
    Z = torch.empty((Bt, 16, 64), device="cuda")
    plan.run(X, Y, W, Z, accumulate=False)
    t = {"CGL": gt.group_coord.cpu().numpy().astype(np.int64),
         "CGI": gt.member_coords[0].cpu().numpy().astype(np.int64),
         "CGJ": gt.member_coords[1].cpu().numpy().astype(np.int64),
         "CGK": gt.member_coords[2].cpu().numpy().astype(np.int64),
         "CGV": gt.values.double().cpu().numpy(), "W": W.double().cpu().numpy()}
    expr = "Z[b,CGI[p,q],w] += CGV[p,q] * X[b,CGJ[p,q],u] * Y[b,CGK[p,q]] * W[CGL[p],u,w]"
    for b0 in (0, 500_000 - 3, Bt - 70):
        sl = slice(b0, b0 + 70)
        tt = dict(t, X=X[sl].double().cpu().numpy(), Y=Y[sl].double().cpu().numpy())
        want = ixo.einsum(expr, tt, "Z", np.zeros((70, 16, 64)))
        assert ixo.max_rel_error(want, Z[sl].double().cpu().numpy()) <= 1e-2
