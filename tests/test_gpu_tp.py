"""GPU parity of K7 (grouped Clebsch–Gordan tensor product) against the C
oracle: the reference corpus form (per-edge W, CUDA-core path, bit-exact in
integer mode) and the shared-weight e3nn form on tcgen05 (bf16 operands,
fp32 accumulation; tolerance 1e-2), including the real-basis l_max = 3 CG
table grouped by path on the device."""
import numpy as np
import pytest

import instances

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

EXPR_B = "Z[b,CGI[p,q],w] += CGV[p,q] * X[b,CGJ[p,q],u] * Y[b,CGK[p,q]] * W[b,CGL[p],u,w]"
EXPR_S = "Z[b,CGI[p,q],w] += CGV[p,q] * X[b,CGJ[p,q],u] * Y[b,CGK[p,q]] * W[CGL[p],u,w]"
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


def run_tp(P, t, out, accumulate=True):
    Z = cuda(out, torch.float32)
    P.tp_grouped(cuda(t["CGL"], torch.int32), cuda(t["CGI"], torch.int32),
                 cuda(t["CGJ"], torch.int32), cuda(t["CGK"], torch.int32),
                 cuda(t["CGV"], torch.float32), cuda(t["X"], torch.bfloat16),
                 cuda(t["Y"], torch.bfloat16), cuda(t["W"], torch.bfloat16), Z,
                 accumulate=accumulate)
    return Z.double().cpu().numpy()


@pytest.mark.parametrize("kind", [1, 0])
def test_tp_acceptance_instances(P, ixo, kind):
    """acceptance.cpp make_grouped_tp (per-edge W): CUDA-core path."""
    for i in range(30 if kind else 15):
        t, expr, on, out = instances.make(ixo, "grouped_tp", kind, 1000 + i)
        if kind == 0:
            t = {k: (bf16_round(v) if k in ("X", "Y", "W") else v) for k, v in t.items()}
        want = ixo.einsum(expr, t, on, out)
        got = run_tp(P, t, out)
        if kind:
            np.testing.assert_array_equal(got.astype(np.int64), want)
        else:
            assert ixo.max_rel_error(want, got) <= TOL_BF16


def cg_grouped(P, ixo, g):
    """Real-basis CG (l_max 3) grouped by path on the device; checked vs oracle."""
    t = ixo.cg_table(3)
    coords = np.stack([t["i"], t["j"], t["k"], t["l"]])
    shape = [16, 16, 16, len(t["paths"])]
    want = ixo.group_coo_tensor(shape, coords, t["v"], 3, g)
    got = P.group_coo_tensor(shape, [cuda(c, torch.int32) for c in coords],
                             cuda(t["v"], torch.float32), 3, g)
    np.testing.assert_array_equal(got.group_coord.cpu().numpy(), want["group_coord"])
    for m in range(3):
        np.testing.assert_array_equal(got.member_coords[m].cpu().numpy(), want["member_coords"][m])
    return {"CGL": want["group_coord"], "CGI": want["member_coords"][0],
            "CGJ": want["member_coords"][1], "CGK": want["member_coords"][2],
            "CGV": want["values"].astype(np.float32).astype(np.float64)}, len(t["paths"])


@pytest.mark.parametrize("g", [4, 16])
def test_tp_tcgen05_real_cg_shared_w(P, ixo, g):
    cg, nl = cg_grouped(P, ixo, g)
    rng = ixo.Rng(3)
    B = 70  # crosses a 64-edge tile
    t = dict(cg)
    t["X"] = bf16_round(ixo.synth_dense(rng, (B, 16, 64)))
    t["Y"] = bf16_round(ixo.synth_dense(rng, (B, 16)))
    t["W"] = bf16_round(ixo.synth_dense(rng, (nl, 64, 64)))
    out = np.zeros((B, 16, 64))
    want = ixo.einsum(EXPR_S, t, "Z", out)
    got = run_tp(P, t, out)
    assert ixo.max_rel_error(want, got) <= TOL_BF16
    primed = ixo.synth_dense(rng, (B, 16, 64))
    want = ixo.einsum(EXPR_S.replace("+=", "="), t, "Z", primed)
    got = run_tp(P, t, primed, accumulate=False)
    assert ixo.max_rel_error(want, got) <= TOL_BF16


def test_tp_tcgen05_random_cg_and_missing_components(P, ixo):
    rng = ixo.Rng(11)
    ni, nj, nk, nl = 12, 9, 7, 5
    coords, vals = ixo.synth_coo_tensor(rng, (ni, nj, nk, nl), 60)
    gt = ixo.group_coo_tensor((ni, nj, nk, nl), coords, vals, 3, 3)
    t = {"CGL": gt["group_coord"], "CGI": gt["member_coords"][0], "CGJ": gt["member_coords"][1],
         "CGK": gt["member_coords"][2], "CGV": gt["values"]}
    B = 130
    t["X"] = bf16_round(ixo.synth_dense(rng, (B, nj, 64)))
    t["Y"] = bf16_round(ixo.synth_dense(rng, (B, nk)))
    t["W"] = bf16_round(ixo.synth_dense(rng, (nl, 64, 64)))
    primed = ixo.synth_dense(rng, (B, ni, 64))
    want = ixo.einsum(EXPR_S, t, "Z", primed)
    got = run_tp(P, t, primed)
    assert ixo.max_rel_error(want, got) <= TOL_BF16


def test_tp_shared_w_other_widths_simt(P, ixo):
    rng = ixo.Rng(5)
    coords, vals = ixo.synth_coo_tensor(rng, (5, 6, 4, 3), 25, 1)
    gt = ixo.group_coo_tensor((5, 6, 4, 3), coords, vals, 3, 2)
    t = {"CGL": gt["group_coord"], "CGI": gt["member_coords"][0], "CGJ": gt["member_coords"][1],
         "CGK": gt["member_coords"][2], "CGV": gt["values"]}
    t["X"] = ixo.synth_dense(rng, (9, 6, 8), 1)
    t["Y"] = ixo.synth_dense(rng, (9, 4), 1)
    t["W"] = ixo.synth_dense(rng, (3, 8, 5), 1)
    out = np.zeros((9, 5, 5), np.int64)
    want = ixo.einsum(EXPR_S, t, "Z", out)
    got = run_tp(P, t, out)
    np.testing.assert_array_equal(got.astype(np.int64), want)


def test_tp_index_errors(P, ixo):
    t, expr, on, out = instances.make(ixo, "grouped_tp", 1, 1234)
    t = dict(t)
    t["CGK"] = t["CGK"].copy()
    t["CGK"].flat[1] = 99
    with pytest.raises(P.IndexRangeError) as e:
        run_tp(P, t, out)
    assert "index tensor CGK value 99 at position [1] out of range for dim 1 of Y" in str(e.value)


def test_tp_plan_reuse_matches_one_shot(P, ixo):
    """TpPlan (validated/reshaped once) equals ixb_tp_grouped bit for bit on
    several batches, on both the tensor-core (shared W) and CUDA-core
    (per-edge W) paths; create reports index errors like the one-shot call."""
    cg, nl = cg_grouped(P, ixo, 4)
    dev = {k: cuda(v, torch.float32 if k == "CGV" else torch.int32) for k, v in cg.items()}
    plan = P.TpPlan(dev["CGL"], dev["CGI"], dev["CGJ"], dev["CGK"], dev["CGV"], 16, 16, 16, nl)
    rng = ixo.Rng(21)
    W = cuda(bf16_round(ixo.synth_dense(rng, (nl, 64, 64))), torch.bfloat16)
    for B in (1, 64, 200):
        X = cuda(bf16_round(ixo.synth_dense(rng, (B, 16, 64))), torch.bfloat16)
        Y = cuda(bf16_round(ixo.synth_dense(rng, (B, 16))), torch.bfloat16)
        Z1 = torch.zeros((B, 16, 64), device="cuda")
        Z2 = torch.zeros((B, 16, 64), device="cuda")
        plan.run(X, Y, W, Z1, accumulate=False)
        P.tp_grouped(dev["CGL"], dev["CGI"], dev["CGJ"], dev["CGK"], dev["CGV"], X, Y, W, Z2,
                     accumulate=False)
        assert torch.equal(Z1, Z2)
    t, expr, on, out = instances.make(ixo, "grouped_tp", 1, 77)
    d = {k: cuda(t[k], torch.float32 if k == "CGV" else torch.int32)
         for k in ("CGL", "CGI", "CGJ", "CGK", "CGV")}
    Bb, ni, Wd = out.shape
    nj, nk, nl2, U = t["X"].shape[1], t["Y"].shape[1], t["W"].shape[1], t["X"].shape[2]
    plan2 = P.TpPlan(d["CGL"], d["CGI"], d["CGJ"], d["CGK"], d["CGV"], ni, nj, nk, nl2, U, Wd,
                     w_per_batch=True)
    Z = cuda(out, torch.float32)
    plan2.run(cuda(t["X"], torch.bfloat16), cuda(t["Y"], torch.bfloat16),
              cuda(t["W"], torch.bfloat16), Z)
    np.testing.assert_array_equal(Z.cpu().numpy().astype(np.int64), ixo.einsum(expr, t, on, out))
    bad = dict(d)
    bad["CGK"] = bad["CGK"].clone()
    bad["CGK"].view(-1)[1] = 99
    with pytest.raises(P.IndexRangeError) as e:
        P.TpPlan(bad["CGL"], bad["CGI"], bad["CGJ"], bad["CGK"], bad["CGV"], ni, nj, nk, nl2, U,
                 Wd, w_per_batch=True)
    assert "index tensor CGK value 99 at position [1] out of range for dim 1 of Y" in str(e.value)


@pytest.mark.parametrize("nchunks", [1, 3, 8])
def test_tp_plan_run_host_matches_device(P, ixo, nchunks):
    """The host-buffer pipelined form (chunks of whole 64-edge tiles) equals
    the device call bit for bit, for `=` and `+=`, with a ragged last chunk."""
    cg, nl = cg_grouped(P, ixo, 4)
    dev = {k: cuda(v, torch.float32 if k == "CGV" else torch.int32) for k, v in cg.items()}
    plan = P.TpPlan(dev["CGL"], dev["CGI"], dev["CGJ"], dev["CGK"], dev["CGV"], 16, 16, 16, nl)
    rng = ixo.Rng(31)
    B = 333
    X = torch.from_numpy(bf16_round(ixo.synth_dense(rng, (B, 16, 64)))).to(torch.bfloat16)
    Y = torch.from_numpy(bf16_round(ixo.synth_dense(rng, (B, 16)))).to(torch.bfloat16)
    W = cuda(bf16_round(ixo.synth_dense(rng, (nl, 64, 64))), torch.bfloat16)
    Z0 = torch.from_numpy(ixo.synth_dense(rng, (B, 16, 64))).float()
    for acc in (False, True):
        Zd = Z0.cuda() if acc else torch.zeros((B, 16, 64), device="cuda")
        plan.run(X.cuda(), Y.cuda(), W, Zd, accumulate=acc)
        Zh = Z0.clone().pin_memory() if acc else torch.zeros((B, 16, 64)).pin_memory()
        plan.run_host(X.pin_memory(), Y.pin_memory(), W, Zh, accumulate=acc, nchunks=nchunks)
        assert torch.equal(Zh, Zd.cpu())


def test_tp_plan_run_host_per_edge_w(P, ixo):
    """Per-edge W[b,l,u,w] (the reference corpus form, CUDA-core kernel): the
    host-buffer form offsets W per chunk and matches the oracle exactly on
    integer data; pageable host buffers work too (no overlap, same result)."""
    t, expr, on, out = instances.make(ixo, "grouped_tp", 1, 91)
    d = {k: cuda(t[k], torch.float32 if k == "CGV" else torch.int32)
         for k in ("CGL", "CGI", "CGJ", "CGK", "CGV")}
    Bb, ni, Wd = out.shape
    nj, nk, nl, U = t["X"].shape[1], t["Y"].shape[1], t["W"].shape[1], t["X"].shape[2]
    plan = P.TpPlan(d["CGL"], d["CGI"], d["CGJ"], d["CGK"], d["CGV"], ni, nj, nk, nl, U, Wd,
                    w_per_batch=True)
    X = torch.from_numpy(t["X"]).to(torch.bfloat16)
    Y = torch.from_numpy(t["Y"]).to(torch.bfloat16)
    W = cuda(t["W"], torch.bfloat16)
    Z = torch.from_numpy(out).float()  # `+=` into the instance's initial output
    plan.run_host(X, Y, W, Z, accumulate=True, nchunks=3)
    np.testing.assert_array_equal(Z.numpy().astype(np.int64), ixo.einsum(expr, t, on, out))
    # 200 edges (4 tiles, 3 chunks): each chunk reads its own slice of the per-edge W
    g = np.random.default_rng(5)
    Bl = 200
    t2 = dict(t, X=g.integers(-2, 3, (Bl, nj, U)).astype(np.int64),
              Y=g.integers(-2, 3, (Bl, nk)).astype(np.int64),
              W=g.integers(-2, 3, (Bl, nl, U, Wd)).astype(np.int64))  # integer kind, like t
    Z2 = torch.zeros((Bl, ni, Wd))
    plan.run_host(torch.from_numpy(t2["X"]).to(torch.bfloat16),
                  torch.from_numpy(t2["Y"]).to(torch.bfloat16),
                  cuda(t2["W"], torch.bfloat16), Z2, accumulate=False, nchunks=3)
    want2 = ixo.einsum(expr, t2, on, np.zeros((Bl, ni, Wd), np.int64))
    np.testing.assert_array_equal(Z2.numpy().astype(np.int64), want2)


def test_tp_tcgen05_rotation_equivariance(P):
    """The tensor-core TP on spherical-harmonic inputs is rotation equivariant:
    X[b, :, u] = a_u Y(r1_b), Y[b, :] = Y(r2_b) (real SH, l <= 3); rotating every
    direction rotates each output irrep block, so the norm of every (edge,
    channel, l3 block) of Z is unchanged. bf16 inputs: held to 2e-2 of the
    block norm scale."""
    from scipy.spatial.transform import Rotation

    from test_cg_pinned import real_sh
    from paper_2510_17505_b200 import synth as S
    cg = S.cg_table(3)
    nl = cg["npaths"]
    l = cg["l"].cuda()
    gt = P.group_coo_tensor([16, 16, 16, nl], [cg["i"].cuda(), cg["j"].cuda(), cg["k"].cuda(), l],
                            cg["v"].cuda(), 3, 4)
    plan = P.TpPlan(gt.group_coord, *gt.member_coords, gt.values, 16, 16, 16, nl)
    rng = np.random.default_rng(5)
    Bn = 200
    r1 = rng.normal(size=(Bn, 3))
    r2 = rng.normal(size=(Bn, 3))
    r1 /= np.linalg.norm(r1, axis=1, keepdims=True)
    r2 /= np.linalg.norm(r2, axis=1, keepdims=True)
    a = rng.uniform(0.5, 1.5, size=64)
    W = torch.from_numpy(rng.normal(size=(nl, 64, 64)) / 8).to(torch.bfloat16).cuda()

    def run(d1, d2):
        sh1 = np.concatenate([real_sh(k, d1) for k in range(4)], axis=1)  # [B, 16]
        sh2 = np.concatenate([real_sh(k, d2) for k in range(4)], axis=1)
        X = torch.from_numpy(sh1[:, :, None] * a[None, None, :]).to(torch.bfloat16).cuda()
        Y = torch.from_numpy(sh2).to(torch.bfloat16).cuda()
        Z = torch.empty((Bn, 16, 64), device="cuda")
        plan.run(X.contiguous(), Y.contiguous(), W, Z, accumulate=False)
        return Z.double()

    R = Rotation.random(random_state=9).as_matrix()
    Z0, Z1 = run(r1, r2), run(r1 @ R.T, r2 @ R.T)
    for l3 in range(4):
        blk = slice(l3 * l3, (l3 + 1) * (l3 + 1))
        n0 = Z0[:, blk, :].norm(dim=1)
        n1 = Z1[:, blk, :].norm(dim=1)
        scale = n0.max().item()
        assert scale > 0
        assert ((n1 - n0).abs().max().item()) <= 2e-2 * scale, l3


def tp_fp64_reference(cg, X, Y, W):
    """Z = sum over CG entries v * Y[:, k] * (X[:, j, :] @ W[l]) in fp64 on the
    device (the einsum of EXPR_S with '=', summed in float64)."""
    Xd, Yd, Wd = X.double(), Y.double(), W.double()
    B = X.shape[0]
    Z = torch.zeros((B, 16, 64), dtype=torch.float64, device="cuda")
    g = cg["CGI"].shape[1]
    for p in range(cg["CGL"].shape[0]):
        l = int(cg["CGL"][p])
        for q in range(g):
            v = float(cg["CGV"][p, q])
            if v == 0.0:
                continue
            i, j, k = int(cg["CGI"][p, q]), int(cg["CGJ"][p, q]), int(cg["CGK"][p, q])
            Z[:, i, :] += v * Yd[:, k:k + 1] * (Xd[:, j, :] @ Wd[l])
    return Z


@pytest.mark.parametrize("B", [148 * 64 * 2 + 37, 148 * 64 * 5])
def test_tp_tcgen05_many_tiles_per_cta(P, ixo, B):
    """Batches of several 64-edge tiles per persistent CTA (ring phases, the
    next tile's X staged while the current one runs, a ragged last tile) for
    `=` and `+=`, against an fp64 reference. The tensor cores see only the
    exact bf16 operands and every sum runs in fp32, so the error is fp32
    rounding (held to 1e-5 relative, tighter than the 1e-2 bf16 contract)."""
    cg, nl = cg_grouped(P, ixo, 4)
    dev = {k: cuda(v, torch.float32 if k == "CGV" else torch.int32) for k, v in cg.items()}
    plan = P.TpPlan(dev["CGL"], dev["CGI"], dev["CGJ"], dev["CGK"], dev["CGV"], 16, 16, 16, nl)
    assert plan.uses_tensor_cores  # the l_max = 3 schedule fits the kernel's shared memory
    gen = torch.Generator(device="cuda").manual_seed(B)
    X = torch.randn((B, 16, 64), device="cuda", generator=gen).to(torch.bfloat16)
    Y = torch.randn((B, 16), device="cuda", generator=gen).to(torch.bfloat16)
    W = (torch.randn((nl, 64, 64), device="cuda", generator=gen) / 8).to(torch.bfloat16)
    want = tp_fp64_reference(cg, X, Y, W)
    Z = torch.full((B, 16, 64), float("nan"), device="cuda")
    plan.run(X, Y, W, Z, accumulate=False)
    scale = want.abs().max().item()
    assert (Z.double() - want).abs().max().item() <= 1e-5 * scale
    Z0 = torch.randn((B, 16, 64), device="cuda", generator=gen)
    Z1 = Z0.clone()
    plan.run(X, Y, W, Z1, accumulate=True)
    assert (Z1.double() - (want + Z0.double())).abs().max().item() <= 1e-5 * scale
