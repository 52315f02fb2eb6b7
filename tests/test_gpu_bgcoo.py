"""GPU parity of K2 (BlockGroupCOO builder) and K4 (BlockGroupCOO SpMM on
tcgen05/TMEM, plus its CUDA-core fallback for other block shapes) against the
C oracle. bf16 inputs with fp32 accumulation: tolerance 1e-2 in
max_rel_error (BASELINE.json north_star); integer-valued inputs are exact
and must match bit-for-bit."""
import numpy as np
import pytest

import instances

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

EXPR = "C[AM[p],bm,n] += AV[p,q,bm,bk] * B[AK[p,q],bk,n]"
TOL_BF16 = 1e-2


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_17505_b200 as P
    P.lib()
    return P


def bf16(x):
    return torch.from_numpy(np.ascontiguousarray(x, np.float64)).to(torch.bfloat16)


def bf16_round(x):
    return bf16(x).double().numpy()


def run(P, t, out, accumulate=True, flags=0):
    C = torch.from_numpy(np.ascontiguousarray(out, np.float64)).float().cuda()
    P.spmm_blockgroupcoo(torch.from_numpy(t["AM"]).int().cuda(),
                         torch.from_numpy(t["AK"]).int().cuda(), bf16(t["AV"]).cuda(),
                         bf16(t["B"]).cuda(), C, accumulate=accumulate, flags=flags)
    return C.cpu().double().numpy()


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_blockgroupcoo_builder_bit_exact(P, ixo, dtype):
    rng = ixo.Rng(8)
    cases = [(4, 4, 2, 2, 2, 0.5), (5, 6, 4, 4, 2, 0.5), (64, 48, 16, 16, 3, 0.3),
             (37, 53, 8, 4, 1, 0.2), (128, 128, 16, 16, 8, 0.1), (16, 16, 16, 16, 1, 1.0),
             (13, 33600, 8, 8, 3, 0.3)]  # > 4096 block columns: several pack tiles per block row
    for rows, cols, bm, bk, g, d in cases:
        a = ixo.synth_block_sparse_matrix(rng, rows, cols, bm, bk, d)
        a = bf16_round(a) if dtype == torch.bfloat16 else a.astype(np.float32).astype(np.float64)
        for gd in (0, 1):
            for gg in (g, 0):
                got = P.dense_to_blockgroupcoo(torch.from_numpy(a).to(dtype).cuda(), bm, bk, gg,
                                               gd)
                gsz = got.group_size
                want = ixo.dense_to_blockgroupcoo(a, bm, bk, gsz, gd)
                for k in ("AM", "AK", "mask"):
                    np.testing.assert_array_equal(getattr(got, k).cpu().numpy(),
                                                  want[k].astype(np.int64 if k != "mask" else np.uint8),
                                                  err_msg=f"{k} {rows}x{cols} {bm}x{bk} gd={gd}")
                np.testing.assert_array_equal(got.AV.double().cpu().numpy(), want["AV"])


def test_blockgroupcoo_tuner_matches_oracle(P, ixo):
    rng = ixo.Rng(2)
    a = bf16_round(ixo.synth_block_sparse_matrix(rng, 512, 512, 16, 16, 0.2))
    got = P.dense_to_blockgroupcoo(bf16(a).cuda(), 16, 16, 0)
    blocks = (np.abs(a).reshape(32, 16, 32, 16).sum(axis=(1, 3)) > 0)
    assert got.group_size == ixo.select(blocks.sum(axis=1).astype(np.int64))
    assert got.num_blocks == blocks.sum()


@pytest.mark.parametrize("kind", [1, 0])
def test_simt_path_acceptance_instances(P, ixo, kind):
    """acceptance.cpp make_blockgroupcoo_spmm (4x4 blocks): CUDA-core path."""
    for i in range(40 if kind else 20):
        t, expr, on, out = instances.make(ixo, "blockgroupcoo_spmm", kind, 1000 + i)
        t = {k: (bf16_round(x) if x.dtype == np.float64 else x) for k, x in t.items()}
        want = ixo.einsum(expr, t, on, out)
        got = run(P, t, out)
        if kind:
            np.testing.assert_array_equal(got.astype(np.int64), want)
        else:
            assert ixo.max_rel_error(want, got) <= TOL_BF16


def make16(ixo, seed, mb, kb, N, bdens, g, kind=1, empty_rows=()):
    rng = ixo.Rng(seed)
    a = ixo.synth_block_sparse_matrix(rng, mb * 16, kb * 16, 16, 16, bdens, kind)
    for r in empty_rows:
        a[r * 16:(r + 1) * 16] = 0
    b = ixo.synth_dense(rng, (kb, 16, N), kind)
    if kind == 0:
        a, b = bf16_round(a), bf16_round(b)
    f = ixo.dense_to_blockgroupcoo(a, 16, 16, g)
    t = {"AM": f["AM"], "AK": f["AK"], "AV": f["AV"], "B": b}
    return t, a, b


@pytest.mark.parametrize("N", [128, 256, 384, 512, 1024])
@pytest.mark.parametrize("g", [1, 3, 8])
def test_tcgen05_path_bit_exact_int(P, ixo, N, g):
    t, a, b = make16(ixo, N + g, 12, 9, N, 0.35, g)
    want = (a.reshape(12 * 16, 9 * 16).astype(np.int64) @
            b.reshape(9 * 16, N).astype(np.int64)).reshape(12, 16, N)
    got = run(P, t, np.zeros((12, 16, N)), flags=2)
    np.testing.assert_array_equal(got.astype(np.int64), want)
    got = run(P, t, np.zeros((12, 16, N)), flags=0)
    np.testing.assert_array_equal(got.astype(np.int64), want)


@pytest.mark.parametrize("N", [256, 512, 1024])
@pytest.mark.parametrize("g", [1, 4])
def test_tcgen05_rows_split_across_many_ctas(P, ixo, N, g):
    """Long block-rows (up to 200 blocks) with few rows: the balanced
    schedule splits each row across many CTAs and the last CTA to arrive
    sums the partials; exact on integer data, for `=` and `+=`, and the
    arrival counters are left clean for the next launch."""
    t, a, b = make16(ixo, 7 + N + g, 3, 200, N, 0.9, g, empty_rows=(1,))
    want = (a.reshape(3 * 16, 200 * 16).astype(np.int64) @
            b.reshape(200 * 16, N).astype(np.int64)).reshape(3, 16, N)
    for _ in range(2):
        got = run(P, t, np.full((3, 16, N), 5.0), accumulate=False, flags=2)
        np.testing.assert_array_equal(got.astype(np.int64), want)
    got = run(P, t, np.full((3, 16, N), 5.0), accumulate=True, flags=2)
    np.testing.assert_array_equal(got.astype(np.int64), want + 5)


def test_tcgen05_path_real_vs_oracle(P, ixo):
    t, a, b = make16(ixo, 77, 10, 14, 256, 0.3, 4, kind=0)
    want = ixo.einsum(EXPR, t, "C", np.zeros((10, 16, 256)))
    got = run(P, t, np.zeros((10, 16, 256)), flags=2)
    err = ixo.max_rel_error(want, got)
    assert err <= TOL_BF16
    assert err <= 1e-5  # bf16 products are exact in fp32; only fp32 summation error remains


def test_tcgen05_assign_accumulate_and_empty_rows(P, ixo):
    t, a, b = make16(ixo, 5, 20, 6, 128, 0.3, 2, empty_rows=(0, 1, 7, 8, 9, 19))
    ref = (a.reshape(320, 96) @ b.reshape(96, 128)).reshape(20, 16, 128)
    primed = ixo.synth_dense(ixo.Rng(3), (20, 16, 128), 1).astype(np.float64)
    got = run(P, t, primed, accumulate=True, flags=2)
    np.testing.assert_array_equal(got, primed + ref)
    got = run(P, t, primed, accumulate=False, flags=2)
    np.testing.assert_array_equal(got, ref)


def test_tcgen05_long_rows_many_stages(P, ixo):
    """Segments far longer than the smem ring and chunks with many segments."""
    t, a, b = make16(ixo, 11, 6, 200, 128, 0.9, 8)
    ref = (a.reshape(96, 3200).astype(np.int64) @ b.reshape(3200, 128).astype(np.int64))
    got = run(P, t, np.zeros((6, 16, 128)), flags=2)
    np.testing.assert_array_equal(got.astype(np.int64).reshape(96, 128), ref)
    t, a, b = make16(ixo, 12, 300, 4, 128, 0.05, 1)
    ref = (a.reshape(4800, 64).astype(np.int64) @ b.reshape(64, 128).astype(np.int64))
    got = run(P, t, np.zeros((300, 16, 128)), flags=2)
    np.testing.assert_array_equal(got.astype(np.int64).reshape(4800, 128), ref)


def test_tcgen05_mixed_long_and_short_rows(P, ixo):
    """Long block-rows (> 256 slots, many pipeline stages and segment
    queue entries) next to short and empty ones."""
    rng = ixo.Rng(21)
    a = ixo.synth_block_sparse_matrix(rng, 80, 6720, 16, 16, 0.7, 1)
    b = ixo.synth_dense(rng, (420, 16, 128), 1)
    a[32:48] = 0  # empty block-row 2
    for r in (1, 3):  # short rows (<= 256 slots) next to long rows 0 and 4
        a[r * 16:(r + 1) * 16, 16 * 40:] = 0
    f = ixo.dense_to_blockgroupcoo(a, 16, 16, 4)
    t = {"AM": f["AM"], "AK": f["AK"], "AV": f["AV"], "B": b}
    ref = (a.reshape(80, 6720).astype(np.int64) @ b.reshape(6720, 128).astype(np.int64))
    got = run(P, t, np.zeros((5, 16, 128)), flags=2)
    np.testing.assert_array_equal(got.astype(np.int64).reshape(80, 128), ref)
    rows = np.bincount(t["AM"], minlength=5) * t["AK"].shape[1]
    assert rows.max() > 256


def test_tcgen05_more_items_than_sms(P, ixo):
    """Far more work items than persistent CTAs: every CTA cycles its TMEM
    accumulator buffers many times."""
    t, a, b = make16(ixo, 31, 3000, 12, 256, 0.2, 2)
    ref = (a.reshape(48000, 192).astype(np.int64) @ b.reshape(192, 256).astype(np.int64))
    got = run(P, t, np.zeros((3000, 16, 256)), accumulate=False, flags=2)
    np.testing.assert_array_equal(got.astype(np.int64).reshape(48000, 256), ref)


def test_tcgen05_deterministic_and_row_block_invariant(P, ixo):
    """Real values: repeated runs are bit-identical, and evaluating a row
    slab alone (a different balanced CTA split, so block-rows that cross a
    CTA boundary are summed from different partials) agrees to fp32
    rounding."""
    t, a, b = make16(ixo, 41, 64, 40, 512, 0.3, 4, kind=0)
    full1 = run(P, t, np.zeros((64, 16, 512)), flags=2)
    full2 = run(P, t, np.zeros((64, 16, 512)), flags=2)
    np.testing.assert_array_equal(full1, full2)
    sel = t["AM"] >= 32
    sub = {"AM": t["AM"][sel] - 32, "AK": t["AK"][sel], "AV": t["AV"][sel], "B": t["B"]}
    part = run(P, sub, np.zeros((32, 16, 512)), flags=2)
    np.testing.assert_allclose(part, full1[32:], rtol=1e-6, atol=1e-5)


def test_tcgen05_unsorted_groups(P, ixo):
    g_np = np.random.default_rng(4)
    G, g, MB, KB, N = 60, 2, 7, 9, 128
    t = {"AM": g_np.integers(0, MB, G).astype(np.int64),
         "AK": g_np.integers(0, KB, (G, g)).astype(np.int64),
         "AV": g_np.integers(-4, 5, (G, g, 16, 16)).astype(np.int64),
         "B": g_np.integers(-4, 5, (KB, 16, N)).astype(np.int64)}
    want = ixo.einsum(EXPR, t, "C", np.zeros((MB, 16, N), np.int64))
    got = run(P, {k: v.astype(np.float64) if k in ("AV", "B") else v for k, v in t.items()},
              np.zeros((MB, 16, N)))
    np.testing.assert_array_equal(got.astype(np.int64), want)


def test_tcgen05_index_errors(P, ixo):
    t, a, b = make16(ixo, 3, 4, 4, 128, 0.5, 2)
    t = dict(t)
    t["AK"] = t["AK"].copy()
    t["AK"].flat[3] = 9
    with pytest.raises(P.IndexRangeError) as e:
        run(P, t, np.zeros((4, 16, 128)), flags=2)
    assert str(e.value) == ("index tensor AK value 9 at position [3] out of range for dim 0 of "
                            "B (extent 4)")
    t, a, b = make16(ixo, 3, 4, 4, 128, 0.5, 2)
    t = dict(t)
    t["AM"] = t["AM"].copy()
    t["AM"][-1] = 4
    with pytest.raises(P.IndexRangeError) as e:
        run(P, t, np.zeros((4, 16, 128)), flags=2)
    assert "index tensor AM value 4" in str(e.value) and "(extent 4)" in str(e.value)


def test_cfg2_full_size_slab_vs_oracle(P, ixo):
    """BASELINE configs[1] (8192^2, 16x16 blocks, 10% blocks, N=512): device
    builder + tcgen05 SpMM; the oracle checks the first 6 block-rows and the
    rest are checked against an exact integer-valued run (column sums)."""
    from paper_2510_17505_b200 import synth as S
    rng = S.Rng(1)
    B = S.synth_dense(rng, (512, 16, 512), S.REAL, torch.bfloat16)
    A = S.synth_block_sparse_matrix(rng, 8192, 8192, 16, 16, 0.10, S.REAL, torch.bfloat16)
    fmt = P.dense_to_blockgroupcoo(A.cuda(), 16, 16, 0)
    assert fmt.group_size == 8
    C = torch.empty((512, 16, 512), device="cuda")
    P.spmm_blockgroupcoo(fmt.AM, fmt.AK, fmt.AV, B.cuda(), C, accumulate=False, flags=2)
    AM = fmt.AM.cpu().numpy()
    sel = AM < 6
    t = {"AM": AM[sel].astype(np.int64), "AK": fmt.AK.cpu().numpy()[sel].astype(np.int64),
         "AV": fmt.AV.double().cpu().numpy()[sel], "B": B.double().numpy()}
    want = ixo.einsum(EXPR, t, "C", np.zeros((6, 16, 512)))
    assert ixo.max_rel_error(want, C[:6].double().cpu().numpy()) <= TOL_BF16
    # whole-output check: C summed over n equals A @ (B summed over n) in fp64
    bs = B.double().sum(dim=2).reshape(8192)
    ref = (A.double() @ bs).reshape(512, 16)
    got = C.double().sum(dim=2).cpu()
    rel = ((got - ref).abs() / torch.maximum(ref.abs(), torch.ones_like(ref))).max().item()
    assert rel <= 1e-3


@pytest.mark.parametrize("nchunks", [0, 1, 3, 8])  # 0: automatic
def test_host_buffer_pipeline_bit_identical(P, ixo, nchunks):
    """ixb_spmm_blockgroupcoo_host (host buffers, chunked H2D/kernel/D2H on
    three streams) equals the device-buffer call bit for bit on integer
    data (real data: to fp32 rounding — each chunk is its own balanced
    launch), for `=` and `+=`, and reports index errors with the same
    message."""
    tr, _, _ = make16(ixo, 52, 40, 30, 256, 0.3, 4, kind=0, empty_rows=(0, 7, 39))
    AMr, AKr = torch.from_numpy(tr["AM"]).int(), torch.from_numpy(tr["AK"]).int()
    AVr, Br = bf16(tr["AV"]), bf16(tr["B"])
    refr = torch.zeros((40, 16, 256), device="cuda")
    P.spmm_blockgroupcoo(AMr.cuda(), AKr.cuda(), AVr.cuda(), Br.cuda(), refr, accumulate=False)
    outr = torch.empty((40, 16, 256)).pin_memory()
    P.spmm_blockgroupcoo_host(AMr, AKr, AVr, Br, outr, accumulate=False, nchunks=nchunks)
    torch.testing.assert_close(outr, refr.cpu(), rtol=1e-6, atol=1e-5)
    t, a, b = make16(ixo, 51, 40, 30, 256, 0.3, 4, kind=1, empty_rows=(0, 7, 39))
    AM = torch.from_numpy(t["AM"]).int()
    AK = torch.from_numpy(t["AK"]).int()
    AV, B = bf16(t["AV"]), bf16(t["B"])
    ref = torch.zeros((40, 16, 256), device="cuda")
    P.spmm_blockgroupcoo(AM.cuda(), AK.cuda(), AV.cuda(), B.cuda(), ref, accumulate=False)
    out = torch.full((40, 16, 256), 7.0).pin_memory()
    P.spmm_blockgroupcoo_host(AM.pin_memory(), AK.pin_memory(), AV.pin_memory(), B.pin_memory(),
                              out, accumulate=False, nchunks=nchunks)
    assert torch.equal(out, ref.cpu())
    primed = torch.randn(40, 16, 256)
    out = primed.clone().pin_memory()
    P.spmm_blockgroupcoo_host(AM, AK, AV, B, out, accumulate=True, nchunks=nchunks)
    ref2 = primed.cuda()
    P.spmm_blockgroupcoo(AM.cuda(), AK.cuda(), AV.cuda(), B.cuda(), ref2, accumulate=True)
    assert torch.equal(out, ref2.cpu())
    bad = AK.clone()
    bad.view(-1)[5] = 30
    with pytest.raises(P.IndexRangeError) as e:
        P.spmm_blockgroupcoo_host(AM, bad, AV, B, out, accumulate=False, nchunks=nchunks)
    assert str(e.value) == ("index tensor AK value 30 at position [5] out of range for dim 0 "
                            "of B (extent 30)")


def test_host_buffer_pipeline_groupcoo_and_unsorted(P, ixo):
    rng = ixo.Rng(8)
    A = ixo.synth_sparse_matrix(rng, 300, 200, 0.05, 1)
    Bn = ixo.synth_dense(rng, (200, 64), 1)
    f = ixo.coo_to_groupcoo(300, 200, *ixo.dense_to_coo(A), 0, 4)
    AM, AK = torch.from_numpy(f["AM"]).int(), torch.from_numpy(f["AK"]).int()
    AV, B = torch.from_numpy(f["AV"]).float(), torch.from_numpy(Bn).float()
    want = torch.from_numpy(A.astype(np.float32) @ Bn.astype(np.float32))
    for nch in (0, 1, 5):  # 0: automatic
        out = torch.empty(300, 64)
        P.spmm_groupcoo_host(AM, AK, AV, B, out, accumulate=False, nchunks=nch)
        assert torch.equal(out, want)
    perm = torch.from_numpy(np.random.default_rng(2).permutation(AM.numel()))
    out = torch.empty(300, 64)
    P.spmm_groupcoo_host(AM[perm], AK[perm], AV[perm], B, out, accumulate=False, nchunks=4)
    assert torch.equal(out, want)
