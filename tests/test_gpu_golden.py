"""GPU runs of the reference's own golden fixtures (tests/golden, produced by
the unmodified reference): every hot-path corpus spec through the drop-in
execute_mode("b200", ...), and the BASELINE config slabs through the device
builders + kernels. Integer-valued fixtures must match bit-for-bit."""
import glob
import os
import zlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CORPUS = sorted(glob.glob(os.path.join(GOLDEN, "corpus_*.npz")))


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_17505_b200 as P
    P.lib()
    return P


@pytest.mark.parametrize("path", CORPUS, ids=[os.path.basename(p) for p in CORPUS])
def test_corpus_through_execute_mode(P, ixo, path):
    d = np.load(path)
    tensors = {k[2:]: d[k] for k in d.files if k.startswith("t_")}
    mo = P.execute_mode("b200", str(d["expr"]), tensors, str(d["out_name"]), d["out"])
    want = d["res_oracle"]
    if want.dtype == np.int64:
        np.testing.assert_array_equal(mo.result.astype(np.int64), want)
    else:
        assert ixo.max_rel_error(want, mo.result) <= P.device_tolerance(str(d["expr"]))


@pytest.mark.parametrize("path", CORPUS, ids=[os.path.basename(p) for p in CORPUS])
def test_corpus_real_values_at_device_tolerance(P, ixo, path):
    """The corpus specs with real values (seeded, rounded to the device's value
    dtype first) against the fp64 oracle at the per-path tolerance: 1e-5 for
    the fp32 GroupCOO / COO SpMM, 1e-2 for bf16 operands."""
    d = np.load(path)
    expr = str(d["expr"])
    tol = P.device_tolerance(expr)
    fp32 = tol < 1e-3
    rng = np.random.default_rng(zlib.crc32(os.path.basename(path).encode()))
    idx = {"AM", "AK", "MAPX", "MAPY", "MAPZ", "CGL", "CGI", "CGJ", "CGK"}
    tensors = {}
    for k in d.files:
        if not k.startswith("t_"):
            continue
        name, v = k[2:], d[k]
        if name in idx:
            tensors[name] = v
            continue
        r = rng.uniform(-1.0, 1.0, v.shape) * (v != 0 if name in ("AV", "CGV", "MAPV") else 1)
        dt = torch.float32 if fp32 or name in ("CGV", "MAPV") else torch.bfloat16
        tensors[name] = torch.from_numpy(r).to(dt).double().numpy()
    out = rng.uniform(-1.0, 1.0, np.asarray(d["out"]).shape)
    want = ixo.einsum(expr, tensors, str(d["out_name"]), out)
    mo = P.execute_mode("b200", expr, tensors, str(d["out_name"]), out)
    assert ixo.max_rel_error(want, mo.result) <= tol


@pytest.mark.parametrize("tag,kind", [("real", 0), ("int", 1)])
def test_cfg1_slab_device(P, ixo, tag, kind):
    d = np.load(os.path.join(GOLDEN, f"cfg1_slab_{tag}.npz"))
    rng = ixo.Rng(1)
    B = ixo.synth_dense(rng, (4096, 128), kind).astype(np.float32)
    A = ixo.synth_sparse_matrix(rng, 64, 4096, 0.01, kind).astype(np.float32)
    fmt = P.dense_to_groupcoo(torch.from_numpy(A).cuda(), g=0)
    assert fmt.group_size == int(d["g"])
    np.testing.assert_array_equal(fmt.AM.cpu().numpy(), d["AM"])
    np.testing.assert_array_equal(fmt.AK.cpu().numpy(), d["AK"])
    C = torch.zeros((64, 128), device="cuda")
    P.spmm_groupcoo(fmt.AM, fmt.AK, fmt.AV, torch.from_numpy(B).cuda(), C, flags=2)
    got = C.double().cpu().numpy()
    if kind:
        np.testing.assert_array_equal(got.astype(np.int64), d["res"])
    else:  # fp32-rounded inputs vs the reference's fp64 result
        assert ixo.max_rel_error(d["res"], got) <= 1e-5


@pytest.mark.parametrize("tag,kind", [("real", 0), ("int", 1)])
def test_cfg2_slab_device(P, ixo, tag, kind):
    d = np.load(os.path.join(GOLDEN, f"cfg2_slab_{tag}.npz"))
    rng = ixo.Rng(1)
    B = ixo.synth_dense(rng, (512, 16, 512), kind)
    A = ixo.synth_block_sparse_matrix(rng, 32, 8192, 16, 16, 0.10, kind)
    bf = lambda x: torch.from_numpy(np.asarray(x, np.float64)).to(torch.bfloat16).cuda()
    fmt = P.dense_to_blockgroupcoo(bf(A), 16, 16, 8)
    np.testing.assert_array_equal(fmt.AM.cpu().numpy(), d["AM"])
    np.testing.assert_array_equal(fmt.AK.cpu().numpy(), d["AK"])
    C = torch.zeros((2, 16, 512), device="cuda")
    P.spmm_blockgroupcoo(fmt.AM, fmt.AK, fmt.AV, bf(B), C, flags=2)
    got = C.double().cpu().numpy()
    if kind:
        np.testing.assert_array_equal(got.astype(np.int64), d["res"])
    else:
        # parity protocol: round the inputs to bf16 first, run
        # the fp64 oracle on the rounded values, compare within 1e-2
        r = lambda x: torch.from_numpy(np.asarray(x)).to(torch.bfloat16).double().numpy()
        bg = ixo.dense_to_blockgroupcoo(r(A), 16, 16, 8)
        t = {"AM": bg["AM"], "AK": bg["AK"], "AV": bg["AV"], "B": r(B)}
        want = ixo.einsum("C[AM[p],bm,n] += AV[p,q,bm,bk] * B[AK[p,q],bk,n]", t, "C",
                          np.zeros((2, 16, 512)))
        assert ixo.max_rel_error(want, got) <= 1e-2
        # and the rounding of the inputs is the only departure from the fixture
        scale = np.abs(bg["AV"]).sum() / 2 * 16 * 2 ** -8
        assert np.abs(d["res"] - got).max() <= scale
