"""GPU checks of the on-disk format layer: .ixt
files load into / save from device buffers bit-exactly against files the
reference wrote (tensor.cpp:176-225); MatrixMarket lands on the device as
the host parser reads it; and `convert` (device builders) reproduces the
reference's cmd_convert directories (driver.cpp:403-514) byte for byte
(arrays) and key for key (manifest). Fixtures: tests/golden/io
(make_io_golden.py)."""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "io")


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_17505_b200 as P
    P.lib()
    return P


def contents():
    return np.load(os.path.join(GOLD, "ixt", "contents.npz"))


def test_load_reference_ixt(P):
    c = contents()
    for name in c.files:
        want = c[name]
        path = os.path.join(GOLD, "ixt", name + ".ixt")
        got = P.load_ixt(path)  # file's own 8-byte type
        assert got.dtype == (torch.int64 if want.dtype == np.int64 else torch.float64)
        np.testing.assert_array_equal(got.cpu().numpy(), want)
        if want.dtype == np.float64:
            np.testing.assert_array_equal(P.load_ixt(path, torch.float32).cpu().numpy(),
                                          want.astype(np.float32))
            assert torch.equal(P.load_ixt(path, torch.bfloat16).cpu(),
                               torch.from_numpy(want).to(torch.bfloat16))
    idx = P.load_ixt(os.path.join(GOLD, "ixt", "idx.ixt"), torch.int32)
    np.testing.assert_array_equal(idx.cpu().numpy(), c["idx"])
    with pytest.raises(P.ShapeError, match=r"position \[0\] does not fit the int32"):
        P.load_ixt(os.path.join(GOLD, "ixt", "int2.ixt"), torch.int32)
    with pytest.raises(P.IxbError, match="cannot be loaded as an integer dtype"):
        P.load_ixt(os.path.join(GOLD, "ixt", "real3.ixt"), torch.int32)


def test_save_matches_reference_bytes(P, tmp_path):
    c = contents()
    for name in c.files:
        t = torch.from_numpy(c[name]).cuda()
        out = str(tmp_path / (name + ".ixt"))
        P.save_ixt(out, t)
        assert open(out, "rb").read() == open(os.path.join(GOLD, "ixt", name + ".ixt"), "rb").read()
    # narrow device dtypes widen exactly
    t = torch.arange(-5, 7, dtype=torch.int32, device="cuda").reshape(3, 4)
    P.save_ixt(str(tmp_path / "i32.ixt"), t)
    assert torch.equal(P.load_ixt(str(tmp_path / "i32.ixt")).cpu(), t.long().cpu())
    b = torch.tensor([1.5, -2.25, 3e-3], dtype=torch.bfloat16, device="cuda")
    P.save_ixt(str(tmp_path / "bf.ixt"), b)
    assert torch.equal(P.load_ixt(str(tmp_path / "bf.ixt")).cpu(), b.double().cpu())
    with pytest.raises(P.IoError, match="refusing to save rank-0 tensor"):
        P.save_ixt(str(tmp_path / "s.ixt"), torch.tensor(1.0, device="cuda"))


def test_chunked_roundtrip(P, tmp_path):
    """Payloads larger than the 32 MiB staging chunks (both directions)."""
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(9_000_123, generator=g, device="cuda", dtype=torch.float64)
    p = str(tmp_path / "big.ixt")
    P.save_ixt(p, x)
    assert os.path.getsize(p) == 16 + 8 + 8 * x.numel()
    assert torch.equal(P.load_ixt(p), x)
    assert torch.equal(P.load_ixt(p, torch.float32), x.float())
    i = torch.randint(0, 2**31 - 1, (5_000_001,), generator=g, device="cuda", dtype=torch.int64)
    i[4_500_000] = 2**31  # out of int32 range, in the second chunk
    P.save_ixt(p, i)
    with pytest.raises(P.ShapeError, match=r"position \[4500000\]"):
        P.load_ixt(p, torch.int32)


@pytest.mark.parametrize("name", sorted(f for f in os.listdir(GOLD) if f.endswith(".mtx")))
def test_matrix_market_to_device(P, name):
    path = os.path.join(GOLD, name)
    host = P.read_matrix_market_host(path)
    for dt in (torch.float64, torch.float32):
        got = P.load_matrix_market(path, dt)
        if "dense" in host:
            assert torch.equal(got.cpu(), torch.from_numpy(host["dense"]).to(dt))
        else:
            assert (got.rows, got.cols) == (host["rows"], host["cols"])
            np.testing.assert_array_equal(got.row.cpu().numpy(), host["row"])
            np.testing.assert_array_equal(got.col.cpu().numpy(), host["col"])
            assert torch.equal(got.values.cpu(), torch.from_numpy(host["values"]).to(dt))


CASES = json.load(open(os.path.join(GOLD, "convert", "cases.json")))


@pytest.mark.parametrize("case", sorted(CASES))
def test_convert_matches_reference(P, case, tmp_path):
    c = CASES[case]
    ref_dir = os.path.join(GOLD, "convert", case)
    out = str(tmp_path / case)
    man = P.convert(os.path.join(GOLD, c["input"]), out, c["format"], c["g"], c["group_dim"],
                    c["block"])
    want = json.load(open(os.path.join(ref_dir, "manifest.json")))
    got = json.load(open(os.path.join(out, "manifest.json")))
    assert got == want
    assert man == want
    for name, file in want["arrays"].items():
        a = open(os.path.join(out, file), "rb").read()
        b = open(os.path.join(ref_dir, file), "rb").read()
        assert a == b, f"{case}: {name} differs"


def test_load_format_then_evaluate(P):
    """A reference-converted GroupCOO directory evaluates on K3 like the
    oracle (C[AM[p],n] += AV[p,q] * B[AK[p,q],n], fp32 tolerance 1e-5)."""
    from oracle import ixo
    fmt, man = P.load_format(os.path.join(GOLD, "convert", "random_auto_d0"), torch.float32)
    assert man["format"] == "groupcoo" and fmt.group_size == man["g"]
    rng = ixo.Rng(9)
    B = ixo.synth_dense(rng, (200, 48))
    C = torch.zeros((300, 48), device="cuda")
    P.spmm_groupcoo(fmt.AM, fmt.AK, fmt.AV, torch.from_numpy(B).float().cuda(), C)
    t = {"AM": fmt.AM.cpu().numpy().astype(np.int64), "AK": fmt.AK.cpu().numpy().astype(np.int64),
         "AV": fmt.AV.double().cpu().numpy(), "B": B.astype(np.float32).astype(np.float64)}
    want = ixo.einsum("C[AM[p],n] += AV[p,q] * B[AK[p,q],n]", t, "C", np.zeros((300, 48)))
    assert ixo.max_rel_error(want, C.double().cpu().numpy()) <= 1e-5
    bg, man = P.load_format(os.path.join(GOLD, "convert", "general_bgcoo"))
    assert man["format"] == "blockgroupcoo" and list(bg.AV.shape[2:]) == man["block"]


MEASURE = json.load(open(os.path.join(GOLD, "convert_measure", "cases.json")))


@pytest.mark.parametrize("case", sorted(MEASURE))
def test_convert_measure_like_reference(P, case, tmp_path):
    """`convert --measure` (driver.cpp:434-460): candidates scored by measured
    time on the device. The reference's directory pins the manifest layout,
    g* and the candidate list; scores are timings, so the chosen g must be
    the first minimum of OUR scores, and the arrays must equal a plain
    `groupcoo` conversion at that g byte for byte."""
    c = MEASURE[case]
    want = json.load(open(os.path.join(GOLD, "convert_measure", case, "manifest.json")))
    out = str(tmp_path / case)
    man = P.convert(os.path.join(GOLD, c["input"]), out, c["format"], c["g"], c["group_dim"],
                    c["block"], measure=True, measure_repeats=3)
    assert list(man) == list(want)
    assert list(man["tuner"]) == list(want["tuner"])
    assert man["tuner"]["scoredBy"] == want["tuner"]["scoredBy"] == "measuredMs"
    assert man["tuner"]["gStar"] == want["tuner"]["gStar"]
    assert [x["g"] for x in man["tuner"]["candidates"]] == \
        [x["g"] for x in want["tuner"]["candidates"]]
    scores = [(x["g"], x["score"]) for x in man["tuner"]["candidates"]]
    assert all(s > 0 for _, s in scores)
    first_min = min(scores, key=lambda gs: gs[1])  # min() keeps the first on a tie
    assert man["g"] == first_min[0]
    plain = str(tmp_path / "plain")
    P.convert(os.path.join(GOLD, c["input"]), plain, "groupcoo", man["g"], c["group_dim"])
    for name, file in man["arrays"].items():
        assert open(os.path.join(out, file), "rb").read() == \
            open(os.path.join(plain, file), "rb").read(), name
    if man["g"] == want["g"]:  # same choice as the reference run: same arrays
        for name, file in want["arrays"].items():
            assert open(os.path.join(out, file), "rb").read() == \
                open(os.path.join(GOLD, "convert_measure", case, file), "rb").read(), name


def test_tune_measured_rejects_column_grouping(P):
    coo = P.load_matrix_market(os.path.join(GOLD, "random_300x200.mtx"), torch.float64)
    with pytest.raises(ValueError):
        P.tune_measured(coo, group_dim=1)
