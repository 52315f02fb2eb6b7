"""CPU checks of the on-disk format layer: the
MatrixMarket parser in libixb (host C++) against the reference's
load_matrix_market (matrix_market.cpp:30-159) on every branch and error
message, and .ixt headers / errors against tensor.cpp:158-225. No device
calls."""
import json
import os
import struct

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "io")
MTX = sorted(f for f in os.listdir(GOLD) if f.endswith(".mtx"))


@pytest.fixture(scope="module")
def P():
    import paper_2510_17505_b200 as P
    try:
        P.lib()
    except Exception as e:  # libixb not built
        pytest.skip(str(e))
    return P


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.int64) if a.dtype == np.float64 else a


@pytest.mark.parametrize("name", MTX)
def test_matrix_market_matches_reference(P, name):
    from oracle import ref
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "ref_io")):
        pytest.skip("reference not built here")
    path = os.path.join(GOLD, name)
    got = P.read_matrix_market_host(path)
    want = ref.load_matrix_market(path)
    assert got.keys() == want.keys()
    for k in want:
        if isinstance(want[k], np.ndarray):
            assert got[k].dtype == want[k].dtype and got[k].shape == want[k].shape, k
            np.testing.assert_array_equal(bits(got[k]), bits(want[k]))
        else:
            assert got[k] == want[k], k


def test_matrix_market_semantics(P):
    """Reader rules, independent of the reference binary: one-based ->
    zero-based, duplicates kept, symmetric mirrored, skew negated, pattern 1,
    array files column-major."""
    d = P.read_matrix_market_host(os.path.join(GOLD, "general_real.mtx"))
    assert (d["rows"], d["cols"]) == (6, 5) and len(d["row"]) == 9
    assert list(d["row"][:2]) == [2, 0] and d["values"][0] == 1.5e-3
    assert d["values"][-1] == 4.0 and d["row"][-1] == 0  # duplicate (1,1) kept
    d = P.read_matrix_market_host(os.path.join(GOLD, "integer_sym.mtx"))
    assert d["values"].dtype == np.int64 and len(d["row"]) == 8  # 2 off-diagonals mirrored
    d = P.read_matrix_market_host(os.path.join(GOLD, "pattern_skew.mtx"))
    np.testing.assert_array_equal(d["values"], [1, -1, 1, -1, 1, -1])
    d = P.read_matrix_market_host(os.path.join(GOLD, "array_general.mtx"))["dense"]
    np.testing.assert_array_equal(d, [[1, 0, 0.3, 8], [0, 0, 0, 0], [-2.5, 4, 0, -1]])
    d = P.read_matrix_market_host(os.path.join(GOLD, "array_skew.mtx"))["dense"]
    np.testing.assert_array_equal(d, -d.T)


def test_matrix_market_errors_match_reference(P):
    msgs = json.load(open(os.path.join(GOLD, "bad", "errors.json")))
    assert len(msgs) >= 14
    for name, msg in msgs.items():
        path = os.path.join(GOLD, "bad", name)
        with pytest.raises(P.IoError) as e:
            P.read_matrix_market_host(path)
        assert str(e.value) == msg.replace("<path>", path), name
    missing = os.path.join(GOLD, "bad", "does_not_exist.mtx")
    with pytest.raises(P.IoError, match="cannot open: " + missing):
        P.read_matrix_market_host(missing)


def test_ixt_info_on_reference_files(P):
    contents = np.load(os.path.join(GOLD, "ixt", "contents.npz"))
    for name in contents.files:
        kind, shape = P.ixt_info(os.path.join(GOLD, "ixt", name + ".ixt"))
        assert shape == list(contents[name].shape)
        assert kind == (1 if contents[name].dtype == np.int64 else 0)


def test_ixt_header_errors(P, tmp_path):
    """load_tensor's header checks and messages (tensor.cpp:197-214)."""
    def write(name, payload):
        p = str(tmp_path / name)
        with open(p, "wb") as f:
            f.write(payload)
        return p

    hdr = struct.pack("<IIII", 0x4E545849, 1, 0, 1)
    cases = {
        "magic.ixt": (struct.pack("<IIII", 0x12345678, 1, 0, 1), "bad magic in "),
        "version.ixt": (struct.pack("<IIII", 0x4E545849, 2, 0, 1), "unsupported version in "),
        "kind.ixt": (struct.pack("<IIII", 0x4E545849, 1, 3, 1), "bad element kind in "),
        "rank0.ixt": (struct.pack("<IIII", 0x4E545849, 1, 0, 0), "bad rank in "),
        "rank17.ixt": (struct.pack("<IIII", 0x4E545849, 1, 0, 17), "bad rank in "),
        "negdim.ixt": (hdr + struct.pack("<q", -1), "negative dimension in "),
        "short.ixt": (hdr[:10], "truncated tensor file: "),
    }
    for name, (payload, msg) in cases.items():
        p = write(name, payload)
        with pytest.raises(P.IoError) as e:
            P.ixt_info(p)
        assert str(e.value) == msg + p
