"""CPU checks of the drop-in boundary: libixb.so loads and exports every
symbol declared in include/ixb.h; host-side logic (parser, workload matcher,
shard planner) behaves like the reference. No device calls."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "ixb.h")).read()
    return sorted(set(re.findall(r"^[A-Za-z_][\w \*]*?\b(ixb_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    import paper_2510_17505_b200 as P
    lib = P.lib()
    decl = declared_symbols()
    assert len(decl) >= 25
    out = subprocess.run(["nm", "-D", "--defined-only", P.lib_path()], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (ixb_\w+)", out))
    missing = [s for s in decl if s not in exported]
    assert not missing, missing
    for s in decl:
        getattr(lib, s)
    assert set(P.abi.EXPORTED) == set(decl)  # every declared entry point has a ctypes signature


def test_library_is_sm100a_only():
    import paper_2510_17505_b200 as P
    out = subprocess.run(["cuobjdump", "--list-elf", P.lib_path()], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_parser_matches_reference_errors(ref):
    from paper_2510_17505_b200.executor import parse
    from paper_2510_17505_b200 import ParseError
    t = {"A": np.array([1, 2], np.int64)}
    for bad in ["C[i] = A[i", "C[i] A[i]", "C[A[B[i]]] = A[i]", "C[i] = A[i] *", "C[] = A[i]",
                "C[i] = A[i] extra"]:
        with pytest.raises(ParseError) as e1:
            parse(bad)
        with pytest.raises(ref.RefError) as e2:
            ref.run(t, bad, "C", np.zeros(2, np.int64), "oracle")
        assert e2.value.code == 2
        assert str(e1.value) == str(e2.value), bad


def test_workload_matcher():
    from paper_2510_17505_b200.executor import match_workload, parse
    import instances
    for name, expr in instances.EXPR.items():
        wl, bind = match_workload(parse(expr))
        assert wl == name, (name, wl)
    wl, bind = match_workload(parse("Y[AM[r],k] = VV[r,s] * D[AK2[r,s],k]"))
    assert wl == "groupcoo_spmm" and bind["B"] == "D" and bind["AK"] == "AK2"
    wl, _ = match_workload(
        parse("Z[b,CGI[p,q],w] += CGV[p,q] * X[b,CGJ[p,q],u] * Y[b,CGK[p,q]] * W[CGL[p],u,w]"))
    assert wl == "grouped_tp_shared"
    assert match_workload(parse("C[y,x] = A[y,r] * B[r,x]"))[0] is None
    assert match_workload(parse("C[AM[p],n] += AV[p,q] * B[AK[p,q],m]"))[0] is None


def test_shard_planner_cuts_at_row_boundaries():
    import paper_2510_17505_b200 as P
    g = np.random.default_rng(0)
    am = np.sort(g.integers(0, 50, 1000)).astype(np.int32)
    for parts in (1, 2, 3, 4, 8):
        b = P.shard_groups(am, parts)
        assert b[0] == 0 and b[-1] == len(am) and np.all(np.diff(b) >= 0)
        for cut in b[1:-1]:
            assert cut in (0, len(am)) or am[cut] != am[cut - 1]
        sizes = np.diff(b)
        assert sizes.max() <= len(am) / parts + np.bincount(am).max() + 1
