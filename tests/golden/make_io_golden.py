"""Generates tests/golden/io/: MatrixMarket inputs covering every branch of
the reference reader (matrix_market.cpp:30-159), malformed files for its
error messages, .ixt files written by the reference's save_tensor
(tensor.cpp:176-195), and `ixsum convert` directories made by the
reference's cmd_convert (driver.cpp:403-514).

Run here (needs /root/reference compiled into oracle/_ref):
    python tests/golden/make_io_golden.py
The outputs are committed; the GPU box only reads them.
"""
import json
import os
import shutil
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "io")

VALID = {
    "general_real.mtx": """%%MatrixMarket matrix coordinate real general
% comment line, then a blank line

6 5 9
3 2 1.5e-3
1 1 -2
6 5 3.
3 2 0.25
2 4 7.125
1 5 -0.5
5 1 1e2
4 3 2.0000001
1 1 4
""",
    "integer_sym.mtx": """%%MatrixMarket matrix coordinate integer symmetric
5 5 6
1 1 3
2 1 -4
3 3 5
5 2 7
4 4 1
5 5 -2
""",
    "pattern_skew.mtx": """%%MatrixMarket Matrix Coordinate Pattern Skew-Symmetric
4 4 3
2 1
4 2
3 1
""",
    "array_general.mtx": """%%MatrixMarket matrix array real general
3 4
1.0
0
-2.5
0
0
4
3e-1
0
0
8
0
-1
""",
    "array_sym_int.mtx": """%%MatrixMarket matrix array integer symmetric
3 3
1
-2
0
5
3
9
""",
    "array_skew.mtx": """%%MatrixMarket matrix array real skew-symmetric
3 3
0
1.5
-2
0
4.25
0
""",
}

BAD = {
    "bad_header.mtx": "%%MatrixMarkt matrix coordinate real general\n1 1 0\n",
    "bad_format.mtx": "%%MatrixMarket matrix sparse real general\n1 1 0\n",
    "bad_field.mtx": "%%MatrixMarket matrix coordinate complex general\n1 1 0\n",
    "bad_symmetry.mtx": "%%MatrixMarket matrix coordinate real hermitian\n1 1 0\n",
    "missing_size.mtx": "%%MatrixMarket matrix coordinate real general\n% only comments\n",
    "bad_size.mtx": "%%MatrixMarket matrix coordinate real general\n3 x 2\n",
    "truncated.mtx": "%%MatrixMarket matrix coordinate real general\n3 3 3\n1 1 1\n2 2 2\n",
    "out_of_bounds.mtx": "%%MatrixMarket matrix coordinate real general\n3 3 1\n4 1 1\n",
    "bad_entry.mtx": "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 x 1\n",
    "bad_real.mtx": "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 1 abc\n",
    "bad_int.mtx": "%%MatrixMarket matrix coordinate integer general\n3 3 1\n1 1 x\n",
    "array_pattern.mtx": "%%MatrixMarket matrix array pattern general\n2 2\n",
    "array_nonsquare_sym.mtx": "%%MatrixMarket matrix array real symmetric\n2 3\n1\n2\n3\n4\n",
    "array_truncated.mtx": "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n",
    "empty.mtx": "",
}


def random_mtx(path, rows, cols, n, seed):
    g = np.random.default_rng(seed)
    r = g.integers(1, rows + 1, n)
    c = g.integers(1, cols + 1, n)
    v = g.standard_normal(n)
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real general\n")
        f.write(f"{rows} {cols} {n}\n")
        for i in range(n):
            f.write(f"{r[i]} {c[i]} {float(v[i])!r}\n")


def main():
    if not ref.available():
        raise SystemExit("oracle/_ref not built (make -C oracle)")
    shutil.rmtree(OUT, ignore_errors=True)
    os.makedirs(os.path.join(OUT, "bad"))
    for name, text in VALID.items():
        with open(os.path.join(OUT, name), "w") as f:
            f.write(text)
    random_mtx(os.path.join(OUT, "random_300x200.mtx"), 300, 200, 2500, 7)
    errors = {}
    for name, text in BAD.items():
        p = os.path.join(OUT, "bad", name)
        with open(p, "w") as f:
            f.write(text)
        try:
            ref.load_matrix_market(p)
            raise SystemExit(f"{name}: expected an error")
        except ref.RefError as e:
            errors[name] = str(e).replace(p, "<path>")
    with open(os.path.join(OUT, "bad", "errors.json"), "w") as f:
        json.dump(errors, f, indent=1, sort_keys=True)

    # reference-written .ixt files (+ their contents for the GPU box)
    g = np.random.default_rng(3)
    tensors = {"real3": g.standard_normal((3, 4, 5)),
               "int2": g.integers(-2**40, 2**40, (7, 3)).astype(np.int64),
               "idx": g.integers(0, 1000, (11,)).astype(np.int64),
               "empty": np.zeros((0, 4)),
               "dense_in": np.where(g.random((6, 8)) < 0.4, g.standard_normal((6, 8)), 0.0)}
    os.makedirs(os.path.join(OUT, "ixt"))
    for k, v in tensors.items():
        ref.save_tensor(os.path.join(OUT, "ixt", k + ".ixt"), v)
    np.savez(os.path.join(OUT, "ixt", "contents.npz"), **tensors)

    # reference convert directories
    cases = {
        "general_coo": ("general_real.mtx", "coo", 1, 0, None),
        "general_g2_d0": ("general_real.mtx", "groupcoo", 2, 0, None),
        "general_g3_d1": ("general_real.mtx", "groupcoo", 3, 1, None),
        "general_auto": ("general_real.mtx", "auto", 1, 0, None),
        "general_bgcoo": ("general_real.mtx", "blockgroupcoo", 2, 0, [2, 2]),
        "intsym_auto": ("integer_sym.mtx", "auto", 1, 0, None),
        "skew_g2": ("pattern_skew.mtx", "groupcoo", 2, 0, None),
        "array_auto": ("array_general.mtx", "auto", 1, 1, None),
        "random_auto_d0": ("random_300x200.mtx", "auto", 1, 0, None),
        "random_auto_d1": ("random_300x200.mtx", "auto", 1, 1, None),
        "skew_bgcoo_d1": ("pattern_skew.mtx", "blockgroupcoo", 2, 1, [2, 2]),
        "intsym_bgcoo_ragged": ("integer_sym.mtx", "blockgroupcoo", 2, 0, [2, 3]),
        "ixt_dense_g2": (os.path.join("ixt", "dense_in.ixt"), "groupcoo", 2, 0, None),
    }
    os.makedirs(os.path.join(OUT, "convert"))
    index = {}
    for name, (inp, fmt, gg, gd, block) in cases.items():
        d = os.path.join(OUT, "convert", name)
        rc = ref.cmd_convert(os.path.join(OUT, inp), d, fmt, gg, gd, block)
        assert rc == 0, (name, rc)
        index[name] = {"input": inp, "format": fmt, "g": gg, "group_dim": gd, "block": block}
    with open(os.path.join(OUT, "convert", "cases.json"), "w") as f:
        json.dump(index, f, indent=1, sort_keys=True)
    print("wrote", OUT)


def measure_cases():
    """`convert --measure` directories (driver.cpp:434-460): the scores are
    wall-clock times, so tests compare the manifest's structure, gStar and
    candidate list, not the scores or (timing-dependent) chosen g."""
    import shutil
    out = os.path.join(OUT, "convert_measure")
    shutil.rmtree(out, ignore_errors=True)
    os.makedirs(out)
    cases = {"random_auto_measure": ("random_300x200.mtx", "auto", 1, 0, None),
             "general_auto_measure": ("general_real.mtx", "auto", 1, 0, None)}
    index = {}
    for name, (inp, fmt, gg, gd, block) in cases.items():
        rc = ref.cmd_convert(os.path.join(OUT, inp), os.path.join(out, name), fmt, gg, gd, block,
                             measure=True)
        assert rc == 0, (name, rc)
        index[name] = {"input": inp, "format": fmt, "g": gg, "group_dim": gd, "block": block}
    with open(os.path.join(out, "cases.json"), "w") as f:
        json.dump(index, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    if "--measure-only" in sys.argv:
        measure_cases()
    else:
        main()
        measure_cases()
