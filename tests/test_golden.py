"""Pins the C oracle against golden fixtures produced by the unmodified
reference (tests/golden/make_golden.py). CPU only; needs no /root/reference,
so it also runs on the GPU box."""
import glob
import json
import os

import numpy as np
import pytest

import instances

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CORPUS = sorted(glob.glob(os.path.join(GOLDEN, "corpus_*.npz")))


def load(path):
    d = np.load(path)
    tensors = {k[2:]: d[k] for k in d.files if k.startswith("t_")}
    return d, tensors


@pytest.mark.parametrize("path", CORPUS, ids=[os.path.basename(p) for p in CORPUS])
def test_corpus_oracle_matches_reference(ixo, path):
    d, tensors = load(path)
    expr, on = str(d["expr"]), str(d["out_name"])
    got = ixo.einsum(expr, tensors, on, d["out"])
    np.testing.assert_array_equal(got, d["res_oracle"])
    if got.dtype == np.int64:
        np.testing.assert_array_equal(d["res_plan"], got)
        np.testing.assert_array_equal(d["res_fused-lazy"], got)


@pytest.mark.parametrize("path", CORPUS, ids=[os.path.basename(p) for p in CORPUS])
def test_corpus_materialize_restated_bit_exact(ixo, path):
    """The C restatement of synth + builders, in materialize order, rebuilds
    every operand the reference materialized for the corpus spec."""
    d, tensors = load(path)
    spec = json.loads(str(d["spec"]))
    mine, out = instances.materialize(ixo, spec)
    assert sorted(mine) == sorted(tensors)
    for k in tensors:
        np.testing.assert_array_equal(mine[k], tensors[k], err_msg=k)
    np.testing.assert_array_equal(out, d["out"])


@pytest.mark.parametrize("tag,kind", [("real", 0), ("int", 1)])
def test_cfg1_slab(ixo, tag, kind):
    d = np.load(os.path.join(GOLDEN, f"cfg1_slab_{tag}.npz"))
    rng = ixo.Rng(1)
    B = ixo.synth_dense(rng, (4096, 128), kind)
    A = ixo.synth_sparse_matrix(rng, 64, 4096, 0.01, kind)
    assert ixo.tensor_hash(B) == int(d["B_hash"]) and ixo.tensor_hash(A) == int(d["A_hash"])
    r, c, v = ixo.dense_to_coo(A)
    g = ixo.select(np.bincount(r, minlength=64).astype(np.int64))
    assert g == int(d["g"])
    gc = ixo.coo_to_groupcoo(64, 4096, r, c, v, 0, g)
    for k in ("AM", "AK", "AV", "mask"):
        np.testing.assert_array_equal(gc[k], d[k])
    t = {"AM": gc["AM"], "AK": gc["AK"], "AV": gc["AV"], "B": B}
    res = ixo.einsum("C[AM[p],n] += AV[p,q] * B[AK[p,q],n]", t, "C", np.zeros_like(d["res"]))
    np.testing.assert_array_equal(res, d["res"])


@pytest.mark.parametrize("tag,kind", [("real", 0), ("int", 1)])
def test_cfg2_slab(ixo, tag, kind):
    d = np.load(os.path.join(GOLDEN, f"cfg2_slab_{tag}.npz"))
    rng = ixo.Rng(1)
    B = ixo.synth_dense(rng, (512, 16, 512), kind)
    A = ixo.synth_block_sparse_matrix(rng, 32, 8192, 16, 16, 0.10, kind)
    assert ixo.tensor_hash(B) == int(d["B_hash"]) and ixo.tensor_hash(A) == int(d["A_hash"])
    bg = ixo.dense_to_blockgroupcoo(A, 16, 16, 8, 0)
    for k in ("AM", "AK", "mask"):
        np.testing.assert_array_equal(bg[k], d[k])
    np.testing.assert_array_equal(bg["AV"].astype(d["AV"].dtype), d["AV"])
    t = {"AM": bg["AM"], "AK": bg["AK"], "AV": bg["AV"], "B": B}
    res = ixo.einsum("C[AM[p],bm,n] += AV[p,q,bm,bk] * B[AK[p,q],bk,n]", t, "C",
                     np.zeros_like(d["res"]))
    np.testing.assert_array_equal(res, d["res"])


def test_builders_fixture(ixo):
    d = np.load(os.path.join(GOLDEN, "builders.npz"))
    for i in range(3):
        A = d[f"m{i}_dense"]
        rows, cols = A.shape
        r, c, v = ixo.dense_to_coo(A)
        for gd in (0, 1):
            for g in (1, 3, 8):
                gc = ixo.coo_to_groupcoo(rows, cols, r, c, v, gd, g)
                for k in ("AM", "AK", "AV", "mask"):
                    np.testing.assert_array_equal(gc[k], d[f"m{i}_gd{gd}_g{g}_{k}"])
            bg = ixo.dense_to_blockgroupcoo(A, 4, 4, 2, gd)
            for k in ("AM", "AK", "AV", "mask"):
                np.testing.assert_array_equal(bg[k], d[f"m{i}_blk_gd{gd}_{k}"])
    for gd in range(4):
        gt = ixo.group_coo_tensor((6, 5, 4, 3), d["t_coords"], d["t_vals"], gd, 3)
        for k in ("group_coord", "member_coords", "values", "mask"):
            np.testing.assert_array_equal(gt[k], d[f"t_gd{gd}_{k}"])
