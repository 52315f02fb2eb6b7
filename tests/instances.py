"""Seeded parity instances (test-side helpers).

Restates the reference acceptance suite's instance makers
(/root/reference/proj/tests/acceptance.cpp:61-162) over either RNG/builder
backend: `oracle.ixo` (the C restatement) or `oracle.ref` (the compiled
reference). Both consume the mt19937_64 stream in the same order, so the
same seed yields bit-identical instances from both.
"""
import numpy as np

EXPR = {
    "coo_spmm": "C[AM[p],n] += AV[p] * B[AK[p],n]",
    "groupcoo_spmm": "C[AM[p],n] += AV[p,q] * B[AK[p,q],n]",
    "blockgroupcoo_spmm": "C[AM[p],bm,n] += AV[p,q,bm,bk] * B[AK[p,q],bk,n]",
    "sparse_conv": "Out[MAPX[p],m] += MAPV[p] * In[MAPY[p],c] * Weight[MAPZ[p],c,m]",
    "grouped_sparse_conv":
        "Out[MAPX[p,q],m] += MAPV[p,q] * In[MAPY[p,q],c] * Weight[MAPZ[p],c,m]",
    "grouped_tp":
        "Z[b,CGI[p,q],w] += CGV[p,q] * X[b,CGJ[p,q],u] * Y[b,CGK[p,q]] * W[b,CGL[p],u,w]",
}
OUT = {"coo_spmm": "C", "groupcoo_spmm": "C", "blockgroupcoo_spmm": "C", "sparse_conv": "Out",
       "grouped_sparse_conv": "Out", "grouped_tp": "Z"}


def make(mod, name, kind, seed):
    """Returns (tensors dict, expr, out_name, out zeros)."""
    rng = mod.Rng(seed)
    pick = rng.uniform_int
    dt = np.int64 if kind == 1 else np.float64
    t = {}
    if name == "coo_spmm":  # acceptance.cpp:61-72
        m, k, n = pick(6, 32), pick(5, 24), pick(2, 8)
        a = mod.synth_sparse_matrix(rng, m, k, 0.25, kind)
        r, c, v = mod.dense_to_coo(a)
        t.update(AV=v, AM=r, AK=c)
        t["B"] = mod.synth_dense(rng, (k, n), kind)
        out = np.zeros((m, n), dt)
    elif name == "groupcoo_spmm":  # acceptance.cpp:74-88
        m, k, n = pick(6, 32), pick(5, 24), pick(2, 8)
        g = pick(1, 4)
        a = mod.synth_sparse_matrix(rng, m, k, 0.3, kind)
        r, c, v = mod.dense_to_coo(a)
        gc = mod.coo_to_groupcoo(m, k, r, c, v, 0, g)
        t.update(AV=gc["AV"], AM=gc["AM"], AK=gc["AK"])
        t["B"] = mod.synth_dense(rng, (k, n), kind)
        out = np.zeros((m, n), dt)
    elif name == "blockgroupcoo_spmm":  # acceptance.cpp:90-105
        bm = bk = 4
        mb, kb, n = pick(2, 8), pick(2, 6), pick(2, 8)
        g = pick(1, 3)
        a = mod.synth_block_sparse_matrix(rng, mb * bm, kb * bk, bm, bk, 0.4, kind)
        b = mod.dense_to_blockgroupcoo(a, bm, bk, g)
        t.update(AV=b["AV"], AM=b["AM"], AK=b["AK"])
        t["B"] = mod.synth_dense(rng, (kb, bk, n), kind)
        out = np.zeros((mb, bm, n), dt)
    elif name in ("sparse_conv", "grouped_sparse_conv"):  # acceptance.cpp:107-137
        grouped = name == "grouped_sparse_conv"
        nx, ny, nz = pick(8, 40), pick(8, 36), pick(3, 9)
        c, m = pick(2, 8), pick(2, 8)
        nnz = pick(4, 64)
        coords, vals = mod.synth_coo_tensor(rng, (nx, ny, nz), nnz, kind)
        if grouped:
            g = pick(1, 4)
            gt = mod.group_coo_tensor((nx, ny, nz), coords, vals, 2, g)
            t["MAPZ"] = gt["group_coord"]
            t["MAPX"] = gt["member_coords"][0]
            t["MAPY"] = gt["member_coords"][1]
            t["MAPV"] = gt["values"]
        else:
            t.update(MAPX=coords[0].copy(), MAPY=coords[1].copy(), MAPZ=coords[2].copy(),
                     MAPV=vals)
        t["In"] = mod.synth_dense(rng, (ny, c), kind)
        t["Weight"] = mod.synth_dense(rng, (nz, c, m), kind)
        out = np.zeros((nx, m), dt)
    elif name == "grouped_tp":  # acceptance.cpp:139-162
        b, ni, nj = pick(2, 6), pick(3, 8), pick(3, 8)
        nk, nl = pick(3, 8), pick(2, 6)
        u, w = pick(2, 8), pick(2, 8)
        nnz = pick(4, 40)
        g = pick(1, 3)
        coords, vals = mod.synth_coo_tensor(rng, (ni, nj, nk, nl), nnz, kind)
        gt = mod.group_coo_tensor((ni, nj, nk, nl), coords, vals, 3, g)
        t["CGL"] = gt["group_coord"]
        t["CGI"] = gt["member_coords"][0]
        t["CGJ"] = gt["member_coords"][1]
        t["CGK"] = gt["member_coords"][2]
        t["CGV"] = gt["values"]
        t["X"] = mod.synth_dense(rng, (b, nj, u), kind)
        t["Y"] = mod.synth_dense(rng, (b, nk), kind)
        t["W"] = mod.synth_dense(rng, (b, nl, u, w), kind)
        out = np.zeros((b, ni, w), dt)
    else:
        raise KeyError(name)
    return t, EXPR[name], OUT[name], out


def materialize(mod, spec):
    """Restates materialize (driver.cpp:165-233) for a run spec dict over a
    backend module: one Rng(seed); dense specs, then index specs, then sparse
    specs in spec order; formats bound like bind_matrix_format /
    bind_tensor_format (driver.cpp:98-161). Returns (tensors, out)."""
    kind = 1 if spec.get("elem") == "int64" else 0
    rng = mod.Rng(spec.get("seed", 0))
    t = {}
    for d in spec.get("dense", []):
        t[d["name"]] = mod.synth_dense(rng, tuple(d["shape"]), kind)
    for ix in spec.get("index", []):
        t[ix["name"]] = np.array([rng.uniform_int(0, max(ix["bound"] - 1, 0))
                                  for _ in range(int(np.prod(ix["shape"])))],
                                 np.int64).reshape(ix["shape"])
    for s in spec.get("sparse", []):
        name, shape, fmt = s["name"], s["shape"], s.get("format", "coo")
        g, gd = s.get("g", 1), s.get("groupDim", 0)
        if len(shape) == 2:
            suf = s.get("suffixes", ["M", "K"])
            if "genBlock" in s:
                a = mod.synth_block_sparse_matrix(rng, shape[0], shape[1], s["genBlock"][0],
                                                  s["genBlock"][1], s.get("blockDensity", 0.1),
                                                  kind)
            else:
                a = mod.synth_sparse_matrix(rng, shape[0], shape[1], s.get("density", 0.1), kind)
            r, c, v = mod.dense_to_coo(a)
            if fmt == "coo":
                t[name + "V"], t[name + suf[0]], t[name + suf[1]] = v, r, c
                continue
            if fmt == "blockgroupcoo":
                b = mod.dense_to_blockgroupcoo(a, s["formatBlock"][0], s["formatBlock"][1], g, gd)
            else:
                if fmt == "auto":
                    occ = np.bincount(r if gd == 0 else c,
                                      minlength=shape[0] if gd == 0 else shape[1])
                    from oracle import ixo
                    g = ixo.select(occ.astype(np.int64))
                b = mod.coo_to_groupcoo(shape[0], shape[1], r, c, v, gd, g)
            gs, ms = (suf[0], suf[1]) if gd == 0 else (suf[1], suf[0])
            t[name + "V"], t[name + gs], t[name + ms] = b["AV"], b["AM"], b["AK"]
        else:
            suf = s.get("suffixes", [chr(ord("I") + i) for i in range(len(shape))])
            nnz = s.get("nnz", -1)
            if nnz < 0:
                nnz = max(1, int(s.get("density", 0.1) * np.prod(shape)))
            coords, vals = mod.synth_coo_tensor(rng, tuple(shape), nnz, kind)
            if fmt == "coo":
                for dd in range(len(shape)):
                    t[name + suf[dd]] = coords[dd].copy()
                t[name + "V"] = vals
            else:
                gt = mod.group_coo_tensor(tuple(shape), coords, vals, gd, g)
                t[name + suf[gd]] = gt["group_coord"]
                m = 0
                for dd in range(len(shape)):
                    if dd != gd:
                        t[name + suf[dd]] = gt["member_coords"][m]
                        m += 1
                t[name + "V"] = gt["values"]
    o = spec["output"]
    out = np.zeros(o["shape"], np.int64 if kind else np.float64)
    return t, out


def occ3112_matrix():
    """The paper's Fig. 4 matrix, occupancy [3,1,1,2] (tests/helpers.hpp:16-21)."""
    return np.array([[1, 2, 0, 3], [0, 4, 0, 0], [0, 0, 5, 0], [6, 0, 0, 7]], dtype=np.float64)
