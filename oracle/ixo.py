"""ctypes wrapper of the plain-C oracle restatement (oracle/ixo.c).

TEST INFRASTRUCTURE ONLY. Arrays are numpy: real = float64, int = int64,
mirroring the reference's `ElemKind { Real64, Int64 }` (tensor.hpp:11).
"""
import ctypes as C
import os

import numpy as np

from . import ORACLE_DIR

_lib = None

REAL, INT = 0, 1


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(ORACLE_DIR, "libixo.so")
        if not os.path.exists(path):
            from . import build
            build()
        L = C.CDLL(path)
        P, I64, D, U64 = C.c_void_p, C.c_int64, C.c_double, C.c_uint64
        sig = {
            "ixo_rng_new": (P, [U64]),
            "ixo_rng_free": (None, [P]),
            "ixo_rng_next": (U64, [P]),
            "ixo_uniform_int": (I64, [P, I64, I64]),
            "ixo_canonical": (D, [P]),
            "ixo_bernoulli": (C.c_int, [P, D]),
            "ixo_uniform_real": (D, [P, D, D]),
            "ixo_synth_dense": (None, [P, C.c_int, I64, P]),
            "ixo_synth_sparse_matrix": (None, [P, C.c_int, I64, I64, D, P]),
            "ixo_synth_block_sparse_matrix": (None, [P, C.c_int, I64, I64, I64, I64, D, P]),
            "ixo_synth_coo_tensor": (I64, [P, C.c_int, C.c_int, P, I64, P, P]),
            "ixo_count_nonzero": (I64, [C.c_int, I64, P]),
            "ixo_dense_to_coo": (None, [C.c_int, I64, I64, P, P, P, P]),
            "ixo_coo_to_groupcoo": (C.c_int, [I64, I64, P, P, C.c_int, P, I64, C.c_int, I64, P,
                                              P, P, P, P]),
            "ixo_dense_to_blockgroupcoo": (C.c_int, [C.c_int, I64, I64, P, I64, I64, I64,
                                                     C.c_int, P, P, P, P, P]),
            "ixo_group_coo_tensor": (C.c_int, [C.c_int, P, P, C.c_int, P, I64, C.c_int, I64, P,
                                               P, P, P, P]),
            "ixo_cost_exact": (I64, [P, I64, I64]),
            "ixo_cost_relaxed": (D, [P, I64, D, C.c_int]),
            "ixo_g_star": (D, [P, I64, C.c_int]),
            "ixo_candidate_group_sizes": (C.c_int, [P, I64, C.c_int, P]),
            "ixo_select": (I64, [P, I64, C.c_int]),
            "ixo_brute_force_optimal": (I64, [P, I64, P]),
            "ixo_einsum": (C.c_int, [C.c_char_p, P, C.c_int, C.c_char_p, C.c_int, C.c_int, P, P,
                                     C.c_char_p, C.c_int]),
            "ixo_max_rel_error": (D, [C.c_int, I64, P, P]),
            "ixo_tensor_hash": (U64, [C.c_int, C.c_int, P, P]),
            "ixo_kernel_map": (I64, [P, I64, P, P, P]),
            "ixo_cg_table": (I64, [C.c_int, P, P, P, P, P, P, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _kind(a):
    return INT if a.dtype == np.int64 else REAL


def _dt(kind):
    return np.int64 if kind == INT else np.float64


class OracleError(Exception):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class Rng:
    """std::mt19937_64 with libstdc++'s distributions (synth.hpp:17)."""

    def __init__(self, seed):
        self._free = lib().ixo_rng_free
        self.h = lib().ixo_rng_new(seed)

    def __del__(self):
        if getattr(self, "h", None):
            self._free(self.h)
            self.h = None

    def next(self):
        return lib().ixo_rng_next(self.h)

    def uniform_int(self, lo, hi):
        return lib().ixo_uniform_int(self.h, lo, hi)

    def canonical(self):
        return lib().ixo_canonical(self.h)


def synth_dense(rng, shape, kind=REAL):
    out = np.empty(shape, dtype=_dt(kind))
    lib().ixo_synth_dense(rng.h, kind, out.size, _p(out))
    return out


def synth_sparse_matrix(rng, rows, cols, density, kind=REAL):
    out = np.empty((rows, cols), dtype=_dt(kind))
    lib().ixo_synth_sparse_matrix(rng.h, kind, rows, cols, density, _p(out))
    return out


def synth_block_sparse_matrix(rng, rows, cols, br, bc, bdens, kind=REAL):
    out = np.empty((rows, cols), dtype=_dt(kind))
    lib().ixo_synth_block_sparse_matrix(rng.h, kind, rows, cols, br, bc, bdens, _p(out))
    return out


def synth_coo_tensor(rng, shape, nnz, kind=REAL):
    shape = np.asarray(shape, dtype=np.int64)
    cap = int(np.prod(shape))
    n = min(nnz, cap)
    coords = np.empty((len(shape), n), dtype=np.int64)
    vals = np.empty(n, dtype=_dt(kind))
    got = lib().ixo_synth_coo_tensor(rng.h, kind, len(shape), _p(shape), nnz, _p(coords), _p(vals))
    assert got == n
    return coords, vals


def dense_to_coo(dense):
    dense = np.ascontiguousarray(dense)
    k = _kind(dense)
    n = lib().ixo_count_nonzero(k, dense.size, _p(dense))
    r = np.empty(n, np.int64)
    c = np.empty(n, np.int64)
    v = np.empty(n, dense.dtype)
    lib().ixo_dense_to_coo(k, dense.shape[0], dense.shape[1], _p(dense), _p(r), _p(c), _p(v))
    return r, c, v


def coo_to_groupcoo(rows, cols, r, c, vals, group_dim, g):
    """Returns dict AM[G], AK[G,g], AV[G,g], mask[G,g] (formats.cpp:115-174)."""
    r = np.ascontiguousarray(r, np.int64)
    c = np.ascontiguousarray(c, np.int64)
    vals = np.ascontiguousarray(vals)
    k = _kind(vals)
    G = C.c_int64(0)
    st = lib().ixo_coo_to_groupcoo(rows, cols, _p(r), _p(c), k, _p(vals), len(r), group_dim, g,
                                   C.byref(G), None, None, None, None)
    if st:
        raise OracleError(st, "coo_to_groupcoo: invalid parameters")
    G = G.value
    AM = np.empty(G, np.int64)
    AK = np.empty((G, g), np.int64)
    AV = np.empty((G, g), vals.dtype)
    mask = np.empty((G, g), np.uint8)
    lib().ixo_coo_to_groupcoo(rows, cols, _p(r), _p(c), k, _p(vals), len(r), group_dim, g,
                              C.byref(C.c_int64(0)), _p(AM), _p(AK), _p(AV), _p(mask))
    return {"AM": AM, "AK": AK, "AV": AV, "mask": mask}


def dense_to_blockgroupcoo(dense, bm, bk, g, group_dim=0):
    dense = np.ascontiguousarray(dense)
    k = _kind(dense)
    G = C.c_int64(0)
    st = lib().ixo_dense_to_blockgroupcoo(k, dense.shape[0], dense.shape[1], _p(dense), bm, bk,
                                          g, group_dim, C.byref(G), None, None, None, None)
    if st:
        raise OracleError(st, "dense_to_blockgroupcoo: invalid parameters")
    G = G.value
    AM = np.empty(G, np.int64)
    AK = np.empty((G, g), np.int64)
    AV = np.empty((G, g, bm, bk), dense.dtype)
    mask = np.empty((G, g), np.uint8)
    lib().ixo_dense_to_blockgroupcoo(k, dense.shape[0], dense.shape[1], _p(dense), bm, bk, g,
                                     group_dim, C.byref(C.c_int64(0)), _p(AM), _p(AK), _p(AV),
                                     _p(mask))
    return {"AM": AM, "AK": AK, "AV": AV, "mask": mask}


def group_coo_tensor(shape, coords, vals, group_dim, g):
    """coords [rank, nnz] → group_coord[G], member_coords[rank-1, G, g], values, mask."""
    shape = np.ascontiguousarray(shape, np.int64)
    coords = np.ascontiguousarray(coords, np.int64)
    vals = np.ascontiguousarray(vals)
    k = _kind(vals)
    rank, nnz = coords.shape
    G = C.c_int64(0)
    st = lib().ixo_group_coo_tensor(rank, _p(shape), _p(coords), k, _p(vals), nnz, group_dim, g,
                                    C.byref(G), None, None, None, None)
    if st:
        raise OracleError(st, "group_coo_tensor: invalid parameters")
    G = G.value
    gc = np.empty(G, np.int64)
    mc = np.empty((rank - 1, G, g), np.int64)
    v = np.empty((G, g), vals.dtype)
    mask = np.empty((G, g), np.uint8)
    lib().ixo_group_coo_tensor(rank, _p(shape), _p(coords), k, _p(vals), nnz, group_dim, g,
                               C.byref(C.c_int64(0)), _p(gc), _p(mc), _p(v), _p(mask))
    return {"group_coord": gc, "member_coords": mc, "values": v, "mask": mask}


def occupancy(coord, extent):
    return np.bincount(np.asarray(coord, np.int64), minlength=extent).astype(np.int64)


def cost_exact(occ, g):
    occ = np.ascontiguousarray(occ, np.int64)
    return lib().ixo_cost_exact(_p(occ), len(occ), g)


def cost_relaxed(occ, g, count_empty_rows=False):
    occ = np.ascontiguousarray(occ, np.int64)
    return lib().ixo_cost_relaxed(_p(occ), len(occ), float(g), int(count_empty_rows))


def g_star(occ, count_empty_rows=False):
    occ = np.ascontiguousarray(occ, np.int64)
    return lib().ixo_g_star(_p(occ), len(occ), int(count_empty_rows))


def candidate_group_sizes(occ, count_empty_rows=False):
    occ = np.ascontiguousarray(occ, np.int64)
    cand = np.zeros(2, np.int64)
    n = lib().ixo_candidate_group_sizes(_p(occ), len(occ), int(count_empty_rows), _p(cand))
    return [int(x) for x in cand[:n]]


def select(occ, count_empty_rows=False):
    occ = np.ascontiguousarray(occ, np.int64)
    return lib().ixo_select(_p(occ), len(occ), int(count_empty_rows))


def brute_force_optimal(occ):
    occ = np.ascontiguousarray(occ, np.int64)
    f = C.c_int64(0)
    g = lib().ixo_brute_force_optimal(_p(occ), len(occ), C.byref(f))
    return None if g == 0 else (g, f.value)


def einsum(expr, tensors, out_name, out):
    """oracle_einsum (plan.cpp:598). `out` primes `+=`; returns a new array."""
    res = np.array(out, copy=True, order="C")
    keep = []
    arr = (_TensorT * max(len(tensors), 1))()
    for i, (name, t) in enumerate(tensors.items()):
        t = np.ascontiguousarray(t)
        if t.dtype not in (np.int64, np.float64):
            raise TypeError(f"oracle tensors are float64/int64, {name} is {t.dtype}")
        sh = np.asarray(t.shape, np.int64)
        keep += [t, sh, name.encode()]
        arr[i].name = keep[-1]
        arr[i].kind = _kind(t)
        arr[i].rank = t.ndim
        arr[i].shape = _p(sh)
        arr[i].data = _p(t)
    osh = np.asarray(res.shape, np.int64)
    err = C.create_string_buffer(512)
    st = lib().ixo_einsum(expr.encode(), C.cast(arr, C.c_void_p), len(tensors), out_name.encode(),
                          _kind(res), res.ndim, _p(osh), _p(res), err, 512)
    if st:
        raise OracleError(st, err.value.decode())
    return res


class _TensorT(C.Structure):
    _fields_ = [("name", C.c_char_p), ("kind", C.c_int), ("rank", C.c_int),
                ("shape", C.c_void_p), ("data", C.c_void_p)]


def max_rel_error(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b, dtype=a.dtype)
    assert a.shape == b.shape
    return lib().ixo_max_rel_error(_kind(a), a.size, _p(a), _p(b))


def tensor_hash(a):
    a = np.ascontiguousarray(a)
    sh = np.asarray(a.shape, np.int64)
    return lib().ixo_tensor_hash(_kind(a), a.ndim, _p(sh), _p(a))


def kernel_map(coords):
    """coords int32 [n,3] → (out, in, offset) sorted by (offset, out)."""
    coords = np.ascontiguousarray(coords, np.int32)
    n = coords.shape[0]
    cnt = lib().ixo_kernel_map(_p(coords), n, None, None, None)
    mo, mi, mz = (np.empty(cnt, np.int64) for _ in range(3))
    lib().ixo_kernel_map(_p(coords), n, _p(mo), _p(mi), _p(mz))
    return mo, mi, mz


def cg_table(l_max):
    """Real-basis CG entries (i, j, k, path, value) and the (l1,l2,l3) paths."""
    npaths = C.c_int(0)
    cnt = lib().ixo_cg_table(l_max, None, None, None, None, None, C.byref(npaths), None)
    ci, cj, ck, cl = (np.empty(cnt, np.int64) for _ in range(4))
    cv = np.empty(cnt, np.float64)
    paths = np.empty((npaths.value, 3), np.int64)
    lib().ixo_cg_table(l_max, _p(ci), _p(cj), _p(ck), _p(cl), _p(cv), C.byref(npaths), _p(paths))
    return {"i": ci, "j": cj, "k": ck, "l": cl, "v": cv, "paths": paths}
