"""ctypes wrapper of the unmodified reference library (oracle/_ref/libixsum_ref.so).

TEST INFRASTRUCTURE ONLY: it is how the tests pin the C restatement and how
bench.py times the reference's own CPU path. `available()` is False when the
library was never built (no /root/reference and no prebuilt copy).
"""
import ctypes as C
import json
import os
import tempfile

import numpy as np

from . import ORACLE_DIR

_lib = None
LIB_PATH = os.path.join(ORACLE_DIR, "_ref", "libixsum_ref.so")


def available():
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)
        P, I64, D, U64, S = C.c_void_p, C.c_int64, C.c_double, C.c_uint64, C.c_char_p
        sig = {
            "ixr_last_error": (S, []),
            "ixr_last_code": (C.c_int, []),
            "ixr_free": (None, [P]),
            "ixr_bag_new": (P, []),
            "ixr_bag_count": (C.c_int, [P]),
            "ixr_bag_name": (S, [P, C.c_int]),
            "ixr_bag_info": (C.c_int, [P, S, P, P]),
            "ixr_bag_read": (C.c_int, [P, S, P]),
            "ixr_bag_set": (None, [P, S, C.c_int, C.c_int, P, P]),
            "ixr_bag_scalar": (D, [P, S]),
            "ixr_bag_text": (S, [P]),
            "ixr_rng_new": (P, [U64]),
            "ixr_rng_free": (None, [P]),
            "ixr_rng_next": (U64, [P]),
            "ixr_uniform_int": (I64, [P, I64, I64]),
            "ixr_synth_dense": (P, [P, C.c_int, C.c_int, P]),
            "ixr_synth_sparse_matrix": (P, [P, C.c_int, I64, I64, D]),
            "ixr_synth_block_sparse_matrix": (P, [P, C.c_int, I64, I64, I64, I64, D]),
            "ixr_synth_coo_tensor": (P, [P, C.c_int, C.c_int, P, I64]),
            "ixr_dense_to_coo": (P, [C.c_int, I64, I64, P]),
            "ixr_coo_to_groupcoo": (P, [I64, I64, P, P, C.c_int, P, I64, C.c_int, C.c_int, I64]),
            "ixr_dense_to_blockgroupcoo": (P, [C.c_int, I64, I64, P, I64, I64, I64, C.c_int]),
            "ixr_group_coo_tensor": (P, [C.c_int, P, P, C.c_int, P, I64, C.c_int, I64]),
            "ixr_tune": (C.c_int, [P, I64, C.c_int, P, P]),
            "ixr_cost_exact": (I64, [P, I64, I64]),
            "ixr_cost_relaxed": (D, [P, I64, D, C.c_int]),
            "ixr_problem_from_spec": (P, [S]),
            "ixr_run": (P, [P, S, S, S, C.c_int]),
            "ixr_count_model": (C.c_int, [I64, I64, P, S, S, P]),
            "ixr_max_rel_error": (D, [C.c_int, I64, P, P]),
            "ixr_tensor_hash": (U64, [C.c_int, C.c_int, P, P]),
            "ixr_load_tensor": (P, [S]),
            "ixr_save_tensor": (C.c_int, [S, C.c_int, C.c_int, P, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class RefError(Exception):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _kind(a):
    return 1 if a.dtype == np.int64 else 0


def _check(h):
    if not h:
        L = lib()
        raise RefError(L.ixr_last_code(), L.ixr_last_error().decode())
    return h


class Bag:
    """Named reference Tensors (+ scalars) owned by the C++ side."""

    def __init__(self, h=-1):
        self._free = lib().ixr_free
        self.h = lib().ixr_bag_new() if h == -1 else _check(h)

    def __del__(self):
        if getattr(self, "h", None):
            self._free(self.h)
            self.h = None

    def names(self):
        L = lib()
        return [L.ixr_bag_name(self.h, i).decode() for i in range(L.ixr_bag_count(self.h))]

    def __contains__(self, name):
        kind = C.c_int(0)
        sh = np.zeros(16, np.int64)
        return lib().ixr_bag_info(self.h, name.encode(), C.byref(kind), _p(sh)) >= 0

    def __getitem__(self, name):
        kind = C.c_int(0)
        sh = np.zeros(16, np.int64)
        rank = lib().ixr_bag_info(self.h, name.encode(), C.byref(kind), _p(sh))
        if rank < 0:
            raise KeyError(name)
        out = np.empty(tuple(sh[:rank]), dtype=np.int64 if kind.value else np.float64)
        lib().ixr_bag_read(self.h, name.encode(), _p(out))
        return out

    def __setitem__(self, name, arr):
        arr = np.ascontiguousarray(arr)
        if arr.dtype not in (np.int64, np.float64):
            arr = arr.astype(np.float64)
        sh = np.asarray(arr.shape, np.int64)
        lib().ixr_bag_set(self.h, name.encode(), _kind(arr), arr.ndim, _p(sh), _p(arr))

    def scalar(self, name):
        return lib().ixr_bag_scalar(self.h, name.encode())

    def text(self):
        return lib().ixr_bag_text(self.h).decode()

    def to_dict(self):
        return {n: self[n] for n in self.names()}


class Rng:
    def __init__(self, seed):
        self._free = lib().ixr_rng_free
        self.h = lib().ixr_rng_new(seed)

    def __del__(self):
        if getattr(self, "h", None):
            self._free(self.h)
            self.h = None

    def next(self):
        return lib().ixr_rng_next(self.h)

    def uniform_int(self, lo, hi):
        return lib().ixr_uniform_int(self.h, lo, hi)


def synth_dense(rng, shape, kind=0):
    sh = np.asarray(shape, np.int64)
    return Bag(lib().ixr_synth_dense(rng.h, kind, len(sh), _p(sh)))["t"]


def synth_sparse_matrix(rng, rows, cols, density, kind=0):
    return Bag(lib().ixr_synth_sparse_matrix(rng.h, kind, rows, cols, density))["t"]


def synth_block_sparse_matrix(rng, rows, cols, br, bc, bdens, kind=0):
    return Bag(lib().ixr_synth_block_sparse_matrix(rng.h, kind, rows, cols, br, bc, bdens))["t"]


def synth_coo_tensor(rng, shape, nnz, kind=0):
    sh = np.asarray(shape, np.int64)
    b = Bag(lib().ixr_synth_coo_tensor(rng.h, kind, len(sh), _p(sh), nnz))
    return b["coords"], b["values"]


def dense_to_coo(dense):
    dense = np.ascontiguousarray(dense)
    b = Bag(lib().ixr_dense_to_coo(_kind(dense), dense.shape[0], dense.shape[1], _p(dense)))
    return b["row_coord"], b["col_coord"], b["values"]


def coo_to_groupcoo(rows, cols, r, c, vals, group_dim, g, canonical=False):
    r = np.ascontiguousarray(r, np.int64)
    c = np.ascontiguousarray(c, np.int64)
    vals = np.ascontiguousarray(vals)
    b = Bag(lib().ixr_coo_to_groupcoo(rows, cols, _p(r), _p(c), _kind(vals), _p(vals), len(r),
                                      int(canonical), group_dim, g))
    d = b.to_dict()
    d["mask"] = d["mask"].astype(np.uint8)
    d["nbytes"] = int(b.scalar("nbytes"))
    d["maskbytes"] = int(b.scalar("maskbytes"))
    d["is_ell"] = bool(b.scalar("is_ell"))
    return d


def dense_to_blockgroupcoo(dense, bm, bk, g, group_dim=0):
    dense = np.ascontiguousarray(dense)
    b = Bag(lib().ixr_dense_to_blockgroupcoo(_kind(dense), dense.shape[0], dense.shape[1],
                                             _p(dense), bm, bk, g, group_dim))
    d = b.to_dict()
    d["mask"] = d["mask"].astype(np.uint8)
    d["nbytes"] = int(b.scalar("nbytes"))
    return d


def group_coo_tensor(shape, coords, vals, group_dim, g):
    sh = np.asarray(shape, np.int64)
    coords = np.ascontiguousarray(coords, np.int64)
    vals = np.ascontiguousarray(vals)
    b = Bag(lib().ixr_group_coo_tensor(len(sh), _p(sh), _p(coords), _kind(vals), _p(vals),
                                       coords.shape[1], group_dim, g))
    d = b.to_dict()
    d["mask"] = d["mask"].astype(np.uint8)
    return d


def tune(occ, count_empty_rows=False):
    occ = np.ascontiguousarray(occ, np.int64)
    out6 = np.zeros(6)
    cands = np.zeros(4)
    if lib().ixr_tune(_p(occ), len(occ), int(count_empty_rows), _p(out6), _p(cands)) != 0:
        raise RefError(lib().ixr_last_code(), lib().ixr_last_error().decode())
    n = int(out6[4])
    return {"gstar": out6[0], "chosen": int(out6[1]),
            "brute": None if out6[2] < 0 else (int(out6[2]), int(out6[3])),
            "candidates": [(int(cands[2 * i]), cands[2 * i + 1]) for i in range(n)]}


def cost_exact(occ, g):
    occ = np.ascontiguousarray(occ, np.int64)
    return lib().ixr_cost_exact(_p(occ), len(occ), g)


def problem_from_spec(spec: dict):
    """load_run_config + materialize (driver.cpp:43-233) of a JSON run spec."""
    with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
        json.dump(spec, f)
        path = f.name
    try:
        return Bag(lib().ixr_problem_from_spec(path.encode()))
    finally:
        os.unlink(path)


def run(tensors, expr, out_name, out, mode="oracle", threads=1):
    """execute_mode (driver.cpp:235-265) over `tensors` + output buffer `out`.

    Returns (result array, scalars dict)."""
    bag = Bag()
    for n, t in tensors.items():
        bag[n] = t
    bag[out_name] = out
    r = Bag(lib().ixr_run(bag.h, expr.encode(), out_name.encode(), mode.encode(), threads))
    sc = {k: r.scalar(k) for k in ("wall_ms", "gathers", "scatters", "atomic_updates",
                                   "kernel_count")}
    return r["result"], sc


def max_rel_error(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b, dtype=a.dtype)
    return lib().ixr_max_rel_error(_kind(a), a.size, _p(a), _p(b))


def tensor_hash(a):
    a = np.ascontiguousarray(a)
    sh = np.asarray(a.shape, np.int64)
    return lib().ixr_tensor_hash(_kind(a), a.ndim, _p(sh), _p(a))


# ---- file formats (test fixtures and parity only)
def ref_io(*args, env=None):
    """Runs oracle/_ref/ref_io (the reference's file-format code in its own
    process); returns (exit code, stdout)."""
    import subprocess
    exe = os.path.join(ORACLE_DIR, "_ref", "ref_io")
    r = subprocess.run([exe, *map(str, args)], capture_output=True, text=True,
                       env=dict(os.environ, **env) if env else None)
    return r.returncode, r.stdout


def load_matrix_market(path):
    """The reference's load_matrix_market (matrix_market.cpp:30-159):
    {"dense"} or {"rows", "cols", "row", "col", "values"}; raises RefError
    with the reference's message."""
    _, out = ref_io("mtx", path)
    d = json.loads(out)
    if "error" in d:
        raise RefError(1, d["error"])
    dt = np.int64 if d["kind"] else np.float64
    if "dense" in d:
        return {"dense": np.asarray(d["dense"], dt).reshape(d["shape"])}
    return {"rows": d["rows"], "cols": d["cols"], "row": np.asarray(d["row"], np.int64),
            "col": np.asarray(d["col"], np.int64), "values": np.asarray(d["values"], dt)}


def cmd_convert(inp, outdir, fmt, g=1, group_dim=0, block=None, prefix="A", measure=False):
    """cmd_convert (driver.cpp:403-514); measure=True is `--measure` (candidates
    scored by the wall clock of the reference SpMM). Returns the exit code."""
    bm, bk = block if block else (0, 0)
    rc, _ = ref_io("convert", inp, outdir, fmt, g, group_dim, bm, bk, prefix,
                   env={"IXR_MEASURE": "1"} if measure else None)
    return rc


def load_tensor(path):
    return Bag(lib().ixr_load_tensor(os.fsencode(path)))["t"]


def save_tensor(path, arr):
    arr = np.ascontiguousarray(arr)
    sh = np.asarray(arr.shape, np.int64)
    if lib().ixr_save_tensor(os.fsencode(path), _kind(arr), arr.ndim, _p(sh), _p(arr)) != 0:
        raise RefError(lib().ixr_last_code(), lib().ixr_last_error().decode())
