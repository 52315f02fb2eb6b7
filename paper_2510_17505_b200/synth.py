"""Seeded synthetic inputs (synth.hpp:13-29) via libixb's host generator.

Same mt19937_64 stream and call order as the reference's synth_*, so a seed
reproduces the reference's operands (values rounded to the device dtype).
Returns host torch tensors (optionally pinned) ready to copy to the device.
"""
import ctypes as C

import numpy as np
import torch

from .abi import check, lib

REAL, INT = 0, 1
_OUT = {torch.float32: 0, torch.bfloat16: 1, torch.float64: 2, torch.int64: 3}


class Rng:
    """One generator shared by all operands, in materialize order (driver.cpp:167)."""

    def __init__(self, seed):
        self._free = lib().ixb_rng_free
        self.h = lib().ixb_rng_new(seed)

    def __del__(self):
        if getattr(self, "h", None):
            self._free(self.h)
            self.h = None

    def next(self):
        return lib().ixb_rng_next(self.h)


def _alloc(shape, dtype, pin):
    return torch.empty(shape, dtype=dtype, pin_memory=pin)


def synth_dense(rng, shape, kind=REAL, dtype=torch.float32, pin=False):
    t = _alloc(shape, dtype, pin)
    check(lib().ixb_synth_dense(rng.h, kind, t.numel(), _OUT[dtype], C.c_void_p(t.data_ptr())))
    return t


def synth_sparse_matrix(rng, rows, cols, density, kind=REAL, dtype=torch.float32, pin=False):
    t = _alloc((rows, cols), dtype, pin)
    check(lib().ixb_synth_sparse_matrix(rng.h, kind, rows, cols, density, _OUT[dtype],
                                        C.c_void_p(t.data_ptr())))
    return t


def synth_block_sparse_matrix(rng, rows, cols, br, bc, bdens, kind=REAL, dtype=torch.float32,
                              pin=False):
    t = _alloc((rows, cols), dtype, pin)
    check(lib().ixb_synth_block_sparse_matrix(rng.h, kind, rows, cols, br, bc, bdens, _OUT[dtype],
                                              C.c_void_p(t.data_ptr())))
    return t


def synth_coo_tensor(rng, shape, nnz, kind=REAL, dtype=torch.float32):
    cap = int(np.prod(shape))
    n = min(nnz, cap)
    coords = torch.empty((len(shape), n), dtype=torch.int32)
    vals = torch.empty(n, dtype=dtype)
    sh = (C.c_int64 * len(shape))(*shape)
    got = C.c_int64(0)
    check(lib().ixb_synth_coo_tensor(rng.h, kind, len(shape), sh, nnz, _OUT[dtype],
                                     C.c_void_p(coords.data_ptr()), C.c_void_p(vals.data_ptr()),
                                     C.byref(got)))
    return coords, vals


def synth_voxel_shells(n_target):
    """cfg5 point cloud: voxelised sphere shells, sorted (x, y, z), int32 [n, 3]."""
    n = C.c_int64(0)
    check(lib().ixb_synth_voxel_shells(n_target, None, C.byref(n)))
    coords = torch.empty((n.value, 3), dtype=torch.int32)
    check(lib().ixb_synth_voxel_shells(n_target, C.c_void_p(coords.data_ptr()), C.byref(n)))
    return coords


def cg_table(l_max=3):
    """Real-basis CG table (host): dict of int32 i, j, k, l, float32 v, npaths."""
    n, npaths = C.c_int64(0), C.c_int32(0)
    check(lib().ixb_cg_table(l_max, None, None, None, None, None, C.byref(n), C.byref(npaths)))
    out = {k: torch.empty(n.value, dtype=torch.int32) for k in ("i", "j", "k", "l")}
    out["v"] = torch.empty(n.value, dtype=torch.float32)
    p = [C.c_void_p(out[k].data_ptr()) for k in ("i", "j", "k", "l", "v")]
    check(lib().ixb_cg_table(l_max, *p, C.byref(n), C.byref(npaths)))
    out["npaths"] = npaths.value
    return out
