"""Reference-shaped builders and evaluators over libixb.so.

Device tensors are torch CUDA tensors (plumbing only). Index arrays are
int32, values float32 or bfloat16. Each function cites the reference entry
point it replaces.
"""
import ctypes as C
from dataclasses import dataclass
from typing import List, Optional

import torch

from .abi import ShapeError, check, lib

# ixb_dtype codes: evaluators take f32/bf16; builders also move f64 (and the
# sorted-run packs int64) values unchanged
_DT = {torch.float32: 0, torch.bfloat16: 1, torch.float64: 2, torch.int64: 4}


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _dtype_code(t):
    if t.dtype not in _DT:
        raise ShapeError(4, f"unsupported value dtype {t.dtype}; use float32, bfloat16 or float64")
    return _DT[t.dtype]


def _dev(t, dtype=None):
    if not t.is_cuda:
        raise ShapeError(4, "ixb operands must be CUDA tensors")
    if dtype is not None and t.dtype != dtype:
        raise ShapeError(4, f"expected {dtype}, got {t.dtype}")
    return t.contiguous()


class _Plan:
    def __init__(self):
        self.h = C.c_void_p()

    def __del__(self):
        if self.h:
            lib().ixb_pack_free(self.h)
            self.h = C.c_void_p()


@dataclass
class GroupCoo:
    """GroupCooMatrix (formats.hpp:38-51) on the device."""
    rows: int
    cols: int
    group_dim: int
    group_size: int
    AM: torch.Tensor     # group_coord [G] int32
    AK: torch.Tensor     # member_coord [G, g] int32
    AV: Optional[torch.Tensor]  # values [G, g]
    mask: torch.Tensor   # pad_mask [G, g] uint8

    def num_groups(self):
        return self.AM.numel()


@dataclass
class BlockGroupCoo:
    """BlockGroupCooMatrix (formats.hpp:63-79) on the device."""
    rows: int
    cols: int
    block_rows: int
    block_cols: int
    group_dim: int
    group_size: int
    AM: torch.Tensor
    AK: torch.Tensor
    AV: torch.Tensor     # [G, g, bM, bK]
    mask: torch.Tensor
    num_blocks: int

    def num_groups(self):
        return self.AM.numel()


@dataclass
class GroupCooTensor:
    """GroupCooTensor (formats.hpp:126-139) on the device."""
    shape: List[int]
    group_dim: int
    group_size: int
    group_coord: torch.Tensor
    member_coords: List[torch.Tensor]
    member_dims: List[int]
    values: Optional[torch.Tensor]
    mask: torch.Tensor

    def num_groups(self):
        return self.group_coord.numel()


def dense_to_coo(dense, stream=None):
    """dense_to_coo (formats.hpp:26): returns (row_coord, col_coord, values)."""
    dense = _dev(dense)
    if dense.dim() != 2:
        raise ShapeError(4, f"dense_to_coo expects a rank-2 tensor, got rank {dense.dim()}")
    plan, nnz = _Plan(), C.c_int64(0)
    check(lib().ixb_dense_to_coo_plan(_ptr(dense), _dtype_code(dense), dense.shape[0],
                                      dense.shape[1], _stream(stream), C.byref(plan.h),
                                      C.byref(nnz)))
    n = nnz.value
    r = torch.empty(n, dtype=torch.int32, device=dense.device)
    c = torch.empty(n, dtype=torch.int32, device=dense.device)
    v = torch.empty(n, dtype=dense.dtype, device=dense.device)
    check(lib().ixb_dense_to_coo_pack(plan.h, _ptr(r), _ptr(c), _ptr(v), _stream(stream)))
    return r, c, v


def coo_to_groupcoo(rows, cols, row_coord, col_coord, values, group_dim, g, canonical=False,
                    stream=None):
    """coo_to_groupcoo (formats.hpp:53). g == 0 selects g with the tuner."""
    r = _dev(row_coord, torch.int32)
    c = _dev(col_coord, torch.int32)
    v = None if values is None else _dev(values)
    plan, G, gout = _Plan(), C.c_int64(0), C.c_int64(0)
    check(lib().ixb_groupcoo_plan(_ptr(r), _ptr(c), r.numel(), rows, cols, int(canonical),
                                  group_dim, g, _stream(stream), C.byref(plan.h), C.byref(G),
                                  C.byref(gout)))
    G, g = G.value, gout.value
    dev = r.device
    AM = torch.empty(G, dtype=torch.int32, device=dev)
    AK = torch.empty((G, g), dtype=torch.int32, device=dev)
    AV = None if v is None else torch.empty((G, g), dtype=v.dtype, device=dev)
    mask = torch.empty((G, g), dtype=torch.uint8, device=dev)
    check(lib().ixb_groupcoo_pack(plan.h, _ptr(v), 0 if v is None else _dtype_code(v), _ptr(AM),
                                  _ptr(AK), _ptr(AV), _ptr(mask), _stream(stream)))
    return GroupCoo(rows, cols, group_dim, g, AM, AK, AV, mask)


def real_count(fmt, stream=None):
    """GroupCooMatrix::real_count (formats.cpp:105-108) of a device format."""
    n = C.c_int64(0)
    check(lib().ixb_mask_real_count(_ptr(fmt.mask), fmt.mask.numel(), _stream(stream),
                                    C.byref(n)))
    return n.value


def pad_count(fmt, stream=None):
    """GroupCooMatrix::pad_count (formats.cpp:110-113)."""
    return fmt.mask.numel() - real_count(fmt, stream)


def is_ell(fmt, stream=None):
    """is_ell (formats.cpp:202-208): one group per distinct grouped coordinate."""
    f = C.c_int(0)
    check(lib().ixb_is_ell(_ptr(fmt.AM), fmt.AM.numel(), _stream(stream), C.byref(f)))
    return bool(f.value)


def ell_view(rows, cols, row_coord, col_coord, values, group_dim=0, canonical=False,
             stream=None):
    """ell_view (formats.cpp:196-200): coo_to_groupcoo with g = max occupancy."""
    coord = _dev(row_coord if group_dim == 0 else col_coord, torch.int32)
    m = C.c_int64(0)
    check(lib().ixb_max_occupancy(_ptr(coord), coord.numel(), rows if group_dim == 0 else cols,
                                  _stream(stream), C.byref(m)))
    return coo_to_groupcoo(rows, cols, row_coord, col_coord, values, group_dim, max(m.value, 1),
                           canonical=canonical, stream=stream)


def groupcoo_to_coo(fmt, stream=None):
    """groupcoo_to_coo (formats.cpp:176-194): the real slots, canonicalized
    (row-major, the g = 1 grouping) -> (row_coord, col_coord, values) on the device."""
    n = real_count(fmt, stream)
    dev = fmt.AM.device
    r = torch.empty(n, dtype=torch.int32, device=dev)
    c = torch.empty(n, dtype=torch.int32, device=dev)
    v = None if fmt.AV is None else torch.empty(n, dtype=fmt.AV.dtype, device=dev)
    G, g = fmt.AK.shape
    check(lib().ixb_groupcoo_to_coo(_ptr(fmt.AM), _ptr(fmt.AK), _ptr(fmt.AV),
                                    0 if v is None else _dtype_code(fmt.AV), _ptr(fmt.mask), G, g,
                                    fmt.group_dim, _ptr(r), _ptr(c), _ptr(v), _stream(stream)))
    if n == 0:
        return r, c, v
    canon = coo_to_groupcoo(fmt.rows, fmt.cols, r, c, v, 0, 1, stream=stream)
    return canon.AM.clone(), canon.AK.reshape(-1).clone(), \
        None if v is None else canon.AV.reshape(-1).clone()


def dense_to_groupcoo(dense, g=0, group_dim=0, stream=None):
    """dense_to_coo + coo_to_groupcoo fused (driver.cpp:101-116 `groupcoo`/`auto`)."""
    dense = _dev(dense)
    if dense.dim() != 2:
        raise ShapeError(4, "dense_to_coo expects a rank-2 tensor")
    plan, G, gout, nnz = _Plan(), C.c_int64(0), C.c_int64(0), C.c_int64(0)
    check(lib().ixb_dense_groupcoo_plan(_ptr(dense), _dtype_code(dense), dense.shape[0],
                                        dense.shape[1], group_dim, g, _stream(stream),
                                        C.byref(plan.h), C.byref(G), C.byref(gout), C.byref(nnz)))
    G, g = G.value, gout.value
    dev = dense.device
    AM = torch.empty(G, dtype=torch.int32, device=dev)
    AK = torch.empty((G, g), dtype=torch.int32, device=dev)
    AV = torch.empty((G, g), dtype=dense.dtype, device=dev)
    mask = torch.empty((G, g), dtype=torch.uint8, device=dev)
    check(lib().ixb_dense_groupcoo_pack(plan.h, _ptr(AM), _ptr(AK), _ptr(AV), _ptr(mask),
                                        _stream(stream)))
    return GroupCoo(dense.shape[0], dense.shape[1], group_dim, g, AM, AK, AV, mask)


def dense_to_blockgroupcoo(dense, block_rows, block_cols, g, group_dim=0, stream=None):
    """dense_to_blockgroupcoo (formats.hpp:81-83). g == 0 selects g with the tuner."""
    dense = _dev(dense)
    if dense.dim() != 2:
        raise ShapeError(4, "dense_to_blockgroupcoo expects a rank-2 tensor")
    plan, G, gout, nb = _Plan(), C.c_int64(0), C.c_int64(0), C.c_int64(0)
    check(lib().ixb_blockgroupcoo_plan(_ptr(dense), _dtype_code(dense), dense.shape[0],
                                       dense.shape[1], block_rows, block_cols, g, group_dim,
                                       _stream(stream), C.byref(plan.h), C.byref(G),
                                       C.byref(gout), C.byref(nb)))
    G, g = G.value, gout.value
    dev = dense.device
    AM = torch.empty(G, dtype=torch.int32, device=dev)
    AK = torch.empty((G, g), dtype=torch.int32, device=dev)
    AV = torch.empty((G, g, block_rows, block_cols), dtype=dense.dtype, device=dev)
    mask = torch.empty((G, g), dtype=torch.uint8, device=dev)
    check(lib().ixb_blockgroupcoo_pack(plan.h, _ptr(AM), _ptr(AK), _ptr(AV), _ptr(mask),
                                       _stream(stream)))
    return BlockGroupCoo(dense.shape[0], dense.shape[1], block_rows, block_cols, group_dim, g,
                         AM, AK, AV, mask, nb.value)


def group_coo_tensor(shape, coords, values, group_dim, g, canonical=False, stream=None):
    """group_coo_tensor (formats.hpp:141). coords: list of rank int32 [nnz] tensors.
    canonical=True asserts the input is already in (group dim, other dims) order."""
    coords = [_dev(c, torch.int32) for c in coords]
    rank = len(coords)
    nnz = coords[0].numel() if rank else 0
    v = None if values is None else _dev(values)
    sh = (C.c_int64 * rank)(*shape)
    cp = (C.c_void_p * rank)(*[c.data_ptr() for c in coords])
    plan, G = _Plan(), C.c_int64(0)
    check(lib().ixb_group_coo_tensor_plan(rank, sh, cp, nnz, group_dim, g, int(canonical),
                                          _stream(stream), C.byref(plan.h), C.byref(G)))
    G = G.value
    dev = coords[0].device
    gc = torch.empty(G, dtype=torch.int32, device=dev)
    dims = [d for d in range(rank) if d != group_dim]
    mcs = [torch.empty((G, g), dtype=torch.int32, device=dev) for _ in dims]
    ov = None if v is None else torch.empty((G, g), dtype=v.dtype, device=dev)
    mask = torch.empty((G, g), dtype=torch.uint8, device=dev)
    mp = (C.c_void_p * max(len(mcs), 1))(*[m.data_ptr() for m in mcs])
    check(lib().ixb_group_coo_tensor_pack(plan.h, _ptr(v), 0 if v is None else _dtype_code(v),
                                          _ptr(gc), mp, _ptr(ov), _ptr(mask), _stream(stream)))
    return GroupCooTensor(list(shape), group_dim, g, gc, mcs, dims, ov, mask)


def emit_operands(fmt, prefix="A", suffix0="M", suffix1="K"):
    """emit_operands (formats.hpp:98-109): named arrays ready to bind."""
    gsuf = suffix0 if fmt.group_dim == 0 else suffix1
    msuf = suffix1 if fmt.group_dim == 0 else suffix0
    return {prefix + "V": fmt.AV, prefix + gsuf: fmt.AM, prefix + msuf: fmt.AK}


def tune_group_size(coord, extent, count_empty_rows=False, stream=None):
    """OccProfile::from_coo + select (tuner.hpp:18,63) on the device."""
    coord = _dev(coord, torch.int32)
    g, gs = C.c_int64(0), C.c_double(0)
    check(lib().ixb_tune_group_size(_ptr(coord), coord.numel(), extent, int(count_empty_rows),
                                    _stream(stream), C.byref(g), C.byref(gs)))
    return g.value, gs.value


def kernel_map(coords, stream=None):
    """K5: submanifold 3x3x3 kernel map (out, in, offset) ordered by (offset, out)."""
    coords = _dev(coords, torch.int32)
    h, n = C.c_void_p(), C.c_int64(0)
    check(lib().ixb_kernel_map_plan(_ptr(coords), coords.shape[0], _stream(stream), C.byref(h),
                                    C.byref(n)))
    try:
        n = n.value
        mo, mi, mz = (torch.empty(n, dtype=torch.int32, device=coords.device) for _ in range(3))
        check(lib().ixb_kernel_map_pack(h, _ptr(mo), _ptr(mi), _ptr(mz), _stream(stream)))
    finally:
        lib().ixb_kernel_map_free(h)
    return mo, mi, mz


class ConvPlan:
    """Inspector/executor form of K6: validates a grouped kernel map and
    indexes it by (output, offset) once; run() evaluates one conv."""

    def __init__(self, MAPZ, MAPX, MAPY, MAPV, n_in, n_off, n_out, flags=0, stream=None):
        self.keep = [t.contiguous() if t is not None else None for t in (MAPZ, MAPX, MAPY, MAPV)]
        MAPZ, MAPX, MAPY, MAPV = self.keep
        G, g = MAPX.shape
        self.n_in, self.n_off, self.n_out = n_in, n_off, n_out
        self._free = lib().ixb_conv_plan_free
        self.h = C.c_void_p()
        check(lib().ixb_conv_plan_create(_ptr(MAPZ), _ptr(MAPX), _ptr(MAPY), _ptr(MAPV), G, g,
                                         n_in, n_off, n_out, flags, _stream(stream),
                                         C.byref(self.h)))

    def _check(self, In, Weight, Out, host):
        if In.dim() != 2 or Weight.dim() != 3:
            raise ShapeError(4, "ConvPlan: In is [n_in, Cin], Weight [n_off, Cin, Cout]")
        cin, cout = In.shape[1], Weight.shape[2]
        _operand("In", In, (self.n_in, cin), torch.bfloat16, device=not host)
        _operand("Weight", Weight, (self.n_off, cin, cout), torch.bfloat16)
        _operand("Out", Out, (self.n_out, cout), torch.float32, device=not host)

    def run(self, In, Weight, Out, accumulate=True, flags=0, stream=None):
        self._check(In, Weight, Out, host=False)
        check(lib().ixb_conv_plan_run(self.h, _ptr(In), In.shape[1], _ptr(Weight),
                                      Weight.shape[2], _ptr(Out), int(accumulate), flags,
                                      _stream(stream)))
        return Out

    def run_host(self, In, Weight, Out, accumulate=True, flags=0, nchunks=8, stream=None):
        """In, Out: host tensors (pinned for overlap); Weight: device. Output
        tiles run in chunks as their input rows land (ixb_conv_plan_run_host)."""
        self._check(In, Weight, Out, host=True)
        check(lib().ixb_conv_plan_run_host(self.h, _ptr(In), In.shape[1], _ptr(Weight),
                                           Weight.shape[2], _ptr(Out), int(accumulate), flags,
                                           nchunks, _stream(stream)))
        return Out

    def __del__(self):
        if getattr(self, "h", None):
            self._free(self.h)
            self.h = None


def spmm_groupcoo(AM, AK, AV, B, C_out, accumulate=True, flags=0, stream=None):
    """K3: C[AM[p],n] (+)= AV[p,q] * B[AK[p,q],n] (fp32). C_out is written in place."""
    AV2 = AV if AV.dim() == 2 else AV.reshape(-1, 1)
    G, g = AV2.shape
    check(lib().ixb_spmm_groupcoo(_ptr(AM), _ptr(AK), _ptr(AV2), G, g, _ptr(B), B.shape[0],
                                  B.shape[1], _ptr(C_out), C_out.shape[0], int(accumulate),
                                  flags, _stream(stream)))
    return C_out


def spmm_blockgroupcoo(AM, AK, AV, B, C_out, accumulate=True, flags=0, stream=None):
    """K4: C[AM[p],bm,n] (+)= AV[p,q,bm,bk] * B[AK[p,q],bk,n] (bf16 -> fp32)."""
    G, g, bm, bk = AV.shape
    check(lib().ixb_spmm_blockgroupcoo(_ptr(AM), _ptr(AK), _ptr(AV), G, g, bm, bk, _ptr(B),
                                       B.shape[0], B.shape[2], _ptr(C_out), C_out.shape[0],
                                       int(accumulate), flags, _stream(stream)))
    return C_out


def conv_grouped(MAPZ, MAPX, MAPY, MAPV, In, Weight, Out, accumulate=True, flags=0,
                 stream=None):
    """K6: Out[MAPX[p,q],m] (+)= MAPV[p,q] * In[MAPY[p,q],c] * Weight[MAPZ[p],c,m]."""
    G, g = MAPX.shape
    check(lib().ixb_conv_grouped(_ptr(MAPZ), _ptr(MAPX), _ptr(MAPY), _ptr(MAPV), G, g, _ptr(In),
                                 In.shape[0], In.shape[1], _ptr(Weight), Weight.shape[0],
                                 Weight.shape[2], _ptr(Out), Out.shape[0], int(accumulate),
                                 flags, _stream(stream)))
    return Out


def tp_grouped(CGL, CGI, CGJ, CGK, CGV, X, Y, W, Z, accumulate=True, flags=0, stream=None):
    """K7: Z[b,CGI[p,q],w] (+)= CGV[p,q] * X[b,CGJ[p,q],u] * Y[b,CGK[p,q]] * W[(b,)CGL[p],u,w]."""
    G, g = CGI.shape
    batch, nj, U = X.shape
    nk = Y.shape[1]
    per_batch = W.dim() == 4
    nl, _, Wd = W.shape[-3:]
    ni = Z.shape[1]
    check(lib().ixb_tp_grouped(_ptr(CGL), _ptr(CGI), _ptr(CGJ), _ptr(CGK), _ptr(CGV), G, g,
                               _ptr(X), _ptr(Y), _ptr(W), int(per_batch), batch, ni, nj, nk, nl,
                               U, Wd, _ptr(Z), int(accumulate), flags, _stream(stream)))
    return Z


def _operand(name, t, shape, dtype, device=True):
    """Shape/dtype/device/contiguity check of a plan operand: the C-ABI only
    receives the batch or channel counts, so a mismatched tensor would be read
    or written out of bounds."""
    if tuple(t.shape) != tuple(shape):
        raise ShapeError(4, f"{name}: expected shape {list(shape)}, got {list(t.shape)}")
    if t.dtype != dtype:
        raise ShapeError(4, f"{name}: expected {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ShapeError(4, f"{name}: must be contiguous")
    if device and not t.is_cuda:
        raise ShapeError(4, f"{name}: must be a CUDA tensor")
    if not device and t.is_cuda:
        raise ShapeError(4, f"{name}: must be a host tensor")
    return t


def _host_out(C_out):
    """Host output buffer of the *_host calls: written in place, so it must be
    contiguous (a .contiguous() copy would silently drop the result)."""
    if C_out.is_cuda or not C_out.is_contiguous() or C_out.dtype != torch.float32:
        raise ShapeError(4, "C_out must be a contiguous float32 host tensor")
    return C_out


def _host(t, dtype=None):
    if t.is_cuda:
        raise ShapeError(4, "host-buffer calls take CPU tensors (pinned for full overlap)")
    if dtype is not None and t.dtype != dtype:
        raise ShapeError(4, f"expected {dtype}, got {t.dtype}")
    return t.contiguous()


def spmm_groupcoo_host(AM, AK, AV, B, C_out, accumulate=True, flags=0, nchunks=0, stream=None):
    """K3 with HOST buffers in and out (execute_mode's shape, driver.cpp:235-265):
    row-boundary chunks pipeline H2D, kernel and D2H on three streams; returns
    with C_out written. Bit-identical to spmm_groupcoo."""
    AM, AK, AV, B = _host(AM, torch.int32), _host(AK, torch.int32), _host(AV), _host(B)
    AV2 = AV if AV.dim() == 2 else AV.reshape(-1, 1)
    G, g = AV2.shape
    check(lib().ixb_spmm_groupcoo_host(_ptr(AM), _ptr(AK), _ptr(AV2), G, g, _ptr(B), B.shape[0],
                                       B.shape[1], _ptr(_host_out(C_out)), C_out.shape[0],
                                       int(accumulate), flags, nchunks, _stream(stream)))
    return C_out


def spmm_blockgroupcoo_host(AM, AK, AV, B, C_out, accumulate=True, flags=0, nchunks=0,
                            stream=None):
    """K4 with HOST buffers in and out (see spmm_groupcoo_host)."""
    AM, AK, AV, B = _host(AM, torch.int32), _host(AK, torch.int32), _host(AV), _host(B)
    G, g, bm, bk = AV.shape
    check(lib().ixb_spmm_blockgroupcoo_host(_ptr(AM), _ptr(AK), _ptr(AV), G, g, bm, bk, _ptr(B),
                                            B.shape[0], B.shape[2], _ptr(_host_out(C_out)),
                                            C_out.shape[0], int(accumulate), flags, nchunks,
                                            _stream(stream)))
    return C_out


class TpPlan:
    """Inspector/executor form of K7: validates a grouped CG table and
    reshapes it (tensor-core job table / CUDA-core slot lists) once;
    run() evaluates one tensor product for any batch. The CG tensors are
    kept alive by the plan."""

    def __init__(self, CGL, CGI, CGJ, CGK, CGV, ni, nj, nk, nl, U=64, Wd=64, w_per_batch=False,
                 flags=0, stream=None):
        self.keep = [t.contiguous() for t in (CGL, CGI, CGJ, CGK, CGV)]
        CGL, CGI, CGJ, CGK, CGV = self.keep
        G, g = CGI.shape
        self.ni, self.nj, self.nk, self.nl, self.U, self.Wd = ni, nj, nk, nl, U, Wd
        self.w_per_batch = bool(w_per_batch)
        self._free = lib().ixb_tp_plan_free
        self.h = C.c_void_p()
        check(lib().ixb_tp_plan_create(_ptr(CGL), _ptr(CGI), _ptr(CGJ), _ptr(CGK), _ptr(CGV), G,
                                       g, int(w_per_batch), ni, nj, nk, nl, U, Wd, flags,
                                       _stream(stream), C.byref(self.h)))

    @property
    def uses_tensor_cores(self):
        """True when the table runs on the V-first tcgen05 kernel."""
        return bool(lib().ixb_tp_plan_uses_tensor_cores(self.h))

    def _check(self, X, Y, W, Z, host):
        if X.dim() != 3:
            raise ShapeError(4, f"TpPlan: X is [batch, {self.nj}, {self.U}]")
        b = X.shape[0]
        _operand("X", X, (b, self.nj, self.U), torch.bfloat16, device=not host)
        _operand("Y", Y, (b, self.nk), torch.bfloat16, device=not host)
        wshape = ((b, self.nl, self.U, self.Wd) if self.w_per_batch else
                  (self.nl, self.U, self.Wd))
        _operand("W", W, wshape, torch.bfloat16)  # device in both forms
        _operand("Z", Z, (b, self.ni, self.Wd), torch.float32, device=not host)

    def run(self, X, Y, W, Z, accumulate=True, flags=0, stream=None):
        self._check(X, Y, W, Z, host=False)
        check(lib().ixb_tp_plan_run(self.h, _ptr(X), _ptr(Y), _ptr(W), X.shape[0], _ptr(Z),
                                    int(accumulate), flags, _stream(stream)))
        return Z

    def run_host(self, X, Y, W, Z, accumulate=True, flags=0, nchunks=8, stream=None):
        """X, Y, Z: host tensors (pinned for overlap); W: device. Chunked
        copy-in / evaluate / copy-out on three streams (ixb_tp_plan_run_host)."""
        self._check(X, Y, W, Z, host=True)
        check(lib().ixb_tp_plan_run_host(self.h, _ptr(X), _ptr(Y), _ptr(W), X.shape[0],
                                         _ptr(Z), int(accumulate), flags, nchunks,
                                         _stream(stream)))
        return Z

    def __del__(self):
        if getattr(self, "h", None):
            self._free(self.h)
            self.h = None


def shard_groups(group_coord_host, parts):
    """Row-boundary group shards for `parts` ranks."""
    import numpy as np
    gc = np.ascontiguousarray(group_coord_host, dtype=np.int32)
    bounds = np.zeros(parts + 1, dtype=np.int64)
    check(lib().ixb_shard_groups(gc.ctypes.data_as(C.c_void_p), gc.size, parts,
                                 bounds.ctypes.data_as(C.c_void_p)))
    return bounds


def count_accesses_model(G, g, other_pointwise_extent):
    """count_accesses_model (plan.cpp:607-631): gathers G*g, scatters G,
    atomic updates G x extent of the pointwise vars outside the group structure."""
    return {"gathers": G * g, "scatters": G, "atomic_updates": G * other_pointwise_extent}
