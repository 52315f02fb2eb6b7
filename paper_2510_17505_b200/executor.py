"""`execute_mode("b200", ...)` — the drop-in evaluator dispatch.

Mirrors execute_mode (driver.cpp:235-265 / driver.hpp:99-101): parse the
indirect Einsum (grammar of expr.cpp:36-181), match it structurally to one
of the hot-path workloads, bind operands on the device and run the sm_100a
kernel. Statements outside the hot path raise — there is no CPU fallback.

Host inputs (numpy fp64/int64 as the reference stores them, or torch CPU
tensors) are converted to the device formats (int32 indices, fp32/bf16
values) and copied in; results come back as float64 numpy arrays with the
output's shape, like ModeResult::result.
"""
import re
import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np
import torch

from . import api
from .abi import BindError, IndexRangeError, ParseError, ShapeError, check, lib

# ---------------------------------------------------------------- grammar


@dataclass
class Index:
    var: str = ""
    tensor: str = ""            # non-empty => indirect
    args: List[str] = field(default_factory=list)

    @property
    def direct(self):
        return not self.tensor


@dataclass
class Access:
    tensor: str
    indices: List[Index]


@dataclass
class Stmt:
    output: Access
    inputs: List[Access]
    accumulate: bool
    vars: List[str]


class _Parser:
    """expr.cpp:36-181 restated (same tokens, messages and positions)."""

    def __init__(self, s):
        self.s, self.pos = s, 0

    def fail(self, msg, pos=None):
        p = self.pos if pos is None else pos
        raise ParseError(2, f"{msg} (at position {p})")

    def ws(self):
        while self.pos < len(self.s) and self.s[self.pos].isspace():
            self.pos += 1

    def peek(self, c):
        self.ws()
        return self.pos < len(self.s) and self.s[self.pos] == c

    def consume(self, tok):
        self.ws()
        if self.s.startswith(tok, self.pos):
            self.pos += len(tok)
            return True
        return False

    def expect(self, c):
        self.ws()
        if self.pos >= len(self.s) or self.s[self.pos] != c:
            self.fail(f"expected '{c}'")
        self.pos += 1

    def ident(self, what):
        self.ws()
        m = re.compile(r"[A-Za-z_][A-Za-z0-9_]*").match(self.s, self.pos)
        if not m:
            self.fail(f"expected {what}")
        self.pos = m.end()
        return m.group(0)

    def access(self):
        name = self.ident("tensor name")
        self.expect("[")
        idx = [self.index()]
        self.ws()
        while self.consume(","):
            idx.append(self.index())
            self.ws()
        self.expect("]")
        return Access(name, idx)

    def index(self):
        name = self.ident("index variable")
        self.ws()
        if not self.peek("["):
            return Index(var=name)
        self.expect("[")
        args = [self.arg()]
        self.ws()
        while self.consume(","):
            args.append(self.arg())
            self.ws()
        self.expect("]")
        return Index(tensor=name, args=args)

    def arg(self):
        self.ws()
        at = self.pos
        v = self.ident("indirection argument")
        self.ws()
        if self.peek("["):
            self.fail("nested indirection is not supported", at)
        return v

    def stmt(self):
        out = self.access()
        self.ws()
        if self.consume("+="):
            acc = True
        elif self.consume("="):
            acc = False
        else:
            self.fail("expected '=' or '+='")
        ins = [self.access()]
        self.ws()
        while self.consume("*"):
            ins.append(self.access())
            self.ws()
        if self.pos != len(self.s):
            self.fail("unexpected trailing input")
        vs = []
        for a in [out] + ins:
            for i in a.indices:
                for v in ([i.var] if i.direct else i.args):
                    if v not in vs:
                        vs.append(v)
        return Stmt(out, ins, acc, vs)


def parse(expr: str) -> Stmt:
    return _Parser(expr).stmt()


# ------------------------------------------------------- workload matching
WORKLOADS = ("groupcoo_spmm", "coo_spmm", "blockgroupcoo_spmm", "grouped_sparse_conv",
             "sparse_conv", "grouped_tp", "grouped_tp_shared")


def _sig(a: Access):
    """Structural signature with variables renamed by first appearance."""
    return [(i.direct, i.var if i.direct else tuple(i.args)) for i in a.indices]


def match_workload(st: Stmt):
    """Returns (workload, binding dict role -> tensor name) or (None, None)."""
    o, ins = st.output, st.inputs
    d = lambda i: i.direct
    try:
        # C[AM[p],n] += AV[p,q] * B[AK[p,q],n]   (and the COO form with [p])
        if len(ins) == 2 and len(o.indices) == 2 and not d(o.indices[0]) and d(o.indices[1]):
            v, b = ins
            p_args = o.indices[0].args
            n = o.indices[1].var
            if (len(b.indices) == 2 and not d(b.indices[0]) and d(b.indices[1])
                    and b.indices[1].var == n and all(d(i) for i in v.indices)):
                vv = [i.var for i in v.indices]
                if len(p_args) == 1 and vv == p_args + b.indices[0].args[1:] and \
                        b.indices[0].args[0] == p_args[0]:
                    wl = "groupcoo_spmm" if len(vv) == 2 else "coo_spmm"
                    if len(vv) in (1, 2) and b.indices[0].args == vv:
                        return wl, {"C": o.tensor, "AM": o.indices[0].tensor, "AV": v.tensor,
                                    "B": b.tensor, "AK": b.indices[0].tensor}
        # C[AM[p],bm,n] += AV[p,q,bm,bk] * B[AK[p,q],bk,n]
        if len(ins) == 2 and len(o.indices) == 3 and not d(o.indices[0]):
            v, b = ins
            p, bm, n = o.indices[0].args, o.indices[1].var, o.indices[2].var
            if (len(v.indices) == 4 and all(d(i) for i in v.indices) and len(b.indices) == 3
                    and not d(b.indices[0])):
                q = v.indices[1].var
                bk = v.indices[3].var
                if ([i.var for i in v.indices] == [p[0], q, bm, bk] and
                        b.indices[0].args == [p[0], q] and b.indices[1].var == bk and
                        b.indices[2].var == n):
                    return "blockgroupcoo_spmm", {"C": o.tensor, "AM": o.indices[0].tensor,
                                                  "AV": v.tensor, "B": b.tensor,
                                                  "AK": b.indices[0].tensor}
        # Out[MAPX[p,q],m] += MAPV[p,q] * In[MAPY[p,q],c] * Weight[MAPZ[p],c,m]
        if len(ins) == 3 and len(o.indices) == 2 and not d(o.indices[0]):
            v, x, w = ins
            pq, m = o.indices[0].args, o.indices[1].var
            if (all(d(i) for i in v.indices) and [i.var for i in v.indices] == pq and
                    len(x.indices) == 2 and x.indices[0].args == pq and d(x.indices[1]) and
                    len(w.indices) == 3 and not d(w.indices[0]) and
                    w.indices[0].args == pq[:1] and w.indices[1].var == x.indices[1].var and
                    w.indices[2].var == m):
                wl = "grouped_sparse_conv" if len(pq) == 2 else "sparse_conv"
                return wl, {"Out": o.tensor, "MAPX": o.indices[0].tensor, "MAPV": v.tensor,
                            "In": x.tensor, "MAPY": x.indices[0].tensor, "Weight": w.tensor,
                            "MAPZ": w.indices[0].tensor}
        # Z[b,CGI[p,q],w] += CGV[p,q] * X[b,CGJ[p,q],u] * Y[b,CGK[p,q]] * W[(b,)CGL[p],u,w]
        if len(ins) == 4 and len(o.indices) == 3 and d(o.indices[0]) and not d(o.indices[1]):
            v, x, y, w = ins
            b, pq, wv = o.indices[0].var, o.indices[1].args, o.indices[2].var
            ok = ([i.var for i in v.indices] == pq and len(x.indices) == 3 and
                  x.indices[0].var == b and x.indices[1].args == pq and d(x.indices[2]) and
                  len(y.indices) == 2 and y.indices[0].var == b and y.indices[1].args == pq)
            u = x.indices[2].var if ok else None
            if ok and len(w.indices) == 4 and w.indices[0].var == b and \
                    w.indices[1].args == pq[:1] and w.indices[2].var == u and \
                    w.indices[3].var == wv:
                wl = "grouped_tp"
            elif ok and len(w.indices) == 3 and w.indices[0].args == pq[:1] and \
                    w.indices[1].var == u and w.indices[2].var == wv:
                wl = "grouped_tp_shared"
            else:
                wl = None
            if wl:
                return wl, {"Z": o.tensor, "CGI": o.indices[1].tensor, "CGV": v.tensor,
                            "X": x.tensor, "CGJ": x.indices[1].tensor, "Y": y.tensor,
                            "CGK": y.indices[1].tensor, "W": w.tensor,
                            "CGL": w.indices[1 if wl == "grouped_tp" else 0].tensor}
    except (AttributeError, IndexError):
        pass
    return None, None


# ------------------------------------------------------------- execution
@dataclass
class ModeResult:
    """ModeResult (driver.hpp:91-97)."""
    result: np.ndarray
    counters: Dict[str, int]
    kernel_count: int
    wall_ms: float


def _to_dev(x, dtype, device, name=None):
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x))
    if dtype == torch.int32 and x.dtype in (torch.int64, torch.uint64) and x.numel():
        # device indices are int32: a value beyond it is out of range for any
        # extent and must raise, not wrap (narrowing is checked, not truncated)
        lo, hi = int(x.min()), int(x.max())
        if lo < -2**31 or hi >= 2**31:
            bad = int((x < -2**31).logical_or(x >= 2**31).nonzero()[0, 0])
            v = int(x.reshape(-1)[bad])
            raise IndexRangeError(6, f"index tensor {name} value {v} at position [{bad}] "
                                     "exceeds the device's int32 range")
    return x.to(device=device, dtype=dtype, non_blocking=True).contiguous()


def _check_shape(name, t, shape):
    if tuple(t.shape) != tuple(shape):
        raise BindError(3, f"tensor {name} shape does not match the statement")


def device_tolerance(expr):
    """Relative tolerance of the b200 result against the fp64 oracle (north_star;
    integration/ixsum_b200_mode.cpp device_tolerance): GroupCOO / COO SpMM run
    fp32 end to end (compensated sums) -> 1e-5; the tensor-core paths take
    bf16 operands with fp32 accumulation -> 1e-2."""
    wl, _ = match_workload(parse(expr))
    return 1e-5 if wl in ("groupcoo_spmm", "coo_spmm") else 1e-2


def execute_mode(mode, expr, tensors, out_name, out, value_dtype=None, device=None,
                 flags=0):
    """execute_mode("b200", ...) over host or device tensors.

    `tensors`: name -> array (reference layout: indices int64, values fp64 —
    or already-device int32 / fp32 / bf16 torch tensors). `out` primes `+=`.
    value_dtype: torch.float32 (default for GroupCOO SpMM and int checks) or
    torch.bfloat16 (default for the tensor-core paths).
    """
    if mode != "b200":
        raise ValueError(f"unknown mode: {mode}")
    device = device or torch.device("cuda", torch.cuda.current_device())
    t0 = time.perf_counter()
    st = parse(expr)
    if st.output.tensor != out_name:
        raise BindError(3, f"unbound tensor {st.output.tensor}")
    for a in st.inputs:
        for nm in [a.tensor] + [i.tensor for i in a.indices if not i.direct]:
            if nm not in tensors:
                raise BindError(3, f"unbound tensor {nm}")
    for nm in [i.tensor for i in st.output.indices if not i.direct]:  # output indirection
        if nm not in tensors:
            raise BindError(3, f"unbound tensor {nm}")
    wl, bind = match_workload(st)
    if wl is None:
        raise ShapeError(4, f"statement is outside the B200 hot path: {expr}")
    ix = lambda n: _to_dev(tensors[bind[n]], torch.int32, device, bind[n])
    acc = st.accumulate
    o_np = out if isinstance(out, np.ndarray) else out.cpu().numpy()
    launches0 = lib().ixb_launch_count()
    if wl in ("groupcoo_spmm", "coo_spmm"):
        vd = value_dtype or torch.float32
        AM, AK = ix("AM"), ix("AK")
        AV = _to_dev(tensors[bind["AV"]], vd, device)
        B = _to_dev(tensors[bind["B"]], vd, device)
        if vd != torch.float32:
            raise ShapeError(4, "GroupCOO SpMM runs in fp32")
        C = _to_dev(o_np, torch.float32, device)
        G = AM.numel()
        g = AV.numel() // max(G, 1) if G else (AK.shape[1] if AK.dim() == 2 else 1)
        _check_shape(bind["AK"], AK, (G, g) if wl == "groupcoo_spmm" else (G,))
        _check_shape(bind["AV"], AV, AK.shape)
        api.spmm_groupcoo(AM, AK, AV.reshape(G, g), B, C, accumulate=acc, flags=flags)
        counters = api.count_accesses_model(G, g, B.shape[1])
        res = C
    elif wl == "blockgroupcoo_spmm":
        vd = value_dtype or torch.bfloat16
        AM, AK = ix("AM"), ix("AK")
        AV = _to_dev(tensors[bind["AV"]], vd, device)
        B = _to_dev(tensors[bind["B"]], vd, device)
        C = _to_dev(o_np, torch.float32, device)
        G, g, bm, bk = AV.shape
        api.spmm_blockgroupcoo(AM, AK, AV, B, C, accumulate=acc, flags=flags)
        counters = api.count_accesses_model(G, g, bm * B.shape[2])
        res = C
    elif wl in ("grouped_sparse_conv", "sparse_conv"):
        vd = value_dtype or torch.bfloat16
        MAPZ, MAPX, MAPY = ix("MAPZ"), ix("MAPX"), ix("MAPY")
        if wl == "sparse_conv":  # COO form = g 1 groups
            MAPX, MAPY = MAPX.reshape(-1, 1), MAPY.reshape(-1, 1)
        MAPV = _to_dev(tensors[bind["MAPV"]], torch.float32, device).reshape(MAPX.shape)
        In = _to_dev(tensors[bind["In"]], vd, device)
        W = _to_dev(tensors[bind["Weight"]], vd, device)
        Out = _to_dev(o_np, torch.float32, device)
        api.conv_grouped(MAPZ, MAPX, MAPY, MAPV, In, W, Out, accumulate=acc, flags=flags)
        counters = api.count_accesses_model(MAPX.shape[0], MAPX.shape[1], W.shape[2])
        res = Out
    else:
        vd = value_dtype or torch.bfloat16
        CGL, CGI, CGJ, CGK = ix("CGL"), ix("CGI"), ix("CGJ"), ix("CGK")
        CGV = _to_dev(tensors[bind["CGV"]], torch.float32, device)
        X = _to_dev(tensors[bind["X"]], vd, device)
        Y = _to_dev(tensors[bind["Y"]], vd, device)
        W = _to_dev(tensors[bind["W"]], vd, device)
        Z = _to_dev(o_np, torch.float32, device)
        api.tp_grouped(CGL, CGI, CGJ, CGK, CGV, X, Y, W, Z, accumulate=acc, flags=flags)
        counters = api.count_accesses_model(CGI.shape[0], CGI.shape[1],
                                            X.shape[0] * W.shape[-1])
        res = Z
    result = res.double().cpu().numpy().reshape(o_np.shape)
    wall = (time.perf_counter() - t0) * 1e3
    return ModeResult(result, counters, int(lib().ixb_launch_count() - launches0), wall)
