"""Row-group / point-block sharding across GPUs.

One process per GPU (torch.distributed; NCCL over NVLink on the GPU box,
gloo in the CPU tests). Groups are sorted by their output coordinate, so a
shard is a contiguous range of groups cut only where the coordinate changes
(ixb_shard_groups): every output row has exactly one owner and keeps its
summation order, hence the gathered result is bit-identical for any number
of ranks. The dense operand is replicated; the only collective is the final
all-gather of the output row slabs (padded to the largest slab, one
all_gather_into_tensor).
"""
from dataclasses import dataclass
from typing import List

import numpy as np
import torch

from . import api


@dataclass
class Shard:
    g0: int  # first group
    g1: int  # one past the last group
    r0: int  # first output row owned
    r1: int  # one past the last output row owned


def shard_plan(group_coord_host, rows, world) -> List[Shard]:
    """Contiguous group ranges of ~equal size cut at row boundaries, and the
    output row slab each rank owns (empty rows between shards go to the
    shard after them; the last shard owns the tail)."""
    gc = np.ascontiguousarray(group_coord_host, dtype=np.int32)
    G = gc.size
    bounds = api.shard_groups(gc, world) if G else np.zeros(world + 1, np.int64)
    starts = [0]
    for r in range(1, world):
        b = int(bounds[r])
        starts.append(int(gc[b]) if b < G else rows)
    starts.append(rows)
    for r in range(1, world + 1):  # monotone (a rank may own an empty slab)
        starts[r] = max(starts[r], starts[r - 1])
    return [Shard(int(bounds[r]), int(bounds[r + 1]), starts[r], starts[r + 1])
            for r in range(world)]


def gather_rows(local, shards, rank, group=None):
    """All-gather of the ranks' output slabs [r1-r0, ...] into the full output
    (every rank receives it). One padded all_gather_into_tensor."""
    import torch.distributed as dist
    world = len(shards)
    tail = tuple(local.shape[1:])
    width = int(np.prod(tail)) if tail else 1
    maxrows = max(s.r1 - s.r0 for s in shards)
    pad = torch.zeros((maxrows, width), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local.reshape(local.shape[0], width)
    buf = torch.empty((world * maxrows, width), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(buf, pad, group=group)
    rows = shards[-1].r1
    out = torch.empty((rows, width), dtype=local.dtype, device=local.device)
    for r, s in enumerate(shards):
        out[s.r0:s.r1] = buf[r * maxrows: r * maxrows + (s.r1 - s.r0)]
    return out.reshape((rows,) + tail)


def _row_view_ptr(local, r0):
    """Device pointer of row 0 of the full output given the slab for rows [r0, ...)."""
    row_bytes = local[0].numel() * local.element_size() if local.shape[0] else 0
    return local.data_ptr() - r0 * row_bytes


def sharded_spmm_groupcoo(fmt, B, shards, rank, group=None, flags=2, stream=None):
    """Rank `rank` evaluates its shard of C[AM[p],n] = AV[p,q] * B[AK[p,q],n]
    into its slab, then all ranks gather the full C. fmt: device GroupCoo."""
    local = spmm_groupcoo_slab(fmt, B, shards[rank], flags, stream)
    return gather_rows(local, shards, rank, group)


def spmm_groupcoo_slab(fmt, B, s, flags=2, stream=None):
    """K3 over one shard's groups into that shard's output slab [r1-r0, N]."""
    import ctypes as C

    from .abi import check, lib
    N = B.shape[1]
    local = torch.zeros((s.r1 - s.r0, N), dtype=torch.float32, device=B.device)
    if s.g1 > s.g0:
        AM, AK, AV = fmt.AM[s.g0:s.g1], fmt.AK[s.g0:s.g1], fmt.AV[s.g0:s.g1]
        st = stream if stream is not None else torch.cuda.current_stream()
        # `+=` into a zeroed slab: no zero-fill outside the rank's rows; the C
        # pointer is offset so absolute row ids land inside the slab
        check(lib().ixb_spmm_groupcoo(C.c_void_p(AM.data_ptr()), C.c_void_p(AK.data_ptr()),
                                      C.c_void_p(AV.data_ptr()), s.g1 - s.g0, fmt.group_size,
                                      C.c_void_p(B.data_ptr()), B.shape[0], N,
                                      C.c_void_p(_row_view_ptr(local, s.r0)), s.r1, 1, flags,
                                      C.c_void_p(st.cuda_stream)))
    return local
