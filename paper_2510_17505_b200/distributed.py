"""Row-group / point-block sharding across GPUs.

One process per GPU (torch.distributed; NCCL over NVLink on the GPU box,
gloo in the CPU tests). Groups are sorted by their output coordinate, so a
shard is a contiguous range of groups cut only where the coordinate changes
(ixb_shard_groups): every output row has exactly one owner and keeps its
summation order, hence the gathered result is bit-identical for any number
of ranks. The dense operand is replicated; the only collective is the final
all-gather of the output row slabs (padded to the largest slab, one
all_gather_into_tensor).

The native path (Comm, ShardPlan, *_sharded at the end) does the same
behind the C-ABI: libixb's own NCCL communicator, C++ shard/chunk planning,
each rank writing straight into its rows of the full output, and the
all-gather as in-place NCCL broadcasts overlapping the next chunk's kernel.
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


class SlabGather:
    """Preallocated form of gather_rows for repeated steps: the rank writes
    its slab straight into `local` (a view of the padded send buffer), and
    __call__ runs one all_gather_into_tensor plus one index_select that drops
    the padding into `out` (the full output, identical on every rank)."""

    def __init__(self, shards, rank, tail, dtype, device, group=None):
        self.group, self.world = group, len(shards)
        self.maxrows = max(max(s.r1 - s.r0 for s in shards), 1)
        s = shards[rank]
        self.pad = torch.zeros((self.maxrows,) + tuple(tail), dtype=dtype, device=device)
        self.local = self.pad[: s.r1 - s.r0]
        self.buf = torch.empty((self.world * self.maxrows,) + tuple(tail), dtype=dtype,
                               device=device)
        idx = [torch.arange(r * self.maxrows, r * self.maxrows + (x.r1 - x.r0))
               for r, x in enumerate(shards)]
        self.idx = torch.cat(idx).to(device)
        self.out = torch.empty((shards[-1].r1,) + tuple(tail), dtype=dtype, device=device)

    def __call__(self):
        import torch.distributed as dist
        if self.world == 1:
            return self.local
        dist.all_gather_into_tensor(self.buf, self.pad, group=self.group)
        torch.index_select(self.buf, 0, self.idx, out=self.out)
        return self.out


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
    local = torch.zeros((s.r1 - s.r0, B.shape[1]), dtype=torch.float32, device=B.device)
    spmm_groupcoo_into(fmt.AM[s.g0:s.g1], fmt.AK[s.g0:s.g1], fmt.AV[s.g0:s.g1], fmt.group_size,
                       B, s, local, flags, stream)
    return local


def spmm_groupcoo_into(AM, AK, AV, g, B, s, local, flags=2, stream=None):
    """K3 over a shard's groups (AM/AK/AV already sliced to [g0, g1)) `+=`
    into the ZEROED slab `local` = rows [s.r0, s.r1). No allocation: the C
    pointer is offset by -r0 rows so absolute row ids land in the slab, and
    `+=` means no zero-fill outside the rank's rows."""
    import ctypes as C

    from .abi import check, lib
    if AM.numel() == 0:
        return local
    st = stream if stream is not None else torch.cuda.current_stream()
    check(lib().ixb_spmm_groupcoo(C.c_void_p(AM.data_ptr()), C.c_void_p(AK.data_ptr()),
                                  C.c_void_p(AV.data_ptr()), AM.numel(), g,
                                  C.c_void_p(B.data_ptr()), B.shape[0], B.shape[1],
                                  C.c_void_p(_row_view_ptr(local, s.r0)), s.r1, 1, flags,
                                  C.c_void_p(st.cuda_stream)))
    return local


# ----------------------------------------------------------- BlockGroupCOO
def sharded_spmm_blockgroupcoo(fmt, B, shards, rank, group=None, flags=2, stream=None):
    """Block-row shards of C[AM[p],bm,n] = AV[p,q,bm,bk] * B[AK[p,q],bk,n]
    (shard_plan over the block-row coordinate AM); all ranks gather C."""
    local = spmm_blockgroupcoo_slab(fmt, B, shards[rank], flags, stream)
    return gather_rows(local, shards, rank, group)


def spmm_blockgroupcoo_slab(fmt, B, s, flags=2, stream=None):
    """K4 over one shard's groups into that shard's block-row slab [r1-r0, bm, N]."""
    local = torch.zeros((s.r1 - s.r0, fmt.AV.shape[2], B.shape[2]), dtype=torch.float32,
                        device=B.device)
    spmm_blockgroupcoo_into(fmt.AM[s.g0:s.g1], fmt.AK[s.g0:s.g1], fmt.AV[s.g0:s.g1], B, s, local,
                            flags, stream)
    return local


def spmm_blockgroupcoo_into(AM, AK, AV, B, s, local, flags=2, stream=None):
    """K4 `+=` into the zeroed block-row slab `local` (see spmm_groupcoo_into)."""
    import ctypes as C

    from .abi import check, lib
    if AM.numel() == 0:
        return local
    G, g, bm, bk = AV.shape
    st = stream if stream is not None else torch.cuda.current_stream()
    check(lib().ixb_spmm_blockgroupcoo(
        C.c_void_p(AM.data_ptr()), C.c_void_p(AK.data_ptr()), C.c_void_p(AV.data_ptr()), G, g,
        bm, bk, C.c_void_p(B.data_ptr()), B.shape[0], B.shape[2],
        C.c_void_p(_row_view_ptr(local, s.r0)), s.r1, 1, flags, C.c_void_p(st.cuda_stream)))
    return local


# ----------------------------------------------------------- sparse conv
def point_blocks(n_out, world):
    """Contiguous output-voxel blocks (voxels are in sorted order, so a block
    is a spatially compact slab) as Shards (groups unused)."""
    bounds = [(n_out * r) // world for r in range(world + 1)]
    return [Shard(0, 0, bounds[r], bounds[r + 1]) for r in range(world)]


def shard_map(mo, mi, mz, s):
    """The pairs of a kernel map (numpy or torch, any order) whose output
    voxel is in [s.r0, s.r1), output index rebased to the slab. Order is
    kept, so a canonical (offset, out) map stays canonical."""
    keep = (mo >= s.r0) & (mo < s.r1)
    return mo[keep] - s.r0, mi[keep], mz[keep]


def conv_shard_plan(mo, mi, mz, n_in, s, g, n_off=27):
    """Point-block shard of a kernel map: keep the pairs whose
    output voxel lies in [s.r0, s.r1), rebase their output index, and group
    them by offset exactly as the full map (the canonical (z, x) order is
    kept by the filter). In is replicated, so input indices stay global.
    Returns a ConvPlan over the slab's n_out = s.r1 - s.r0 rows."""
    mo_l, mi_l, mz_l = shard_map(mo, mi, mz, s)
    n_local = s.r1 - s.r0
    ones = torch.ones(mo_l.numel(), dtype=torch.float32, device=mo.device)
    gt = api.group_coo_tensor([n_local, n_in, n_off], [mo_l, mi_l, mz_l], ones, 2, g,
                              canonical=True)
    plan = api.ConvPlan(gt.group_coord, gt.member_coords[0], gt.member_coords[1], gt.values,
                        n_in, n_off, n_local)
    plan.keep_map = gt
    return plan


def sharded_conv(plan_local, In, Weight, shards, rank, group=None):
    """Rank `rank` runs its point-block plan into its Out slab; all ranks
    gather the full Out."""
    s = shards[rank]
    local = torch.empty((s.r1 - s.r0, Weight.shape[2]), dtype=torch.float32, device=In.device)
    if s.r1 > s.r0:
        plan_local.run(In, Weight, local, accumulate=False)
    return gather_rows(local, shards, rank, group)


# ----------------------------------------------------------- tensor product
def edge_blocks(batch, world):
    """Contiguous edge ranges (X, Y, Z are sharded; W is replicated)."""
    return point_blocks(batch, world)


def sharded_tp(plan, X, Y, W, shards, rank, group=None, gather=True):
    """Rank `rank` evaluates Z for its edge range; the all-gather of Z is only
    needed when every rank wants the full output."""
    s = shards[rank]
    local = torch.empty((s.r1 - s.r0, plan.ni, plan.Wd), dtype=torch.float32, device=X.device)
    if s.r1 > s.r0:
        plan.run(X[s.r0:s.r1], Y[s.r0:s.r1], W, local, accumulate=False)
    return gather_rows(local, shards, rank, group) if gather else local


# ----------------------------------------------- C-ABI sharded evaluation
# The native multi-GPU path (include/ixb.h "Sharded evaluation"): NCCL
# communicator owned by libixb, shard + chunk plan in C++, every rank writing
# its rows straight into the FULL output and the all-gather (grouped in-place
# broadcasts) overlapping the next chunk's kernel. The torch.distributed
# helpers above remain for CPU/gloo checks of the partitioning.
SHARD_NO_COMM, SHARD_COMM_ONLY = 8, 16


class Comm:
    """libixb's NCCL communicator over the ranks of `group` (default: the
    whole job). Rank 0's id travels over torch.distributed (any backend)."""

    def __init__(self, world, rank, group=None):
        import ctypes as C

        from .abi import check, lib
        self.world, self.rank = world, rank
        idb = (C.c_char * 128)()
        if rank == 0 and world == 1:
            check(lib().ixb_comm_unique_id(idb))
        if world > 1:
            import torch.distributed as dist
            if rank == 0:
                check(lib().ixb_comm_unique_id(idb))
            obj = [bytes(idb)]
            dist.broadcast_object_list(obj, src=0, group=group)
            C.memmove(idb, obj[0], 128)
        self.h = C.c_void_p()
        check(lib().ixb_comm_init(idb, world, rank, C.byref(self.h)))

    def broadcast(self, *tensors, root=0, stream=None):
        """In-place NCCL broadcast of device tensors from `root` (replicating
        the format and the dense operand once, outside any timed step)."""
        import ctypes as C

        from .abi import check, lib
        for t in tensors:
            assert t.is_contiguous() and t.is_cuda
            check(lib().ixb_comm_broadcast(self.h, C.c_void_p(t.data_ptr()),
                                           t.numel() * t.element_size(), root, _stream(stream)))

    def __del__(self):
        if getattr(self, "h", None):
            try:
                from .abi import lib
                lib().ixb_comm_free(self.h)
            except Exception:  # interpreter shutdown: the process exit frees it
                pass
            self.h = None


class ShardPlan:
    """Row-aligned group shards of a sorted group-coordinate array (the
    replicated format's AM, on the device), each cut into `nchunks`
    row-aligned chunks (ixb_shard_plan_create)."""

    def __init__(self, AM, rows, world, rank, nchunks=4, stream=None):
        import ctypes as C

        from .abi import check, lib
        self.world, self.rank, self.nchunks, self.rows = world, rank, nchunks, rows
        st = stream if stream is not None else torch.cuda.current_stream()
        self.h = C.c_void_p()
        check(lib().ixb_shard_plan_create(C.c_void_p(AM.data_ptr()), AM.numel(), rows, world,
                                          rank, nchunks, C.c_void_p(st.cuda_stream),
                                          C.byref(self.h)))

    def chunk(self, rank, c):
        """(g0, g1, r0, r1) of chunk c of `rank`."""
        import ctypes as C

        from .abi import check, lib
        v = [C.c_int64() for _ in range(4)]
        check(lib().ixb_shard_plan_chunk(self.h, rank, c, *[C.byref(x) for x in v]))
        return tuple(x.value for x in v)

    def rows_of(self, rank):
        return self.chunk(rank, 0)[2], self.chunk(rank, self.nchunks - 1)[3]

    def __del__(self):
        if getattr(self, "h", None):
            try:
                from .abi import lib
                lib().ixb_shard_plan_free(self.h)
            except Exception:  # interpreter shutdown: the process exit frees it
                pass
            self.h = None


def _stream(stream):
    import ctypes as C
    st = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(st.cuda_stream)


def spmm_groupcoo_sharded(plan, fmt, B, C_full, comm=None, flags=2, stream=None):
    """Rank plan.rank evaluates its chunks of `C = AV * B[AK]` into its rows
    of C_full [M, N] and all ranks' rows are broadcast in place: every rank
    ends with the whole C (comm None: world 1 or flags & SHARD_NO_COMM)."""
    import ctypes as C

    from .abi import check, lib
    check(lib().ixb_spmm_groupcoo_sharded(
        plan.h, C.c_void_p(fmt.AK.data_ptr()), C.c_void_p(fmt.AV.data_ptr()), fmt.group_size,
        C.c_void_p(B.data_ptr()), B.shape[0], B.shape[1], C.c_void_p(C_full.data_ptr()), flags,
        comm.h if comm is not None else None, _stream(stream)))
    return C_full


def spmm_blockgroupcoo_sharded(plan, fmt, B, C_full, comm=None, flags=2, stream=None):
    """Block-row form of spmm_groupcoo_sharded: C_full [MB, 16, N]."""
    import ctypes as C

    from .abi import check, lib
    G, g, bm, bk = fmt.AV.shape
    check(lib().ixb_spmm_blockgroupcoo_sharded(
        plan.h, C.c_void_p(fmt.AK.data_ptr()), C.c_void_p(fmt.AV.data_ptr()), g, bm, bk,
        C.c_void_p(B.data_ptr()), B.shape[0], B.shape[2], C.c_void_p(C_full.data_ptr()), flags,
        comm.h if comm is not None else None, _stream(stream)))
    return C_full


def conv_sharded(local_plan, In, Weight, Out_full, world, rank, nchunks=4, comm=None, flags=0,
                 stream=None):
    """Rank `rank` runs its point-block plan (conv_shard_plan over
    point_blocks(n, world)[rank]) in `nchunks` tile chunks into its rows of
    Out_full [n, 64]; the rows are all-gathered in place as they finish."""
    import ctypes as C

    from .abi import check, lib
    check(lib().ixb_conv_plan_run_sharded(
        local_plan.h if local_plan is not None else None, C.c_void_p(In.data_ptr()), In.shape[1],
        C.c_void_p(Weight.data_ptr()), Weight.shape[2], C.c_void_p(Out_full.data_ptr()),
        Out_full.shape[0], world, rank, nchunks, flags, comm.h if comm is not None else None,
        _stream(stream)))
    return Out_full
