"""ctypes binding of libixb.so (include/ixb.h). Loud failure, no fallback."""
import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None


def lib_path():
    # IXB_LIB_PATH: load an alternative build of the same library (perf experiments)
    return os.environ.get("IXB_LIB_PATH") or os.path.join(_HERE, "libixb.so")


class IxbError(RuntimeError):
    """Base of the reference-mirroring exceptions; .code is the ixb_status."""

    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class ParseError(IxbError):       # expr.hpp:57-62, exit code 2
    pass


class BindError(IxbError):        # plan.hpp:68-70, exit code 3
    pass


class ShapeError(IxbError):       # tensor.hpp:79-81 / InferenceError, exit code 4
    pass


class IndexRangeError(IxbError):  # plan.hpp:64-66, exit code 6
    pass


class IoError(IxbError):          # tensor.hpp:75-77 (reference CLI exit code 1)
    pass


_BY_CODE = {2: ParseError, 3: BindError, 4: ShapeError, 6: IndexRangeError, 8: IoError}

_SIGS = {
    "ixb_last_error": (C.c_char_p, []),
    "ixb_version": (C.c_int, []),
    "ixb_last_index_error": (C.c_int, [C.c_void_p] * 4),
    "ixb_check_errors": (C.c_int, [C.c_void_p]),
    "ixb_sm_count": (C.c_int, []),
    "ixb_launch_count": (C.c_int64, []),
    "ixb_pack_free": (None, [C.c_void_p]),
    "ixb_dense_to_coo_plan": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_void_p,
                                        C.c_void_p, C.c_void_p]),
    "ixb_dense_to_coo_pack": (C.c_int, [C.c_void_p] * 5),
    "ixb_groupcoo_plan": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                                    C.c_int, C.c_int, C.c_int64, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_void_p]),
    "ixb_groupcoo_pack": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int] + [C.c_void_p] * 5),
    "ixb_dense_groupcoo_plan": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int,
                                          C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p]),
    "ixb_dense_groupcoo_pack": (C.c_int, [C.c_void_p] * 6),
    "ixb_blockgroupcoo_plan": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                         C.c_int64, C.c_int64, C.c_int, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_void_p]),
    "ixb_blockgroupcoo_pack": (C.c_int, [C.c_void_p] * 6),
    "ixb_group_coo_tensor_plan": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int,
                                            C.c_int64, C.c_int, C.c_void_p, C.c_void_p,
                                            C.c_void_p]),
    "ixb_group_coo_tensor_pack": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int] + [C.c_void_p] * 5),
    "ixb_tune_group_size": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_void_p,
                                      C.c_void_p, C.c_void_p]),
    "ixb_spmm_groupcoo": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                    C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int64,
                                    C.c_int, C.c_int, C.c_void_p]),
    "ixb_spmm_blockgroupcoo": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                         C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_int64,
                                         C.c_int64, C.c_void_p, C.c_int64, C.c_int, C.c_int,
                                         C.c_void_p]),
    "ixb_kernel_map_plan": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                      C.c_void_p]),
    "ixb_kernel_map_pack": (C.c_int, [C.c_void_p] * 5),
    "ixb_kernel_map_free": (None, [C.c_void_p]),
    "ixb_conv_plan_create": (C.c_int, [C.c_void_p] * 4 + [C.c_int64] * 5 +
                             [C.c_int, C.c_void_p, C.c_void_p]),
    "ixb_conv_plan_run": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                    C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "ixb_conv_plan_run_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                         C.c_int64, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                         C.c_void_p]),
    "ixb_conv_plan_free": (None, [C.c_void_p]),
    "ixb_conv_grouped": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                   C.c_int64, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p,
                                   C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_int, C.c_int,
                                   C.c_void_p]),
    "ixb_tp_grouped": (C.c_int, [C.c_void_p] * 5 + [C.c_int64, C.c_int64] + [C.c_void_p] * 3 +
                       [C.c_int] + [C.c_int64] * 7 + [C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "ixb_spmm_blockgroupcoo_host": (C.c_int, [C.c_void_p] * 3 + [C.c_int64] * 4 +
                                    [C.c_void_p] + [C.c_int64] * 2 + [C.c_void_p, C.c_int64,
                                                                      C.c_int, C.c_int, C.c_int,
                                                                      C.c_void_p]),
    "ixb_spmm_groupcoo_host": (C.c_int, [C.c_void_p] * 3 + [C.c_int64] * 2 + [C.c_void_p] +
                               [C.c_int64] * 2 + [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int,
                                                  C.c_void_p]),
    "ixb_tp_plan_create": (C.c_int, [C.c_void_p] * 5 + [C.c_int64, C.c_int64, C.c_int] +
                           [C.c_int64] * 6 + [C.c_int, C.c_void_p, C.c_void_p]),
    "ixb_tp_plan_run": (C.c_int, [C.c_void_p] * 4 + [C.c_int64, C.c_void_p, C.c_int, C.c_int,
                                                     C.c_void_p]),
    "ixb_tp_plan_free": (None, [C.c_void_p]),
    "ixb_tp_plan_uses_tensor_cores": (C.c_int, [C.c_void_p]),
    "ixb_mask_real_count": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "ixb_is_ell": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "ixb_max_occupancy": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]),
    "ixb_groupcoo_to_coo": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                      C.c_int64, C.c_int64, C.c_int, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p]),
    "ixb_tp_plan_run_host": (C.c_int, [C.c_void_p] * 4 + [C.c_int64, C.c_void_p, C.c_int,
                                                          C.c_int, C.c_int, C.c_void_p]),
    "ixb_shard_groups": (C.c_int, [C.c_void_p, C.c_int64, C.c_int, C.c_void_p]),
    "ixb_tune_brute": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                                 C.c_void_p]),
    "ixb_tune_report": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ixb_ixt_info": (C.c_int, [C.c_char_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ixb_ixt_load": (C.c_int, [C.c_char_p, C.c_void_p, C.c_int, C.c_void_p]),
    "ixb_ixt_save": (C.c_int, [C.c_char_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p,
                               C.c_void_p]),
    "ixb_mtx_read": (C.c_int, [C.c_char_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                               C.c_void_p, C.c_void_p]),
    "ixb_mtx_to_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                    C.c_void_p]),
    "ixb_mtx_to_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ixb_mtx_free": (None, [C.c_void_p]),
    "ixb_rng_new": (C.c_void_p, [C.c_uint64]),
    "ixb_rng_free": (None, [C.c_void_p]),
    "ixb_rng_next": (C.c_uint64, [C.c_void_p]),
    "ixb_synth_dense": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_int, C.c_void_p]),
    "ixb_synth_sparse_matrix": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_double,
                                          C.c_int, C.c_void_p]),
    "ixb_synth_block_sparse_matrix": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_int64,
                                                C.c_int64, C.c_int64, C.c_double, C.c_int,
                                                C.c_void_p]),
    "ixb_synth_coo_tensor": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int64,
                                       C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ixb_synth_voxel_shells": (C.c_int, [C.c_int64, C.c_void_p, C.c_void_p]),
    "ixb_cg_table": (C.c_int, [C.c_int] + [C.c_void_p] * 7),
    "ixb_comm_unique_id": (C.c_int, [C.c_void_p]),
    "ixb_comm_init": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "ixb_comm_free": (None, [C.c_void_p]),
    "ixb_comm_broadcast": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_void_p]),
    "ixb_shard_plan_create": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_int,
                                        C.c_int, C.c_void_p, C.c_void_p]),
    "ixb_shard_plan_chunk": (C.c_int, [C.c_void_p, C.c_int, C.c_int] + [C.c_void_p] * 4),
    "ixb_shard_plan_free": (None, [C.c_void_p]),
    "ixb_spmm_groupcoo_sharded": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                            C.c_void_p, C.c_int64, C.c_int64, C.c_void_p,
                                            C.c_int, C.c_void_p, C.c_void_p]),
    "ixb_spmm_blockgroupcoo_sharded": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                                 C.c_int64, C.c_int64, C.c_void_p, C.c_int64,
                                                 C.c_int64, C.c_void_p, C.c_int, C.c_void_p,
                                                 C.c_void_p]),
    "ixb_conv_plan_run_sharded": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                            C.c_int64, C.c_void_p, C.c_int64, C.c_int, C.c_int,
                                            C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
}

EXPORTED = tuple(_SIGS)


def lib():
    """Loads libixb.so (raises if it was never built — no fallback)."""
    global _lib
    if _lib is None:
        path = lib_path()
        if not os.path.exists(path):
            raise IxbError(1, f"libixb.so not built at {path}; run __graft_entry__.build()")
        L = C.CDLL(path)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(code):
    if code != 0:
        msg = lib().ixb_last_error().decode()
        raise _BY_CODE.get(code, IxbError)(code, msg)
