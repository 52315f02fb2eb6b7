"""ixsum-b200 — B200-native executor for Insum's indirect Einsums.

Python mirror of the reference's hot-path API (/root/reference/proj/include/
ixsum/{formats,plan,driver}.hpp) over the C-ABI in include/ixb.h
(libixb.so, hand-written sm_100a kernels). torch is used only for device
memory and streams. There is no CPU fallback: if libixb.so is missing, or
no CUDA device is present, every call raises.

Names and argument meaning follow the reference:
  dense_to_coo, coo_to_groupcoo, dense_to_blockgroupcoo, group_coo_tensor,
  emit_operands, execute_mode("b200", ...)
Errors raise the reference's exception classes (ParseError, BindError,
ShapeError, IndexRangeError, IoError) with the reference's message content.
On-disk formats (.ixt, MatrixMarket, convert directories) load straight to
the device: see `io`.
"""
from .abi import (BindError, IxbError, IndexRangeError, IoError, ParseError, ShapeError, lib,
                  lib_path)
from .api import (BlockGroupCoo, GroupCoo, GroupCooTensor, dense_to_blockgroupcoo,
                  dense_to_coo, dense_to_groupcoo, coo_to_groupcoo, emit_operands,
                  group_coo_tensor, kernel_map, tune_group_size, spmm_groupcoo,
                  spmm_blockgroupcoo, conv_grouped, tp_grouped, shard_groups, ConvPlan, TpPlan,
                  spmm_groupcoo_host, spmm_blockgroupcoo_host,
                  count_accesses_model, real_count, pad_count, is_ell, ell_view,
                  groupcoo_to_coo)
from .executor import device_tolerance, execute_mode, match_workload, WORKLOADS
from . import io
from .io import (ixt_info, load_ixt, save_ixt, load_matrix_market, read_matrix_market_host,
                 save_format, load_format, convert, tune_report, tune_measured)

__all__ = [
    "lib", "lib_path", "IxbError", "ParseError", "BindError", "ShapeError", "IndexRangeError",
    "IoError",
    "GroupCoo", "BlockGroupCoo", "GroupCooTensor", "dense_to_coo", "coo_to_groupcoo",
    "dense_to_groupcoo", "dense_to_blockgroupcoo", "group_coo_tensor", "emit_operands",
    "kernel_map", "tune_group_size", "spmm_groupcoo", "spmm_blockgroupcoo", "conv_grouped",
    "tp_grouped", "shard_groups", "ConvPlan", "TpPlan", "spmm_groupcoo_host",
    "spmm_blockgroupcoo_host", "count_accesses_model", "real_count", "pad_count", "is_ell",
    "ell_view", "groupcoo_to_coo", "device_tolerance", "execute_mode", "match_workload",
    "WORKLOADS", "io", "ixt_info", "load_ixt", "save_ixt", "load_matrix_market",
    "read_matrix_market_host", "save_format", "load_format", "convert", "tune_report", "tune_measured",
]
