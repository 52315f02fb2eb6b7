/*
 * ixb.h — C-ABI of the B200-native executor for Insum's indirect Einsums.
 *
 * Drop-in boundary for the hot path of the reference toolkit `ixsum`
 * (/root/reference/proj/include/ixsum): the format builders and the four
 * indirect-Einsum evaluators. Plain pointers and sizes only — no C++ or torch
 * types. All device pointers are CUDA device memory on the current device;
 * every call is stream-ordered on `stream` (NULL = legacy default stream).
 *
 * Index arrays are int32 on the device (the reference stores int64,
 * formats.hpp:43-45); values are fp32 or bf16 with fp32 accumulation (the
 * reference is fp64/int64, tensor.hpp:11). See DESIGN.md for layouts.
 *
 * Return codes map 1:1 onto the reference's exception classes and CLI exit
 * codes (driver.hpp:19-27, report_error driver.cpp:571-580):
 *   IXB_OK 0, IXB_FAILURE 1 (std::runtime_error / std::invalid_argument),
 *   IXB_PARSE 2 (ParseError), IXB_BIND 3 (BindError), IXB_SHAPE 4
 *   (ShapeError / InferenceError), IXB_INDEX_RANGE 6 (IndexRangeError),
 *   IXB_CUDA 7 (device failure — no reference equivalent), IXB_IO 8 (IoError;
 *   the reference CLI reports it with exit code 1).
 * The message of the last failure on the calling thread is ixb_last_error().
 */
#ifndef IXB_H
#define IXB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* ixb_stream; /* == cudaStream_t */

enum ixb_status {
  IXB_OK = 0,
  IXB_FAILURE = 1,
  IXB_PARSE = 2,
  IXB_BIND = 3,
  IXB_SHAPE = 4,
  IXB_INDEX_RANGE = 6,
  IXB_CUDA = 7,
  IXB_IO = 8
};

/* Device element types. Evaluators take IXB_F32 / IXB_BF16 values; the
 * sorted-run builders (ixb_groupcoo_pack, ixb_group_coo_tensor_pack) also
 * carry 8-byte values (IXB_F64 / IXB_I64) unchanged, and the file I/O
 * below converts between the files' real64/int64 and any of these. */
enum ixb_dtype { IXB_F32 = 0, IXB_BF16 = 1, IXB_F64 = 2, IXB_I32 = 3, IXB_I64 = 4, IXB_U8 = 5 };

/* Evaluator flags. */
enum ixb_flags {
  /* Evaluator returns without synchronising; index-range errors found by the
   * kernel are reported by the next ixb_check_errors() call. */
  IXB_ASYNC = 1,
  /* Caller asserts the group-coordinate array (AM / MAPX-groups / CGL ...)
   * is non-decreasing, as every ixb builder produces it. Without the flag
   * the evaluator verifies it (one extra pass + sync) and falls back to a
   * stable permutation when it is not sorted. */
  IXB_GROUPS_SORTED = 2,
  /* Skip the in-kernel index range checks (inputs already validated). */
  IXB_UNCHECKED = 4,
  /* Sharded evaluation only (instrumentation): evaluate this rank's chunks
   * without the output all-gather, or run only the all-gather. */
  IXB_SHARD_NO_COMM = 8,
  IXB_SHARD_COMM_ONLY = 16
};

const char* ixb_last_error(void);
int ixb_version(void);
/* Details of the last IXB_INDEX_RANGE failure on this thread: which operand
 * (evaluator-specific order, gathers before scatters), flat position, value
 * and the extent it violated. */
int ixb_last_index_error(int* operand, int64_t* position, int64_t* value, int64_t* extent);
/* Reports (and clears) index-range errors recorded by IXB_ASYNC calls on this
 * device; synchronises `stream`. */
int ixb_check_errors(ixb_stream stream);
/* Number of SMs of the current device (148 on B200). */
int ixb_sm_count(void);
/* Number of ixb kernels launched by this process (for launch accounting). */
int64_t ixb_launch_count(void);

/* ======================================================================
 * Builders (K1/K2 + rank-n grouping). Two phases: *_plan computes sizes
 * (one device->host sync) and keeps device temporaries in the opaque
 * ixb_pack; *_pack writes caller-allocated outputs and may be called with
 * several value arrays; ixb_pack_free releases it.
 * Outputs reproduce the reference bit-for-bit (after int32->int64 widening).
 * ==================================================================== */
typedef struct ixb_pack ixb_pack;
void ixb_pack_free(ixb_pack* plan);

/* dense_to_coo (formats.hpp:26, formats.cpp:24-46): row-major scan of a
 * dense [rows, cols] matrix, entries != 0 kept. */
int ixb_dense_to_coo_plan(const void* dense, int dtype, int64_t rows, int64_t cols,
                          ixb_stream stream, ixb_pack** plan, int64_t* nnz);
int ixb_dense_to_coo_pack(ixb_pack* plan, int32_t* row_coord, int32_t* col_coord, void* values,
                          ixb_stream stream);

/* coo_to_groupcoo (formats.hpp:53, formats.cpp:115-174): stable sort by
 * (group coordinate, member coordinate), runs split into ceil(occ/g) groups,
 * tail padded with the last real member and value 0. `canonical` != 0 asserts
 * the input is already sorted by (row, col) (CooMatrix::canonical).
 * g == 0 selects g with the reference tuner (tuner.cpp:100-118; the
 * `format: auto` path of driver.cpp:106-113); *g_out returns the g used. */
int ixb_groupcoo_plan(const int32_t* row_coord, const int32_t* col_coord, int64_t nnz,
                      int64_t rows, int64_t cols, int canonical, int group_dim, int64_t g,
                      ixb_stream stream, ixb_pack** plan, int64_t* num_groups, int64_t* g_out);
/* AV: [G, g] of `dtype`; mask: [G, g] u8 (1 = real) or NULL. `values` may be
 * NULL when only the index arrays are wanted. */
int ixb_groupcoo_pack(ixb_pack* plan, const void* values, int dtype, int32_t* AM, int32_t* AK,
                      void* AV, uint8_t* mask, ixb_stream stream);

/* dense_to_coo + coo_to_groupcoo fused for a dense [rows, cols] source
 * (group_dim 0 or 1; g == 0 -> tuner). */
int ixb_dense_groupcoo_plan(const void* dense, int dtype, int64_t rows, int64_t cols,
                            int group_dim, int64_t g, ixb_stream stream, ixb_pack** plan,
                            int64_t* num_groups, int64_t* g_out, int64_t* nnz);
int ixb_dense_groupcoo_pack(ixb_pack* plan, int32_t* AM, int32_t* AK, void* AV, uint8_t* mask,
                            ixb_stream stream);

/* dense_to_blockgroupcoo (formats.hpp:81-83, formats.cpp:224-292): a bM x bK
 * block is stored iff any element != 0 (in the device dtype); block COO is
 * grouped like coo_to_groupcoo; ragged edges and pad slots are zero.
 * g == 0 -> tuner on block occupancy. AV: [G, g, bM, bK] of `dtype`. */
int ixb_blockgroupcoo_plan(const void* dense, int dtype, int64_t rows, int64_t cols, int64_t bm,
                           int64_t bk, int64_t g, int group_dim, ixb_stream stream,
                           ixb_pack** plan, int64_t* num_groups, int64_t* g_out,
                           int64_t* num_blocks);
int ixb_blockgroupcoo_pack(ixb_pack* plan, int32_t* AM, int32_t* AK, void* AV, uint8_t* mask,
                           ixb_stream stream);

/* group_coo_tensor (formats.hpp:141, formats.cpp:417-479): rank-n COO
 * (coords: `rank` device arrays of nnz int32) grouped along group_dim; sort
 * key (group coord, then the other dims in order), stable. `canonical` != 0
 * asserts the input is already in that order (e.g. ixb_kernel_map output). */
int ixb_group_coo_tensor_plan(int rank, const int64_t* shape, const int32_t* const* coords,
                              int64_t nnz, int group_dim, int64_t g, int canonical,
                              ixb_stream stream, ixb_pack** plan, int64_t* num_groups);
/* member_coords: rank-1 device arrays [G, g] (dims in order, group_dim skipped). */
int ixb_group_coo_tensor_pack(ixb_pack* plan, const void* values, int dtype,
                              int32_t* group_coord, int32_t* const* member_coords, void* out_values,
                              uint8_t* mask, ixb_stream stream);

/* Reference tuner over a device occupancy source (tuner.cpp:31-118):
 * coord: nnz int32 coordinates in [0, extent). */
/* select's full TuneReport (tuner.hpp:43-63): g*, the power-of-two
 * candidates (at most 2) and their cost_exact scores, and the chosen g —
 * what the convert manifest's "tuner" block records (driver.cpp:460-470). */
int ixb_tune_report(const int32_t* coord, int64_t nnz, int64_t extent, int count_empty_rows,
                    ixb_stream stream, int64_t* g, double* gstar, int64_t* cand_g,
                    double* cand_score, int* ncand);
/* brute_force_optimal (tuner.cpp:86-97), the TuneReport's brute_optimal:
 * argmin over g in [1, max occ] of cost_exact (ties -> smaller g). *g = 0 for an
 * empty profile (the reference's nullopt). */
int ixb_tune_brute(const int32_t* coord, int64_t nnz, int64_t extent, ixb_stream stream,
                   int64_t* g, int64_t* cost);
int ixb_tune_group_size(const int32_t* coord, int64_t nnz, int64_t extent, int count_empty_rows,
                        ixb_stream stream, int64_t* g_out, double* gstar_out);

/* GroupCOO helpers (formats.hpp:49-58), device arrays in, host scalars out:
 * real_count of a pad mask (pad_count = slots - real; formats.cpp:105-113),
 * is_ell — no two consecutive groups share a coordinate (formats.cpp:202-208),
 * the occupancy maximum ell_view groups by (g = max(max_occ, 1),
 * formats.cpp:196-200), and groupcoo_to_coo (formats.cpp:176-194): the
 * real slots in slot order into caller buffers of real_count entries
 * (values of `dtype`, or NULL); the reference then canonicalizes, which the
 * g = 1 grouping does (ixb_groupcoo_plan/pack with g = 1). */
int ixb_mask_real_count(const uint8_t* mask, int64_t slots, ixb_stream stream, int64_t* real);
int ixb_is_ell(const int32_t* group_coord, int64_t G, ixb_stream stream, int* is_ell);
int ixb_max_occupancy(const int32_t* coord, int64_t nnz, int64_t extent, ixb_stream stream,
                      int64_t* max_occ);
int ixb_groupcoo_to_coo(const int32_t* group_coord, const int32_t* member_coord,
                        const void* values, int dtype, const uint8_t* mask, int64_t G, int64_t g,
                        int group_dim, int32_t* row_out, int32_t* col_out, void* val_out,
                        ixb_stream stream);

/* ======================================================================
 * Evaluators. Each validates indices in-kernel (unless IXB_UNCHECKED);
 * `accumulate` != 0 is `+=` (the output's contents prime the sum),
 * accumulate == 0 is `=` (plan.cpp:540). Results are run-to-run
 * deterministic: no floating-point atomics; each output row has one owner
 * that sums its groups in group order.
 * ==================================================================== */

/* K3 — GroupCOO SpMM, `C[AM[p],n] += AV[p,q] * B[AK[p,q],n]`
 * (corpus/unstructured_spmm.json:2). AV [G,g], B [K,N], C [M,N], fp32.
 * g == 1 is the COO SpMM `C[AM[p],n] += AV[p] * B[AK[p],n]`.
 * Operands for ixb_last_index_error: 0 = AK, 1 = AM. */
int ixb_spmm_groupcoo(const int32_t* AM, const int32_t* AK, const float* AV, int64_t G, int64_t g,
                      const float* B, int64_t K, int64_t N, float* C, int64_t M, int accumulate,
                      int flags, ixb_stream stream);

/* K4 — BlockGroupCOO SpMM on tcgen05/TMEM,
 * `C[AM[p],bm,n] += AV[p,q,bm,bk] * B[AK[p,q],bk,n]` (corpus/structured_spmm.json:2).
 * AV [G,g,16,16] bf16, B [KB,16,N] bf16, C [MB,16,N] fp32. bm = bk = 16,
 * N % 128 == 0. Operands: 0 = AK, 1 = AM. */
int ixb_spmm_blockgroupcoo(const int32_t* AM, const int32_t* AK, const void* AV, int64_t G,
                           int64_t g, int64_t bm, int64_t bk, const void* B, int64_t KB,
                           int64_t N, float* C, int64_t MB, int accumulate, int flags,
                           ixb_stream stream);

/* K5 — submanifold 3x3x3 kernel map over n voxels (coords [n,3] int32,
 * unique). Pairs (out i, in j, offset z) with coord[j] == coord[i] + delta(z),
 * z = (dx+1)*9 + (dy+1)*3 + (dz+1), ordered by (z, i) — the canonical order
 * of group_coo_tensor(map, 2, g) input. The plan counts the pairs (one
 * device->host read); pack writes them and reads `coords` again, so coords
 * must stay valid until pack. */
typedef struct ixb_kmap ixb_kmap;
int ixb_kernel_map_plan(const int32_t* coords, int64_t n, ixb_stream stream, ixb_kmap** plan,
                        int64_t* num_pairs);
int ixb_kernel_map_pack(ixb_kmap* plan, int32_t* map_out, int32_t* map_in, int32_t* map_off,
                        ixb_stream stream);
void ixb_kernel_map_free(ixb_kmap* plan);

/* K6 — grouped sparse convolution,
 * `Out[MAPX[p,q],m] += MAPV[p,q] * In[MAPY[p,q],c] * Weight[MAPZ[p],c,m]`
 * (corpus/grouped_sparse_conv.json:2). In [n_in, Cin] bf16, Weight
 * [n_off, Cin, Cout] bf16, MAPV [G,g] fp32 (NULL = all ones), Out
 * [n_out, Cout] fp32. Operands: 0 = MAPY, 1 = MAPZ, 2 = MAPX. */
int ixb_conv_grouped(const int32_t* MAPZ, const int32_t* MAPX, const int32_t* MAPY,
                     const float* MAPV, int64_t G, int64_t g, const void* In, int64_t n_in,
                     int64_t Cin, const void* Weight, int64_t n_off, int64_t Cout, float* Out,
                     int64_t n_out, int accumulate, int flags, ixb_stream stream);
/* Inspector/executor split of K6 for a map reused across calls (one conv
 * layer stack over one point cloud): the plan validates the map and builds
 * its (output, offset) index once; run evaluates In/Weight -> Out. */
typedef struct ixb_conv_plan ixb_conv_plan;
int ixb_conv_plan_create(const int32_t* MAPZ, const int32_t* MAPX, const int32_t* MAPY,
                         const float* MAPV, int64_t G, int64_t g, int64_t n_in, int64_t n_off,
                         int64_t n_out, int flags, ixb_stream stream, ixb_conv_plan** plan);
int ixb_conv_plan_run(ixb_conv_plan* plan, const void* In, int64_t Cin, const void* Weight,
                      int64_t Cout, float* Out, int accumulate, int flags, ixb_stream stream);
/* Host-buffer form of ixb_conv_plan_run: In [n_in, Cin] bf16 and Out
 * [n_out, Cout] fp32 are HOST arrays (pinned for overlap), Weight a device
 * array. Builder-made (unit) maps run in `nchunks` groups of output tiles:
 * In streams in row order and each group starts once the input rows it reads
 * have landed, while earlier groups' Out rows copy back. Returns with Out
 * written, bit-identical to the device-buffer call. */
int ixb_conv_plan_run_host(ixb_conv_plan* plan, const void* In, int64_t Cin, const void* Weight,
                           int64_t Cout, float* Out, int accumulate, int flags, int nchunks,
                           ixb_stream stream);
void ixb_conv_plan_free(ixb_conv_plan* plan);

/* K7 — grouped Clebsch–Gordan tensor product,
 * `Z[b,CGI[p,q],w] += CGV[p,q] * X[b,CGJ[p,q],u] * Y[b,CGK[p,q]] * W[CGL[p],u,w]`
 * (corpus/grouped_tensor_product.json:2 with `w_per_batch` = 1; the
 * shared-weight form `W[CGL[p],u,w]` with w_per_batch = 0). X [B,nj,U] bf16,
 * Y [B,nk] bf16, W [(B,)nl,U,Wd] bf16, CGV [G,g] fp32, Z [B,ni,Wd] fp32.
 * Operands: 0 = CGJ, 1 = CGK, 2 = CGL, 3 = CGI. */
int ixb_tp_grouped(const int32_t* CGL, const int32_t* CGI, const int32_t* CGJ, const int32_t* CGK,
                   const float* CGV, int64_t G, int64_t g, const void* X, const void* Y,
                   const void* W, int w_per_batch, int64_t batch, int64_t ni, int64_t nj,
                   int64_t nk, int64_t nl, int64_t U, int64_t Wd, float* Z, int accumulate,
                   int flags, ixb_stream stream);
/* Inspector/executor split of K7 for a CG table reused across calls (every
 * layer of an equivariant network applies the same table): the plan
 * validates the table (same errors as ixb_tp_grouped) and reshapes it once;
 * run evaluates X/Y/W -> Z for any batch. The CG arrays must outlive the
 * plan. ixb_tp_grouped == create + run + free. */
typedef struct ixb_tp_plan ixb_tp_plan;
int ixb_tp_plan_create(const int32_t* CGL, const int32_t* CGI, const int32_t* CGJ,
                       const int32_t* CGK, const float* CGV, int64_t G, int64_t g, int w_per_batch,
                       int64_t ni, int64_t nj, int64_t nk, int64_t nl, int64_t U, int64_t Wd,
                       int flags, ixb_stream stream, ixb_tp_plan** plan);
int ixb_tp_plan_run(ixb_tp_plan* plan, const void* X, const void* Y, const void* W, int64_t batch,
                    float* Z, int accumulate, int flags, ixb_stream stream);
void ixb_tp_plan_free(ixb_tp_plan* plan);
/* 1 if the plan runs on the tensor-core (V-first) kernel, 0 if its shape or
 * table size sends it to the CUDA-core kernel. */
int ixb_tp_plan_uses_tensor_cores(const ixb_tp_plan* plan);
/* Host-buffer form of ixb_tp_plan_run: X [batch, nj, U] bf16, Y [batch, nk]
 * bf16 and Z [batch, ni, Wd] fp32 are HOST arrays (pinned for overlap), W a
 * device array. The batch is cut into `nchunks` runs of whole 64-edge tiles
 * whose copy-in, evaluation and copy-out overlap on three streams; returns
 * with Z written, bit-identical to the device-buffer call. */
int ixb_tp_plan_run_host(ixb_tp_plan* plan, const void* X, const void* Y, const void* W,
                         int64_t batch, float* Z, int accumulate, int flags, int nchunks,
                         ixb_stream stream);

/* Host-buffer forms of the SpMM evaluators (the shape of the reference's
 * execute_mode: host Tensors in, host result out). All arrays are HOST
 * memory (pinned for full overlap); the call returns with C written. The
 * groups are cut into `nchunks` ranges at output-row boundaries: B is copied
 * first, then chunk i's format H2D, its kernel and its C rows D2H run on
 * three streams, so transfers overlap each other and the kernels (the small
 * index arrays go whole, right after B, when small next to the values).
 * nchunks <= 0 picks 2 chunks for GroupCOO and one per ~2 MB of values in +
 * C rows out (2..8) for BlockGroupCOO. Results and errors are bit-identical
 * to the device-buffer calls. */
int ixb_spmm_blockgroupcoo_host(const int32_t* AM, const int32_t* AK, const void* AV, int64_t G,
                                int64_t g, int64_t bm, int64_t bk, const void* B, int64_t KB,
                                int64_t N, float* C, int64_t MB, int accumulate, int flags,
                                int nchunks, ixb_stream stream);
int ixb_spmm_groupcoo_host(const int32_t* AM, const int32_t* AK, const float* AV, int64_t G,
                           int64_t g, const float* B, int64_t K, int64_t N, float* C, int64_t M,
                           int accumulate, int flags, int nchunks, ixb_stream stream);

/* ======================================================================
 * On-disk formats straight to/from the device.
 * ==================================================================== */
/* .ixt tensor files (tensor.hpp:65-73, tensor.cpp:158-225,
 * docs/file-formats.md): header query; load into a device buffer of
 * `dtype` (int64 files -> IXB_I32 are range-checked; real64 -> int dtypes
 * refused); save a device array (float dtypes as real64, integer dtypes as
 * int64), bitwise-compatible with the reference's save_tensor. Errors and
 * messages follow load_tensor / save_tensor (IXB_IO). */
int ixb_ixt_info(const char* path, int* kind, int* rank, int64_t* dims16);
int ixb_ixt_load(const char* path, void* dst, int dtype, ixb_stream stream);
int ixb_ixt_save(const char* path, const void* src, int dtype, int rank, const int64_t* dims,
                 ixb_stream stream);

/* MatrixMarket (matrix_market.hpp:16, matrix_market.cpp:30-159): parsed on
 * the host with the reference's rules and messages (one-based -> zero-based,
 * duplicates kept, symmetric/skew-symmetric expanded, array files dense
 * column-major -> row-major); then copied to the device as COO (int32
 * coordinates + values of `dtype`) or as a dense [rows, cols] array.
 * kind: 0 real64, 1 int64 (integer field). nnz = entries after expansion
 * (rows*cols for array files). ixb_mtx_to_host copies the 8-byte host form
 * (rows/cols int64, values double or int64 by kind). */
typedef struct ixb_mtx ixb_mtx;
int ixb_mtx_read(const char* path, ixb_mtx** mtx, int* is_dense, int* kind, int64_t* rows,
                 int64_t* cols, int64_t* nnz);
int ixb_mtx_to_device(const ixb_mtx* mtx, int32_t* row, int32_t* col, void* values, int dtype,
                      ixb_stream stream);
int ixb_mtx_to_host(const ixb_mtx* mtx, int64_t* row, int64_t* col, void* values);
void ixb_mtx_free(ixb_mtx* mtx);

/* ======================================================================
 * Multi-GPU sharding (host-side planning). Cuts G sorted
 * groups into `parts` contiguous ranges of ~equal slot count, cutting only
 * where the group coordinate changes, so no output row spans two ranks and
 * per-row summation order (hence every bit of the result) is independent
 * of `parts`. group_coord is a HOST array here. bounds: parts+1 entries.
 * ==================================================================== */
int ixb_shard_groups(const int32_t* group_coord_host, int64_t G, int parts, int64_t* bounds);

/* Sharded evaluation across the GPUs of one node, one process per GPU
 * (north_star: "shard across one 8xB200 box by row-group / point-block
 * partition with a replicated dense operand; NCCL over NVLink only for the
 * final output all-gather"). The reference's single-process evaluators
 * (execute_plan plan.hpp:82, interpret_kernel kernel.hpp:184) have no
 * multi-process form; these entries are what a multi-GPU `execute_mode`
 * would call on each rank.
 *
 * Communicator: NCCL (libnccl.so.2, loaded at first use). Rank 0 creates a
 * 128-byte id, the caller distributes it (any side channel), every rank
 * calls ixb_comm_init (world == 1 builds a 1-rank communicator; a null
 * comm with world == 1 evaluates without any collective). */
typedef struct ixb_comm ixb_comm;
int ixb_comm_unique_id(void* id128);
int ixb_comm_init(const void* id128, int world, int rank, ixb_comm** comm);
void ixb_comm_free(ixb_comm* comm);
/* In-place broadcast of `bytes` of a device buffer from `root` (the
 * one-time replication of the format and dense operand). */
int ixb_comm_broadcast(ixb_comm* comm, void* buf, int64_t bytes, int root, ixb_stream stream);

/* Shard plan over a sorted group-coordinate array (DEVICE, the replicated
 * format's AM): every rank's row-aligned group range (ixb_shard_groups),
 * each cut into `nchunks` row-aligned chunks. One device->host copy. */
typedef struct ixb_shard_plan ixb_shard_plan;
int ixb_shard_plan_create(const int32_t* group_coord, int64_t G, int64_t rows, int world,
                          int rank, int nchunks, ixb_stream stream, ixb_shard_plan** plan);
int ixb_shard_plan_chunk(const ixb_shard_plan* plan, int rank, int chunk, int64_t* g0,
                         int64_t* g1, int64_t* r0, int64_t* r1);
void ixb_shard_plan_free(ixb_shard_plan* plan);

/* `=` evaluation of the plan's rank into its rows of the FULL output C
 * (GroupCOO C[M,N] fp32; BlockGroupCOO C[MB,16,N] fp32), then every rank's
 * rows are broadcast in place so that, stream-ordered on return, every rank
 * holds the whole C. Chunk c's broadcasts (one NCCL group, side stream)
 * overlap chunk c+1's kernel. AK/AV/B are the full replicated operands. */
int ixb_spmm_groupcoo_sharded(const ixb_shard_plan* plan, const int32_t* AK, const float* AV,
                              int64_t g, const float* B, int64_t K, int64_t N, float* C,
                              int flags, ixb_comm* comm, ixb_stream stream);
int ixb_spmm_blockgroupcoo_sharded(const ixb_shard_plan* plan, const int32_t* AK, const void* AV,
                                   int64_t g, int64_t bm, int64_t bk, const void* B, int64_t KB,
                                   int64_t N, float* C, int flags, ixb_comm* comm,
                                   ixb_stream stream);
/* Point-block conv: `local` is this rank's plan over output voxels
 * [n_total*rank/world, n_total*(rank+1)/world) (the kernel map filtered to
 * that block, output index re-based; In replicated). Evaluates the block in
 * `nchunks` tile-aligned chunks into its rows of the FULL Out [n_total,
 * Cout] and all-gathers Out as above. */
int ixb_conv_plan_run_sharded(ixb_conv_plan* local, const void* In, int64_t Cin,
                              const void* Weight, int64_t Cout, float* Out, int64_t n_total,
                              int world, int rank, int nchunks, int flags, ixb_comm* comm,
                              ixb_stream stream);

/* ======================================================================
 * Seeded synthetic inputs, host side (synth.hpp:13-29): std::mt19937_64 and
 * libstdc++'s distributions consumed exactly like synth.cpp:10-106, so one
 * seed reproduces the reference's operands. `kind` 0 = real (+-U[0.125,1]),
 * 1 = int (+-{1..4}); `out` 0 = f32, 1 = bf16, 2 = f64, 3 = i64 (host arrays).
 * ==================================================================== */
typedef struct ixb_rng ixb_rng;
ixb_rng* ixb_rng_new(uint64_t seed);
void ixb_rng_free(ixb_rng* rng);
uint64_t ixb_rng_next(ixb_rng* rng);
int ixb_synth_dense(ixb_rng* rng, int kind, int64_t numel, int out, void* dst);
int ixb_synth_sparse_matrix(ixb_rng* rng, int kind, int64_t rows, int64_t cols, double density,
                            int out, void* dst);
int ixb_synth_block_sparse_matrix(ixb_rng* rng, int kind, int64_t rows, int64_t cols, int64_t br,
                                  int64_t bc, double block_density, int out, void* dst);
/* Real-basis Clebsch–Gordan table for l_max (cfg4's CG operand; host
 * arrays, NULL to count): entries (i, j, k, path, value) in (path, i, j, k)
 * generation order; paths (l1,l2,l3) with the triangle rule and even
 * l1+l2+l3 (23 paths / 353 entries for l_max = 3). */
int ixb_cg_table(int l_max, int32_t* ci, int32_t* cj, int32_t* ck, int32_t* cl, float* cv,
                 int64_t* count, int32_t* npaths);
/* cfg5 point cloud: voxelised sphere shells (R = 282) in (x,y,z) order,
 * n_target voxels, coords [n, 3] int32 (NULL to count). */
int ixb_synth_voxel_shells(int64_t n_target, int32_t* coords, int64_t* n_out);
/* coords: [rank, nnz] int32 (capacity >= min(nnz, prod(shape))); *nnz_out = realised nnz. */
int ixb_synth_coo_tensor(ixb_rng* rng, int kind, int rank, const int64_t* shape, int64_t nnz,
                         int out, int32_t* coords, void* values, int64_t* nnz_out);

#ifdef __cplusplus
}
#endif
#endif /* IXB_H */
