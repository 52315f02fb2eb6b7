/*
 * ixo — CPU ORACLE (test infrastructure only; never linked into the product).
 *
 * Plain-C restatement of the reference algorithms on the hot path of
 * arxiv/paper_2510_17505 (the `ixsum` toolkit under /root/reference/proj):
 *   - the seeded synthetic inputs (synth.cpp:10-106) bit-for-bit, including
 *     libstdc++'s mt19937_64 / uniform_int / bernoulli / uniform_real streams;
 *   - the format builders dense_to_coo (formats.cpp:24-46), coo_to_groupcoo
 *     (:115-174), dense_to_blockgroupcoo (:224-292), group_coo_tensor (:417-479);
 *   - the group-size tuner (tuner.cpp:31-118);
 *   - the brute-force evaluator oracle_einsum (plan.cpp:579-605) over the
 *     expression grammar (expr.cpp:36-181), with the same range checks and
 *     messages (plan.cpp:249-259);
 *   - max_rel_error / tensor_hash (tensor.cpp:124-156);
 *   - new, reference-absent KATs: the submanifold voxel kernel map and the
 *     real-basis Clebsch–Gordan table (SURVEY.md §8c "not pinned").
 *
 * PARITY PINNING: tests/test_oracle_vs_ref.py checks every function here
 * against the unmodified reference compiled in place (oracle/_ref), and
 * tests/test_oracle_kat.py against the reference unit tests' known answers.
 * Kernel map and CG have no reference implementation: they are pinned by
 * brute-force and sympy cross-checks instead.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library.
 */
#ifndef IXO_H
#define IXO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { IXO_REAL = 0, IXO_INT = 1 };
/* Status codes mirror report_error (driver.cpp:571-580). */
enum {
  IXO_OK = 0, IXO_FAILURE = 1, IXO_PARSE = 2, IXO_BIND = 3, IXO_SHAPE = 4, IXO_INDEX_RANGE = 6
};

/* ---- std::mt19937_64 + libstdc++ distributions ---- */
typedef struct ixo_rng ixo_rng;
ixo_rng* ixo_rng_new(uint64_t seed);
void ixo_rng_free(ixo_rng* r);
uint64_t ixo_rng_next(ixo_rng* r);
int64_t ixo_uniform_int(ixo_rng* r, int64_t a, int64_t b);
double ixo_canonical(ixo_rng* r);
int ixo_bernoulli(ixo_rng* r, double p);
double ixo_uniform_real(ixo_rng* r, double a, double b);

/* ---- synth.hpp:17-29 (out buffers are caller-allocated) ---- */
void ixo_synth_dense(ixo_rng* r, int kind, int64_t numel, void* out);
void ixo_synth_sparse_matrix(ixo_rng* r, int kind, int64_t rows, int64_t cols, double density,
                             void* out);
void ixo_synth_block_sparse_matrix(ixo_rng* r, int kind, int64_t rows, int64_t cols,
                                   int64_t br, int64_t bc, double bdens, void* out);
/* coords_out: [rank, nnz_cap]; returns the realised nnz = min(nnz, capacity). */
int64_t ixo_synth_coo_tensor(ixo_rng* r, int kind, int rank, const int64_t* shape, int64_t nnz,
                             int64_t* coords_out, void* vals_out);

/* ---- builders ---- */
int64_t ixo_count_nonzero(int kind, int64_t n, const void* data);
/* dense_to_coo: row-major scan; arrays sized by ixo_count_nonzero. */
void ixo_dense_to_coo(int kind, int64_t rows, int64_t cols, const void* data, int64_t* row_coord,
                      int64_t* col_coord, void* values);
/* coo_to_groupcoo. Call with AM==NULL to get G only. */
int ixo_coo_to_groupcoo(int64_t rows, int64_t cols, const int64_t* r, const int64_t* c, int kind,
                        const void* vals, int64_t nnz, int group_dim, int64_t g, int64_t* G_out,
                        int64_t* AM, int64_t* AK, void* AV, uint8_t* mask);
/* dense_to_blockgroupcoo. Call with AM==NULL to get G only. AV: [G,g,bm,bk]. */
int ixo_dense_to_blockgroupcoo(int kind, int64_t rows, int64_t cols, const void* data, int64_t bm,
                               int64_t bk, int64_t g, int group_dim, int64_t* G_out, int64_t* AM,
                               int64_t* AK, void* AV, uint8_t* mask);
/* group_coo_tensor. coords: [rank, nnz]; member_coords: [rank-1, G, g]. */
int ixo_group_coo_tensor(int rank, const int64_t* shape, const int64_t* coords, int kind,
                         const void* vals, int64_t nnz, int group_dim, int64_t g, int64_t* G_out,
                         int64_t* group_coord, int64_t* member_coords, void* values,
                         uint8_t* mask);

/* ---- tuner ---- */
int64_t ixo_cost_exact(const int64_t* occ, int64_t n, int64_t g);
double ixo_cost_relaxed(const int64_t* occ, int64_t n, double g, int count_empty_rows);
double ixo_g_star(const int64_t* occ, int64_t n, int count_empty_rows);
/* returns number of candidates (1 or 2) written to cand[]. */
int ixo_candidate_group_sizes(const int64_t* occ, int64_t n, int count_empty_rows, int64_t* cand);
int64_t ixo_select(const int64_t* occ, int64_t n, int count_empty_rows);
/* brute force argmin F(g) over [1, max occ]; returns g (0 for empty), *f_out = F(g). */
int64_t ixo_brute_force_optimal(const int64_t* occ, int64_t n, int64_t* f_out);

/* ---- oracle_einsum ---- */
typedef struct {
  const char* name;
  int kind;
  int rank;
  const int64_t* shape;
  const void* data;
} ixo_tensor;

/* Evaluates `expr` over `tensors`; `out` holds the output buffer: its
 * contents prime `+=` and receive the result. err receives the reference's
 * message on failure. */
int ixo_einsum(const char* expr, const ixo_tensor* tensors, int ntensors, const char* out_name,
               int out_kind, int out_rank, const int64_t* out_shape, void* out, char* err,
               int errlen);

double ixo_max_rel_error(int kind, int64_t n, const void* a, const void* b);
uint64_t ixo_tensor_hash(int kind, int rank, const int64_t* shape, const void* data);

/* ---- reference-absent KATs ---- */
/* Submanifold 3x3x3 kernel map over voxels sorted by (x,y,z): every pair
 * (out i, in j, offset z) with coord[j] == coord[i] + delta(z),
 * z = (dx+1)*9 + (dy+1)*3 + (dz+1). Output sorted by (z, i). Returns count
 * (call with outputs NULL to count). */
int64_t ixo_kernel_map(const int32_t* coords /*[n,3]*/, int64_t n, int64_t* map_out,
                       int64_t* map_in, int64_t* map_off);

/* Real-basis Clebsch–Gordan table for l_max; paths (l1,l2,l3) with
 * |l1-l2|<=l3<=l1+l2 and (l1+l2+l3) even, ordered by (l1,l2,l3). Entries
 * (i, j, k, path, value) with |value| > 1e-12; i indexes the output irrep
 * (offset l3^2 + m3), j the X irrep (l1^2+m1), k the Y irrep (l2^2+m2).
 * Returns count; call with NULL outputs to count. paths_out: [npaths, 3]. */
int64_t ixo_cg_table(int l_max, int64_t* ci, int64_t* cj, int64_t* ck, int64_t* cl, double* cv,
                     int* npaths, int64_t* paths_out);

#ifdef __cplusplus
}
#endif
#endif
