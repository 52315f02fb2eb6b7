/*
 * ixo.c — CPU ORACLE, test infrastructure only. See ixo.h for scope and the
 * reference file:line each function restates. Plain C11, scalar, single
 * threaded: it is the checker, never the thing measured or shipped.
 */
#include "ixo.h"

#include <ctype.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ======================================================================
 * std::mt19937_64 (ISO C++ [rand.eng.mers] parameters)
 * ==================================================================== */
#define MT_N 312
#define MT_M 156
struct ixo_rng {
  uint64_t mt[MT_N];
  int idx;
};

ixo_rng* ixo_rng_new(uint64_t seed) {
  ixo_rng* r = (ixo_rng*)malloc(sizeof(ixo_rng));
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i) {
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  }
  r->idx = MT_N;
  return r;
}

void ixo_rng_free(ixo_rng* r) { free(r); }

static void mt_twist(ixo_rng* r) {
  const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
  const uint64_t a = 0xB5026F5AA96619E9ULL;
  for (int i = 0; i < MT_N; ++i) {
    uint64_t y = (r->mt[i] & upper) | (r->mt[(i + 1) % MT_N] & lower);
    r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ (y >> 1) ^ ((y & 1ULL) ? a : 0ULL);
  }
  r->idx = 0;
}

uint64_t ixo_rng_next(ixo_rng* r) {
  if (r->idx >= MT_N) mt_twist(r);
  uint64_t z = r->mt[r->idx++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= z >> 43;
  return z;
}

/* libstdc++ uniform_int_distribution<int64_t>: Lemire nearly-divisionless
 * downscale with 128-bit products (bits/uniform_int_dist.h, GCC 13). */
int64_t ixo_uniform_int(ixo_rng* r, int64_t a, int64_t b) {
  uint64_t urange = (uint64_t)b - (uint64_t)a;
  uint64_t ret;
  if (urange == UINT64_MAX) {
    ret = ixo_rng_next(r);
  } else {
    uint64_t erange = urange + 1;
    unsigned __int128 prod = (unsigned __int128)ixo_rng_next(r) * erange;
    uint64_t low = (uint64_t)prod;
    if (low < erange) {
      uint64_t thresh = (0 - erange) % erange;
      while (low < thresh) {
        prod = (unsigned __int128)ixo_rng_next(r) * erange;
        low = (uint64_t)prod;
      }
    }
    ret = (uint64_t)(prod >> 64);
  }
  return (int64_t)(ret + (uint64_t)a);
}

/* std::generate_canonical<double, 53> over a 64-bit engine: one draw. */
double ixo_canonical(ixo_rng* r) {
  double ret = (double)ixo_rng_next(r) / 18446744073709551616.0;
  if (ret >= 1.0) ret = nextafter(1.0, 0.0);
  return ret;
}

int ixo_bernoulli(ixo_rng* r, double p) { return ixo_canonical(r) < p; }

double ixo_uniform_real(ixo_rng* r, double a, double b) {
  return ixo_canonical(r) * (b - a) + a;
}

/* ======================================================================
 * synth.cpp
 * ==================================================================== */
static int64_t nonzero_int(ixo_rng* r) { /* synth.cpp:10-15 */
  int64_t v = ixo_uniform_int(r, 1, 4);
  return ixo_bernoulli(r, 0.5) ? v : -v;
}

static double nonzero_real(ixo_rng* r) { /* synth.cpp:17-22 */
  double v = ixo_uniform_real(r, 0.125, 1.0);
  return ixo_bernoulli(r, 0.5) ? v : -v;
}

static void put_nonzero(ixo_rng* r, int kind, void* out, int64_t i) {
  if (kind == IXO_INT) {
    ((int64_t*)out)[i] = nonzero_int(r);
  } else {
    ((double*)out)[i] = nonzero_real(r);
  }
}

static void zero_fill(int kind, int64_t n, void* out) {
  (void)kind;
  memset(out, 0, (size_t)n * 8);
}

void ixo_synth_dense(ixo_rng* r, int kind, int64_t numel, void* out) { /* synth.cpp:36-40 */
  for (int64_t i = 0; i < numel; ++i) put_nonzero(r, kind, out, i);
}

void ixo_synth_sparse_matrix(ixo_rng* r, int kind, int64_t rows, int64_t cols, double density,
                             void* out) { /* synth.cpp:42-54 */
  int64_t n = rows * cols;
  zero_fill(kind, n, out);
  for (int64_t i = 0; i < n; ++i) {
    if (!ixo_bernoulli(r, density)) continue;
    put_nonzero(r, kind, out, i);
  }
}

void ixo_synth_block_sparse_matrix(ixo_rng* r, int kind, int64_t rows, int64_t cols,
                                   int64_t br, int64_t bc, double bdens,
                                   void* out) { /* synth.cpp:56-78 */
  zero_fill(kind, rows * cols, out);
  int64_t gr = (rows + br - 1) / br, gc = (cols + bc - 1) / bc;
  for (int64_t bi = 0; bi < gr; ++bi) {
    for (int64_t bj = 0; bj < gc; ++bj) {
      if (!ixo_bernoulli(r, bdens)) continue;
      int64_t ie = (bi + 1) * br < rows ? (bi + 1) * br : rows;
      int64_t je = (bj + 1) * bc < cols ? (bj + 1) * bc : cols;
      for (int64_t i = bi * br; i < ie; ++i) {
        for (int64_t j = bj * bc; j < je; ++j) put_nonzero(r, kind, out, i * cols + j);
      }
    }
  }
}

/* open-addressing set of flat coordinates */
typedef struct {
  int64_t* keys;
  int64_t cap;
} flatset;

static int flatset_insert(flatset* s, int64_t key) {
  uint64_t h = (uint64_t)key * 0x9E3779B97F4A7C15ULL;
  int64_t i = (int64_t)(h % (uint64_t)s->cap);
  while (s->keys[i] != -1) {
    if (s->keys[i] == key) return 0;
    i = (i + 1) % s->cap;
  }
  s->keys[i] = key;
  return 1;
}

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

int64_t ixo_synth_coo_tensor(ixo_rng* r, int kind, int rank, const int64_t* shape, int64_t nnz,
                             int64_t* coords_out, void* vals_out) { /* synth.cpp:80-106 */
  int64_t capacity = 1;
  for (int d = 0; d < rank; ++d) capacity *= shape[d];
  if (nnz > capacity) nnz = capacity;
  flatset s;
  s.cap = 4 * nnz + 16;
  s.keys = (int64_t*)malloc((size_t)s.cap * 8);
  for (int64_t i = 0; i < s.cap; ++i) s.keys[i] = -1;
  int64_t* picked = (int64_t*)malloc((size_t)(nnz > 0 ? nnz : 1) * 8);
  int64_t np = 0;
  while (np < nnz) {
    int64_t flat = 0;
    for (int d = 0; d < rank; ++d) flat = flat * shape[d] + ixo_uniform_int(r, 0, shape[d] - 1);
    if (flatset_insert(&s, flat)) picked[np++] = flat;
  }
  /* std::sort of coordinate vectors == ascending row-major flat index */
  qsort(picked, (size_t)np, 8, cmp_i64);
  for (int64_t p = 0; p < np; ++p) {
    int64_t f = picked[p];
    for (int d = rank - 1; d >= 0; --d) {
      coords_out[d * np + p] = f % shape[d];
      f /= shape[d];
    }
  }
  ixo_synth_dense(r, kind, np, vals_out);
  free(picked);
  free(s.keys);
  return np;
}

/* ======================================================================
 * formats.cpp
 * ==================================================================== */
static int is_zero(int kind, const void* data, int64_t i) { /* formats.cpp:10-12 */
  return kind == IXO_INT ? ((const int64_t*)data)[i] == 0 : ((const double*)data)[i] == 0.0;
}

static void copy_elem(int kind, void* dst, int64_t di, const void* src, int64_t si) {
  (void)kind;
  memcpy((char*)dst + di * 8, (const char*)src + si * 8, 8);
}

int64_t ixo_count_nonzero(int kind, int64_t n, const void* data) {
  int64_t c = 0;
  for (int64_t i = 0; i < n; ++i) c += !is_zero(kind, data, i);
  return c;
}

void ixo_dense_to_coo(int kind, int64_t rows, int64_t cols, const void* data, int64_t* row_coord,
                      int64_t* col_coord, void* values) { /* formats.cpp:24-46 */
  int64_t p = 0;
  for (int64_t i = 0; i < rows; ++i) {
    for (int64_t j = 0; j < cols; ++j) {
      int64_t flat = i * cols + j;
      if (!is_zero(kind, data, flat)) {
        row_coord[p] = i;
        col_coord[p] = j;
        copy_elem(kind, values, p, data, flat);
        ++p;
      }
    }
  }
}

/* Stable merge sort of `order` under a multi-key lexicographic compare
 * (keys[k][idx], k = 0..nkeys-1) — std::stable_sort semantics. */
typedef struct {
  const int64_t* const* keys;
  int nkeys;
} keyset;

static int key_less(const keyset* ks, int64_t a, int64_t b) {
  for (int k = 0; k < ks->nkeys; ++k) {
    int64_t x = ks->keys[k][a], y = ks->keys[k][b];
    if (x != y) return x < y;
  }
  return 0;
}

static void stable_sort_idx(int64_t* order, int64_t n, const keyset* ks) {
  int64_t* tmp = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * 8);
  for (int64_t w = 1; w < n; w *= 2) {
    for (int64_t lo = 0; lo < n; lo += 2 * w) {
      int64_t mid = lo + w < n ? lo + w : n, hi = lo + 2 * w < n ? lo + 2 * w : n;
      int64_t i = lo, j = mid, o = lo;
      while (i < mid && j < hi) {
        /* take from the right only when strictly less: stability */
        if (key_less(ks, order[j], order[i])) tmp[o++] = order[j++];
        else tmp[o++] = order[i++];
      }
      while (i < mid) tmp[o++] = order[i++];
      while (j < hi) tmp[o++] = order[j++];
    }
    memcpy(order, tmp, (size_t)n * 8);
  }
  free(tmp);
}

/* Shared run-splitting core of coo_to_groupcoo / group_coo_tensor
 * (formats.cpp:137-164, 445-470). `order` is sorted; gcoord is the grouped
 * coordinate. Emits slot sources (-1 = pad). Returns G. */
static int64_t split_runs(const int64_t* order, int64_t n, const int64_t* gcoord, int64_t g,
                          int64_t* group_coord, int64_t* slot_src) {
  int64_t G = 0, i = 0;
  while (i < n) {
    int64_t run_end = i;
    while (run_end < n && gcoord[order[run_end]] == gcoord[order[i]]) ++run_end;
    for (int64_t start = i; start < run_end; start += g) {
      if (group_coord) group_coord[G] = gcoord[order[i]];
      int64_t take = run_end - start < g ? run_end - start : g;
      if (slot_src) {
        for (int64_t k = 0; k < g; ++k) slot_src[G * g + k] = k < take ? order[start + k] : -1;
      }
      ++G;
    }
    i = run_end;
  }
  return G;
}

int ixo_coo_to_groupcoo(int64_t rows, int64_t cols, const int64_t* r, const int64_t* c, int kind,
                        const void* vals, int64_t nnz, int group_dim, int64_t g, int64_t* G_out,
                        int64_t* AM, int64_t* AK, void* AV,
                        uint8_t* mask) { /* formats.cpp:115-174 */
  (void)rows;
  (void)cols;
  if (g < 1) return IXO_SHAPE;
  if (group_dim != 0 && group_dim != 1) return IXO_SHAPE;
  const int64_t* gcoord = group_dim == 0 ? r : c;
  const int64_t* mcoord = group_dim == 0 ? c : r;
  int64_t* order = (int64_t*)malloc((size_t)(nnz > 0 ? nnz : 1) * 8);
  for (int64_t i = 0; i < nnz; ++i) order[i] = i;
  const int64_t* kk[2] = {gcoord, mcoord};
  keyset ks = {kk, 2};
  stable_sort_idx(order, nnz, &ks);
  int64_t G = split_runs(order, nnz, gcoord, g, NULL, NULL);
  *G_out = G;
  if (AM) {
    int64_t* src = (int64_t*)malloc((size_t)(G * g > 0 ? G * g : 1) * 8);
    split_runs(order, nnz, gcoord, g, AM, src);
    for (int64_t s = 0; s < G * g; ++s) {
      if (src[s] >= 0) {
        AK[s] = mcoord[src[s]];
        copy_elem(kind, AV, s, vals, src[s]);
        mask[s] = 1;
      } else {
        AK[s] = AK[s - 1]; /* pad repeats the last real member (formats.cpp:156-157) */
        memset((char*)AV + s * 8, 0, 8);
        mask[s] = 0;
      }
    }
    free(src);
  }
  free(order);
  return IXO_OK;
}

int ixo_dense_to_blockgroupcoo(int kind, int64_t rows, int64_t cols, const void* data, int64_t bm,
                               int64_t bk, int64_t g, int group_dim, int64_t* G_out, int64_t* AM,
                               int64_t* AK, void* AV,
                               uint8_t* mask) { /* formats.cpp:224-292 */
  if (bm < 1 || bk < 1) return IXO_SHAPE;
  if (g < 1) return IXO_SHAPE;
  int64_t gr = (rows + bm - 1) / bm, gcn = (cols + bk - 1) / bk;
  int64_t cap = gr * gcn;
  int64_t* br = (int64_t*)malloc((size_t)(cap > 0 ? cap : 1) * 8);
  int64_t* bc = (int64_t*)malloc((size_t)(cap > 0 ? cap : 1) * 8);
  int64_t nb = 0;
  for (int64_t bi = 0; bi < gr; ++bi) {
    for (int64_t bj = 0; bj < gcn; ++bj) {
      int any = 0;
      int64_t ie = (bi + 1) * bm < rows ? (bi + 1) * bm : rows;
      int64_t je = (bj + 1) * bk < cols ? (bj + 1) * bk : cols;
      for (int64_t i = bi * bm; i < ie && !any; ++i) {
        for (int64_t j = bj * bk; j < je; ++j) {
          if (!is_zero(kind, data, i * cols + j)) {
            any = 1;
            break;
          }
        }
      }
      if (any) {
        br[nb] = bi;
        bc[nb] = bj;
        ++nb;
      }
    }
  }
  double* zeros = (double*)calloc((size_t)(nb > 0 ? nb : 1), 8);
  int64_t G = 0;
  int st = ixo_coo_to_groupcoo(gr, gcn, br, bc, kind, zeros, nb, group_dim, g, &G, NULL, NULL,
                               NULL, NULL);
  if (st != IXO_OK) goto done;
  *G_out = G;
  if (AM) {
    double* dummy = (double*)malloc((size_t)(G * g > 0 ? G * g : 1) * 8);
    ixo_coo_to_groupcoo(gr, gcn, br, bc, kind, zeros, nb, group_dim, g, &G, AM, AK, dummy, mask);
    free(dummy);
    memset(AV, 0, (size_t)(G * g * bm * bk) * 8);
    for (int64_t p = 0; p < G; ++p) {
      for (int64_t q = 0; q < g; ++q) {
        int64_t slot = p * g + q;
        if (!mask[slot]) continue;
        int64_t rb = group_dim == 0 ? AM[p] : AK[slot];
        int64_t cb = group_dim == 0 ? AK[slot] : AM[p];
        for (int64_t i = 0; i < bm; ++i) {
          for (int64_t j = 0; j < bk; ++j) {
            int64_t si = rb * bm + i, sj = cb * bk + j;
            if (si >= rows || sj >= cols) continue;
            copy_elem(kind, AV, (slot * bm + i) * bk + j, data, si * cols + sj);
          }
        }
      }
    }
  }
done:
  free(zeros);
  free(br);
  free(bc);
  return st;
}

int ixo_group_coo_tensor(int rank, const int64_t* shape, const int64_t* coords, int kind,
                         const void* vals, int64_t nnz, int group_dim, int64_t g, int64_t* G_out,
                         int64_t* group_coord, int64_t* member_coords, void* values,
                         uint8_t* mask) { /* formats.cpp:417-479 */
  (void)shape;
  if (g < 1) return IXO_SHAPE;
  if (group_dim < 0 || group_dim >= rank) return IXO_SHAPE;
  int64_t* order = (int64_t*)malloc((size_t)(nnz > 0 ? nnz : 1) * 8);
  for (int64_t i = 0; i < nnz; ++i) order[i] = i;
  const int64_t* kk[16];
  int nk = 0;
  kk[nk++] = coords + group_dim * nnz;
  for (int d = 0; d < rank; ++d) {
    if (d != group_dim) kk[nk++] = coords + d * nnz;
  }
  keyset ks = {kk, nk};
  stable_sort_idx(order, nnz, &ks);
  const int64_t* gcoord = coords + group_dim * nnz;
  int64_t G = split_runs(order, nnz, gcoord, g, NULL, NULL);
  *G_out = G;
  if (group_coord) {
    int64_t* src = (int64_t*)malloc((size_t)(G * g > 0 ? G * g : 1) * 8);
    split_runs(order, nnz, gcoord, g, group_coord, src);
    int m = 0;
    for (int d = 0; d < rank; ++d) {
      if (d == group_dim) continue;
      int64_t* mc = member_coords + (int64_t)m * G * g;
      for (int64_t s = 0; s < G * g; ++s) {
        mc[s] = src[s] >= 0 ? coords[d * nnz + src[s]] : mc[s - 1];
      }
      ++m;
    }
    for (int64_t s = 0; s < G * g; ++s) {
      if (src[s] >= 0) {
        copy_elem(kind, values, s, vals, src[s]);
        mask[s] = 1;
      } else {
        memset((char*)values + s * 8, 0, 8);
        mask[s] = 0;
      }
    }
    free(src);
  }
  free(order);
  return IXO_OK;
}

/* ======================================================================
 * tuner.cpp
 * ==================================================================== */
static int64_t occ_total(const int64_t* occ, int64_t n) {
  int64_t s = 0;
  for (int64_t i = 0; i < n; ++i) s += occ[i];
  return s;
}
static int64_t occ_nonzero(const int64_t* occ, int64_t n) {
  int64_t c = 0;
  for (int64_t i = 0; i < n; ++i) c += occ[i] > 0;
  return c;
}
static int64_t occ_max(const int64_t* occ, int64_t n) {
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i) m = occ[i] > m ? occ[i] : m;
  return m;
}

int64_t ixo_cost_exact(const int64_t* occ, int64_t n, int64_t g) { /* tuner.cpp:31-36 */
  if (g < 1) return -1;
  int64_t groups = 0;
  for (int64_t i = 0; i < n; ++i) groups += (occ[i] + g - 1) / g;
  return (g + 1) * groups;
}

double ixo_cost_relaxed(const int64_t* occ, int64_t n, double g, int count_empty_rows) {
  double s = (double)occ_total(occ, n);
  double nn = (double)(count_empty_rows ? n : occ_nonzero(occ, n));
  return s + s / g + nn * g + nn; /* tuner.cpp:46-51 */
}

double ixo_g_star(const int64_t* occ, int64_t n, int count_empty_rows) { /* tuner.cpp:60-65 */
  if (occ_total(occ, n) == 0) return 1.0;
  double nn = (double)(count_empty_rows ? n : occ_nonzero(occ, n));
  if (nn <= 0) return 1.0;
  return sqrt((double)occ_total(occ, n) / nn);
}

int ixo_candidate_group_sizes(const int64_t* occ, int64_t n, int count_empty_rows,
                              int64_t* cand) { /* tuner.cpp:67-84 */
  if (occ_total(occ, n) == 0) {
    cand[0] = 1;
    return 1;
  }
  double gs = ixo_g_star(occ, n, count_empty_rows);
  int64_t lo = 1;
  while (lo * 2 <= (int64_t)gs) lo *= 2;
  int64_t hi = lo;
  while ((double)hi < gs) hi *= 2;
  int64_t cap = 1, mo = occ_max(occ, n);
  while (cap * 2 <= mo) cap *= 2;
  lo = lo < 1 ? 1 : (lo > cap ? cap : lo);
  hi = hi < 1 ? 1 : (hi > cap ? cap : hi);
  cand[0] = lo;
  if (lo == hi) return 1;
  cand[1] = hi;
  return 2;
}

int64_t ixo_select(const int64_t* occ, int64_t n, int count_empty_rows) { /* tuner.cpp:100-118 */
  int64_t cand[2];
  int nc = ixo_candidate_group_sizes(occ, n, count_empty_rows, cand);
  int64_t chosen = cand[0];
  double best = (double)ixo_cost_exact(occ, n, cand[0]);
  for (int i = 0; i < nc; ++i) {
    double sc = (double)ixo_cost_exact(occ, n, cand[i]);
    if (sc < best) {
      best = sc;
      chosen = cand[i];
    }
  }
  return chosen;
}

int64_t ixo_brute_force_optimal(const int64_t* occ, int64_t n, int64_t* f_out) {
  if (occ_total(occ, n) == 0) return 0; /* tuner.cpp:86-98 */
  int64_t best_g = 1, best_f = ixo_cost_exact(occ, n, 1), mo = occ_max(occ, n);
  for (int64_t g = 2; g <= mo; ++g) {
    int64_t f = ixo_cost_exact(occ, n, g);
    if (f < best_f) {
      best_f = f;
      best_g = g;
    }
  }
  *f_out = best_f;
  return best_g;
}

/* ======================================================================
 * oracle_einsum: parser (expr.cpp:36-181) + odometer (plan.cpp:579-594)
 * ==================================================================== */
#define MAXN 32
#define MAXD 8
typedef struct {
  char tensor[MAXN];
  int nidx;
  int indirect[MAXD];         /* 0 direct, 1 indirect */
  char var[MAXD][MAXN];       /* direct var, or index-tensor name */
  int nargs[MAXD];
  char args[MAXD][MAXD][MAXN];
} access_t;

typedef struct {
  access_t out;
  access_t in[MAXD];
  int nin;
  int accumulate;
  char vars[2 * MAXD * MAXD][MAXN];
  int nvars;
} stmt_t;

typedef struct {
  const char* s;
  size_t pos;
  char* err;
  int errlen;
  int failed;
} parser_t;

static void pfail(parser_t* p, const char* msg) {
  if (!p->failed) snprintf(p->err, (size_t)p->errlen, "%s (at position %zu)", msg, p->pos);
  p->failed = 1;
}
static void skip_ws(parser_t* p) {
  while (p->s[p->pos] && isspace((unsigned char)p->s[p->pos])) ++p->pos;
}
static int peekc(parser_t* p, char c) {
  skip_ws(p);
  return p->s[p->pos] == c;
}
static int consume(parser_t* p, const char* tok) {
  skip_ws(p);
  size_t n = strlen(tok);
  if (strncmp(p->s + p->pos, tok, n) == 0) {
    p->pos += n;
    return 1;
  }
  return 0;
}
static void expect(parser_t* p, char c) {
  skip_ws(p);
  if (p->s[p->pos] != c) {
    char m[32];
    snprintf(m, sizeof m, "expected '%c'", c);
    pfail(p, m);
    return;
  }
  ++p->pos;
}
static void parse_ident(parser_t* p, const char* what, char* out) {
  skip_ws(p);
  size_t st = p->pos;
  char c = p->s[p->pos];
  if (c && (isalpha((unsigned char)c) || c == '_')) {
    ++p->pos;
    while (p->s[p->pos] && (isalnum((unsigned char)p->s[p->pos]) || p->s[p->pos] == '_')) ++p->pos;
    size_t n = p->pos - st < MAXN - 1 ? p->pos - st : MAXN - 1;
    memcpy(out, p->s + st, n);
    out[n] = 0;
    return;
  }
  char m[64];
  snprintf(m, sizeof m, "expected %s", what);
  pfail(p, m);
  out[0] = 0;
}
static void parse_access(parser_t* p, access_t* a) {
  memset(a, 0, sizeof *a);
  parse_ident(p, "tensor name", a->tensor);
  expect(p, '[');
  do {
    if (p->failed) return;
    int d = a->nidx++;
    parse_ident(p, "index variable", a->var[d]);
    skip_ws(p);
    if (peekc(p, '[')) {
      expect(p, '[');
      a->indirect[d] = 1;
      do {
        size_t at;
        skip_ws(p);
        at = p->pos;
        parse_ident(p, "indirection argument", a->args[d][a->nargs[d]++]);
        skip_ws(p);
        if (peekc(p, '[')) {
          p->pos = at;
          pfail(p, "nested indirection is not supported");
          return;
        }
        skip_ws(p);
      } while (!p->failed && consume(p, ","));
      expect(p, ']');
    }
    skip_ws(p);
  } while (!p->failed && consume(p, ","));
  expect(p, ']');
}
static void add_var(stmt_t* st, const char* v) {
  for (int i = 0; i < st->nvars; ++i) {
    if (!strcmp(st->vars[i], v)) return;
  }
  strcpy(st->vars[st->nvars++], v);
}
static void scan_vars(stmt_t* st, const access_t* a) {
  for (int d = 0; d < a->nidx; ++d) {
    if (!a->indirect[d]) add_var(st, a->var[d]);
    else for (int k = 0; k < a->nargs[d]; ++k) add_var(st, a->args[d][k]);
  }
}
static int parse_stmt(const char* s, stmt_t* st, char* err, int errlen) {
  parser_t p = {s, 0, err, errlen, 0};
  memset(st, 0, sizeof *st);
  parse_access(&p, &st->out);
  if (p.failed) return IXO_PARSE;
  skip_ws(&p);
  if (consume(&p, "+=")) st->accumulate = 1;
  else if (consume(&p, "=")) st->accumulate = 0;
  else pfail(&p, "expected '=' or '+='");
  if (p.failed) return IXO_PARSE;
  parse_access(&p, &st->in[st->nin++]);
  skip_ws(&p);
  while (!p.failed && consume(&p, "*")) {
    if (st->nin >= MAXD) {
      pfail(&p, "too many factors");
      break;
    }
    parse_access(&p, &st->in[st->nin++]);
    skip_ws(&p);
  }
  if (!p.failed && p.s[p.pos]) pfail(&p, "unexpected trailing input");
  if (p.failed) return IXO_PARSE;
  scan_vars(st, &st->out);
  for (int i = 0; i < st->nin; ++i) scan_vars(st, &st->in[i]);
  return IXO_OK;
}

typedef struct {
  const ixo_tensor* t;
  int64_t strides[MAXD];
  int direct_slot[MAXD];
  const ixo_tensor* idx_t[MAXD];
  int arg_slot[MAXD][MAXD];
  int nargs[MAXD];
  const char* idx_name[MAXD];
} compiled_t;

static const ixo_tensor* find_t(const ixo_tensor* ts, int n, const char* name) {
  for (int i = 0; i < n; ++i) {
    if (!strcmp(ts[i].name, name)) return &ts[i];
  }
  return NULL;
}
static int var_slot(const stmt_t* st, const char* v) {
  for (int i = 0; i < st->nvars; ++i) {
    if (!strcmp(st->vars[i], v)) return i;
  }
  return -1;
}

static int errf(char* err, int errlen, int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(err, (size_t)errlen, fmt, ap);
  va_end(ap);
  return code;
}

/* infer_extents (expr.cpp:236-283) fused with validate_bindings (plan.cpp:199-247). */
static int note_extent(int64_t* ext, int slot, int64_t e, const char* var, char* err, int errlen) {
  if (ext[slot] < 0) ext[slot] = e;
  else if (ext[slot] != e)
    return errf(err, errlen, IXO_SHAPE, "extent conflict for %s: %lld vs %lld", var,
                (long long)ext[slot], (long long)e);
  return IXO_OK;
}

static int infer_access(const stmt_t* st, const access_t* a, const ixo_tensor* t,
                        const ixo_tensor* ts, int nt, int64_t* ext, char* err, int errlen) {
  if (t->rank != a->nidx)
    return errf(err, errlen, IXO_SHAPE, "rank mismatch: %s has rank %d but is accessed with %d indices",
                a->tensor, t->rank, a->nidx);
  for (int d = 0; d < a->nidx; ++d) {
    int rc;
    if (!a->indirect[d]) {
      rc = note_extent(ext, var_slot(st, a->var[d]), t->shape[d], a->var[d], err, errlen);
      if (rc) return rc;
    } else {
      const ixo_tensor* it = find_t(ts, nt, a->var[d]);
      if (!it) return errf(err, errlen, IXO_SHAPE, "no shape given for tensor %s", a->var[d]);
      if (it->rank != a->nargs[d])
        return errf(err, errlen, IXO_SHAPE,
                    "rank mismatch: index tensor %s has rank %d but is accessed with %d indices",
                    a->var[d], it->rank, a->nargs[d]);
      for (int k = 0; k < a->nargs[d]; ++k) {
        rc = note_extent(ext, var_slot(st, a->args[d][k]), it->shape[k], a->args[d][k], err,
                         errlen);
        if (rc) return rc;
      }
    }
  }
  return IXO_OK;
}

static int compile_access(const stmt_t* st, const access_t* a, const ixo_tensor* t,
                          const ixo_tensor* ts, int nt, compiled_t* c, char* err, int errlen) {
  memset(c, 0, sizeof *c);
  c->t = t;
  int64_t s = 1;
  for (int d = t->rank - 1; d >= 0; --d) {
    c->strides[d] = s;
    s *= t->shape[d];
  }
  for (int d = 0; d < a->nidx; ++d) {
    if (!a->indirect[d]) {
      c->direct_slot[d] = var_slot(st, a->var[d]);
    } else {
      const ixo_tensor* it = find_t(ts, nt, a->var[d]);
      if (!it) return errf(err, errlen, IXO_BIND, "unbound tensor %s", a->var[d]);
      if (it->kind != IXO_INT)
        return errf(err, errlen, IXO_BIND, "index tensor %s must be int64, got real64", a->var[d]);
      c->direct_slot[d] = -1;
      c->idx_t[d] = it;
      c->idx_name[d] = a->var[d];
      c->nargs[d] = a->nargs[d];
      for (int k = 0; k < a->nargs[d]; ++k) c->arg_slot[d][k] = var_slot(st, a->args[d][k]);
    }
  }
  return IXO_OK;
}

/* CompiledAccess::flat_at with checked_index (plan.cpp:249-259, 316-335). */
static int flat_at(const compiled_t* c, const int64_t* pt, int64_t* flat, const char* tname,
                   char* err, int errlen) {
  int64_t f = 0;
  for (int d = 0; d < c->t->rank; ++d) {
    int64_t idx;
    if (c->direct_slot[d] >= 0) {
      idx = pt[c->direct_slot[d]];
    } else {
      const ixo_tensor* it = c->idx_t[d];
      int64_t iflat = 0;
      for (int k = 0; k < c->nargs[d]; ++k) iflat = iflat * it->shape[k] + pt[c->arg_slot[d][k]];
      idx = ((const int64_t*)it->data)[iflat];
      if (idx < 0 || idx >= c->t->shape[d])
        return errf(err, errlen, IXO_INDEX_RANGE,
                    "index tensor %s value %lld at position [%lld] out of range for dim %d of %s "
                    "(extent %lld)",
                    c->idx_name[d], (long long)idx, (long long)iflat, d, tname,
                    (long long)c->t->shape[d]);
    }
    f += c->strides[d] * idx;
  }
  *flat = f;
  return IXO_OK;
}

int ixo_einsum(const char* expr, const ixo_tensor* tensors, int ntensors, const char* out_name,
               int out_kind, int out_rank, const int64_t* out_shape, void* out, char* err,
               int errlen) {
  stmt_t st;
  int rc = parse_stmt(expr, &st, err, errlen);
  if (rc) return rc;
  ixo_tensor outt = {out_name, out_kind, out_rank, out_shape, out};
  /* shapes of every named tensor must exist (infer_extents) */
  int64_t ext[2 * MAXD * MAXD];
  for (int i = 0; i < st.nvars; ++i) ext[i] = -1;
  if (strcmp(st.out.tensor, out_name) != 0)
    return errf(err, errlen, IXO_BIND, "output buffer %s does not match statement output %s",
                out_name, st.out.tensor);
  rc = infer_access(&st, &st.out, &outt, tensors, ntensors, ext, err, errlen);
  if (rc) return rc;
  const ixo_tensor* ins[MAXD];
  for (int i = 0; i < st.nin; ++i) {
    ins[i] = find_t(tensors, ntensors, st.in[i].tensor);
    if (!ins[i]) return errf(err, errlen, IXO_SHAPE, "no shape given for tensor %s", st.in[i].tensor);
    rc = infer_access(&st, &st.in[i], ins[i], tensors, ntensors, ext, err, errlen);
    if (rc) return rc;
  }
  for (int i = 0; i < st.nin; ++i) {
    if (ins[i]->kind != out_kind)
      return errf(err, errlen, IXO_BIND, "tensor %s is %s but the output buffer is %s",
                  st.in[i].tensor, ins[i]->kind ? "int64" : "real64", out_kind ? "int64" : "real64");
  }
  compiled_t oc, ic[MAXD];
  rc = compile_access(&st, &st.out, &outt, tensors, ntensors, &oc, err, errlen);
  if (rc) return rc;
  for (int i = 0; i < st.nin; ++i) {
    rc = compile_access(&st, &st.in[i], ins[i], tensors, ntensors, &ic[i], err, errlen);
    if (rc) return rc;
  }
  int64_t onum = 1;
  for (int d = 0; d < out_rank; ++d) onum *= out_shape[d];
  if (!st.accumulate) memset(out, 0, (size_t)onum * 8);
  int64_t total = 1;
  for (int i = 0; i < st.nvars; ++i) total *= ext[i];
  if (total == 0) return IXO_OK;
  int64_t pt[2 * MAXD * MAXD];
  memset(pt, 0, sizeof pt);
  for (;;) {
    int64_t f;
    if (out_kind == IXO_INT) {
      int64_t prod = 1;
      for (int i = 0; i < st.nin; ++i) {
        rc = flat_at(&ic[i], pt, &f, st.in[i].tensor, err, errlen);
        if (rc) return rc;
        prod *= ((const int64_t*)ins[i]->data)[f];
      }
      rc = flat_at(&oc, pt, &f, out_name, err, errlen);
      if (rc) return rc;
      ((int64_t*)out)[f] += prod;
    } else {
      double prod = 1.0;
      for (int i = 0; i < st.nin; ++i) {
        rc = flat_at(&ic[i], pt, &f, st.in[i].tensor, err, errlen);
        if (rc) return rc;
        prod *= ((const double*)ins[i]->data)[f];
      }
      rc = flat_at(&oc, pt, &f, out_name, err, errlen);
      if (rc) return rc;
      ((double*)out)[f] += prod;
    }
    int i = st.nvars - 1;
    for (; i >= 0; --i) {
      if (++pt[i] < ext[i]) break;
      pt[i] = 0;
    }
    if (i < 0) break;
  }
  return IXO_OK;
}

/* tensor.cpp:124-136 */
double ixo_max_rel_error(int kind, int64_t n, const void* a, const void* b) {
  double worst = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double x = kind == IXO_INT ? (double)((const int64_t*)a)[i] : ((const double*)a)[i];
    double y = kind == IXO_INT ? (double)((const int64_t*)b)[i] : ((const double*)b)[i];
    double den = fabs(x);
    if (fabs(y) > den) den = fabs(y);
    if (1.0 > den) den = 1.0;
    double e = fabs(x - y) / den;
    if (e > worst) worst = e;
  }
  return worst;
}

/* tensor.cpp:138-156 (FNV-1a) */
uint64_t ixo_tensor_hash(int kind, int rank, const int64_t* shape, const void* data) {
  uint64_t h = 1469598103934665603ULL;
#define MIX(p, n)                                             \
  do {                                                        \
    const unsigned char* b_ = (const unsigned char*)(p);      \
    for (size_t i_ = 0; i_ < (size_t)(n); ++i_) {             \
      h ^= b_[i_];                                            \
      h *= 1099511628211ULL;                                  \
    }                                                         \
  } while (0)
  uint64_t k = kind == IXO_REAL ? 0 : 1;
  MIX(&k, 8);
  int64_t n = 1;
  for (int d = 0; d < rank; ++d) {
    MIX(&shape[d], 8);
    n *= shape[d];
  }
  MIX(data, n * 8);
#undef MIX
  return h;
}

/* ======================================================================
 * Kernel map (reference-absent)
 * ==================================================================== */
typedef struct {
  int64_t key;
  int64_t idx;
} kv_t;

static int cmp_kv(const void* a, const void* b) {
  int64_t x = ((const kv_t*)a)->key, y = ((const kv_t*)b)->key;
  return (x > y) - (x < y);
}

static int64_t vox_key(int64_t x, int64_t y, int64_t z) {
  /* coordinates are biased into [0, 2^21) */
  return ((x + (1 << 20)) << 42) | ((y + (1 << 20)) << 21) | (z + (1 << 20));
}

int64_t ixo_kernel_map(const int32_t* coords, int64_t n, int64_t* map_out, int64_t* map_in,
                       int64_t* map_off) {
  kv_t* tab = (kv_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(kv_t));
  for (int64_t i = 0; i < n; ++i) {
    tab[i].key = vox_key(coords[3 * i], coords[3 * i + 1], coords[3 * i + 2]);
    tab[i].idx = i;
  }
  qsort(tab, (size_t)n, sizeof(kv_t), cmp_kv);
  int64_t cnt = 0;
  for (int z = 0; z < 27; ++z) {
    int dx = z / 9 - 1, dy = (z / 3) % 3 - 1, dz = z % 3 - 1;
    for (int64_t i = 0; i < n; ++i) {
      kv_t probe;
      probe.key = vox_key((int64_t)coords[3 * i] + dx, (int64_t)coords[3 * i + 1] + dy,
                          (int64_t)coords[3 * i + 2] + dz);
      kv_t* hit = (kv_t*)bsearch(&probe, tab, (size_t)n, sizeof(kv_t), cmp_kv);
      if (!hit) continue;
      if (map_out) {
        map_out[cnt] = i;
        map_in[cnt] = hit->idx;
        map_off[cnt] = z;
      }
      ++cnt;
    }
  }
  free(tab);
  return cnt;
}

/* ======================================================================
 * Real-basis Clebsch–Gordan (reference-absent)
 * ==================================================================== */
static double lfact(int n) { return lgamma((double)n + 1.0); }

/* Complex-basis <l1 m1 l2 m2 | l3 m3> via the Racah formula. */
static double cg_complex(int l1, int m1, int l2, int m2, int l3, int m3) {
  if (m1 + m2 != m3) return 0.0;
  if (abs(m1) > l1 || abs(m2) > l2 || abs(m3) > l3) return 0.0;
  if (l3 < abs(l1 - l2) || l3 > l1 + l2) return 0.0;
  double pre = 0.5 * (log(2.0 * l3 + 1.0) + lfact(l3 + l1 - l2) + lfact(l3 - l1 + l2) +
                      lfact(l1 + l2 - l3) - lfact(l1 + l2 + l3 + 1) + lfact(l3 + m3) +
                      lfact(l3 - m3) + lfact(l1 - m1) + lfact(l1 + m1) + lfact(l2 - m2) +
                      lfact(l2 + m2));
  double sum = 0.0;
  for (int k = 0; k <= l1 + l2 + l3; ++k) {
    int a = l1 + l2 - l3 - k, b = l1 - m1 - k, c = l2 + m2 - k, d = l3 - l2 + m1 + k,
        e = l3 - l1 - m2 + k;
    if (a < 0 || b < 0 || c < 0 || d < 0 || e < 0) continue;
    double t = -(lfact(k) + lfact(a) + lfact(b) + lfact(c) + lfact(d) + lfact(e));
    sum += ((k & 1) ? -1.0 : 1.0) * exp(pre + t);
  }
  return sum;
}

/* Real spherical-harmonic basis change U[l]: real_m = sum_mu U[m][mu] complex_mu,
 * real index r = m + l. Entries are complex: stored as (re, im). */
static void real_basis(int l, double* ure, double* uim) {
  int n = 2 * l + 1;
  memset(ure, 0, (size_t)(n * n) * sizeof(double));
  memset(uim, 0, (size_t)(n * n) * sizeof(double));
  const double s = 1.0 / sqrt(2.0);
  for (int m = -l; m <= l; ++m) {
    int r = m + l;
    if (m == 0) {
      ure[r * n + l] = 1.0;
    } else if (m > 0) {
      ure[r * n + (-m + l)] = s;
      ure[r * n + (m + l)] = (m & 1) ? -s : s;
    } else {
      int am = -m;
      uim[r * n + (m + l)] = s;                   /* i/sqrt2 * Y_{l,-|m|} */
      uim[r * n + (am + l)] = (am & 1) ? s : -s;  /* -i/sqrt2 * (-1)^m Y_{l,|m|} */
    }
  }
}

int64_t ixo_cg_table(int l_max, int64_t* ci, int64_t* cj, int64_t* ck, int64_t* cl, double* cv,
                     int* npaths, int64_t* paths_out) {
  int64_t cnt = 0;
  int path = 0;
  for (int l1 = 0; l1 <= l_max; ++l1) {
    for (int l2 = 0; l2 <= l_max; ++l2) {
      for (int l3 = 0; l3 <= l_max; ++l3) {
        if (l3 < abs(l1 - l2) || l3 > l1 + l2 || ((l1 + l2 + l3) & 1)) continue;
        int n1 = 2 * l1 + 1, n2 = 2 * l2 + 1, n3 = 2 * l3 + 1;
        double u1r[64], u1i[64], u2r[64], u2i[64], u3r[64], u3i[64];
        real_basis(l1, u1r, u1i);
        real_basis(l2, u2r, u2i);
        real_basis(l3, u3r, u3i);
        /* C_real[a,b,c] = sum conj(U1[a,mu1]) conj(U2[b,mu2]) U3[c,mu3] C(mu1,mu2,mu3):
         * coupling real X (index a) and real Y (index b) into real Z (index c). */
        for (int c = 0; c < n3; ++c) {
          for (int a = 0; a < n1; ++a) {
            for (int b = 0; b < n2; ++b) {
              double re = 0.0, im = 0.0;
              for (int m1 = -l1; m1 <= l1; ++m1) {
                for (int m2 = -l2; m2 <= l2; ++m2) {
                  int m3 = m1 + m2;
                  if (abs(m3) > l3) continue;
                  double cgv = cg_complex(l1, m1, l2, m2, l3, m3);
                  if (cgv == 0.0) continue;
                  /* x = U3[c,m3] * conj(U1[a,m1]) * conj(U2[b,m2]) */
                  double ar = u1r[a * n1 + m1 + l1], ai = -u1i[a * n1 + m1 + l1];
                  double br = u2r[b * n2 + m2 + l2], bi = -u2i[b * n2 + m2 + l2];
                  double cr = u3r[c * n3 + m3 + l3], ci_ = u3i[c * n3 + m3 + l3];
                  double tr = ar * br - ai * bi, ti = ar * bi + ai * br;
                  double xr = tr * cr - ti * ci_, xi = tr * ci_ + ti * cr;
                  re += cgv * xr;
                  im += cgv * xi;
                }
              }
              (void)im; /* even l1+l2+l3: the coupling is real */
              if (fabs(re) > 1e-12) {
                if (ci) {
                  ci[cnt] = l3 * l3 + c;
                  cj[cnt] = l1 * l1 + a;
                  ck[cnt] = l2 * l2 + b;
                  cl[cnt] = path;
                  cv[cnt] = re;
                }
                ++cnt;
              }
            }
          }
        }
        if (paths_out) {
          paths_out[3 * path] = l1;
          paths_out[3 * path + 1] = l2;
          paths_out[3 * path + 2] = l3;
        }
        ++path;
      }
    }
  }
  if (npaths) *npaths = path;
  return cnt;
}
