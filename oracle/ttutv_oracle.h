/*
 * TEST INFRASTRUCTURE ONLY -- never linked into the product.
 *
 * ttutv_oracle: a plain-C restatement of the reference CPU path for TT-UTV
 * (/root/reference/proj/src/{factor,tt_decomp,kernels,tt,tensor_ops,generators}.cpp),
 * written from the algorithm with the same floating-point operation order (no FMA
 * contraction), so it is pinned BITWISE against the reference library built in
 * oracle/_ref and against the committed golden fixtures (tests/golden/).
 *
 * Storage: column-major matrices, first-index-fastest tensors, int64 0-based perms.
 * Return codes: 0 ok, 1 argument error, 4 numerical error (Jacobi non-convergence).
 */
#ifndef TTUTV_ORACLE_H
#define TTUTV_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* generators.cpp:13-48 */
typedef struct orc_rng { uint64_t state; int has_spare; double spare; } orc_rng;
void orc_rng_init(orc_rng* r, uint64_t seed);
uint64_t orc_rng_u64(orc_rng* r);
double orc_rng_uniform(orc_rng* r);
double orc_rng_normal(orc_rng* r);
int64_t orc_rng_uniform_int(orc_rng* r, int64_t lo, int64_t hi);
void orc_gen_gaussian(int64_t count, uint64_t seed, double* out);
/* A(i) = 1 / (sum of 1-based indices - shift); shift = 0 is gen_hilbert (generators.cpp:50-60) */
void orc_gen_hilbert(const int64_t* dims, int d, double shift, double* out);
/* gen_planted_tt cores concatenated in core order (generators.cpp:62-79) */
void orc_gen_planted_cores(const int64_t* dims, int d, const int64_t* ranks, uint64_t seed, double* out);

/* kernels.cpp */
double orc_sum_squares_serial(const double* x, int64_t n);
double orc_sum_squares(const double* x, int64_t n); /* 4096-element blocks, block order */
void orc_matmul(const double* a, int64_t ar, int64_t ac, int ta, const double* b, int64_t br, int64_t bc, int tb,
                double* c);

/* factor.cpp */
int orc_qr_col_pivot(const double* a, int64_t m, int64_t n, double* q, double* r, int64_t* perm);
int orc_utv(const double* a, int64_t m, int64_t n, int lower, int refine, double* u, double* t, double* v);
int orc_svd(const double* a, int64_t m, int64_t n, int max_sweeps, double pair_tol, double* u, double* s,
            double* v);
/* kind 0 svd (t = p-vector s), 1 ulv, 2 urv; rank > 0 fixed, else eps. */
int orc_truncate(int kind, const double* u, const double* t, const double* v, int64_t m, int64_t n, int64_t p,
                 int64_t rank, double eps, int64_t* rank_out, double* residual, double* u1, double* t11,
                 double* v1);

/* tt.cpp / tensor_ops.cpp */
int orc_reconstruct(const double* cores, const int64_t* dims, const int64_t* ranks, int d, double* out);
double orc_rse(const double* est, const double* truth, int64_t n);

/* tt_decomp.cpp: method 0 svd 1 ulv 2 urv; sweep 0 l2r 1 r2l; retain 0 l11 1 full column.
 * cores_out: capacity `cap` doubles, cores concatenated; core_dims: 3*d; step_errors d-1;
 * ranks_chosen d+1; scalars: bound, bound_kind, input_norm. Returns 0 or an error code. */
int orc_decompose(const double* a, const int64_t* dims, int d, int method, int sweep, int fixed_rank,
                  const int64_t* ranks, double eps, const double* weights, int nweights, int refine, int retain,
                  double* cores_out, int64_t cap, int64_t* core_dims, double* step_errors, int64_t* ranks_chosen,
                  double* bound, int* bound_kind, double* input_norm);

const char* orc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
