/*
 * ttutv_b200.h -- C-ABI of the B200-native TT-UTV engine.
 *
 * This is the drop-in boundary: plain pointers, sizes and status codes, no C++ or
 * torch types. The C++ API in include/ttutv_b200/ttutv.hpp (namespace ttutv, the same
 * names and signatures as the reference's include/ttutv/*.hpp) is a thin layer over
 * these entry points, and any FFI (ctypes, cgo, JNI) can bind them directly
 * (see INTEGRATION.md).
 *
 * Every entry point replaces one reference interface (paths relative to
 * /root/reference/proj):
 *   ttg_decompose          <- decompose()                 include/ttutv/tt_decomp.hpp:100
 *                             and the seven named sweeps   include/ttutv/tt_decomp.hpp:69-97
 *   ttg_verify_bound       <- verify_bound()              include/ttutv/tt_decomp.hpp:105
 *   ttg_qr_col_pivot       <- qr_col_pivot()              include/ttutv/factor.hpp:19
 *   ttg_svd                <- svd()                       include/ttutv/factor.hpp:35
 *   ttg_utv                <- ulv() / urv()               include/ttutv/factor.hpp:56-57
 *   ttg_truncate           <- truncate_fixed_rank/tol()   include/ttutv/factor.hpp:73-82
 *   ttg_reconstruct        <- reconstruct()               include/ttutv/tt.hpp:60
 *   ttg_frobenius_norm     <- frobenius_norm()            include/ttutv/tensor_ops.hpp:26
 *   ttg_rse                <- rse()                       include/ttutv/tensor_ops.hpp:30
 *
 * Storage conventions are the reference's: matrices are column-major
 * ((i,j) -> data[i + j*rows], include/ttutv/matrix.hpp:36), tensors are flat with the
 * first index fastest (include/ttutv/dense_tensor.hpp:13-15), cores are
 * (r_{k-1}, I_k, r_k) tensors in the same order, perms are 0-based int64 source columns.
 *
 * Error convention: every call returns a ttg_status. Codes 1..6 correspond 1:1 to the
 * reference exception classes (include/ttutv/errors.hpp:10-54); the message is available
 * from ttg_last_error() on the calling thread. The C++ layer rethrows the matching class.
 *
 * Threading: calls are reentrant; each host thread gets its own CUDA stream on the
 * current device. ttg_decompose calls from several host threads take turns: host inputs
 * are uploaded one at a time and the decompositions hold the device one at a time (an
 * upload overlaps another caller's compute). Results are bitwise deterministic for a given
 * input and device.
 */
#ifndef TTUTV_B200_H
#define TTUTV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum ttg_status {
    TTG_OK = 0,
    TTG_ERR_ARGUMENT = 1,  /* ttutv::ArgumentError  */
    TTG_ERR_INDEX = 2,     /* ttutv::IndexError     */
    TTG_ERR_PARSE = 3,     /* ttutv::ParseError     */
    TTG_ERR_NUMERICAL = 4, /* ttutv::NumericalError */
    TTG_ERR_RESOURCE = 5,  /* ttutv::ResourceError  */
    TTG_ERR_INVARIANT = 6, /* ttutv::InvariantError */
    TTG_ERR_INTERNAL = 7,  /* any other ttutv::Error */
    TTG_ERR_CUDA = 8       /* CUDA runtime failure (no reference analogue; maps to Error) */
} ttg_status;

enum { TTG_METHOD_SVD = 0, TTG_METHOD_ULV = 1, TTG_METHOD_URV = 2 };
enum { TTG_SWEEP_L2R = 0, TTG_SWEEP_R2L = 1 };
enum { TTG_RETAIN_L11_ONLY = 0, TTG_RETAIN_FULL_COLUMN = 1 };
enum { TTG_BOUND_RSS = 0, TTG_BOUND_PLAIN_SUM = 1 };
/* QLP policy. EARLY_EXIT (default) stops each pivoted pass as soon as the kept block is
 * provably the one the full factorisation would produce;
 * FULL runs all p = min(m,n) steps of both passes exactly as the reference does;
 * BITWISE is FULL with cuts of at most 32 rows (of W) run bitwise like the reference's
 * qr_col_pivot in both passes (long sums as sequential chains): an ulp-decided rank (BASELINE
 * config 2 at eps 1e-8) is then the reference's. Much slower on those cuts (~0.1-0.3 s). */
enum { TTG_QLP_EARLY_EXIT = 0, TTG_QLP_FULL = 1, TTG_QLP_BITWISE = 2 };

/* Mirrors DecompConfig + FixedRank/FixedTol (tt_decomp.hpp:24-45). */
typedef struct ttg_config {
    int method;            /* TTG_METHOD_* */
    int sweep;             /* TTG_SWEEP_*  */
    int fixed_rank;        /* nonzero: ranks[0..d] used; zero: eps + weights */
    const int64_t* ranks;  /* rank chain (r_0..r_d) when fixed_rank */
    int nranks;            /* its length; validated against d+1 like FixedRank */
    double eps;            /* relative tolerance when !fixed_rank */
    const double* weights; /* may be NULL when nweights == 0 (equal split) */
    int nweights;
    int refine_passes;     /* default 1 */
    int retain;            /* TTG_RETAIN_*, right-to-left ULV only */
    int debug_checks;
    int qlp_policy;        /* TTG_QLP_* */
} ttg_config;

typedef struct ttg_result ttg_result; /* opaque; owns device and host buffers */

/* ---- library / device ------------------------------------------------------- */
const char* ttg_last_error(void);
int ttg_abi_version(void);
int ttg_device_count(void);
ttg_status ttg_set_device(int device);
/* Number of CUDA kernels this thread has launched (monotone counter; for bench/tests). */
int64_t ttg_kernel_launches(void);
ttg_status ttg_synchronize(void);
/* Grow this device's stream-ordered memory pool to hold at least `bytes` (allocate and
 * free once; the pool keeps freed memory), so later calls do not pay for pool growth. */
ttg_status ttg_reserve(int64_t bytes);
/* The calling thread's CUDA stream (cudaStream_t), on which every kernel of this thread
 * is launched; lets a harness record events on the same stream. */
void* ttg_stream(void);
/* Event timing of the dominant kernel (pass-1 streaming GEMV) for roofline reports:
 * enable, run, then read (host sync) the launch count, summed device time and summed
 * algorithmic bytes since the last read. */
ttg_status ttg_profile_enable(int on);
int64_t ttg_profile_read(double* total_ms, double* algorithmic_bytes);
/* Per-kernel totals of everything drained by ttg_profile_read since the last reset:
 * name (static string), summed device ms, algorithmic bytes and launches for each pass-1
 * stream kernel variant. Returns the number of kernels (<= max are written). */
int ttg_profile_kernels(int max, const char** names, double* ms, double* bytes, int64_t* launches);
void ttg_profile_reset_kernels(void);
/* Phase split of the persistent pass-1 loop (k_pass1_big<v>, v < 8), device time of CTA 0
 * in ms summed over steps since the last reset: out24[v*3 + 0] reflector, [+1] stream
 * (through the first grid barrier), [+2] guard (through the second). Host sync. */
ttg_status ttg_profile_big_phases(double* out24, int reset);

/* ---- files straight to and from the device --------------------------------------
 * The reference's binary containers (include/ttutv/io.hpp:10-19): TTUTVTEN dense tensors
 * and TTUTVCOR trains. Payloads stream through pinned chunks (the file read of one chunk
 * overlapping the H2D copy of the previous one), so a tensor file never has a host copy;
 * header checks, messages and offsets are read_tensor()'s (src/io.cpp:151-161).
 *   ttg_tensor_file_header    <- read_tensor() header      src/io.cpp:151-161 (host only)
 *   ttg_tensor_file_to_device <- read_tensor() payload
 *   ttg_decompose_file        <- read_tensor() + decompose()
 *   ttg_result_write_file     <- write_tt()                src/io.cpp:163-174
 * dims must hold 255 entries. On TTG_ERR_PARSE, ttg_last_error_offset() is the byte
 * offset the reference's ParseError carries. */
ttg_status ttg_tensor_file_header(const char* path, int* order, int64_t* dims);
ttg_status ttg_tensor_file_to_device(const char* path, double* dst, int64_t capacity);
int64_t ttg_last_error_offset(void);

/* ---- tensor-train sweeps ---------------------------------------------------- */
/* a: tensor of shape dims[0..d-1], first index fastest. a_on_device selects whether `a`
 * is a host pointer (copied in, timed in the report) or a device pointer (read in place).
 * Device inputs: the engine works on its own non-blocking per-thread stream (ttg_stream()); it
 * waits for the work already queued on the legacy default stream before reading `a`, but work
 * the caller queued on other streams must be complete (or ordered before ttg_stream()) first. */
ttg_status ttg_decompose(const double* a, const int64_t* dims, int d, const ttg_config* cfg,
                         int a_on_device, ttg_result** out);
/* ttg_decompose() on the tensor in a TTUTVTEN file, read straight to the device. */
ttg_status ttg_decompose_file(const char* path, const ttg_config* cfg, ttg_result** out);
void ttg_result_free(ttg_result* res);
/* The result's train as a TTUTVCOR file, byte-identical to the reference's write_tt(). */
ttg_status ttg_result_write_file(const ttg_result* res, const char* path);
int ttg_result_order(const ttg_result* res);
void ttg_result_core_dims(const ttg_result* res, int k, int64_t dims3[3]); /* k is 0-based */
ttg_status ttg_result_core_copy(const ttg_result* res, int k, double* host_out);
const double* ttg_result_core_device(const ttg_result* res, int k);
/* step_errors: d-1 (unfolding order); ranks_chosen: d+1; ranks_requested: d+1 or 0.
 * Returns the number of ranks_requested entries written (0 for tolerance mode). */
int ttg_result_report(const ttg_result* res, double* step_errors, int64_t* ranks_chosen,
                      int64_t* ranks_requested, double* bound, int* bound_kind,
                      double* input_norm, double* wall_time_ms);
int ttg_result_warning_count(const ttg_result* res);
const char* ttg_result_warning(const ttg_result* res, int i);
/* step_errors above are the reference's residual_from_mass, sqrt(max(0, kept[p] - kept[r]))
 * (src/factor.cpp:507-510), which cancels below ~1e-8 |A|_F (config 1 reports 0 like the
 * reference). This writes beside them, per cut in unfolding order, the discarded mass
 * computed directly (unseen pass-1 rows + discarded pass-2 columns, no subtraction), or -1
 * for cuts of the general path (refine != 1, TT-SVD, Alg. 4). Returns d-1. */
int ttg_result_direct_errors(const ttg_result* res, double* out);
/* The kept-mass vector the cut's rank rule used (fast path): kept[0..s] over the s pass-2
 * columns computed, in the reference's order (factor.cpp:479-499), then kept[p] (the total,
 * |R1[:s]|^2 + the exact trailing mass when s < p) as the last entry. Writes min(max, count)
 * entries and returns count (0 for general-path cuts). For margin logs of ulp-decided ranks
 * (kept[r] - target in ulps). */
int ttg_result_cut_kept(const ttg_result* res, int cut, double* kept, int max);
/* Per-cut diagnostics (cut = 0..d-2 in unfolding order):
 *   diag: |T_ii| of the kept block, i < r (the "per-unfolding diagonal estimates"),
 *   info[0] pivoted steps run in pass 1, info[1] p = min(m,n), info[2] rank kept,
 *   info[3] early-exit extensions, info[4..5] m, n of the cut matrix.
 * Returns the number of diag entries written (<= max). */
int ttg_result_cut_diag(const ttg_result* res, int cut, double* diag, int max, int64_t info[6]);

/* achieved = |A - reconstruct(tt)|_F computed on device (reconstruct fused with the
 * difference norm). Throws (returns) TTG_ERR_INVARIANT when achieved exceeds
 * bound + slack_rel * |A|_F, like verify_bound (tt_decomp.cpp:445-462). */
ttg_status ttg_verify_bound(const double* a, int a_on_device, const ttg_result* res,
                            double slack_rel, double* achieved);
/* |A - reconstruct(tt)|_F / |A|_F on device (no element cap: Â is never materialised). */
ttg_status ttg_result_rse(const ttg_result* res, const double* a, int a_on_device, double* rse);
/* Dense reconstruction of the result's train into `out` (device pointer when
 * out_on_device, else host), reconstruct() (tt.cpp:52-73) without an element cap. */
ttg_status ttg_result_reconstruct(const ttg_result* res, double* out, int out_on_device);

/* One completion step on device buffers of n entries (the reference's loop body,
 * completion.cpp:161-186, with a step size of 1): y holds the reconstruction X on entry;
 * on exit y = observed on the mask (mask != 0) and X elsewhere. Also returns
 *   stats[0] = sum_mask (X - observed)^2     stats[1] = sum_mask observed^2
 *   stats[2] = sum (X - truth)^2             stats[3] = sum truth^2
 *   stats[4] = max truth                     (truth may be NULL: stats[2..4] = 0)
 * with deterministic fixed-order reductions. */
ttg_status ttg_completion_reset(double* y, const double* observed, const double* mask,
                                const double* truth, int64_t n, double stats[5]);

/* complete() / initial_guess() (include/ttutv/completion.hpp:73-81, completion.cpp:121-211) on
 * the device: X_0 = Retract(P_Omega(M)), X_i = Retract(X_{i-1} + step_size P_Omega(M - X_{i-1})),
 * with the reference's trace, 20-iteration divergence run and 5-iteration stop window. The
 * fields mirror CompletionConfig (completion.hpp:40-55); extension: nranks == 0 with eps > 0
 * retracts at the prescribed accuracy eps (rank-adaptive, equal rss weights), the retraction
 * config 4 of BASELINE.json needs. `linear` holds the observations' 0-based linear indices
 * (strictly increasing, like ObservationMask), `values` their values; with on_device the
 * pointers (linear, values, truth) are device memory. truth may be NULL. */
typedef struct ttg_completion_config {
    const int64_t* ranks; /* target chain (r_0..r_d), or NULL with nranks = 0 (rank-adaptive) */
    int nranks;
    double eps;           /* rank-adaptive retraction tolerance (nranks == 0) */
    int retraction;       /* TTG_METHOD_*; URV sweeps right to left, the others left to right */
    double step_size;     /* default 1 */
    int max_iters;        /* default 500 */
    double stop_tol;      /* default 1e-6; 0 disables */
    int refine_passes;    /* default 2 */
    int64_t dense_cap;    /* default 1e7 */
} ttg_completion_config;
typedef struct ttg_completion ttg_completion; /* opaque */
ttg_status ttg_complete(const int64_t* linear, const double* values, int64_t count, const int64_t* dims, int d,
                        const ttg_completion_config* cfg, const double* truth, int on_device,
                        ttg_completion** out);
void ttg_completion_free(ttg_completion* c);
int ttg_completion_iterations(const ttg_completion* c);
int ttg_completion_status(const ttg_completion* c); /* 0 converged, 1 max_iters, 2 diverged */
const char* ttg_completion_note(const ttg_completion* c);
/* per iteration 1..n: observed RSE, full RSE and PSNR (only with truth: else untouched),
 * cumulative wall ms; initial3 (nullable) = the initial guess's observed RSE, full RSE, PSNR */
void ttg_completion_trace(const ttg_completion* c, double* rse_observed, double* rse_full, double* psnr,
                          double* wall_time_ms, double* initial3);
/* rank chain (d+1 entries) of iterate `iter` (0 = the initial guess); returns d+1 or 0 */
int ttg_completion_ranks(const ttg_completion* c, int iter, int64_t* ranks);
/* the final iterate's train (owned by the completion handle) */
const ttg_result* ttg_completion_result(const ttg_completion* c);

/* ---- multi-GPU: column-sharded sweeps (no reference analogue) --------
 * One process (or host thread) per GPU. A communicator is an NCCL communicator over the
 * ranks (NVLink / NVSwitch inside a B200 box), or a loopback group whose endpoints are
 * host threads of one process sharing one GPU (tests). The reference is single-process;
 * these entry points extend ttg_decompose and return the same ttg_result, with the cores
 * replicated on every rank. */
typedef struct ttg_comm ttg_comm; /* opaque */
/* 128-byte NCCL unique id: create on one rank, hand to every rank (any side channel). */
ttg_status ttg_comm_nccl_unique_id(unsigned char id[128]);
ttg_status ttg_comm_nccl_create(const unsigned char id[128], int nranks, int rank, ttg_comm** out);
/* nranks endpoints in `out[0..nranks-1]`; endpoint g must be driven by its own host thread. */
ttg_status ttg_comm_loopback_create(int nranks, ttg_comm** out);
/* A communicator over a host transport the caller provides (gloo, MPI, sockets): fn must
 * all-gather `bytes` from every rank into recv (nranks * bytes, rank order) and return 0. The
 * engine stages the exchanged buffers through pinned host memory. */
typedef int (*ttg_host_allgather)(const void* send, void* recv, size_t bytes, void* user);
ttg_status ttg_comm_callback_create(int nranks, int rank, ttg_host_allgather fn, void* user, ttg_comm** out);
void ttg_comm_free(ttg_comm* comm);
/* The block of the first unfolding a rank owns: out = {lo, hi, rows, cols}. ULV (l2r):
 * columns [lo, hi) of c = A(i1; i2..id), a contiguous slice of A, rows x cols = I1 x (hi-lo).
 * URV (r2l): rows [lo, hi) of c = A(i1..i(d-1); id), a (hi-lo) x Id column-major block. */
ttg_status ttg_shard_range(const int64_t* dims, int d, int method, int nranks, int rank, int64_t out[4]);
/* ttg_decompose over the ranks of `comm`: a_local is this rank's block (ttg_shard_range).
 * Pass 1 of the first cut runs column-sharded (one all-gather of a pivot record per step),
 * its pass 2 reduces the ranks' TSQR triangles, and the carry is all-gathered once; the
 * remaining cuts run replicated. ULV-L2R and URV-R2L with refine_passes = 1. */
ttg_status ttg_decompose_sharded(const double* a_local, const int64_t* dims, int d, const ttg_config* cfg,
                                 int a_on_device, ttg_comm* comm, ttg_result** out);

/* ---- factor level (host buffers, column-major) ------------------------------ */
/* q: m x p, r: p x n, perm: n. Any of the outputs may be NULL. */
ttg_status ttg_qr_col_pivot(const double* a, int64_t m, int64_t n, double* q, double* r,
                            int64_t* perm);
/* lower != 0: ULV (t lower-triangular), else URV. u: m x p, t: p x p, v: n x p. */
ttg_status ttg_utv(const double* a, int64_t m, int64_t n, int lower, int refine_passes,
                   double* u, double* t, double* v);
/* Economy SVD (one-sided Jacobi on the p x p triangle of a pivoted QR). u: m x p, s: p,
 * v: n x p. max_sweeps / pair_tol as SvdOptions (factor.hpp:30-33). */
ttg_status ttg_svd(const double* a, int64_t m, int64_t n, int max_sweeps, double pair_tol,
                   double* u, double* s, double* v);
/* kind: 0 svd (t is diag(s) given as the p-vector s), 1 ulv, 2 urv.
 * rank > 0: fixed rank; rank == 0: tolerance eps. Outputs u1 m x r, t11 r x r, v1 n x r
 * (caller sizes them for r = p). */
ttg_status ttg_truncate(int kind, const double* u, const double* t, const double* v, int64_t m,
                        int64_t n, int64_t p, int64_t rank, double eps, int64_t* rank_out,
                        double* residual, double* u1, double* t11, double* v1);

/* ---- tensor ops ------------------------------------------------------------- */
/* cores: concatenated (r_{k-1}, I_k, r_k) blocks; ranks: d+1; dims: d. out: prod(dims). */
ttg_status ttg_reconstruct(const double* cores, const int64_t* dims, const int64_t* ranks, int d,
                           int64_t element_cap, double* out);
ttg_status ttg_frobenius_norm(const double* a, int64_t count, int a_on_device, double* out);
/* kernels::sum_squares (kernels.cpp:84-102): the 4096-blocked sum of squares, no sqrt */
ttg_status ttg_sum_squares(const double* a, int64_t count, int a_on_device, double* out);
ttg_status ttg_rse(const double* estimate, const double* truth, int64_t count, double* out);
/* |x - y|_2 over count entries (verify_bound's achieved error, tt_decomp.cpp:449-454). */
ttg_status ttg_diff_norm(const double* x, const double* y, int64_t count, double* out);
/* C = op(A) op(B) on the device (DMMA tiles), host buffers, column-major; op = transpose
 * when ta/tb is nonzero (kernels::matmul, include/ttutv/kernels.hpp:21). */
/* Tensor algebra (host buffers in and out, computed on the device):
 *   mode_product  tensor_ops.cpp:49-80: out = tensor x_k mat (mat is m_rows x m_cols, m_cols
 *                 must equal dims[k-1]; k is 1-based); bitwise the reference's (same sums)
 *   kron          tensor_ops.cpp:82-93 (column-major (ar br) x (ac bc)); bitwise
 *   psnr          tensor_ops.cpp:113-126: 10 log10(max(truth)^2 / mse), +inf when mse == 0
 *   reverse_indices  tensor_ops.cpp:128-143: out has dims reversed, out(i_d..i_1) = a(i_1..i_d)
 *   reverse_tt    tt.cpp:108-123: cores (packed back to back, core k = ranks[k] x dims[k] x
 *                 ranks[k+1]) of the reversed train, packed in the new core order */
ttg_status ttg_mode_product(const double* x, const int64_t* dims, int d, int k, const double* m,
                            int64_t m_rows, int64_t m_cols, double* out);
ttg_status ttg_kron(const double* a, int64_t ar, int64_t ac, const double* b, int64_t br, int64_t bc,
                    double* out);
ttg_status ttg_psnr(const double* estimate, const double* truth, int64_t count, double* out);
ttg_status ttg_reverse_indices(const double* a, const int64_t* dims, int d, double* out);
ttg_status ttg_reverse_tt(const double* cores, const int64_t* dims, const int64_t* ranks, int d,
                          double* out);
/* C = alpha op(A) op(B) + beta C on DEVICE buffers, column-major, on this thread's stream
 * (ttg_stream()), no synchronisation: the engine's FP64 tensor-core (DMMA) GEMM -- a 128 x 128
 * cp.async-pipelined kernel for aligned operands with even leading dimensions, split over K for
 * long reductions with a deterministic combine. The dense kernel of the carry/Gram/reconstruct
 * contractions, exported for measurement and for callers that keep data on the device. */
ttg_status ttg_gemm_device(int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha, const double* A,
                           int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc);
ttg_status ttg_matmul(const double* a, int64_t a_rows, int64_t a_cols, int ta, const double* b,
                      int64_t b_rows, int64_t b_cols, int tb, double* c);

#ifdef __cplusplus
}
#endif
#endif /* TTUTV_B200_H */
