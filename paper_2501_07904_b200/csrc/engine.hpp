// Host-side engine interfaces (internal; the public boundary is include/ttutv_b200.h).
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"

namespace ttg {

// Storage of the k x N matrix W whose columns are pivoted in pass 1.
//   Col: W(i,j) = W[i + j*ld]  (the unfolding c itself, ULV / left-to-right)
//   Row: W(i,j) = W[i*ld + j]  (c^T read in place from a column-major c, URV / right-to-left)
enum class Layout { Col = 0, Row = 1 };

// ---------------------------------------------------------------------------
// Multi-GPU plumbing (comm.cu). One rank per GPU; every exchange on the data path is an
// all-gather of a small device buffer, ordered on the calling thread's stream, followed
// by a fixed-order combine, so every rank derives bitwise identical decisions.
// ---------------------------------------------------------------------------
class Comm {
public:
    virtual ~Comm() = default;
    virtual int rank() const = 0;
    virtual int size() const = 0;
    // recv (device, size() * bytes) <- every rank's send (device, bytes), in rank order.
    virtual void allgather(const void* send, void* recv, size_t bytes) = 0;
    // Point-to-point round (every rank calls it): send `bytes` to rank `to` and receive `bytes`
    // from rank `from`; -1 skips either side. Only when has_p2p().
    virtual bool has_p2p() const { return false; }
    virtual void sendrecv(const void* send, int to, void* recv, int from, size_t bytes) {
        (void)send; (void)to; (void)recv; (void)from; (void)bytes;
        fail(8, "this communicator has no point-to-point transport");
    }
};
// Sum of one double per rank, combined in rank order (host result, identical everywhere).
double global_sum(Comm& comm, double local);
std::unique_ptr<Comm> make_nccl_comm(const unsigned char id[128], int nranks, int rank);
void nccl_unique_id(unsigned char id[128]);
// In-process group of `nranks` endpoints for one GPU, one host thread per endpoint (tests):
// the exchange is a host barrier around device copies, no kernel ever waits on another.
std::vector<std::unique_ptr<Comm>> make_loopback_group(int nranks);
// A communicator whose all-gather is a host callback: recv (size() * bytes, rank order) <-
// every rank's send (bytes); returns 0 on success.
typedef int (*ttg_host_allgather_fn)(const void* send, void* recv, size_t bytes, void* user);
std::unique_ptr<Comm> make_callback_comm(int nranks, int rank, ttg_host_allgather_fn fn, void* user);

// Column sharding of pass 1: this engine holds columns [col_off, col_off + N) of a
// k x N_global matrix whose other columns live on the other ranks of `comm`.
struct ShardSpec {
    Comm* comm = nullptr;
    int64_t col_off = 0;
    int64_t N_global = 0;
};

// ---------------------------------------------------------------------------
// Pass 1: greedy column-pivoted Householder QR of a k x N matrix W. W is never written.
// The orthogonal factor Q_t = H_0...H_{t-1} is kept in compact WY form
// Q_t = I - Y_t T_t Y_t^T (Y: k x t reflectors, T: t x t upper), so one step costs
// O(k t) besides one streaming GEMV over W: R(t,j) = q_t^T w_j for every unpivoted
// column, with the norm downdate of factor.cpp:98-107. Any prefix of steps equals the
// prefix of the reference's qr_col_pivot (factor.cpp:62-135) in exact arithmetic: same
// pivots (same tie rule), same R rows, and Q[:, :s] = its first s economy-Q columns.
//
// Sharded (ShardSpec): positions are global; every step each rank exports its best local
// candidate with its column, the records are all-gathered, and every rank picks the same
// winner (norm desc, global position asc) and builds the same reflector from the winner's
// column, then streams its own columns. Q and the reflectors are replicated; R rows and
// norms stay local.
// ---------------------------------------------------------------------------
struct LzArgs;

class WideQrcp {
public:
    // subspace: allow the subspace (lazy-exact) stream (fixed-rank cuts; see qrcp_wide.cu)
    WideQrcp(const double* W, int64_t k, int64_t N, int64_t ld, Layout layout, int64_t cap_steps,
             const ShardSpec* shard = nullptr, bool subspace = false);
    void run_to(int64_t steps);  // advance the greedy factorisation to `steps` (<= p)
    int64_t steps() const { return steps_; }
    int64_t p() const { return p_; }
    int64_t k() const { return k_; }
    int64_t N() const { return N_; }  // local columns
    bool sharded() const { return comm_ != nullptr; }
    Comm* comm() const { return comm_; }
    // Trailing mass sum_j nu_j of the not-yet-pivoted columns from the downdated norms
    // (host sync). Below ~1e-16 of a column's norm the downdates are rounding noise.
    double trailing_mass();
    // Recomputes every unpivoted norm exactly from the projection residual
    // |w_j - Q[:, :s] R(0:s, j)|^2 (one GEMM over W; also resets cref like the guard) and
    // returns the exact trailing mass.
    double refresh_exact();

    const double* Q() const { return explicit_ ? Qx_.get() : Qt_.get(); }  // columns 0..steps-1 = economy Q
    const double* R() const { return R_.get(); }       // rows 0..steps-1, row t at R + t*N
    const int64_t* perm() const { return perm_.get(); } // position -> column (global when sharded)
    const int64_t* piv() const { return piv_.get(); }   // step -> local column (-1: other rank)
    const double* diag() const { return diag_.get(); }  // R(t,t)
    int64_t R_stride() const { return N_; }

private:
    void grow(int64_t cap);
    void step();
    void reflect_step(int64_t t);
    void explicit_step(int64_t t);
    void to_explicit(int64_t t);
    void gemv_step(int64_t t);
    void guard_step(int64_t t);
    void sub_step(int64_t t);
    double* qptr() { return explicit_ ? Qx_.get() : Qt_.get(); }

    const double* W_;
    int64_t k_, N_, ld_, p_;
    Layout layout_;
    int64_t steps_ = 0, cap_ = 0;
    int ncand_ = 0, ngc_ = 0, mode_ = 0, nchunk_ = 1, ksplit_ = 1;  // stream / guard candidate slots
    Comm* comm_ = nullptr;
    int64_t off_ = 0, Ng_ = 0;
    DevBuf<double> nu_, cref_, R_, diag_, beta_, mass_;
    DevBuf<double> Y_, T_, Qt_, wv_, yv_, part_, vecs_, kpart_;  // WY state and scratch
    DevBuf<double> rec_, recs_;  // sharded: this rank's pivot record, all ranks' records
    bool explicit_ = false;      // explicit k x k Q (long factorisations)
    DevBuf<double> Qx_, exz_;
    DevBuf<double> Wt_;  // row-layout copy of a narrow Col W for k_pass1_big<5>
    bool big_ = false;           // ... with the large-W stream variants (k_pass1_big)
    bool coop_ = false;          // persistent cooperative step loop (small / medium W)
    // subspace (lazy-exact) pivoting: R rows from Z = E^T W while q_t stays in span(E)
    bool sub_ = false;
    int subc_ = 8;  // predicted directions (basis size cap)
    bool coop_ok_ = false, big_ok_ = false;  // the persistent loop, for after a subspace fallback
    int ncand_coop_ = 0, sms_ = 0;
    int sub_hits();
    DevBuf<double> E_, a_, Z_;
    DevBuf<int> subi_;  // [0] basis size nE, [1] hit flag of the current step
    DevBuf<int> nflag2_;
    bool coop_run(int64_t steps);
    DevBuf<int64_t> pos_, perm_, piv_, flags_;
    DevBuf<Cand> cand_;
    DevBuf<int> nflag_;
    // candidate (lazy-exact) pivoting for narrow W (qrcp_wide.cu, k_lz_*)
    bool lz_ = false, lzw_ = false;  // narrow (k <= 32) / wide (k <= 512) variant
    int lz_nubest() const;
    int64_t lz_buf() const;
    static int lz_tails();
    int64_t lz_run_first_ = 0;  // first step of the current run (its first choice is a launch of its own)
    int64_t lz_host_exact_ = 0;  // step of the last exact pass the host knows of (forced passes)
    DevBuf<int64_t> lzst_, lzidx_, lzposc_;
    DevBuf<Cand> lzubest_;
    DevBuf<double> lzsd_, lzwc_, lznuc_, lzcrefc_;
    DevBuf<int> lzhist_;
    LzArgs lz_args();
    void lz_step(int64_t t);
    void lz_refresh(int64_t t1, bool force);
};

// ---------------------------------------------------------------------------
// Bitwise pass 1 for narrow W (k <= 32): the reference's qr_col_pivot operation for operation
// on a row-major working copy (qrcp_exact.cu), for tolerance-mode cuts whose rank the rounding
// of pass 1 decides (BASELINE config 2).
// ---------------------------------------------------------------------------
class ExactQrcp {
public:
    ExactQrcp(const double* W, int64_t k, int64_t N, int64_t ld, Layout layout);
    void run_to(int64_t s);
    int64_t steps() const { return steps_; }
    int64_t p() const { return p_; }
    double trailing_mass_exact();
    void r_rows(double* R, int64_t s) const;  // rows 0..s-1 by original column, row t at R + t N
    void form_q(double* Q, int64_t s) const;  // economy Q columns 0..s-1, k x s
    const int64_t* perm() const { return perm_.get(); }
    const double* diag() const { return diag_.get(); }

private:
    int64_t k_, N_, p_, steps_ = 0;
    int grid_ = 1;
    DevBuf<double> work_, cn_, cr_, betas_, diag_, cand_, step_;
    DevBuf<int64_t> pos_, perm_;
};

// Bitwise qr_col_pivot of a tall N x s work matrix (s <= 32, column-major, overwritten): R over
// positions (s x s, ld s), the permutation (position -> column) and each pivot's norm^2 at its
// step. Its long sums are sequential chains (one warp each), as in the reference.
void exact_tall_qrcp(double* work, int64_t N, int64_t s, double* R, int64_t* perm, double* pnorm);

// ---------------------------------------------------------------------------
// Pass 2 (and any tall QRCP): in-place Householder QR with column pivoting of an
// N x n column-major matrix B with n moderate, mirroring factor.cpp:62-135 step by step
// (pivot, dlarfg reflector, reflector application, norm downdate with the 1e-16
// recompute guard). Reduction over the long dimension is split across CTAs with a
// fixed-order combine, so results are deterministic.
// ---------------------------------------------------------------------------
class TallQrcp {
public:
    TallQrcp(double* B, int64_t N, int64_t n, int64_t ld);
    void run(int64_t steps);     // steps <= min(N, n)
    int64_t steps() const { return steps_; }
    // R over final positions (steps x n, col-major, ldo >= steps): R(t,q) for q >= t, 0 below.
    void extract_r(double* out, int64_t ldo) const;
    const int64_t* perm() const { return colmap_.get(); } // position -> physical column
    const double* pivot_norm2() const { return pnorm_.get(); } // nu of the pivot at its step
    const double* beta() const { return beta_.get(); }
    // Explicit economy Q columns 0..q-1 (N x q, col-major, ldq >= N).
    void form_q(double* Qout, int64_t q, int64_t ldq);
    // Rows 0..steps-1 of R indexed by ORIGINAL column (row t at out + t*ldo), the layout
    // the wide engine produces; exact zeros below the diagonal.
    void r_rows_by_column(double* out, int64_t ldo) const;
    // Trailing mass of the not-yet-pivoted columns, exactly: the sum of squares of rows
    // steps.. of the in-place updated columns (host sync).
    double trailing_mass_exact() const;
    int64_t p() const { return p_; }
    int64_t N() const { return N_; }
    int64_t n() const { return n_; }

private:
    double* B_;
    int64_t N_, n_, ld_, p_;
    int64_t steps_ = 0;
    int nblk_ = 0;
    int64_t rows_per_blk_ = 0;
    bool col_mode_ = false;  // one CTA per trailing column per step (N <= 25600)
    bool run_persist(int64_t steps);
    DevBuf<double> nu_, cref_, R_, part_, tq_, beta_, v0_, pnorm_;
    DevBuf<double> Vp_, F_;  // persistent blocked engine (panel state)
    DevBuf<int64_t> colmap_, pos_;
    DevBuf<int> flag_;
};

// ---------------------------------------------------------------------------
// TSQR and small pivoted QR (tsqr.cu)
// ---------------------------------------------------------------------------
// R factor (s x s, upper, col-major ld = s) of the N x s matrix B (column t at B + t*ld),
// by a Householder TSQR tree in shared memory (one HBM pass over B). Requires tsqr_fits(s).
bool tsqr_fits(int64_t s);
// Upper Cholesky factor R (G = R^T R) of an s x s Gram matrix, one CTA (s^2 doubles of
// shared memory). Returns false (R unusable) unless G is numerically positive definite
// with min R_ii >= min_ratio * max R_ii (host sync).
bool cholesky_r(const double* G, int64_t s, double min_ratio, double* R);
void tsqr_r(const double* B, int64_t N, int64_t s, int64_t ld, double* Rout);
// One-CTA qr_col_pivot of a matrix that fits in shared memory (small_qrcp_fits): the
// reference algorithm step for step. perm[n], R (p x n over positions, ld = p), pnorm[p]
// (norm^2 of each pivot when chosen), Q (m x p, optional).
bool small_qrcp_fits(int64_t m, int64_t n);
void small_qrcp(const double* A, int64_t m, int64_t n, int64_t lda, int64_t* perm, double* R, double* pnorm,
                double* Q);

// ---------------------------------------------------------------------------
// Dense helpers on device buffers (column-major).
// ---------------------------------------------------------------------------
// C(m x n) = op(A) * op(B) with FP64 tensor-core (DMMA) tiles.
void gemm(bool ta, bool tb, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda,
          const double* B, int64_t ldb, double* C, int64_t ldc, double alpha = 1.0,
          double beta = 0.0);
void transpose(const double* A, int64_t m, int64_t n, int64_t lda, double* B, int64_t ldb);
// C (n x n) = op(A) op(A)^T with op(A) = A^T (ta, A k x n) or A (A n x k): symmetric tiles only
// on the DMMA kernel, the lower triangle mirrored.
void syrk(bool ta, int64_t n, int64_t k, const double* A, int64_t lda, double* C, int64_t ldc);
// G (s x s, ld s) = B^T B for a tall N x s block, s <= 32, on the DMMA tensor cores.
void gram_small(const double* B, int64_t N, int64_t s, int64_t ld, double* G);
// Deterministic sum of squares of a contiguous buffer (fixed 4096-element blocks combined
// in block order, the reference's blocking, kernels.cpp:84-102).
double sum_squares(const double* x, int64_t n);
// sum_i (x_i - y_i)^2 with the same blocking.
double diff_squares(const double* x, const double* y, int64_t n);

}  // namespace ttg
