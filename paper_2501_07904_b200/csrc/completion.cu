// Tensor completion on the device (completion.hpp / completion.cpp, BASELINE config 4):
//   X_0 = Retract(P_Omega(M))                                  initial_guess  (:121-129)
//   X_i = Retract(X_{i-1} + alpha P_Omega(M - X_{i-1}))        complete       (:161-170)
// with the trace of completion.cpp:172-207 (observed RSE, full RSE and PSNR against a ground
// truth, the 20-step divergence run and the 5-iteration stop window). The retraction is the
// device sweep (fixed rank like the reference, or -- the extension config 4 needs --
// rank-adaptive at a prescribed accuracy), the iterate is reconstructed on the device, and
// the dense iterate, observations and truth stay in HBM for the whole loop.
#include <chrono>
#include <cmath>
#include <string>

#include "completion.hpp"

namespace ttg {
namespace {

constexpr int kStopWindow = 5;   // completion.cpp:21
constexpr int kDivergeRun = 20;  // completion.cpp:22
constexpr int64_t kChunk = 4096;

// dense observation tensors from the mask's (0-based, increasing) linear indices
__global__ void k_scatter_obs(const int64_t* __restrict__ idx, const double* __restrict__ vals, int64_t count,
                              double* dvals, double* dmask) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        dvals[idx[i]] = vals[i];
        dmask[idx[i]] = 1.0;
    }
}

// stepped = x + alpha (v - x) on the observed entries, x elsewhere (completion.cpp:163-167:
// the product rounded, then the sum)
__global__ void k_comp_step(const double* __restrict__ x, const double* __restrict__ v,
                            const double* __restrict__ mask, double alpha, int64_t n, double* out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double xi = x[i];
        out[i] = mask[i] != 0.0 ? __dadd_rn(xi, __dmul_rn(alpha, __dsub_rn(v[i], xi))) : xi;
    }
}

// per 4096-entry chunk: observed error^2, full error^2, truth^2, max truth (chunks combined in
// order on the host: deterministic)
__global__ void __launch_bounds__(256) k_comp_stats(const double* __restrict__ x, const double* __restrict__ v,
                                                    const double* __restrict__ mask,
                                                    const double* __restrict__ truth, int64_t n, double* part) {
    __shared__ double sd[8];
    __shared__ double smx[8];
    const int64_t nchunk = cdiv(n, kChunk);
    for (int64_t b = blockIdx.x; b < nchunk; b += gridDim.x) {
        const int64_t lo = b * kChunk, hi = min(n, lo + kChunk);
        double so = 0.0, sf = 0.0, st = 0.0, mx = -INFINITY;
        for (int64_t i = lo + threadIdx.x; i < hi; i += 256) {
            const double xi = x[i];
            if (mask[i] != 0.0) {
                const double d = xi - v[i];
                so = fma(d, d, so);
            }
            if (truth) {
                const double d = xi - truth[i];
                sf = fma(d, d, sf);
                st = fma(truth[i], truth[i], st);
                mx = fmax(mx, truth[i]);
            }
        }
        so = block_sum(so, sd);
        sf = block_sum(sf, sd);
        st = block_sum(st, sd);
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        __syncthreads();
        if ((threadIdx.x & 31) == 0) smx[threadIdx.x >> 5] = mx;
        __syncthreads();
        if (threadIdx.x == 0) {
            double m = smx[0];
            for (int w = 1; w < 8; ++w) m = fmax(m, smx[w]);
            part[4 * b + 0] = so;
            part[4 * b + 1] = sf;
            part[4 * b + 2] = st;
            part[4 * b + 3] = m;
        }
    }
}

struct Stats {
    double obs_err2 = 0.0, full_err2 = 0.0, truth2 = 0.0, max_truth = -INFINITY;
};

Stats stats_of(const double* x, const double* v, const double* mask, const double* truth, int64_t n) {
    const int64_t nchunk = cdiv(n, kChunk);
    DevBuf<double> part((size_t)(4 * nchunk));
    const int grid = (int)std::min<int64_t>(nchunk, (int64_t)sm_count() * 8);
    TTG_LAUNCH(k_comp_stats, grid, 256, 0, stream(), x, v, mask, truth, n, part.get());
    const std::vector<double> h = part.to_host((size_t)(4 * nchunk));
    Stats s;
    for (int64_t b = 0; b < nchunk; ++b) {
        s.obs_err2 += h[(size_t)(4 * b)];
        s.full_err2 += h[(size_t)(4 * b + 1)];
        s.truth2 += h[(size_t)(4 * b + 2)];
        s.max_truth = std::max(s.max_truth, h[(size_t)(4 * b + 3)]);
    }
    return s;
}

int grid_of(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), (int64_t)sm_count() * 16)); }

}  // namespace

CompletionRun complete(const int64_t* idx, const double* vals, int64_t count, const std::vector<int64_t>& dims,
                       const CompletionSpec& spec, const double* truth) {
    using Clock = std::chrono::steady_clock;
    const auto start = Clock::now();
    const int64_t d = (int64_t)dims.size();
    int64_t n = 1;
    for (int64_t v : dims) n *= v;
    if (count < 1) argument_error("observation set is empty");
    if (n > spec.dense_cap)
        resource_error("completion would materialize " + std::to_string(n) + " elements (cap " +
                       std::to_string(spec.dense_cap) + ")");
    if (!spec.adaptive && (int64_t)spec.ranks.size() != d + 1)
        argument_error("rank chain has " + std::to_string(spec.ranks.size()) + " entries, expected " +
                       std::to_string(d + 1));
    if (spec.adaptive && !(spec.eps > 0.0)) argument_error("tolerance must be >= 0");
    if (spec.step_size < 0.0) argument_error("step size must be >= 0");
    if (spec.max_iters < 1) argument_error("max_iters must be >= 1");
    if (spec.stop_tol < 0.0) argument_error("stop_tol must be >= 0");

    // expected chain after clamping against the unfolding sizes (completion.cpp:144-151)
    std::vector<int64_t> expected = spec.ranks;
    if (!spec.adaptive) {
        int64_t left = 1;
        for (int64_t k = 1; k < d; ++k) {
            left *= dims[(size_t)(k - 1)];
            expected[(size_t)k] = std::min(expected[(size_t)k], std::min(left, n / left));
        }
    }
    SweepConfig sc;
    sc.method = spec.retraction;
    sc.sweep = spec.retraction == 2 ? 1 : 0;  // URV right to left, the others left to right (:92-104)
    sc.fixed_rank = !spec.adaptive;
    sc.ranks = spec.ranks;
    sc.eps = spec.eps;
    sc.refine = spec.refine_passes;

    DevBuf<double> v((size_t)n), mask((size_t)n), x((size_t)n), stepped((size_t)n);
    v.zero();
    mask.zero();
    TTG_LAUNCH(k_scatter_obs, grid_of(count), 256, 0, stream(), idx, vals, count, v.get(), mask.get());
    const double obs_norm = std::sqrt(sum_squares(v.get(), n));  // values_norm (completion.cpp:62-64)

    CompletionRun run;
    auto retract = [&](const double* y) {
        TTResult r = decompose(y, dims, sc);
        std::vector<const double*> cores;
        std::vector<int64_t> ranks{1};
        for (size_t k = 0; k < r.cores.size(); ++k) {
            cores.push_back(r.cores[k].get());
            ranks.push_back(r.core_dims[k][2]);
        }
        reconstruct(cores, dims, ranks, x.get());
        if (!spec.adaptive && r.ranks_chosen != expected) {
            // ranks may collapse only when the iterate is exactly zero (completion.cpp:107-117)
            if (sum_squares(x.get(), n) != 0.0) {
                std::string got, want;
                for (size_t i = 0; i < r.ranks_chosen.size(); ++i) {
                    got += (i ? "," : "") + std::to_string(r.ranks_chosen[i]);
                    want += (i ? "," : "") + std::to_string(expected[i]);
                }
                invariant_error("iterate left the fixed-rank set: ranks (" + got + ") vs expected (" + want + ")");
            }
        }
        run.ranks.push_back(r.ranks_chosen);
        return r;
    };
    auto record = [&](std::vector<double>& obs, std::vector<double>& full, std::vector<double>& ps) {
        const Stats s = stats_of(x.get(), v.get(), mask.get(), truth, n);
        obs.push_back(obs_norm > 0.0 ? std::sqrt(s.obs_err2) / obs_norm : std::sqrt(s.obs_err2));
        if (truth) {
            if (s.truth2 == 0.0) argument_error("rse: truth has zero norm (domain error)");
            full.push_back(std::sqrt(s.full_err2) / std::sqrt(s.truth2));
            const double mse = s.full_err2 / (double)n;
            ps.push_back(mse == 0.0 ? INFINITY : 10.0 * std::log10(s.max_truth * s.max_truth / mse));
        }
    };

    // initial guess: retraction of the observations embedded in zeros
    run.tt = retract(v.get());
    record(run.initial_obs, run.initial_full, run.initial_psnr);

    int rising = 0;
    for (int iter = 1; iter <= spec.max_iters; ++iter) {
        TTG_LAUNCH(k_comp_step, grid_of(n), 256, 0, stream(), x.get(), v.get(), mask.get(), spec.step_size, n,
                   stepped.get());
        run.tt = retract(stepped.get());
        record(run.rse_observed, run.rse_full, run.psnr);
        run.wall_ms.push_back(std::chrono::duration<double, std::milli>(Clock::now() - start).count());
        const size_t t = run.rse_observed.size();
        if (t >= 2 && run.rse_observed[t - 1] > run.rse_observed[t - 2]) {
            if (++rising >= kDivergeRun) {
                run.status = 2;
                run.note = "observed error rose for " + std::to_string(kDivergeRun) +
                           " consecutive iterations (iteration " + std::to_string(iter) + ")";
                break;
            }
        } else {
            rising = 0;
        }
        if (spec.stop_tol > 0.0 && t >= (size_t)kStopWindow + 1) {
            const double prev = run.rse_observed[t - 1 - kStopWindow];
            const double change = std::abs(run.rse_observed[t - 1] - prev);
            if (change < spec.stop_tol * std::max(prev, 1e-300)) {
                run.status = 0;
                break;
            }
        }
    }
    sync();
    return run;
}

}  // namespace ttg
