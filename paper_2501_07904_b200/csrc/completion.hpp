// Device tensor completion (completion.hpp:40-81 of the reference, plus a rank-adaptive
// retraction). Internal; the public boundary is ttg_complete in include/ttutv_b200.h.
#pragma once

#include <string>
#include <vector>

#include "sweep.hpp"

namespace ttg {

struct CompletionSpec {
    std::vector<int64_t> ranks;  // fixed-rank chain (r_0..r_d) unless adaptive
    bool adaptive = false;       // extension: retraction at a prescribed accuracy eps
    double eps = 0.0;
    int retraction = 0;          // 0 svd, 1 ulv, 2 urv
    double step_size = 1.0;
    int max_iters = 500;
    double stop_tol = 1e-6;
    int refine_passes = 2;
    int64_t dense_cap = 10'000'000;
};

struct CompletionRun {
    TTResult tt;                                // the last iterate's train
    std::vector<std::vector<int64_t>> ranks;    // [0] initial guess, [i] iteration i
    std::vector<double> rse_observed, rse_full, psnr, wall_ms;  // iterations 1..n
    std::vector<double> initial_obs, initial_full, initial_psnr; // the initial guess (0 or 1 entry)
    int status = 1;                             // 0 converged, 1 max_iters, 2 diverged
    std::string note;
};

// idx / vals / truth are device pointers (truth may be null); idx 0-based, strictly increasing.
CompletionRun complete(const int64_t* idx, const double* vals, int64_t count, const std::vector<int64_t>& dims,
                       const CompletionSpec& spec, const double* truth);

}  // namespace ttg
