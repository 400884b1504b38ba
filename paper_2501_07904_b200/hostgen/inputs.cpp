// Seeded synthetic inputs for the BASELINE configs -- harness code
// for bench.py and the tests, NOT the product path and not linked into libttutv_b200.so.
//
// The reference builds its fixtures with a splitmix64 generator and Box-Muller normals
// (src/generators.cpp:13-48), dense trains with gen_planted_tt -> reconstruct
// (generators.cpp:62-79, tt.cpp:52-73 over kernels::matmul, kernels.cpp:48-69) and norms with
// the 4096-blocked sum of squares (kernels.cpp:84-102). This file restates those published
// algorithms so that bench.py can build exactly the buffers the reference's own generators
// give (bitwise: same glibc libm calls, products and sums in the same order, no FMA --
// compiled with -ffp-contract=off for the default x86-64 target), without linking the
// reference. Pinned bitwise against the reference in tests/test_inputs_cpu.py.
//
// Parallelism changes nothing: splitmix64's state after k draws is seed + k*golden, so
// normal pair j (draws 2j, 2j+1) is computed independently; matmul sums over l in order for
// every output element whatever the loop nest.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numbers>
#include <vector>

namespace {

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;

inline uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// draw number k (0-based) of Rng(seed)
inline uint64_t draw(uint64_t seed, uint64_t k) { return mix(seed + (k + 1) * kGolden); }
inline double uniform_of(uint64_t x) { return static_cast<double>(x >> 11) * 0x1.0p-53; }

// normals [first, first + n) of Rng(seed)'s normal() stream; `first` must be even
void normals(uint64_t seed, int64_t first, int64_t n, double* out) {
    const int64_t pair0 = first / 2, pairs = (n + 1) / 2;
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < pairs; ++j) {
        const uint64_t k = 2 * static_cast<uint64_t>(pair0 + j);
        const double u1 = 1.0 - uniform_of(draw(seed, k));
        const double u2 = uniform_of(draw(seed, k + 1));
        const double radius = std::sqrt(-2.0 * std::log(u1));
        const double angle = 2.0 * std::numbers::pi * u2;
        out[2 * j] = radius * std::cos(angle);
        if (2 * j + 1 < n) out[2 * j + 1] = radius * std::sin(angle);
    }
}

// c (m x n) = a (m x k) * b (k x n), column-major, the reference's summation order
void matmul(const double* a, const double* b, double* c, int64_t m, int64_t k, int64_t n) {
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < n; ++j) {
        double* cj = c + j * m;
        for (int64_t i = 0; i < m; ++i) cj[i] = 0.0;
        for (int64_t l = 0; l < k; ++l) {
            const double bv = b[l + j * k];
            const double* al = a + l * m;
            for (int64_t i = 0; i < m; ++i) cj[i] += al[i] * bv;
        }
    }
}

}  // namespace

extern "C" {

// Rng(seed).next_u64() for draws [0, n)
void tig_u64(uint64_t seed, int64_t n, uint64_t* out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = draw(seed, static_cast<uint64_t>(i));
}

// gen_gaussian: n normals of Rng(seed)
void tig_gaussian(uint64_t seed, int64_t n, double* out) { normals(seed, 0, n, out); }

// Rng(seed).uniform() for draws [0, n)
void tig_uniform(uint64_t seed, int64_t n, double* out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = uniform_of(draw(seed, static_cast<uint64_t>(i)));
}

// sum_squares (kernels.cpp:84-102): 4096-element blocks summed in order, then combined in order
double tig_sum_squares(const double* x, int64_t n) {
    constexpr int64_t kBlock = 4096;
    const int64_t blocks = (n + kBlock - 1) / kBlock;
    if (blocks <= 1) {
        double s = 0.0;
        for (int64_t i = 0; i < n; ++i) s += x[i] * x[i];
        return s;
    }
    std::vector<double> part(static_cast<size_t>(blocks));
#pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < blocks; ++b) {
        const int64_t lo = b * kBlock, hi = lo + kBlock < n ? lo + kBlock : n;
        double s = 0.0;
        for (int64_t i = lo; i < hi; ++i) s += x[i] * x[i];
        part[static_cast<size_t>(b)] = s;
    }
    double t = 0.0;
    for (double p : part) t += p;
    return t;
}

// gen_planted_tt(shape, ranks, seed) cores back to back (core k: ranks[k] x dims[k] x ranks[k+1],
// first index fastest), all drawn from one Rng in core order
void tig_planted_cores(const int64_t* dims, int d, const int64_t* ranks, uint64_t seed, double* out) {
    int64_t total = 0;
    for (int k = 0; k < d; ++k) total += ranks[k] * dims[k] * ranks[k + 1];
    normals(seed, 0, total, out);
}

// reconstruct (tt.cpp:52-73): B <- B * left_unfolding(core k), left to right. `work` must hold
// the largest intermediate (the full tensor); `out` receives the dense tensor.
void tig_contract(const double* cores, const int64_t* dims, int d, const int64_t* ranks, double* out,
                  double* work) {
    const double* core = cores;
    int64_t left = dims[0];
    const int64_t n0 = ranks[0] * dims[0] * ranks[1];
    double* cur = (d % 2 == 1) ? out : work;  // the last product lands in `out`
    double* nxt = (d % 2 == 1) ? work : out;
    std::memcpy(cur, core, sizeof(double) * static_cast<size_t>(n0));
    core += n0;
    for (int k = 1; k < d; ++k) {
        const int64_t rl = ranks[k], nk = dims[k], rr = ranks[k + 1];
        matmul(cur, core, nxt, left, rl, nk * rr);  // (left x rl) * (rl x nk rr)
        core += rl * nk * rr;
        left *= nk;
        double* t = cur;
        cur = nxt;
        nxt = t;
    }
}

// a = a0 + s * e elementwise (numpy's `a0 + s * e`: the product rounded, then the sum)
void tig_add_scaled(double* a0, const double* e, double s, int64_t n) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) a0[i] = a0[i] + s * e[i];
}

// scale in place: x *= s
void tig_scale(double* x, double s, int64_t n) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) x[i] = x[i] * s;
}

// Config 4: 64 axis-aligned Gaussian blobs on an n^3 grid. Blob
// parameters from Rng(seed) in the order c_x, c_y, c_z (uniform * n), w_x, w_y, w_z
// (4 + 28 uniform, used as the standard deviation), amplitude (0.2 + 0.8 uniform).
// V(x, y, z) = sum over blobs in order of amp * (gx * gy * gz), g = exp(-0.5 ((t - c) / w)^2);
// storage x + n y + n^2 z (first index fastest).
void tig_blobs(int64_t n, int nblobs, uint64_t seed, double* out) {
    std::vector<double> p(static_cast<size_t>(nblobs) * 7);
    for (int b = 0; b < nblobs; ++b)
        for (int q = 0; q < 7; ++q) {
            const double u = uniform_of(draw(seed, static_cast<uint64_t>(b) * 7 + q));
            p[static_cast<size_t>(b) * 7 + q] = q < 3 ? u * static_cast<double>(n) : q < 6 ? 4.0 + 28.0 * u : 0.2 + 0.8 * u;
        }
    std::vector<double> g(static_cast<size_t>(nblobs) * 3 * static_cast<size_t>(n));
    for (int b = 0; b < nblobs; ++b)
        for (int a = 0; a < 3; ++a)
            for (int64_t t = 0; t < n; ++t) {
                const double z = (static_cast<double>(t) - p[static_cast<size_t>(b) * 7 + a]) / p[static_cast<size_t>(b) * 7 + 3 + a];
                g[(static_cast<size_t>(b) * 3 + a) * static_cast<size_t>(n) + static_cast<size_t>(t)] = std::exp(-0.5 * z * z);
            }
#pragma omp parallel for schedule(static)
    for (int64_t zz = 0; zz < n; ++zz)
        for (int64_t y = 0; y < n; ++y)
            for (int64_t x = 0; x < n; ++x) {
                double v = 0.0;
                for (int b = 0; b < nblobs; ++b) {
                    const double* gb = g.data() + static_cast<size_t>(b) * 3 * static_cast<size_t>(n);
                    v += p[static_cast<size_t>(b) * 7 + 6] * (gb[x] * gb[n + y] * gb[2 * n + zz]);
                }
                out[x + n * (y + n * zz)] = v;
            }
}

// Bernoulli(prob) mask: 1.0 where Rng(seed).uniform() < prob, per entry in storage order;
// returns the number of observed entries
int64_t tig_bernoulli_mask(uint64_t seed, double prob, int64_t n, double* out) {
    int64_t count = 0;
#pragma omp parallel for schedule(static) reduction(+ : count)
    for (int64_t i = 0; i < n; ++i) {
        const bool on = uniform_of(draw(seed, static_cast<uint64_t>(i))) < prob;
        out[i] = on ? 1.0 : 0.0;
        count += on;
    }
    return count;
}

}  // extern "C"
