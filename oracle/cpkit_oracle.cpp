// cpkit_oracle.cpp — CPU restatement of the reference cpkit solver path.
//
// TEST INFRASTRUCTURE ONLY. This file is the parity checker for the B200
// product in paper_1910_12331_b200/. It may only be loaded by tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg.
// The product library never links or calls it.
//
// Why a restatement: the reference (/root/reference/proj) needs Eigen 3 and
// vendored nlohmann/json, CLI11 and doctest headers; none exist in this image
// and there is no network, so the reference cannot be compiled.
// Every function below follows the reference file:line it cites, including
// loop order and the descending mode order of contractions. Dense products
// are sequential-k loops (Eigen's blocked summation order is not knowable
// without Eigen; parity is therefore held to the reference tests' own
// Frobenius-relative tolerances, test_tensor_core.cpp:30-32).
//
// Pinned by: every known-answer test of the reference suites for this path
// (tests/test_oracle_kats.py lists them with their reference file:line).
//
// Build: oracle/Makefile -> oracle/build/libcpkit_oracle.so (C ABI below).

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <limits>
#include <map>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace orc {

// ---------------------------------------------------------------- errors
// errors.hpp:9-49 taxonomy; codes match cpkit.h:30-39.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void invalid(const std::string& m) { throw Error(1, m); }
[[noreturn]] void singular(const std::string& m) { throw Error(4, m); }
[[noreturn]] void numerical(const std::string& m) { throw Error(5, m); }
[[noreturn]] void limit(const std::string& m) { throw Error(6, m); }

// ---------------------------------------------------------------- threads
int g_threads = 1;

void parallel_rows(std::int64_t n, const std::function<void(std::int64_t, std::int64_t)>& fn) {
    const int t = std::max(1, std::min<int>(g_threads, static_cast<int>(std::min<std::int64_t>(n, 1 << 20))));
    if (t <= 1 || n < 64) {
        fn(0, n);
        return;
    }
    std::vector<std::thread> pool;
    const std::int64_t chunk = (n + t - 1) / t;
    for (int i = 0; i < t; ++i) {
        const std::int64_t lo = i * chunk, hi = std::min(n, lo + chunk);
        if (lo >= hi) break;
        pool.emplace_back([&, lo, hi] { fn(lo, hi); });
    }
    for (auto& th : pool) th.join();
}

// ---------------------------------------------------------------- rng
// rng.hpp:11-46 (SplitMix64 keyed mixer, 53-bit uniforms, Box-Muller).
inline std::uint64_t mix64(std::uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
inline std::uint64_t derive(std::uint64_t h, std::uint64_t v) {
    return mix64(h ^ (v * 0xD6E8FEB86659FD93ull + 0xA0761D6478BD642Full));
}
inline std::uint64_t keyed(std::uint64_t seed, std::uint64_t stream, std::uint64_t index,
                           std::uint64_t salt) {
    return derive(derive(derive(mix64(seed), stream), index), salt);
}
inline double to_unit(std::uint64_t bits) { return static_cast<double>(bits >> 11) * 0x1.0p-53; }
inline double uniform(std::uint64_t seed, std::uint64_t stream, std::uint64_t index, double a,
                      double b) {
    return a + (b - a) * to_unit(keyed(seed, stream, index, 0));
}
inline double gaussian(std::uint64_t seed, std::uint64_t stream, std::uint64_t index) {
    const double u1 = static_cast<double>((keyed(seed, stream, index, 1) >> 11) + 1) * 0x1.0p-53;
    const double u2 = to_unit(keyed(seed, stream, index, 2));
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
}
// harness.cpp:19-20, :378-391
constexpr std::uint64_t kProblemTag = 0x50524F42;
constexpr std::uint64_t kInitTag = 0x494E4954;
std::uint64_t problem_seed(std::uint64_t master, int rank, int problem) {
    return derive(derive(derive(mix64(master), kProblemTag), static_cast<std::uint64_t>(rank)),
                  static_cast<std::uint64_t>(problem));
}
std::uint64_t init_seed(std::uint64_t master, int rank, int problem, int init) {
    return derive(derive(derive(derive(mix64(master), kInitTag), static_cast<std::uint64_t>(rank)),
                         static_cast<std::uint64_t>(problem)),
                  static_cast<std::uint64_t>(init));
}

// ---------------------------------------------------------------- Matrix
// matrix_ops.hpp:9-10: row-major dense double matrix.
struct Mat {
    std::int64_t r = 0, c = 0;
    std::vector<double> d;
    Mat() = default;
    Mat(std::int64_t rows, std::int64_t cols, double v = 0.0)
        : r(rows), c(cols), d(static_cast<std::size_t>(rows * cols), v) {}
    double& operator()(std::int64_t i, std::int64_t j) { return d[static_cast<std::size_t>(i * c + j)]; }
    double operator()(std::int64_t i, std::int64_t j) const {
        return d[static_cast<std::size_t>(i * c + j)];
    }
    static Mat identity(std::int64_t n) {
        Mat m(n, n);
        for (std::int64_t i = 0; i < n; ++i) m(i, i) = 1.0;
        return m;
    }
    double norm() const {  // Eigen .norm(): sqrt of the plain sum of squares
        double s = 0.0;
        for (double v : d) s += v * v;
        return std::sqrt(s);
    }
    double sum() const {
        double s = 0.0;
        for (double v : d) s += v;
        return s;
    }
    bool all_finite() const {
        for (double v : d)
            if (!std::isfinite(v)) return false;
        return true;
    }
};

// C (m x n) = A (m x k) * B (k x n); each entry summed in ascending k.
// Row loop is threaded; per-entry summation order is thread-independent.
// Cache blocking only regroups independent entries: 8 rows share each row of
// B and a 256-column strip of C stays in L1; every entry still accumulates
// a(i,0) b(0,j), a(i,1) b(1,j), ... in that order from 0.0.
void gemm_nn(const double* __restrict a, const double* __restrict b, double* __restrict c, std::int64_t m,
             std::int64_t n, std::int64_t k) {
    constexpr std::int64_t kRows = 8, kCols = 256;
    const std::int64_t blocks = (m + kRows - 1) / kRows;
    parallel_rows(blocks, [&](std::int64_t lo, std::int64_t hi) {
        for (std::int64_t blk = lo; blk < hi; ++blk) {
            const std::int64_t i0 = blk * kRows, i1 = std::min(m, i0 + kRows);
            for (std::int64_t j0 = 0; j0 < n; j0 += kCols) {
                const std::int64_t j1 = std::min(n, j0 + kCols);
                for (std::int64_t i = i0; i < i1; ++i)
                    for (std::int64_t j = j0; j < j1; ++j) c[i * n + j] = 0.0;
                for (std::int64_t kk = 0; kk < k; ++kk) {
                    const double* bk = b + kk * n;
                    for (std::int64_t i = i0; i < i1; ++i) {
                        const double aik = a[i * k + kk];
                        double* ci = c + i * n;
                        for (std::int64_t j = j0; j < j1; ++j) ci[j] += aik * bk[j];
                    }
                }
            }
        }
    });
}
Mat mul(const Mat& a, const Mat& b) {
    Mat c(a.r, b.c);
    gemm_nn(a.d.data(), b.d.data(), c.d.data(), a.r, b.c, a.c);
    return c;
}
Mat transpose(const Mat& a) {
    Mat t(a.c, a.r);
    for (std::int64_t i = 0; i < a.r; ++i)
        for (std::int64_t j = 0; j < a.c; ++j) t(j, i) = a(i, j);
    return t;
}
// matrix_ops.cpp:23-28
Mat hadamard(const Mat& a, const Mat& b) {
    if (a.r != b.r || a.c != b.c) invalid("hadamard: shape mismatch");
    Mat o(a.r, a.c);
    for (std::size_t i = 0; i < a.d.size(); ++i) o.d[i] = a.d[i] * b.d[i];
    return o;
}
// matrix_ops.cpp:9-21 (test-only in the reference)
Mat khatri_rao(const Mat& a, const Mat& b) {
    if (a.c != b.c) invalid("khatri_rao: column counts differ");
    Mat o(a.r * b.r, a.c);
    for (std::int64_t i = 0; i < a.r; ++i)
        for (std::int64_t j = 0; j < b.r; ++j)
            for (std::int64_t k = 0; k < a.c; ++k) o(i * b.r + j, k) = b(j, k) * a(i, k);
    return o;
}
// matrix_ops.cpp:30-34: S = A^T A, then S = 0.5 (S + S^T)
Mat gram(const Mat& a) {
    Mat g(a.c, a.c);
    for (std::int64_t i = 0; i < a.r; ++i)
        for (std::int64_t x = 0; x < a.c; ++x) {
            const double v = a(i, x);
            for (std::int64_t y = 0; y < a.c; ++y) g(x, y) += v * a(i, y);
        }
    Mat s(a.c, a.c);
    for (std::int64_t x = 0; x < a.c; ++x)
        for (std::int64_t y = 0; y < a.c; ++y) s(x, y) = 0.5 * (g(x, y) + g(y, x));
    return s;
}

// matrix_ops.cpp:41-56: LLT of S + lambda I with one jitter retry.
// Eigen's LLT reports failure when a pivot is <= 0.
bool llt_inplace(Mat& a) {
    const std::int64_t n = a.r;
    for (std::int64_t j = 0; j < n; ++j) {
        double x = a(j, j);
        for (std::int64_t k = 0; k < j; ++k) x -= a(j, k) * a(j, k);
        if (x <= 0.0) return false;
        const double l = std::sqrt(x);
        a(j, j) = l;
        for (std::int64_t i = j + 1; i < n; ++i) {
            double y = a(i, j);
            for (std::int64_t k = 0; k < j; ++k) y -= a(i, k) * a(j, k);
            a(i, j) = y / l;
        }
    }
    for (std::int64_t i = 0; i < n; ++i)
        for (std::int64_t j = i + 1; j < n; ++j) a(i, j) = 0.0;
    return true;
}
Mat factor_shifted(const Mat& s, double lambda) {
    const std::int64_t n = s.r;
    Mat shifted = s;
    for (std::int64_t i = 0; i < n; ++i) shifted(i, i) += lambda;
    Mat l = shifted;
    if (llt_inplace(l)) return l;
    double tr = 0.0;
    for (std::int64_t i = 0; i < n; ++i) tr += s(i, i);
    const double jitter = 1e-12 * tr / static_cast<double>(n);
    for (std::int64_t i = 0; i < n; ++i) shifted(i, i) += jitter;
    l = shifted;
    if (!llt_inplace(l)) singular("spd_solve: factorization failed after jitter retry");
    return l;
}
// Solves (L L^T) x = b in place for each column of b^T, i.e. each row of y.
void llt_solve_rows(const Mat& l, Mat& y) {
    const std::int64_t n = l.r;
    for (std::int64_t row = 0; row < y.r; ++row) {
        double* v = &y.d[static_cast<std::size_t>(row * n)];
        for (std::int64_t i = 0; i < n; ++i) {
            double s = v[i];
            for (std::int64_t k = 0; k < i; ++k) s -= l(i, k) * v[k];
            v[i] = s / l(i, i);
        }
        for (std::int64_t i = n; i-- > 0;) {
            double s = v[i];
            for (std::int64_t k = i + 1; k < n; ++k) s -= l(k, i) * v[k];
            v[i] = s / l(i, i);
        }
    }
}
// matrix_ops.cpp:60-71: Y (S + lambda I) = B
Mat spd_solve(const Mat& s, const Mat& b, double lambda) {
    if (s.r != s.c) invalid("spd_solve: S must be square");
    if (b.c != s.r) invalid("spd_solve: B column count must match S");
    Mat l = factor_shifted(s, lambda);
    Mat y = b;  // rows of Y are the solved columns of Y^T
    llt_solve_rows(l, y);
    return y;
}
// matrix_ops.cpp:73-81
Mat spd_inverse(const Mat& s, double lambda) {
    if (s.r != s.c) invalid("spd_inverse: S must be square");
    Mat l = factor_shifted(s, lambda);
    Mat inv = Mat::identity(s.r);  // symmetric input: rows == columns
    llt_solve_rows(l, inv);
    inv = transpose(inv);
    Mat o(s.r, s.r);
    for (std::int64_t i = 0; i < s.r; ++i)
        for (std::int64_t j = 0; j < s.r; ++j) o(i, j) = 0.5 * (inv(i, j) + inv(j, i));
    return o;
}

// ---------------------------------------------------------------- tensor
// tensor.hpp:16-48
struct Tensor {
    std::vector<std::uint64_t> dims;
    const double* data = nullptr;  // borrowed, row-major (last index fastest)
    std::uint64_t size = 0;
    std::size_t order() const { return dims.size(); }
};
// tensor.cpp:61-67 (sequential sum of squares)
double norm2(const Tensor& t) {
    double acc = 0.0;
    for (std::uint64_t i = 0; i < t.size; ++i) acc += t.data[i] * t.data[i];
    return acc;
}

// ---------------------------------------------------------------- model
// kruskal.hpp:15-26
struct Model {
    std::vector<std::uint64_t> dims;
    std::int64_t rank = 0;
    std::vector<Mat> factors;
    std::size_t order() const { return dims.size(); }
    void validate() const {  // kruskal.cpp:27-40
        if (dims.empty() || rank < 1) invalid("model needs order >= 1 and rank >= 1");
        if (factors.size() != dims.size()) invalid("model factor count does not match order");
        for (std::size_t n = 0; n < dims.size(); ++n) {
            if (static_cast<std::uint64_t>(factors[n].r) != dims[n] || factors[n].c != rank)
                invalid("model factor shape mismatch");
            if (!factors[n].all_finite()) invalid("model factor contains non-finite entries");
        }
    }
};

// ---------------------------------------------------------------- MTTKRP
// mttkrp.hpp:15-20
struct Partial {
    std::vector<std::size_t> kept_modes;
    std::vector<std::uint64_t> kept_dims;
    std::int64_t rank = 0;
    std::vector<double> data;
};
std::uint64_t dim_product(const std::vector<std::uint64_t>& d, std::size_t lo, std::size_t hi) {
    std::uint64_t p = 1;
    for (std::size_t m = lo; m < hi; ++m) p *= d[m];
    return p;
}
// mttkrp.cpp:29-77
Partial contract_mode(const Partial& p, std::size_t mode_id, const Mat& a) {
    const std::size_t pos = static_cast<std::size_t>(
        std::find(p.kept_modes.begin(), p.kept_modes.end(), mode_id) - p.kept_modes.begin());
    const std::uint64_t outer = dim_product(p.kept_dims, 0, pos);
    const std::uint64_t sm = p.kept_dims[pos];
    const std::uint64_t inner = dim_product(p.kept_dims, pos + 1, p.kept_dims.size());
    const std::int64_t rank = (p.rank > 0) ? p.rank : a.c;
    const std::uint64_t R = static_cast<std::uint64_t>(rank);

    Partial out;
    out.kept_modes = p.kept_modes;
    out.kept_modes.erase(out.kept_modes.begin() + static_cast<std::ptrdiff_t>(pos));
    out.kept_dims = p.kept_dims;
    out.kept_dims.erase(out.kept_dims.begin() + static_cast<std::ptrdiff_t>(pos));
    out.rank = rank;
    out.data.assign(outer * inner * R, 0.0);

    if (p.rank == 0) {
        if (inner == 1) {
            // :46-53 one GEMM (outer x sm) * (sm x R)
            gemm_nn(p.data.data(), a.d.data(), out.data.data(), static_cast<std::int64_t>(outer),
                    rank, static_cast<std::int64_t>(sm));
            return out;
        }
        // :55-62 per-outer slice^T (inner x sm) * A (sm x R), summed over sm ascending
        parallel_rows(static_cast<std::int64_t>(outer), [&](std::int64_t lo, std::int64_t hi) {
            for (std::int64_t o = lo; o < hi; ++o) {
                const double* slice = p.data.data() + static_cast<std::uint64_t>(o) * sm * inner;
                double* dst = out.data.data() + static_cast<std::uint64_t>(o) * inner * R;
                for (std::uint64_t im = 0; im < sm; ++im) {
                    const double* arow = a.d.data() + im * R;
                    const double* srow = slice + im * inner;
                    for (std::uint64_t j = 0; j < inner; ++j) {
                        const double s = srow[j];
                        double* drow = dst + j * R;
                        for (std::uint64_t r = 0; r < R; ++r) drow[r] += s * arow[r];
                    }
                }
            }
        });
    } else {
        // :63-75 Hadamard-weighted reduction over the contracted kept mode
        parallel_rows(static_cast<std::int64_t>(outer), [&](std::int64_t lo, std::int64_t hi) {
            for (std::int64_t o = lo; o < hi; ++o) {
                double* dst = out.data.data() + static_cast<std::uint64_t>(o) * inner * R;
                for (std::uint64_t im = 0; im < sm; ++im) {
                    const double* src =
                        p.data.data() + ((static_cast<std::uint64_t>(o) * sm + im) * inner) * R;
                    const double* arow = a.d.data() + im * R;
                    for (std::uint64_t j = 0; j < inner; ++j)
                        for (std::uint64_t r = 0; r < R; ++r) dst[j * R + r] += src[j * R + r] * arow[r];
                }
            }
        });
    }
    return out;
}
// mttkrp.cpp:79-87 (the reference copies the whole tensor here)
Partial tensor_as_partial(const Tensor& t) {
    Partial p;
    p.kept_modes.resize(t.order());
    for (std::size_t m = 0; m < t.order(); ++m) p.kept_modes[m] = m;
    p.kept_dims = t.dims;
    p.rank = 0;
    p.data.assign(t.data, t.data + t.size);
    return p;
}
// mttkrp.cpp:89-92
Mat partial_to_matrix(const Partial& p) {
    Mat m(static_cast<std::int64_t>(p.kept_dims[0]), p.rank);
    m.d = p.data;
    return m;
}
// mttkrp.cpp:94-116
void check_inputs(const Tensor& t, const std::vector<Mat>& f, std::size_t mode) {
    if (t.order() < 2) invalid("mttkrp: tensor order must be at least 2");
    if (mode >= t.order()) invalid("mttkrp: mode out of range");
    if (f.size() != t.order()) invalid("mttkrp: factor count does not match order");
    const std::int64_t rank = f[0].c;
    for (std::size_t m = 0; m < t.order(); ++m) {
        if (f[m].c != rank) invalid("mttkrp: rank mismatch across factors");
        if (static_cast<std::uint64_t>(f[m].r) != t.dims[m])
            invalid("mttkrp: factor rows do not match extent");
    }
}
// mttkrp.cpp:118-126: contract highest mode first
Partial contract_set(Partial p, std::vector<std::size_t> modes, const std::vector<Mat>& f,
                     int* counter) {
    std::sort(modes.begin(), modes.end(), std::greater<>());
    for (std::size_t m : modes) {
        if (p.rank == 0 && counter != nullptr) ++(*counter);
        p = contract_mode(p, m, f[m]);
    }
    return p;
}
// mttkrp.hpp:35-54
struct Workspace {
    std::map<std::uint64_t, Partial> cache;
    int full_contractions = 0;
    void note_factor_update(std::size_t mode) {  // mttkrp.cpp:136-145
        const std::uint64_t bit = 1ull << mode;
        for (auto it = cache.begin(); it != cache.end();) {
            if (it->first & bit)
                it = cache.erase(it);
            else
                ++it;
        }
    }
};
// mttkrp.cpp:149-158 (naive, uncached)
Mat mttkrp(const Tensor& t, const std::vector<Mat>& f, std::size_t mode) {
    check_inputs(t, f, mode);
    std::vector<std::size_t> others;
    for (std::size_t m = 0; m < t.order(); ++m)
        if (m != mode) others.push_back(m);
    return partial_to_matrix(contract_set(tensor_as_partial(t), others, f, nullptr));
}
// mttkrp.cpp:160-189 (dimension tree)
Mat mttkrp(const Tensor& t, const std::vector<Mat>& f, std::size_t mode, Workspace& ws) {
    check_inputs(t, f, mode);
    const std::size_t order = t.order();
    const std::size_t half = (order + 1) / 2;
    std::vector<std::size_t> contracted, remaining;
    if (mode < half) {
        for (std::size_t m = half; m < order; ++m) contracted.push_back(m);
        for (std::size_t m = 0; m < half; ++m)
            if (m != mode) remaining.push_back(m);
    } else {
        for (std::size_t m = 0; m < half; ++m) contracted.push_back(m);
        for (std::size_t m = half; m < order; ++m)
            if (m != mode) remaining.push_back(m);
    }
    std::uint64_t key = 0;
    for (std::size_t m : contracted) key |= (1ull << m);
    auto it = ws.cache.find(key);
    if (it == ws.cache.end()) {
        Partial root = contract_set(tensor_as_partial(t), contracted, f, &ws.full_contractions);
        it = ws.cache.emplace(key, std::move(root)).first;
    }
    return partial_to_matrix(contract_set(it->second, remaining, f, &ws.full_contractions));
}

// ---------------------------------------------------------------- Gamma / residual
// kruskal.hpp:32-39
struct GammaSet {
    std::vector<Mat> grams;
    std::vector<std::vector<Mat>> pairwise;
    const Mat& gamma(std::size_t n, std::size_t p) const { return pairwise[n][p]; }
};
// kruskal.cpp:42-65
GammaSet build_gamma_set(const Model& model) {
    const std::size_t order = model.order();
    if (order < 2) invalid("build_gamma_set: order must be at least 2");
    GammaSet gs;
    for (const auto& a : model.factors) gs.grams.push_back(gram(a));
    gs.pairwise.assign(order, std::vector<Mat>(order));
    for (std::size_t n = 0; n < order; ++n)
        for (std::size_t p = n; p < order; ++p) {
            Mat g(model.rank, model.rank, 1.0);
            for (std::size_t m = 0; m < order; ++m) {
                if (m == n || m == p) continue;
                g = hadamard(g, gs.grams[m]);
            }
            gs.pairwise[n][p] = g;
            if (p != n) gs.pairwise[p][n] = g;
        }
    return gs;
}
// kruskal.cpp:67-92 (dense evaluation, reference per-entry order)
std::vector<double> reconstruct(const Model& model) {
    // kruskal.cpp:76-90 per entry: acc = sum_r (((1 A_0) A_1) ... A_{N-1}), r
    // ascending, separate multiply and add. The product over modes 0..N-2 is
    // the same for every last-mode index, so it is formed once per prefix row
    // (the same roundings); the last-mode loop then runs across j.
    std::uint64_t total = 1;
    for (auto d : model.dims) total *= d;
    const std::size_t order = model.order();
    std::vector<double> t(total);
    const std::uint64_t R = static_cast<std::uint64_t>(model.rank);
    const std::uint64_t sl = model.dims[order - 1];
    const std::uint64_t rows = total / sl;
    std::vector<double> bt(R * sl);  // last factor transposed: bt[r][j]
    for (std::uint64_t j = 0; j < sl; ++j)
        for (std::uint64_t r = 0; r < R; ++r) bt[r * sl + j] = model.factors[order - 1].d[j * R + r];
    parallel_rows(static_cast<std::int64_t>(rows), [&](std::int64_t lo, std::int64_t hi) {
        std::vector<double> pre(R);
        std::vector<std::uint64_t> idx(order, 0);
        for (std::int64_t f = lo; f < hi; ++f) {
            std::uint64_t q = static_cast<std::uint64_t>(f);
            for (std::size_t m = order - 1; m-- > 0;) {
                idx[m] = q % model.dims[m];
                q /= model.dims[m];
            }
            for (std::uint64_t r = 0; r < R; ++r) {
                double prod = 1.0;
                for (std::size_t n = 0; n + 1 < order; ++n) prod *= model.factors[n].d[idx[n] * R + r];
                pre[r] = prod;
            }
            double* __restrict a = t.data() + static_cast<std::uint64_t>(f) * sl;
            for (std::uint64_t j = 0; j < sl; ++j) a[j] = 0.0;
            for (std::uint64_t r = 0; r < R; ++r) {
                const double pr = pre[r];
                const double* __restrict br = bt.data() + r * sl;
                for (std::uint64_t j = 0; j < sl; ++j) a[j] += pr * br[j];
            }
        }
    });
    return t;
}

// ---------------------------------------------------------------- keyed noise
// Restatement of the product's noise definition (BASELINE configs 2 and 5:
// Gaussian noise scaled to rel ||X||_F; SURVEY.md §8d stream 0x4E01). The
// reference generates no noise; the product defines it so that a GPU and this
// CPU restatement produce the same bits: rng.hpp:40-46's Box-Muller with log
// and cos evaluated by fixed polynomial programs of correctly rounded
// +, -, *, /, sqrt (this file is built with -ffp-contract=off), keyed at each
// entry's global flat index; ||X||^2 and ||E||^2 summed in a fixed
// column-block order that does not depend on how the last mode is sharded.
constexpr int kNoiseBlocks = 256;
double portable_log(double u) {
    std::uint64_t bits;
    std::memcpy(&bits, &u, 8);
    int e = static_cast<int>((bits >> 52) & 0x7FF) - 1022;
    bits = (bits & 0x000FFFFFFFFFFFFFull) | (static_cast<std::uint64_t>(1022) << 52);
    double m;
    std::memcpy(&m, &bits, 8);
    if (m < 0x1.6a09e667f3bcdp-1) {
        m *= 2.0;
        e -= 1;
    }
    const double s = (m - 1.0) / (m + 1.0), z = s * s;
    static const double kl[14] = {0x1.0000000000000p+0, 0x1.5555555555555p-2, 0x1.999999999999ap-3,
                                  0x1.2492492492492p-3, 0x1.c71c71c71c71cp-4, 0x1.745d1745d1746p-4,
                                  0x1.3b13b13b13b14p-4, 0x1.1111111111111p-4, 0x1.e1e1e1e1e1e1ep-5,
                                  0x1.af286bca1af28p-5, 0x1.8618618618618p-5, 0x1.642c8590b2164p-5,
                                  0x1.47ae147ae147bp-5, 0x1.2f684bda12f68p-5};
    double p = kl[13];
    for (int i = 12; i >= 0; --i) p = p * z + kl[i];
    const double de = static_cast<double>(e);
    return de * 0x1.62e42fee00000p-1 + (de * 0x1.a39ef35793c76p-33 + (2.0 * s) * p);
}
double portable_cos_2pi(double u) {
    const double t = u * 4.0;
    const int k = static_cast<int>(t);
    const double r = t - static_cast<double>(k);
    const double th = r * 0x1.921fb54442d18p+0, z = th * th;
    static const double kc[14] = {0x1.0000000000000p+0,  -0x1.0000000000000p-1, 0x1.5555555555555p-5,
                                  -0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-16,  -0x1.27e4fb7789f5cp-22,
                                  0x1.1eed8eff8d898p-29,  -0x1.93974a8c07c9dp-37, 0x1.ae7f3e733b81fp-45,
                                  -0x1.6827863b97d97p-53, 0x1.e542ba4020225p-62,  -0x1.0ce396db7f853p-70,
                                  0x1.f2cf01972f578p-80,  -0x1.88e85fc6a4e59p-89};
    static const double ks[13] = {0x1.0000000000000p+0,  -0x1.5555555555555p-3, 0x1.1111111111111p-7,
                                  -0x1.a01a01a01a01ap-13, 0x1.71de3a556c734p-19,  -0x1.ae64567f544e4p-26,
                                  0x1.6124613a86d09p-33,  -0x1.ae7f3e733b81fp-41, 0x1.952c77030ad4ap-49,
                                  -0x1.2f49b46814157p-57, 0x1.71b8ef6dcf572p-66,  -0x1.761b413163819p-75,
                                  0x1.3f3ccdd165fa9p-84};
    double cc = kc[13], ss = ks[12];
    for (int i = 12; i >= 0; --i) cc = cc * z + kc[i];
    for (int i = 11; i >= 0; --i) ss = ss * z + ks[i];
    ss *= th;
    switch (k & 3) {
        case 0: return cc;
        case 1: return -ss;
        case 2: return -cc;
        default: return ss;
    }
}
double noise_gaussian(std::uint64_t base, std::uint64_t gidx) {
    const std::uint64_t h = derive(base, gidx);
    const double u1 = static_cast<double>((derive(h, 1) >> 11) + 1) * 0x1.0p-53;
    const double u2 = static_cast<double>(derive(h, 2) >> 11) * 0x1.0p-53;
    return std::sqrt(-2.0 * portable_log(u1)) * portable_cos_2pi(u2);
}
// x (full tensor, last extent sl) += scale E; returns {scale, ||X||^2, ||E||^2}
std::array<double, 3> add_noise(double* x, const std::vector<std::uint64_t>& dims, std::uint64_t seed, double rel) {
    std::uint64_t total = 1;
    for (auto d : dims) total *= d;
    const std::uint64_t sl = dims.back(), rows = total / sl;
    const std::uint64_t blk = (rows + kNoiseBlocks - 1) / kNoiseBlocks;
    const std::uint64_t base = derive(mix64(seed), 0x4E01);
    std::vector<double> part(2 * kNoiseBlocks * sl, 0.0);  // [X | E][block][column]
    parallel_rows(kNoiseBlocks, [&](std::int64_t lo, std::int64_t hi) {
        for (std::int64_t b = lo; b < hi; ++b) {
            double* px = part.data() + static_cast<std::uint64_t>(b) * sl;
            double* pe = part.data() + (kNoiseBlocks + static_cast<std::uint64_t>(b)) * sl;
            const std::uint64_t r1 = std::min(rows, (static_cast<std::uint64_t>(b) + 1) * blk);
            for (std::uint64_t r = static_cast<std::uint64_t>(b) * blk; r < r1; ++r)
                for (std::uint64_t j = 0; j < sl; ++j) {
                    const double v = x[r * sl + j];
                    px[j] += v * v;
                    const double g = noise_gaussian(base, r * sl + j);
                    pe[j] += g * g;
                }
        }
    });
    double nx = 0.0, ne = 0.0;
    for (std::uint64_t j = 0; j < sl; ++j) {
        double cx = 0.0, ce = 0.0;
        for (int b = 0; b < kNoiseBlocks; ++b) {
            cx += part[static_cast<std::uint64_t>(b) * sl + j];
            ce += part[(kNoiseBlocks + static_cast<std::uint64_t>(b)) * sl + j];
        }
        nx += cx;
        ne += ce;
    }
    // (columns in ascending j: the GPU sums rank blocks in rank order, i.e. the same order)
    const double scale = rel * std::sqrt(nx) / std::sqrt(ne);
    parallel_rows(static_cast<std::int64_t>(rows), [&](std::int64_t lo, std::int64_t hi) {
        for (std::uint64_t e = static_cast<std::uint64_t>(lo) * sl; e < static_cast<std::uint64_t>(hi) * sl; ++e)
            x[e] += scale * noise_gaussian(base, e);
    });
    return {scale, nx, ne};
}
// kruskal.cpp:94-118
std::pair<double, double> residual_fitness(const Model& model, const Tensor& x, double xnorm2,
                                           const Mat* last) {
    if (!(xnorm2 > 0.0)) invalid("residual_fitness: tensor norm must be positive");
    const std::size_t l = model.order() - 1;
    Mat local;
    if (last == nullptr) {
        local = mttkrp(x, model.factors, l);
        last = &local;
    }
    double cross = 0.0;
    for (std::size_t i = 0; i < last->d.size(); ++i) cross += last->d[i] * model.factors[l].d[i];
    Mat all(model.rank, model.rank, 1.0);
    for (const auto& a : model.factors) all = hadamard(all, gram(a));
    const double model_norm2 = all.sum();
    double res2 = xnorm2 - 2.0 * cross + model_norm2;
    if (res2 < 0.0) res2 = 0.0;
    const double r = std::sqrt(res2 / xnorm2);
    return {r, 1.0 - r};
}

// ---------------------------------------------------------------- GN
enum class RegMode { constant = 0, varying = 1 };
enum class RegShape { identity = 0, diagonal = 1 };
// gauss_newton.hpp:19-34
struct RegSchedule {
    RegMode mode = RegMode::constant;
    RegShape shape = RegShape::identity;
    double lambda = 1e-3, mu = 2.0, lower = 1e-6, upper = 1e-2;
    int direction = 0;  // 0 down, 1 up
    void validate() const {  // gauss_newton.cpp:33-45
        if (lambda < 0) invalid("schedule: lambda must be nonnegative");
        if (mode == RegMode::varying) {
            if (!(mu > 1.0)) invalid("schedule: mu must exceed 1");
            if (!(lower > 0.0) || !(lower < upper)) invalid("schedule: need 0 < lower < upper");
        }
    }
};
// gauss_newton.cpp:47-59
RegSchedule schedule_next(RegSchedule s) {
    if (s.mode == RegMode::constant) return s;
    if (s.direction == 0) {
        s.lambda /= s.mu;
        if (s.lambda < s.lower) s.direction = 1;
    } else {
        s.lambda *= s.mu;
        if (s.lambda > s.upper) s.direction = 0;
    }
    return s;
}
struct GnConfig {  // gauss_newton.hpp:50-62
    double grad_tol = 0.0, residual_tol = 5e-5, step_tol = 1e-7;
    int max_iters = 500;
    double cg_tol = 1e-3;
    int cg_max_iters = 0;
    RegSchedule schedule;
    bool armijo = false;
    double c1 = 1e-4, shrink = 0.5;
    int max_backtracks = 20;
    int cg_beta = 0;  // 0 standard, 1 stale_denominator
    void validate() const {  // gauss_newton.cpp:61-79
        schedule.validate();
        if (grad_tol < 0 || residual_tol < 0 || step_tol < 0) invalid("gn config: negative tolerance");
        if (max_iters < 0 || cg_max_iters < 0) invalid("gn config: negative iteration cap");
        if (!(cg_tol > 0)) invalid("gn config: cg_tol must be positive");
        if (armijo) {
            if (!(c1 > 0 && c1 < 1) || !(shrink > 0 && shrink < 1) || max_backtracks < 1)
                invalid("gn config: bad armijo parameters");
        }
    }
};
// gauss_newton.cpp:81-94
std::vector<Mat> gradient(const Model& model, const std::vector<Mat>& mk, const GammaSet& gs) {
    if (mk.size() != model.order()) invalid("gradient: need one MTTKRP per mode");
    std::vector<Mat> g;
    for (std::size_t n = 0; n < model.order(); ++n) {
        Mat t = mul(model.factors[n], gs.gamma(n, n));
        for (std::size_t i = 0; i < t.d.size(); ++i) t.d[i] -= mk[n].d[i];
        g.push_back(std::move(t));
    }
    return g;
}
// gauss_newton.cpp:96-136 (reference loop order: identity/diag term, then p ascending)
std::vector<Mat> hessian_matvec(const Model& model, const GammaSet& gs, const std::vector<Mat>& w,
                                double lambda, RegShape shape) {
    const std::size_t order = model.order();
    if (w.size() != order) invalid("hessian_matvec: need one block per mode");
    for (std::size_t n = 0; n < order; ++n)
        if (w[n].r != model.factors[n].r || w[n].c != model.rank)
            invalid("hessian_matvec: block shape mismatch");
    std::vector<Mat> u;
    for (std::size_t n = 0; n < order; ++n) {
        Mat un(w[n].r, w[n].c);
        const Mat& gnn = gs.gamma(n, n);
        for (std::int64_t i = 0; i < un.r; ++i)
            for (std::int64_t r = 0; r < un.c; ++r)
                un(i, r) = (shape == RegShape::identity) ? lambda * w[n](i, r)
                                                         : w[n](i, r) * (lambda * gnn(r, r));
        for (std::size_t p = 0; p < order; ++p) {
            Mat add;
            if (p == n) {
                add = mul(w[n], gnn);
            } else {
                Mat b = mul(transpose(model.factors[p]), w[p]);
                Mat d = hadamard(gs.gamma(n, p), b);
                add = mul(model.factors[n], transpose(d));
            }
            for (std::size_t i = 0; i < un.d.size(); ++i) un.d[i] += add.d[i];
        }
        u.push_back(std::move(un));
    }
    return u;
}
// gauss_newton.cpp:138-188: dense J^T J (columns mode-major, column-major per factor)
Mat explicit_jtj(const Model& model, std::uint64_t var_cap) {
    model.validate();
    const std::size_t order = model.order();
    const std::int64_t rank = model.rank;
    std::uint64_t vars = 0;
    std::vector<std::uint64_t> off(order, 0);
    for (std::size_t n = 0; n < order; ++n) {
        off[n] = vars;
        vars += model.dims[n] * static_cast<std::uint64_t>(rank);
    }
    if (vars > var_cap) limit("explicit_jtj: variable count exceeds cap");
    std::uint64_t rows = 1;
    for (auto d : model.dims) rows *= d;
    Mat jac(static_cast<std::int64_t>(rows), static_cast<std::int64_t>(vars));
    std::vector<std::uint64_t> idx(order, 0);
    std::vector<double> pre(order + 1), suf(order + 1);
    for (std::uint64_t f = 0; f < rows; ++f) {
        for (std::int64_t r = 0; r < rank; ++r) {
            pre[0] = 1.0;
            for (std::size_t m = 0; m < order; ++m)
                pre[m + 1] = pre[m] * model.factors[m](static_cast<std::int64_t>(idx[m]), r);
            suf[order] = 1.0;
            for (std::size_t m = order; m-- > 0;)
                suf[m] = suf[m + 1] * model.factors[m](static_cast<std::int64_t>(idx[m]), r);
            for (std::size_t n = 0; n < order; ++n) {
                const std::uint64_t col = off[n] + static_cast<std::uint64_t>(r) * model.dims[n] + idx[n];
                jac(static_cast<std::int64_t>(f), static_cast<std::int64_t>(col)) = -(pre[n] * suf[n + 1]);
            }
        }
        for (std::size_t m = order; m-- > 0;) {
            if (++idx[m] < model.dims[m]) break;
            idx[m] = 0;
        }
    }
    return gram(jac);
}
// gauss_newton.cpp:190-207
std::vector<Mat> build_preconditioner(const GammaSet& gs, double lambda, RegShape shape) {
    if (lambda < 0) invalid("build_preconditioner: lambda must be nonnegative");
    std::vector<Mat> pinv;
    for (std::size_t n = 0; n < gs.grams.size(); ++n) {
        if (shape == RegShape::identity) {
            pinv.push_back(spd_inverse(gs.gamma(n, n), lambda));
        } else {
            Mat s = gs.gamma(n, n);
            for (std::int64_t i = 0; i < s.r; ++i) s(i, i) *= (1.0 + lambda);
            pinv.push_back(spd_inverse(s, 0.0));
        }
    }
    return pinv;
}
// gauss_newton.cpp:246-265
double norm_sum(const std::vector<Mat>& ms) {
    double acc = 0.0;
    for (const auto& m : ms) acc += m.norm();
    return acc;
}
double dot_sum(const std::vector<Mat>& a, const std::vector<Mat>& b) {
    double acc = 0.0;
    for (std::size_t n = 0; n < a.size(); ++n) {
        double s = 0.0;
        for (std::size_t i = 0; i < a[n].d.size(); ++i) s += a[n].d[i] * b[n].d[i];
        acc += s;
    }
    return acc;
}
bool all_finite(const std::vector<Mat>& ms) {
    for (const auto& m : ms)
        if (!m.all_finite()) return false;
    return true;
}
// gauss_newton.cpp:267-275
int default_cg_cap(const Model& model) {
    std::uint64_t total = 0;
    for (auto d : model.dims) total += d * static_cast<std::uint64_t>(model.rank);
    return static_cast<int>(std::min<std::uint64_t>(total, 10ull * static_cast<std::uint64_t>(model.rank)));
}
struct CgResult {
    std::vector<Mat> v;
    int iterations = 0;
    bool hit_cap = false, breakdown = false;
};
// gauss_newton.cpp:279-349
CgResult cp_cg(const Model& model, const GammaSet& gs, const std::vector<Mat>& g, double lambda,
               const GnConfig& cfg) {
    const std::size_t order = model.order();
    if (g.size() != order) invalid("cp_cg: need one gradient block per mode");
    const RegShape shape = cfg.schedule.shape;
    const int cap = cfg.cg_max_iters > 0 ? cfg.cg_max_iters : default_cg_cap(model);
    std::vector<Mat> v, rres, z, w, q;
    for (std::size_t n = 0; n < order; ++n) v.emplace_back(g[n].r, g[n].c);
    CgResult out;
    const double gnorm = norm_sum(g);
    if (gnorm == 0.0) {
        out.v = v;
        return out;
    }
    const std::vector<Mat> pinv = build_preconditioner(gs, lambda, shape);
    for (std::size_t n = 0; n < order; ++n) {
        Mat r = g[n];
        for (double& x : r.d) x = -x;
        z.push_back(mul(r, pinv[n]));
        rres.push_back(std::move(r));
    }
    w = z;
    double rz = dot_sum(rres, z);
    const double target = cfg.cg_tol * gnorm;
    int it = 0;
    while (norm_sum(rres) > target) {
        if (it >= cap) {
            out.hit_cap = true;
            break;
        }
        q = hessian_matvec(model, gs, w, lambda, shape);
        const double wq = dot_sum(w, q);
        if (!(wq > 0.0)) {
            out.breakdown = true;
            break;
        }
        const double alpha = rz / wq;
        for (std::size_t n = 0; n < order; ++n) {
            for (std::size_t i = 0; i < v[n].d.size(); ++i) {
                v[n].d[i] += alpha * w[n].d[i];
                rres[n].d[i] -= alpha * q[n].d[i];
            }
            z[n] = mul(rres[n], pinv[n]);
        }
        const double rz_new = dot_sum(rres, z);
        const double beta = (cfg.cg_beta == 0) ? rz_new / rz : rz_new / wq;
        for (std::size_t n = 0; n < order; ++n)
            for (std::size_t i = 0; i < w[n].d.size(); ++i) w[n].d[i] = z[n].d[i] + beta * w[n].d[i];
        rz = rz_new;
        ++it;
        if (!all_finite(v) || !all_finite(rres)) numerical("cp_cg: non-finite iterate");
    }
    out.v = std::move(v);
    out.iterations = it;
    return out;
}
struct GnStepDiag {  // gauss_newton.hpp:117-131
    int halt = 0;  // 0 none, 1 residual, 2 gradient
    bool stepped = false;
    double residual_before = 1.0, residual_after = 1.0, grad_norm = 0.0, lambda = 0.0;
    int cg_iters = 0;
    double step_norm = 0.0, alpha = 1.0;
    bool armijo_exhausted = false, cg_hit_cap = false, cg_breakdown = false;
};
// gauss_newton.cpp:360-449
GnStepDiag gn_step(const Tensor& x, Model& model, Workspace& ws, const GnConfig& cfg,
                   RegSchedule& schedule, double xnorm2) {
    const std::size_t order = model.order();
    GnStepDiag diag;
    std::vector<Mat> mk;
    for (std::size_t n = 0; n < order; ++n) mk.push_back(mttkrp(x, model.factors, n, ws));
    GammaSet gs = build_gamma_set(model);
    auto [res, fit] = residual_fitness(model, x, xnorm2, &mk.back());
    (void)fit;
    diag.residual_before = res;
    diag.residual_after = res;
    if (res < cfg.residual_tol) {
        diag.halt = 1;
        return diag;
    }
    std::vector<Mat> g = gradient(model, mk, gs);
    diag.grad_norm = 0.0;
    for (const auto& gn : g) diag.grad_norm += gn.norm();
    if (diag.grad_norm <= cfg.grad_tol) {
        diag.halt = 2;
        return diag;
    }
    diag.lambda = schedule.lambda;
    CgResult cg = cp_cg(model, gs, g, diag.lambda, cfg);
    diag.cg_iters = cg.iterations;
    diag.cg_hit_cap = cg.hit_cap;
    diag.cg_breakdown = cg.breakdown;
    double alpha = 1.0, residual_after = -1.0;
    if (cfg.armijo) {
        const double f0 = 0.5 * res * res * xnorm2;
        double gv = 0.0;
        for (std::size_t n = 0; n < order; ++n) {
            double s = 0.0;
            for (std::size_t i = 0; i < g[n].d.size(); ++i) s += g[n].d[i] * cg.v[n].d[i];
            gv += s;
        }
        Model trial = model;
        bool accepted = false;
        for (int t = 0; t < cfg.max_backtracks; ++t) {
            for (std::size_t n = 0; n < order; ++n)
                for (std::size_t i = 0; i < trial.factors[n].d.size(); ++i)
                    trial.factors[n].d[i] = model.factors[n].d[i] + alpha * cg.v[n].d[i];
            const double r_trial = residual_fitness(trial, x, xnorm2, nullptr).first;
            const double f_trial = 0.5 * r_trial * r_trial * xnorm2;
            if (f_trial <= f0 + cfg.c1 * alpha * gv) {
                accepted = true;
                residual_after = r_trial;
                break;
            }
            alpha *= cfg.shrink;
        }
        if (!accepted) {
            diag.armijo_exhausted = true;
            for (std::size_t n = 0; n < order; ++n)
                for (std::size_t i = 0; i < trial.factors[n].d.size(); ++i)
                    trial.factors[n].d[i] = model.factors[n].d[i] + alpha * cg.v[n].d[i];
            residual_after = residual_fitness(trial, x, xnorm2, nullptr).first;
        }
        model = std::move(trial);
    } else {
        for (std::size_t n = 0; n < order; ++n)
            for (std::size_t i = 0; i < model.factors[n].d.size(); ++i)
                model.factors[n].d[i] += cg.v[n].d[i];
    }
    diag.alpha = alpha;
    diag.step_norm = 0.0;
    for (const auto& vn : cg.v) diag.step_norm += alpha * vn.norm();
    for (std::size_t n = 0; n < order; ++n) ws.note_factor_update(n);
    if (!all_finite(model.factors)) numerical("gn_step: non-finite factors after update");
    if (residual_after < 0.0) residual_after = residual_fitness(model, x, xnorm2, nullptr).first;
    diag.residual_after = residual_after;
    diag.stepped = true;
    schedule = schedule_next(schedule);
    return diag;
}

// report.hpp:21-40
struct Record {
    int iteration;
    double residual, fitness, lambda;
    int cg_iters;
    double seconds;
};
enum Status { converged_residual = 0, converged_step = 1, cap_hit = 2, numerical_failure = 3 };

// gauss_newton.cpp:451-494
int gn_optimize(const Tensor& x, Model& model, const GnConfig& cfg, std::vector<Record>& recs) {
    cfg.validate();
    model.validate();
    const double xnorm2 = norm2(x);
    if (!(xnorm2 > 0.0)) invalid("gn_optimize: tensor norm must be positive");
    int status = cap_hit;
    Workspace ws;
    RegSchedule schedule = cfg.schedule;
    const auto t0 = std::chrono::steady_clock::now();
    for (int iter = 1; iter <= cfg.max_iters; ++iter) {
        GnStepDiag d = gn_step(x, model, ws, cfg, schedule, xnorm2);
        if (d.halt == 1) {
            status = converged_residual;
            break;
        }
        if (d.halt == 2) {
            status = converged_step;
            break;
        }
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        recs.push_back({iter, d.residual_after, 1.0 - d.residual_after, d.lambda, d.cg_iters, s});
        if (d.residual_after < cfg.residual_tol) {
            status = converged_residual;
            break;
        }
        if (d.step_norm < cfg.step_tol) {
            status = converged_step;
            break;
        }
    }
    return status;
}

// ---------------------------------------------------------------- ALS
struct AlsConfig {  // als.hpp:11-22
    int max_sweeps = 10000;
    double residual_tol = 5e-5, step_tol = 1e-7, lambda0 = 0.0, decay_factor = 2.0;
    int decay_every = 0;  // 0 = unset
    void validate() const {  // als.cpp:10-20
        if (max_sweeps < 0 || residual_tol < 0 || step_tol < 0 || lambda0 < 0)
            invalid("als config: negative tolerance, cap or lambda");
        if (decay_factor < 1.0) invalid("als config: decay_factor must be >= 1");
        if (decay_every < 0) invalid("als config: decay_every must be positive");
    }
};
struct SweepDiag {
    double step_norm = 0.0;
    int full_contractions = 0;
    Mat last;
};
// als.cpp:22-52
SweepDiag als_sweep(const Tensor& x, Model& model, double lambda, Workspace& ws) {
    model.validate();
    const std::size_t order = model.order();
    ws.full_contractions = 0;
    std::vector<Mat> grams;
    for (const auto& a : model.factors) grams.push_back(gram(a));
    SweepDiag diag;
    for (std::size_t n = 0; n < order; ++n) {
        Mat gamma(model.rank, model.rank, 1.0);
        for (std::size_t m = 0; m < order; ++m)
            if (m != n) gamma = hadamard(gamma, grams[m]);
        Mat mn = mttkrp(x, model.factors, n, ws);
        Mat a_new = spd_solve(gamma, mn, lambda);
        Mat diff = a_new;
        for (std::size_t i = 0; i < diff.d.size(); ++i) diff.d[i] -= model.factors[n].d[i];
        diag.step_norm += diff.norm();
        model.factors[n] = std::move(a_new);
        ws.note_factor_update(n);
        grams[n] = gram(model.factors[n]);
        if (n == order - 1) diag.last = std::move(mn);
    }
    diag.full_contractions = ws.full_contractions;
    return diag;
}
// als.cpp:54-94
int als_optimize(const Tensor& x, Model& model, const AlsConfig& cfg, std::vector<Record>& recs) {
    cfg.validate();
    model.validate();
    const double xnorm2 = norm2(x);
    if (!(xnorm2 > 0.0)) invalid("als_optimize: tensor norm must be positive");
    int status = cap_hit;
    Workspace ws;
    const auto t0 = std::chrono::steady_clock::now();
    for (int sweep = 1; sweep <= cfg.max_sweeps; ++sweep) {
        double lambda = cfg.lambda0;
        if (cfg.decay_every > 0)
            lambda /= std::pow(cfg.decay_factor, static_cast<double>((sweep - 1) / cfg.decay_every));
        SweepDiag d = als_sweep(x, model, lambda, ws);
        auto [res, fit] = residual_fitness(model, x, xnorm2, &d.last);
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        recs.push_back({sweep, res, fit, lambda, 0, s});
        if (res < cfg.residual_tol) {
            status = converged_residual;
            break;
        }
        if (d.step_norm < cfg.step_tol) {
            status = converged_step;
            break;
        }
    }
    return status;
}

}  // namespace orc

// =====================================================================
// C ABI for ctypes (tests / bench baseline only).
// Factor blocks are passed as one concatenated row-major buffer, mode-major.
// =====================================================================
namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const orc::Error& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 7;
    }
}
orc::Tensor make_tensor(const std::uint64_t* dims, int order, const double* data) {
    orc::Tensor t;
    t.dims.assign(dims, dims + order);
    t.size = 1;
    for (int m = 0; m < order; ++m) t.size *= dims[m];
    t.data = data;
    return t;
}
std::vector<orc::Mat> read_blocks(const std::uint64_t* rows, int order, std::int64_t rank,
                                  const double* buf) {
    std::vector<orc::Mat> out;
    std::size_t at = 0;
    for (int m = 0; m < order; ++m) {
        orc::Mat a(static_cast<std::int64_t>(rows[m]), rank);
        std::memcpy(a.d.data(), buf + at, a.d.size() * 8);
        at += a.d.size();
        out.push_back(std::move(a));
    }
    return out;
}
void write_blocks(const std::vector<orc::Mat>& ms, double* buf) {
    std::size_t at = 0;
    for (const auto& m : ms) {
        std::memcpy(buf + at, m.d.data(), m.d.size() * 8);
        at += m.d.size();
    }
}
orc::Model make_model(const std::uint64_t* dims, int order, std::int64_t rank, const double* f) {
    orc::Model m;
    m.dims.assign(dims, dims + order);
    m.rank = rank;
    m.factors = read_blocks(dims, order, rank, f);
    return m;
}
orc::GammaSet read_gamma(int order, std::int64_t rank, const double* grams, const double* pair) {
    orc::GammaSet gs;
    const std::size_t rr = static_cast<std::size_t>(rank * rank);
    for (int n = 0; n < order; ++n) {
        orc::Mat g(rank, rank);
        std::memcpy(g.d.data(), grams + n * rr, rr * 8);
        gs.grams.push_back(g);
    }
    gs.pairwise.assign(order, std::vector<orc::Mat>(order));
    for (int n = 0; n < order; ++n)
        for (int p = 0; p < order; ++p) {
            orc::Mat g(rank, rank);
            std::memcpy(g.d.data(), pair + (n * order + p) * rr, rr * 8);
            gs.pairwise[n][p] = g;
        }
    return gs;
}
}  // namespace

extern "C" {

// Flat GN config mirroring GnConfig (gauss_newton.hpp:50-62).
struct orc_gn_config {
    double grad_tol, residual_tol, step_tol;
    int max_iters;
    double cg_tol;
    int cg_max_iters;
    int reg_mode;   // 0 constant, 1 varying
    int reg_shape;  // 0 identity, 1 diagonal
    double lambda, mu, lower, upper;
    int armijo;
    double c1, shrink;
    int max_backtracks;
    int cg_beta;
};
struct orc_als_config {
    int max_sweeps;
    double residual_tol, step_tol, lambda0, decay_factor;
    int decay_every;
};
struct orc_record {
    int iteration;
    double residual, fitness, lambda;
    int cg_iters;
    double seconds;
};

const char* orc_last_error(void) { return g_err.c_str(); }
void orc_set_threads(int t) { orc::g_threads = t < 1 ? 1 : t; }
int orc_get_threads(void) { return orc::g_threads; }

uint64_t orc_mix64(uint64_t x) { return orc::mix64(x); }
uint64_t orc_keyed(uint64_t s, uint64_t st, uint64_t i, uint64_t salt) { return orc::keyed(s, st, i, salt); }
double orc_uniform(uint64_t s, uint64_t st, uint64_t i, double a, double b) { return orc::uniform(s, st, i, a, b); }
double orc_noise_gaussian(uint64_t seed, uint64_t gidx) {
    return orc::noise_gaussian(orc::derive(orc::mix64(seed), 0x4E01), gidx);
}
int orc_add_noise(const uint64_t* dims, int order, double* x, uint64_t seed, double rel, double* out3) {
    return guarded([&] {
        auto r = orc::add_noise(x, std::vector<std::uint64_t>(dims, dims + order), seed, rel);
        if (out3) std::memcpy(out3, r.data(), 3 * 8);
    });
}
double orc_gaussian(uint64_t s, uint64_t st, uint64_t i) { return orc::gaussian(s, st, i); }
uint64_t orc_problem_seed(uint64_t m, int r, int p) { return orc::problem_seed(m, r, p); }
uint64_t orc_init_seed(uint64_t m, int r, int p, int i) { return orc::init_seed(m, r, p, i); }

// generators.cpp:32-76: kind 0 uniform(a,b), 1 gaussian
int orc_random_model(const uint64_t* dims, int order, int64_t rank, uint64_t seed, int kind, double a,
                     double b, double* out) {
    return guarded([&] {
        if (rank < 1) orc::invalid("random_model: rank must be positive");
        if (kind == 0 && !(a < b)) orc::invalid("random_model: uniform needs a < b");
        std::size_t at = 0;
        for (int n = 0; n < order; ++n)
            for (uint64_t i = 0; i < dims[n]; ++i)
                for (int64_t r = 0; r < rank; ++r) {
                    const uint64_t idx = i * static_cast<uint64_t>(rank) + static_cast<uint64_t>(r);
                    out[at++] = kind == 0 ? orc::uniform(seed, n, idx, a, b) : orc::gaussian(seed, n, idx);
                }
    });
}
int orc_reconstruct(const uint64_t* dims, int order, int64_t rank, const double* factors, double* out) {
    return guarded([&] {
        auto m = make_model(dims, order, rank, factors);
        auto t = orc::reconstruct(m);
        std::memcpy(out, t.data(), t.size() * 8);
    });
}
double orc_norm2(const uint64_t* dims, int order, const double* x) { return orc::norm2(make_tensor(dims, order, x)); }

int orc_mttkrp_naive(const uint64_t* dims, int order, const double* x, int64_t rank,
                     const double* factors, int mode, double* out) {
    return guarded([&] {
        auto t = make_tensor(dims, order, x);
        auto f = read_blocks(dims, order, rank, factors);
        auto m = orc::mttkrp(t, f, static_cast<std::size_t>(mode));
        std::memcpy(out, m.d.data(), m.d.size() * 8);
    });
}
// All modes in ascending order through one workspace (the GN pattern,
// gauss_newton.cpp:366-370). Returns the full-contraction count.
int orc_mttkrp_tree_all(const uint64_t* dims, int order, const double* x, int64_t rank,
                        const double* factors, double* out, int* contractions) {
    return guarded([&] {
        auto t = make_tensor(dims, order, x);
        auto f = read_blocks(dims, order, rank, factors);
        orc::Workspace ws;
        std::vector<orc::Mat> ms;
        for (int n = 0; n < order; ++n) ms.push_back(orc::mttkrp(t, f, static_cast<std::size_t>(n), ws));
        write_blocks(ms, out);
        *contractions = ws.full_contractions;
    });
}
int orc_gram(const double* a, int64_t rows, int64_t cols, double* out) {
    return guarded([&] {
        orc::Mat m(rows, cols);
        std::memcpy(m.d.data(), a, m.d.size() * 8);
        auto g = orc::gram(m);
        std::memcpy(out, g.d.data(), g.d.size() * 8);
    });
}
// grams_out: N*R*R; pair_out: N*N*R*R ([n][p] blocks)
int orc_gamma_set(const uint64_t* dims, int order, int64_t rank, const double* factors,
                  double* grams_out, double* pair_out) {
    return guarded([&] {
        auto m = make_model(dims, order, rank, factors);
        auto gs = orc::build_gamma_set(m);
        const std::size_t rr = static_cast<std::size_t>(rank * rank);
        for (int n = 0; n < order; ++n) std::memcpy(grams_out + n * rr, gs.grams[n].d.data(), rr * 8);
        for (int n = 0; n < order; ++n)
            for (int p = 0; p < order; ++p)
                std::memcpy(pair_out + (n * order + p) * rr, gs.pairwise[n][p].d.data(), rr * 8);
    });
}
// last_mttkrp may be NULL (naive contraction inside, kruskal.cpp:102-105)
int orc_residual(const uint64_t* dims, int order, const double* x, int64_t rank, const double* factors,
                 double xnorm2, const double* last_mttkrp, double* r, double* f) {
    return guarded([&] {
        auto t = make_tensor(dims, order, x);
        auto m = make_model(dims, order, rank, factors);
        orc::Mat last;
        const orc::Mat* lp = nullptr;
        if (last_mttkrp) {
            last = orc::Mat(static_cast<int64_t>(dims[order - 1]), rank);
            std::memcpy(last.d.data(), last_mttkrp, last.d.size() * 8);
            lp = &last;
        }
        auto [rr, ff] = orc::residual_fitness(m, t, xnorm2, lp);
        *r = rr;
        *f = ff;
    });
}
int orc_gradient(const uint64_t* dims, int order, int64_t rank, const double* factors,
                 const double* mttkrps, const double* grams, const double* pair, double* out) {
    return guarded([&] {
        auto m = make_model(dims, order, rank, factors);
        auto mk = read_blocks(dims, order, rank, mttkrps);
        auto gs = read_gamma(order, rank, grams, pair);
        write_blocks(orc::gradient(m, mk, gs), out);
    });
}
int orc_hessian_matvec(const uint64_t* dims, int order, int64_t rank, const double* factors,
                       const double* grams, const double* pair, const double* w, double lambda,
                       int shape, double* out) {
    return guarded([&] {
        auto m = make_model(dims, order, rank, factors);
        auto gs = read_gamma(order, rank, grams, pair);
        auto ww = read_blocks(dims, order, rank, w);
        write_blocks(orc::hessian_matvec(m, gs, ww, lambda, static_cast<orc::RegShape>(shape)), out);
    });
}
int orc_explicit_jtj(const uint64_t* dims, int order, int64_t rank, const double* factors,
                     uint64_t var_cap, double* out) {
    return guarded([&] {
        auto m = make_model(dims, order, rank, factors);
        auto h = orc::explicit_jtj(m, var_cap);
        std::memcpy(out, h.d.data(), h.d.size() * 8);
    });
}
int orc_preconditioner(int order, int64_t rank, const double* grams, const double* pair, double lambda,
                       int shape, double* out) {
    return guarded([&] {
        auto gs = read_gamma(order, rank, grams, pair);
        auto p = orc::build_preconditioner(gs, lambda, static_cast<orc::RegShape>(shape));
        const std::size_t rr = static_cast<std::size_t>(rank * rank);
        for (int n = 0; n < order; ++n) std::memcpy(out + n * rr, p[n].d.data(), rr * 8);
    });
}
int orc_spd_solve(const double* s, int64_t n, const double* b, int64_t rows, double lambda, double* out) {
    return guarded([&] {
        orc::Mat S(n, n), B(rows, n);
        std::memcpy(S.d.data(), s, S.d.size() * 8);
        std::memcpy(B.d.data(), b, B.d.size() * 8);
        auto y = orc::spd_solve(S, B, lambda);
        std::memcpy(out, y.d.data(), y.d.size() * 8);
    });
}
int orc_spd_inverse(const double* s, int64_t n, double lambda, double* out) {
    return guarded([&] {
        orc::Mat S(n, n);
        std::memcpy(S.d.data(), s, S.d.size() * 8);
        auto y = orc::spd_inverse(S, lambda);
        std::memcpy(out, y.d.data(), y.d.size() * 8);
    });
}
static orc::GnConfig gn_cfg(const orc_gn_config* c) {
    orc::GnConfig g;
    g.grad_tol = c->grad_tol;
    g.residual_tol = c->residual_tol;
    g.step_tol = c->step_tol;
    g.max_iters = c->max_iters;
    g.cg_tol = c->cg_tol;
    g.cg_max_iters = c->cg_max_iters;
    g.schedule.mode = static_cast<orc::RegMode>(c->reg_mode);
    g.schedule.shape = static_cast<orc::RegShape>(c->reg_shape);
    g.schedule.lambda = c->lambda;
    g.schedule.mu = c->mu;
    g.schedule.lower = c->lower;
    g.schedule.upper = c->upper;
    g.armijo = c->armijo != 0;
    g.c1 = c->c1;
    g.shrink = c->shrink;
    g.max_backtracks = c->max_backtracks;
    g.cg_beta = c->cg_beta;
    return g;
}
int orc_cp_cg(const uint64_t* dims, int order, int64_t rank, const double* factors, const double* grams,
              const double* pair, const double* g, double lambda, const orc_gn_config* cfg, double* v_out,
              int* iters, int* hit_cap, int* breakdown) {
    return guarded([&] {
        auto m = make_model(dims, order, rank, factors);
        auto gs = read_gamma(order, rank, grams, pair);
        auto gg = read_blocks(dims, order, rank, g);
        auto res = orc::cp_cg(m, gs, gg, lambda, gn_cfg(cfg));
        write_blocks(res.v, v_out);
        *iters = res.iterations;
        *hit_cap = res.hit_cap;
        *breakdown = res.breakdown;
    });
}
// One gn_step on (x, factors) with a fresh workspace; factors updated in place.
// diag_out: [halt, stepped, residual_before, residual_after, grad_norm, lambda,
//            cg_iters, step_norm, alpha, armijo_exhausted, cg_hit_cap, cg_breakdown]
int orc_gn_step(const uint64_t* dims, int order, const double* x, int64_t rank, double* factors,
                const orc_gn_config* cfg, double xnorm2, double* diag_out) {
    return guarded([&] {
        auto t = make_tensor(dims, order, x);
        auto m = make_model(dims, order, rank, factors);
        auto c = gn_cfg(cfg);
        orc::Workspace ws;
        orc::RegSchedule s = c.schedule;
        auto d = orc::gn_step(t, m, ws, c, s, xnorm2);
        write_blocks(m.factors, factors);
        const double vals[12] = {double(d.halt), double(d.stepped), d.residual_before, d.residual_after,
                                 d.grad_norm, d.lambda, double(d.cg_iters), d.step_norm, d.alpha,
                                 double(d.armijo_exhausted), double(d.cg_hit_cap), double(d.cg_breakdown)};
        std::memcpy(diag_out, vals, sizeof vals);
    });
}
// factors in/out; recs must hold max_iters entries; *nrec and *status out.
int orc_gn_optimize(const uint64_t* dims, int order, const double* x, int64_t rank, double* factors,
                    const orc_gn_config* cfg, orc_record* recs, int* nrec, int* status) {
    return guarded([&] {
        auto t = make_tensor(dims, order, x);
        auto m = make_model(dims, order, rank, factors);
        std::vector<orc::Record> rr;
        int st;
        try {
            st = orc::gn_optimize(t, m, gn_cfg(cfg), rr);
        } catch (...) {
            throw;
        }
        write_blocks(m.factors, factors);
        for (std::size_t i = 0; i < rr.size(); ++i)
            recs[i] = {rr[i].iteration, rr[i].residual, rr[i].fitness, rr[i].lambda, rr[i].cg_iters, rr[i].seconds};
        *nrec = static_cast<int>(rr.size());
        *status = st;
    });
}
int orc_als_sweep(const uint64_t* dims, int order, const double* x, int64_t rank, double* factors,
                  double lambda, double* step_norm, int* contractions, double* last_out) {
    return guarded([&] {
        auto t = make_tensor(dims, order, x);
        auto m = make_model(dims, order, rank, factors);
        orc::Workspace ws;
        auto d = orc::als_sweep(t, m, lambda, ws);
        write_blocks(m.factors, factors);
        *step_norm = d.step_norm;
        *contractions = d.full_contractions;
        if (last_out) std::memcpy(last_out, d.last.d.data(), d.last.d.size() * 8);
    });
}
int orc_als_optimize(const uint64_t* dims, int order, const double* x, int64_t rank, double* factors,
                     const orc_als_config* cfg, orc_record* recs, int* nrec, int* status) {
    return guarded([&] {
        auto t = make_tensor(dims, order, x);
        auto m = make_model(dims, order, rank, factors);
        orc::AlsConfig c;
        c.max_sweeps = cfg->max_sweeps;
        c.residual_tol = cfg->residual_tol;
        c.step_tol = cfg->step_tol;
        c.lambda0 = cfg->lambda0;
        c.decay_factor = cfg->decay_factor;
        c.decay_every = cfg->decay_every;
        std::vector<orc::Record> rr;
        int st = orc::als_optimize(t, m, c, rr);
        write_blocks(m.factors, factors);
        for (std::size_t i = 0; i < rr.size(); ++i)
            recs[i] = {rr[i].iteration, rr[i].residual, rr[i].fitness, rr[i].lambda, rr[i].cg_iters, rr[i].seconds};
        *nrec = static_cast<int>(rr.size());
        *status = st;
    });
}
int orc_schedule_next(int mode, double* lambda, double mu, double lower, double upper, int* direction) {
    orc::RegSchedule s;
    s.mode = static_cast<orc::RegMode>(mode);
    s.lambda = *lambda;
    s.mu = mu;
    s.lower = lower;
    s.upper = upper;
    s.direction = *direction;
    s = orc::schedule_next(s);
    *lambda = s.lambda;
    *direction = s.direction;
    return 0;
}

}  // extern "C"
