// TEST INFRASTRUCTURE ONLY — the CHECKER, never the product.
//
// CPU restatement (f64, plain C++, no Eigen) of the reference's sparse-FFN
// executor path. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline leg may load this library (oracle/liboracle.so); the product
// (paper_2603_14110_b200/) never links or calls it.
//
// Follows, line for line:
//   /root/reference/proj/include/sparsegate/common.hpp:52-95   det_sum/det_dot/tree_sum, relu
//   /root/reference/proj/include/sparsegate/types.hpp:31-105   validation semantics
//   /root/reference/proj/include/sparsegate/ffn_exec.hpp:56-244 executors, stats, op counts
//   /root/reference/proj/include/sparsegate/synthetic.hpp:15-108 fixtures (same RNG call order)
//
// It adds what the reference does not return: the predicted index set P and
// the gate-revalidated survivor set V, plus the f64 pre-activations and their
// absolute-value scales used to classify near-threshold neurons.
//
// Pinning: tests/test_oracle.py checks this file bit-for-bit against the real
// reference headers compiled into oracle/_ref/libsgref.so (oracle/ref_driver.cpp)
// and against the committed golden vectors in tests/golden/.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <vector>

namespace {

thread_local std::string g_last_error;

constexpr std::size_t kReduceBlock = 64;  // common.hpp:52

// common.hpp:56-65
double tree_sum(const double* v, std::size_t n) {
    if (n == 0) return 0.0;
    if (n == 1) return v[0];
    const std::size_t half = n / 2;
    return tree_sum(v, half) + tree_sum(v + half, n - half);
}

// common.hpp:70-76
double det_sum(const double* v, std::size_t n) {
    double total = 0.0;
    for (std::size_t base = 0; base < n; base += kReduceBlock) {
        total += tree_sum(v + base, std::min(kReduceBlock, n - base));
    }
    return total;
}

// common.hpp:79-90
double det_dot(const double* a, const double* b, std::size_t n) {
    double buf[kReduceBlock];
    double total = 0.0;
    for (std::size_t base = 0; base < n; base += kReduceBlock) {
        const std::size_t m = std::min(kReduceBlock, n - base);
        for (std::size_t j = 0; j < m; ++j) buf[j] = a[base + j] * b[base + j];
        total += tree_sum(buf, m);
    }
    return total;
}

bool all_finite(const double* p, std::int64_t n) {
    for (std::int64_t i = 0; i < n; ++i) {
        if (!std::isfinite(p[i])) return false;
    }
    return true;
}

struct Fail {
    int code;  // 2 DataError, 3 PropertyViolation (common.hpp:20-37)
    std::string msg;
};

// ffn_exec.hpp:68-76
double gated_value(double g, double u, int act) {
    if (g <= 0.0) return 0.0;
    if (act == 1 && u <= 0.0) return 0.0;
    return g * u;
}

struct Weights {
    std::int64_t d, D;
    int act;
    const double* gate;  // D x d
    const double* up;    // D x d
    const double* down;  // d x D (reference layout, types.hpp:19-24)
};

struct Pred {
    std::int64_t r, rank_field;
    const double* A;  // D x r
    const double* B;  // r x d
    const double* bias;
};

// types.hpp:31-51 + ffn_exec.hpp:56-65 (shapes are implied by the C ABI;
// the finiteness scans run on every call exactly like the reference).
void check_input(const Weights& w, const double* x, std::int64_t x_len, bool scan) {
    if (w.d < 1 || w.D < 1) throw Fail{2, "ffn weights: gate must be at least 1x1"};
    if (scan && (!all_finite(w.gate, w.D * w.d) || !all_finite(w.up, w.D * w.d) ||
                 !all_finite(w.down, w.D * w.d))) {
        throw Fail{2, "ffn weights: non-finite entries"};
    }
    if (x_len != w.d) throw Fail{2, "ffn input length does not match hidden size"};
    if (!all_finite(x, x_len)) throw Fail{2, "ffn input has non-finite entries"};
}

// types.hpp:82-105
void validate_pred(const Pred& p, std::int64_t d, std::int64_t D, bool scan) {
    if (p.rank_field != p.r) throw Fail{2, "predictor: rank field disagrees with factor shapes"};
    if (p.r < 1 || p.r > std::min(D, d)) throw Fail{2, "predictor: rank out of range"};
    if (scan && (!all_finite(p.A, D * p.r) || !all_finite(p.B, p.r * d))) {
        throw Fail{2, "predictor: non-finite factor entries"};
    }
}

// ffn_exec.hpp:80-94 — y_j = det_sum_k (z_k == 0 ? +0 : z_k * down[j, idx_k]).
void down_project(const Weights& w, const std::vector<std::int64_t>& idx,
                  const std::vector<double>& z, double* y) {
    const std::size_t n = idx.size();
    std::vector<double> terms(n);
    for (std::int64_t j = 0; j < w.d; ++j) {
        const double* row = w.down + j * w.D;
        for (std::size_t k = 0; k < n; ++k) terms[k] = z[k] == 0.0 ? 0.0 : z[k] * row[idx[k]];
        y[j] = det_sum(terms.data(), n);
    }
}

// ffn_exec.hpp:125-146. Also returns pre (f64) per neuron when asked.
std::int64_t predict_mask(const Pred& p, std::int64_t d, std::int64_t D, const double* x,
                          std::int64_t x_len, bool scan, std::uint8_t* mask, double* pre_out) {
    validate_pred(p, d, D, scan);
    if (x_len != d) throw Fail{2, "predictor input length does not match hidden size"};
    std::vector<double> t(static_cast<std::size_t>(p.r));
    for (std::int64_t j = 0; j < p.r; ++j) t[j] = det_dot(p.B + j * d, x, d);
    std::int64_t count = 0;
    for (std::int64_t i = 0; i < D; ++i) {
        const double pre = det_dot(p.A + i * p.r, t.data(), p.r) + p.bias[i];
        const bool on = pre > 0.0;  // strict, ffn_exec.hpp:141
        mask[i] = on ? 1 : 0;
        count += on ? 1 : 0;
        if (pre_out) pre_out[i] = pre;
    }
    return count;
}

struct Stats {
    double predicted_sparsity;
    double realized_sparsity;
    std::int64_t multiplies;
    std::int32_t pipeline;  // 0 dense, 1 parallel, 2 sequential
    std::int32_t pad;
};

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const Fail& f) {
        g_last_error = f.msg;
        return f.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return 1;
    }
}

}  // namespace

extern "C" {

const char* sgo_last_error() { return g_last_error.c_str(); }

double sgo_det_dot(const double* a, const double* b, std::int64_t n) {
    return det_dot(a, b, static_cast<std::size_t>(n));
}
double sgo_det_sum(const double* v, std::int64_t n) {
    return det_sum(v, static_cast<std::size_t>(n));
}

// ffn_exec.hpp:103-122
int sgo_dense_ffn(std::int64_t d, std::int64_t D, int act, const double* gate, const double* up,
                  const double* down, const double* x, std::int64_t x_len, int scan, double* y,
                  Stats* stats) {
    return guarded([&] {
        const Weights w{d, D, act, gate, up, down};
        check_input(w, x, x_len, scan != 0);
        std::vector<std::int64_t> idx(static_cast<std::size_t>(D));
        std::vector<double> z(static_cast<std::size_t>(D));
        for (std::int64_t i = 0; i < D; ++i) {
            idx[i] = i;
            const double g = det_dot(gate + i * d, x, d);
            const double u = det_dot(up + i * d, x, d);
            z[i] = gated_value(g, u, act);
        }
        down_project(w, idx, z, y);
        if (stats) *stats = Stats{0.0, 0.0, 3 * d * D, 0, 0};
    });
}

int sgo_predict_mask(std::int64_t d, std::int64_t D, std::int64_t r, std::int64_t rank_field,
                     const double* A, const double* B, const double* bias, const double* x,
                     std::int64_t x_len, std::uint8_t* mask, std::int64_t* count, double* pre) {
    return guarded([&] {
        const Pred p{r, rank_field, A, B, bias};
        *count = predict_mask(p, d, D, x, x_len, true, mask, pre);
    });
}

// ffn_exec.hpp:149-178 (pipeline 1) and :183-218 (pipeline 2). Extra outputs
// (any may be NULL): P[p] ascending predicted-active indices, V[v] ascending
// gate-revalidated survivors (sequential; equals {k in P: g_k > 0} for
// parallel too), g[p] gate pre-activations over P, z[p] gated values over P.
int sgo_sparse_ffn(int pipeline, std::int64_t d, std::int64_t D, int act, const double* gate,
                   const double* up, const double* down, std::int64_t r, std::int64_t rank_field,
                   const double* A, const double* B, const double* bias, const double* x,
                   std::int64_t x_len, int scan, double* y, Stats* stats, std::int32_t* P_out,
                   std::int64_t* p_out, std::int32_t* V_out, std::int64_t* v_out, double* g_out,
                   double* z_out) {
    return guarded([&] {
        const Weights w{d, D, act, gate, up, down};
        check_input(w, x, x_len, scan != 0);
        const Pred pr{r, rank_field, A, B, bias};
        std::vector<std::uint8_t> mask(static_cast<std::size_t>(D));
        predict_mask(pr, d, D, x, x_len, scan != 0, mask.data(), nullptr);
        std::vector<std::int64_t> idx;  // stage 2 compaction, ffn_exec.hpp:189-195
        for (std::int64_t i = 0; i < D; ++i) {
            if (mask[i]) idx.push_back(i);
        }
        std::vector<double> z(idx.size(), 0.0);
        std::int64_t revalidated = 0;
        std::int64_t nv = 0;
        for (std::size_t k = 0; k < idx.size(); ++k) {
            const double g = det_dot(gate + idx[k] * d, x, d);
            if (g_out) g_out[k] = g;
            if (pipeline == 1) {  // ffn_exec.hpp:163-167: no revalidation
                const double u = det_dot(up + idx[k] * d, x, d);
                z[k] = gated_value(g, u, act);
            } else if (g > 0.0) {  // ffn_exec.hpp:196-205
                ++revalidated;
                const double u = det_dot(up + idx[k] * d, x, d);
                z[k] = gated_value(g, u, act);
            }
            if (g > 0.0 && V_out) V_out[nv] = static_cast<std::int32_t>(idx[k]);
            if (g > 0.0) ++nv;
            if (P_out) P_out[k] = static_cast<std::int32_t>(idx[k]);
        }
        if (z_out) std::copy(z.begin(), z.end(), z_out);
        down_project(w, idx, z, y);
        const auto predicted = static_cast<std::int64_t>(idx.size());
        Stats s{};
        s.predicted_sparsity = 1.0 - static_cast<double>(predicted) / static_cast<double>(D);
        if (pipeline == 1) {  // ffn_exec.hpp:173-180
            s.multiplies = r * (d + D) + 3 * d * predicted;
            s.realized_sparsity = s.predicted_sparsity;
            s.pipeline = 1;
        } else {  // ffn_exec.hpp:209-216
            s.multiplies = r * (d + D) + d * predicted + 2 * d * revalidated;
            s.realized_sparsity =
                1.0 - static_cast<double>(revalidated) / static_cast<double>(D);
            s.pipeline = 2;
        }
        if (stats) *stats = s;
        if (p_out) *p_out = predicted;
        if (v_out) *v_out = nv;
    });
}

// ffn_exec.hpp:229-244
int sgo_op_count_model(std::int64_t d, std::int64_t D, std::int64_t r, double s, double sp,
                       std::int64_t* dense, double* sparse, double* ratio) {
    return guarded([&] {
        if (d < 1 || D < 1 || r < 0) {
            throw Fail{2, "op count model: dimensions must be positive and rank nonnegative"};
        }
        if (!(0.0 <= s && s <= sp && sp <= 1.0)) throw Fail{2, "op count model: need 0 <= s <= s' <= 1"};
        *dense = 3 * d * D;
        *sparse = static_cast<double>(r) * static_cast<double>(d + D) +
                  static_cast<double>(d) * (1.0 - s) * static_cast<double>(D) +
                  2.0 * static_cast<double>(d) * (1.0 - sp) * static_cast<double>(D);
        *ratio = static_cast<double>(*dense) / *sparse;
    });
}

// Near-threshold scales (not in the reference):
//   pre_scale_i = sum_j |A_ij| * (sum_k |B_jk x_k|) + |bias_i|   (finite bias only)
//   gate_scale_i = sum_k |gate_ik x_k|
// An index-set disagreement between the GPU (fp32 accumulation) and this f64
// oracle is admissible only where |pre_i| <= eps * pre_scale_i (for P) or
// |g_i| <= eps * gate_scale_i (for V).
void sgo_threshold_scales(std::int64_t d, std::int64_t D, std::int64_t r, const double* A,
                          const double* B, const double* bias, const double* gate,
                          const double* x, double* pre_scale, double* gate_scale) {
    std::vector<double> tabs(static_cast<std::size_t>(r), 0.0);
    for (std::int64_t j = 0; j < r; ++j) {
        double s = 0.0;
        for (std::int64_t k = 0; k < d; ++k) s += std::fabs(B[j * d + k] * x[k]);
        tabs[j] = s;
    }
    for (std::int64_t i = 0; i < D; ++i) {
        if (pre_scale) {
            double s = std::isfinite(bias[i]) ? std::fabs(bias[i]) : 0.0;
            for (std::int64_t j = 0; j < r; ++j) s += std::fabs(A[i * r + j]) * tabs[j];
            pre_scale[i] = s;
        }
        if (gate_scale) {
            double s = 0.0;
            for (std::int64_t k = 0; k < d; ++k) s += std::fabs(gate[i * d + k] * x[k]);
            gate_scale[i] = s;
        }
    }
}

// ---- synthetic.hpp:15-108 restated ---------------------------------------
double sgo_normal_quantile(double p) {
    if (!(p > 0.0 && p < 1.0)) return std::nan("");
    double z = 0.0;
    for (int iter = 0; iter < 60; ++iter) {
        const double cdf = 0.5 * std::erfc(-z / std::sqrt(2.0));
        const double pdf = std::exp(-0.5 * z * z) / std::sqrt(2.0 * M_PI);
        const double step = (cdf - p) / pdf;
        z -= step;
        if (std::abs(step) < 1e-14) break;
    }
    return z;
}

static void fill_gaussian(std::mt19937_64& rng, std::int64_t n, double mean, double stddev,
                          double* out) {
    std::normal_distribution<double> dist(mean, stddev);  // fresh per matrix, synthetic.hpp:34
    for (std::int64_t i = 0; i < n; ++i) {
        const double v = dist(rng);
        if (out) out[i] = v;
    }
}

int sgo_synthetic(std::int64_t hidden, std::int64_t inter, std::int64_t calib_tokens,
                  std::int64_t eval_tokens, int /*activation*/, double natural_sparsity,
                  std::uint64_t seed, double* gate, double* up, double* down, double* calib,
                  double* eval) {
    return guarded([&] {
        if (hidden < 1 || inter < 1 || calib_tokens < 1 || eval_tokens < 0) {
            throw Fail{2, "synthetic fixture: invalid sizes"};
        }
        if (!(natural_sparsity > 0.0 && natural_sparsity < 1.0)) {
            throw Fail{2, "synthetic fixture: natural sparsity must lie in (0, 1)"};
        }
        const auto d = static_cast<double>(hidden);
        const double z = sgo_normal_quantile(natural_sparsity);
        double shift = z * std::sqrt(2.0);
        shift = z * std::sqrt(2.0 + shift * shift / d);
        std::mt19937_64 rng(seed);
        fill_gaussian(rng, inter * hidden, -shift / d, 1.0 / std::sqrt(d), gate);
        fill_gaussian(rng, inter * hidden, 0.0, 1.0 / std::sqrt(d), up);
        fill_gaussian(rng, hidden * inter, 0.0, 1.0 / std::sqrt(static_cast<double>(inter)), down);
        fill_gaussian(rng, hidden * calib_tokens, 1.0, 1.0, calib);
        fill_gaussian(rng, hidden * eval_tokens, 1.0, 1.0, eval);
    });
}

}  // extern "C"
