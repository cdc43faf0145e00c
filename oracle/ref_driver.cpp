// TEST INFRASTRUCTURE ONLY — the CHECKER, never the product.
//
// Compiles the reference's own hot-path headers, unmodified, straight from
// /root/reference/proj/include/sparsegate/ (common.hpp, types.hpp,
// ffn_exec.hpp, synthetic.hpp, parallel.hpp) against oracle/eigen_shim, and
// exports a C ABI so that Python tests can run the real reference executor
// (build recipe: oracle/Makefile, output oracle/_ref/libsgref.so, git-ignored).
//
// Used for: (1) pinning the restatement oracle/sg_oracle.cpp bit-for-bit,
// (2) generating the golden fixtures in tests/golden/ (tests/golden/make_golden.py),
// (3) the `cpu_baseline` / `--impl reference` legs of bench.py (kind
// "reference"), timed with the reference's own parallel_for over tokens
// (parallel.hpp:26-50, as cmd_run does at tools/sparsegate_main.cpp:241).
#include "sparsegate/calibration.hpp"
#include "sparsegate/ffn_exec.hpp"
#include "sparsegate/parallel.hpp"
#include "sparsegate/synthetic.hpp"

#include <chrono>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>

using namespace sparsegate;

namespace {

thread_local std::string g_last_error;

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const DataError& e) {
        g_last_error = e.what();
        return 2;
    } catch (const PropertyViolation& e) {
        g_last_error = e.what();
        return 3;
    } catch (const IoError& e) {
        g_last_error = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return 1;
    }
}

Mat to_mat(const double* p, std::int64_t rows, std::int64_t cols) {
    Mat m(rows, cols);
    if (rows * cols > 0) {
        std::memcpy(m.data(), p, sizeof(double) * static_cast<std::size_t>(rows * cols));
    }
    return m;
}

Vec to_vec(const double* p, std::int64_t n) {
    Vec v(n);
    if (n > 0) {
        std::memcpy(v.data(), p, sizeof(double) * static_cast<std::size_t>(n));
    }
    return v;
}

void from_mat(const Mat& m, double* out) {
    if (m.size() > 0) {
        std::memcpy(out, m.data(), sizeof(double) * static_cast<std::size_t>(m.size()));
    }
}

struct StatsOut {
    double predicted_sparsity;
    double realized_sparsity;
    std::int64_t multiplies;
    std::int32_t pipeline;
    std::int32_t pad;
};

void write_stats(const ExecStats& s, StatsOut* out) {
    if (out == nullptr) {
        return;
    }
    out->predicted_sparsity = s.predicted_sparsity;
    out->realized_sparsity = s.realized_sparsity;
    out->multiplies = s.multiplies;
    out->pipeline = static_cast<std::int32_t>(s.pipeline);
    out->pad = 0;
}

struct RefLayer {
    FfnWeights w;
    Predictor pred;
    bool has_pred = false;
};

}  // namespace

extern "C" {

const char* sgref_last_error() { return g_last_error.c_str(); }

// ---- RNG streams exactly as the reference tests draw them -----------------
void* sgref_rng_new(std::uint64_t seed) { return new std::mt19937_64(seed); }
void sgref_rng_free(void* rng) { delete static_cast<std::mt19937_64*>(rng); }

// test_support.hpp:48-58 (random_matrix) — row-major rows x cols.
void sgref_random_matrix(void* rng, std::int64_t rows, std::int64_t cols, double stddev,
                         double* out) {
    auto& g = *static_cast<std::mt19937_64*>(rng);
    std::normal_distribution<double> dist(0.0, stddev);
    for (std::int64_t i = 0; i < rows * cols; ++i) {
        out[i] = dist(g);
    }
}

// synthetic.hpp:32-42 (random_gaussian), via the reference function itself.
void sgref_random_gaussian(void* rng, std::int64_t rows, std::int64_t cols, double mean,
                           double stddev, double* out) {
    auto& g = *static_cast<std::mt19937_64*>(rng);
    from_mat(random_gaussian(g, rows, cols, mean, stddev), out);
}

double sgref_uniform(void* rng, double a, double b) {
    auto& g = *static_cast<std::mt19937_64*>(rng);
    std::uniform_real_distribution<double> u(a, b);
    return u(g);
}

double sgref_normal_quantile(double p) { return normal_quantile(p); }

// calibration.hpp:61-96 + :128-205 — the reference's own build_instance +
// greedy_calibrate on scores / weights (D x T row-major): bias[D], achieved
// sparsity and total damage. Used to build the reference bench arm's inputs.
int sgref_greedy_calibrate(const double* scores, const double* weights, std::int64_t D,
                           std::int64_t T, int eta, double target, double* bias,
                           double* achieved, double* damage) {
    return guarded([&] {
        Mat s(D, T), w(D, T);
        std::memcpy(s.data(), scores, sizeof(double) * static_cast<std::size_t>(D * T));
        std::memcpy(w.data(), weights, sizeof(double) * static_cast<std::size_t>(D * T));
        const CalibResult r = greedy_calibrate(build_instance(s, w, eta), target);
        for (std::int64_t i = 0; i < D; ++i) bias[i] = r.bias(i);
        if (achieved) *achieved = r.achieved_sparsity;
        if (damage) *damage = r.total_damage;
    });
}

// synthetic.hpp:80-108. Outputs row-major: gate DxH, up DxH, down HxD,
// calib H x calib_tokens, eval H x eval_tokens (any output may be NULL).
int sgref_synthetic(std::int64_t hidden, std::int64_t inter, std::int64_t calib_tokens,
                    std::int64_t eval_tokens, int activation, double natural_sparsity,
                    std::uint64_t seed, double* gate, double* up, double* down, double* calib,
                    double* eval) {
    return guarded([&] {
        SyntheticConfig cfg;
        cfg.hidden = hidden;
        cfg.inter = inter;
        cfg.calib_tokens = calib_tokens;
        cfg.eval_tokens = eval_tokens;
        cfg.activation = activation == 1 ? Activation::DReLU : Activation::ReGLU;
        cfg.natural_sparsity = natural_sparsity;
        cfg.seed = seed;
        const SyntheticFixture f = make_synthetic_fixture(cfg);
        if (gate) from_mat(f.weights.gate, gate);
        if (up) from_mat(f.weights.up, up);
        if (down) from_mat(f.weights.down, down);
        if (calib) from_mat(f.calib.x_cols, calib);
        if (eval) from_mat(f.eval.x_cols, eval);
    });
}

// ---- executor (ffn_exec.hpp) ---------------------------------------------
void* sgref_layer_new(std::int64_t d, std::int64_t D, int activation, const double* gate,
                      const double* up, const double* down, std::int64_t r, const double* A,
                      const double* B, const double* bias) {
    auto* L = new RefLayer;
    L->w.gate = to_mat(gate, D, d);
    L->w.up = to_mat(up, D, d);
    L->w.down = to_mat(down, d, D);
    L->w.activation = activation == 1 ? Activation::DReLU : Activation::ReGLU;
    if (A != nullptr && B != nullptr && bias != nullptr) {
        L->pred.A = to_mat(A, D, r);
        L->pred.B = to_mat(B, r, d);
        L->pred.bias = to_vec(bias, D);
        L->pred.rank = r;
        L->has_pred = true;
    }
    return L;
}

void sgref_layer_free(void* layer) { delete static_cast<RefLayer*>(layer); }

// pipeline: 0 dense, 1 parallel, 2 sequential (ffn_exec.hpp:32 enum order).
// Runs `tokens` columns of xs (token-major: tokens x d) with the reference's
// parallel_for; ys is tokens x d. Returns wall seconds through *elapsed.
int sgref_layer_run(void* layer, int pipeline, const double* xs, std::int64_t tokens,
                    double* ys, StatsOut* stats, double* elapsed) {
    auto* L = static_cast<RefLayer*>(layer);
    return guarded([&] {
        const std::int64_t d = L->w.gate.cols();
        if (pipeline != 0 && !L->has_pred) {
            throw std::invalid_argument("layer has no predictor");
        }
        std::vector<FfnResult> results(static_cast<std::size_t>(tokens));
        std::vector<std::string> errors(static_cast<std::size_t>(tokens));
        const auto t0 = std::chrono::steady_clock::now();
        parallel_for(static_cast<std::size_t>(tokens), [&](std::size_t t) {
            try {
                const Vec x = to_vec(xs + t * d, d);
                if (pipeline == 0) {
                    results[t] = dense_ffn(L->w, x);
                } else if (pipeline == 1) {
                    results[t] = sparse_ffn_parallel(L->w, L->pred, x);
                } else {
                    results[t] = sparse_ffn_sequential(L->w, L->pred, x);
                }
            } catch (const std::exception& e) {
                errors[t] = e.what();
            }
        });
        const auto t1 = std::chrono::steady_clock::now();
        if (elapsed) *elapsed = std::chrono::duration<double>(t1 - t0).count();
        for (std::size_t t = 0; t < errors.size(); ++t) {
            if (!errors[t].empty()) {
                throw DataError(errors[t]);
            }
        }
        for (std::int64_t t = 0; t < tokens; ++t) {
            if (ys) std::memcpy(ys + t * d, results[t].y.data(), sizeof(double) * d);
            if (stats) write_stats(results[t].stats, stats + t);
        }
    });
}

int sgref_dense_ffn(std::int64_t d, std::int64_t D, int activation, const double* gate,
                    const double* up, const double* down, const double* x, std::int64_t x_len,
                    double* y, StatsOut* stats) {
    return guarded([&] {
        FfnWeights w;
        w.gate = to_mat(gate, D, d);
        w.up = to_mat(up, D, d);
        w.down = to_mat(down, d, D);
        w.activation = activation == 1 ? Activation::DReLU : Activation::ReGLU;
        const FfnResult r = dense_ffn(w, to_vec(x, x_len));
        std::memcpy(y, r.y.data(), sizeof(double) * static_cast<std::size_t>(r.y.size()));
        write_stats(r.stats, stats);
    });
}

int sgref_sparse_ffn(int pipeline, std::int64_t d, std::int64_t D, int activation,
                     const double* gate, const double* up, const double* down, std::int64_t r,
                     std::int64_t rank_field, const double* A, const double* B,
                     const double* bias, const double* x, std::int64_t x_len, double* y,
                     StatsOut* stats) {
    return guarded([&] {
        FfnWeights w;
        w.gate = to_mat(gate, D, d);
        w.up = to_mat(up, D, d);
        w.down = to_mat(down, d, D);
        w.activation = activation == 1 ? Activation::DReLU : Activation::ReGLU;
        Predictor p;
        p.A = to_mat(A, D, r);
        p.B = to_mat(B, r, d);
        p.bias = to_vec(bias, D);
        p.rank = rank_field;
        const Vec xv = to_vec(x, x_len);
        const FfnResult res = pipeline == 1 ? sparse_ffn_parallel(w, p, xv)
                                            : sparse_ffn_sequential(w, p, xv);
        std::memcpy(y, res.y.data(), sizeof(double) * static_cast<std::size_t>(res.y.size()));
        write_stats(res.stats, stats);
    });
}

int sgref_predict_mask(std::int64_t d, std::int64_t D, std::int64_t r, std::int64_t rank_field,
                       const double* A, const double* B, const double* bias, const double* x,
                       std::int64_t x_len, std::uint8_t* mask, std::int64_t* count) {
    return guarded([&] {
        Predictor p;
        p.A = to_mat(A, D, r);
        p.B = to_mat(B, r, d);
        p.bias = to_vec(bias, D);
        p.rank = rank_field;
        const Mask m = predict_mask(p, to_vec(x, x_len));
        std::memcpy(mask, m.active.data(), m.active.size());
        *count = m.predicted_active_count;
    });
}

int sgref_op_count_model(std::int64_t d, std::int64_t D, std::int64_t r, double s,
                         double s_prime, std::int64_t* dense, double* sparse, double* ratio) {
    return guarded([&] {
        const OpCounts c = op_count_model(d, D, r, s, s_prime);
        *dense = c.dense;
        *sparse = c.sparse;
        *ratio = c.ratio;
    });
}

double sgref_det_dot(const double* a, const double* b, std::int64_t n) {
    return det_dot(a, b, static_cast<std::size_t>(n));
}

double sgref_det_sum(const double* v, std::int64_t n) {
    return det_sum(v, static_cast<std::size_t>(n));
}

unsigned sgref_thread_budget() { return thread_budget(); }

}  // extern "C"
