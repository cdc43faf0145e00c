// sparsegate-b200 — drop-in for /root/reference/proj/include/sparsegate/factorization.hpp
// (data-whitened truncated-SVD predictor construction, factorization.hpp:18-157),
// implemented over the C ABI's offline producer (csrc/sg_offline.cu: the large
// products on the GPU, no Eigen). Same names, argument meaning and DataError cases.
//
// SVD: the reference's Eigen BDCSVD is exact. Here min(D, d) <= 1024 (and
// D * d <= 4M) runs the exact one-sided Jacobi SVD on the host; larger shapes the
// randomized rank-(r+32) range finder (4 power iterations) on the GPU, so spectral.singular_values then
// holds the leading rank + 1 values only.
#pragma once

#include "sparsegate/types.hpp"
#include "sparsegate_c.h"

#include <array>
#include <string>
#include <utility>
#include <vector>

namespace sparsegate {

struct WhiteningResult {
    Mat S;
    Mat S_inv;
    double lambda = 0.0;
};

// factorization.hpp:26-29: lambda = m * epsilon * mu, mu = trace(X X^T) / d.
struct DampingPolicy {
    double epsilon = 1e-10;
    std::array<double, 4> multipliers{0.0, 1.0, 10.0, 100.0};
};

namespace fdetail {
inline void check(sg_status s) {
    if (s == SG_OK) return;
    const std::string msg = sg_last_error();
    if (s == SG_ERR_DATA) throw DataError(msg);
    if (s == SG_ERR_PROPERTY) throw PropertyViolation(msg);
    throw DeviceError(msg);
}
inline bool exact_ok(Index rows, Index cols) {
    return std::min(rows, cols) <= 1024 && rows * cols <= 4'000'000;
}
}  // namespace fdetail

inline WhiteningResult cholesky_whitening(const ActivationBatch& X, const DampingPolicy& policy = {}) {
    validate(X);
    const Index d = X.hidden_size();
    WhiteningResult r;
    r.S = Mat(d, d);
    r.S_inv = Mat(d, d);
    fdetail::check(sg_cholesky_whitening(X.x_cols.data(), d, X.tokens(), policy.epsilon, policy.multipliers.data(),
                                         static_cast<int32_t>(policy.multipliers.size()), r.S.data(),
                                         r.S_inv.data(), &r.lambda));
    return r;
}

enum class WhiteningMode { Whitened, Naive };

struct SpectralInfo {
    Vec singular_values;
    double sigma_r_plus_1 = 0.0;
};

struct BuildResult {
    Predictor predictor;
    SpectralInfo spectral;
    WhiteningMode mode = WhiteningMode::Whitened;
    double lambda = 0.0;
};

namespace detail {
inline Vec singular_values_of(const Mat& m) {
    const bool exact = fdetail::exact_ok(m.rows(), m.cols());
    const Index k = exact ? std::min(m.rows(), m.cols()) : std::min<Index>(std::min(m.rows(), m.cols()), 64);
    Vec s(k);
    fdetail::check(sg_singular_values(m.data(), m.rows(), m.cols(), exact ? 0 : 1, k, 0, s.data()));
    return s;
}
}  // namespace detail

// factorization.hpp:93-144: A = U_r Σ_r, B = V_r^T S^-1 (whitened) or V_r^T (naive).
inline BuildResult build_predictor(const Mat& w_gate, const ActivationBatch& X, Index rank,
                                   WhiteningMode mode = WhiteningMode::Whitened, const DampingPolicy& policy = {}) {
    const Index D = w_gate.rows(), d = w_gate.cols();
    if (rank < 1 || rank > std::min(D, d))
        throw DataError("predictor rank " + std::to_string(rank) + " out of range [1, " +
                        std::to_string(std::min(D, d)) + "]");
    if (!all_finite(w_gate)) throw DataError("gate matrix has non-finite entries");
    const bool whitened = mode == WhiteningMode::Whitened;
    if (whitened && X.hidden_size() != d)
        throw DataError("calibration batch hidden size " + std::to_string(X.hidden_size()) +
                        " does not match gate columns " + std::to_string(d));
    if (whitened) validate(X);
    const bool exact = fdetail::exact_ok(D, d);
    const Index n_sv = exact ? std::min(D, d) : std::min(std::min(D, d), rank + 1);
    BuildResult out;
    out.mode = mode;
    Predictor& p = out.predictor;
    p.A = Mat(D, rank);
    p.B = Mat(rank, d);
    p.bias = Vec::Zero(D);
    p.rank = rank;
    out.spectral.singular_values = Vec(n_sv);
    fdetail::check(sg_build_predictor(w_gate.data(), D, d, whitened ? X.x_cols.data() : nullptr,
                                      whitened ? X.tokens() : 0, rank, whitened ? 1 : 0, exact ? 0 : 1, 0,
                                      policy.epsilon, policy.multipliers.data(),
                                      static_cast<int32_t>(policy.multipliers.size()), p.A.data(), p.B.data(),
                                      out.spectral.singular_values.data(), n_sv, &out.spectral.sigma_r_plus_1,
                                      &out.lambda));
    return out;
}

// factorization.hpp:147-155: largest singular value of W - A B.
inline double residual_spectral_norm(const Mat& w, const Predictor& pred) {
    if (pred.A.rows() != w.rows() || pred.B.cols() != w.cols())
        throw DataError("residual: predictor shape does not match weight matrix");
    const Mat residual = w - pred.A * pred.B;
    const bool exact = fdetail::exact_ok(residual.rows(), residual.cols());
    double s = 0.0;
    fdetail::check(sg_singular_values(residual.data(), residual.rows(), residual.cols(), exact ? 0 : 1, 1, 0, &s));
    return s;
}

}  // namespace sparsegate
