// sparsegate-b200 — C++ drop-in for the reference executor API
//   /root/reference/proj/include/sparsegate/ffn_exec.hpp (+ types.hpp, common.hpp)
// implemented over the C ABI (include/sparsegate_c.h, libsparsegate_b200.so).
//
// Same names, argument meaning and error behaviour as the reference:
//   dense_ffn              ffn_exec.hpp:103-122
//   predict_mask           ffn_exec.hpp:125-146
//   sparse_ffn_parallel    ffn_exec.hpp:149-178
//   sparse_ffn_sequential  ffn_exec.hpp:183-218
//   op_count_model         ffn_exec.hpp:229-244
//   gating_error           ffn_exec.hpp:256-285
//   FfnWeights / Predictor / validate   types.hpp:21-105
//   Error / IoError / DataError / PropertyViolation   common.hpp:20-37
// Mat / Vec / the domain types come from sparsegate/common.hpp and types.hpp:
// the reference's own Eigen types when <Eigen/Dense> is available, minimal
// stand-ins otherwise. Values are f64 on the host; the device computes with bf16
// weights and fp32 arithmetic.
//
// The reference functions are stateless. A GPU needs resident weights, so the
// stateless calls here keep a per-thread cache of device layers keyed by the
// weight / predictor buffers (address, shape and a digest of their full
// contents: an in-place change re-uploads — and re-validates — the layer, as the
// reference validates on every call), or use the explicit
// sparsegate::gpu::Layer / Context objects.
#pragma once

#include "sparsegate/types.hpp"
#include "sparsegate_c.h"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

namespace sparsegate {

namespace detail {
inline void check(sg_status s) {
    if (s == SG_OK) return;
    const std::string msg = sg_last_error();
    switch (s) {
        case SG_ERR_DATA: throw DataError(msg);
        case SG_ERR_PROPERTY: throw PropertyViolation(msg);
        case SG_ERR_IO: throw IoError(msg);
        default: throw DeviceError(msg);
    }
}
}  // namespace detail

// ---- executor types (ffn_exec.hpp:27-52) ----
struct Mask {
    std::vector<std::uint8_t> active;
    Index predicted_active_count = 0;
};

enum class Pipeline { Dense, Parallel, Sequential };
inline std::string to_string(Pipeline p) {
    switch (p) {
        case Pipeline::Dense: return "dense";
        case Pipeline::Parallel: return "parallel";
        default: return "sequential";
    }
}

struct ExecStats {
    double predicted_sparsity = 0.0;
    double realized_sparsity = 0.0;
    std::int64_t multiplies = 0;
    Pipeline pipeline = Pipeline::Dense;
};

struct FfnResult {
    Vec y;
    ExecStats stats;
};

struct OpCounts {
    std::int64_t dense = 0;
    double sparse = 0.0;
    double ratio = 0.0;
};

struct GatingError {
    double error_norm = 0.0;
    double relative = 0.0;
};

// ---- explicit device objects ----
namespace gpu {

class Context {
   public:
    Context(int device, Index max_hidden, Index max_inter, Index max_rank) {
        detail::check(sg_ctx_create(device, max_hidden, max_inter, max_rank, &ctx_));
    }
    ~Context() {
        if (ctx_) sg_ctx_destroy(ctx_);
    }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    sg_ctx* get() const { return ctx_; }

   private:
    sg_ctx* ctx_ = nullptr;
};

// One layer (or d_ff shard) resident in HBM. w and/or pred may be null.
class Layer {
   public:
    Layer(const FfnWeights* w, const Predictor* pred, int device = 0, int shard_index = 0,
          int shard_count = 1, bool interleave = false) {
        sg_layer_desc d{};
        if (w) {
            validate(*w);
            d.hidden = w->hidden_size();
            d.inter = w->inter_size();
            d.activation = w->activation == Activation::DReLU ? SG_DRELU : SG_REGLU;
            d.gate = w->gate.data();
            d.up = w->up.data();
            d.down = w->down.data();
        }
        if (pred) {
            validate(*pred);
            if (w && pred->hidden_size() != w->hidden_size())
                throw DataError("predictor input length does not match hidden size");
            if (w && pred->inter_size() != w->inter_size())
                throw DataError("predictor intermediate size does not match weights");
            d.hidden = pred->hidden_size();
            d.inter = pred->inter_size();
            d.rank = pred->rank;
            d.pred_A = pred->A.data();
            d.pred_B = pred->B.data();
            d.bias = pred->bias.data();
            d.bias_dtype = SG_F64;
        }
        if (!w && !pred) throw DataError("layer needs weights and/or a predictor");
        d.weight_dtype = SG_F64;
        d.device = device;
        d.shard_index = shard_index;
        d.shard_count = shard_count;
        d.shard_interleave = interleave ? 1 : 0;
        detail::check(sg_layer_create(&d, &layer_));
        hidden_ = d.hidden;
        inter_ = d.inter;
        rank_ = d.rank;
        device_ = device;
    }
    ~Layer() {
        if (layer_) sg_layer_destroy(layer_);
    }
    Layer(const Layer&) = delete;
    Layer& operator=(const Layer&) = delete;

    sg_layer* get() const { return layer_; }
    Index hidden() const { return hidden_; }
    Index inter() const { return inter_; }
    Index local_inter() const { return sg_layer_local_inter(layer_); }
    Index rank() const { return rank_; }
    int device() const { return device_; }
    // Gate rows of the first `rows` neurons of every CTA block fetched before the
    // mask (sg_layer_set_hot_rows): timing only, results unchanged.
    void set_hot_rows(Index rows) { detail::check(sg_layer_set_hot_rows(layer_, rows)); }

    // Host x (f64) -> host y (f64) and the reference's ExecStats.
    FfnResult forward(Context& ctx, Pipeline p, const Vec& x, void* stream = nullptr) const {
        FfnResult r;
        r.y = Vec(hidden_);
        sg_exec_stats st{};
        detail::check(sg_ffn_forward(ctx.get(), layer_, static_cast<sg_pipeline>(p), x.data(), SG_F64,
                                     x.size(), r.y.data(), SG_F64, &st, stream));
        r.stats.predicted_sparsity = st.predicted_sparsity;
        r.stats.realized_sparsity = st.realized_sparsity;
        r.stats.multiplies = st.multiplies;
        r.stats.pipeline = static_cast<Pipeline>(st.pipeline);
        return r;
    }

    Mask predict(Context& ctx, const Vec& x, void* stream = nullptr) const {
        Mask m;
        m.active.assign(static_cast<size_t>(local_inter()), 0);
        int64_t cnt = 0;
        detail::check(sg_predict_mask(ctx.get(), layer_, x.data(), SG_F64, x.size(), m.active.data(),
                                      &cnt, stream));
        m.predicted_active_count = cnt;
        return m;
    }

   private:
    sg_layer* layer_ = nullptr;
    Index hidden_ = 0, inter_ = 0, rank_ = 0;
    int device_ = 0;
};

namespace detail {
// Digest of a buffer's full contents (64-bit FNV-1a over 8-byte words, then a
// splitmix finaliser).
inline std::uint64_t mix64(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
inline std::uint64_t fingerprint(const double* p, Index n, std::uint64_t salt) {
    std::uint64_t h = 0xcbf29ce484222325ull ^ mix64(salt ^ static_cast<std::uint64_t>(n));
    for (Index i = 0; i < n; ++i) {
        std::uint64_t b;
        std::memcpy(&b, p + i, 8);
        h = (h ^ b) * 0x100000001b3ull;
    }
    return mix64(h);
}
using Key = std::tuple<const void*, const void*, const void*, Index, Index, Index, int, std::uint64_t>;
inline Key key_of(const FfnWeights* w, const Predictor* p) {
    std::uint64_t f = 0;
    const void *a = nullptr, *b = nullptr, *c = nullptr;
    Index d = 0, D = 0, r = 0;
    int act = 0;
    if (w) {
        a = w->gate.data();
        b = w->down.data();
        d = w->hidden_size();
        D = w->inter_size();
        act = static_cast<int>(w->activation);
        f = mix64(f ^ fingerprint(w->gate.data(), w->gate.size(), 1));
        f = mix64(f ^ fingerprint(w->up.data(), w->up.size(), 2));
        f = mix64(f ^ fingerprint(w->down.data(), w->down.size(), 3));
    }
    if (p) {
        c = p->A.data();
        r = p->rank;
        f = mix64(f ^ fingerprint(p->A.data(), p->A.size(), 4));
        f = mix64(f ^ fingerprint(p->B.data(), p->B.size(), 5));
        f = mix64(f ^ fingerprint(p->bias.data(), p->bias.size(), 6));
    }
    return Key{a, b, c, d, D, r, act, f};
}
struct Cache {
    std::map<Key, std::unique_ptr<Layer>> layers;
    std::unique_ptr<Context> ctx;
    Index cd = 0, cD = 0, cr = 0;
};
inline Cache& cache() {
    thread_local Cache c;
    return c;
}
}  // namespace detail

inline void clear_cache() {
    detail::cache().layers.clear();
    detail::cache().ctx.reset();
}

inline const Layer& layer_for(const FfnWeights* w, const Predictor* p) {
    auto& c = detail::cache();
    const auto k = detail::key_of(w, p);
    auto it = c.layers.find(k);
    if (it == c.layers.end()) {
        if (c.layers.size() >= 64) c.layers.clear();  // bounded
        it = c.layers.emplace(k, std::make_unique<Layer>(w, p)).first;
    }
    return *it->second;
}

inline Context& context_for(const Layer& l) {
    auto& c = detail::cache();
    const Index r = l.rank() > 0 ? l.rank() : 1;
    if (!c.ctx || l.hidden() > c.cd || l.inter() > c.cD || r > c.cr) {
        c.cd = std::max(c.cd, l.hidden());
        c.cD = std::max(c.cD, l.inter());
        c.cr = std::max(c.cr, r);
        c.ctx.reset();
        c.ctx = std::make_unique<Context>(l.device(), c.cd, c.cD, c.cr);
    }
    return *c.ctx;
}

}  // namespace gpu

// ---- the reference API ----
inline FfnResult dense_ffn(const FfnWeights& w, const Vec& x) {
    const auto& l = gpu::layer_for(&w, nullptr);
    return l.forward(gpu::context_for(l), Pipeline::Dense, x);
}

// The standalone mask is exact: f64 on the GPU in det_dot order (sg_predict_mask_f64),
// so it equals the reference bit for bit; the executors' internal masks use the
// layer's bf16 predictor (gpu::Layer::predict is that one).
inline Mask predict_mask(const Predictor& pred, const Vec& x) {
    validate(pred);
    if (x.size() != pred.hidden_size()) throw DataError("predictor input length does not match hidden size");
    Mask m;
    m.active.assign(static_cast<std::size_t>(pred.inter_size()), 0);
    std::int64_t cnt = 0;
    detail::check(sg_predict_mask_f64(0, pred.A.data(), pred.B.data(), pred.bias.data(),
                                      pred.inter_size(), pred.rank, pred.hidden_size(), x.data(),
                                      m.active.data(), &cnt));
    m.predicted_active_count = cnt;
    return m;
}

inline FfnResult sparse_ffn_parallel(const FfnWeights& w, const Predictor& pred, const Vec& x) {
    const auto& l = gpu::layer_for(&w, &pred);
    return l.forward(gpu::context_for(l), Pipeline::Parallel, x);
}

inline FfnResult sparse_ffn_sequential(const FfnWeights& w, const Predictor& pred, const Vec& x) {
    const auto& l = gpu::layer_for(&w, &pred);
    return l.forward(gpu::context_for(l), Pipeline::Sequential, x);
}

inline OpCounts op_count_model(std::int64_t d, std::int64_t D, std::int64_t r, double s,
                               double s_prime) {
    OpCounts c;
    detail::check(sg_op_count_model(d, D, r, s, s_prime, &c.dense, &c.sparse, &c.ratio));
    return c;
}

// ffn_exec.hpp:251-285: the exact dropped-gate-mass formula under the (device)
// predictor mask; the gate projection is evaluated on the host in f64 with the
// reference's det_dot / det_sum, and the closed form is cross-checked against
// the direct masked difference as the reference does.
inline GatingError gating_error(const FfnWeights& w, const Predictor& pred, const Vec& x) {
    validate(w);
    if (x.size() != w.hidden_size())  // ffn_exec.hpp:58-63
        throw DataError("ffn input length " + std::to_string(x.size()) + " does not match hidden size " +
                        std::to_string(w.hidden_size()));
    if (!all_finite(x)) throw DataError("ffn input has non-finite entries");
    const Mask mask = predict_mask(pred, x);
    const Index D = w.inter_size(), d = w.hidden_size();
    std::vector<double> formula_terms(static_cast<size_t>(D)), direct_terms(static_cast<size_t>(D));
    for (Index i = 0; i < D; ++i) {
        const double a = relu(det_dot(w.gate.data() + i * d, x.data(), static_cast<size_t>(d)));
        const bool on = mask.active[static_cast<size_t>(i)] != 0;
        formula_terms[static_cast<size_t>(i)] = on ? 0.0 : a * a;
        const double diff = a - (on ? a : 0.0);
        direct_terms[static_cast<size_t>(i)] = diff * diff;
    }
    const double formula = std::sqrt(det_sum(formula_terms.data(), formula_terms.size()));
    const double direct = std::sqrt(det_sum(direct_terms.data(), direct_terms.size()));
    if (std::abs(formula - direct) > 1e-12 * std::max(1.0, std::abs(direct)))
        throw PropertyViolation("gating error: closed form disagrees with direct difference");
    const double x_norm = std::sqrt(det_dot(x.data(), x.data(), static_cast<size_t>(x.size())));
    if (x_norm == 0.0) throw DataError("gating error: zero input has no relative form");
    GatingError err;
    err.error_norm = formula;
    err.relative = formula / x_norm;
    return err;
}

}  // namespace sparsegate
