// Exercises include/sparsegate/ffn_exec.hpp (the C++ drop-in) the way a
// reference caller would. Mode "cpu": host-only entry points (no device calls).
// Mode "gpu": the executor on cuda:0, with known answers from
// /root/reference/proj/tests/ffn_exec_tests.cpp.
//   g++ -std=c++17 -O2 -Iinclude tests/cpp/header_check.cpp
//       -Lpaper_2603_14110_b200 -lsparsegate_b200 -Wl,-rpath,<abs pkg dir>
#include "sparsegate/ffn_exec.hpp"

#include <cstdio>
#include <random>
#include <string>

using namespace sparsegate;

static int fails = 0;
#define CHECK(c)                                                         \
    do {                                                                 \
        if (!(c)) {                                                      \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);     \
            ++fails;                                                     \
        }                                                                \
    } while (0)

template <class E, class F>
static bool throws(F f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static Mat random_mat(std::mt19937_64& g, Index r, Index c) {
    std::normal_distribution<double> n(0.0, 1.0);
    Mat m(r, c);
    for (Index i = 0; i < r; ++i)
        for (Index j = 0; j < c; ++j) m(i, j) = n(g);
    return m;
}

static void cpu_checks() {
    // ffn_exec_tests.cpp:256-279
    const OpCounts c = op_count_model(4096, 11008, 256, 0.5, 0.9);
    CHECK(c.dense == 135266304);
    CHECK(std::abs(c.sparse - 35428761.6) < 1e-6);
    char buf[32];
    std::snprintf(buf, sizeof buf, "%.2f", c.ratio);
    CHECK(std::string(buf) == "3.82");
    CHECK(throws<DataError>([] { op_count_model(64, 256, 8, 0.9, 0.5); }));
    CHECK(throws<DataError>([] { op_count_model(0, 256, 8, 0.5, 0.9); }));
    // types.hpp validation
    FfnWeights w{Mat::Zero(4, 2), Mat::Zero(4, 2), Mat::Zero(3, 4), Activation::ReGLU};
    CHECK(throws<DataError>([&] { validate(w); }));
    w.down = Mat::Zero(2, 4);
    validate(w);
    w.up(1, 1) = std::nan("");
    CHECK(throws<DataError>([&] { validate(w); }));
    Predictor p{Mat::Zero(4, 2), Mat::Zero(2, 3), Vec::Zero(4), 2};
    validate(p);
    p.bias(0) = INFINITY;  // calibrated +inf biases are legal
    validate(p);
    p.rank = 3;
    CHECK(throws<DataError>([&] { validate(p); }));
    CHECK(std::string(sg_version()).rfind("sparsegate-b200", 0) == 0);
    int64_t b, s, n;
    CHECK(sg_shard_range(11008, 3, 8, 1, &b, &s, &n) == SG_OK && b == 3 && s == 8 && n == 1376);
}

static void gpu_checks() {
    // ffn_exec_tests.cpp:51-82: 2x2 dense known answers
    FfnWeights w{Mat(2, 2), Mat::Identity(2, 2), Mat::Identity(2, 2), Activation::ReGLU};
    w.gate << 1, 0, -1, 0;
    Vec x11(2), xnan(2), x3(3);
    x11 << 1, 1;
    xnan << 1, std::nan("");
    x3 << 1, 1, 1;
    const FfnResult r = dense_ffn(w, x11);
    CHECK(r.y[0] == 1.0 && r.y[1] == 0.0);
    CHECK(r.stats.multiplies == 12 && r.stats.pipeline == Pipeline::Dense);
    CHECK(throws<DataError>([&] { dense_ffn(w, xnan); }));
    CHECK(throws<DataError>([&] { dense_ffn(w, x3); }));
    w.up << -1, 0, 0, 1;
    const FfnResult r2 = dense_ffn(w, x11);
    if (r2.y[0] != -1.0) std::printf("reglu y = (%g, %g)\n", r2.y[0], r2.y[1]);
    CHECK(r2.y[0] == -1.0);
    w.activation = Activation::DReLU;
    CHECK(dense_ffn(w, x11).y[0] == 0.0);

    // exact predictor (A = gate, B = I): mask = gate support; all-active == dense
    std::mt19937_64 g(29);
    for (Activation act : {Activation::ReGLU, Activation::DReLU}) {
        FfnWeights rw{random_mat(g, 48, 16), random_mat(g, 48, 16), random_mat(g, 16, 48), act};
        Predictor all{rw.gate, Mat::Identity(16, 16), Vec::Zero(48), 16};
        all.bias.setConstant(1e12);
        Vec x(16);
        std::normal_distribution<double> nd(0.0, 1.0);
        for (Index i = 0; i < 16; ++i) x[i] = nd(g);
        const FfnResult a = sparse_ffn_sequential(rw, all, x), d = dense_ffn(rw, x);
        double err = 0, nrm = 0;
        for (Index i = 0; i < 16; ++i) {
            err += (a.y[i] - d.y[i]) * (a.y[i] - d.y[i]);
            nrm += d.y[i] * d.y[i];
        }
        CHECK(err <= 1e-10 * nrm);
        CHECK(a.stats.predicted_sparsity == 0.0);
        Predictor exact{rw.gate, Mat::Identity(16, 16), Vec::Zero(48), 16};
        const Mask m = predict_mask(exact, x);
        Index cnt = 0;
        for (auto v : m.active) cnt += v;
        CHECK(cnt == m.predicted_active_count);
        const GatingError ge = gating_error(rw, exact, x);
        CHECK(ge.error_norm >= 0.0 && ge.relative >= 0.0);
    }
}

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "cpu";
    try {
        cpu_checks();
        if (mode == "gpu") gpu_checks();
    } catch (const std::exception& e) {
        std::printf("FAIL exception: %s\n", e.what());
        return 2;
    }
    std::printf("%s: %d failure(s)\n", mode.c_str(), fails);
    return fails ? 1 : 0;
}
