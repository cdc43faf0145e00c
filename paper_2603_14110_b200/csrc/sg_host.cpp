// sparsegate-b200 host library: the C ABI (include/sparsegate_c.h).
//
// Host responsibilities, each mirroring a reference contract:
//   * sg_layer_create: validate ONCE (types.hpp:31-51 FfnWeights, :82-105
//     Predictor), round to bf16, pad rows to 128-B pitches, transpose `down`
//     (reference d x D, types.hpp:19-24) to neuron-major and pack it behind the
//     matching `up` row, upload.
//   * sg_ffn_forward*: the executor entry points (ffn_exec.hpp:103-218); input
//     checks of detail::check_input (ffn_exec.hpp:56-65); ExecStats formulas
//     (ffn_exec.hpp:120, :173-180, :209-216).
//   * sg_op_count_model: ffn_exec.hpp:229-244 verbatim semantics.
//   * sg_synthetic_fixture*: synthetic.hpp:15-108 (same mt19937_64 stream).
//   * sg_greedy_calibrate: calibration.hpp:61-96 and :128-205 (offline producer).
#include "sparsegate_c.h"
#include "sg_internal.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <limits>
#include <numeric>
#include <queue>
#include <random>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

struct sg_layer {
    int device = 0;
    int64_t d = 0, D_full = 0, D_local = 0, r = 0;
    int act = 0;
    bool has_pred = false;
    bool has_w = false;
    int pitch_d = 0, pitch_r = 0;
    int64_t gbase = 0, gstride = 1;
    void* dmem = nullptr;
    size_t bytes = 0;
    std::vector<int> gidx;  // local -> global when a layout order was given (else empty)
    sg::LayerView view{};
    sg::LayerView* repdev = nullptr;  // [64] copies of view: small batches as one stack launch
    uint64_t id = 0;                  // unique per (layer, view contents): bumped by set_hot_rows
    sg::TcMaps tcmaps{};              // weight tensor maps of the tensor-core batch path
    bool has_tcmaps = false;
    int tc_brows = 0;                 // its neurons per block (sg::tc_block_rows)
};

struct sg_ctx {
    int device = 0;
    int G = 0;
    int64_t max_d = 0, max_D = 0, max_r = 0;
    int pitch_dmax = 0, pitch_rmax = 0;
    void* dmem = nullptr;
    sg::WorkView W{};
    float* xdev = nullptr;
    float* ydev = nullptr;
    uint8_t* maskdev = nullptr;
    float* xpin = nullptr;
    float* ypin = nullptr;
    const sg_layer* last_layer = nullptr;
    int last_pipeline = 0;
    // device descriptor tables, one per distinct stack (keyed by layer ids, never
    // mutated or freed before the ctx: a captured CUDA graph may replay one)
    std::map<std::vector<uint64_t>, sg::LayerView*> tables;
    std::vector<const sg_layer*> last_stack;
    unsigned long long* sbits = nullptr;  // [2][max_D] per-layer P / V bits of stack calls
    bool stack_sets = false;
    bool last_stack_bits = false;          // the last stack call recorded them
    float* xsdev = nullptr;  // host-entry staging for stacks
    float* ysdev = nullptr;
    size_t xs_cap = 0;
    uint64_t* dbgdev = nullptr;
    int dbg_layers = 0;
    // batched decode workspace (allocated on first use)
    void* bmem = nullptr;
    sg::BatchArgs bw{};
    float* bxdev = nullptr;  // host-entry staging [64][max_d]
    float* bydev = nullptr;
    const sg_layer* blast = nullptr;
    int blast_B = 0;
    bool blast_stack = false;  // the last batch ran as a stack launch (small B)
    int blast_path = 0;        // 0 stack, 1 legacy mma.sync kernels, 2 tensor cores (tcgen05)
    // tensor-core batch workspace (allocated on first use)
    void* tmem_ws = nullptr;
    sg::TcArgs tw{};
    std::map<int, sg::TcMaps> tcmaps_ws;  // workspace maps per nb (box height N = 2 nb)
    // X^T prepared by the last tensor-core launch for the next one: valid for a call on
    // `layer` with `batch` tokens whose input is hs + res == prep_h + prep_y
    struct {
        bool valid = false;
        const sg_layer* layer = nullptr;
        const float* h = nullptr;
        const float* y = nullptr;
        int batch = 0;
    } tc_prep;
    std::map<std::vector<int>, int*> tc_orders;  // device claim orders per unit geometry
    unsigned long long* tc_trace = nullptr;      // optional unit trace (sg_ctx_enable_tc_trace)
    size_t tc_trace_cap = 0;
    bool tc_trace_on = false;
    int tc_last_units = 0;
    const int* tc_last_order = nullptr;
};

constexpr int kMaxStackLayers = 1024;

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_layer_ids{1};

sg_status fail(sg_status s, const std::string& msg) {
    g_err = msg;
    return s;
}

#define SG_CUDA(call)                                                                      \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            return fail(SG_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

int round_up(int64_t v, int64_t a) { return static_cast<int>((v + a - 1) / a * a); }

// f64 -> f32 (RNE, hardware cast) -> bf16 (RNE on the f32 bits), NaN kept quiet.
inline uint16_t f32_to_bf16(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x007fffffu) != 0) {
        return static_cast<uint16_t>((u >> 16) | 0x0040u);
    }
    const uint32_t lsb = (u >> 16) & 1u;
    u += 0x7fffu + lsb;
    return static_cast<uint16_t>(u >> 16);
}
inline uint16_t to_bf16(const void* base, int dtype, int64_t i) {
    switch (dtype) {
        case SG_F64: return f32_to_bf16(static_cast<float>(static_cast<const double*>(base)[i]));
        case SG_F32: return f32_to_bf16(static_cast<const float*>(base)[i]);
        default: return static_cast<const uint16_t*>(base)[i];
    }
}
inline bool finite_at(const void* base, int dtype, int64_t i) {
    switch (dtype) {
        case SG_F64: return std::isfinite(static_cast<const double*>(base)[i]);
        case SG_F32: return std::isfinite(static_cast<const float*>(base)[i]);
        default: return (static_cast<const uint16_t*>(base)[i] & 0x7f80u) != 0x7f80u;
    }
}

// Parallel for over [0, n) in contiguous blocks on hardware threads.
void par_for(int64_t n, const std::function<void(int64_t, int64_t)>& fn) {
    unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int64_t workers = std::min<int64_t>(hw, std::max<int64_t>(1, n / 64));
    if (workers <= 1) {
        fn(0, n);
        return;
    }
    std::vector<std::thread> pool;
    for (int64_t w = 0; w < workers; ++w) {
        pool.emplace_back([&, w] { fn(n * w / workers, n * (w + 1) / workers); });
    }
    for (auto& t : pool) t.join();
}

bool all_finite(const void* p, int dtype, int64_t n) {
    std::atomic<bool> ok{true};
    par_for(n, [&](int64_t a, int64_t b) {
        for (int64_t i = a; i < b && ok.load(std::memory_order_relaxed); ++i) {
            if (!finite_at(p, dtype, i)) ok = false;
        }
    });
    return ok;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                   CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                   CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<EncodeTiledFn>(f);
    }();
    return fn;
}
// 2-D bf16 map: `cols` x `rows`, row stride `row_elems`, box {64, box_rows}, 128-B swizzle.
bool make_map(CUtensorMap* m, const void* base, int64_t cols, int64_t rows, int64_t row_elems,
              int box_rows) {
    EncodeTiledFn fn = encode_tiled();
    if (fn == nullptr) return false;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(row_elems) * 2};
    cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
    cuuint32_t es[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int64_t local_to_global(const sg_layer* L, int64_t k) {
    return L->gidx.empty() ? L->gbase + k * L->gstride : L->gidx[static_cast<size_t>(k)];
}

// interleaved (neuron base + k*S) or contiguous near-equal blocks.
void shard_map(int64_t D, int64_t si, int64_t S, bool interleave, int64_t* base, int64_t* stride,
               int64_t* count) {
    if (S > 1 && interleave) {
        *base = si;
        *stride = S;
        *count = si < D ? (D - si + S - 1) / S : 0;
    } else {
        const int64_t lo = D * si / S, hi = D * (si + 1) / S;
        *base = lo;
        *stride = 1;
        *count = hi - lo;
    }
}

sg_exec_stats stats_from_counts(int64_t d, int64_t D, int64_t r, int pipeline, int64_t p, int64_t v) {
    sg_exec_stats s{};
    s.pipeline = pipeline;
    s.predicted_active = p;
    s.revalidated = v;
    if (pipeline == SG_PIPELINE_DENSE) {  // ffn_exec.hpp:118-121
        s.multiplies = int64_t{3} * d * D;
        s.predicted_sparsity = 0.0;
        s.realized_sparsity = 0.0;
    } else if (pipeline == SG_PIPELINE_PARALLEL) {  // ffn_exec.hpp:173-180
        s.multiplies = r * (d + D) + int64_t{3} * d * p;
        s.predicted_sparsity = 1.0 - static_cast<double>(p) / static_cast<double>(D);
        s.realized_sparsity = s.predicted_sparsity;
    } else {  // ffn_exec.hpp:209-216
        s.multiplies = r * (d + D) + d * p + int64_t{2} * d * v;
        s.predicted_sparsity = 1.0 - static_cast<double>(p) / static_cast<double>(D);
        s.realized_sparsity = 1.0 - static_cast<double>(v) / static_cast<double>(D);
    }
    return s;
}

sg_exec_stats make_stats(const sg_layer* L, int pipeline, int64_t p, int64_t v) {
    return stats_from_counts(L->d, L->D_local, L->r, pipeline, p, v);
}

// Batches up to this size run through the persistent single-token executor (one
// stack launch, token b as layer b). Measured on B200 (7B, 8-layer stack, tokens/s,
// persistent vs row streaming): B = 3 4616 / 4020, 4 4883 / 4831, 5 4997 / 5867,
// 6 5136 / 6928. SG_BATCH_STACK_MAX overrides (0 = always the batched path).
int small_batch_limit() {
    static const int v = [] {
        const char* e = std::getenv("SG_BATCH_STACK_MAX");
        return e ? std::atoi(e) : 1;
    }();
    return v;
}

sg::WorkView work_for(sg_ctx* ctx, const float* x, float* y) {
    sg::WorkView W = ctx->W;
    W.x = x;
    W.y = y;
    return W;
}

sg_status check_pair(sg_ctx* ctx, const sg_layer* L) {
    if (ctx == nullptr || L == nullptr) return fail(SG_ERR_USAGE, "null ctx or layer");
    if (ctx->device != L->device) return fail(SG_ERR_USAGE, "ctx and layer on different devices");
    if (L->d > ctx->max_d || L->D_local > ctx->max_D || L->r > ctx->max_r)
        return fail(SG_ERR_USAGE, "layer exceeds the ctx bounds (max_hidden/max_inter/max_rank)");
    return SG_OK;
}

sg_status read_x(const void* x, sg_dtype dt, int64_t n, int64_t d, float* out, const char* what) {
    if (x == nullptr) return fail(SG_ERR_USAGE, "null x");
    if (n != d) {  // ffn_exec.hpp:58-60 / :127-129
        return fail(SG_ERR_DATA, std::string(what) + " input length " + std::to_string(n) +
                                     " does not match hidden size " + std::to_string(d));
    }
    for (int64_t i = 0; i < n; ++i) {
        double v;
        if (dt == SG_F64) v = static_cast<const double*>(x)[i];
        else if (dt == SG_F32) v = static_cast<const float*>(x)[i];
        else return fail(SG_ERR_USAGE, "x dtype must be SG_F64 or SG_F32");
        if (!std::isfinite(v)) {  // ffn_exec.hpp:61-63
            return fail(SG_ERR_DATA, std::string(what) + " input has non-finite entries");
        }
        out[i] = static_cast<float>(v);
    }
    return SG_OK;
}

sg_status stack_launch(sg_ctx* C, const sg_layer* const* layers, int32_t n,
                              sg_pipeline pipeline, const float* xs, float* ys, int32_t chain,
                              void* stream, unsigned long long* mbits, unsigned long long* vbits,
                              const sg::LayerView* views_dev = nullptr) {
    if (C == nullptr || layers == nullptr || n < 1 || n > kMaxStackLayers || chain < 0 || chain > 2)
        return fail(SG_ERR_USAGE, "bad arguments");
    if (xs == nullptr || ys == nullptr) return fail(SG_ERR_USAGE, "null xs/ys");
    const sg_layer* L0 = layers[0];
    for (int i = 0; i < n; ++i) {
        const sg_layer* L = layers[i];
        if (sg_status s = check_pair(C, L); s != SG_OK) return s;
        if (L->d != L0->d || L->D_local != L0->D_local || L->r != L0->r)
            return fail(SG_ERR_USAGE, "all layers of a stack must share hidden/inter/rank");
        if (pipeline != SG_PIPELINE_DENSE && !L->has_pred)
            return fail(SG_ERR_USAGE, "sparse pipeline needs layers with predictors");
        if (!L->has_w) return fail(SG_ERR_USAGE, "predictor-only layer cannot run the FFN");
    }
    DeviceGuard dg(C->device);
    auto st = static_cast<cudaStream_t>(stream);
    if (views_dev != nullptr) {
        // caller-provided descriptor table (no upload: graph-capture safe)
        SG_CUDA(cudaMemsetAsync(C->W.stats, 0, static_cast<size_t>(n) * 4 * sizeof(int), st));
        sg::WorkView W = work_for(C, xs, ys);
        W.mbits = mbits;
        W.vbits = vbits;
        const int e = sg::launch_layers(views_dev, n, L0->view, W, xs, ys, chain,
                                        static_cast<int>(L0->d), pipeline, C->G, st);
        if (e != 0) return fail(SG_ERR_CUDA, std::string("launch: ") +
                                                 cudaGetErrorString(static_cast<cudaError_t>(e)));
        C->last_layer = layers[n - 1];
        C->last_pipeline = pipeline;
        C->last_stack.clear();
        return SG_OK;
    }
    // The (tiny) descriptor table of a stack is uploaded once per distinct stack
    // (layer ids, not pointers: a freed and re-created layer at a recycled address
    // gets a new id), so repeated calls — and CUDA-graph capture after a first
    // warm call — issue nothing but the kernel launch.
    std::vector<uint64_t> key(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) key[static_cast<size_t>(i)] = layers[i]->id;
    sg::LayerView* table = nullptr;
    if (auto it = C->tables.find(key); it != C->tables.end()) {
        table = it->second;
    } else {
        std::vector<sg::LayerView> views(n);
        for (int i = 0; i < n; ++i) views[i] = layers[i]->view;
        SG_CUDA(cudaMalloc(&table, sizeof(sg::LayerView) * n));
        SG_CUDA(cudaMemcpy(table, views.data(), sizeof(sg::LayerView) * n, cudaMemcpyHostToDevice));
        C->tables.emplace(std::move(key), table);
    }
    SG_CUDA(cudaMemsetAsync(C->W.stats, 0, static_cast<size_t>(n) * 4 * sizeof(int), st));
    sg::WorkView W = work_for(C, xs, ys);
    W.mbits = mbits;
    W.vbits = vbits;
    const int e = sg::launch_layers(table, n, L0->view, W, xs, ys, chain,
                                    static_cast<int>(L0->d), pipeline, C->G, st);
    if (e != 0) return fail(SG_ERR_CUDA, std::string("launch: ") +
                                             cudaGetErrorString(static_cast<cudaError_t>(e)));
    C->last_layer = layers[n - 1];
    C->last_pipeline = pipeline;
    C->last_stack.assign(layers, layers + n);
    return SG_OK;
}

}  // namespace

// ---- internals shared with sg_comm.cpp (the sharded stack) ----
sg_status sg_internal_fail(sg_status st, const std::string& msg) { return fail(st, msg); }

// Validates a stack for a sequence of per-layer launches and zeroes its stats slots.
sg_status sg_internal_begin_stack(sg_ctx* C, const sg_layer* const* layers, int32_t n, sg_pipeline pipeline,
                                  void* stream) {
    if (C == nullptr || layers == nullptr || n < 1 || n > kMaxStackLayers) return fail(SG_ERR_USAGE, "bad arguments");
    for (int i = 0; i < n; ++i) {
        if (sg_status s = check_pair(C, layers[i]); s != SG_OK) return s;
        if (layers[i]->d != layers[0]->d) return fail(SG_ERR_USAGE, "all layers of a stack must share hidden");
        if (pipeline != SG_PIPELINE_DENSE && !layers[i]->has_pred)
            return fail(SG_ERR_USAGE, "sparse pipeline needs layers with predictors");
        if (!layers[i]->has_w) return fail(SG_ERR_USAGE, "predictor-only layer cannot run the FFN");
    }
    DeviceGuard dg(C->device);
    SG_CUDA(cudaMemsetAsync(C->W.stats, 0, static_cast<size_t>(n) * 4 * sizeof(int), static_cast<cudaStream_t>(stream)));
    C->last_stack.assign(layers, layers + n);
    C->last_pipeline = pipeline;
    C->last_layer = layers[n - 1];
    C->last_stack_bits = false;
    return SG_OK;
}

// One layer launch writing stats slot `slot` (the stack's per-layer {p, v, bad, pipe}).
sg_status sg_internal_forward_layer(sg_ctx* C, const sg_layer* L, sg_pipeline pipeline, const float* x,
                                    const float* xres, float* y, int slot, void* stream) {
    DeviceGuard dg(C->device);
    sg::WorkView W = work_for(C, x, y);
    W.xres = xres;
    W.stats = C->W.stats + 4 * slot;
    const int e = sg::launch_layer(L->view, W, pipeline, C->G, stream);
    if (e != 0) return fail(SG_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(static_cast<cudaError_t>(e)));
    return SG_OK;
}

extern "C" {

const char* sg_last_error(void) { return g_err.c_str(); }
int64_t sg_layer_hidden(const sg_layer* L) { return L ? L->d : 0; }
const char* sg_version(void) { return "sparsegate-b200 0.1 (sm_100a)"; }

sg_status sg_op_count_model(int64_t d, int64_t D, int64_t r, double s, double sp, int64_t* dense,
                            double* sparse, double* ratio) {
    if (d < 1 || D < 1 || r < 0) {
        return fail(SG_ERR_DATA, "op count model: dimensions must be positive and rank nonnegative");
    }
    if (!(0.0 <= s && s <= sp && sp <= 1.0)) {
        return fail(SG_ERR_DATA, "op count model: need 0 <= s <= s' <= 1");
    }
    const int64_t dn = 3 * d * D;
    const double sps = static_cast<double>(r) * static_cast<double>(d + D) +
                       static_cast<double>(d) * (1.0 - s) * static_cast<double>(D) +
                       2.0 * static_cast<double>(d) * (1.0 - sp) * static_cast<double>(D);
    if (dense) *dense = dn;
    if (sparse) *sparse = sps;
    if (ratio) *ratio = static_cast<double>(dn) / sps;
    return SG_OK;
}

sg_status sg_shard_range(int64_t inter, int32_t shard_index, int32_t shard_count,
                         int32_t shard_interleave, int64_t* base, int64_t* stride, int64_t* count) {
    if (inter < 1) return fail(SG_ERR_DATA, "shard range: inter must be positive");
    const int64_t S = shard_count > 1 ? shard_count : 1;
    const int64_t si = S > 1 ? shard_index : 0;
    if (si < 0 || si >= S) return fail(SG_ERR_USAGE, "shard_index out of range");
    if (base == nullptr || stride == nullptr || count == nullptr) return fail(SG_ERR_USAGE, "null output");
    shard_map(inter, si, S, shard_interleave != 0, base, stride, count);
    return SG_OK;
}

sg_status sg_exec_stats_from_counts(int64_t hidden, int64_t inter, int64_t rank, sg_pipeline pipeline,
                                    int64_t predicted_active, int64_t revalidated, sg_exec_stats* out) {
    if (hidden < 1 || inter < 1 || rank < 0) return fail(SG_ERR_DATA, "stats: bad dimensions");
    if (pipeline < SG_PIPELINE_DENSE || pipeline > SG_PIPELINE_SEQUENTIAL)
        return fail(SG_ERR_USAGE, "stats: unknown pipeline");
    if (predicted_active < 0 || predicted_active > inter || revalidated < 0 ||
        revalidated > predicted_active)
        return fail(SG_ERR_USAGE, "stats: counts out of range");
    if (out == nullptr) return fail(SG_ERR_USAGE, "null output");
    *out = stats_from_counts(hidden, inter, rank, pipeline, predicted_active, revalidated);
    return SG_OK;
}

void sg_round_bf16(const double* in, uint16_t* out, int64_t n) {
    par_for(n, [&](int64_t a, int64_t b) {
        for (int64_t i = a; i < b; ++i) out[i] = f32_to_bf16(static_cast<float>(in[i]));
    });
}

sg_status sg_layer_create(const sg_layer_desc* desc, sg_layer** out) {
    if (desc == nullptr || out == nullptr) return fail(SG_ERR_USAGE, "null argument");
    *out = nullptr;
    const int64_t d = desc->hidden, D = desc->inter;
    if (d < 1 || D < 1) {  // types.hpp:34-37
        return fail(SG_ERR_DATA, "ffn weights: gate must be at least 1x1, got " +
                                     std::to_string(D) + "x" + std::to_string(d));
    }
    const bool has_w = desc->gate != nullptr || desc->up != nullptr || desc->down != nullptr;
    if (has_w && (desc->gate == nullptr || desc->up == nullptr || desc->down == nullptr))
        return fail(SG_ERR_USAGE, "gate/up/down must be given together");
    const int wdt = desc->weight_dtype;
    if (wdt != SG_F64 && wdt != SG_F32 && wdt != SG_BF16) return fail(SG_ERR_USAGE, "bad weight dtype");
    const bool has_pred = desc->pred_A != nullptr || desc->pred_B != nullptr || desc->bias != nullptr;
    int64_t r = 0;
    if (has_pred) {
        if (!desc->pred_A || !desc->pred_B || !desc->bias)
            return fail(SG_ERR_USAGE, "pred_A, pred_B and bias must be given together");
        r = desc->rank;
        if (r < 1 || r > std::min(D, d)) {  // types.hpp:92-95
            return fail(SG_ERR_DATA, "predictor: rank " + std::to_string(r) + " out of range [1, " +
                                         std::to_string(std::min(D, d)) + "]");
        }
        if (desc->bias_dtype != SG_F64 && desc->bias_dtype != SG_F32)
            return fail(SG_ERR_USAGE, "bias dtype must be SG_F64 or SG_F32");
    }
    if (!has_w && !has_pred) return fail(SG_ERR_USAGE, "layer needs weights and/or a predictor");
    if (d > (1 << 20) || D > (1 << 30)) return fail(SG_ERR_USAGE, "layer too large");
    // types.hpp:48-50 / :102-104 — once, here, instead of on every call.
    if (has_w && (!all_finite(desc->gate, wdt, D * d) || !all_finite(desc->up, wdt, D * d) ||
                  !all_finite(desc->down, wdt, D * d))) {
        return fail(SG_ERR_DATA, "ffn weights: non-finite entries");
    }
    if (has_pred && (!all_finite(desc->pred_A, wdt, D * r) || !all_finite(desc->pred_B, wdt, r * d))) {
        return fail(SG_ERR_DATA, "predictor: non-finite factor entries");
    }

    auto L = new sg_layer;
    L->device = desc->device;
    L->d = d;
    L->D_full = D;
    L->r = r;
    L->act = desc->activation == SG_DRELU ? 1 : 0;
    L->has_pred = has_pred;
    L->has_w = has_w;
    L->pitch_d = round_up(d, 64);
    L->pitch_r = has_pred ? round_up(r, 64) : 64;
    // shard -> local neuron list
    const int S = desc->shard_count > 1 ? desc->shard_count : 1;
    const int si = S > 1 ? desc->shard_index : 0;
    if (si < 0 || si >= S) {
        delete L;
        return fail(SG_ERR_USAGE, "shard_index out of range");
    }
    shard_map(D, si, S, S > 1 && desc->shard_interleave, &L->gbase, &L->gstride, &L->D_local);
    if (L->D_local < 1) {
        delete L;
        return fail(SG_ERR_USAGE, "shard holds no neurons");
    }
    const int64_t Dl = L->D_local, pd = L->pitch_d, pr = L->pitch_r;
    if (desc->neuron_order) {
        // layout order of this shard's neurons: their order of appearance in neuron_order
        std::vector<int64_t> pos(static_cast<size_t>(D), -1);
        for (int64_t i = 0; i < D; ++i) {
            const int64_t g = desc->neuron_order[i];
            if (g < 0 || g >= D || pos[static_cast<size_t>(g)] >= 0) {
                delete L;
                return fail(SG_ERR_DATA, "neuron_order is not a permutation of 0..inter-1");
            }
            pos[static_cast<size_t>(g)] = i;
        }
        std::vector<int64_t> mine(static_cast<size_t>(Dl));
        for (int64_t k = 0; k < Dl; ++k) mine[static_cast<size_t>(k)] = L->gbase + k * L->gstride;
        std::sort(mine.begin(), mine.end(), [&](int64_t a, int64_t b) {
            return pos[static_cast<size_t>(a)] < pos[static_cast<size_t>(b)];
        });
        L->gidx.assign(mine.begin(), mine.end());
    }
    // device layout: [B r x pd][A Dl x pr][gate Dl x pd][ud Dl x 2pd][bias Dl f32]
    const size_t nB = static_cast<size_t>(has_pred ? r : 0) * pd;
    const size_t nA = static_cast<size_t>(has_pred ? Dl : 0) * pr;
    const size_t nG = static_cast<size_t>(has_w ? Dl : 0) * pd;
    const size_t nUD = static_cast<size_t>(has_w ? Dl : 0) * 2 * pd;
    const size_t offB = 0, offA = offB + nB, offG = offA + nA, offUD = offG + nG;
    const size_t n16 = offUD + nUD;
    const size_t bias_off = (n16 * 2 + 255) / 256 * 256;
    const size_t gidx_off = bias_off + static_cast<size_t>(Dl) * 4;
    const size_t total = gidx_off + (L->gidx.empty() ? 0 : static_cast<size_t>(Dl) * 4);
    std::vector<uint16_t> host(n16, 0);
    std::vector<float> hbias(static_cast<size_t>(Dl), 0.f);
    const bool down_nm = desc->down_neuron_major != 0;
    par_for(Dl, [&](int64_t a, int64_t b) {
        for (int64_t k = a; k < b; ++k) {
            const int64_t n = local_to_global(L, k);
            uint16_t* g = host.data() + offG + k * pd;
            uint16_t* u = host.data() + offUD + k * 2 * pd;
            uint16_t* dn = u + pd;
            for (int64_t j = 0; has_w && j < d; ++j) {
                g[j] = to_bf16(desc->gate, wdt, n * d + j);
                u[j] = to_bf16(desc->up, wdt, n * d + j);
                dn[j] = down_nm ? to_bf16(desc->down, wdt, n * d + j)
                                : to_bf16(desc->down, wdt, j * D + n);  // column n of d x D
            }
            if (has_pred) {
                uint16_t* arow = host.data() + offA + k * pr;
                for (int64_t j = 0; j < r; ++j) arow[j] = to_bf16(desc->pred_A, wdt, n * r + j);
                hbias[k] = desc->bias_dtype == SG_F64
                               ? static_cast<float>(static_cast<const double*>(desc->bias)[n])
                               : static_cast<const float*>(desc->bias)[n];
            }
        }
    });
    if (has_pred) {
        par_for(r, [&](int64_t a, int64_t b) {
            for (int64_t j = a; j < b; ++j)
                for (int64_t k = 0; k < d; ++k)
                    host[offB + j * pd + k] = to_bf16(desc->pred_B, wdt, j * d + k);
        });
    }
    DeviceGuard dg(desc->device);
    cudaError_t e = cudaMalloc(&L->dmem, total);
    if (e == cudaSuccess) e = cudaMemcpy(L->dmem, host.data(), n16 * 2, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(static_cast<char*>(L->dmem) + bias_off, hbias.data(), Dl * 4,
                       cudaMemcpyHostToDevice);
    if (e == cudaSuccess && !L->gidx.empty())
        e = cudaMemcpy(static_cast<char*>(L->dmem) + gidx_off, L->gidx.data(), Dl * 4,
                       cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        if (L->dmem) cudaFree(L->dmem);
        delete L;
        return fail(SG_ERR_CUDA, std::string("layer upload: ") + cudaGetErrorString(e));
    }
    L->bytes = total;
    auto* base = static_cast<uint16_t*>(L->dmem);
    sg::LayerView& V = L->view;
    V.d = static_cast<int>(d);
    V.D = static_cast<int>(Dl);
    V.r = static_cast<int>(r);
    V.pitch_d = L->pitch_d;
    V.pitch_r = L->pitch_r;
    V.act = L->act;
    V.gbase = static_cast<int>(L->gbase);
    V.gstride = static_cast<int>(L->gstride);
    V.B = has_pred ? base + offB : nullptr;
    V.A = has_pred ? base + offA : nullptr;
    V.gate = has_w ? base + offG : nullptr;
    V.ud = has_w ? base + offUD : nullptr;
    V.bias = reinterpret_cast<const float*>(static_cast<char*>(L->dmem) + bias_off);
    V.gidx = L->gidx.empty() ? nullptr
                             : reinterpret_cast<const int*>(static_cast<char*>(L->dmem) + gidx_off);
    L->id = g_layer_ids.fetch_add(1);
    if (has_w) {
        // tensor maps of the batched tensor-core path (sg_batch_tc.cu)
        sg::TcMaps& tm = L->tcmaps;
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, L->device);
        const int br = sg::tc_block_rows(Dl, sms);
        L->tc_brows = br;
        bool ok = make_map(&tm.gate, V.gate, pd, Dl, pd, br) && make_map(&tm.up, V.ud, pd, Dl, 2 * pd, br) &&
                  make_map(&tm.down, V.ud + pd, pd, Dl, 2 * pd, 16) &&
                  make_map(&tm.down64, V.ud + pd, pd, Dl, 2 * pd, 64) &&
                  make_map(&tm.down128, V.ud + pd, pd, Dl, 2 * pd, 128);
        if (ok && has_pred)
            ok = make_map(&tm.A, V.A, pr, Dl, pr, br) && make_map(&tm.Bp, V.B, pd, r, pd, 128);
        L->has_tcmaps = ok;
    }
    if (has_w && has_pred) {
        // 64 copies of the view: small batches run as one stack launch (token b =
        // "layer" b); allocated here, never by a (possibly captured) forward call
        std::vector<sg::LayerView> views(64, L->view);
        e = cudaMalloc(&L->repdev, sizeof(sg::LayerView) * views.size());
        if (e == cudaSuccess)
            e = cudaMemcpy(L->repdev, views.data(), sizeof(sg::LayerView) * views.size(),
                           cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            sg_layer_destroy(L);
            return fail(SG_ERR_CUDA, std::string("layer upload: ") + cudaGetErrorString(e));
        }
    }
    *out = L;
    return SG_OK;
}

sg_status sg_layer_destroy(sg_layer* L) {
    if (L == nullptr) return SG_OK;
    DeviceGuard dg(L->device);
    if (L->dmem) cudaFree(L->dmem);
    if (L->repdev) cudaFree(L->repdev);
    delete L;
    return SG_OK;
}

int64_t sg_layer_local_inter(const sg_layer* L) { return L ? L->D_local : 0; }
int64_t sg_layer_global_index(const sg_layer* L, int64_t k) { return L ? local_to_global(L, k) : -1; }
int64_t sg_layer_device_bytes(const sg_layer* L) { return L ? static_cast<int64_t>(L->bytes) : 0; }

sg_status sg_layer_set_hot_rows(sg_layer* L, int64_t rows) {
    if (L == nullptr || rows < 0) return fail(SG_ERR_USAGE, "sg_layer_set_hot_rows: bad arguments");
    L->view.hot = static_cast<int>(rows < L->D_local ? rows : L->D_local);
    L->id = g_layer_ids.fetch_add(1);  // stacks built from now on get a fresh descriptor table
    if (L->repdev) {
        // refreshed in place (synchronously): a graph captured earlier keeps a
        // valid table; the hot prefix changes only when rows arrive, not results
        DeviceGuard dg(L->device);
        std::vector<sg::LayerView> views(64, L->view);
        SG_CUDA(cudaMemcpy(L->repdev, views.data(), sizeof(sg::LayerView) * views.size(),
                           cudaMemcpyHostToDevice));
    }
    return SG_OK;
}

sg_status sg_ctx_create(int32_t device, int64_t max_hidden, int64_t max_inter, int64_t max_rank,
                        sg_ctx** out) {
    if (out == nullptr || max_hidden < 1 || max_inter < 1 || max_rank < 0)
        return fail(SG_ERR_USAGE, "bad ctx bounds");
    *out = nullptr;
    DeviceGuard dg(device);
    sg::LaunchInfo info{};
    const int qe = sg::query_launch_info(device, &info);
    if (qe != 0) return fail(SG_ERR_CUDA, std::string("device query: ") +
                                             cudaGetErrorString(static_cast<cudaError_t>(qe)));
    auto C = new sg_ctx;
    C->device = device;
    C->G = info.num_sms;
    C->max_d = max_hidden;
    C->max_D = max_inter;
    C->max_r = std::max<int64_t>(max_rank, 1);
    C->pitch_dmax = round_up(max_hidden, 64);
    C->pitch_rmax = round_up(C->max_r, 64);
    const int G = C->G;
    const size_t Dm = static_cast<size_t>(max_inter) + 32;
    // carve one allocation (256-B aligned pieces)
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off += (bytes + 255) / 256 * 256;
        return o;
    };
    const size_t o_t = take(C->pitch_rmax * 32);  // one 32-B sector per t value
    const size_t o_cnt = take(2 * G * 32);  // one 32-B sector per CTA count
    const size_t o_plist = take(Dm * 4), o_P = take(Dm * 4), o_gP = take(Dm * 4);
    const size_t o_gN = take(Dm * 4);
    const size_t o_rec = take(Dm * 8), o_V = take(Dm * 4), o_zV = take(Dm * 4);
    const size_t o_vseg = take(Dm * 8);
    const size_t o_zD = take(Dm * 4);
    const size_t o_ypart = take(static_cast<size_t>(G) * C->pitch_dmax * 4);
    const size_t o_bar = take(8 * 256);
    const size_t o_ytag = take(static_cast<size_t>(C->pitch_dmax) * 8);
    const size_t o_stats = take(4 * 4 * kMaxStackLayers);
    const size_t o_x = take(C->pitch_dmax * 4), o_y = take(C->pitch_dmax * 4);
    const size_t o_mask = take(Dm);
    cudaError_t e = cudaMalloc(&C->dmem, off);
    if (e == cudaSuccess) e = cudaMemset(C->dmem, 0, off);
    if (e == cudaSuccess) e = cudaMallocHost(&C->xpin, C->pitch_dmax * 4);
    if (e == cudaSuccess) e = cudaMallocHost(&C->ypin, C->pitch_dmax * 4);
    if (e != cudaSuccess) {
        if (C->dmem) cudaFree(C->dmem);
        if (C->xpin) cudaFreeHost(C->xpin);
        delete C;
        return fail(SG_ERR_CUDA, std::string("ctx alloc: ") + cudaGetErrorString(e));
    }
    char* b = static_cast<char*>(C->dmem);
    sg::WorkView& W = C->W;
    W.t = reinterpret_cast<float*>(b + o_t);
    W.cnt = reinterpret_cast<int*>(b + o_cnt);
    W.plist = reinterpret_cast<int*>(b + o_plist);
    W.P = reinterpret_cast<int*>(b + o_P);
    W.gP = reinterpret_cast<float*>(b + o_gP);
    W.gN = reinterpret_cast<float*>(b + o_gN);
    W.rec = reinterpret_cast<int*>(b + o_rec);
    W.vseg = reinterpret_cast<int*>(b + o_vseg);
    W.V = reinterpret_cast<int*>(b + o_V);
    W.zV = reinterpret_cast<float*>(b + o_zV);
    W.zD = reinterpret_cast<float*>(b + o_zD);
    W.ypart = reinterpret_cast<float*>(b + o_ypart);
    W.bar = reinterpret_cast<unsigned long long*>(b + o_bar);
    W.ytag = reinterpret_cast<uint32_t*>(b + o_ytag);
    W.stats = reinterpret_cast<int*>(b + o_stats);
    if (const char* f = std::getenv("SG_FLAGS")) W.flags = std::atoi(f);
    C->xdev = reinterpret_cast<float*>(b + o_x);
    C->ydev = reinterpret_cast<float*>(b + o_y);
    C->maskdev = reinterpret_cast<uint8_t*>(b + o_mask);
    *out = C;
    return SG_OK;
}

sg_status sg_ctx_destroy(sg_ctx* C) {
    if (C == nullptr) return SG_OK;
    DeviceGuard dg(C->device);
    if (C->dmem) cudaFree(C->dmem);
    if (C->xpin) cudaFreeHost(C->xpin);
    if (C->ypin) cudaFreeHost(C->ypin);
    for (auto& kv : C->tables) cudaFree(kv.second);
    if (C->sbits) cudaFree(C->sbits);
    if (C->xsdev) cudaFree(C->xsdev);
    if (C->ysdev) cudaFree(C->ysdev);
    if (C->dbgdev) cudaFree(C->dbgdev);
    if (C->bmem) cudaFree(C->bmem);
    if (C->tmem_ws) cudaFree(C->tmem_ws);
    for (auto& kv : C->tc_orders) cudaFree(kv.second);
    if (C->tc_trace) cudaFree(C->tc_trace);
    delete C;
    return SG_OK;
}

// ---- batched decode ------------------------------------------------------------
namespace {
sg_status batch_workspace(sg_ctx* C) {
    if (C->bmem) return SG_OK;
    const int M = sg::batch_max();
    const size_t Dm = static_cast<size_t>(C->max_D), pd = static_cast<size_t>(C->pitch_dmax),
                 pr = static_cast<size_t>(C->pitch_rmax);
    const size_t pv = (Dm + 63) / 64 * 64;
    const int tsplit = 16;
    // split-K of the down GEMM (SG_BATCH_DSPLIT overrides; the partial buffer is
    // sized for sg::kDpSplits)
    const int dsplit = [] {
        const char* e = std::getenv("SG_BATCH_DSPLIT");
        const int v = e ? std::atoi(e) : 0;  // 0: per call (see sg_ffn_forward_batch)
        return v < 0 ? 0 : (v > sg::kDpSplits ? sg::kDpSplits : v);
    }();
    // split-K of the gate / up GEMMs (SG_BATCH_GSPLIT overrides; the partial buffer
    // is sized for sg::kGpSplits)
    const int gsplit = [] {
        const char* e = std::getenv("SG_BATCH_GSPLIT");
        const int v = e ? std::atoi(e) : 0;  // 0: per call (see sg_ffn_forward_batch)
        return v < 0 ? 0 : (v > sg::kGpSplits ? sg::kGpSplits : v);
    }();
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off += (bytes + 255) / 256 * 256;
        return o;
    };
    const size_t o_xh = take(M * pd * 2), o_xl = take(M * pd * 2), o_tp = take(tsplit * pr * M * 4),
                 o_th = take(M * pr * 2), o_tl = take(M * pr * 2), o_mb = take(Dm * 8),
                 o_uf = take(Dm * 4), o_pc = take(M * 4), o_pl = take(Dm * 4), o_np = take(4),
                 o_G = take(Dm * M * 4), o_vb = take(Dm * 8), o_vf = take(Dm * 4), o_vc = take(M * 4),
                 o_vl = take(Dm * 4), o_nv = take(4), o_Z = take(Dm * M * 4), o_zh = take(M * pv * 2),
                 o_zl = take(M * pv * 2), o_yp = take(sg::kDpSplits * M * pd * 4), o_bx = take(M * pd * 4),
                 o_by = take(M * pd * 4), o_gp = take(sg::kGpSplits * pv * M * 4), o_tk = take(16 * 4),
                 o_bad = take(4);
    DeviceGuard dg(C->device);
    cudaError_t e = cudaMalloc(&C->bmem, off);
    if (e == cudaSuccess) e = cudaMemset(C->bmem, 0, off);
    if (e != cudaSuccess) {
        C->bmem = nullptr;
        return fail(SG_ERR_CUDA, std::string("batch workspace: ") + cudaGetErrorString(e));
    }
    char* b = static_cast<char*>(C->bmem);
    sg::BatchArgs& a = C->bw;
    a.pitch_v = static_cast<int>(pv);
    a.tsplit = tsplit;
    a.dsplit = dsplit;
    a.gsplit = gsplit;
    {  // SG_BATCH_GDOT=0: gate / up through the tensor-core tiles at every batch size
        const char* e = std::getenv("SG_BATCH_GDOT");
        a.gdot = e ? std::atoi(e) != 0 : 1;
    }
    a.sms = C->G;
    a.gp = reinterpret_cast<float*>(b + o_gp);
    a.xh = reinterpret_cast<uint16_t*>(b + o_xh);
    a.xl = reinterpret_cast<uint16_t*>(b + o_xl);
    a.tp = reinterpret_cast<float*>(b + o_tp);
    a.th = reinterpret_cast<uint16_t*>(b + o_th);
    a.tl = reinterpret_cast<uint16_t*>(b + o_tl);
    a.mbits = reinterpret_cast<uint64_t*>(b + o_mb);
    a.uflag = reinterpret_cast<int*>(b + o_uf);
    a.pcount = reinterpret_cast<int*>(b + o_pc);
    a.plist = reinterpret_cast<int*>(b + o_pl);
    a.np = reinterpret_cast<int*>(b + o_np);
    a.G = reinterpret_cast<float*>(b + o_G);
    a.vbits = reinterpret_cast<uint64_t*>(b + o_vb);
    a.vflag = reinterpret_cast<int*>(b + o_vf);
    a.vcount = reinterpret_cast<int*>(b + o_vc);
    a.vlist = reinterpret_cast<int*>(b + o_vl);
    a.nv = reinterpret_cast<int*>(b + o_nv);
    a.ticket = reinterpret_cast<int*>(b + o_tk);
    a.bad = reinterpret_cast<int*>(b + o_bad);
    a.Z = reinterpret_cast<float*>(b + o_Z);
    a.zh = reinterpret_cast<uint16_t*>(b + o_zh);
    a.zl = reinterpret_cast<uint16_t*>(b + o_zl);
    a.yp = reinterpret_cast<float*>(b + o_yp);
    C->bxdev = reinterpret_cast<float*>(b + o_bx);
    C->bydev = reinterpret_cast<float*>(b + o_by);
    return SG_OK;
}
}  // namespace

namespace {
int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

constexpr int kTcBlk = 128;   // block capacity of the tensor-core kernel (rows of an M = 128 tile)
constexpr int kTcSMax = 4;    // block ranges of the down units (the y finisher sums <= 4)
constexpr int kTcKTMax = 4;   // K slices of the predictor's T units (the finisher sums <= 4)

// blocks of a layer at most: one per SM, or D / 128 for very wide layers
size_t tc_block_cap(const sg_ctx* C) {
    return std::max<size_t>(static_cast<size_t>(C->G), (static_cast<size_t>(C->max_D) + kTcBlk - 1) / kTcBlk) + 8;
}

sg_status tc_workspace(sg_ctx* C) {
    if (C->tmem_ws) return SG_OK;
    const size_t pd = static_cast<size_t>(C->pitch_dmax);
    const size_t nblk = tc_block_cap(C), ndt = (pd + 127) / 128, Dm = static_cast<size_t>(C->max_D);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off += (bytes + 255) / 256 * 256;
        return o;
    };
    const size_t o_x = take(128 * pd * 2), o_tp = take(kTcKTMax * 256 * 64 * 4), o_th = take(128 * 256 * 2),
                 o_mb = take(Dm * 8), o_vb = take(Dm * 8), o_vl = take(nblk * kTcBlk * 4), o_vc = take(nblk * 4),
                 o_z = take(128 * nblk * kTcBlk * 2), o_y = take(kTcSMax * ndt * 128 * 64 * 4),
                 o_cnt = take((64 + 64 + 4) * 4),
                 o_fl = take(static_cast<size_t>(sg::tc_flag_ints(static_cast<int>(nblk), static_cast<int>(ndt))) * 4);
    DeviceGuard dg(C->device);
    cudaError_t e = cudaMalloc(&C->tmem_ws, off);
    if (e == cudaSuccess) e = cudaMemset(C->tmem_ws, 0, off);
    if (e != cudaSuccess) {
        C->tmem_ws = nullptr;
        return fail(SG_ERR_CUDA, std::string("tensor-core batch workspace: ") + cudaGetErrorString(e));
    }
    char* b = static_cast<char*>(C->tmem_ws);
    sg::TcArgs& a = C->tw;
    a.xhl = reinterpret_cast<uint16_t*>(b + o_x);
    a.tpart = reinterpret_cast<float*>(b + o_tp);
    a.thl = reinterpret_cast<uint16_t*>(b + o_th);
    a.mbits = reinterpret_cast<uint64_t*>(b + o_mb);
    a.vbits = reinterpret_cast<uint64_t*>(b + o_vb);
    a.vlist = reinterpret_cast<int*>(b + o_vl);
    a.vcnt = reinterpret_cast<int*>(b + o_vc);
    a.zhl = reinterpret_cast<uint16_t*>(b + o_z);
    a.ypart = reinterpret_cast<float*>(b + o_y);
    a.pcount = reinterpret_cast<int*>(b + o_cnt);
    a.vcount = a.pcount + 64;
    a.bad = a.pcount + 128;
    a.flags = reinterpret_cast<int*>(b + o_fl);
    a.zpitch = static_cast<int>(nblk * kTcBlk);
    a.xpitch = static_cast<int>(pd);
    return SG_OK;
}

// Largest divisor k <= want of the 64-wide K chunks of pitch (so each slice is whole chunks).
int k_slices(int pitch, int want) {
    const int chunks = pitch / 64;
    for (int k = std::min(want, chunks); k > 1; --k)
        if (chunks % k == 0) return k;
    return 1;
}

// The claim order of the tensor-core kernel's units (sg_batch_tc.cu): X, the T
// slices, the GU blocks, with each block range's DOWN units merged in `lag` claims
// after the range's last GU block (about one wave of the grid: by then the range's
// blocks are streaming in), so no unit waits for a whole previous phase.
// Topological by construction.
std::vector<int> tc_schedule(const sg::TcArgs& a, int NX, int KT, int lag, int NPF) {
    auto code = [](int t, int i, int j) { return (t << 24) | (i << 8) | j; };
    enum { X = 1, T, GU, DOWN, PF };  // sg_batch_tc.cu UnitType
    std::vector<int> order;
    for (int k = 0; k < NX; ++k) order.push_back(code(X, k, 0));
    for (int h = 0; h < (a.r > 128 ? 2 : 1); ++h)
        for (int k = 0; k < KT; ++k) order.push_back(code(T, k, h));
    struct Item {
        int code, ready_at;
    };
    std::vector<Item> downs;
    // range sr: chunks of rchunk blocks sr, sr + S, ... (sg_batch_tc.cu range_block); its last block
    const int kTcChunk = a.rchunk;
    const int chunks = (a.nblk + kTcChunk - 1) / kTcChunk;
    auto range_last = [&](int sr) {
        if (sr >= chunks) return -1;
        const int p = sr + (chunks - 1 - sr) / a.S * a.S;
        return std::min(a.nblk - 1, kTcChunk * p + kTcChunk - 1);
    };
    size_t di = 0;
    for (int b = 0; b < a.nblk; ++b) {
        while (di < downs.size() && downs[di].ready_at <= static_cast<int>(order.size()))
            order.push_back(downs[di++].code);
        order.push_back(code(GU, b, 0));
        for (int sr = 0; sr < a.S; ++sr)
            if (b == range_last(sr))
                for (int dt = 0; dt < a.ndt; ++dt)
                    downs.push_back({code(DOWN, dt, sr), static_cast<int>(order.size()) + lag});
    }

    for (; di < downs.size(); ++di) order.push_back(downs[di].code);
    for (int k = 0; k < NPF; ++k) order.push_back(code(PF, k, 0));  // claimed by SMs without down work
    return order;
}

// One tensor-core launch: B tokens through one layer (dense != 0: every row, no predictor).
sg_status tc_forward(sg_ctx* C, const sg_layer* L, const float* xs, int B, float* ys, void* stream,
                     int dense, const float* xres = nullptr, const sg_layer* next = nullptr,
                     const float* next_xs = nullptr) {
    if (sg_status s = tc_workspace(C); s != SG_OK) return s;
    sg::TcArgs a = C->tw;
    a.B = B;
    a.nb = (B + 7) / 8 * 8;
    a.N = 2 * a.nb;
    a.d = static_cast<int>(L->d);
    a.D = static_cast<int>(L->D_local);
    a.r = static_cast<int>(L->r);
    a.pitch_d = L->pitch_d;
    a.pitch_r = L->pitch_r;
    a.act = L->act;
    a.brows = L->tc_brows;
    a.nblk = (a.D + a.brows - 1) / a.brows;
    if (static_cast<size_t>(a.nblk) > tc_block_cap(C))
        return fail(SG_ERR_USAGE, "tensor-core batch: layer has more blocks than the ctx workspace holds");
    a.ndt = (a.pitch_d + 127) / 128;  // d tiles of 128 outputs (the down units' M)
    a.dense = dense;
    // a block's down rows stream whole once its survivors reach this density (per
    // 1024; SG_TC_TILE_U): a row gather moves a fraction of the tile rate per SM (on
    // B200 even a block with a sixth of its rows surviving streams faster whole), so by
    // default every block with a survivor is tiled and only empty blocks are skipped
    a.tile_u = env_int("SG_TC_TILE_U", 1);
    a.dbg = env_int("SG_TC_DBG", 0);
    a.x = xs;
    a.xres = xres;
    a.y = ys;
    a.bias = L->view.bias;
    a.ud = L->view.ud;
    // default: S contiguous block ranges (longest runs of tiled blocks, fewest walker
    // steps); SG_TC_RCHUNK = c > 0 interleaves chunks of c blocks, -1 picks ~8-block
    // chunks with the chunk count a multiple of S (138 blocks: 16 chunks of 9)
    a.S = std::max(1, std::min({env_int("SG_TC_S", 4), kTcSMax, a.nblk}));
    a.rchunk = env_int("SG_TC_RCHUNK", 0);  // default: contiguous ranges (measured best once the walk was cheap)
    if (a.rchunk < 0) {
        a.rchunk = 8;
        for (int k = std::max(1, (a.nblk + 4 * a.S) / (8 * a.S)); k >= 1; --k) {
            const int c = (a.nblk + a.S * k - 1) / (a.S * k);
            if ((a.nblk + c - 1) / c == a.S * k) {
                a.rchunk = c;
                break;
            }
        }
    }
    if (a.rchunk == 0) a.rchunk = (a.nblk + a.S - 1) / a.S;
    a.S = std::max(1, std::min(a.S, (a.nblk + a.rchunk - 1) / a.rchunk));  // each range: >= 1 chunk
    const int KT = dense ? 0 : k_slices(a.pitch_d, kTcKTMax);
    a.kst = KT ? a.pitch_d / KT : 0;
    a.kt = KT;
    // x -> X^T hi / lo: about 256 (token, 8-column) items per unit, so each epilogue
    // thread issues its loads in one round
    // the previous launch may have written this call's X^T already (x = h + y formed in its
    // y finishers): then no X units
    const auto& pp = C->tc_prep;
    a.x_ready = pp.valid && pp.layer == L && pp.batch == B &&
                ((xs == pp.h && xres == pp.y) || (pp.h == nullptr && xres == nullptr && xs == pp.y));
    // (up to 32 tokens: past that the finishers' extra X^T stores cost more than the X
    // split they save, measured B = 64 106 -> 111 µs/layer)
    a.prep = next != nullptr && next != L && next->d == L->d && next->pitch_d == L->pitch_d && a.nb <= 32 ? 1 : 0;
    a.nh = next_xs;
    C->tc_prep.valid = a.prep != 0;
    C->tc_prep.layer = next;
    C->tc_prep.h = next_xs;
    C->tc_prep.y = ys;
    C->tc_prep.batch = B;
    const int NX = a.x_ready ? 0 : std::max(8, std::min(128, a.nb * (a.pitch_d / 8) / 256));
    a.u_T = NX;
    a.u_GU = a.u_T + KT * (a.r > 128 ? 2 : 1);
    a.u_DOWN = a.u_GU + a.nblk;
    // L2 prefetch of the next layer's gate / up rows (their leading SG_TC_PF eighths)
    const int pf8 = env_int("SG_TC_PF", 0);  // measured neutral to slower with evict-first weights: off
    const int NPF = (next != nullptr && next->has_w && pf8 > 0) ? 32 : 0;
    a.pf_gate = NPF ? next->view.gate : nullptr;
    a.pf_ud = NPF ? next->view.ud : nullptr;
    a.pf_D = NPF ? static_cast<int>(next->D_local) : 0;
    a.pf_pitch = NPF ? next->pitch_d : 0;
    a.pf_units = NPF;
    a.pf_bytes = NPF ? static_cast<uint32_t>(next->pitch_d * 2 * std::min(pf8, 8) / 8 / 16 * 16) : 0;
    a.u_end = a.u_DOWN + a.ndt * a.S + NPF;
    {  // the claim order for this unit geometry, uploaded once per ctx (graph-capture safe after)
        const int lag = env_int("SG_TC_LAG", C->G);
        std::vector<int> key = {a.nblk, a.ndt, a.S, a.dense, NX, KT, lag, NPF, a.rchunk};  // (NX = 0: X^T prepared)
        auto oit = C->tc_orders.find(key);
        if (oit == C->tc_orders.end()) {
            const std::vector<int> order = tc_schedule(a, NX, KT, lag, NPF);
            if (static_cast<int>(order.size()) != a.u_end)
                return fail(SG_ERR_CUDA, "tensor-core schedule: unit count mismatch");
            int* dev = nullptr;
            DeviceGuard dg0(C->device);
            SG_CUDA(cudaMalloc(&dev, order.size() * sizeof(int)));
            SG_CUDA(cudaMemcpy(dev, order.data(), order.size() * sizeof(int), cudaMemcpyHostToDevice));
            oit = C->tc_orders.emplace(key, dev).first;
        }
        a.order = oit->second;
        a.n_units = a.u_end;
    }
    a.trace = C->tc_trace_on && C->tc_trace_cap >= static_cast<size_t>(a.n_units) ? C->tc_trace : nullptr;
    C->tc_last_units = a.n_units;
    C->tc_last_order = a.order;
    // workspace maps for this nb (box height N), cached per ctx
    auto it = C->tcmaps_ws.find(a.nb);
    if (it == C->tcmaps_ws.end()) {
        sg::TcMaps m{};
        if (!make_map(&m.xhl, a.xhl, C->pitch_dmax, a.N, C->pitch_dmax, a.N) ||
            !make_map(&m.thl, a.thl, 256, a.N, 256, a.N) ||
            !make_map(&m.zhl, a.zhl, a.zpitch, a.N, a.zpitch, a.N))
            return fail(SG_ERR_CUDA, "cuTensorMapEncodeTiled failed (workspace maps)");
        it = C->tcmaps_ws.emplace(a.nb, m).first;
    }
    // the workspace pitches are the ctx maxima: X^T / T^T rows use them
    sg::TcMaps maps = L->tcmaps;
    maps.xhl = it->second.xhl;
    maps.thl = it->second.thl;
    maps.zhl = it->second.zhl;
    DeviceGuard dg(C->device);
    // (no memset between launches: a graph node between two launches would cut their
    // programmatic dependent launch; the kernel's last CTA publishes and re-zeroes the
    // non-finite flag itself)
    const int e = sg::launch_batch_tc(maps, a, C->G, stream);
    if (e != 0) return fail(SG_ERR_CUDA, std::string("tensor-core batch launch: ") +
                                             cudaGetErrorString(static_cast<cudaError_t>(e)));
    return SG_OK;
}
}  // namespace

sg_status sg_ffn_forward_batch(sg_ctx* C, const sg_layer* L, const float* xs, int32_t batch,
                               float* ys, void* stream) {
    if (sg_status s = check_pair(C, L); s != SG_OK) return s;
    if (!L->has_pred || !L->has_w) return fail(SG_ERR_USAGE, "batched decode needs weights and a predictor");
    if (batch < 1 || batch > sg::batch_max())
        return fail(SG_ERR_USAGE, "batch must be in [1, " + std::to_string(sg::batch_max()) + "]");
    if (xs == nullptr || ys == nullptr) return fail(SG_ERR_USAGE, "null buffers");
    if (sg_status s = batch_workspace(C); s != SG_OK) return s;
    DeviceGuard dg(C->device);
    if (batch <= small_batch_limit() && batch <= kMaxStackLayers) {
        C->tc_prep.valid = false;  // (a prepared X^T is for the tensor-core call that follows it)
        // few tokens: one persistent launch with token b as "layer" b of a stack
        // (unchained; same per-token results), predicted / survivor bits per token
        auto st = static_cast<cudaStream_t>(stream);
        const size_t bits = static_cast<size_t>(L->D_local) * sizeof(uint64_t);
        SG_CUDA(cudaMemsetAsync(C->bw.mbits, 0, bits, st));
        SG_CUDA(cudaMemsetAsync(C->bw.vbits, 0, bits, st));
        std::vector<const sg_layer*> rep(static_cast<size_t>(batch), L);
        if (sg_status s = stack_launch(C, rep.data(), batch, SG_PIPELINE_SEQUENTIAL, xs, ys, 0, stream,
                                       reinterpret_cast<unsigned long long*>(C->bw.mbits),
                                       reinterpret_cast<unsigned long long*>(C->bw.vbits), L->repdev);
            s != SG_OK)
            return s;
        C->blast = L;
        C->blast_B = batch;
        C->blast_stack = true;
        C->blast_path = 0;
        return SG_OK;
    }
    if (L->has_tcmaps && L->r <= 256 && L->d <= 8192 && !env_int("SG_BATCH_LEGACY", 0)) {
        // tensor cores: one persistent tcgen05 launch (sg_batch_tc.cu)
        if (sg_status s = tc_forward(C, L, xs, batch, ys, stream, 0); s != SG_OK) return s;
        C->blast = L;
        C->blast_B = batch;
        C->blast_stack = false;
        C->blast_path = 2;
        return SG_OK;
    }
    C->tc_prep.valid = false;
    sg::BatchArgs a = C->bw;
    a.B = batch;
    // split-K of the gate / up GEMMs: enough CTAs for ~2 full waves of the union
    // tiles (measured at the 7B shape: 7 best up to B = 32, 4 at B = 64)
    if (a.gsplit == 0) a.gsplit = batch <= 32 ? 7 : 4;
    // split-K of the down GEMM (B > 16; measured at the 7B shape with the stage
    // depths below, B = 32: 4 best; B = 64: split 4 / 8 / 12 = 29.6k / 33.5k / 31.5k
    // tokens/s)
    if (a.dsplit == 0) a.dsplit = batch <= 32 ? 4 : 8;
    {  // cp.async depth of the GEMM tiles (SG_BATCH_STAGES overrides: 2, 3, 4 or 6)
        static const int st = [] {
            const char* e = std::getenv("SG_BATCH_STAGES");
            return e ? std::atoi(e) : 0;
        }();
        // measured at the 7B shape (8-layer stack), 64-wide K chunks: B = 64: 6 / 4 /
        // 3 / 2 stages = 19.3k / 26.0k / 26.0k / 31.5k tokens/s (smem per CTA bounds
        // the CTAs per SM, and the tiles are latency-bound per warp); 32-wide K
        // chunks (shipped): B = 64: 4 / 3 / 2 = 28.7k / 33.5k / 31.6k, B = 32:
        // 19.4k / 19.1k / 18.0k; B <= 16 (T / mask tiles only): no difference
        a.stages = st >= 2 && st <= 4 ? st : st == 6 ? 6 : (batch > 32 ? 3 : 4);
    }
    a.nb = (batch + 7) / 8 * 8;
    a.d = static_cast<int>(L->d);
    a.D = static_cast<int>(L->D_local);
    a.r = static_cast<int>(L->r);
    a.pitch_d = L->pitch_d;
    a.pitch_r = L->pitch_r;
    a.act = L->act;
    a.Bm = L->view.B;
    a.A = L->view.A;
    a.bias = L->view.bias;
    a.gate = L->view.gate;
    a.ud = L->view.ud;
    a.gate = L->view.gate;
    a.ud = L->view.ud;
    SG_CUDA(cudaMemsetAsync(a.bad, 0, sizeof(int), static_cast<cudaStream_t>(stream)));
    const int e = sg::launch_batch(a, xs, ys, stream);
    if (e != 0) return fail(SG_ERR_CUDA, std::string("batch launch: ") +
                                             cudaGetErrorString(static_cast<cudaError_t>(e)));
    C->blast = L;
    C->blast_B = batch;
    C->blast_stack = false;
    C->blast_path = 1;
    return SG_OK;
}

sg_status sg_ffn_forward_batch_dense(sg_ctx* C, const sg_layer* L, const float* xs, int32_t batch,
                                     float* ys, void* stream) {
    if (sg_status s = check_pair(C, L); s != SG_OK) return s;
    if (!L->has_w || !L->has_tcmaps) return fail(SG_ERR_USAGE, "dense batched decode needs weights");
    if (batch < 1 || batch > 64) return fail(SG_ERR_USAGE, "batch must be in [1, 64]");
    if (xs == nullptr || ys == nullptr) return fail(SG_ERR_USAGE, "null buffers");
    if (L->d > 8192) return fail(SG_ERR_USAGE, "hidden too large for the tensor-core path");
    if (sg_status s = tc_forward(C, L, xs, batch, ys, stream, 1); s != SG_OK) return s;
    C->blast = L;
    C->blast_B = batch;
    C->blast_stack = false;
    C->blast_path = 3;
    return SG_OK;
}

sg_status sg_ffn_forward_batch_res(sg_ctx* C, const sg_layer* L, const float* xs, const float* xres,
                                   int32_t batch, float* ys, int32_t dense, const sg_layer* next,
                                   const float* next_xs, void* stream) {
    if (xres == nullptr && next == nullptr && !(C && C->tc_prep.valid))
        return dense ? sg_ffn_forward_batch_dense(C, L, xs, batch, ys, stream)
                     : sg_ffn_forward_batch(C, L, xs, batch, ys, stream);
    if (sg_status s = check_pair(C, L); s != SG_OK) return s;
    if (batch == 1 && !dense && L->has_pred && L->has_w) {
        // one token: the persistent single-token executor with the residual formed while
        // x is staged (the tensor-core launch would stream every gate / up row for it)
        if (xs == nullptr || ys == nullptr) return fail(SG_ERR_USAGE, "null buffers");
        if (sg_status s = batch_workspace(C); s != SG_OK) return s;
        C->tc_prep.valid = false;
        DeviceGuard dg(C->device);
        auto st = static_cast<cudaStream_t>(stream);
        const size_t bits = static_cast<size_t>(L->D_local) * sizeof(uint64_t);
        SG_CUDA(cudaMemsetAsync(C->bw.mbits, 0, bits, st));
        SG_CUDA(cudaMemsetAsync(C->bw.vbits, 0, bits, st));
        SG_CUDA(cudaMemsetAsync(C->W.stats, 0, 4 * sizeof(int), st));
        sg::WorkView W = work_for(C, xs, ys);
        W.xres = xres;
        W.mbits = reinterpret_cast<unsigned long long*>(C->bw.mbits);
        W.vbits = reinterpret_cast<unsigned long long*>(C->bw.vbits);
        W.bitpos = 0;
        const int e = sg::launch_layer(L->view, W, SG_PIPELINE_SEQUENTIAL, C->G, stream);
        if (e != 0) return fail(SG_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(static_cast<cudaError_t>(e)));
        C->blast = L;
        C->blast_B = 1;
        C->blast_stack = true;
        C->blast_path = 0;
        return SG_OK;
    }
    if (!L->has_w || !L->has_tcmaps || (!dense && !L->has_pred) || L->r > 256 || L->d > 8192)
        return fail(SG_ERR_USAGE, "residual batched decode runs on the tensor-core path only");
    if (batch < 1 || batch > 64) return fail(SG_ERR_USAGE, "batch must be in [1, 64]");
    if (xs == nullptr || ys == nullptr) return fail(SG_ERR_USAGE, "null buffers");
    if (sg_status s = batch_workspace(C); s != SG_OK) return s;
    DeviceGuard dg(C->device);
    if (next != nullptr && next->device != L->device) return fail(SG_ERR_USAGE, "next layer on another device");
    if (sg_status s = tc_forward(C, L, xs, batch, ys, stream, dense ? 1 : 0, xres, next, next_xs); s != SG_OK)
        return s;
    C->blast = L;
    C->blast_B = batch;
    C->blast_stack = false;
    C->blast_path = dense ? 3 : 2;
    return SG_OK;
}

sg_status sg_ctx_enable_tc_trace(sg_ctx* C, int32_t max_units) {
    if (C == nullptr || max_units < 0) return fail(SG_ERR_USAGE, "bad arguments");
    DeviceGuard dg(C->device);
    if (C->tc_trace) cudaFree(C->tc_trace);
    C->tc_trace = nullptr;
    C->tc_trace_cap = 0;
    C->tc_trace_on = max_units > 0;
    if (max_units > 0) {
        SG_CUDA(cudaMalloc(&C->tc_trace, static_cast<size_t>(max_units) * 8 * 8));
        SG_CUDA(cudaMemset(C->tc_trace, 0, static_cast<size_t>(max_units) * 8 * 8));
        C->tc_trace_cap = static_cast<size_t>(max_units);
    }
    return SG_OK;
}

sg_status sg_ctx_read_tc_trace(sg_ctx* C, void* stream, int32_t max_units, uint64_t* out, int32_t* n_units) {
    if (C == nullptr || out == nullptr || !C->tc_trace) return fail(SG_ERR_USAGE, "tc trace not enabled");
    DeviceGuard dg(C->device);
    SG_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    const int n = std::min<int>(max_units, C->tc_last_units);
    SG_CUDA(cudaMemcpy(out, C->tc_trace, static_cast<size_t>(n) * 8 * 8, cudaMemcpyDeviceToHost));
    if (n_units) *n_units = n;
    return SG_OK;
}

sg_status sg_tc_unit_codes(sg_ctx* C, int32_t* out, int32_t max_units) {
    if (C == nullptr || out == nullptr || C->tc_last_order == nullptr) return fail(SG_ERR_USAGE, "no tc call");
    DeviceGuard dg(C->device);
    const int n = std::min<int>(max_units, C->tc_last_units);
    SG_CUDA(cudaMemcpy(out, C->tc_last_order, static_cast<size_t>(n) * 4, cudaMemcpyDeviceToHost));
    return SG_OK;
}

sg_status sg_ctx_read_batch(sg_ctx* C, void* stream, int32_t batch, sg_exec_stats* stats,
                            uint64_t* pred_bits, uint64_t* surv_bits) {
    if (C == nullptr || C->blast == nullptr) return fail(SG_ERR_USAGE, "no batched call on this ctx");
    if (batch != C->blast_B) return fail(SG_ERR_USAGE, "batch differs from the last batched call");
    DeviceGuard dg(C->device);
    SG_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    const sg_layer* L = C->blast;
    int pc[64], vc[64];
    bool bad = false;
    if (C->blast_stack) {
        std::vector<int> st4(static_cast<size_t>(batch) * 4);
        SG_CUDA(cudaMemcpy(st4.data(), C->W.stats, st4.size() * sizeof(int), cudaMemcpyDeviceToHost));
        for (int b = 0; b < batch; ++b) {
            pc[b] = st4[4 * b];
            vc[b] = st4[4 * b + 1];
            bad |= st4[4 * b + 2] != 0;  // the device non-finite flag of token b
        }
    } else if (C->blast_path >= 2) {
        // tensor-core path: the per-token counts are the bit columns' popcounts (the
        // kernel keeps only the bits)
        int flag = 0;
        SG_CUDA(cudaMemcpy(&flag, C->tw.bad + 1, sizeof(int), cudaMemcpyDeviceToHost));  // published copy
        bad = flag != 0;
        std::vector<uint64_t> mb(static_cast<size_t>(L->D_local)), vb(static_cast<size_t>(L->D_local));
        if (C->blast_path == 2)
            SG_CUDA(cudaMemcpy(mb.data(), C->tw.mbits, sizeof(uint64_t) * mb.size(), cudaMemcpyDeviceToHost));
        SG_CUDA(cudaMemcpy(vb.data(), C->tw.vbits, sizeof(uint64_t) * vb.size(), cudaMemcpyDeviceToHost));
        for (int b = 0; b < batch; ++b) pc[b] = vc[b] = 0;
        for (size_t n = 0; n < vb.size(); ++n)
            for (int b = 0; b < batch; ++b) {
                pc[b] += static_cast<int>((mb[n] >> b) & 1ull);
                vc[b] += static_cast<int>((vb[n] >> b) & 1ull);
            }
    } else {
        int flag = 0;
        SG_CUDA(cudaMemcpy(pc, C->bw.pcount, sizeof(int) * batch, cudaMemcpyDeviceToHost));
        SG_CUDA(cudaMemcpy(vc, C->bw.vcount, sizeof(int) * batch, cudaMemcpyDeviceToHost));
        SG_CUDA(cudaMemcpy(&flag, C->bw.bad, sizeof(int), cudaMemcpyDeviceToHost));
        bad = flag != 0;
    }
    const int pipe = C->blast_path == 3 ? SG_PIPELINE_DENSE : SG_PIPELINE_SEQUENTIAL;
    for (int b = 0; stats && b < batch; ++b) stats[b] = make_stats(L, pipe, pc[b], vc[b]);
    const bool tc = C->blast_path >= 2;
    if (pred_bits)
        SG_CUDA(cudaMemcpy(pred_bits, tc ? C->tw.mbits : C->bw.mbits, sizeof(uint64_t) * L->D_local,
                           cudaMemcpyDeviceToHost));
    if (surv_bits)
        SG_CUDA(cudaMemcpy(surv_bits, tc ? C->tw.vbits : C->bw.vbits, sizeof(uint64_t) * L->D_local,
                           cudaMemcpyDeviceToHost));
    if (bad) return fail(SG_ERR_DATA, "ffn input has non-finite entries");  // ffn_exec.hpp:61-63
    return SG_OK;
}

sg_status sg_ffn_forward_batch_host(sg_ctx* C, const sg_layer* L, const float* xs_host,
                                    int32_t batch, float* ys_host, sg_exec_stats* stats,
                                    void* stream) {
    if (sg_status s = check_pair(C, L); s != SG_OK) return s;
    if (xs_host == nullptr || ys_host == nullptr || batch < 1 || batch > sg::batch_max())
        return fail(SG_ERR_USAGE, "bad batch buffers");
    for (int64_t i = 0; i < static_cast<int64_t>(batch) * L->d; ++i)
        if (!std::isfinite(xs_host[i])) return fail(SG_ERR_DATA, "input: non-finite entries");
    if (sg_status s = batch_workspace(C); s != SG_OK) return s;
    DeviceGuard dg(C->device);
    auto st = static_cast<cudaStream_t>(stream);
    const size_t bytes = static_cast<size_t>(batch) * L->d * 4;
    SG_CUDA(cudaMemcpyAsync(C->bxdev, xs_host, bytes, cudaMemcpyHostToDevice, st));
    if (sg_status s = sg_ffn_forward_batch(C, L, C->bxdev, batch, C->bydev, stream); s != SG_OK) return s;
    SG_CUDA(cudaMemcpyAsync(ys_host, C->bydev, bytes, cudaMemcpyDeviceToHost, st));
    return sg_ctx_read_batch(C, stream, batch, stats, nullptr, nullptr);
}

sg_status sg_ffn_forward_device(sg_ctx* C, const sg_layer* L, sg_pipeline pipeline,
                                const float* x, float* y, void* stream) {
    if (sg_status s = check_pair(C, L); s != SG_OK) return s;
    if (pipeline != SG_PIPELINE_DENSE && !L->has_pred)
        return fail(SG_ERR_USAGE, "sparse pipeline needs a layer with a predictor");
    if (pipeline < 0 || pipeline > 2) return fail(SG_ERR_USAGE, "bad pipeline");
    if (!L->has_w) return fail(SG_ERR_USAGE, "predictor-only layer cannot run the FFN");
    if (x == nullptr || y == nullptr) return fail(SG_ERR_USAGE, "null x/y");
    DeviceGuard dg(L->device);
    // per-layer counts are accumulated with integer atomics by the kernel
    SG_CUDA(cudaMemsetAsync(C->W.stats, 0, 4 * sizeof(int), static_cast<cudaStream_t>(stream)));
    const int e = sg::launch_layer(L->view, work_for(C, x, y), pipeline, C->G, stream);
    if (e != 0) {
        return fail(SG_ERR_CUDA, std::string("launch: ") +
                                     cudaGetErrorString(static_cast<cudaError_t>(e)));
    }
    C->last_layer = L;
    C->last_pipeline = pipeline;
    return SG_OK;
}

sg_status sg_ctx_read_stats(sg_ctx* C, void* stream, sg_exec_stats* out) {
    if (C == nullptr || out == nullptr) return fail(SG_ERR_USAGE, "null argument");
    if (C->last_layer == nullptr) return fail(SG_ERR_USAGE, "no forward call on this ctx");
    DeviceGuard dg(C->device);
    SG_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    int st[4];
    SG_CUDA(cudaMemcpy(st, C->W.stats, sizeof(st), cudaMemcpyDeviceToHost));
    const int pipe = C->last_pipeline;
    const int64_t p = pipe == SG_PIPELINE_DENSE ? C->last_layer->D_local : st[0];
    const int64_t v = pipe == SG_PIPELINE_DENSE ? C->last_layer->D_local : st[1];
    *out = make_stats(C->last_layer, pipe, p, v);
    if (st[2] != 0) return fail(SG_ERR_DATA, "ffn input has non-finite entries");
    return SG_OK;
}

sg_status sg_ctx_read_sets(sg_ctx* C, void* stream, int32_t* P, int64_t* p, int32_t* V, int64_t* v,
                           float* g, float* z) {
    if (C == nullptr) return fail(SG_ERR_USAGE, "null ctx");
    if (C->last_layer == nullptr || C->last_pipeline == SG_PIPELINE_DENSE)
        return fail(SG_ERR_USAGE, "no sparse forward call on this ctx");
    DeviceGuard dg(C->device);
    SG_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    int st[4];
    SG_CUDA(cudaMemcpy(st, C->W.stats, sizeof(st), cudaMemcpyDeviceToHost));
    if (p) *p = st[0];
    if (v) *v = st[1];
    if (P && st[0] > 0) SG_CUDA(cudaMemcpy(P, C->W.P, st[0] * 4, cudaMemcpyDeviceToHost));
    if (g && st[0] > 0) SG_CUDA(cudaMemcpy(g, C->W.gP, st[0] * 4, cudaMemcpyDeviceToHost));
    if (V && st[1] > 0) SG_CUDA(cudaMemcpy(V, C->W.V, st[1] * 4, cudaMemcpyDeviceToHost));
    if (z && st[1] > 0) SG_CUDA(cudaMemcpy(z, C->W.zV, st[1] * 4, cudaMemcpyDeviceToHost));
    if (!C->last_layer->gidx.empty()) {
        // segments follow the layout order: report ascending global indices
        auto sort_pairs = [](int32_t* idx, float* val, int n) {
            if (!idx || n <= 1) return;
            std::vector<std::pair<int32_t, float>> t(static_cast<size_t>(n));
            for (int i = 0; i < n; ++i) t[static_cast<size_t>(i)] = {idx[i], val ? val[i] : 0.f};
            std::sort(t.begin(), t.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
            for (int i = 0; i < n; ++i) {
                idx[i] = t[static_cast<size_t>(i)].first;
                if (val) val[i] = t[static_cast<size_t>(i)].second;
            }
        };
        sort_pairs(P, g, st[0]);
        sort_pairs(V, z, st[1]);
    }
    return SG_OK;
}

sg_status sg_predict_mask(sg_ctx* C, const sg_layer* L, const void* x, sg_dtype x_dtype,
                          int64_t x_len, uint8_t* mask, int64_t* count, void* stream) {
    if (sg_status s = check_pair(C, L); s != SG_OK) return s;
    if (!L->has_pred) return fail(SG_ERR_USAGE, "layer has no predictor");
    if (sg_status s = read_x(x, x_dtype, x_len, L->d, C->xpin, "predictor"); s != SG_OK) return s;
    DeviceGuard dg(L->device);
    auto st = static_cast<cudaStream_t>(stream);
    SG_CUDA(cudaMemcpyAsync(C->xdev, C->xpin, L->d * 4, cudaMemcpyHostToDevice, st));
    SG_CUDA(cudaMemsetAsync(C->W.stats, 0, 4 * sizeof(int), st));
    const int e = sg::launch_predict(L->view, work_for(C, C->xdev, C->ydev), C->maskdev, C->G, st);
    if (e != 0) return fail(SG_ERR_CUDA, std::string("launch: ") +
                                             cudaGetErrorString(static_cast<cudaError_t>(e)));
    int stv[4];
    SG_CUDA(cudaMemcpyAsync(stv, C->W.stats, sizeof(stv), cudaMemcpyDeviceToHost, st));
    if (mask) SG_CUDA(cudaMemcpyAsync(mask, C->maskdev, L->D_local, cudaMemcpyDeviceToHost, st));
    SG_CUDA(cudaStreamSynchronize(st));
    if (count) *count = stv[0];
    return SG_OK;
}

sg_status sg_ffn_forward(sg_ctx* C, const sg_layer* L, sg_pipeline pipeline, const void* x,
                         sg_dtype x_dtype, int64_t x_len, void* y, sg_dtype y_dtype,
                         sg_exec_stats* stats, void* stream) {
    if (sg_status s = check_pair(C, L); s != SG_OK) return s;
    if (y == nullptr) return fail(SG_ERR_USAGE, "null y");
    if (y_dtype != SG_F64 && y_dtype != SG_F32) return fail(SG_ERR_USAGE, "y dtype must be f64/f32");
    if (sg_status s = read_x(x, x_dtype, x_len, L->d, C->xpin, "ffn"); s != SG_OK) return s;
    DeviceGuard dg(L->device);
    auto st = static_cast<cudaStream_t>(stream);
    SG_CUDA(cudaMemcpyAsync(C->xdev, C->xpin, L->d * 4, cudaMemcpyHostToDevice, st));
    if (sg_status s = sg_ffn_forward_device(C, L, pipeline, C->xdev, C->ydev, stream); s != SG_OK)
        return s;
    SG_CUDA(cudaMemcpyAsync(C->ypin, C->ydev, L->d * 4, cudaMemcpyDeviceToHost, st));
    sg_exec_stats tmp{};
    if (sg_status s = sg_ctx_read_stats(C, stream, &tmp); s != SG_OK) return s;
    if (stats) *stats = tmp;
    if (y_dtype == SG_F64) {
        auto* yd = static_cast<double*>(y);
        for (int64_t i = 0; i < L->d; ++i) yd[i] = static_cast<double>(C->ypin[i]);
    } else {
        std::memcpy(y, C->ypin, L->d * 4);
    }
    return SG_OK;
}

sg_status sg_ffn_forward_layers(sg_ctx* C, const sg_layer* const* layers, int32_t n,
                                sg_pipeline pipeline, const float* xs, float* ys, int32_t chain,
                                void* stream) {
    if (C != nullptr && C->stack_sets && n >= 1 && n <= 64 && pipeline != SG_PIPELINE_DENSE) {
        DeviceGuard dg(C->device);
        SG_CUDA(cudaMemsetAsync(C->sbits, 0, static_cast<size_t>(C->max_D) * 16,
                                static_cast<cudaStream_t>(stream)));
        const sg_status s = stack_launch(C, layers, n, pipeline, xs, ys, chain, stream, C->sbits,
                                         C->sbits + C->max_D);
        C->last_stack_bits = s == SG_OK;
        return s;
    }
    if (C) C->last_stack_bits = false;
    return stack_launch(C, layers, n, pipeline, xs, ys, chain, stream, nullptr, nullptr);
}

sg_status sg_ctx_enable_stack_sets(sg_ctx* C, int32_t enable) {
    if (C == nullptr) return fail(SG_ERR_USAGE, "null ctx");
    DeviceGuard dg(C->device);
    if (enable && C->sbits == nullptr)
        SG_CUDA(cudaMalloc(&C->sbits, static_cast<size_t>(C->max_D) * 16));
    C->stack_sets = enable != 0;
    return SG_OK;
}

sg_status sg_ctx_read_stack_sets(sg_ctx* C, void* stream, int32_t layer, int32_t* P, int64_t* p,
                                 int32_t* V, int64_t* v) {
    if (C == nullptr || !C->last_stack_bits)
        return fail(SG_ERR_USAGE, "no stack call recorded index sets on this ctx");
    if (layer < 0 || static_cast<size_t>(layer) >= C->last_stack.size() || layer >= 64)
        return fail(SG_ERR_USAGE, "layer out of range of the last stack call");
    DeviceGuard dg(C->device);
    SG_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    const sg_layer* L = C->last_stack[static_cast<size_t>(layer)];
    const size_t Dl = static_cast<size_t>(L->D_local);
    std::vector<unsigned long long> bits(2 * Dl);
    SG_CUDA(cudaMemcpy(bits.data(), C->sbits, Dl * 8, cudaMemcpyDeviceToHost));
    SG_CUDA(cudaMemcpy(bits.data() + Dl, C->sbits + C->max_D, Dl * 8, cudaMemcpyDeviceToHost));
    std::vector<int32_t> ps, vs;
    for (size_t k = 0; k < Dl; ++k) {
        const int32_t g = static_cast<int32_t>(local_to_global(L, static_cast<int64_t>(k)));
        if ((bits[k] >> layer) & 1ull) ps.push_back(g);
        if ((bits[Dl + k] >> layer) & 1ull) vs.push_back(g);
    }
    std::sort(ps.begin(), ps.end());
    std::sort(vs.begin(), vs.end());
    if (P) std::copy(ps.begin(), ps.end(), P);
    if (V) std::copy(vs.begin(), vs.end(), V);
    if (p) *p = static_cast<int64_t>(ps.size());
    if (v) *v = static_cast<int64_t>(vs.size());
    return SG_OK;
}


sg_status sg_ctx_enable_phase_timing(sg_ctx* C, int32_t max_layers) {
    if (C == nullptr || max_layers < 0) return fail(SG_ERR_USAGE, "bad arguments");
    DeviceGuard dg(C->device);
    if (C->dbgdev) cudaFree(C->dbgdev);
    C->dbgdev = nullptr;
    C->dbg_layers = 0;
    C->W.dbg = nullptr;
    if (max_layers == 0) return SG_OK;
    const size_t bytes = static_cast<size_t>(max_layers) * C->G * 32 * 8;
    SG_CUDA(cudaMalloc(&C->dbgdev, bytes));
    SG_CUDA(cudaMemset(C->dbgdev, 0, bytes));
    C->dbg_layers = max_layers;
    C->W.dbg = C->dbgdev;
    return SG_OK;
}

sg_status sg_ctx_read_phase_timing(sg_ctx* C, void* stream, int32_t n, uint64_t* out,
                                   int32_t* num_ctas) {
    if (C == nullptr || out == nullptr || n < 1 || n > C->dbg_layers)
        return fail(SG_ERR_USAGE, "phase timing not enabled for that many layers");
    DeviceGuard dg(C->device);
    SG_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    SG_CUDA(cudaMemcpy(out, C->dbgdev, static_cast<size_t>(n) * C->G * 32 * 8,
                       cudaMemcpyDeviceToHost));
    if (num_ctas) *num_ctas = C->G;
    return SG_OK;
}

sg_status sg_ctx_read_stack_stats(sg_ctx* C, void* stream, int32_t n, sg_exec_stats* out) {
    if (C == nullptr || out == nullptr) return fail(SG_ERR_USAGE, "null argument");
    if (n < 1 || static_cast<size_t>(n) > C->last_stack.size())
        return fail(SG_ERR_USAGE, "no stack call with that many layers on this ctx");
    DeviceGuard dg(C->device);
    SG_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    std::vector<int> st(4 * static_cast<size_t>(n));
    SG_CUDA(cudaMemcpy(st.data(), C->W.stats, st.size() * 4, cudaMemcpyDeviceToHost));
    bool bad = false;
    for (int l = 0; l < n; ++l) {
        const sg_layer* L = C->last_stack[l];
        const int pipe = C->last_pipeline;
        const int64_t p = pipe == SG_PIPELINE_DENSE ? L->D_local : st[4 * l];
        const int64_t v = pipe == SG_PIPELINE_DENSE ? L->D_local : st[4 * l + 1];
        out[l] = make_stats(L, pipe, p, v);
        bad |= st[4 * l + 2] != 0;
    }
    if (bad) return fail(SG_ERR_DATA, "ffn input has non-finite entries");
    return SG_OK;
}

sg_status sg_ffn_forward_layers_host(sg_ctx* C, const sg_layer* const* layers, int32_t n,
                                     sg_pipeline pipeline, const float* xs_host, float* ys_host,
                                     int32_t chain, sg_exec_stats* stats, void* stream) {
    if (C == nullptr || layers == nullptr || n < 1 || xs_host == nullptr || ys_host == nullptr)
        return fail(SG_ERR_USAGE, "bad arguments");
    const size_t d = static_cast<size_t>(layers[0]->d);
    const size_t need = d * static_cast<size_t>(n) * 4;
    DeviceGuard dg(C->device);
    if (C->xs_cap < need) {
        if (C->xsdev) cudaFree(C->xsdev);
        if (C->ysdev) cudaFree(C->ysdev);
        C->xsdev = C->ysdev = nullptr;
        C->xs_cap = 0;
        SG_CUDA(cudaMalloc(&C->xsdev, need));
        SG_CUDA(cudaMalloc(&C->ysdev, need));
        C->xs_cap = need;
    }
    auto st = static_cast<cudaStream_t>(stream);
    SG_CUDA(cudaMemcpyAsync(C->xsdev, xs_host, chain == 1 ? d * 4 : need, cudaMemcpyHostToDevice, st));
    if (sg_status s = sg_ffn_forward_layers(C, layers, n, pipeline, C->xsdev, C->ysdev, chain, stream);
        s != SG_OK)
        return s;
    SG_CUDA(cudaMemcpyAsync(ys_host, C->ysdev, need, cudaMemcpyDeviceToHost, st));
    if (stats) return sg_ctx_read_stack_stats(C, stream, n, stats);
    SG_CUDA(cudaStreamSynchronize(st));
    return SG_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// synthetic.hpp:15-108
// ---------------------------------------------------------------------------
static double normal_quantile(double p) {
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

template <typename Sink>
static sg_status synthetic_stream(int64_t hidden, int64_t inter, int64_t calib_tokens,
                                  int64_t eval_tokens, double ns, uint64_t seed, Sink&& sink) {
    if (hidden < 1 || inter < 1 || calib_tokens < 1 || eval_tokens < 0)
        return fail(SG_ERR_DATA, "synthetic fixture: invalid sizes");
    if (!(ns > 0.0 && ns < 1.0))
        return fail(SG_ERR_DATA, "synthetic fixture: natural sparsity must lie in (0, 1)");
    const auto d = static_cast<double>(hidden);
    const double z = normal_quantile(ns);
    double shift = z * std::sqrt(2.0);
    shift = z * std::sqrt(2.0 + shift * shift / d);
    std::mt19937_64 rng(seed);
    const double means[5] = {-shift / d, 0.0, 0.0, 1.0, 1.0};
    const double sds[5] = {1.0 / std::sqrt(d), 1.0 / std::sqrt(d),
                           1.0 / std::sqrt(static_cast<double>(inter)), 1.0, 1.0};
    const int64_t counts[5] = {inter * hidden, inter * hidden, hidden * inter,
                               hidden * calib_tokens, hidden * eval_tokens};
    for (int m = 0; m < 5; ++m) {
        std::normal_distribution<double> dist(means[m], sds[m]);  // fresh per matrix
        for (int64_t i = 0; i < counts[m]; ++i) sink(m, i, dist(rng));
    }
    return SG_OK;
}

extern "C" {

sg_status sg_synthetic_fixture(int64_t hidden, int64_t inter, int64_t calib_tokens,
                               int64_t eval_tokens, double ns, uint64_t seed, double* gate,
                               double* up, double* down, double* calib, double* eval) {
    double* outs[5] = {gate, up, down, calib, eval};
    return synthetic_stream(hidden, inter, calib_tokens, eval_tokens, ns, seed,
                            [&](int m, int64_t i, double v) {
                                if (outs[m]) outs[m][i] = v;
                            });
}

sg_status sg_synthetic_fixture_bf16(int64_t hidden, int64_t inter, int64_t calib_tokens,
                                    int64_t eval_tokens, double ns, uint64_t seed, uint16_t* gate,
                                    uint16_t* up, uint16_t* down_t, double* calib, double* eval) {
    return synthetic_stream(hidden, inter, calib_tokens, eval_tokens, ns, seed,
                            [&](int m, int64_t i, double v) {
                                switch (m) {
                                    case 0: if (gate) gate[i] = f32_to_bf16(static_cast<float>(v)); break;
                                    case 1: if (up) up[i] = f32_to_bf16(static_cast<float>(v)); break;
                                    case 2:
                                        if (down_t) {  // down is hidden x inter: (j, n) -> down_t[n, j]
                                            const int64_t j = i / inter, n = i % inter;
                                            down_t[n * hidden + j] = f32_to_bf16(static_cast<float>(v));
                                        }
                                        break;
                                    case 3: if (calib) calib[i] = v; break;
                                    default: if (eval) eval[i] = v; break;
                                }
                            });
}

// ---------------------------------------------------------------------------
// calibration.hpp:61-96 (build_instance) + :128-205 (greedy_calibrate)
// ---------------------------------------------------------------------------
sg_status sg_greedy_calibrate(const double* scores, const double* weights, int64_t D, int64_t T,
                              int32_t eta, double target, double* bias, double* achieved,
                              double* total_damage) {
    if (scores == nullptr || weights == nullptr || bias == nullptr) return fail(SG_ERR_USAGE, "null argument");
    if (D < 1 || T < 1) return fail(SG_ERR_DATA, "calibration instance: need at least one neuron and one sample");
    if (eta < 1) return fail(SG_ERR_DATA, "calibration instance: eta must be >= 1");
    for (int64_t i = 0; i < D * T; ++i)
        if (weights[i] < 0.0) return fail(SG_ERR_DATA, "calibration instance: negative damage weight");
    if (!(target > 0.0 && target <= 1.0)) return fail(SG_ERR_DATA, "target sparsity must lie in (0, 1]");
    // build_instance: per-neuron stable co-sort by score; cumulative costs.
    std::vector<double> ss(D * T), sw(D * T), cum(D * (T + 1));
    par_for(D, [&](int64_t a, int64_t b) {
        std::vector<int64_t> order(T);
        for (int64_t i = a; i < b; ++i) {
            std::iota(order.begin(), order.end(), int64_t{0});
            const double* row = scores + i * T;
            std::stable_sort(order.begin(), order.end(),
                             [&](int64_t x, int64_t y) { return row[x] < row[y]; });
            cum[i * (T + 1)] = 0.0;
            for (int64_t k = 0; k < T; ++k) {
                ss[i * T + k] = row[order[k]];
                sw[i * T + k] = weights[i * T + order[k]];
                cum[i * (T + 1) + k + 1] = cum[i * (T + 1) + k] + sw[i * T + k];
            }
        }
    });
    auto threshold_at = [&](int64_t i, int64_t k) {
        return k == 0 ? -std::numeric_limits<double>::infinity() : ss[i * T + k - 1];
    };
    auto realized_drops = [&](int64_t i, double tau) {
        const double* row = ss.data() + i * T;
        return static_cast<int64_t>(std::upper_bound(row, row + T, tau) - row);
    };
    const double total = static_cast<double>(D) * static_cast<double>(T);
    std::vector<int64_t> k(D, 0), realized(D, 0);
    int64_t realized_total = 0;
    for (int64_t i = 0; i < D; ++i) {
        int64_t fr = 0;
        while (fr < T && sw[i * T + fr] == 0.0) ++fr;
        k[i] = fr;
        realized[i] = realized_drops(i, threshold_at(i, fr));
        realized_total += realized[i];
    }
    auto increment = [&](int64_t i) {
        const int64_t cur = k[i];
        const int64_t next = std::min<int64_t>(cur + eta, T);
        return cum[i * (T + 1) + next] - cum[i * (T + 1) + cur];
    };
    using HeapEntry = std::tuple<double, int64_t, int64_t>;
    std::priority_queue<HeapEntry, std::vector<HeapEntry>, std::greater<>> heap;
    for (int64_t i = 0; i < D; ++i)
        if (k[i] < T) heap.emplace(increment(i), i, k[i]);
    while (static_cast<double>(realized_total) / total < target) {
        int64_t chosen = -1;
        while (!heap.empty()) {
            const auto [inc, i, snap] = heap.top();
            (void)inc;
            heap.pop();
            if (snap != k[i]) continue;
            chosen = i;
            break;
        }
        if (chosen < 0) {
            return fail(SG_ERR_PROPERTY,
                        "greedy calibration ran out of samples before the target; this state "
                        "should be unreachable");
        }
        int64_t& ptr = k[chosen];
        ptr = std::min<int64_t>(ptr + eta, T);
        const int64_t nr = realized_drops(chosen, threshold_at(chosen, ptr));
        realized_total += nr - realized[chosen];
        realized[chosen] = nr;
        if (ptr < T) heap.emplace(increment(chosen), chosen, ptr);
    }
    double dmg = 0.0;
    for (int64_t i = 0; i < D; ++i) {
        bias[i] = -threshold_at(i, k[i]);
        dmg += cum[i * (T + 1) + k[i]];
    }
    if (achieved) *achieved = static_cast<double>(realized_total) / total;
    if (total_damage) *total_damage = dmg;
    return SG_OK;
}

}  // extern "C"
