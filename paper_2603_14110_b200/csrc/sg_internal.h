// Internal declarations shared by the host ABI (sg_host.cpp) and the device
// code (sg_kernels.cu). Not part of the public ABI (include/sparsegate_c.h).
#pragma once

#include <cstdio>  // (device printf of the bounds-checked build)

#include <cuda.h>

#include <cstdint>

namespace sg {

// Device-resident layer (one shard). All matrices bf16 (uint16 bit patterns),
// rows padded with zeros to a pitch that is a multiple of 64 elements (128 B)
// so every row start is 128-B aligned for cp.async.bulk and LDG.128.
struct LayerView {
    int d;        // hidden
    int D;        // local (shard) inter
    int r;        // predictor rank (0 = dense-only layer)
    int pitch_d;  // round_up(d, 64)
    int pitch_r;  // round_up(r, 64)
    int act;      // 0 ReGLU, 1 dReLU
    int gbase;    // global index of local neuron k = gbase + k * gstride
    int gstride;
    const uint16_t* B;     // r x pitch_d        (reference Predictor::B, types.hpp:75)
    const uint16_t* A;     // D x pitch_r        (reference Predictor::A, types.hpp:74)
    const float* bias;     // D                  (types.hpp:76, +inf kept)
    const uint16_t* gate;  // D x pitch_d        (types.hpp:22)
    const uint16_t* ud;    // D x 2*pitch_d : row k = [up_k | down_k] (down neuron-major)
    const int* gidx;       // global index of local neuron k (null: gbase + k * gstride)
    int hot;               // leading neurons of each CTA block whose gate rows are fetched
                           // before the mask is known (sg_layer_set_hot_rows; 0 = off)
    int pad_[3];
};

// Per-context device workspace (one per stream). Sizes are bounded by the
// ctx's max_inter (Dmax), max_hidden (pitch) and the SM count (G).
// Bounds checks of the device paths' computed global indices (row gathers, list and
// output writes): compiled in only for the checked variant (make checked ->
// libsparsegate_b200_checked.so, SG_LIB=checked), where a violation prints its
// site and traps — the stand-in for compute-sanitizer, which this GPU pool bars.
#ifdef SG_BOUNDS_CHECK
#define SG_CHECK(cond)                                                                   \
    do {                                                                                 \
        if (!(cond)) {                                                                   \
            printf("SG_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, \
                   __LINE__, static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x)); \
            asm volatile("trap;");                                                       \
        }                                                                                \
    } while (0)
#else
#define SG_CHECK(cond) \
    do {               \
    } while (0)
#endif

struct WorkView {
    const float* x;       // [d] input (caller's device buffer)
    const float* xres;    // optional [d] added to x while it is staged (residual chains), or null
    float* y;             // [d] output (caller's device buffer)
    float* t;             // [pitch_r] predictor low-rank activations
    int* cnt;             // [2*gpad] per-CTA predicted counts, then survivor counts
    int* plist;           // [Dmax] per-CTA local predicted lists at neuron-range offsets
    int* P;               // [Dmax] compacted GLOBAL predicted indices, by P position
    float* gP;            // [Dmax] gate pre-activation, by P position (output)
    float* gN;            // [Dmax] gate pre-activation per (local) neuron
    int* rec;             // [2*Dmax] int2 {local neuron or -1, z bits}, by P position
    int* vseg;            // [2*Dmax] int2 per-CTA survivor segments at item-range offsets
    int* V;               // [Dmax] compacted GLOBAL survivor indices
    float* zV;            // [Dmax] gated value per survivor
    float* zD;            // [Dmax] dense pipeline: z per neuron
    float* ypart;         // [G * pitch_dmax] per-CTA partial outputs
    uint32_t* ytag;       // [2 * pitch_dmax] {y bits, tag} published by phase D inside a stack
    unsigned long long* bar;  // 8 grid-barrier counters, 256 B apart (see grid_barrier)
    int* stats;           // [4 per layer] p, v, nonfinite(x), pipeline
    uint64_t* dbg;        // optional [layers][G][16] globaltimer phase stamps (or null)
    unsigned long long* mbits;  // optional [D]: bit `bitpos` set for predicted neurons
    unsigned long long* vbits;  // optional [D]: bit `bitpos` set for survivors
    int bitpos;                 //   (small batches run as a stack, token b = layer b)
    int flags;            // experiment switches (SG_FLAGS env, default 0): 2 no survivor-row
                          // L2 prefetch; bits 8-15 consumer-group override, bits 16-23
                          // ring-slot override (timing studies only; results unchanged)
};

struct LaunchInfo {
    int num_sms;
    int max_smem;  // opt-in dynamic shared memory per block
};

// Launch one layer of the given pipeline (0 dense, 1 parallel, 2 sequential)
// on `stream`. Returns a cudaError_t value.
int launch_layer(const LayerView& L, const WorkView& W, int pipeline, int num_ctas, void* stream);
// Predictor only: t and per-neuron mask bytes into mask_out (device, D bytes).
int launch_predict(const LayerView& L, const WorkView& W, uint8_t* mask_out, int num_ctas,
                   void* stream);
// Multi-layer: runs n layers (device array of LayerView) inside one persistent launch.
int launch_layers(const LayerView* layers_dev, int n, const LayerView& first, const WorkView& W,
                  const float* xs, float* ys, int chain, int pitch_stride, int pipeline,
                  int num_ctas, void* stream);
int query_launch_info(int device, LaunchInfo* info);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device), thread-safe.
int ensure_smem_attr(const void* kernel, int smem);

// Batched decode (sg_batch.cu): one layer, B <= batch_max() tokens.
constexpr int kGpSplits = 8;  // capacity of BatchArgs::gp in split-K partials
constexpr int kDpSplits = 12; // capacity of BatchArgs::yp in split-K partials
struct BatchArgs {
    int B;        // tokens
    int nb;       // B rounded up to a multiple of 8
    int d, D, r;  // hidden, local inter, rank
    int pitch_d, pitch_r, pitch_v;  // pitch_v: survivor-position pitch of Z (>= round_up(D, 64))
    int act;
    int tsplit, dsplit, gsplit;     // split-K of the T, down and gate/up GEMMs
    int gdot;                       // B <= 16: gate / up on the CUDA cores (rows_dot_kernel)
    int stages;                     // cp.async depth of the GEMM tiles (3, 4 or 6)
    int sms;                        // SM count (grid of the row-streaming down kernel)
    // layer
    const uint16_t* Bm;  // predictor B, r x pitch_d
    const uint16_t* A;   // D x pitch_r
    const float* bias;
    const uint16_t* gate;
    const uint16_t* ud;
    // workspace
    uint16_t *xh, *xl;       // [64][pitch_d]
    float* tp;               // [tsplit][pitch_r][64]
    uint16_t *th, *tl;       // [64][pitch_r]
    uint64_t* mbits;         // [D] predicted-active bit per token
    int* uflag;              // [D] union of the predicted sets
    int* pcount;             // [64] |P_b|
    int* plist;              // [D] union, ascending
    int* np;
    float* G;                // [D][64] gate pre-activations
    uint64_t* vbits;         // [D] survivor bit per token
    int* vflag;              // [D]
    int* vcount;             // [64] |V_b|
    int* vlist;              // [D]
    int* nv;
    int* ticket;             // [16] blocks-done tickets: [0] gate_epi (its last block compacts V),
                             // [1 + tile] t_kernel row tiles (the last split reduces T); reset to 0
    float* Z;                // [D][64] gated values
    uint16_t *zh, *zl;       // [64][pitch_v]
    float* yp;               // [dsplit][64][pitch_d]
    float* gp;               // [gsplit][pitch_v][64] gate / up split-K partials
    int* bad;                // [1] set when an input token has a non-finite entry
};
int batch_max();
int launch_batch(const BatchArgs& a, const float* xs, float* ys, void* stream);

// Batched decode on the tensor cores (sg_batch_tc.cu): one persistent launch per
// layer, tcgen05.mma with TMEM accumulators, weight rows by TMA tiles (down rows of
// sparse blocks by cp.async gathers).
struct TcMaps {            // TMA tensor maps (bf16, SWIZZLE_128B, 64-element inner box)
    CUtensorMap xhl;       // X^T hi/lo   [N][xpitch]         box {64, N}
    CUtensorMap thl;       // T^T hi/lo   [N][256]            box {64, N}
    CUtensorMap zhl;       // Z^T hi/lo   [N][zpitch]         box {64, N}
    CUtensorMap Bp;        // predictor B [r][pitch_d]        box {64, 128}
    CUtensorMap A;         // predictor A [D][pitch_r]        box {64, brows}
    CUtensorMap gate;      // gate rows   [D][pitch_d]        box {64, brows}
    CUtensorMap up;        // up rows     [D][pitch_d], row stride 2*pitch_d (ud, first half)   box {64, brows}
    CUtensorMap down;      // down rows   [D][pitch_d], row stride 2*pitch_d (ud + pitch_d)     box {64, 16}
    CUtensorMap down64;    // the same rows                                                     box {64, 64}
    CUtensorMap down128;   // the same rows                                                     box {64, 128}
};
// Rows per neuron block of the tensor-core path for a layer of D (local) rows on a
// device with `sms` SMs: about one block per SM beside the predictor's units, so the
// gate / up streaming needs no split-K (sg_batch_tc.cu).
int tc_block_rows(int64_t D, int sms);
struct TcArgs {
    int B, nb, N;          // tokens, B rounded up to 8, MMA N = 2*nb (hi | lo columns)
    int d, D, r, pitch_d, pitch_r, act;
    int brows;             // neurons per block (<= 128: rows of one M = 128 tile)
    int nblk;              // neuron blocks
    int kst, kt;           // K of a T unit, K slices of T (T units: kt per 128-row half of rank)
    int ndt, S;            // d tiles of 128 outputs, block ranges of the down GEMM (S <= 4)
    int rchunk;            // consecutive blocks per interleave step of the ranges
    int dense;             // 1: dense comparator (no predictor; every row)
    int tile_u;            // per-1024 survivor density at which DOWN tiles a block, not gathers
    int dbg;               // experiment switches (SG_TC_DBG; 1: down stages skip their weight copies)
    int nstages, stage_bytes;  // smem ring: stages x bytes (set by launch_batch_tc from N)
    int u_T, u_GU, u_DOWN, u_end;  // unit counts by type (prefix sums: X, T, GU, DOWN; PF last)
    const uint16_t* pf_gate;  // optional: the next layer's gate rows [pf_D][pf_pitch] to prefetch
    const uint16_t* pf_ud;    //   and its [up | down] rows (up halves prefetched)
    int pf_D, pf_pitch, pf_units;
    uint32_t pf_bytes;        //   leading bytes of each row into L2
    const int* order;      // [n_units] claim order: type << 24 | i << 8 | j (host-built)
    int n_units;
    unsigned long long* trace;  // optional [n_units][8] stamps (tools/tc_trace.py)
    int zpitch;            // slots of Z^T per row (block capacity 128 x blocks)
    int xpitch;            // elements per X^T row (the ctx's max pitch)
    const float* x;        // [B][d] input tokens
    const float* xres;     // optional [B][d] added to x while it is split (residual chains)
    float* y;              // [B][d] outputs
    const float* bias;     // [D]
    const uint16_t* ud;    // [D][2*pitch_d]    [up | down] rows (down rows gathered by cp.async)
    uint16_t* xhl;         // [N][xpitch]
    float* tpart;          // [KT][256][nb]
    uint16_t* thl;         // [N][256]
    uint64_t* mbits;       // [D] predicted bit per token
    uint64_t* vbits;       // [D] survivor bit per token
    int* vlist;            // [nblk][128] survivor rows of a block (row in block), ascending
    int* vcnt;             // [nblk] survivor rows | 1 << 16 when DOWN streams the block whole
    uint16_t* zhl;         // [N][zpitch]
    float* ypart;          // [S][ndt*128][nb]
    int* pcount;           // [64] |P_b|   (pcount, vcount, bad: zeroed by the host per call)
    int* vcount;           // [64] |V_b|
    int* bad;              // [4] non-finite flags: [0] this launch's x, [1] published for the
                           //   last completed launch, [2] / [3] the next launch's x (prep)
    int prep;              // 1: the y finishers also write the NEXT launch's X^T (x = nh + y)
    const float* nh;       //   its residual input h_{l+1} [B][d] (or null: x = y)
    int x_ready;           // 1: X^T was prepared by the previous launch (no X units)
    int* flags;            // dataflow counters, reset by the last CTA of every launch
};
int tc_smem_bytes(int nstages, int stage_bytes);
int tc_flag_ints(int nblk, int ndt);
int launch_batch_tc(const TcMaps& maps, const TcArgs& a, int grid, void* stream);

}  // namespace sg
