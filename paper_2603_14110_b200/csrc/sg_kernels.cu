// sparsegate-b200 device code: the sparse gated-FFN decode executor for sm_100a.
//
// One persistent, cooperative launch per layer (or per stack of layers) runs
// the five stages of the reference's sequential pipeline
// (/root/reference/proj/include/sparsegate/ffn_exec.hpp:183-218). CTA c owns a
// contiguous range of neurons [n0, n1) and the predictor rows j = c + k*G.
//
//   start    cp.async.bulk: this CTA's rows of B and its slice of A -> smem;
//            cp.async: its bias slice; the gate rows of its block's hot prefix
//            (the first sg_layer_set_hot_rows neurons of the layout) -> ring
//            slots (all x-independent: issued during the previous layer's tail)
//            x: inside a stack, the previous layer's y is polled as tagged values
//   phase A  stage 1a  t = B·x  (rows j = c + k*G)    (ffn_exec.hpp:133-136)
//            --- t exchanged as tagged values (no grid barrier) ---
//   phase B  stage 1b  pre = A·t + bias > 0 -> mask  (ffn_exec.hpp:139-144)
//            stage 2   warp-ballot compaction -> this CTA's predicted list
//                                                     (ffn_exec.hpp:189-195)
//   phase C  stage 3   its predicted gate rows -> smem ring (cp.async.bulk,
//                      one issuing lane per slot, mbarriers); 4-warp groups
//                      with x in registers compute g; revalidation g > 0
//                                                     (ffn_exec.hpp:196-201)
//                      survivors' [up | down] rows are prefetched to L2
//            stage 4   survivors: u = up·x, z = gated(g, u)  (:202-203, :68-76)
//            stage 5a  partial y = Σ z·down over its survivors (one pass with 4)
//            --- grid barrier ---
//   phase D  stage 5b  y: CTA c sums the G partials of its column slice in a
//                      fixed order                   (ffn_exec.hpp:80-94)
//                      and, inside a stack, publishes it tagged for the next layer
//
// No grid barrier between stages 2 and 3: a CTA streams its OWN predicted
// rows, so the P prefix (needed only for the P/V outputs) is computed in
// phase D, and only when the caller asks for the index sets.
//
// Dense (ffn_exec.hpp:103-122) and parallel (:149-178) pipelines reuse phases
// C/D with gate+up rows fetched together.
//
// Determinism: no floating-point atomics. Every dot product has a fixed
// thread -> chunk assignment and a fixed reduction tree; every partial sum is
// over a fixed, ordered set (a CTA's own rows in ascending neuron order), and
// the G partials are summed in CTA order. Repeated calls are bit-identical.
//
// Code size matters: the per-layer path must fit the SM instruction cache
// (~32 KB), so cold paths (index-set outputs, barriers) are out of line and
// the phase-timing instrumentation is compiled only with -DSG_PHASE_TIMING.
#include "sg_internal.h"

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <utility>

namespace sg {
namespace {

constexpr int kWarps = 16;                // compute warps
constexpr int kCThreads = kWarps * 32;    // 512 compute threads
constexpr int kThreads = kCThreads + 32;  // + one producer warp (cp.async.bulk issue)
constexpr int kMaxSlots = 32;             // ring slots (upper bound)
constexpr int kRowsA = 2;                 // phase A rows reduced per pass (r = 256 over 148 CTAs: <= 2)
constexpr int kGroupWarps = 4;            // phase C: a row is reduced by a group of 4 warps
constexpr int kGroups = kWarps / kGroupWarps;
constexpr int kGroupThreads = kGroupWarps * 32;
constexpr int kXRegChunks = 4;            // x chunks per thread held in registers (pitch_d <= 4096)
constexpr int kSvChunk = 12;              // survivor [up | down] rows staged per round (stage 4/5a)
constexpr int kSector = 8;                // ints per 32-B sector

// Shared memory: small fixed arrays, then one large region that is, in turn,
// the B/A staging buffer (phases A/B), the cp.async.bulk ring (phase C) and
// the survivor list + reduction scratch (stages 4/5) — never live at once.
struct SmemPlan {
    int off_slotn;  // int[kMaxSlots]   neuron of each ring slot
    int off_uses;   // int[kMaxSlots]   fills of each ring slot before the current layer
    int off_off;    // int[G+1]         predictor-kernel prefix scratch
    int off_mask;   // uint8[mask_cap]  phase B mask bytes
    int off_bias;   // float[mask_cap]  this CTA's bias slice / dense z slice
    int off_misc;   // int[32]          block-level scalars
    int off_lv;     // LayerView[2]     this and the next layer's view (stack launches)
    int off_reda;   // float[512]       reduction scratch (phases A, C, stage 4, phase D)
    int off_items;  // int[item_cap]    this CTA's predicted neurons
    int off_recs;   // int2[item_cap]   per-item {neuron or -1, g or z}
    int off_xs;     // float[pitch_d]
    int off_ts;     // float[pitch_r]
    int off_big;
    int big_bytes;
    int ns;          // ring slots, a multiple of kc
    int kc;          // consumer groups; slot s is always consumed by group s % kc
    int slot_bytes;
    int stage_b;     // B rows of this CTA staged in smem (phase A)
    int as_bytes;    // A slice capacity in smem (0 = stream A from HBM)
    int stage_off;   // staged B rows / A slice: [stage_off, big_bytes) of the big region
    int pre_slots;   // ring slots below stage_off (free while phases A/B run)
    int mask_cap;
    int item_cap;
    int off_sv;      // int2[item_cap] survivor list {n, g} (sequential pipeline), float[kSvChunk] z
    int sv_chunk;    // survivor [up | down] rows staged per round: min(kSvChunk, big / row)
    int total;
};

struct Smem {
    uint64_t* full;
    uint64_t* empty;
    uint64_t* abar;
    int* slotn;
    int* uses;
    int* off;
    uint8_t* mask;
    float* bias;
    int* misc;
    LayerView* lv;
    float* reda;
    int* items;
    int2* recs;
    int2* svl;
    float* xs;
    float* ts;
    uint8_t* big;
};

__device__ __forceinline__ Smem carve(uint8_t* base, const SmemPlan& S) {
    Smem m;
    m.full = reinterpret_cast<uint64_t*>(base);
    m.empty = m.full + kMaxSlots;
    m.abar = m.empty + kMaxSlots;
    m.slotn = reinterpret_cast<int*>(base + S.off_slotn);
    m.uses = reinterpret_cast<int*>(base + S.off_uses);
    m.off = reinterpret_cast<int*>(base + S.off_off);
    m.mask = base + S.off_mask;
    m.bias = reinterpret_cast<float*>(base + S.off_bias);
    m.misc = reinterpret_cast<int*>(base + S.off_misc);
    m.lv = reinterpret_cast<LayerView*>(base + S.off_lv);
    m.reda = reinterpret_cast<float*>(base + S.off_reda);
    m.items = reinterpret_cast<int*>(base + S.off_items);
    m.recs = reinterpret_cast<int2*>(base + S.off_recs);
    m.svl = reinterpret_cast<int2*>(base + S.off_sv);
    m.xs = reinterpret_cast<float*>(base + S.off_xs);
    m.ts = reinterpret_cast<float*>(base + S.off_ts);
    m.big = base + S.off_big;
    return m;
}

// Per-thread persistent state across phases/layers.
struct RunState {
    uint32_t auses;     // staging-barrier phases consumed so far
    uint64_t bar_base;  // grid-barrier counter base (lanes 0..7 of warp 0)
    uint32_t bar_k;     // grid barriers passed in this launch
    uint32_t tag0;      // grid barriers completed before this launch (exchange tags)
};

// ---------------------------------------------------------------------------
// PTX helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "SG_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra SG_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 1-D bulk copy global -> shared through the TMA engine, completion counted on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// Streaming 128-bit weight load: read-only path, no L1 allocation.
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ uint64_t ld_acquire_u64(const unsigned long long* p) {
    uint64_t v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

#ifdef SG_PHASE_TIMING
__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define SG_STAMP(dbg, k)                                         \
    do {                                                         \
        if ((dbg) && threadIdx.x == 0) (dbg)[k] = globaltimer(); \
    } while (0)
#define SG_DBG_PARAM , uint64_t* dbg
#define SG_DBG_ARG , dbg
#else
#define SG_STAMP(dbg, k) \
    do {                 \
    } while (0)
#define SG_DBG_PARAM
#define SG_DBG_ARG
#endif

// 8 bf16 weights (one 16-B chunk) against 8 fp32 activations, in element order.
__device__ __forceinline__ float dot8(const uint4 w, const float* x, float acc) {
    const float4 a = *reinterpret_cast<const float4*>(x);
    const float4 b = *reinterpret_cast<const float4*>(x + 4);
    acc = fmaf(__uint_as_float(w.x << 16), a.x, acc);
    acc = fmaf(__uint_as_float(w.x & 0xffff0000u), a.y, acc);
    acc = fmaf(__uint_as_float(w.y << 16), a.z, acc);
    acc = fmaf(__uint_as_float(w.y & 0xffff0000u), a.w, acc);
    acc = fmaf(__uint_as_float(w.z << 16), b.x, acc);
    acc = fmaf(__uint_as_float(w.z & 0xffff0000u), b.y, acc);
    acc = fmaf(__uint_as_float(w.w << 16), b.z, acc);
    acc = fmaf(__uint_as_float(w.w & 0xffff0000u), b.w, acc);
    return acc;
}
__device__ __forceinline__ float dot8r(const uint4 w, const float* x, float acc) {
    acc = fmaf(__uint_as_float(w.x << 16), x[0], acc);
    acc = fmaf(__uint_as_float(w.x & 0xffff0000u), x[1], acc);
    acc = fmaf(__uint_as_float(w.y << 16), x[2], acc);
    acc = fmaf(__uint_as_float(w.y & 0xffff0000u), x[3], acc);
    acc = fmaf(__uint_as_float(w.z << 16), x[4], acc);
    acc = fmaf(__uint_as_float(w.z & 0xffff0000u), x[5], acc);
    acc = fmaf(__uint_as_float(w.w << 16), x[6], acc);
    acc = fmaf(__uint_as_float(w.w & 0xffff0000u), x[7], acc);
    return acc;
}
// acc[e] += z * w[e] for the 8 bf16 of one chunk.
__device__ __forceinline__ void axpy8(const uint4 w, float z, float* acc) {
    acc[0] = fmaf(z, __uint_as_float(w.x << 16), acc[0]);
    acc[1] = fmaf(z, __uint_as_float(w.x & 0xffff0000u), acc[1]);
    acc[2] = fmaf(z, __uint_as_float(w.y << 16), acc[2]);
    acc[3] = fmaf(z, __uint_as_float(w.y & 0xffff0000u), acc[3]);
    acc[4] = fmaf(z, __uint_as_float(w.z << 16), acc[4]);
    acc[5] = fmaf(z, __uint_as_float(w.z & 0xffff0000u), acc[5]);
    acc[6] = fmaf(z, __uint_as_float(w.w << 16), acc[6]);
    acc[7] = fmaf(z, __uint_as_float(w.w & 0xffff0000u), acc[7]);
}
// Butterfly sum: every lane ends with the same bits.
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    return v;
}
__device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ffn_exec.hpp:68-76 in fp32 (canonical +0 when suppressed).
__device__ __forceinline__ float gated(float g, float u, int act) {
    const bool on = g > 0.f && (act == 0 || u > 0.f);
    return on ? g * u : 0.f;
}

// Balanced split of n items over G parts: part c starts at c*n/G (32-bit safe
// for c <= 1024 and n < 2^21).
__device__ __forceinline__ int split_lo(int c, int G, int n) {
    return static_cast<int>(static_cast<unsigned>(c) * static_cast<unsigned>(n) /
                            static_cast<unsigned>(G));
}

// Values exchanged between CTAs through global memory (per-CTA counts, the
// predictor's t) are written as whole 32-B sectors, one sector per value.
__device__ __forceinline__ void st_sector(int* p, int v) {
    asm volatile(
        "st.global.v4.b32 [%0], {%1, %2, %2, %2};\n\tst.global.v4.b32 [%0+16], {%2, %2, %2, %2};" ::"l"(
            p),
        "r"(v), "r"(0)
        : "memory");
}
__device__ __forceinline__ int gpad() { return static_cast<int>(gridDim.x) * kSector; }

// Data-carrying exchange: a value and a launch-unique tag in ONE 64-bit store,
// so a reader polls the value itself instead of a barrier and then the value.
__device__ __forceinline__ void st_tagged(void* p, float v, uint32_t tag) {
    asm volatile("st.relaxed.gpu.global.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(__float_as_uint(v)),
                 "r"(tag)
                 : "memory");
}
__device__ __forceinline__ float ld_tagged(const void* p, uint32_t tag) {
    uint32_t v, t;
    do {
        asm volatile("ld.relaxed.gpu.global.v2.u32 {%0, %1}, [%2];" : "=r"(v), "=r"(t) : "l"(p) : "memory");
    } while (t != tag);
    return __uint_as_float(v);
}

// ---------------------------------------------------------------------------
// Grid barrier on kBarCounters monotonically increasing 64-bit counters
// (each in its own 256-B block, so they live in different L2 slices). CTA c
// arrives on counter c % kBarCounters; every barrier adds exactly n_j to
// counter j, so between barriers counter j is a multiple of n_j and each
// launch recovers its base as floor(v / n_j) * n_j even if early CTAs already
// arrived. No reset, no generation flag. Split phase: grid_arrive() publishes
// this CTA's writes, grid_wait() returns once every CTA has arrived; work that
// does not depend on other CTAs may run in between. All CTAs are co-resident
// (cooperative launch, one per SM).
// ---------------------------------------------------------------------------
constexpr int kBarCounters = 8;
constexpr int kBarStride = 32;  // u64 elements between counters (256 B)

__device__ __forceinline__ int bar_share(int j) {  // CTAs arriving on counter j
    return (static_cast<int>(gridDim.x) - j + kBarCounters - 1) / kBarCounters;
}
__device__ __forceinline__ void grid_barrier_init(const WorkView& W, RunState& rs) {
    if (threadIdx.x < kBarCounters) {
        const int n = bar_share(threadIdx.x);
        const uint64_t v = ld_acquire_u64(W.bar + threadIdx.x * kBarStride);
        rs.bar_base = n > 0 ? v - v % static_cast<uint64_t>(n) : v;
    }
    if (threadIdx.x < 32) __syncwarp();
    rs.bar_k = 0;
}
__device__ __forceinline__ void grid_arrive(const WorkView& W, RunState& rs) {
    __syncthreads();
    rs.bar_k += 1;
    if (threadIdx.x == 0) {
        // release is cumulative: the block's writes, ordered before this
        // thread by the barrier above, are published with it
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(
                         W.bar + (blockIdx.x % kBarCounters) * kBarStride)
                     : "memory");
    }
}
__device__ __forceinline__ void grid_wait(const WorkView& W, RunState& rs) {
    if (threadIdx.x < 32) {
        if (threadIdx.x < kBarCounters) {
            const int j = threadIdx.x;
            const uint64_t target = rs.bar_base + static_cast<uint64_t>(rs.bar_k) *
                                                      static_cast<uint64_t>(bar_share(j));
            while (ld_acquire_u64(W.bar + j * kBarStride) < target) {
            }
        }
        // the lanes left the spin at different times: reconverge warp 0, or it
        // stays split and its later shuffles take the slow divergent path
        __syncwarp();
    }
    __syncthreads();
}
__device__ __forceinline__ void grid_barrier(const WorkView& W, RunState& rs) {
    grid_arrive(W, rs);
    grid_wait(W, rs);
}

// Exclusive prefix of the per-CTA sector counts cnt[i*kSector], i < G, into
// off[0..G] (off[G] = total). One warp; loads first.
__device__ __noinline__ void warp_prefix(const int* cnt, int* off, int G, int lane) {
    int carry = 0;
    for (int base = 0; base < G; base += 128) {
        int v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int i = base + k * 32 + lane;
            v[k] = i < G ? __ldcg(cnt + i * kSector) : 0;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int i = base + k * 32 + lane;
            int incl = v[k];
#pragma unroll
            for (int m = 1; m < 32; m <<= 1) {
                const int o = __shfl_up_sync(0xffffffffu, incl, m);
                if (lane >= m) incl += o;
            }
            if (i < G) off[i] = carry + incl - v[k];
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
    }
    if (lane == 0) off[G] = carry;
    __syncwarp();
}

// ---------------------------------------------------------------------------
// Staging of one layer's predictor weights for this CTA (weights only, so it
// may run during the previous layer's tail): B rows and the A slice by bulk
// copy on `abar`, the bias slice by cp.async. Returns whether abar was armed.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool stage_weights(const LayerView& L, const Smem& sm,
                                           const SmemPlan& S, bool use_as) {
    const int G = gridDim.x, c = blockIdx.x;
    const int n0 = split_lo(c, G, L.D), n1 = split_lo(c + 1, G, L.D);
    for (int k = threadIdx.x; k < n1 - n0; k += kThreads) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(sm.bias + k)),
                     "l"(L.bias + n0 + k)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    const int nB = c < L.r ? (L.r - c + G - 1) / G : 0;
    const uint32_t row_bytes = static_cast<uint32_t>(L.pitch_d) * 2u;
    const uint32_t bytesB = S.stage_b ? static_cast<uint32_t>(nB) * row_bytes : 0u;
    const uint32_t bytesA = use_as ? static_cast<uint32_t>(n1 - n0) * L.pitch_r * 2u : 0u;
    if (bytesA + bytesB == 0) return false;
    if ((threadIdx.x >> 5) == kWarps) {
        const int lane = threadIdx.x & 31;
        // WAR vs. the generic-proxy reads of this region earlier in the layer
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const uint64_t pol = policy_evict_first();
        if (lane == 0) mbar_expect_tx(sm.abar, bytesA + bytesB);
        __syncwarp();
        for (int q = lane; q < nB && bytesB; q += 31)
            bulk_g2s(sm.big + S.stage_off + static_cast<size_t>(q) * row_bytes,
                     L.B + static_cast<size_t>(c + q * G) * L.pitch_d, row_bytes, sm.abar, pol);
        if (bytesA && lane == 31)
            bulk_g2s(sm.big + S.stage_off + bytesB, L.A + static_cast<size_t>(n0) * L.pitch_r, bytesA,
                     sm.abar, pol);
        __syncwarp();
    }
    return true;
}

// Hot prefix of the sequential pipeline: the gate rows of the first h neurons
// of this CTA's block go into ring slots 0..h-1 (free while phases A/B use the
// staging area at the top of the big region) before x or the mask is known.
// phase_mask keeps them as items 0..h-1; phase C drops the ones it rejected.
// Called when the ring is idle (layer start, or the previous layer's tail).
__device__ __forceinline__ void preissue_hot(const LayerView& L, const Smem& sm,
                                             const SmemPlan& S) {
    const int G = gridDim.x, c = blockIdx.x;
    const int n0 = split_lo(c, G, L.D), n1 = split_lo(c + 1, G, L.D);
    int h = L.hot < S.pre_slots ? L.hot : S.pre_slots;
    if (h > S.ns) h = S.ns;
    if (h > n1 - n0) h = n1 - n0;
    if (h < 0) h = 0;
    if ((threadIdx.x >> 5) == kWarps) {
        const int lane = threadIdx.x & 31;
        if (lane == 0) sm.misc[4] = h;
        if (lane < h) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            const uint32_t row_bytes = static_cast<uint32_t>(L.pitch_d) * 2u;
            const uint32_t use = static_cast<uint32_t>(sm.uses[lane]);
            if (use > 0) mbar_wait(sm.empty + lane, (use - 1) & 1u);
            sm.slotn[lane] = n0 + lane;
            mbar_expect_tx(sm.full + lane, row_bytes);
            bulk_g2s(sm.big + static_cast<size_t>(lane) * S.slot_bytes,
                     L.gate + static_cast<size_t>(n0 + lane) * L.pitch_d, row_bytes, sm.full + lane,
                     policy_evict_first());
        }
        __syncwarp();
    }
}

// Stage x (fp32, length d) into smem, zero-padded to pitch_d; flag non-finite.
// xres (optional): added element-wise (fp32) — x_l = xs_l + y_{l-1} of a residual
// chain run as separate launches (the sharded path, sg_comm.cpp).
__device__ __forceinline__ bool stage_x(const float* x, int d, int pitch_d, float* xs,
                                        const float* xres = nullptr) {
    bool bad = false;
    if (xres != nullptr) {
        for (int i = threadIdx.x; i < pitch_d; i += kThreads) {
            const float v = i < d ? __ldcg(xres + i) + __ldcg(x + i) : 0.f;
            xs[i] = v;
            bad |= !isfinite(v);
        }
        return __syncthreads_or(bad) != 0;
    }
    if ((d & 3) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
        for (int i = threadIdx.x * 4; i < pitch_d; i += kThreads * 4) {
            const float4 w = i < d ? __ldcg(reinterpret_cast<const float4*>(x + i))
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
            *reinterpret_cast<float4*>(xs + i) = w;
            bad |= !isfinite(w.x) || !isfinite(w.y) || !isfinite(w.z) || !isfinite(w.w);
        }
    } else {
        for (int i = threadIdx.x; i < pitch_d; i += kThreads) {
            const float v = i < d ? __ldcg(x + i) : 0.f;
            xs[i] = v;
            bad |= !isfinite(v);
        }
    }
    return __syncthreads_or(bad) != 0;
}

// Inside a stack, layer l+1 starts without a grid barrier: phase D of layer l
// publishes y as tagged values and the next stage x polls them (chained: all
// of y is the next x — plus, for the residual chain, this layer's own token
// xres: x_{l+1} = h_{l+1} + y_l, the residual-stream dependency of a decoder;
// unchained: one value per CTA slice, which orders the layers — a CTA only
// reuses ypart once every CTA has finished reading it).
__device__ __forceinline__ bool stage_x_poll(const float* x, const float* xres, const WorkView& W,
                                             int d, int pitch_d, float* xs, uint32_t tag) {
    bool bad = false;
    const int tid = threadIdx.x;
    if (x == nullptr) {
        constexpr int kIn = 8;
        for (int i0 = tid; i0 < pitch_d; i0 += kIn * kThreads) {
            uint32_t v[kIn], t[kIn];
            float h[kIn];
#pragma unroll
            for (int k = 0; k < kIn; ++k) {
                const int i = i0 + k * kThreads;
                v[k] = 0u;
                t[k] = tag;
                h[k] = 0.f;
                if (i < d) {
                    asm volatile("ld.relaxed.gpu.global.v2.u32 {%0, %1}, [%2];"
                                 : "=r"(v[k]), "=r"(t[k])
                                 : "l"(W.ytag + 2 * i)
                                 : "memory");
                    if (xres) h[k] = __ldcg(xres + i);
                }
            }
#pragma unroll
            for (int k = 0; k < kIn; ++k) {
                const int i = i0 + k * kThreads;
                if (i >= pitch_d) continue;
                float f = __uint_as_float(v[k]);
                if (t[k] != tag) f = ld_tagged(W.ytag + 2 * i, tag);
                if (xres) f = h[k] + f;
                xs[i] = f;
                bad |= !isfinite(f);
            }
        }
        return __syncthreads_or(bad) != 0;
    }
    const int G = gridDim.x;
    constexpr int kXV = 4;  // float4 per thread held across the poll
    if ((d & 3) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 && pitch_d <= kXV * 4 * kThreads) {
        // this layer's x does not depend on the previous layer: its loads are
        // in flight while the previous layer's completion is polled
        float4 v[kXV];
#pragma unroll
        for (int k = 0; k < kXV; ++k) {
            const int i = (tid + k * kThreads) * 4;
            v[k] = i < d ? __ldcg(reinterpret_cast<const float4*>(x + i)) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        if (tid < G) {
            const int col = split_lo(tid, G, d);
            if (col < split_lo(tid + 1, G, d)) (void)ld_tagged(W.ytag + 2 * col, tag);
        }
#pragma unroll
        for (int k = 0; k < kXV; ++k) {
            const int i = (tid + k * kThreads) * 4;
            if (i < pitch_d) {
                *reinterpret_cast<float4*>(xs + i) = v[k];
                bad |= !isfinite(v[k].x) || !isfinite(v[k].y) || !isfinite(v[k].z) || !isfinite(v[k].w);
            }
        }
        return __syncthreads_or(bad) != 0;
    }
    if (tid < G) {
        const int col = split_lo(tid, G, d);
        if (col < split_lo(tid + 1, G, d)) (void)ld_tagged(W.ytag + 2 * col, tag);
    }
    return stage_x(x, d, pitch_d, xs);
}

// ---------------------------------------------------------------------------
// Phase A: t = B·x (fp32), rows j = c + q*G ; block-reduced in fixed order.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int rows_b(const LayerView& L) {  // predictor rows c + k*G
    const int G = gridDim.x, c = blockIdx.x;
    return c < L.r ? (L.r - c + G - 1) / G : 0;
}
__device__ void phase_t(const LayerView& L, const WorkView& W, const Smem& sm, const SmemPlan& S,
                        bool staged_b, uint32_t tag, int nB) {
    const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int nch = L.pitch_d >> 3;
    const uint16_t* bs = reinterpret_cast<const uint16_t*>(sm.big + S.stage_off);
    for (int q0 = 0; q0 < nB; q0 += kRowsA) {
        float acc[kRowsA];
#pragma unroll
        for (int q = 0; q < kRowsA; ++q) acc[q] = 0.f;
        if (tid < kCThreads) {
            for (int ch = tid; ch < nch; ch += kCThreads) {
                uint4 w[kRowsA];
#pragma unroll
                for (int q = 0; q < kRowsA; ++q) {
                    const int qq = q0 + q;
                    if (qq >= nB)
                        w[q] = make_uint4(0, 0, 0, 0);
                    else if (staged_b)
                        w[q] = *reinterpret_cast<const uint4*>(
                            bs + static_cast<size_t>(qq) * L.pitch_d + ch * 8);
                    else
                        w[q] = ldg_stream(L.B + static_cast<size_t>(c + qq * G) * L.pitch_d +
                                          ch * 8);
                }
#pragma unroll
                for (int q = 0; q < kRowsA; ++q) acc[q] = dot8(w[q], sm.xs + ch * 8, acc[q]);
            }
#pragma unroll
            for (int q = 0; q < kRowsA; ++q) {
                const float s = warp_sum(acc[q]);
                if (lane == 0) sm.reda[q * kWarps + warp] = s;
            }
        }
        __syncthreads();
        if (tid < kRowsA && q0 + tid < nB) {
            float s = 0.f;
            for (int w = 0; w < kWarps; ++w) s += sm.reda[tid * kWarps + w];
            st_tagged(reinterpret_cast<int*>(W.t) + (c + (q0 + tid) * G) * kSector, s, tag);
        }
        __syncthreads();
    }
}

// 32-B chunk of x as two LDS.128 (scalar loads at a 32-B thread stride would
// be 8-way bank conflicts).
__device__ __forceinline__ void load_x8(const float* xs, int ch, bool ok, float* v) {
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
    if (ok) {
        a = *reinterpret_cast<const float4*>(xs + ch * 8);
        b = *reinterpret_cast<const float4*>(xs + ch * 8 + 4);
    }
    v[0] = a.x;
    v[1] = a.y;
    v[2] = a.z;
    v[3] = a.w;
    v[4] = b.x;
    v[5] = b.y;
    v[6] = b.z;
    v[7] = b.w;
}
// Sum of v[0..7] over the 32 lanes, transposed: 9 shuffles instead of 40.
// Afterwards lane l holds the total of item 4*(l>>4 & 1) + 2*(l>>3 & 1) + (l>>2 & 1).
__device__ __forceinline__ float warp_sum8(float* v, int lane) {
    const bool hi16 = lane & 16;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float send = hi16 ? v[i] : v[i + 4];
        const float keep = hi16 ? v[i + 4] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    const bool hi8 = lane & 8;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const float send = hi8 ? v[i] : v[i + 2];
        const float keep = hi8 ? v[i + 2] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    const bool hi4 = lane & 4;
    {
        const float send = hi4 ? v[0] : v[1];
        const float keep = hi4 ? v[1] : v[0];
        v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    float s = v[0];
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    return s;
}

// All of t (tagged: no grid barrier between stages 1a and 1b) and the bias slice.
__device__ __forceinline__ void poll_t(const LayerView& L, const WorkView& W, const Smem& sm,
                                       uint32_t tag) {
    for (int i = threadIdx.x; i < L.pitch_r; i += kThreads)
        sm.ts[i] = i < L.r ? ld_tagged(W.t + i * kSector, tag) : 0.f;
    asm volatile("cp.async.wait_all;" ::: "memory");  // the bias slice
    __syncthreads();
}

// ---------------------------------------------------------------------------
// Phase B: mask over this CTA's neuron range + warp-ballot compaction into
// its predicted list (smem items[], global plist at n0, count).
// ---------------------------------------------------------------------------
__device__ void phase_mask(const LayerView& L, const WorkView& W, const Smem& sm, const SmemPlan& S,
                           bool use_as, bool staged_b, uint8_t* mask_out, uint32_t tag SG_DBG_PARAM) {
    const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int n0 = split_lo(c, G, L.D), n1 = split_lo(c + 1, G, L.D);
    const int nB = c < L.r ? (L.r - c + G - 1) / G : 0;
    const uint16_t* as = reinterpret_cast<const uint16_t*>(
        sm.big + S.stage_off + (staged_b ? static_cast<size_t>(nB) * L.pitch_d * 2 : 0));
    const int nchr = L.pitch_r >> 3;
    // the setup above (divisions, parameter-bank reads) is pinned here, before
    // the wait for t, so its latency hides under the exchange
    asm volatile("" ::"r"(n0), "r"(n1), "l"(as), "r"(nchr));
    poll_t(L, W, sm, tag);
    if (use_as && nchr <= 32) {
        // A slice in smem, r <= 256: warp w takes 8 neurons per pass; lane l
        // holds t chunk l in registers and dots chunk l of the 8 rows (each row
        // read contiguously), then one transposed warp reduction. Order fixed
        // per neuron: the 8 products of chunk l, then the butterfly.
        float tr[8];
        load_x8(sm.ts, lane, lane < nchr, tr);
        const uint32_t abase = smem_u32(as) + static_cast<uint32_t>(lane * 16);
        for (int base = warp * 8; warp < kWarps && base < n1 - n0; base += kWarps * 8) {
            float part[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                uint4 w = make_uint4(0u, 0u, 0u, 0u);
                if (base + j < n1 - n0 && lane < nchr)
                    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                                 : "r"(abase + static_cast<uint32_t>((base + j) * L.pitch_r * 2)));
                part[j] = dot8r(w, tr, 0.f);
            }
                const float sum = warp_sum8(part, lane);
                const int k = base + ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
            if ((lane & 3) == 0 && k < n1 - n0) {
                const float pre = sum + sm.bias[k];
                const uint8_t on = pre > 0.f ? 1 : 0;  // strict, ffn_exec.hpp:141
                sm.mask[k] = on;
                if (mask_out) mask_out[n0 + k] = on;
                if (on && W.mbits) atomicOr(W.mbits + n0 + k, 1ull << W.bitpos);
            }
            }
    } else {
        // 4 lanes per neuron, 128 neurons per pass; lane sub covers chunks
        // sub + 4i, starting at i = (global index & 1) so the two neurons sharing a
        // quarter-warp read different banks. Order fixed per neuron.
        const int nchr = L.pitch_r >> 3;
        const int nq = nchr >> 2;  // chunks per lane (pitch_r >= 64 -> nq >= 2)
        for (int base = 0; base < n1 - n0; base += kCThreads / 4) {
            const int k = base + (tid >> 2), sub = tid & 3;
            float acc = 0.f;
            if (tid < kCThreads && k < n1 - n0) {
                const int n = n0 + k;
                const uint16_t* arow = use_as ? as + static_cast<size_t>(k) * L.pitch_r
                                              : L.A + static_cast<size_t>(n) * L.pitch_r;
                const int rot = (L.gbase + n * L.gstride) & 1;
                for (int i = 0; i < nq; ++i) {
                    int ii = i + rot;
                    if (ii >= nq) ii -= nq;
                    const int ch = sub + 4 * ii;
                    const uint4 w = use_as ? *reinterpret_cast<const uint4*>(arow + ch * 8)
                                           : ldg_stream(arow + ch * 8);
                    acc = dot8(w, sm.ts + ch * 8, acc);
                }
            }
            acc += __shfl_xor_sync(0xffffffffu, acc, 1);
            acc += __shfl_xor_sync(0xffffffffu, acc, 2);
            if (tid < kCThreads && sub == 0 && k < n1 - n0) {
                const float pre = acc + sm.bias[k];
                const uint8_t on = pre > 0.f ? 1 : 0;  // strict, ffn_exec.hpp:141
                sm.mask[k] = on;
                if (mask_out) mask_out[n0 + k] = on;
                if (on && W.mbits) atomicOr(W.mbits + n0 + k, 1ull << W.bitpos);
            }
        }
    }
    __syncthreads();
    if (warp == 0) {
        // P list (ascending) and the phase C item list: the hot prefix fetched
        // ahead of the mask (items 0..hpre-1 = the block's first neurons, kept
        // whether predicted or not), then the other predicted neurons
        const int hpre = sm.misc[4];
        int run = 0, irun = hpre;
        for (int base = 0; base < n1 - n0; base += 32) {
            const int k = base + lane;
            const bool on = k < n1 - n0 && sm.mask[k];
            const unsigned b = __ballot_sync(0xffffffffu, on);
            const unsigned bi = __ballot_sync(0xffffffffu, on && k >= hpre);
            const unsigned below = (1u << lane) - 1u;
            SG_CHECK(!on || (n0 + run + __popc(b & below) < L.D && n0 + k < L.D));
            if (on) W.plist[n0 + run + __popc(b & below)] = n0 + k;
            if (k < hpre) sm.items[k] = n0 + k;
            if (on && k >= hpre) sm.items[irun + __popc(bi & below)] = n0 + k;
            run += __popc(b);
            irun += __popc(bi);
        }
        if (lane == 0) {
            st_sector(W.cnt + c * kSector, run);
            sm.misc[0] = run;
            sm.misc[3] = irun;
            if (run && !mask_out) atomicAdd(W.stats + 0, run);  // p (integer: order-free)
        }
    }
    __syncthreads();
}

// ---- phase C row dot: a group of 4 warps (128 threads) per row ----------
// Thread gt of a group owns chunks gt, gt+128, ... of every row and keeps the
// matching x values in registers, so the per-row shared-memory traffic is the
// row itself only. Row value = (thread chain over its chunks, ascending)
// -> warp butterfly -> the 4 warps summed in order.
struct XRegs {
    float v[kXRegChunks][8];
};
__device__ __forceinline__ void load_xregs(const float* xs, int nch, int gt, XRegs& X) {
#pragma unroll
    for (int k = 0; k < kXRegChunks; ++k) {
        const int ch = gt + k * kGroupThreads;
        load_x8(xs, ch, ch < nch, X.v[k]);
    }
}
// kRows smem rows sharing the x registers; red is this group's scratch
// [2 parities][kGroupWarps][4]; par alternates per call.
template <int kRows>
__device__ __forceinline__ void group_dot(const uint16_t* const* rows, const XRegs& X,
                                          const float* xs, int nch, int gt, int grp, float* red,
                                          int& par, float* out) {
    float acc[kRows];
#pragma unroll
    for (int q = 0; q < kRows; ++q) acc[q] = 0.f;
#pragma unroll
    for (int k = 0; k < kXRegChunks; ++k) {
        const int ch = gt + k * kGroupThreads;
        if (ch < nch) {
#pragma unroll
            for (int q = 0; q < kRows; ++q)
                acc[q] = dot8r(*reinterpret_cast<const uint4*>(rows[q] + ch * 8), X.v[k], acc[q]);
        }
    }
    // chunks beyond the register window (pitch_d > 4096): x from smem
    for (int ch = gt + kXRegChunks * kGroupThreads; ch < nch; ch += kGroupThreads) {
#pragma unroll
        for (int q = 0; q < kRows; ++q)
            acc[q] = dot8(*reinterpret_cast<const uint4*>(rows[q] + ch * 8), xs + ch * 8, acc[q]);
    }
    const int gw = gt >> 5, lane = gt & 31;
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1)
#pragma unroll
        for (int q = 0; q < kRows; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], m);
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < kRows; ++q) red[(par * kGroupWarps + gw) * 4 + q] = acc[q];
    }
    named_bar(1 + grp, kGroupThreads);
#pragma unroll
    for (int q = 0; q < kRows; ++q) {
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < kGroupWarps; ++w) s += red[(par * kGroupWarps + w) * 4 + q];
        out[q] = s;
    }
    par ^= 1;
}

// group_dot with x read from shared memory (same chunk map, same fmaf order per
// row — dot8 and dot8r are one chain — so the result is bitwise group_dot's);
// used where the x registers would not fit next to other live state.
template <int kRows>
__device__ __forceinline__ void group_dot_xs(const uint16_t* const* rows, const float* xs, int nch,
                                             int gt, int grp, float* red, int& par, float* out) {
    float acc[kRows];
#pragma unroll
    for (int q = 0; q < kRows; ++q) acc[q] = 0.f;
    for (int ch = gt; ch < nch; ch += kGroupThreads) {
#pragma unroll
        for (int q = 0; q < kRows; ++q)
            acc[q] = dot8(*reinterpret_cast<const uint4*>(rows[q] + ch * 8), xs + ch * 8, acc[q]);
    }
    const int gw = gt >> 5, lane = gt & 31;
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1)
#pragma unroll
        for (int q = 0; q < kRows; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], m);
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < kRows; ++q) red[(par * kGroupWarps + gw) * 4 + q] = acc[q];
    }
    named_bar(1 + grp, kGroupThreads);
#pragma unroll
    for (int q = 0; q < kRows; ++q) {
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < kGroupWarps; ++w) s += red[(par * kGroupWarps + w) * 4 + q];
        out[q] = s;
    }
    par ^= 1;
}

// ---------------------------------------------------------------------------
// Phase C: gather-GEMV over this CTA's items through the cp.async.bulk ring.
//   kPipe 2 (sequential): items = own predicted rows; slot = gate row.
//   kPipe 1 (parallel):   items = own predicted rows; slot = gate row + up row.
//   kPipe 0 (dense):      items = own neuron range;   slot = gate row + up row.
// Sparse pipelines record {neuron or -1, g (seq) or z (par)} per item and end
// with this CTA's survivor list (P order) in the big region.
// ---------------------------------------------------------------------------
template <int kPipe>
__device__ void phase_gather(const LayerView& L, const WorkView& W, const Smem& sm,
                             const SmemPlan& S) {
    const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int nch = L.pitch_d >> 3;
    const uint32_t row_bytes = static_cast<uint32_t>(L.pitch_d) * 2u;
    const int n0 = split_lo(c, G, L.D);
    const int nitems = kPipe == 0 ? split_lo(c + 1, G, L.D) - n0 : sm.misc[3];
    const int ns = S.ns;
    // item j lives in slot j % ns as that slot's fill uses[slot] + j / ns

    if (warp == kWarps) {
        // ---- producer warp: lane s issues every item of ring slot s (s < ns),
        // in order. One issuing thread per slot: a single thread issuing all
        // cp.async.bulk copies caps an SM near 22 GB/s (tools/microbench_gather.cu).
        const uint64_t pol = policy_evict_first();
        const int slot = lane;
        // WAR vs. the generic reads of the staging area under the last slots
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (slot < ns) {
            const uint32_t u0 = static_cast<uint32_t>(sm.uses[slot]);
            const int hpre = kPipe == 2 ? sm.misc[4] : 0;  // items already issued (hot prefix)
            for (int j = slot; j < nitems; j += ns) {
                if (j < hpre) continue;
                const int n = kPipe == 0 ? n0 + j : sm.items[j];
                SG_CHECK(n >= 0 && n < L.D);
                const uint32_t use = u0 + static_cast<uint32_t>(j / ns);
                if (use > 0) mbar_wait(sm.empty + slot, (use - 1) & 1u);
                sm.slotn[slot] = n;
                uint8_t* dst = sm.big + static_cast<size_t>(slot) * S.slot_bytes;
                if (kPipe == 2) {
                    mbar_expect_tx(sm.full + slot, row_bytes);
                    bulk_g2s(dst, L.gate + static_cast<size_t>(n) * L.pitch_d, row_bytes,
                             sm.full + slot, pol);
                } else {
                    mbar_expect_tx(sm.full + slot, 2 * row_bytes);
                    bulk_g2s(dst, L.gate + static_cast<size_t>(n) * L.pitch_d, row_bytes,
                             sm.full + slot, pol);
                    bulk_g2s(dst + row_bytes, L.ud + static_cast<size_t>(n) * 2 * L.pitch_d,
                             row_bytes, sm.full + slot, pol);
                }
            }
        }
        __syncwarp();
    } else {
        // ---- compute groups: group g < kc (4 warps) consumes the items
        // j with j % kc == g, in order, two per iteration. ns is a multiple of
        // kc, so every slot is consumed by one group, phase after phase, and a
        // parity wait can never run a phase ahead of the barrier.
        const int kc = S.kc;
        const int grp = warp / kGroupWarps, gt = tid % kGroupThreads;
        XRegs X;
        load_xregs(sm.xs, nch, gt, X);
        float* red = sm.reda + grp * (2 * kGroupWarps * 4);
        int par = 0;
        for (int j = grp; grp < kc && j < nitems; j += 2 * kc) {
            const bool two = j + kc < nitems;
            int slot[2], n[2];
            const uint16_t* r[4];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int jj = two ? j + h * kc : j;
                slot[h] = jj % ns;
                if (h == 0 || two)
                    mbar_wait(sm.full + slot[h],
                              (static_cast<uint32_t>(sm.uses[slot[h]]) + jj / ns) & 1u);
                n[h] = sm.slotn[slot[h]];
                const uint16_t* srow = reinterpret_cast<const uint16_t*>(
                    sm.big + static_cast<size_t>(slot[h]) * S.slot_bytes);
                r[2 * h] = srow;
                r[2 * h + 1] = srow + L.pitch_d;
            }
            __syncwarp();  // lanes leave the spins at different times: reconverge
            float res[4] = {0.f, 0.f, 0.f, 0.f};
            if (kPipe == 2) {
                const uint16_t* rr[2] = {r[0], r[2]};
                float o[2];
                group_dot<2>(rr, X, sm.xs, nch, gt, grp, red, par, o);
                res[0] = o[0];
                res[2] = o[1];
            } else {
                group_dot<4>(r, X, sm.xs, nch, gt, grp, red, par, res);
            }
            // the group barrier inside group_dot follows every read of the slots
            if (gt == 0) {
                mbar_arrive(sm.empty + slot[0]);
                if (two) mbar_arrive(sm.empty + slot[1]);
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (h == 1 && !two) break;
                const float g = res[2 * h];
                const float u = res[2 * h + 1];
                const int nn = n[h];
                if (kPipe == 0) {
                    SG_CHECK(gt != 0 || (nn >= 0 && nn < L.D));
                    if (gt == 0) W.zD[nn] = gated(g, u, L.act);
                    continue;
                }
                // a hot-prefix item the mask rejected is dropped (never in P)
                const int jj = j + h * kc;
                const bool inP = kPipe != 2 || jj >= sm.misc[4] || sm.mask[jj];
                const bool sv = inP && g > 0.f;  // revalidation, ffn_exec.hpp:200 (strict)
                // a survivor's [up | down] rows (16 KB, contiguous) go to L2 now for
                // stages 4 and 5a: one bulk prefetch, kept in L2 ahead of the
                // evict-first gate stream (SG_FLAGS bit 2: per-line LSU prefetches)
                if (sv && !(W.flags & 2)) {
                    const char* a = reinterpret_cast<const char*>(
                        L.ud + static_cast<size_t>(nn) * 2 * L.pitch_d);
                    if (W.flags & 4) {
                        for (int off = gt * 128; off < 4 * L.pitch_d; off += kGroupThreads * 128)
                            asm volatile("prefetch.global.L2 [%0];" ::"l"(a + off));
                    } else if (gt == 0) {
                        uint64_t keep;
                        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
                        asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(a),
                                     "r"(static_cast<uint32_t>(4 * L.pitch_d)), "l"(keep)
                                     : "memory");
                    }
                }
                if (gt == 0) {
                    if (kPipe == 2 && sv && W.vbits) atomicOr(W.vbits + nn, 1ull << W.bitpos);
                    if (inP) W.gN[nn] = g;  // gate pre-activation per neuron (P output)
                    int2 rec;
                    rec.x = sv ? nn : -1;
                    rec.y = __float_as_int(kPipe == 2 ? g : (sv ? gated(g, u, L.act) : 0.f));
                    sm.recs[jj] = rec;
                }
            }
        }
    }
    __syncthreads();
    if (tid < ns && nitems > tid) sm.uses[tid] += (nitems - tid + ns - 1) / ns;
    if (tid == 0) sm.misc[4] = 0;
    if (kPipe == 0) __syncthreads();
    if (kPipe != 0) {
        // survivors of this CTA's items, in P order -> smem list + global segment
        int2* list = kPipe == 2 ? sm.svl : reinterpret_cast<int2*>(sm.big);
        if (warp == 0) {
            int run = 0;
            for (int base = 0; base < nitems; base += 32) {
                const int j = base + lane;
                const int2 rr = j < nitems ? sm.recs[j] : make_int2(-1, 0);
                const bool on = rr.x >= 0;
                const unsigned b = __ballot_sync(0xffffffffu, on);
                if (on) {
                    const int dst = run + __popc(b & ((1u << lane) - 1u));
                    SG_CHECK(n0 + dst < L.D);
                    list[dst] = rr;
                    reinterpret_cast<int2*>(W.vseg)[n0 + dst] = rr;
                }
                run += __popc(b);
            }
            if (lane == 0) {
                sm.misc[1] = run;
                st_sector(W.cnt + gpad() + c * kSector, run);
                if (run) atomicAdd(W.stats + 1, run);  // v (integer: order-free)
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Stages 4+5a of the sequential pipeline, per CTA, after its gate stream. The
// survivors' [up | down] rows (16 KB each, contiguous, sent to L2 during the
// gate stream) are bulk-copied into shared memory in groups of sv_chunk / 2,
// alternating between two row buffers so one group lands while another is computed.
// The up rows are dotted by the 4-warp groups with phase C's reduction (same
// chunk map and order, x from shared memory), so u — and z, y — are bitwise
// those of the dense and parallel pipelines; threads 0..m-1 form
// z = gated(g, u) (ffn_exec.hpp:202-203, :68-76), and thread t adds z·down for
// chunks t and t + 512 into its partial y, survivors in P order.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void survivor_updown(const LayerView& L, const WorkView& W,
                                                const Smem& sm, const SmemPlan& S, RunState& rs) {
    const int c = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nch = L.pitch_d >> 3;
    const int n0 = split_lo(c, gridDim.x, L.D);
    const int nsv = sm.misc[1];
    const uint32_t ud_bytes = static_cast<uint32_t>(L.pitch_d) * 4u;
    float* zs = reinterpret_cast<float*>(sm.svl + S.item_cap);  // after the list
    const int ch0 = tid, ch1 = tid + kCThreads;
    const bool comp = tid < kCThreads;
    const bool h0 = comp && ch0 < nch, h1 = comp && ch1 < nch;
    // u = up·x with phase C's row reduction (group_dot: 4-warp groups, x chunks
    // gt + 128k in registers), so u — and therefore z and y — are bitwise the
    // same as in the dense / parallel pipelines (ffn_exec_tests.cpp:124-137, :171-192)
    const int grp = warp / kGroupWarps, gt = tid % kGroupThreads;
#ifdef SG_SV_XREGS
    XRegs X;
    load_xregs(sm.xs, nch, gt, X);
#endif
    float* gred = sm.reda + grp * (2 * kGroupWarps * 4);
    int gpar = 0;
    float* us = sm.reda + kGroups * 2 * kGroupWarps * 4;  // u of the group's rows
    float a0[8], a1[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        a0[e] = 0.f;
        a1[e] = 0.f;
    }
    // groups of `half` survivors alternate between two row buffers (barriers
    // full[kMaxSlots-2+b], never used by the ring): group g + 2 is fetched while
    // group g + 1 is computed, so a CTA with more survivors than fit at once does
    // not pay a second exposed L2 round trip
    const int half = S.sv_chunk / 2;
    int* bu = sm.uses + kMaxSlots - 2;  // fills of the two buffer barriers so far
    const uint64_t pol = policy_evict_first();
    auto issue = [&](int g) {  // producer warp
        const int r0 = g * half;
        const int m = nsv - r0 < half ? nsv - r0 : half;
        if (m <= 0) return;
        uint64_t* bar = sm.full + kMaxSlots - 2 + (g & 1);
        if (lane == 0) mbar_expect_tx(bar, static_cast<uint32_t>(m) * ud_bytes);
        __syncwarp();
        SG_CHECK(lane >= m || (sm.svl[r0 + lane].x >= 0 && sm.svl[r0 + lane].x < L.D));
        if (lane < m)
            bulk_g2s(sm.big + static_cast<size_t>((g & 1) * half + lane) * ud_bytes,
                     L.ud + static_cast<size_t>(sm.svl[r0 + lane].x) * 2 * L.pitch_d, ud_bytes, bar,
                     pol);
        __syncwarp();
    };
    if (warp == kWarps) {
        // the ring's last generic reads ended at a block barrier
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(0);
        issue(1);
    }
    const int ngroups = nsv > 0 ? (nsv + half - 1) / half : 0;
    for (int g = 0; g < ngroups; ++g) {
        const int r0 = g * half;
        const int m = nsv - r0 < half ? nsv - r0 : half;  // <= kBatch
        const uint8_t* rows = sm.big + static_cast<size_t>((g & 1) * half) * ud_bytes;
        mbar_wait(sm.full + kMaxSlots - 2 + (g & 1), static_cast<uint32_t>(bu[g & 1] + (g >> 1)) & 1u);
        __syncwarp();
        if (comp) {
            // rows grp and grp + 4 of the group (m <= 8)
            const int j0 = grp, j1 = grp + kGroups;
            const uint16_t* rr[2] = {
                reinterpret_cast<const uint16_t*>(rows + static_cast<size_t>(j0) * ud_bytes),
                reinterpret_cast<const uint16_t*>(rows + static_cast<size_t>(j1) * ud_bytes)};
            float o[2];
            if (j1 < m) {
#ifdef SG_SV_XREGS
                group_dot<2>(rr, X, sm.xs, nch, gt, grp, gred, gpar, o);
#else
                group_dot_xs<2>(rr, sm.xs, nch, gt, grp, gred, gpar, o);
#endif
                if (gt == 0) {
                    us[j0] = o[0];
                    us[j1] = o[1];
                }
            } else if (j0 < m) {
#ifdef SG_SV_XREGS
                group_dot<1>(rr, X, sm.xs, nch, gt, grp, gred, gpar, o);
#else
                group_dot_xs<1>(rr, sm.xs, nch, gt, grp, gred, gpar, o);
#endif
                if (gt == 0) us[j0] = o[0];
            }
        }
        __syncthreads();
        if (tid < m) {
            const float u = us[tid];
            int2 e = sm.svl[r0 + tid];
            const float z = gated(__int_as_float(e.y), u, L.act);
            zs[tid] = z;
            e.y = __float_as_int(z);
            SG_CHECK(n0 + r0 + tid < L.D);
            reinterpret_cast<int2*>(W.vseg)[n0 + r0 + tid] = e;
        }
        __syncthreads();  // zs complete
        if (comp) {
            for (int i = 0; i < m; ++i) {
                const uint16_t* dn =
                    reinterpret_cast<const uint16_t*>(rows + static_cast<size_t>(i) * ud_bytes) + L.pitch_d;
                const float z = zs[i];
                if (z == 0.f) continue;  // zero-z slots contribute nothing (ffn_exec.hpp:89-92)
                if (h0) axpy8(*reinterpret_cast<const uint4*>(dn + ch0 * 8), z, a0);
                if (h1) axpy8(*reinterpret_cast<const uint4*>(dn + ch1 * 8), z, a1);
            }
        }
        __syncthreads();  // the group's rows and zs are no longer read
        if (warp == kWarps) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(g + 2);
        }
    }
    if (tid < 2) bu[tid] += (ngroups + 1 - tid) / 2;  // buffer 0: ceil(n/2), buffer 1: floor(n/2)
    // this CTA's partial y
    if (h0) {
        float4* dst = reinterpret_cast<float4*>(W.ypart + static_cast<size_t>(c) * L.pitch_d + ch0 * 8);
        dst[0] = make_float4(a0[0], a0[1], a0[2], a0[3]);
        dst[1] = make_float4(a0[4], a0[5], a0[6], a0[7]);
    }
    if (h1) {
        float4* dst = reinterpret_cast<float4*>(W.ypart + static_cast<size_t>(c) * L.pitch_d + ch1 * 8);
        dst[0] = make_float4(a1[0], a1[1], a1[2], a1[3]);
        dst[1] = make_float4(a1[4], a1[5], a1[6], a1[7]);
    }
}

// ---------------------------------------------------------------------------
// Stage 5a for the dense and parallel pipelines: partial y over this CTA's
// list, streaming whole down rows (thread t owns chunks t, t+512, ...), rows
// in list order, kU rows in flight per thread. Dense: the list is the CTA's
// neuron range with z from zD; parallel: the survivor list of phase C.
// ---------------------------------------------------------------------------
template <int kPipe>
__device__ void partial_down(const LayerView& L, const WorkView& W, const Smem& sm) {
    const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x;
    const int nch = L.pitch_d >> 3;
    const int n0 = split_lo(c, G, L.D), n1 = split_lo(c + 1, G, L.D);
    const int2* list = reinterpret_cast<const int2*>(sm.big);
    float* zs = sm.bias;  // dense: z of this CTA's neurons (<= mask_cap)
    int cnt;
    if (kPipe == 0) {
        cnt = n1 - n0;
        for (int k = tid; k < cnt; k += kThreads) zs[k] = W.zD[n0 + k];
        __syncthreads();
    } else {
        cnt = sm.misc[1];
    }
    constexpr int kU = 8;
    for (int ch = tid; tid < kCThreads && ch < nch; ch += kCThreads) {
        float acc[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = 0.f;
        const uint16_t* col = L.ud + L.pitch_d + static_cast<size_t>(ch) * 8;
        for (int k = 0; k < cnt; k += kU) {
            uint4 w[kU];
            float z[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int kk = k + u;
                int n = 0;
                z[u] = 0.f;
                if (kk < cnt) {
                    if (kPipe == 0) {
                        n = n0 + kk;
                        z[u] = zs[kk];
                    } else {
                        const int2 e = list[kk];
                        n = e.x;
                        z[u] = __int_as_float(e.y);
                    }
                }
                w[u] = kk < cnt ? ldg_stream(col + static_cast<size_t>(n) * 2 * L.pitch_d)
                                : make_uint4(0, 0, 0, 0);
            }
            // zero-z slots (and the padding) contribute nothing, exactly as in
            // survivor_updown, so all pipelines sum the same terms in one order
#pragma unroll
            for (int u = 0; u < kU; ++u)
                if (z[u] != 0.f) axpy8(w[u], z[u], acc);
        }
        float4* dst = reinterpret_cast<float4*>(W.ypart + static_cast<size_t>(c) * L.pitch_d + ch * 8);
        dst[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
        dst[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
    }
}

// P and V index-set outputs (ascending global indices) for the caller: prefixes
// over the per-CTA predicted / survivor counts; this CTA copies its own
// segments. One warp; only for the last layer of a launch.
__device__ __noinline__ void write_index_sets(int gbase, int gstride, const int* gidx, int D,
                                              const int* cnt, const int* plist, const float* gN,
                                              const int* vseg_raw, int* P, float* gP, int* V,
                                              float* zV) {
    const int G = gridDim.x, c = blockIdx.x, lane = threadIdx.x & 31;
    int carryP = 0, carryV = 0, mineP = 0, mineV = 0;
    for (int base = 0; base < G; base += 32) {
        const int i = base + lane;
        const int vp = i < G ? __ldcg(cnt + i * kSector) : 0;
        const int vv = i < G ? __ldcg(cnt + gpad() + i * kSector) : 0;
        int ip = vp, iv = vv;
#pragma unroll
        for (int m = 1; m < 32; m <<= 1) {
            const int op = __shfl_up_sync(0xffffffffu, ip, m);
            const int ov = __shfl_up_sync(0xffffffffu, iv, m);
            if (lane >= m) {
                ip += op;
                iv += ov;
            }
        }
        if (i == c) {
            mineP = carryP + ip - vp;
            mineV = carryV + iv - vv;
        }
        carryP += __shfl_sync(0xffffffffu, ip, 31);
        carryV += __shfl_sync(0xffffffffu, iv, 31);
    }
    mineP = __reduce_add_sync(0xffffffffu, mineP);
    mineV = __reduce_add_sync(0xffffffffu, mineV);
    const int n0 = split_lo(c, G, D);
    const int cntP = __ldcg(cnt + c * kSector);
    for (int k = lane; k < cntP; k += 32) {
        const int n = __ldcg(plist + n0 + k);
        SG_CHECK(n >= 0 && n < D && mineP + k < D);
        P[mineP + k] = gidx ? __ldg(gidx + n) : gbase + n * gstride;
        gP[mineP + k] = __ldcg(gN + n);
    }
    const int cntV = __ldcg(cnt + gpad() + c * kSector);
    const int2* seg = reinterpret_cast<const int2*>(vseg_raw) + n0;
    for (int k = lane; k < cntV; k += 32) {
        const int2 e = __ldcg(seg + k);
        SG_CHECK(e.x >= 0 && e.x < D && mineV + k < D);
        V[mineV + k] = gidx ? __ldg(gidx + e.x) : gbase + e.x * gstride;
        zV[mineV + k] = __int_as_float(e.y);
    }
    __syncwarp();
}

// ---------------------------------------------------------------------------
// Phase D (after a grid barrier): CTA c sums the G partials of its column
// range in fixed order (contiguous groups of partials, then the groups).
// ---------------------------------------------------------------------------
// Phase D's index arithmetic, computed before the partial barrier's wait so
// its latency (divisions, parameter reads) hides under the barrier.
struct DownPlan {
    int c0, ncols, ngrp, g0, g1;
    const float* src;  // this thread's first partial (column c0 + tid % ncols)
};
__device__ __forceinline__ DownPlan down_plan(const LayerView& L, const WorkView& W) {
    const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x;
    DownPlan p;
    p.c0 = split_lo(c, G, L.d);
    p.ncols = split_lo(c + 1, G, L.d) - p.c0;
    p.ngrp = p.ncols > 0 ? kCThreads / p.ncols : 0;
    if (p.ngrp > 32) p.ngrp = 32;
    p.g0 = p.g1 = 0;
    p.src = W.ypart;
    if (p.ncols > 0 && tid < p.ngrp * p.ncols) {
        const int grp = tid / p.ncols;
        p.g0 = split_lo(grp, p.ngrp, G);
        p.g1 = split_lo(grp + 1, p.ngrp, G);
        p.src = W.ypart + static_cast<size_t>(p.g0) * L.pitch_d + p.c0 + tid % p.ncols;
    }
    asm volatile("" ::"r"(p.c0), "r"(p.ncols), "r"(p.ngrp), "r"(p.g0), "r"(p.g1), "l"(p.src));
    return p;
}

template <int kPipe>
__device__ void phase_down(const LayerView& L, const WorkView& W, const Smem& sm, float* y,
                           bool want_sets, bool publish, uint32_t ytag, const DownPlan& dp) {
    const int tid = threadIdx.x;
    if (kPipe != 0 && want_sets && (tid >> 5) == kWarps)
        write_index_sets(L.gbase, L.gstride, L.gidx, L.D, W.cnt, W.plist, W.gN, W.vseg, W.P, W.gP,
                         W.V, W.zV);
    const int c0 = dp.c0, ncols = dp.ncols, ngrp = dp.ngrp;
    float* part = sm.reda;  // the big region may hold the next layer's hot prefix
    if (ncols > 0) {
        if (tid < ngrp * ncols) {
            const int g0 = dp.g0, g1 = dp.g1;
            // all loads in flight before the (ordered) sum: one L2 round trip
            constexpr int kPer = 12;
            const float* src = dp.src;
            float v[kPer];
#pragma unroll
            for (int i = 0; i < kPer; ++i)
                v[i] = g0 + i < g1 ? __ldcg(src + static_cast<size_t>(i) * L.pitch_d) : 0.f;
            float s = 0.f;
#pragma unroll
            for (int i = 0; i < kPer; ++i)
                if (g0 + i < g1) s += v[i];
            for (int g = g0 + kPer; g < g1; ++g)
                s += __ldcg(src + static_cast<size_t>(g - g0) * L.pitch_d);
            part[tid] = s;
        }
        __syncthreads();
        if (tid < ncols) {
            float s = 0.f;
            for (int grp = 0; grp < ngrp; ++grp) s += part[grp * ncols + tid];
            SG_CHECK(c0 + tid < L.d);
            y[c0 + tid] = s;
            if (publish) st_tagged(W.ytag + 2 * (c0 + tid), s, ytag);
        }
    }
    __syncthreads();
}

// One layer. Returns whether it already staged the next layer's weights.
template <int kPipe>
__device__ bool run_layer(const LayerView& L, const WorkView& W, const Smem& sm,
                          const SmemPlan& S, RunState& rs, const float* x, float* y,
                          bool first_layer, int chain, int lidx, bool want_sets,
                          const LayerView* next, bool prestaged) {
    const int c = blockIdx.x, tid = threadIdx.x;
#ifdef SG_PHASE_TIMING
    uint64_t* dbg =
        W.dbg ? W.dbg + (static_cast<size_t>(lidx) * gridDim.x + c) * 32 : nullptr;
#else
    (void)lidx;
#endif
    SG_STAMP(dbg, 0);
    const bool use_as = kPipe != 0 && S.as_bytes > 0;
    bool staged = prestaged;
    // weights of this layer (independent of x), unless the previous layer
    // already staged them during its tail
    if (kPipe != 0 && !prestaged) {
        staged = stage_weights(L, sm, S, use_as);
        if (kPipe == 2) preissue_hot(L, sm, S);
    }
    SG_STAMP(dbg, 1);
    // phase A's row count and the ring / survivor parameters, read before the
    // x wait so their latency hides under it
    const int nB = rows_b(L);
    asm volatile("" ::"r"(nB), "r"(S.stage_off), "r"(S.ns), "r"(S.kc), "r"(S.slot_bytes),
                 "r"(S.sv_chunk), "r"(S.item_cap));
    // no grid barrier between the layers of a stack: the previous layer's y
    // arrives tagged (its tag: the partial barrier it followed)
    const bool bad = first_layer ? stage_x(x, L.d, L.pitch_d, sm.xs, W.xres)
                                 : stage_x_poll(chain ? nullptr : x, chain == 2 ? x : nullptr, W,
                                                L.d, L.pitch_d, sm.xs,
                                                rs.tag0 + rs.bar_k);
    if (c == 0 && tid == 0) {
        // p and v (stats[0], [1]) are zeroed by the host before the launch
        W.stats[2] = bad ? 1 : 0;
        W.stats[3] = kPipe;
    }
    SG_STAMP(dbg, 2);
    if (kPipe != 0) {
        if (staged) {
            mbar_wait(sm.abar, rs.auses & 1u);
            __syncwarp();
            rs.auses += 1;
        }
        // t travels with its tag: no grid barrier between stages 1a and 1b
        const uint32_t tag = rs.tag0 + rs.bar_k + 1u;
        phase_t(L, W, sm, S, S.stage_b != 0, tag, nB);
        SG_STAMP(dbg, 3);
        SG_STAMP(dbg, 4);
        phase_mask(L, W, sm, S, use_as, S.stage_b != 0, nullptr, tag SG_DBG_ARG);
        SG_STAMP(dbg, 6);
    }
    phase_gather<kPipe>(L, W, sm, S);
    SG_STAMP(dbg, 14);
    if (kPipe == 2) {
        survivor_updown(L, W, sm, S, rs);
    } else {
        partial_down<kPipe>(L, W, sm);
    }
    SG_STAMP(dbg, 7);
    // stage the next layer's predictor weights and hot prefix during the
    // barrier: this CTA's ring and survivor rows are done, phase D uses reda
    grid_arrive(W, rs);
    bool next_staged = false;
    if (kPipe != 0 && next != nullptr) {
        next_staged = stage_weights(*next, sm, S, use_as);
        if (kPipe == 2) preissue_hot(*next, sm, S);
    }
    const DownPlan dp = down_plan(L, W);
    grid_wait(W, rs);
    SG_STAMP(dbg, 8);
    phase_down<kPipe>(L, W, sm, y, want_sets, next != nullptr, rs.tag0 + rs.bar_k, dp);
    SG_STAMP(dbg, 9);
    return next_staged;
}

__device__ __noinline__ void init_barriers(uint64_t* bars) {
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2 * kMaxSlots + 1; ++i) mbar_init(bars + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
}

template <int kPipe>
__global__ void __launch_bounds__(kThreads, 1)
    ffn_kernel(const LayerView* __restrict__ layers, int nlayers, LayerView L0, WorkView W,
               SmemPlan S, const float* xs, float* ys, int chain, int xstride) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const Smem sm = carve(smem_raw, S);
    init_barriers(sm.full);
    RunState rs{0u, 0ull, 0u, 0u};
    grid_barrier_init(W, rs);
    if (threadIdx.x < kMaxSlots) sm.uses[threadIdx.x] = 0;
    if (threadIdx.x == 0) sm.misc[4] = 0;
    // barriers completed by all earlier launches on this workspace: a tag base
    // that no value left in the exchange buffers can carry yet
    if (threadIdx.x == 0) sm.misc[9] = static_cast<int>(rs.bar_base / static_cast<uint64_t>(bar_share(0)));
    bool prestaged = false;
    // layer views live in shared memory: the next one is copied during the
    // current layer, so a layer never starts with a global-memory round trip
    constexpr int kLvWords = static_cast<int>(sizeof(LayerView) / 4);
    static_assert(sizeof(LayerView) % 16 == 0, "LayerView is copied in 16-B pieces");
    if (threadIdx.x == 0) {
        if (layers) {
            for (int k = 0; k < kLvWords; ++k)
                reinterpret_cast<int*>(sm.lv)[k] = __ldg(reinterpret_cast<const int*>(layers) + k);
        } else {
            sm.lv[0] = L0;
        }
    }
    __syncthreads();
    rs.tag0 = static_cast<uint32_t>(sm.misc[9]);
    for (int l = 0; l < nlayers; ++l) {
        if (layers && l + 1 < nlayers && threadIdx.x < kLvWords / 4) {
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                             smem_u32(reinterpret_cast<int4*>(sm.lv + ((l + 1) & 1)) + threadIdx.x)),
                         "l"(reinterpret_cast<const int4*>(layers + l + 1) + threadIdx.x)
                         : "memory");
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        const LayerView L = sm.lv[l & 1];
        const LayerView* next = (layers && l + 1 < nlayers) ? layers + l + 1 : nullptr;
        // chain 1: x_l = y_{l-1}; chain 2 (residual): x_l = xs_l + y_{l-1}; 0: x_l = xs_l
        const float* x = (chain == 1 && l > 0) ? ys + static_cast<size_t>(l - 1) * xstride
                                               : xs + static_cast<size_t>(l) * xstride;
        float* y = ys + static_cast<size_t>(l) * xstride;
        WorkView Wl = W;
        Wl.stats = W.stats + 4 * l;  // per-layer {p, v, nonfinite, pipeline}
        Wl.bitpos = l;
        prestaged = run_layer<kPipe>(L, Wl, sm, S, rs, x, y, l == 0, chain, l, l == nlayers - 1,
                                     next, prestaged);
        if (layers && l + 1 < nlayers) {
            if (threadIdx.x < kLvWords / 4) asm volatile("cp.async.wait_all;" ::: "memory");
            __syncthreads();
        }
    }
}

// Predictor-only kernel (sg_predict_mask): phases A and B, weights streamed.
__global__ void __launch_bounds__(kThreads, 1)
    predict_kernel(LayerView L, WorkView W, SmemPlan S, uint8_t* mask_out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const Smem sm = carve(smem_raw, S);
    init_barriers(sm.full);
    RunState rs{0u, 0ull, 0u, 0u};
    grid_barrier_init(W, rs);
    if (threadIdx.x == 0) sm.misc[4] = 0;
    if (threadIdx.x == 0) sm.misc[9] = static_cast<int>(rs.bar_base / static_cast<uint64_t>(bar_share(0)));
    stage_weights(L, sm, S, false);  // bias only (S.stage_b == 0)
    const bool bad = stage_x(W.x, L.d, L.pitch_d, sm.xs);  // (block barrier inside)
    rs.tag0 = static_cast<uint32_t>(sm.misc[9]);
    if (blockIdx.x == 0 && threadIdx.x == 0) W.stats[2] = bad ? 1 : 0;
    const uint32_t tag = rs.tag0 + 1u;
    phase_t(L, W, sm, S, false, tag, rows_b(L));
#ifdef SG_PHASE_TIMING
    uint64_t* dbg = nullptr;
#endif
    phase_mask(L, W, sm, S, false, false, mask_out, tag SG_DBG_ARG);
    grid_barrier(W, rs);
    if (threadIdx.x < 32 && blockIdx.x == 0) {
        warp_prefix(W.cnt, sm.off, gridDim.x, threadIdx.x);
        if (threadIdx.x == 0) W.stats[0] = sm.off[gridDim.x];
    }
}

int align_up(int v, int a) { return (v + a - 1) / a * a; }

// Shared-memory plan for a layer shape at G CTAs.
bool make_plan(int G, int pitch_d, int r, int pitch_r, int Dl, int pipe, int max_smem,
               SmemPlan* S, int kc_override = 0, int ns_override = 0) {
    int off = 3 * kMaxSlots * 8;  // full, empty, abar
    off = align_up(off, 128);
    S->off_slotn = off;
    off += kMaxSlots * 4;
    S->off_uses = off;
    off += kMaxSlots * 4;
    S->off_off = off = align_up(off, 16);
    off += (G + 1) * 4;
    S->mask_cap = align_up((Dl + G - 1) / G + 1, 16);
    S->off_mask = off = align_up(off, 16);
    off += S->mask_cap;
    S->off_bias = off = align_up(off, 16);
    off += S->mask_cap * 4;
    S->off_misc = off = align_up(off, 16);
    off += 32 * 4;
    S->off_lv = off = align_up(off, 16);
    off += 2 * static_cast<int>(sizeof(LayerView));
    S->off_reda = off = align_up(off, 16);
    off += 512 * 4;  // phase A: kRowsA*kWarps; C: kGroups*2*kGroupWarps*4; 4: 2*kWarps*kBatch; D: kCThreads
    S->item_cap = (Dl + G - 1) / G + 2;
    S->off_items = off = align_up(off, 16);
    off += S->item_cap * 4;
    S->off_recs = off = align_up(off, 16);
    off += S->item_cap * 8;
    S->off_sv = off = align_up(off, 16);
    off += S->item_cap * 8 + kSvChunk * 4;
    S->off_xs = off = align_up(off, 128);
    off += pitch_d * 4;
    S->off_ts = off = align_up(off, 128);
    off += pitch_r * 4;
    S->off_big = off = align_up(off, 1024);
    const int avail = max_smem - off;
    if (avail < S->item_cap * 8) return false;
    // phases A/B staging
    const int nB = (r + G - 1) / G;
    const int b_bytes = nB * pitch_d * 2;
    int as_bytes = 0;
    if (pipe != 0) as_bytes = align_up(((Dl + G - 1) / G + 1) * pitch_r * 2, 16);
    S->stage_b = (pipe != 0 && b_bytes + as_bytes <= avail) ? 1 : 0;
    if (!S->stage_b && pipe != 0 && as_bytes > avail) as_bytes = 0;
    S->as_bytes = as_bytes;
    // the staging area sits at the top of the big region, under the ring's last slots
    S->stage_off = (avail - (S->stage_b ? b_bytes : 0) - as_bytes) / 128 * 128;
    // phase C ring
    S->slot_bytes = (pipe == 2 ? 1 : 2) * pitch_d * 2;
    S->pre_slots = S->stage_off / S->slot_bytes;
    int ns_max = avail / S->slot_bytes;
    if (ns_max > kMaxSlots - 2) ns_max = kMaxSlots - 2;  // full[kMaxSlots-2..]: survivor buffers
    if (ns_max < 1) return false;
    int kc = ns_max < kGroups ? ns_max : kGroups;
    if (kc_override > 0 && kc_override < kc) kc = kc_override;
    if (ns_override > 0 && ns_override < ns_max) ns_max = ns_override;
    if (ns_max < kc) kc = ns_max;
    S->kc = kc;
    S->ns = kc * (ns_max / kc);
    S->big_bytes = avail;
    S->sv_chunk = avail / (pitch_d * 4) < kSvChunk ? avail / (pitch_d * 4) : kSvChunk;
    if (pipe == 2 && S->sv_chunk < 2) return false;  // two survivor row buffers
    S->total = max_smem;
    return true;
}

}  // namespace

// Raise a kernel's dynamic-smem cap once per (kernel, device): the attribute is
// per device context, so a ctx on a second device in the same process needs its
// own call. Process-wide, mutex-protected; errors propagate.
int ensure_smem_attr(const void* kernel, int smem) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> done;
    std::lock_guard<std::mutex> lock(mu);
    auto it = done.find({kernel, dev});
    if (it != done.end() && it->second >= smem) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    done[{kernel, dev}] = smem;
    return cudaSuccess;
}

namespace {

template <typename K>
int launch_coop(K kernel, int G, int smem, cudaStream_t stream, void** args) {
    const int e = ensure_smem_attr(reinterpret_cast<const void*>(kernel), smem);
    if (e != cudaSuccess) return e;
    return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kernel), dim3(G),
                                       dim3(kThreads), args, static_cast<size_t>(smem), stream);
}

int smem_budget() {
    int dev = 0;
    cudaGetDevice(&dev);
    int max_smem = 0;
    cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return max_smem - 1024;
}

int launch_ffn(const LayerView* layers_dev, int nlayers, const LayerView& L0, const WorkView& W,
               const float* xs, float* ys, int chain, int xstride, int pipeline, int G,
               cudaStream_t stream) {
    SmemPlan S;
    if (!make_plan(G, L0.pitch_d, L0.r, L0.pitch_r, L0.D, pipeline, smem_budget(), &S,
                   (W.flags >> 8) & 0xff, (W.flags >> 16) & 0xff))
        return cudaErrorInvalidConfiguration;
    WorkView Wc = W;
    void* args[] = {(void*)&layers_dev, (void*)&nlayers, (void*)&L0, (void*)&Wc, (void*)&S,
                    (void*)&xs, (void*)&ys, (void*)&chain, (void*)&xstride};
    switch (pipeline) {
        case 0: return launch_coop(ffn_kernel<0>, G, S.total, stream, args);
        case 1: return launch_coop(ffn_kernel<1>, G, S.total, stream, args);
        default: return launch_coop(ffn_kernel<2>, G, S.total, stream, args);
    }
}

}  // namespace

int launch_layer(const LayerView& L, const WorkView& W, int pipeline, int num_ctas, void* stream) {
    return launch_ffn(nullptr, 1, L, W, W.x, W.y, 0, 0, pipeline, num_ctas,
                      static_cast<cudaStream_t>(stream));
}

int launch_layers(const LayerView* layers_dev, int n, const LayerView& first, const WorkView& W,
                  const float* xs, float* ys, int chain, int pitch_stride, int pipeline,
                  int num_ctas, void* stream) {
    return launch_ffn(layers_dev, n, first, W, xs, ys, chain, pitch_stride, pipeline, num_ctas,
                      static_cast<cudaStream_t>(stream));
}

int launch_predict(const LayerView& L, const WorkView& W, uint8_t* mask_out, int num_ctas,
                   void* stream) {
    SmemPlan S;
    if (!make_plan(num_ctas, L.pitch_d, L.r, L.pitch_r, L.D, 0, smem_budget(), &S))
        return cudaErrorInvalidConfiguration;
    S.stage_b = 0;
    S.as_bytes = 0;
    LayerView Lc = L;
    WorkView Wc = W;
    void* args[] = {(void*)&Lc, (void*)&Wc, (void*)&S, (void*)&mask_out};
    return launch_coop(predict_kernel, num_ctas, S.total, static_cast<cudaStream_t>(stream),
                       args);
}

int query_launch_info(int device, LaunchInfo* info) {
    cudaError_t e = cudaDeviceGetAttribute(&info->num_sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    return cudaDeviceGetAttribute(&info->max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
}

}  // namespace sg
