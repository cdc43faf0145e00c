// sparsegate-b200 device code: the sparse gated-FFN decode executor for sm_100a.
//
// One persistent, cooperative launch per layer (or per stack of layers) runs
// the five stages of the reference's sequential pipeline
// (/root/reference/proj/include/sparsegate/ffn_exec.hpp:183-218):
//
//   phase A  stage 1a  t = B·x                       (ffn_exec.hpp:133-136)
//            --- grid barrier ---
//   phase B  stage 1b  pre = A·t + bias > 0 -> mask  (ffn_exec.hpp:139-144)
//            stage 2   per-CTA warp-ballot compaction (ffn_exec.hpp:189-195)
//            --- grid barrier ---
//   phase C  stage 3   gather-GEMV over predicted gate rows, staged into a
//                      shared-memory ring by cp.async.bulk (TMA bulk engine) +
//                      mbarriers; revalidation g > 0      (ffn_exec.hpp:196-201)
//            stage 4   survivors only: up row -> z = gated(g, u) (ffn_exec.hpp:202-203, :68-76)
//            second compaction (survivor list)
//            --- grid barrier ---
//   phase D  stage 5   down projection over neuron-major rows, column-sliced
//                      with a fixed-order cross-CTA reduction (ffn_exec.hpp:80-94)
//
// Dense (ffn_exec.hpp:103-122) and parallel (ffn_exec.hpp:149-178) pipelines
// reuse phases C/D with gate+up rows fetched together.
//
// Determinism: no floating-point atomics. Every dot product has a fixed lane
// -> chunk assignment and a fixed shuffle tree, so a given row gives the same
// bits whichever CTA/warp computes it; the down projection sums each column
// in a fixed order over (survivor position, warp, group). Repeated calls are
// bit-identical, and the sequential and parallel pipelines are bit-identical
// on the same mask (the reference's determinism contract, ffn_exec.hpp:3-15).
#include "sg_internal.h"

#include <cuda_runtime.h>

#include <cstdint>

namespace sg {
namespace {

constexpr int kWarps = 16;                  // compute warps
constexpr int kCThreads = kWarps * 32;      // 512 compute threads
constexpr int kThreads = kCThreads + 32;    // + one producer warp (cp.async.bulk issue)
constexpr int kMaxSlots = 32;               // ring slots (upper bound)
constexpr int kSliceChunks = 32;            // phase D: 32 lanes x 16 B
constexpr int kSliceCols = kSliceChunks * 8;  // = 256 output columns per slice
constexpr int kRowsA = 4;                   // phase A rows reduced per pass

struct SmemPlan {
    int off_slotn;  // int[kMaxSlots]
    int off_off;    // int[G+1]   P prefix
    int off_voff;   // int[G+1]   V prefix
    int off_red;    // float[kWarps*32*8]
    int off_mask;   // uint8[mask_cap]
    int off_xs;     // float[pitch_d]
    int off_ts;     // float[pitch_r]
    int off_as;     // uint16[as_cap]
    int off_ring;   // ns * slot_bytes
    int ns;
    int slot_bytes;
    int as_cap_bytes;
    int mask_cap;
    int total;
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
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
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
__device__ __forceinline__ uint32_t ld_acquire(const unsigned* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

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

// Canonical row dot: lane l owns chunks l, l+32, ... and accumulates them in
// order; then the butterfly. Identical for rows read from smem or global.
template <bool kSmem>
__device__ __forceinline__ float row_dot(const uint16_t* row, const float* xs, int nch, int lane) {
    float acc = 0.f;
    if (kSmem) {
        for (int c = lane; c < nch; c += 32)
            acc = dot8(*reinterpret_cast<const uint4*>(row + c * 8), xs + c * 8, acc);
    } else {
        // Issue the whole row's loads first (up to 16 x 16 B per lane in flight).
        int c = lane;
        for (; c + 32 * 15 < nch; c += 32 * 16) {
            uint4 w[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) w[k] = ldg_stream(row + (c + 32 * k) * 8);
#pragma unroll
            for (int k = 0; k < 16; ++k) acc = dot8(w[k], xs + (c + 32 * k) * 8, acc);
        }
        for (; c < nch; c += 32) acc = dot8(ldg_stream(row + c * 8), xs + c * 8, acc);
    }
    return warp_sum(acc);
}
// Two rows (gate, up) sharing the x loads; per-row accumulation identical to row_dot.
__device__ __forceinline__ void row_dot2(const uint16_t* r0, const uint16_t* r1, const float* xs,
                                         int nch, int lane, float& o0, float& o1) {
    float a0 = 0.f, a1 = 0.f;
    for (int c = lane; c < nch; c += 32) {
        a0 = dot8(*reinterpret_cast<const uint4*>(r0 + c * 8), xs + c * 8, a0);
        a1 = dot8(*reinterpret_cast<const uint4*>(r1 + c * 8), xs + c * 8, a1);
    }
    o0 = warp_sum(a0);
    o1 = warp_sum(a1);
}

// ffn_exec.hpp:68-76 in fp32 (canonical +0 when suppressed).
__device__ __forceinline__ float gated(float g, float u, int act) {
    if (!(g > 0.f)) return 0.f;
    if (act == 1 && !(u > 0.f)) return 0.f;
    return g * u;
}

__device__ __forceinline__ int split_lo(int c, int G, int n) {
    return static_cast<int>((static_cast<long long>(c) * n) / G);
}

// Sense-free grid barrier (count returns to 0, generation advances). All CTAs
// are co-resident (cooperative launch, one CTA per SM).
__device__ __forceinline__ void grid_barrier(unsigned* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t gen = ld_acquire(bar + 1);
        __threadfence();
        const unsigned arrived = atomicAdd(bar, 1u);
        if (arrived == gridDim.x - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            st_release(bar + 1, gen + 1);
        } else {
            while (ld_acquire(bar + 1) == gen) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// Exclusive prefix of cnt[0..G) into off[0..G], off[G] = total. Warp 0 only.
__device__ __forceinline__ void warp_prefix(const int* cnt, int* off, int G, int lane) {
    int carry = 0;
    for (int base = 0; base < G; base += 32) {
        const int i = base + lane;
        const int v = i < G ? __ldcg(cnt + i) : 0;
        int incl = v;
#pragma unroll
        for (int m = 1; m < 32; m <<= 1) {
            const int o = __shfl_up_sync(0xffffffffu, incl, m);
            if (lane >= m) incl += o;
        }
        if (i < G) off[i] = carry + incl - v;
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) off[G] = carry;
}

// Owner CTA s of list position pos: off[s] <= pos < off[s+1] (off ascending).
__device__ __forceinline__ int owner_of(const int* off, int G, int pos) {
    int lo = 0, hi = G;  // off[lo] <= pos < off[hi]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (off[mid] <= pos) lo = mid; else hi = mid;
    }
    return lo;
}

struct Smem {
    uint64_t* full;
    uint64_t* empty;
    uint64_t* abar;
    int* slotn;
    int* off;
    int* voff;
    float* red;
    uint8_t* mask;
    float* xs;
    float* ts;
    uint16_t* as;
    uint8_t* ring;
};

__device__ __forceinline__ Smem carve(uint8_t* base, const SmemPlan& S) {
    Smem m;
    m.full = reinterpret_cast<uint64_t*>(base);
    m.empty = m.full + kMaxSlots;
    m.abar = m.empty + kMaxSlots;
    m.slotn = reinterpret_cast<int*>(base + S.off_slotn);
    m.off = reinterpret_cast<int*>(base + S.off_off);
    m.voff = reinterpret_cast<int*>(base + S.off_voff);
    m.red = reinterpret_cast<float*>(base + S.off_red);
    m.mask = base + S.off_mask;
    m.xs = reinterpret_cast<float*>(base + S.off_xs);
    m.ts = reinterpret_cast<float*>(base + S.off_ts);
    m.as = reinterpret_cast<uint16_t*>(base + S.off_as);
    m.ring = base + S.off_ring;
    return m;
}

// Per-CTA persistent pipeline state (identical in every thread of the CTA).
struct RingState {
    uint32_t seq;   // items pushed through the ring so far (this launch)
    uint32_t auses; // A-slice barrier uses so far
};

// ---------------------------------------------------------------------------
// Phase A: t = B·x (fp32), rows j = c, c+G, ... ; block-reduced in fixed order.
// ---------------------------------------------------------------------------
__device__ void phase_t(const LayerView& L, const WorkView& W, const Smem& sm) {
    const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int nch = L.pitch_d >> 3;
    for (int j0 = c; j0 < L.r; j0 += kRowsA * G) {
        float acc[kRowsA];
#pragma unroll
        for (int q = 0; q < kRowsA; ++q) acc[q] = 0.f;
        if (tid < kCThreads) {
            for (int ch = tid; ch < nch; ch += kCThreads) {
                uint4 w[kRowsA];
#pragma unroll
                for (int q = 0; q < kRowsA; ++q) {
                    const int j = j0 + q * G;
                    w[q] = j < L.r ? ldg_stream(L.B + static_cast<size_t>(j) * L.pitch_d + ch * 8)
                                   : make_uint4(0, 0, 0, 0);
                }
#pragma unroll
                for (int q = 0; q < kRowsA; ++q) acc[q] = dot8(w[q], sm.xs + ch * 8, acc[q]);
            }
#pragma unroll
            for (int q = 0; q < kRowsA; ++q) {
                const float s = warp_sum(acc[q]);
                if (lane == 0) sm.red[q * kWarps + warp] = s;
            }
        }
        __syncthreads();
        if (tid < kRowsA) {
            const int j = j0 + tid * G;
            if (j < L.r) {
                float s = 0.f;
                for (int w = 0; w < kWarps; ++w) s += sm.red[tid * kWarps + w];
                W.t[j] = s;
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Phase B: mask over this CTA's neuron range + warp-ballot compaction.
// ---------------------------------------------------------------------------
__device__ void phase_mask(const LayerView& L, const WorkView& W, const Smem& sm, bool use_as,
                           RingState& rs, uint8_t* mask_out) {
    const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int n0 = split_lo(c, G, L.D), n1 = split_lo(c + 1, G, L.D);
    for (int i = tid; i < L.pitch_r; i += kThreads) sm.ts[i] = i < L.r ? __ldcg(W.t + i) : 0.f;
    if (use_as && n1 > n0) {
        mbar_wait(sm.abar, rs.auses & 1u);
    }
    if (n1 > n0) rs.auses += use_as ? 1u : 0u;
    __syncthreads();
    const int nchr = L.pitch_r >> 3;
    if (warp < kWarps) {
        for (int n = n0 + warp; n < n1; n += kWarps) {
            const uint16_t* arow = use_as ? sm.as + static_cast<size_t>(n - n0) * L.pitch_r
                                          : L.A + static_cast<size_t>(n) * L.pitch_r;
            float acc = 0.f;
            for (int ch = lane; ch < nchr; ch += 32) {
                const uint4 w = use_as ? *reinterpret_cast<const uint4*>(arow + ch * 8)
                                       : ldg_stream(arow + ch * 8);
                acc = dot8(w, sm.ts + ch * 8, acc);
            }
            acc = warp_sum(acc);
            if (lane == 0) {
                const float pre = acc + __ldg(L.bias + n);
                const uint8_t on = pre > 0.f ? 1 : 0;  // strict, ffn_exec.hpp:141
                sm.mask[n - n0] = on;
                if (mask_out) mask_out[n] = on;
            }
        }
    }
    __syncthreads();
    if (warp == 0) {
        int run = 0;
        for (int base = 0; base < n1 - n0; base += 32) {
            const int k = base + lane;
            const bool on = k < n1 - n0 && sm.mask[k];
            const unsigned b = __ballot_sync(0xffffffffu, on);
            if (on) W.plist[n0 + run + __popc(b & ((1u << lane) - 1u))] = n0 + k;
            run += __popc(b);
        }
        if (lane == 0) W.cnt[c] = run;
    }
}

// ---------------------------------------------------------------------------
// Phase C: gather-GEMV over list items through the cp.async.bulk ring.
//   kPipe 2 (sequential): items = P positions; slot = gate row; survivors fetch
//                         their up row directly (LDG) -> z.
//   kPipe 1 (parallel):   items = P positions; slot = gate row + up row.
//   kPipe 0 (dense):      items = neurons of this CTA's range; slot = gate + up.
// ---------------------------------------------------------------------------
template <int kPipe>
__device__ void phase_gather(const LayerView& L, const WorkView& W, const Smem& sm,
                             const SmemPlan& S, RingState& rs, int& i0_out, int& i1_out) {
    const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int nch = L.pitch_d >> 3;
    const uint32_t row_bytes = static_cast<uint32_t>(L.pitch_d) * 2u;
    int i0, i1;
    if (kPipe == 0) {
        i0 = split_lo(c, G, L.D);
        i1 = split_lo(c + 1, G, L.D);
    } else {
        if (warp == 0) warp_prefix(W.cnt, sm.off, G, lane);
        __syncthreads();
        const int p = sm.off[G];
        i0 = split_lo(c, G, p);
        i1 = split_lo(c + 1, G, p);
        if (c == 0 && tid == 0) W.stats[0] = p;
    }
    i0_out = i0;
    i1_out = i1;
    const int nitems = i1 - i0;
    const uint32_t seq0 = rs.seq;
    const int ns = S.ns;

    if (warp == kWarps) {
        // ---- producer warp: one lane issues the bulk copies ----
        if (lane == 0 && nitems > 0) {
            const uint64_t pol = policy_evict_first();
            int s = 0, k = 0;
            if (kPipe != 0) {
                s = owner_of(sm.off, G, i0);
                k = i0 - sm.off[s];
            }
            for (int j = 0; j < nitems; ++j) {
                int n;
                if (kPipe == 0) {
                    n = i0 + j;
                } else {
                    while (k >= sm.off[s + 1] - sm.off[s]) {
                        ++s;
                        k = 0;
                    }
                    n = __ldcg(W.plist + split_lo(s, G, L.D) + k);
                    ++k;
                }
                const uint32_t q = seq0 + j;
                const int slot = static_cast<int>(q % ns);
                const uint32_t use = q / ns;
                if (use > 0) mbar_wait(sm.empty + slot, (use - 1) & 1u);
                sm.slotn[slot] = n;
                uint8_t* dst = sm.ring + static_cast<size_t>(slot) * S.slot_bytes;
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
    } else {
        // ---- compute warps ----
        for (int j = warp; j < nitems; j += kWarps) {
            const uint32_t q = seq0 + j;
            const int slot = static_cast<int>(q % ns);
            mbar_wait(sm.full + slot, (q / ns) & 1u);
            const int n = sm.slotn[slot];
            const uint16_t* srow =
                reinterpret_cast<const uint16_t*>(sm.ring + static_cast<size_t>(slot) * S.slot_bytes);
            float g, u = 0.f;
            if (kPipe == 2) {
                g = row_dot<true>(srow, sm.xs, nch, lane);
            } else {
                row_dot2(srow, srow + L.pitch_d, sm.xs, nch, lane, g, u);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(sm.empty + slot);  // slot free: reads are done
            const int it = i0 + j;
            if (kPipe == 0) {
                if (lane == 0) W.zD[n] = gated(g, u, L.act);
            } else {
                const bool sv = g > 0.f;  // revalidation, ffn_exec.hpp:200 (strict)
                if (kPipe == 2 && sv) {
                    u = row_dot<false>(L.ud + static_cast<size_t>(n) * 2 * L.pitch_d, sm.xs, nch,
                                       lane);
                }
                if (lane == 0) {
                    W.P[it] = L.gbase + n * L.gstride;
                    W.Pl[it] = n;
                    W.gP[it] = g;
                    W.surv[it] = sv ? 1 : 0;
                    W.zP[it] = sv ? gated(g, u, L.act) : 0.f;
                }
            }
        }
    }
    rs.seq = seq0 + static_cast<uint32_t>(nitems > 0 ? nitems : 0);
    __syncthreads();
    if (kPipe != 0 && warp == 0) {
        // second compaction: survivors of this CTA's item range, in P order.
        int run = 0;
        for (int base = 0; base < nitems; base += 32) {
            const int j = base + lane;
            const bool on = j < nitems && W.surv[i0 + j] != 0;
            const unsigned b = __ballot_sync(0xffffffffu, on);
            if (on) {
                const int dst = i0 + run + __popc(b & ((1u << lane) - 1u));
                W.vlist[dst] = W.Pl[i0 + j];
                W.zlist[dst] = W.zP[i0 + j];
            }
            run += __popc(b);
        }
        if (lane == 0) W.cnt[G + c] = run;
    }
}

// ---------------------------------------------------------------------------
// Phase D: y = sum over list positions of z * down_row, column-sliced.
// Work item = (column slice of 256, position group q of Q). Each item is
// reduced over its 16 warps in fixed order; the Q group partials of a slice are
// summed in fixed q order by whichever CTA arrives last.
// ---------------------------------------------------------------------------
template <int kPipe>
__device__ void phase_down(const LayerView& L, const WorkView& W, const Smem& sm, float* y,
                           int p_total_i0_unused) {
    (void)p_total_i0_unused;
    const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int nch = L.pitch_d >> 3;
    int v;       // list length
    int p = 0;   // P length (sparse)
    if (kPipe == 0) {
        v = L.D;
    } else {
        if (warp == 0) warp_prefix(W.cnt + G, sm.voff, G, lane);
        __syncthreads();
        v = sm.voff[G];
        p = sm.off[G];
        // publish this CTA's survivor segment as the compacted global V list
        const int i0 = split_lo(c, G, p);
        const int cntc = sm.voff[c + 1] - sm.voff[c];
        for (int k = tid; k < cntc; k += kThreads) {
            const int n = W.vlist[i0 + k];
            W.V[sm.voff[c] + k] = L.gbase + n * L.gstride;
            W.zV[sm.voff[c] + k] = W.zlist[i0 + k];
        }
        if (c == 0 && tid == 0) W.stats[1] = v;
    }
    const int nslices = (nch + kSliceChunks - 1) / kSliceChunks;
    int Q = G / nslices;
    if (Q < 1) Q = 1;
    const int nitems = nslices * Q;
    for (int item = c; item < nitems; item += G) {
        const int slice = item % nslices;
        const int q = item / nslices;
        const int g0 = split_lo(q, Q, v), g1 = split_lo(q + 1, Q, v);
        const int chunk = slice * kSliceChunks + lane;
        const bool col_ok = chunk < nch;
        float acc[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = 0.f;
        if (warp < kWarps) {
            // positions handled by this warp: g0 + warp + 16*k
            for (int pass = g0 + warp; pass < g1; pass += kWarps * 32) {
                // lane l resolves position pass + 16*l
                const int mypos = pass + kWarps * lane;
                int myn = 0;
                float myz = 0.f;
                if (mypos < g1) {
                    if (kPipe == 0) {
                        myn = mypos;
                        myz = __ldcg(W.zD + mypos);
                    } else {
                        const int s = owner_of(sm.voff, G, mypos);
                        const int src = split_lo(s, G, p) + (mypos - sm.voff[s]);
                        myn = __ldcg(W.vlist + src);
                        myz = __ldcg(W.zlist + src);
                    }
                }
                const int cnt = min(32, (g1 - pass + kWarps - 1) / kWarps);
                int k = 0;
                for (; k + 4 <= cnt; k += 4) {
                    uint4 w[4];
                    float z[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int n = __shfl_sync(0xffffffffu, myn, k + u);
                        z[u] = __shfl_sync(0xffffffffu, myz, k + u);
                        w[u] = col_ok ? ldg_stream(L.ud + static_cast<size_t>(n) * 2 * L.pitch_d +
                                                   L.pitch_d + chunk * 8)
                                      : make_uint4(0, 0, 0, 0);
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) axpy8(w[u], z[u], acc);
                }
                for (; k < cnt; ++k) {
                    const int n = __shfl_sync(0xffffffffu, myn, k);
                    const float z = __shfl_sync(0xffffffffu, myz, k);
                    const uint4 w = col_ok ? ldg_stream(L.ud + static_cast<size_t>(n) * 2 *
                                                                   L.pitch_d +
                                                        L.pitch_d + chunk * 8)
                                           : make_uint4(0, 0, 0, 0);
                    axpy8(w, z, acc);
                }
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) sm.red[(warp * 32 + lane) * 8 + e] = acc[e];
        }
        __syncthreads();
        // fixed-order sum over the 16 warps: thread t -> (lane t>>3, element t&7)
        float s = 0.f;
        const int col = slice * kSliceCols + tid;  // tid in [0,256): chunk lane tid>>3, elem tid&7
        if (tid < kSliceCols) {
            const int l = tid >> 3, e = tid & 7;
            for (int w = 0; w < kWarps; ++w) s += sm.red[(w * 32 + l) * 8 + e];
            if (Q == 1) {
                if (col < L.d) y[col] = s;
            } else {
                W.ypart[static_cast<size_t>(q) * L.pitch_d + col] = s;
                __threadfence();
            }
        }
        if (Q > 1) {
            __shared__ int s_last;
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                const unsigned prev = atomicAdd(W.slice_ctr + slice, 1u);
                s_last = prev == static_cast<unsigned>(Q - 1);
                if (s_last) W.slice_ctr[slice] = 0u;  // self-reset for the next use
                __threadfence();
            }
            __syncthreads();
            if (s_last && tid < kSliceCols && col < L.d) {
                float tot = 0.f;
                for (int qq = 0; qq < Q; ++qq)
                    tot += __ldcg(W.ypart + static_cast<size_t>(qq) * L.pitch_d + col);
                y[col] = tot;
            }
        }
        __syncthreads();
    }
}

// Stage x (fp32, length d) into smem, zero-padded to pitch_d; flag non-finite.
__device__ __forceinline__ bool stage_x(const float* x, int d, int pitch_d, float* xs) {
    bool bad = false;
    for (int i = threadIdx.x; i < pitch_d; i += kThreads) {
        const float v = i < d ? __ldcg(x + i) : 0.f;
        xs[i] = v;
        bad |= !isfinite(v);
    }
    return __syncthreads_or(bad) != 0;
}

template <int kPipe>
__device__ void run_layer(const LayerView& L, const WorkView& W, const Smem& sm,
                          const SmemPlan& S, RingState& rs, const float* x, float* y,
                          bool first_layer) {
    const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x;
    const bool use_as = kPipe != 0 && S.as_cap_bytes > 0;
    // A-slice prefetch (does not depend on x): overlaps phase A and barrier 1.
    if (use_as && tid == kCThreads) {
        const int n0 = split_lo(c, G, L.D), n1 = split_lo(c + 1, G, L.D);
        if (n1 > n0) {
            const uint32_t bytes = static_cast<uint32_t>(n1 - n0) * L.pitch_r * 2u;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // WAR vs. last layer's reads
            mbar_expect_tx(sm.abar, bytes);
            bulk_g2s(sm.as, L.A + static_cast<size_t>(n0) * L.pitch_r, bytes, sm.abar,
                     policy_evict_first());
        }
    }
    if (!first_layer) grid_barrier(W.bar);  // previous layer's y is complete
    const bool bad = stage_x(x, L.d, L.pitch_d, sm.xs);
    if (c == 0 && tid == 0) {
        W.stats[2] = bad ? 1 : 0;
        W.stats[3] = kPipe;
    }
    int i0 = 0, i1 = 0;
    if (kPipe != 0) {
        phase_t(L, W, sm);
        grid_barrier(W.bar);
        phase_mask(L, W, sm, use_as, rs, nullptr);
        grid_barrier(W.bar);
    }
    phase_gather<kPipe>(L, W, sm, S, rs, i0, i1);
    grid_barrier(W.bar);
    phase_down<kPipe>(L, W, sm, y, 0);
}

__device__ __forceinline__ void init_barriers(const Smem& sm) {
    if (threadIdx.x == 0) {
        for (int i = 0; i < kMaxSlots; ++i) {
            mbar_init(sm.full + i, 1);
            mbar_init(sm.empty + i, 1);
        }
        mbar_init(sm.abar, 1);
        fence_mbar_init();
    }
    __syncthreads();
}

template <int kPipe>
__global__ void __launch_bounds__(kThreads, 1)
    ffn_kernel(const LayerView* __restrict__ layers, int nlayers, LayerView L0, WorkView W,
               SmemPlan S, const float* xs, float* ys, int chain, int xstride) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const Smem sm = carve(smem_raw, S);
    init_barriers(sm);
    RingState rs{0u, 0u};
    for (int l = 0; l < nlayers; ++l) {
        const LayerView L = layers ? layers[l] : L0;
        const float* x = (chain && l > 0) ? ys + static_cast<size_t>(l - 1) * xstride
                                          : xs + static_cast<size_t>(l) * xstride;
        float* y = ys + static_cast<size_t>(l) * xstride;
        WorkView Wl = W;
        Wl.stats = W.stats + 4 * l;  // per-layer {p, v, nonfinite, pipeline}
        run_layer<kPipe>(L, Wl, sm, S, rs, x, y, l == 0);
    }
}

// Predictor-only kernel (sg_predict_mask): phases A and B.
__global__ void __launch_bounds__(kThreads, 1)
    predict_kernel(LayerView L, WorkView W, SmemPlan S, uint8_t* mask_out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const Smem sm = carve(smem_raw, S);
    init_barriers(sm);
    RingState rs{0u, 0u};
    const bool bad = stage_x(W.x, L.d, L.pitch_d, sm.xs);
    if (blockIdx.x == 0 && threadIdx.x == 0) W.stats[2] = bad ? 1 : 0;
    phase_t(L, W, sm);
    grid_barrier(W.bar);
    phase_mask(L, W, sm, false, rs, mask_out);
    grid_barrier(W.bar);
    if (threadIdx.x < 32 && blockIdx.x == 0) {
        warp_prefix(W.cnt, sm.off, gridDim.x, threadIdx.x);
        if (threadIdx.x == 0) W.stats[0] = sm.off[gridDim.x];
    }
}

int align_up(int v, int a) { return (v + a - 1) / a * a; }

// Shared-memory plan for a layer shape at G CTAs.
bool make_plan(int G, int pitch_d, int pitch_r, int Dl, int pipe, int max_smem, SmemPlan* S) {
    int off = 3 * kMaxSlots * 8;  // full, empty, abar (+ spare)
    off = align_up(off, 128);
    S->off_slotn = off;
    off += kMaxSlots * 4;
    S->off_off = off = align_up(off, 16);
    off += (G + 1) * 4;
    S->off_voff = off = align_up(off, 16);
    off += (G + 1) * 4;
    S->off_red = off = align_up(off, 128);
    off += kWarps * 32 * 8 * 4;
    S->mask_cap = align_up((Dl + G - 1) / G + 1, 16);
    S->off_mask = off;
    off += S->mask_cap;
    S->off_xs = off = align_up(off, 128);
    off += pitch_d * 4;
    S->off_ts = off = align_up(off, 128);
    off += pitch_r * 4;
    S->off_as = off = align_up(off, 128);
    int as_bytes = 0;
    if (pipe != 0) {
        as_bytes = ((Dl + G - 1) / G + 1) * pitch_r * 2;
        if (as_bytes > 64 * 1024) as_bytes = 0;  // fall back to streaming A from HBM
    }
    S->as_cap_bytes = as_bytes;
    off += as_bytes;
    S->off_ring = off = align_up(off, 128);
    S->slot_bytes = (pipe == 2 ? 1 : 2) * pitch_d * 2;
    int ns = (max_smem - off) / S->slot_bytes;
    if (ns > kMaxSlots) ns = kMaxSlots;
    if (ns < 2) return false;
    S->ns = ns;
    S->total = off + ns * S->slot_bytes;
    return true;
}

template <typename K>
int launch_coop(K kernel, int G, int smem, cudaStream_t stream, void** args) {
    // Raise the dynamic-smem cap once per kernel (per process; one device per process).
    static thread_local const void* set_for[8] = {};
    static thread_local int set_smem[8] = {};
    const void* key = reinterpret_cast<const void*>(kernel);
    int slot = 0;
    while (slot < 8 && set_for[slot] != nullptr && set_for[slot] != key) ++slot;
    if (slot == 8 || set_for[slot] != key || set_smem[slot] < smem) {
        cudaError_t e =
            cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        if (slot < 8) {
            set_for[slot] = key;
            set_smem[slot] = smem;
        }
    }
    return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kernel), dim3(G),
                                       dim3(kThreads), args, static_cast<size_t>(smem), stream);
}

int launch_ffn(const LayerView* layers_dev, int nlayers, const LayerView& L0, const WorkView& W,
               const float* xs, float* ys, int chain, int xstride, int pipeline, int G,
               cudaStream_t stream) {
    int dev = 0;
    cudaGetDevice(&dev);
    int max_smem = 0;
    cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    SmemPlan S;
    if (!make_plan(G, L0.pitch_d, L0.pitch_r, L0.D, pipeline, max_smem, &S))
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
    int dev = 0;
    cudaGetDevice(&dev);
    int max_smem = 0;
    cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    SmemPlan S;
    if (!make_plan(num_ctas, L.pitch_d, L.pitch_r, L.D, 0, max_smem, &S))
        return cudaErrorInvalidConfiguration;
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
