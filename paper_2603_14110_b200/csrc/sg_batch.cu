// sparsegate-b200: batched decode (BASELINE.json configs[4]) — B tokens, one layer.
//
// Per token the result means exactly what sparse_ffn_sequential
// (/root/reference/proj/include/sparsegate/ffn_exec.hpp:183-218) returns for
// that token alone: its own predicted set P_b (pre > 0, :141), survivors V_b
// (g > 0, :200), gated values (:68-76) and y_b over V_b. The batch shares the
// weight traffic: every gate row of the union of the P_b and every [up|down]
// row of the union of the V_b is read ONCE and multiplied against all tokens
// on the tensor cores (the gathered block is a real dense contraction).
//
// Stages (one launch each; all orders fixed, so results are deterministic):
//   x -> bf16 hi/lo          x = hi + lo with both bf16 (relative error ~2^-16,
//                            inside the 2^-14 parity band; tests/parity_util.py)
//   T  = Bp x                gathered-row GEMM, split-K, fixed-order reduction
//   pre = A T + bias         same GEMM over all D rows; epilogue: mask bits per
//                            neuron (one bit per token), union flag, per-token |P|
//   U_P                      ascending compaction of the union (one CTA scan)
//   G = gate[U_P] x          epilogue: survivor bits = mask & (G > 0), union, |V|
//   U_V                      ascending compaction
//   U = up[U_V] x            epilogue: z = gated(G, U) on survivor bits, else +0
//   Y = sum_{U_V} down z     split-K over U_V, fixed-order reduction
//
// GEMM tiles: 4 warps, 64 rows x Bp (<= 64) tokens, K chunks of 64 through a
// 2-stage cp.async pipeline; fragments by ldmatrix; mma.sync.m16n8k16 bf16 with
// fp32 accumulation (hi and lo parts are two MMAs into the same accumulator).
#include "sg_internal.h"

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <type_traits>

namespace sg {
namespace {

// Programmatic dependent launch (opt-in, see pdl_enabled): every kernel of the
// batched path can be launched with programmatic stream serialization, so the
// next kernel's CTAs are set up while this one drains. Each kernel first waits for its predecessor grid to
// complete (griddepcontrol.wait, unconditionally and before any memory access:
// the ordering is exactly that of plain stream order, transitively), then
// allows its own dependents to launch.
#define SG_PDL_ENTRY()                                          \
    do {                                                        \
        asm volatile("griddepcontrol.wait;" ::: "memory");      \
        asm volatile("griddepcontrol.launch_dependents;" :::);  \
    } while (0)


constexpr int kBM = 64;                  // rows per CTA tile
constexpr int kBK = 32;                  // K per pipeline stage
constexpr int kCh = kBK / 8;             // 16-B chunks per row per stage
constexpr int kTickets = 16;  // ints at BatchArgs::ticket: [0] gate_epi, [1 + tile] t_kernel
constexpr int kBWarps = 4;               // one m16 slice per warp
constexpr int kBThreads = kBWarps * 32;
constexpr int kRowPad = kBK + 8;         // smem row stride (bf16): conflict-free ldmatrix
constexpr int kMaxBatch = 64;

__device__ __forceinline__ uint32_t smem_u32b(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp16(void* dst, const void* src, bool ok) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32b(dst)), "l"(src),
                 "r"(ok ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void ldsm_x4(const void* p, uint32_t& a, uint32_t& b, uint32_t& c,
                                        uint32_t& d) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                 : "r"(smem_u32b(p)));
}
__device__ __forceinline__ void ldsm_x4_t(const void* p, uint32_t& a, uint32_t& b, uint32_t& c,
                                          uint32_t& d) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                 : "r"(smem_u32b(p)));
}
__device__ __forceinline__ void ldsm_x2(const void* p, uint32_t& a, uint32_t& b) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0, %1}, [%2];"
                 : "=r"(a), "=r"(b)
                 : "r"(smem_u32b(p)));
}
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
        "{%8, %9}, {%0, %1, %2, %3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// ---------------------------------------------------------------------------
// Gathered-row GEMM: acc[r][n] = sum_k W[row(r)][k] * (Xh[n][k] + Xl[n][k]),
// r over this CTA's 64 rows, n < nb (a multiple of 8), k over [k0, k1).
// W rows: row(r) = rows ? rows[r] : r, pitch wp elements; X: [nb][xp] bf16.
// TRANS_A: W is stored [k][m] (m contiguous, pitch wp) — the down projection,
// where "rows" index K (neurons) and the 64-wide tile runs over m.
// ---------------------------------------------------------------------------
constexpr int kStages = 6;  // cp.async pipeline depth (K chunks in flight), default

__host__ __device__ constexpr int a_elems(bool trans) { return trans ? kBK * (kBM + 8) : kBM * kRowPad; }
__host__ __device__ inline int stage_elems(bool trans, int nb) { return a_elems(trans) + 2 * nb * kRowPad; }

template <bool TRANS_A, int kStages>
__device__ __forceinline__ void gemm_tile_s(const uint16_t* __restrict__ W, int wp,
                                          const int* __restrict__ rows, int nrows, int m0,
                                          const uint16_t* __restrict__ Xh,
                                          const uint16_t* __restrict__ Xl, int xp, int nb, int k0,
                                          int k1, uint16_t* sm, float (*acc)[4]) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ntile = nb >> 3;
    constexpr int kA = a_elems(TRANS_A);
    const int se = stage_elems(TRANS_A, nb);
    const int nk = k1 > k0 ? (k1 - k0 + kBK - 1) / kBK : 0;
    auto load = [&](int st, int kb) {
        uint16_t* a = sm + st * se;
        uint16_t* xh = a + kA;
        uint16_t* xl = xh + nb * kRowPad;
        if (!TRANS_A) {
            for (int i = tid; i < kBM * kCh; i += kBThreads) {
                const int r = i / kCh, p = i % kCh;
                const int gr = m0 + r;
                const bool ok = gr < nrows;
                const int row = ok ? (rows ? rows[gr] : gr) : 0;
                cp16(a + r * kRowPad + p * 8, W + static_cast<size_t>(row) * wp + kb + p * 8, ok);
            }
        } else {
            // 64 k (neurons) x 64 m: row k is the m-slice [m0, m0+64) of neuron rows[k]
            for (int i = tid; i < kBK * 8; i += kBThreads) {
                const int r = i >> 3, p = i & 7;
                const int gk = kb + r;
                const bool ok = gk < k1;
                const int row = ok ? rows[gk] : 0;
                cp16(a + r * (kBM + 8) + p * 8, W + static_cast<size_t>(row) * wp + m0 + p * 8, ok);
            }
        }
        for (int i = tid; i < nb * kCh; i += kBThreads) {
            const int n = i / kCh, p = i % kCh;
            cp16(xh + n * kRowPad + p * 8, Xh + static_cast<size_t>(n) * xp + kb + p * 8, true);
            cp16(xl + n * kRowPad + p * 8, Xl + static_cast<size_t>(n) * xp + kb + p * 8, true);
        }
    };
#pragma unroll
    for (int t = 0; t < kMaxBatch / 8; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[t][e] = 0.f;
    // prologue: chunks 0 .. kStages-2 in flight (one commit group each, empty ones too)
    for (int s = 0; s < kStages - 1; ++s) {
        if (s < nk) load(s, k0 + s * kBK);
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int it = 0; it < nk; ++it) {
        asm volatile("cp.async.wait_group %0;" ::"n"(kStages - 2) : "memory");
        __syncthreads();  // chunk `it` visible to all; stage (it-1) % S free to refill
        {
            const int nx = it + kStages - 1;
            if (nx < nk) load(nx % kStages, k0 + nx * kBK);
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        const uint16_t* a = sm + (it % kStages) * se;
        const uint16_t* xh = a + kA;
        const uint16_t* xl = xh + nb * kRowPad;
#pragma unroll
        for (int ks = 0; ks < kBK; ks += 16) {
            uint32_t af[4];
            if (!TRANS_A) {
                const int r = warp * 16 + (lane & 15);
                const int kk = ks + (lane >> 4) * 8;
                ldsm_x4(a + r * kRowPad + kk, af[0], af[1], af[2], af[3]);
            } else {
                // matrices: (m 0-7, k 0-7), (m 8-15, k 0-7), (m 0-7, k 8-15), (m 8-15, k 8-15)
                const int q = lane >> 3, rr = lane & 7;
                const int kk = ks + (q >> 1) * 8 + rr;
                const int mm = warp * 16 + (q & 1) * 8;
                ldsm_x4_t(a + kk * (kBM + 8) + mm, af[0], af[1], af[2], af[3]);
            }
#pragma unroll
            for (int t = 0; t < kMaxBatch / 8; ++t) {
                if (t < ntile) {
                    const int n = t * 8 + (lane & 7);
                    const int kk = ks + ((lane >> 3) & 1) * 8;
                    uint32_t b0, b1;
                    ldsm_x2(xh + n * kRowPad + kk, b0, b1);
                    mma16816(acc[t], af, b0, b1);
                    ldsm_x2(xl + n * kRowPad + kk, b0, b1);
                    mma16816(acc[t], af, b0, b1);
                }
            }
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
}

// pipeline depth chosen per call (BatchArgs::stages): fewer stages at large B
// so more CTAs fit per SM
template <bool TRANS_A>
__device__ __forceinline__ void gemm_tile(int stages, const uint16_t* __restrict__ W, int wp,
                                          const int* __restrict__ rows, int nrows, int m0,
                                          const uint16_t* __restrict__ Xh,
                                          const uint16_t* __restrict__ Xl, int xp, int nb, int k0,
                                          int k1, uint16_t* sm, float (*acc)[4]) {
    if (stages == 2)
        gemm_tile_s<TRANS_A, 2>(W, wp, rows, nrows, m0, Xh, Xl, xp, nb, k0, k1, sm, acc);
    else if (stages == 3)
        gemm_tile_s<TRANS_A, 3>(W, wp, rows, nrows, m0, Xh, Xl, xp, nb, k0, k1, sm, acc);
    else if (stages == 4)
        gemm_tile_s<TRANS_A, 4>(W, wp, rows, nrows, m0, Xh, Xl, xp, nb, k0, k1, sm, acc);
    else
        gemm_tile_s<TRANS_A, kStages>(W, wp, rows, nrows, m0, Xh, Xl, xp, nb, k0, k1, sm, acc);
}

// acc -> out[(split * cap + row) * 64 + n] for the CTA's rows (fp32 partial sums)
__device__ __forceinline__ void store_partial(float (*acc)[4], float* out, int cap, int split, int m0,
                                              int nrows, int nb) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int t = 0; t < kMaxBatch / 8; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            if (t >= nb / 8) continue;
            const int row = m0 + warp * 16 + (lane >> 2) + (e >> 1) * 8;
            const int n = t * 8 + (lane & 3) * 2 + (e & 1);
            if (row < nrows) out[(static_cast<size_t>(split) * cap + row) * kMaxBatch + n] = acc[t][e];
        }
}

// Per-token counts of the set bits of this warp's rows (each lane may carry up to
// two rows' masks; duplicates across a lane group must be zero) -> one atomicAdd
// per token per warp (integer: order-free).
__device__ __forceinline__ void count_tokens(uint64_t m0, uint64_t m1, int B, int* counts) {
    const int lane = threadIdx.x & 31;
    for (int n = 0; n < B; ++n) {
        const unsigned c = __popc(__ballot_sync(0xffffffffu, (m0 >> n) & 1ull)) +
                           __popc(__ballot_sync(0xffffffffu, (m1 >> n) & 1ull));
        if (lane == 0 && c) atomicAdd(counts + n, static_cast<int>(c));
    }
}

// x (fp32 [B][d]) -> bf16 hi/lo [nb][pitch] (zero padded rows and columns)
// Also clears the call's counters and survivor flags / bits (in place of
// memsets, which would break the programmatic-launch chain).
__global__ void split_x_kernel(const float* __restrict__ x, int B, int d, int nb, int pitch,
                               uint16_t* __restrict__ hi, uint16_t* __restrict__ lo, BatchArgs a) {
    SG_PDL_ENTRY();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < kMaxBatch) {
        a.pcount[i] = 0;
        a.vcount[i] = 0;
    }
    if (i < a.D) {
        a.vflag[i] = 0;
        a.vbits[i] = 0ull;
    }
    if (i >= nb * pitch) return;
    const int n = i / pitch, k = i - n * pitch;
    const float v = (n < B && k < d) ? x[static_cast<size_t>(n) * d + k] : 0.f;
    if (!isfinite(v)) atomicOr(a.bad, 1);  // check_input, ffn_exec.hpp:61-63
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    const __nv_bfloat16 l = __float2bfloat16_rn(v - __bfloat162float(h));
    hi[i] = __bfloat16_as_ushort(h);
    lo[i] = __bfloat16_as_ushort(l);
}

// T partials: tp[split][j][n] over K slice `split`
// fuse != 0: the last of the tsplit blocks of a row tile sums its splits in
// order into T hi/lo (what t_reduce_kernel does, one kernel boundary less)
__global__ void __launch_bounds__(kBThreads) t_kernel(BatchArgs a, int fuse) {
    SG_PDL_ENTRY();
    extern __shared__ __align__(128) uint16_t smb[];
    float acc[kMaxBatch / 8][4];
    const int kslice = ((a.pitch_d + a.tsplit - 1) / a.tsplit + kBK - 1) / kBK * kBK;
    const int k0 = min(a.pitch_d, blockIdx.y * kslice), k1 = min(a.pitch_d, k0 + kslice);
    gemm_tile<false>(a.stages, a.Bm, a.pitch_d, nullptr, a.r, blockIdx.x * kBM, a.xh, a.xl, a.pitch_d, a.nb, k0,
                     k1, smb, acc);
    store_partial(acc, a.tp, a.pitch_r, blockIdx.y, blockIdx.x * kBM, a.r, a.nb);
    if (!fuse) return;
    __shared__ int last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(a.ticket + 1 + blockIdx.x, 1) == static_cast<int>(gridDim.y) - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    const int m0 = blockIdx.x * kBM;
    for (int o = threadIdx.x; o < kBM * a.nb; o += blockDim.x) {
        const int n = o / kBM, j = m0 + o % kBM;
        float s = 0.f;  // padding columns (r <= j < pitch_r = tiles * kBM) get +0
        if (j < a.r)
            for (int sp = 0; sp < a.tsplit; ++sp)
            s += __ldcg(a.tp + (static_cast<size_t>(sp) * a.pitch_r + j) * kMaxBatch + n);
        const __nv_bfloat16 h = __float2bfloat16_rn(s);
        const __nv_bfloat16 l = __float2bfloat16_rn(s - __bfloat162float(h));
        a.th[static_cast<size_t>(n) * a.pitch_r + j] = __bfloat16_as_ushort(h);
        a.tl[static_cast<size_t>(n) * a.pitch_r + j] = __bfloat16_as_ushort(l);
    }
    if (threadIdx.x == 0) a.ticket[1 + blockIdx.x] = 0;
}

// T = sum of the splits in order -> bf16 hi/lo [nb][pitch_r]
__global__ void t_reduce_kernel(BatchArgs a) {
    SG_PDL_ENTRY();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.nb * a.pitch_r) return;
    const int n = i / a.pitch_r, j = i - n * a.pitch_r;
    float s = 0.f;
    if (j < a.r)
        for (int sp = 0; sp < a.tsplit; ++sp)
            s += a.tp[(static_cast<size_t>(sp) * a.pitch_r + j) * kMaxBatch + n];
    const __nv_bfloat16 h = __float2bfloat16_rn(s);
    const __nv_bfloat16 l = __float2bfloat16_rn(s - __bfloat162float(h));
    a.th[i] = __bfloat16_as_ushort(h);
    a.tl[i] = __bfloat16_as_ushort(l);
}

// pre = A T + bias over all D rows: mask bits, union flags, per-token |P|
__global__ void __launch_bounds__(kBThreads) mask_kernel(BatchArgs a) {
    SG_PDL_ENTRY();
    extern __shared__ __align__(128) uint16_t smb[];
    __shared__ int scnt[kMaxBatch];  // per-token |P| of this block's rows
    for (int i = threadIdx.x; i < kMaxBatch; i += blockDim.x) scnt[i] = 0;
    __syncthreads();
    float acc[kMaxBatch / 8][4];
    gemm_tile<false>(a.stages, a.A, a.pitch_r, nullptr, a.D, blockIdx.x * kBM, a.th, a.tl, a.pitch_r, a.nb, 0,
                     a.pitch_r, smb, acc);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t bits[2] = {0ull, 0ull};
    const int rb = blockIdx.x * kBM + warp * 16 + (lane >> 2);
#pragma unroll
    for (int t = 0; t < kMaxBatch / 8; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            if (t >= a.nb / 8) continue;
            const int h = e >> 1, row = rb + h * 8;
            const int n = t * 8 + (lane & 3) * 2 + (e & 1);
            if (row < a.D && n < a.B && acc[t][e] + a.bias[row] > 0.f)  // strict, ffn_exec.hpp:141
                bits[h] |= 1ull << n;
        }
    for (int h = 0; h < 2; ++h) {
        bits[h] |= __shfl_xor_sync(0xffffffffu, bits[h], 1);
        bits[h] |= __shfl_xor_sync(0xffffffffu, bits[h], 2);
        const int row = rb + h * 8;
        if ((lane & 3) == 0 && row < a.D) {
            a.mbits[row] = bits[h];
            a.uflag[row] = bits[h] != 0ull;
        }
        if ((lane & 3) != 0 || row >= a.D) bits[h] = 0ull;  // count each row once
    }
    count_tokens(bits[0], bits[1], a.B, scnt);
    __syncthreads();
    for (int n = threadIdx.x; n < a.B; n += blockDim.x)
        if (scnt[n] != 0) atomicAdd(a.pcount + n, scnt[n]);
}

// ascending compaction of flags[0..D), D <= 16384, into list, count into *count
// (one CTA): element j*1024 + t is read by thread t (coalesced), each warp
// ballots it, one block-wide scan over the (j, warp) counts gives every warp's
// output offset for every j, the flags stay in the ballot masks.
constexpr int kCompactPer = 16;
// one 1024-thread block; flags read through L2 (written by other blocks of the
// calling kernel when fused into gate_epi)
__device__ __forceinline__ void compact_ballot_block(const int* __restrict__ flag, int D,
                                                     int* __restrict__ list, int* __restrict__ count) {
    __shared__ int woff[kCompactPer * 32];
    __shared__ int wsum[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per = (D + 1023) / 1024;
    uint32_t m[kCompactPer];
    int f[kCompactPer];  // all flag loads in flight before the first ballot
#pragma unroll
    for (int j = 0; j < kCompactPer; ++j) {
        const int i = j * 1024 + tid;
        f[j] = j < per && i < D ? __ldcg(flag + i) : 0;
    }
#pragma unroll
    for (int j = 0; j < kCompactPer; ++j) {
        m[j] = 0u;
        if (j < per) {
            m[j] = __ballot_sync(0xffffffffu, f[j] != 0);
            if (lane == 0) woff[j * 32 + warp] = __popc(m[j]);
        }
    }
    __syncthreads();
    const int v = tid < per * 32 ? woff[tid & (kCompactPer * 32 - 1)] : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const int w = wsum[lane];
        int wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += u;
        }
        wsum[lane] = wi - w;  // exclusive
        if (lane == 31) *count = wi;
    }
    __syncthreads();
    if (tid < per * 32) woff[tid] = wsum[warp] + incl - v;
    __syncthreads();
    const uint32_t below = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < kCompactPer; ++j)
        if (j < per && ((m[j] >> lane) & 1u)) list[woff[j * 32 + warp] + __popc(m[j] & below)] = j * 1024 + tid;
}
__global__ void __launch_bounds__(1024) compact_ballot_kernel(const int* __restrict__ flag, int D,
                                                              int* __restrict__ list,
                                                              int* __restrict__ count) {
    SG_PDL_ENTRY();
    compact_ballot_block(flag, D, list, count);
}

// ascending compaction of flags[0..D) into list, count into *count (one CTA):
// thread t scans a contiguous run, one block-wide exclusive scan, then writes.
__global__ void __launch_bounds__(1024) compact_kernel(const int* __restrict__ flag, int D,
                                                       int* __restrict__ list, int* __restrict__ count) {
    SG_PDL_ENTRY();
    __shared__ int wsum[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per = (D + 1023) / 1024;
    const int i0 = tid * per, i1 = min(D, i0 + per);
    int c = 0;
    for (int i = i0; i < i1; ++i) c += flag[i] != 0;
    int incl = c;
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, m);
        if (lane >= m) incl += o;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int w = wsum[lane], wi = w;
#pragma unroll
        for (int m = 1; m < 32; m <<= 1) {
            const int o = __shfl_up_sync(0xffffffffu, wi, m);
            if (lane >= m) wi += o;
        }
        wsum[lane] = wi - w;  // exclusive
        if (lane == 31) *count = wi;
    }
    __syncthreads();
    int pos = wsum[warp] + incl - c;
    for (int i = i0; i < i1; ++i)
        if (flag[i]) list[pos++] = i;
}

// gate[U_P] x, split-K partials: gp[split][pos][n]
__global__ void __launch_bounds__(kBThreads) gate_kernel(BatchArgs a) {
    SG_PDL_ENTRY();
    extern __shared__ __align__(128) uint16_t smb[];
    const int np = *a.np;
    if (blockIdx.x * kBM >= np) return;
    const int kslice = ((a.pitch_d + a.gsplit - 1) / a.gsplit + kBK - 1) / kBK * kBK;
    const int k0 = min(a.pitch_d, blockIdx.y * kslice), k1 = min(a.pitch_d, k0 + kslice);
    float acc[kMaxBatch / 8][4];
    gemm_tile<false>(a.stages, a.gate, a.pitch_d, a.plist, np, blockIdx.x * kBM, a.xh, a.xl, a.pitch_d, a.nb, k0,
                     k1, smb, acc);
    store_partial(acc, a.gp, a.pitch_v, blockIdx.y, blockIdx.x * kBM, np, a.nb);
}

// g = sum of the splits in order; survivor bits = mask & (g > 0) (ffn_exec.hpp:200),
// union flags, per-token |V|; G stored per neuron. One warp per neuron: lane n, n+32.
__device__ __forceinline__ void gate_epi_neuron(const BatchArgs& a, int pos, int lane, int* scnt) {
    const int nid = a.plist[pos];
    const uint64_t mb = a.mbits[nid];
    uint64_t bits = 0ull;
    // all split partials in flight first, then summed in split order
    float pg[2][kGpSplits];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int sp = 0; sp < kGpSplits; ++sp) {
            const int n = lane + 32 * h;
            pg[h][sp] = n < a.nb && sp < a.gsplit
                            ? a.gp[(static_cast<size_t>(sp) * a.pitch_v + pos) * kMaxBatch + n]
                            : 0.f;
        }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int n = lane + 32 * h;
        if (n >= a.nb) continue;
        float g = 0.f;
#pragma unroll
        for (int sp = 0; sp < kGpSplits; ++sp)
            if (sp < a.gsplit) g += pg[h][sp];
        a.G[static_cast<size_t>(nid) * kMaxBatch + n] = g;
        if (n < a.B && ((mb >> n) & 1ull) && g > 0.f) bits |= 1ull << n;
    }
    bits = static_cast<uint64_t>(__reduce_or_sync(0xffffffffu, static_cast<unsigned>(bits))) |
           (static_cast<uint64_t>(__reduce_or_sync(0xffffffffu, static_cast<unsigned>(bits >> 32))) << 32);
    if (lane == 0) {
        a.vbits[nid] = bits;
        a.vflag[nid] = bits != 0ull;
    }
    // per-token |V|: counted in the block's shared counters (integer, order-free);
    // one global atomic per token per block (same-address global atomics from
    // every warp left the kernel drain-stalled: 24 us at B = 64)
    if (lane < a.B && ((bits >> lane) & 1ull)) atomicAdd(scnt + lane, 1);
    if (lane + 32 < a.B && ((bits >> (lane + 32)) & 1ull)) atomicAdd(scnt + lane + 32, 1);
}

// 1024-thread blocks, one predicted neuron per warp. fuse != 0: the last block to finish compacts the
// survivor union (one kernel boundary less than a separate compaction launch)
__global__ void __launch_bounds__(1024) gate_epi_kernel(BatchArgs a, int fuse) {
    SG_PDL_ENTRY();
    const int np = *a.np;
    const int pos = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    __shared__ int scnt[kMaxBatch];
    if (threadIdx.x < kMaxBatch) scnt[threadIdx.x] = 0;
    __syncthreads();
    if (pos < np) gate_epi_neuron(a, pos, lane, scnt);
    __syncthreads();
    if (threadIdx.x < a.B && scnt[threadIdx.x] != 0) atomicAdd(a.vcount + threadIdx.x, scnt[threadIdx.x]);
    if (!fuse) return;
    __shared__ int last;
    __threadfence();  // this block's vflag writes before its ticket
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(a.ticket, 1) == static_cast<int>(gridDim.x) - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    compact_ballot_block(a.vflag, a.D, a.vlist, a.nv);
    if (threadIdx.x == 0) *a.ticket = 0;
}

// up[U_V] x, split-K partials: gp[split][pos][n] (the gate partials are consumed)
__global__ void __launch_bounds__(kBThreads) up_kernel(BatchArgs a) {
    SG_PDL_ENTRY();
    extern __shared__ __align__(128) uint16_t smb[];
    const int nv = *a.nv;
    if (blockIdx.x * kBM >= nv) return;
    const int kslice = ((a.pitch_d + a.gsplit - 1) / a.gsplit + kBK - 1) / kBK * kBK;
    const int k0 = min(a.pitch_d, blockIdx.y * kslice), k1 = min(a.pitch_d, k0 + kslice);
    float acc[kMaxBatch / 8][4];
    gemm_tile<false>(a.stages, a.ud, 2 * a.pitch_d, a.vlist, nv, blockIdx.x * kBM, a.xh, a.xl, a.pitch_d, a.nb, k0,
                     k1, smb, acc);
    store_partial(acc, a.gp, a.pitch_v, blockIdx.y, blockIdx.x * kBM, nv, a.nb);
}

// u = sum of the splits; z = gated(g, u) on survivor bits (ffn_exec.hpp:202-203,
// :68-76), else +0 -> Z per (neuron, token) and Z hi/lo [n][pos] for the down GEMM
// (split_z = 0: the row-streamed down projection reads Z only; no hi/lo copy)
__global__ void up_epi_kernel(BatchArgs a, int split_z) {
    SG_PDL_ENTRY();
    const int nv = *a.nv;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int pos = i / a.nb, n = i - pos * a.nb;
    if (pos >= nv) return;
    const int nid = a.vlist[pos];
    float z = 0.f;
    if (n < a.B && ((a.vbits[nid] >> n) & 1ull)) {
        float pu[kGpSplits];  // all split partials in flight first, summed in split order
#pragma unroll
        for (int sp = 0; sp < kGpSplits; ++sp)
            pu[sp] = sp < a.gsplit ? a.gp[(static_cast<size_t>(sp) * a.pitch_v + pos) * kMaxBatch + n] : 0.f;
        const float g = a.G[static_cast<size_t>(nid) * kMaxBatch + n];
        float u = 0.f;
#pragma unroll
        for (int sp = 0; sp < kGpSplits; ++sp)
            if (sp < a.gsplit) u += pu[sp];
        z = (g > 0.f && (a.act == 0 || u > 0.f)) ? g * u : 0.f;
    }
    a.Z[static_cast<size_t>(nid) * kMaxBatch + n] = z;
    if (!split_z) return;
    const __nv_bfloat16 h = __float2bfloat16_rn(z);
    const __nv_bfloat16 l = __float2bfloat16_rn(z - __bfloat162float(h));
    a.zh[static_cast<size_t>(n) * a.pitch_v + pos] = __bfloat16_as_ushort(h);
    a.zl[static_cast<size_t>(n) * a.pitch_v + pos] = __bfloat16_as_ushort(l);
}

// zero the Z hi/lo columns [nv, round_up(nv, 64)) so the last K chunk adds +0
__global__ void zpad_kernel(BatchArgs a) {
    SG_PDL_ENTRY();
    const int nv = *a.nv;
    const int padto = (nv + kBK - 1) / kBK * kBK;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int w = padto - nv;
    if (i >= w * a.nb) return;
    const int n = i / w, pos = nv + (i - n * w);
    a.zh[static_cast<size_t>(n) * a.pitch_v + pos] = 0;
    a.zl[static_cast<size_t>(n) * a.pitch_v + pos] = 0;
}

// Y partials: Yp[split][n][m] = sum over survivor positions of split of down[.][m] z
__global__ void __launch_bounds__(kBThreads) down_kernel(BatchArgs a) {
    SG_PDL_ENTRY();
    extern __shared__ __align__(128) uint16_t smb[];
    const int nv = *a.nv;
    const int chunks = (nv + kBK - 1) / kBK;
    const int per = (chunks + a.dsplit - 1) / a.dsplit;
    const int k0 = blockIdx.y * per * kBK, k1 = min(nv, k0 + per * kBK);
    float acc[kMaxBatch / 8][4];
    // down rows of neuron k live in ud at k * 2 pitch_d + pitch_d
    gemm_tile<true>(a.stages, a.ud + a.pitch_d, 2 * a.pitch_d, a.vlist, nv, blockIdx.x * kBM, a.zh, a.zl,
                    a.pitch_v, a.nb, k0, k1 > k0 ? k1 : k0, smb, acc);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int t = 0; t < kMaxBatch / 8; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            if (t >= a.nb / 8) continue;
            const int m = blockIdx.x * kBM + warp * 16 + (lane >> 2) + (e >> 1) * 8;
            const int n = t * 8 + (lane & 3) * 2 + (e & 1);
            if (m < a.pitch_d)
                a.yp[(static_cast<size_t>(blockIdx.y) * kMaxBatch + n) * a.pitch_d + m] = acc[t][e];
        }
}

__global__ void y_reduce_kernel(BatchArgs a, float* __restrict__ y) {
    SG_PDL_ENTRY();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.B * a.d) return;
    const int n = i / a.d, m = i - n * a.d;
    float s = 0.f;
    for (int sp = 0; sp < a.dsplit; ++sp) s += a.yp[(static_cast<size_t>(sp) * kMaxBatch + n) * a.pitch_d + m];
    y[i] = s;
}

// Down projection for small batches (nb <= 16) on the CUDA cores, streaming
// whole row pieces: CTA (rg, cg) takes the survivor-union positions of row
// group rg and the 1024 columns of column group cg (2 KB contiguous per row;
// the GEMM tile reads 128 B per row at a 16 KB stride). Thread = (row lane rl,
// column thread ct): CP columns x TB tokens of fp32 accumulators over the rows
// rl, rl + RL, ... of its group in order; the RL lanes are summed in order
// through shared memory, then the row groups in order by y_rows_reduce.
// Rows arrive through a kDrStages-deep cp.async ring: each thread copies (and
// later reads) its own CP columns of each row; the rows' z values are copied by
// the first TB / 4 threads of each row lane (one __syncthreads per step).
// Deterministic; bits differ from the tensor-core path (tolerance-checked).
constexpr int kDrCols = 1024;  // columns per column group
constexpr int kDrStages = 4;   // ring depth (steps of U rows per row lane)
constexpr int kDrU = 4;        // rows per row lane per step
constexpr int kDrIdx = 1024;   // row ids staged in smem per CTA
template <int TB>
constexpr int down_rows_smem() {
    constexpr int CP = 64 / TB, RL = 512 / (kDrCols / CP);
    constexpr int ring = kDrStages * kDrU * 512 * CP * 2 + kDrStages * kDrU * RL * TB * 4;
    constexpr int red = 512 * TB * CP * 4;
    return ring > red ? ring : red;
}
template <int TB>
__global__ void __launch_bounds__(512) down_rows_kernel(BatchArgs a, int ncg, int nrg) {
    SG_PDL_ENTRY();
    constexpr int CP = 64 / TB;            // columns per thread
    constexpr int T = kDrCols / CP;        // threads per row piece
    constexpr int RL = 512 / T;            // row lanes
    constexpr int U = kDrU;
    constexpr int NS = kDrStages;
    using WV = typename std::conditional<CP == 8, uint4, uint2>::type;
    extern __shared__ __align__(16) float red[];  // [RL][T][TB*CP] after the loop
    WV* wring = reinterpret_cast<WV*>(red);                              // [NS][U][512]
    float* zring = reinterpret_cast<float*>(wring + NS * U * 512);       // [NS][U][RL][TB]
    const int nv = *a.nv;
    const int cg = blockIdx.x % ncg, rg = blockIdx.x / ncg;
    const int tid = threadIdx.x, rl = tid / T, ct = tid % T;
    const int col = cg * kDrCols + ct * CP;
    const int p0 = static_cast<int>(static_cast<long long>(rg) * nv / nrg);
    const int p1 = static_cast<int>(static_cast<long long>(rg + 1) * nv / nrg);
    const int nsteps = (p1 - p0 + U * RL - 1) / (U * RL);
    // the group's neuron ids, staged once (the copies then issue without a
    // dependent global load each)
    __shared__ int sidx[kDrIdx];
    for (int i = tid; i < p1 - p0 && i < kDrIdx; i += 512) sidx[i] = __ldg(a.vlist + p0 + i);
    __syncthreads();
    float acc[TB][CP];
#pragma unroll
    for (int b = 0; b < TB; ++b)
#pragma unroll
        for (int e = 0; e < CP; ++e) acc[b][e] = 0.f;
    const bool okc = col < a.pitch_d;
    const uint16_t* base = a.ud + a.pitch_d + col;
    auto issue = [&](int k, int stg) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int pos = p0 + rl + (k * U + u) * RL;
            const bool ok = pos < p1;
            const int nid = !ok ? 0 : pos - p0 < kDrIdx ? sidx[pos - p0] : __ldg(a.vlist + pos);
            const uint16_t* src = base + static_cast<size_t>(nid) * 2 * a.pitch_d;
            const uint32_t dst = smem_u32b(wring + (stg * U + u) * 512 + tid);
            if (CP == 8)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
                             "r"(ok && okc ? 16 : 0)
                             : "memory");
            else
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src),
                             "r"(ok && okc ? 8 : 0)
                             : "memory");
            if (ct < TB / 4)
                cp16(zring + ((stg * U + u) * RL + rl) * TB + ct * 4,
                     a.Z + static_cast<size_t>(nid) * kMaxBatch + ct * 4, ok);
        }
    };
#pragma unroll
    for (int k = 0; k < NS - 1; ++k) {
        if (k < nsteps) issue(k, k);
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int k = 0; k < nsteps; ++k) {
        asm volatile("cp.async.wait_group %0;" ::"n"(NS - 2) : "memory");
        __syncthreads();  // step k's z visible; the stage read at step k - 1 is free
        {
            const int kn = k + NS - 1;
            if (kn < nsteps) issue(kn, kn % NS);
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        const int stg = k % NS;
        // rows in position order (u ascending): the accumulation order per thread
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const WV wv = wring[(stg * U + u) * 512 + tid];
            uint32_t w[CP / 2];
            if constexpr (CP == 8) {
                w[0] = wv.x; w[1] = wv.y; w[2] = wv.z; w[3] = wv.w;
            } else {
                w[0] = wv.x; w[1] = wv.y;
            }
            const float4* zr = reinterpret_cast<const float4*>(zring + ((stg * U + u) * RL + rl) * TB);
#pragma unroll
            for (int b4 = 0; b4 < TB / 4; ++b4) {
                const float4 zq = zr[b4];
                const float zz[4] = {zq.x, zq.y, zq.z, zq.w};
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int i = 0; i < CP / 2; ++i) {
                        acc[b4 * 4 + q][2 * i] =
                            fmaf(zz[q], __uint_as_float(w[i] << 16), acc[b4 * 4 + q][2 * i]);
                        acc[b4 * 4 + q][2 * i + 1] =
                            fmaf(zz[q], __uint_as_float(w[i] & 0xffff0000u), acc[b4 * 4 + q][2 * i + 1]);
                    }
            }
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();  // the ring is reused as the reduction area
    float* mine = red + (static_cast<size_t>(rl) * T + ct) * (TB * CP);
#pragma unroll
    for (int b = 0; b < TB; ++b)
#pragma unroll
        for (int e = 0; e < CP; ++e) mine[b * CP + e] = acc[b][e];
    __syncthreads();
    // row lanes summed in order; all threads, one (token, column) output each per pass
    for (int o = tid; o < a.B * kDrCols; o += 512) {
        const int b = o / kDrCols, cc = o - b * kDrCols, c = cg * kDrCols + cc;
        if (c >= a.pitch_d) continue;
        const float* q = red + static_cast<size_t>(cc / CP) * (TB * CP) + b * CP + cc % CP;
        float s = 0.f;
#pragma unroll
        for (int l = 0; l < RL; ++l) s += q[static_cast<size_t>(l) * T * (TB * CP)];
        a.gp[(static_cast<size_t>(rg) * TB + b) * a.pitch_d + c] = s;
    }
}

// Gate / up projections for small batches (nb <= 16) on the CUDA cores:
// gp[cg][pos][n] = sum over the 1024 columns of column group cg of
// W[rows[pos]][c] * x[n][c], x exact fp32 (no hi/lo split). CTA (cg, rg) stages
// its column group of x in smem and its 16 warps stream whole 2-KB row pieces:
// warp step s covers positions p0 + s*R .. +R of row group rg (steps dealt to the
// warps round-robin), lane l takes the 16-B chunks l + 32 i (i < 4) of every row,
// so a warp has 4R 16-B loads per lane in flight. The R x TB lane partials are
// summed by a fixed transposed butterfly (lane j ends with output j); the column
// groups are summed in order by gate_epi / up_epi. Deterministic.
template <int TB>
__global__ void __launch_bounds__(512) rows_dot_kernel(BatchArgs a, const float* __restrict__ xs,
                                                       const uint16_t* __restrict__ W, int wp,
                                                       const int* __restrict__ rows,
                                                       const int* __restrict__ count, int ncg,
                                                       int nrg) {
    SG_PDL_ENTRY();
    constexpr int R = 32 / TB;  // rows per warp step: R x TB = 32 outputs
    extern __shared__ __align__(16) float4 xsm[];  // [TB][2][128]: chunk ch, half h
    const int cg = blockIdx.x % ncg, rg = blockIdx.x / ncg;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int c0 = cg * kDrCols;
    const int n = *count;
    const int p0 = static_cast<int>(static_cast<long long>(rg) * n / nrg);
    const int p1 = static_cast<int>(static_cast<long long>(rg + 1) * n / nrg);
    // the group's row ids, staged once with x (no dependent global load per step)
    __shared__ int sidx[kDrIdx];
    for (int i = tid; i < p1 - p0 && i < kDrIdx; i += 512) sidx[i] = __ldg(rows + p0 + i);
    for (int i = tid; i < TB * 256; i += 512) {
        const int b = i >> 8, q = i & 255, ch = q >> 1, h = q & 1;
        const int c = c0 + ch * 8 + h * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (b < a.B) {
            const float* src = xs + static_cast<size_t>(b) * a.d;
            if (c + 0 < a.d) v.x = src[c + 0];
            if (c + 1 < a.d) v.y = src[c + 1];
            if (c + 2 < a.d) v.z = src[c + 2];
            if (c + 3 < a.d) v.w = src[c + 3];
        }
        xsm[(b * 2 + h) * 128 + ch] = v;
    }
    __syncthreads();
    for (int pos0 = p0 + warp * R; pos0 < p1; pos0 += 16 * R) {
        uint4 w[R][4];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const bool ok = pos0 + r < p1;
            const int rid = !ok ? 0 : pos0 + r - p0 < kDrIdx ? sidx[pos0 + r - p0] : __ldg(rows + pos0 + r);
            const uint16_t* src = W + static_cast<size_t>(rid) * wp + c0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int c = (lane + 32 * i) * 8;
                w[r][i] = ok && c0 + c < a.pitch_d ? __ldg(reinterpret_cast<const uint4*>(src + c))
                                                   : make_uint4(0u, 0u, 0u, 0u);
            }
        }
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int b = 0; b < TB; ++b) {
                const float4 xa = xsm[(b * 2) * 128 + lane + 32 * i];
                const float4 xb = xsm[(b * 2 + 1) * 128 + lane + 32 * i];
                const float xv[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const uint32_t wv[4] = {w[r][i].x, w[r][i].y, w[r][i].z, w[r][i].w};
                    float s = v[r * TB + b];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        s = fmaf(__uint_as_float(wv[e] << 16), xv[2 * e], s);
                        s = fmaf(__uint_as_float(wv[e] & 0xffff0000u), xv[2 * e + 1], s);
                    }
                    v[r * TB + b] = s;
                }
            }
        // transposed butterfly: after the level with offset o, v[j] (j < o) holds
        // index j + (lane & o ? o : 0) summed over the lanes that differ in bit o
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int j = 0; j < o; ++j) {
                const float send = up ? v[j] : v[j + o];
                const float keep = up ? v[j + o] : v[j];
                v[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
        }
        const int r = lane / TB, b = lane % TB, pos = pos0 + r;
        if (pos < p1) a.gp[(static_cast<size_t>(cg) * a.pitch_v + pos) * kMaxBatch + b] = v[0];
    }
}

template <int TB>
__global__ void y_rows_reduce_kernel(BatchArgs a, int nrg, float* __restrict__ y) {
    SG_PDL_ENTRY();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.B * a.d) return;
    const int n = i / a.d, m = i - n * a.d;
    float s = 0.f;
    for (int rg = 0; rg < nrg; ++rg) s += a.gp[(static_cast<size_t>(rg) * TB + n) * a.pitch_d + m];
    y[i] = s;
}

int gemm_smem(bool trans, int nb, int stages) { return stages * stage_elems(trans, nb) * 2; }

// Launch with programmatic stream serialization when SG_PDL=1. Off by default:
// measured on B200 (8-layer 7B stack in a CUDA graph, tokens/s, PDL vs plain):
// B = 5 6587 / 6514, 8 9714 / 9799, 16 12218 / 12318, 32 19942 / 20547,
// 64 35072 / 35131 (tools/pdl_ab.sh). griddepcontrol.wait is a no-op in a
// kernel launched without the attribute.
// SG_BATCH_FUSE bit 0: survivor compaction in gate_epi's last block; bit 1: T
// reduced by t_kernel's last split block. Off by default: the serial last-block
// work costs more than the kernel boundary it saves in a CUDA graph (B200, 7B
// 8-layer stack, tokens/s for fuse 0 / 1 / 2 / 3: B = 5 6532 / 6340 / 6269 / 6100,
// B = 8 9837 / 9564 / 9463 / 9220, B = 16 12300 / 12086 / 11313 / 11137;
// tools/fuse_ab.sh).
int fuse_mask() {
    static const int v = [] {
        const char* e = std::getenv("SG_BATCH_FUSE");
        return e ? std::atoi(e) : 0;
    }();
    return v;
}
bool pdl_enabled() {
    static const bool v = [] {
        const char* e = std::getenv("SG_PDL");
        return e && std::atoi(e) != 0;
    }();
    return v;
}
template <typename... KArgs, typename... Args>
void launch(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

}  // namespace

int batch_max() { return kMaxBatch; }

int launch_batch(const BatchArgs& a0, const float* xs, float* ys, void* stream_) {
    cudaStream_t st = static_cast<cudaStream_t>(stream_);
    BatchArgs a = a0;
    const int sm_rows = gemm_smem(false, a.nb, a.stages), sm_down = gemm_smem(true, a.nb, a.stages);
    {
        const int mx = gemm_smem(false, kMaxBatch, kStages);
        int e = 0;
        for (const void* k : {reinterpret_cast<const void*>(t_kernel), reinterpret_cast<const void*>(mask_kernel),
                              reinterpret_cast<const void*>(gate_kernel), reinterpret_cast<const void*>(up_kernel)})
            if (!e) e = ensure_smem_attr(k, mx);
        if (!e) e = ensure_smem_attr(reinterpret_cast<const void*>(down_kernel), gemm_smem(true, kMaxBatch, kStages));
        if (e) return e;
    }
    {
        int n = a.nb * a.pitch_d;
        if (n < a.D) n = a.D;
        if (n < kMaxBatch) n = kMaxBatch;
        launch(split_x_kernel, (n + 255) / 256, 256, 0, st, xs, a.B, a.d, a.nb, a.pitch_d, a.xh, a.xl, a);
    }
    {
        // small batches: T reduced by the last split block of each row tile
        const int tiles = (a.r + kBM - 1) / kBM;
        const int fuse = (fuse_mask() & 2) && a.nb <= 16 && tiles <= kTickets - 1;
        launch(t_kernel, dim3(tiles, a.tsplit), kBThreads, sm_rows, st, a, fuse);
        if (!fuse) {
            const int n = a.nb * a.pitch_r;
            launch(t_reduce_kernel, (n + 255) / 256, 256, 0, st, a);
        }
    }
    launch(mask_kernel, (a.D + kBM - 1) / kBM, kBThreads, sm_rows, st, a);
    if (a.D <= kCompactPer * 1024)
        launch(compact_ballot_kernel, 1, 1024, 0, st, a.uflag, a.D, a.plist, a.np);
    else
        launch(compact_kernel, 1, 1024, 0, st, a.uflag, a.D, a.plist, a.np);
    // small batches: gate / up row pieces streamed on the CUDA cores (x exact fp32,
    // one partial per column group); larger: the tensor-core GEMM tiles, split-K
    const int ncg = (a.pitch_d + kDrCols - 1) / kDrCols;
    const bool dot_rows = a.nb <= 16 && ncg <= kGpSplits && a.gdot;
    const int dtb = a.nb <= 8 ? 8 : 16;
    const int dgrid = ncg * (a.sms / ncg < 1 ? 1 : a.sms / ncg);
    const int dsm = dtb * 256 * 16;
    if (dot_rows) {
        int e = ensure_smem_attr(reinterpret_cast<const void*>(rows_dot_kernel<8>), 16 * 256 * 16);
        if (!e) e = ensure_smem_attr(reinterpret_cast<const void*>(rows_dot_kernel<16>), 16 * 256 * 16);
        if (e) return e;
        a.gsplit = ncg;
        auto k = dtb == 8 ? rows_dot_kernel<8> : rows_dot_kernel<16>;
        launch(k, dgrid, 512, dsm, st, a, xs, a.gate, a.pitch_d, a.plist, a.np, ncg, dgrid / ncg);
    } else {
        launch(gate_kernel, dim3((a.D + kBM - 1) / kBM, a.gsplit), kBThreads, sm_rows, st, a);
    }
    if (a.D <= kCompactPer * 1024 && (fuse_mask() & 1)) {
        launch(gate_epi_kernel, (a.D + 31) / 32, 1024, 0, st, a, 1);
    } else {
        launch(gate_epi_kernel, (a.D + 31) / 32, 1024, 0, st, a, 0);
        if (a.D <= kCompactPer * 1024)
            launch(compact_ballot_kernel, 1, 1024, 0, st, a.vflag, a.D, a.vlist, a.nv);
        else
            launch(compact_kernel, 1, 1024, 0, st, a.vflag, a.D, a.vlist, a.nv);
    }
    if (dot_rows) {
        auto k = dtb == 8 ? rows_dot_kernel<8> : rows_dot_kernel<16>;
        launch(k, dgrid, 512, dsm, st, a, xs, a.ud, 2 * a.pitch_d, a.vlist, a.nv, ncg, dgrid / ncg);
    } else {
        launch(up_kernel, dim3((a.D + kBM - 1) / kBM, a.gsplit), kBThreads, sm_rows, st, a);
    }
    // small batches: whole-row-piece streaming on the CUDA cores (partials reuse gp,
    // free after up_epi); larger: the tensor-core GEMM over Z hi/lo
    const int tb = a.nb <= 8 ? 8 : 16;
    const size_t cap = static_cast<size_t>(kGpSplits) * a.pitch_v * kMaxBatch;  // floats in gp
    int nrg = a.sms / ncg;
    if (static_cast<size_t>(nrg) * tb * a.pitch_d > cap)
        nrg = static_cast<int>(cap / (static_cast<size_t>(tb) * a.pitch_d));
    const bool rows_path = a.nb <= 16 && nrg >= 8;
    launch(up_epi_kernel, (a.D * a.nb + 255) / 256, 256, 0, st, a, rows_path ? 0 : 1);
    if (rows_path) {
        const int smem = tb == 8 ? down_rows_smem<8>() : down_rows_smem<16>();
        int e = ensure_smem_attr(reinterpret_cast<const void*>(down_rows_kernel<8>), down_rows_smem<8>());
        if (!e) e = ensure_smem_attr(reinterpret_cast<const void*>(down_rows_kernel<16>), down_rows_smem<16>());
        if (e) return e;
        const int n = a.B * a.d;
        if (tb == 8) {
            launch(down_rows_kernel<8>, ncg * nrg, 512, smem, st, a, ncg, nrg);
            launch(y_rows_reduce_kernel<8>, (n + 255) / 256, 256, 0, st, a, nrg, ys);
        } else {
            launch(down_rows_kernel<16>, ncg * nrg, 512, smem, st, a, ncg, nrg);
            launch(y_rows_reduce_kernel<16>, (n + 255) / 256, 256, 0, st, a, nrg, ys);
        }
        return static_cast<int>(cudaGetLastError());
    }
    launch(zpad_kernel, (kBK * kMaxBatch + 255) / 256, 256, 0, st, a);
    launch(down_kernel, dim3((a.pitch_d + kBM - 1) / kBM, a.dsplit), kBThreads, sm_down, st, a);
    {
        const int n = a.B * a.d;
        launch(y_reduce_kernel, (n + 255) / 256, 256, 0, st, a, ys);
    }
    return static_cast<int>(cudaGetLastError());
}

}  // namespace sg
