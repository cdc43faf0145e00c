// sparsegate-b200: batched decode (BASELINE.json configs[4]) on the 5th-generation
// tensor cores — B in [2, 64] tokens through one layer, ONE persistent launch.
//
// Per token the result means exactly what sparse_ffn_sequential
// (/root/reference/proj/include/sparsegate/ffn_exec.hpp:183-218) returns for that
// token alone: its predicted set P_b (pre > 0, :141), survivors V_b (g > 0, :200),
// gated values (:68-76) and y_b over V_b (:80-94). The batch shares the weight
// traffic: every gate row of the union of the P_b and every up / down row of the
// union of the V_b is read ONCE from HBM and multiplied against all B tokens.
//
// Numerics: x (and t, z) enter the tensor cores as bf16 hi + lo pairs (x = hi + lo,
// relative error ~2^-17, inside the 2^-14 parity band of tests/parity_util.py);
// the two halves are the N = 2*nb columns of one MMA (hi tokens, then lo tokens) and
// are summed in the epilogue, fp32 accumulation in TMEM throughout.
//
// Work decomposition (a dataflow of units claimed from one global counter in
// topological order, so a unit only ever waits for units claimed before it — no
// co-residency assumption, no grid barrier):
//   X    split x -> bf16 hi/lo rows of X^T (K-major B operand), zero the counters
//   T    T^T = Bp X^T over a K slice (M = 256 predictor rows, split-K KT)
//   TR   fixed-order sum of the KT partials -> bf16 hi/lo T (B operand of PRE)
//   PRE  neuron block i (256 rows of A): pre = A T + bias > 0 -> per-token mask
//        bits, union list of the block (ascending), |P_b| counts
//   GATE block i, K slice: g = gate[union rows] X (rows by TMA tile::gather4);
//        slice 0 sums the other slices' partials in order, then survivor bits
//        (mask & g > 0), the block's survivor list, |V_b|
//   UP   block i, K slice: u = up[survivor rows] X; slice 0: z = gated(g, u) on
//        the token's survivor bit, else +0 -> bf16 hi/lo Z^T (K-major)
//   DOWN d tile (256 outputs) x block range s: y_s = down^T[rows] Z (the
//        neuron-major down rows gathered as an MN-major A operand)
//   YR   y = fixed-order sum of the S block-range partials
// All reductions have a fixed order, no float atomics: bit-identical on rerun.
//
// CTA: warp 0 = TMA producer (claims units, waits their inputs, gathers rows),
// warp 1 = MMA issuer (tcgen05.mma, one elected lane; TMEM: two accumulator
// buffers of 256 columns), warps 2-5 = epilogue (tcgen05.ld; one TMEM lane
// quarter each) and the non-MMA units. 4 smem stages of 48 KB.
#include "sg_internal.h"

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace sg {
namespace {

// 8 warps = 2 per SM sub-partition, so a thread may hold up to 255 registers (a 9th
// warp would put 3 on one sub-partition and cap them at 168)
constexpr int kProdThreads = 96;   // warps 0-2: producers (cp.async row gathers, TMA tiles)
constexpr int kMmaWarp = 3;         // warp 3: MMA issuer; warps 4-7: epilogue
constexpr int kEpiBase = 128;
constexpr int kTcThreads = 256;
constexpr int kLag = 3;             // stages a producer thread keeps in flight before arriving
constexpr int kStages = 4;
constexpr int kStageA = 32768;  // 256 rows x 64 K bf16 (two M = 128 sub-tiles)
constexpr int kStageB = 16384;  // <= 128 rows (N) x 64 K bf16
constexpr int kStageBytes = kStageA + kStageB;
constexpr int kUQ = 4;          // unit queue depth (producer lead)
constexpr int kBlk = 128;       // neurons per block: one M = 128 tile of gate and of up rows
constexpr int kTRows = 256;     // predictor rows of a T unit (rank <= 256: two M = 128 tiles)

enum UnitType : int { U_STOP = 0, U_X, U_T, U_TR, U_PRE, U_GU, U_DOWN };

struct Unit {
    int type;
    int a, b;    // block / tile index, K slice / block-range index
    int nst;     // smem stages (MMA units)
    int nsub;    // M = 128 sub-tiles carrying rows (1 or 2)
    int cnt;     // rows of the unit (gather units)
    int acc;     // TMEM accumulator buffer
    int pad;     // GU: the block's rows are contiguous (TMA tiles), not gathered
    int u;       // index in the claim order
};

// ---- PTX wrappers -----------------------------------------------------------
__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "TC_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra TC_WAIT_%=;\n}" ::"r"(su32(b)),
        "r"(par)
        : "memory");
}
__device__ __forceinline__ void tma_tile(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            su32(dst)),
        "l"(m), "r"(c0), "r"(c1), "r"(su32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* m, int c0, int r0, int r1,
                                            int r2, int r3, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(su32(dst)),
        "l"(m), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// UMMA shared-memory descriptor, SWIZZLE_128B (sm_100 version 1).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) |
           (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
           (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
// kind::f16 instruction descriptor: bf16 x bf16 -> f32, M = 128.
__device__ __forceinline__ uint32_t idesc(int N, int a_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(a_mn) << 15) |
           (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);
}
__device__ __forceinline__ void umma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
        "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     su32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
// 8 fp32 columns of this warp's TMEM lane quarter (call tmem_wait before use)
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7])
                 : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
__device__ __forceinline__ bool epi_bar_or(int v) {  // epi_bar + OR of v over the epilogue threads
    uint32_t out;
    asm volatile("{\n\t.reg .pred p, q;\n\tsetp.ne.u32 p, %1, 0;\n\tbar.red.or.pred q, 1, 128, p;\n\t"
                 "selp.u32 %0, 1, 0, q;\n}"
                 : "=r"(out)
                 : "r"(v)
                 : "memory");
    return out != 0;
}
__device__ __forceinline__ void prod_bar() { asm volatile("bar.sync 2, %0;" ::"n"(kProdThreads) : "memory"); }
// 16-B global -> shared copy on the LSU path (row gathers: a TMA tile::gather4 moves
// only 512 B per instruction, ~14 GB/s per SM on B200 — tools/bw_tma.cu)
__device__ __forceinline__ void cp16(uint32_t dst, const void* src, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// this thread's copies of the stage have landed: make them visible to the tensor
// cores (async proxy) and count the thread on the stage's full barrier
__device__ __forceinline__ void stage_arrive(uint64_t* bar) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive(bar);
}


__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Acquire a dataflow counter; the proxy fence orders this thread's later TMA reads
// (async proxy) after the generic-proxy writes the counter published.
__device__ __forceinline__ void wait_count(const int* p, int target) {
    while (ld_acquire(p) < target) __nanosleep(64);
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ bool flag_ready(const int* p, int target) { return ld_acquire(p) >= target; }
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// unit trace (diagnostics): [u][0] claim, [1] inputs ready, [2] loads issued,
// [3] epilogue start, [4] epilogue end, [5] SM id
#define TC_TRACE(a, u, k, v)                                                         \
    do {                                                                             \
        if ((a).trace != nullptr && (u) >= 0 && (u) < (a).n_units)                   \
            (a).trace[static_cast<size_t>(u) * 8 + (k)] = (v);                      \
    } while (0)

// Publish this thread's (or, after a CTA-level barrier, the CTA's) global writes —
// generic-proxy stores included, for later TMA reads — then count.
__device__ __forceinline__ void signal(int* p) {
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __threadfence();
    atomicAdd(p, 1);
}

__device__ __forceinline__ void split_bf16(float v, uint16_t& hi, uint16_t& lo) {
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    hi = __bfloat16_as_ushort(h);
    lo = __bfloat16_as_ushort(__float2bfloat16_rn(v - __bfloat162float(h)));
}
// ffn_exec.hpp:68-76 in fp32 (canonical +0 when suppressed)
__device__ __forceinline__ float gated(float g, float u, int act) {
    return (g > 0.f && (act == 0 || u > 0.f)) ? g * u : 0.f;
}

// ---- unit table ---------------------------------------------------------------
// The host lays the units out in one claim order (TcArgs::order, built by
// sg_host.cpp tc_schedule): the predictor chain first, then the GATE units block by
// block (the K slices of a block KS-1 .. 0, the owner that sums the others'
// partials last), with a block's UP units, a block range's DOWN units and a d
// tile's YR units merged in about one wave of claims after the units they depend
// on. Every unit's inputs come from units earlier in the order, so the dataflow
// cannot deadlock, and no phase waits for a whole previous phase.
__device__ __forceinline__ int unit_type(const TcArgs& a, int u, int& i, int& j) {
    if (u >= a.n_units) return U_STOP;
    const int code = __ldg(a.order + u);
    i = (code >> 8) & 0xffff;
    j = code & 0xff;
    return code >> 24;
}
__device__ __forceinline__ int blk_rows(const TcArgs& a, int blk) {
    const int r = a.D - blk * kBlk;
    return r < kBlk ? r : kBlk;
}
__device__ __forceinline__ int range_lo(const TcArgs& a, int s) { return s * a.nblk / a.S; }
// A block whose listed rows are a large enough share of its rows is loaded whole by
// TMA tiles (128 contiguous rows per instruction) instead of gathered row by row:
// gathers stream ~26 GB/s per SM, tiles ~55 (tools/bw_tma.cu), so above ~45 %
// density the tile is faster even though it also reads the unlisted rows. The
// decision is a function of the block's count only, so every unit (and the UP
// epilogue that lays out Z for DOWN) agrees on it.
__device__ __forceinline__ bool blk_tiled(const TcArgs& a, int cnt, int blk, int thr) {
    return a.dense || cnt * 1024 >= thr * blk_rows(a, blk);
}
// vcnt[blk] = survivor rows | kVTiled when DOWN streams the block whole (GU epilogue)
constexpr int kVTiled = 1 << 16;
__device__ __forceinline__ int vcnt_rows(int raw) { return raw & (kVTiled - 1); }
__device__ __forceinline__ bool vcnt_tiled(int raw) { return (raw & kVTiled) != 0; }

// flags layout (ints), zeroed by the last CTA of every launch
__device__ __forceinline__ int* fl_work(const TcArgs& a) { return a.flags; }
__device__ __forceinline__ int* fl_exit(const TcArgs& a) { return a.flags + 1; }
__device__ __forceinline__ int* fl_x(const TcArgs& a) { return a.flags + 2; }
__device__ __forceinline__ int* fl_t(const TcArgs& a) { return a.flags + 3; }
__device__ __forceinline__ int* fl_tr(const TcArgs& a) { return a.flags + 4; }
__device__ __forceinline__ int* fl_pre(const TcArgs& a, int b) { return a.flags + 32 + b; }
__device__ __forceinline__ int* fl_gpart(const TcArgs& a, int b) { return a.flags + 32 + a.nblk + b; }
__device__ __forceinline__ int* fl_gu(const TcArgs& a, int b) { return a.flags + 32 + 2 * a.nblk + b; }
__device__ __forceinline__ int* fl_down(const TcArgs& a, int t) { return a.flags + 32 + 3 * a.nblk + t; }
__device__ __forceinline__ int flag_count(const TcArgs& a) { return 32 + 3 * a.nblk + a.ndt; }
// GU units load without waiting for the block's mask: the dense comparator, and
// batches wide enough that the union of the masks covers most rows anyway
__device__ __forceinline__ bool gu_static(const TcArgs& a) { return a.dense || a.tile_all; }

struct TcSmem {
    uint64_t full[kStages], empty[kStages], tfull[2], tempty[2], uqf[kUQ], uqe[kUQ];
    Unit uq[kUQ];
    uint32_t tmem;
    int rows[kBlk];      // producer: gather rows of the current unit (global neuron index)
    Unit pu;             // producer: the unit being loaded
    int pready;          // producer: its inputs and queue slot are available now
    int flag[kBlk];      // epilogue: per-row flags / positions
    int cnt[64];         // epilogue: per-token counts
    int wsum[16];        // epilogue: per-(sub-tile, quarter) counts
    int last;            // epilogue: this unit was the last of its group (it reduces)
    alignas(16) uint16_t zst[2][8][kBlk];  // epilogue: Z hi / lo of 8 tokens x the block's slots
};

// ---- producer: claim, wait, load ---------------------------------------------
// 96 threads (warps 0-2). Thread 0 is the controller: it claims units, checks and
// waits their inputs and publishes them. Contiguous rows (T, PRE, the dense
// comparator) and the B operands come by TMA tiles from the controller; gathered
// rows (the union / survivor rows of GATE, UP, DOWN) by 16-B cp.async from every
// producer thread, written in the 128-B-swizzled UMMA layout. Each thread keeps kLag
// stages of its copies in flight, then (wait_group, proxy fence) arrives on the
// stage's full barrier (kProdThreads + 1 arrivals: the threads + the controller's expect_tx).
// Before any blocking wait on another unit or on the epilogue every thread flushes
// its pending arrivals, so no stage of an earlier unit is held back.
__device__ __forceinline__ bool unit_inputs_ready(const TcArgs& a, int type, int i, int j) {
    switch (type) {
        case U_T: return flag_ready(fl_x(a), a.u_T);
        case U_PRE: return flag_ready(fl_tr(a), a.u_PRE - a.u_TR);
        case U_GU: return gu_static(a) ? flag_ready(fl_x(a), a.u_T) : flag_ready(fl_pre(a, i), 1);
        case U_DOWN: return flag_ready(fl_gu(a, range_lo(a, j)), 1);  // later blocks: as they stream
        case U_TR: return flag_ready(fl_t(a), a.u_TR - a.u_T);
        default: return true;  // U_X
    }
}
__device__ __forceinline__ void unit_inputs_wait(const TcArgs& a, int type, int i, int j) {
    switch (type) {
        case U_T: wait_count(fl_x(a), a.u_T); break;
        case U_PRE: wait_count(fl_tr(a), a.u_PRE - a.u_TR); break;
        case U_GU:
            if (gu_static(a)) wait_count(fl_x(a), a.u_T);
            else wait_count(fl_pre(a, i), 1);
            break;
        case U_TR: wait_count(fl_t(a), a.u_TR - a.u_T); break;
        case U_DOWN: wait_count(fl_gu(a, range_lo(a, j)), 1); break;
        default: break;
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ void producer(const TcArgs& a, const TcMaps& M, TcSmem& S, uint8_t* stages) {
    const int pt = threadIdx.x;  // 0..127
    const uint64_t pol = policy_evict_first();
    const uint32_t bbytes = static_cast<uint32_t>(a.N) * 128u;
    const uint32_t sbase = su32(stages);
    int seq = 0, accseq = 0;
    int n = 0;         // stages issued by this thread (all producer threads agree)
    int pending = 0;   // of which not yet arrived
    uint32_t ephase = 0;  // bit s: parity of empty[s] to wait for
    auto flush = [&] {
        cp_wait<0>();
        for (; pending > 0; --pending) stage_arrive(&S.full[(n - pending) % kStages]);
    };
    for (;;) {
        // ---- claim the next unit of the order (controller), then everyone sees it
        if (pt == 0) {
            const int u = atomicAdd(fl_work(a), 1);
            int i = 0, j = 0;
            const int type = unit_type(a, u, i, j);
            S.pu = Unit{type, i, j, 0, 0, 0, 0, 0, u};
            TC_TRACE(a, u, 0, gtimer());
            bool ready = unit_inputs_ready(a, type, i, j);
            if (ready && seq >= kUQ) {  // and its queue slot
                uint32_t okw;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                    "selp.u32 %0, 1, 0, p;\n}"
                    : "=r"(okw)
                    : "r"(su32(&S.uqe[seq % kUQ])), "r"(((seq / kUQ) - 1) & 1)
                    : "memory");
                ready = okw != 0;
            }
            S.pready = ready && type != U_STOP;
        }
        prod_bar();
        Unit un = S.pu;
        if (!S.pready) {
            // a blocking wait: no stage of this CTA's own earlier units may stay held
            // back meanwhile (their epilogues may be what the others wait for)
            flush();
            if (pt == 0) {
                unit_inputs_wait(a, un.type, un.a, un.b);
                if (seq >= kUQ) mbar_wait(&S.uqe[seq % kUQ], ((seq / kUQ) - 1) & 1);
            }
        }
        if (pt == 0) {
            asm volatile("fence.proxy.async.global;" ::: "memory");
            TC_TRACE(a, un.u, 1, gtimer());
            unsigned smid;
            asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
            TC_TRACE(a, un.u, 5, smid);
        }
        prod_bar();
        const int type = un.type, i = un.a, j = un.b;
        // ---- the unit's geometry and rows
        if (type == U_T) {
            un.nst = a.kst / 64;
            un.nsub = a.r > 128 ? 2 : 1;
        } else if (type == U_PRE) {
            un.nst = a.pitch_r / 64;
            un.nsub = blk_rows(a, i) > 128 ? 2 : 1;
        } else if (type == U_GU) {
            // sub-tile 0 = gate rows, 1 = up rows (the same rows of both matrices)
            bool tiled = true;
            int cnt = blk_rows(a, i);
            if (!gu_static(a)) {
                wait_count(fl_pre(a, i), 1);  // (set: orders the list reads below)
                const int listed = __ldcg(a.ucnt + i);
                tiled = listed > 0 && blk_tiled(a, listed, i, a.tile_g);
                if (!tiled) {
                    cnt = listed;  // the block's union rows, gathered
                    for (int k = pt; k < cnt; k += kProdThreads) S.rows[k] = i * kBlk + __ldcg(a.ulist + i * kBlk + k);
                }
            }
            un.cnt = cnt;
            un.nsub = cnt > 0 ? 2 : 0;
            un.nst = cnt > 0 ? a.ksg / 64 : 0;
            un.pad = tiled;
        } else if (type == U_DOWN) {
            un.nst = 1;  // the stage count unfolds block by block (producer / MMA walk the range)
            un.nsub = 1;
        }
        const bool mma_unit = type == U_T || type == U_PRE || type == U_GU || type == U_DOWN;
        if (mma_unit) un.acc = accseq++ & 1;
        prod_bar();  // S.rows complete
        if (pt == 0) {
            const int slot = seq % kUQ;
            S.uq[slot] = un;
            mbar_arrive(&S.uqf[slot]);
        }
        ++seq;
        if (type == U_STOP) break;
        if (!mma_unit || un.nst == 0) continue;

        // ---- one stage per 64-wide K chunk
        auto begin_stage = [&](uint8_t*& As, uint32_t& as, uint64_t*& bar) {
            const int s = n % kStages;
            mbar_wait(&S.empty[s], (ephase >> s) & 1u);
            ephase ^= 1u << s;
            As = stages + s * kStageBytes;
            as = sbase + s * kStageBytes;
            bar = &S.full[s];
        };
        auto end_stage = [&] {
            cp_commit();
            ++n;
            if (++pending > kLag) {
                cp_wait<kLag>();
                stage_arrive(&S.full[(n - pending) % kStages]);
                --pending;
            }
        };
        if (type == U_T || type == U_PRE || un.pad) {
            // contiguous rows: TMA tiles (T: predictor B rows; PRE: A rows; GU: gate + up
            // rows of the block). No thread copies: arrive at once, nothing held back.
            flush();
            const CUtensorMap* am = type == U_T ? &M.Bp : &M.A;
            const CUtensorMap* bm = type == U_PRE ? &M.thl : &M.xhl;
            const int k0 = type == U_T ? i * a.kst : type == U_PRE ? 0 : j * a.ksg;
            const int r0 = type == U_T ? 0 : i * kBlk;
            for (int st = 0; st < un.nst; ++st) {
                uint8_t* As;
                uint32_t as;
                uint64_t* bar;
                begin_stage(As, as, bar);
                if (pt == 0) {
                    mbar_expect_tx(bar, un.nsub * 16384u + bbytes);
                    for (int t = 0; t < un.nsub; ++t)
                        tma_tile(As + t * 16384, type == U_GU ? (t ? &M.up : &M.gate) : am, k0 + st * 64,
                                 type == U_GU ? r0 : r0 + t * 128, bar);
                    tma_tile(As + kStageA, bm, k0 + st * 64, 0, bar);
                }
                mbar_arrive(bar);
                ++n;
            }
        } else if (type == U_GU) {
            // the block's union rows of gate (sub-tile 0) and up (sub-tile 1), gathered
            const int k0 = j * a.ksg;
            const int jj = pt & 7;  // this thread's 16-B chunk of every row it copies
            for (int st = 0; st < un.nst; ++st) {
                uint8_t* As;
                uint32_t as;
                uint64_t* bar;
                begin_stage(As, as, bar);
                const int kc = k0 + st * 64;
                if (pt == 0) {
                    mbar_expect_tx(bar, bbytes);
                    tma_tile(As + kStageA, &M.xhl, kc, 0, bar);
                }
#pragma unroll 4
                for (int r = pt >> 3; r < un.cnt; r += kProdThreads / 8) {
                    const size_t row = static_cast<size_t>(S.rows[r]);
                    const uint32_t dst = as + (r >> 3) * 1024 + (r & 7) * 128 + ((jj ^ (r & 7)) << 4);
                    cp16(dst, a.gate + row * a.pitch_d + kc + jj * 8, pol);
                    cp16(dst + 16384, a.ud + row * 2 * a.pitch_d + kc + jj * 8, pol);
                }
                end_stage();
            }
        } else {  // U_DOWN: K = survivor slots of the block range, A = down rows (MN-major)
            const int m0 = i * 128;
            for (int blk = range_lo(a, j); blk < range_lo(a, j + 1); ++blk) {
                // blocks become ready in order while the unit streams: a blocking wait
                // first releases this thread's held-back stages
                if (!flag_ready(fl_gu(a, blk), 1)) {
                    flush();
                    wait_count(fl_gu(a, blk), 1);
                }
                const int v = __ldcg(a.vcnt + blk);
                if (vcnt_rows(v) == 0) continue;
                if (vcnt_tiled(v)) {
                    // the block's down rows by TMA tiles: 64 k-rows x 2 atoms of 64 outputs;
                    // Z holds zeros for the rows that are not survivors (GU epilogue)
                    flush();
                    for (int c0 = 0; c0 < blk_rows(a, blk); c0 += 64) {
                        uint8_t* As;
                        uint32_t as;
                        uint64_t* bar;
                        begin_stage(As, as, bar);
                        if (pt == 0) {
                            mbar_expect_tx(bar, 2u * 8192u + bbytes);
                            for (int atom = 0; atom < 2; ++atom)
                                tma_tile(As + atom * 8192, &M.down, m0 + atom * 64, blk * kBlk + c0, bar);
                            tma_tile(As + kStageA, &M.zhl, blk * kBlk + c0, 0, bar);
                        }
                        mbar_arrive(bar);
                        ++n;
                    }
                    continue;
                }
                const int cnt = vcnt_rows(v);
                prod_bar();  // the previous block's rows are no longer read
                for (int k = pt; k < cnt; k += kProdThreads)
                    S.rows[k] = blk * kBlk + __ldcg(a.vlist + blk * kBlk + k);
                prod_bar();
                for (int c0 = 0; c0 < cnt; c0 += 64) {
                    uint8_t* As;
                    uint32_t as;
                    uint64_t* bar;
                    begin_stage(As, as, bar);
                    if (pt == 0) {
                        mbar_expect_tx(bar, bbytes);
                        tma_tile(As + kStageA, &M.zhl, blk * kBlk + c0, 0, bar);
                    }
                    // 64 k-rows x 2 atoms of 64 outputs: 1024 chunks of 16 B. Slots past the
                    // block's survivors repeat its last row (finite data against Z = 0: they
                    // add exact zeros).
#pragma unroll 4
                    for (int q = pt; q < 1024; q += kProdThreads) {
                        const int r = q >> 4, atom = (q >> 3) & 1, jj = q & 7;
                        const int row = S.rows[min(c0 + r, cnt - 1)];
                        const uint16_t* src = a.ud + static_cast<size_t>(row) * 2 * a.pitch_d + a.pitch_d + m0 +
                                              atom * 64 + jj * 8;
                        cp16(as + atom * 8192 + (r >> 3) * 1024 + (r & 7) * 128 + ((jj ^ (r & 7)) << 4), src, pol);
                    }
                    end_stage();
                }
            }
        }
        if (pt == 0) TC_TRACE(a, un.u, 2, gtimer());
    }
}

// ---- MMA issuer ----------------------------------------------------------------
__device__ void mma_issuer(const TcArgs& a, TcSmem& S, uint8_t* stages) {
    const int lane = threadIdx.x & 31;
    int seq = 0, stage = 0;
    uint32_t fphase = 0, tphase = 0;  // full[] / tempty[] phases
    int uses[2] = {0, 0};
    for (;;) {
        const int slot = seq % kUQ;
        mbar_wait(&S.uqf[slot], (seq / kUQ) & 1);
        const Unit un = S.uq[slot];
        ++seq;
        const bool mma_unit = un.type == U_T || un.type == U_PRE || un.type == U_GU || un.type == U_DOWN;
        if (mma_unit) {
            const int acc = un.acc;
            if (uses[acc] > 0) mbar_wait(&S.tempty[acc], (tphase >> acc) & 1u), tphase ^= 1u << acc;
            uses[acc]++;
            tc_fence_after();
            const uint32_t dcol = S.tmem + static_cast<uint32_t>(acc * 256);
            const bool mn = un.type == U_DOWN;
            const uint32_t id = idesc(a.N, mn ? 1 : 0);
            // down: K steps of 16 survivor slots; the last stage of a block may be partial
            int dblk = mn ? range_lo(a, un.b) : 0, dleft = 0;
            const int dend = mn ? range_lo(a, un.b + 1) : 0;
            bool dtiled = false;
            for (int st = 0;; ++st) {
                int ksteps = 4;
                if (mn) {
                    while (dleft <= 0 && dblk < dend) {
                        wait_count(fl_gu(a, dblk), 1);  // orders the vcnt read
                        const int v = __ldcg(a.vcnt + dblk);
                        dtiled = vcnt_tiled(v);
                        dleft = dtiled ? blk_rows(a, dblk) : vcnt_rows(v);
                        ++dblk;
                    }
                    if (dleft <= 0) break;
                    const int here = dleft < 64 ? dleft : 64;
                    ksteps = dtiled ? 4 : (here + 15) / 16;
                    dleft -= 64;
                } else if (st >= un.nst) {
                    break;
                }
                mbar_wait(&S.full[stage], (fphase >> stage) & 1u);
                fphase ^= 1u << stage;
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t As = su32(stages + stage * kStageBytes), Bs = As + kStageA;
                    for (int t = 0; t < un.nsub; ++t) {
                        for (int k = 0; k < ksteps; ++k) {
                            uint64_t ad, bd;
                            if (mn) {  // MN-major SW128: atoms of 64 outputs x 64 k-rows (8 KB)
                                ad = sdesc(As + t * 16384 + k * 2048, 8192, 1024);
                            } else {   // K-major SW128: rows of 128 B, 8-row groups of 1 KB
                                ad = sdesc(As + t * 16384 + k * 32, 16, 1024);
                            }
                            bd = sdesc(Bs + k * 32, 16, 1024);
                            umma(dcol + t * a.N, ad, bd, id, (st | k) != 0);
                        }
                    }
                    umma_commit(&S.empty[stage]);
                }
                __syncwarp();
                stage = (stage + 1) % kStages;
            }
            if (lane == 0) umma_commit(&S.tfull[acc]);
            __syncwarp();
        }
        if (lane == 0) mbar_arrive(&S.uqe[slot]);
        if (un.type == U_STOP) break;
    }
}

// ---- epilogue helpers ------------------------------------------------------------
// hi + lo accumulator columns of this thread's TMEM lane (row) for tokens c0..c0+15 of
// sub-tile t: four tcgen05.ld issued back to back, one wait (tokens >= nb read stale
// columns, ignored by the callers).
__device__ __forceinline__ void acc16(const TcArgs& a, uint32_t tbase, int quarter, int accbuf, int t,
                                      int c0, float* v) {
    float h[16], l[16];
    const uint32_t addr = tbase + (static_cast<uint32_t>(quarter * 32) << 16) +
                          static_cast<uint32_t>(accbuf * 256 + t * a.N + c0);
    tmem_ld8(addr, h);
    tmem_ld8(addr + 8u, h + 8);
    tmem_ld8(addr + static_cast<uint32_t>(a.nb), l);
    tmem_ld8(addr + static_cast<uint32_t>(a.nb) + 8u, l + 8);
    tmem_wait();
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = h[e] + l[e];
}
__device__ __forceinline__ void acc8(const TcArgs& a, uint32_t tbase, int quarter, int accbuf, int t,
                                     int c0, float* v) {
    float h[8], l[8];
    const uint32_t addr = tbase + (static_cast<uint32_t>(quarter * 32) << 16) +
                          static_cast<uint32_t>(accbuf * 256 + t * a.N + c0);
    tmem_ld8(addr, h);
    tmem_ld8(addr + static_cast<uint32_t>(a.nb), l);
    tmem_wait();
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = h[e] + l[e];
}
__device__ __forceinline__ void ld16(const float* p, float* v) {  // 16 floats, 16-B aligned
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const float4 f = __ldcg(reinterpret_cast<const float4*>(p) + q);
        v[4 * q] = f.x;
        v[4 * q + 1] = f.y;
        v[4 * q + 2] = f.z;
        v[4 * q + 3] = f.w;
    }
}
__device__ __forceinline__ void st16(float* p, const float* v, int n) {  // n in {8, 16}
#pragma unroll
    for (int q = 0; q < 4; ++q)
        if (4 * q < n) reinterpret_cast<float4*>(p)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
}

// ascending compaction of S.flag[0..n) (non-zero = keep) into out_list (the kept k),
// by the first epilogue warp; returns the count to all epilogue threads
__device__ int epi_compact(TcSmem& S, int n, int et, int* out_list) {
    __shared__ int total;
    if (et < 32) {
        int run = 0;
        for (int b0 = 0; b0 < kBlk; b0 += 32) {
            const int k = b0 + et;
            const bool on = k < n && S.flag[k] != 0;
            const unsigned bal = __ballot_sync(0xffffffffu, on);
            if (on) out_list[run + __popc(bal & ((1u << et) - 1u))] = k;
            run += __popc(bal);
        }
        if (et == 0) total = run;
    }
    epi_bar();
    return total;
}

// per-token counts of the set bits over the 128 epilogue rows (S.cnt, smem)
__device__ __forceinline__ void count_bits(TcSmem& S, uint64_t bits, int B, int lane) {
    for (int b = 0; b < B; ++b) {
        const unsigned bal = __ballot_sync(0xffffffffu, (bits >> b) & 1ull);
        if (lane == 0 && bal) atomicAdd(&S.cnt[b], __popc(bal));
    }
}

// Count this unit's (already CTA-synchronised) writes into a group of `total`; true
// on every epilogue thread iff it was the last arrival, which then reads the others'
// writes (release by their fence + add, acquire by this fence after the add).
__device__ __forceinline__ bool arrive_last(int* p, int total, TcSmem& S, int et) {
    if (et == 0) {
        __threadfence();
        const int last = atomicAdd(p, 1) == total - 1;
        if (last) __threadfence();
        S.last = last;
    }
    epi_bar();
    return S.last != 0;
}

// g, u of this thread's row for every token: the KS slice partials summed in slice
// order 0, 1, ..., KS-1 — this unit's own slice j straight from TMEM (sub-tiles 0 / 1),
// the others from gpart — then z = gated(g, u) on the survivor bits (ffn_exec.hpp:200,
// :68-76). GC chunks of 8 tokens per round of loads; partials held per slice index
// (NS >= KS) so no register array is indexed at run time. With two slices the order is
// moot (a + b == b + a exactly): NS = 1 holds just the other one.
template <int GC, int NS>
__device__ __forceinline__ void gu_reduce(const TcArgs& a, const TcSmem& S, int quarter, int acc, int j, int KS,
                                          const float* rowpart, size_t sstride, bool mine, uint64_t mb,
                                          float* z, uint64_t& sbits) {
    const int nb = a.nb;
#pragma unroll
    for (int c0 = 0; c0 < 64; c0 += 8 * GC) {
        if (c0 >= nb) continue;  // warp-uniform
        float4 q[NS][GC][4];
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            const int sl = NS == 1 ? 1 - j : s;
            if (sl >= KS || sl == j || !mine) continue;
#pragma unroll
            for (int gc = 0; gc < GC; ++gc) {
                const int c = c0 + 8 * gc;
                if (c >= nb) continue;
                const float4* sg = reinterpret_cast<const float4*>(rowpart + sl * sstride + c);
                const float4* su = reinterpret_cast<const float4*>(rowpart + sl * sstride + nb + c);
                q[s][gc][0] = __ldcg(sg);
                q[s][gc][1] = __ldcg(sg + 1);
                q[s][gc][2] = __ldcg(su);
                q[s][gc][3] = __ldcg(su + 1);
            }
        }
#pragma unroll
        for (int gc = 0; gc < GC; ++gc) {
            const int c = c0 + 8 * gc;
            if (c >= nb) continue;
            float g[8], u[8];
            acc8(a, S.tmem, quarter, acc, 0, c, g);
            acc8(a, S.tmem, quarter, acc, 1, c, u);
            if (!mine) continue;
            if (NS == 1) {
                if (KS == 2) {
                    const float4 a0 = q[0][gc][0], a1 = q[0][gc][1], b0 = q[0][gc][2], b1 = q[0][gc][3];
                    g[0] += a0.x; g[1] += a0.y; g[2] += a0.z; g[3] += a0.w;
                    g[4] += a1.x; g[5] += a1.y; g[6] += a1.z; g[7] += a1.w;
                    u[0] += b0.x; u[1] += b0.y; u[2] += b0.z; u[3] += b0.w;
                    u[4] += b1.x; u[5] += b1.y; u[6] += b1.z; u[7] += b1.w;
                }
            } else {
                float gs[8], us[8];
#pragma unroll
                for (int s = 0; s < NS; ++s) {  // slice order
                    if (s >= KS) break;
                    float gv[8], uv[8];
                    if (s == j) {
#pragma unroll
                        for (int e = 0; e < 8; ++e) gv[e] = g[e], uv[e] = u[e];
                    } else {
                        const float4 a0 = q[s][gc][0], a1 = q[s][gc][1], b0 = q[s][gc][2], b1 = q[s][gc][3];
                        gv[0] = a0.x; gv[1] = a0.y; gv[2] = a0.z; gv[3] = a0.w;
                        gv[4] = a1.x; gv[5] = a1.y; gv[6] = a1.z; gv[7] = a1.w;
                        uv[0] = b0.x; uv[1] = b0.y; uv[2] = b0.z; uv[3] = b0.w;
                        uv[4] = b1.x; uv[5] = b1.y; uv[6] = b1.z; uv[7] = b1.w;
                    }
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        gs[e] = s == 0 ? gv[e] : gs[e] + gv[e];
                        us[e] = s == 0 ? uv[e] : us[e] + uv[e];
                    }
                }
#pragma unroll
                for (int e = 0; e < 8; ++e) g[e] = gs[e], u[e] = us[e];
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const bool sv = ((mb >> (c + e)) & 1ull) && g[e] > 0.f;
                if (sv) sbits |= 1ull << (c + e);
                z[c + e] = sv ? gated(g[e], u[e], a.act) : 0.f;
            }
        }
    }
}

// y rows of d tile i (this thread's row m): the S range partials in range order, this
// unit's own range j from TMEM (zeros when it had no rows), the others from ypart.
template <int GC, int NR>
__device__ __forceinline__ void down_reduce(const TcArgs& a, const TcSmem& S, int quarter, int acc, int j,
                                            bool have, int m) {
    const int nb = a.nb, R = a.S;
    const size_t rs = static_cast<size_t>(a.ndt) * 128 * nb;  // between ranges
    const float* rowp = a.ypart + static_cast<size_t>(m) * nb;
#pragma unroll
    for (int c0 = 0; c0 < 64; c0 += 8 * GC) {
        if (c0 >= nb) continue;  // warp-uniform
        float4 q[NR][GC][2];
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            if (r >= R || r == j || m >= a.d) continue;
#pragma unroll
            for (int gc = 0; gc < GC; ++gc) {
                const int c = c0 + 8 * gc;
                if (c >= nb) continue;
                const float4* src = reinterpret_cast<const float4*>(rowp + r * rs + c);
                q[r][gc][0] = __ldcg(src);
                q[r][gc][1] = __ldcg(src + 1);
            }
        }
#pragma unroll
        for (int gc = 0; gc < GC; ++gc) {
            const int c = c0 + 8 * gc;
            if (c >= nb) continue;
            float own[8], y[8];
            if (have) {
                acc8(a, S.tmem, quarter, acc, 0, c, own);
            } else {
#pragma unroll
                for (int e = 0; e < 8; ++e) own[e] = 0.f;
            }
            if (m >= a.d) continue;
#pragma unroll
            for (int r = 0; r < NR; ++r) {  // range order
                if (r >= R) break;
                float v[8];
                if (r == j) {
#pragma unroll
                    for (int e = 0; e < 8; ++e) v[e] = own[e];
                } else {
                    const float4 a0 = q[r][gc][0], a1 = q[r][gc][1];
                    v[0] = a0.x; v[1] = a0.y; v[2] = a0.z; v[3] = a0.w;
                    v[4] = a1.x; v[5] = a1.y; v[6] = a1.z; v[7] = a1.w;
                }
#pragma unroll
                for (int e = 0; e < 8; ++e) y[e] = r == 0 ? v[e] : y[e] + v[e];
            }
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (c + e < a.B) a.y[static_cast<size_t>(c + e) * a.d + m] = y[e];
        }
    }
}

// ---- epilogue -----------------------------------------------------------------
__device__ void epilogue(const TcArgs& a, TcSmem& S) {
    const int et = threadIdx.x - kEpiBase;     // 0..127
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int quarter = warp & 3;              // TMEM lane quarter of this warp
    int seq = 0;
    uint32_t tphase = 0;
    const uint64_t bmask = a.B >= 64 ? ~0ull : ((1ull << a.B) - 1ull);
    const int nb = a.nb;
    for (;;) {
        const int slot = seq % kUQ;
        mbar_wait(&S.uqf[slot], (seq / kUQ) & 1);
        const Unit un = S.uq[slot];
        ++seq;
        if (un.type == U_STOP) break;
        const int i = un.a, j = un.b;
        const bool mma_unit = un.type == U_T || un.type == U_PRE || un.type == U_GU || un.type == U_DOWN;
        bool have = false;
        if (mma_unit) {
            have = un.nst > 0;  // DOWN: recomputed below from the range's survivor counts
            mbar_wait(&S.tfull[un.acc], (tphase >> un.acc) & 1u);
            tphase ^= 1u << un.acc;
            tc_fence_after();
        }
        if (et == 0) TC_TRACE(a, un.u, 3, gtimer());
        const int row0 = quarter * 32 + lane;  // this thread's row of each sub-tile
        const int acc = un.acc;

        if (un.type == U_X) {
            // x (fp32 [B][d]) -> X^T hi rows 0..nb-1, lo rows nb..2nb-1 (bf16 [N][xpitch]):
            // this unit's share of the (token, 8-column chunk) items, float4 loads
            const int nch = a.pitch_d / 8, items = nb * nch;
            const int per = (items + a.u_T - 1) / a.u_T;
            const int w0 = i * per, w1 = min(items, w0 + per);
            bool bad = false;
            const bool vec = (a.d & 7) == 0;
            for (int wb = w0 + et; wb < w1; wb += 4 * 128) {  // 4 items per thread: loads first
                float v[4][8];
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const int w = wb + h * 128;
                    const int b = w / nch, k0 = (w % nch) * 8;
                    if (w < w1 && b < a.B && vec && k0 < a.d) {
                        const float4* src = reinterpret_cast<const float4*>(a.x + static_cast<size_t>(b) * a.d + k0);
                        const float4 f0 = __ldg(src), f1 = __ldg(src + 1);
                        v[h][0] = f0.x; v[h][1] = f0.y; v[h][2] = f0.z; v[h][3] = f0.w;
                        v[h][4] = f1.x; v[h][5] = f1.y; v[h][6] = f1.z; v[h][7] = f1.w;
                    } else {
#pragma unroll
                        for (int e = 0; e < 8; ++e)
                            v[h][e] = (w < w1 && b < a.B && k0 + e < a.d) ? __ldg(a.x + static_cast<size_t>(b) * a.d + k0 + e) : 0.f;
                    }
                }
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const int w = wb + h * 128;
                    if (w >= w1) break;
                    const int b = w / nch, k0 = (w % nch) * 8;
                    uint16_t hi[8], lo[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        bad |= !isfinite(v[h][e]);
                        split_bf16(v[h][e], hi[e], lo[e]);
                    }
                    uint4 vh, vl;
                    vh.x = hi[0] | (uint32_t(hi[1]) << 16); vh.y = hi[2] | (uint32_t(hi[3]) << 16);
                    vh.z = hi[4] | (uint32_t(hi[5]) << 16); vh.w = hi[6] | (uint32_t(hi[7]) << 16);
                    vl.x = lo[0] | (uint32_t(lo[1]) << 16); vl.y = lo[2] | (uint32_t(lo[3]) << 16);
                    vl.z = lo[4] | (uint32_t(lo[5]) << 16); vl.w = lo[6] | (uint32_t(lo[7]) << 16);
                    *reinterpret_cast<uint4*>(a.xhl + static_cast<size_t>(b) * a.xpitch + k0) = vh;
                    *reinterpret_cast<uint4*>(a.xhl + static_cast<size_t>(nb + b) * a.xpitch + k0) = vl;
                }
            }
            if (bad) atomicOr(a.bad, 1);  // check_input, ffn_exec.hpp:61-63
            asm volatile("fence.proxy.async.global;" ::: "memory");
            epi_bar();
            if (et == 0) signal(fl_x(a));
        } else if (un.type == U_T) {
            // partial T^T over K slice i: tpart[i][row][b], hi + lo summed
            for (int t = 0; t < un.nsub; ++t) {
                const int row = t * 128 + row0;
                for (int c = 0; c < nb; c += 16) {
                    float v[16];
                    acc16(a, S.tmem, quarter, acc, t, c, v);
                    st16(a.tpart + (static_cast<size_t>(i) * kTRows + row) * nb + c, v, min(16, nb - c));
                }
            }
            tc_fence_before();
            epi_bar();
            if (et == 0) {
                mbar_arrive(&S.tempty[acc]);
                signal(fl_t(a));
            }
        } else if (un.type == U_TR) {
            // rows [4i, 4i+4) x nb tokens: fixed-order sum of the KT slices, all loads first
            const int KT = a.u_TR - a.u_T;
            wait_count(fl_t(a), KT);
            for (int w = et; w < 4 * nb; w += 128) {
                const int row = i * 4 + w / nb, b = w % nb;
                const float* src = a.tpart + static_cast<size_t>(row) * nb + b;
                float s = 0.f;
                for (int k0 = 0; k0 < KT; k0 += 16) {  // fixed order over the K slices
                    float p[16];
#pragma unroll
                    for (int k = 0; k < 16; ++k)
                        p[k] = k0 + k < KT ? __ldcg(src + static_cast<size_t>(k0 + k) * kTRows * nb) : 0.f;
#pragma unroll
                    for (int k = 0; k < 16; ++k)
                        if (k0 + k < KT) s += p[k];
                }
                uint16_t hi, lo;
                split_bf16(row < a.r ? s : 0.f, hi, lo);
                a.thl[static_cast<size_t>(b) * 256 + row] = hi;
                a.thl[static_cast<size_t>(nb + b) * 256 + row] = lo;
            }
            asm volatile("fence.proxy.async.global;" ::: "memory");
            epi_bar();
            if (et == 0) signal(fl_tr(a));
        } else if (un.type == U_PRE) {
            // mask bits per neuron (strict pre > 0, ffn_exec.hpp:141), union list
            const int rows = blk_rows(a, i);
            if (et < 64) S.cnt[et] = 0;
            epi_bar();
            {
                const int k = row0, t = 0;
                uint64_t bits = 0;
                {
                    const bool mine = k < rows;
                    const float bias = mine ? __ldg(a.bias + i * kBlk + k) : 0.f;
                    for (int c = 0; c < nb; c += 16) {
                        float v[16];
                        acc16(a, S.tmem, quarter, acc, t, c, v);
#pragma unroll
                        for (int e = 0; e < 16; ++e)
                            if (c + e < nb && v[e] + bias > 0.f) bits |= 1ull << (c + e);
                    }
                    bits = mine ? (bits & bmask) : 0ull;
                    if (mine) {
                        a.mbits[i * kBlk + k] = bits;
                        a.vbits[i * kBlk + k] = 0ull;
                    }
                }
                S.flag[k] = bits != 0;
                count_bits(S, bits, a.B, lane);
            }
            tc_fence_before();
            epi_bar();
            if (et == 0) mbar_arrive(&S.tempty[acc]);
            const int n = epi_compact(S, rows, et, a.ulist + i * kBlk);
            if (et < a.B && S.cnt[et]) atomicAdd(a.pcount + et, S.cnt[et]);
            if (et == 0) {
                a.ucnt[i] = n;
                signal(fl_pre(a, i));
            }
            epi_bar();
        } else if (un.type == U_GU) {
            // block i (128 neurons), K slice j: g (sub-tile 0) and u (sub-tile 1) partials;
            // the last slice of the block to finish reduces them (no unit ever waits for
            // another's epilogue)
            const int KS = a.KSg, cnt = un.cnt, k = row0;
            const size_t pw = 2 * static_cast<size_t>(nb);  // floats per partial row: g | u
            const size_t sstride = static_cast<size_t>(a.nblk) * kBlk * pw;  // between slices
            const float* rowpart = a.gpart + (static_cast<size_t>(i) * kBlk + k) * pw;
            bool fin = true;
            if (KS > 1) {
                float* dst = a.gpart + static_cast<size_t>(j) * sstride + (static_cast<size_t>(i) * kBlk + k) * pw;
                if (un.nsub > 0)  // warp-uniform
                    for (int t = 0; t < 2; ++t)
                        for (int c = 0; c < nb; c += 16) {
                            float v[16];
                            acc16(a, S.tmem, quarter, acc, t, c, v);
                            if (k < cnt) st16(dst + t * nb + c, v, min(16, nb - c));
                        }
                epi_bar();
                if (et == 0) TC_TRACE(a, un.u, 6, gtimer());
                fin = arrive_last(fl_gpart(a, i), KS, S, et);
            }
            if (et == 0) TC_TRACE(a, un.u, 7, gtimer());
            if (!fin) {
                tc_fence_before();
                epi_bar();
                if (et == 0) mbar_arrive(&S.tempty[acc]);
            } else {
                // survivors V_b = P_b & g > 0; z = gated(g, u) on V_b, else +0
                if (!a.dense) wait_count(fl_pre(a, i), 1);  // mask bits (set long before, as a rule)
                if (et < 64) S.cnt[et] = 0;
                epi_bar();
                const bool mine = un.nsub > 0 && k < cnt;
                const int lrow = un.pad ? k : (mine ? __ldcg(a.ulist + i * kBlk + k) : 0);  // row in block
                const int n = i * kBlk + lrow;
                const uint64_t mb = a.dense ? bmask : (mine ? __ldcg(a.mbits + n) : 0ull);
                float z[64];
#pragma unroll
                for (int e = 0; e < 64; ++e) z[e] = 0.f;
                uint64_t sbits = 0;
#ifdef SG_TC_FINTRACE
                if (et == 0) TC_TRACE(a, un.u, 5, gtimer());
#endif
                if (un.nsub > 0) gu_reduce<4, 1>(a, S, quarter, acc, j, KS, rowpart, sstride, mine, mb, z, sbits);
#ifdef SG_TC_FINTRACE
                epi_bar();
                if (et == 0) TC_TRACE(a, un.u, 6, gtimer());
#endif
                tc_fence_before();
                sbits &= bmask;
                if (mine) a.vbits[n] = sbits;
                count_bits(S, sbits, a.B, lane);
                // survivor slots: ascending rows (positions k ascend with the local row)
                const bool keep = sbits != 0;
                const unsigned bal = __ballot_sync(0xffffffffu, keep);
                if (lane == 0) S.wsum[quarter] = __popc(bal);
                epi_bar();
                if (et == 0) mbar_arrive(&S.tempty[acc]);
                int before = 0;
                for (int q = 0; q < quarter; ++q) before += S.wsum[q];
                const int nv = S.wsum[0] + S.wsum[1] + S.wsum[2] + S.wsum[3];
                const int slot_c = before + __popc(bal & ((1u << lane) - 1u));
                // DOWN streams a tiled GU block whole (Z slot = row) when its survivors are
                // dense enough, else gathers the survivor rows (Z slot = survivor position);
                // the slots up to the next 64 are exact zeros either way
                const bool dtile = un.pad && nv > 0 && blk_tiled(a, nv, i, a.tile_u);
                const int pad_to = dtile ? (blk_rows(a, i) + 63) / 64 * 64 : (nv + 63) / 64 * 64;
                // this thread's slots: its z (if any) and an exact-zero padding slot (if any)
                int zslot = -1, pslot = -1;
                if (dtile) {
                    if (mine) zslot = lrow;
                    else if (k < pad_to) pslot = k;
                } else {
                    if (keep) {
                        zslot = slot_c;
                        a.vlist[i * kBlk + slot_c] = lrow;
                    }
                    if (k >= nv && k < pad_to) pslot = k;
                }
                // Z^T rows are K-major (slots contiguous per token): stage 8 tokens at a time
                // in smem, then store whole 16-B runs of 8 slots
                const int chunks = pad_to / 8;
#pragma unroll
                for (int c = 0; c < 64; c += 8) {
                    if (c >= nb) continue;  // uniform
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        uint16_t hi, lo;
                        split_bf16(z[c + e], hi, lo);
                        if (zslot >= 0) S.zst[0][e][zslot] = hi, S.zst[1][e][zslot] = lo;
                        if (pslot >= 0) S.zst[0][e][pslot] = 0, S.zst[1][e][pslot] = 0;
                    }
                    epi_bar();
                    for (int w = et; w < 16 * chunks; w += 128) {
                        const int row = w / chunks, ch = w % chunks, hl = row >> 3, e = row & 7;
                        const uint4 v = *reinterpret_cast<const uint4*>(&S.zst[hl][e][ch * 8]);
                        *reinterpret_cast<uint4*>(a.zhl + static_cast<size_t>(hl * nb + c + e) * a.zpitch +
                                                  static_cast<size_t>(i) * kBlk + ch * 8) = v;
                    }
                    epi_bar();
                }
                if (et < a.B && S.cnt[et]) atomicAdd(a.vcount + et, S.cnt[et]);
#ifdef SG_TC_FINTRACE
                epi_bar();
                if (et == 0) TC_TRACE(a, un.u, 7, gtimer());
#endif
                asm volatile("fence.proxy.async.global;" ::: "memory");  // Z is read by TMA
                epi_bar();
                if (et == 0) {
                    a.vcnt[i] = nv | (dtile ? kVTiled : 0);
                    signal(fl_gu(a, i));
                }
            }
        } else if (un.type == U_DOWN) {
            // partial y over block range j for d tile i (128 outputs): ypart[j][m][b]; the
            // last range of the d tile to finish sums the S partials in range order into y
            const int m = i * 128 + row0;
            {  // did the range hold any survivor row (else the accumulator was never written)
                int hv = 0;
                for (int blk = range_lo(a, j) + et; blk < range_lo(a, j + 1); blk += 128)
                    hv |= vcnt_rows(__ldcg(a.vcnt + blk)) > 0;
                have = epi_bar_or(hv);
            }
            bool fin = true;
            if (a.S > 1) {
                float* dst = a.ypart + (static_cast<size_t>(j) * a.ndt * 128 + m) * nb;
                for (int c = 0; c < nb; c += 16) {
                    float v[16];
                    if (have) {
                        acc16(a, S.tmem, quarter, acc, 0, c, v);
                    } else {
#pragma unroll
                        for (int e = 0; e < 16; ++e) v[e] = 0.f;
                    }
                    st16(dst + c, v, min(16, nb - c));
                }
                epi_bar();
                if (et == 0) TC_TRACE(a, un.u, 6, gtimer());
                fin = arrive_last(fl_down(a, i), a.S, S, et);
            }
            if (et == 0) TC_TRACE(a, un.u, 7, gtimer());
            if (fin) down_reduce<2, 4>(a, S, quarter, acc, j, have, m);
            tc_fence_before();
            epi_bar();
            if (et == 0) mbar_arrive(&S.tempty[acc]);
        }
        if (et == 0) {
            TC_TRACE(a, un.u, 4, gtimer());
            mbar_arrive(&S.uqe[slot]);
        }
    }
}

__global__ void __launch_bounds__(kTcThreads, 1) tc_kernel(const __grid_constant__ TcMaps maps, const TcArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* stages = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    TcSmem& S = *reinterpret_cast<TcSmem*>(stages + kStages * kStageBytes);
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&S.full[s], kProdThreads + 1);  // the producer threads + the expect_tx
            mbar_init(&S.empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&S.tfull[s], 1);
            mbar_init(&S.tempty[s], 1);
        }
        for (int s = 0; s < kUQ; ++s) {
            mbar_init(&S.uqf[s], 1);
            mbar_init(&S.uqe[s], 2);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&S.tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // the producer waits on empty[] before every stage: pre-arrive the first round
    if (threadIdx.x == 0)
        for (int s = 0; s < kStages; ++s) mbar_arrive(&S.empty[s]);
    __syncthreads();
    if (warp < kMmaWarp) {
        producer(a, maps, S, stages);
    } else if (warp == kMmaWarp) {
        mma_issuer(a, S, stages);
    } else {
        epilogue(a, S);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == kMmaWarp) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(S.tmem));
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(fl_exit(a), 1) == static_cast<int>(gridDim.x) - 1) {
            // last CTA out: every other CTA has finished; reset the dataflow counters
            __threadfence();
            for (int k = 0; k < flag_count(a); ++k) a.flags[k] = 0;
            __threadfence();
        }
    }
}

}  // namespace

int tc_smem_bytes() { return kStages * kStageBytes + static_cast<int>(sizeof(TcSmem)) + 1024; }
int tc_flag_ints(int nblk, int ndt) { return 32 + 3 * nblk + ndt; }

int launch_batch_tc(const TcMaps& maps, const TcArgs& a, int grid, void* stream) {
    const int smem = tc_smem_bytes();
    const int e = ensure_smem_attr(reinterpret_cast<const void*>(tc_kernel), smem);
    if (e) return e;
    tc_kernel<<<grid, kTcThreads, smem, static_cast<cudaStream_t>(stream)>>>(maps, a);
    return static_cast<int>(cudaGetLastError());
}

}  // namespace sg
