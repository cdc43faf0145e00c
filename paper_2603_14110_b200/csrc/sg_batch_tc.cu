// sparsegate-b200: batched decode (BASELINE.json configs[4]) on the 5th-generation
// tensor cores — B in [2, 64] tokens through one layer, ONE persistent launch.
//
// Per token the result means exactly what sparse_ffn_sequential
// (/root/reference/proj/include/sparsegate/ffn_exec.hpp:183-218) returns for that
// token alone: its predicted set P_b (pre > 0, :141), survivors V_b (g > 0, :200),
// gated values (:68-76) and y_b over V_b (:80-94). The batch shares the weight
// traffic: every weight row is read ONCE from HBM and multiplied against all B tokens.
//
// Numerics: x (and t, z) enter the tensor cores as bf16 hi + lo pairs (x = hi + lo,
// relative error ~2^-17, inside the 2^-14 parity band of tests/parity_util.py);
// the two halves are the N = 2*nb columns of one MMA (hi tokens, then lo tokens) and
// are summed in the epilogue, fp32 accumulation in TMEM throughout.
//
// Why the gate / up rows are streamed whole: the union of B tokens' predicted sets
// covers most rows already at B = 2-4 (about 2/3 of them at B = 4 on the bench
// layers), and a row gather runs at a fraction of the TMA tile rate, so the batch
// reads every gate and up row by TMA tiles and applies the masks in the epilogue;
// the down rows, needed only for the union of the SURVIVOR sets (a quarter to a half
// of the rows), are gathered per block when sparse enough, else tiled too.
//
// Work decomposition (a dataflow of units claimed from one global counter in a
// host-built topological order, so a unit only ever waits for units claimed before
// it — no co-residency assumption, no grid barrier):
//   X    split x -> bf16 hi/lo rows of X^T (K-major B operand)
//   T    T^T = Bp X^T over a K slice (M = 256 predictor rows); the last slice to finish
//        sums the KT partials in slice order -> bf16 hi/lo T^T
//   GU   neuron block i (brows <= 128 rows, one block per SM: no split-K): g = gate X,
//        u = up X and — sparse — pre = A T, all into TMEM; the epilogue derives the
//        tokens' mask bits (pre + bias > 0), survivors (mask & g > 0), z = gated(g, u),
//        the block's survivor list and Z^T (bf16 hi/lo, K-major)
//   DOWN d tile (128 outputs) x block range s: y_s = down^T[rows] Z, streaming the
//        range's blocks as they complete (survivor rows gathered, or whole blocks by
//        TMA tiles when dense enough); the last range of a tile to finish sums the S
//        partials in range order into y
// All reductions have a fixed order, no float atomics: bit-identical on rerun.
//
// CTA (256 threads = 2 warps per SM sub-partition, so up to 255 registers): warps
// 0-2 = producer (claims units, waits their inputs, TMA tiles / cp.async row
// gathers), warp 3 = MMA issuer (tcgen05.mma from one lane; TMEM: two accumulator
// buffers of 256 columns), warps 4-7 = epilogue (tcgen05.ld; one TMEM lane quarter
// each) and the non-MMA units. 4 smem stages of 48 KB.
#include "sg_internal.h"

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <algorithm>
#include <cstdlib>

namespace sg {
namespace {

constexpr int kProdThreads = 96;  // warps 0-2: producers
constexpr int kMmaWarp = 3;       // warp 3: MMA issuer; warps 4-7: epilogue
constexpr int kEpiBase = 128;
constexpr int kTcThreads = 256;
constexpr int kLag = 3;           // stages a producer thread keeps in flight before arriving
constexpr int kStagesMax = 6;     // smem ring depth at most (a.nstages: as many as fit)
constexpr int kStageA = 32768;    // two M = 128 A tiles of 64 K (bf16)
constexpr int kStageB = 16384;    // <= 128 rows (N) x 64 K bf16 (B area: a.stage_bytes - kStageA)
constexpr int kUQ = 4;            // unit queue depth (producer lead)
constexpr int kBlk = 128;         // neurons per block at most (one M = 128 tile)
constexpr int kTRows = 256;       // predictor rows (rank <= 256: two M = 128 tiles)

enum UnitType : int { U_STOP = 0, U_X, U_T, U_GU, U_DOWN, U_PF };

struct Unit {
    int type;
    int a, b;    // block / tile index, K slice / block-range index
    int nst;     // smem stages (MMA units; DOWN: unfolds while streaming)
    int nsub;    // A sub-tiles per stage (T: 128-row halves; GU: gate, up)
    int cnt;     // rows of the unit
    int acc;     // TMEM accumulator buffer
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
__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t par) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(su32(b)), "r"(par)
        : "memory");
    return ok != 0;
}
// TMA tile with an L2 policy: weight tiles are read once per launch (evict-first), the
// X^T / T^T / Z^T operand tiles are re-read by every block / d tile (evict-last)
__device__ __forceinline__ void tma_tile_ef(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* bar,
                                            uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(su32(dst)),
        "l"(m), "r"(c0), "r"(c1), "r"(su32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
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
// D (+)= A B, issued by the whole (converged) warp: one elected lane executes it and
// the operands stay warp-uniform (no per-lane operand broadcast loop around the MMA)
__device__ __forceinline__ void umma_warp(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
        "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void umma_commit_warp(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(su32(bar))
        : "memory");
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
// 16 fp32 columns of this warp's TMEM lane quarter (call tmem_wait before use)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
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
// 16-B global -> shared copy on the LSU path (row gathers)
__device__ __forceinline__ void cp16(uint32_t dst, const void* src, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// the warp's copies of the stage have landed: make them visible to the tensor cores
// (async proxy) and count the warp on the stage's full barrier (one arrival per
// producer warp: a barrier word updated by 96 threads per stage costs more than the
// stage's data takes to arrive)
constexpr int kFullArrivals = kProdThreads / 32 + 1;  // the producer warps + the expect_tx
__device__ __forceinline__ void stage_arrive(uint64_t* bar) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
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
// [3] epilogue start, [4] epilogue end, [5] SM id, [6] / [7] epilogue-internal stamps
#define TC_TRACE(a, u, k, v)                                                         \
    do {                                                                             \
        if ((a).trace != nullptr && (u) >= 0 && (u) < (a).n_units)                   \
            (a).trace[static_cast<size_t>(u) * 8 + (k)] = (v);                       \
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
// sg_host.cpp tc_schedule): X, the predictor's T slices, the GU blocks, and each
// block range's DOWN units merged in about one wave of claims after its last GU
// block. Every unit's inputs come from units earlier in the order, so the dataflow
// cannot deadlock.
__device__ __forceinline__ int unit_type(const TcArgs& a, int u, int& i, int& j) {
    if (u >= a.n_units) return U_STOP;
    const int code = __ldg(a.order + u);
    i = (code >> 8) & 0xffff;
    j = code & 0xff;
    return code >> 24;
}
__device__ __forceinline__ int blk_rows(const TcArgs& a, int blk) {
    const int r = a.D - blk * a.brows;
    return r < a.brows ? r : a.brows;
}
// The S block ranges of the DOWN units interleave chunks of a.rchunk consecutive
// blocks (range j: chunks j, j + S, j + 2S, ...), so every range mixes the layout's
// leading (hot) and trailing (cold) blocks and the ranges carry about equal survivor
// rows, while a chunk's tiled blocks still stream as one run of full stages; block k
// of range j (>= nblk: past its end).
__device__ __forceinline__ int range_block(const TcArgs& a, int j, int k) {
    return (j + (k / a.rchunk) * a.S) * a.rchunk + k % a.rchunk;
}
// DOWN streams a block whole by TMA tiles (reading its non-survivor rows too, against
// Z = 0) once its survivors are a large enough share of its rows: a row gather moves
// a fraction of the tile rate per SM.
__device__ __forceinline__ bool down_tiled(const TcArgs& a, int nv, int blk) {
    return a.dense || nv * 1024 >= a.tile_u * blk_rows(a, blk);
}
// vcnt[blk] = survivor rows | kVTiled when DOWN streams the block whole (GU epilogue)
constexpr int kVTiled = 1 << 16;
__device__ __forceinline__ int vcnt_rows(int raw) { return raw & (kVTiled - 1); }
__device__ __forceinline__ bool vcnt_tiled(int raw) { return (raw & kVTiled) != 0; }

// The DOWN stages of a block range, walked identically by the producer and the MMA
// issuer. Z slots are neuron rows (a gathered block packs its survivors at the start of
// its own rows), so consecutive tiled blocks form one run of contiguous rows cut into
// full 64-row stages; a gathered block's survivor slots are cut into stages of their
// own. A stage covers `rows` K rows (its MMA runs ceil(rows / 16) K steps; the Z
// slots up to the next 16 are exact zeros).
struct DownWalk {
    int j, k, done;   // the range, its next block index, all blocks visited
    int run0, run1;   // tiled rows not yet staged
    int pend, pv;     // a block that does not extend the run, its vcnt
    int gblk, g0, g1; // the gathered block being staged: survivor positions [g0, g1)
    int cb, cp;       // block k = range_block(j, k), incrementally: chunk base, position in it
};
struct DownStage {
    int tiled;  // 1: rows [row0, row0 + rows); 0: block gblk's survivors [c0, c0 + rows)
    int row0, rows, gblk, c0;
    int kd;     // K rows the stage's smem layout holds (128: tiled stages when Z fits twice)
};
// TMEM accumulator regions (512 columns). Normally two buffers of 256; a sparse GU
// unit past 85 tokens needs g | u | pre = 3N columns, so then region 0 = [0, 3N) holds
// the GU and T units and region 1 = [3N, 512) (>= N) the DOWN units: a down unit's
// MMAs still overlap the GU epilogue on the same SM.
__device__ __forceinline__ bool tmem_split(const TcArgs& a) { return !a.dense && 3 * a.N > 256; }
__device__ __forceinline__ uint32_t acc_base(const TcArgs& a, int acc) {
    return acc == 0 ? 0u : static_cast<uint32_t>(tmem_split(a) ? 3 * a.N : 256);
}
// tiled down stages take 128 K rows when the Z tile of 128 slots fits the B area
__device__ __forceinline__ int down_kd(const TcArgs& a) { return a.N <= 64 ? 128 : 64; }
__device__ __forceinline__ DownWalk down_walk(const TcArgs& a, int j) {
    return DownWalk{j, 0, 0, 0, 0, -1, 0, 0, 0, 0, j * a.rchunk, 0};
}
template <class Wait>
__device__ __forceinline__ bool down_next(const TcArgs& a, DownWalk& w, DownStage& st, Wait&& wait) {
    for (;;) {
        const int kd = down_kd(a);
        if (w.g0 < w.g1) {
            st = DownStage{0, 0, min(kd, w.g1 - w.g0), w.gblk, w.g0, kd};
            w.g0 += kd;
            return true;
        }
        if (w.run1 - w.run0 >= kd || (w.run1 > w.run0 && (w.pend >= 0 || w.done))) {
            st = DownStage{1, w.run0, min(kd, w.run1 - w.run0), 0, 0, kd};
            w.run0 += st.rows;
            return true;
        }
        if (w.pend >= 0) {  // the run is staged: now the block behind it
            if (vcnt_tiled(w.pv)) {
                w.run0 = w.run1 = w.pend * a.brows;
                w.run1 += blk_rows(a, w.pend);
            } else {  // (an empty block: nothing)
                w.gblk = w.pend;
                w.g0 = 0;
                w.g1 = vcnt_rows(w.pv);
            }
            w.pend = -1;
            continue;
        }
        if (w.done) return false;
        const int blk = w.cb + w.cp;  // range_block(a, w.j, w.k)
        if (blk >= a.nblk) {
            w.done = 1;
            continue;
        }
        if (++w.cp == a.rchunk) {
            w.cp = 0;
            w.cb += a.S * a.rchunk;
        }
        const int v = wait(w.k++, blk);  // the block's vcnt once it is complete
        if (vcnt_tiled(v) && w.run1 > w.run0 && w.run1 == blk * a.brows) {
            w.run1 += blk_rows(a, blk);  // contiguous with the run: extend it
        } else if (vcnt_tiled(v) && w.run1 == w.run0) {
            w.run0 = w.run1 = blk * a.brows;
            w.run1 += blk_rows(a, blk);
        } else {
            w.pend = blk;
            w.pv = v;
        }
    }
}

// flags layout (ints), zeroed by the last CTA of every launch
__device__ __forceinline__ int* fl_work(const TcArgs& a) { return a.flags; }
__device__ __forceinline__ int* fl_exit(const TcArgs& a) { return a.flags + 1; }
__device__ __forceinline__ int* fl_x(const TcArgs& a) { return a.flags + 2; }
__device__ __forceinline__ int* fl_t(const TcArgs& a, int h) { return a.flags + 3 + 2 * h; }  // T partials of half h
__device__ __forceinline__ int* fl_tr(const TcArgs& a) { return a.flags + 4; }  // T^T halves ready
// predictor row halves (M = 128 tiles) of the T units
__device__ __forceinline__ int t_halves(const TcArgs& a) { return a.r > 128 ? 2 : 1; }
__device__ __forceinline__ int* fl_gu(const TcArgs& a, int b) { return a.flags + 32 + b; }
__device__ __forceinline__ int* fl_down(const TcArgs& a, int t) { return a.flags + 32 + a.nblk + t; }
__device__ __forceinline__ int flag_count(const TcArgs& a) { return 32 + a.nblk + a.ndt; }

// what the MMA issuer needs of a DOWN stage (written by the producer's controller
// before it arrives on the stage's full barrier)
struct StageInfo {
    int ksteps;  // K steps of 16 (0: no data)
    int kd;      // K rows of the stage's layout
    int last;    // the unit's final (empty) stage
};
struct TcSmem {
    uint64_t full[kStagesMax], empty[kStagesMax], tfull[2], tempty[2], uqf[kUQ], uqe[kUQ];
    uint64_t bbar[kUQ];  // a queued GU unit's predictor bias landed in bias[slot]
    StageInfo sinfo[kStagesMax];
    Unit uq[kUQ];
    uint32_t tmem;
    int rows[kBlk];      // producer: gather rows of the current block (global neuron index)
    int dvc[kProdThreads];  // producer: vcnt of the DOWN unit's blocks found complete at its start (-1: not yet)
    Unit pu;             // producer: the unit being claimed
    int pready;          // producer: its inputs and queue slot are available now
    int cnt[64];         // epilogue: per-token counts
    int wsum[8];         // epilogue: per-quarter counts
    int last;            // epilogue: this unit was the last of its group (it reduces)
    alignas(16) uint16_t zst[2][16][kBlk];  // epilogue: hi / lo of 16 tokens x 128 rows, staged
    alignas(16) float bias[kUQ][kBlk];      // a queued GU unit's predictor bias (bulk-copied at claim)
};
constexpr int kTcSmemPad = (static_cast<int>(sizeof(TcSmem)) + 1023) / 1024 * 1024;

// ---- producer: claim, wait, load ---------------------------------------------
// 96 threads (warps 0-2). Thread 0 is the controller: it claims units, checks and
// waits their inputs and publishes them. Contiguous rows and the B operands come by
// TMA tiles from the controller; gathered down rows by 16-B cp.async from every
// producer thread, written in the 128-B-swizzled UMMA layout. For gathered stages
// each thread keeps kLag stages of its copies in flight, then (wait_group, proxy
// fence, warp sync) arrives on the stage's full barrier once per warp (kFullArrivals:
// the warps + the controller's expect_tx); tile stages arrive at once. Before any blocking
// wait every thread flushes its pending arrivals, so no stage is held back.
__device__ __forceinline__ bool unit_inputs_ready(const TcArgs& a, int type, int j) {
    switch (type) {
        case U_T:
        case U_GU: return flag_ready(fl_x(a), a.u_T);
        case U_DOWN: return flag_ready(fl_gu(a, range_block(a, j, 0)), 1);  // later blocks: as they stream
        default: return true;  // U_X
    }
}
__device__ __forceinline__ void unit_inputs_wait(const TcArgs& a, int type, int j) {
    switch (type) {
        case U_T:
        case U_GU: wait_count(fl_x(a), a.u_T); break;
        case U_DOWN: wait_count(fl_gu(a, range_block(a, j, 0)), 1); break;
        default: break;
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ void producer(const TcArgs& a, const TcMaps& M, TcSmem& S, uint8_t* stages) {
    const int pt = threadIdx.x;  // 0..95
    const uint64_t pol = policy_evict_first(), pol_last = policy_evict_last();
    const uint32_t bbytes = static_cast<uint32_t>(a.N) * 128u;
    const uint32_t abytes = static_cast<uint32_t>(a.brows) * 128u;  // one block's rows x 64 K
    const uint32_t sbase = su32(stages);
    int seq = 0, accseq = 0;
    int n = 0;         // stages issued by this thread (all producer threads agree)
    int pending = 0;   // of which not yet arrived
    int spos = 0;      // n % a.nstages (the ring slot of stage n)
    const int nst = a.nstages;
    auto back = [&](int k) { return spos - k < 0 ? spos - k + nst : spos - k; };  // slot of stage n - k
    auto advance = [&] {
        ++n;
        spos = spos + 1 == nst ? 0 : spos + 1;
    };
    uint32_t ephase = 0;  // bit s: parity of empty[s] to wait for
    auto flush = [&] {
        cp_wait<0>();
        for (; pending > 0; --pending) stage_arrive(&S.full[back(pending)]);
    };
#ifdef SG_TC_FINTRACE
    unsigned long long ewait = 0;  // ns the controller spent waiting for free stages (this unit)
#endif
    auto begin_stage = [&](uint8_t*& As, uint32_t& as, uint64_t*& bar) {
        const int s = spos;
#ifdef SG_TC_FINTRACE
        const unsigned long long t0 = gtimer();
        mbar_wait(&S.empty[s], (ephase >> s) & 1u);
        ewait += gtimer() - t0;
#else
        mbar_wait(&S.empty[s], (ephase >> s) & 1u);
#endif
        ephase ^= 1u << s;
        As = stages + s * a.stage_bytes;
        as = sbase + s * a.stage_bytes;
        bar = &S.full[s];
    };
    auto end_gather_stage = [&] {
        cp_commit();
        advance();
        if (++pending > kLag) {
            cp_wait<kLag>();
            stage_arrive(&S.full[back(pending)]);
            --pending;
        }
    };
    auto end_tile_stage = [&](uint64_t* bar) {  // (no copies of this warp: arrive now)
        __syncwarp();
        if ((pt & 31) == 0) mbar_arrive(bar);
        advance();
    };
    // a cross-CTA wait inside a unit: release this thread's held-back stages first
    auto wait_flag = [&](const int* p, int target) {
        if (!flag_ready(p, target)) {
            flush();
            wait_count(p, target);
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");
    };
    for (;;) {
        // ---- claim the next unit of the order (controller), then everyone sees it
        if (pt == 0) {
            const int u = atomicAdd(fl_work(a), 1);
            int i = 0, j = 0;
            const int type = unit_type(a, u, i, j);
            S.pu = Unit{type, i, j, 0, 0, 0, 0, u};
            TC_TRACE(a, u, 0, gtimer());
            bool ready = unit_inputs_ready(a, type, j);
            if (ready && seq >= kUQ) ready = mbar_test(&S.uqe[seq % kUQ], ((seq / kUQ) - 1) & 1);
            S.pready = ready && type != U_STOP;
        }
        prod_bar();
        Unit un = S.pu;
        if (!S.pready) {
            flush();
            if (pt == 0) {
                unit_inputs_wait(a, un.type, un.b);
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
        // ---- the unit's geometry
        if (type == U_T) {
            un.nst = a.kst / 64;
            un.nsub = 1;  // predictor rows [128 j, 128 j + 128)
        } else if (type == U_GU) {
            un.cnt = blk_rows(a, i);
            un.nsub = 2;
            un.nst = a.pitch_d / 64 + (a.dense ? 0 : a.pitch_r / 64);
        } else if (type == U_DOWN) {
            un.nst = 1;  // the stage count unfolds block by block
            un.nsub = 1;
        }
        const bool mma_unit = type == U_T || type == U_GU || type == U_DOWN;
        if (mma_unit) un.acc = tmem_split(a) ? (type == U_DOWN ? 1 : 0) : (accseq++ & 1);
        if (pt == 0) {
            const int slot = seq % kUQ;
            S.uq[slot] = un;
            if (type == U_GU && !a.dense) {
                // the block's predictor bias, for the epilogue, long before it is needed
                const uint32_t bytes = static_cast<uint32_t>((un.cnt * 4 + 15) / 16 * 16);
                mbar_expect_tx(&S.bbar[slot], bytes);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        su32(&S.bias[slot][0])),
                    "l"(a.bias + static_cast<size_t>(i) * a.brows), "r"(bytes), "r"(su32(&S.bbar[slot]))
                    : "memory");
            }
            mbar_arrive(&S.uqf[slot]);
        }
        ++seq;
        if (type == U_STOP) break;
        if (type == U_PF) {
            // the NEXT layer's gate and up rows, the leading pf_bytes of each, into L2
            // while this layer's down units stream (HBM has headroom then): its GU units
            // find that share of their weights in L2. Slice i of the next layer's rows.
            const int nrows = a.pf_D, n0 = static_cast<int>(static_cast<int64_t>(i) * nrows / a.pf_units),
                      n1 = static_cast<int>(static_cast<int64_t>(i + 1) * nrows / a.pf_units);
            for (int q = n0 * 2 + pt; q < n1 * 2; q += kProdThreads) {
                const int n = q >> 1;
                const uint16_t* src = (q & 1) ? a.pf_ud + static_cast<size_t>(n) * 2 * a.pf_pitch
                                              : a.pf_gate + static_cast<size_t>(n) * a.pf_pitch;
                asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(src),
                             "r"(a.pf_bytes), "l"(pol_last)
                             : "memory");
            }
            continue;
        }
        if (!mma_unit) continue;

        uint8_t* As;
        uint32_t as;
        uint64_t* bar;
        if (type == U_T) {
            flush();
            const int k0 = i * a.kst;
            for (int st = 0; st < un.nst; ++st) {
                begin_stage(As, as, bar);
                if (pt == 0) mbar_expect_tx(bar, un.nsub * 16384u + bbytes);
                if (pt == 0) tma_tile_ef(As, &M.Bp, k0 + st * 64, j * 128, bar, pol);
                else if (pt == 1) tma_tile_ef(As + kStageA, &M.xhl, k0 + st * 64, 0, bar, pol_last);
                end_tile_stage(bar);
            }
        } else if (type == U_GU) {
            // gate rows (sub-tile 0) and up rows (sub-tile 1) of the block over all of K,
            // then (sparse) the block's predictor rows A against T^T
            flush();
            const int r0 = i * a.brows;
            for (int st = 0; st < a.pitch_d / 64; ++st) {
                begin_stage(As, as, bar);
                // (the three copies issued by three lanes of warp 0 side by side)
                if (pt == 0) mbar_expect_tx(bar, 2u * abytes + bbytes);
                if (pt < 3) {
                    if (pt == 0) tma_tile_ef(As, &M.gate, st * 64, r0, bar, pol);
                    else if (pt == 1) tma_tile_ef(As + 16384, &M.up, st * 64, r0, bar, pol);
                    else tma_tile_ef(As + kStageA, &M.xhl, st * 64, 0, bar, pol_last);
                }
                end_tile_stage(bar);
            }
            if (!a.dense) {
                wait_flag(fl_tr(a), t_halves(a));
                for (int st = 0; st < a.pitch_r / 64; ++st) {
                    begin_stage(As, as, bar);
                    if (pt == 0) mbar_expect_tx(bar, abytes + bbytes);
                    if (pt == 0) tma_tile_ef(As, &M.A, st * 64, r0, bar, pol);
                    else if (pt == 1) tma_tile_ef(As + kStageA, &M.thl, st * 64, 0, bar, pol_last);
                    end_tile_stage(bar);
                }
            }
        } else {  // U_DOWN: K = Z slots of the block range, A = down rows (MN-major)
            const int m0 = i * 128;
            DownWalk w = down_walk(a, j);
            DownStage ds;
            // the range's completion flags and counts, one round of loads for all blocks;
            // a block found incomplete is waited for, then the rest are read again
#ifdef SG_TC_FINTRACE
            unsigned long long nfetch = 0, fetch_ns = 0;
#endif
            auto fetch = [&] {
                prod_bar();
                const int blk = range_block(a, j, pt);
                S.dvc[pt] = (blk < a.nblk && flag_ready(fl_gu(a, blk), 1)) ? __ldcg(a.vcnt + blk) : -1;
                prod_bar();
            };
            fetch();
            auto wait_blk = [&](int k, int blk) {
                if (k >= kProdThreads) {
                    wait_flag(fl_gu(a, blk), 1);
                    return __ldcg(a.vcnt + blk);
                }
                if (S.dvc[k] < 0) {
#ifdef SG_TC_FINTRACE
                    const unsigned long long f0 = gtimer();
#endif
                    wait_flag(fl_gu(a, blk), 1);
                    fetch();
#ifdef SG_TC_FINTRACE
                    ++nfetch;
                    fetch_ns += gtimer() - f0;
#endif
                }
                return S.dvc[k];
            };
            int cnt = 0;
#ifdef SG_TC_FINTRACE
            int nstg = 0;
#endif
#ifdef SG_TC_FINTRACE
            unsigned long long walk_ns = 0;
            auto next = [&] {
                const unsigned long long w0 = gtimer();
                const bool r = down_next(a, w, ds, wait_blk);
                walk_ns += gtimer() - w0;
                return r;
            };
#else
            auto next = [&] { return down_next(a, w, ds, wait_blk); };
#endif
            while (next()) {
#ifdef SG_TC_FINTRACE
                if (pt == 0 && nstg++ == 0) TC_TRACE(a, un.u, 6, gtimer());
#endif
                if (ds.tiled) {
                    // rows by TMA tiles into 2 atoms of 64 outputs x kd k-rows (64-row boxes,
                    // 16-row boxes for the tail); Z: kd / 64 boxes of 64 slots
                    flush();
                    const int full = ds.rows / 64, nbox = (ds.rows % 64 + 15) / 16, nz = ds.kd / 64;
                    begin_stage(As, as, bar);
                    if (pt == 0) {
                        S.sinfo[spos] = StageInfo{(ds.rows + 15) / 16, ds.kd, 0};
                        mbar_expect_tx(bar, (a.dbg & 1 ? 0u : static_cast<uint32_t>(full * 8192 + nbox * 2048) * 2u) +
                                                (a.dbg & 2 ? 0u : nz * bbytes));
                    }
                    // one copy per lane of warp 0: lane q < 2 * per issues A box q % per of
                    // atom q / per (a full 128-row stage: one box per atom), the next nz
                    // lanes the Z boxes
                    const bool b128 = full == 2 && nbox == 0;
                    const int per = b128 ? 1 : full + nbox;
                    if (pt < 2 * per && !(a.dbg & 1)) {
                        const int atom = pt >= per, q = pt - atom * per;
                        uint8_t* dst = As + atom * ds.kd * 128;
                        if (b128)
                            tma_tile_ef(dst, &M.down128, m0 + atom * 64, ds.row0, bar, pol);
                        else if (q < full)
                            tma_tile_ef(dst + q * 8192, &M.down64, m0 + atom * 64, ds.row0 + q * 64, bar, pol);
                        else
                            tma_tile_ef(dst + full * 8192 + (q - full) * 2048, &M.down, m0 + atom * 64,
                                        ds.row0 + full * 64 + (q - full) * 16, bar, pol);
                    } else if (pt >= 2 * per && pt < 2 * per + nz && !(a.dbg & 2)) {
                        const int z = pt - 2 * per;
                        tma_tile_ef(As + kStageA + z * a.N * 128, &M.zhl, ds.row0 + z * 64, 0, bar, pol_last);
                    }
                    end_tile_stage(bar);
                    continue;
                }
                if (ds.c0 == 0) {  // a new gathered block: its survivor rows
                    cnt = w.g1;
                    prod_bar();  // the previous block's rows are no longer read
                    SG_CHECK(cnt <= kBlk && ds.gblk < a.nblk);
                    for (int k = pt; k < cnt; k += kProdThreads)
                        S.rows[k] = ds.gblk * a.brows + __ldcg(a.vlist + ds.gblk * kBlk + k);
                    prod_bar();
                }
                const int nz = ds.kd / 64, r16 = (ds.rows + 15) / 16 * 16;
                begin_stage(As, as, bar);
                if (pt == 0) {
                    S.sinfo[spos] = StageInfo{r16 / 16, ds.kd, 0};
                    mbar_expect_tx(bar, nz * bbytes);
                    for (int z = 0; z < nz; ++z)
                        tma_tile_ef(As + kStageA + z * a.N * 128, &M.zhl, ds.gblk * a.brows + ds.c0 + z * 64, 0, bar,
                                    pol_last);
                }
                // the stage's k-rows (to the next 16) x 2 atoms of 64 outputs, 16-B chunks;
                // rows past the block's survivors repeat its last row (finite data against
                // Z = 0: they add exact zeros)
#pragma unroll 4
                for (int q = pt; q < r16 * 16; q += kProdThreads) {
                    const int r = q >> 4, atom = (q >> 3) & 1, jj = q & 7;
                    const int row = S.rows[min(ds.c0 + r, cnt - 1)];
                    SG_CHECK(row >= 0 && row < a.D);
                    const uint16_t* src = a.ud + static_cast<size_t>(row) * 2 * a.pitch_d + a.pitch_d + m0 +
                                          atom * 64 + jj * 8;
                    cp16(as + atom * ds.kd * 128 + (r >> 3) * 1024 + (r & 7) * 128 + ((jj ^ (r & 7)) << 4), src, pol);
                }
                end_gather_stage();
            }
#ifdef SG_TC_FINTRACE
            if (pt == 0) TC_TRACE(a, un.u, 5, (static_cast<unsigned long long>(nstg) << 40) | (nfetch << 32) | fetch_ns);
            if (pt == 0) TC_TRACE(a, un.u, 7, walk_ns);
#endif
            // the terminating stage (no data) tells the MMA issuer the unit is complete
            flush();
            begin_stage(As, as, bar);
            if (pt == 0) {
                S.sinfo[spos] = StageInfo{0, 64, 1};
                mbar_arrive(bar);  // (the expect_tx arrival, with no bytes)
            }
            end_tile_stage(bar);
        }
#ifdef SG_TC_FINTRACE
        if (pt == 0) TC_TRACE(a, un.u, 2, ewait);
        ewait = 0;
#else
        if (pt == 0) TC_TRACE(a, un.u, 2, gtimer());
#endif
    }
    flush();
}

// ---- MMA issuer ----------------------------------------------------------------
__device__ void mma_issuer(const TcArgs& a, TcSmem& S, uint8_t* stages) {
    const int lane = threadIdx.x & 31;
    int seq = 0, stage = 0;
    uint32_t fphase = 0, tphase = 0;  // full[] / tempty[] phases
    int uses[2] = {0, 0};
    auto take_buffer = [&](int b) {
        if (uses[b] > 0) mbar_wait(&S.tempty[b], (tphase >> b) & 1u), tphase ^= 1u << b;
        uses[b]++;
    };
    // one smem stage: nsub A sub-tiles x ksteps K steps of 16 into columns dcol (+ t * N);
    // kd = K rows of the stage's layout (MN-major A atoms of 64 outputs x kd rows, K-major
    // B in kd / 64 atoms of 64 K)
    auto run_stage = [&](int nsub, int ksteps, bool mn, uint32_t dcol, uint32_t id, bool first, int kd = 64) {
        mbar_wait(&S.full[stage], (fphase >> stage) & 1u);
        fphase ^= 1u << stage;
        tc_fence_after();
        {
            const uint32_t As = su32(stages + stage * a.stage_bytes), Bs = As + kStageA;
            for (int t = 0; t < nsub; ++t)
                for (int k = 0; k < ksteps; ++k) {
                    // MN-major SW128: atoms of 64 outputs x 64 k-rows (8 KB); K-major SW128:
                    // rows of 128 B, 8-row groups of 1 KB
                    const uint64_t ad = mn ? sdesc(As + t * 16384 + k * 2048, kd * 128, 1024)
                                           : sdesc(As + t * 16384 + k * 32, 16, 1024);
                    const uint32_t bk = Bs + (k >> 2) * a.N * 128 + (k & 3) * 32;
                    umma_warp(dcol + t * a.N, ad, sdesc(bk, 16, 1024), id, (first && k == 0) ? 0u : 1u);
                }
            umma_commit_warp(&S.empty[stage]);
        }
        __syncwarp();
        stage = stage + 1 == a.nstages ? 0 : stage + 1;
    };
    for (;;) {
        const int slot = seq % kUQ;
        mbar_wait(&S.uqf[slot], (seq / kUQ) & 1);
        const Unit un = S.uq[slot];
        ++seq;
        const bool mma_unit = un.type == U_T || un.type == U_GU || un.type == U_DOWN;
        if (mma_unit) {
            const int acc = un.acc;
            take_buffer(acc);
            tc_fence_after();
            const uint32_t dcol = S.tmem + acc_base(a, acc);
            if (un.type == U_T) {
                for (int st = 0; st < un.nst; ++st) run_stage(un.nsub, 4, false, dcol, idesc(a.N, 0), st == 0);
            } else if (un.type == U_GU) {
                const int ngu = a.pitch_d / 64;
                for (int st = 0; st < ngu; ++st) run_stage(2, 4, false, dcol, idesc(a.N, 0), st == 0);
                for (int st = ngu; st < un.nst; ++st)  // pre = A T into columns 2N..3N
                    run_stage(1, 4, false, dcol + 2 * a.N, idesc(a.N, 0), st == ngu);
            } else {
                // down: the producer's stages in order, each with its K steps (StageInfo),
                // until the terminating one
                for (int st = 0;; ++st) {
                    mbar_wait(&S.full[stage], (fphase >> stage) & 1u);
                    const StageInfo si = S.sinfo[stage];
                    if (si.last) {
                        fphase ^= 1u << stage;
                        if (lane == 0) mbar_arrive(&S.empty[stage]);
                        __syncwarp();
                        stage = stage + 1 == a.nstages ? 0 : stage + 1;
                        break;
                    }
                    run_stage(1, a.dbg & 4 ? 0 : si.ksteps, true, dcol, idesc(a.N, 1), st == 0, si.kd);
                }
            }
            if (lane == 0) {
                umma_commit(&S.tfull[acc]);
            }
            __syncwarp();
        }
        if (lane == 0) mbar_arrive(&S.uqe[slot]);
        if (un.type == U_STOP) break;
    }
}

// ---- epilogue helpers ------------------------------------------------------------
// hi + lo accumulator columns of this thread's TMEM lane (row) for tokens c0..c0+15
// of sub-tile column block t (columns t*N ..): four tcgen05.ld back to back, one wait
// (tokens >= nb read unused columns, ignored by the callers).
__device__ __forceinline__ void acc16(const TcArgs& a, uint32_t tbase, int quarter, int accbuf, int t, int c0,
                                      float* v) {
    float h[16], l[16];
    const uint32_t addr = tbase + (static_cast<uint32_t>(quarter * 32) << 16) +
                          acc_base(a, accbuf) + static_cast<uint32_t>(t * a.N + c0);
    tmem_ld8(addr, h);
    tmem_ld8(addr + 8u, h + 8);
    tmem_ld8(addr + static_cast<uint32_t>(a.nb), l);
    tmem_ld8(addr + static_cast<uint32_t>(a.nb) + 8u, l + 8);
    tmem_wait();
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = h[e] + l[e];
}
__device__ __forceinline__ void st16(float* p, const float* v, int n) {  // n in {8, 16}
#pragma unroll
    for (int q = 0; q < 4; ++q)
        if (4 * q < n) reinterpret_cast<float4*>(p)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
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

// Store E (8 or 16) tokens' hi / lo values of this thread's row `slot` (v[e] for
// token c + e; slot < 0: none) — or, for `zslot`, exact zeros — into the K-major bf16
// rows dst[(c + e) * pitch + slot] (hi) and dst[(nb + c + e) * pitch + slot] (lo),
// slots [0, nslots), through smem so the global stores are whole 16-B runs of 8 slots.
template <int E>
__device__ __forceinline__ void store_hilo(TcSmem& S, int et, const float* v, int slot, int zslot, uint16_t* dst,
                                           size_t pitch, int nb, int c, int nslots) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
        uint16_t hi, lo;
        split_bf16(v[e], hi, lo);
        if (slot >= 0) S.zst[0][e][slot] = hi, S.zst[1][e][slot] = lo;
        if (zslot >= 0) S.zst[0][e][zslot] = 0, S.zst[1][e][zslot] = 0;
    }
    epi_bar();
    const int chunks = nslots / 8;
    for (int w = et; w < 2 * E * chunks; w += 128) {
        const int row = w / chunks, ch = w % chunks, hl = row / E, e = row % E;
        const uint4 q = *reinterpret_cast<const uint4*>(&S.zst[hl][e][ch * 8]);
        SG_CHECK(ch * 8 + 8 <= kBlk && hl * nb + c + e < 2 * nb);
        *reinterpret_cast<uint4*>(dst + static_cast<size_t>(hl * nb + c + e) * pitch + ch * 8) = q;
    }
    epi_bar();
}

// ---- epilogue -----------------------------------------------------------------
__device__ void epilogue(const TcArgs& a, TcSmem& S) {
    const int et = threadIdx.x - kEpiBase;     // 0..127
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int quarter = warp & 3;              // TMEM lane quarter of this warp
    int seq = 0;
    uint32_t tphase = 0, bphase = 0;  // tfull[] / bbar[] phases
    const uint64_t bmask = a.B >= 64 ? ~0ull : ((1ull << a.B) - 1ull);
    const int nb = a.nb;
    auto wait_acc = [&](int b) {
        mbar_wait(&S.tfull[b], (tphase >> b) & 1u);
        tphase ^= 1u << b;
    };
    for (;;) {
        const int slot = seq % kUQ;
        mbar_wait(&S.uqf[slot], (seq / kUQ) & 1);
        const Unit un = S.uq[slot];
        ++seq;
        if (un.type == U_STOP) break;
        const int i = un.a, j = un.b;
        const bool mma_unit = un.type == U_T || un.type == U_GU || un.type == U_DOWN;
        if (mma_unit) {
            wait_acc(un.acc);
            tc_fence_after();
        }
        if (et == 0) TC_TRACE(a, un.u, 3, gtimer());
        const int row0 = quarter * 32 + lane;  // this thread's row of the M = 128 tile
        const int acc = un.acc;
        auto release = [&] {  // the unit's TMEM buffers are free again
            tc_fence_before();
            epi_bar();
            if (et == 0) {
                mbar_arrive(&S.tempty[acc]);
            }
        };

        if (un.type == U_X) {
            // x (fp32 [B][d]) -> X^T hi rows 0..nb-1, lo rows nb..2nb-1 (bf16 [N][xpitch]):
            // this unit's share of the (token, 8-column chunk) items, 4 per thread per
            // round of loads
            const int nch = a.pitch_d / 8, items = nb * nch;
            const int per = (items + a.u_T - 1) / a.u_T;
            const int w0 = i * per, w1 = min(items, w0 + per);
            bool bad = false;
            const bool vec = (a.d & 7) == 0;
            for (int wb = w0 + et; wb < w1; wb += 4 * 128) {
                float v[4][8];
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const int w = wb + h * 128;
                    const int b = w / nch, k0 = (w % nch) * 8;
                    if (w < w1 && b < a.B && vec && k0 < a.d) {
                        const float4* src = reinterpret_cast<const float4*>(a.x + static_cast<size_t>(b) * a.d + k0);
                        float4 f0 = __ldg(src), f1 = __ldg(src + 1);
                        if (a.xres) {  // residual input: x = h + r, summed in fp32 before the split
                            const float4* rs = reinterpret_cast<const float4*>(a.xres + static_cast<size_t>(b) * a.d + k0);
                            const float4 r0 = __ldcg(rs), r1 = __ldcg(rs + 1);
                            f0.x += r0.x; f0.y += r0.y; f0.z += r0.z; f0.w += r0.w;
                            f1.x += r1.x; f1.y += r1.y; f1.z += r1.z; f1.w += r1.w;
                        }
                        v[h][0] = f0.x; v[h][1] = f0.y; v[h][2] = f0.z; v[h][3] = f0.w;
                        v[h][4] = f1.x; v[h][5] = f1.y; v[h][6] = f1.z; v[h][7] = f1.w;
                    } else {
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            const bool in = w < w1 && b < a.B && k0 + e < a.d;
                            const size_t o = static_cast<size_t>(b) * a.d + k0 + e;
                            v[h][e] = in ? __ldg(a.x + o) + (a.xres ? __ldcg(a.xres + o) : 0.f) : 0.f;
                        }
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
            // partial T^T of predictor rows [128 j, 128 j + 128) over K slice i ->
            // tpart[i][row][b]; the last slice of the half to finish sums its KT partials in
            // slice order (its own straight from TMEM) -> T^T hi / lo (the B operand of the
            // GU units' predictor MMA), zero past the rank
            const int KT = a.kt, row = j * 128 + row0;
            for (int c = 0; c < nb; c += 16) {
                float v[16];
                acc16(a, S.tmem, quarter, acc, 0, c, v);
                st16(a.tpart + (static_cast<size_t>(i) * kTRows + row) * nb + c, v, min(16, nb - c));
            }
            epi_bar();
            if (arrive_last(fl_t(a, j), KT, S, et)) {
                const float* src = a.tpart + static_cast<size_t>(row) * nb;
                const uint32_t tl = S.tmem + (static_cast<uint32_t>(quarter * 32) << 16) + acc_base(a, acc);
                for (int c = 0; c < nb; c += 8) {
                    // the other slices' loads first, then this slice's TMEM columns
                    float4 q[4][2];
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (k < KT && k != i && row < a.r) {
                            const float4* p = reinterpret_cast<const float4*>(src + static_cast<size_t>(k) * kTRows * nb + c);
                            q[k][0] = __ldcg(p);
                            q[k][1] = __ldcg(p + 1);
                        }
                    float h[8], l[8], s[8];
                    tmem_ld8(tl + c, h);
                    tmem_ld8(tl + nb + c, l);
                    tmem_wait();
#pragma unroll
                    for (int k = 0; k < 4; ++k) {  // fixed order: slices 0, 1, ... (own at i)
                        if (k >= KT) break;
                        const float v[8] = {q[k][0].x, q[k][0].y, q[k][0].z, q[k][0].w,
                                            q[k][1].x, q[k][1].y, q[k][1].z, q[k][1].w};
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            const float t = k == i ? h[e] + l[e] : v[e];
                            s[e] = k == 0 ? t : s[e] + t;
                        }
                    }
                    if (row >= a.r)
#pragma unroll
                        for (int e = 0; e < 8; ++e) s[e] = 0.f;
                    store_hilo<8>(S, et, s, row0, -1, a.thl + j * 128, 256, nb, c, 128);
                }
                asm volatile("fence.proxy.async.global;" ::: "memory");  // T^T is read by TMA
                epi_bar();
                if (et == 0) signal(fl_tr(a));
            }
            release();
        } else if (un.type == U_GU) {
            // block i: g (columns 0..N), u (N..2N), pre (2N..3N, sparse) of this thread's
            // row; mask P_b = pre + bias > 0 (ffn_exec.hpp:141), survivors V_b = P_b &
            // g > 0 (:200), z = gated(g, u) on V_b, else +0. (The per-token counts are
            // the bit columns' popcounts, taken when the host reads the stats.)
            const int cnt = un.cnt, k = row0;
            const bool mine = k < cnt;
            const int n = i * a.brows + k;
            float bias = 0.f;
            if (!a.dense) {  // (bulk-copied to smem when the unit was queued)
                mbar_wait(&S.bbar[slot], (bphase >> slot) & 1u);
                bphase ^= 1u << slot;
                if (mine) bias = S.bias[slot][k];
            }
            const uint32_t tl = S.tmem + (static_cast<uint32_t>(quarter * 32) << 16) + acc_base(a, acc);
            float z[64];
            uint64_t mb = 0, sbits = 0;
#pragma unroll
            for (int c = 0; c < 64; c += 16) {
#pragma unroll
                for (int e = 0; e < 16; ++e) z[c + e] = 0.f;
                if (c >= nb) continue;  // uniform
                // this chunk's g, u (and pre) hi + lo columns: all loads, one wait
                float gh[16], gl[16], uh[16], ul[16], ph[16], pl[16];
                tmem_ld16(tl + c, gh);
                tmem_ld16(tl + nb + c, gl);
                tmem_ld16(tl + a.N + c, uh);
                tmem_ld16(tl + a.N + nb + c, ul);
                if (!a.dense) {
                    tmem_ld16(tl + 2 * a.N + c, ph);
                    tmem_ld16(tl + 2 * a.N + nb + c, pl);
                }
                tmem_wait();
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const bool pm = a.dense || (ph[e] + pl[e]) + bias > 0.f;
                    const float g = gh[e] + gl[e], u = uh[e] + ul[e];
                    if (pm) mb |= 1ull << (c + e);
                    const bool sv = pm && g > 0.f;
                    if (sv) sbits |= 1ull << (c + e);
                    z[c + e] = sv ? gated(g, u, a.act) : 0.f;
                }
            }
            release();
#ifdef SG_TC_FINTRACE
            if (et == 0) TC_TRACE(a, un.u, 5, gtimer());
#endif
            mb = mine ? (mb & bmask) : 0ull;
            sbits = mine ? (sbits & bmask) : 0ull;
            SG_CHECK(!mine || n < a.D);
            if (mine) {
                a.vbits[n] = sbits;
                if (!a.dense) a.mbits[n] = mb;
            }
            // survivor slots: ascending rows
            const bool keep = sbits != 0;
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (lane == 0) S.wsum[quarter] = __popc(bal);
            epi_bar();
            int before = 0;
            for (int q = 0; q < quarter; ++q) before += S.wsum[q];
            const int nv = S.wsum[0] + S.wsum[1] + S.wsum[2] + S.wsum[3];
            const int slot_c = before + __popc(bal & ((1u << lane) - 1u));
#ifdef SG_TC_FINTRACE
            if (et == 0) TC_TRACE(a, un.u, 6, gtimer());
#endif
            // DOWN streams the block whole (Z slot = row) when its survivors are dense
            // enough, else gathers the survivor rows (Z slot = survivor position); the
            // slots up to the next 16 are exact zeros either way
            const bool dtile = nv > 0 && down_tiled(a, nv, i);
            const int pad_to = dtile ? (cnt + 15) / 16 * 16 : (nv + 15) / 16 * 16;
            SG_CHECK(static_cast<size_t>(i) * a.brows + pad_to <= static_cast<size_t>(a.zpitch));
            int zslot = -1, pslot = -1;
            if (dtile) {
                if (mine) zslot = k;
                else if (k < pad_to) pslot = k;
            } else {
                if (keep) {
                    zslot = slot_c;
                    SG_CHECK(slot_c < cnt && i < a.nblk);
                    a.vlist[i * kBlk + slot_c] = k;
                }
                if (k >= nv && k < pad_to) pslot = k;
            }
#pragma unroll
            for (int c = 0; c < 64; c += 16) {
                if (c >= nb) continue;  // uniform
                if (c + 16 <= nb)
                    store_hilo<16>(S, et, z + c, zslot, pslot, a.zhl + static_cast<size_t>(i) * a.brows, a.zpitch, nb,
                                   c, pad_to);
                else
                    store_hilo<8>(S, et, z + c, zslot, pslot, a.zhl + static_cast<size_t>(i) * a.brows, a.zpitch, nb,
                                  c, pad_to);
            }
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
        } else if (un.type == U_DOWN) {
            // partial y over block range j for d tile i (128 outputs): ypart[j][m][b]; the
            // last range of the d tile to finish sums the S partials in range order into y
            const int m = i * 128 + row0;
            bool have;
            {  // did the range hold any survivor row (else the accumulator was never written)
                int hv = 0;
                for (int k = et, blk; (blk = range_block(a, j, k)) < a.nblk; k += 128)
                    hv |= vcnt_rows(__ldcg(a.vcnt + blk)) > 0;
                have = epi_bar_or(hv);
            }
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
            release();
#ifndef SG_TC_FINTRACE
            if (et == 0) TC_TRACE(a, un.u, 6, gtimer());
#endif
            if (arrive_last(fl_down(a, i), a.S, S, et)) {
                // y rows of d tile i: the S range partials in range order, 2 chunks of 8
                // tokens per round of loads
                bool xbad = false;
                const size_t rs = static_cast<size_t>(a.ndt) * 128 * nb;
                const float* rowp = a.ypart + static_cast<size_t>(m) * nb;
                for (int c0 = 0; c0 < nb; c0 += 16) {
                    float4 q[4][2][2];
                    float nv[16];  // (prep) the next launch's residual input, same round of loads
#pragma unroll
                    for (int r = 0; r < 4; ++r)
#pragma unroll
                        for (int h = 0; h < 2; ++h)
                            if (r < a.S && c0 + 8 * h < nb && m < a.d) {
                                const float4* src = reinterpret_cast<const float4*>(rowp + r * rs + c0 + 8 * h);
                                q[r][h][0] = __ldcg(src);
                                q[r][h][1] = __ldcg(src + 1);
                            }
#pragma unroll
                    for (int e = 0; e < 16; ++e)
                        nv[e] = (a.prep && a.nh && c0 + e < a.B && m < a.d)
                                    ? __ldcg(a.nh + static_cast<size_t>(c0 + e) * a.d + m)
                                    : 0.f;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int c = c0 + 8 * h;
                        if (c >= nb) continue;
                        float y[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                        if (m < a.d) {
#pragma unroll
                            for (int r = 0; r < 4; ++r)  // fixed order: ranges 0, 1, ..., S-1
                                if (r < a.S) {
                                    y[0] += q[r][h][0].x; y[1] += q[r][h][0].y; y[2] += q[r][h][0].z; y[3] += q[r][h][0].w;
                                    y[4] += q[r][h][1].x; y[5] += q[r][h][1].y; y[6] += q[r][h][1].z; y[7] += q[r][h][1].w;
                                }
#pragma unroll
                            for (int e = 0; e < 8; ++e)
                                if (c + e < a.B) a.y[static_cast<size_t>(c + e) * a.d + m] = y[e];
                        }
                        if (a.prep) {
                            // the NEXT launch's X^T column m: x = h_next + y (h_next may be
                            // absent: x = y), split into bf16 hi / lo through smem staging —
                            // the next launch then runs no X units (every GU unit of this
                            // launch has finished)
                            float xv[8];
#pragma unroll
                            for (int e = 0; e < 8; ++e) {
                                const int b = c + e;
                                xv[e] = 0.f;
                                if (b < a.B && m < a.d) xv[e] = y[e] + nv[8 * h + e];
                                xbad |= !isfinite(xv[e]);
                            }
                            store_hilo<8>(S, et, xv, row0, -1, a.xhl + static_cast<size_t>(i) * 128, a.xpitch, nb, c,
                                          min(128, a.pitch_d - i * 128));
                        }
                    }
                }
                if (xbad) atomicOr(a.bad + 2, 1);  // the next launch's check_input
            }
        }
        if (et == 0) {
            TC_TRACE(a, un.u, 4, gtimer());
            mbar_arrive(&S.uqe[slot]);
        }
    }
}

__global__ void __launch_bounds__(kTcThreads, 1) tc_kernel(const __grid_constant__ TcMaps maps, const TcArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // [TcSmem | ring of a.nstages x a.stage_bytes], the ring 1024-B aligned (SW128 atoms)
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    TcSmem& S = *reinterpret_cast<TcSmem*>(base);
    uint8_t* stages = base + kTcSmemPad;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int s = 0; s < a.nstages; ++s) {
            mbar_init(&S.full[s], kFullArrivals);
            mbar_init(&S.empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&S.tfull[s], 1);
            mbar_init(&S.tempty[s], 1);
        }
        for (int s = 0; s < kUQ; ++s) {
            mbar_init(&S.uqf[s], 1);
            mbar_init(&S.uqe[s], 2);
            mbar_init(&S.bbar[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x == 32) {  // warm the TMA descriptor cache with every map this CTA may use
        const CUtensorMap* ms[] = {&maps.xhl, &maps.thl, &maps.zhl, &maps.Bp, &maps.A,
                                   &maps.gate, &maps.up, &maps.down, &maps.down64, &maps.down128};
        for (const CUtensorMap* m : ms)
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
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
        for (int s = 0; s < a.nstages; ++s) mbar_arrive(&S.empty[s]);
    // (programmatic dependent launch: everything above overlapped the previous launch's
    // tail; from here on the previous launch's outputs and counters are read)
    asm volatile("griddepcontrol.wait;" ::: "memory");
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
    if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" :::);
    if (warp == kMmaWarp) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(S.tmem));
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(fl_exit(a), 1) == static_cast<int>(gridDim.x) - 1) {
            // last CTA out: every other CTA has finished; reset the dataflow counters and
            // publish the non-finite flag (read by sg_ctx_read_batch), zero for the next
            __threadfence();
            for (int k = 0; k < flag_count(a); ++k) a.flags[k] = 0;
            // bad: [0] this launch's x, [1] published, [2] the x this launch prepared for
            // the next one, [3] that flag carried into the next launch
            a.bad[1] = __ldcg(a.bad) | (a.x_ready ? __ldcg(a.bad + 3) : 0);
            a.bad[0] = 0;
            a.bad[3] = __ldcg(a.bad + 2);
            a.bad[2] = 0;
            __threadfence();
        }
    }
}

}  // namespace

int tc_block_rows(int64_t D, int sms) {
    constexpr int kReserve = 4;  // SMs left beside one GU block per SM (the T units)
    const int64_t g = sms > kReserve + 1 ? sms - kReserve : 1;
    const int64_t per = ((D + g - 1) / g + 15) / 16 * 16;  // multiple of 16: one MMA K step
    return static_cast<int>(per > kBlk ? kBlk : per);
}

int tc_smem_bytes(int nstages, int stage_bytes) { return 1024 + kTcSmemPad + nstages * stage_bytes; }

// the smem ring for MMA N: stages of the two A tiles + the larger B operand of a stage
// (the GU / T token tile of N rows x 64 K, or a down stage's Z tile of kd = 128 slots x N
// when N <= 64), as many as the opt-in shared memory holds (SG_TC_STAGES caps it)
void tc_ring(TcArgs& a) {
    const int bneed = (a.N <= 64 ? 2 : 1) * a.N * 128;
    a.stage_bytes = kStageA + (bneed + 1023) / 1024 * 1024;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const char* cap = std::getenv("SG_TC_STAGES");
    int ns = (optin - 1024 - kTcSmemPad) / a.stage_bytes;
    ns = std::min({ns, kStagesMax, cap ? std::atoi(cap) : kStagesMax});
    a.nstages = std::max(kLag + 1, ns);  // (a producer thread holds kLag stages back)
}
int tc_flag_ints(int nblk, int ndt) { return 32 + nblk + ndt; }

int launch_batch_tc(const TcMaps& maps, const TcArgs& a_in, int grid, void* stream) {
    TcArgs a = a_in;
    tc_ring(a);
    const int smem = tc_smem_bytes(a.nstages, a.stage_bytes);
    const int e = ensure_smem_attr(reinterpret_cast<const void*>(tc_kernel), smem);
    if (e) return e;
    // programmatic dependent launch (SG_TC_PDL=0 disables): the next launch on the
    // stream sets up its CTAs while this one drains
    static const bool pdl = [] {
        const char* e = std::getenv("SG_TC_PDL");
        return e == nullptr || std::atoi(e) != 0;
    }();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kTcThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, tc_kernel, maps, a);
    return static_cast<int>(cudaGetLastError());
}

}  // namespace sg
