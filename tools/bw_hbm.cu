// HBM streaming-rate probe for the batched tensor-core kernel's weight layouts (the
// matrices are 4x the L2, so every byte comes from HBM). 148 CTAs, one producer
// lane issuing into a ring of `stages` x 32 KB, one consumer warp releasing stages.
//   mode 0: GU pattern, row-major [D][K] weights: per stage two 2-D boxes of 128 rows x
//           64 K (128 B of each 8-KB row), the unit walks K for a 128-row block
//   mode 1: the same bytes pre-packed tile by tile (each 16-KB box contiguous in HBM):
//           two 1-D cp.async.bulk of 16 KB per stage
//   mode 2: DOWN pattern on the interleaved [D][2*4096] up|down rows: boxes of 64 rows
//           x 64 outputs (128 B of each 16-KB row), four per stage
//   mode 3: DOWN pre-packed d-tile-major ([tile][D][128 outputs]): one 32-KB bulk copy
//   mode 4: the batch kernel's DOWN units: CTA c < 128 streams d tile c % 32 (128
//           outputs) over row range c / 32 of 4, 128-row stages (2 atoms x 2 boxes of
//           64 rows), as the tcgen05 kernel does
//   mode 5: as 4 with d tiles of 256 outputs (64 units of 4 atoms)
//   mode 6: as 4, but the 32 units of a range start their row walk at staggered rows
//           (no two SMs read the same rows at the same time)
// Prints GB/s per mode and ring depth.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/bw_hbm.cu -o tools/bw_hbm
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
            su32(b)),
        "r"(par)
        : "memory");
}
__device__ __forceinline__ void tile(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            su32(dst)),
        "l"(m), "r"(c0), "r"(c1), "r"(su32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(bar))
                 : "memory");
}

struct Maps {
    CUtensorMap gate, up, down;
};
constexpr int kStage = 32768, kMaxStages = 6;
constexpr int D = 4 * 11008 / 128 * 128, K = 4096;  // 4 layers' worth of rows: 4x the L2

__global__ void __launch_bounds__(64, 1) stream(const __grid_constant__ Maps M, int mode, int nst, const char* packed,
                                              unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[kMaxStages], empty[kMaxStages];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // work: mode 0/1: (128-row block, 64-K chunk) stages, both matrices; 2/3: (64-row
    // group, 256-output half-tile) stages
    int total = (mode < 2) ? (D / 256) * (K / 64) : (D / 64) * (K / 256);
    if (mode >= 4) total = 0;
    int n = 0;
    if (mode >= 4) {  // unit-major DOWN streaming: rows of one range, one column slab
        const bool stag = mode == 6;
        if (mode == 6) mode = 4;
        const int tiles = mode == 4 ? 32 : 16, atoms = mode == 4 ? 2 : 4;
        const int c = blockIdx.x;
        if (c < tiles * 4) {
            const int dt = c % tiles, rg = c / tiles, rows = D / 4, r0 = rg * rows;
            const int nstage = rows / (mode == 4 ? 128 : 64);
            if (warp == 0 && lane == 0) {
                for (int st0 = 0; st0 < nstage; ++st0, ++n) {
                    const int st = stag ? (st0 + dt * nstage / tiles) % nstage : st0;
                    const int s = n % nst;
                    if (n >= nst) mbar_wait(&empty[s], ((n / nst) - 1) & 1);
                    uint8_t* dst = sm + s * kStage;
                    mbar_expect_tx(&full[s], kStage);
                    for (int a = 0; a < atoms; ++a)
                        for (int f = 0; f < (mode == 4 ? 2 : 1); ++f)
                            tile(dst + a * (mode == 4 ? 16384 : 8192) + f * 8192, &M.down, dt * atoms * 64 + a * 64,
                                 r0 + st * (mode == 4 ? 128 : 64) + f * 64, &full[s]);
                }
            } else if (warp == 1) {
                unsigned long long acc = 0;
                for (int st = 0; st < nstage; ++st, ++n) {
                    const int s = n % nst;
                    mbar_wait(&full[s], (n / nst) & 1);
                    acc += sm[s * kStage + lane * 64];
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[s]);
                }
                if (lane == 0) atomicAdd(sink, acc);
            }
        }
    } else if (warp == 0 && lane == 0) {
        for (int u = blockIdx.x; u < total; u += gridDim.x, ++n) {
            const int s = n % nst;
            if (n >= nst) mbar_wait(&empty[s], ((n / nst) - 1) & 1);
            uint8_t* dst = sm + s * kStage;
            mbar_expect_tx(&full[s], kStage);
            if (mode == 0) {
                const int blk = u / (K / 64), kc = (u % (K / 64)) * 64;
                tile(dst, &M.gate, kc, blk * 128, &full[s]);
                tile(dst + 16384, &M.up, kc, blk * 128, &full[s]);
            } else if (mode == 1) {
                bulk(dst, packed + static_cast<size_t>(u) * 32768, 16384, &full[s]);
                bulk(dst + 16384, packed + static_cast<size_t>(u) * 32768 + 16384, 16384, &full[s]);
            } else if (mode == 2) {
                const int g = u / (K / 256), m0 = (u % (K / 256)) * 256;
                for (int a = 0; a < 4; ++a) tile(dst + a * 8192, &M.down, m0 + a * 64, g * 64, &full[s]);
            } else {
                bulk(dst, packed + static_cast<size_t>(u) * 32768, 32768, &full[s]);
            }
        }
    } else if (warp == 1) {
        unsigned long long acc = 0;
        for (int u = blockIdx.x; u < total; u += gridDim.x, ++n) {
            const int s = n % nst;
            mbar_wait(&full[s], (n / nst) & 1);
            acc += sm[s * kStage + lane * 64];
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        if (lane == 0) atomicAdd(sink, acc);
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    const size_t mat = size_t(D) * K * 2;  // one [D][K] bf16 matrix
    char *gate, *ud, *packed;
    cudaMalloc(&gate, mat);
    cudaMalloc(&ud, 2 * mat);
    cudaMalloc(&packed, 2 * mat);
    cudaMemset(gate, 1, mat);
    cudaMemset(ud, 1, 2 * mat);
    cudaMemset(packed, 1, 2 * mat);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<EncodeFn>(f);
    Maps M;
    auto mk = [&](CUtensorMap* m, void* base, uint64_t cols, uint64_t rows, uint64_t stride_el, uint32_t box_rows) {
        cuuint64_t dims[2] = {cols, rows};
        cuuint64_t st[1] = {stride_el * 2};
        cuuint32_t box[2] = {64, box_rows}, es[2] = {1, 1};
        CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) std::printf("encode failed %d\n", int(r));
    };
    mk(&M.gate, gate, K, D / 2, K, 128);                 // gate half of the rows
    mk(&M.up, gate + mat / 2, K, D / 2, K, 128);         // "up": the other half (same bytes total)
    mk(&M.down, ud + K * 2, K, D, 2 * K, 64);            // down rows of the interleaved matrix
    const int smem = kMaxStages * kStage + 1024;
    cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const char* names[] = {"GU row-major 2x box{64,128}", "GU packed 2x bulk 16KB", "DOWN interleaved 4x box{64,64}",
                           "DOWN packed bulk 32KB", "DOWN units 32 tiles x 4 ranges", "DOWN units 16 tiles x 4 ranges",
                           "DOWN units staggered rows"};
    for (int mode = 0; mode < 7; ++mode) {
        for (int nst : {4, 6}) {
            // modes 0/1 read gate+up halves (D/2 rows each x K) = mat bytes; 2/3 the down half of ud = mat
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            stream<<<148, 64, smem>>>(M, mode, nst, packed, sink);
            cudaEventRecord(a);
            const int it = 3;
            for (int k = 0; k < it; ++k) stream<<<148, 64, smem>>>(M, mode, nst, packed, sink);
            cudaEventRecord(b);
            cudaError_t e = cudaDeviceSynchronize();
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            const double bytes = double(it) * (mode < 2 ? (size_t(D) / 256) * (K / 64) : (size_t(D) / 64) * (K / 256)) * kStage;
            // (modes 4/5 move the same bytes: every down row once)
            std::printf("%-32s stages %d: %8.1f GB/s  (%s)\n", names[mode], nst, bytes / (ms * 1e-3) / 1e9,
                        cudaGetErrorString(e));
        }
    }
    return 0;
}
