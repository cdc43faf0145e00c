// TMA streaming-rate probe for the batched tensor-core kernel's load patterns:
// every CTA streams its share of a D x K bf16 weight matrix (K = 4096, the 7B
// gate shape) through a 4-stage ring of 32 KB stages (256 rows x 64 K), either
//   mode 0: two 2-D tile boxes of 128 rows x 64 K per stage,
//   mode 1: 64 tile::gather4 (4 rows x 64 K each) per stage, issued by 32 lanes,
//   mode 2: the same 64 gather4 issued by one lane,
//   mode 3: gather4 of a permuted (random) row order, 32 lanes,
//   mode 4: 32 2-D boxes of 8 rows x 64 K per stage (32 lanes)
//   mode 5: 16-B cp.async from 128 threads (random rows, 128-B swizzled placement),
//           each thread arriving on the stage barrier after cp.async.wait_group + proxy fence
//   mode 6: as 5 without the proxy fence
//   mode 7: as 5 but arriving through cp.async.mbarrier.arrive.noinc (no wait, no fence)
// and a consumer warp releases each stage as soon as it lands. Prints GB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/bw_tma.cu -o tools/bw_tma
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

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
__device__ __forceinline__ void g4(void* dst, const CUtensorMap* m, int c0, int r0, int r1, int r2, int r3,
                                   uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
            su32(dst)),
        "l"(m), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(bar))
        : "memory");
}

struct Maps {
    CUtensorMap box128, box1, box8;
};

constexpr int kStages = 4, kStage = 32768;

__global__ void __launch_bounds__(160, 1) stream(const __grid_constant__ Maps M, int D, int K, int mode,
                                               const int* perm, unsigned long long* sink, const void* gw) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[kStages], empty[kStages];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const bool cpa = mode >= 5;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], cpa ? 128 : 1);
            mbar_init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int blocks = D / 256, kch = K / 64;
    const int units = blocks * kch;  // (256-row block, 64-K chunk) stage units
    int n = 0;
    if (cpa && warp < 4) {
        const int pt = threadIdx.x;
        const uint16_t* W = reinterpret_cast<const uint16_t*>(gw);
        int pend = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++n) {
            const int s = n % kStages;
            if (n >= kStages) mbar_wait(&empty[s], ((n / kStages) - 1) & 1);
            const uint32_t dst = su32(sm + s * kStage);
            const int r0 = (u / kch) * 256, kc = (u % kch) * 64, jj = pt & 7;
            for (int r = pt >> 3; r < 256; r += 16) {
                const uint16_t* src = W + static_cast<size_t>(perm[r0 + r]) * K + kc + jj * 8;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + (r >> 3) * 1024 + (r & 7) * 128 + ((jj ^ (r & 7)) << 4)), "l"(src) : "memory");
            }
            if (mode == 7) {
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[s])) : "memory");
                continue;
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            if (++pend > 2) {
                asm volatile("cp.async.wait_group 2;" ::: "memory");
                if (mode == 5) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive(&full[(n - 2) % kStages]);
                --pend;
            }
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        for (; pend > 0; --pend) mbar_arrive(&full[(n - pend) % kStages]);
    } else if (!cpa && warp == 0) {
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++n) {
            const int s = n % kStages;
            if (n >= kStages) mbar_wait(&empty[s], ((n / kStages) - 1) & 1);
            uint8_t* dst = sm + s * kStage;
            const int r0 = (u / kch) * 256, kc = (u % kch) * 64;
            if (lane == 0) mbar_expect_tx(&full[s], kStage);
            __syncwarp();
            if (mode == 0) {
                if (lane == 0) {
                    tile(dst, &M.box128, kc, r0, &full[s]);
                    tile(dst + 16384, &M.box128, kc, r0 + 128, &full[s]);
                }
            } else if (mode == 4) {
                tile(dst + lane * 1024, &M.box8, kc, r0 + lane * 8, &full[s]);
            } else {
                for (int g = (mode == 2 ? 0 : lane); g < 64; g += (mode == 2 ? 1 : 32)) {
                    if (mode == 2 && lane != 0) break;
                    int r[4];
                    for (int q = 0; q < 4; ++q) {
                        const int row = r0 + 4 * g + q;
                        r[q] = mode == 3 ? perm[row] : row;
                    }
                    g4(dst + g * 512, &M.box1, kc, r[0], r[1], r[2], r[3], &full[s]);
                }
            }
            __syncwarp();
        }
    } else if (warp == (cpa ? 4 : 1)) {
        unsigned long long acc = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++n) {
            const int s = n % kStages;
            mbar_wait(&full[s], (n / kStages) & 1);
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

int main(int argc, char** argv) {
    setvbuf(stdout, nullptr, _IONBF, 0);
    const int D = 11008 / 256 * 256, K = 4096;
    void* w;
    cudaMalloc(&w, size_t(D) * K * 2);
    cudaMemset(w, 1, size_t(D) * K * 2);
    std::vector<int> perm(D);
    for (int i = 0; i < D; ++i) perm[i] = i;
    srand(1);
    for (int i = D - 1; i > 0; --i) std::swap(perm[i], perm[rand() % (i + 1)]);
    int* dperm;
    cudaMalloc(&dperm, D * 4);
    cudaMemcpy(dperm, perm.data(), D * 4, cudaMemcpyHostToDevice);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<EncodeFn>(f);
    Maps M;
    auto mk = [&](CUtensorMap* m, int box_rows) {
        cuuint64_t dims[2] = {cuuint64_t(K), cuuint64_t(D)};
        cuuint64_t st[1] = {cuuint64_t(K) * 2};
        cuuint32_t box[2] = {64, cuuint32_t(box_rows)}, es[2] = {1, 1};
        enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    };
    mk(&M.box128, 128);
    mk(&M.box1, 1);
    mk(&M.box8, 8);
    const int smem = kStages * kStage + 1024;
    cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const char* names[] = {"tile 128 rows", "gather4 x32 lanes", "gather4 1 lane", "gather4 random rows",
                           "tile 8 rows x32 lanes", "cp.async 128 thr random", "cp.async no fence",
                           "cp.async arrive.noinc"};
    for (int grid : {sms, 86, 43}) {
        for (int mode = 0; mode < 8; ++mode) {
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            stream<<<grid, 160, smem>>>(M, D, K, mode, dperm, sink, w);
            cudaEventRecord(a);
            for (int it = 0; it < 5; ++it) stream<<<grid, 160, smem>>>(M, D, K, mode, dperm, sink, w);
            cudaEventRecord(b);
            cudaError_t e = cudaDeviceSynchronize();
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            const double bytes = 5.0 * D * K * 2;
            std::printf("grid %3d %-24s %8.1f GB/s  (%s)\n", grid, names[mode], bytes / (ms * 1e-3) / 1e9,
                        cudaGetErrorString(e));
        }
    }
    return 0;
}
