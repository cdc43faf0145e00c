// Probe of the sm_100a building blocks of the batched decode kernel (sg_batch_tc.cu):
//   1. TMA 2D tile loads (SWIZZLE_128B) + tcgen05.mma kind::f16 with K-major A and B,
//      accumulator in TMEM, tcgen05.ld epilogue;
//   2. TMA tile::gather4 of arbitrary weight rows into a K-major SW128 A tile;
//   3. gather4 of neuron-major rows as an MN-major SW128 A operand (the down GEMM),
//      trying the two LBO/SBO assignments.
// Exact small-integer data: every result must match the CPU bit for bit.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/probe_tc.cu -o tools/probe_tc
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                                \
    do {                                                                                     \
        cudaError_t e_ = (x);                                                                \
        if (e_ != cudaSuccess) {                                                             \
            std::printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            std::exit(1);                                                                    \
        }                                                                                    \
    } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
                 : "memory");
}
// bounded wait: returns false on timeout
__device__ __forceinline__ bool mbar_wait(uint64_t* b, uint32_t par) {
    for (int it = 0; it < (1 << 22); ++it) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(su32(b)), "r"(par)
            : "memory");
        if (ok) return true;
    }
    return false;
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            su32(dst)),
        "l"(m), "r"(c0), "r"(c1), "r"(su32(bar))
        : "memory");
}
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* m, int c0, int r0, int r1, int r2,
                                        int r3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
            su32(dst)),
        "l"(m), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(bar))
        : "memory");
}
__device__ __forceinline__ uint64_t sdesc(const void* p, uint32_t lbo, uint32_t sbo) {
    const uint32_t a = su32(p);
    return static_cast<uint64_t>((a >> 4) & 0x3FFF) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
           (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, int a_mn, int b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(a_mn) << 15) |
           (static_cast<uint32_t>(b_mn) << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
           (static_cast<uint32_t>(M >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
        "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ void tld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

struct Maps {
    CUtensorMap a_tile, b_tile, a_g4, w_g4;
};

// mode 0: A K-major by tile; 1: A K-major by gather4 (rows idx); 2/3: MN-major A by gather4,
// LBO/SBO = (8K, 1K) / (1K, 8K). N = 32 columns. Output D[256][32] (two M=128 sub-tiles for mode 2/3).
__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ Maps maps, const int* idx, int mode,
                                                float* out, int* status) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* As = sm;            // 32 KB
    uint8_t* Bs = sm + 32768;    // 4 KB per 64-K stage (32 rows x 128 B) x 2 stages
    __shared__ uint64_t bar_load, bar_mma;
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(&bar_load, 1);
        mbar_init(&bar_mma, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tbase;
    if (threadIdx.x == 0) {
        uint32_t bytes = 0;
        if (mode == 0) {  // A 128 x 64 tile (K 0..63), B 32 x 64
            tma2d(As, &maps.a_tile, 0, 0, &bar_load);
            tma2d(As + 16384, &maps.a_tile, 64, 0, &bar_load);  // K 64..127
            bytes += 32768;
        } else if (mode == 1) {  // 128 rows gathered, K 0..63 and 64..127
            for (int kb = 0; kb < 2; ++kb)
                for (int g = 0; g < 32; ++g)
                    gather4(As + kb * 16384 + g * 512, &maps.a_g4, kb * 64, idx[4 * g], idx[4 * g + 1],
                            idx[4 * g + 2], idx[4 * g + 3], &bar_load);
            bytes += 32768;
        } else {  // MN-major: 64 k-rows (gathered) x 256 m (4 atoms of 64), one 64-K stage
            for (int j = 0; j < 4; ++j)
                for (int g = 0; g < 16; ++g)
                    gather4(As + j * 8192 + g * 512, &maps.w_g4, j * 64, idx[4 * g], idx[4 * g + 1],
                            idx[4 * g + 2], idx[4 * g + 3], &bar_load);
            bytes += 32768;
        }
        tma2d(Bs, &maps.b_tile, 0, 0, &bar_load);
        tma2d(Bs + 4096, &maps.b_tile, 64, 0, &bar_load);
        bytes += 8192;
        mbar_expect_tx(&bar_load, bytes);
        if (!mbar_wait(&bar_load, 0)) {
            status[0] = 1;
        } else {
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t idK = idesc(128, 32, 0, 0), idMN = idesc(128, 32, 1, 0);
            if (mode <= 1) {
                for (int kb = 0; kb < 2; ++kb)
                    for (int k = 0; k < 4; ++k)
                        mma(tmem, sdesc(As + kb * 16384 + k * 32, 16, 1024), sdesc(Bs + kb * 4096 + k * 32, 16, 1024),
                            idK, kb | k);
            } else {
                const uint32_t lbo = mode == 2 ? 8192 : 1024, sbo = mode == 2 ? 1024 : 8192;
                for (int t = 0; t < 2; ++t)
                    for (int k = 0; k < 4; ++k) {
                        const uint32_t koff = k * 2048;  // 16 k-rows of 128 B
                        mma(tmem + t * 32, sdesc(As + t * 16384 + koff, lbo, sbo), sdesc(Bs + k * 32, 16, 1024),
                            idMN, k);
                    }
            }
            commit(&bar_mma);
        }
    }
    __syncthreads();
    if (status[0] == 0) {
        if (!mbar_wait(&bar_mma, 0)) status[0] = 2;
        asm volatile("tcgen05.fence::after_thread_sync;");
        __syncwarp();
        const int row = warp * 32 + lane;
        for (int t = 0; t < (mode >= 2 ? 2 : 1); ++t)
            for (int c = 0; c < 32; c += 16) {
                float v[16];
                tld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + t * 32 + c, v);
                for (int i = 0; i < 16; ++i) out[(t * 128 + row) * 32 + c + i] = v[i];
            }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn encode_fn() {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    return reinterpret_cast<EncodeFn>(f);
}
static CUtensorMap make_map(void* base, uint64_t cols, uint64_t rows, uint32_t box_c, uint32_t box_r) {
    CUtensorMap m;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 2};
    cuuint32_t box[2] = {box_c, box_r};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) std::printf("encode failed (%d) box %u x %u\n", int(r), box_c, box_r);
    return m;
}

int main() {
    const int R = 512, K = 128, N = 32, WM = 256;
    std::vector<uint16_t> A(R * K), B(N * K), W(R * WM);
    std::vector<float> Af(R * K), Bf(N * K), Wf(R * WM);
    srand(7);
    auto mk = [](float v) {
        __nv_bfloat16 h = __float2bfloat16(v);
        uint16_t u;
        std::memcpy(&u, &h, 2);
        return u;
    };
    for (int i = 0; i < R * K; ++i) { Af[i] = float(rand() % 9 - 4); A[i] = mk(Af[i]); }
    for (int i = 0; i < N * K; ++i) { Bf[i] = float(rand() % 9 - 4); B[i] = mk(Bf[i]); }
    for (int i = 0; i < R * WM; ++i) { Wf[i] = float(rand() % 9 - 4); W[i] = mk(Wf[i]); }
    std::vector<int> idx(128);
    for (int i = 0; i < 128; ++i) idx[i] = (i * 37 + 11) % R;
    void *dA, *dB, *dW, *dI, *dO, *dS;
    CK(cudaMalloc(&dA, A.size() * 2));
    CK(cudaMalloc(&dB, B.size() * 2));
    CK(cudaMalloc(&dW, W.size() * 2));
    CK(cudaMalloc(&dI, 128 * 4));
    CK(cudaMalloc(&dO, 256 * 32 * 4));
    CK(cudaMalloc(&dS, 4));
    CK(cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dW, W.data(), W.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dI, idx.data(), 128 * 4, cudaMemcpyHostToDevice));
    CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    int fails = 0;
    for (int g4box : {1, 4}) {
        Maps maps;
        maps.a_tile = make_map(dA, K, R, 64, 128);
        maps.b_tile = make_map(dB, K, N, 64, N);
        maps.a_g4 = make_map(dA, K, R, 64, g4box);
        maps.w_g4 = make_map(dW, WM, R, 64, g4box);
        for (int mode = 0; mode < 4; ++mode) {
            if (mode == 0 && g4box == 4) continue;
            CK(cudaMemset(dO, 0, 256 * 32 * 4));
            CK(cudaMemset(dS, 0, 4));
            probe<<<1, 128, 64 * 1024>>>(maps, static_cast<int*>(dI), mode, static_cast<float*>(dO),
                                         static_cast<int*>(dS));
            cudaError_t e = cudaDeviceSynchronize();
            int st = -1;
            std::vector<float> o(256 * 32);
            if (e == cudaSuccess) {
                CK(cudaMemcpy(&st, dS, 4, cudaMemcpyDeviceToHost));
                CK(cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost));
            }
            int bad = 0, rows = mode >= 2 ? 256 : 128;
            for (int m = 0; m < rows && e == cudaSuccess; ++m)
                for (int n = 0; n < N; ++n) {
                    double ref = 0;
                    if (mode == 0)
                        for (int k = 0; k < K; ++k) ref += Af[m * K + k] * Bf[n * K + k];
                    else if (mode == 1)
                        for (int k = 0; k < K; ++k) ref += Af[idx[m] * K + k] * Bf[n * K + k];
                    else
                        for (int k = 0; k < 64; ++k) ref += Wf[idx[k] * WM + m] * Bf[n * K + k];
                    if (o[m * 32 + n] != static_cast<float>(ref)) ++bad;
                }
            std::printf("gather4 box rows %d mode %d: %s status %d mismatches %d\n", g4box, mode,
                        cudaGetErrorString(e), st, bad);
            if (e != cudaSuccess) return 2;
            fails += bad != 0 || st != 0;
        }
    }
    std::printf("probe done, failing cases: %d\n", fails);
    return 0;
}
