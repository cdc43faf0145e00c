// Microbenchmark: gathering random 8-KB rows on B200, bulk-copy ring vs LDG.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/mb tools/microbench_gather.cu
// Each CTA (one per SM) reads `per_cta` rows of `row_bytes` chosen at random
// (or sequentially) from a large matrix, and reduces them (so loads are used).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                           \
    do {                                                                                \
        cudaError_t e = (x);                                                            \
        if (e != cudaSuccess) {                                                         \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));            \
            exit(1);                                                                    \
        }                                                                               \
    } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p "
        "bra W_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// ring: warp 16 lane 0 produces; warps 0..kc-1 consume slot s = q % ns (ns multiple of kc)
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__global__ void ring_kernel(const uint8_t* __restrict__ mat, const int* __restrict__ rows,
                            int per_cta, int row_bytes, int ns, int kc, int split,
                            float* out, int hint, int nprod = 1, unsigned long long* tlog = nullptr) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm);
    uint64_t* empty = full + 64;
    uint8_t* ring = sm + 1024;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int i = 0; i < ns; ++i) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    int* srows = reinterpret_cast<int*>(sm + 1024 + ns * row_bytes);
    for (int j = tid; j < per_cta; j += blockDim.x) srows[j] = rows[blockIdx.x * per_cta + j];
    __syncthreads();
    const int* myrows = srows;
    float acc = 0.f;
    const unsigned long long t0 = gtime();
    unsigned long long tfirst = 0;
    if (warp == 16) {
        if (lane < nprod) {
            for (int j = lane; j < per_cta; j += nprod) {
                const int slot = j % ns;
                const int use = j / ns;
                if (use > 0) mbar_wait(empty + slot, (use - 1) & 1);
                mbar_expect_tx(full + slot, row_bytes);
                const uint8_t* src = mat + static_cast<size_t>(myrows[j]) * row_bytes;
                const int piece = row_bytes / split;
                uint64_t pol;
                asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
                for (int p = 0; p < split; ++p) {
                    if (hint)
                        bulk_g2s_hint(ring + static_cast<size_t>(slot) * row_bytes + p * piece,
                                      src + p * piece, piece, full + slot, pol);
                    else
                        bulk_g2s(ring + static_cast<size_t>(slot) * row_bytes + p * piece,
                                 src + p * piece, piece, full + slot);
                }
            }
        }
    } else if (warp < kc) {
        for (int j = warp; j < per_cta; j += kc) {
            const int slot = j % ns;
            mbar_wait(full + slot, (j / ns) & 1);
            if (j == 0 && lane == 0) tfirst = gtime();
            const uint4* r = reinterpret_cast<const uint4*>(ring + static_cast<size_t>(slot) * row_bytes);
            for (int c = lane; c < row_bytes / 16; c += 32) {
                const uint4 v = r[c];
                acc += __uint_as_float(v.x) + __uint_as_float(v.w);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + slot);
        }
    }
    if (acc == 12345.f) out[blockIdx.x] = acc;
    __syncthreads();
    if (tlog && tid == 0) {
        tlog[blockIdx.x * 2] = tfirst - t0;
        tlog[blockIdx.x * 2 + 1] = gtime() - t0;
    }
}

// LDG: each warp takes rows j = warp, warp+16, ...; kU rows in flight per warp
template <int kU>
__global__ void ldg_kernel(const uint8_t* __restrict__ mat, const int* __restrict__ rows,
                           int per_cta, int row_bytes, float* out) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    __shared__ int srows[1024];
    for (int j = tid; j < per_cta; j += blockDim.x) srows[j] = rows[blockIdx.x * per_cta + j];
    __syncthreads();
    const int* myrows = srows;
    float acc = 0.f;
    const int nch = row_bytes / 16;
    for (int j0 = warp * kU; j0 < per_cta; j0 += 16 * kU) {
        for (int c = lane; c < nch; c += 32 * 4) {
            uint4 v[kU][4];
#pragma unroll
            for (int u = 0; u < kU; ++u)
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int cc = c + 32 * k;
                    v[u][k] = (j0 + u < per_cta && cc < nch)
                                  ? ldg_stream(mat + static_cast<size_t>(myrows[j0 + u]) * row_bytes + cc * 16)
                                  : make_uint4(0, 0, 0, 0);
                }
#pragma unroll
            for (int u = 0; u < kU; ++u)
#pragma unroll
                for (int k = 0; k < 4; ++k) acc += __uint_as_float(v[u][k].x) + __uint_as_float(v[u][k].w);
        }
    }
    if (acc == 12345.f) out[blockIdx.x] = acc;
}

// contiguous streaming read of `bytes_per_cta` per CTA (roofline check)
__global__ void stream_kernel(const uint4* __restrict__ mat, size_t n16_per_cta, float* out) {
    const uint4* p = mat + blockIdx.x * n16_per_cta;
    float acc = 0.f;
    for (size_t i = threadIdx.x; i < n16_per_cta; i += blockDim.x * 8) {
        uint4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
            v[k] = i + k * blockDim.x < n16_per_cta ? ldg_stream(p + i + k * blockDim.x) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += __uint_as_float(v[k].x);
    }
    if (acc == 12345.f) out[blockIdx.x] = acc;
}

// L2 prefetch of all rows then ring (rows come from L2)
__global__ void prefetch_kernel(const uint8_t* __restrict__ mat, const int* __restrict__ rows,
                                int per_cta, int row_bytes) {
    const int* myrows = rows + blockIdx.x * per_cta;
    for (int j = threadIdx.x; j < per_cta; j += blockDim.x)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                         mat + static_cast<size_t>(myrows[j]) * row_bytes),
                     "r"(row_bytes)
                     : "memory");
}

int main(int argc, char** argv) {
    const int per_cta = argc > 1 ? atoi(argv[1]) : 38;
    const int row_bytes = argc > 2 ? atoi(argv[2]) : 8192;
    const size_t nrows_layer = 11008;
    const int reps = 32;
    const size_t nrows_total = nrows_layer * reps;
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    uint8_t* mat;
    CK(cudaMalloc(&mat, nrows_total * row_bytes));
    // non-uniform contents (avoid any compression effects)
    {
        std::vector<uint32_t> h(1 << 20);
        std::mt19937 g(7);
        for (auto& v : h) v = g();
        for (size_t off = 0; off < nrows_total * row_bytes; off += h.size() * 4) {
            const size_t n = std::min(h.size() * 4, nrows_total * row_bytes - off);
            CK(cudaMemcpy(mat + off, h.data(), n, cudaMemcpyHostToDevice));
        }
    }
    float* out;
    CK(cudaMalloc(&out, 4096));
    std::mt19937 rng(1);
    const size_t per_rep = static_cast<size_t>(nsm) * per_cta;
    std::vector<int> hr(reps * per_rep), hs(reps * per_rep);
    for (int r = 0; r < reps; ++r) {
        std::vector<int> perm(nrows_total);
        for (size_t i = 0; i < nrows_total; ++i) perm[i] = static_cast<int>(i);
        std::shuffle(perm.begin(), perm.end(), rng);
        std::vector<int> pick(perm.begin(), perm.begin() + per_rep);
        std::sort(pick.begin(), pick.end());
        for (size_t i = 0; i < per_rep; ++i) {
            hr[r * per_rep + i] = pick[i];
            hs[r * per_rep + i] = static_cast<int>((r * per_rep + i) % nrows_total);
        }
    }
    int *rows, *seq;
    CK(cudaMalloc(&rows, hr.size() * 4));
    CK(cudaMalloc(&seq, hs.size() * 4));
    CK(cudaMemcpy(rows, hr.data(), hr.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(seq, hs.data(), hs.size() * 4, cudaMemcpyHostToDevice));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double bytes = static_cast<double>(per_rep) * row_bytes;
    auto run = [&](const char* name, auto launch) {
        for (int r = 0; r < 3; ++r) launch(r);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r) launch(r);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1000.0 / reps;
        printf("%-44s %8.2f us/launch  %7.0f GB/s\n", name, us, bytes / (us * 1e-6) / 1e9);
    };
    CK(cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    {
        unsigned long long* tlog;
        CK(cudaMalloc(&tlog, nsm * 16));
        std::vector<unsigned long long> ht(nsm * 2);
        for (int ns : {8, 16, 24}) {
            for (int np : {1, 8, 24}) {
                if (np > ns) continue;
                double f = 0, l = 0, fm = 0, lm = 0;
                for (int r = 0; r < 8; ++r) {
                    ring_kernel<<<nsm, 544, 1024 + ns * row_bytes + per_cta * 4>>>(
                        mat, rows + r * per_rep, per_cta, row_bytes, ns, 16 < ns ? 16 : (ns >= 16 ? 16 : ns), 1, out, 1, np, tlog);
                    CK(cudaDeviceSynchronize());
                    CK(cudaMemcpy(ht.data(), tlog, nsm * 16, cudaMemcpyDeviceToHost));
                    for (int i = 0; i < nsm; ++i) {
                        f += ht[2 * i];
                        l += ht[2 * i + 1];
                        fm = fm > ht[2 * i] ? fm : ht[2 * i];
                        lm = lm > ht[2 * i + 1] ? lm : ht[2 * i + 1];
                    }
                }
                printf("ring ns=%2d nprod=%2d: first row mean %.2f us (max %.2f), done mean %.2f us (max %.2f)\n",
                       ns, np, f / (8 * nsm) / 1000, fm / 1000, l / (8 * nsm) / 1000, lm / 1000);
            }
        }
    }
    const int maxslots = (220 * 1024 - per_cta * 4) / row_bytes;
    for (int hint : {0, 1}) {
        for (int ns : {4, 8, 16, 24}) {
            if (ns > maxslots) continue;
            const int kc = ns < 16 ? ns : 16;
            char nm[96];
            snprintf(nm, 96, "ring random hint=%d kc=%d ns=%d", hint, kc, ns - ns % kc);
            const int nsr = ns - ns % kc;
            run(nm, [&](int r) {
                ring_kernel<<<nsm, 544, 1024 + nsr * row_bytes + per_cta * 4>>>(
                    mat, rows + r * per_rep, per_cta, row_bytes, nsr, kc, 1, out, hint);
            });
        }
    }
    for (int np : {2, 4, 8, 16}) {
        char nm[96];
        snprintf(nm, 96, "ring random hint=1 kc=16 ns=16 nprod=%d", np);
        run(nm, [&](int r) {
            ring_kernel<<<nsm, 544, 1024 + 16 * row_bytes + per_cta * 4>>>(
                mat, rows + r * per_rep, per_cta, row_bytes, 16, 16, 1, out, 1, np);
        });
    }
    for (int sp : {2, 4}) {
        char nm[96];
        snprintf(nm, 96, "ring random kc=16 ns=16 split=%d nprod=16", sp);
        run(nm, [&](int r) {
            ring_kernel<<<nsm, 544, 1024 + 16 * row_bytes + per_cta * 4>>>(
                mat, rows + r * per_rep, per_cta, row_bytes, 16, 16, sp, out, 1, 16);
        });
    }
    for (int ns : {8, 16, 24}) {
        if (ns > maxslots) continue;
        const int kc = ns < 16 ? ns : 16, nsr = ns - ns % kc;
        char nm[96];
        snprintf(nm, 96, "ring SEQ hint=1 kc=%d ns=%d", kc, nsr);
        run(nm, [&](int r) {
            ring_kernel<<<nsm, 544, 1024 + nsr * row_bytes + per_cta * 4>>>(
                mat, seq + r * per_rep, per_cta, row_bytes, nsr, kc, 1, out, 1);
        });
    }
    run("ldg random kU=1", [&](int r) {
        ldg_kernel<1><<<nsm, 512>>>(mat, rows + r * per_rep, per_cta, row_bytes, out);
    });
    run("ldg random kU=2", [&](int r) {
        ldg_kernel<2><<<nsm, 512>>>(mat, rows + r * per_rep, per_cta, row_bytes, out);
    });
    run("ldg random kU=4", [&](int r) {
        ldg_kernel<4><<<nsm, 512>>>(mat, rows + r * per_rep, per_cta, row_bytes, out);
    });
    run("ldg seq kU=2", [&](int r) {
        ldg_kernel<2><<<nsm, 512>>>(mat, seq + r * per_rep, per_cta, row_bytes, out);
    });
    run("stream (contiguous per CTA, same bytes)", [&](int r) {
        stream_kernel<<<nsm, 512>>>(reinterpret_cast<const uint4*>(mat) + r * per_rep * row_bytes / 16 % (nrows_total * row_bytes / 16 / 2),
                                    static_cast<size_t>(per_cta) * row_bytes / 16, out);
    });
    run("prefetch-L2 random (issue only)", [&](int r) {
        prefetch_kernel<<<nsm, 64>>>(mat, rows + r * per_rep, per_cta, row_bytes);
    });
    return 0;
}
