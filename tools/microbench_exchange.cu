// Microbenchmark: cost of reading per-CTA values written by all CTAs right
// before a grid barrier (the P-count prefix of phase C).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_exchange tools/microbench_exchange.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t gt() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint64_t ld_acq(const unsigned long long* p) {
    uint64_t v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ void gbar(unsigned long long* ctr, uint64_t target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
        while (ld_acq(ctr) < target) {
        }
    }
    __syncthreads();
}

constexpr int kMaxPrefixChunks = 8;
constexpr int kSector = 8;
__device__ __forceinline__ void warp_prefix(const int* cnt, int* off, int G, int lane) {
    int v[kMaxPrefixChunks];
#pragma unroll
    for (int k = 0; k < kMaxPrefixChunks; ++k) {
        const int i = k * 32 + lane;
        v[k] = i < G ? __ldcg(cnt + i * kSector) : 0;
    }
    int carry = 0;
#pragma unroll
    for (int k = 0; k < kMaxPrefixChunks; ++k) {
        const int i = k * 32 + lane;
        int incl = v[k];
#pragma unroll
        for (int m = 1; m < 32; m <<= 1) {
            const int o = __shfl_up_sync(0xffffffffu, incl, m);
            if (lane >= m) incl += o;
        }
        if (i < G) off[i] = carry + incl - v[k];
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) off[G] = carry;
}

// mode 0: plain 4-B stores; 1: 32-B sector stores; 2: atomicExch
__global__ void k(int* cnt, unsigned long long* ctr, uint64_t base, int mode, uint64_t* out,
                  const uint4* big, int touch_big) {
    const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x;
    uint64_t t0 = gt();
    // optionally stream some memory first (like the phases before)
    float acc = 0.f;
    if (touch_big) {
        for (int i = tid; i < 4096; i += blockDim.x) acc += __uint_as_float(big[c * 4096 + i].x);
    }
    if (tid == 0) {
        if (mode == 0) cnt[c] = c + 1;
        else if (mode == 1) {
            asm volatile("st.global.v4.b32 [%0], {%1, %2, %2, %2};\n\tst.global.v4.b32 [%0+16], {%2, %2, %2, %2};" ::"l"(cnt + c * 8), "r"(c + 1), "r"(0) : "memory");
        } else {
            atomicExch(cnt + c * 8, c + 1);
        }
    }
    gbar(ctr, base + G);
    uint64_t t1 = gt();
    int s = 0;
    if (tid < 32) {
        for (int i = tid; i < G; i += 32) s += __ldcg(cnt + (mode == 0 ? i : i * 8));
        s = __reduce_add_sync(0xffffffffu, s);
    }
    uint64_t t2 = gt();
    int s2 = 0;
    if (tid < 32) {
        for (int i = tid; i < G; i += 32) s2 += __ldcg(cnt + (mode == 0 ? i : i * 8));
        s2 = __reduce_add_sync(0xffffffffu, s2);
    }
    uint64_t t3 = gt();
    __shared__ int off[300];
    if (mode != 0 && tid < 32) warp_prefix(cnt, off, G, tid);
    __syncthreads();
    uint64_t t4 = gt();
    if (tid == 0) {
        out[c * 4 + 0] = t4 - t3;
        out[c * 4 + 1] = t2 - t1;
        out[c * 4 + 2] = t3 - t2;
        out[c * 4 + 3] = s + s2 + (acc == 1.2345f);
    }
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    int* cnt;
    unsigned long long* ctr;
    uint64_t* out;
    uint4* big;
    cudaMalloc(&cnt, nsm * 32);
    cudaMalloc(&ctr, 256);
    cudaMalloc(&out, nsm * 32);
    cudaMalloc(&big, (size_t)nsm * 4096 * 16);
    cudaMemset(ctr, 0, 256);
    cudaMemset(big, 0, (size_t)nsm * 4096 * 16);
    uint64_t base = 0;
    uint64_t h[4096];
    for (int touch = 0; touch < 2; ++touch)
        for (int mode = 0; mode < 3; ++mode) {
            for (int rep = 0; rep < 5; ++rep) {
                k<<<nsm, 544>>>(cnt, ctr, base, mode, out, big, touch);
                base += nsm;
            }
            cudaDeviceSynchronize();
            cudaMemcpy(h, out, nsm * 32, cudaMemcpyDeviceToHost);
            double a = 0, b = 0, cc = 0;
            uint64_t mb = 0;
            for (int i = 0; i < nsm; ++i) {
                a += h[i * 4];
                b += h[i * 4 + 1];
                cc += h[i * 4 + 2];
                if (h[i * 4 + 1] > mb) mb = h[i * 4 + 1];
            }
            printf("touch=%d mode=%d  warp_prefix %.2f us  first read %.2f us (max %.2f)  second read %.2f us\n",
                   touch, mode, a / nsm / 1000, b / nsm / 1000, mb / 1000.0, cc / nsm / 1000);
        }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
