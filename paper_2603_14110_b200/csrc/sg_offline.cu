// sparsegate-b200: the offline producer of the hot path's inputs, in C++ without
// Eigen: the predictor factors A, B and the calibration's
// proxy scores / damage weights, i.e.
//   factorization.hpp:31-64   cholesky_whitening  (Gram X X^T + damping ladder, LLT,
//                                                  S^-1 by triangular inversion)
//   factorization.hpp:93-144  build_predictor     (SVD of W S or W; A = U_r Σ_r,
//                                                  B = V_r^T S^-1)
//   calibration.hpp:20-46     damage_weights, proxy_scores
// The large products run on the GPU (a tiled f64 GEMM, below); the small dense
// factorizations (Cholesky, triangular inverse, symmetric eigenproblems of
// (r+p) x (r+p)) run on the host. Two SVD modes:
//   exact       one-sided Jacobi on the host (the f64 reference answer; small shapes)
//   randomized  rank-(r+p) range finder with power iterations, CholeskyQR2 on the
//               GPU, the small core by a Jacobi eigen-decomposition (bench shapes:
//               a 7B-size 11008 x 4096 predictor in well under a second of GPU time)
// All f64.
#include "sparsegate_c.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <functional>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

sg_status sg_internal_fail(sg_status s, const std::string& msg);

namespace {

// ---------------------------------------------------------------------------
// GPU f64 GEMM: C[M x N] = alpha * op(A) op(B) + beta * C, row-major; op = transpose
// when t* != 0 (A is K x M then). 64 x 64 tiles, 256 threads, 4 x 4 outputs each.
// ---------------------------------------------------------------------------
constexpr int kT = 64, kK = 16;

__global__ void __launch_bounds__(256) dgemm_kernel(int M, int N, int K, double alpha, const double* __restrict__ A,
                                                    int lda, int tA, const double* __restrict__ B, int ldb, int tB,
                                                    double beta, double* __restrict__ C, int ldc) {
    __shared__ double As[kK][kT + 1];
    __shared__ double Bs[kK][kT + 1];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int m0 = blockIdx.y * kT, n0 = blockIdx.x * kT;
    double acc[4][4] = {};
    for (int k0 = 0; k0 < K; k0 += kK) {
        for (int e = threadIdx.x; e < kK * kT; e += 256) {
            const int kk = e / kT, mm = e % kT;
            const int m = m0 + mm, k = k0 + kk;
            double a = 0.0;
            if (m < M && k < K) a = tA ? A[static_cast<size_t>(k) * lda + m] : A[static_cast<size_t>(m) * lda + k];
            As[kk][mm] = a;
            const int n = n0 + mm;
            double b = 0.0;
            if (n < N && k < K) b = tB ? B[static_cast<size_t>(n) * ldb + k] : B[static_cast<size_t>(k) * ldb + n];
            Bs[kk][mm] = b;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < kK; ++kk) {
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
            if (m < M && n < N) {
                double* c = C + static_cast<size_t>(m) * ldc + n;
                *c = alpha * acc[i][j] + (beta == 0.0 ? 0.0 : beta * *c);
            }
        }
}

// damage_weights epilogue (calibration.hpp:27-35): w = (act(g) * up')^2 * |down_col|^2
__global__ void damage_kernel(const double* gp, const double* up,
                              const double* dn2, int D, int T, int act, double* w) {  // w may alias gp
    const size_t n = static_cast<size_t>(D) * T;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < n;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const double g = gp[e] > 0.0 ? gp[e] : 0.0;
        double u = up[e];
        if (act == 1) u = u > 0.0 ? u : 0.0;
        const double inner = g * u;
        w[e] = inner * inner * dn2[e / T];
    }
}

// common.hpp:52-90 det_dot on the device, bit for bit: products rounded one by one
// (no FMA contraction), blocks of 64 reduced by the balanced binary tree (split at
// n/2), block results accumulated left to right.
__device__ double tree_sum_dev(const double* v, int n) {
    if (n == 0) return 0.0;
    if (n == 1) return v[0];
    const int half = n / 2;
    return __dadd_rn(tree_sum_dev(v, half), tree_sum_dev(v + half, n - half));
}
__device__ double det_dot_dev(const double* a, const double* b, int n) {
    double buf[64];
    double total = 0.0;
    for (int base = 0; base < n; base += 64) {
        const int m = n - base < 64 ? n - base : 64;
        for (int j = 0; j < m; ++j) buf[j] = __dmul_rn(a[base + j], b[base + j]);
        total = __dadd_rn(total, tree_sum_dev(buf, m));
    }
    return total;
}
// predict_mask (ffn_exec.hpp:125-146) in f64: t = B x (rows), then pre_i = A_i . t + b_i
__global__ void predict_t_kernel(const double* B, const double* x, int r, int d, double* t) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < r) t[j] = det_dot_dev(B + static_cast<size_t>(j) * d, x, d);
}
__global__ void predict_pre_kernel(const double* A, const double* t, const double* bias, int D, int r,
                                   uint8_t* mask, int* count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= D) return;
    const double pre = __dadd_rn(det_dot_dev(A + static_cast<size_t>(i) * r, t, r), bias[i]);
    const bool on = pre > 0.0;
    mask[i] = on ? 1 : 0;
    if (on) atomicAdd(count, 1);
}

struct Dev {
    double* p = nullptr;
    Dev() = default;
    explicit Dev(size_t n) { cudaMalloc(&p, n * sizeof(double)); }
    ~Dev() {
        if (p) cudaFree(p);
    }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
};

cudaError_t gemm(int M, int N, int K, double alpha, const double* A, int lda, int tA, const double* B, int ldb,
                 int tB, double beta, double* C, int ldc) {
    dim3 grid((N + kT - 1) / kT, (M + kT - 1) / kT);
    dgemm_kernel<<<grid, 256>>>(M, N, K, alpha, A, lda, tA, B, ldb, tB, beta, C, ldc);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// host dense kernels
// ---------------------------------------------------------------------------
void par_rows(int64_t n, const std::function<void(int64_t, int64_t)>& fn) {
    const int64_t hw = std::max(1u, std::thread::hardware_concurrency());
    const int64_t w = std::min<int64_t>(hw, std::max<int64_t>(1, n / 16));
    if (w <= 1) {
        fn(0, n);
        return;
    }
    std::vector<std::thread> ts;
    for (int64_t k = 0; k < w; ++k) ts.emplace_back([&, k] { fn(n * k / w, n * (k + 1) / w); });
    for (auto& t : ts) t.join();
}

// In-place Cholesky of a symmetric positive definite n x n (row-major, lower used):
// right-looking, trailing update threaded over rows. false if not positive definite.
bool cholesky(std::vector<double>& a, int64_t n) {
    for (int64_t k = 0; k < n; ++k) {
        double d = a[k * n + k];
        if (!(d > 0.0) || !std::isfinite(d)) return false;
        d = std::sqrt(d);
        a[k * n + k] = d;
        for (int64_t i = k + 1; i < n; ++i) a[i * n + k] /= d;
        par_rows(n - k - 1, [&](int64_t lo, int64_t hi) {
            for (int64_t i = k + 1 + lo; i < k + 1 + hi; ++i) {
                const double lik = a[i * n + k];
                for (int64_t j = k + 1; j <= i; ++j) a[i * n + j] -= lik * a[j * n + k];
            }
        });
    }
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = i + 1; j < n; ++j) a[i * n + j] = 0.0;
    return true;
}

// Inverse of a lower-triangular n x n L (row-major): columns solved independently.
std::vector<double> lower_inverse(const std::vector<double>& L, int64_t n) {
    std::vector<double> inv(static_cast<size_t>(n * n), 0.0);
    par_rows(n, [&](int64_t lo, int64_t hi) {
        for (int64_t c = lo; c < hi; ++c) {
            for (int64_t i = c; i < n; ++i) {
                double s = i == c ? 1.0 : 0.0;
                for (int64_t k = c; k < i; ++k) s -= L[i * n + k] * inv[k * n + c];
                inv[i * n + c] = s / L[i * n + i];
            }
        }
    });
    return inv;
}

// Cyclic Jacobi eigen-decomposition of a symmetric n x n S (row-major): eigenvalues
// (descending) and eigenvectors as columns of V (row-major n x n).
void sym_eig(std::vector<double> S, int64_t n, std::vector<double>& w, std::vector<double>& V) {
    V.assign(static_cast<size_t>(n * n), 0.0);
    for (int64_t i = 0; i < n; ++i) V[i * n + i] = 1.0;
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0.0, tot = 0.0;
        for (int64_t i = 0; i < n; ++i)
            for (int64_t j = 0; j < n; ++j) {
                tot += S[i * n + j] * S[i * n + j];
                if (i != j) off += S[i * n + j] * S[i * n + j];
            }
        if (off <= 1e-30 * tot) break;
        for (int64_t p = 0; p < n - 1; ++p)
            for (int64_t q = p + 1; q < n; ++q) {
                const double apq = S[p * n + q];
                if (std::abs(apq) < 1e-300) continue;
                const double theta = (S[q * n + q] - S[p * n + p]) / (2.0 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
                for (int64_t k = 0; k < n; ++k) {  // S <- J^T S J
                    const double skp = S[k * n + p], skq = S[k * n + q];
                    S[k * n + p] = c * skp - s * skq;
                    S[k * n + q] = s * skp + c * skq;
                }
                for (int64_t k = 0; k < n; ++k) {
                    const double spk = S[p * n + k], sqk = S[q * n + k];
                    S[p * n + k] = c * spk - s * sqk;
                    S[q * n + k] = s * spk + c * sqk;
                }
                for (int64_t k = 0; k < n; ++k) {
                    const double vkp = V[k * n + p], vkq = V[k * n + q];
                    V[k * n + p] = c * vkp - s * vkq;
                    V[k * n + q] = s * vkp + c * vkq;
                }
            }
    }
    std::vector<int64_t> ord(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) ord[i] = i;
    std::sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return S[a * n + a] > S[b * n + b]; });
    w.resize(static_cast<size_t>(n));
    std::vector<double> Vs(static_cast<size_t>(n * n));
    for (int64_t j = 0; j < n; ++j) {
        w[j] = S[ord[j] * n + ord[j]];
        for (int64_t i = 0; i < n; ++i) Vs[i * n + j] = V[i * n + ord[j]];
    }
    V.swap(Vs);
}

// Exact thin SVD of M (m x n row-major, m >= n) by one-sided Jacobi on the columns
// of a column-major working copy: U (m x n), s (n, descending), V (n x n), row-major.
void jacobi_svd(const double* M, int64_t m, int64_t n, std::vector<double>& U, std::vector<double>& s,
                std::vector<double>& V) {
    std::vector<double> A(static_cast<size_t>(m * n));  // column-major
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) A[j * m + i] = M[i * n + j];
    std::vector<double> Vc(static_cast<size_t>(n * n), 0.0);  // column-major
    for (int64_t j = 0; j < n; ++j) Vc[j * n + j] = 1.0;
    // round-robin pairing: n/2 disjoint pairs per step, run in parallel
    const int64_t nn = n + (n & 1);
    std::vector<int64_t> ring(static_cast<size_t>(nn));
    for (int64_t i = 0; i < nn; ++i) ring[i] = i;
    for (int sweep = 0; sweep < 40; ++sweep) {
        std::atomic<int64_t> rotations{0};
        for (int64_t step = 0; step < nn - 1; ++step) {
            par_rows(nn / 2, [&](int64_t lo, int64_t hi) {
                int64_t local = 0;
                for (int64_t k = lo; k < hi; ++k) {
                    int64_t p = ring[k], q = ring[nn - 1 - k];
                    if (p >= n || q >= n) continue;
                    if (p > q) std::swap(p, q);
                    double* ap = A.data() + p * m;
                    double* aq = A.data() + q * m;
                    double alpha = 0, beta = 0, gamma = 0;
                    for (int64_t i = 0; i < m; ++i) {
                        alpha += ap[i] * ap[i];
                        beta += aq[i] * aq[i];
                        gamma += ap[i] * aq[i];
                    }
                    if (std::abs(gamma) <= 1e-15 * std::sqrt(alpha * beta) || gamma == 0.0) continue;
                    ++local;
                    const double zeta = (beta - alpha) / (2.0 * gamma);
                    const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
                    const double c = 1.0 / std::sqrt(1.0 + t * t), sn = c * t;
                    for (int64_t i = 0; i < m; ++i) {
                        const double x = ap[i], y = aq[i];
                        ap[i] = c * x - sn * y;
                        aq[i] = sn * x + c * y;
                    }
                    double* vp = Vc.data() + p * n;
                    double* vq = Vc.data() + q * n;
                    for (int64_t i = 0; i < n; ++i) {
                        const double x = vp[i], y = vq[i];
                        vp[i] = c * x - sn * y;
                        vq[i] = sn * x + c * y;
                    }
                }
                rotations += local;
            });
            // rotate the ring (position 0 fixed)
            const int64_t last = ring[nn - 1];
            for (int64_t i = nn - 1; i > 1; --i) ring[i] = ring[i - 1];
            ring[1] = last;
        }
        if (rotations.load() == 0) break;
    }
    std::vector<double> norms(static_cast<size_t>(n));
    for (int64_t j = 0; j < n; ++j) {
        double a = 0;
        for (int64_t i = 0; i < m; ++i) a += A[j * m + i] * A[j * m + i];
        norms[j] = std::sqrt(a);
    }
    std::vector<int64_t> ord(static_cast<size_t>(n));
    for (int64_t j = 0; j < n; ++j) ord[j] = j;
    std::sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return norms[a] > norms[b]; });
    U.assign(static_cast<size_t>(m * n), 0.0);
    V.assign(static_cast<size_t>(n * n), 0.0);
    s.resize(static_cast<size_t>(n));
    for (int64_t jj = 0; jj < n; ++jj) {
        const int64_t j = ord[jj];
        s[jj] = norms[j];
        const double inv = norms[j] > 0 ? 1.0 / norms[j] : 0.0;
        for (int64_t i = 0; i < m; ++i) U[i * n + jj] = A[j * m + i] * inv;
        for (int64_t i = 0; i < n; ++i) V[i * n + jj] = Vc[j * n + i];
    }
}

#define OFF_CUDA(call)                                                                                 \
    do {                                                                                              \
        cudaError_t e_ = (call);                                                                      \
        if (e_ != cudaSuccess) return sg_internal_fail(SG_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// Q (m x l, device) <- orthonormal basis of the columns of Y (device), CholeskyQR2.
sg_status cholqr2(double* Y, int64_t m, int64_t l) {
    Dev G(static_cast<size_t>(l * l)), Rinv(static_cast<size_t>(l * l)), T(static_cast<size_t>(m * l));
    for (int pass = 0; pass < 2; ++pass) {
        OFF_CUDA(gemm(static_cast<int>(l), static_cast<int>(l), static_cast<int>(m), 1.0, Y, static_cast<int>(l), 1, Y,
                      static_cast<int>(l), 0, 0.0, G.p, static_cast<int>(l)));
        std::vector<double> g(static_cast<size_t>(l * l));
        OFF_CUDA(cudaMemcpy(g.data(), G.p, g.size() * 8, cudaMemcpyDeviceToHost));
        // tiny ridge keeps a rank-deficient sketch factorizable (its extra columns are noise)
        double tr = 0;
        for (int64_t i = 0; i < l; ++i) tr += g[i * l + i];
        for (int64_t i = 0; i < l; ++i) g[i * l + i] += 1e-14 * tr / static_cast<double>(l);
        if (!cholesky(g, l)) return sg_internal_fail(SG_ERR_DATA, "randomized SVD: sketch is not full rank");
        // Y R^-1 with R = L^T: (L^-1)^T on the right
        std::vector<double> li = lower_inverse(g, l);
        OFF_CUDA(cudaMemcpy(Rinv.p, li.data(), li.size() * 8, cudaMemcpyHostToDevice));
        OFF_CUDA(gemm(static_cast<int>(m), static_cast<int>(l), static_cast<int>(l), 1.0, Y, static_cast<int>(l), 0,
                      Rinv.p, static_cast<int>(l), 1, 0.0, T.p, static_cast<int>(l)));
        OFF_CUDA(cudaMemcpy(Y, T.p, static_cast<size_t>(m * l) * 8, cudaMemcpyDeviceToDevice));
    }
    return SG_OK;
}

// Rank-k truncated SVD of M (m x n, host row-major): U (m x k), s (k), V (n x k), by a
// randomized range finder of width l = k + oversample with `power` iterations.
sg_status randomized_svd(const double* M_host, int64_t m, int64_t n, int64_t k, int64_t oversample, int power,
                         uint64_t seed, std::vector<double>* U, std::vector<double>& s, std::vector<double>* V) {
    const int64_t l = std::min<int64_t>(std::min(m, n), k + oversample);
    Dev M(static_cast<size_t>(m * n)), Om(static_cast<size_t>(n * l)), Y(static_cast<size_t>(m * l)),
        Z(static_cast<size_t>(n * l)), Bs(static_cast<size_t>(l * n));
    OFF_CUDA(cudaMemcpy(M.p, M_host, static_cast<size_t>(m * n) * 8, cudaMemcpyHostToDevice));
    std::vector<double> om(static_cast<size_t>(n * l));
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> nd(0.0, 1.0);
    for (auto& v : om) v = nd(rng);
    OFF_CUDA(cudaMemcpy(Om.p, om.data(), om.size() * 8, cudaMemcpyHostToDevice));
    const int im = static_cast<int>(m), in = static_cast<int>(n), il = static_cast<int>(l);
    OFF_CUDA(gemm(im, il, in, 1.0, M.p, in, 0, Om.p, il, 0, 0.0, Y.p, il));  // Y = M Om
    if (sg_status st = cholqr2(Y.p, m, l); st != SG_OK) return st;
    for (int it = 0; it < power; ++it) {
        OFF_CUDA(gemm(in, il, im, 1.0, M.p, in, 1, Y.p, il, 0, 0.0, Z.p, il));  // Z = M^T Q
        if (sg_status st = cholqr2(Z.p, n, l); st != SG_OK) return st;
        OFF_CUDA(gemm(im, il, in, 1.0, M.p, in, 0, Z.p, il, 0, 0.0, Y.p, il));  // Y = M Z
        if (sg_status st = cholqr2(Y.p, m, l); st != SG_OK) return st;
    }
    OFF_CUDA(gemm(il, in, im, 1.0, Y.p, il, 1, M.p, in, 0, 0.0, Bs.p, in));  // Bs = Q^T M (l x n)
    // SVD of the l x n core through the eigen-decomposition of Bs Bs^T (l x l)
    Dev Gd(static_cast<size_t>(l * l));
    OFF_CUDA(gemm(il, il, in, 1.0, Bs.p, in, 0, Bs.p, in, 1, 0.0, Gd.p, il));
    std::vector<double> g(static_cast<size_t>(l * l)), w, Ub;
    OFF_CUDA(cudaMemcpy(g.data(), Gd.p, g.size() * 8, cudaMemcpyDeviceToHost));
    sym_eig(g, l, w, Ub);
    s.resize(static_cast<size_t>(k));
    for (int64_t j = 0; j < k; ++j) s[j] = std::sqrt(std::max(w[j], 0.0));
    if (U || V) {
        std::vector<double> ubk(static_cast<size_t>(l * k));
        for (int64_t i = 0; i < l; ++i)
            for (int64_t j = 0; j < k; ++j) ubk[i * k + j] = Ub[i * l + j];
        Dev Ubk(static_cast<size_t>(l * k)), Ud(static_cast<size_t>(m * k)), Vd(static_cast<size_t>(n * k));
        OFF_CUDA(cudaMemcpy(Ubk.p, ubk.data(), ubk.size() * 8, cudaMemcpyHostToDevice));
        const int ik = static_cast<int>(k);
        if (U) {
            OFF_CUDA(gemm(im, ik, il, 1.0, Y.p, il, 0, Ubk.p, ik, 0, 0.0, Ud.p, ik));  // U = Q Ub
            U->resize(static_cast<size_t>(m * k));
            OFF_CUDA(cudaMemcpy(U->data(), Ud.p, U->size() * 8, cudaMemcpyDeviceToHost));
        }
        if (V) {  // V = Bs^T Ub / s
            OFF_CUDA(gemm(in, ik, il, 1.0, Bs.p, in, 1, Ubk.p, ik, 0, 0.0, Vd.p, ik));
            V->resize(static_cast<size_t>(n * k));
            OFF_CUDA(cudaMemcpy(V->data(), Vd.p, V->size() * 8, cudaMemcpyDeviceToHost));
            for (int64_t i = 0; i < n; ++i)
                for (int64_t j = 0; j < k; ++j) (*V)[i * k + j] = s[j] > 0 ? (*V)[i * k + j] / s[j] : 0.0;
        }
    }
    OFF_CUDA(cudaDeviceSynchronize());
    return SG_OK;
}

// Thin SVD of M (m x n row-major) truncated to k: exact (Jacobi) or randomized.
sg_status svd_k(const double* M, int64_t m, int64_t n, int64_t k, int mode, uint64_t seed, std::vector<double>* U,
                std::vector<double>& s, std::vector<double>* V) {
    if (mode == 1) return randomized_svd(M, m, n, k, 32, 4, seed, U, s, V);
    const bool tr = m < n;  // Jacobi wants rows >= cols: work on M^T and swap U, V
    const int64_t rm = tr ? n : m, rn = tr ? m : n;
    std::vector<double> Mt;
    const double* src = M;
    if (tr) {
        Mt.resize(static_cast<size_t>(m * n));
        for (int64_t i = 0; i < m; ++i)
            for (int64_t j = 0; j < n; ++j) Mt[j * m + i] = M[i * n + j];
        src = Mt.data();
    }
    std::vector<double> Uf, sf, Vf;
    jacobi_svd(src, rm, rn, Uf, sf, Vf);
    s.assign(sf.begin(), sf.begin() + k);
    auto take = [&](const std::vector<double>& X, int64_t rows, std::vector<double>* out) {
        out->resize(static_cast<size_t>(rows * k));
        for (int64_t i = 0; i < rows; ++i)
            for (int64_t j = 0; j < k; ++j) (*out)[i * k + j] = X[i * rn + j];
    };
    if (U) take(tr ? Vf : Uf, m, U);
    if (V) take(tr ? Uf : Vf, n, V);
    return SG_OK;
}

bool finite_all(const double* p, int64_t n) {
    for (int64_t i = 0; i < n; ++i)
        if (!std::isfinite(p[i])) return false;
    return true;
}

}  // namespace

extern "C" {

sg_status sg_cholesky_whitening(const double* X, int64_t d, int64_t T, double epsilon, const double* multipliers,
                                int32_t n_mult, double* S, double* S_inv, double* lambda) {
    if (X == nullptr || d < 1 || T < 1 || (n_mult > 0 && multipliers == nullptr))
        return sg_internal_fail(SG_ERR_USAGE, "cholesky_whitening: bad arguments");
    if (!finite_all(X, d * T)) return sg_internal_fail(SG_ERR_DATA, "activation batch: non-finite entries");
    // Gram X X^T on the GPU
    Dev Xd(static_cast<size_t>(d * T)), Gd(static_cast<size_t>(d * d));
    OFF_CUDA(cudaMemcpy(Xd.p, X, static_cast<size_t>(d * T) * 8, cudaMemcpyHostToDevice));
    OFF_CUDA(gemm(static_cast<int>(d), static_cast<int>(d), static_cast<int>(T), 1.0, Xd.p, static_cast<int>(T), 0,
                  Xd.p, static_cast<int>(T), 1, 0.0, Gd.p, static_cast<int>(d)));
    std::vector<double> gram(static_cast<size_t>(d * d));
    OFF_CUDA(cudaMemcpy(gram.data(), Gd.p, gram.size() * 8, cudaMemcpyDeviceToHost));
    double mu = 0.0;
    for (int64_t i = 0; i < d; ++i) mu += gram[i * d + i];
    mu /= static_cast<double>(d);
    std::ostringstream attempted;
    for (int32_t k = 0; k < n_mult; ++k) {  // factorization.hpp:39-57: the damping ladder
        const double lam = multipliers[k] * epsilon * mu;
        std::vector<double> a = gram;
        for (int64_t i = 0; i < d; ++i) a[i * d + i] += lam;
        if (cholesky(a, d)) {
            if (S) std::memcpy(S, a.data(), a.size() * 8);
            if (S_inv) {
                std::vector<double> inv = lower_inverse(a, d);
                std::memcpy(S_inv, inv.data(), inv.size() * 8);
            }
            if (lambda) *lambda = lam;
            return SG_OK;
        }
        attempted << (k > 0 ? ", " : "") << lam;
    }
    return sg_internal_fail(SG_ERR_DATA, "cholesky whitening failed for every damping value {" + attempted.str() +
                                             "}; calibration data is degenerate");
}

sg_status sg_singular_values(const double* M, int64_t rows, int64_t cols, int32_t svd_mode, int64_t k,
                             uint64_t seed, double* out) {
    if (M == nullptr || out == nullptr || rows < 1 || cols < 1 || k < 1 || k > std::min(rows, cols))
        return sg_internal_fail(SG_ERR_USAGE, "singular_values: bad arguments");
    std::vector<double> s;
    if (sg_status st = svd_k(M, rows, cols, k, svd_mode, seed, nullptr, s, nullptr); st != SG_OK) return st;
    std::memcpy(out, s.data(), static_cast<size_t>(k) * 8);
    return SG_OK;
}

sg_status sg_build_predictor(const double* W, int64_t D, int64_t d, const double* X, int64_t T, int64_t rank,
                             int32_t whitened, int32_t svd_mode, uint64_t seed, double epsilon,
                             const double* multipliers, int32_t n_mult, double* A, double* B, double* sv,
                             int64_t n_sv, double* sigma_r1, double* lambda) {
    if (W == nullptr || A == nullptr || B == nullptr || D < 1 || d < 1)
        return sg_internal_fail(SG_ERR_USAGE, "build_predictor: bad arguments");
    if (rank < 1 || rank > std::min(D, d))  // factorization.hpp:97-100
        return sg_internal_fail(SG_ERR_DATA, "predictor rank " + std::to_string(rank) + " out of range [1, " +
                                                 std::to_string(std::min(D, d)) + "]");
    if (!finite_all(W, D * d)) return sg_internal_fail(SG_ERR_DATA, "gate matrix has non-finite entries");
    std::vector<double> target(W, W + D * d), S, Sinv;
    double lam = 0.0;
    if (whitened) {
        if (X == nullptr || T < 1)
            return sg_internal_fail(SG_ERR_DATA, "calibration batch hidden size 0 does not match gate columns " +
                                                     std::to_string(d));
        S.resize(static_cast<size_t>(d * d));
        Sinv.resize(static_cast<size_t>(d * d));
        if (sg_status st = sg_cholesky_whitening(X, d, T, epsilon, multipliers, n_mult, S.data(), Sinv.data(), &lam);
            st != SG_OK)
            return st;
        // target = W S on the GPU
        Dev Wd(static_cast<size_t>(D * d)), Sd(static_cast<size_t>(d * d)), Td(static_cast<size_t>(D * d));
        OFF_CUDA(cudaMemcpy(Wd.p, W, target.size() * 8, cudaMemcpyHostToDevice));
        OFF_CUDA(cudaMemcpy(Sd.p, S.data(), S.size() * 8, cudaMemcpyHostToDevice));
        OFF_CUDA(gemm(static_cast<int>(D), static_cast<int>(d), static_cast<int>(d), 1.0, Wd.p, static_cast<int>(d), 0,
                      Sd.p, static_cast<int>(d), 0, 0.0, Td.p, static_cast<int>(d)));
        OFF_CUDA(cudaMemcpy(target.data(), Td.p, target.size() * 8, cudaMemcpyDeviceToHost));
    }
    const int64_t kk = std::min<int64_t>(std::min(D, d), std::max<int64_t>(rank + 1, n_sv));
    std::vector<double> U, s, V;
    if (sg_status st = svd_k(target.data(), D, d, kk, svd_mode, seed, &U, s, &V); st != SG_OK)
        return st;
    const int64_t ks = static_cast<int64_t>(s.size());
    // A = U_r diag(s_r) (D x r); B = V_r^T (S^-1 when whitened) (r x d)
    for (int64_t i = 0; i < D; ++i)
        for (int64_t j = 0; j < rank; ++j) A[i * rank + j] = U[i * ks + j] * s[j];
    std::vector<double> Vt(static_cast<size_t>(rank * d));
    for (int64_t j = 0; j < rank; ++j)
        for (int64_t c = 0; c < d; ++c) Vt[j * d + c] = V[c * ks + j];
    if (whitened) {
        Dev Vd(Vt.size()), Id(Sinv.size()), Bd(Vt.size());
        OFF_CUDA(cudaMemcpy(Vd.p, Vt.data(), Vt.size() * 8, cudaMemcpyHostToDevice));
        OFF_CUDA(cudaMemcpy(Id.p, Sinv.data(), Sinv.size() * 8, cudaMemcpyHostToDevice));
        OFF_CUDA(gemm(static_cast<int>(rank), static_cast<int>(d), static_cast<int>(d), 1.0, Vd.p, static_cast<int>(d),
                      0, Id.p, static_cast<int>(d), 0, 0.0, Bd.p, static_cast<int>(d)));
        OFF_CUDA(cudaMemcpy(B, Bd.p, Vt.size() * 8, cudaMemcpyDeviceToHost));
    } else {
        std::memcpy(B, Vt.data(), Vt.size() * 8);
    }
    if (sv)
        for (int64_t j = 0; j < n_sv; ++j) sv[j] = j < ks ? s[j] : 0.0;
    if (sigma_r1) {  // σ_{r+1}(W): of W itself (factorization.hpp:137-140)
        *sigma_r1 = 0.0;
        if (rank < std::min(D, d)) {
            if (!whitened) {
                *sigma_r1 = rank < ks ? s[rank] : 0.0;
            } else {
                std::vector<double> sw;
                if (sg_status st = svd_k(W, D, d, rank + 1, svd_mode, seed + 1, nullptr, sw, nullptr); st != SG_OK)
                    return st;
                *sigma_r1 = sw[rank];
            }
        }
    }
    if (lambda) *lambda = lam;
    return SG_OK;
}

sg_status sg_proxy_scores(const double* A, const double* B, int64_t D, int64_t r, int64_t d, const double* X,
                          int64_t T, double* scores) {
    if (!A || !B || !X || !scores || D < 1 || r < 1 || d < 1 || T < 1)
        return sg_internal_fail(SG_ERR_USAGE, "proxy_scores: bad arguments");
    if (!finite_all(X, d * T)) return sg_internal_fail(SG_ERR_DATA, "activation batch: non-finite entries");
    Dev Ad(static_cast<size_t>(D * r)), Bd(static_cast<size_t>(r * d)), Xd(static_cast<size_t>(d * T)),
        Td(static_cast<size_t>(r * T)), Sd(static_cast<size_t>(D * T));
    OFF_CUDA(cudaMemcpy(Ad.p, A, static_cast<size_t>(D * r) * 8, cudaMemcpyHostToDevice));
    OFF_CUDA(cudaMemcpy(Bd.p, B, static_cast<size_t>(r * d) * 8, cudaMemcpyHostToDevice));
    OFF_CUDA(cudaMemcpy(Xd.p, X, static_cast<size_t>(d * T) * 8, cudaMemcpyHostToDevice));
    // calibration.hpp:39-46: A (B X)
    OFF_CUDA(gemm(static_cast<int>(r), static_cast<int>(T), static_cast<int>(d), 1.0, Bd.p, static_cast<int>(d), 0,
                  Xd.p, static_cast<int>(T), 0, 0.0, Td.p, static_cast<int>(T)));
    OFF_CUDA(gemm(static_cast<int>(D), static_cast<int>(T), static_cast<int>(r), 1.0, Ad.p, static_cast<int>(r), 0,
                  Td.p, static_cast<int>(T), 0, 0.0, Sd.p, static_cast<int>(T)));
    OFF_CUDA(cudaMemcpy(scores, Sd.p, static_cast<size_t>(D * T) * 8, cudaMemcpyDeviceToHost));
    return SG_OK;
}

sg_status sg_damage_weights(const double* gate, const double* up, const double* down, int64_t D, int64_t d,
                            int32_t activation, const double* X, int64_t T, double* weights) {
    if (!gate || !up || !down || !X || !weights || D < 1 || d < 1 || T < 1)
        return sg_internal_fail(SG_ERR_USAGE, "damage_weights: bad arguments");
    if (!finite_all(X, d * T)) return sg_internal_fail(SG_ERR_DATA, "activation batch: non-finite entries");
    Dev Gd(static_cast<size_t>(D * d)), Ud(static_cast<size_t>(D * d)), Xd(static_cast<size_t>(d * T)),
        GP(static_cast<size_t>(D * T)), UP(static_cast<size_t>(D * T)), N2(static_cast<size_t>(D));
    OFF_CUDA(cudaMemcpy(Gd.p, gate, static_cast<size_t>(D * d) * 8, cudaMemcpyHostToDevice));
    OFF_CUDA(cudaMemcpy(Ud.p, up, static_cast<size_t>(D * d) * 8, cudaMemcpyHostToDevice));
    OFF_CUDA(cudaMemcpy(Xd.p, X, static_cast<size_t>(d * T) * 8, cudaMemcpyHostToDevice));
    // calibration.hpp:28-35: gate X, up X, |down column|^2
    OFF_CUDA(gemm(static_cast<int>(D), static_cast<int>(T), static_cast<int>(d), 1.0, Gd.p, static_cast<int>(d), 0,
                  Xd.p, static_cast<int>(T), 0, 0.0, GP.p, static_cast<int>(T)));
    OFF_CUDA(gemm(static_cast<int>(D), static_cast<int>(T), static_cast<int>(d), 1.0, Ud.p, static_cast<int>(d), 0,
                  Xd.p, static_cast<int>(T), 0, 0.0, UP.p, static_cast<int>(T)));
    std::vector<double> n2(static_cast<size_t>(D), 0.0);
    for (int64_t j = 0; j < d; ++j)
        for (int64_t i = 0; i < D; ++i) n2[i] += down[j * D + i] * down[j * D + i];
    OFF_CUDA(cudaMemcpy(N2.p, n2.data(), n2.size() * 8, cudaMemcpyHostToDevice));
    damage_kernel<<<1024, 256>>>(GP.p, UP.p, N2.p, static_cast<int>(D), static_cast<int>(T), activation, GP.p);
    OFF_CUDA(cudaGetLastError());
    OFF_CUDA(cudaMemcpy(weights, GP.p, static_cast<size_t>(D * T) * 8, cudaMemcpyDeviceToHost));
    return SG_OK;
}

sg_status sg_predict_mask_f64(int32_t device, const double* A, const double* B, const double* bias, int64_t D,
                              int64_t r, int64_t d, const double* x, uint8_t* mask, int64_t* count) {
    if (!A || !B || !bias || !x || !mask || D < 1 || r < 1 || d < 1)
        return sg_internal_fail(SG_ERR_USAGE, "predict_mask_f64: bad arguments");
    OFF_CUDA(cudaSetDevice(device));
    Dev Ad(static_cast<size_t>(D * r)), Bd(static_cast<size_t>(r * d)), bd(static_cast<size_t>(D)),
        xd(static_cast<size_t>(d)), td(static_cast<size_t>(r)), md(static_cast<size_t>(D + 15) / 8 + 1);
    OFF_CUDA(cudaMemcpy(Ad.p, A, static_cast<size_t>(D * r) * 8, cudaMemcpyHostToDevice));
    OFF_CUDA(cudaMemcpy(Bd.p, B, static_cast<size_t>(r * d) * 8, cudaMemcpyHostToDevice));
    OFF_CUDA(cudaMemcpy(bd.p, bias, static_cast<size_t>(D) * 8, cudaMemcpyHostToDevice));
    OFF_CUDA(cudaMemcpy(xd.p, x, static_cast<size_t>(d) * 8, cudaMemcpyHostToDevice));
    auto* cnt = reinterpret_cast<int*>(md.p);
    auto* m8 = reinterpret_cast<uint8_t*>(md.p) + 8;
    OFF_CUDA(cudaMemset(cnt, 0, sizeof(int)));
    predict_t_kernel<<<static_cast<int>((r + 127) / 128), 128>>>(Bd.p, xd.p, static_cast<int>(r), static_cast<int>(d),
                                                                 td.p);
    OFF_CUDA(cudaGetLastError());
    predict_pre_kernel<<<static_cast<int>((D + 127) / 128), 128>>>(Ad.p, td.p, bd.p, static_cast<int>(D),
                                                                   static_cast<int>(r), m8, cnt);
    OFF_CUDA(cudaGetLastError());
    int c = 0;
    OFF_CUDA(cudaMemcpy(mask, m8, static_cast<size_t>(D), cudaMemcpyDeviceToHost));
    OFF_CUDA(cudaMemcpy(&c, cnt, sizeof(int), cudaMemcpyDeviceToHost));
    if (count) *count = c;
    return SG_OK;
}

}  // extern "C"
