// GPU-side kernel-table precompute: the cascade
// refinements of the scaling function and of the boundary functions
// (kernel.cpp:31-77 via wavelet.cpp:192-311) run on the device; the host keeps
// the cheap cell-mass quadrature and the 2^q-point sequency FWHT.  Every
// product and sum is rounded separately (__dmul_rn / __dadd_rn, no FMA
// contraction) in the host's order, so the tables are bit-identical to the
// host path and to the reference.
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

#include "cww_launch.h"

namespace cww {

namespace {

// phi on the 2^-r grid over [a, b] from the 2^-(r-1) grid (refine in cww_host.cpp)
__global__ void k_refine(const double* __restrict__ prev, long long nprev, double* __restrict__ cur, long long n,
                         long long a2r, long long half, long long lo, const double* __restrict__ h, int nu,
                         double s2) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const long long x2 = a2r + t;
    double acc = 0.0;
    for (int u = -nu + 1; u <= nu; ++u) {
        const long long i = x2 - u * half - lo;
        if (i >= 0 && i < nprev) acc = __dadd_rn(acc, __dmul_rn(h[u + nu - 1], prev[i]));
    }
    cur[t] = __dmul_rn(s2, acc);
}

// one refinement of the nu boundary functions (cascade_edges in cww_host.cpp):
// nxt[m][t] = sqrt2 (sum_k A[m][k] cur[k][t] + sum_li B[m][li] il[t - (nu+li) 2^(r-1) - a 2^(r-1)])
__global__ void k_refine_edges(const double* __restrict__ cur, long long stride, long long ncur_base, int r, int nu,
                               const double* __restrict__ A, const double* __restrict__ B,
                               const double* __restrict__ il, long long nil, long long a, double s2,
                               double* __restrict__ nxt) {
    const int m = blockIdx.y, W = 2 * nu - 1;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long n = (long long)(nu + m) * (1ll << r) + 1;
    if (t >= n) return;
    double acc = 0.0;
    for (int k = 0; k < nu; ++k) {
        const long long nk = (long long)(nu + k) * ncur_base + 1;  // length of cur[k]
        if (t < nk) acc = __dadd_rn(acc, __dmul_rn(A[m * nu + k], cur[k * stride + t]));
    }
    const long long hr = 1ll << (r - 1);
    for (int li = 0; li <= 2 * m; ++li) {
        const long long idx = t - (long long)(nu + li) * hr - a * hr;
        const double iv = (idx >= 0 && idx < nil) ? il[idx] : 0.0;
        acc = __dadd_rn(acc, __dmul_rn(B[m * W + li], iv));
    }
    nxt[m * stride + t] = __dmul_rn(s2, acc);
}

struct DBuf {
    double* p = nullptr;
    ~DBuf() {
        if (p) cudaFree(p);
    }
    cudaError_t alloc(size_t n) { return cudaMalloc(&p, n * sizeof(double)); }
};

}  // namespace

// Interior cascade levels 0..R of phi over [-nu+1, nu] (lev[r] has (2nu-1) 2^r + 1
// samples); all levels are returned (the edge cascade reads them).
cudaError_t cascade_gpu(const std::vector<double>& h, const std::vector<double>& phi, int nu, int R,
                        std::vector<std::vector<double>>& lev) {
    const int a = -nu + 1, b = nu;
    const double s2 = std::sqrt(2.0);
    lev.assign(size_t(R) + 1, {});
    lev[0] = phi;
    DBuf dh, d0, d1;
    const long long nmax = (long long)(b - a) * (1ll << R) + 1;
    cudaError_t e;
    if ((e = dh.alloc(h.size())) != cudaSuccess || (e = d0.alloc(size_t(nmax))) != cudaSuccess ||
        (e = d1.alloc(size_t(nmax))) != cudaSuccess)
        return e;
    if ((e = cudaMemcpy(dh.p, h.data(), h.size() * 8, cudaMemcpyHostToDevice)) != cudaSuccess) return e;
    if ((e = cudaMemcpy(d0.p, phi.data(), phi.size() * 8, cudaMemcpyHostToDevice)) != cudaSuccess) return e;
    double* prev = d0.p;
    double* cur = d1.p;
    long long nprev = (long long)phi.size();
    for (int r = 1; r <= R; ++r) {
        const long long n = (long long)(b - a) * (1ll << r) + 1, half = 1ll << (r - 1), lo = (long long)a * half;
        k_refine<<<(unsigned)((n + 255) / 256), 256>>>(prev, nprev, cur, n, (long long)a * (1ll << r), half, lo,
                                                       dh.p, nu, s2);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        lev[size_t(r)].resize(size_t(n));
        if ((e = cudaMemcpy(lev[size_t(r)].data(), cur, size_t(n) * 8, cudaMemcpyDeviceToHost)) != cudaSuccess)
            return e;
        std::swap(prev, cur);
        nprev = n;
    }
    return cudaSuccess;
}

// Boundary-function cascade (cascade_edges): start values cur0[m] (nu + m + 1
// samples, computed on the host), interior levels lev[0..R]; returns the nu
// functions at resolution 2^-R ((nu + m) 2^R + 1 samples each).
cudaError_t cascade_edges_gpu(const std::vector<std::vector<double>>& cur0,
                              const std::vector<std::vector<double>>& lev, const std::vector<double>& A,
                              const std::vector<double>& B, int nu, int R, std::vector<std::vector<double>>& out) {
    const int a = -nu + 1;
    const double s2 = std::sqrt(2.0);
    const long long stride = (long long)(2 * nu - 1) * (1ll << R) + 1;  // >= (nu + m) 2^R + 1
    DBuf dc, dn, dA, dB, dil;
    cudaError_t e;
    if ((e = dc.alloc(size_t(nu * stride))) != cudaSuccess || (e = dn.alloc(size_t(nu * stride))) != cudaSuccess ||
        (e = dA.alloc(A.size())) != cudaSuccess || (e = dB.alloc(B.size())) != cudaSuccess ||
        (e = dil.alloc(lev[size_t(R)].size())) != cudaSuccess)
        return e;
    if ((e = cudaMemcpy(dA.p, A.data(), A.size() * 8, cudaMemcpyHostToDevice)) != cudaSuccess) return e;
    if ((e = cudaMemcpy(dB.p, B.data(), B.size() * 8, cudaMemcpyHostToDevice)) != cudaSuccess) return e;
    for (int m = 0; m < nu; ++m)
        if ((e = cudaMemcpy(dc.p + m * stride, cur0[size_t(m)].data(), cur0[size_t(m)].size() * 8,
                            cudaMemcpyHostToDevice)) != cudaSuccess)
            return e;
    double* cur = dc.p;
    double* nxt = dn.p;
    for (int r = 1; r <= R; ++r) {
        const auto& il = lev[size_t(r - 1)];
        if ((e = cudaMemcpy(dil.p, il.data(), il.size() * 8, cudaMemcpyHostToDevice)) != cudaSuccess) return e;
        const long long nlast = (long long)(2 * nu - 1) * (1ll << r) + 1;
        // cur[k] has (nu + k) 2^(r-1) + 1 samples: ncur_base = 2^(r-1)
        k_refine_edges<<<dim3((unsigned)((nlast + 255) / 256), (unsigned)nu), 256>>>(
            cur, stride, 1ll << (r - 1), r, nu, dA.p, dB.p, dil.p, (long long)il.size(), a, s2, nxt);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        std::swap(cur, nxt);
    }
    out.assign(size_t(nu), {});
    for (int m = 0; m < nu; ++m) {
        const long long n = (long long)(nu + m) * (1ll << R) + 1;
        out[size_t(m)].resize(size_t(n));
        if ((e = cudaMemcpy(out[size_t(m)].data(), cur + m * stride, size_t(n) * 8, cudaMemcpyDeviceToHost)) !=
            cudaSuccess)
            return e;
    }
    return cudaSuccess;
}

}  // namespace cww
