// Device kernels of the least-squares driver (generalised sampling, SPEC.md
// gs_solve: CG on the normal equations A* A x = A* y).
// The operator applications are the library's own forward/adjoint launches;
// these kernels are the CGLS vector algebra, batched (one system per vector)
// with device-resident scalars so an iteration needs no host round trip.
// Reductions are deterministic (fixed partition, fixed tree order).
#include <cuda_runtime.h>

#include "cww_launch.h"

namespace cww {

namespace {

constexpr int kRedNT = 256;

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) red[w] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x < 32) {
        t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    }
    return t;  // valid in thread 0
}

// part[v * nblk + blk] = sum over the blk-th span of a[v] .* b[v]
__global__ void __launch_bounds__(kRedNT) k_dot_partial(const double* __restrict__ a, const double* __restrict__ b,
                                                        long long n, double* part, int nblk) {
    __shared__ double red[kRedNT / 32];
    const long long v = blockIdx.y;
    const long long chunk = (n + nblk - 1) / nblk;
    const long long lo = blockIdx.x * chunk, hi = lo + chunk < n ? lo + chunk : n;
    const double* av = a + v * n;
    const double* bv = b + v * n;
    double acc = 0.0;
    for (long long i = lo + threadIdx.x; i < hi; i += kRedNT) acc = fma(av[i], bv[i], acc);
    const double s = block_sum(acc, red);
    if (threadIdx.x == 0) part[v * nblk + blockIdx.x] = s;
}

__global__ void __launch_bounds__(kRedNT) k_dot_final(const double* part, int nblk, double* out) {
    __shared__ double red[kRedNT / 32];
    const int v = blockIdx.x;
    double acc = 0.0;
    for (int i = threadIdx.x; i < nblk; i += kRedNT) acc += part[(long long)v * nblk + i];
    const double s = block_sum(acc, red);
    if (threadIdx.x == 0) out[v] = s;
}

// x += alpha p, r -= alpha q with alpha = gam / qq (0 for converged systems)
__global__ void k_cgls_xr(double* x, double* r, const double* __restrict__ p, const double* __restrict__ q,
                          long long nx, long long nr, const double* gam, const double* qq, const int* active) {
    const long long v = blockIdx.y;
    const double den = qq[v];
    const double alpha = (active[v] && den > 0.0) ? gam[v] / den : 0.0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nx; i += stride)
        x[v * nx + i] = fma(alpha, p[v * nx + i], x[v * nx + i]);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nr; i += stride)
        r[v * nr + i] = fma(-alpha, q[v * nr + i], r[v * nr + i]);
}

// p = s + beta p with beta = gnew / gold
__global__ void k_cgls_p(double* p, const double* __restrict__ s, long long nx, const double* gnew,
                         const double* gold) {
    const long long v = blockIdx.y;
    const double beta = gold[v] > 0.0 ? gnew[v] / gold[v] : 0.0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nx; i += stride)
        p[v * nx + i] = fma(beta, p[v * nx + i], s[v * nx + i]);
}

// active[v] = ||s_v|| > tol * s0_v  (s0 = ||A* y|| of the initial residual)
__global__ void k_cgls_flags(const double* gam, const double* s0, double tol, int* active, long long batch) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < batch) active[v] = sqrt(gam[v]) > tol * s0[v] ? 1 : 0;
}

__global__ void k_sqrt(const double* a, double* out, long long batch) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < batch) out[v] = sqrt(a[v]);
}

// r = y - r
__global__ void k_sub_from(double* r, const double* __restrict__ y, long long n) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) r[i] = y[i] - r[i];
}

int grid_x(long long n, long long batch) {
    long long g = (n + 255) / 256;
    long long cap = (148 * 8 + batch - 1) / batch;
    if (cap < 1) cap = 1;
    return (int)(g < cap ? g : cap);
}

// ---- Chambolle-Pock for QCBP (SPEC.md cs_solve) ----
// dual, step 1: t = xi / sigma + A zbar - y  (in place in xi)
__global__ void k_cp_dual_t(double* xi, const double* __restrict__ w, const double* __restrict__ y, double inv_sigma,
                            long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        xi[i] = fma(xi[i], inv_sigma, w[i] - y[i]);
}
// dual, step 2: xi = sigma (1 - min(1, sqrt(eta) / ||t||)) t  (= prox of sigma F*,
// F the indicator of the ball ||. - y|| <= sqrt(eta), by Moreau's identity)
__global__ void k_cp_dual_scale(double* xi, const double* tt, double sigma, double sqrt_eta, long long nr) {
    const long long v = blockIdx.y;
    const double nt = sqrt(tt[v]);
    const double c = nt > sqrt_eta ? sqrt_eta / nt : 1.0;
    const double f = sigma * (1.0 - c);
    double* x = xi + v * nr;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nr; i += (long long)gridDim.x * blockDim.x)
        x[i] *= f;
}
// primal: z' = soft(z - tau s, tau); zbar = 2 z' - z; s <- z' - z (for the stopping test)
__global__ void k_cp_primal(double* z, double* zbar, double* s, double tau, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double zo = z[i];
        const double u = zo - tau * s[i];
        const double zn = u > tau ? u - tau : (u < -tau ? u + tau : 0.0);
        z[i] = zn;
        zbar[i] = 2.0 * zn - zo;
        s[i] = zn - zo;
    }
}
// s = a - b
__global__ void k_sub(double* s, const double* __restrict__ a, const double* __restrict__ b, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        s[i] = a[i] - b[i];
}

unsigned flat_grid(long long n) {
    long long g = (n + 255) / 256;
    return (unsigned)(g > 148 * 8 ? 148 * 8 : (g < 1 ? 1 : g));
}

}  // namespace

cudaError_t launch_cp_dual(double* xi, const double* w, const double* y, double sigma, double sqrt_eta,
                           long long nr, long long batch, double* part, double* tt, cudaStream_t st) {
    k_cp_dual_t<<<flat_grid(nr * batch), 256, 0, st>>>(xi, w, y, 1.0 / sigma, nr * batch);
    if (cudaError_t e = launch_dot(xi, xi, nr, batch, part, tt, st); e != cudaSuccess) return e;
    k_cp_dual_scale<<<dim3(grid_x(nr, batch), (unsigned)batch), 256, 0, st>>>(xi, tt, sigma, sqrt_eta, nr);
    return cudaGetLastError();
}

cudaError_t launch_cp_primal(double* z, double* zbar, double* s, double tau, long long n, cudaStream_t st) {
    k_cp_primal<<<flat_grid(n), 256, 0, st>>>(z, zbar, s, tau, n);
    return cudaGetLastError();
}

cudaError_t launch_sub(double* s, const double* a, const double* b, long long n, cudaStream_t st) {
    k_sub<<<flat_grid(n), 256, 0, st>>>(s, a, b, n);
    return cudaGetLastError();
}

int dot_nblk(long long n, long long batch) {
    long long per = (n + kRedNT * 8 - 1) / (kRedNT * 8);  // >= 8 elements per thread
    long long cap = (148 * 4 + batch - 1) / batch;
    long long nb = per < cap ? per : cap;
    return (int)(nb < 1 ? 1 : nb);
}

cudaError_t launch_dot(const double* a, const double* b, long long n, long long batch, double* part,
                       double* out, cudaStream_t st) {
    const int nblk = dot_nblk(n, batch);
    for (long long b0 = 0; b0 < batch; b0 += 65535) {
        const long long nb = batch - b0 < 65535 ? batch - b0 : 65535;
        k_dot_partial<<<dim3(nblk, (unsigned)nb), kRedNT, 0, st>>>(a + b0 * n, b + b0 * n, n, part + b0 * nblk, nblk);
    }
    k_dot_final<<<(unsigned)batch, kRedNT, 0, st>>>(part, nblk, out);
    return cudaGetLastError();
}

cudaError_t launch_cgls_xr(double* x, double* r, const double* p, const double* q, long long nx, long long nr,
                           long long batch, const double* gam, const double* qq, const int* active,
                           cudaStream_t st) {
    k_cgls_xr<<<dim3(grid_x(nx > nr ? nx : nr, batch), (unsigned)batch), 256, 0, st>>>(x, r, p, q, nx, nr, gam, qq,
                                                                                       active);
    return cudaGetLastError();
}

cudaError_t launch_cgls_p(double* p, const double* s, long long nx, long long batch, const double* gnew,
                          const double* gold, cudaStream_t st) {
    k_cgls_p<<<dim3(grid_x(nx, batch), (unsigned)batch), 256, 0, st>>>(p, s, nx, gnew, gold);
    return cudaGetLastError();
}

cudaError_t launch_cgls_flags(const double* gam, const double* s0, double tol, int* active, long long batch,
                              cudaStream_t st) {
    k_cgls_flags<<<(unsigned)((batch + 255) / 256), 256, 0, st>>>(gam, s0, tol, active, batch);
    return cudaGetLastError();
}

cudaError_t launch_sqrt(const double* a, double* out, long long batch, cudaStream_t st) {
    k_sqrt<<<(unsigned)((batch + 255) / 256), 256, 0, st>>>(a, out, batch);
    return cudaGetLastError();
}

cudaError_t launch_sub_from(double* r, const double* y, long long n, cudaStream_t st) {
    long long g = (n + 255) / 256;
    if (g > 148 * 8) g = 148 * 8;
    k_sub_from<<<(unsigned)g, 256, 0, st>>>(r, y, n);
    return cudaGetLastError();
}

}  // namespace cww
