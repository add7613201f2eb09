// Dispatch over the wavelet order and the non-templated utility kernels
// (standalone FWHT, sequency permutation table, Walsh sign rows).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <vector>

#include "cww_device.cuh"
#include "cww_launch.h"

namespace cww {

#define DECL(N)                                                                     \
    cudaError_t launch_small_nu##N(const SmallArgs&, bool, cudaStream_t);           \
    cudaError_t launch_wv_nu##N(const SmallArgs&, bool, cudaStream_t);              \
    long long small_smem_nu##N(int, int, int, bool, bool);                                \
    cudaError_t launch_large_nu##N(int, const LargeArgs&, cudaStream_t);            \
    cudaError_t launch_wav_nu##N(const WavArgs&, cudaStream_t);                    \
    cudaError_t launch_pyr_nu##N(bool, const PyrArgs&, cudaStream_t);               \
    cudaError_t launch_normal_rows_nu##N(const NormArgs&, cudaStream_t);               \
    cudaError_t launch_normal_rows_reg_nu##N(const NormArgs&, cudaStream_t);
DECL(1) DECL(2) DECL(3) DECL(4) DECL(5) DECL(6)
#undef DECL

#define SWITCH_NU(nu, call)                  \
    switch (nu) {                            \
        case 1: return call(1);              \
        case 2: return call(2);              \
        case 3: return call(3);              \
        case 4: return call(4);              \
        case 5: return call(5);              \
        case 6: return call(6);              \
    }

cudaError_t launch_wv(int nu, const SmallArgs& a, bool adj, cudaStream_t st) {
#define C(N) launch_wv_nu##N(a, adj, st)
    SWITCH_NU(nu, C)
#undef C
    return cudaErrorInvalidValue;
}

cudaError_t launch_small(int nu, const SmallArgs& a, bool adj, cudaStream_t st) {
#define C(N) launch_small_nu##N(a, adj, st)
    SWITCH_NU(nu, C)
#undef C
    return cudaErrorInvalidValue;
}

long long small_smem_query(int nu, int V, int j, int q, bool adj, bool vf) {
#define C(N) small_smem_nu##N(V, j, q, adj, vf)
    SWITCH_NU(nu, C)
#undef C
    return -1;
}

cudaError_t launch_large(int nu, int which, const LargeArgs& a, cudaStream_t st) {
#define C(N) launch_large_nu##N(which, a, st)
    SWITCH_NU(nu, C)
#undef C
    return cudaErrorInvalidValue;
}

cudaError_t launch_ana_fixup(int nu, const LargeArgs& a, cudaStream_t st) { return launch_large(nu, 4, a, st); }

__global__ void k_f32_f64(const float* __restrict__ in, double* __restrict__ out, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        out[i] = (double)in[i];
}
__global__ void k_f64_f32(const double* __restrict__ in, float* __restrict__ out, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        out[i] = (float)in[i];  // round to nearest
}
static unsigned conv_grid(long long n) {
    long long g = (n + 255) / 256;
    return (unsigned)(g > 148 * 16 ? 148 * 16 : (g < 1 ? 1 : g));
}
cudaError_t launch_convert_f32_f64(const float* in, double* out, long long n, cudaStream_t st) {
    k_f32_f64<<<conv_grid(n), 256, 0, st>>>(in, out, n);
    return cudaGetLastError();
}
cudaError_t launch_convert_f64_f32(const double* in, float* out, long long n, cudaStream_t st) {
    k_f64_f32<<<conv_grid(n), 256, 0, st>>>(in, out, n);
    return cudaGetLastError();
}

cudaError_t launch_wav(int nu, const WavArgs& w, cudaStream_t st) {
#define C(N) launch_wav_nu##N(w, st)
    SWITCH_NU(nu, C)
#undef C
    return cudaErrorInvalidValue;
}

cudaError_t launch_pyr(int nu, bool analysis, const PyrArgs& a, cudaStream_t st) {
#define C(N) launch_pyr_nu##N(analysis, a, st)
    SWITCH_NU(nu, C)
#undef C
    return cudaErrorInvalidValue;
}

// Sampling mask P_Omega (fastop.cpp:253-281): one vector per blockIdx.y,
// sorted indices -> nearly contiguous full-vector accesses.
__global__ void k_mask(double* full, long long nfull, const uint64_t* __restrict__ idx, long long cnt,
                       double* y, int scatter) {
    const long long b = blockIdx.y;
    double* fb = full + b * nfull;
    double* yb = y + b * cnt;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
         i += (long long)gridDim.x * blockDim.x) {
        const long long k = (long long)__ldg(idx + i);
        if (scatter) fb[k] = yb[i];
        else yb[i] = fb[k];
    }
}

cudaError_t launch_mask(double* full, long long nfull, const uint64_t* idx, long long cnt, double* y,
                        long long batch, bool scatter, cudaStream_t st) {
    if (cnt == 0 || batch == 0) return cudaSuccess;
    long long blocks = (cnt + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    for (long long b0 = 0; b0 < batch; b0 += 65535) {
        const long long nb = batch - b0 < 65535 ? batch - b0 : 65535;
        k_mask<<<dim3((unsigned)blocks, (unsigned)nb), 256, 0, st>>>(full + b0 * nfull, nfull, idx, cnt,
                                                                     y + b0 * cnt, scatter ? 1 : 0);
    }
    return cudaGetLastError();
}

bool normal_reg_ok(int nu, int j, int r0, int use_idwt) {
    (void)nu;
    return use_idwt && j >= 9 && j <= 12 && r0 < kRegLog;
}

cudaError_t launch_normal_rows(int nu, const NormArgs& a, cudaStream_t st) {
    if (normal_reg_ok(nu, a.j, a.r0, a.use_idwt) && (a.V <= 1 || a.es > 0)) {
#define C(N) launch_normal_rows_reg_nu##N(a, st)
        SWITCH_NU(nu, C)
#undef C
    }
#define C(N) launch_normal_rows_nu##N(a, st)
    SWITCH_NU(nu, C)
#undef C
    return cudaErrorInvalidValue;
}

// Batched out-of-place transpose of rows x cols fp64 matrices: 32 x 32 tiles
// through shared memory (odd row stride: conflict-free both ways).
__global__ void k_transpose(const double* __restrict__ in, double* __restrict__ out, long long rows,
                            long long cols) {
    __shared__ double tile[32][33];
    const long long base = (long long)blockIdx.z * rows * cols;
    const long long bx = (long long)blockIdx.x * 32, by = (long long)blockIdx.y * 32;  // column / row tile
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
#pragma unroll
    for (int r = 0; r < 32; r += 8) {
        const long long row = by + ty + r, col = bx + tx;
        if (row < rows && col < cols) tile[ty + r][tx] = in[base + row * cols + col];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 32; r += 8) {
        const long long orow = bx + ty + r, ocol = by + tx;  // out is cols x rows
        if (orow < cols && ocol < rows) out[base + orow * rows + ocol] = tile[tx][ty + r];
    }
}

cudaError_t launch_transpose_rect(const double* in, double* out, long long rows, long long cols, long long batch,
                                  cudaStream_t st) {
    const unsigned gx = (unsigned)((cols + 31) / 32), gy = (unsigned)((rows + 31) / 32);
    for (long long b0 = 0; b0 < batch; b0 += 65535) {
        const long long nb = batch - b0 < 65535 ? batch - b0 : 65535;
        k_transpose<<<dim3(gx, gy, (unsigned)nb), dim3(32, 8), 0, st>>>(in + b0 * rows * cols, out + b0 * rows * cols,
                                                                         rows, cols);
    }
    return cudaGetLastError();
}

cudaError_t launch_transpose(const double* in, double* out, long long n, long long batch, cudaStream_t st) {
    return launch_transpose_rect(in, out, n, n, batch, st);
}

// Unpack of the distributed transpose: rank r's block arrives as recv[r][i][k]
// (already transposed by the sender); local row i (length P*m) is the
// concatenation over r.  Grid-stride over the output in row order (m = 2^lm):
// reads and writes both run along k, 16 bytes per thread.
__global__ void k_unpack_blocks(const double2* __restrict__ recv, double2* __restrict__ x, int lm, int P,
                                long long total2) {
    const long long m2 = (1ll << lm) >> 1;  // double2 per block row
    const long long row2 = m2 * P;          // double2 per local row
    for (long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x; f < total2;
         f += (long long)gridDim.x * blockDim.x) {
        const long long i = f / row2, c = f - i * row2;
        const long long r = c / m2, k = c - r * m2;
        x[f] = recv[(r * (m2 << lm)) + i * m2 + k];
    }
}

cudaError_t launch_unpack_blocks(const double* recv, double* x, long long m, int P, cudaStream_t st) {
    int lm = 0;
    while ((1ll << lm) < m) ++lm;
    if ((1ll << lm) != m || m < 2) return cudaErrorInvalidValue;
    const long long total2 = m * m * P / 2;
    long long blocks = (total2 + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_unpack_blocks<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<const double2*>(recv),
                                                     reinterpret_cast<double2*>(x), lm, P, total2);
    return cudaGetLastError();
}

long long large_nslot(int nu, int q, int j, int kl, int ng) {
    const int nt = 256;
    const int kh = (j - kLogB) - kl, R1 = 1 << kl, R2 = 1 << kh;
    if (large_cta_red(nu, q)) return R1 / ng;  // one slot per adj2 CTA
    int items = ng * R2;
    int iters = (items + nt - 1) / nt;
    return (long long)(R1 / ng) * (nt / 32) * iters;  // one slot per (CTA, iteration, warp)
}


// In-place natural / sequency FWHT of vectors of length 2^bits <= 2^13 (one
// CTA per vector, shared memory).
__global__ void k_fwht_small(double* v, int bits, int sequency) {
    extern __shared__ double sm[];
    const int n = 1 << bits, tid = threadIdx.x, nt = blockDim.x;
    double* x = v + (long long)blockIdx.x * n;
    for (int i = tid; i < n; i += nt) sm[i] = x[i];
    __syncthreads();
    for (int hb = 0; hb < bits; ++hb) {
        int h = 1 << hb;
        for (int i = tid; i < n / 2; i += nt) {
            int lo = ((i >> hb) << (hb + 1)) | (i & (h - 1));
            double a = sm[lo], b = sm[lo + h];
            sm[lo] = a + b;
            sm[lo + h] = a - b;
        }
        __syncthreads();
    }
    for (int i = tid; i < n; i += nt) {
        unsigned src = sequency ? brev_bits((unsigned)(i ^ (i >> 1)), bits) : (unsigned)i;
        x[i] = sm[src];
    }
}

// Large FWHT (bits > 13): passes over groups of index bits, each a tile of
// 2^nb rows x W columns in shared memory (element (r, c) <-> index
// hi * 2^(lo+nb) + r * 2^lo + inner0 + c), radix-2 stages in place in the
// tile, one HBM read + write per pass:
//   pass 1: bits [0, 13)      contiguous chunks of 8192 (W = 1),
//   pass k: bits [lo, lo+10)  2^nb x 8 tiles (64-byte row segments).
// Sequency order (fwht_sequency, walsh.cpp:88-98: out[n] = nat[bitrev(gray(n))])
// is fused into the last pass, which covers the top bits: column c's 2^nb
// results land in one aligned block of 2^nb outputs, n = n0(c) ^
// gray^-1(bitrev_nb(r)), stored in destination order (coalesced).  Passes
// run in place except that the sequency result alternates v -> scratch -> v.
constexpr int kFwhtTileLog = 13;  // doubles per tile: 64 KB
constexpr int kFwhtLW = 3;        // strided passes: 8 columns

__device__ __forceinline__ unsigned gray_inv_u(unsigned x) {
    x ^= x >> 1;
    x ^= x >> 2;
    x ^= x >> 4;
    x ^= x >> 8;
    x ^= x >> 16;
    return x;
}

__global__ void __launch_bounds__(256) k_fwht_pass(const double* __restrict__ src, double* dst, int bits, int lo,
                                                    int nb, int lw, int seq_out) {
    extern __shared__ double T[];  // [2^nb rows][W + 1 (odd stride when W > 1)]
    const int W = 1 << lw, RS = W > 1 ? W + 1 : 1, tid = threadIdx.x, nt = blockDim.x;
    const long long n = 1ll << bits;
    const int ninner = lo > lw ? 1 << (lo - lw) : 1;   // column blocks per (vector, hi)
    const long long nhi = 1ll << (bits - lo - nb);
    long long blk = blockIdx.x;
    const long long ib = blk % ninner;
    blk /= ninner;
    const long long hi = blk % nhi, v = blk / nhi;
    const long long base = v * n + hi * (1ll << (lo + nb)) + ib * W;
    const int R = 1 << nb;
    for (int f = tid; f < R * W; f += nt) {
        const int r = f >> lw, c = f & (W - 1);
        T[r * RS + c] = __ldcs(src + base + ((long long)r << lo) + c);
    }
    __syncthreads();
    for (int hb = 0; hb < nb; ++hb) {
        const int h = 1 << hb;
        for (int f = tid; f < (R >> 1) * W; f += nt) {
            const int i = f >> lw, c = f & (W - 1);
            const int r0 = ((i >> hb) << (hb + 1)) | (i & (h - 1));
            const double a = T[r0 * RS + c], b = T[(r0 + h) * RS + c];
            T[r0 * RS + c] = a + b;
            T[(r0 + h) * RS + c] = a - b;
        }
        __syncthreads();
    }
    if (!seq_out) {
        for (int f = tid; f < R * W; f += nt) {
            const int r = f >> lw, c = f & (W - 1);
            dst[base + ((long long)r << lo) + c] = T[r * RS + c];
        }
        return;
    }
    // last pass (lo + nb == bits): natural index k = r 2^lo + inner, inner = ib W + c;
    // destination n = gray^-1(bitrev_bits(k)) = n0(c) ^ gray^-1(bitrev_nb(r))
    for (int f = tid; f < R * W; f += nt) {
        const int c = f >> nb, t = f & (R - 1);
        const unsigned inner = (unsigned)(ib * W + c);
        const unsigned n0 = gray_inv_u(brev_bits(inner, bits));
        const unsigned u = (unsigned)t ^ (n0 & (unsigned)(R - 1));  // = gray^-1(bitrev_nb(r))
        const int r = (int)brev_bits(u ^ (u >> 1), nb);             // gray(u), reversed
        dst[v * n + (long long)((n0 & ~(unsigned)(R - 1)) | (unsigned)t)] = T[r * RS + c];
    }
}

__global__ void k_seq_perm(uint32_t* perm, int bits) {
    const long long n = 1ll << bits;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        unsigned g = (unsigned)(i ^ (i >> 1));
        perm[i] = brev_bits(g, bits);
    }
}

__global__ void k_sign_rows(const uint64_t* pos, long long npos, int jb, double* out) {
    const long long n = 1ll << jb, tot = npos * n;
    for (long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x; f < tot;
         f += (long long)gridDim.x * blockDim.x) {
        long long ip = f / n, r = f % n;
        unsigned long long vv = jb ? (__brevll(pos[ip]) >> (64 - jb)) : 0ull;
        unsigned long long mask = vv ^ (vv << 1);
        out[f] = (__popcll((unsigned long long)r & mask) & 1) ? -1.0 : 1.0;
    }
}


cudaError_t launch_fwht(double* v, int bits, long long batch, int sequency, double* scratch,
                        cudaStream_t st) {
    if (bits <= 13) {
        long long smem = (1ll << bits) * 8;
        opt_in_smem(reinterpret_cast<const void*>(k_fwht_small));
        k_fwht_small<<<(unsigned)batch, 256, smem, st>>>(v, bits, sequency);
        return cudaGetLastError();
    }
    if (sequency && !scratch) return cudaErrorInvalidValue;
    // passes: [0, 13) contiguous, then <= 10 bits each with 8-column tiles
    struct Pass { int lo, nb, lw; };
    std::vector<Pass> ps{{0, kFwhtTileLog, 0}};
    for (int lo = kFwhtTileLog; lo < bits;) {
        const int nb = bits - lo < kFwhtTileLog - kFwhtLW ? bits - lo : kFwhtTileLog - kFwhtLW;
        ps.push_back({lo, nb, kFwhtLW});
        lo += nb;
    }
    cudaFuncSetAttribute(k_fwht_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    const double* src = v;
    for (size_t i = 0; i < ps.size(); ++i) {
        const Pass& p = ps[i];
        const bool last = i + 1 == ps.size();
        // sequency: the second-to-last pass writes scratch, the last scatters back into v
        double* dst = (sequency && i + 2 == ps.size()) ? scratch : v;
        const int W = 1 << p.lw, RS = W > 1 ? W + 1 : 1;
        const long long smem = (long long)(1 << p.nb) * RS * 8;
        const long long blocks = batch * (1ll << (bits - p.lo - p.nb)) * (p.lo > p.lw ? 1ll << (p.lo - p.lw) : 1);
        if (blocks > 0x7fffffffll) return cudaErrorInvalidValue;
        k_fwht_pass<<<(unsigned)blocks, 256, smem, st>>>(src, dst, bits, p.lo, p.nb, p.lw, (sequency && last) ? 1 : 0);
        src = dst;
    }
    return cudaGetLastError();
}

cudaError_t launch_seq_perm(uint32_t* perm, int bits, cudaStream_t st) {
    k_seq_perm<<<148 * 4, 256, 0, st>>>(perm, bits);
    return cudaGetLastError();
}

cudaError_t launch_sign_rows(const uint64_t* pos, long long npos, int j, double* out,
                             cudaStream_t st) {
    k_sign_rows<<<148 * 4, 256, 0, st>>>(pos, npos, j, out);
    return cudaGetLastError();
}

}  // namespace cww
