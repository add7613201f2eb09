#pragma once
// sm_100a kernel templates of the Walsh->wavelet change-of-basis operator.
//
//   small path  (M <= kSmallMax): one CTA per group of V vectors runs the whole
//               composed map in shared memory:
//                 forward  k_small_fwd : IDWT (all levels) -> H_A -> stencil+edges
//                                        -> H_B -> sequency-ordered store
//                 adjoint  k_small_adj : sequency-ordered load -> H_B -> correlation
//                                        stencil (+edge sums) -> H_A -> overlap-add
//                                        -> DWT (all levels) -> store
//   large path  (M > kSmallMax): wavelet levels as separate passes, then a
//               two-pass Hadamard with an L2-resident intermediate G of
//               A x (B+2h) doubles:
//                 forward  k_large_fwd1 (contiguous chunks: halo/mask + H over the
//                          low K bits)  ->  k_large_fwd2 (strided: H over the high
//                          K bits + stencil + H_B + sequency store)
//                 adjoint  k_large_adj2 (strided: load + H_B + correlation + H over
//                          the high N bits)  ->  k_large_adj1 (contiguous: H over
//                          the low bits + overlap-add + edges)
//
// Reference correspondence: fastop.cpp:100-175 (forward_1d / adjoint_1d),
// fastop.cpp:196-227 (2D driver), wavelet.cpp:367-514 (dwt_apply levels),
// walsh.cpp:41-98 (FWHT), fastop.cpp:54-98 (edge terms).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "cww_device.cuh"
#include "cww_launch.h"

namespace cww {

constexpr int kKMax = 32;  // register-staged outputs per thread (in-place levels)

// ============================================================================
// small path
// ============================================================================

template <int NU, int LOGB>
struct SmallSmem {
    using G = Geo<NU, LOGB>;
    // doubles: filters | EV[V][2nu] | ES/W[V][S][2NP] | EPW[V][slots][S][2NP] | region
    static __host__ __device__ long long filt() { return FiltSmem<NU>::SIZE; }
};

// shared-memory footprint (bytes) of one small-path CTA
template <int NU, int LOGB>
inline long long small_smem_bytes(int V, int j, int q, bool adj, bool vf) {
    using G = Geo<NU, LOGB>;
    const int a = j - LOGB, A = 1 << a, S = 1 << q;
    long long d = FiltSmem<NU>::SIZE + (long long)V * 2 * NU + (long long)V * S * 2 * G::NP;
    if (adj) {  // edge partial-sum slots, as computed in k_small_adj
        int L = vf ? ((32 / V) < A ? (32 / V) : A) : (A < 32 ? A : 32);
        int nslot = A / L > 0 ? A / L : 1;
        d += (long long)V * (nslot + 1) * S * 2 * G::NP;
    }
    long long region = (long long)V * A * G::RS;
    long long xs = (long long)V << j;
    d += region > xs ? region : xs;
    return d * 8;
}

// Load the staged filters (h | g | edge matrices are contiguous in the table).
template <int NU>
__device__ __forceinline__ void stage_filters(double* filt, const SmallArgs& p, int tid, int nt) {
    for (int i = tid; i < FiltSmem<NU>::SIZE; i += nt) filt[i] = p.tab[p.t.o_h + i];
}

template <int NU, int LOGB, int NT>
__global__ void __launch_bounds__(NT) k_small_fwd(SmallArgs p) {
    using G = Geo<NU, LOGB>;
    constexpr int B = G::B, H = G::H, CW = G::CW, RS = G::RS, NP = G::NP;
    extern __shared__ double sm[];
    const int tid = threadIdx.x;
    const int j = p.j, M = 1 << j, a = j - LOGB, A = 1 << a, S = 1 << p.q;
    const int V = p.V;
    const long long v0 = (long long)blockIdx.x * V;
    const int nv = (int)((p.nvec - v0) < V ? (p.nvec - v0) : V);
    double* filt = sm;
    double* EV = filt + FiltSmem<NU>::SIZE;
    double* ES = EV + V * 2 * NU;
    double* X = ES + V * S * 2 * NP;
    double* T = X;  // the tile overlaps X (all X reads finish before the tile is written)
    const long long tst = (long long)A * RS;

    stage_filters<NU>(filt, p, tid, NT);
    const long long tot = (long long)nv * M;
    const bool vf = p.lin.vfast();
    for (long long f = tid; f < tot; f += NT) {
        int v = vf ? (int)(f % nv) : (int)(f >> j);
        int i = vf ? (int)(f / nv) : (int)(f & (M - 1));
        X[(long long)v * M + i] = p.in[p.lin.at(v0 + v, i)];
    }
    __syncthreads();
    FiltSmem<NU> F{filt};

    // IDWT levels r0+1 .. j-1 in place (register staged), wavelet.cpp:505-513
    const int lev0 = p.use_idwt ? p.r0 + 1 : j + 1;
    for (int lev = lev0; lev < j; ++lev) {
        const int n = 1 << lev;
        const int total = nv << lev;
        double r[kKMax];
#pragma unroll
        for (int k = 0; k < kKMax; ++k) {
            int o = tid + k * NT;
            if (o < total) r[k] = idwt_sample<NU>(F, X + (long long)(o >> lev) * M, n, o & (n - 1), p.vmp);
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kKMax; ++k) {
            int o = tid + k * NT;
            if (o < total) X[(long long)(o >> lev) * M + (o & (n - 1))] = r[k];
        }
        __syncthreads();
    }
    // final level (or plain copy) -> registers -> extended tile
    {
        double r[kKMax];
        const int total = nv << j;
#pragma unroll
        for (int k = 0; k < kKMax; ++k) {
            int o = tid + k * NT;
            if (o < total) {
                const double* xv = X + (long long)(o >> j) * M;
                int i = o & (M - 1);
                r[k] = (lev0 <= j) ? idwt_sample<NU>(F, xv, M, i, p.vmp) : xv[i];
            }
        }
        __syncthreads();
        // halo cells without a source: row 0 left halo, row A-1 right halo
        for (int f = tid; f < nv * 2 * H; f += NT) {
            int v = f / (2 * H), c = f % (2 * H);
            double* t = T + v * tst;
            if (c < H) t[tile_idx(0, c, RS, 0)] = 0.0;
            else t[tile_idx(A - 1, B + c, RS, brev_bits(A - 1, a))] = 0.0;
        }
#pragma unroll
        for (int k = 0; k < kKMax; ++k) {
            int o = tid + k * NT;
            if (o < total) {
                int v = o >> j, i = o & (M - 1);
                double val = r[k];
                if (NU > 1 && (i < NU || i >= M - NU)) {  // interior mask; edge columns kept aside
                    EV[v * 2 * NU + (i < NU ? i : NU + i - (M - NU))] = val;
                    val = 0.0;
                }
                double* t = T + v * tst;
                int K = i >> LOGB, kl = i & (B - 1);
                t[tile_idx(K, kl + H, RS, brev_bits(K, a))] = val;
                if (kl < H && K > 0) t[tile_idx(K - 1, B + H + kl, RS, brev_bits(K - 1, a))] = val;
                if (kl >= B - H && K < A - 1) t[tile_idx(K + 1, kl - (B - H), RS, brev_bits(K + 1, a))] = val;
            }
        }
    }
    __syncthreads();
    // edge contributions es[v][s][pos] = sum_c em[s][pos][c] xi_edge[c]
    if (NU > 1) {
        for (int f = tid; f < nv * S * 2 * NP; f += NT) {
            int v = f / (S * 2 * NP), sp = f % (S * 2 * NP);
            const double* em = p.tab + p.t.o_em + (long long)sp * 2 * NU;
            double acc = 0.0;
#pragma unroll
            for (int c = 0; c < 2 * NU; ++c) acc += em[c] * EV[v * 2 * NU + c];
            ES[f] = acc;
        }
    }
    tile_hadamard(T, nv, a, 0, a, CW, RS, tst, tid, NT);
    __syncthreads();

    // row stage: stencil + edges + H_B + sequency-ordered store
    const bool of = p.lout.vfast();
    const int items = nv * A * S;
    for (int w = tid; w < items; w += NT) {
        int v, wlo, s;
        if (of) {
            v = w % nv;
            int rest = w / nv;
            wlo = rest % A;
            s = rest / A;
        } else {
            wlo = w % A;
            int rest = w / A;
            s = rest % S;
            v = rest / S;
        }
        const int N = (int)brev_bits(wlo, a);
        const double* t = T + v * tst;
        double row[CW];
#pragma unroll
        for (int e = 0; e < CW; ++e) row[e] = t[tile_idx(N, e, RS, wlo)];
        double kap[2 * H + 1];
#pragma unroll
        for (int l = 0; l <= 2 * H; ++l) kap[l] = __ldg(p.tab + p.t.o_kap + l * S + s);
        double z[B];
#pragma unroll
        for (int k = 0; k < B; ++k) {
            double acc = 0.0;
#pragma unroll
            for (int l = -H; l <= H; ++l) acc += kap[l + H] * row[k - l + H];
            z[k] = acc;
        }
        if (NU > 1) {
            const double* es = ES + (v * S + s) * 2 * NP;
            const double sg = (a > 0 && (__popc(N) & 1)) ? -1.0 : 1.0;
#pragma unroll
            for (int i = 0; i < NP; ++i) z[i] += es[i];
#pragma unroll
            for (int i = 0; i < NP; ++i) z[B - NP + i] += sg * es[NP + i];
        }
        hadamard_reg<LOGB>(z);
#pragma unroll
        for (int nl = 0; nl < B; ++nl) {
            unsigned g = (brev_bits(nl, LOGB) << a) | (unsigned)wlo;
            int r = (int)gray_inv(g);
            if (s & 1) r = M - 1 - r;
            p.out[p.lout.at(v0 + v, (long long)s * M + r)] = z[nl];
        }
    }
}

// Warp all-reduce over the lanes that share a vector (deterministic butterfly).
__device__ __forceinline__ double seg_allreduce(double x, int lo_off, int hi_off) {
    for (int off = lo_off; off < hi_off; off <<= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
    return x;
}

template <int NU, int LOGB, int NT>
__global__ void __launch_bounds__(NT) k_small_adj(SmallArgs p) {
    using G = Geo<NU, LOGB>;
    constexpr int B = G::B, H = G::H, CW = G::CW, RS = G::RS, NP = G::NP;
    extern __shared__ double sm[];
    const int tid = threadIdx.x, lane = tid & 31;
    const int j = p.j, M = 1 << j, a = j - LOGB, A = 1 << a, S = 1 << p.q;
    const int V = p.V;
    const long long v0 = (long long)blockIdx.x * V;
    const int nv = (int)((p.nvec - v0) < V ? (p.nvec - v0) : V);
    const bool vf = p.lin.vfast();
    // lanes of a warp that share one vector: a contiguous (non-vfast) or
    // strided (vfast) subset; L of them per warp, EPW slots per vector A/L
    const int L = vf ? ((32 / V) < A ? (32 / V) : A) : (A < 32 ? A : 32);
    const int nslot = A / L > 0 ? A / L : 1;
    double* filt = sm;
    double* EV = filt + FiltSmem<NU>::SIZE;  // unused (edge values), kept for layout symmetry
    double* W = EV + V * 2 * NU;              // [V][S][2NP]
    double* EPW = W + V * S * 2 * NP;         // [V][nslot+1][S][2NP]
    double* X = EPW + (long long)V * (nslot + 1) * S * 2 * NP;
    double* T = X;
    const long long tst = (long long)A * RS;
    stage_filters<NU>(filt, p, tid, NT);

    // row stage: sequency-ordered load + H_B + correlation stencil (+ edge partials)
    const int items = V * A;  // padded to V so that lane->vector is a fixed pattern
    const int iters = (items + NT - 1) / NT;
    for (int it = 0; it < iters; ++it) {
        int w = tid + it * NT;
        int v, wlo;
        if (vf) {
            v = w % V;
            wlo = (w / V) % A;
        } else {
            wlo = w % A;
            v = w / A;
        }
        const bool act = (w < items) && (v < nv);
        const int N = (int)brev_bits(wlo, a);
        const double sg = (a > 0 && (__popc(N) & 1)) ? -1.0 : 1.0;
        double acc[CW];
#pragma unroll
        for (int e = 0; e < CW; ++e) acc[e] = 0.0;
        for (int s = 0; s < S; ++s) {
            double y[B];
#pragma unroll
            for (int nl = 0; nl < B; ++nl) {
                unsigned g = (brev_bits(nl, LOGB) << a) | (unsigned)wlo;
                int r = (int)gray_inv(g);
                if (s & 1) r = M - 1 - r;
                y[nl] = act ? p.in[p.lin.at(v0 + v, (long long)s * M + r)] : 0.0;
            }
            hadamard_reg<LOGB>(y);
            double kap[2 * H + 1];
#pragma unroll
            for (int l = 0; l <= 2 * H; ++l) kap[l] = __ldg(p.tab + p.t.o_kap + l * S + s);
#pragma unroll
            for (int e = 0; e < CW; ++e) {
#pragma unroll
                for (int l = -H; l <= H; ++l) {
                    const int k = e - H + l;
                    if (k >= 0 && k < B) acc[e] += kap[l + H] * y[k];
                }
            }
            if (NU > 1) {  // transform-domain values at the 4nu-2 edge positions
                const int lo_off = vf ? V : 1;
                const int hi_off = vf ? 32 : L;
                const bool leader = vf ? (lane < V) : ((lane & (L - 1)) == 0);
                const int slot = (it * NT + (tid & ~31)) / (vf ? V : 1) / L % nslot;
#pragma unroll
                for (int i = 0; i < 2 * NP; ++i) {
                    double val = i < NP ? y[i] : sg * y[B - NP + (i - NP)];
                    val = seg_allreduce(val, lo_off, hi_off);
                    if (leader && act) EPW[(((long long)v * (nslot + 1) + slot) * S + s) * 2 * NP + i] = val;
                }
            }
        }
        if (act) {
            double* t = T + v * tst;
#pragma unroll
            for (int e = 0; e < CW; ++e) t[tile_idx(N, e, RS, wlo)] = acc[e];
        }
    }
    __syncthreads();
    tile_hadamard(T, nv, a, 0, a, CW, RS, tst, tid, NT);
    __syncthreads();
    if (NU > 1) {  // W[v][s][pos] = sum over rows (fixed order)
        for (int f = tid; f < nv * S * 2 * NP; f += NT) {
            int v = f / (S * 2 * NP), sp = f % (S * 2 * NP);
            double acc = 0.0;
            for (int sl = 0; sl < nslot; ++sl) acc += EPW[((long long)v * (nslot + 1) + sl) * S * 2 * NP + sp];
            W[f] = acc;
        }
        __syncthreads();
    }
    // overlap-add + interior mask + edge columns -> registers -> X
    {
        double r[kKMax];
        const int total = nv << j;
#pragma unroll
        for (int k = 0; k < kKMax; ++k) {
            int o = tid + k * NT;
            if (o < total) {
                int v = o >> j, i = o & (M - 1);
                const double* t = T + v * tst;
                int K = i >> LOGB, kl = i & (B - 1);
                double val = t[tile_idx(K, kl + H, RS, brev_bits(K, a))];
                if (kl < H && K > 0) val += t[tile_idx(K - 1, B + H + kl, RS, brev_bits(K - 1, a))];
                if (kl >= B - H && K < A - 1) val += t[tile_idx(K + 1, kl - (B - H), RS, brev_bits(K + 1, a))];
                if (NU > 1 && (i < NU || i >= M - NU)) {
                    int c = i < NU ? i : NU + i - (M - NU);
                    const double* wv = W + v * S * 2 * NP;
                    double e = 0.0;
                    for (int sp = 0; sp < S * 2 * NP; ++sp) e += p.tab[p.t.o_em + (long long)sp * 2 * NU + c] * wv[sp];
                    val = e;
                }
                r[k] = val;
            }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kKMax; ++k) {
            int o = tid + k * NT;
            if (o < total) X[(long long)(o >> j) * M + (o & (M - 1))] = r[k];
        }
        __syncthreads();
    }
    // DWT levels j .. r0+1 in place (wavelet.cpp:497-504)
    FiltSmem<NU> F{filt};
    if (p.use_idwt) {
        for (int lev = j; lev > p.r0; --lev) {
            const int n = 1 << lev;
            const int total = nv << lev;
            double r[kKMax];
#pragma unroll
            for (int k = 0; k < kKMax; ++k) {
                int o = tid + k * NT;
                if (o < total) r[k] = dwt_sample<NU>(F, X + (long long)(o >> lev) * M, n, o & (n - 1), p.vmp);
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < kKMax; ++k) {
                int o = tid + k * NT;
                if (o < total) X[(long long)(o >> lev) * M + (o & (n - 1))] = r[k];
            }
            __syncthreads();
        }
    }
    const long long tot = (long long)nv * M;
    const bool of = p.lout.vfast();
    for (long long f = tid; f < tot; f += NT) {
        int v = of ? (int)(f % nv) : (int)(f >> j);
        int i = of ? (int)(f / nv) : (int)(f & (M - 1));
        p.out[p.lout.at(v0 + v, i)] = X[(long long)v * M + i];
    }
}

// ============================================================================
// wavelet levels in global memory (large path)
// ============================================================================

// One IDWT level: fine[i] for i < n from c = lo[0:n/2] (workspace, stride
// lo_vs) and d = x-layout elements [n/2, n) of the op input.
template <int NU>
__global__ void k_idwt_level(const double* tab, Tables t, const double* lo, long long lo_vs,
                             const double* x, Layout lx, long long xv0, double* out,
                             long long out_vs, int lev, int nvec, int vmp) {
    __shared__ double filt[FiltSmem<NU>::SIZE];
    for (int i = threadIdx.x; i < FiltSmem<NU>::SIZE; i += blockDim.x) filt[i] = tab[t.o_h + i];
    __syncthreads();
    FiltSmem<NU> F{filt};
    const int n = 1 << lev, half = n >> 1;
    const long long tot = (long long)nvec << lev;
    for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < tot;
         o += (long long)gridDim.x * blockDim.x) {
        int v = (int)(o >> lev), i = (int)(o & (n - 1));
        const double* c = lo + v * lo_vs;
        // gather form with c from the workspace and d read through the layout
        double acc = 0.0;
        if (!vmp) {
#pragma unroll
            for (int k = 0; k < NU; ++k) {
                int u = -NU + 1 + 2 * k + ((i + NU + 1) & 1);
                int tt = (i - u) % n;
                if (tt < 0) tt += n;
                int mm = tt >> 1;
                acc += F.h(u) * c[mm] + F.g(u) * __ldg(x + lx.at(xv0 + v, half + mm));
            }
        } else {
#pragma unroll
            for (int k = 0; k < NU; ++k) {
                int u = -NU + 1 + 2 * k + ((i + NU + 1) & 1);
                int mm = (i - u) >> 1;
                if (mm >= NU && mm < half - NU)
                    acc += F.h(u) * c[mm] + F.g(u) * __ldg(x + lx.at(xv0 + v, half + mm));
            }
            constexpr int W = 2 * NU - 1;
#pragma unroll
            for (int side = 0; side < 2; ++side) {
                int ii = side ? n - 1 - i : i;
                if (ii < 3 * NU - 1) {
#pragma unroll
                    for (int m = 0; m < NU; ++m) {
                        int row = side ? half - 1 - m : m;
                        double cm = c[row], dm = __ldg(x + lx.at(xv0 + v, half + row));
                        if (ii < NU) acc += F.A(side)[m * NU + ii] * cm + F.Aw(side)[m * NU + ii] * dm;
                        else if (ii - NU <= 2 * m)
                            acc += F.Bm(side)[m * W + ii - NU] * cm + F.Bw(side)[m * W + ii - NU] * dm;
                    }
                }
            }
        }
        out[v * out_vs + i] = acc;
    }
}

// One DWT level: from fine samples in[0:n] (workspace) write the coarse half
// to cout[0:n/2] (workspace) and the detail half directly to the op output
// elements [n/2, n).
template <int NU>
__global__ void k_dwt_level(const double* tab, Tables t, const double* in, long long in_vs,
                            double* cout, long long cout_vs, double* y, Layout ly, long long yv0,
                            int lev, int nvec, int vmp) {
    __shared__ double filt[FiltSmem<NU>::SIZE];
    for (int i = threadIdx.x; i < FiltSmem<NU>::SIZE; i += blockDim.x) filt[i] = tab[t.o_h + i];
    __syncthreads();
    FiltSmem<NU> F{filt};
    const int n = 1 << lev, half = n >> 1;
    const long long tot = (long long)nvec << lev;
    for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < tot;
         o += (long long)gridDim.x * blockDim.x) {
        int v = (int)(o >> lev), i = (int)(o & (n - 1));
        double val = dwt_sample<NU>(F, in + v * in_vs, n, i, vmp);
        if (i < half) cout[v * cout_vs + i] = val;
        else y[ly.at(yv0 + v, i)] = val;
    }
}

// Coarse levels in one CTA per vector (shared memory), both directions.
//   inverse: levels r0+1..Lc of x (layout) -> out[0:2^Lc] (workspace)
//   forward: levels Lc..r0+1 of in[0:2^Lc] (workspace) -> y layout [0:2^Lc)
template <int NU>
__global__ void k_wav_coarse(const double* tab, Tables t, const double* src, Layout ls,
                             long long sv0, long long src_vs, double* dst, Layout ld,
                             long long dv0, long long dst_vs, int r0, int Lc, int inverse,
                             int vmp) {
    extern __shared__ double sm[];
    double* filt = sm;
    double* X = sm + FiltSmem<NU>::SIZE;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int i = tid; i < FiltSmem<NU>::SIZE; i += nt) filt[i] = tab[t.o_h + i];
    const int n = 1 << Lc;
    const int v = blockIdx.x;
    for (int i = tid; i < n; i += nt)
        X[i] = inverse ? src[ls.at(sv0 + v, i)] : src[v * src_vs + i];
    __syncthreads();
    FiltSmem<NU> F{filt};
    double r[kKMax];
    for (int step = 0; step < Lc - r0; ++step) {
        int lev = inverse ? r0 + 1 + step : Lc - step;
        int m = 1 << lev;
#pragma unroll
        for (int k = 0; k < kKMax; ++k) {
            int o = tid + k * nt;
            if (o < m) r[k] = inverse ? idwt_sample<NU>(F, X, m, o, vmp) : dwt_sample<NU>(F, X, m, o, vmp);
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kKMax; ++k) {
            int o = tid + k * nt;
            if (o < m) X[o] = r[k];
        }
        __syncthreads();
    }
    for (int i = tid; i < n; i += nt) {
        if (inverse) dst[v * dst_vs + i] = X[i];
        else dst[ld.at(dv0 + v, i)] = X[i];
    }
}

// ============================================================================
// large path: two-pass Hadamard over K with an L2-resident intermediate
// ============================================================================
// G layout per vector: [A rows][CW] (row = K_hi * R1 + n_lo after pass 1).

template <int NU, int NT>
__global__ void __launch_bounds__(NT) k_large_fwd1(LargeArgs p) {
    using Gm = Geo<NU, kLogB>;
    constexpr int B = Gm::B, H = Gm::H, CW = Gm::CW, RS = Gm::RS;
    extern __shared__ double sm[];
    const int tid = threadIdx.x;
    const int j = p.j, M = 1 << j, a = j - kLogB, A = 1 << a;
    const int kl = p.kl, R1 = 1 << kl;
    const int chunk = blockIdx.x, v = blockIdx.y;
    const double* xi = p.xi + (long long)v * p.xi_vs;  // IDWT result (or input via layout)
    double* T = sm;
    // load rows K in [chunk*R1, (chunk+1)*R1) with halos; rows of the tile are
    // local K_lo, swizzled by bitrev_kl(K_lo) (the pass-2 lanes vary K_hi,
    // which is not stored here, so any fixed swizzle is fine).
    const long long base = (long long)chunk * R1 * B - H;
    const int span = R1 * B + 2 * H;
    for (int f = tid; f < R1 * CW; f += NT) {
        int rl = f / CW, e = f % CW;
        long long pos = (long long)(chunk * R1 + rl) * B + e - H;
        double val = 0.0;
        if (pos >= 0 && pos < M) {
            val = p.xi_is_input ? __ldg(p.in + p.lin.at(p.v0 + v, pos)) : __ldg(xi + pos);
            if (NU > 1 && (pos < NU || pos >= M - NU)) val = 0.0;
        }
        T[tile_idx(rl, e, RS, brev_bits(rl, kl))] = val;
    }
    (void)base;
    (void)span;
    // capture the raw edge values (first / last chunk)
    if (NU > 1 && tid < 2 * NU) {
        int c = tid;
        long long pos = c < NU ? c : (M - NU) + (c - NU);
        int owner = (int)((pos / B) / R1);
        if (owner == chunk) {
            double val = p.xi_is_input ? p.in[p.lin.at(p.v0 + v, pos)] : xi[pos];
            p.ev[(long long)v * 2 * NU + c] = val;
        }
    }
    __syncthreads();
    tile_hadamard(T, 1, kl, 0, kl, CW, RS, 0, tid, NT);
    __syncthreads();
    double* g = p.G + (long long)v * A * CW + (long long)chunk * R1 * CW;
    for (int f = tid; f < R1 * CW; f += NT) {
        int rl = f / CW, e = f % CW;
        g[f] = T[tile_idx(rl, e, RS, brev_bits(rl, kl))];
    }
}

template <int NU, int NT>
__global__ void __launch_bounds__(NT) k_large_fwd2(LargeArgs p) {
    using Gm = Geo<NU, kLogB>;
    constexpr int B = Gm::B, H = Gm::H, CW = Gm::CW, RS = Gm::RS, NP = Gm::NP;
    extern __shared__ double sm[];
    const int tid = threadIdx.x;
    const int j = p.j, M = 1 << j, a = j - kLogB, A = 1 << a, S = 1 << p.q;
    const int kl = p.kl, R1 = 1 << kl, kh = a - kl, R2 = 1 << kh;
    const int NG = p.ng;  // n_lo values per CTA
    const int nlo0 = blockIdx.x * NG, v = blockIdx.y;
    double* ES = sm;                    // [S][2NP]
    double* T = sm + S * 2 * NP;        // NG tiles of R2 rows
    const long long tst = (long long)R2 * RS;
    const double* g = p.G + (long long)v * A * CW;
    for (int f = tid; f < NG * R2 * CW; f += NT) {
        int e = f % CW, rest = f / CW;
        int khi = rest % R2, ng = rest / R2;
        double val = g[((long long)khi * R1 + nlo0 + ng) * CW + e];
        T[ng * tst + tile_idx(khi, e, RS, brev_bits(khi, kh))] = val;
    }
    if (NU > 1) {
        for (int f = tid; f < S * 2 * NP; f += NT) {
            const double* em = p.tab + p.t.o_em + (long long)f * 2 * NU;
            double acc = 0.0;
#pragma unroll
            for (int c = 0; c < 2 * NU; ++c) acc += em[c] * p.ev[(long long)v * 2 * NU + c];
            ES[f] = acc;
        }
    }
    __syncthreads();
    tile_hadamard(T, NG, kh, 0, kh, CW, RS, tst, tid, NT);
    __syncthreads();
    const int items = NG * R2 * S;
    for (int w = tid; w < items; w += NT) {
        int wlo = w % R2, rest = w / R2;
        int s = rest % S, ng = rest / S;
        const int nhi = (int)brev_bits(wlo, kh);
        const int nlo = nlo0 + ng;
        const int N = nhi * R1 + nlo;
        const double* t = T + ng * tst;
        double row[CW];
#pragma unroll
        for (int e = 0; e < CW; ++e) row[e] = t[tile_idx(nhi, e, RS, wlo)];
        double kap[2 * H + 1];
#pragma unroll
        for (int l = 0; l <= 2 * H; ++l) kap[l] = __ldg(p.tab + p.t.o_kap + l * S + s);
        double z[B];
#pragma unroll
        for (int k = 0; k < B; ++k) {
            double acc = 0.0;
#pragma unroll
            for (int l = -H; l <= H; ++l) acc += kap[l + H] * row[k - l + H];
            z[k] = acc;
        }
        if (NU > 1) {
            const double* es = ES + s * 2 * NP;
            const double sg = (__popc(N) & 1) ? -1.0 : 1.0;
#pragma unroll
            for (int i = 0; i < NP; ++i) z[i] += es[i];
#pragma unroll
            for (int i = 0; i < NP; ++i) z[B - NP + i] += sg * es[NP + i];
        }
        hadamard_reg<kLogB>(z);
        // g = bitrev_j(N*B + n_lo) = bitrev5(n_lo)*A + bitrev_kl(nlo)*R2 + wlo
        const unsigned glo = (brev_bits(nlo, kl) << kh) | (unsigned)wlo;
#pragma unroll
        for (int nl = 0; nl < B; ++nl) {
            unsigned gg = (brev_bits(nl, kLogB) << a) | glo;
            int r = (int)gray_inv(gg);
            if (s & 1) r = M - 1 - r;
            p.out[p.lout.at(p.v0 + v, (long long)s * M + r)] = z[nl];
        }
    }
}

template <int NU, int NT>
__global__ void __launch_bounds__(NT) k_large_adj2(LargeArgs p) {
    using Gm = Geo<NU, kLogB>;
    constexpr int B = Gm::B, H = Gm::H, CW = Gm::CW, RS = Gm::RS, NP = Gm::NP;
    extern __shared__ double sm[];
    const int tid = threadIdx.x, lane = tid & 31;
    const int j = p.j, M = 1 << j, a = j - kLogB, A = 1 << a, S = 1 << p.q;
    const int kl = p.kl, R1 = 1 << kl, kh = a - kl, R2 = 1 << kh;
    const int NG = p.ng;
    const int nlo0 = blockIdx.x * NG, v = blockIdx.y;
    double* T = sm;
    const long long tst = (long long)R2 * RS;
    const int L = R2 < 32 ? R2 : 32;  // lanes per warp sharing one n_lo tile
    const int items = NG * R2;
    const int iters = (items + NT - 1) / NT;
    for (int it = 0; it < iters; ++it) {
        int w = tid + it * NT;
        int wlo = w % R2, ng = w / R2;
        bool act = w < items;
        const int nhi = (int)brev_bits(wlo, kh);
        const int nlo = nlo0 + (act ? ng : 0);
        const int N = nhi * R1 + nlo;
        const double sg = (__popc(N) & 1) ? -1.0 : 1.0;
        const unsigned glo = (brev_bits(nlo, kl) << kh) | (unsigned)wlo;
        double acc[CW];
#pragma unroll
        for (int e = 0; e < CW; ++e) acc[e] = 0.0;
        for (int s = 0; s < S; ++s) {
            double y[B];
#pragma unroll
            for (int nl = 0; nl < B; ++nl) {
                unsigned gg = (brev_bits(nl, kLogB) << a) | glo;
                int r = (int)gray_inv(gg);
                if (s & 1) r = M - 1 - r;
                y[nl] = act ? p.in[p.lin.at(p.v0 + v, (long long)s * M + r)] : 0.0;
            }
            hadamard_reg<kLogB>(y);
            double kap[2 * H + 1];
#pragma unroll
            for (int l = 0; l <= 2 * H; ++l) kap[l] = __ldg(p.tab + p.t.o_kap + l * S + s);
#pragma unroll
            for (int e = 0; e < CW; ++e) {
#pragma unroll
                for (int l = -H; l <= H; ++l) {
                    const int k = e - H + l;
                    if (k >= 0 && k < B) acc[e] += kap[l + H] * y[k];
                }
            }
            if (NU > 1) {
                // partial sums over this warp's rows; one slot per (CTA, warp, iter)
                const long long slot = ((long long)blockIdx.x * ((NT / 32) * iters) + it * (NT / 32) + (tid >> 5));
#pragma unroll
                for (int i = 0; i < 2 * NP; ++i) {
                    double val = act ? (i < NP ? y[i] : sg * y[B - NP + (i - NP)]) : 0.0;
                    val = seg_allreduce(val, 1, 32);
                    if (lane == 0) p.epw[(((long long)v * p.nslot + slot) * S + s) * 2 * NP + i] = val;
                }
            }
        }
        (void)L;
        if (act) {
#pragma unroll
            for (int e = 0; e < CW; ++e) T[ng * tst + tile_idx(nhi, e, RS, wlo)] = acc[e];
        }
    }
    __syncthreads();
    tile_hadamard(T, NG, kh, 0, kh, CW, RS, tst, tid, NT);
    __syncthreads();
    // write G'[v][khi*R1 + nlo][e]
    double* g = p.G + (long long)v * A * CW;
    for (int f = tid; f < NG * R2 * CW; f += NT) {
        int e = f % CW, rest = f / CW;
        int khi = rest % R2, ng = rest / R2;
        g[((long long)khi * R1 + nlo0 + ng) * CW + e] = T[ng * tst + tile_idx(khi, e, RS, brev_bits(khi, kh))];
    }
}

template <int NU, int NT>
__global__ void __launch_bounds__(NT) k_large_adj1(LargeArgs p) {
    using Gm = Geo<NU, kLogB>;
    constexpr int B = Gm::B, H = Gm::H, CW = Gm::CW, RS = Gm::RS, NP = Gm::NP;
    extern __shared__ double sm[];
    const int tid = threadIdx.x;
    const int j = p.j, M = 1 << j, a = j - kLogB, A = 1 << a, S = 1 << p.q;
    const int kl = p.kl, R1 = 1 << kl;
    const int chunk = blockIdx.x, v = blockIdx.y;
    double* Wv = sm;                 // [S][2NP]
    double* nb = Wv + S * 2 * NP;    // [2][H]: neighbour-row halo sums
    double* T = nb + 2 * (H > 0 ? H : 1);
    const double* g = p.G + (long long)v * A * CW;
    for (int f = tid; f < R1 * CW; f += NT) {
        int rl = f / CW, e = f % CW;
        T[tile_idx(rl, e, RS, brev_bits(rl, kl))] = g[((long long)chunk * R1 + rl) * CW + e];
    }
    // halo contributions from the neighbouring chunks' boundary rows:
    //   previous chunk, last local row (K_lo = R1-1): sum_nlo (-1)^popc(nlo) G[(c-1)R1+nlo][B+H+k]
    //   next chunk, first local row (K_lo = 0):      sum_nlo G[(c+1)R1+nlo][k]
    if (tid < 2 * H) {
        int side = tid / H, k = tid % H;
        double acc = 0.0;
        if (side == 0 && chunk > 0) {
            for (int nl = 0; nl < R1; ++nl) {
                double val = g[((long long)(chunk - 1) * R1 + nl) * CW + B + H + k];
                acc += (__popc(nl) & 1) ? -val : val;
            }
        } else if (side == 1 && (chunk + 1) * R1 < A) {
            for (int nl = 0; nl < R1; ++nl) acc += g[((long long)(chunk + 1) * R1 + nl) * CW + k];
        }
        nb[side * H + k] = acc;
    }
    const bool has_edge = NU > 1 && (chunk == 0 || (chunk + 1) * R1 >= A);
    if (has_edge) {
        for (int f = tid; f < S * 2 * NP; f += NT) {
            double acc = 0.0;
            for (long long sl = 0; sl < p.nslot; ++sl) acc += p.epw[((long long)v * p.nslot + sl) * S * 2 * NP + f];
            Wv[f] = acc;
        }
    }
    __syncthreads();
    tile_hadamard(T, 1, kl, 0, kl, CW, RS, 0, tid, NT);
    __syncthreads();
    double* xo = p.xo + (long long)v * p.xo_vs;
    for (int f = tid; f < R1 * B; f += NT) {
        int rl = f / B, k = f % B;
        long long pos = ((long long)chunk * R1 + rl) * B + k;
        double val = T[tile_idx(rl, k + H, RS, brev_bits(rl, kl))];
        if (k < H) val += rl > 0 ? T[tile_idx(rl - 1, B + H + k, RS, brev_bits(rl - 1, kl))] : nb[k];
        if (k >= B - H) {
            int kk = k - (B - H);
            val += rl < R1 - 1 ? T[tile_idx(rl + 1, kk, RS, brev_bits(rl + 1, kl))] : nb[H + kk];
        }
        if (NU > 1 && (pos < NU || pos >= M - NU)) {
            int c = pos < NU ? (int)pos : NU + (int)(pos - (M - NU));
            double e = 0.0;
            for (int sp = 0; sp < S * 2 * NP; ++sp) e += p.tab[p.t.o_em + (long long)sp * 2 * NU + c] * Wv[sp];
            val = e;
        }
        if (p.xo_is_output) p.out[p.lout.at(p.v0 + v, pos)] = val;
        else xo[pos] = val;
    }
}

}  // namespace cww
