#pragma once
// Warp-per-vector kernels of the composed operator for M = 2^10 (the 2D
// configurations' 1024-point rows and columns, and 1D j = 10): one warp owns
// one vector end to end.  With B = 32 the extended tile has A = 32 rows, so
// lane l owns tile row K = l: the row is built / consumed in registers, H_A
// (the Hadamard transform across rows) is a 5-stage shuffle butterfly across
// the lanes, and the wavelet levels run warp-private and in place in the
// vector's shared-memory region (register-staged: read, __syncwarp, write).
// CTA barriers remain only around the staging of vector-fast layouts (the 2D
// column passes, where one warp's element stride is a whole image row): the
// CTA's 8 consecutive vectors are moved cooperatively, 8 adjacent doubles per
// row, through the warps' regions.
//
//   k_wv_fwd: inputs -> IDWT levels r0+1..9 in place -> level 10 as pairs ->
//             padded xi -> row K per lane (+ halos) -> edge values -> H_A
//             across lanes -> per block s: stencil + edges + H_B in registers
//             -> sequency-ordered store     (fastop.cpp:100-137,
//             wavelet.cpp:447-483, walsh.cpp:41-98)
//   k_wv_adj: per block s: sequency-ordered load -> H_B -> edge sums (warp
//             reduction) -> correlation into the row accumulator -> H_A
//             across lanes -> overlap-add (shuffles) + edge positions ->
//             padded xi -> DWT levels 10..r0+1 in place ([c_r0 | d_r0 | ... |
//             d_9], the output layout) -> store  (fastop.cpp:139-175,
//             wavelet.cpp:403-445)
#include "cww_kernels.cuh"

namespace cww {

constexpr int kWvJ = 10;                     // M = 1024
// per-warp region: 1024 + 64 pads (+2); = 2 (mod 16), so that the cooperative
// staging's half-warps (8 regions x 2 consecutive doubles) cover 16 distinct
// 8-byte banks (= 4 (mod 16) measured 2-way conflicts there: cfg4 1.439 -> 1.413 ms)
constexpr int kWvXS = 1090;
constexpr int kWvNT = 256;                   // 8 warps = 8 vectors per CTA
constexpr int kWvV = kWvNT / 32;
#ifndef WV_MINB
#define WV_MINB 2
#endif

// padded position: one pad per 32 so that lane l's row (33 l + c) is conflict free
__device__ __forceinline__ int wv_pad(int p) { return p + (p >> 5); }
// the adjoint's coefficient vector: one pad per 16, conflict free for every
// lane stride up to 16 (the register level's 16-row segments per lane)
__device__ __forceinline__ int p16(int k) { return k + (k >> 4); }

// staging index of sequency position q: a half-warp (lanes = rows 0..15 or 16..31)
// touches positions 2g + (g & 1) + const, g = 0..15, whose 8-byte banks collide
// pairwise (g, g + 8); flipping bit 0 where bit 4 is set separates them, and
// keeps every aligned pair of positions together (the cooperative copies)
__device__ __forceinline__ int wv_sq(int q) { return q ^ ((q >> 4) & 1); }

// element REL (compile time, may be < 0 or >= P) relative to this lane's first
// sample of a level distributed P per lane (wrapping across lanes 31 <-> 0)
template <int P, int REL>
__device__ __forceinline__ double lane_rel(const double (&c)[P], int lane) {
    if constexpr (REL >= 0 && REL < P) {
        return c[REL];
    } else if constexpr (REL < 0) {
        constexpr int SO = (-REL + P - 1) / P, IDX = REL + SO * P;
        return __shfl_sync(0xffffffffu, c[IDX], (lane - SO) & 31);
    } else {
        constexpr int SO = REL / P, IDX = REL - SO * P;
        return __shfl_sync(0xffffffffu, c[IDX], (lane + SO) & 31);
    }
}

// w[i] = element T0 + i relative to this lane's first sample, i < N
template <int P, int T0, int N, int I = 0>
__device__ __forceinline__ void lane_window(const double (&c)[P], double (&w)[N], int lane) {
    if constexpr (I < N) {
        w[I] = lane_rel<P, T0 + I>(c, lane);
        lane_window<P, T0, N, I + 1>(c, w, lane);
    }
}

template <int NU>
inline long long wv_smem_bytes(int S) {
    return (long long)(FiltSmem<NU>::SIZE + small_ke_size(NU, S) + 2 + kWvV * (kWvXS + S * 2 * (2 * NU - 1))) * 8;
}

// H_A across the lanes (lane = row K, natural order) for every column of r
template <int N>
__device__ __forceinline__ void lane_hadamard(double (&r)[N], int lane) {
#pragma unroll
    for (int b = 0; b < 5; ++b) {
        const bool up = (lane >> b) & 1;
#pragma unroll
        for (int e = 0; e < N; ++e) {
            const double t = __shfl_xor_sync(0xffffffffu, r[e], 1 << b);
            r[e] = up ? t - r[e] : r[e] + t;
        }
    }
}

// elements [off, off + cnt) of the CTA's vectors: vector-fast layouts (v adjacent
// in memory) cooperatively, 8 vectors x 4 consecutive elements per warp access;
// XB[v * kWvXS + k].  Thread tid always serves vector tid & 7 and elements
// k = tid / 8 + 32 i, so its addresses step linearly when the layout's element
// index is linear (esh >= 62: image columns, column panels).  Callers bracket
// with __syncthreads.
template <bool SQ = false>
__device__ __forceinline__ void wv_coop_load(double* XB, const double* in, const Layout& L, long long v0, int nv,
                                             long long off, int cnt, int tid) {
    constexpr int U = 8;
    const int v = tid & (kWvV - 1), k0 = tid / kWvV;
    double* xb = XB + v * kWvXS;
    if (v >= nv) return;
    if (L.esh >= 62) {
        const double* src = in + L.vbase(v0 + v) + (off + k0) * L.es;
        const long long st = 32 * L.es;
        for (int i0 = 0; i0 < cnt / 32; i0 += U) {
            double r[U];
#pragma unroll
            for (int u = 0; u < U; ++u) r[u] = __ldg(src + (i0 + u) * st);
#pragma unroll
            for (int u = 0; u < U; ++u) xb[SQ ? wv_sq(k0 + 32 * (i0 + u)) : k0 + 32 * (i0 + u)] = r[u];
        }
        return;
    }
    for (int k = k0; k < cnt; k += 32) xb[SQ ? wv_sq(k) : k] = __ldg(in + L.at(v0 + v, off + k));
}
template <bool PAD = false, bool SQ = false>
__device__ __forceinline__ void wv_coop_store(const double* XB, double* out, const Layout& L, long long v0, int nv,
                                              long long off, int cnt, int tid) {
    const int v = tid & (kWvV - 1), k0 = tid / kWvV;
    const double* xb = XB + v * kWvXS;
    if (v >= nv) return;
    if (L.esh >= 62) {
        double* dst = out + L.vbase(v0 + v) + (off + k0) * L.es;
        const long long st = 32 * L.es;
#pragma unroll 8
        for (int i = 0; i < cnt / 32; ++i) dst[i * st] = xb[PAD ? p16(k0 + 32 * i) : (SQ ? wv_sq(k0 + 32 * i) : k0 + 32 * i)];
        return;
    }
    for (int k = k0; k < cnt; k += 32) out[L.at(v0 + v, off + k)] = xb[PAD ? p16(k) : (SQ ? wv_sq(k) : k)];
}
// one vector's elements [off, off + cnt) by its own warp (lanes over k):
// contiguous layouts as 16-byte loads, others element-wise
__device__ __forceinline__ void wv_warp_load(double* X, const double* vb, const Layout& L, long long off, int cnt,
                                             int lane) {
    constexpr int U = 8;
    if (L.contig() && ((reinterpret_cast<uintptr_t>(vb + off)) & 15) == 0) {
        const double2* s2 = reinterpret_cast<const double2*>(vb + off);
        double2* d2 = reinterpret_cast<double2*>(X);
        for (int k0 = lane; k0 < cnt / 2; k0 += U * 32) {
            double2 r[U];
#pragma unroll
            for (int u = 0; u < U; ++u) r[u] = k0 + 32 * u < cnt / 2 ? __ldg(s2 + k0 + 32 * u) : make_double2(0.0, 0.0);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (k0 + 32 * u < cnt / 2) d2[k0 + 32 * u] = r[u];
        }
        return;
    }
    for (int k0 = lane; k0 < cnt; k0 += U * 32) {
        double r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) r[u] = k0 + 32 * u < cnt ? __ldg(vb + L.eoff(off + k0 + 32 * u)) : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (k0 + 32 * u < cnt) X[k0 + 32 * u] = r[u];
    }
}

// one analysis level n -> n/2 (n <= 512) in place in the p16-padded
// coefficient vector (c to [0:n/2], d to [n/2:n]); register-staged
template <int NU>
__device__ __forceinline__ void wv_dwt_level(const FiltSmem<NU>& F, const Taps<NU>& tp, double* X, int n, bool vmp,
                                             int lane) {
    constexpr int EL = FiltSmem<NU>::EL;
    constexpr int KM = (1 << (kWvJ - 1)) / 2 / 32;
    const int half = n >> 1;
    auto xv = [&](int i) { return X[p16(i)]; };
    double cc[KM], dd[KM];
    const int rlo = vmp ? NU : 0, rhi = vmp ? half - NU : half;
#pragma unroll
    for (int k = 0; k < KM; ++k) {
        const int mm = rlo + lane + 32 * k;
        if (mm < rhi) {
            double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
            const int i0 = 2 * mm - NU + 1;
            const bool wrap = !vmp && !(i0 >= 0 && i0 + 2 * NU <= n);
#pragma unroll
            for (int u = 0; u < 2 * NU; ++u) {
                const double x = xv(wrap ? ((i0 + u) & (n - 1)) : i0 + u);
                if (u & 1) {
                    a1 = fma(tp.h[u], x, a1);
                    b1 = fma(tp.g[u], x, b1);
                } else {
                    a0 = fma(tp.h[u], x, a0);
                    b0 = fma(tp.g[u], x, b0);
                }
            }
            cc[k] = a0 + a1;
            dd[k] = b0 + b1;
        }
    }
    double ce = 0.0, de = 0.0;  // VMP edge rows mm < NU, mm >= half - NU: one per lane
    if (vmp && lane < 2 * NU) {
        const int side = lane < NU ? 0 : 1;
        const int m = side ? lane - NU : lane;  // row half-1-m on the right
        const double* ra = F.ana(side, 0, m);
        const double* rb = F.ana(side, 1, m);
#pragma unroll
        for (int kk = 0; kk < EL; ++kk) {
            const double x = xv(side ? n - 1 - kk : kk);
            ce = fma(ra[kk], x, ce);
            de = fma(rb[kk], x, de);
        }
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < KM; ++k) {
        const int mm = rlo + lane + 32 * k;
        if (mm < rhi) {
            X[p16(mm)] = cc[k];
            X[p16(half + mm)] = dd[k];
        }
    }
    if (vmp && lane < 2 * NU) {
        const int mm = lane < NU ? lane : half - 1 - (lane - NU);
        X[p16(mm)] = ce;
        X[p16(half + mm)] = de;
    }
    __syncwarp();
}

// one synthesis level n/2 -> n in place in x[0:n] (c = x[0:n/2], d = x[n/2:n]):
// interior pairs from register taps, VMP edge samples one per lane; every lane
// reads first, then the warp writes (padded destination when PADDED)
template <int NU, int KP, bool PADDED>
__device__ __forceinline__ void wv_idwt_level(const FiltSmem<NU>& F, const Taps<NU>& tp, double* x, int n, bool vmp,
                                              int lane) {
    constexpr int EL = FiltSmem<NU>::EL;
    const int np = n >> 1;
    auto dst = [&](int i) -> double& { return x[PADDED ? wv_pad(i) : i]; };
    if (vmp && n < 8 * NU) {  // coarsest VMP levels: the generic edge code for every sample
        double o[2];
#pragma unroll
        for (int k = 0; k < 2; ++k)
            if (lane + 32 * k < n) o[k] = idwt_one<NU>(F, x, x + np, n, lane + 32 * k, true);
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 2; ++k)
            if (lane + 32 * k < n) dst(lane + 32 * k) = o[k];
        __syncwarp();
        return;
    }
    const int mlo = vmp ? (EL + 1) >> 1 : 0, mhi = vmp ? (n - EL) >> 1 : np;
    double o[2 * KP];
    // interior pairs as quads (pairs m, m + 1 from one window of nu + 2 samples,
    // read as 16-byte pairs when the window start m - OFF is even): lane l takes
    // quads l, l + 32, ...; an odd pair count leaves one pair for the last lane
    constexpr int KQ = KP / 2;
    const int nq = (mhi - mlo) >> 1;
    const bool odd = ((mhi - mlo) & 1) != 0;
#pragma unroll
    for (int k = 0; k < KQ; ++k) {
        const int q = lane + 32 * k;
        if (q < nq) idwt_quad_inner<NU>(tp, x, x + np, n, mlo + 2 * q, vmp, o + 4 * k);
    }
    double ol0 = 0.0, ol1 = 0.0;
    if (odd && lane == 31) idwt_pair_inner<NU>(tp, x, x + np, n, mhi - 1, vmp, ol0, ol1);
    const int nl = 2 * mlo, nr = n - 2 * mhi;  // VMP edge samples (<= 36 of them: up to 2 per lane)
    double oe[2] = {0.0, 0.0};
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int k = lane + 32 * r;
        if (k < nl + nr) oe[r] = idwt_one<NU>(F, x, x + np, n, k < nl ? k : 2 * mhi + (k - nl), true);
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < KQ; ++k) {
        const int q = lane + 32 * k;
        if (q < nq) {
            const int m = mlo + 2 * q;
            dst(2 * m) = o[4 * k];
            dst(2 * m + 1) = o[4 * k + 1];
            dst(2 * m + 2) = o[4 * k + 2];
            dst(2 * m + 3) = o[4 * k + 3];
        }
    }
    if (odd && lane == 31) {
        dst(2 * (mhi - 1)) = ol0;
        dst(2 * (mhi - 1) + 1) = ol1;
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int k = lane + 32 * r;
        if (k < nl + nr) dst(k < nl ? k : 2 * mhi + (k - nl)) = oe[r];
    }
    __syncwarp();
}

template <int NU>
__global__ void __launch_bounds__(kWvNT, WV_MINB) k_wv_fwd(SmallArgs p) {
    using G = Geo<NU, kLogB>;
    constexpr int B = G::B, H = G::H, CW = G::CW, NP = G::NP;
    constexpr int M = 1 << kWvJ, A = M >> kLogB, a = kWvJ - kLogB;
    extern __shared__ double sm[];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int S = 1 << p.q;
    const long long v0 = (long long)blockIdx.x * kWvV;
    const int nv = (int)((p.nvec - v0) < kWvV ? (p.nvec - v0) : kWvV);
    const bool act = w < nv;
    double* filt = sm;
    double* KE = filt + FiltSmem<NU>::SIZE;
    double* XB = KE + small_ke_size(NU, S);
    XB += (reinterpret_cast<uintptr_t>(XB) >> 3) & 1;  // 16-byte aligned regions
    double* X = XB + w * kWvXS;
    double* WS = XB + kWvV * kWvXS + w * S * 2 * NP;  // this warp's edge contributions es[S][2NP]
    stage_filters<NU>(filt, p.tab, p.t, tid, kWvNT);
    stage_ke<NU>(KE, p.tab, p.t, S, tid, kWvNT);
    if (p.lin.vfast()) wv_coop_load(XB, p.in, p.lin, v0, nv, 0, M, tid);
    else if (act) wv_warp_load(X, p.in + p.lin.vbase(v0 + w), p.lin, 0, M, lane);
    __syncthreads();
    const FiltSmem<NU> F{filt};
    const bool vmp = NU > 1 && p.vmp != 0;
    const bool idwt = p.use_idwt && p.r0 < kWvJ;
    const double* KAP = KE;
    const double* EM = KE + (2 * NU - 1) * S;
    const bool ovf = p.lout.vfast();
    if (!act && !ovf) return;  // (vector-fast outputs: every warp joins the store barriers)

    double E[CW];
    if (act) {
        // xi = level 10: levels r0+1 .. 9 in place, level 10 written padded
        if (idwt) {
            const Taps<NU> tp(F);
            for (int lev = p.r0 + 1; lev < kWvJ; ++lev) wv_idwt_level<NU, 8, false>(F, tp, X, 1 << lev, vmp, lane);
            wv_idwt_level<NU, 16, true>(F, tp, X, M, vmp, lane);
        } else {  // FastOp: xi is the input itself
            double o[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) o[k] = X[lane + 32 * k];
            __syncwarp();
#pragma unroll
            for (int k = 0; k < 32; ++k) X[wv_pad(lane + 32 * k)] = o[k];
            __syncwarp();
        }
        // extended row K = lane: positions 32 K - H .. 32 K + 32 + H (0 outside [0, M))
#pragma unroll
        for (int e = 0; e < CW; ++e) {
            const int pos = lane * B + e - H;
            E[e] = (pos >= 0 && pos < M) ? X[wv_pad(pos)] : 0.0;
        }
        // edge positions (pos < NU, pos >= M - NU): 0 in the tile; their raw values
        // feed es[s][pos] = sum_c em[s][pos][c] xi_edge[c] (this warp's smem)
        if (NU > 1) {
            for (int f = lane; f < S * 2 * NP; f += 32) {
                const double* em = EM + f * 2 * NU;
                double acc = 0.0;
#pragma unroll
                for (int c = 0; c < 2 * NU; ++c) acc = fma(em[c], X[wv_pad(c < NU ? c : M - NU + (c - NU))], acc);
                WS[f] = acc;
            }
        }
        if (NU > 1 && lane == 0) {
#pragma unroll
            for (int c = 0; c < NU; ++c) E[H + c] = 0.0;
        }
        if (NU > 1 && lane == A - 1) {
#pragma unroll
            for (int c = 0; c < NU; ++c) E[H + B - NU + c] = 0.0;
        }
        lane_hadamard<CW>(E, lane);
    }
    // row stage: lane = logical row N = lane, i.e. physical row wlo = bitrev5(N)
    const int wlo = (int)brev_bits((unsigned)lane, a);
    const double sg = (__popc(lane) & 1) ? -1.0 : 1.0;
    double* ob = p.out + p.lout.vbase(v0 + (act ? w : 0));
    for (int s = 0; s < S; ++s) {
        const unsigned rw = gray_inv((unsigned)wlo) ^ ((s & 1) ? (unsigned)(M - 1) : 0u);
        if (act) {
            double z[B];
            row_fwd<NU, kLogB>(E, wlo, KAP + s, S, NU > 1 ? WS + s * 2 * NP : nullptr, sg, z);
            if (!ovf) {
                row_store<kLogB>(ob + p.lout.eoff((long long)s * M), p.lout, a, rw, z);
            } else {  // block s staged in the region (sequency positions), stored by the CTA
#pragma unroll
                for (int nl = 0; nl < B; ++nl) X[wv_sq((int)(gray_inv_hi(nl, kLogB, a) ^ rw))] = z[nl];
            }
        }
        if (ovf) {
            __syncthreads();
            wv_coop_store<false, true>(XB, p.out, p.lout, v0, nv, (long long)s * M, M, tid);
            __syncthreads();
        }
    }
}

template <int NU>
__global__ void __launch_bounds__(kWvNT, WV_MINB) k_wv_adj(SmallArgs p) {
    using G = Geo<NU, kLogB>;
    constexpr int B = G::B, H = G::H, CW = G::CW, NP = G::NP;
    constexpr int M = 1 << kWvJ, A = M >> kLogB, a = kWvJ - kLogB;
    constexpr int EL = FiltSmem<NU>::EL;
    extern __shared__ double sm[];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int S = 1 << p.q;
    const long long v0 = (long long)blockIdx.x * kWvV;
    const int nv = (int)((p.nvec - v0) < kWvV ? (p.nvec - v0) : kWvV);
    const bool act = w < nv;
    double* filt = sm;
    double* KE = filt + FiltSmem<NU>::SIZE;
    double* XB = KE + small_ke_size(NU, S);
    XB += (reinterpret_cast<uintptr_t>(XB) >> 3) & 1;
    double* X = XB + w * kWvXS;
    double* WS = XB + kWvV * kWvXS + w * S * 2 * NP;  // this warp's edge sums [S][2NP]
    stage_filters<NU>(filt, p.tab, p.t, tid, kWvNT);
    stage_ke<NU>(KE, p.tab, p.t, S, tid, kWvNT);
    __syncthreads();
    const bool ivf = p.lin.vfast(), ovf = p.lout.vfast();
    if (!act && !ivf && !ovf) return;
    const FiltSmem<NU> F{filt};
    const bool vmp = NU > 1 && p.vmp != 0;
    const double* KAP = KE;
    const double* EM = KE + (2 * NU - 1) * S;
    const int wlo = (int)brev_bits((unsigned)lane, a);  // lane = logical row N
    const double sg = (__popc(lane) & 1) ? -1.0 : 1.0;
    const double* ib = p.in + p.lin.vbase(v0 + (act ? w : 0));
    double acc[CW];
#pragma unroll
    for (int e = 0; e < CW; ++e) acc[e] = 0.0;
    for (int s = 0; s < S; ++s) {
        const unsigned rw = gray_inv((unsigned)wlo) ^ ((s & 1) ? (unsigned)(M - 1) : 0u);
        if (ivf) {  // block s of the CTA's vectors through the regions
            if (s > 0) __syncthreads();
            wv_coop_load<true>(XB, p.in, p.lin, v0, nv, (long long)s * M, M, tid);
            __syncthreads();
        }
        if (!act) continue;
        double y[B];
        if (ivf) {
#pragma unroll
            for (int nl = 0; nl < B; ++nl) y[nl] = X[wv_sq((int)(gray_inv_hi(nl, kLogB, a) ^ rw))];
        } else {
            row_load<kLogB>(ib + p.lin.eoff((long long)s * M), p.lin, a, rw, true, y);
        }
        hadamard_reg<kLogB>(y);
        if (NU > 1) {  // edge sums over the rows: W[s][i] = sum_N (i < NP ? y[i] : sg y[B-NP+i-NP]),
                       // through this warp's region (free here), rows summed in order
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 2 * NP; ++i) X[i * 33 + lane] = i < NP ? y[i] : sg * y[B - NP + (i - NP)];
            __syncwarp();
            if (lane < 2 * NP) {
                double t0 = 0.0, t1 = 0.0;
#pragma unroll
                for (int l = 0; l < 32; l += 2) {
                    t0 += X[lane * 33 + l];
                    t1 += X[lane * 33 + l + 1];
                }
                WS[s * 2 * NP + lane] = t0 + t1;
            }
            __syncwarp();
        }
        row_adj_accum<NU, kLogB>(acc, wlo, KAP + s, S, y, false);
    }
    if (ivf) __syncthreads();  // the regions are this warp's again
    double* ob = p.out + p.lout.vbase(v0 + (act ? w : 0));
    if (act) {
        lane_hadamard<CW>(acc, lane);
        // overlap-add: xi[32 K + c] = acc[H + c] + right halo of row K - 1 (c < H)
        // + left halo of row K + 1 (c >= B - H)
        double xi[B];
#pragma unroll
        for (int c = 0; c < B; ++c) xi[c] = acc[H + c];
#pragma unroll
        for (int c = 0; c < H; ++c) {
            const double fromprev = __shfl_up_sync(0xffffffffu, acc[B + H + c], 1);
            const double fromnext = __shfl_down_sync(0xffffffffu, acc[c], 1);
            if (lane > 0) xi[c] += fromprev;
            if (lane < A - 1) xi[B - H + c] += fromnext;
        }
        __syncwarp();  // WS visible
        if (NU > 1 && (lane == 0 || lane == A - 1)) {  // edge positions: sum_sp em[sp][c] W[sp]
#pragma unroll
            for (int k = 0; k < NU; ++k) {
                const int c = lane == 0 ? k : NU + k;
                const double* em = EM + c;
                double e0 = 0.0, e1 = 0.0;
                const int nsp = S * 2 * NP;
                int sp = 0;
                for (; sp + 2 <= nsp; sp += 2) {
                    e0 = fma(em[sp * 2 * NU], WS[sp], e0);
                    e1 = fma(em[(sp + 1) * 2 * NU], WS[sp + 1], e1);
                }
                if (sp < nsp) e0 = fma(em[sp * 2 * NU], WS[sp], e0);
                xi[lane == 0 ? k : B - NU + k] = e0 + e1;
            }
        }
        const bool dwt = p.use_idwt && p.r0 < kWvJ;
        if (!dwt) {  // FastOp adjoint: xi is the output
#pragma unroll
            for (int c = 0; c < B; ++c) X[p16(lane * B + c)] = xi[c];
        } else {
            // level 10 -> 9 straight from the rows in registers (lane l: rows 16 l ..
            // 16 l + 15 from xi[32 l - NU + 1 .. 32 l + 31 + NU], halos by shuffles),
            // c_9 and d_9 into the p16-padded coefficient vector; then levels
            // 9 .. r0 + 1 in place there, which ends as [c_r0 | d_r0 | ... | d_9]
            const Taps<NU> tp(F);
            constexpr int WN = B + 2 * NU - 2;
            double xw[WN];
            lane_window<B, -NU + 1, WN>(xi, xw, lane);
#pragma unroll
            for (int t = 0; t < B / 2; ++t) {
                const int mm = (B / 2) * lane + t;
                double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
                for (int u = 0; u < 2 * NU; ++u) {
                    const double x = xw[2 * t + u];
                    if (u & 1) {
                        a1 = fma(tp.h[u], x, a1);
                        b1 = fma(tp.g[u], x, b1);
                    } else {
                        a0 = fma(tp.h[u], x, a0);
                        b0 = fma(tp.g[u], x, b0);
                    }
                }
                X[p16(mm)] = a0 + a1;
                X[p16(M / 2 + mm)] = b0 + b1;
            }
            if (vmp && (lane == 0 || lane == A - 1)) {  // VMP edge rows: dense rows over this lane's own samples
                const int side = lane == 0 ? 0 : 1;
                constexpr int EL = FiltSmem<NU>::EL;
#pragma unroll
                for (int m = 0; m < NU; ++m) {
                    const double* ra = F.ana(side, 0, m);
                    const double* rb = F.ana(side, 1, m);
                    double ce = 0.0, de = 0.0;
#pragma unroll
                    for (int kk = 0; kk < EL; ++kk) {
                        const double x = side ? xi[B - 1 - kk] : xi[kk];
                        ce = fma(ra[kk], x, ce);
                        de = fma(rb[kk], x, de);
                    }
                    const int mm = side ? M / 2 - 1 - m : m;
                    X[p16(mm)] = ce;
                    X[p16(M / 2 + mm)] = de;
                }
            }
            __syncwarp();
            for (int n = M / 2; n > (1 << p.r0); n >>= 1) wv_dwt_level<NU>(F, tp, X, n, vmp, lane);
        }
        __syncwarp();
    }
    if (!ovf) {
        if (act) {
#pragma unroll 8
            for (int k = lane; k < M; k += 32) ob[p.lout.eoff(k)] = X[p16(k)];
        }
        return;
    }
    __syncthreads();
    wv_coop_store<true>(XB, p.out, p.lout, v0, nv, 0, M, tid);
}

}  // namespace cww
