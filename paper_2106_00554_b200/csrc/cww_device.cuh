// Device building blocks of the sm_100a Walsh->wavelet operator.
//
// Algorithm.  With M = 2^j, N = 2^(j+q), S = 2^q and the
// position index split k = K*B + k_lo (B = 2^b, A = 2^a, a = j - b), the
// reference's forward product (fastop.cpp:100-137: 2nu-1 N-point FWHTs +
// permuted gathers + 4nu-2 edge axpys) is computed as
//
//   Xi~   = (H_A (x) I_B) applied to the overlapped "extended tile"
//           E[K][e] = xi_int[K*B + e - h],  e in [0, B + 2h), h = nu - 1
//   z_s[N][k]  = sum_l kap_l(s) Xi~[N][k - l + h]  (+ edge terms)        (stencil)
//   alpha_s[r] = (H_B z_s[N])[n_lo],  r = gray^-1(bitrev_j(N*B + n_lo)),
//                r -> M-1-r for odd s                                    (sequency write)
//
// H_A is shared by all 2^q blocks s, so the fp64 butterfly count per input
// element is a(1 + 2h/B) + S*b instead of the reference's 2(2nu-1)(j+q).
// The adjoint (fastop.cpp:139-175) is the exact transpose of every step.
// kap is pre-scaled by 2^(-j/2); the odd-s sign pattern sigma_s is applied as
// an index reversal (FWHT_seq(sigma . z)[r] = FWHT_seq(z)[M-1-r]).
#pragma once
#include <cstdint>

namespace cww {

constexpr int kMaxNu = 6;
constexpr int kLogB = 5;  // row length B = 32 for j >= 5

// ---- per-op constant tables (device global memory, see cww_host.cpp) -------
struct Tables {
    // offsets (in doubles) into the table block
    int o_kap;  // [2h+1][S]   kap[(l+h)*S + s] = 2^(-j/2) kappa_l(s)
    int o_em;   // [S][2(2nu-1)][2nu]  edge matrix (positions x edge columns), scaled
    int o_h;    // [2nu] hbar_u, u = -nu+1..nu
    int o_g;    // [2nu] gbar_u
    int o_ef;   // [2][ A(nu*nu) | B(nu*(2nu-1)) | Aw | Bw ]  left, right
    int o_syn;  // [2 sides][3nu-1][2 bands][2nu]  dense synthesis edge blocks
    int o_ana;  // [2 sides][2 bands][nu][3nu-1]   dense analysis edge rows
    int n;      // total doubles
};

// Generic strided/tiled address of element i of vector v (in doubles):
//   (v >> vsh)*vb + (v & vmask)*vs + (i >> esh)*eb + (i & emask)*es
struct Layout {
    long long vb, vs, eb, es;
    int vsh, esh;
    __host__ __device__ long long at(long long v, long long i) const {
        long long vm = (vsh >= 62) ? v : (v & ((1ll << vsh) - 1));
        long long vh = (vsh >= 62) ? 0 : (v >> vsh);
        long long im = (esh >= 62) ? i : (i & ((1ll << esh) - 1));
        long long ih = (esh >= 62) ? 0 : (i >> esh);
        return vh * vb + vm * vs + ih * eb + im * es;
    }
    __host__ __device__ long long vbase(long long v) const {
        return (vsh >= 62) ? v * vs : (v >> vsh) * vb + (v & ((1ll << vsh) - 1)) * vs;
    }
    __host__ __device__ long long eoff(long long i) const {
        return (esh >= 62) ? i * es : (i >> esh) * eb + (i & ((1ll << esh) - 1)) * es;
    }
    __host__ __device__ bool contig() const { return esh >= 62 && es == 1; }
    // consecutive vectors are adjacent in memory: lanes should vary v first
    __host__ __device__ bool vfast() const { return vs == 1; }
};

__device__ __forceinline__ unsigned brev_bits(unsigned v, int bits) {
    return bits == 0 ? 0u : (__brev(v) >> (32 - bits));
}

__device__ __forceinline__ unsigned gray_inv(unsigned g) {
    g ^= g >> 1;
    g ^= g >> 2;
    g ^= g >> 4;
    g ^= g >> 8;
    g ^= g >> 16;
    return g;
}

// Extended-tile geometry for compile-time NU / LOGB.
template <int NU, int LOGB>
struct Geo {
    static constexpr int B = 1 << LOGB;
    static constexpr int H = NU - 1;
    static constexpr int CW = B + 2 * H;             // used columns per row
    static constexpr int RS = CW | 1;                // odd smem row stride: conflict-free for
                                                     // both row-wise and column-wise lanes
    static constexpr int NP = 2 * NU - 1;            // edge positions per side
    // large strided passes: even row stride (16-byte aligned rows for the bulk
    // copies), = 2 (mod 4) so row-per-lane reads are at most 2-way conflicted
    static constexpr int RSL = (CW % 4 == 2) ? CW : CW + 2;
};

// Tile element (physical row, e) lives at row * RS + e with an odd row
// stride RS, which is bank-conflict free both for lanes that walk a row and
// for lanes that walk consecutive rows.  Tiles store logical row K at physical row bitrev_a(K): the
// Hadamard matrix is invariant under reversing the bits of both indices, so
// H_A runs on physical rows with plain strides and the row stage reads
// physical row w (= logical N = bitrev(w)) for consecutive lanes w.
__device__ __forceinline__ int tile_idx(int row, int e, int RS, int sw) {
    (void)sw;
    return row * RS + e;
}

// In-register natural-order Hadamard butterflies over R bits.
template <int R>
__device__ __forceinline__ void hadamard_reg(double* x) {
#pragma unroll
    for (int hb = 0; hb < R; ++hb) {
        const int h = 1 << hb;
#pragma unroll
        for (int i = 0; i < (1 << R); ++i) {
            if ((i & h) == 0) {
                double a = x[i], b = x[i + h];
                x[i] = a + b;
                x[i + h] = a - b;
            }
        }
    }
}

// One radix-2^R pass of H_A along the physical row index of V tiles held in
// smem (rows 0..2^a-1, columns 0..CW-1), over row bits [lo, lo+R).
template <int R, int CW, int RS>
__device__ __forceinline__ void tile_hadamard_pass(double* T, int V, int a, int lo, int tstride,
                                                   int tid, int nt) {
    const int groups = (1 << a) >> R;
    const int items = V * CW * groups;
    // (e, rest) = (it % CW, it / CW), stepped incrementally (no division per item)
    int e = tid % CW, rest = tid / CW;
    const int de = nt % CW, dr = nt / CW;
    for (int it = tid; it < items; it += nt) {
        const int fb = rest & (groups - 1);
        const int v = rest >> (a - R);
        const int low = fb & ((1 << lo) - 1);
        const int row0 = ((fb >> lo) << (lo + R)) | low;
        double* t = T + v * tstride + row0 * RS + e;
        double x[1 << R];
#pragma unroll
        for (int k = 0; k < (1 << R); ++k) x[k] = t[(k << lo) * RS];
        hadamard_reg<R>(x);
#pragma unroll
        for (int k = 0; k < (1 << R); ++k) t[(k << lo) * RS] = x[k];
        e += de;
        rest += dr;
        if (e >= CW) {
            e -= CW;
            ++rest;
        }
    }
}

// H_A restricted to row bits [lo, hi), passes of <= MAXR bits (registers:
// 2^MAXR doubles per thread), __syncthreads after each.  Inlined variant
// (no call frame) for kernels whose register budget is tight.
template <int CW, int RS, int MAXR = 5>
__device__ __forceinline__ void tile_hadamard_inl(double* T, int V, int a, int lo, int hi, int tstride,
                                                  int tid, int nt) {
    static_assert(MAXR >= 1 && MAXR <= 5, "pass width");
    while (lo < hi) {
        const int r = hi - lo < MAXR ? hi - lo : MAXR;
        // only passes of <= MAXR bits are instantiated (register budget)
        if (r == 1) tile_hadamard_pass<1, CW, RS>(T, V, a, lo, tstride, tid, nt);
        else if (MAXR >= 2 && r == 2) tile_hadamard_pass<(MAXR >= 2 ? 2 : 1), CW, RS>(T, V, a, lo, tstride, tid, nt);
        else if (MAXR >= 3 && r == 3) tile_hadamard_pass<(MAXR >= 3 ? 3 : 1), CW, RS>(T, V, a, lo, tstride, tid, nt);
        else if (MAXR >= 4 && r == 4) tile_hadamard_pass<(MAXR >= 4 ? 4 : 1), CW, RS>(T, V, a, lo, tstride, tid, nt);
        else tile_hadamard_pass<MAXR, CW, RS>(T, V, a, lo, tstride, tid, nt);
        __syncthreads();
        lo += r;
    }
}

template <int CW, int RS, int MAXR = 5>
__device__ __noinline__ void tile_hadamard(double* T, int V, int a, int lo, int hi, int tstride,
                                           int tid, int nt) {
    while (lo < hi) {
        const int r = hi - lo < MAXR ? hi - lo : MAXR;
        switch (r) {
            case 1: tile_hadamard_pass<1, CW, RS>(T, V, a, lo, tstride, tid, nt); break;
            case 2: tile_hadamard_pass<2, CW, RS>(T, V, a, lo, tstride, tid, nt); break;
            case 3: tile_hadamard_pass<3, CW, RS>(T, V, a, lo, tstride, tid, nt); break;
            case 4: tile_hadamard_pass<4, CW, RS>(T, V, a, lo, tstride, tid, nt); break;
            default: tile_hadamard_pass<5, CW, RS>(T, V, a, lo, tstride, tid, nt); break;
        }
        __syncthreads();
        lo += r;
    }
}

// ---- wavelet levels (gather form of wavelet.cpp:367-483) --------------------
// Filters staged in shared memory: h[2nu], g[2nu], then per side
// A[nu*nu], B[nu*(2nu-1)], Aw[nu*nu], Bw[nu*(2nu-1)].
template <int NU>
struct FiltSmem {
    static constexpr int W = 2 * NU - 1;
    static constexpr int SIDE = 2 * NU * NU + 2 * NU * W;
    static constexpr int EL = 3 * NU - 1;  // edge-region width of one level
    static constexpr int CI = 2 * NU;      // coarse/detail inputs an edge sample reads
    static constexpr int SYN = 2 * EL * 2 * CI;
    static constexpr int ANA = 2 * 2 * NU * EL;
    static constexpr int SIZE = 4 * NU + 2 * SIDE + SYN + ANA;
    const double* f;
    // dense synthesis edge block, layout [side][band][k][i]: coefficient of
    // c[k] (band 0) / d[k] (band 1) in edge sample i is syn(side, i, band)[k * EL]
    __device__ const double* syn(int side, int i, int band) const {
        return f + 4 * NU + 2 * SIDE + (side * 2 + band) * CI * EL + i;
    }
    // dense analysis edge row m (band 0 coarse, 1 detail)
    __device__ const double* ana(int side, int band, int m) const {
        return f + 4 * NU + 2 * SIDE + SYN + ((side * 2 + band) * NU + m) * EL;
    }
    __device__ double h(int u) const { return f[u + NU - 1]; }
    __device__ double g(int u) const { return f[2 * NU + u + NU - 1]; }
    __device__ const double* A(int side) const { return f + 4 * NU + side * SIDE; }
    __device__ const double* Bm(int side) const { return A(side) + NU * NU; }
    __device__ const double* Aw(int side) const { return Bm(side) + NU * W; }
    __device__ const double* Bw(int side) const { return Aw(side) + NU * NU; }
};

// Synthesis (one IDWT level): fine sample i of a length-n level from
// c = x[0:n/2], d = x[n/2:n].
template <int NU>
__device__ __noinline__ double idwt_sample_full2(const FiltSmem<NU> F, const double* c,
                                                 const double* d, int n, int i, bool vmp) {
    const int half = n >> 1;
    double acc = 0.0;
    if (!vmp) {  // periodic: scratch[(2mm+u) mod n] += hbar c + gbar d (387-400)
#pragma unroll
        for (int k = 0; k < NU; ++k) {
            int u = -NU + 1 + 2 * k + ((i + NU + 1) & 1);  // u == i (mod 2)
            int t = i - u;
            t %= n;
            if (t < 0) t += n;
            int mm = t >> 1;
            acc += F.h(u) * c[mm] + F.g(u) * d[mm];
        }
        return acc;
    }
    // interior columns nu <= mm < half-nu (475-481)
#pragma unroll
    for (int k = 0; k < NU; ++k) {
        int u = -NU + 1 + 2 * k + ((i + NU + 1) & 1);
        int mm = (i - u) >> 1;
        if (mm >= NU && mm < half - NU) acc += F.h(u) * c[mm] + F.g(u) * d[mm];
    }
    constexpr int W = 2 * NU - 1;
    // left and right edge columns (edge_cols, 454-473)
#pragma unroll
    for (int side = 0; side < 2; ++side) {
        int ii = side ? n - 1 - i : i;
        if (ii < 3 * NU - 1) {
            const double* A = F.A(side);
            const double* Aw = F.Aw(side);
            const double* Bm = F.Bm(side);
            const double* Bw = F.Bw(side);
#pragma unroll
            for (int m = 0; m < NU; ++m) {
                int row = side ? half - 1 - m : m;
                double cm = c[row], dm = d[row];
                if (ii < NU) {
                    acc += A[m * NU + ii] * cm + Aw[m * NU + ii] * dm;
                } else {
                    int li = ii - NU;
                    if (li <= 2 * m) acc += Bm[m * W + li] * cm + Bw[m * W + li] * dm;
                }
            }
        }
    }
    return acc;
}

// Analysis (one DWT level): output o of a length-n level (coarse o < n/2,
// detail o >= n/2) from the fine samples x[0:n] (369-385, 403-445).
template <int NU>
__device__ __noinline__ double dwt_sample_full(const FiltSmem<NU> F, const double* x, int n, int o,
                                               bool vmp) {
    const int half = n >> 1;
    const bool det = o >= half;
    const int mm = det ? o - half : o;
    double acc = 0.0;
    if (!vmp) {
#pragma unroll
        for (int u = -NU + 1; u <= NU; ++u) {
            int t = 2 * mm + u;
            t %= n;
            if (t < 0) t += n;
            acc += (det ? F.g(u) : F.h(u)) * x[t];
        }
        return acc;
    }
    constexpr int W = 2 * NU - 1;
    if (mm < NU || mm >= half - NU) {
        int side = mm < NU ? 0 : 1;
        int m = side ? half - 1 - mm : mm;
        const double* A = det ? F.Aw(side) : F.A(side);
        const double* Bm = det ? F.Bw(side) : F.Bm(side);
#pragma unroll
        for (int k = 0; k < NU; ++k) acc += A[m * NU + k] * x[side ? n - 1 - k : k];
#pragma unroll
        for (int li = 0; li < W; ++li)
            if (li <= 2 * m) acc += Bm[m * W + li] * x[side ? n - 1 - NU - li : NU + li];
        return acc;
    }
#pragma unroll
    for (int u = -NU + 1; u <= NU; ++u) acc += (det ? F.g(u) : F.h(u)) * x[2 * mm + u];
    return acc;
}

// Interior synthesis/analysis taps held in registers.
template <int NU>
struct Taps {
    double h[2 * NU], g[2 * NU];
    __device__ __forceinline__ explicit Taps(const FiltSmem<NU>& F) {
#pragma unroll
        for (int k = 0; k < 2 * NU; ++k) {
            h[k] = F.f[k];
            g[k] = F.f[2 * NU + k];
        }
    }
};

// Synthesis of one fine sample i of a length-n level from c = cv[0:n/2],
// d = dv[0:n/2].  Periodic: masked (mod n) indices, exact everywhere.  VMP:
// the interior formula for 3nu-1 <= i <= n-3nu; the first/last 3nu-1 samples
// from the dense level-independent edge blocks (valid for n >= 8nu); the
// generic edge code only for the few coarsest levels (n < 8nu).
template <int NU>
__device__ __forceinline__ double idwt_one(const FiltSmem<NU>& F, const double* cv, const double* dv,
                                           int n, int i, bool vmp) {
    const int half = n >> 1;
    const int par = (i + NU + 1) & 1;
    if (!vmp) {
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int k = 0; k < NU; ++k) {
            const int u = -NU + 1 + 2 * k + par;
            const int mm = ((i - u) & (n - 1)) >> 1;
            a0 = fma(F.h(u), cv[mm], a0);
            a1 = fma(F.g(u), dv[mm], a1);
        }
        return a0 + a1;
    }
    constexpr int EL = FiltSmem<NU>::EL, CI = FiltSmem<NU>::CI;
    if (n < 8 * NU) return idwt_sample_full2<NU>(F, cv, dv, n, i, vmp);
    if (i < EL || i >= n - EL) {
        const int side = i < EL ? 0 : 1;
        const int ii = side ? n - 1 - i : i;
        const double* sc = F.syn(side, ii, 0);
        const double* sd = F.syn(side, ii, 1);
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;  // four short chains (latency)
#pragma unroll
        for (int k = 0; k < CI; ++k) {
            const int idx = side ? half - 1 - k : k;
            if (k & 1) {
                a1 = fma(sc[k * EL], cv[idx], a1);
                b1 = fma(sd[k * EL], dv[idx], b1);
            } else {
                a0 = fma(sc[k * EL], cv[idx], a0);
                b0 = fma(sd[k * EL], dv[idx], b0);
            }
        }
        return (a0 + a1) + (b0 + b1);
    }
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int k = 0; k < NU; ++k) {
        const int u = -NU + 1 + 2 * k + par;
        const int mm = (i - u) >> 1;
        a0 = fma(F.h(u), cv[mm], a0);
        a1 = fma(F.g(u), dv[mm], a1);
    }
    return a0 + a1;
}

// Paired synthesis: fine samples 2m and 2m+1 share one window of nu+1 coarse
// and nu+1 detail samples (periodic: masked indices, always; VMP: interior
// pairs), otherwise two single samples.
template <int NU>
__device__ __forceinline__ void idwt_pair(const FiltSmem<NU>& F, const double* cv, const double* dv,
                                          int n, int m, bool vmp, double& o0, double& o1) {
    const int i = 2 * m;
    const int half = n >> 1;
    const bool inner = !vmp || (i >= 3 * NU - 1 && i + 1 <= n - 3 * NU);
    if (inner) {
        constexpr int OFF = (NU + 1) / 2;  // window c[m-OFF .. m-OFF+NU]
        double cw[NU + 1], dw[NU + 1];
#pragma unroll
        for (int k = 0; k <= NU; ++k) {
            const int idx = vmp ? m - OFF + k : ((m - OFF + k) & (half - 1));
            cw[k] = cv[idx];
            dw[k] = dv[idx];
        }
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int u = -NU + 1; u <= NU; ++u) {
            if ((u & 1) == 0) {  // even u feeds the even sample: mm = m - u/2
                const int idx = OFF - u / 2;
                a0 += F.h(u) * cw[idx] + F.g(u) * dw[idx];
            } else {  // odd u feeds the odd sample: mm = m - (u-1)/2
                const int idx = OFF - (u - 1) / 2;
                a1 += F.h(u) * cw[idx] + F.g(u) * dw[idx];
            }
        }
        o0 = a0;
        o1 = a1;
        return;
    }
    o0 = idwt_one<NU>(F, cv, dv, n, i, vmp);
    o1 = idwt_one<NU>(F, cv, dv, n, i + 1, vmp);
}

// Interior pair with register taps (caller guarantees the pair is interior
// for VMP; periodic: masked indices, any pair).
template <int NU>
__device__ __forceinline__ void idwt_pair_inner(const Taps<NU>& tp, const double* cv, const double* dv,
                                                int n, int m, bool vmp, double& o0, double& o1) {
    constexpr int OFF = (NU + 1) / 2;
    const int half = n >> 1;
    double cw[NU + 1], dw[NU + 1];
#pragma unroll
    for (int k = 0; k <= NU; ++k) {
        const int idx = vmp ? m - OFF + k : ((m - OFF + k) & (half - 1));
        cw[k] = cv[idx];
        dw[k] = dv[idx];
    }
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;  // four independent chains
#pragma unroll
    for (int u = -NU + 1; u <= NU; ++u) {
        if ((u & 1) == 0) {
            const int idx = OFF - u / 2;
            a0 += tp.h[u + NU - 1] * cw[idx];
            b0 += tp.g[u + NU - 1] * dw[idx];
        } else {
            const int idx = OFF - (u - 1) / 2;
            a1 += tp.h[u + NU - 1] * cw[idx];
            b1 += tp.g[u + NU - 1] * dw[idx];
        }
    }
    o0 = a0 + b0;
    o1 = a1 + b1;
}

// Two interior pairs (samples 2m .. 2m+3) from one window of nu+2 coarse and
// nu+2 detail samples (periodic: masked indices).
template <int NU>
__device__ __forceinline__ void idwt_quad_inner(const Taps<NU>& tp, const double* cv, const double* dv,
                                                int n, int m, bool vmp, double* o) {
    constexpr int OFF = (NU + 1) / 2;
    const int half = n >> 1;
    constexpr int NW = (NU + 3) / 2;  // double2 pairs covering the nu + 2 window
    double cw[2 * NW], dw[2 * NW];
    const double* c0 = cv + (m - OFF);
    const double* d0 = dv + (m - OFF);
    if (vmp && ((reinterpret_cast<uintptr_t>(c0) | reinterpret_cast<uintptr_t>(d0)) & 15) == 0) {
        // 16-byte aligned windows (lanes 2 pairs apart): half the shared-memory
        // wavefronts of the scalar loads (the extra sample of an odd window stays
        // inside the level: m + 2 + nu - OFF < half for interior quads)
#pragma unroll
        for (int k = 0; k < NW; ++k) {
            const double2 a = reinterpret_cast<const double2*>(c0)[k];
            const double2 b = reinterpret_cast<const double2*>(d0)[k];
            cw[2 * k] = a.x;
            cw[2 * k + 1] = a.y;
            dw[2 * k] = b.x;
            dw[2 * k + 1] = b.y;
        }
    } else {
#pragma unroll
        for (int k = 0; k <= NU + 1; ++k) {
            const int idx = vmp ? m - OFF + k : ((m - OFF + k) & (half - 1));
            cw[k] = cv[idx];
            dw[k] = dv[idx];
        }
    }
#pragma unroll
    for (int p = 0; p < 2; ++p) {  // pair m + p: window shifted by p
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
        for (int u = -NU + 1; u <= NU; ++u) {
            if ((u & 1) == 0) {
                const int idx = OFF - u / 2 + p;
                a0 += tp.h[u + NU - 1] * cw[idx];
                b0 += tp.g[u + NU - 1] * dw[idx];
            } else {
                const int idx = OFF - (u - 1) / 2 + p;
                a1 += tp.h[u + NU - 1] * cw[idx];
                b1 += tp.g[u + NU - 1] * dw[idx];
            }
        }
        o[2 * p] = a0 + b0;
        o[2 * p + 1] = a1 + b1;
    }
}

// Analysis: coarse and detail row mm of a length-n level from x[0:n].
// Periodic: masked indices.  VMP: interior rows use the 2nu taps, the nu
// edge rows per side the dense [A|B] / [Aw|Bw] rows (any level n >= 4nu).
template <int NU>
__device__ __forceinline__ void dwt_pair(const FiltSmem<NU>& F, const double* x, int n, int mm,
                                         bool vmp, double& c, double& d) {
    const int half = n >> 1;
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;  // two chains per output (latency)
    if (!vmp) {
#pragma unroll
        for (int u = -NU + 1; u <= NU; ++u) {
            const double xv = x[(2 * mm + u) & (n - 1)];
            if (u & 1) {
                a1 = fma(F.h(u), xv, a1);
                b1 = fma(F.g(u), xv, b1);
            } else {
                a0 = fma(F.h(u), xv, a0);
                b0 = fma(F.g(u), xv, b0);
            }
        }
    } else if (mm >= NU && mm < half - NU) {
#pragma unroll
        for (int u = -NU + 1; u <= NU; ++u) {
            const double xv = x[2 * mm + u];
            if (u & 1) {
                a1 = fma(F.h(u), xv, a1);
                b1 = fma(F.g(u), xv, b1);
            } else {
                a0 = fma(F.h(u), xv, a0);
                b0 = fma(F.g(u), xv, b0);
            }
        }
    } else {
        constexpr int EL = FiltSmem<NU>::EL;
        const int side = mm < NU ? 0 : 1;
        const int m = side ? half - 1 - mm : mm;
        const double* ra = F.ana(side, 0, m);
        const double* rb = F.ana(side, 1, m);
#pragma unroll
        for (int k = 0; k < EL; ++k) {
            const double xv = x[side ? n - 1 - k : k];
            if (k & 1) {
                a1 = fma(ra[k], xv, a1);
                b1 = fma(rb[k], xv, b1);
            } else {
                a0 = fma(ra[k], xv, a0);
                b0 = fma(rb[k], xv, b0);
            }
        }
    }
    c = a0 + a1;
    d = b0 + b1;
}


// Asynchronous 16-byte global -> shared copy (both addresses 16-byte aligned).
__device__ __forceinline__ void cp_async16(double* sdst, const double* gsrc) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gsrc) : "memory");
}

// Asynchronous 8-byte global -> shared copy (LDGSTS): many loads in flight
// per thread without register staging.
__device__ __forceinline__ void cp_async8(double* sdst, const double* gsrc) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// ---- bulk copies (TMA engine: cp.async.bulk, SASS UBLKCP) + mbarrier ---------
// global -> shared copies complete on an mbarrier (transaction bytes); shared
// -> global copies are tracked per thread with bulk groups.  Addresses 16-byte
// aligned, sizes multiples of 16.
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
// arrive (count 1) and add `bytes` to the transactions the current phase waits for
__device__ __forceinline__ void mbar_arrive_expect(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_addr(sdst)),
        "l"(gsrc), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst), "r"(smem_addr(ssrc)),
                 "r"(bytes)
                 : "memory");
}
// L2 prefetch of bytes (multiple of 16) at a 16-byte aligned global address
__device__ __forceinline__ void l2_prefetch(const void* gsrc, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(gsrc), "r"(bytes) : "memory");
}
// L2 prefetch of the doubles [src, src + n) clipped to [lim_lo, lim_hi) and
// widened to 16-byte granules inside those limits
__device__ __forceinline__ void l2_prefetch_span(const double* src, int n, const double* lim_lo,
                                                 const double* lim_hi) {
    uintptr_t a = reinterpret_cast<uintptr_t>(src < lim_lo ? lim_lo : src);
    uintptr_t b = reinterpret_cast<uintptr_t>(src + n > lim_hi ? lim_hi : src + n);
    a = (a + 15) & ~uintptr_t(15);
    b &= ~uintptr_t(15);
    if (b > a) l2_prefetch(reinterpret_cast<const void*>(a), (unsigned)(b - a));
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
// this thread's bulk stores have finished READING shared memory
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
// make this thread's generic-proxy shared-memory writes visible to the async proxy
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// ---- window geometry of the multilevel (pyramid) wavelet kernels ------------
// Index ranges [lo, hi).  Periodic ranges are LOGICAL (may start below 0 or end
// past the level length; entries are read modulo the length): periodic
// synthesis and analysis are translation-equivariant, so a window never needs
// to be clipped or collapsed.  VMP ranges are physical (clipped).
struct Win {
    int lo, hi;
};

// Coarse/detail window (level n/2) read by the synthesis of fine samples f of
// level n (wavelet.cpp:447-483 in gather form).  VMP: the first/last 3nu-1
// fine samples read coarse entries [0, 2nu) / [n/2-2nu, n/2) (dense edge
// blocks); levels n < 8nu use the generic edge code on the whole level.
__host__ __device__ inline Win syn_need(int nu, int n, Win f, bool vmp) {
    const int half = n >> 1;
    Win c{(f.lo - nu) >> 1, ((f.hi + nu - 2) >> 1) + 1};
    if (!vmp) return c;
    if (n < 8 * nu) return Win{0, half};
    const int EL = 3 * nu - 1, CI = 2 * nu;
    if (c.lo < 0) c.lo = 0;
    if (c.hi > half) c.hi = half;
    if (f.lo < EL) {
        c.lo = 0;
        if (c.hi < CI) c.hi = CI;
    }
    if (f.hi > n - EL) {
        c.hi = half;
        if (c.lo > half - CI) c.lo = half - CI;
    }
    return c;
}

// Fine window (level n) read by the analysis of coarse/detail rows r of a
// length-n level (wavelet.cpp:369-385, 403-445).  VMP edge rows (the first /
// last nu) read the first / last 3nu-1 fine samples.
__host__ __device__ inline Win ana_need(int nu, int n, Win r, bool vmp) {
    const int half = n >> 1;
    Win w{2 * r.lo - nu + 1, 2 * r.hi + nu - 1};
    if (!vmp) return w;
    const int EL = 3 * nu - 1;
    if (w.lo < 0) w.lo = 0;
    if (w.hi > n) w.hi = n;
    if (r.lo < nu) {
        w.lo = 0;
        if (w.hi < EL) w.hi = EL;
    }
    if (r.hi > half - nu) {
        w.hi = n;
        if (w.lo > n - EL) w.lo = n - EL;
    }
    return w;
}

// gray^-1(bitrev_5(nl) << a): gray^-1 is linear over XOR and
// gray^-1(x << a) = (gray^-1(x) << a) | (parity(x) ? 2^a - 1 : 0).
// compile-time friendly (constexpr) bit reversal and inverse Gray code
__host__ __device__ constexpr unsigned brev_c(int v, int bits) {
    unsigned r = 0;
    for (int b = 0; b < bits; ++b) r |= (unsigned)((v >> b) & 1) << (bits - 1 - b);
    return r;
}
__host__ __device__ constexpr unsigned brev_c5(int v) { return brev_c(v, 5); }
__host__ __device__ constexpr unsigned gray_inv_c(unsigned g) {
    return g ^ (g >> 1) ^ (g >> 2) ^ (g >> 3) ^ (g >> 4) ^ (g >> 5) ^ (g >> 6) ^ (g >> 7);
}

__device__ __forceinline__ unsigned gray_inv_hi(int nl, int logb, int a) {
    const unsigned x = brev_bits((unsigned)nl, logb);
    const unsigned gx = gray_inv(x);
    return (gx << a) | ((__popc(x) & 1) ? ((1u << a) - 1u) : 0u);
}

// Sequency-ordered row access (row_store / row_load / the large adjoint):
// element nl of a row sits at gray_inv_hi(nl) ^ rw, rw = gray_inv(w) ^ (odd
// block ? M - 1 : 0) with gray_inv(w) < A.  Since gray_inv_hi(nl) = gx * A |
// (parity(bitrev(nl)) ? A - 1 : 0), the address is pe/po + gx * step: two
// base pointers by parity and a compile-time multiple of one stride, valid
// whenever the layout is affine over multiples of A (plain strides, or a
// tiled layout whose tile width divides A).
__device__ __forceinline__ bool seq_linear(const Layout& L, int a) { return L.esh >= 62 || a >= L.esh; }

template <int LOGB, class P>
__device__ __forceinline__ void seq_ptrs(P* ob, const Layout& L, int a, unsigned rw, P*& pe, P*& po,
                                         long long& step) {
    const long long A = 1ll << a;
    const bool odd = (rw >> a) != 0u;
    const unsigned rl = rw & (unsigned)(A - 1);
    const long long ea = L.eoff(A);
    const long long base = odd ? (long long)((1 << LOGB) - 1) * ea : 0ll;
    pe = ob + L.eoff(rl) + base;
    po = ob + L.eoff(rl ^ (unsigned)(A - 1)) + base;
    step = odd ? -ea : ea;
}

// One warp copies w contiguous doubles global -> shared asynchronously; when
// source and destination share their 16-byte phase the body moves in 16-byte
// pieces (half the copy instructions), an unaligned head / odd tail singly.
__device__ __forceinline__ void warp_copy_span(double* dst, const double* src, int w, int lane) {
    if (((reinterpret_cast<uintptr_t>(dst) ^ reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
        const int head = (reinterpret_cast<uintptr_t>(src) & 15) ? 1 : 0;
        if (lane == 0 && head && w > 0) cp_async8(dst, src);
        const int body = (w - head) >> 1;
        for (int t = lane; t < body; t += 32) cp_async16(dst + head + 2 * t, src + head + 2 * t);
        if (lane == 0 && w > head && ((w - head) & 1)) cp_async8(dst + w - 1, src + w - 1);
    } else {
        for (int t = lane; t < w; t += 32) cp_async8(dst + t, src + t);
    }
}

}  // namespace cww
