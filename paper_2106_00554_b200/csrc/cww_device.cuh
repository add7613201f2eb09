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
    static constexpr int RS = ((CW + 15) / 16) * 16;  // smem row stride (doubles)
    static constexpr int NP = 2 * NU - 1;            // edge positions per side
};

// Bank-conflict-free addressing of tile element (row, e): the column index is
// XOR-swizzled within its 16-double group by the low 4 bits of the lane-varying
// index (bitrev_a(row) for rows visited in bit-reversed order by the row stage).
__device__ __forceinline__ int tile_idx(int row, int e, int RS, int sw) {
    return row * RS + (e ^ (sw & 15));
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

// One radix-2^R pass of H_A along the row index of V tiles held in smem
// (rows 0..A-1 of each tile, columns 0..CW-1), over row bits [lo, lo+R).
template <int R>
__device__ void tile_hadamard_pass(double* T, int V, int a, int lo, int CW, int RS,
                                   long long tstride, int tid, int nt) {
    const int A = 1 << a;
    const int groups = A >> R;
    const long long items = (long long)V * CW * groups;
    for (long long it = tid; it < items; it += nt) {
        int e = (int)(it % CW);
        long long rest = it / CW;
        int fb = (int)(rest % groups);
        int v = (int)(rest / groups);
        int low = fb & ((1 << lo) - 1);
        int row0 = ((fb >> lo) << (lo + R)) | low;
        double* t = T + v * tstride;
        double x[1 << R];
#pragma unroll
        for (int k = 0; k < (1 << R); ++k) {
            int row = row0 + (k << lo);
            x[k] = t[tile_idx(row, e, RS, brev_bits(row, a))];
        }
        hadamard_reg<R>(x);
#pragma unroll
        for (int k = 0; k < (1 << R); ++k) {
            int row = row0 + (k << lo);
            t[tile_idx(row, e, RS, brev_bits(row, a))] = x[k];
        }
    }
}

// Full H_A (a row bits) in passes of <= 5 bits, restricted to bits [lo, hi).
static __device__ __noinline__ void tile_hadamard(double* T, int V, int a, int lo, int hi, int CW, int RS,
                              long long tstride, int tid, int nt) {
    while (lo < hi) {
        int r = hi - lo < 5 ? hi - lo : 5;
        switch (r) {
            case 1: tile_hadamard_pass<1>(T, V, a, lo, CW, RS, tstride, tid, nt); break;
            case 2: tile_hadamard_pass<2>(T, V, a, lo, CW, RS, tstride, tid, nt); break;
            case 3: tile_hadamard_pass<3>(T, V, a, lo, CW, RS, tstride, tid, nt); break;
            case 4: tile_hadamard_pass<4>(T, V, a, lo, CW, RS, tstride, tid, nt); break;
            default: tile_hadamard_pass<5>(T, V, a, lo, CW, RS, tstride, tid, nt); break;
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
    static constexpr int SIZE = 4 * NU + 2 * SIDE;
    const double* f;
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
__device__ __noinline__ double idwt_sample_full(const FiltSmem<NU> F, const double* x, int n, int i,
                                                bool vmp) {
    const int half = n >> 1;
    const double* c = x;
    const double* d = x + half;
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

// Fast paths: away from both ends (3nu-1 <= i <= n-3nu) every synthesis term
// is an interior column and no index wraps, for both boundary modes; the
// rest goes through the out-of-line full sample.
template <int NU>
__device__ __forceinline__ double idwt_sample(const FiltSmem<NU>& F, const double* x, int n, int i,
                                              bool vmp) {
    if (i >= 3 * NU - 1 && i <= n - 3 * NU) {
        const int half = n >> 1;
        const int par = (i + NU + 1) & 1;
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < NU; ++k) {
            int u = -NU + 1 + 2 * k + par;
            int mm = (i - u) >> 1;
            acc += F.h(u) * x[mm] + F.g(u) * x[half + mm];
        }
        return acc;
    }
    return idwt_sample_full<NU>(F, x, n, i, vmp);
}

// analysis: coarse/detail rows NU <= mm < half-NU use the plain 2nu taps
template <int NU>
__device__ __forceinline__ double dwt_sample(const FiltSmem<NU>& F, const double* x, int n, int o,
                                             bool vmp) {
    const int half = n >> 1;
    const bool det = o >= half;
    const int mm = det ? o - half : o;
    if (mm >= NU && mm < half - NU) {
        const double* f = det ? F.f + 2 * NU : F.f;
        double acc = 0.0;
#pragma unroll
        for (int u = -NU + 1; u <= NU; ++u) acc += f[u + NU - 1] * x[2 * mm + u];
        return acc;
    }
    return dwt_sample_full<NU>(F, x, n, o, vmp);
}

}  // namespace cww
