#pragma once
// sm_100a kernel templates of the Walsh->wavelet change-of-basis operator.
//
//   small path  (M <= 2^kSmallMaxLog): one CTA per group of V vectors (V*M <= 4096)
//               runs the whole composed map in shared memory:
//                 k_small_fwd : IDWT levels (ping-pong) -> extended tile -> H_A
//                               -> stencil + edges -> H_B -> sequency-ordered store
//                 k_small_adj : sequency-ordered load -> H_B -> correlation stencil
//                               (+ edge sums) -> H_A -> overlap-add -> DWT levels
//                               (details stored as produced)
//   large path  (M > 2^kSmallMaxLog): wavelet levels as separate passes, then a
//               two-pass Hadamard with an L2-resident intermediate G[A][B+2h]:
//                 k_large_fwd1 (contiguous chunks: halo/mask + H over the low K
//                 bits) -> k_large_fwd2 (strided: H over the high K bits + row stage)
//                 k_large_adj2 (strided: row stage + H over the high N bits)
//                 -> k_large_adj1 (contiguous: H over the low bits + overlap-add + edges)
//
// Tiles and G store logical row K at physical row bitrev(K) (see tile_idx).
//
// Reference correspondence: fastop.cpp:100-175 (forward_1d / adjoint_1d),
// fastop.cpp:196-227 (2D driver), wavelet.cpp:367-514 (dwt_apply levels),
// walsh.cpp:41-98 (FWHT), fastop.cpp:54-98 (edge terms).
#include <cuda_runtime.h>

#include <cstdint>

#include "cww_device.cuh"
#include "cww_launch.h"

namespace cww {

constexpr int kSmallNT = 256;  // threads per small-path CTA (2 CTAs per SM)
constexpr int kWarpLev = 8;  // wavelet levels of <= 256 samples run warp-private
#ifndef CWW_CONTIG_MAXR
#define CWW_CONTIG_MAXR 4  // large contiguous passes: widest in-register Hadamard pass (bits)
#endif
#ifndef CWW_CONTIG_MINB
#define CWW_CONTIG_MINB 3  // large contiguous passes: CTAs per SM (the 76 KB tile allows 3;
                           // 4 forced 64 registers with spills; 2: cfg3 adj1 0.335 vs 0.354 ms
                           // but fwd1 and every config-2 launch slower)
#endif

// Optional per-phase cycle stamps (build with -DCWW_PHASE_TIMING): thread 0 of
// each CTA records clock64() at phase boundaries into cww_phase_buf.
#ifdef CWW_PHASE_TIMING
__device__ long long cww_phase_buf[1 << 20];
#define PHASE(k)                                                                         \
    do {                                                                                 \
        if (threadIdx.x == 0 && blockIdx.x < (1 << 20) / 16)                             \
            cww_phase_buf[blockIdx.x * 16 + (k)] = clock64();                            \
    } while (0)
#else
#define PHASE(k) \
    do {         \
    } while (0)
#endif

// ---------------------------------------------------------------------------
// row stages (shared by the small and large paths)
// ---------------------------------------------------------------------------

// Forward row: z = H_B( stencil_s(row) + edges ).  trow: physical tile row
// (sw unused: odd row stride), kp: &kap[0][s] (stride S), es: edge contributions [2NP] or null.
// VEC2: trow is 16-byte aligned and read as double2 pairs (the large strided
// passes: row stride = 2 (mod 4) doubles makes 16-byte row-per-lane reads
// bank-conflict free, where 8-byte ones would be 2-way conflicted)
template <int NU, int LOGB, bool VEC2 = false>
__device__ __forceinline__ void row_fwd(const double* trow, int sw, const double* kp, int S,
                                        const double* es, double sgR, double* z) {
    using G = Geo<NU, LOGB>;
    constexpr int B = G::B, H = G::H, CW = G::CW, NP = G::NP;
    double kap[2 * H + 1];
#pragma unroll
    for (int l = 0; l <= 2 * H; ++l) kap[l] = kp[l * S];
#pragma unroll
    for (int k = 0; k < B; ++k) z[k] = 0.0;
    double2 pr = make_double2(0.0, 0.0);
#pragma unroll
    for (int e = 0; e < CW; ++e) {  // z[k] = sum_l kap[l] row[k - l + h], streamed over e
        double r;
        if constexpr (VEC2) {
            if ((e & 1) == 0) pr = reinterpret_cast<const double2*>(trow)[e >> 1];
            r = (e & 1) ? pr.y : pr.x;
        } else {
            r = trow[e];
        }
#pragma unroll
        for (int l = -H; l <= H; ++l) {
            const int k = e + l - H;
            if (k >= 0 && k < B) z[k] += kap[l + H] * r;
        }
    }
    if (NU > 1 && es) {
#pragma unroll
        for (int i = 0; i < NP; ++i) z[i] += es[i];
#pragma unroll
        for (int i = 0; i < NP; ++i) z[B - NP + i] += sgR * es[NP + i];
    }
    hadamard_reg<LOGB>(z);
}

// Adjoint row: tile row (+)= correlation_s(y), y already H_B-transformed.
template <int NU, int LOGB>
__device__ __forceinline__ void row_adj_accum(double* trow, int sw, const double* kp, int S,
                                              const double* y, bool first) {
    using G = Geo<NU, LOGB>;
    constexpr int B = G::B, H = G::H, CW = G::CW;
    double kap[2 * H + 1];
#pragma unroll
    for (int l = 0; l <= 2 * H; ++l) kap[l] = kp[l * S];
#pragma unroll
    for (int e = 0; e < CW; ++e) {
        double acc = 0.0;
#pragma unroll
        for (int l = -H; l <= H; ++l) {
            const int k = e - H + l;
            if (k >= 0 && k < B) acc += kap[l + H] * y[k];
        }
        trow[e] = first ? acc : trow[e] + acc;
    }
}

// Adjoint row with software pipelining: as the correlation stream passes
// column e, y[e - 2H] is dead and its register receives the next block's
// element (nxt: that block's base pointer, or null on the last block), so the
// next block's 32 loads are in flight while this block is consumed.
template <int NU, int LOGB>
__device__ __forceinline__ void row_adj_accum_pf(double* trow, const double* kp, int S, double* y, bool first,
                                                 const double* pe, const double* po, long long step) {
    using G = Geo<NU, LOGB>;
    constexpr int B = G::B, H = G::H, CW = G::CW;
    static_assert(CW % 2 == 0, "double2 row pairs");
    double kap[2 * H + 1];
#pragma unroll
    for (int l = 0; l <= 2 * H; ++l) kap[l] = kp[l * S];
    double2* trow2 = reinterpret_cast<double2*>(trow);  // 16-byte aligned rows (row stride = 2 mod 4)
    double accp = 0.0;
#pragma unroll
    for (int e = 0; e < CW; ++e) {
        double acc = 0.0;
#pragma unroll
        for (int l = -H; l <= H; ++l) {
            const int k = e - H + l;
            if (k >= 0 && k < B) acc += kap[l + H] * y[k];
        }
        if (e & 1) {  // the pair (e - 1, e) as one 16-byte read-modify-write
            double2 t = first ? make_double2(0.0, 0.0) : trow2[e >> 1];
            t.x += accp;
            t.y += acc;
            trow2[e >> 1] = t;
        } else {
            accp = acc;
        }
        const int kd = e - 2 * H;  // last use of y[kd] was this column
        if (kd >= 0 && kd < B && pe) {
            const unsigned xb = brev_c(kd, LOGB);
            y[kd] = __ldcs(((__popc(xb) & 1) ? po : pe) + (long long)gray_inv_c(xb) * step);  // streamed once
        }
    }
}

// Store / load one row's B sequency-ordered values: element index
// s*M + (gray^-1(bitrev_b(nl) << a) ^ rw), specialised by layout kind.
template <int LOGB>
__device__ __forceinline__ void row_store(double* ob, const Layout& L, int a, unsigned rw, const double* z) {
    if (seq_linear(L, a)) {
        double *pe, *po;
        long long step;
        seq_ptrs<LOGB>(ob, L, a, rw, pe, po, step);
#pragma unroll
        for (int nl = 0; nl < (1 << LOGB); ++nl) {
            const unsigned x = brev_c(nl, LOGB);
            ((__popc(x) & 1) ? po : pe)[(long long)gray_inv_c(x) * step] = z[nl];
        }
    } else {
#pragma unroll
        for (int nl = 0; nl < (1 << LOGB); ++nl) ob[L.eoff(gray_inv_hi(nl, LOGB, a) ^ rw)] = z[nl];
    }
}

template <int LOGB>
__device__ __forceinline__ void row_load(const double* ib, const Layout& L, int a, unsigned rw, bool act,
                                         double* y) {
    if (!act) {
#pragma unroll
        for (int nl = 0; nl < (1 << LOGB); ++nl) y[nl] = 0.0;
    } else if (seq_linear(L, a)) {
        const double *pe, *po;
        long long step;
        seq_ptrs<LOGB>(ib, L, a, rw, pe, po, step);
#pragma unroll
        for (int nl = 0; nl < (1 << LOGB); ++nl) {
            const unsigned x = brev_c(nl, LOGB);
            y[nl] = __ldg(((__popc(x) & 1) ? po : pe) + (long long)gray_inv_c(x) * step);
        }
    } else {
#pragma unroll
        for (int nl = 0; nl < (1 << LOGB); ++nl) y[nl] = __ldg(ib + L.eoff(gray_inv_hi(nl, LOGB, a) ^ rw));
    }
}

// Deterministic segmented transpose-reduce.  The lanes that differ only in
// the bits `segbits` form one segment (e.g. the lanes sharing a vector).  Each
// lane holds R values; afterwards the segment's sums are spread over its lanes:
// v[0..cnt) of a lane with leader == true hold the sums of the original values
// base*cnt .. base*cnt+cnt-1.  Each step over one segment bit halves the values
// a lane keeps (R/2 + R/4 + ... shuffles instead of R per bit).
template <int R, unsigned SEG>
__device__ __forceinline__ int seg_transpose_reduce(double* v, int lane, int& cnt, bool& leader) {
    int n = R, base = 0;
    unsigned rem = 0;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        if (!(SEG & (unsigned)off)) continue;
        if (n > 1) {
            const bool upper = (lane & off) != 0;
            n >>= 1;
#pragma unroll
            for (int i = 0; i < R / 2; ++i) {
                if (i < n) {
                    const double send = upper ? v[i] : v[i + n];
                    const double keep = upper ? v[i + n] : v[i];
                    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
                }
            }
            base = (base << 1) | (upper ? 1 : 0);
        } else {
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
            rem |= (unsigned)off;
        }
    }
    cnt = n;
    leader = (lane & rem) == 0;
    return base;
}

// Reduce the edge values ev[R] over a lane segment and store the sums
// dst[idx] (idx < nval) from the leader lanes; SEG must be compile-time so
// every register index is static.
template <int R, unsigned SEG, bool ACC = false>
__device__ __forceinline__ void seg_reduce_store(double* ev, int lane, int nval, bool live, double* dst,
                                                 bool acc = false) {
    int cnt;
    bool leader;
    const int base = seg_transpose_reduce<R, SEG>(ev, lane, cnt, leader);
    if (leader && live) {
#pragma unroll
        for (int k2 = 0; k2 < R; ++k2) {
            const int idx = base * cnt + k2;
            if (k2 < cnt && idx < nval) {
                if (ACC && acc) dst[idx] += ev[k2];
                else dst[idx] = ev[k2];
            }
        }
    }
}

template <int R>
__device__ __forceinline__ void seg_reduce_store_rt(double* ev, int lane, unsigned seg, int nval, bool live,
                                                    double* dst) {
    switch (seg) {
        case 31u: seg_reduce_store<R, 31u>(ev, lane, nval, live, dst); break;
        case 30u: seg_reduce_store<R, 30u>(ev, lane, nval, live, dst); break;
        case 28u: seg_reduce_store<R, 28u>(ev, lane, nval, live, dst); break;
        case 24u: seg_reduce_store<R, 24u>(ev, lane, nval, live, dst); break;
        case 16u: seg_reduce_store<R, 16u>(ev, lane, nval, live, dst); break;
        case 15u: seg_reduce_store<R, 15u>(ev, lane, nval, live, dst); break;
        case 7u: seg_reduce_store<R, 7u>(ev, lane, nval, live, dst); break;
        case 3u: seg_reduce_store<R, 3u>(ev, lane, nval, live, dst); break;
        case 1u: seg_reduce_store<R, 1u>(ev, lane, nval, live, dst); break;
        default: seg_reduce_store<R, 0u>(ev, lane, nval, live, dst); break;
    }
}

// Warp all-reduce over the lanes that share a vector (deterministic butterfly).
__device__ __forceinline__ double seg_allreduce(double x, int lo_off, int hi_off) {
    for (int off = lo_off; off < hi_off; off <<= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
    return x;
}

// ---------------------------------------------------------------------------
// wavelet level bodies (cooperative over `nthr` threads starting at `t0`)
// ---------------------------------------------------------------------------

// Synthesis of level n for one vector: fine[0:n] from cs[0:n/2], ds[0:n/2].
// Interior pairs share a window; the 2(3nu-1) edge samples are separate
// (dense edge blocks), so the interior loop is branch-free.
template <int NU>
__device__ __forceinline__ void idwt_level_vec(const FiltSmem<NU>& F, const double* cs, const double* ds,
                                               double* dst, int n, bool vmp, int t0, int nthr) {
    const int half = n >> 1;
    if (vmp && n < 8 * NU) {  // coarsest levels: generic edge code
        for (int i = t0; i < n; i += nthr) dst[i] = idwt_sample_full2<NU>(F, cs, ds, n, i, true);
        return;
    }
    constexpr int EL = FiltSmem<NU>::EL;
    const int mlo = vmp ? (EL + 1) >> 1 : 0;
    const int mhi = vmp ? (n - EL) >> 1 : half;
    const Taps<NU> tp(F);
    // two adjacent pairs (four samples) per thread share one window of nu+2
    const int nq = (mhi - mlo) >> 1;
    for (int qi = t0; qi < nq; qi += nthr) {
        const int m = mlo + 2 * qi;
        double o[4];
        idwt_quad_inner<NU>(tp, cs, ds, n, m, vmp, o);
        dst[2 * m] = o[0];
        dst[2 * m + 1] = o[1];
        dst[2 * m + 2] = o[2];
        dst[2 * m + 3] = o[3];
    }
    if (((mhi - mlo) & 1) && t0 == 0) {
        const int m = mhi - 1;
        double o0, o1;
        idwt_pair_inner<NU>(tp, cs, ds, n, m, vmp, o0, o1);
        dst[2 * m] = o0;
        dst[2 * m + 1] = o1;
    }
    if (vmp) {
        const int nl = 2 * mlo, nr = n - 2 * mhi;  // edge samples [0, nl) and [2 mhi, n)
        for (int k = nthr - 1 - t0; k < nl + nr; k += nthr) {  // last threads: fewest pairs
            const int i = k < nl ? k : 2 * mhi + (k - nl);
            dst[i] = idwt_one<NU>(F, cs, ds, n, i, true);
        }
    }
}

// Barrier over the G threads of group gid (NT threads per CTA): the whole
// CTA, one warp (or less: __syncwarp is a superset), or a named barrier.
template <int NT>
__device__ __forceinline__ void group_sync(int gid, int G, int ngroups) {
    if (G >= NT) {
        __syncthreads();
    } else if (G <= 32) {  // the warp's active groups (a group never spans warps)
        const int g0 = (int)(threadIdx.x & ~31u) / G;
        const int nact = min(32 / G, ngroups - g0);
        const unsigned mask = nact >= 32 / G ? 0xffffffffu : ((1u << (nact * G)) - 1u);
        __syncwarp(mask);
    } else {  // G > 32 implies at most 4 groups; immediate ids keep the barrier count low
        switch (gid) {
            case 0: asm volatile("bar.sync 1, %0;" ::"r"(G) : "memory"); break;
            case 1: asm volatile("bar.sync 2, %0;" ::"r"(G) : "memory"); break;
            case 2: asm volatile("bar.sync 3, %0;" ::"r"(G) : "memory"); break;
            default: asm volatile("bar.sync 4, %0;" ::"r"(G) : "memory"); break;
        }
    }
}

// Synthesis levels r0+1 .. j-1 of one vector by a thread group; returns the
// coarse input of the final level j (cbuf, or xv when there is no earlier
// level).  Level t (lev = r0+1+t) reads c from xv (t = 0) or the previous
// buffer and d = xv[2^(lev-1) : 2^lev]; it writes p0/p1 alternately, and the
// last one (level j-1) writes cbuf.
template <int NU, int NT>
__device__ __forceinline__ const double* idwt_group(const FiltSmem<NU>& F, const double* xv, double* p0,
                                                    double* p1, double* cbuf, int j, int r0, bool vmp,
                                                    int gt, int G, int gid, int ngroups) {
    const double* src = xv;
    int lev = r0 + 1;
    for (; lev < j; ++lev) {
        const int n = 1 << lev;
        double* dst = (lev == j - 1) ? cbuf : (src == p0 ? p1 : p0);
        idwt_level_vec<NU>(F, src, xv + (n >> 1), dst, n, vmp, gt, G);
        group_sync<NT>(gid, G, ngroups);
        src = dst;
    }
    return src;
}

// ---------------------------------------------------------------------------
// small path
// ---------------------------------------------------------------------------

// edge partial-sum slots of k_small_adj (lanes sharing a vector per warp)
__host__ __device__ inline int small_adj_lanes(int A, int V, bool vf) {
    return vf ? ((32 / V) < A ? (32 / V) : A) : (A < 32 ? A : 32);
}

// per-vector tile stride: >= A*RS and == 16/V (mod 16), so lanes that walk
// (vector, row) pairs hit distinct banks
__host__ __device__ inline int small_tile_stride(int ars, int V) {
    const int t = V >= 16 ? 1 : 16 / V;
    return ((ars + 15) / 16) * 16 + (t & 15);
}

// shared copy of kap[2h+1][S] and the edge matrix em[S][2NP][2nu]
__host__ __device__ inline int small_ke_size(int nu, int S) {
    return (2 * nu - 1) * S + S * 2 * (2 * nu - 1) * 2 * nu;
}

template <int NU>
__device__ __forceinline__ void stage_ke(double* ke, const double* tab, const Tables& t, int S, int tid,
                                         int nt) {
    const int nk = (2 * NU - 1) * S, ne = S * 2 * (2 * NU - 1) * 2 * NU;
    for (int i = tid; i < nk; i += nt) ke[i] = tab[t.o_kap + i];
    for (int i = tid; i < ne; i += nt) ke[nk + i] = tab[t.o_em + i];
}

template <int NU, int LOGB>
inline long long small_smem_bytes(int V, int j, int q, bool adj, bool vf) {
    using G = Geo<NU, LOGB>;
    const int a = j - LOGB, A = 1 << a, S = 1 << q;
    long long d = FiltSmem<NU>::SIZE + small_ke_size(NU, S) + (long long)V * 2 * NU +
                  (long long)V * S * 2 * G::NP;
    if (adj) {
        const int L = small_adj_lanes(A, V, vf);
        const int nslot = A / L > 0 ? A / L : 1;
        d += (long long)V * nslot * S * 2 * G::NP;
    }
    d += (long long)V << j;          // X
    d += (long long)V << (j > 0 ? j - 1 : 0);  // C (final-level coarse input / DWT ping)
    d += 3;                          // 16-byte phase slack of X, C and the tiles
    d += (long long)V * small_tile_stride(A * G::RS, V);  // tiles (also wavelet ping-pong / output staging)
    return d * 8;
}

template <int NU>
__device__ __forceinline__ void stage_filters(double* filt, const double* tab, const Tables& t,
                                              int tid, int nt) {
    for (int i = tid; i < FiltSmem<NU>::SIZE; i += nt) filt[i] = tab[t.o_h + i];
}

__device__ __forceinline__ int ilog2(int v) { return 31 - __clz(v); }

template <int NU, int LOGB, int NT>
__global__ void __launch_bounds__(NT, 2) k_small_fwd(SmallArgs p) {
    const bool vmp_ = NU > 1 && p.vmp != 0;  // VMP needs nu >= 2: no VMP code in the Haar kernels
    using G = Geo<NU, LOGB>;
    constexpr int B = G::B, H = G::H, CW = G::CW, RS = G::RS, NP = G::NP;
    extern __shared__ double sm[];
    const int tid = threadIdx.x;
    const int j = p.j, M = 1 << j, a = j - LOGB, A = 1 << a, S = 1 << p.q;
    const int V = p.V, lV = ilog2(V);
    const long long v0 = (long long)blockIdx.x * V;
    const int nv = (int)((p.nvec - v0) < V ? (p.nvec - v0) : V);
    double* filt = sm;
    double* KE = filt + FiltSmem<NU>::SIZE;  // kap | em
    double* EV = KE + small_ke_size(NU, S);
    double* ES = EV + V * 2 * NU;
    // 16-byte aligned X, C and tile bases: the synthesis quads then read their
    // windows as double2 pairs (idwt_quad_inner); slack in small_smem_bytes
    auto al2 = [](double* q) { return q + ((reinterpret_cast<uintptr_t>(q) >> 3) & 1); };
    double* X = al2(ES + V * S * 2 * NP);
    double* C = al2(X + V * M);
    double* T = al2(C + (V * M >> 1));
    const int tst = small_tile_stride(A * RS, V);
    const int hM = M >> 1;
    const double* KAP = KE;
    const double* EM = KE + (2 * NU - 1) * S;
    // thread groups: G threads per vector (V divides NT)
    const int Gs = NT / V, gid = tid / Gs, gt = tid % Gs;

    PHASE(0);
    stage_filters<NU>(filt, p.tab, p.t, tid, NT);
    stage_ke<NU>(KE, p.tab, p.t, S, tid, NT);
    constexpr int U = 4;  // 16-byte loads in flight per thread
    if (p.in_block == 1 && M >= 2) {  // V vectors back to back: 16-byte copy
        const double2* blk = reinterpret_cast<const double2*>(p.in + p.lin.vbase(v0));
        const int tot2 = (nv * M) >> 1;
        for (int f0 = tid; f0 < tot2; f0 += U * NT) {
            double2 r[U];
#pragma unroll
            for (int u = 0; u < U; ++u) r[u] = f0 + u * NT < tot2 ? __ldg(blk + f0 + u * NT) : make_double2(0.0, 0.0);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int f = f0 + u * NT;
                if (f < tot2) {
                    X[2 * f] = r[u].x;
                    X[2 * f + 1] = r[u].y;
                }
            }
        }
    } else if (p.in_block == 2 && V >= 2) {  // [M][V] interleaved block (column panel)
        const double2* blk = reinterpret_cast<const double2*>(p.in + p.lin.vbase(v0));
        const int tot2 = (V * M) >> 1;
        for (int f0 = tid; f0 < tot2; f0 += U * NT) {
            double2 r[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int f = f0 + u * NT;
                r[u] = (f < tot2 && ((2 * f) & (V - 1)) < nv) ? __ldg(blk + f) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int f = f0 + u * NT;
                const int v = (2 * f) & (V - 1), i = (2 * f) >> lV;
                if (f < tot2 && v < nv) {
                    X[v * M + i] = r[u].x;
                    X[(v + 1) * M + i] = r[u].y;
                }
            }
        }
    } else {
        const bool vf = p.lin.vfast();
        for (int f = tid; f < V * M; f += NT) {
            const int v = vf ? f & (V - 1) : f >> j;
            const int i = vf ? f >> lV : f & (M - 1);
            if (v < nv) X[v * M + i] = __ldg(p.in + p.lin.vbase(v0 + v) + p.lin.eoff(i));
        }
    }
    __syncthreads();
    PHASE(1);
    const FiltSmem<NU> F{filt};
    const bool idwt = p.use_idwt && p.r0 < j;

    // per-vector group: IDWT levels r0+1 .. j (wavelet.cpp:505-513); the final
    // level writes the extended tile directly (interior mask, edge values -> EV)
    if (gid < nv) {
        const int v = gid;
        const double* xv = X + v * M;
        double* tv = T + v * tst;
        const double* cfin = xv;
        // Haar (nu = 1, periodic, non-overlapping 2-tap filters): every fine sample is
        // its own chain c_r0 -> level j through one coefficient per level, so all the
        // levels run in ONE phase without barriers (wavelet.cpp:387-400 per step)
        constexpr bool haar = NU == 1;
        if (idwt && !haar) cfin = idwt_group<NU, NT>(F, xv, tv, tv + hM, C + v * hM, j, p.r0, vmp_, gt, Gs, gid,
                                                          nv);
        PHASE(2);
        auto put = [&](int i, double val) {
            if (NU > 1 && (i < NU || i >= M - NU)) {
                EV[v * 2 * NU + (i < NU ? i : NU + i - (M - NU))] = val;
                val = 0.0;
            }
            const int ph = (int)brev_bits((unsigned)(i >> LOGB), a);
            tv[ph * RS + (i & (B - 1)) + H] = val;
        };
        if (!idwt) {
            for (int i = gt; i < M; i += Gs) put(i, xv[i]);
        } else if (haar) {
            const double h0 = F.h(0), h1 = F.h(1), g0 = F.g(0), g1 = F.g(1);
            const int r0 = p.r0;
            for (int i = gt; i < M; i += Gs) {
                double val = xv[i >> (j - r0)];  // c_r0
                for (int l = r0; l < j; ++l) {   // level l + 1 from level l: fine[2m + u] = h_u c[m] + g_u d[m]
                    const int idx = i >> (j - l - 1);
                    const double d = xv[(1 << l) + (idx >> 1)];
                    val = (idx & 1) ? h1 * val + g1 * d : h0 * val + g0 * d;
                }
                put(i, val);
            }
        } else if (vmp_ && M < 8 * NU) {
            for (int i = gt; i < M; i += Gs) put(i, idwt_sample_full2<NU>(F, cfin, xv + hM, M, i, true));
        } else {
            constexpr int EL = FiltSmem<NU>::EL;
            const int mlo = vmp_ ? (EL + 1) >> 1 : 0;
            const int mhi = vmp_ ? (M - EL) >> 1 : hM;
            const Taps<NU> tp(F);
            if (NU > 1 && vmp_ && B >= 2) {  // interior pairs hold no edge position: both samples in one tile row
                for (int m = mlo + gt; m < mhi; m += Gs) {
                    double o0, o1;
                    idwt_pair_inner<NU>(tp, cfin, xv + hM, M, m, true, o0, o1);
                    double* d = tv + (int)brev_bits((unsigned)((2 * m) >> LOGB), a) * RS + ((2 * m) & (B - 1)) + H;
                    d[0] = o0;
                    d[1] = o1;
                }
                const int nl = 2 * mlo, nr = M - 2 * mhi;
                for (int k2 = Gs - 1 - gt; k2 < nl + nr; k2 += Gs) {
                    const int i = k2 < nl ? k2 : 2 * mhi + (k2 - nl);
                    put(i, idwt_one<NU>(F, cfin, xv + hM, M, i, true));
                }
            } else {
                for (int m = mlo + gt; m < mhi; m += Gs) {
                    double o0, o1;
                    idwt_pair_inner<NU>(tp, cfin, xv + hM, M, m, vmp_, o0, o1);
                    put(2 * m, o0);
                    put(2 * m + 1, o1);
                }
                if (vmp_) {
                    const int nl = 2 * mlo, nr = M - 2 * mhi;
                    for (int k2 = Gs - 1 - gt; k2 < nl + nr; k2 += Gs) {
                        const int i = k2 < nl ? k2 : 2 * mhi + (k2 - nl);
                        put(i, idwt_one<NU>(F, cfin, xv + hM, M, i, true));
                    }
                }
            }
        }
        group_sync<NT>(gid, Gs, nv);
        PHASE(3);
        // halo columns of this vector's tile: copies of the neighbouring rows
        if (H > 0) {
            for (int f = gt; f < A * 2 * H; f += Gs) {
                const int c = f % (2 * H), K = f / (2 * H);
                const int ph = (int)brev_bits((unsigned)K, a);
                double val = 0.0;
                if (c < H) {  // left halo e = c <- row K-1, column (B - H + c) + H
                    if (K > 0) val = tv[(int)brev_bits((unsigned)(K - 1), a) * RS + B + c];
                    tv[ph * RS + c] = val;
                } else {      // right halo e = B + c <- row K+1, column (c - H) + H
                    if (K < A - 1) val = tv[(int)brev_bits((unsigned)(K + 1), a) * RS + c];
                    tv[ph * RS + B + c] = val;
                }
            }
        }
        if (NU > 1) {  // es[v][s][pos] = sum_c em[s][pos][c] xi_edge[c]
            for (int f = gt; f < S * 2 * NP; f += Gs) {
                const double* em = EM + f * 2 * NU;
                double acc = 0.0;
#pragma unroll
                for (int c = 0; c < 2 * NU; ++c) acc += em[c] * EV[v * 2 * NU + c];
                ES[v * S * 2 * NP + f] = acc;
            }
        }
    }
    __syncthreads();
    PHASE(4);
    PHASE(5);
    tile_hadamard<CW, RS>(T, nv, a, 0, a, tst, tid, NT);
    PHASE(6);

    // row stage: stencil + edges + H_B + sequency-ordered store
    const bool of = p.lout.vfast();
    const int items = V * A * S;
    for (int w = tid; w < items; w += NT) {
        int v, wlo, s;
        if (of) {  // lanes vary the vector first (V is a power of two)
            v = w & (V - 1);
            const int rest = w >> lV;
            wlo = rest & (A - 1);
            s = rest >> a;
        } else {
            wlo = w & (A - 1);
            const int rest = w >> a;
            s = rest & (S - 1);
            v = rest >> p.q;
        }
        if (v >= nv) continue;
        const double sg = (__popc(wlo) & 1) ? -1.0 : 1.0;  // popc(N) = popc(bitrev(N))
        double z[B];
        row_fwd<NU, LOGB>(T + v * tst + wlo * RS, wlo, KAP + s, S,
                          NU > 1 ? ES + (v * S + s) * 2 * NP : nullptr, sg, z);
        const unsigned rw = gray_inv((unsigned)wlo) ^ ((s & 1) ? (unsigned)(M - 1) : 0u);
        row_store<LOGB>(p.out + p.lout.vbase(v0 + v) + p.lout.eoff((long long)s * M), p.lout, a, rw, z);
    }
    PHASE(7);
}

template <int NU, int LOGB, int NT>
__global__ void __launch_bounds__(NT, 2) k_small_adj(SmallArgs p) {
    const bool vmp_ = NU > 1 && p.vmp != 0;  // VMP needs nu >= 2: no VMP code in the Haar kernels
    using G = Geo<NU, LOGB>;
    constexpr int B = G::B, H = G::H, CW = G::CW, RS = G::RS, NP = G::NP;
    extern __shared__ double sm[];
    const int tid = threadIdx.x, lane = tid & 31;
    const int j = p.j, M = 1 << j, a = j - LOGB, A = 1 << a, S = 1 << p.q;
    const int V = p.V, lV = ilog2(V);
    const long long v0 = (long long)blockIdx.x * V;
    const int nv = (int)((p.nvec - v0) < V ? (p.nvec - v0) : V);
    const bool vf = p.lin.vfast();
    const int L = small_adj_lanes(A, V, vf);
    const int nslot = A / L > 0 ? A / L : 1;
    double* filt = sm;
    double* KE = filt + FiltSmem<NU>::SIZE;  // kap | em
    double* EV = KE + small_ke_size(NU, S);  // unused here; keeps the layout of k_small_fwd
    double* W = EV + V * 2 * NU;              // [V][S][2NP]
    const double* KAP = KE;
    const double* EM = KE + (2 * NU - 1) * S;
    double* EPW = W + V * S * 2 * NP;         // [V][nslot][S][2NP]
    // X and C (the analysis ping-pong) start at the 8-byte phase that puts each
    // analysis row's first tap 2mm - nu + 1 on a 16-byte boundary (double2 tap
    // pairs); one slack double each (small_smem_bytes)
    auto pair_al = [](double* q) {
        return q + ((((reinterpret_cast<uintptr_t>(q) >> 3) & 1) + 1 - NU) & 1);
    };
    double* X = pair_al(EPW + V * nslot * S * 2 * NP);
    double* C = pair_al(X + V * M);
    double* T = C + (V * M >> 1) + 1;
    const int tst = small_tile_stride(A * RS, V);
    const int hM = M >> 1;
    const int Gs = NT / V, gid = tid / Gs, gt = tid % Gs;
    PHASE(0);
    stage_filters<NU>(filt, p.tab, p.t, tid, NT);
    stage_ke<NU>(KE, p.tab, p.t, S, tid, NT);
    __syncthreads();

    // row stage: sequency-ordered load + H_B + correlation (+ edge partials)
    const int items = V * A;  // padded to V: the lane -> vector pattern is fixed
    const int iters = (items + NT - 1) / NT;
    for (int it = 0; it < iters; ++it) {
        const int w = tid + it * NT;
        int v, wlo;
        if (vf) {
            v = w & (V - 1);
            wlo = (w >> lV) & (A - 1);
        } else {
            wlo = w & (A - 1);
            v = w >> a;
        }
        const bool act = (w < items) && (v < nv);
        const double sg = (__popc(wlo) & 1) ? -1.0 : 1.0;
        const double* ib0 = p.in + p.lin.vbase(v0 + (act ? v : 0));
        for (int s = 0; s < S; ++s) {
            double y[B];
            const unsigned rw = gray_inv((unsigned)wlo) ^ ((s & 1) ? (unsigned)(M - 1) : 0u);
            row_load<LOGB>(ib0 + p.lin.eoff((long long)s * M), p.lin, a, rw, act, y);
            hadamard_reg<LOGB>(y);
            if (NU > 1) {  // transform-domain values at the 4nu-2 edge positions
                // V, L and nslot are powers of two: ((it*NT + warp base) / (vf ? V : 1) / L) % nslot
                const int slot = ((it * NT + (tid & ~31)) >> ((vf ? lV : 0) + ilog2(L))) & (nslot - 1);
                constexpr int R = 2 * NP <= 16 ? 16 : 32;
                double ev[R];
#pragma unroll
                for (int i = 0; i < R; ++i)
                    ev[i] = (act && i < 2 * NP) ? (i < NP ? y[i] : sg * y[B - NP + (i - NP)]) : 0.0;
                const unsigned segbits = vf ? (31u & ~(unsigned)(V - 1)) : (unsigned)(L - 1);
                // v is uniform over a segment; a segment is live iff its warp starts
                // inside the padded item range and its vector exists
                const bool live = v < nv && (it * NT + (tid & ~31)) < items;
                seg_reduce_store_rt<R>(ev, lane, segbits, 2 * NP, live,
                                       EPW + ((v * nslot + slot) * S + s) * 2 * NP);
            }
            if (act) row_adj_accum<NU, LOGB>(T + v * tst + wlo * RS, wlo, KAP + s, S, y, s == 0);
        }
    }
    __syncthreads();
    PHASE(1);
    tile_hadamard<CW, RS>(T, nv, a, 0, a, tst, tid, NT);
    PHASE(2);
    if (NU > 1) {  // W[v][s][pos] = sum over rows (fixed order)
        for (int f = tid; f < nv * S * 2 * NP; f += NT) {
            const int v = f / (S * 2 * NP), sp = f % (S * 2 * NP);
            double acc = 0.0;
            for (int sl = 0; sl < nslot; ++sl) acc += EPW[(v * nslot + sl) * S * 2 * NP + sp];
            W[f] = acc;
        }
        __syncthreads();
    }
    // overlap-add + interior mask + edge columns -> X
    if constexpr (B == 32) {  // one tile row per warp, lane = column: row indices are warp-uniform
        const int lane = tid & 31;
        const int hside = lane < H ? -1 : (lane >= B - H ? 1 : 0);
        const int hcol = lane < H ? B + H + lane : lane - (B - H);
        for (int r = tid >> 5; r < nv * A; r += NT / 32) {
            const int v = r >> a, K = r & (A - 1);
            const double* t = T + v * tst;
            double val = t[(int)brev_bits((unsigned)K, a) * RS + lane + H];
            if (hside != 0) {
                const int Kn = K + hside;
                if (Kn >= 0 && Kn < A) val += t[(int)brev_bits((unsigned)Kn, a) * RS + hcol];
            }
            const int i = K * B + lane;
            if (NU > 1 && (K == 0 || K == A - 1) && (i < NU || i >= M - NU)) {
                const int c = i < NU ? i : NU + i - (M - NU);
                const double* wv = W + v * S * 2 * NP;
                double e0 = 0.0, e1 = 0.0, e2 = 0.0, e3 = 0.0;
                const int nsp = S * 2 * NP;
                int sp = 0;
                for (; sp + 4 <= nsp; sp += 4) {
                    e0 += EM[sp * 2 * NU + c] * wv[sp];
                    e1 += EM[(sp + 1) * 2 * NU + c] * wv[sp + 1];
                    e2 += EM[(sp + 2) * 2 * NU + c] * wv[sp + 2];
                    e3 += EM[(sp + 3) * 2 * NU + c] * wv[sp + 3];
                }
                for (; sp < nsp; ++sp) e0 += EM[sp * 2 * NU + c] * wv[sp];
                val = (e0 + e1) + (e2 + e3);
            }
            X[v * M + i] = val;
        }
    } else
    for (int o = tid; o < nv * M; o += NT) {
        const int v = o >> j, i = o & (M - 1);
        const double* t = T + v * tst;
        const int K = i >> LOGB, kl = i & (B - 1);
        const int ph = (int)brev_bits((unsigned)K, a);
        double val = t[ph * RS + kl + H];
        if (kl < H && K > 0) val += t[(int)brev_bits((unsigned)(K - 1), a) * RS + B + H + kl];
        if (kl >= B - H && K < A - 1) val += t[(int)brev_bits((unsigned)(K + 1), a) * RS + kl - (B - H)];
        if (NU > 1 && (i < NU || i >= M - NU)) {
            const int c = i < NU ? i : NU + i - (M - NU);
            const double* wv = W + v * S * 2 * NP;
            double e0 = 0.0, e1 = 0.0, e2 = 0.0, e3 = 0.0;
            const int nsp = S * 2 * NP;  // multiple of 2; four independent chains
            int sp = 0;
            for (; sp + 4 <= nsp; sp += 4) {
                e0 += EM[sp * 2 * NU + c] * wv[sp];
                e1 += EM[(sp + 1) * 2 * NU + c] * wv[sp + 1];
                e2 += EM[(sp + 2) * 2 * NU + c] * wv[sp + 2];
                e3 += EM[(sp + 3) * 2 * NU + c] * wv[sp + 3];
            }
            for (; sp < nsp; ++sp) e0 += EM[sp * 2 * NU + c] * wv[sp];
            val = (e0 + e1) + (e2 + e3);
        }
        X[o] = val;
    }
    __syncthreads();
    PHASE(3);
    // DWT levels j .. r0+1 (wavelet.cpp:497-504) per vector group; the output
    // vector is staged in the (now free) tile area and stored block-wide.
    const FiltSmem<NU> F{filt};
    const bool of = p.lout.vfast();
    const bool dwt = p.use_idwt && p.r0 < j;
    if (dwt && gid < nv) {
        const int v = gid;
        double* ov = T + v * tst;  // staged output [c_r0 | d_r0 | ... | d_(j-1)]
        double* xv = X + v * M;
        double* cv = C + v * hM;
        const double* src = xv;
        for (int lev = j; lev > p.r0; --lev) {
            const int t = j - lev, n = 1 << lev, half = n >> 1;
            const bool last = lev == p.r0 + 1;
            double* dst = last ? ov : ((t & 1) ? xv : cv);  // coarse rows ping-pong C <-> X
            const double* s2 = src;
            if (NU > 1 && vmp_ && half >= 2 * NU + 2 && (s2 == xv || s2 == cv)) {  // (no code for Haar)
                // interior rows [NU, half - NU): nu aligned double2 tap pairs per row
                // (s2 + 2mm - nu + 1 is 16-byte aligned: pair_al above); then the
                // 2 NU edge rows on the last threads
                const Taps<NU> tp(F);
                for (int mm = NU + gt; mm < half - NU; mm += Gs) {
                    const double2* xp = reinterpret_cast<const double2*>(s2 + 2 * mm - NU + 1);
                    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
                    for (int k = 0; k < NU; ++k) {
                        const double2 pr = xp[k];
                        a0 = fma(tp.h[2 * k], pr.x, a0);
                        b0 = fma(tp.g[2 * k], pr.x, b0);
                        a1 = fma(tp.h[2 * k + 1], pr.y, a1);
                        b1 = fma(tp.g[2 * k + 1], pr.y, b1);
                    }
                    ov[half + mm] = b0 + b1;
                    dst[mm] = a0 + a1;
                }
                for (int k2 = Gs - 1 - gt; k2 < 2 * NU; k2 += Gs) {
                    const int mm = k2 < NU ? k2 : half - 2 * NU + k2;
                    double c, d;
                    dwt_pair<NU>(F, s2, n, mm, true, c, d);
                    ov[half + mm] = d;
                    dst[mm] = c;
                }
            } else {
                for (int mm = gt; mm < half; mm += Gs) {
                    double c, d;
                    dwt_pair<NU>(F, s2, n, mm, vmp_, c, d);
                    ov[half + mm] = d;
                    dst[mm] = c;
                }
            }
            group_sync<NT>(gid, Gs, nv);
            src = dst;
        }
    }
    __syncthreads();
    PHASE(4);
    const double* res = dwt ? T : X;
    const int rst = dwt ? tst : M;
    if (p.lout.esh >= 62 && (p.lout.vsh >= 62 || (p.lout.vsh >= lV && nv == V))) {
        // plain strides within the CTA's V vectors: no tiling arithmetic per element
        const long long vs = p.lout.vs, es = p.lout.es;
        double* o0 = p.out + p.lout.vbase(v0);
        for (int f = tid; f < V * M; f += NT) {
            const int v = of ? f & (V - 1) : f >> j;
            const int i = of ? f >> lV : f & (M - 1);
            if (v < nv) o0[v * vs + i * es] = res[v * rst + i];
        }
    } else {
        for (int f = tid; f < V * M; f += NT) {
            const int v = of ? f & (V - 1) : f >> j;
            const int i = of ? f >> lV : f & (M - 1);
            if (v < nv) p.out[p.lout.at(v0 + v, i)] = res[v * rst + i];
        }
    }
    __syncthreads();
    PHASE(5);
}

// ---------------------------------------------------------------------------
// wavelet levels in global memory (large path)
// ---------------------------------------------------------------------------

// Coarse levels in one CTA per vector (shared memory ping-pong).
//   inverse: levels r0+1..Lc of x (layout) -> dst[0:2^Lc] (workspace, dst_vs)
//   forward: levels Lc..r0+1 of src[0:2^Lc] (workspace) -> y layout [0:2^Lc)
template <int NU>
__global__ void __launch_bounds__(256) k_wav_coarse(const double* tab, Tables t, const double* src,
                                                    Layout ls, long long sv0, long long src_vs,
                                                    double* dst, Layout ld, long long dv0,
                                                    long long dst_vs, int r0, int Lc, int inverse,
                                                    int vmp) {
    extern __shared__ double sm[];
    double* filt = sm;
    const int n = 1 << Lc;
    double* X = sm + FiltSmem<NU>::SIZE;  // [n] input
    double* P0 = X + n;                   // [n] ping
    double* P1 = P0 + n;                  // [n] pong
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int i = tid; i < FiltSmem<NU>::SIZE; i += nt) filt[i] = tab[t.o_h + i];
    const int v = blockIdx.x;
    for (int i = tid; i < n; i += nt) X[i] = inverse ? src[ls.at(sv0 + v, i)] : src[v * src_vs + i];
    __syncthreads();
    const FiltSmem<NU> F{filt};
    const double* cur = X;
    double* nxt = P0;
    if (inverse) {
        for (int lev = r0 + 1; lev <= Lc; ++lev) {
            const int m = 1 << lev, half = m >> 1;
            idwt_level_vec<NU>(F, cur, X + half, nxt, m, vmp, tid, nt);
            __syncthreads();
            cur = nxt;
            nxt = (nxt == P0) ? P1 : P0;
        }
        for (int i = tid; i < n; i += nt) dst[v * dst_vs + i] = cur[i];
    } else {
        for (int lev = Lc; lev > r0; --lev) {
            const int m = 1 << lev, half = m >> 1;
            for (int k = tid; k < half; k += nt) {
                double c, d;
                dwt_pair<NU>(F, cur, m, k, vmp, c, d);
                dst[ld.at(dv0 + v, half + k)] = d;
                nxt[k] = c;
            }
            __syncthreads();
            cur = nxt;
            nxt = (nxt == P0) ? P1 : P0;
        }
        for (int i = tid; i < (1 << r0); i += nt) dst[ld.at(dv0 + v, i)] = cur[i];
    }
}

// ---------------------------------------------------------------------------
// windowed multilevel synthesis (large path forward: every chunk builds its
// own pyramid of level windows straight from x, coarse to fine)
// ---------------------------------------------------------------------------

// Fine samples [lo, hi) of level n from windows cw = c[clo .. chi), dw =
// d[clo .. chi) (same range; periodic: entries taken modulo n/2), written to
// out[i - lo] (or, when put != nullptr, handed to put(i, value)).
// put2(i, a, b), i even, stores the sample pair (i, i + 1) (one 16-byte store
// where the destination keeps sample i at i's 16-byte phase).
template <int NU, class Put, class Put2>
__device__ __forceinline__ void idwt_window(const FiltSmem<NU>& F, const Taps<NU>& tp, const double* cw,
                                            const double* dw, int clo, int n, int lo, int hi, bool vmp,
                                            int t0, int nthr, Put&& put, Put2&& put2) {
    const double* cv = cw - clo;  // absolute (logical) coarse index
    const double* dv = dw - clo;
    if (vmp && n < 8 * NU) {
        for (int i = lo + t0; i < hi; i += nthr) put(i, idwt_sample_full2<NU>(F, cv, dv, n, i, true));
        return;
    }
    constexpr int EL = FiltSmem<NU>::EL;
    int mlo = (lo + 1) >> 1, mhi = hi >> 1;  // pairs (2m, 2m+1) fully inside [lo, hi)
    if (vmp) {
        mlo = max(mlo, (EL + 1) >> 1);
        mhi = min(mhi, (n - EL) >> 1);
    }
    auto pair = [&](int m, double& o0, double& o1) {
        constexpr int OFF = (NU + 1) / 2;
        double c[NU + 1], d[NU + 1];
#pragma unroll
        for (int k = 0; k <= NU; ++k) {
            c[k] = cv[m - OFF + k];
            d[k] = dv[m - OFF + k];
        }
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
        for (int u = -NU + 1; u <= NU; ++u) {
            if ((u & 1) == 0) {
                a0 += tp.h[u + NU - 1] * c[OFF - u / 2];
                b0 += tp.g[u + NU - 1] * d[OFF - u / 2];
            } else {
                a1 += tp.h[u + NU - 1] * c[OFF - (u - 1) / 2];
                b1 += tp.g[u + NU - 1] * d[OFF - (u - 1) / 2];
            }
        }
        o0 = a0 + b0;
        o1 = a1 + b1;
    };
    for (int m = mlo + t0; m < mhi; m += nthr) {
        double o0, o1;
        pair(m, o0, o1);
        put2(2 * m, o0, o1);
    }
    // the rest of [lo, hi): partial pairs at the window ends and VMP edge samples
    const int nl = 2 * mlo - lo, nr = hi - 2 * mhi;
    for (int k = nthr - 1 - t0; k < nl + nr; k += nthr) {
        const int i = k < nl ? lo + k : 2 * mhi + (k - nl);
        if (!vmp) {
            const int par = (i + NU + 1) & 1;
            double acc = 0.0;
#pragma unroll
            for (int q = 0; q < NU; ++q) {
                const int u = -NU + 1 + 2 * q + par;
                const int mm = (i - u) >> 1;  // logical index, inside the window
                acc += F.h(u) * cv[mm] + F.g(u) * dv[mm];  // runtime tap index: smem, not registers
            }
            put(i, acc);
        } else {
            put(i, idwt_one<NU>(F, cv, dv, n, i, true));
        }
    }
}

// Analysis rows mm of a length-n level from a window addressed by LOGICAL
// fine index (x = window - window.lo): periodic rows need no masking.
template <int NU>
__device__ __forceinline__ void dwt_pair_log(const FiltSmem<NU>& F, const Taps<NU>& tp, const double* x,
                                             int n, int mm, bool vmp, double& c, double& d) {
    const int half = n >> 1;
    if (!vmp || (mm >= NU && mm < half - NU)) {
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
        for (int u = -NU + 1; u <= NU; ++u) {
            const double xv = x[2 * mm + u];
            if (u & 1) {
                a1 += tp.h[u + NU - 1] * xv;
                b1 += tp.g[u + NU - 1] * xv;
            } else {
                a0 += tp.h[u + NU - 1] * xv;
                b0 += tp.g[u + NU - 1] * xv;
            }
        }
        c = a0 + a1;
        d = b0 + b1;
        return;
    }
    constexpr int EL = FiltSmem<NU>::EL;
    const int side = mm < NU ? 0 : 1;
    const int m = side ? half - 1 - mm : mm;
    const double* ra = F.ana(side, 0, m);
    const double* rb = F.ana(side, 1, m);
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;  // two chains per output (latency)
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
    c = a0 + a1;
    d = b0 + b1;
}

// ---------------------------------------------------------------------------
// large path: multilevel wavelet pyramids (one launch for many levels)
// ---------------------------------------------------------------------------
// Warp-granular synthesis pyramid: every WARP owns one chunk of 2^cb fine
// samples of level `top` and runs its own cone (windows, prefetch, levels)
// with __syncwarp only -- no CTA barrier after the filter staging, so the
// warps of a CTA (and of the other resident CTAs) overlap their load,
// compute and store phases freely.
// One warp's synthesis cone, part 1 (lane 0): the windows of fine samples
// [lo, hi) of level p.top down to level p.bot.  Per-warp scratch wb: ints
// wlo/whi/doff (48 doubles), then P, Q (p.wmax each) and the detail windows D.
template <int NU>
__device__ __forceinline__ void warp_syn_windows(const PyrArgs& p, double* wb, int lo, int hi, bool vmp) {
    int* wlo = reinterpret_cast<int*>(wb);
    int* whi = wlo + 32;
    int* doff = wlo + 64;
    Win f{lo, hi};
    for (int lev = p.top; lev >= p.bot; --lev) {
        wlo[lev] = f.lo;
        whi[lev] = f.hi;
        if (lev > p.bot) {
            f = syn_need(NU, 1 << lev, f, vmp);
            if (f.hi - f.lo > (((p.top - lev) & 1) ? p.wmax2 : p.wmax)) __trap();  // slot size
        }
    }
    int off = 0;  // even offsets, room for the bulk copies' 16-byte rounding on both sides
    for (int lev = p.bot + 1; lev <= p.top; ++lev) {
        doff[lev] = off;
        off += (whi[lev - 1] - wlo[lev - 1] + 2) & ~1;
    }
    if (off > p.dsum) __trap();
}

// part 2 (the whole warp, after the windows are visible): prefetch the
// level-bot coarse window and every level's detail window, synthesise up to
// level p.top and hand the top samples to put(i, value).
template <int NU, class Put, class Put2>
__device__ __forceinline__ void warp_syn_run(const PyrArgs& p, const FiltSmem<NU>& F, const Taps<NU>& tp,
                                             double* wb, int v, int lane, bool vmp, Put&& put, Put2&& put2) {
    const int* wlo = reinterpret_cast<const int*>(wb);
    const int* whi = wlo + 32;
    const int* doff = wlo + 64;
    // level lev's window sits in buffer (lev - bot) & 1; the host sized slot 0 (wmax)
    // for the level top-1 window and slot 1 (wmax2) for the other parity
    const bool swap01 = ((p.top - 1 - p.bot) & 1) != 0;
    double* P = wb + 48;
    double* Q = P + (swap01 ? p.wmax2 : p.wmax);
    double* D = P + p.wmax + p.wmax2;
    const double* xb = p.x + p.lx.vbase(p.xv0 + v);
    const double* cs = p.src_is_x ? xb : p.src + v * p.src_vs;
    // Every staged window keeps sample i at an address of i's 16-byte phase
    // (slot bases are 16-byte aligned: + (lo & 1)), so that a window is ONE bulk
    // copy (TMA engine: full 128-byte shared-memory wavefronts, where cp.async
    // writes land sector by sector) from lo & ~1, an even number of samples --
    // lane 0 the level-bot coarse window, lane i the details d_{bot+i-1}; all
    // complete on this warp's mbarrier (count = number of windows)
    uint64_t* wbar = reinterpret_cast<uint64_t*>(D + p.dsum);
    const bool bulk = vmp && ((reinterpret_cast<uintptr_t>(xb) | reinterpret_cast<uintptr_t>(cs)) & 15) == 0;
    if (bulk) {
        if (lane <= p.top - p.bot) {
            const int L = lane == 0 ? p.bot : p.bot + lane - 1;
            const int lo = wlo[L], w = whi[L] - lo;
            const double* src = lane == 0 ? cs : xb + (1 << L);
            double* dst = lane == 0 ? P : D + doff[L + 1];
            const int cnt = ((lo & 1) + w + 1) & ~1;
            mbar_arrive_expect(wbar, (unsigned)(cnt * 8));
            bulk_g2s(dst, src + (lo & ~1), (unsigned)(cnt * 8), wbar);
        }
    } else {
        {
            const int lo = wlo[p.bot], w = whi[p.bot] - lo, hb = 1 << p.bot;
            double* pp = P + (lo & 1);
            for (int t = lane; t < w; t += 32) cp_async8(pp + t, cs + (vmp ? lo + t : ((lo + t) & (hb - 1))));
        }
        for (int lev = p.bot + 1; lev <= p.top; ++lev) {  // details of level lev (half = 2^(lev-1))
            const int lo = wlo[lev - 1], w = whi[lev - 1] - lo, hf = 1 << (lev - 1);
            const double* ds = xb + hf;
            double* dd = D + doff[lev] + (lo & 1);
            // (16-byte window copies measured slower here: cfg2 49.8 vs 47.3 us)
            for (int t = lane; t < w; t += 32) cp_async8(dd + t, ds + (vmp ? lo + t : ((lo + t) & (hf - 1))));
        }
    }
    if (p.pfd > 0) {
        // L2 prefetch of the windows of the warp with this index in the CTA pfd
        // linear block indices ahead (this warp's windows shifted by whole chunks)
        const long long lin = (long long)blockIdx.y * gridDim.x + blockIdx.x + p.pfd;
        if (lin < (long long)gridDim.x * gridDim.y && lane <= p.top - p.bot) {
            const long long v2 = lin / gridDim.x;
            const long long dc = ((long long)(lin % gridDim.x) - (long long)blockIdx.x) * (blockDim.x >> 5);
            const double* xb2 = p.x + p.lx.vbase(p.xv0 + v2);
            const int L = p.bot + lane - 1;  // lane 0: the coarse window of level bot; lane i: details d_{bot+i-1}
            const int LL = lane == 0 ? p.bot : L, sh = p.cb - (p.top - LL);
            if (sh >= 0) {
                const long long lo2 = wlo[LL] + dc * (1ll << sh);
                const int w = whi[LL] - wlo[LL];
                const double* b0 = lane == 0 ? (p.src_is_x ? xb2 : p.src + v2 * p.src_vs) : xb2 + (1ll << LL);
                l2_prefetch_span(b0 + lo2, w, b0, b0 + (1ll << LL));
            }
        }
    }
    if (bulk) mbar_wait(wbar, 0);
    else cp_async_wait_all();
    __syncwarp();
    for (int lev = p.bot + 1; lev <= p.top; ++lev) {
        const int n = 1 << lev;
        const int clo = wlo[lev - 1], lo = wlo[lev], hi = whi[lev];
        const double* dw = D + doff[lev] + (clo & 1);
        const double* cwin = P + (clo & 1);
        if (lev < p.top) {
            double* q = Q + (lo & 1) - lo;  // the computed window at its samples' 16-byte phase too: pair stores
            idwt_window<NU>(F, tp, cwin, dw, clo, n, lo, hi, vmp, lane, 32, [&](int i, double val) { q[i] = val; },
                            [&](int i, double a, double b) { *reinterpret_cast<double2*>(q + i) = make_double2(a, b); });
            __syncwarp();
        } else {
            idwt_window<NU>(F, tp, cwin, dw, clo, n, lo, hi, vmp, lane, 32, put, put2);
        }
        double* t0 = P;
        P = Q;
        Q = t0;
    }
}

// Warp-granular synthesis pyramid: every WARP owns one chunk of 2^cb fine
// samples of level `top` and runs its own cone (windows, prefetch, levels)
// with __syncwarp only -- no CTA barrier after the filter staging, so the
// warps of a CTA (and of the other resident CTAs) overlap their load,
// compute and store phases freely.
template <int NU>
__global__ void __launch_bounds__(256) k_idwt_wpyr(PyrArgs p) {
    extern __shared__ double sm[];
    constexpr int FS = FiltSmem<NU>::SIZE;
    double* filt = sm;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5, nt = blockDim.x;
    double* wb = sm + FS + wid * (48 + p.wmax + p.wmax2 + p.dsum + 2);  // + this warp's mbarrier
    const int c = blockIdx.x * nw + wid, v = blockIdx.y;
    const bool vmp = p.vmp != 0;
    for (int i = tid; i < FS; i += nt) filt[i] = p.tab[p.t.o_h + i];
    if (lane == 0) {
        warp_syn_windows<NU>(p, wb, c << p.cb, (c + 1) << p.cb, vmp);
        mbar_init(reinterpret_cast<uint64_t*>(wb + 48 + p.wmax + p.wmax2 + p.dsum), (unsigned)(p.top - p.bot + 1));
    }
    __syncthreads();  // filters (CTA-wide) and the windows
    const FiltSmem<NU> F{filt};
    const Taps<NU> tp(F);
    double* ob = p.out + v * p.out_vs;
    // (16-byte pair stores when this vector's output starts 16-byte aligned)
    const bool oal = (reinterpret_cast<uintptr_t>(ob) & 15) == 0;
    warp_syn_run<NU>(p, F, tp, wb, v, lane, vmp, [&](int i, double val) { ob[i] = val; },
                     [&](int i, double a, double b) {
                         if (oal) {
                             *reinterpret_cast<double2*>(ob + i) = make_double2(a, b);
                         } else {
                             ob[i] = a;
                             ob[i + 1] = b;
                         }
                     });
}

// Coarse tail of an analysis pyramid launch: the last CTA of vector v to
// finish (atomic ticket) loads the whole level-bot coarse vector from cws and
// runs levels bot..r0+1 in shared memory (`buf`: 2 * 2^bot doubles).
template <int NU>
__device__ __forceinline__ void dwt_coarse_tail(const PyrArgs& p, const FiltSmem<NU>& F, double* buf, int v,
                                                int tid, int nt) {
    __shared__ unsigned s_last;
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(p.cnt + v, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const bool vmp = p.vmp != 0;
    double* yb = p.y + p.ly.vbase(p.yv0 + v);
    const int n0 = 1 << p.bot;
    // both ping-pong halves at the phase that puts tap 2k - nu + 1 on a 16-byte
    // boundary: interior rows read nu double2 pairs (host slack: 2 doubles)
    buf += (((reinterpret_cast<uintptr_t>(buf) >> 3) & 1) + 1 - NU) & 1;
    double* cur = buf;
    double* nxt = buf + n0;
    for (int i = tid; i < n0; i += nt) cur[i] = __ldcg(p.cws + v * p.cws_vs + i);
    __syncthreads();
    const Taps<NU> tp(F);
    for (int lev = p.bot; lev > p.r0; --lev) {
        const int m = 1 << lev, half = m >> 1;
        for (int k = tid; k < half; k += nt) {
            double cc, dd;
            if (NU > 1 && vmp && k >= NU && k < half - NU) {
                const double2* xp = reinterpret_cast<const double2*>(cur + 2 * k - NU + 1);
                double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
                for (int q = 0; q < NU; ++q) {
                    const double2 pr = xp[q];
                    a0 = fma(tp.h[2 * q], pr.x, a0);
                    b0 = fma(tp.g[2 * q], pr.x, b0);
                    a1 = fma(tp.h[2 * q + 1], pr.y, a1);
                    b1 = fma(tp.g[2 * q + 1], pr.y, b1);
                }
                cc = a0 + a1;
                dd = b0 + b1;
            } else {
                dwt_pair<NU>(F, cur, m, k, vmp, cc, dd);
            }
            yb[half + k] = dd;
            nxt[k] = cc;
        }
        __syncthreads();
        double* t0 = cur;
        cur = nxt;
        nxt = t0;
    }
    for (int i = tid; i < (1 << p.r0); i += nt) yb[i] = cur[i];
    if (tid == 0) p.cnt[v] = 0u;  // ticket ready for the next launch
}

// Warp-granular analysis pyramid (steps top..bot+1, optional tail): every WARP
// owns rows [c, c+1) * 2^(s-1-lognc) of each step, loads its cone's fine
// window and writes its detail rows and its level-bot coarse rows (to cws, or
// the output when bot == r0).  __syncwarp only.
template <int NU>
__global__ void __launch_bounds__(256) k_dwt_wpyr(PyrArgs p) {
    extern __shared__ double sm[];
    constexpr int FS = FiltSmem<NU>::SIZE;
    double* filt = sm;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    const int per = 64 + p.wmax + p.wmax2 + 2;  // slot 0: windows of steps top, top-2, ...; slot 1: the others; mbarrier
    double* wb = sm + FS + wid * per;
    uint64_t* wbar = reinterpret_cast<uint64_t*>(wb + 64 + p.wmax + p.wmax2);  // this warp's window landed
    int* rlo = reinterpret_cast<int*>(wb);
    int* rhi = rlo + 32;
    int* xlo = rlo + 64;
    int* xhi = rlo + 96;
    double* X = wb + 64;
    double* Y = X + p.wmax;
    const int c = blockIdx.x * nw + wid, v = blockIdx.y;
    const bool vmp = p.vmp != 0;
    const int lnc = p.top - p.cb;
    for (int i = tid; i < FS; i += blockDim.x) filt[i] = p.tab[p.t.o_h + i];
    if (lane == 0) {
        mbar_init(wbar, 1);
        Win r{c << (p.bot - lnc), (c + 1) << (p.bot - lnc)};
        for (int s = p.bot + 1; s <= p.top; ++s) {
            const Win w = ana_need(NU, 1 << s, r, vmp);
            rlo[s] = r.lo;
            rhi[s] = r.hi;
            xlo[s] = w.lo;
            xhi[s] = w.hi;
            if (w.hi - w.lo > (((p.top - s) & 1) ? p.wmax2 : p.wmax)) __trap();  // slot size
            r = w;
        }
    }
    __syncthreads();
    // Every window is stored so that sample 2mm - nu + 1 of each row mm sits at a
    // 16-byte boundary: the 2nu-tap rows then read nu double2 pairs (half the
    // shared-memory wavefronts of 2nu scalar loads at a 16-byte lane stride).
    // (slack: +1 in both slots)
    auto pair_al = [&](double* base, int x0) {  // shifted slot start for a window from x0
        const int par = (int)((reinterpret_cast<uintptr_t>(base) >> 3) & 1);
        return ((par + 1 - NU - x0) & 1) ? base + 1 : base;
    };
    double* const S0 = X;  // slot bases (unshifted)
    double* const S1 = Y;
    bool bulk = false;
    {
        const double* src = p.src + v * p.src_vs;
        const int lo = xlo[p.top], w = xhi[p.top] - lo, n = 1 << p.top;
        X = pair_al(S0, lo);
        // the window as ONE bulk copy (TMA engine: full 128-byte shared-memory
        // wavefronts, where cp.async writes land sector by sector) when source and
        // slot share their 16-byte phase (odd nu): widened to 16-byte bounds --
        // one sample before (slot slack) and / or after (n is even) the window
        const double* s0 = src + lo;
        double* d0 = X;
        int cnt = w;
        if (reinterpret_cast<uintptr_t>(s0) & 15) {
            --s0;
            --d0;
            ++cnt;
        }
        cnt = (cnt + 1) & ~1;
        bulk = vmp && (reinterpret_cast<uintptr_t>(d0) & 15) == 0 && d0 >= S0;
        if (bulk) {
            if (lane == 0) {
                mbar_arrive_expect(wbar, (unsigned)(cnt * 8));
                bulk_g2s(d0, s0, (unsigned)(cnt * 8), wbar);
            }
        } else if (vmp) {
            warp_copy_span(X, src + lo, w, lane);  // 16-byte copies when the phases agree
        } else {
            for (int t = lane; t < w; t += 32) cp_async8(X + t, src + ((lo + t) & (n - 1)));
        }
    }
    if (p.pfd > 0 && lane == 0) {  // L2 prefetch of the window of this warp index in the CTA pfd blocks ahead
        const long long lin = (long long)blockIdx.y * gridDim.x + blockIdx.x + p.pfd;
        if (lin < (long long)gridDim.x * gridDim.y) {
            const long long v2 = lin / gridDim.x;
            const long long dc = ((long long)(lin % gridDim.x) - (long long)blockIdx.x) * nw;
            const double* s2 = p.src + v2 * p.src_vs;
            l2_prefetch_span(s2 + xlo[p.top] + dc * (1ll << p.cb), xhi[p.top] - xlo[p.top], s2, s2 + (1ll << p.top));
        }
    }
    if (bulk) mbar_wait(wbar, 0);
    else cp_async_wait_all();
    __syncwarp();
    const FiltSmem<NU> F{filt};
    const Taps<NU> tp(F);
    double* yb = p.y + p.ly.vbase(p.yv0 + v);  // large path: contiguous 1D output
    bool xin0 = true;  // X lives in slot 0
    for (int s = p.top; s > p.bot; --s) {
        const int n = 1 << s, half = n >> 1;
        const int lo = rlo[s], hi = rhi[s];
        const int plo = c << (s - 1 - lnc), phi = (c + 1) << (s - 1 - lnc);
        const double* xv = X - xlo[s];
        Y = pair_al(xin0 ? S1 : S0, lo);  // the next step reads rows [lo, hi) as its window
        double* yv = Y - lo;
        const bool last = s == p.bot + 1;
        for (int mm = lo + lane; mm < hi; mm += 32) {
            double c0, d0;
            if (!vmp || (mm >= NU && mm < half - NU)) {  // interior: nu aligned pairs
                const double2* xp = reinterpret_cast<const double2*>(xv + 2 * mm - NU + 1);
                double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
                for (int k = 0; k < NU; ++k) {
                    const double2 pr = xp[k];  // u = 2k - nu + 1 (.x) and u + 1 (.y)
                    a0 = fma(tp.h[2 * k], pr.x, a0);
                    b0 = fma(tp.g[2 * k], pr.x, b0);
                    a1 = fma(tp.h[2 * k + 1], pr.y, a1);
                    b1 = fma(tp.g[2 * k + 1], pr.y, b1);
                }
                c0 = a0 + a1;
                d0 = b0 + b1;
            } else {
                dwt_pair_log<NU>(F, tp, xv, n, mm, vmp, c0, d0);
            }
            if (!last) yv[mm] = c0;
            if (mm >= plo && mm < phi) {
                yb[half + mm] = d0;
                if (last) {
                    if (p.cws) p.cws[v * p.cws_vs + mm] = c0;
                    else yb[mm] = c0;
                }
            }
        }
        __syncwarp();
        X = Y;
        xin0 = !xin0;
    }
    if (p.tail) dwt_coarse_tail<NU>(p, F, sm + FS, v, tid, blockDim.x);
}

// ---------------------------------------------------------------------------
// normal form along rows: out_v = N1 in_v, N1 = W G W^-1 (use_idwt) or G
// ---------------------------------------------------------------------------
// V rows per CTA (V * M <= 4096), three smem buffers of V*M doubles: A holds
// the input (coarse + all details), the IDWT ping-pongs through B/C, the band
// product lands in A, the DWT ping-pongs back through B/C and streams the
// detail rows straight to `out` (which may alias `in`: every row is fully
// staged before any write).  Every level loop runs over (row, index) pairs.
// One analysis level of one vector: coarse c[0:n/2] -> dstc, detail rows ->
// dstd[k] (any address space).  Interior rows with register taps, edge rows
// (VMP) / all rows (periodic, masked) through dwt_pair.
template <int NU>
__device__ __forceinline__ void dwt_level_vec(const FiltSmem<NU>& F, const Taps<NU>& tp, const double* x,
                                              double* dstc, double* dstd, int n, bool vmp, int t0, int nthr,
                                              long long dstride = 1) {
    const int half = n >> 1;
    const int klo = vmp ? NU : (NU + 1) / 2 + 1, khi = vmp ? half - NU : half - NU;
    for (int k = klo + t0; k < khi; k += nthr) {
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
        for (int u = -NU + 1; u <= NU; ++u) {
            const double xv = x[2 * k + u];
            if (u & 1) {
                a1 = fma(tp.h[u + NU - 1], xv, a1);
                b1 = fma(tp.g[u + NU - 1], xv, b1);
            } else {
                a0 = fma(tp.h[u + NU - 1], xv, a0);
                b0 = fma(tp.g[u + NU - 1], xv, b0);
            }
        }
        dstc[k] = a0 + a1;
        dstd[k * dstride] = b0 + b1;
    }
    const int nl = klo, nr = half - khi;
    for (int r = nthr - 1 - t0; r < nl + nr; r += nthr) {  // boundary rows
        const int k = r < nl ? r : khi + (r - nl);
        double c, d;
        dwt_pair<NU>(F, x, n, k, vmp, c, d);
        dstc[k] = c;
        dstd[k * dstride] = d;
    }
}

// Band product y = G x of one vector (G: see NormArgs); interior rows use
// the Toeplitz row held in registers (half-bandwidth B = 2nu - 2).
template <int NU>
__device__ __forceinline__ void band_vec(const double* __restrict__ gE, const double (&gI)[4 * NU - 3], int E,
                                         const double* x, double* y, int M, bool wrap, int t0, int nthr) {
    constexpr int B = 2 * NU - 2, W = 2 * B + 1;
    for (int i = E + t0; i < M - E; i += nthr) {
        double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
        for (int d = 0; d < W; ++d) {
            if (d & 1) acc1 = fma(gI[d], x[i + d - B], acc1);
            else acc0 = fma(gI[d], x[i + d - B], acc0);
        }
        y[i] = acc0 + acc1;
    }
    for (int r = t0; r < 2 * E; r += nthr) {  // edge rows: tabulated band
        const int i = r < E ? r : M - 2 * E + r;
        const double* g = gE + r * W;
        double acc = 0.0;
#pragma unroll
        for (int d = 0; d < W; ++d) {
            int k = i + d - B;
            if (wrap) k &= M - 1;
            if (k >= 0 && k < M) acc = fma(g[d], x[k], acc);
        }
        y[i] = acc;
    }
}

template <int NU, int NT>
__global__ void __launch_bounds__(NT, 2) k_normal_rows(NormArgs p) {
    PHASE(0);
    // smem: filters | band edge rows | A, B, C [V][M] each.  A holds the
    // staged input (coarse + every level's details); the synthesis ping-pongs
    // B/C, the band product lands in A (free by then), the analysis ping-pongs
    // B/C and streams detail rows to `out` (may alias `in`: rows are staged).
    extern __shared__ double sm[];
    constexpr int FS = FiltSmem<NU>::SIZE;
    constexpr int W = 4 * NU - 3;
    double* filt = sm;
    const int j = p.j, M = 1 << j, tid = threadIdx.x;
    const long long v0 = (long long)blockIdx.x * p.V;
    const int nv = (int)(p.nvec - v0 < p.V ? p.nvec - v0 : p.V);
    double* gE = sm + FS;  // [2E][W] edge rows of the band
    double* A = gE + 2 * p.E * W;
    double* B = A + p.V * M;
    double* Cb = B + p.V * M;
    const bool vmp = p.vmp != 0;
    for (int i = tid; i < FS; i += NT) filt[i] = p.tab[p.t.o_h + i];
    for (int i = tid; i < 2 * p.E * W; i += NT) gE[i] = p.band[i];
    double gI[W];
#pragma unroll
    for (int d = 0; d < W; ++d) gI[d] = __ldg(p.band + 2 * p.E * W + d);
    for (int t = tid; t < nv * M; t += NT) cp_async8(A + t, p.in + (v0 + (t >> j)) * p.in_vs + (t & (M - 1)));
    cp_async_wait_all();
    __syncthreads();
    PHASE(1);
    const FiltSmem<NU> F{filt};
    const Taps<NU> tp(F);
    const bool wav = p.use_idwt && p.r0 < j;
    double* fine = A;
    if (wav) {
        double* src = A;  // level-r0 coarse rows live at the start of each input row
        for (int lev = p.r0 + 1; lev <= j; ++lev) {
            const int n = 1 << lev, half = n >> 1;
            double* dst = (src == B) ? Cb : B;
            for (int v = 0; v < nv; ++v)
                idwt_level_vec<NU>(F, src + v * M, A + v * M + half, dst + v * M, n, vmp, tid, NT);
            __syncthreads();
            src = dst;
        }
        fine = src;
    }
    PHASE(2);
    double* Y = wav ? A : B;  // A is free once the details are consumed
    for (int v = 0; v < nv; ++v) band_vec<NU>(gE, gI, p.E, fine + v * M, Y + v * M, M, !vmp, tid, NT);
    __syncthreads();
    PHASE(3);
    if (!wav) {
        for (int t = tid; t < nv * M; t += NT) p.out[(v0 + (t >> j)) * p.out_vs + (t & (M - 1))] = Y[t];
        return;
    }
    double* cur = Y;
    for (int lev = j; lev > p.r0; --lev) {
        const int n = 1 << lev, half = n >> 1;
        double* dst = (cur == B) ? Cb : B;
        for (int v = 0; v < nv; ++v)
            dwt_level_vec<NU>(F, tp, cur + v * M, dst + v * M, p.out + (v0 + v) * p.out_vs + half, n, vmp, tid, NT);
        __syncthreads();
        cur = dst;
    }
    PHASE(4);
    const int nc = 1 << p.r0;
    for (int t = tid; t < nv * nc; t += NT) {
        const int v = t >> p.r0, i = t & (nc - 1);
        p.out[(v0 + v) * p.out_vs + i] = cur[v * M + i];
    }
    PHASE(5);
}

// ---------------------------------------------------------------------------
// register-resident normal rows: 2^9 <= M <= 2^12, one row per CTA, 256 threads
// ---------------------------------------------------------------------------
// Above 2^kRegLog samples every thread owns a contiguous segment of each
// level: a synthesis level turns its K coarse values into 2K fine values
// that are exactly the next level's input segment, so levels chain in
// registers.  Only the halos (a few values from the neighbouring segments)
// and the VMP edge samples read a shared-memory copy of the level.  The
// analysis runs the same way downward.  Levels <= 2^kRegLog and the band
// edge rows use the shared-memory helpers.

// Register levels keep a shared-memory copy of each level for the halos in a
// padded layout (one spare double per 32) so that the segment stores / loads
// of a warp (lane stride 2K doubles) are bank-conflict free.
__device__ __forceinline__ int pidx(int i) { return i + (i >> 5); }

// synthesis of a length-n level: coarse segment c[K] (indices m0..) -> fine f[2K].
// cs: copy of the coarse level (padded when PADIN), ds: details (plain).
template <int NU, int K, bool PADIN>
__device__ __forceinline__ void syn_seg(const FiltSmem<NU>& F, const Taps<NU>& tp, const double* cs,
                                        const double* ds, int n, int m0, bool vmp, const double (&c)[K],
                                        double (&f)[2 * K]) {
    constexpr int OFF = (NU + 1) / 2, WN = K + NU + 1;
    const int half = n >> 1;
    auto cat = [&](int i) { return PADIN ? cs[pidx(i)] : cs[i]; };
    double cw[WN], dw[WN];
#pragma unroll
    for (int w = 0; w < WN; ++w) {
        int idx = m0 - OFF + w;
        const bool ok = !vmp || (idx >= 0 && idx < half);
        idx &= half - 1;
        if (w >= OFF && w < OFF + K) cw[w] = c[w - OFF];
        else cw[w] = ok ? cat(idx) : 0.0;
        dw[w] = ok ? ds[pidx(idx)] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < K; ++q) {
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
        for (int u = -NU + 1; u <= NU; ++u) {
            if ((u & 1) == 0) {
                const int idx = OFF - u / 2 + q;
                a0 = fma(tp.h[u + NU - 1], cw[idx], a0);
                b0 = fma(tp.g[u + NU - 1], dw[idx], b0);
            } else {
                const int idx = OFF - (u - 1) / 2 + q;
                a1 = fma(tp.h[u + NU - 1], cw[idx], a1);
                b1 = fma(tp.g[u + NU - 1], dw[idx], b1);
            }
        }
        f[2 * q] = a0 + b0;
        f[2 * q + 1] = a1 + b1;
    }
}

// analysis rows k0..k0+K of a length-n level from the fine segment x[2K];
// xs: padded copy of the fine level (halos, VMP edge rows)
template <int NU, int K>
__device__ __forceinline__ void ana_seg(const FiltSmem<NU>& F, const Taps<NU>& tp, const double* xs, int n, int k0,
                                        bool vmp, const double (&x)[2 * K], double (&c)[K], double (&d)[K]) {
    constexpr int WL = NU - 1, WN = 2 * K + 2 * NU - 2;
    double xw[WN];
#pragma unroll
    for (int w = 0; w < WN; ++w) {
        int idx = 2 * k0 - WL + w;
        const bool ok = !vmp || (idx >= 0 && idx < n);
        idx &= n - 1;
        if (w >= WL && w < WL + 2 * K) xw[w] = x[w - WL];
        else xw[w] = ok ? xs[pidx(idx)] : 0.0;
    }
#pragma unroll
    for (int r = 0; r < K; ++r) {
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
        for (int u = -NU + 1; u <= NU; ++u) {
            const double xv = xw[2 * r + u + WL];
            if (u & 1) {
                a1 = fma(tp.h[u + NU - 1], xv, a1);
                b1 = fma(tp.g[u + NU - 1], xv, b1);
            } else {
                a0 = fma(tp.h[u + NU - 1], xv, a0);
                b0 = fma(tp.g[u + NU - 1], xv, b0);
            }
        }
        c[r] = a0 + a1;
        d[r] = b0 + b1;
    }
}

// synthesis levels with K coarse values per thread, recursing up to KT; the
// level written by each step goes (padded) to `dst`, the next step swaps.
template <int NU, int K, int KT, bool PADIN, int RNT>
__device__ __forceinline__ void syn_up(const FiltSmem<NU>& F, const Taps<NU>& tp, const double* xin,
                                       const double* cs, double* dst, double* alt, bool vmp, const double (&c)[K],
                                       double (&fine)[2 * KT], double*& top) {
    const int tid = threadIdx.x;
    const int half = K * RNT, n = 2 * half;
    double f[2 * K];
    const double* ds = xin + pidx(half);  // details of this level (xin padded)
    syn_seg<NU, K, PADIN>(F, tp, cs, ds, n, tid * K, vmp, c, f);
    constexpr int EL = FiltSmem<NU>::EL, CI = FiltSmem<NU>::CI;
    const int i0 = 2 * K * tid;
    const bool edge = vmp && (i0 < EL || i0 + 2 * K > n - EL);
#pragma unroll
    for (int q = 0; q < 2 * K; ++q)
        if (!(edge && (i0 + q < EL || i0 + q >= n - EL))) dst[pidx(i0 + q)] = f[q];
    if (vmp && tid < 2 * EL) {  // VMP edge samples from the dense edge blocks, one per helper thread
        const int side = tid < EL ? 0 : 1, ii = side ? tid - EL : tid, i = side ? n - 1 - ii : ii;
        const double* sc = F.syn(side, ii, 0);
        const double* sd = F.syn(side, ii, 1);
        double a0 = 0.0, a1 = 0.0;  // two chains (this helper warp gates the barrier)
#pragma unroll
        for (int k = 0; k < CI; ++k) {
            const int idx = side ? half - 1 - k : k;
            const double cv = PADIN ? cs[pidx(idx)] : cs[idx];
            a0 = fma(sc[k * EL], cv, a0);
            a1 = fma(sd[k * EL], ds[pidx(idx)], a1);
        }
        dst[pidx(i)] = a0 + a1;
    }
    __syncthreads();
    if (edge) {
#pragma unroll
        for (int q = 0; q < 2 * K; ++q)
            if (i0 + q < EL || i0 + q >= n - EL) f[q] = dst[pidx(i0 + q)];
    }
    if constexpr (K == KT) {
#pragma unroll
        for (int q = 0; q < 2 * K; ++q) fine[q] = f[q];
        top = dst;
    } else {
        syn_up<NU, 2 * K, KT, true, RNT>(F, tp, xin, dst, alt, dst, vmp, f, fine, top);
    }
}

// analysis levels with 2K fine values per thread, recursing down to K = 1;
// xs: padded copy of the level being analysed, other: free padded buffer;
// the K = 1 step leaves its 2^RLOG coarse values PLAIN in `low`
template <int NU, int K, int RNT>
__device__ __forceinline__ void ana_down(const FiltSmem<NU>& F, const Taps<NU>& tp, double* out, long long es,
                                         double* xs, double* other, double* low, bool vmp, const double (&x)[2 * K]) {
    const int tid = threadIdx.x;
    const int half = K * RNT;
    double c[K], d[K];
    const int n = 2 * half, k0 = tid * K;
    ana_seg<NU, K>(F, tp, xs, n, k0, vmp, x, c, d);
    const bool edge = vmp && (k0 < NU || k0 + K > half - NU);
    auto is_edge = [&](int k) { return k < NU || k >= half - NU; };
    double* od = out + (half + k0) * es;
#pragma unroll
    for (int r = 0; r < K; ++r)
        if (!(edge && is_edge(k0 + r))) od[r * es] = d[r];
    if (vmp && tid < 2 * NU) {  // VMP edge rows (wavelet.cpp:403-445), one per helper thread
        constexpr int EL = FiltSmem<NU>::EL;
        const int side = tid < NU ? 0 : 1, m = side ? tid - NU : tid, k = side ? half - 1 - m : m;
        const double* ra = F.ana(side, 0, m);
        const double* rb = F.ana(side, 1, m);
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
        for (int q = 0; q < EL; ++q) {
            const double xv = xs[pidx(side ? n - 1 - q : q)];
            if (q & 1) {
                a1 = fma(ra[q], xv, a1);
                b1 = fma(rb[q], xv, b1);
            } else {
                a0 = fma(ra[q], xv, a0);
                b0 = fma(rb[q], xv, b0);
            }
        }
        const double a = a0 + a1, b = b0 + b1;
        out[(half + k) * es] = b;
        if (K == 1) low[k] = a;
        else other[pidx(k)] = a;
    }
    if constexpr (K == 1) {
        if (!edge) low[tid] = c[0];
        __syncthreads();
    } else {
#pragma unroll
        for (int r = 0; r < K; ++r)
            if (!(edge && is_edge(k0 + r))) other[pidx(k0 + r)] = c[r];
        __syncthreads();
        if (edge) {
#pragma unroll
            for (int r = 0; r < K; ++r)
                if (is_edge(k0 + r)) c[r] = other[pidx(k0 + r)];
        }
        double x2[K];
#pragma unroll
        for (int r = 0; r < K; ++r) x2[r] = c[r];
        ana_down<NU, K / 2, RNT>(F, tp, out, es, other, xs, low, vmp, x2);
    }
}

template <int NU, int J, int RNT>
__global__ void __launch_bounds__(RNT, 2) k_normal_rows_reg(NormArgs p) {
    constexpr int RLOG = RNT == 512 ? 9 : (RNT == 256 ? 8 : 7);  // levels <= 2^RLOG: shared memory
    constexpr int M = 1 << J, KT = M / (2 * RNT), FT = 2 * KT;  // fine values per thread
    constexpr int FS = FiltSmem<NU>::SIZE, W = 4 * NU - 3, Bw = 2 * NU - 2, PM = M + M / 32;
    constexpr int NL = 1 << RLOG;
    static_assert(NL == RNT, "one level-RLOG value per thread");
    extern __shared__ double sm[];
    double* filt = sm;
    double* gE = sm + FS;
    double* X = gE + 2 * p.E * W;  // staged input row, padded (coarse + every level's details)
    double* Pa = X + PM;           // padded level copies
    double* Pb = Pa + PM;
    double* L0 = Pb + PM;          // plain buffers of the coarse (<= 2^RLOG) levels
    double* L1 = L0 + NL;
    double* XL = L1 + NL;          // plain copy of the input's first 2^RLOG values
    const int tid = threadIdx.x;
    const bool vmp = p.vmp != 0;
    for (int i = tid; i < FS; i += RNT) filt[i] = p.tab[p.t.o_h + i];
    for (int i = tid; i < 2 * p.E * W; i += RNT) gE[i] = p.band[i];
    double gI[W];
#pragma unroll
    for (int d = 0; d < W; ++d) gI[d] = __ldg(p.band + 2 * p.E * W + d);
    const long long v = blockIdx.x;
    const long long es = p.es > 0 ? p.es : 1;
    const long long vb = p.es > 0 ? (v / p.vpi) * p.ivs + (v % p.vpi) * p.in_vs : v * p.in_vs;
    const double* xg = p.in + vb;
    double* out = p.out + (p.es > 0 ? vb : v * p.out_vs);
#pragma unroll
    for (int r = 0; r < M / RNT; ++r) cp_async8(X + pidx(tid + r * RNT), xg + (tid + r * RNT) * es);
    cp_async8(XL + tid, xg + tid * es);  // RNT == 2^RLOG
    if (tid == 0 && p.pfd > 0 && p.es <= 0 && v + p.pfd < p.nvec)  // a later CTA's row into L2
        l2_prefetch_span(p.in + (v + p.pfd) * p.in_vs, M, p.in, p.in + p.nvec * p.in_vs);
    cp_async_wait_all();
    __syncthreads();
    const FiltSmem<NU> F{filt};
    const Taps<NU> tp(F);
    // coarse synthesis levels r0+1 .. RLOG (plain shared memory)
    const int nc = 1 << p.r0;
    const double* src = XL;  // the level-r0 coarse values lead the input row
    double* dst = L0;
    for (int lev = p.r0 + 1; lev <= RLOG; ++lev) {
        const int n = 1 << lev;
        idwt_level_vec<NU>(F, src, XL + (n >> 1), dst, n, vmp, tid, RNT);
        __syncthreads();
        src = dst;
        dst = (dst == L0) ? L1 : L0;
    }
    // register levels RLOG+1 .. J
    double fine[FT];
    double* top = nullptr;
    {
        const double c1[1] = {src[tid]};
        syn_up<NU, 1, KT, false, RNT>(F, tp, X, src, Pa, Pb, vmp, c1, fine, top);
    }
    double* fre = (top == Pa) ? Pb : Pa;
    // band product in registers (halos / edge rows from the padded top level)
    double y[FT];
    {
        const int i0 = tid * FT;
        constexpr int WN = FT + 2 * Bw;
        double xw[WN];
#pragma unroll
        for (int w = 0; w < WN; ++w) {
            const int idx = i0 - Bw + w;
            if (w >= Bw && w < Bw + FT) xw[w] = fine[w - Bw];
            else xw[w] = (!vmp || (idx >= 0 && idx < M)) ? top[pidx(idx & (M - 1))] : 0.0;
        }
#pragma unroll
        for (int r = 0; r < FT; ++r) {
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int d = 0; d < W; ++d) {
                if (d & 1) a1 = fma(gI[d], xw[r + d], a1);
                else a0 = fma(gI[d], xw[r + d], a0);
            }
            y[r] = a0 + a1;
        }
    }
    const int i0 = tid * FT;
    const bool bedge = i0 < p.E || i0 + FT > M - p.E;
#pragma unroll
    for (int r = 0; r < FT; ++r)
        if (!(bedge && (i0 + r < p.E || i0 + r >= M - p.E))) fre[pidx(i0 + r)] = y[r];
    if (tid < 2 * p.E) {  // tabulated edge rows of the band, one per helper thread
        const int i = tid < p.E ? tid : M - 2 * p.E + tid;
        double acc = 0.0;
#pragma unroll
        for (int d = 0; d < W; ++d) {
            int k = i + d - Bw;
            if (!vmp) k &= M - 1;
            if (k >= 0 && k < M) acc = fma(gE[tid * W + d], top[pidx(k)], acc);
        }
        fre[pidx(i)] = acc;
    }
    __syncthreads();
    if (bedge) {
#pragma unroll
        for (int r = 0; r < FT; ++r)
            if (i0 + r < p.E || i0 + r >= M - p.E) y[r] = fre[pidx(i0 + r)];
    }
    // analysis: register levels J .. RLOG+1, then the coarse levels (plain)
    ana_down<NU, KT, RNT>(F, tp, out, es, fre, top, L0, vmp, y);
    double* cur = L0;
    double* nxt = L1;
    for (int lev = RLOG; lev > p.r0; --lev) {
        const int n = 1 << lev, half = n >> 1;
        dwt_level_vec<NU>(F, tp, cur, nxt, out + half * es, n, vmp, tid, RNT, es);
        __syncthreads();
        double* t0 = cur;
        cur = nxt;
        nxt = t0;
    }
    for (int i = tid; i < nc; i += RNT) out[i * es] = cur[i];
}

// fused finest synthesis level in forward pass 1: the chunk's coarse / detail
// windows are staged in this many pieces; window length (doubles, even) of a
// piece of `pairs` output pairs
constexpr int kFusePieces = 4;
__host__ __device__ constexpr int fuse_window(int pairs, int nu) { return (pairs + nu + 3) & ~1; }

// ---------------------------------------------------------------------------
// large path: two-pass Hadamard over K with an L2-resident intermediate
// ---------------------------------------------------------------------------
// G per vector: [2^kh chunks][R1 physical rows][CW]; chunk c = K_hi (forward
// pass 1 output) and physical row rho = bitrev_kl(N_lo).

template <int NU, int NT>
__global__ void __launch_bounds__(NT, CWW_CONTIG_MINB) k_large_fwd1(LargeArgs p) {
    using Gm = Geo<NU, kLogB>;
    // the contiguous pass's tile rows are unpadded (RS = CW): its lane patterns walk
    // columns only, and the tile is then byte-for-byte the chunk's G block
    constexpr int B = Gm::B, H = Gm::H, CW = Gm::CW, RS = CW;
    extern __shared__ double sm[];
    const int tid = threadIdx.x;
    const int j = p.j, M = 1 << j, a = j - kLogB, A = 1 << a;
    const int kl = p.kl, R1 = 1 << kl;
    const int chunk = blockIdx.x, v = blockIdx.y;
    const double* xi = p.xi + (long long)v * p.xi_vs;
    double* T = sm;
    const double* src = p.xi_is_input ? p.in + p.lin.vbase(p.v0 + v) : xi;  // large path: contiguous
    const long long cbase = (long long)chunk * R1 * B;
    const bool echunk = NU > 1 && (chunk == 0 || cbase + R1 * B >= M);  // holds edge positions
    if (p.fuse_top) {
        // the finest synthesis level (wavelet.cpp:447-483 gather form) straight
        // into the tile.  The chunk's c_{j-1} / d_{j-1} windows are staged in
        // kFusePieces pieces by bulk copies (TMA engine, one mbarrier phase per
        // piece); pair m -> samples 2m, 2m+1 from window entries
        // m-OFF .. m-OFF+NU; VMP edge samples / periodic wrap via idwt_one
        // from global memory (first / last chunk only)
        const FiltSmem<NU> F{p.tab + p.t.o_h};
        const Taps<NU> tp(F);
        const bool vmp = p.vmp != 0;
        const int half = M >> 1;
        const double* cv = p.xi + (long long)v * p.xi_vs;
        const double* dv = p.in + p.lin.vbase(p.v0 + v) + half;
        constexpr int OFF = (NU + 1) / 2, EL = FiltSmem<NU>::EL;
        const int mlo = vmp ? (EL + 1) >> 1 : OFF, mhi = vmp ? (M - EL) >> 1 : half - (NU - OFF);
        const int m0 = (int)(cbase >> 1);
        const int ppairs = R1 * B / 2 / kFusePieces;
        const int WP = fuse_window(ppairs, NU);
        // two window buffers (ring): piece pc + 1 lands while piece pc is consumed
        uint64_t* bar = reinterpret_cast<uint64_t*>(T + R1 * RS);  // [2]
        double* Wb = T + R1 * RS + 2;                               // [2][C | D][WP]
        const bool al = ((reinterpret_cast<uintptr_t>(cv) | reinterpret_cast<uintptr_t>(dv)) & 15) == 0;
        auto win = [&](int pc, int& ws, int& len) {
            const int mp = m0 + pc * ppairs;
            ws = max(0, (mp - OFF) & ~1);
            len = min(half, (mp + ppairs + NU - OFF + 1) & ~1) - ws;
        };
        auto issue = [&](int pc) {  // thread 0: bulk copies of piece pc into buffer pc & 1
            int ws, len;
            win(pc, ws, len);
            double* Cw = Wb + (pc & 1) * 2 * WP;
            mbar_arrive_expect(bar + (pc & 1), (unsigned)(2 * len * 8));
            bulk_g2s(Cw, cv + ws, (unsigned)(len * 8), bar + (pc & 1));
            bulk_g2s(Cw + WP, dv + ws, (unsigned)(len * 8), bar + (pc & 1));
        };
        if (tid == 0) {
            mbar_init(bar, 1);
            mbar_init(bar + 1, 1);
        }
        __syncthreads();
        if (al && tid == 0) {
            issue(0);
            if (kFusePieces > 1) issue(1);
        }
        for (int pc = 0; pc < kFusePieces; ++pc) {
            const int mp = m0 + pc * ppairs;
            int ws, len;
            win(pc, ws, len);
            double* Cw = Wb + (pc & 1) * 2 * WP;
            double* Dw = Cw + WP;
            if (al) {
                mbar_wait(bar + (pc & 1), (unsigned)((pc >> 1) & 1));
            } else {  // caller's buffer only 8-byte aligned: element-wise async copies
                for (int t = tid; t < len; t += NT) {
                    cp_async8(Cw + t, cv + ws + t);
                    cp_async8(Dw + t, dv + ws + t);
                }
                cp_async_wait_all();
                __syncthreads();
            }
            for (int t = tid; t < ppairs; t += NT) {
                const int m = mp + t;
                double o0, o1;
                if (m >= mlo && m < mhi) {
                    const double* cw = Cw + (m - OFF - ws);
                    const double* dw = Dw + (m - OFF - ws);
                    double c[NU + 1], d[NU + 1];
#pragma unroll
                    for (int k = 0; k <= NU; ++k) {
                        c[k] = cw[k];
                        d[k] = dw[k];
                    }
                    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
                    for (int u = -NU + 1; u <= NU; ++u) {
                        if ((u & 1) == 0) {
                            a0 = fma(tp.h[u + NU - 1], c[OFF - u / 2], a0);
                            b0 = fma(tp.g[u + NU - 1], d[OFF - u / 2], b0);
                        } else {
                            a1 = fma(tp.h[u + NU - 1], c[OFF - (u - 1) / 2], a1);
                            b1 = fma(tp.g[u + NU - 1], d[OFF - (u - 1) / 2], b1);
                        }
                    }
                    o0 = a0 + b0;
                    o1 = a1 + b1;
                } else {
                    o0 = idwt_one<NU>(F, cv, dv, M, 2 * m, vmp);
                    o1 = idwt_one<NU>(F, cv, dv, M, 2 * m + 1, vmp);
                }
                const int pos = 2 * m, rl = (pos - (int)cbase) >> kLogB, col = pos & (B - 1);
                double* dst = T + (int)brev_bits((unsigned)rl, kl) * RS + H + col;
                if (echunk && (pos < NU || pos + 1 >= M - NU)) {  // edge positions: raw value to ev, 0 in the tile
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int q = pos + e;
                        const double o = e ? o1 : o0;
                        if (q < NU || q >= M - NU) {
                            p.ev[(long long)v * 2 * NU + (q < NU ? q : NU + (q - (M - NU)))] = o;
                            dst[e] = 0.0;
                        } else {
                            dst[e] = o;
                        }
                    }
                } else {
                    dst[0] = o0;
                    dst[1] = o1;
                }
            }
            __syncthreads();  // buffer pc & 1 is free: refill it with piece pc + 2
            if (al && tid == 0 && pc + 2 < kFusePieces) issue(pc + 2);
        }
        if (H > 0 && tid < 2 * H) {  // outer halos: samples of the neighbouring chunks
            const bool left = tid < H;
            const int c = left ? tid : tid - H;
            const long long pos = left ? cbase - H + c : cbase + (long long)R1 * B + c;
            double* dst = left ? T + c : T + (int)brev_bits((unsigned)(R1 - 1), kl) * RS + B + H + c;
            *dst = (pos >= 0 && pos < M && !(NU > 1 && (pos < NU || pos >= M - NU)))
                       ? idwt_one<NU>(F, cv, dv, M, (int)pos, vmp)
                       : 0.0;
        }
    } else {
        // each source sample once, into its row's own columns [H, B + H): one
        // warp per logical row, lane = column (coalesced, warp-uniform row math)
        const int lane = tid & 31;
        for (int rl = tid >> 5; rl < R1; rl += NT / 32) {
            const long long pos = cbase + (long long)rl * B + lane;
            double* dst = T + (int)brev_bits((unsigned)rl, kl) * RS + H + lane;
            if (echunk && (pos < NU || pos >= M - NU)) *dst = 0.0;  // edge position (edge terms)
            else cp_async8(dst, src + pos);
        }
        if (H > 0 && tid < 2 * H) {  // the chunk's outer halos come from the neighbouring chunks
            const bool left = tid < H;
            const int c = left ? tid : tid - H;
            const long long pos = left ? cbase - H + c : cbase + (long long)R1 * B + c;
            double* dst = left ? T + c : T + (int)brev_bits((unsigned)(R1 - 1), kl) * RS + B + H + c;
            if (pos >= 0 && pos < M && !(NU > 1 && (pos < NU || pos >= M - NU))) cp_async8(dst, src + pos);
            else *dst = 0.0;
        }
    }
    if (NU > 1 && !p.fuse_top && tid < 2 * NU) {  // raw edge values (first / last chunk)
        const int c = tid;
        const long long pos = c < NU ? c : (M - NU) + (c - NU);
        if ((int)((pos / B) / R1) == chunk)
            p.ev[(long long)v * 2 * NU + c] = p.xi_is_input ? p.in[p.lin.at(p.v0 + v, pos)] : xi[pos];
    }
    cp_async_wait_all();
    __syncthreads();
    if (H > 0) {  // inner halos: copies of the neighbouring rows' own columns
        // (thread = (physical row, halo column): consecutive lanes walk consecutive
        // physical rows, whose 36-double stride spreads them over the banks)
        for (int f = tid; f < R1 * 2 * H; f += NT) {
            const int ph = f / (2 * H), c = f % (2 * H);
            const int K = (int)brev_bits((unsigned)ph, kl);  // this row's halos from its neighbours
            if (c < H) {  // right halo: the next row's first columns
                if (K + 1 < R1) T[ph * RS + B + H + c] = T[(int)brev_bits((unsigned)(K + 1), kl) * RS + H + c];
            } else {      // left halo: the previous row's last columns
                if (K > 0) T[ph * RS + (c - H)] = T[(int)brev_bits((unsigned)(K - 1), kl) * RS + B + (c - H)];
            }
        }
        __syncthreads();
    }
    tile_hadamard_inl<CW, RS, CWW_CONTIG_MAXR>(T, 1, kl, 0, kl, 0, tid, NT);
    double* g = p.G + (long long)v * A * CW + (long long)chunk * R1 * CW;
    // tile == G block: one bulk store (TMA engine) once every thread's last
    // Hadamard writes are visible to the async proxy
    static_assert(CW % 2 == 0, "16-byte bulk G stores");
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
        bulk_s2g(g, T, (unsigned)(R1 * CW * 8));
        bulk_commit();
        bulk_wait_read();
    }
}

// Persistent variant of the fused forward pass 1 (16-byte aligned inputs):
// every CTA walks tasks (vector, chunk) blockIdx.x, +gridDim.x, ...; the
// window pieces form one ring across the CTA's tasks, so the next task's
// first two pieces land during this task's halo / Hadamard / store phases,
// and the G block's bulk store overlaps the next task's first piece.
template <int NU, int NT>
__global__ void __launch_bounds__(NT, 2) k_large_fwd1_fz(LargeArgs p) {
    using Gm = Geo<NU, kLogB>;
    constexpr int B = Gm::B, H = Gm::H, CW = Gm::CW, RS = CW;
    constexpr int OFF = (NU + 1) / 2, EL = FiltSmem<NU>::EL, KP = kFusePieces;
    extern __shared__ double sm[];
    const int tid = threadIdx.x;
    const int j = p.j, M = 1 << j, a = j - kLogB, A = 1 << a, half = M >> 1;
    const int kl = p.kl, R1 = 1 << kl, nch = A >> kl;
    const long long ntask = (long long)nch * p.nvec;
    double* T = sm;
    uint64_t* bar = reinterpret_cast<uint64_t*>(T + R1 * RS);  // [2]
    double* Wb = T + R1 * RS + 2;                               // [2][C | D][WP]
    const int ppairs = R1 * B / 2 / KP;
    const int WP = fuse_window(ppairs, NU);
    const FiltSmem<NU> F{p.tab + p.t.o_h};
    const Taps<NU> tp(F);
    const bool vmp = p.vmp != 0;
    const int mlo = vmp ? (EL + 1) >> 1 : OFF, mhi = vmp ? (M - EL) >> 1 : half - (NU - OFF);
    auto task_of = [&](long long lp) { return (long long)blockIdx.x + (lp / KP) * gridDim.x; };
    // thread 0: bulk copies of this CTA's ring piece lp into buffer lp & 1
    auto issue = [&](long long lp) {
        const long long t = task_of(lp);
        if (t >= ntask) return;
        const int v = (int)(t / nch), chunk = (int)(t % nch), pc = (int)(lp % KP);
        const double* cv = p.xi + (long long)v * p.xi_vs;
        const double* dv = p.in + p.lin.vbase(p.v0 + v) + half;
        const int mp = chunk * R1 * B / 2 + pc * ppairs;
        const int ws = max(0, (mp - OFF) & ~1);
        const int len = min(half, (mp + ppairs + NU - OFF + 1) & ~1) - ws;
        double* Cw = Wb + (lp & 1) * 2 * WP;
        mbar_arrive_expect(bar + (lp & 1), (unsigned)(2 * len * 8));
        bulk_g2s(Cw, cv + ws, (unsigned)(len * 8), bar + (lp & 1));
        bulk_g2s(Cw + WP, dv + ws, (unsigned)(len * 8), bar + (lp & 1));
    };
    if (tid == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
    }
    __syncthreads();
    if (tid == 0) {
        issue(0);
        issue(1);
    }
    long long lp = 0;
    for (long long t = blockIdx.x; t < ntask; t += gridDim.x) {
        const int v = (int)(t / nch), chunk = (int)(t % nch);
        const double* cv = p.xi + (long long)v * p.xi_vs;
        const double* dv = p.in + p.lin.vbase(p.v0 + v) + half;
        const long long cbase = (long long)chunk * R1 * B;
        const bool echunk = NU > 1 && (chunk == 0 || cbase + R1 * B >= M);
        const int m0 = (int)(cbase >> 1);
        if (tid == 0) bulk_wait_read();  // the previous task's G store has read the tile
        __syncthreads();
        for (int pc = 0; pc < KP; ++pc, ++lp) {
            const int mp = m0 + pc * ppairs;
            const int ws = max(0, (mp - OFF) & ~1);
            const double* Cw = Wb + (lp & 1) * 2 * WP;
            const double* Dw = Cw + WP;
            mbar_wait(bar + (lp & 1), (unsigned)((lp >> 1) & 1));
            for (int q = tid; q < ppairs; q += NT) {
                const int m = mp + q;
                double o0, o1;
                if (m >= mlo && m < mhi) {
                    const double* cw = Cw + (m - OFF - ws);
                    const double* dw = Dw + (m - OFF - ws);
                    double c[NU + 1], d[NU + 1];
#pragma unroll
                    for (int k = 0; k <= NU; ++k) {
                        c[k] = cw[k];
                        d[k] = dw[k];
                    }
                    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
                    for (int u = -NU + 1; u <= NU; ++u) {
                        if ((u & 1) == 0) {
                            a0 = fma(tp.h[u + NU - 1], c[OFF - u / 2], a0);
                            b0 = fma(tp.g[u + NU - 1], d[OFF - u / 2], b0);
                        } else {
                            a1 = fma(tp.h[u + NU - 1], c[OFF - (u - 1) / 2], a1);
                            b1 = fma(tp.g[u + NU - 1], d[OFF - (u - 1) / 2], b1);
                        }
                    }
                    o0 = a0 + b0;
                    o1 = a1 + b1;
                } else {
                    o0 = idwt_one<NU>(F, cv, dv, M, 2 * m, vmp);
                    o1 = idwt_one<NU>(F, cv, dv, M, 2 * m + 1, vmp);
                }
                const int pos = 2 * m, rl = (pos - (int)cbase) >> kLogB, col = pos & (B - 1);
                double* dst = T + (int)brev_bits((unsigned)rl, kl) * RS + H + col;
                if (echunk && (pos < NU || pos + 1 >= M - NU)) {
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int q2 = pos + e;
                        const double o = e ? o1 : o0;
                        if (q2 < NU || q2 >= M - NU) {
                            p.ev[(long long)v * 2 * NU + (q2 < NU ? q2 : NU + (q2 - (M - NU)))] = o;
                            dst[e] = 0.0;
                        } else {
                            dst[e] = o;
                        }
                    }
                } else {
                    dst[0] = o0;
                    dst[1] = o1;
                }
            }
            __syncthreads();  // buffer lp & 1 is free: refill it with ring piece lp + 2
            if (tid == 0) issue(lp + 2);
        }
        if (H > 0 && tid < 2 * H) {  // outer halos: samples of the neighbouring chunks
            const bool left = tid < H;
            const int c = left ? tid : tid - H;
            const long long pos = left ? cbase - H + c : cbase + (long long)R1 * B + c;
            double* dst = left ? T + c : T + (int)brev_bits((unsigned)(R1 - 1), kl) * RS + B + H + c;
            *dst = (pos >= 0 && pos < M && !(NU > 1 && (pos < NU || pos >= M - NU)))
                       ? idwt_one<NU>(F, cv, dv, M, (int)pos, vmp)
                       : 0.0;
        }
        __syncthreads();
        if (H > 0) {  // inner halos: copies of the neighbouring rows' own columns
            // (thread = (physical row, halo column): consecutive lanes walk consecutive
            // physical rows, whose 36-double stride spreads them over the banks)
            for (int f = tid; f < R1 * 2 * H; f += NT) {
                const int ph = f / (2 * H), c = f % (2 * H);
                const int K = (int)brev_bits((unsigned)ph, kl);  // this row's halos from its neighbours
                if (c < H) {  // right halo: the next row's first columns
                    if (K + 1 < R1) T[ph * RS + B + H + c] = T[(int)brev_bits((unsigned)(K + 1), kl) * RS + H + c];
                } else {      // left halo: the previous row's last columns
                    if (K > 0) T[ph * RS + (c - H)] = T[(int)brev_bits((unsigned)(K - 1), kl) * RS + B + (c - H)];
                }
            }
            __syncthreads();
        }
        tile_hadamard_inl<CW, RS, CWW_CONTIG_MAXR>(T, 1, kl, 0, kl, 0, tid, NT);
        double* g = p.G + (long long)v * A * CW + (long long)chunk * R1 * CW;
        fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
            bulk_s2g(g, T, (unsigned)(R1 * CW * 8));
            bulk_commit();
        }
    }
    if (tid == 0) bulk_wait_read();
}

template <int NU, int NT>
__global__ void __launch_bounds__(NT, 2) k_large_fwd2(LargeArgs p) {
    using Gm = Geo<NU, kLogB>;
    constexpr int B = Gm::B, CW = Gm::CW, RS = Gm::RSL, NP = Gm::NP;
    extern __shared__ double sm[];
    const int tid = threadIdx.x;
    const int j = p.j, M = 1 << j, a = j - kLogB, A = 1 << a, S = 1 << p.q;
    const int kl = p.kl, R1 = 1 << kl, kh = a - kl, R2 = 1 << kh;
    const int NG = p.ng, lng = 31 - __clz(NG);
    const int rho0 = blockIdx.x * NG, v = blockIdx.y;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm);  // G rows landed
    double* ES = sm + 2;            // [S][2NP]
    double* T = ES + S * 2 * NP;    // NG tiles of R2 physical rows (16-byte aligned rows)
    const int tst = R2 * RS;
    const double* g = p.G + (long long)v * A * CW;
    if (tid == 0) mbar_init(bar, 1);
    __syncthreads();
    if (tid == 0) mbar_arrive_expect(bar, (unsigned)(NG * R2 * CW * 8));
    // one bulk copy (TMA engine) per G row: row (khi, rho0 + ng) -> physical row bitrev(khi) of sub-tile ng
    for (int f = tid; f < NG * R2; f += NT) {
        const int ng = f & (NG - 1), khi = f >> lng;  // NG = 2^lng
        const int ph = (int)brev_bits((unsigned)khi, kh);
        bulk_g2s(T + ng * tst + ph * RS, g + ((long long)khi * R1 + rho0 + ng) * CW, (unsigned)(CW * 8), bar);
    }
    if (NU > 1) {
        for (int f = tid; f < S * 2 * NP; f += NT) {
            const double* em = p.tab + p.t.o_em + f * 2 * NU;
            double acc = 0.0;
#pragma unroll
            for (int c = 0; c < 2 * NU; ++c) acc += __ldg(em + c) * p.ev[(long long)v * 2 * NU + c];
            ES[f] = acc;
        }
    }
    mbar_wait(bar, 0);
    __syncthreads();
    tile_hadamard<CW, RS>(T, NG, kh, 0, kh, tst, tid, NT);
    double* ob = p.out + p.lout.vbase(p.v0 + v);
    const int items = NG * R2 * S;
    for (int w = tid; w < items; w += NT) {
        const int wlo = w & (R2 - 1), rest = w >> kh;
        const int s = rest & (S - 1), ng = rest >> p.q;
        const int rho = rho0 + ng;  // = bitrev_kl(N_lo)
        const double sg = ((__popc(wlo) + __popc(rho)) & 1) ? -1.0 : 1.0;
        double z[B];
        row_fwd<NU, kLogB, true>(T + ng * tst + wlo * RS, wlo, p.tab + p.t.o_kap + s, S,
                           NU > 1 ? ES + s * 2 * NP : nullptr, sg, z);
        // g = bitrev_j(N*B + n_lo) = bitrev5(n_lo)*A + bitrev_kl(N_lo)*R2 + bitrev_kh(N_hi)
        // element index gray_inv_hi(nl) ^ rw = (gx ^ rh) * A + (low a bits), with
        // rw = gray_inv(glo) ^ (odd s ? M - 1 : 0): rh = 0 or 31, and the low
        // part rl or rl ^ (A - 1) by the parity of bitrev5(nl) -- two base
        // pointers and a compile-time multiple of +-A per store
        const unsigned glo = ((unsigned)rho << kh) | (unsigned)wlo;
        const unsigned rl = gray_inv(glo) ^ ((s & 1) ? (unsigned)(A - 1) : 0u);
        double* os = ob + (long long)s * M;  // large path: contiguous 1D output
        const int stp = (s & 1) ? -A : A;
        double* pe = os + rl + ((s & 1) ? 31ll * A : 0ll);
        double* po = os + (rl ^ (unsigned)(A - 1)) + ((s & 1) ? 31ll * A : 0ll);
#pragma unroll
        for (int nl = 0; nl < B; ++nl) {
            const unsigned x = brev_c5(nl);
            const int gx = (int)gray_inv_c(x);
            __stcs(((__popc(x) & 1) ? po : pe) + (long long)gx * stp, z[nl]);  // evict-first: streamed out
        }
    }
}

template <int NU, int NT>
__global__ void __launch_bounds__(NT, 2) k_large_adj2(LargeArgs p) {
    using Gm = Geo<NU, kLogB>;
    constexpr int B = Gm::B, CW = Gm::CW, RS = Gm::RSL, NP = Gm::NP;
    extern __shared__ double sm[];
    const int tid = threadIdx.x, lane = tid & 31;
    const int j = p.j, M = 1 << j, a = j - kLogB, A = 1 << a, S = 1 << p.q;
    const int kl = p.kl, R1 = 1 << kl, kh = a - kl, R2 = 1 << kh;
    const int NG = p.ng, lng = 31 - __clz(NG);
    const int rho0 = blockIdx.x * NG, v = blockIdx.y;
    double* T = sm;
    const int tst = R2 * RS;
    const int items = NG * R2;
    const int iters = (items + NT - 1) / NT;
    const int FE = S * 2 * NP;                     // edge sums per vector
    double* red = sm + NG * tst;                   // [NT/32 warps][FE]
    const double* ib = p.in + p.lin.vbase(p.v0 + v);
    for (int it = 0; it < iters; ++it) {
        const int w = tid + it * NT;
        const int wlo = w & (R2 - 1), ng = w >> kh;
        const bool act = w < items;
        const int rho = rho0 + (act ? ng : 0);
        const double sg = ((__popc(wlo) + __popc(rho)) & 1) ? -1.0 : 1.0;
        const unsigned glo = ((unsigned)rho << kh) | (unsigned)wlo;
        const unsigned gi = gray_inv(glo);
        double y[B];
        const Layout lc{0, 0, 0, 1, 62, 62};  // large path: contiguous 1D input
        if (act) {  // block s = 0; later blocks are prefetched by the row stage
            const double *pe, *po;
            long long step;
            seq_ptrs<kLogB>(ib, lc, a, gi, pe, po, step);
#pragma unroll
            for (int nl = 0; nl < B; ++nl) {
                const unsigned x = brev_c(nl, kLogB);
                y[nl] = __ldcs(((__popc(x) & 1) ? po : pe) + (long long)gray_inv_c(x) * step);  // streamed once
            }
        } else {
#pragma unroll
            for (int nl = 0; nl < B; ++nl) y[nl] = 0.0;
        }
        // L2 prefetches (warp 0, one 2^kh-double run per lane and sub-tile) of this
        // CTA's later blocks, p.pfs blocks ahead of the row stage's register loads
        auto pf_block = [&](const double* ibn, int bx, int s2) {
            const unsigned x = brev_bits((unsigned)tid, kLogB);
            const long long gx = (long long)gray_inv(x);
            for (int g2 = 0; g2 < NG; ++g2) {
                const unsigned gl0 = (unsigned)(bx * NG + g2) << kh;
                unsigned rl0 = gray_inv(gl0) & (unsigned)(A - 1);
                if (__popc(x) & 1) rl0 ^= (unsigned)(A - 1);
                long long idx = gx * A + rl0;
                if (s2 & 1) idx ^= (long long)(M - 1);  // odd blocks are mirrored
                // (an 8-byte aligned input: the 16-byte granules from the one holding the run's start)
                l2_prefetch(reinterpret_cast<const void*>(reinterpret_cast<uintptr_t>(
                                ibn + (long long)s2 * M + (idx & ~(long long)(R2 - 1))) & ~uintptr_t(15)),
                            (unsigned)(R2 * 8));
            }
        };
        if (it == 0 && tid < 32) {
            for (int s2 = 1; s2 <= p.pfs && s2 < S; ++s2) pf_block(ib, (int)blockIdx.x, s2);
        }
        for (int s = 0; s < S; ++s) {
            if (it == 0 && tid < 32 && p.pfs > 0 && s > 0 && s + p.pfs < S) pf_block(ib, (int)blockIdx.x, s + p.pfs);
            hadamard_reg<kLogB>(y);
            if (NU > 1) {  // per-warp partial sums, one slot per (CTA, iteration, warp)
                constexpr int R = 2 * NP <= 16 ? 16 : 32;
                double ev[R];
#pragma unroll
                for (int i = 0; i < R; ++i)
                    ev[i] = (act && i < 2 * NP) ? (i < NP ? y[i] : sg * y[B - NP + (i - NP)]) : 0.0;
                if (p.cta_red) {
                    seg_reduce_store<R, 31u, true>(ev, lane, 2 * NP, true, red + (tid >> 5) * FE + s * 2 * NP, it > 0);
                } else {
                    const long long slot = (long long)blockIdx.x * ((NT / 32) * iters) + it * (NT / 32) + (tid >> 5);
                    seg_reduce_store<R, 31u>(ev, lane, 2 * NP, true, p.epw + (((long long)v * p.nslot + slot) * S + s) * 2 * NP);
                }
            }
            if (act) {
                const double *pe = nullptr, *po = nullptr;
                long long step = 0;
                if (s + 1 < S)
                    seq_ptrs<kLogB>(ib + (long long)(s + 1) * M, lc, a, gi ^ (((s + 1) & 1) ? (unsigned)(M - 1) : 0u),
                                    pe, po, step);
                row_adj_accum_pf<NU, kLogB>(T + ng * tst + wlo * RS, p.tab + p.t.o_kap + s, S, y, s == 0, pe, po,
                                            step);
            }
        }
    }
    __syncthreads();
    if (NU > 1 && p.cta_red) {  // one slot per CTA: the warps' sums in a fixed order
        for (int f = tid; f < FE; f += NT) {
            double acc = 0.0;
#pragma unroll
            for (int w = 0; w < NT / 32; ++w) acc += red[w * FE + f];
            p.epw[((long long)v * p.nslot + blockIdx.x) * FE + f] = acc;
        }
    }
    tile_hadamard<CW, RS>(T, NG, kh, 0, kh, tst, tid, NT);
    // physical row ph of sub-tile ng is logical K_hi = bitrev_kh(ph): one bulk
    // store (TMA engine) per G row once the last Hadamard writes are visible
    // to the async proxy
    fence_proxy_async();
    __syncthreads();
    double* g = p.G + (long long)v * A * CW;
    for (int f = tid; f < NG * R2; f += NT) {
        const int ng = f & (NG - 1), khi = f >> lng;  // NG = 2^lng
        bulk_s2g(g + ((long long)khi * R1 + rho0 + ng) * CW, T + ng * tst + (int)brev_bits((unsigned)khi, kh) * RS,
                 (unsigned)(CW * 8));
    }
    bulk_commit();
    bulk_wait_read();
}

template <int NU, int NT>
__global__ void __launch_bounds__(NT, CWW_CONTIG_MINB) k_large_adj1(LargeArgs p) {
    using Gm = Geo<NU, kLogB>;
    // unpadded tile rows (RS = CW): the chunk's G block loads as one 16-byte copy
    constexpr int B = Gm::B, H = Gm::H, CW = Gm::CW, RS = CW, NP = Gm::NP;
    extern __shared__ double sm[];
    const int tid = threadIdx.x;
    const int j = p.j, M = 1 << j, a = j - kLogB, A = 1 << a, S = 1 << p.q;
    const int kl = p.kl, R1 = 1 << kl;
    const int chunk = blockIdx.x, v = blockIdx.y;
    const int FE = S * 2 * NP;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm);  // G block landed
    double* Wv = sm + 2;             // [S][2NP]
    double* nb = Wv + FE;            // [2][H]: neighbour-row halo sums
    double* T = nb + 2 * NU;
    double* red = T + R1 * RS;       // reduction scratch: [NT/32][2H] and [NT/FE][FE]
    const double* g = p.G + (long long)v * A * CW;
    static_assert(CW % 2 == 0, "16-byte bulk G loads");
    if (tid == 0) {  // the chunk's G block: one bulk copy (TMA engine)
        mbar_init(bar, 1);
        mbar_arrive_expect(bar, (unsigned)(R1 * CW * 8));
        bulk_g2s(T, g + (long long)chunk * R1 * CW, (unsigned)(R1 * CW * 8), bar);
        // L2 prefetch of the G block of the CTA that will take this one's place
        const long long lin = (long long)blockIdx.y * gridDim.x + blockIdx.x + p.pfd1;
        if (p.pfd1 > 0 && lin < (long long)gridDim.x * gridDim.y)
            l2_prefetch(p.G + ((lin / gridDim.x) * A + (lin % gridDim.x) * R1) * CW, (unsigned)(R1 * CW * 8));
    }
    // halo contributions from the neighbouring chunks' boundary rows (sums over
    // the physical rows rho of their Hadamard rows; popc is bit-reversal invariant):
    //   previous chunk, last logical row:  sum_rho (-1)^popc(rho) G[(c-1)R1+rho][B+H+k]
    //   next chunk, first logical row:     sum_rho G[(c+1)R1+rho][k]
    // one row per thread, then a fixed-order warp/CTA reduction
    if (NU > 1) {
        double hs[2 * H > 0 ? 2 * H : 1];
        const bool prev = chunk > 0, next = (chunk + 1) * R1 < A;
#pragma unroll
        for (int k = 0; k < H; ++k) {
            double a0 = 0.0, a1 = 0.0;
            for (int nl = tid; nl < R1; nl += NT) {
                if (prev) {
                    const double val = __ldg(g + ((long long)(chunk - 1) * R1 + nl) * CW + B + H + k);
                    a0 += (__popc(nl) & 1) ? -val : val;
                }
                if (next) a1 += __ldg(g + ((long long)(chunk + 1) * R1 + nl) * CW + k);
            }
            hs[k] = a0;
            hs[H + k] = a1;
        }
#pragma unroll
        for (int k = 0; k < 2 * H; ++k)
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) hs[k] += __shfl_xor_sync(0xffffffffu, hs[k], off);
        if ((tid & 31) == 0) {
#pragma unroll
            for (int k = 0; k < 2 * H; ++k) red[(tid >> 5) * 2 * H + k] = hs[k];
        }
    }
    const bool has_edge = NU > 1 && (chunk == 0 || (chunk + 1) * R1 >= A);
    const int nr = FE <= NT ? NT / FE : 1;  // slot lanes per edge sum
    double* red2 = red + (NT / 32) * 2 * NU;  // [nr][FE]
    for (int idx = tid; has_edge && idx < nr * FE; idx += NT) {
        const int f = idx % FE, r = idx / FE;
        const double* e0 = p.epw + (long long)v * p.nslot * FE + f;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        long long sl = r;
        for (; sl + 3 * nr < p.nslot; sl += 4 * nr) {
            a0 += e0[sl * FE];
            a1 += e0[(sl + nr) * FE];
            a2 += e0[(sl + 2 * nr) * FE];
            a3 += e0[(sl + 3 * nr) * FE];
        }
        for (; sl < p.nslot; sl += nr) a0 += e0[sl * FE];
        red2[r * FE + f] = (a0 + a1) + (a2 + a3);
    }
    __syncthreads();    // (also publishes the barrier's initialisation)
    mbar_wait(bar, 0);
    if (NU > 1 && tid < 2 * H) {
        double acc = 0.0;
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) acc += red[w * 2 * H + tid];
        nb[tid] = acc;
    }
    for (int f = tid; has_edge && f < FE; f += NT) {
        double acc = 0.0;
        for (int r = 0; r < nr; ++r) acc += red2[r * FE + f];
        Wv[f] = acc;
    }
    __syncthreads();
    tile_hadamard_inl<CW, RS, CWW_CONTIG_MAXR>(T, 1, kl, 0, kl, 0, tid, NT);
    double* xo = p.xo + (long long)v * p.xo_vs;
    double* ob = p.out + p.lout.vbase(p.v0 + v);
    static_assert(B == 32, "one tile row per warp");
    const int lane = tid & 31;
    // per lane: which halo (if any) it adds, and from which column of the neighbour row
    const int hside = lane < H ? -1 : (lane >= B - H ? 1 : 0);
    const int hcol = lane < H ? B + H + lane : lane - (B - H);
    const double nbv = hside < 0 ? nb[lane] : (hside > 0 ? nb[H + lane - (B - H)] : 0.0);
    const long long base = (long long)chunk * R1 * B;
    const bool fana = p.fuse_ana != 0;
    // xi of the chunk: to the workspace / output, or (fused analysis) in place
    // into the tile's own columns [H, B + H) -- each (row, column) is read and
    // written by one thread only, and the halo columns stay intact
    double* xw = (p.xo_is_output || fana) ? nullptr : xo + base + lane;
    if (!has_edge && (fana || xw)) {
        // interior chunks: the tile's columns [H, B + H) already hold xi except for
        // the 2H columns per row that receive a neighbour row's halo: (row, halo
        // column) per thread, in place (the halo columns themselves are never
        // written); then the fused analysis reads the tile, or a plain coalesced
        // copy sends xi to the workspace
        if (NU > 1) {
            // (consecutive lanes walk consecutive PHYSICAL rows: the row stride of 36
            // doubles spreads them over the banks; logical order would not)
            for (int idx = tid; idx < R1 * 2 * H; idx += NT) {
                const int ph = idx / (2 * H), hh = idx - ph * 2 * H;
                const int r = (int)brev_bits((unsigned)ph, kl);
                const bool left = hh < H;
                const int c = left ? hh : B - 2 * H + hh;  // xi column
                const int rn = left ? r - 1 : r + 1;
                const double add = (rn >= 0 && rn < R1)
                                       ? T[(int)brev_bits((unsigned)rn, kl) * RS + (left ? B + H + c : c - (B - H))]
                                       : nb[hh];
                T[ph * RS + H + c] += add;
            }
        }
        if (!fana) {
            __syncthreads();
#pragma unroll 4
            for (int rl = tid >> 5; rl < R1; rl += NT / 32)
                xw[rl * B] = T[(int)brev_bits((unsigned)rl, kl) * RS + lane + H];
        }
    } else {
        for (int rl = tid >> 5; rl < R1; rl += NT / 32) {  // logical local row K_lo, lane = column
            const int ph = (int)brev_bits((unsigned)rl, kl);
            double val = T[ph * RS + lane + H];
            if (hside != 0) {  // overlap-add of the previous row's right / the next row's left halo
                const int rn = rl + hside;
                val += (rn >= 0 && rn < R1) ? T[(int)brev_bits((unsigned)rn, kl) * RS + hcol] : nbv;
            }
            if (has_edge) {
                const long long pos = base + (long long)rl * B + lane;
                const long long rpos = pos - lane;  // warp-uniform: does this row hold an edge position?
                if ((rpos < NU || rpos + B > M - NU) && (pos < NU || pos >= M - NU)) {
                    const int c = pos < NU ? (int)pos : NU + (int)(pos - (M - NU));
                    const double* em = p.tab + p.t.o_em + c;
                    double e0 = 0.0, e1 = 0.0, e2 = 0.0, e3 = 0.0;
                    const int nsp = S * 2 * NP;
                    int sp = 0;
                    for (; sp + 4 <= nsp; sp += 4) {
                        e0 += __ldg(em + sp * 2 * NU) * Wv[sp];
                        e1 += __ldg(em + (sp + 1) * 2 * NU) * Wv[sp + 1];
                        e2 += __ldg(em + (sp + 2) * 2 * NU) * Wv[sp + 2];
                        e3 += __ldg(em + (sp + 3) * 2 * NU) * Wv[sp + 3];
                    }
                    for (; sp < nsp; ++sp) e0 += __ldg(em + sp * 2 * NU) * Wv[sp];
                    val = (e0 + e1) + (e2 + e3);
                }
            }
            if (fana) T[ph * RS + lane + H] = val;
            else if (xw) xw[rl * B] = val;
            else ob[p.lout.eoff(base + (long long)rl * B + lane)] = val;
        }
    }
    if (!fana) return;
    __syncthreads();
    // finest analysis level (wavelet.cpp:403-445 gather form) from the chunk's xi:
    // c[m] = sum_u hbar_u xi[2m+u], d[m] = sum_u gbar_u xi[2m+u], u = -NU+1..NU;
    // VMP edge rows from the dense edge rows (chunk-local); rows whose window
    // straddles a chunk boundary P (m in [P/2 - FL, P/2 - FL + NS)) get this
    // chunk's partial sums, completed by k_ana_fixup
    {
        constexpr int FL = NU / 2, NS = NU / 2 + NU / 2;  // straddling rows per boundary
        constexpr int EL = FiltSmem<NU>::EL;
        const FiltSmem<NU> F{p.tab + p.t.o_h};
        const Taps<NU> tp(F);
        const bool vmp = p.vmp != 0;
        const int half = M >> 1, CH = R1 * B, nch = M / CH;
        const int m0 = (int)(base >> 1);
        auto xiv = [&](int pos) -> double {  // pos inside this chunk
            const int r = (pos - (int)base) >> kLogB;
            return T[(int)brev_bits((unsigned)r, kl) * RS + H + (pos & (B - 1))];
        };
        const bool lb = !vmp || chunk > 0, rb = !vmp || chunk + 1 < nch;  // boundaries with partials
        const int mlo = m0 + (lb ? NS - FL : 0), mhi = m0 + CH / 2 - (rb ? FL : 0);
        double* cws = xo;  // c_{j-1}
        double* dout = ob + half;
        if (!has_edge) {
            // interior chunks: 16 pairs per tile row, thread = (row, pair t); the
            // window xi[32 r + 2t - H .. + 2nu) is the row's extended columns
            // e = 2t .. 2t + 2nu - 1 (nu aligned 16-byte loads), except e < H
            // (previous row's last columns) and e >= B + H (next row's first)
            static_assert(B == 32, "16 pairs per row");
            const int t = tid & 15;
            const bool lo_x = NU > 1 && 2 * t < H, hi_x = NU > 1 && 2 * t + 2 * NU - 1 >= B + H;
            for (int r = tid >> 4; r < R1; r += NT / 16) {
                const int m = m0 + 16 * r + t;
                const double* row = T + (int)brev_bits((unsigned)r, kl) * RS;
                const double2* rp = reinterpret_cast<const double2*>(row + 2 * t);
                double x[2 * NU];
#pragma unroll
                for (int i = 0; i < NU; ++i) {
                    const double2 pr = rp[i];
                    x[2 * i] = pr.x;
                    x[2 * i + 1] = pr.y;
                }
                if (lo_x && r > 0) {
                    const double* rq = T + (int)brev_bits((unsigned)(r - 1), kl) * RS + B;
#pragma unroll
                    for (int k = 0; k < H; ++k)
                        if (2 * t + k < H) x[k] = rq[2 * t + k];
                }
                if (hi_x && r + 1 < R1) {
                    const double* rq = T + (int)brev_bits((unsigned)(r + 1), kl) * RS - B;
#pragma unroll
                    for (int k = 2 * NU - H; k < 2 * NU; ++k)
                        if (2 * t + k >= B + H) x[k] = rq[2 * t + k];
                }
                double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
                for (int k = 0; k < 2 * NU; k += 2) {
                    a0 = fma(tp.h[k], x[k], a0);
                    b0 = fma(tp.g[k], x[k], b0);
                    a1 = fma(tp.h[k + 1], x[k + 1], a1);
                    b1 = fma(tp.g[k + 1], x[k + 1], b1);
                }
                if (m >= mlo && m < mhi) {
                    cws[m] = a0 + a1;
                    dout[m] = b0 + b1;
                }
            }
        } else
        for (int m = mlo + tid; m < mhi; m += NT) {
            double c, d;
            if (vmp && (m < NU || m >= half - NU)) {
                const int side = m < NU ? 0 : 1;
                const int mm = side ? half - 1 - m : m;
                const double* ra = F.ana(side, 0, mm);
                const double* rb2 = F.ana(side, 1, mm);
                double a0 = 0.0, b0 = 0.0;
#pragma unroll
                for (int k = 0; k < EL; ++k) {
                    const double xv = xiv(side ? M - 1 - k : k);
                    a0 = fma(ra[k], xv, a0);
                    b0 = fma(rb2[k], xv, b0);
                }
                c = a0;
                d = b0;
            } else {
                double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
                for (int u = -NU + 1; u <= NU; ++u) {
                    const double xv = xiv(2 * m + u);
                    if (u & 1) {
                        a1 = fma(tp.h[u + NU - 1], xv, a1);
                        b1 = fma(tp.g[u + NU - 1], xv, b1);
                    } else {
                        a0 = fma(tp.h[u + NU - 1], xv, a0);
                        b0 = fma(tp.g[u + NU - 1], xv, b0);
                    }
                }
                c = a0 + a1;
                d = b0 + b1;
            }
            cws[m] = c;
            dout[m] = d;
        }
        // partial sums of the straddling rows: left boundary (this chunk is its
        // right side) and right boundary (left side); unwrapped positions
        if (tid < 2 * NS) {
            const bool right = tid >= NS;
            const int i = right ? tid - NS : tid;
            if (right ? rb : lb) {
                const int P = (int)base + (right ? CH : 0);
                const int m = P / 2 - FL + i;
                double a0 = 0.0, b0 = 0.0;
#pragma unroll
                for (int u = -NU + 1; u <= NU; ++u) {
                    const int pos = 2 * m + u;
                    if (pos >= (int)base && pos < (int)base + CH) {
                        const double xv = xiv(pos);
                        a0 = fma(tp.h[u + NU - 1], xv, a0);
                        b0 = fma(tp.g[u + NU - 1], xv, b0);
                    }
                }
                const int bidx = right ? (chunk + 1) % nch : chunk;  // boundary at P (P = M wraps to 0)
                double* pp = p.apart + (((long long)v * nch + bidx) * NU + i) * 4 + (right ? 0 : 2);
                pp[0] = a0;
                pp[1] = b0;
            }
        }
    }
}

// Completes the finest-level analysis rows that straddle adjoint pass-1 chunk
// boundaries: one thread per (vector, boundary, row); c / d = left + right
// partial sums (fixed order).  VMP has no boundary at 0 / M.
template <int NU>
__global__ void k_ana_fixup(LargeArgs p) {
    constexpr int FL = NU / 2, NS = NU / 2 + NU / 2;
    const int M = 1 << p.j, half = M >> 1, CH = (1 << p.kl) << kLogB, nch = M / CH;
    const long long tot = p.nvec * nch * NS;
    for (long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x; f < tot; f += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(f % NS);
        const int b = (int)((f / NS) % nch);
        const long long v = f / ((long long)NS * nch);
        if (p.vmp && b == 0) continue;
        const double* pp = p.apart + ((v * nch + b) * NU + i) * 4;
        const int m = (((b * CH) >> 1) - FL + i + half) & (half - 1);
        p.xo[v * p.xo_vs + m] = pp[0] + pp[2];
        (p.out + p.lout.vbase(p.v0 + v))[half + m] = pp[1] + pp[3];
    }
}

}  // namespace cww
