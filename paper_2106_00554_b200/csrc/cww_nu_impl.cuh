// Per-wavelet-order launchers.  Each cww_nu<N>.cu defines CWW_NU and includes
// this file, so the kernel templates for one order compile in their own
// translation unit (parallel build, bounded compile time).
#pragma once
#include "cww_kernels.cuh"
#include "cww_warp.cuh"


#ifndef CWW_NU
#error "define CWW_NU before including cww_nu_impl.cuh"
#endif

#define CWW_CAT2(a, b) a##b
#define CWW_CAT(a, b) CWW_CAT2(a, b)
#define CWW_FN(name) CWW_CAT(name, CWW_NU)

namespace cww {

#define CWW_NT 256

namespace {
constexpr int J0 = CWW_NU == 1 ? 0 : (CWW_NU == 2 ? 2 : (CWW_NU <= 4 ? 3 : 4));

template <int LOGB>
cudaError_t small_t(const SmallArgs& a, bool adj, cudaStream_t st) {
    if constexpr (LOGB < J0) {
        return cudaErrorInvalidValue;  // j >= J0 is validated on the host
    } else {
        int grid = (int)((a.nvec + a.V - 1) / a.V);
        long long smem = small_smem_bytes<CWW_NU, LOGB>(a.V, a.j, a.q, adj, adj ? a.lin.vfast() : a.lout.vfast());
        if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
        if (adj) {
            auto k = k_small_adj<CWW_NU, LOGB, kSmallNT>;
            opt_in_smem(reinterpret_cast<const void*>(k));
            if (cudaError_t e = launch_k(k, grid, kSmallNT, smem, st, a); e != cudaSuccess) return e;
        } else {
            auto k = k_small_fwd<CWW_NU, LOGB, kSmallNT>;
            opt_in_smem(reinterpret_cast<const void*>(k));
            if (cudaError_t e = launch_k(k, grid, kSmallNT, smem, st, a); e != cudaSuccess) return e;
        }
        return cudaGetLastError();
    }
}
}  // namespace

cudaError_t CWW_FN(launch_small_nu)(const SmallArgs& a, bool adj, cudaStream_t st) {
    switch (a.j < kLogB ? a.j : kLogB) {
        case 0: return small_t<0>(a, adj, st);
        case 1: return small_t<1>(a, adj, st);
        case 2: return small_t<2>(a, adj, st);
        case 3: return small_t<3>(a, adj, st);
        case 4: return small_t<4>(a, adj, st);
        default: return small_t<5>(a, adj, st);
    }
}

long long CWW_FN(small_smem_nu)(int V, int j, int q, bool adj, bool vf) {
    switch (j < kLogB ? j : kLogB) {
        case 0: return small_smem_bytes<CWW_NU, 0>(V, j, q, adj, vf);
        case 1: return small_smem_bytes<CWW_NU, 1>(V, j, q, adj, vf);
        case 2: return small_smem_bytes<CWW_NU, 2>(V, j, q, adj, vf);
        case 3: return small_smem_bytes<CWW_NU, 3>(V, j, q, adj, vf);
        case 4: return small_smem_bytes<CWW_NU, 4>(V, j, q, adj, vf);
        default: return small_smem_bytes<CWW_NU, 5>(V, j, q, adj, vf);
    }
}

cudaError_t CWW_FN(launch_wv_nu)(const SmallArgs& a, bool adj, cudaStream_t st) {
    if (a.j != kWvJ) return cudaErrorInvalidValue;
    const int grid = (int)((a.nvec + kWvNT / 32 - 1) / (kWvNT / 32));
    const long long smem = wv_smem_bytes<CWW_NU>(1 << a.q);
    if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    if (adj) {
        auto k = k_wv_adj<CWW_NU>;
        opt_in_smem(reinterpret_cast<const void*>(k));
        if (cudaError_t e = launch_k(k, grid, kWvNT, smem, st, a); e != cudaSuccess) return e;
    } else {
        auto k = k_wv_fwd<CWW_NU>;
        opt_in_smem(reinterpret_cast<const void*>(k));
        if (cudaError_t e = launch_k(k, grid, kWvNT, smem, st, a); e != cudaSuccess) return e;
    }
    return cudaGetLastError();
}

cudaError_t CWW_FN(launch_large_nu)(int which, const LargeArgs& a, cudaStream_t st) {
    using Gm = Geo<CWW_NU, kLogB>;
    const int acnt = a.j - kLogB, kh = acnt - a.kl, R1 = 1 << a.kl, R2 = 1 << kh;
    const int S = 1 << a.q;
    dim3 g1(1u << kh, (unsigned)a.nvec), g2((unsigned)(R1 / a.ng), (unsigned)a.nvec);
    long long s1 = ((long long)R1 * Gm::CW) * 8;  // contiguous passes: unpadded tile rows
    long long s2 = (2 + (long long)a.ng * R2 * Gm::RSL + S * 2 * Gm::NP) * 8;  // + mbarrier
    const long long FE = (long long)S * 2 * Gm::NP;
    long long s1a = s1 + (2 + FE + 2 * CWW_NU + (CWW_NT / 32) * 2 * CWW_NU + (FE > CWW_NT ? FE : CWW_NT)) * 8;
    long long s2a = s2 + (a.cta_red ? (CWW_NT / 32) * FE * 8 : 0);
    switch (which) {
        case 0: {
            if (a.fuse_top)  // + mbarrier + the coarse / detail windows of one piece
                s1 += (2 + 4ll * fuse_window(R1 * (1 << kLogB) / 2 / kFusePieces, CWW_NU)) * 8;  // 2 buffers
            auto k = k_large_fwd1<CWW_NU, CWW_NT>;
            opt_in_smem(reinterpret_cast<const void*>(k));
            if (cudaError_t e = launch_k(k, g1, CWW_NT, s1, st, a); e != cudaSuccess) return e;
            break;
        }
        case 1: {
            auto k = k_large_fwd2<CWW_NU, CWW_NT>;
            opt_in_smem(reinterpret_cast<const void*>(k));
            if (cudaError_t e = launch_k(k, g2, CWW_NT, s2, st, a); e != cudaSuccess) return e;
            break;
        }
        case 2: {
            auto k = k_large_adj2<CWW_NU, CWW_NT>;
            opt_in_smem(reinterpret_cast<const void*>(k));
            if (cudaError_t e = launch_k(k, g2, CWW_NT, s2a, st, a); e != cudaSuccess) return e;
            break;
        }
        case 5: {  // persistent fused forward pass 1: as many CTAs as fit on the device
            s1 += (2 + 4ll * fuse_window(R1 * (1 << kLogB) / 2 / kFusePieces, CWW_NU)) * 8;
            auto k = k_large_fwd1_fz<CWW_NU, CWW_NT>;
            opt_in_smem(reinterpret_cast<const void*>(k));
            int dev = 0, nsm = 0, per = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, CWW_NT, (size_t)s1);
            const long long ntask = (long long)(1 << kh) * a.nvec;
            long long grid = (long long)nsm * (per > 0 ? per : 1);
            if (grid > ntask) grid = ntask;
            if (cudaError_t e = launch_k(k, (int)grid, CWW_NT, s1, st, a); e != cudaSuccess) return e;
            break;
        }
        case 4: {  // straddling finest-level analysis rows (fused adjoint pass 1)
            const long long tot = a.nvec * (R1 ? (1ll << a.j) / ((long long)R1 << kLogB) : 0) * (CWW_NU / 2) * 2;
            if (tot == 0) return cudaSuccess;
            const long long g = (tot + 255) / 256;
            k_ana_fixup<CWW_NU><<<(unsigned)(g < 148 * 8 ? g : 148 * 8), 256, 0, st>>>(a);
            break;
        }
        default: {
            auto k = k_large_adj1<CWW_NU, CWW_NT>;
            opt_in_smem(reinterpret_cast<const void*>(k));
            if (cudaError_t e = launch_k(k, g1, CWW_NT, s1a, st, a); e != cudaSuccess) return e;
            break;
        }
    }
    return cudaGetLastError();
}

cudaError_t CWW_FN(launch_pyr_nu)(bool analysis, const PyrArgs& a, cudaStream_t st) {
    constexpr long long FS = FiltSmem<CWW_NU>::SIZE;
    const int nchunk = 1 << (a.top - a.cb);  // one chunk per warp
    const int nw = nchunk < 8 ? nchunk : 8;
    const dim3 grid((unsigned)(nchunk / nw), (unsigned)a.nvec);
    if (analysis) {
        long long nb = (long long)nw * (64ll + a.wmax + a.wmax2 + 2);
        if (a.tail && nb < (2ll << a.bot) + 2) nb = (2ll << a.bot) + 2;  // + 16-byte phase slack
        const long long smem = (FS + nb) * 8;
        if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
        auto k = k_dwt_wpyr<CWW_NU>;
        opt_in_smem(reinterpret_cast<const void*>(k));
        if (cudaError_t e = launch_k(k, grid, 32 * nw, smem, st, a); e != cudaSuccess) return e;
    } else {
        const long long smem = (FS + (long long)nw * (48ll + a.wmax + a.wmax2 + a.dsum + 2)) * 8;
        if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
        auto k = k_idwt_wpyr<CWW_NU>;
        opt_in_smem(reinterpret_cast<const void*>(k));
        if (cudaError_t e = launch_k(k, grid, 32 * nw, smem, st, a); e != cudaSuccess) return e;
    }
    return cudaGetLastError();
}

cudaError_t CWW_FN(launch_normal_rows_nu)(const NormArgs& a, cudaStream_t st) {
    const long long smem = (FiltSmem<CWW_NU>::SIZE + 2ll * a.E * (4 * CWW_NU - 3) + 3ll * a.V * (1ll << a.j)) * 8;
    if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    const unsigned grid = (unsigned)((a.nvec + a.V - 1) / a.V);
    auto k = k_normal_rows<CWW_NU, 256>;
    opt_in_smem(reinterpret_cast<const void*>(k));
    if (cudaError_t e = launch_k(k, grid, 256, smem, st, a); e != cudaSuccess) return e;
    return cudaGetLastError();
}

namespace {
template <int J, int RNT>
cudaError_t normal_reg_t(const NormArgs& a, cudaStream_t st) {
    constexpr int RLOG = RNT == 512 ? 9 : 8;
    const long long smem = (FiltSmem<CWW_NU>::SIZE + 2ll * a.E * (4 * CWW_NU - 3) +
                            3ll * ((1 << J) + (1 << J) / 32) + 3ll * (1 << RLOG)) * 8;
    auto k = k_normal_rows_reg<CWW_NU, J, RNT>;
    opt_in_smem(reinterpret_cast<const void*>(k));
    if (cudaError_t e = launch_k(k, dim3((unsigned)a.nvec), dim3(RNT), (size_t)smem, st, a); e != cudaSuccess)
        return e;
    return cudaGetLastError();
}
}  // namespace

// register-resident variant: use_idwt, 2^9 <= M <= 2^12, r0 < kRegLog
cudaError_t CWW_FN(launch_normal_rows_reg_nu)(const NormArgs& a, cudaStream_t st) {
    switch (a.j) {
        case 9: return normal_reg_t<9, 256>(a, st);
        case 10: return normal_reg_t<10, 256>(a, st);
        case 11: return normal_reg_t<11, 256>(a, st);
        case 12: return normal_reg_t<12, 256>(a, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t CWW_FN(launch_wav_nu)(const WavArgs& w, cudaStream_t st) {
    const int nt = 256;
    if (w.kind == 0) {
        long long smem = (FiltSmem<CWW_NU>::SIZE + 3 * (1ll << w.lev)) * 8;
        auto k = k_wav_coarse<CWW_NU>;
        opt_in_smem(reinterpret_cast<const void*>(k));
        if (cudaError_t e = launch_k(k, dim3((unsigned)w.nvec), dim3(nt), (size_t)smem, st, w.tab, w.t, w.src, w.ls,
                                     w.sv0, w.src_vs, w.dst, w.ld, w.dv0, w.dst_vs, w.r0, w.lev, w.inverse, w.vmp);
            e != cudaSuccess)
            return e;
    }
    return cudaGetLastError();
}

}  // namespace cww

#ifndef CWW_PHASE_NU
#define CWW_PHASE_NU 4
#endif
#if defined(CWW_PHASE_TIMING) && CWW_NU == CWW_PHASE_NU
extern "C" int cww_debug_phase_read(long long* host, size_t n) {
    return (int)cudaMemcpyFromSymbol(host, cww::cww_phase_buf, n * sizeof(long long));
}
#endif
