// Kernel argument blocks and launcher prototypes shared by cww_host.cpp and
// cww_kernels.cu.  Plain structs passed by value (kernel parameter space).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <set>
#include <utility>
#include <vector>

#include "cww_device.cuh"
#include "../../include/cww_b200.h"

namespace cww {

// Kernel launch through cudaLaunchKernelEx (typed arguments).
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

constexpr int kSmallMaxLog = 12;
constexpr int kRegNT = 256, kRegLog = 8;  // register-resident normal rows: threads, shared-memory levels <= 2^8  // M <= 2^12: whole map in one CTA's shared memory

struct SmallArgs {
    const double* tab;  // per-op device table block
    Tables t;
    const double* in;
    double* out;
    Layout lin, lout;
    long long nvec;  // vectors in this launch
    int V;           // vectors per CTA (power of two)
    int j, q, r0, use_idwt, vmp;
    int in_block;  // 1: a CTA's V input vectors are one contiguous block; 2: an
                   // interleaved [M][V] block (column panel); 0: generic layout
};

// Opts kernel k in to the device's full dynamic shared memory (227 KB minus the
// kernel's static part), once per (kernel, device).  The attribute is per
// kernel and process-wide: setting it to each launch's own footprint would
// race between host threads launching the same kernel with different sizes.
inline cudaError_t opt_in_smem(const void* k) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    if (cudaError_t e = cudaGetDevice(&dev); e != cudaSuccess) return e;
    std::lock_guard<std::mutex> g(mu);
    if (done.count({k, dev})) return cudaSuccess;
    cudaFuncAttributes fa{};
    if (cudaError_t e = cudaFuncGetAttributes(&fa, k); e != cudaSuccess) return e;
    if (cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             227 * 1024 - (int)fa.sharedSizeBytes);
        e != cudaSuccess)
        return e;
    done.insert({k, dev});
    return cudaSuccess;
}

struct LargeArgs {
    const double* tab;
    Tables t;
    int j, q, kl, ng;  // kl: low K bits handled by the contiguous pass; ng: n_lo per CTA
    int r0, use_idwt, vmp;
    long long nvec;
    long long v0;      // global index of the first vector (for the I/O layouts)
    // forward pass 1 source: xi workspace (xi_vs per vector) or the op input
    const double* xi;
    long long xi_vs;
    int xi_is_input;
    // 1: xi holds the level-(j-1) coarse vector and pass 1 synthesises level j
    // itself (details d_{j-1} = in[2^(j-1) : 2^j]), so xi never reaches HBM
    int fuse_top;
    const double* in;
    Layout lin;
    // intermediate G: [nvec][A][CW]; edge values ev: [nvec][2nu]
    double* G;
    double* ev;
    // adjoint edge partial sums: [nvec][nslot][S][2(2nu-1)]
    double* epw;
    long long nslot;
    int cta_red;  // 1: adj2 reduces its warps' edge sums in smem (one slot per CTA)
    // outputs
    double* out;
    Layout lout;
    double* xo;  // adjoint pass-1 destination (workspace) unless xo_is_output
    long long xo_vs;
    int xo_is_output;
    // 1: adjoint pass 1 runs the finest analysis level itself: d_{j-1} to the
    // output, c_{j-1} to xo; the pairs whose filter window straddles a chunk
    // boundary get per-side partial sums apart[nvec][2^kh][NU][2 sides][c, d],
    // summed by launch_ana_fixup
    int fuse_ana;
    double* apart;
    // L2 prefetches: adjoint pass 1 prefetches the G block of the CTA pfd1 linear
    // block indices ahead; adjoint pass 2 its own sequency blocks pfs ahead (0: off)
    int pfd1, pfs;
};

struct WavArgs {
    int kind;  // 0: coarse levels (one CTA per vector, shared memory)
    int V;
    const double* tab;
    Tables t;
    long long nvec;
    int lev;  // level (kind 1/2) or Lc (kind 0)
    int r0, inverse, vmp;
    // coarse: src via ls (inverse) or src + v*src_vs (forward); dst via dst_vs (inverse) or ld
    const double* src;
    Layout ls;
    long long sv0, src_vs;
    double* dst;
    Layout ld;
    long long dv0, dst_vs;
    // level kernels: x/lx (idwt detail source), y/ly (dwt detail sink)
    const double* x;
    Layout lx;
    long long xv0;
    double* y;
    Layout ly;
    long long yv0;
};

// Multilevel wavelet pyramids (large path), one chunk of 2^cb samples of
// level `top` per warp.  Synthesis: levels bot+1..top,
// coarse c_bot from src (or the op input x when src_is_x), details from x, top
// level to out.  Analysis: steps top..bot+1 from src (fine level top), details
// to y, coarse c_bot to cws (or y when cws == nullptr); tail: the last CTA per
// vector runs levels bot..r0+1 (cnt: one zeroed ticket per vector).
struct PyrArgs {
    const double* tab;
    Tables t;
    long long nvec;
    int vmp, top, bot, cb, r0, tail;
    int wmax;  // window buffer length (doubles), from pyr_wmax_*: the larger ping-pong slot
    int wmax2; // the other ping-pong slot (levels alternate: about half of wmax)
    int dsum;  // synthesis: total detail-window length over all levels
    const double* x;
    Layout lx;
    long long xv0;
    const double* src;
    long long src_vs;
    int src_is_x;
    double* out;
    long long out_vs;
    double* y;
    Layout ly;
    long long yv0;
    double* cws;
    long long cws_vs;
    unsigned* cnt;
    int pfd;  // L2 prefetch distance in CTAs (0: off)
};

cudaError_t launch_pyr(int nu, bool analysis, const PyrArgs& a, cudaStream_t st);

// Normal form of the full-mask operator along one axis (SURVEY.md 8d "K10
// normal-op form"): U* U = sum_s (D_s + E_s)^T H^T H (D_s + E_s) and H^T H =
// M I, so U* U is a symmetric BANDED matrix G (half-bandwidth b = 2nu - 2,
// wrapping for periodic boundaries).  N1 = W G W^-1 for the ComposedOp.
// band: rows [0, E) gL[E][2b+1], rows [M-E, M) gR[E][2b+1], other rows the
// Toeplitz row gI[2b+1]; entry d of row i multiplies x[i + d - b].
struct NormArgs {
    const double* tab;
    Tables t;
    const double* band;  // gL | gR | gI
    int E, b;
    const double* in;
    double* out;
    long long in_vs, out_vs, nvec;
    int j, r0, use_idwt, vmp, V;
    // register kernel only: vector v starts at (v / vpi) * ivs + (v % vpi) * vs and
    // its elements are es apart (columns of row-major images: vpi = M, ivs = M^2,
    // vs = 1, es = M); es = 0 means the contiguous layout above
    long long vpi, ivs, es;
    int pfd;  // register kernel, contiguous rows: L2 prefetch of the row pfd CTAs ahead (0: off)
};
cudaError_t launch_normal_rows(int nu, const NormArgs& a, cudaStream_t st);
// fp32 I/O conversions (grid-stride)
cudaError_t launch_convert_f32_f64(const float* in, double* out, long long n, cudaStream_t st);
cudaError_t launch_convert_f64_f32(const double* in, float* out, long long n, cudaStream_t st);
// record an error message for cww_last_error() (host translation units)
cww_status set_error(cww_status st, const char* msg);
// add n kernel launches to cww_kernel_launches() (host translation units)
void note_launches(int n);
// distributed transpose: x[i][r*m + k] = recv[r][i][k] (P blocks of m x m, rows of M = P*m)
cudaError_t launch_unpack_blocks(const double* recv, double* x, long long m, int P, cudaStream_t st);
// the register-resident kernel serves this shape (strided layouts need it)
bool normal_reg_ok(int nu, int j, int r0, int use_idwt);
// Batched out-of-place transpose of n x n fp64 matrices (matrix stride n*n).
cudaError_t launch_transpose(const double* in, double* out, long long n, long long batch, cudaStream_t st);
// Batched out-of-place transpose of rows x cols matrices (out: cols x rows).
cudaError_t launch_transpose_rect(const double* in, double* out, long long rows, long long cols, long long batch,
                                  cudaStream_t st);

// Largest window (over all CTAs and levels) of a synthesis pyramid producing
// chunks of 2^cb samples of level top from level bot.
// Also returns the largest total detail-window length of one CTA (dsum) and,
// in *wm2, the largest window of the other ping-pong slot: level lev's window
// lives in slot (top-1-lev) & 1 (slot 0 = the level top-1 window, the largest).
inline int pyr_wmax_syn(int nu, int top, int bot, int cb, bool vmp, int* dsum, int* wm2 = nullptr) {
    int wm[2] = {1, 1}, ds = 1;
    for (long long c = 0; c < (1ll << (top - cb)); ++c) {
        Win f{int(c << cb), int((c + 1) << cb)};
        int sum = 0;
        for (int lev = top; lev > bot; --lev) {
            f = syn_need(nu, 1 << lev, f, vmp);  // window of level lev-1
            const int slot = (top - lev) & 1;
            if (f.hi - f.lo > wm[slot]) wm[slot] = f.hi - f.lo;
            sum += f.hi - f.lo;
        }
        if (sum > ds) ds = sum;
    }
    *dsum = ds;
    if (wm2) {
        *wm2 = wm[1];
        return wm[0];
    }
    return wm[0] > wm[1] ? wm[0] : wm[1];
}

// Same for an analysis pyramid (steps top..bot+1, chunks of 2^cb at level top);
// the input window of step s lives in slot (top - s) & 1, *wm2 = slot 1's max.
inline int pyr_wmax_ana(int nu, int top, int bot, int cb, bool vmp, int* wm2 = nullptr) {
    int wm[2] = {1, 1};
    const int lnc = top - cb;
    for (long long c = 0; c < (1ll << lnc); ++c) {
        Win r{int(c << (bot - lnc)), int((c + 1) << (bot - lnc))};
        for (int s = bot + 1; s <= top; ++s) {
            r = ana_need(nu, 1 << s, r, vmp);  // input window of step s
            const int slot = (top - s) & 1;
            if (r.hi - r.lo > wm[slot]) wm[slot] = r.hi - r.lo;
        }
    }
    if (wm2) {
        *wm2 = wm[1];
        return wm[0];
    }
    return wm[0] > wm[1] ? wm[0] : wm[1];
}
cudaError_t launch_small(int nu, const SmallArgs& a, bool adj, cudaStream_t st);
// warp-per-vector kernels for M = 2^10 (cww_warp.cuh)
cudaError_t launch_wv(int nu, const SmallArgs& a, bool adj, cudaStream_t st);
long long small_smem_query(int nu, int V, int j, int q, bool adj, bool vf);
cudaError_t launch_large(int nu, int which, const LargeArgs& a, cudaStream_t st);
// finest-level analysis pairs straddling adjoint pass-1 chunk boundaries: c / d = left + right partials
cudaError_t launch_ana_fixup(int nu, const LargeArgs& a, cudaStream_t st);
long long large_nslot(int nu, int q, int j, int kl, int ng);
// adj2 keeps per-warp edge sums in smem when they are small (<= 256 values)
inline bool large_cta_red(int nu, int q) { return (2 * (2 * nu - 1)) << q <= 256; }
cudaError_t launch_wav(int nu, const WavArgs& w, cudaStream_t st);
cudaError_t launch_fwht(double* v, int bits, long long batch, int sequency, double* scratch,
                        cudaStream_t st);
cudaError_t launch_seq_perm(uint32_t* perm, int bits, cudaStream_t st);
// GPU kernel-table cascades (cww_ktable.cu): interior levels 0..R of phi, and
// the nu boundary functions from their start values cur0.
cudaError_t cascade_gpu(const std::vector<double>& h, const std::vector<double>& phi, int nu, int R,
                        std::vector<std::vector<double>>& lev);
cudaError_t cascade_edges_gpu(const std::vector<std::vector<double>>& cur0,
                              const std::vector<std::vector<double>>& lev, const std::vector<double>& A,
                              const std::vector<double>& B, int nu, int R, std::vector<std::vector<double>>& out);
// CGLS vector algebra (cww_solver.cu)
int dot_nblk(long long n, long long batch);
cudaError_t launch_dot(const double* a, const double* b, long long n, long long batch, double* part,
                       double* out, cudaStream_t st);
cudaError_t launch_cgls_xr(double* x, double* r, const double* p, const double* q, long long nx, long long nr,
                           long long batch, const double* gam, const double* qq, const int* active,
                           cudaStream_t st);
cudaError_t launch_cgls_p(double* p, const double* s, long long nx, long long batch, const double* gnew,
                          const double* gold, cudaStream_t st);
cudaError_t launch_cgls_flags(const double* gam, const double* s0, double tol, int* active, long long batch,
                              cudaStream_t st);
cudaError_t launch_sqrt(const double* a, double* out, long long batch, cudaStream_t st);
cudaError_t launch_sub_from(double* r, const double* y, long long n, cudaStream_t st);
// Chambolle-Pock vector algebra (cs_solve): dual prox (tt: per-system ||t||^2),
// primal soft-threshold step, s = a - b
cudaError_t launch_cp_dual(double* xi, const double* w, const double* y, double sigma, double sqrt_eta,
                           long long nr, long long batch, double* part, double* tt, cudaStream_t st);
cudaError_t launch_cp_primal(double* z, double* zbar, double* s, double tau, long long n, cudaStream_t st);
cudaError_t launch_sub(double* s, const double* a, const double* b, long long n, cudaStream_t st);
// Sampling-mask epilogues: gather y[b][i] = full[b][idx[i]] (scatter = false) or
// scatter full[b][idx[i]] = y[b][i] (scatter = true; full pre-zeroed).
cudaError_t launch_mask(double* full, long long nfull, const uint64_t* idx, long long cnt, double* y,
                        long long batch, bool scatter, cudaStream_t st);
cudaError_t launch_sign_rows(const uint64_t* pos, long long npos, int j, double* out,
                             cudaStream_t st);

}  // namespace cww
