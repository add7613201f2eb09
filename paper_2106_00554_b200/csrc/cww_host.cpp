// Host side of the B200 operator: spec validation, CWWF filter loading, the
// Walsh-coefficient (kernel) table, edge-term tables, the per-op device table
// block, call orchestration and the extern "C" ABI declared in
// include/cww_b200.h.
//
// Reference correspondence (paths under /root/reference/proj):
//   WaveletSpec::min_level / validate        src/wavelet.cpp:16-39
//   load_filters (CWWF + CRC32)              src/wavelet.cpp:123-186, include/cww/crc32.hpp
//   cascade / refine / left-edge cascade     src/wavelet.cpp:192-311
//   cell_masses / compute_kernel_table       src/kernel.cpp:14-77
//   FastOp ctor checks, build_edge_terms     src/fastop.cpp:27-98
//   FastOp / ComposedOp forward & adjoint    src/fastop.cpp:100-281 (run on the GPU here)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <atomic>
#include <map>
#include <string>
#include <vector>

#include "../../include/cww_b200.h"
#include "cww_launch.h"

using cww::Layout;

namespace {

thread_local std::string g_err;

cww_status fail(cww_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

#define CUDA_TRY(expr)                                                                 \
    do {                                                                               \
        cudaError_t e_ = (expr);                                                       \
        if (e_ != cudaSuccess) return fail(CWW_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
    } while (0)

// ---------------------------------------------------------------------------
// filters
// ---------------------------------------------------------------------------
struct Filters {
    int family = 0, nu = 1;
    std::vector<double> h, g, phi;         // 2nu each
    std::vector<double> E[2], A[2], B[2], Aw[2], Bw[2];  // [0] left, [1] right
};

uint32_t crc32_zlib(const unsigned char* p, size_t n) {
    static uint32_t table[256];
    static std::once_flag once;
    std::call_once(once, [] {
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
            table[i] = c;
        }
    });
    uint32_t c = 0xFFFFFFFFu;
    for (size_t i = 0; i < n; ++i) c = table[(c ^ p[i]) & 0xFFu] ^ (c >> 8);
    return c ^ 0xFFFFFFFFu;
}

int spec_min_level(int nu) {
    if (nu == 1) return 0;
    int j = 0;
    while ((1 << j) < 2 * nu) ++j;
    return j;
}

std::string default_data_dir();

cww_status load_filters(int family, int nu, const char* dir_in, Filters& f) {
    f = Filters{};
    f.family = family;
    f.nu = nu;
    if (nu == 1) {  // Haar, built in
        double s = 1.0 / std::sqrt(2.0);
        f.h = {s, s};
        f.g = {s, -s};
        f.phi = {1.0, 0.0};
        return CWW_OK;
    }
    std::string dir = (dir_in && *dir_in) ? dir_in : default_data_dir();
    std::string path = dir + "/" + (family == 0 ? "db" : "sym") + std::to_string(nu) + ".cwwf";
    FILE* fp = std::fopen(path.c_str(), "rb");
    if (!fp) return fail(CWW_ERR_DATA_IO, "cannot open filter data file: %s", path.c_str());
    std::vector<unsigned char> b;
    unsigned char buf[4096];
    size_t got;
    while ((got = std::fread(buf, 1, sizeof buf, fp)) > 0) b.insert(b.end(), buf, buf + got);
    std::fclose(fp);
    if (b.size() < 20) return fail(CWW_ERR_DATA_IO, "truncated filter data file: %s", path.c_str());
    uint32_t stored;
    std::memcpy(&stored, b.data() + b.size() - 4, 4);
    if (crc32_zlib(b.data(), b.size() - 4) != stored)
        return fail(CWW_ERR_DATA_IO, "checksum failure in filter data file: %s", path.c_str());
    if (std::memcmp(b.data(), "CWWF", 4) != 0)
        return fail(CWW_ERR_DATA_IO, "bad magic in filter data file: %s", path.c_str());
    size_t pos = 4, end = b.size() - 4;
    auto u32 = [&](uint32_t& v) {
        if (pos + 4 > end) return false;
        std::memcpy(&v, b.data() + pos, 4);
        pos += 4;
        return true;
    };
    auto mat = [&](uint32_t rows, uint32_t cols, std::vector<double>& dst) {
        uint32_t r, c;
        if (!u32(r) || !u32(c) || r != rows || c != cols) return false;
        size_t n = size_t(r) * c;
        if (pos + 8 * n > end) return false;
        dst.resize(n);
        std::memcpy(dst.data(), b.data() + pos, 8 * n);
        pos += 8 * n;
        return true;
    };
    uint32_t ver, fam, fnu, nmat;
    if (!u32(ver) || !u32(fam) || !u32(fnu) || !u32(nmat))
        return fail(CWW_ERR_DATA_IO, "truncated filter data file: %s", path.c_str());
    if (ver != 1) return fail(CWW_ERR_DATA_IO, "unsupported filter data version in %s", path.c_str());
    if (fam != uint32_t(family) || fnu != uint32_t(nu))
        return fail(CWW_ERR_DATA_IO, "filter data header does not match requested wavelet: %s", path.c_str());
    if (nmat != 13) return fail(CWW_ERR_DATA_IO, "unexpected matrix count in %s", path.c_str());
    uint32_t L = 2 * nu, W = L - 1, V = nu;
    bool ok = mat(1, L, f.h) && mat(1, L, f.g) && mat(1, L, f.phi);
    for (int e = 0; e < 2 && ok; ++e)
        ok = mat(V, W, f.E[e]) && mat(V, V, f.A[e]) && mat(V, W, f.B[e]) && mat(V, V, f.Aw[e]) &&
             mat(V, W, f.Bw[e]);
    if (!ok) return fail(CWW_ERR_DATA_IO, "filter data shape mismatch or truncation in %s", path.c_str());
    double s = 0;
    for (double x : f.h) s += x;
    if (std::fabs(s - std::sqrt(2.0)) > 1e-10)
        return fail(CWW_ERR_DATA_IO, "corrupt filter data (lowpass sum != sqrt2): %s", path.c_str());
    return CWW_OK;
}

// ---------------------------------------------------------------------------
// cascade and kernel table (host precompute, untimed; the cascade optionally
// on the GPU, bit-identical: cww_ktable.cu)
// ---------------------------------------------------------------------------
thread_local bool g_gpu_cascade = false;
struct Samples {
    std::vector<double> v;
    long left = 0;  // support_left (integer)
    int R = 0;
    double at(long g) const {
        long i = g - left * (1l << R);
        return (i < 0 || i >= long(v.size())) ? 0.0 : v[size_t(i)];
    }
};

// phi(x) = sqrt2 sum_u h_u phi(2x-u) on the 2^-r grid over [a, b]
std::vector<double> refine(const std::vector<double>& prev, int r, int a, int b,
                           const std::vector<double>& h, int nu) {
    long n = long(b - a) * (1l << r) + 1, half = 1l << (r - 1), lo = long(a) * half;
    std::vector<double> cur(size_t(n), 0.0);
    const double s2 = std::sqrt(2.0);
    for (long t = 0; t < n; ++t) {
        long x2 = long(a) * (1l << r) + t;  // 2x on the (r-1) grid
        double acc = 0.0;
        for (int u = -nu + 1; u <= nu; ++u) {
            long i = x2 - u * half - lo;
            if (i >= 0 && i < long(prev.size())) acc += h[size_t(u + nu - 1)] * prev[size_t(i)];
        }
        cur[size_t(t)] = s2 * acc;
    }
    return cur;
}

// left-edge functions 0..nu-1 in construction coordinates (support [0, nu+m])
std::vector<std::vector<double>> cascade_edges(const std::vector<double>& h,
                                               const std::vector<double>& phi,
                                               const std::vector<double>& E,
                                               const std::vector<double>& A,
                                               const std::vector<double>& B, int nu, int R) {
    const int a = -nu + 1, W = 2 * nu - 1;
    std::vector<std::vector<double>> lev(static_cast<size_t>(R) + 1);
    if (g_gpu_cascade) {
        if (cww::cascade_gpu(h, phi, nu, R, lev) != cudaSuccess) return {};
    } else {
        lev[0] = phi;
        for (int r = 1; r <= R; ++r) lev[size_t(r)] = refine(lev[size_t(r - 1)], r, a, nu, h, nu);
    }
    std::vector<std::vector<double>> cur(static_cast<size_t>(nu));
    for (int m = 0; m < nu; ++m) {
        cur[size_t(m)].assign(size_t(nu + m + 1), 0.0);
        for (long k = 0; k <= nu + m; ++k) {
            double acc = 0.0;
            for (int i = 0; i < W; ++i) {
                long arg = k - (-nu + 1 + i);
                if (arg > -nu && arg < nu) acc += E[size_t(m * W + i)] * phi[size_t(arg + nu - 1)];
            }
            cur[size_t(m)][size_t(k)] = acc;
        }
    }
    if (g_gpu_cascade) {
        std::vector<std::vector<double>> out;
        if (cww::cascade_edges_gpu(cur, lev, A, B, nu, R, out) != cudaSuccess) return {};
        return out;
    }
    const double s2 = std::sqrt(2.0);
    for (int r = 1; r <= R; ++r) {
        std::vector<std::vector<double>> nxt(static_cast<size_t>(nu));
        const auto& il = lev[size_t(r - 1)];
        for (int m = 0; m < nu; ++m) {
            long n = long(nu + m) * (1l << r) + 1;
            nxt[size_t(m)].assign(size_t(n), 0.0);
            for (long t = 0; t < n; ++t) {
                double acc = 0.0;
                for (int k = 0; k < nu; ++k)
                    if (t < long(cur[size_t(k)].size())) acc += A[size_t(m * nu + k)] * cur[size_t(k)][size_t(t)];
                for (int li = 0; li <= 2 * m; ++li) {
                    long idx = t - long(nu + li) * (1l << (r - 1)) - long(a) * (1l << (r - 1));
                    double iv = (idx >= 0 && idx < long(il.size())) ? il[size_t(idx)] : 0.0;
                    acc += B[size_t(m * W + li)] * iv;
                }
                nxt[size_t(m)][size_t(t)] = s2 * acc;
            }
        }
        cur.swap(nxt);
    }
    return cur;
}

void fwht_seq_host(std::vector<double>& v) {
    size_t n = v.size();
    for (size_t h = 1; h < n; h <<= 1)
        for (size_t i = 0; i < n; i += 2 * h)
            for (size_t k = i; k < i + h; ++k) {
                double a = v[k], b = v[k + h];
                v[k] = a + b;
                v[k + h] = a - b;
            }
    unsigned bits = 0;
    while ((size_t(1) << bits) < n) ++bits;
    std::vector<double> t(v);
    for (size_t i = 0; i < n; ++i) {
        size_t g = i ^ (i >> 1), r = 0;
        for (unsigned b = 0; b < bits; ++b) r |= ((g >> b) & 1u) << (bits - 1 - b);
        v[i] = t[r];
    }
}

std::vector<double> cell_masses(const Samples& s, long x0, int q) {
    const int R = s.R;
    size_t cells = size_t(1) << q;
    long per = 1l << (R - q);
    double h = std::ldexp(1.0, -R);
    std::vector<double> out(cells, 0.0);
    long base = x0 * (1l << R);
    for (size_t c = 0; c < cells; ++c) {
        long st = base + long(c) * per;
        double acc = 0.5 * (s.at(st) + s.at(st + per));
        for (long i = 1; i < per; ++i) acc += s.at(st + i);
        out[c] = acc * h;
    }
    return out;
}

struct KernelTable {
    std::vector<double> interior, left, right;
};

cww_status kernel_table(const Filters& f, int vmp, int q, int R, KernelTable& t) {
    const int nu = f.nu, W = 2 * nu - 1;
    const size_t S = size_t(1) << q;
    if (R < q) return fail(CWW_ERR_SPEC, "kernel quadrature requires R >= q");
    t.interior.assign(size_t(W) * S, 0.0);
    if (nu == 1) {  // Haar: kappa_0(s) = delta_{s0} exactly
        t.interior[0] = 1.0;
        return CWW_OK;
    }
    Samples in;
    in.R = R;
    in.left = -nu + 1;
    if (g_gpu_cascade) {
        std::vector<std::vector<double>> lev;
        if (cww::cascade_gpu(f.h, f.phi, nu, R, lev) != cudaSuccess)
            return fail(CWW_ERR_CUDA, "GPU kernel-table cascade failed");
        in.v = std::move(lev[size_t(R)]);
    } else {
        in.v = f.phi;
        for (int r = 1; r <= R; ++r) in.v = refine(in.v, r, -nu + 1, nu, f.h, nu);
    }
    for (int l = -nu + 1; l <= nu - 1; ++l) {
        auto m = cell_masses(in, l, q);
        fwht_seq_host(m);
        std::copy(m.begin(), m.end(), t.interior.begin() + long(l + nu - 1) * long(S));
    }
    if (!vmp) return CWW_OK;
    t.left.assign(size_t(nu * W) * S, 0.0);
    t.right.assign(size_t(nu * W) * S, 0.0);
    auto L = cascade_edges(f.h, f.phi, f.E[0], f.A[0], f.B[0], nu, R);
    std::vector<double> hr(f.h.rbegin(), f.h.rend()), pr(f.phi.rbegin(), f.phi.rend());
    auto Rt = cascade_edges(hr, pr, f.E[1], f.A[1], f.B[1], nu, R);
    if (L.size() != size_t(nu) || Rt.size() != size_t(nu))
        return fail(CWW_ERR_CUDA, "GPU kernel-table edge cascade failed");
    for (int m = 0; m < nu; ++m) {
        Samples sl;
        sl.R = R;
        sl.left = 0;
        sl.v = L[size_t(m)];
        Samples sr;
        sr.R = R;
        sr.left = -(nu + m);
        sr.v.assign(Rt[size_t(m)].rbegin(), Rt[size_t(m)].rend());
        for (int l = 0; l <= nu - 1 + m; ++l) {
            auto ms = cell_masses(sl, l, q);
            fwht_seq_host(ms);
            std::copy(ms.begin(), ms.end(), t.left.begin() + long(m * W + l) * long(S));
        }
        for (int tt = 0; tt <= nu + m - 1; ++tt) {
            auto ms = cell_masses(sr, tt - (nu + m), q);
            fwht_seq_host(ms);
            std::copy(ms.begin(), ms.end(), t.right.begin() + long(m * W + tt) * long(S));
        }
    }
    return CWW_OK;
}

// ---- kernel-table cache: CWWK files (kernel.cpp:79-198) --------------------
// "CWWK" | u32 version (1) | u32 family | u32 nu | u32 boundary | u32 q | u32 R
// | 3 x (u32 count, count f64: interior, left, right) | u32 CRC-32 of all
// preceding bytes; little-endian, as the reference writes it.
constexpr uint32_t kCwwkVersion = 1;

struct CwwkHeader {
    int family = 0, nu = 0, vmp = 0, q = 0, R = 0;
};

std::string cwwk_filename(int family, int nu, int vmp, int q, int R) {
    return std::string("cwwk_") + (family == 0 ? "db" : "sym") + std::to_string(nu) + "_" +
           (vmp ? "vmp" : "periodic") + "_q" + std::to_string(q) + "_R" + std::to_string(R) + "_v" +
           std::to_string(kCwwkVersion) + ".bin";
}

cww_status cwwk_save(const KernelTable& t, const CwwkHeader& h, const std::string& path) {
    std::vector<unsigned char> b;
    auto put = [&](const void* p, size_t n) {
        const auto* c = static_cast<const unsigned char*>(p);
        b.insert(b.end(), c, c + n);
    };
    auto u32 = [&](uint32_t v) { put(&v, 4); };
    auto arr = [&](const std::vector<double>& a) {
        u32(uint32_t(a.size()));
        put(a.data(), a.size() * 8);
    };
    put("CWWK", 4);
    u32(kCwwkVersion);
    u32(uint32_t(h.family));
    u32(uint32_t(h.nu));
    u32(uint32_t(h.vmp));
    u32(uint32_t(h.q));
    u32(uint32_t(h.R));
    arr(t.interior);
    arr(t.left);
    arr(t.right);
    const uint32_t crc = crc32_zlib(b.data(), b.size());
    u32(crc);
    FILE* fp = std::fopen(path.c_str(), "wb");
    if (!fp) return fail(CWW_ERR_DATA_IO, "cannot write kernel cache: %s", path.c_str());
    const size_t w = std::fwrite(b.data(), 1, b.size(), fp);
    const int c = std::fclose(fp);
    if (w != b.size() || c != 0) return fail(CWW_ERR_DATA_IO, "short write to kernel cache: %s", path.c_str());
    return CWW_OK;
}

cww_status cwwk_load(const std::string& path, KernelTable& t, CwwkHeader& h) {
    FILE* fp = std::fopen(path.c_str(), "rb");
    if (!fp) return fail(CWW_ERR_DATA_IO, "cannot open kernel cache: %s", path.c_str());
    std::vector<unsigned char> b;
    unsigned char buf[4096];
    size_t got;
    while ((got = std::fread(buf, 1, sizeof buf, fp)) > 0) b.insert(b.end(), buf, buf + got);
    std::fclose(fp);
    if (b.size() < 32) return fail(CWW_ERR_DATA_IO, "truncated kernel cache: %s", path.c_str());
    uint32_t stored;
    std::memcpy(&stored, b.data() + b.size() - 4, 4);
    if (crc32_zlib(b.data(), b.size() - 4) != stored)
        return fail(CWW_ERR_DATA_IO, "checksum failure in kernel cache: %s", path.c_str());
    if (std::memcmp(b.data(), "CWWK", 4) != 0)
        return fail(CWW_ERR_DATA_IO, "bad magic in kernel cache: %s", path.c_str());
    size_t pos = 4;
    const size_t end = b.size() - 4;
    auto u32 = [&]() {
        uint32_t v = 0;
        if (pos + 4 <= end) std::memcpy(&v, b.data() + pos, 4);
        pos += 4;
        return v;
    };
    if (u32() != kCwwkVersion) return fail(CWW_ERR_DATA_IO, "kernel cache version mismatch: %s", path.c_str());
    h.family = int(u32());
    h.nu = int(u32());
    h.vmp = int(u32());
    h.q = int(u32());
    h.R = int(u32());
    auto arr = [&](std::vector<double>& a) {
        const uint32_t n = u32();
        if (pos > end || pos + size_t(n) * 8 > end) return false;
        a.resize(n);
        std::memcpy(a.data(), b.data() + pos, size_t(n) * 8);
        pos += size_t(n) * 8;
        return true;
    };
    if (!arr(t.interior) || !arr(t.left) || !arr(t.right))
        return fail(CWW_ERR_DATA_IO, "truncated kernel cache payload: %s", path.c_str());
    if (h.nu < 1 || h.nu > 6 || h.q < 0 || h.q > 20)
        return fail(CWW_ERR_DATA_IO, "kernel cache shape mismatch (header): %s", path.c_str());
    const size_t W = size_t(2 * h.nu - 1), S = size_t(1) << h.q;
    if (t.interior.size() != W * S)
        return fail(CWW_ERR_DATA_IO, "kernel cache shape mismatch (interior): %s", path.c_str());
    const size_t edge = h.vmp ? size_t(h.nu) * W * S : 0;
    if (t.left.size() != edge || t.right.size() != edge)
        return fail(CWW_ERR_DATA_IO, "kernel cache shape mismatch (edge): %s", path.c_str());
    return CWW_OK;
}

// get_kernel_table (kernel.cpp:173-198): a valid, matching cache file is
// used; a missing / corrupt one is recomputed silently, a stale one with a
// note; the computed table is written back (failures noted, not fatal).
cww_status cached_kernel_table(const Filters& f, int family, int vmp, int q, int R, const std::string& dir,
                               KernelTable& t) {
    std::string path;
    if (!dir.empty()) {
        path = dir + "/" + cwwk_filename(family, f.nu, vmp, q, R);
        KernelTable c;
        CwwkHeader h;
        const std::string saved = g_err;
        if (cwwk_load(path, c, h) == CWW_OK) {
            if (h.family == family && h.nu == f.nu && h.vmp == vmp && h.q == q && h.R == R) {
                t = std::move(c);
                return CWW_OK;
            }
            std::fprintf(stderr, "cww: stale kernel cache %s, recomputing\n", path.c_str());
        }
        g_err = saved;
    }
    cww_status s = kernel_table(f, vmp, q, R, t);
    if (s != CWW_OK || path.empty()) return s;
    CwwkHeader h{family, f.nu, vmp, q, R};
    const std::string saved = g_err;
    if (cwwk_save(t, h, path) != CWW_OK) {
        std::fprintf(stderr, "cww: %s (continuing without cache)\n", g_err.c_str());
        g_err = saved;
    }
    return CWW_OK;
}

std::string cache_dir_of(const char* flag) {  // resolve_cache_dir (kernel.cpp:167-171)
    if (flag && *flag) return flag;
    if (const char* e = std::getenv("CWW_CACHE_DIR"); e && *e) return e;
    return "";
}

std::string default_data_dir() {
    if (const char* e = std::getenv("CWW_DATA_DIR"); e && *e) return e;
#ifdef CWW_DEFAULT_DATA_DIR
    return CWW_DEFAULT_DATA_DIR;
#else
    return "data";
#endif
}

// ---- launch instrumentation ------------------------------------------------
std::atomic<unsigned long long> g_launches{0};
std::atomic<int> g_prof_on{0};
struct ProfRec {
    const char* name;
    cudaEvent_t a, b;
};
std::mutex g_prof_mu;
std::vector<ProfRec> g_prof;

struct Prof {  // RAII bracket around one launcher call
    const char* name;
    cudaStream_t st;
    cudaEvent_t a = nullptr, b = nullptr;
    int kernels;
    Prof(const char* n, cudaStream_t s, int k = 1) : name(n), st(s), kernels(k) {
        if (g_prof_on.load()) {
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a, st);
        }
    }
    ~Prof() {
        g_launches += (unsigned long long)kernels;
        if (a) {
            cudaEventRecord(b, st);
            std::lock_guard<std::mutex> lk(g_prof_mu);
            g_prof.push_back({name, a, b});
        }
    }
};

// One VMP synthesis level (wavelet.cpp:447-483 semantics), used only to
// extract the level-independent edge blocks below.
std::vector<double> level_inverse_vmp_host(const Filters& f, const std::vector<double>& x) {
    const size_t n = x.size(), half = n / 2, NV = size_t(f.nu);
    const int nu = f.nu, W = 2 * nu - 1;
    std::vector<double> s(n, 0.0);
    for (int band = 0; band < 2; ++band)
        for (int side = 0; side < 2; ++side) {
            const auto& A = band ? f.Aw[side] : f.A[side];
            const auto& B = band ? f.Bw[side] : f.B[side];
            for (size_t m = 0; m < NV; ++m) {
                size_t row = side ? half - 1 - m : m;
                double c = x[(band ? half : 0) + row];
                for (size_t k = 0; k < NV; ++k) s[side ? n - 1 - k : k] += A[m * NV + k] * c;
                for (int li = 0; li <= 2 * int(m); ++li) {
                    size_t l = NV + size_t(li);
                    s[side ? n - 1 - l : l] += B[m * size_t(W) + size_t(li)] * c;
                }
            }
        }
    for (size_t mm = NV; mm + NV < half; ++mm) {
        double c = x[mm], d = x[half + mm];
        for (int u = -nu + 1; u <= nu; ++u) s[size_t(long(2 * mm) + u)] += f.h[size_t(u + nu - 1)] * c + f.g[size_t(u + nu - 1)] * d;
    }
    return s;
}

// One periodic synthesis / analysis level and one VMP analysis level
// (wavelet.cpp:369-445 semantics), for the dense coarse block below.
std::vector<double> level_inverse_periodic_host(const Filters& f, const std::vector<double>& x) {
    const size_t n = x.size(), half = n / 2;
    const int nu = f.nu;
    std::vector<double> s(n, 0.0);
    for (size_t mm = 0; mm < half; ++mm)
        for (int u = -nu + 1; u <= nu; ++u) {
            size_t idx = size_t(((long long)(2 * mm) + u + 2 * (long long)n) % (long long)n);
            s[idx] += f.h[size_t(u + nu - 1)] * x[mm] + f.g[size_t(u + nu - 1)] * x[half + mm];
        }
    return s;
}

std::vector<double> level_forward_host(const Filters& f, const std::vector<double>& x, bool vmp) {
    const size_t n = x.size(), half = n / 2, NV = size_t(f.nu);
    const int nu = f.nu, W = 2 * nu - 1;
    std::vector<double> s(n, 0.0);
    if (!vmp) {
        for (size_t mm = 0; mm < half; ++mm)
            for (int u = -nu + 1; u <= nu; ++u) {
                size_t idx = size_t(((long long)(2 * mm) + u + 2 * (long long)n) % (long long)n);
                s[mm] += f.h[size_t(u + nu - 1)] * x[idx];
                s[half + mm] += f.g[size_t(u + nu - 1)] * x[idx];
            }
        return s;
    }
    for (int band = 0; band < 2; ++band)
        for (int side = 0; side < 2; ++side) {
            const auto& A = band ? f.Aw[side] : f.A[side];
            const auto& B = band ? f.Bw[side] : f.B[side];
            for (size_t m = 0; m < NV; ++m) {
                double acc = 0.0;
                for (size_t k = 0; k < NV; ++k) acc += A[m * NV + k] * x[side ? n - 1 - k : k];
                for (int li = 0; li <= 2 * int(m); ++li) {
                    size_t l = NV + size_t(li);
                    acc += B[m * size_t(W) + size_t(li)] * x[side ? n - 1 - l : l];
                }
                s[(band ? half : 0) + (side ? half - 1 - m : m)] = acc;
            }
        }
    for (size_t mm = NV; mm + NV < half; ++mm)
        for (int u = -nu + 1; u <= nu; ++u) {
            size_t idx = size_t((long long)(2 * mm) + u);
            s[mm] += f.h[size_t(u + nu - 1)] * x[idx];
            s[half + mm] += f.g[size_t(u + nu - 1)] * x[idx];
        }
    return s;
}

struct EdgeTerm {
    uint64_t p;
    int col;
    long row;  // offset into the concatenated table interior|left|right
};

}  // namespace

// ---------------------------------------------------------------------------
// the op
// ---------------------------------------------------------------------------
struct cww_op {
    cww_op_desc d{};
    int nu = 1, vmp = 0, r0 = 0, dim = 1, device = 0;
    int nsm = 148;  // SM count of the device (L2 prefetch distances)
    unsigned j = 0, q = 0;
    long long M = 1, N = 1, S = 1;
    Filters f;
    KernelTable kt;
    std::vector<EdgeTerm> terms;
    cww::Tables tabs{};
    double* d_tab = nullptr;
    std::string data_dir;
    // subsampled output (ComposedOp with a SamplingMask, fastop.cpp:231-281)
    std::vector<uint64_t> mask;
    uint64_t* d_mask = nullptr;
    bool masked = false;
    long long full_out = 0;  // output size of the unmasked operator
    // banded normal form G = U* U along one axis (built on first use)
    struct Gram {
        std::once_flag once;
        bool ok = false;
        int E = 0, b = 0;
        double* d = nullptr;
    };
    std::shared_ptr<Gram> gram = std::make_shared<Gram>();
    // side streams of the large path's slice pipeline (created on first use,
    // non-blocking; every call forks onto them from the caller's stream and
    // joins back, so they are only ordering, never shared state)
};

namespace {

// device table block: kap | em | h | g | edge filters
cww_status build_tables(cww_op& op) {
    const int nu = op.nu, W = 2 * nu - 1, NP = 2 * nu - 1;
    const long long S = op.S, M = op.M;
    const double scale = 1.0 / std::sqrt(double(M));
    std::vector<double> tab;
    cww::Tables& t = op.tabs;
    t.o_kap = 0;
    for (int l = 0; l < W; ++l)
        for (long long s = 0; s < S; ++s) tab.push_back(scale * op.kt.interior[size_t(l * S + s)]);
    t.o_em = int(tab.size());
    std::vector<double> em(size_t(S * 2 * NP * 2 * nu), 0.0);
    if (nu > 1) {
        const long long ofs_left = W * S, ofs_right = W * S + nu * W * S;
        (void)ofs_left;
        (void)ofs_right;
        for (const auto& e : op.terms) {
            int pi = e.p < uint64_t(NP) ? int(e.p) : NP + int(e.p - uint64_t(M - NP));
            int c = e.col < nu ? e.col : nu + int(e.col - (M - nu));
            const double* kap = nullptr;
            std::vector<double> all;
            all.insert(all.end(), op.kt.interior.begin(), op.kt.interior.end());
            all.insert(all.end(), op.kt.left.begin(), op.kt.left.end());
            all.insert(all.end(), op.kt.right.begin(), op.kt.right.end());
            kap = all.data() + e.row;
            for (long long s = 0; s < S; ++s) em[size_t(((s * 2 * NP) + pi) * 2 * nu + c)] += scale * kap[s];
        }
    }
    tab.insert(tab.end(), em.begin(), em.end());
    t.o_h = int(tab.size());
    tab.insert(tab.end(), op.f.h.begin(), op.f.h.end());
    t.o_g = int(tab.size());
    tab.insert(tab.end(), op.f.g.begin(), op.f.g.end());
    t.o_ef = int(tab.size());
    for (int side = 0; side < 2; ++side) {
        auto put = [&](const std::vector<double>& m, size_t n) {
            for (size_t i = 0; i < n; ++i) tab.push_back(i < m.size() ? m[i] : 0.0);
        };
        put(op.f.A[side], size_t(nu * nu));
        put(op.f.B[side], size_t(nu * W));
        put(op.f.Aw[side], size_t(nu * nu));
        put(op.f.Bw[side], size_t(nu * W));
    }
    // Dense edge blocks of one VMP level (valid for n >= 8 nu; coarser levels
    // use the generic path):  synthesis  out[i] = sum_k Sc[i][k] c[k] + Sd[i][k] d[k],
    // i < 3nu-1, k < 2nu (right side mirrored: i -> n-1-i, k -> half-1-k);
    // analysis  row m < nu: sum_k Da[m][k] x[k], k < 3nu-1 (A | B restricted to
    // li <= 2m as in wavelet.cpp:419-423; detail rows from Aw | Bw).
    t.o_syn = int(tab.size());
    const int EL = 3 * nu - 1, CI = 2 * nu;
    if (nu == 1) tab.insert(tab.end(), size_t(2 * EL * 2 * CI + 2 * 2 * nu * EL), 0.0);
    if (nu > 1) {
        const size_t n = size_t(16 * nu), half = n / 2;
        std::vector<double> syn(size_t(2 * EL * 2 * CI), 0.0);
        for (int band = 0; band < 2; ++band)
            for (int k = 0; k < CI; ++k)
                for (int side = 0; side < 2; ++side) {
                    std::vector<double> x(n, 0.0);
                    size_t idx = side ? half - 1 - size_t(k) : size_t(k);
                    x[(band ? half : 0) + idx] = 1.0;
                    auto y = level_inverse_vmp_host(op.f, x);
                    for (int i = 0; i < EL; ++i)  // [side][band][k][i]: lanes (i) read consecutively
                        syn[size_t(((side * 2 + band) * CI + k) * EL + i)] = y[side ? n - 1 - size_t(i) : size_t(i)];
                }
        tab.insert(tab.end(), syn.begin(), syn.end());
    }
    t.o_ana = int(tab.size());
    if (nu > 1) {
        std::vector<double> ana(size_t(2 * 2 * nu * EL), 0.0);
        for (int side = 0; side < 2; ++side)
            for (int band = 0; band < 2; ++band) {
                const auto& A = band ? op.f.Aw[side] : op.f.A[side];
                const auto& B = band ? op.f.Bw[side] : op.f.B[side];
                for (int m = 0; m < nu; ++m) {
                    double* row = ana.data() + ((side * 2 + band) * nu + m) * EL;
                    for (int k = 0; k < nu; ++k) row[k] = A[size_t(m * nu + k)];
                    for (int li = 0; li <= 2 * m; ++li) row[nu + li] = B[size_t(m * W + li)];
                }
            }
        tab.insert(tab.end(), ana.begin(), ana.end());
    }
    t.n = int(tab.size());
    CUDA_TRY(cudaMalloc(&op.d_tab, tab.size() * sizeof(double)));
    CUDA_TRY(cudaMemcpy(op.d_tab, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice));
    return CWW_OK;
}

// Prop. 4.1 edge decomposition, grouped by position (fastop.cpp:54-98)
void build_edge_terms(cww_op& op) {
    op.terms.clear();
    if (op.nu < 2) return;
    const int nu = op.nu, W = 2 * nu - 1;
    const long long S = op.S, M = op.M;
    const long ofs_left = long(W * S), ofs_right = long(W * S + nu * W * S);
    if (op.vmp) {
        for (int m = 0; m < nu; ++m)
            for (int l = 0; l <= nu - 1 + m; ++l) op.terms.push_back({uint64_t(l), m, ofs_left + long(m * W + l) * long(S)});
        for (int mb = 0; mb < nu; ++mb)
            for (int t = 0; t <= nu + mb - 1; ++t)
                op.terms.push_back({uint64_t(M + t - (nu + mb)), int(M - 1 - mb), ofs_right + long(mb * W + t) * long(S)});
    } else {
        for (int side = 0; side < 2; ++side)
            for (int k = 0; k < nu; ++k) {
                int col = side ? int(M - nu + k) : k;
                for (int l = -nu + 1; l <= nu - 1; ++l) {
                    long long pos = (col + l) % M;
                    if (pos < 0) pos += M;
                    op.terms.push_back({uint64_t(pos), col, long(l + nu - 1) * long(S)});
                }
            }
    }
    std::stable_sort(op.terms.begin(), op.terms.end(),
                     [](const EdgeTerm& a, const EdgeTerm& b) { return a.p < b.p; });
}

cww_status validate(const cww_op_desc* d) {
    if (d->precision != CWW_FP64 && d->precision != CWW_FP32) return fail(CWW_ERR_INVALID_ARG, "precision must be CWW_FP64 or CWW_FP32");
    if (d->family != 0 && d->family != 1) return fail(CWW_ERR_INVALID_ARG, "bad family");
    if (d->boundary != 0 && d->boundary != 1) return fail(CWW_ERR_INVALID_ARG, "bad boundary");
    if (d->nu < 1 || d->nu > 6)
        return fail(CWW_ERR_SPEC, "unsupported vanishing moments: %d (supported: 1..6)", d->nu);
    if (d->nu == 1 && d->boundary == 1)
        return fail(CWW_ERR_SPEC, "vmp boundary requires nu >= 2 (Haar has no boundary functions)");
    if (d->nu == 1 && d->family == 1) return fail(CWW_ERR_SPEC, "sym1 is identical to Haar; use db1");
    if (d->dim != 1 && d->dim != 2) return fail(CWW_ERR_SPEC, "FastOp dim must be 1 or 2");
    const int J0 = spec_min_level(d->nu);
    if (int(d->j) < J0) return fail(CWW_ERR_SPEC, "FastOp: j must be >= ceil(log2(2 nu))");
    if (d->nu >= 2 && d->q < 1) return fail(CWW_ERR_SPEC, "FastOp: q must be >= 1");
    if (d->j + d->q > 30) return fail(CWW_ERR_UNSUPPORTED, "j + q must be <= 30");
    // the two-pass large path holds 2^(j-5) tile rows in two shared-memory
    // passes of <= 512 rows each (one 2^23-point vector per pass pair)
    if (d->j > 23) return fail(CWW_ERR_UNSUPPORTED, "j must be <= 23 (M = 2^23 wavelet coefficients per axis)");
    if (d->j < 1) return fail(CWW_ERR_UNSUPPORTED, "j must be >= 1 (M = 1 is not supported)");
    if (d->q > 10) return fail(CWW_ERR_UNSUPPORTED, "q must be <= 10");
    if (d->dim == 2 && d->j + d->q > 17)
        return fail(CWW_ERR_UNSUPPORTED, "2D: j + q must be <= 17 (N^2 doubles of one image must fit a device)");
    int r0 = d->min_level < 0 ? J0 : d->min_level;
    if (r0 > int(d->j)) return fail(CWW_ERR_SPEC, "dwt: j below the coarsest admissible level");
    if (d->boundary == 1 && r0 < J0)
        return fail(CWW_ERR_SPEC, "vmp DWT requires min_level >= ceil(log2(2 nu)) = %d", J0);
    int R = d->kernel_resolution > 0 ? d->kernel_resolution : 14;
    if (R < int(d->q) || R > 24) return fail(CWW_ERR_SPEC, "kernel resolution must be in [q, 24]");
    return CWW_OK;
}

cudaStream_t S_(void* s) { return static_cast<cudaStream_t>(s); }

// 1D layout helpers
Layout lay_contig(long long len) { return Layout{0, len, 0, 1, 62, 62}; }

// largest power of two V <= cap with V*M <= 4096 (one small-path CTA)

int small_V(long long M, long long nvec, int cap = 32) {
    int V = 1;
    while (V * 2 <= cap && (V * 2) * M <= 4096 && V * 2 <= nvec) V *= 2;
    return V;
}

struct DevBuf {
    double* p = nullptr;
    cudaStream_t st = nullptr;
    ~DevBuf() {
        if (p) cudaFreeAsync(p, st);
    }
    cudaError_t alloc(size_t n, cudaStream_t s) {
        st = s;
        return cudaMallocAsync(&p, n * sizeof(double), s);
    }
};

cww::SmallArgs small_args(const cww_op* op, const double* in, Layout lin, double* out,
                          Layout lout, long long nvec, int V) {
    cww::SmallArgs a{};
    a.tab = op->d_tab;
    a.t = op->tabs;
    a.in = in;
    a.out = out;
    a.lin = lin;
    a.lout = lout;
    a.nvec = nvec;
    a.V = V;
    a.j = int(op->j);
    a.q = int(op->q);
    a.r0 = op->r0;
    a.use_idwt = op->d.use_idwt;
    a.vmp = op->vmp;
    return a;
}

cww_status run_small(const cww_op* op, const double* in, Layout lin, double* out, Layout lout,
                     long long nvec, bool adj, cudaStream_t st, bool wav = true) {
    if (nvec == 0) return CWW_OK;
    // warp-per-vector kernels (cww_warp.cuh) for large batches of 2^10-point
    // vectors; a few vectors run faster on the CTA-per-group kernels (every
    // thread of the CTA on one vector: cfg1 0.014 vs 0.018 ms)
    if (op->j == 10 && wav && nvec >= 256) {
        auto a = small_args(op, in, lin, out, lout, nvec, 8);
        Prof pr(adj ? "wv_adj" : "wv_fwd", st);
        CUDA_TRY(cww::launch_wv(op->nu, a, adj, st));
        return CWW_OK;
    }
    int V = small_V(op->M, nvec);
    const bool vf = adj ? lin.vfast() : lout.vfast();
    while (V > 1 && cww::small_smem_query(op->nu, V, int(op->j), int(op->q), adj, vf) > 200 * 1024) V /= 2;
    if (cww::small_smem_query(op->nu, V, int(op->j), int(op->q), adj, vf) > 227 * 1024)
        return fail(CWW_ERR_UNSUPPORTED, "shared-memory footprint too large for nu=%d j=%u q=%u", op->nu, op->j, op->q);
    auto a = small_args(op, in, lin, out, lout, nvec, V);
    if (!wav) a.use_idwt = 0;  // 2D: the wavelet transform of this axis runs as a separate panel pass
    // block-contiguous inputs allow a plain 16-byte copy (forward kernel); the
    // caller's buffer is only guaranteed 8-byte aligned, so a misaligned base
    // (e.g. x + 1) takes the element-wise path
    const long long M = op->M;
    const bool al16 = (reinterpret_cast<uintptr_t>(in) & 15) == 0;
    if (!al16) {
    } else if (lin.contig() && (V == 1 || (lin.vsh >= 62 && lin.vs == M))) a.in_block = 1;
    else if (lin.vs == 1 && lin.esh >= 62 && lin.es == V && lin.vsh < 62 && (1ll << lin.vsh) == V &&
             lin.vb == M * V)
        a.in_block = 2;
    Prof pr(adj ? "small_adj" : "small_fwd", st);
    CUDA_TRY(cww::launch_small(op->nu, a, adj, st));
    return CWW_OK;
}


// Wavelet pyramid plan of the large path
constexpr int kPyrSynBot = 10;      // coarse levels <= 10: k_wav_coarse (one CTA per vector)
constexpr int kWpyrLog = 9;         // warp pyramids: 2^9 samples of the top level per warp
constexpr int kWpyrAnaLevels = 3;   // analysis steps per pyramid launch

cww::PyrArgs pyr_args(const cww_op* op, long long nvec) {
    cww::PyrArgs y{};
    y.tab = op->d_tab;
    y.t = op->tabs;
    y.nvec = nvec;
    y.vmp = op->vmp;
    y.r0 = op->r0;
    y.pfd = 3 * op->nsm / 2;  // L2 prefetch 1.5 waves of CTAs ahead (measured at config 3)
    return y;
}

// Multilevel synthesis W^-1 (wavelet.cpp:487-514, Inverse) of nvec vectors of
// length M > 2^12 read through `lin`: the coarse levels r0+1..10 in one CTA per
// vector (k_wav_coarse), then chained warp pyramids of <= 6 (j <= 17) or 4
// levels each.  The level-j samples land contiguously (M apart) in w0 or w1;
// *xi points at them.
cww_status synth_chain(const cww_op* op, const double* in, Layout lin, long long nvec, double* w0, double* w1,
                       const double** xi, cudaStream_t st, int jt = -1) {
    const int j = jt < 0 ? int(op->j) : jt, nu = op->nu;
    const long long M = op->M;
    int bot = std::max(op->r0, std::min(kPyrSynBot, j - 1));
    const double* src = nullptr;  // level-bot coarse vector (nullptr: the op input)
    long long src_vs = 0;
    if (bot > op->r0) {
        cww::WavArgs w{};
        w.tab = op->d_tab;
        w.t = op->tabs;
        w.nvec = nvec;
        w.r0 = op->r0;
        w.vmp = op->vmp;
        w.kind = 0;
        w.lev = bot;
        w.inverse = 1;
        w.src = in;
        w.ls = lin;
        w.dst = w1;
        w.dst_vs = 1ll << bot;
        Prof pr("wav_coarse", st);
        CUDA_TRY(cww::launch_wav(nu, w, st));
        src = w1;
        src_vs = 1ll << bot;
    }
    double* bufs[2] = {w0, w1};
    while (bot < j) {
        const int top = std::min(j, bot + (j <= 17 ? 6 : 4));
        cww::PyrArgs y = pyr_args(op, nvec);
        y.top = top;
        y.bot = bot;
        y.cb = std::min(top, kWpyrLog);
        y.wmax = cww::pyr_wmax_syn(nu, y.top, y.bot, y.cb, op->vmp != 0, &y.dsum, &y.wmax2);
        // even slot sizes (16-byte aligned slot bases) with room for the bulk copies'
        // rounding to 16-byte bounds on both sides of every window
        y.wmax = (y.wmax + 3) & ~1;
        y.wmax2 = (y.wmax2 + 3) & ~1;
        y.dsum = (y.dsum + 2 * (y.top - y.bot) + 1) & ~1;
        y.x = in;
        y.lx = lin;
        y.src_is_x = src ? 0 : 1;
        y.src = src;
        y.src_vs = src_vs;
        y.out = bufs[src == w0 ? 1 : 0];  // never overwrite the level being read
        y.out_vs = M;
        {
            Prof pr("idwt_pyr", st);
            CUDA_TRY(cww::launch_pyr(nu, false, y, st));
        }
        src = y.out;
        src_vs = M;
        bot = top;
    }
    *xi = src;  // nullptr: no level to synthesise (level j is the op input's coarse part)
    return CWW_OK;
}

// Multilevel analysis W (wavelet.cpp:487-514, Forward) of nvec contiguous
// level-j vectors in w0 (M apart; clobbered) into coefficients through
// `lout`: chained warp pyramids of <= 3 steps; the launch that reaches level
// <= 10 finishes the coarse levels in its last CTA per vector (atomic ticket).
cww_status analysis_chain(const cww_op* op, double* w0, double* w1, double* out, Layout lout, long long nvec,
                          cudaStream_t st, int top = -1) {
    const long long M = op->M;
    const int nu = op->nu;
    unsigned* cnt = nullptr;
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&cnt), size_t(nvec) * sizeof(unsigned), st));
    struct CntFree {
        unsigned* p;
        cudaStream_t s;
        ~CntFree() { cudaFreeAsync(p, s); }
    } cnt_free{cnt, st};
    CUDA_TRY(cudaMemsetAsync(cnt, 0, size_t(nvec) * sizeof(unsigned), st));
    int T = top < 0 ? int(op->j) : top;  // level of the samples in w0
    const double* src = w0;
    double* sink[2] = {w1, w0};
    for (int it = 0;; ++it) {
        const int cb = std::min(T, kWpyrLog);
        const int bot = std::max({op->r0, T - kWpyrAnaLevels, T - cb});
        const bool tail = bot > op->r0 && bot <= std::max(kPyrSynBot, op->r0);
        cww::PyrArgs y = pyr_args(op, nvec);
        y.top = T;
        y.bot = bot;
        y.cb = cb;
        y.tail = tail ? 1 : 0;
        y.wmax = cww::pyr_wmax_ana(nu, T, bot, cb, op->vmp != 0, &y.wmax2) + 2;  // 16-byte phase shift + bulk-copy rounding
        y.wmax2 += 1;
        y.wmax += (y.wmax + y.wmax2) & 1;  // even per-warp stride: every warp's slots start 16-byte aligned
        y.src = src;
        y.src_vs = M;
        y.y = out;
        y.ly = lout;
        y.cws = bot == op->r0 ? nullptr : sink[it & 1];
        y.cws_vs = M;
        y.cnt = cnt;
        {
            Prof pr("dwt_pyr", st);
            CUDA_TRY(cww::launch_pyr(nu, true, y, st));
        }
        if (bot == op->r0 || tail) break;
        T = bot;
        src = y.cws;
    }
    return CWW_OK;
}

// ---- large path (1D, M > 2^12) ----
struct LargePlan {
    int kl, ng, ng_adj;  // kl: low K bits of the contiguous passes; ng: fwd2 sub-tiles per CTA; ng_adj: adj2
};
LargePlan large_plan(unsigned j) {
    int a = int(j) - cww::kLogB;
    int kl = (a + 1) / 2;
    if (kl > 8) kl = 8;    // pass-1 tiles of 256 rows (3 CTAs per SM) ...
    if (a - kl > 9) kl = a - 9;  // ... unless pass 2 would exceed 512 rows (j = 23: 512 x 512 rows)
    int kh = a - kl;
    int ng = 1;
    while (ng * (1 << kh) < 128 && ng * 2 <= (1 << kl)) ng *= 2;
    int ng_adj = 1;  // adj2 runs one tile row per thread: fill the CTA
    while (ng_adj * (1 << kh) < 256 && ng_adj * 2 <= (1 << kl)) ng_adj *= 2;
    return {kl, ng, ng_adj};
}

// Vectors per slice of the large path: whole batches per launch (the
// passes need the full grid to stream; L2-sized slices, also pipelined over
// 2-6 side streams, measured 13-38% slower at config 3), split
// only to bound the intermediates' memory (w0, w1, G) to 4 GiB.
long long large_slice(const cww_op* op, long long nvec) {
    const long long M = op->M, A = M >> cww::kLogB, CW = 32 + 2 * (op->nu - 1);
    const long long per = 8 * (2 * M + A * CW);
    return std::max(1ll, std::min(nvec, (4ll << 30) / per));
}

struct LargeBufs {
    DevBuf w0, w1, G, ev, epw, apart;
};

cww_status run_large_slice(const cww_op* op, const double* in, Layout lin, double* out, Layout lout,
                           long long nvec, bool adj, LargeBufs& B, cudaStream_t st) {
    const int nu = op->nu;
    const long long M = op->M;
    const auto pl = large_plan(op->j);
    const bool idwt = op->d.use_idwt && op->r0 < int(op->j);
    cww::LargeArgs a{};
    a.tab = op->d_tab;
    a.t = op->tabs;
    a.j = int(op->j);
    a.q = int(op->q);
    a.kl = pl.kl;
    a.ng = pl.ng;
    a.nvec = nvec;
    a.v0 = 0;
    a.in = in;
    a.lin = lin;
    a.G = B.G.p;
    a.ev = B.ev.p;
    a.epw = B.epw.p;
    a.nslot = cww::large_nslot(nu, int(op->q), int(op->j), pl.kl, pl.ng_adj);
    a.cta_red = cww::large_cta_red(nu, int(op->q)) ? 1 : 0;
    a.out = out;
    a.lout = lout;
    a.r0 = op->r0;
    a.use_idwt = op->d.use_idwt;
    a.vmp = op->vmp;
    // L2 prefetch distances (measured at config 3: 3/4 of a wave ahead for the
    // contiguous pass, one sequency block ahead in the strided pass)
    a.pfd1 = 3 * op->nsm / 4;
    a.pfs = pl.ng_adj == 1 ? 1 : 0;  // (sub-tiled CTAs: many short runs, the prefetches cost more than they hide)
    if (!adj) {
        // levels r0+1 .. j-1 by the pyramids and level j inside pass 1 (fuse_top)
        // when the batch's xi would not stay L2-resident (> 32 MB); else the
        // pyramids write xi and pass 1 reads it back from L2
        const double* xi = nullptr;
        long long xi_vs = M;
        const bool fuse = idwt && nvec * M * 8 > (32ll << 20);
        if (idwt) {
            cww_status s = synth_chain(op, in, lin, nvec, B.w0.p, B.w1.p, &xi, st, int(op->j) - (fuse ? 1 : 0));
            if (s != CWW_OK) return s;
            if (!xi) {  // r0 = j - 1 (fused): the input's first half is the level-(j-1) coarse vector
                xi = in + lin.vbase(0);
                xi_vs = lin.vbase(1) - lin.vbase(0);
            }
        }
        a.xi = xi;
        a.xi_vs = xi_vs;
        a.xi_is_input = idwt ? 0 : 1;
        a.fuse_top = fuse ? 1 : 0;
        {
            Prof pr("large_fwd1", st);
            // fused: the persistent ring kernel when the detail windows can be bulk-copied
            const bool al = fuse && ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(xi)) & 15) == 0 &&
                            (lin.vbase(1) - lin.vbase(0)) % 2 == 0 && xi_vs % 2 == 0;
            CUDA_TRY(cww::launch_large(nu, al ? 5 : 0, a, st));
        }
        Prof pr("large_fwd2", st);
        CUDA_TRY(cww::launch_large(nu, 1, a, st));
        return CWW_OK;
    }
    a.ng = pl.ng_adj;
    {
        Prof pr("large_adj2", st);
        CUDA_TRY(cww::launch_large(nu, 2, a, st));
    }
    // the finest analysis level inside pass 1 when the batch's xi would not
    // stay L2-resident (> 32 MB): d_{j-1} straight to the output, c_{j-1} to
    // the workspace (or, for r0 = j - 1, to the output's coarse half)
    const bool fana = idwt && nvec * M * 8 > (32ll << 20);
    const bool last = fana && op->r0 == int(op->j) - 1;
    a.xo = last ? out : (idwt ? B.w0.p : nullptr);
    a.xo_vs = last ? lout.vbase(1) - lout.vbase(0) : M;
    a.xo_is_output = idwt ? 0 : 1;
    a.fuse_ana = fana ? 1 : 0;
    a.apart = B.apart.p;
    {
        Prof pr("large_adj1", st);
        CUDA_TRY(cww::launch_large(nu, 3, a, st));
    }
    if (fana && nu > 1) {
        Prof pr("ana_fixup", st);
        CUDA_TRY(cww::launch_ana_fixup(nu, a, st));
    }
    if (!idwt || last) return CWW_OK;
    return analysis_chain(op, B.w0.p, B.w1.p, out, lout, nvec, st, fana ? int(op->j) - 1 : int(op->j));
}

// Forward (IDWT, pass 1, pass 2) or adjoint (pass 2, pass 1, DWT) of nvec
// contiguous vectors, slice by slice (large_slice) through one set of
// slice-sized intermediates.
cww_status run_large(const cww_op* op, const double* in, Layout lin, double* out, Layout lout, long long nvec,
                     bool adj, cudaStream_t st) {
    if (nvec == 0) return CWW_OK;
    const long long M = op->M;
    const int nu = op->nu, NP = 2 * nu - 1, CW = 32 + 2 * (nu - 1);
    const long long A = M >> cww::kLogB;
    const auto pl = large_plan(op->j);
    const bool idwt = op->d.use_idwt && op->r0 < int(op->j);
    const long long sl = large_slice(op, nvec);
    const long long nslot = cww::large_nslot(nu, int(op->q), int(op->j), pl.kl, pl.ng_adj);
    LargeBufs B;
    CUDA_TRY(B.G.alloc(size_t(sl * A * CW), st));
    CUDA_TRY(B.ev.alloc(size_t(sl * 2 * nu), st));
    if (idwt) {
        CUDA_TRY(B.w0.alloc(size_t(sl * M), st));
        CUDA_TRY(B.w1.alloc(size_t(sl * M), st));
    }
    if (adj) {
        CUDA_TRY(B.epw.alloc(size_t(sl * nslot * op->S * 2 * NP + 1), st));
        CUDA_TRY(B.apart.alloc(size_t(sl * (A >> pl.kl) * nu * 4 + 1), st));
    }
    for (long long v0 = 0; v0 < nvec; v0 += sl) {
        const long long nv = std::min(sl, nvec - v0);
        cww_status s = run_large_slice(op, in + lin.vbase(v0), lin, out + lout.vbase(v0), lout, nv, adj, B, st);
        if (s != CWW_OK) return s;
    }
    return CWW_OK;
}

cww_status run_1d(const cww_op* op, const double* in, double* out, long long nvec, bool adj,
                  cudaStream_t st) {
    Layout lin = lay_contig(adj ? op->N : op->M), lout = lay_contig(adj ? op->M : op->N);
    if (op->j <= unsigned(cww::kSmallMaxLog)) return run_small(op, in, lin, out, lout, nvec, adj, st);
    return run_large(op, in, lin, out, lout, nvec, adj, st);
}

// 2D: rows then columns (forward), columns then rows (adjoint), with the
// M x N intermediate stored in column panels of VC columns: [N/VC][M][VC].
// Above 2^12 per axis (large path): every pass runs on contiguous rows, with
// batched out-of-place transposes between the passes.
cww_status run_2d(const cww_op* op, const double* in, double* out, long long batch, bool adj,
                  cudaStream_t st) {
    const long long M = op->M, N = op->N;
    const int j = int(op->j), jq = int(op->j + op->q);
    cww_status s;
    if (j > cww::kSmallMaxLog) {
        // forward:  T = rows(X) (M x N), T^T (N x M), Z = rows(T^T) = Y^T (N x N), Y = Z^T
        // adjoint:  Y^T (N x N), V^T = rows(Y^T) (N x M), V (M x N), X = rows(V) (M x M)
        DevBuf t1, t2;
        CUDA_TRY(t1.alloc(size_t(batch * std::max(M * N, N * N)), st));
        CUDA_TRY(t2.alloc(size_t(batch * std::max(M * N, N * N)), st));
        if (!adj) {
            if ((s = run_large(op, in, lay_contig(M), t1.p, lay_contig(N), batch * M, false, st)) != CWW_OK) return s;
            {
                Prof pr("transpose", st);
                CUDA_TRY(cww::launch_transpose_rect(t1.p, t2.p, M, N, batch, st));
            }
            if ((s = run_large(op, t2.p, lay_contig(M), t1.p, lay_contig(N), batch * N, false, st)) != CWW_OK)
                return s;
            Prof pr("transpose", st);
            CUDA_TRY(cww::launch_transpose_rect(t1.p, out, N, N, batch, st));
            return CWW_OK;
        }
        {
            Prof pr("transpose", st);
            CUDA_TRY(cww::launch_transpose_rect(in, t1.p, N, N, batch, st));
        }
        if ((s = run_large(op, t1.p, lay_contig(N), t2.p, lay_contig(M), batch * N, true, st)) != CWW_OK) return s;
        {
            Prof pr("transpose", st);
            CUDA_TRY(cww::launch_transpose_rect(t2.p, t1.p, N, M, batch, st));
        }
        return run_large(op, t1.p, lay_contig(N), out, lay_contig(M), batch * M, true, st);
    }
    int VC = small_V(M, N, 16);
    int lvc = 0;
    while ((1 << lvc) < VC) ++lvc;
    DevBuf T;
    CUDA_TRY(T.alloc(size_t(batch * M * N), st));
    // row vectors: v = b*M + m ; column vectors: v = b*N + n
    Layout x_rows{0, M, 0, 1, 62, 62};                     // x[v*M + i]
    Layout t_rows{M * N, VC, M * VC, 1, j, lvc};           // T: (v>>j)*MN + (v&(M-1))*VC + (i>>lvc)*M*VC + (i&(VC-1))
    Layout t_cols{M * VC, 1, 0, VC, lvc, 62};              // T: (v>>lvc)*M*VC + (v&(VC-1)) + i*VC
    Layout y_cols{N * N, 1, 0, N, jq, 62};                 // y: (v>>jq)*N^2 + (v&(N-1)) + i*N
    if (!adj) {
        if ((s = run_small(op, in, x_rows, T.p, t_rows, batch * M, false, st)) != CWW_OK) return s;
        return run_small(op, T.p, t_cols, out, y_cols, batch * N, false, st);
    }
    if ((s = run_small(op, in, y_cols, T.p, t_cols, batch * N, true, st)) != CWW_OK) return s;
    return run_small(op, T.p, t_rows, out, x_rows, batch * M, true, st);
}

cww_status run_full(const cww_op* op, const double* in, double* out, long long batch, bool adj,
                    cudaStream_t st) {
    if (op->dim == 1) return run_1d(op, in, out, batch, adj, st);
    return run_2d(op, in, out, batch, adj, st);
}

cww_status run(const cww_op* op, const double* in, double* out, long long batch, bool adj,
               cudaStream_t st) {
    int cur = -1;
    CUDA_TRY(cudaGetDevice(&cur));
    if (cur != op->device) CUDA_TRY(cudaSetDevice(op->device));
    if (!op->masked) return run_full(op, in, out, batch, adj, st);
    // subsampled mask (fastop.cpp:253-281): full operator + gather / scatter
    const long long cnt = (long long)op->mask.size();
    DevBuf full;
    CUDA_TRY(full.alloc(size_t(batch * op->full_out), st));
    if (!adj) {
        cww_status s = run_full(op, in, full.p, batch, false, st);
        if (s != CWW_OK) return s;
        Prof pr("mask_gather", st);
        CUDA_TRY(cww::launch_mask(full.p, op->full_out, op->d_mask, cnt, out, batch, false, st));
        return CWW_OK;
    }
    CUDA_TRY(cudaMemsetAsync(full.p, 0, size_t(batch * op->full_out) * sizeof(double), st));
    {
        Prof pr("mask_scatter", st);
        CUDA_TRY(cww::launch_mask(full.p, op->full_out, op->d_mask, cnt, const_cast<double*>(in), batch,
                                  true, st));
    }
    return run_full(op, full.p, out, batch, true, st);
}

}  // namespace

// ---------------------------------------------------------------------------
// extern "C" ABI
// ---------------------------------------------------------------------------
extern "C" {

const char* cww_last_error(void) { return g_err.c_str(); }
}  // extern "C"

// shared with the other host translation units (cww_dist.cpp)
cww_status cww::set_error(cww_status st, const char* msg) {
    g_err = msg;
    return st;
}
void cww::note_launches(int n) { g_launches += (unsigned long long)n; }

extern "C" {
const char* cww_version(void) { return "cww_b200 0.1 (sm_100a)"; }

void cww_op_desc_init(cww_op_desc* d) {
    if (!d) return;
    std::memset(d, 0, sizeof *d);
    d->family = CWW_DAUBECHIES;
    d->nu = 2;
    d->boundary = CWW_VMP;
    d->j = 3;
    d->q = 1;
    d->dim = 1;
    d->min_level = -1;
    d->use_idwt = 0;
    d->kernel_resolution = 0;
    d->device = -1;
    d->data_dir = nullptr;
    d->mask = nullptr;
    d->mask_len = 0;
    d->cache_dir = nullptr;
    d->gpu_kernel_table = 0;
    d->precision = CWW_FP64;
}

cww_status cww_op_create(const cww_op_desc* desc, cww_op** out) {
    if (!desc || !out) return fail(CWW_ERR_INVALID_ARG, "null argument");
    *out = nullptr;
    cww_status s = validate(desc);
    if (s != CWW_OK) return s;
    if (desc->mask && desc->mask_len) {  // SamplingMask::validate (fastop.cpp:19-25)
        const long long n1 = 1ll << (desc->j + desc->q);
        const uint64_t nout = uint64_t(desc->dim == 2 ? n1 * n1 : n1);
        for (size_t i = 0; i < desc->mask_len; ++i) {
            if (desc->mask[i] >= nout) return fail(CWW_ERR_SPEC, "sampling mask index out of range");
            if (i > 0 && desc->mask[i] <= desc->mask[i - 1])
                return fail(CWW_ERR_SPEC, "sampling mask indices must be sorted and unique");
        }
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(CWW_ERR_CUDA, "no CUDA device available (the operator has no CPU fallback)");
    auto op = std::make_unique<cww_op>();
    op->d = *desc;
    op->nu = desc->nu;
    op->vmp = desc->boundary;
    op->j = desc->j;
    op->q = desc->q;
    op->dim = desc->dim;
    op->M = 1ll << desc->j;
    op->N = 1ll << (desc->j + desc->q);
    op->S = 1ll << desc->q;
    op->r0 = desc->min_level < 0 ? spec_min_level(desc->nu) : desc->min_level;
    op->data_dir = desc->data_dir ? desc->data_dir : "";
    if (desc->device >= 0) {
        if (desc->device >= ndev) return fail(CWW_ERR_CUDA, "device %d not present", desc->device);
        op->device = desc->device;
    } else {
        CUDA_TRY(cudaGetDevice(&op->device));
    }
    CUDA_TRY(cudaSetDevice(op->device));
    CUDA_TRY(cudaDeviceGetAttribute(&op->nsm, cudaDevAttrMultiProcessorCount, op->device));
    if ((s = load_filters(desc->family, desc->nu, op->data_dir.c_str(), op->f)) != CWW_OK) return s;
    int R = desc->kernel_resolution > 0 ? desc->kernel_resolution : 14;
    g_gpu_cascade = desc->gpu_kernel_table != 0;
    s = cached_kernel_table(op->f, desc->family, desc->boundary, int(desc->q), R, cache_dir_of(desc->cache_dir),
                            op->kt);
    g_gpu_cascade = false;
    if (s != CWW_OK) return s;
    build_edge_terms(*op);
    if ((s = build_tables(*op)) != CWW_OK) return s;
    op->full_out = op->dim == 2 ? op->N * op->N : op->N;
    if (desc->mask && desc->mask_len) {
        if (desc->mask_len != size_t(op->full_out)) {  // sorted + unique + full length = identity
            op->mask.assign(desc->mask, desc->mask + desc->mask_len);
            op->masked = true;
            CUDA_TRY(cudaMalloc(&op->d_mask, op->mask.size() * sizeof(uint64_t)));
            CUDA_TRY(cudaMemcpy(op->d_mask, op->mask.data(), op->mask.size() * sizeof(uint64_t),
                                cudaMemcpyHostToDevice));
        }
    }
    op->d.mask = nullptr;  // the caller's arrays / strings are not retained
    op->d.cache_dir = nullptr;
    op->d.data_dir = nullptr;
    // keep freed workspace in the stream-ordered pool between calls
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, op->device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    *out = op.release();
    return CWW_OK;
}

cww_status cww_op_destroy(cww_op* op) {
    if (!op) return CWW_OK;
    if (op->d_tab) cudaFree(op->d_tab);
    if (op->d_mask) cudaFree(op->d_mask);
    if (op->gram->d) cudaFree(op->gram->d);
    delete op;
    return CWW_OK;
}

cww_status cww_op_sizes(const cww_op* op, size_t* in, size_t* out) {
    if (!op) return fail(CWW_ERR_INVALID_ARG, "null op");
    size_t i = size_t(op->M), o = size_t(op->N);
    if (op->dim == 2) i *= i, o *= o;
    if (op->masked) o = op->mask.size();  // ComposedOp::rows (fastop.cpp:237-239)
    if (in) *in = i;
    if (out) *out = o;
    return CWW_OK;
}

static cww_status check_lens(const cww_op* op, size_t in_len, size_t out_len, size_t batch,
                             bool adj, const char* what) {
    if (!op) return fail(CWW_ERR_INVALID_ARG, "null op");
    size_t ni, no;
    cww_op_sizes(op, &ni, &no);
    if (adj) std::swap(ni, no);
    if (in_len != ni * batch || out_len != no * batch)
        return fail(CWW_ERR_DIMENSION, "%s: dimension mismatch", what);
    return CWW_OK;
}

cww_status cww_forward(const cww_op* op, const double* x, size_t x_len, double* y, size_t y_len,
                       size_t batch, void* stream) {
    cww_status s = check_lens(op, x_len, y_len, batch, false, "forward");
    if (s != CWW_OK) return s;
    if (op->d.precision != CWW_FP64) return fail(CWW_ERR_INVALID_ARG, "op created with precision fp32: use cww_forward_f32");
    if (batch == 0) return CWW_OK;
    if (!x || !y) return fail(CWW_ERR_INVALID_ARG, "null buffer");
    return run(op, x, y, (long long)batch, false, S_(stream));
}

cww_status cww_adjoint(const cww_op* op, const double* y, size_t y_len, double* x, size_t x_len,
                       size_t batch, void* stream) {
    cww_status s = check_lens(op, y_len, x_len, batch, true, "adjoint");
    if (s != CWW_OK) return s;
    if (op->d.precision != CWW_FP64) return fail(CWW_ERR_INVALID_ARG, "op created with precision fp32: use cww_adjoint_f32");
    if (batch == 0) return CWW_OK;
    if (!x || !y) return fail(CWW_ERR_INVALID_ARG, "null buffer");
    return run(op, y, x, (long long)batch, true, S_(stream));
}

// fp32 I/O: convert on entry, fp64 kernels, round once on exit
static cww_status run_f32(const cww_op* op, const float* in, size_t in_len, float* out, size_t out_len,
                          size_t batch, bool adj, void* stream) {
    cww_status s = check_lens(op, in_len, out_len, batch, adj, adj ? "adjoint" : "forward");
    if (s != CWW_OK) return s;
    if (op->d.precision != CWW_FP32) return fail(CWW_ERR_INVALID_ARG, "op created with precision fp64: use cww_%s",
                                                 adj ? "adjoint" : "forward");
    if (batch == 0) return CWW_OK;
    if (!in || !out) return fail(CWW_ERR_INVALID_ARG, "null buffer");
    cudaStream_t st = S_(stream);
    CUDA_TRY(cudaSetDevice(op->device));
    DevBuf din, dout;
    CUDA_TRY(din.alloc(in_len, st));
    CUDA_TRY(dout.alloc(out_len, st));
    {
        Prof pr("f32_in", st);
        CUDA_TRY(cww::launch_convert_f32_f64(in, din.p, (long long)in_len, st));
    }
    if ((s = run(op, din.p, dout.p, (long long)batch, adj, st)) != CWW_OK) return s;
    Prof pr("f32_out", st);
    CUDA_TRY(cww::launch_convert_f64_f32(dout.p, out, (long long)out_len, st));
    return CWW_OK;
}

cww_status cww_forward_f32(const cww_op* op, const float* x, size_t x_len, float* y, size_t y_len, size_t batch,
                           void* stream) {
    return run_f32(op, x, x_len, y, y_len, batch, false, stream);
}

cww_status cww_adjoint_f32(const cww_op* op, const float* y, size_t y_len, float* x, size_t x_len, size_t batch,
                           void* stream) {
    return run_f32(op, y, y_len, x, x_len, batch, true, stream);
}

// ---- banded normal form (U* U along one axis) -----------------------------
// Probes G = U* U with the op's own FastOp kernels on unit vectors: the
// first / last E columns, one interior column, and two verification columns.
// G is symmetric, so probed column i gives row i's band.  Rows outside the
// edge strips must equal the interior (Toeplitz) row, else the normal form is
// not used (the op falls back to forward + adjoint).
void build_gram(const cww_op* op) {
    const long long M = op->M;
    const int b = 2 * op->nu - 2, w = 2 * b + 1;
    if (M < 4 * (b + 2) || M < 64) return;
    cww_op u = *op;  // the plain 1D FastOp over the same device tables
    u.d.use_idwt = 0;
    u.dim = 1;
    u.masked = false;
    const bool wrap = !op->vmp;
    int E = std::min<long long>(6 * op->nu + 4, M / 4);
    std::vector<long long> cols;
    for (int i = 0; i < E; ++i) cols.push_back(i);
    for (int i = 0; i < E; ++i) cols.push_back(M - E + i);
    cols.push_back(M / 2);
    cols.push_back(E);
    cols.push_back(M - E - 1);
    const long long nc = (long long)cols.size(), N = op->N;
    std::vector<double> band(size_t(nc) * w, 0.0);
    cudaStream_t st;
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return;
    const long long chunk = std::max<long long>(1, std::min<long long>(nc, (256ll << 20) / (8 * (N + M))));
    double *e = nullptr, *f = nullptr;
    bool good = cudaMallocAsync(&e, size_t(chunk * M) * 8, st) == cudaSuccess &&
                cudaMallocAsync(&f, size_t(chunk * N) * 8, st) == cudaSuccess;
    for (long long c0 = 0; good && c0 < nc; c0 += chunk) {
        const long long cn = std::min(chunk, nc - c0);
        good = cudaMemsetAsync(e, 0, size_t(cn * M) * 8, st) == cudaSuccess;
        const double one = 1.0;
        for (long long c = 0; good && c < cn; ++c)
            good = cudaMemcpyAsync(e + c * M + cols[size_t(c0 + c)], &one, 8, cudaMemcpyHostToDevice, st) ==
                   cudaSuccess;
        good = good && run_1d(&u, e, f, cn, false, st) == CWW_OK && run_1d(&u, f, e, cn, true, st) == CWW_OK;
        for (long long c = 0; good && c < cn; ++c) {
            const long long k = cols[size_t(c0 + c)];
            for (int d = 0; d < w && good; ++d) {
                long long i = k + d - b;
                if (wrap) i &= M - 1;
                else if (i < 0 || i >= M) continue;
                good = cudaMemcpyAsync(&band[size_t((c0 + c) * w + d)], e + c * M + i, 8, cudaMemcpyDeviceToHost,
                                       st) == cudaSuccess;
            }
        }
        good = good && cudaStreamSynchronize(st) == cudaSuccess;
    }
    if (e) cudaFreeAsync(e, st);
    if (f) cudaFreeAsync(f, st);
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    cudaGetLastError();
    if (!good) return;
    // verification columns E and M-E-1 against the interior row
    const double* gI = &band[size_t(2 * E) * w];
    double mx = 0.0;
    for (int d = 0; d < w; ++d) mx = std::max(mx, std::fabs(gI[d]));
    for (int v = 1; v <= 2; ++v)
        for (int d = 0; d < w; ++d)
            if (std::fabs(band[size_t((2 * E + v) * w + d)] - gI[d]) > 1e-12 * mx) return;
    // band rows: column k probed = row k (symmetry): entry d multiplies x[k + d - b]
    std::vector<double> tab(size_t(2 * E + 1) * w);
    std::copy(band.begin(), band.begin() + size_t(2 * E + 1) * w, tab.begin());
    double* d = nullptr;
    if (cudaMalloc(&d, tab.size() * 8) != cudaSuccess) return;
    if (cudaMemcpy(d, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaFree(d);
        return;
    }
    op->gram->d = d;
    op->gram->E = E;
    op->gram->b = b;
    op->gram->ok = true;
}

cww::NormArgs norm_args(const cww_op* op, double* x, long long nvec) {
    cww::NormArgs a{};
    a.tab = op->d_tab;
    a.t = op->tabs;
    a.band = op->gram->d;
    a.E = op->gram->E;
    a.b = op->gram->b;
    a.in = x;
    a.out = x;
    a.in_vs = a.out_vs = op->M;
    a.nvec = nvec;
    a.j = int(op->j);
    a.r0 = op->r0;
    a.use_idwt = op->d.use_idwt;
    a.vmp = op->vmp;
    a.V = cww::normal_reg_ok(op->nu, int(op->j), op->r0, op->d.use_idwt) ? 1 : int(std::max<long long>(1, 4096 / op->M));
    a.pfd = op->nsm;  // L2 prefetch one CTA per SM ahead (config 5: row passes 17.86 -> 17.25 ms per 100)
    return a;
}

// x <- (A* A)^iters x with the banded form along every axis.  1D: rows in
// place.  2D (A* A = N1 (x) N1): each iteration applies N1 to the rows,
// transposes, applies N1 to the rows again -- the result is transposed, so
// iterations alternate between x and the work buffer and an odd count ends
// with one transpose back.
cww_status normal_banded(const cww_op* op, double* x, double* w, long long batch, int iters, cudaStream_t st) {
    const long long M = op->M;
    if (op->dim == 1) {
        cww::NormArgs a = norm_args(op, x, batch);
        for (int it = 0; it < iters; ++it) {
            Prof pr("normal_rows", st);
            CUDA_TRY(cww::launch_normal_rows(op->nu, a, st));
        }
        return CWW_OK;
    }
    double* cur = x;
    double* oth = w;
    for (int it = 0; it < iters; ++it) {
        cww::NormArgs a = norm_args(op, cur, batch * M);
        {
            Prof pr("normal_rows", st);
            CUDA_TRY(cww::launch_normal_rows(op->nu, a, st));
        }
        {
            Prof pr("transpose", st);
            CUDA_TRY(cww::launch_transpose(cur, oth, M, batch, st));
        }
        a = norm_args(op, oth, batch * M);
        {
            Prof pr("normal_rows", st);
            CUDA_TRY(cww::launch_normal_rows(op->nu, a, st));
        }
        std::swap(cur, oth);  // cur now holds (A* A x)^T of the iterate, or the iterate itself after two
    }
    if (cur != x) {  // odd iteration count: result is transposed in w
        Prof pr("transpose", st);
        CUDA_TRY(cww::launch_transpose(cur, x, M, batch, st));
    }
    return CWW_OK;
}

cww_status cww_normal(const cww_op* op, double* x, size_t x_len, double* work, size_t work_len,
                      size_t batch, int iters, void* stream) {
    if (!op) return fail(CWW_ERR_INVALID_ARG, "null op");
    size_t ni, no;
    cww_op_sizes(op, &ni, &no);
    if (x_len != ni * batch) return fail(CWW_ERR_DIMENSION, "normal: dimension mismatch");
    if (work && work_len < no * batch) return fail(CWW_ERR_DIMENSION, "normal: work buffer too small");
    cudaStream_t st = S_(stream);
    DevBuf wb;
    double* w = work;
    if (!w) {
        CUDA_TRY(wb.alloc(no * batch, st));
        w = wb.p;
    }
    CUDA_TRY(cudaSetDevice(op->device));
    if (!op->masked && op->M <= 4096) {
        std::call_once(op->gram->once, [op] { build_gram(op); });
        if (op->gram->ok) return normal_banded(op, x, w, (long long)batch, iters, st);
    }
    for (int it = 0; it < iters; ++it) {
        cww_status s = run(op, x, w, (long long)batch, false, st);
        if (s != CWW_OK) return s;
        if ((s = run(op, w, x, (long long)batch, true, st)) != CWW_OK) return s;
    }
    return CWW_OK;
}

// Least-squares driver (generalised sampling, SPEC.md gs_solve; SURVEY.md 8f
// row f1): CGLS on A* A x = A* y with A this op (masked or full), batched.
// Stops when every system's relative normal-equation residual
// ||A*(y - A x)|| / ||A* y|| <= residual_tol, or after max_iters.
// CG on the normal equations with the banded normal form N = A* A (full-mask
// ops): b = A* y once, then one banded N application per iteration instead of
// a forward and an adjoint.  Same stopping rule as CGLS: ||b - N x|| / ||b||.
cww_status gs_solve_normal(const cww_op* op, const double* y, double* x, long long B, double tol,
                           int max_iters, bool use_x0, int* iters_out, double* resid_out, cudaStream_t st) {
    size_t ni, no;
    cww_op_sizes(op, &ni, &no);
    const long long nx = (long long)ni;
    DevBuf bv, r, pv, qv, wv, part, sc;
    CUDA_TRY(bv.alloc(size_t(B * nx), st));
    CUDA_TRY(r.alloc(size_t(B * nx), st));
    CUDA_TRY(pv.alloc(size_t(B * nx), st));
    CUDA_TRY(qv.alloc(size_t(B * nx), st));
    CUDA_TRY(wv.alloc(size_t(B * nx), st));
    CUDA_TRY(part.alloc(size_t(B * cww::dot_nblk(nx, B)), st));
    CUDA_TRY(sc.alloc(size_t(5 * B), st));
    double* gam[2] = {sc.p, sc.p + B};
    double* pq = sc.p + 2 * B;
    double* s0 = sc.p + 3 * B;
    int* active = reinterpret_cast<int*>(sc.p + 4 * B);
    const size_t bytes = size_t(B * nx) * sizeof(double);
    cww_status rs;
    if ((rs = run(op, y, bv.p, B, true, st)) != CWW_OK) return rs;  // b = A* y
    if (use_x0) {  // r = b - N x0
        CUDA_TRY(cudaMemcpyAsync(qv.p, x, bytes, cudaMemcpyDeviceToDevice, st));
        if ((rs = normal_banded(op, qv.p, wv.p, B, 1, st)) != CWW_OK) return rs;
        CUDA_TRY(cudaMemcpyAsync(r.p, qv.p, bytes, cudaMemcpyDeviceToDevice, st));
        Prof pr("cg_vec", st);
        CUDA_TRY(cww::launch_sub_from(r.p, bv.p, B * nx, st));
    } else {
        CUDA_TRY(cudaMemsetAsync(x, 0, bytes, st));
        CUDA_TRY(cudaMemcpyAsync(r.p, bv.p, bytes, cudaMemcpyDeviceToDevice, st));
    }
    {
        Prof pr("cg_vec", st, 6);
        CUDA_TRY(cww::launch_dot(bv.p, bv.p, nx, B, part.p, gam[1], st));  // ||A* y||: the reference norm
        CUDA_TRY(cww::launch_sqrt(gam[1], s0, B, st));
        CUDA_TRY(cww::launch_dot(r.p, r.p, nx, B, part.p, gam[0], st));
        CUDA_TRY(cww::launch_cgls_flags(gam[0], s0, tol, active, B, st));
    }
    CUDA_TRY(cudaMemcpyAsync(pv.p, r.p, bytes, cudaMemcpyDeviceToDevice, st));
    std::vector<double> hg(size_t(2 * B));
    auto residuals = [&](const double* g, bool& done) -> cww_status {
        CUDA_TRY(cudaMemcpyAsync(hg.data(), g, size_t(B) * sizeof(double), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaMemcpyAsync(hg.data() + B, s0, size_t(B) * sizeof(double), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        done = true;
        for (long long b = 0; b < B; ++b) {
            const double n0 = hg[size_t(B + b)];
            const double rel = n0 > 0.0 ? std::sqrt(hg[size_t(b)]) / n0 : 0.0;
            if (resid_out) resid_out[b] = rel;
            if (rel > tol) done = false;
        }
        return CWW_OK;
    };
    int it = 0, cur = 0;
    bool done = false;
    for (; it < max_iters; ++it) {
        if ((rs = residuals(gam[cur], done)) != CWW_OK) return rs;
        if (done) break;
        CUDA_TRY(cudaMemcpyAsync(qv.p, pv.p, bytes, cudaMemcpyDeviceToDevice, st));
        if ((rs = normal_banded(op, qv.p, wv.p, B, 1, st)) != CWW_OK) return rs;  // q = N p
        {
            Prof pr("cg_vec", st, 3);
            CUDA_TRY(cww::launch_dot(pv.p, qv.p, nx, B, part.p, pq, st));
            CUDA_TRY(cww::launch_cgls_xr(x, r.p, pv.p, qv.p, nx, nx, B, gam[cur], pq, active, st));
        }
        {
            Prof pr("cg_vec", st, 4);
            CUDA_TRY(cww::launch_dot(r.p, r.p, nx, B, part.p, gam[cur ^ 1], st));
            CUDA_TRY(cww::launch_cgls_p(pv.p, r.p, nx, B, gam[cur ^ 1], gam[cur], st));
            CUDA_TRY(cww::launch_cgls_flags(gam[cur ^ 1], s0, tol, active, B, st));
        }
        cur ^= 1;
    }
    if (!done && (rs = residuals(gam[cur], done)) != CWW_OK) return rs;
    if (iters_out) *iters_out = it;
    if (!done) {
        double worst = 0.0;
        for (long long b = 0; b < B; ++b) {
            const double n0 = hg[size_t(B + b)];
            worst = std::max(worst, n0 > 0.0 ? std::sqrt(hg[size_t(b)]) / n0 : 0.0);
        }
        return fail(CWW_ERR_NOT_CONVERGED, "gs_solve: CG did not converge in %d iterations (relative residual %.3e)",
                    it, worst);
    }
    return CWW_OK;
}

cww_status gs_solve(const cww_op* op, const double* y, double* x, long long B, double tol, int max_iters,
                    bool use_x0, int* iters_out, double* resid_out, cudaStream_t st) {
    size_t ni, no;
    cww_op_sizes(op, &ni, &no);
    const long long nx = (long long)ni, nr = (long long)no;
    DevBuf r, sv, pv, qv, part, sc;
    CUDA_TRY(r.alloc(size_t(B * nr), st));
    CUDA_TRY(qv.alloc(size_t(B * nr), st));
    CUDA_TRY(sv.alloc(size_t(B * nx), st));
    CUDA_TRY(pv.alloc(size_t(B * nx), st));
    const long long nb = std::max(cww::dot_nblk(nx, B), cww::dot_nblk(nr, B));
    CUDA_TRY(part.alloc(size_t(B * nb), st));
    CUDA_TRY(sc.alloc(size_t(5 * B), st));  // gam[2B] | qq | s0 | active (as int)
    double* gam[2] = {sc.p, sc.p + B};
    double* qq = sc.p + 2 * B;
    double* s0 = sc.p + 3 * B;
    int* active = reinterpret_cast<int*>(sc.p + 4 * B);
    cww_status rs;
    if (use_x0) {
        if ((rs = run(op, x, r.p, B, false, st)) != CWW_OK) return rs;
        Prof pr("cg_vec", st);
        CUDA_TRY(cww::launch_sub_from(r.p, y, B * nr, st));
    } else {
        CUDA_TRY(cudaMemsetAsync(x, 0, size_t(B * nx) * sizeof(double), st));
        CUDA_TRY(cudaMemcpyAsync(r.p, y, size_t(B * nr) * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
    if (use_x0) {  // reference norm ||A* y||
        if ((rs = run(op, y, sv.p, B, true, st)) != CWW_OK) return rs;
        Prof pr("cg_vec", st, 3);
        CUDA_TRY(cww::launch_dot(sv.p, sv.p, nx, B, part.p, gam[1], st));
        CUDA_TRY(cww::launch_sqrt(gam[1], s0, B, st));
    }
    if ((rs = run(op, r.p, sv.p, B, true, st)) != CWW_OK) return rs;
    {
        Prof pr("cg_vec", st, 4);
        CUDA_TRY(cww::launch_dot(sv.p, sv.p, nx, B, part.p, gam[0], st));
        if (!use_x0) CUDA_TRY(cww::launch_sqrt(gam[0], s0, B, st));
        CUDA_TRY(cww::launch_cgls_flags(gam[0], s0, tol, active, B, st));
    }
    CUDA_TRY(cudaMemcpyAsync(pv.p, sv.p, size_t(B * nx) * sizeof(double), cudaMemcpyDeviceToDevice, st));
    std::vector<double> hg(size_t(2 * B));
    auto residuals = [&](const double* g, bool& done) -> cww_status {
        CUDA_TRY(cudaMemcpyAsync(hg.data(), g, size_t(B) * sizeof(double), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaMemcpyAsync(hg.data() + B, s0, size_t(B) * sizeof(double), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        done = true;
        for (long long b = 0; b < B; ++b) {
            const double n0 = hg[size_t(B + b)];
            const double rel = n0 > 0.0 ? std::sqrt(hg[size_t(b)]) / n0 : 0.0;
            if (resid_out) resid_out[b] = rel;
            if (rel > tol) done = false;
        }
        return CWW_OK;
    };
    int it = 0, cur = 0;
    bool done = false;
    for (; it < max_iters; ++it) {
        if ((rs = residuals(gam[cur], done)) != CWW_OK) return rs;
        if (done) break;
        if ((rs = run(op, pv.p, qv.p, B, false, st)) != CWW_OK) return rs;  // q = A p
        {
            Prof pr("cg_vec", st, 3);
            CUDA_TRY(cww::launch_dot(qv.p, qv.p, nr, B, part.p, qq, st));
            CUDA_TRY(cww::launch_cgls_xr(x, r.p, pv.p, qv.p, nx, nr, B, gam[cur], qq, active, st));
        }
        if ((rs = run(op, r.p, sv.p, B, true, st)) != CWW_OK) return rs;  // s = A* r
        {
            Prof pr("cg_vec", st, 4);
            CUDA_TRY(cww::launch_dot(sv.p, sv.p, nx, B, part.p, gam[cur ^ 1], st));
            CUDA_TRY(cww::launch_cgls_p(pv.p, sv.p, nx, B, gam[cur ^ 1], gam[cur], st));
            CUDA_TRY(cww::launch_cgls_flags(gam[cur ^ 1], s0, tol, active, B, st));
        }
        cur ^= 1;
    }
    if (!done && (rs = residuals(gam[cur], done)) != CWW_OK) return rs;
    if (iters_out) *iters_out = it;
    if (!done) {
        double worst = 0.0;
        for (long long b = 0; b < B; ++b) {
            const double n0 = hg[size_t(B + b)];
            worst = std::max(worst, n0 > 0.0 ? std::sqrt(hg[size_t(b)]) / n0 : 0.0);
        }
        return fail(CWW_ERR_NOT_CONVERGED, "gs_solve: CG did not converge in %d iterations (relative residual %.3e)",
                    it, worst);
    }
    return CWW_OK;
}

static cww_status host_call(const cww_op* op, const double* in, size_t in_len, double* out,
                            size_t out_len, size_t batch, bool adj) {
    cww_status s = check_lens(op, in_len, out_len, batch, adj, adj ? "adjoint" : "forward");
    if (s != CWW_OK) return s;
    if (op->d.precision != CWW_FP64) return fail(CWW_ERR_INVALID_ARG, "op created with precision fp32: use the f32 entry points");
    if (batch == 0) return CWW_OK;
    CUDA_TRY(cudaSetDevice(op->device));
    cudaStream_t st;
    CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    double *din = nullptr, *dout = nullptr;
    cww_status rs = CWW_OK;
    cudaError_t e = cudaMallocAsync(&din, in_len * 8, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&dout, out_len * 8, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(din, in, in_len * 8, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) rs = fail(CWW_ERR_CUDA, "host staging: %s", cudaGetErrorString(e));
    if (rs == CWW_OK) rs = run(op, din, dout, (long long)batch, adj, st);
    if (rs == CWW_OK) {
        e = cudaMemcpyAsync(out, dout, out_len * 8, cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) rs = fail(CWW_ERR_CUDA, "host staging: %s", cudaGetErrorString(e));
    }
    if (din) cudaFreeAsync(din, st);
    if (dout) cudaFreeAsync(dout, st);
    e = cudaStreamSynchronize(st);
    if (rs == CWW_OK && e != cudaSuccess) rs = fail(CWW_ERR_CUDA, "%s", cudaGetErrorString(e));
    cudaStreamDestroy(st);
    return rs;
}

// Compressed-sensing reconstruction (SPEC.md cs_solve, Eq. QCBP; SURVEY.md 8f
// row f2): min ||z||_1 subject to ||A z - y||^2 <= eta, A = this op (masked
// ComposedOp in the CS use case), by the Chambolle-Pock primal-dual iteration
// with F = indicator of the ball ||. - y|| <= sqrt(eta), G = ||.||_1, K = A:
//   xi  <- prox_{sigma F*}(xi + sigma A zbar) = sigma (1 - min(1, sqrt(eta)/||t||)) t,
//          t = xi / sigma + A zbar - y                       (Moreau)
//   z'  <- soft(z - tau A* xi, tau);  zbar <- 2 z' - z
// tau = sigma = 0.99 / L with L^2 = lambda_max(A* A) from a power iteration.
// Stops (checked every kCheck iterations) when every system has
// ||z' - z|| <= tol ||z'|| and ||A z - y||^2 <= eta + tol ||y||^2.
static cww_status cs_solve(const cww_op* op, const double* y, double* z, long long B, double eta, double tol,
                           int max_iters, int* iters_out, double* resid_out, cudaStream_t st) {
    size_t ni, no;
    cww_op_sizes(op, &ni, &no);
    const long long nx = (long long)ni, nr = (long long)no;
    DevBuf zbar, s, xi, w, part, sc;
    CUDA_TRY(zbar.alloc(size_t(B * nx), st));
    CUDA_TRY(s.alloc(size_t(B * nx), st));
    CUDA_TRY(xi.alloc(size_t(B * nr), st));
    CUDA_TRY(w.alloc(size_t(B * nr), st));
    const long long nb = std::max(cww::dot_nblk(nx, B), cww::dot_nblk(nr, B));
    CUDA_TRY(part.alloc(size_t(B * nb), st));
    CUDA_TRY(sc.alloc(size_t(5 * B), st));  // tt | dz2 | z2 | r2 | y2
    double *tt = sc.p, *dz2 = sc.p + B, *z2 = sc.p + 2 * B, *r2 = sc.p + 3 * B, *y2 = sc.p + 4 * B;
    cww_status rs;
    // L^2 = lambda_max(A* A): power iteration from A* y_0 (||A|| <= ~1, no rescaling needed)
    double L2 = 1.0;
    {
        if ((rs = run(op, y, s.p, 1, true, st)) != CWW_OK) return rs;
        double prev = 0.0;
        for (int k = 0; k < 30; ++k) {
            if ((rs = run(op, s.p, w.p, 1, false, st)) != CWW_OK) return rs;
            if ((rs = run(op, w.p, zbar.p, 1, true, st)) != CWW_OK) return rs;
            {
                Prof pr("cp_vec", st, 4);
                CUDA_TRY(cww::launch_dot(s.p, s.p, nx, 1, part.p, tt, st));
                CUDA_TRY(cww::launch_dot(zbar.p, zbar.p, nx, 1, part.p, dz2, st));
            }
            double h[2];
            CUDA_TRY(cudaMemcpyAsync(h, tt, sizeof(double), cudaMemcpyDeviceToHost, st));
            CUDA_TRY(cudaMemcpyAsync(h + 1, dz2, sizeof(double), cudaMemcpyDeviceToHost, st));
            CUDA_TRY(cudaStreamSynchronize(st));
            if (!(h[0] > 0.0)) break;  // A* y = 0: any step size works
            const double lam = std::sqrt(h[1] / h[0]);
            std::swap(s.p, zbar.p);
            if (k > 4 && std::fabs(lam - prev) <= 1e-6 * lam) {
                L2 = lam;
                break;
            }
            prev = lam;
            L2 = lam;
        }
    }
    const double L = std::sqrt(std::max(L2, 1e-300)) * 1.02;
    const double tau = 0.99 / L, sigma = 0.99 / L, seta = std::sqrt(eta);
    CUDA_TRY(cudaMemsetAsync(z, 0, size_t(B * nx) * sizeof(double), st));
    CUDA_TRY(cudaMemsetAsync(zbar.p, 0, size_t(B * nx) * sizeof(double), st));
    CUDA_TRY(cudaMemsetAsync(xi.p, 0, size_t(B * nr) * sizeof(double), st));
    {
        Prof pr("cp_vec", st, 2);
        CUDA_TRY(cww::launch_dot(y, y, nr, B, part.p, y2, st));
    }
    std::vector<double> h(size_t(4 * B));
    constexpr int kCheck = 20;
    int it = 0;
    bool done = false;
    auto check = [&]() -> cww_status {
        if ((rs = run(op, z, w.p, B, false, st)) != CWW_OK) return rs;  // A z - y
        {
            Prof pr("cp_vec", st, 7);
            CUDA_TRY(cww::launch_sub(w.p, w.p, y, B * nr, st));
            CUDA_TRY(cww::launch_dot(w.p, w.p, nr, B, part.p, r2, st));
            CUDA_TRY(cww::launch_dot(s.p, s.p, nx, B, part.p, dz2, st));
            CUDA_TRY(cww::launch_dot(z, z, nx, B, part.p, z2, st));
        }
        CUDA_TRY(cudaMemcpyAsync(h.data(), dz2, size_t(4 * B) * sizeof(double), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        done = true;
        for (long long b = 0; b < B; ++b) {
            const double d2 = h[size_t(b)], zz = h[size_t(B + b)], rr = h[size_t(2 * B + b)],
                         yy = h[size_t(3 * B + b)];
            if (resid_out) resid_out[b] = rr;
            if (!(d2 <= tol * tol * zz) || !(rr <= eta + tol * yy)) done = false;
        }
        return CWW_OK;
    };
    while (it < max_iters) {
        if ((rs = run(op, zbar.p, w.p, B, false, st)) != CWW_OK) return rs;  // A zbar
        {
            Prof pr("cp_vec", st, 4);
            CUDA_TRY(cww::launch_cp_dual(xi.p, w.p, y, sigma, seta, nr, B, part.p, tt, st));
        }
        if ((rs = run(op, xi.p, s.p, B, true, st)) != CWW_OK) return rs;  // A* xi
        {
            Prof pr("cp_vec", st);
            CUDA_TRY(cww::launch_cp_primal(z, zbar.p, s.p, tau, B * nx, st));
        }
        ++it;
        if (it % kCheck == 0 || it == max_iters) {
            if ((rs = check()) != CWW_OK) return rs;
            if (done) break;
        }
    }
    if (iters_out) *iters_out = it;
    if (done) return CWW_OK;
    if (it == 0 && (rs = check()) != CWW_OK) return rs;
    if (done) return CWW_OK;
    // classify the failure: is eta below the least-squares residual (infeasible)?
    double worst = 0.0;
    for (long long b = 0; b < B; ++b) worst = std::max(worst, h[size_t(2 * B + b)]);
    {
        DevBuf xl;
        CUDA_TRY(xl.alloc(size_t(B * nx), st));
        cww_status g = gs_solve(op, y, xl.p, B, 1e-12, int(std::min<long long>(4 * nx + 100, 100000)), false,
                                nullptr, nullptr, st);
        if (g == CWW_OK || g == CWW_ERR_NOT_CONVERGED) {
            if ((rs = run(op, xl.p, w.p, B, false, st)) != CWW_OK) return rs;
            CUDA_TRY(cww::launch_sub(w.p, w.p, y, B * nr, st));
            CUDA_TRY(cww::launch_dot(w.p, w.p, nr, B, part.p, r2, st));
            std::vector<double> ls(static_cast<size_t>(B));
            CUDA_TRY(cudaMemcpyAsync(ls.data(), r2, size_t(B) * sizeof(double), cudaMemcpyDeviceToHost, st));
            CUDA_TRY(cudaStreamSynchronize(st));
            for (long long b = 0; b < B; ++b)
                if (ls[size_t(b)] > eta * (1.0 + 1e-9) + 1e-300)
                    return fail(CWW_ERR_INFEASIBLE,
                                "cs_solve: eta = %.3e is below the least-squares residual %.3e of system %lld", eta,
                                ls[size_t(b)], b);
        }
    }
    return fail(CWW_ERR_NOT_CONVERGED, "cs_solve: no convergence in %d iterations (residual^2 %.3e, eta %.3e)", it,
                worst, eta);
}

cww_status cww_cs_solve(const cww_op* op, const double* y, size_t y_len, double* x, size_t x_len, size_t batch,
                        double eta, double tol, int max_iters, int* iters, double* residuals, void* stream) {
    cww_status s = check_lens(op, x_len, y_len, batch, false, "cs_solve");
    if (s != CWW_OK) return s;
    if (iters) *iters = 0;
    if (batch == 0) return CWW_OK;
    if (!x || !y) return fail(CWW_ERR_INVALID_ARG, "null buffer");
    if (max_iters < 0 || !(tol >= 0.0) || !(eta >= 0.0)) return fail(CWW_ERR_INVALID_ARG, "cs_solve: bad parameters");
    CUDA_TRY(cudaSetDevice(op->device));
    return cs_solve(op, y, x, (long long)batch, eta, tol, max_iters, iters, residuals, S_(stream));
}

cww_status cww_gs_solve(const cww_op* op, const double* y, size_t y_len, double* x, size_t x_len,
                        size_t batch, double residual_tol, int max_iters, int use_x0, int* iters,
                        double* residuals, void* stream) {
    cww_status s = check_lens(op, x_len, y_len, batch, false, "gs_solve");
    if (s != CWW_OK) return s;
    if (iters) *iters = 0;
    if (batch == 0) return CWW_OK;
    if (!x || !y) return fail(CWW_ERR_INVALID_ARG, "null buffer");
    if (max_iters < 0 || !(residual_tol >= 0.0)) return fail(CWW_ERR_INVALID_ARG, "gs_solve: bad parameters");
    CUDA_TRY(cudaSetDevice(op->device));
    if (!op->masked && op->M <= 4096) {
        std::call_once(op->gram->once, [op] { build_gram(op); });
        if (op->gram->ok)
            return gs_solve_normal(op, y, x, (long long)batch, residual_tol, max_iters, use_x0 != 0, iters,
                                   residuals, S_(stream));
    }
    return gs_solve(op, y, x, (long long)batch, residual_tol, max_iters, use_x0 != 0, iters, residuals,
                    S_(stream));
}

cww_status cww_kernel_table_save(int family, int nu, int boundary, unsigned q, int resolution,
                                 const char* data_dir, const char* path) {
    if (!path) return fail(CWW_ERR_INVALID_ARG, "null path");
    if (nu < 1 || nu > 6 || family < 0 || family > 1 || boundary < 0 || boundary > 1 || q > 20)
        return fail(CWW_ERR_SPEC, "unsupported kernel table spec");
    if (q < 1) return fail(CWW_ERR_SPEC, "kernel table requires q >= 1");  // kernel.cpp:32-33
    if (nu < 2) return fail(CWW_ERR_SPEC, "kernel tables are for nu >= 2 (Haar uses the FWHT/DWT composition)");
    Filters f;
    cww_status s = load_filters(family, nu, data_dir, f);
    if (s != CWW_OK) return s;
    const int R = resolution > 0 ? resolution : 14;
    KernelTable t;
    if ((s = kernel_table(f, boundary, int(q), R, t)) != CWW_OK) return s;
    return cwwk_save(t, CwwkHeader{family, nu, boundary, int(q), R}, path);
}

cww_status cww_kernel_table_load(const char* path, int* header, double* interior, size_t ni, double* left,
                                 size_t nl, double* right, size_t nr, size_t* counts) {
    if (!path) return fail(CWW_ERR_INVALID_ARG, "null path");
    KernelTable t;
    CwwkHeader h;
    cww_status s = cwwk_load(path, t, h);
    if (s != CWW_OK) return s;
    if (header) {
        header[0] = h.family;
        header[1] = h.nu;
        header[2] = h.vmp;
        header[3] = h.q;
        header[4] = h.R;
    }
    if (counts) {
        counts[0] = t.interior.size();
        counts[1] = t.left.size();
        counts[2] = t.right.size();
    }
    if ((interior && ni < t.interior.size()) || (left && nl < t.left.size()) || (right && nr < t.right.size()))
        return fail(CWW_ERR_DIMENSION, "kernel table buffers too small");
    if (interior) std::memcpy(interior, t.interior.data(), t.interior.size() * 8);
    if (left) std::memcpy(left, t.left.data(), t.left.size() * 8);
    if (right) std::memcpy(right, t.right.data(), t.right.size() * 8);
    return CWW_OK;
}

// Chunk-pipelined host staging for pinned buffers: H2D (side stream), compute
// (caller stream), D2H (second side stream), one event per chunk and stage.
static bool is_pinned(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

struct SideStreams {  // per host thread and device: created once
    cudaStream_t in = nullptr, out = nullptr;
    int device = -1;
};

static cww_status host_call_async(const cww_op* op, const double* in, size_t in_len, double* out,
                                  size_t out_len, size_t batch, bool adj, cudaStream_t st) {
    cww_status s = check_lens(op, in_len, out_len, batch, adj, adj ? "adjoint" : "forward");
    if (s != CWW_OK) return s;
    if (op->d.precision != CWW_FP64) return fail(CWW_ERR_INVALID_ARG, "op created with precision fp32: use the f32 entry points");
    if (batch == 0) return CWW_OK;
    if (!in || !out) return fail(CWW_ERR_INVALID_ARG, "null buffer");
    if (!is_pinned(in) || !is_pinned(out)) return host_call(op, in, in_len, out, out_len, batch, adj);
    CUDA_TRY(cudaSetDevice(op->device));
    constexpr size_t zc_max = size_t(256) << 10;
    if ((in_len + out_len) * sizeof(double) <= zc_max && op->M <= (1ll << cww::kSmallMaxLog)) {
        // tiny transforms (small path: each input read once, each output written
        // once): the kernels read / write the pinned buffers over PCIe directly
        // (zero-copy) -- no copy launches on the latency-bound path
        cudaPointerAttributes ai{}, ao{};
        if (cudaPointerGetAttributes(&ai, in) == cudaSuccess && cudaPointerGetAttributes(&ao, out) == cudaSuccess &&
            ai.devicePointer && ao.devicePointer)
            return run(op, static_cast<const double*>(ai.devicePointer), static_cast<double*>(ao.devicePointer),
                       (long long)batch, adj, st);
        cudaGetLastError();
    }
    if ((in_len + out_len) * sizeof(double) <= (size_t(2) << 20)) {  // small: one stream, no pipeline
        double *din = nullptr, *dout = nullptr;
        CUDA_TRY(cudaMallocAsync(&din, in_len * sizeof(double), st));
        CUDA_TRY(cudaMallocAsync(&dout, out_len * sizeof(double), st));
        CUDA_TRY(cudaMemcpyAsync(din, in, in_len * sizeof(double), cudaMemcpyHostToDevice, st));
        if ((s = run(op, din, dout, (long long)batch, adj, st)) != CWW_OK) return s;
        CUDA_TRY(cudaMemcpyAsync(out, dout, out_len * sizeof(double), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaFreeAsync(din, st));
        CUDA_TRY(cudaFreeAsync(dout, st));
        return CWW_OK;
    }
    thread_local SideStreams ss;
    if (ss.device != op->device) {
        CUDA_TRY(cudaStreamCreateWithFlags(&ss.in, cudaStreamNonBlocking));
        CUDA_TRY(cudaStreamCreateWithFlags(&ss.out, cudaStreamNonBlocking));
        ss.device = op->device;
    }
    const size_t ni = in_len / batch, no = out_len / batch;
    constexpr size_t target = size_t(64) << 20;  // input+output per chunk (tuned: 8-256 MB)
    size_t cb = std::max<size_t>(1, target / ((ni + no) * sizeof(double)));
    cb = std::min(cb, batch);
    const size_t nch = (batch + cb - 1) / cb;
    double *din = nullptr, *dout = nullptr;
    CUDA_TRY(cudaMallocAsync(&din, in_len * sizeof(double), st));
    CUDA_TRY(cudaMallocAsync(&dout, out_len * sizeof(double), st));
    std::vector<cudaEvent_t> ev(2 * nch + 2, nullptr);
    for (auto& e : ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cudaEvent_t e_start = ev[2 * nch], e_done = ev[2 * nch + 1];
    CUDA_TRY(cudaEventRecord(e_start, st));  // buffers allocated, caller's prior work ordered
    CUDA_TRY(cudaStreamWaitEvent(ss.in, e_start, 0));
    for (size_t k = 0; k < nch; ++k) {
        const size_t b0 = k * cb, nb = std::min(cb, batch - b0);
        CUDA_TRY(cudaMemcpyAsync(din + b0 * ni, in + b0 * ni, nb * ni * sizeof(double), cudaMemcpyHostToDevice,
                                 ss.in));
        CUDA_TRY(cudaEventRecord(ev[2 * k], ss.in));
        CUDA_TRY(cudaStreamWaitEvent(st, ev[2 * k], 0));
        if ((s = run(op, din + b0 * ni, dout + b0 * no, (long long)nb, adj, st)) != CWW_OK) return s;
        CUDA_TRY(cudaEventRecord(ev[2 * k + 1], st));
        CUDA_TRY(cudaStreamWaitEvent(ss.out, ev[2 * k + 1], 0));
        CUDA_TRY(cudaMemcpyAsync(out + b0 * no, dout + b0 * no, nb * no * sizeof(double), cudaMemcpyDeviceToHost,
                                 ss.out));
    }
    CUDA_TRY(cudaEventRecord(e_done, ss.out));
    CUDA_TRY(cudaStreamWaitEvent(st, e_done, 0));  // the caller's stream sees the results
    CUDA_TRY(cudaFreeAsync(din, st));
    CUDA_TRY(cudaFreeAsync(dout, st));
    for (auto& e : ev) cudaEventDestroy(e);  // destruction is deferred until the events complete
    return CWW_OK;
}

cww_status cww_forward_host_async(const cww_op* op, const double* x, size_t x_len, double* y, size_t y_len,
                                  size_t batch, void* stream) {
    return host_call_async(op, x, x_len, y, y_len, batch, false, S_(stream));
}

cww_status cww_adjoint_host_async(const cww_op* op, const double* y, size_t y_len, double* x, size_t x_len,
                                  size_t batch, void* stream) {
    return host_call_async(op, y, y_len, x, x_len, batch, true, S_(stream));
}

cww_status cww_forward_host(const cww_op* op, const double* x, size_t x_len, double* y,
                            size_t y_len, size_t batch) {
    return host_call(op, x, x_len, y, y_len, batch, false);
}

cww_status cww_adjoint_host(const cww_op* op, const double* y, size_t y_len, double* x,
                            size_t x_len, size_t batch) {
    return host_call(op, y, y_len, x, x_len, batch, true);
}

// In-place multilevel DWT / IDWT of `batch` vectors (1D) or images (2D,
// rows then columns: dwt_apply_2d) on the op's spec, j and r0
// (wavelet.cpp:487-536).  M <= 2^12: one CTA per vector (k_wav_coarse,
// through the data's layout).  Larger M: the large path's warp pyramids
// (synth_chain / analysis_chain) on contiguous rows; 2D columns via batched
// transposes.
cww_status cww_dwt(const cww_op* op, double* data, size_t len, size_t batch, int dir, void* stream) {
    if (!op) return fail(CWW_ERR_INVALID_ARG, "null op");
    if (!data && batch) return fail(CWW_ERR_INVALID_ARG, "null buffer");
    if (dir != CWW_DWT_FORWARD && dir != CWW_DWT_INVERSE) return fail(CWW_ERR_INVALID_ARG, "dwt: bad direction");
    size_t ni;
    cww_op_sizes(op, &ni, nullptr);
    if (len != ni * batch) return fail(CWW_ERR_DIMENSION, "dwt: bad input length");
    if (batch == 0 || op->r0 >= int(op->j)) return CWW_OK;
    CUDA_TRY(cudaSetDevice(op->device));
    cudaStream_t st = S_(stream);
    const long long M = op->M;
    const int nu = op->nu;
    const bool inverse = dir == CWW_DWT_INVERSE;
    const long long nvec = (long long)batch * (op->dim == 2 ? M : 1);
    if (M > (1ll << cww::kSmallMaxLog)) {
        // contiguous rows through the pyramids; 2D: rows, transpose, rows, transpose back
        DevBuf w0, w1, tr;
        CUDA_TRY(w0.alloc(size_t(nvec * M), st));
        CUDA_TRY(w1.alloc(size_t(nvec * M), st));
        if (op->dim == 2) CUDA_TRY(tr.alloc(size_t(nvec * M), st));
        auto rows = [&](double* buf) -> cww_status {  // in place on nvec contiguous rows of buf
            if (inverse) {
                const double* xi = nullptr;
                cww_status s = synth_chain(op, buf, lay_contig(M), nvec, w0.p, w1.p, &xi, st);
                if (s != CWW_OK) return s;
                CUDA_TRY(cudaMemcpyAsync(buf, xi, size_t(nvec * M) * 8, cudaMemcpyDeviceToDevice, st));
                return CWW_OK;
            }
            CUDA_TRY(cudaMemcpyAsync(w0.p, buf, size_t(nvec * M) * 8, cudaMemcpyDeviceToDevice, st));
            return analysis_chain(op, w0.p, w1.p, buf, lay_contig(M), nvec, st);
        };
        cww_status s = rows(data);
        if (s != CWW_OK || op->dim == 1) return s;
        {
            Prof pr("transpose", st);
            CUDA_TRY(cww::launch_transpose(data, tr.p, M, (long long)batch, st));
        }
        if ((s = rows(tr.p)) != CWW_OK) return s;
        Prof pr("transpose", st);
        CUDA_TRY(cww::launch_transpose(tr.p, data, M, (long long)batch, st));
        return CWW_OK;
    }
    auto pass = [&](Layout l, long long nv) -> cww_status {  // k_wav_coarse: 3 * 2^j doubles of smem
        cww::WavArgs w{};
        w.kind = 0;
        w.tab = op->d_tab;
        w.t = op->tabs;
        w.nvec = nv;
        w.lev = int(op->j);
        w.r0 = op->r0;
        w.inverse = inverse;
        w.vmp = op->vmp;
        // in place: both sides through the layout (src read fully before writes)
        DevBuf tmp;
        CUDA_TRY(tmp.alloc(size_t(nv * M), st));
        w.src = data;
        w.ls = l;
        w.sv0 = 0;
        w.src_vs = M;
        if (inverse) {
            w.dst = tmp.p;
            w.dst_vs = M;
            Prof pr("wav_coarse", st, 2);
            CUDA_TRY(cww::launch_wav(nu, w, st));
            // copy back through the layout with a forward "coarse" of zero levels
            cww::WavArgs c = w;
            c.inverse = 0;
            c.r0 = int(op->j);
            c.src = tmp.p;
            c.src_vs = M;
            c.dst = data;
            c.ld = l;
            c.dv0 = 0;
            CUDA_TRY(cww::launch_wav(nu, c, st));
        } else {
            // gather into contiguous scratch, transform, scatter back
            cww::WavArgs g = w;
            g.inverse = 1;
            g.r0 = int(op->j);
            g.dst = tmp.p;
            g.dst_vs = M;
            Prof pr("wav_coarse", st, 2);
            CUDA_TRY(cww::launch_wav(nu, g, st));
            cww::WavArgs f = w;
            f.inverse = 0;
            f.src = tmp.p;
            f.src_vs = M;
            f.dst = data;
            f.ld = l;
            f.dv0 = 0;
            CUDA_TRY(cww::launch_wav(nu, f, st));
        }
        return CWW_OK;
    };
    if (op->dim == 1) return pass(lay_contig(M), nvec);
    // 2D: rows (v = b*M + r: x[v*M + i]) then columns (v = b*M + c: x[(v>>j)*M^2 + (v&(M-1)) + i*M])
    cww_status s = pass(Layout{0, M, 0, 1, 62, 62}, nvec);
    if (s != CWW_OK) return s;
    return pass(Layout{M * M, 1, 0, M, int(op->j), 62}, nvec);
}

cww_status cww_fwht(double* v, unsigned bits, size_t batch, int sequency, void* stream) {
    if (!v && batch) return fail(CWW_ERR_INVALID_ARG, "null buffer");
    if (bits > 30) return fail(CWW_ERR_UNSUPPORTED, "length too large");
    if (batch == 0) return CWW_OK;
    cudaStream_t st = S_(stream);
    DevBuf scr;
    if (bits > 13 && sequency) CUDA_TRY(scr.alloc(size_t(batch) << bits, st));
    Prof pr("fwht", st, bits <= 13 ? 1 : 1 + (int(bits) - 13 + 9) / 10);
    CUDA_TRY(cww::launch_fwht(v, int(bits), (long long)batch, sequency, scr.p, st));
    return CWW_OK;
}

cww_status cww_sequency_perm(unsigned bits, uint32_t* perm, void* stream) {
    if (!perm) return fail(CWW_ERR_INVALID_ARG, "null buffer");
    if (bits > 31) return fail(CWW_ERR_UNSUPPORTED, "bits must be <= 31");
    Prof pr("seq_perm", S_(stream));
    CUDA_TRY(cww::launch_seq_perm(perm, int(bits), S_(stream)));
    return CWW_OK;
}

cww_status cww_walsh_sign_rows(const uint64_t* p, size_t npos, unsigned j, double* signs, void* stream) {
    if ((!p || !signs) && npos) return fail(CWW_ERR_INVALID_ARG, "null buffer");
    if (j > 30) return fail(CWW_ERR_UNSUPPORTED, "j must be <= 30");
    if (npos == 0) return CWW_OK;
    Prof pr("sign_rows", S_(stream));
    CUDA_TRY(cww::launch_sign_rows(p, (long long)npos, int(j), signs, S_(stream)));
    return CWW_OK;
}

cww_status cww_op_kernel_table(const cww_op* op, double* interior, size_t ni, double* left,
                               size_t nl, double* right, size_t nr) {
    if (!op) return fail(CWW_ERR_INVALID_ARG, "null op");
    if (interior) {
        if (ni < op->kt.interior.size()) return fail(CWW_ERR_DIMENSION, "interior buffer too small");
        std::copy(op->kt.interior.begin(), op->kt.interior.end(), interior);
    }
    if (left && !op->kt.left.empty()) {
        if (nl < op->kt.left.size()) return fail(CWW_ERR_DIMENSION, "left buffer too small");
        std::copy(op->kt.left.begin(), op->kt.left.end(), left);
    }
    if (right && !op->kt.right.empty()) {
        if (nr < op->kt.right.size()) return fail(CWW_ERR_DIMENSION, "right buffer too small");
        std::copy(op->kt.right.begin(), op->kt.right.end(), right);
    }
    return CWW_OK;
}

cww_status cww_op_edge_terms(const cww_op* op, uint64_t* p, int32_t* col, int64_t* row, size_t cap,
                             size_t* n) {
    if (!op || !n) return fail(CWW_ERR_INVALID_ARG, "null argument");
    *n = op->terms.size();
    for (size_t i = 0; i < op->terms.size() && i < cap; ++i) {
        if (p) p[i] = op->terms[i].p;
        if (col) col[i] = op->terms[i].col;
        if (row) row[i] = op->terms[i].row;
    }
    return CWW_OK;
}

// test_rng semantics (proj/tests/test_util.hpp:10-27) + SURVEY.md 8d inputs
cww_status cww_synth(int kind, uint64_t seed, unsigned j, int r0, double density, int dim, double* out) {
    if (!out) return fail(CWW_ERR_INVALID_ARG, "null buffer");
    if (j > 28) return fail(CWW_ERR_UNSUPPORTED, "j too large");
    struct Rng {
        uint64_t s;
        uint64_t u64() {
            s ^= s << 13;
            s ^= s >> 7;
            s ^= s << 17;
            return s * 0x2545F4914F6CDD1Dull;
        }
        double uni() { return double(u64() >> 11) * 0x1.0p-53; }
        double normal() {
            double u1 = uni(), u2 = uni();
            if (u1 < 1e-300) u1 = 1e-300;
            return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
        }
    } rng{seed * 0x9E3779B97F4A7C15ull + 1};
    const size_t side = size_t(1) << j, n = dim == 2 ? side * side : side;
    auto level = [&](uint64_t i) {
        if (i < (uint64_t(2) << r0)) return r0;
        int l = 0;
        while ((i >> (l + 1)) != 0) ++l;
        return l;
    };
    size_t k = density >= 1.0 ? n : size_t(std::llround(density * double(n)));
    std::vector<uint32_t> idx;
    if (k < n) {
        idx.resize(n);
        for (size_t i = 0; i < n; ++i) idx[i] = uint32_t(i);
        for (size_t i = 0; i < k; ++i) {
            size_t t = i + size_t(rng.u64() % uint64_t(n - i));
            std::swap(idx[i], idx[t]);
        }
        std::memset(out, 0, n * sizeof(double));
    }
    for (size_t i = 0; i < k; ++i) {
        size_t pos = idx.empty() ? i : idx[i];
        double v = rng.normal();
        if (kind == 1) {
            int lev = dim == 2 ? std::max(level(pos / side), level(pos % side)) : level(pos);
            v = std::ldexp(v, -lev);
        }
        out[pos] = v;
    }
    return CWW_OK;
}

void cww_profile_enable(int on) { g_prof_on = on ? 1 : 0; }

unsigned long long cww_kernel_launches(void) { return g_launches.load(); }

cww_status cww_profile_dump(char* json, size_t cap) {
    std::vector<ProfRec> recs;
    {
        std::lock_guard<std::mutex> lk(g_prof_mu);
        recs.swap(g_prof);
    }
    std::map<std::string, std::pair<double, long>> agg;
    cww_status st = CWW_OK;
    for (auto& r : recs) {
        float ms = 0.f;
        cudaError_t e = cudaEventSynchronize(r.b);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, r.a, r.b);
        if (e != cudaSuccess) st = fail(CWW_ERR_CUDA, "profile: %s", cudaGetErrorString(e));
        auto& x = agg[r.name];
        x.first += ms;
        x.second += 1;
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    std::string out = "{";
    for (auto& [k, v] : agg) {
        char buf[160];
        std::snprintf(buf, sizeof buf, "%s\"%s\": [%.6f, %ld]", out.size() > 1 ? ", " : "", k.c_str(), v.first, v.second);
        out += buf;
    }
    out += "}";
    if (json && cap) {
        std::strncpy(json, out.c_str(), cap - 1);
        json[cap - 1] = 0;
    }
    return st;
}

}  // extern "C"
