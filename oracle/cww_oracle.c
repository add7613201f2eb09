/* TEST INFRASTRUCTURE ONLY -- CPU oracle, see cww_oracle.h.
 *
 * Plain-C restatement of the reference's hot path.  Each function cites the
 * reference code it follows (paths under /root/reference/proj).  Written for
 * clarity, not speed: the parity tests run it at sizes that finish in
 * seconds.  The arithmetic order deliberately follows the reference (same
 * butterfly order, same accumulation order) so that it agrees with the
 * compiled reference to the last few ulps.
 */
#define _GNU_SOURCE
#include "cww_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];
static int fail(const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return 1;
}
const char* orc_last_error(void) { return g_err; }

/* ---- CRC-32, zlib polynomial (proj/include/cww/crc32.hpp:10-24) ---------- */
uint32_t orc_crc32(const void* data, size_t len) {
    const unsigned char* p = (const unsigned char*)data;
    uint32_t c = 0xFFFFFFFFu;
    for (size_t i = 0; i < len; ++i) {
        c ^= p[i];
        for (int k = 0; k < 8; ++k) c = (c >> 1) ^ (0xEDB88320u & (0u - (c & 1u)));
    }
    return c ^ 0xFFFFFFFFu;
}

/* J0 = ceil(log2(2 nu)), 0 for Haar (wavelet.cpp:16-21) */
int orc_min_level(int nu) {
    if (nu == 1) return 0;
    int j = 0;
    while ((1 << j) < 2 * nu) ++j;
    return j;
}

/* ---- CWWF loader (wavelet.cpp:123-186, format gen_wavelet_data.py:453-467) */
static int rd_u32(const unsigned char* b, size_t sz, size_t* pos, uint32_t* v) {
    if (*pos + 4 > sz) return 1;
    memcpy(v, b + *pos, 4);
    *pos += 4;
    return 0;
}

static int rd_mat(const unsigned char* b, size_t sz, size_t* pos, uint32_t rows, uint32_t cols,
                  double* dst) {
    uint32_t r, c;
    if (rd_u32(b, sz, pos, &r) || rd_u32(b, sz, pos, &c)) return fail("truncated filter file");
    if (r != rows || c != cols) return fail("filter data shape mismatch");
    size_t n = (size_t)r * c;
    if (*pos + 8 * n > sz) return fail("truncated filter file");
    memcpy(dst, b + *pos, 8 * n);
    *pos += 8 * n;
    return 0;
}

int orc_load_filters(int family, int nu, const char* data_dir, orc_filters* f) {
    memset(f, 0, sizeof *f);
    f->family = family;
    f->nu = nu;
    if (nu < 1 || nu > ORC_MAX_NU) return fail("unsupported vanishing moments");
    if (nu == 1) { /* built-in Haar (wavelet.cpp:104-113) */
        double s = 1.0 / sqrt(2.0);
        f->h[0] = s, f->h[1] = s;
        f->g[0] = s, f->g[1] = -s;
        f->phi[0] = 1.0, f->phi[1] = 0.0;
        return 0;
    }
    char path[4096];
    snprintf(path, sizeof path, "%s/%s%d.cwwf", data_dir ? data_dir : ".",
             family == 0 ? "db" : "sym", nu);
    FILE* fp = fopen(path, "rb");
    if (!fp) return fail("cannot open filter data file");
    fseek(fp, 0, SEEK_END);
    long sz = ftell(fp);
    fseek(fp, 0, SEEK_SET);
    unsigned char* b = (unsigned char*)malloc((size_t)(sz > 0 ? sz : 1));
    size_t got = fread(b, 1, (size_t)sz, fp);
    fclose(fp);
    int rc = 1;
    if (sz < 20 || got != (size_t)sz) { fail("truncated filter file"); goto out; }
    uint32_t stored;
    memcpy(&stored, b + sz - 4, 4);
    if (orc_crc32(b, (size_t)sz - 4) != stored) { fail("checksum failure in filter file"); goto out; }
    if (memcmp(b, "CWWF", 4) != 0) { fail("bad magic in filter file"); goto out; }
    size_t pos = 4, end = (size_t)sz - 4;
    uint32_t ver, fam, fnu, nmat;
    if (rd_u32(b, end, &pos, &ver) || rd_u32(b, end, &pos, &fam) || rd_u32(b, end, &pos, &fnu) ||
        rd_u32(b, end, &pos, &nmat)) { fail("truncated filter file"); goto out; }
    if (ver != 1 || fam != (uint32_t)family || fnu != (uint32_t)nu || nmat != 13) {
        fail("filter header mismatch");
        goto out;
    }
    uint32_t L = 2 * nu, W = L - 1, V = nu;
    if (rd_mat(b, end, &pos, 1, L, f->h) || rd_mat(b, end, &pos, 1, L, f->g) ||
        rd_mat(b, end, &pos, 1, L, f->phi))
        goto out;
    for (int e = 0; e < 2; ++e) {
        if (rd_mat(b, end, &pos, V, W, f->E[e]) || rd_mat(b, end, &pos, V, V, f->A[e]) ||
            rd_mat(b, end, &pos, V, W, f->B[e]) || rd_mat(b, end, &pos, V, V, f->Aw[e]) ||
            rd_mat(b, end, &pos, V, W, f->Bw[e]))
            goto out;
    }
    double s = 0;
    for (uint32_t i = 0; i < L; ++i) s += f->h[i];
    if (fabs(s - sqrt(2.0)) > 1e-10) { fail("corrupt filter data"); goto out; }
    rc = 0;
out:
    free(b);
    return rc;
}

/* ---- Walsh primitives (walsh.hpp:25-62, walsh.cpp:20-131) ---------------- */
static uint64_t bitrev(uint64_t v, unsigned bits) {
    uint64_t r = 0;
    for (unsigned i = 0; i < bits; ++i) r = (r << 1) | ((v >> i) & 1u);
    return r;
}

uint64_t orc_seq_to_nat(uint64_t n, unsigned bits) { return bitrev(n ^ (n >> 1), bits); }

/* Def. 3.1: exponent sum_i (n_{i-1} + n_i) x_i with x_i the i-th binary digit
 * of p / 2^j (walsh.cpp:20-31). */
int orc_walsh_eval(uint64_t n, uint64_t p, unsigned j) {
    unsigned par = 0;
    for (unsigned i = 1; i <= j; ++i)
        if ((p >> (j - i)) & 1u) par ^= (unsigned)(((n >> (i - 1)) ^ (n >> i)) & 1u);
    return par ? -1 : 1;
}

/* w_r(p/2^j) for r < 2^j (walsh.cpp:123-131) */
void orc_walsh_sign_row(uint64_t p, unsigned j, double* sign) {
    uint64_t v = bitrev(p, j), mask = v ^ (v << 1);
    for (uint64_t r = 0; r < (1ull << j); ++r)
        sign[r] = (__builtin_popcountll(r & mask) & 1) ? -1.0 : 1.0;
}

static int is_pow2(size_t n) { return n && !(n & (n - 1)); }

/* Radix-2 natural-order FWHT, stages h = 1, 2, 4, ... (walsh.cpp:41-52).
 * The reference's cache-blocked recursion (walsh.cpp:58-72) performs the
 * same butterflies on the same operands, so the results are identical. */
int orc_fwht_natural(double* v, size_t n) {
    if (!is_pow2(n)) return fail("length is not a power of two");
    for (size_t h = 1; h < n; h <<= 1)
        for (size_t i = 0; i < n; i += 2 * h)
            for (size_t k = i; k < i + h; ++k) {
                double a = v[k], b = v[k + h];
                v[k] = a + b;
                v[k + h] = a - b;
            }
    return 0;
}

/* natural FWHT + gather out[n] = nat[bitrev(gray(n))] (walsh.cpp:88-98) */
int orc_fwht_sequency(double* v, size_t n) {
    if (orc_fwht_natural(v, n)) return 1;
    unsigned bits = 0;
    while ((1ull << bits) < n) ++bits;
    double* t = (double*)malloc(n * sizeof(double));
    memcpy(t, v, n * sizeof(double));
    for (size_t i = 0; i < n; ++i) v[i] = t[orc_seq_to_nat(i, bits)];
    free(t);
    return 0;
}

/* ---- cascade (wavelet.cpp:192-311) ----------------------------------------
 * Samples on the grid of spacing 2^-r over the support.  Interior refinement:
 * phi(x) = sqrt2 sum_u hbar_u phi(2x - u)  (refine_interior, 195-214). */
static double* refine(const double* prev, long prev_n, int r, int a, int b, const double* hb,
                      int nu, long* out_n) {
    long n = (long)(b - a) * (1l << r) + 1, half = 1l << (r - 1), lo = (long)a * half;
    double* cur = (double*)calloc((size_t)n, sizeof(double));
    double s2 = sqrt(2.0);
    for (long t = 0; t < n; ++t) {
        long tpos = (long)a * (1l << r) + t;
        double acc = 0.0;
        for (int u = -nu + 1; u <= nu; ++u) {
            long i = tpos - u * half - lo;
            if (i >= 0 && i < prev_n) acc += hb[u + nu - 1] * prev[i];
        }
        cur[t] = s2 * acc;
    }
    *out_n = n;
    return cur;
}

/* left-edge cascade in construction coordinates, support [0, nu+m]
 * (cascade_left_all, 217-277); returns samples of edge function m. */
static double* cascade_left(const double* hb, const double* phi_int, const double* E,
                            const double* A, const double* B, int nu, int R, int mwant,
                            long* out_n) {
    int a = -nu + 1, b = nu, W = 2 * nu - 1;
    double** lev = (double**)calloc((size_t)R + 1, sizeof(double*));
    long* lev_n = (long*)calloc((size_t)R + 1, sizeof(long));
    lev[0] = (double*)malloc((size_t)(2 * nu) * sizeof(double));
    memcpy(lev[0], phi_int, (size_t)(2 * nu) * sizeof(double));
    lev_n[0] = 2 * nu;
    for (int r = 1; r <= R; ++r) lev[r] = refine(lev[r - 1], lev_n[r - 1], r, a, b, hb, nu, &lev_n[r]);

    double* cur[ORC_MAX_NU];
    long cur_n[ORC_MAX_NU];
    for (int m = 0; m < nu; ++m) { /* integer-grid values from E (238-250) */
        cur_n[m] = nu + m + 1;
        cur[m] = (double*)calloc((size_t)cur_n[m], sizeof(double));
        for (long k = 0; k <= nu + m; ++k) {
            double acc = 0.0;
            for (int i = 0; i < W; ++i) {
                long arg = k - (-nu + 1 + i);
                if (arg > -nu && arg < nu) acc += E[m * W + i] * phi_int[arg + nu - 1];
            }
            cur[m][k] = acc;
        }
    }
    double s2 = sqrt(2.0);
    for (int r = 1; r <= R; ++r) { /* 253-275 */
        double* nxt[ORC_MAX_NU];
        long nxt_n[ORC_MAX_NU];
        for (int m = 0; m < nu; ++m) {
            nxt_n[m] = ((long)(nu + m) << r) + 1;
            nxt[m] = (double*)calloc((size_t)nxt_n[m], sizeof(double));
            for (long t = 0; t < nxt_n[m]; ++t) {
                double acc = 0.0;
                for (int k = 0; k < nu; ++k)
                    if (t < cur_n[k]) acc += A[m * nu + k] * cur[k][t];
                for (int li = 0; li <= 2 * m; ++li) {
                    long idx = t - (long)(nu + li) * (1l << (r - 1)) - (long)a * (1l << (r - 1));
                    double iv = (idx >= 0 && idx < lev_n[r - 1]) ? lev[r - 1][idx] : 0.0;
                    acc += B[m * W + li] * iv;
                }
                nxt[m][t] = s2 * acc;
            }
        }
        for (int m = 0; m < nu; ++m) {
            free(cur[m]);
            cur[m] = nxt[m];
            cur_n[m] = nxt_n[m];
        }
    }
    for (int m = 0; m < nu; ++m)
        if (m != mwant) free(cur[m]);
    for (int r = 0; r <= R; ++r) free(lev[r]);
    free(lev);
    free(lev_n);
    *out_n = cur_n[mwant];
    return cur[mwant];
}

long orc_cascade(const orc_filters* f, int kind, int m, int R, double* out, size_t cap,
                 int* support_left) {
    int nu = f->nu;
    double* v = NULL;
    long n = 0;
    if (R < 1) return -fail("cascade resolution must be >= 1");
    if (kind == 0) { /* 285-292 */
        long pn = 2 * nu;
        double* p = (double*)malloc((size_t)pn * sizeof(double));
        memcpy(p, f->phi, (size_t)pn * sizeof(double));
        for (int r = 1; r <= R; ++r) {
            double* q = refine(p, pn, r, -nu + 1, nu, f->h, nu, &n);
            free(p);
            p = q;
            pn = n;
        }
        v = p;
        n = pn;
        *support_left = -nu + 1;
    } else {
        if (nu < 2 || m < 0 || m >= nu) return -fail("bad edge function request");
        if (kind == 1) {
            v = cascade_left(f->h, f->phi, f->E[0], f->A[0], f->B[0], nu, R, m, &n);
            *support_left = 0;
        } else { /* reflect the left construction of the reversed filter (302-310) */
            double hr[2 * ORC_MAX_NU], pr[2 * ORC_MAX_NU];
            for (int i = 0; i < 2 * nu; ++i) hr[i] = f->h[2 * nu - 1 - i], pr[i] = f->phi[2 * nu - 1 - i];
            double* w = cascade_left(hr, pr, f->E[1], f->A[1], f->B[1], nu, R, m, &n);
            v = (double*)malloc((size_t)n * sizeof(double));
            for (long i = 0; i < n; ++i) v[i] = w[n - 1 - i];
            free(w);
            *support_left = -(nu + m);
        }
    }
    if (out) {
        if ((size_t)n > cap) {
            free(v);
            return -fail("cascade output buffer too small");
        }
        memcpy(out, v, (size_t)n * sizeof(double));
    }
    free(v);
    return n;
}

/* ---- DWT (wavelet.cpp:367-536) -------------------------------------------- */
static void level_periodic(const orc_filters* f, double* x, size_t n, int inverse, double* s) {
    size_t half = n / 2;
    int nu = f->nu;
    memset(s, 0, n * sizeof(double));
    for (size_t mm = 0; mm < half; ++mm) {
        if (!inverse) { /* 369-385 */
            double c = 0, d = 0;
            for (int u = -nu + 1; u <= nu; ++u) {
                size_t idx = (size_t)(((long long)(2 * mm) + u + 2 * (long long)n) % (long long)n);
                c += f->h[u + nu - 1] * x[idx];
                d += f->g[u + nu - 1] * x[idx];
            }
            s[mm] = c;
            s[half + mm] = d;
        } else { /* 387-400 */
            double c = x[mm], d = x[half + mm];
            for (int u = -nu + 1; u <= nu; ++u) {
                size_t idx = (size_t)(((long long)(2 * mm) + u + 2 * (long long)n) % (long long)n);
                s[idx] += f->h[u + nu - 1] * c + f->g[u + nu - 1] * d;
            }
        }
    }
    memcpy(x, s, n * sizeof(double));
}

/* One VMP step.  Edge rows m < nu use A (nu x nu) on the first nu samples and
 * the first 2m+1 columns of B on samples nu..nu+2m; the right edge is the
 * mirror image (index n-1-k, row half-1-m).  Interior rows use the 2nu-tap
 * filters (403-483). */
static void level_vmp(const orc_filters* f, double* x, size_t n, int inverse, double* s) {
    size_t half = n / 2;
    int nu = f->nu, W = 2 * nu - 1;
    memset(s, 0, n * sizeof(double));
    for (int band = 0; band < 2; ++band) {        /* scaling (A,B) then wavelet (Aw,Bw) */
        for (int e = 0; e < 2; ++e) {             /* left then right edge */
            const double* A = band ? f->Aw[e] : f->A[e];
            const double* B = band ? f->Bw[e] : f->B[e];
            size_t base = band ? half : 0;
            for (int m = 0; m < nu; ++m) {
                size_t row = e ? half - 1 - (size_t)m : (size_t)m;
                if (!inverse) {
                    double acc = 0.0;
                    for (int k = 0; k < nu; ++k) acc += A[m * nu + k] * x[e ? n - 1 - (size_t)k : (size_t)k];
                    for (int li = 0; li <= 2 * m; ++li) {
                        size_t l = (size_t)(nu + li);
                        acc += B[m * W + li] * x[e ? n - 1 - l : l];
                    }
                    s[base + row] = acc;
                } else {
                    double c = x[base + row];
                    for (int k = 0; k < nu; ++k) s[e ? n - 1 - (size_t)k : (size_t)k] += A[m * nu + k] * c;
                    for (int li = 0; li <= 2 * m; ++li) {
                        size_t l = (size_t)(nu + li);
                        s[e ? n - 1 - l : l] += B[m * W + li] * c;
                    }
                }
            }
        }
    }
    for (size_t mm = (size_t)nu; mm + (size_t)nu < half; ++mm) {
        if (!inverse) {
            double c = 0, d = 0;
            for (int u = -nu + 1; u <= nu; ++u) {
                size_t idx = (size_t)((long long)(2 * mm) + u);
                c += f->h[u + nu - 1] * x[idx];
                d += f->g[u + nu - 1] * x[idx];
            }
            s[mm] = c;
            s[half + mm] = d;
        } else {
            double c = x[mm], d = x[half + mm];
            for (int u = -nu + 1; u <= nu; ++u) {
                size_t idx = (size_t)((long long)(2 * mm) + u);
                s[idx] += f->h[u + nu - 1] * c + f->g[u + nu - 1] * d;
            }
        }
    }
    memcpy(x, s, n * sizeof(double));
}

/* multilevel, levels j..min_level+1 (Forward) or min_level+1..j (Inverse)
 * (dwt_apply, 487-514) */
int orc_dwt(const orc_filters* f, int boundary, unsigned j, double* data, int inverse,
            int min_level) {
    int j0 = min_level < 0 ? orc_min_level(f->nu) : min_level;
    if ((int)j < j0) return fail("dwt: j below the coarsest admissible level");
    if (boundary == 1 && f->nu < 2) return fail("dwt: vmp requires nu >= 2");
    size_t n = (size_t)1 << j;
    double* s = (double*)malloc(n * sizeof(double));
    if (!inverse) {
        for (int lev = (int)j; lev > j0; --lev) {
            if (boundary == 0) level_periodic(f, data, (size_t)1 << lev, 0, s);
            else level_vmp(f, data, (size_t)1 << lev, 0, s);
        }
    } else {
        for (int lev = j0 + 1; lev <= (int)j; ++lev) {
            if (boundary == 0) level_periodic(f, data, (size_t)1 << lev, 1, s);
            else level_vmp(f, data, (size_t)1 << lev, 1, s);
        }
    }
    free(s);
    return 0;
}

/* rows, then columns (dwt_apply_2d, 524-536) */
int orc_dwt2d(const orc_filters* f, int boundary, unsigned j, double* data, int inverse,
              int min_level) {
    size_t n = (size_t)1 << j;
    double* col = (double*)malloc(n * sizeof(double));
    int rc = 0;
    for (size_t r = 0; r < n && !rc; ++r) rc = orc_dwt(f, boundary, j, data + r * n, inverse, min_level);
    for (size_t c = 0; c < n && !rc; ++c) {
        for (size_t r = 0; r < n; ++r) col[r] = data[r * n + c];
        rc = orc_dwt(f, boundary, j, col, inverse, min_level);
        for (size_t r = 0; r < n; ++r) data[r * n + c] = col[r];
    }
    free(col);
    return rc;
}

/* ---- kernel table (kernel.cpp:14-77) -------------------------------------- */
/* composite trapezoid of the samples over [x0, x0+1) split into 2^q cells
 * (cell_masses, 14-29) */
static void cell_masses(const double* v, long vn, int sl, int R, long x0, int q, double* out) {
    long cells = 1l << q, per = 1l << (R - q), base = x0 * (1l << R), off = (long)sl * (1l << R);
    double h = ldexp(1.0, -R);
#define AT(g) ((((g) - off) >= 0 && ((g) - off) < vn) ? v[(g) - off] : 0.0)
    for (long c = 0; c < cells; ++c) {
        long st = base + c * per;
        double acc = 0.5 * (AT(st) + AT(st + per));
        for (long i = 1; i < per; ++i) acc += AT(st + i);
        out[c] = acc * h;
    }
#undef AT
}

int orc_kernel_table(const orc_filters* f, int boundary, int q, int R, double* interior,
                     double* left, double* right) {
    if (q < 1) return fail("kernel table requires q >= 1");
    if (f->nu < 2) return fail("kernel tables are for nu >= 2");
    if (R < q) return fail("kernel quadrature requires R >= q");
    int nu = f->nu;
    long S = 1l << q, W = 2 * nu - 1;
    int sl;
    long n = orc_cascade(f, 0, 0, R, NULL, 0, &sl);
    double* v = (double*)malloc((size_t)n * sizeof(double));
    orc_cascade(f, 0, 0, R, v, (size_t)n, &sl);
    memset(interior, 0, (size_t)(W * S) * sizeof(double));
    for (int l = -nu + 1; l <= nu - 1; ++l) {
        double* row = interior + (long)(l + nu - 1) * S;
        cell_masses(v, n, sl, R, l, q, row);
        orc_fwht_sequency(row, (size_t)S);
    }
    free(v);
    if (boundary == 1) {
        memset(left, 0, (size_t)(nu * W * S) * sizeof(double));
        memset(right, 0, (size_t)(nu * W * S) * sizeof(double));
        for (int m = 0; m < nu; ++m) {
            for (int side = 1; side <= 2; ++side) {
                n = orc_cascade(f, side, m, R, NULL, 0, &sl);
                v = (double*)malloc((size_t)n * sizeof(double));
                orc_cascade(f, side, m, R, v, (size_t)n, &sl);
                for (int t = 0; t <= nu - 1 + m; ++t) {
                    long x0 = side == 1 ? t : t - (nu + m); /* right: l' = t-(nu+m) */
                    double* row = (side == 1 ? left : right) + ((long)m * W + t) * S;
                    cell_masses(v, n, sl, R, x0, q, row);
                    orc_fwht_sequency(row, (size_t)S);
                }
                free(v);
            }
        }
    }
    return 0;
}

/* ---- FastOp + compositions (fastop.cpp:27-302) ----------------------------- */
typedef struct {
    uint64_t p;
    int col;
    long row; /* offset of the kappa row (2^q values) in op->ktab */
} edge_term;

struct orc_op {
    orc_filters f;
    int boundary, nu, dim, r0;
    unsigned j, q;
    double* ktab; /* interior | left | right, reference layout (kernel.hpp:23-38) */
    long kint, kleft, kright;
    edge_term* terms;
    long nterms;
};

static void add_term(orc_op* o, uint64_t p, long row, int col) {
    /* stable insertion by position (the grouping of fastop.cpp:85-97) */
    long i = o->nterms++;
    while (i > 0 && o->terms[i - 1].p > p) {
        o->terms[i] = o->terms[i - 1];
        --i;
    }
    o->terms[i].p = p;
    o->terms[i].col = col;
    o->terms[i].row = row;
}

/* Prop. 4.1 edge decomposition (build_edge_terms, fastop.cpp:54-98) */
static void build_edges(orc_op* o) {
    int nu = o->nu;
    long S = 1l << o->q, W = 2 * nu - 1;
    uint64_t M = 1ull << o->j;
    o->terms = (edge_term*)calloc((size_t)(4 * nu * W + 4), sizeof(edge_term));
    o->nterms = 0;
    if (o->boundary == 1) {
        for (int m = 0; m < nu; ++m)
            for (int l = 0; l <= nu - 1 + m; ++l) add_term(o, (uint64_t)l, o->kleft + (m * W + l) * S, m);
        for (int mb = 0; mb < nu; ++mb)
            for (int t = 0; t <= nu + mb - 1; ++t)
                add_term(o, M + (uint64_t)(t - (nu + mb)), o->kright + (mb * W + t) * S,
                         (int)M - 1 - mb);
    } else {
        for (int side = 0; side < 2; ++side)
            for (int k = 0; k < nu; ++k) {
                int col = side ? (int)M - nu + k : k;
                for (int l = -nu + 1; l <= nu - 1; ++l) {
                    long long pos = ((long long)col + l) % (long long)M;
                    if (pos < 0) pos += (long long)M;
                    add_term(o, (uint64_t)pos, o->kint + (l + nu - 1) * S, col);
                }
            }
    }
}

orc_op* orc_op_create(int family, int nu, int boundary, unsigned j, unsigned q, int dim,
                      int min_level, const char* data_dir) {
    if (nu < 1 || nu > ORC_MAX_NU) { fail("unsupported vanishing moments"); return NULL; }
    if (nu == 1 && boundary == 1) { fail("vmp boundary requires nu >= 2"); return NULL; }
    if (dim != 1 && dim != 2) { fail("dim must be 1 or 2"); return NULL; }
    if ((int)j < orc_min_level(nu)) { fail("j below the coarsest admissible level"); return NULL; }
    if (nu >= 2 && q < 1) { fail("q must be >= 1"); return NULL; }
    orc_op* o = (orc_op*)calloc(1, sizeof(orc_op));
    if (orc_load_filters(family, nu, data_dir, &o->f)) { free(o); return NULL; }
    o->boundary = boundary;
    o->nu = nu;
    o->dim = dim;
    o->j = j;
    o->q = q;
    o->r0 = min_level < 0 ? orc_min_level(nu) : min_level;
    if (o->r0 > (int)j) { fail("r0 above j"); free(o); return NULL; }
    if (nu >= 2) {
        long S = 1l << q, W = 2 * nu - 1;
        o->kint = 0;
        o->kleft = W * S;
        o->kright = W * S + nu * W * S;
        o->ktab = (double*)calloc((size_t)(W * S + 2 * nu * W * S), sizeof(double));
        if (orc_kernel_table(&o->f, boundary, (int)q, 14, o->ktab, o->ktab + o->kleft,
                             o->ktab + o->kright)) {
            free(o->ktab);
            free(o);
            return NULL;
        }
        build_edges(o);
    }
    return o;
}

void orc_op_destroy(orc_op* o) {
    if (!o) return;
    free(o->ktab);
    free(o->terms);
    free(o);
}

long orc_op_edge_terms(const orc_op* o, uint64_t* p, int* col, long* row, long cap) {
    for (long i = 0; i < o->nterms && i < cap; ++i) {
        p[i] = o->terms[i].p;
        col[i] = o->terms[i].col;
        row[i] = o->terms[i].row;
    }
    return o->nterms;
}

/* Alg. 1 forward: sum_l D_l(H_l(xi)) over interior columns, then the edge
 * columns position by position (forward_1d, fastop.cpp:100-137). */
static void fwd1(const orc_op* o, const double* xi, double* alpha) {
    size_t M = (size_t)1 << o->j, N = (size_t)1 << (o->j + o->q), S = (size_t)1 << o->q;
    unsigned bits = o->j + o->q;
    int nu = o->nu;
    double scale = 1.0 / sqrt((double)M);
    memset(alpha, 0, N * sizeof(double));
    double* scr = (double*)malloc(N * sizeof(double));
    for (int l = -nu + 1; l <= nu - 1 && M >= 2 * (size_t)nu + 1; ++l) {
        memset(scr, 0, N * sizeof(double));
        for (size_t m = (size_t)nu; m + (size_t)nu < M; ++m) scr[(size_t)((long long)m + l) << o->q] = xi[m];
        orc_fwht_natural(scr, N);
        const double* kr = o->ktab + o->kint + (long)(l + nu - 1) * (long)S;
        for (size_t n = 0; n < N; ++n) alpha[n] += scale * kr[n >> o->j] * scr[orc_seq_to_nat(n, bits)];
    }
    double* sign = (double*)malloc(M * sizeof(double));
    double cval[64];
    for (long t0 = 0; t0 < o->nterms;) {
        long t1 = t0;
        uint64_t p = o->terms[t0].p;
        for (size_t s = 0; s < S; ++s) cval[s] = 0.0;
        for (; t1 < o->nterms && o->terms[t1].p == p; ++t1)
            for (size_t s = 0; s < S; ++s) cval[s] += xi[o->terms[t1].col] * o->ktab[o->terms[t1].row + (long)s];
        orc_walsh_sign_row(p, o->j, sign);
        for (size_t s = 0; s < S; ++s) {
            double w = scale * cval[s];
            if ((p & 1) && (s & 1)) w = -w;
            if (w == 0.0) continue;
            for (size_t r = 0; r < M; ++r) alpha[s * M + r] += w * sign[r];
        }
        t0 = t1;
    }
    free(sign);
    free(scr);
}

/* transpose of fwd1 (adjoint_1d, fastop.cpp:139-175) */
static void adj1(const orc_op* o, const double* alpha, double* xi) {
    size_t M = (size_t)1 << o->j, N = (size_t)1 << (o->j + o->q), S = (size_t)1 << o->q;
    unsigned bits = o->j + o->q;
    int nu = o->nu;
    double scale = 1.0 / sqrt((double)M);
    memset(xi, 0, M * sizeof(double));
    double* scr = (double*)malloc(N * sizeof(double));
    for (int l = -nu + 1; l <= nu - 1 && M >= 2 * (size_t)nu + 1; ++l) {
        const double* kr = o->ktab + o->kint + (long)(l + nu - 1) * (long)S;
        for (size_t n = 0; n < N; ++n) scr[n] = scale * kr[n >> o->j] * alpha[n];
        orc_fwht_natural(scr, N);
        for (size_t m = (size_t)nu; m + (size_t)nu < M; ++m)
            xi[m] += scr[orc_seq_to_nat((size_t)((long long)m + l) << o->q, bits)];
    }
    double* sign = (double*)malloc(M * sizeof(double));
    double tp[64];
    for (long t0 = 0; t0 < o->nterms;) {
        uint64_t p = o->terms[t0].p;
        orc_walsh_sign_row(p, o->j, sign);
        for (size_t s = 0; s < S; ++s) {
            double acc = 0.0;
            for (size_t r = 0; r < M; ++r) acc += alpha[s * M + r] * sign[r];
            if ((p & 1) && (s & 1)) acc = -acc;
            tp[s] = scale * acc;
        }
        long t1 = t0;
        for (; t1 < o->nterms && o->terms[t1].p == p; ++t1) {
            double acc = 0.0;
            for (size_t s = 0; s < S; ++s) acc += o->ktab[o->terms[t1].row + (long)s] * tp[s];
            xi[o->terms[t1].col] += acc;
        }
        t0 = t1;
    }
    free(sign);
    free(scr);
}

/* Haar composition for nu = 1 (HaarFullRankOp fastop.cpp:285-302
 * generalised to r0 and q): IDWT -> sequency FWHT -> 1/sqrt(M); rows >= M are 0. */
static void haar_fwd(const orc_op* o, const double* x, double* y, int use_idwt) {
    size_t M = (size_t)1 << o->j, N = (size_t)1 << (o->j + o->q);
    double* v = (double*)malloc(M * sizeof(double));
    memcpy(v, x, M * sizeof(double));
    if (use_idwt) orc_dwt(&o->f, 0, o->j, v, 1, o->r0);
    orc_fwht_sequency(v, M);
    double scale = 1.0 / sqrt((double)M);
    for (size_t i = 0; i < M; ++i) y[i] = scale * v[i];
    for (size_t i = M; i < N; ++i) y[i] = 0.0;
    free(v);
}

static void haar_adj(const orc_op* o, const double* y, double* x, int use_idwt) {
    size_t M = (size_t)1 << o->j;
    memcpy(x, y, M * sizeof(double));
    orc_fwht_sequency(x, M);
    double scale = 1.0 / sqrt((double)M);
    for (size_t i = 0; i < M; ++i) x[i] *= scale;
    if (use_idwt) orc_dwt(&o->f, 0, o->j, x, 0, o->r0);
}

/* alpha = G xi G^T: rows, then columns (forward_2d, fastop.cpp:196-210) */
static void fwd2(const orc_op* o, const double* xi, double* alpha) {
    size_t M = (size_t)1 << o->j, N = (size_t)1 << (o->j + o->q);
    double* tmp = (double*)malloc(M * N * sizeof(double));
    double *col = (double*)malloc(M * sizeof(double)), *out = (double*)malloc(N * sizeof(double));
    for (size_t r = 0; r < M; ++r) fwd1(o, xi + r * M, tmp + r * N);
    for (size_t c = 0; c < N; ++c) {
        for (size_t r = 0; r < M; ++r) col[r] = tmp[r * N + c];
        fwd1(o, col, out);
        for (size_t r = 0; r < N; ++r) alpha[r * N + c] = out[r];
    }
    free(tmp), free(col), free(out);
}

/* xi = G^T alpha G: columns, then rows (adjoint_2d, fastop.cpp:212-227) */
static void adj2(const orc_op* o, const double* alpha, double* xi) {
    size_t M = (size_t)1 << o->j, N = (size_t)1 << (o->j + o->q);
    double* tmp = (double*)malloc(M * N * sizeof(double));
    double *col = (double*)malloc(N * sizeof(double)), *out = (double*)malloc(M * sizeof(double));
    for (size_t c = 0; c < N; ++c) {
        for (size_t r = 0; r < N; ++r) col[r] = alpha[r * N + c];
        adj1(o, col, out);
        for (size_t r = 0; r < M; ++r) tmp[r * N + c] = out[r];
    }
    for (size_t r = 0; r < M; ++r) adj1(o, tmp + r * N, xi + r * M);
    free(tmp), free(col), free(out);
}

/* ComposedOp with a full mask (fastop.cpp:241-281), with min_level = r0. */
int orc_op_forward(orc_op* o, const double* z, double* y, int use_idwt) {
    if (o->nu == 1) {
        if (o->dim != 1) return fail("Haar composition is 1D only");
        haar_fwd(o, z, y, use_idwt);
        return 0;
    }
    size_t M = (size_t)1 << o->j, n_in = o->dim == 1 ? M : M * M;
    double* x = (double*)malloc(n_in * sizeof(double));
    memcpy(x, z, n_in * sizeof(double));
    int rc = 0;
    if (use_idwt)
        rc = o->dim == 1 ? orc_dwt(&o->f, o->boundary, o->j, x, 1, o->r0)
                         : orc_dwt2d(&o->f, o->boundary, o->j, x, 1, o->r0);
    if (!rc) {
        if (o->dim == 1) fwd1(o, x, y);
        else fwd2(o, x, y);
    }
    free(x);
    return rc;
}

int orc_op_adjoint(orc_op* o, const double* y, double* z, int use_idwt) {
    if (o->nu == 1) {
        if (o->dim != 1) return fail("Haar composition is 1D only");
        haar_adj(o, y, z, use_idwt);
        return 0;
    }
    if (o->dim == 1) adj1(o, y, z);
    else adj2(o, y, z);
    if (!use_idwt) return 0;
    return o->dim == 1 ? orc_dwt(&o->f, o->boundary, o->j, z, 0, o->r0)
                       : orc_dwt2d(&o->f, o->boundary, o->j, z, 0, o->r0);
}

/* ---- seeded inputs -------------------------------------------------------- */
/* test_rng: splitmix-style seed, xorshift 13/7/17, multiplier, 53-bit
 * uniform, Box-Muller normal (proj/tests/test_util.hpp:10-27) */
typedef struct { uint64_t s; } rng_t;
static void rng_init(rng_t* r, uint64_t seed) { r->s = seed * 0x9E3779B97F4A7C15ull + 1; }
static uint64_t rng_u64(rng_t* r) {
    r->s ^= r->s << 13;
    r->s ^= r->s >> 7;
    r->s ^= r->s << 17;
    return r->s * 0x2545F4914F6CDD1Dull;
}
static double rng_uniform(rng_t* r) { return (double)(rng_u64(r) >> 11) * 0x1.0p-53; }
static double rng_normal(rng_t* r) {
    double u1 = rng_uniform(r), u2 = rng_uniform(r);
    if (u1 < 1e-300) u1 = 1e-300;
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

void orc_rng_normals(uint64_t seed, double* out, size_t n) {
    rng_t r;
    rng_init(&r, seed);
    for (size_t i = 0; i < n; ++i) out[i] = rng_normal(&r);
}

/* wavelet level of 1D index i: r0 for the coarse block and the first detail
 * band, floor(log2 i) above */
static int level_of(uint64_t i, int r0) {
    if (i < (2ull << r0)) return r0;
    int l = 0;
    while ((i >> (l + 1)) != 0) ++l;
    return l;
}

/* kind 0: N(0,1); kind 1: N(0,1) * 2^-level (level(r,c) = max of the two in
 * 2D).  density < 1: only round(density * n) entries nonzero, positions drawn
 * first by a partial Fisher-Yates shuffle (index = i + u64 % (n - i)), then
 * the values in that order; the rest are 0. */
int orc_synth(int kind, uint64_t seed, unsigned j, int r0, double density, int dim,
              double* out) {
    size_t side = (size_t)1 << j, n = dim == 2 ? side * side : side;
    rng_t r;
    rng_init(&r, seed);
    size_t k = density >= 1.0 ? n : (size_t)llround(density * (double)n);
    uint32_t* idx = NULL;
    if (k < n) {
        idx = (uint32_t*)malloc(n * sizeof(uint32_t));
        for (size_t i = 0; i < n; ++i) idx[i] = (uint32_t)i;
        for (size_t i = 0; i < k; ++i) {
            size_t t = i + (size_t)(rng_u64(&r) % (uint64_t)(n - i));
            uint32_t tmp = idx[i];
            idx[i] = idx[t];
            idx[t] = tmp;
        }
        memset(out, 0, n * sizeof(double));
    }
    for (size_t i = 0; i < k; ++i) {
        size_t pos = idx ? idx[i] : i;
        double v = rng_normal(&r);
        if (kind == 1) {
            int lev = dim == 2 ? (level_of(pos / side, r0) > level_of(pos % side, r0)
                                      ? level_of(pos / side, r0)
                                      : level_of(pos % side, r0))
                               : level_of(pos, r0);
            v = ldexp(v, -lev);
        }
        out[pos] = v;
    }
    free(idx);
    return 0;
}
