/* TEST INFRASTRUCTURE ONLY -- the CPU oracle (checker) for the Walsh->wavelet
 * change-of-basis hot path.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it; the product never links it.
 *
 * A plain-C restatement of the reference algorithm (citations are
 * /root/reference/proj paths).  Parity is pinned two ways ("Oracle"):
 *   - against the compiled reference itself (oracle/_ref/libcwwref.so, built
 *     by oracle/Makefile from the unmodified sources), and
 *   - against committed golden vectors tests/golden/ (npz files) produced by that
 *     reference (tests/golden/make_golden.py), plus the known-answer checks
 *     of the reference's own suites (proj/tests/test_walsh.cpp,
 *     proj/tests/test_wavelet.cpp) restated in tests/test_oracle.py.
 */
#ifndef CWW_ORACLE_H
#define CWW_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_NU 6

/* FilterSet (proj/include/cww/wavelet.hpp:51-69).  Edge matrices are row
 * major, nu x nu (A, Aw) or nu x (2nu-1) (E, B, Bw). */
typedef struct {
    int family; /* 0 Daubechies, 1 Symlet */
    int nu;
    double h[2 * ORC_MAX_NU];   /* hbar_u, u = -nu+1..nu */
    double g[2 * ORC_MAX_NU];   /* gbar_u */
    double phi[2 * ORC_MAX_NU]; /* phi(k), k = -nu+1..nu */
    double E[2][ORC_MAX_NU * (2 * ORC_MAX_NU - 1)];
    double A[2][ORC_MAX_NU * ORC_MAX_NU];
    double B[2][ORC_MAX_NU * (2 * ORC_MAX_NU - 1)];
    double Aw[2][ORC_MAX_NU * ORC_MAX_NU];
    double Bw[2][ORC_MAX_NU * (2 * ORC_MAX_NU - 1)];
} orc_filters; /* index [0] = left edge, [1] = right edge */

const char* orc_last_error(void);

uint32_t orc_crc32(const void* data, size_t len);
int orc_min_level(int nu);
int orc_load_filters(int family, int nu, const char* data_dir, orc_filters* out);

/* walsh.hpp */
uint64_t orc_seq_to_nat(uint64_t n, unsigned bits);
int orc_walsh_eval(uint64_t n, uint64_t p, unsigned j);
void orc_walsh_sign_row(uint64_t p, unsigned j, double* sign);
int orc_fwht_natural(double* v, size_t n);
int orc_fwht_sequency(double* v, size_t n);

/* wavelet.hpp: cascade samples of the interior (kind 0), left (1) or right
 * (2) scaling function; returns the sample count, fills *support_left. */
long orc_cascade(const orc_filters* f, int kind, int m, int R, double* out, size_t cap,
                 int* support_left);
int orc_dwt(const orc_filters* f, int boundary, unsigned j, double* data, int inverse,
            int min_level);
int orc_dwt2d(const orc_filters* f, int boundary, unsigned j, double* data, int inverse,
              int min_level);

/* kernel.hpp */
int orc_kernel_table(const orc_filters* f, int boundary, int q, int R, double* interior,
                     double* left, double* right);

/* fastop.hpp: an operator handle (FastOp + the ComposedOp/Haar compositions) */
typedef struct orc_op orc_op;
orc_op* orc_op_create(int family, int nu, int boundary, unsigned j, unsigned q, int dim,
                      int min_level, const char* data_dir);
void orc_op_destroy(orc_op* op);
int orc_op_forward(orc_op* op, const double* x, double* y, int use_idwt);
int orc_op_adjoint(orc_op* op, const double* y, double* x, int use_idwt);
/* edge terms after the reference's grouping by position (fastop.cpp:54-98):
 * writes up to cap (p, col, table-row offset) triples; returns the count. */
long orc_op_edge_terms(const orc_op* op, uint64_t* p, int* col, long* row, long cap);

/* test_rng semantics (proj/tests/test_util.hpp:10-27) and the seeded
 * synthetic inputs of SURVEY.md section 8d. */
void orc_rng_normals(uint64_t seed, double* out, size_t n);
int orc_synth(int kind, uint64_t seed, unsigned j, int r0, double density, int dim,
              double* out);

#ifdef __cplusplus
}
#endif
#endif
