/*
 * cww_b200 -- C ABI of the B200-native Walsh->wavelet change-of-basis operator.
 *
 * Drop-in boundary for the reference library's hot path (reference sources
 * under /root/reference/proj):
 *
 *   reference (C++, proj/include/cww/fastop.hpp)            this ABI
 *   ---------------------------------------------------------------------------
 *   FastOp(filters, spec, j, q, kernels, dim)   :46-47     cww_op_create(desc{use_idwt=0})
 *   ComposedOp(op, SamplingMask::full, true)    :114-127   cww_op_create(desc{use_idwt=1})
 *   HaarFullRankOp(j)                           :131-142   cww_op_create(desc{nu=1, q=0})
 *   LinearOp::rows()/cols(), FastOp::
 *     input_size()/output_size()                :16-17,57-58 cww_op_sizes
 *   FastOp::forward / forward_1d / forward_2d   :62-69     cww_forward   (device pointers)
 *   FastOp::adjoint / adjoint_1d / adjoint_2d   :63-72     cww_adjoint   (device pointers)
 *   LinearOp::forward(span, span) (host spans)  :18        cww_forward_host
 *   LinearOp::adjoint(span, span) (host spans)  :19        cww_adjoint_host
 *   dwt_apply / dwt_apply_2d (wavelet.hpp)      :115-129   cww_dwt
 *   fwht_sequency / fwht_natural (walsh.hpp)    :53-58     cww_fwht
 *   sequency_to_natural_index (walsh.hpp)       :60-62     cww_sequency_perm
 *   walsh_sign_row (walsh.hpp)                  :66        cww_walsh_sign_rows
 *   compute_kernel_table (kernel.hpp)           :46-47     cww_op_kernel_table
 *   save/load_kernel_table, get_kernel_table    :49-60     cww_kernel_table_save/_load, desc.cache_dir
 *   CwwError (std::runtime_error) thrown        wavelet.hpp:11-13  -> cww_status + cww_last_error()
 *
 * All arithmetic is IEEE fp64.  Batches are batch-major and contiguous: item b
 * of a forward input starts at x + b*input_size.  Outputs are fully
 * overwritten (as fastop.cpp:103,142).  The handle is immutable after create,
 * so concurrent calls on distinct streams are safe (the reference's const-pure
 * forward/adjoint).  There is no CPU fallback: every entry point
 * that computes runs hand-written sm_100a kernels and fails with
 * CWW_ERR_CUDA when no CUDA device is usable.
 */
#ifndef CWW_B200_H
#define CWW_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    CWW_OK = 0,
    CWW_ERR_INVALID_ARG = 1, /* null pointer, bad enum                       */
    CWW_ERR_DIMENSION = 2,   /* "dimension mismatch" (fastop.cpp:102,141,...) */
    CWW_ERR_SPEC = 3,        /* invalid spec / j / q (fastop.cpp:31-45)        */
    CWW_ERR_DATA_IO = 4,     /* filter-data or kernel-cache file errors        */
    CWW_ERR_CUDA = 5,        /* CUDA runtime error or no device                */
    CWW_ERR_NCCL = 6,
    CWW_ERR_UNSUPPORTED = 7,
    CWW_ERR_INTERNAL = 8,
    CWW_ERR_NOT_CONVERGED = 9, /* gs_solve / cs_solve: no convergence at max_iters  */
    CWW_ERR_INFEASIBLE = 10    /* cs_solve: eta below the least-squares residual    */
} cww_status;

typedef enum { CWW_DAUBECHIES = 0, CWW_SYMLET = 1 } cww_family;       /* wavelet.hpp:15 */
typedef enum { CWW_PERIODIC = 0, CWW_VMP = 1 } cww_boundary;          /* wavelet.hpp:16 */
typedef enum { CWW_DWT_FORWARD = 0, CWW_DWT_INVERSE = 1 } cww_dwt_dir; /* wavelet.hpp:111 */

typedef struct {
    int family;            /* cww_family                                        */
    int nu;                /* vanishing moments 1..6 (1 = Haar, periodic only)  */
    int boundary;          /* cww_boundary                                      */
    unsigned j;            /* M = 2^j                                           */
    unsigned q;            /* N = 2^(j+q); q >= 1 for nu >= 2, q >= 0 for Haar  */
    int dim;               /* 1 or 2                                            */
    int min_level;         /* coarsest DWT level r0 of the composition; -1 = J0 */
    int use_idwt;          /* 1: ComposedOp (U W^-1 / W U*); 0: FastOp (U / U*) */
    int kernel_resolution; /* cascade/quadrature resolution R; 0 = 14           */
    int device;            /* CUDA device ordinal; -1 = current                 */
    const char* data_dir;  /* CWWF directory; NULL = $CWW_DATA_DIR or built-in  */
    /* Sampling mask P_Omega of ComposedOp(op, SamplingMask, use_idwt)
     * (fastop.hpp:33-39, fastop.cpp:12-25, 231-281): sorted, unique output
     * indices (host memory, copied at create).  NULL / mask_len == output
     * size = full mask.  A subsampled op has output_size = mask_len: forward
     * gathers the masked rows, adjoint scatters into zeros first. */
    const uint64_t* mask;
    size_t mask_len;
    /* Kernel-table cache directory (get_kernel_table, kernel.cpp:173-198):
     * NULL/"" = $CWW_CACHE_DIR, else no cache.  A valid matching CWWK file is
     * loaded instead of recomputing the table; otherwise the table is computed
     * and written back. */
    const char* cache_dir;
    /* 1: run the kernel-table cascade (kernel.cpp:31-77) on the GPU; the
     * table is bit-identical to the host computation (separately rounded
     * products and sums in the host's order). */
    int gpu_kernel_table;
    /* I/O precision: CWW_FP64 (cww_forward / cww_adjoint on
     * double buffers) or CWW_FP32 (cww_forward_f32 / cww_adjoint_f32 on float
     * buffers; the arithmetic stays fp64, the results are rounded to fp32 once
     * on output: relative error ~1e-7 against the fp64 path). */
    int precision;
} cww_op_desc;

typedef enum { CWW_FP64 = 0, CWW_FP32 = 1 } cww_precision;

typedef struct cww_op cww_op;

/* thread-local description of the last error on this thread */
const char* cww_last_error(void);
const char* cww_version(void);

void cww_op_desc_init(cww_op_desc* d);
cww_status cww_op_create(const cww_op_desc* desc, cww_op** out);
cww_status cww_op_destroy(cww_op* op);
cww_status cww_op_sizes(const cww_op* op, size_t* input_size, size_t* output_size);

/* Device-pointer entry points (the measured path).  x: batch*input_size,
 * y: batch*output_size doubles in device memory; stream = cudaStream_t
 * (NULL = legacy default stream).  Asynchronous with respect to the host. */
cww_status cww_forward(const cww_op* op, const double* x, size_t x_len, double* y,
                       size_t y_len, size_t batch, void* stream);
cww_status cww_adjoint(const cww_op* op, const double* y, size_t y_len, double* x,
                       size_t x_len, size_t batch, void* stream);
/* fp32 I/O (ops created with desc.precision = CWW_FP32): float device
 * buffers, batch-major as above; converted to fp64 on entry and rounded to
 * fp32 on exit around the fp64 kernels. */
cww_status cww_forward_f32(const cww_op* op, const float* x, size_t x_len, float* y, size_t y_len,
                           size_t batch, void* stream);
cww_status cww_adjoint_f32(const cww_op* op, const float* y, size_t y_len, float* x, size_t x_len,
                           size_t batch, void* stream);
/* x <- (U* U)^iters x  (adjoint(forward(x)) repeated; the normal operator
 * of a least-squares / CG loop).  work: NULL or batch*output_size doubles. */
cww_status cww_normal(const cww_op* op, double* x, size_t x_len, double* work,
                      size_t work_len, size_t batch, int iters, void* stream);

/* Kernel-table cache files (CWWK, kernel.cpp:79-164; device-free).  save:
 * compute the table of (family, nu, boundary, q, R; R <= 0 = 14) from the
 * filter data and write it (save_kernel_table).  load: read and validate
 * (CRC, magic, version, shapes -- the reference's messages); header[5] =
 * family, nu, boundary, q, R; counts[3] = interior/left/right lengths (always
 * written); arrays copied when non-NULL (CWW_ERR_DIMENSION if too small). */
cww_status cww_kernel_table_save(int family, int nu, int boundary, unsigned q, int resolution,
                                 const char* data_dir, const char* path);
cww_status cww_kernel_table_load(const char* path, int* header, double* interior, size_t ni, double* left,
                                 size_t nl, double* right, size_t nr, size_t* counts);

/* Least-squares reconstruction (generalised sampling, the reference spec's
 * gs_solve; its src/reconstruct.cpp is empty): CGLS on the
 * normal equations A* A x = A* y with A = this op (full or masked), for
 * `batch` independent systems (device pointers, batch-major).  Stops when
 * every system's relative normal-equation residual ||A*(y - A x)|| / ||A* y||
 * <= residual_tol (checked once per iteration), else returns
 * CWW_ERR_NOT_CONVERGED after max_iters with x = the last iterate.  use_x0:
 * start from the x passed in (else 0).  iters / residuals (batch doubles,
 * host) may be NULL. */
cww_status cww_gs_solve(const cww_op* op, const double* y, size_t y_len, double* x, size_t x_len,
                        size_t batch, double residual_tol, int max_iters, int use_x0, int* iters,
                        double* residuals, void* stream);

/* Compressed-sensing reconstruction (the reference spec's cs_solve, QCBP,
 * SPEC.md:421-429; its src/reconstruct.cpp is empty):
 *   min ||x||_1  subject to  ||A x - y||^2 <= eta
 * with A = this op (typically a masked ComposedOp), by the Chambolle-Pock
 * primal-dual iteration (step sizes from a power-iteration estimate of
 * ||A||), for `batch` independent systems (device pointers, batch-major),
 * starting from x = 0.  Stops when every system's relative iterate change
 * is <= tol and ||A x - y||^2 <= eta + tol ||y||^2 (checked every 20
 * iterations); otherwise CWW_ERR_INFEASIBLE when eta is below the
 * least-squares residual, else CWW_ERR_NOT_CONVERGED (x = last iterate).
 * residuals (batch doubles, host, may be NULL): ||A x - y||^2. */
cww_status cww_cs_solve(const cww_op* op, const double* y, size_t y_len, double* x, size_t x_len,
                        size_t batch, double eta, double tol, int max_iters, int* iters,
                        double* residuals, void* stream);

/* Host-pointer entry points: a literal drop-in for the reference's span API.
 * Stages through pinned buffers and synchronises before returning. */
cww_status cww_forward_host(const cww_op* op, const double* x, size_t x_len, double* y,
                            size_t y_len, size_t batch);
cww_status cww_adjoint_host(const cww_op* op, const double* y, size_t y_len, double* x,
                            size_t x_len, size_t batch);

/* Asynchronous host-pointer entry points for PINNED host buffers (cudaHostAlloc
 * / cudaHostRegister; pageable buffers take the synchronous path): the batch
 * is split into chunks whose host-to-device copy, compute and device-to-host
 * copy run on three streams, so copies in both PCIe directions overlap the
 * compute and each other.  Tiny transforms (input + output <= 256 KB,
 * small path only) skip the copies: the kernels read and
 * write the pinned buffers over PCIe directly (zero-copy).  Enqueued behind
 * `stream`, which is made to wait for the last copy; returns without
 * synchronising. */
cww_status cww_forward_host_async(const cww_op* op, const double* x, size_t x_len, double* y,
                                  size_t y_len, size_t batch, void* stream);
cww_status cww_adjoint_host_async(const cww_op* op, const double* y, size_t y_len, double* x,
                                  size_t x_len, size_t batch, void* stream);

/* Multilevel DWT (dir = CWW_DWT_FORWARD, analysis) or IDWT (CWW_DWT_INVERSE)
 * of `batch` device vectors (dim 1: 2^j, dim 2: 2^j x 2^j row-major), in
 * place, using the op's filters, boundary and min_level (dwt_apply,
 * wavelet.cpp:487-536). */
cww_status cww_dwt(const cww_op* op, double* data, size_t len, size_t batch, int dir,
                   void* stream);

/* In-place sequency-ordered (natural = 0) unnormalised FWHT of `batch`
 * device vectors of length n = 2^bits (walsh.cpp:81-98). */
cww_status cww_fwht(double* v, unsigned bits, size_t batch, int sequency, void* stream);

/* perm[n] = bit_reverse(gray(n), bits) for n < 2^bits, computed on the
 * device (the reference's FastOp::perm_ table, fastop.cpp:47-50). */
cww_status cww_sequency_perm(unsigned bits, uint32_t* perm_dev, void* stream);

/* signs[i*2^j + r] = w_r(p_i / 2^j) for each of npos positions (device
 * buffers; walsh.cpp:123-131). */
cww_status cww_walsh_sign_rows(const uint64_t* p_dev, size_t npos, unsigned j,
                               double* signs_dev, void* stream);

/* Host copies of the op's Walsh-coefficient table, reference layout
 * (kernel.hpp:23-38): interior (2nu-1)*2^q; left, right nu*(2nu-1)*2^q (VMP). */
cww_status cww_op_kernel_table(const cww_op* op, double* interior, size_t n_interior,
                               double* left, size_t n_left, double* right, size_t n_right);
/* Edge terms (position p, column, kappa row offset into the table above)
 * grouped by position as fastop.cpp:54-98; returns the count in *n. */
cww_status cww_op_edge_terms(const cww_op* op, uint64_t* p, int32_t* col, int64_t* row,
                             size_t cap, size_t* n);

/* Seeded synthetic inputs (test_rng semantics of
 * proj/tests/test_util.hpp:10-27), host memory.  kind 0: N(0,1); kind 1:
 * N(0,1)*2^-level; density < 1: sparse.  n = 2^j (dim 1) or 4^j (dim 2). */
cww_status cww_synth(int kind, uint64_t seed, unsigned j, int r0, double density, int dim,
                     double* out);

/* ---- multi-GPU ------------------------------------------
 * The reference's only parallelism is the std::thread fan-out over rows and
 * columns of FastOp::forward_2d / adjoint_2d (fastop.cpp:179-192).
 *
 * Batch sharding over the devices of one box (independent vectors / images,
 * configs 2-4): one op per listed device; the *_host calls split the batch
 * into contiguous shards (the first batch % ndev one item longer), run each
 * on its device from its own host thread and return when all are done. */
typedef struct cww_multi cww_multi;
cww_status cww_multi_create(const cww_op_desc* desc, int ndev, const int* devices, cww_multi** out);
cww_status cww_multi_destroy(cww_multi* mu);
cww_status cww_multi_forward_host(const cww_multi* mu, const double* x, size_t x_len, double* y,
                                  size_t y_len, size_t batch);
cww_status cww_multi_adjoint_host(const cww_multi* mu, const double* y, size_t y_len, double* x,
                                  size_t x_len, size_t batch);

/* Row-partitioned 2D operator (config 5: one 2^j x 2^j image, rows split over
 * nranks processes, one GPU each).  desc.dim must be 2 (full mask).  Each
 * rank holds M/nranks consecutive rows (row-major, device memory on
 * desc.device).  The separable passes run locally on rows; every pass is
 * followed by a distributed transpose: local rectangular transpose (blocks
 * bound for rank q become contiguous) -> grouped ncclSend/ncclRecv of
 * nranks blocks of (M/nranks)^2 doubles -> unpack kernel.  NCCL is loaded at
 * run time (libnccl.so.2).  Bootstrap: rank 0 calls cww_nccl_unique_id, the
 * caller broadcasts the 128 bytes, every rank calls cww_dist_create. */
typedef struct cww_dist cww_dist;
cww_status cww_nccl_unique_id(unsigned char* id, size_t len);
cww_status cww_dist_create(const cww_op_desc* desc, int rank, int nranks, const unsigned char* id,
                           size_t id_len, cww_dist** out);
cww_status cww_dist_destroy(cww_dist* d);
/* rows_per_rank = M / nranks, row_len = M */
cww_status cww_dist_rows(const cww_dist* d, size_t* rows_per_rank, size_t* row_len);
/* x_rows <- this rank's rows of (U* U)^iters X (cww_normal of the whole image) */
cww_status cww_dist_normal(cww_dist* d, double* x_rows, size_t len, int iters, void* stream);
/* The same partition and exchange with nranks virtual ranks inside one
 * process on one device (device-copy exchange instead of NCCL; every rank's
 * phase completes before the next phase starts): the partition logic on a
 * single GPU.  x_rows[r]: rank r's rows. */
cww_status cww_dist_create_local(const cww_op_desc* desc, int nranks, cww_dist** out);
cww_status cww_dist_normal_local(cww_dist* d, double* const* x_rows, size_t len, int iters, void* stream);

/* Instrumentation: when enabled, every kernel launch is bracketed by CUDA
 * events on its own stream; cww_profile_dump synchronises them and writes
 * {"<kernel>": [total_ms, launches], ...} (then clears the record).
 * cww_kernel_launches counts every kernel this library has launched. */
void cww_profile_enable(int on);
cww_status cww_profile_dump(char* json, size_t cap);
unsigned long long cww_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* CWW_B200_H */
