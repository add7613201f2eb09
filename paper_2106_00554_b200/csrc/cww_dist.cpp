// Multi-GPU entry points of the C ABI.
//
// The reference's only parallelism is the std::thread fan-out of
// FastOp::forward_2d / adjoint_2d over rows and columns
// (/root/reference/proj/src/fastop.cpp:179-192, parallel_for).  On one
// 8 x B200 box the work shards two ways:
//
//   cww_multi_*  independent vectors / images (configs 2-4): the batch is split
//                into contiguous shards, one per device, each run by its own
//                host thread through the single-device host API (no data-path
//                collective).  One process drives every listed device.
//   cww_dist_*   one image too large to want on one GPU (config 5): rows are
//                partitioned over P ranks (one process per GPU, NCCL
//                communicator); every separable pass is followed by a
//                distributed transpose = local rectangular transpose (the
//                blocks bound for rank q become contiguous) -> grouped
//                ncclSend / ncclRecv of P blocks of (M/P)^2 doubles over
//                NVLink / NVSwitch -> unpack kernel (local row i = the
//                concatenation of the received blocks' row i).
//
// NCCL is resolved at run time (dlopen of libnccl.so.2: inside a PyTorch
// process this is the already-loaded torch NCCL), so the library has no link
// dependency on it and single-GPU use never touches it.  A "local" dist
// handle simulates P ranks inside one process on one device with the same
// pack / unpack kernels and a device-copy exchange (the tests' oracle check
// of the partition logic on a single GPU: no rank ever waits on another).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdarg>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/cww_b200.h"
#include "cww_launch.h"

namespace {

cww_status err(cww_status st, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
cww_status err(cww_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    return cww::set_error(st, buf);
}

#define DCUDA(expr)                                                                                 \
    do {                                                                                            \
        cudaError_t e_ = (expr);                                                                    \
        if (e_ != cudaSuccess) return err(CWW_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
    } while (0)

struct Nccl {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
    static Nccl api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
            return;
        }
        auto sym = [&](const char* n) { return dlsym(h, n); };
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
        api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
        api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
        api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.GroupStart && api.GroupEnd &&
                 api.Send && api.Recv && api.GetErrorString;
        if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
    });
    return api;
}

#define DNCCL(expr)                                                                                   \
    do {                                                                                              \
        ncclResult_t r_ = (expr);                                                                     \
        if (r_ != ncclSuccess) return err(CWW_ERR_NCCL, "%s: %s", #expr, nccl().GetErrorString(r_)); \
    } while (0)

}  // namespace

struct cww_dist {
    cww_op* op = nullptr;  // 1D operator on the image rows (desc with dim = 1)
    int rank = 0, P = 1, device = 0;
    long long M = 0, m = 0;  // image side, rows per rank
    bool local = false;      // P virtual ranks in this process (device-copy exchange)
    ncclComm_t comm = nullptr;
    std::vector<double*> send, recv;  // per (virtual) rank: P blocks of m x m
    double* work = nullptr;           // cww_normal work buffer (unused by the banded form)
    size_t work_len = 0;
};

struct cww_multi {
    std::vector<cww_op*> ops;  // one per listed device
    size_t nin = 0, nout = 0;
};

namespace {

cww_status dist_alloc(cww_dist* d) {
    const int nb = d->local ? d->P : 1;
    DCUDA(cudaSetDevice(d->device));
    for (int r = 0; r < nb; ++r) {
        double *s = nullptr, *q = nullptr;
        DCUDA(cudaMalloc(&s, size_t(d->P) * d->m * d->m * sizeof(double)));
        d->send.push_back(s);
        DCUDA(cudaMalloc(&q, size_t(d->P) * d->m * d->m * sizeof(double)));
        d->recv.push_back(q);
    }
    size_t ni = 0, no = 0;
    cww_op_sizes(d->op, &ni, &no);
    d->work_len = no * size_t(d->m);
    DCUDA(cudaMalloc(&d->work, d->work_len * sizeof(double)));
    return CWW_OK;
}

cww_status dist_common(const cww_op_desc* desc, int nranks, cww_dist* d) {
    if (!desc) return err(CWW_ERR_INVALID_ARG, "null desc");
    if (desc->dim != 2) return err(CWW_ERR_UNSUPPORTED, "row-partitioned operator: desc.dim must be 2");
    if (desc->mask && desc->mask_len) return err(CWW_ERR_UNSUPPORTED, "row-partitioned operator: full mask only");
    if (nranks < 1) return err(CWW_ERR_INVALID_ARG, "nranks must be >= 1");
    d->M = 1ll << desc->j;
    d->P = nranks;
    if (d->M % nranks != 0 || d->M / nranks < 2)
        return err(CWW_ERR_DIMENSION, "M = %lld rows do not split into %d ranks of >= 2", d->M, nranks);
    d->m = d->M / nranks;
    cww_op_desc d1 = *desc;
    d1.dim = 1;  // the separable passes are the 1D operator on rows
    cww_status s = cww_op_create(&d1, &d->op);
    if (s != CWW_OK) return s;
    cudaGetDevice(&d->device);
    if (desc->device >= 0) d->device = desc->device;
    return CWW_OK;
}

// rows x of every (virtual) rank <- the same rows of the transposed image
cww_status dist_transpose(cww_dist* d, double* const* xs, cudaStream_t st) {
    const long long m = d->m, M = d->M, blk = m * m;
    const int nb = d->local ? d->P : 1;
    for (int r = 0; r < nb; ++r)  // pack: the blocks bound for rank q become contiguous (and transposed)
        DCUDA(cww::launch_transpose_rect(xs[r], d->send[size_t(r)], m, M, 1, st));
    if (d->local) {
        for (int r = 0; r < d->P; ++r)
            for (int q = 0; q < d->P; ++q)
                DCUDA(cudaMemcpyAsync(d->recv[size_t(q)] + r * blk, d->send[size_t(r)] + q * blk,
                                      size_t(blk) * sizeof(double), cudaMemcpyDeviceToDevice, st));
    } else {
        Nccl& n = nccl();
        DNCCL(n.GroupStart());
        for (int q = 0; q < d->P; ++q) {
            DNCCL(n.Send(d->send[0] + q * blk, size_t(blk), ncclFloat64, q, d->comm, st));
            DNCCL(n.Recv(d->recv[0] + q * blk, size_t(blk), ncclFloat64, q, d->comm, st));
        }
        DNCCL(n.GroupEnd());
    }
    for (int r = 0; r < nb; ++r) DCUDA(cww::launch_unpack_blocks(d->recv[size_t(r)], xs[r], m, d->P, st));
    cww::note_launches(2 * nb);  // pack transposes + unpacks
    return CWW_OK;
}

cww_status dist_rows_normal(cww_dist* d, double* const* xs, cudaStream_t st) {
    const int nb = d->local ? d->P : 1;
    const size_t n = size_t(d->m) * size_t(d->M);
    for (int r = 0; r < nb; ++r) {
        cww_status s = cww_normal(d->op, xs[r], n, d->work, d->work_len, size_t(d->m), 1, st);
        if (s != CWW_OK) return s;
    }
    return CWW_OK;
}

// x <- (U*U)^iters x with A*A = N1 (x) N1: per iteration N1 on
// the local rows, a distributed transpose, N1 on the local rows again (the
// result is transposed); an odd count ends with one transpose back.
cww_status dist_normal(cww_dist* d, double* const* xs, int iters, cudaStream_t st) {
    if (iters < 0) return err(CWW_ERR_INVALID_ARG, "iters must be >= 0");
    DCUDA(cudaSetDevice(d->device));
    for (int it = 0; it < iters; ++it) {
        cww_status s = dist_rows_normal(d, xs, st);
        if (s == CWW_OK) s = dist_transpose(d, xs, st);
        if (s == CWW_OK) s = dist_rows_normal(d, xs, st);
        if (s != CWW_OK) return s;
    }
    if (iters & 1) return dist_transpose(d, xs, st);
    return CWW_OK;
}

}  // namespace

extern "C" {

cww_status cww_nccl_unique_id(unsigned char* id, size_t len) {
    if (!id || len < NCCL_UNIQUE_ID_BYTES) return err(CWW_ERR_INVALID_ARG, "id buffer must hold 128 bytes");
    Nccl& n = nccl();
    if (!n.ok) return err(CWW_ERR_NCCL, "%s", n.why.c_str());
    ncclUniqueId u;
    DNCCL(n.GetUniqueId(&u));
    std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
    return CWW_OK;
}

cww_status cww_dist_create(const cww_op_desc* desc, int rank, int nranks, const unsigned char* id, size_t id_len,
                           cww_dist** out) {
    if (!out) return err(CWW_ERR_INVALID_ARG, "null out");
    *out = nullptr;
    if (!id || id_len < NCCL_UNIQUE_ID_BYTES) return err(CWW_ERR_INVALID_ARG, "NCCL unique id (128 bytes) required");
    if (rank < 0 || rank >= nranks) return err(CWW_ERR_INVALID_ARG, "rank %d outside [0, %d)", rank, nranks);
    Nccl& n = nccl();
    if (!n.ok) return err(CWW_ERR_NCCL, "%s", n.why.c_str());
    auto* d = new cww_dist;
    d->rank = rank;
    cww_status s = dist_common(desc, nranks, d);
    if (s == CWW_OK) {
        ncclUniqueId u;
        std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
        cudaSetDevice(d->device);
        ncclResult_t r = n.CommInitRank(&d->comm, nranks, u, rank);
        if (r != ncclSuccess) s = err(CWW_ERR_NCCL, "ncclCommInitRank: %s", n.GetErrorString(r));
    }
    if (s == CWW_OK) s = dist_alloc(d);
    if (s != CWW_OK) {
        cww_dist_destroy(d);
        return s;
    }
    *out = d;
    return CWW_OK;
}

cww_status cww_dist_create_local(const cww_op_desc* desc, int nranks, cww_dist** out) {
    if (!out) return err(CWW_ERR_INVALID_ARG, "null out");
    *out = nullptr;
    auto* d = new cww_dist;
    d->local = true;
    cww_status s = dist_common(desc, nranks, d);
    if (s == CWW_OK) s = dist_alloc(d);
    if (s != CWW_OK) {
        cww_dist_destroy(d);
        return s;
    }
    *out = d;
    return CWW_OK;
}

cww_status cww_dist_destroy(cww_dist* d) {
    if (!d) return CWW_OK;
    cudaSetDevice(d->device);
    for (double* p : d->send) cudaFree(p);
    for (double* p : d->recv) cudaFree(p);
    if (d->work) cudaFree(d->work);
    if (d->comm) nccl().CommDestroy(d->comm);
    if (d->op) cww_op_destroy(d->op);
    delete d;
    return CWW_OK;
}

cww_status cww_dist_rows(const cww_dist* d, size_t* rows_per_rank, size_t* row_len) {
    if (!d) return err(CWW_ERR_INVALID_ARG, "null handle");
    if (rows_per_rank) *rows_per_rank = size_t(d->m);
    if (row_len) *row_len = size_t(d->M);
    return CWW_OK;
}

cww_status cww_dist_normal(cww_dist* d, double* x_rows, size_t len, int iters, void* stream) {
    if (!d || !x_rows) return err(CWW_ERR_INVALID_ARG, "null argument");
    if (d->local) return err(CWW_ERR_INVALID_ARG, "local handle: use cww_dist_normal_local");
    if (len != size_t(d->m) * size_t(d->M)) return err(CWW_ERR_DIMENSION, "normal: dimension mismatch");
    double* xs[1] = {x_rows};
    return dist_normal(d, xs, iters, static_cast<cudaStream_t>(stream));
}

cww_status cww_dist_normal_local(cww_dist* d, double* const* x_rows, size_t len, int iters, void* stream) {
    if (!d || !x_rows) return err(CWW_ERR_INVALID_ARG, "null argument");
    if (!d->local) return err(CWW_ERR_INVALID_ARG, "NCCL handle: use cww_dist_normal");
    if (len != size_t(d->m) * size_t(d->M)) return err(CWW_ERR_DIMENSION, "normal: dimension mismatch");
    for (int r = 0; r < d->P; ++r)
        if (!x_rows[r]) return err(CWW_ERR_INVALID_ARG, "null rows of rank %d", r);
    return dist_normal(d, x_rows, iters, static_cast<cudaStream_t>(stream));
}

cww_status cww_multi_create(const cww_op_desc* desc, int ndev, const int* devices, cww_multi** out) {
    if (!desc || !out || ndev < 1 || !devices) return err(CWW_ERR_INVALID_ARG, "null argument or ndev < 1");
    *out = nullptr;
    auto* mu = new cww_multi;
    for (int i = 0; i < ndev; ++i) {
        cww_op_desc di = *desc;
        di.device = devices[i];
        cww_op* op = nullptr;
        cww_status s = cww_op_create(&di, &op);
        if (s != CWW_OK) {
            cww_multi_destroy(mu);
            return s;
        }
        mu->ops.push_back(op);
    }
    cww_op_sizes(mu->ops[0], &mu->nin, &mu->nout);
    *out = mu;
    return CWW_OK;
}

cww_status cww_multi_destroy(cww_multi* mu) {
    if (!mu) return CWW_OK;
    for (cww_op* op : mu->ops) cww_op_destroy(op);
    delete mu;
    return CWW_OK;
}

static cww_status multi_call(const cww_multi* mu, const double* in, size_t in_len, double* out, size_t out_len,
                             size_t batch, bool adj) {
    if (!mu || ((!in || !out) && batch)) return err(CWW_ERR_INVALID_ARG, "null argument");
    const size_t ni = adj ? mu->nout : mu->nin, no = adj ? mu->nin : mu->nout;
    if (in_len != ni * batch || out_len != no * batch)
        return err(CWW_ERR_DIMENSION, "%s: dimension mismatch", adj ? "adjoint" : "forward");
    const size_t P = mu->ops.size();
    std::vector<cww_status> st(P, CWW_OK);
    std::vector<std::string> msg(P);
    std::vector<std::thread> th;
    for (size_t r = 0; r < P; ++r) {
        // shard_batch: contiguous shards, the first batch % P one vector longer
        const size_t base = batch / P, rem = batch % P;
        const size_t start = r * base + std::min(r, rem), cnt = base + (r < rem ? 1 : 0);
        if (cnt == 0) continue;
        th.emplace_back([&, r, start, cnt] {
            cww_op* op = mu->ops[r];
            st[r] = adj ? cww_adjoint_host(op, in + start * ni, cnt * ni, out + start * no, cnt * no, cnt)
                        : cww_forward_host(op, in + start * ni, cnt * ni, out + start * no, cnt * no, cnt);
            if (st[r] != CWW_OK) msg[r] = cww_last_error();
        });
    }
    for (auto& t : th) t.join();
    for (size_t r = 0; r < P; ++r)
        if (st[r] != CWW_OK) return err(st[r], "device shard %zu: %s", r, msg[r].c_str());
    return CWW_OK;
}

cww_status cww_multi_forward_host(const cww_multi* mu, const double* x, size_t x_len, double* y, size_t y_len,
                                  size_t batch) {
    return multi_call(mu, x, x_len, y, y_len, batch, false);
}

cww_status cww_multi_adjoint_host(const cww_multi* mu, const double* y, size_t y_len, double* x, size_t x_len,
                                  size_t batch) {
    return multi_call(mu, y, y_len, x, x_len, batch, true);
}

}  // extern "C"
