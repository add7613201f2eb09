// Header-only C++ veneer over the C ABI (cww_b200.h) with the reference
// library's operator shapes, so reference C++ callers (dense_from_fastop,
// FastOpLinear users, the intended CG / PBDW / CS solvers) switch by changing
// the namespace:
//
//   reference (proj/include/cww/fastop.hpp)        here
//   struct LinearOp { rows, cols, forward, adjoint } cww_b200::LinearOp     (fastop.hpp:14-31)
//   class FastOp(filters, spec, j, q, kernels, dim) cww_b200::FastOp(spec, j, q, dim)  (:44-92)
//   class ComposedOp(op, mask, use_idwt)           cww_b200::ComposedOp(op, [mask,] use_idwt, r0) (:114-127)
//   struct SamplingMask                             cww_b200::SamplingMask (:33-39)
//   class HaarFullRankOp(j)                        cww_b200::HaarFullRankOp(j)  (:131-142)
//   CwwError                                       cww_b200::CwwError (wavelet.hpp:11-13)
//
// forward/adjoint(span, span) take HOST spans (staged through the GPU,
// synchronous, like the reference); forward_device/adjoint_device take
// device pointers and a stream (asynchronous, the fast path).
#pragma once
#include <cstddef>
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "cww_b200.h"

namespace cww_b200 {

struct CwwError : std::runtime_error {
    cww_status status;
    CwwError(cww_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

inline void check(cww_status s) {
    if (s != CWW_OK) throw CwwError(s, cww_last_error());
}

enum class Family { Daubechies = CWW_DAUBECHIES, Symlet = CWW_SYMLET };
enum class Boundary { Periodic = CWW_PERIODIC, Vmp = CWW_VMP };

struct WaveletSpec {
    Family family = Family::Daubechies;
    int nu = 2;
    Boundary boundary = Boundary::Vmp;
    int min_level() const {
        if (nu == 1) return 0;
        int j = 0;
        while ((1 << j) < 2 * nu) ++j;
        return j;
    }
};

// SamplingMask (fastop.hpp:33-39): sorted, unique output indices; empty = full.
struct SamplingMask {
    std::vector<std::uint64_t> indices;
    static SamplingMask full(std::uint64_t) { return {}; }
    std::size_t size() const { return indices.size(); }
};

struct LinearOp {
    virtual ~LinearOp() = default;
    virtual std::size_t rows() const = 0;
    virtual std::size_t cols() const = 0;
    virtual void forward(std::span<const double> x, std::span<double> y) const = 0;
    virtual void adjoint(std::span<const double> y, std::span<double> x) const = 0;
    std::vector<double> forward_copy(std::span<const double> x) const {
        std::vector<double> y(rows());
        forward(x, y);
        return y;
    }
    std::vector<double> adjoint_copy(std::span<const double> y) const {
        std::vector<double> x(cols());
        adjoint(y, x);
        return x;
    }
};

// One handle (FastOp when use_idwt = 0, ComposedOp when 1).
class Op : public LinearOp {
public:
    Op(const WaveletSpec& s, unsigned j, unsigned q, int dim, bool use_idwt, int min_level = -1,
       const char* data_dir = nullptr, int device = -1, const SamplingMask* mask = nullptr) {
        cww_op_desc d;
        cww_op_desc_init(&d);
        d.family = int(s.family);
        d.nu = s.nu;
        d.boundary = int(s.boundary);
        d.j = j;
        d.q = q;
        d.dim = dim;
        d.min_level = min_level;
        d.use_idwt = use_idwt ? 1 : 0;
        d.device = device;
        d.data_dir = data_dir;
        if (mask && !mask->indices.empty()) {
            d.mask = mask->indices.data();
            d.mask_len = mask->indices.size();
        }
        cww_op* h = nullptr;
        check(cww_op_create(&d, &h));
        h_.reset(h, [](cww_op* p) { cww_op_destroy(p); });
        check(cww_op_sizes(h, &in_, &out_));
    }
    std::size_t rows() const override { return out_; }
    std::size_t cols() const override { return in_; }
    std::size_t input_size() const { return in_; }
    std::size_t output_size() const { return out_; }
    void forward(std::span<const double> x, std::span<double> y) const override {
        check(cww_forward_host(h_.get(), x.data(), x.size(), y.data(), y.size(), x.size() / in_));
    }
    void adjoint(std::span<const double> y, std::span<double> x) const override {
        check(cww_adjoint_host(h_.get(), y.data(), y.size(), x.data(), x.size(), y.size() / out_));
    }
    // device pointers, `batch` vectors, cudaStream_t passed as void*
    void forward_device(const double* x, double* y, std::size_t batch, void* stream) const {
        check(cww_forward(h_.get(), x, batch * in_, y, batch * out_, batch, stream));
    }
    void adjoint_device(const double* y, double* x, std::size_t batch, void* stream) const {
        check(cww_adjoint(h_.get(), y, batch * out_, x, batch * in_, batch, stream));
    }
    // pinned host buffers: chunk-pipelined H2D / compute / D2H behind `stream` (no sync)
    void forward_host_async(const double* x, double* y, std::size_t batch, void* stream) const {
        check(cww_forward_host_async(h_.get(), x, batch * in_, y, batch * out_, batch, stream));
    }
    void adjoint_host_async(const double* y, double* x, std::size_t batch, void* stream) const {
        check(cww_adjoint_host_async(h_.get(), y, batch * out_, x, batch * in_, batch, stream));
    }
    // x <- (A* A)^iters x on device memory (banded normal form for full masks)
    void normal_device(double* x, std::size_t batch, int iters, void* stream) const {
        check(cww_normal(h_.get(), x, batch * in_, nullptr, 0, batch, iters, stream));
    }
    const cww_op* handle() const { return h_.get(); }

private:
    std::shared_ptr<cww_op> h_;
    std::size_t in_ = 0, out_ = 0;
};

class FastOp : public Op {
public:
    FastOp(const WaveletSpec& s, unsigned j, unsigned q, int dim = 1)
        : Op(s, j, q, dim, false), spec_(s), j_(j), q_(q), dim_(dim) {}
    void forward_1d(std::span<const double> x, std::span<double> y) const { forward(x, y); }
    void adjoint_1d(std::span<const double> y, std::span<double> x) const { adjoint(y, x); }
    void forward_2d(std::span<const double> x, std::span<double> y) const { forward(x, y); }
    void adjoint_2d(std::span<const double> y, std::span<double> x) const { adjoint(y, x); }
    void set_threads(int) {}
    const WaveletSpec& spec() const { return spec_; }
    unsigned j() const { return j_; }
    unsigned q() const { return q_; }
    int dim() const { return dim_; }

private:
    WaveletSpec spec_;
    unsigned j_, q_;
    int dim_;
};

class ComposedOp : public Op {
public:
    // full sampling mask; r0 (min_level) -1 = the spec's J0 as in the reference
    ComposedOp(const FastOp& op, bool use_idwt = true, int min_level = -1)
        : Op(op.spec(), op.j(), op.q(), op.dim(), use_idwt, min_level) {}
    // ComposedOp(op, SamplingMask, use_idwt) (fastop.hpp:116): rows() = mask size
    ComposedOp(const FastOp& op, const SamplingMask& mask, bool use_idwt, int min_level = -1)
        : Op(op.spec(), op.j(), op.q(), op.dim(), use_idwt, min_level, nullptr, -1, &mask) {}
};

class HaarFullRankOp : public Op {
public:
    explicit HaarFullRankOp(unsigned j, unsigned q = 0, int min_level = 0)
        : Op(WaveletSpec{Family::Daubechies, 1, Boundary::Periodic}, j, q, 1, true, min_level) {}
};

}  // namespace cww_b200
