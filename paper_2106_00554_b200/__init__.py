"""B200-native Walsh -> wavelet change-of-basis operator (arXiv 2106.00554).

Python host side mirroring the reference C++ library's operator interface
(/root/reference/proj/include/cww/fastop.hpp, wavelet.hpp, walsh.hpp) over
the C ABI in include/cww_b200.h (libcww_b200.so, hand-written sm_100a CUDA):

    reference                                   here
    ------------------------------------------  -----------------------------------
    WaveletSpec{family, nu, boundary}           WaveletSpec(family, nu, boundary)
    FastOp(filters, spec, j, q, kernels, dim)   FastOp(spec, j, q, dim)
    FastOp::forward/adjoint(span, span)         FastOp.forward(x, y=None) / .adjoint
    FastOp::forward_1d/_2d, adjoint_1d/_2d      same names
    ComposedOp(op, SamplingMask::full, true)    ComposedOp(op, mask=None, use_idwt=True,
                                                           min_level=None)
    HaarFullRankOp(j)                           HaarFullRankOp(j)
    dwt_apply / dwt_apply_2d                    dwt_apply / dwt_apply_2d
    fwht_sequency / fwht_natural                fwht_sequency / fwht_natural
    sequency_to_natural_index, walsh_sign_row   sequency_perm / walsh_sign_rows
    compute_kernel_table                        FastOp.kernel_table()
    CwwError                                    CwwError

Inputs may be CUDA tensors (float64; the device path, on torch's current
stream) or host arrays (numpy; staged through pinned buffers, a literal
drop-in for the reference's span API).  A leading batch dimension is
accepted.  There is no CPU fallback: without the built library or a CUDA
device every compute call raises CwwError.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from typing import Optional

import numpy as np

__all__ = [
    "CwwError", "Family", "Boundary", "WaveletSpec", "parse_wavelet_name", "LinearOp", "FastOp",
    "FastOpLinear", "ComposedOp", "HaarFullRankOp", "SamplingMask", "dwt_apply", "dwt_apply_2d",
    "fwht_sequency", "fwht_natural", "sequency_perm", "walsh_sign_rows", "synth", "library_path",
    "profile_enable", "profile_dump", "kernel_launches",
]

_PKG = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_PKG, os.environ.get("CWW_LIB_NAME", "libcww_b200.so"))
DATA_DIR = os.path.join(_PKG, "data")


class CwwError(RuntimeError):
    """Mirror of the reference's CwwError (wavelet.hpp:11-13) carrying the C status."""

    def __init__(self, msg: str, status: int = 8):
        super().__init__(msg)
        self.status = status


class Family(enum.IntEnum):
    Daubechies = 0
    Symlet = 1


class Boundary(enum.IntEnum):
    Periodic = 0
    Vmp = 1


class _Desc(C.Structure):
    _fields_ = [("family", C.c_int), ("nu", C.c_int), ("boundary", C.c_int), ("j", C.c_uint),
                ("q", C.c_uint), ("dim", C.c_int), ("min_level", C.c_int), ("use_idwt", C.c_int),
                ("kernel_resolution", C.c_int), ("device", C.c_int), ("data_dir", C.c_char_p),
                ("mask", C.c_void_p), ("mask_len", C.c_size_t), ("cache_dir", C.c_char_p),
                ("gpu_kernel_table", C.c_int), ("precision", C.c_int)]


_lib = None


def library_path() -> str:
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise CwwError(f"CUDA library not built: {_LIB_PATH} (run paper_2106_00554_b200/build.py)", 5)
    L = C.CDLL(_LIB_PATH)
    vp, sz, dp = C.c_void_p, C.c_size_t, C.c_void_p
    L.cww_last_error.restype = C.c_char_p
    L.cww_version.restype = C.c_char_p
    L.cww_op_create.argtypes = [C.POINTER(_Desc), C.POINTER(vp)]
    L.cww_op_destroy.argtypes = [vp]
    L.cww_op_sizes.argtypes = [vp, C.POINTER(sz), C.POINTER(sz)]
    for name in ("cww_forward", "cww_adjoint"):
        getattr(L, name).argtypes = [vp, dp, sz, dp, sz, sz, vp]
    for name in ("cww_forward_host", "cww_adjoint_host"):
        getattr(L, name).argtypes = [vp, dp, sz, dp, sz, sz]
    L.cww_normal.argtypes = [vp, dp, sz, dp, sz, sz, C.c_int, vp]
    L.cww_forward_host_async.argtypes = [vp, dp, sz, dp, sz, sz, vp]
    L.cww_forward_f32.argtypes = [vp, dp, sz, dp, sz, sz, vp]
    L.cww_adjoint_f32.argtypes = [vp, dp, sz, dp, sz, sz, vp]
    L.cww_adjoint_host_async.argtypes = [vp, dp, sz, dp, sz, sz, vp]
    L.cww_gs_solve.argtypes = [vp, dp, sz, dp, sz, sz, C.c_double, C.c_int, C.c_int,
                               C.POINTER(C.c_int), dp, vp]
    L.cww_cs_solve.argtypes = [vp, dp, sz, dp, sz, sz, C.c_double, C.c_double, C.c_int,
                               C.POINTER(C.c_int), dp, vp]
    L.cww_dwt.argtypes = [vp, dp, sz, sz, C.c_int, vp]
    L.cww_fwht.argtypes = [dp, C.c_uint, sz, C.c_int, vp]
    L.cww_sequency_perm.argtypes = [C.c_uint, dp, vp]
    L.cww_walsh_sign_rows.argtypes = [dp, sz, C.c_uint, dp, vp]
    L.cww_op_kernel_table.argtypes = [vp, dp, sz, dp, sz, dp, sz]
    L.cww_op_edge_terms.argtypes = [vp, dp, dp, dp, sz, C.POINTER(sz)]
    L.cww_synth.argtypes = [C.c_int, C.c_uint64, C.c_uint, C.c_int, C.c_double, C.c_int, dp]
    L.cww_profile_enable.argtypes = [C.c_int]
    L.cww_profile_dump.argtypes = [C.c_char_p, sz]
    L.cww_kernel_launches.restype = C.c_ulonglong
    _lib = L
    return L


def _check(rc: int):
    if rc != 0:
        raise CwwError(_load().cww_last_error().decode(), rc)


def _torch():
    import torch  # noqa: PLC0415  (torch is plumbing: device memory + streams)
    return torch


def _is_tensor(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def _stream_ptr(t) -> int:
    torch = _torch()
    return torch.cuda.current_stream(t.device).cuda_stream


def _np_ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# ---------------------------------------------------------------------------
class WaveletSpec:
    """WaveletSpec (wavelet.hpp:18-29): family, vanishing moments, boundary."""

    def __init__(self, family: Family = Family.Daubechies, nu: int = 2,
                 boundary: Boundary = Boundary.Vmp):
        self.family = Family(family)
        self.nu = int(nu)
        self.boundary = Boundary(boundary)

    def min_level(self) -> int:
        """ceil(log2(2 nu)) for nu >= 2, 0 for Haar (wavelet.cpp:16-21)."""
        if self.nu == 1:
            return 0
        j = 0
        while (1 << j) < 2 * self.nu:
            j += 1
        return j

    def name(self) -> str:
        return ("db" if self.family == Family.Daubechies else "sym") + str(self.nu)

    def boundary_name(self) -> str:
        return "periodic" if self.boundary == Boundary.Periodic else "vmp"

    def validate(self) -> None:
        """wavelet.cpp:31-39"""
        if self.nu < 1 or self.nu > 6:
            raise CwwError(f"unsupported vanishing moments: {self.nu} (supported: 1..6)", 3)
        if self.nu == 1 and self.boundary == Boundary.Vmp:
            raise CwwError("vmp boundary requires nu >= 2 (Haar has no boundary functions)", 3)
        if self.nu == 1 and self.family == Family.Symlet:
            raise CwwError("sym1 is identical to Haar; use db1", 3)

    def __repr__(self):
        return f"WaveletSpec({self.name()}, {self.boundary_name()})"


def parse_wavelet_name(name: str, boundary: Boundary) -> WaveletSpec:
    """wavelet.cpp:41-58"""
    if name in ("haar", "db1"):
        spec = WaveletSpec(Family.Daubechies, 1, boundary)
    elif name.startswith("db"):
        spec = WaveletSpec(Family.Daubechies, int(name[2:]), boundary)
    elif name.startswith("sym"):
        spec = WaveletSpec(Family.Symlet, int(name[3:]), boundary)
    else:
        raise CwwError("unknown wavelet name: " + name, 3)
    spec.validate()
    return spec


class SamplingMask:
    """SamplingMask (fastop.hpp:33-39): sorted, unique output indices Omega.
    full(n) is the identity (fastop.cpp:12-17); validate(n) raises like the
    reference (fastop.cpp:19-25).  A subsampled ComposedOp gathers the masked
    rows on the GPU (forward) and scatters into zeros (adjoint)."""

    def __init__(self, indices=None, n: Optional[int] = None):
        self.indices = None if indices is None else np.ascontiguousarray(indices, dtype=np.uint64)
        self.n = n

    @staticmethod
    def full(n: int) -> "SamplingMask":
        return SamplingMask(None, n)

    def size(self) -> int:
        return int(self.n) if self.indices is None else int(self.indices.size)

    def validate(self, n: int) -> None:
        if self.indices is None:
            return
        idx = self.indices
        if idx.size and int(idx.max()) >= n:
            raise CwwError("sampling mask index out of range", 3)
        if idx.size > 1 and not np.all(idx[1:] > idx[:-1]):
            raise CwwError("sampling mask indices must be sorted and unique", 3)

    def is_full(self, n: int) -> bool:
        if self.indices is None:
            return True
        return self.indices.size == n and np.array_equal(self.indices, np.arange(n, dtype=np.uint64))


class LinearOp:
    """LinearOp (fastop.hpp:14-31): rows/cols and forward/adjoint."""

    def rows(self) -> int:
        raise NotImplementedError

    def cols(self) -> int:
        raise NotImplementedError

    def forward_copy(self, x):
        return self.forward(x)

    def adjoint_copy(self, y):
        return self.adjoint(y)


class _Handle:
    def __init__(self, spec: WaveletSpec, j: int, q: int, dim: int, min_level: int, use_idwt: bool,
                 kernel_resolution: int = 0, device: Optional[int] = None,
                 data_dir: Optional[str] = None, mask: Optional[np.ndarray] = None,
                 cache_dir: Optional[str] = None, gpu_kernel_table: bool = False, precision: str = "fp64"):
        L = _load()
        m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint64)
        d = _Desc(int(spec.family), spec.nu, int(spec.boundary), j, q, dim, min_level,
                  1 if use_idwt else 0, kernel_resolution, -1 if device is None else device,
                  (data_dir or DATA_DIR).encode(), None if m is None else m.ctypes.data,
                  0 if m is None else m.size, None if cache_dir is None else cache_dir.encode(),
                  1 if gpu_kernel_table else 0, 1 if precision == "fp32" else 0)
        self.fp32 = precision == "fp32"
        h = C.c_void_p()
        _check(L.cww_op_create(C.byref(d), C.byref(h)))
        self.h = h
        self.L = L
        self.device = device
        if device is None:  # the op lives on the device that was current at creation
            try:
                import torch
                self.device = torch.cuda.current_device() if torch.cuda.is_available() else None
            except ImportError:  # pragma: no cover
                pass
        self._inflight = []  # (event, inp, out) of asynchronous pinned-host calls
        ni, no = C.c_size_t(), C.c_size_t()
        _check(L.cww_op_sizes(h, C.byref(ni), C.byref(no)))
        self.nin, self.nout = ni.value, no.value

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            self.L.cww_op_destroy(h)
            self.h = None

    def _apply(self, inp, out, adjoint: bool):
        nin, nout = (self.nout, self.nin) if adjoint else (self.nin, self.nout)
        if self.fp32:  # fp32 I/O: float32 CUDA tensors (cww_*_f32)
            torch = _torch()
            if not (_is_tensor(inp) and inp.is_cuda and inp.dtype == torch.float32):
                raise CwwError("fp32 op: expected a float32 CUDA tensor", 1)
            inp = inp.contiguous()
            if inp.numel() % nin:
                raise CwwError(("adjoint" if adjoint else "forward") + ": dimension mismatch", 2)
            batch = inp.numel() // nin
            shape = (nout,) if inp.dim() == 1 else tuple(inp.shape[:-1]) + (nout,)
            if out is None:
                out = torch.empty(shape, dtype=torch.float32, device=inp.device)
            fn = self.L.cww_adjoint_f32 if adjoint else self.L.cww_forward_f32
            _check(fn(self.h, inp.data_ptr(), inp.numel(), out.data_ptr(), out.numel(), batch, _stream_ptr(inp)))
            return out
        if _is_tensor(inp):
            torch = _torch()
            if (not inp.is_cuda and inp.is_pinned() and _is_tensor(out) and not out.is_cuda and out.is_pinned()
                    and inp.dtype == torch.float64 and out.dtype == torch.float64 and inp.is_contiguous()
                    and out.is_contiguous()):
                # pinned host tensors: chunk-pipelined copies / compute, asynchronous on the
                # current CUDA stream (cww_*_host_async); synchronise before reading `out`
                if inp.numel() % nin or out.numel() != (inp.numel() // nin) * nout:
                    raise CwwError(("adjoint" if adjoint else "forward") + ": dimension mismatch", 2)
                batch = inp.numel() // nin
                fn = self.L.cww_adjoint_host_async if adjoint else self.L.cww_forward_host_async
                dev = torch.device("cuda", self.device) if self.device is not None else torch.device("cuda")
                stream = torch.cuda.current_stream(dev)
                _check(fn(self.h, inp.data_ptr(), inp.numel(), out.data_ptr(), out.numel(), batch,
                          stream.cuda_stream))
                # torch's pinned-memory allocator does not see this use: keep both
                # buffers alive until the stream has finished with them
                if not torch.cuda.is_current_stream_capturing():
                    self._inflight = [r for r in self._inflight if not r[0].query()]
                    ev = torch.cuda.Event()
                    ev.record(stream)
                    self._inflight.append((ev, inp, out))
                return out
            if not inp.is_cuda:
                inp = inp.detach().numpy()
            else:
                if inp.dtype != torch.float64:
                    raise CwwError("expected a float64 tensor", 1)
                inp = inp.contiguous()
                if inp.numel() % nin:
                    raise CwwError(("adjoint" if adjoint else "forward") + ": dimension mismatch", 2)
                batch = inp.numel() // nin
                shape = (nout,) if inp.dim() == 1 else tuple(inp.shape[:-1]) + (nout,)
                if out is None:
                    out = torch.empty(shape, dtype=torch.float64, device=inp.device)
                elif not (out.is_cuda and out.dtype == torch.float64 and out.is_contiguous()):
                    raise CwwError("output must be a contiguous float64 CUDA tensor", 1)
                fn = self.L.cww_adjoint if adjoint else self.L.cww_forward
                _check(fn(self.h, inp.data_ptr(), inp.numel(), out.data_ptr(), out.numel(), batch,
                          _stream_ptr(inp)))
                return out
        a = np.ascontiguousarray(inp, dtype=np.float64)
        if a.size % nin:
            raise CwwError(("adjoint" if adjoint else "forward") + ": dimension mismatch", 2)
        batch = a.size // nin
        shape = (nout,) if a.ndim <= 1 else tuple(a.shape[:-1]) + (nout,)
        o = np.empty(shape, dtype=np.float64) if out is None else out
        if not (isinstance(o, np.ndarray) and o.dtype == np.float64 and o.flags.c_contiguous):
            raise CwwError("output must be a contiguous float64 array", 1)
        fn = self.L.cww_adjoint_host if adjoint else self.L.cww_forward_host
        _check(fn(self.h, _np_ptr(a), a.size, _np_ptr(o), o.size, batch))
        return o


class FastOp:
    """P_N U P_M and its adjoint (fastop.hpp:41-92) on the GPU.

    FastOp(spec, j, q, dim=1): M = 2^j wavelet-side scaling coefficients, N =
    2^(j+q) sequency-ordered Walsh coefficients.  The reference's explicit
    FilterSet / KernelTable arguments are built internally by the same
    algorithms (CWWF data, R = 14 cascade quadrature)."""

    def __init__(self, spec: WaveletSpec, j: int, q: int, dim: int = 1, *,
                 kernel_resolution: int = 0, device: Optional[int] = None,
                 data_dir: Optional[str] = None, cache_dir: Optional[str] = None,
                 gpu_kernel_table: bool = False, precision: str = "fp64"):
        spec.validate()
        if precision not in ("fp64", "fp32"):
            raise CwwError("precision must be 'fp64' or 'fp32'", 1)
        if spec.nu < 2:
            raise CwwError("FastOp requires nu >= 2; use HaarFullRankOp for Haar", 3)
        self._spec, self._j, self._q, self._dim = spec, int(j), int(q), int(dim)
        self._opts = dict(kernel_resolution=kernel_resolution, device=device, data_dir=data_dir,
                          cache_dir=cache_dir, gpu_kernel_table=gpu_kernel_table, precision=precision)
        self._h = _Handle(spec, self._j, self._q, self._dim, -1, False, **self._opts)

    def M(self) -> int:
        return 1 << self._j

    def N(self) -> int:
        return 1 << (self._j + self._q)

    def j(self) -> int:
        return self._j

    def q(self) -> int:
        return self._q

    def dim(self) -> int:
        return self._dim

    def spec(self) -> WaveletSpec:
        return self._spec

    def input_size(self) -> int:
        return self._h.nin

    def output_size(self) -> int:
        return self._h.nout

    def set_threads(self, t: int) -> None:  # fastop.hpp:60 -- the GPU ignores it
        pass

    def forward(self, x, y=None):
        return self._h._apply(x, y, False)

    def adjoint(self, y, x=None):
        return self._h._apply(y, x, True)

    def _dim_guard(self, want: int, what: str):
        if self._dim != want:
            raise CwwError(f"{what}: dimension mismatch", 2)

    def forward_1d(self, x, y=None):
        self._dim_guard(1, "forward_1d")
        return self.forward(x, y)

    def adjoint_1d(self, y, x=None):
        self._dim_guard(1, "adjoint_1d")
        return self.adjoint(y, x)

    def forward_2d(self, x, y=None):
        self._dim_guard(2, "forward_2d")
        return self.forward(x, y)

    def adjoint_2d(self, y, x=None):
        self._dim_guard(2, "adjoint_2d")
        return self.adjoint(y, x)

    def normal(self, x, iters: int = 1, work=None):
        """x <- (U* U)^iters x in place on a CUDA tensor (banded normal form)."""
        return _normal(self._h, x, iters, work)

    def kernel_table(self):
        """(interior, left, right) in the reference layout (kernel.hpp:23-38)."""
        nu, S = self._spec.nu, 1 << self._q
        W = 2 * nu - 1
        it = np.zeros(W * S)
        le = np.zeros(nu * W * S)
        ri = np.zeros(nu * W * S)
        _check(_load().cww_op_kernel_table(self._h.h, _np_ptr(it), it.size, _np_ptr(le), le.size,
                                           _np_ptr(ri), ri.size))
        return it, le, ri

    def edge_terms(self):
        """[(p, col, kappa row offset)] grouped by position (fastop.cpp:54-98)."""
        cap = 1024
        p = np.zeros(cap, np.uint64)
        col = np.zeros(cap, np.int32)
        row = np.zeros(cap, np.int64)
        n = C.c_size_t()
        _check(_load().cww_op_edge_terms(self._h.h, _np_ptr(p), _np_ptr(col), _np_ptr(row), cap,
                                         C.byref(n)))
        return [(int(p[i]), int(col[i]), int(row[i])) for i in range(n.value)]


class FastOpLinear(LinearOp):
    """fastop.hpp:94-109"""

    def __init__(self, op: FastOp):
        self.op = op

    def rows(self):
        return self.op.output_size()

    def cols(self):
        return self.op.input_size()

    def forward(self, x, y=None):
        return self.op.forward(x, y)

    def adjoint(self, y, x=None):
        return self.op.adjoint(y, x)


class ComposedOp(LinearOp):
    """z -> U W^-1 z and y -> W U* y (fastop.hpp:111-127, fastop.cpp:231-281),
    with the IDWT/DWT fused into the GPU operator.  min_level (r0) defaults to
    the spec's J0 as in the reference; the benchmark configs pass r0 = J0+1."""

    def __init__(self, op: FastOp, mask: Optional[SamplingMask] = None, use_idwt: bool = True,
                 min_level: Optional[int] = None):
        if mask is not None:
            mask.validate(op.output_size())
        self.op = op
        self.mask = mask
        self.use_idwt = bool(use_idwt)
        self.r0 = op.spec().min_level() if min_level is None else int(min_level)
        sub = mask is not None and not mask.is_full(op.output_size())
        self._h = _Handle(op.spec(), op.j(), op.q(), op.dim(), self.r0, self.use_idwt,
                          mask=mask.indices if sub else None, **op._opts)

    def rows(self):
        return self._h.nout

    def cols(self):
        return self._h.nin

    def forward(self, z, y=None):
        return self._h._apply(z, y, False)

    def adjoint(self, y, z=None):
        return self._h._apply(y, z, True)

    def normal(self, x, iters: int = 1, work=None):
        """x <- (A* A)^iters x in place on a CUDA tensor (the CG / least-squares
        inner loop; config 5).  work: optional output_size buffer."""
        return _normal(self._h, x, iters, work)

    def handle(self):
        return self._h


def _normal(h, x, iters, work):
    torch = _torch()
    if not (_is_tensor(x) and x.is_cuda and x.dtype == torch.float64 and x.is_contiguous()):
        raise CwwError("normal() needs a contiguous float64 CUDA tensor", 1)
    batch = x.numel() // h.nin
    wp, wn = (0, 0) if work is None else (work.data_ptr(), work.numel())
    _check(h.L.cww_normal(h.h, x.data_ptr(), x.numel(), wp, wn, batch, int(iters), _stream_ptr(x)))
    return x


class HaarFullRankOp(LinearOp):
    """The square Haar operator H W^-1 (fastop.hpp:129-142): Haar periodic IDWT
    (min_level 0), sequency FWHT, 1/sqrt(M).  Also generalises to the config-1
    composition (q >= 1, r0 >= 0), whose rows n >= M vanish."""

    def __init__(self, j: int, q: int = 0, min_level: int = 0, device: Optional[int] = None):
        self._j, self._q = int(j), int(q)
        spec = WaveletSpec(Family.Daubechies, 1, Boundary.Periodic)
        self._h = _Handle(spec, self._j, self._q, 1, int(min_level), True, device=device)

    def rows(self):
        return self._h.nout

    def cols(self):
        return self._h.nin

    def forward(self, x, y=None):
        return self._h._apply(x, y, False)

    def adjoint(self, y, x=None):
        return self._h._apply(y, x, True)

    def normal(self, x, iters: int = 1, work=None):
        """x <- (A* A)^iters x in place on a CUDA tensor."""
        return _normal(self._h, x, iters, work)

    def handle(self):
        return self._h


# ---------------------------------------------------------------------------
# free functions over device tensors
def gs_solve(op, y, residual_tol: float = 1e-10, max_iters: int = 1000, x0=None, raise_on_fail: bool = True):
    """Generalised-sampling least squares (SPEC.md gs_solve, min_z ||A z - y||
    with A = op): CGLS on A* A x = A* y on the GPU (cww_gs_solve), batched over
    the leading dimension of y (a contiguous float64 CUDA tensor).  Returns
    (x, iterations, relative normal-equation residuals).  Raises CwwError
    (status 9) when max_iters is reached above tolerance, unless raise_on_fail
    is False."""
    torch = _torch()
    h = op._h
    y = _dev_tensor(y, "gs_solve")
    if y.numel() % h.nout:
        raise CwwError("gs_solve: dimension mismatch", 2)
    batch = y.numel() // h.nout
    shape = (h.nin,) if y.dim() == 1 else tuple(y.shape[:-1]) + (h.nin,)
    if x0 is None:
        x = torch.empty(shape, dtype=torch.float64, device=y.device)
    else:
        x = _dev_tensor(x0, "gs_solve x0").clone()
    it = C.c_int(0)
    res = np.zeros(batch)
    rc = h.L.cww_gs_solve(h.h, y.data_ptr(), y.numel(), x.data_ptr(), x.numel(), batch,
                          float(residual_tol), int(max_iters), 0 if x0 is None else 1, C.byref(it),
                          _np_ptr(res), _stream_ptr(y))
    if rc != 0 and (raise_on_fail or rc != 9):
        _check(rc)
    return x, it.value, res


def cs_solve(op, y, eta: float, tol: float = 1e-8, max_iters: int = 20000, raise_on_fail: bool = True):
    """Compressed-sensing reconstruction (SPEC.md cs_solve, QCBP): min ||x||_1
    subject to ||A x - y||^2 <= eta with A = op (typically a masked
    ComposedOp), by Chambolle-Pock primal-dual iterations on the GPU
    (cww_cs_solve), batched over the leading dimension of y (a contiguous
    float64 CUDA tensor).  Returns (x, iterations, ||A x - y||^2 per system).
    Raises CwwError status 10 when eta is infeasible (below the least-squares
    residual) and status 9 at max_iters (unless raise_on_fail is False)."""
    torch = _torch()
    h = op._h
    y = _dev_tensor(y, "cs_solve")
    if y.numel() % h.nout:
        raise CwwError("cs_solve: dimension mismatch", 2)
    batch = y.numel() // h.nout
    shape = (h.nin,) if y.dim() == 1 else tuple(y.shape[:-1]) + (h.nin,)
    x = torch.empty(shape, dtype=torch.float64, device=y.device)
    it = C.c_int(0)
    res = np.zeros(batch)
    rc = h.L.cww_cs_solve(h.h, y.data_ptr(), y.numel(), x.data_ptr(), x.numel(), batch, float(eta), float(tol),
                          int(max_iters), C.byref(it), _np_ptr(res), _stream_ptr(y))
    if rc != 0 and (raise_on_fail or rc not in (9,)):
        _check(rc)
    return x, it.value, res


def kernel_table_save(spec: WaveletSpec, q: int, path: str, resolution: int = 14,
                      data_dir: Optional[str] = None) -> None:
    """save_kernel_table (kernel.cpp:95-117): compute the kappa tables of
    (spec, q, R) and write a CWWK cache file (host only, no device)."""
    L = _load()
    L.cww_kernel_table_save.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint, C.c_int, C.c_char_p, C.c_char_p]
    _check(L.cww_kernel_table_save(int(spec.family), spec.nu, int(spec.boundary), int(q), int(resolution),
                                   (data_dir or DATA_DIR).encode(), path.encode()))


def kernel_table_load(path: str) -> dict:
    """load_kernel_table (kernel.cpp:119-164): read and validate a CWWK file
    (CRC, magic, version, shapes).  Returns header fields and the arrays."""
    L = _load()
    dp, sz = C.c_void_p, C.c_size_t
    L.cww_kernel_table_load.argtypes = [C.c_char_p, C.POINTER(C.c_int), dp, sz, dp, sz, dp, sz,
                                        C.POINTER(C.c_size_t)]
    hdr = (C.c_int * 5)()
    cnt = (C.c_size_t * 3)()
    _check(L.cww_kernel_table_load(path.encode(), hdr, None, 0, None, 0, None, 0, cnt))
    it, le, ri = (np.empty(int(cnt[k])) for k in range(3))
    _check(L.cww_kernel_table_load(path.encode(), hdr, _np_ptr(it), it.size, _np_ptr(le), le.size,
                                   _np_ptr(ri), ri.size, cnt))
    return {"family": hdr[0], "nu": hdr[1], "boundary": hdr[2], "q": hdr[3], "R": hdr[4],
            "interior": it, "left": le, "right": ri}


def kernel_cache_filename(spec: WaveletSpec, q: int, resolution: int = 14) -> str:
    """kernel_cache_filename (kernel.cpp:161-165)."""
    return f"cwwk_{spec.name()}_{'periodic' if spec.boundary == Boundary.Periodic else 'vmp'}_q{q}_R{resolution}_v1.bin"


def _dev_tensor(v, what):
    torch = _torch()
    if not (_is_tensor(v) and v.is_cuda and v.dtype == torch.float64 and v.is_contiguous()):
        raise CwwError(f"{what}: expected a contiguous float64 CUDA tensor", 1)
    return v


def dwt_apply(spec: WaveletSpec, j: int, data, inverse: bool, min_level: int = -1, dim: int = 1):
    """In-place multilevel DWT / IDWT of CUDA tensor `data` (wavelet.cpp:487-536);
    a leading batch dimension is allowed."""
    data = _dev_tensor(data, "dwt_apply")
    h = _Handle(spec, j, 0 if spec.nu == 1 else 1, dim, min_level, True)
    batch = data.numel() // h.nin
    _check(h.L.cww_dwt(h.h, data.data_ptr(), data.numel(), batch, 1 if inverse else 0,
                       _stream_ptr(data)))
    return data


def dwt_apply_2d(spec: WaveletSpec, j: int, data, inverse: bool, min_level: int = -1):
    return dwt_apply(spec, j, data, inverse, min_level, dim=2)


def _fwht(v, sequency: int):
    v = _dev_tensor(v, "fwht")
    n = v.shape[-1]
    bits = n.bit_length() - 1
    if n <= 0 or (1 << bits) != n:
        raise CwwError("length is not a power of two", 1)
    _check(_load().cww_fwht(v.data_ptr(), bits, v.numel() // n, sequency, _stream_ptr(v)))
    return v


def fwht_sequency(v):
    """In-place sequency-ordered FWHT (walsh.cpp:88-98) of a CUDA tensor."""
    return _fwht(v, 1)


def fwht_natural(v):
    """In-place natural-order FWHT (walsh.cpp:81-86) of a CUDA tensor."""
    return _fwht(v, 0)


def sequency_perm(bits: int, device=None):
    """perm[n] = bit_reverse(gray(n), bits), computed on the GPU (int64 tensor)."""
    torch = _torch()
    dev = torch.device("cuda") if device is None else torch.device(device)
    out = torch.empty(1 << bits, dtype=torch.int32, device=dev)
    _check(_load().cww_sequency_perm(bits, out.data_ptr(), torch.cuda.current_stream(dev).cuda_stream))
    return out.to(torch.int64) & 0xFFFFFFFF


def walsh_sign_rows(positions, j: int, device=None):
    """rows[i, r] = w_r(p_i / 2^j) (walsh.cpp:123-131), on the GPU."""
    torch = _torch()
    dev = torch.device("cuda") if device is None else torch.device(device)
    p = torch.as_tensor(np.asarray(positions, dtype=np.int64), device=dev)
    out = torch.empty((p.numel(), 1 << j), dtype=torch.float64, device=dev)
    _check(_load().cww_walsh_sign_rows(p.data_ptr(), p.numel(), j, out.data_ptr(),
                                       torch.cuda.current_stream(dev).cuda_stream))
    return out


def profile_enable(on: bool = True) -> None:
    """Bracket every kernel launch with CUDA events on its stream."""
    _load().cww_profile_enable(1 if on else 0)


def profile_dump() -> dict:
    """{kernel: (total_ms, launches)} since the last dump (synchronises)."""
    import json
    buf = C.create_string_buffer(1 << 16)
    _check(_load().cww_profile_dump(buf, len(buf)))
    return {k: (v[0], int(v[1])) for k, v in json.loads(buf.value.decode()).items()}


def kernel_launches() -> int:
    """Number of kernels this library has launched in this process."""
    return int(_load().cww_kernel_launches())


def synth(kind: int, seed: int, j: int, r0: int, density: float, dim: int = 1) -> np.ndarray:
    """Seeded synthetic inputs of SURVEY.md 8d (test_rng semantics), host array."""
    n = (1 << j) if dim == 1 else (1 << (2 * j))
    out = np.empty(n)
    _check(_load().cww_synth(kind, seed, j, r0, density, dim, _np_ptr(out)))
    return out
