"""TEST INFRASTRUCTURE ONLY -- ctypes bindings for the CPU oracle.

`Oracle`   : oracle/liboracle.so, the plain-C restatement (cww_oracle.c).
`Reference`: oracle/_ref/libcwwref.so, the unmodified reference library built
             from /root/reference/proj/src by oracle/Makefile (ref_shim.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import
this module; the product path (paper_2106_00554_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
DATA_DIR = os.path.join(REPO, "paper_2106_00554_b200", "data")
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcwwref.so")

_dp = C.POINTER(C.c_double)


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def build(ref: bool = True) -> None:
    """Builds liboracle.so (always possible) and, when the reference sources
    are present, oracle/_ref/libcwwref.so."""
    targets = ["liboracle"]
    if ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


class OracleError(RuntimeError):
    pass


class Oracle:
    """The C restatement.  Families: 0 Daubechies, 1 Symlet; boundary: 0
    periodic, 1 vmp (the reference enums, wavelet.hpp:15-16)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = C.CDLL(path)
        self.L = L
        L.orc_last_error.restype = C.c_char_p
        L.orc_seq_to_nat.restype = C.c_uint64
        L.orc_seq_to_nat.argtypes = [C.c_uint64, C.c_uint]
        L.orc_walsh_eval.argtypes = [C.c_uint64, C.c_uint64, C.c_uint]
        L.orc_walsh_sign_row.argtypes = [C.c_uint64, C.c_uint, _dp]
        L.orc_fwht_natural.argtypes = [_dp, C.c_size_t]
        L.orc_fwht_sequency.argtypes = [_dp, C.c_size_t]
        L.orc_dwt.argtypes = [C.c_void_p, C.c_int, C.c_uint, _dp, C.c_int, C.c_int]
        L.orc_dwt2d.argtypes = [C.c_void_p, C.c_int, C.c_uint, _dp, C.c_int, C.c_int]
        L.orc_load_filters.argtypes = [C.c_int, C.c_int, C.c_char_p, C.c_void_p]
        L.orc_kernel_table.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp]
        L.orc_cascade.restype = C.c_long
        L.orc_cascade.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, _dp, C.c_size_t,
                                  C.POINTER(C.c_int)]
        L.orc_op_create.restype = C.c_void_p
        L.orc_op_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint, C.c_uint, C.c_int,
                                    C.c_int, C.c_char_p]
        L.orc_op_destroy.argtypes = [C.c_void_p]
        L.orc_op_forward.argtypes = [C.c_void_p, _dp, _dp, C.c_int]
        L.orc_op_adjoint.argtypes = [C.c_void_p, _dp, _dp, C.c_int]
        L.orc_op_edge_terms.restype = C.c_long
        L.orc_op_edge_terms.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_int),
                                        C.POINTER(C.c_long), C.c_long]
        L.orc_rng_normals.argtypes = [C.c_uint64, _dp, C.c_size_t]
        L.orc_synth.argtypes = [C.c_int, C.c_uint64, C.c_uint, C.c_int, C.c_double, C.c_int, _dp]
        L.orc_min_level.argtypes = [C.c_int]
        L.orc_crc32.restype = C.c_uint32
        L.orc_crc32.argtypes = [C.c_char_p, C.c_size_t]

    def _check(self, rc):
        if rc != 0:
            raise OracleError(self.L.orc_last_error().decode())

    # ---- walsh
    def seq_to_nat(self, n: int, bits: int) -> int:
        return int(self.L.orc_seq_to_nat(n, bits))

    def walsh_eval(self, n: int, p: int, j: int) -> int:
        return int(self.L.orc_walsh_eval(n, p, j))

    def sign_row(self, p: int, j: int) -> np.ndarray:
        s = np.empty(1 << j)
        self.L.orc_walsh_sign_row(p, j, _ptr(s))
        return s

    def fwht_natural(self, v) -> np.ndarray:
        v = np.array(v, dtype=np.float64, copy=True)
        self._check(self.L.orc_fwht_natural(_ptr(v), v.size))
        return v

    def fwht_sequency(self, v) -> np.ndarray:
        v = np.array(v, dtype=np.float64, copy=True)
        self._check(self.L.orc_fwht_sequency(_ptr(v), v.size))
        return v

    # ---- filters / dwt / kernel table
    def filters(self, family: int, nu: int):
        buf = C.create_string_buffer(8 * 1024)
        self._check(self.L.orc_load_filters(family, nu, DATA_DIR.encode(), buf))
        return buf

    def dwt(self, family, nu, boundary, j, data, inverse, min_level=-1, dim=1):
        f = self.filters(family, nu)
        d = np.array(data, dtype=np.float64, copy=True)
        fn = self.L.orc_dwt if dim == 1 else self.L.orc_dwt2d
        self._check(fn(f, boundary, j, _ptr(d), int(inverse), min_level))
        return d

    def kernel_table(self, family, nu, boundary, q, R=14):
        f = self.filters(family, nu)
        W, S = 2 * nu - 1, 1 << q
        it = np.zeros(W * S)
        le = np.zeros(nu * W * S)
        ri = np.zeros(nu * W * S)
        self._check(self.L.orc_kernel_table(f, boundary, q, R, _ptr(it), _ptr(le), _ptr(ri)))
        return it, le, ri

    def cascade(self, family, nu, kind, m, R):
        f = self.filters(family, nu)
        sl = C.c_int(0)
        n = self.L.orc_cascade(f, kind, m, R, None, 0, C.byref(sl))
        if n < 0:
            raise OracleError(self.L.orc_last_error().decode())
        v = np.empty(n)
        self.L.orc_cascade(f, kind, m, R, _ptr(v), n, C.byref(sl))
        return v, sl.value

    def min_level(self, nu: int) -> int:
        return int(self.L.orc_min_level(nu))

    def crc32(self, b: bytes) -> int:
        return int(self.L.orc_crc32(b, len(b)))

    # ---- inputs
    def normals(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n)
        self.L.orc_rng_normals(seed, _ptr(out), n)
        return out

    def synth(self, kind, seed, j, r0, density, dim=1) -> np.ndarray:
        n = (1 << j) if dim == 1 else (1 << (2 * j))
        out = np.empty(n)
        self._check(self.L.orc_synth(kind, seed, j, r0, density, dim, _ptr(out)))
        return out

    def op(self, family, nu, boundary, j, q, dim=1, r0=-1):
        return OracleOp(self, family, nu, boundary, j, q, dim, r0)


class OracleOp:
    def __init__(self, orc: Oracle, family, nu, boundary, j, q, dim, r0):
        self.o = orc
        self.h = orc.L.orc_op_create(family, nu, boundary, j, q, dim, r0, DATA_DIR.encode())
        if not self.h:
            raise OracleError(orc.L.orc_last_error().decode())
        self.M, self.N, self.dim = 1 << j, 1 << (j + q), dim
        self.nin = self.M if dim == 1 else self.M * self.M
        self.nout = self.N if dim == 1 else self.N * self.N

    def __del__(self):
        if getattr(self, "h", None):
            self.o.L.orc_op_destroy(self.h)
            self.h = None

    def forward(self, x, use_idwt=True):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self.nout)
        self.o._check(self.o.L.orc_op_forward(self.h, _ptr(x), _ptr(y), int(use_idwt)))
        return y

    def adjoint(self, y, use_idwt=True):
        y = np.ascontiguousarray(y, dtype=np.float64)
        x = np.empty(self.nin)
        self.o._check(self.o.L.orc_op_adjoint(self.h, _ptr(y), _ptr(x), int(use_idwt)))
        return x

    def forward_masked(self, mask, x, use_idwt=True):
        """ComposedOp::forward with a subsampled mask (fastop.cpp:253-259):
        full forward, then y[i] = full[mask[i]]."""
        return self.forward(x, use_idwt)[np.asarray(mask, dtype=np.int64)]

    def adjoint_masked(self, mask, y, use_idwt=True):
        """ComposedOp::adjoint with a subsampled mask (fastop.cpp:265-270):
        scatter into zeros, then the full adjoint."""
        full = np.zeros(self.nout)
        full[np.asarray(mask, dtype=np.int64)] = y
        return self.adjoint(full, use_idwt)

    def edge_terms(self):
        cap = 512
        p = (C.c_uint64 * cap)()
        col = (C.c_int * cap)()
        row = (C.c_long * cap)()
        n = self.o.L.orc_op_edge_terms(self.h, p, col, row, cap)
        return [(int(p[i]), int(col[i]), int(row[i])) for i in range(n)]


class Reference:
    """The compiled, unmodified reference (oracle/_ref/libcwwref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build(ref=True)
        if not os.path.exists(path):
            raise OracleError("reference library not built (needs /root/reference)")
        L = C.CDLL(path)
        self.L = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_fwht_natural.argtypes = [_dp, C.c_size_t]
        L.ref_fwht_sequency.argtypes = [_dp, C.c_size_t]
        L.ref_seq_to_nat.restype = C.c_ulonglong
        L.ref_seq_to_nat.argtypes = [C.c_ulonglong, C.c_uint]
        L.ref_walsh_sign_row.argtypes = [C.c_ulonglong, C.c_uint, _dp]
        L.ref_walsh_eval.argtypes = [C.c_ulonglong, C.c_ulonglong, C.c_uint]
        L.ref_dwt.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint, _dp, C.c_int, C.c_int, C.c_int,
                              C.c_char_p]
        L.ref_kernel_table.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_char_p,
                                       _dp, _dp, _dp]
        L.ref_op_create.restype = C.c_void_p
        L.ref_op_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint, C.c_uint, C.c_int,
                                    C.c_int, C.c_char_p]
        L.ref_op_destroy.argtypes = [C.c_void_p]
        L.ref_op_forward.argtypes = [C.c_void_p, _dp, _dp, C.c_int]
        L.ref_op_adjoint.argtypes = [C.c_void_p, _dp, _dp, C.c_int]
        L.ref_haar_fullrank.argtypes = [C.c_uint, _dp, _dp, C.c_int]
        L.ref_composed_masked.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_int,
                                          _dp, _dp]
        L.ref_kernel_cache_save.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_char_p,
                                            C.c_char_p]
        L.ref_kernel_cache_load.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.c_void_p, C.c_void_p,
                                            C.c_void_p, C.POINTER(C.c_size_t)]
        L.ref_bench.restype = C.c_double
        L.ref_bench.argtypes = [C.c_void_p, C.c_int, _dp, _dp, C.c_size_t, C.c_int, C.c_int,
                                C.c_int]
        L.ref_min_level.argtypes = [C.c_int]

    def _check(self, rc):
        if rc != 0:
            raise OracleError(self.L.ref_last_error().decode())

    def fwht_natural(self, v):
        v = np.array(v, dtype=np.float64, copy=True)
        self._check(self.L.ref_fwht_natural(_ptr(v), v.size))
        return v

    def fwht_sequency(self, v):
        v = np.array(v, dtype=np.float64, copy=True)
        self._check(self.L.ref_fwht_sequency(_ptr(v), v.size))
        return v

    def seq_to_nat(self, n, bits):
        return int(self.L.ref_seq_to_nat(n, bits))

    def sign_row(self, p, j):
        s = np.empty(1 << j)
        self._check(self.L.ref_walsh_sign_row(p, j, _ptr(s)))
        return s

    def walsh_eval(self, n, p, j):
        return int(self.L.ref_walsh_eval(n, p, j))

    def dwt(self, family, nu, boundary, j, data, inverse, min_level=-1, dim=1):
        d = np.array(data, dtype=np.float64, copy=True)
        self._check(self.L.ref_dwt(family, nu, boundary, j, _ptr(d), int(inverse), min_level,
                                   dim, DATA_DIR.encode()))
        return d

    def kernel_cache_save(self, family, nu, boundary, q, path, R=14):
        """The reference's save_kernel_table of its own computed table."""
        self._check(self.L.ref_kernel_cache_save(family, nu, boundary, q, R, DATA_DIR.encode(),
                                                 path.encode()))

    def kernel_cache_load(self, path):
        """The reference's load_kernel_table: (header, interior, left, right)."""
        hdr = (C.c_int * 5)()
        cnt = (C.c_size_t * 3)()
        big = [np.empty(1 << 16) for _ in range(3)]
        self._check(self.L.ref_kernel_cache_load(path.encode(), hdr, big[0].ctypes.data, big[1].ctypes.data,
                                                 big[2].ctypes.data, cnt))
        return list(hdr), big[0][:cnt[0]].copy(), big[1][:cnt[1]].copy(), big[2][:cnt[2]].copy()

    def kernel_table(self, family, nu, boundary, q, R=14):
        W, S = 2 * nu - 1, 1 << q
        it = np.zeros(W * S)
        le = np.zeros(nu * W * S)
        ri = np.zeros(nu * W * S)
        self._check(self.L.ref_kernel_table(family, nu, boundary, q, R, DATA_DIR.encode(),
                                            _ptr(it), _ptr(le), _ptr(ri)))
        return it, le, ri

    def haar_fullrank(self, j, v, adjoint=False):
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.empty_like(v)
        self._check(self.L.ref_haar_fullrank(j, _ptr(v), _ptr(out), int(adjoint)))
        return out

    def op(self, family, nu, boundary, j, q, dim=1, r0=-1):
        return ReferenceOp(self, family, nu, boundary, j, q, dim, r0)


class ReferenceOp:
    def __init__(self, ref: Reference, family, nu, boundary, j, q, dim, r0):
        self.r = ref
        self.h = ref.L.ref_op_create(family, nu, boundary, j, q, dim, r0, DATA_DIR.encode())
        if not self.h:
            raise OracleError(ref.L.ref_last_error().decode())
        self.M, self.N, self.dim = 1 << j, 1 << (j + q), dim
        self.nin = self.M if dim == 1 else self.M * self.M
        self.nout = self.N if dim == 1 else self.N * self.N

    def __del__(self):
        if getattr(self, "h", None):
            self.r.L.ref_op_destroy(self.h)
            self.h = None

    def forward(self, x, use_idwt=True):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self.nout)
        self.r._check(self.r.L.ref_op_forward(self.h, _ptr(x), _ptr(y), int(use_idwt)))
        return y

    def adjoint(self, y, use_idwt=True):
        y = np.ascontiguousarray(y, dtype=np.float64)
        x = np.empty(self.nin)
        self.r._check(self.r.L.ref_op_adjoint(self.h, _ptr(y), _ptr(x), int(use_idwt)))
        return x

    def masked(self, mask, v, adjoint=False, use_idwt=True):
        """The reference ComposedOp(op, SamplingMask{mask}, use_idwt) (fastop.cpp:231-281)."""
        m = np.ascontiguousarray(mask, dtype=np.uint64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.empty(self.nin if adjoint else m.size)
        self.r._check(self.r.L.ref_composed_masked(self.h, m.ctypes.data, m.size, int(use_idwt),
                                                   int(adjoint), _ptr(v), _ptr(out)))
        return out

    def bench(self, mode, inp, out, batch, threads, iters=1, use_idwt=True) -> float:
        t = self.r.L.ref_bench(self.h, mode, _ptr(inp), _ptr(out), batch, threads, iters,
                               int(use_idwt))
        if t < 0:
            raise OracleError(self.r.L.ref_last_error().decode())
        return t
