"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every
symbol include/cww_b200.h declares, validates specs like the reference
(fastop.cpp:31-45, wavelet.cpp:31-39) and refuses to compute without a GPU
(no CPU fallback).  No compute calls here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "cww_b200.h")


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(cww_[a-z_0-9]+)\s*\(", txt)))


def test_library_loads_and_exports_all_symbols():
    import paper_2106_00554_b200 as cw
    L = cw._load()
    names = _declared()
    assert len(names) >= 18
    for n in names:
        assert hasattr(L, n), n
    assert b"sm_100a" in L.cww_version()


def _desc(**kw):
    import paper_2106_00554_b200 as cw
    d = cw._Desc()
    cw._load().cww_op_desc_init(C.byref(d))
    for k, v in kw.items():
        setattr(d, k, v)
    d.data_dir = cw.DATA_DIR.encode()
    return d


@pytest.mark.parametrize("kw,status", [
    (dict(nu=7), 3), (dict(nu=0), 3), (dict(nu=1, boundary=1), 3), (dict(nu=1, family=1, boundary=0), 3),
    (dict(nu=4, j=2), 3), (dict(nu=2, q=0), 3), (dict(dim=3), 3), (dict(nu=4, j=6, min_level=2), 3),
    (dict(nu=2, j=5, min_level=6), 3), (dict(family=5), 1), (dict(nu=2, j=17, q=1, dim=2), 7),
    (dict(nu=3, j=24, q=1), 7), (dict(nu=3, j=20, q=2, precision=2), 1),
])
def test_spec_validation(kw, status):
    import paper_2106_00554_b200 as cw
    L = cw._load()
    d = _desc(**kw)
    h = C.c_void_p()
    assert L.cww_op_create(C.byref(d), C.byref(h)) == status
    assert L.cww_last_error()


def test_no_cpu_fallback():
    import torch
    import paper_2106_00554_b200 as cw
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    L = cw._load()
    d = _desc(nu=2, j=5, q=1)
    h = C.c_void_p()
    assert L.cww_op_create(C.byref(d), C.byref(h)) == 5  # CWW_ERR_CUDA
    assert b"no CUDA device" in L.cww_last_error()
    with pytest.raises(cw.CwwError):
        cw.FastOp(cw.WaveletSpec(cw.Family.Daubechies, 2, cw.Boundary.Vmp), 5, 1)


def test_python_spec_mirror():
    import paper_2106_00554_b200 as cw
    s = cw.parse_wavelet_name("db4", cw.Boundary.Vmp)
    assert s.nu == 4 and s.min_level() == 3 and s.name() == "db4"
    assert cw.parse_wavelet_name("sym6", cw.Boundary.Vmp).family == cw.Family.Symlet
    assert cw.parse_wavelet_name("haar", cw.Boundary.Periodic).nu == 1
    with pytest.raises(cw.CwwError):
        cw.parse_wavelet_name("coif3", cw.Boundary.Vmp)
    with pytest.raises(cw.CwwError):
        cw.WaveletSpec(cw.Family.Daubechies, 1, cw.Boundary.Vmp).validate()


@pytest.mark.parametrize("args", [(0, 1001, 10, 1, 1.0, 1), (1, 1002, 16, 4, 1.0, 1),
                                  (0, 1003, 14, 4, 0.1, 1), (1, 1004, 6, 4, 0.05, 2),
                                  (0, 1005, 7, 3, 0.02, 2)])
def test_synth_matches_oracle(orc, args):
    """The product's seeded-input generator equals the oracle's test_rng port."""
    import paper_2106_00554_b200 as cw
    kind, seed, j, r0, dens, dim = args
    assert np.array_equal(cw.synth(kind, seed, j, r0, dens, dim), orc.synth(kind, seed, j, r0, dens, dim))


def test_header_documents_reference_interfaces():
    txt = open(HEADER).read()
    for cite in ("fastop.hpp", "wavelet.hpp", "walsh.hpp", "kernel.hpp"):
        assert cite in txt


def test_c_and_cpp_headers_compile_and_link(tmp_path):
    """A C caller (cww_b200.h) and a reference-style C++ caller
    (cww_b200.hpp: LinearOp / FastOp / ComposedOp over spans) build and link
    against the in-tree library."""
    import shutil
    import subprocess
    import paper_2106_00554_b200 as cw
    lib = cw.library_path()
    c_src = tmp_path / "c_caller.c"
    c_src.write_text('#include "cww_b200.h"\n#include <stdio.h>\nint main(void){cww_op_desc d; '
                     'cww_op_desc_init(&d); cww_op* h=0; cww_status s=cww_op_create(&d,&h); '
                     'printf("%d %s\\n",(int)s,cww_last_error()); return 0;}\n')
    cpp_src = tmp_path / "cpp_caller.cpp"
    cpp_src.write_text('#include "cww_b200.hpp"\n#include <vector>\nint main(){ try { '
                       'cww_b200::WaveletSpec s{cww_b200::Family::Daubechies, 4, cww_b200::Boundary::Vmp};'
                       ' cww_b200::FastOp op(s, 6, 2); cww_b200::ComposedOp c(op, true, 4);'
                       ' cww_b200::SamplingMask m{{1, 5, 9}}; cww_b200::ComposedOp cm(op, m, true);'
                       ' std::vector<double> x(c.cols()), y(c.rows()); c.forward(x, y); }'
                       ' catch (const cww_b200::CwwError& e) { return e.status == CWW_ERR_CUDA ? 0 : 1; }'
                       ' return 0; }\n')
    inc = os.path.join(REPO, "include")
    libdir = os.path.dirname(lib)
    gcc, gxx = shutil.which("gcc"), shutil.which("g++")
    r = subprocess.run([gcc, "-std=c11", "-I", inc, str(c_src), "-o", str(tmp_path / "c_caller"),
                        lib, f"-Wl,-rpath,{libdir}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([gxx, "-std=c++20", "-I", inc, str(cpp_src), "-o", str(tmp_path / "cpp_caller"),
                        lib, f"-Wl,-rpath,{libdir}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(tmp_path / "c_caller")], capture_output=True, text=True)
    assert out.returncode == 0
    run = subprocess.run([str(tmp_path / "cpp_caller")], capture_output=True, text=True)
    assert run.returncode == 0, run.stdout + run.stderr


@pytest.mark.parametrize("mask,status", [([0, 5, 3], 3), ([0, 1, 1], 3), ([0, 1 << 20], 3)])
def test_mask_validation(mask, status):
    """SamplingMask::validate (fastop.cpp:19-25): unsorted, duplicate or
    out-of-range indices are rejected before any device work."""
    import paper_2106_00554_b200 as cw
    L = cw._load()
    m = np.array(mask, dtype=np.uint64)
    d = _desc(nu=2, j=5, q=1)
    d.mask = m.ctypes.data
    d.mask_len = m.size
    h = C.c_void_p()
    assert L.cww_op_create(C.byref(d), C.byref(h)) == status
    assert b"sampling mask" in L.cww_last_error()


def test_python_mask_mirror():
    import paper_2106_00554_b200 as cw
    m = cw.SamplingMask([1, 4, 9])
    m.validate(16)
    assert m.size() == 3 and not m.is_full(16)
    assert cw.SamplingMask.full(8).is_full(8)
    assert cw.SamplingMask(np.arange(8)).is_full(8)
    with pytest.raises(cw.CwwError, match="out of range"):
        cw.SamplingMask([1, 16]).validate(16)
    with pytest.raises(cw.CwwError, match="sorted and unique"):
        cw.SamplingMask([3, 2]).validate(16)
