"""CWWK kernel-table cache files (kernel.cpp:79-198):
byte-identical to the reference's save_kernel_table (committed fixtures
written by the reference, tests/golden/make_golden.py), the reference's
validation behaviour on damaged files, and the live reference both ways when
it is built here.  Host-only (no GPU); the op-side cache use is in
tests/test_gpu_parity.py."""
import os
import shutil
import struct
import zlib

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")
FIXTURES = [(0, 2, 1, 1), (1, 3, 0, 3), (0, 4, 1, 2)]


def _name(fam, nu, bnd, q):
    return f"cwwk_{'db' if fam == 0 else 'sym'}{nu}_{'vmp' if bnd else 'periodic'}_q{q}_R14_v1.bin"


@pytest.mark.parametrize("case", FIXTURES)
def test_save_is_byte_identical_to_reference_fixture(tmp_path, case):
    import paper_2106_00554_b200 as cw
    fam, nu, bnd, q = case
    spec = cw.WaveletSpec(cw.Family(fam), nu, cw.Boundary(bnd))
    assert cw.kernel_cache_filename(spec, q) == _name(*case)
    out = tmp_path / _name(*case)
    cw.kernel_table_save(spec, q, str(out))
    assert out.read_bytes() == open(os.path.join(GOLD, _name(*case)), "rb").read()


@pytest.mark.parametrize("case", FIXTURES)
def test_load_reference_fixture_matches_oracle_table(orc, case):
    import paper_2106_00554_b200 as cw
    fam, nu, bnd, q = case
    t = cw.kernel_table_load(os.path.join(GOLD, _name(*case)))
    assert (t["family"], t["nu"], t["boundary"], t["q"], t["R"]) == (fam, nu, bnd, q, 14)
    it, le, ri = orc.kernel_table(fam, nu, bnd, q)
    assert np.array_equal(t["interior"], it)
    if bnd:
        assert np.array_equal(t["left"], le) and np.array_equal(t["right"], ri)
    else:  # periodic tables hold the interior array only (kernel.hpp:12-13)
        assert t["left"].size == 0 and t["right"].size == 0


def _rewrite(path, body):
    """Write `body` with a valid trailing CRC-32."""
    with open(path, "wb") as f:
        f.write(body + struct.pack("<I", zlib.crc32(body) & 0xFFFFFFFF))


def _damaged(tmp_path):
    src = open(os.path.join(GOLD, _name(0, 4, 1, 2)), "rb").read()
    body = src[:-4]
    cases = {}
    p = tmp_path / "flip.bin"
    b = bytearray(src)
    b[40] ^= 0x55
    p.write_bytes(bytes(b))
    cases["checksum failure"] = p
    p = tmp_path / "short.bin"
    p.write_bytes(src[:20])
    cases["truncated kernel cache"] = p
    p = tmp_path / "magic.bin"
    _rewrite(p, b"XWWK" + body[4:])
    cases["bad magic"] = p
    p = tmp_path / "version.bin"
    _rewrite(p, body[:4] + struct.pack("<I", 2) + body[8:])
    cases["version mismatch"] = p
    p = tmp_path / "payload.bin"
    _rewrite(p, body[:28] + struct.pack("<I", 1 << 20) + body[32:])
    cases["truncated kernel cache payload"] = p
    p = tmp_path / "shape.bin"
    n_int = struct.unpack("<I", body[28:32])[0]
    _rewrite(p, body[:28] + struct.pack("<I", n_int - 1) + body[32:32 + 8 * (n_int - 1)] + body[32 + 8 * n_int:])
    cases["shape mismatch (interior)"] = p
    cases["cannot open kernel cache"] = tmp_path / "missing.bin"
    return cases


def test_damaged_files_rejected_like_the_reference(tmp_path):
    import paper_2106_00554_b200 as cw
    for msg, path in _damaged(tmp_path).items():
        with pytest.raises(cw.CwwError, match=msg.replace("(", r"\(").replace(")", r"\)")) as e:
            cw.kernel_table_load(str(path))
        assert e.value.status == 4, msg


def test_live_reference_round_trips(tmp_path, orc):
    """With the reference built here: it reads our files, we read its files,
    and both reject the same damaged files with the same messages."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle"))
    try:
        from oracle_py import OracleError, Reference
        ref = Reference()
    except Exception as e:  # noqa: BLE001
        pytest.skip(f"reference not built here: {e}")
    import paper_2106_00554_b200 as cw
    for fam, nu, bnd, q in [(0, 5, 1, 1), (1, 6, 0, 2), (0, 3, 1, 3)]:
        spec = cw.WaveletSpec(cw.Family(fam), nu, cw.Boundary(bnd))
        ours, theirs = tmp_path / "ours.bin", tmp_path / "theirs.bin"
        cw.kernel_table_save(spec, q, str(ours))
        ref.kernel_cache_save(fam, nu, bnd, q, str(theirs))
        assert ours.read_bytes() == theirs.read_bytes()
        h, it, le, ri = ref.kernel_cache_load(str(ours))
        t = cw.kernel_table_load(str(theirs))
        assert h == [t["family"], t["nu"], t["boundary"], t["q"], t["R"]]
        assert np.array_equal(it, t["interior"]) and np.array_equal(le, t["left"])
    for msg, path in _damaged(tmp_path).items():
        with pytest.raises(OracleError) as e:
            ref.kernel_cache_load(str(path))
        assert msg in str(e.value), (msg, str(e.value))


def test_spec_errors():
    import paper_2106_00554_b200 as cw
    with pytest.raises(cw.CwwError, match="q >= 1"):
        cw.kernel_table_save(cw.WaveletSpec(cw.Family.Daubechies, 3, cw.Boundary.Vmp), 0, "/tmp/x.bin")
    with pytest.raises(cw.CwwError, match="nu >= 2"):
        cw.kernel_table_save(cw.WaveletSpec(cw.Family.Daubechies, 1, cw.Boundary.Periodic), 1, "/tmp/x.bin")
