"""Pins the CPU oracle (oracle/cww_oracle.c) before it is trusted as the checker:
  * against golden vectors produced by the UNMODIFIED reference
    (tests/golden/golden.npz, tests/golden/make_golden.py);
  * against the compiled reference itself when oracle/_ref is present;
  * against the known-answer / property checks of the reference's own test
    suites (proj/tests/test_walsh.cpp, proj/tests/test_wavelet.cpp), restated.
"""
import math
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


# ---- golden vectors (reference outputs) ------------------------------------
def test_golden_operator_cases(orc, gold):
    cases = sorted({k.split("_")[0] for k in gold.files if k.startswith("c") and k.endswith("_case")})
    assert len(cases) >= 15
    for c in cases:
        fam, nu, bnd, j, q, dim, r0 = (int(v) for v in gold[c + "_case"])
        op = orc.op(fam, nu, bnd, j, q, dim, r0)
        x, y = gold[c + "_x"], gold[c + "_y"]
        for use in (0, 1):
            k = f"{c}_fwd{use}"
            if k not in gold.files:
                continue
            assert rel(op.forward(x, use), gold[k]) <= 1e-14, (c, use)
            assert rel(op.adjoint(y, use), gold[f"{c}_adj{use}"]) <= 1e-14, (c, use)


def test_golden_kernel_tables_bit_exact(orc, gold):
    n = 0
    for k in gold.files:
        if not (k.startswith("k_") and k.endswith("_int")):
            continue
        _, fam, nu, bnd, q, _ = k.split("_")
        it, le, ri = orc.kernel_table(int(fam), int(nu), int(bnd), int(q))
        base = k[: -len("_int")]
        assert np.array_equal(it, gold[base + "_int"]), k
        assert np.array_equal(le, gold[base + "_left"]), k
        assert np.array_equal(ri, gold[base + "_right"]), k
        n += 1
    assert n == 60


def test_golden_fwht_perm_signs_dwt(orc, gold):
    v = gold["fwht_in"]
    assert np.array_equal(orc.fwht_sequency(v), gold["fwht_seq"])
    assert np.array_equal(orc.fwht_natural(v), gold["fwht_nat"])
    perm = np.array([orc.seq_to_nat(n, 13) for n in range(1 << 13)])
    assert np.array_equal(perm, gold["perm_13"])
    signs = np.stack([orc.sign_row(p, 6) for p in range(64)])
    assert np.array_equal(signs, gold["sign_j6"])
    for k in gold.files:
        if k.startswith("dwt_") and k.endswith("_x"):
            _, nu, bnd, j, r0, _ = k.split("_")
            base = k[:-2]
            x = gold[k]
            fwd = orc.dwt(0, int(nu), int(bnd), int(j), x, 0, int(r0))
            inv = orc.dwt(0, int(nu), int(bnd), int(j), x, 1, int(r0))
            assert rel(fwd, gold[base + "_fwd"]) <= 1e-15
            assert rel(inv, gold[base + "_inv"]) <= 1e-15


def test_golden_masked_composed_op(orc, gold):
    """Subsampled ComposedOp (SamplingMask, fastop.cpp:231-281): the oracle's
    gather/scatter restatement against the reference's own outputs."""
    cases = sorted({k.split("_")[0] for k in gold.files if k.startswith("m") and k.endswith("_case")})
    assert len(cases) >= 4
    for c in cases:
        fam, nu, bnd, j, q, dim = (int(v) for v in gold[c + "_case"])
        op = orc.op(fam, nu, bnd, j, q, dim, -1)
        mask = gold[c + "_mask"]
        assert mask.size < op.nout and np.all(np.diff(mask.astype(np.int64)) > 0)
        for use in (0, 1):
            assert rel(op.forward_masked(mask, gold[c + "_x"], use), gold[f"{c}_fwd{use}"]) <= 1e-14
            assert rel(op.adjoint_masked(mask, gold[c + "_y"], use), gold[f"{c}_adj{use}"]) <= 1e-14


# ---- live reference (this container, or a prebuilt oracle/_ref) ------------
@pytest.mark.parametrize("case", [
    (0, 2, 1, 8, 1, 1, 3), (0, 4, 1, 9, 2, 1, 4), (0, 3, 1, 10, 2, 1, 4), (1, 5, 0, 8, 2, 1, -1),
    (0, 6, 1, 8, 1, 1, -1), (0, 1, 0, 10, 1, 1, 1), (0, 4, 1, 5, 1, 2, 4), (0, 2, 1, 5, 1, 2, 3),
])
def test_oracle_matches_reference(orc, ref, case):
    fam, nu, bnd, j, q, dim, r0 = case
    o, r = orc.op(*case), ref.op(*case)
    x, y = orc.normals(11, o.nin), orc.normals(12, o.nout)
    for use in (0, 1):
        assert rel(o.forward(x, use), r.forward(x, use)) <= 1e-14
        assert rel(o.adjoint(y, use), r.adjoint(y, use)) <= 1e-14


def test_edge_terms_match_reference_layout(orc):
    # VMP: 2 * sum_m (nu+m) terms; positions [0, 2nu-2] and [M-2nu+1, M-1]
    for nu in range(2, 7):
        j = orc.min_level(nu) + 2
        M = 1 << j
        terms = orc.op(0, nu, 1, j, 1).edge_terms()
        assert len(terms) == 2 * sum(nu + m for m in range(nu))
        ps = sorted({t[0] for t in terms})
        assert ps == list(range(2 * nu - 1)) + list(range(M - 2 * nu + 1, M))
        assert [t[0] for t in terms] == sorted(t[0] for t in terms)
        pterms = orc.op(0, nu, 0, j, 1).edge_terms()
        assert len(pterms) == 2 * nu * (2 * nu - 1)
        assert sorted({t[0] for t in pterms}) == ps


# ---- restated known-answer checks of proj/tests/test_walsh.cpp ---------------
def _walsh_brute(n, p, j):  # test_walsh.cpp:16-25
    e = 0
    for i in range(1, j + 1):
        xi = (p >> (j - i)) & 1
        e += (((n >> (i - 1)) & 1) + ((n >> i) & 1)) * xi
    return -1 if e % 2 else 1


def test_walsh_eval_bruteforce(orc):  # test_walsh.cpp:52-61
    for j in range(7):
        for p in range(1 << j):
            assert orc.walsh_eval(0, p, j) == 1
    assert orc.walsh_eval(1, 3, 2) == -1
    for n in range(64):
        for p in range(64):
            assert orc.walsh_eval(n, p, 6) == _walsh_brute(n, p, 6)


def test_walsh_symmetry_and_sign_changes(orc):  # test_walsh.cpp:75-104
    for j in range(1, 7):
        for n in range(1 << j):
            for l in range(1 << j):
                assert orc.walsh_eval(n, l, j) == orc.walsh_eval(l, n, j)
    for r in range(1, 7):
        for n in range(1 << r):
            row = [orc.walsh_eval(n, k, r) for k in range(1 << r)]
            assert sum(row[i] != row[i - 1] for i in range(1, len(row))) == n


def test_fwht_known_answers(orc):  # test_walsh.cpp:106-116
    ones = orc.fwht_sequency(np.ones(8))
    assert ones[0] == 8.0 and np.all(ones[1:] == 0.0)
    d = np.zeros(8)
    d[0] = 1.0
    assert np.all(orc.fwht_sequency(d) == 1.0)


def test_fwht_vs_dense_sequency_hadamard(orc):  # test_walsh.cpp:118-132
    for r in (3, 4, 5, 6):
        n = 1 << r
        v = orc.normals(22 + r, n)
        H = np.array([[orc.walsh_eval(a, k, r) for k in range(n)] for a in range(n)], float)
        assert np.allclose(orc.fwht_sequency(v), H @ v, rtol=1e-12, atol=1e-12)


def test_fwht_involution(orc):  # test_walsh.cpp:134-150
    for r in range(3, 13):
        n = 1 << r
        v = orc.normals(33, n)
        w = orc.fwht_sequency(orc.fwht_sequency(v))
        assert rel(w, n * v) <= 1e-13


def test_sign_row_vs_walsh_eval(orc):  # test_walsh.cpp:175-185
    for j in (3, 5):
        for p in range(1 << j):
            s = orc.sign_row(p, j)
            assert all(s[r] == orc.walsh_eval(r, p, j) for r in range(1 << j))


# ---- restated checks of proj/tests/test_wavelet.cpp -------------------------
def test_min_level():  # test_wavelet.cpp:56-57
    from oracle_py import Oracle
    o = Oracle()
    assert o.min_level(2) == 2 and o.min_level(6) == 4 and o.min_level(1) == 0


def test_dwt_forward_inverse_identity(orc):  # test_wavelet.cpp:162-176
    for bnd in (0, 1):
        for nu in (2, 4, 6):
            j = orc.min_level(nu) + 2
            v = orc.normals(7, 1 << j)
            w = orc.dwt(0, nu, bnd, j, orc.dwt(0, nu, bnd, j, v, 0), 1)
            assert np.max(np.abs(v - w)) <= 1e-12


def test_dwt_norm_conservation(orc):  # test_wavelet.cpp:178-193
    for bnd in (0, 1):
        for nu in (2, 3, 5):
            j = orc.min_level(nu) + 3
            v = orc.normals(8, 1 << j)
            w = orc.dwt(1, nu, bnd, j, v, 0)
            tol = 1e-12 if bnd == 0 else 1e-10
            assert abs(np.linalg.norm(w) - np.linalg.norm(v)) / np.linalg.norm(v) <= tol


def test_dwt_haar_constant(orc):  # test_wavelet.cpp:195-201
    w = orc.dwt(0, 1, 0, 3, np.ones(8), 0, 0)
    assert w[0] == pytest.approx(math.sqrt(8.0))
    assert np.allclose(w[1:], 0.0)


def test_dwt_periodic_shift(orc):  # test_wavelet.cpp:209-230
    j, n = 5, 32
    v = orc.normals(55, n)
    sh = np.roll(v, 2)
    wv = orc.dwt(0, 3, 0, j, v, 0, j - 1)
    ws = orc.dwt(0, 3, 0, j, sh, 0, j - 1)
    h = n // 2
    for m in range(h):
        assert ws[(m + 1) % h] == pytest.approx(wv[m], rel=1e-12, abs=1e-12)
        assert ws[h + (m + 1) % h] == pytest.approx(wv[h + m], rel=1e-12, abs=1e-12)


def test_dwt2d_round_trip(orc):  # test_wavelet.cpp:259-270
    v = orc.normals(66, 256)
    w = orc.dwt(0, 2, 1, 4, orc.dwt(0, 2, 1, 4, v, 0, dim=2), 1, dim=2)
    assert np.max(np.abs(v - w)) <= 1e-11


def test_cascade_partition_of_unity(orc):  # test_wavelet.cpp:100-115
    for nu in (2, 3, 4, 5, 6):
        v, sl = orc.cascade(0, nu, 0, 0, 8)
        w = np.ones_like(v)
        w[0] = w[-1] = 0.5
        assert float(np.sum(w * v)) * 2.0 ** -8 == pytest.approx(1.0, rel=1e-12)


def test_filter_file_errors(orc, tmp_path):  # test_wavelet.cpp:87-89 + CRC
    from oracle_py import OracleError, DATA_DIR
    with pytest.raises(OracleError):
        orc.L.orc_load_filters(0, 4, str(tmp_path).encode(), orc.filters(0, 2)) and (_ for _ in ()).throw(
            OracleError(orc.L.orc_last_error().decode()))
    raw = bytearray(open(os.path.join(DATA_DIR, "db3.cwwf"), "rb").read())
    assert orc.crc32(bytes(raw[:-4])) == int.from_bytes(raw[-4:], "little")


# ---- kernel-table invariants (SPEC.md kernel module) ------------------------
def test_kernel_table_bessel_and_nesting(orc):
    for nu in (2, 3, 4):
        it1, le1, ri1 = orc.kernel_table(0, nu, 1, 1)
        it2, le2, ri2 = orc.kernel_table(0, nu, 1, 2)
        W = 2 * nu - 1
        for l in range(W):
            row2 = it2[l * 4:(l + 1) * 4]
            assert float(np.sum(row2 ** 2)) <= 1.0 + 1e-12
            # q-nesting: the q=2 table restricted to s < 2 equals the q=1 table
            assert np.allclose(row2[:2], it1[l * 2:(l + 1) * 2], atol=1e-12)


# ---- synthetic inputs follow test_rng (test_util.hpp:10-27) -----------------
def test_rng_semantics(orc):
    def py_rng(seed, n):
        m = (1 << 64) - 1
        s = (seed * 0x9E3779B97F4A7C15 + 1) & m
        out = []
        for _ in range(n):
            vals = []
            for _ in range(2):
                s ^= (s << 13) & m
                s ^= s >> 7
                s ^= (s << 17) & m
                vals.append(((s * 0x2545F4914F6CDD1D) & m) >> 11)
            u1, u2 = vals[0] * 2.0 ** -53, vals[1] * 2.0 ** -53
            u1 = max(u1, 1e-300)
            out.append(math.sqrt(-2.0 * math.log(u1)) * math.cos(6.283185307179586 * u2))
        return np.array(out)
    assert np.array_equal(orc.normals(1003, 64), py_rng(1003, 64))


def test_synth_shapes(orc):
    x = orc.synth(0, 3000, 12, 4, 0.1)
    assert np.count_nonzero(x) == round(0.1 * 4096)
    y = orc.synth(1, 2000, 8, 4, 1.0)
    assert np.all(np.abs(y[512 // 2:]) <= 2.0 ** -7 * 10)
    z = orc.synth(1, 4000, 5, 4, 0.05, dim=2)
    assert np.count_nonzero(z) == round(0.05 * 1024)
