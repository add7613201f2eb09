"""Generates tests/golden/golden.npz from the UNMODIFIED reference library
(oracle/_ref/libcwwref.so, built by oracle/Makefile from /root/reference).

Run here (the reference exists only in this container):
    python tests/golden/make_golden.py
The committed fixture pins the oracle restatement on the GPU box, where
/root/reference does not exist.  Inputs use the oracle's test_rng port
(seeded normals), which tests/test_oracle.py checks against the reference's
generator semantics."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(REPO, "oracle"))
from oracle_py import Oracle, Reference  # noqa: E402

# (family, nu, boundary, j, q, dim, r0)
CASES = [
    (0, 2, 1, 3, 1, 1, -1), (0, 2, 1, 6, 1, 1, 3), (0, 3, 1, 5, 2, 1, 4), (0, 4, 1, 6, 2, 1, 4),
    (0, 4, 1, 4, 1, 1, -1), (0, 5, 1, 5, 1, 1, -1), (0, 6, 1, 6, 2, 1, -1), (1, 3, 1, 6, 1, 1, -1),
    (1, 4, 1, 5, 3, 1, -1), (0, 2, 0, 5, 1, 1, -1), (0, 3, 0, 6, 2, 1, -1), (1, 6, 0, 6, 1, 1, -1),
    (0, 1, 0, 10, 1, 1, 1), (0, 1, 0, 6, 0, 1, 0), (0, 1, 0, 7, 2, 1, 3),
    (0, 2, 1, 4, 1, 2, 3), (0, 4, 1, 4, 1, 2, 4), (0, 3, 0, 4, 1, 2, -1),
]

# (family, nu, boundary, j, q, dim, sampled fraction) for masked ComposedOps
MASKED = [(0, 2, 1, 5, 1, 1, 0.25), (0, 4, 1, 6, 2, 1, 0.1), (1, 3, 0, 6, 1, 1, 0.5),
          (0, 3, 1, 4, 1, 2, 0.2)]

# kernel-cache fixtures (family, nu, boundary, q)
CWWK = [(0, 2, 1, 1), (1, 3, 0, 3), (0, 4, 1, 2)]


def main():
    o, r = Oracle(), Reference()
    out = {}
    for ci, (fam, nu, bnd, j, q, dim, r0) in enumerate(CASES):
        op = r.op(fam, nu, bnd, j, q, dim, r0)
        x = o.normals(7000 + ci, op.nin)
        y = o.normals(8000 + ci, op.nout)
        key = f"c{ci}"
        out[key + "_case"] = np.array([fam, nu, bnd, j, q, dim, r0])
        out[key + "_x"] = x
        out[key + "_y"] = y
        for use in (0, 1):
            if nu == 1 and use == 0 and q == 0:
                continue
            out[key + f"_fwd{use}"] = op.forward(x, use)
            out[key + f"_adj{use}"] = op.adjoint(y, use)
    # kernel tables
    for fam in (0, 1):
        for nu in range(2, 7):
            for bnd in (0, 1):
                for q in (1, 2, 3):
                    it, le, ri = r.kernel_table(fam, nu, bnd, q)
                    k = f"k_{fam}_{nu}_{bnd}_{q}"
                    out[k + "_int"], out[k + "_left"], out[k + "_right"] = it, le, ri
    # FWHT / sign rows / DWT known vectors
    v = o.normals(42, 1 << 10)
    out["fwht_in"] = v
    out["fwht_seq"] = r.fwht_sequency(v)
    out["fwht_nat"] = r.fwht_natural(v)
    out["perm_13"] = np.array([r.seq_to_nat(n, 13) for n in range(1 << 13)], dtype=np.int64)
    out["sign_j6"] = np.stack([r.sign_row(p, 6) for p in range(64)])
    for nu, bnd, j, r0 in [(2, 1, 7, 3), (4, 1, 8, 4), (3, 0, 7, -1), (1, 0, 8, 0), (6, 1, 7, -1)]:
        x = o.normals(900 + nu * 10 + bnd, 1 << j)
        k = f"dwt_{nu}_{bnd}_{j}_{r0}"
        out[k + "_x"] = x
        out[k + "_fwd"] = r.dwt(0, nu, bnd, j, x, 0, r0)
        out[k + "_inv"] = r.dwt(0, nu, bnd, j, x, 1, r0)
    # subsampled ComposedOp (SamplingMask; the reference's ComposedOp uses r0 = J0)
    rng = np.random.default_rng(2106)
    for mi, (fam, nu, bnd, j, q, dim, frac) in enumerate(MASKED):
        op = r.op(fam, nu, bnd, j, q, dim, -1)
        cnt = max(1, int(frac * op.nout))
        mask = np.sort(rng.choice(op.nout, cnt, replace=False)).astype(np.uint64)
        x = o.normals(9100 + mi, op.nin)
        y = o.normals(9200 + mi, cnt)
        k = f"m{mi}"
        out[k + "_case"] = np.array([fam, nu, bnd, j, q, dim])
        out[k + "_mask"] = mask
        out[k + "_x"] = x
        out[k + "_y"] = y
        for use in (0, 1):
            out[k + f"_fwd{use}"] = op.masked(mask, x, adjoint=False, use_idwt=use)
            out[k + f"_adj{use}"] = op.masked(mask, y, adjoint=True, use_idwt=use)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    # CWWK kernel-cache files written by the reference's save_kernel_table
    for fam, nu, bnd, q in CWWK:
        name = f"cwwk_{'db' if fam == 0 else 'sym'}{nu}_{'vmp' if bnd else 'periodic'}_q{q}_R14_v1.bin"
        r.kernel_cache_save(fam, nu, bnd, q, os.path.join(HERE, name))
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
