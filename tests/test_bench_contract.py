"""bench.py contract helpers (CPU): every kernel the bench can name as the
dominant one has algorithmic bytes, and the committed traffic table parses."""
import json
import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_algorithmic_bytes_cover_the_kernels(cfg):
    import bench
    c = bench.CONFIGS[cfg]
    fam, nu, bnd, j, q, dim, r0, batch = c[:8]
    if cfg == 5:
        names = ["normal_rows", "transpose"]
    elif dim == 2 or j <= 12:
        names = ["small_fwd", "small_adj"]
    else:
        names = ["idwt_pyr", "dwt_pyr", "wav_coarse", "large_fwd1", "large_fwd2", "large_adj2", "large_adj1"]
    for k in names:
        assert bench.algorithmic_bytes(c, k, batch) > 0, k


def test_traffic_table_entries():
    tr = json.load(open(os.path.join(REPO, "profiles", "r01_traffic.json")))
    for cfg in "12345":
        entries = tr[cfg] if isinstance(tr[cfg], list) else [tr[cfg]]
        assert entries and all(e["bytes"] > 0 and e["kernel"] for e in entries)
