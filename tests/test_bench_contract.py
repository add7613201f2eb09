"""bench.py contract helpers (CPU): the per-kernel algorithmic bytes are the
SURVEY 8(d) bytes split over the kernels of a step (intermediates excluded),
both arms print the same config dict, the batch shards cover the global
batch, and the committed traffic tables parse."""
import glob
import json
import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def _kernels(cfg):
    fam, nu, bnd, j, q, dim = cfg[:6]
    if j == 10 and dim == 2:
        return ["wv_fwd", "wv_adj"]  # warp-per-vector kernels (M = 2^10, large batches)
    if dim == 2 or j <= 12:
        return ["small_fwd", "small_adj"]
    return ["wav_coarse", "idwt_pyr", "large_fwd1", "large_fwd2", "large_adj2", "large_adj1", "dwt_pyr"]


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_kernel_bytes_sum_to_the_path_bytes(cfg):
    import bench
    c = bench.CONFIGS[cfg]
    batch = c[7]
    total = sum(bench.algorithmic_bytes(c, k, batch) for k in _kernels(c))
    assert total == 2 * batch * bench.path_bytes(c)
    assert max(bench.algorithmic_bytes(c, k, batch) for k in _kernels(c)) > 0


def test_normal_form_bytes():
    import bench
    c = bench.CONFIGS[5]
    assert bench.algorithmic_bytes(c, "normal_rows", 1) == 16.0 * (1 << 24) * 2 * bench.CFG5_ITERS


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_shards_cover_the_batch(cfg, world):
    import bench
    got = [bench.shard(cfg, world, r) for r in range(world)]
    if cfg in (2, 3, 4) and world > 1:
        pos = 0
        for s, n in got:
            assert s == pos and n > 0
            pos += n
        assert pos == bench.CONFIGS[cfg][7]
    else:
        assert all(g == (0, bench.CONFIGS[cfg][7]) for g in got)


def test_default_config_is_the_2_23_target():
    import bench
    c = bench.CONFIGS[bench.DEFAULT_CONFIG]
    assert (c[3], c[4], c[7]) == (21, 2, 32)


def test_config_dict_is_arm_independent():
    import bench
    for cfg in bench.CONFIGS:
        for w in (1, 2, 8):
            assert bench.config_dict(cfg, w) == json.loads(json.dumps(bench.config_dict(cfg, w)))


def test_traffic_table_entries():
    for path in glob.glob(os.path.join(REPO, "profiles", "r*_traffic.json")):
        tr = json.load(open(path))
        for cfg, entries in tr.items():
            if cfg == "source":
                continue
            entries = entries if isinstance(entries, list) else [entries]
            assert entries and all(e["bytes"] > 0 and e["kernel"] for e in entries), path
