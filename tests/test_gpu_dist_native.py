"""Native multi-GPU entry points (csrc/cww_dist.cpp) on one GPU.

* cww_dist_*_local: the row partition of config 5 with P virtual ranks in one
  process (the same pack / unpack kernels; a device-copy exchange instead of
  NCCL), against the single-GPU normal operator of the whole image, which is
  itself checked against the compiled reference (test_gpu_reference.py).
* cww_dist_* over a real NCCL communicator of one rank.
* cww_multi_*: the batch split over two shards on device 0.
"""
import numpy as np
import pytest
import torch

import paper_2106_00554_b200 as cw
from paper_2106_00554_b200 import dist as cdist

pytestmark = pytest.mark.gpu


def _image(orc, j, r0, seed):
    return orc.synth(0, seed, j, r0, 0.02, 2)


def _full_normal(spec, j, q, r0, x, iters, dev):
    op = cw.ComposedOp(cw.FastOp(spec, j, q, 2), None, True, r0)
    t = torch.as_tensor(x, device=dev).clone()
    op.normal(t, iters=iters)
    return t.cpu().numpy()


@pytest.mark.parametrize("P", [1, 2, 4])
@pytest.mark.parametrize("iters", [1, 2, 3])
@pytest.mark.parametrize("case", [(2, 1, 7, 1, 3), (4, 1, 8, 1, 4), (3, 0, 6, 2, -1)])
def test_local_partition_matches_single_gpu(orc, cuda, P, iters, case):
    nu, bnd, j, q, r0 = case
    spec = cw.WaveletSpec(cw.Family.Daubechies, nu, cw.Boundary(bnd))
    M = 1 << j
    x = _image(orc, j, r0 if r0 >= 0 else spec.min_level(), 900 + j)
    want = _full_normal(spec, j, q, r0, x, iters, cuda)
    d = cdist.NativeRowPartitioned2D(spec, j, q, r0, nranks=P, local=True)
    m = M // P
    rows = [torch.as_tensor(x.reshape(M, M)[r * m:(r + 1) * m], device=cuda).contiguous() for r in range(P)]
    d.normal(rows, iters)
    got = torch.cat(rows).cpu().numpy().reshape(-1)
    err = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert err <= 1e-13, err


def test_local_partition_config5_shape(orc, cuda):
    """Config 5's exact shape (db2 VMP, r0 = 3, 4096^2, q = 1) on 4 virtual ranks."""
    spec = cw.WaveletSpec(cw.Family.Daubechies, 2, cw.Boundary.Vmp)
    j, q, r0, P = 12, 1, 3, 4
    M = 1 << j
    x = _image(orc, j, r0, 5000)
    want = _full_normal(spec, j, q, r0, x, 1, cuda)
    d = cdist.NativeRowPartitioned2D(spec, j, q, r0, nranks=P, local=True)
    m = M // P
    rows = [torch.as_tensor(x.reshape(M, M)[r * m:(r + 1) * m], device=cuda).contiguous() for r in range(P)]
    d.normal(rows, 1)
    got = torch.cat(rows).cpu().numpy().reshape(-1)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-13


@pytest.mark.parametrize("iters", [1, 2])
def test_nccl_single_rank(orc, cuda, iters):
    spec = cw.WaveletSpec(cw.Family.Daubechies, 2, cw.Boundary.Vmp)
    j, q, r0 = 8, 1, 3
    x = _image(orc, j, r0, 77)
    want = _full_normal(spec, j, q, r0, x, iters, cuda)
    d = cdist.NativeRowPartitioned2D(spec, j, q, r0, rank=0, nranks=1, nccl_id=cdist.nccl_unique_id())
    t = torch.as_tensor(x, device=cuda).clone()
    d.normal(t, iters)
    torch.cuda.synchronize()
    assert np.linalg.norm(t.cpu().numpy() - want) / np.linalg.norm(want) <= 1e-13


def test_dist_rejects_bad_partition(cuda):
    spec = cw.WaveletSpec(cw.Family.Daubechies, 2, cw.Boundary.Vmp)
    with pytest.raises(cw.CwwError) as e:
        cdist.NativeRowPartitioned2D(spec, 4, 1, 3, nranks=16, local=True)
    assert e.value.status == 2


@pytest.mark.parametrize("batch", [1, 3, 8])
def test_multi_device_shards(orc, cuda, batch):
    spec = cw.WaveletSpec(cw.Family.Daubechies, 3, cw.Boundary.Vmp)
    j, q, r0 = 14, 2, 4
    op = cw.ComposedOp(cw.FastOp(spec, j, q, 1), None, True, r0)
    mu = cdist.MultiDeviceOp(spec, j, q, 1, r0, [0, 0])
    x = np.stack([orc.synth(0, 10 + b, j, r0, 0.1, 1) for b in range(batch)])
    y = np.stack([orc.normals(20 + b, 1 << (j + q)) for b in range(batch)])
    fx, ay = mu.forward(x), mu.adjoint(y)
    assert np.array_equal(fx, op.forward(x)) and np.array_equal(ay, op.adjoint(y))
