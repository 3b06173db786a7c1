"""The training harness's torch V-cycle (paper_2604_23265_b200/train.py MgNet, NEXT-4) against the fp64
oracle V-cycle on the CPU: same packed weights (R20), same data flow, so weights trained
through the torch copy mean the same network in mgnet_create / mgnet_vcycle; and the weight count matches
the oracle's packing.  Runs without a GPU."""
import numpy as np
import pytest

import workloads as W
from oracle import rte as O

torch = pytest.importorskip("torch")


@pytest.mark.parametrize("L,C0,N,M,nu", [(1, 8, 8, 4, 2), (3, 8, 16, 8, 2), (2, 16, 8, 8, 1)])
def test_torch_mgnet_equals_oracle_vcycle(L, C0, N, M, nu):
    from paper_2604_23265_b200 import train as TR
    rng = np.random.default_rng(L * 100 + C0)
    w = rng.normal(0.0, 0.05, TR.weight_count(M, L, C0, nu)).astype(np.float32)
    onet = O.make_mgnet(w, M, L, C0, nu)            # (validates the count against the oracle's packing)
    r = rng.standard_normal((2, N, N, M))
    z_ref = r + O.vcycle(onet, r, add_identity=False)
    net = TR.MgNet(M, L, C0, nu, w, device="cpu", dtype=torch.float64)
    with torch.no_grad():
        z = net(torch.from_numpy(r)).numpy()
    assert np.linalg.norm(z - z_ref) <= 1e-12 * np.linalg.norm(z_ref - r)
    assert np.array_equal(net.flat(), w)


def test_cosine_schedule_endpoints():
    from paper_2604_23265_b200 import train as TR
    assert TR.cosine_lr(0, 100) == pytest.approx(1e-3)
    assert TR.cosine_lr(50, 100) == pytest.approx(5e-4)
    assert TR.cosine_lr(100, 100) == pytest.approx(0.0, abs=1e-15)
