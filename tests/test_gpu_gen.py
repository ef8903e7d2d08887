"""Device synthetic generator (ircur_gen_baseline) == the numpy generator
of oracle.baseline_problem_blocked, bit for bit, including row shards."""

import numpy as np
import pytest
import torch

from oracle import ircur_oracle as orc
from paper_2010_07422_b200 import gen

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("shape", [(257, 193), (64, 1000)])
def test_device_generator_bitwise(dtype, shape):
    n1, n2 = shape
    D, linf, a = orc.baseline_problem_blocked(n1, n2, 4, 0.2, 9, dtype=dtype, block_rows=50)
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    Dd, linf_d, a_d = gen.baseline_problem_device(n1, n2, 4, 0.2, 9, dtype=tdt)
    np.testing.assert_array_equal(Dd.cpu().numpy(), D)
    assert linf_d == linf and a_d == a


def test_device_generator_row_shards():
    n1, n2 = 301, 211
    D, linf, a = orc.baseline_problem_blocked(n1, n2, 3, 0.1, 4)
    stats = []
    for r0, nl in ((0, 100), (100, 150), (250, 51)):
        mx, q = gen._call(None, 1, n2, n1, n2, r0, nl, 3, *_factors(n1, n2, 3, 4), 0.1, 0.0,
                          gen.factors(n1, n2, 3, 4)[2], torch.cuda.current_stream().cuda_stream)
        stats.append((mx, q))
    tot = (max(s[0] for s in stats), sum(s[1] for s in stats))

    def reduce(mx, q):
        return tot

    parts = [gen.baseline_problem_device(n1, n2, 3, 0.1, 4, dtype=torch.float64, row0=r0, nrows=nl,
                                         stats_reduce=reduce)
             for r0, nl in ((0, 100), (100, 150), (250, 51))]
    np.testing.assert_array_equal(torch.cat([p[0] for p in parts]).cpu().numpy(), D)
    assert all(p[1] == linf and p[2] == a for p in parts)


def _factors(n1, n2, r, seed):
    W, V, _ = gen.factors(n1, n2, r, seed)
    return torch.from_numpy(W).cuda(), torch.from_numpy(V).cuda()
