"""cfg5 — BASELINE.json's headline problem — against the CPU oracle at full size.

n1 = n2 = 1e5 fp32 (40 GB), r = 10, alpha = 0.2, gamma = 0.7, eps = 1e-5,
resampled, zeta0 = max|L|, data seed 0, solver seed 1: exactly the bench.py
workload.  The host copy of D comes from the numpy generator
(`orc.baseline_problem_blocked`), the device copy from the device generator,
which reproduces it bit for bit (tests/test_gpu_gen.py).  The oracle
(the reference loop, solver.py:304-416, in fp64 arithmetic on the fp32
values) runs to tol on the host's cores, about a minute.

Checked (tests/parity.py): identical index sets, per-iteration set sizes and
thresholds; the iteration count within one (fp32) and the strips compared at
the oracle's iteration; e_k; C, R, S_rows, S_cols over the whole strips at
1e-4; the outlier-support flip count and its distance to the threshold; and
L = C U^+ R on four random 2000 x 2000 blocks.  The oracle's measured wall
time is written to gpurun_out/cfg5_oracle.json (the measured CPU time behind
bench.py's cpu_baseline).
"""

import json
import os
import time

import numpy as np
import pytest
import torch

from oracle import ircur_oracle as orc
import parity

pytestmark = pytest.mark.gpu

N, RANK, ALPHA, GAMMA, EPS = 100000, 10, 0.2, 0.7, 1e-5
DATA_SEED, SOLVER_SEED = 0, 1


def _L_block(C, W, V, inv, R, ri, ci):
    # L(ri, ci) = C(ri,:) V diag(inv) W^T R(:, ci)  (solver.py:211-213)
    return C[ri] @ (V @ ((W.T @ R[:, ci]) * inv[:, None]))


def test_cfg5_matches_oracle():
    import paper_2010_07422_b200 as ir
    from paper_2010_07422_b200 import _build, gen

    _build.build()
    if torch.cuda.get_device_properties(0).total_memory < 60e9:
        pytest.skip("cfg5 needs a B200-class device")
    t0 = time.perf_counter()
    Dh, linf, _ = orc.baseline_problem_blocked(N, N, RANK, ALPHA, DATA_SEED, dtype=np.float32)
    t_gen = time.perf_counter() - t0
    kw = dict(rank=RANK, eps=EPS, zeta0=linf, gamma=GAMMA, mode="resampled", max_iter=100)
    iter_s = []

    def on_iter(k, sec):
        iter_s.append(sec)
        return False

    t0 = time.perf_counter()
    ref = orc.solve(Dh, seed=SOLVER_SEED, upcast=False, record_x=True, on_iter=on_iter, **kw)
    t_oracle = time.perf_counter() - t0
    iter_s.append(None)  # the converging iteration returns before on_iter

    Dd, linf_d, _ = gen.baseline_problem_device(N, N, RANK, ALPHA, DATA_SEED, dtype=torch.float32)
    assert linf_d == linf
    # spot check: the device matrix is the host matrix
    rows = np.random.default_rng(3).choice(N, 8, replace=False)
    np.testing.assert_array_equal(Dd[torch.from_numpy(rows).cuda()].cpu().numpy(), Dh[rows])

    def resolve(mi, e):
        cfg = ir.SolverConfig(seed=ir.RngSeed(SOLVER_SEED), **{**kw, "max_iter": mi, "eps": e})
        return ir.solve(Dd, cfg, device=0)

    out = resolve(kw["max_iter"], EPS)
    rec = parity.check(out, ref, True, resolve=resolve, name="cfg5")
    cur, sp, tr = resolve(ref.iterations, 1e-300) if out[2].iterations != ref.iterations else out
    rng = np.random.default_rng(5)
    blocks = []
    for _ in range(4):
        ri = np.sort(rng.choice(N, 2000, replace=False))
        ci = np.sort(rng.choice(N, 2000, replace=False))
        pf = cur.core_pinv
        Lm = _L_block(cur.C, pf.W, pf.V, pf.inv_sigma, cur.R, ri, ci)
        Lr = _L_block(ref.C, ref.W, ref.V, ref.inv_sigma, ref.R, ri, ci)
        blocks.append(parity.rel(Lm, Lr))
    rec["rel_L_blocks"] = blocks
    report = {"config": "cfg5", "n1": N, "n2": N, "rank": RANK, "alpha": ALPHA, "gamma": GAMMA,
              "eps": EPS, "mode": "resampled", "cores": os.cpu_count(),
              "oracle_seconds": t_oracle, "oracle_iterations": ref.iterations,
              "oracle_iter_seconds": iter_s, "host_generation_seconds": t_gen,
              "oracle_note": "oracle port (fp64 arithmetic, strips upcast per gather; the reference's "
                             "whole-matrix fp64 upcast + finite check is not included)",
              "gpu_iterations": out[2].iterations, "gpu_errors": list(out[2].errors),
              "oracle_errors": list(ref.errors), "parity": rec}
    os.makedirs("gpurun_out", exist_ok=True)
    with open(os.path.join("gpurun_out", "cfg5_oracle.json"), "w") as f:
        json.dump(report, f, indent=1, default=float)
    assert max(blocks) <= 1e-4, blocks
    del Dd
    ir.clear_cache()
    torch.cuda.empty_cache()
