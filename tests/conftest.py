"""Shared pytest configuration: the `gpu` marker and golden-fixture helpers."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def golden_names():
    return sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz"))


def load_golden(name):
    """Return (D, meta, arrays) for one fixture; regenerates D when the
    fixture stores generator arguments instead of the matrix."""
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    arrs = {k: z[k] for k in z.files if k not in ("meta", "D")}
    if "D" in z.files:
        D = z["D"]
    else:
        from oracle.ircur_oracle import baseline_problem
        g = meta["gen"]
        D = baseline_problem(g["n1"], g["n2"], g["rank"], g["alpha"], g["seed"])[0]
    return D, meta, arrs


def solver_kwargs(meta):
    keys = ("rank", "eps", "zeta0", "gamma", "c_rows", "c_cols", "mode", "max_iter", "seed")
    return {k: meta[k] for k in keys if k in meta}


@pytest.fixture(scope="session")
def golden():
    return load_golden


def pytest_sessionfinish(session, exitstatus):
    """Write the parity records (flip counts, worst errors) of this session
    to gpurun_out/parity_stats.json (tests/parity.py)."""
    try:
        import parity
    except Exception:
        return
    if not parity.STATS:
        return
    out = os.path.join(ROOT, "gpurun_out")
    path = os.path.join(out, "parity_stats.json")
    try:
        os.makedirs(out, exist_ok=True)
        old = []
        if os.path.exists(path):  # several pytest sessions in one call: append
            with open(path) as f:
                old = json.load(f)
        with open(path, "w") as f:
            json.dump(old + parity.STATS, f, indent=1, default=float)
    except OSError:
        pass
