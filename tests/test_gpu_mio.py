"""BIN matrix files to and from device memory (mio.py:66-121 format),
checked against a numpy restatement of the reference's writer and reader."""

import struct

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def write_ref(M, path):
    """The reference's write_matrix (mio.py:66-79) restated: header + F-order f8."""
    with open(path, "wb") as fh:
        fh.write(struct.pack("<4sii", b"IRCM", M.shape[0], M.shape[1]))
        fh.write(np.asarray(M, dtype="<f8").tobytes(order="F"))


@pytest.fixture(scope="module")
def mio():
    from paper_2010_07422_b200 import _build, mio as m
    _build.build()
    return m


@pytest.mark.parametrize("shape", [(1, 1), (37, 53), (300, 257), (1000, 70)])
@pytest.mark.parametrize("block_cols", [None, 7])
def test_read_bitexact_and_shards(mio, tmp_path, shape, block_cols):
    M = np.random.default_rng(sum(shape)).standard_normal(shape)
    p = tmp_path / "m.bin"
    write_ref(M, p)
    D = mio.read_matrix_device(p, block_cols=block_cols).cpu().numpy()
    np.testing.assert_array_equal(D, M)
    D32 = mio.read_matrix_device(p, dtype=torch.float32, block_cols=block_cols).cpu().numpy()
    np.testing.assert_array_equal(D32, M.astype(np.float32))
    if shape[0] > 2:
        r0, nr = shape[0] // 3, shape[0] // 2
        S = mio.read_matrix_device(p, row0=r0, nrows=nr, block_cols=block_cols).cpu().numpy()
        np.testing.assert_array_equal(S, M[r0:r0 + nr])


def test_write_round_trip_bytes(mio, tmp_path):
    M = np.random.default_rng(3).standard_normal((123, 77))
    a, b = tmp_path / "a.bin", tmp_path / "b.bin"
    write_ref(M, a)
    mio.write_matrix_device(torch.from_numpy(M).cuda(), b, block_cols=10)
    assert a.read_bytes() == b.read_bytes()
    M32 = M.astype(np.float32)
    mio.write_matrix_device(torch.from_numpy(M32).cuda(), b)
    write_ref(M32.astype(np.float64), a)
    assert a.read_bytes() == b.read_bytes()


def test_format_errors_match_reference_offsets(mio, tmp_path):
    M = np.arange(12.0).reshape(3, 4)
    p = tmp_path / "e.bin"
    write_ref(M, p)
    raw = p.read_bytes()
    cases = [
        (raw[:7], "truncated header", 7),
        (b"XXXX" + raw[4:], "bad magic", 0),
        (struct.pack("<4sii", b"IRCM", -1, 4) + raw[12:], "negative dimensions", 4),
        (raw[:-8], "truncated payload", len(raw) - 8),
        (raw + b"\0", "trailing bytes", len(raw)),
    ]
    for data, msg, off in cases:
        p.write_bytes(data)
        with pytest.raises(mio.FormatError, match=msg) as ei:
            mio.read_matrix_device(p)
        assert ei.value.offset == off
    # the first non-finite value in file (column-major) order
    M2 = M.copy()
    M2[2, 1] = np.nan   # flat file index 1*3 + 2 = 5
    M2[0, 3] = np.inf   # flat index 9
    M2[1, 0] = -np.inf  # flat index 1  <- first
    write_ref(M2, p)
    with pytest.raises(mio.FormatError, match="non-finite") as ei:
        mio.read_matrix_device(p, block_cols=1)
    assert ei.value.offset == 12 + 8 * 1


def test_read_then_solve_equals_array_solve(mio, tmp_path):
    import paper_2010_07422_b200 as ir
    from oracle.ircur_oracle import baseline_problem
    D = baseline_problem(180, 150, 3, 0.1, 6)[0]
    p = tmp_path / "d.bin"
    write_ref(D, p)
    cfg = ir.SolverConfig(rank=3, gamma=0.7, mode="resampled", seed=ir.RngSeed(2))
    a = ir.solve(mio.read_matrix_device(p), cfg)
    b = ir.solve(D, cfg, device=0)
    assert a[2].errors == b[2].errors
    np.testing.assert_array_equal(a[0].C, b[0].C)
