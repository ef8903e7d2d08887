"""Video background/foreground frames on the device vs the reference's
run_video chunk computation (cli.py:217-230) evaluated on the oracle's
factors (cur_eval_cols association, matrix_to_frames rounding)."""

import numpy as np
import pytest

from oracle import ircur_oracle as orc

pytestmark = pytest.mark.gpu


def ref_frames(C, W, V, inv, R, D, cols, h, w):
    low = C @ (V @ ((W.T @ R[:, cols]) * inv[:, None]))   # cur_eval_cols (solver.py:189-195)
    resid = np.abs(D[:, cols] - low)
    peaks = resid.max(axis=0)
    peaks[peaks == 0.0] = 1.0
    fg = resid * (255.0 / peaks)
    to8 = lambda M: np.clip(np.rint(M), 0, 255).astype(np.uint8).reshape((h, w, M.shape[1]), order="F").transpose(2, 0, 1)  # noqa: E731
    return to8(low), to8(fg)


def test_video_frames_match_reference(tmp_path):
    import paper_2010_07422_b200 as ir
    from paper_2010_07422_b200 import _build, video
    from paper_2010_07422_b200.gen import video_problem
    _build.build()
    h, w, f = 24, 32, 120
    D, L, S = video_problem(frames=f, height=h, width=w, rank=2, n_blocks=3, block=6, seed=1, dtype=np.float64)
    D = D * 100.0 + 50.0  # pixel-like range so rounding and clamping matter
    cfg = ir.SolverConfig(rank=2, eps=1e-9, gamma=0.7, mode="resampled", max_iter=60, seed=ir.RngSeed(3))
    ref = orc.solve(D, rank=2, eps=1e-9, gamma=0.7, mode="resampled", max_iter=60, seed=3)
    trace, bg, fg = video.run_video_device(D, cfg, h, w, chunk=50)
    assert trace.iterations == ref.iterations
    rbg, rfg = [], []
    for s in range(0, f, 50):
        a, b = ref_frames(ref.C, ref.W, ref.V, ref.inv_sigma, ref.R, D, np.arange(s, min(s + 50, f)), h, w)
        rbg.append(a)
        rfg.append(b)
    rbg, rfg = np.concatenate(rbg), np.concatenate(rfg)
    for mine, theirs in ((bg, rbg), (fg, rfg)):
        assert mine.shape == theirs.shape == (f, h, w)
        diff = np.abs(mine.astype(int) - theirs.astype(int))
        assert diff.max() <= 1 and (diff > 0).mean() <= 1e-3  # only rounding ties
    trace2, _, _ = video.run_video_device(D, cfg, h, w, chunk=50, out_dir=tmp_path)
    pgm = (tmp_path / "foreground" / "frame_00007.pgm").read_bytes()
    assert pgm.startswith(f"P5\n{w} {h}\n255\n".encode()) and pgm.endswith(fg[7].tobytes())
