"""Frame schedules and discrepancy weights (inputs)."""
from __future__ import annotations

import numpy as np


def _blocks(blocks):
    """[(count, seconds), ...] -> (start_min, dur_min) float64 arrays, contiguous from t=0."""
    durs = []
    for count, sec in blocks:
        durs += [sec / 60.0] * count
    dur = np.array(durs, dtype=np.float64)
    start = np.concatenate([[0.0], np.cumsum(dur)[:-1]])
    return start, dur


def fdg22():
    """Config 1: 22 frames over 50 min: 8x15 s, 4x60 s, 4x120 s, 6x360 s."""
    return _blocks([(8, 15), (4, 60), (4, 120), (6, 360)])


def tb35():
    """Config 4: 35 frames over 50 min: 12x10 s, 6x30 s, 5x60 s, 12x200 s (P:269 count)."""
    return _blocks([(12, 10), (6, 30), (5, 60), (12, 200)])


def uniform_frames(n: int, seconds: float = 60.0):
    """n contiguous frames of equal length (config 2: 61x60 s; config 3: 90x60 s)."""
    return _blocks([(n, seconds)])


def decay_weights(start, dur, half_life_min: float) -> np.ndarray:
    """w_f = dt_f exp(-lambda mid_f), normalised to mean 1 (FP32).

    Reading (R6): the inverse of sigma_t^2 / C_t of the P:220 noise model with the
    data-dependent C_t dropped.  The method takes w as an input; this only generates it.
    """
    lam = np.log(2.0) / half_life_min
    mid = np.asarray(start) + 0.5 * np.asarray(dur)
    w = np.asarray(dur) * np.exp(-lam * mid)
    w = w / w.mean()
    return w.astype(np.float32)
