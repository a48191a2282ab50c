"""Seeded synthetic inputs (SURVEY.md §8(d) "Ray sets"): camera rays are deterministic bit for bit
(generated once on the host, the same bits for the oracle and the GPU), and bench.py records the
SHA-256 of every ray buffer it traces."""
from __future__ import annotations

import hashlib

import numpy as np

from inputs import rays as R


def _sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_camera_rays_are_deterministic():
    for name in ("menger", "terrain", "city", "sparse"):
        a, pa = R.camera(name, scale=16)
        b, pb = R.camera(name, scale=16)
        assert a.dtype == np.float32 and a.shape[1] == 8
        assert _sha(a) == _sha(b) and np.array_equal(pa, pb)


def test_adversarial_and_random_sets_are_seeded():
    assert _sha(R.adversarial_rays(2000, (64, 64, 64), 7)) == _sha(R.adversarial_rays(2000, (64, 64, 64), 7))
    assert _sha(R.adversarial_rays(2000, (64, 64, 64), 7)) != _sha(R.adversarial_rays(2000, (64, 64, 64), 8))
    assert _sha(R.random_rays(2000, (64, 64, 64), 3)) == _sha(R.random_rays(2000, (64, 64, 64), 3))
