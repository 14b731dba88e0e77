"""The generator is deterministic and bit-identical to the pinned manifest (synth/volumes.py)."""
import numpy as np
import pytest

from synth import volumes as V


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_manifest_small(name):
    c = V.generate(name)
    spec = V.CONFIGS[name]
    assert c.shape == (spec.X, spec.Y, spec.Z) and c.dtype == np.int32
    assert c.min() >= 0 and c.max() <= 255
    assert V.sha256_volume(c) == V.MANIFEST[name]


def test_chunking_invariant():
    a = V.generate("C2", x_chunk=128)
    b = V.generate("C2", x_chunk=7)
    assert np.array_equal(a, b)


def test_dsin_accuracy():
    t = np.linspace(-20, 20, 2001)
    assert np.max(np.abs(V.dsin(t) - np.sin(t))) < 1e-14
    assert np.max(np.abs(V.dcos(t) - np.cos(t))) < 1e-14


def test_noise_moments():
    n = V.noise(9, np.arange(200000, dtype=np.uint64))
    assert abs(n.mean()) < 0.01 and abs(n.std() - 1.0) < 0.01


def test_tiny_cases_ranges():
    for seed in range(1000, 1200):
        c, d = V.tiny_case(seed)
        X, Y, Z = c.shape
        assert 1 <= X <= 5 and 1 <= Y <= 5 and 1 <= Z <= 12 and 0 <= d <= 4
