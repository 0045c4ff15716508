"""Philox4x32-10 (oracle/philox.py) pinned to the published known-answer vectors
(tests/golden/philox_kat.json) and Box-Muller to the N(0,1) moments."""
import json
import os

import numpy as np

from oracle.philox import gaussian_block, philox4x32_10

KAT = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "philox_kat.json")))


def test_known_answer_vectors():
    for v in KAT["vectors"]:
        c = [int(x, 16) for x in v["ctr"]]
        k = [int(x, 16) for x in v["key"]]
        out = philox4x32_10(*c, *k)
        assert [int(x) for x in out] == [int(x, 16) for x in v["out"]]


def test_vectorised_equals_scalar():
    i = np.arange(64, dtype=np.uint32)
    vec = np.stack(philox4x32_10(i, 3, 4, 5, 77, 88), axis=1)
    for j in (0, 17, 63):
        assert [int(x) for x in vec[j]] == [int(x) for x in philox4x32_10(j, 3, 4, 5, 77, 88)]


def test_gaussian_moments_and_determinism():
    E = gaussian_block(2000, 50, seed=123, stream=4, ctx=1, tag=2)
    assert E.shape == (2000, 50)
    z = E.ravel()
    assert abs(z.mean()) < 4 / np.sqrt(z.size)
    assert abs(z.var() - 1) < 6 * np.sqrt(2 / z.size)
    assert abs(np.mean(z ** 4) - 3) < 0.1  # Gaussian kurtosis
    assert np.array_equal(E, gaussian_block(2000, 50, seed=123, stream=4, ctx=1, tag=2))
    assert not np.array_equal(E, gaussian_block(2000, 50, seed=123, stream=4, ctx=1, tag=3))
    # column-major linear index: prefix of a taller block is NOT the same; same n, fewer cols is
    assert np.array_equal(E[:, :10], gaussian_block(2000, 10, seed=123, stream=4, ctx=1, tag=2))
