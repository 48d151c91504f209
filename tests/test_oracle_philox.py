"""Pins for oracle/philox.py (CPU)."""
import numpy as np
import pytest

from oracle import philox

# Known-answer vectors for Philox4x32-10 published with Random123 (Salmon et al., SC'11;
# the kat_vectors file of the Random123 distribution): (counter, key) -> output.
KAT = [
    ((0x00000000, 0x00000000, 0x00000000, 0x00000000), (0x00000000, 0x00000000),
     (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF), (0xFFFFFFFF, 0xFFFFFFFF),
     (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("ctr,key,out", KAT)
def test_philox_known_answers(ctr, key, out):
    got = philox.philox4x32_10(*ctr, *key)
    assert tuple(int(x) for x in got) == out


def test_philox_vectorised_matches_scalar():
    rng = np.random.default_rng(0)
    c = rng.integers(0, 2**32, size=(4, 64), dtype=np.uint64)
    k0, k1 = 0x12345678, 0x9ABCDEF0
    vec = philox.philox4x32_10(c[0], c[1], c[2], c[3], k0, k1)
    for t in range(64):
        sc = philox.philox4x32_10(int(c[0, t]), int(c[1, t]), int(c[2, t]), int(c[3, t]), k0, k1)
        assert tuple(int(v[t]) for v in vec) == tuple(int(s) for s in sc)


def test_stream_layout_distinguishes_purposes_and_is_uniform():
    idx = np.arange(200_000, dtype=np.uint64)
    a = philox.stream(7, philox.PURPOSE_INIT, 0, 2, 0, idx)
    b = philox.stream(7, philox.PURPOSE_REGROW, 0, 2, 0, idx)
    assert not np.array_equal(a[0], b[0])
    u = a[0].astype(np.float64) / 2**32
    # mean and variance of U(0,1) within 6 sigma
    n = len(u)
    assert abs(u.mean() - 0.5) < 6 * np.sqrt(1 / 12 / n)
    assert abs(u.var() - 1 / 12) < 0.002
    # 64-bit counter: the high word of idx is used
    hi = philox.stream(7, 1, 0, 2, 0, np.array([1 << 32], dtype=np.uint64))
    lo = philox.stream(7, 1, 0, 2, 0, np.array([0], dtype=np.uint64))
    assert int(hi[0][0]) != int(lo[0][0])
