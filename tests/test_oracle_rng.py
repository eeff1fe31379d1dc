"""Pins for oracle/rng.py (R1): public splitmix64 known answers and
agreement of the pure-Python and NumPy implementations."""
import numpy as np

from oracle import rng


def test_splitmix64_known_answers(golden):
    for ctr, val in golden("splitmix64_kat.txt"):
        assert rng.u(0, int(ctr)) == int(val, 16)
        assert int(rng.u_np(0, np.array([int(ctr)], dtype=np.uint64))[0]) == int(val, 16)


def test_numpy_matches_python():
    r = np.random.default_rng(0)
    ctr = r.integers(0, 2**63, size=500, dtype=np.uint64)
    for key in (0, 1, 0xDEADBEEF, rng.key_hash(5), rng.key_diag(5)):
        got = rng.u_np(key, ctr)
        want = [rng.u(key, int(c)) for c in ctr]
        assert [int(x) for x in got] == want


def test_mulhi_matches_exact():
    r = np.random.default_rng(1)
    x = r.integers(0, 2**64 - 1, size=2000, dtype=np.uint64, endpoint=True)
    x[:3] = [0, 2**64 - 1, 2**63]
    for m in (1, 2, 3, 7, 256, 1792, 7168, 16384, 2**31 - 1):
        got = rng.mulhi_np(x, m)
        want = [(int(v) * m) >> 64 for v in x]
        assert [int(g) for g in got] == want
        assert int(got.max()) < m


def test_domain_separation():
    # D must be independent of S_h: distinct keys per label and seed.
    keys = {rng.key_hash(s) for s in range(64)} | {rng.key_diag(s) for s in range(64)}
    assert len(keys) == 128
