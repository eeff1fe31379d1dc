"""Counter-based random stream used to draw S and D (oracle side).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper fixes only the *distribution* of the draws: "independently for each
j in [n], we sample without replacement i_1..i_s in [m] uniformly at random and
let S_{i_k j} = +-1/sqrt(s)" and "D is a random n x n diagonal
matrix with +-1 independent entries ... S_h ... independent of D" (P:L793,
P:L799).  It is silent on the generator.  DESIGN.md reading R1 fixes one so that
bucket lists can be compared bit-exactly:

    mix64(z)     = splitmix64 finaliser (Steele, Lea & Flood 2014)
    u(key, ctr)  = mix64(key + (ctr + 1) * GAMMA)  mod 2^64
                 = output number ctr+1 of a splitmix64 generator whose state
                   starts at ``key``
    key_HASH     = mix64(seed ^ 0x48415348)   ("HASH")
    key_DIAG     = mix64(seed ^ 0x44494147)   ("DIAG")

Pinned by the public splitmix64 known answers for state 0
(tests/golden/splitmix64_kat.txt).  Two implementations live here, a pure-Python
one on ints (``mix64``, ``u``) and a NumPy one on uint64 arrays (``mix64_np``,
``u_np``); tests check that they agree.
"""
import numpy as np

MASK64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15
C1 = 0xBF58476D1CE4E5B9
C2 = 0x94D049BB133111EB
LABEL_HASH = 0x48415348
LABEL_DIAG = 0x44494147


def mix64(z):
    """splitmix64 finaliser on a Python int (mod 2^64)."""
    z &= MASK64
    z ^= z >> 30
    z = (z * C1) & MASK64
    z ^= z >> 27
    z = (z * C2) & MASK64
    z ^= z >> 31
    return z


def u(key, ctr):
    """Output number ctr+1 of splitmix64 started at state ``key`` (Python ints)."""
    return mix64((key + (ctr + 1) * GAMMA) & MASK64)


def key_hash(seed):
    """Stream key for the rows and signs of S_h (R1)."""
    return mix64((seed & MASK64) ^ LABEL_HASH)


def key_diag(seed):
    """Stream key for the diagonal D, independent of S_h."""
    return mix64((seed & MASK64) ^ LABEL_DIAG)


def mulhi(x, m):
    """floor(x * m / 2^64): maps a 64-bit uniform to [0, m) (Python ints)."""
    return (x * m) >> 64


# ---------------------------------------------------------------- NumPy versions
_U64 = np.uint64


def mix64_np(z):
    """splitmix64 finaliser on a uint64 array (NumPy wraps mod 2^64)."""
    z = np.asarray(z, dtype=_U64).copy()
    with np.errstate(over="ignore"):
        z ^= z >> _U64(30)
        z *= _U64(C1)
        z ^= z >> _U64(27)
        z *= _U64(C2)
        z ^= z >> _U64(31)
    return z


def u_np(key, ctr):
    """Vectorised ``u``: key is a Python int, ctr a uint64 array."""
    ctr = np.asarray(ctr, dtype=_U64)
    with np.errstate(over="ignore"):
        z = _U64(key) + (ctr + _U64(1)) * _U64(GAMMA)
    return mix64_np(z)


def mulhi_np(x, m):
    """floor(x * m / 2^64) for uint64 array x and 1 <= m < 2^32."""
    if not (1 <= m < (1 << 32)):
        raise ValueError("m out of range for mulhi_np")
    x = np.asarray(x, dtype=_U64)
    mm = _U64(m)
    hi = x >> _U64(32)
    lo = x & _U64(0xFFFFFFFF)
    with np.errstate(over="ignore"):
        # x*m = hi*m*2^32 + lo*m; both hi*m and lo*m fit in 64 bits since m < 2^32
        t = hi * mm + ((lo * mm) >> _U64(32))
    return t >> _U64(32)
