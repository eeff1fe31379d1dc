"""hash_gen has two transposes: the stable LSD radix sort and the
count / fill / per-bucket-sort path used for short buckets.  Their output is the
unique canonical bucket list, so on the same inputs both must equal the oracle
bit for bit.  SKH_HASH_RADIX=1 forces the radix path (read once per process,
hence the subprocess)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import numpy as np, sys
sys.path.insert(0, %r)
import paper_2105_11815_b200 as skh
from oracle import hashing
ok = True
for (n, m, s, row0, blk, stride) in [(65536, 1792, 1, 0, 0, 0), (131072 // 8, 7168, 2, 0, 0, 0),
                                     (4096, 256, 2, 0, 0, 0), (3000, 64, 3, 7, 0, 0), (8000, 500, 2, 5, 100, 1000),
                                     (20000, 70000, 2, 0, 0, 0)]:
    k = np.arange(n)
    gid = row0 + k if blk <= 0 else row0 + (k // blk) * stride + (k % blk)
    bl = skh.hash_gen(31, m, s, n, row0=row0, blk=blk, stride=stride, want_cols=True)
    ptr, rows, signs = hashing.bucket_lists(31, gid, m, s)
    ok &= np.array_equal(bl.ptr.cpu().numpy(), ptr)
    ok &= np.array_equal(bl.rows.cpu().numpy(), rows)
    ok &= np.array_equal(bl.signs.cpu().numpy(), signs)
    cr, cs = hashing.draw_columns(31, gid, m, s)
    ok &= np.array_equal(bl.col_rows.cpu().numpy().reshape(n, s), cr)
print("OK" if ok else "MISMATCH")
"""


@pytest.mark.parametrize("force_radix", ["0", "1"])
def test_both_transposes_bitexact(force_radix):
    import paper_2105_11815_b200.build as b
    b.build()
    env = dict(os.environ, SKH_HASH_RADIX=force_radix)
    script = SCRIPT.replace("%r", repr(ROOT))
    r = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().endswith("OK"), r.stdout[-2000:]
