"""The planner's pass-width cap (SKH_FWHT_KMAX) only changes how
the stages are grouped into HBM passes: every cap stays bit-identical to the
oracle.  The cap is read once per process, so each runs in a subprocess."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import numpy as np, torch, sys
sys.path.insert(0, %r)
import paper_2105_11815_b200 as skh
from oracle import hadamard, sketch
ok = True
for (nrows, nvalid, d, lo, hi, diag, row0) in [(2048, 2000, 64, 0, 11, True, 0), (4096, 4096, 96, 1, 11, False, 0),
                                            (1 << 14, 1 << 14, 64, 0, 14, True, 3), (512, 512, 130, 0, 9, True, 0)]:
    X = np.random.default_rng(nrows + d).standard_normal((nvalid, d))
    Y = skh.rht_stages(77, torch.from_numpy(X).cuda(), lo, hi, nrows=nrows, row0=row0, apply_diag=diag).cpu().numpy()
    Z = np.zeros((nrows, d)); Z[:nvalid] = X
    if diag:
        Z[:nvalid] *= hadamard.diag_signs(77, np.arange(row0, row0 + nvalid))[:, None].astype(float)
    hadamard.fwht_stages(Z, lo, hi)
    ok &= np.array_equal(Y.view(np.int64), Z.view(np.int64))
A = np.random.default_rng(1).standard_normal((1 << 13, 64))
SA, _ = skh.rht_dense(5, torch.from_numpy(A).cuda(), None, 112, 1)
ok &= np.array_equal(SA.cpu().numpy(), sketch.rht_sketch(5, A, None, 112, 1)[0])
print("OK" if ok else "MISMATCH")
"""


@pytest.mark.parametrize("kmax", ["4", "8", "11"])
def test_pass_width_cap_bitexact(kmax):
    import paper_2105_11815_b200.build as b
    b.build()
    env = dict(os.environ, SKH_FWHT_KMAX=kmax)
    r = subprocess.run([sys.executable, "-c", SCRIPT % ROOT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().endswith("OK"), r.stdout[-2000:]
