"""The five BASELINE.json workloads (shapes and structure only).

C1-C5 follow BASELINE.json ``configs`` in order; they stand in for the paper's
Test Sets 1-2.  The Florida collection (Test Set 3)
is not available and is not reproduced.
"""
from dataclasses import dataclass


@dataclass(frozen=True)
class Workload:
    name: str
    kind: str          # dense_gauss | dense_coherent | csr
    n: int
    d: int
    m: int
    s: int
    seed: int
    hd: bool           # apply D + Walsh-Hadamard before hashing
    nnz_row: int = 0   # CSR only
    note: str = ""

    @property
    def a_bytes(self):
        """Bytes of A as streamed: n*d*8 dense; CSR = val + col_idx + row_ptr."""
        if self.kind == "csr":
            nnz = self.n * self.nnz_row
            return nnz * 8 + nnz * 4 + (self.n + 1) * 8
        return self.n * self.d * 8

    def scaled(self, n=None, d=None, m=None, name=None):
        """A smaller replica with the same structure (for parity at test size)."""
        return Workload(name or self.name + "-small", self.kind, n or self.n, d or self.d,
                        m or self.m, self.s, self.seed, self.hd, self.nnz_row, self.note)


C1 = Workload("C1", "dense_gauss", 4096, 64, 256, 2, 1, False,
              note="Dense A 4096x64 iid N(0,1), b N(0,1); s=2, m=256; seed 1")
C2 = Workload("C2", "dense_gauss", 65536, 1024, 1792, 1, 2, True,
              note="Dense incoherent A 65536x1024 N(0,1); D + Walsh-Hadamard, s=1, m=1792; seed 2")
C3 = Workload("C3", "dense_coherent", 131072, 4096, 7168, 2, 3, False,
              note="Dense coherent A 131072x4096; s=2, m=7168; seed 3 (no H D)")
C3HD = Workload("C3HD", "dense_coherent", 131072, 4096, 7168, 2, 3, True,
                note="C3 with D + Walsh-Hadamard")
C4 = Workload("C4", "csr", 1048576, 8192, 16384, 3, 4, False, nnz_row=8,
              note="CSR A 1048576x8192, 8 nnz/row, N(0,1); s=3, m=16384; seed 4")
C5 = Workload("C5", "dense_gauss", 2097152, 4096, 7168, 1, 5, True,
              note="Dense A 2097152x4096 N(0,1) (64 GiB); D + Walsh-Hadamard, s=1, m=7168; seed 5")

ALL = {w.name: w for w in (C1, C2, C3, C3HD, C4, C5)}
