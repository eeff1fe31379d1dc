"""CPU ORACLE for the s-hashing sketch hot path of Ski-LLS (arXiv 2105.11815).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import, call or
execute anything in this package.  The product path
(``paper_2105_11815_b200``) never imports it, and this package never imports the
product path: the two share no code, tables or constants.  The only shared module
is ``synth`` (seeded input generators, which hold none of the method's
arithmetic).

Citation format: ``P:L123`` is line 123 of the paper's text
(/root/reference/PAPER.md), ``S:L123`` a line of SPEC.md; ``DESIGN.md R<k>`` is a
reading of the paper recorded in DESIGN.md §3.

What each module computes (all fp64, plain NumPy, slow on purpose):

* ``rng``       - splitmix64 counter-based stream (R1, the paper is
                  silent on the RNG).  Pinned: public splitmix64
                  known-answer values (tests/golden/splitmix64_kat.txt).
* ``hashing``   - the s-hashing matrix S of Def. ``def::sampling_and_hashing``
                  (P:L269-272): s distinct rows per column, entries +-1/sqrt(s);
                  explicit triples, dense S and bucket lists.  Pinned: structure
                  invariants, chi^2 uniformity, sign balance, unbiasedness
                  E||Sx||^2 = ||x||^2 (P:L272 footnote), Example 1's birthday
                  bound, pure-Python vs vectorised agreement.
* ``hadamard``  - D and the Walsh-Hadamard H of Def. ``def::HRHT``:
                  H by Sylvester recursion, H by the P:L796 formula, and the
                  radix-2 fast transform.  Pinned: Sylvester == formula
                  entrywise, H^2 = I, n=2 worked value, H e_0, H 1,
                  orthogonality, Tropp's coherence bound.
* ``sketch``    - Algorithm 1 Step 1: SA and Sb for dense A, CSR A and
                  the HRHT S_h H D A.  Pinned: dense materialised S @ A vs
                  bucket-order sums, A = I gives S, scipy.sparse cross-check,
                  linearity, subspace-embedding band (R11),
                  negative control for coherent A without H D,
                  sketch-QR-preconditioned LSQR vs normal equations.
* ``variant``   - the s-hashing variant T of Def. 7.  Pinned:
                  Lemma 8, collision probability, s = 1 reduction.
* ``lls``       - Algorithm 1 Steps 2-5: QR, x_s, LSQR with the
                  (7.1) stop.  Pinned: scipy's LSQR, lstsq.
* ``hartley``   - HR-DHT S_h F D (eq. (6.1)).  Pinned: explicit
                  (6.1) matrix, involution, Parseval, n = 2 WHT identity.
* ``sampling``  - SR-DHT S_s F D (eq. (7.2)) and the Fig. 1 experiment
                  (P:L1284-1297).  Pinned: chi^2, collision rate, explicit S_s.
* ``probes``    - Freivalds identities w^T(SA)v = (S^T w)^T(Av) for sizes the
                  oracle cannot materialise.  Pinned: equals the dense product on
                  small sizes.

Parity status: every function above is pinned by at least one test in
``tests/test_oracle_*.py`` against something other than itself; none is
"parity unpinned".  The absolute value of one SA entry at BASELINE size has no
external reference; it is pinned only through the properties above.
"""
