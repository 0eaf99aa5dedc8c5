"""Float64 CPU oracle for arXiv 1410.7455 (Povey, Zhang & Khudanpur, Kaldi nnet2).

TEST INFRASTRUCTURE ONLY.  Nothing in the product path (``paper_1410_7455_b200``)
may import, call, link or execute anything under ``oracle/``.  The only callers are
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs.

The oracle is a plain, slow, obviously-correct NumPy float64 transcription of the
paper.  Every function cites the PAPER.md passage it follows (``P:n`` = line n of
PAPER.md; section / equation label given alongside).  Library primitives used as
single steps: ``numpy.linalg.eigh`` (symmetric eigendecomposition), ``cholesky``,
``inv``/``solve`` and ``@`` (matmul).  No blocking, fusion or reordering beyond the
paper's own algorithm.

Modules
-------
online_ng   Appendix B: online NG-SGD preconditioner (efficient B.5 form, the naive
            D x D defining form of B.1-B.2, init B.3.2, reorthogonalisation B.3.1).
simple_ng   Appendix A: simple NG-SGD (efficient form and per-row held-out brute force).
nnet        Section 2 + C.6 + 4.6-4.7: p-norm/softmax DNN forward/backward and the
            preconditioned minibatch update with the C.3 max-change guard.
training    Section 3: learning-rate schedule, max-change scale, parameter averaging.

Parity status: every function is pinned by tests in ``tests/test_oracle_*.py``
(``-m "not gpu"``) against worked examples, closed forms, invariants and brute force.
Parity unpinned: initialisation on near-degenerate spectra
(lambda_R ~= lambda_{R+1}); the reorthogonalisation path on non-injected data.
"""
