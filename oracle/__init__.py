"""CPU oracle for randUTV (arXiv:2002.06960, Sec. 3.1) -- TEST INFRASTRUCTURE ONLY.

This package is a plain, slow, obviously-correct FP64 implementation of what the
GPU hot path computes.  It exists to *check* the CUDA library, never to stand in
for it.  Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import, call or execute anything
under ``oracle/``.  The product path (``paper_2002_06960_b200``) never imports
it, and the oracle never imports the product path: the two share no code,
helpers, constants or tables.  Inputs both sides consume come from
``paper_2002_06960_b200/inputs.py``, which holds no randUTV arithmetic.

Citation convention: ``P:L`` = line L of PAPER.md (the paper's LaTeX source),
followed by the section / equation / figure it falls in.  Where the paper is
silent or garbled, the reading taken is the one listed in DESIGN.md §"Readings"
(labels A1..A22 follow SURVEY.md §8(c)).

Modules
-------
philox      O1  counter-based Gaussian G^(i)            (reading A7)
householder O3  dlarfg-convention Householder QR         (A9)
            O4  compact-WY T factor (forward, columnwise)
jacobi      O8  one-sided (Hestenes) Jacobi SVD           (A10)
randutv     O2, O5-O7, O9-O11 the blocked loop and the truncated variant
            
bruteforce  explicit-matrix mini-oracle for tiny n (forms every H_j, every
            orthogonal factor, and multiplies literally)
hqrrp       H1-H6 the paper's first method, HQRRP (randomized blocked
            column-pivoted QR) and its partial variant
"""
