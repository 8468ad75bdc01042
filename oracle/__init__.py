"""CPU oracle for the IsoRank pair-similarity hot path — TEST INFRASTRUCTURE ONLY.

Nothing in ``paper_1707_02423_b200`` imports this package.  Only ``tests/``,
``__graft_entry__.smoke()`` (as the checker) and ``bench.py``'s CPU-baseline
leg / ``--impl reference`` arm may import, link or execute anything here.

Two restatements of the reference algorithm (``/root/reference`` is the
public ``sasscfg`` package, pure Python + numpy):

* ``isorank_np``  — numpy, small cases, readable line-by-line against
  ``pkg/src/sasscfg/similarity.py:85-173`` and ``matrix.py:74-114``.
* ``isorank_ref.c`` (built to ``oracle/build/liboracle.so``, bound by
  ``oracle.ffi``) — plain C, OpenMP over pairs, used for bulk parity sweeps
  and as the CPU baseline ("port") in ``bench.py``.

Both replace only the reference's materialised Kronecker mat-vec
``kron(A',B')^T @ x`` (``similarity.py:133,140``) by the identical two-product
form ``A'^T X B'`` (``X`` = ``x`` reshaped row-major N x N).  Every other step —
bilinear size normalisation, row normalisation with uniform zero rows, the
damped update, L1 renormalisation, L1 change, stopping rule, greedy matching
tie rule and the distance formula — follows the reference operation by
operation.  Parity of the restatement is PINNED against the reference itself:
``tests/golden/`` holds vectors produced by importing ``sasscfg`` from
``/root/reference`` (script ``tests/golden/make_golden.py``), and
``tests/test_oracle.py`` checks both restatements against them.
"""
