"""ORACLE — test infrastructure only.

A plain, slow, CPU (numpy/scipy, complex float64) implementation of what the
hybrid DH^2 recompression of arXiv 1809.04384 computes, written directly from
PAPER.md.  Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import it.  The product path
(``paper_1809_04384_b200``) never imports, links or executes anything here, and
this package imports nothing from the product path: the two share only the
seeded input generators in ``synth/``.

Modules
  structure  -- cluster tree, boxes, directions, block tree, row/col pair closure (PAPER §2)
  interp     -- Chebyshev grids, Lagrange polynomials, quadrature, V, E, S (PAPER §2, Eq. 4, Eq. 10)
  recompress -- "O-fast": §3.2 basis weights, total weights, truncation, projection
  dense      -- "O-dense": §3.1 compression applied to the densely expanded far field
  ops        -- matvec, storage accounting, error identities

Pins: every function is checked by ``tests/test_oracle_*.py`` (``-m "not gpu"``)
against closed forms, invariants, brute force on tiny inputs and the paper's own
identities; see DESIGN.md §"Oracle pins" for the list.  Nothing is "parity
unpinned" except the absolute magnitude of the interpolation error, for which the
paper gives no constant (we pin its monotone decay in m instead).
"""
