"""CPU ORACLE — test infrastructure only.

Plain, slow, obviously-correct NumPy (fp64) implementation of what the hot path computes,
written from PAPER.md (arXiv 2506.14424) and the readings G1-G25 of SURVEY.md §8(c)
(listed again in DESIGN.md).  Full-tensor quadrature: every basis function and gradient
is tabulated at every volume / face quadrature point and the integrals are evaluated by
dense sums - no sum factorisation, no blocking, no fusion.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import this package.  The CUDA library
(paper_2506_14424_b200) never imports, links or executes anything here, and this package
never imports the CUDA library: the two share no code.

Parity status (DESIGN.md §Oracle pins): every public function is pinned by at least one
`-m "not gpu"` test in tests/test_oracle_*.py against properties the paper and the
mathematics fix.  Conventions G1-G3, G6 (basis, quadrature, penalty length scale, face
viscosity) are convention-pinned, not paper-pinned: the paper prints no operator value.
"""
