"""CPU oracle for the hot path -- TEST INFRASTRUCTURE ONLY.

A plain-numpy restatement of the reference algorithm (h2bem, arXiv 2001.05523)
for the functions the GPU path replaces: quadrature rules, touching-pair
classification, regular and Sauter-Schwab Galerkin pair integrals, dense
SLP/DLP blocks, and the H^2 matvec over explicit operator data.  Every
function cites the reference file:line it restates.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this package, and only as the checker / the timed CPU baseline.  The
product package (paper_2001_05523_b200) never imports it.

Pinning: tests/test_oracle.py checks this oracle against the golden vectors
in tests/golden/ produced by running the reference itself
(tests/golden/make_golden.py) -- rules bit-for-bit, pair integrals and dense
blocks to 1e-12, the H^2 matvec to 1e-12 on the reference's own operator.
"""
