"""TEST INFRASTRUCTURE ONLY — CPU oracle for the bidomain PCG hot path.

A restatement of the reference algorithm (/root/reference/pkg/src/bidomain:
system.py, precond.py, krylov.py, ionic.py, simulate.py) in numpy/scipy, with
the IC(0) factorisation sweep also restated in C (ic0_oracle.c) for the large
configurations.  Every function cites the reference file:line it follows.

Pinned against the reference itself: tests/golden/make_golden.py imports the
real reference (with a cvxopt/matplotlib shim) in the build container and
commits its outputs as fixtures; tests/test_oracle_golden.py checks this
oracle against them (bit-exact where the reference arithmetic is reproduced,
tolerance-checked at the CHOLMOD/SuperLU boundary).

Only tests/, __graft_entry__.smoke() and bench.py (its cpu_baseline leg and
`--impl reference`) may import this package, and only as the checker / the
CPU reference arm — never as the product path.
"""
