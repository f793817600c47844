"""CPU oracle for the B200 SpMV + Krylov path -- TEST INFRASTRUCTURE ONLY.

A NumPy restatement of the reference's CPU algorithm (the `opalg` package,
/root/reference/pkg/src/opalg; numpy 2.3.5 defines the summation orders) used
as the parity checker. Every function cites the reference file:line it
follows. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import it -- never the product package.

Parity pinning: tests/golden/make_golden.py runs the reference itself (in the
build container, where /root/reference exists) on the same inputs and commits
its outputs as tests/golden/*.npz; tests/test_oracle_golden.py checks this
restatement against those vectors bit-for-bit (SpMV, generators, Jacobi
inverses, iteration counts and residual histories). The layouts of Ell /
Sellp / Hybrid and the power-law generator have no reference implementation
(SPEC.md:294): for those the oracle *is* the specification and parity is
pinned through the format-independent SpMV result against the reference Csr.
"""
