"""CPU fp64 ORACLE for the paper's matrix-free system model (arXiv 1812.03358).

TEST INFRASTRUCTURE ONLY.  Nothing in the product path (paper_1812_03358_b200/,
include/, the CUDA library) may import, call, link or execute anything under
`oracle/`; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may.  The oracle shares no code with the CUDA path; the
only common module is `workloads/` (seeded input recipes, no method arithmetic).

It is a plain, slow, literal transcription of the paper in fp64:

* optics.py    -- ray transforms T_D, R_f, composition, inverse (§2.1)
* transport.py -- 1D transport entries of B^{pq}_k from the L2 inner products
                  (eqn,xport / xport,ip / xport,int), V^p
* camera.py    -- single-lens and plenoptic cameras (§2.6), slice
                  collapse and factored plenoptic chain (§3); the
                  explicit dense A for tiny inputs ("would produce the same
                  results") and a matrix-free sparse fp64 path for larger ones
* rotation.py  -- Theta = D S_z S_x S_y and the shear operators E (§3.1)
* system.py    -- A_c = camera o collapse o rotation (§3.2)
* pwls.py      -- PWLS cost, gains, gradient, regulariser, majoriser, FISTA
                  (§5, Appendix A)

Readings of silent/garbled passages are SURVEY.md §8(c) Z1-Z24 and are listed in
DESIGN.md.  Pins (what each function is checked against, other than itself) are
in tests/test_oracle_*.py.  Parity unpinned vs the paper: the absolute scale of y
(reading Z7) and the FISTA trajectory (tab,alg missing; reading Z18).
"""
