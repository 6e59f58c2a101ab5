"""ORACLE — test infrastructure only.

A plain, slow, CPU fp64 transcription of what the hot path computes (PAPER.md
arXiv 2510.22077, Li & Mehmani), written from the paper and SURVEY.md §8(c)'s
readings, for checking the CUDA path.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import or run anything in this package.  The
product library (``paper_2510_22077_b200``) never imports it and shares no
code with it; the only common dependency is the seeded input generator in
``synth/`` (images and random vectors, none of the method's arithmetic).

Modules
-------
grid          D1 clean-up, canonical DOF numbering, face classification
mac           residual r(x), Jacobian J(x), modified Jacobian J~_w (Eq. Ax=b, Eq. mod_res)
decomposition D2-D10 watershed primaries, interfaces, duals, mask band
gplmm         W, Q, fold C(.), P, R, P^, R^, A°, M_G, M_dp, M (Eqs. permute..restrict_FVM, iMG, Mdp)
krylov        right-preconditioned flexible GMRES with MGS
newton        Newton driver and the steady / transient pipelines

Parity status: every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` except the decomposition (D2-D10), whose result
is an algorithm the paper does not specify (P:156 defers to an external
reference): it is pinned only by invariants and hand-built fixtures —
"parity unpinned" against the paper for the exact labelling.  Krylov
iteration counts are likewise unpinned by the paper (its figures are absent).
"""
