"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct complex128 NumPy/SciPy implementation of the
hot path of Bootland & Rees, "Multipreconditioning with directional sweeping
methods for high-frequency Helmholtz problems" (arXiv 2408.11929), in the
discretisation the north star fixes (P1 FEM on a "/"-triangulated grid).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2408_11929_b200``) never imports it and shares no code
with it; the only common module is ``helm_inputs`` (seeded input generators,
no method arithmetic).

Citations: ``P:Lnn`` = PAPER.md line nn (LaTeX source), with the equation /
section named; ``D1..D12`` and ``A1..A27`` = the definitions and readings of
SURVEY.md §8(c), restated in DESIGN.md §3.

Modules
  p1      -- D1-D5 grid, coefficients, assembly of A, load vector, manufactured data
  strips  -- D6-D8 strip geometry, local matrices, transmission corrections
  sweep   -- D9 forward/backward double sweeps and single sweeps, gathers;
             D12 exact-Schur test mode
  krylov  -- D10 selective MPGMRES (BCGS2 and paper-count modes), textbook
             right-preconditioned GMRES, complete MPGMRES (small scale)

Parity status: every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_pins.py`` (Pin-1 .. Pin-14 of SURVEY.md §8(c)).  The
iteration counts on C1-C5 are "parity unpinned" beyond oracle-vs-GPU (there is
no published P1 number to pin them to).
"""
