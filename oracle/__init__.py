"""CPU oracle for the D3Q19 binary-fluid lattice-Boltzmann step.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import anything
under ``oracle/``.  The product path (``paper_1609_01479_b200``) never imports
it, and this package imports nothing from the product path: the two share no
code, tables or constants.

Modules
-------
lb_ref    plain NumPy fp64 transcription of the step, ``np.roll`` for every shift
lb_brute  per-site scalar loops (pure Python floats) for tiny lattices and for
          single sampled sites of large lattices
lb_mrt    the NEXT-3 collision variant: chemical stress in f's equilibrium,
          three-rate MRT (readings R23-R27)
lb_ch     the NEXT-2 variant: phi as a field, finite-difference Cahn-Hilliard
          with first-order upwind advection (readings R29-R33)
lb_lc     the NEXT-4 workload: Landau-de Gennes Q tensor, Beris-Edwards LC
          update and chemical stress driving the LB fluid (readings R34-R45)

Citations: ``P:NNN`` = PAPER.md line NNN (Gray & Stratford, arXiv 1609.01479);
``S:NNN`` = SPEC.md line NNN; ``Rk`` = reading k of the DESIGN.md ledger (the
paper contains no binary-fluid equations, so every equation is a reading).
"""
