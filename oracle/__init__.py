"""CPU fp64 oracle for the structure-preserving reduced FDTD hot path.

TEST INFRASTRUCTURE ONLY.  Nothing under ``oracle/`` is part of the product:
only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import it.  The CUDA path
(``paper_1406_7042_b200``) never imports it, and it never imports the CUDA
path or the host preprocessing library (``paper_1406_7042_b200.prep``); the
two share no code.  Inputs common to both come only from ``synth/`` (seeded
scenario generators that hold none of the method's arithmetic) and from the
fp64 problem description the preprocessing emits (the F13 shared-input rule,
DESIGN.md §3).

Everything here is written to be checked against the paper by eye:
plain NumPy/SciPy fp64, sparse matrices built entry by entry from the
definitions, no blocking or fusion.  Citations are ``P:n`` =
``/root/reference/PAPER.md`` line ``n`` (the reference tree is not needed at
run time).

Modules
-------
yee          Eq. (3) assembly on uniform 1-D / 2-D (Ez/Hx/Hy) / 3-D Yee grids.
matrix_form  Eqs. (4)-(6): R, F, B, the literal recursion, energy x^T R x,
             update-matrix eigenvalues.
stability    Eq. (1) CFL, Eqs. (25)-(26) singular-value criterion, §III-A
             enforcement, the hybrid split enforcement (reading R7).
reduction    Eqs. (9)-(16) projection, Eq. (19) expansion points, transfer
             function for moment-matching checks.
hybrid       Coarse grid + refined box as one system of form (3)
             (reading R4; not in the paper).
problem_step The reduced-hybrid recursion (4)/(12) driven by a problem
             description: what the GPU must match.
physics      Analytic cavity resonances and spectral peak picking.

Parity status of every function is listed in DESIGN.md §4 ("pinned by").
"""
