"""Seeded synthetic scenario generators - the ONLY code shared by the CUDA path
(via the host preprocessing library) and the oracle.

It holds none of the method's arithmetic: it draws random numbers, lays out
geometry (cell sizes, permittivity maps, refined boxes, PEC strips), samples
the source waveforms in fp64 and fixes the time step of each configuration.
Everything the paper's method computes (assembly, projection, enforcement,
stepping) lives on either side, written twice, independently.

Recipes follow SURVEY.md §8(d) "Synthetic inputs" (RNG = NumPy PCG64, seed =
14067042 + config id, draws in the listed order); deviations are listed in
DESIGN.md §7.
"""
from .scenarios import (C0, MU0, EPS0, scenario, config_ids, gaussian_tau,
                        gaussian_derivative_tau)  # noqa: F401
