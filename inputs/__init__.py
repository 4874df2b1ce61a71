"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds ONLY the physical description of each workload (grid size,
permeability / storage coefficients, fracture cells and their adjacency,
transfer coefficients, Dirichlet data, the NLMC-style synthetic coarse
transmissibilities).  It contains none of the method's arithmetic: no
transmissibility, mass, coupling or boundary assembly, no time stepping and no
linear algebra.  Both ``oracle/`` (CPU reference) and
``paper_2209_01158_b200`` (the CUDA product path) import it and assemble their
own operators from it independently.
"""
from .generator import (  # noqa: F401
    CONV_VERSION,
    CONFIGS,
    make,
    make_fine,
    crop_fine,
    make_paper_analogue,
    make_nlmc,
    fracture_network,
)
