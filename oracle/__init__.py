"""CPU oracle for the decoupled multicontinuum time step — TEST INFRASTRUCTURE ONLY.

This package is the plain, slow, obviously-correct reference that the CUDA
path (``paper_2209_01158_b200``) is checked against.  It is NOT part of the
product: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import or execute anything
here.  It shares no code with the CUDA path; both read the physical inputs
produced by ``inputs/`` and assemble their own operators.

Modules
-------
assemble  Eq. app-md / app-tc / app-mc assembly of M, A = D + Q, F
          from the generator's physical inputs, with readings C1-C12.
schemes   coupled backward Euler, Eq. ct-mc, and the decoupled
          D-scheme, Eq. si-mc with A0 = blockdiag(A), solved
          with SciPy sparse LU (SuperLU) factorisations, or plain Jacobi-PCG.
cg        a plain Jacobi-preconditioned CG in NumPy, for the CG
          unit pins.
flux_pcg.c / fluxcg
          plain C + OpenMP Jacobi-PCG on the unassembled flux-form operator and the
          coupled / D-scheme steppers built on it (relres 1e-13), for the sizes a
          sparse factorisation cannot take (configs 2 and 4); the
          C library is compiled on first use (gcc) or by __graft_entry__.build().

nlmc      the NLMC multiscale space of PAPER.md §4.1: bases of Eq. eq:basis per oversampled
          region (KKT systems, SuperLU), R, the coarse system in flux form (readings
          C30-C33), pinned by tests/test_nlmc_oracle.py.

Every function is pinned by ``tests/test_oracle_*.py`` against closed forms,
brute force and the paper's / SPEC's worked examples.
"""
