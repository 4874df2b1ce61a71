"""B200-native decoupled multicontinuum time stepping (arXiv 2209.01158).

The product is ``libmc.so`` (C ABI: ``include/mc.h``; CUDA sources: ``csrc/``),
built in-tree for sm_100a by ``paper_2209_01158_b200.build``.  ``mc`` is its thin
ctypes binding.  Importing this package does not load the library; ``mc.load()``
(or constructing ``mc.Problem``) does, and raises if it has not been built.
"""
from . import mc  # noqa: F401
from .mc import Problem, load, MCError, permeability_order  # noqa: F401

__all__ = ["mc", "Problem", "load", "MCError"]
