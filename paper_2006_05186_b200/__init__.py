"""B200-native multi-frequency H^2 + ACA single-layer apply (arXiv 2006.05186).

The product is the C-ABI library libbem.so (include/bem.h) built from csrc/;
this package is its thin binding.  See DESIGN.md.
"""
from .bem import (BEM_MODE_COMBINED, BEM_MODE_DENSE, BEM_MODE_H2ACA, BEM_MODE_H2ONLY, BEM_SKEL_FACTORS, BEM_SKEL_Z,
                  BemError, Operator, Tree, cqm_forward, cqm_frequencies, cqm_inverse, cqm_mot_solve, cqm_solve,
                  debug_fastmath, debug_pinned, dirichlet_solve, fp64_peak, lib, solve_multifreq)

__all__ = ["BEM_MODE_COMBINED", "BEM_MODE_DENSE", "BEM_MODE_H2ACA", "BEM_MODE_H2ONLY", "BEM_SKEL_FACTORS", "BEM_SKEL_Z",
           "BemError", "Operator", "Tree", "cqm_forward", "cqm_frequencies", "cqm_inverse", "cqm_mot_solve", "cqm_solve",
           "debug_fastmath", "debug_pinned", "dirichlet_solve", "fp64_peak", "lib", "solve_multifreq"]
