"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds the input recipe only (configs, vertex arrays, right-hand-side
functions, random vectors) and none of the method's arithmetic.  It is the one
module both `oracle/` and the product path may import.
"""
from .configs import CONFIGS, Config, get_config  # noqa: F401
from .generate import (  # noqa: F401
    vertices, rhs_function, exact_solution, dirichlet_function, random_free_rhs,
    parity_vector, small_config, coefficient_function, coefficient_b4, coefficient_samples, strip_vertices,
)
