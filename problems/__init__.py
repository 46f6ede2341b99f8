"""Seeded synthetic input generators (configs C1-C5 of BASELINE.json).

This package is shared by the oracle (`oracle/`), the tests and `bench.py`.
It holds NO arithmetic of the hierarchical method itself: it only builds the
sparse SPD operators, coordinates, extruded column ids and right-hand sides
that both the oracle and the CUDA path consume.  See DESIGN.md "Input recipe".
"""
from .generators import (Problem, gen_poisson2d, gen_laplace3d, gen_slab,
                         gen_stokes_q1, gen_config, gen_family, grf, rhs, CONFIGS)

__all__ = ["Problem", "gen_poisson2d", "gen_laplace3d", "gen_slab",
           "gen_stokes_q1", "gen_config", "gen_family", "grf", "rhs", "CONFIGS"]
