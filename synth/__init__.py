"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This package holds ONLY input generators (surface meshes, seeded vectors and the
named workload configurations).  It contains none of the recompression method's
arithmetic, so both the oracle (``oracle/``) and the product path
(``paper_1809_04384_b200``) may consume it without sharing code with each other.
"""
from .meshes import sphere_mesh, cube_mesh, mesh_for
from .vectors import seeded_vector
from .configs import CONFIGS, get_config

__all__ = ["sphere_mesh", "cube_mesh", "mesh_for", "seeded_vector", "CONFIGS", "get_config"]
