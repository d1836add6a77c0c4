"""Seeded synthetic inputs shared by the oracle (tests) and the CUDA path (bench/tests).

This package holds NONE of the method's arithmetic: it only draws permeability
fields, source cells and fault multipliers with the shapes and value
distributions of BASELINE.json's five configs ("Synthetic
inputs").  Both `oracle/` and `paper_2001_01624_b200/` consume its output; it
imports neither.
"""
from .configs import Problem, make_problem, CONFIGS  # noqa: F401
