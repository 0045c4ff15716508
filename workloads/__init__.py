"""workloads/ -- seeded synthetic inputs shared by the oracle tests and the CUDA path.

Holds NONE of the method's arithmetic (no projection, no eigensolver, no Ritz step): only
the matrix sequences of BASELINE.json's configs (C1..C5) and the spectrum-preserving
variant C3-R, each returned with its planted spectrum / eigenbasis so tests can form the
closed-form expectation themselves. Recipes: DESIGN.md §4 (restating SURVEY.md §8.d.3).
"""
from .generators import (  # noqa: F401
    C1, C2, C2CL, C3, C3R, C4, planted, sym, drift_sequence, rotation_sequence, c4_blocks,
    maxcut_graph,
)
