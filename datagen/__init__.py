"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

Holds none of the method's arithmetic (DESIGN.md §3 "input recipe")."""
from .configs import CONFIGS, EXPERIMENTS, PAPER_RHO, PARITY, Config, Dataset, get, make_dataset, make_sources  # noqa: F401
from .sources import gg_beta  # noqa: F401
