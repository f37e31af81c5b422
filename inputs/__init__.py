"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

Holds none of the method's arithmetic."""
from . import configs, synth  # noqa: F401
