"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

Holds none of the sketch's arithmetic (see synth/gen.py).  ``synth.device``
wraps the CUDA generator (libsynth.so) that writes the same values straight
into device memory for the large workloads.
"""
from . import configs, gen  # noqa: F401
