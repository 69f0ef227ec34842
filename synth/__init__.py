"""Seeded synthetic inputs shared by the oracle (tests) and the CUDA path (bench/tests).

This package holds only input *generation* (random draws, sampling from a known
Kronecker-sum Gaussian, QR for orthonormal factors).  It contains none of the
method's arithmetic (no Gram spectra, no eigenvalue solve, no recomposition or
sparsification).  See ``synth.gen`` for the recipes.
"""
from .gen import *  # noqa: F401,F403
