"""B200-native PDGraph scoring hot path (arXiv 2506.14851, Hermes).

Drop-in, GPU-backed replacements for the reference's policy runtime:
``sched`` (Gittins evaluator), ``queue`` (device-resident scoring queue).
Importing needs no GPU; every compute call does (no CPU fallback).
"""

from . import errors
from ._lib import PdgDeviceError, PdgError

__all__ = ["errors", "PdgError", "PdgDeviceError"]
__version__ = "0.1.0"
