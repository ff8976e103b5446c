"""B200-native hot path for Anderson-accelerated FWI/LSRTM (arXiv:2008.11778).

The drop-in API mirrors the reference package ``seisopt``: ``gradients``
(fwi_synthetic, fwi_gradient, BornKernel, lsrtm_objective, FwiObjective,
LsrtmObjective), ``anderson`` (AAWindow, aa_weights, aa_step, minimize_aa) and
the data-model types in ``model``.  All arithmetic runs in hand-written sm_100a
CUDA inside ``libseisgpu.so`` behind a C ABI (``include/seisgpu.h``); the CUDA
library is loaded lazily on first use and its absence is an error, never a
fallback.
"""

from .model import (AcquisitionGeometry, EvalCounters, Grid2D, ObjectiveEval,  # noqa: F401
                    ReflectivityModel, ShotGather, SimConfig, SourceWavelet,
                    StabilityError, VelocityModel, make_ricker)

__all__ = ["AcquisitionGeometry", "EvalCounters", "Grid2D", "ObjectiveEval",
           "ReflectivityModel", "ShotGather", "SimConfig", "SourceWavelet",
           "StabilityError", "VelocityModel", "make_ricker"]
