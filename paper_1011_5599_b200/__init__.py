"""B200-native HyperANF engine (arXiv:1011.5599), drop-in for the reference's
C++ engine surface (/root/reference/proj/include/hyperanf/engine.hpp).

The hot path -- seeding, the register-wise max over successors, the
estimator and the N(t) reduction -- runs as hand-written sm_100a kernels in
libhanf.so, reached through its C-ABI (include/hanf.h).  This package is the
Python mirror of that surface; there is no CPU fallback.
"""
from ._lib import (CapacityError, CudaError, GuardError, IoError, ParseError,  # noqa: F401
                   LIB_PATH, lib)
from .engine import (EngineConfig, IterationReport, NfEngine, NfEstimate,  # noqa: F401
                     SketchParams, Termination, estimate_nf, multirun, ExactNf,
                     exact_nf)
from .graph import (Graph, gen_barabasi_albert, gen_clique_path, gen_copying,  # noqa: F401
                    gen_erdos_renyi, gen_rmat, gen_uniform_random, load_csr, save_csr,
                    transpose)
from .stats import (aggregate_runs, cdf_from_nf, diameter_interval,  # noqa: F401
                    distance_distribution, distribution_from_cdf, effective_diameter,
                    precision_from_error, precision_from_eta, precision_from_m)

__all__ = [
    "EngineConfig", "IterationReport", "NfEngine", "NfEstimate", "SketchParams",
    "Termination", "estimate_nf", "multirun", "ExactNf", "exact_nf", "Graph", "transpose", "gen_uniform_random",
    "gen_clique_path", "gen_erdos_renyi", "gen_rmat", "gen_copying",
    "gen_barabasi_albert", "save_csr", "load_csr", "cdf_from_nf",
    "distribution_from_cdf", "distance_distribution", "effective_diameter",
    "diameter_interval", "precision_from_m", "precision_from_eta",
    "precision_from_error", "aggregate_runs", "GuardError", "ParseError", "IoError",
    "CudaError", "CapacityError",
]
