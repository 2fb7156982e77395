"""B200-native gDP2d constrained-Delaunay refinement (arXiv 2007.00324).

The refinement loop runs as hand-written sm_100a kernels in lib/libgdp2d.so
behind the C ABI of include/gdp2d.h; this package is the host-side mirror of
the reference's cdtref interface (refine.hpp:651) plus its PSLG/mesh I/O.
"""
from .gdp2d import (CHEW, RUPPERT, CapacityExceeded, CdtError, build_cdt, EngineConfig, Engine, Mesh, MeshError,
                    PinnedPool,
                    QualityCriteria, RuleFlags, RunReport, circumcenters, make_params,
                    predicates, radius_edge_to_theta, refine)

__all__ = ["CHEW", "RUPPERT", "CapacityExceeded", "CdtError", "build_cdt", "EngineConfig", "Engine", "Mesh", "MeshError",
           "PinnedPool",
           "QualityCriteria", "RuleFlags", "RunReport", "circumcenters", "make_params",
           "predicates", "radius_edge_to_theta", "refine"]
