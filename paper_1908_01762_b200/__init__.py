"""B200-native SISPH hot path (arXiv 1908.01762): sm_100a CUDA kernels behind a
C ABI (include/sisph.h), with a thin ctypes binding.

    from paper_1908_01762_b200 import Simulation
"""
from .sisph import (EXPORTED, FIELDS, LocalGroup, Simulation, SisphError, default_nccl_lib,  # noqa: F401
                    domain, lib, make_dist, nccl_unique_id, params_from_dict, sisph_dist, sisph_domain,
                    sisph_params, sisph_step_report, slab_bounds, slab_owner)

__all__ = ["Simulation", "SisphError", "domain", "params_from_dict", "lib", "FIELDS", "EXPORTED", "LocalGroup",
           "make_dist", "nccl_unique_id", "slab_bounds", "slab_owner", "default_nccl_lib"]
