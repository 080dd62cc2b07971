"""B200-native time-marching hot path of arXiv 1609.07114 (FDTD with embedded reduced-order models).

The product is libfdtdrom.so (C ABI in include/fdtdrom.h, CUDA kernels for sm_100a);
``fdtdrom`` is its thin ctypes binding.  Build with ``python -m paper_1609_07114_b200.build``.
"""
from .fdtdrom import (FDTDError, Simulation, build_rom, from_scene, halo_plan, lib, nccl_unique_id,  # noqa: F401
                      pass_regions, step_group)

__all__ = ["Simulation", "FDTDError", "build_rom", "from_scene", "halo_plan", "lib", "nccl_unique_id", "pass_regions",
           "step_group"]
