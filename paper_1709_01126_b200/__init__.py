"""B200-native (sm_100a) fp64 PCG solve of the POT3D potential-field problem
(arXiv 1709.01126): C-ABI library libpot3d.so + thin Python binding."""
from .pot3d import (CLOSED_WALL, PC1, PC2, SOURCE_SURFACE, Pot3d, Pot3dError,  # noqa: F401
                    gather_slabs, library, nccl_unique_id, slab_bounds)

__all__ = ["Pot3d", "Pot3dError", "library", "nccl_unique_id", "slab_bounds", "gather_slabs",
           "SOURCE_SURFACE", "CLOSED_WALL", "PC1", "PC2"]
