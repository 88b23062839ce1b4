"""B200-native laplacianFoam hot path (arxiv 2507.18268): C-ABI CUDA library
liblfoam.so (include/lfoam.h) + thin ctypes binding + host-side domain
decomposition.  See DESIGN.md."""
from .lfoam import (Context, Mesh, Ldu, LfoamError, controls, lib, LIB_PATH,  # noqa: F401
                    SIGNATURES, KERNELS)

__all__ = ["Context", "Mesh", "Ldu", "LfoamError", "controls", "lib", "LIB_PATH"]
