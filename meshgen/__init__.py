"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the method (no assembly, no Amul, no
solver): it only lays out blockMesh-style hex meshes in OpenFOAM LDU face
addressing, their closed-form geometry, and initial fields.  Both sides
(``oracle/`` and ``paper_2507_18268_b200``) consume its output; neither
imports the other.

Recipe (SURVEY.md §8(d) "Configs as concrete
synthetic inputs"): unit cube [0,1]^3, cell c = i + N*j + N^2*k, internal
faces upper-triangular, six patches xmin,xmax,ymin,ymax,zmin,zmax, DT=1,
dt=0.2, fixedValue 0 walls, T0 = sin(pi x) sin(pi y) sin(pi z).
"""
from .cube import (Mesh, Patch, block_mesh, permute_mesh, sine_field, canonical_field,
                   CANONICAL_AMPLITUDE,
                   cosine_field, multimode_field, random_field, hot_plate,
                   cube_counts, mesh_points_faces, CONFIGS, config_mesh,
                   skewed_block_mesh, with_geometry, PATCH_NAMES,
                   skewed_config_mesh, SKEW_SHEAR, layered_dt_field,
                   PROTOCOL_MESHES, PROTOCOL, protocol_mesh,
                   relabel_mesh, colour_order, colour_mesh)

__all__ = ["Mesh", "Patch", "block_mesh", "permute_mesh", "sine_field", "canonical_field",
           "CANONICAL_AMPLITUDE",
           "cosine_field", "multimode_field", "random_field", "hot_plate",
           "cube_counts", "mesh_points_faces", "CONFIGS", "config_mesh",
           "skewed_block_mesh", "with_geometry", "PATCH_NAMES",
           "skewed_config_mesh", "SKEW_SHEAR", "layered_dt_field",
           "PROTOCOL_MESHES", "PROTOCOL", "protocol_mesh",
           "relabel_mesh", "colour_order", "colour_mesh"]
