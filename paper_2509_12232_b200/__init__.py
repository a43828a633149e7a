"""paper_2509_12232_b200 -- the vecdock docking hot path, B200-native.

Scope: AutoDock4-type scoring of GA populations of
ligand poses (pose -> grid-map gathers + pairwise intra energy) and the GA
loop that closes it, as hand-written sm_100a CUDA kernels behind the C-ABI
of include/vecdock_b200.h, with a host-side mirror of the reference's
Python interface (same names, arguments, rounding and errors).
"""

from .chem import (DESOLV_LABEL, ELEC_LABEL, AtomParams, ParameterTable, TermWeights,
                   default_parameter_table, parse_parameter_table)
from .context import BackendUnavailable, ScoreBreakdown, ScoringContext, prepare_context
from .gridmaps import (GridFormatError, GridMapSet, GridSpec, build_grid_maps, read_grid_set,
                       trilinear_lookup, write_grid_set)
from .topology import (LigandTopology, NonbondPairList, Protein, RotatableBond,
                       build_fragment_masks, build_nonbond_pairlist)

__all__ = [
    "AtomParams", "BackendUnavailable", "DESOLV_LABEL", "ELEC_LABEL", "GridFormatError",
    "GridMapSet", "GridSpec", "LigandTopology", "NonbondPairList", "ParameterTable", "Protein",
    "RotatableBond", "ScoreBreakdown", "ScoringContext", "TermWeights", "build_fragment_masks",
    "build_grid_maps", "build_nonbond_pairlist", "default_parameter_table",
    "parse_parameter_table", "prepare_context", "read_grid_set", "trilinear_lookup",
    "write_grid_set",
]


def __getattr__(name):
    # device-facing modules load lazily so host-only use never dlopens CUDA
    import importlib

    lazy = {
        "CudaBackend": ("backend", "CudaBackend"), "get_backend": ("backend", "get_backend"),
        "list_backends": ("backend", "list_backends"), "score_pose": ("backend", "score_pose"),
        "score_population": ("backend", "score_population"),
        "inter_energy": ("backend", "inter_energy"), "intra_energy": ("backend", "intra_energy"),
        "register_reference_backend": ("backend", "register_reference_backend"),
        "GaConfig": ("ga", "GaConfig"), "dock": ("ga", "dock"),
        "DockingResult": ("ga", "DockingResult"),
        "ScreenConfig": ("screening", "ScreenConfig"), "screen_batch": ("screening", "screen_batch"),
        "apply_pose": ("pose", "apply_pose"), "pose_population": ("pose", "pose_population"),
    }
    if name in lazy:
        mod, attr = lazy[name]
        return getattr(importlib.import_module(f".{mod}", __name__), attr)
    raise AttributeError(name)
