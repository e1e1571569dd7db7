"""B200-native distributed MoE-layer forward behind the `moeplace` placement API.

The reference (arXiv 2508.12851, package `moeplace`) chooses which experts
live on which server; this package executes the layer those placements imply
on B200 GPUs: hand-written sm_100a kernels (router + histogram, permute +
NVLink dispatch, tcgen05 grouped SwiGLU, combine + NVLink return, peer-copy
migration) behind the C ABI in include/moeplace_b200.h.
"""

from .errors import DimensionMismatch, InfeasibleError, UnplacedExpertError
from .shapes import DEEPSEEK, MIXTRAL, QWEN, SHAPES, TOY, LayerShape, get_shape, slot_caps
from .routing import dispatch_accounting, route_table, route_table_for, slot_map

__all__ = [
    "B200MoELayer", "DEEPSEEK", "MigrationController", "DimensionMismatch", "InfeasibleError", "LayerShape", "MIXTRAL", "QWEN",
    "SHAPES", "TOY", "UnplacedExpertError", "dispatch_accounting", "get_shape", "route_table",
    "route_table_for", "slot_caps", "slot_map",
]


def __getattr__(name):
    # the layer pulls in torch + the CUDA library; import it lazily
    if name == "B200MoELayer":
        from .layer import B200MoELayer
        return B200MoELayer
    if name == "MigrationController":
        from .controller import MigrationController
        return MigrationController
    raise AttributeError(name)
