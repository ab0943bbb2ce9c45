"""B200-native exact readability metrics (drop-in for glare.metrics' oracle).

The five metric functions keep the reference's signatures and outputs
(/root/reference/pkg/src/glare/metrics/__init__.py:11-25) and run on
hand-written sm_100a kernels through the C ABI in include/glare_b200.h.
"""

from .enhanced import (
    crossing_angle_stats,
    edge_crossing_angle_enhanced,
    edge_crossing_enhanced,
    node_occlusion_grid,
)
from .layout import fr_layout, generate_layout, random_layout
from .metrics import (
    CrossingRecords,
    DeviceGraph,
    _crossing_scan,
    crossing_count_and_angle,
    edge_crossing,
    edge_crossing_angle,
    edge_length_variation,
    minimum_angle,
    node_occlusion,
)
from .model import (
    IDEAL_ANGLE_DEFAULT,
    METRIC_FIELDS,
    GlareError,
    InputError,
    InvariantError,
    LayoutGraph,
    MetricParams,
    ParameterError,
    SchemaError,
    normalize_edges,
)

__all__ = [
    "crossing_angle_stats",
    "edge_crossing_angle_enhanced",
    "edge_crossing_enhanced",
    "node_occlusion_grid",
    "fr_layout",
    "generate_layout",
    "random_layout",
    "CrossingRecords",
    "DeviceGraph",
    "GlareError",
    "IDEAL_ANGLE_DEFAULT",
    "InputError",
    "InvariantError",
    "LayoutGraph",
    "METRIC_FIELDS",
    "MetricParams",
    "ParameterError",
    "SchemaError",
    "_crossing_scan",
    "crossing_count_and_angle",
    "edge_crossing",
    "edge_crossing_angle",
    "edge_length_variation",
    "minimum_angle",
    "node_occlusion",
    "normalize_edges",
]
