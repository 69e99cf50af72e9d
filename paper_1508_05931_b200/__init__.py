"""B200-native gScan 2D convex hull (arXiv 1508.05931), drop-in for the
reference's hull2d::full_pipeline path. See DESIGN.md and include/gscan.h."""
from .hull2d import (  # noqa: F401
    CoincidentWithAnchor,
    CollectiveError,
    DeviceError,
    EmptyInput,
    Engine,
    Error,
    Hull,
    IndexOutOfRange,
    IoError,
    LengthMismatch,
    ParseError,
    PipelineConfig,
    PipelineResult,
    StageStats,
    TooFewPoints,
    TooLarge,
    ZeroChunks,
    default_engine,
    full_pipeline,
    generate,
    generate_grid,
    hull,
    load_points,
    save_soa,
)
from ._native import LIB_PATH, NativeUnavailable  # noqa: F401
