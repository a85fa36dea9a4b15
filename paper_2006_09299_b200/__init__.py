"""B200-native (sm_100a) run-based FG/BG connected-component labeling and analysis.

The compute path is ``librunlab_gpu.so`` (hand-written CUDA, C ABI in
``include/runlab_gpu.h``); this package is the Python mirror of the reference's
``runlab`` interface on top of it.  There is no CPU fallback.
"""
from .runlab import (  # noqa: F401
    NO_LABEL, BatchResult, ComponentRecord, ComponentTree, Connectivity, EquivalenceTable,
    Labeler, LabelingConfig, LabelingResult, LogicError, StepTimes, adjacency_tree,
    binarize_labels, components, default_labeler, euler_number, holes, label_image,
    timed_label_image)

__all__ = [
    "NO_LABEL", "BatchResult", "ComponentRecord", "ComponentTree", "Connectivity",
    "EquivalenceTable", "Labeler", "LabelingConfig", "LabelingResult", "LogicError", "StepTimes",
    "adjacency_tree", "binarize_labels", "components", "default_labeler", "euler_number", "holes",
    "label_image", "timed_label_image",
]
