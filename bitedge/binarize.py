"""`bitedge.binarize` (reference: SPEC.md:226-271, module not shipped) -> B200
implementation: fixed threshold, fused threshold + edges, Otsu."""
from paper_1401_5245_b200.binarize import otsu_threshold, threshold, threshold_edges  # noqa: F401
