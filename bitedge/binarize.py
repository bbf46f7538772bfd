"""`bitedge.binarize` (reference: SPEC.md:226-271, module not shipped) -> B200
implementation of the fixed threshold (Otsu is out of scope)."""
from paper_1401_5245_b200.binarize import threshold, threshold_edges  # noqa: F401
