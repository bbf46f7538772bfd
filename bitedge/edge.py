"""`bitedge.edge` (reference: SPEC.md:132-224, module not shipped) -> B200 implementation."""
from paper_1401_5245_b200.edge import (  # noqa: F401
    FOUR_NEIGHBORS, NEIGHBOR_OFFSETS, Neighborhood, at_most_one_black_8neighbor, build_mask,
    detect_edges_mask, detect_edges_scan, edge_set, fundamental_edge, fundamental_edges,
    is_edge_point, neighborhood)
