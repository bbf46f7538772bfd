"""`bitedge.cuda` -- device tensor API (new)."""
from paper_1401_5245_b200.cuda import *  # noqa: F401,F403
from paper_1401_5245_b200.cuda import (  # noqa: F401
    count_black, edges_general, edges_halo, edges_packed, pack_edges_u8, pack_u8, scan_edges,
    unpack_u8)
