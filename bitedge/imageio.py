"""`bitedge.imageio` (reference: SPEC.md:273-316, module not shipped) -> B200
implementation: PBM with the P4 payload decoded/encoded on the device, and the
PGM reader (host-side header + payload parse)."""
from paper_1401_5245_b200.pbm import (  # noqa: F401
    detect_pbm, parse_header, read_pbm, read_pgm, write_pbm)
