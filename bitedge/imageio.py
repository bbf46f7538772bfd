"""`bitedge.imageio` PBM part (reference: SPEC.md:273-316, module not shipped) -> B200
implementation with the P4 payload decoded/encoded on the device (PGM is out of scope)."""
from paper_1401_5245_b200.pbm import detect_pbm, parse_header, read_pbm, write_pbm  # noqa: F401
