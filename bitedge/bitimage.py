"""`bitedge.bitimage` (reference: pkg/src/bitedge/bitimage.py) -> B200 implementation."""
from paper_1401_5245_b200.bitimage import (  # noqa: F401
    WORD_BITS, BitImage, BorderPolicy, Direction, PixelColor, first_difference)
