"""Test-side helpers: host construction of the int32 layout words that
realb_moe_align builds on the device (include/realb.h), so the GEMM kernels can
be unit-tested on arbitrary group sizes (the builder lives in the package:
moe.host_layout)."""

from paper_2604_19503_b200 import _lib
from paper_2604_19503_b200.moe import host_layout  # noqa: F401


def layout_words(E, nchunks):
    return int(_lib.load().realb_layout_words(E, nchunks))
