"""Test-side helpers: host construction of the int32 layout words that
realb_moe_align builds on the device (include/realb.h), so the GEMM kernels can
be unit-tested on arbitrary group sizes."""

import numpy as np

from paper_2604_19503_b200 import _lib


def layout_words(E, nchunks):
    return int(_lib.load().realb_layout_words(E, nchunks))


def host_layout(counts, prec, nchunks=1):
    """counts: [E] rows per expert; prec: [E] 0/1. Returns (layout int32, rows_used)."""
    counts = np.asarray(counts, np.int64)
    prec = np.asarray(prec, np.int64)
    E = len(counts)
    lay = np.zeros(layout_words(E, nchunks), np.int32)
    padded = (counts + 127) // 128 * 128
    row_start = np.concatenate([[0], np.cumsum(padded)[:-1]])
    lay[8:8 + E] = row_start
    lay[8 + E:8 + 2 * E] = counts
    for p in (0, 1):
        g = np.flatnonzero(prec == p)
        base = 8 + 3 * E + p * (2 * E + 1)
        lay[base:base + len(g)] = g
        mt = padded[g] // 128
        lay[base + E:base + E + len(g) + 1] = np.concatenate([[0], np.cumsum(mt)])
        pbase = 8 + 3 * E + 2 * (2 * E + 1) + p * (E + 1)
        lay[pbase:pbase + len(g) + 1] = np.concatenate([[0], np.cumsum((mt + 1) // 2)])
        lay[1 + p] = len(g)
    lay[0] = int(padded.sum())
    return lay, int(padded.sum())
