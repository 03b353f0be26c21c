"""Shared test helpers (comparison metrics only; no method arithmetic)."""
import numpy as np


def normalized_err(G, Gref):
    """max |G_ij - Gref_ij| / sqrt(Gref_ii Gref_jj) over all entries and drops (reading R9)."""
    G = np.asarray(G)
    Gref = np.asarray(Gref)
    d = np.real(np.diagonal(Gref, axis1=-2, axis2=-1))
    scale = np.sqrt(np.abs(d[..., :, None] * d[..., None, :]))
    return float(np.max(np.abs(G - Gref) / scale))
