"""Shared helpers for reading tests/golden/golden.npz."""

import ast
import hashlib

import numpy as np


def digest(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return np.frombuffer(h.digest(), np.uint8)


def cases(g, prefix):
    """Distinct case ids under ``prefix`` (e.g. 'mdps' -> ['0', '1', ...])."""
    ids = sorted({k.split("/")[1] for k in g.files if k.startswith(prefix + "/")},
                 key=lambda s: (len(s), s))
    return ids


def mdps_kwargs(g, t):
    kw = ast.literal_eval(str(g[f"mdps/{t}/kw"]))
    if f"mdps/{t}/curve" in g.files:
        kw["curve"] = g[f"mdps/{t}/curve"]
    return kw
