"""Loader for the golden fixtures generated from the real reference
(tests/golden/make_golden.py)."""
import json
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
_META = None
_ARR = None


def meta():
    global _META
    if _META is None:
        with open(os.path.join(HERE, "golden.json")) as f:
            _META = json.load(f)
    return _META


def arrays():
    global _ARR
    if _ARR is None:
        _ARR = dict(np.load(os.path.join(HERE, "golden.npz")))
    return _ARR


def layer_case(name):
    m = meta()["layers"][name]
    a = arrays()
    return m, a[f"{name}__x"], a[f"{name}__w"], a[f"{name}__out_fully_fused"]


LAYER_NAMES = sorted(meta()["layers"])
