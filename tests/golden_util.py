"""Loaders for the committed golden fixtures (made by tests/golden/make_golden.py)."""

from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def cases(name):
    d = np.load(GOLDEN / f"{name}.npz")
    n = int(d["n_cases"])
    out = []
    for i in range(n):
        pre = f"c{i}_"
        out.append({k[len(pre):]: d[k] for k in d.files if k.startswith(pre)})
    return out


def toy_bundle_path(ci):
    return GOLDEN / f"toy_eps{[0, 2, 5][ci]}.bin"
