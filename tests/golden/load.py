"""Loads the reference-generated golden fixtures (see make_golden.py)."""
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def load_golden(body):
    z = np.load(os.path.join(HERE, f"{body}.npz"))
    tconst = float(z["__thres_const__"])
    keys = sorted({k.split("/")[0] for k in z.files if not k.startswith("__")})
    cases = []
    for key in keys:
        c = {"name": f"{body}:{key}", "source": str(z["__source__"])}
        for part in ("A", "B", "thres", "dis", "R"):
            if f"{key}/{part}" in z.files:
                c[part] = z[f"{key}/{part}"].astype(np.float64)
        if not np.isnan(tconst):
            c["thres_const"] = tconst
        cases.append(c)
    return cases
