"""Loader for the committed reference fixtures in tests/golden (see make_golden.py)."""
import os
from collections import defaultdict

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def solves():
    z = np.load(os.path.join(HERE, "reference_solves.npz"), allow_pickle=False)
    out = defaultdict(dict)
    for key in z.files:
        name, field = key.split("__", 1)
        out[name][field] = z[key]
    for d in out.values():
        for f in ("ab", "bb"):
            if d[f].size == 0:
                d[f] = None
        for f in ("tile", "status", "events"):
            d[f] = int(d[f])
        for f in ("alpha", "omega", "pivot"):
            d[f] = float(d[f])
        d["origin"] = str(d["origin"])
    return dict(out)


def guards():
    return np.load(os.path.join(HERE, "guards.npz"))


def robust_updates():
    z = np.load(os.path.join(HERE, "robust_update.npz"))
    out = []
    for k in sorted(z.files, key=int):
        v = z[k]
        m, k_, n = int(v[0]), int(v[1]), int(v[2])
        g, al, be, st, s, nr = v[3:9]
        o = 9
        c = v[o:o + m * n].reshape((m, n), order="F"); o += m * n
        a = v[o:o + m * k_].reshape((m, k_), order="F"); o += m * k_
        b = v[o:o + k_ * n].reshape((k_, n), order="F"); o += k_ * n
        y = v[o:o + m * n].reshape((m, n), order="F")
        out.append(dict(c=c, a=a, b=b, g=g, al=al, be=be, status=int(st), scale=s, norm=nr, y=y))
    return out


def rel_inf_diff(got, want):
    """tests/support/oracles.cpp:75-81"""
    d = np.abs(got - want).sum(axis=1).max() if got.size else 0.0
    r = np.abs(want).sum(axis=1).max() if want.size else 0.0
    return d / r if r else d
