"""Loader for tests/golden/*.npz (made by oracle/make_golden.py from the
unmodified reference).  Inputs are regenerated from seeds by the oracle."""
import glob
import os

import numpy as np

from oracle import hbs_oracle as O

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names():
    """Reduced-size fixtures (oracle/make_golden.py)."""
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz"))
                  if not os.path.basename(p).startswith("full_"))


def full_names():
    """Full BASELINE-size fixtures (oracle/make_golden_full.py): scalars only."""
    return sorted(os.path.basename(p)[5:-4] for p in glob.glob(os.path.join(GOLDEN_DIR, "full_*.npz")))


def load_full(name):
    """Parameters, reference scalars and the host-side seeded inputs of a
    full-size case: the truth operator (OracleFactorization or dense array)
    and Omega / Psi = gaussian(N, s, 0, stream 0 / 1) (linalg.py:23-32)."""
    g = np.load(os.path.join(GOLDEN_DIR, "full_" + name + ".npz"))
    n, leaf, k, r, s = (int(v) for v in g["params"])
    decay = float(g["decay"])
    kind = str(g["kind"])
    truth = O.baseline_generator(n, leaf, k, seed=0, decay=None if decay < 0 else decay) if kind == "hbs" else None
    return dict(fixture=g, n=n, leaf=leaf, k=k, r=r, s=s, kind=kind, truth=truth, literal=(r == k),
                omega=O.gaussian(n, s, 0, O.STREAM_OMEGA), psi=O.gaussian(n, s, 0, O.STREAM_PSI),
                x=O.gaussian(n, 4, 0, 4))


def load(name):
    g = np.load(os.path.join(GOLDEN_DIR, name + ".npz"))
    n, leaf, k, r, s = (int(v) for v in g["params"])
    decay = float(g["decay"])
    kind = str(g["kind"])
    truth = O.baseline_generator(n, leaf, k, seed=0, decay=None if decay < 0 else decay) if kind == "hbs" \
        else O.ellipse_log_kernel(n)
    om, ps, y, z = O.samples_from(truth, s, 0)
    return dict(fixture=g, n=n, leaf=leaf, k=k, r=r, s=s, truth=truth, samples=(om, ps, y, z),
                literal=(r == k), x=O.gaussian(n, 4, 0, 4))
