"""Relative-error verification on the device (§8(f) row 2).

`power_method_relnorm` restates `linalg.py:93-129`: both norms are estimated
by `iters` power iterations on the Gram operator x <- op_t(op(x)), from the
same seeded start vector (stream STREAM_POWER, moving to the next stream on a
zero draw).  `estimate_rel_err` is `bench.py:79-90`: E = oracle - compressed,
through matvecs only.  Operators may take/return numpy or CUDA tensors; the
iteration itself runs on the device.
"""

import numpy as np
import torch

from .compress import STREAM_POWER, gaussian_matrix
from .errors import DimensionError
from .factorization import apply_matrix


def _as_col(x, device):
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.asarray(x, dtype=np.float64))
    t = t.to(device=device, dtype=torch.float64)
    return t.reshape(-1, 1) if t.ndim == 1 else t


def _device_op(op, device):
    """Wrap a matvec handle for the device iteration.  Handles marked
    `hbs_device_aware` (the compressed factorization's apply, in-house
    samplers) take the CUDA column as is; any other callable follows the
    reference contract (linalg.py:108-129): a 1-D numpy vector in, a vector
    out."""
    if getattr(op, "hbs_device_aware", False):
        return op

    def host(x):
        y = op(x.detach().cpu().numpy().reshape(-1))
        return _as_col(y, device)
    return host


def _device_aware(fn):
    fn.hbs_device_aware = True
    return fn


def _gram_norm(op, op_t, x0, iters):
    x = x0 / torch.linalg.norm(x0)
    est = 0.0
    for _ in range(iters):
        y = _as_col(op_t(op(x)), x.device)
        gain = float(torch.linalg.norm(y))
        if gain == 0.0:
            return 0.0
        est = float(np.sqrt(gain))
        x = y / gain
    return est


def power_method_relnorm(op_e, op_et, op_a, op_at, n, iters=20, seed=0, device=None):
    """Estimate ||E|| / ||A|| from matvec handles only (linalg.py:108-129)."""
    if iters < 1:
        raise DimensionError("power method needs at least one iteration")
    dev = torch.device(device) if device is not None else torch.device("cuda")
    stream = STREAM_POWER
    x0 = gaussian_matrix(n, 1, seed, stream)
    while not np.linalg.norm(x0) > 0.0:
        stream += 1
        x0 = gaussian_matrix(n, 1, seed, stream)
    x0 = torch.from_numpy(x0).to(dev)
    op_e, op_et, op_a, op_at = (_device_op(o, dev) for o in (op_e, op_et, op_a, op_at))
    e_norm = _gram_norm(op_e, op_et, x0, iters)
    a_norm = _gram_norm(op_a, op_at, x0, iters)
    if a_norm == 0.0:
        raise ValueError("reference operator norm estimate is zero; relative error undefined")
    return e_norm / a_norm


def estimate_rel_err(oracle, f, iters=20, seed=0):
    """Power-method ||A_oracle - A_f|| / ||A_oracle|| (bench.py:79-90) with the
    compressed factorization applied on the device.  A device-aware oracle
    (MatVecOracle.device_aware) takes CUDA columns; any other oracle gets numpy
    n x 1 arrays, as in the reference."""
    dev = f.device

    if getattr(oracle, "device_aware", False):
        def a(x):
            return _as_col(oracle.apply_batch(x), dev)

        def at(x):
            return _as_col(oracle.apply_transpose_batch(x), dev)
    else:
        def a(x):
            return _as_col(oracle.apply_batch(x.detach().cpu().numpy()), dev)

        def at(x):
            return _as_col(oracle.apply_transpose_batch(x.detach().cpu().numpy()), dev)

    ops = [_device_aware(fn) for fn in (lambda x: a(x) - apply_matrix(f, x), lambda x: at(x) - apply_matrix(f, x, True),
                                        a, at)]
    return power_method_relnorm(*ops, oracle.n, iters=iters, seed=seed, device=dev)
