"""Device samplers behind the black-box boundary (operators.py:213-228).

`dense_oracle` keeps the explicit matrix in HBM and multiplies on the FP64
tensor cores (`hbs_dense_apply`); `hbs_oracle` applies a telescoping
factorization with the level-batched up/root/down sweep (`hbs_apply`).  Both
accept numpy (returns numpy) or CUDA tensors (returns CUDA tensors).
"""

import numpy as np
import torch

from . import _native
from .errors import DimensionError
from .factorization import HbsFactorization, apply_matrix
from .matvec import MatVecOracle


def dense_apply(a_dev: torch.Tensor, x, transpose=False, stream=None):
    """A x or A^T x for a device-resident dense A (n x n, float64)."""
    host = not isinstance(x, torch.Tensor)
    xd = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(a_dev.device) if host \
        else x.to(device=a_dev.device, dtype=torch.float64).contiguous()
    n, c = xd.shape
    out = torch.empty_like(xd)
    st = stream if stream is not None else torch.cuda.current_stream(a_dev.device).cuda_stream
    rc = _native.lib().hbs_dense_apply(n, c, a_dev.data_ptr(), xd.data_ptr(), out.data_ptr(),
                                       1 if transpose else 0, st)
    _native.check(rc, "hbs_dense_apply")
    return out.cpu().numpy() if host else out


def dense_oracle(a, device=None) -> MatVecOracle:
    """Wrap an explicit square matrix as a black-box oracle (operators.py:213-218)."""
    if isinstance(a, torch.Tensor):
        a_dev = a.to(device=device or a.device, dtype=torch.float64).contiguous()
    else:
        a = np.asarray(a, dtype=np.float64)
        a_dev = torch.from_numpy(np.ascontiguousarray(a)).to(device or "cuda")
    if a_dev.ndim != 2 or a_dev.shape[0] != a_dev.shape[1]:
        raise DimensionError(f"dense oracle needs a square matrix, got shape {tuple(a_dev.shape)}")
    return MatVecOracle(a_dev.shape[0], lambda x: dense_apply(a_dev, x), lambda x: dense_apply(a_dev, x, True),
                        device_aware=True)


def hbs_oracle(f: HbsFactorization) -> MatVecOracle:
    """Matrix-free oracle of a telescoping factorization (operators.py:221-228)."""
    return MatVecOracle(f.n, lambda x: apply_matrix(f, x), lambda x: apply_matrix(f, x, transpose=True),
                        device_aware=True)


def log_kernel_matrix(n: int, device=None) -> torch.Tensor:
    """Config-3 operator (ellipse log kernel) generated on the device."""
    dev = torch.device(device) if device is not None else torch.device("cuda")
    a = torch.empty(n, n, dtype=torch.float64, device=dev)
    rc = _native.lib().hbs_fill_log_kernel(n, 0, n, a.data_ptr(), torch.cuda.current_stream(dev).cuda_stream)
    _native.check(rc, "hbs_fill_log_kernel")
    return a
