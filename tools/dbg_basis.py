import sys; sys.path.insert(0, "/root/repo")
import numpy as np
from tests.test_gpu_kernels import basis_qr
rows, r = 40, 40
rng = np.random.default_rng(rows * 100 + r)
blocks = [rng.standard_normal((rows, r)) for _ in range(3)]
for rep in range(3):
    qs = basis_qr(blocks, r)
    for bi, (b, q) in enumerate(zip(blocks, qs)):
        qr = np.linalg.qr(b)[0]
        err = np.abs(q - qr).max(axis=0)
        bad = np.where(err > 1e-10)[0]
        print(rep, bi, "bad cols", bad, "orth %.1e" % np.linalg.norm(q.T @ q - np.eye(r)),
              "span %.1e" % np.linalg.norm(b - q @ (q.T @ b)), "sign flip?" , [np.abs(q[:, c] + qr[:, c]).max() < 1e-10 for c in bad])
