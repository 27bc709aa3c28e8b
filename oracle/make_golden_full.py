"""Reference error scalars at the FULL BASELINE sizes (test infrastructure).

Run in the build container, where /root/reference exists (takes ~25 min, the
config-4 cases dominate):

    python oracle/make_golden_full.py [case ...]

For every case the UNMODIFIED reference is driven through its own public API
on the BASELINE seeded inputs:

  * truth operator: `hbs_oracle.baseline_generator` (seed 0, stream 3) mapped
    onto a reference `HbsFactorization`, or the config-3 ellipse log kernel
    as a dense array;
  * samples: `hbs.draw_samples(oracle, s, seed=0)` (compress.py:132-141) with
    the reference's own `hbs_oracle` / `dense_oracle` (operators.py:213-228),
    i.e. Omega / Psi = gaussian_matrix(N, s, 0, stream 0 / 1);
  * compression: `hbs.compress_from_samples` (compress.py:236-280);
  * error: ||(A_ref - A) x|| / ||A x|| with x = gaussian(N, 4, 0, stream 4).

Only scalars and the reference's apply of x (all 4 columns for N <= 2^16,
the first column for the config-4 twin) are stored in
tests/golden/full_<case>.npz; the GPU tests regenerate the same inputs from
the seeds, sample them on the device and gate the GPU factorization against
the truth at 10x the reference's error (literal, r = k) or 1e-10 (oversampled
twins, r = k + 8, s = 3r) -- SURVEY.md section 8(c).
"""

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
REF = "/root/reference/pkg/src"

# name: (n, leaf, k, r, s, decay, kind)
FULL_CASES = {
    "c2_literal": (1 << 16, 64, 32, 32, 96, None, "hbs"),
    "c2_twin": (1 << 16, 64, 32, 40, 120, None, "hbs"),
    "c3_literal": (1 << 15, 80, 40, 40, 120, None, "logkernel"),
    "c3_twin": (1 << 15, 80, 40, 48, 144, None, "logkernel"),
    "c4_literal": (1 << 20, 128, 64, 64, 192, 0.9, "hbs"),
    "c4_twin": (1 << 20, 128, 64, 72, 216, 0.9, "hbs"),
}


def to_reference(hbs, of):
    """OracleFactorization -> reference HbsFactorization (factorization.py:25-40)."""
    tree = hbs.build_tree(of.n, int(np.diff(of.bounds[of.depth]).max()))
    assert tree.depth == of.depth
    u, v, d = {}, {}, {}
    for level in range(1, of.depth + 1):
        for j in range(1 << level):
            nid = (1 << level) - 1 + j
            u[nid], v[nid], d[nid] = of.U[level][j], of.V[level][j], of.D[level][j]
    return hbs.HbsFactorization(tree, of.rank, u, v, d, of.root)


def log_kernel_blocked(n, block=4096):
    """The config-3 operator in row blocks (same values as ellipse_log_kernel)."""
    t = 2.0 * np.pi * np.arange(n) / n
    x = np.stack((np.cos(t), 0.5 * np.sin(t)), axis=1)
    a = np.empty((n, n))
    for i0 in range(0, n, block):
        i1 = min(n, i0 + block)
        diff = x[i0:i1, None, :] - x[None, :, :]
        dist = np.sqrt((diff ** 2).sum(-1))
        idx = np.arange(i0, i1)
        dist[idx - i0, idx] = 1.0
        blk = np.log(dist)
        blk[idx - i0, idx] = 1.0
        a[i0:i1] = blk
    return a


def run_case(hbs, O, name, out_dir):
    from hbs import operators
    n, leaf, k, r, s, decay, kind = FULL_CASES[name]
    t0 = time.perf_counter()
    if kind == "hbs":
        truth = O.baseline_generator(n, leaf, k, seed=0, decay=decay)
        oracle = operators.hbs_oracle(to_reference(hbs, truth))
        true_apply = lambda x: O.apply(truth, x)
    else:
        a = log_kernel_blocked(n)
        oracle = operators.dense_oracle(a)
        true_apply = lambda x: a @ x
    tree = hbs.build_tree(n, leaf)
    samples = hbs.draw_samples(oracle, s, 0)
    t1 = time.perf_counter()
    cfg = hbs.CompressionConfig(rank=r, leaf_threshold=leaf, probes=s)
    f = hbs.compress_from_samples(samples, tree, cfg)
    t2 = time.perf_counter()
    x = O.gaussian(n, 4, 0, 4)
    ref_ax = hbs.apply_matrix(f, x)
    true_ax = true_apply(x)
    err = float(np.linalg.norm(ref_ax - true_ax) / np.linalg.norm(true_ax))
    extra = {}
    if n <= (1 << 16):
        extra["ref_ax"] = ref_ax
    elif r > k:   # oversampled config-4 twin: one column (8 MB) for the 1e-10 gate vs the reference
        extra["ref_ax"] = ref_ax[:, :1]
    np.savez_compressed(
        os.path.join(out_dir, f"full_{name}.npz"),
        params=np.array([n, leaf, k, r, s], dtype=np.int64),
        decay=np.array(-1.0 if decay is None else decay),
        kind=np.array(kind),
        depth=np.array(tree.depth),
        omega_sum=np.array(samples.omega.sum()), psi_sum=np.array(samples.psi.sum()),
        y_sum=np.array(samples.y.sum()), z_sum=np.array(samples.z.sum()),
        true_ax_sum=np.array(true_ax.sum()),
        ref_err_vs_truth=np.array(err),
        ref_compress_s=np.array(t2 - t1),
        **extra,
    )
    print(f"{name}: N={n} depth={tree.depth} ref err vs truth {err:.3e}  "
          f"(inputs {t1 - t0:.1f} s, compress {t2 - t1:.1f} s)", flush=True)


def main():
    sys.path.insert(0, REF)
    import hbs
    from oracle import hbs_oracle as O
    out_dir = os.path.join(os.path.dirname(HERE), "tests", "golden")
    names = sys.argv[1:] or list(FULL_CASES)
    for name in names:
        run_case(hbs, O, name, out_dir)


if __name__ == "__main__":
    main()
