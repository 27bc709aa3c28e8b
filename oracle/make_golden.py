"""Generate tests/golden/*.npz from the UNMODIFIED reference (run in the build
container, where /root/reference exists):

    python oracle/make_golden.py

Each fixture stores the case parameters, the reference's root core, a few
per-node blocks, its apply of a fixed probe x = gaussian(N, 4, 0, stream=4),
and the true operator's apply of the same x.  Inputs are NOT stored: they are
regenerated bit-exactly from the seeds (numpy PCG64 streams), which the
fixtures also pin via checksums of omega / y.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
REF = "/root/reference/pkg/src"

# name: (n, leaf, k, r, s, decay, kind)
CASES = {
    "c1_literal": (4096, 32, 16, 16, 48, None, "hbs"),
    "c1_twin": (4096, 32, 16, 24, 72, None, "hbs"),
    "c2_shape_twin": (4096, 64, 32, 40, 120, None, "hbs"),
    "c2_shape_literal": (4096, 64, 32, 32, 96, None, "hbs"),
    "c4_shape_twin": (2048, 128, 64, 72, 216, 0.9, "hbs"),
    "c4_shape_literal": (2048, 128, 64, 64, 192, 0.9, "hbs"),
    "c3_shape_literal": (2048, 80, 40, 40, 120, None, "logkernel"),
    "c3_shape_twin": (2048, 80, 40, 48, 144, None, "logkernel"),
    "uneven_333": (333, 24, 4, 8, 32, None, "hbs"),
    "depth_one": (40, 20, 3, 6, 26, None, "hbs"),
}


def build_case(name):
    from oracle import hbs_oracle as O
    n, leaf, k, r, s, decay, kind = CASES[name]
    if kind == "hbs":
        truth = O.baseline_generator(n, leaf, k, seed=0, decay=decay)
    else:
        truth = O.ellipse_log_kernel(n)
    om, ps, y, z = O.samples_from(truth, s, 0)
    return truth, (om, ps, y, z)


def main():
    sys.path.insert(0, REF)
    import hbs
    from oracle import hbs_oracle as O
    out_dir = os.path.join(os.path.dirname(HERE), "tests", "golden")
    os.makedirs(out_dir, exist_ok=True)
    for name, (n, leaf, k, r, s, decay, kind) in CASES.items():
        truth, (om, ps, y, z) = build_case(name)
        tree = hbs.build_tree(n, leaf)
        f = hbs.compress_from_samples(hbs.SampleSet(om, ps, y, z), tree,
                                      hbs.CompressionConfig(rank=r, leaf_threshold=leaf))
        x = O.gaussian(n, 4, 0, 4)
        ref_ax = hbs.apply_matrix(f, x)
        ref_atx = hbs.apply_matrix(f, x, transpose=True)
        true_ax = truth @ x if isinstance(truth, np.ndarray) else O.apply(truth, x)
        # The literal (r == k) configs are rounding-chaotic: record the spread
        # of the reference's own error under 1e-16 relative perturbations of Y, Z.
        perturbed = []
        if r == k:
            for pseed in range(6):
                rng = np.random.default_rng(pseed)
                yp = y * (1 + 1e-16 * rng.standard_normal(y.shape))
                zp = z * (1 + 1e-16 * rng.standard_normal(z.shape))
                fp = hbs.compress_from_samples(hbs.SampleSet(om, ps, yp, zp), tree,
                                               hbs.CompressionConfig(rank=r, leaf_threshold=leaf))
                pax = hbs.apply_matrix(fp, x)
                perturbed.append(np.linalg.norm(pax - true_ax) / np.linalg.norm(true_ax))
        leaves = tree.leaves()
        first_leaf, lvl1 = leaves[0].id, tree.nodes_at_level(1)[0].id
        np.savez_compressed(
            os.path.join(out_dir, f"{name}.npz"),
            params=np.array([n, leaf, k, r, s], dtype=np.int64),
            decay=np.array(-1.0 if decay is None else decay),
            kind=np.array(kind),
            root=f.root_disc,
            ref_ax=ref_ax, ref_atx=ref_atx, true_ax=true_ax,
            leaf_id=np.array(first_leaf), leaf_u=f.u_bases[first_leaf], leaf_v=f.v_bases[first_leaf],
            leaf_d=f.discs[first_leaf],
            l1_id=np.array(lvl1), l1_u=f.u_bases[lvl1], l1_v=f.v_bases[lvl1], l1_d=f.discs[lvl1],
            omega_sum=np.array(om.sum()), y_sum=np.array(y.sum()), z_sum=np.array(z.sum()),
            ref_err_vs_truth=np.array(np.linalg.norm(ref_ax - true_ax) / np.linalg.norm(true_ax)),
            ref_err_perturbed=np.array(perturbed, dtype=np.float64),
        )
        print(name, "ref err vs truth %.3e" % (np.linalg.norm(ref_ax - true_ax) / np.linalg.norm(true_ax)),
              "perturbed max %.3e" % (max(perturbed) if perturbed else 0.0))


if __name__ == "__main__":
    main()
