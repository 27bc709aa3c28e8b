"""The per-node stage API (stages.py) on the GPU, re-expressing the
reference's stage tests (pkg/tests/test_compress.py:159-257, test_linalg.py)
against the drop-in: nullspace / col follow LAPACK conventions, lstsq_right
solves and screens, the discrepancy and root match dense formulas, and a
sweep driven stage by stage equals compress_from_samples as an operator."""
import numpy as np
import pytest
import torch

import paper_2205_02990_b200 as hb
from oracle import hbs_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    hb._native.lib()


@pytest.mark.parametrize("rows,cols,k", [(30, 90, 30), (60, 90, 30), (128, 192, 64), (21, 45, 9)])
def test_nullspace_lapack_convention(rows, cols, k):
    rng = np.random.default_rng(rows + cols)
    b = rng.standard_normal((rows, cols))
    p = hb.nullspace(b, k)
    assert isinstance(p, np.ndarray) and p.shape == (cols, k)
    want = np.linalg.qr(b.T, mode="complete")[0][:, cols - k:]
    assert np.abs(p - want).max() <= 1e-12
    assert np.linalg.norm(b @ p) <= 1e-12 * np.linalg.norm(b)
    with pytest.raises(hb.DimensionError):
        hb.nullspace(b, cols - rows + 1)


@pytest.mark.parametrize("rows,cols,k", [(128, 64, 64), (64, 64, 30), (40, 70, 12)])
def test_col_lapack_convention(rows, cols, k):
    rng = np.random.default_rng(rows * cols)
    b = rng.standard_normal((rows, cols))
    q = hb.col(b, k)
    want = np.linalg.qr(b)[0][:, :k]
    assert np.abs(q - want).max() <= 1e-12
    with pytest.raises(hb.DimensionError):
        hb.col(b, min(rows, cols) + 1)


def test_lstsq_right_planted_and_screen():
    rng = np.random.default_rng(7)
    m = rng.standard_normal((40, 120))
    x = rng.standard_normal((17, 40))
    got = hb.lstsq_right(x @ m, m)
    assert np.abs(got - x).max() <= 1e-12 * np.abs(x).max()
    dev = hb.lstsq_right(torch.from_numpy(x @ m).cuda(), torch.from_numpy(m).cuda())
    assert isinstance(dev, torch.Tensor) and dev.is_cuda
    bad = m.copy()
    bad[3] = bad[2]                       # two identical probe rows (test_linalg.py:142-145)
    with pytest.raises(hb.IllConditionedProbeError):
        hb.lstsq_right(x @ bad, bad)
    with pytest.raises(hb.DimensionError):
        hb.lstsq_right(x, m.T)


def _dense_case(n=512, leaf=24, k=8, r=12, s=36):
    a = O.dense(O.baseline_generator(n, leaf, k, seed=2))
    samples = hb.draw_samples(hb.dense_oracle(a), s, seed=0)
    host = hb.SampleSet(*(np.asarray(m.cpu() if isinstance(m, torch.Tensor) else m) for m in
                          (samples.omega, samples.psi, samples.y, samples.z)))
    return a, host, hb.build_tree(n, leaf), r, leaf


def test_leaf_discrepancy_matches_dense_formula():
    a, samples, tree, r, leaf = _dense_case()
    node = tree.leaves()[3]
    ns = hb.leaf_node_samples(samples, node)
    u, v, _, _ = hb.compress_node_bases(ns, r)
    d = hb.compute_discrepancy(u, v, ns)
    att = a[node.begin:node.end, node.begin:node.end]
    want = att - u @ (u.T @ att @ v) @ v.T
    assert np.linalg.norm(d - want) <= 1e-10 * np.linalg.norm(att)
    assert np.linalg.norm(u.T @ u - np.eye(r)) <= 1e-12


def test_stage_sweep_equals_compress_from_samples():
    """The reference's level loop (compress.py:250-280) written with the stage
    API reproduces compress_from_samples as an operator."""
    a, samples, tree, r, leaf = _dense_case()
    state, ub, vb, db = {}, {}, {}, {}
    for level in range(tree.depth, 0, -1):
        for node in tree.nodes_at_level(level):
            if node.is_leaf:
                ns = hb.leaf_node_samples(samples, node)
            else:
                ns = hb.lift_to_parent(state.pop(node.children[0]), state.pop(node.children[1]))
                assert ns.omega_t.shape == (2 * r, samples.probes)
            u, v, _, _ = hb.compress_node_bases(ns, r)
            d = hb.compute_discrepancy(u, v, ns)
            ub[node.id], vb[node.id], db[node.id] = u, v, d
            state[node.id] = hb.CompressedNode(u, v, d, ns)
    root = tree.nodes[0]
    ns = hb.lift_to_parent(state.pop(root.children[0]), state.pop(root.children[1]))
    core = hb.compute_root(ns)
    f_stage = hb.HbsFactorization(tree, r, ub, vb, db, core)
    f = hb.compress_from_samples(samples, tree, hb.CompressionConfig(rank=r, leaf_threshold=leaf))
    x = O.gaussian(tree.n, 3, 0, 4)
    ref = a @ x
    err_stage = np.linalg.norm(hb.apply_matrix(f_stage, x) - ref) / np.linalg.norm(ref)
    err = np.linalg.norm(hb.apply_matrix(f, x) - ref) / np.linalg.norm(ref)
    assert err_stage <= 1e-10 and err <= 1e-10
    rep = hb.storage(f)
    assert rep.total_floats == sum(lv.basis_floats + lv.disc_floats for lv in rep.levels)
    assert rep.floats_per_dof == rep.total_floats / tree.n
