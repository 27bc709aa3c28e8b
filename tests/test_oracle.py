"""CPU: the oracle restatement is pinned to the reference (golden fixtures made
from the unmodified reference, and the live reference when present)."""
import numpy as np
import pytest

from oracle import hbs_oracle as O
from tests import golden_cases

CASES = golden_cases.names()


def test_golden_fixtures_exist():
    assert len(CASES) >= 8


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_golden(name):
    c = golden_cases.load(name)
    g = c["fixture"]
    om, ps, y, z = c["samples"]
    # inputs regenerate bit-exactly from the seeds
    assert om.sum() == float(g["omega_sum"])
    assert np.isclose(y.sum(), float(g["y_sum"]), rtol=1e-12, atol=1e-9)
    f = O.compress(om, ps, y, z, O.level_bounds(c["n"], _depth(c)), c["r"])
    ax = O.apply(f, c["x"])
    ref = g["ref_ax"]
    err = np.linalg.norm(ax - ref) / np.linalg.norm(ref)
    # same LAPACK calls in the same order: agreement to rounding of the host BLAS
    bar = 1e-6 * max(float(g["ref_err_vs_truth"]), 1e-12) / 1e-12 if c["literal"] else 1e-12
    assert err <= max(bar, 1e-12), err
    np.testing.assert_allclose(f.root, g["root"], rtol=0, atol=1e-8 * np.abs(g["root"]).max()
                               if c["literal"] else 1e-11 * np.abs(g["root"]).max())


def _depth(c):
    from paper_2205_02990_b200.tree import tree_depth
    return tree_depth(c["n"], c["leaf"])


def test_oracle_bitwise_equals_live_reference(reference_hbs):
    hbs = reference_hbs
    n, m, k, r, s = 1024, 32, 16, 24, 72
    g = O.baseline_generator(n, m, k, seed=3)
    om, ps, y, z = O.samples_from(g, s, 0)
    f = O.compress(om, ps, y, z, g.bounds, r)
    fr = hbs.compress_from_samples(hbs.SampleSet(om, ps, y, z), hbs.build_tree(n, m),
                                   hbs.CompressionConfig(rank=r, leaf_threshold=m))
    assert np.array_equal(f.root, fr.root_disc)
    for nid in (1, 2, 40, 62):
        u, v, d = f.node_blocks(nid)
        assert np.array_equal(u, fr.u_bases[nid])
        assert np.array_equal(v, fr.v_bases[nid])
        assert np.array_equal(d, fr.discs[nid])


def test_oracle_apply_matches_reference_apply(reference_hbs):
    hbs = reference_hbs
    g = O.baseline_generator(333, 24, 4, seed=1)
    tree = hbs.build_tree(333, 24)
    blocks = {}
    for lvl in range(1, tree.depth + 1):
        for j, nd in enumerate(tree.nodes_at_level(lvl)):
            blocks[nd.id] = (g.U[lvl][j], g.V[lvl][j], g.D[lvl][j])
    fr = hbs.HbsFactorization(tree, 4, {i: b[0] for i, b in blocks.items()}, {i: b[1] for i, b in blocks.items()},
                              {i: b[2] for i, b in blocks.items()}, g.root)
    x = O.gaussian(333, 3, 0, 4)
    assert np.allclose(O.apply(g, x), hbs.apply_matrix(fr, x), rtol=0, atol=1e-12)
    assert np.allclose(O.apply(g, x, transpose=True), hbs.apply_matrix(fr, x, transpose=True), rtol=0, atol=1e-12)
    assert np.allclose(O.dense(g), hbs.to_dense(fr), rtol=0, atol=1e-12)


def test_oracle_ill_conditioned_box_reported():
    n, s, r = 16, 6, 1
    om = O.gaussian(n, s, 36, 0)
    om[1] = om[0]
    ps = O.gaussian(n, s, 36, 1)
    with pytest.raises(O.ProbeRankError) as exc:
        O.compress(om, ps, om.copy(), ps.copy(), O.level_bounds(n, 3), r)
    assert exc.value.level == 3 and exc.value.box == 0


def test_gaussian_stream_frozen():
    # test_linalg.py:9-11 frozen mean / variance of seed 7, stream 0
    g = O.gaussian(10000, 1, 7, 0)
    np.testing.assert_allclose(g.mean(), -0.01581890868143026, rtol=1e-12)
    np.testing.assert_allclose(g.var(ddof=1), 0.9942184780399852, rtol=1e-12)


def test_power_method_matches_reference_semantics(reference_hbs):
    """verify.power_method_relnorm restates linalg.py:108-129 (same start
    stream) and, like the reference, hands plain callables 1-D numpy vectors."""
    pytest.importorskip("torch")
    from paper_2205_02990_b200.verify import power_method_relnorm
    rng = np.random.default_rng(7)
    a = rng.standard_normal((32, 32))
    d = np.ones(32)
    d[0] = 3.0
    ops = (lambda x: d * x, lambda x: d * x, lambda x: a @ x, lambda x: a.T @ x)
    mine = power_method_relnorm(*ops, 32, iters=20, seed=4, device="cpu")
    ref = reference_hbs.power_method_relnorm(*ops, 32, iters=20, seed=4)
    assert abs(mine - ref) <= 1e-12 * ref
