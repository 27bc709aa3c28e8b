"""The reference's compressor tests (pkg/tests/test_compress.py,
test_acceptance.py) re-expressed against the drop-in API on the GPU.
Dense ground truth comes from the oracle's generator (random_hbs is a test
generator of the reference, outside the hot path)."""
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


def dense_hbs(n, m, k, seed):
    return O.dense(O.baseline_generator(n, m, k, seed=seed))


def rel2(a, b):
    return np.linalg.norm(a - b, 2) / np.linalg.norm(b, 2)


def to_dense(f):
    n = f.n
    return hb.apply_matrix(f, np.eye(n))


class TestDrawSamples:   # test_compress.py:49-65
    def test_identity_oracle(self):
        s = hb.draw_samples(hb.dense_oracle(np.eye(12)), 5, seed=0)
        np.testing.assert_array_equal(s.y, s.omega)
        np.testing.assert_array_equal(s.z, s.psi)

    def test_counters_advance_exactly(self):
        o = hb.dense_oracle(np.eye(12))
        hb.draw_samples(o, 7, seed=0)
        assert o.matvec_count == (7, 7)

    def test_diagonal_action(self):
        d = np.arange(1.0, 11.0)
        s = hb.draw_samples(hb.dense_oracle(np.diag(d)), 4, seed=1)
        np.testing.assert_allclose(s.y, d[:, None] * s.omega)


class TestCompress:      # test_compress.py:280-393
    def test_exact_rank_recovery(self):
        n, k, r, m = 960, 10, 15, 30
        a = dense_hbs(n, m, k, 27)
        o = hb.dense_oracle(a)
        f = hb.compress(o, hb.CompressionConfig(rank=r, leaf_threshold=m, probes=45, seed=28))
        assert rel2(to_dense(f), a) <= 1e-10
        assert o.matvec_count == (45, 45)

    def test_diagonal_matrix(self):
        a = np.diag(np.linspace(1.0, 2.0, 200))
        f = hb.compress(hb.dense_oracle(a), hb.CompressionConfig(rank=5, leaf_threshold=10, seed=29))
        assert rel2(to_dense(f), a) <= 1e-12

    def test_probe_budget_is_exact(self):
        n = 128
        a = dense_hbs(n, 16, 4, 30)
        o = hb.dense_oracle(a)
        cfg = hb.CompressionConfig(rank=6, leaf_threshold=16, seed=31)
        s = cfg.validate_for(hb.build_tree(n, 16))
        hb.compress(o, cfg)
        assert o.matvec_count == (s, s)

    def test_deterministic_bitwise(self):
        a = dense_hbs(96, 12, 3, 32)
        cfg = hb.CompressionConfig(rank=5, leaf_threshold=12, seed=33)
        f1, f2 = hb.compress(hb.dense_oracle(a), cfg), hb.compress(hb.dense_oracle(a), cfg)
        assert np.array_equal(f1.root_disc, f2.root_disc)
        for nid in f1.u_bases:
            assert np.array_equal(f1.u_bases[nid], f2.u_bases[nid])
            assert np.array_equal(f1.discs[nid], f2.discs[nid])

    def test_oversampling_monotonicity(self):
        a = dense_hbs(960, 30, 5, 11)
        med = {}
        for rank in (7, 15):
            errs = [rel2(to_dense(hb.compress(hb.dense_oracle(a), hb.CompressionConfig(rank=rank, leaf_threshold=30,
                                                                                          seed=seed))), a)
                    for seed in range(10)]
            med[rank] = np.median(errs)
        assert med[15] <= med[7]

    def test_arithmetic_scales_linearly(self):
        madds = {}
        for n in (2048, 4096):
            tree = hb.build_tree(n, 10)
            g = O.baseline_generator(n, 10, 2, seed=34)
            om, ps, y, z = O.samples_from(g, 15, 35)
            with hb.flops.count_madds() as c:
                hb.compress_from_samples(hb.SampleSet(om, ps, y, z), tree, hb.CompressionConfig(rank=5, leaf_threshold=10))
            madds[n] = c.madds
        assert 1.8 <= madds[4096] / madds[2048] <= 2.3

    def test_ill_conditioned_probe_names_node(self):
        n = 16
        tree = hb.build_tree(n, 2)
        cfg = hb.CompressionConfig(rank=1, leaf_threshold=2, probes=6, seed=36)
        om = hb.gaussian_matrix(n, 6, 36, 0)
        om[1] = om[0]
        ps = hb.gaussian_matrix(n, 6, 36, 1)
        with pytest.raises(hb.IllConditionedProbeError) as exc:
            hb.compress_from_samples(hb.SampleSet(om, ps, om.copy(), ps.copy()), tree, cfg)
        assert exc.value.node_id == (1 << tree.depth) - 1   # first leaf
        assert exc.value.level == tree.depth

    def test_depth_one_tree(self):
        n, k, r, m = 40, 3, 6, 20
        assert hb.build_tree(n, m).depth == 1
        a = dense_hbs(n, m, k, 40)
        f = hb.compress(hb.dense_oracle(a), hb.CompressionConfig(rank=r, leaf_threshold=m, seed=41))
        assert rel2(to_dense(f), a) <= 1e-11

    def test_uneven_leaves(self):
        n, k, r, m = 333, 4, 8, 24
        tree = hb.build_tree(n, m)
        assert tree.min_leaf_size != tree.max_leaf_size
        a = dense_hbs(n, m, k, 42)
        f = hb.compress(hb.dense_oracle(a), hb.CompressionConfig(rank=r, leaf_threshold=m, seed=43))
        assert rel2(to_dense(f), a) <= 1e-10

    def test_compressed_bases_are_orthonormal(self):
        a = dense_hbs(200, 20, 4, 37)
        hb.compress(hb.dense_oracle(a), hb.CompressionConfig(rank=8, leaf_threshold=20, seed=38)).validate()

    def test_scaling_commutes(self):   # test_compress.py:267-277
        a = np.random.default_rng(25).standard_normal((64, 64))
        cfg = hb.CompressionConfig(rank=4, leaf_threshold=8, seed=26)
        f1 = hb.compress(hb.dense_oracle(a), cfg)
        f2 = hb.compress(hb.dense_oracle(3.0 * a), cfg)
        assert np.linalg.norm(f2.root_disc - 3.0 * f1.root_disc) <= 1e-12 * np.linalg.norm(f1.root_disc)

    def test_zero_matrix(self):        # test_compress.py:259-265 via the full sweep
        f = hb.compress(hb.dense_oracle(np.zeros((16, 16))), hb.CompressionConfig(rank=3, leaf_threshold=8, probes=17))
        np.testing.assert_allclose(f.root_disc, 0.0, atol=1e-12)
        np.testing.assert_allclose(to_dense(f), 0.0, atol=1e-12)

    def test_block_diagonal_operator(self):  # off-diagonal blocks vanish: D carries everything
        rng = np.random.default_rng(16)
        import scipy.linalg
        a = scipy.linalg.block_diag(*(rng.standard_normal((8, 8)) for _ in range(8)))
        f = hb.compress(hb.dense_oracle(a), hb.CompressionConfig(rank=2, leaf_threshold=8, probes=24))
        assert rel2(to_dense(f), a) <= 1e-10


@pytest.mark.parametrize("k,depth", [(1, 1), (5, 2), (10, 3), (5, 4)])
def test_acceptance_exact_rank_power_method(k, depth):   # test_acceptance.py:27-46
    from paper_2205_02990_b200.verify import estimate_rel_err
    r = k + 5
    m = 2 * r
    n = m * (1 << depth)
    tree = hb.build_tree(n, m)
    assert tree.depth == depth
    a = dense_hbs(n, m, k, 7)
    o = hb.dense_oracle(a)
    f = hb.compress(o, hb.CompressionConfig(rank=r, leaf_threshold=m, probes=3 * r, seed=3))
    assert estimate_rel_err(o, f, iters=20, seed=0) <= 1e-9


def test_hbs_sampler_large_n_matches_dense_blocks():
    """Matrix-free sampler at a size that is never densified, checked on a few
    random entries against the telescoping definition."""
    g = O.baseline_generator(8192, 32, 8, seed=5)
    tree = hb.build_tree(8192, 32)
    ub, vb, db = {}, {}, {}
    for lvl in range(1, tree.depth + 1):
        for j, nd in enumerate(tree.nodes_at_level(lvl)):
            ub[nd.id], vb[nd.id], db[nd.id] = g.U[lvl][j], g.V[lvl][j], g.D[lvl][j]
    f = hb.HbsFactorization(tree, 8, ub, vb, db, g.root)
    x = O.gaussian(8192, 3, 0, 4)
    assert np.linalg.norm(hb.apply_matrix(f, x) - O.apply(g, x)) <= 1e-13 * np.linalg.norm(O.apply(g, x))
