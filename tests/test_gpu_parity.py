"""GPU parity: the CUDA path (through the C-ABI) against the oracle and the
reference's golden fixtures.

Parity contract:
  * oversampled twins (r > k): ||(A_gpu - A_ref) x|| / ||A_ref x|| <= 1e-10;
  * literal configs (r = k, rounding-chaotic in the reference itself):
    ||(A_gpu - A) x|| / ||A x|| <= 10 x the reference's own error vs the truth,
    where "the reference's own error" is the max over the reference run on the
    exact samples and on six 1e-16-relative perturbations of (Y, Z) (recorded
    in the golden fixture by oracle/make_golden.py with the real reference);
  * node-level: projectors U U^T, V V^T and D of the first leaf / level-1 node
    within 1e-10 of the reference when the case is well conditioned.
"""
import numpy as np
import pytest
import torch

import paper_2205_02990_b200 as hb
from oracle import hbs_oracle as O
from tests import golden_cases

pytestmark = pytest.mark.gpu

CASES = golden_cases.names()


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    hb._native.lib()   # fail loudly if the extension is missing


def gpu_compress(samples, n, leaf, r, tol=1e-10):
    tree = hb.build_tree(n, leaf)
    return hb.compress_from_samples(hb.SampleSet(*samples), tree,
                                    hb.CompressionConfig(rank=r, leaf_threshold=leaf, ill_conditioning_tol=tol))


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("name", CASES)
def test_golden_operator_parity(name):
    c = golden_cases.load(name)
    g = c["fixture"]
    f = gpu_compress(c["samples"], c["n"], c["leaf"], c["r"])
    ax = hb.apply_matrix(f, c["x"])
    atx = hb.apply_matrix(f, c["x"], transpose=True)
    ref_err = max([float(g["ref_err_vs_truth"])] + [float(v) for v in g["ref_err_perturbed"]])
    err_truth = rel(ax, g["true_ax"])
    if c["literal"]:
        assert err_truth <= 10.0 * ref_err, (err_truth, ref_err)
    else:
        assert rel(ax, g["ref_ax"]) <= 1e-10
        assert rel(atx, g["ref_atx"]) <= 1e-10
        assert err_truth <= 1e-10


@pytest.mark.parametrize("name", [n for n in CASES if "literal" in n and "c3" not in n])
def test_leaf_projectors_literal(name):
    """r == k and nullity == r at the leaves: span(U), span(V) and D of a leaf
    are unique, so they must match the reference's node for node.  (Config 3
    is excluded: its leaf samples Y P are numerically rank deficient --
    sigma_min/sigma_max ~ 3e-17 -- so span(U) is rounding-determined there,
    in the reference as much as here.)"""
    c = golden_cases.load(name)
    g = c["fixture"]
    f = gpu_compress(c["samples"], c["n"], c["leaf"], c["r"])
    nid = int(g["leaf_id"])
    u, v, d = f.u_bases[nid], f.v_bases[nid], f.discs[nid]
    ur, vr, dr = g["leaf_u"], g["leaf_v"], g["leaf_d"]
    assert np.linalg.norm(u @ u.T - ur @ ur.T) <= 1e-9
    assert np.linalg.norm(v @ v.T - vr @ vr.T) <= 1e-9
    assert np.linalg.norm(d - dr) <= 1e-9 * np.linalg.norm(dr)
    assert np.linalg.norm(u.T @ u - np.eye(c["r"])) <= 1e-12


@pytest.mark.parametrize("name", [n for n in CASES if "twin" in n and "c3" not in n])
def test_leaf_bases_contain_true_range_twin(name):
    """r > k: U is the true rank-k range plus r - k rounding-determined
    directions (not unique, also in the reference).  The invariant is that
    span(U) contains the generator's leaf basis."""
    c = golden_cases.load(name)
    f = gpu_compress(c["samples"], c["n"], c["leaf"], c["r"])
    truth = c["truth"]
    L = f.tree.depth
    for j in (0, (1 << L) - 1):
        nid = (1 << L) - 1 + j
        u, v = f.u_bases[nid], f.v_bases[nid]
        ut, vt = truth.U[L][j], truth.V[L][j]
        assert np.linalg.norm(ut - u @ (u.T @ ut)) <= 1e-10
        assert np.linalg.norm(vt - v @ (v.T @ vt)) <= 1e-10
        assert np.linalg.norm(u.T @ u - np.eye(c["r"])) <= 1e-12


def test_dense_sampler_matches_numpy():
    rng = np.random.default_rng(0)
    a = rng.standard_normal((300, 300))
    x = rng.standard_normal((300, 77))
    o = hb.dense_oracle(a)
    assert rel(o.apply_batch(x), a @ x) <= 1e-14
    assert rel(o.apply_transpose_batch(x), a.T @ x) <= 1e-14
    assert o.matvec_count == (77, 77)


def test_log_kernel_generator():
    a = hb.log_kernel_matrix(512).cpu().numpy()
    assert np.abs(a - O.ellipse_log_kernel(512)).max() <= 1e-13


def test_hbs_sampler_matches_oracle_apply():
    g = O.baseline_generator(333, 24, 4, seed=1)
    tree = hb.build_tree(333, 24)
    ub, vb, db = {}, {}, {}
    for lvl in range(1, tree.depth + 1):
        for j, nd in enumerate(tree.nodes_at_level(lvl)):
            ub[nd.id], vb[nd.id], db[nd.id] = g.U[lvl][j], g.V[lvl][j], g.D[lvl][j]
    f = hb.HbsFactorization(tree, 4, ub, vb, db, g.root)
    x = O.gaussian(333, 5, 0, 4)
    assert rel(hb.apply_matrix(f, x), O.apply(g, x)) <= 1e-14
    assert rel(hb.apply_matrix(f, x, transpose=True), O.apply(g, x, transpose=True)) <= 1e-14
    o = hb.hbs_oracle(f)
    assert rel(o.apply_batch(x), O.apply(g, x)) <= 1e-14


def test_deterministic_bitwise():
    c = golden_cases.load("c1_twin")
    f1 = gpu_compress(c["samples"], c["n"], c["leaf"], c["r"])
    f2 = gpu_compress(c["samples"], c["n"], c["leaf"], c["r"])
    assert np.array_equal(f1.root_disc, f2.root_disc)
    for lvl in range(1, f1.tree.depth + 1):
        for a, b in zip(f1.levels[lvl], f2.levels[lvl]):
            assert torch.equal(a, b)


def test_device_resident_samples_match_host_samples():
    c = golden_cases.load("uneven_333")
    dev = [torch.from_numpy(m).cuda() for m in c["samples"]]
    f_host = gpu_compress(c["samples"], c["n"], c["leaf"], c["r"])
    f_dev = gpu_compress(dev, c["n"], c["leaf"], c["r"])
    assert np.array_equal(f_host.root_disc, f_dev.root_disc)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_subtree_partition_on_one_gpu_bitwise(world):
    """The multi-GPU geometry (per-rank subtrees, concatenated level-lg lifts,
    replicated top) run sequentially on one GPU equals the single-GPU sweep
    bit for bit."""
    from paper_2205_02990_b200.distributed import compress_partitioned_on_one_device
    c = golden_cases.load("c1_twin")
    tree = hb.build_tree(c["n"], c["leaf"])
    cfg = hb.CompressionConfig(rank=c["r"], leaf_threshold=c["leaf"])
    f = hb.compress_from_samples(hb.SampleSet(*c["samples"]), tree, cfg)
    blocks, root = compress_partitioned_on_one_device(c["samples"], tree, cfg, world)
    assert np.array_equal(root, f.root_disc)
    for nid, (u, v, d) in blocks.items():
        assert np.array_equal(u, f.u_bases[nid])
        assert np.array_equal(v, f.v_bases[nid])
        assert np.array_equal(d, f.discs[nid])


@pytest.mark.parametrize("world", [2, 8])
def test_subtree_partition_bitwise_config4_shape(world):
    """Same, at the config-4 box shape (128-row boxes, s = 192, r = 64), where
    every (box, side) runs the persistent pipelined probe kernel: a box's bits
    must not depend on how many boxes share its launch (one rank's level of 8
    boxes vs the single-GPU level of 64)."""
    import torch
    from paper_2205_02990_b200 import synthetic
    from paper_2205_02990_b200.distributed import compress_partitioned_on_one_device
    n, leaf, k, s = 1 << 13, 128, 64, 192
    tree = hb.build_tree(n, leaf)
    gen = synthetic.device_generator(tree, k, seed=5, decay=0.9)
    samples = tuple(m.cpu().numpy() for m in synthetic.device_samples(gen, s))
    cfg = hb.CompressionConfig(rank=k, leaf_threshold=leaf)
    f = hb.compress_from_samples(hb.SampleSet(*samples), tree, cfg)
    blocks, root = compress_partitioned_on_one_device(samples, tree, cfg, world)
    assert np.array_equal(root, f.root_disc)
    for nid, (u, v, d) in blocks.items():
        assert np.array_equal(u, f.u_bases[nid])
        assert np.array_equal(v, f.v_bases[nid])
        assert np.array_equal(d, f.discs[nid])


@pytest.mark.parametrize("world", [1, 2, 4])
def test_distributed_sampler_and_compressor_emulated(world):
    """Subtree-partitioned sampler (local up, level-lg exchange, replicated top,
    local down) and compressor, with `world` ranks emulated on one GPU by
    concatenation in place of the NCCL all-gathers: the sampler equals the
    single-GPU telescoping apply of the same operator, and compressing its
    samples reproduces the operator."""
    import torch
    from paper_2205_02990_b200 import synthetic
    from paper_2205_02990_b200.distributed import DistributedOperator, SubtreePartition
    n, leaf, k, r, s = 4096, 32, 12, 20, 60
    tree = hb.build_tree(n, leaf)
    parts = [SubtreePartition(tree, world, g, k) for g in range(world)]
    ops = [synthetic.partitioned_generator(p, k, seed=3) for p in parts]
    # assemble the same operator as one HbsFactorization for the reference apply
    ub, vb, db = {}, {}, {}
    blocks_all = {}
    from paper_2205_02990_b200.distributed import DistributedFactorization, EngineResult
    for p, op in zip(parts, ops):
        for src_blocks, src_geo, first in ((op.local_blocks, op.local_geo, {lv: f for lv, _, f in p.local_specs}),
                                           (op.top_blocks, op.top_geo, {lv: 0 for lv, _, _ in p.top_specs})):
            res = EngineResult(src_blocks, {lv: g.begins_host for lv, g in src_geo.items()}, first, None, None, None)
            blocks_all.update(DistributedFactorization(p, res, None).host_blocks(res))
    for nid, (u, v, d) in blocks_all.items():
        ub[nid], vb[nid], db[nid] = u, v, d
    full = hb.HbsFactorization(tree, k, ub, vb, db, ops[0].root.cpu().numpy())
    x = torch.from_numpy(O.gaussian(n, 5, 0, 4)).cuda()
    for transpose in (False, True):
        want = hb.apply_matrix(full, x, transpose=transpose)
        if world == 1:
            got = ops[0].apply(x, transpose)
        else:
            qh = [op.up_local(x[p.begin:p.end].contiguous(), transpose) for p, op in zip(parts, ops)]
            qtop = torch.cat([q[parts[0].lg] for q in qh])
            ulg = ops[0].top(qtop, transpose)
            got = torch.cat([op.down_local(x[p.begin:p.end].contiguous(), q, ulg[p.rank * k:(p.rank + 1) * k], transpose)
                             for p, op, q in zip(parts, ops, qh)])
        assert float(torch.linalg.norm(got - want) / torch.linalg.norm(want)) <= 1e-14
    # ... and compressing samples of that operator with the same partition
    # (per-rank subtrees, concatenated level-lg lifts, replicated top) gives a
    # factorization that reproduces it (oversampled: r = k + 8, s = 3r)
    from paper_2205_02990_b200.distributed import compress_partitioned_on_one_device
    om, ps = O.gaussian(n, s, 11, 0), O.gaussian(n, s, 11, 1)
    y = hb.apply_matrix(full, om)
    z = hb.apply_matrix(full, ps, transpose=True)
    cfg = hb.CompressionConfig(rank=r, leaf_threshold=leaf)
    blocks, root = compress_partitioned_on_one_device((om, ps, y, z), tree, cfg, world)
    fc = hb.HbsFactorization(tree, r, {i: b[0] for i, b in blocks.items()}, {i: b[1] for i, b in blocks.items()},
                             {i: b[2] for i, b in blocks.items()}, root)
    xs = x.cpu().numpy()
    for transpose in (False, True):
        want = hb.apply_matrix(full, xs, transpose=transpose)
        got = hb.apply_matrix(fc, xs, transpose=transpose)
        assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-10


def test_power_method_relnorm_device():
    """Device power method (linalg.py:108-129 semantics) on a compressed operator:
    the exact-rank twin compresses to ~1e-13, and E == A reports exactly 1."""
    from paper_2205_02990_b200.verify import estimate_rel_err, power_method_relnorm
    c = golden_cases.load("c1_twin")
    f = gpu_compress(c["samples"], c["n"], c["leaf"], c["r"])
    o = hb.dense_oracle(O.dense(c["truth"]))
    assert estimate_rel_err(o, f, iters=20, seed=0) <= 1e-10
    ident = lambda x: x
    assert power_method_relnorm(ident, ident, ident, ident, 64, iters=5) == 1.0


def test_hbsf_round_trip_device(tmp_path):
    from paper_2205_02990_b200.serialize import load_factorization, save_factorization
    c = golden_cases.load("uneven_333")
    f = gpu_compress(c["samples"], c["n"], c["leaf"], c["r"])
    save_factorization(f, tmp_path / "f.hbsf")
    g = load_factorization(tmp_path / "f.hbsf")
    x = c["x"]
    assert np.array_equal(hb.apply_matrix(f, x), hb.apply_matrix(g, x))


def _pinned(a):
    t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
    t.copy_(torch.from_numpy(a))
    return t


@pytest.mark.parametrize("name", ["c1_twin", "uneven_333", "c4_shape_literal"])
def test_pinned_host_pipeline_bitwise(name):
    """Host samples take the overlapped path (subtree-chunked uploads -- pinned
    arrays directly, pageable numpy arrays staged through pinned buffers --,
    per-level downloads on a second stream); results equal the plain level
    sweep on device-resident samples bit for bit, and the dict views come back
    already on the host."""
    c = golden_cases.load(name)
    tree = hb.build_tree(c["n"], c["leaf"])
    cfg = hb.CompressionConfig(rank=c["r"], leaf_threshold=c["leaf"])
    plain = hb.compress_from_samples(hb.SampleSet(*(torch.from_numpy(m).cuda() for m in c["samples"])), tree, cfg)
    keep = [_pinned(m) for m in c["samples"]]
    for piped in (hb.compress_from_samples(hb.SampleSet(*(t.numpy() for t in keep)), tree, cfg),
                  hb.compress_from_samples(hb.SampleSet(*c["samples"]), tree, cfg)):
        assert ("root" in piped._host) and all((lv, "d") in piped._host for lv in range(1, tree.depth + 1))
        assert np.array_equal(plain.root_disc, piped.root_disc)
        for nid in plain.u_bases:
            assert np.array_equal(plain.u_bases[nid], piped.u_bases[nid])
            assert np.array_equal(plain.discs[nid], piped.discs[nid])


def test_pinned_host_pipeline_failure_names_node():
    n, m = 4096, 32
    g = O.baseline_generator(n, m, 16, seed=0)
    om, ps, y, z = O.samples_from(g, 72, 0)
    lo = int(O.level_bounds(n, 7)[7][77])
    om[lo + 1] = om[lo]
    keep = [_pinned(a) for a in (om, ps, y, z)]
    with pytest.raises(hb.IllConditionedProbeError) as exc:
        hb.compress_from_samples(hb.SampleSet(*(t.numpy() for t in keep)), hb.build_tree(n, m),
                                 hb.CompressionConfig(rank=24, leaf_threshold=m))
    assert exc.value.level == 7 and exc.value.node_id == 127 + 77


def _expanded(ub, level_of, L):
    """Bases in original coordinates: leaf U, parent blockdiag(U_a, U_b) U_tau."""
    out = {}
    for level in range(L, 0, -1):
        for j in range(1 << level):
            nid = (1 << level) - 1 + j
            u = ub(level, j)
            if level < L:
                ca, cb = out[(level + 1, 2 * j)], out[(level + 1, 2 * j + 1)]
                r = ca.shape[1]
                u = np.vstack([ca @ u[:r], cb @ u[r:]])
            out[(level, j)] = u
    return out


@pytest.mark.parametrize("n,leaf,r,s", [(512, 32, 8, 48), (512, 32, 16, 48), (1024, 64, 32, 96), (1000, 128, 64, 192),
                                        (1970, 128, 64, 192)])
def test_oversampled_null_space_matches_reference(n, leaf, r, s):
    """The reference keeps the LAST r columns of LAPACK's complete Householder
    Q of Omega_tau^T (linalg.py:52-62), so when nullity s - n_tau > r the
    picked subspace depends on the exact reflectors, not only on
    null(Omega_tau).  A full-rank dense operator makes every off-diagonal
    block full rank, so any other pick would move the bases by O(1).  The
    nested bases, expanded to original coordinates (the parent's U acts on
    its children's bases), must match the reference node for node.  s > 3r:
    LAPACK-signed bases at every level (raw node bases match too); s = 3r:
    parents have nullity exactly r, the CholeskyQR2 bases are used and only
    the expanded bases are comparable.  The s = 192 cases have leaves of 125
    and 123 / 124 rows: the SMSP-split probe kernel runs them zero-padded to
    128 columns (identity reflectors), which must not move the pick."""
    rng = np.random.default_rng(77)
    a = rng.standard_normal((n, n)) / np.sqrt(n)
    om, ps = O.gaussian(n, s, 5, 0), O.gaussian(n, s, 5, 1)
    y, z = a @ om, a.T @ ps
    tree = hb.build_tree(n, leaf)
    f = gpu_compress((om, ps, y, z), n, leaf, r)
    ref = O.compress(om, ps, y, z, O.level_bounds(n, tree.depth), r)
    L = tree.depth
    gu = _expanded(lambda l, j: f.u_bases[(1 << l) - 1 + j], None, L)
    gv = _expanded(lambda l, j: f.v_bases[(1 << l) - 1 + j], None, L)
    ru = _expanded(lambda l, j: ref.U[l][j], None, L)
    rv = _expanded(lambda l, j: ref.V[l][j], None, L)
    for key in ru:
        assert np.linalg.norm(gu[key] @ gu[key].T - ru[key] @ ru[key].T) <= 1e-8, key
        assert np.linalg.norm(gv[key] @ gv[key].T - rv[key] @ rv[key].T) <= 1e-8, key
        if s > 3 * r:
            level, j = key
            u = f.u_bases[(1 << level) - 1 + j]
            assert np.linalg.norm(u @ u.T - ref.U[level][j] @ ref.U[level][j].T) <= 1e-8, key


@pytest.mark.parametrize("k,r,s", [(12, 16, 160), (24, 40, 192)])
def test_leaf_over_128_rows(k, r, s):
    """Leaves of 144 rows exceed the 128 TMEM lanes.  s = 160: the fused
    kernel keeps Y in L2 there (group Y streams it per panel) and in TMEM at
    the parents; s = 192: Omega^T no longer fits in shared memory and the
    separate QR / apply-Q kernels run.  All must reproduce the oracle."""
    n, leaf = 2304, 144
    truth = O.baseline_generator(n, leaf, k, seed=9)
    om, ps, y, z = O.samples_from(truth, s, 9)
    tree = hb.build_tree(n, leaf)
    assert tree.level_sizes(tree.depth).max() == 144
    f = gpu_compress((om, ps, y, z), n, leaf, r)
    ref = O.compress(om, ps, y, z, O.level_bounds(n, tree.depth), r)
    x = O.gaussian(n, 4, 0, 4)
    got, want = hb.apply_matrix(f, x), O.apply(ref, x)
    assert rel(got, want) <= 1e-10
    assert rel(got, O.apply(truth, x)) <= 1e-10


def test_chunked_levels_bitwise():
    """A workspace cap splits levels into box chunks that reuse one scratch
    (config 5's leaf level on one GPU); the result is bitwise the unchunked
    sweep."""
    c = golden_cases.load("c2_shape_twin")
    tree = hb.build_tree(c["n"], c["leaf"])
    quad = [torch.from_numpy(m).cuda() for m in c["samples"]]
    full = hb.CompressPlan(tree, c["s"], c["r"])
    full.run(*quad)
    small = hb.CompressPlan(tree, c["s"], c["r"], max_workspace_bytes=1 << 20)
    assert small.chunks, "the 1 MB cap must chunk the deep levels"
    small.run(*quad)
    torch.cuda.synchronize()
    assert torch.equal(full.root, small.root)
    for lvl in range(1, tree.depth + 1):
        for a, b in zip(full.levels[lvl], small.levels[lvl]):
            assert torch.equal(a, b)
    assert torch.equal(full.status, small.status)


def test_graph_replay_equals_stream_launches():
    """CompressPlan.run_graph (one CUDA-graph replay per sweep) leaves the same
    bits as the plain launch sequence, for repeated replays."""
    import torch
    from paper_2205_02990_b200 import synthetic
    n, leaf, k, s = 1 << 12, 128, 64, 192
    tree = hb.build_tree(n, leaf)
    gen = synthetic.device_generator(tree, k, seed=2, decay=0.9)
    quad = synthetic.device_samples(gen, s)
    plan = hb.CompressPlan(tree, s, k)
    plan.run(*quad)
    torch.cuda.synchronize()
    want = [[m.clone() for m in plan.levels[lv]] for lv in sorted(plan.levels)] + [[plan.root.clone()]]
    for m in (m for lv in plan.levels.values() for m in lv):
        m.zero_()
    plan.root.zero_()
    for _ in range(2):
        nk = plan.run_graph(*quad)
    torch.cuda.synchronize()
    plan.raise_for_status()
    assert nk > 0
    got = [[m for m in plan.levels[lv]] for lv in sorted(plan.levels)] + [[plan.root]]
    for a, b in zip(want, got):
        for x, y in zip(a, b):
            assert torch.equal(x, y)


def test_sigma_screen_window_is_one_sided():
    """The documented difference of the ill-conditioning screen (DESIGN.md
    section 6): the reference tests sigma_min / sigma_max of the probe block
    (linalg.py:73-78), the GPU path min|R_ii| / max|R_ii| of its QR factor,
    which is an upper bound of that ratio -- so it never raises where the
    reference would not.  A Kahan block (|R_ii| = s^i, far smaller sigma_min)
    sits in the window between the two: with a tolerance inside the window the
    oracle rejects the block and the GPU stage accepts it; with the tolerance
    above the diag(R) ratio both reject it."""
    rows, cols = 32, 48
    c, sn = 0.5, np.sqrt(0.75)
    kahan = np.diag(sn ** np.arange(rows)) @ (np.eye(rows) - c * np.triu(np.ones((rows, rows)), 1))
    m = np.zeros((rows, cols))
    m[:, :rows] = kahan.T                                  # M^T = [K; 0]: R = K up to signs
    b = O.gaussian(8, cols, 2, 0)
    sv = np.linalg.svd(kahan, compute_uv=False)
    diag_ratio, sigma_ratio = sn ** (rows - 1), sv[-1] / sv[0]
    assert sigma_ratio < 1e-3 * diag_ratio                 # a real window
    tol = float(np.sqrt(diag_ratio * sigma_ratio))         # sigma ratio < tol < diag(R) ratio
    x, ratio = O.right_solve(b, m, tol)
    assert x is None and ratio < tol                       # the reference's test rejects the block
    got = hb.lstsq_right(b, m, tol)                        # inside the window: accepted (documented)
    assert np.all(np.isfinite(np.asarray(got)))
    with pytest.raises(hb.IllConditionedProbeError):
        hb.lstsq_right(b, m, 2.0 * diag_ratio)
    x, _ = O.right_solve(b, m, 2.0 * diag_ratio)
    assert x is None


def test_level_hint_does_not_change_results():
    """hbs_level_hint only lets the library skip launches that would find no
    box: a sweep whose levels are hinted as uniform (the default) and one with
    the hint withheld (min_rows = 0: unknown) leave the same bits, and the
    hinted sweep performs fewer launches."""
    import torch
    from paper_2205_02990_b200 import synthetic
    n, leaf, k, s = 1 << 12, 128, 64, 192
    tree = hb.build_tree(n, leaf)
    gen = synthetic.device_generator(tree, k, seed=4, decay=0.9)
    quad = synthetic.device_samples(gen, s)
    lib = hb._native.lib()
    outs, launches = [], []
    for hinted in (True, False):
        plan = hb.CompressPlan(tree, s, k)
        if not hinted:
            for g in plan.geometry.values():
                g.min_rows = 0
        n0 = lib.hbs_launch_counter()
        plan.run(*quad)
        torch.cuda.synchronize()
        plan.raise_for_status()
        launches.append(lib.hbs_launch_counter() - n0)
        outs.append([m.clone() for lv in sorted(plan.levels) for m in plan.levels[lv]] + [plan.root.clone()])
    assert launches[0] < launches[1]
    for a, b in zip(*outs):
        assert torch.equal(a, b)
