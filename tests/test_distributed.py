"""Multi-process (gloo, CPU) tests of the subtree-partitioned driver
(paper_2205_02990_b200/distributed.py).

The per-level work runs through a CPU engine built on the oracle, so these
tests exercise exactly the host logic the GPU path uses: row partition,
per-level geometry, the single all-gather of lifted halves, replicated top
levels, failure agreement, and the gathered result -- which must equal the
single-process oracle bit for bit (partitioning changes no per-node
arithmetic)."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import hbs_oracle as O
from paper_2205_02990_b200 import CompressionConfig, IllConditionedProbeError, build_tree
from paper_2205_02990_b200.distributed import EngineResult, SubtreePartition, compress_distributed


class OracleEngine:
    """CPU engine for tests: the oracle's per-node restatement, packed like CompressPlan."""

    def as_tensor(self, a):
        return a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))

    def run(self, tree, specs, quad, s, r, tol, with_root):
        q = [m.numpy() for m in quad]
        levels, begins, first = {}, {}, {}
        for level, b, f in specs:
            us, vs, ds = [], [], []
            lifted = [np.empty(((b.size - 1) * r, s)) for _ in range(4)]
            for j in range(b.size - 1):
                blk = [m[b[j] - b[0]:b[j + 1] - b[0]] for m in q]
                try:
                    u, v, d = O.node_step(*blk, r, tol)
                except O.ProbeRankError:
                    return EngineResult(levels, begins, first, None, None, (level, (1 << level) - 1 + f + j))
                us.append(u), vs.append(v), ds.append(d.ravel())
                for dst, part in zip(lifted, O.lift_rows(u, v, d, *blk)):
                    dst[j * r:(j + 1) * r] = part
            levels[level] = tuple(torch.from_numpy(np.concatenate(x)) for x in (us, vs, ds))
            begins[level], first[level] = b, f
            q = lifted
        root, fail = None, None
        if with_root:
            root, _ = O.right_solve(q[2], q[0], tol)
            if root is None:
                fail = (0, 0)
        return EngineResult(levels, begins, first, tuple(torch.from_numpy(m) for m in q), root, fail)


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


CASE = dict(n=2048, leaf=32, k=16, r=24, s=72)


def _problem(n, leaf, k, r, s, break_leaf=None):
    g = O.baseline_generator(n, leaf, k, seed=0)
    om, ps, y, z = O.samples_from(g, s, 0)
    if break_leaf is not None:
        lo = int(O.level_bounds(n, g.depth)[g.depth][break_leaf])
        om[lo + 1] = om[lo]
    return g, (om, ps, y, z)


def _worker(rank, world, port, outdir, break_leaf):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        c = CASE
        tree = build_tree(c["n"], c["leaf"])
        _, samples = _problem(c["n"], c["leaf"], c["k"], c["r"], c["s"], break_leaf)
        part = SubtreePartition(tree, world, rank, c["r"])
        local = [m[part.begin:part.end] for m in samples]
        try:
            f = compress_distributed(local, tree, CompressionConfig(rank=c["r"], leaf_threshold=c["leaf"]),
                                     engine=OracleEngine())
            blocks, root = f.gather()
            np.savez(os.path.join(outdir, f"rank{rank}.npz"), root=root,
                     ids=np.array(sorted(blocks)),
                     **{f"u{i}": blocks[i][0] for i in blocks}, **{f"v{i}": blocks[i][1] for i in blocks},
                     **{f"d{i}": blocks[i][2] for i in blocks})
        except IllConditionedProbeError as exc:
            np.savez(os.path.join(outdir, f"rank{rank}.npz"), err=np.array([exc.level, exc.node_id]))
    finally:
        dist.destroy_process_group()


def _run(world, break_leaf=None):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d, break_leaf), nprocs=world, join=True)
        return [dict(np.load(os.path.join(d, f"rank{i}.npz"))) for i in range(world)]


@pytest.mark.parametrize("world", [2, 4])
def test_subtree_partition_bitwise_equals_single_process(world):
    c = CASE
    _, (om, ps, y, z) = _problem(c["n"], c["leaf"], c["k"], c["r"], c["s"])
    tree = build_tree(c["n"], c["leaf"])
    ref = O.compress(om, ps, y, z, O.level_bounds(c["n"], tree.depth), c["r"])
    outs = _run(world)
    for out in outs:   # every rank holds the same gathered factorization
        assert np.array_equal(out["root"], ref.root)
        assert len(out["ids"]) == (1 << (tree.depth + 1)) - 2
        for nid in out["ids"]:
            u, v, d = ref.node_blocks(int(nid))
            assert np.array_equal(out[f"u{nid}"], u)
            assert np.array_equal(out[f"v{nid}"], v)
            assert np.array_equal(out[f"d{nid}"], d)


def test_failure_is_agreed_across_ranks():
    # duplicated probe rows in leaf 40 (owned by rank 1 of 2): every rank
    # raises for the same node / level as the single-process oracle.
    c = CASE
    _, (om, ps, y, z) = _problem(c["n"], c["leaf"], c["k"], c["r"], c["s"], break_leaf=40)
    tree = build_tree(c["n"], c["leaf"])
    with pytest.raises(O.ProbeRankError) as exc:
        O.compress(om, ps, y, z, O.level_bounds(c["n"], tree.depth), c["r"])
    want = [exc.value.level, (1 << exc.value.level) - 1 + exc.value.box]
    outs = _run(2, break_leaf=40)
    for out in outs:
        assert list(out["err"]) == want


def test_partition_geometry():
    tree = build_tree(333, 24)
    for world in (1, 2, 4):
        spans = []
        for rank in range(world):
            p = SubtreePartition(tree, world, rank, 8)
            spans.append((p.begin, p.end))
            leaf = p.local_specs[0]
            assert leaf[0] == tree.depth and leaf[1][0] == 0 and leaf[1][-1] == p.rows
            assert [s[0] for s in p.local_specs] == list(range(tree.depth, max(p.lg, 1) - 1, -1))
        assert spans[0][0] == 0 and spans[-1][1] == 333
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
