"""`.hbsf` I/O (CPU tests): bit-exact round trips from the packed layout and
byte compatibility with the reference's format (serialize.py:1-91)."""
import numpy as np
import pytest

from oracle import hbs_oracle as O
from paper_2205_02990_b200 import FormatError, HbsFactorization, build_tree
from paper_2205_02990_b200.serialize import load_factorization, save_factorization


def _fact(n, leaf, k, seed, device="cpu"):
    g = O.baseline_generator(n, leaf, k, seed=seed)
    tree = build_tree(n, leaf)
    ub, vb, db = {}, {}, {}
    for lvl in range(1, tree.depth + 1):
        for j, nd in enumerate(tree.nodes_at_level(lvl)):
            ub[nd.id], vb[nd.id], db[nd.id] = g.U[lvl][j], g.V[lvl][j], g.D[lvl][j]
    return HbsFactorization(tree, k, ub, vb, db, g.root, device=device), (ub, vb, db, g.root)


def _same(f, g):
    assert f.n == g.n and f.rank == g.rank and f.tree.depth == g.tree.depth
    assert np.array_equal(f.root_disc, g.root_disc)
    for nid in f.u_bases:
        assert np.array_equal(f.u_bases[nid], g.u_bases[nid])
        assert np.array_equal(f.v_bases[nid], g.v_bases[nid])
        assert np.array_equal(f.discs[nid], g.discs[nid])


@pytest.mark.parametrize("n,leaf,k", [(100, 12, 4), (101, 12, 4), (333, 24, 4), (40, 20, 3)])
def test_bitwise_round_trip(tmp_path, n, leaf, k):
    f, _ = _fact(n, leaf, k, seed=1)
    p = tmp_path / "f.hbsf"
    save_factorization(f, p)
    _same(f, load_factorization(p, device="cpu"))


def test_files_interchange_with_reference(tmp_path, reference_hbs):
    hbs = reference_hbs
    f, (ub, vb, db, root) = _fact(101, 12, 4, seed=2)
    ref = hbs.HbsFactorization(hbs.build_tree(101, 12), 4, ub, vb, db, root)
    mine, theirs = tmp_path / "mine.hbsf", tmp_path / "ref.hbsf"
    save_factorization(f, mine)
    hbs.save_factorization(ref, theirs)
    assert mine.read_bytes() == theirs.read_bytes()
    _same(load_factorization(theirs, device="cpu"), f)
    g = hbs.load_factorization(mine)
    for nid in ub:
        assert np.array_equal(g.u_bases[nid], ub[nid]) and np.array_equal(g.discs[nid], db[nid])


def test_format_errors(tmp_path):
    f, _ = _fact(64, 8, 3, seed=3)
    p = tmp_path / "f.hbsf"
    save_factorization(f, p)
    raw = p.read_bytes()
    (tmp_path / "magic.hbsf").write_bytes(b"XXXX" + raw[4:])
    (tmp_path / "ver.hbsf").write_bytes(raw[:4] + (7).to_bytes(4, "little") + raw[8:])
    (tmp_path / "trunc.hbsf").write_bytes(raw[:-9])
    (tmp_path / "trail.hbsf").write_bytes(raw + b"\0")
    (tmp_path / "short.hbsf").write_bytes(raw[:10])
    for name in ("magic", "ver", "trunc", "trail", "short"):
        with pytest.raises(FormatError):
            load_factorization(tmp_path / f"{name}.hbsf", device="cpu")
