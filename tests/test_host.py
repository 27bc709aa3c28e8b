"""CPU tests of the host-side logic: tree, configuration checks, madd
accounting, and the C-ABI library surface (loads and exports every symbol
declared in include/hbs_b200.h -- no compute calls without a GPU)."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2205_02990_b200 import CompressionConfig, ConfigurationError, DimensionError, build_tree, flops
from paper_2205_02990_b200 import _native
from paper_2205_02990_b200.compress import _charge_madds, _check_configuration

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("n,m", [(4096, 32), (333, 24), (40, 20), (2 ** 15, 80), (21, 4), (1000, 7), (17, 2), (3, 2)])
def test_tree_matches_reference(reference_hbs, n, m):
    a, b = reference_hbs.build_tree(n, m), build_tree(n, m)
    assert a.depth == b.depth
    assert [(x.id, x.level, x.begin, x.end, x.parent, x.children) for x in a.nodes] == \
           [(x.id, x.level, x.begin, x.end, x.parent, x.children) for x in b.nodes]
    for lv in range(b.depth + 1):
        assert [nd.begin for nd in b.nodes_at_level(lv)] == list(b.level_begin(lv)[:-1])


def test_tree_errors():
    for n, m in ((1, 2), (10, 1), (8, 8)):
        with pytest.raises(ConfigurationError):
            build_tree(n, m)


def test_config_validation_matches_reference():
    # compress.py:49-70 (test_compress.py:395-402)
    tree = build_tree(64, 8)
    with pytest.raises(ConfigurationError):
        CompressionConfig(rank=9, leaf_threshold=8).validate_for(tree)
    with pytest.raises(ConfigurationError):
        CompressionConfig(rank=2, leaf_threshold=8, probes=9).validate_for(tree)
    with pytest.raises(ConfigurationError):
        CompressionConfig(rank=0, leaf_threshold=8).validate_for(tree)
    assert CompressionConfig(rank=3, leaf_threshold=8).validate_for(tree) == 11


def test_shape_errors_before_launch():
    tree = build_tree(96, 12)
    with pytest.raises(ConfigurationError):
        _check_configuration(tree, 14, 5)          # nullity 14 - 12 < 5 at the leaves
    with pytest.raises(DimensionError):
        _check_configuration(tree, 60, 13)         # rank wider than a 12-row leaf


def test_madd_accounting_equals_reference(reference_hbs):
    """The drop-in charges exactly the reference's per-node madd formulas
    (compress.py:170,173,194,213; linalg.py:42,60,81,89)."""
    hbs = reference_hbs
    from oracle import hbs_oracle as O
    for n, m, r in ((512, 10, 5), (333, 24, 8), (1024, 32, 16)):
        tree = build_tree(n, m)
        s = CompressionConfig(rank=r, leaf_threshold=m).validate_for(tree)
        g = O.baseline_generator(n, m, max(1, r - 5), seed=1)
        om, ps, y, z = O.samples_from(g, s, 0)
        with hbs.flops.count_madds() as ref_counter:
            hbs.compress_from_samples(hbs.SampleSet(om, ps, y, z), hbs.build_tree(n, m),
                                      hbs.CompressionConfig(rank=r, leaf_threshold=m))
        with flops.count_madds() as mine:
            _charge_madds(tree, s, r)
        assert mine.madds == ref_counter.madds


def test_madds_scale_linearly():
    """test_compress.py:337-351 / test_acceptance.py:146-167 on the charged counts."""
    counts = []
    for n in (2048, 4096, 16384, 32768):
        tree = build_tree(n, 10)
        with flops.count_madds() as c:
            _charge_madds(tree, 15, 5)
        counts.append(c.madds / n)
    assert max(counts) / min(counts) <= 1.1


def test_library_exports_every_header_symbol():
    header = open(os.path.join(ROOT, "include", "hbs_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:const\s+char\*|int|void|unsigned long long)\s+(hbs_\w+)\s*\(", header, re.M))
    assert len(declared) >= 15
    assert declared == set(_native.SIGNATURES)
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built")
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert b"sm_100a" in _native.lib().hbs_b200_version()


def test_no_cpu_fallback_without_library(monkeypatch, tmp_path):
    monkeypatch.setattr(_native, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(_native, "_lib", None)
    with pytest.raises(_native.NativeError):
        _native.lib()
