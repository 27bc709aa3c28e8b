"""Run records / CLI (mirrors the reference's bench.py / cli.py)."""
import json

import numpy as np
import pytest
import torch

from paper_2205_02990_b200 import cli, runs


def test_record_csv_schema_matches_reference():
    rec = runs.RunRecord("synthetic", 4096, 16, 32, 48, 0, 0.1, 0.2, 0.3, 1e-12, 40.5, 48, 48)
    # the CSV schema is the reference's 13 columns (bench.py:31); the GPU
    # fields (device, n_gpus, rows_per_s, roofline_frac, generator) are JSON-only
    assert runs.CSV_HEADER.split(",") == [f.name for f in rec.__dataclass_fields__.values()][:13]
    assert rec.csv_row().split(",")[0] == "synthetic" and len(rec.csv_row().split(",")) == 13
    row = json.loads(rec.json_row())
    assert row["matvecs_at"] == 48
    assert {"device", "n_gpus", "rows_per_s", "roofline_frac", "generator"} <= set(row)


def test_cli_configuration_error_exit_code(capsys):
    # rank above the leaf size: rejected before any device work (exit 2)
    assert cli.main(["compress", "--problem", "synthetic", "--n", "256", "--rank", "40", "--leaf", "32"]) == 2
    assert "configuration error" in capsys.readouterr().err


def test_unknown_problem_rejected():
    with pytest.raises(SystemExit):
        cli.main(["compress", "--problem", "bie-dl", "--n", "256", "--rank", "8", "--leaf", "32"])


@pytest.mark.gpu
def test_run_once_synthetic_on_gpu(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = runs.CompressionConfig(rank=16, leaf_threshold=32, seed=3)
    rec, f = runs.run_with_factorization("synthetic", 4096, cfg)
    assert rec.s == 48 and rec.matvecs_a == 48 and rec.matvecs_at == 48
    assert rec.rel_err < 1e-10 and rec.t_compress > 0 and rec.floats_per_dof > 0
    out = tmp_path / "sweep.csv"
    recs = runs.sweep("synthetic", [1024, 2048], cfg, out)
    lines = out.read_text().strip().splitlines()
    assert lines[0] == runs.CSV_HEADER and len(lines) == 3 and all(r.rel_err < 1e-10 for r in recs)
    hbsf = tmp_path / "f.hbsf"
    assert cli.main(["compress", "--problem", "synthetic", "--n", "4096", "--rank", "16", "--leaf", "32",
                     "--seed", "3", "--json", "--save", str(hbsf)]) == 0
    assert cli.main(["verify", "--load", str(hbsf), "--problem", "synthetic", "--n", "4096", "--rank", "16",
                     "--leaf", "32", "--seed", "3"]) == 0


@pytest.mark.gpu
def test_run_once_log_kernel_on_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rec = runs.run_once("log-kernel", 2048, runs.CompressionConfig(rank=40, leaf_threshold=64, seed=0))
    assert np.isfinite(rec.rel_err) and rec.rel_err < 1e-6
