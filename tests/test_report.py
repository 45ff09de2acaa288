"""Table-1 arithmetic (paper_1811_12174_b200/report.py) pinned to the paper's own printed
table: from the epoch times of PAPER.md Table 1 the report must reproduce the
printed speedups 1.97x / 1.93x / 2.01x / 1.83x and scalings 98.5 / 95.0 / 95.4 / 87.3 %, at
the paper's printed precision.  Golden values: tests/golden/table1.json (cited).  CPU only."""
import json
import os

import pytest

from paper_1811_12174_b200 import report

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "table1.json")


def test_reproduces_paper_table1():
    g = json.load(open(GOLDEN))
    times = {int(r["gpus"]): r["seconds"] for r in g["rows"]}
    rows = report.table1_rows(times)
    for r, want in zip(rows, g["rows"]):
        assert r["gpus"] == want["gpus"]
        if want["speedup_prev"] is None:
            assert r["speedup_prev"] is None and r["scaling_pct"] is None
            continue
        assert f"{r['speedup_prev']:.2f}" == f"{want['speedup_prev']:.2f}", r
        assert f"{r['scaling_pct']:.1f}" == f"{want['scaling_pct']:.1f}", r
    txt = report.format_rows(rows)
    assert "1.97x" in txt and "87.3" in txt


def test_weak_scaling_step_times_map_to_epochs():
    """Perfect weak scaling (equal step time at every N) is 100 % scaling and an N/prev
    speedup; a 2x slower step at N = 2 is 50 %."""
    eps = {n: report.epoch_seconds(100.0, n, 64, 1_281_167) for n in (1, 2, 4, 8)}
    rows = report.table1_rows(eps)
    assert all(abs(r["scaling_pct"] - 100.0) < 1e-9 for r in rows[1:])
    assert all(abs(r["speedup_prev"] - 2.0) < 1e-9 for r in rows[1:])
    rows = report.table1_rows({1: report.epoch_seconds(100.0, 1, 64, 6400),
                               2: report.epoch_seconds(200.0, 2, 64, 6400)})
    assert abs(rows[1]["scaling_pct"] - 50.0) < 1e-9


def test_needs_one_gpu_row():
    with pytest.raises(ValueError):
        report.table1_rows({2: 1.0, 4: 0.5})


def test_unet3d_model_matches_config3_parameter_count():
    """scripts/train_ddp.py's 3D U-Net is the network whose gradient set BASELINE config 3
    all-reduces: 19,075,523 fp32 parameters in 64 tensors (
    synthetic_inputs.UNET3D_PARAMS)."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
    import synthetic_inputs as si
    import train_ddp
    m = train_ddp.UNet3D()
    ps = list(m.parameters())
    assert sum(p.numel() for p in ps) == si.UNET3D_PARAMS == 19_075_523
    assert len(ps) == 64
