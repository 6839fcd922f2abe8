"""CPU tests of host-side logic that needs no GPU: the quant lab's report/CSV plumbing
and seeding, and the synthetic OutlierSpec generator's contract."""
import csv
import io

import pytest
import torch

import synthetic


def test_outlier_spec_generator_contract():
    a = synthetic.outlier_matrix(64, 1024, 1, base_std=2.0, outlier_rate=1e-3, outlier_scale=100.0)
    b = synthetic.outlier_matrix(64, 1024, 1, base_std=2.0, outlier_rate=1e-3, outlier_scale=100.0)
    assert torch.equal(a, b)                                    # deterministic per seed
    assert a.abs().max().item() == pytest.approx(200.0)         # outliers at +-scale * base_std
    frac = (a.abs() == 200.0).float().mean().item()
    assert 2e-4 < frac < 3e-3                                   # ~ outlier_rate
    z = synthetic.outlier_matrix(64, 1024, 1, outlier_rate=0.0)
    assert z.abs().max().item() < 6.5                           # pure Gaussian
    with pytest.raises(ValueError):
        synthetic.outlier_matrix(4, 16, 1, outlier_rate=1.5)
    with pytest.raises(ValueError):
        synthetic.outlier_matrix(4, 16, 1, outlier_scale=0.5)


def test_quant_lab_report_csv_and_seeds():
    from paper_2412_08832_b200 import quant_lab
    spec = quant_lab.OutlierSpec(rows=4, cols=16, seed=7)
    assert quant_lab.trial_seed(spec, 0) != quant_lab.trial_seed(spec, 1)
    assert quant_lab.trial_seed(spec, 3) == quant_lab.trial_seed(quant_lab.OutlierSpec(rows=4, cols=16, seed=7), 3)
    rep = {"per_trial": [{"trial": 0, "mse_plain": 2.0, "mse_rotated": 1.0, "max_abs_plain": 9.0, "max_abs_rotated": 3.0},
                         {"trial": 1, "mse_plain": 1.0, "mse_rotated": 4.0, "max_abs_plain": 8.0, "max_abs_rotated": 2.0}],
           "aggregate": {"mse_plain": 1.5, "mse_rotated": 2.5, "win_rate": 0.5, "max_abs_plain": 9.0,
                         "max_abs_rotated": 3.0}}
    buf = io.StringIO()
    quant_lab.write_csv(rep, buf)
    rows = list(csv.reader(io.StringIO(buf.getvalue())))
    assert rows[0] == ["trial", "mse_plain", "mse_rotated", "max_abs_plain", "max_abs_rotated", "win_rate"]
    assert len(rows) == 4 and rows[-1][0] == "aggregate" and float(rows[-1][-1]) == 0.5
