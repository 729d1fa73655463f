"""Eq. 4 throughput model and the Sec. 7.2 alternatives
(P:1371-1388): closed forms and the paper's own worked numbers."""
import math

import pytest

from paper_2007_13005_b200 import throughput as tp


def test_single_dnn_min():
    # one DNN, alpha = 1: T_hat = min(T_pre, T_exec)
    assert tp.eq4_min(5900.0, [4200.0]) == 4200.0
    assert tp.eq4_min(3000.0, [4200.0]) == 3000.0


def test_paper_sec72_numbers():
    # preprocessing 5.9k, DNN execution 4.2k, pipelined 3.6k im/s;
    # Smol's min() model predicts 4.2k (16% above measured, "only incurs a 16%
    # overhead"), Tahoma's model (sum) predicts ~2.5k ("a 30% error").
    e = tp.model_errors(3600.0, 5900.0, [4200.0])
    assert e["min"]["predicted"] == 4200.0
    assert e["min"]["rel_error"] == pytest.approx(0.1667, abs=1e-3)
    assert e["sum"]["predicted"] == pytest.approx(1 / (1 / 5900 + 1 / 4200))
    assert e["sum"]["predicted"] == pytest.approx(2453.5, abs=1.0)          # "2.5k"
    assert e["sum"]["rel_error"] == pytest.approx(0.318, abs=0.01)          # "a 30% error"


def test_cascade_harmonic():
    # two-stage cascade: every input runs model 1, a fraction 0.1 runs model 2
    t1, t2 = 10000.0, 1000.0
    d = tp.dnn_stage([t1, t2], [1.0, 0.1])
    assert d == pytest.approx(1.0 / (1 / t1 + 0.1 / t2))
    assert d == pytest.approx(5000.0)
    assert tp.eq4_min(1e9, [t1, t2], [1.0, 0.1]) == pytest.approx(5000.0)
    # alpha_j = 0 removes a stage
    assert tp.dnn_stage([t1, t2], [1.0, 0.0]) == pytest.approx(t1)


def test_sum_le_min_and_limits():
    for pre, ex in ((1e6, 3e4), (3e4, 1e6), (5e4, 5e4)):
        assert tp.sum_model(pre, [ex]) <= tp.eq4_min(pre, [ex])
    # equal stages: sum model halves the rate, min keeps it
    assert tp.sum_model(5e4, [5e4]) == pytest.approx(2.5e4)
    # preprocessing infinitely fast: every model reduces to DNN execution
    assert tp.sum_model(1e300, [3e4]) == pytest.approx(3e4)
    assert math.isclose(tp.exec_only(1.0, [3e4]), 3e4)


def test_validation():
    with pytest.raises(ValueError):
        tp.dnn_stage([], [])
    with pytest.raises(ValueError):
        tp.dnn_stage([1.0], [1.5])
    with pytest.raises(ValueError):
        tp.eq4_min(0.0, [1.0])
