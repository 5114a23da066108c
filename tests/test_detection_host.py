"""f4: host-side H0/H1 bookkeeping of the PCE detector (P:259 threshold 60,
strict S:310).  Pure host logic over PCE scores; no GPU needed."""
import numpy as np
import pytest

import paper_1909_04573_b200 as prnu


def test_detection_rates_strict_threshold():
    M = np.array([[100.0, 60.0, 3.0],
                  [60.0, 61.0, -5.0],
                  [0.0, 80.0, 60.0]])
    r = prnu.detection_rates(M)
    assert r["n_h1"] == 3 and r["n_h0"] == 6
    assert r["tpr"] == pytest.approx(2 / 3)        # 60.0 on the diagonal is not a match (strict >)
    assert r["fpr"] == pytest.approx(1 / 6)        # only the 80.0 off-diagonal entry
    with pytest.raises(ValueError):
        prnu.detection_rates(np.zeros((2, 3)))


def test_roc_extremes_and_auc():
    fpr, tpr, auc = prnu.roc([5, 6, 7], [1, 2, 3])      # perfect separation
    assert auc == pytest.approx(1.0) and fpr[-1] == 1.0 and tpr[-1] == 1.0
    fpr, tpr, auc = prnu.roc([1, 2, 3], [5, 6, 7])      # perfectly wrong
    assert auc == pytest.approx(0.0)
    rng = np.random.default_rng(0)                       # identical distributions -> AUC ~ 1/2
    _, _, auc = prnu.roc(rng.normal(size=4000), rng.normal(size=4000))
    assert abs(auc - 0.5) < 0.03
    assert np.all(np.diff(fpr) >= 0) and np.all(np.diff(tpr) >= 0)
