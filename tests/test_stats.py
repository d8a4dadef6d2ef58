"""Host statistics of the paper's experiments (paper_cs_0605069_b200/stats.py) on
hand-made inputs whose answers are worked out in the comments.  CPU only."""
import math

import numpy as np

from paper_cs_0605069_b200 import stats


def test_paired_ratio_worked_example():
    # frames: (PUS, SUS) = (10, 5), (20, 11), (-1, 7), (8, -1), (30, 15)
    tp = [10, 20, -1, 8, 30]
    ts = [5, 11, 7, -1, 15]
    r = stats.paired_ratio(tp, ts)
    assert r["paired"] == 3 and r["nonconv_pus"] == 1 and r["nonconv_sus"] == 1
    assert math.isclose(r["mean_t_sus"], 31 / 3) and math.isclose(r["mean_t_pus"], 20.0)
    assert math.isclose(r["ratio_of_means"], 31 / 60)
    q = np.array([0.5, 0.55, 0.5])
    assert math.isclose(r["mean_ratio"], q.mean()) and math.isclose(r["std_ratio"], q.std())


def test_paired_ratio_nothing_paired():
    r = stats.paired_ratio([-1, -1], [3, -1])
    assert r["paired"] == 0 and "ratio_of_means" not in r


def test_delta_p_curve_worked_example():
    # nbits = 10.  PUS frame: correct bits 2, 4, 6, 8, 10 (converges at t = 4);
    # SUS frame: 2, 6, 10, 10, 10 (converges at t = 2; the frozen tail is excluded).
    tp = np.array([[2, 4, 6, 8, 10]])
    ts = np.array([[2, 6, 10, 10, 10]])
    res = stats.delta_p_curve(tp, [4], ts, [2], nbits=10, bins=[0, 50, 100])
    # PUS transitions: P=20 -> +20, 40 -> +20 (bin 0); 60 -> +20, 80 -> +20 (bin 1)
    # SUS transitions: P=20 -> +40 (bin 0); 60 -> +40 (bin 1)
    assert res["count_pus"] == [2, 2] and res["count_sus"] == [1, 1]
    assert res["mean_dP_pus"] == [20.0, 20.0] and res["mean_dP_sus"] == [40.0, 40.0]
    assert res["ratio_pus_over_sus"] == [0.5, 0.5]


def test_delta_p_curve_nonconverged_uses_every_transition():
    # never converges (-1): all 3 transitions count, including a loss of correct bits
    tr = np.array([[5, 7, 6, 9]])
    res = stats.delta_p_curve(tr, [-1], tr, [-1], nbits=10, bins=[0, 100])
    assert res["count_pus"] == [3]
    assert math.isclose(res["mean_dP_pus"][0], (20 - 10 + 30) / 3)
    assert res["ratio_pus_over_sus"] == [1.0]
