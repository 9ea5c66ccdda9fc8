"""Assembly flop models: closed-form check on a hand-made leaf table."""
import numpy as np

from paper_1706_09384_b200.flops import PAIR_FLOPS, survey_flops


def test_survey_flops_closed_form():
    # one dense leaf (ignored by the factor terms) and two admissible leaves
    table = np.array([[0, 0, 10, 0, 10], [1, 0, 10, 20, 40], [1, 20, 40, 0, 10]], np.int64)
    steps = np.array([0, 4, 2])
    kb = np.array([0, 12, 6])
    ka = np.array([0, 7, 3])
    f, parts = survey_flops(table, steps, kb, ka, 3, "U", 1000)
    d = 3
    exp = {
        "pairs": PAIR_FLOPS["U"] * 1000,
        "residual": 8 * (d / 2) * 30 * (144 + 36),
        "qr": 8 * 2 * d * 30 * (144 + 36),
        "form": 8 * d * 30 * (12 * 7 + 6 * 3),
        "svd": 8 * 22 * (12 ** 3 + 6 ** 3),
    }
    for k, v in exp.items():
        assert abs(parts[k] - v) <= 1e-9 * max(v, 1), k
    assert abs(f - sum(exp.values())) <= 1e-9 * f
