"""The test-only near-exact sketch (tests/accurate_sketch.py) against exact
rational arithmetic on a few entries (CPU torch: the slice products are exact
under any fp64 GEMM)."""
from fractions import Fraction

import numpy as np
import torch

from accurate_sketch import accurate_sketch


def test_accurate_sketch_is_correctly_rounded_ish():
    rng = np.random.default_rng(3)
    K = 3000
    om = rng.standard_normal((5, K))
    mm = rng.standard_normal((K, 4)) * np.exp(rng.standard_normal((K, 1)) * 3)  # wide dynamic range
    y = accurate_sketch(torch.from_numpy(om), torch.from_numpy(mm)).numpy()
    for i in range(5):
        for j in range(4):
            exact = sum(Fraction(float(om[i, l])) * Fraction(float(mm[l, j])) for l in range(K))
            ex = float(exact)
            assert abs(y[i, j] - ex) <= 4 * np.spacing(abs(ex)), (i, j, y[i, j], ex)
