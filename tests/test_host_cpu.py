"""CPU: host-side helpers -- config constructions and bench bookkeeping."""
import numpy as np

from paper_2105_07076_b200.configs import CONFIGS, make_np, spectrum


def test_configs_follow_baseline():
    c = CONFIGS
    assert (c["cfg1"].m, c["cfg1"].n, c["cfg1"].k, c["cfg1"].p) == (500, 1000, 50, -1)
    assert (c["cfg2"].m, c["cfg2"].n, c["cfg2"].k, c["cfg2"].p) == (2000, 4000, 100, 10)
    assert (c["cfg3"].batch, c["cfg3"].m, c["cfg3"].n, c["cfg3"].k) == (4096, 64, 256, 16)
    assert (c["cfg4"].m, c["cfg4"].n, c["cfg4"].k, c["cfg4"].p) == (16384, 16384, 256, 16)
    assert (c["cfg5"].m, c["cfg5"].n, c["cfg5"].k, c["cfg5"].p) == (65536, 4096, 64, 8)


def test_spectra():
    s1 = spectrum("cfg1", 500)
    assert s1[0] == 1.0 and np.isclose(s1[25], 0.1)
    s4 = spectrum("cfg4", 300)
    assert np.all(s4[:128] == 1.0) and np.isclose(s4[128], 1.0) and np.isclose(s4[137], 0.01)


def test_small_constructions_have_the_spectrum():
    a = make_np("cfg1", seed=3, scale=0.2)  # 100 x 200
    sv = np.linalg.svd(a, compute_uv=False)
    np.testing.assert_allclose(sv, spectrum("cfg1", 100), rtol=1e-10, atol=1e-14)
    b = make_np("cfg3", seed=3, scale=4 / 4096)
    assert b.shape == (4, 256, 64)
    sv = np.linalg.svd(b[0].T, compute_uv=False)
    assert sv[15] / sv[16] > 1e3  # clear gap at k = 16
    c = make_np("cfg5", seed=3, scale=1 / 64)
    assert c.shape == (8192, 73) and c.min() >= 0.0


def test_bench_stage_work():
    import bench
    w = bench.stage_work(CONFIGS["cfg4"], 16384)
    assert w["sketch"]["flops"] == 2.0 * 272 * 16384 * 16384
    w5 = bench.stage_work(CONFIGS["cfg5"], 4096)
    assert w5["sketch"]["flops"] == 2.0 * 72 * 4096 * 65536  # dual: Omega (72 x 4096) on A^T
