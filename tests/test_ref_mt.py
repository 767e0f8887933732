"""The multithreaded reference composition used at full size (tests and
bench.py's reference arm) must be bit-identical to the reference called once
on one thread: matmul and solve_triangular are split by column blocks, which
changes no arithmetic (matrix.cpp:28-48, solve.cpp:23-53)."""
import numpy as np
import pytest


@pytest.mark.parametrize("threads", [1, 3, 8])
def test_sketch_id_mt_bit_identical(ref, threads):
    rng = np.random.default_rng(7)
    a = np.asfortranarray(rng.standard_normal((120, 333)) * np.exp(-np.arange(333) / 40.0))
    om = np.asfortranarray(rng.standard_normal((25, 120)))
    c1, z1, cc1 = ref.sketch_id(a, 20, om)
    c2, z2, cc2, t = ref.sketch_id_mt(a, 20, om, threads=threads)
    assert np.array_equal(c1, c2) and np.array_equal(z1, z2) and np.array_equal(cc1, cc2)
    assert set(t) == {"omega", "matmul", "qr", "solve", "select"}


def test_sketch_id_mt_dual_and_generated_omega(ref):
    rng = np.random.default_rng(8)
    a = np.asfortranarray(rng.random((200, 64)) @ rng.random((64, 90)))  # stored tall: M = a^T (90 x 200)
    om = ref.generate(1, 30, 90, 5)
    at = np.asfortranarray(a.T)
    c1, z1, cc1 = ref.sketch_id(at, 24, om)
    c2, z2, cc2, _ = ref.sketch_id_mt(a, 24, None, l=30, seed=5, transposed=True, threads=4)
    assert np.array_equal(c1, c2) and np.array_equal(z1, z2) and np.array_equal(cc1, cc2)


def test_sketch_id_mt_k_equals_n(ref):
    rng = np.random.default_rng(9)
    a = np.asfortranarray(rng.standard_normal((12, 6)))
    om = np.asfortranarray(rng.standard_normal((8, 12)))
    c1, z1, _ = ref.sketch_id(a, 6, om)
    c2, z2, _, _ = ref.sketch_id_mt(a, 6, om, threads=4)
    assert np.array_equal(c1, c2) and np.array_equal(z1, z2)


def test_optim_id_batch_mt(ref):
    rng = np.random.default_rng(10)
    b = rng.standard_normal((9, 30, 16))  # 9 matrices 16 x 30, b[i].T column-major
    cols, z, _ = ref.optim_id_batch_mt(b, 4, threads=4)
    for i in range(9):
        c, zz, _ = ref.optim_id(np.asfortranarray(b[i].T), 4)
        assert np.array_equal(c, cols[i]) and np.array_equal(zz, z[i].T)
