"""Generate tests/golden/reference_cases.npz from the REFERENCE library itself.

Runs oracle/_ref/libidkit_ref.so (the unmodified /root/reference sources built
by `make -C oracle ref`) on the known-answer inputs of the reference's own
tests (proj/tests/test_qr.cpp, test_id.cpp, test_solve.cpp, acceptance.cpp)
and on composed sketch cases, and stores inputs and outputs.  The CPU test
tests/test_oracle_golden.py then pins our restatement (oracle/liboracle.so)
against these fixtures bit for bit, even where the reference is absent.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import OracleError, Reference  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_cases.npz")


def main():
    ref = Reference()
    g = ref.gaussian_matrix
    cases = {}

    def put(name, **arrs):
        for k, v in arrs.items():
            cases[f"{name}/{k}"] = np.asarray(v)

    # ---- qr_column_pivoted (test_qr.cpp) ----
    qr_inputs = {
        "qr_identity4": (np.eye(4), 4),                       # :40-47
        "qr_gs_8x6": (g(8, 6, 11), 6),                        # :65-76
        "qr_partial_10x8": (g(10, 8, 17), 3),                 # :102-115
        "qr_prefix_20x25_full": (g(20, 25, 13), 20),          # :93-100
        "qr_prefix_20x25_9": (g(20, 25, 13), 9),
        "qr_wide_37x101": (g(37, 101, 6), 20),
    }
    zc = np.zeros((6, 4))
    gg = g(6, 2, 23)
    zc[:, 0], zc[:, 2] = gg[:, 0], gg[:, 1]
    qr_inputs["qr_zero_columns"] = (zc, 4)                    # :123-134
    ln = np.zeros((5, 4))
    u = g(5, 1, 7)[:, 0]
    ln[:, 0], ln[:, 1], ln[:, 2], ln[:, 3] = u, 0.01 * np.arange(1, 6), 10.0 * u, 0.02
    qr_inputs["qr_largest_first"] = (ln, 1)                   # :49-63
    ties = np.zeros((8, 17))
    for j in range(17):
        ties[j % 8, j] = 1.0
    qr_inputs["qr_exact_ties"] = (ties, 8)
    for name, (a, s) in qr_inputs.items():
        q, r, perm = ref.qr_column_pivoted(a, s)
        put(name, a=a, steps=s, q=q, r=r, perm=perm)
    order, norms = ref.gram_schmidt_pivoted(g(8, 6, 11), 6)   # tests/support/oracles.hpp:83-138
    put("gs_oracle_8x6", order=order, norms=norms)

    # ---- optim_id / optim_rid / id_auto (test_id.cpp) ----
    uv = np.zeros((6, 3))
    uv[0, 0], uv[0, 1], uv[1, 2] = 1.0, 2.0, 1.0
    det_inputs = {"id_identity5": (np.eye(5), 5), "id_u2uv": (uv, 2), "id_14x20": (g(14, 20, 2), 6),
                  "id_15x22": (g(15, 22, 4), 7), "id_30x24": (g(30, 24, 5), 10), "id_12x12": (g(12, 12, 20), 12)}
    for name, (a, k) in det_inputs.items():
        cols, z, approx = ref.optim_id(a, k)
        put(name, a=a, k=k, cols=cols, z=z, approx=approx)
    rid_inputs = {"rid_14x20": (g(14, 20, 2), 6, 0.2, 3), "rid_identity10": (np.eye(10), 10, 0.2, 17),
                  "rid_18x26": (g(18, 26, 6), 8, 0.2, 1234), "rid_16x16": (g(16, 16, 11), 6, 0.2, 77)}
    for name, (a, k, frac, seed) in rid_inputs.items():
        cols, z, approx = ref.optim_rid(a, k, frac, seed)
        put(name, a=a, k=k, frac=frac, seed=seed, cols=cols, z=z, approx=approx)
    for name, (a, k, rnd) in {"auto_tall_40x12": (g(40, 12, 10), 5, 0), "auto_tall_rid": (g(40, 12, 10), 5, 1)}.items():
        cols, z, approx, tr = ref.id_auto(a, k, rnd, seed=9, frac=0.2)
        put(name, a=a, k=k, randomized=rnd, cols=cols, z=z, approx=approx, transposed=tr)
    # error contract (test_id.cpp:109-129)
    bad = np.zeros((10, 12))
    gg = g(10, 2, 8)
    bad[:, 3], bad[:, 9] = gg[:, 0], gg[:, 1]
    try:
        ref.optim_id(bad, 3)
        code = 0
    except OracleError as e:
        code = {"SingularMatrixError": 2, "NotPositiveDefiniteError": 3}.get(type(e).__name__, 9)
    put("err_det_rank_deficient", a=bad, k=3, code=code)
    bad2 = np.zeros((4, 6))
    gg = g(4, 2, 7)
    bad2[:, 0], bad2[:, 1] = gg[:, 0], gg[:, 1]
    try:
        ref.optim_rid(bad2, 3, 0.0, 5)
        code = 0
    except OracleError as e:
        code = {"SingularMatrixError": 2, "NotPositiveDefiniteError": 3}.get(type(e).__name__, 9)
    put("err_rid_rank_deficient", a=bad2, k=3, code=code)

    # ---- composed sketch ID with the reference's generate() ----
    for name, (m, n, k, p, seed) in {"sketch_60x90": (60, 90, 12, 4, 2), "sketch_30x200": (30, 200, 9, 3, 8)}.items():
        a = g(m, n, seed)
        a[:, ::5] *= 2.0
        omega = ref.generate(1, k + p, m, seed + 100)
        cols, z, c = ref.sketch_id(a, k, omega)
        put(name, a=a, k=k, omega=omega, cols=cols, z=z, c=c)

    # ---- solvers (test_solve.cpp, acceptance.cpp:357-371) ----
    gs = g(8, 8, 44)
    spd = gs.T @ gs + np.eye(8)
    b = g(8, 3, 45)
    put("solve_posdef", s=spd, b=b, x=ref.solve_posdef(spd, b))
    t = np.triu(g(9, 9, 3)) + 4.0 * np.eye(9)
    bb = g(9, 4, 4)
    put("solve_upper", t=t, b=bb, x=ref.solve_triangular(t, bb, True))
    put("solve_lower", t=t.T.copy(), b=bb, x=ref.solve_triangular(np.asfortranarray(t.T), bb, False))
    sym = g(9, 9, 46)
    sym = sym + sym.T
    put("solve_indefinite", s=sym, b=g(9, 3, 47), x=ref.solve_symmetric_indefinite(sym, g(9, 3, 47)))

    # ---- RNG streams (random.cpp) ----
    put("rng", gaussian=ref.generate(1, 7, 5, 123), uniform=ref.generate(2, 7, 5, 123),
        boolean=ref.generate(0, 7, 5, 123), swr=ref.sample_without_replacement(1000, 50, 99),
        mix=np.array([ref.mix_seed(20260601, "gaussian")], dtype=np.uint64))

    np.savez_compressed(OUT, **cases)
    print(f"wrote {OUT}: {len(cases)} arrays, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()
