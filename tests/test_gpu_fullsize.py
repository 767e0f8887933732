"""Full-size parity on every BASELINE.json configuration against the reference
library itself (oracle/_ref, compiled from /root/reference/proj/src).

* cfg1 / cfg2: the reference at full size (optim_id; the composed sketch path
  with the same Omega).
* cfg3: all 4096 matrices -- the throughput kernel against the reference's
  optim_id (identical pivots, Z within 1e-10) and the exact kernel against the
  composition qr_column_pivoted -> solve_triangular -> select_columns
  (bit-identical).
* cfg4 (16384^2, k = 256, p = 16) and cfg5 (65536 x 4096 dual, k = 64, p = 8):
  our Philox Omega is copied to the host and handed verbatim to the reference
  composition matmul -> qr_column_pivoted -> solve_triangular ->
  select_columns, run on all host threads by column blocks (bit-identical to
  the single-threaded calls; ref_sketch_id_mt).

Tolerances (BASELINE.json north_star): identical column indices;
||dZ||_F / ||Z||_F <= 1e-10; relative error ||A - CZ||_F / ||A||_F within
1e-10 relative (above the fp64 floor of evaluating it); C bit-identical.
cfg4 at full size is at the conditioning limit of fp64: the reference's own
sequential 16384-term sums move its Z by ~1e-10 from the exact solution, so
the default DMMA sketch is held to "pivots and C identical, Z at least as
close to a near-exact solution as the reference's" and the strict 1e-10 is
asserted with the sketch in the reference's arithmetic
(IDK_SKETCH_REFERENCE_ORDER), which isolates everything after the sketch.  Every measured number goes to
gpurun_out/parity_records.json (copied to profiles/parity_r02.json).
"""
import time

import numpy as np
import pytest

from conftest import rel
from paper_2105_07076_b200.configs import CONFIGS, make_np, make_torch

pytestmark = pytest.mark.gpu
ZTOL = 1e-10


@pytest.fixture(scope="module")
def idk():
    import paper_2105_07076_b200 as idk
    return idk


def _dev(a):
    import torch
    return torch.from_numpy(np.asfortranarray(a, dtype=np.float64)).cuda()


def test_cfg1_full(idk, ref, parity_record):
    a = make_np("cfg1", seed=101)
    t0 = time.perf_counter()
    rcols, rz, rapprox = ref.optim_id(a, 50)
    t_ref = time.perf_counter() - t0
    r = idk.optim_id(_dev(a), 50)
    cols, z, c = r.cols.cpu().numpy(), r.z.cpu().numpy(), r.c.cpu().numpy()
    e = np.linalg.norm(a - c @ z) / np.linalg.norm(a)
    re_ = np.linalg.norm(a - rapprox) / np.linalg.norm(a)
    parity_record["cfg1"] = {"reference": "optim_id (id.cpp:29-45)", "shape": [500, 1000], "k": 50,
                             "pivots_identical": bool(np.array_equal(cols, rcols)), "dz_rel": rel(z, rz),
                             "rel_error": e, "ref_rel_error": re_, "d_rel_error_rel": abs(e - re_) / re_,
                             "ref_seconds_1thread": t_ref}
    assert np.array_equal(cols, rcols)
    assert rel(z, rz) <= ZTOL
    assert abs(e - re_) <= ZTOL * re_


def test_cfg2_full(idk, ref, parity_record):
    a = make_np("cfg2", seed=102)
    k, p = 100, 10
    om = idk.sketch_omega(k + p, 2000, 102)
    r = idk.sketch_rid(_dev(a), k, p, seed=102)
    omh = np.asfortranarray(om.cpu().numpy())
    t0 = time.perf_counter()
    rcols, rz, rc, tms = ref.sketch_id_mt(a, k, omh, threads=1)
    t_ref = time.perf_counter() - t0
    cols, z, c = r.cols.cpu().numpy(), r.z.cpu().numpy(), r.c.cpu().numpy()
    e = np.linalg.norm(a - c @ z) / np.linalg.norm(a)
    re_ = np.linalg.norm(a - rc @ rz) / np.linalg.norm(a)
    parity_record["cfg2"] = {"reference": "matmul -> qr_column_pivoted -> solve_triangular -> select_columns",
                             "shape": [2000, 4000], "k": k, "p": p, "omega": "device Philox, passed verbatim",
                             "pivots_identical": bool(np.array_equal(cols, rcols)), "dz_rel": rel(z, rz),
                             "c_bit_identical": bool(np.array_equal(c, rc)), "rel_error": e, "ref_rel_error": re_,
                             "d_rel_error_rel": abs(e - re_) / re_, "ref_seconds_1thread": t_ref,
                             "ref_stage_seconds": tms}
    assert np.array_equal(cols, rcols)
    assert rel(z, rz) <= ZTOL
    assert np.array_equal(c, rc)
    assert abs(e - re_) <= ZTOL * re_


def test_cfg3_all_4096(idk, ref, parity_record):
    import torch
    cfg = CONFIGS["cfg3"]
    a = make_np("cfg3", seed=103)  # (4096, 256, 64): a[b].T is matrix b
    assert a.shape == (4096, 256, 64)
    t0 = time.perf_counter()
    rcols, rz, _ = ref.optim_id_batch_mt(a, cfg.k)
    t_ref = time.perf_counter() - t0
    da = torch.from_numpy(a).cuda()
    ctx = idk.context(0)
    cols, z, c = (x.cpu().numpy() for x in idk.optim_id_batched(da, cfg.k))
    piv_ok = np.array_equal(cols, rcols)
    dz = max(rel(z[b], rz[b]) for b in range(a.shape[0]))
    c_ok = all(np.array_equal(c[b], a[b][cols[b]]) for b in range(a.shape[0]))
    # exact kernel vs the composition, bit for bit, on every matrix
    ctx.set_batched_exact(True)
    try:
        ecols, ez, ec = (x.cpu().numpy() for x in idk.optim_id_batched(da, cfg.k))
    finally:
        ctx.set_batched_exact(False)
    exact_ok = True
    for b in range(a.shape[0]):
        ccols, cz, cc = ref.sketch_id(np.asfortranarray(a[b].T), cfg.k, None)
        exact_ok &= bool(np.array_equal(ecols[b], ccols) and np.array_equal(ez[b].T, cz)
                         and np.array_equal(ec[b].T, cc))
    parity_record["cfg3"] = {"reference": "optim_id per matrix (id.cpp:29-45), all host threads",
                             "matrices": int(a.shape[0]), "shape": [64, 256], "k": cfg.k,
                             "pivots_identical_all": bool(piv_ok), "dz_rel_max": dz,
                             "c_bit_identical_all": bool(c_ok),
                             "exact_kernel_bit_identical_to_composition_all": bool(exact_ok),
                             "ref_seconds_all_threads": t_ref}
    assert piv_ok
    assert dz <= ZTOL
    assert c_ok
    assert exact_ok


def _rel_error_dev(a, c, z, transposed):
    """||A - C Z||_F / ||A||_F on the GPU (test-only checker; torch GEMM)."""
    import torch
    if transposed:
        d = a - (c @ z).t()
    else:
        d = a - c @ z
    e = float(torch.linalg.norm(d) / torch.linalg.norm(a))
    del d
    torch.cuda.empty_cache()
    return e


# Relative-error agreement: 1e-10 relative (north_star) above the fp64 floor of
# evaluating ||A - CZ||_F / ||A||_F itself (16 ulps of 1): cfg5's error is
# 1e-7, where 1e-10 relative would be 1e-17 absolute, below what any fp64
# evaluation of the residual resolves.
def _err_close(e, re_):
    return abs(e - re_) <= 1e-10 * re_ + 16 * 2.0 ** -53


@pytest.mark.parametrize("name", ["cfg4", "cfg5"])
def test_full_size_vs_reference(idk, ref, parity_record, name):
    """Default (DMMA) sketch against the reference composition, plus both
    against a near-exact sketch (tests/accurate_sketch.py) run through the
    reference's own CPQR and solve: at cfg4 (cond(R11) ~ 1.7e4, K = 16384)
    two correctly working fp64 pipelines differ by ~1e-10 in Z, the size of
    the reference's own summation error, so we also assert that our Z is at
    least as close to the near-exact solution as the reference's is."""
    import os
    import torch
    from accurate_sketch import accurate_sketch
    cfg = CONFIGS[name]
    seed = 104 if name == "cfg4" else 105
    a = make_torch(name, seed=seed)
    tall = cfg.m > cfg.n
    mm, nn = (cfg.n, cfg.m) if tall else (cfg.m, cfg.n)  # M = A^T for the dual
    r = idk.id_auto(a, cfg.k, idk.RANDOMIZED, seed=seed, p=cfg.p)
    assert r.transposed == tall
    om = idk.sketch_omega(cfg.l, mm, seed)
    cols, z, c = r.cols.cpu().numpy(), r.z.cpu().numpy(), r.c.cpu().numpy()
    ah = np.asfortranarray(a.cpu().numpy())
    omh = np.asfortranarray(om.cpu().numpy())
    t0 = time.perf_counter()
    rcols, rz, rc, tms = ref.sketch_id_mt(ah, cfg.k, omh, transposed=tall)
    t_ref = time.perf_counter() - t0
    del ah
    # near-exact Y through the reference's qr_column_pivoted + solve_triangular
    y_acc = np.asfortranarray(accurate_sketch(om, a.t() if tall else a).cpu().numpy())
    acols, az, _ = ref.sketch_id(y_acc, cfg.k, None, want_c=False)
    del y_acc
    torch.cuda.empty_cache()
    piv = bool(np.array_equal(cols, rcols))
    dz = rel(z, rz)
    dz_ours_acc, dz_ref_acc = rel(z, az), rel(rz, az)
    c_ok = bool(np.array_equal(c, rc))
    e = _rel_error_dev(a, r.c, r.z, tall)
    re_ = _rel_error_dev(a, torch.from_numpy(rc).cuda(), torch.from_numpy(rz).cuda(), tall)
    parity_record[name] = {
        "reference": ("matmul(Omega, transpose(A)) -> qr_column_pivoted -> solve_triangular -> select_columns"
                      if tall else "matmul(Omega, A) -> qr_column_pivoted -> solve_triangular -> select_columns"),
        "shape": [cfg.m, cfg.n], "k": cfg.k, "p": cfg.p, "dual": tall, "sketch": "DMMA (default)",
        "omega": "device Philox (idk_sketch_omega), copied to host, passed verbatim to the reference",
        "pivots_identical": piv, "pivots_matching_prefix": int(np.argmin(np.append(cols == rcols, False))),
        "dz_rel": dz, "c_bit_identical": c_ok, "rel_error": e, "ref_rel_error": re_,
        "d_rel_error_abs": abs(e - re_), "d_rel_error_rel": abs(e - re_) / re_,
        "near_exact_sketch": {"pivots_identical": bool(np.array_equal(acols, rcols)),
                              "dz_rel_ours_vs_near_exact": dz_ours_acc, "dz_rel_reference_vs_near_exact": dz_ref_acc,
                              "how": "Ozaki splitting of Omega and M into 4 x 19-bit slices, exact slice GEMMs, "
                                     "then the reference's qr_column_pivoted + solve_triangular"},
        "ref_seconds_wall": t_ref, "ref_stage_seconds": tms, "ref_threads": len(os.sched_getaffinity(0)),
        "note": "reference matmul / solve_triangular split by column blocks over threads: bit-identical to one call"}
    assert piv
    assert c_ok
    assert _err_close(e, re_)
    assert np.array_equal(acols, rcols)
    # ours is no further from the near-exact solution than the reference is
    assert dz_ours_acc <= dz_ref_acc * 1.05, (dz_ours_acc, dz_ref_acc)
    assert dz <= 2 * ZTOL, dz  # ~1e-10 at cfg4 is the reference's own error (see near_exact_sketch)


@pytest.mark.parametrize("name", ["cfg4", "cfg5"])
def test_full_size_reference_order_sketch(idk, ref, parity_record, name):
    """With the sketch computed in the reference matmul's own arithmetic
    (IDK_SKETCH_REFERENCE_ORDER: Y bit-identical), everything after it --
    CPQR, Z solve, gather -- matches the reference within the north_star's
    1e-10 on Z at full size."""
    import torch
    cfg = CONFIGS[name]
    seed = 104 if name == "cfg4" else 105
    a = make_torch(name, seed=seed)
    tall = cfg.m > cfg.n
    mm = cfg.n if tall else cfg.m
    ctx = idk.context(0)
    ctx.set_sketch_order(ctx.SKETCH_REFERENCE_ORDER)
    try:
        t0 = time.perf_counter()
        r = idk.id_auto(a, cfg.k, idk.RANDOMIZED, seed=seed, p=cfg.p)
        torch.cuda.synchronize()
        t_gpu = time.perf_counter() - t0
    finally:
        ctx.set_sketch_order(ctx.SKETCH_DMMA)
    om = idk.sketch_omega(cfg.l, mm, seed)
    ah = np.asfortranarray(a.cpu().numpy())
    rcols, rz, rc, _ = ref.sketch_id_mt(ah, cfg.k, np.asfortranarray(om.cpu().numpy()), transposed=tall)
    del ah
    cols, z, c = r.cols.cpu().numpy(), r.z.cpu().numpy(), r.c.cpu().numpy()
    dz = rel(z, rz)
    parity_record[name + "_reference_order_sketch"] = {
        "sketch": "IDK_SKETCH_REFERENCE_ORDER (Y bit-identical to the reference's matmul)",
        "pivots_identical": bool(np.array_equal(cols, rcols)), "dz_rel": dz,
        "c_bit_identical": bool(np.array_equal(c, rc)), "gpu_seconds_wall": t_gpu}
    assert np.array_equal(cols, rcols)
    assert dz <= ZTOL, dz
    assert np.array_equal(c, rc)
