"""Error contract of the C ABI (include/idkit_b200.h): every entry validates its
arguments and reports the reference's error class (errors.hpp:9-19,
id.cpp:14-18, qr.cpp:45-46) as a status code with a message, never a crash."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2105_07076_b200 as idk
    return idk.context(0)


@pytest.fixture(scope="module")
def bufs():
    import torch
    a = torch.randn(40, 60, dtype=torch.float64, device="cuda").t().contiguous().t()  # 40 x 60, ld 40
    cols = torch.empty(60, dtype=torch.int64, device="cuda")
    z = torch.empty(60 * 60, dtype=torch.float64, device="cuda")
    c = torch.empty(40 * 60, dtype=torch.float64, device="cuda")
    return a, cols, z, c


def P(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def test_invalid_shapes_and_pointers(ctx, bufs):
    a, cols, z, c = bufs
    L = ctx.lib
    INVALID = 1
    cases = [
        L.idk_optim_id(ctx.h, P(a), 40, 60, 40, 0, P(cols), P(z), P(c)),          # k = 0
        L.idk_optim_id(ctx.h, P(a), 40, 60, 40, 41, P(cols), P(z), P(c)),         # k > min(m, n)
        L.idk_optim_id(ctx.h, P(a), 40, 60, 30, 5, P(cols), P(z), P(c)),          # lda < m
        L.idk_optim_id(ctx.h, P(a), 40, 60, 40, 5, None, P(z), P(c)),             # null cols
        L.idk_optim_id(ctx.h, P(a), 0, 60, 40, 1, P(cols), P(z), P(c)),           # empty
        L.idk_sketch_rid(ctx.h, P(a), 40, 60, 40, 0, 5, -1, 1, 0, None, P(cols), P(z), P(c)),   # p < 0
        L.idk_sketch_rid(ctx.h, P(a), 40, 60, 40, 0, 5, 2, 1, 2, None, P(cols), P(z), P(c)),    # verbatim, no omega
        L.idk_sketch_rid(ctx.h, P(a), 40, 60, 40, 0, 5, 2, 1, 7, None, P(cols), P(z), P(c)),    # bad omega mode
        L.idk_optim_rid(ctx.h, P(a), 40, 60, 40, 0, 5, -0.5, 1, P(cols), P(z), P(c)),           # fraction < 0
        L.idk_id_auto(ctx.h, P(a), 40, 60, 40, 5, 3, 1, 2, 0, None, P(cols), P(z), P(c), None),  # bad method
        L.idk_qr_column_pivoted(ctx.h, P(a), 40, 60, 40, 0, None, None, None),                 # steps = 0
        L.idk_qr_column_pivoted(ctx.h, P(a), 40, 60, 40, 41, None, None, None),                # steps > min
        L.idk_optim_id_batched(ctx.h, P(a), 2, 40, 30, 40, 100, 5, P(cols), P(z), P(c)),       # stride < lda*n
        L.idk_set_cpqr_mode(ctx.h, 9),
        L.idk_set_concurrency(ctx.h, 0),
        L.idk_matmul_ref(ctx.h, P(a), 40, 60, 10, P(a), 60, 60, P(c), 40),                     # lda < m
    ]
    for i, rc in enumerate(cases):
        assert rc == INVALID, (i, rc, ctx.lib.idk_last_error(ctx.h))
    assert L.idk_optim_id(ctx.h, P(a), 40, 60, 40, 0, P(cols), P(z), P(c)) == INVALID
    assert "k must lie in [1, min(rows, cols)]" in ctx.lib.idk_last_error(ctx.h).decode()  # id.cpp:16-17


def test_status_strings_and_abi_version(ctx):
    L = ctx.lib
    assert L.idk_abi_version() >= 1
    for code, text in [(0, "ok"), (1, "invalid argument"), (2, "singular matrix"), (3, "not positive definite")]:
        assert L.idk_status_string(code).decode() == text


def test_empty_batches_are_noops(ctx, bufs):
    a, cols, z, c = bufs
    L = ctx.lib
    arr = (C.c_void_p * 1)()
    assert L.idk_id_auto_batch(ctx.h, 0, arr, 40, 60, 40, 5, 0, None, 0, 0, arr, arr, None, None) == 0
    assert L.idk_optim_id_batched(ctx.h, P(a), 0, 40, 60, 40, 2400, 5, P(cols), P(z), P(c)) == 0


def test_handle_survives_errors(ctx, bufs):
    """An invalid call leaves the handle usable (the next valid call succeeds)."""
    import paper_2105_07076_b200 as idk
    a, cols, z, c = bufs
    assert ctx.lib.idk_optim_id(ctx.h, P(a), 40, 60, 40, 99, P(cols), P(z), P(c)) == 1
    r = idk.optim_id(a, 5)
    assert len(set(r.cols.tolist())) == 5
