"""The communicator layer of the C-ABI (tsqr_ctx_*): the butterfly rounds of
Alg. TSQR:par ([TR] P:1667-1707) run INSIDE one collective C call per operation.

CPU: argument validation before anything is enqueued, and NCCL's unique id.
GPU: G contexts of one process joined by the library's loopback transport (each rank's
call synchronises its own stream before posting its message, so no kernel ever waits
on another rank's), one host thread per rank, against the oracle's global tree over
the same plan -- R replicated bitwise, Q^T C in tree order, the replicated thin part,
Q, and the round trip Q (Q^T C) = C.  And a one-rank NCCL communicator (this GPU)
equals the plain local call bit for bit."""
import ctypes
import threading

import numpy as np
import pytest
import torch

import oracle as orc
import paper_0808_2664_b200 as T
from paper_0808_2664_b200 import _lib, inputs


def test_ctx_validation_without_gpu():
    L = _lib.lib()
    fake = ctypes.c_void_p(0x1000)
    h = ctypes.c_void_p(None)
    assert L.tsqr_ctx_factor(None, 100, 10, fake, 100, None, 0, None, None, ctypes.byref(h)) == 1
    assert L.tsqr_ctx_apply_qt(None, None, None, 0, 0, None, 0, None) == 1
    assert L.tsqr_ctx_apply_q(None, None, None, 0, 0, None) == 1
    assert L.tsqr_ctx_form_q(None, None, None, 0, None) == 1
    assert L.tsqr_ctx_set_comm(None, None, 2, 0) == 1
    assert L.tsqr_ctx_info(None, None, None) == 1
    assert L.tsqr_ctx_destroy(None) == 0
    assert L.tsqr_ctx_create(0, None) == 1
    assert L.tsqr_get_unique_id(None) == 1
    hub = ctypes.c_void_p(None)
    assert L.tsqr_loopback_create(3, ctypes.byref(hub)) == 3       # the butterfly needs a power of two
    assert L.tsqr_loopback_create(0, ctypes.byref(hub)) == 1
    assert L.tsqr_loopback_create(4, ctypes.byref(hub)) == 0
    assert L.tsqr_ctx_set_loopback(None, hub, 0) == 1
    assert L.tsqr_loopback_destroy(hub) == 0
    assert "NCCL" in L.tsqr_status_string(6).decode()
    if not torch.cuda.is_available():
        assert L.tsqr_ctx_create(0, ctypes.byref(h)) == 5            # no device: a CUDA error, no handle
        assert h.value is None


def _reference(m, n, b, s, G, k, c):
    A = inputs.to_numpy_colmajor(inputs.gaussian(m, n, 0))
    C = inputs.to_numpy_colmajor(inputs.gaussian(m, k, 1))
    f = orc.tsqr_factor(A, orc.plan(m, n, b, s, G, c))
    return f.R, orc.tsqr_apply_qt(f, C.copy()), orc.tsqr_form_q(f)


@pytest.mark.gpu
@pytest.mark.parametrize("G,m,n,b,s,k", [(2, 20000, 50, 4096, 1366, 64), (4, 40000, 32, 4096, 4096, 128),
                                         (8, 8 * 4096 + 100, 64, 4096, 4096, 70), (8, 50000, 16, 2048, 128, 16),
                                         (2, 12000, 200, 2048, 2048, 64), (4, 16000, 100, 2048, 2048, 20)])
def test_ctx_loopback_collectives(G, m, n, b, s, k):
    hub = T.Loopback(G)
    rows = [T.slab(m, n, b, G, r) for r in range(G)]
    out, errs = {}, []

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            ctx = T.Ctx(0).set_loopback(hub, r)
            assert ctx.info() == (G, r)
            row0, ml = rows[r]
            with torch.cuda.stream(st):
                A = inputs.gaussian_rows(row0, ml, n, 0).cuda()
                C = inputs.gaussian_rows(row0, ml, k, 1).cuda()
                C0 = C.clone()
                top = torch.empty((k, n), dtype=torch.float64, device="cuda")
            R, tree = ctx.factor(A, b, s, stream=st)
            ctx.apply_qt(tree, C, top, stream=st)
            with torch.cuda.stream(st):
                QtC = C.clone()
            Q = ctx.form_q(tree, stream=st)
            ctx.apply_q(tree, C, stream=st)                    # back to C0
            st.synchronize()
            out[r] = tuple(inputs.to_numpy_colmajor(x).copy() for x in (R, QtC, top, Q, C, C0))
            tree.free()
            ctx.free()
        except Exception as e:                                  # noqa: BLE001 -- reported below
            errs.append((r, repr(e)))

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    c = T.plan_info(rows[0][1], n, block_rows=b, tile_rows=s, nranks=G, rank=0)["chunk_rows"]
    Rref, QtC_ref, Qref = _reference(m, n, b, s, G, k, c)
    for r, (row0, ml) in enumerate(rows):
        R, QtC, top, Q, back, C0 = out[r]
        assert np.array_equal(R, out[0][0])                     # R replicated bitwise
        assert np.all(np.tril(R, -1) == 0.0)
        assert orc.rel_fro(orc.sign_normalise(R), orc.sign_normalise(Rref)) <= 1e-11
        assert orc.rel_fro(QtC, QtC_ref[row0:row0 + ml]) <= 1e-11
        assert orc.rel_fro(top, QtC_ref[:n]) <= 1e-11           # thin part on every rank
        assert orc.rel_fro(Q, Qref[row0:row0 + ml]) <= 1e-11
        assert orc.rel_fro(back, C0) <= 1e-13


@pytest.mark.gpu
def test_ctx_nccl_one_rank_equals_local():
    m, n, b, s, k = 100_000, 50, 4096, 1366, 16
    ctx = T.Ctx(0).set_comm(T.Ctx.unique_id(), 1, 0)
    assert ctx.info() == (1, 0)
    At = inputs.gaussian(m, n, 3).cuda()
    Ct = inputs.gaussian(m, k, 4).cuda()
    A1, A2, C1, C2 = At.clone(), At.clone(), Ct.clone(), Ct.clone()
    R1, t1 = ctx.factor(A1, b, s)
    ctx.apply_qt(t1, C1)
    Q1 = ctx.form_q(t1)
    R2, t2 = T.factor(A2, b, s)
    T.apply_qt(t2, C2)
    Q2 = T.form_q(t2)
    torch.cuda.synchronize()
    assert torch.equal(R1, R2) and torch.equal(A1, A2) and torch.equal(C1, C2) and torch.equal(Q1, Q2)
    t1.free()
    t2.free()
    ctx.free()


@pytest.mark.gpu
def test_measure_fp64_peak():
    dmma, dfma = T.measure_fp64_peak()
    # B200: 148 SMs x 64 FP64 FMA/clk x 2 x <= 1.965 GHz = 37.2 TFLOP/s
    assert 20.0 < dmma < 40.0 and 15.0 < dfma < 40.0, (dmma, dfma)
