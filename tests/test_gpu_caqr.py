"""GPU parity of CAQR (right-looking QR with TSQR panels, Sec. 3; Alg. CAQR:j
[TR] P:3992-4048) through the C-ABI against the oracle's CAQR on the same panel plans.
Tolerances as test_gpu_parity.py (BASELINE.json north_star)."""
import numpy as np
import pytest
import torch

import oracle as orc
import paper_0808_2664_b200 as T
from paper_0808_2664_b200 import inputs

pytestmark = pytest.mark.gpu

TOL_R = 1e-11
TOL_INV = 1e-13


def _np(t):
    return inputs.to_numpy_colmajor(t)


CASES = [
    # (m, N, panel, b, s)
    (3000, 100, 32, 1000, 250),      # 4 narrow panels (64-row chunks), last one 4 columns
    (5000, 300, 64, 2048, 512),      # panel 64: 40-row chunks; N > TSQR_MAX_N
    (2000, 300, 128, 1000, 1000),    # wide panels (compact-WY leaves), last one 44 columns
    (4000, 70, 50, 4096, 1024),      # one row block per panel, ragged last panel (20)
    (777, 37, 10, 250, 90),          # small ragged everything
    (500, 500, 100, 500, 500),       # square: the last panel has exactly its own rows
]


@pytest.mark.parametrize("m,N,panel,b,s", CASES)
def test_caqr_parity(m, N, panel, b, s):
    At = inputs.gaussian(m, N, 0)
    A0 = _np(At).copy()
    Ad = At.cuda()
    R, h = T.caqr(Ad, panel, block_rows=b, tile_rows=s, debug=True)
    Q = T.caqr_form_q(h)
    Ct = inputs.gaussian(m, 9, 1)
    C0 = _np(Ct).copy()
    Cd = Ct.cuda()
    T.caqr_apply_qt(h, Cd)
    torch.cuda.synchronize()
    QtC = _np(Cd).copy()
    T.caqr_apply_q(h, Cd)
    torch.cuda.synchronize()
    cf = orc.caqr_factor(A0, panel, b, s, chunk=lambda w: T.plan_info(m, w, block_rows=b, tile_rows=s)["chunk_rows"])
    Rg, Qg = _np(R), _np(Q)
    assert np.all(np.tril(Rg, -1) == 0.0)
    assert orc.rel_fro(orc.sign_normalise(Rg), orc.sign_normalise(cf.R)) <= TOL_R
    assert orc.rel_fro(Qg, orc.caqr_form_q(cf)) <= TOL_R
    assert np.linalg.norm(A0 - Qg @ Rg) / np.linalg.norm(A0) <= TOL_INV
    assert np.linalg.norm(Qg.T @ Qg - np.eye(N)) <= TOL_INV * np.sqrt(N / 64)
    assert orc.rel_fro(QtC, orc.caqr_apply_qt(cf, C0)) <= TOL_R
    assert np.linalg.norm(_np(Cd) - C0) <= 1e-13 * np.linalg.norm(C0)
    h.free()


def test_caqr_handle_reuse_bitwise():
    m, N, panel = 6000, 150, 48
    At = inputs.gaussian(m, N, 5).cuda()
    A1 = At.clone()
    R1, h = T.caqr(A1, panel, block_rows=2000, tile_rows=500)
    A2 = At.clone()
    R2, h = T.caqr(A2, panel, block_rows=2000, tile_rows=500, handle=h)
    torch.cuda.synchronize()
    assert torch.equal(R1, R2) and torch.equal(A1, A2)
    h.free()
