"""GPU parity of the sequential (out-of-HBM) TSQR: R of a host-resident matrix streamed in row
slabs ([TR] Alg. sequential TSQR P:1725-1753) against the oracle's sequential TSQR on the same
slabs and plans; the streamed-back slabs against the one-GPU factor of each slab."""
import numpy as np
import pytest
import torch

import oracle as orc
import paper_0808_2664_b200 as T
from paper_0808_2664_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,slab,b,s", [(20000, 50, 4096, 4096, 1024), (9000, 16, 2000, 1000, 250),
                                          (12345, 64, 3000, 3000, 1000), (5000, 100, 2048, 2048, 1024),
                                          (3000, 200, 1000, 1000, 1000), (700, 24, 5000, 700, 175),
                                          (4100, 33, 1000, 1000, 500)])
def test_streamed_parity(m, n, slab, b, s):
    At = inputs.gaussian(m, n, 0).pin_memory()
    A0 = inputs.to_numpy_colmajor(At).copy()
    Y = torch.empty_like(At).pin_memory()
    R = T.factor_streamed(At, slab, block_rows=b, tile_rows=s, Y_host=Y)
    torch.cuda.synchronize()
    c = T.plan_info(min(m, slab), n, block_rows=b, tile_rows=s)["chunk_rows"]
    Ro = orc.sequential_tsqr_r(A0, slab, b, s, c)
    Rg = inputs.to_numpy_colmajor(R)
    assert np.all(np.tril(Rg, -1) == 0.0)
    assert orc.rel_fro(orc.sign_normalise(Rg), orc.sign_normalise(Ro)) <= 1e-11
    assert np.array_equal(inputs.to_numpy_colmajor(At), A0)              # A is read only
    # every streamed-back slab equals the one-GPU factor of that slab
    for r0, rows in orc.slab_ranges(m, n, slab):
        Ad = At[:, r0:r0 + rows].contiguous().cuda()
        T.factor(Ad, b, s)[1].free()
        assert torch.equal(Ad.cpu(), Y[:, r0:r0 + rows])


# ----------------------------------------------------- the streamed factor's Q (8(f) row 3)
@pytest.mark.parametrize("m,n,slab,b,s,k", [(20000, 50, 4096, 4096, 1024, 16), (9000, 16, 2000, 1000, 250, 40),
                                            (12345, 64, 3000, 3000, 1000, 64), (5000, 100, 2048, 2048, 1024, 8),
                                            (3000, 200, 1000, 1000, 1000, 70), (700, 24, 5000, 700, 175, 3),
                                            (4100, 33, 1000, 1000, 500, 33)])
def test_streamed_q(m, n, slab, b, s, k):
    """Q and Q^T C of a streamed factor (Alg. TSQR:seq keeps every slab's Q factors in slow
    memory, [TR] P:1725-1753) against the oracle.  Thin Q and Q_thin^T C are unique up to the
    signs R's diagonal fixes, whatever the tree, so they are compared with the
    oracle's TSQR of all of A (its own plan) after sign normalisation; the full Q^T C (tree
    order) by ||Q^T C|| = ||C|| and the round trip Q (Q^T C) = C."""
    At = inputs.gaussian(m, n, 0).pin_memory()
    A0 = inputs.to_numpy_colmajor(At).copy()
    Y = torch.empty_like(At).pin_memory()
    R, st = T.factor_streamed_q(At, slab, Y, block_rows=b, tile_rows=s)
    Q = T.streamed_form_q(st)
    Ct = inputs.gaussian(m, k, 1).pin_memory()
    C0 = inputs.to_numpy_colmajor(Ct).copy()
    top = torch.empty((k, n), dtype=torch.float64).pin_memory()
    T.streamed_apply_qt(st, Ct, top)
    QtC = inputs.to_numpy_colmajor(Ct).copy()
    T.streamed_apply_q(st, Ct)
    back = inputs.to_numpy_colmajor(Ct).copy()
    torch.cuda.synchronize()
    Rg, Qg, topg = (inputs.to_numpy_colmajor(x) for x in (R, Q, top))
    f = orc.tsqr_factor(A0.copy(), orc.plan(m, n, b, s))
    Ro, Qo = orc.sign_normalise(f.R, orc.tsqr_form_q(f))
    Rn, Qn = orc.sign_normalise(Rg, Qg)
    assert orc.rel_fro(Rn, Ro) <= 1e-11
    assert orc.rel_fro(Qn, Qo) <= 1e-11
    assert np.linalg.norm(Qg.T @ Qg - np.eye(n)) <= 1e-13
    assert np.linalg.norm(A0 - Qg @ Rg) / np.linalg.norm(A0) <= 1e-13
    sg = np.where(np.diag(Rg) < 0, -1.0, 1.0)
    assert orc.rel_fro(topg * sg[:, None], Qo.T @ C0) <= 1e-11          # Q_thin^T C on the host
    assert np.array_equal(QtC[:n], topg)                                  # ... and in C's head rows
    assert abs(np.linalg.norm(QtC) - np.linalg.norm(C0)) <= 1e-13 * np.linalg.norm(C0)
    assert orc.rel_fro(back, C0) <= 1e-13
    st.free()
