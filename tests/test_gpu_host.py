"""The host-buffer end-to-end call (tsqr_qr_host, bench.py's e2e path): HOST A in, R and the
explicit Q (or Q^T C) out in host memory.  For n <= 64 with Q it runs pipelined over slabs of
whole tiles (copy-in under the leaf stage, copy-out under the form-Q leaves); the kernels, the
plan and therefore the bytes are those of the device path -- checked bit for bit against
tsqr_factor + tsqr_form_q / tsqr_apply_qt on the same plan, and against the oracle on a small
case."""
import numpy as np
import pytest
import torch

import oracle as orc
import paper_0808_2664_b200 as T
from paper_0808_2664_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,b,s", [(1 << 22, 32, 4096, 4096), (3_000_000, 50, 4096, 1024),
                                     (600_001, 64, 4096, 4096), (5000, 16, 512, 128), (4096, 24, 4096, 4096)])
def test_host_qr_matches_device_path(m, n, b, s):
    At = torch.cat([inputs.gaussian_rows(r, min(1 << 20, m - r), n, 0) for r in range(0, m, 1 << 20)], 1)
    Ah = At.pin_memory()
    hq = T.HostQR()
    R, Q, _ = hq(Ah, block_rows=b, tile_rows=s)
    R2, Q2, _ = hq(Ah, block_rows=b, tile_rows=s)           # workspace reuse, repeat determinism
    Ad = At.cuda()
    Rd, tree = T.factor(Ad, b, s)
    Qd = T.form_q(tree)
    torch.cuda.synchronize()
    assert torch.equal(R, Rd.cpu()) and torch.equal(Q, Qd.cpu())
    assert torch.equal(R, R2) and torch.equal(Q, Q2)
    assert torch.equal(Ah, At)                               # A is read only
    tree.free()
    hq.free()


def test_host_qr_strided_apply_and_oracle():
    m, n, b, s, k = 20_000, 40, 4096, 1024, 12
    At = inputs.gaussian(m, n, 5)
    Ct = inputs.gaussian(m, k, 6)
    big = torch.zeros((n, m + 3), dtype=torch.float64).pin_memory()
    big[:, :m] = At
    Ah = big[:, :m]                                          # host lda = m + 3
    hq = T.HostQR()
    R, Q, _ = hq(Ah, block_rows=b, tile_rows=s)
    Ch = Ct.clone().pin_memory()
    R2, _, C = hq(Ah, block_rows=b, tile_rows=s, C_host=Ch, want_q=False)   # the unpipelined Q^T C path
    c = T.plan_info(m, n, block_rows=b, tile_rows=s)["chunk_rows"]
    f = orc.tsqr_factor(inputs.to_numpy_colmajor(At).copy(), orc.plan(m, n, b, s, 1, c))
    Rg, Qg = inputs.to_numpy_colmajor(R), inputs.to_numpy_colmajor(Q)
    assert orc.rel_fro(orc.sign_normalise(Rg), orc.sign_normalise(f.R)) <= 1e-11
    assert orc.rel_fro(Qg, orc.tsqr_form_q(f)) <= 1e-11
    assert torch.equal(R, R2)
    assert orc.rel_fro(inputs.to_numpy_colmajor(C), orc.tsqr_apply_qt(f, inputs.to_numpy_colmajor(Ct))) <= 1e-11
    hq.free()
