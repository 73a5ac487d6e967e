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
