"""GPU parity of the q-ary structured combine (Alg. QR:qnxn, [TR] P:1957-1979) against the
oracle's combine_q: R, the reflectors' v parts and tau (kappa ~ 1, same reflector sequence)."""
import numpy as np
import pytest
import torch

import oracle as orc
import paper_0808_2664_b200 as T

pytestmark = pytest.mark.gpu


def _pack(R):
    n = R.shape[0]
    return np.concatenate([R[:c + 1, c] for c in range(n)])


def _unpack(p, n):
    R = np.zeros((n, n))
    for c in range(n):
        R[:c + 1, c] = p[c * (c + 1) // 2:(c + 1) * (c + 2) // 2]
    return R


@pytest.mark.parametrize("q,n", [(2, 16), (3, 50), (4, 64), (8, 64), (5, 100), (2, 256), (8, 200), (1, 9), (16, 33)])
def test_combine_q_parity(q, n):
    rng = np.random.default_rng(7 * q + n)
    Rs = [np.triu(rng.standard_normal((n, n))) for _ in range(q)]
    packed = torch.from_numpy(np.concatenate([_pack(R) for R in Rs])).cuda()
    tau = T.combine_stacked(packed, q, n)
    torch.cuda.synchronize()
    R, Ys, to = orc.combine_q(Rs)
    got = packed.cpu().numpy().reshape(q, -1)
    assert orc.rel_fro(_unpack(got[0], n), R) <= 1e-13
    for i in range(1, q):
        assert orc.rel_fro(_unpack(got[i], n), Ys[i - 1]) <= 1e-13
    assert orc.rel_fro(tau.cpu().numpy(), to) <= 1e-13
