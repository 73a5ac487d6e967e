"""The chunk engine's warp-to-warp hand-offs under timing stress.

The default build orders each hand-off by program order only (a warp's shared-memory
accesses performed in issue order).  The jitter build
(-DTSQR_HANDOFF_JITTER, libtsqr_jitter.so) puts pseudo-random __nanosleep delays
between every data store and its counter release and after every counter read, so
any read that relied on an unordered access would see stale data.  Both builds must
give bitwise-identical factors, Q and Q^T C (the hand-offs decide only WHEN a value is
read, never which) and match the oracle."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle as orc
import paper_0808_2664_b200 as T
from paper_0808_2664_b200 import _build, inputs

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# narrow configurations of every chunk height: (m, n, b, s, k)
SHAPES = [(300_000, 50, 4096, 1366, 16), (200_000, 64, 4096, 4096, 8), (200_000, 32, 4096, 4096, 128),
          (100_000, 16, 512, 512, 4), (50_000, 40, 4096, 1000, 7)]

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_0808_2664_b200 as T
from paper_0808_2664_b200 import inputs
out = {}
for i, (m, n, b, s, k) in enumerate(eval(sys.argv[3])):
    for rep in range(3):
        A = inputs.gaussian(m, n, 40 + i).cuda()
        C = inputs.gaussian(m, k, 50 + i).cuda()
        R, tree = T.factor(A, b, s)
        T.apply_qt(tree, C)
        Q = T.form_q(tree)
        torch.cuda.synchronize()
        cur = [x.cpu().numpy() for x in (R, A, C, Q)]
        if rep == 0:
            ref = cur
        else:
            assert all(np.array_equal(a, b2) for a, b2 in zip(ref, cur)), "run-to-run difference"
        tree.free()
    for name, x in zip("RACQ", ref):
        out[f"{i}{name}"] = x
np.savez(sys.argv[2], **out)
"""


def _run(lib, path):
    env = dict(os.environ)
    if lib:
        env["TSQR_LIBRARY"] = lib
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, path, repr(SHAPES)], env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    return np.load(path)


def test_jitter_build_bitwise_equal(tmp_path):
    jit = _build.JITTER_LIB
    if not os.path.exists(jit):
        _build.build_variant(jit, ["-DTSQR_HANDOFF_JITTER"])
    base = _run(None, str(tmp_path / "base.npz"))
    jitter = _run(jit, str(tmp_path / "jitter.npz"))
    for key in base.files:
        assert np.array_equal(base[key], jitter[key]), key
    for i, (m, n, b, s, k) in enumerate(SHAPES):                  # and the oracle, same plan
        c = T.plan_info(m, n, block_rows=b, tile_rows=s)["chunk_rows"]
        A0 = inputs.to_numpy_colmajor(inputs.gaussian(m, n, 40 + i))
        f = orc.tsqr_factor(A0, orc.plan(m, n, b, s, 1, c), threads=8)
        R = base[f"{i}R"].T
        assert orc.rel_fro(orc.sign_normalise(R), orc.sign_normalise(f.R)) <= 1e-11
