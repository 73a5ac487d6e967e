"""CPU-only tests of the product library: it loads, exports every symbol that
include/tsqr.h declares, and its host logic (plan, slabs, butterfly indexing,
argument validation) agrees with the independently written oracle plan."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle as orc
import paper_0808_2664_b200 as T
from paper_0808_2664_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_symbols_exported():
    hdr = open(os.path.join(ROOT, "include", "tsqr.h")).read()
    declared = set(re.findall(r"^\s*(?:tsqr_status_t|const char \*)\s*(tsqr_\w+)\s*\(", hdr, re.M))
    assert declared == set(_lib.SYMBOLS)
    L = _lib.lib()
    for name in declared:
        assert hasattr(L, name), name


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings():
    L = _lib.lib()
    for s in range(7):
        assert len(L.tsqr_status_string(s)) > 0


def _oracle_nodes(p):
    return sorted(zip(p.node_a.tolist(), p.node_b.tolist(), p.node_stage.tolist(), p.node_level.tolist()))


@pytest.mark.parametrize("m,n,b,s", [
    (4096, 16, 512, 128), (1_000_000, 50, 4096, 96), (100_000, 64, 2048, 96), (5000, 50, 4096, 192),
    (1010, 16, 500, 190), (1020, 16, 500, 190), (64, 64, 64, 64), (3000, 24, 700, 175), (777, 5, 100, 30),
    (100, 40, 100, 30), (8 * 4096 + 100, 64, 4096, 96),
    (33_554_432 // 64, 32, 4096, 96),
])
def test_plan_matches_oracle(m, n, b, s):
    e = T.plan_export(m, n, block_rows=b, tile_rows=s)
    p = orc.plan(m, n, b, s, 1)
    assert np.array_equal(e["tile_row0"], p.tile_row0)
    assert np.array_equal(e["tile_rows"], p.tile_rows)
    mine = sorted(zip(e["node_a"].tolist(), e["node_b"].tolist(), e["node_stage"].tolist(), e["node_level"].tolist()))
    assert mine == _oracle_nodes(p)
    info = T.plan_info(m, n, block_rows=b, tile_rows=s)
    assert info["ntiles"] == p.ntiles and info["nnodes"] == p.nnodes == p.ntiles - 1
    # the tiles' flat chains: chunk rows and the chunk count the oracle derives from them
    pc = orc.plan(m, n, b, s, 1, info["chunk_rows"])
    assert info["chunk_rows"] in (32, 40, 48, 64, 128, 256) and info["nchunks"] == pc.tile_chunk0[-1]


@pytest.mark.parametrize("m,n,b,G", [(1_000_000, 50, 4096, 8), (100_000, 64, 2048, 4), (33_554_432, 32, 4096, 8),
                                     (4096 * 3 + 20, 16, 4096, 2), (5000, 8, 100, 16), (5000, 40, 100, 16)])
def test_slabs_match_oracle_ranks(m, n, b, G):
    s = min(192, b)
    p = orc.plan(m, n, b, s, G)
    for r in range(G):
        row0, ml = T.slab(m, n, b, G, r)
        rows = p.tile_rows[p.tile_rank == r]
        assert row0 == p.tile_row0[p.tile_rank == r][0]
        assert ml == rows.sum()
        # the rank's local plan reproduces the oracle's tiles of that rank
        e = T.plan_export(ml, n, block_rows=b, tile_rows=s, nranks=G, rank=r)
        assert np.array_equal(e["tile_rows"], rows)


def test_butterfly_indexing():
    # Alg. TSQR:par / butterfly indices: partner r xor 2^(k-1), lower on top;
    # log2 G rounds per rank (Table 1: log P messages).
    for G in (2, 4, 8):
        rounds = int(np.log2(G))
        assert T.plan_info(4096, 8, nranks=G, rank=0, block_rows=512)["cross_rounds"] == rounds
        for k in range(1, rounds + 1):
            roles = []
            for r in range(G):
                p, lo, role = T.cross_partner(G, r, k)
                assert p == r ^ (1 << (k - 1)) and lo == (r < p)
                assert T.cross_partner(G, p, k)[0] == r
                roles.append(role)
            # one lower-leftmost and one upper-leftmost rank per group of 2^k
            assert roles.count(1) == G >> k and roles.count(2) == G >> k
        # every rank r > 0 is the upper-leftmost in exactly one round (its head gets a complement)
        for r in range(1, G):
            assert sum(T.cross_partner(G, r, k)[2] == 2 for k in range(1, rounds + 1)) == 1
    with pytest.raises(_lib.TsqrError):
        T.cross_partner(6, 0, 1)
    with pytest.raises(_lib.TsqrError):
        T.cross_partner(4, 0, 3)


def _factor_status(m, n, A, lda, R, ldr, o):
    h = ctypes.c_void_p(None)
    return _lib.lib().tsqr_factor(m, n, A, lda, R, ldr, ctypes.byref(o) if o is not None else None, None,
                                  ctypes.byref(h)), h


def test_factor_validation_without_gpu():
    # every rejection happens on the host before anything is enqueued (no GPU needed)
    o = T.api.opts(block_rows=64, tile_rows=64)
    fake = ctypes.c_void_p(0x1000)
    assert _factor_status(10, 20, fake, 10, None, 0, o)[0] == 2          # m < n
    assert _factor_status(300, 257, fake, 300, None, 0, o)[0] == 3       # n > TSQR_MAX_N
    # wide n (> 64): one CTA per tile, at most 2304 rows
    assert _factor_status(5000, 65, fake, 5000, None, 0, T.api.opts(block_rows=5000, tile_rows=2400))[0] == 3
    assert _factor_status(100, 10, None, 100, None, 0, o)[0] == 1        # null A
    assert _factor_status(100, 10, fake, 99, None, 0, o)[0] == 1         # lda < m
    assert _factor_status(100, 10, fake, 100, fake, 9, o)[0] == 1        # ldr < n
    assert _factor_status(100, 10, fake, 100, None, 0, T.api.opts(block_rows=64, tile_rows=(1 << 30) + 1))[0] == 3
    assert _factor_status(100, 40, fake, 100, None, 0, T.api.opts(block_rows=30, tile_rows=30))[0] == 2  # block < n
    assert _factor_status(1000, 10, fake, 1000, None, 0, T.api.opts(block_rows=64, nranks=3))[0] == 3
    with pytest.raises(_lib.TsqrError):
        T.plan_info(100, 10, block_rows=64, tile_rows=1 << 31)


def test_apply_validation_without_gpu():
    L = _lib.lib()
    assert L.tsqr_apply_qt(None, None, 0, 0, None, 0, None) == 1
    assert L.tsqr_form_q(None, None, 0, None) == 1
    assert L.tsqr_cross_factor(None, 1, None, None, 0, None) == 1
    assert L.tsqr_tree_free(None) == 0
    assert L.tsqr_apply_q(None, None, 0, 0, None) == 1
    assert L.tsqr_cross_apply_q(None, 1, None, 0, None, None, 0, 0, None) == 1
    assert L.tsqr_cross_factor_gathered(None, None, None, 0, None) == 1


def test_caqr_validation_without_gpu():
    L = _lib.lib()
    fake = ctypes.c_void_p(0x1000)
    h = ctypes.c_void_p(None)
    o = T.api.opts(block_rows=256, tile_rows=128)

    def st(m, N, A, lda, panel, R, ldr, opts=o):
        return L.tsqr_caqr_factor(m, N, A, lda, panel, R, ldr, ctypes.byref(opts), None, ctypes.byref(h))

    assert st(100, 200, fake, 100, 32, fake, 200) == 2                  # m < N
    assert st(1000, 0, fake, 1000, 32, fake, 1) == 2                    # N < 1
    assert st(1000, 100, None, 1000, 32, fake, 100) == 1                # null A
    assert st(1000, 100, fake, 1000, 32, None, 100) == 1                # null R
    assert st(1000, 100, fake, 999, 32, fake, 100) == 1                 # lda < m
    assert st(1000, 100, fake, 1000, 32, fake, 99) == 1                 # ldr < N
    assert st(1000, 100, fake, 1000, 0, fake, 100) == 1                 # panel < 1
    assert st(1000, 100, fake, 1000, 257, fake, 100) == 3               # panel > TSQR_MAX_N
    assert st(1000, 100, fake, 1000, 32, fake, 100, T.api.opts(block_rows=256, nranks=2)) == 3
    assert h.value is None                                              # nothing created
    assert L.tsqr_caqr_apply_qt(None, None, 0, 0, None) == 1
    assert L.tsqr_caqr_apply_q(None, None, 0, 0, None) == 1
    assert L.tsqr_caqr_form_q(None, None, 0, None) == 1
    assert L.tsqr_caqr_free(None) == 0
