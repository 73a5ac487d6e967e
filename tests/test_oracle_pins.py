"""Pins of the CPU oracle to things other than itself (worked examples, closed
forms, textbook / library special cases, invariants, brute force).

Every check here is independent of the oracle's own arithmetic: explicit
reflector matrices are built with numpy from the returned (v, tau), LAPACK is
reached through numpy/torch, MGS in long double is a different algorithm.
Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n.
"""
import os

import numpy as np
import pytest
import scipy.linalg

import oracle as orc

EPS = np.finfo(np.float64).eps


def _golden_rows(path):
    rows = []
    with open(path) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


def _rng(seed):
    return np.random.default_rng(seed)


def _explicit_tile_q(F, tau, rows, n):
    """Q = H_0 H_1 ... H_{n-1} as an explicit rows x rows matrix (numpy)."""
    Q = np.eye(rows)
    for j in range(n):
        v = np.zeros(rows)
        v[j] = 1.0
        v[j + 1:] = F[j + 1:rows, j]
        Q = Q @ (np.eye(rows) - tau[j] * np.outer(v, v))
    return Q


def _explicit_node_q(Y1, tau):
    n = Y1.shape[0]
    Q = np.eye(2 * n)
    for j in range(n):
        v = np.zeros(2 * n)
        v[j] = 1.0
        v[n:n + j + 1] = Y1[:j + 1, j]
        Q = Q @ (np.eye(2 * n) - tau[j] * np.outer(v, v))
    return Q


# --------------------------------------------------------------------- house
def test_house_worked_example(golden_dir):
    (row,) = _golden_rows(os.path.join(golden_dir, "house_3_4.txt"))
    w0, w1, v0, v1, tau, beta = map(float, row)
    v, t, b = orc.house([w0, w1])
    assert v[0] == v0 and v[1] == v1 and t == tau and b == beta


def test_house_special_cases():
    # x = (c,0,0), c > 0 -> tau = 0, beta = c ; x = 0 -> tau = 0, beta = 0
    v, t, b = orc.house([2.5, 0.0, 0.0])
    assert t == 0.0 and b == 2.5 and list(v) == [1.0, 0.0, 0.0]
    v, t, b = orc.house([0.0, 0.0, 0.0])
    assert t == 0.0 and b == 0.0
    # reading R2: a negative pivot with a zero tail is left alone (H = I)
    v, t, b = orc.house([-3.0, 0.0])
    assert t == 0.0 and b == -3.0
    # sign(0) = +1 -> beta = -||x||
    v, t, b = orc.house([0.0, 3.0, 4.0])
    assert b == -5.0 and t == 1.0


@pytest.mark.parametrize("seed", range(5))
def test_house_annihilates(seed):
    w = _rng(seed).standard_normal(7) * 10.0 ** _rng(seed + 100).integers(-5, 5)
    v, t, b = orc.house(w)
    H = np.eye(len(w)) - t * np.outer(v, v)
    hw = H @ w
    assert abs(hw[0] - b) <= 8 * EPS * np.linalg.norm(w)
    assert np.linalg.norm(hw[1:]) <= 8 * EPS * np.linalg.norm(w)
    assert np.linalg.norm(H.T @ H - np.eye(len(w))) <= 16 * EPS
    assert abs(b) == pytest.approx(np.linalg.norm(w), rel=4 * EPS)
    assert 1.0 <= t <= 2.0              # LAPACK property of dlarfg for real data
    assert np.sign(b) == -np.sign(w[0])


# ----------------------------------------------------------------------- hqr
GRID = [(8, 3), (64, 6), (128, 32), (512, 64)]   # S:649 acceptance grid (n <= 64)


@pytest.mark.parametrize("m,n", GRID)
def test_hqr_vs_long_double_mgs(m, n):
    A = _rng(m * 1000 + n).standard_normal((m, n))
    F, tau = orc.hqr(A)
    _, Rm = orc.mgs_ld(A)
    assert orc.rel_fro(orc.sign_normalise(np.triu(F[:n])), Rm) <= 1e-13


@pytest.mark.parametrize("m,n", GRID + [(300, 40)])
def test_hqr_vs_lapack(m, n):
    A = _rng(m + n).standard_normal((m, n))
    F, tau = orc.hqr(A)
    Rl = np.linalg.qr(A, mode="r")
    assert orc.rel_fro(orc.sign_normalise(np.triu(F[:n])), orc.sign_normalise(Rl)) <= 1e-13


def test_hqr_identity_columns():
    # A = I(:,1:n) -> R = I, tau = 0 exactly
    A = np.eye(10)[:, :4]
    F, tau = orc.hqr(A)
    assert np.all(tau == 0.0)
    assert np.array_equal(np.triu(F[:4]), np.eye(4))


@pytest.mark.parametrize("m,n", [(8, 3), (64, 6), (40, 40)])
def test_hqr_invariants(m, n):
    A = _rng(7 * m + n).standard_normal((m, n))
    F, tau = orc.hqr(A)
    Q = _explicit_tile_q(F, tau, m, n)[:, :n]
    R = np.triu(F[:n])
    assert np.linalg.norm(A - Q @ R) / np.linalg.norm(A) <= 1e-14
    assert np.linalg.norm(Q.T @ Q - np.eye(n)) <= 1e-14
    # Corollary 1 identity: R^T R = A^T A
    assert np.linalg.norm(R.T @ R - A.T @ A) / np.linalg.norm(A) ** 2 <= 1e-14


def test_hqr_rank_deficient_zero_column():
    # reading R2: a zero column gives tau = 0 (H = I), no error
    A = _rng(3).standard_normal((20, 5))
    A[:, 2] = 0.0
    A[:, 4] = A[:, 0]
    F, tau = orc.hqr(A)
    Q = _explicit_tile_q(F, tau, 20, 5)[:, :5]
    assert np.linalg.norm(A - Q @ np.triu(F[:5])) <= 1e-14 * np.linalg.norm(A)
    assert np.all(np.isfinite(F))


# ------------------------------------------------------------------- combine
def test_combine_sparsity_matches_paper(golden_dir):
    # eq. fact_2rs, P:1051-1083 (the 5x5 example)
    pat = _golden_rows(os.path.join(golden_dir, "fact_2rs_pattern.txt"))
    rng = _rng(11)
    Ra = np.triu(rng.standard_normal((5, 5)))
    Rb = np.triu(rng.standard_normal((5, 5)))
    R, Y1, tau, _ = orc.combine(Ra, Rb)
    V = np.vstack([np.eye(5), Y1])
    for i in range(10):
        for j in range(5):
            c = pat[i][j]
            if c == "1":
                assert V[i, j] == 1.0
            elif c == ".":
                assert V[i, j] == 0.0
            else:
                assert V[i, j] != 0.0


@pytest.mark.parametrize("n", [1, 2, 8, 32, 64])
def test_combine_vs_dense_qr(n):
    rng = _rng(n)
    Ra = np.triu(rng.standard_normal((n, n)))
    Rb = np.triu(rng.standard_normal((n, n)))
    R, Y1, tau, _ = orc.combine(Ra, Rb)
    S = np.vstack([Ra, Rb])
    F, _ = orc.hqr(S)                                       # dense, unstructured
    assert orc.rel_fro(orc.sign_normalise(R), orc.sign_normalise(np.triu(F[:n]))) <= 1e-13
    assert orc.rel_fro(orc.sign_normalise(R), orc.sign_normalise(np.linalg.qr(S, mode="r"))) <= 1e-13
    # Y1 strictly lower is exactly zero
    assert np.all(np.tril(Y1, -1) == 0.0)
    # explicit node Q: Q^T [Ra; Rb] = [R; 0]
    Q = _explicit_node_q(Y1, tau)
    out = Q.T @ S
    assert np.linalg.norm(out[:n] - R) <= 1e-13 * np.linalg.norm(S)
    assert np.linalg.norm(out[n:]) <= 1e-13 * np.linalg.norm(S)


def test_combine_identity_zero():
    # R0 = I, R1 = 0 -> R = I, tau = 0
    R, Y1, tau, _ = orc.combine(np.eye(6), np.zeros((6, 6)))
    assert np.array_equal(R, np.eye(6)) and np.all(tau == 0.0) and np.all(Y1 == 0.0)


def test_combine_flop_count():
    # (2/3) n^3 for the structured QR of two triangles
    _, _, _, fl = orc.combine(np.triu(np.ones((64, 64))), np.triu(np.ones((64, 64))))
    ratio = fl / (2.0 / 3.0 * 64 ** 3)
    assert 1.0 <= ratio <= 1.1


# -------------------------------------------------------------------- T build
@pytest.mark.parametrize("rows,k", [(6, 3), (40, 8), (64, 64)])
def test_build_t_leaf(rows, k):
    A = _rng(rows + k).standard_normal((rows, k))
    F, tau = orc.hqr(A)
    Y = np.tril(F, -1)
    Y[np.arange(k), np.arange(k)] = 1.0
    T = orc.build_t(F, tau)
    Qexp = _explicit_tile_q(F, tau, rows, k)
    assert np.linalg.norm(np.eye(rows) - Y @ T @ Y.T - Qexp) <= 1e-13 * rows
    assert np.all(np.tril(T, -1) == 0.0) and np.array_equal(np.diag(T), tau)


@pytest.mark.parametrize("n", [3, 16, 33])
def test_build_t_node(n):
    rng = _rng(50 + n)
    R, Y1, tau, _ = orc.combine(np.triu(rng.standard_normal((n, n))), np.triu(rng.standard_normal((n, n))))
    T = orc.build_t_node(Y1, tau)
    Y = np.vstack([np.eye(n), Y1])
    assert np.linalg.norm(np.eye(2 * n) - Y @ T @ Y.T - _explicit_node_q(Y1, tau)) <= 1e-13 * n
    # the paper's Alg. YT:scaled T' satisfies rho_1...rho_n = I + Y T' Y^T with T' = -T (reading R3)
    assert np.linalg.norm(np.eye(2 * n) + Y @ (-T) @ Y.T - _explicit_node_q(Y1, tau)) <= 1e-13 * n


# ---------------------------------------------------------------------- plan
def _plan_nodes(p):
    return [(int(l), int(a), int(b)) for a, b, l in zip(p.node_a, p.node_b, p.node_level)]


def test_plan_eq4_tree(golden_dir):
    ref = [tuple(map(int, r)) for r in _golden_rows(os.path.join(golden_dir, "eq4_binary_tree_p4.txt"))]
    p = orc.plan(4 * 32, 8, 32)
    assert _plan_nodes(p) == ref


def test_plan_promotion_p5(golden_dir):
    ref = [tuple(map(int, r)) for r in _golden_rows(os.path.join(golden_dir, "build_tree_p5.txt"))]
    p = orc.plan(5 * 32, 8, 32)
    assert _plan_nodes(p) == ref
    widths = [5]
    for lev in range(1, 4):
        widths.append(widths[-1] - int(np.sum(p.node_level == lev)))
    assert widths == [5, 3, 2, 1]


def test_plan_config_shapes():
    p = orc.plan(4096, 16, 512)                  # config 1: 8 leaves, depth 3
    assert p.ntiles == 8 and p.nnodes == 7 and p.node_level.max() == 3
    p = orc.plan(1_000_000, 50, 4096)            # config 2: 245 blocks, last one 576 rows
    assert p.ntiles == 245 and p.tile_rows[-1] == 576
    assert p.node_level.max() == int(np.ceil(np.log2(245)))
    p = orc.plan(100_000, 200, 2048)             # config 3: 49 blocks, last 1696 rows
    assert p.ntiles == 49 and p.tile_rows[-1] == 1696
    p = orc.plan(1_000_000, 50, 4096, 256, 8)    # runs of 31,31,31,31,31,30,30,30 blocks
    blocks_per_rank = []
    for r in range(8):
        rows = p.tile_rows[p.tile_rank == r].sum()
        blocks_per_rank.append(int(np.ceil(rows / 4096)))
    assert blocks_per_rank == [31, 31, 31, 31, 31, 30, 30, 30]
    # every tile is >= n rows and <= s rows; tiles cover 0..m-1 contiguously
    assert np.all(p.tile_rows >= 50) and np.all(p.tile_rows <= 256)
    assert p.tile_row0[0] == 0 and np.all(p.tile_row0[1:] == np.cumsum(p.tile_rows)[:-1])
    assert p.tile_row0[-1] + p.tile_rows[-1] == 1_000_000
    # rank stage: G - 1 nodes, depth log2 G (Table 1: log P messages)
    assert np.sum(p.node_stage == 2) == 7 and p.node_level[p.node_stage == 2].max() == 3
    # a binary tree over L tiles has L - 1 nodes
    assert p.nnodes == p.ntiles - 1


def test_plan_remainder_rules():
    # remainder >= n becomes its own block; < n merges into the last block (reading R6)
    p = orc.plan(1000 + 10, 16, 500)
    assert list(p.tile_rows) == [500, 510]
    # tiles of even height: 250 row pairs over 3 tiles -> 84, 83, rest
    p = orc.plan(1000 + 10, 16, 500, 200)
    assert list(p.tile_rows) == [168, 166, 166, 170, 170, 170]
    assert all(r0 % 2 == 0 for r0 in p.tile_row0)
    # an odd block: the last tile takes the odd row
    p = orc.plan(1011, 16, 500, 200)
    assert list(p.tile_rows) == [168, 166, 166, 170, 170, 171]
    # even heights would leave a tile shorter than n: plain near-equal heights
    p = orc.plan(99, 49, 99, 50)
    assert list(p.tile_rows) == [50, 49]
    p = orc.plan(1000 + 16, 16, 500)
    assert list(p.tile_rows) == [500, 500, 16]
    # s < n: tiles are never shorter than n (t = min(ceil(h/s), floor(h/n)))
    p = orc.plan(100, 40, 100, 30)
    assert list(p.tile_rows) == [50, 50]
    p = orc.plan(100, 64, 100, 96)
    assert list(p.tile_rows) == [100]


@pytest.mark.parametrize("args", [(5, 8, 4, 4, 1), (64, 8, 16, 16, 3), (64, 8, 32, 32, 4), (64, 8, 4, 4, 1)])
def test_plan_rejects(args):
    with pytest.raises(ValueError):
        orc.plan(*args[:3], s=args[3], G=args[4])


# ---------------------------------------------------------------------- TSQR
@pytest.mark.parametrize("c", [0, 32])
@pytest.mark.parametrize("m,n,b,s,G", [
    (64, 6, 16, 16, 4),                 # S:218 P=4 binary on 64x6
    (4096, 16, 512, 512, 1),            # config 1
    (3000, 24, 700, 256, 2),
    (2048, 64, 512, 256, 4),
    (1500, 33, 400, 128, 1),
])
def test_tsqr_r_vs_flat(m, n, b, s, G, c):
    A = _rng(m + n + b).standard_normal((m, n))
    f = orc.tsqr_factor(A, orc.plan(m, n, b, s, G, c))
    Rflat = np.triu(orc.hqr(A)[0][:n])
    assert np.all(np.tril(f.R, -1) == 0.0)
    assert orc.rel_fro(orc.sign_normalise(f.R), orc.sign_normalise(Rflat)) <= 1e-13
    assert np.linalg.norm(f.R.T @ f.R - A.T @ A) / np.linalg.norm(A) ** 2 <= 1e-14


def test_tsqr_tree_independence():
    # any tree gives the same R modulo signs
    A = _rng(5).standard_normal((2048, 20))
    Rs = [orc.sign_normalise(orc.tsqr_factor(A, orc.plan(2048, 20, b, s, G)).R)
          for (b, s, G) in [(2048, 2048, 1), (256, 256, 1), (512, 64, 2), (128, 40, 8)]]
    for R in Rs[1:]:
        assert orc.rel_fro(R, Rs[0]) <= 1e-13


def test_tsqr_r_vs_mgs_tiny():
    A = _rng(9).standard_normal((64, 6))
    f = orc.tsqr_factor(A, orc.plan(64, 6, 16, 16, 1))
    _, Rm = orc.mgs_ld(A)
    assert orc.rel_fro(orc.sign_normalise(f.R), Rm) <= 1e-13


@pytest.mark.parametrize("m,n,b,s,G,k,c", [(512, 8, 128, 64, 2, 5, 0), (1200, 16, 300, 150, 1, 16, 0),
                                           (512, 8, 128, 64, 2, 5, 16), (1200, 16, 300, 150, 1, 16, 32),
                                           (1000, 40, 500, 500, 1, 7, 32)])
def test_tsqr_apply_qt_closed_forms(m, n, b, s, G, k, c):
    rng = _rng(m * k)
    A = rng.standard_normal((m, n))
    p = orc.plan(m, n, b, s, G, c)
    f = orc.tsqr_factor(A, p)
    # Q^T A = [R; 0] in tree order
    QtA = orc.tsqr_apply_qt(f, A)
    assert np.linalg.norm(QtA[:n] - f.R) <= 1e-14 * np.linalg.norm(A) * 10
    assert np.linalg.norm(QtA[n:]) <= 1e-14 * np.linalg.norm(A) * 10
    C = rng.standard_normal((m, k))
    QtC = orc.tsqr_apply_qt(f, C)
    assert abs(np.linalg.norm(QtC) - np.linalg.norm(C)) <= 1e-14 * np.linalg.norm(C) * 10
    back = orc.tsqr_apply_q(f, QtC)
    assert np.linalg.norm(back - C) <= 1e-14 * np.linalg.norm(C) * 10
    Q = orc.tsqr_form_q(f)
    assert np.linalg.norm(QtC[:n] - Q.T @ C) <= 1e-13 * np.linalg.norm(C)


@pytest.mark.parametrize("m,n,b,s,G,c", [(4096, 16, 512, 512, 1, 0), (3000, 30, 1000, 200, 2, 0),
                                         (4096, 16, 512, 512, 1, 64), (3000, 30, 1000, 200, 2, 32),
                                         (2000, 50, 1000, 1000, 1, 32)])
def test_tsqr_form_q(m, n, b, s, G, c):
    A = _rng(m - n).standard_normal((m, n))
    f = orc.tsqr_factor(A, orc.plan(m, n, b, s, G, c))
    Q = orc.tsqr_form_q(f)
    assert np.linalg.norm(A - Q @ f.R) / np.linalg.norm(A) <= 1e-13
    assert np.linalg.norm(Q.T @ Q - np.eye(n)) <= 1e-13
    # kappa ~ 1: Q = A R^{-1} by an independent triangular solve
    Qs = scipy.linalg.solve_triangular(f.R, A.T, trans="T", lower=False).T
    assert np.linalg.norm(Q - Qs) / np.linalg.norm(Qs) <= 1e-12


def test_tsqr_orthonormal_input():
    # A with orthonormal columns: Q^ = A, R^ = I
    Qa, _ = np.linalg.qr(_rng(1).standard_normal((1024, 12)))
    f = orc.tsqr_factor(Qa, orc.plan(1024, 12, 256, 128, 1))
    Rn, Qn = orc.sign_normalise(f.R, orc.tsqr_form_q(f))
    assert np.linalg.norm(Rn - np.eye(12)) <= 1e-13
    assert np.linalg.norm(Qn - Qa) <= 1e-13


def test_tsqr_ill_conditioned_invariants():
    # the C4 recipe at a small size: sigma log-spaced 1 .. 1e-10
    rng = _rng(2)
    n = 16
    G = rng.standard_normal((4096, n))
    sig = 10.0 ** (-10.0 * np.arange(n) / (n - 1))
    V, _ = np.linalg.qr(rng.standard_normal((n, n)))
    A = (G * sig) @ V.T
    for c in (0, 32):
        f = orc.tsqr_factor(A, orc.plan(4096, n, 512, 256, 1, c))
        Q = orc.tsqr_form_q(f)
        assert np.linalg.norm(A - Q @ f.R) / np.linalg.norm(A) <= 1e-13
        assert np.linalg.norm(Q.T @ Q - np.eye(n)) <= 1e-13
        assert np.linalg.norm(f.R.T @ f.R - A.T @ A) / np.linalg.norm(A) ** 2 <= 1e-14
        Rflat = np.linalg.qr(A, mode="r")
        assert orc.rel_fro(orc.sign_normalise(f.R), orc.sign_normalise(Rflat)) <= 1e-13


def test_mgs_ld_pins():
    Q, R = orc.mgs_ld(np.array([[3.0], [4.0]]))
    assert R[0, 0] == 5.0 and np.allclose(Q[:, 0], [0.6, 0.8], rtol=0, atol=1e-16)
    A = _rng(4).standard_normal((50, 7))
    Q, R = orc.mgs_ld(A)
    assert orc.rel_fro(R, orc.sign_normalise(np.linalg.qr(A, mode="r"))) <= 1e-14
    assert np.linalg.norm(Q.T @ Q - np.eye(7)) <= 1e-14


# ------------------------------------------------- flat-chain tile QR (leaves)
@pytest.mark.parametrize("rows,n", [(100, 7), (257, 16), (64, 64), (200, 50)])
def test_chain_c0_is_hqr(rows, n):
    # c = 0 and c >= rows are the paper's plain leaf QR (DGEQR2), bit for bit
    A = _rng(rows * n).standard_normal((rows, n))
    F0, t0 = orc.hqr(A)
    for c in (0, rows, rows + 5):
        F, t = orc.chain_qr(A, c)
        assert np.array_equal(F, F0) and np.array_equal(t[0], t0)


@pytest.mark.parametrize("rows,n,c", [(200, 16, 32), (200, 50, 32), (97, 40, 32), (130, 64, 32),
                                      (300, 24, 64), (64, 64, 32), (77, 50, 32), (50, 16, 8),
                                      (203, 50, 40), (170, 44, 48)])
def test_chain_equals_stacked_hqr(rows, n, c):
    # Sequential TSQR: every chunk step is qr([R; A_k]) with R the
    # upper trapezoid so far.  Dense hqr of the explicitly stacked matrix
    # (zero-padded to n rows while it is wide) touches the same nonzeros -- R's
    # zeros and the padding add exact zeros -- so it must agree bit for bit:
    # the chunk's taus, its reflector tails, and R after every chunk.
    A = _rng(rows + 7 * n + c).standard_normal((rows, n))
    F, tau = orc.chain_qr(A, c)
    Rk = np.zeros((0, n))
    for k, r0 in enumerate(range(0, rows, c)):
        h = min(c, rows - r0)
        r = Rk.shape[0]
        S = np.vstack([Rk, A[r0:r0 + h], np.zeros((max(0, n - r - h), n))])
        Fs, ts = orc.hqr(S)
        kk = min(n, r + h)                                 # reflectors this chunk has
        assert np.array_equal(tau[k][:kk], ts[:kk]) and np.all(tau[k][kk:] == 0.0)
        for i in range(h):                                 # tails: tile row > column
            cols = min(n, r0 + i)
            assert np.array_equal(F[r0 + i, :cols], Fs[r + i, :cols])
        Rk = np.triu(Fs[:kk])
    assert np.array_equal(np.triu(F[:n]), Rk)


@pytest.mark.parametrize("rows,n,c", [(300, 20, 32), (256, 64, 32), (1000, 50, 32), (1000, 50, 40), (700, 40, 48)])
def test_chain_r_vs_lapack_and_q(rows, n, c):
    A = _rng(rows - n + c).standard_normal((rows, n))
    F, tau = orc.chain_qr(A, c)
    R = np.triu(F[:n])
    assert orc.rel_fro(orc.sign_normalise(R), orc.sign_normalise(np.linalg.qr(A, mode="r"))) <= 1e-13
    p = orc.plan(rows, n, rows, rows, 1, c)             # one tile: Q from the stored reflectors
    f = orc.tsqr_factor(A, p)
    assert np.array_equal(f.A, F) and np.array_equal(f.tau_tile, tau)
    Q = orc.tsqr_form_q(f)
    assert np.linalg.norm(A - Q @ R) / np.linalg.norm(A) <= 1e-13
    assert np.linalg.norm(Q.T @ Q - np.eye(n)) <= 1e-13


# ------------------------------------------------------------------- CAQR
@pytest.mark.parametrize("m,N,panel,b,s,c", [(600, 40, 16, 200, 100, 0), (777, 37, 10, 250, 90, 16),
                                              (300, 300, 64, 300, 300, 0), (1000, 70, 70, 400, 200, 0)])
def test_caqr_pins(m, N, panel, b, s, c):
    """CAQR (Sec. 3; Alg. CAQR:j [TR] P:3992-4048) pinned to LAPACK's R (unique up to
    signs for a full-rank A), A = QR, Q^T Q = I, the inverse pair apply_q(apply_qt(C)) = C and the
    thin part of Q^T C = R^-T A^T C."""
    rng = np.random.default_rng(3)
    A = np.asfortranarray(rng.standard_normal((m, N)))
    cf = orc.caqr_factor(A, panel, b, s, chunk=lambda w: min(c, 8 * ((w + 7) // 8)) if c else 0)
    R = cf.R
    assert np.all(np.tril(R, -1) == 0.0)
    Rl = scipy.linalg.qr(A, mode="r")[0][:N]
    assert orc.rel_fro(orc.sign_normalise(R), orc.sign_normalise(Rl)) <= 1e-12
    Q = orc.caqr_form_q(cf)
    assert np.linalg.norm(A - Q @ R) / np.linalg.norm(A) <= 1e-14
    assert np.linalg.norm(Q.T @ Q - np.eye(N)) <= 1e-13
    C = rng.standard_normal((m, 5))
    QtC = orc.caqr_apply_qt(cf, C)
    assert np.linalg.norm(orc.caqr_apply_q(cf, QtC) - C) <= 1e-13 * np.linalg.norm(C)
    thin = scipy.linalg.solve_triangular(R, A.T @ C, trans="T")
    assert orc.rel_fro(QtC[:N], thin) <= 1e-12


def test_caqr_single_panel_is_tsqr():
    """panel >= N: CAQR is exactly one TSQR (same plan, bitwise)."""
    A = np.asfortranarray(np.random.default_rng(4).standard_normal((900, 24)))
    cf = orc.caqr_factor(A, 32, 300, 100)
    f = orc.tsqr_factor(A.copy(order="F"), orc.plan(900, 24, 300, 100, 1, 0))
    assert np.array_equal(cf.R, f.R)
    assert np.array_equal(orc.caqr_form_q(cf), orc.tsqr_form_q(f))


# ------------------------------------------------------ sequential (streamed) TSQR
def test_slab_ranges():
    assert orc.slab_ranges(1000, 10, 300) == [(0, 300), (300, 300), (600, 300), (900, 100)]
    assert orc.slab_ranges(905, 10, 300) == [(0, 300), (300, 300), (600, 305)]
    assert orc.slab_ranges(200, 10, 300) == [(0, 200)]


@pytest.mark.parametrize("m,n,slab,b,s,c", [(3000, 20, 700, 350, 175, 0), (2500, 40, 1000, 500, 250, 16),
                                             (1200, 100, 500, 500, 500, 0)])
def test_sequential_tsqr_pins(m, n, slab, b, s, c):
    """Flat tree over slabs pinned to LAPACK's R (unique up to signs, full rank) and to
    R^T R = A^T A; one slab is exactly the parallel TSQR (bitwise)."""
    A = np.asfortranarray(np.random.default_rng(6).standard_normal((m, n)))
    R = orc.sequential_tsqr_r(A, slab, b, s, c)
    assert np.all(np.tril(R, -1) == 0.0)
    Rl = scipy.linalg.qr(A, mode="r")[0][:n]
    assert orc.rel_fro(orc.sign_normalise(R), orc.sign_normalise(Rl)) <= 1e-12
    assert np.linalg.norm(R.T @ R - A.T @ A) / np.linalg.norm(A) ** 2 <= 1e-14
    one = orc.sequential_tsqr_r(A, m, b, s, c)
    assert np.array_equal(one, orc.tsqr_factor(A.copy(order="F"), orc.plan(m, n, b, s, 1, c)).R)


# ------------------------------------------------------------- q-ary combine
def _q_from_combine(Ys, tau, n):
    """Explicit Q (qn x n) of Alg. QR:qnxn: the reflectors applied to [I_n; 0] in reverse."""
    q = len(Ys) + 1
    Q = np.zeros((q * n, n))
    Q[:n] = np.eye(n)
    for j in range(n - 1, -1, -1):
        I = [j] + [i * n + r for i in range(1, q) for r in range(j + 1)]
        v = np.concatenate([[1.0]] + [Ys[i - 1][:j + 1, j] for i in range(1, q)])
        Q[I] -= tau[j] * np.outer(v, v @ Q[I])
    return Q


@pytest.mark.parametrize("q,n", [(2, 5), (3, 8), (4, 17), (8, 33), (5, 64)])
def test_combine_q_pins(q, n):
    rng = np.random.default_rng(q * 100 + n)
    Rs = [np.triu(rng.standard_normal((n, n))) for _ in range(q)]
    R, Ys, tau = orc.combine_q(Rs)
    S = np.vstack(Rs)
    Rl = scipy.linalg.qr(S, mode="r")[0][:n]
    assert orc.rel_fro(orc.sign_normalise(R), orc.sign_normalise(Rl)) <= 1e-13
    Q = _q_from_combine(Ys, tau, n)
    assert np.linalg.norm(Q @ R - S) / np.linalg.norm(S) <= 1e-14
    assert np.linalg.norm(Q.T @ Q - np.eye(n)) <= 1e-13
    if q == 2:                                            # the binary combine (C oracle)
        Rb, Y1, tb, _ = orc.combine(Rs[0], Rs[1])
        assert orc.rel_fro(R, Rb) <= 1e-14 and orc.rel_fro(Ys[0], Y1) <= 1e-14 and orc.rel_fro(tau, tb) <= 1e-14


# ------------------------------------------------------- CholeskyQR (8(f) row 4)
def test_cholqr_worked_example(golden_dir):
    """Alg. CholeskyQR ([TR] P:1410-1419) on the hand-worked 2x2 case."""
    (row,) = _golden_rows(os.path.join(golden_dir, "cholqr_2x2.txt"))
    v = [float(x) for x in row]
    A = np.array([[v[0], v[1]], [v[2], v[3]]])
    info, R, Q = orc.cholqr(A)
    assert info == 0
    np.testing.assert_allclose(R, [[v[4], v[5]], [0.0, v[6]]], rtol=0, atol=4 * EPS * 5)
    # q2 = (a2 - 2.2 q1) / 0.4 cancels (1 - 1.32) and divides by 0.4: ~10 eps of rounding
    np.testing.assert_allclose(Q, [[v[7], v[8]], [v[9], v[10]]], rtol=0, atol=32 * EPS)


@pytest.mark.parametrize("m,n,seed", [(200, 8, 0), (1000, 16, 1), (3000, 33, 2)])
def test_cholqr_matches_lapack_householder_r(m, n, seed):
    """kappa(A) ~ 1: CholeskyQR's R is the QR factor's R with a positive diagonal (R is
    unique up to the signs of its rows), so it equals LAPACK's Householder R
    after sign normalisation; Q = A R^{-1} equals an independent triangular solve."""
    A = _rng(seed).standard_normal((m, n))
    info, R, Q = orc.cholqr(A)
    assert info == 0
    assert np.all(np.diag(R) > 0) and np.all(np.tril(R, -1) == 0)
    Rl = np.linalg.qr(A, mode="r")
    Rl = Rl * np.sign(np.diag(Rl))[:, None]
    assert np.linalg.norm(R - Rl) / np.linalg.norm(Rl) <= 1e-13
    Qs = scipy.linalg.solve_triangular(R, A.T, trans="T", lower=False).T     # R^T Q^T = A^T
    assert np.linalg.norm(Q - Qs) <= 1e-13 * np.sqrt(n)
    assert np.linalg.norm(Q.T @ Q - np.eye(n)) <= 1e-13


def test_cholqr_orthonormal_input():
    """A with orthonormal columns: W = I exactly up to rounding, so R = I and Q = A."""
    A, _ = np.linalg.qr(_rng(5).standard_normal((500, 12)))
    info, R, Q = orc.cholqr(A)
    assert info == 0
    assert np.linalg.norm(R - np.eye(12)) <= 1e-14
    assert np.linalg.norm(Q - A) <= 1e-14


def test_cholqr_breakdown_on_zero_column():
    """A zero column makes the leading minor of that order of W = A^T A zero: Alg.
    CholeskyQR line 2 breaks down exactly there (info = column + 1)."""
    A = _rng(6).standard_normal((100, 6))
    A[:, 3] = 0.0
    info, _, _ = orc.cholqr(A)
    assert info == 4


def test_cholqr_orthogonality_degrades_as_kappa_squared():
    """"the Q factor computed by CholeskyQR loses orthogonality proportionally to
    kappa_2(A)^2", while Householder QR's Q stays orthogonal: on the C4
    recipe (sigma log-spaced 1 .. 1/kappa, reading R15) the orthogonality error grows by
    >= 1e5 from kappa = 1e2 to 1e5 (kappa^2 grows 1e6) and stays within c kappa^2 eps."""
    import torch
    from paper_0808_2664_b200 import inputs
    errs = {}
    for kappa in (1e2, 1e5):
        A = inputs.to_numpy_colmajor(inputs.conditioned(4096, 16, seed=0, kappa=kappa))
        info, R, Q = orc.cholqr(A)
        assert info == 0
        errs[kappa] = np.linalg.norm(Q.T @ Q - np.eye(16))
        assert errs[kappa] <= 50 * kappa ** 2 * EPS
        # and the factorisation itself is still backward stable: ||A - QR|| small
        assert np.linalg.norm(A - Q @ R) / np.linalg.norm(A) <= 1e-12
    assert errs[1e5] >= 1e5 * errs[1e2]
    F = A.copy(order="F")
    tau = np.zeros(16)
    orc.lib().orc_hqr(orc._i64(4096), orc._i64(16), orc._d(F), orc._i64(4096), orc._d(tau))
    Qh = _explicit_tile_q(F, tau, 4096, 16)[:, :16]
    assert np.linalg.norm(Qh.T @ Qh - np.eye(16)) <= 1e-13
