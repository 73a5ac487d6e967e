"""Multi-rank (row-sharded) TSQR: the butterfly driver of paper_0808_2664_b200.dist.

CPU (gloo, world size 2 and 4): the SAME round logic as the product (RankState,
torch.distributed point-to-point exchange) runs with an oracle-backed engine; its
per-rank R, Q^T C rows and Q rows must equal the oracle's single global tree over
the same plan (the butterfly of Alg. TSQR:par is the binary tree over
rank roots with every rank holding a replica).

GPU (marked gpu): the product CudaEngine over G virtual ranks in one process on
one GPU (loopback exchange between rounds, no kernel ever waits on another).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as orc
from paper_0808_2664_b200 import dist as tdist
from paper_0808_2664_b200 import inputs


# ------------------------------------------------------------ oracle engine
def _np(t):
    return t.numpy().T


def _node_apply(Y1, tau, Ca, Cb, forward):
    n = Y1.shape[0]
    order = range(n) if forward else range(n - 1, -1, -1)
    for j in order:
        y = Y1[:j + 1, j]
        w = Ca[j] + y @ Cb[:j + 1]
        Ca[j] -= tau[j] * w
        Cb[:j + 1] -= tau[j] * np.outer(y, w)


class OracleTree:
    pass


class OracleEngine:
    """Test-only engine: the oracle's kernels behind the product's engine interface."""

    def factor_local(self, A, b, s, nranks, rank):
        t = OracleTree()
        ml, n = A.shape[1], A.shape[0]
        t.f = orc.tsqr_factor(_np(A), orc.plan(ml, n, b, s, 1))
        t.R = t.f.R.copy()
        t.nranks, t.rank, t.n = nranks, rank, n
        t.cross = []
        R = torch.from_numpy(np.ascontiguousarray(t.R.T))
        return R, t

    def empty(self, shape, like):
        return torch.empty(shape, dtype=torch.float64)

    def pack(self, t, out):
        n = t.n
        out.numpy()[:] = np.concatenate([t.R[:c + 1, c] for c in range(n)])

    def cross_factor(self, t, rnd, recv, R):
        n = t.n
        P = np.zeros((n, n))
        pk = recv.numpy()
        for c in range(n):
            P[:c + 1, c] = pk[c * (c + 1) // 2:(c + 1) * (c + 2) // 2]
        partner = t.rank ^ (1 << (rnd - 1))
        Ra, Rb = (t.R, P) if t.rank < partner else (P, t.R)
        Rn, Y1, tau, _ = orc.combine(Ra, Rb)
        t.cross.append((Y1, tau))
        t.R = Rn
        R.numpy()[:] = Rn.T

    def cross_factor_gathered(self, t, all_packed, R):
        n, G = t.n, t.nranks
        npk = n * (n + 1) // 2
        packs = all_packed.numpy().reshape(G, npk)

        def unpack(pk):
            P = np.zeros((n, n))
            for c in range(n):
                P[:c + 1, c] = pk[c * (c + 1) // 2:(c + 1) * (c + 2) // 2]
            return P

        def group(r, g):                      # R of ranks g*2^r .. (g+1)*2^r - 1
            if r == 0:
                return unpack(packs[g])
            return orc.combine(group(r - 1, 2 * g), group(r - 1, 2 * g + 1))[0]

        for rnd in range(1, int(np.log2(G)) + 1):
            P = group(rnd - 1, (t.rank >> (rnd - 1)) ^ 1)
            pk = torch.from_numpy(np.concatenate([P[:c + 1, c] for c in range(n)]))
            self.cross_factor(t, rnd, pk, R)

    def apply_local(self, t, C, top):
        out = orc.tsqr_apply_qt(t.f, _np(C))
        C.numpy()[:] = out.T
        top.numpy()[:] = out[:t.n].T

    def cross_apply(self, t, rnd, top, ptop, C):
        partner = t.rank ^ (1 << (rnd - 1))
        mine, theirs = _np(top).copy(), _np(ptop).copy()
        Ca, Cb = (mine, theirs) if t.rank < partner else (theirs, mine)
        Y1, tau = t.cross[rnd - 1]
        _node_apply(Y1, tau, Ca, Cb, True)
        top.numpy()[:] = Ca.T
        pos = t.rank & ((1 << rnd) - 1)
        if pos == 0:
            C.numpy()[:, :t.n] = Ca.T
        elif pos == 1 << (rnd - 1):
            C.numpy()[:, :t.n] = Cb.T

    def cross_apply_q(self, t, rnd, top, ptop, C):
        partner = t.rank ^ (1 << (rnd - 1))
        mine, theirs = _np(top).copy(), _np(ptop).copy()
        Ca, Cb = (mine, theirs) if t.rank < partner else (theirs, mine)
        Y1, tau = t.cross[rnd - 1]
        _node_apply(Y1, tau, Ca, Cb, False)
        keep = Ca if t.rank < partner else Cb
        top.numpy()[:] = keep.T
        C.numpy()[:, :t.n] = keep.T

    def apply_q_local(self, t, C):
        out = orc.tsqr_apply_q(t.f, _np(C))
        C.numpy()[:] = out.T

    def form_q(self, t):
        n = t.n
        X = np.eye(n)
        for rnd in range(len(t.cross), 0, -1):
            Y1, tau = t.cross[rnd - 1]
            Xa, Xb = X.copy(), np.zeros((n, n))
            _node_apply(Y1, tau, Xa, Xb, False)
            X = Xa if ((t.rank >> (rnd - 1)) & 1) == 0 else Xb
        ml = t.f.plan.m
        Q0 = np.zeros((ml, n), order="F")
        Q0[:n] = X
        Q = orc.tsqr_apply_q(t.f, Q0)
        return torch.from_numpy(np.ascontiguousarray(Q.T))


# -------------------------------------------------------------- reference
def _global_reference(m, n, b, s, G, k, c=0):
    A = inputs.to_numpy_colmajor(inputs.gaussian(m, n, 0))
    C = inputs.to_numpy_colmajor(inputs.gaussian(m, k, 1))
    f = orc.tsqr_factor(A, orc.plan(m, n, b, s, G, c))
    Z = inputs.to_numpy_colmajor(inputs.gaussian(m, k, 2))
    return f.R, orc.tsqr_apply_qt(f, C.copy()), orc.tsqr_form_q(f), orc.tsqr_apply_q(f, Z)


def _free_port():
    with socket.socket() as sck:
        sck.bind(("127.0.0.1", 0))
        return sck.getsockname()[1]


def _worker(rank, world, port, m, n, b, s, k, q, cross="butterfly"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_0808_2664_b200 import api
        row0, ml = api.slab(m, n, b, world, rank)
        A = inputs.gaussian_rows(row0, ml, n, 0)
        C = inputs.gaussian_rows(row0, ml, k, 1)
        st = tdist.factor(A, b, s, engine=OracleEngine(), cross=cross)
        C0 = C.clone()
        tdist.apply_qt(st, C)
        QtC = C.clone()
        tdist.apply_q(st, C)                                   # back to C0
        back = _np(C).copy()
        Z = inputs.gaussian_rows(row0, ml, k, 2)
        tdist.apply_q(st, Z)
        Q = tdist.form_q(st)
        q.put((rank, row0, ml, _np(st.R).copy(), _np(QtC).copy(), _np(st.top).copy(), _np(Q).copy(), st.sent,
               back, _np(C0).copy(), _np(Z).copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,m,n,b,s,k,cross", [(2, 3000, 12, 500, 250, 7, "butterfly"),
                                                   (4, 5000, 8, 300, 100, 5, "butterfly"),
                                                   (2, 2 * 4096 + 37, 16, 4096, 512, 3, "butterfly"),
                                                   (4, 5000, 8, 300, 100, 5, "allgather")])
def test_butterfly_gloo(world, m, n, b, s, k, cross):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, b, s, k, q, cross)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    Rref, QtC_ref, Qref, QZ_ref = _global_reference(m, n, b, s, world, k)
    rounds = int(np.log2(world))
    for rank, row0, ml, R, C, top, Q, sent, back, C0, QZ in sorted(res, key=lambda x: x[0]):
        assert np.array_equal(R, Rref)                              # replicated and bitwise equal
        assert orc.rel_fro(C, QtC_ref[row0:row0 + ml]) <= 1e-13     # tree-order rows of this rank
        assert orc.rel_fro(top, QtC_ref[:n]) <= 1e-13              # thin part replicated
        assert orc.rel_fro(Q, Qref[row0:row0 + ml]) <= 1e-13
        assert orc.rel_fro(back, C0) <= 1e-13                       # apply_q(apply_qt(C)) = C
        assert orc.rel_fro(QZ, QZ_ref[row0:row0 + ml]) <= 1e-13     # Q Z = the global tree's
        # apply Q: a rank exchanges only in the rounds where it is a group head
        heads = [r for r in range(1, rounds + 1) if tdist.head_role(rank, r)]
        assert sorted(-r for r, _ in sent if r < 0) == sorted(2 * heads)
        if cross == "allgather":                                    # one all-gather of the packed R
            assert [w for r_, w in sent if r_ == 0] == [n * (n + 1) // 2]
            assert [w for r_, w in sent if r_ > 0] == [n * k] * rounds
            continue
        sent = [x for x in sent if x[0] > 0]
        # counts (Table 1; Cor. 2): log2 G messages of n(n+1)/2 words
        fac = [w for r_, w in sent if True][:rounds]
        assert len(sent) == 2 * rounds
        assert all(w == n * (n + 1) // 2 for w in fac)
        assert all(w == n * k for w in [w for _, w in sent][rounds:])


@pytest.mark.parametrize("G,m,n,b,s,k", [(2, 20000, 12, 4096, 512, 5), (4, 9000, 8, 1000, 250, 3)])
def test_butterfly_virtual_oracle(G, m, n, b, s, k):
    """The loopback driver (the one the GPU tests use) with the oracle engine: apply Q^T,
    apply Q (each round's sent buffer is also the partner's receive buffer) and the
    round trip, against the global tree."""
    from paper_0808_2664_b200 import api
    rows = [api.slab(m, n, b, G, r) for r in range(G)]
    eng = OracleEngine()
    states = tdist.factor_virtual([inputs.gaussian_rows(r0, ml, n, 0) for r0, ml in rows], b, s, engine=eng)
    cs = [inputs.gaussian_rows(r0, ml, k, 1) for r0, ml in rows]
    c0 = [C.clone() for C in cs]
    zs = [inputs.gaussian_rows(r0, ml, k, 2) for r0, ml in rows]
    tdist.apply_qt_virtual(states, cs)
    Rref, QtC_ref, Qref, QZ_ref = _global_reference(m, n, b, s, G, k)
    for (r0, ml), C in zip(rows, cs):
        assert orc.rel_fro(_np(C), QtC_ref[r0:r0 + ml]) <= 1e-13
    tdist.apply_q_virtual(states, cs)
    tdist.apply_q_virtual(states, zs)
    for (r0, ml), C, C0, Z in zip(rows, cs, c0, zs):
        assert orc.rel_fro(_np(C), _np(C0)) <= 1e-13
        assert orc.rel_fro(_np(Z), QZ_ref[r0:r0 + ml]) <= 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("G,m,n,b,s", [(8, 50000, 16, 2048, 128), (4, 40000, 50, 4096, 192), (2, 12000, 200, 2048, 2048),
                                       (8, 8 * 4096 + 100, 64, 4096, 96), (4, 16000, 100, 2048, 2048)])
def test_allgather_cross_equals_butterfly_cuda(G, m, n, b, s):
    """The all-gather variant of the cross-GPU combine leaves every rank's tree in the butterfly's
    state: R, Q^T C and Q bitwise equal."""
    from paper_0808_2664_b200 import api
    rows = [api.slab(m, n, b, G, r) for r in range(G)]
    out = {}
    for cross in ("butterfly", "allgather"):
        slabs = [inputs.gaussian_rows(r0, ml, n, 0).cuda() for r0, ml in rows]
        cs = [inputs.gaussian_rows(r0, ml, 7, 1).cuda() for r0, ml in rows]
        states = tdist.factor_virtual(slabs, b, s, cross=cross)
        tdist.apply_qt_virtual(states, cs)
        Qs = [tdist.form_q(st) for st in states]
        torch.cuda.synchronize()
        out[cross] = ([st.R.clone() for st in states], cs, Qs)
        for st in states:
            st.tree.free()
    for x, y in zip(out["butterfly"], out["allgather"]):
        for a_, b_ in zip(x, y):
            assert torch.equal(a_, b_)


@pytest.mark.gpu
@pytest.mark.parametrize("G,m,n,b,s,k", [(2, 20000, 50, 4096, 96, 64), (4, 40000, 32, 4096, 192, 128),
                                         (8, 50000, 16, 2048, 128, 16), (8, 8 * 4096 + 100, 64, 4096, 96, 70), (2, 2 * 4096 + 30, 32, 4096, 64, 32),
                                         (2, 12000, 200, 2048, 2048, 64), (4, 16000, 100, 2048, 2048, 20)])
def test_butterfly_virtual_ranks_cuda(G, m, n, b, s, k):
    from paper_0808_2664_b200 import api
    slabs, cs, rows = [], [], []
    for r in range(G):
        row0, ml = api.slab(m, n, b, G, r)
        rows.append((row0, ml))
        slabs.append(inputs.gaussian_rows(row0, ml, n, 0).cuda())
        cs.append(inputs.gaussian_rows(row0, ml, k, 1).cuda())
    states = tdist.factor_virtual(slabs, b, s)
    c0 = [C.clone() for C in cs]
    tdist.apply_qt_virtual(states, cs)
    Qs = [tdist.form_q(st) for st in states]
    qtc = [C.clone() for C in cs]
    tdist.apply_q_virtual(states, cs)                               # back to C
    zs = [inputs.gaussian_rows(row0, ml, k, 2).cuda() for row0, ml in rows]
    tdist.apply_q_virtual(states, zs)
    torch.cuda.synchronize()
    c = api.plan_info(rows[0][1], n, block_rows=b, tile_rows=s, nranks=G, rank=0)["chunk_rows"]
    Rref, QtC_ref, Qref, QZ_ref = _global_reference(m, n, b, s, G, k, c)
    for st, (row0, ml), C, Q, C0, Cb, Z in zip(states, rows, qtc, Qs, c0, cs, zs):
        R = inputs.to_numpy_colmajor(st.R)
        assert np.array_equal(R, inputs.to_numpy_colmajor(states[0].R))   # bitwise replicated
        assert orc.rel_fro(orc.sign_normalise(R), orc.sign_normalise(Rref)) <= 1e-11
        assert orc.rel_fro(inputs.to_numpy_colmajor(C), QtC_ref[row0:row0 + ml]) <= 1e-11
        assert orc.rel_fro(inputs.to_numpy_colmajor(st.top), QtC_ref[:n]) <= 1e-11
        assert orc.rel_fro(inputs.to_numpy_colmajor(Q), Qref[row0:row0 + ml]) <= 1e-11
        assert orc.rel_fro(inputs.to_numpy_colmajor(Cb), inputs.to_numpy_colmajor(C0)) <= 1e-13
        assert orc.rel_fro(inputs.to_numpy_colmajor(Z), QZ_ref[row0:row0 + ml]) <= 1e-11
    for st in states:
        st.tree.free()
