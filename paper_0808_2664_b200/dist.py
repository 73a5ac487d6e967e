"""Row-sharded multi-GPU TSQR: Alg. TSQR:par as a butterfly all-reduction
(butterfly indices P:3955-3975).

One process per GPU.  Each rank factors its contiguous slab of whole row blocks
(tsqr_slab) with the single-GPU kernels, then runs log2(G) rounds: pack the
current R (n(n+1)/2 words, the Cor. 2 minimum), exchange it with
partner r XOR 2^(k-1) over NCCL (torch.distributed point-to-point, NVLink), and
run the structured combine on [R_lower; R_upper] -- both partners compute the
same node, so R ends replicated.  Apply Q^T exchanges the n x k
R coordinates per round, apply Q (its inverse) the same between the group heads;
form Q needs no communication (every rank holds the
node factors on its root-to-leaf path).

Product path (NCCL process group, the default engine): a thin caller of the
C-ABI's communicator layer -- rank 0's NCCL unique id is broadcast over the
process group, every rank joins a libtsqr context (tsqr_ctx_set_comm), and each
operation is ONE collective C call that runs every round inside the library
(grouped ncclSend/ncclRecv on the call's stream; `CtxState`).

Test path: the same round logic written in Python (`RankState`), driven by
torch.distributed point-to-point (gloo, `factor`, `apply_qt`) or by an
in-process loopback over virtual ranks (`*_virtual`), with the arithmetic of an
engine: `CudaEngine` calls libtsqr.so's per-round entry points; the CPU tests
substitute an oracle-backed engine.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import api


class CudaEngine:
    """The product engine: every step is a libtsqr.so call on the current stream.
    stage_timing: record device events around the local leaf / tree stages (Tree.stage_ms)."""

    def __init__(self, stage_timing: bool = False):
        self.stage_timing = stage_timing

    def factor_local(self, A, block_rows, tile_rows, nranks, rank, tree=None):
        return api.factor(A, block_rows, tile_rows, nranks=nranks, rank=rank, tree=tree,
                          stage_timing=self.stage_timing)

    def empty(self, shape, like):
        return torch.empty(shape, dtype=torch.float64, device=like.device)

    def pack(self, tree, out):
        return api.pack_r(tree, out)

    def cross_factor(self, tree, rnd, recv, R):
        api.cross_factor(tree, rnd, recv, R)

    def cross_factor_gathered(self, tree, all_packed, R):
        api.cross_factor_gathered(tree, all_packed, R)

    def apply_local(self, tree, C, top):
        api.apply_qt(tree, C, top)

    def cross_apply(self, tree, rnd, top, partner_top, C):
        api.cross_apply_qt(tree, rnd, top, partner_top, C)

    def cross_apply_q(self, tree, rnd, top, partner_top, C):
        api.cross_apply_q(tree, rnd, top, partner_top, C)

    def apply_q_local(self, tree, C):
        api.apply_q(tree, C)

    def form_q(self, tree):
        return api.form_q(tree)


def head_role(rank: int, rnd: int) -> int:
    """1: leftmost rank of the 2^rnd group (lower half), 2: leftmost of its upper half, 0: other
    (tsqr_cross_partner's head_role)."""
    pos = rank & ((1 << rnd) - 1)
    return 1 if pos == 0 else (2 if pos == 1 << (rnd - 1) else 0)


def rounds_of(nranks: int) -> int:
    r = 0
    while (1 << r) < nranks:
        r += 1
    if (1 << r) != nranks:
        raise ValueError("nranks must be a power of two")
    return r


@dataclass
class RankState:
    engine: object
    rank: int
    nranks: int
    n: int = 0
    tree: object = None
    R: object = None
    top: object = None
    C: object = None
    sent: list = field(default_factory=list)      # (round, words) per message, for the count pins

    # ---------------------------------------------------------------- factor
    def factor_local(self, A, block_rows, tile_rows, tree=None):
        self.n = A.shape[0]
        if tree is None:
            self.R, self.tree = self.engine.factor_local(A, block_rows, tile_rows, self.nranks, self.rank)
        else:                                        # reuse a previous factor's workspace
            self.R, self.tree = self.engine.factor_local(A, block_rows, tile_rows, self.nranks, self.rank, tree=tree)

    def factor_send(self, rnd):
        buf = self.engine.empty((self.n * (self.n + 1) // 2,), self.R)
        self.engine.pack(self.tree, buf)
        self.sent.append((rnd, buf.numel()))
        return buf

    def factor_finish(self, rnd, recv):
        self.engine.cross_factor(self.tree, rnd, recv, self.R)

    def factor_gathered_finish(self, all_packed):
        # every round from the all-gathered leaf R's (the factor_send(0) of every rank)
        self.engine.cross_factor_gathered(self.tree, all_packed, self.R)

    # ----------------------------------------------------------------- apply
    def apply_local(self, C):
        k = C.shape[0]
        self.C = C
        self.top = self.engine.empty((k, self.n), C)
        self.engine.apply_local(self.tree, C, self.top)

    def apply_send(self, rnd):
        buf = self.top.clone()
        self.sent.append((rnd, buf.numel()))
        return buf

    def apply_finish(self, rnd, recv):
        self.engine.cross_apply(self.tree, rnd, self.top, recv, self.C)

    # ------------------------------------------------------ apply Q (reverse)
    # Rounds log2 G .. 1: in round k only the two group heads take part -- the
    # lower holds the group's R coordinates, the upper this node's complement
    # (both in their C head rows, where apply_qt left them); each keeps its half of
    # Q_node [lower; upper], which is its subgroup's R coordinates one round down.
    def apply_q_send(self, rnd, C):
        if head_role(self.rank, rnd) == 0:
            return None
        buf = C[:, :self.n].contiguous()                  # n x k head rows, ld n
        self.sent.append((-rnd, buf.numel()))
        return buf

    def apply_q_finish(self, rnd, recv, C):
        mine = C[:, :self.n].contiguous()                 # the sent buffer may be the partner's recv
        self.engine.cross_apply_q(self.tree, rnd, mine, recv, C)


@dataclass
class CtxState:
    """A factor done by the C communicator layer (tsqr_ctx_factor): R replicated."""
    ctx: object
    tree: object
    R: object
    rank: int
    nranks: int
    top: object = None


_CTX = {}


def nccl_ctx(group=None):
    """The libtsqr context of this process for `group` (NCCL backend), created once:
    rank 0's ncclUniqueId is broadcast over the group, then every rank joins."""
    import torch.distributed as dist
    key = id(group)
    if key not in _CTX:
        rank, nranks = dist.get_rank(group), dist.get_world_size(group)
        box = [api.Ctx.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0, group=group)
        _CTX[key] = api.Ctx(torch.cuda.current_device()).set_comm(box[0], nranks, rank)
    return _CTX[key]


def _use_ctx(engine, group, cross) -> bool:
    import torch.distributed as dist
    return (engine is None or type(engine) is CudaEngine) and cross == "butterfly" and \
        dist.get_backend(group) == "nccl"


def _exchange(send: torch.Tensor, partner: int, group=None) -> torch.Tensor:
    import torch.distributed as dist
    if send.is_cuda and dist.get_backend(group) == "gloo":
        # gloo moves host memory only: stage a device buffer through the host
        return _exchange(send.cpu(), partner, group).to(send.device)
    recv = torch.empty_like(send)
    ops = [dist.P2POp(dist.isend, send, partner, group), dist.P2POp(dist.irecv, recv, partner, group)]
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    return recv


def _all_gather(send: torch.Tensor, group=None) -> torch.Tensor:
    import torch.distributed as dist
    if send.is_cuda and dist.get_backend(group) == "gloo":
        return _all_gather(send.cpu(), group).to(send.device)
    G = dist.get_world_size(group)
    if dist.get_backend(group) == "nccl":
        out = torch.empty((G * send.numel(),), dtype=send.dtype, device=send.device)
        dist.all_gather_into_tensor(out, send, group=group)
        return out
    parts = [torch.empty_like(send) for _ in range(G)]
    dist.all_gather(parts, send, group=group)
    return torch.cat(parts)


# ------------------------------------------------------ torch.distributed drivers
def factor(A_local, block_rows: int, tile_rows: int = 0, engine=None, group=None, tree=None,
           cross: str = "butterfly") -> RankState:
    """Collective over the process group: returns the rank state (R replicated in .R).
    tree: a previous factor's tree of the same shape, whose workspace is reused.
    cross: "butterfly" (log2 G pairwise exchanges) or "allgather" (one all-gather of the
    packed leaf R's, the rounds recomputed locally; bitwise the same R and tree state)."""
    import torch.distributed as dist
    rank, nranks = dist.get_rank(group), dist.get_world_size(group)
    if _use_ctx(engine, group, cross):             # product path: one collective C call
        ctx = nccl_ctx(group)
        R, t = ctx.factor(A_local, block_rows, tile_rows, tree=tree,
                          stage_timing=bool(engine is not None and engine.stage_timing))
        return CtxState(ctx, t, R, rank, nranks)
    st = RankState(engine or CudaEngine(), rank, nranks)
    st.factor_local(A_local, block_rows, tile_rows, tree)
    if cross == "allgather":
        if nranks > 1:
            st.factor_gathered_finish(_all_gather(st.factor_send(0), group))
        return st
    if cross != "butterfly":
        raise ValueError("cross must be 'butterfly' or 'allgather'")
    for rnd in range(1, rounds_of(nranks) + 1):
        partner = rank ^ (1 << (rnd - 1))
        recv = _exchange(st.factor_send(rnd), partner, group)
        st.factor_finish(rnd, recv)
    return st


def apply_qt(st: RankState, C_local, group=None):
    """Collective: C_local <- rows of Q^T C (tree order); st.top = Q_thin^T C on every rank."""
    if isinstance(st, CtxState):
        st.top = torch.empty((C_local.shape[0], st.R.shape[0]), dtype=torch.float64, device=C_local.device)
        st.ctx.apply_qt(st.tree, C_local, st.top)
        return C_local, st.top
    st.apply_local(C_local)
    for rnd in range(1, rounds_of(st.nranks) + 1):
        partner = st.rank ^ (1 << (rnd - 1))
        recv = _exchange(st.apply_send(rnd), partner, group)
        st.apply_finish(rnd, recv)
    return C_local, st.top


def apply_q(st: RankState, C_local, group=None):
    """Collective: C_local <- rows of Q C, C in tree order (the inverse of apply_qt)."""
    if isinstance(st, CtxState):
        return st.ctx.apply_q(st.tree, C_local)
    for rnd in range(rounds_of(st.nranks), 0, -1):
        send = st.apply_q_send(rnd, C_local)
        if send is None:
            continue
        recv = _exchange(send, st.rank ^ (1 << (rnd - 1)), group)
        st.apply_q_finish(rnd, recv, C_local)
    st.engine.apply_q_local(st.tree, C_local)
    return C_local


def form_q(st: RankState):
    """Local (communication-free) explicit Q rows of this rank."""
    if isinstance(st, CtxState):
        return st.ctx.form_q(st.tree)
    return st.engine.form_q(st.tree)


# ------------------------------------------------------- loopback (virtual) drivers
def factor_virtual(slabs, block_rows: int, tile_rows: int = 0, engine=None, cross: str = "butterfly") -> list:
    """All ranks in one process, exchanging by reference between rounds (no kernel of one
    rank ever waits on another's: each round's sends are complete before any finish)."""
    nranks = len(slabs)
    eng = engine or CudaEngine()
    states = [RankState(eng, r, nranks) for r in range(nranks)]
    for st, A in zip(states, slabs):
        st.factor_local(A, block_rows, tile_rows)
    if cross == "allgather":
        if nranks > 1:
            all_packed = torch.cat([st.factor_send(0) for st in states])
            for st in states:
                st.factor_gathered_finish(all_packed)
        return states
    for rnd in range(1, rounds_of(nranks) + 1):
        sends = [st.factor_send(rnd) for st in states]
        for st in states:
            st.factor_finish(rnd, sends[st.rank ^ (1 << (rnd - 1))])
    return states


def apply_qt_virtual(states, C_slabs):
    for st, C in zip(states, C_slabs):
        st.apply_local(C)
    for rnd in range(1, rounds_of(len(states)) + 1):
        sends = [st.apply_send(rnd) for st in states]
        for st in states:
            st.apply_finish(rnd, sends[st.rank ^ (1 << (rnd - 1))])
    return C_slabs


def apply_q_virtual(states, C_slabs):
    for rnd in range(rounds_of(len(states)), 0, -1):
        sends = [st.apply_q_send(rnd, C) for st, C in zip(states, C_slabs)]
        for st, C in zip(states, C_slabs):
            if sends[st.rank] is not None:
                st.apply_q_finish(rnd, sends[st.rank ^ (1 << (rnd - 1))], C)
    for st, C in zip(states, C_slabs):
        st.engine.apply_q_local(st.tree, C)
    return C_slabs
