"""Subtree-sharded factorization across ranks.

Nested-dissection subtrees are independent: every rank factors the subtrees
it owns with no communication; the few fronts above the cut (the "top") are
dealt to ranks height by height so siblings factor in parallel. The exchange
step is a child update crossing ranks: after each height with such an edge,
each such update travels from the child's owner to the parent's owner only,
point to point, in its own compressed form -- the reference's UpdateRep
(hodlr.py:429-470): the update HODLR's leaves and low-rank / dense blocks
behind a node table whose pointers are offsets, then W and V^T -- and the
receiver rebases the table, so the parent's sampler reads exactly the numbers
it reads on one GPU (multifrontal.py:329-348). ``compressed=False`` keeps the
earlier path: every cut update densified and all-reduced to every rank. The preconditioner apply
(mf_solve, multifrontal.py:533-560) runs the global apply levels on each
rank's fronts and all-reduces the contribution buffer (upward) and x
(downward) only at level boundaries where a dependency crosses ranks, then x
once more at the end: every rank holds the full solution, bitwise equal to the
single-GPU factor's. GMRES (krylov.py:68-161) runs replicated on every rank on
top of that apply.

Collectives go through torch.distributed: NCCL directly on the library's CUDA
stream (device buffers, stream ordered), or gloo through host staging (tests).
"""
from __future__ import annotations

import ctypes as C
import traceback

import numpy as np

from .ordering import etree_handle
from . import _lib
from .multifrontal import ACCELERATED, CONVENTIONAL, MfFactorization, MfParams, mf_factorize
from .sparse import SparseMatrix


def subtree_costs(tree):
    """Per-node work proxy (front_size^2 * max(n_pivot, 1)) and its subtree sums."""
    nodes = tree.nodes
    n_nodes = len(nodes)
    own = np.zeros(n_nodes)
    sub = np.zeros(n_nodes)
    for v in tree.post_order:
        nd = nodes[v]
        own[v] = float(nd.front_size) ** 2 * max(nd.n_pivot, 1)
        sub[v] = own[v] + sum(sub[c] for c in nd.children)
    return own, sub


class SubtreePartition:
    """Owner rank for every elimination-tree node.

    The largest piece is split (its root joins the top, its children become
    pieces) until there are at least 2*world pieces and no piece exceeds an
    equal share; pieces (whole subtrees) are dealt largest-first to the least
    loaded rank (LPT). Top nodes are then dealt height by height, children
    before parents, balancing each height's work across ranks so sibling top
    fronts factor in parallel. Deterministic: every rank computes the same cut."""

    def __init__(self, tree, world, max_splits=None):
        if world < 1:
            raise ValueError("world size must be positive")
        self.world = world
        nodes = tree.nodes
        own, sub = subtree_costs(tree)
        self.top = []
        pieces = [] if tree.root is None else [tree.root]
        max_splits = max_splits if max_splits is not None else 64 * world
        if world > 1:
            splits = 0
            while pieces and splits < max_splits:
                total = sum(sub[p] for p in pieces)
                big = max(pieces, key=lambda v: (sub[v], -v))
                if len(pieces) >= 2 * world and sub[big] <= total / world:
                    break
                kids = list(nodes[big].children)
                if not kids:
                    break
                pieces.remove(big)
                self.top.append(big)
                pieces.extend(kids)
                splits += 1
        load = [0.0] * world
        self.owner = {}
        for p in sorted(pieces, key=lambda v: (-sub[v], v)):
            r = min(range(world), key=lambda q: (load[q], q))
            self.owner[p] = r
            load[r] += sub[p]
        n_nodes = len(nodes)
        self.node_owner = np.full(n_nodes, -1, dtype=np.int64)
        for p, r in self.owner.items():
            stack = [p]
            while stack:
                v = stack.pop()
                self.node_owner[v] = r
                stack.extend(nodes[v].children)
        # top nodes by height (children first), balanced per height
        height = {}
        for v in tree.post_order:
            height[v] = 1 + max((height[c] for c in nodes[v].children), default=-1)
        by_h = {}
        for v in self.top:
            by_h.setdefault(height[v], []).append(v)
        for h in sorted(by_h):
            at_h = [0.0] * world
            for v in sorted(by_h[h], key=lambda v: (-own[v], v)):
                r = min(range(world), key=lambda q: (at_h[q], load[q], q))
                self.node_owner[v] = r
                at_h[r] += own[v]
                load[r] += own[v]
        self.load = load
        self.pieces = pieces

    def owners(self):
        """int32 owner rank per etree node id (the mfh_shard_t owner array)."""
        return self.node_owner.astype(np.int32)


class _CudaArray:
    def __init__(self, ptr, count):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


class TorchExchange:
    """mfh_exchange_fn over a torch.distributed group: in-place all-reduce SUM
    of a device buffer that the library produced on its stream."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self.group = group
        self.device_collective = dist.get_backend(group) == "nccl"
        ctx = _lib.context()
        self.stream = torch.cuda.ExternalStream(ctx.info()[0])
        self.calls = 0
        self.bytes = 0
        self.p2p_calls = 0
        self.p2p_bytes = 0
        self.cfn = _lib.EXCHANGE_FN(self._call)
        self.pfn = _lib.P2P_FN(self._p2p)

    def _call(self, user, dptr, count):
        import torch
        import torch.distributed as dist
        try:
            t = torch.as_tensor(_CudaArray(dptr, count), device="cuda")
            with torch.cuda.stream(self.stream):
                if self.device_collective:
                    dist.all_reduce(t, group=self.group)  # stream ordered on the library stream
                else:
                    h = t.cpu()
                    dist.all_reduce(h, group=self.group)
                    t.copy_(h)
                    self.stream.synchronize()
            self.calls += 1
            self.bytes += 8 * int(count)
            return 0
        except Exception:  # the library turns a nonzero return into an error
            traceback.print_exc()
            return 1


    def _p2p(self, user, nops, bufs, counts, peers, sends):
        """mfh_p2p_fn: one group of sends / receives of device buffers (NCCL
        batch_isend_irecv on the library stream, or gloo through host staging)."""
        import torch
        import torch.distributed as dist
        try:
            ts = [torch.as_tensor(_CudaArray(bufs[i], counts[i]), device="cuda") for i in range(nops)]
            with torch.cuda.stream(self.stream):
                if self.device_collective:
                    ops = [dist.P2POp(dist.isend if sends[i] else dist.irecv, ts[i], int(peers[i]), group=self.group)
                           for i in range(nops)]
                    for w in dist.batch_isend_irecv(ops):
                        w.wait()
                else:
                    self.stream.synchronize()
                    host = [t.cpu() if sends[i] else torch.empty(int(counts[i]), dtype=torch.float64)
                            for i, t in enumerate(ts)]
                    reqs = [(dist.isend if sends[i] else dist.irecv)(host[i], int(peers[i]), group=self.group)
                            for i in range(nops)]
                    for r in reqs:
                        r.wait()
                    for i in range(nops):
                        if not sends[i]:
                            ts[i].copy_(host[i])
                    self.stream.synchronize()
            self.p2p_calls += 1
            self.p2p_bytes += 8 * sum(int(counts[i]) for i in range(nops) if sends[i])
            return 0
        except Exception:
            traceback.print_exc()
            return 1


def mf_factorize_sharded(A, tree, mode=ACCELERATED, params=None, group=None, partition=None, compressed=True):
    """mf_factorize over torch.distributed ranks: this rank's subtrees and top
    fronts; returns a factorization whose stats cover the whole tree and whose
    apply / GMRES return the full solution on every rank."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return mf_factorize(A, tree, mode, params)
    rank = dist.get_rank(group)
    if mode not in (CONVENTIONAL, ACCELERATED):
        raise ValueError(f"unknown mode '{mode}'")
    params = params or MfParams()
    if not isinstance(A, SparseMatrix):
        A = SparseMatrix(A)
    part = partition or SubtreePartition(tree, world)
    owners = part.owners()
    ex = TorchExchange(group)
    sh = _lib.mfh_shard_t(owners.ctypes.data_as(C.POINTER(C.c_int32)), rank, ex.cfn, None,
                          ex.pfn if compressed else _lib.P2P_FN())
    ctx = _lib.context()
    ip, ix, dv = A.csr_arrays()
    p = _lib.mfh_params(int(min(params.n_c, 2**62)), float(params.eps), int(params.d),
                        int(params.n_leaf), -1 if params.max_rank is None else int(params.max_rank))
    h = C.c_void_p()
    _lib.check(_lib.lib().mfh_factorize_sharded(ctx.handle, etree_handle(tree), A.n_rows, _lib.ptr(ip), _lib.ptr(ix),
                                                _lib.ptr(dv), 1 if mode == ACCELERATED else 0, C.byref(p),
                                                C.byref(sh), C.byref(h)))
    F = MfFactorization(h, mode, params, tree, ctx)
    F._shard = (ex, owners, sh, part)  # the callback and owner array live as long as the factor
    F.partition = part
    F.exchange = ex
    return F


def gmres_sharded(A, b, F, tol=1e-6, max_iter=4000, restart=100):
    """GMRES distributed over the ranks of a sharded factorization
    (``mfh_gmres_sharded``): each rank owns the rows and Krylov-vector entries
    of its pivots, SpMV reads the coupled entries of other ranks from an
    all-reduced halo buffer, Gram-Schmidt is CGS2 with one all-reduce of the
    dot products per pass. Collective; every rank passes the same ``A`` and
    ``b`` and gets the whole solution (krylov.py:68-161 semantics; iteration
    counts within one of ``gmres``)."""
    from .krylov import ConvergenceHistory
    if not getattr(F, "_shard", None):
        raise ValueError("gmres_sharded needs a factorization from mf_factorize_sharded")
    if not isinstance(A, SparseMatrix):
        A = SparseMatrix(A)
    b = np.ascontiguousarray(b, dtype=np.float64)
    n = A.n_rows
    x = np.empty(n)
    ip, ix, dv = A.csr_arrays()
    hist = np.empty(max(1, int(max_iter)))
    nh, its, conv = C.c_int64(), C.c_int64(), C.c_int()
    _lib.check(_lib.lib().mfh_gmres_sharded(F._h, n, _lib.ptr(ip), _lib.ptr(ix), _lib.ptr(dv), _lib.ptr(b),
                                            _lib.ptr(x), float(tol), int(max_iter), int(restart), _lib.ptr(hist),
                                            C.byref(nh), C.byref(its), C.byref(conv)))
    return x, ConvergenceHistory([float(v) for v in hist[:nh.value]], bool(conv.value), int(its.value))
