"""Subtree-partitioned multi-GPU compression.

One process per GPU; G = 2^lg ranks.  Rank g owns the level-lg node
2^lg - 1 + g, i.e. the contiguous rows [begin, end) of that node, and
receives only those rows of Omega, Psi, Y, Z.  It compresses its subtree
(levels L .. lg, every per-node computation identical to the single-GPU
sweep), producing its level-lg node's lifted half: 4 x (r x s) fp64
(compress.py:209-219).  One all-gather of those halves (393 KB per rank at
config 4) gives every rank the level-(lg-1) quadruple; the few top levels
(2^lg - 2 nodes) and the root are then finished redundantly on every rank,
so no rank waits on another afterwards.  Per-node arithmetic is unchanged,
so the gathered factorization equals the single-GPU one bit for bit.

The per-level work is delegated to an engine: `CudaEngine` (the product
path, `CompressPlan` on the rank's device).  Tests substitute a CPU engine to
exercise this host logic with the gloo backend.
"""

from dataclasses import dataclass

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _native
from .compress import CompressionConfig, CompressPlan, _check_configuration, raise_ill_conditioned
from .errors import ConfigurationError
from .factorization import LevelGeometry
from .tree import ClusterTree


class SubtreePartition:
    """Row range and per-level geometry of rank `rank` of `world`."""

    def __init__(self, tree: ClusterTree, world: int, rank: int, r: int):
        if world < 1 or world & (world - 1):
            raise ConfigurationError(f"world size must be a power of two, got {world}")
        lg = world.bit_length() - 1
        if lg >= tree.depth:
            raise ConfigurationError(f"{world} ranks need a tree deeper than {tree.depth} levels")
        self.tree, self.world, self.rank, self.r, self.lg = tree, world, rank, r, lg
        top = tree.level_begin(lg)
        self.begin, self.end = int(top[rank]), int(top[rank + 1])
        self.local_specs = []
        for level in range(tree.depth, max(lg, 1) - 1, -1):
            nb = 1 << (level - lg)
            first = rank * nb
            if level == tree.depth:
                begins = tree.level_begin(level)[first:first + nb + 1] - self.begin
            else:
                begins = np.arange(nb + 1, dtype=np.int64) * 2 * r
            self.local_specs.append((level, begins, first))
        self.top_specs = [(level, np.arange((1 << level) + 1, dtype=np.int64) * 2 * r, 0)
                          for level in range(lg - 1, 0, -1)]

    @property
    def rows(self) -> int:
        return self.end - self.begin


@dataclass
class EngineResult:
    """Packed per-level blocks (same layout as CompressPlan / include/hbs_b200.h)."""
    levels: dict          # level -> (U (rows x r), V (rows x r), D flat)
    begins: dict          # level -> row starts (numpy, relative)
    first_box: dict       # level -> global index of the first box
    top_quad: tuple       # lifted quadruple of the last compressed level
    root: object          # 2r x 2r core or None
    failure: object       # (level, node id) of the first failing node, or None


class CudaEngine:
    """Product engine: one CompressPlan on the current CUDA device."""

    def __init__(self, device=None):
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())

    def run(self, tree, specs, quad, s, r, tol, with_root):
        plan = CompressPlan(tree, s, r, tol, device=self.device, specs=specs, with_root=with_root)
        if specs:
            plan.run(*quad)
        else:
            plan.top_quad = tuple(quad)
            if with_root:
                plan.run_root(quad[0], quad[2])
        return EngineResult(levels={lv: plan.levels[lv] for lv, _, _ in specs},
                            begins={lv: b for lv, b, _ in specs}, first_box={lv: f for lv, _, f in specs},
                            top_quad=plan.top_quad, root=plan.root if with_root else None,
                            failure=plan.first_failure())

    def as_tensor(self, a):
        return a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a)).to(self.device)


def _all_gather_flat(out, inp, group):
    """all_gather_into_tensor over NCCL; over other backends (gloo: the CPU
    multi-process tests, or CUDA ranks without NCCL) the tensors are staged
    through host memory."""
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, inp, group=group)
        return out
    world = dist.get_world_size(group)
    host = inp.detach().cpu().contiguous()
    parts = [torch.empty_like(host) for _ in range(world)]
    dist.all_gather(parts, host, group=group)
    out.copy_(torch.cat(parts).to(out.device))
    return out


def _agree_on_failure(fail, group):
    """All ranks adopt the first failure in sweep order (deepest level,
    lowest node id) so they raise the same IllConditionedProbeError."""
    world = dist.get_world_size(group)
    code = torch.tensor([-1 if fail is None else fail[0], -1 if fail is None else fail[1]], dtype=torch.int64)
    if dist.get_backend(group) == "nccl":
        code = code.cuda()
    out = [torch.empty_like(code) for _ in range(world)]
    dist.all_gather(out, code, group=group)
    cands = [(int(t[0]), int(t[1])) for t in out if int(t[0]) >= 0]
    if not cands:
        return None
    level = max(c[0] for c in cands)
    return level, min(c[1] for c in cands if c[0] == level)


def compress_distributed(local_samples, tree: ClusterTree, config: CompressionConfig, group=None, engine=None):
    """Compress with subtree partitioning across the ranks of `group`.

    `local_samples` = (omega, psi, y, z) restricted to this rank's rows
    (SubtreePartition.begin .. end).  Returns a DistributedFactorization whose
    top levels and root are replicated on every rank."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    engine = engine or CudaEngine()
    quad = tuple(engine.as_tensor(m) for m in local_samples)
    s, r, tol = quad[0].shape[1], config.rank, config.ill_conditioning_tol
    _check_configuration(tree, s, r)
    part = SubtreePartition(tree, world, rank, r)
    if quad[0].shape[0] != part.rows:
        raise ConfigurationError(f"rank {rank} owns rows [{part.begin}, {part.end}) but got {quad[0].shape[0]}")
    local = engine.run(tree, part.local_specs, quad, s, r, tol, with_root=(world == 1))
    if world == 1:
        if local.failure is not None:
            raise_ill_conditioned(*local.failure, tol)
        return DistributedFactorization(part, local, None)
    fail = _agree_on_failure(local.failure, group)
    if fail is not None:
        raise_ill_conditioned(*fail, tol)
    # one all-gather of the level-lg lifted halves: (world, 4, r, s)
    half = torch.stack([m.reshape(r, s) for m in local.top_quad]).contiguous().reshape(-1)
    gathered = torch.empty(world * half.numel(), dtype=half.dtype, device=half.device)
    _all_gather_flat(gathered, half, group)
    gathered = gathered.reshape(world, 4, r, s)
    top_quad = tuple(gathered[:, i].reshape(world * r, s).contiguous() for i in range(4))
    top = engine.run(tree, part.top_specs, top_quad, s, r, tol, with_root=True)
    if top.failure is not None:
        raise_ill_conditioned(*top.failure, tol)
    return DistributedFactorization(part, local, top)


class DistributedFactorization:
    """This rank's subtree blocks plus the replicated top levels and root."""

    def __init__(self, partition, local: EngineResult, top):
        self.partition, self.local, self.top = partition, local, top

    @property
    def root(self):
        return (self.top or self.local).root

    def host_blocks(self, result: EngineResult):
        """{node id: (U, V, D)} as numpy for one engine result."""
        out = {}
        r = self.partition.r
        for level, (u, v, d) in result.levels.items():
            b = result.begins[level]
            u, v, d = (t.cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t) for t in (u, v, d))
            sq = 0
            for j in range(b.size - 1):
                lo, hi = int(b[j] - b[0]), int(b[j + 1] - b[0])
                rows = hi - lo
                nid = (1 << level) - 1 + result.first_box[level] + j
                out[nid] = (u[lo:hi], v[lo:hi], d[sq:sq + rows * rows].reshape(rows, rows))
                sq += rows * rows
        del r
        return out

    def gather(self, group=None):
        """All blocks of the whole tree on every rank: ({node id: (U, V, D)}, root) as numpy."""
        blocks = self.host_blocks(self.local)
        if self.top is not None:
            blocks.update(self.host_blocks(self.top))
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        if world > 1:
            parts = [None] * world
            dist.all_gather_object(parts, blocks, group=group)
            blocks = {}
            for p in parts:
                blocks.update(p)
        root = self.root
        root = root.cpu().numpy() if isinstance(root, torch.Tensor) else np.asarray(root)
        return blocks, root


def compress_partitioned_on_one_device(samples, tree: ClusterTree, config: CompressionConfig, world: int,
                                       engine=None):
    """Run the `world` subtrees one after another on one device and replace the
    all-gather with a concatenation -- the single-GPU emulation of
    compress_distributed (same per-level geometry, no collective).  Returns
    ({node id: (U, V, D)}, root) as numpy."""
    engine = engine or CudaEngine()
    quad = tuple(engine.as_tensor(m) for m in samples)
    s, r, tol = quad[0].shape[1], config.rank, config.ill_conditioning_tol
    _check_configuration(tree, s, r)
    blocks, halves = {}, []
    for rank in range(world):
        part = SubtreePartition(tree, world, rank, r)
        local = engine.run(tree, part.local_specs, tuple(m[part.begin:part.end] for m in quad), s, r, tol,
                           with_root=(world == 1))
        if local.failure is not None:
            raise_ill_conditioned(*local.failure, tol)
        blocks.update(DistributedFactorization(part, local, None).host_blocks(local))
        halves.append(local.top_quad)
        if world == 1:
            root = local.root
            return blocks, (root.cpu().numpy() if isinstance(root, torch.Tensor) else np.asarray(root))
    top_quad = tuple(torch.cat([h[i] for h in halves]) for i in range(4))
    part = SubtreePartition(tree, world, 0, r)
    top = engine.run(tree, part.top_specs, top_quad, s, r, tol, with_root=True)
    if top.failure is not None:
        raise_ill_conditioned(*top.failure, tol)
    blocks.update(DistributedFactorization(part, top, None).host_blocks(top))
    root = top.root
    return blocks, (root.cpu().numpy() if isinstance(root, torch.Tensor) else np.asarray(root))


# ---------------------------------------------------------------------------
# Distributed telescoping operator (the HBS sampler of SURVEY 8(e)) and a
# preallocated distributed compressor for repeated runs (bench.py).
# ---------------------------------------------------------------------------

def _level_arrays(geo: dict, blocks: dict, lo: int, hi: int, which: int):
    n = hi + 1
    nbox = (ctypes.c_int64 * n)()
    rb = _native.ptr_array([0] * n)
    sq = _native.ptr_array([0] * n)
    bp = _native.ptr_array([0] * n)
    for lv in range(lo, hi + 1):
        nbox[lv] = geo[lv].nbox
        rb[lv] = geo[lv].row_begin.data_ptr()
        sq[lv] = geo[lv].sq_off.data_ptr()
        bp[lv] = blocks[lv][which].data_ptr()
    return nbox, rb, sq, bp


class DistributedOperator:
    """A telescoping factorization split by subtree: this rank's levels
    lg..L (its boxes only) plus the replicated top levels 1..lg-1 and root.
    `apply` is the distributed sampler: local upward pass, one all-gather of
    qhat at level lg (r x c per rank), the top levels on every rank, then the
    local downward pass (factorization.py:89-143 split at level lg)."""

    def __init__(self, partition: SubtreePartition, local_blocks: dict, local_geo: dict, top_blocks: dict,
                 top_geo: dict, root, group=None):
        self.part, self.group = partition, group
        self.local_blocks, self.local_geo = local_blocks, local_geo
        self.top_blocks, self.top_geo, self.root = top_blocks, top_geo, root
        self.device = root.device

    # the three phases of `apply`, exposed so that a single-device test can
    # emulate several ranks (concatenation in place of the all-gather)
    def up_local(self, q, transpose=False):
        part, r = self.part, self.part.r
        L, lo = part.tree.depth, max(part.lg, 1)
        c = q.shape[1]
        f64 = dict(dtype=torch.float64, device=self.device)
        qhat = {lv: torch.empty(self.local_geo[lv].nbox * r, c, **f64) for lv in range(lo, L + 1)}
        nbox, rb, sq, bp = _level_arrays(self.local_geo, self.local_blocks, lo, L, 0 if transpose else 1)
        qp = _native.ptr_array([0] * (L + 1))
        for lv in range(lo, L + 1):
            qp[lv] = qhat[lv].data_ptr()
        st = torch.cuda.current_stream(self.device).cuda_stream
        _native.check(_native.lib().hbs_apply_up(L, lo, r, c, nbox, rb, sq, bp, q.data_ptr(), qp, st),
                      "hbs_apply_up")
        return qhat

    def top(self, qtop, transpose=False):
        """qtop: level-lg qhat of all ranks ((world r) x c, rank order) -> uhat at level lg, all ranks."""
        part, r, lg = self.part, self.part.r, self.part.lg
        c = qtop.shape[1]
        lib, st = _native.lib(), torch.cuda.current_stream(self.device).cuda_stream
        f64 = dict(dtype=torch.float64, device=self.device)
        tq = {lv: torch.empty((1 << lv) * r, c, **f64) for lv in range(1, lg)}
        tu = {lv: torch.empty((1 << lv) * r, c, **f64) for lv in range(1, lg + 1)}
        tqp, tup = _native.ptr_array([0] * (lg + 1)), _native.ptr_array([0] * (lg + 1))
        for lv in range(1, lg):
            tqp[lv] = tq[lv].data_ptr()
        for lv in range(1, lg + 1):
            tup[lv] = tu[lv].data_ptr()
        q1 = qtop
        if lg >= 2:
            tn, trb, tsq, tbp = _level_arrays(self.top_geo, self.top_blocks, 1, lg - 1, 0 if transpose else 1)
            _native.check(lib.hbs_apply_up(lg - 1, 1, r, c, tn, trb, tsq, tbp, qtop.data_ptr(), tqp, st),
                          "hbs_apply_up(top)")
            q1 = tq[1]
        _native.check(lib.hbs_apply_root(r, c, self.root.data_ptr(), 1 if transpose else 0, q1.data_ptr(),
                                         tu[1].data_ptr(), st), "hbs_apply_root")
        if lg >= 2:
            tn, trb, tsq, tbp = _level_arrays(self.top_geo, self.top_blocks, 1, lg - 1, 1 if transpose else 0)
            _, _, _, tdp = _level_arrays(self.top_geo, self.top_blocks, 1, lg - 1, 2)
            _native.check(lib.hbs_apply_down(1, lg - 1, r, c, tn, trb, tsq, 2 * r, tbp, tdp, 1 if transpose else 0,
                                             tup, tqp, qtop.data_ptr(), tu[lg].data_ptr(), st), "hbs_apply_down(top)")
        return tu[lg]

    def down_local(self, q, qhat, uhat_lg, transpose=False):
        part, r = self.part, self.part.r
        L, lo = part.tree.depth, max(part.lg, 1)
        c = q.shape[1]
        f64 = dict(dtype=torch.float64, device=self.device)
        uhat = {lv: torch.empty(self.local_geo[lv].nbox * r, c, **f64) for lv in range(lo + 1, L + 1)}
        uhat[lo] = uhat_lg.contiguous()
        up_, qp = _native.ptr_array([0] * (L + 1)), _native.ptr_array([0] * (L + 1))
        for lv in range(lo, L + 1):
            up_[lv], qp[lv] = uhat[lv].data_ptr(), qhat[lv].data_ptr()
        out = torch.empty_like(q)
        nbox, rb, sq, bp = _level_arrays(self.local_geo, self.local_blocks, lo, L, 1 if transpose else 0)
        _, _, _, dp = _level_arrays(self.local_geo, self.local_blocks, lo, L, 2)
        st = torch.cuda.current_stream(self.device).cuda_stream
        _native.check(_native.lib().hbs_apply_down(lo, L, r, c, nbox, rb, sq, self.local_geo[L].max_rows, bp, dp,
                                                   1 if transpose else 0, up_, qp, q.data_ptr(), out.data_ptr(), st),
                      "hbs_apply_down")
        return out

    def apply(self, q, transpose=False):
        """Distributed A q (A^T q) for this rank's rows of q."""
        part, r = self.part, self.part.r
        q = q.contiguous()
        qhat = self.up_local(q, transpose)
        if part.world == 1:
            st = torch.cuda.current_stream(self.device).cuda_stream
            u1 = torch.empty(2 * r, q.shape[1], dtype=torch.float64, device=self.device)
            _native.check(_native.lib().hbs_apply_root(r, q.shape[1], self.root.data_ptr(), 1 if transpose else 0,
                                                       qhat[1].data_ptr(), u1.data_ptr(), st), "hbs_apply_root")
            return self.down_local(q, qhat, u1, transpose)
        lg = part.lg
        qtop = torch.empty(part.world * r * q.shape[1], dtype=torch.float64, device=self.device)
        _all_gather_flat(qtop, qhat[lg].reshape(-1), self.group)
        ulg = self.top(qtop.reshape(part.world * r, q.shape[1]), transpose)
        return self.down_local(q, qhat, ulg[part.rank * r:(part.rank + 1) * r], transpose)


class DistributedCompressor:
    """Preallocated subtree-partitioned compressor (CUDA): `run` enqueues the
    local sweep, the all-gather of lifted halves and the replicated top sweep;
    `operator()` wraps the result as a DistributedOperator."""

    def __init__(self, tree: ClusterTree, partition: SubtreePartition, s: int, tol: float = 1e-10, device=None,
                 group=None):
        self.part, self.s, self.group = partition, s, group
        r = partition.r
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.local = CompressPlan(tree, s, r, tol, device=self.device, specs=partition.local_specs,
                                  with_root=(partition.world == 1))
        self.top = None
        if partition.world > 1:
            self.top = CompressPlan(tree, s, r, tol, device=self.device, specs=partition.top_specs, with_root=True)
            self.gathered = torch.empty(partition.world * 4 * r * s, dtype=torch.float64, device=self.device)
            self.top_quad = [torch.empty(partition.world * r, s, dtype=torch.float64, device=self.device)
                             for _ in range(4)]
            self.half = torch.empty(4, r, s, dtype=torch.float64, device=self.device)

    def run(self, omega, psi, y, z):
        self.local.run(omega, psi, y, z)
        if self.top is None:
            return
        w, r, s = self.part.world, self.part.r, self.s
        for i, m in enumerate(self.local.top_quad):
            self.half[i].copy_(m.reshape(r, s))
        _all_gather_flat(self.gathered, self.half.reshape(-1), self.group)
        g = self.gathered.reshape(w, 4, r, s)
        for i in range(4):
            self.top_quad[i].copy_(g[:, i].reshape(w * r, s))
        if self.top.specs:
            self.top.run(*self.top_quad)
        else:
            self.top.top_quad = tuple(self.top_quad)
            self.top.run_root(self.top_quad[0], self.top_quad[2])

    def raise_for_status(self):
        fail = self.local.first_failure()
        if self.top is not None:
            fail = _agree_on_failure(fail, self.group)
            if fail is None:
                fail = self.top.first_failure()
        if fail is not None:
            raise_ill_conditioned(*fail, self.local.tol)

    def operator(self) -> DistributedOperator:
        top_blocks = {} if self.top is None else {lv: self.top.levels[lv] for lv, _, _ in self.top.specs}
        top_geo = {} if self.top is None else {lv: self.top.geometry[lv] for lv, _, _ in self.top.specs}
        root = self.local.root if self.top is None else self.top.root
        return DistributedOperator(self.part, {lv: self.local.levels[lv] for lv, _, _ in self.part.local_specs},
                                   {lv: self.local.geometry[lv] for lv, _, _ in self.part.local_specs},
                                   top_blocks, top_geo, root, self.group)
