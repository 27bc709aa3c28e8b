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

import numpy as np
import torch
import torch.distributed as dist

from .compress import CompressionConfig, CompressPlan, _check_configuration, raise_ill_conditioned
from .errors import ConfigurationError
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
        for level in range(tree.depth, lg - 1, -1):
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
    dist.all_gather_into_tensor(gathered, half, group=group)
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
