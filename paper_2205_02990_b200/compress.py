"""Reference-compatible compression API on the B200 kernels.

Mirrors `pkg/src/hbs/compress.py`: `CompressionConfig` (32-70), `SampleSet`
(73-94), `draw_samples` (132-141), `compress_from_samples` (236-280) and
`compress` (283-290).  The per-node Python loop of the reference is replaced
by one C-ABI call per tree level (`hbs_compress_level`, all boxes of the
level at once) plus `hbs_compress_root`; the sample quadruple, the lifted
parent quadruples and the factorization stay resident in HBM.

Error semantics follow the reference sweep order: the first failing node of
the deepest failing level (ascending id) raises IllConditionedProbeError with
its node id and level (compress.py:260-265, 274-279).
"""

import ctypes
import os
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _native, flops
from .errors import ConfigurationError, DimensionError, IllConditionedProbeError
from .factorization import HbsFactorization, tree_geometry
from .tree import ClusterTree, build_tree

DEFAULT_ILL_CONDITIONING_TOL = 1e-10   # linalg.py:20
STREAM_OMEGA, STREAM_PSI, STREAM_POWER, STREAM_SYNTHETIC = 0, 1, 2, 3   # linalg.py:15-18


@dataclass(frozen=True)
class CompressionConfig:
    """rank r, leaf threshold m, probe count s (None -> max(r + max leaf, 3r)),
    seed, ill-conditioning tolerance (compress.py:32-70)."""

    rank: int
    leaf_threshold: int
    probes: int | None = None
    seed: int = 0
    ill_conditioning_tol: float = DEFAULT_ILL_CONDITIONING_TOL

    def resolved_probes(self, tree: ClusterTree) -> int:
        if self.probes is not None:
            return self.probes
        return max(self.rank + tree.max_leaf_size, 3 * self.rank)

    def validate_for(self, tree: ClusterTree) -> int:
        if self.rank < 1:
            raise ConfigurationError(f"rank must be positive, got {self.rank}")
        if self.leaf_threshold < self.rank:
            raise ConfigurationError(
                f"leaf threshold {self.leaf_threshold} < rank {self.rank}: leaf bases would be wider than tall")
        if tree.min_leaf_size < self.rank:
            raise ConfigurationError(
                f"smallest leaf has {tree.min_leaf_size} rows < rank {self.rank}; "
                "lower the rank or raise the leaf threshold")
        s = self.resolved_probes(tree)
        s_min = max(self.rank + tree.max_leaf_size, 3 * self.rank)
        if s < s_min:
            raise ConfigurationError(f"probe count {s} below the required max(r + max leaf, 3r) = {s_min}")
        return s


@dataclass(frozen=True)
class SampleSet:
    """Probe quadruple (omega, psi, y = A omega, z = A^T psi): numpy arrays
    (host) or float64 CUDA tensors (device-resident, no copy)."""

    omega: object
    psi: object
    y: object
    z: object

    def __post_init__(self):
        shapes = {tuple(m.shape) for m in (self.omega, self.psi, self.y, self.z)}
        if len(shapes) != 1:
            raise DimensionError(f"sample matrices must share one shape, got {shapes}")

    @property
    def n(self) -> int:
        return self.omega.shape[0]

    @property
    def probes(self) -> int:
        return self.omega.shape[1]


def gaussian_matrix(n: int, s: int, seed: int, stream: int = 0) -> np.ndarray:
    """Seeded n x s standard normals, the reference's PCG64 substreams
    (linalg.py:23-32), so host samples are bit-identical to the reference's."""
    if n < 1 or s < 1:
        raise DimensionError(f"gaussian_matrix needs positive dimensions, got {n} x {s}")
    gen = np.random.Generator(np.random.PCG64(np.random.SeedSequence(entropy=seed, spawn_key=(stream,))))
    return gen.standard_normal((n, s))


def draw_samples(oracle, s: int, seed: int) -> SampleSet:
    """Draw Omega, Psi and push one batch through each oracle direction
    (compress.py:132-141)."""
    if s < 1:
        raise DimensionError(f"need at least one probe column, got {s}")
    omega = gaussian_matrix(oracle.n, s, seed, STREAM_OMEGA)
    psi = gaussian_matrix(oracle.n, s, seed, STREAM_PSI)
    return SampleSet(omega=omega, psi=psi, y=oracle.apply_batch(omega), z=oracle.apply_transpose_batch(psi))


def _size_t():
    return ctypes.c_size_t()


def tree_level_specs(tree: ClusterTree, rank: int, top_level: int = 1):
    """(level, row starts, first box index) for levels L .. top_level of a whole tree."""
    specs = []
    for level in range(tree.depth, top_level - 1, -1):
        if level == tree.depth:
            begins = tree.level_begin(level)
        else:
            begins = np.arange((1 << level) + 1, dtype=np.int64) * 2 * rank
        specs.append((level, begins, 0))
    return specs


class CompressPlan:
    """Buffers + launch sequence of a level sweep on one device.

    `specs` lists the levels to compress, deepest first, as (level, row starts
    of the level's boxes, index of the first box within the global level);
    the default is the whole tree of `tree`.  With `with_root` the root core
    is solved after the last (level-1) sweep.  Everything is allocated up
    front, so `run()` only enqueues kernels on a stream: it can be timed with
    CUDA events or captured in a CUDA graph.  After `run`, `top_quad` holds
    the lifted quadruple of the last compressed level (the multi-GPU hand-off)."""

    def __init__(self, tree: ClusterTree, s: int, rank: int, tol: float = DEFAULT_ILL_CONDITIONING_TOL,
                 device=None, specs=None, with_root=None, out_levels=None, max_workspace_bytes=None,
                 parent_geometry=None):
        self.tree, self.s, self.rank, self.tol = tree, s, rank, tol
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        r = rank
        self.specs = specs if specs is not None else tree_level_specs(tree, r)
        self.with_root = (self.specs[-1][0] == 1) if with_root is None else with_root
        dev, f64 = self.device, torch.float64
        lib = _native.lib()
        from .factorization import LevelGeometry
        self.geometry, self.first_box, self.levels = {}, {}, {}
        # A level whose per-box scratch exceeds the cap runs in contiguous box
        # chunks that reuse one workspace (the reference's level loop,
        # compress.py:250-269, has no such limit on the host; config 5's leaf
        # level needs ~110 GB of scratch at once).
        cap = max_workspace_bytes if max_workspace_bytes is not None else _workspace_cap(dev)
        self.chunks = {}
        ws, lift_rows = 0, []
        for level, begins, first in self.specs:
            # (parent_geometry: whole-level geometries already on the device; slice them there)
            g = (LevelGeometry.slice_of(parent_geometry[level], first, len(begins) - 1)
                 if parent_geometry is not None and level in parent_geometry else LevelGeometry(begins, dev))
            self.geometry[level], self.first_box[level] = g, first
            if out_levels is not None and level in out_levels:   # caller-owned (views of full levels)
                self.levels[level] = out_levels[level]
            else:
                self.levels[level] = (torch.empty(g.total_rows, r, dtype=f64, device=dev),
                                      torch.empty(g.total_rows, r, dtype=f64, device=dev),
                                      torch.empty(g.sq_total, dtype=f64, device=dev))
            sz = _size_t()
            _native.check(lib.hbs_level_workspace_bytes(g.nbox, g.max_rows, s, r, ctypes.byref(sz)), "workspace")
            if sz.value > cap and g.nbox > 1:
                per_box = sz.value / g.nbox
                nchunk = max(1, int(cap // per_box))
                while True:
                    _native.check(lib.hbs_level_workspace_bytes(nchunk, g.max_rows, s, r, ctypes.byref(sz)),
                                  "workspace")
                    if sz.value <= cap or nchunk == 1:
                        break
                    nchunk = max(1, nchunk * 7 // 8)
                parts = []
                for b0 in range(0, g.nbox, nchunk):
                    b1 = min(g.nbox, b0 + nchunk)
                    parts.append((b0, b1, LevelGeometry(g.begins_host[b0:b1 + 1], dev),
                                  torch.zeros(2 * (b1 - b0), dtype=torch.int32, device=dev)))
                self.chunks[level] = parts
            ws = max(ws, sz.value)
            lift_rows.append(g.nbox * r)
        if self.with_root:   # (one small upload; the host pipeline's subtree plans have no root)
            self.geometry[0] = LevelGeometry(np.array([0, 2 * r], dtype=np.int64), dev)
        sz = _size_t()
        _native.check(lib.hbs_root_workspace_bytes(2 * r, s, ctypes.byref(sz)), "workspace")
        ws = max(ws, sz.value)
        self.workspace = torch.empty(ws // 8 + 1, dtype=f64, device=dev)
        self.workspace_bytes = ws
        # lifted quadruples, ping-pong between consecutive levels
        sizes = [max(lift_rows[0::2] or [1]), max(lift_rows[1::2] or [1])]
        self.lift = [[torch.empty(rows, s, dtype=f64, device=dev) for _ in range(4)] for rows in sizes]
        nstat = sum(2 * self.geometry[lv].nbox for lv, _, _ in self.specs) + 1
        self.status = torch.zeros(nstat, dtype=torch.int32, device=dev)
        self.root = torch.empty(2 * r, 2 * r, dtype=f64, device=dev)
        self.top_quad = None

    def _status_slices(self):
        out, off = {}, 0
        for level, _, _ in self.specs:
            n = 2 * self.geometry[level].nbox
            out[level] = self.status[off:off + n]
            off += n
        out[0] = self.status[off:off + 1]
        return out

    def run_level(self, idx, quad, stream, box_range=None, chunk_geo=None, status=None):
        """Enqueue one level (spec index `idx`) on `stream`; `box_range` =
        (b0, b1) restricts it to a contiguous run of boxes (whose geometry
        `chunk_geo` holds rows relative to box b0).  Returns the lift buffers."""
        lib = _native.lib()
        level = self.specs[idx][0]
        r, s = self.rank, self.s
        g = self.geometry[level]
        u, v, d = self.levels[level]
        out = self.lift[idx % 2]
        if box_range is None:
            b0, geo, row0, sq0, stat = 0, g, 0, 0, self._status_slices()[level]
        else:
            b0, b1 = box_range
            geo, row0, sq0 = chunk_geo, int(g.begins_host[b0] - g.begins_host[0]), int(g.sq_host[b0])
            stat = status
        q = [m[row0:] for m in quad]
        lib.hbs_level_hint(geo.min_rows)
        rc = lib.hbs_compress_level(
            geo.nbox, geo.row_begin.data_ptr(), geo.sq_off.data_ptr(), geo.max_rows, s, r, self.tol,
            q[0].data_ptr(), q[1].data_ptr(), q[2].data_ptr(), q[3].data_ptr(),
            u[row0:].data_ptr(), v[row0:].data_ptr(), d[sq0:].data_ptr(),
            out[0][b0 * r:].data_ptr(), out[1][b0 * r:].data_ptr(), out[2][b0 * r:].data_ptr(),
            out[3][b0 * r:].data_ptr(),
            self.workspace.data_ptr(), self.workspace_bytes, stat.data_ptr(), stream)
        _native.check(rc, f"hbs_compress_level(level {level})")
        return tuple(m[:g.nbox * r] for m in out)

    def run_level_profiled(self, idx, quad, stream):
        """One level (all its chunks) with per-phase CUDA-event timing
        (hbs_compress_level_profiled, synchronising); returns (lift outputs,
        six phase times in ms summed over the chunks).  Measurement only."""
        lib = _native.lib()
        level = self.specs[idx][0]
        r, s = self.rank, self.s
        g = self.geometry[level]
        u, v, d = self.levels[level]
        out = self.lift[idx % 2]
        buf = (ctypes.c_float * 6)()
        total = [0.0] * 6
        parts = self.chunks.get(level) or [(0, g.nbox, g, self._status_slices()[level])]
        for b0, b1, geo, stat in parts:
            row0, sq0 = int(g.begins_host[b0] - g.begins_host[0]), int(g.sq_host[b0])
            q = [m[row0:] for m in quad]
            lib.hbs_level_hint(geo.min_rows)
            rc = lib.hbs_compress_level_profiled(
                geo.nbox, geo.row_begin.data_ptr(), geo.sq_off.data_ptr(), geo.max_rows, s, r, self.tol,
                *(m.data_ptr() for m in q), u[row0:].data_ptr(), v[row0:].data_ptr(), d[sq0:].data_ptr(),
                *(m[b0 * r:].data_ptr() for m in out), self.workspace.data_ptr(), self.workspace_bytes,
                stat.data_ptr(), stream, buf)
            _native.check(rc, f"profiled level {level}")
            total = [a + b for a, b in zip(total, buf)]
        return tuple(m[:g.nbox * r] for m in out), total

    def run(self, omega, psi, y, z, stream=None, first=0):
        """Enqueue the level sweep (compress.py:250-279) on `stream`, from spec
        index `first` (the quadruple given is that level's input)."""
        st = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        quad = (omega, psi, y, z)
        slices = self._status_slices()
        for idx in range(first, len(self.specs)):
            level = self.specs[idx][0]
            if level not in self.chunks:
                quad = self.run_level(idx, quad, st)
                continue
            nbox = self.geometry[level].nbox
            lvl_status = slices[level].view(2, nbox)
            torch_stream = torch.cuda.ExternalStream(st, device=self.device) if stream is not None else None
            out = None
            for b0, b1, geo, cst in self.chunks[level]:
                out = self.run_level(idx, quad, st, box_range=(b0, b1), chunk_geo=geo, status=cst)
                with torch.cuda.stream(torch_stream) if torch_stream is not None else _nullcontext():
                    lvl_status[:, b0:b1].copy_(cst.view(2, b1 - b0))
            quad = out
        self.top_quad = quad
        if self.with_root:
            self.run_root(quad[0], quad[2], stream=st)

    def run_graph(self, omega, psi, y, z):
        """The same sweep replayed from a CUDA graph (captured on first use for
        this quadruple's addresses, after one plain run that sets the kernels'
        attributes): the ~230 launches of a sweep become one graph launch,
        which removes the host launch gaps between the short kernels of the
        upper levels.  Returns the number of kernels of this library in the
        graph (the launches one replay performs)."""
        key = tuple(m.data_ptr() for m in (omega, psi, y, z))
        if getattr(self, "_graph_key", None) != key:
            lib = _native.lib()
            self.run(omega, psi, y, z)
            torch.cuda.synchronize(self.device)
            graph = torch.cuda.CUDAGraph()
            n0 = lib.hbs_launch_counter()
            with torch.cuda.graph(graph):
                self.run(omega, psi, y, z)
            self._graph, self._graph_key, self._graph_quad = graph, key, self.top_quad
            self._graph_launches = int(lib.hbs_launch_counter() - n0)
        self._graph.replay()
        self.top_quad = self._graph_quad
        return self._graph_launches

    def run_root(self, omega_root, y_root, stream=None):
        """Root core D_root = Y_root Omega_root^+ (compress.py:230-233)."""
        lib = _native.lib()
        st = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        g0 = self.geometry[0]
        rc = lib.hbs_compress_root(g0.row_begin.data_ptr(), g0.sq_off.data_ptr(), 2 * self.rank, self.s, self.tol,
                                   omega_root.data_ptr(), y_root.data_ptr(), self.root.data_ptr(),
                                   self.workspace.data_ptr(), self.workspace_bytes, self._status_slices()[0].data_ptr(),
                                   st)
        _native.check(rc, "hbs_compress_root")

    def first_failure(self):
        """(level, node id) of the first failing box in sweep order, or None
        (one device->host read of all statuses)."""
        host = self.status.cpu().numpy()
        if not host.any():
            return None
        off = 0
        for level, _, _ in self.specs:
            nbox = self.geometry[level].nbox
            blk = host[off:off + 2 * nbox].reshape(2, nbox)
            off += 2 * nbox
            bad = np.nonzero(blk.any(axis=0))[0]
            if bad.size:
                return level, (1 << level) - 1 + self.first_box[level] + int(bad[0])
        if self.with_root and host[off]:
            return 0, 0
        return None

    def raise_for_status_from(self, first_idx):
        """Like raise_for_status but ignoring the specs before `first_idx`
        (their statuses were checked elsewhere, e.g. per leaf chunk)."""
        host = self.status.cpu().numpy()
        off = 0
        for idx, (level, _, _) in enumerate(self.specs):
            nbox = self.geometry[level].nbox
            blk = host[off:off + 2 * nbox].reshape(2, nbox)
            off += 2 * nbox
            if idx < first_idx:
                continue
            bad = np.nonzero(blk.any(axis=0))[0]
            if bad.size:
                raise_ill_conditioned(level, (1 << level) - 1 + self.first_box[level] + int(bad[0]), self.tol)
        if self.with_root and host[off]:
            raise_ill_conditioned(0, 0, self.tol)

    def raise_for_status(self):
        """Raise like the reference for the first failing node in sweep order."""
        fail = self.first_failure()
        if fail is not None:
            raise_ill_conditioned(*fail, self.tol)

    def factorization(self) -> HbsFactorization:
        geo = [self.geometry[level] for level in range(self.tree.depth + 1)]
        levels = [None] + [self.levels[level] for level in range(1, self.tree.depth + 1)]
        return HbsFactorization.from_device(self.tree, self.rank, geo, levels, self.root)


def raise_ill_conditioned(level, node_id, tol):
    raise IllConditionedProbeError(
        f"node {node_id} (level {level}): probe matrix is rank deficient within tolerance {tol:g}; "
        "increase the probe count s", node_id=node_id, level=level)


def _check_configuration(tree: ClusterTree, s: int, r: int):
    """Shape-only failures of compress_node_bases / col, in sweep order
    (compress.py:164-168, linalg.py:329-331)."""
    for level in range(tree.depth, 0, -1):
        sizes = tree.level_sizes(level) if level == tree.depth else np.full(1 << level, 2 * r)
        short = np.nonzero(s - sizes < r)[0]
        thin = np.nonzero(sizes < r)[0]
        if short.size or thin.size:
            first = min(short.min() if short.size else 1 << 62, thin.min() if thin.size else 1 << 62)
            rows = int(sizes[first])
            if s - rows < r:
                raise ConfigurationError(
                    f"probe count {s} leaves nullity {s - rows} < rank {r} for a {rows}-row node; "
                    "increase the probe count s")
            raise DimensionError(f"cannot extract {r} basis columns from a {rows} x {r} matrix")


class _nullcontext:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


def _workspace_cap(dev) -> int:
    """Per-level scratch cap: HBS_MAX_WORKSPACE_GB, else a quarter of the
    device's memory (45 GB on a B200)."""
    env = os.environ.get("HBS_MAX_WORKSPACE_GB")
    if env:
        return int(float(env) * (1 << 30))
    return int(torch.cuda.get_device_properties(dev).total_memory // 4)


def _device_tensor(a, device):
    if isinstance(a, torch.Tensor):
        if a.dtype != torch.float64:
            raise DimensionError(f"samples must be float64, got {a.dtype}")
        return a.to(device).contiguous()
    arr = np.ascontiguousarray(a, dtype=np.float64)
    t = torch.from_numpy(arr)
    if device.type == "cuda":
        if not t.is_pinned():
            t = t.pin_memory()
        t = t.to(device, non_blocking=True)
    return t


def _charge_madds(tree: ClusterTree, s: int, r: int):
    """Host-side madd charge identical to the reference's per-node calls."""
    total = 0
    for level in range(tree.depth, 0, -1):
        sizes = tree.level_sizes(level) if level == tree.depth else np.full(1 << level, 2 * r)
        for rows in np.unique(sizes):
            cnt = int((sizes == rows).sum())
            total += cnt * (flops.node_compress_madds(int(rows), s, r) + flops.lift_madds(int(rows), s, r))
    total += flops.root_madds(2 * r, s)
    flops.add_madds(total)


def _host_view(a):
    """torch view of a host numpy array (float64, C-contiguous; copied only if
    it is not), else None for device tensors."""
    if isinstance(a, torch.Tensor):
        return None
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))


def _compress_host_subtrees(host, tree: ClusterTree, config: CompressionConfig, dev, chunks: int = None):
    """Host samples in (pinned, or pageable staged through pinned buffers),
    host-materialised factorization out, with the
    transfers hidden behind the compute by subtree: the rows are uploaded as
    `chunks` contiguous subtrees (one H2D stream), each subtree is compressed
    from its leaves up to its own root as soon as its rows have arrived (the
    single-device form of the multi-GPU partition, distributed.py), its
    U, V, D go back to pinned host memory on a second copy stream while the
    next subtree computes, and the few top levels plus the root run on the
    concatenated subtree-root lifts at the end.  Per-node arithmetic is that
    of the level sweep, so the result is bitwise identical to it
    (test_host_subtree_pipeline_bitwise)."""
    from .distributed import SubtreePartition
    from .factorization import LevelGeometry
    n, s = host[0].shape
    r, tol = config.rank, config.ill_conditioning_tol
    L = tree.depth
    _t = [time.perf_counter()] if os.environ.get("HBS_HOST_TIMING") else None
    if chunks is None:
        chunks = int(os.environ.get("HBS_HOST_CHUNKS", "16"))
    world = 1
    while world * 2 <= chunks and (world * 2).bit_length() - 1 < L:
        world *= 2
    full = {lv: b for lv, b, _ in tree_level_specs(tree, r)}
    geo = {lv: LevelGeometry(full[lv], dev) for lv in full}
    f64 = torch.float64
    levels = {lv: (torch.empty(g.total_rows, r, dtype=f64, device=dev), torch.empty(g.total_rows, r, dtype=f64, device=dev),
                   torch.empty(g.sq_total, dtype=f64, device=dev)) for lv, g in geo.items()}
    hosts = {lv: tuple(torch.empty(t.shape, dtype=f64, pin_memory=True) for t in ts) for lv, ts in levels.items()}
    comp = torch.cuda.current_stream(dev)
    h2d, copy = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    dq = [torch.empty(n, s, dtype=f64, device=dev) for _ in range(4)]
    parts = [SubtreePartition(tree, world, g, r) for g in range(world)]
    def views(specs):
        out = {}
        for lv, begins, first in specs:
            g, nb = geo[lv], len(begins) - 1
            r0, r1 = int(g.begins_host[first]), int(g.begins_host[first + nb])
            q0, q1 = int(g.sq_host[first]), int(g.sq_host[first + nb])
            out[lv] = (r0, r1, q0, q1)
        return out

    def drain(specs, plan):       # level blocks of `plan` -> pinned host, on the copy stream
        done = torch.cuda.Event()
        done.record(comp)
        copy.wait_event(done)
        with torch.cuda.stream(copy):
            for lv, (r0, r1, q0, q1) in views(specs).items():
                u, v, d = levels[lv]
                hu, hv, hd = hosts[lv]
                hu[r0:r1].copy_(u[r0:r1], non_blocking=True)
                hv[r0:r1].copy_(v[r0:r1], non_blocking=True)
                hd[q0:q1].copy_(d[q0:q1], non_blocking=True)

    def out_views(specs):
        return {lv: (levels[lv][0][r0:r1], levels[lv][1][r0:r1], levels[lv][2][q0:q1])
                for lv, (r0, r1, q0, q1) in views(specs).items()}

    # every plan (buffers, geometry uploads) is built before any compute is
    # enqueued, so the launches of consecutive subtrees go out back to back
    plans = [CompressPlan(tree, s, r, tol, dev, specs=p.local_specs, with_root=(world == 1),
                          out_levels=out_views(p.local_specs), parent_geometry=geo) for p in parts]
    tspecs = parts[0].top_specs
    top = plans[0] if world == 1 else CompressPlan(tree, s, r, tol, dev, specs=tspecs, with_root=True,
                                                   out_levels=out_views(tspecs), parent_geometry=geo)
    # (uploads after the plans: their small geometry copies must not queue
    # behind gigabytes of H2D on the copy engine)
    if _t is not None:
        _t.append(time.perf_counter())
    def upload(p, src):          # rows of one subtree, host -> device on the H2D stream
        with torch.cuda.stream(h2d):
            for i in range(4):
                dq[i][p.begin:p.end].copy_(src[i], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(h2d)
        return ev

    if all(h.is_pinned() for h in host):
        # all uploads back to back on the H2D stream, then the launches
        arrived = [upload(p, [h[p.begin:p.end] for h in host]) for p in parts]
        for p, ev, plan in zip(parts, arrived, plans):
            comp.wait_event(ev)
            plan.run(*[m[p.begin:p.end] for m in dq], stream=comp.cuda_stream)
            drain(p.local_specs, plan)
    else:
        # ordinary (pageable) numpy arrays, the reference's calling convention:
        # each subtree's rows are staged through one of two pinned buffer sets
        # (a multi-threaded host copy) while the previous subtree is in flight
        rows = max(p.end - p.begin for p in parts)
        stage = [[torch.empty(rows, s, dtype=f64, pin_memory=True) for _ in range(4)] for _ in range(2)]
        in_flight = [None, None]
        for idx, (p, plan) in enumerate(zip(parts, plans)):
            buf = stage[idx % 2]
            if in_flight[idx % 2] is not None:
                in_flight[idx % 2].synchronize()      # the upload that last used this buffer set
            nr = p.end - p.begin
            for i in range(4):
                buf[i][:nr].copy_(host[i][p.begin:p.end])
            ev = upload(p, [b[:nr] for b in buf])
            in_flight[idx % 2] = ev
            comp.wait_event(ev)
            plan.run(*[m[p.begin:p.end] for m in dq], stream=comp.cuda_stream)
            drain(p.local_specs, plan)
    if world > 1:
        with torch.cuda.stream(comp):
            top_quad = tuple(torch.cat([pl.top_quad[i] for pl in plans]) for i in range(4))
        if tspecs:
            top.run(*top_quad, stream=comp.cuda_stream)
            drain(tspecs, top)
        else:
            top.run_root(top_quad[0], top_quad[2], stream=comp.cuda_stream)
        plans = plans + [top]
    if _t is not None:
        _t.append(time.perf_counter())
    torch.cuda.synchronize(dev)
    if _t is not None:
        _t.append(time.perf_counter())
        print("host pipeline: plans built %.1f ms, enqueued %.1f ms, device done %.1f ms" % tuple(1e3 * (x - _t[0]) for x in _t[1:]), flush=True)
    fails = [f for f in (pl.first_failure() for pl in plans) if f is not None]
    if fails:
        level, nid = min(fails, key=lambda f: (-f[0], f[1]))
        raise_ill_conditioned(level, nid, tol)
    geo_list = [geo.get(lv, top.geometry[0] if lv == 0 else None) for lv in range(L + 1)]
    f = HbsFactorization.from_device(tree, r, geo_list, [None] + [levels[lv] for lv in range(1, L + 1)], top.root)
    for lv, (hu, hv, hd) in hosts.items():
        f._host[(lv, "u")], f._host[(lv, "v")], f._host[(lv, "d")] = hu.numpy(), hv.numpy(), hd.numpy()
    f._host["root"] = top.root.cpu().numpy()
    # (the device copies of the samples and the plans' workspaces are freed
    # here: the synchronize above ordered every use of them)
    f._host_keepalive = hosts
    del dq, plans, top
    return f


def compress_from_samples(samples: SampleSet, tree: ClusterTree, config: CompressionConfig,
                          device=None) -> HbsFactorization:
    """Level sweep on an already-drawn probe quadruple (compress.py:236-280),
    on the GPU.  Host (numpy) samples are uploaded once; CUDA tensors are used
    in place.  The returned factorization is device-resident."""
    if samples.n != tree.n:
        raise DimensionError(f"samples are for n={samples.n}, tree has n={tree.n}")
    s, r = samples.probes, config.rank
    _check_configuration(tree, s, r)
    if device is None:
        dev = samples.omega.device if isinstance(samples.omega, torch.Tensor) else torch.device("cuda")
    else:
        dev = torch.device(device)
    if dev.type != "cuda":
        raise DimensionError("the compressor runs on a CUDA device only (no CPU fallback)")
    hostv = [_host_view(m) for m in (samples.omega, samples.psi, samples.y, samples.z)]
    if all(h is not None for h in hostv) and tree.depth >= 2:
        f = _compress_host_subtrees(hostv, tree, config, dev)
        if flops.counting():
            _charge_madds(tree, s, r)
        return f
    quad = [_device_tensor(m, dev) for m in (samples.omega, samples.psi, samples.y, samples.z)]
    plan = CompressPlan(tree, s, r, config.ill_conditioning_tol, dev)
    plan.run(*quad)
    plan.raise_for_status()
    if flops.counting():
        _charge_madds(tree, s, r)
    return plan.factorization()


def compress(oracle, config: CompressionConfig) -> HbsFactorization:
    """Build the tree, draw exactly s probes per direction, sweep
    (compress.py:283-290)."""
    tree = build_tree(oracle.n, config.leaf_threshold)
    s = config.validate_for(tree)
    samples = draw_samples(oracle, s, config.seed)
    return compress_from_samples(samples, tree, config)
