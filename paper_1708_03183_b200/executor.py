"""Execute loop chains on the B200: untiled reference-order execution and the
fused tiled executor.

Same entry points as the reference (``executor.py:163-245``):
``execute_untiled(chain, bindings, datasets, registry)`` and
``execute_schedule(schedule, chain, bindings, datasets, registry,
exchange=None, use_local_maps=False, max_workers=None)``.

Differences, all B200-motivated:

* ``Dataset.values`` is a float64 tensor resident in HBM (element-major, as in
  the reference); numpy input is uploaded once.  ``Dataset.numpy()`` reads
  it back.
* Kernel bodies are native device functions (``libltcuda.so``); the registry
  maps kernel ids to them.  Python callables cannot run on the device and are
  rejected at registration: there is no CPU fallback.
* Execution is stream-ordered and asynchronous; ``ExecutionReport`` phase
  times come from CUDA events and are resolved on first access.
* ``max_workers`` is accepted and ignored (colour classes run as one launch).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .chain import LoopChain
from .errors import ExecutionError, StaleScheduleError

THREADS_ENV = "LOOPTILE_THREADS"


def _to_device_tensor(values):
    import torch
    if isinstance(values, torch.Tensor):
        t = values.detach().to(torch.float64).reshape(-1)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(values, dtype=np.float64)).ravel())
    if torch.cuda.is_available() and t.device.type != "cuda":
        t = t.to("cuda")
    return t.contiguous()


@dataclass
class Dataset:
    """Values attached to an iteration space, values_per_element reals each.

    Reference ``executor.py:25-43``; ``values`` lives on the GPU.
    """

    name: str
    space: object
    values_per_element: int
    values: object

    def __post_init__(self):
        self.values = _to_device_tensor(self.values)
        if self.values.numel() != self.space.total * self.values_per_element:
            raise ExecutionError(
                f"dataset {self.name!r}: {self.values.numel()} values for "
                f"{self.space.total} x {self.values_per_element}")

    def copy(self) -> "Dataset":
        return Dataset(self.name, self.space, self.values_per_element, self.values.clone())

    def numpy(self) -> np.ndarray:
        return self.values.detach().cpu().numpy()


@dataclass(frozen=True)
class NativeKernel:
    """Handle of a device kernel body compiled into libltcuda.so."""

    name: str
    id: int
    nargs: int


def native_kernel(name: str) -> NativeKernel:
    from . import _lib
    kid, nargs = _lib.kernel_lookup(name)
    return NativeKernel(name, kid, nargs)


class KernelRegistry:
    """Kernel bodies by id; an id registers once (reference ``executor.py:46-61``).

    ``body`` is a :class:`NativeKernel` or the name of one.
    """

    def __init__(self):
        self._kernels: dict[str, tuple] = {}

    def register(self, kernel_id: str, body, nargs: int) -> None:
        if kernel_id in self._kernels:
            raise ExecutionError(f"kernel {kernel_id!r} already registered")
        if isinstance(body, str):
            body = native_kernel(body)
        if not isinstance(body, NativeKernel):
            raise ExecutionError(
                f"kernel {kernel_id!r}: bodies must be native device kernels "
                f"(native_kernel(name)); Python callables have no GPU path and "
                f"there is no CPU fallback")
        if body.nargs != nargs:
            raise ExecutionError(
                f"kernel {kernel_id!r}: native body {body.name!r} takes {body.nargs} "
                f"args, registered with {nargs}")
        self._kernels[kernel_id] = (body, nargs)

    def get(self, kernel_id: str):
        try:
            return self._kernels[kernel_id]
        except KeyError:
            raise ExecutionError(f"kernel {kernel_id!r} not registered") from None

    def __contains__(self, kernel_id: str) -> bool:
        return kernel_id in self._kernels


@dataclass(frozen=True)
class KernelBinding:
    """Dataset names paired positionally with a loop's descriptors."""

    kernel: str
    args: tuple[str, ...]


class _EventPhases(dict):
    """phase -> seconds, resolved from CUDA events on first read."""

    def __init__(self):
        super().__init__()
        self._pending: list[tuple[str, object, object]] = []

    def _resolve(self):
        if self._pending:
            for name, a, b in self._pending:
                b.synchronize()
                dict.__setitem__(self, name, dict.get(self, name, 0.0)
                                 + a.elapsed_time(b) * 1e-3)
            self._pending = []

    def add_events(self, name, start, end):
        self._pending.append((name, start, end))

    def __getitem__(self, k):
        self._resolve()
        return dict.__getitem__(self, k)

    def get(self, k, default=None):
        self._resolve()
        return dict.get(self, k, default)

    def items(self):
        self._resolve()
        return dict.items(self)


@dataclass
class ExecutionReport:
    """Per-phase times and tile counts for one tiled execution (``executor.py:72-95``)."""

    phase_seconds: dict = field(default_factory=_EventPhases)
    tiles_per_color: dict[int, int] = field(default_factory=dict)
    bytes_exchanged: int = 0
    launches: int = 0

    PHASES = ("exchange_start", "core", "exchange_wait", "boundary")

    def to_text(self) -> str:
        lines = ["execution report"]
        for phase in self.PHASES:
            lines.append(f"  {phase}: {self.phase_seconds.get(phase, 0.0) * 1e3:.3f} ms")
        for color in sorted(self.tiles_per_color):
            lines.append(f"  color {color}: {self.tiles_per_color[color]} tiles")
        lines.append(f"  bytes exchanged: {self.bytes_exchanged}")
        return "\n".join(lines)

    def to_kv(self) -> str:
        items = [f"phase.{p}={self.phase_seconds.get(p, 0.0):.9f}" for p in self.PHASES]
        items += [f"tiles.color{c}={n}" for c, n in sorted(self.tiles_per_color.items())]
        items.append(f"bytes_exchanged={self.bytes_exchanged}")
        return "\n".join(items)


def check_bindings(chain: LoopChain, bindings, datasets: dict) -> None:
    """Reference ``executor.py:98-119``, same messages."""
    if len(bindings) != len(chain.loops):
        raise ExecutionError(f"{len(bindings)} bindings for {len(chain.loops)} loops")
    for loop, binding in zip(chain.loops, bindings):
        if binding.kernel != loop.kernel:
            raise ExecutionError(
                f"loop {loop.index} expects kernel {loop.kernel!r}, bound {binding.kernel!r}")
        if len(binding.args) != len(loop.descriptors):
            raise ExecutionError(
                f"loop {loop.index}: {len(binding.args)} args for "
                f"{len(loop.descriptors)} descriptors")
        for d, name in zip(loop.descriptors, binding.args):
            if name not in datasets:
                raise ExecutionError(f"loop {loop.index}: dataset {name!r} missing")
            ds = datasets[name]
            wanted = loop.space if d.is_direct else d.map.target
            if ds.space is not wanted and ds.space.name != wanted.name:
                raise ExecutionError(
                    f"loop {loop.index}: dataset {name!r} lives on "
                    f"{ds.space.name!r}, descriptor needs {wanted.name!r}")


class _BoundChain:
    """ctypes image of (chain, kernel ids, dataset pointers), cached per call site."""

    def __init__(self, chain, bindings, datasets, registry):
        from . import _lib
        ids = []
        for loop in chain.loops:
            body, nargs = registry.get(loop.kernel)
            if nargs != len(loop.descriptors):
                raise ExecutionError(
                    f"kernel {loop.kernel!r} takes {nargs} args, loop {loop.index} "
                    f"has {len(loop.descriptors)} descriptors")
            ids.append(body.id)
        self.desc = _lib.ChainDesc(chain, kernel_ids=ids)
        entries = []
        for loop, binding in zip(chain.loops, bindings):
            for d, name in zip(loop.descriptors, binding.args):
                ds = datasets[name]
                t = ds.values
                if t.device.type != "cuda" or t.dtype.itemsize != 8 or not t.is_contiguous():
                    raise ExecutionError(
                        f"dataset {name!r} must be a contiguous float64 CUDA tensor")
                entries.append((t, ds.space.total, ds.values_per_element))
        self.tensors = [e[0] for e in entries]
        self.args = _lib.make_args(entries)


_BIND_CACHE: dict = {}


def _bind(chain, bindings, datasets, registry) -> _BoundChain:
    key = (id(chain), tuple(bindings), id(registry),
           tuple((n, ds.values.data_ptr(), ds.values_per_element)
                 for n, ds in sorted(datasets.items())))
    hit = _BIND_CACHE.get(key)
    if hit is not None and hit[0] is chain:
        return hit[1]
    bc = _BoundChain(chain, bindings, datasets, registry)
    if len(_BIND_CACHE) > 64:
        _BIND_CACHE.clear()
    _BIND_CACHE[key] = (chain, bc)
    return bc


def execute_untiled(chain: LoopChain, bindings, datasets: dict, registry: KernelRegistry) -> None:
    """The semantic reference order on the GPU: loops in order, elements ascending.

    Mapped increments are applied per target in ascending (element, k) order
    (ordered gather through the CSR inverse map), so results are bitwise those
    of the reference's sequential ``execute_untiled``.
    """
    from . import _lib
    check_bindings(chain, bindings, datasets)
    bc = _bind(chain, bindings, datasets, registry)
    _lib.execute_untiled(bc.desc, bc.args)


def execute_schedule(schedule, chain: LoopChain, bindings, datasets: dict,
                     registry: KernelRegistry, exchange=None, use_local_maps: bool = False,
                     max_workers: int | None = None) -> ExecutionReport:
    """Run the tiled schedule: core colours, halo wait, boundary colours (Alg. 2).

    ``exchange`` follows the reference protocol: ``begin()`` before the core
    phase, ``end()`` between core and boundary, ``bytes_exchanged``.  Each
    colour class is one launch of the fused tile kernel; T_ne never runs.
    """
    import torch
    from . import _lib
    if schedule.fingerprint != chain.fingerprint:
        raise StaleScheduleError("schedule was inspected for a different chain")
    if schedule.n_loops != len(chain.loops):
        raise StaleScheduleError("schedule loop count differs from chain")
    check_bindings(chain, bindings, datasets)
    bc = _bind(chain, bindings, datasets, registry)
    handle = schedule.device_handle(chain)

    report = ExecutionReport()
    colors, regions = schedule.tile_colors()
    for c, r in zip(colors.tolist(), regions.tolist()):
        if r != 2:
            report.tiles_per_color[c] = report.tiles_per_color.get(c, 0) + 1

    stream = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ev[0].record(stream)
    if exchange is not None:
        exchange.begin()
    ev[1].record(stream)
    info = _lib.execute(handle, bc.desc, bc.args, _lib.PHASE_CORE, use_local_maps)
    ev[2].record(stream)
    if exchange is not None:
        exchange.end()
        report.bytes_exchanged = getattr(exchange, "bytes_exchanged", 0)
    ev[3].record(stream)
    info2 = _lib.execute(handle, bc.desc, bc.args, _lib.PHASE_BOUNDARY, use_local_maps)
    ev[4].record(stream)
    report.launches = info.launches + info2.launches
    for name, a, b in zip(ExecutionReport.PHASES, ev[:-1], ev[1:]):
        report.phase_seconds.add_events(name, a, b)
    return report


class TiledRunner:
    """Pre-bound tiled execution of one (schedule, chain, datasets) triple.

    The steady-state form of :func:`execute_schedule` for time-stepping
    drivers: validation and plan building happen once; ``__call__`` issues
    the colour-phase launches of both regions (no halo exchange) with no host
    synchronisation, so it can be captured into a CUDA graph (``graph``).
    """

    def __init__(self, schedule, chain: LoopChain, bindings, datasets: dict,
                 registry: KernelRegistry, use_local_maps: bool = True, repeats: int = 1):
        from . import _lib
        if schedule.fingerprint != chain.fingerprint:
            raise StaleScheduleError("schedule was inspected for a different chain")
        check_bindings(chain, bindings, datasets)
        self._lib = _lib
        self.bound = _bind(chain, bindings, datasets, registry)
        self.handle = schedule.device_handle(chain)
        self.use_local_maps = use_local_maps
        self.repeats = repeats
        # build the execution plan outside any capture, without executing the
        # chain (the datasets are untouched until the first call)
        info = _lib.prepare(self.handle, self.bound.desc, self.bound.args,
                            _lib.PHASE_CORE | _lib.PHASE_BOUNDARY, repeats, use_local_maps)
        self.launches_per_call = info.launches
        self.executor = {0: "global", 1: "staged", 2: "dataflow"}[info.staged]
        self.smem_bytes = info.smem_bytes
        self.queue_order = ("wavefront" if info.wave_order else "colour-major") \
            if info.staged == 2 else None
        self.wide_build = bool(info.wide_build)

    def __call__(self):
        """Execute the chain ``repeats`` times (one persistent launch when dataflow)."""
        if self.repeats == 1:
            return self._lib.execute(self.handle, self.bound.desc, self.bound.args,
                                     self._lib.PHASE_CORE | self._lib.PHASE_BOUNDARY,
                                     self.use_local_maps)
        return self._lib.execute_repeat(self.handle, self.bound.desc, self.bound.args,
                                        self.repeats, self.use_local_maps)

    def with_exchange(self, exchange):
        """One chain execution around a halo exchange (Alg. 2 order):
        ``begin()``, core colour classes, ``end()``, boundary colour classes."""
        lib = self._lib
        exchange.begin()
        a = lib.execute(self.handle, self.bound.desc, self.bound.args, lib.PHASE_CORE,
                        self.use_local_maps)
        exchange.end()
        b = lib.execute(self.handle, self.bound.desc, self.bound.args, lib.PHASE_BOUNDARY,
                        self.use_local_maps)
        return a.launches + b.launches

    def graph(self, repeats: int = 1):
        """CUDA graph replaying ``repeats`` chain executions back to back.

        Capturing executes nothing: the plan was built by the constructor, so
        the datasets change only when the graph is replayed."""
        import torch
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(repeats):
                self()
        return g


class UntiledRunner:
    """Pre-bound :func:`execute_untiled` (the GPU "original version" baseline)."""

    def __init__(self, chain: LoopChain, bindings, datasets: dict, registry: KernelRegistry):
        from . import _lib
        check_bindings(chain, bindings, datasets)
        self._lib = _lib
        self.bound = _bind(chain, bindings, datasets, registry)
        self.launches_per_call = self().launches

    def __call__(self):
        return self._lib.execute_untiled(self.bound.desc, self.bound.args)


# -- result comparison (executor.py:250-273) ---------------------------------------------

def _host(values) -> np.ndarray:
    if hasattr(values, "detach"):
        return values.detach().cpu().numpy()
    return np.asarray(values)


def integer_valued(values) -> bool:
    v = _host(values)
    return bool(np.all(v == np.rint(v)))


def diff_datasets(reference: dict, candidate: dict, rtol: float = 1e-12,
                  limit: int = 10) -> list[tuple]:
    """First ``limit`` (dataset, element, ref, got) mismatches; integer-valued
    reference data compared exactly, else within ``rtol``."""
    diffs = []
    for name in sorted(reference):
        ref, got = _host(reference[name].values), _host(candidate[name].values)
        if integer_valued(ref):
            bad = np.flatnonzero(ref != got)
        else:
            bad = np.flatnonzero(~np.isclose(got, ref, rtol=rtol, atol=0.0))
        k = reference[name].values_per_element
        for flat in bad[:limit - len(diffs)]:
            diffs.append((name, int(flat // k), float(ref[flat]), float(got[flat])))
        if len(diffs) >= limit:
            break
    return diffs
