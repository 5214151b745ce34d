"""ctypes binding of ``libltcuda.so`` (C ABI: ``include/looptile_cuda.h``).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).
There is no fallback: if the shared object is missing, importing any compute
entry point raises ``ImportError``; if no B200 is visible, creating the device
context raises ``ExecutionError`` from ``LT_E_CUDA``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
import weakref

import numpy as np

from .errors import (ColoringLimitError, DepthExceededError, ExecutionError,
                     InspectionError, InvalidChainError, PartitionBugError,
                     StaleScheduleError)

LIB_PATH = os.environ.get("LT_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libltcuda.so")

LT_OK = 0
_ERRORS = {
    -1: InvalidChainError,
    -2: DepthExceededError,
    -3: InspectionError,
    -4: ColoringLimitError,
    -5: ExecutionError,
    -6: StaleScheduleError,
    -7: PartitionBugError,
    -8: ValueError,
    -9: ExecutionError,  # CUDA failure / no device: no CPU fallback exists
}
PHASE_CORE, PHASE_BOUNDARY = 1, 2


class LtSpace(C.Structure):
    _fields_ = [("core", C.c_int64), ("boundary", C.c_int64), ("nonexec", C.c_int64)]


class LtMap(C.Structure):
    _fields_ = [("source", C.c_int32), ("target", C.c_int32), ("arity", C.c_int32),
                ("reserved", C.c_int32), ("values", C.c_void_p)]


class LtDesc(C.Structure):
    _fields_ = [("map", C.c_int32), ("mode", C.c_int32)]


class LtLoop(C.Structure):
    _fields_ = [("space", C.c_int32), ("n_desc", C.c_int32), ("kernel", C.c_int32),
                ("reserved", C.c_int32), ("desc", C.POINTER(LtDesc))]


class LtChain(C.Structure):
    _fields_ = [("n_spaces", C.c_int32), ("n_maps", C.c_int32), ("n_loops", C.c_int32),
                ("depth", C.c_int32), ("spaces", C.POINTER(LtSpace)),
                ("maps", C.POINTER(LtMap)), ("loops", C.POINTER(LtLoop))]


class LtArg(C.Structure):
    _fields_ = [("values", C.c_void_p), ("n_elements", C.c_int64), ("vpe", C.c_int32),
                ("reserved", C.c_int32)]


class LtScheduleInfo(C.Structure):
    _fields_ = [("mode", C.c_int32), ("n_loops", C.c_int32), ("n_tiles", C.c_int32),
                ("n_core_tiles", C.c_int32), ("n_boundary_tiles", C.c_int32),
                ("rounds", C.c_int32), ("n_colors", C.c_int32), ("reserved", C.c_int32),
                ("partition_s", C.c_double), ("coloring_s", C.c_double),
                ("projection_tiling_s", C.c_double), ("local_maps_s", C.c_double),
                ("total_s", C.c_double)]


class LtExecInfo(C.Structure):
    _fields_ = [("launches", C.c_int32), ("n_colors", C.c_int32), ("elements", C.c_int64),
                ("staged", C.c_int32), ("smem_bytes", C.c_int32), ("wave_order", C.c_int32),
                ("wide_build", C.c_int32)]


# every symbol the header declares, with (restype, argtypes)
_P = C.c_void_p
_I32P = C.POINTER(C.c_int32)
_I64P = C.POINTER(C.c_int64)
SIGNATURES = {
    "lt_abi_version": (C.c_int, []),
    "lt_last_error": (C.c_char_p, []),
    "lt_ctx_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "lt_ctx_destroy": (C.c_int, [_P]),
    "lt_ctx_set_stream": (C.c_int, [_P, _P]),
    "lt_ctx_synchronize": (C.c_int, [_P]),
    "lt_ctx_forget_map": (C.c_int, [_P, _P]),
    "lt_kernel_lookup": (C.c_int, [C.c_char_p, _I32P, _I32P]),
    "lt_kernel_count": (C.c_int, []),
    "lt_kernel_name": (C.c_char_p, [C.c_int32]),
    "lt_ctx_set_kernel_params": (C.c_int, [_P, C.c_int32, _P, C.c_int64]),
    "lt_invert_map": (C.c_int, [_P, _P, C.c_int64, C.c_int32, C.c_int64, _P, _P]),
    "lt_inspect": (C.c_int, [_P, C.POINTER(LtChain), C.c_int64, C.c_int32, C.POINTER(_P)]),
    "lt_schedule_import": (C.c_int, [_P, C.POINTER(LtChain), C.c_int32, C.c_int32, _P, _P,
                                     C.c_int32, C.POINTER(_P), C.POINTER(_P),
                                     C.POINTER(_P)]),
    "lt_schedule_info_get": (C.c_int, [_P, C.POINTER(LtScheduleInfo)]),
    "lt_schedule_tiles": (C.c_int, [_P, _P, _P]),
    "lt_schedule_lists": (C.c_int, [_P, C.c_int32, _P, _P]),
    "lt_schedule_tile_of": (C.c_int, [_P, C.c_int32, C.POINTER(_P), _I64P]),
    "lt_schedule_local_map": (C.c_int, [_P, C.c_int32, C.c_int32, _P]),
    "lt_schedule_destroy": (C.c_int, [_P]),
    "lt_execute": (C.c_int, [_P, _P, C.POINTER(LtChain), C.POINTER(LtArg), C.c_int32,
                             C.c_int32, C.POINTER(LtExecInfo)]),
    "lt_execute_repeat": (C.c_int, [_P, _P, C.POINTER(LtChain), C.POINTER(LtArg), C.c_int32,
                                    C.c_int32, C.POINTER(LtExecInfo)]),
    "lt_prepare": (C.c_int, [_P, _P, C.POINTER(LtChain), C.POINTER(LtArg), C.c_int32,
                             C.c_int32, C.c_int32, C.POINTER(LtExecInfo)]),
    "lt_check_legality": (C.c_int, [_P, _P, C.POINTER(LtChain), _I64P, _I64P,
                                    C.POINTER(C.c_int32)]),
    "lt_execute_untiled": (C.c_int, [_P, C.POINTER(LtChain), C.POINTER(LtArg),
                                     C.POINTER(LtExecInfo)]),
    "lt_halo_pack": (C.c_int, [_P, _P, C.c_int32, _P, C.c_int64, _P]),
    "lt_halo_unpack": (C.c_int, [_P, _P, C.c_int32, _P, C.c_int64, _P]),
    "lt_rcm_order": (C.c_int, [C.c_int64, _P, _P, _P]),
    "lt_gather_rows": (C.c_int, [_P, _P, C.c_int32, _P, C.c_int64, _P]),
    "lt_partition_seed": (C.c_int, [_P, C.POINTER(LtSpace), C.c_int64, _P, _I32P, _I32P]),
    "lt_assign": (C.c_int, [_P, _P, C.c_int64, C.c_int32, _P, _P]),
    "lt_seed_adjacency": (C.c_int, [_P, _P, C.c_int64, C.c_int32, C.c_int64, _P, C.c_int32, _P,
                                    C.c_int64, _I64P]),
    "lt_color_tiles": (C.c_int, [C.c_int32, _P, C.c_int32, _P, C.c_int64, _P]),
    "lt_project": (C.c_int, [_P, C.POINTER(LtChain), C.c_int32, _P, _P, C.c_int32,
                             C.POINTER(_P), _P, _P, C.c_int64, _I64P]),
    "lt_tile_loop": (C.c_int, [_P, C.POINTER(LtChain), C.c_int32, C.POINTER(_P), _P, _P,
                               C.c_int32, C.c_int32, _P, C.c_int32, _P, C.c_int64, _I64P]),
}

_lib = None
_lock = threading.Lock()


def load() -> C.CDLL:
    """Load libltcuda.so once (raises ImportError when it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc sm_100a); "
                    f"the looptile B200 path has no CPU fallback")
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(status: int) -> None:
    if status != LT_OK:
        msg = load().lt_last_error().decode(errors="replace")
        raise _ERRORS.get(status, RuntimeError)(msg)


# ---- device context ------------------------------------------------------------

class Context:
    def __init__(self, device: int):
        self.device = device
        h = C.c_void_p()
        check(load().lt_ctx_create(device, C.byref(h)))
        self.handle = h

    def bind_stream(self):
        import torch
        stream = torch.cuda.current_stream(self.device).cuda_stream
        check(load().lt_ctx_set_stream(self.handle, C.c_void_p(stream)))
        return self.handle


_contexts: dict[int, Context] = {}


def context(device: int | None = None) -> Context:
    import torch
    if not torch.cuda.is_available():
        raise ExecutionError("no CUDA device available; the looptile B200 executor has "
                             "no CPU fallback")
    dev = torch.cuda.current_device() if device is None else int(device)
    ctx = _contexts.get(dev)
    if ctx is None:
        ctx = _contexts[dev] = Context(dev)
    return ctx


def forget_map(ptr: int) -> None:
    if _lib is None:
        return
    for ctx in list(_contexts.values()):
        _lib.lt_ctx_forget_map(ctx.handle, C.c_void_p(ptr))


# ---- kernels ---------------------------------------------------------------------

def kernel_lookup(name: str) -> tuple[int, int]:
    kid, nargs = C.c_int32(), C.c_int32()
    check(load().lt_kernel_lookup(name.encode(), C.byref(kid), C.byref(nargs)))
    return kid.value, nargs.value


def kernel_names() -> list[str]:
    lib = load()
    return [lib.lt_kernel_name(i).decode() for i in range(lib.lt_kernel_count())]


def set_kernel_params(kernel_id: int, params: np.ndarray, device: int | None = None) -> None:
    ctx = context(device)
    p = np.ascontiguousarray(params, dtype=np.float64)
    check(load().lt_ctx_set_kernel_params(ctx.handle, kernel_id, p.ctypes.data, len(p)))


# ---- chain marshalling -------------------------------------------------------------

class ChainDesc:
    """Keeps the ctypes image of a LoopChain (and the device map buffers) alive."""

    def __init__(self, chain, kernel_ids=None, device=None):
        spaces = list(chain.spaces)
        sidx = {s: i for i, s in enumerate(spaces)}
        midx = {id(m): i for i, m in enumerate(chain.maps)}
        self.space_index = sidx
        self.map_index = midx
        self.spaces = (LtSpace * len(spaces))(
            *[LtSpace(s.core_size, s.boundary_size, s.nonexec_size) for s in spaces])
        self.map_tensors = [m.device_values(device) for m in chain.maps]
        for m, t in zip(chain.maps, self.map_tensors):
            _register_map_finalizer(m, t)
        self.maps = (LtMap * max(len(chain.maps), 1))(
            *[LtMap(sidx[m.source], sidx[m.target], m.arity, 0, t.data_ptr())
              for m, t in zip(chain.maps, self.map_tensors)])
        self.descs = []
        loops = []
        for j, lp in enumerate(chain.loops):
            arr = (LtDesc * len(lp.descriptors))(
                *[LtDesc(-1 if d.map is None else midx[id(d.map)], d.mode.code)
                  for d in lp.descriptors])
            self.descs.append(arr)
            kid = -1 if kernel_ids is None else kernel_ids[j]
            loops.append(LtLoop(sidx[lp.space], len(lp.descriptors), kid, 0,
                                C.cast(arr, C.POINTER(LtDesc))))
        self.loops = (LtLoop * len(loops))(*loops)
        self.struct = LtChain(len(spaces), len(chain.maps), len(loops), chain.depth,
                              C.cast(self.spaces, C.POINTER(LtSpace)),
                              C.cast(self.maps, C.POINTER(LtMap)),
                              C.cast(self.loops, C.POINTER(LtLoop)))

    @property
    def ref(self):
        return C.byref(self.struct)


_finalized: set[int] = set()


def _register_map_finalizer(mesh_map, tensor) -> None:
    ptr = tensor.data_ptr()
    if ptr in _finalized:
        return
    _finalized.add(ptr)

    def _drop(p=ptr):
        _finalized.discard(p)
        forget_map(p)

    weakref.finalize(mesh_map, _drop)


# ---- inspector ------------------------------------------------------------------------

def invert_map(mesh_map) -> tuple[np.ndarray, np.ndarray]:
    import torch
    ctx = context()
    vals = mesh_map.device_values()
    n_src, n_tgt, a = mesh_map.source.total, mesh_map.target.total, mesh_map.arity
    off = torch.empty(n_tgt + 1, dtype=torch.int32, device=vals.device)
    src = torch.empty(max(n_src * a, 1), dtype=torch.int32, device=vals.device)
    check(load().lt_invert_map(ctx.bind_stream(), vals.data_ptr(), n_src, a, n_tgt,
                               off.data_ptr(), src.data_ptr()))
    return (off.cpu().numpy().astype(np.int64),
            src[:n_src * a].cpu().numpy().astype(np.int64))


class ScheduleHandle:
    """Owns an ``lt_schedule*``; destroyed with the Python object."""

    def __init__(self, handle: C.c_void_p, ctx: Context, chain_desc: ChainDesc):
        self.handle = handle
        self.ctx = ctx
        self.chain_desc = chain_desc  # keeps device map buffers alive
        self._fin = weakref.finalize(self, _destroy_schedule, handle.value)

    def info(self) -> LtScheduleInfo:
        out = LtScheduleInfo()
        check(load().lt_schedule_info_get(self.handle, C.byref(out)))
        return out

    def tiles(self, n_tiles: int) -> tuple[np.ndarray, np.ndarray]:
        colors = np.empty(n_tiles, dtype=np.int32)
        regions = np.empty(n_tiles, dtype=np.int32)
        check(load().lt_schedule_tiles(self.handle, colors.ctypes.data, regions.ctypes.data))
        return colors, regions

    def lists(self, loop: int, n_tiles: int, n_elements: int) -> tuple[np.ndarray, np.ndarray]:
        offsets = np.empty(n_tiles + 1, dtype=np.int32)
        elements = np.empty(max(n_elements, 1), dtype=np.int32)
        check(load().lt_schedule_lists(self.handle, loop, offsets.ctypes.data,
                                       elements.ctypes.data))
        return offsets, elements[:n_elements]

    def local_map(self, loop: int, map_index: int, size: int) -> np.ndarray:
        out = np.empty(max(size, 1), dtype=np.int32)
        check(load().lt_schedule_local_map(self.handle, loop, map_index, out.ctypes.data))
        return out[:size]


def _destroy_schedule(ptr):
    if _lib is not None and ptr:
        _lib.lt_schedule_destroy(C.c_void_p(ptr))


def inspect(chain, ts: int, mode_code: int) -> ScheduleHandle:
    ctx = context()
    cd = ChainDesc(chain, device=ctx.device)
    h = C.c_void_p()
    check(load().lt_inspect(ctx.bind_stream(), cd.ref, int(ts), mode_code, C.byref(h)))
    return ScheduleHandle(h, ctx, cd)


def import_schedule(chain, mode_code: int, colors, regions, rounds: int,
                    lists: list[tuple[np.ndarray, np.ndarray]]) -> ScheduleHandle:
    ctx = context()
    cd = ChainDesc(chain, device=ctx.device)
    n_tiles = len(colors)
    col = np.ascontiguousarray(colors, dtype=np.int32)
    reg = np.ascontiguousarray(regions, dtype=np.int32)
    keep = []
    offs = (C.c_void_p * len(lists))()
    elems = (C.c_void_p * len(lists))()
    for j, (o, e) in enumerate(lists):
        o = np.ascontiguousarray(o, dtype=np.int32)
        e = np.ascontiguousarray(e, dtype=np.int32)
        if len(e) == 0:
            e = np.zeros(1, dtype=np.int32)
        keep += [o, e]
        offs[j] = o.ctypes.data
        elems[j] = e.ctypes.data
    h = C.c_void_p()
    check(load().lt_schedule_import(ctx.bind_stream(), cd.ref, mode_code, n_tiles,
                                    col.ctypes.data, reg.ctypes.data, rounds, offs, elems,
                                    C.byref(h)))
    return ScheduleHandle(h, ctx, cd)


# ---- step-level inspector ------------------------------------------------------------

def _dev_i32(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(
        torch.device("cuda", torch.cuda.current_device()))


def _pairs_call(fn, *args):
    cap = 1 << 16
    while True:
        buf = np.empty(cap, dtype=np.int64)
        n = C.c_int64()
        check(fn(*args, buf.ctypes.data, cap, C.byref(n)))
        if n.value <= cap:
            v = buf[:n.value]
            return [(int(x >> 32), int(x & 0xffffffff)) for x in v]
        cap = n.value


def partition_seed(space, ts: int) -> tuple[np.ndarray, int, int]:
    import torch
    ctx = context()
    sig = torch.empty(max(space.total, 1), dtype=torch.int32, device="cuda")
    m, k = C.c_int32(), C.c_int32()
    sp = LtSpace(space.core_size, space.boundary_size, space.nonexec_size)
    check(load().lt_partition_seed(ctx.bind_stream(), C.byref(sp), int(ts), sig.data_ptr(),
                                   C.byref(m), C.byref(k)))
    return sig[:space.total].cpu().numpy().astype(np.int64), m.value, k.value


def assign(sigma: np.ndarray, n_tiles: int) -> tuple[np.ndarray, np.ndarray]:
    import torch
    ctx = context()
    s = _dev_i32(sigma)
    off = torch.empty(n_tiles + 1, dtype=torch.int32, device="cuda")
    el = torch.empty(max(len(sigma), 1), dtype=torch.int32, device="cuda")
    check(load().lt_assign(ctx.bind_stream(), s.data_ptr(), len(sigma), n_tiles, off.data_ptr(),
                           el.data_ptr()))
    return off.cpu().numpy().astype(np.int64), el[:len(sigma)].cpu().numpy().astype(np.int64)


def seed_adjacency(seed_map, sigma0: np.ndarray, n_tiles: int) -> list[tuple[int, int]]:
    ctx = context()
    vals = seed_map.device_values()
    s = _dev_i32(sigma0)
    return _pairs_call(load().lt_seed_adjacency, ctx.bind_stream(), vals.data_ptr(),
                       seed_map.source.total, seed_map.arity, seed_map.target.total, s.data_ptr(),
                       n_tiles)


def color_tiles(regions, mode_code: int, pairs) -> np.ndarray:
    reg = np.ascontiguousarray(regions, dtype=np.int32)
    pr = np.array([(a << 32) | b for a, b in pairs] or [0], dtype=np.int64)
    out = np.empty(len(reg), dtype=np.int32)
    check(load().lt_color_tiles(len(reg), reg.ctypes.data, mode_code, pr.ctypes.data,
                                len(pairs), out.ctypes.data))
    return out


class LoopChainDesc:
    """ctypes image of a one-loop chain (the loop's spaces and maps)."""

    def __init__(self, loop):
        import types
        spaces, maps = [loop.space], []
        for d in loop.descriptors:
            if d.map is not None:
                if all(m is not d.map for m in maps):
                    maps.append(d.map)
                for sp in (d.map.source, d.map.target):
                    if sp not in spaces:
                        spaces.append(sp)
        from .chain import Loop
        fake = types.SimpleNamespace(spaces=tuple(spaces), maps=tuple(maps), depth=1,
                                     loops=(Loop(0, loop.space, loop.descriptors, loop.kernel),))
        self.desc = ChainDesc(fake)
        self.spaces = spaces


def project(loop, sigma: np.ndarray, colors: np.ndarray, phi: dict) -> list[tuple[int, int]]:
    """phi: space name -> int64 numpy assignment (updated in place)."""
    import torch
    ctx = context()
    lc = LoopChainDesc(loop)
    bufs, present = [], np.zeros(len(lc.spaces), dtype=np.int32)
    for i, sp in enumerate(lc.spaces):
        if sp.name in phi:
            bufs.append(_dev_i32(phi[sp.name]))
            present[i] = 1
        else:
            bufs.append(torch.full((max(sp.total, 1),), -1, dtype=torch.int32, device="cuda"))
    ptrs = (C.c_void_p * len(bufs))(*[b.data_ptr() for b in bufs])
    sig, col = _dev_i32(sigma), _dev_i32(colors)
    pairs = _pairs_call(load().lt_project, ctx.bind_stream(), lc.desc.ref, 0, sig.data_ptr(),
                        col.data_ptr(), len(colors), ptrs, present.ctypes.data)
    for i, sp in enumerate(lc.spaces):
        if present[i]:
            phi[sp.name] = bufs[i][:sp.total].cpu().numpy().astype(np.int64)
    return pairs


def tile_loop(loop, colors: np.ndarray, phi: dict, detect: bool, tne: int = -1):
    import torch
    ctx = context()
    lc = LoopChainDesc(loop)
    bufs, present = [], np.zeros(len(lc.spaces), dtype=np.int32)
    for i, sp in enumerate(lc.spaces):
        if sp.name in phi:
            bufs.append(_dev_i32(phi[sp.name]))
            present[i] = 1
        else:
            bufs.append(torch.full((max(sp.total, 1),), -1, dtype=torch.int32, device="cuda"))
    ptrs = (C.c_void_p * len(bufs))(*[b.data_ptr() for b in bufs])
    col = _dev_i32(colors)
    out = torch.empty(max(loop.space.total, 1), dtype=torch.int32, device="cuda")
    pairs = _pairs_call(load().lt_tile_loop, ctx.bind_stream(), lc.desc.ref, 0, ptrs,
                        present.ctypes.data, col.data_ptr(), len(colors), tne, out.data_ptr(),
                        int(detect))
    return out[:loop.space.total].cpu().numpy().astype(np.int64), pairs


def gather_rows(mesh_map, elements: np.ndarray) -> np.ndarray:
    import torch
    ctx = context()
    el = _dev_i32(elements)
    out = torch.empty(max(len(elements) * mesh_map.arity, 1), dtype=torch.int32, device="cuda")
    check(load().lt_gather_rows(ctx.bind_stream(), mesh_map.device_values().data_ptr(),
                                mesh_map.arity, el.data_ptr(), len(elements), out.data_ptr()))
    return out[:len(elements) * mesh_map.arity].cpu().numpy().astype(np.int64)


# ---- executor ---------------------------------------------------------------------------

def make_args(arg_list) -> C.Array:
    """arg_list: [(tensor, n_elements, vpe), ...] loop-major, one per descriptor."""
    arr = (LtArg * len(arg_list))()
    for i, (t, n, k) in enumerate(arg_list):
        arr[i] = LtArg(t.data_ptr(), n, k, 0)
    return arr


def execute(sched: ScheduleHandle, chain_desc: ChainDesc, args, phases: int,
            use_local_maps: bool) -> LtExecInfo:
    info = LtExecInfo()
    check(load().lt_execute(sched.ctx.bind_stream(), sched.handle, chain_desc.ref, args,
                            phases, int(bool(use_local_maps)), C.byref(info)))
    return info


def execute_repeat(sched: ScheduleHandle, chain_desc: ChainDesc, args, repeats: int,
                   use_local_maps: bool) -> LtExecInfo:
    info = LtExecInfo()
    check(load().lt_execute_repeat(sched.ctx.bind_stream(), sched.handle, chain_desc.ref, args,
                                   int(repeats), int(bool(use_local_maps)), C.byref(info)))
    return info


def prepare(sched: ScheduleHandle, chain_desc: ChainDesc, args, phases: int, repeats: int,
            use_local_maps: bool) -> LtExecInfo:
    """Build the execution plan of a later execute/execute_repeat; launches nothing."""
    info = LtExecInfo()
    check(load().lt_prepare(sched.ctx.bind_stream(), sched.handle, chain_desc.ref, args,
                            int(phases), int(repeats), int(bool(use_local_maps)),
                            C.byref(info)))
    return info


def check_legality(sched: ScheduleHandle, chain_desc: ChainDesc) -> dict:
    pairs, red, ovf = C.c_int64(0), C.c_int64(0), C.c_int32(0)
    check(load().lt_check_legality(sched.ctx.bind_stream(), sched.handle, chain_desc.ref,
                                   C.byref(pairs), C.byref(red), C.byref(ovf)))
    out = {"pairs": pairs.value, "reductions": red.value}
    if ovf.value:
        out["overflow"] = True
    return out


def execute_untiled(chain_desc: ChainDesc, args) -> LtExecInfo:
    ctx = context()
    info = LtExecInfo()
    check(load().lt_execute_untiled(ctx.bind_stream(), chain_desc.ref, args, C.byref(info)))
    return info


def halo_pack(values, vpe: int, rows, out) -> None:
    ctx = context()
    check(load().lt_halo_pack(ctx.bind_stream(), values.data_ptr(), vpe, rows.data_ptr(),
                              rows.numel(), out.data_ptr()))


def halo_unpack(values, vpe: int, rows, src) -> None:
    ctx = context()
    check(load().lt_halo_unpack(ctx.bind_stream(), values.data_ptr(), vpe, rows.data_ptr(),
                                rows.numel(), src.data_ptr()))


# ---- host data-layout pass ----------------------------------------------------------------

def rcm_order(offsets: np.ndarray, neighbours: np.ndarray) -> np.ndarray:
    n = len(offsets) - 1
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    nb = np.ascontiguousarray(neighbours, dtype=np.int64)
    if len(nb) == 0:
        nb = np.zeros(1, dtype=np.int64)
    out = np.empty(max(n, 1), dtype=np.int64)
    check(load().lt_rcm_order(n, off.ctypes.data, nb.ctypes.data, out.ctypes.data))
    return out[:n]
