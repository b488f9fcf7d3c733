"""ctypes binding of libhubgpu.so (include/hubgpu.h).

The library is built in-tree (``make -C paper_1704_06258_b200/csrc``) and is
the ONLY compute path of this package: there is no CPU fallback.  Loading it
needs no GPU; every compute entry point raises ``RuntimeError`` when no CUDA
device is visible.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import threading
import weakref
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libhubgpu.so"
# tuning only (tools/ab_k3.py): another in-tree build of the same library
if os.environ.get("HUBGPU_LIB_VARIANT"):
    LIB_PATH = LIB_PATH.with_name(f"libhubgpu_{os.environ['HUBGPU_LIB_VARIANT']}.so")

HG_OK, HG_EARG, HG_ECUDA, HG_ENODEV, HG_ESTATE = 0, 1, 2, 3, 4
HG_HOST, HG_DEVICE = 0, 1
FLAG_SYMMETRIC, FLAG_WEIGHTS_EXACT, FLAG_TENSOR_OK = 1, 2, 4
FIT_AUTO, FIT_FP64, FIT_TENSOR, FIT_TC_PAIR, FIT_TC_PAIR_FULL = 0, 1, 2, 5, 6
RNG_MODES = {"replay": 0, "philox": 1}  # hg_ga_params.rng
FIT_NAMES = {"auto": FIT_AUTO, "fp64": FIT_FP64, "tensor": FIT_TENSOR, "tensor-pair": FIT_TC_PAIR,
             "tensor-pair-full": FIT_TC_PAIR_FULL}

_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_u64p = C.POINTER(C.c_uint64)
_u8p = C.POINTER(C.c_uint8)
_f64p = C.POINTER(C.c_double)
_vp = C.c_void_p


class GaParamsC(C.Structure):
    _fields_ = [("islands_total", C.c_int32), ("island_lo", C.c_int32),
                ("island_hi", C.c_int32), ("pop_size", C.c_int32),
                ("strength", C.c_int32), ("strict_paper", C.c_int32), ("rng", C.c_int32),
                ("seed", C.c_uint64)]


# name -> (restype, argtypes); the exported surface of include/hubgpu.h
SIGNATURES = {
    "hg_last_error": (C.c_char_p, []),
    "hg_version": (C.c_int, []),
    "hg_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "hg_instance_create": (C.c_int, [C.c_int, C.c_int, C.c_int, _f64p, _f64p, _f64p, _f64p,
                                     C.c_double, _i64p, C.c_double, C.c_double, C.c_double,
                                     _vp, C.POINTER(_vp)]),
    "hg_instance_free": (None, [_vp]),
    "hg_instance_info": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                   C.POINTER(C.c_int)]),
    "hg_instance_stream": (C.c_int, [_vp, C.POINTER(_vp)]),
    "hg_instance_set_fitness": (C.c_int, [_vp, C.c_int]),
    "hg_instance_set_exact": (C.c_int, [_vp, C.c_int]),
    "hg_pairwise_leaves": (C.c_int, [C.c_int64, C.POINTER(C.c_uint32), C.c_int,
                                     C.POINTER(C.c_int)]),
    "hg_instance_exact": (C.c_int, [_vp, C.POINTER(C.c_int)]),
    "hg_instance_fitness": (C.c_int, [_vp, C.POINTER(C.c_int)]),
    "hg_synchronize": (C.c_int, [_vp]),
    "hg_allocate": (C.c_int, [_vp, C.c_int64, _i64p, _i64p]),
    "hg_evaluate": (C.c_int, [_vp, C.c_int64, _vp, _vp, _vp]),  # int64*, int64*, double*
    "hg_evaluate_unique": (C.c_int, [_vp, C.c_int64, _i64p, _f64p, _i64p]),
    "hg_pop_create": (C.c_int, [_vp, C.c_int64, C.POINTER(_vp)]),
    "hg_pop_free": (None, [_vp]),
    "hg_pop_load_hubs": (C.c_int, [_vp, C.c_int64, _vp, C.c_int]),
    "hg_pop_evaluate": (C.c_int, [_vp, C.c_int64]),
    "hg_pop_read": (C.c_int, [_vp, C.c_int64, _vp, C.c_int]),
    "hg_pop_launches_per_evaluate": (C.c_int, [_vp]),
    "hg_pop_last_fitness_ms": (C.c_int, [_vp, C.POINTER(C.c_float)]),
    "hg_pop_last_allocate_ms": (C.c_int, [_vp, C.POINTER(C.c_float)]),
    "hg_debug_tc_timing": (C.c_int, [_u64p]),
    "hg_debug_tc_trace": (C.c_int, [_u64p]),
    "hg_launch_count": (C.c_int, [_u64p]),
    "hg_fitness_work": (C.c_int, [_vp, C.c_int64, _f64p]),
    "hg_correct": (C.c_int, [_vp, C.c_int64, _u8p, _i64p]),
    "hg_crossover": (C.c_int, [C.c_int, C.c_int, C.c_int64, _u8p, _u8p, _i64p, _u8p, _u8p]),
    "hg_swap": (C.c_int, [C.c_int, C.c_int, C.c_int64, _u8p, _i64p, _i64p, _u8p]),
    "hg_ga_create": (C.c_int, [_vp, C.POINTER(GaParamsC), C.POINTER(_vp)]),
    "hg_ga_free": (None, [_vp]),
    "hg_ga_reseed": (C.c_int, [_vp, C.c_uint64]),
    "hg_ga_begin_round": (C.c_int, [_vp, _i64p]),
    "hg_ga_generations": (C.c_int, [_vp, C.c_int]),
    "hg_ga_round_results": (C.c_int, [_vp, _f64p, _i64p]),
    "hg_ga_last_children": (C.c_int, [_vp, _i64p, _f64p]),
    "hg_ga_draw_counters": (C.c_int, [_vp, _u64p]),
    "hg_ga_launches_per_generation": (C.c_int, [_vp]),
    "hg_generate_urand": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_uint64, _f64p, _f64p]),
    "hg_restricted_optimum": (C.c_int, [_vp, C.c_uint64, _i64p, _f64p, _u64p]),
    "hg_philox4x32_10": (None, [C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                C.POINTER(C.c_uint32)]),
    "hg_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(_vp)]),
    "hg_host_free": (None, [_vp]),
}

_lib = None
_lock = threading.Lock()


def load() -> C.CDLL:
    """Load libhubgpu.so (once).  Raises if it was not built: there is no
    fallback path."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with "
                    "`make -C paper_1704_06258_b200/csrc` (or __graft_entry__.build())")
            lib = C.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


class HubGpuError(RuntimeError):
    pass


def check(rc: int) -> None:
    if rc == HG_OK:
        return
    msg = load().hg_last_error().decode(errors="replace")
    if rc == HG_EARG:
        raise ValueError(msg)
    if rc == HG_ENODEV:
        raise HubGpuError(msg)
    raise HubGpuError(f"libhubgpu error {rc}: {msg}")


def launch_count() -> int:
    """Kernels libhubgpu has launched in this process (hg_launch_count)."""
    v = C.c_uint64()
    check(load().hg_launch_count(C.byref(v)))
    return v.value


def device_count() -> int:
    c = C.c_int(0)
    check(load().hg_device_count(C.byref(c)))
    return c.value


_device = int(os.environ.get("HUBGPU_DEVICE", os.environ.get("LOCAL_RANK", "0")))
# transfer-term kernel for new device instances: auto (tensor cores when the
# flows allow the exact u8 GEMM), fp64 (K3 gather) or tensor (K3-TC/P, also
# named tensor-pair)
_fit_default = FIT_NAMES[os.environ.get("HUBGPU_FITNESS", "auto")]


def set_fitness_default(kind: str) -> None:
    """A FIT_NAMES key for device instances created from now on (a tensor-core
    choice the instance cannot run -- non-integer flows, p > 128 or
    n > 16384 -- leaves it on 'auto')."""
    global _fit_default
    _fit_default = FIT_NAMES[kind]


_exact_default = os.environ.get("HUBGPU_EXACT", "0") not in ("", "0")


def set_exact_default(on: bool) -> None:
    """Cost sums in numpy's pairwise order (bit-identical to the reference's
    np.sum) for every evaluation from now on; off: fixed-order sums within
    ~1 ulp.  GA objects keep the mode they were created with."""
    global _exact_default
    _exact_default = bool(on)


def exact_default() -> bool:
    return _exact_default


def set_device(index: int) -> None:
    """Select the CUDA device new device instances are created on."""
    global _device
    _device = int(index)


def current_device() -> int:
    return _device


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(ctype)


# ---------------------------------------------------------------------------
# device-resident instances, cached on the (immutable) Instance object
# ---------------------------------------------------------------------------


class DeviceInstance:
    """Owns an hg_inst handle: HBM-resident dist / flow / derived vectors."""

    def __init__(self, inst, device: int, stream=None):
        lib = load()
        self.n, self.p = inst.n, inst.p
        self.device = device
        h = _vp()
        dist = np.ascontiguousarray(inst.dist, dtype=np.float64)
        flow = np.ascontiguousarray(inst.flow, dtype=np.float64)
        out_flow = np.ascontiguousarray(inst.out_flow, dtype=np.float64)
        in_flow = np.ascontiguousarray(inst.in_flow, dtype=np.float64)
        rank = np.ascontiguousarray(inst.middle_rank, dtype=np.int64)
        check(lib.hg_instance_create(device, inst.n, inst.p, ptr(dist, _f64p), ptr(flow, _f64p),
                                     ptr(out_flow, _f64p), ptr(in_flow, _f64p),
                                     float(inst.total_flow), ptr(rank, _i64p),
                                     float(inst.chi), float(inst.alpha), float(inst.delta),
                                     stream, C.byref(h)))
        self.handle = h
        self._fin = weakref.finalize(self, lib.hg_instance_free, h)
        n_, p_, flags = C.c_int(), C.c_int(), C.c_int()
        check(lib.hg_instance_info(h, C.byref(n_), C.byref(p_), C.byref(flags)))
        self.flags = flags.value
        if _fit_default == FIT_FP64:
            self.set_fitness(_fit_default)
        elif _fit_default != FIT_AUTO and self.flags & FLAG_TENSOR_OK:
            try:
                self.set_fitness(_fit_default)
            except ValueError:
                pass  # this variant does not fit the instance: keep auto

    def set_fitness(self, kind: int) -> None:
        check(load().hg_instance_set_fitness(self.handle, int(kind)))

    def set_exact(self, on: bool) -> None:
        check(load().hg_instance_set_exact(self.handle, int(bool(on))))
        self._exact = bool(on)

    @property
    def exact(self) -> bool:
        v = C.c_int()
        check(load().hg_instance_exact(self.handle, C.byref(v)))
        return bool(v.value)

    def sync_exact(self) -> None:
        """Follow the module default (set_exact_default)."""
        if getattr(self, "_exact", None) != _exact_default:
            self.set_exact(_exact_default)

    @property
    def fitness_kernel(self) -> str:
        """'fp64', 'tensor-pair' (K3-TC/P on the triangular fold of W when the
        costs are symmetric and the sums fixed-order) or 'tensor-pair-full'."""
        k = C.c_int()
        check(load().hg_instance_fitness(self.handle, C.byref(k)))
        return {v: n for n, v in FIT_NAMES.items()}[k.value]

    @property
    def stream(self) -> int:
        s = _vp()
        check(load().hg_instance_stream(self.handle, C.byref(s)))
        return s.value or 0

    def synchronize(self) -> None:
        check(load().hg_synchronize(self.handle))

    def allocate(self, hubs: np.ndarray) -> np.ndarray:
        hubs = np.ascontiguousarray(hubs, dtype=np.int64).reshape(-1, self.p)
        out = np.empty((hubs.shape[0], self.n), dtype=np.int64)
        check(load().hg_allocate(self.handle, hubs.shape[0], ptr(hubs, _i64p), ptr(out, _i64p)))
        return out

    def evaluate(self, hubs: np.ndarray, alloc: np.ndarray | None = None,
                 unique: bool = False) -> np.ndarray:
        self.sync_exact()
        hubs = np.ascontiguousarray(hubs, dtype=np.int64).reshape(-1, self.p)
        B = hubs.shape[0]
        # results land by DMA in a pooled page-locked buffer (a pageable
        # destination costs the driver a staging copy)
        out = pinned_array((B, 4), np.float64)
        if unique and alloc is None:
            groups = C.c_int64()
            check(load().hg_evaluate_unique(self.handle, B, ptr(hubs, _i64p), ptr(out, _f64p),
                                            C.byref(groups)))
            self.last_groups = groups.value
            return out
        ap = None
        if alloc is not None:
            alloc = np.ascontiguousarray(alloc, dtype=np.int64).reshape(B, self.n)
            ap = alloc.ctypes.data
        # plain addresses: the hot end-to-end path skips ctypes pointer objects
        check(load().hg_evaluate(self.handle, B, hubs.ctypes.data, ap, out.ctypes.data))
        return out

    def mma_ops(self, B: int) -> float:
        """int8 tensor operations the fitness kernel issues for B hub sets."""
        v = C.c_double()
        check(load().hg_fitness_work(self.handle, int(B), C.byref(v)))
        return v.value

    def correct(self, masks: np.ndarray) -> np.ndarray:
        masks = np.ascontiguousarray(masks, dtype=np.uint8).reshape(-1, self.n)
        out = np.empty((masks.shape[0], self.p), dtype=np.int64)
        check(load().hg_correct(self.handle, masks.shape[0], ptr(masks, _u8p), ptr(out, _i64p)))
        return out


_inst_lock = threading.Lock()


def device_instance(inst, device: int | None = None) -> DeviceInstance:
    """The instance's device copy on `device` (built once, also when several
    threads ask at the same time: the Instance is shareable, hm/model.py:35)."""
    dev = _device if device is None else int(device)
    cache = inst.__dict__.get("_hubgpu_dev")
    d = cache.get(dev) if cache is not None else None
    if d is not None:
        return d
    with _inst_lock:
        cache = inst.__dict__.get("_hubgpu_dev")
        if cache is None:
            cache = {}
            object.__setattr__(inst, "_hubgpu_dev", cache)
        d = cache.get(dev)
        if d is None:
            d = DeviceInstance(inst, dev)
            cache[dev] = d
    return d


# ---------------------------------------------------------------------------
# population and GA handles
# ---------------------------------------------------------------------------


class DevicePopulation:
    """A device-resident population buffer (hg_pop) bound to one instance."""

    def __init__(self, dinst: DeviceInstance, capacity: int):
        lib = load()
        self.dinst = dinst
        self.capacity = int(capacity)
        h = _vp()
        check(lib.hg_pop_create(dinst.handle, self.capacity, C.byref(h)))
        self.handle = h
        self._fin = weakref.finalize(self, lib.hg_pop_free, h)

    def load_hubs(self, hubs32, where: int = HG_HOST, count: int | None = None) -> None:
        """hubs32: int32 numpy array (host) or a device pointer (int) with where=HG_DEVICE."""
        if where == HG_HOST:
            hubs32 = np.ascontiguousarray(hubs32, dtype=np.int32).reshape(-1, self.dinst.p)
            count = hubs32.shape[0]
            p = hubs32.ctypes.data
        else:
            p = int(hubs32)
        check(load().hg_pop_load_hubs(self.handle, int(count), p, where))

    def evaluate(self, count: int) -> None:
        self.dinst.sync_exact()
        check(load().hg_pop_evaluate(self.handle, int(count)))

    def read(self, count: int, out=None, where: int = HG_HOST):
        if where == HG_HOST:
            if out is None:
                out = np.empty((count, 4), dtype=np.float64)
            check(load().hg_pop_read(self.handle, int(count), out.ctypes.data, HG_HOST))
            return out
        check(load().hg_pop_read(self.handle, int(count), int(out), HG_DEVICE))
        return out

    def last_fitness_ms(self) -> float:
        v = C.c_float()
        check(load().hg_pop_last_fitness_ms(self.handle, C.byref(v)))
        return v.value

    def last_allocate_ms(self) -> float:
        v = C.c_float()
        check(load().hg_pop_last_allocate_ms(self.handle, C.byref(v)))
        return v.value

    @property
    def launches_per_evaluate(self) -> int:
        return load().hg_pop_launches_per_evaluate(self.handle)


class DeviceGa:
    """Islands [lo, hi) of an island-GA run on one device (hg_ga)."""

    def __init__(self, dinst: DeviceInstance, islands_total: int, lo: int, hi: int,
                 pop_size: int, strength: int, strict: bool, seed: int, rng: str = "replay"):
        lib = load()
        self.dinst = dinst
        self.lo, self.hi = lo, hi
        self.pop = pop_size
        prm = GaParamsC(islands_total, lo, hi, pop_size, strength, 1 if strict else 0,
                        RNG_MODES[rng], seed & ((1 << 64) - 1))
        h = _vp()
        dinst.sync_exact()  # the GA keeps the summation mode it is created with
        self.exact = dinst.exact
        check(lib.hg_ga_create(dinst.handle, C.byref(prm), C.byref(h)))
        self.handle = h
        self._fin = weakref.finalize(self, lib.hg_ga_free, h)

    @property
    def n_local(self) -> int:
        return self.hi - self.lo

    def reseed(self, seed: int) -> None:
        check(load().hg_ga_reseed(self.handle, seed & ((1 << 64) - 1)))

    def begin_round(self, hubs: np.ndarray) -> None:
        hubs = np.ascontiguousarray(hubs, dtype=np.int64)
        check(load().hg_ga_begin_round(self.handle, ptr(hubs, _i64p)))

    def generations(self, count: int) -> None:
        check(load().hg_ga_generations(self.handle, int(count)))

    def round_results(self):
        raw = np.empty(self.n_local, dtype=np.float64)
        hubs = np.empty((self.n_local, self.dinst.p), dtype=np.int64)
        check(load().hg_ga_round_results(self.handle, ptr(raw, _f64p), ptr(hubs, _i64p)))
        return raw, hubs

    def last_children(self):
        B = self.n_local * self.pop
        hubs = np.empty((B, self.dinst.p), dtype=np.int64)
        raw = np.empty(B, dtype=np.float64)
        check(load().hg_ga_last_children(self.handle, ptr(hubs, _i64p), ptr(raw, _f64p)))
        return hubs, raw

    def draw_counters(self) -> np.ndarray:
        out = np.empty((self.n_local, 3), dtype=np.uint64)
        check(load().hg_ga_draw_counters(self.handle, ptr(out, _u64p)))
        return out

    @property
    def launches_per_generation(self) -> int:
        return load().hg_ga_launches_per_generation(self.handle)


def crossover_masks(a: np.ndarray, b: np.ndarray, cuts: np.ndarray, device: int | None = None):
    a = np.ascontiguousarray(a, dtype=np.uint8)
    b = np.ascontiguousarray(b, dtype=np.uint8)
    B, n = a.reshape(-1, a.shape[-1]).shape
    cuts = np.ascontiguousarray(cuts, dtype=np.int64).reshape(B)
    c1 = np.empty((B, n), dtype=np.uint8)
    c2 = np.empty((B, n), dtype=np.uint8)
    check(load().hg_crossover(_device if device is None else device, n, B, ptr(a, _u8p),
                              ptr(b, _u8p), ptr(cuts, _i64p), ptr(c1, _u8p), ptr(c2, _u8p)))
    return c1, c2


def swap_masks(masks: np.ndarray, r_close: np.ndarray, r_open: np.ndarray,
               device: int | None = None) -> np.ndarray:
    masks = np.ascontiguousarray(masks, dtype=np.uint8)
    B, n = masks.reshape(-1, masks.shape[-1]).shape
    rc = np.ascontiguousarray(r_close, dtype=np.int64).reshape(B)
    ro = np.ascontiguousarray(r_open, dtype=np.int64).reshape(B)
    out = np.empty((B, n), dtype=np.uint8)
    check(load().hg_swap(_device if device is None else device, n, B, ptr(masks, _u8p),
                         ptr(rc, _i64p), ptr(ro, _i64p), ptr(out, _u8p)))
    return out


# ---------------------------------------------------------------------------
# device generator, GPU restricted optimum
# ---------------------------------------------------------------------------


def generate_urand_arrays(n: int, p: int, seed: int, device: int | None = None):
    """(dist, flow) of generate_urand(n, p, seed, .) computed on the GPU
    (hm/io.py:188-210 bit for bit)."""
    dist = np.empty((n, n), dtype=np.float64)
    flow = np.empty((n, n), dtype=np.float64)
    check(load().hg_generate_urand(_device if device is None else int(device), int(n), int(p),
                                   int(seed) & 0xFFFFFFFFFFFFFFFF, ptr(dist, _f64p),
                                   ptr(flow, _f64p)))
    return dist, flow


def restricted_optimum(dinst: "DeviceInstance", limit: int):
    """(best hubs int64[p], best raw, C(n, p)) over every p-subset."""
    hubs = np.empty(dinst.p, dtype=np.int64)
    raw = C.c_double()
    count = C.c_uint64()
    dinst.sync_exact()
    check(load().hg_restricted_optimum(dinst.handle, int(limit), ptr(hubs, _i64p), C.byref(raw),
                                       C.byref(count)))
    return hubs, raw.value, count.value


def philox4x32_10(key, ctr) -> list[int]:
    """One Philox4x32-10 block (the GA's rng='philox' generator), host side."""
    k = (C.c_uint32 * 2)(*[int(v) & 0xFFFFFFFF for v in key])
    c = (C.c_uint32 * 4)(*[int(v) & 0xFFFFFFFF for v in ctr])
    out = (C.c_uint32 * 4)()
    load().hg_philox4x32_10(k, c, out)
    return list(out)


# ---------------------------------------------------------------------------
# pooled page-locked result buffers
# ---------------------------------------------------------------------------


class _PinnedPool:
    """Page-locked blocks by size; a block returns to the pool when the numpy
    array built on it (and every view of it) is garbage-collected.

    Each block is wrapped in an instance of a per-size ctypes array subclass
    whose ``__del__`` hands the block back: numpy arrays over it (and every
    view, numpy's base chain ends at the buffer exporter) keep that instance
    alive, so the block is reused only after its last view is gone.  (Cheaper
    than a weakref.finalize per array: ~2 us per result array.)"""

    KEEP = 8  # cached free blocks per size

    def __init__(self):
        self._free: dict[int, list[int]] = {}
        self._types: dict[int, type] = {}
        self._lock = threading.Lock()

    def _block_type(self, nbytes: int) -> type:
        t = self._types.get(nbytes)
        if t is None:
            pool = self

            def _del(block, _n=nbytes, _addressof=C.addressof):
                try:
                    pool._give_back(_n, _addressof(block))
                except Exception:  # interpreter shutdown: the process frees it
                    pass

            t = type(f"_PinnedBlock{nbytes}", (C.c_char * nbytes,), {"__del__": _del})
            self._types[nbytes] = t
        return t

    def array(self, shape, dtype) -> np.ndarray:
        dtype = np.dtype(dtype)
        nbytes = math.prod(shape) * dtype.itemsize
        if nbytes == 0:
            return np.empty(shape, dtype=dtype)
        with self._lock:
            blocks = self._free.get(nbytes)
            addr = blocks.pop() if blocks else None
        if addr is None:
            p = _vp()
            check(load().hg_host_alloc(nbytes, C.byref(p)))
            addr = p.value
        raw = self._block_type(nbytes).from_address(addr)
        return np.frombuffer(raw, dtype=dtype).reshape(shape)

    def _give_back(self, nbytes: int, addr: int) -> None:
        with self._lock:
            blocks = self._free.setdefault(nbytes, [])
            if len(blocks) < self.KEEP:
                blocks.append(addr)
                return
        load().hg_host_free(addr)


_pinned = _PinnedPool()


def pinned_array(shape, dtype) -> np.ndarray:
    return _pinned.array(shape, dtype)


def pairwise_leaves(m: int) -> np.ndarray:
    """The exact mode's leaf table for an m-term np.sum (hg_pairwise_leaves)."""
    cnt = C.c_int()
    check(load().hg_pairwise_leaves(int(m), None, 0, C.byref(cnt)))
    out = np.zeros(max(cnt.value, 1), dtype=np.uint32)
    check(load().hg_pairwise_leaves(int(m), out.ctypes.data_as(C.POINTER(C.c_uint32)),
                                    out.size, C.byref(cnt)))
    return out[:cnt.value]
