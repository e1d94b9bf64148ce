"""ctypes binding of the C-ABI in ``include/ttagg_b200.h``.

The shared library ``libttagg_b200.so`` is built in-tree by
``__graft_entry__.build()`` (nvcc, sm_100a).  There is no CPU fallback: if the
library is missing or no CUDA device is present, every operator raises.
"""

from __future__ import annotations

import ctypes
import os
import threading
import weakref

import numpy as np

__all__ = [
    "LIB_PATH",
    "load",
    "lib_error",
    "Context",
    "get_context",
    "DeviceKernel",
    "EXPORTED_SYMBOLS",
    "TTAGG_HOST_PTRS",
    "TTAGG_WANT_P",
    "TTAGG_WANT_Q",
]

# TTAGG_LIB: development override (A/B builds of the same sources with -D switches)
LIB_PATH = os.environ.get("TTAGG_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libttagg_b200.so")

TTAGG_OK = 0
TTAGG_ERR_ARG = 1
TTAGG_ERR_SIZE = 2
TTAGG_ERR_EMPTY = 3
TTAGG_ERR_NONFINITE = 4
TTAGG_ERR_CUDA = 5
TTAGG_ERR_UNSUPPORTED = 6
TTAGG_ERR_NOMEM = 7
TTAGG_ERR_NCCL = 8
TTAGG_HOST_PTRS = 1
TTAGG_WANT_P = 2
TTAGG_WANT_Q = 4
KIND_CP = 1
KIND_TT = 2
KIND_DENSE = 3

_c_int64_p = ctypes.POINTER(ctypes.c_int64)
_c_double_p = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p

# name -> (restype, argtypes); every symbol declared in include/ttagg_b200.h
_SIGNATURES = {
    "ttagg_version": (ctypes.c_int, []),
    "ttagg_last_error": (ctypes.c_char_p, []),
    "ttagg_geometry": (ctypes.c_int, [ctypes.c_int64, _c_int64_p]),
    "ttagg_ctx_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_vp)]),
    "ttagg_ctx_destroy": (ctypes.c_int, [_vp]),
    "ttagg_cp_upload": (
        ctypes.c_int,
        [_vp, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(_vp), _c_int64_p,
         ctypes.c_int64, ctypes.POINTER(_vp)],
    ),
    "ttagg_cp_upload_dedup": (
        ctypes.c_int,
        [_vp, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(_vp), _c_int64_p,
         ctypes.c_int64, ctypes.POINTER(_vp)],
    ),
    "ttagg_tt_upload": (
        ctypes.c_int,
        [_vp, ctypes.c_int, ctypes.c_int64, _c_int64_p, ctypes.POINTER(_vp), ctypes.POINTER(_vp)],
    ),
    "ttagg_dense_upload": (
        ctypes.c_int,
        [_vp, ctypes.c_int, ctypes.c_int64, _vp, ctypes.POINTER(_vp)],
    ),
    "ttagg_kernel_free": (ctypes.c_int, [_vp]),
    "ttagg_kernel_info": (ctypes.c_int, [_vp, _c_int64_p]),
    "ttagg_rhs": (
        ctypes.c_int,
        [_vp, ctypes.POINTER(_vp), ctypes.c_int, _vp, _vp, _vp, _vp, ctypes.c_int, _vp],
    ),
    "ttagg_rhs_perm": (
        ctypes.c_int,
        [_vp, ctypes.POINTER(_vp), ctypes.c_int, _vp, _vp, ctypes.c_double, _vp, _vp],
    ),
    "ttagg_permute": (ctypes.c_int, [_vp, ctypes.c_int64, _vp, _vp, ctypes.c_int, _vp]),
    "ttagg_stage": (
        ctypes.c_int,
        [_vp, ctypes.c_int64, _vp, _vp, ctypes.c_double, _vp, _vp, _vp],
    ),
    "ttagg_rk2": (
        ctypes.c_int,
        [_vp, ctypes.POINTER(_vp), ctypes.c_int, _vp, ctypes.c_double, ctypes.c_double,
         ctypes.c_int64, ctypes.c_int64, _vp, _c_int64_p, _c_int64_p, ctypes.c_int, _vp],
    ),
    "ttagg_profile_enable": (ctypes.c_int, [_vp, ctypes.c_int]),
    "ttagg_profile_read": (ctypes.c_int, [_vp, _c_double_p]),
    "ttagg_launch_count": (ctypes.c_int, [_vp, _c_int64_p]),
    "ttagg_debug_poison": (ctypes.c_int, [_vp, ctypes.c_int]),
    "ttagg_group_create": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.POINTER(_vp)]),
    "ttagg_group_destroy": (ctypes.c_int, [_vp]),
    "ttagg_group_size": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_int)]),
    "ttagg_group_ctx": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.POINTER(_vp)]),
    "ttagg_group_rhs": (ctypes.c_int, [_vp, ctypes.POINTER(_vp), ctypes.c_int, _vp, _vp, _vp, _vp]),
    "ttagg_group_rk2": (
        ctypes.c_int,
        [_vp, ctypes.POINTER(_vp), ctypes.c_int, _vp, ctypes.c_double, ctypes.c_double, ctypes.c_int64,
         ctypes.c_int64, _vp, _c_int64_p, _c_int64_p],
    ),
}
EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_LIB = None
_LOCK = threading.RLock()
# opt-in: CP kernels are uploaded with identical columns deduplicated
# (ttagg_cp_upload_dedup); set through paper_1905_09071_b200.dedup_identical_columns
DEDUP = False


def load():
    """Load the extension (raises if it has not been built)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    with _LOCK:
        if _LIB is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"CUDA extension {LIB_PATH} is missing; build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback)"
                )
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _LIB = lib
    return _LIB


def lib_error() -> str:
    return load().ttagg_last_error().decode("utf-8", "replace")


class TTaggError(RuntimeError):
    pass


def check(rc: int, what: str):
    if rc == TTAGG_OK:
        return
    msg = lib_error()
    # error classes mirror the reference (rhs.py / kernels.py raise KernelError / ValueError)
    from .kernels import KernelError

    if rc in (TTAGG_ERR_ARG, TTAGG_ERR_SIZE, TTAGG_ERR_EMPTY):
        raise KernelError(msg)
    if rc == TTAGG_ERR_NONFINITE:
        raise ValueError(msg)
    raise TTaggError(f"{what} failed (code {rc}): {msg}")


def geometry(n_classes: int):
    out = (ctypes.c_int64 * 3)()
    check(load().ttagg_geometry(int(n_classes), out), "ttagg_geometry")
    return int(out[0]), int(out[1]), int(out[2])


class DeviceKernel:
    """One uploaded collision kernel (device-resident, perm layout)."""

    def __init__(self, ctx: "Context", handle, kind: int, order: int, n_classes: int):
        self.ctx = ctx
        self.handle = handle
        self.kind = kind
        self.order = order
        self.n_classes = n_classes
        self._fin = weakref.finalize(self, _free_kernel, handle)

    def info(self):
        out = (ctypes.c_int64 * 8)()
        check(load().ttagg_kernel_info(self.handle, out), "ttagg_kernel_info")
        return [int(x) for x in out]


def _free_kernel(handle):
    try:
        load().ttagg_kernel_free(handle)
    except Exception:
        pass


class Context:
    """Per-device engine context (workspaces, twiddle tables, upload cache)."""

    def __init__(self, device: int = 0):
        lib = load()
        h = _vp()
        check(lib.ttagg_ctx_create(int(device), ctypes.byref(h)), "ttagg_ctx_create")
        self.handle = h
        self.device = device
        self._cache = {}  # id(kernel object) -> (weakref, DeviceKernel)
        self._lock = threading.RLock()

    @classmethod
    def _wrap(cls, handle, device: int) -> "Context":
        """A context owned by a device group (not destroyed through this object)."""
        self = cls.__new__(cls)
        self.handle = handle
        self.device = device
        self._cache = {}
        self._lock = threading.RLock()
        return self

    # -- uploads -----------------------------------------------------------
    def upload_cp(self, factors, rank_subset=None, dedup=False) -> DeviceKernel:
        lib = load()
        fs = [np.ascontiguousarray(f, dtype=np.float64) for f in factors]
        d = len(fs)
        n_classes, rank = fs[0].shape
        ptrs = (_vp * d)(*[f.ctypes.data for f in fs])
        if rank_subset is not None:
            sub = np.ascontiguousarray(rank_subset, dtype=np.int64)
            sub_p = sub.ctypes.data_as(_c_int64_p)
            n_sub = sub.size
        else:
            sub_p, n_sub = None, 0
        h = _vp()
        fn = "ttagg_cp_upload_dedup" if dedup else "ttagg_cp_upload"
        check(getattr(lib, fn)(self.handle, d, n_classes, rank, ptrs, sub_p, n_sub, ctypes.byref(h)), fn)
        return DeviceKernel(self, h, KIND_CP, d, n_classes)

    def upload_tt(self, cores) -> DeviceKernel:
        lib = load()
        cs = [np.ascontiguousarray(c, dtype=np.float64) for c in cores]
        d = len(cs)
        n_classes = cs[0].shape[1]
        ranks = np.array([1] + [c.shape[2] for c in cs], dtype=np.int64)
        ptrs = (_vp * d)(*[c.ctypes.data for c in cs])
        h = _vp()
        check(
            lib.ttagg_tt_upload(self.handle, d, n_classes, ranks.ctypes.data_as(_c_int64_p), ptrs,
                                ctypes.byref(h)),
            "ttagg_tt_upload",
        )
        return DeviceKernel(self, h, KIND_TT, d, n_classes)

    def upload_dense(self, values) -> DeviceKernel:
        lib = load()
        v = np.ascontiguousarray(values, dtype=np.float64)
        d, n_classes = v.ndim, v.shape[0]
        h = _vp()
        check(lib.ttagg_dense_upload(self.handle, d, n_classes, v.ctypes.data, ctypes.byref(h)),
              "ttagg_dense_upload")
        return DeviceKernel(self, h, KIND_DENSE, d, n_classes)

    def device_kernel(self, kernel, rank_subset=None) -> DeviceKernel:
        """Upload once per (immutable) kernel object; cached by identity (kernels.py:129-134)."""
        dedup = DEDUP and hasattr(kernel, "factors")
        key = (id(kernel), None if rank_subset is None else tuple(int(r) for r in rank_subset), dedup)
        with self._lock:
            hit = self._cache.get(key)
            if hit is not None and hit[0]() is kernel:
                return hit[1]
            if hasattr(kernel, "factors"):
                dk = self.upload_cp(kernel.factors, rank_subset, dedup=dedup)
            elif hasattr(kernel, "cores"):
                if rank_subset is not None:
                    raise NotImplementedError("rank sharding of TT kernels")
                dk = self.upload_tt(kernel.cores)
            elif hasattr(kernel, "values"):
                if rank_subset is not None:
                    raise NotImplementedError("rank sharding of dense kernels")
                dk = self.upload_dense(kernel.values)
            else:
                from .kernels import KernelError

                raise KernelError(
                    f"unsupported kernel representation {type(kernel).__name__} on the GPU path"
                )
            try:
                ref = weakref.ref(kernel, lambda _r, k=key: self._cache.pop(k, None))
            except TypeError:
                ref = lambda k=kernel: k  # noqa: E731  (object without weakref support)
            self._cache[key] = (ref, dk)
            return dk

    # -- compute -------------------------------------------------------------
    def _pinned(self, N: int, count: int):
        """Fresh host arrays in page-locked memory (torch's caching host
        allocator) so the device->host copies run at full PCIe speed."""
        try:
            import torch

            return [torch.empty(N, dtype=torch.float64, pin_memory=True).numpy() for _ in range(count)]
        except Exception:
            return [np.empty(N) for _ in range(count)]

    def rhs_host(self, dkernels, n: np.ndarray, want_p=True, want_q=True, outputs=("p", "q", "s")):
        """Host-pointer RHS: returns dict of fresh numpy arrays."""
        lib = load()
        n = np.ascontiguousarray(n, dtype=np.float64)
        N = n.size
        # outputs land in page-locked memory (DMA target, no extra host copy);
        # the state is staged by the library itself (one call, no GIL hand-offs)
        if N >= 1 << 16:
            res = dict(zip(outputs, self._pinned(N, len(outputs))))
        else:
            res = {name: np.empty(N) for name in outputs}
        arr = (_vp * len(dkernels))(*[k.handle for k in dkernels])
        flags = TTAGG_HOST_PTRS | (TTAGG_WANT_P if want_p else 0) | (TTAGG_WANT_Q if want_q else 0)
        ptr = lambda name: res[name].ctypes.data if name in res else None  # noqa: E731
        with self._lock:
            check(
                lib.ttagg_rhs(self.handle, arr, len(dkernels), n.ctypes.data, ptr("p"), ptr("q"),
                              ptr("s"), flags, None),
                "ttagg_rhs",
            )
        return res

    def rhs_device(self, dkernels, n_ptr, p_ptr, q_ptr, s_ptr, stream_ptr=None, want_p=True, want_q=True):
        lib = load()
        arr = (_vp * len(dkernels))(*[k.handle for k in dkernels])
        flags = (TTAGG_WANT_P if want_p else 0) | (TTAGG_WANT_Q if want_q else 0)
        with self._lock:
            check(
                lib.ttagg_rhs(self.handle, arr, len(dkernels), n_ptr, p_ptr, q_ptr, s_ptr, flags,
                              stream_ptr),
                "ttagg_rhs",
            )

    def rhs_perm(self, dkernels, n_perm_ptr, k_perm_ptr, alpha, s_perm_ptr, stream_ptr=None):
        lib = load()
        arr = (_vp * len(dkernels))(*[k.handle for k in dkernels])
        with self._lock:
            check(
                lib.ttagg_rhs_perm(self.handle, arr, len(dkernels), n_perm_ptr, k_perm_ptr,
                                   float(alpha), s_perm_ptr, stream_ptr),
                "ttagg_rhs_perm",
            )

    def permute(self, n_classes, in_ptr, out_ptr, direction, stream_ptr=None):
        check(load().ttagg_permute(self.handle, int(n_classes), in_ptr, out_ptr, int(direction), stream_ptr),
              "ttagg_permute")

    def stage(self, n_classes, base_ptr, s_ptr, a, out_ptr, diag_ptr, stream_ptr=None):
        with self._lock:
            check(load().ttagg_stage(self.handle, int(n_classes), base_ptr, s_ptr, float(a), out_ptr,
                                     diag_ptr, stream_ptr), "ttagg_stage")

    def rk2_host(self, dkernels, n0: np.ndarray, t0: float, dt: float, steps: int, record_every: int):
        lib = load()
        n = np.array(n0, dtype=np.float64, copy=True)
        nrows = steps // record_every + 1
        rec = np.zeros((nrows, 5))
        fail = ctypes.c_int64(0)
        neg = ctypes.c_int64(0)
        arr = (_vp * len(dkernels))(*[k.handle for k in dkernels])
        with self._lock:
            check(
                lib.ttagg_rk2(self.handle, arr, len(dkernels), n.ctypes.data, float(t0), float(dt),
                              int(steps), int(record_every), rec.ctypes.data, ctypes.byref(fail),
                              ctypes.byref(neg), TTAGG_HOST_PTRS, None),
                "ttagg_rk2",
            )
        return n, rec, int(fail.value), int(neg.value)

    def profile(self, on: bool):
        check(load().ttagg_profile_enable(self.handle, 1 if on else 0), "ttagg_profile_enable")

    def debug_poison(self, on: bool):
        """NaN-fill every scratch buffer before use (initialisation check, ttagg_debug_poison)."""
        check(load().ttagg_debug_poison(self.handle, int(bool(on))), "ttagg_debug_poison")

    def launch_count(self) -> int:
        out = ctypes.c_int64(0)
        check(load().ttagg_launch_count(self.handle, ctypes.byref(out)), "ttagg_launch_count")
        return int(out.value)

    def profile_read(self):
        """{(cls, d): (ms, launches)} since the last read; cls 0/1/2/3 = pass A/B/C/other."""
        out = (ctypes.c_double * 72)()
        check(load().ttagg_profile_read(self.handle, out), "ttagg_profile_read")
        res = {}
        for cls in range(4):
            for d in range(9):
                ms, cnt = out[(cls * 9 + d) * 2], out[(cls * 9 + d) * 2 + 1]
                if cnt:
                    res[(cls, d)] = (float(ms), int(cnt))
        return res


_CONTEXTS: dict[int, Context] = {}


def group_rank_split(d: int, R: int, n_dev: int):
    """CP rank terms of one order over a device group: LPT (parallel.py's
    lpt_rank_shards) rotated by the order, so that orders with fewer rank
    terms than devices land on different devices.  Every rank exactly once."""
    from .parallel import lpt_rank_shards

    shards = lpt_rank_shards({d: R}, n_dev)
    return [list(shards[(i + d) % n_dev].get(d, [])) for i in range(n_dev)]


class Group:
    """Several GPUs of this process as one rank-sharded engine (ttagg_group_*).

    Each kernel object is split once into per-device shards — CP rank terms
    by LPT (cost ~ d^2, rhs.py:375-381 is linear in the rank sum), TT cores by
    slices of the first internal rank (construct.tt_rank_shard), a dense
    order whole on the first device — and uploaded to that device's context;
    every RHS is the all-reduced sum of the partials."""

    def __init__(self, devices):
        lib = load()
        devs = [int(x) for x in devices]
        if not devs:
            raise ValueError("a device group needs at least one device")
        arr = (ctypes.c_int * len(devs))(*devs)
        h = _vp()
        check(lib.ttagg_group_create(arr, len(devs), ctypes.byref(h)), "ttagg_group_create")
        self.handle = h
        self.devices = devs
        self.ctxs = []
        for i, dv in enumerate(devs):
            c = _vp()
            check(lib.ttagg_group_ctx(h, i, ctypes.byref(c)), "ttagg_group_ctx")
            self.ctxs.append(Context._wrap(c, dv))
        self._cache = {}
        self._lock = threading.RLock()

    def close(self):
        """Free the shards (before their contexts go) and the group."""
        if self.handle:
            with self._lock:
                for _, shards in self._cache.values():
                    for dk in shards:
                        if dk is not None:
                            dk._fin()  # ttagg_kernel_free now, not at garbage collection
                self._cache.clear()
            for c in self.ctxs:
                c._cache.clear()
            load().ttagg_group_destroy(self.handle)
            self.handle = None

    def shards(self, kernel):
        """Per-device DeviceKernel (or None) for one kernel object, cached by identity."""
        key = (id(kernel), DEDUP and hasattr(kernel, "factors"))
        with self._lock:
            hit = self._cache.get(key)
            if hit is not None and hit[0]() is kernel:
                return hit[1]
            n = len(self.ctxs)
            out = [None] * n
            if hasattr(kernel, "factors"):
                d = len(kernel.factors)
                R = kernel.factors[0].shape[1]
                for i, sub in enumerate(group_rank_split(d, R, n)):
                    if sub:
                        out[i] = self.ctxs[i].upload_cp(kernel.factors, rank_subset=sub, dedup=key[1])
            elif hasattr(kernel, "cores"):
                from .construct import tt_rank_shard

                for i in range(n):
                    sl = tt_rank_shard(kernel.cores, n, i) if n > 1 else kernel.cores
                    if sl is not None:
                        out[i] = self.ctxs[i].upload_tt(sl)
            elif hasattr(kernel, "values"):
                out[0] = self.ctxs[0].upload_dense(kernel.values)
            else:
                from .kernels import KernelError

                raise KernelError(f"unsupported kernel representation {type(kernel).__name__} on the GPU path")
            try:
                ref = weakref.ref(kernel, lambda _r, k=key: self._cache.pop(k, None))
            except TypeError:
                ref = lambda k=kernel: k  # noqa: E731
            self._cache[key] = (ref, out)
            return out

    def _table(self, kernels):
        cols = [self.shards(k) for k in kernels]
        n = len(self.ctxs)
        flat = [cols[j][i].handle if cols[j][i] is not None else None for i in range(n) for j in range(len(cols))]
        return (_vp * len(flat))(*flat), len(cols)

    def rhs_host(self, kernels, n: np.ndarray, outputs=("p", "q", "s")):
        n = np.ascontiguousarray(n, dtype=np.float64)
        if n.size >= 1 << 16:  # page-locked outputs: direct device-to-host copies
            res = dict(zip(outputs, self.ctxs[0]._pinned(n.size, len(outputs))))
        else:
            res = {name: np.empty(n.size) for name in outputs}
        arr, nk = self._table(kernels)
        ptr = lambda name: res[name].ctypes.data if name in res else None  # noqa: E731
        with self._lock:
            check(load().ttagg_group_rhs(self.handle, arr, nk, n.ctypes.data, ptr("p"), ptr("q"), ptr("s")),
                  "ttagg_group_rhs")
        return res

    def rk2_host(self, kernels, n0: np.ndarray, t0: float, dt: float, steps: int, record_every: int):
        n = np.array(n0, dtype=np.float64, copy=True)
        rec = np.zeros((steps // record_every + 1, 5))
        fail = ctypes.c_int64(0)
        neg = ctypes.c_int64(0)
        arr, nk = self._table(kernels)
        with self._lock:
            check(load().ttagg_group_rk2(self.handle, arr, nk, n.ctypes.data, float(t0), float(dt), int(steps),
                                         int(record_every), rec.ctypes.data, ctypes.byref(fail),
                                         ctypes.byref(neg)), "ttagg_group_rk2")
        return n, rec, int(fail.value), int(neg.value)


_GROUP = None
_GROUP_ENV_READ = False


def set_group(devices) -> "Group | None":
    """Route rhs_total / integrate through a device group (None: one device)."""
    global _GROUP, _GROUP_ENV_READ
    with _LOCK:
        _GROUP_ENV_READ = True
        old, _GROUP = _GROUP, (Group(devices) if devices else None)
    if old is not None:
        old.close()
    return _GROUP


def active_group() -> "Group | None":
    """The device group in use ($TTAGG_DEVICES="0,1,..." selects one at first use)."""
    global _GROUP_ENV_READ
    if not _GROUP_ENV_READ:
        with _LOCK:
            if not _GROUP_ENV_READ:
                _GROUP_ENV_READ = True
                env = os.environ.get("TTAGG_DEVICES", "").strip()
                if env:
                    globals()["_GROUP"] = Group([int(x) for x in env.split(",") if x.strip()])
    return _GROUP


def get_context(device: int | None = None) -> Context:
    """Context of the given device (default: $TTAGG_DEVICE, else $LOCAL_RANK, else 0)."""
    if device is None:
        device = int(os.environ.get("TTAGG_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    with _LOCK:
        ctx = _CONTEXTS.get(device)
        if ctx is None:
            ctx = Context(device)
            _CONTEXTS[device] = ctx
    return ctx
