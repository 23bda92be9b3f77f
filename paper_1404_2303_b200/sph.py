"""Thin ctypes binding over libsph (include/sph.h): argument marshalling only.

Every step of the path runs in libsph's CUDA kernels; this module never computes
SPH quantities and has no CPU fallback: if libsph.so is missing or no CUDA device is
present, the calls raise.

Arrays may be torch tensors (CUDA or CPU; fp32 / int32, contiguous) or numpy arrays
(host); their raw pointers are handed to the C ABI, which detects host vs device
pointers itself.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os

import numpy as np

from .build import LIB

_lib = None


class SphError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{msg} (status {status})")
        self.status = status


SPH_OK, SPH_E_ARG, SPH_E_DOMAIN, SPH_E_STATE, SPH_E_NOCONV, SPH_E_CUDA, SPH_E_NCCL, SPH_E_OOM = (
    0, -1, -2, -3, -4, -5, -6, -7)
SPH_F_SYNC = 1
SPH_F_COUNT_CANDIDATES = 2
SPH_F_DIAGNOSTICS = 4
SPH_F_SYMMETRIC = 8
ABI_VERSION = 2


class Config(ctypes.Structure):
    _fields_ = [
        ("abi_version", ctypes.c_int32), ("box", ctypes.c_double * 3), ("gamma", ctypes.c_float),
        ("n_ngb", ctypes.c_float), ("n_ngb_tol", ctypes.c_float), ("max_h_iter", ctypes.c_int32),
        ("alpha", ctypes.c_float), ("balsara_eps", ctypes.c_float), ("split_count", ctypes.c_int32),
        ("split_fraction", ctypes.c_float), ("top_edge_factor", ctypes.c_float),
        ("h_margin", ctypes.c_float), ("sort_min_len", ctypes.c_int32), ("flags", ctypes.c_uint32), ("rank", ctypes.c_int32),
        ("nranks", ctypes.c_int32), ("slab_lo", ctypes.c_double), ("slab_hi", ctypes.c_double),
        ("halo_width", ctypes.c_double), ("row_cap", ctypes.c_int32), ("list_cap", ctypes.c_int32),
        ("group_container", ctypes.c_int32), ("cold_margin", ctypes.c_float),
    ]


class Stats(ctypes.Structure):
    _fields_ = [
        ("n_pairs", ctypes.c_int64), ("n_directed", ctypes.c_int64), ("n_candidates", ctypes.c_int64),
        ("n_unconverged", ctypes.c_int64), ("n_rebuilds", ctypes.c_int64), ("h_iters", ctypes.c_int32),
        ("n_levels", ctypes.c_int32), ("n_cells", ctypes.c_int64), ("n_leaves", ctypes.c_int64),
        ("n_pair_slots", ctypes.c_int64), ("ms_build", ctypes.c_double), ("ms_density", ctypes.c_double),
        ("ms_force", ctypes.c_double), ("ms_halo", ctypes.c_double), ("halo_sent", ctypes.c_int64),
        ("halo_recv", ctypes.c_int64), ("ms_kernel_density_full", ctypes.c_double),
        ("ms_kernel_force", ctypes.c_double), ("n_candidates_density_full", ctypes.c_int64),
        ("ms_kernel_walk_nb", ctypes.c_double), ("ms_kernel_hsolve", ctypes.c_double),
        ("ms_kernel_walk_union", ctypes.c_double), ("n_nb_entries", ctypes.c_int64),
        ("n_walk_launches", ctypes.c_int64), ("n_borderline", ctypes.c_int64),
        ("n_borderline_force", ctypes.c_int64), ("n_coincident", ctypes.c_int64),
        ("n_nb_sources", ctypes.c_int64), ("n_union_sources", ctypes.c_int64), ("cells_reused", ctypes.c_int32),
        ("ms_kernel_sort", ctypes.c_double), ("sort_key_bits", ctypes.c_int32), ("sort_passes", ctypes.c_int32),
        ("n_h_evals", ctypes.c_int64),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


#: every symbol include/sph.h declares (checked by tests/test_abi.py)
EXPORTS = ("sph_config_default", "sph_create", "sph_destroy", "sph_set_allocator",
           "sph_status_string", "sph_last_error", "sph_build_cells", "sph_density", "sph_force",
           "sph_kernel_launches", "sph_build_cells_halo", "sph_halo_select", "sph_export_state",
           "sph_import_halo_state", "sph_x_histogram", "sph_guess_h", "sph_comm_unique_id", "sph_comm_init",
           "sph_halo_counts", "sph_halo_exchange", "sph_allreduce", "sph_kick", "sph_drift", "sph_timestep", "sph_set_active", "sph_update_cells", "sph_kick_each", "sph_neighbour_min",
           "sph_debug_export", "sph_pair_ablation", "sph_halo_pack", "sph_timebins", "sph_timebins_wake",
           "sph_x_histogram_weighted", "sph_slab_leavers", "sph_halo_required", "sph_set_halo_width", "sph_step",
           "sph_ipc_alloc", "sph_ipc_open", "sph_ipc_event_create", "sph_ipc_event_open", "sph_ipc_event_record",
           "sph_ipc_event_wait")


def load(path: str | None = None):
    """Load libsph.so (no compute: safe without a GPU)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    path = path or os.environ.get("SPH_LIB", LIB)
    if not os.path.exists(path):
        raise FileNotFoundError(f"libsph.so not built ({path}); run `python -m paper_1404_2303_b200.build`")
    lib = ctypes.CDLL(path)
    P, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    lib.sph_config_default.argtypes = [ctypes.POINTER(Config), ctypes.c_double, ctypes.c_double, ctypes.c_double]
    lib.sph_config_default.restype = None
    lib.sph_create.argtypes = [ctypes.POINTER(Config), i32, P, ctypes.POINTER(P)]
    lib.sph_destroy.argtypes = [P]
    lib.sph_set_allocator.argtypes = [P, P, P, P]
    lib.sph_status_string.argtypes = [i32]
    lib.sph_status_string.restype = ctypes.c_char_p
    lib.sph_last_error.argtypes = [P]
    lib.sph_last_error.restype = ctypes.c_char_p
    lib.sph_build_cells.argtypes = [P, i64, P, P]
    lib.sph_density.argtypes = [P, P, P, P, P, P, P, P, P, P, ctypes.POINTER(Stats)]
    lib.sph_force.argtypes = [P, P, P, P, P, ctypes.POINTER(Stats)]
    lib.sph_kernel_launches.argtypes = [P]
    lib.sph_kernel_launches.restype = i64
    lib.sph_build_cells_halo.argtypes = [P, i64, i64, P, P]
    lib.sph_halo_select.argtypes = [P, i64, P, ctypes.c_double, ctypes.c_double, ctypes.c_double, P, P, P]
    lib.sph_export_state.argtypes = [P, i64, P, P]
    lib.sph_import_halo_state.argtypes = [P, P]
    lib.sph_x_histogram.argtypes = [P, i64, P, ctypes.c_double, ctypes.c_double, ctypes.c_int32, P]
    lib.sph_guess_h.argtypes = [P, i64, P, P]
    lib.sph_x_histogram_weighted.argtypes = [P, i64, P, P, ctypes.c_double, ctypes.c_double, ctypes.c_int32, P]
    lib.sph_slab_leavers.argtypes = [P, i64, P, ctypes.c_double, ctypes.c_double, P, P, P]
    lib.sph_halo_required.argtypes = [P, P]
    lib.sph_set_halo_width.argtypes = [P, ctypes.c_double]
    lib.sph_ipc_alloc.argtypes = [P, i64, ctypes.POINTER(ctypes.c_void_p), P]
    lib.sph_ipc_open.argtypes = [P, P, ctypes.POINTER(ctypes.c_void_p)]
    lib.sph_ipc_event_create.argtypes = [P, ctypes.POINTER(ctypes.c_int32), P]
    lib.sph_ipc_event_open.argtypes = [P, P, ctypes.POINTER(ctypes.c_int32)]
    lib.sph_ipc_event_record.argtypes = [P, ctypes.c_int32]
    lib.sph_ipc_event_wait.argtypes = [P, ctypes.c_int32]
    lib.sph_step.argtypes = [P, i64, P, P, P, P, P, P, P, P, P, ctypes.POINTER(Stats), ctypes.POINTER(Stats)]
    lib.sph_comm_unique_id.argtypes = [P]
    lib.sph_comm_init.argtypes = [P, P]
    lib.sph_halo_counts.argtypes = [P, i64, i64, P, P]
    lib.sph_halo_exchange.argtypes = [P, ctypes.c_int32, P, i64, P, i64, P, i64, P, i64]
    lib.sph_allreduce.argtypes = [P, P, i64, ctypes.c_int32, ctypes.c_int32]
    lib.sph_kick.argtypes = [P, i64, P, P, P, P, ctypes.c_float]
    lib.sph_set_active.argtypes = [P, i64, P]
    lib.sph_update_cells.argtypes = [P, P, P]
    lib.sph_kick_each.argtypes = [P, i64, P, P, P, P, P]
    lib.sph_neighbour_min.argtypes = [P, P, P]
    lib.sph_debug_export.argtypes = [P, ctypes.c_int32, P, i64, P]
    lib.sph_pair_ablation.argtypes = [P, ctypes.c_int32, P, P]
    lib.sph_halo_pack.argtypes = [P, P, P, P, P, P, i64, P, P]
    lib.sph_timebins.argtypes = [P, i64, P, P, ctypes.c_float, ctypes.c_double, ctypes.c_int32, i64, P, P,
                                 ctypes.c_int32, P]
    lib.sph_timebins_wake.argtypes = [P, i64, P, P, i64, P, P, ctypes.c_double, P]
    lib.sph_drift.argtypes = [P, i64, P, P, ctypes.c_float]
    lib.sph_timestep.argtypes = [P, i64, P, P, ctypes.c_float, P, P]
    if path == LIB or path is None:
        _lib = lib
    return lib


def default_config(box=(1.0, 1.0, 1.0), **kw) -> Config:
    cfg = Config()
    load().sph_config_default(ctypes.byref(cfg), *map(float, box))
    for k, v in kw.items():
        if k == "box":
            continue
        if not hasattr(cfg, k):
            raise KeyError(k)
        setattr(cfg, k, v)
    return cfg


def _ptr(a, dtype=np.float32):
    """Raw pointer of a torch tensor or numpy array (no copy; must be contiguous)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if a.dtype != dtype or not a.flags.c_contiguous:
            raise TypeError(f"expected a C-contiguous {np.dtype(dtype)} array")
        return a.ctypes.data
    import torch  # torch is plumbing only (device memory)
    if isinstance(a, torch.Tensor):
        want = {np.float32: torch.float32, np.int32: torch.int32, np.int64: torch.int64}[dtype]
        if a.dtype != want or not a.is_contiguous():
            raise TypeError(f"expected a contiguous {want} tensor")
        return a.data_ptr()
    raise TypeError(f"unsupported array type {type(a)}")


@dataclasses.dataclass
class DensityResult:
    h: object
    rho: object
    omega: object = None
    n_nbr: object = None
    div: object = None
    curl: object = None
    stats: dict = None


@dataclasses.dataclass
class ForceResult:
    a: object
    dudt: object
    vsig: object = None
    n_nbr_force: object = None
    stats: dict = None


class Context:
    """One libsph context (one GPU, one stream)."""

    def __init__(self, config: Config | None = None, device: int = 0, stream: int | None = None, **kw):
        self.lib = load()
        self.cfg = config if config is not None else default_config(**kw)
        if stream is None:
            # order the context after torch's work: its current stream on that device (a
            # legacy default stream has handle 0, and libsph then creates a blocking stream,
            # which is ordered after the legacy stream too)
            import torch
            if torch.cuda.is_available():
                stream = torch.cuda.current_stream(torch.device("cuda", int(device))).cuda_stream or None
        h = ctypes.c_void_p()
        st = self.lib.sph_create(ctypes.byref(self.cfg), int(device), stream, ctypes.byref(h))
        if st != SPH_OK:
            raise SphError(st, self.lib.sph_status_string(st).decode())
        self.h = h
        self.n = 0

    def _check(self, st):
        if st != SPH_OK:
            raise SphError(st, self.lib.sph_last_error(self.h).decode() or self.lib.sph_status_string(st).decode())

    def close(self):
        if getattr(self, "h", None):
            self.lib.sph_destroy(self.h)
            self.h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def kernel_launches(self) -> int:
        return int(self.lib.sph_kernel_launches(self.h))

    # -- the three calls of include/sph.h ------------------------------------------
    def build_cells(self, x, h0=None):
        n = int(x.shape[0])
        self._check(self.lib.sph_build_cells(self.h, n, _ptr(x), _ptr(h0)))
        self.n = n

    def step(self, x, v, m, u, h0=None, out=None):
        """build_cells + density + force in one call (include/sph.h sph_step: the host <-> device
        copies of host arrays overlap the work). out: dict of preallocated h, rho, a, dudt
        (host or device, like x). Returns (DensityResult, ForceResult) with those outputs."""
        n = int(x.shape[0])
        self.n = n
        out = out if out is not None else self._alloc_like(v, dict(h=(), rho=(), a=(3,), dudt=()))
        sd, sf = Stats(), Stats()
        self._check(self.lib.sph_step(self.h, n, _ptr(x), _ptr(h0), _ptr(v), _ptr(m), _ptr(u), _ptr(out["h"]),
                                      _ptr(out["rho"]), _ptr(out["a"]), _ptr(out["dudt"]), ctypes.byref(sd),
                                      ctypes.byref(sf)))
        return (DensityResult(out["h"], out["rho"], None, None, None, None, sd.as_dict()),
                ForceResult(out["a"], out["dudt"], None, None, sf.as_dict()))

    def update_cells(self, x, h0):
        """New positions and h of the same particles; keeps the cells when they moved little
        (include/sph.h sph_update_cells)."""
        self._check(self.lib.sph_update_cells(self.h, _ptr(x), _ptr(h0)))

    def build_cells_halo(self, x, n_own, h0=None):
        """x holds n_own owned particles followed by halo (source-only) particles."""
        n = int(x.shape[0])
        self._check(self.lib.sph_build_cells_halo(self.h, int(n_own), n - int(n_own), _ptr(x), _ptr(h0)))
        self.n = int(n_own)

    def halo_select(self, x, lo, hi, width):
        """Indices of the particles within `width` of the slab faces: (idx_lo, idx_hi)."""
        import torch
        n = int(x.shape[0])
        dev = x.device if isinstance(x, torch.Tensor) else torch.device("cpu")
        ilo = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        ihi = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        cnt = np.zeros(2, dtype=np.int64)
        self._check(self.lib.sph_halo_select(self.h, n, _ptr(x), float(lo), float(hi), float(width),
                                             _ptr(ilo, np.int32), _ptr(ihi, np.int32), cnt.ctypes.data))
        return ilo[: int(cnt[0])], ihi[: int(cnt[1])]

    def slab_leavers(self, x, lo, hi):
        """Indices of the particles outside [lo, hi): (x < lo, x >= hi)."""
        import torch
        n = int(x.shape[0])
        dev = x.device if isinstance(x, torch.Tensor) else torch.device("cpu")
        ilo = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        ihi = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        cnt = np.zeros(2, dtype=np.int64)
        self._check(self.lib.sph_slab_leavers(self.h, n, _ptr(x) if n else None, float(lo), float(hi),
                                              _ptr(ilo, np.int32), _ptr(ihi, np.int32), cnt.ctypes.data))
        return ilo[: int(cnt[0])], ihi[: int(cnt[1])]

    # -- CUDA IPC (peer-store halo, include/sph.h sph_ipc_*) ---------------------------
    def ipc_alloc(self, nbytes):
        """(device address, 64-byte handle) of a new buffer other processes can open."""
        p = ctypes.c_void_p()
        h = ctypes.create_string_buffer(64)
        self._check(self.lib.sph_ipc_alloc(self.h, int(nbytes), ctypes.byref(p), h))
        return int(p.value), bytes(h.raw)

    def ipc_open(self, handle: bytes):
        p = ctypes.c_void_p()
        self._check(self.lib.sph_ipc_open(self.h, ctypes.create_string_buffer(handle, 64), ctypes.byref(p)))
        return int(p.value)

    def ipc_event_create(self):
        i = ctypes.c_int32()
        h = ctypes.create_string_buffer(64)
        self._check(self.lib.sph_ipc_event_create(self.h, ctypes.byref(i), h))
        return int(i.value), bytes(h.raw)

    def ipc_event_open(self, handle: bytes):
        i = ctypes.c_int32()
        self._check(self.lib.sph_ipc_event_open(self.h, ctypes.create_string_buffer(handle, 64), ctypes.byref(i)))
        return int(i.value)

    def ipc_event_record(self, eid: int):
        self._check(self.lib.sph_ipc_event_record(self.h, int(eid)))

    def ipc_event_wait(self, eid: int):
        self._check(self.lib.sph_ipc_event_wait(self.h, int(eid)))

    def halo_required(self) -> float:
        """The largest owned h of the last density call (the halo width it needs)."""
        v = ctypes.c_double(0.0)
        self._check(self.lib.sph_halo_required(self.h, ctypes.byref(v)))
        return float(v.value)

    def set_halo_width(self, width: float):
        self._check(self.lib.sph_set_halo_width(self.h, float(width)))

    def x_histogram_weighted(self, x, w, lo, hi, nbins):
        import torch
        dev = x.device if isinstance(x, torch.Tensor) else torch.device("cpu")
        out = torch.zeros(nbins, dtype=torch.int64, device=dev)
        n = int(x.shape[0])
        self._check(self.lib.sph_x_histogram_weighted(self.h, n, _ptr(x) if n else None,
                                                      _ptr(w, np.int32) if n else None, float(lo), float(hi),
                                                      int(nbins), _ptr(out, np.int64)))
        return out

    def halo_pack(self, x, v, m, u, h0, idx, out=None):
        """[k, 9] rows {x, v, m, u, h0} of the owned particles idx (device), one libsph kernel;
        out: a preallocated [k, 9] device tensor (e.g. a peer's IPC buffer, `device_view`)."""
        import torch
        k = int(idx.shape[0])
        out = out if out is not None else torch.empty(k, 9, dtype=torch.float32, device=idx.device)
        if k:
            self._check(self.lib.sph_halo_pack(self.h, _ptr(x), _ptr(v), _ptr(m), _ptr(u), _ptr(h0), k,
                                               _ptr(idx, np.int32), _ptr(out)))
        return out

    def export_state(self, idx, out=None):
        import torch
        k = int(idx.shape[0])
        out = out if out is not None else torch.empty(k, 5, dtype=torch.float32, device=idx.device)
        if k:
            self._check(self.lib.sph_export_state(self.h, k, _ptr(idx, np.int32), _ptr(out)))
        return out

    def import_halo_state(self, state):
        self._check(self.lib.sph_import_halo_state(self.h, _ptr(state) if state.shape[0] else None))

    def guess_h(self, x):
        import torch
        out = torch.empty(int(x.shape[0]), dtype=torch.float32, device=x.device)
        self._check(self.lib.sph_guess_h(self.h, int(x.shape[0]), _ptr(x), _ptr(out)))
        return out

    def x_histogram(self, x, lo, hi, nbins):
        import torch
        dev = x.device if isinstance(x, torch.Tensor) else torch.device("cpu")
        out = torch.zeros(nbins, dtype=torch.int64, device=dev)
        n = int(x.shape[0])
        self._check(self.lib.sph_x_histogram(self.h, n, _ptr(x) if n else None, float(lo), float(hi), int(nbins),
                                             _ptr(out, np.int64)))
        return out

    # -- allocator hook (include/sph.h sph_set_allocator) ---------------------------
    def use_torch_allocator(self):
        """Route libsph's device buffers through torch's caching allocator (before the first
        build). The callbacks count allocations and releases (self.alloc_counts)."""
        import torch
        dev = torch.cuda.current_device()
        self.alloc_counts = {"alloc": 0, "free": 0, "bytes": 0}
        AF = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
        RF = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)

        def _alloc(nbytes, stream, user):
            self.alloc_counts["alloc"] += 1
            self.alloc_counts["bytes"] += int(nbytes)
            return torch.cuda.caching_allocator_alloc(int(nbytes), dev, int(stream or 0))

        def _free(ptr, stream, user):
            self.alloc_counts["free"] += 1
            torch.cuda.caching_allocator_delete(int(ptr))

        self._alloc_cbs = (AF(_alloc), RF(_free))            # kept alive with the context
        self._check(self.lib.sph_set_allocator(self.h, ctypes.cast(self._alloc_cbs[0], ctypes.c_void_p),
                                               ctypes.cast(self._alloc_cbs[1], ctypes.c_void_p), None))

    # -- NCCL transport of the slab ring (include/sph.h) ------------------------------
    @staticmethod
    def comm_unique_id() -> bytes:
        buf = (ctypes.c_uint8 * 128)()
        st = load().sph_comm_unique_id(buf)
        if st != SPH_OK:
            raise SphError(st, "sph_comm_unique_id: " + load().sph_status_string(st).decode())
        return bytes(buf)

    def comm_init(self, uid: bytes):
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        self._check(self.lib.sph_comm_init(self.h, buf))

    def halo_exchange(self, send_lo, send_hi):
        """send_lo [n_lo, w] -> lower neighbour, send_hi [n_hi, w] -> upper neighbour (device
        float32); returns (rows from the lower neighbour, rows from the upper neighbour)."""
        import torch
        w = int(send_lo.shape[1])
        m = np.zeros(2, dtype=np.int64)
        self._check(self.lib.sph_halo_counts(self.h, int(send_lo.shape[0]), int(send_hi.shape[0]), m.ctypes.data,
                                             m.ctypes.data + 8))
        r_lo = torch.empty(int(m[0]), w, dtype=torch.float32, device=send_lo.device)
        r_hi = torch.empty(int(m[1]), w, dtype=torch.float32, device=send_lo.device)
        p = lambda t: _ptr(t) if t.shape[0] else None
        self._check(self.lib.sph_halo_exchange(self.h, w, p(send_lo), int(send_lo.shape[0]), p(send_hi),
                                               int(send_hi.shape[0]), p(r_lo), int(m[0]), p(r_hi), int(m[1])))
        return r_lo, r_hi

    def allreduce_(self, t, op: str = "sum"):
        """In-place all-reduce of a device float64 / int64 tensor (op "sum" or "max")."""
        import torch
        dt = {torch.float64: 0, torch.int64: 1}[t.dtype]
        if not t.is_contiguous():
            raise TypeError("expected a contiguous tensor")
        self._check(self.lib.sph_allreduce(self.h, t.data_ptr() if t.numel() else None, int(t.numel()), dt,
                                           {"sum": 0, "max": 1}[op]))
        return t

    _EXPORT = {"perm": (0, np.uint32, 1), "groups": (1, np.int32, 4), "list_off": (2, np.int64, 1),
               "list_len": (3, np.int32, 1), "list": (4, np.uint32, 1), "nodes": (5, np.int32, 4),
               "sortoff": (6, np.int64, 1), "sorted": (7, np.dtype([("key", np.float32), ("idx", np.int32)]), 1),
               "xh": (8, np.float32, 4)}

    def export(self, what: str) -> np.ndarray:
        """A copy of one of the context's internal arrays (include/sph.h sph_debug_export)."""
        code, dt, w = self._EXPORT[what]
        cnt = ctypes.c_int64()
        self._check(self.lib.sph_debug_export(self.h, code, None, 0, ctypes.byref(cnt)))
        out = np.zeros((cnt.value, w) if w > 1 else cnt.value, dtype=dt)
        if cnt.value:
            self._check(self.lib.sph_debug_export(self.h, code, out.ctypes.data, cnt.value, ctypes.byref(cnt)))
        return out

    def pair_ablation(self, sorted: bool, rho_out=None) -> dict:
        """The paper's cell-pair density loops on a uniform grid (include/sph.h
        sph_pair_ablation): naive double loop or the presorted sweeps."""
        c = np.zeros(16, dtype=np.int64)
        self._check(self.lib.sph_pair_ablation(self.h, int(bool(sorted)), _ptr(rho_out), c.ctypes.data))
        keys = ("tests", "hits", "pairs_face", "pairs_edge", "pairs_corner", "pass_face", "pass_edge",
                "pass_corner", "inrange_face", "inrange_edge", "inrange_corner", "cells_x", "ns_loop", "ns_presort")
        return {k: int(v) for k, v in zip(keys, c)}

    def set_active(self, mask=None):
        """Targets of the next build / density / force: bool or uint8 array [n] (caller
        order), None for all (include/sph.h sph_set_active)."""
        if mask is None:
            self._check(self.lib.sph_set_active(self.h, 0, None))
            return
        import torch
        m = mask.to(torch.uint8).contiguous() if isinstance(mask, torch.Tensor) else \
            np.ascontiguousarray(mask, dtype=np.uint8)
        ptr = m.data_ptr() if isinstance(m, torch.Tensor) else m.ctypes.data
        self._check(self.lib.sph_set_active(self.h, int(m.shape[0]), ptr))

    # -- the step around the hot path (include/sph.h sph_kick / sph_drift / sph_timestep) ----
    def kick(self, v, a, dt, u=None, dudt=None):
        self._check(self.lib.sph_kick(self.h, int(v.shape[0]), _ptr(v), _ptr(u), _ptr(a), _ptr(dudt), float(dt)))

    def kick_each(self, v, a, dt, u=None, dudt=None):
        """Per-particle kick: dt is a device float32 array [n] (0 = unchanged)."""
        self._check(self.lib.sph_kick_each(self.h, int(v.shape[0]), _ptr(v), _ptr(u), _ptr(a), _ptr(dudt), _ptr(dt)))

    def neighbour_min(self, val, out):
        """out[j] = min(out[j], val[i]) over the last force call's targets i and their force
        neighbours j (device float32 arrays, caller order)."""
        self._check(self.lib.sph_neighbour_min(self.h, _ptr(val), _ptr(out)))
        return out

    def timebins(self, h, vsig, c_cfl, dt_min, n_bins, ti, active=None, ticks_in=None, cap2=False, out=None):
        """Power-of-two steps in dt_min ticks (include/sph.h sph_timebins); int64 device arrays."""
        import torch
        out = out if out is not None else torch.empty(int(h.shape[0]), dtype=torch.int64, device=h.device)
        a = active.to(torch.uint8).contiguous() if active is not None else None
        self._check(self.lib.sph_timebins(self.h, int(h.shape[0]), _ptr(h), _ptr(vsig), float(c_cfl), float(dt_min),
                                          int(n_bins), int(ti), a.data_ptr() if a is not None else None,
                                          _ptr(ticks_in, np.int64), int(bool(cap2)), _ptr(out, np.int64)))
        return out

    def timebins_wake(self, active, lim, ti_end, ti_begin, ticks, dt_min):
        """Limiter wake-up in place on `ticks`; returns the opening-kick corrections (include/sph.h)."""
        import torch
        kick = torch.empty(int(ticks.shape[0]), dtype=torch.float32, device=ticks.device)
        a = active.to(torch.uint8).contiguous() if active is not None else None
        self._check(self.lib.sph_timebins_wake(self.h, int(ticks.shape[0]), a.data_ptr() if a is not None else None,
                                               _ptr(lim), int(ti_end), _ptr(ti_begin, np.int64), _ptr(ticks, np.int64),
                                               float(dt_min), _ptr(kick)))
        return kick

    def drift(self, x, v, dt):
        self._check(self.lib.sph_drift(self.h, int(x.shape[0]), _ptr(x), _ptr(v), float(dt)))

    def timestep(self, h, vsig, c_cfl=0.25, per_particle=False):
        """Eq. 6: min_i C_CFL 2 h_i / vsig_i (and the per-particle dt if asked)."""
        import torch
        out = torch.empty_like(h) if per_particle else None
        dmin = ctypes.c_float()
        self._check(self.lib.sph_timestep(self.h, int(h.shape[0]), _ptr(h), _ptr(vsig), float(c_cfl), _ptr(out),
                                          ctypes.byref(dmin)))
        return (dmin.value, out) if per_particle else dmin.value

    def density(self, v, m, u, out=None, stats: Stats | None = None, check=True):
        """out: dict of preallocated output arrays (h, rho, omega, n_nbr, div, curl)."""
        out = out if out is not None else self._alloc_like(v, dict(h=(), rho=(), omega=(), n_nbr=("i",),
                                                                   div=(), curl=(3,)))
        st = stats if stats is not None else Stats()
        rc = self.lib.sph_density(self.h, _ptr(v), _ptr(m), _ptr(u), _ptr(out["h"]), _ptr(out["rho"]),
                                  _ptr(out.get("omega")), _ptr(out.get("n_nbr"), np.int32),
                                  _ptr(out.get("div")), _ptr(out.get("curl")), ctypes.byref(st))
        if check:
            self._check(rc)
        return DensityResult(out["h"], out["rho"], out.get("omega"), out.get("n_nbr"), out.get("div"),
                             out.get("curl"), st.as_dict())

    def force(self, like, out=None, stats: Stats | None = None):
        out = out if out is not None else self._alloc_like(like, dict(a=(3,), dudt=(), vsig=(),
                                                                      n_nbr_force=("i",)))
        st = stats if stats is not None else Stats()
        self._check(self.lib.sph_force(self.h, _ptr(out["a"]), _ptr(out["dudt"]), _ptr(out.get("vsig")),
                                       _ptr(out.get("n_nbr_force"), np.int32), ctypes.byref(st)))
        return ForceResult(out["a"], out["dudt"], out.get("vsig"), out.get("n_nbr_force"), st.as_dict())

    def _alloc_like(self, like, spec):
        n = self.n
        out = {}
        for k, sh in spec.items():
            is_int = "i" in sh
            shape = (n,) + tuple(s for s in sh if s != "i")
            if isinstance(like, np.ndarray):
                out[k] = np.zeros(shape, dtype=np.int32 if is_int else np.float32)
            else:
                import torch
                out[k] = torch.zeros(shape, dtype=torch.int32 if is_int else torch.float32, device=like.device)
        return out


class _DevArray:
    """A raw device address as a CUDA array (__cuda_array_interface__ v3), for zero-copy
    torch views of IPC buffers."""

    def __init__(self, ptr: int, shape, typestr="<f4"):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": tuple(int(s) for s in shape),
                                         "typestr": typestr, "strides": None, "version": 3}


def device_view(ptr: int, shape, device=None):
    """float32 torch tensor viewing `shape` elements at device address ptr (no copy)."""
    import torch
    return torch.as_tensor(_DevArray(ptr, shape), device=device or torch.device("cuda", torch.cuda.current_device()))
