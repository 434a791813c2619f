"""Python binding of libtinv.so (include/tinv.h): argument marshalling only.

Every step of the path runs in the library's sm_100a kernels; this module only turns
torch tensors / numpy arrays into pointers.  There is no CPU fallback: if the shared
library is missing or no CUDA device is usable, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtinv.so")
if os.environ.get("TINV_LIB_VARIANT"):   # performance A/B of two in-tree builds (libtinv_<variant>.so)
    LIB_PATH = os.path.join(_HERE, "libtinv_" + os.environ["TINV_LIB_VARIANT"] + ".so")

EXPORTS = ("tinv_create", "tinv_eigvecs", "tinv_eigvecs_host", "tinv_destroy", "tinv_strerror",
           "tinv_set_profiling", "tinv_get_stats", "tinv_abi_version", "tinv_partition",
           "tinv_eigvals", "tinv_eig", "tinv_set_virtual_ranks", "tinv_set_resident", "tinv_set_reorth",
           "tinv_set_lookahead", "tinv_set_host_exchange", "tinv_debug_peer_map", "tinv_plan",
           "tinv_set_deferred")

# include/tinv.h tinv_allgather_fn: int (*)(const void* send, void* recv, size_t bytes, void* ctx)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)

KERNEL_NAMES = ("prep", "batched_lu", "finalize", "cwy", "misc", "total")
PHASE_NAMES = ("first", "A", "R1", "TT", "BC", "R2", "TN", "D", "test", "solve_fwd", "solve_back", "solve_wait", "st_wait", "st_body", "st_sync", "st_blkend")


class TinvConfig(C.Structure):
    _fields_ = [("device", C.c_int), ("nranks", C.c_int), ("rank", C.c_int),
                ("nccl_id", C.c_void_p), ("stream", C.c_void_p)]


class TinvStats(C.Structure):
    _fields_ = [("n", C.c_int64), ("nclusters", C.c_int64), ("max_cluster", C.c_int64),
                ("n_clustered", C.c_int64), ("nflagged", C.c_int64), ("iters_hist", C.c_int64 * 8),
                ("launches", C.c_int64), ("group_syncs", C.c_int64), ("ngroups", C.c_int64),
                ("cwy_ctas", C.c_int64), ("resident_groups", C.c_int64), ("reorth_bytes", C.c_double), ("solve_bytes", C.c_double),
                ("kernel_ms", C.c_double * 6), ("kernel_launches", C.c_int64 * 6),
                ("cwy_phase_ms", C.c_double * 16), ("dz_parked", C.c_int64), ("dz_redo", C.c_int64),
                ("dz_ms", C.c_double)]

    def as_dict(self):
        return {
            "n": self.n, "nclusters": self.nclusters, "max_cluster": self.max_cluster,
            "n_clustered": self.n_clustered, "nflagged": self.nflagged,
            "iters_hist": list(self.iters_hist), "launches": self.launches,
            "group_syncs": self.group_syncs, "ngroups": self.ngroups, "cwy_ctas": self.cwy_ctas,
            "resident_groups": self.resident_groups,
            "reorth_bytes": self.reorth_bytes, "solve_bytes": self.solve_bytes,
            "kernel_ms": dict(zip(KERNEL_NAMES, list(self.kernel_ms))),
            "kernel_launches": dict(zip(KERNEL_NAMES, list(self.kernel_launches))),
            "cwy_phase_ms": dict(zip(PHASE_NAMES, list(self.cwy_phase_ms))),
            "dz_parked": self.dz_parked, "dz_redo": self.dz_redo, "dz_ms": self.dz_ms,
        }


class TinvError(RuntimeError):
    pass


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libtinv.so and declare the C signatures (no CUDA needed for this step)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise TinvError(f"{path} is missing: build it with __graft_entry__.build() (make -C paper_1209_1910_b200/csrc)")
    L = C.CDLL(path)
    P = C.c_void_p
    I64 = C.c_int64
    L.tinv_create.argtypes = [C.POINTER(P), C.POINTER(TinvConfig)]
    L.tinv_create.restype = C.c_int
    L.tinv_eigvecs.argtypes = [P, I64, P, P, P, P, I64, C.c_uint64]
    L.tinv_eigvecs.restype = C.c_int
    L.tinv_eigvecs_host.argtypes = [P, I64, P, P, P, P, I64, C.c_uint64]
    L.tinv_eigvecs_host.restype = C.c_int
    L.tinv_destroy.argtypes = [P]
    L.tinv_destroy.restype = C.c_int
    L.tinv_strerror.argtypes = [C.c_int]
    L.tinv_strerror.restype = C.c_char_p
    L.tinv_set_profiling.argtypes = [P, C.c_int]
    L.tinv_set_profiling.restype = C.c_int
    L.tinv_get_stats.argtypes = [P, C.POINTER(TinvStats)]
    L.tinv_get_stats.restype = C.c_int
    L.tinv_abi_version.argtypes = []
    L.tinv_set_resident.restype = C.c_int
    L.tinv_set_resident.argtypes = [P, C.c_int]
    L.tinv_set_reorth.restype = C.c_int
    L.tinv_set_reorth.argtypes = [P, C.c_int]
    L.tinv_set_lookahead.restype = C.c_int
    L.tinv_set_lookahead.argtypes = [P, C.c_int]
    L.tinv_set_deferred.restype = C.c_int
    L.tinv_set_deferred.argtypes = [P, C.c_int]
    L.tinv_set_host_exchange.restype = C.c_int
    L.tinv_set_host_exchange.argtypes = [P, ALLGATHER_FN, P]
    L.tinv_debug_peer_map.restype = C.c_int
    L.tinv_debug_peer_map.argtypes = [P, C.c_size_t, C.c_uint64, P]
    L.tinv_set_virtual_ranks.restype = C.c_int
    L.tinv_set_virtual_ranks.argtypes = [P, C.c_int]
    L.tinv_eigvals.restype = C.c_int
    L.tinv_eigvals.argtypes = [P, I64, P, P, P]
    L.tinv_eig.restype = C.c_int
    L.tinv_eig.argtypes = [P, I64, P, P, P, P, I64, C.c_uint64]
    L.tinv_partition.restype = C.c_int
    L.tinv_partition.argtypes = [I64, I64, P, C.c_int, P, P]
    L.tinv_plan.restype = C.c_int
    L.tinv_plan.argtypes = [I64, I64, P, C.c_int, P, P, P]
    L.tinv_abi_version.restype = C.c_int
    _lib = L
    return L


def strerror(code: int) -> str:
    return load_library().tinv_strerror(int(code)).decode()


class Tinv:
    """Handle on one GPU (tinv_create).  ``stream`` defaults to torch's current stream."""

    def __init__(self, device: int = 0, stream=None, nranks: int = 1, rank: int = 0, nccl_id: bytes | None = None):
        import torch

        if not torch.cuda.is_available():
            raise TinvError("no CUDA device: libtinv has no CPU fallback")
        self._torch = torch
        L = load_library()
        self.device = device
        self.nranks = nranks
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        self._idbuf = None
        cfg = TinvConfig(device, nranks, rank, None, C.c_void_p(stream.cuda_stream))
        if nccl_id is not None:
            self._idbuf = C.create_string_buffer(bytes(nccl_id), 128)
            cfg.nccl_id = C.cast(self._idbuf, C.c_void_p)
        h = C.c_void_p()
        rc = L.tinv_create(C.byref(h), C.byref(cfg))
        if rc != 0:
            raise TinvError(f"tinv_create failed: {rc} ({strerror(rc)})")
        self._h = h
        self._L = L

    def close(self):
        if getattr(self, "_h", None):
            self._L.tinv_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_profiling(self, on: bool = True):
        self._L.tinv_set_profiling(self._h, 1 if on else 0)

    def stats(self) -> dict:
        s = TinvStats()
        self._L.tinv_get_stats(self._h, C.byref(s))
        return s.as_dict()

    def eigvecs(self, d, e, w, Z=None, seed: int = 1, check: bool = True):
        """Device path: d, e, w are float64 CUDA tensors; returns (Z, info) with Z an
        (n, n) tensor whose COLUMNS are the eigenvectors (column-major storage)."""
        torch = self._torch
        n = int(d.shape[0])
        for name, t in (("d", d), ("w", w)) + ((("e", e),) if n > 1 else ()):
            if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
                raise TinvError(f"{name} must be a contiguous float64 CUDA tensor")
        if Z is None:
            Zt = torch.empty((n, n), dtype=torch.float64, device=d.device)  # Zt[j] = column j
        else:
            Zt = Z
        rc = self._L.tinv_eigvecs(self._h, n, C.c_void_p(d.data_ptr()),
                                  C.c_void_p(e.data_ptr()) if n > 1 else None,
                                  C.c_void_p(w.data_ptr()), C.c_void_p(Zt.data_ptr()), n, int(seed))
        if rc < 0 and check:
            raise TinvError(f"tinv_eigvecs failed: {rc} ({strerror(rc)})")
        return Zt.t(), rc

    def set_resident(self, enable: bool):
        rc = self._L.tinv_set_resident(self._h, int(bool(enable)))
        if rc:
            raise TinvError(f"tinv_set_resident failed: {rc}")

    def set_reorth(self, mode: str):
        """'cwy' (Alg. 4, reduced sequence §3.3.2, default), 'mgs' (Alg. 1, classical modified
        Gram-Schmidt) or 'ordinary' (Alg. 4 in the ordinary sequence of §3.3.1)."""
        code = {"cwy": 0, "mgs": 1, "ordinary": 2}[mode]
        rc = self._L.tinv_set_reorth(self._h, code)
        if rc:
            raise TinvError(f"tinv_set_reorth failed: {rc}")

    def set_lookahead(self, b: int):
        """Blocked look-ahead block size (include/tinv.h tinv_set_lookahead; 0/1 = off)."""
        rc = self._L.tinv_set_lookahead(self._h, int(b))
        if rc:
            raise TinvError(f"tinv_set_lookahead failed: {rc}")

    def set_deferred(self, enable: bool):
        """Deferred final pass D (include/tinv.h tinv_set_deferred; default on)."""
        rc = self._L.tinv_set_deferred(self._h, int(bool(enable)))
        if rc:
            raise TinvError(f"tinv_set_deferred failed: {rc}")

    def set_host_exchange(self, allgather):
        """Exchange the CUDA IPC handles through ``allgather(send: bytes, nbytes) -> bytes`` (a
        host all-gather over the ranks, e.g. torch.distributed on gloo) instead of NCCL
        (include/tinv.h tinv_set_host_exchange; diagnostics / tests)."""
        def _fn(send, recv, nbytes, _ctx):
            try:
                out = allgather(C.string_at(send, nbytes), nbytes)
                C.memmove(recv, out, len(out))
                return 0
            except Exception:
                return 1
        self._xchg = ALLGATHER_FN(_fn)   # keep the trampoline alive
        rc = self._L.tinv_set_host_exchange(self._h, self._xchg, None)
        if rc:
            raise TinvError(f"tinv_set_host_exchange failed: {rc}")

    def debug_peer_map(self, nbytes: int, tag: int):
        """tinv_debug_peer_map: map every rank's workspace over CUDA IPC and read each rank's tag
        through the mapping; returns the list of tags (collective)."""
        n = self.nranks
        out = (C.c_uint64 * n)()
        rc = self._L.tinv_debug_peer_map(self._h, int(nbytes), int(tag), out)
        if rc:
            raise TinvError(f"tinv_debug_peer_map failed: {rc} ({strerror(rc)})")
        return list(out)

    def set_virtual_ranks(self, nranks: int):
        rc = self._L.tinv_set_virtual_ranks(self._h, int(nranks))
        if rc:
            raise TinvError(f"tinv_set_virtual_ranks failed: {rc}")

    def eigvals(self, d, e, check: bool = True):
        """Device path: eigenvalues of T (Sturm bisection, tinv_eigvals); d, e float64 CUDA
        tensors; returns w (CUDA tensor, ascending)."""
        torch = self._torch
        n = int(d.shape[0])
        for name, t in (("d", d),) + ((("e", e),) if n > 1 else ()):
            if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
                raise TinvError(f"{name} must be a contiguous float64 CUDA tensor")
        w = torch.empty(n, dtype=torch.float64, device=d.device)
        rc = self._L.tinv_eigvals(self._h, n, C.c_void_p(d.data_ptr()),
                                  C.c_void_p(e.data_ptr()) if n > 1 else None, C.c_void_p(w.data_ptr()))
        if rc < 0 and check:
            raise TinvError(f"tinv_eigvals failed: {rc} ({strerror(rc)})")
        return w

    def eig(self, d, e, seed: int = 1, check: bool = True):
        """All eigenpairs from (d, e): (w, Z, info) via tinv_eig."""
        torch = self._torch
        n = int(d.shape[0])
        w = torch.empty(n, dtype=torch.float64, device=d.device)
        Zt = torch.empty((n, n), dtype=torch.float64, device=d.device)
        rc = self._L.tinv_eig(self._h, n, C.c_void_p(d.data_ptr()), C.c_void_p(e.data_ptr()) if n > 1 else None,
                              C.c_void_p(w.data_ptr()), C.c_void_p(Zt.data_ptr()), n, int(seed))
        if rc < 0 and check:
            raise TinvError(f"tinv_eig failed: {rc} ({strerror(rc)})")
        return w, Zt.t(), rc

    def eigvecs_host(self, d, e, w, Z=None, seed: int = 1, check: bool = True):
        """End-to-end path with host buffers (numpy or pinned CPU tensors)."""
        n = int(np.asarray(d).shape[0]) if not hasattr(d, "data_ptr") else int(d.shape[0])

        def ptr(a):
            if a is None:
                return None
            if hasattr(a, "data_ptr"):
                return C.c_void_p(a.data_ptr())
            return a.ctypes.data_as(C.c_void_p)

        if Z is None:
            Z = np.empty((n, n), dtype=np.float64)  # row j = column j of the column-major Z
        rc = self._L.tinv_eigvecs_host(self._h, n, ptr(d), ptr(e) if n > 1 else None, ptr(w), ptr(Z), n, int(seed))
        if rc < 0 and check:
            raise TinvError(f"tinv_eigvecs_host failed: {rc} ({strerror(rc)})")
        return Z, rc


def eigvecs(d, e, w, seed: int = 1, device: int = 0):
    """One-shot convenience wrapper (creates and destroys a handle)."""
    h = Tinv(device)
    try:
        Z, rc = h.eigvecs(d, e, w, seed=seed)
        return Z, rc, h.stats()
    finally:
        h.close()


def partition(cstart, nranks: int):
    """Column ranges [(lo, hi)] per rank computed by the library's multi-rank partitioner
    (tinv_partition: host-only, no device).  ``cstart`` is the cluster table (length
    nclus + 1, cstart[0] = 0, cstart[-1] = n)."""
    import numpy as np

    cs = np.ascontiguousarray(cstart, dtype=np.int32)
    nclus = cs.shape[0] - 1
    lo = np.zeros(nranks, dtype=np.int32)
    hi = np.zeros(nranks, dtype=np.int32)
    L = load_library()
    rc = L.tinv_partition(int(cs[-1]), nclus, cs.ctypes.data, int(nranks), lo.ctypes.data, hi.ctypes.data)
    if rc != 0:
        raise TinvError(rc, L.tinv_strerror(rc).decode())
    return list(zip(lo.tolist(), hi.tolist()))


def plan(cstart, nranks: int):
    """(ranges, split): tinv_plan -- the column ranges of tinv_partition and the index of the
    cluster whose rows every rank shares (-1: none)."""
    import numpy as np

    cs = np.ascontiguousarray(cstart, dtype=np.int32)
    nclus = cs.shape[0] - 1
    lo = np.zeros(nranks, dtype=np.int32)
    hi = np.zeros(nranks, dtype=np.int32)
    sp = C.c_int(-2)
    L = load_library()
    rc = L.tinv_plan(int(cs[-1]), nclus, cs.ctypes.data, int(nranks), lo.ctypes.data, hi.ctypes.data, C.byref(sp))
    if rc != 0:
        raise TinvError(rc, L.tinv_strerror(rc).decode())
    return list(zip(lo.tolist(), hi.tolist())), sp.value
