"""Thin ctypes binding of libtusq.so (include/tusq.h).  Argument marshalling only: every step of
the path runs in the library (host ECM/TEM in C++, device work in its sm_100a kernels).  There is
no fallback: if the shared library is missing or fails to load, importing this module raises."""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, os.environ.get("TUSQ_LIB_NAME", "libtusq.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(nvcc, sm_100a) -- there is no CPU fallback")
_lib = C.CDLL(LIB_PATH)

OK, ERR_INVALID_ARG, ERR_UNSUPPORTED, ERR_OOM, ERR_CUDA, ERR_NCCL, ERR_CAPACITY, ERR_INTERNAL = range(8)
EXEC_NO_FUSE, EXEC_NO_RESET, EXEC_NO_SAMPLE, EXEC_NO_FOLD, EXEC_PLAN_ONLY, EXEC_PROFILE = 0x1, 0x2, 0x4, 0x8, 0x10, 0x20
EXEC_CONTINUE, EXEC_NO_BATCH, EXEC_NO_LIVE = 0x40, 0x80, 0x100
APPLY_INVERSE, APPLY_UNFUSED, APPLY_PLAN_ONLY = 0x1, 0x2, 0x4

OP_DTYPE = np.dtype([("kind", "<u4"), ("q0", "<u4"), ("q1", "<u4"), ("_pad", "<u4"), ("theta", "<f8")])


class Noise(C.Structure):
    _fields_ = [("p1", C.c_double), ("p2", C.c_double), ("p_meas", C.c_double), ("flags", C.c_uint32),
                ("_pad", C.c_uint32), ("pauli1", C.c_double * 3), ("pauli2", C.c_double * 3),
                ("pauli_meas", C.c_double * 3)]


NOISE_PAULI = 0x1


class Prune(C.Structure):
    _fields_ = [("alpha_num", C.c_uint32), ("alpha_den", C.c_uint32), ("beta", C.c_uint32), ("enabled", C.c_uint32)]


class TreeInfo(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in ["S1", "S2", "S3", "p0", "n_sig", "n_insig", "n_selected", "n_leaves",
                                          "n_sites", "n_ops", "edges", "dftt_ops", "naive_ops"]]


class Exec(C.Structure):
    _fields_ = [("precision", C.c_uint32), ("mode", C.c_uint32), ("device", C.c_int32), ("flags", C.c_uint32),
                ("d_state", C.c_void_p), ("state_bytes", C.c_uint64), ("stream", C.c_void_p),
                ("leaf_begin", C.c_uint64), ("leaf_end", C.c_uint64), ("reanchor_budget", C.c_uint64),
                ("fuse_qubits", C.c_uint32), ("_pad", C.c_uint32), ("edge_eps", C.c_double), ("comm", C.c_void_p)]


class RunStats(C.Structure):
    _fields_ = [("leaves", C.c_uint64), ("resets", C.c_uint64), ("gate_apps", C.c_uint64),
                ("launches", C.c_uint64), ("sweeps", C.c_uint64), ("draws", C.c_uint64),
                ("edge_draws", C.c_uint64), ("hbm_bytes", C.c_double), ("sample_bytes", C.c_double),
                ("host_seconds", C.c_double), ("gate_kernel_launches", C.c_uint64),
                ("gate_kernel_seconds", C.c_double), ("gate_kernel_bytes", C.c_double),
                ("fused_launches", C.c_uint64), ("exchanges", C.c_uint64),
                ("sample_kernel_seconds", C.c_double), ("device_seconds", C.c_double),
                ("reduce_seconds", C.c_double), ("h2d_bytes", C.c_double), ("d2h_bytes", C.c_double),
                ("sampled_vectors", C.c_uint64), ("dense_sweep_launches", C.c_uint64),
                ("dense_sweep_seconds", C.c_double), ("dense_sweep_bytes", C.c_double)]

    def to_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_u8p, _u32p, _u64p, _vp = C.POINTER(C.c_uint8), C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.c_void_p
_sigs = {
    "tusq_build_error_tree": [C.c_uint32, _vp, C.c_uint64, C.POINTER(Noise), C.c_uint64, C.c_uint64,
                              C.POINTER(Prune), C.POINTER(_vp)],
    "tusq_tree_get_info": [_vp, C.POINTER(TreeInfo)],
    "tusq_tree_serialize": [_vp, _vp, _u64p],
    "tusq_tree_leaf": [_vp, C.c_uint64, _u64p, _u64p, _u32p, _u32p],
    "tusq_tree_partition": [_vp, C.c_uint32, C.c_uint32, _u64p],
    "tusq_run_tree": [_vp, C.POINTER(Exec), _u64p, C.POINTER(RunStats)],
    "tusq_sample": [_vp, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64, _vp, _vp],
    "tusq_apply_ops": [_vp, C.c_uint32, C.c_uint32, _vp, C.c_uint64, C.c_uint32, _vp],
    "tusq_init_basis": [_vp, C.c_uint32, C.c_uint32, C.c_uint64, C.c_double, C.c_double, _vp],
    "tusq_comm_unique_id": [_vp],
    "tusq_comm_init": [_vp, C.c_int, C.c_int, C.c_int, C.POINTER(_vp)],
    "tusq_comm_init_local": [C.c_int, C.c_int, C.POINTER(_vp)],
    "tusq_reduce_slots": [_vp, _u64p, C.c_uint64, _vp],
    "tusq_twirl_decoherence": [C.c_double, C.c_double, C.c_double, C.POINTER(C.c_double)],
}
for _name, _args in _sigs.items():
    getattr(_lib, _name).argtypes = _args
    getattr(_lib, _name).restype = C.c_int
_lib.tusq_tree_free.argtypes = [_vp]
_lib.tusq_tree_free.restype = None
_lib.tusq_comm_free.argtypes = [_vp]
_lib.tusq_comm_free.restype = None
_lib.tusq_last_error.restype = C.c_char_p
_lib.tusq_version.restype = C.c_char_p

EXPORTED = list(_sigs) + ["tusq_tree_free", "tusq_comm_free", "tusq_last_error", "tusq_version"]
MODE_REPLICA, MODE_SHARDED = 0, 1


class TusqError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = _lib.tusq_last_error().decode(errors="replace")
        super().__init__(f"{where}: status {status}: {msg}")
        self.status = status


def _check(st: int, where: str):
    if st != OK:
        raise TusqError(st, where)


def _ptr(x) -> Optional[int]:
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if hasattr(x, "cuda_stream"):
        return x.cuda_stream
    raise TypeError(f"cannot take a device pointer of {type(x)}")


def pack_ops(ops: Sequence[Tuple[int, int, int, float]]) -> np.ndarray:
    a = np.zeros(max(len(ops), 1), dtype=OP_DTYPE)
    for i, (k, q0, q1, th) in enumerate(ops):
        a[i] = (k, q0, q1, 0, th)
    return a


def version() -> str:
    return _lib.tusq_version().decode()


class Tree:
    """Library-owned ECM + TEM tree (tusq_tree*)."""

    def __init__(self, handle: int, n: int):
        self.h = C.c_void_p(handle)
        self.n = n

    def __del__(self):
        if getattr(self, "h", None) is not None and self.h.value:
            _lib.tusq_tree_free(self.h)
            self.h = None

    def info(self) -> dict:
        o = TreeInfo()
        _check(_lib.tusq_tree_get_info(self.h, C.byref(o)), "tusq_tree_get_info")
        return {k: int(getattr(o, k)) for k, _ in TreeInfo._fields_}

    @property
    def n_leaves(self) -> int:
        return self.info()["n_leaves"]

    def serialize(self) -> bytes:
        n = C.c_uint64(0)
        _check(_lib.tusq_tree_serialize(self.h, None, C.byref(n)), "tusq_tree_serialize")
        buf = (C.c_uint8 * n.value)()
        _check(_lib.tusq_tree_serialize(self.h, buf, C.byref(n)), "tusq_tree_serialize")
        return bytes(buf)

    def leaf(self, l: int):
        cnt, off, m = C.c_uint64(), C.c_uint64(), C.c_uint32(0)
        st = _lib.tusq_tree_leaf(self.h, l, C.byref(cnt), C.byref(off), None, C.byref(m))
        if st not in (OK, ERR_CAPACITY):
            _check(st, "tusq_tree_leaf")
        buf = np.zeros(3 * max(m.value, 1), dtype=np.uint32)
        _check(_lib.tusq_tree_leaf(self.h, l, C.byref(cnt), C.byref(off), buf.ctypes.data_as(_u32p), C.byref(m)),
               "tusq_tree_leaf")
        tr = [(int(buf[3 * i]), int(buf[3 * i + 1]), int(buf[3 * i + 2])) for i in range(m.value)]
        return tr, int(cnt.value), int(off.value)

    def partition(self, nranks: int, precision: int = 128) -> np.ndarray:
        b = np.zeros(nranks + 1, dtype=np.uint64)
        _check(_lib.tusq_tree_partition(self.h, nranks, precision, b.ctypes.data_as(_u64p)), "tusq_tree_partition")
        return b


def build_error_tree(n: int, ops, p1: float, p2: float, p_meas: float, shots: int, seed: int,
                     alpha=(1, 100), beta: int = 100, prune: bool = True, pauli=None) -> Tree:
    """pauli: None (depolarizing p1/p2 + bit flip p_meas) or three (pX, pY, pZ) triples for the
    1q-gate, 2q-gate and readout sites (TUSQ_NOISE_PAULI; p1/p2/p_meas are then ignored)."""
    a = pack_ops(ops)
    h = C.c_void_p()
    nz = Noise(p1, p2, p_meas, 0, 0)
    if pauli is not None:
        nz.flags = NOISE_PAULI
        for dst, src in zip((nz.pauli1, nz.pauli2, nz.pauli_meas), pauli):
            for i in range(3):
                dst[i] = float(src[i])
    pr = Prune(alpha[0], alpha[1], beta, 1 if prune else 0)
    _check(_lib.tusq_build_error_tree(n, a.ctypes.data, len(ops), C.byref(nz), shots, seed, C.byref(pr), C.byref(h)),
           "tusq_build_error_tree")
    return Tree(h.value, n)


def run_tree(tree: Tree, precision: int = 128, d_state=None, state_bytes: int = 0, stream=None,
             leaf_begin: int = 0, leaf_end: int = 0, flags: int = 0, reanchor_budget: int = 0,
             fuse_qubits: int = 0, edge_eps: float = 0.0, device: int = -1, out_slots: Optional[np.ndarray] = None,
             comm: Optional["Comm"] = None, mode: Optional[int] = None):
    """Returns (slots u64[S1], stats dict).  d_state: device pointer (int) or tensor; None = library-allocated.
    comm: a Comm -> TUSQ_MODE_SHARDED by default (d_state then holds this process's shards); with
    mode=MODE_REPLICA an NCCL Comm of the replica ranks sums the slot arrays inside the library."""
    info = tree.info()
    if out_slots is None:
        out_slots = np.zeros(info["S1"], dtype=np.uint64)
    if not (isinstance(out_slots, np.ndarray) and out_slots.dtype == np.uint64 and out_slots.flags.c_contiguous
            and out_slots.ndim == 1 and out_slots.size >= info["S1"]):
        raise ValueError(f"out_slots must be a C-contiguous 1-d uint64 array of at least S1 = {info['S1']} entries")
    if d_state is not None and not state_bytes and hasattr(d_state, "numel"):
        state_bytes = d_state.numel() * d_state.element_size()
    if mode is None:
        mode = MODE_SHARDED if comm is not None else MODE_REPLICA
    ex = Exec(precision, mode, device, flags, _ptr(d_state),
              state_bytes, _ptr(stream), leaf_begin, leaf_end, reanchor_budget, fuse_qubits, 0, edge_eps,
              comm.h if comm is not None else None)
    stats = RunStats()
    _check(_lib.tusq_run_tree(tree.h, C.byref(ex), out_slots.ctypes.data_as(_u64p), C.byref(stats)), "tusq_run_tree")
    return out_slots, stats.to_dict()


class Comm:
    """Sharded-mode communicator (tusq_comm): Comm.local(nshards) drives all shards from this process
    on one device; Comm.nccl(uid, nranks, rank, device) is one rank of a one-process-per-GPU job."""

    def __init__(self, h: int, nranks: int):
        self.h, self.nranks = h, nranks

    @staticmethod
    def unique_id() -> bytes:
        b = (C.c_uint8 * 128)()
        _check(_lib.tusq_comm_unique_id(C.cast(b, _vp)), "tusq_comm_unique_id")
        return bytes(b)

    @classmethod
    def nccl(cls, uid: bytes, nranks: int, rank: int, device: int = -1) -> "Comm":
        b = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = _vp()
        _check(_lib.tusq_comm_init(C.cast(b, _vp), nranks, rank, device, C.byref(h)), "tusq_comm_init")
        return cls(h.value, nranks)

    @classmethod
    def local(cls, nshards: int, device: int = -1) -> "Comm":
        h = _vp()
        _check(_lib.tusq_comm_init_local(nshards, device, C.byref(h)), "tusq_comm_init_local")
        return cls(h.value, nshards)

    def free(self):
        if self.h:
            _lib.tusq_comm_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def sample(d_state, n: int, precision: int, n_draws: int, seed: int, leaf: int, d_out, stream=None):
    _check(_lib.tusq_sample(_ptr(d_state), n, precision, n_draws, seed, leaf, _ptr(d_out), _ptr(stream)), "tusq_sample")


def apply_ops(d_state, n: int, precision: int, ops, flags: int = 0, stream=None):
    a = pack_ops(ops)
    _check(_lib.tusq_apply_ops(_ptr(d_state), n, precision, a.ctypes.data, len(ops), flags, _ptr(stream)),
           "tusq_apply_ops")


def init_basis(d_state, n: int, precision: int, index: int, re: float = 1.0, im: float = 0.0, stream=None):
    _check(_lib.tusq_init_basis(_ptr(d_state), n, precision, index, re, im, _ptr(stream)), "tusq_init_basis")


def reduce_slots(comm: "Comm", slots: np.ndarray, stream=None) -> np.ndarray:
    """Sum the replica ranks' (disjoint) host slot arrays in place over an NCCL Comm (tusq_reduce_slots)."""
    if not (isinstance(slots, np.ndarray) and slots.dtype == np.uint64 and slots.flags.c_contiguous):
        raise ValueError("slots must be a C-contiguous uint64 array")
    _check(_lib.tusq_reduce_slots(comm.h, slots.ctypes.data_as(_u64p), slots.size, _ptr(stream)), "tusq_reduce_slots")
    return slots


def twirl_decoherence(t: float, T1: float, T2: float):
    """(pX, pY, pZ) of the Pauli-twirled decoherence channel (Eq. 2) -- tusq_twirl_decoherence."""
    out = (C.c_double * 3)()
    _check(_lib.tusq_twirl_decoherence(t, T1, T2, out), "tusq_twirl_decoherence")
    return tuple(out)
