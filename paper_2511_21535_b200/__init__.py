"""paper_2511_21535_b200 -- B200-native (sm_100a) MLFMA near-field (P2P) operator with the data-redundancy layout
of arXiv 2511.21535.

This module is the thin Python binding over the C ABI of libp2p.so (include/p2p.h): argument marshalling only --
every step of the path (binning, Morton keys, radix sort, box scan, neighbour lists, restructure, evaluation,
scatter) runs in the library's CUDA kernels.  PyTorch supplies device memory, streams and process groups.  There
is NO CPU fallback: if libp2p.so is missing or no CUDA device is present the calls raise.

Functions with the C names (p2p_plan_create, p2p_restructure, p2p_eval, p2p_set_charges, p2p_destroy,
p2p_get_info, p2p_copy_out, p2p_comm_*, p2p_status_string, p2p_last_error, p2p_kernel_launch_count) take raw
pointers / ints exactly like the ABI; `Plan` and `nearfield` are conveniences over them taking torch tensors.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libp2p.so")

# ---- enums (include/p2p.h) ----
P2P_OK, P2P_ERR_INVALID_ARGUMENT, P2P_ERR_OUT_OF_DOMAIN, P2P_ERR_OUT_OF_MEMORY, P2P_ERR_CUDA, P2P_ERR_NCCL, \
    P2P_ERR_BAD_STATE, P2P_ERR_UNSUPPORTED = range(8)
P2P_GRAVITY, P2P_HELMHOLTZ2D = 0, 1
P2P_FP32, P2P_FP64 = 0, 1
P2P_REDUNDANT, P2P_INDEXED, P2P_INDEXED_BITWISE, P2P_PAIRREC = 0, 1, 2, 3
(P2P_ARR_PERM, P2P_ARR_SORTED_KEYS, P2P_ARR_BOX_KEYS, P2P_ARR_BOX_START, P2P_ARR_NBR_OFF, P2P_ARR_NBR_BOX,
 P2P_ARR_NBR_SLOT, P2P_ARR_RED_OFF, P2P_ARR_RED, P2P_ARR_PAIRREC) = range(10)

# the layouts one p2p_restructure serves (P2P_PAIRREC needs p2p_restructure_pairs)
LAYOUTS = {"redundant": P2P_REDUNDANT, "indexed": P2P_INDEXED, "indexed_bitwise": P2P_INDEXED_BITWISE}

EXPORTED = ["p2p_plan_create", "p2p_plan_update", "p2p_plan_update_host", "p2p_restructure",
            "p2p_restructure_pairs", "p2p_get_pairrec_size", "p2p_adaptive_leaves", "p2p_adaptive_neighbours", "p2p_adaptive_eval",
            "p2p_eval",
            "p2p_eval_host", "p2p_set_charges", "p2p_destroy",
            "p2p_get_info", "p2p_copy_out", "p2p_comm_unique_id", "p2p_comm_create", "p2p_comm_destroy",
            "p2p_partition_splitters", "p2p_get_splitters", "p2p_loopback_group_create", "p2p_loopback_group_destroy",
            "p2p_comm_create_loopback", "p2p_comm_create_ipc", "p2p_adaptive_enable", "p2p_adaptive_disable",
            "p2p_status_string", "p2p_last_error", "p2p_kernel_launch_count",
            "p2p_abi_version"]


class P2PConfig(C.Structure):
    _fields_ = [("dim", C.c_int32), ("kernel", C.c_int), ("precision", C.c_int), ("box_size", C.c_double),
                ("lo", C.c_double * 3), ("nbox", C.c_int32 * 3), ("periodic_mask", C.c_uint32),
                ("softening", C.c_double), ("wavenumber", C.c_double), ("points_per_box", C.c_int32),
                ("stream", C.c_void_p), ("comm", C.c_void_p)]


class P2PInfo(C.Structure):
    _fields_ = [("n_local", C.c_int64), ("n_boxes", C.c_int64), ("n_nbr", C.c_int64), ("n_red", C.c_int64),
                ("n_pairs", C.c_int64), ("n_items", C.c_int64), ("key_bits", C.c_int32),
                ("sort_passes", C.c_int32)]


class P2PError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_status_name(status)}: {msg}")
        self.status = status


_lib = None


def lib() -> C.CDLL:
    """Load libp2p.so (fails loudly when it has not been built: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                              f"g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
        L = C.CDLL(LIB_PATH)
        p, i64, u64 = C.c_void_p, C.c_int64, C.c_uint64
        sig = {
            "p2p_plan_create": (C.c_int, [C.POINTER(P2PConfig), i64, p, p, C.POINTER(C.c_void_p)]),
            "p2p_plan_update": (C.c_int, [p, i64, p, p]),
            "p2p_plan_update_host": (C.c_int, [p, i64, p, p]),
            "p2p_eval_host": (C.c_int, [p, C.c_int, p, p]),
            "p2p_restructure": (C.c_int, [p]),
            "p2p_restructure_pairs": (C.c_int, [p]),
            "p2p_adaptive_leaves": (C.c_int, [p, C.c_int32, C.c_int32, p, p, p, i64, C.POINTER(C.c_int64)]),
            "p2p_adaptive_eval": (C.c_int, [p, C.c_int32, C.c_int32, C.c_int, p, p, p, i64, C.POINTER(C.c_int64)]),
            "p2p_adaptive_neighbours": (C.c_int, [p, C.c_int32, C.c_int32, p, p, p, i64, i64, C.POINTER(C.c_int64),
                                                  C.POINTER(C.c_int64)]),
            "p2p_get_pairrec_size": (C.c_int, [p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
            "p2p_eval": (C.c_int, [p, C.c_int, p, p]),
            "p2p_set_charges": (C.c_int, [p, p]),
            "p2p_destroy": (None, [p]),
            "p2p_get_info": (C.c_int, [p, C.POINTER(P2PInfo)]),
            "p2p_copy_out": (C.c_int, [p, C.c_int, p, C.c_size_t]),
            "p2p_comm_unique_id": (C.c_int, [p]),
            "p2p_comm_create": (C.c_int, [C.c_int, C.c_int, p, C.POINTER(C.c_void_p)]),
            "p2p_comm_destroy": (None, [p]),
            "p2p_status_string": (C.c_char_p, [C.c_int]),
            "p2p_last_error": (C.c_char_p, []),
            "p2p_kernel_launch_count": (u64, []),
            "p2p_abi_version": (C.c_int, []),
            "p2p_partition_splitters": (C.c_int, [p, i64, C.c_int, C.c_int, C.c_int, p]),
            "p2p_get_splitters": (C.c_int, [p, p, C.c_int]),
            "p2p_loopback_group_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
            "p2p_loopback_group_destroy": (None, [p]),
            "p2p_comm_create_loopback": (C.c_int, [p, C.c_int, C.POINTER(C.c_void_p)]),
            "p2p_comm_create_ipc": (C.c_int, [C.c_int, C.c_int, C.c_char_p, C.POINTER(C.c_void_p)]),
            "p2p_adaptive_enable": (C.c_int, [p, C.c_int, C.c_int]),
            "p2p_adaptive_disable": (C.c_int, [p]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _status_name(s: int) -> str:
    try:
        return lib().p2p_status_string(int(s)).decode()
    except Exception:  # noqa: BLE001 -- only used to format an error message
        return f"status {s}"


def _check(s: int):
    if s != P2P_OK:
        raise P2PError(s, lib().p2p_last_error().decode())


def _host_array(a, dtype):
    """a contiguous host array of the plan's dtype (torch CPU tensor kept as is, numpy converted)"""
    import torch
    if isinstance(a, np.ndarray):
        a = torch.from_numpy(np.ascontiguousarray(a))
    if a.is_cuda:
        raise P2PError(P2P_ERR_INVALID_ARGUMENT, "host array expected (use update / eval for device tensors)")
    return a.to(dtype).contiguous()


def _host_ptr(a) -> int:
    return a.data_ptr()


# ---- ABI-shaped functions (raw pointers) ----
def p2p_plan_create(cfg: P2PConfig, n_local: int, positions: int, charges: int) -> int:
    out = C.c_void_p()
    _check(lib().p2p_plan_create(C.byref(cfg), int(n_local), C.c_void_p(positions), C.c_void_p(charges),
                                 C.byref(out)))
    return out.value


def p2p_plan_update(plan: int, n_local: int, positions: int, charges: int):
    _check(lib().p2p_plan_update(C.c_void_p(plan), int(n_local), C.c_void_p(positions), C.c_void_p(charges)))


def p2p_plan_update_host(plan: int, n_local: int, positions_host: int, charges_host: int):
    _check(lib().p2p_plan_update_host(C.c_void_p(plan), int(n_local), C.c_void_p(positions_host),
                                      C.c_void_p(charges_host)))


def p2p_eval_host(plan: int, layout: int, potential_host: int, field_host: int | None):
    _check(lib().p2p_eval_host(C.c_void_p(plan), int(layout), C.c_void_p(potential_host),
                               C.c_void_p(field_host or None)))


def p2p_restructure(plan: int):
    _check(lib().p2p_restructure(C.c_void_p(plan)))


def p2p_adaptive_leaves(plan: int, t: int, min_bits: int, capacity: int):
    """(prefix length, prefix, first sorted particle) of every adaptive leaf, Morton order"""
    cap = max(int(capacity), 1)
    ln, px, st = np.empty(cap, np.uint32), np.empty(cap, np.uint32), np.empty(cap, np.uint32)
    nl = C.c_int64()
    _check(lib().p2p_adaptive_leaves(C.c_void_p(plan), int(t), int(min_bits), ln.ctypes.data_as(C.c_void_p),
                                     px.ctypes.data_as(C.c_void_p), st.ctypes.data_as(C.c_void_p), cap,
                                     C.byref(nl)))
    n = int(nl.value)
    return ln[:n].copy(), px[:n].copy(), st[:n].copy()


def p2p_adaptive_neighbours(plan: int, t: int, min_bits: int, cap_leaves: int, cap_entries: int):
    """closed neighbour CSR of the adaptive leaves: (off[L + 1], leaf[E], image code[E])"""
    off = np.empty(max(int(cap_leaves), 1), np.uint32)
    nbr = np.empty(max(int(cap_entries), 1), np.uint32)
    code = np.empty(max(int(cap_entries), 1), np.uint8)
    nl, ne = C.c_int64(), C.c_int64()
    _check(lib().p2p_adaptive_neighbours(C.c_void_p(plan), int(t), int(min_bits), off.ctypes.data_as(C.c_void_p),
                                         nbr.ctypes.data_as(C.c_void_p), code.ctypes.data_as(C.c_void_p),
                                         off.size, nbr.size, C.byref(nl), C.byref(ne)))
    L, E = int(nl.value), int(ne.value)
    return off[:L + 1].copy(), nbr[:E].copy(), code[:E].copy()


def p2p_adaptive_eval(plan: int, t: int, min_bits: int, potential: int | None, field: int | None,
                      red_out: np.ndarray | None = None, layout: int = 0) -> int:
    """redundant runs + REDUNDANT eval (or the INDEXED baseline) over the adaptive leaves; returns the
    record count"""
    nr = C.c_int64()
    _check(lib().p2p_adaptive_eval(C.c_void_p(plan), int(t), int(min_bits), int(layout), C.c_void_p(potential or None),
                                   C.c_void_p(field or None),
                                   red_out.ctypes.data_as(C.c_void_p) if red_out is not None else None,
                                   int(red_out.shape[0]) if red_out is not None else 0, C.byref(nr)))
    return int(nr.value)


def p2p_restructure_pairs(plan: int):
    _check(lib().p2p_restructure_pairs(C.c_void_p(plan)))


def p2p_get_pairrec_size(plan: int) -> tuple:
    r, t = C.c_int64(), C.c_int64()
    _check(lib().p2p_get_pairrec_size(C.c_void_p(plan), C.byref(r), C.byref(t)))
    return int(r.value), int(t.value)


def p2p_eval(plan: int, layout: int, potential: int, field: int | None):
    _check(lib().p2p_eval(C.c_void_p(plan), int(layout), C.c_void_p(potential), C.c_void_p(field or None)))


def p2p_set_charges(plan: int, charges: int):
    _check(lib().p2p_set_charges(C.c_void_p(plan), C.c_void_p(charges)))


def p2p_destroy(plan: int):
    lib().p2p_destroy(C.c_void_p(plan))


def p2p_get_info(plan: int) -> P2PInfo:
    info = P2PInfo()
    _check(lib().p2p_get_info(C.c_void_p(plan), C.byref(info)))
    return info


def p2p_copy_out(plan: int, which: int, dst: np.ndarray):
    _check(lib().p2p_copy_out(C.c_void_p(plan), int(which), dst.ctypes.data_as(C.c_void_p), dst.nbytes))


def p2p_comm_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    _check(lib().p2p_comm_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


def p2p_comm_create(nranks: int, rank: int, uid: bytes) -> int:
    out = C.c_void_p()
    buf = (C.c_ubyte * 128).from_buffer_copy(uid)
    _check(lib().p2p_comm_create(int(nranks), int(rank), C.cast(buf, C.c_void_p), C.byref(out)))
    return out.value


def p2p_comm_destroy(comm: int):
    lib().p2p_comm_destroy(C.c_void_p(comm))


def p2p_partition_splitters(hist: np.ndarray, shift: int, key_bits: int, nranks: int) -> np.ndarray:
    h = np.ascontiguousarray(np.asarray(hist, dtype=np.uint64))
    out = np.zeros(nranks + 1, np.uint32)
    _check(lib().p2p_partition_splitters(h.ctypes.data_as(C.c_void_p), h.shape[0], int(shift), int(key_bits),
                                         int(nranks), out.ctypes.data_as(C.c_void_p)))
    return out


def p2p_get_splitters(plan: int, nranks: int) -> np.ndarray:
    out = np.zeros(nranks + 1, np.uint32)
    _check(lib().p2p_get_splitters(plan, out.ctypes.data_as(C.c_void_p), int(nranks) + 1))
    return out


def p2p_loopback_group_create(nranks: int) -> int:
    out = C.c_void_p()
    _check(lib().p2p_loopback_group_create(int(nranks), C.byref(out)))
    return out.value


def p2p_loopback_group_destroy(group: int):
    lib().p2p_loopback_group_destroy(C.c_void_p(group))


def p2p_comm_create_ipc(nranks: int, rank: int, name: str) -> int:
    """multi-process communicator over CUDA IPC peer memory (include/p2p.h); `name` = a fresh token shared by all
    ranks (rank 0 draws it, the caller broadcasts it)"""
    out = C.c_void_p()
    _check(lib().p2p_comm_create_ipc(int(nranks), int(rank), name.encode(), C.byref(out)))
    return out.value


def p2p_adaptive_enable(plan: int, t: int, min_bits: int = 9):
    _check(lib().p2p_adaptive_enable(plan, int(t), int(min_bits)))


def p2p_adaptive_disable(plan: int):
    _check(lib().p2p_adaptive_disable(plan))


def p2p_comm_create_loopback(group: int, rank: int) -> int:
    out = C.c_void_p()
    _check(lib().p2p_comm_create_loopback(C.c_void_p(group), int(rank), C.byref(out)))
    return out.value


def p2p_status_string(s: int) -> str:
    return lib().p2p_status_string(int(s)).decode()


def p2p_last_error() -> str:
    return lib().p2p_last_error().decode()


def p2p_kernel_launch_count() -> int:
    return int(lib().p2p_kernel_launch_count())


def p2p_abi_version() -> int:
    return int(lib().p2p_abi_version())


# ---- torch conveniences ----
def make_config(kernel: int, precision: int, h: float, lo, nbox, periodic: int = 0, eps: float = 0.0,
                k: float = 0.0, t: int = 0, stream=None) -> P2PConfig:
    cfg = P2PConfig()
    cfg.dim = 3 if kernel == P2P_GRAVITY else 2
    cfg.kernel = kernel
    cfg.precision = precision
    cfg.box_size = float(h)
    lo = list(lo) + [0.0] * (3 - len(lo))
    nb = list(nbox) + [1] * (3 - len(nbox))
    for d in range(3):
        cfg.lo[d] = float(lo[d])
        cfg.nbox[d] = int(nb[d])
    cfg.periodic_mask = int(periodic)
    cfg.softening = float(eps)
    cfg.wavenumber = float(k)
    cfg.points_per_box = int(t)
    cfg.stream = stream
    cfg.comm = None
    return cfg


def _stream_handle(stream) -> int | None:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _check_inputs(kernel: int, positions, charges, dtype=None, device=None):
    """the C ABI cannot see dtypes or shapes: reject mismatches here (argument checking, no arithmetic)"""
    import torch
    dim = 3 if kernel == P2P_GRAVITY else 2
    if positions.dtype not in (torch.float32, torch.float64):
        raise P2PError(P2P_ERR_INVALID_ARGUMENT, f"positions must be float32 or float64, got {positions.dtype}")
    if dtype is not None and positions.dtype != dtype:
        raise P2PError(P2P_ERR_INVALID_ARGUMENT, f"positions dtype {positions.dtype} != the plan's {dtype}")
    if charges.dtype != positions.dtype:
        raise P2PError(P2P_ERR_INVALID_ARGUMENT,
                       f"charges dtype {charges.dtype} != positions dtype {positions.dtype}")
    if positions.dim() != 2 or positions.shape[1] != dim:
        raise P2PError(P2P_ERR_INVALID_ARGUMENT, f"positions must be [N][{dim}], got {tuple(positions.shape)}")
    n = positions.shape[0]
    want = (n,) if kernel == P2P_GRAVITY else (n, 2)
    if tuple(charges.shape) != want:
        raise P2PError(P2P_ERR_INVALID_ARGUMENT, f"charges must be {list(want)}, got {tuple(charges.shape)}")
    if positions.device != charges.device or (device is not None and positions.device.type != device):
        raise P2PError(P2P_ERR_INVALID_ARGUMENT, "positions and charges must be on the same (expected) device")


class Plan:
    """RAII wrapper of a p2p_plan over torch CUDA tensors (positions [N][dim], charges [N] real or [N][2] complex)."""

    def __init__(self, kernel: int, positions, charges, h: float, lo, nbox, periodic: int = 0, eps: float = 0.0,
                 k: float = 0.0, t: int = 0, stream=None, comm: int | None = None):
        import torch
        assert positions.is_cuda and charges.is_cuda, "positions / charges must be CUDA tensors"
        _check_inputs(kernel, positions, charges)
        positions = positions.contiguous()
        charges = charges.contiguous()
        prec = P2P_FP64 if positions.dtype == torch.float64 else P2P_FP32
        self.kernel, self.precision = kernel, prec
        self.dtype = positions.dtype
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        self.cfg = make_config(kernel, prec, h, lo, nbox, periodic, eps, k, t, self.stream.cuda_stream)
        self.cfg.comm = comm
        self.n = int(positions.shape[0])
        self._handle = p2p_plan_create(self.cfg, self.n, positions.data_ptr(), charges.data_ptr())
        self._info = p2p_get_info(self._handle)

    @property
    def info(self) -> P2PInfo:
        """sizes of the current structures (synchronises once after an asynchronous update())"""
        if self._info is None:
            self._info = p2p_get_info(self.handle)
        return self._info

    @property
    def handle(self) -> int:
        if not self._handle:
            raise P2PError(P2P_ERR_BAD_STATE, "plan destroyed")
        return self._handle

    def update(self, positions, charges):
        """a PhotoNs-like time step: rebuild a1..a5 for moved particles, asynchronously (no host sync); the
        sizes in self.info refresh lazily (refresh_info() synchronises and reports input errors)."""
        _check_inputs(self.kernel, positions, charges, self.dtype, "cuda")
        positions = positions.contiguous()
        charges = charges.contiguous()
        self.n = int(positions.shape[0])
        p2p_plan_update(self.handle, self.n, positions.data_ptr(), charges.data_ptr())
        self._keep = (positions, charges)
        self._info = None

    def update_host(self, positions, charges):
        """update() from HOST arrays (numpy or CPU tensors; page-locked memory makes the copy asynchronous):
        the library copies them to the device on the plan's stream (p2p_plan_update_host).  The arrays must stay
        alive until the stream passes the copy."""
        positions = _host_array(positions, self.dtype)
        charges = _host_array(charges, self.dtype)
        _check_inputs(self.kernel, positions, charges, self.dtype, "cpu")
        self.n = int(positions.shape[0])
        p2p_plan_update_host(self.handle, self.n, _host_ptr(positions), _host_ptr(charges))
        self._keep = (positions, charges)
        self._info = None

    def eval_host(self, layout: int = P2P_REDUNDANT, potential=None, field=None, want_field: bool = True):
        """eval() into HOST arrays (p2p_eval_host: device results copied back, valid on return)"""
        import torch
        if potential is None:
            potential = torch.empty(self.n, dtype=self.dtype, pin_memory=True)
        if field is None and want_field:
            field = torch.empty((self.n, 3), dtype=self.dtype, pin_memory=True)
        p2p_eval_host(self.handle, layout, _host_ptr(potential), _host_ptr(field) if field is not None else None)
        return potential, field

    def refresh_info(self):
        self._info = p2p_get_info(self.handle)
        return self._info

    def restructure(self):
        p2p_restructure(self.handle)

    def enable_adaptive(self, t: int, min_bits: int = 9):
        """SURVEY NEXT-1 on the per-step path: run update / restructure / eval over adaptive leaves with threshold t
        (p2p_adaptive_enable; measures the current input once, then every step is asynchronous)"""
        _check(lib().p2p_adaptive_enable(self.handle, int(t), int(min_bits)))
        self.adaptive = (int(t), int(min_bits))
        self._info = None

    def disable_adaptive(self):
        _check(lib().p2p_adaptive_disable(self.handle))
        self.adaptive = None
        self._info = None

    def restructure_pairs(self):
        """the thread-level pair records of P2P_PAIRREC"""
        p2p_restructure_pairs(self.handle)

    def set_charges(self, charges):
        want = (self.n,) if self.kernel == P2P_GRAVITY else (self.n, 2)
        if charges.dtype != self.dtype or tuple(charges.shape) != want or not charges.is_cuda:
            raise P2PError(P2P_ERR_INVALID_ARGUMENT, f"charges must be a CUDA {self.dtype} tensor of shape {want}")
        p2p_set_charges(self.handle, charges.contiguous().data_ptr())

    def eval(self, layout: int = P2P_REDUNDANT, potential=None, field=None, want_field: bool = True):
        import torch
        dev = torch.device("cuda", torch.cuda.current_device())
        if self.kernel == P2P_GRAVITY:
            if potential is None:
                potential = torch.empty(self.n, dtype=self.dtype, device=dev)
            if field is None and want_field:
                field = torch.empty((self.n, 3), dtype=self.dtype, device=dev)
            p2p_eval(self.handle, layout, potential.data_ptr(), field.data_ptr() if field is not None else None)
            return potential, field
        if potential is None:
            potential = torch.empty((self.n, 2), dtype=self.dtype, device=dev)
        p2p_eval(self.handle, layout, potential.data_ptr(), None)
        return potential

    def copy_out(self, which: int) -> np.ndarray:
        i = self.refresh_info()
        f64 = self.precision == P2P_FP64
        if which == P2P_ARR_PERM or which == P2P_ARR_SORTED_KEYS:
            a = np.empty(i.n_local, np.uint32)
        elif which == P2P_ARR_BOX_KEYS:
            a = np.empty(i.n_boxes, np.uint32)
        elif which in (P2P_ARR_BOX_START, P2P_ARR_NBR_OFF):
            a = np.empty(i.n_boxes + 1, np.uint32)
        elif which == P2P_ARR_NBR_BOX:
            a = np.empty(i.n_nbr, np.uint32)
        elif which == P2P_ARR_NBR_SLOT:
            a = np.empty(i.n_nbr, np.uint8)
        elif which == P2P_ARR_RED_OFF:
            a = np.empty(i.n_boxes + 1, np.uint64)
        elif which == P2P_ARR_RED:
            if self.kernel == P2P_GRAVITY:
                a = np.empty((i.n_red, 4), np.float64 if f64 else np.float32)
            else:
                a = np.empty(i.n_red, np.complex128 if f64 else np.complex64)
        elif which == P2P_ARR_PAIRREC:
            nrec, _ = p2p_get_pairrec_size(self.handle)
            a = np.empty((nrec, 4), np.float64 if f64 else np.float32)
        else:
            raise ValueError(which)
        if i.n_local == 0:
            return a[:0] if a.ndim == 1 else a
        p2p_copy_out(self.handle, which, a)
        return a

    def close(self):
        if self._handle:
            p2p_destroy(self._handle)
            self._handle = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass


def nearfield(kernel: int, positions, charges, h: float, lo, nbox, periodic: int = 0, eps: float = 0.0,
              k: float = 0.0, t: int = 0, layout: int = P2P_REDUNDANT, comm: int | None = None):
    """One-shot public API: plan -> restructure -> eval -> destroy.  Accepts host (CPU) or device tensors; host
    inputs are copied to the device and the results back to the host (the end-to-end path bench.py times)."""
    import torch
    host = not positions.is_cuda
    dev = torch.device("cuda", torch.cuda.current_device())
    pos_d = positions.to(dev, non_blocking=True) if host else positions
    q_d = charges.to(dev, non_blocking=True) if host else charges
    with Plan(kernel, pos_d, q_d, h, lo, nbox, periodic, eps, k, t, comm=comm) as plan:
        if layout == P2P_REDUNDANT:
            plan.restructure()
        out = plan.eval(layout)
    if not host:
        return out
    if kernel == P2P_GRAVITY:
        return out[0].to("cpu", non_blocking=False), out[1].to("cpu", non_blocking=False)
    return out.to("cpu", non_blocking=False)
