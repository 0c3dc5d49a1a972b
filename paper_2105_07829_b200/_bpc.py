"""ctypes binding of libbpc.so (include/bpc.h): argument marshalling only.

Every step of the hot path runs in libbpc's CUDA kernels and NCCL calls; this
module only converts torch tensors / numpy arrays to pointers.  There is no
CPU fallback: if libbpc.so is missing or fails to load, import raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libbpc.so")

BPC_OK = 0
STATUS = {0: "ok", 1: "invalid argument", 2: "size mismatch", 3: "empty block", 4: "k too large",
          5: "unsupported kind", 6: "bad state", 7: "non-finite gradient", 8: "CUDA error",
          9: "NCCL error", 10: "out of memory"}
BUF_SEND, BUF_RECV, BUF_P, BUF_WORKER_ERR, BUF_SERVER_ERR, BUF_M, BUF_V = range(7)
TIMER_NAMES = ("compress", "server", "update", "push", "pull")
EXCHANGE_P2P, EXCHANGE_NCCL = 0, 1
OPT_ADAM, OPT_LANS, OPT_NAG = 0, 1, 2
EXCHANGE_NAMES = ("p2p", "nccl", "nvls")


class BpcError(RuntimeError):
    def __init__(self, status, msg=""):
        self.status = status
        super().__init__(f"bpc status {status} ({STATUS.get(status, '?')}){': ' + msg if msg else ''}")


class Compressor(C.Structure):
    _fields_ = [("kind", C.c_int32), ("k_num", C.c_uint32), ("k_den", C.c_uint32), ("bits", C.c_uint32),
                ("randk_scaled", C.c_int32), ("use_ef", C.c_int32), ("f16_values", C.c_int32)]


class Config(C.Structure):
    _fields_ = [("world_size", C.c_int32), ("rank", C.c_int32), ("device", C.c_int32),
                ("cuda_stream", C.c_void_p), ("nccl_unique_id", C.c_void_p), ("seed", C.c_uint64),
                ("num_tensors", C.c_uint32), ("tensor_numel", C.POINTER(C.c_uint64)),
                ("tensor_offset", C.POINTER(C.c_uint64)), ("chunk_elems", C.c_uint64),
                ("size_threshold_bytes", C.c_uint64), ("comp", Compressor), ("beta1", C.c_float),
                ("beta2", C.c_float), ("eps", C.c_float), ("weight_decay", C.c_float),
                ("check_finite", C.c_int32), ("exchange", C.c_int32), ("optimizer", C.c_int32),
                ("lans_alpha_l", C.c_float), ("lans_alpha_u", C.c_float), ("momentum", C.c_float),
                ("unit_mode", C.c_int32)]


class ChunkInfo(C.Structure):
    _fields_ = [("tensor", C.c_uint32), ("raw", C.c_int32), ("owner", C.c_uint32), ("k", C.c_uint32),
                ("offset", C.c_uint64), ("len", C.c_uint64), ("payload_offset", C.c_uint64),
                ("payload_bytes", C.c_uint64), ("recv_offset", C.c_uint64), ("server_err_offset", C.c_uint64)]


class PlanSummary(C.Structure):
    _fields_ = [("num_chunks", C.c_uint32), ("num_compressed", C.c_uint32), ("num_owned", C.c_uint32),
                ("cluster_ctas", C.c_uint32), ("flat_elems", C.c_uint64), ("send_bytes", C.c_uint64),
                ("recv_slot_bytes", C.c_uint64), ("server_err_elems", C.c_uint64), ("payload_total", C.c_uint64)]


EXPORTS = ["bpc_get_unique_id", "bpc_init", "bpc_plan", "bpc_connect_local", "bpc_compress", "bpc_aggregate", "bpc_exchange_push",
           "bpc_server", "bpc_exchange_pull", "bpc_step", "bpc_sync", "bpc_finalize", "bpc_get_plan",
           "bpc_get_chunk", "bpc_peer_segment", "bpc_buffer", "bpc_copy_state", "bpc_load_state",
           "bpc_get_exchange", "bpc_get_step", "bpc_set_step", "bpc_set_timing", "bpc_get_timing", "bpc_launch_count",
           "bpc_status_string", "bpc_last_error"]

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        sigs = {
            "bpc_get_unique_id": [P], "bpc_init": [C.POINTER(Config), C.POINTER(C.c_void_p)],
            "bpc_connect_local": [P, C.c_int32],
            "bpc_plan": [C.POINTER(Config), C.POINTER(PlanSummary), C.POINTER(ChunkInfo), C.c_uint32],
            "bpc_compress": [P, P], "bpc_aggregate": [P], "bpc_exchange_push": [P], "bpc_server": [P],
            "bpc_exchange_pull": [P], "bpc_step": [P, P, C.c_float], "bpc_sync": [P], "bpc_finalize": [P],
            "bpc_get_plan": [P, C.POINTER(PlanSummary)], "bpc_get_chunk": [P, C.c_uint32, C.POINTER(ChunkInfo)],
            "bpc_peer_segment": [P, C.c_int32, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)],
            "bpc_buffer": [P, C.c_int32, C.POINTER(C.c_void_p), C.POINTER(C.c_uint64)],
            "bpc_copy_state": [P, C.c_int32, P, C.c_uint64], "bpc_load_state": [P, C.c_int32, P, C.c_uint64],
            "bpc_get_exchange": [P, C.POINTER(C.c_int32)], "bpc_get_step": [P, C.POINTER(C.c_uint32)], "bpc_set_step": [P, C.c_uint32],
            "bpc_set_timing": [P, C.c_int32], "bpc_get_timing": [P, P, P], "bpc_launch_count": [P],
            "bpc_status_string": [C.c_int], "bpc_last_error": [P],
        }
        for name, args in sigs.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.bpc_launch_count.restype = C.c_uint64
        L.bpc_status_string.restype = C.c_char_p
        L.bpc_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def _check(status, ctx=None):
    if status != BPC_OK:
        msg = lib().bpc_last_error(ctx).decode() if ctx else ""
        raise BpcError(status, msg)


def unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib().bpc_get_unique_id(buf))
    return bytes(buf)


def make_config(numels, offsets, comp, *, world_size=1, rank=0, device=0, stream=0, nccl_id=None,
                seed=0, chunk_elems=1 << 18, threshold_bytes=1 << 20, beta1=0.9, beta2=0.999, eps=1e-6,
                weight_decay=0.0, check_finite=0, exchange=0, optimizer=0, lans_alpha_l=0.01,
                lans_alpha_u=10.0, momentum=0.9, unit_mode=0):
    numel = np.ascontiguousarray(numels, dtype=np.uint64)
    offset = np.ascontiguousarray(offsets, dtype=np.uint64)
    idbuf = (C.c_uint8 * 128).from_buffer_copy(nccl_id) if nccl_id is not None else None
    cfg = Config(world_size, rank, device, stream, C.cast(idbuf, C.c_void_p) if idbuf is not None else None,
                 seed, len(numel), numel.ctypes.data_as(C.POINTER(C.c_uint64)),
                 offset.ctypes.data_as(C.POINTER(C.c_uint64)), chunk_elems, threshold_bytes,
                 Compressor(comp.kind, comp.k_num, comp.k_den, comp.bits, comp.randk_scaled, comp.use_ef,
                            getattr(comp, "f16", 0)),
                 beta1, beta2, eps, weight_decay, check_finite, exchange, optimizer, lans_alpha_l,
                 lans_alpha_u, momentum, unit_mode)
    cfg._keep = (numel, offset, idbuf)   # keep the arrays alive with the struct
    return cfg


def plan(cfg: Config):
    """Host-only planning: (PlanSummary, [ChunkInfo])."""
    s = PlanSummary()
    _check(lib().bpc_plan(C.byref(cfg), C.byref(s), None, 0))
    arr = (ChunkInfo * max(1, s.num_chunks))()
    _check(lib().bpc_plan(C.byref(cfg), C.byref(s), arr, s.num_chunks))
    return s, list(arr[:s.num_chunks])


def connect_local(contexts) -> None:
    """bpc_connect_local: one process's contexts (rank r at index r) as one P2P
    exchange group with direct device pointers (see bpc.h for the issue order)."""
    arr = (C.c_void_p * len(contexts))(*[c.h.value for c in contexts])
    _check(lib().bpc_connect_local(arr, len(contexts)), contexts[0].h)


def _device_f32(t, name, numel, device):
    """Marshalling check of a caller buffer: contiguous fp32 on the context's
    device with at least the plan's flat_elems values (libbpc checks alignment)."""
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if t.dtype != torch.float32 or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous float32 tensor")
    if t.device.type != "cuda" or t.device.index != device:
        raise ValueError(f"{name} must live on cuda:{device} (got {t.device})")
    if t.numel() < numel:
        raise ValueError(f"{name} has {t.numel()} elements, the plan needs {numel}")
    return C.c_void_p(t.data_ptr())


class _CAI:
    """Wraps a device pointer for torch.as_tensor (zero copy)."""

    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3}


class Context:
    """One rank's libbpc context (bpc_ctx)."""

    def __init__(self, cfg: Config):
        self.cfg = cfg
        h = C.c_void_p()
        _check(lib().bpc_init(C.byref(cfg), C.byref(h)))
        self.h = h
        self._flat = self.summary().flat_elems

    # ---- the hot path
    def compress(self, grad):
        _check(lib().bpc_compress(self.h, _device_f32(grad, "grad", self._flat, self.cfg.device)), self.h)

    def aggregate(self):
        _check(lib().bpc_aggregate(self.h), self.h)

    def exchange_push(self):
        _check(lib().bpc_exchange_push(self.h), self.h)

    def server(self):
        _check(lib().bpc_server(self.h), self.h)

    def exchange_pull(self):
        _check(lib().bpc_exchange_pull(self.h), self.h)

    def step(self, params, lr: float):
        _check(lib().bpc_step(self.h, _device_f32(params, "params", self._flat, self.cfg.device), C.c_float(lr)),
               self.h)

    def sync(self):
        _check(lib().bpc_sync(self.h), self.h)

    def finalize(self):
        if self.h:
            _check(lib().bpc_finalize(self.h))
            self.h = None

    def __del__(self):
        try:
            self.finalize()
        except Exception:
            pass

    # ---- introspection
    def summary(self) -> PlanSummary:
        s = PlanSummary()
        _check(lib().bpc_get_plan(self.h, C.byref(s)), self.h)
        return s

    def chunk(self, c: int) -> ChunkInfo:
        ci = ChunkInfo()
        _check(lib().bpc_get_chunk(self.h, c, C.byref(ci)), self.h)
        return ci

    def chunks(self):
        return [self.chunk(c) for c in range(self.summary().num_chunks)]

    def peer_segment(self, r: int):
        o, b = C.c_uint64(), C.c_uint64()
        _check(lib().bpc_peer_segment(self.h, r, C.byref(o), C.byref(b)), self.h)
        return o.value, b.value

    def buffer(self, which: int):
        """Device buffer as a torch uint8 tensor (zero copy)."""
        import torch
        p, b = C.c_void_p(), C.c_uint64()
        _check(lib().bpc_buffer(self.h, which, C.byref(p), C.byref(b)), self.h)
        if b.value == 0:
            return torch.empty(0, dtype=torch.uint8, device="cuda")
        return torch.as_tensor(_CAI(p.value, b.value), device="cuda")

    def copy_state(self, which: int) -> np.ndarray:
        p, b = C.c_void_p(), C.c_uint64()
        _check(lib().bpc_buffer(self.h, which, C.byref(p), C.byref(b)), self.h)
        out = np.zeros(max(b.value, 1), dtype=np.uint8)
        if b.value:
            _check(lib().bpc_copy_state(self.h, which, out.ctypes.data_as(C.c_void_p), b.value), self.h)
        return out[:b.value]

    def load_state(self, which: int, data: np.ndarray):
        data = np.ascontiguousarray(data).view(np.uint8)
        _check(lib().bpc_load_state(self.h, which, data.ctypes.data_as(C.c_void_p), data.size), self.h)

    @property
    def exchange(self) -> str:
        """Exchange transport in use: "p2p" (NVLink peer stores) or "nccl"."""
        m = C.c_int32()
        _check(lib().bpc_get_exchange(self.h, C.byref(m)), self.h)
        return EXCHANGE_NAMES[m.value]

    def set_step(self, t: int):
        """Resume at optimizer step t (after load_state of e, e~, m, v)."""
        _check(lib().bpc_set_step(self.h, t), self.h)

    @property
    def t(self) -> int:
        t = C.c_uint32()
        _check(lib().bpc_get_step(self.h, C.byref(t)), self.h)
        return t.value

    def set_timing(self, enable: bool):
        _check(lib().bpc_set_timing(self.h, int(enable)), self.h)

    def timing(self):
        ms = (C.c_float * 5)()
        cnt = (C.c_uint32 * 5)()
        _check(lib().bpc_get_timing(self.h, ms, cnt), self.h)
        return {n: (ms[i], cnt[i]) for i, n in enumerate(TIMER_NAMES)}

    def launch_count(self) -> int:
        return lib().bpc_launch_count(self.h)
