"""ctypes wrapper of the plain C oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: import it from tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never from the product
package. It shares no code with paper_2105_07829_b200/.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "oracle.c")
CFLAGS = ["-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared", "-Wall"]


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "oracle.h"))):
        subprocess.check_call(["gcc", *CFLAGS, "-o", LIB_PATH, SRC, "-lm"])
    return LIB_PATH


class _Comp(C.Structure):
    _fields_ = [("kind", C.c_int32), ("k_num", C.c_uint32), ("k_den", C.c_uint32),
                ("bits", C.c_uint32), ("randk_scaled", C.c_int32), ("use_ef", C.c_int32),
                ("f16", C.c_int32)]


class _Cfg(C.Structure):
    _fields_ = [("n", C.c_uint32), ("seed", C.c_uint64), ("num_tensors", C.c_uint32),
                ("numel", C.POINTER(C.c_uint64)), ("offset", C.POINTER(C.c_uint64)),
                ("chunk_elems", C.c_uint64), ("threshold_bytes", C.c_uint64), ("comp", _Comp),
                ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("weight_decay", C.c_float), ("optimizer", C.c_int32), ("alpha_l", C.c_float),
                ("alpha_u", C.c_float), ("momentum", C.c_float)]


class _Chunk(C.Structure):
    _fields_ = [("tensor", C.c_uint32), ("offset", C.c_uint64), ("len", C.c_uint64),
                ("raw", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        L.orc_philox4x32_10.argtypes = [C.POINTER(C.c_uint32)] * 3
        L.orc_rng_word.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32]
        L.orc_rng_word.restype = C.c_uint32
        L.orc_pairwise_sum.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_pairwise_sum.restype = C.c_double
        L.orc_topk_k.argtypes = [C.POINTER(_Comp), C.c_uint64]
        L.orc_topk_k.restype = C.c_uint64
        L.orc_payload_bytes.argtypes = [C.POINTER(_Comp), C.c_int, C.c_uint64]
        L.orc_payload_bytes.restype = C.c_uint64
        L.orc_compress.argtypes = [C.POINTER(_Comp), C.c_int, C.c_void_p, C.c_uint64, C.c_uint64,
                                   C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p]
        L.orc_decompress.argtypes = [C.POINTER(_Comp), C.c_int, C.c_void_p, C.c_uint64, C.c_void_p]
        L.orc_plan.argtypes = [C.POINTER(_Cfg), C.c_void_p, C.c_int64]
        L.orc_plan.restype = C.c_int64
        L.orc_round.argtypes = [C.POINTER(_Cfg), C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_float,
                                C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_push_pull.argtypes = [C.c_uint32, C.c_uint64, C.c_void_p, C.c_void_p]
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_get_threads.restype = C.c_int
        L.orc_adam.argtypes = [C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                               C.c_uint32, C.c_float, C.c_float, C.c_float, C.c_float, C.c_float]
        L.orc_nag.argtypes = [C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_float, C.c_float, C.c_float]
        L.orc_lans_block.argtypes = [C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_uint32, C.c_float, C.c_float, C.c_float, C.c_float, C.c_float,
                                     C.c_float, C.c_float]
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)


def comp_struct(kind, k_num=1, k_den=1000, bits=7, randk_scaled=0, use_ef=1) -> _Comp:
    return _Comp(kind, k_num, k_den, bits, randk_scaled, use_ef)


def _comp_of(c) -> _Comp:
    if isinstance(c, _Comp):
        return c
    return _Comp(c.kind, c.k_num, c.k_den, c.bits, c.randk_scaled, c.use_ef, getattr(c, "f16", 0))


def philox(ctr, key) -> list[int]:
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    o = (C.c_uint32 * 4)()
    lib().orc_philox4x32_10(c, k, o)
    return list(o)


def rng_word(seed, j, chunk, t, stage, rank) -> int:
    return lib().orc_rng_word(seed, j, chunk, t, stage, rank)


def pairwise_sum(a) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return lib().orc_pairwise_sum(_ptr(a), a.size)


def topk_k(comp, L) -> int:
    c = _comp_of(comp)
    return lib().orc_topk_k(C.byref(c), L)


def payload_bytes(comp, raw, L) -> int:
    c = _comp_of(comp)
    return lib().orc_payload_bytes(C.byref(c), int(raw), L)


def compress(comp, x, *, raw=0, seed=0, chunk=0, t=1, stage=0, rank=0) -> bytes:
    c = _comp_of(comp)
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.zeros(max(1, payload_bytes(c, raw, x.size)), dtype=np.uint8)
    rc = lib().orc_compress(C.byref(c), int(raw), _ptr(x), x.size, seed, chunk, t, stage, rank, _ptr(out))
    if rc:
        raise ValueError("orc_compress failed")
    return out[:payload_bytes(c, raw, x.size)].tobytes()


def decompress(comp, payload: bytes, L: int, *, raw=0) -> np.ndarray:
    c = _comp_of(comp)
    buf = np.frombuffer(payload, dtype=np.uint8).copy()
    out = np.zeros(max(L, 1), dtype=np.float32)
    rc = lib().orc_decompress(C.byref(c), int(raw), _ptr(buf), L, _ptr(out))
    if rc:
        raise ValueError("malformed payload")
    return out[:L]


class Cfg:
    """Holds the ctypes config plus the arrays it points to."""

    def __init__(self, n, numels, offsets, comp, *, seed=0, chunk_elems=1 << 18,
                 threshold_bytes=1 << 20, beta1=0.9, beta2=0.999, eps=1e-6, weight_decay=0.0,
                 optimizer="adam", alpha_l=0.01, alpha_u=10.0, momentum=0.9):
        self.numel = np.ascontiguousarray(numels, dtype=np.uint64)
        self.offset = np.ascontiguousarray(offsets, dtype=np.uint64)
        self.s = _Cfg(n, seed, len(self.numel),
                      self.numel.ctypes.data_as(C.POINTER(C.c_uint64)),
                      self.offset.ctypes.data_as(C.POINTER(C.c_uint64)),
                      chunk_elems, threshold_bytes, _comp_of(comp), beta1, beta2, eps, weight_decay,
                      {"adam": 0, "lans": 1, "nag": 2}[optimizer], alpha_l, alpha_u, momentum)

    @classmethod
    def from_workload(cls, wcfg, n=None):
        from workloads import layout
        numels = wcfg.tensor_numels()
        offs, _ = layout(numels)
        return cls(wcfg.n if n is None else n, numels, offs, wcfg.comp, seed=wcfg.seed,
                   chunk_elems=wcfg.chunk_elems, threshold_bytes=wcfg.threshold_bytes,
                   beta1=wcfg.beta1, beta2=wcfg.beta2, eps=wcfg.eps, weight_decay=wcfg.weight_decay,
                   optimizer=getattr(wcfg, "optimizer", "adam"), alpha_l=getattr(wcfg, "alpha_l", 0.01),
                   alpha_u=getattr(wcfg, "alpha_u", 10.0), momentum=getattr(wcfg, "momentum", 0.9))

    def plan(self) -> list[tuple[int, int, int, int]]:
        n = lib().orc_plan(C.byref(self.s), None, 0)
        if n < 0:
            raise ValueError("bad plan config")
        arr = (_Chunk * max(n, 1))()
        lib().orc_plan(C.byref(self.s), arr, n)
        return [(a.tensor, a.offset, a.len, a.raw) for a in arr[:n]]

    def payload_layout(self) -> list[tuple[int, int]]:
        """(byte offset, size) of each chunk's payload in the oracle's packed
        payload stream (chunk order, no padding)."""
        out, off = [], 0
        for (_, _, L, raw) in self.plan():
            b = payload_bytes(self.s.comp, raw, L)
            out.append((off, b))
            off += b
        return out


class State:
    """Oracle-side optimizer + EF state for n workers over a flat buffer of D."""

    def __init__(self, n, D, x0):
        self.n, self.D = n, D
        self.e = np.zeros((n, D), dtype=np.float32)
        self.et = np.zeros(D, dtype=np.float32)
        self.m = np.zeros(D, dtype=np.float32)
        self.v = np.zeros(D, dtype=np.float32)
        self.x = np.array(x0, dtype=np.float32, copy=True)
        self.t = 1


def round_(cfg: Cfg, st: State, grads: np.ndarray, lr: float, want_payloads=True):
    """One Alg. 5 step. Returns (delta payload stream per worker, p stream, g~)."""
    grads = np.ascontiguousarray(grads, dtype=np.float32).reshape(st.n, st.D)
    total = sum(b for _, b in cfg.payload_layout())
    delta = np.zeros((st.n, max(total, 1)), dtype=np.uint8) if want_payloads else None
    p = np.zeros(max(total, 1), dtype=np.uint8) if want_payloads else None
    gt = np.zeros(st.D, dtype=np.float32)
    rc = lib().orc_round(C.byref(cfg.s), st.D, _ptr(grads), _ptr(st.e), _ptr(st.et), _ptr(st.m),
                         _ptr(st.v), _ptr(st.x), st.t, lr,
                         _ptr(delta) if want_payloads else None,
                         _ptr(p) if want_payloads else None, _ptr(gt))
    if rc:
        raise RuntimeError("orc_round failed")
    st.t += 1
    return delta, p, gt


def set_threads(n: int) -> None:
    """Host threads of round_ (OpenMP over units; results identical for any n)."""
    lib().orc_set_threads(int(n))


def get_threads() -> int:
    return lib().orc_get_threads()


def push_pull(grads: np.ndarray) -> np.ndarray:
    grads = np.ascontiguousarray(grads, dtype=np.float32)
    n, D = grads.shape
    out = np.zeros(D, dtype=np.float32)
    lib().orc_push_pull(n, D, _ptr(grads), _ptr(out))
    return out


def lans_block(gt, m, v, x, t, lr, beta1, beta2, eps, wd, alpha_l=0.01, alpha_u=10.0):
    """One LANS / CLAN block update in place (Alg. 5 lines 12-18, R22)."""
    for a in (m, v, x):
        assert a.dtype == np.float32 and a.flags["C_CONTIGUOUS"]
    gt = np.ascontiguousarray(gt, dtype=np.float32)
    lib().orc_lans_block(gt.size, _ptr(gt), _ptr(m), _ptr(v), _ptr(x), t, lr, beta1, beta2, eps, wd,
                         alpha_l, alpha_u)


def nag(gt, vel, x, lr, mu, wd):
    """One NAG step in place (R24); vel is the velocity."""
    for a in (vel, x):
        assert a.dtype == np.float32 and a.flags["C_CONTIGUOUS"]
    gt = np.ascontiguousarray(gt, dtype=np.float32)
    lib().orc_nag(gt.size, _ptr(gt), _ptr(vel), _ptr(x), lr, mu, wd)


def adam(gt, m, v, x, t, lr, beta1, beta2, eps, wd):
    for a in (m, v, x):
        assert a.dtype == np.float32 and a.flags["C_CONTIGUOUS"]
    gt = np.ascontiguousarray(gt, dtype=np.float32)
    lib().orc_adam(gt.size, _ptr(gt), _ptr(m), _ptr(v), _ptr(x), t, lr, beta1, beta2, eps, wd)
