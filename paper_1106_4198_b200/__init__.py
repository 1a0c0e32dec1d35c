"""B200-native online / batch Itakura-Saito NMF engine (sm_100a).

The product is the C-ABI shared library ``lib/libisnmf_b200.so`` declared in
``include/isnmf_b200.h`` and the header-only C++ API in ``include/isnmf/``
(same names as the reference's proj/include/isnmf).  This module is a thin
ctypes face of that C ABI for the tests and bench.py.  There is no CPU
fallback: if the library cannot be loaded or no CUDA device is usable, every
compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# ISNMF_LIB selects another build of the same library (the debug build, make debug)
LIB_PATH = os.environ.get("ISNMF_LIB") or os.path.join(_HERE, "lib", "libisnmf_b200.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "isnmf_b200.h")

ERRORS = {
    1: "ShapeMismatch", 2: "EmptyDataset", 3: "NegativeInput", 4: "NonPositiveInit", 5: "ZeroColumn",
    6: "InconsistentStats", 7: "NumericalFailure", 8: "DivergedObjective", 9: "NonFiniteEntry",
    10: "NegativeEntry", 11: "IoError", 12: "UnsupportedFormat", 13: "TooShort", 14: "AllSilent",
    20: "CudaError", 21: "InvalidArgument", 22: "Unsupported",
}
RESTART = {"warm": 0, "fresh": 1}


class EngineError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERRORS.get(code, str(code))


class OnlineConfig(C.Structure):
    _fields_ = [("F", C.c_int64), ("K", C.c_int64), ("beta", C.c_int32), ("inner_iters", C.c_int32),
                ("epsilon", C.c_double), ("restart", C.c_int32), ("flags", C.c_int32), ("seed", C.c_uint64),
                ("n_store", C.c_int64), ("max_chunk", C.c_int64)]


_lib = None

D, I32, I64, U64, VP = C.c_double, C.c_int32, C.c_int64, C.c_uint64, C.c_void_p
_SIGS = {
    "isnmf_last_error": ([], C.c_char_p),
    "isnmf_device_info": ([C.c_char_p, I64], C.c_int),
    "isnmf_is_divergence": ([VP, I64, VP, I64, D, VP], C.c_int),
    "isnmf_objective": ([VP, VP, VP, I64, I64, I64, D, VP], C.c_int),
    "isnmf_solve_h": ([VP, VP, VP, I64, I64, I64, C.c_int, D, VP], C.c_int),
    "isnmf_batch_stats": ([VP, VP, VP, I64, I64, I64, D, VP, VP], C.c_int),
    "isnmf_update_w": ([VP, VP, VP, I64, I64, VP], C.c_int),
    "isnmf_rescale_dictionary": ([VP, VP, VP, I64, I64, VP, I64], C.c_int),
    "isnmf_online_create": ([VP, VP], C.c_int),
    "isnmf_online_destroy": ([VP], C.c_int),
    "isnmf_online_set_dictionary": ([VP, VP, VP, VP], C.c_int),
    "isnmf_online_get_dictionary": ([VP, VP, VP, VP], C.c_int),
    "isnmf_online_set_pending": ([VP, VP, VP, D, U64], C.c_int),
    "isnmf_online_get_pending": ([VP, VP, VP, VP, VP], C.c_int),
    "isnmf_online_set_counters": ([VP, U64, U64, D], C.c_int),
    "isnmf_online_get_counters": ([VP, VP, VP, VP, VP, VP], C.c_int),
    "isnmf_online_set_warm_h": ([VP, VP], C.c_int),
    "isnmf_online_fill_warm_h": ([VP, D], C.c_int),
    "isnmf_online_get_warm_h": ([VP, VP], C.c_int),
    "isnmf_online_run": ([VP, VP, I64, I64, VP, U64, D, VP], C.c_int),
    "isnmf_online_enqueue": ([VP, VP, I64, I64, VP, U64, D], C.c_int),
    "isnmf_online_synchronize": ([VP], C.c_int),
    "isnmf_online_get_trace": ([VP, VP, VP, VP, I64, VP], C.c_int),
    "isnmf_online_clear_trace": ([VP], C.c_int),
    "isnmf_online_get_last_h": ([VP, VP, I64], C.c_int),
    "isnmf_online_launch_count": ([VP], I64),
    "isnmf_online_solver": ([VP, C.c_char_p, I64], C.c_int),
    "isnmf_online_commit": ([VP], C.c_int),
    "isnmf_host_alloc": ([I64], VP),
    "isnmf_host_free": ([VP], None),
    "isnmf_online_profile_begin": ([VP, C.c_int32], C.c_int),
    "isnmf_online_profile_end": ([VP, VP, VP, VP, VP, VP], C.c_int),
    "isnmf_batch_train": ([VP, I64, I64, I64, I64, VP, VP, U64, D, D, VP, VP, VP, VP, VP, VP], C.c_int),
    "isnmf_batch_profile": ([I32, VP, VP], C.c_int),
    "isnmf_evaluate_heldout": ([VP, I64, I64, I64, VP, I64, D, C.c_int32, U64, VP], C.c_int),
    "isnmf_stft_power": ([VP, I64, C.c_int32, C.c_int32, VP, I64, VP], C.c_int),
    "isnmf_discard_silence": ([VP, I64, I64, D, VP, VP], C.c_int),
}


def header_symbols():
    """Every function name declared in include/isnmf_b200.h."""
    import re
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int|int64_t|void\*|void)\s+(isnmf_\w+)\(", txt, re.M)))


def lib():
    """Loads the engine library; raises if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"isnmf-b200 engine library not built: {LIB_PATH} (run `make` or build())")
        L = C.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise EngineError(rc, lib().isnmf_last_error().decode())


def _p(a):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):  # torch tensor (device memory for the bench)
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)


def _f(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def device_info():
    buf = C.create_string_buffer(4096)
    _check(lib().isnmf_device_info(buf, 4096))
    import json
    return json.loads(buf.value.decode())


# ---- stateless kernels (kernels.hpp) --------------------------------------------
def is_divergence(y, x, eps):
    y, x = np.ascontiguousarray(y, np.float64), np.ascontiguousarray(x, np.float64)
    out = D()
    _check(lib().isnmf_is_divergence(_p(y), y.size, _p(x), x.size, eps, C.byref(out)))
    return out.value


def objective(v, w, h, eps):
    v, w, h = _f(v), _f(w), _f(h)
    out = D()
    _check(lib().isnmf_objective(_p(v), _p(w), _p(h), w.shape[0], w.shape[1], v.shape[1], eps, C.byref(out)))
    return out.value


def solve_h(v, w, h0, iters, eps):
    one = np.ndim(v) == 1
    v = _f(np.asarray(v).reshape(-1, 1) if one else v)
    h0 = _f(np.asarray(h0).reshape(-1, 1) if one else h0)
    w = _f(w)
    out = np.empty(h0.shape, order="F")
    _check(lib().isnmf_solve_h(_p(v), _p(w), _p(h0), w.shape[0], w.shape[1], v.shape[1], iters, eps, _p(out)))
    return out[:, 0] if one else out


def batch_stats(v, w, h, eps):
    v, w, h = _f(v), _f(w), _f(h)
    a = np.empty(w.shape, order="F")
    b = np.empty(w.shape, order="F")
    _check(lib().isnmf_batch_stats(_p(v), _p(w), _p(h), w.shape[0], w.shape[1], v.shape[1], eps, _p(a), _p(b)))
    return a, b


def update_w(a, b, w_prev):
    a, b, w_prev = _f(a), _f(b), _f(w_prev)
    out = np.empty(a.shape, order="F")
    _check(lib().isnmf_update_w(_p(a), _p(b), _p(w_prev), a.shape[0], a.shape[1], _p(out)))
    return out


def rescale_dictionary(w, a, b, warm_h=None):
    w, a, b = _f(w).copy(order="F"), _f(a).copy(order="F"), _f(b).copy(order="F")
    h = _f(warm_h).copy(order="F") if warm_h is not None else None
    _check(lib().isnmf_rescale_dictionary(_p(w), _p(a), _p(b), w.shape[0], w.shape[1], _p(h),
                                          h.shape[1] if h is not None else 0))
    return w, a, b, h


# ---- online engine ----------------------------------------------------------------
class Online:
    """Device-resident OnlineState (online.hpp:224-248) behind the C ABI."""

    def __init__(self, F, K, beta, inner_iters, epsilon=1e-12, restart="warm", seed=1, n_store=0, max_chunk=0,
                 generic=False, pair=None):
        # pair: None = the engine's choice, False = never K1C (2-SM tcgen05 solve), True = K1C at any size
        flags = (1 if generic else 0) | {None: 0, False: 2, True: 4}[pair]
        cfg = OnlineConfig(F=F, K=K, beta=beta, inner_iters=inner_iters, epsilon=epsilon, restart=RESTART[restart],
                           seed=seed, n_store=n_store, max_chunk=max_chunk, flags=flags)
        h = C.c_void_p()
        _check(lib().isnmf_online_create(C.byref(h), C.byref(cfg)))
        self._h = h
        self.F, self.K, self.beta, self.n_store = F, K, beta, n_store

    def close(self):
        if getattr(self, "_h", None) is not None and _lib is not None:
            _lib.isnmf_online_destroy(self._h)
            self._h = None

    __del__ = close

    def set_dictionary(self, w=None, a=None, b=None):
        w, a, b = (None if x is None else _f(x) for x in (w, a, b))
        _check(lib().isnmf_online_set_dictionary(self._h, _p(w), _p(a), _p(b)))

    def set_pending(self, pa=None, pb=None, pending_div=0.0, pending_count=0):
        pa, pb = (None if x is None else _f(x) for x in (pa, pb))
        _check(lib().isnmf_online_set_pending(self._h, _p(pa), _p(pb), pending_div, pending_count))

    def set_counters(self, t=0, commits=0, rho=1.0):
        _check(lib().isnmf_online_set_counters(self._h, t, commits, rho))

    def set_warm_h(self, warm_h):
        warm_h = _f(warm_h)
        _check(lib().isnmf_online_set_warm_h(self._h, _p(warm_h)))

    def fill_warm_h(self, value):
        _check(lib().isnmf_online_fill_warm_h(self._h, value))

    def state(self, warm_h=False):
        F, K = self.F, self.K
        out = {n: np.empty((F, K), order="F") for n in ("w", "a", "b", "pending_a", "pending_b")}
        _check(lib().isnmf_online_get_dictionary(self._h, _p(out["w"]), _p(out["a"]), _p(out["b"])))
        pdiv, pcnt = D(), U64()
        _check(lib().isnmf_online_get_pending(self._h, _p(out["pending_a"]), _p(out["pending_b"]), C.byref(pdiv),
                                              C.byref(pcnt)))
        t, c, rho, ld, lo = U64(), U64(), D(), D(), D()
        _check(lib().isnmf_online_get_counters(self._h, C.byref(t), C.byref(c), C.byref(rho), C.byref(ld),
                                               C.byref(lo)))
        out.update(t=t.value, commits=c.value, rho=rho.value, last_delta=ld.value, last_minibatch_obj=lo.value,
                   pending_div=pdiv.value, pending_count=pcnt.value)
        if warm_h:
            wh = np.empty((K, self.n_store), order="F")
            _check(lib().isnmf_online_get_warm_h(self._h, _p(wh)))
            out["warm_h"] = wh
        return out

    def run(self, frames, n=None, ldv=None, index=None, budget=(1 << 64) - 1, eta=0.0):
        """frames: numpy (F x n, fp32, column-major) or a torch tensor (n x ldv, fp32, device or pinned)."""
        if hasattr(frames, "data_ptr"):
            n = frames.shape[0] if n is None else n
            ldv = frames.stride(0) if ldv is None else ldv
        else:
            frames = np.asfortranarray(frames, dtype=np.float32)
            n = frames.shape[1] if n is None else n
            ldv = frames.shape[0] if ldv is None else ldv
        idx = None if index is None else np.ascontiguousarray(index, dtype=np.uint64)
        stopped = I32()
        _check(lib().isnmf_online_run(self._h, _p(frames), ldv, n, _p(idx), budget, eta, C.byref(stopped)))
        return bool(stopped.value)

    def enqueue(self, frames, n, ldv, index=None, budget=(1 << 64) - 1, eta=0.0):
        idx = None if index is None else np.ascontiguousarray(index, dtype=np.uint64)
        _check(lib().isnmf_online_enqueue(self._h, _p(frames), ldv, n, _p(idx), budget, eta))

    def synchronize(self):
        _check(lib().isnmf_online_synchronize(self._h))

    def trace(self, cap=1 << 20):
        cnt_max = cap
        s = np.empty(cnt_max, dtype=np.uint64)
        o = np.empty(cnt_max)
        sec = np.empty(cnt_max)
        n = I64()
        _check(lib().isnmf_online_get_trace(self._h, _p(s), _p(o), _p(sec), cnt_max, C.byref(n)))
        k = n.value
        return s[:k].copy(), o[:k].copy(), sec[:k].copy()

    def clear_trace(self):
        _check(lib().isnmf_online_clear_trace(self._h))

    def last_h(self, n):
        h = np.empty((self.K, n), order="F")
        _check(lib().isnmf_online_get_last_h(self._h, _p(h), n))
        return h

    def commit(self):
        _check(lib().isnmf_online_commit(self._h))

    def solver(self):
        buf = C.create_string_buffer(16)
        _check(lib().isnmf_online_solver(self._h, buf, 16))
        return buf.value.decode()

    def launch_count(self):
        return int(lib().isnmf_online_launch_count(self._h))


class Profile:
    """CUDA events on the engine's own stream: the whole region, and with
    per_kernel=True also around every K1 / K2 launch."""

    def __init__(self, online, per_kernel=True):
        self.o = online
        self.per_kernel = per_kernel
        self._span = None

    def start(self):
        _check(lib().isnmf_online_profile_begin(self.o._h, 1 if self.per_kernel else 0))

    def stop(self):
        ms, nl, nf, span, tail = D(), I64(), I64(), D(), D()
        _check(lib().isnmf_online_profile_end(self.o._h, C.byref(ms), C.byref(nl), C.byref(nf), C.byref(span),
                                              C.byref(tail)))
        self._span = span.value
        return dict(solve_ms=ms.value, solve_launches=nl.value, solve_frames=nf.value, span_ms=span.value,
                    tail_ms=tail.value)

    def span_ms(self):
        return self._span


def batch_train(v32, w0, h0, max_epochs, eps=1e-12, eta=0.0):
    """batch.hpp:84-143 on the device. v32: F x N fp32 numpy (or torch [N, ldv])."""
    w0, h0 = _f(w0), _f(h0)
    F, K = w0.shape
    N = h0.shape[1]
    if hasattr(v32, "data_ptr"):
        ldv = v32.stride(0)
    else:
        v32 = np.asfortranarray(v32, dtype=np.float32)
        ldv = F
    w = np.empty((F, K), order="F")
    h = np.empty((K, N), order="F")
    obj = np.empty(max(1, max_epochs))
    ep, o0, ld = U64(), D(), D()
    _check(lib().isnmf_batch_train(_p(v32), ldv, F, N, K, _p(w0), _p(h0), max_epochs, eps, eta, _p(w), _p(h),
                                   _p(obj), C.byref(ep), C.byref(o0), C.byref(ld)))
    return dict(w=w, h=h, obj=obj[:ep.value].copy(), epochs=ep.value, initial_obj=o0.value, last_delta=ld.value)


def batch_profile(enable=-1):
    """CUDA-event device time (ms) and kernel launches of the last batch_train call
    (enable=1/0 switches the timing on/off first)."""
    ms, n = D(), I64()
    _check(lib().isnmf_batch_profile(enable, C.byref(ms), C.byref(n)))
    return ms.value, n.value


def evaluate_heldout(test32, w, eps=1e-12, inner_iters=100, seed=0x45):
    """harness.hpp:17-37 on the device. test32: F x N fp32 numpy (or torch [N, ldt])."""
    w = _f(w)
    F, K = w.shape
    if hasattr(test32, "data_ptr"):
        ldt, N = test32.stride(0), test32.shape[0]
    else:
        test32 = np.asfortranarray(test32, dtype=np.float32)
        ldt, N = F, test32.shape[1]
    out = D()
    _check(lib().isnmf_evaluate_heldout(_p(test32), ldt, F, N, _p(w), K, eps, inner_iters, seed, C.byref(out)))
    return out.value


def stft_power(samples, window=512, hop=256):
    """audio.hpp:121-153 on the device: bins x frames fp64 power spectrogram."""
    x = np.ascontiguousarray(samples, dtype=np.float64)
    frames = (x.size - window) // hop + 1 if window >= 2 and hop >= 1 and x.size >= window else 0
    out = np.zeros((window // 2 + 1 if window >= 2 else 1, max(frames, 0)), order="F")
    got = I64()
    _check(lib().isnmf_stft_power(_p(x), x.size, window, hop, _p(out), out.shape[1], C.byref(got)))
    return out


def discard_silence(spec, threshold_db=-60.0):
    """audio.hpp:164-187 on the device: the ascending indices of the retained frames."""
    spec = np.asfortranarray(spec, dtype=np.float64)
    keep = np.empty(max(spec.shape[1], 1), dtype=np.int64)
    n = I64()
    _check(lib().isnmf_discard_silence(_p(spec), spec.shape[0], spec.shape[1], threshold_db, _p(keep), C.byref(n)))
    return keep[:n.value].copy()
