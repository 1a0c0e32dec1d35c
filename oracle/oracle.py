"""TEST INFRASTRUCTURE ONLY — ctypes face of the CPU fp64 oracle.

Wraps oracle/_build/liboracle.so (built from isnmf_oracle.hpp + oracle_capi.cpp
by `make -C oracle`).  Used by tests/, __graft_entry__.smoke() as the checker
and bench.py's CPU baseline / --impl reference arm; never by the product.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "_build", "liboracle.so")

CODES = {
    1: "ShapeMismatch", 2: "EmptyDataset", 3: "NegativeInput", 4: "NonPositiveInit",
    5: "ZeroColumn", 6: "InconsistentStats", 7: "NumericalFailure", 8: "DivergedObjective",
    9: "NonFiniteEntry", 10: "NegativeEntry", 11: "IoError",
}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{CODES.get(code, code)}: {msg}")
        self.code = code
        self.kind = CODES.get(code, str(code))


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            build()
        _lib = C.CDLL(_LIB)
        _lib.oracle_last_error.restype = C.c_char_p
        for name in ("oracle_splitmix64", "oracle_mix_seed"):
            getattr(_lib, name).restype = C.c_uint64
            getattr(_lib, name).argtypes = [C.c_uint64] * (1 if name == "oracle_splitmix64" else 2)
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _fortran(a):
    """Column-major fp64 copy (the reference's Eigen layout)."""
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _check(rc):
    if rc != 0:
        raise OracleError(rc, lib().oracle_last_error().decode())


D = C.c_double
I64 = C.c_int64
U64 = C.c_uint64


def splitmix64(x):
    return lib().oracle_splitmix64(U64(x))


def mix_seed(s, t):
    return lib().oracle_mix_seed(U64(s), U64(t))


def uniform01(seed, n):
    out = np.empty(n)
    lib().oracle_uniform01(U64(seed), I64(n), _p(out))
    return out


def cycle_permutation(seed, cycle, n):
    out = np.empty(n, dtype=np.uint64)
    lib().oracle_cycle_permutation(U64(seed), U64(cycle), U64(n), _p(out))
    return out


def random_positive(rows, cols, seed, lo=0.05, hi=2.0):
    """test_core.cpp:17-24 / test_kernels.cpp:13-20 — column-major fill."""
    u = uniform01(seed, rows * cols)
    return (lo + (hi - lo) * u).reshape(cols, rows).T.copy(order="F")


def is_divergence(y, x, eps):
    y, x = _f64(y), _f64(x)
    out = D()
    _check(lib().oracle_is_divergence(_p(y), I64(y.size), _p(x), I64(x.size), D(eps), C.byref(out)))
    return out.value


def objective(v, w, h, eps):
    v, w, h = _fortran(v), _fortran(w), _fortran(h)
    out = D()
    _check(lib().oracle_objective(_p(v), _p(w), _p(h), I64(w.shape[0]), I64(w.shape[1]), I64(v.shape[1]), D(eps),
                                  C.byref(out)))
    return out.value


def solve_h(v, w, h0, iters, eps):
    """v: F or F x N; h0: K or K x N."""
    v1 = np.ndim(v) == 1
    v, h0, w = _fortran(np.atleast_2d(v).T if v1 else v), _fortran(np.atleast_2d(h0).T if v1 else h0), _fortran(w)
    out = np.empty_like(h0, order="F")
    _check(lib().oracle_solve_h(_p(v), _p(w), _p(h0), I64(v.shape[0]), I64(h0.shape[0]), I64(v.shape[1]),
                                C.c_int(iters), D(eps), _p(out)))
    return out[:, 0] if v1 else out


def sample_stats(v, w, h, eps):
    """Sum over columns of kernels.hpp:112-121 (accumulate_sample_stats)."""
    v1 = np.ndim(v) == 1
    v, h, w = _fortran(np.atleast_2d(v).T if v1 else v), _fortran(np.atleast_2d(h).T if v1 else h), _fortran(w)
    F, K = w.shape
    a = np.empty((F, K), order="F")
    b = np.empty((F, K), order="F")
    _check(lib().oracle_sample_stats(_p(v), _p(w), _p(h), I64(F), I64(K), I64(v.shape[1]), D(eps), _p(a), _p(b)))
    return a, b


def batch_stats(v, w, h, eps):
    v, w, h = _fortran(v), _fortran(w), _fortran(h)
    F, K = w.shape
    a = np.empty((F, K), order="F")
    b = np.empty((F, K), order="F")
    _check(lib().oracle_batch_stats(_p(v), _p(w), _p(h), I64(F), I64(K), I64(v.shape[1]), D(eps), _p(a), _p(b)))
    return a, b


def update_w(a, b, w_prev):
    a, b, w_prev = _fortran(a), _fortran(b), _fortran(w_prev)
    if a.shape != b.shape or a.shape != w_prev.shape:
        # shape errors come from the C side for parity of the error type
        pass
    F, K = a.shape
    w = np.empty((F, K), order="F")
    if a.shape != b.shape or a.shape != w_prev.shape:
        raise OracleError(1, "update_w: shape mismatch")
    _check(lib().oracle_update_w(_p(a), _p(b), _p(w_prev), I64(F), I64(K), _p(w)))
    return w


def aux_value(a, b, w):
    a, b, w = _fortran(a), _fortran(b), _fortran(w)
    out = D()
    _check(lib().oracle_aux_value(_p(a), _p(b), _p(w), I64(a.shape[0]), I64(a.shape[1]), C.byref(out)))
    return out.value


def aux_constant(v, w, h, eps):
    v, w, h = _fortran(v), _fortran(w), _fortran(h)
    out = D()
    _check(lib().oracle_aux_constant(_p(v), _p(w), _p(h), I64(w.shape[0]), I64(w.shape[1]), I64(v.shape[1]),
                                     D(eps), C.byref(out)))
    return out.value


def rescale_dictionary(w, a, b, warm_h=None):
    """Returns rescaled copies (w, a, b, warm_h)."""
    w, a, b = _fortran(w).copy(order="F"), _fortran(a).copy(order="F"), _fortran(b).copy(order="F")
    H = _fortran(warm_h).copy(order="F") if warm_h is not None else None
    if H is not None and H.shape[0] != w.shape[1]:
        raise OracleError(1, "rescale_dictionary: warm_h rows vs W cols")
    if w.shape != a.shape or w.shape != b.shape:
        raise OracleError(1, "rescale_dictionary: shapes")
    _check(lib().oracle_rescale_dictionary(_p(w), _p(a), _p(b), I64(w.shape[0]), I64(w.shape[1]), _p(H),
                                           I64(H.shape[1] if H is not None else 0)))
    return w, a, b, H


def frobenius_delta(a, b):
    a, b = _fortran(np.atleast_2d(a)), _fortran(np.atleast_2d(b))
    out = D()
    _check(lib().oracle_frobenius_delta(_p(a), I64(a.shape[0]), I64(a.shape[1]), _p(b), I64(b.shape[0]),
                                        I64(b.shape[1]), C.byref(out)))
    return out.value


def config_check(k=8, epsilon=1e-12, eta=-1.0, beta=1000, r=0.7, inner_iters=0, restart="warm", n_seeds=5,
                 init_stats_weight=1.0, F=1, K=1):
    it = C.c_int()
    et = D()
    _check(lib().oracle_config_check(C.c_int(k), D(epsilon), D(eta), C.c_int(beta), D(r), C.c_int(inner_iters),
                                     C.c_int(0 if restart == "warm" else 1), C.c_int(n_seeds), D(init_stats_weight),
                                     I64(F), I64(K), C.byref(it), C.byref(et)))
    return it.value, et.value


def fresh_h_init(v, w, eps, seed, t):
    v, w = _f64(v), _fortran(w)
    h = np.empty(w.shape[1])
    _check(lib().oracle_fresh_h_init(_p(v), _p(w), I64(w.shape[0]), I64(w.shape[1]), D(eps), U64(seed), U64(t),
                                     _p(h)))
    return h


def default_h0(v, w, eps=1e-12):
    v, w = _fortran(v), _fortran(w)
    h = np.empty((w.shape[1], v.shape[1]), order="F")
    _check(lib().oracle_default_h0(_p(v), _p(w), I64(w.shape[0]), I64(w.shape[1]), I64(v.shape[1]), D(eps), _p(h)))
    return h


def evaluate_heldout(w, test, eps=1e-12, inner_iters=100, seed=0x45):
    """harness.hpp:17-37."""
    w, test = _fortran(w), _fortran(test)
    out = D()
    _check(lib().oracle_evaluate_heldout(_p(w), _p(test), I64(w.shape[0]), I64(w.shape[1]), I64(test.shape[0]),
                                         I64(test.shape[1]), D(eps), C.c_int(inner_iters), C.c_uint64(seed),
                                         C.byref(out)))
    return out.value


def heldout_h0(w, test, eps=1e-12, seed=0x45):
    w, test = _fortran(w), _fortran(test)
    h = np.empty((w.shape[1], test.shape[1]), order="F")
    _check(lib().oracle_heldout_h0(_p(w), _p(test), I64(w.shape[0]), I64(w.shape[1]), I64(test.shape[1]), D(eps),
                                   C.c_uint64(seed), _p(h)))
    return h


def init_from_samples(v, k, seed, eps=1e-12):
    v = _fortran(v)
    w = np.empty((v.shape[0], k), order="F")
    _check(lib().oracle_init_from_samples(_p(v), I64(v.shape[0]), I64(v.shape[1]), C.c_int(k), U64(seed), D(eps),
                                          _p(w)))
    return w


class Online:
    """online.hpp:224-419 restated: make_online_state + online_resume."""

    def __init__(self, w0, *, beta, r=1.0, inner_iters=0, restart="warm", seed=1, epsilon=1e-12, eta=0.0,
                 budget=None, init_stats_weight=1.0, dataset_size=None, dataset=None):
        w0 = _fortran(w0)
        self.F, self.K = w0.shape
        ds = _fortran(dataset) if dataset is not None else None
        h = C.c_void_p()
        budget = (1 << 63) if budget is None else budget
        _check(lib().oracle_online_create(C.byref(h), _p(w0), I64(self.F), I64(self.K), C.c_int(beta), D(r),
                                          C.c_int(inner_iters), C.c_int(0 if restart == "warm" else 1), U64(seed),
                                          D(epsilon), D(eta), U64(budget), D(init_stats_weight),
                                          C.c_int(dataset_size is not None), U64(dataset_size or 0), _p(ds),
                                          I64(ds.shape[1] if ds is not None else 0)))
        self._h = h
        self.warm_n = ds.shape[1] if ds is not None else 0

    def __del__(self):
        if getattr(self, "_h", None) is not None and _lib is not None:
            _lib.oracle_online_destroy(self._h)
            self._h = None

    def set(self, w=None, a=None, b=None, pending_a=None, pending_b=None, warm_h=None, rho=-1.0, t=0, commits=0):
        arrs = [None if x is None else _fortran(x) for x in (w, a, b, pending_a, pending_b, warm_h)]
        if arrs[5] is not None:
            self.warm_n = arrs[5].shape[1]
        _check(lib().oracle_online_set(self._h, *[_p(x) for x in arrs], I64(self.warm_n), D(rho), U64(t), U64(commits)))

    def state(self, warm_h=False):
        F, K = self.F, self.K
        out = {n: np.empty((F, K), order="F") for n in ("w", "a", "b", "pending_a", "pending_b")}
        wh = np.empty((K, self.warm_n), order="F") if (warm_h and self.warm_n) else None
        t, c = U64(), U64()
        sc = np.empty(6)
        _check(lib().oracle_online_get(self._h, _p(out["w"]), _p(out["a"]), _p(out["b"]), _p(out["pending_a"]),
                                       _p(out["pending_b"]), _p(wh), C.byref(t), C.byref(c), _p(sc)))
        out.update(t=t.value, commits=c.value, last_delta=sc[0], last_minibatch_obj=sc[1], pending_div=sc[2],
                   pending_count=int(sc[3]), rho=sc[4], final_train_obj=sc[5])
        if wh is not None:
            out["warm_h"] = wh
        return out

    def run(self, v, index=None, index_base=0, trace_cap=1 << 20):
        """Visit the columns of v (F x n, fp32 or fp64) in order."""
        v = np.asarray(v)
        is32 = v.dtype == np.float32
        v = np.asfortranarray(v, dtype=np.float32 if is32 else np.float64)
        n = v.shape[1]
        idx = None if index is None else np.ascontiguousarray(index, dtype=np.uint64)
        tt = np.empty(min(trace_cap, n + 1), dtype=np.uint64)
        to = np.empty(min(trace_cap, n + 1))
        nt = I64()
        _check(lib().oracle_online_run(self._h, _p(v), C.c_int(is32), I64(n), _p(idx), U64(index_base), _p(tt),
                                       _p(to), I64(tt.size), C.byref(nt)))
        return tt[:nt.value].copy(), to[:nt.value].copy()

    def step(self, frame, index):
        fr = _f64(frame)
        _check(lib().oracle_online_step(self._h, _p(fr), I64(fr.size), U64(index)))

    def commit(self):
        _check(lib().oracle_online_commit(self._h))


def batch_train(v, w0, h0, max_epochs, eps=1e-12, eta=0.0):
    v, w0, h0 = _fortran(v), _fortran(w0), _fortran(h0)
    F, K = w0.shape
    N = v.shape[1]
    w = np.empty((F, K), order="F")
    h = np.empty((K, N), order="F")
    obj = np.empty(max(1, max_epochs))
    ep = I64()
    o0 = D()
    ld = D()
    _check(lib().oracle_batch_train(_p(v), _p(w0), _p(h0), I64(F), I64(K), I64(N), U64(max_epochs), D(eps), D(eta),
                                    _p(w), _p(h), _p(obj), C.byref(ep), C.byref(o0), C.byref(ld)))
    return dict(w=w, h=h, obj=obj[:ep.value].copy(), epochs=ep.value, initial_obj=o0.value, last_delta=ld.value)


def baseline_online(v32, w0, a0, b0, beta, iters, rho, eps=1e-12, threads=1):
    """CPU baseline: warm-ones online pass over fp32 frames; returns (W, last obj)."""
    v32 = np.asfortranarray(v32, dtype=np.float32)
    w0, a0, b0 = _fortran(w0), _fortran(a0), _fortran(b0)
    F, K = w0.shape
    w = np.empty((F, K), order="F")
    obj = D()
    _check(lib().oracle_baseline_online(_p(v32), I64(F), I64(K), I64(v32.shape[1]), C.c_int(beta), C.c_int(iters),
                                        D(eps), D(rho), _p(w0), _p(a0), _p(b0), C.c_int(threads), _p(w),
                                        C.byref(obj)))
    return w, obj.value
