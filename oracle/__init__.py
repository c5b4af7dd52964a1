"""CPU oracle for the AttnCache hot path (arXiv 2510.25979) — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package.  The product
path (``paper_2510_25979_b200``) never imports it and shares no code with it.

The arithmetic lives in ``attncache_oracle.c`` (plain C, fp64 accumulation,
OpenMP over independent units); this module only compiles it with gcc and
marshals numpy arrays.  See that file's header for the paper passages each
function follows.  Every function here has pins in
``tests/test_oracle_pins.py``; none is "parity unpinned".

Storage dtypes are named ``"f32"``, ``"f16"``, ``"bf16"``.  bf16 data is passed
as ``np.uint16`` arrays holding the raw bit patterns (numpy has no bf16).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "attncache_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_DT = {"f32": 0, "f16": 1, "bf16": 2}
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile attncache_oracle.c into liboracle.so with gcc (-O2 -fopenmp)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            P, I64, I32, F32, D = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                   ctypes.c_float, ctypes.c_double)
            lib.oracle_search.argtypes = [P, I64, P, I64, I32, I32, F32, P, P, P, P]
            lib.oracle_scores.argtypes = [P, P, I32, I32, P, P, I64, P]
            lib.oracle_apply.argtypes = [P, I32, P, P, I32, P, I64, I32, I32, P]
            lib.oracle_attend.argtypes = [P, P, P, I32, P, I64, I32, I32, D, P]
            lib.oracle_attention_map.argtypes = [P, P, I32, P, I64, I32, I32, D, P]
            lib.oracle_rope.argtypes = [P, I32, I64, I32, I32, D, P]
            lib.oracle_project.argtypes = [P, I64, I32, I32, P, P, I32, P, P, I32, P]
            lib.oracle_linear.argtypes = [P, I64, I32, P, I32, I32, P]
            lib.oracle_decode.argtypes = [P, I64, I32]
            lib.oracle_decode.restype = D
            lib.oracle_set_threads.argtypes = [I32]
            lib.oracle_get_threads.restype = I32
            _lib = lib
    return _lib


def _raw(a: np.ndarray, dtype: str) -> np.ndarray:
    want = {"f32": np.float32, "f16": np.float16, "bf16": np.uint16}[dtype]
    a = np.ascontiguousarray(a)
    if a.dtype != want:
        raise TypeError(f"oracle: expected {np.dtype(want)} storage for {dtype}, got {a.dtype}")
    return a


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def set_threads(n: int) -> None:
    _load().oracle_set_threads(int(n))


def get_threads() -> int:
    return int(_load().oracle_get_threads())


def decode(a: np.ndarray, dtype: str) -> np.ndarray:
    """Exact fp64 values of stored elements (uses the oracle's own decoders)."""
    a = _raw(a, dtype).reshape(-1)
    lib = _load()
    return np.array([lib.oracle_decode(_ptr(a), i, _DT[dtype]) for i in range(a.size)], dtype=np.float64)


def search(q: np.ndarray, x: np.ndarray, dtype: str, tau: float):
    """Alg. 1 l.255-257: brute-force exact top-1 (lowest index on ties) and the >= tau gate.

    q: [B][D], x: [N][D] in storage dtype.  Returns (idx int64[B], s1 f64[B], s2 f64[B], hit u8[B]).
    """
    q = _raw(q, dtype)
    x = _raw(x, dtype)
    B = q.shape[0]
    N = x.shape[0] if x.ndim == 2 else 0
    D = q.shape[1]
    if N and x.shape[1] != D:
        raise ValueError("feature dims differ")
    idx = np.empty(B, np.int64)
    s1 = np.empty(B, np.float64)
    s2 = np.empty(B, np.float64)
    hit = np.empty(B, np.uint8)
    _load().oracle_search(_ptr(q), B, _ptr(x), N, D, _DT[dtype], float(tau),
                          _ptr(idx), _ptr(s1), _ptr(s2), _ptr(hit))
    return idx, s1, s2, hit


def scores(q: np.ndarray, x: np.ndarray, dtype: str, qb, xi) -> np.ndarray:
    """fp64 inner products q[qb[p]] . x[xi[p]]."""
    q = _raw(q, dtype)
    x = _raw(x, dtype)
    qb = np.ascontiguousarray(qb, dtype=np.int64)
    xi = np.ascontiguousarray(xi, dtype=np.int64)
    if qb.size and (qb.min() < 0 or qb.max() >= q.shape[0] or xi.min() < 0 or xi.max() >= x.shape[0]):
        raise IndexError("oracle.scores: pair index out of range")
    out = np.empty(qb.size, np.float64)
    _load().oracle_scores(_ptr(q), _ptr(x), q.shape[1], _DT[dtype], _ptr(qb), _ptr(xi), qb.size, _ptr(out))
    return out


def apply(A: np.ndarray, a_dtype: str, a_off, V: np.ndarray, v_dtype: str, v_off, S: int, d: int) -> np.ndarray:
    """Alg. 2 l.375: O_u = A_u . V_u for units u with A_u at A.flat[a_off[u]:] ([S][S]) and
    V_u at V.flat[v_off[u]:] ([S][d]).  Returns f64 [n_units][S][d]."""
    A = _raw(A, a_dtype).reshape(-1)
    V = _raw(V, v_dtype).reshape(-1)
    a_off = np.ascontiguousarray(a_off, dtype=np.int64)
    v_off = np.ascontiguousarray(v_off, dtype=np.int64)
    n = a_off.size
    if v_off.size != n:
        raise ValueError("offset lists differ in length")
    if n and (a_off.min() < 0 or a_off.max() + S * S > A.size or v_off.min() < 0 or v_off.max() + S * d > V.size):
        raise IndexError("oracle.apply: unit out of range")
    O = np.empty((n, S, d), np.float64)
    _load().oracle_apply(_ptr(A), _DT[a_dtype], _ptr(a_off), _ptr(V), _DT[v_dtype], _ptr(v_off), n, S, d, _ptr(O))
    return O


def attend(Q: np.ndarray, K: np.ndarray, V: np.ndarray, dtype: str, off, S: int, d: int, scale: float | None = None):
    """Alg. 2 l.376-381 / Eq. 5: O_u = softmax(Q_u K_u^T * scale, causal) . V_u (scale default 1/sqrt(d))."""
    Q = _raw(Q, dtype).reshape(-1)
    K = _raw(K, dtype).reshape(-1)
    V = _raw(V, dtype).reshape(-1)
    off = np.ascontiguousarray(off, dtype=np.int64)
    if not (Q.size == K.size == V.size):
        raise ValueError("Q, K, V sizes differ")
    if off.size and (off.min() < 0 or off.max() + S * d > Q.size):
        raise IndexError("oracle.attend: unit out of range")
    scale = 1.0 / np.sqrt(d) if scale is None else float(scale)
    O = np.empty((off.size, S, d), np.float64)
    _load().oracle_attend(_ptr(Q), _ptr(K), _ptr(V), _DT[dtype], _ptr(off), off.size, S, d, scale, _ptr(O))
    return O


def attention_map(Q: np.ndarray, K: np.ndarray, dtype: str, off, S: int, d: int, scale: float | None = None):
    """Eq. 5 causal probabilities P_u = softmax(Q_u K_u^T * scale, causal), f64 [n_units][S][S]."""
    Q = _raw(Q, dtype).reshape(-1)
    K = _raw(K, dtype).reshape(-1)
    off = np.ascontiguousarray(off, dtype=np.int64)
    if off.size and (off.min() < 0 or off.max() + S * d > Q.size):
        raise IndexError("oracle.attention_map: unit out of range")
    scale = 1.0 / np.sqrt(d) if scale is None else float(scale)
    P = np.empty((off.size, S, S), np.float64)
    _load().oracle_attention_map(_ptr(Q), _ptr(K), _DT[dtype], _ptr(off), off.size, S, d, scale, _ptr(P))
    return P


def rope(X: np.ndarray, dtype: str, S: int, d: int, base: float = 10000.0) -> np.ndarray:
    """Alg. 2 l.379 rotary_pos_emb (rotate-half convention, R29) of [units][S][d] -> f64."""
    X = _raw(X, dtype).reshape(-1)
    if X.size % (S * d) or d % 2:
        raise ValueError("X must hold whole [S][d] units with d even")
    Y = np.empty(X.size, np.float64)
    _load().oracle_rope(_ptr(X), _DT[dtype], X.size // (S * d), S, d, float(base), _ptr(Y))
    return Y.reshape(-1, S, d)


def project(h: np.ndarray, dtype: str, W1: np.ndarray, b1: np.ndarray, W2: np.ndarray, b2: np.ndarray) -> np.ndarray:
    """Alg. 1 l.254 feature_projector (readings R30-R32): f = normalize(W2 relu(W1 h + b1) + b2).

    h: [B][E], W1: [Hd][E], W2: [D][Hd] in storage dtype; b1, b2 float32.  Returns f64 [B][D]."""
    h = _raw(h, dtype)
    W1 = _raw(W1, dtype)
    W2 = _raw(W2, dtype)
    b1 = np.ascontiguousarray(b1, dtype=np.float32)
    b2 = np.ascontiguousarray(b2, dtype=np.float32)
    B, E = h.shape
    Hd, D = W1.shape[0], W2.shape[0]
    if W1.shape != (Hd, E) or W2.shape != (D, Hd) or b1.shape != (Hd,) or b2.shape != (D,):
        raise ValueError("oracle.project: shapes disagree")
    f = np.empty((B, D), np.float64)
    _load().oracle_project(_ptr(h), B, E, _DT[dtype], _ptr(W1), _ptr(b1), Hd, _ptr(W2), _ptr(b2), D, _ptr(f))
    return f


def linear(X: np.ndarray, W: np.ndarray, dtype: str) -> np.ndarray:
    """Alg. 2 l.372 / l.377-378 projections (f4): Y = X W^T, X [M][K], W [N][K] (nn.Linear layout) -> f64 [M][N]."""
    X = _raw(X, dtype)
    W = _raw(W, dtype)
    M, K = X.shape
    N = W.shape[0]
    if W.shape[1] != K:
        raise ValueError("oracle.linear: X [M][K] and W [N][K] disagree on K")
    Y = np.empty((M, N), np.float64)
    _load().oracle_linear(_ptr(X), M, K, _ptr(W), N, _DT[dtype], _ptr(Y))
    return Y
