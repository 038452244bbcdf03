"""CPU oracle for the V:N:M hot path — TEST INFRASTRUCTURE ONLY.

Python face of ``oracle/venom_oracle.c`` (plain C, fp64, scalar loops written from the paper;
see that file's header for what each function follows and how it is pinned). Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may
import this package. The product package ``paper_2310_02065_b200`` never imports it and shares no
code with it.

Arrays cross the boundary as numpy ``uint16`` bit patterns (fp16 or bf16, selected by ``dtype``
0 / 1) plus ``uint8`` metadata / column_idx, exactly the byte layouts DESIGN.md fixes.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "venom_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

OK = 0
INVALID_ARGUMENT = 1
NON_DIVISIBLE_ROWS = 2
NON_DIVISIBLE_COLS = 3
UNSUPPORTED_PATTERN = 4
UNSUPPORTED_DTYPE = 5
NON_FINITE = 6
CORRUPT_METADATA = 7
INVALID_MASK = 10

F16, BF16 = 0, 1


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"oracle {what} failed with status {status}")
        self.status = status


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2, no fast-math, OpenMP over independent rows)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        P, I64, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        lib.oracle_decode.restype = ctypes.c_double
        lib.oracle_decode.argtypes = [ctypes.c_uint16, I]
        lib.oracle_validate.argtypes = [I64, I64, I, I, I]
        lib.oracle_compress.argtypes = [P, I64, I64, I64, I, I, I, I, P, P, P]
        lib.oracle_decompress.argtypes = [P, P, P, I64, I64, I, I, I, I, P, I64]
        lib.oracle_spmm_compressed.argtypes = [P, P, P, I64, I64, I, I, I, I, P, I64, I64, P, P, I64]
        lib.oracle_gemm_dense.argtypes = [P, I64, I64, I64, I, P, I64, I64, P, P, I64]
        lib.oracle_num_threads.argtypes = []
        lib.oracle_set_num_threads.argtypes = [I]
        lib.oracle_expand_2to4.argtypes = [P, P, P, I64, I64, I, I, I, P, P, P]
        lib.oracle_compress_masked.argtypes = [P, I64, I64, I64, I, P, I64, I, I, I, P, P, P]
        lib.oracle_energy.argtypes = [P, I64, I64, I64, I, P, I64, P]
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def sizes(R: int, K: int, V: int, M: int):
    """(values elements, metadata bytes, column_idx bytes) — PAPER.md:194-195."""
    G = K // M
    return R * G * 2, R * ((G + 1) // 2), (R // V) * G * 4


def decode(bits: int, dtype: int) -> float:
    return _load().oracle_decode(int(bits), int(dtype))


def validate(R, K, V, N, M) -> int:
    return _load().oracle_validate(R, K, V, N, M)


def num_threads() -> int:
    return _load().oracle_num_threads()


def set_num_threads(n: int) -> None:
    """Thread count of the OpenMP loops (timing legs only; n <= 0 = all host cores)."""
    _load().oracle_set_num_threads(int(n))


def compress(A: np.ndarray, dtype: int, V: int, M: int, N: int = 2, check: bool = True):
    """A: (R, K) uint16 bit patterns (row stride may exceed K). Returns (values, metadata, column_idx)
    as ((R, K/M, 2) uint16, (R, ceil(K/M/2)) uint8, (R/V, K/M, 4) uint8)."""
    A = np.asarray(A)
    assert A.dtype == np.uint16 and A.ndim == 2 and A.strides[1] == 2
    R, K = A.shape
    lda = A.strides[0] // 2
    G = K // M if M > 0 else 0
    values = np.zeros((R, max(G, 0), 2), np.uint16)
    metadata = np.zeros((R, (max(G, 0) + 1) // 2), np.uint8)
    cidx = np.zeros((R // V if V > 0 else 0, max(G, 0), 4), np.uint8)
    st = _load().oracle_compress(_ptr(A), R, K, lda, dtype, V, N, M,
                                 _ptr(values), _ptr(metadata), _ptr(cidx))
    if st != OK:
        if check:
            raise OracleError(st, "compress")
        return st
    return values, metadata, cidx


def compress_masked(A: np.ndarray, mask: np.ndarray, dtype: int, V: int, M: int, N: int = 2,
                    check: bool = True):
    """Compression with the kept set given by an external V:N:M mask (uint8, non-zero = keep);
    see oracle_compress_masked. Same outputs as compress()."""
    A = np.asarray(A)
    mask = np.asarray(mask)
    assert A.dtype == np.uint16 and A.ndim == 2 and A.strides[1] == 2
    assert mask.dtype == np.uint8 and mask.shape == A.shape and mask.strides[1] == 1
    R, K = A.shape
    G = K // M if M > 0 else 0
    values = np.zeros((R, max(G, 0), 2), np.uint16)
    metadata = np.zeros((R, (max(G, 0) + 1) // 2), np.uint8)
    cidx = np.zeros((R // V if V > 0 else 0, max(G, 0), 4), np.uint8)
    st = _load().oracle_compress_masked(_ptr(A), R, K, A.strides[0] // 2, dtype, _ptr(mask),
                                        mask.strides[0], V, N, M, _ptr(values), _ptr(metadata), _ptr(cidx))
    if st != OK:
        if check:
            raise OracleError(st, "compress_masked")
        return st
    return values, metadata, cidx


def energy(A: np.ndarray, values: np.ndarray, dtype: int):
    """(kept sum, dense sum, energy) in fp64 — PAPER.md:305-309; see oracle_energy."""
    A = np.asarray(A)
    assert A.dtype == np.uint16 and A.ndim == 2 and A.strides[1] == 2
    v = np.ascontiguousarray(values).reshape(-1)
    out = np.zeros(3, np.float64)
    st = _load().oracle_energy(_ptr(A), A.shape[0], A.shape[1], A.strides[0] // 2, dtype, _ptr(v),
                               v.size, _ptr(out))
    if st != OK:
        raise OracleError(st, "energy")
    return float(out[0]), float(out[1]), float(out[2])


def decompress(values, metadata, column_idx, R: int, K: int, dtype: int, V: int, M: int,
               N: int = 2, check: bool = True):
    out = np.zeros((R, K), np.uint16)
    st = _load().oracle_decompress(_ptr(np.ascontiguousarray(values)), _ptr(np.ascontiguousarray(metadata)),
                                   _ptr(np.ascontiguousarray(column_idx)), R, K, dtype, V, N, M,
                                   _ptr(out), K)
    if st != OK:
        if check:
            raise OracleError(st, "decompress")
        return st
    return out


def expand_2to4(values, metadata, column_idx, R: int, K: int, V: int, M: int, N: int = 2,
                check: bool = True):
    """V:N:M (M % 4 == 0) -> the same matrix as V:2:4 over the original K (see the C source)."""
    G2 = K // 4
    v2 = np.zeros((R, G2, 2), np.uint16)
    m2 = np.zeros((R, (G2 + 1) // 2), np.uint8)
    c2 = np.zeros((R // V, G2, 4), np.uint8)
    st = _load().oracle_expand_2to4(_ptr(np.ascontiguousarray(values)), _ptr(np.ascontiguousarray(metadata)),
                                    _ptr(np.ascontiguousarray(column_idx)), R, K, V, N, M,
                                    _ptr(v2), _ptr(m2), _ptr(c2))
    if st != OK:
        if check:
            raise OracleError(st, "expand_2to4")
        return st
    return v2, m2, c2


def spmm(values, metadata, column_idx, R: int, K: int, dtype: int, V: int, M: int,
         B: np.ndarray, bias=None, N: int = 2) -> np.ndarray:
    """fp64 C = decompress(A)·B (+ bias) straight on the compressed operand. B: (K, T) uint16
    (row stride may exceed T, e.g. a column subset of a wider matrix)."""
    assert B.dtype == np.uint16 and B.ndim == 2 and B.strides[1] == 2 and B.shape[0] == K
    T = B.shape[1]
    ldb = B.strides[0] // 2
    C = np.zeros((R, T), np.float64)
    st = _load().oracle_spmm_compressed(_ptr(np.ascontiguousarray(values)), _ptr(np.ascontiguousarray(metadata)),
                                        _ptr(np.ascontiguousarray(column_idx)), R, K, dtype, V, N, M,
                                        _ptr(B), T, ldb,
                                        _ptr(None if bias is None else np.ascontiguousarray(bias)), _ptr(C), T)
    if st != OK:
        raise OracleError(st, "spmm")
    return C


def gemm_dense(A: np.ndarray, B: np.ndarray, dtype: int, bias=None) -> np.ndarray:
    """fp64 C = A·B (+ bias), k ascending; A (R, K), B (K, T) uint16 bit patterns."""
    A = np.ascontiguousarray(A)
    assert B.dtype == np.uint16 and B.strides[1] == 2
    R, K = A.shape
    T = B.shape[1]
    C = np.zeros((R, T), np.float64)
    st = _load().oracle_gemm_dense(_ptr(A), R, K, K, dtype, _ptr(B), T, B.strides[0] // 2,
                                   _ptr(None if bias is None else np.ascontiguousarray(bias)), _ptr(C), T)
    if st != OK:
        raise OracleError(st, "gemm_dense")
    return C
