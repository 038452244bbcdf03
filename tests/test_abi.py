"""C-ABI boundary checks that need no GPU: the library builds/loads, exports every symbol the
header declares, and rejects bad arguments synchronously (before any device access)."""
from __future__ import annotations

import ctypes
import os
import re

import pytest

import paper_2310_02065_b200 as venom

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    import glob
    src = "".join(open(f).read() for f in sorted(glob.glob(os.path.join(ROOT, "include", "*.h"))))
    return sorted(set(re.findall(r"\b(venom_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    venom.build()
    return venom.lib()


def test_exports_every_declared_symbol(L):
    names = _declared_symbols()
    assert {"venom_compress", "venom_spmm", "venom_decompress"} <= set(names)
    for n in names:
        assert hasattr(L, n), n
    assert set(venom.EXPORTED) == set(names)


def test_status_strings_and_version(L):
    assert L.venom_status_string(0) == b"ok"
    assert b"sm_100a" in L.venom_version()
    assert L.venom_kernels_per_call() == 1


@pytest.mark.parametrize("R,K,V,N,M,expect", [
    (1024, 4096, 64, 2, 8, 0), (10, 16, 4, 2, 8, 2), (8, 8, 4, 2, 3, 4), (8, 12, 4, 2, 8, 3),
    (8, 16, 4, 3, 8, 4), (8, 512, 4, 2, 512, 4), (8, 16, 0, 2, 8, 1),
])
def test_compressed_sizes_and_validation(L, R, K, V, N, M, expect):
    nv, nm, nc = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    st = L.venom_compressed_sizes(R, K, venom._Format(V, N, M), ctypes.byref(nv), ctypes.byref(nm),
                                  ctypes.byref(nc))
    assert st == expect
    if st == 0:
        G = K // M
        assert (nv.value, nm.value, nc.value) == (R * G * 2, R * ((G + 1) // 2), (R // V) * G * 4)


def _spmm(L, R=256, K=512, V=128, M=8, T=64, ldb=64, ldc=64, n=2, dt=0):
    P = ctypes.c_void_p
    fake = P(0x10000)  # never dereferenced: validation fails first
    return L.venom_spmm(fake, fake, fake, R, K, venom._Format(V, n, M), fake, T, ldb, fake, ldc,
                        P(0), dt, P(0))


def test_expand_argument_errors(L):
    P = ctypes.c_void_p
    fake = P(0x10000)

    def ex(R=256, K=512, V=64, M=8, dt=0, n=2):
        return L.venom_expand_2to4(fake, fake, fake, R, K, dt, venom._Format(V, n, M), fake, fake, fake,
                                   P(0), P(0))
    assert ex(M=10, K=500) == 4   # M % 4 != 0: no 2:4 re-encoding
    assert ex(R=200) == 2         # V does not divide R
    assert ex(K=500) == 3         # M does not divide K
    assert ex(dt=3) == 5
    assert ex(n=1) == 4


def test_metadata_tc_sizes_and_errors(L):
    P = ctypes.c_void_p
    f = venom._Format
    assert L.venom_metadata_tc_bytes(1024, 4096, f(64, 2, 8)) == 8 * 16 * 128 * 16  # 8 tiles, 16 k-stages
    assert L.venom_metadata_tc_bytes(130, 320, f(13, 2, 10)) == 2 * 1 * 128 * 16
    assert L.venom_metadata_tc_bytes(130, 320, f(7, 2, 10)) == -1  # V does not divide R
    fake = P(0x10000)
    # any G (a partial last 4-group word is completed with 0x4): G = 6 reaches the device check
    assert L.venom_order_metadata(fake, 256, 8 * 6, f(64, 2, 8), P(0x10008), P(0)) == 1  # misaligned
    assert L.venom_order_metadata(fake, 256, 500, f(64, 2, 8), fake, P(0)) == 3
    assert L.venom_order_metadata(fake, 256, 512, f(64, 2, 8), P(0x10008), P(0)) == 1  # misaligned


def test_values_padded_sizes_and_errors(L):
    """The K' tail's execution form (venom_pad_values): R·ceil(G/4)·4 groups of 4 bytes."""
    P = ctypes.c_void_p
    f = venom._Format
    assert L.venom_values_padded_bytes(256, 330, f(64, 2, 10)) == 256 * 36 * 4  # G = 33 -> 36
    assert L.venom_values_padded_bytes(128, 640, f(64, 2, 10)) == 128 * 64 * 4  # G = 64: no padding
    assert L.venom_values_padded_bytes(130, 320, f(7, 2, 10)) == -1
    fake = P(0x10000)
    assert L.venom_pad_values(fake, 256, 330, f(64, 2, 10), P(0x10008), P(0)) == 1  # misaligned out
    assert L.venom_pad_values(fake, 256, 333, f(64, 2, 10), fake, P(0)) == 3
    assert L.venom_pad_values(P(0), 0, 330, f(64, 2, 10), fake, P(0)) == 0  # R = 0: nothing to do


def test_compress_2to4_argument_errors(L):
    P = ctypes.c_void_p
    fake = P(0x10000)

    def c24(R=256, K=512, V=64, M=8, lda=512, dt=0):
        return L.venom_compress_2to4(fake, R, K, lda, dt, venom._Format(V, 2, M), fake, fake, fake, fake,
                                     fake, P(0), P(0))
    assert c24(M=4) == 4          # nothing to re-encode (M % 8)
    assert c24(V=24, R=240) == 4  # V % 16
    assert c24(M=24, K=24 * 20, lda=480) == 4  # M does not divide 128
    assert c24(R=200) == 2
    assert c24(lda=100) == 1
    assert c24(dt=3) == 5


def test_spmm_argument_errors(L):
    assert _spmm(L, R=384, V=96, K=640, M=10) == 4   # gather: V not in {32,64} ∪ 128N; dense-K: M ∤ 128
    assert _spmm(L, K=12 * 6, M=12) == 4       # gather: G = 6 not a multiple of 4; dense-K: M = 12
    assert _spmm(L, K=8 * 6, M=8) == 4         # G = 6: neither strategy (TMA row stride 4G % 16)
    assert _spmm(L, T=60, ldb=64, ldc=64) == 1  # T % 8
    assert _spmm(L, ldb=32) == 1               # ldb < T
    assert _spmm(L, ldc=68) == 1               # ldc % 8
    assert _spmm(L, R=200) == 2                # V does not divide R
    assert _spmm(L, K=500) == 3                # M does not divide K
    assert _spmm(L, n=1) == 4
    assert _spmm(L, dt=3) == 5


def test_compress_argument_errors(L):
    P = ctypes.c_void_p
    f = P(0x10000)
    assert L.venom_compress(f, 10, 16, 16, 0, venom._Format(4, 2, 8), f, f, f, P(0), P(0)) == 2
    assert L.venom_compress(f, 8, 16, 8, 0, venom._Format(4, 2, 8), f, f, f, P(0), P(0)) == 1  # lda < K
    assert L.venom_compress(f, 8, 16, 16, 7, venom._Format(4, 2, 8), f, f, f, P(0), P(0)) == 5
    assert L.venom_decompress(f, f, f, 8, 16, 0, venom._Format(4, 2, 3), f, 16, P(0), P(0)) == 4


def test_masked_compress_and_energy_argument_errors(L):
    P = ctypes.c_void_p
    f = P(0x10000)
    fmt = venom._Format(4, 2, 8)
    assert L.venom_compress_masked(f, 10, 16, 16, f, 16, 0, fmt, f, f, f, P(0), P(0)) == 2  # V ∤ R
    assert L.venom_compress_masked(f, 8, 16, 16, f, 8, 0, fmt, f, f, f, P(0), P(0)) == 1   # ldm < K
    assert L.venom_compress_masked(f, 8, 16, 16, P(0), 16, 0, fmt, f, f, f, P(0), P(0)) == 1  # no mask
    assert L.venom_compress_masked(f, 8, 16, 16, f, 16, 3, fmt, f, f, f, P(0), P(0)) == 5
    assert L.venom_energy(f, 8, 16, 8, f, 4, 0, f, P(0)) == 1      # lda < K
    assert L.venom_energy(f, 8, 16, 16, f, 4, 0, P(0), P(0)) == 1  # no output
    assert L.venom_energy(f, 8, 16, 16, f, 4, 9, f, P(0)) == 5
    assert L.venom_status_string(10) == b"mask is not V:N:M"


def test_no_cpu_fallback_without_device(L):
    """On a GPU-less host a valid call must fail loudly (CUDA / arch error), never compute."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    P = ctypes.c_void_p
    buf = (ctypes.c_uint8 * 4096)()
    p = P(ctypes.addressof(buf) + (16 - ctypes.addressof(buf) % 16) % 16)
    st = L.venom_spmm(p, p, p, 128, 128, venom._Format(64, 2, 8), p, 8, 8, p, 8, P(0), 0, P(0))
    assert st in (8, 9)


@pytest.mark.parametrize("V,M,expect", [(32, 8, 1), (128, 8, 1), (256, 8, 0), (32, 16, 1), (64, 16, 0),
                                        (128, 16, 0), (256, 16, 0), (32, 32, 0), (64, 32, 0), (128, 4, 0),
                                        (64, 10, 0)])
def test_planner_operand_form(L, V, M, expect):
    """venom_prefer_2to4 follows the measured V-scaling crossover (DESIGN.md planner table,
    profiles/r02b_vscaling.txt): the V:2:4 form for M = 8 below V = 256 or V·M < 1024; never for
    M = 4 (already 2:4) or M % 4 != 0."""
    assert L.venom_prefer_2to4(4096, 4096 if M != 10 else 4160, 4096, venom._Format(V, 2, M)) == expect
