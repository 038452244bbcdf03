"""venom-b200: the data-parallel hot path of VENOM / Spatha (arXiv 2310.02065) for NVIDIA B200.

Thin ctypes binding over ``libvenom.so`` (C ABI in ``include/venom.h``). This module only
marshals arguments: PyTorch provides device memory and the current stream; every step of the
path (compression, decompression, SpMM) runs in the sm_100a kernels of ``csrc/``. There is no
CPU fallback: if the library is missing or the device is not sm_100, calls raise.

Paper vocabulary: a V:N:M matrix keeps, per V×M block, 4 columns
(``column_idx``, the paper's *column-loc*) and per row 2 of those 4 (``values`` + 2-bit
*m-indices* packed in ``metadata``). ``spmm`` computes C = A·B (+ bias) like
``spatha.spmm(values, columns, metadata, input, bias)``.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libvenom.so")

OK = 0
STATUS_NAMES = {
    0: "VENOM_OK", 1: "VENOM_ERR_INVALID_ARGUMENT", 2: "VENOM_ERR_NON_DIVISIBLE_ROWS",
    3: "VENOM_ERR_NON_DIVISIBLE_COLS", 4: "VENOM_ERR_UNSUPPORTED_PATTERN",
    5: "VENOM_ERR_UNSUPPORTED_DTYPE", 6: "VENOM_ERR_NON_FINITE", 7: "VENOM_ERR_CORRUPT_METADATA",
    8: "VENOM_ERR_ARCH", 9: "VENOM_ERR_CUDA", 10: "VENOM_ERR_INVALID_MASK",
}
EXPORTED = ["venom_compressed_sizes", "venom_compress", "venom_decompress", "venom_spmm",
            "venom_spmm_ex", "venom_expand_2to4", "venom_compress_2to4", "venom_prefer_2to4",
            "venom_metadata_tc_bytes", "venom_values_padded_bytes", "venom_pad_values",
            "venom_order_metadata", "venom_kernels_per_call", "venom_status_string",
            "venom_version", "venom_compress_masked", "venom_energy",
            # include/venom_encoder.h (encoder layout helpers, not the V:N:M method)
            "venom_enc_add_layernorm", "venom_enc_heads_to_fm"]


class VenomError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: {STATUS_NAMES.get(status, status)}")
        self.status = status


class _Format(ctypes.Structure):
    _fields_ = [("v", ctypes.c_int32), ("n", ctypes.c_int32), ("m", ctypes.c_int32)]


class _Opts(ctypes.Structure):
    _fields_ = [("tile_t", ctypes.c_int32), ("stages", ctypes.c_int32), ("max_ctas", ctypes.c_int32),
                ("strategy", ctypes.c_int32), ("cta_pair", ctypes.c_int32),
                ("metadata_tc", ctypes.c_void_p), ("c_transposed", ctypes.c_int32),
                ("b_kmajor", ctypes.c_int32), ("activation", ctypes.c_int32), ("group_n", ctypes.c_int32),
                ("c_peers", ctypes.POINTER(ctypes.c_void_p)), ("n_peers", ctypes.c_int32),
                ("values_padded", ctypes.c_void_p), ("b_scratch", ctypes.c_void_p)]


STRATEGY_AUTO, STRATEGY_GATHER, STRATEGY_DENSE_K = 0, 1, 2
# spmm(gelu=...): opts.activation (include/venom.h): GELU erf form (True / "erf") or tanh form ("tanh")
_ACTIVATIONS = {False: 0, None: 0, True: 1, "erf": 1, "tanh": 2}


_lib = None


def lib() -> ctypes.CDLL:
    """Load libvenom.so (built by ``build()`` / ``__graft_entry__.build()``); raise if absent."""
    global _lib
    if _lib is None:
        # VENOM_LIB selects another build of the same ABI (tools/ablate.py: libvenom_ablation.so)
        path = os.environ.get("VENOM_LIB") or LIB_PATH
        if not os.path.exists(path):
            raise RuntimeError(f"libvenom.so not built ({path}); run python -m "
                               "paper_2310_02065_b200.build — there is no CPU fallback")
        L = ctypes.CDLL(path)
        P, I64, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        L.venom_compressed_sizes.argtypes = [I64, I64, _Format, P, P, P]
        L.venom_compress.argtypes = [P, I64, I64, I64, ctypes.c_int, _Format, P, P, P, P, P]
        L.venom_decompress.argtypes = [P, P, P, I64, I64, ctypes.c_int, _Format, P, I64, P, P]
        L.venom_spmm.argtypes = [P, P, P, I64, I64, _Format, P, I64, I64, P, I64, P, ctypes.c_int, P]
        L.venom_expand_2to4.argtypes = [P, P, P, I64, I64, ctypes.c_int, _Format, P, P, P, P, P]
        L.venom_prefer_2to4.argtypes = [I64, I64, I64, _Format]
        L.venom_metadata_tc_bytes.argtypes = [I64, I64, _Format]
        L.venom_metadata_tc_bytes.restype = I64
        L.venom_order_metadata.argtypes = [P, I64, I64, _Format, P, P]
        L.venom_values_padded_bytes.argtypes = [I64, I64, _Format]
        L.venom_values_padded_bytes.restype = I64
        L.venom_pad_values.argtypes = [P, I64, I64, _Format, P, P]
        L.venom_pad_values.restype = ctypes.c_int
        L.venom_compress_2to4.argtypes = [P, I64, I64, I64, ctypes.c_int, _Format, P, P, P, P, P, P, P]
        L.venom_compress_masked.argtypes = [P, I64, I64, I64, P, I64, ctypes.c_int, _Format, P, P, P, P, P]
        L.venom_energy.argtypes = [P, I64, I64, I64, P, I64, ctypes.c_int, P, P]
        L.venom_enc_add_layernorm.argtypes = [P, P, P, P, I64, I64, ctypes.c_float, ctypes.c_int, P, P, I64, P]
        L.venom_enc_heads_to_fm.argtypes = [P, I64, I64, I64, I64, I64, I64, I64, ctypes.c_int, P, I64, P]
        L.venom_prefer_2to4.restype = ctypes.c_int
        L.venom_spmm_ex.argtypes = [P, P, P, I64, I64, _Format, P, I64, I64, P, I64, P, ctypes.c_int,
                                    ctypes.POINTER(_Opts), P]
        for fn in ("venom_compressed_sizes", "venom_compress", "venom_decompress", "venom_spmm",
                   "venom_spmm_ex", "venom_expand_2to4", "venom_order_metadata", "venom_compress_2to4"):
            getattr(L, fn).restype = ctypes.c_int
        L.venom_status_string.argtypes = [ctypes.c_int]
        L.venom_status_string.restype = ctypes.c_char_p
        L.venom_version.restype = ctypes.c_char_p
        L.venom_kernels_per_call.restype = I32
        _lib = L
    return _lib


def build(force: bool = False) -> str:
    from .build import build as _b
    return _b(force=force)


def _dt(t: torch.dtype) -> int:
    if t == torch.float16:
        return 0
    if t == torch.bfloat16:
        return 1
    raise VenomError(5, f"dtype {t}")


def _stream(device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _check(st: int, what: str):
    if st != OK:
        raise VenomError(st, what)


@dataclass
class VNMTensor:
    """A V:N:M-compressed R×K matrix (Fig 3). N is always 2."""
    values: torch.Tensor      # dtype[R, K/M, 2]
    metadata: torch.Tensor    # uint8[R, ceil(K/M/2)]
    column_idx: torch.Tensor  # uint8[R/V, K/M, 4]
    R: int
    K: int
    V: int
    M: int
    N: int = 2
    metadata_tc: Optional[torch.Tensor] = None  # uint8, tensor-core order (order_metadata)
    values_padded: Optional[torch.Tensor] = None  # rows padded to 4 groups (pad_values; G % 4 != 0)

    @property
    def dtype(self) -> torch.dtype:
        return self.values.dtype

    @property
    def nnz(self) -> int:
        return self.R * (self.K // self.M) * 2

    def fmt(self) -> _Format:
        return _Format(self.V, self.N, self.M)


def compressed_sizes(R: int, K: int, V: int, M: int, N: int = 2):
    nv, nm, nc = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _check(lib().venom_compressed_sizes(R, K, _Format(V, N, M), ctypes.byref(nv), ctypes.byref(nm),
                                        ctypes.byref(nc)), "venom_compressed_sizes")
    return nv.value, nm.value, nc.value


def compress(A: torch.Tensor, V: int, M: int, N: int = 2, status: Optional[torch.Tensor] = None,
             check: bool = False, out: Optional[VNMTensor] = None) -> VNMTensor:
    """Magnitude V:N:M compression on the GPU. ``status`` (int32[1] on the
    device) receives data-dependent errors; ``check=True`` allocates one and synchronises to read
    it (raising on non-finite input)."""
    assert A.is_cuda and A.dim() == 2 and A.stride(1) == 1, "A: 2-D CUDA tensor, unit column stride"
    R, K = A.shape
    nv, nm, nc = compressed_sizes(R, K, V, M, N)
    G = K // M
    if out is not None:
        assert (out.R, out.K, out.V, out.M) == (R, K, V, M) and out.dtype == A.dtype
        values, metadata, column_idx = out.values, out.metadata, out.column_idx
    else:
        values = torch.empty((R, G, 2), dtype=A.dtype, device=A.device)
        metadata = torch.empty((R, (G + 1) // 2), dtype=torch.uint8, device=A.device)
        column_idx = torch.empty((R // V, G, 4), dtype=torch.uint8, device=A.device)
    if check and status is None:
        status = torch.zeros(1, dtype=torch.int32, device=A.device)
    st = lib().venom_compress(ctypes.c_void_p(A.data_ptr()), R, K, A.stride(0), _dt(A.dtype),
                              _Format(V, N, M), ctypes.c_void_p(values.data_ptr()),
                              ctypes.c_void_p(metadata.data_ptr()), ctypes.c_void_p(column_idx.data_ptr()),
                              ctypes.c_void_p(status.data_ptr() if status is not None else 0),
                              _stream(A.device))
    _check(st, "venom_compress")
    if check:
        s = int(status.item())
        _check(s, "venom_compress (device status)")
    if out is not None:
        if out.metadata_tc is not None:
            # the tensor-core-ordered copy of the old metadata would pair stale m-indices with the
            # new values in spmm: re-derive it from the new metadata (same stream, in order)
            order_metadata(out, out=out.metadata_tc)
        return out
    return VNMTensor(values, metadata, column_idx, R, K, V, M, N)


def compress_masked(A: torch.Tensor, mask: torch.Tensor, V: int, M: int, N: int = 2,
                    status: Optional[torch.Tensor] = None, check: bool = False) -> VNMTensor:
    """V:N:M compression of ``A`` with the kept set given by an external V:N:M ``mask`` (uint8 or
    bool, non-zero keeps; e.g. from a second-order pruner). The result is exactly
    A∘mask. ``check=True`` raises on a non-V:N:M mask or non-finite input."""
    assert A.is_cuda and A.dim() == 2 and A.stride(1) == 1, "A: 2-D CUDA tensor, unit column stride"
    if mask.dtype == torch.bool:
        mask = mask.view(torch.uint8)
    assert mask.dtype == torch.uint8 and mask.shape == A.shape and mask.stride(1) == 1 and mask.device == A.device
    R, K = A.shape
    compressed_sizes(R, K, V, M, N)
    G = K // M
    values = torch.empty((R, G, 2), dtype=A.dtype, device=A.device)
    metadata = torch.empty((R, (G + 1) // 2), dtype=torch.uint8, device=A.device)
    column_idx = torch.empty((R // V, G, 4), dtype=torch.uint8, device=A.device)
    if check and status is None:
        status = torch.zeros(1, dtype=torch.int32, device=A.device)
    st = lib().venom_compress_masked(ctypes.c_void_p(A.data_ptr()), R, K, A.stride(0),
                                     ctypes.c_void_p(mask.data_ptr()), mask.stride(0), _dt(A.dtype),
                                     _Format(V, N, M), ctypes.c_void_p(values.data_ptr()),
                                     ctypes.c_void_p(metadata.data_ptr()), ctypes.c_void_p(column_idx.data_ptr()),
                                     ctypes.c_void_p(status.data_ptr() if status is not None else 0),
                                     _stream(A.device))
    _check(st, "venom_compress_masked")
    if check:
        _check(int(status.item()), "venom_compress_masked (device status)")
    return VNMTensor(values, metadata, column_idx, R, K, V, M, N)


def energy(A: torch.Tensor, kept: "VNMTensor | torch.Tensor", out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Energy of a pruning on the GPU: float64[3] {Σ|kept|, Σ|dense|, energy}.
    ``kept`` is a compressed operand (its values) or any tensor of kept values."""
    assert A.is_cuda and A.dim() == 2 and A.stride(1) == 1
    vals = kept.values if isinstance(kept, VNMTensor) else kept
    assert vals.is_contiguous() and vals.dtype == A.dtype
    if out is None:
        out = torch.empty(3, dtype=torch.float64, device=A.device)
    st = lib().venom_energy(ctypes.c_void_p(A.data_ptr()), A.shape[0], A.shape[1], A.stride(0),
                            ctypes.c_void_p(vals.data_ptr()), vals.numel(), _dt(A.dtype),
                            ctypes.c_void_p(out.data_ptr()), _stream(A.device))
    _check(st, "venom_energy")
    return out


def enc_add_layernorm(x: torch.Tensor, y: torch.Tensor, w: torch.Tensor, b: torch.Tensor, eps: float,
                      out_tm: torch.Tensor, out_fm: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Encoder helper (include/venom_encoder.h): out_tm = LayerNorm(x + y) token-major [T, h], and
    the same values feature-major into out_fm [h, >= T] (row stride may exceed T)."""
    T, h = x.shape
    for t in (x, y, out_tm):
        assert t.is_contiguous() and t.shape == (T, h) and t.dtype == x.dtype
    if out_fm is not None:
        assert out_fm.stride(1) == 1 and out_fm.shape[0] >= h and out_fm.shape[1] >= T  # rows >= h untouched
    _check(lib().venom_enc_add_layernorm(
        ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(w.data_ptr()),
        ctypes.c_void_p(b.data_ptr()), T, h, float(eps), _dt(x.dtype), ctypes.c_void_p(out_tm.data_ptr()),
        ctypes.c_void_p(out_fm.data_ptr() if out_fm is not None else 0),
        out_fm.stride(0) if out_fm is not None else 0, _stream(x.device)), "venom_enc_add_layernorm")
    return out_tm


def enc_heads_to_fm(a: torch.Tensor, out_fm: torch.Tensor) -> torch.Tensor:
    """Encoder helper: attention output a [B, H, S, D] (any strides, D contiguous) -> feature-major
    out_fm[h*D + d, b*S + s]."""
    B_, H_, S_, D_ = a.shape
    assert a.stride(3) == 1 and out_fm.stride(1) == 1
    _check(lib().venom_enc_heads_to_fm(
        ctypes.c_void_p(a.data_ptr()), B_, H_, S_, D_, a.stride(0), a.stride(1), a.stride(2), _dt(a.dtype),
        ctypes.c_void_p(out_fm.data_ptr()), out_fm.stride(0), _stream(a.device)), "venom_enc_heads_to_fm")
    return out_fm


def decompress(x: VNMTensor, out: Optional[torch.Tensor] = None, status: Optional[torch.Tensor] = None,
               check: bool = False) -> torch.Tensor:
    """V:N:M -> dense (inverse of Fig 3); +0.0 at every pruned position."""
    if out is None:
        out = torch.empty((x.R, x.K), dtype=x.dtype, device=x.values.device)
    assert out.stride(1) == 1
    if check and status is None:
        status = torch.zeros(1, dtype=torch.int32, device=out.device)
    st = lib().venom_decompress(ctypes.c_void_p(x.values.data_ptr()), ctypes.c_void_p(x.metadata.data_ptr()),
                                ctypes.c_void_p(x.column_idx.data_ptr()), x.R, x.K, _dt(x.dtype), x.fmt(),
                                ctypes.c_void_p(out.data_ptr()), out.stride(0),
                                ctypes.c_void_p(status.data_ptr() if status is not None else 0),
                                _stream(out.device))
    _check(st, "venom_decompress")
    if check:
        _check(int(status.item()), "venom_decompress (device status)")
    return out


def spmm(x: VNMTensor, B: torch.Tensor, bias: Optional[torch.Tensor] = None,
         out: Optional[torch.Tensor] = None, tile_t: int = 0, stages: int = 0,
         max_ctas: int = 0, strategy: int = STRATEGY_AUTO, cta_pair: int = 0,
         use_metadata_tc: bool = True, transposed_out: bool = False,
         b_kmajor: bool = False, gelu=False, group_n: int = 0,
         c_peers=None) -> torch.Tensor:
    """C = A_vnm · B (+ bias) on the sparse tensor cores.
    B: dtype[K, T] (row stride may exceed T); returns / fills C: dtype[R, T], or with
    ``transposed_out`` the token-major C^T: dtype[T, R] (row stride may exceed R). When x carries
    tensor-core-ordered metadata (order_metadata) it is used unless use_metadata_tc is False.
    ``b_kmajor``: B is token-major dtype[T, K] (read natively by M = 4 operands; transposed once into
    a scratch buffer for M > 4); with ``transposed_out`` this is
    ``F.linear(B, decompress(x))`` on PyTorch-layout activations. ``gelu``: GELU after the bias in
    the epilogue (row-major B and C): True / "erf" the erf form, "tanh" the tanh form. ``c_peers``: the fused all-gather — device addresses (or
    tensors) where the epilogue also stores C, same layout and leading dimension (tp.py)."""
    assert B.is_cuda and B.dim() == 2 and B.stride(1) == 1 and B.shape[1 if b_kmajor else 0] == x.K
    assert B.dtype == x.dtype
    T = B.shape[0 if b_kmajor else 1]
    shape = (T, x.R) if transposed_out else (x.R, T)
    if out is None:
        out = torch.empty(shape, dtype=x.dtype, device=B.device)
    assert out.stride(1) == 1 and tuple(out.shape) == shape
    if bias is not None:
        assert bias.dtype == x.dtype and bias.is_contiguous() and bias.numel() == x.R
    mtc = x.metadata_tc.data_ptr() if (use_metadata_tc and x.metadata_tc is not None) else None
    vpad = x.values_padded.data_ptr() if (mtc is not None and x.values_padded is not None) else None
    peers = None
    if c_peers:
        # fused all-gather: device addresses (ints or tensors) of the peer output slices
        addrs = [p if isinstance(p, int) else p.data_ptr() for p in c_peers]
        peers = (ctypes.c_void_p * len(addrs))(*addrs)
    scratch = None
    if b_kmajor and x.M != 4:
        # the gathered operand reads feature-major B: the library transposes B^T into this scratch
        scratch = torch.empty((x.K, T), dtype=B.dtype, device=B.device)
    if gelu not in _ACTIVATIONS:
        raise ValueError(f"gelu must be False, True / 'erf' or 'tanh', not {gelu!r}")
    opts = _Opts(tile_t, stages, max_ctas, strategy, cta_pair, mtc, 1 if transposed_out else 0,
                 1 if b_kmajor else 0, _ACTIVATIONS[gelu], group_n,
                 ctypes.cast(peers, ctypes.POINTER(ctypes.c_void_p)) if peers is not None else None,
                 len(c_peers) if c_peers else 0, vpad, scratch.data_ptr() if scratch is not None else None)
    st = lib().venom_spmm_ex(ctypes.c_void_p(x.values.data_ptr()),
                             ctypes.c_void_p(x.metadata.data_ptr() if x.metadata.numel() else 0),
                             ctypes.c_void_p(x.column_idx.data_ptr() if x.column_idx.numel() else 0),
                             x.R, x.K, x.fmt(),
                             ctypes.c_void_p(B.data_ptr()), T, B.stride(0),
                             ctypes.c_void_p(out.data_ptr()), out.stride(0),
                             ctypes.c_void_p(bias.data_ptr() if bias is not None else 0),
                             _dt(x.dtype), ctypes.byref(opts), _stream(B.device))
    _check(st, "venom_spmm")
    return out


def compress_2to4(A: torch.Tensor, V: int, M: int, status: Optional[torch.Tensor] = None,
                  check: bool = False, out=None):
    """Fused compress + V:2:4 execution form (venom_compress_2to4): returns (x, y) where x is the
    canonical V:N:M operand (== compress(A)) and y the same matrix as V:2:4 with tensor-core-ordered
    metadata (y.metadata / y.column_idx are empty: spmm does not read them)."""
    assert A.is_cuda and A.dim() == 2 and A.stride(1) == 1
    R, K = A.shape
    dev = A.device
    if out is None:
        x = VNMTensor(torch.empty((R, K // M, 2), dtype=A.dtype, device=dev),
                      torch.empty((R, (K // M + 1) // 2), dtype=torch.uint8, device=dev),
                      torch.empty((R // V, K // M, 4), dtype=torch.uint8, device=dev), R, K, V, M)
        y = VNMTensor(torch.empty((R, K // 4, 2), dtype=A.dtype, device=dev),
                      torch.empty(0, dtype=torch.uint8, device=dev), torch.empty(0, dtype=torch.uint8, device=dev),
                      R, K, V, 4, metadata_tc=torch.empty(max(metadata_tc_bytes(R, K, V, 4), 16),
                                                          dtype=torch.uint8, device=dev))
    else:
        x, y = out
    if check and status is None:
        status = torch.zeros(1, dtype=torch.int32, device=dev)
    st = lib().venom_compress_2to4(ctypes.c_void_p(A.data_ptr()), R, K, A.stride(0), _dt(A.dtype), _Format(V, 2, M),
                                   ctypes.c_void_p(x.values.data_ptr()), ctypes.c_void_p(x.metadata.data_ptr()),
                                   ctypes.c_void_p(x.column_idx.data_ptr()), ctypes.c_void_p(y.values.data_ptr()),
                                   ctypes.c_void_p(y.metadata_tc.data_ptr()),
                                   ctypes.c_void_p(status.data_ptr() if status is not None else 0), _stream(dev))
    _check(st, "venom_compress_2to4")
    if check:
        _check(int(status.item()), "venom_compress_2to4 (device status)")
    return x, y


def metadata_tc_bytes(R: int, K: int, V: int, M: int) -> int:
    n = lib().venom_metadata_tc_bytes(R, K, _Format(V, 2, M))
    if n < 0:
        raise VenomError(4, "venom_metadata_tc_bytes")
    return n


def order_metadata(x: VNMTensor, out: Optional[torch.Tensor] = None) -> VNMTensor:
    """Attach the metadata in tensor-core order (the paper's storage-order idea)
    to x, in place; spmm then loads it with TMA instead of permuting metadata on the fly."""
    n = metadata_tc_bytes(x.R, x.K, x.V, x.M)
    if out is None:
        out = x.metadata_tc if (x.metadata_tc is not None and x.metadata_tc.numel() == n) else \
            torch.empty(max(n, 16), dtype=torch.uint8, device=x.metadata.device)
    st = lib().venom_order_metadata(ctypes.c_void_p(x.metadata.data_ptr()), x.R, x.K, x.fmt(),
                                    ctypes.c_void_p(out.data_ptr()), _stream(x.metadata.device))
    _check(st, "venom_order_metadata")
    x.metadata_tc = out
    if (x.K // x.M) % 4 != 0:
        pad_values(x)  # the K' tail's other execution-form array
    return x


def pad_values(x: VNMTensor) -> VNMTensor:
    """Attach the values with rows padded to a multiple of 4 groups (include/venom.h
    venom_pad_values) to x, in place: with metadata_tc, spmm then runs any G = K/M (a K' tail)."""
    n = lib().venom_values_padded_bytes(x.R, x.K, x.fmt())
    if n < 0:
        raise VenomError(4, "venom_values_padded_bytes")
    buf = x.values_padded
    if buf is None or buf.numel() * buf.element_size() != max(n, 16):
        buf = torch.empty(max(n, 16) // 2, dtype=x.dtype, device=x.values.device)
    st = lib().venom_pad_values(ctypes.c_void_p(x.values.data_ptr()), x.R, x.K, x.fmt(),
                                ctypes.c_void_p(buf.data_ptr()), _stream(x.values.device))
    _check(st, "venom_pad_values")
    x.values_padded = buf
    return x


def expand_2to4(x: VNMTensor, out: Optional[VNMTensor] = None, status: Optional[torch.Tensor] = None,
                check: bool = False) -> VNMTensor:
    """The same matrix as V:2:4 over the original K (M % 4 == 0): the dense-K execution form."""
    R, K, V = x.R, x.K, x.V
    G2 = K // 4
    dev = x.values.device
    if out is None:
        out = VNMTensor(torch.empty((R, G2, 2), dtype=x.dtype, device=dev),
                        torch.empty((R, (G2 + 1) // 2), dtype=torch.uint8, device=dev),
                        torch.empty((R // V, G2, 4), dtype=torch.uint8, device=dev), R, K, V, 4)
    if check and status is None:
        status = torch.zeros(1, dtype=torch.int32, device=dev)
    st = lib().venom_expand_2to4(ctypes.c_void_p(x.values.data_ptr()), ctypes.c_void_p(x.metadata.data_ptr()),
                                 ctypes.c_void_p(x.column_idx.data_ptr()), R, K, _dt(x.dtype), x.fmt(),
                                 ctypes.c_void_p(out.values.data_ptr()), ctypes.c_void_p(out.metadata.data_ptr()),
                                 ctypes.c_void_p(out.column_idx.data_ptr()),
                                 ctypes.c_void_p(status.data_ptr() if status is not None else 0),
                                 _stream(dev))
    _check(st, "venom_expand_2to4")
    if check:
        _check(int(status.item()), "venom_expand_2to4 (device status)")
    return out


def prefers_2to4(R: int, K: int, T: int, V: int, M: int) -> bool:
    """Whether the library's planner runs this shape faster as the V:2:4 re-encoding (expand_2to4)
    than straight on the V:N:M operand (venom_prefer_2to4)."""
    return bool(lib().venom_prefer_2to4(R, K, T, _Format(V, 2, M)))


def version() -> str:
    return lib().venom_version().decode()
