"""One tiny call of every kernel family and SpMM instantiation, for compute-sanitizer
(memcheck / racecheck / synccheck): python tools/sanitize.py. Checks results loosely against
torch on the decompressed operand so a silent corruption also fails."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2310_02065_b200 as venom  # noqa: E402


def check(C, A_dense, B, bias=None, tol=2e-2, transposed=False, bk=False, gelu=False):
    ref = A_dense.float() @ (B.float().t() if bk else B.float())
    if bias is not None:
        ref += bias.float()[:, None]
    if gelu:
        ref = torch.nn.functional.gelu(ref)
    got = C.float().t() if transposed else C.float()
    err = (got - ref).norm() / ref.norm().clamp_min(1e-30)
    assert err < tol, float(err)


def main():
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(1)
    cases = [  # R, K, T, V, M
        (256, 512, 256, 128, 16), (256, 512, 128, 64, 8), (128, 512, 64, 32, 16), (512, 512, 256, 256, 16),
        (256, 512, 256, 128, 4), (512, 1024, 480, 128, 4), (128, 640, 64, 64, 10)]
    for (R, K, T, V, M) in cases:
        A = (torch.randn(R, K, generator=g, device=dev) * 0.02).half()
        B = torch.randn(K, T, generator=g, device=dev).half()
        bias = torch.randn(R, generator=g, device=dev).half()
        x = venom.compress(A, V=V, M=M, check=True)
        D = venom.decompress(x, check=True)
        for use_tc in (False, True):
            if use_tc:
                venom.order_metadata(x)
            check(venom.spmm(x, B, bias=bias, use_metadata_tc=use_tc), D, B, bias)
        check(venom.spmm(x, B, transposed_out=True), D, B, transposed=True)
        check(venom.spmm(x, B, bias=bias, gelu=True), D, B, bias, gelu=True)
        for pair in (1, 2):
            try:
                check(venom.spmm(x, B, cta_pair=pair), D, B)
            except venom.VenomError:
                pass  # not available for this V
        if M in (4, 8, 16, 32):
            for pair in (1, 2):
                check(venom.spmm(x, B, strategy=venom.STRATEGY_DENSE_K, cta_pair=pair), D, B)
        if M == 4:
            Bt = B.t().contiguous()
            check(venom.spmm(x, Bt, b_kmajor=True), D, Bt, bk=True)
            if T % 240 == 0 or T >= 240:
                check(venom.spmm(x, B, tile_t=240), D, B)
        if M % 8 == 0 and 128 % M == 0 and V % 16 == 0:
            x2, y = venom.compress_2to4(A, V=V, M=M, check=True)
            check(venom.spmm(y, B, bias=bias), D, B, bias)
        if M % 4 == 0:
            venom.expand_2to4(x, check=True)
    # round 2b: the K' tail (G = 33: padded values + metadata_tc), V = 64 tile 64 (M64), the
    # fused all-gather fan-out (row-major and token-major C through the TMA-store epilogue)
    A = (torch.randn(128, 330, generator=g, device=dev) * 0.02).half()
    B = torch.randn(330, 64, generator=g, device=dev).half()
    x = venom.order_metadata(venom.compress(A, V=64, M=10, check=True))
    D = venom.decompress(x, check=True)
    check(venom.spmm(x, B), D, B)
    check(venom.spmm(x, B, transposed_out=True), D, B, transposed=True)
    A = (torch.randn(192, 640, generator=g, device=dev) * 0.02).half()
    B = torch.randn(640, 136, generator=g, device=dev).half()
    x = venom.order_metadata(venom.compress(A, V=64, M=8, check=True))
    D = venom.decompress(x, check=True)
    check(venom.spmm(x, B, tile_t=64), D, B)
    for ct in (False, True):
        shape = (136, 192) if ct else (192, 136)
        peers = [torch.empty(shape, dtype=torch.float16, device=dev) for _ in range(2)]
        C = venom.spmm(x, B, transposed_out=ct, c_peers=peers)
        check(C, D, B, transposed=ct)
        assert all(torch.equal(q, C) for q in peers)
    # compressor routes: streaming kernel (tall blocks), tile kernel (lda not 16-byte pitched)
    A = (torch.randn(512, 1024, generator=g, device=dev) * 0.02).half()
    venom.compress(A, V=256, M=128, check=True)
    Ab = torch.randn(256, 1030, generator=g, device=dev).half()[:, :1020]
    venom.compress(Ab, V=64, M=10, check=True)
    torch.cuda.synchronize()
    print("sanitize driver: all calls ok")


if __name__ == "__main__":
    main()
