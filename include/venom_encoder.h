/*
 * venom_encoder.h — auxiliary layout kernels for the sparse BERT encoder (
 * paper_2310_02065_b200/encoder.py). NOT part of the V:N:M method: they move activations between
 * the token-major layout attention and LayerNorm use and the feature-major layout the SpMM's B
 * operand uses (reading #14), so the encoder needs no strided torch copies.
 *
 * Conventions as in venom.h: every pointer is a DEVICE pointer owned by the caller; the library
 * never allocates and never synchronises; argument errors return synchronously and launch nothing.
 * Element type: fp16 or bf16 (venom_dtype_t); statistics in fp32.
 */
#ifndef VENOM_ENCODER_H
#define VENOM_ENCODER_H

#include "venom.h"

#ifdef __cplusplus
extern "C" {
#endif

/*
 * Residual add + LayerNorm with a dual-layout write:
 *   z[t][:] = x[t][:] + y[t][:];  out_tm[t][:] = (z - mean(z)) / sqrt(var(z) + eps) * w + b
 * and, if out_fm != NULL, the same values transposed: out_fm[f][t] (feature-major, row stride
 * ld_fm >= T). x, y, out_tm: dtype[T][h] contiguous rows; w, b: dtype[h]. h % 256 == 0, h <= 1024,
 * T % 32 == 0, ld_fm % 8 == 0 (else VENOM_ERR_INVALID_ARGUMENT). Variance is the biased one
 * (torch.nn.functional.layer_norm).
 */
venom_status_t venom_enc_add_layernorm(const void* x, const void* y, const void* w, const void* b,
                                       int64_t T, int64_t h, float eps, venom_dtype_t dt,
                                       void* out_tm, void* out_fm, int64_t ld_fm,
                                       venom_stream_t stream);

/*
 * Attention output [B][H][S][D] (strides in elements: sb, sh, ss; D contiguous) -> feature-major
 * out_fm[h*D + d][b*S + s] (row stride ld_fm >= B*S). D == 64, S % 64 == 0, ld_fm % 8 == 0.
 */
venom_status_t venom_enc_heads_to_fm(const void* a, int64_t B, int64_t H, int64_t S, int64_t D,
                                     int64_t sb, int64_t sh, int64_t ss, venom_dtype_t dt,
                                     void* out_fm, int64_t ld_fm, venom_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* VENOM_ENCODER_H */
