// Model forward entry points (see lstm_simt.cu).
#pragma once
#include "common.cuh"

namespace recmg {
size_t fwd_fp32_smem_bytes(const recmg_model_shape *m);
int model_pack(const recmg_model_shape *m, const float *raw, void *packed, cudaStream_t s);
int model_forward_fp32(const recmg_model_shape *m, const float *embed_id, const void *packed,
                       const int32_t *gid, const int32_t *tid, int64_t batch, float *logits,
                       uint8_t *bits, int32_t *pf_gid, cudaStream_t s,
                       int64_t decode_ids = 0);
}  // namespace recmg
