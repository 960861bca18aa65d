// Tensor-core (tcgen05) LSTM forwards: layout of the packed TC blob.
#pragma once
#include "common.cuh"

namespace recmg {

struct TcLayout {              // byte offsets into the TC blob
    int64_t phase_off[3], phase_len[3];  // B-image groups loaded together into smem
    int64_t b_off[16];                   // B image (hi, then lo) offset within its phase
    int nb;
    int64_t pid[2];                      // folded token tables (enc, dec) [ids][256] fp32
    size_t spart_off, smem_bytes;
    size_t const_off;                    // per-unit constants in shared memory
    int64_t img64, img256, dslot;        // B image bytes (N = 64 / 256); caching decoder slot
    int64_t eslot;                       // prefetch encoder slot (Wh0 <-> Wx1)
    int64_t swap_off;                    // prefetch: DEC-B swap region (bytes in smem)
    int64_t total;
};

bool tc_supported(const recmg_model_shape *m);
TcLayout tc_layout(const recmg_model_shape *m);
int model_pack_tc(const recmg_model_shape *m, const float *raw, const float *embed_id,
                  const int64_t *offsets, void *packed_dense, void *tc_blob, cudaStream_t s);
int model_forward_tc(const recmg_model_shape *m, const void *packed_dense, const void *tc_blob,
                     const int32_t *gid, const int32_t *tid, int64_t batch, float *logits,
                     uint8_t *bits, int32_t *pf_gid, void *ws, size_t ws_bytes, cudaStream_t s,
                     long long *prof = nullptr, int64_t decode_ids = 0,
                     bool single = false, int32_t *progress = nullptr,
                     int64_t piece_chunks = 0);
int wait_progress(const int32_t *progress, int32_t target, cudaStream_t s);
size_t tc_workspace_bytes(const recmg_model_shape *m, int64_t batch);
int set_model_sm_budget(int n);
int model_sm_budget();

}  // namespace recmg
