// K1 / K2: fp32 forward of the caching model (1 LSTM stack, causal attention,
// l_in outputs) and the prefetch model (2 stacks, l_out slot queries) over a
// tile of MC chunks per CTA.  Exact-fp32 path: fp32 storage, fp32 FMA,
// accurate tanhf/expf.  Reference: model.py:103-212 (see per-block cites).
//
// Per CTA, everything a chunk needs lives in shared memory:
//   Hs[d][L*MC]   encoder top-layer states (model.py:144)       j-major so a
//   Ep[d][L*MC]   enc_pre = Hs @ att_enc   (model.py:160)        warp reads
//                                                                 consecutive
//   A[K][MC]      GEMM operand (concat of inputs, k-major)       (pos,chunk)
//   h,c[stack][d][MC], q[d][MC], ctx[d][MC], comb[d][MC], probs.
// Gate GEMMs: thread item = (hidden unit j, 4 chunks); one float4 of the
// gate-interleaved weights x one float4 of A per k -> 16 FMA.
#include "lstm.cuh"
#include "model_layout.cuh"

namespace recmg {

constexpr int kMC = 16;        // chunks per CTA
constexpr int kThreads = 256;

struct FwdArgs {
    recmg_model_shape m;
    PackedLayout pl;
    const float *embed_id;
    const float *w;        // packed blob
    const int32_t *gid, *tid;
    int64_t batch;
    float *logits;
    uint8_t *bits;
    int32_t *pf_gid;
};

__device__ __forceinline__ float sigm(float x) { return 1.0f / (1.0f + expf(-x)); }

// One LSTM step for all MC chunks of the tile (model.py:103-112).
// A[K][MC] (smem), W [K][d] float4 (global, gate-interleaved), bias [d] float4.
__device__ __forceinline__ void lstm_cell_step(const float *__restrict__ A, int K,
                                               const float4 *__restrict__ W,
                                               const float4 *__restrict__ bias, float *c,
                                               float *h, int d) {
    const int items = d * (kMC / 4);
    for (int it = threadIdx.x; it < items; it += kThreads) {
        const int j = it % d, cg = it / d;
        const float4 b = __ldg(bias + j);
        float4 acc[4];
#pragma unroll
        for (int r = 0; r < 4; r++) acc[r] = b;
        const float *a = A + cg * 4;
#pragma unroll 4
        for (int k = 0; k < K; k++) {
            const float4 wv = __ldg(W + (int64_t)k * d + j);
            const float4 av = *reinterpret_cast<const float4 *>(a + k * kMC);
            acc[0].x += av.x * wv.x; acc[0].y += av.x * wv.y; acc[0].z += av.x * wv.z; acc[0].w += av.x * wv.w;
            acc[1].x += av.y * wv.x; acc[1].y += av.y * wv.y; acc[1].z += av.y * wv.z; acc[1].w += av.y * wv.w;
            acc[2].x += av.z * wv.x; acc[2].y += av.z * wv.y; acc[2].z += av.z * wv.z; acc[2].w += av.z * wv.w;
            acc[3].x += av.w * wv.x; acc[3].y += av.w * wv.y; acc[3].z += av.w * wv.z; acc[3].w += av.w * wv.w;
        }
#pragma unroll
        for (int r = 0; r < 4; r++) {
            const int ch = cg * 4 + r;
            const float ig = sigm(acc[r].x), fg = sigm(acc[r].y);
            const float gg = tanhf(acc[r].z), og = sigm(acc[r].w);
            const float cn = fg * c[j * kMC + ch] + ig * gg;
            c[j * kMC + ch] = cn;
            h[j * kMC + ch] = og * tanhf(cn);
        }
    }
}

// out[j][MC] = act( sum_k A[k][MC] * Wm[k][j] + b[j] ), plain row-major W [K][d]
template <bool TANH>
__device__ __forceinline__ void dense_step(const float *__restrict__ A, int K,
                                           const float *__restrict__ Wm,
                                           const float *__restrict__ b, float *out, int d) {
    const int items = d * (kMC / 4);
    for (int it = threadIdx.x; it < items; it += kThreads) {
        const int j = it % d, cg = it / d;
        const float bj = b ? __ldg(b + j) : 0.0f;
        float acc0 = bj, acc1 = bj, acc2 = bj, acc3 = bj;
        const float *a = A + cg * 4;
#pragma unroll 4
        for (int k = 0; k < K; k++) {
            const float wv = __ldg(Wm + (int64_t)k * d + j);
            const float4 av = *reinterpret_cast<const float4 *>(a + k * kMC);
            acc0 += av.x * wv; acc1 += av.y * wv; acc2 += av.z * wv; acc3 += av.w * wv;
        }
        if (TANH) { acc0 = tanhf(acc0); acc1 = tanhf(acc1); acc2 = tanhf(acc2); acc3 = tanhf(acc3); }
        *reinterpret_cast<float4 *>(out + j * kMC + cg * 4) = make_float4(acc0, acc1, acc2, acc3);
    }
}

__global__ void __launch_bounds__(kThreads)
lstm_fwd_fp32_kernel(FwdArgs a) {
    extern __shared__ __align__(16) float sm[];
    const int d = a.m.dim, L = a.m.l_in, stacks = a.m.stacks;
    const bool caching = a.m.kind == RECMG_MODEL_CACHING;
    const int T = caching ? L : a.m.l_out;
    const int LM = L * kMC;
    const int64_t c0 = (int64_t)blockIdx.x * kMC;
    const int tid = threadIdx.x;
    const PackedLayout &pl = a.pl;
    const float *w = a.w;

    float *Hs = sm;                       // [d][L*MC]
    float *Ep = Hs + d * LM;              // [d][L*MC]
    float *A = Ep + d * LM;               // [4d][MC]
    float *hst = A + 4 * d * kMC;         // [stacks][d][MC]
    float *cst = hst + stacks * d * kMC;  // [stacks][d][MC]
    float *q = cst + stacks * d * kMC;    // [d][MC]
    float *ctx = q + d * kMC;             // [d][MC]
    float *comb = ctx + d * kMC;          // [d][MC]
    float *sc = comb + d * kMC;           // [L][MC] scores / attention weights
    int32_t *gsm = (int32_t *)(sc + L * kMC);  // [L][MC] gid
    int32_t *tsm = gsm + L * kMC;              // [L][MC] tid

    // chunk ids (pad rows beyond batch with id 0; their outputs are dropped)
    for (int i = tid; i < LM; i += kThreads) {
        const int t = i / kMC, ch = i % kMC;
        const int64_t row = c0 + ch;
        gsm[i] = row < a.batch ? a.gid[row * L + t] : 0;
        tsm[i] = row < a.batch ? a.tid[row * L + t] : 0;
    }
    for (int i = tid; i < 2 * stacks * d * kMC; i += kThreads) hst[i] = 0.0f;  // h and c = 0 (model.py:134-136)
    __syncthreads();

    // token of step t into A rows [0, 2d): [E_id[gid]; E_tab[tid]]  (model.py:148-153)
    auto load_token = [&](int t) {
        const float *etab = w + pl.embed_table;
        for (int i = tid; i < 2 * d * kMC; i += kThreads) {
            const int k = i / kMC, ch = i % kMC;
            const int g = gsm[t * kMC + ch], tb = tsm[t * kMC + ch];
            A[i] = k < d ? __ldg(a.embed_id + (int64_t)g * d + k) : __ldg(etab + (int64_t)tb * d + (k - d));
        }
    };
    auto copy_rows = [&](float *dst, const float *src, int rows) {
        for (int i = tid; i < rows * kMC; i += kThreads) dst[i] = src[i];
    };

    // ---------------- encoder  (model.py:131-145) ----------------
    for (int t = 0; t < L; t++) {
        for (int k = 0; k < stacks; k++) {
            const int in = (k == 0) ? 2 * d : d;
            if (k == 0) load_token(t);
            else copy_rows(A, hst + (k - 1) * d * kMC, d);
            copy_rows(A + in * kMC, hst + k * d * kMC, d);
            __syncthreads();
            lstm_cell_step(A, in + d, (const float4 *)(w + pl.enc_w[k]),
                           (const float4 *)(w + pl.enc_b[k]), cst + k * d * kMC, hst + k * d * kMC, d);
            __syncthreads();
        }
        // top-layer state -> Hs[:, t]
        const float *ht = hst + (stacks - 1) * d * kMC;
        for (int i = tid; i < d * kMC; i += kThreads) {
            const int j = i / kMC, ch = i % kMC;
            Hs[j * LM + t * kMC + ch] = ht[i];
        }
        __syncthreads();
    }
    // enc_pre = Hs @ att_enc  (model.py:159-160): items (j, 4 columns of L*MC)
    {
        const float *Wa = w + pl.att_enc;
        const int cols4 = LM / 4;
        for (int it = tid; it < d * cols4; it += kThreads) {
            const int j = it % d, c4 = it / d;
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int k = 0; k < d; k++) {
                const float wv = __ldg(Wa + k * d + j);
                const float4 hv = *reinterpret_cast<const float4 *>(Hs + k * LM + c4 * 4);
                acc.x += hv.x * wv; acc.y += hv.y * wv; acc.z += hv.z * wv; acc.w += hv.w * wv;
            }
            *reinterpret_cast<float4 *>(Ep + j * LM + c4 * 4) = acc;
        }
    }
    // decoder state restarts at zero (model.py:161-163)
    for (int i = tid; i < 2 * stacks * d * kMC; i += kThreads) hst[i] = 0.0f;
    __syncthreads();

    // ---------------- decoder  (model.py:156-181) ----------------
    const float *hv_att = w + pl.att_v;
    for (int t = 0; t < T; t++) {
        const float *htop = hst + (stacks - 1) * d * kMC;
        // query = h_top(t-1) @ att_dec  (model.py:118)
        dense_step<false>(htop, d, w + pl.att_dec, nullptr, q, d);
        __syncthreads();
        // scores_j = v . tanh(enc_pre_j + q), causal mask j > t  (model.py:119-121,166-169)
        const int npos = caching ? (t + 1) : L;
        for (int i = tid; i < L * kMC; i += kThreads) {
            const int pos = i / kMC, ch = i % kMC;
            float s = -INFINITY;
            if (pos < npos) {
                s = 0.0f;
                for (int j = 0; j < d; j++)
                    s += tanhf(Ep[j * LM + i] + q[j * kMC + ch]) * __ldg(hv_att + j);
            }
            sc[i] = s;
        }
        __syncthreads();
        // softmax over positions (autodiff.py:226-236)
        for (int ch = tid; ch < kMC; ch += kThreads) {
            float mx = -INFINITY;
            for (int pos = 0; pos < npos; pos++) mx = fmaxf(mx, sc[pos * kMC + ch]);
            float sum = 0.0f;
            for (int pos = 0; pos < npos; pos++) {
                const float e = expf(sc[pos * kMC + ch] - mx);
                sc[pos * kMC + ch] = e;
                sum += e;
            }
            const float inv = 1.0f / sum;
            for (int pos = 0; pos < L; pos++) sc[pos * kMC + ch] = pos < npos ? sc[pos * kMC + ch] * inv : 0.0f;
        }
        __syncthreads();
        // context = sum_j a_j H_j  (model.py:123)
        for (int i = tid; i < d * kMC; i += kThreads) {
            const int j = i / kMC, ch = i % kMC;
            float s = 0.0f;
            for (int pos = 0; pos < npos; pos++) s += sc[pos * kMC + ch] * Hs[j * LM + pos * kMC + ch];
            ctx[i] = s;
        }
        __syncthreads();
        // decoder LSTM stack: layer 0 input [x_t ; ctx] (model.py:172-176)
        for (int k = 0; k < stacks; k++) {
            int K;
            const float4 *W, *B;
            if (k == 0) {
                if (caching) {
                    load_token(t);
                    copy_rows(A + 2 * d * kMC, ctx, d);
                    copy_rows(A + 3 * d * kMC, hst, d);
                    K = 4 * d;
                    W = (const float4 *)(w + pl.dec_w[0]);
                    B = (const float4 *)(w + pl.dec_b[0]);
                } else {
                    // slot part folded into slot_proj at pack time (model.py:208-209)
                    copy_rows(A, ctx, d);
                    copy_rows(A + d * kMC, hst, d);
                    K = 2 * d;
                    W = (const float4 *)(w + pl.dec_w[0]) + (int64_t)2 * d * d;
                    B = (const float4 *)(w + pl.slot_proj) + (int64_t)t * d;
                }
            } else {
                copy_rows(A, hst + (k - 1) * d * kMC, d);
                copy_rows(A + d * kMC, hst + k * d * kMC, d);
                K = 2 * d;
                W = (const float4 *)(w + pl.dec_w[k]);
                B = (const float4 *)(w + pl.dec_b[k]);
            }
            __syncthreads();
            lstm_cell_step(A, K, W, B, cst + k * d * kMC, hst + k * d * kMC, d);
            __syncthreads();
        }
        // combined = tanh([h_top ; ctx] @ comb_w + comb_b)  (model.py:177-178)
        copy_rows(A, htop, d);
        copy_rows(A + d * kMC, ctx, d);
        __syncthreads();
        dense_step<true>(A, 2 * d, w + pl.comb_w, w + pl.comb_b, comb, d);
        __syncthreads();
        // logit = combined @ head_w + head_b  (model.py:179, pre-sigmoid)
        for (int ch = tid; ch < kMC; ch += kThreads) {
            float s = __ldg(w + pl.head_b);
            for (int j = 0; j < d; j++) s += comb[j * kMC + ch] * __ldg(w + pl.head_w + j);
            const int64_t row = c0 + ch;
            if (row < a.batch) {
                a.logits[row * T + t] = s;
                if (caching && a.bits) a.bits[row * T + t] = s >= 0.0f ? 1 : 0;  // runtime.py:192
                if (!caching && a.pf_gid) {
                    // decode_indices in float64 (model.py:250-258)
                    const double po = 1.0 / (1.0 + exp(-(double)s));
                    const int64_t V = a.m.total_ids;
                    double gg = floor(po * (double)(V - 1) + 0.5);
                    gg = fmin(fmax(gg, 0.0), (double)(V - 1));
                    a.pf_gid[row * T + t] = (int32_t)gg;
                }
            }
        }
        __syncthreads();
    }
}

size_t fwd_fp32_smem_bytes(const recmg_model_shape *m) {
    const size_t d = m->dim, L = m->l_in, st = m->stacks;
    size_t floats = 2 * d * L * kMC + 4 * d * kMC + 2 * st * d * kMC + 3 * d * kMC + L * kMC;
    return floats * 4 + 2 * L * kMC * 4;
}

// ---------------------------------------------------------------------------
// packing: raw _shapes blob -> packed layout
__global__ void pack_kernel(recmg_model_shape m, RawLayout r, PackedLayout p, const float *raw,
                            float *out) {
    const int64_t d = m.dim;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    auto inter = [&](int64_t dst, int64_t wx, int64_t wh, int64_t kin, int64_t bsrc, int64_t bdst) {
        const int64_t rows = kin + d, cols = 4 * d;
        for (int64_t i = tid; i < rows * cols; i += stride) {
            const int64_t k = i / cols, c = i % cols;  // c = 4*j + gate
            const int64_t j = c / 4, gate = c % 4;
            out[dst + i] = k < kin ? raw[wx + k * 4 * d + gate * d + j]
                                   : raw[wh + (k - kin) * 4 * d + gate * d + j];
        }
        for (int64_t i = tid; i < 4 * d; i += stride) out[bdst + i] = raw[bsrc + (i % 4) * d + i / 4];
    };
    for (int k = 0; k < m.stacks; k++) {
        inter(p.enc_w[k], r.enc_wx[k], r.enc_wh[k], k == 0 ? 2 * d : d, r.enc_b[k], p.enc_b[k]);
        inter(p.dec_w[k], r.dec_wx[k], r.dec_wh[k], k == 0 ? 3 * d : d, r.dec_b[k], p.dec_b[k]);
    }
    auto copy = [&](int64_t dst, int64_t src, int64_t nfl) {
        for (int64_t i = tid; i < nfl; i += stride) out[dst + i] = raw[src + i];
    };
    copy(p.att_enc, r.att_enc, d * d);
    copy(p.att_dec, r.att_dec, d * d);
    copy(p.att_v, r.att_v, d);
    copy(p.comb_w, r.comb_w, 2 * d * d);
    copy(p.comb_b, r.comb_b, d);
    copy(p.head_w, r.head_w, d);
    copy(p.head_b, r.head_b, 1);
    copy(p.embed_table, r.embed_table, (int64_t)m.n_tables * d);
    if (m.kind == RECMG_MODEL_PREFETCH) {
        copy(p.slot_embed, r.slot_embed, (int64_t)m.l_out * 2 * d);
        // slot_proj[t][4j+gate] = dec0_b + slot_embed[t] @ dec0_wx[0:2d]  (model.py:208-209)
        for (int64_t i = tid; i < (int64_t)m.l_out * 4 * d; i += stride) {
            const int64_t t = i / (4 * d), c = i % (4 * d), j = c / 4, gate = c % 4;
            float s = raw[r.dec_b[0] + gate * d + j];
            for (int64_t k = 0; k < 2 * d; k++)
                s += raw[r.slot_embed + t * 2 * d + k] * raw[r.dec_wx[0] + k * 4 * d + gate * d + j];
            out[p.slot_proj + i] = s;
        }
    }
}

int model_pack(const recmg_model_shape *m, const float *raw, void *packed, cudaStream_t s) {
    RawLayout r = raw_layout(m);
    PackedLayout p = packed_layout(m);
    RECMG_CUDA_TRY(cudaMemsetAsync(packed, 0, p.total * sizeof(float), s));
    pack_kernel<<<2 * kSmCount, 256, 0, s>>>(*m, r, p, raw, (float *)packed);
    RECMG_LAUNCH_CHECK();
    return RECMG_OK;
}

int model_forward_fp32(const recmg_model_shape *m, const float *embed_id, const void *packed,
                       const int32_t *gid, const int32_t *tid, int64_t batch, float *logits,
                       uint8_t *bits, int32_t *pf_gid, cudaStream_t s, int64_t decode_ids) {
    if (batch <= 0) return RECMG_OK;
    FwdArgs a;
    a.m = *m;
    a.pl = packed_layout(m);
    if (decode_ids > 0) a.m.total_ids = decode_ids;   // decode scale only (table shards)
    a.embed_id = embed_id;
    a.w = (const float *)packed;
    a.gid = gid;
    a.tid = tid;
    a.batch = batch;
    a.logits = logits;
    a.bits = bits;
    a.pf_gid = pf_gid;
    const size_t smem = fwd_fp32_smem_bytes(m);
    if (smem > 227 * 1024) return RECMG_E_INVALID_CONFIG;
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        RECMG_CUDA_TRY(cudaFuncSetAttribute(lstm_fwd_fp32_kernel,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = smem;
    }
    const int64_t grid = (batch + kMC - 1) / kMC;
    lstm_fwd_fp32_kernel<<<(unsigned)grid, kThreads, smem, s>>>(a);
    RECMG_LAUNCH_CHECK();
    return RECMG_OK;
}

}  // namespace recmg
