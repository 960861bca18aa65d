// Packed (kernel) layout of the dense model weights.  The raw input blob is
// every array of _shapes (model.py:54-80) except embed_id, row-major, in
// _shapes order.  The packed blob interleaves each LSTM layer's [Wx; Wh]
// columns gate-minor (col' = 4*j + gate, gates i,f,g,o = model.py:106-109)
// so one float4 holds the four gates of one hidden unit.
#pragma once
#include "common.cuh"

namespace recmg {

struct RawLayout {  // float offsets into the raw blob
    int64_t embed_table, att_enc, att_dec, att_v, comb_w, comb_b, head_w, head_b;
    int64_t enc_wx[4], enc_wh[4], enc_b[4], dec_wx[4], dec_wh[4], dec_b[4];
    int64_t slot_embed, total;
};

struct PackedLayout {  // float offsets into the packed blob (16 B aligned)
    int64_t enc_w[4], enc_b[4], dec_w[4], dec_b[4];  // [Kin+d][4d], [4d]
    int64_t att_enc, att_dec, att_v, comb_w, comb_b, head_w, head_b, slot_embed, embed_table;
    int64_t slot_proj;  // prefetch: slot_embed[t] @ dec0_wx[0:2d] + dec0_b, [l_out][4d] interleaved
    int64_t total;
};

constexpr int kMaxStacks = 4;

inline bool shape_ok(const recmg_model_shape *m) {
    return m && (m->kind == RECMG_MODEL_CACHING || m->kind == RECMG_MODEL_PREFETCH) && m->dim >= 1 &&
           m->dim <= 128 && m->stacks >= 1 && m->stacks <= kMaxStacks && m->l_in >= 1 &&
           m->l_in <= 32 && m->l_out >= 1 && m->l_out <= 32 && m->n_tables >= 1 &&
           m->total_ids >= 1 && m->total_ids < (int64_t)kGidMask;
}

inline RawLayout raw_layout(const recmg_model_shape *m) {
    const int64_t d = m->dim;
    RawLayout r{};
    int64_t o = 0;
    r.embed_table = o; o += m->n_tables * d;
    r.att_enc = o; o += d * d;
    r.att_dec = o; o += d * d;
    r.att_v = o; o += d;
    r.comb_w = o; o += 2 * d * d;
    r.comb_b = o; o += d;
    r.head_w = o; o += d;
    r.head_b = o; o += 1;
    for (int k = 0; k < m->stacks; k++) {
        const int64_t ein = k == 0 ? 2 * d : d, din = k == 0 ? 3 * d : d;
        r.enc_wx[k] = o; o += ein * 4 * d;
        r.enc_wh[k] = o; o += d * 4 * d;
        r.enc_b[k] = o; o += 4 * d;
        r.dec_wx[k] = o; o += din * 4 * d;
        r.dec_wh[k] = o; o += d * 4 * d;
        r.dec_b[k] = o; o += 4 * d;
    }
    r.slot_embed = o;
    if (m->kind == RECMG_MODEL_PREFETCH) o += (int64_t)m->l_out * 2 * d;
    r.total = o;
    return r;
}

inline PackedLayout packed_layout(const recmg_model_shape *m) {
    const int64_t d = m->dim;
    PackedLayout p{};
    int64_t o = 0;
    auto take = [&](int64_t n) { int64_t r = o; o += (n + 3) / 4 * 4; return r; };
    for (int k = 0; k < m->stacks; k++) {
        const int64_t ein = k == 0 ? 2 * d : d, din = k == 0 ? 3 * d : d;
        p.enc_w[k] = take((ein + d) * 4 * d);
        p.enc_b[k] = take(4 * d);
        p.dec_w[k] = take((din + d) * 4 * d);
        p.dec_b[k] = take(4 * d);
    }
    p.att_enc = take(d * d);
    p.att_dec = take(d * d);
    p.att_v = take(d);
    p.comb_w = take(2 * d * d);
    p.comb_b = take(d);
    p.head_w = take(d);
    p.head_b = take(1);
    p.slot_embed = take(m->kind == RECMG_MODEL_PREFETCH ? (int64_t)m->l_out * 2 * d : 0);
    p.slot_proj = take(m->kind == RECMG_MODEL_PREFETCH ? (int64_t)m->l_out * 4 * d : 0);
    p.embed_table = take(m->n_tables * d);
    p.total = o;
    return p;
}

}  // namespace recmg
