// K1 / K2 on the 5th-gen tensor cores: fp32-parity LSTM + attention forwards
// with every GEMM on tcgen05 (kind::f16, fp32 accumulation in TMEM).
//
// Precision: each GEMM is the 3-product split x*w ~= xh*wh + xh*wl + xl*wh
// with xh = fp16(x), xl = fp16(x - xh) (same for w), accumulated in fp32;
// that is ~22 significant bits per product, i.e. fp32-class logits (the
// 1e-3 parity bar; tests/test_gpu_model.py).  Elementwise math stays fp32.
//
// Tile = 128 chunks = 128 TMEM lanes; 512 threads: warp w serves TMEM lane
// quadrant (w & 3) and hidden units [16*(w>>2), +16), so every chunk row is
// owned by four threads.  TMEM (512 columns):
//   [0,256)   Z   gate pre-activations, gate-interleaved (col 4j+g)
//   [256,320) Q   attention query / enc_pre of the previous step
//   [320,384) C   comb accumulator (caching) / h1 operand (prefetch)
//   [384,512) A   fp16 hi|lo operands (h, ctx / h0, ctx)
// Weights live in shared memory as fp16 hi/lo B images in the no-swizzle
// K-major core-matrix layout (umma.cuh), loaded per phase.  The layer-0
// token projection x_t @ Wx + b is folded into per-id tables at pack time
// (Pid = E_id @ Wx[:d], Ptab = E_tab @ Wx[d:2d] + b), so z starts as
// Pid[gid] + Ptab[tid] written into Z with tcgen05.st.
// Encoder states H_t and enc_pre_t = H_t @ att_enc go to a per-CTA L2
// scratch for the attention of every decoder step (model.py:115-124).
#include <vector>

#include "lstm.cuh"
#include "lstm_tc.cuh"
#include "model_layout.cuh"
#include "umma.cuh"

namespace recmg {

namespace {

constexpr uint32_t COL_Z = 0, COL_Q = 256, COL_C = 320, COL_A = 384;
// A operand sub-regions (32 columns = 64 fp16 each)
constexpr uint32_t A_H_HI = COL_A + 0, A_H_LO = COL_A + 32, A_X_HI = COL_A + 64,
                   A_X_LO = COL_A + 96;                  // caching: h, ctx
constexpr uint32_t P_H0_HI = COL_A + 0, P_H0_LO = COL_A + 32, P_CTX_HI = COL_A + 64,
                   P_CTX_LO = COL_A + 96, P_H1_HI = COL_C, P_H1_LO = COL_C + 32;  // prefetch

// threads per chunk row: 4 (512 threads, 16 hidden units each) for both
// models -- measured; with the smaller shared-memory layouts the caching model
// also gains from the 16 warps (2 threads per row were best at 191 KB)
template <int KIND> struct PartsOf { static constexpr int value = 4; };

__device__ __forceinline__ float ftanh(float x) {
    return 1.0f - __fdividef(2.0f, 1.0f + __expf(2.0f * x));
}

// The epilogues are bound by the SFU (MUFU: ex2 + rcp per sigmoid/tanh at
// 16 lanes/clk/SM).  rcp4 replaces four reciprocals of denominators d >= 1 by
// one MUFU.RCP and nine FMULs; clamping each d at 2^31 keeps the product of
// four finite and changes 1/d by < 5e-10 absolute.
__device__ __forceinline__ float frcp(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
constexpr float kDenMax = 2147483648.0f;
__device__ __forceinline__ void rcp4(float &a, float &b, float &c, float &d) {
    a = fminf(a, kDenMax); b = fminf(b, kDenMax); c = fminf(c, kDenMax); d = fminf(d, kDenMax);
    const float ab = a * b, cd = c * d;
    const float r = frcp(ab * cd);
    const float rab = r * cd, rcd = r * ab;
    const float ia = rab * b, ib = rab * a, ic = rcd * d, id = rcd * c;
    a = ia; b = ib; c = ic; d = id;
}
// 1 / (1 + e^(-x)) and tanh = 1 - 2 / (1 + e^(2x)) denominators
__device__ __forceinline__ float sig_den(float x) { return 1.0f + __expf(-x); }
__device__ __forceinline__ float tanh_den(float x) { return 1.0f + __expf(2.0f * x); }
// The gate pre-activations arrive pre-scaled (packing multiplies every gate
// column of the LSTM weights, folded token tables, layer-1 biases and slot
// projections by gate_scale): z' = -log2(e) z for i, f, o and 2 log2(e) z for
// g, so each gate's denominator is one MUFU.EX2 with no FMUL in front.
constexpr float kLog2e = 1.4426950408889634f;
__host__ __device__ __forceinline__ float gate_scale(int g) {
    return g == 2 ? 2.0f * kLog2e : -kLog2e;
}
__device__ __forceinline__ float ex2f(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float ex2_den(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return 1.0f + r;
}

// Attention scores tanh(e + q) (model.py:118) use e^(2(e+q)) = e^(2e) e^(2q):
// the encoder stores X = e^(2e) once per position, each decoder step
// computes e^(2q) once, and every (position, unit) pair costs one FFMA and a
// quarter MUFU.RCP instead of ex2 + rcp.  Exponents beyond +-kExpLim fall
// back to the direct form (raw e kept for that position / q out of range).
// kExpLim = 11 bounds each denominator by 1 + e^22 < 2^32, so the product
// of four stays finite and score_fast needs no clamps (|e|, |q| < 4.5 at init
// 0.4 / 0.6; at init 1.0 about 5% of positions take the direct form).
constexpr float kExpLim = 11.0f;

struct TcArgs {
    recmg_model_shape m;
    TcLayout tl;
    PackedLayout pl;
    const uint8_t *blob;   // TC blob (B images + folded tables)
    const float *dense;    // fp32 packed blob (biases, att_v, comb, head, slot_proj)
    const int32_t *gid, *tid;
    int64_t batch;
    float *logits;
    uint8_t *bits;
    int32_t *pf_gid;
    float *scratch;        // [gridDim.x][2][L][8][128] 32-byte pairs (scratch_at)
    int *tile_counter;     // dynamic tile scheduler (zeroed before the launch)
    int *progress;         // nullable: finished tiles per piece (piece = tile / piece_tiles)
    int64_t piece_tiles;
    long long *prof;       // PROF builds: per-CTA cycles per phase [grid][16]
};

// Phase cycle accounting (thread 0's timeline = the CTA's critical path);
// compiled only into the diagnostic recmg_model_forward_profile variant.
template <bool PROF>
struct PhaseClock {
    long long acc[16];
    long long last;
    int cur;
    __device__ __forceinline__ void start() {
        if constexpr (PROF) {
#pragma unroll
            for (int i = 0; i < 16; i++) acc[i] = 0;
            last = clock64();
            cur = 15;
        }
    }
    __device__ __forceinline__ void mark(int next) {
        if constexpr (PROF) {
            const long long t = clock64();
#pragma unroll
            for (int i = 0; i < 16; i++)
                if (i == cur) acc[i] += t - last;
            last = t;
            cur = next;
        }
    }
    __device__ __forceinline__ void flush(long long *out) {
        if constexpr (PROF) {
            mark(15);
#pragma unroll
            for (int i = 0; i < 16; i++) out[i] = acc[i];
        }
    }
};

// ---- per-thread helpers ------------------------------------------------------
// Unit ownership: the gate product Z is issued as two N = 128 halves (units
// 0-31, then 32-63) with their own commits, and every thread owns HU units of
// EACH half -- part p holds units [HU p, HU p + HU) and [32 + HU p, 32 + HU p + HU)
// -- so all warps start their cell on the first half while the tensor pipe
// still runs the second.  Local unit k < HU is in half 0, k >= HU in half 1.
template <int PARTS>
struct Ctx {
    static constexpr int U = 64 / PARTS;       // hidden units per thread
    static constexpr int HU = U / 2;           // units per Z half
    static constexpr int NQ = U / 4;           // float4 per scratch position
    static constexpr int NT = 128 * PARTS;     // threads
    int tid, warp, lane, quad, part, row;
    uint32_t tbase, lane_addr;  // tmem base, + lane quadrant
    // global hidden unit of local unit k
    __device__ __forceinline__ int unit(int k) const {
        return (k < HU ? 0 : 32 - HU) + HU * part + k;
    }
    // Z column (gate-interleaved, 4 per unit) of the first gate of local unit k
    __device__ __forceinline__ uint32_t zcol(int k) const { return 4u * (uint32_t)unit(k); }
};

// all threads: copy a phase's B images (bytes [off, off+len) of the blob) to smem
template <int NT>
__device__ __forceinline__ void load_phase(uint8_t *smem, const uint8_t *blob, int64_t off,
                                           int64_t len, int tid) {
    const int4 *src = reinterpret_cast<const int4 *>(blob + off);
    int4 *dst = reinterpret_cast<int4 *>(smem);
    for (int64_t i = tid; i < len / 16; i += NT) dst[i] = __ldg(src + i);
    umma::fence_proxy_async();
    __syncthreads();
}

// the same with one TMA bulk copy stream (thread 0 issues, everyone waits on
// the byte-counting barrier): no register round trip per 16 B
__device__ __forceinline__ void load_phase_tma(uint8_t *smem, const uint8_t *blob, int64_t off,
                                               int64_t len, int tid, uint64_t *bar,
                                               uint32_t &ph) {
    umma::fence_proxy_async();   // order this thread's generic smem writes (s_part) before the TMA
    __syncthreads();             // every reader of the old contents is done
    if (tid == 0) {
        umma::mbar_expect_tx(bar, (uint32_t)len);
        for (int64_t o = 0; o < len; o += 32768)
            umma::bulk_g2s(smem + o, blob + off + o, (uint32_t)imin64(32768, len - o), bar);
    }
    umma::mbar_wait(bar, ph);
    ph ^= 1u;
}

// thread 0: TMA-copy `len` bytes of the blob at `off` to smem `dst`, arriving on bar
// (the caller arms the barrier with the total of all pieces first)
__device__ __forceinline__ void tma_piece(uint8_t *dst, const uint8_t *blob, int64_t off,
                                          int64_t len, uint64_t *bar) {
    for (int64_t o = 0; o < len; o += 32768)
        umma::bulk_g2s(dst + o, blob + off + o, (uint32_t)imin64(32768, len - o), bar);
}

// the three split products for one B matrix: d (+)= a * b, K = 64 (4 k-steps)
// SINGLE: the reduced-precision variant (RECMG_PREC_TC16) keeps only xh * wh
template <bool SINGLE>
__device__ __forceinline__ void mma3x(uint32_t d, uint32_t a_hi, uint32_t a_lo, uint32_t b_saddr,
                                      uint32_t lo_off, int N, bool acc) {
    const uint32_t idesc = umma::idesc_f16(128, N);
    // one descriptor built per B image; the k-steps and the lo image only move
    // its 16 B-granular start field (+16 per 256 B k-step), so each MMA costs
    // one independent add instead of a dependent shift/mask chain
    const uint64_t dh = umma::make_desc(b_saddr, 128, 1024);
    const uint64_t dl = dh + (uint64_t)(lo_off >> 4);
#pragma unroll
    for (int ks = 0; ks < 4; ks++)
        umma::mma_ts(d, a_hi + 8 * ks, dh + (uint64_t)(16 * ks), idesc, (acc || ks > 0) ? 1u : 0u);
    if (SINGLE) return;
#pragma unroll
    for (int ks = 0; ks < 4; ks++)
        umma::mma_ts(d, a_hi + 8 * ks, dl + (uint64_t)(16 * ks), idesc, 1u);
#pragma unroll
    for (int ks = 0; ks < 4; ks++)
        umma::mma_ts(d, a_lo + 8 * ks, dh + (uint64_t)(16 * ks), idesc, 1u);
}
template <bool SINGLE>
__device__ __forceinline__ void mma3(uint32_t d, uint32_t a_hi, uint32_t a_lo, uint32_t b_saddr,
                                     int N, bool acc) {
    mma3x<SINGLE>(d, a_hi, a_lo, b_saddr, (uint32_t)N * 128u, N, acc);  // lo image follows hi
}
// half h of an N = 256 gate product into Z: B rows [128h, 128h + 128) start
// 16 KB into the hi (and lo) image of the N = 256 B matrix, D = Z columns [128h, +128)
template <bool SINGLE>
__device__ __forceinline__ void mma3_zhalf(uint32_t tbase, uint32_t a_hi, uint32_t a_lo,
                                           uint32_t b_saddr, bool acc, int h) {
    mma3x<SINGLE>(tbase + COL_Z + 128u * h, a_hi, a_lo, b_saddr + 16384u * h, 32768u, 128, acc);
}

// Z (+)= a * b for an N = 256 gate product; SPLIT: as two N = 128 halves
// committed to bar_a / bar_b (the cell starts on the first half), else one
// product committed to bar_a only (measured per model and phase: the split
// pays where the products are long -- the prefetch model's two-operand layers --
// and costs where one N = 256 product is short)
template <bool SINGLE, bool SPLIT, bool BOTH = false>
__device__ __forceinline__ void zproduct(uint32_t tbase, uint32_t a_hi, uint32_t a_lo,
                                         uint32_t b_saddr, bool acc, uint64_t *bar_a,
                                         uint64_t *bar_b) {
    if constexpr (SPLIT) {
        mma3_zhalf<SINGLE>(tbase, a_hi, a_lo, b_saddr, acc, 0);
        umma::commit(bar_a);
        mma3_zhalf<SINGLE>(tbase, a_hi, a_lo, b_saddr, acc, 1);
        umma::commit(bar_b);
    } else {
        mma3<SINGLE>(tbase + COL_Z, a_hi, a_lo, b_saddr, 256, acc);
        umma::commit(bar_a);
        if constexpr (BOTH) umma::commit(bar_b);   // the caller's cell waits on both
    }
}
// Z (+)= a1 * b1 + a2 * b2 (two operands, e.g. h0 Wx1 + h1 Wh1), split as above;
// unsplit it commits both barriers
template <bool SINGLE, bool SPLIT>
__device__ __forceinline__ void zproduct2(uint32_t tbase, uint32_t a1_hi, uint32_t a1_lo,
                                          uint32_t b1, bool acc1, uint32_t a2_hi, uint32_t a2_lo,
                                          uint32_t b2, uint64_t *bar_a, uint64_t *bar_b) {
    if constexpr (SPLIT) {
#pragma unroll
        for (int hf = 0; hf < 2; hf++) {
            mma3_zhalf<SINGLE>(tbase, a1_hi, a1_lo, b1, acc1, hf);
            mma3_zhalf<SINGLE>(tbase, a2_hi, a2_lo, b2, true, hf);
            umma::commit(hf == 0 ? bar_a : bar_b);
        }
    } else {
        mma3<SINGLE>(tbase + COL_Z, a1_hi, a1_lo, b1, 256, acc1);
        mma3<SINGLE>(tbase + COL_Z, a2_hi, a2_lo, b2, 256, true);
        umma::commit(bar_a);
        umma::commit(bar_b);
    }
}

// the four warps of a TMEM lane quadrant (warps q, q+4, q+8, q+12: the four
// parts of the quadrant's 32 rows) -- all a row's partial scores and head
// terms are exchanged within them, so the exchange needs no CTA barrier
#ifndef RECMG_QUAD_SYNC
#define RECMG_QUAD_SYNC 1
#endif
__device__ __forceinline__ void quad_sync(int quad) {
    if constexpr (RECMG_QUAD_SYNC)
        asm volatile("bar.sync %0, 128;" ::"r"(1 + quad) : "memory");
    else
        __syncthreads();
}

// sync point after threads wrote TMEM operands / before the MMA issue
__device__ __forceinline__ void tmem_writes_done() {
    umma::tmem_st_wait();
    umma::fence_before();
    __syncthreads();
}

__device__ __forceinline__ void wait_mma(uint64_t *mbar, uint32_t &phase) {
    umma::mbar_wait(mbar, phase);
    phase ^= 1u;
    umma::fence_after();
}

template <int N>
__device__ __forceinline__ void st_cols(uint32_t taddr, const uint32_t (&r)[N]) {
    if constexpr (N == 16) umma::tmem_st16(taddr, r);
    else if constexpr (N == 8) umma::tmem_st8(taddr, r);
    else umma::tmem_st4(taddr, r);
}

// the two half-sized column runs of an operand region (fp16 pairs: unit u at
// column u / 2) that hold this thread's units
template <int PARTS>
__device__ __forceinline__ void st_op_halves(const Ctx<PARTS> &c, uint32_t col,
                                             const uint32_t (&r)[Ctx<PARTS>::U / 2]) {
    constexpr int Q = Ctx<PARTS>::HU / 2;
    uint32_t r0[Q], r1[Q];
#pragma unroll
    for (int m = 0; m < Q; m++) { r0[m] = r[m]; r1[m] = r[Q + m]; }
    st_cols<Q>(c.lane_addr + col + (uint32_t)c.unit(0) / 2, r0);
    st_cols<Q>(c.lane_addr + col + (uint32_t)c.unit(Ctx<PARTS>::HU) / 2, r1);
}

// this thread's U units as fp16 hi|lo into an A operand region (32 columns each)
template <bool SINGLE, int PARTS>
__device__ __forceinline__ void store_operand(const Ctx<PARTS> &c, uint32_t col_hi,
                                              uint32_t col_lo, const float (&v)[Ctx<PARTS>::U]) {
    constexpr int H = Ctx<PARTS>::U / 2;
    uint32_t hi[H], lo[H];
#pragma unroll
    for (int m = 0; m < H; m++) {
        const __half2 h = __floats2half2_rn(v[2 * m], v[2 * m + 1]);
        const float2 hf = __half22float2(h);
        hi[m] = *reinterpret_cast<const uint32_t *>(&h);
        lo[m] = umma::pack_half2(v[2 * m] - hf.x, v[2 * m + 1] - hf.y);
    }
    st_op_halves(c, col_hi, hi);
    if (!SINGLE) st_op_halves(c, col_lo, lo);
}

// zero this thread's unit columns of a per-unit fp32 region (Q)
template <int PARTS>
__device__ __forceinline__ void zero_units(const Ctx<PARTS> &c, uint32_t col) {
    static_assert(Ctx<PARTS>::HU == 8, "two 8-column runs");
    const uint32_t z[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    umma::tmem_st8(c.lane_addr + col + c.unit(0), z);
    umma::tmem_st8(c.lane_addr + col + c.unit(8), z);
}

template <int PARTS>
__device__ __forceinline__ void zero_operand(const Ctx<PARTS> &c, uint32_t col_hi, uint32_t col_lo) {
    constexpr int H = Ctx<PARTS>::U / 2;
    uint32_t z[H];
#pragma unroll
    for (int m = 0; m < H; m++) z[m] = 0u;
    st_op_halves(c, col_hi, z);
    st_op_halves(c, col_lo, z);
}

// folded-table row loads: kept in L1 (hot ids repeat within a tile) but
// first out of L2, so the per-tile H / key scratch that every decoder step
// re-reads stays L2-resident (measured: caching -2.2%, prefetch -1.6% vs plain
// __ldg; an L2 evict_last policy on the scratch instead, or L1::no_allocate
// scratch loads, were slower -- DESIGN.md)
#ifndef RECMG_ROW_L1
#define RECMG_ROW_L1 0
#endif
#if RECMG_ROW_L1 == 0
#define RECMG_ROW_L1_Q "L1::evict_last"
#elif RECMG_ROW_L1 == 1
#define RECMG_ROW_L1_Q "L1::evict_normal"
#elif RECMG_ROW_L1 == 2
#define RECMG_ROW_L1_Q "L1::evict_first"
#else
#define RECMG_ROW_L1_Q "L1::no_allocate"
#endif
__device__ __forceinline__ float4 row_ld(const float4 *p) {
    float4 v;
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("ld.global.nc." RECMG_ROW_L1_Q ".L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
    return v;
}
#ifndef RECMG_ROW_V8
#define RECMG_ROW_V8 1
#endif
// the same as one 256-bit load (LDG.256, sm_100): a full 32 B sector per lane,
// half the load instructions and L1 tag lookups of two LDG.128
__device__ __forceinline__ void row_ld8(const float4 *p, float4 &a, float4 &b) {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("ld.global.nc." RECMG_ROW_L1_Q ".L2::cache_hint.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                 : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z),
                   "=f"(b.w)
                 : "l"(p), "l"(pol));
}

// Folded-table row of the NEXT step, gathered while the current step's MMA
// and epilogue run: the first NPRE float4 are loaded early into registers,
// the rest when the row is committed into Z (after the cell has read Z).
template <int PARTS, int NPRE_>
struct RowStageN;
// early float4 of the next row per phase: measured per model and phase --
// the register allocation is the whole story (caching decoder at 8: ~240 B
// of spills, +11%; caching encoder at 4 with decoder 4: +23%; prefetch
// encoder at 12: +3%)
#ifndef RECMG_NPRE_ENC_C
#define RECMG_NPRE_ENC_C 12
#endif
#ifndef RECMG_NPRE_ENC_P
#define RECMG_NPRE_ENC_P 8
#endif
#ifndef RECMG_NPRE_DEC
#define RECMG_NPRE_DEC 4
#endif

template <int PARTS, int NPRE_>
struct RowStageN {
    using C = Ctx<PARTS>;
    static constexpr int NF4 = C::U;            // 4U floats = U float4
    static constexpr int NH = C::HU;            // float4 per Z half (4 HU floats)
    static constexpr int NPRE = PARTS == 4 ? NPRE_ : 16;
    static_assert(NPRE % 4 == 0 && NH % 4 == 0, "loads and commits are whole 64-byte blocks");
    float4 x[NPRE];
    const float4 *src;   // this thread's first-half run; the second half is +128 floats
    // float4 i of this thread's row part: half i / NH, float4 i % NH of that half's run
    __device__ __forceinline__ const float4 *at(int i) const {
        return src + (i >= NH ? 32 : 0) + (i % NH);
    }
    __device__ __forceinline__ void prefetch(const C &c, const float *pid, int32_t g) {
        src = reinterpret_cast<const float4 *>(pid + (int64_t)g * 256 + c.zcol(0));
        if constexpr (RECMG_ROW_V8) {
#pragma unroll
            for (int q = 0; q < NPRE; q += 2) row_ld8(at(q), x[q], x[q + 1]);
        } else {
#pragma unroll
            for (int q = 0; q < NPRE; q++) x[q] = row_ld(at(q));
        }
    }
    __device__ __forceinline__ void commit(const C &c) {
#pragma unroll
        for (int blk = 0; blk < NF4 / 4; blk++) {
            uint32_t r[16];
            float4 late[4];
            if constexpr (RECMG_ROW_V8) {
                if (blk * 4 >= NPRE) {
                    row_ld8(at(blk * 4), late[0], late[1]);
                    row_ld8(at(blk * 4 + 2), late[2], late[3]);
                }
            }
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const int i = blk * 4 + q;
                const float4 u = i < NPRE ? x[i < NPRE ? i : 0]
                                 : (RECMG_ROW_V8 ? late[q] : row_ld(at(i)));
                r[4 * q + 0] = __float_as_uint(u.x);
                r[4 * q + 1] = __float_as_uint(u.y);
                r[4 * q + 2] = __float_as_uint(u.z);
                r[4 * q + 3] = __float_as_uint(u.w);
            }
            umma::tmem_st16(c.lane_addr + COL_Z + c.zcol(4 * blk), r);
        }
    }
};

// Z[my 4U columns] = row (same for every chunk: prefetch slot projection)
template <int PARTS>
__device__ __forceinline__ void init_z_from_row(const Ctx<PARTS> &c, const float *rowp) {
    constexpr int NC = 4 * Ctx<PARTS>::U;
#pragma unroll
    for (int blk = 0; blk < NC / 16; blk++) {
        const float4 *a = reinterpret_cast<const float4 *>(rowp + c.zcol(4 * blk));
        uint32_t r[16];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const float4 x = a[q];
            r[4 * q + 0] = __float_as_uint(x.x);
            r[4 * q + 1] = __float_as_uint(x.y);
            r[4 * q + 2] = __float_as_uint(x.z);
            r[4 * q + 3] = __float_as_uint(x.w);
        }
        umma::tmem_st16(c.lane_addr + COL_Z + c.zcol(4 * blk), r);
    }
}

struct NoMid {
    __device__ __forceinline__ void operator()() const {}
};

// LSTM cell on this thread's U hidden units (model.py:103-112)
// mid() runs between the two Z halves (the wait for the second half's commit)
template <bool BIAS, int PARTS, class Mid = NoMid>
__device__ __forceinline__ void cell(const Ctx<PARTS> &c, const float *bias,
                                     float (&cs)[Ctx<PARTS>::U], float (&h)[Ctx<PARTS>::U],
                                     Mid mid = Mid()) {
    constexpr int U = Ctx<PARTS>::U;
    static_assert(Ctx<PARTS>::HU == 8, "one loop iteration per Z half");
    const float4 *b4 = reinterpret_cast<const float4 *>(bias);   // gate-interleaved per unit
#pragma unroll
    for (int blk = 0; blk < U / 4; blk += 2) {
        if (blk == 2) mid();
        float z0[16], z1[16];
        umma::tmem_ld16(c.lane_addr + COL_Z + c.zcol(4 * blk), z0);
        umma::tmem_ld16(c.lane_addr + COL_Z + c.zcol(4 * blk + 4), z1);
        umma::tmem_ld_wait();
#pragma unroll
        for (int g4 = 0; g4 < 2; g4++) {
            float og[4], dc[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int j = 4 * blk + 4 * g4 + u;
                const float *z = g4 == 0 ? &z0[4 * u] : &z1[4 * u];
                float zi = z[0], zf = z[1], zg = z[2], zo = z[3];
                if (BIAS) {
                    const float4 bb = b4[c.unit(j)];
                    zi += bb.x; zf += bb.y; zg += bb.z; zo += bb.w;
                }
                float ig = ex2_den(zi), fg = ex2_den(zf), gd = ex2_den(zg), o = ex2_den(zo);
                rcp4(ig, fg, gd, o);
                // the cell state is kept scaled by 2 log2(e): c' = f c' + i (2 log2(e) g)
                const float gg = fmaf(-4.0f * kLog2e, gd, 2.0f * kLog2e);
                cs[j] = fg * cs[j] + ig * gg;
                og[u] = o;
                dc[u] = ex2_den(cs[j]);
            }
            rcp4(dc[0], dc[1], dc[2], dc[3]);
#pragma unroll
            for (int u = 0; u < 4; u++) h[4 * blk + 4 * g4 + u] = og[u] * fmaf(-2.0f, dc[u], 1.0f);
        }
    }
}

// this thread's U unit columns (col + unit) of a per-unit TMEM region
template <int PARTS>
__device__ __forceinline__ void readU(const Ctx<PARTS> &c, uint32_t col,
                                      float (&v)[Ctx<PARTS>::U]) {
    static_assert(Ctx<PARTS>::HU == 8, "two 8-column runs");
    float t0[8], t1[8];
    umma::tmem_ld8(c.lane_addr + col + c.unit(0), t0);
    umma::tmem_ld8(c.lane_addr + col + c.unit(8), t1);
    umma::tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 8; i++) { v[i] = t0[i]; v[8 + i] = t1[i]; }
}

// scratch position j of this thread: NQ float4 as NQ/2 32-byte pairs at
// pair index ((j*8 + NQ/2*part + u/2)*128 + row); consecutive rows of a warp
// are consecutive 32 B -> one LDG.256 / STG.256 per pair, fully coalesced
template <int PARTS>
__device__ __forceinline__ float4 *scratch_at(float *base, const Ctx<PARTS> &c, int j, int u) {
    return reinterpret_cast<float4 *>(base) +
           ((int64_t)(j * 8 + Ctx<PARTS>::NQ / 2 * c.part + u / 2) * 128 + c.row) * 2 + (u & 1);
}

// all NQ float4 of scratch position j (256-bit loads)
template <int PARTS>
__device__ __forceinline__ void scr_ld_pos(float *base, const Ctx<PARTS> &c, int j,
                                           float4 (&x)[Ctx<PARTS>::NQ]) {
#pragma unroll
    for (int u = 0; u < Ctx<PARTS>::NQ; u += 2) {
        const float4 *p = scratch_at(base, c, j, u);
        asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(x[u].x), "=f"(x[u].y), "=f"(x[u].z), "=f"(x[u].w), "=f"(x[u + 1].x),
                       "=f"(x[u + 1].y), "=f"(x[u + 1].z), "=f"(x[u + 1].w)
                     : "l"(p));
    }
}

template <int PARTS>
__device__ __forceinline__ void storeU(float *base, const Ctx<PARTS> &c, int j,
                                       const float (&v)[Ctx<PARTS>::U]) {
#pragma unroll
    for (int u = 0; u < Ctx<PARTS>::NQ; u += 2)
        asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                     ::"l"(scratch_at(base, c, j, u)), "f"(v[4 * u]), "f"(v[4 * u + 1]),
                       "f"(v[4 * u + 2]), "f"(v[4 * u + 3]), "f"(v[4 * u + 4]), "f"(v[4 * u + 5]),
                       "f"(v[4 * u + 6]), "f"(v[4 * u + 7])
                     : "memory");
}

// encoder: position j of the attention keys, stored as X = e^(2e) (bit j of
// rawmask clear) or as raw e when any of this thread's units is out of range
template <int PARTS>
__device__ __forceinline__ void store_keys(float *Es, const Ctx<PARTS> &c, int j,
                                           float (&e)[Ctx<PARTS>::U], uint32_t &rawmask) {
    constexpr int U = Ctx<PARTS>::U;
    bool ok = true;
#pragma unroll
    for (int k = 0; k < U; k++) ok = ok && fabsf(e[k]) <= 0.5f * kExpLim;   // |2e| <= kExpLim
    if (ok) {
#pragma unroll
        for (int k = 0; k < U; k++) e[k] = ex2f(e[k] * (2.0f * kLog2e));   // = __expf(2e) bit for bit
    } else {
        rawmask |= 1u << j;
    }
    storeU(Es, c, j, e);
}

// sum_u v_u tanh(e_u + q_u) over this thread's units for one position
template <int NQ>
__device__ __forceinline__ float score_fast(const float4 (&x)[NQ], const float (&qx)[4 * NQ],
                                            const float4 (&vr)[NQ]) {
    // per 4 units: sum v_k / d_k as one fraction over d_a d_b d_c d_d (each
    // d in [1, 2^32), so the product stays finite), one MUFU.RCP per 4 units
    float s0 = 0.0f, s1 = 0.0f;
#pragma unroll
    for (int u = 0; u < NQ; u++) {
        const float4 v = vr[u];
        const float a = fmaf(x[u].x, qx[4 * u + 0], 1.0f), b = fmaf(x[u].y, qx[4 * u + 1], 1.0f);
        const float cc = fmaf(x[u].z, qx[4 * u + 2], 1.0f), d = fmaf(x[u].w, qx[4 * u + 3], 1.0f);
        const float dab = a * b, dcd = cc * d;
        const float nab = fmaf(v.x, b, v.y * a), ncd = fmaf(v.z, d, v.w * cc);
        const float num = fmaf(nab, dcd, ncd * dab);
        const float r = frcp(dab * dcd);
        if (u & 1) s1 = fmaf(num, r, s1);
        else s0 = fmaf(num, r, s0);
    }
    return -2.0f * (s0 + s1);   // + sum_u v_u by the caller
}

// direct form: raw keys (raw) or keys stored as X = e^(2e) recovered by log
template <int NQ>
__device__ __forceinline__ float score_slow(const float4 (&x)[NQ], const float (&q)[4 * NQ],
                                            const float4 (&vr)[NQ], bool raw) {
    float s = 0.0f;
#pragma unroll
    for (int u = 0; u < NQ; u++) {
        const float4 v = vr[u];
        const float4 e = raw ? x[u] : make_float4(0.5f * __logf(x[u].x), 0.5f * __logf(x[u].y),
                                                  0.5f * __logf(x[u].z), 0.5f * __logf(x[u].w));
        s += v.x * ftanh(e.x + q[4 * u + 0]);
        s += v.y * ftanh(e.y + q[4 * u + 1]);
        s += v.z * ftanh(e.z + q[4 * u + 2]);
        s += v.w * ftanh(e.w + q[4 * u + 3]);
    }
    return s;
}

// partial attention scores over this thread's units (model.py:118-119),
// two positions per iteration so 2*NQ loads are in flight
#ifndef RECMG_SCORE_POS
#define RECMG_SCORE_POS 4
#endif
// partial attention scores over this thread's units (model.py:118-119) from
// the query in TMEM column col_q.  Warps whose positions and query are all in
// the fast (exponential-product) range -- the common case -- run a loop that
// keeps no raw query in registers and has RECMG_SCORE_POS positions' loads in
// flight; otherwise the two-position loop with the direct-form fallback runs.
template <int PARTS>
__device__ __forceinline__ void attn_scores(const Ctx<PARTS> &c, float *Es, int npos,
                                            uint32_t col_q, const float *vp,
                                            float vsum, uint32_t rawmask, float *s_part, int L) {
    constexpr int NQ = Ctx<PARTS>::NQ;
    constexpr int U = Ctx<PARTS>::U;
    const float4 *v4 = reinterpret_cast<const float4 *>(vp);   // float4 u of mine: unit(4u) / 4
    float qx[U];
    bool qok = true;
    {
        float q[U];
        readU(c, col_q, q);
#pragma unroll
        for (int k = 0; k < U; k++) {
            qok = qok && fabsf(q[k]) <= 0.5f * kExpLim;
            qx[k] = ex2f(q[k] * (2.0f * kLog2e));
        }
    }
    const uint32_t npmask = npos >= 32 ? 0xFFFFFFFFu : ((1u << npos) - 1u);
    const uint32_t slow = (qok ? rawmask : 0xFFFFFFFFu) & npmask;
    float4 vr[NQ];   // this thread's att_v units, loaded once per step
#pragma unroll
    for (int u = 0; u < NQ; u++) vr[u] = v4[c.unit(4 * u) / 4];
    float *sp = s_part + (c.part * L) * 128 + c.row;
    if (!__any_sync(0xFFFFFFFFu, slow != 0u)) {
        constexpr int P = RECMG_SCORE_POS;
        int j = 0;
        for (; j + P <= npos; j += P) {
            float4 e[P][NQ];
#pragma unroll
            for (int i = 0; i < P; i++) scr_ld_pos(Es, c, j + i, e[i]);
#pragma unroll
            for (int i = 0; i < P; i++) sp[(j + i) * 128] = vsum + score_fast<NQ>(e[i], qx, vr);
        }
        for (; j < npos; j++) {
            float4 e0[NQ];
            scr_ld_pos(Es, c, j, e0);
            sp[j * 128] = vsum + score_fast<NQ>(e0, qx, vr);
        }
        return;
    }
    float q[U];   // warp-uniform reload for the direct form
    readU(c, col_q, q);
    auto score = [&](const float4 (&x)[NQ], int j) {
        return ((slow >> j) & 1u) ? score_slow<NQ>(x, q, vr, (rawmask >> j) & 1u)
                                  : vsum + score_fast<NQ>(x, qx, vr);
    };
    int j = 0;
    for (; j + 2 <= npos; j += 2) {
        float4 e0[NQ], e1[NQ];
        scr_ld_pos(Es, c, j, e0); scr_ld_pos(Es, c, j + 1, e1);
        sp[j * 128] = score(e0, j);
        sp[(j + 1) * 128] = score(e1, j + 1);
    }
    if (j < npos) {
        float4 e0[NQ];
        scr_ld_pos(Es, c, j, e0);
        sp[j * 128] = score(e0, j);
    }
}

template <int PARTS>
__device__ __forceinline__ float full_score(const float *s_part, int L, int j, int row) {
    float s = 0.0f;
#pragma unroll
    for (int p = 0; p < PARTS; p++) s += s_part[(p * L + j) * 128 + row];
    return s;
}

template <int NQ>
__device__ __forceinline__ void acc_ctx(float (&ctx)[4 * NQ], float e, const float4 (&h)[NQ]) {
#pragma unroll
    for (int u = 0; u < NQ; u++) {
        ctx[4 * u + 0] += e * h[u].x;
        ctx[4 * u + 1] += e * h[u].y;
        ctx[4 * u + 2] += e * h[u].z;
        ctx[4 * u + 3] += e * h[u].w;
    }
}

#ifndef RECMG_CTX_POS
#define RECMG_CTX_POS 3
#endif
constexpr float kShiftMax = 40.0f;   // e^(-2 * 40) = 1.8e-35 > FLT_MIN

// softmax over positions + context on this thread's units (model.py:120-123)
template <int PARTS>
__device__ __forceinline__ void attn_context(const Ctx<PARTS> &c, float *Hs, int npos,
                                             const float *s_part, int L, float vabs,
                                             float (&ctx)[Ctx<PARTS>::U]) {
    constexpr int NQ = Ctx<PARTS>::NQ;
    // softmax shift (autodiff.py:226-236 uses the max): every score is
    // sum_u v_u tanh(.), so |s| <= vabs = sum_u |v_u| and e^(s - vabs) stays a
    // normal float while vabs <= kShiftMax; the shift cancels in the ratio, so
    // the max pass is skipped.  Larger |v| falls back to the max.
    float mx = vabs;
    if (vabs > kShiftMax) {
        mx = -INFINITY;
        for (int j = 0; j < npos; j++) mx = fmaxf(mx, full_score<PARTS>(s_part, L, j, c.row));
    }
#pragma unroll
    for (int k = 0; k < 4 * NQ; k++) ctx[k] = 0.0f;
    float sum = 0.0f;
    int j = 0;
    constexpr int P = RECMG_CTX_POS;   // positions' loads in flight
    for (; j + P <= npos; j += P) {
        float4 hv[P][NQ];
#pragma unroll
        for (int i = 0; i < P; i++) scr_ld_pos(Hs, c, j + i, hv[i]);
#pragma unroll
        for (int i = 0; i < P; i++) {
            const float e = __expf(full_score<PARTS>(s_part, L, j + i, c.row) - mx);
            sum += e;
            acc_ctx<NQ>(ctx, e, hv[i]);
        }
    }
    for (; j + 2 <= npos; j += 2) {
        float4 h0[NQ], h1[NQ];
        scr_ld_pos(Hs, c, j, h0); scr_ld_pos(Hs, c, j + 1, h1);
        const float e0 = __expf(full_score<PARTS>(s_part, L, j, c.row) - mx);
        const float e1 = __expf(full_score<PARTS>(s_part, L, j + 1, c.row) - mx);
        sum += e0 + e1;
        acc_ctx<NQ>(ctx, e0, h0);
        acc_ctx<NQ>(ctx, e1, h1);
    }
    if (j < npos) {
        float4 h0[NQ];
        scr_ld_pos(Hs, c, j, h0);
        const float e0 = __expf(full_score<PARTS>(s_part, L, j, c.row) - mx);
        sum += e0;
        acc_ctx<NQ>(ctx, e0, h0);
    }
    const float inv = __fdividef(1.0f, sum);
#pragma unroll
    for (int k = 0; k < 4 * NQ; k++) ctx[k] *= inv;
}

// partial head: sum_k tanh(comb_k + b_k) * w_k over my units (model.py:177-179)
template <int PARTS>
__device__ __forceinline__ float head_partial(const Ctx<PARTS> &c, uint32_t col,
                                              const float *comb_b, const float *head_w) {
    constexpr int U = Ctx<PARTS>::U;
    float v[U];
    readU(c, col, v);
    float s[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    const float4 *cb4 = reinterpret_cast<const float4 *>(comb_b);
    const float4 *hw4 = reinterpret_cast<const float4 *>(head_w);
#pragma unroll
    for (int k = 0; k < U; k += 4) {
        const float4 cb = cb4[c.unit(k) / 4], hw = hw4[c.unit(k) / 4];
        float d[4] = {ex2_den(v[k] + cb.x), ex2_den(v[k + 1] + cb.y), ex2_den(v[k + 2] + cb.z),
                      ex2_den(v[k + 3] + cb.w)};
        rcp4(d[0], d[1], d[2], d[3]);
        s[0] += fmaf(-2.0f, d[0], 1.0f) * hw.x;
        s[1] += fmaf(-2.0f, d[1], 1.0f) * hw.y;
        s[2] += fmaf(-2.0f, d[2], 1.0f) * hw.z;
        s[3] += fmaf(-2.0f, d[3], 1.0f) * hw.w;
    }
    return (s[0] + s[1]) + (s[2] + s[3]);
}

__device__ __forceinline__ void emit_logit(const TcArgs &a, int64_t chunk, int T, int t, float s,
                                           bool caching) {
    if (chunk >= a.batch) return;
    a.logits[chunk * T + t] = s;
    if (caching) {
        if (a.bits) a.bits[chunk * T + t] = s >= 0.0f ? 1 : 0;   // runtime.py:192
    } else if (a.pf_gid) {
        const double po = 1.0 / (1.0 + exp(-(double)s));          // model.py:250-258
        const int64_t V = a.m.total_ids;
        double gg = floor(po * (double)(V - 1) + 0.5);
        gg = fmin(fmax(gg, 0.0), (double)(V - 1));
        a.pf_gid[chunk * T + t] = (int32_t)gg;
    }
}

}  // namespace

// ---------------------------------------------------------------------------
// phases: 0 enc table init+sync, 1 enc MMA wait, 2 enc epilogue, 3 dec init+sync,
// 4 dec MMA1 wait, 5 dec head+scores+sync, 6 dec softmax/ctx+sync, 7 dec MMA2 wait,
// 8 dec cell, 9 weight loads, 10 prefetch layer-1 MMA wait, 11 prefetch layer-1 cell
// MODE bit 0: phase-cycle instrumentation; bit 1: single-product GEMMs (TC16)
#ifndef RECMG_ZSPLIT_CENC
#define RECMG_ZSPLIT_CENC 0
#endif
#ifndef RECMG_ZSPLIT_CDEC
#define RECMG_ZSPLIT_CDEC 0
#endif
constexpr bool kSplitCEnc = RECMG_ZSPLIT_CENC != 0;   // caching encoder Z += h Wh
constexpr bool kSplitCDec = RECMG_ZSPLIT_CDEC != 0;   // caching decoder Z += ctx Wc
#ifndef RECMG_ZSPLIT_P
#define RECMG_ZSPLIT_P 15
#endif
constexpr bool kSplitPL0 = (RECMG_ZSPLIT_P & 1) != 0;  // prefetch encoder layer 0
constexpr bool kSplitPL1 = (RECMG_ZSPLIT_P & 2) != 0;  // prefetch encoder layer 1
constexpr bool kSplitPD0 = (RECMG_ZSPLIT_P & 4) != 0;  // prefetch decoder layer 0
constexpr bool kSplitPD1 = (RECMG_ZSPLIT_P & 8) != 0;  // prefetch decoder layer 1

template <int KIND, int MODE>
__global__ void __launch_bounds__(128 * PartsOf<KIND>::value, 1) lstm_tc_kernel(TcArgs a) {
    constexpr bool PROF = (MODE & 1) != 0;
    constexpr bool SINGLE = (MODE & 2) != 0;
    PhaseClock<PROF> pc;
    pc.start();
    constexpr int PARTS = PartsOf<KIND>::value;
    using C = Ctx<PARTS>;
    constexpr int U = C::U;
    constexpr int NT = C::NT;
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t mbar, mbar2;   // caching: mbar2 tracks the MMAs split off
    __shared__ uint64_t mbar3;         // second N = 128 half of a gate product
    __shared__ uint64_t tma_bar;       // async weight loads / swaps
    __shared__ uint64_t tma_bar2;      // prefetch decoder: reload of the weights s_part overlays
    __shared__ uint32_t tmem_base_s;
    __shared__ float lpart[PARTS][128];
    __shared__ int s_tile;
    constexpr bool caching = (KIND == RECMG_MODEL_CACHING);
    const int L = a.m.l_in;
    const int T = caching ? L : a.m.l_out;
    float *s_part = reinterpret_cast<float *>(smem + a.tl.spart_off);

    C c;
    c.tid = threadIdx.x;
    c.warp = c.tid >> 5;
    c.lane = c.tid & 31;
    c.quad = c.warp & 3;
    c.part = c.warp >> 2;
    c.row = 32 * c.quad + c.lane;
    if (c.tid == 0) {
        umma::mbar_init(&mbar, 1);
        umma::mbar_init(&mbar2, 1);
        umma::mbar_init(&mbar3, 1);
        umma::mbar_init(&tma_bar, 1);
        umma::mbar_init(&tma_bar2, 1);
    }
    if (c.warp == 0) umma::tmem_alloc<512>(&tmem_base_s);
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    c.tbase = tmem_base_s;
    c.lane_addr = c.tbase + ((uint32_t)(32 * c.quad) << 16);
    uint32_t phase = 0, phase2 = 0, phase3 = 0, tphase = 0, tphase2 = 0;
    const uint32_t sbase = umma::smem_u32(smem);
    const TcLayout &tl = a.tl;
    const PackedLayout &pl = a.pl;
    const float *pid_enc = reinterpret_cast<const float *>(a.blob + tl.pid[0]);
    const float *pid_dec = reinterpret_cast<const float *>(a.blob + tl.pid[1]);
    float *Hs = a.scratch + (int64_t)blockIdx.x * 2 * L * 128 * 64;
    float *Es = Hs + (int64_t)L * 128 * 64;
    // the per-unit constants every step reads (layer-1 biases, att_v, comb bias,
    // head weights, prefetch slot projections) live in shared memory: broadcast
    // LDS instead of LDG, the L1 tag stage is kept for the row gathers
    float *cst = reinterpret_cast<float *>(smem + tl.const_off);
    {
        const int nslot = caching ? 0 : a.m.l_out * 256;
        for (int i = c.tid; i < 704 + nslot; i += NT) {
            float v = 0.0f;
            if (i < 512) {
                if (!caching) v = __ldg(a.dense + (i < 256 ? pl.enc_b[1] + i : pl.dec_b[1] + i - 256));
            } else if (i < 576) {
                v = __ldg(a.dense + pl.att_v + i - 512);
            } else if (i < 640) {
                v = __ldg(a.dense + pl.comb_b + i - 576);
            } else if (i < 704) {
                v = __ldg(a.dense + pl.head_w + i - 640);
            } else {
                v = __ldg(a.dense + pl.slot_proj + i - 704);
            }
            cst[i] = v;
        }
        __syncthreads();
    }
    const float *enc_b1 = cst, *dec_b1 = cst + 256;
    const float *att_v = cst + 512;
    const float *comb_b = cst + 576;
    const float *head_w = cst + 640;
    const float *slot_proj = cst + 704;
    const float head_b = __ldg(a.dense + pl.head_b);
    float vsum = 0.0f;   // sum of this thread's att_v units (score_fast)
    for (int k = 0; k < U; k++) vsum += att_v[c.unit(k)];
    float vabs = 0.0f;   // sum over all d units of |att_v| (attn_context's shift)
    for (int k = 0; k < 64; k++) vabs += fabsf(att_v[k]);
    const int64_t n_tiles = (a.batch + 127) / 128;

    // dynamic tile scheduler: a CTA that starts late (its SM busy with a
    // co-scheduled replay CTA) simply takes fewer tiles
    if (c.tid == 0) s_tile = atomicAdd(a.tile_counter, 1);
    __syncthreads();
    for (int64_t tile = s_tile; tile < n_tiles;) {
        const int64_t chunk = tile * 128 + c.row;
        const int64_t crow = chunk < a.batch ? chunk : a.batch - 1;  // clamp pad rows
        const int32_t *gid = a.gid + crow * L;
        float cs0[U], cs1[U], h[U];

        // ====================== encoder (model.py:131-145) ======================
        pc.mark(9);
        if (caching) {
            load_phase_tma(smem, a.blob, tl.phase_off[0], tl.phase_len[0], c.tid, &tma_bar,
                           tphase);
        } else {
            // prefetch encoder layout (small shared memory = more L1 for the
            // folded-table rows): Wh1 | att_enc resident at [0, 80 KB), one
            // 64 KB slot holding Wh0 for layer 0 and Wx1 for layer 1 (TMA swaps)
            umma::fence_proxy_async();
            __syncthreads();
            if (c.tid == 0) {
                umma::mbar_expect_tx(&tma_bar, (uint32_t)(tl.img256 + tl.img64 + tl.img256));
                tma_piece(smem, a.blob, tl.phase_off[0] + tl.b_off[2], tl.img256 + tl.img64,
                          &tma_bar);
                tma_piece(smem + tl.eslot, a.blob, tl.phase_off[0] + tl.b_off[0], tl.img256,
                          &tma_bar);
            }
            wait_mma(&tma_bar, tphase);
        }
#pragma unroll
        for (int k = 0; k < U; k++) { cs0[k] = 0.0f; cs1[k] = 0.0f; }
        if (caching) {
            zero_operand(c, A_H_HI, A_H_LO);
        } else {
            zero_operand(c, P_H0_HI, P_H0_LO);
            zero_operand(c, P_H1_HI, P_H1_LO);
        }
        uint32_t rawmask = 0;   // attention key positions stored raw (store_keys)
        RowStageN<PARTS, caching ? RECMG_NPRE_ENC_C : RECMG_NPRE_ENC_P> stage;
        stage.prefetch(c, pid_enc, __ldg(gid));
        // the id of the row gathered at step t (for step t + 1) is loaded one
        // step earlier still, so the gather's address is in a register when the
        // step reaches it (prefetch -0.6%, caching encoder -0.7%)
#ifndef RECMG_GID_AHEAD_C
#define RECMG_GID_AHEAD_C 1
#endif
        int32_t g_ahead = ((!caching || RECMG_GID_AHEAD_C) && L > 1) ? __ldg(gid + 1) : 0;
        stage.commit(c);
        for (int t = 0; t <= L; t++) {
            const bool last = (t == L);   // t == L: only enc_pre of the last state
            pc.mark(0);
            tmem_writes_done();
            pc.mark(1);
            if (caching) {
                // Q first (its own barrier), then Z: the keys of step t-1 are
                // stored while the long N=256 Z product still runs
                if (c.tid == 0) {
                    umma::fence_after();
                    mma3<SINGLE>(c.tbase + COL_Q, c.tbase + A_H_HI, c.tbase + A_H_LO,
                         sbase + tl.b_off[1], 64, false);                  // Q = h att_enc
                    umma::commit(&mbar);
                    if (!last)                                    // Z += h Wh
                        zproduct<SINGLE, kSplitCEnc>(c.tbase, c.tbase + A_H_HI, c.tbase + A_H_LO,
                                                     sbase + tl.b_off[0], true, &mbar2, &mbar3);
                }
                pc.mark(12);
                if (t + 1 < L) {
                    if constexpr (RECMG_GID_AHEAD_C) {
                        const int32_t g1 = g_ahead;
                        if (t + 2 < L) g_ahead = __ldg(gid + t + 2);
                        stage.prefetch(c, pid_enc, g1);
                    } else {
                        stage.prefetch(c, pid_enc, __ldg(gid + t + 1));
                    }
                }
                pc.mark(13);
                wait_mma(&mbar, phase);
                pc.mark(2);
                if (t >= 1) {
                    float ep[U];
                    readU(c, COL_Q, ep);
                    store_keys(Es, c, t - 1, ep, rawmask);
                }
                if (!last) {
                    wait_mma(&mbar2, phase2);
                    if constexpr (kSplitCEnc)
                        cell<false>(c, nullptr, cs0, h, [&] { wait_mma(&mbar3, phase3); });
                    else
                        cell<false>(c, nullptr, cs0, h);
                    store_operand<SINGLE>(c, A_H_HI, A_H_LO, h);
                    storeU(Hs, c, t, h);
                    if (t + 1 < L) stage.commit(c);
                }
            } else {
                // Q = h1(t-1) att_enc (barrier 2) right behind layer 0: it only
                // needs h1(t-1), so it runs under the layer-0 cell and the keys
                // of step t-1 are ready before the layer-1 product finishes
                if (t >= 1 && !last) wait_mma(&tma_bar, tphase);   // Wh0 back in the slot
                if (c.tid == 0) {
                    umma::fence_after();
                    if (!last) {
                        // layer 0: Z = Pid + Ptab + h0 Wh0 (slot)
                        zproduct<SINGLE, kSplitPL0, true>(c.tbase, c.tbase + P_H0_HI,
                                                          c.tbase + P_H0_LO, sbase + tl.eslot,
                                                          true, &mbar, &mbar3);
                    }
                    if (t >= 1) {
                        mma3<SINGLE>(c.tbase + COL_Q, c.tbase + P_H1_HI, c.tbase + P_H1_LO,
                             sbase + tl.img256, 64, false);               // att_enc
                        umma::commit(&mbar2);
                    }
                }
                if (!last) {
                    wait_mma(&mbar, phase);
                    pc.mark(2);
                    cell<false>(c, nullptr, cs0, h, [&] {
                        wait_mma(&mbar3, phase3);
                        if (c.tid == 0) {   // Wh0 done: Wx1 into the slot under the layer-0 cell
                            umma::mbar_expect_tx(&tma_bar, (uint32_t)tl.img256);
                            tma_piece(smem + tl.eslot, a.blob, tl.phase_off[0] + tl.b_off[1],
                                      tl.img256, &tma_bar);
                        }
                    });
                    store_operand<SINGLE>(c, P_H0_HI, P_H0_LO, h);
                    pc.mark(15);
                    wait_mma(&tma_bar, tphase);                    // Wx1 in the slot
                    pc.mark(14);
                    tmem_writes_done();
                    pc.mark(12);
                    // layer 1: Z = h0 Wx1 + h1 Wh1 (+b1 in the cell)
                    if (c.tid == 0) {
                        umma::fence_after();
                        zproduct2<SINGLE, kSplitPL1>(c.tbase, c.tbase + P_H0_HI, c.tbase + P_H0_LO,
                                                     sbase + tl.eslot, false,      // Wx1 (slot)
                                                     c.tbase + P_H1_HI, c.tbase + P_H1_LO,
                                                     sbase, &mbar, &mbar3);        // Wh1
                    }
                }
                if (t + 1 < L) {
                    const int32_t g1 = g_ahead;
                    if (t + 2 < L) g_ahead = __ldg(gid + t + 2);
                    stage.prefetch(c, pid_enc, g1);
                }
                pc.mark(13);
                if (t >= 1) {
                    wait_mma(&mbar2, phase2);
                    float ep[U];
                    readU(c, COL_Q, ep);
                    store_keys(Es, c, t - 1, ep, rawmask);
                }
                pc.mark(10);
                if (!last) {
                    wait_mma(&mbar, phase);
                    pc.mark(11);
                    cell<true>(c, enc_b1, cs1, h, [&] {
                        wait_mma(&mbar3, phase3);
                        if (t + 1 < L && c.tid == 0) {   // Wx1 done: Wh0 back for the next step
                            umma::mbar_expect_tx(&tma_bar, (uint32_t)tl.img256);
                            tma_piece(smem + tl.eslot, a.blob, tl.phase_off[0] + tl.b_off[0],
                                      tl.img256, &tma_bar);
                        }
                    });
                    store_operand<SINGLE>(c, P_H1_HI, P_H1_LO, h);
                    storeU(Hs, c, t, h);
                    if (t + 1 < L) stage.commit(c);
                }
            }
        }
        __syncthreads();  // scratch rows are read back by the same threads that wrote them

        // ====================== decoder (model.py:156-181) ======================
#pragma unroll
        for (int k = 0; k < U; k++) { cs0[k] = 0.0f; cs1[k] = 0.0f; }
        pc.mark(9);
        if (caching) {
            // decoder layout (shared memory kept small: the L1 that holds the
            // folded-table rows is what is left of the 256 KB): att_dec |
            // Wcomb_h | Wcomb_c resident at [0, 48 KB), then one 64 KB slot
            // that holds Wh_d for GEMM1 and Wc_d for GEMM2 (TMA swaps)
            umma::fence_proxy_async();
            __syncthreads();
            if (c.tid == 0) {
                umma::mbar_expect_tx(&tma_bar, (uint32_t)(2 * tl.img64 + tl.img256 + tl.img64));
                tma_piece(smem, a.blob, tl.phase_off[1] + tl.b_off[3], 2 * tl.img64, &tma_bar);
                tma_piece(smem + 2 * tl.img64, a.blob, tl.phase_off[1] + tl.b_off[6], tl.img64,
                          &tma_bar);
                tma_piece(smem + tl.dslot, a.blob, tl.phase_off[1] + tl.b_off[2], tl.img256,
                          &tma_bar);
            }
            wait_mma(&tma_bar, tphase);
        } else {
            // prefetch: the rotating region starts with att_dec | Wcomb_h | Wcomb_c
            load_phase_tma(smem, a.blob, tl.phase_off[1] + tl.b_off[4], 3 * tl.img64, c.tid,
                           &tma_bar, tphase);
        }
        float lsum;
        if (caching) {
            zero_operand(c, A_H_HI, A_H_LO);
            zero_operand(c, A_X_HI, A_X_LO);
            zero_units(c, COL_Q);
            RowStageN<PARTS, RECMG_NPRE_DEC> dstage;
            dstage.prefetch(c, pid_dec, __ldg(gid));
#ifndef RECMG_GID_AHEAD_D
#define RECMG_GID_AHEAD_D 0
#endif
            int32_t gd_ahead = (RECMG_GID_AHEAD_D && T > 1) ? __ldg(gid + 1) : 0;
            dstage.commit(c);
            for (int t = 0; t <= T; t++) {
                const bool last = (t == T);   // t == T: only finish comb_{T-1}
                pc.mark(3);
                if (t >= 1) {
                    wait_mma(&mbar2, phase2);                  // C = ctx Wcomb_c of step t-1
                    if (!last) wait_mma(&tma_bar, tphase);     // Wh_d back in the slot
                    wait_mma(&tma_bar2, tphase2);              // att_dec | Wcomb_h over s_part
                }
                tmem_writes_done();
                pc.mark(4);
                // GEMM1 on h_{t-1}: Z += h Wh_d ; [Q | C] += h [att_dec | Wcomb_h]
                // (one N = 128 product: Q was zeroed after the previous step's
                // scores, C holds ctx_{t-1} Wcomb_c) first (barrier 1), Z += h Wh_d
                // after (barrier 2): the head and the attention run while the N=256
                // product finishes
                if (c.tid == 0) {
                    umma::fence_after();
                    mma3<SINGLE>(c.tbase + COL_Q, c.tbase + A_H_HI, c.tbase + A_H_LO,
                         sbase, 128, true);                              // att_dec | Wcomb_h
                    umma::commit(&mbar);
                    if (!last) {
                        mma3<SINGLE>(c.tbase + COL_Z, c.tbase + A_H_HI, c.tbase + A_H_LO,
                             sbase + tl.dslot, 256, true);               // Wh_d (slot)
                        umma::commit(&mbar2);
                    }
                }
                wait_mma(&mbar, phase);
                pc.mark(5);
                if (t >= 1) lpart[c.part][c.row] = head_partial(c, COL_C, comb_b, head_w);
                if (!last) {
                    attn_scores(c, Es, t + 1, COL_Q, att_v, vsum, rawmask, s_part, L);  // causal: j <= t
                    zero_units(c, COL_Q);   // Q accumulates from zero in the next GEMM1
                }
                quad_sync(c.quad);   // the rows' partial scores / head terms
                if (t >= 1 && c.part == 0) {
                    lsum = head_b;
#pragma unroll
                    for (int p = 0; p < PARTS; p++) lsum += lpart[p][c.row];
                    emit_logit(a, chunk, T, t - 1, lsum, true);
                }
                if (last) break;
                pc.mark(6);
                // Z += h Wh_d is long done: swap Wc_d into the slot under the context
                wait_mma(&mbar2, phase2);
                if (c.tid == 0) {
                    umma::mbar_expect_tx(&tma_bar, (uint32_t)tl.img256);
                    tma_piece(smem + tl.dslot, a.blob, tl.phase_off[1] + tl.b_off[5], tl.img256,
                              &tma_bar);
                }
                float ctx[U];
                attn_context(c, Hs, t + 1, s_part, L, vabs, ctx);
                store_operand<SINGLE>(c, A_X_HI, A_X_LO, ctx);
                wait_mma(&tma_bar, tphase);   // Wc_d in the slot
                umma::fence_proxy_async();    // s_part reads done before the TMA overwrites them
                tmem_writes_done();
                // s_part overlays att_dec | Wcomb_h (idle until the next GEMM1): reload
                if (c.tid == 0) {
                    umma::mbar_expect_tx(&tma_bar2, (uint32_t)(2 * tl.img64));
                    tma_piece(smem, a.blob, tl.phase_off[1] + tl.b_off[3], 2 * tl.img64,
                              &tma_bar2);
                }
                pc.mark(7);
                // GEMM2 on ctx_t: Z += ctx Wc (barrier 1, the cell needs it) ;
                // C = ctx Wcomb_c (barrier 2, read by the next step's head)
                if (c.tid == 0) {
                    umma::fence_after();
                    zproduct<SINGLE, kSplitCDec>(c.tbase, c.tbase + A_X_HI, c.tbase + A_X_LO,
                                                 sbase + tl.dslot, true, &mbar, &mbar3);  // Wc_d

                    mma3<SINGLE>(c.tbase + COL_C, c.tbase + A_X_HI, c.tbase + A_X_LO,
                         sbase + 2 * tl.img64, 64, false);               // Wcomb_c
                    umma::commit(&mbar2);
                }
                if (t + 1 < T) {
                    if constexpr (RECMG_GID_AHEAD_D) {
                        const int32_t g1 = gd_ahead;
                        if (t + 2 < T) gd_ahead = __ldg(gid + t + 2);
                        dstage.prefetch(c, pid_dec, g1);
                    } else {
                        dstage.prefetch(c, pid_dec, __ldg(gid + t + 1));
                    }
                }
                wait_mma(&mbar, phase);
                pc.mark(8);
                // Wc_d done (and so every earlier MMA): swap Wh_d back under the cell
                // (the last step's GEMM1 has no Z product, so it is not needed then)
                auto swap_whd = [&] {
                    if (t + 1 < T && c.tid == 0) {
                        umma::mbar_expect_tx(&tma_bar, (uint32_t)tl.img256);
                        tma_piece(smem + tl.dslot, a.blob, tl.phase_off[1] + tl.b_off[2],
                                  tl.img256, &tma_bar);
                    }
                };
                if constexpr (kSplitCDec) {
                    cell<false>(c, nullptr, cs0, h, [&] { wait_mma(&mbar3, phase3); swap_whd(); });
                } else {
                    swap_whd();
                    cell<false>(c, nullptr, cs0, h);
                }
                store_operand<SINGLE>(c, A_H_HI, A_H_LO, h);
                if (t + 1 < T) dstage.commit(c);
            }
        } else {
            zero_operand(c, P_H0_HI, P_H0_LO);
            zero_operand(c, P_H1_HI, P_H1_LO);
            zero_operand(c, P_CTX_HI, P_CTX_LO);
            // One 128 KB weight region at [0, 128 KB) rotates through the step:
            // att_dec | Wcomb_h | Wcomb_c (GEMM1) -> Wctx0 | Wh0 (GEMM2) ->
            // Wx1 | Wh1 (layer 1), each load issued by TMA as soon as the previous
            // occupant's MMAs completed and hidden under the attention / the cells;
            // s_part sits above it, so shared memory is 158 KB (L1 92 KB)
            const int64_t dec_a = tl.phase_off[1];
            for (int t = 0; t <= T; t++) {
                const bool last = (t == T);
                // GEMM1: [comb | Q] = h1 [Wcomb_h | att_dec] into Z[0:128) (one
                // N = 128 product over the stacked image), then comb += ctx Wcomb_c
                pc.mark(3);
                if (t >= 1) wait_mma(&tma_bar2, tphase2);   // att_dec | Wcomb back in the region
                tmem_writes_done();
                pc.mark(4);
                if (c.tid == 0) {
                    umma::fence_after();
                    mma3<SINGLE>(c.tbase + COL_Z, c.tbase + P_H1_HI, c.tbase + P_H1_LO,
                         sbase, 128, false);                             // Wcomb_h | att_dec
                    if (t >= 1)
                        mma3<SINGLE>(c.tbase + COL_Z, c.tbase + P_CTX_HI, c.tbase + P_CTX_LO,
                             sbase + 2 * tl.img64, 64, true);            // Wcomb_c
                    umma::commit(&mbar);
                }
                wait_mma(&mbar, phase);
                // GEMM1 done: Wctx0 | Wh0 into the region under the head and attention
                if (!last && c.tid == 0) {
                    umma::mbar_expect_tx(&tma_bar, (uint32_t)(2 * tl.img256));
                    tma_piece(smem, a.blob, dec_a + tl.b_off[7], 2 * tl.img256, &tma_bar);
                }
                pc.mark(5);
                if (t >= 1) lpart[c.part][c.row] = head_partial(c, COL_Z, comb_b, head_w);
                if (!last) {
                    attn_scores(c, Es, L, COL_Z + 64, att_v, vsum, rawmask, s_part, L);  // non-causal
                }
                quad_sync(c.quad);   // the rows' partial scores / head terms
                if (t >= 1 && c.part == 0) {
                    lsum = head_b;
#pragma unroll
                    for (int p = 0; p < PARTS; p++) lsum += lpart[p][c.row];
                    emit_logit(a, chunk, T, t - 1, lsum, false);
                }
                if (last) break;
                pc.mark(6);
                float ctx[U];
                attn_context(c, Hs, L, s_part, L, vabs, ctx);
                store_operand<SINGLE>(c, P_CTX_HI, P_CTX_LO, ctx);
                // layer 0: Z = slot_proj[t] + ctx Wctx0 + h0 Wh0   (model.py:208-209)
                init_z_from_row(c, slot_proj + t * 256);
                wait_mma(&tma_bar, tphase);                      // Wctx0 | Wh0 in the region
                tmem_writes_done();
                pc.mark(7);
                if (c.tid == 0) {
                    umma::fence_after();
                    zproduct2<SINGLE, kSplitPD0>(c.tbase, c.tbase + P_CTX_HI, c.tbase + P_CTX_LO,
                                                 sbase, true,                       // Wctx0
                                                 c.tbase + P_H0_HI, c.tbase + P_H0_LO,
                                                 sbase + tl.img256, &mbar, &mbar3);  // Wh0
                }
                wait_mma(&mbar, phase);
                pc.mark(8);
                cell<false>(c, nullptr, cs0, h, [&] {
                    wait_mma(&mbar3, phase3);
                    // GEMM2 done: DEC-B (Wx1 | Wh1) into the region under the layer-0 cell
                    if (c.tid == 0) {
                        umma::mbar_expect_tx(&tma_bar, (uint32_t)tl.phase_len[2]);
                        tma_piece(smem, a.blob, tl.phase_off[2], tl.phase_len[2], &tma_bar);
                    }
                });
                store_operand<SINGLE>(c, P_H0_HI, P_H0_LO, h);
                // layer 1 (DEC-B weights): Z = h0 Wx1 + h1 Wh1 (+ b1)
                pc.mark(9);
                wait_mma(&tma_bar, tphase);
                tmem_writes_done();
                if (c.tid == 0) {
                    umma::fence_after();
                    zproduct2<SINGLE, kSplitPD1>(c.tbase, c.tbase + P_H0_HI, c.tbase + P_H0_LO,
                                                 sbase + tl.b_off[9], false,
                                                 c.tbase + P_H1_HI, c.tbase + P_H1_LO,
                                                 sbase + tl.b_off[10], &mbar, &mbar3);
                }
                pc.mark(10);
                wait_mma(&mbar, phase);
                pc.mark(11);
                cell<true>(c, dec_b1, cs1, h, [&] {
                    wait_mma(&mbar3, phase3);
                    // layer 1 done: att_dec | Wcomb back for the next step's GEMM1
                    if (c.tid == 0) {
                        umma::mbar_expect_tx(&tma_bar2, (uint32_t)(3 * tl.img64));
                        tma_piece(smem, a.blob, dec_a + tl.b_off[4], 3 * tl.img64, &tma_bar2);
                    }
                });
                store_operand<SINGLE>(c, P_H1_HI, P_H1_LO, h);
            }
        }
        // progress signal for a consumer on another stream (recmg_wait_progress):
        // every thread's outputs of this tile are made visible device-wide, then
        // one arrival per tile is released on its piece's counter
        if (a.progress) __threadfence();
        __syncthreads();
        if (c.tid == 0) {
            if (a.progress) {
                const int64_t piece = tile / a.piece_tiles;
                asm volatile("red.release.gpu.global.add.s32 [%0], 1;"
                             ::"l"(a.progress + piece) : "memory");
            }
            s_tile = atomicAdd(a.tile_counter, 1);
        }
        __syncthreads();
        tile = s_tile;
    }
    if (PROF && c.tid == 0) pc.flush(a.prof + blockIdx.x * 16);
    umma::fence_before();
    __syncthreads();
    if (c.warp == 0) umma::tmem_free<512>(c.tbase);
}

// ---------------------------------------------------------------------------
// packing: B images (fp16 hi/lo, core-matrix layout) and the folded token tables
namespace {

struct BSpec {
    int64_t src;      // float offset in the raw blob of W[k0][0]
    int64_t ld;       // row stride of W (floats)
    int N;            // output columns
    int gates;        // 1: B row n = 4j+g reads W column g*d+j, scaled by gate_scale(g);
                      // 0: identity; 2: identity, scaled by 2 log2(e) (W_comb: the head's
                      // tanh denominators then need no FMUL)
    int64_t dst;      // byte offset of the hi image in the TC blob
    int row0 = 0;     // first B row written (several matrices stacked along N in one image)
    int img_n = 0;    // N of the whole image (lo image at dst + img_n * 128); 0 = N
};

__global__ void bimage_kernel(const float *raw, uint8_t *out, BSpec s, int d) {
    const int64_t total = (int64_t)s.N * 64;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int n = (int)(i / 64), k = (int)(i % 64);
        const int col = s.gates == 1 ? ((n & 3) * d + (n >> 2)) : n;
        const float w = raw[s.src + (int64_t)k * s.ld + col] *
                        (s.gates == 1 ? gate_scale(n & 3) : s.gates == 2 ? 2.0f * kLog2e : 1.0f);
        const __half hi = __float2half_rn(w);
        const __half lo = __float2half_rn(w - __half2float(hi));
        const uint32_t off = umma::kmajor_offset(n + s.row0, k, 64);
        const int64_t img_n = s.img_n ? s.img_n : s.N;
        *reinterpret_cast<__half *>(out + s.dst + off) = hi;
        *reinterpret_cast<__half *>(out + s.dst + img_n * 128 + off) = lo;
    }
}

// out[r][4j+g] = bias[g*d+j] + sum_k E[r][k] W[k][g*d+j]
//                             + sum_k Et[tab(r)][k] Wt[k][g*d+j]      (fp32)
// i.e. the whole layer-0 token projection [E_id[r]; E_tab[tab(r)]] @ Wx + b
// of model.py:105,148-153 for every id r, tab(r) = searchsorted(offsets, r).
__global__ void proj_fold_kernel(const float *E, int64_t rows, int d, const float *W,
                                 const float *Et, const float *Wt, const int64_t *offsets,
                                 int n_tables, const float *bias, float *out) {
    extern __shared__ float e_s[];  // [32][2d]
    const int n = threadIdx.x;       // 0..4d-1
    const int j = n >> 2, g = n & 3;
    const int col = g * d + j;
    for (int64_t r0 = (int64_t)blockIdx.x * 32; r0 < rows; r0 += (int64_t)gridDim.x * 32) {
        __syncthreads();
        for (int i = threadIdx.x; i < 32 * d; i += blockDim.x) {
            const int64_t r = r0 + i / d;
            float e = 0.0f, et = 0.0f;
            if (r < rows) {
                e = E[r * d + (i % d)];
                int lo = 0, hi = n_tables;   // offsets[lo] <= r < offsets[hi]
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (offsets[mid] <= r) lo = mid; else hi = mid;
                }
                et = Et[(int64_t)lo * d + (i % d)];
            }
            e_s[(i / d) * 2 * d + (i % d)] = e;
            e_s[(i / d) * 2 * d + d + (i % d)] = et;
        }
        __syncthreads();
        float acc[32];
        const float b = bias[col];
#pragma unroll
        for (int q = 0; q < 32; q++) acc[q] = b;
        for (int k = 0; k < d; k++) {
            const float w = __ldg(W + (int64_t)k * 4 * d + col);
            const float wt = __ldg(Wt + (int64_t)k * 4 * d + col);
#pragma unroll
            for (int q = 0; q < 32; q++) acc[q] += e_s[q * 2 * d + k] * w + e_s[q * 2 * d + d + k] * wt;
        }
#pragma unroll
        for (int q = 0; q < 32; q++)
            if (r0 + q < rows) out[(r0 + q) * 4 * d + n] = acc[q] * gate_scale(g);
    }
}

}  // namespace

bool tc_supported(const recmg_model_shape *m) {
    return shape_ok(m) && m->dim == 64 && m->l_in <= 16 && m->l_out <= 16 &&
           ((m->kind == RECMG_MODEL_CACHING && m->stacks == 1) ||
            (m->kind == RECMG_MODEL_PREFETCH && m->stacks == 2));
}

TcLayout tc_layout(const recmg_model_shape *m) {
    TcLayout t{};
    const int64_t V = m->total_ids, T = m->n_tables;
    int64_t o = 0;
    auto img = [&](int N) { int64_t r = o; o += (int64_t)N * 256; return r; };  // hi+lo bytes
    if (m->kind == RECMG_MODEL_CACHING) {
        // ENC {Wh_e, att_enc} | DEC {Wh_d, att_dec, Wcomb_h, Wc_d, Wcomb_c}
        t.phase_off[0] = o;
        t.b_off[0] = img(256) - t.phase_off[0];
        t.b_off[1] = img(64) - t.phase_off[0];
        t.phase_len[0] = o - t.phase_off[0];
        t.phase_off[1] = o;
        t.b_off[2] = img(256) - t.phase_off[1];
        t.b_off[3] = img(64) - t.phase_off[1];
        t.b_off[4] = img(64) - t.phase_off[1];
        t.b_off[5] = img(256) - t.phase_off[1];
        t.b_off[6] = img(64) - t.phase_off[1];
        t.phase_len[1] = o - t.phase_off[1];
        t.nb = 7;
    } else {
        // ENC {Wh0, Wx1, Wh1, att_enc} | DEC-A {att_dec, Wcomb_h, Wcomb_c, Wctx0, Wh0}
        // | DEC-B {Wx1, Wh1}
        t.phase_off[0] = o;
        t.b_off[0] = img(256) - t.phase_off[0];
        t.b_off[1] = img(256) - t.phase_off[0];
        t.b_off[2] = img(256) - t.phase_off[0];
        t.b_off[3] = img(64) - t.phase_off[0];
        t.phase_len[0] = o - t.phase_off[0];
        t.phase_off[1] = o;
        t.b_off[4] = img(64) - t.phase_off[1];
        t.b_off[5] = img(64) - t.phase_off[1];
        t.b_off[6] = img(64) - t.phase_off[1];
        t.b_off[7] = img(256) - t.phase_off[1];
        t.b_off[8] = img(256) - t.phase_off[1];
        t.phase_len[1] = o - t.phase_off[1];
        t.phase_off[2] = o;
        t.b_off[9] = img(256) - t.phase_off[2];
        t.b_off[10] = img(256) - t.phase_off[2];
        t.phase_len[2] = o - t.phase_off[2];
        t.nb = 11;
        t.swap_off = t.b_off[7];   // DEC-B swaps in over Wctx0 | Wh0
        if (t.phase_len[1] - t.swap_off != t.phase_len[2]) t.swap_off = -1;  // (never)
    }
    o = (o + 255) / 256 * 256;
    const int ntab = m->kind == RECMG_MODEL_CACHING ? 2 : 1;
    for (int i = 0; i < 2; i++) {
        if (i < ntab) {
            t.pid[i] = o; o += V * 256 * 4;
            o = (o + 255) / 256 * 256;
        } else {
            t.pid[i] = t.pid[0];
        }
    }
    (void)T;
    const size_t spart = (size_t)(m->kind == RECMG_MODEL_CACHING ? PartsOf<RECMG_MODEL_CACHING>::value : PartsOf<RECMG_MODEL_PREFETCH>::value) * m->l_in * 128 * 4;
    t.spart_off = 176 * 1024;
    t.img64 = 64 * 256;
    t.img256 = 256 * 256;
    t.dslot = 3 * t.img64;
    // caching: the partial scores overlay att_dec | Wcomb_h (reloaded each step)
    if (m->kind == RECMG_MODEL_CACHING) t.spart_off = 0;
    // prefetch: encoder Wh1 | att_enc | slot (144 KB); decoder DEC-A (176 KB) with
    // s_part overlaying att_dec | Wcomb_h | Wcomb_c, reloaded every step
    t.eslot = t.img256 + t.img64;
    if (m->kind == RECMG_MODEL_PREFETCH) t.spart_off = (size_t)(2 * t.img256);   // 128 KB
    size_t wmax = 0;
    for (int i = 0; i < 3; i++) wmax = wmax > (size_t)t.phase_len[i] ? wmax : (size_t)t.phase_len[i];
    if (m->kind == RECMG_MODEL_CACHING)   // encoder 80 KB, decoder 112 KB (R1 + slot)
        wmax = (size_t)(t.dslot + t.img256) > (size_t)t.phase_len[0] ? (size_t)(t.dslot + t.img256)
                                                                     : (size_t)t.phase_len[0];
    if (m->kind == RECMG_MODEL_PREFETCH) wmax = (size_t)(t.eslot + t.img256);   // encoder 144 KB
    t.smem_bytes = wmax > t.spart_off + spart ? wmax : t.spart_off + spart;
    // per-unit constants (lstm_tc_kernel: biases, att_v, comb_b, head_w, slot_proj)
    t.const_off = (t.smem_bytes + 15) / 16 * 16;
    t.smem_bytes = t.const_off + (size_t)(704 + (m->kind == RECMG_MODEL_CACHING ? 0 : m->l_out * 256)) * 4;
    t.total = o;
    return t;
}

// x[i] *= gate_scale(i & 3) over gate-interleaved [.][4d] rows
__global__ void gate_scale_kernel(float *x, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        x[i] *= gate_scale((int)(i & 3));
}

__global__ void scale_kernel(float *x, int64_t n, float sc) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        x[i] *= sc;
}

int model_pack_tc(const recmg_model_shape *m, const float *raw, const float *embed_id,
                  const int64_t *offsets, void *packed_dense, void *tc_blob, cudaStream_t s) {
    int rc = model_pack(m, raw, packed_dense, s);
    if (rc) return rc;
    {   // the gate rows the TC kernels read from the dense blob: layer >= 1
        // biases (added in the cell) and the prefetch slot projections (Z init)
        const PackedLayout p = packed_layout(m);
        float *dense = (float *)packed_dense;
        for (int k = 1; k < m->stacks; k++) {
            gate_scale_kernel<<<1, 256, 0, s>>>(dense + p.enc_b[k], 4 * m->dim);
            RECMG_LAUNCH_CHECK();
            gate_scale_kernel<<<1, 256, 0, s>>>(dense + p.dec_b[k], 4 * m->dim);
            RECMG_LAUNCH_CHECK();
        }
        if (m->kind == RECMG_MODEL_PREFETCH) {
            gate_scale_kernel<<<4, 256, 0, s>>>(dense + p.slot_proj, (int64_t)m->l_out * 4 * m->dim);
            RECMG_LAUNCH_CHECK();
        }
        scale_kernel<<<1, 64, 0, s>>>(dense + p.comb_b, m->dim, 2.0f * kLog2e);   // head bias
        RECMG_LAUNCH_CHECK();
    }
    const RawLayout r = raw_layout(m);
    const TcLayout t = tc_layout(m);
    const int d = m->dim;
    uint8_t *out = (uint8_t *)tc_blob;
    std::vector<BSpec> specs;
    auto spec = [&](int phase, int b, int64_t src, int64_t ld, int N, int gates) {
        BSpec x{src, ld, N, gates, t.phase_off[phase] + t.b_off[b]};
        specs.push_back(x);
    };
    if (m->kind == RECMG_MODEL_CACHING) {
        spec(0, 0, r.enc_wh[0], 4 * d, 256, 1);
        spec(0, 1, r.att_enc, d, 64, 0);
        spec(1, 2, r.dec_wh[0], 4 * d, 256, 1);
        // att_dec | Wcomb_h (rows 0..d-1: the h part) stacked as one N = 128 image
        spec(1, 3, r.att_dec, d, 64, 0);
        specs.back().img_n = 128;
        spec(1, 3, r.comb_w, d, 64, 2);
        specs.back().row0 = 64;
        specs.back().img_n = 128;
        spec(1, 5, r.dec_wx[0] + 2 * d * 4 * d, 4 * d, 256, 1); // rows 2d..3d-1: ctx part
        spec(1, 6, r.comb_w + d * d, d, 64, 2);               // rows d..2d-1: ctx part
    } else {
        spec(0, 0, r.enc_wh[0], 4 * d, 256, 1);
        spec(0, 1, r.enc_wx[1], 4 * d, 256, 1);
        spec(0, 2, r.enc_wh[1], 4 * d, 256, 1);
        spec(0, 3, r.att_enc, d, 64, 0);
        // Wcomb_h (h part) | att_dec stacked as one N = 128 image at b_off[4]
        spec(1, 4, r.comb_w, d, 64, 2);
        specs.back().img_n = 128;
        spec(1, 4, r.att_dec, d, 64, 0);
        specs.back().row0 = 64;
        specs.back().img_n = 128;
        spec(1, 6, r.comb_w + d * d, d, 64, 2);
        spec(1, 7, r.dec_wx[0] + 2 * d * 4 * d, 4 * d, 256, 1);
        spec(1, 8, r.dec_wh[0], 4 * d, 256, 1);
        spec(2, 9, r.dec_wx[1], 4 * d, 256, 1);
        spec(2, 10, r.dec_wh[1], 4 * d, 256, 1);
    }
    for (const BSpec &x : specs) {
        bimage_kernel<<<64, 256, 0, s>>>(raw, out, x, d);
        RECMG_LAUNCH_CHECK();
    }
    // folded token tables: P[r] = [E_id[r]; E_tab[tab(r)]] @ Wx[0:2d] + b
    const int ntab = m->kind == RECMG_MODEL_CACHING ? 2 : 1;
    for (int i = 0; i < ntab; i++) {
        const int64_t wx = (i == 0) ? r.enc_wx[0] : r.dec_wx[0];
        const int64_t bb = (i == 0) ? r.enc_b[0] : r.dec_b[0];
        const int64_t blocks = imin64((m->total_ids + 31) / 32, 64 * kSmCount);
        proj_fold_kernel<<<(unsigned)blocks, 4 * d, 2 * 32 * d * 4, s>>>(
            embed_id, m->total_ids, d, raw + wx, raw + r.embed_table,
            raw + wx + (int64_t)d * 4 * d, offsets, m->n_tables, raw + bb,
            (float *)(out + t.pid[i]));
        RECMG_LAUNCH_CHECK();
    }
    return RECMG_OK;
}

static int g_model_sm_budget = kSmCount;

int model_sm_budget() { return g_model_sm_budget; }
int set_model_sm_budget(int n) {
    const int prev = g_model_sm_budget;
    g_model_sm_budget = n < 1 ? 1 : (n > kSmCount ? kSmCount : n);
    return prev;
}

int model_forward_tc(const recmg_model_shape *m, const void *packed_dense, const void *tc_blob,
                     const int32_t *gid, const int32_t *tid, int64_t batch, float *logits,
                     uint8_t *bits, int32_t *pf_gid, void *ws, size_t ws_bytes, cudaStream_t s,
                     long long *prof, int64_t decode_ids, bool single, int32_t *progress,
                     int64_t piece_chunks) {
    if (batch <= 0) return RECMG_OK;
    if (progress && (piece_chunks <= 0 || piece_chunks % 128 != 0)) return RECMG_E_INVALID_CONFIG;
    const int64_t n_tiles = (batch + 127) / 128;
    const int grid = (int)imin64(n_tiles, g_model_sm_budget);
    if (ws_bytes < tc_workspace_bytes(m, batch)) return RECMG_E_WORKSPACE;
    TcArgs a;
    a.m = *m;
    a.tl = tc_layout(m);
    a.pl = packed_layout(m);
    if (decode_ids > 0) a.m.total_ids = decode_ids;   // decode scale only (table shards)
    a.blob = (const uint8_t *)tc_blob;
    a.dense = (const float *)packed_dense;
    a.gid = gid;
    a.tid = tid;
    a.batch = batch;
    a.logits = logits;
    a.bits = bits;
    a.pf_gid = pf_gid;
    a.tile_counter = (int *)ws;
    a.progress = progress;
    a.piece_tiles = progress ? piece_chunks / 128 : 1;
    a.scratch = (float *)((char *)ws + 256);
    RECMG_CUDA_TRY(cudaMemsetAsync(a.tile_counter, 0, sizeof(int), s));
    a.prof = prof;
    const int smem = (int)a.tl.smem_bytes;
#define RECMG_TC_LAUNCH(K, P)                                                                 \
    do {                                                                                      \
        RECMG_CUDA_TRY(cudaFuncSetAttribute(lstm_tc_kernel<K, P>,                             \
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); \
        lstm_tc_kernel<K, P><<<grid, 128 * PartsOf<K>::value, smem, s>>>(a);                   \
    } while (0)
    if (m->kind == RECMG_MODEL_CACHING) {
        if (prof) RECMG_TC_LAUNCH(RECMG_MODEL_CACHING, 1);
        else if (single) RECMG_TC_LAUNCH(RECMG_MODEL_CACHING, 2);
        else RECMG_TC_LAUNCH(RECMG_MODEL_CACHING, 0);
    } else {
        if (prof) RECMG_TC_LAUNCH(RECMG_MODEL_PREFETCH, 1);
        else if (single) RECMG_TC_LAUNCH(RECMG_MODEL_PREFETCH, 2);
        else RECMG_TC_LAUNCH(RECMG_MODEL_PREFETCH, 0);
    }
#undef RECMG_TC_LAUNCH
    RECMG_LAUNCH_CHECK();
    return RECMG_OK;
}

__global__ void wait_progress_kernel(const int32_t *p, int32_t target) {
    for (;;) {
        int32_t v;
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
        if (v >= target) break;
        __nanosleep(500);
    }
}

int wait_progress(const int32_t *progress, int32_t target, cudaStream_t s) {
    wait_progress_kernel<<<1, 1, 0, s>>>(progress, target);
    RECMG_LAUNCH_CHECK();
    return RECMG_OK;
}

size_t tc_workspace_bytes(const recmg_model_shape *m, int64_t batch) {
    const int64_t n_tiles = (batch + 127) / 128;
    const int64_t grid = imin64(n_tiles > 0 ? n_tiles : 1, kSmCount);
    return 256 + (size_t)grid * 2 * m->l_in * 128 * 64 * sizeof(float);
}

}  // namespace recmg
