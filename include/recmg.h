/*
 * recmg.h — C ABI of the B200-native RecMG hot path (paper_2511_08568_b200).
 *
 * The reference (arxiv 2511.08568 `embcache`, /root/reference/pkg/src/embcache)
 * is pure Python + numpy and has no FFI; each entry point below replaces the
 * Python function cited beside it, with the same argument meaning and the
 * same error categories (errors.py), expressed as status codes.  The binding
 * a maintainer would add on the reference side is in INTEGRATION.md.
 *
 * Conventions
 *   - All array pointers are DEVICE pointers unless the name says `host`.
 *   - Every call is stream-ordered on `stream` (a cudaStream_t, NULL = legacy
 *     default stream); no call synchronises, allocates, or keeps hidden state.
 *     Scratch comes from a caller-owned workspace sized by *_workspace_bytes.
 *   - Buffer state (the GPU embedding-buffer metadata) is caller-owned device
 *     memory of recmg_buffer_state_bytes(); recmg_buffer_reset() empties it.
 *     Replays continue from whatever state they are given, so a trace can be
 *     replayed batch by batch.
 *   - Global ids are int32 (every configured vocabulary is < 2^30 ids).
 */
#ifndef RECMG_H
#define RECMG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: one per errors.py category on this path ------------ */
typedef enum {
    RECMG_OK = 0,
    RECMG_E_INVALID_CONFIG = -1, /* InvalidConfigError   errors.py:15-18      */
    RECMG_E_VOCAB_MISMATCH = -2, /* VocabularyMismatchError errors.py:51-54   */
    RECMG_E_OUT_OF_VOCAB = -3,   /* OutOfVocabularyError errors.py:57-60      */
    RECMG_E_BUFFER_STATE = -4,   /* ValueError / KeyError raised by
                                    PriorityBuffer (runtime.py:69-70,79-80,
                                    85-88,104) and load_embeddings (:124-128) */
    RECMG_E_NON_FINITE = -5,     /* NumericalError errors.py:75-78            */
    RECMG_E_CUDA = -6,           /* CUDA launch / runtime failure             */
    RECMG_E_WORKSPACE = -7       /* workspace smaller than *_workspace_bytes   */
} recmg_status;

const char *recmg_status_string(int status);
/* "error" category string of errors.py for a status (e.g. "invalid-config") */
const char *recmg_status_category(int status);

/* ---- buffer configuration --------------------------------------------- */
enum { RECMG_POLICY_PRIORITY = 0, /* Alg. 1/2 priority-decay buffer (runtime.py:41-141) */
       RECMG_POLICY_LRU = 1,      /* LRU comparator (cache_sim.py:92-106)              */
       RECMG_POLICY_LRU_PF = 2,   /* LRU + prefetch tags: replay_policy_only with a
                                     prefetcher (runtime.py:304-349); recmg_replay
                                     ignores the bits                             */
       RECMG_POLICY_LFU = 3,      /* cache_sim.py:109-137 (ties -> least recent)   */
       RECMG_POLICY_SRRIP = 4,    /* cache_sim.py:140-170; max rrpv in
                                     eviction_speed                                */
       RECMG_POLICY_OPTGEN = 5 }; /* Belady / optgen, cache_sim.py:173-249          */

typedef struct {
    int64_t capacity;       /* BufferConfig.capacity (runtime.py:29-38) /
                               CacheConfig.capacity (cache_sim.py:30-58)          */
    int32_t ways;           /* 0 = fully associative (the reference buffer);
                               >0 = ways per set, set = gid % (capacity/ways)     */
    int32_t eviction_speed; /* BufferConfig.eviction_speed, default 4             */
    int32_t policy;         /* RECMG_POLICY_*                                     */
    int32_t reserved;
    int64_t total_ids;      /* Trace.total_ids (trace.py:75-77)                   */
} recmg_buffer_cfg;

/* Counters of one replay; cache_hits..prefetch_useful are BreakdownReport's
 * integer fields (runtime.py:153-162), the rest are the spy-visible counts
 * (populate calls, prefetched add calls, resident count at the end).       */
typedef struct {
    int64_t cache_hits;
    int64_t prefetch_hits;
    int64_t on_demand;
    int64_t prefetch_issued;
    int64_t prefetch_useful;
    int64_t evictions;
    int64_t prefetch_inserts;
    int64_t occupancy;
} recmg_counters;

/* Bytes of device state for `cfg` (tags, priorities/tags or LRU clocks,
 * per-set counts, and for sets wider than 32 ways an id->slot map over
 * total_ids).  Replaces PriorityBuffer.__init__ (runtime.py:48-56).          */
size_t recmg_buffer_state_bytes(const recmg_buffer_cfg *cfg);
/* Empty the buffer.  Validation = BufferConfig.validate (runtime.py:34-38)
 * and CacheConfig.validate (cache_sim.py:43-50).                            */
int recmg_buffer_reset(const recmg_buffer_cfg *cfg, void *state, void *stream);

/* ---- chunked replay through the buffer  (runtime.py:220-283) ----------- */
/* Number of chunks chunk() emits (trace.py:226-250).                        */
int64_t recmg_num_chunks(int64_t n, int32_t l_in, int32_t l_out, int32_t window_ratio);

int recmg_replay_workspace_bytes(const recmg_buffer_cfg *cfg, int64_t n, int32_t l_in,
                                 int32_t l_out, int32_t window_ratio, int32_t pf_stride,
                                 size_t *bytes);
/*
 * replay (runtime.py:220-283) with the model decisions already computed:
 *   gids[n]            Trace.gid_array
 *   bits[K*l_in]       caching bits 0/1 (runtime.py:181-193); NULL = all 0
 *                      (caching_params None, runtime.py:184-185)
 *   pf[K*pf_stride]    prefetch gids per chunk, -1 padded (runtime.py:196-210);
 *                      NULL = no prefetcher
 *   counters           device recmg_counters, ACCUMULATED into (zero it first)
 *   cov_num, cov_den   device uint16[K] (nullable): |set(P_k) & set(W_k)| and
 *                      |set(W_k)| so the host can form the float64 coverage in
 *                      chunk order (runtime.py:276,282) via recmg_coverage_mean
 *   access_class[n]    nullable: 0 cache hit, 1 prefetch hit, 2 on-demand
 * Status: RECMG_E_INVALID_CONFIG for a bad cfg / l_in / l_out / window_ratio
 * (trace.py:233-236).  Bits must be 0/1: the model path only emits 0/1, and
 * the host mirror rejects other caching_fn output with ValueError before
 * any launch (runtime.py:124-128); a nonzero byte here is read as 1.
 */
int recmg_replay(const recmg_buffer_cfg *cfg, void *state, const int32_t *gids, int64_t n,
                 int32_t l_in, int32_t l_out, int32_t window_ratio, const uint8_t *bits,
                 const int32_t *pf, int32_t pf_stride, recmg_counters *counters,
                 uint16_t *cov_num, uint16_t *cov_den, uint8_t *access_class, void *ws,
                 size_t ws_bytes, void *stream);

/* The same replay over chunks [k_begin, k_end) only (k_end = -1: all), with
 * the tail accesses appended when with_tail (requires k_end = last chunk).
 * Consecutive ranges on one state reproduce recmg_replay exactly, so a trace
 * can be replayed piece by piece while later pieces are still being scored.
 * bits / pf / cov_* / access_class are indexed globally (chunk k, access i). */
int recmg_replay_chunks(const recmg_buffer_cfg *cfg, void *state, const int32_t *gids, int64_t n,
                        int32_t l_in, int32_t l_out, int32_t window_ratio, int64_t k_begin,
                        int64_t k_end, int32_t with_tail, const uint8_t *bits, const int32_t *pf,
                        int32_t pf_stride, recmg_counters *counters, uint16_t *cov_num,
                        uint16_t *cov_den, uint8_t *access_class, void *ws, size_t ws_bytes,
                        void *stream);

/* recmg_replay_chunks with flags.  RECMG_REPLAY_SKIP_STATS: the per-chunk
 * prefetch statistics (prefetch_issued / prefetch_useful and the coverage
 * counts of runtime.py:271-276) of this range were already produced by
 * recmg_prefetch_stats, so only the buffer replay runs.                     */
#define RECMG_REPLAY_SKIP_STATS 1
int recmg_replay_chunks_ex(const recmg_buffer_cfg *cfg, void *state, const int32_t *gids,
                           int64_t n, int32_t l_in, int32_t l_out, int32_t window_ratio,
                           int64_t k_begin, int64_t k_end, int32_t with_tail, const uint8_t *bits,
                           const int32_t *pf, int32_t pf_stride, recmg_counters *counters,
                           uint16_t *cov_num, uint16_t *cov_den, uint8_t *access_class,
                           void *ws, size_t ws_bytes, int32_t flags, void *stream);
/* recmg_replay_chunks_ex with the 32-way LRU comparator (cache_sim.py:92-106,
 * simulate() over the same accesses) fused into the same launch: it replays
 * the serves of the priority replay's own partitioned events (both buffers
 * have the same sets), so it needs no event build or partition of its own.
 * lru_cfg: policy RECMG_POLICY_LRU, the same sets, ways (<= 32) and total_ids
 * as cfg; lru_state its state (recmg_buffer_reset), lru_hits_misses [2] int64
 * accumulates (hits, misses) like recmg_simulate_ex's.  No access classes.
 * RECMG_E_INVALID_CONFIG when the geometries differ (run recmg_simulate_ex). */
int recmg_replay_chunks_lru(const recmg_buffer_cfg *cfg, void *state, const int32_t *gids,
                            int64_t n, int32_t l_in, int32_t l_out, int32_t window_ratio,
                            int64_t k_begin, int64_t k_end, int32_t with_tail,
                            const uint8_t *bits, const int32_t *pf, int32_t pf_stride,
                            recmg_counters *counters, uint16_t *cov_num, uint16_t *cov_den,
                            const recmg_buffer_cfg *lru_cfg, void *lru_state,
                            int64_t *lru_hits_misses, void *ws, size_t ws_bytes, int32_t flags,
                            void *stream);
/* The prefetch statistics of chunks [k_begin, k_end) alone: they depend only
 * on the ids and the decoded prefetch ids (runtime.py:271-276), not on the
 * buffer, so they can run as soon as the prefetch forward is done.          */
int recmg_prefetch_stats(const int32_t *gids, int64_t n, int32_t l_in, int32_t l_out,
                         int32_t window_ratio, int64_t k_begin, int64_t k_end, const int32_t *pf,
                         int32_t pf_stride, recmg_counters *counters, uint16_t *cov_num,
                         uint16_t *cov_den, void *stream);

/* Host: sequential float64 mean of num/den in chunk order (runtime.py:276,282). */
double recmg_coverage_mean(const uint16_t *host_num, const uint16_t *host_den, int64_t K);
/* Host: acc + the same left-to-right float64 sum over `count` chunks, for
 * summing the coverage piece by piece in chunk order as pieces complete.    */
double recmg_coverage_accumulate(const uint16_t *host_num, const uint16_t *host_den, int64_t count,
                                 double acc);

/* ---- policy-only simulation  (cache_sim.py:223-260, LRU) --------------- */
int recmg_simulate_workspace_bytes(const recmg_buffer_cfg *cfg, int64_t n, size_t *bytes);
/* simulate(trace, CacheConfig(capacity, policy, ways)) for LRU, and for
 * LFU / SRRIP / OPTGEN, any ways per set (sets wider than 4096 ways keep
 * their ways in global memory, one CTA per set): hits/misses
 * accumulated into device int64[2]; per_access_hit[n] (nullable) as
 * SimResult.per_access_hit.  Use recmg_simulate_ex for OPTGEN keep bits.    */
int recmg_simulate(const recmg_buffer_cfg *cfg, void *state, const int32_t *gids, int64_t n,
                   uint8_t *per_access_hit, int64_t *hits_misses, void *ws, size_t ws_bytes,
                   void *stream);

/* As recmg_simulate, plus keep_decisions[n] (OPTGEN only, nullable):
 * SimResult.keep_decisions of simulate_optgen (cache_sim.py:199-220).       */
int recmg_simulate_ex(const recmg_buffer_cfg *cfg, void *state, const int32_t *gids, int64_t n,
                      uint8_t *per_access_hit, uint8_t *keep_decisions, int64_t *hits_misses,
                      void *ws, size_t ws_bytes, void *stream);

/* ---- single buffer operations (PriorityBuffer object API) -------------- */
enum {
    RECMG_OP_ADD = 0,          /* add(gid, arg=priority, flag=prefetched) runtime.py:83-91 */
    RECMG_OP_POPULATE = 1,     /* populate() -> victim gid              runtime.py:100-112 */
    RECMG_OP_REFERENCE = 2,    /* reference(gid) -> 0/1                 runtime.py:93-98   */
    RECMG_OP_SET_PRIORITY = 3, /* set_priority(gid, arg)                runtime.py:78-81   */
    RECMG_OP_QUERY = 4         /* -> resident ? priority : -1           runtime.py:61-71   */
};
/* result: device int64[2] = {status (0 or RECMG_E_BUFFER_STATE), value}.   */
int recmg_buffer_op(const recmg_buffer_cfg *cfg, void *state, int32_t op, int64_t gid,
                    int64_t arg, int32_t flag, int64_t *result, void *stream);

/* ---- embedding rows: host gathers (K5) and EmbeddingBag pooling (K6) ---- */
/* Not in the reference; parity = torch embedding_bag(sum).
 * host_rows: [total_ids x dim] fp32 in pinned, mapped host memory (UVA);
 * buf_rows: [capacity x dim] fp32 in HBM, row = buffer slot (set*ways+way);
 * loaded: int32 [capacity], the id whose row each slot holds (-1 = none).  */
/* Copy the row of every slot whose occupant changed since the last refresh
 * (zero-copy PCIe reads); *copied (device int64) += rows copied.  ways <= 32. */
int recmg_rows_refresh(const recmg_buffer_cfg *cfg, const void *state, int32_t *loaded,
                       const float *host_rows, int32_t dim, float *buf_rows, int64_t *copied,
                       void *stream);
/* out[b] = sum of the rows of gids[bag_offsets[b] .. bag_offsets[b+1]) in
 * order; each row read from its HBM slot when resident, else from host
 * memory.  src_counts (device int64[2], nullable) += {from HBM, from host}. */
int recmg_embedding_bag(const recmg_buffer_cfg *cfg, const void *state, const int32_t *gids,
                        const int64_t *bag_offsets, int64_t n_bags, const float *buf_rows,
                        const float *host_rows, int32_t dim, float *out, int64_t *src_counts,
                        void *stream);

/* ---- K7 fused: pooled all-to-all over NVLink peer memory (DLRM mode) --- */
/* EmbeddingBag(sum) of n_bags = batch x Tg bags (bag b*Tg + j = sample b,
 * local table j) whose epilogue stores each pooled row directly into the
 * receiving rank's output: sample b goes to rank b / (batch/world), row
 * [b % (batch/world)][table_global[j]] of that rank's [batch/world, n_tables,
 * dim] buffer (peer_out[rank'] = its CUDA-IPC-mapped pointer).  The last
 * block then publishes `epoch` (> every earlier epoch) into slot [rank] of
 * every receiver's flag array (peer_flags[rank']) at system scope, and the
 * stream waits until all `world` slots of this rank's `flags` reach `epoch`:
 * after the call (stream order) this rank's output holds every table's
 * pooled row for its samples.  flags: world uint64 + one uint32 counter,
 * zero-initialised (recmg_peer_alloc).  Replaces pooling + all_to_all_single. */
int recmg_embedding_bag_a2a(const recmg_buffer_cfg *cfg, const void *state, const int32_t *gids,
                            const int64_t *bag_offsets, int64_t n_bags, const float *buf_rows,
                            const float *host_rows, int32_t dim, int32_t batch, int32_t world,
                            int32_t rank, int32_t n_tables, const int32_t *table_global,
                            float *const *peer_out, unsigned long long *const *peer_flags,
                            unsigned long long *flags, uint64_t epoch, int64_t *src_counts,
                            void *stream);
/* Peer memory for the exchange: a dedicated zeroed cudaMalloc, its CUDA IPC
 * handle (64 bytes, host), and its mapping in another rank's process.       */
int recmg_peer_alloc(size_t bytes, void **dev_ptr);
int recmg_peer_free(void *dev_ptr);
int recmg_peer_handle(void *dev_ptr, uint8_t *host_handle64);
int recmg_peer_open(const uint8_t *host_handle64, void **dev_ptr);
int recmg_peer_close(void *dev_ptr);

/* ---- models  (neural/model.py) ----------------------------------------- */
enum { RECMG_MODEL_CACHING = 0, RECMG_MODEL_PREFETCH = 1 };
enum {
    RECMG_PREC_FP32 = 0, /* SIMT: fp32 weights, fp32 FMA, any dim <= 64            */
    RECMG_PREC_TC32 = 1, /* tcgen05: every GEMM as the fp16 hi/lo 3-product split
                            with fp32 accumulation in TMEM (fp32-class logits);
                            dim 64, l_in/l_out <= 16, 1 (caching) / 2 (prefetch)
                            stacks; token projection folded into per-id tables   */
    RECMG_PREC_TC16 = 2  /* reduced-precision variant of TC32 (the north star's
                            "bf16 variant, reported separately"): ONE fp16 product
                            per GEMM (x_hi * w_hi), same packed weights and
                            kernels; logits ~1e-3..1e-1 off, decisions reported
                            as agreement rates against TC32                    */
};

typedef struct {
    int32_t kind;      /* ModelParameters.kind (model.py:28-38)   */
    int32_t dim;       /* d                                       */
    int32_t stacks;    /* LSTM layers per encoder/decoder         */
    int32_t l_in;      /* input chunk length (15)                 */
    int32_t l_out;     /* prefetch outputs (5)                    */
    int32_t n_tables;  /* len(table_sizes)                        */
    int64_t total_ids; /* sum(table_sizes)                        */
} recmg_model_shape;

/* Floats of the raw dense blob: every array of _shapes (model.py:54-80)
 * except embed_id, row-major, concatenated in _shapes order.               */
int64_t recmg_model_dense_floats(const recmg_model_shape *shape);
/* Bytes of the packed (kernel-layout) weights for a precision; 0 if that
 * precision does not support the shape.  TC32 includes the folded token
 * tables (total_ids x 4*dim fp32 per layer-0 projection).                  */
size_t recmg_model_packed_bytes(const recmg_model_shape *shape, int32_t precision);
/* Re-lay the raw dense blob into the kernel layout (gate-interleaved LSTM
 * weights).  Ingests init_params / load_checkpoint arrays (model.py:83-100,
 * checkpoint.py:48-79) after a float64 -> float32 cast.                    */
int recmg_model_pack(const recmg_model_shape *shape, const float *dense_raw, void *packed,
                     int32_t precision, void *stream);
/* TC32 packing also needs embed_id [total_ids x dim] fp32 and the table
 * offsets [n_tables+1] int64 (device): the layer-0 token projection
 * [E_id[r]; E_tab[tab(r)]] @ Wx + b is folded into one row per id r.  The
 * TC32 forward then ignores embed_id and tid.  A TC-packed buffer serves
 * RECMG_PREC_TC32 / TC16 only: its gate columns, folded rows, layer-1
 * biases, slot projections and W_comb / comb bias are stored pre-scaled for
 * exp2 (-log2 e, 2 log2 e), so RECMG_PREC_FP32 needs its own
 * recmg_model_pack buffer.                                                  */
int recmg_model_pack_tc(const recmg_model_shape *shape, const float *dense_raw,
                        const float *embed_id, const int64_t *table_offsets, void *packed,
                        void *stream);
/* Scratch bytes recmg_model_forward needs for `batch` chunks.              */
size_t recmg_model_workspace_bytes(const recmg_model_shape *shape, int32_t precision,
                                   int64_t batch);
/*
 * forward_caching_batch (model.py:184-196) / forward_prefetch_batch
 * (model.py:199-212) over `batch` chunks:
 *   embed_id[total_ids*dim]   fp32 id embeddings
 *   gid, tid [batch*l_in]     int32
 *   logits   [batch*l_in] (caching) or [batch*l_out] (prefetch), pre-sigmoid
 *   bits     caching, nullable: (sigmoid >= 0.5) = (logit >= 0)  runtime.py:192
 *   pf_gid   prefetch, nullable: decode_indices in float64       model.py:250-258
 */
int recmg_model_forward(const recmg_model_shape *shape, int32_t precision,
                        const float *embed_id, const void *packed, const int32_t *gid,
                        const int32_t *tid, int64_t batch, float *logits, uint8_t *bits,
                        int32_t *pf_gid, void *ws, size_t ws_bytes, void *stream);

/* recmg_model_forward for a table shard: the model's
 * vocabulary (shape->total_ids, n_tables, the packed folded tables and
 * gid/tid) is the shard's local one, while the prefetch decode keeps the
 * global id scale of model.py:255, floor(po*(decode_ids-1)+0.5) over the
 * whole layout (decode_ids = 0: shape->total_ids, i.e. recmg_model_forward). */
int recmg_model_forward_ex(const recmg_model_shape *shape, int32_t precision,
                           const float *embed_id, const void *packed, const int32_t *gid,
                           const int32_t *tid, int64_t batch, int64_t decode_ids, float *logits,
                           uint8_t *bits, int32_t *pf_gid, void *ws, size_t ws_bytes,
                           void *stream);

/* recmg_model_forward_ex (TC32 / TC16 only) that also reports progress for a
 * consumer on another stream: every finished tile of 128 chunks adds one to
 * progress[(tile * 128) / piece_chunks] (device int32 counters, zeroed by the
 * caller; piece_chunks a multiple of 128), released after the tile's logits,
 * bits and decoded ids are visible device-wide.  Lets one forward launch over
 * the whole trace feed a piecewise replay without launch boundaries between
 * the pieces (pipeline.HotPath).                                            */
int recmg_model_forward_signal(const recmg_model_shape *shape, int32_t precision,
                               const float *embed_id, const void *packed, const int32_t *gid,
                               const int32_t *tid, int64_t batch, int64_t decode_ids,
                               float *logits, uint8_t *bits, int32_t *pf_gid, void *ws,
                               size_t ws_bytes, int32_t *progress, int64_t piece_chunks,
                               void *stream);
/* Stream-ordered wait: work queued on `stream` after this call starts once
 * progress[piece] >= target (acquire; one 1-thread kernel that polls).      */
int recmg_wait_progress(const int32_t *progress, int64_t piece, int32_t target, void *stream);

/* Upper bound on the CTAs (= SMs) the TC32 forwards occupy (default 148);
 * returns the previous value.  Leaving a few SMs to the replay lets a
 * pipelined replay of earlier chunks run beside the forwards.              */
int recmg_set_model_sm_budget(int n);

/* ---- trace helpers ----------------------------------------------------- */
/* tid[i] = table of gids[i] given table offsets[n_tables+1] (device), the
 * searchsorted of trace.py:86 / index_of_global trace.py:44-51.             */
int recmg_table_ids(const int32_t *gids, int64_t n, const int64_t *offsets, int32_t n_tables,
                    int32_t *tid, void *stream);
/* Host: body of the text trace format (read_trace, trace.py:172-204):
 * parses "table_id,row_id" lines of host_buf from byte `pos` into global
 * ids (host_out, up to cap, appended at *n_out) while every line has the
 * plain form and is in range; stops at the first other line (*stop_pos =
 * its first byte, for the caller's reference-rule reader) or at len.
 * *lines_done = lines consumed, blank lines included.                        */
int recmg_trace_parse_text(const char *host_buf, int64_t len, int64_t pos,
                           const int64_t *host_offsets, int32_t n_tables, int32_t *host_out,
                           int64_t cap, int64_t *n_out, int64_t *stop_pos, int64_t *lines_done);
/* Table shard: for every global gid, its row in the
 * shard's local vocabulary and its local table.  table_local[n_tables] maps
 * a global table to its local index (-1: another shard's, then both outputs
 * are -1); local_offsets[n_local+1] are the local table offsets.  The
 * models of a shard are packed over the local vocabulary and run with
 * recmg_model_forward_ex(decode_ids = global total_ids).                    */
int recmg_shard_local_ids(const int32_t *gids, int64_t n, const int64_t *offsets,
                          int32_t n_tables, const int32_t *table_local,
                          const int64_t *local_offsets, int32_t *local_gids,
                          int32_t *local_tids, void *stream);
/* Host: the sticky-pool pass of generate_trace (trace.py:144-160), given
 * the already-drawn zipf gids and coins.  Returns 0.                        */
int recmg_trace_pool_pass(const int64_t *host_zipf_gids, const double *host_sticky_coin,
                          const double *host_pool_coin, int64_t n, double stickiness,
                          int32_t pool_size, int64_t *host_out_gids);

/* ---- streamed generator (trace.py:124-161 without materialising it) ---- */
/* pcg[4] = numpy PCG64 {state_hi, state_lo, inc_hi, inc_lo} as
 * default_rng(seed) holds it right after permutation(V).                    */
/* Host: count doubles of Generator.random() starting `skip` outputs ahead
 * of pcg (PCG64.advance + next_double), on `threads` host threads.          */
int recmg_pcg64_uniforms(const uint64_t pcg[4], int64_t skip, int64_t count, double *host_out,
                         int32_t threads);
/* Host: guide[b] = #{j : cdf[j] <= b / 2^guide_log2}, b = 0..2^guide_log2
 * (host_guide has 2^guide_log2 + 1 entries).                                */
int recmg_trace_guide(const double *host_cdf, int64_t V, int32_t guide_log2, int64_t *host_guide);
/* Host: accesses [i0, i0+count) of generate_trace(n_total accesses): the
 * zipf draw choice(V, p) == cdf.searchsorted(random(), 'right') mapped
 * through rank_to_gid, the two coin streams, and the sticky-pool pass with
 * its state (host_pool[pool_size], *host_pool_len; start empty, len 0)
 * carried from the previous block.  Blocks must be generated in order.     */
int recmg_trace_generate_block(const uint64_t pcg[4], int64_t n_total, int64_t i0, int64_t count,
                               const double *host_cdf, int64_t V, const int64_t *host_guide,
                               int32_t guide_log2, const int64_t *host_rank_to_gid,
                               double stickiness, int32_t pool_size, int64_t *host_pool,
                               int32_t *host_pool_len, int32_t *host_out_gids, int32_t threads);

/* ---- diagnostics -------------------------------------------------------- */
/* tcgen05 self-test GEMM: D[128 x N] (fp32, row-major) = A[128 x K] * B[N x K]^T
 * with A, B fp16 row-major; A staged in shared memory (a_in_tmem = 0) or in
 * tensor memory (1).  Pins the descriptor / TMEM layouts of the LSTM kernels. */
int recmg_selftest_umma(const void *A, const void *B, float *D, int N, int K, int a_in_tmem,
                        void *stream);

/* ---- instrumentation --------------------------------------------------- */
/* TC32 forward with per-CTA phase cycle counters (prof: device int64
 * [148][16]); diagnostic build of the same kernel (scripts/tc_phases.py).   */
int recmg_model_forward_profile(const recmg_model_shape *shape, const void *packed,
                                const int32_t *gid, const int32_t *tid, int64_t batch,
                                float *logits, void *ws, size_t ws_bytes, long long *prof,
                                void *stream);
/* Kernels this library has launched since it was loaded (host counter).   */
uint64_t recmg_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* RECMG_H */
