/* ecoserve.h -- C ABI of the B200-native PaDG instance hot path.
 *
 * EcoServe (arXiv 2504.18154) runs every serving instance in temporally
 * disaggregated phases (Sec. 3.2.1): a prefill-only phase
 * over a batch of new requests, and a decode-only phase over the running set,
 * switched by the instance scheduler under the macro
 * instance's routing (Alg. 1/2). This header exposes those two
 * phases as calls on an instance object, plus the host-side macro scheduler.
 * The computation inside a phase is the Llama-family decoder of Eq. 1-3
 * with the readings listed in DESIGN.md section 3.
 *
 * Conventions
 *  - Every function returns ecoserve_status; nothing throws across the ABI.
 *  - Pointers documented "device" are CUDA device pointers on the instance's
 *    device; "host" are CPU pointers. Sizes are element counts unless noted.
 *  - Borrowed memory (weights, prepared buffer, KV pool, stream) is allocated by
 *    the caller and must outlive the instance. The library owns its host state
 *    (allocator, block tables, request table) and its device workspace.
 *  - CUDA errors are sticky: the instance reports dead in its status and every
 *    later call returns ECOSERVE_ERR_CUDA. ecoserve_last_error() explains.
 *  - An instance is single-threaded (one worker thread per GPU); a macro object
 *    is single-threaded (the dispatcher thread).
 */
#ifndef ECOSERVE_H_
#define ECOSERVE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ECOSERVE_OK = 0,
  ECOSERVE_ERR_INVALID_ARG = 1, /* bad pointer/size/shape; nothing changed */
  ECOSERVE_ERR_KV_EXHAUSTED = 2, /* not enough free KV blocks; all-or-nothing: nothing allocated */
  ECOSERVE_ERR_STATE = 3,        /* unknown or duplicate req_id, decode before prefill, dead instance */
  ECOSERVE_ERR_UNSUPPORTED = 4,  /* shape/feature this build does not implement */
  ECOSERVE_ERR_CUDA = 5,         /* sticky CUDA error */
  ECOSERVE_ERR_NCCL = 6,
  ECOSERVE_ERR_NUMERIC = 7       /* NaN logits (reading A6: greedy sampling of NaN is an error);
                                    sticky like CUDA errors: the instance is marked dead, since
                                    its weights or KV can no longer be trusted */
} ecoserve_status;

/* Model shape, Table 1 notation: L, H, M, D plus the GQA
 * kv-head count, SwiGLU width F and vocabulary V (reading A1). */
typedef struct {
  int32_t n_layers;   /* L */
  int32_t hidden;     /* H, multiple of 64 */
  int32_t n_heads;    /* M */
  int32_t n_kv_heads; /* Mkv, divides M, M/Mkv <= 16 */
  int32_t head_dim;   /* D in {32, 64, 128} */
  int32_t ffn_dim;    /* F, multiple of 64 */
  int32_t vocab;      /* V */
  float rope_theta;   /* reading A3 */
  float rms_eps;      /* reading A4 */
  int32_t tp_size;    /* 1, or 2: a TP pair splitting heads, kv heads and FFN
                         columns; every size query and buffer below is then per rank */
} ecoserve_model_shape;

/* Paged KV pool (PagedAttention). Layout, block-major so a
 * block migrates as one contiguous copy:
 *   pool[num_blocks][n_layers][2 (K,V)][n_kv_heads][block_tokens][head_dim] bf16
 * `pool` is a borrowed device pointer of ecoserve_kv_pool_bytes() bytes; the
 * instance zero-fills it at creation. block_tokens must be 64. */
typedef struct {
  int32_t block_tokens;
  int64_t num_blocks;
  void* pool;
} ecoserve_kv_pool;

/* Raw weights, bf16, matrices [out][in] row-major (device pointers):
 *   embed [V][H], lm_head [V][H] (untied), final_norm [H];
 *   layers[l][0..8] = attn_norm [H], wq [M*D][H], wk [Mkv*D][H], wv [Mkv*D][H],
 *                     wo [H][M*D], ffn_norm [H], w_gate [F][H], w_up [F][H],
 *                     w_down [H][F].
 * wq/wk/wv/w_gate/w_up are read only during ecoserve_instance_create (they are
 * re-laid-out into the prepared buffer); all others are read by every phase. */
typedef struct {
  const void* embed;
  const void* lm_head;
  const void* final_norm;
  const void* const* layers; /* host array of n_layers*9 device pointers */
} ecoserve_weights;

/* Engine configuration (NULL = defaults in brackets). */
typedef struct {
  int32_t token_budget;  /* max prompt tokens per prefill batch T [16384] */
  int32_t max_batch;     /* max decode batch B [512]; also max requests per prefill batch */
  int32_t max_positions; /* max prompt + output length [16384] */
  int32_t debug_hidden;  /* keep per-layer residuals of the last phase call [0] */
} ecoserve_engine_config;

/* One request handed to a prefill phase. The prompt is copied during the call. */
typedef struct {
  int64_t req_id;
  const int32_t* prompt; /* host [prompt_len], token ids in [0, V) */
  int32_t prompt_len;    /* S >= 1 */
  int32_t max_new_tokens;/* G >= 1, counts the prefill token (reading A7) */
} ecoserve_request;

typedef struct {
  int32_t alive;          /* 0 after a sticky CUDA error */
  int32_t n_requests;     /* resident (unfinished + finished-not-released) */
  int64_t blocks_total;
  int64_t blocks_used;
} ecoserve_instance_status;

typedef struct {
  int64_t req_id;
  int32_t prompt_len;
  int32_t n_generated;    /* tokens produced so far, incl. the prefill token */
  int32_t finished;       /* n_generated == max_new_tokens */
  int32_t n_blocks;
} ecoserve_req_status;

typedef struct ecoserve_instance ecoserve_instance;

/* Writes a fresh NCCL unique id (128 bytes) to host `out` for a TP pair. */
ecoserve_status ecoserve_nccl_unique_id(void* out);

/* Bytes of the KV pool for `num_blocks` blocks (layout above). <0 on bad args. */
int64_t ecoserve_kv_pool_bytes(const ecoserve_model_shape* shape, int32_t block_tokens, int64_t num_blocks);
/* Bytes of the caller-allocated prepared-weight buffer (fused, re-laid-out QKV
 * and gate/up matrices). <0 on bad args. */
int64_t ecoserve_prepared_weight_bytes(const ecoserve_model_shape* shape);

/* Create an instance on `device`. `prepared` is a caller-allocated device buffer
 * of ecoserve_prepared_weight_bytes(); `cuda_stream` is a borrowed cudaStream_t
 * (NULL = the library creates its own).
 * TP=2 (shape->tp_size == 2): each rank of the pair (one process
 * per GPU) calls create concurrently with tp_rank 0/1 and the same 128-byte
 * nccl_unique_id (from ecoserve_nccl_unique_id on one rank, broadcast by the
 * caller). `raw` then holds the rank's shard: wq/wk/wv/w_gate/w_up rows and
 * wo/w_down columns of heads [r*M/2, (r+1)*M/2), kv heads [r*Mkv/2, ..) and FFN
 * columns [r*F/2, ..); embed, LM head and norms are replicated. The residual
 * stream is all-reduced (fp32 sum) after the O and down projections; both ranks
 * return identical tokens. tp_size 1 requires tp_rank 0 and nccl_unique_id NULL. */
ecoserve_status ecoserve_instance_create(const ecoserve_model_shape* shape, const ecoserve_kv_pool* kv,
                                         const ecoserve_weights* raw, void* prepared, int32_t device,
                                         int32_t tp_rank, const void* nccl_unique_id, void* cuda_stream,
                                         const ecoserve_engine_config* cfg, ecoserve_instance** out);

/* Prefill-only phase: admit n new requests, run their
 * prompts through the model in batches of <= token_budget tokens, write their
 * KV into the pool, and return each request's first (greedy) token in
 * first_tokens (host [n]). All-or-nothing on ECOSERVE_ERR_KV_EXHAUSTED /
 * INVALID_ARG / STATE (duplicate or resident req_id). Synchronous: returns when
 * the tokens are on the host. */
ecoserve_status ecoserve_prefill_phase(ecoserve_instance* inst, const ecoserve_request* reqs, int32_t n,
                                       int32_t* first_tokens);

/* Decode-only phase (rows a13-a16): `steps` decode iterations over the running
 * set req_ids[0..n) with continuous batching (a request leaves the batch once it
 * has max_new_tokens tokens). tokens is host [n][steps]: the token produced for
 * request i at step s, or -1 when the request had already finished.
 * n_finished (host, may be NULL) receives the number of requests finished by
 * the end of the call. A new KV block is allocated at every 64-token boundary;
 * ECOSERVE_ERR_KV_EXHAUSTED leaves the step that could not allocate undone. */
ecoserve_status ecoserve_decode_phase(ecoserve_instance* inst, const int64_t* req_ids, int32_t n, int32_t steps,
                                      int32_t* tokens, int32_t* n_finished);

/* Hybrid batching (chunked prefill: the Sarathi-style NoDG baseline
 * on these kernels). One forward pass over prompt chunks and decode tokens together:
 * each chunk continues its request's prompt where the previous chunk ended (a new
 * req_id starts at token 0 and registers the request; prompt / prompt_len /
 * max_new_tokens are read only then); each decode_ids[k] (a prefilled, unfinished
 * request) advances by one token. Chunk rows attend to the request's cached K / V
 * plus the chunk (causal); decode rows use the split-K decode attention.
 * chunk_tokens[i]: the request's first token if chunk i completes its prompt, else -1;
 * decode_tokens[k]: the next token. All-or-nothing on validation errors
 * (INVALID_ARG, STATE for chunks of prefilled or decodes of unprefilled requests,
 * KV_EXHAUSTED). n_chunks + n_decode <= max_batch, total tokens <= token_budget. */
typedef struct {
  int64_t req_id;
  const int32_t* prompt;   /* host, the full prompt (first chunk only) */
  int32_t prompt_len;
  int32_t max_new_tokens;
  int32_t chunk_len;       /* tokens of this chunk */
} ecoserve_chunk;

ecoserve_status ecoserve_hybrid_step(ecoserve_instance* inst, const ecoserve_chunk* chunks, int32_t n_chunks,
                                     const int64_t* decode_ids, int32_t n_decode, int32_t* chunk_tokens,
                                     int32_t* decode_tokens);

/* KV migration between instances (mitosis contraction and
 * rebalancing move a running request with its paged KV instead of recomputing it).
 * A request's KV is blocks of the pool's block-major layout, so it moves as
 * n_blocks contiguous copies of ecoserve_kv_pool_bytes(shape, 64, 1) bytes each. */
typedef struct {
  int64_t req_id;
  int32_t prompt_len;
  int32_t max_new_tokens;
  int32_t n_generated;  /* >= 1 (prefilled) */
  int32_t last_token;   /* the token the next decode step feeds */
  int32_t n_blocks;     /* KV blocks the request holds */
} ecoserve_req_state;
/* Copies the request's blocks, in logical order, into `dst` (device pointer on
 * any device, UVA; >= n_blocks * block bytes) and its prompt into `prompt`
 * (host, >= prompt_len); fills *state. The request stays resident (release it
 * after the destination imported it). Synchronous. */
ecoserve_status ecoserve_kv_export(ecoserve_instance* inst, int64_t req_id, void* dst, int64_t dst_bytes,
                                   int32_t* prompt, int32_t prompt_cap, ecoserve_req_state* state);
/* Allocates state->n_blocks blocks, copies them from `src` (device, any device)
 * and registers the request so decode phases continue it. All-or-nothing:
 * KV_EXHAUSTED / STATE (resident req_id) leave the instance unchanged. Synchronous. */
ecoserve_status ecoserve_kv_import(ecoserve_instance* inst, const ecoserve_req_state* state, const int32_t* prompt,
                                   const void* src);

/* Free the KV blocks of the given requests and forget them. */
ecoserve_status ecoserve_release(ecoserve_instance* inst, const int64_t* req_ids, int32_t n);

/* Instance status plus up to `cap` per-request records (host). */
ecoserve_status ecoserve_get_status(const ecoserve_instance* inst, ecoserve_instance_status* out,
                                    ecoserve_req_status* reqs, int32_t cap);

/* Debug (engine_config.debug_hidden = 1): residual stream of `req_id` after
 * layer `layer` (0 = embedding output, L = after the last layer) from the last
 * phase call, fp32 host out [rows][H], rows = prompt_len (prefill) or 1
 * (decode, last step). */
ecoserve_status ecoserve_debug_hidden(ecoserve_instance* inst, int64_t req_id, int32_t layer, float* out);

/* Debug (engine_config.debug_hidden = 1): replace the token the next decode
 * step of `req_id` feeds (the request's last generated token) by `token`, so a
 * test can teacher-force the oracle's greedy sequence (the
 * GPU's argmax is compared with the oracle's at every step whose oracle top-2
 * margin exceeds 5e-2). Only the fed id changes: n_generated, KV growth and
 * the returned tokens are unaffected. INVALID_ARG if token is outside
 * [0, vocab); UNSUPPORTED without debug_hidden; STATE if the request is
 * unknown, not yet prefilled or finished. Host-only, no device work. */
ecoserve_status ecoserve_debug_force_token(ecoserve_instance* inst, int64_t req_id, int32_t token);

/* Device-side timing of the phase work, measured with CUDA events on the
 * instance stream: a phase interval starts after its inputs are resident in HBM
 * (after the host->device copy) and ends before the device->host token copy.
 * With profiling level 2 every kernel launch is also bracketed by events and
 * accumulated per kernel class with its algorithmic work. */
typedef struct {
  double prefill_ms, decode_ms;
  int64_t prefill_tokens, decode_tokens;
  int64_t launches;                          /* kernels launched by the phases */
  /* level 2 only */
  double gemm_prefill_ms, gemm_prefill_flop; int64_t gemm_prefill_launches;
  double gemm_decode_ms, gemm_decode_bytes;  int64_t gemm_decode_launches; /* weight bytes streamed */
  double attn_prefill_ms, attn_prefill_flop; int64_t attn_prefill_launches;
  double attn_decode_ms, attn_decode_bytes;  int64_t attn_decode_launches;  /* KV bytes read */
  double other_ms;                           int64_t other_launches;
  int64_t h2d_bytes, d2h_bytes;              /* host<->device bytes the phases copied */
} ecoserve_timing;

/* level 0 off, 1 phase intervals (default), 2 + per-kernel-class events */
ecoserve_status ecoserve_set_profiling(ecoserve_instance* inst, int32_t level);
ecoserve_status ecoserve_get_timing(ecoserve_instance* inst, ecoserve_timing* out, int32_t reset);

void ecoserve_instance_destroy(ecoserve_instance* inst);
const char* ecoserve_last_error(const ecoserve_instance* inst);

/* ------------------------------------------------------------------------
 * Host-only macro-instance scheduler (Alg. 1 InterSchedule P:476-497 with the
 * prose probing of P:556-559 (reading A9), Alg. 2 CheckConstraints P:499-540,
 * readings A10-A14, A18). All times are int64 nanoseconds.
 * ------------------------------------------------------------------------ */
typedef struct ecoserve_macro ecoserve_macro;

typedef struct {
  int32_t n_instances;
  int64_t slo_ttft_ns;
  int64_t slo_tpot_ns;
  int32_t reserve_tokens;      /* R of reading A14 */
  int32_t block_tokens;        /* 64 */
  int32_t probe_printed;       /* 0: cyclic probe (prose, A9); 1: Alg. 1 as printed */
  /* prefill predictor: either the integer cost model a + (b S + c S^2)/1000
   * (b, c in ps) when n_table == 0, or piecewise-linear over (table_len, table_ns). */
  int64_t cost_a_ns, cost_b_ps, cost_c_ps;
  int32_t n_table;
  const int64_t* table_len;    /* host [n_table], strictly increasing */
  const int64_t* table_ns;     /* host [n_table] */
  const int64_t* total_blocks; /* host [n_instances] */
} ecoserve_macro_config;

typedef struct {
  int64_t req_id;
  int64_t arrival_ns;
  int32_t prompt_len;
} ecoserve_route_req;

typedef struct {
  int64_t req_id;
  int64_t arrival_ns;
  int32_t prompt_len;
  int64_t t_first_ns;   /* -1 until the first token */
  int32_t n_generated;
  int32_t finished;
} ecoserve_sched_req;

typedef struct {
  int32_t phase;        /* 0 idle, 1 prefill, 2 decode */
  int64_t t_switch_ns;  /* last phase switch (Alg. 2 t_switch) */
  int64_t total_blocks;
  int32_t alive;
} ecoserve_sched_status;

typedef struct {
  int64_t req_id;
  int32_t instance;
} ecoserve_routed;

ecoserve_status ecoserve_macro_create(const ecoserve_macro_config* cfg, ecoserve_macro** out);
/* Alg. 1. *inst = chosen instance, or -1 (Deferred: the caller queues it with
 * ecoserve_macro_defer and retries with ecoserve_macro_drain_deferred).
 * outcomes (host, may be NULL, cap n_instances) receives the Alg. 2 result of
 * each probed instance in probe order (0 ok, 1 TTFT, 2 TPOT, 3 KV); *n_probed
 * (may be NULL) their count. */
ecoserve_status ecoserve_macro_route(ecoserve_macro* m, const ecoserve_route_req* req, int64_t now_ns, int32_t* inst,
                                     int32_t* outcomes, int32_t* n_probed);
/* Alg. 2 alone, against instance `inst` (no state change). *result as above. */
ecoserve_status ecoserve_macro_check(const ecoserve_macro* m, int32_t inst, const ecoserve_route_req* req,
                                     int64_t now_ns, int32_t* result);
ecoserve_status ecoserve_macro_defer(ecoserve_macro* m, const ecoserve_route_req* req);
/* Status push of instance `inst`: per-request records overwrite the
 * macro's view by req_id; finished ones are dropped. */
ecoserve_status ecoserve_macro_update_status(ecoserve_macro* m, int32_t inst, const ecoserve_sched_status* st,
                                             const ecoserve_sched_req* reqs, int32_t n);
/* Retry deferred requests FIFO, stopping at the first still-Deferred one. */
ecoserve_status ecoserve_macro_drain_deferred(ecoserve_macro* m, int64_t now_ns, ecoserve_routed* out, int32_t cap,
                                              int32_t* n);
int32_t ecoserve_macro_prev_idx(const ecoserve_macro* m);
int64_t ecoserve_macro_predict_prefill_ns(const ecoserve_macro* m, int32_t prompt_len);
void ecoserve_macro_destroy(ecoserve_macro* m);

/* ------------------------------------------------------------------------
 * Mitosis scaling (Sec. 3.5).
 * ------------------------------------------------------------------------ */
enum {
  ECOSERVE_MITOSIS_CREATE = 0,       /* first macro created (a1 = index) */
  ECOSERVE_MITOSIS_ADD = 1,          /* one instance added to macro a1 */
  ECOSERVE_MITOSIS_ADD_SPLIT = 2,    /* added to a1, which then split off a new macro a2 of N_l */
  ECOSERVE_MITOSIS_REMOVE = 3,       /* one instance removed from macro a1 */
  ECOSERVE_MITOSIS_REMOVE_MERGE = 4, /* one removed from a1, then macros a1 and a2 merged */
  ECOSERVE_MITOSIS_REMOVE_MACRO = 5  /* the last instance of the only macro removed */
};
/* One expansion (expand = 1) or contraction (0) step over the macro sizes
 * (host array sizes[*n_macros], creation order, capacity cap) with bounds
 * N_l <= N_u (Fig. 7: expansion fills the first macro below N_u, splitting off a
 * new macro of N_l when all are full; contraction shrinks the smallest macro to
 * N_l, then its partner, merging the pair into N_u - 1 once they total N_u).
 * action (host [3]) = {kind, a1, a2}. */
ecoserve_status ecoserve_mitosis_step(int32_t* sizes, int32_t* n_macros, int32_t cap, int32_t n_l, int32_t n_u,
                                      int32_t expand, int32_t* action);

/* InstanceHandler: the serializable proxy of an instance handed from
 * one macro scheduler to another (no re-initialisation, no KV movement). */
typedef struct {
  int64_t actor_id;
  int32_t device;
  int32_t tp_size;
  int32_t tp_rank;
  int64_t kv_blocks;
  char address[64];    /* e.g. "host:port/gpu" (NUL-terminated) */
} ecoserve_instance_handler;
/* Returns the encoded size (> 0) written to out, or -(needed bytes) if cap is too small. */
int32_t ecoserve_handler_serialize(const ecoserve_instance_handler* h, uint8_t* out, int32_t cap);
/* ECOSERVE_ERR_UNSUPPORTED on an unknown wire version, INVALID_ARG on a malformed buffer. */
ecoserve_status ecoserve_handler_deserialize(const uint8_t* in, int32_t n, ecoserve_instance_handler* h);

/* Virtual-clock discrete-event simulation of a macro instance of n identical
 * instances under the integer cost model (decision-parity mode):
 * prefill batch = sum of predicted prefill ns; decode step =
 * d + e*B + (f * sum(context))/1000 ns. Outputs per request (host arrays of n_req):
 * instance, t_first, t_decode_begin, t_done (-1 if never admitted), and n_preempt
 * (may be NULL): how often the request was preempted for recompute under KV
 * pressure (reading A14: when the reservation R is below the true output length, a
 * decode step preempts the latest-arrived batch members until the grown batch fits
 * the pool; they are re-prefilled with prompt + generated tokens from the front of
 * the queue, TD-Pipe P:1112). ECOSERVE_ERR_KV_EXHAUSTED if one request needs more
 * blocks than a whole instance pool (the outputs are then partial). */
typedef struct {
  int64_t cost_d_ns, cost_e_ns, cost_f_ps;
  int32_t token_budget;
} ecoserve_des_config;

ecoserve_status ecoserve_des_run(const ecoserve_macro_config* mcfg, const ecoserve_des_config* dcfg,
                                 const int64_t* arrival_ns, const int32_t* prompt_len, const int32_t* output_len,
                                 int32_t n_req, int32_t* inst, int64_t* t_first, int64_t* t_decode_begin,
                                 int64_t* t_done, int64_t* route_log /* host [cap][3]: (t_ns, req, inst), may be NULL */,
                                 int32_t route_log_cap, int32_t* n_route_log, int32_t* n_preempt);

#ifdef __cplusplus
}
#endif
#endif /* ECOSERVE_H_ */
