/* smoe.h — C ABI of the B200 speculative expert-prefetch MoE decode path.
 *
 * Drop-in boundary for the reference's decode-path API
 * (/root/reference/proj/include/specmoe).  Plain pointers and sizes only; no
 * CUDA or torch types.  Every function returns an int status:
 *   0 = ok, 1 = invalid argument (the reference throws std::invalid_argument,
 *   CLI exit 2), 2 = runtime / CUDA error (std::runtime_error, CLI exit 3);
 * the message is available from smoe_last_error() on the calling thread.
 * INTEGRATION.md shows the reference-side binding (a C++ shim rethrowing
 * the matching exception, and a ctypes stub).
 */
#ifndef SMOE_H
#define SMOE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct smoe_session smoe_session;

/* ModelConfig (model.hpp:28-47).  gating: 0 softmax-topk-renorm, 1 topk-softmax. */
typedef struct smoe_config {
    int32_t layers, experts, top_k, hidden, expert_hidden, vocab, head_dim;
    float eps;
    uint64_t seed;
    int32_t gating;
} smoe_config;

/* Session options.  cache_fraction caps the HBM slot pool per layer at
 * max(top_k, ceil(cache_fraction * experts)) slots (NEW: the reference keeps
 * exactly two k-expert buffers, executor.cpp:115-122).  copy_latency_us is
 * ExecutorOptions::copy_latency_us (executor.hpp:23-29); deadlock_s the
 * device-side wait limit (the reference's deadlock timeout, executor.cpp:124-128). */
typedef struct smoe_options {
    int32_t device;
    float cache_fraction;
    int32_t max_positions;
    int32_t copy_latency_us;
    double deadlock_s;
    int32_t ep_rank;   /* expert parallelism: this rank owns experts e % ep_world == ep_rank */
    int32_t ep_world;  /* 1 = single GPU (default when 0) */
} smoe_options;

/* EstimatorConfig (estimator.hpp:20-39). */
typedef struct smoe_estimator_config {
    int32_t d, m, n, experts, layers;
    float eps;
} smoe_estimator_config;

/* TrainHyper (estimator.hpp:151-160) and CurvePoint (estimator.hpp:162-166). */
typedef struct smoe_train_hyper {
    double lr;
    int32_t batch_tokens;
    int64_t max_steps;
    int64_t eval_every;
    double val_fraction;
    uint64_t seed;
    int32_t k;
    double early_stop_hit_rate;
} smoe_train_hyper;
typedef struct smoe_curve_point {
    int64_t tokens_seen;
    double val_kl;
    double val_hit_rate;
} smoe_curve_point;

/* Predictor kinds (PredictorKind, speculation.hpp:64): -1 none,
 * 0 baseline-s, 1 router-pf, 2 est-pf, 3 hybrid, 4 oracle. */
enum { SMOE_PRED_NONE = -1, SMOE_PRED_BASELINE_S = 0, SMOE_PRED_ROUTER_PF = 1,
       SMOE_PRED_EST_PF = 2, SMOE_PRED_HYBRID = 3, SMOE_PRED_ORACLE = 4 };
/* OffloadMode (executor.hpp:18). */
enum { SMOE_ON_DEMAND = 0, SMOE_PREFETCH = 1 };

/* One copy-lane request (MeasuredEvent kCopy, executor.hpp:31-37, plus the
 * cache outcome).  start/end are device-timed ms from the decode origin. */
typedef struct smoe_copy_event {
    int32_t seq, layer, step, hits, misses;
    int64_t bytes;
    double start_ms, end_ms;
} smoe_copy_event;

/* One measured lane event (MeasuredEvent, executor.hpp:31-37): lane 0 compute /
 * 1 copy; kind 0 attn / 1 gate / 2 expert / 3 copy; token = decode step index. */
typedef struct smoe_event {
    int32_t lane, kind, layer, token;
    double start_ms, end_ms;
} smoe_event;

const char* smoe_last_error(void);

/* Creates a session: allocates the pinned bf16 expert store, HBM slot pool,
 * dense weights, streams and the copy-scheduler thread.  Replaces building a
 * Model and the TwoLaneEngine (executor.cpp:41-216). */
int smoe_session_create(const smoe_config* cfg, const smoe_options* opt, smoe_session** out);
int smoe_session_destroy(smoe_session* s);

/* build_model (model.cpp:112-158) generated on the GPU, every weight rounded
 * to bf16 (RNE). */
int smoe_init_weights_seeded(smoe_session* s);
/* Loads one f32 tensor of a reference Model by its bundle name
 * (model.cpp:194-254: "embedding", "layer3.wq", "layer0.expert5.w_down", ...);
 * rounded to bf16 on the way in. */
int smoe_load_tensor(smoe_session* s, const char* name, const float* data, int64_t count);
/* DefaultVectorTable [L][E][H] (speculation.hpp:18-33). */
int smoe_load_default_vectors(smoe_session* s, const float* d, int64_t count);
/* init_estimator_params<float> (estimator.cpp:54-75): the flat parameter
 * block (param_count() floats, estimator.cpp:29-33) for config c and seed. */
int smoe_estimator_param_count(const smoe_estimator_config* c, int64_t* n);
int smoe_estimator_init(const smoe_estimator_config* c, uint64_t seed, float* flat, int64_t cap);
/* train_estimator (estimator.cpp:374-450) on the GPU: KL distillation with
 * hand-derived gradients and Adam, bit-exact with the reference.  The
 * DistillDataset (estimator.hpp:117-131) is given flat: inputs
 * [tokens][layers_predicting][d], targets [tokens][layers_predicting][E].
 * Writes the trained flat params and the validation curve (n_curve points;
 * at most curve_cap stored).  train_ms (nullable): device time of the
 * training steps, evaluation excluded.  Needs no session. */
int smoe_train_estimator(const smoe_estimator_config* c, uint64_t seed, const float* inputs,
                         const float* targets, int64_t tokens, int32_t layers_predicting,
                         const smoe_train_hyper* h, float* params_out, int64_t params_cap,
                         smoe_curve_point* curve_out, int32_t curve_cap, int32_t* n_curve,
                         double* train_ms);
/* EstimatorParams flat layout (estimator.hpp:41-72). */
int smoe_load_estimator(smoe_session* s, const smoe_estimator_config* c, const float* flat,
                        int64_t count);
/* make_predictor (speculation.cpp:330-346).  hybrid_map: layers-1 kind codes
 * (nullable -> all router-pf), only for SMOE_PRED_HYBRID. */
int smoe_set_predictor(smoe_session* s, int32_t kind, const int32_t* hybrid_map);
int smoe_set_cache_fraction(smoe_session* s, float cache_fraction);

/* New decode sequence (DecodeState reset).  max_steps sizes the per-step
 * record buffers; trace_full = 1 also records s, r, m, logits, gates and raw
 * expert outputs per (step, layer) (LayerTraceRecord, model.hpp:94-103). */
int smoe_reset(smoe_session* s, int32_t max_steps, int32_t trace_full);
/* Prefill with true routing, one forward_decode per token (model.cpp:355-389). */
int smoe_prefill(smoe_session* s, const int32_t* tokens, int32_t n);
/* Batched prefill: the same results as smoe_prefill (KV cache, next token,
 * every later decode step), all n tokens per layer at once — dense weights
 * and each executed expert are streamed once per layer, experts loaded into
 * the slot pool in waves.  The prompt's per-token trace rows are not recorded.
 * Single GPU; with the Oracle predictor it falls back to smoe_prefill. */
int smoe_prefill_batched(smoe_session* s, const int32_t* tokens, int32_t n);
/* Expert GEMMs of smoe_prefill_batched: mode 0 (default) exact — the
 * reference's sequential f32 chains, bit-identical to smoe_prefill; mode 1
 * tensor cores (tcgen05, M = 128 tokens of an expert, activations as bf16
 * hi + lo, f32 accumulation in TMEM) — the hidden states then agree with the
 * reference to a stated tolerance, not bit for bit (tests/test_gpu_prefill_tc.py).
 * Needs hidden and expert_hidden to be multiples of 64. */
int smoe_set_prefill_mode(smoe_session* s, int32_t mode);
/* Decode GEMV arithmetic for every single-sequence decode kernel (qkv, wo,
 * routers / predictor, expert gate/up and down, unembed): mode 0 (default)
 * exact — each output row one sequential f32 chain in the reference's column
 * order, bit-identical to the reference (linear, numerics.cpp:136-147);
 * mode 1 tolerance — four packed fused multiply-add partial sums per row, so
 * the kernels are HBM-bound; hidden states and logits then agree with the
 * reference within the stated tolerance and router ids are exact except
 * reported near-ties (tests/test_gpu_fast.py).  Rebuilds the step graphs. */
int smoe_set_decode_mode(smoe_session* s, int32_t mode);
/* n_steps greedy decode steps on the device (speculative_forward semantics in
 * SMOE_PREFETCH mode, forward_decode in SMOE_ON_DEMAND mode). */
int smoe_decode(smoe_session* s, int32_t mode, int32_t n_steps, int32_t use_graph);
/* Teacher-forced decode: step i consumes tokens[i] instead of the previous
 * argmax (the reference's trace workload over random_token_stream,
 * trace.cpp:187-211, run through speculative_forward in SMOE_PREFETCH mode).
 * The argmax of every step is still recorded (smoe_read_tokens). */
int smoe_decode_stream(smoe_session* s, int32_t mode, const int32_t* tokens, int32_t n_steps);
/* run_offloaded_decode (executor.cpp:326-359): prefill + n_new-1 decode steps;
 * out_tokens[n_new]; per_token_ms[n_new-1] (device-timed, nullable). */
int smoe_run_offloaded_decode(smoe_session* s, const int32_t* prompt, int32_t n_prompt,
                              int32_t n_new, int32_t mode, int32_t* out_tokens,
                              double* per_token_ms);
/* run_offloaded_decode returning the whole ExecutorResult (executor.hpp:39-44):
 * tokens, the measured lane events of the same run (CUDA events around each
 * layer's attention / routing / expert phases and the copy lane; no CUDA
 * graph), per_token_ms[n_new-1] and max_resident_layers (the most layers whose
 * experts were requested and not yet consumed at once; the reference's bound
 * is 2, executor.cpp:159-162).  events (nullable) holds up to cap events;
 * *n_events = the total. */
int smoe_run_offloaded_decode_ex(smoe_session* s, const int32_t* prompt, int32_t n_prompt,
                                 int32_t n_new, int32_t mode, int32_t* out_tokens,
                                 double* per_token_ms, smoe_event* events, int32_t cap,
                                 int32_t* n_events, int32_t* max_resident_layers);
/* One host-driven step: token in, logits[vocab] out, returns the argmax token
 * through *next (end-to-end API: H2D of the token, D2H of the logits). */
int smoe_step(smoe_session* s, int32_t mode, int32_t token, float* logits_out, int32_t* next);
/* accumulate_default_vectors over random_token_stream(ntok, vocab, seed) with
 * resets every seq_len tokens (speculation.cpp:23-83, trace.cpp:187-211), on
 * the GPU; loads the table into the session and copies it out (nullable). */
int smoe_calibrate(smoe_session* s, int64_t ntok, uint64_t seed, int32_t seq_len,
                   float* d_out, int64_t* counts_out);

/* Results. */
int smoe_steps_done(smoe_session* s, int32_t* n);
int smoe_read_tokens(smoe_session* s, int32_t* out, int32_t n);
/* field: id_true, id_exec, id_pred ([steps][L][K] int32), g_true, g_exec,
 * g_pred ([steps][L][K]), s, r, m ([steps][L][H]), lg_true, lg_pred
 * ([steps][L][E]; lg_pred row l = prediction for layer l), y ([steps][L][K][H]),
 * logits ([steps][vocab]), tok_in ([steps] input token of each step). */
int smoe_read_trace(smoe_session* s, const char* field, void* out, int64_t n_elems);
/* Trace bundle of steps [first, first + n) in the reference's format
 * (TraceWriter, trace.cpp:60-122; MOET files, moet.hpp:3-9): manifest.json
 * plus token_ids, s, r, m, router_logits (true router), expert_ids /
 * expert_gates (executed decision, ids as f32) and expert_outputs (raw) .moet
 * files in `dir`, readable by the reference's TraceReader.  Needs
 * smoe_reset(..., trace_full = 1). */
/* build_distill_dataset (speculation.cpp:437-484) from captured trace steps
 * [first, first+n) (needs smoe_reset with trace_full=1), on the GPU:
 * mode 0 (DistillInput::kQuasiHidden, needs default vectors): inputs are
 * q_l = rms_norm(r_l + layer_default(executed_l), gain_{l+1}); mode 1
 * (kSNext): s_{l+1}.  targets: the true router logits of layer l+1.
 * inputs [n][L-1][H], targets [n][L-1][E] (host). */
int smoe_build_distill_dataset(smoe_session* s, int32_t first, int32_t n, int32_t mode, float* inputs,
                               float* targets);
/* B independent sequences decoded together (batch 1-16 configs): for every
 * sequence b, generate(model, prompts[b], n_new, predictor)
 * (speculation.cpp:401-421) — prompt via the true path, then on-demand
 * (mode 0, forward_decode) or speculative (mode 1, Algorithm 1 with the
 * router-pf predictor) steps — with the B tokens of a step sharing every
 * weight stream and expert load.  Each sequence's tokens and logits equal
 * its single-sequence run.  prompts [B][prompt_len]; out_tokens [B][n_new];
 * out_logits (nullable) [B][n_new][V]; step_ms (nullable): mean wall ms per
 * decode step (prompt excluded).  Does not touch the session's own decode
 * state. */
int smoe_batch_generate(smoe_session* s, int32_t batch, const int32_t* prompts, int32_t prompt_len,
                        int32_t n_new, int32_t mode, int32_t* out_tokens, float* out_logits,
                        double* step_ms);
/* Diagnostics: y = exp(x) computed on the GPU by the device restatement of
 * glibc's exp(double) that every f64 softmax / silu on the path uses
 * (exp_glibc.cuh); equal to the host libm's exp bit for bit. */
int smoe_exp(const double* x, double* y, int64_t n);
/* Diagnostics: make_decision (model.cpp:258-274) of `rows` logits rows
 * [rows][E] on the GPU through the decision routine every router, predictor
 * and estimator on the path uses; ids / gates [rows][K]. */
int smoe_decide(const float* logits, int32_t rows, int32_t E, int32_t K, int32_t gating, int32_t* ids,
                float* gates);
/* Router-pf predictions `depth` layers ahead (multi-layer-
 * ahead prefetch study) from captured steps (trace_full=1, default vectors
 * loaded): ids[t][l][:] = top-k of gate_l . rms_norm(r_{l-depth} +
 * layer_default(executed_{l-depth}), gain_l); -1 for l < depth.  depth 1 is
 * the paper's router-pf predictor (speculation.cpp:206-228). */
int smoe_predict_ahead(smoe_session* s, int32_t first, int32_t n, int32_t depth, int32_t* ids);
int smoe_write_trace_bundle(smoe_session* s, const char* dir, int32_t first, int32_t n,
                            int32_t seq_len, const char* source, uint64_t seed);
int smoe_token_ms(smoe_session* s, double* out, int32_t cap, int32_t* n);
/* Per-layer cache hits/misses [L], total H2D bytes, summed copy-lane busy ms,
 * number of copy requests. */
int smoe_counters(smoe_session* s, int64_t* hits, int64_t* misses, int64_t* h2d_bytes,
                  double* copy_ms, int32_t* requests);
int smoe_copy_events(smoe_session* s, smoe_copy_event* out, int32_t cap, int32_t* n);
/* Slots per layer actually allocated. */
int smoe_cache_slots(smoe_session* s, int32_t* slots);
/* Expert parallelism.  Each rank creates its session with
 * ep_rank/ep_world (its pinned store, slot pool and copy lane hold only its
 * shard), then connects to the exchange buffers and arrival counters of all
 * ranks: either raw device pointers (ranks sharing a process; smoe_ep_buffers
 * gives each rank's own) or CUDA IPC handles (one process per GPU; 128 bytes
 * per rank from smoe_ep_ipc_handles — the handle of the allocation holding
 * the rank's exchange region plus the region's offset in it, since a peer's
 * opened pointer is the allocation base — exchanged by the caller, e.g. with
 * torch.distributed).  After connecting, every decode step combines expert
 * outputs across ranks through peer memory; results equal the single-GPU path. */
int smoe_ep_buffers(smoe_session* s, void** xbuf, void** counters);
int smoe_ep_ipc_handles(smoe_session* s, unsigned char* out128);
int smoe_ep_connect(smoe_session* s, void* const* xbufs, void* const* counters);
int smoe_ep_connect_ipc(smoe_session* s, const unsigned char* handles);
/* Copies every expert into HBM (cache_fraction 1.0 only): the model is fully
 * resident, decode posts no copy requests and never waits on the copy lane. */
int smoe_preload_all(smoe_session* s);
/* Clears cache hit/miss counters, copy records and step timings (state kept). */
int smoe_clear_stats(smoe_session* s);
/* Average device time (us) per launch of each per-layer kernel, CUDA events on
 * the compute stream over L back-to-back launches (one per layer, weights
 * larger than L2), `reps` repetitions.  out_us[9]: qkv, attn, wo, router,
 * ffn_gate_up (on-demand form: decision from this layer's router), ffn_down,
 * final, ffn (the whole expert FFN as decode launches it: the one-launch fused
 * kernel when active, else gate/up + down), ffn_gate_up_prefetch (the form the
 * prefetch path launches for layers >= 1: decision published a layer ahead,
 * weight stream started before the PDL wait).  Needs a completed prefetch
 * decode step (resident experts). */
int smoe_profile_kernels(smoe_session* s, int32_t reps, double* out_us);
/* H2D GB/s of expert-sized copies from the pinned store into HBM. */
int smoe_measure_link(smoe_session* s, int32_t n_copies, double* gbps);
/* Kernel launches in one captured decode step (-1 before the first capture). */
int smoe_kernels_per_step(smoe_session* s, int32_t mode, int32_t* n);
/* Decode with a per-layer lane timeline (no CUDA graph; CUDA events around
 * attention, routing and expert phases, plus the copy lane): the measured
 * event log of run_offloaded_decode (executor.cpp:239-322).  tokens: forced
 * inputs (nullable = greedy).  Returns up to cap events through out, total in *n. */
int smoe_timeline(smoe_session* s, int32_t mode, const int32_t* tokens, int32_t n_steps,
                  smoe_event* out, int32_t cap, int32_t* n);

/* Reporting (host-only, no GPU needed). */
/* simulate_on_demand / simulate_prefetch (schedule.cpp:92-148) + breakdown
 * (schedule.cpp:205-217) + analytic_improvement (Eq. 1, schedule.cpp:150-155).
 * cold_start_copy < 0 means "use t_copy[0]". */
int smoe_simulate(int32_t layers, const double* t_attn, const double* t_gate,
                  const double* t_expert, const double* t_copy, double cold_start_copy,
                  int32_t mode, double* tpot, double* fractions3, double* analytic);
/* Trace-driven two-lane schedule with a per-layer slot cache (SURVEY §8f
 * row 4; extends simulate_prefetch / simulate_on_demand, schedule.cpp:92-148).
 * exec_ids [tokens][layers][k]: executed experts; pred_ids [tokens][layers][k]:
 * the prediction for layer l made at layer l-1 (lookahead >= 1); pred2_ids:
 * the prediction for layer l made at layer l-2 (lookahead 2).  policy 0 LRU,
 * 1 LFU; one copy of t_copy_expert per expert, single FIFO copy lane.
 * out4 = {mean TPOT, on-demand (stall) copies, speculative copies, useful
 * speculative copies} per measured token (tokens after warm_tokens). */
typedef struct smoe_cache_sim {
    int32_t tokens, layers, k, capacity, policy, lookahead, warm_tokens;
} smoe_cache_sim;
int smoe_simulate_cache(const smoe_cache_sim* c, const int32_t* exec_ids, const int32_t* pred_ids,
                        const int32_t* pred2_ids, const double* t_attn, const double* t_gate,
                        const double* t_expert, double t_copy_expert, double* out4);
/* per_token_reports (executor.cpp:361-382) then breakdown, averaged over tokens:
 * fractions {compute, copy on the critical path, idle}. */
int smoe_breakdown(const smoe_event* events, int32_t n, double* mean_fractions3,
                   double* mean_tpot);
/* Per-layer online hit rates of a recorded decode: exec_ids / true_ids
 * [steps][layers][k] (smoe_read_trace id_exec / id_true of the decode steps);
 * rates[layers-1], entry l-1 = mean recall_at_k at layer l (the predictor
 * dispatched at l-1).  Host-only. */
int smoe_layer_hit_rates(const int32_t* exec_ids, const int32_t* true_ids, int32_t steps, int32_t layers,
                         int32_t k, double* rates);
/* Hybrid map selection from per-layer hit rates:
 * rates [n_kinds][layers-1] of the candidate predictors kinds[] (SMOE_PRED_*
 * baseline-s / router-pf / est-pf).  threshold > 0: kinds[0] unless its rate
 * is below the threshold, then the best other; threshold <= 0: best per layer.
 * map_out[layers-1] feeds smoe_set_predictor(SMOE_PRED_HYBRID, map).  Host-only. */
int smoe_select_hybrid_map(const double* rates, const int32_t* kinds, int32_t n_kinds, int32_t layers,
                           double threshold, int32_t* map_out);
/* recall_at_k (metrics.cpp:9-20) and rank_alignment (metrics.cpp:22-28). */
int smoe_recall_at_k(const int32_t* pred, const int32_t* truth, int32_t k, double* recall,
                     int32_t* rank_match);

/* Which variants this session runs: out[0] expert FFN fused into one launch
 * (1) or gate/up + down kernels (0); out[1] split-attention CTAs; out[2]
 * host-ordered copy waits (profiler / sanitizer attached or
 * SMOE_HOST_ORDERED=1); out[3] device-side all-hit release; out[4] NUMA node
 * the pinned expert store is bound to (-1: not bound — single-node host);
 * out[5] expert blocks held exponent-packed in the pinned store; out[6]
 * link bytes per 1000 raw expert bytes; out[7] copy-lane decode kernels
 * (k_xp_unpack) launched so far in this process. */
int smoe_path_info(smoe_session* s, int32_t* out, int32_t cap);

/* Lossless exponent packing of one bf16 expert block ("xp11", engine.h):
 * the pinned store's wire format (~11 bits per Gaussian-like weight instead of
 * 16; SMOE_STORE_PACK=0 keeps the store raw).  Host only, no GPU needed.
 * smoe_xp_pack writes at most `cap` bytes and sets *packed_bytes (0: the block
 * does not pack — n % 8 != 0 or too many escapes); smoe_xp_unpack restores the
 * n raw values (n from the block header).  Replaces no reference function: the
 * reference copies raw experts (executor.cpp:138-198). */
int smoe_xp_pack(const uint16_t* raw, int64_t n, uint8_t* out, int64_t cap, int64_t* packed_bytes);
int smoe_xp_unpack(const uint8_t* packed, uint16_t* out, int64_t n);

/* Diagnostics: request counter, error flag, scheduler progress, ready[L], req_seq[L]. */
int smoe_debug_state(smoe_session* s, int32_t* out, int32_t cap);

#ifdef __cplusplus
}
#endif

#endif /* SMOE_H */
