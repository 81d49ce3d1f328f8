// kernels.h — host-callable launchers for the sm_100a kernels in kernels.cu.
// Every launcher enqueues on the given stream and returns the launch error.
// DevModel / DevState / DevCtl are passed by value (kernel parameters), so a
// captured CUDA graph replays with the same pointers; all per-token dynamic
// values (position, token, request numbers) live in device memory.
#pragma once
#include "smoe_dev.h"

#include <cuda_runtime.h>

#include <string>

namespace smoe {

// Weight init (model.cpp:112-158 stream semantics, counter-based splitmix64):
// element n of the reference's row-major [R][C] tensor is
// f32(gaussian_n(seed) * f64(stddev)), rounded to bf16 (RNE) and written to
// `out` in the given layout (row_offset shifts rows inside a row-tiled block
// that packs several matrices, e.g. [wq; wk; wv]).
enum GenLayout : int { kRowMajor = 0, kRowTiled = 1, kGateUp = 2 };
cudaError_t launch_gen_bf16(uint64_t seed, float stddev, int R, int C, int tile_cols, int layout,
                            int which, int row_offset, uint16_t* out, cudaStream_t s);

struct RouterLaunch {
    int layer;
    int do_true;        // evaluate the true router of `layer`
    int pred_kind;      // PredKind used to predict layer+1 (kNone = no prediction here)
    int exec_from;      // 0: exec = true decision, 1: exec = pred decision of `layer`, -1: leave
    int post_exec;      // post (layer, exec ids) to the mailbox
    int post_pred;      // post (layer+1, pred ids) to the mailbox
    int step_tag;       // mailbox step tag
    int quasi_ready;    // st.rd / ssq_rd of `layer` hold r_l + d_l (k_wo computed them)
};

// token = stream ? stream[*step] : *token_src (stream: teacher-forced decode input)
cudaError_t launch_embed(const DevModel& m, const DevState& st, const int* token_src,
                         cudaStream_t s, const int* stream = nullptr, const int* step = nullptr);
cudaError_t launch_qkv(const DevModel& m, const DevState& st, int layer, cudaStream_t s);
cudaError_t launch_attn(const DevModel& m, const DevState& st, double* scratch, int layer,
                        cudaStream_t s);
// rd_from_pred: also form rd_l = r_l + d_l from the decision predicted for
// `layer` (id_pred / g_pred), for the predictor's q_l.
cudaError_t launch_wo(const DevModel& m, const DevState& st, const DevCtl& ctl, int layer,
                      cudaStream_t s, int rd_from_pred = 0);
// logging-only true routers of layers l0 .. l0+nl-1 in one launch (prefetch mode)
cudaError_t launch_log_routers(const DevModel& m, const DevState& st, const DevCtl& ctl, int l0,
                               int nl, int step_tag, cudaStream_t s);
// L2 prefetch of the resident expert blocks of the decision predicted for `layer`
cudaError_t launch_l2_prefetch(const DevModel& m, const DevState& st, const DevCtl& ctl, int layer,
                               cudaStream_t s);
// rd_l = r_l + d_l of the executed decision (id_exec) after the true router
cudaError_t launch_quasi_rd(const DevModel& m, const DevState& st, int layer, cudaStream_t s);
cudaError_t launch_router(const DevModel& m, const DevState& st, const DevCtl& ctl,
                          const RouterLaunch& rl, const DevState* shadow, cudaStream_t s);
cudaError_t launch_estimator(const DevModel& m, const DevState& st, const DevCtl& ctl,
                             int layer, int post_pred, int step_tag, cudaStream_t s);
// exec_src 1: run the decision predicted for `layer` (id_pred / g_pred);
// s_from_r 1: normalise r_l inside the kernel (routers run concurrently).
cudaError_t launch_ffn(const DevModel& m, const DevState& st, const DevCtl& ctl, int layer,
                       cudaStream_t s, int exec_src = 0, int s_from_r = 0);
size_t attn_scratch_bytes(int cap);  // split / fast attention scratch for a KV capacity
cudaError_t launch_mark_decided(const DevState& st, int L, cudaStream_t s);
cudaError_t launch_ffn_part(const DevModel& m, const DevState& st, const DevCtl& ctl, int layer,
                            int part, cudaStream_t s);
cudaError_t launch_final(const DevModel& m, const DevState& st, const DevCtl& ctl,
                         int record_token, cudaStream_t s);

// Default-vector calibration: f64 sums of raw expert outputs in token order
// (speculation.cpp:28-42), frozen to f32 means (speculation.cpp:49-58).
cudaError_t launch_dv_accum(const DevModel& m, const DevState& st, double* sums,
                            long long* counts, int layer, cudaStream_t s);
cudaError_t launch_dv_freeze(const double* sums, const long long* counts, float* dv,
                             long long LE, int H, cudaStream_t s);

// Per-step record capture (LayerTraceRecord, model.hpp:94-103).
struct TraceDev {
    int* step;          // device step counter
    int cap;            // steps allocated
    int full;           // 0: ids only (hit-rate history), 1: all fields
    float *s, *r, *m, *lg_true, *g_true, *g_exec, *lg_pred, *g_pred, *y, *logits;
    int *id_true, *id_exec, *id_pred;
    int* tok_in;        // [cap] input token per step
};
cudaError_t launch_trace(const DevModel& m, const DevState& st, const TraceDev& tr,
                         cudaStream_t s);

// exp_glibc over n doubles (device buffers) — the parity check of the device exp.
cudaError_t launch_exp_glibc(const double* x, double* y, long long n, cudaStream_t s);
cudaError_t launch_decide(const float* logits, int rows, int E, int K, int gating, int* ids, float* gates,
                          cudaStream_t s);

// DistillDatasetBuilder (speculation.cpp:437-471) over trace steps [first, first+n).
cudaError_t launch_distill(const DevModel& m, const TraceDev& tr, int first, int n, int mode, float* inputs,
                           float* targets, cudaStream_t s);

// Router-pf ids `depth` layers ahead over trace steps; out [n][L][K] (rows < depth untouched).
// Expands one exponent-packed expert block (xp11, engine.h) from `src` (HBM
// staging) into the bf16 slot `dst` (n elements); on the copy stream.
cudaError_t launch_xp_unpack(const uint8_t* src, uint16_t* dst, long long n, cudaStream_t s);
long long xp_unpack_launches();  // k_xp_unpack launches so far (process-wide)
cudaError_t launch_pred_ahead(const DevModel& m, const TraceDev& tr, int first, int n, int depth, int* out,
                              cudaStream_t s);

cudaError_t launch_trace_y(const DevModel& m, const DevState& st, const TraceDev& tr, int layer,
                           cudaStream_t s);

// ---- batched prefill (prefill.cu) ----
struct PrefillDev {
    int P;              // tokens in this prefill
    int pos0;           // KV position of token 0
    int attn_smem_positions;
    const int* tokens;  // [P]
    float* X;           // [P][Hp] residual stream (layer input)
    double* ssqx;       // [P][Hp/32] rms partials of X
    float* Q;           // [P][D]
    float* ctx;         // [P][D]
    float* R;           // [P][Hp] r_l
    double* ssqr;       // [P][Hp/32]
    float* lg;          // [P][E] true router logits
    int* ids;           // [P][K]
    float* gates;       // [P][K]
    int* cnt;           // [E] tokens per expert
    int* off;           // [E+1]
    int* fill;          // [E]
    int* list;          // [P*K] entries t*K+i grouped by expert
    float* Hb;          // [P*K][Hmp]
    float* Y;           // [P*K][Hp] raw expert rows per (token, slot)
    double* attn_scratch;  // [P][2*cap] when contexts exceed the smem budget
    float* scale;       // [P] rms scale of the vector being normalised (per stage)
    int* chunk_u;       // [max chunks] wave expert index of each (expert, 8-token chunk)
    int* chunk_c;       // [max chunks] chunk index within the expert's token list
    int* dev_step;      // ctl.step (token records)
    int* trace_step;    // trace step counter (nullable)
    // batched decode (Session::batch_generate): token t is sequence t, all at
    // position pos0, each with its own KV cache at bkc/bvc + t * bkv_stride
    float* bkc;         // nullable (prefill of one sequence)
    float* bvc;
    long long bkv_stride;
    float* RD;          // [P][Hp] r_l + d_l (router-pf predictor input)
    double* ssqrd;      // [P][Hp/32]
    float* lgp;         // [P][E] predicted logits
    int* pids;          // [2][P][K] predicted decisions (double-buffered by layer parity)
    float* pgates;      // [2][P][K]
    float* logits;      // [P][V] final logits
    int* next;          // [P] argmax tokens
    int* nchunks;       // device-built (expert, chunk) list length (resident batches), nullable
    const int* pos_dev; // batched decode under a CUDA graph: the position lives on the device
};
constexpr int kMaxWave = 128;
struct PfWave {
    int n;
    int e[kMaxWave];
    int slot[kMaxWave];
};
int pf_attn_smem_positions();
cudaError_t pf_preload();
cudaError_t launch_pf_embed(const DevModel& m, const PrefillDev& pf, cudaStream_t s);
cudaError_t launch_pf_layer_dense(const DevModel& m, const DevState& st, const PrefillDev& pf, int layer,
                                  cudaStream_t s);
// chains: tokens per chunk worth computing (at most 8; fewer for small batches)
cudaError_t launch_pf_experts(const DevModel& m, const PrefillDev& pf, int layer, const PfWave& wv,
                              int chunks, cudaStream_t s, int chains = 8);
cudaError_t launch_pf_mix(const DevModel& m, const PrefillDev& pf, cudaStream_t s);
// batched decode under EP: publish this rank's expert rows to every rank and
// wait for every rank's rows of this layer (mix then reads the exchange buffer)
cudaError_t launch_pf_ep_combine(const DevModel& m, const PrefillDev& pf, const DevEP& ep, int layer, int* error,
                                 long long spin_limit, cudaStream_t s);
// tensor-core expert GEMMs of the batched prefill (prefill_tc.cu, tolerance
// mode): items = (wave expert, 128-token block) pairs in pf.chunk_u / chunk_c;
// apk: packed-activation scratch of tc_pack_bytes(m, items)
bool tc_prefill_supported(const DevModel& m);
size_t tc_pack_bytes(const DevModel& m, int items);
cudaError_t tc_preload();
cudaError_t launch_pf_experts_tc(const DevModel& m, const PrefillDev& pf, int layer, const PfWave& wv, int items,
                                 uint16_t* apk, cudaStream_t s);
// batched decode pieces (prefill.cu)
cudaError_t launch_pf_attn_block(const DevModel& m, const DevState& st, const PrefillDev& pf, int layer,
                                 cudaStream_t s);
cudaError_t launch_pf_route(const DevModel& m, const PrefillDev& pf, int layer, cudaStream_t s);
// executed decision := pids/pgates[buf] (Algorithm 1, l >= 1), then counts / lists
cudaError_t launch_pf_exec_pred(const DevModel& m, const PrefillDev& pf, int buf, cudaStream_t s);
// router-pf prediction for layer+1 from r_l and the executed decision -> pids/pgates[buf]
cudaError_t launch_pf_predict(const DevModel& m, const PrefillDev& pf, int layer, int buf, cudaStream_t s);
// baseline-s prediction for layer+1 (gate_{l+1} over s_l) -> pids/pgates[buf]
cudaError_t launch_pf_predict_baseline_s(const DevModel& m, const PrefillDev& pf, int layer, int buf,
                                         cudaStream_t s);
// q_l = rms_norm(r_l + d_l, gain_{l+1}) materialised as [P][H] (estimator input)
cudaError_t launch_pf_quasi_q(const DevModel& m, const PrefillDev& pf, int layer, float* qn, cudaStream_t s);
// make_decision on pf.lgp -> pids/pgates[buf]
cudaError_t launch_pf_decide_pred(const DevModel& m, const PrefillDev& pf, int buf, cudaStream_t s);
// final rms_norm + unembed + argmax for every token -> pf.logits, pf.next
// resident experts: the (expert, chunk) list is built on the device from the
// counts (no host round trip); wv must map every expert u < E to its slot.
cudaError_t launch_pf_experts_dev(const DevModel& m, const PrefillDev& pf, int layer, const PfWave& wv,
                                  int max_chunks, cudaStream_t s, int ep_rank = 0, int ep_world = 1);
cudaError_t launch_pf_final(const DevModel& m, const PrefillDev& pf, cudaStream_t s);
cudaError_t launch_pf_handoff(const DevModel& m, const DevState& st, const PrefillDev& pf, cudaStream_t s);

int max_dynamic_smem_needed(const DevModel& m);
// k_ffn_down_rb's shared memory (K rings + K staged h vectors) fits one CTA
int down_rb_ok(const DevModel& m);
std::string kernel_limit_violation(const DevModel& m);     // "" when every kernel fits
std::string estimator_limit_violation(const DevModel& m);  // after the estimator dims are set
int attn_grid_for(const DevModel& m, int device);
int ffn_fused_ok(const DevModel& m, int device);  // 1: launch_ffn uses the one-launch k_ffn
int ffn_cs_fused_ok(const DevModel& m, int device);  // 1: tolerance mode uses the one-launch k_ffn_cs
cudaError_t preload_kernels();
// Number of kernel launches enqueued by the launchers so far (host counter).
long long launch_counter();

}  // namespace smoe
