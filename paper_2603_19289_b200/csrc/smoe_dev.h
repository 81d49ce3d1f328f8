// smoe_dev.h — device-side data layout shared by the host engine (engine.cpp)
// and the sm_100a kernels (kernels.cu).  Plain C++ (no CUDA headers) so the
// host engine can be compiled by g++.
//
// HBM layout:
//   * every weight matrix the decode path streams is stored as *row tiles*:
//     [R/32][cols][32] bf16 — 32 consecutive output rows interleaved per input
//     column, so one warp (lane = output row) reads 64 contiguous bytes per
//     column and a CTA stages a [chunk of columns x 32 rows] tile with one
//     cp.async.bulk.  Each lane keeps the reference's *sequential* f32 dot
//     product (numerics.cpp:136-147) for its row, so results are bit-identical.
//   * an expert (l, e) is one contiguous block of expert_elems bf16:
//       gate/up part  [Hmp/16][H][16][2]  (virtual row 2r = w_gate row r,
//                                          2r+1 = w_up row r)
//       down part     [Hp/32][Hmp][32]
//     which is exactly one cudaMemcpyAsync between the pinned host store and
//     an HBM slot.
#pragma once
#include <cstddef>
#include <cstdint>

namespace smoe {

constexpr int kMaxK = 16;         // top-k limit
constexpr int kMaxE = 1024;       // experts per layer limit
constexpr int kMaxD = 256;        // head_dim limit
constexpr int kRowTile = 32;      // rows per warp tile
constexpr int kMailboxRing = 1024;

enum PredKind : int { kBaselineS = 0, kRouterPF = 1, kEstPF = 2, kHybrid = 3, kOracle = 4, kNone = -1 };
enum Gating : int { kSoftmaxTopK = 0, kTopKSoftmax = 1 };

#ifdef __CUDACC__
#define SMOE_HD __host__ __device__
#else
#define SMOE_HD
#endif
SMOE_HD inline int round_up(int a, int b) { return (a + b - 1) / b * b; }

// One mailbox entry (pinned, mapped host memory).  Device writes the body,
// __threadfence_system(), then `seq` last; the host scheduler polls `seq`.
struct MailboxEntry {
    volatile int seq;   // request number (monotonic, 1-based)
    int layer;
    int step;           // decode step (-1 prefill / shadow)
    int nids;
    int ids[kMaxK];
    int flags;          // kMbAllHit: the device found every (local) id resident
                        // and released the layer itself; host: bookkeeping only
    int pad[11];
};
constexpr int kMbAllHit = 1;

struct DevModel {
    int L, E, K, H, Hm, V, D;
    float eps;
    int gating;
    int Hmp;            // Hm padded to 16 (gate/up tiles hold 16 rows x {gate,up})
    int Hp;             // H padded to 32 (down / Wo row tiles)
    int Ep, Vp, QKVp;   // router / unembed / qkv rows padded to 32
    int cap;            // KV capacity (positions)
    float inv_sqrt_d;   // 1.0f / sqrtf(D), computed on the host like model.cpp:336
    int fast;           // decode GEMV arithmetic: 0 exact (reference order), 1 tolerance (run_fast)
    const uint16_t* emb;      // [V][H] row-major bf16
    const uint16_t* unemb;    // row tiles of unembed [V][H]
    const float* final_gain;  // [H]
    const float* attn_gain;   // [L][H]
    const float* moe_gain;    // [L][H]
    const uint16_t* wqkv;     // [L] x row tiles of [wq; wk; wv] (3D x H)
    const uint16_t* wo;       // [L] x row tiles of wo (H x D)
    const uint16_t* gate;     // [L] x row tiles of gate (E x H)
    const float* rope;        // [cap][D/2][2] cos, sin (host libm, model.cpp:309-321)
    long long qkv_stride, wo_stride, gate_stride;  // elements per layer
    // expert cache
    const uint16_t* slots;    // [L*C][expert_elems]
    const int* slot_of;       // [L][E] -> slot index in layer, -1 = absent
    int C;
    long long expert_elems, gu_elems;
    // speculation artifacts
    const float* dv;          // [L][E][H] default vectors (f32)
    // estimator (f32 row tiles): A (dm x d), B (mlp x dm), C (dm x mlp), W_head (E x dm)
    int est_d, est_dm, est_mlp;
    float est_eps;
    const float* est_a;
    const float* est_pos;     // [L][dm]
    const float* est_b;
    const float* est_c;
    const float* est_gain;
    const float* est_bias;
    const float* est_head;
    const int* hybrid;        // [L-1] predictor kind per layer
    // split decode attention (contexts beyond kAttnSplitMin positions):
    // attn_grid CTAs when that many are co-resident (occupancy checked at
    // session creation), else 1 (single-CTA path); the CTAs' flag wait is
    // bounded by attn_spin cycles and reports through *attn_err
    int attn_grid;
    int* attn_err;
    long long attn_spin;
    int ffn_fused;      // expert FFN as one launch (k_ffn) when its grid is co-resident
    int ffn_cs_fused;   // tolerance mode: expert FFN as one launch (k_ffn_cs) when co-resident
    int ffn_gud;        // tolerance mode, one GPU: gate/up + column-split down (k_ffn_gud + k_down_reduce)
    int down_rb;        // tolerance mode, one GPU: down as one CTA per row block, K warps (k_ffn_down_rb)
    int attn_fast_grid; // tolerance-mode attention CTAs (0: sized for the KV capacity); any value is
                        // correct, the host sizes it for the positions a decode call reaches
};

// Per-stream decode state (the main stream, and the Oracle's shadow stream).
struct DevState {
    float* x;          // [Hp] residual input of the current layer
    float* r;          // [L][Hp]
    float* s;          // [L][Hp]
    float* m;          // [L][Hp]
    float* q;          // [D]   attention query (after RoPE)
    float* ctx;        // [D]
    float* kc;         // [L][cap][D]
    float* vc;         // [L][cap][D]
    float* lg_true;    // [L][E]
    int* id_true;      // [L][K]
    float* g_true;     // [L][K]
    int* id_exec;      // [L][K]
    float* g_exec;     // [L][K]
    float* lg_pred;    // [L][E]  index = predicted layer (l+1)
    int* id_pred;      // [L][K]
    float* g_pred;     // [L][K]
    float* quasi;      // [Hp]  q_l of the last prediction (router-pf / est-pf)
    float* est_z;      // [dm]
    float* est_act;    // [mlp]
    float* est_xn;     // [dm] gain*xhat + bias
    float* h;          // [K][Hmp]
    float* y;          // [K][Hp]  raw expert outputs (decision order)
    float* dpart;      // [K][Hmp/16][Hp] tolerance-mode down partials per 16-column slice of h
    float* logits;     // [V]
    int* pos;          // position
    int* token;        // current token
    int* tok_in;       // input token of the current step (for the trace)
    int* counters;     // last-CTA counters [64]
    int* down_cnt;     // [Hp/32] k_ffn_down per-row-block arrival counters (self-resetting)
    int* log_cnt;      // [L] last-CTA counters of the batched logging routers
    // rms_norm statistics, computed by the kernel that produces the vector:
    // f64 partial sums of squares per 32-row block (Hp/32 per vector), summed
    // by consumers in a fixed order (rms_scale_from_partials).
    double* ssq_x;     // [L+1][Hp/32]  x entering layer l (index L: final norm)
    double* ssq_r;     // [L][Hp/32]    r_l (pre-MoE residual)
    // q_l prologue fused into k_wo when the executed decision of layer l is
    // known before it (prefetch mode, l >= 1): rd_l = r_l + d_l with d_l the
    // layer_default of that decision (speculation.cpp:104-121), and its
    // rms_norm partials; the predictor then only scales it (gain_{l+1}).
    float* rd;         // [L][Hp]
    // decision handshake for the expert kernels' early start (prefetch mode):
    // k_embed bumps pass_id at every pass; the predictor that decides layer l
    // publishes dec_ready[l] = pass_id after the decision and its copy request
    int* pass_id;      // [1]
    int* dec_ready;    // [L]
    int* gu_done;      // [L][K] gate/up CTAs finished, monotonic (fused k_ffn)
    int* ffn_epoch;    // [L] completed k_ffn launches per layer
    double* ssq_rd;    // [L][Hp/32]
    int* ep_arrive;    // [L] EP: this rank's k_ffn_down CTAs done (self-resetting)
};

// Expert parallelism: expert e of every layer lives on rank
// e % world.  Combine without summation: each rank writes the raw outputs of
// its local experts into every rank's exchange buffer (peer memory over
// NVLink, or the same device when ranks share a GPU) and bumps each rank's
// per-layer arrival counter with a system-scope atomic; every rank then mixes
// all k rows in decision order, so EP results equal single-GPU results bit
// for bit.
constexpr int kMaxEP = 8;
constexpr int kEpBatchMax = 16;  // batched decode under EP: sequences per step (BASELINE configs 2-3: B <= 16)
struct DevEP {
    int rank, world;
    float* xbuf[kMaxEP];  // rank p's exchange buffer [2][K][Hp] (layer parity), mapped here
    int* cnt[kMaxEP];     // rank p's arrival counters [L] (monotonic)
    int* epoch;           // this rank's combines completed per layer [L]
    // batched decode: the same scheme over the step's B·k expert rows
    float* bxbuf[kMaxEP];  // rank p's [2][kEpBatchMax * K][Hp] (layer parity)
    int* bcnt[kMaxEP];     // rank p's batched arrival counters [L] (monotonic)
    int* bepoch;           // this rank's batched combines completed per layer [L]
    int* bdone;            // [L] this rank's publish CTAs (self-resetting)
};

// Cross-stream control block (device memory unless noted).
struct DevCtl {
    MailboxEntry* mailbox;   // mapped pinned host memory, kMailboxRing entries
    int* req_counter;        // requests issued so far
    int* req_seq;            // [L] request number the next FFN at layer l waits for
    int* ready;              // [L] last completed request number per layer (copy stream writes)
    int* error;              // device-detected error code (deadlock etc.)
    int* step;               // decode step counter
    int* tokens_out;         // [max_steps]
    long long spin_limit;    // clock64 cycles before declaring a deadlock
    int resident;            // 1: every expert is resident (no requests, no waits)
    // 1: a request whose (local) ids are all resident per slot_of releases its
    // layer on the device (ready = seq) without the host round trip
    int fast_hit;
    // 1: the host orders the compute stream after the copy stream with a CUDA
    // event before every expert kernel (no device spin on ready; no graphs) —
    // for kernel-serialising tools (ncu, compute-sanitizer)
    int host_ordered;
    DevEP ep;
};

}  // namespace smoe
