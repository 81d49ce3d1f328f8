// engine.h — host C++ runtime of the B200 speculative expert-prefetch decode
// path.  Replaces the reference's TwoLaneEngine / offloaded_forward /
// run_offloaded_decode (executor.cpp:41-359) with:
//   * ExpertStore   — pinned host memory holding every expert as one
//                     contiguous bf16 block in the kernels' tile layout;
//   * SlotCache     — per-layer HBM slot pool capped at C slots, LRU
//                     replacement, per-layer hit/miss table (NEW: the
//                     reference double-buffers k experts, executor.cpp:115-122);
//   * CopyScheduler — a host thread that polls a mapped-memory mailbox the
//                     router kernel writes (predicted / routed ids), issues
//                     cudaMemcpyAsync H2D for misses on the copy stream, then
//                     publishes the slot table and a per-layer ready value
//                     (cuStreamWriteValue32) the expert kernels wait on;
//   * Session       — device weights, decode state, CUDA-graph-captured token
//                     steps for on-demand and prefetch modes.
#pragma once
#include "kernels.h"
#include "smoe_dev.h"

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace smoe {

struct ModelCfg {
    int L, E, K, H, Hm, V, D;
    float eps;
    uint64_t seed;
    int gating;
    void validate() const;  // model.cpp:25-37 invariants (+ this path's limits)
};

struct SessionOpts {
    int device = 0;
    float cache_fraction = 1.0f;  // HBM slots per layer = max(K, ceil(frac * E))
    int max_positions = 4096;     // KV capacity
    int copy_latency_us = 0;      // injected per copy request (ExecutorOptions parity)
    double deadlock_s = 10.0;     // device spin limit before "deadlock suspected"
    int ep_rank = 0;              // expert parallelism: this rank owns experts e % ep_world == ep_rank
    int ep_world = 1;
};

struct EstCfg {
    int d, m, n, E, L;
    float eps;
};

struct TimelineEvent {  // MeasuredEvent (executor.hpp:31-37)
    int lane, kind, layer, token;
    double start_ms, end_ms;
};

struct CopyRecord {  // one mailbox request as the copy lane saw it
    int seq, layer, step, hits, misses;
    long long bytes;
    int ev;  // index into the event pool, -1 if none
};

// Exponent-packed bf16 expert blocks ("xp11", lossless).  Sign and mantissa
// of bf16 weights are incompressible, but the 8-bit exponent of weights drawn
// around a fixed scale spans a few binades (Q30 init: 3 exponents hold 75 % of
// the weights, entropy 2.55 bits), so each exponent is coded with two levels:
//   primary    2 bits: 0/1/2 = the block's three most frequent exponents,
//              3 = a secondary code follows;
//   secondary  4 bits, in element order: exponent = base + c for c < 15 (the
//              15-binade window holding the most non-primary weights), 15 =
//              escape (zeros, subnormals, outliers: the raw value is listed).
// A block of n bf16 weights (n % 256 == 0) becomes
//   [32 B header: magic, n/256 groups, n_secondary, n_escape, p0, p1, p2, base]
//   [n/4 B primary codes: element i in bits 2(i%4) of byte i/4]
//   [n/256 x u32: secondary codes before each 256-weight group]
//   [ceil(n_secondary/2) B secondary codes: code k in the low nibble of byte
//    k/2 for even k, the high nibble for odd k]  (padded to 16 B)
//   [n B sign<<7 | mantissa]
//   [n_escape x 8 B: u32 index, u16 raw value, u16 0 — ascending index]
// ~11.1 bits per Q30 weight on the wire instead of 16 (0.70 of raw).
constexpr uint32_t kXpMagic = 0x31315058u;  // "XP11"
constexpr int kXpHeader = 32;
constexpr int kXpGroup = 256;  // weights per group (one warp decodes a group)
inline long long xp_pad16(long long b) { return (b + 15) / 16 * 16; }
// byte offsets of the sections of a packed block
inline long long xp_off_groups(long long n) { return kXpHeader + n / 4; }
inline long long xp_off_sec(long long n) { return xp_off_groups(n) + xp_pad16(4 * (n / kXpGroup)); }
inline long long xp_off_sm(long long n, long long nsec) { return xp_off_sec(n) + xp_pad16((nsec + 1) / 2); }
inline long long xp_off_esc(long long n, long long nsec) { return xp_off_sm(n, nsec) + n; }
// packed size of a block with `nsec` secondary codes and `nesc` escapes
inline long long xp_bytes(long long n, long long nsec, long long nesc) { return xp_off_esc(n, nsec) + nesc * 8; }
// Packs `raw` (n bf16) into `out` (capacity `cap` bytes).  Returns the packed
// size, or 0 when the block is not worth packing (n % 256, or it would be
// larger than 7/8 of the raw bytes, or it does not fit `cap`).
long long xp_pack(const uint16_t* raw, long long n, uint8_t* out, long long cap);
// Inverse of xp_pack (host side; the device side is k_xp_unpack).
void xp_unpack(const uint8_t* in, uint16_t* out);

class ExpertStore {
public:
    ExpertStore(long long n_experts, long long elems_per_expert, int device);
    ~ExpertStore();
    uint16_t* expert(long long i) { return base_ + i * elems_; }
    long long bytes_per_expert() const { return elems_ * 2; }
    int numa_node() const { return node_; }  // -1: not NUMA-bound (single node / unknown)
    // packed size of block i on the wire (0: stored raw)
    long long packed_bytes(long long i) const { return packed_[i]; }
    long long wire_bytes(long long i) const { return packed_[i] ? packed_[i] : elems_ * 2; }
    long long max_packed_bytes() const { return elems_ * 2 * 7 / 8 + 64; }
    // packs every raw block in place (host threads); returns blocks packed
    long long pack_all();
    // restores block i to raw bf16 (before a partial rewrite of its weights)
    void unpack(long long i);
    long long blocks() const { return n_; }

private:
    uint16_t* base_ = nullptr;
    long long n_, elems_;
    size_t mapped_ = 0;  // mmap'd + cudaHostRegister'ed (NUMA-bound) when > 0
    int node_ = -1;
    std::vector<long long> packed_;  // [n_] packed bytes, 0 = raw
};

class SlotCache {
public:
    SlotCache(int L, int E, int C);
    // Returns the (slot, expert) pairs that must be copied for this request.
    std::vector<std::pair<int, int>> request(int layer, const int* ids, int n, int* hits,
                                             int* misses);
    const std::vector<int>& slot_row(int layer) const { return expert_slot_[layer]; }
    int capacity() const { return C_; }
    long long hits(int l) const { return hits_[l]; }
    long long misses(int l) const { return misses_[l]; }
    void clear_stats();
    void invalidate();

private:
    int L_, E_, C_;
    long long clock_ = 0;
    std::vector<std::vector<int>> expert_slot_;   // [L][E] -> slot or -1
    std::vector<std::vector<int>> slot_expert_;   // [L][C] -> expert or -1
    std::vector<std::vector<long long>> stamp_;   // [L][C]
    std::vector<std::vector<long long>> freq_;    // [L][E] requests seen (LFU)
    bool lfu_ = false;
    std::vector<long long> hits_, misses_;
};

class Session;

class CopyScheduler {
public:
    explicit CopyScheduler(Session* s);
    ~CopyScheduler();
    void start();
    void stop();
    std::string error();  // first error seen by the thread ("" if none)
    std::vector<CopyRecord> records();
    void clear_records();
    int next_seq() const { return next_seq_.load(); }  // requests handled = next_seq() - 1
    long long polls = 0;

private:
    void loop();
    void handle(const MailboxEntry& e);
    Session* s_;
    std::thread th_;
    std::atomic<bool> stop_{false};
    std::mutex mu_;
    std::string err_;
    std::vector<CopyRecord> recs_;
    std::atomic<int> next_seq_{1};
    int stage_idx_ = 0;
    int ev_next_ = 0;
};

class Session {
public:
    Session(const ModelCfg& cfg, const SessionOpts& opts);
    ~Session();

    // --- weights -------------------------------------------------------------
    void init_weights_seeded();  // build_model (model.cpp:112-158) on the GPU, bf16
    void load_tensor(const std::string& name, const float* data, long long n);  // from f32
    void load_default_vectors(const float* d);  // [L][E][H]
    void load_estimator(const EstCfg& c, const float* flat);
    void set_predictor(int kind, const int* hybrid_map);
    void set_cache_fraction(float frac);
    // Copies every expert into HBM (needs cache_fraction 1.0): the whole model
    // is resident, so no copy requests are posted and no waits happen.
    void preload_all();

    // --- decode --------------------------------------------------------------
    void reset(int max_steps, int trace_full);
    void prefill(const int* tokens, int n);               // true routing per token
    // all n prompt tokens per layer at once (prefill.cu); same results
    void prefill_batched(const int* tokens, int n);
    // 0: exact (sequential f32 chains, bit-identical to token-by-token prefill);
    // 1: tensor-core expert GEMMs (tcgen05, bf16x2 activations, f32 accumulate;
    // a stated tolerance instead of bit parity)
    void set_prefill_mode(int mode);
    void set_decode_mode(int mode);
    int decode_mode() const { return dm_.fast; }
    // B independent sequences decoded together (generate, speculation.cpp:401-421,
    // per sequence): prompts [B][P], out_tokens [B][n_new], out_logits
    // (nullable) [B][n_new][V] = the logits each output token was taken from.
    // mode 0 on-demand (true routing), 1 prefetch (Algorithm 1, router-pf).
    void batch_generate(int B, const int* prompts, int P, int n_new, int mode, int* out_tokens,
                        float* out_logits, double* step_ms);
    void decode(int mode, int n_steps, int use_graph);    // greedy, device-driven
    // Teacher-forced decode: step i consumes tokens[i] instead of the previous
    // argmax (the reference's trace workload, trace.cpp:187-211, fed through
    // speculative_forward).  Greedy argmax is still recorded per step.
    void decode_stream(int mode, const int* tokens, int n_steps);
    // Non-graph decode recording CUDA events around each layer's attention,
    // routing and expert phases plus the copy lane (tokens nullable = greedy).
    void decode_timeline(int mode, const int* tokens, int n_steps, std::vector<TimelineEvent>& out);
    int step_host(int mode, int token, float* logits_out);  // host token in, logits out
    void calibrate(long long ntok, uint64_t seed, int seq_len, float* d_out, long long* c_out);

    // --- results -------------------------------------------------------------
    int steps_done();
    void read_tokens(int* out, int n);
    void read_trace(const char* field, void* out, long long n_elems);
    // build_distill_dataset (speculation.cpp:476-484) from captured steps:
    // mode 0 quasi-hidden inputs (needs default vectors), 1 s_{l+1}.
    void build_distill_dataset(int first, int n, int mode, float* inputs, float* targets);
    // router-pf predictions `depth` layers ahead from captured steps (ids [n][L][K], -1 where l < depth)
    void predict_ahead(int first, int n, int depth, int* ids);
    void write_trace_bundle(const std::string& dir, int first, int n, int seq_len,
                            const std::string& source, unsigned long long seed);
    std::vector<double> token_ms();  // device-timed duration of each decode() step
    void counters(long long* hits, long long* misses, long long* bytes, double* copy_ms,
                  int* requests);
    std::vector<CopyRecord> copy_records() { return sched_->records(); }
    double event_ms(int ev_pair, int which);  // 0 start, 1 end; relative to run origin
    double step_event_ms(int i, int which);

    const ModelCfg& cfg() const { return cfg_; }
    int slots_per_layer() const { return C_; }
    // --- expert parallelism ----------------------------------------------------
    bool is_local(int e) const { return e % opts_.ep_world == opts_.ep_rank; }
    int local_experts() const {
        return (cfg_.E - opts_.ep_rank + opts_.ep_world - 1) / opts_.ep_world;
    }
    long long store_index(int l, int e) const {
        return static_cast<long long>(l) * el_max_ + e / opts_.ep_world;
    }
    int slots_for(float frac) const;
    void ep_buffers(void** xbuf, void** cnt);
    void ep_ipc_handles(unsigned char* out128);
    void ep_connect(void* const* xbufs, void* const* cnts);
    unsigned char* locate_ep_region(unsigned char* base, unsigned long long off,
                                    const unsigned long long tag[2]);
    void ep_connect_ipc(const unsigned char* handles);  // world x 128 bytes
    void debug_state(int* out, int cap);
    void clear_stats();
    // Average device time (us) per launch of each per-layer kernel, timed with
    // CUDA events on the compute stream over L back-to-back launches (one per
    // layer, so the streamed weights exceed L2), repeated `reps` times.
    // out[8]: qkv, attn, wo, router, ffn_gate_up, ffn_down, final, ffn (the expert FFN
    // as decode launches it: one fused launch when active, else gate/up + down).
    void profile_kernels(int reps, double* out);
    // H2D GB/s of expert-sized copies from the pinned store (same allocation and
    // copy size as the scheduler) into an HBM scratch block.
    double measure_link(int n_copies);
    int kernels_per_step(int mode) const;
    bool host_ordered() const { return host_ordered_; }
    // {expert FFN fused into one launch, split-attention CTAs, host-ordered copy waits, device hit
    //  path, NUMA node the pinned expert store is bound to (-1: not bound)}
    void path_info(int* out, int cap) const;

    // used by the scheduler
    friend class CopyScheduler;

private:
    void alloc();
    void free_all();
    void build_devmodel();
    void enqueue_step(int mode, int is_prefill, int record, int calibrating, cudaStream_t s,
                      int stream = 0);
    void enqueue_pass(DevState& st, int mode, int pred_kind_enabled, int calibrating,
                      int step_tag, int record, cudaStream_t s);
    void check_device_error();
    // host-ordered mode (ctl_.host_ordered): every request posted so far has
    // been handled by the copy scheduler, and stream `s` waits for its copies
    void host_copy_barrier(cudaStream_t s);
    void sync();
    void set_token(int tok);

    ModelCfg cfg_;
    SessionOpts opts_;
    int C_ = 0;
    DevModel dm_{};
    DevState st_{}, sh_{};
    DevCtl ctl_{};
    TraceDev tr_{};

    // device allocations (owned)
    std::vector<void*> dev_allocs_;
    void* dalloc(size_t bytes);
    void pf_waves(const PrefillDev& pf, int layer, const std::vector<int>& cnt);
    void h2d(void* dst, const void* src, size_t n, const char* what);
    void d2h(void* dst, const void* src, size_t n, const char* what);
    void dset(void* p, int v, size_t n, const char* what);
    uint16_t *d_emb_ = nullptr, *d_unemb_ = nullptr, *d_wqkv_ = nullptr, *d_wo_ = nullptr,
             *d_gate_ = nullptr, *d_slots_ = nullptr;
    float *d_final_gain_ = nullptr, *d_attn_gain_ = nullptr, *d_moe_gain_ = nullptr,
          *d_rope_ = nullptr, *d_dv_ = nullptr;
    int* d_slot_of_ = nullptr;
    double* d_attn_scratch_ = nullptr;
    double* d_dv_sums_ = nullptr;
    long long* d_dv_counts_ = nullptr;
    float* d_est_ = nullptr;
    int* d_hybrid_ = nullptr;
    int* d_prompt_tok_ = nullptr;
    int el_max_ = 0;                       // store blocks per layer = ceil(E / ep_world)
    unsigned char* d_ep_region_ = nullptr;  // EP region: tag | counters | exchange buffer
    unsigned long long ep_tag_[2] = {0, 0};
    float* d_xbuf_ = nullptr;              // EP exchange buffer [2][K][Hp]
    PrefillDev pf_{};                      // batched-prefill buffers (sized for pf_cap_ tokens)
    PrefillDev bd_{};                      // batched-decode buffers (sized for bd_cap_ sequences)
    int bd_cap_ = 0;
    long long batch_prefetched_bytes_ = 0;  // batched decode: expert bytes copied one layer ahead
    std::atomic<long long> direct_bytes_{0};  // link bytes of host-driven copies (batched waves / prefetch)
    int pf_tc_ = 0;                         // batched prefill expert GEMMs on tcgen05 (tolerance mode)
    uint16_t* d_tc_apk_ = nullptr;          // packed activations of the tensor-core prefill
    size_t tc_apk_cap_ = 0;
    int* bd_nchunks_ = nullptr;
    float* bd_qn_ = nullptr;          // [B][H] q_l for the batched estimator
    int* bd_pos_ = nullptr;           // device position of a graph-captured batched step
    float* d_est_flat_ = nullptr;     // estimator params, flat layout (estimator.hpp:41-72)
    size_t est_flat_n_ = 0;
    std::vector<void*> bd_allocs_;
    int pf_cap_ = 0;
    int* d_cnt_ = nullptr;                 // EP arrival counters [L]
    int* d_epoch_ = nullptr;               // EP combines done [L]
    int* d_bepoch_ = nullptr;              // EP batched combines done [L]
    int* d_bdone_ = nullptr;               // EP batched publish CTAs [L] (self-resetting)
    void ep_batch_ptrs(float* xbuf, int** bcnt, float** bxbuf) const;
    std::vector<void*> ipc_opened_;

    // packed expert copies (xp11): H2D of the packed block into a staging ring
    // slot, then k_xp_unpack into the HBM slot, both on `s` (FIFO: a ring slot
    // is reused kXpRing copies later, after its decode ran)
    // The decodes run on their own highest-priority stream (s_unpack_), so
    // expert i+1's H2D overlaps expert i's decode; a ring slot's next H2D waits
    // for its previous decode (ev_xp_), and join_unpack() orders a stream
    // after every decode issued so far (before a ready flag / slot use).
    static constexpr int kXpRing = 8;
    unsigned char* d_xp_stage_ = nullptr;
    long long xp_stride_ = 0;
    std::atomic<long long> xp_next_{0};
    cudaStream_t s_unpack_ = nullptr;
    cudaEvent_t ev_h2d_[kXpRing] = {}, ev_xp_[kXpRing] = {}, ev_unp_join_ = nullptr;
    std::atomic<int> xp_pending_{0};  // decodes issued since the last join_unpack
    bool store_packed_ = false;       // some expert block is packed: request tails run on s_unpack_
    cudaEvent_t ev_h2d_tail_ = nullptr, ev_hostord2_ = nullptr;
    void join_unpack(cudaStream_t s);
    bool pack_store_ = std::getenv("SMOE_STORE_PACK") == nullptr || std::atoi(std::getenv("SMOE_STORE_PACK")) != 0;
    // copies expert (layer, e) from the pinned store into `dst`; returns the bytes moved over the link
    long long copy_expert(int layer, int expert, uint16_t* dst, cudaStream_t s, const char* what);

    // host
    std::unique_ptr<ExpertStore> store_;
    std::unique_ptr<SlotCache> cache_;
    std::unique_ptr<CopyScheduler> sched_;
    MailboxEntry* h_mailbox_ = nullptr;
    int* h_stage_ = nullptr;  // pinned slot-table staging ring [256][E]
    int* h_token_ = nullptr;  // pinned token staging [2]
    float* h_logits_ = nullptr;
    cudaStream_t s_comp_ = nullptr, s_copy_ = nullptr;
    cudaStream_t s_side_ = nullptr;               // routers/predictors in prefetch mode
    cudaStream_t s_log_ = nullptr;                // logging-only true routers (lowest priority)
    // L2 warm-up of the next layer's experts (k_l2_prefetch): measured slower on Q30
    // (competes with the attention kernels for HBM), so off unless requested
    bool l2_prefetch_ = std::getenv("SMOE_L2_PREFETCH") != nullptr;
    std::vector<cudaEvent_t> ev_fork_, ev_join_;  // per layer
    cudaEvent_t ev_side_end_ = nullptr;           // side stream fully done (before k_final)
    cudaEvent_t ev_log_end_ = nullptr;            // log stream fully done (before k_final)
    std::vector<cudaEvent_t> ev_copy_;  // pairs
    std::vector<cudaEvent_t> ev_step_;  // pairs per decode step
    cudaEvent_t ev_origin_ = nullptr;
    cudaEvent_t ev_hostord_ = nullptr;  // host-ordered mode: copy stream -> compute stream
    bool host_ordered_ = false;
    int n_step_events_ = 0;

    int pred_kind_ = kNone;
    std::vector<int> hybrid_;
    bool have_dv_ = false, have_est_ = false;
    EstCfg est_{};
    int max_steps_ = 0, trace_full_ = 0;
    int steps_ = 0;

    std::map<long long, cudaGraphExec_t> graphs_;
    std::map<long long, int> graph_kernels_;
    cudaGraphExec_t get_graph(int mode, int stream = 0);
    void size_attn_grid(int pos_end);
    int host_pos_ = 0;  // position mirror for step_host's attention grid (advisory)
    int* d_stream_ = nullptr;
    // timeline recording (decode_timeline): event pairs per (step, layer, phase)
    struct TlRec {
        std::vector<TimelineEvent> meta;                      // times filled after sync
        std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;  // per meta entry
        int step = 0;
    };
    TlRec* tl_ = nullptr;
    int tl_begin(int lane, int kind, int layer, cudaStream_t s);
    void tl_end(int idx, cudaStream_t s);
    void upload_stream(const int* tokens, int n_steps);
    void drop_graphs();
};

}  // namespace smoe
