// ref_driver.cpp — TEST INFRASTRUCTURE ONLY (never on the product path).
//
// A thin extern "C" shim over the *unmodified* reference library
// (/root/reference/proj/src, compiled by oracle/Makefile into oracle/_ref/).
// It lets the Python tests / golden-fixture generator / bench.py's
// cpu_baseline leg drive the reference through its own public C++ API
// (proj/include/specmoe/*.hpp).  Nothing here re-implements reference math:
// every number comes from the reference's own functions.
//
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline /
// --impl reference) may load the resulting oracle/_ref/libspecmoe_ref.so.

#include "specmoe/estimator.hpp"
#include "specmoe/executor.hpp"
#include "specmoe/metrics.hpp"
#include "specmoe/model.hpp"
#include "specmoe/numerics.hpp"
#include "specmoe/schedule.hpp"
#include "specmoe/speculation.hpp"
#include "specmoe/trace.hpp"

#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

using namespace specmoe;

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

// Round-to-nearest-even f32 -> bf16 -> f32 (the value the GPU stores).
float round_bf16(float x) {
    std::uint32_t u;
    std::memcpy(&u, &x, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    u &= 0xFFFF0000u;
    float y;
    std::memcpy(&y, &u, 4);
    return y;
}

void round_mat(Mat& m) {
    for (float& x : m.data) x = round_bf16(x);
}

Mat* find_mat(Model& m, const std::string& name) {
    if (name == "embedding") return &m.embedding;
    if (name == "unembed") return &m.unembed;
    // layer{l}.{wq,wk,wv,wo,gate} | layer{l}.expert{e}.{w_gate,w_up,w_down}
    if (name.rfind("layer", 0) != 0) return nullptr;
    std::size_t dot = name.find('.');
    int l = std::stoi(name.substr(5, dot - 5));
    if (l < 0 || l >= m.config.layers) return nullptr;
    LayerWeights& w = m.layers[l];
    std::string rest = name.substr(dot + 1);
    if (rest == "wq") return &w.wq;
    if (rest == "wk") return &w.wk;
    if (rest == "wv") return &w.wv;
    if (rest == "wo") return &w.wo;
    if (rest == "gate") return &w.gate;
    if (rest.rfind("expert", 0) == 0) {
        std::size_t d2 = rest.find('.');
        int e = std::stoi(rest.substr(6, d2 - 6));
        if (e < 0 || e >= m.config.experts) return nullptr;
        std::string t = rest.substr(d2 + 1);
        if (t == "w_gate") return &w.experts[e].w_gate;
        if (t == "w_up") return &w.experts[e].w_up;
        if (t == "w_down") return &w.experts[e].w_down;
    }
    return nullptr;
}

Vec* find_vec(Model& m, const std::string& name) {
    if (name == "final_norm_gain") return &m.final_norm_gain;
    if (name.rfind("layer", 0) != 0) return nullptr;
    std::size_t dot = name.find('.');
    int l = std::stoi(name.substr(5, dot - 5));
    if (l < 0 || l >= m.config.layers) return nullptr;
    std::string rest = name.substr(dot + 1);
    if (rest == "attn_norm_gain") return &m.layers[l].attn_norm_gain;
    if (rest == "moe_norm_gain") return &m.layers[l].moe_norm_gain;
    return nullptr;
}

// Records every predict_next call (the decision the executor will run next).
class RecordingPredictor final : public Predictor {
public:
    explicit RecordingPredictor(std::unique_ptr<Predictor> inner) : inner_(std::move(inner)) {}
    std::string_view name() const override { return inner_->name(); }
    Prediction predict_next(const Model& model, const Context& ctx) override {
        Prediction p = inner_->predict_next(model, ctx);
        if (sink_logits) {
            const int L = model.config.layers, E = model.config.experts, K = model.config.top_k;
            const std::size_t base = static_cast<std::size_t>(step) * (L - 1) + ctx.layer;
            if (!p.logits.empty())
                std::memcpy(sink_logits + base * E, p.logits.data(), sizeof(float) * E);
            for (int i = 0; i < K; ++i) {
                sink_ids[base * K + i] = p.decision.ids[i];
                sink_gates[base * K + i] = p.decision.gates[i];
            }
        }
        return p;
    }
    void observe_prompt_token(const Model& m, int t) override { inner_->observe_prompt_token(m, t); }
    void begin_token(const Model& m, int t) override { inner_->begin_token(m, t); }

    std::unique_ptr<Predictor> inner_;
    int step = 0;
    float* sink_logits = nullptr;
    int* sink_ids = nullptr;
    float* sink_gates = nullptr;
};

struct TraceBuffers {
    float* s;       // [S][L][H]
    float* r;       // [S][L][H]
    float* m;       // [S][L][H]
    float* logits;  // [S][L][E]  true router logits on the actual stream
    int* ids;       // [S][L][K]  executed decision
    float* gates;   // [S][L][K]
    float* outputs; // [S][L][K][H] raw expert outputs (nullable)
    float* final_logits; // [S][vocab]
};

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_free_model(void* h) { delete static_cast<Model*>(h); }

// build_model (model.cpp:112-158); optionally rounds every weight matrix to
// bf16 in place so the oracle sees exactly the values the GPU stores.
int ref_build_model(int L, int E, int K, int H, int Hm, int vocab, int hd, float eps,
                    std::uint64_t seed, int gating, int round_weights, void** out) {
    return guard([&] {
        ModelConfig c;
        c.layers = L;
        c.experts = E;
        c.top_k = K;
        c.hidden = H;
        c.expert_hidden = Hm;
        c.vocab = vocab;
        c.head_dim = hd;
        c.eps = eps;
        c.seed = seed;
        c.gating = gating == 0 ? GatingOrder::kSoftmaxThenTopK : GatingOrder::kTopKThenSoftmax;
        auto* m = new Model(build_model(c));
        if (round_weights) {
            round_mat(m->embedding);
            round_mat(m->unembed);
            for (LayerWeights& w : m->layers) {
                round_mat(w.wq);
                round_mat(w.wk);
                round_mat(w.wv);
                round_mat(w.wo);
                round_mat(w.gate);
                for (ExpertWeights& x : w.experts) {
                    round_mat(x.w_gate);
                    round_mat(x.w_up);
                    round_mat(x.w_down);
                }
            }
        }
        *out = m;
    });
}

// A Model with build_model's shapes (model.cpp:112-158) but zero weights, for
// callers that fill the tensors themselves (the bench fills it with the
// oracle's multithreaded generator; values are identical, tests pin that).
int ref_alloc_model(int L, int E, int K, int H, int Hm, int vocab, int hd, float eps,
                    std::uint64_t seed, int gating, void** out) {
    return guard([&] {
        ModelConfig c;
        c.layers = L;
        c.experts = E;
        c.top_k = K;
        c.hidden = H;
        c.expert_hidden = Hm;
        c.vocab = vocab;
        c.head_dim = hd;
        c.eps = eps;
        c.seed = seed;
        c.gating = gating == 0 ? GatingOrder::kSoftmaxThenTopK : GatingOrder::kTopKThenSoftmax;
        c.validate();
        auto* m = new Model();
        m->config = c;
        m->embedding = Mat(vocab, H);
        m->unembed = Mat(vocab, H);
        m->final_norm_gain.assign(H, 1.0f);
        m->layers.resize(L);
        for (LayerWeights& w : m->layers) {
            w.attn_norm_gain.assign(H, 1.0f);
            w.moe_norm_gain.assign(H, 1.0f);
            w.wq = Mat(hd, H);
            w.wk = Mat(hd, H);
            w.wv = Mat(hd, H);
            w.wo = Mat(H, hd);
            w.gate = Mat(E, H);
            w.experts.resize(E);
            for (ExpertWeights& x : w.experts) {
                x.w_gate = Mat(Hm, H);
                x.w_up = Mat(Hm, H);
                x.w_down = Mat(H, Hm);
            }
        }
        *out = m;
    });
}

// Returns the element count of a named tensor (0 if unknown); copies when out != null.
std::int64_t ref_model_tensor(void* h, const char* name, float* out) {
    Model& m = *static_cast<Model*>(h);
    if (Mat* mt = find_mat(m, name)) {
        if (out) std::memcpy(out, mt->data.data(), mt->data.size() * 4);
        return static_cast<std::int64_t>(mt->data.size());
    }
    if (Vec* v = find_vec(m, name)) {
        if (out) std::memcpy(out, v->data(), v->size() * 4);
        return static_cast<std::int64_t>(v->size());
    }
    return 0;
}

std::int64_t ref_model_set_tensor(void* h, const char* name, const float* in) {
    Model& m = *static_cast<Model*>(h);
    if (Mat* mt = find_mat(m, name)) {
        std::memcpy(mt->data.data(), in, mt->data.size() * 4);
        return static_cast<std::int64_t>(mt->data.size());
    }
    if (Vec* v = find_vec(m, name)) {
        std::memcpy(v->data(), in, v->size() * 4);
        return static_cast<std::int64_t>(v->size());
    }
    return 0;
}

// --- default vectors (speculation.cpp:23-83, trace.cpp:187-211) -------------

void ref_free_table(void* t) { delete static_cast<std::shared_ptr<const DefaultVectorTable>*>(t); }

int ref_calibrate_default_vectors(void* h, std::int64_t ntok, std::uint64_t seed, int seq_len,
                                  void** out) {
    return guard([&] {
        const Model& m = *static_cast<Model*>(h);
        const std::vector<int> toks = random_token_stream(ntok, m.config.vocab, seed);
        DefaultVectorAccumulator acc(m.config.layers, m.config.experts, m.config.hidden);
        stream_decode_trace(m, toks, seq_len,
                            [&](std::int64_t, const TraceToken& tok) { acc.add_token(tok); });
        *out = new std::shared_ptr<const DefaultVectorTable>(
            std::make_shared<DefaultVectorTable>(acc.freeze()));
    });
}

int ref_table_from(int L, int E, int H, const float* d, const std::int64_t* counts, void** out) {
    return guard([&] {
        auto t = std::make_shared<DefaultVectorTable>(DefaultVectorTable::zeros(L, E, H));
        for (std::size_t i = 0; i < t->d.size(); ++i) {
            std::memcpy(t->d[i].data(), d + i * H, sizeof(float) * H);
            t->counts[i] = counts ? counts[i] : 0;
        }
        *out = new std::shared_ptr<const DefaultVectorTable>(t);
    });
}

int ref_table_get(void* h, float* d, std::int64_t* counts) {
    return guard([&] {
        const DefaultVectorTable& t = **static_cast<std::shared_ptr<const DefaultVectorTable>*>(h);
        for (std::size_t i = 0; i < t.d.size(); ++i) {
            std::memcpy(d + i * t.hidden, t.d[i].data(), sizeof(float) * t.hidden);
            if (counts) counts[i] = t.counts[i];
        }
    });
}

// --- estimator (estimator.cpp:54-167) ----------------------------------------

void ref_free_estimator(void* e) { delete static_cast<std::shared_ptr<const EstimatorParams>*>(e); }

int ref_estimator_init(int d, int mred, int nexp, int E, int L, float eps, std::uint64_t seed,
                       void** out, std::int64_t* count) {
    return guard([&] {
        EstimatorConfig c;
        c.d = d;
        c.m = mred;
        c.n = nexp;
        c.experts = E;
        c.layers = L;
        c.eps = eps;
        c.seed = seed;
        auto p = std::make_shared<EstimatorParams>(init_estimator_params<float>(c));
        *count = static_cast<std::int64_t>(p->flat.size());
        *out = new std::shared_ptr<const EstimatorParams>(p);
    });
}

int ref_estimator_get(void* h, float* flat) {
    return guard([&] {
        const EstimatorParams& p = **static_cast<std::shared_ptr<const EstimatorParams>*>(h);
        std::memcpy(flat, p.flat.data(), p.flat.size() * 4);
    });
}

int ref_estimator_set(void* h, const float* flat) {
    return guard([&] {
        auto& sp = *static_cast<std::shared_ptr<const EstimatorParams>*>(h);
        auto p = std::make_shared<EstimatorParams>(*sp);
        std::memcpy(p->flat.data(), flat, p->flat.size() * 4);
        sp = p;
    });
}

int ref_estimator_logits(void* h, const float* q, int layer, float* out) {
    return guard([&] {
        const EstimatorParams& p = **static_cast<std::shared_ptr<const EstimatorParams>*>(h);
        Vec qv(q, q + p.config.d);
        Vec lg = estimator_logits(p, qv, layer);
        std::memcpy(out, lg.data(), lg.size() * 4);
    });
}

// train_estimator (estimator.cpp:374-450) on a DistillDataset given as flat
// arrays.  curve: n_curve x {tokens_seen, val_kl, val_hit_rate} as doubles.
int ref_train_estimator(int d, int mred, int nexp, int E, int L, float eps, std::uint64_t seed,
                        const float* inputs, const float* targets, std::int64_t tokens, double lr,
                        int batch, std::int64_t max_steps, std::int64_t eval_every,
                        double val_fraction, std::uint64_t hseed, int k, double early_stop,
                        float* params_out, double* curve_out, int curve_cap, int* n_curve) {
    return guard([&] {
        EstimatorConfig c;
        c.d = d;
        c.m = mred;
        c.n = nexp;
        c.experts = E;
        c.layers = L;
        c.eps = eps;
        c.seed = seed;
        DistillDataset data;
        data.d = d;
        data.experts = E;
        data.layers_predicting = L - 1;
        data.tokens = tokens;
        data.inputs.assign(inputs, inputs + tokens * (L - 1) * d);
        data.targets.assign(targets, targets + tokens * (L - 1) * E);
        TrainHyper h;
        h.lr = lr;
        h.batch_tokens = batch;
        h.max_steps = max_steps;
        h.eval_every = eval_every;
        h.val_fraction = val_fraction;
        h.seed = hseed;
        h.k = k;
        h.early_stop_hit_rate = early_stop;
        TrainResult r = train_estimator(data, c, h);
        std::memcpy(params_out, r.params.flat.data(), r.params.flat.size() * 4);
        *n_curve = static_cast<int>(r.curve.size());
        for (int i = 0; i < *n_curve && i < curve_cap; ++i) {
            curve_out[3 * i] = static_cast<double>(r.curve[i].tokens_seen);
            curve_out[3 * i + 1] = r.curve[i].val_kl;
            curve_out[3 * i + 2] = r.curve[i].val_hit_rate;
        }
    });
}

// DistillDatasetBuilder (speculation.cpp:437-471) fed with the records of
// forward_decode over `prompt` (one sequence from a fresh DecodeState).
// mode 0 quasi-hidden (table required), 1 s_{l+1}.
int ref_distill_dataset(void* h, const int* prompt, int P, void* table, int mode, float* inputs,
                        float* targets) {
    return guard([&] {
        const Model& model = *static_cast<Model*>(h);
        const int L = model.config.layers;
        const DefaultVectorTable* tb =
            table ? static_cast<std::shared_ptr<const DefaultVectorTable>*>(table)->get() : nullptr;
        DistillDatasetBuilder b(model, tb, mode == 0 ? DistillInput::kQuasiHidden : DistillInput::kSNext, P);
        DecodeState state(L);
        for (int i = 0; i < P; ++i) {
            TraceToken tok;
            tok.token_id = prompt[i];
            tok.layers.resize(static_cast<std::size_t>(L));
            TraceSink sink = [&](int l, const LayerTraceRecord& rec) { tok.layers[static_cast<std::size_t>(l)] = rec; };
            forward_decode(model, state, prompt[i], &sink);
            b.add_token(tok);
        }
        DistillDataset d = b.take();
        std::memcpy(inputs, d.inputs.data(), d.inputs.size() * 4);
        std::memcpy(targets, d.targets.data(), d.targets.size() * 4);
    });
}

// --- predictors (speculation.cpp:167-346) ------------------------------------

void ref_free_predictor(void* p) { delete static_cast<RecordingPredictor*>(p); }

// kind: 0 baseline-s, 1 router-pf, 2 est-pf, 3 hybrid, 4 oracle.
// hybrid_map: L-1 entries of kind codes (nullable -> all router-pf).
int ref_make_predictor(int kind, void* table, void* est, const int* hybrid_map, int L,
                       void** out) {
    return guard([&] {
        PredictorArtifacts art;
        if (table) art.table = *static_cast<std::shared_ptr<const DefaultVectorTable>*>(table);
        if (est) art.estimator = *static_cast<std::shared_ptr<const EstimatorParams>*>(est);
        if (hybrid_map) {
            HybridMap hm(static_cast<std::size_t>(L - 1));
            for (int l = 0; l < L - 1; ++l) hm[l] = static_cast<PredictorKind>(hybrid_map[l]);
            art.hybrid_map = hm;
        }
        *out = new RecordingPredictor(make_predictor(static_cast<PredictorKind>(kind), art, L));
    });
}

// generate() (speculation.cpp:401-421) re-driven step by step through the
// public forward_decode / speculative_forward so every per-(step, layer)
// record can be captured.  Step s < P is prefill token s; step P+i is decode
// step i.  S = P + n_new - 1 steps.  pred may be null (true path).
// pred_* buffers ([S][L-1][E] / [S][L-1][K]) record every predict_next call.
int ref_generate_trace(void* h, const int* prompt, int P, int n_new, void* pred,
                       int* out_tokens, float* s, float* r, float* m, float* logits, int* ids,
                       float* gates, float* outputs, float* final_logits, float* pred_logits,
                       int* pred_ids, float* pred_gates) {
    return guard([&] {
        const Model& model = *static_cast<Model*>(h);
        const ModelConfig& c = model.config;
        const int L = c.layers, H = c.hidden, E = c.experts, K = c.top_k;
        auto* rp = static_cast<RecordingPredictor*>(pred);
        if (rp) {
            rp->sink_logits = pred_logits;
            rp->sink_ids = pred_ids;
            rp->sink_gates = pred_gates;
        }
        int step = 0;
        TraceSink sink = [&](int l, const LayerTraceRecord& rec) {
            const std::size_t b = static_cast<std::size_t>(step) * L + l;
            if (s) std::memcpy(s + b * H, rec.s.data(), H * 4);
            if (r) std::memcpy(r + b * H, rec.r.data(), H * 4);
            if (m) std::memcpy(m + b * H, rec.m.data(), H * 4);
            if (logits) std::memcpy(logits + b * E, rec.router_logits.data(), E * 4);
            for (int i = 0; i < K; ++i) {
                if (ids) ids[b * K + i] = rec.decision.ids[i];
                if (gates) gates[b * K + i] = rec.decision.gates[i];
                if (outputs && !rec.expert_outputs.empty())
                    std::memcpy(outputs + (b * K + i) * H, rec.expert_outputs[i].data(), H * 4);
            }
        };
        if (P < 1) throw std::invalid_argument("generate: empty prompt");
        DecodeState state(L);
        Vec lg;
        for (int i = 0; i < P; ++i, ++step) {
            if (rp) rp->step = step;
            lg = forward_decode(model, state, prompt[i], &sink);
            if (final_logits) std::memcpy(final_logits + static_cast<std::size_t>(step) * c.vocab, lg.data(), c.vocab * 4);
            if (rp) rp->observe_prompt_token(model, prompt[i]);
        }
        int next = argmax_token(lg);
        for (int i = 0; i < n_new; ++i) {
            out_tokens[i] = next;
            if (i + 1 == n_new) break;
            if (rp) rp->step = step;
            lg = rp ? speculative_forward(model, state, next, *rp, &sink)
                    : forward_decode(model, state, next, &sink);
            if (final_logits) std::memcpy(final_logits + static_cast<std::size_t>(step) * c.vocab, lg.data(), c.vocab * 4);
            next = argmax_token(lg);
            ++step;
        }
    });
}

// Plain generate() as the reference ships it (used for CPU timing).
int ref_generate(void* h, const int* prompt, int P, int n_new, void* pred, int* out_tokens,
                 double* prefill_s, double* decode_s) {
    return guard([&] {
        const Model& model = *static_cast<Model*>(h);
        auto* rp = static_cast<RecordingPredictor*>(pred);
        if (rp) rp->sink_logits = nullptr;
        // Same body as generate(), with a clock around the two phases.
        DecodeState state(model.config.layers);
        Vec lg;
        auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < P; ++i) {
            lg = forward_decode(model, state, prompt[i]);
            if (rp) rp->observe_prompt_token(model, prompt[i]);
        }
        auto t1 = std::chrono::steady_clock::now();
        int next = argmax_token(lg);
        for (int i = 0; i < n_new; ++i) {
            out_tokens[i] = next;
            if (i + 1 == n_new) break;
            lg = rp ? speculative_forward(model, state, next, *rp) : forward_decode(model, state, next);
            next = argmax_token(lg);
        }
        auto t2 = std::chrono::steady_clock::now();
        if (prefill_s) *prefill_s = std::chrono::duration<double>(t1 - t0).count();
        if (decode_s) *decode_s = std::chrono::duration<double>(t2 - t1).count();
    });
}

// run_offloaded_decode (executor.cpp:326-359).  mode 0 on_demand, 1 prefetch.
int ref_offloaded_decode(void* h, const int* prompt, int P, int n_new, void* pred, int mode,
                         std::int64_t latency_us, double deadlock_factor, int* out_tokens,
                         double* per_token_us, int* max_resident) {
    return guard([&] {
        const Model& model = *static_cast<Model*>(h);
        auto* rp = static_cast<RecordingPredictor*>(pred);
        if (rp) rp->sink_logits = nullptr;
        ExecutorOptions o;
        o.mode = mode == 0 ? OffloadMode::kOnDemand : OffloadMode::kPrefetch;
        o.copy_latency_us = latency_us;
        o.deadlock_factor = deadlock_factor;
        ExecutorResult res = run_offloaded_decode(model, std::span<const int>(prompt, P), n_new,
                                                  rp, o);
        for (std::size_t i = 0; i < res.tokens.size(); ++i) out_tokens[i] = res.tokens[i];
        for (std::size_t i = 0; i < res.per_token_us.size(); ++i) per_token_us[i] = res.per_token_us[i];
        if (max_resident) *max_resident = res.max_resident_layers;
    });
}

// --- leaf numerics (numerics.cpp, model.cpp:258-304) -------------------------

// The reference's own trace capture (cmd_trace, main.cpp:90-147): the true path
// over `tokens` with state resets every seq_len tokens (stream_decode_trace,
// trace.cpp:187-203), written by TraceWriter (trace.cpp:60-122).
int ref_write_trace(void* h, const int* tokens, std::int64_t n, int seq_len, const char* dir,
                    const char* source, std::uint64_t seed) {
    return guard([&] {
        const Model& m = *static_cast<Model*>(h);
        TraceManifest man;
        man.config = m.config;
        man.tokens = n;
        man.seq_len = seq_len;
        man.source = source;
        man.seed = seed;
        TraceWriter w(dir, man);
        stream_decode_trace(m, std::span<const int>(tokens, static_cast<size_t>(n)), seq_len,
                            [&](std::int64_t, const TraceToken& t) { w.add_token(t.token_id, t.layers); });
        w.finish();
    });
}

std::uint64_t ref_derive_seed(std::uint64_t seed, const char* label) { return derive_seed(seed, label); }

void ref_gaussian_stream(std::uint64_t seed, float stddev, std::int64_t n, float* out) {
    Rng rng(seed);
    for (std::int64_t i = 0; i < n; ++i) out[i] = rng.next_gaussian(stddev);
}

int ref_softmax(const float* v, int n, float* out) {
    return guard([&] {
        Vec o = softmax(Vec(v, v + n));
        std::memcpy(out, o.data(), n * 4);
    });
}

int ref_top_k(const float* v, int n, int k, int* idx) {
    return guard([&] {
        TopK t = top_k(Vec(v, v + n), k);
        for (int i = 0; i < k; ++i) idx[i] = t.indices[i];
    });
}

int ref_rms_norm(const float* v, const float* g, int n, float eps, float* out) {
    return guard([&] {
        Vec o = rms_norm(Vec(v, v + n), Vec(g, g + n), eps);
        std::memcpy(out, o.data(), n * 4);
    });
}

float ref_silu(float x) { return silu(x); }

int ref_make_decision(const float* logits, int E, int k, int gating, int* ids, float* gates) {
    return guard([&] {
        RouterDecision d = make_decision(Vec(logits, logits + E), k,
                                         gating == 0 ? GatingOrder::kSoftmaxThenTopK
                                                     : GatingOrder::kTopKThenSoftmax);
        for (int i = 0; i < k; ++i) {
            ids[i] = d.ids[i];
            gates[i] = d.gates[i];
        }
    });
}

int ref_linear(const float* w, int rows, int cols, const float* x, float* out) {
    return guard([&] {
        Mat m(rows, cols);
        std::memcpy(m.data.data(), w, sizeof(float) * rows * cols);
        Vec o = linear(m, Vec(x, x + cols));
        std::memcpy(out, o.data(), rows * 4);
    });
}

int ref_layer_default(void* table, const int* ids, const float* gates, int k, int layer,
                      float* out) {
    return guard([&] {
        const DefaultVectorTable& t = **static_cast<std::shared_ptr<const DefaultVectorTable>*>(table);
        RouterDecision d;
        d.ids.assign(ids, ids + k);
        d.gates.assign(gates, gates + k);
        Vec o = layer_default(t, d, layer);
        std::memcpy(out, o.data(), o.size() * 4);
    });
}

// --- schedule model (schedule.cpp:92-217) ------------------------------------

int ref_simulate(int L, const double* attn, const double* gate, const double* expert,
                 const double* copy, double cold, int prefetch, double* tpot, double* fracs,
                 double* analytic) {
    return guard([&] {
        TimingModel tm;
        tm.t_attn.assign(attn, attn + L);
        tm.t_gate_topk.assign(gate, gate + L);
        tm.t_expert.assign(expert, expert + L);
        tm.t_copy.assign(copy, copy + L);
        tm.cold_start_copy = cold;
        ScheduleReport rep = prefetch ? simulate_prefetch(tm) : simulate_on_demand(tm);
        *tpot = rep.tpot;
        BreakdownFractions f = breakdown(rep);
        fracs[0] = f.compute_frac;
        fracs[1] = f.copy_frac;
        fracs[2] = f.idle_frac;
        *analytic = analytic_improvement(tm);
    });
}

// per_token_reports (executor.cpp:361-382) + breakdown over an event list.
int ref_breakdown_events(const int* lane, const int* kind, const int* layer, const int* token,
                         const double* start_us, const double* end_us, int n, double* mean_fr,
                         double* mean_tpot) {
    return guard([&] {
        ExecutorResult r;
        for (int i = 0; i < n; ++i)
            r.events.push_back({lane[i] == 0 ? Lane::kCompute : Lane::kCopy,
                                static_cast<EventKind>(kind[i]), layer[i], start_us[i], end_us[i],
                                token[i]});
        auto reps = per_token_reports(r);
        double acc[3] = {0, 0, 0}, tp = 0;
        int c = 0;
        for (auto& rep : reps) {
            if (rep.events.empty()) continue;
            BreakdownFractions f = breakdown(rep);
            acc[0] += f.compute_frac;
            acc[1] += f.copy_frac;
            acc[2] += f.idle_frac;
            tp += rep.tpot;
            ++c;
        }
        for (int k = 0; k < 3; ++k) mean_fr[k] = c ? acc[k] / c : 0;
        *mean_tpot = c ? tp / c : 0;
    });
}

} // extern "C"
