// capi.cpp — extern "C" boundary (include/smoe.h) over the C++ Session.
// Exceptions never cross the ABI: std::invalid_argument -> 1, others -> 2,
// message kept in a thread-local string (the reference's exception
// convention, SURVEY §8b "Errors").
#include "../../include/smoe.h"

#include "engine.h"
#include <vector>
#include <algorithm>
#include <map>
#include "train.h"

#include <cstring>
#include <string>

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
    } catch (...) {
        g_err = "unknown error";
        return 2;
    }
}

}  // namespace

void smoe_set_last_error(const std::string& msg) { g_err = msg; }

namespace {
smoe::Session* S(smoe_session* s) {
    if (!s) throw std::invalid_argument("null session");
    return reinterpret_cast<smoe::Session*>(s);
}
}  // namespace

extern "C" {

const char* smoe_last_error(void) { return g_err.c_str(); }

int smoe_session_create(const smoe_config* cfg, const smoe_options* opt, smoe_session** out) {
    return guard([&] {
        if (!cfg || !out) throw std::invalid_argument("null argument");
        smoe::ModelCfg c{cfg->layers, cfg->experts, cfg->top_k, cfg->hidden, cfg->expert_hidden,
                         cfg->vocab, cfg->head_dim, cfg->eps, cfg->seed, cfg->gating};
        smoe::SessionOpts o;
        if (opt) {
            o.device = opt->device;
            o.cache_fraction = opt->cache_fraction;
            o.max_positions = opt->max_positions;
            o.copy_latency_us = opt->copy_latency_us;
            o.deadlock_s = opt->deadlock_s > 0 ? opt->deadlock_s : 10.0;
            o.ep_rank = opt->ep_rank;
            o.ep_world = opt->ep_world > 0 ? opt->ep_world : 1;
        }
        *out = reinterpret_cast<smoe_session*>(new smoe::Session(c, o));
    });
}

int smoe_session_destroy(smoe_session* s) {
    return guard([&] { delete S(s); });
}

int smoe_init_weights_seeded(smoe_session* s) {
    return guard([&] { S(s)->init_weights_seeded(); });
}

int smoe_load_tensor(smoe_session* s, const char* name, const float* data, int64_t count) {
    return guard([&] {
        if (!name || !data) throw std::invalid_argument("null argument");
        S(s)->load_tensor(name, data, count);
    });
}

int smoe_load_default_vectors(smoe_session* s, const float* d, int64_t count) {
    return guard([&] {
        const auto& c = S(s)->cfg();
        if (!d || count != static_cast<int64_t>(c.L) * c.E * c.H)
            throw std::invalid_argument("default vectors must be [L][E][H]");
        S(s)->load_default_vectors(d);
    });
}

int smoe_load_estimator(smoe_session* s, const smoe_estimator_config* c, const float* flat,
                        int64_t count) {
    return guard([&] {
        if (!c || !flat) throw std::invalid_argument("null argument");
        if (c->m <= 1 || c->n <= 1 || c->d % c->m != 0)
            throw std::invalid_argument("estimator: m and n must be > 1, d divisible by m");
        const int64_t dm = c->d / c->m, mlp = dm * c->n;
        const int64_t want = c->d * dm + static_cast<int64_t>(c->layers) * dm + 2 * mlp * dm +
                             2 * dm + dm * c->experts;
        if (count != want) throw std::invalid_argument("estimator: flat parameter count mismatch");
        smoe::EstCfg e{c->d, c->m, c->n, c->experts, c->layers, c->eps};
        S(s)->load_estimator(e, flat);
    });
}

int smoe_set_predictor(smoe_session* s, int32_t kind, const int32_t* hybrid_map) {
    return guard([&] { S(s)->set_predictor(kind, hybrid_map); });
}

int smoe_set_cache_fraction(smoe_session* s, float f) {
    return guard([&] { S(s)->set_cache_fraction(f); });
}

int smoe_reset(smoe_session* s, int32_t max_steps, int32_t trace_full) {
    return guard([&] {
        if (max_steps < 0) throw std::invalid_argument("max_steps must be >= 0");
        S(s)->reset(max_steps, trace_full);
    });
}

int smoe_prefill_batched(smoe_session* s, const int32_t* tokens, int32_t n) {
    return guard([&] {
        if (!tokens && n > 0) throw std::invalid_argument("null tokens");
        S(s)->prefill_batched(tokens, n);
    });
}

int smoe_prefill(smoe_session* s, const int32_t* tokens, int32_t n) {
    return guard([&] {
        if (!tokens && n > 0) throw std::invalid_argument("null tokens");
        S(s)->prefill(tokens, n);
    });
}

int smoe_decode(smoe_session* s, int32_t mode, int32_t n_steps, int32_t use_graph) {
    return guard([&] {
        if (mode != 0 && mode != 1) throw std::invalid_argument("unknown offload mode");
        S(s)->decode(mode, n_steps, use_graph);
    });
}

int smoe_decode_stream(smoe_session* s, int32_t mode, const int32_t* tokens, int32_t n_steps) {
    return guard([&] {
        if (mode != 0 && mode != 1) throw std::invalid_argument("unknown offload mode");
        if (!tokens && n_steps > 0) throw std::invalid_argument("null tokens");
        S(s)->decode_stream(mode, tokens, n_steps);
    });
}

int smoe_run_offloaded_decode(smoe_session* s, const int32_t* prompt, int32_t n_prompt,
                              int32_t n_new, int32_t mode, int32_t* out_tokens,
                              double* per_token_ms) {
    return guard([&] {
        if (n_prompt < 1 || !prompt) throw std::invalid_argument("offloaded decode: empty prompt");
        if (n_new < 1) throw std::invalid_argument("offloaded decode: n_new must be >= 1");
        if (mode != 0 && mode != 1) throw std::invalid_argument("unknown offload mode");
        smoe::Session* ss = S(s);
        ss->reset(n_prompt + n_new, 0);
        ss->prefill(prompt, n_prompt);
        ss->decode(mode, n_new - 1, 1);
        std::vector<int> toks(n_prompt + n_new - 1);
        ss->read_tokens(toks.data(), static_cast<int>(toks.size()));
        for (int i = 0; i < n_new; ++i) out_tokens[i] = toks[n_prompt - 1 + i];
        if (per_token_ms) {
            auto v = ss->token_ms();
            for (size_t i = 0; i < v.size() && i < static_cast<size_t>(n_new - 1); ++i) per_token_ms[i] = v[i];
        }
    });
}

// ExecutorResult (executor.hpp:39-44) in full: the decode runs with the
// measured lane events (CUDA events per phase, no graph), so tokens, events,
// per-token times and the residency bound come from the same run, like the
// reference's (executor.cpp:326-408).  max_resident_layers: the most layers
// whose experts were requested (copy issued or hit) and not yet consumed by
// their expert kernel at any instant (the reference's bound is 2,
// executor.cpp:159-162; Algorithm 1 keeps it at 2 here too).
int smoe_run_offloaded_decode_ex(smoe_session* s, const int32_t* prompt, int32_t n_prompt,
                                 int32_t n_new, int32_t mode, int32_t* out_tokens,
                                 double* per_token_ms, smoe_event* events, int32_t cap,
                                 int32_t* n_events, int32_t* max_resident_layers) {
    return guard([&] {
        if (n_prompt < 1 || !prompt) throw std::invalid_argument("offloaded decode: empty prompt");
        if (n_new < 1) throw std::invalid_argument("offloaded decode: n_new must be >= 1");
        if (mode != 0 && mode != 1) throw std::invalid_argument("unknown offload mode");
        smoe::Session* ss = S(s);
        ss->reset(n_prompt + n_new, 0);
        ss->prefill(prompt, n_prompt);
        std::vector<smoe::TimelineEvent> ev;
        ss->decode_timeline(mode, nullptr, n_new - 1, ev);
        std::vector<int> toks(n_prompt + n_new - 1);
        ss->read_tokens(toks.data(), static_cast<int>(toks.size()));
        for (int i = 0; i < n_new; ++i) out_tokens[i] = toks[n_prompt - 1 + i];
        const int steps = n_new - 1;
        std::vector<double> t0(steps, 1e300), t1(steps, -1e300);
        for (const auto& e : ev)
            if (e.lane == 0 && e.token >= 0 && e.token < steps) {
                t0[e.token] = std::min(t0[e.token], e.start_ms);
                t1[e.token] = std::max(t1[e.token], e.end_ms);
            }
        if (per_token_ms)
            for (int i = 0; i < steps; ++i) per_token_ms[i] = t1[i] - t0[i];
        // residency: interval [decision end (request posted), expert end] per
        // (token, layer).  The routing events are recorded in issue order: on
        // demand, routing at layer l decides l; in prefetch mode the first one
        // of a token (the true router of layer 0) decides layer 0 and every
        // later one at layer l is the predictor deciding l + 1.
        std::map<std::pair<int, int>, std::pair<double, double>> span;
        std::map<int, int> seen0;
        for (const auto& e : ev) {
            if (e.lane != 0 || e.token < 0) continue;
            int dl = e.layer;
            if (e.kind == 1 && mode == 1 && !(e.layer == 0 && seen0[e.token]++ == 0)) dl = e.layer + 1;
            auto& sp = span.try_emplace({e.token, dl}, 1e300, -1e300).first->second;
            if (e.kind == 1) sp.first = std::min(sp.first, e.end_ms);  // request posted
            if (e.kind == 2) sp.second = std::max(sp.second, e.end_ms);
        }
        std::vector<std::pair<double, int>> marks;
        for (auto& [k, sp] : span)
            if (sp.first < sp.second) {
                marks.push_back({sp.first, +1});
                marks.push_back({sp.second, -1});
            }
        std::sort(marks.begin(), marks.end(),
                  [](const auto& a, const auto& b) { return a.first < b.first || (a.first == b.first && a.second < b.second); });
        int cur = 0, mx = 0;
        for (auto& mk : marks) mx = std::max(mx, cur += mk.second);
        if (max_resident_layers) *max_resident_layers = mx;
        const int m = static_cast<int>(ev.size()) < cap ? static_cast<int>(ev.size()) : cap;
        if (events)
            for (int i = 0; i < m; ++i)
                events[i] = smoe_event{ev[i].lane, ev[i].kind, ev[i].layer, ev[i].token, ev[i].start_ms,
                                       ev[i].end_ms};
        if (n_events) *n_events = static_cast<int32_t>(ev.size());
    });
}

int smoe_step(smoe_session* s, int32_t mode, int32_t token, float* logits_out, int32_t* next) {
    return guard([&] {
        if (mode != 0 && mode != 1) throw std::invalid_argument("unknown offload mode");
        const int t = S(s)->step_host(mode, token, logits_out);
        if (next) *next = t;
    });
}

int smoe_calibrate(smoe_session* s, int64_t ntok, uint64_t seed, int32_t seq_len, float* d_out,
                   int64_t* counts_out) {
    return guard([&] {
        S(s)->calibrate(ntok, seed, seq_len, d_out, reinterpret_cast<long long*>(counts_out));
    });
}

int smoe_steps_done(smoe_session* s, int32_t* n) {
    return guard([&] { *n = S(s)->steps_done(); });
}

int smoe_read_tokens(smoe_session* s, int32_t* out, int32_t n) {
    return guard([&] { S(s)->read_tokens(out, n); });
}

int smoe_read_trace(smoe_session* s, const char* field, void* out, int64_t n) {
    return guard([&] { S(s)->read_trace(field, out, n); });
}

int smoe_build_distill_dataset(smoe_session* s, int32_t first, int32_t n, int32_t mode, float* inputs,
                               float* targets) {
    return guard([&] { S(s)->build_distill_dataset(first, n, mode, inputs, targets); });
}

int smoe_predict_ahead(smoe_session* s, int32_t first, int32_t n, int32_t depth, int32_t* ids) {
    return guard([&] { S(s)->predict_ahead(first, n, depth, ids); });
}

int smoe_batch_generate(smoe_session* s, int32_t batch, const int32_t* prompts, int32_t prompt_len,
                        int32_t n_new, int32_t mode, int32_t* out_tokens, float* out_logits,
                        double* step_ms) {
    return guard([&] {
        S(s)->batch_generate(batch, prompts, prompt_len, n_new, mode, out_tokens, out_logits, step_ms);
    });
}

int smoe_write_trace_bundle(smoe_session* s, const char* dir, int32_t first, int32_t n,
                            int32_t seq_len, const char* source, uint64_t seed) {
    return guard([&] { S(s)->write_trace_bundle(dir, first, n, seq_len, source ? source : "", seed); });
}

int smoe_token_ms(smoe_session* s, double* out, int32_t cap, int32_t* n) {
    return guard([&] {
        auto v = S(s)->token_ms();
        const int m = static_cast<int>(v.size()) < cap ? static_cast<int>(v.size()) : cap;
        for (int i = 0; i < m; ++i) out[i] = v[i];
        *n = static_cast<int32_t>(v.size());
    });
}

int smoe_counters(smoe_session* s, int64_t* hits, int64_t* misses, int64_t* h2d_bytes,
                  double* copy_ms, int32_t* requests) {
    return guard([&] {
        long long b = 0;
        int req = 0;
        double ms = 0;
        S(s)->counters(reinterpret_cast<long long*>(hits), reinterpret_cast<long long*>(misses), &b,
                       &ms, &req);
        if (h2d_bytes) *h2d_bytes = b;
        if (copy_ms) *copy_ms = ms;
        if (requests) *requests = req;
    });
}

int smoe_copy_events(smoe_session* s, smoe_copy_event* out, int32_t cap, int32_t* n) {
    return guard([&] {
        smoe::Session* ss = S(s);
        ss->counters(nullptr, nullptr, nullptr, nullptr, nullptr);  // syncs both streams
        auto recs = ss->copy_records();
        int m = 0;
        for (const auto& r : recs) {
            if (m >= cap) break;
            smoe_copy_event& e = out[m++];
            e.seq = r.seq;
            e.layer = r.layer;
            e.step = r.step;
            e.hits = r.hits;
            e.misses = r.misses;
            e.bytes = r.bytes;
            e.start_ms = r.ev >= 0 ? ss->event_ms(r.ev, 0) : -1.0;
            e.end_ms = r.ev >= 0 ? ss->event_ms(r.ev, 1) : -1.0;
        }
        *n = static_cast<int32_t>(recs.size());
    });
}

int smoe_cache_slots(smoe_session* s, int32_t* slots) {
    return guard([&] {
        smoe::Session* ss = S(s);
        const auto& c = ss->cfg();
        (void)c;
        *slots = ss->slots_per_layer();
    });
}

int smoe_timeline(smoe_session* s, int32_t mode, const int32_t* tokens, int32_t n_steps,
                  smoe_event* out, int32_t cap, int32_t* n) {
    return guard([&] {
        if (mode != 0 && mode != 1) throw std::invalid_argument("unknown offload mode");
        std::vector<smoe::TimelineEvent> ev;
        S(s)->decode_timeline(mode, tokens, n_steps, ev);
        const int m = static_cast<int>(ev.size()) < cap ? static_cast<int>(ev.size()) : cap;
        for (int i = 0; i < m; ++i)
            out[i] = smoe_event{ev[i].lane, ev[i].kind, ev[i].layer, ev[i].token, ev[i].start_ms,
                                ev[i].end_ms};
        *n = static_cast<int32_t>(ev.size());
    });
}

int smoe_set_decode_mode(smoe_session* s, int32_t mode) {
    return guard([&] { S(s)->set_decode_mode(mode); });
}

int smoe_set_prefill_mode(smoe_session* s, int32_t mode) {
    return guard([&] { S(s)->set_prefill_mode(mode); });
}

int smoe_path_info(smoe_session* s, int32_t* out, int32_t cap) {
    return guard([&] { S(s)->path_info(out, cap); });
}

int smoe_xp_pack(const uint16_t* raw, int64_t n, uint8_t* out, int64_t cap, int64_t* packed_bytes) {
    return guard([&] {
        if (!raw || !out || !packed_bytes || n < 0 || cap < 0) throw std::invalid_argument("xp_pack: bad arguments");
        *packed_bytes = smoe::xp_pack(raw, n, out, cap);
    });
}

int smoe_xp_unpack(const uint8_t* packed, uint16_t* out, int64_t n) {
    return guard([&] {
        if (!packed || !out) throw std::invalid_argument("xp_unpack: bad arguments");
        uint32_t hdr[4];
        std::memcpy(hdr, packed, sizeof hdr);
        if (hdr[0] != smoe::kXpMagic) throw std::invalid_argument("xp_unpack: not a packed expert block");
        if (static_cast<int64_t>(hdr[1]) * smoe::kXpGroup != n)
            throw std::invalid_argument("xp_unpack: element count mismatch");
        smoe::xp_unpack(packed, out);
    });
}

int smoe_debug_state(smoe_session* s, int32_t* out, int32_t cap) {
    return guard([&] { S(s)->debug_state(out, cap); });
}

int smoe_ep_buffers(smoe_session* s, void** xbuf, void** counters) {
    return guard([&] {
        if (!xbuf || !counters) throw std::invalid_argument("null argument");
        S(s)->ep_buffers(xbuf, counters);
    });
}

int smoe_ep_ipc_handles(smoe_session* s, unsigned char* out128) {
    return guard([&] {
        if (!out128) throw std::invalid_argument("null argument");
        S(s)->ep_ipc_handles(out128);
    });
}

int smoe_ep_connect(smoe_session* s, void* const* xbufs, void* const* counters) {
    return guard([&] {
        if (!xbufs || !counters) throw std::invalid_argument("null argument");
        S(s)->ep_connect(xbufs, counters);
    });
}

int smoe_ep_connect_ipc(smoe_session* s, const unsigned char* handles) {
    return guard([&] {
        if (!handles) throw std::invalid_argument("null argument");
        S(s)->ep_connect_ipc(handles);
    });
}

int smoe_preload_all(smoe_session* s) {
    return guard([&] { S(s)->preload_all(); });
}

int smoe_clear_stats(smoe_session* s) {
    return guard([&] { S(s)->clear_stats(); });
}

int smoe_profile_kernels(smoe_session* s, int32_t reps, double* out_us) {
    return guard([&] {
        if (reps < 1 || !out_us) throw std::invalid_argument("profile: reps >= 1 and out[7] required");
        S(s)->profile_kernels(reps, out_us);
    });
}

int smoe_measure_link(smoe_session* s, int32_t n_copies, double* gbps) {
    return guard([&] {
        if (n_copies < 1 || !gbps) throw std::invalid_argument("measure_link: n_copies >= 1");
        *gbps = S(s)->measure_link(n_copies);
    });
}

int smoe_kernels_per_step(smoe_session* s, int32_t mode, int32_t* n) {
    return guard([&] { *n = S(s)->kernels_per_step(mode); });
}

}  // extern "C"

namespace {
smoe::EstTrainCfg est_cfg(const smoe_estimator_config* c, uint64_t seed) {
    if (!c) throw std::invalid_argument("null estimator config");
    return smoe::EstTrainCfg{c->d, c->m, c->n, c->experts, c->layers, c->eps, seed};
}
}  // namespace

int smoe_estimator_param_count(const smoe_estimator_config* c, int64_t* n) {
    return guard([&] { *n = static_cast<int64_t>(smoe::estimator_init_params(est_cfg(c, 0)).size()); });
}

int smoe_estimator_init(const smoe_estimator_config* c, uint64_t seed, float* flat, int64_t cap) {
    return guard([&] {
        const std::vector<float> p = smoe::estimator_init_params(est_cfg(c, seed));
        if (cap < static_cast<int64_t>(p.size())) throw std::invalid_argument("estimator init: buffer too small");
        std::memcpy(flat, p.data(), p.size() * 4);
    });
}

int smoe_train_estimator(const smoe_estimator_config* c, uint64_t seed, const float* inputs,
                         const float* targets, int64_t tokens, int32_t layers_predicting,
                         const smoe_train_hyper* h, float* params_out, int64_t params_cap,
                         smoe_curve_point* curve_out, int32_t curve_cap, int32_t* n_curve,
                         double* train_ms) {
    return guard([&] {
        if (!h || !inputs || !targets || !params_out) throw std::invalid_argument("train: null argument");
        const smoe::EstTrainCfg cfg = est_cfg(c, seed);
        const int64_t need = static_cast<int64_t>(smoe::estimator_init_params(cfg).size());
        if (params_cap < need) throw std::invalid_argument("train: params buffer too small");
        const smoe::EstTrainHyper hy{h->lr, h->batch_tokens, h->max_steps, h->eval_every,
                                     h->val_fraction, h->seed, h->k, h->early_stop_hit_rate};
        const std::vector<smoe::EstCurvePoint> curve = smoe::train_estimator_gpu(
            cfg, inputs, targets, tokens, layers_predicting, hy, params_out, train_ms);
        if (n_curve) *n_curve = static_cast<int32_t>(curve.size());
        for (size_t i = 0; i < curve.size() && static_cast<int64_t>(i) < curve_cap && curve_out; ++i)
            curve_out[i] = smoe_curve_point{curve[i].tokens_seen, curve[i].val_kl, curve[i].val_hit_rate};
    });
}

int smoe_decide(const float* logits, int32_t rows, int32_t E, int32_t K, int32_t gating, int32_t* ids,
                float* gates) {
    return guard([&] {
        if (rows < 0 || E < 1 || E > smoe::kMaxE || K < 1 || K > E || K > smoe::kMaxK || (gating != 0 && gating != 1))
            throw std::invalid_argument("smoe_decide: bad arguments");
        if (rows == 0) return;
        float *dl = nullptr, *dg = nullptr;
        int* di = nullptr;
        auto ck = [](cudaError_t e) {
            if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error in smoe_decide: ") + cudaGetErrorString(e));
        };
        ck(cudaMalloc(&dl, 4ull * rows * E));
        ck(cudaMalloc(&di, 4ull * rows * K));
        ck(cudaMalloc(&dg, 4ull * rows * K));
        cudaError_t e = cudaMemcpy(dl, logits, 4ull * rows * E, cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = smoe::launch_decide(dl, rows, E, K, gating, di, dg, nullptr);
        if (e == cudaSuccess) e = cudaMemcpy(ids, di, 4ull * rows * K, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess) e = cudaMemcpy(gates, dg, 4ull * rows * K, cudaMemcpyDeviceToHost);
        cudaFree(dl);
        cudaFree(di);
        cudaFree(dg);
        ck(e);
    });
}

int smoe_exp(const double* x, double* y, int64_t n) {
    return guard([&] {
        if (n < 0 || (n && (!x || !y))) throw std::invalid_argument("smoe_exp: bad arguments");
        double *dx = nullptr, *dy = nullptr;
        auto ck = [](cudaError_t e) {
            if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error in smoe_exp: ") + cudaGetErrorString(e));
        };
        ck(cudaMalloc(&dx, 8 * std::max<int64_t>(n, 1)));
        ck(cudaMalloc(&dy, 8 * std::max<int64_t>(n, 1)));
        cudaError_t e = cudaMemcpy(dx, x, 8 * n, cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = smoe::launch_exp_glibc(dx, dy, n, nullptr);
        if (e == cudaSuccess) e = cudaMemcpy(y, dy, 8 * n, cudaMemcpyDeviceToHost);
        cudaFree(dx);
        cudaFree(dy);
        ck(e);
    });
}
