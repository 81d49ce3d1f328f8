// specmoe_b200.cpp — the C++ drop-in (specmoe_b200.hpp) over the C ABI.
//
// Maps the reference's decode API onto include/smoe.h: the Model's tensors
// are uploaded once per Model object (the reference treats Model as
// immutable and shareable) into a session that keeps the pinned
// bf16 expert store, the HBM slot pool and the copy lane; the predictor's
// artifacts (default-vector table, estimator, hybrid map) are uploaded per
// call.  Errors come back as the reference's exception types.
#include "specmoe_b200.hpp"

#include "../../include/smoe.h"

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>

namespace specmoe_b200 {

namespace {

void check(int rc) {
    if (rc == 0) return;
    const std::string msg = smoe_last_error();
    if (rc == 1) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

int pred_code(specmoe::PredictorKind k) {
    switch (k) {
    case specmoe::PredictorKind::kBaselineS: return SMOE_PRED_BASELINE_S;
    case specmoe::PredictorKind::kRouterPF: return SMOE_PRED_ROUTER_PF;
    case specmoe::PredictorKind::kEstPF: return SMOE_PRED_EST_PF;
    case specmoe::PredictorKind::kHybridPF: return SMOE_PRED_HYBRID;
    case specmoe::PredictorKind::kOracle: return SMOE_PRED_ORACLE;
    }
    throw std::invalid_argument("unknown predictor kind");
}

DeviceOptions g_opts;

// One session per (Model object, device options), weights uploaded once.
struct Cached {
    smoe_session* s = nullptr;
    int max_positions = 0;
    float cache_fraction = 0.0f;
    bool resident = false;
};
std::mutex g_mu;
std::map<const specmoe::Model*, Cached> g_sessions;

void upload_model(smoe_session* s, const specmoe::Model& model) {
    const auto& c = model.config;
    auto put = [&](const std::string& name, const float* p, size_t n) {
        check(smoe_load_tensor(s, name.c_str(), p, static_cast<int64_t>(n)));
    };
    put("embedding", model.embedding.data.data(), model.embedding.data.size());
    put("unembed", model.unembed.data.data(), model.unembed.data.size());
    put("final_norm_gain", model.final_norm_gain.data(), model.final_norm_gain.size());
    for (int l = 0; l < c.layers; ++l) {
        const auto& w = model.layers[static_cast<size_t>(l)];
        const std::string p = "layer" + std::to_string(l) + ".";
        put(p + "attn_norm_gain", w.attn_norm_gain.data(), w.attn_norm_gain.size());
        put(p + "moe_norm_gain", w.moe_norm_gain.data(), w.moe_norm_gain.size());
        put(p + "wq", w.wq.data.data(), w.wq.data.size());
        put(p + "wk", w.wk.data.data(), w.wk.data.size());
        put(p + "wv", w.wv.data.data(), w.wv.data.size());
        put(p + "wo", w.wo.data.data(), w.wo.data.size());
        put(p + "gate", w.gate.data.data(), w.gate.data.size());
        for (int e = 0; e < c.experts; ++e) {
            const auto& x = w.experts[static_cast<size_t>(e)];
            const std::string q = p + "expert" + std::to_string(e) + ".";
            put(q + "w_gate", x.w_gate.data.data(), x.w_gate.data.size());
            put(q + "w_up", x.w_up.data.data(), x.w_up.data.size());
            put(q + "w_down", x.w_down.data.data(), x.w_down.data.size());
        }
    }
}

smoe_session* session_for(const specmoe::Model& model, int positions, bool resident,
                          const specmoe::ExecutorOptions* eo) {
    model.config.validate();  // the reference's own invariants first (model.cpp:25-37)
    const auto& c = model.config;
    Cached& cs = g_sessions[&model];
    const float frac = resident ? 1.0f : g_opts.cache_fraction;
    if (!cs.s || cs.max_positions < positions) {
        if (cs.s) smoe_session_destroy(cs.s);
        cs = Cached{};
        smoe_config cfg{c.layers, c.experts, c.top_k, c.hidden, c.expert_hidden, c.vocab, c.head_dim,
                        c.eps, c.seed, c.gating == specmoe::GatingOrder::kSoftmaxThenTopK ? 0 : 1};
        smoe_options opt{};
        opt.device = g_opts.device;
        opt.cache_fraction = frac;
        opt.max_positions = std::max(positions, 256);
        opt.deadlock_s = 10.0;
        opt.ep_world = 1;
        smoe_session* s = nullptr;
        check(smoe_session_create(&cfg, &opt, &s));
        cs.s = s;
        cs.max_positions = opt.max_positions;
        cs.cache_fraction = frac;
        upload_model(s, model);
    }
    if (cs.cache_fraction != frac) {
        check(smoe_set_cache_fraction(cs.s, frac));
        cs.cache_fraction = frac;
        cs.resident = false;
    }
    if (resident && !cs.resident) {
        check(smoe_preload_all(cs.s));
        cs.resident = true;
    }
    (void)eo;
    return cs.s;
}

// The predictor's artifacts into the session; returns the SMOE_PRED_* code.
int install_predictor(smoe_session* s, const specmoe::Model& model, specmoe::Predictor* predictor) {
    if (!predictor) {
        check(smoe_set_predictor(s, SMOE_PRED_NONE, nullptr));
        return SMOE_PRED_NONE;
    }
    auto* gp = dynamic_cast<GpuPredictor*>(predictor);
    if (!gp)
        throw std::invalid_argument(
            "specmoe_b200: the predictor must come from specmoe_b200::make_* (the B200 decode runs "
            "predictions on the device; there is no CPU fallback)");
    const auto& c = model.config;
    const auto& art = gp->artifacts();
    if (art.table) {
        const auto& t = *art.table;
        if (t.layers != c.layers || t.experts != c.experts || t.hidden != c.hidden)
            throw std::invalid_argument("default-vector table shape does not match the model");
        std::vector<float> flat(static_cast<size_t>(c.layers) * c.experts * c.hidden);
        for (size_t i = 0; i < t.d.size(); ++i)
            std::copy(t.d[i].begin(), t.d[i].end(), flat.begin() + static_cast<std::ptrdiff_t>(i) * c.hidden);
        check(smoe_load_default_vectors(s, flat.data(), static_cast<int64_t>(flat.size())));
    }
    if (art.estimator) {
        const auto& ec = art.estimator->config;
        smoe_estimator_config e{ec.d, ec.m, ec.n, ec.experts, ec.layers, ec.eps};
        check(smoe_load_estimator(s, &e, art.estimator->flat.data(),
                                  static_cast<int64_t>(art.estimator->flat.size())));
    }
    const int kind = pred_code(gp->kind());
    std::vector<int32_t> hyb;
    if (kind == SMOE_PRED_HYBRID && art.hybrid_map)
        for (auto k : *art.hybrid_map) hyb.push_back(pred_code(k));
    check(smoe_set_predictor(s, kind, hyb.empty() ? nullptr : hyb.data()));
    return kind;
}

}  // namespace

// ---------------------------------------------------------------- predictors

GpuPredictor::GpuPredictor(specmoe::PredictorKind kind, specmoe::PredictorArtifacts art)
    : kind_(kind), art_(std::move(art)) {}

std::string_view GpuPredictor::name() const {
    switch (kind_) {
    case specmoe::PredictorKind::kBaselineS: return "baseline-s";
    case specmoe::PredictorKind::kRouterPF: return "router-pf";
    case specmoe::PredictorKind::kEstPF: return "est-pf";
    case specmoe::PredictorKind::kHybridPF: return "hybrid";
    case specmoe::PredictorKind::kOracle: return "oracle";
    }
    return "unknown";
}

specmoe::Predictor::Prediction GpuPredictor::predict_next(const specmoe::Model&, const Context&) {
    throw std::invalid_argument("specmoe_b200::GpuPredictor predicts on the device only "
                                "(pass it to specmoe_b200::run_offloaded_decode / generate)");
}

std::unique_ptr<specmoe::Predictor> make_baseline_s() {
    return std::make_unique<GpuPredictor>(specmoe::PredictorKind::kBaselineS, specmoe::PredictorArtifacts{});
}

std::unique_ptr<specmoe::Predictor> make_router_pf(std::shared_ptr<const specmoe::DefaultVectorTable> table) {
    if (!table) throw std::invalid_argument("router-pf: missing default-vector table");
    return std::make_unique<GpuPredictor>(specmoe::PredictorKind::kRouterPF,
                                          specmoe::PredictorArtifacts{std::move(table), nullptr, std::nullopt});
}

std::unique_ptr<specmoe::Predictor> make_est_pf(std::shared_ptr<const specmoe::DefaultVectorTable> table,
                                                std::shared_ptr<const specmoe::EstimatorParams> estimator) {
    if (!estimator) throw std::invalid_argument("est-pf: missing estimator");
    return std::make_unique<GpuPredictor>(
        specmoe::PredictorKind::kEstPF,
        specmoe::PredictorArtifacts{std::move(table), std::move(estimator), std::nullopt});
}

std::unique_ptr<specmoe::Predictor> make_hybrid_pf(std::shared_ptr<const specmoe::DefaultVectorTable> table,
                                                   std::shared_ptr<const specmoe::EstimatorParams> estimator,
                                                   specmoe::HybridMap map) {
    return std::make_unique<GpuPredictor>(
        specmoe::PredictorKind::kHybridPF,
        specmoe::PredictorArtifacts{std::move(table), std::move(estimator), std::move(map)});
}

std::unique_ptr<specmoe::Predictor> make_oracle() {
    return std::make_unique<GpuPredictor>(specmoe::PredictorKind::kOracle, specmoe::PredictorArtifacts{});
}

std::unique_ptr<specmoe::Predictor> make_predictor(specmoe::PredictorKind kind,
                                                   const specmoe::PredictorArtifacts& art, int layers) {
    switch (kind) {
    case specmoe::PredictorKind::kBaselineS: return specmoe_b200::make_baseline_s();
    case specmoe::PredictorKind::kRouterPF: return specmoe_b200::make_router_pf(art.table);
    case specmoe::PredictorKind::kEstPF: return specmoe_b200::make_est_pf(art.table, art.estimator);
    case specmoe::PredictorKind::kHybridPF:
        if (!art.hybrid_map) throw std::invalid_argument("hybrid: missing hybrid map");
        if (static_cast<int>(art.hybrid_map->size()) != layers - 1)
            throw std::invalid_argument("hybrid map must have layers-1 entries");
        return specmoe_b200::make_hybrid_pf(art.table, art.estimator, *art.hybrid_map);
    case specmoe::PredictorKind::kOracle: return specmoe_b200::make_oracle();
    }
    throw std::invalid_argument("unknown predictor kind");
}

void set_device_options(const DeviceOptions& o) {
    if (!(o.cache_fraction > 0.0f && o.cache_fraction <= 1.0f))
        throw std::invalid_argument("cache_fraction must be in (0, 1]");
    std::lock_guard<std::mutex> g(g_mu);
    g_opts = o;
}

// ------------------------------------------------------------------ decode

specmoe::ExecutorResult run_offloaded_decode(const specmoe::Model& model, std::span<const int> prompt,
                                             int n_new, specmoe::Predictor* predictor,
                                             const specmoe::ExecutorOptions& options) {
    if (prompt.empty()) throw std::invalid_argument("offloaded decode: empty prompt");
    if (n_new < 1) throw std::invalid_argument("offloaded decode: n_new must be >= 1");
    const bool prefetch = options.mode == specmoe::OffloadMode::kPrefetch;
    if (prefetch && !predictor) throw std::invalid_argument("offloaded decode: prefetch mode needs a predictor");
    if (options.copy_latency_us < 0) throw std::invalid_argument("offloaded decode: negative copy latency");
    std::lock_guard<std::mutex> g(g_mu);
    const int P = static_cast<int>(prompt.size());
    smoe_session* s = session_for(model, P + n_new + 8, false, &options);
    install_predictor(s, model, prefetch ? predictor : nullptr);
    std::vector<int32_t> pr(prompt.begin(), prompt.end()), toks(static_cast<size_t>(n_new));
    std::vector<double> per(static_cast<size_t>(std::max(n_new - 1, 1)));
    const int cap = 1 << 18;
    std::vector<smoe_event> ev(static_cast<size_t>(cap));
    int32_t nev = 0, max_res = 0;
    check(smoe_run_offloaded_decode_ex(s, pr.data(), P, n_new, prefetch ? SMOE_PREFETCH : SMOE_ON_DEMAND,
                                       toks.data(), per.data(), ev.data(), cap, &nev, &max_res));
    specmoe::ExecutorResult r;
    r.tokens.assign(toks.begin(), toks.end());
    for (int i = 0; i < n_new - 1; ++i) r.per_token_us.push_back(per[static_cast<size_t>(i)] * 1000.0);
    static const specmoe::EventKind kinds[] = {specmoe::EventKind::kAttn, specmoe::EventKind::kGate,
                                               specmoe::EventKind::kExpert, specmoe::EventKind::kCopy};
    for (int i = 0; i < std::min(nev, cap); ++i) {
        const smoe_event& e = ev[static_cast<size_t>(i)];
        r.events.push_back({e.lane == 0 ? specmoe::Lane::kCompute : specmoe::Lane::kCopy,
                            kinds[std::clamp(e.kind, 0, 3)], e.layer, e.start_ms * 1000.0, e.end_ms * 1000.0,
                            e.token});
    }
    r.max_resident_layers = max_res;
    return r;
}

std::vector<int> generate(const specmoe::Model& model, std::span<const int> prompt, int n_new,
                          specmoe::Predictor* predictor) {
    if (prompt.empty()) throw std::invalid_argument("generate: empty prompt");
    if (n_new < 1) throw std::invalid_argument("generate: n_new must be >= 1");
    std::lock_guard<std::mutex> g(g_mu);
    const int P = static_cast<int>(prompt.size());
    smoe_session* s = session_for(model, P + n_new + 8, true, nullptr);
    const int kind = install_predictor(s, model, predictor);
    std::vector<int32_t> pr(prompt.begin(), prompt.end()), toks(static_cast<size_t>(n_new));
    check(smoe_run_offloaded_decode(s, pr.data(), P, n_new, kind == SMOE_PRED_NONE ? SMOE_ON_DEMAND : SMOE_PREFETCH,
                                    toks.data(), nullptr));
    return std::vector<int>(toks.begin(), toks.end());
}

}  // namespace specmoe_b200
