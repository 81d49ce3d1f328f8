// dropin_check.cpp — TEST INFRASTRUCTURE ONLY.
//
// Links the UNMODIFIED reference objects (oracle/_ref/obj) with the B200 C++
// drop-in (paper_2603_19289_b200/libspecmoe_b200_dropin.so) and runs both on
// the same reference Model: the reference's run_offloaded_decode / generate
// (CPU, executor.cpp / speculation.cpp) against specmoe_b200::
// run_offloaded_decode / generate (GPU), predictors from each side's own
// make_* factories.  Called by tests/test_gpu_dropin.py through ctypes.
#include "specmoe_b200.hpp"

#include "specmoe/executor.hpp"
#include "specmoe/model.hpp"
#include "specmoe/speculation.hpp"

#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;

float round_bf16(float x) {
    std::uint32_t u;
    std::memcpy(&u, &x, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    u &= 0xFFFF0000u;
    float y;
    std::memcpy(&y, &u, 4);
    return y;
}

void round_mat(specmoe::Mat& m) {
    for (float& v : m.data) v = round_bf16(v);
}

}  // namespace

extern "C" const char* dropin_last_error() { return g_err.c_str(); }

// kind: -1 none, 0 baseline-s, 1 router-pf.  mode: 0 on_demand, 1 prefetch.
// out: ref_tokens[n_new], b200_tokens[n_new], gen_ref[n_new], gen_b200[n_new],
// info[4] = {b200 max_resident_layers, b200 events, ref max_resident_layers, ref events}.
extern "C" int dropin_check(int L, int E, int K, int H, int Hm, int V, int D, std::uint64_t seed, int mode,
                            int kind, const int* prompt, int P, int n_new, float cache_fraction, int* ref_tokens,
                            int* b200_tokens, int* gen_ref, int* gen_b200, int* info) {
    try {
        specmoe::ModelConfig cfg;
        cfg.layers = L; cfg.experts = E; cfg.top_k = K; cfg.hidden = H; cfg.expert_hidden = Hm;
        cfg.vocab = V; cfg.head_dim = D; cfg.seed = seed;
        specmoe::Model model = specmoe::build_model(cfg);
        // the values the GPU stores (bf16): both sides then see identical weights
        round_mat(model.embedding);
        round_mat(model.unembed);
        for (auto& lw : model.layers) {
            round_mat(lw.wq); round_mat(lw.wk); round_mat(lw.wv); round_mat(lw.wo); round_mat(lw.gate);
            for (auto& ex : lw.experts) { round_mat(ex.w_gate); round_mat(ex.w_up); round_mat(ex.w_down); }
        }
        auto table = std::make_shared<specmoe::DefaultVectorTable>(specmoe::DefaultVectorTable::zeros(L, E, H));
        std::uint64_t z = seed * 0x9E3779B97F4A7C15ull + 1;
        for (auto& d : table->d)
            for (float& v : d) {
                z = z * 6364136223846793005ull + 1442695040888963407ull;
                v = static_cast<float>(static_cast<std::int64_t>(z >> 40) - (1ll << 23)) * 1e-8f;
            }
        std::unique_ptr<specmoe::Predictor> rp, bp, rp2, bp2;
        if (kind == 0) {
            rp = specmoe::make_baseline_s(); bp = specmoe_b200::make_baseline_s();
            rp2 = specmoe::make_baseline_s(); bp2 = specmoe_b200::make_baseline_s();
        } else if (kind == 1) {
            rp = specmoe::make_router_pf(table); bp = specmoe_b200::make_router_pf(table);
            rp2 = specmoe::make_router_pf(table); bp2 = specmoe_b200::make_router_pf(table);
        }
        specmoe::ExecutorOptions opt;
        opt.mode = mode ? specmoe::OffloadMode::kPrefetch : specmoe::OffloadMode::kOnDemand;
        opt.copy_latency_us = 1;
        opt.deadlock_factor = 1e8;
        std::span<const int> pr(prompt, static_cast<size_t>(P));
        const specmoe::ExecutorResult a = specmoe::run_offloaded_decode(model, pr, n_new, rp.get(), opt);
        specmoe_b200::set_device_options({0, cache_fraction});
        const specmoe::ExecutorResult b = specmoe_b200::run_offloaded_decode(model, pr, n_new, bp.get(), opt);
        for (int i = 0; i < n_new; ++i) {
            ref_tokens[i] = a.tokens[static_cast<size_t>(i)];
            b200_tokens[i] = b.tokens[static_cast<size_t>(i)];
        }
        const std::vector<int> ga = specmoe::generate(model, pr, n_new, rp2.get());
        const std::vector<int> gb = specmoe_b200::generate(model, pr, n_new, bp2.get());
        for (int i = 0; i < n_new; ++i) {
            gen_ref[i] = ga[static_cast<size_t>(i)];
            gen_b200[i] = gb[static_cast<size_t>(i)];
        }
        info[0] = b.max_resident_layers;
        info[1] = static_cast<int>(b.events.size());
        info[2] = a.max_resident_layers;
        info[3] = static_cast<int>(a.events.size());
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

// A CPU predictor from the reference's own factory is refused (no CPU fallback).
extern "C" int dropin_reject_cpu_predictor() {
    try {
        specmoe::ModelConfig cfg;
        cfg.layers = 2; cfg.experts = 4; cfg.top_k = 2; cfg.hidden = 16; cfg.expert_hidden = 16;
        cfg.vocab = 16; cfg.head_dim = 8; cfg.seed = 1;
        specmoe::Model model = specmoe::build_model(cfg);
        auto p = specmoe::make_baseline_s();
        specmoe::ExecutorOptions opt;
        opt.mode = specmoe::OffloadMode::kPrefetch;
        const int prompt[2] = {1, 2};
        specmoe_b200::run_offloaded_decode(model, std::span<const int>(prompt, 2), 3, p.get(), opt);
        g_err = "accepted a CPU predictor";
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}
