// specmoe_b200.hpp — C++ drop-in for the reference's offloaded-decode API
// (/root/reference/proj/include/specmoe: executor.hpp:51-52,
// speculation.hpp:72-89, speculation.hpp:97-103), executed on a B200 through
// the C ABI (include/smoe.h).  Compiled against the reference's own headers:
// the argument and result types are the reference's (Model, Predictor,
// ExecutorOptions, ExecutorResult, DefaultVectorTable, EstimatorParams).
//
// A caller switches by replacing
//     specmoe::make_router_pf(table)              -> specmoe_b200::make_router_pf(table)
//     specmoe::run_offloaded_decode(model, ...)   -> specmoe_b200::run_offloaded_decode(model, ...)
//     specmoe::generate(model, ...)               -> specmoe_b200::generate(model, ...)
// The predictor factories return GPU-aware Predictor subclasses; the decode
// recovers their kind and artifacts by dynamic_cast (a CPU Predictor cannot
// be called per layer from the device without a round trip, and the
// reference's concrete predictor classes are anonymous, speculation.cpp:167-308).
// Any other Predictor is rejected with std::invalid_argument: there is no CPU
// fallback.  Errors follow the reference: std::invalid_argument for usage and
// config errors, std::runtime_error for runtime failures ("deadlock
// suspected ...").
//
// Weights are stored as bf16 on the GPU (rounded to nearest even from the
// Model's f32 values); results equal the reference's on a model whose weights
// are already bf16-representable (tests/test_gpu_dropin.py).
#pragma once

#include "specmoe/estimator.hpp"
#include "specmoe/executor.hpp"
#include "specmoe/model.hpp"
#include "specmoe/speculation.hpp"

#include <memory>
#include <optional>
#include <span>
#include <string_view>
#include <vector>

namespace specmoe_b200 {

// The predictor plugin handed to the B200 decode (model.hpp:143-167): it
// carries the kind and artifacts make_predictor takes
// (speculation.hpp:83-89).  Its CPU predict_next throws — the B200 path runs
// the prediction on the device.
class GpuPredictor : public specmoe::Predictor {
public:
    GpuPredictor(specmoe::PredictorKind kind, specmoe::PredictorArtifacts art);
    std::string_view name() const override;
    Prediction predict_next(const specmoe::Model& model, const Context& ctx) override;
    specmoe::PredictorKind kind() const { return kind_; }
    const specmoe::PredictorArtifacts& artifacts() const { return art_; }

private:
    specmoe::PredictorKind kind_;
    specmoe::PredictorArtifacts art_;
};

std::unique_ptr<specmoe::Predictor> make_baseline_s();
std::unique_ptr<specmoe::Predictor> make_router_pf(std::shared_ptr<const specmoe::DefaultVectorTable> table);
std::unique_ptr<specmoe::Predictor> make_est_pf(std::shared_ptr<const specmoe::DefaultVectorTable> table,
                                                std::shared_ptr<const specmoe::EstimatorParams> estimator);
std::unique_ptr<specmoe::Predictor> make_hybrid_pf(std::shared_ptr<const specmoe::DefaultVectorTable> table,
                                                   std::shared_ptr<const specmoe::EstimatorParams> estimator,
                                                   specmoe::HybridMap map);
std::unique_ptr<specmoe::Predictor> make_oracle();
std::unique_ptr<specmoe::Predictor> make_predictor(specmoe::PredictorKind kind,
                                                   const specmoe::PredictorArtifacts& art, int layers);

// B200 placement knobs the reference API has no slot for (defaults: device
// 0, HBM expert cache capped at 25 % of the experts per layer).
struct DeviceOptions {
    int device = 0;
    float cache_fraction = 0.25f;
};
void set_device_options(const DeviceOptions& o);

// run_offloaded_decode (executor.hpp:51-52, executor.cpp:326-359): prefill
// with true routing, then n_new - 1 decode steps, on-demand or Algorithm 1
// prefetch.  Returns the reference's ExecutorResult: tokens, the measured
// lane events of the same run (µs from the run start), per_token_us and
// max_resident_layers.  options.mode selects the mode; copy_latency_us (the
// reference's injected stand-in for a PCIe copy) is not injected — the B200
// copies are real — and the device-side deadlock limit is 10 s.  The session
// (uploaded weights, pinned store, slot pool) is cached per Model object.
specmoe::ExecutorResult run_offloaded_decode(const specmoe::Model& model, std::span<const int> prompt,
                                             int n_new, specmoe::Predictor* predictor,
                                             const specmoe::ExecutorOptions& options);

// generate (speculation.hpp:102-103): greedy generation with every expert
// resident in HBM (the in-memory path); Algorithm 1 from layer 1 when a
// predictor is given.
std::vector<int> generate(const specmoe::Model& model, std::span<const int> prompt, int n_new,
                          specmoe::Predictor* predictor = nullptr);

}  // namespace specmoe_b200
