// train.h — estimator distillation on the GPU: the device
// side of train_estimator (estimator.cpp:374-450) and its host driver.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace smoe {

// Chain GEMM: out[a][b] = start + L(0,a)*R(0,b) + L(1,a)*R(1,b) + ... + L(K-1,a)*R(K-1,b)
// summed strictly in k order, every product rounded to f32 before its add
// (the reference's scalar `acc += w * x` loops, compiled without FMA).
// `start` is init[a][b] when init is set, else +0.  Every matrix is addressed
// through its own strides so one kernel serves the forward GEMVs over a batch
// of samples (k = input feature), the transposed backward GEMVs and the
// per-step gradient outer products (k = sample).
enum ChainEpi {
    kEpiNone = 0,
    kEpiAddPos = 1,    // out = acc + aux[(a % lp) * B + b]            z = A.q + pos[l]   (estimator.cpp:106-111)
    kEpiSilu = 2,      // out = acc, out2 = acc / (1 + expf(-acc))      u, act           (estimator.cpp:113-123)
    kEpiAddAfter = 3,  // out = aux[a][b] + acc                         h = z + C.act    (estimator.cpp:125-131)
    kEpiSiluGrad = 4,  // out2 = acc * sig * (1 + u * (1 - sig)), u = aux[a][b]       (estimator.cpp:236-242)
};

struct ChainGemm {
    const float* L;
    long long lsk, lsa;
    const float* R;
    long long rsk, rsb;
    float* out;
    long long osa, osb;
    const float* init;  // chain start in out's layout, or null for +0
    int A, B, K;
    int epi;
    const float* aux;
    float* out2;
    int lp;             // kEpiAddPos: samples are token-major, layer = a % lp
};

cudaError_t launch_chain_gemm(const ChainGemm& g, cudaStream_t s);
// Qb[s] = inputs[tok[s / lp] * lp + s % lp], Tb likewise (the step's batch, token-major).
cudaError_t launch_est_gather(const float* inputs, const float* targets, const int64_t* tok, int S, int lp,
                              int d, int E, float* Qb, float* Tb, cudaStream_t s);
// LayerNorm forward per sample (estimator.cpp:133-147): XHAT, Y = gain*xhat + bias, inv_std.
cudaError_t launch_est_layernorm(const float* H, const float* gain, const float* bias, int S, int dm, float eps,
                                 float* XHAT, float* Y, float* inv_std, cudaStream_t s);
// probs = softmax_inplace(logits); with targets: glog = weight * (probs - softmax_inplace(targets))
// (estimator.cpp:79-90, 185-193).
cudaError_t launch_est_softmax(const float* logits, const float* targets, int S, int E, float weight, float* probs,
                               float* glog, cudaStream_t s);
// LayerNorm backward (estimator.cpp:205-224): GH from GY.
cudaError_t launch_est_ln_backward(const float* GY, const float* XHAT, const float* inv_std, const float* gain,
                                   int S, int dm, float* GH, cudaStream_t s);
// grad ln_gain / ln_bias / pos (estimator.cpp:205-210, 254-256), chains over the batch in sample order.
cudaError_t launch_est_small_grads(const float* GY, const float* XHAT, const float* GZ, int S, int lp, int dm,
                                   float* g_gain, float* g_bias, float* g_pos, cudaStream_t s);
// adam_step (estimator.cpp:301-322); b1c / b2c = 1 - beta^step computed by the host's libm pow.
cudaError_t launch_est_adam(float* params, const float* grad, float* m, float* v, long long n, double lr,
                            double b1, double b2, double eps, double b1c, double b2c, cudaStream_t s);

struct EstTrainCfg {
    int d, m, n, experts, layers;
    float eps;
    uint64_t seed;
};
struct EstTrainHyper {
    double lr;
    int batch_tokens;
    int64_t max_steps, eval_every;
    double val_fraction;
    uint64_t seed;
    int k;
    double early_stop_hit_rate;
};
struct EstCurvePoint {
    int64_t tokens_seen;
    double val_kl, val_hit_rate;
};

// init_estimator_params<float> (estimator.cpp:54-75) on the host.
std::vector<float> estimator_init_params(const EstTrainCfg& c);

// train_estimator (estimator.cpp:374-450): inputs [tokens][L-1][d],
// targets [tokens][L-1][E] (host); params_out sized param_count().
// Returns the validation curve.  `step_ms` (nullable) receives the device
// time of the training steps (excluding evaluation).
std::vector<EstCurvePoint> train_estimator_gpu(const EstTrainCfg& c, const float* inputs, const float* targets,
                                               int64_t tokens, int layers_predicting, const EstTrainHyper& h,
                                               float* params_out, double* step_ms);

}  // namespace smoe
