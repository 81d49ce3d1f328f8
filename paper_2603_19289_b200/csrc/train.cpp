// train.cpp — host driver of estimator distillation on the GPU
// (train_estimator, estimator.cpp:374-450).
//
// The host keeps what is sequential by nature and cheap: the epoch shuffles
// (Rng, numerics.hpp:35-64), Adam's bias corrections (libm pow, as the
// reference), and the validation metrics over the logits the GPU produced
// (recall@k, numerics.cpp top_k; KL, numerics.cpp:118-134), summed in the
// reference's order.  Everything proportional to the parameter count runs on
// the device (train.cu).
#include "train.h"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <stdexcept>
#include <string>

namespace smoe {

namespace {

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

// Rng (numerics.hpp:35-64) and derive_seed (numerics.cpp:20-35).
struct HostRng {
    uint64_t st;
    uint64_t next_u64() {
        uint64_t z = (st += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    double next_gaussian() {
        double s = 0.0;
        for (int i = 0; i < 12; ++i) s += next_double();
        return s - 6.0;
    }
};

uint64_t derive_seed_h(uint64_t seed, const std::string& label) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (unsigned char c : label) {
        h ^= c;
        h *= 0x100000001b3ull;
    }
    uint64_t z = seed ^ h;
    for (int i = 0; i < 2; ++i) {
        z += 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z = z ^ (z >> 31);
    }
    return z;
}

// EstimatorConfig::validate (estimator.cpp:19-27), same messages.
void validate(const EstTrainCfg& c) {
    if (c.d < 1) throw std::invalid_argument("estimator: d must be >= 1");
    if (c.m <= 1 || c.n <= 1) throw std::invalid_argument("estimator: m and n must be > 1");
    if (c.d % c.m != 0) throw std::invalid_argument("estimator: d must be divisible by m");
    if (c.d / c.m < 1) throw std::invalid_argument("estimator: latent width must be >= 1");
    if (c.experts < 1) throw std::invalid_argument("estimator: E must be >= 1");
    if (c.layers < 1) throw std::invalid_argument("estimator: L must be >= 1");
    if (!(c.eps > 0.0f)) throw std::invalid_argument("estimator: eps must be > 0");
}

// Flat layout (estimator.hpp:41-72).
struct Layout {
    size_t dm, mlp, a, pos, b, c, gain, bias, head, total;
    explicit Layout(const EstTrainCfg& cf) {
        dm = static_cast<size_t>(cf.d / cf.m);
        mlp = dm * static_cast<size_t>(cf.n);
        a = 0;
        pos = a + dm * cf.d;
        b = pos + static_cast<size_t>(cf.layers) * dm;
        c = b + mlp * dm;
        gain = c + dm * mlp;
        bias = gain + dm;
        head = bias + dm;
        total = head + static_cast<size_t>(cf.experts) * dm;
    }
};

// softmax (numerics.cpp:37-54): f64 exponentials and normaliser.
std::vector<float> softmax_f64(const float* v, int n) {
    float mx = v[0];
    for (int i = 0; i < n; ++i) {
        if (!std::isfinite(v[i])) throw std::invalid_argument("softmax: non-finite input");
        mx = std::max(mx, v[i]);
    }
    std::vector<double> e(n);
    double z = 0.0;
    for (int i = 0; i < n; ++i) {
        e[i] = std::exp(static_cast<double>(v[i]) - static_cast<double>(mx));
        z += e[i];
    }
    std::vector<float> out(n);
    for (int i = 0; i < n; ++i) out[i] = static_cast<float>(e[i] / z);
    return out;
}

// The top-k SET under (value desc, index asc) (numerics.cpp:56-71); recall
// only needs the set.
std::vector<int> top_k_set(const float* v, int n, int k) {
    std::vector<int> idx(n);
    std::iota(idx.begin(), idx.end(), 0);
    std::partial_sort(idx.begin(), idx.begin() + k, idx.end(), [&](int a, int b) {
        if (v[a] != v[b]) return v[a] > v[b];
        return a < b;
    });
    idx.resize(k);
    return idx;
}

void check_distribution(const float* p, int n, const char* name) {
    double sum = 0.0;
    for (int i = 0; i < n; ++i) {
        const float x = p[i];
        if (!(x >= 0.0f) || x > 1.0f + 1e-5f)
            throw std::invalid_argument(std::string("kl_divergence: ") + name + " is not a distribution");
        sum += x;
    }
    if (std::abs(sum - 1.0) > 1e-4)
        throw std::invalid_argument(std::string("kl_divergence: ") + name + " does not sum to 1");
}

// kl_divergence (numerics.cpp:118-134).
double kl_div(const float* p, const float* q, int n) {
    check_distribution(p, n, "p");
    check_distribution(q, n, "q");
    double kl = 0.0;
    for (int i = 0; i < n; ++i) {
        if (p[i] == 0.0f) continue;
        if (q[i] == 0.0f) throw std::invalid_argument("kl_divergence: q has zero mass where p > 0");
        kl += static_cast<double>(p[i]) * std::log(static_cast<double>(p[i]) / static_cast<double>(q[i]));
    }
    if (kl < 0.0 && kl > -1e-12) kl = 0.0;
    return kl;
}

struct DevBuf {
    float* p = nullptr;
    void alloc(size_t n) { ck(cudaMalloc(&p, std::max<size_t>(n, 1) * 4), "estimator training alloc"); }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

}  // namespace

std::vector<float> estimator_init_params(const EstTrainCfg& c) {
    validate(c);
    const Layout lo(c);
    std::vector<float> p(lo.total, 0.0f);
    auto fill = [&](size_t off, size_t count, const char* label, double stddev) {
        HostRng rng{derive_seed_h(c.seed, std::string("estimator.") + label)};
        for (size_t i = 0; i < count; ++i) p[off + i] = static_cast<float>(rng.next_gaussian() * stddev);
    };
    fill(lo.a, lo.dm * c.d, "a", 1.0 / std::sqrt(static_cast<double>(c.d)));
    fill(lo.pos, static_cast<size_t>(c.layers) * lo.dm, "pos", 0.02);
    fill(lo.b, lo.mlp * lo.dm, "b", 1.0 / std::sqrt(static_cast<double>(lo.dm)));
    fill(lo.c, lo.dm * lo.mlp, "c", 1.0 / std::sqrt(static_cast<double>(lo.mlp)));
    fill(lo.head, static_cast<size_t>(c.experts) * lo.dm, "w_head", 1.0 / std::sqrt(static_cast<double>(lo.dm)));
    for (size_t i = 0; i < lo.dm; ++i) p[lo.gain + i] = 1.0f;
    return p;
}

std::vector<EstCurvePoint> train_estimator_gpu(const EstTrainCfg& c, const float* inputs, const float* targets,
                                               int64_t tokens, int layers_predicting, const EstTrainHyper& h,
                                               float* params_out, double* step_ms) {
    validate(c);
    if (tokens < 1) throw std::invalid_argument("train: empty dataset");
    if (layers_predicting != c.layers - 1 || layers_predicting < 1)
        throw std::invalid_argument("train: dataset does not match estimator config");
    if (h.k < 1 || h.k > c.experts) throw std::invalid_argument("train: invalid k");
    if (h.batch_tokens < 1) throw std::invalid_argument("train: batch_tokens must be >= 1");
    if (h.eval_every < 1) throw std::invalid_argument("train: eval_every must be >= 1");
    const int64_t val_tokens =
        std::max<int64_t>(1, static_cast<int64_t>(static_cast<double>(tokens) * h.val_fraction));
    const int64_t train_tokens = tokens - val_tokens;
    if (train_tokens < 1) throw std::invalid_argument("train: no training tokens after split");

    const Layout lo(c);
    const int lp = layers_predicting, d = c.d, E = c.experts, B = h.batch_tokens;
    const int dm = static_cast<int>(lo.dm), mlp = static_cast<int>(lo.mlp);
    const int ev_tok = std::max(B, 32);                       // validation chunk (tokens)
    const size_t S = static_cast<size_t>(std::max(B, ev_tok)) * lp;  // samples per buffer
    std::vector<float> params = estimator_init_params(c);

    cudaStream_t st;
    ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "estimator training stream");
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{st};
    DevBuf din, dtg, P, G, M, V, Qb, Tb, Z, U, ACT, Hh, XH, Y, INV, LOG, PROB, GLOG, GY, GH, GU, GZ;
    const size_t nsamp = static_cast<size_t>(tokens) * lp;
    din.alloc(nsamp * d);
    dtg.alloc(nsamp * E);
    P.alloc(lo.total);
    G.alloc(lo.total);
    M.alloc(lo.total);
    V.alloc(lo.total);
    Qb.alloc(S * d);
    Tb.alloc(S * E);
    for (DevBuf* b : {&Z, &Hh, &XH, &Y, &GY, &GH, &GZ}) b->alloc(S * dm);
    for (DevBuf* b : {&U, &ACT, &GU}) b->alloc(S * mlp);
    for (DevBuf* b : {&LOG, &PROB, &GLOG}) b->alloc(S * E);
    INV.alloc(S);
    int64_t* dtok = nullptr;
    ck(cudaMalloc(&dtok, 8ull * B * std::max<int64_t>(1, std::min<int64_t>(h.eval_every, h.max_steps))),
       "estimator training alloc");
    struct TokGuard {
        int64_t* p;
        ~TokGuard() { cudaFree(p); }
    } tg{dtok};
    ck(cudaMemcpyAsync(din.p, inputs, nsamp * d * 4, cudaMemcpyHostToDevice, st), "dataset upload");
    ck(cudaMemcpyAsync(dtg.p, targets, nsamp * E * 4, cudaMemcpyHostToDevice, st), "dataset upload");
    ck(cudaMemcpyAsync(P.p, params.data(), lo.total * 4, cudaMemcpyHostToDevice, st), "params upload");
    ck(cudaMemsetAsync(G.p, 0, lo.total * 4, st), "grad reset");  // pos[L-1] grad stays +0
    ck(cudaMemsetAsync(M.p, 0, lo.total * 4, st), "adam reset");
    ck(cudaMemsetAsync(V.p, 0, lo.total * 4, st), "adam reset");

    const float* pA = P.p + lo.a;
    const float* pPos = P.p + lo.pos;
    const float* pB = P.p + lo.b;
    const float* pC = P.p + lo.c;
    const float* pGain = P.p + lo.gain;
    const float* pBias = P.p + lo.bias;
    const float* pHead = P.p + lo.head;
    auto gemm = [&](ChainGemm g, const char* what) { ck(launch_chain_gemm(g, st), what); };

    // estimator_forward<float> (estimator.cpp:94-161) for n samples (token-major,
    // layer = sample % lp) of inputs q; tg != null also produces glog.
    auto forward = [&](const float* q, const float* tgt, int n, float weight) {
        gemm({q, 1, d, pA, 1, d, Z.p, dm, 1, nullptr, n, dm, d, kEpiAddPos, pPos, nullptr, lp}, "estimator z");
        gemm({Z.p, 1, dm, pB, 1, dm, U.p, mlp, 1, nullptr, n, mlp, dm, kEpiSilu, nullptr, ACT.p, lp}, "estimator u");
        gemm({ACT.p, 1, mlp, pC, 1, mlp, Hh.p, dm, 1, nullptr, n, dm, mlp, kEpiAddAfter, Z.p, nullptr, lp},
             "estimator h");
        ck(launch_est_layernorm(Hh.p, pGain, pBias, n, dm, c.eps, XH.p, Y.p, INV.p, st), "estimator layernorm");
        gemm({Y.p, 1, dm, pHead, 1, dm, LOG.p, E, 1, nullptr, n, E, dm, kEpiNone, nullptr, nullptr, lp},
             "estimator head");
        ck(launch_est_softmax(LOG.p, tgt, n, E, weight, PROB.p, GLOG.p, st), "estimator softmax");
    };

    // estimator_backward<float> (estimator.cpp:171-258) for the n samples of
    // the batch, gradients accumulated in sample order (each element's chain
    // restarts at +0 per step, as the reference zeroes grad).
    auto backward = [&](int n) {
        gemm({GLOG.p, 1, E, pHead, dm, 1, GY.p, dm, 1, nullptr, n, dm, E, kEpiNone, nullptr, nullptr, lp},
             "estimator g_y");
        ck(launch_est_ln_backward(GY.p, XH.p, INV.p, pGain, n, dm, GH.p, st), "estimator ln backward");
        gemm({GH.p, 1, dm, pC, mlp, 1, nullptr, mlp, 1, nullptr, n, mlp, dm, kEpiSiluGrad, U.p, GU.p, lp},
             "estimator g_u");
        gemm({GU.p, 1, mlp, pB, dm, 1, GZ.p, dm, 1, GH.p, n, dm, mlp, kEpiNone, nullptr, nullptr, lp},
             "estimator g_z");
        gemm({GLOG.p, E, 1, Y.p, dm, 1, G.p + lo.head, dm, 1, nullptr, E, dm, n, kEpiNone, nullptr, nullptr, lp},
             "estimator grad w_head");
        ck(launch_est_small_grads(GY.p, XH.p, GZ.p, n, lp, dm, G.p + lo.gain, G.p + lo.bias, G.p + lo.pos, st),
           "estimator grad ln/pos");
        gemm({GH.p, dm, 1, ACT.p, mlp, 1, G.p + lo.c, mlp, 1, nullptr, dm, mlp, n, kEpiNone, nullptr, nullptr, lp},
             "estimator grad c");
        gemm({GU.p, mlp, 1, Z.p, dm, 1, G.p + lo.b, dm, 1, nullptr, mlp, dm, n, kEpiNone, nullptr, nullptr, lp},
             "estimator grad b");
        gemm({GZ.p, dm, 1, Qb.p, d, 1, G.p + lo.a, d, 1, nullptr, dm, d, n, kEpiNone, nullptr, nullptr, lp},
             "estimator grad a");
    };

    std::vector<float> hlog, hprob;
    // eval_hit_rate (estimator.cpp:340-372) on tokens [train_tokens, tokens).
    auto eval_point = [&](int64_t seen, std::vector<EstCurvePoint>& curve) {
        std::vector<double> per_layer(lp, 0.0);
        std::vector<int64_t> counts(lp, 0);
        double kl_sum = 0.0;
        int64_t n = 0;
        for (int64_t t0 = train_tokens; t0 < tokens; t0 += ev_tok) {
            const int nt = static_cast<int>(std::min<int64_t>(ev_tok, tokens - t0));
            const int ns = nt * lp;
            forward(din.p + static_cast<size_t>(t0) * lp * d, nullptr, ns, 0.0f);
            hlog.resize(static_cast<size_t>(ns) * E);
            hprob.resize(static_cast<size_t>(ns) * E);
            ck(cudaMemcpyAsync(hlog.data(), LOG.p, hlog.size() * 4, cudaMemcpyDeviceToHost, st), "eval logits");
            ck(cudaMemcpyAsync(hprob.data(), PROB.p, hprob.size() * 4, cudaMemcpyDeviceToHost, st), "eval probs");
            ck(cudaStreamSynchronize(st), "eval");
            for (int i = 0; i < ns; ++i) {
                const int l = i % lp;
                const float* pred = hlog.data() + static_cast<size_t>(i) * E;
                const float* truth = targets + (static_cast<size_t>(t0) * lp + i) * E;
                const std::vector<int> tp = top_k_set(pred, E, h.k), tt = top_k_set(truth, E, h.k);
                int hits = 0;
                for (int a : tp)
                    for (int b : tt)
                        if (a == b) {
                            ++hits;
                            break;
                        }
                per_layer[l] += static_cast<double>(hits) / static_cast<double>(h.k);
                ++counts[l];
                const std::vector<float> tprob = softmax_f64(truth, E);
                kl_sum += kl_div(tprob.data(), hprob.data() + static_cast<size_t>(i) * E, E);
                ++n;
            }
        }
        double total = 0.0;
        for (int l = 0; l < lp; ++l) {
            if (counts[l] > 0) per_layer[l] /= static_cast<double>(counts[l]);
            total += per_layer[l];
        }
        const double mean = total / lp;
        curve.push_back({seen, n > 0 ? kl_sum / static_cast<double>(n) : 0.0, mean});
        return mean;
    };

    std::vector<EstCurvePoint> curve;
    double hit = eval_point(0, curve);
    double ms_total = 0.0;
    if (!(h.early_stop_hit_rate > 0.0 && hit >= h.early_stop_hit_rate)) {
        std::vector<int64_t> order(static_cast<size_t>(train_tokens));
        std::iota(order.begin(), order.end(), 0);
        int64_t cursor = 0, epoch = 0, seen = 0;
        auto reshuffle = [&]() {
            HostRng rng{derive_seed_h(h.seed, "train-epoch-" + std::to_string(epoch))};
            for (size_t i = order.size(); i > 1; --i) {
                const auto j = static_cast<size_t>(rng.next_u64() % i);
                std::swap(order[i - 1], order[j]);
            }
        };
        reshuffle();
        const float weight = 1.0f / static_cast<float>(B * lp);
        const double b1 = 0.9, b2 = 0.999, aeps = 1e-8;  // AdamConfig (estimator.hpp:133-138)
        cudaEvent_t e0, e1;
        ck(cudaEventCreate(&e0), "event");
        ck(cudaEventCreate(&e1), "event");
        std::vector<int64_t> sched;
        for (int64_t step = 1; step <= h.max_steps;) {
            // one segment = the steps up to the next evaluation point
            const int64_t last = std::min(h.max_steps, ((step - 1) / h.eval_every + 1) * h.eval_every);
            sched.clear();
            for (int64_t s2 = step; s2 <= last; ++s2)
                for (int bt = 0; bt < B; ++bt) {
                    if (cursor >= train_tokens) {
                        cursor = 0;
                        ++epoch;
                        reshuffle();
                    }
                    sched.push_back(order[static_cast<size_t>(cursor++)]);
                }
            ck(cudaMemcpyAsync(dtok, sched.data(), sched.size() * 8, cudaMemcpyHostToDevice, st), "schedule upload");
            ck(cudaEventRecord(e0, st), "event");
            for (int64_t s2 = step; s2 <= last; ++s2) {
                const int n = B * lp;
                ck(launch_est_gather(din.p, dtg.p, dtok + (s2 - step) * B, n, lp, d, E, Qb.p, Tb.p, st),
                   "estimator gather");
                forward(Qb.p, Tb.p, n, weight);
                backward(n);
                const double b1c = 1.0 - std::pow(b1, static_cast<double>(s2));
                const double b2c = 1.0 - std::pow(b2, static_cast<double>(s2));
                ck(launch_est_adam(P.p, G.p, M.p, V.p, static_cast<long long>(lo.total), h.lr, b1, b2, aeps, b1c,
                                   b2c, st),
                   "estimator adam");
            }
            ck(cudaEventRecord(e1, st), "event");
            ck(cudaStreamSynchronize(st), "estimator training");
            float ms = 0.0f;
            ck(cudaEventElapsedTime(&ms, e0, e1), "event");
            ms_total += ms;
            seen += (last - step + 1) * B;
            step = last + 1;
            if (last % h.eval_every == 0 || last == h.max_steps) {
                hit = eval_point(seen, curve);
                if (h.early_stop_hit_rate > 0.0 && hit >= h.early_stop_hit_rate) break;
            }
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    }
    ck(cudaMemcpyAsync(params.data(), P.p, lo.total * 4, cudaMemcpyDeviceToHost, st), "params download");
    ck(cudaStreamSynchronize(st), "estimator training");
    std::copy(params.begin(), params.end(), params_out);
    if (step_ms) *step_ms = ms_total;
    return curve;
}

}  // namespace smoe
