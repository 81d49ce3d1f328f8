// train.cu — device side of estimator distillation (train_estimator,
// estimator.cpp:374-450): forward over a batch of samples, hand-derived
// backward, gradient accumulation over the batch, Adam.
//
// Bit-exact with the reference by construction: every scalar the reference
// computes in a sequential f32 loop is produced here by ONE thread walking the
// same index order (products rounded before each add, no FMA: the library is
// built with --fmad=false and the intrinsics below are the _rn forms).  What
// runs in parallel are only independent chains: different outputs of a GEMV,
// different samples of the batch, different gradient elements.  A gradient
// element's chain over the samples of a step is sample-ordered, which is the
// order the reference's per-sample backward accumulates into `grad`.
#include "train.h"

#include "expf_glibc.cuh"

namespace smoe {

namespace {

constexpr int kKC = 16, kGemmThreads = 256;
constexpr int kPad = 4;  // keeps the k-contiguous tile stores off a single bank

// 16x16 threads, each owning a TM x TN block of independent chains; the CTA
// tile is (16*TM) x (16*TN).  A thread's columns are TN/4 float4 groups 64
// apart (rows likewise for TM >= 4) so a warp's shared-memory reads are
// contiguous.  Products are formed two at a time with FMUL2 (each lane of the
// pair rounded separately, exactly like two FMULs) and added with scalar
// FADDs in k order.  Tiles are double-buffered: the next k chunk is fetched
// into registers while the current one is consumed.
template <int TM>
__device__ __forceinline__ int row_of(int t, int i) {
    if constexpr (TM % 4 == 0) return (i >> 2) * 64 + t * 4 + (i & 3);
    else return t * TM + i;
}

template <int TM, int TN>  // TM even, TN a multiple of 4
__global__ void __launch_bounds__(kGemmThreads, (TM * TN >= 64) ? 1 : 2) k_chain_gemm(ChainGemm g) {
    constexpr int TA = 16 * TM, TB = 16 * TN;
    constexpr int LPT = kKC * TA / kGemmThreads, RPT = kKC * TB / kGemmThreads;
    __shared__ __align__(16) float Ls[2][kKC][TA + kPad];
    __shared__ __align__(16) float Rs[2][kKC][TB + kPad];
    const int tid = threadIdx.x, ta = tid >> 4, tb = tid & 15;
    const int a0 = blockIdx.y * TA, b0 = blockIdx.x * TB;
    float acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const int a = a0 + row_of<TM>(ta, i), b = b0 + row_of<TN>(tb, j);
            acc[i][j] = (g.init && a < g.A && b < g.B) ? g.init[a * g.osa + b * g.osb] : 0.0f;
        }
    const bool l_acontig = g.lsa == 1, r_bcontig = g.rsb == 1;
    float lr[LPT], rr[RPT];
    auto fetch = [&](int k0) {
#pragma unroll
        for (int q = 0; q < LPT; ++q) {
            const int idx = tid + q * kGemmThreads;
            const int kk = l_acontig ? idx / TA : idx % kKC, aa = l_acontig ? idx % TA : idx / kKC;
            const int a = a0 + aa, k = k0 + kk;
            lr[q] = (a < g.A && k < g.K) ? __ldg(g.L + k * g.lsk + a * g.lsa) : 0.0f;
        }
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const int idx = tid + q * kGemmThreads;
            const int kk = r_bcontig ? idx / TB : idx % kKC, bb = r_bcontig ? idx % TB : idx / kKC;
            const int b = b0 + bb, k = k0 + kk;
            rr[q] = (b < g.B && k < g.K) ? __ldg(g.R + k * g.rsk + b * g.rsb) : 0.0f;
        }
    };
    auto stash = [&](int buf) {
#pragma unroll
        for (int q = 0; q < LPT; ++q) {
            const int idx = tid + q * kGemmThreads;
            const int kk = l_acontig ? idx / TA : idx % kKC, aa = l_acontig ? idx % TA : idx / kKC;
            Ls[buf][kk][aa] = lr[q];
        }
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const int idx = tid + q * kGemmThreads;
            const int kk = r_bcontig ? idx / TB : idx % kKC, bb = r_bcontig ? idx % TB : idx / kKC;
            Rs[buf][kk][bb] = rr[q];
        }
    };
    fetch(0);
    stash(0);
    __syncthreads();
    int buf = 0;
    for (int k0 = 0; k0 < g.K; k0 += kKC) {
        const int kc = min(kKC, g.K - k0);
        const bool more = k0 + kKC < g.K;
        if (more) fetch(k0 + kKC);
        auto step = [&](int kk) {
            float av[TM], bv[TN];
            if constexpr (TM % 4 == 0) {
#pragma unroll
                for (int i = 0; i < TM; i += 4) {
                    const float4 v = *reinterpret_cast<const float4*>(&Ls[buf][kk][row_of<TM>(ta, i)]);
                    av[i] = v.x, av[i + 1] = v.y, av[i + 2] = v.z, av[i + 3] = v.w;
                }
            } else {
#pragma unroll
                for (int i = 0; i < TM; i += 2) {
                    const float2 v = *reinterpret_cast<const float2*>(&Ls[buf][kk][ta * TM + i]);
                    av[i] = v.x, av[i + 1] = v.y;
                }
            }
#pragma unroll
            for (int j = 0; j < TN; j += 4) {
                const float4 v = *reinterpret_cast<const float4*>(&Rs[buf][kk][row_of<TN>(tb, j)]);
                bv[j] = v.x, bv[j + 1] = v.y, bv[j + 2] = v.z, bv[j + 3] = v.w;
            }
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; j += 2) {
                    const float2 pr = __fmul2_rn(make_float2(av[i], av[i]), make_float2(bv[j], bv[j + 1]));
                    acc[i][j] = __fadd_rn(acc[i][j], pr.x);
                    acc[i][j + 1] = __fadd_rn(acc[i][j + 1], pr.y);
                }
        };
        if (kc == kKC) {
#pragma unroll
            for (int kk = 0; kk < kKC; ++kk) step(kk);
        } else {
            for (int kk = 0; kk < kc; ++kk) step(kk);  // never touches k >= K (keeps -0 chains exact)
        }
        if (more) stash(buf ^ 1);
        __syncthreads();
        buf ^= 1;
    }
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const int a = a0 + row_of<TM>(ta, i), b = b0 + row_of<TN>(tb, j);
            if (a >= g.A || b >= g.B) continue;
            const long long o = a * g.osa + b * g.osb;
            const float v = acc[i][j];
            switch (g.epi) {
                case kEpiAddPos:
                    g.out[o] = __fadd_rn(v, g.aux[static_cast<long long>(a % g.lp) * g.B + b]);
                    break;
                case kEpiSilu:
                    g.out[o] = v;
                    g.out2[o] = __fdiv_rn(v, __fadd_rn(1.0f, expf_glibc(-v)));
                    break;
                case kEpiAddAfter:
                    g.out[o] = __fadd_rn(g.aux[o], v);
                    break;
                case kEpiSiluGrad: {
                    const float u = g.aux[o];
                    const float sig = __fdiv_rn(1.0f, __fadd_rn(1.0f, expf_glibc(-u)));
                    if (g.out) g.out[o] = v;
                    g.out2[o] = __fmul_rn(__fmul_rn(v, sig), __fadd_rn(1.0f, __fmul_rn(u, __fsub_rn(1.0f, sig))));
                    break;
                }
                default:
                    g.out[o] = v;
            }
        }
}

__global__ void k_est_gather(const float* inputs, const float* targets, const int64_t* tok, int lp, int d, int E,
                             float* Qb, float* Tb) {
    const int s = blockIdx.x;
    const long long src = tok[s / lp] * lp + s % lp;
    for (int i = threadIdx.x; i < d; i += blockDim.x) Qb[static_cast<long long>(s) * d + i] = inputs[src * d + i];
    for (int i = threadIdx.x; i < E; i += blockDim.x) Tb[static_cast<long long>(s) * E + i] = targets[src * E + i];
}

// estimator.cpp:133-147: mean, variance (two sequential f32 chains), inv_std,
// xhat; y = gain * xhat + bias as the head consumes it (estimator.cpp:153).
__global__ void k_est_layernorm(const float* H, const float* gain, const float* bias, int dm, float eps, float* XHAT,
                                float* Y, float* inv_std) {
    extern __shared__ float sh[];
    const int s = blockIdx.x;
    const float* h = H + static_cast<long long>(s) * dm;
    for (int j = threadIdx.x; j < dm; j += blockDim.x) sh[j] = h[j];
    __shared__ float st[2];
    __syncthreads();
    if (threadIdx.x == 0) {
        float mean = 0.0f;
        for (int j = 0; j < dm; ++j) mean = __fadd_rn(mean, sh[j]);
        mean = __fdiv_rn(mean, static_cast<float>(dm));
        float var = 0.0f;
        for (int j = 0; j < dm; ++j) {
            const float c = __fsub_rn(sh[j], mean);
            var = __fadd_rn(var, __fmul_rn(c, c));
        }
        var = __fdiv_rn(var, static_cast<float>(dm));
        st[0] = mean;
        st[1] = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, eps)));
        inv_std[s] = st[1];
    }
    __syncthreads();
    const float mean = st[0], is = st[1];
    for (int j = threadIdx.x; j < dm; j += blockDim.x) {
        const float xh = __fmul_rn(__fsub_rn(sh[j], mean), is);
        XHAT[static_cast<long long>(s) * dm + j] = xh;
        Y[static_cast<long long>(s) * dm + j] = __fadd_rn(__fmul_rn(gain[j], xh), bias[j]);
    }
}

// softmax_inplace<float> (estimator.cpp:79-90) of n values in smem: the max is
// order-free, the exponentials are independent, the normaliser is one
// sequential chain.
__device__ void softmax_f32_block(float* v, int n, float* red) {
    float mx = -__int_as_float(0x7f800000);
    for (int i = threadIdx.x; i < n; i += blockDim.x) mx = fmaxf(mx, v[i]);
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    __syncwarp();
    for (int i = threadIdx.x; i < n; i += blockDim.x) v[i] = expf_glibc(__fsub_rn(v[i], mx));
    __syncwarp();
    if (threadIdx.x == 0) {
        float z = 0.0f;
        for (int i = 0; i < n; ++i) z = __fadd_rn(z, v[i]);
        red[0] = z;
    }
    __syncwarp();
    const float z = red[0];
    for (int i = threadIdx.x; i < n; i += blockDim.x) v[i] = __fdiv_rn(v[i], z);
    __syncwarp();
}

// One warp per sample.
__global__ void __launch_bounds__(32) k_est_softmax(const float* logits, const float* targets, int E, float weight,
                                                    float* probs, float* glog) {
    extern __shared__ float sm[];
    float* p = sm;
    float* t = sm + E;
    float* red = sm + 2 * E;
    const long long s = blockIdx.x;
    for (int i = threadIdx.x; i < E; i += 32) p[i] = logits[s * E + i];
    if (targets)
        for (int i = threadIdx.x; i < E; i += 32) t[i] = targets[s * E + i];
    __syncwarp();
    softmax_f32_block(p, E, red);
    for (int i = threadIdx.x; i < E; i += 32) probs[s * E + i] = p[i];
    if (!targets) return;
    softmax_f32_block(t, E, red + 1);
    for (int i = threadIdx.x; i < E; i += 32) glog[s * E + i] = __fmul_rn(weight, __fsub_rn(p[i], t[i]));
}

// estimator.cpp:205-224.
__global__ void k_est_ln_backward(const float* GY, const float* XHAT, const float* inv_std, const float* gain, int dm,
                                  float* GH) {
    extern __shared__ float sh[];
    float* gx = sh;
    float* xh = sh + dm;
    __shared__ float st[2];
    const long long s = blockIdx.x;
    for (int j = threadIdx.x; j < dm; j += blockDim.x) {
        xh[j] = XHAT[s * dm + j];
        gx[j] = __fmul_rn(GY[s * dm + j], gain[j]);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float m1 = 0.0f, m2 = 0.0f;
        for (int j = 0; j < dm; ++j) {
            m1 = __fadd_rn(m1, gx[j]);
            m2 = __fadd_rn(m2, __fmul_rn(gx[j], xh[j]));
        }
        st[0] = __fdiv_rn(m1, static_cast<float>(dm));
        st[1] = __fdiv_rn(m2, static_cast<float>(dm));
    }
    __syncthreads();
    const float m1 = st[0], m2 = st[1], is = inv_std[s];
    for (int j = threadIdx.x; j < dm; j += blockDim.x)
        GH[s * dm + j] = __fmul_rn(is, __fsub_rn(__fsub_rn(gx[j], m1), __fmul_rn(xh[j], m2)));
}

// blockIdx.y == 0: ln_gain / ln_bias grads; y = 1 + l: pos[l] grad.
__global__ void k_est_small_grads(const float* GY, const float* XHAT, const float* GZ, int S, int lp, int dm,
                                  float* g_gain, float* g_bias, float* g_pos) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= dm) return;
    constexpr int U = 16;  // loads of U samples issued ahead of their sequential adds
    if (blockIdx.y == 0) {
        float gg = 0.0f, gb = 0.0f;
        for (int s0 = 0; s0 < S; s0 += U) {
            float gy[U], xh[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long long o = static_cast<long long>(min(s0 + u, S - 1)) * dm + j;
                gy[u] = GY[o];
                xh[u] = XHAT[o];
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (s0 + u < S) {
                    gg = __fadd_rn(gg, __fmul_rn(gy[u], xh[u]));
                    gb = __fadd_rn(gb, gy[u]);
                }
        }
        g_gain[j] = gg;
        g_bias[j] = gb;
    } else {
        const int l = blockIdx.y - 1;
        float gp = 0.0f;
        for (int s0 = l; s0 < S; s0 += U * lp) {
            float gz[U];
#pragma unroll
            for (int u = 0; u < U; ++u) gz[u] = GZ[static_cast<long long>(min(s0 + u * lp, S - 1)) * dm + j];
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (s0 + u * lp < S) gp = __fadd_rn(gp, gz[u]);
        }
        g_pos[static_cast<long long>(l) * dm + j] = gp;
    }
}

// adam_step (estimator.cpp:301-322), f64 update of f32 state.
__global__ void k_est_adam(float* params, const float* grad, float* m, float* v, long long n, double lr, double b1,
                           double b2, double eps, double b1c, double b2c) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double gi = grad[i];
    const double mi = __dadd_rn(__dmul_rn(b1, static_cast<double>(m[i])), __dmul_rn(__dsub_rn(1.0, b1), gi));
    const double vi = __dadd_rn(__dmul_rn(b2, static_cast<double>(v[i])),
                                __dmul_rn(__dmul_rn(__dsub_rn(1.0, b2), gi), gi));
    m[i] = static_cast<float>(mi);
    v[i] = static_cast<float>(vi);
    const double mhat = __ddiv_rn(mi, b1c), vhat = __ddiv_rn(vi, b2c);
    const double upd = __ddiv_rn(__dmul_rn(lr, mhat), __dadd_rn(__dsqrt_rn(vhat), eps));
    params[i] = __fsub_rn(params[i], static_cast<float>(upd));
}

}  // namespace

// Largest per-thread block that still gives every SM a CTA: no split-k is
// possible (each chain is sequential), so narrow outputs take small tiles.
cudaError_t launch_chain_gemm(const ChainGemm& g, cudaStream_t s) {
    if (g.A <= 0 || g.B <= 0) return cudaSuccess;
    auto ctas = [&](int t) { return static_cast<long long>((g.A + t - 1) / t) * ((g.B + t - 1) / t); };
    if (ctas(128) >= 2 * 148) {
        k_chain_gemm<8, 8><<<dim3((g.B + 127) / 128, (g.A + 127) / 128), kGemmThreads, 0, s>>>(g);
    } else if (ctas(64) >= 148) {
        k_chain_gemm<4, 4><<<dim3((g.B + 63) / 64, (g.A + 63) / 64), kGemmThreads, 0, s>>>(g);
    } else {
        k_chain_gemm<2, 4><<<dim3((g.B + 63) / 64, (g.A + 31) / 32), kGemmThreads, 0, s>>>(g);
    }
    return cudaGetLastError();
}

cudaError_t launch_est_gather(const float* inputs, const float* targets, const int64_t* tok, int S, int lp, int d,
                              int E, float* Qb, float* Tb, cudaStream_t s) {
    k_est_gather<<<S, 256, 0, s>>>(inputs, targets, tok, lp, d, E, Qb, Tb);
    return cudaGetLastError();
}

cudaError_t launch_est_layernorm(const float* H, const float* gain, const float* bias, int S, int dm, float eps,
                                 float* XHAT, float* Y, float* inv_std, cudaStream_t s) {
    k_est_layernorm<<<S, 128, dm * 4, s>>>(H, gain, bias, dm, eps, XHAT, Y, inv_std);
    return cudaGetLastError();
}

cudaError_t launch_est_softmax(const float* logits, const float* targets, int S, int E, float weight, float* probs,
                               float* glog, cudaStream_t s) {
    k_est_softmax<<<S, 32, (2 * E + 2) * 4, s>>>(logits, targets, E, weight, probs, glog);
    return cudaGetLastError();
}

cudaError_t launch_est_ln_backward(const float* GY, const float* XHAT, const float* inv_std, const float* gain,
                                   int S, int dm, float* GH, cudaStream_t s) {
    k_est_ln_backward<<<S, 128, 2 * dm * 4, s>>>(GY, XHAT, inv_std, gain, dm, GH);
    return cudaGetLastError();
}

cudaError_t launch_est_small_grads(const float* GY, const float* XHAT, const float* GZ, int S, int lp, int dm,
                                   float* g_gain, float* g_bias, float* g_pos, cudaStream_t s) {
    k_est_small_grads<<<dim3((dm + 127) / 128, lp + 1), 128, 0, s>>>(GY, XHAT, GZ, S, lp, dm, g_gain, g_bias, g_pos);
    return cudaGetLastError();
}

cudaError_t launch_est_adam(float* params, const float* grad, float* m, float* v, long long n, double lr,
                            double b1, double b2, double eps, double b1c, double b2c, cudaStream_t s) {
    k_est_adam<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(params, grad, m, v, n, lr, b1, b2, eps, b1c,
                                                                       b2c);
    return cudaGetLastError();
}

}  // namespace smoe
