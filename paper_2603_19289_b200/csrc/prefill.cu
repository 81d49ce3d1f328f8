// prefill.cu — batched prefill: all P prompt tokens go
// through a layer together, with true routing (forward_decode semantics,
// model.cpp:355-389), so every dense weight is streamed once per layer instead
// of once per token and every executed expert once per layer instead of once
// per token that selected it.
//
// Arithmetic contract: identical to the per-token path (kernels.cu) — each
// (row, token) dot product is the reference's sequential f32 chain in column
// order (run_multi: one weight stream, T independent chains per lane), the
// f64 softmax / rms steps are the same, the mixture is summed in decision
// order.  The prefilled KV cache, the last token's logits and every later
// decode step therefore equal the token-by-token prefill bit for bit
// (tests/test_gpu.py::test_batched_prefill_*).
//
// Orchestration (Session::prefill_batched): per layer, qkv -> attention ->
// wo -> router -> decisions + per-expert token lists on the device; the host
// reads the union of executed experts, loads them into HBM slots in waves of
// at most C experts (cache fraction permitting) and runs the gate/up and down
// kernels per wave; then the per-token mixture.
#include "kernels.h"
#include "smoe_chain.cuh"

namespace smoe {

namespace {

constexpr int kPT = 8;  // tokens per CTA (independent chains per lane)
constexpr int kPW = 12;  // max warps per CTA: row tiles sharing one staging of the token inputs
using PipePF = WarpPipe<uint16_t, 3, kCCf>;  // 4 KB chunks, 12 KB per warp
using PipePD = PipePF;
constexpr int kPipeStride = (PipePF::kBytes + 127) & ~127;  // per-warp pipe footprint, 128-aligned
// one-warp CTAs (small batches: few row tiles per token group) have the SM's
// shared memory to themselves: a 64 KB in-flight window instead of 12 KB
using PipeDeep = WarpPipe<uint16_t, 4, 256>;
template <class Pipe>
__host__ __device__ constexpr int pipe_stride() { return (Pipe::kBytes + 127) & ~127; }

// run_multi with as many chains as the CTA has tokens (1, 2, 4 or 8): a
// batch of one sequence must not pay for eight chains.
template <class Pipe>
__device__ __forceinline__ void run_multi_n(Pipe& pipe, const uint16_t* tile, int cols, const float* xs, int stride,
                                            int nt, float (&acc)[kPT]) {
    if (nt <= 1) {
        float a[1];
        run_multi<1>(pipe, tile, cols, xs, stride, nt, a);
        acc[0] = a[0];
    } else if (nt <= 2) {
        float a[2];
        run_multi<2>(pipe, tile, cols, xs, stride, nt, a);
        acc[0] = a[0], acc[1] = a[1];
    } else if (nt <= 4) {
        float a[4];
        run_multi<4>(pipe, tile, cols, xs, stride, nt, a);
#pragma unroll
        for (int t = 0; t < 4; ++t) acc[t] = a[t];
    } else {
        run_multi<kPT>(pipe, tile, cols, xs, stride, nt, acc);
    }
}

__device__ __forceinline__ void pf_prologue() {
    pdl_wait();
    pdl_trigger();
}

// xs[t][*] = (v_t * scale_t) * gain (rms_norm, numerics.cpp:72-84) for the
// tokens of this CTA; scale_t precomputed per token by k_pf_scales from the
// producer's f64 partials (same fixed order as the per-token path).
__device__ void pf_stage_norm(const DevModel& m, const float* V, const float* scales, const float* gain,
                              const int* tok_of, int nt, float* xs, int xstride) {
    const int H = m.H;
    for (int t = 0; t < nt; ++t) {
        const int tok = tok_of[t];
        const float scale = __ldcg(scales + tok);
        const float4* v4 = reinterpret_cast<const float4*>(V + static_cast<long long>(tok) * m.Hp);
        const float4* g4 = reinterpret_cast<const float4*>(gain);
        float4* o4 = reinterpret_cast<float4*>(xs + t * xstride);
#pragma unroll 4
        for (int i = threadIdx.x; i < (H >> 2); i += blockDim.x) {
            const float4 a = __ldcg(v4 + i), g = __ldg(g4 + i);
            o4[i] = make_float4(a.x * scale * g.x, a.y * scale * g.y, a.z * scale * g.z, a.w * scale * g.w);
        }
    }
    __syncthreads();
}

}  // namespace

// per-token rms scale from the f64 partials of V (one warp per token)
__global__ void __launch_bounds__(32) k_pf_scales(DevModel m, PrefillDev pf, const double* ssq) {
    pf_prologue();
    const int t = blockIdx.x, nb = m.Hp / 32;
    const float s = rms_scale_from_partials(ssq + static_cast<long long>(t) * nb, nb, m.H, m.eps);
    if (threadIdx.x == 0) pf.scale[t] = s;
}

// ------------------------------------------------------------------ embed --
__global__ void __launch_bounds__(32) k_pf_embed(DevModel m, PrefillDev pf) {
    pf_prologue();
    const int t = blockIdx.y, j = blockIdx.x * 32 + threadIdx.x;
    const int tok = pf.tokens[t];
    const float v = j < m.H ? bf2f(m.emb[static_cast<long long>(tok) * m.H + j]) : 0.0f;
    pf.X[static_cast<long long>(t) * m.Hp + j] = v;
    warp_ssq_partial(v, pf.ssqx + static_cast<long long>(t) * (m.Hp / 32) + blockIdx.x);
}

// -------------------------------------------------------------------- qkv --
// q, k, v for kPT tokens per CTA (model.cpp:325-333), RoPE at position
// pos0 + t, K/V appended to the layer's cache, q kept per token.
template <class Pipe>
__global__ void __launch_bounds__(32 * kPW) k_pf_qkv(DevModel m, DevState st, PrefillDev pf, int layer) {
    const int H = m.H, Hr = round_up(H, 32), D = m.D, w = threadIdx.x >> 5;
    float* xs = reinterpret_cast<float*>(g_smem);  // [kPT][Hr]
    unsigned char* pipe_mem = align128(reinterpret_cast<unsigned char*>(xs + kPT * Hr)) + w * pipe_stride<Pipe>();
    const int rb = blockIdx.x * (blockDim.x >> 5) + w, t0 = blockIdx.y * kPT, nt = min(kPT, pf.P - t0);
    const bool has_tile = rb * 32 < m.QKVp;
    const uint16_t* tile = m.wqkv + layer * m.qkv_stride + static_cast<long long>(rb) * H * 32;
    Pipe pipe;
    pipe.init(pipe_mem);
    if (has_tile) pipe.prime(tile, H);
    pf_prologue();
    const int p0 = pf.pos_dev ? __ldcg(pf.pos_dev) : pf.pos0;
    int tok_of[kPT];
#pragma unroll
    for (int t = 0; t < kPT; ++t) tok_of[t] = t0 + t;
    pf_stage_norm(m, pf.X, pf.scale, m.attn_gain + static_cast<long long>(layer) * H, tok_of, nt, xs, Hr);
    if (!has_tile) return;
    float acc[kPT];
    run_multi_n(pipe, tile, H, xs, Hr, nt, acc);
    const int lane = threadIdx.x & 31, R = rb * 32 + lane;
#pragma unroll
    for (int t = 0; t < kPT; ++t) {
        float a = acc[t];
        const float other = __shfl_xor_sync(0xffffffffu, a, 1);
        if (t >= nt) continue;
        const int pos = pf.bkc ? p0 : pf.pos0 + t0 + t;
        if (R < 2 * D) {  // RoPE pair (2i, 2i+1), model.cpp:309-321
            const int i = (R % D) >> 1;
            const float c = m.rope[(static_cast<long long>(pos) * (D / 2) + i) * 2];
            const float s = m.rope[(static_cast<long long>(pos) * (D / 2) + i) * 2 + 1];
            const bool even = (R & 1) == 0;
            const float x0 = even ? a : other, x1 = even ? other : a;
            a = even ? (x0 * c - x1 * s) : (x0 * s + x1 * c);
        }
        const long long kv = (static_cast<long long>(layer) * m.cap + pos) * D +
                             (pf.bkc ? static_cast<long long>(t0 + t) * pf.bkv_stride : 0);
        if (R < D)
            pf.Q[static_cast<long long>(t0 + t) * D + R] = a;
        else if (R < 2 * D)
            (pf.bkc ? pf.bkc : st.kc)[kv + R - D] = a;
        else if (R < 3 * D)
            (pf.bkc ? pf.bvc : st.vc)[kv + R - 2 * D] = a;
    }
}

// -------------------------------------------------------------- attention --
// scores / softmax / context for token t over positions 0 .. pos0 + t
// (model.cpp:335-351), one CTA per token; the same operation order as k_attn.
constexpr int kPfAttnThreads = 256;
__global__ void __launch_bounds__(kPfAttnThreads) k_pf_attn(DevModel m, DevState st, PrefillDev pf,
                                                             int layer) {
    pf_prologue();
    const int p0 = pf.pos_dev ? __ldcg(pf.pos_dev) : pf.pos0;
    const int D = m.D, t = blockIdx.x, n = (pf.bkc ? p0 : pf.pos0 + t) + 1;
    float* red = reinterpret_cast<float*>(g_smem);  // [32]
    float* qs = red + 32;                           // [D]
    double* e = reinterpret_cast<double*>(qs + kMaxD);
    float* sc = reinterpret_cast<float*>(e + n);
    if ((pf.bkc ? (pf.pos_dev ? m.cap : p0 + 1) : pf.pos0 + pf.P) > pf.attn_smem_positions) {  // global scratch
        e = pf.attn_scratch + static_cast<long long>(t) * 2 * m.cap;
        sc = reinterpret_cast<float*>(e + m.cap);
    }
    const long long seq = pf.bkc ? static_cast<long long>(t) * pf.bkv_stride : 0;
    const float* K = (pf.bkc ? pf.bkc : st.kc) + seq + static_cast<long long>(layer) * m.cap * D;
    const float* V = (pf.bkc ? pf.bvc : st.vc) + seq + static_cast<long long>(layer) * m.cap * D;
    for (int i = threadIdx.x; i < D; i += blockDim.x) qs[i] = __ldcg(pf.Q + static_cast<long long>(t) * D + i);
    __syncthreads();
    float lmax = -INFINITY;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const float4* kj = reinterpret_cast<const float4*>(K + static_cast<long long>(j) * D);
        float acc = 0.0f;
        for (int i = 0; i < D / 4; ++i) {
            const float4 kv = __ldcg(kj + i);
            acc = acc + qs[4 * i] * kv.x;
            acc = acc + qs[4 * i + 1] * kv.y;
            acc = acc + qs[4 * i + 2] * kv.z;
            acc = acc + qs[4 * i + 3] * kv.w;
        }
        const float v = acc * m.inv_sqrt_d;
        sc[j] = v;
        lmax = fmaxf(lmax, v);
    }
    const float mx = block_max_f(lmax, red);
    for (int j = threadIdx.x; j < n; j += blockDim.x)
        e[j] = exp_glibc(static_cast<double>(sc[j]) - static_cast<double>(mx));
    __syncthreads();
    __shared__ double zs;
    if (threadIdx.x == 0) {  // f64 partition in index order, numerics.cpp:46-49
        double z = 0.0;
        for (int j = 0; j < n; ++j) z += e[j];
        zs = z;
    }
    __syncthreads();
    const double z = zs;
    for (int j = threadIdx.x; j < n; j += blockDim.x) sc[j] = static_cast<float>(e[j] / z);
    __syncthreads();
    const int i = threadIdx.x;
    if (i < D) {
        float acc = 0.0f;
        for (int j = 0; j < n; ++j) acc = acc + sc[j] * __ldcg(V + static_cast<long long>(j) * D + i);
        pf.ctx[static_cast<long long>(t) * D + i] = acc;
    }
}

// --------------------------------------------------------------------- wo --
// r = x + wo . ctx (model.cpp:352, 380) for kPT tokens, rms partials of r.
__global__ void __launch_bounds__(32 * kPW) k_pf_wo(DevModel m, PrefillDev pf, int layer) {
    const int D = m.D, w = threadIdx.x >> 5;
    float* xs = reinterpret_cast<float*>(g_smem);  // [kPT][kMaxD]
    unsigned char* pipe_mem = align128(reinterpret_cast<unsigned char*>(xs + kPT * kMaxD)) + w * kPipeStride;
    const int rb = blockIdx.x * (blockDim.x >> 5) + w, t0 = blockIdx.y * kPT, nt = min(kPT, pf.P - t0);
    const bool has_tile = rb * 32 < m.Hp;
    const uint16_t* tile = m.wo + layer * m.wo_stride + static_cast<long long>(rb) * D * 32;
    PipePD pipe;
    pipe.init(pipe_mem);
    if (has_tile) pipe.prime(tile, D);
    pf_prologue();
    for (int t = 0; t < nt; ++t)
        for (int i = threadIdx.x; i < D; i += blockDim.x)
            xs[t * kMaxD + i] = __ldcg(pf.ctx + static_cast<long long>(t0 + t) * D + i);
    __syncthreads();
    if (!has_tile) return;
    float acc[kPT];
    run_multi_n(pipe, tile, D, xs, kMaxD, nt, acc);
    const int j = rb * 32 + (threadIdx.x & 31);
    for (int t = 0; t < nt; ++t) {
        const long long o = static_cast<long long>(t0 + t) * m.Hp + j;
        const float r = j < m.H ? __ldcg(pf.X + o) + acc[t] : 0.0f;
        pf.R[o] = r;
        warp_ssq_partial(r, pf.ssqr + static_cast<long long>(t0 + t) * (m.Hp / 32) + rb);
    }
}

// ----------------------------------------------------------------- router --
// true router logits gate . rms_norm(r, moe_gain) (model.cpp:276-281).
template <class Pipe>
__global__ void __launch_bounds__(32 * kPW) k_pf_router(DevModel m, PrefillDev pf, int layer) {
    const int H = m.H, Hr = round_up(H, 32), E = m.E, w = threadIdx.x >> 5;
    float* xs = reinterpret_cast<float*>(g_smem);  // [kPT][Hr]
    unsigned char* pipe_mem = align128(reinterpret_cast<unsigned char*>(xs + kPT * Hr)) + w * pipe_stride<Pipe>();
    const int rb = blockIdx.x * (blockDim.x >> 5) + w, t0 = blockIdx.y * kPT, nt = min(kPT, pf.P - t0);
    const bool has_tile = rb * 32 < m.Ep;
    const uint16_t* tile = m.gate + layer * m.gate_stride + static_cast<long long>(rb) * H * 32;
    Pipe pipe;
    pipe.init(pipe_mem);
    if (has_tile) pipe.prime(tile, H);
    pf_prologue();
    int tok_of[kPT];
#pragma unroll
    for (int t = 0; t < kPT; ++t) tok_of[t] = t0 + t;
    pf_stage_norm(m, pf.R, pf.scale, m.moe_gain + static_cast<long long>(layer) * H, tok_of, nt, xs, Hr);
    if (!has_tile) return;
    float acc[kPT];
    run_multi_n(pipe, tile, H, xs, Hr, nt, acc);
    const int e = rb * 32 + (threadIdx.x & 31);
    if (e < E)
        for (int t = 0; t < nt; ++t) pf.lg[static_cast<long long>(t0 + t) * E + e] = acc[t];
}

// make_decision per token (model.cpp:258-274) and per-expert counts.
__global__ void __launch_bounds__(32) k_pf_decide(DevModel m, PrefillDev pf) {
    pf_prologue();
    __shared__ double se[kMaxE];
    __shared__ float sp[kMaxE];
    const int t = blockIdx.x, K = m.K;
    warp_decision(pf.lg + static_cast<long long>(t) * m.E, m.E, K, m.gating, sp, se, pf.ids + t * K,
                  pf.gates + t * K);
    __syncwarp();
    if (threadIdx.x < K) atomicAdd(pf.cnt + __ldcg(pf.ids + t * K + threadIdx.x), 1);
}

// offsets of the per-expert (token, slot) lists: exclusive scan over E (1 CTA)
__global__ void k_pf_offsets(DevModel m, PrefillDev pf) {
    pf_prologue();
    if (threadIdx.x == 0) {
        int s = 0;
        for (int e = 0; e < m.E; ++e) {
            pf.off[e] = s;
            s += pf.cnt[e];
            pf.fill[e] = 0;
        }
        pf.off[m.E] = s;
    }
}

// list entries t * K + i grouped by expert (order inside a group is free: every
// (token, expert) pair is computed independently and mixed per token later)
__global__ void __launch_bounds__(32) k_pf_scatter(DevModel m, PrefillDev pf) {
    pf_prologue();
    const int t = blockIdx.x, K = m.K;
    if (threadIdx.x < K) {
        const int e = pf.ids[t * K + threadIdx.x];
        const int slot = pf.off[e] + atomicAdd(pf.fill + e, 1);
        pf.list[slot] = t * K + threadIdx.x;
    }
}

// ---------------------------------------------------------------- experts --
// gate/up: grid (Hmp/16, wave experts, token chunks of kPT); h = silu(g) * u.
// T = chains per lane (tokens per CTA actually used): 8 for prefill, the
// next power of two of the batch for batched decode.
template <int T>
__device__ __forceinline__ void run_multi_t(PipePF& pipe, const uint16_t* tile, int cols, const float* xs, int stride,
                                            int nt, float (&acc)[kPT]) {
    if constexpr (T == kPT) {
        run_multi<kPT>(pipe, tile, cols, xs, stride, nt, acc);
    } else if constexpr (T == 0) {  // per-chunk dispatch (batched decode: chunks of 1-8 tokens)
        run_multi_n(pipe, tile, cols, xs, stride, nt, acc);
    } else {
        float a[T];
        run_multi<T>(pipe, tile, cols, xs, stride, nt, a);
#pragma unroll
        for (int t = 0; t < T; ++t) acc[t] = a[t];
    }
}

template <int T>
__global__ void __launch_bounds__(32 * kPW) k_pf_gu(DevModel m, PrefillDev pf, int layer, PfWave wv) {
    const int H = m.H, Hr = round_up(H, 32), K = m.K, w = threadIdx.x >> 5;
    float* xs = reinterpret_cast<float*>(g_smem);  // [kPT][Hr]
    unsigned char* pipe_mem = align128(reinterpret_cast<unsigned char*>(xs + kPT * Hr)) + w * kPipeStride;
    pf_prologue();
    if (pf.nchunks && static_cast<int>(blockIdx.y) >= __ldcg(pf.nchunks)) return;
    const int u = __ldcg(pf.chunk_u + blockIdx.y), e = wv.e[u];
    const int rb = blockIdx.x * (blockDim.x >> 5) + w;
    const int b0 = pf.off[e], cnt = pf.off[e + 1] - b0, c0 = __ldcg(pf.chunk_c + blockIdx.y) * kPT;
    const int nt = min(kPT, cnt - c0);
    const bool has_tile = rb * 16 < m.Hmp;
    const uint16_t* tile = m.slots + (static_cast<long long>(layer) * m.C + wv.slot[u]) * m.expert_elems +
                           static_cast<long long>(rb) * H * 32;
    PipePF pipe;
    pipe.init(pipe_mem, kL2Normal);  // expert tiles are re-read by the other token chunks
    if (has_tile) pipe.prime(tile, H);
    int ent[kPT], tok_of[kPT];
#pragma unroll
    for (int t = 0; t < kPT; ++t) {
        ent[t] = t < nt ? __ldcg(pf.list + b0 + c0 + t) : 0;
        tok_of[t] = ent[t] / K;
    }
    pf_stage_norm(m, pf.R, pf.scale, m.moe_gain + static_cast<long long>(layer) * H, tok_of, nt, xs, Hr);
    if (!has_tile) return;
    float acc[kPT];
    run_multi_t<T>(pipe, tile, H, xs, Hr, nt, acc);
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int t = 0; t < (T == 0 ? kPT : T); ++t) {
        const float up = __shfl_xor_sync(0xffffffffu, acc[t], 1);
        if (t < nt && (lane & 1) == 0)
            pf.Hb[static_cast<long long>(ent[t]) * m.Hmp + rb * 16 + (lane >> 1)] = silu_ref(acc[t]) * up;
    }
}

// down: grid (Hp/32, wave experts, token chunks); raw expert rows into Y.
template <int T>
__global__ void __launch_bounds__(32 * kPW) k_pf_down(DevModel m, PrefillDev pf, int layer, PfWave wv, int tpb) {
    // tpb: tokens staged at a time (8, or fewer when Hmp * 4 B per token would
    // not fit, e.g. Mixtral's 14336); the tile is streamed once per staging.
    const int Hmp = m.Hmp, w = threadIdx.x >> 5;
    float* xs = reinterpret_cast<float*>(g_smem);  // [tpb][Hmp]
    unsigned char* pipe_mem = align128(reinterpret_cast<unsigned char*>(xs + tpb * Hmp)) + w * kPipeStride;
    pf_prologue();
    if (pf.nchunks && static_cast<int>(blockIdx.y) >= __ldcg(pf.nchunks)) return;
    const int u = __ldcg(pf.chunk_u + blockIdx.y), e = wv.e[u];
    const int rb = blockIdx.x * (blockDim.x >> 5) + w;
    const int b0 = pf.off[e], cnt = pf.off[e + 1] - b0, c0 = __ldcg(pf.chunk_c + blockIdx.y) * kPT;
    const int nt = min(kPT, cnt - c0);
    const bool has_tile = rb * 32 < m.Hp;
    const uint16_t* tile = m.slots + (static_cast<long long>(layer) * m.C + wv.slot[u]) * m.expert_elems +
                           m.gu_elems + static_cast<long long>(rb) * Hmp * 32;
    PipePD pipe;
    pipe.init(pipe_mem, kL2Normal);  // expert tiles are re-read by the other token chunks
    if (has_tile) pipe.prime(tile, m.Hm);
    int ent[kPT];
#pragma unroll
    for (int t = 0; t < kPT; ++t) ent[t] = t < nt ? __ldcg(pf.list + b0 + c0 + t) : 0;
    const int j = rb * 32 + (threadIdx.x & 31);
    for (int s0 = 0; s0 < nt; s0 += tpb) {
        const int ns = min(tpb, nt - s0);
        if (s0) __syncthreads();  // every warp is done with the previous staging
        for (int t = 0; t < ns; ++t) {
            const float4* h4 = reinterpret_cast<const float4*>(pf.Hb + static_cast<long long>(ent[s0 + t]) * Hmp);
            for (int i = threadIdx.x; i < Hmp / 4; i += blockDim.x)
                reinterpret_cast<float4*>(xs + t * Hmp)[i] = __ldcg(h4 + i);
        }
        __syncthreads();
        if (has_tile) {
            float acc[kPT];
            if (tpb == kPT)
                run_multi_t<T>(pipe, tile, m.Hm, xs, Hmp, ns, acc);
            else
                run_multi_n(pipe, tile, m.Hm, xs, Hmp, ns, acc);
            if (j < m.H)
                for (int t = 0; t < ns; ++t) pf.Y[static_cast<long long>(ent[s0 + t]) * m.Hp + j] = acc[t];
        }
    }
}

// mixture in decision order (model.cpp:297-301), x = r + m, rms partials of x.
__global__ void __launch_bounds__(32) k_pf_mix(DevModel m, PrefillDev pf) {
    pf_prologue();
    const int t = blockIdx.y, rb = blockIdx.x, j = rb * 32 + threadIdx.x, K = m.K;
    float xv = 0.0f;
    if (j < m.H) {
        float out = 0.0f;
        for (int i = 0; i < K; ++i)
            out += __ldcg(pf.gates + t * K + i) * __ldcg(pf.Y + (static_cast<long long>(t) * K + i) * m.Hp + j);
        xv = __ldcg(pf.R + static_cast<long long>(t) * m.Hp + j) + out;
    }
    pf.X[static_cast<long long>(t) * m.Hp + j] = xv;
    warp_ssq_partial(xv, pf.ssqx + static_cast<long long>(t) * (m.Hp / 32) + rb);
}

// ------------------------------------------- batched decode under EP ----
// The single-token combine (kernels.cu k_ffn_down / k_ep_mix) over a step's
// B·k expert rows: every rank computed the rows Y[t·k + i] of the entries
// whose expert it owns; k_pf_ep_publish stores those rows into every rank's
// batched exchange buffer (peer memory; one writer per row), fences them
// system-wide, and the last of its CTAs makes ONE system-scope arrival on
// every rank's per-layer counter; k_pf_ep_wait (one CTA) waits for all
// `world` arrivals of this layer's step; k_pf_mix then reads the rows from the
// exchange buffer — the same rows, mixed in the same decision order, so the
// result equals the single-GPU batch bit for bit.  Layer parity double-
// buffers the exchange (a rank arrives for layer l only after its own layer-l
// work, so no rank can be two layers ahead of a peer).
__global__ void __launch_bounds__(128) k_pf_ep_publish(DevModel m, PrefillDev pf, DevEP ep, int layer) {
    pf_prologue();
    const int ent = blockIdx.x, K = m.K;
    const int e = __ldcg(pf.ids + ent);
    if (e % ep.world == ep.rank) {
        const long long o = (static_cast<long long>(layer & 1) * kEpBatchMax * K + ent) * m.Hp;
        const float4* src = reinterpret_cast<const float4*>(pf.Y + static_cast<long long>(ent) * m.Hp);
        for (int p = 0; p < ep.world; ++p) {
            float4* dst = reinterpret_cast<float4*>(ep.bxbuf[p] + o);
            for (int j = threadIdx.x; j < m.Hp / 4; j += blockDim.x) __stcg(dst + j, __ldcg(src + j));
        }
    }
    __threadfence_system();
    if (last_cta(ep.bdone + layer, gridDim.x) && threadIdx.x == 0) {
        __threadfence_system();
        for (int p = 0; p < ep.world; ++p) atomicAdd_system(ep.bcnt[p] + layer, 1);
    }
}

__global__ void __launch_bounds__(32) k_pf_ep_wait(DevEP ep, int layer, int* error, long long spin_limit) {
    pf_prologue();
    if (threadIdx.x != 0) return;
    const int want = (ep.bepoch[layer] + 1) * ep.world;
    const int* c = ep.bcnt[ep.rank] + layer;
    const long long t0 = clock64();
    for (;;) {
        int v;
        asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
        if (v >= want) break;
        if (*(volatile int*)error) break;
        if (clock64() - t0 > spin_limit) {
            atomicCAS(error, 0, 5000 + layer);  // EP batched combine: a peer never arrived
            break;
        }
        __nanosleep(64);
    }
    ep.bepoch[layer] += 1;
    __threadfence();
}

// hands the last token to the per-token state: x, its final-norm partials,
// position and input token, so k_final produces the prefill's next token.
__global__ void __launch_bounds__(32) k_pf_handoff(DevModel m, DevState st, PrefillDev pf) {
    pf_prologue();
    const int t = pf.P - 1, rb = blockIdx.x, j = rb * 32 + threadIdx.x;
    st.x[j] = __ldcg(pf.X + static_cast<long long>(t) * m.Hp + j);
    if (threadIdx.x == 0) {
        st.ssq_x[static_cast<long long>(m.L) * (m.Hp / 32) + rb] = __ldcg(pf.ssqx + static_cast<long long>(t) * (m.Hp / 32) + rb);
        if (rb == 0) {
            *st.pos = pf.pos0 + t;
            *st.tok_in = pf.tokens[t];
            // token / trace records of the P - 1 earlier steps are skipped, so
            // the last prefill token and later decode steps keep their indices
            *pf.dev_step = *pf.dev_step + t;  // k_final records the last token at t
            if (pf.trace_step) *pf.trace_step = *pf.trace_step + pf.P;  // no trace rows
        }
    }
}

// ------------------------------------------------------ batched decode --
// Normalised GEMV for kPT tokens per CTA: out[t][row] = W . ((V_t * scale_t) * gain)
// (predictor: gate_{l+1} over q_l; final: unembed over h).
template <class Pipe>
__global__ void __launch_bounds__(32 * kPW) k_pf_gemvn(DevModel m, PrefillDev pf, const float* V, const float* gain,
                                                       const uint16_t* W, int rows, float* out, int out_stride) {
    const int H = m.H, Hr = round_up(H, 32), w = threadIdx.x >> 5;
    float* xs = reinterpret_cast<float*>(g_smem);  // [kPT][Hr]
    unsigned char* pipe_mem = align128(reinterpret_cast<unsigned char*>(xs + kPT * Hr)) + w * pipe_stride<Pipe>();
    const int rb = blockIdx.x * (blockDim.x >> 5) + w, t0 = blockIdx.y * kPT, nt = min(kPT, pf.P - t0);
    const bool has_tile = rb * 32 < round_up(rows, 32);
    const uint16_t* tile = W + static_cast<long long>(rb) * H * 32;
    Pipe pipe;
    pipe.init(pipe_mem);
    if (has_tile) pipe.prime(tile, H);
    pf_prologue();
    int tok_of[kPT];
#pragma unroll
    for (int t = 0; t < kPT; ++t) tok_of[t] = t0 + t;
    pf_stage_norm(m, V, pf.scale, gain, tok_of, nt, xs, Hr);
    if (!has_tile) return;
    float acc[kPT];
    run_multi_n(pipe, tile, H, xs, Hr, nt, acc);
    const int r = rb * 32 + (threadIdx.x & 31);
    if (r < rows)
        for (int t = 0; t < nt; ++t) out[static_cast<long long>(t0 + t) * out_stride + r] = acc[t];
}

// make_decision per token on predicted logits -> pids/pgates[buf]
__global__ void __launch_bounds__(32) k_pf_decide_pred(DevModel m, PrefillDev pf, int buf) {
    pf_prologue();
    __shared__ double se[kMaxE];
    __shared__ float sp[kMaxE];
    const int t = blockIdx.x, K = m.K;
    const long long o = (static_cast<long long>(buf) * pf.P + t) * K;
    warp_decision(pf.lgp + static_cast<long long>(t) * m.E, m.E, K, m.gating, sp, se, pf.pids + o, pf.pgates + o);
}

// executed decision of every token := its prediction (Algorithm 1, l >= 1); counts
__global__ void __launch_bounds__(32) k_pf_take_pred(DevModel m, PrefillDev pf, int buf) {
    pf_prologue();
    const int t = blockIdx.x, K = m.K;
    if (threadIdx.x < K) {
        const long long o = (static_cast<long long>(buf) * pf.P + t) * K + threadIdx.x;
        const int e = __ldcg(pf.pids + o);
        pf.ids[t * K + threadIdx.x] = e;
        pf.gates[t * K + threadIdx.x] = __ldcg(pf.pgates + o);
        atomicAdd(pf.cnt + e, 1);
    }
}

// rd = r_l + layer_default(executed_l) (speculation.cpp:104-121) and its rms
// partials; grid (Hp/32, P).
__global__ void __launch_bounds__(32) k_pf_quasi(DevModel m, PrefillDev pf, int layer) {
    pf_prologue();
    const int t = blockIdx.y, rb = blockIdx.x, j = rb * 32 + threadIdx.x, K = m.K;
    float rd = 0.0f;
    if (j < m.H) {
        float d = 0.0f;
        for (int i = 0; i < K; ++i) {
            const int e = __ldcg(pf.ids + t * K + i);
            d = d + __ldcg(pf.gates + t * K + i) * __ldcg(m.dv + (static_cast<long long>(layer) * m.E + e) * m.H + j);
        }
        rd = __ldcg(pf.R + static_cast<long long>(t) * m.Hp + j) + d;
    }
    pf.RD[static_cast<long long>(t) * m.Hp + j] = rd;
    warp_ssq_partial(rd, pf.ssqrd + static_cast<long long>(t) * (m.Hp / 32) + rb);
}

// q_l materialised for the estimator (est-pf): Qn[t] = (RD_t * scale_t) * gain
// (rms_norm, numerics.cpp:72-84); grid (ceil(H/32), P).
__global__ void __launch_bounds__(32) k_pf_normq(DevModel m, PrefillDev pf, const float* gain, float* qn) {
    pf_prologue();
    const int t = blockIdx.y, j = blockIdx.x * 32 + threadIdx.x;
    if (j < m.H)
        qn[static_cast<long long>(t) * m.H + j] =
            (__ldcg(pf.RD + static_cast<long long>(t) * m.Hp + j) * __ldcg(pf.scale + t)) * gain[j];
}

// (expert, 8-token chunk) work list from the per-expert counts, expert order
// (wave = every expert, wave index = expert id; under EP only this rank's
// experts e % ep_world == ep_rank get work items)
__global__ void k_pf_chunks(DevModel m, PrefillDev pf, int ep_rank, int ep_world) {
    pf_prologue();
    if (threadIdx.x == 0) {
        int k = 0;
        for (int e = ep_rank; e < m.E; e += ep_world)
            for (int q = 0; q < (pf.cnt[e] + kPT - 1) / kPT; ++q) {
                pf.chunk_u[k] = e;
                pf.chunk_c[k] = q;
                ++k;
            }
        *pf.nchunks = k;
    }
}

// argmax_token (model.cpp:391-396): first maximum of each token's logits
__global__ void __launch_bounds__(32) k_pf_argmax(DevModel m, PrefillDev pf) {
    pf_prologue();
    const int t = blockIdx.x;
    const float* lg = pf.logits + static_cast<long long>(t) * m.V;
    float best = -INFINITY;
    int bi = 0x7fffffff;
    for (int i = threadIdx.x; i < m.V; i += 32) {
        const float v = lg[i];
        if (v > best) {  // first maximum within the lane's strided subsequence
            best = v;
            bi = i;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) {
            best = ov;
            bi = oi;
        }
    }
    if (threadIdx.x == 0) pf.next[t] = bi == 0x7fffffff ? 0 : bi;
}

// ---------------------------------------------------------------- launchers --
namespace {
size_t vecf(int n) { return static_cast<size_t>(round_up(n, 32)) * 4; }
// Warps per CTA for a kernel whose token staging takes `stage` bytes: as many
// row tiles (each with its own 16 KB pipe) as fit next to it, up to kPW.
constexpr size_t kPfSmemBudget = 220 * 1024;
// Warps per CTA: maximise resident row-tile warps per SM (CTAs per SM x W,
// each warp with its own pipe next to the CTA's token staging), discounted by
// the idle warps of the last CTA over the kernel's `tiles` row tiles.
int pf_warps(size_t stage, int tiles, long long groups) {
    // few row tiles x token groups (small batches): one warp per CTA, so the
    // tiles stream through as many SMs as possible
    if (groups <= 2 && static_cast<long long>(tiles) * groups <= 2 * 148) return 1;
    int best = 1;
    double best_score = -1.0;
    for (int w = kPW; w >= 1; --w) {
        const size_t smem = stage + 128 + static_cast<size_t>(w) * kPipeStride;
        if (smem > kPfSmemBudget) continue;
        const int per_sm = static_cast<int>((228 * 1024) / (smem + 1024));
        const double used = static_cast<double>(tiles) / (((tiles + w - 1) / w) * w);
        const double score = std::min(per_sm * w, 16) * used;
        if (score > best_score + 1e-9) {
            best_score = score;
            best = w;
        }
    }
    return best;
}
size_t pf_smem(size_t stage, int w) {
    return stage + 128 + static_cast<size_t>(w) * (w == 1 ? pipe_stride<PipeDeep>() : kPipeStride);
}
size_t pf_h_stage(const DevModel& m) { return kPT * vecf(m.H); }
size_t pf_wo_stage(const DevModel&) { return kPT * kMaxD * 4; }
// tokens staged at a time by k_pf_down: 8 unless a token's h row is too large
// (a power of two: run_multi reads every one of its T <= tpb staged rows)
int pf_down_tpb(const DevModel& m) {
    const size_t row = static_cast<size_t>(m.Hmp) * 4;
    int t = kPT;
    while (t > 1 && static_cast<size_t>(t) * row > 200 * 1024) t >>= 1;
    return t;
}
size_t pf_down_stage(const DevModel& m) { return pf_down_tpb(m) * static_cast<size_t>(m.Hmp) * 4; }
int cdiv(int a, int b) { return (a + b - 1) / b; }
size_t pf_attn_smem(const DevModel& m, int npos) {
    return (32 + kMaxD) * 4 + static_cast<size_t>(npos) * 12;
}
}  // namespace

int pf_attn_smem_positions() { return 12 * 1024; }

cudaError_t pf_preload() {
    const void* fns[] = {(const void*)k_pf_embed, (const void*)k_pf_qkv<PipePF>, (const void*)k_pf_qkv<PipeDeep>,
                         (const void*)k_pf_attn,
                         (const void*)k_pf_wo, (const void*)k_pf_router<PipePF>,
                         (const void*)k_pf_router<PipeDeep>, (const void*)k_pf_decide,
                         (const void*)k_pf_offsets, (const void*)k_pf_scatter, (const void*)k_pf_gu<0>,
                         (const void*)k_pf_gu<8>, (const void*)k_pf_down<0>, (const void*)k_pf_down<8>, (const void*)k_pf_mix, (const void*)k_pf_handoff,
                         (const void*)k_pf_scales, (const void*)k_pf_gemvn<PipePF>,
                         (const void*)k_pf_gemvn<PipeDeep>, (const void*)k_pf_decide_pred,
                         (const void*)k_pf_take_pred, (const void*)k_pf_quasi, (const void*)k_pf_argmax,
                         (const void*)k_pf_chunks, (const void*)k_pf_normq, (const void*)k_pf_ep_publish,
                         (const void*)k_pf_ep_wait};
    for (const void* f : fns) {
        cudaFuncAttributes a;
        cudaError_t e = cudaFuncGetAttributes(&a, f);
        if (e != cudaSuccess) return e;
        // opt-in maximum per block (227 KB on sm_100) minus the static shared memory
        e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(227 * 1024 - a.sharedSizeBytes));
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_pf_embed(const DevModel& m, const PrefillDev& pf, cudaStream_t s) {
    PDL(k_pf_embed, dim3(m.Hp / 32, pf.P), 32, 0, s, m, pf);
    return cudaGetLastError();
}

cudaError_t launch_gemvn(const DevModel& m, const PrefillDev& pf, int tiles, int tg, const float* V,
                         const float* gain, const uint16_t* W, int rows, float* out, int out_stride, cudaStream_t s) {
    const int w = pf_warps(pf_h_stage(m), tiles, tg);
    if (w == 1)
        PDL(k_pf_gemvn<PipeDeep>, dim3(tiles, tg), 32, pf_smem(pf_h_stage(m), 1), s, m, pf, V, gain, W, rows, out,
            out_stride);
    else
        PDL(k_pf_gemvn<PipePF>, dim3(cdiv(tiles, w), tg), 32 * w, pf_smem(pf_h_stage(m), w), s, m, pf, V, gain, W,
            rows, out, out_stride);
    return cudaGetLastError();
}

cudaError_t launch_pf_attn_block(const DevModel& m, const DevState& st, const PrefillDev& pf, int layer,
                                 cudaStream_t s) {
    const int tg = (pf.P + kPT - 1) / kPT;
    PDL(k_pf_scales, pf.P, 32, 0, s, m, pf, static_cast<const double*>(pf.ssqx));
    const int wh = pf_warps(pf_h_stage(m), m.QKVp / 32, tg), ww = pf_warps(pf_wo_stage(m), m.Hp / 32, tg);
    if (wh == 1)
        PDL(k_pf_qkv<PipeDeep>, dim3(m.QKVp / 32, tg), 32, pf_smem(pf_h_stage(m), 1), s, m, st, pf, layer);
    else
        PDL(k_pf_qkv<PipePF>, dim3(cdiv(m.QKVp / 32, wh), tg), 32 * wh, pf_smem(pf_h_stage(m), wh), s, m, st, pf, layer);
    const int nmax = pf.bkc ? (pf.pos_dev ? m.cap : pf.pos0 + 1) : pf.pos0 + pf.P;
    const int npos = nmax <= pf.attn_smem_positions ? nmax : 0;
    PDL(k_pf_attn, pf.P, kPfAttnThreads, pf_attn_smem(m, npos), s, m, st, pf, layer);
    PDL(k_pf_wo, dim3(cdiv(m.Hp / 32, ww), tg), 32 * ww, pf_smem(pf_wo_stage(m), ww), s, m, pf, layer);
    return cudaGetLastError();
}

cudaError_t launch_pf_route(const DevModel& m, const PrefillDev& pf, int layer, cudaStream_t s) {
    const int tg = (pf.P + kPT - 1) / kPT;
    PDL(k_pf_scales, pf.P, 32, 0, s, m, pf, static_cast<const double*>(pf.ssqr));
    const int wr = pf_warps(pf_h_stage(m), m.Ep / 32, tg);
    if (wr == 1)
        PDL(k_pf_router<PipeDeep>, dim3(m.Ep / 32, tg), 32, pf_smem(pf_h_stage(m), 1), s, m, pf, layer);
    else
        PDL(k_pf_router<PipePF>, dim3(cdiv(m.Ep / 32, wr), tg), 32 * wr, pf_smem(pf_h_stage(m), wr), s, m, pf, layer);
    PDL(k_pf_decide, pf.P, 32, 0, s, m, pf);
    PDL(k_pf_offsets, 1, 32, 0, s, m, pf);
    PDL(k_pf_scatter, pf.P, 32, 0, s, m, pf);
    return cudaGetLastError();
}

cudaError_t launch_pf_layer_dense(const DevModel& m, const DevState& st, const PrefillDev& pf, int layer,
                                  cudaStream_t s) {
    cudaError_t e = launch_pf_attn_block(m, st, pf, layer, s);
    return e != cudaSuccess ? e : launch_pf_route(m, pf, layer, s);
}

cudaError_t launch_pf_exec_pred(const DevModel& m, const PrefillDev& pf, int buf, cudaStream_t s) {
    // the router's scales of r_l feed the expert kernels (pf_stage_norm of R)
    PDL(k_pf_scales, pf.P, 32, 0, s, m, pf, static_cast<const double*>(pf.ssqr));
    PDL(k_pf_take_pred, pf.P, 32, 0, s, m, pf, buf);
    PDL(k_pf_offsets, 1, 32, 0, s, m, pf);
    PDL(k_pf_scatter, pf.P, 32, 0, s, m, pf);
    return cudaGetLastError();
}

cudaError_t launch_pf_predict(const DevModel& m, const PrefillDev& pf, int layer, int buf, cudaStream_t s) {
    const int tg = (pf.P + kPT - 1) / kPT;
    PDL(k_pf_quasi, dim3(m.Hp / 32, pf.P), 32, 0, s, m, pf, layer);
    PDL(k_pf_scales, pf.P, 32, 0, s, m, pf, static_cast<const double*>(pf.ssqrd));
    cudaError_t e = launch_gemvn(m, pf, m.Ep / 32, tg, pf.RD, m.moe_gain + static_cast<long long>(layer + 1) * m.H,
                                 m.gate + (layer + 1) * m.gate_stride, m.E, pf.lgp, m.E, s);
    if (e != cudaSuccess) return e;
    PDL(k_pf_decide_pred, pf.P, 32, 0, s, m, pf, buf);
    return cudaGetLastError();
}

cudaError_t launch_pf_experts_dev(const DevModel& m, const PrefillDev& pf, int layer, const PfWave& wv,
                                  int max_chunks, cudaStream_t s, int ep_rank, int ep_world) {
    PDL(k_pf_chunks, 1, 32, 0, s, m, pf, ep_rank, ep_world);
    return launch_pf_experts(m, pf, layer, wv, max_chunks, s, 0);
}

cudaError_t launch_pf_predict_baseline_s(const DevModel& m, const PrefillDev& pf, int layer, int buf,
                                         cudaStream_t s) {
    // BaselineS (speculation.cpp:180-190): gate_{l+1} over s_l = rms_norm(r_l, gain_l)
    const int tg = (pf.P + kPT - 1) / kPT;
    PDL(k_pf_scales, pf.P, 32, 0, s, m, pf, static_cast<const double*>(pf.ssqr));
    cudaError_t e = launch_gemvn(m, pf, m.Ep / 32, tg, pf.R, m.moe_gain + static_cast<long long>(layer) * m.H,
                                 m.gate + (layer + 1) * m.gate_stride, m.E, pf.lgp, m.E, s);
    if (e != cudaSuccess) return e;
    PDL(k_pf_decide_pred, pf.P, 32, 0, s, m, pf, buf);
    return cudaGetLastError();
}

cudaError_t launch_pf_quasi_q(const DevModel& m, const PrefillDev& pf, int layer, float* qn, cudaStream_t s) {
    PDL(k_pf_quasi, dim3(m.Hp / 32, pf.P), 32, 0, s, m, pf, layer);
    PDL(k_pf_scales, pf.P, 32, 0, s, m, pf, static_cast<const double*>(pf.ssqrd));
    PDL(k_pf_normq, dim3(cdiv(m.H, 32), pf.P), 32, 0, s, m, pf, m.moe_gain + static_cast<long long>(layer + 1) * m.H,
        qn);
    return cudaGetLastError();
}

cudaError_t launch_pf_decide_pred(const DevModel& m, const PrefillDev& pf, int buf, cudaStream_t s) {
    PDL(k_pf_decide_pred, pf.P, 32, 0, s, m, pf, buf);
    return cudaGetLastError();
}

cudaError_t launch_pf_final(const DevModel& m, const PrefillDev& pf, cudaStream_t s) {
    const int tg = (pf.P + kPT - 1) / kPT;
    PDL(k_pf_scales, pf.P, 32, 0, s, m, pf, static_cast<const double*>(pf.ssqx));
    cudaError_t e = launch_gemvn(m, pf, m.Vp / 32, tg, pf.X, m.final_gain, m.unemb, m.V, pf.logits, m.V, s);
    if (e != cudaSuccess) return e;
    PDL(k_pf_argmax, pf.P, 32, 0, s, m, pf);
    return cudaGetLastError();
}

template <int T>
cudaError_t launch_pf_experts_t(const DevModel& m, const PrefillDev& pf, int layer, const PfWave& wv, int chunks,
                                cudaStream_t s) {
    const int wh = pf_warps(pf_h_stage(m), m.Hmp / 16, chunks), wd = pf_warps(pf_down_stage(m), m.Hp / 32, chunks);
    PDL(k_pf_gu<T>, dim3(cdiv(m.Hmp / 16, wh), chunks), 32 * wh, pf_smem(pf_h_stage(m), wh), s, m, pf, layer, wv);
    PDL(k_pf_down<T>, dim3(cdiv(m.Hp / 32, wd), chunks), 32 * wd, pf_smem(pf_down_stage(m), wd), s, m, pf, layer,
        wv, pf_down_tpb(m));
    return cudaGetLastError();
}

cudaError_t launch_pf_experts(const DevModel& m, const PrefillDev& pf, int layer, const PfWave& wv,
                              int chunks, cudaStream_t s, int chains) {
    // `chunks` = number of (expert, 8-token chunk) work items in pf.chunk_u / chunk_c;
    // the router's scales (of r_l) are still in pf.scale
    // chains < 8: small batches whose chunks hold 1-8 tokens -> per-chunk dispatch
    if (chains < kPT) return launch_pf_experts_t<0>(m, pf, layer, wv, chunks, s);
    return launch_pf_experts_t<kPT>(m, pf, layer, wv, chunks, s);
}

cudaError_t launch_pf_ep_combine(const DevModel& m, const PrefillDev& pf, const DevEP& ep, int layer, int* error,
                                 long long spin_limit, cudaStream_t s) {
    PDL(k_pf_ep_publish, pf.P * m.K, 128, 0, s, m, pf, ep, layer);
    PDL(k_pf_ep_wait, 1, 32, 0, s, ep, layer, error, spin_limit);
    return cudaGetLastError();
}

cudaError_t launch_pf_mix(const DevModel& m, const PrefillDev& pf, cudaStream_t s) {
    PDL(k_pf_mix, dim3(m.Hp / 32, pf.P), 32, 0, s, m, pf);
    return cudaGetLastError();
}

cudaError_t launch_pf_handoff(const DevModel& m, const DevState& st, const PrefillDev& pf, cudaStream_t s) {
    PDL(k_pf_handoff, m.Hp / 32, 32, 0, s, m, st, pf);
    return cudaGetLastError();
}

}  // namespace smoe
