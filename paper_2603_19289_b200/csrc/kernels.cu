// kernels.cu — sm_100a kernels for the speculative expert-prefetch decode path.
//
// Arithmetic contract: every f32 dot product is the
// reference's sequential `acc += w[c] * x[c]` (numerics.cpp:136-147) with a
// separately rounded product (the file is compiled with --fmad=false; the
// reference's x86-64 build emits no FMA).  One lane owns one output row and
// walks the columns in order; parallelism comes from rows, experts and
// layers, never from splitting a dot product.  Weights stream HBM -> smem
// with cp.async.bulk (TMA bulk copies, SASS UBLKCP) into a per-warp
// multi-stage ring guarded by mbarriers, so the sequential FADD chains run
// at chain latency while the copy engine keeps bytes in flight.
// f64 reductions (rms_norm sum of squares, softmax partition) are
// tree-ordered; their ~1e-16 relative differences vanish in the f32
// rounding of the result except at measure-zero midpoints (reported by the
// parity tests as exact-match fractions).
#include "kernels.h"

#include <atomic>
#include "smoe_chain.cuh"
#include "expf_glibc.cuh"

#ifdef SMOE_KTRACE
// Device-side kernel timeline (instrumented builds only, tools/ktrace_run.py):
// per (kernel kind, layer) the first CTA entry, the first CTA past its PDL
// wait and the last CTA exit, in globaltimer ns, min/max over CTAs.
namespace smoe {

constexpr int kKtKinds = 17, kKtLayers = 128;
__device__ unsigned long long g_kt[kKtKinds * kKtLayers][4];
__device__ __forceinline__ unsigned long long kt_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
struct KTrace {
    int slot;
    __device__ KTrace(int kind, int layer) : slot(kind * kKtLayers + (layer & (kKtLayers - 1))) {
        if (threadIdx.x == 0) {
            const unsigned long long t = kt_now();
            atomicMin(&g_kt[slot][0], t);
            atomicMax(&g_kt[slot][3], t);  // last CTA to start
        }
    }
    __device__ void waited() const {
        if (threadIdx.x == 0) atomicMin(&g_kt[slot][1], kt_now());
    }
    __device__ ~KTrace() {
        if (threadIdx.x == 0) atomicMax(&g_kt[slot][2], kt_now());
    }
};
}  // namespace smoe
extern "C" int smoe_ktrace_reset() {
    static unsigned long long h[smoe::kKtKinds * smoe::kKtLayers][4];
    for (auto& r : h) { r[0] = ~0ull; r[1] = ~0ull; r[2] = 0; r[3] = 0; }
    return cudaMemcpyToSymbol(smoe::g_kt, h, sizeof(h)) == cudaSuccess ? 0 : 1;
}
extern "C" int smoe_ktrace_read(unsigned long long* out) {
    return cudaMemcpyFromSymbol(out, smoe::g_kt, sizeof(smoe::g_kt)) == cudaSuccess ? 0 : 1;
}
#define KTRACE(kind, layer) const KTrace kt_(kind, layer)
#define KT_WAITED() kt_.waited()
#else
#define KTRACE(kind, layer)
#define KT_WAITED()
#endif

#include <cstdio>
#include <string>
#include <cstdlib>

namespace smoe {

// Tolerance-mode code paths are compiled out of the exact-only object the SASS
// guard inspects (Makefile build/kernels_exact.o, tests/test_sass.py): that
// build proves the exact chains carry no fused multiply-add.
#ifdef SMOE_EXACT_ONLY
#define SMOE_FAST(m) false
#else
#define SMOE_FAST(m) ((m).fast != 0)
#endif

// A decode GEMV row chain in the session's arithmetic mode (DevModel::fast).
template <typename Pipe>
__device__ __forceinline__ float chain_run(Pipe& p, const DevModel& m, const uint16_t* tile, int cols,
                                          const float* xs) {
    return SMOE_FAST(m) ? p.run_fast(tile, cols, xs) : p.run(tile, cols, xs);
}




// The decision for `layer` (and its copy request) is complete: release it to
// the expert kernel of `layer`, which may start before its own PDL wait.
__device__ __forceinline__ void publish_decision(const DevState& st, int layer) {
    __threadfence();
    const int p = __ldcg(st.pass_id);
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(st.dec_ready + layer), "r"(p) : "memory");
}

// dst := src for one decision (single thread): every load issued before the
// first store, so the K round trips overlap instead of serialising behind
// the stores.
__device__ __forceinline__ void copy_decision(const int* sid, const float* sg, int* did, float* dg, int k) {
    int iv[kMaxK];
    float gv[kMaxK];
#pragma unroll
    for (int i = 0; i < kMaxK; ++i)
        if (i < k) {
            iv[i] = __ldcg(sid + i);
            gv[i] = __ldcg(sg + i);
        }
#pragma unroll
    for (int i = 0; i < kMaxK; ++i)
        if (i < k) {
            did[i] = iv[i];
            dg[i] = gv[i];
        }
}

// Mailbox post (single thread): request copies of `ids` for `layer`.
//
// Device-side hit path: when every id this rank owns is already resident
// (slot_of >= 0; the copy stream updates slot_of only after the expert's
// bytes landed, and a layer's slots change only while serving a later request
// of the same layer, which the compute order puts after this layer's experts
// ran), the layer is released here (ready = seq) instead of after a host
// round trip; the entry still goes to the host for LRU order and hit counts.
__device__ void post_request(const DevModel& m, const DevCtl& ctl, int layer, int step, const int* ids,
                             int k) {
    const int seq = *ctl.req_counter + 1;
    *ctl.req_counter = seq;
    ctl.req_seq[layer] = seq;
    MailboxEntry* e = ctl.mailbox + (seq % kMailboxRing);
    // all loads first: a load after a store to (possibly aliasing) memory
    // would otherwise wait for it, one L2 round trip per id
    int v[kMaxK], so[kMaxK];
#pragma unroll
    for (int i = 0; i < kMaxK; ++i)
        if (i < k) v[i] = __ldcg(ids + i);
#pragma unroll
    for (int i = 0; i < kMaxK; ++i)
        if (i < k) {
            const bool local = ctl.ep.world == 1 || v[i] % ctl.ep.world == ctl.ep.rank;
            so[i] = local ? __ldcg(m.slot_of + layer * m.E + v[i]) : 0;
        }
    bool all_hit = ctl.fast_hit != 0;
#pragma unroll
    for (int i = 0; i < kMaxK; ++i)
        if (i < k && so[i] < 0) all_hit = false;
    e->layer = layer;
    e->step = step;
    e->nids = k;
    e->flags = all_hit ? kMbAllHit : 0;
#pragma unroll
    for (int i = 0; i < kMaxK; ++i)
        if (i < k) e->ids[i] = v[i];
    __threadfence_system();
    e->seq = seq;
    if (all_hit) {  // ready only grows (the host never writes it for an all-hit entry)
        __threadfence();
        atomicMax(ctl.ready + layer, seq);
    }
}

// ------------------------------------------------------------- weight init --

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Rng::next_gaussian (numerics.cpp:10-14) for draw block n: 12 uniforms from
// the counter-based splitmix64 stream, summed in order in f64, minus 6.
__device__ __forceinline__ double gaussian_at(uint64_t seed, unsigned long long n) {
    double s = 0.0;
    uint64_t st = seed + (12ull * n) * 0x9E3779B97F4A7C15ull;
#pragma unroll
    for (int j = 0; j < 12; ++j) {
        st += 0x9E3779B97F4A7C15ull;
        s = __dadd_rn(s, __dmul_rn(__ull2double_rn(mix64(st) >> 11), 0x1.0p-53));
    }
    return __dadd_rn(s, -6.0);
}

__device__ __forceinline__ uint16_t f2bf_rne(float x) {
    uint32_t u = __float_as_uint(x);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

// Thread per destination element (coalesced writes).  Row-tiled layouts
// cover rows [0, Rtile) x tile_cols; elements outside the tensor are left.
__global__ void k_gen_bf16(uint64_t seed, double stddev, int R, int C, int tile_cols,
                           int layout, int which, int row_off, long long total, uint16_t* out) {
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long d = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; d < total;
         d += stride) {
        long long r, c;
        if (layout == kRowMajor) {
            r = d / C;
            c = d % C;
        } else {
            const long long tile = static_cast<long long>(tile_cols) * 32;
            const long long rb = d / tile, rem = d % tile;
            const long long lane = (rem % 256) / 8;
            c = (rem / 256) * 8 + (rem % 8);
            if (c >= C) continue;
            const long long vr = rb * 32 + lane;
            if (layout == kRowTiled) {
                r = vr - row_off;
            } else {  // kGateUp: virtual row 2r + which
                if ((vr & 1) != which) continue;
                r = vr >> 1;
            }
            if (r < 0 || r >= R) continue;
        }
        const double g = gaussian_at(seed, static_cast<unsigned long long>(r * C + c));
        out[d] = f2bf_rne(static_cast<float>(__dmul_rn(g, stddev)));
    }
}

// ------------------------------------------------------------- attention --

__global__ void k_embed(DevModel m, DevState st, const int* token_src, const int* stream,
                        const int* step) {
    KTRACE(0, 0);
    pdl_wait();
    KT_WAITED();
    pdl_trigger();  // after our own dependency: dependents launch at most one kernel ahead
    const int tok = stream ? stream[*step] : *token_src;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *st.token = tok;
        *st.tok_in = tok;
        *st.pass_id = *st.pass_id + 1;  // read by later kernels of this pass only
    }
    const int j = blockIdx.x * 32 + threadIdx.x;  // grid Hp/32 x 32
    const float v = j < m.H ? bf2f(m.emb[static_cast<long long>(tok) * m.H + j]) : 0.0f;
    st.x[j] = v;
    warp_ssq_partial(v, st.ssq_x + blockIdx.x);  // layer 0's input
}

// q, k, v = W{q,k,v} . rms_norm(x, attn_gain) (model.cpp:325-333), RoPE on q
// and k (model.cpp:309-321, cos/sin precomputed on the host with libm), k and v
// appended to the layer's KV cache at `pos`.  One warp per 32-row tile.
__global__ void __launch_bounds__(32 * kSplitWarps) k_qkv(DevModel m, DevState st, int layer) {
    KTRACE(1, layer);
    PHASE_DECL
    PHASE();
    uint64_t* bar = reinterpret_cast<uint64_t*>(g_smem);
    double* red = reinterpret_cast<double*>(g_smem + 64);
    float* xs = reinterpret_cast<float*>(g_smem + 128);
    float* gs = xs + round_up(m.H, 32);
    unsigned char* pipe_mem = align128(reinterpret_cast<unsigned char*>(gs + round_up(m.H, 32)));
    const int rb = blockIdx.x;
    const uint16_t* tile = m.wqkv + layer * m.qkv_stride + static_cast<long long>(rb) * m.H * 32;
    // exact: one warp, the tile's sequential chains; fast: kSplitWarps warps
    // split the columns (SplitLdg), weights loaded into registers right here
    PipeBL pipe;
    SplitG sp;
    if (SMOE_FAST(m)) {
        sp.prime(tile, m.H);
    } else {
        pipe.init(pipe_mem);
        pipe.prime(tile, m.H);
    }
    Stager sg;
    sg.init(bar);
    sg.add(gs, m.attn_gain + static_cast<long long>(layer) * m.H, m.H * 4);  // static: before the PDL wait
    pdl_wait();
    KT_WAITED();
    pdl_trigger();  // after our own dependency: dependents launch at most one kernel ahead
    sg.add(xs, st.x, m.H * 4);
    // the epilogue's position and RoPE factors load while the chain runs
    const int lane = threadIdx.x & 31;
    const int R = rb * 32 + lane;
    const int D = m.D;
    const int pos = *st.pos;
    float c = 1.0f, s = 0.0f;
    if (R < 2 * D) {
        const int i = (R % D) >> 1;
        c = m.rope[(static_cast<long long>(pos) * (D / 2) + i) * 2];
        s = m.rope[(static_cast<long long>(pos) * (D / 2) + i) * 2 + 1];
    }
    PHASE();
    const float scale = rms_scale_from_partials(st.ssq_x + static_cast<long long>(layer) * (m.Hp / 32),
                                                m.Hp / 32, m.H, m.eps);
    sg.wait();
    PHASE();
    block_apply_norm(xs, gs, m.H, scale, xs);
    PHASE();
    float acc = SMOE_FAST(m) ? sp.run(tile, m.H, xs, reinterpret_cast<float*>(pipe_mem)) : pipe.run(tile, m.H, xs);
    if (threadIdx.x >= 32) return;  // fast mode: warp 0 holds the rows
    PHASE();
    const float other = __shfl_xor_sync(0xffffffffu, acc, 1);
    if (R < 2 * D) {  // RoPE pair (2i, 2i+1) lives in lanes (2i', 2i'+1)
        const bool even = (R & 1) == 0;
        const float x0 = even ? acc : other, x1 = even ? other : acc;
        acc = even ? (x0 * c - x1 * s) : (x0 * s + x1 * c);
    }
    const long long kv = (static_cast<long long>(layer) * m.cap + pos) * D;
    if (R < D)
        st.q[R] = acc;
    else if (R < 2 * D)
        st.kc[kv + R - D] = acc;
    else if (R < 3 * D)
        st.vc[kv + R - 2 * D] = acc;
    PHASE();
    PHASE_DUMP("qkv [pre, stage, norm, chain, epi]");
#ifdef SMOE_PHASES
    if (blockIdx.x == 0 && threadIdx.x == 0) printf("qkv chain waits (cycles): %lld\n", pipe.wait_cyc);
#endif
}

// scores / softmax / context (model.cpp:335-351), one CTA of kAttnThreads.
// Keys, then values, stream through 2-chunk rings of kAttnChunk positions,
// copied global -> smem with cp.async (16 B per thread, L2 only).  Key rows
// are padded to D+4 floats so that thread j's LDS.128 of its own row is
// bank-conflict-free (8 rows per phase cover all 32 banks); thread j owns
// position j's dot product (sequential over head dims), thread i owns
// context dim i (sequential over positions).  Rows of earlier positions are
// final before this step, so the first chunks are fetched BEFORE the PDL
// wait; only row `pos` (written by k_qkv of this step) and q wait for it.
constexpr int kAttnChunk = 64;
constexpr int kAttnThreads = 256;
constexpr int kAttnSmemPositions = 4096;

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// rows [p0, p0+pn) of a [cap][D] f32 cache into smem rows of `stride` floats;
// row `skip` (the current position, not yet written) is left out.
__device__ __forceinline__ void attn_fetch(float* dst, const float* src, int p0, int pn, int D,
                                           int stride, int skip) {
    const int per = D / 4;  // 16-byte pieces per row
    for (int t = threadIdx.x; t < pn * per; t += blockDim.x) {
        const int r = t / per, c = (t % per) * 4;
        if (p0 + r == skip) continue;
        cp_async16(dst + r * stride + c, src + static_cast<long long>(p0 + r) * D + c);
    }
}

__device__ __forceinline__ void attn_single(const DevModel& m, const DevState& st, double* scratch, int layer) {
    const int D = m.D, KS = D + 4;  // padded key row stride (floats)
    float* red = reinterpret_cast<float*>(g_smem);                     // [32]
    float* qs = reinterpret_cast<float*>(g_smem + 256);                // [kMaxD]
    float* kt = qs + kMaxD;                                            // [2][chunk][D+4]
    float* vt = kt + 2 * kAttnChunk * KS;                              // [2][chunk][D]
    double* e = reinterpret_cast<double*>(vt + 2 * kAttnChunk * D);    // [n] (smem when it fits)
    float* sc = reinterpret_cast<float*>(e + m.cap);
    if (m.cap > kAttnSmemPositions) {  // long contexts: f64/f32 scratch in global
        e = scratch;
        sc = reinterpret_cast<float*>(scratch + m.cap);
    }
    const long long base = static_cast<long long>(layer) * m.cap * D;
    const float* K = st.kc + base;
    const float* V = st.vc + base;
    // st.pos is only advanced by k_final, which completed before this grid could launch
    const int pos = __ldcg(st.pos);
    const int n = pos + 1;
    const int nch = (n + kAttnChunk - 1) / kAttnChunk;
    auto fetch_k = [&](int c, int skip) {
        attn_fetch(kt + (c & 1) * kAttnChunk * KS, K, c * kAttnChunk, min(kAttnChunk, n - c * kAttnChunk), D,
                   KS, skip);
    };
    auto fetch_v = [&](int c, int skip) {
        attn_fetch(vt + (c & 1) * kAttnChunk * D, V, c * kAttnChunk, min(kAttnChunk, n - c * kAttnChunk), D, D,
                   skip);
    };
    // prefetch (groups 0, 1): K chunks 0-1 and, for short contexts, V chunks 0-1
    fetch_k(0, pos);
    if (nch > 1) fetch_k(1, pos);
    cp_async_commit();
    const bool v_early = nch <= 2;
    if (v_early) {
        fetch_v(0, pos);
        if (nch > 1) fetch_v(1, pos);
    }
    cp_async_commit();
    pdl_wait();
    pdl_trigger();  // after our own dependency: dependents launch at most one kernel ahead
    // q and the current position's key/value row (written by k_qkv)
    for (int t = threadIdx.x; t < D / 4; t += blockDim.x) {
        cp_async16(qs + 4 * t, st.q + 4 * t);
        const int c = pos / kAttnChunk, r = pos % kAttnChunk;
        if (c < 2) {
            cp_async16(kt + (c & 1) * kAttnChunk * KS + r * KS + 4 * t, K + static_cast<long long>(pos) * D + 4 * t);
            if (v_early)
                cp_async16(vt + (c & 1) * kAttnChunk * D + r * D + 4 * t, V + static_cast<long long>(pos) * D + 4 * t);
        }
    }
    cp_async_commit();
    // pass 1: scores
    float lmax = -INFINITY;
    // chunk c + 2 is fetched into chunk c's slot as soon as c is consumed, so
    // one chunk load is always in flight behind the one being scored
    for (int c = 0; c < nch; ++c) {
        if (c >= 1 && c + 1 < nch)
            cp_async_wait<1>();  // chunk c landed; chunk c + 1's group may still be pending
        else
            cp_async_wait<0>();
        __syncthreads();
        const float* t = kt + (c & 1) * kAttnChunk * KS;
        const int p0 = c * kAttnChunk;
        const int pn = min(kAttnChunk, n - p0);
        for (int j = threadIdx.x; j < pn; j += blockDim.x) {
            const float* kj = t + j * KS;
            float acc = 0.0f;
            for (int i = 0; i < D; i += 4) {
                const float4 kv = *reinterpret_cast<const float4*>(kj + i);
                const float4 qv = *reinterpret_cast<const float4*>(qs + i);
                acc = acc + qv.x * kv.x;
                acc = acc + qv.y * kv.y;
                acc = acc + qv.z * kv.z;
                acc = acc + qv.w * kv.w;
            }
            const float v = acc * m.inv_sqrt_d;
            sc[p0 + j] = v;
            lmax = fmaxf(lmax, v);
        }
        __syncthreads();  // the ring slot is refilled now
        if (c + 2 < nch) {  // (row pos included: the chunk loads after the PDL wait)
            fetch_k(c + 2, -1);
            cp_async_commit();
        }
    }
    if (!v_early) {  // stream values: first two chunks now, the rest in pass 2
        fetch_v(0, -1);
        if (nch > 1) fetch_v(1, -1);
        cp_async_commit();
    }
    const float mx = block_max_f(lmax, red);
    for (int j = threadIdx.x; j < n; j += blockDim.x)
        e[j] = exp_glibc(static_cast<double>(sc[j]) - static_cast<double>(mx));
    __syncthreads();
    __shared__ double zs;
    if (threadIdx.x == 0) {  // f64 partition in index order, as numerics.cpp:46-49
        double z = 0.0;
        for (int j = 0; j < n; ++j) z += e[j];
        zs = z;
    }
    __syncthreads();
    const double z = zs;
    for (int j = threadIdx.x; j < n; j += blockDim.x) sc[j] = static_cast<float>(e[j] / z);
    __syncthreads();
    float acc = 0.0f;
    const int i = threadIdx.x;
    for (int c = 0; c < nch; ++c) {
        if (c >= 1 && c + 1 < nch)
            cp_async_wait<1>();
        else
            cp_async_wait<0>();
        __syncthreads();
        const float* t = vt + (c & 1) * kAttnChunk * D;
        const int p0 = c * kAttnChunk;
        const int pn = min(kAttnChunk, n - p0);
        if (i < D)
            for (int j = 0; j < pn; ++j) acc = acc + sc[p0 + j] * t[j * D + i];
        __syncthreads();
        if (c + 2 < nch) {
            fetch_v(c + 2, -1);
            cp_async_commit();
        }
    }
    if (i < D) st.ctx[i] = acc;
}

// Long contexts (more than kAttnSplitMin positions): kAttnSplit CTAs share the
// work with the same arithmetic as attn_single.  Each CTA scores its slice of
// positions (one sequential chain per position), the last CTA to arrive forms
// the softmax (max is order-free; the f64 partition is one sequential chain in
// index order, numerics.cpp:46-49) and publishes the probabilities; then each
// CTA produces its slice of the D context outputs (one sequential chain over
// the positions per output).  All kAttnSplit CTAs are co-resident, so waiting
// on the last one is safe.  Scratch: e [cap] f64 | p [cap] f32 | ctl | maxes.
// the dynamic shared memory k_attn is launched with (attn_smem on the host)
__device__ __forceinline__ size_t attn_smem_bytes(const DevModel& m) {
    size_t bts = 256 + kMaxD * 4 + 2ull * kAttnChunk * (2 * m.D + 4) * 4;
    if (m.cap <= kAttnSmemPositions) bts += static_cast<size_t>(m.cap) * 12;
    return bts;
}

constexpr int kAttnSplit = 16;
constexpr int kAttnSplitMin = 512;

__global__ void __launch_bounds__(kAttnThreads) k_attn(DevModel m, DevState st, double* scratch, int layer) {
    KTRACE(2, layer);
    // st.pos is only advanced by k_final, which completed before this grid could launch
    const int n = __ldcg(st.pos) + 1;
    if (n <= kAttnSplitMin || gridDim.x == 1) {
        if (blockIdx.x == 0) attn_single(m, st, scratch, layer);
        return;
    }
    const int D = m.D, G = gridDim.x, b = blockIdx.x;
    PHASE_DECL
    PHASE();
    float* red = reinterpret_cast<float*>(g_smem);       // [32]
    float* qs = reinterpret_cast<float*>(g_smem + 256);  // [kMaxD]
    double* eg = scratch;
    float* pg = reinterpret_cast<float*>(scratch + m.cap);
    int* ctl = reinterpret_cast<int*>(pg + m.cap);       // [0] arrivals, [1] published generation
    float* mxs = reinterpret_cast<float*>(ctl + 32);     // [G] per-CTA maxima
    const long long base = static_cast<long long>(layer) * m.cap * D;
    const float* K = st.kc + base;
    const float* V = st.vc + base;
    pdl_wait();
    KT_WAITED();
    pdl_trigger();
    for (int t = threadIdx.x; t < D; t += blockDim.x) qs[t] = __ldcg(st.q + t);
    __syncthreads();
    const int per = (n + G - 1) / G, j0 = b * per, j1 = min(n, j0 + per);
    float lmax = -INFINITY;
    for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
        const float4* kj = reinterpret_cast<const float4*>(K + static_cast<long long>(j) * D);
        float acc = 0.0f;
#pragma unroll 8
        for (int i = 0; i < D / 4; ++i) {
            const float4 kv = __ldcg(kj + i);
            acc = acc + qs[4 * i] * kv.x;
            acc = acc + qs[4 * i + 1] * kv.y;
            acc = acc + qs[4 * i + 2] * kv.z;
            acc = acc + qs[4 * i + 3] * kv.w;
        }
        const float v = acc * m.inv_sqrt_d;
        pg[j] = v;  // scores; replaced by probabilities below
        lmax = fmaxf(lmax, v);
    }
    const float mb = block_max_f(lmax, red);
    PHASE();
    __shared__ int s_gen, s_last;
    __shared__ double zs;
    if (threadIdx.x == 0) {
        mxs[b] = mb;
        __threadfence();
        const int old = atomicAdd(ctl, 1);
        s_gen = old / G;
        s_last = (old % G) == G - 1;
    }
    __syncthreads();
    const int gen = s_gen;
    // staging area behind q: the exponentials (last CTA), then p and V slices
    unsigned char* stage = g_smem + 256 + kMaxD * 4;
    const int cap_s = static_cast<int>((attn_smem_bytes(m) - 256 - kMaxD * 4) / 8);  // f64 slots
    if (s_last) {
        __threadfence();
        float mx = -INFINITY;
        for (int k = 0; k < G; ++k) mx = fmaxf(mx, __ldcg(mxs + k));
        double* es = n <= cap_s ? reinterpret_cast<double*>(stage) : eg;
        for (int j = threadIdx.x; j < n; j += blockDim.x)
            es[j] = exp_glibc(static_cast<double>(__ldcg(pg + j)) - static_cast<double>(mx));
        __syncthreads();
        PHASE();
        if (threadIdx.x == 0) {  // f64 partition in index order, as numerics.cpp:46-49
            double z = 0.0;
            int j = 0;
            for (; j + 32 <= n; j += 32) {  // loads of a block in flight together, adds in order
                double ev[32];
#pragma unroll
                for (int u = 0; u < 32; ++u) ev[u] = es[j + u];
#pragma unroll
                for (int u = 0; u < 32; ++u) z += ev[u];
            }
            for (; j < n; ++j) z += es[j];
            zs = z;
        }
        __syncthreads();
        PHASE();
        for (int j = threadIdx.x; j < n; j += blockDim.x) pg[j] = static_cast<float>(es[j] / zs);
        __syncthreads();
        PHASE();
        if (threadIdx.x == 0) {
            __threadfence();
            asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(ctl + 1), "r"(gen + 1) : "memory");
        }
    }
    // bounded like every other device wait: the attn_grid CTAs are co-resident
    // by construction (occupancy checked at session creation), and a stall
    // here (e.g. an SM-limited context) is reported instead of hanging
    __shared__ int s_abort;
    if (threadIdx.x == 0) {
        s_abort = 0;
        const long long t0 = clock64();
        while (ld_acquire(ctl + 1) < gen + 1) {
            if (*(volatile int*)m.attn_err) {
                s_abort = 1;
                break;
            }
            if (clock64() - t0 > m.attn_spin) {
                atomicCAS(m.attn_err, 0, 4000 + layer);
                s_abort = 1;
                break;
            }
            __nanosleep(32);
        }
    }
    __syncthreads();
    if (s_abort) return;
    PHASE();
    // context slice: outputs [i0, i0 + ipc), p and V[:, slice] staged in chunks
    // of positions, one sequential chain per output over all positions
    const int ipc = (D + G - 1) / G, i0 = b * ipc, ni = max(0, min(ipc, D - i0));
    float* ps = reinterpret_cast<float*>(stage);
    const int chunk = max(32, min(n, static_cast<int>(cap_s * 8 / (4 * (1 + ipc)))) / 32 * 32);
    float* vs = ps + chunk;
    float acc = 0.0f;
    for (int c0 = 0; c0 < n; c0 += chunk) {
        const int cn = min(chunk, n - c0);
        if (c0) __syncthreads();
        if ((ipc & 3) == 0 && ni == ipc && (reinterpret_cast<uintptr_t>(pg + c0) & 15) == 0) {  // cp.async
            const int q4 = ipc >> 2;                           // float4 per row slice
            for (int x = threadIdx.x; x < (cn + 3) / 4; x += blockDim.x)
                if (4 * x + 3 < cn)
                    cp_async16(ps + 4 * x, pg + c0 + 4 * x);
                else
                    for (int j = 4 * x; j < cn; ++j) ps[j] = __ldcg(pg + c0 + j);
            for (int x = threadIdx.x; x < cn * q4; x += blockDim.x) {
                const int j = x / q4, k = x % q4;
                cp_async16(vs + j * ipc + 4 * k, V + static_cast<long long>(c0 + j) * D + i0 + 4 * k);
            }
            cp_async_commit();
            cp_async_wait<0>();
        } else {
            for (int j = threadIdx.x; j < cn; j += blockDim.x) ps[j] = __ldcg(pg + c0 + j);
            for (int x = threadIdx.x; x < cn * ni; x += blockDim.x) {
                const int j = x / ni, k = x % ni;
                vs[j * ipc + k] = __ldcg(V + static_cast<long long>(c0 + j) * D + i0 + k);
            }
        }
        __syncthreads();
        if (threadIdx.x < ni) {
            int j = 0;
            for (; j + 8 <= cn; j += 8) {  // operands of a block loaded together, chain in order
                float pv[8], vv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    pv[u] = ps[j + u];
                    vv[u] = vs[(j + u) * ipc + threadIdx.x];
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) acc = acc + pv[u] * vv[u];
            }
            for (; j < cn; ++j) acc = acc + ps[j] * vs[j * ipc + threadIdx.x];
        }
    }
    if (threadIdx.x < ni) st.ctx[i0 + threadIdx.x] = acc;
    PHASE();
#ifdef SMOE_PHASES
    if (threadIdx.x == 0 && (b == 0 || s_last))
        phase_print(s_last ? "attn split LAST [start, scores, exps, z, p, flag, context]"
                           : "attn split cta0 [start, scores, flag wait, context]", ph_, nph_);
#endif
}

// Tolerance-mode decode attention (DevModel::fast): split-K "flash decoding".
// The positions are sliced over the CTAs that have any (grid sized for the KV
// capacity, up to kAttnFastCtas; at least kAttnFastChunk positions each).  A
// CTA streams its K and V rows through a 2-chunk cp.async ring in shared
// memory (rows before `pos` are final, so the first chunks are requested
// before the PDL wait), thread j scores position j of a chunk (q . k_j, four
// f32 partial sums), and the CTA keeps an online softmax: running max m, sum
// l and context acc (thread i owns dim i), rescaled by exp(m_old - m) per
// chunk.  CTAs publish (m, l, acc[D]); the last to arrive merges them in CTA
// order, normalises and writes ctx.  Same math as softmax + context
// (model.cpp:337-351) up to f32 rounding (f32 exp, no sequential f64
// partition): a 16 k-token context streams its 16 MB of K/V per layer at HBM
// rate instead of one f64 chain over all positions.
constexpr int kAttnFastThreads = 128;  // >= head_dim (thread i owns context dim i)
constexpr int kAttnFastChunk = 32;     // positions per ring slot (66 KB of ring at head_dim 128: 3 CTAs per SM)
constexpr int kAttnFastCtas = 296;     // 2 per SM
__device__ __forceinline__ float* attn_fast_scratch(const DevModel& m, double* scratch) {
    return reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(scratch) + 16ull * m.cap + 1024);
}
bool attn_fast_ok(const DevModel& m) { return SMOE_FAST(m) && m.D % 4 == 0 && m.D <= kAttnFastThreads; }
size_t attn_fast_smem(const DevModel& m) { return 2ull * kAttnFastChunk * (2 * m.D + 4) * 4; }
constexpr int kAttnGroup = 32;  // flash-decoding merge: partials per first-level group (one 32-load batch)
constexpr int kAttnGroups = (kAttnFastCtas + kAttnGroup - 1) / kAttnGroup;
size_t attn_scratch_bytes(int cap) {
    // e/p | CTA partials [kAttnFastCtas][kMaxD+2] | counters (64 B) | group partials | group counters
    return 16ull * cap + 1024 + static_cast<size_t>(kAttnFastCtas) * (kMaxD + 2) * 4 + 64 +
           static_cast<size_t>(kAttnGroups) * (kMaxD + 2) * 4 + 4 * (kAttnGroups + 1) + 64;
}

// Merge n online-softmax partials (m_q, l_q, acc_q[D]) at src (stride
// kMaxD + 2): M = max m_q, f_q = exp(m_q - M), L = sum f_q l_q (fixed-order
// block tree), acc = sum_q f_q acc_q (thread i: dim i, 32 loads in flight).
// Every step is parallel over the partials; the order is fixed, so the
// result is deterministic.  Whole block; returns M and L in every thread and
// acc in threads < D.
__device__ __forceinline__ void attn_merge(const float* src, int n, int D, float* fq, float* lq, float* red,
                                           float& M, float& L, float& acc) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = blockDim.x >> 5;
    float mx = -INFINITY;
    for (int q = tid; q < n; q += blockDim.x) {
        const float* pq = src + static_cast<long long>(q) * (kMaxD + 2);
        const float mq = __ldcg(pq);
        fq[q] = mq;
        lq[q] = __ldcg(pq + 1);
        mx = fmaxf(mx, mq);
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) red[w] = mx;
    __syncthreads();
    M = red[0];
    for (int q = 1; q < nw; ++q) M = fmaxf(M, red[q]);
    __syncthreads();  // red reused below
    float lt = 0.0f;
    for (int q = tid; q < n; q += blockDim.x) {
        const float f = __expf(fq[q] - M);
        fq[q] = f;
        lt = fmaf(f, lq[q], lt);
    }
    for (int o = 16; o > 0; o >>= 1) lt += __shfl_xor_sync(0xffffffffu, lt, o);
    if (lane == 0) red[w] = lt;
    __syncthreads();  // fq complete, red holds the warp sums
    L = 0.0f;
    for (int q = 0; q < nw; ++q) L += red[q];
    float a = 0.0f;
    if (tid < D) {
        constexpr int kB = 32;
        int q = 0;
        for (; q + kB <= n; q += kB) {
            float v[kB];
#pragma unroll
            for (int u = 0; u < kB; ++u) v[u] = __ldcg(src + static_cast<long long>(q + u) * (kMaxD + 2) + 2 + tid);
#pragma unroll
            for (int u = 0; u < kB; ++u) a = fmaf(fq[q + u], v[u], a);
        }
        for (; q < n; ++q) a = fmaf(fq[q], __ldcg(src + static_cast<long long>(q) * (kMaxD + 2) + 2 + tid), a);
    }
    acc = a;
    __syncthreads();  // fq / lq / red free
}

__global__ void __launch_bounds__(kAttnFastThreads) k_attn_fast(DevModel m, DevState st, double* scratch,
                                                                int layer) {
    KTRACE(2, layer);
    const int D = m.D, KS = D + 4;  // padded key rows: thread j's LDS.128 of row j is conflict-free
    __shared__ __align__(16) float qs[kAttnFastThreads];
    __shared__ float red[kAttnFastThreads / 32];
    __shared__ int s_last;
    float* kt = reinterpret_cast<float*>(g_smem);  // [2][chunk][D+4]
    float* vt = kt + 2 * kAttnFastChunk * KS;      // [2][chunk][D]
    __shared__ float ps[2 * kAttnFastChunk];
    const long long base = static_cast<long long>(layer) * m.cap * D;
    const float* K = st.kc + base;
    const float* V = st.vc + base;
    float* part = attn_fast_scratch(m, scratch);  // [G][kMaxD + 2]: m, l, acc
    int* cnt = reinterpret_cast<int*>(part + kAttnFastCtas * (kMaxD + 2));
    // st.pos is only advanced by k_final, which completed before this grid could launch
    const int pos = __ldcg(st.pos), n = pos + 1, b = blockIdx.x;
    const int ppc = max(2 * kAttnFastChunk, (n + gridDim.x - 1) / gridDim.x);  // both chunks in the ring
    const int G = (n + ppc - 1) / ppc;  // CTAs with positions
    if (b >= G) {  // no positions: leave at once (an exit counts as the PDL trigger)
#ifdef SMOE_ATTN_IDLE_WAIT
        pdl_wait();
        pdl_trigger();
#endif
        return;
    }
    // a slice of <= 2 chunks (every CTA up to ~19 k positions, and the one
    // CTA of a short context) is one pass over both ring slots as a single
    // 64-position chunk: one softmax round instead of two
    const int j0 = b * ppc, j1 = min(n, j0 + ppc);
    const int CH = j1 - j0 <= 2 * kAttnFastChunk ? 2 * kAttnFastChunk : kAttnFastChunk;
    const int nch = (j1 - j0 + CH - 1) / CH;
    auto fetch = [&](int c, int skip) {
        const int p0 = j0 + c * CH, pn = min(CH, j1 - p0);
        float* kd = kt + (c & 1) * CH * KS;
        float* vd = vt + (c & 1) * CH * D;
        const int per = D / 4;
        for (int t = threadIdx.x; t < pn * per; t += blockDim.x) {
            const int r = t / per, q4 = (t % per) * 4;
            if (p0 + r == skip) continue;
            cp_async16(kd + r * KS + q4, K + static_cast<long long>(p0 + r) * D + q4);
            cp_async16(vd + r * D + q4, V + static_cast<long long>(p0 + r) * D + q4);
        }
    };
    fetch(0, pos);  // rows before pos are final: requested before the PDL wait
    cp_async_commit();
    if (nch > 1) fetch(1, pos);
    cp_async_commit();
    pdl_wait();  // q and row pos come from k_qkv
    KT_WAITED();
    pdl_trigger();
    for (int t = threadIdx.x; t < D / 4; t += blockDim.x) {
        cp_async16(qs + 4 * t, st.q + 4 * t);
        const int c = (pos - j0) / CH, r = (pos - j0) % CH;
        if (pos >= j0 && pos < j1 && c < 2) {
            cp_async16(kt + (c & 1) * CH * KS + r * KS + 4 * t, K + static_cast<long long>(pos) * D + 4 * t);
            cp_async16(vt + (c & 1) * CH * D + r * D + 4 * t, V + static_cast<long long>(pos) * D + 4 * t);
        }
    }
    cp_async_commit();
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = blockDim.x >> 5;
    float mrun = -INFINITY, lrun = 0.0f, acc = 0.0f;
    for (int c = 0; c < nch; ++c) {
        if (c >= 1 && c + 1 < nch)
            cp_async_wait<1>();  // chunk c landed; chunk c + 1 may still be in flight
        else
            cp_async_wait<0>();  // (c = 0: q and row pos too)
        __syncthreads();
        const int p0 = j0 + c * CH, pn = min(CH, j1 - p0);
        const float* kc = kt + (c & 1) * CH * KS;
        const float* vc = vt + (c & 1) * CH * D;
        float sj = -INFINITY;
        if (tid < pn) {
            const float* kj = kc + tid * KS;
            float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll 8
            for (int i = 0; i < D; i += 4) {
                const float4 kv = *reinterpret_cast<const float4*>(kj + i);
                const float4 qv = *reinterpret_cast<const float4*>(qs + i);
                a0 = fmaf(qv.x, kv.x, a0);
                a1 = fmaf(qv.y, kv.y, a1);
                a2 = fmaf(qv.z, kv.z, a2);
                a3 = fmaf(qv.w, kv.w, a3);
            }
            sj = ((a0 + a1) + (a2 + a3)) * m.inv_sqrt_d;
        }
        float cm = sj;
        for (int o = 16; o > 0; o >>= 1) cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, o));
        if (lane == 0) red[w] = cm;
        __syncthreads();
        cm = red[0];
        for (int q = 1; q < nw; ++q) cm = fmaxf(cm, red[q]);
        const float mn = fmaxf(mrun, cm);
        const float sc = __expf(mrun - mn);  // 0 on the first chunk
        const float p = tid < pn ? __expf(sj - mn) : 0.0f;
        if (tid < CH) ps[tid] = p;
        float cs = p;
        for (int o = 16; o > 0; o >>= 1) cs += __shfl_xor_sync(0xffffffffu, cs, o);
        __syncthreads();  // red (max) read by all; ps complete
        if (lane == 0) red[w] = cs;
        __syncthreads();
        float csum = 0.0f;
        for (int q = 0; q < nw; ++q) csum += red[q];
        lrun = lrun * sc + csum;
        mrun = mn;
        if (tid < D) {
            float a = acc * sc;
            for (int j = 0; j < pn; ++j) a = fmaf(ps[j], vc[j * D + tid], a);
            acc = a;
        }
        __syncthreads();  // ring slot and ps free
        if (c + 2 < nch) {
            fetch(c + 2, -1);
            cp_async_commit();
        }
    }
    if (G == 1) {  // one CTA holds every position: no merge
        if (tid < D) st.ctx[tid] = acc / lrun;
        return;
    }
    // two-level merge: the last CTA of each group of kAttnGroup (32) merges the
    // group's partials into a group partial, the last group merges those
    // (a single last-arriver merging every CTA serially bounded long contexts)
    float* pb = part + static_cast<long long>(b) * (kMaxD + 2);
    if (tid == 0) {
        pb[0] = mrun;
        pb[1] = lrun;
    }
    if (tid < D) pb[2 + tid] = acc;
    float* gpart = reinterpret_cast<float*>(cnt + 16);  // [kAttnGroups][kMaxD+2]
    int* gcnt = reinterpret_cast<int*>(gpart + kAttnGroups * (kMaxD + 2));  // [kAttnGroups + 1]
    const int g = b / kAttnGroup, ng = (G + kAttnGroup - 1) / kAttnGroup;
    const int gsize = min(kAttnGroup, G - g * kAttnGroup);
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        s_last = atomicAdd(gcnt + g, 1) == gsize - 1;
        if (s_last) gcnt[g] = 0;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    __shared__ float fq[kAttnFastCtas];
    __shared__ float lq[kAttnFastCtas];
    float M, Lt, a;
    attn_merge(part + static_cast<long long>(g) * kAttnGroup * (kMaxD + 2), gsize, D, fq, lq, red, M, Lt, a);
    if (ng == 1) {
        if (tid < D) st.ctx[tid] = a / Lt;
        return;
    }
    float* gp = gpart + static_cast<long long>(g) * (kMaxD + 2);
    if (tid == 0) {
        gp[0] = M;
        gp[1] = Lt;
    }
    if (tid < D) gp[2 + tid] = a;
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        s_last = atomicAdd(gcnt + kAttnGroups, 1) == ng - 1;
        if (s_last) gcnt[kAttnGroups] = 0;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    attn_merge(gpart, ng, D, fq, lq, red, M, Lt, a);
    if (tid < D) st.ctx[tid] = a / Lt;
}

// attn_out = wo . ctx; r = x + attn_out (model.cpp:352, 380).
// SMOE_DOWN_L2=1: k_ffn_gu warms L2 with the down-projection blocks (measured
// neutral on Q30: down gets faster, gate/up slower by as much)
__device__ int g_down_l2_dev = 0;
__device__ int g_fused_l2_dev = 1;  // fused k_ffn: L2 prefetch of the down block (SMOE_FUSED_NO_L2PF=1: off)

// Wait (thread 0) until the predictor of layer-1 published this layer's
// decision for the current pass (publish_decision).
__device__ __forceinline__ void wait_decision(const DevState& st, const DevCtl& ctl, int layer) {
    if (threadIdx.x == 0) {
        const int want = __ldcg(st.pass_id);
        const long long t0 = clock64();
        for (;;) {
            int v;
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(st.dec_ready + layer) : "memory");
            if (v == want) break;
            if (*(volatile int*)ctl.error) break;
            if (clock64() - t0 > ctl.spin_limit) {
                atomicCAS(ctl.error, 0, 1000 + layer);
                break;
            }
            __nanosleep(64);
        }
    }
    __syncwarp();
}

// layer_default (speculation.cpp:104-117) for row j of a decision of K
// experts: d_j = sum_i g_i * D[layer][e_i][j] in decision order (f32).  The K
// loads (one coalesced 128-byte line per warp and expert) are all in flight.
__device__ __forceinline__ float layer_default_row(const DevModel& m, const int* ids, const float* gts,
                                                   int layer, int j) {
    float dv[kMaxK], gv[kMaxK];
#pragma unroll
    for (int i = 0; i < kMaxK; ++i) {
        if (i < m.K) {
            const int e = __ldcg(ids + i);
            gv[i] = __ldcg(gts + i);
            dv[i] = __ldcg(m.dv + (static_cast<long long>(layer) * m.E + e) * m.H + j);
        }
    }
    float d = 0.0f;
#pragma unroll
    for (int i = 0; i < kMaxK; ++i)
        if (i < m.K) d = d + gv[i] * dv[i];
    return d;
}

__global__ void __launch_bounds__(32) k_wo(DevModel m, DevState st, DevCtl ctl, int layer,
                                           int rd_from_pred) {
    KTRACE(3, layer);
    uint64_t* bar = reinterpret_cast<uint64_t*>(g_smem);
    float* xs = reinterpret_cast<float*>(g_smem + 128);
    float* xr = xs + kMaxD;  // residual rows of this tile
    unsigned char* pipe_mem = align128(reinterpret_cast<unsigned char*>(xr + 32));
    PipeB pipe;
    pipe.init(pipe_mem);
    pipe.prime(m.wo + layer * m.wo_stride + static_cast<long long>(blockIdx.x) * m.D * 32, m.D);
    Stager sg;
    sg.init(bar);
    const int rb = blockIdx.x;
    const int j = rb * 32 + (threadIdx.x & 31);
    // d_l of the decision predicted for this layer (for q_l): once the
    // predictor of layer-1 has published it (device flag, not the PDL edge),
    // its default-vector rows load while the attention still runs
    float d = 0.0f;
    if (rd_from_pred) {
        wait_decision(st, ctl, layer);
        if (j < m.H) d = layer_default_row(m, st.id_pred + layer * m.K, st.g_pred + layer * m.K, layer, j);
    }
    pdl_wait();
    KT_WAITED();
    pdl_trigger();  // after our own dependency: dependents launch at most one kernel ahead
    sg.add(xs, st.ctx, m.D * 4);
    sg.add(xr, st.x + blockIdx.x * 32, 32 * 4);
    sg.wait();
    const uint16_t* tile = m.wo + layer * m.wo_stride + static_cast<long long>(rb) * m.D * 32;
    const float acc = chain_run(pipe, m, tile, m.D, xs);
    const float r = j < m.H ? xr[threadIdx.x & 31] + acc : 0.0f;
    if (j < m.H) st.r[static_cast<long long>(layer) * m.Hp + j] = r;
    warp_ssq_partial(r, st.ssq_r + static_cast<long long>(layer) * (m.Hp / 32) + rb);
    if (rd_from_pred) {  // rd_l = r_l + d_l (speculation.cpp:119-121) and its rms_norm partial
        const float rd = j < m.H ? r + d : 0.0f;
        if (j < m.H) st.rd[static_cast<long long>(layer) * m.Hp + j] = rd;
        warp_ssq_partial(rd, st.ssq_rd + static_cast<long long>(layer) * (m.Hp / 32) + rb);
    }
}

// rd_l = r_l + d_l of the executed decision (id_exec / g_exec) when it is only
// known after k_wo (layer 0 in prefetch mode, where the true router decides):
// grid Hp/32 x 32, launched on the side stream ahead of the predictor.
__global__ void __launch_bounds__(32) k_quasi_rd(DevModel m, DevState st, int layer) {
    pdl_wait();
    pdl_trigger();
    const int rb = blockIdx.x, j = rb * 32 + (threadIdx.x & 31);
    float rd = 0.0f;
    if (j < m.H) {
        const float d = layer_default_row(m, st.id_exec + layer * m.K, st.g_exec + layer * m.K, layer, j);
        rd = __ldcg(st.r + static_cast<long long>(layer) * m.Hp + j) + d;
        st.rd[static_cast<long long>(layer) * m.Hp + j] = rd;
    }
    warp_ssq_partial(rd, st.ssq_rd + static_cast<long long>(layer) * (m.Hp / 32) + rb);
}

// ---------------------------------------------------------------- router --
//
// CTA groups: [0, nT) true-router row tiles of gate_l over s_l;
// [nT, nT+nP) predictor row tiles of gate_{l+1} over the predictor input
// (baseline-s: s_l; router-pf / est-pf: q_l = rms_norm(r_l + d_l, gain_{l+1})).
// The last CTA turns logits into decisions, fixes the executed decision and
// posts the copy requests.

// layer_default (speculation.cpp:104-117) + quasi_hidden (speculation.cpp:119-121)
// over the decision executed at `layer` (pred_l when this launch also fixes
// exec).  r, the K default-vector rows and gain_{l+1} are staged in smem.
__device__ void compute_quasi(const DevModel& m, const DevState& st, int layer, int exec_from,
                              float* qs, float* rs, float* gs, float* dvs, double* red,
                              Stager& sg) {
    const int H = m.H, K = m.K, Hr = round_up(H, 32);
    __shared__ int s_ids[kMaxK];
    __shared__ float s_g[kMaxK];
    if (threadIdx.x < K) {
        s_ids[threadIdx.x] = (exec_from == 1 ? st.id_pred : st.id_exec)[layer * K + threadIdx.x];
        s_g[threadIdx.x] = (exec_from == 1 ? st.g_pred : st.g_exec)[layer * K + threadIdx.x];
    }
    __syncthreads();
    sg.add(rs, st.r + static_cast<long long>(layer) * m.Hp, H * 4);
    sg.add(gs, m.moe_gain + static_cast<long long>(layer + 1) * H, H * 4);
    for (int i = 0; i < K; ++i)
        sg.add(dvs + i * Hr, m.dv + (static_cast<long long>(layer) * m.E + s_ids[i]) * H, H * 4);
    sg.wait();
    for (int j = threadIdx.x; j < H; j += blockDim.x) {
        float d = 0.0f;
        for (int i = 0; i < K; ++i) d = d + s_g[i] * dvs[i * Hr + j];
        rs[j] = rs[j] + d;
    }
    __syncthreads();
    block_rms_norm(rs, gs, H, m.eps, qs, red);
}

__global__ void __launch_bounds__(32 * kRouterSplitWarps) k_router(DevModel m, DevState st, DevCtl ctl,
                                               RouterLaunch rl, DevState sh, int has_shadow) {
    KTRACE(rl.do_true ? 4 : 13, rl.layer);
    PHASE_DECL
    PHASE();
    // gridDim.y > 1: the logging true routers of layers rl.layer .. +gridDim.y-1
    // in one launch (one y-slice per layer, per-layer last-CTA counters)
    const int H = m.H, E = m.E, K = m.K, l = rl.layer + static_cast<int>(blockIdx.y), Hr = round_up(H, 32);
    uint64_t* bar = reinterpret_cast<uint64_t*>(g_smem);
    double* red = reinterpret_cast<double*>(g_smem + 64);  // [kRouterSplitWarps] (block reductions)
    float* xs = reinterpret_cast<float*>(g_smem + 256);
    float* rs = xs + Hr;
    float* gs = rs + Hr;
    // [K][Hr] default-vector rows, only for a router-pf / est-pf q_l not
    // prepared by k_wo (router_smem sizes the launch by the same condition)
    float* dvs = gs + Hr;
    const bool needs_dv = (rl.pred_kind == kRouterPF || rl.pred_kind == kEstPF) && !rl.quasi_ready;
    unsigned char* pipe_mem = align128(reinterpret_cast<unsigned char*>(dvs + (needs_dv ? K * Hr : 0)));
    const int nT = rl.do_true ? m.Ep / 32 : 0;
    const bool gemv_pred = rl.pred_kind == kBaselineS || rl.pred_kind == kRouterPF;
    const int nP = gemv_pred ? m.Ep / 32 : 0;
    const int nQ = (rl.pred_kind == kEstPF) ? 1 : 0;  // est-pf: one CTA writes q_l
    const int b = blockIdx.x;
    PipeR pipe;
    SplitG spl;  // fast mode: kSplitWarps warps split the columns of the tile
    const uint16_t* tile = nullptr;
    if (b < nT + nP) {
        const bool is_true = b < nT;
        const int rb = is_true ? b : b - nT;
        tile = m.gate + (is_true ? l : l + 1) * m.gate_stride + static_cast<long long>(rb) * H * 32;
        if (SMOE_FAST(m)) {
            spl.prime(tile, H);
        } else {
            pipe.init(pipe_mem, kL2EvictLast);
            pipe.prime(tile, H);
        }
    }
    Stager sg;
    sg.init(bar);
    // the norm gains are static: staged before the PDL wait, the activations after
    const bool norm_s = b < nT || (b < nT + nP && rl.pred_kind == kBaselineS);
    const bool norm_q = !norm_s && b < nT + nP + nQ && rl.quasi_ready;
    if (norm_s) sg.add(gs, m.moe_gain + static_cast<long long>(l) * H, H * 4);
    if (norm_q) sg.add(gs, m.moe_gain + static_cast<long long>(l + 1) * H, H * 4);
    pdl_wait();
    KT_WAITED();
    PHASE();
    pdl_trigger();  // after our own dependency: dependents launch at most one kernel ahead
    if (norm_s) {
        sg.add(rs, st.r + static_cast<long long>(l) * m.Hp, H * 4);
        const float scale = rms_scale_from_partials(st.ssq_r + static_cast<long long>(l) * (m.Hp / 32),
                                                    m.Hp / 32, H, m.eps);
        sg.wait();
        block_apply_norm(rs, gs, H, scale, xs);
        if (b == 0 && rl.do_true)
            for (int j = threadIdx.x; j < H; j += blockDim.x) st.s[static_cast<long long>(l) * m.Hp + j] = xs[j];
    } else if (b < nT + nP + nQ) {
        if (rl.quasi_ready) {  // q_l = rms_norm(r_l + d_l, gain_{l+1}) from k_wo's rd_l
            sg.add(rs, st.rd + static_cast<long long>(l) * m.Hp, H * 4);
            const float scale = rms_scale_from_partials(
                st.ssq_rd + static_cast<long long>(l) * (m.Hp / 32), m.Hp / 32, H, m.eps);
            sg.wait();
            block_apply_norm(rs, gs, H, scale, xs);
        } else {
            compute_quasi(m, st, l, rl.exec_from, xs, rs, gs, dvs, red, sg);
        }
        if (b == nT)
            for (int j = threadIdx.x; j < H; j += blockDim.x) st.quasi[j] = xs[j];
    }
    PHASE();
    if (b < nT + nP) {
        const bool is_true = b < nT;
        const int rb = is_true ? b : b - nT;
        const float acc = SMOE_FAST(m) ? spl.run(tile, H, xs, reinterpret_cast<float*>(pipe_mem)) : pipe.run(tile, H, xs);
        const int e = rb * 32 + (threadIdx.x & 31);
        if (threadIdx.x < 32 && e < E) {
            if (is_true)
                st.lg_true[static_cast<long long>(l) * E + e] = acc;
            else
                st.lg_pred[static_cast<long long>(l + 1) * E + e] = acc;
        }
    }
    PHASE();
    // ---- finalize: the true-router CTAs and the predictor CTAs each elect
    // their own last CTA, so the two decisions run in parallel; the predictor's
    // copy request is posted without waiting for the (logging-only) true one.
    const bool in_true = b < nT;
    const bool has_b = static_cast<int>(gridDim.x) > nT;  // predictor / quasi CTAs exist
    int* gate_cnt = gridDim.y > 1 ? st.log_cnt + l : st.counters + (in_true ? 0 : 4);
    if (!last_cta(gate_cnt, in_true ? nT : gridDim.x - nT)) return;
    if (threadIdx.x >= 32) return;  // the decision is one warp's
    PHASE();
    double* se = reinterpret_cast<double*>(pipe_mem);            // [E]
    float* sp = reinterpret_cast<float*>(pipe_mem + kMaxE * 8);  // [E]
    if (in_true) {
        if (SMOE_FAST(m) && E <= 256)
            warp_decision_fast(st.lg_true + static_cast<long long>(l) * E, E, K, st.id_true + l * K,
                               st.g_true + l * K);
        else
            warp_decision(st.lg_true + static_cast<long long>(l) * E, E, K, m.gating, sp, se,
                          st.id_true + l * K, st.g_true + l * K);
        if (threadIdx.x == 0 && rl.exec_from == 0) {
            copy_decision(st.id_true + l * K, st.g_true + l * K, st.id_exec + l * K, st.g_exec + l * K, K);
            if (rl.post_exec && !ctl.resident) post_request(m, ctl, l, rl.step_tag, st.id_exec + l * K, K);
        }
    }
    if (!in_true || !has_b) {
        if (gemv_pred)
        {
            if (SMOE_FAST(m) && E <= 256)
                warp_decision_fast(st.lg_pred + static_cast<long long>(l + 1) * E, E, K, st.id_pred + (l + 1) * K,
                                   st.g_pred + (l + 1) * K);
            else
                warp_decision(st.lg_pred + static_cast<long long>(l + 1) * E, E, K, m.gating, sp, se,
                              st.id_pred + (l + 1) * K, st.g_pred + (l + 1) * K);
        }
        if (threadIdx.x == 0) {
            if (rl.pred_kind == kOracle && has_shadow) {  // Oracle: shadow true decisions (speculation.cpp:296-305)
                for (int i = 0; i < K; ++i) {
                    st.id_pred[(l + 1) * K + i] = sh.id_true[(l + 1) * K + i];
                    st.g_pred[(l + 1) * K + i] = sh.g_true[(l + 1) * K + i];
                }
            }
            if (rl.post_pred && !ctl.resident)
                post_request(m, ctl, l + 1, rl.step_tag, st.id_pred + (l + 1) * K, K);
            if ((gemv_pred || rl.pred_kind == kOracle) && l + 1 < m.L) publish_decision(st, l + 1);
            if (rl.exec_from == 1)
                copy_decision(st.id_pred + l * K, st.g_pred + l * K, st.id_exec + l * K, st.g_exec + l * K, K);
        }
        if (rl.pred_kind == kOracle && has_shadow)
            for (int e = threadIdx.x; e < E; e += blockDim.x)
                st.lg_pred[static_cast<long long>(l + 1) * E + e] = sh.lg_true[static_cast<long long>(l + 1) * E + e];
    }
#ifdef SMOE_PHASES
    PHASE();
    if (threadIdx.x == 0)
        phase_print(rl.do_true ? "true router [pdl, stage+norm, chain, lastcta, decide]"
                               : "predictor [pdl, stage+norm, chain, lastcta, decide]",
                    ph_, nph_);
#ifdef DECISION_TIMING
    if (threadIdx.x == 0 && !rl.do_true)
        printf("predictor decision [stage, softmax, topk, gates] (cycles): %lld %lld %lld %lld\n",
               g_dec_t[1] - g_dec_t[0], g_dec_t[2] - g_dec_t[1], g_dec_t[3] - g_dec_t[2], g_dec_t[4] - g_dec_t[3]);
#endif
#endif
}

// --------------------------------------------------------------- estimator --
// estimator_forward<float> (estimator.cpp:94-161), f32 throughout; stage kernels:
//  A: z = A.q + pos[l]   B: act = silu_f32(B.z)   C: h = z + C.act, LayerNorm
//  head: logits = W_head.(gain*xhat + bias), decision, mailbox.

__global__ void __launch_bounds__(32) k_est_stage(DevModel m, DevState st, DevCtl ctl, int layer,
                                                  int stage, int post_pred, int step_tag) {
    KTRACE(5 + stage, layer);
    const int dm = m.est_dm, mlp = m.est_mlp;
    float* xs = reinterpret_cast<float*>(g_smem);
    int cols;
    const float* in;
    const float* tiles;
    if (stage == 0) {
        cols = m.est_d;
        in = st.quasi;
        tiles = m.est_a;
    } else if (stage == 1) {
        cols = dm;
        in = st.est_z;
        tiles = m.est_b;
    } else if (stage == 2) {
        cols = mlp;
        in = st.est_act;
        tiles = m.est_c;
    } else {
        cols = dm;
        in = st.est_xn;
        tiles = m.est_head;
    }
    uint64_t* bar = reinterpret_cast<uint64_t*>(g_smem + round_up(cols, 32) * 4);
    unsigned char* pipe_mem = align128(g_smem + round_up(cols, 32) * 4 + 64);
    const int rb = blockIdx.x;
    PipeF pipe;
    pipe.init(pipe_mem);
    pipe.prime(tiles + static_cast<long long>(rb) * cols * 32, cols);
    Stager sg;
    sg.init(bar);
    pdl_wait();
    KT_WAITED();
    pdl_trigger();  // after our own dependency: dependents launch at most one kernel ahead
    sg.add(xs, in, cols * 4);
    sg.wait();
    const float acc = pipe.run(tiles + static_cast<long long>(rb) * cols * 32, cols, xs);
    const int row = rb * 32 + (threadIdx.x & 31);
    if (stage == 0) {
        if (row < dm) st.est_z[row] = acc + m.est_pos[static_cast<long long>(layer) * dm + row];
    } else if (stage == 1) {
        if (row < mlp) st.est_act[row] = acc / (1.0f + expf_glibc(-acc));
    } else if (stage == 2) {
        if (row < dm) st.est_xn[row] = st.est_z[row] + acc;  // h (normalised below)
    } else {
        if (row < m.E) st.lg_pred[static_cast<long long>(layer + 1) * m.E + row] = acc;
    }
    if (stage == 0 || stage == 1) return;
    if (!last_cta(st.counters + 1, gridDim.x)) return;
    if (stage == 2) {  // LayerNorm, mean/var in f32 sequential (estimator.cpp:137-151)
        if (threadIdx.x == 0) {
            float* h = st.est_xn;
            float mean = 0.0f;
            for (int j = 0; j < dm; ++j) mean += h[j];
            mean /= static_cast<float>(dm);
            float var = 0.0f;
            for (int j = 0; j < dm; ++j) {
                const float c = h[j] - mean;
                var += c * c;
            }
            var /= static_cast<float>(dm);
            const float inv_std = 1.0f / sqrtf(var + m.est_eps);
            for (int j = 0; j < dm; ++j) {
                const float xhat = (h[j] - mean) * inv_std;
                h[j] = m.est_gain[j] * xhat + m.est_bias[j];
            }
        }
        return;
    }
    // stage 3: decision + mailbox
    double* se = reinterpret_cast<double*>(pipe_mem);
    float* sp = reinterpret_cast<float*>(pipe_mem + kMaxE * 8);
    warp_decision(st.lg_pred + static_cast<long long>(layer + 1) * m.E, m.E, m.K, m.gating, sp,
                  se, st.id_pred + (layer + 1) * m.K, st.g_pred + (layer + 1) * m.K);
    if (threadIdx.x == 0 && post_pred && !ctl.resident)
        post_request(m, ctl, layer + 1, step_tag, st.id_pred + (layer + 1) * m.K, m.K);
    if (threadIdx.x == 0 && layer + 1 < m.L) publish_decision(st, layer + 1);
}

// ------------------------------------------------------------- expert FFN --
//
// expert_ffn (model.cpp:283-288) for every executed expert, read from its HBM
// slot.  gate/up: grid (Hmp/16, K), one warp per 16-row tile (lanes 2r, 2r+1
// hold gate row r and up row r); h = silu(g) * u.

__device__ void wait_ready(const DevCtl& ctl, int layer) {
    if (ctl.resident || ctl.host_ordered) return;  // host-ordered: a stream event did it
    if (threadIdx.x == 0) {
        const int want = __ldcg(ctl.req_seq + layer);
        const long long t0 = clock64();
        while (ld_acquire(ctl.ready + layer) < want) {
            if (*(volatile int*)ctl.error) break;
            __nanosleep(128);
            if (clock64() - t0 > ctl.spin_limit) {
                atomicCAS(ctl.error, 0, 1000 + layer);
                break;
            }
        }
    }
    __syncthreads();
}

// exec_src 0: the executed decision is id_exec/g_exec[layer] (fixed by the
// router before this kernel); 1: it is the decision predicted at layer-1
// (id_pred/g_pred[layer]) — prefetch mode, where the routers of this layer
// run concurrently on a side stream (Alg. 1: the predicted experts are known
// before the layer starts).  s_from_r: compute s_l = rms_norm(r_l, moe_gain_l)
// here instead of reading the router's copy.
// gate/up role of one (16-row block rb, executed expert i).  `fused`: the down
// role runs in the same grid and waits on gu_done[layer][i].
__device__ __forceinline__ void ffn_gu_body(const DevModel& m, const DevState& st, const DevCtl& ctl,
                                            int layer, int exec_src, int s_from_r, int rb, int i,
                                            bool fused) {
    KTRACE(9, layer);
    // counts this CTA towards gu_done[layer][i] on every exit path, so a down
    // CTA never waits for a gate/up CTA that left early (EP peer expert, error)
    struct Done {
        const DevState& st;
        int idx;
        bool on;
        __device__ ~Done() {
            if (on && threadIdx.x == 0) {
                __threadfence();
                atomicAdd(st.gu_done + idx, 1);
            }
        }
    } done{st, layer * m.K + i, fused};
    PHASE_DECL
    PHASE();
    // prefetch mode: the executed decision was published by the predictor of
    // layer l-1 on the side stream (publish_decision); wait for that flag, not
    // for the PDL edge, and start the copy wait and weight stream before the
    // PDL wait, overlapping the attention tail.  On-demand: the router of this
    // layer (our predecessor) decides, so wait for it first.
    const bool early = exec_src != 0;
    if (early) {
        wait_decision(st, ctl, layer);
    } else {
        pdl_wait();
        KT_WAITED();
    }
    const int H = m.H;
    const int e = __ldcg((exec_src ? st.id_pred : st.id_exec) + layer * m.K + i);
    if (ctl.ep.world > 1 && e % ctl.ep.world != ctl.ep.rank) return;  // a peer runs it
    wait_ready(ctl, layer);
    if (*(volatile int*)ctl.error) return;
    uint64_t* bar = reinterpret_cast<uint64_t*>(g_smem);
    float* xs = reinterpret_cast<float*>(g_smem + 128);
    // only the input vector is staged (the gain is read once from L2 by the
    // norm), which keeps k_ffn_gu at ~41 KB so five CTAs fit per SM and the
    // next launch's CTAs are resident (weights primed) while this one drains;
    // the fused grid keeps 2 vectors of room for h (gu_stage_floats)
    unsigned char* pipe_mem =
        align128(reinterpret_cast<unsigned char*>(xs + (fused ? 2 : 1) * round_up(H, 32)));
    const int slot = __ldcg(m.slot_of + layer * m.E + e);
    if (slot < 0) {
        if (threadIdx.x == 0) atomicCAS(ctl.error, 0, 2000 + layer);
        return;
    }
    const uint16_t* tile = m.slots + (static_cast<long long>(layer) * m.C + slot) * m.expert_elems +
                           static_cast<long long>(rb) * H * 32;
    PipeGU pipe;
    pipe.init(pipe_mem, kL2EvictFirst);
    pipe.prime(tile, H);
    if ((g_down_l2_dev || (fused && g_fused_l2_dev)) && threadIdx.x == 0) {
        // warm L2 with this CTA's share of the expert's down-projection block,
        // so k_ffn_down streams it from L2 while our gate/up stream runs on HBM
        const char* dn = reinterpret_cast<const char*>(
            m.slots + (static_cast<long long>(layer) * m.C + slot) * m.expert_elems + m.gu_elems);
        const long long bytes = static_cast<long long>(m.Hp) * m.Hmp * 2;
        const int parts = m.Hmp / 16;
        const long long part = ((bytes + parts - 1) / parts + 15) / 16 * 16;
        const long long b0 = part * rb, b1 = min(bytes, b0 + part);
        for (long long o = b0; o < b1; o += 65536) {
            const uint32_t nb = static_cast<uint32_t>(min(65536LL, b1 - o)) & ~15u;
            if (nb) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(dn + o), "r"(nb) : "memory");
        }
    }
    if (early) {
        pdl_wait();
        KT_WAITED();
    }
    // every CTA is past its copy wait: k_ffn_down may now read ids / slot_of and
    // stream its weights before its own PDL wait
    pdl_trigger();
    PHASE();
    Stager sg;
    sg.init(bar);
    if (s_from_r) {
        sg.add(xs, st.r + static_cast<long long>(layer) * m.Hp, H * 4);
        const float scale = rms_scale_from_partials(st.ssq_r + static_cast<long long>(layer) * (m.Hp / 32),
                                                    m.Hp / 32, H, m.eps);
        sg.wait();
        block_apply_norm(xs, m.moe_gain + static_cast<long long>(layer) * H, H, scale, xs);
    } else {
        sg.add(xs, st.s + static_cast<long long>(layer) * m.Hp, H * 4);
        sg.wait();
    }
    PHASE();
    const float acc = chain_run(pipe, m, tile, H, xs);
    PHASE();
    const float up = __shfl_xor_sync(0xffffffffu, acc, 1);
    const int lane = threadIdx.x & 31;
    if ((lane & 1) == 0) {
        const int row = rb * 16 + (lane >> 1);
        st.h[static_cast<long long>(i) * m.Hmp + row] = silu_ref(acc) * up;
    }
    PHASE();
    PHASE_DUMP("ffn_gu [pdl, ready+stage+norm, chain, epi]");
#ifdef SMOE_PHASES
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
        printf("ffn_gu chain waits (cycles): %lld\n", pipe.wait_cyc);
#endif
    if (fused) __syncwarp();  // h rows written by every lane before the count (Done)
}

__global__ void __launch_bounds__(32) k_ffn_gu(DevModel m, DevState st, DevCtl ctl, int layer,
                                               int exec_src, int s_from_r) {
    ffn_gu_body(m, st, ctl, layer, exec_src, s_from_r, blockIdx.x, blockIdx.y, false);
}

// Gate/up with W row-tile warps per CTA (grid (ceil(Hmp/16 / W), K)).  Same
// arithmetic as k_ffn_gu — every lane still walks one SwiGLU row's columns in
// order — but the warps of a CTA sit on distinct SM sub-partitions (warp w on
// SMSP w % 4), so no two chains share an issue slot, and the input staging
// and norm are shared by the W warps.  Selected by gu_warps (launch_ffn).
template <int W>
__global__ void __launch_bounds__(32 * W) k_ffn_gu_w(DevModel m, DevState st, DevCtl ctl, int layer,
                                                     int exec_src, int s_from_r) {
    KTRACE(9, layer);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, i = blockIdx.y;
    const int rb = blockIdx.x * W + warp;
    const bool active = rb < m.Hmp / 16;
    const bool early = exec_src != 0;  // prefetch mode: decision published a layer ahead
    if (early) {
        wait_decision(st, ctl, layer);
    } else {
        pdl_wait();
        KT_WAITED();
    }
    __syncthreads();
    const int H = m.H;
    const int e = __ldcg((exec_src ? st.id_pred : st.id_exec) + layer * m.K + i);
    if (ctl.ep.world > 1 && e % ctl.ep.world != ctl.ep.rank) return;  // a peer runs it (CTA-uniform)
    wait_ready(ctl, layer);
    if (__syncthreads_or(*(volatile int*)ctl.error)) return;
    uint64_t* bar = reinterpret_cast<uint64_t*>(g_smem);
    float* xs = reinterpret_cast<float*>(g_smem + 128);
    unsigned char* pipe_mem = align128(reinterpret_cast<unsigned char*>(xs + round_up(H, 32))) +
                              warp * round_up(PipeGU::kBytes, 128);
    const int slot = __ldcg(m.slot_of + layer * m.E + e);
    if (slot < 0) {
        if (threadIdx.x == 0) atomicCAS(ctl.error, 0, 2000 + layer);
        return;
    }
    const uint16_t* tile = m.slots + (static_cast<long long>(layer) * m.C + slot) * m.expert_elems +
                           static_cast<long long>(rb) * H * 32;
    PipeGU pipe;
    if (active) {
        pipe.init(pipe_mem, kL2EvictFirst);
        pipe.prime(tile, H);
    }
    if (early) {
        pdl_wait();
        KT_WAITED();
    }
    pdl_trigger();  // every CTA is past its copy wait (k_ffn_down reads ids / slot_of early)
    Stager sg;
    sg.init(bar);
    if (s_from_r) {
        sg.add(xs, st.r + static_cast<long long>(layer) * m.Hp, H * 4);
        const float scale = rms_scale_from_partials(st.ssq_r + static_cast<long long>(layer) * (m.Hp / 32),
                                                    m.Hp / 32, H, m.eps);
        sg.wait();
        block_apply_norm(xs, m.moe_gain + static_cast<long long>(layer) * H, H, scale, xs);
    } else {
        sg.add(xs, st.s + static_cast<long long>(layer) * m.Hp, H * 4);
        sg.wait();
    }
    if (!active) return;
    const float acc = chain_run(pipe, m, tile, H, xs);
    const float up = __shfl_xor_sync(0xffffffffu, acc, 1);
    if ((lane & 1) == 0) st.h[static_cast<long long>(i) * m.Hmp + rb * 16 + (lane >> 1)] = silu_ref(acc) * up;
}

// ---------------------------------------------- tolerance-mode expert FFN --
//
// Column-split expert GEMVs (DevModel::fast only).  The exact kernels give
// each 32-row tile to ONE warp, because the reference's dot product is one
// sequential sum; with one warp per SM sub-partition that stream is issue-
// latency bound (ncu, profiles/r02_ncu_fast_summary.csv: ~4 cycles per
// instruction, DRAM at 38 % of peak).  In tolerance mode the tile's columns
// are split over kCsWarps warps of the CTA (warp w: a contiguous range of
// 8-column groups, its own cp.async.bulk pipe of 8 KB chunks), each lane
// keeps packed-FFMA partial sums of its row, and warp 0 adds the warps'
// partials in warp order (deterministic) before the usual epilogue.  4x the
// warps in flight for the same bytes; the CTA still fits three per SM.
// Measured on Q30 (16 layers, tools/kbench.py): 10.3 us per launch in the
// prefetch form against 12.1 us for the one-warp tile.  Also measured and
// dropped: 8 warps (one CTA per SM: 17 us), 3-stage pipes (two CTAs per SM:
// 14 us), register-streamed LDG tiles (18 us), and the same split for the
// down projection (8.5 us against 7.5 us for the one-warp k_ffn_down, whose
// whole 48 KB tile is in flight per warp).
#ifndef SMOE_CS_WARPS
#define SMOE_CS_WARPS 4
#endif
#ifndef SMOE_CS_S
#define SMOE_CS_S 2
#endif
#ifndef SMOE_CS_CC
#define SMOE_CS_CC 128
#endif
constexpr int kCsWarps = SMOE_CS_WARPS;
using PipeCs = WarpPipe<uint16_t, SMOE_CS_S, SMOE_CS_CC>;  // gate/up: 2 x 8 KB per warp


// this warp's column range [c0, c0 + n) of a `cols`-column tile
__device__ __forceinline__ void cs_range(int cols, int& c0, int& n) {
    const int ng = (cols + 7) / 8, per = (ng + kCsWarps - 1) / kCsWarps, w = threadIdx.x >> 5;
    c0 = min(ng, w * per) * 8;
    n = max(0, min(cols - c0, per * 8));
}

// red: [kCsWarps][32] floats; returns the row sum in warp 0 (others: 0)
__device__ __forceinline__ float cs_reduce(float part, float* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    red[w * 32 + lane] = part;
    __syncthreads();
    float s = 0.0f;
    if (w == 0) {
#pragma unroll
        for (int q = 0; q < kCsWarps; ++q) s += red[q * 32 + lane];
    }
    return s;
}

// this warp's ring behind the red / staging areas (k_ffn_gu_cs, k_ffn_cs)
__device__ __forceinline__ unsigned char* cs_pipe_mem(const DevModel& m) {
    float* xs = reinterpret_cast<float*>(g_smem + 128) + kCsWarps * 32;
    return align128(reinterpret_cast<unsigned char*>(xs + round_up(max(m.H, m.Hmp), 32))) +
           (threadIdx.x >> 5) * round_up(PipeCs::kBytes, 128);
}

// Gate/up of one (16-row block rb, executed expert i) by the CTA's kCsWarps
// warps.  `fused`: the down projection runs in the same grid (k_ffn_cs) and
// waits on gu_done[layer][i], counted here on every exit path.
template <bool DOWN = false>
__device__ __forceinline__ void gu_cs_unit(const DevModel& m, const DevState& st, const DevCtl& ctl, int layer,
                                           int exec_src, int s_from_r, int rb, int i, bool fused, PipeCs& pipe) {
    struct Done {  // a down CTA never waits for a gate/up CTA that left early
        const DevState& st;
        int idx;
        bool on;
        __device__ ~Done() {
            if (on && threadIdx.x == 0) {
                __threadfence();
                atomicAdd(st.gu_done + idx, 1);
            }
        }
    } done{st, layer * m.K + i, fused};
    KTRACE(9, layer);
    const int lane = threadIdx.x & 31;
    const bool early = exec_src != 0;  // prefetch mode: decision published a layer ahead
    GainRegs gr;  // the MoE norm gain is static: in registers before any wait
    if (s_from_r) gr.load(m.moe_gain + static_cast<long long>(layer) * m.H, m.H);
    if (early) {
        wait_decision(st, ctl, layer);
    } else {
        pdl_wait();
        KT_WAITED();
    }
    __syncthreads();
    const int H = m.H;
    const int e = __ldcg((exec_src ? st.id_pred : st.id_exec) + layer * m.K + i);
    if (ctl.ep.world > 1 && e % ctl.ep.world != ctl.ep.rank) return;  // a peer runs it (CTA-uniform)
    wait_ready(ctl, layer);
    if (__syncthreads_or(*(volatile int*)ctl.error)) return;
    uint64_t* bar = reinterpret_cast<uint64_t*>(g_smem);
    float* red = reinterpret_cast<float*>(g_smem + 128);
    float* xs = red + kCsWarps * 32;
    const int slot = __ldcg(m.slot_of + layer * m.E + e);
    if (slot < 0) {
        if (threadIdx.x == 0) atomicCAS(ctl.error, 0, 2000 + layer);
        return;
    }
    int c0, nc;
    cs_range(H, c0, nc);
    const uint16_t* tile = m.slots + (static_cast<long long>(layer) * m.C + slot) * m.expert_elems +
                           static_cast<long long>(rb) * H * 32 + static_cast<long long>(c0) * 32;
    if (nc > 0) pipe.prime(tile, nc);
    if (early) {
        pdl_wait();
        KT_WAITED();
    }
    pdl_trigger();  // every CTA is past its copy wait (k_ffn_down reads ids / slot_of early)
    Stager sg;
    sg.init(bar);
    if (s_from_r) {
        sg.add(xs, st.r + static_cast<long long>(layer) * m.Hp, H * 4);
        const float scale = rms_scale_from_partials(st.ssq_r + static_cast<long long>(layer) * (m.Hp / 32),
                                                    m.Hp / 32, H, m.eps);
        sg.wait();
        block_apply_norm_regs(xs, gr, m.moe_gain + static_cast<long long>(layer) * H, H, scale, xs);
    } else {
        sg.add(xs, st.s + static_cast<long long>(layer) * m.Hp, H * 4);
        sg.wait();
    }
    // tolerance mode only (launch_gu); SMOE_FAST is constant 0 in the exact-only object
    const float part = nc > 0 && SMOE_FAST(m) ? pipe.run_fast(tile, nc, xs + c0) : 0.0f;
    // DOWN (k_ffn_gud): this warp's share of the down block's 16-column slice
    // [16 rb, 16 rb + 16) — one 1 KB piece per 32-row tile — streams into the
    // ring right behind the gate/up chunks, before the cross-warp reduction
    const int nrt = m.Hp / 32, per = (nrt + kCsWarps - 1) / kCsWarps, w = threadIdx.x >> 5;
    const int t0 = min(nrt, w * per), tn = max(0, min(nrt - t0, per));
    constexpr int kTpc = PipeCs::kChunkElems / 512;  // 1 KB pieces per ring chunk
    const int nchd = (tn + kTpc - 1) / kTpc;
    const uint16_t* dsrc = m.slots + (static_cast<long long>(layer) * m.C + slot) * m.expert_elems + m.gu_elems +
                           static_cast<long long>(t0) * m.Hmp * 32 + rb * 512;
    if (DOWN && lane == 0)
        for (int c = 0; c < PipeCs::kS && c < nchd; ++c)
            pipe.issue_gather(dsrc + static_cast<long long>(c) * kTpc * m.Hmp * 32, static_cast<long long>(m.Hmp) * 32,
                              min(kTpc, tn - c * kTpc), 512, pipe.ctr + c);
    const float acc = cs_reduce(part, red);
    if (threadIdx.x < 32) {
        const float up = __shfl_xor_sync(0xffffffffu, acc, 1);
        const float hv = silu_ref(acc) * up;
        if ((lane & 1) == 0) st.h[static_cast<long long>(i) * m.Hmp + rb * 16 + (lane >> 1)] = hv;
        if (DOWN && (lane & 1) == 0) xs[lane >> 1] = hv;  // xs is free: every warp is past its sums
    }
    if (fused) __syncthreads();  // h rows written before the count (Done)
    if (!DOWN || !SMOE_FAST(m)) return;
    __syncthreads();
    float hr[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) hr[c] = xs[c];
    float* out = st.dpart + (static_cast<long long>(i) * (m.Hmp / 16) + rb) * m.Hp + static_cast<long long>(t0) * 32;
    for (int c = 0; c < nchd; ++c) {
        const uint32_t cb = pipe.wait_chunk(pipe.ctr + c);
        const int np = min(kTpc, tn - c * kTpc);
        for (int p = 0; p < np; ++p) {
            const uint4 g0 = lds128(cb + p * 1024 + lane * 16), g1 = lds128(cb + p * 1024 + 512 + lane * 16);
            float a = lo_bf(g0.x) * hr[0];
            a = a + hi_bf(g0.x) * hr[1];
            a = a + lo_bf(g0.y) * hr[2];
            a = a + hi_bf(g0.y) * hr[3];
            a = a + lo_bf(g0.z) * hr[4];
            a = a + hi_bf(g0.z) * hr[5];
            a = a + lo_bf(g0.w) * hr[6];
            a = a + hi_bf(g0.w) * hr[7];
            a = a + lo_bf(g1.x) * hr[8];
            a = a + hi_bf(g1.x) * hr[9];
            a = a + lo_bf(g1.y) * hr[10];
            a = a + hi_bf(g1.y) * hr[11];
            a = a + lo_bf(g1.z) * hr[12];
            a = a + hi_bf(g1.z) * hr[13];
            a = a + lo_bf(g1.w) * hr[14];
            a = a + hi_bf(g1.w) * hr[15];
            __stcg(out + (c * kTpc + p) * 32 + lane, a);
        }
        __syncwarp();
        if (c + PipeCs::kS < nchd && lane == 0) {
            const int cn = c + PipeCs::kS;
            pipe.issue_gather(dsrc + static_cast<long long>(cn) * kTpc * m.Hmp * 32, static_cast<long long>(m.Hmp) * 32,
                              min(kTpc, tn - cn * kTpc), 512, pipe.ctr + cn);
        }
    }
    pipe.ctr += nchd;
}

__global__ void __launch_bounds__(32 * kCsWarps) k_ffn_gu_cs(DevModel m, DevState st, DevCtl ctl, int layer,
                                                            int exec_src, int s_from_r) {
    PipeCs pipe;  // one ring per warp (its mbarriers are initialised once per launch)
    pipe.init(cs_pipe_mem(m), kL2EvictFirst);
    gu_cs_unit(m, st, ctl, layer, exec_src, s_from_r, blockIdx.x, blockIdx.y, false, pipe);
}

// Tolerance-mode expert FFN on one GPU as two launches without a cross-CTA
// wait between gate/up and down: CTA (rb, i) computes the 16 h values of
// rows [16 rb, 16 rb + 16) of expert i (as k_ffn_gu_cs) and then the down
// projection's partial over exactly those 16 columns of h for all H rows,
// its 16-column slice of the down block (Hp/32 pieces of 1 KB) streamed
// through the same per-warp ring right behind the gate/up chunks.  So the
// layer's 75 MB of expert weights stream in ONE launch with no CTA waiting
// for another; k_down_reduce then sums the Hmp/16 partials of each row in
// slice order (deterministic), mixes the experts in decision order
// (model.cpp:297-301) and adds the residual, like k_ffn_down's epilogue.
// Opt-in (SMOE_FFN_GUD=1): the fused launch streams its 75 MB in ~15 µs
// (5.0 TB/s, vs 9.9 + 7.5 µs for the pair), but the reduction launch costs
// ~4 µs after it (device timeline), so the layer is ~1 µs slower.
__global__ void __launch_bounds__(32 * kCsWarps) k_ffn_gud(DevModel m, DevState st, DevCtl ctl, int layer,
                                                          int exec_src, int s_from_r) {
    PipeCs pipe;
    pipe.init(cs_pipe_mem(m), kL2EvictFirst);
    gu_cs_unit<true>(m, st, ctl, layer, exec_src, s_from_r, blockIdx.x, blockIdx.y, false, pipe);
}

__global__ void __launch_bounds__(32 * kMaxK) k_down_reduce(DevModel m, DevState st, DevCtl ctl, int layer,
                                                            int exec_src) {
    KTRACE(16, layer);
    __shared__ float ys[kMaxK][32];
    pdl_wait();
    KT_WAITED();
    pdl_trigger();
    const int K = m.K, q = threadIdx.x >> 5, lane = threadIdx.x & 31, rb = blockIdx.x, j = rb * 32 + lane;
    const int ncb = m.Hmp / 16;
    if (*(volatile int*)ctl.error) return;
    // warp 0's mixture inputs, loaded up front (independent of the partial sums)
    const float* gts = (exec_src ? st.g_pred : st.g_exec) + layer * K;
    float gv[kMaxK], rv = 0.0f;
    if (q == 0) {
#pragma unroll
        for (int k = 0; k < kMaxK; ++k) gv[k] = k < K ? __ldcg(gts + k) : 0.0f;
        if (j < m.H) rv = __ldcg(st.r + static_cast<long long>(layer) * m.Hp + j);
    }
    if (q < K) {
        const float* p = st.dpart + static_cast<long long>(q) * ncb * m.Hp + j;
        float y = 0.0f;
        for (int c0 = 0; c0 < ncb; c0 += 64) {  // 64 loads in flight (one L2 round trip), then the sum in order
            float v[64];
#pragma unroll
            for (int u = 0; u < 64; ++u) v[u] = c0 + u < ncb ? __ldcg(p + static_cast<long long>(c0 + u) * m.Hp) : 0.0f;
#pragma unroll
            for (int u = 0; u < 64; ++u)
                if (c0 + u < ncb) y = y + v[u];
        }
        ys[q][lane] = y;
        if (j < m.H) st.y[static_cast<long long>(q) * m.Hp + j] = y;
    }
    __syncthreads();
    if (q != 0) return;
    float xv = 0.0f;
    if (j < m.H) {
        float out = 0.0f;
#pragma unroll
        for (int k = 0; k < kMaxK; ++k)
            if (k < K) out += gv[k] * ys[k][lane];
        st.m[static_cast<long long>(layer) * m.Hp + j] = out;
        xv = rv + out;
        st.x[j] = xv;
    }
    warp_ssq_partial(xv, st.ssq_x + static_cast<long long>(layer + 1) * (m.Hp / 32) + rb);
}

__device__ __forceinline__ void down_block_epilogue(const DevModel& m, const DevState& st, const float* gts,
                                                    int layer, int rb, int i, float acc);

// Tolerance-mode expert FFN in ONE launch (single GPU; every CTA co-resident,
// checked at session creation): CTA b first computes gate/up unit
// (b % (Hmp/16), b / (Hmp/16)) as k_ffn_gu_cs, then claims down items
// (32-row block, expert) from an atomic counter — gate/up units are never
// claimed, so a claimed item only waits for CTAs that are already running.
// For each item the CTA primes the item's down weights (4 warps x a column
// slice) BEFORE waiting for the expert's gate/up units (gu_done), so the down
// weights stream while the last gate/up tiles finish; then h, the 4-warp
// column-split sums, and k_ffn_down's epilogue.  One launch per layer: no
// down-kernel launch gap, ramp or gate/up tail.
__global__ void __launch_bounds__(32 * kCsWarps) k_ffn_cs(DevModel m, DevState st, DevCtl ctl, int layer,
                                                         int exec_src, int s_from_r) {
    KTRACE(15, layer);
    const int ngu_x = m.Hmp / 16, nrb = m.Hp / 32, items = nrb * m.K;
    const int epoch = __ldcg(st.ffn_epoch + layer);  // before this launch's last CTA bumps it
    // one ring per warp for the whole launch: the down items continue its
    // chunk count (re-initialising the mbarriers between runs stalled the TMA)
    PipeCs pipe;
    pipe.init(cs_pipe_mem(m), kL2EvictFirst);
    gu_cs_unit(m, st, ctl, layer, exec_src, s_from_r, blockIdx.x % ngu_x, blockIdx.x / ngu_x, true, pipe);
    const int* ids = (exec_src ? st.id_pred : st.id_exec) + layer * m.K;
    const float* gts = (exec_src ? st.g_pred : st.g_exec) + layer * m.K;
    float* red = reinterpret_cast<float*>(g_smem + 128);
    float* hs = red + kCsWarps * 32;
    const int target = (epoch + 1) * ngu_x;
    __shared__ int s_it;
    for (;;) {
        __syncthreads();  // every warp is done with the previous item's smem
        if (threadIdx.x == 0) s_it = atomicAdd(st.counters + 6, 1);
        __syncthreads();
        const int it = s_it;
        if (__syncthreads_or(*(volatile int*)ctl.error) || it >= items) break;
        const int i = it / nrb, rb = it % nrb;
        const int e = __ldcg(ids + i);
        const int slot = __ldcg(m.slot_of + layer * m.E + e);
        if (slot < 0) {
            if (threadIdx.x == 0) atomicCAS(ctl.error, 0, 2000 + layer);
            break;
        }
        int c0, nc;
        cs_range(m.Hm, c0, nc);
        const uint16_t* tile = m.slots + (static_cast<long long>(layer) * m.C + slot) * m.expert_elems + m.gu_elems +
                               static_cast<long long>(rb) * m.Hmp * 32 + static_cast<long long>(c0) * 32;
        if (nc > 0) pipe.prime(tile, nc);  // weights do not depend on h: stream them now
        if (threadIdx.x == 0) {  // this expert's h rows are complete
            const int* cnt = st.gu_done + layer * m.K + i;
            const long long t0 = clock64();
            for (;;) {
                int v;
                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
                if (v >= target || *(volatile int*)ctl.error) break;
                if (clock64() - t0 > ctl.spin_limit) {
                    atomicCAS(ctl.error, 0, 1000 + layer);
                    break;
                }
                __nanosleep(32);
            }
        }
        if (__syncthreads_or(*(volatile int*)ctl.error)) break;
        const float4* h4 = reinterpret_cast<const float4*>(st.h + static_cast<long long>(i) * m.Hmp);
        for (int t = threadIdx.x; t < m.Hmp / 4; t += blockDim.x) reinterpret_cast<float4*>(hs)[t] = __ldcg(h4 + t);
        __syncthreads();
        const float part = nc > 0 && SMOE_FAST(m) ? pipe.run_fast(tile, nc, hs + c0) : 0.0f;
        const float acc = cs_reduce(part, red);
        if (threadIdx.x < 32) down_block_epilogue(m, st, gts, layer, rb, i, acc);
    }
    if (last_cta(st.counters + 5, gridDim.x) && threadIdx.x == 0) {
        st.counters[6] = 0;  // every CTA has left its claim loop
        st.ffn_epoch[layer] = epoch + 1;
    }
}

// Single-GPU epilogue of one 32-row block of executed expert i's down
// projection: the raw rows y_i; the last of the K arrivals on the block
// (device-scope counter, threadfence pattern) forms the gate-weighted mixture
// in decision order (model.cpp:297-301), the residual x = r + m
// (model.cpp:386) and the rms_norm partial of x for the next layer.
__device__ __forceinline__ void down_block_epilogue(const DevModel& m, const DevState& st, const float* gts,
                                                    int layer, int rb, int i, float acc) {
    const int K = m.K, lane = threadIdx.x & 31, j = rb * 32 + lane;
    if (j < m.H) st.y[static_cast<long long>(i) * m.Hp + j] = acc;
    __threadfence();
    __syncwarp();
    int last = 0;
    if (lane == 0) last = atomicAdd(st.down_cnt + rb, 1) == K - 1;
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) return;
    __threadfence();
    if (lane == 0) st.down_cnt[rb] = 0;
    float xv = 0.0f;
    if (j < m.H) {
        // all loads first (independent, one L2 round trip), then the mixture in
        // decision order
        float yv[kMaxK], gv[kMaxK];
#pragma unroll
        for (int q = 0; q < kMaxK; ++q) {
            yv[q] = q < K ? __ldcg(st.y + static_cast<long long>(q) * m.Hp + j) : 0.0f;
            gv[q] = q < K ? gts[q] : 0.0f;
        }
        const float rv = __ldcg(st.r + static_cast<long long>(layer) * m.Hp + j);
        float out = 0.0f;
#pragma unroll
        for (int q = 0; q < kMaxK; ++q)
            if (q < K) out += gv[q] * yv[q];
        st.m[static_cast<long long>(layer) * m.Hp + j] = out;
        xv = rv + out;
        st.x[j] = xv;
    }
    warp_ssq_partial(xv, st.ssq_x + static_cast<long long>(layer + 1) * (m.Hp / 32) + rb);
}

// down: grid (Hp/32, K), one warp per (32-row block, executed expert), so the
// 25 MB of Q30 down weights stream through every SM.  Each CTA writes its raw
// expert rows y_i; the last of the K CTAs of a row block (device-scope arrival
// counter, threadfence pattern) forms the gate-weighted mixture in decision
// order (model.cpp:297-301), the residual x = r + m (model.cpp:386) and the
// rms_norm partial of x for the next layer.
__device__ __forceinline__ void ffn_down_body(const DevModel& m, const DevState& st, const DevCtl& ctl,
                                              int layer, int exec_src, int rb, int i, bool fused,
                                              int gu_target) {
    KTRACE(10, layer);
    PHASE_DECL
    PHASE();
    // separate kernel: ids and slot_of are final once every k_ffn_gu CTA passed
    // its copy wait (its PDL trigger point), so the weight stream starts before
    // our PDL wait; fused grid: this CTA waits for the decision and the copy
    // itself, and for the gate/up CTAs of its expert (gu_done) before reading h.
    const int K = m.K, Hmp = m.Hmp, lane = threadIdx.x & 31;
    if (fused) {
        if (exec_src != 0) {
            wait_decision(st, ctl, layer);
        } else {
            pdl_wait();
            KT_WAITED();
        }
        wait_ready(ctl, layer);
    }
    float* hs = reinterpret_cast<float*>(g_smem + 128);  // [Hmp] this expert's hidden state
    unsigned char* pipe_mem = align128(reinterpret_cast<unsigned char*>(hs + Hmp));
    const int* ids = (exec_src ? st.id_pred : st.id_exec) + layer * K;
    const float* gts = (exec_src ? st.g_pred : st.g_exec) + layer * K;
    const int e = __ldcg(ids + i);
    const bool local = ctl.ep.world == 1 || e % ctl.ep.world == ctl.ep.rank;
    const int j = rb * 32 + lane;
    const int slot = local ? __ldcg(m.slot_of + layer * m.E + e) : 0;
    PipeD pipe;
    const uint16_t* tile = nullptr;
    if (local && slot >= 0) {
        tile = m.slots + (static_cast<long long>(layer) * m.C + slot) * m.expert_elems + m.gu_elems +
               static_cast<long long>(rb) * Hmp * 32;
        pipe.init(pipe_mem, kL2EvictFirst);
        pipe.prime(tile, m.Hm);
    }
    pdl_wait();
    KT_WAITED();
    pdl_trigger();  // after our own dependency: dependents launch at most one kernel ahead
    PHASE();
    if (fused && local && threadIdx.x == 0) {  // the gate/up CTAs of this expert are done
        const int* cnt = st.gu_done + layer * K + i;
        const long long t0 = clock64();
        for (;;) {
            int v;
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
            if (v >= gu_target) break;
            if (*(volatile int*)ctl.error) break;
            if (clock64() - t0 > ctl.spin_limit) {
                atomicCAS(ctl.error, 0, 1000 + layer);
                break;
            }
            __nanosleep(32);
        }
    }
    __syncwarp();
    if (*(volatile int*)ctl.error) return;
    float acc = 0.0f;
    if (local) {
        if (slot < 0) {
            if (lane == 0) atomicCAS(ctl.error, 0, 2000 + layer);
            return;
        }
        PHASE();
        // h (written by k_ffn_gu, L2-resident): direct 16-byte loads, 8 in flight per lane
        const float4* h4 = reinterpret_cast<const float4*>(st.h + static_cast<long long>(i) * Hmp);
        for (int t0 = 0; t0 < Hmp / 4; t0 += 8 * 32) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int t = t0 + u * 32 + lane;
                if (t < Hmp / 4) v[u] = __ldcg(h4 + t);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int t = t0 + u * 32 + lane;
                if (t < Hmp / 4) reinterpret_cast<float4*>(hs)[t] = v[u];
            }
        }
        __syncwarp();
        PHASE();
        acc = chain_run(pipe, m, tile, m.Hm, hs);
        PHASE();
    }
    if (ctl.ep.world > 1) {
        // EP: the owning rank publishes these expert rows to every rank (peer
        // stores over NVLink), fences them system-wide and counts the CTA on a
        // local per-layer counter; the last of the K x Hp/32 local CTAs (owner
        // or not) then makes ONE system-scope arrival on every rank's counter.
        // A rank therefore arrives for layer l only after all its CTAs of l
        // ran, which keeps the ranks within one layer of each other (the
        // layer-parity double buffer of the exchange relies on it).
        if (local && j < m.H) {
            const long long o = (static_cast<long long>(layer & 1) * K + i) * m.Hp + j;
            for (int p = 0; p < ctl.ep.world; ++p) __stcg(ctl.ep.xbuf[p] + o, acc);
        }
        __syncwarp();
        if (lane == 0) {
            __threadfence_system();
            if (atomicAdd(st.ep_arrive + layer, 1) == K * static_cast<int>(gridDim.x) - 1) {
                st.ep_arrive[layer] = 0;
                __threadfence_system();
                for (int p = 0; p < ctl.ep.world; ++p) atomicAdd_system(ctl.ep.cnt[p] + layer, 1);
            }
        }
        return;
    }
    down_block_epilogue(m, st, gts, layer, rb, i, acc);
    PHASE();
#ifdef SMOE_PHASES
    if (rb == 0 && lane == 0)
        phase_print("ffn_down(last) [pdl, ids+slot, stage, chain, y+fence+atomic, mix]", ph_, nph_);
#endif
}

#ifndef SMOE_DR_S
#define SMOE_DR_S 2
#endif
#ifndef SMOE_DR_CC
#define SMOE_DR_CC 128
#endif
using PipeDR = WarpPipe<uint16_t, SMOE_DR_S, SMOE_DR_CC>;  // k_ffn_down_rb: per-warp ring (2 x 8 KB)

// Tolerance-mode down projection, one GPU (the default when its shared memory
// fits: Q30 152 KB): CTA rb owns the 32-row block rb of
// ALL k executed experts (warp q: expert q's 48 KB tile through its own 2 x 8
// KB ring, primed before the PDL wait), so the mixture in decision order
// (model.cpp:297-301), the residual and the rms partial of x are formed in
// shared memory — no y round trip through global memory, no device-scope
// fence / arrival counter as k_ffn_down's last-of-k CTA needs.
__global__ void __launch_bounds__(32 * kMaxK) k_ffn_down_rb(DevModel m, DevState st, DevCtl ctl, int layer,
                                                           int exec_src) {
    KTRACE(10, layer);
    const int K = m.K, Hmp = m.Hmp, q = threadIdx.x >> 5, lane = threadIdx.x & 31, rb = blockIdx.x;
    const int j = rb * 32 + lane;
    __shared__ float ys[kMaxK][32];
    float* hs = reinterpret_cast<float*>(g_smem) + static_cast<long long>(q) * Hmp;  // [K][Hmp]
    unsigned char* pipe_mem = align128(reinterpret_cast<unsigned char*>(reinterpret_cast<float*>(g_smem) + K * Hmp)) +
                              q * round_up(PipeDR::kBytes, 128);
    const int* ids = (exec_src ? st.id_pred : st.id_exec) + layer * K;
    const float* gts = (exec_src ? st.g_pred : st.g_exec) + layer * K;
    // ids / slot_of are final once every gate/up CTA passed its copy wait (its PDL trigger)
    const int e = __ldcg(ids + q);
    const int slot = __ldcg(m.slot_of + layer * m.E + e);
    PipeDR pipe;
    pipe.init(pipe_mem, kL2EvictFirst);
    const uint16_t* tile = m.slots + (static_cast<long long>(layer) * m.C + slot) * m.expert_elems + m.gu_elems +
                           static_cast<long long>(rb) * Hmp * 32;
    if (slot >= 0) pipe.prime(tile, m.Hm);
    pdl_wait();
    KT_WAITED();
    pdl_trigger();
    if (__syncthreads_or(*(volatile int*)ctl.error)) return;
    if (slot < 0) {  // (per warp) report; the warp contributes 0 and the CTA finishes together
        if (lane == 0) atomicCAS(ctl.error, 0, 2000 + layer);
    }
    float gv = 0.0f, rv = 0.0f;
    if (q == 0) {
        if (lane < K) gv = __ldcg(gts + lane);
        if (j < m.H) rv = __ldcg(st.r + static_cast<long long>(layer) * m.Hp + j);
    }
    float y = 0.0f;
    if (slot >= 0) {
        // h (k_ffn_gu_cs's rows of expert q, L2-resident): 16-byte loads, all in flight
        const float4* h4 = reinterpret_cast<const float4*>(st.h + static_cast<long long>(q) * Hmp);
        for (int t0 = 0; t0 < Hmp / 4; t0 += 8 * 32) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int t = t0 + u * 32 + lane;
                if (t < Hmp / 4) v[u] = __ldcg(h4 + t);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int t = t0 + u * 32 + lane;
                if (t < Hmp / 4) reinterpret_cast<float4*>(hs)[t] = v[u];
            }
        }
        __syncwarp();
        y = SMOE_FAST(m) ? pipe.run_fast(tile, m.Hm, hs) : 0.0f;
        if (j < m.H) st.y[static_cast<long long>(q) * m.Hp + j] = y;
    }
    ys[q][lane] = y;
    __syncthreads();
    if (q != 0) return;
    float out = 0.0f;
    for (int k = 0; k < K; ++k) out += __shfl_sync(0xffffffffu, gv, k) * ys[k][lane];
    float xv = 0.0f;
    if (j < m.H) {
        st.m[static_cast<long long>(layer) * m.Hp + j] = out;
        xv = rv + out;
        st.x[j] = xv;
    }
    warp_ssq_partial(xv, st.ssq_x + static_cast<long long>(layer + 1) * (m.Hp / 32) + rb);
}

__global__ void __launch_bounds__(32) k_ffn_down(DevModel m, DevState st, DevCtl ctl, int layer,
                                                 int exec_src) {
    ffn_down_body(m, st, ctl, layer, exec_src, blockIdx.x, blockIdx.y, false, 0);
}

// The expert FFN of a layer in ONE launch (single GPU, when every CTA of the
// grid is co-resident — attn_grid-style occupancy check at session creation):
//
//  phase 1  CTA b = gate/up of (16-row block b % (Hmp/16), expert b / (Hmp/16))
//           exactly as k_ffn_gu, plus an L2 prefetch of its share of the
//           expert's down-projection block, so the down weights stream from
//           HBM while the gate/up chains run (one HBM pass over all 3·H·Hm
//           weights per expert);
//  phase 2  the CTAs that finished their gate/up claim down items (atomic
//           counter): a pair of 32-row blocks of one expert, primed from L2
//           into the same shared-memory pipe, started once that expert's
//           gate/up blocks are all done (gu_done, monotonic; target from the
//           per-layer launch epoch); two independent chains per lane
//           (run_pair), then the usual mixture epilogue.
//
// Every dot product is still one lane walking the reference's column order,
// so results equal the split kernels bit for bit.
__global__ void __launch_bounds__(32) k_ffn(DevModel m, DevState st, DevCtl ctl, int layer,
                                            int exec_src, int s_from_r) {
    KTRACE(15, layer);
    const int ngu_x = m.Hmp / 16, nrb = m.Hp / 32, npair = (nrb + 1) / 2, items = npair * m.K;
    const int epoch = __ldcg(st.ffn_epoch + layer);  // before this launch's last CTA bumps it
    const int b = blockIdx.x;
    ffn_gu_body(m, st, ctl, layer, exec_src, s_from_r, b % ngu_x, b / ngu_x, true);
    const int lane = threadIdx.x & 31;
    const int* ids = (exec_src ? st.id_pred : st.id_exec) + layer * m.K;
    const float* gts = (exec_src ? st.g_pred : st.g_exec) + layer * m.K;
    float* hs = reinterpret_cast<float*>(g_smem + 128);  // reuses the gate/up input staging
    unsigned char* pipe_mem = align128(reinterpret_cast<unsigned char*>(hs + 2 * round_up(m.H, 32)));
    const int target = (epoch + 1) * ngu_x;
    PHASE_DECL
    PHASE();
    for (;;) {
        int it = 0;
        if (lane == 0) it = atomicAdd(st.counters + 6, 1);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it >= items || *(volatile int*)ctl.error) break;
        const int i = it / npair, pr = it % npair, rb0 = 2 * pr, rb1 = 2 * pr + 1;
        const bool two = rb1 < nrb;
        const int e = __ldcg(ids + i);
        const int slot = __ldcg(m.slot_of + layer * m.E + e);
        if (slot < 0) {
            if (lane == 0) atomicCAS(ctl.error, 0, 2000 + layer);
            break;
        }
        const uint16_t* dn = m.slots + (static_cast<long long>(layer) * m.C + slot) * m.expert_elems + m.gu_elems;
        const uint16_t* ta = dn + static_cast<long long>(rb0) * m.Hmp * 32;
        const uint16_t* tb = dn + static_cast<long long>(two ? rb1 : rb0) * m.Hmp * 32;
        if (lane == 0) {  // this expert's h rows are complete
            const int* cnt = st.gu_done + layer * m.K + i;
            const long long t0 = clock64();
            for (;;) {
                int v;
                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
                if (v >= target || *(volatile int*)ctl.error) break;
                if (clock64() - t0 > ctl.spin_limit) {
                    atomicCAS(ctl.error, 0, 1000 + layer);
                    break;
                }
                __nanosleep(32);
            }
        }
        __syncwarp();
        if (*(volatile int*)ctl.error) break;
        PHASE();
        // h loads go out before the weight stream (they would queue behind it)
        const float4* h4 = reinterpret_cast<const float4*>(st.h + static_cast<long long>(i) * m.Hmp);
        constexpr int kHv = 8;
        float4 hv[kHv];
        const int nh4 = m.Hmp / 4;
#pragma unroll
        for (int u = 0; u < kHv; ++u) {
            const int t = u * 32 + lane;
            if (t < nh4) hv[u] = __ldcg(h4 + t);
        }
        // the gate/up phase's pipe is drained: fresh barriers for this item
        PipeGU pipe;
        pipe.init(pipe_mem, kL2EvictFirst);
        if (two)
            prime_pair(pipe, ta, tb, m.Hm);
        else
            pipe.prime(ta, m.Hm);
#pragma unroll
        for (int u = 0; u < kHv; ++u) {
            const int t = u * 32 + lane;
            if (t < nh4) reinterpret_cast<float4*>(hs)[t] = hv[u];
        }
        for (int t = kHv * 32 + lane; t < nh4; t += 32) reinterpret_cast<float4*>(hs)[t] = __ldcg(h4 + t);
        __syncwarp();
        PHASE();
        if (two) {
            float acc_a, acc_b;
            run_pair(pipe, ta, tb, m.Hm, hs, acc_a, acc_b);
            PHASE();
            down_block_epilogue(m, st, gts, layer, rb0, i, acc_a);
            down_block_epilogue(m, st, gts, layer, rb1, i, acc_b);
            PHASE();
        } else {
            const float acc = chain_run(pipe, m, ta, m.Hm, hs);
            down_block_epilogue(m, st, gts, layer, rb0, i, acc);
        }
    }
#ifdef SMOE_PHASES
    if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == 200))
        phase_print("ffn down phase [start->primed, gu_done wait, h stage, chain, epilogue]", ph_, nph_);
#endif
    if (last_cta(st.counters + 5, gridDim.x) && threadIdx.x == 0) {
        st.counters[6] = 0;  // every CTA has left its claim loop
        st.ffn_epoch[layer] = epoch + 1;
    }
}

// L2 prefetch of the experts a decision will execute (prefetch mode): issued on
// the side stream right after the predictor of layer l-1, it streams layer l's
// resident expert blocks (cache hits; misses are still in flight over PCIe and
// are skipped) into L2 while the attention of layer l runs, so the expert
// kernels of layer l read L2 instead of HBM.  grid (parts, K), one thread
// issues cp.async.bulk.prefetch.L2 (SASS UBLKPF) in 64 KB pieces.
__global__ void __launch_bounds__(32) k_l2_prefetch(DevModel m, DevState st, DevCtl ctl, int layer) {
    KTRACE(14, layer);
    pdl_wait();
    KT_WAITED();
    pdl_trigger();
    if (threadIdx.x != 0) return;
    const int i = blockIdx.y;
    const int e = __ldcg(st.id_pred + layer * m.K + i);
    if (ctl.ep.world > 1 && e % ctl.ep.world != ctl.ep.rank) return;
    const int slot = __ldcg(m.slot_of + layer * m.E + e);
    if (slot < 0) return;  // not resident yet (copy in flight)
    const char* base = reinterpret_cast<const char*>(
        m.slots + (static_cast<long long>(layer) * m.C + slot) * m.expert_elems);
    const long long bytes = m.expert_elems * 2;
    const long long part = ((bytes + gridDim.x - 1) / gridDim.x + 15) / 16 * 16;
    const long long b0 = part * blockIdx.x, b1 = min(bytes, b0 + part);
    for (long long o = b0; o < b1; o += 65536) {
        const uint32_t n = static_cast<uint32_t>(min(65536LL, b1 - o)) & ~15u;
        if (n) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + o), "r"(n) : "memory");
    }
}

// EP combine: wait until every rank's down-projection CTAs of this layer have
// published their rows (system-scope acquire on the arrival counter), then
// mix all k raw outputs in decision order (model.cpp:297-301) and add the
// residual — identical arithmetic to the single-GPU epilogue.
__global__ void __launch_bounds__(32) k_ep_mix(DevModel m, DevState st, DevCtl ctl, int layer,
                                               int exec_src) {
    KTRACE(11, layer);
    pdl_wait();
    KT_WAITED();
    pdl_trigger();  // after our own dependency: dependents launch at most one kernel ahead
    const int K = m.K, lane = threadIdx.x & 31, rb = blockIdx.x, j = rb * 32 + lane;
    __shared__ int s_ok;
    if (threadIdx.x == 0) {
        const long long target = (static_cast<long long>(ctl.ep.epoch[layer]) + 1) * ctl.ep.world;
        const int* cnt = ctl.ep.cnt[ctl.ep.rank] + layer;
        const long long t0 = clock64();
        int ok = 1;
        for (;;) {
            int v;
            asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
            if (v >= target) break;
            if (*(volatile int*)ctl.error || clock64() - t0 > ctl.spin_limit) {
                atomicCAS(ctl.error, 0, 3000 + layer);
                ok = 0;
                break;
            }
            __nanosleep(64);
        }
        s_ok = ok;
    }
    __syncthreads();
    float xv = 0.0f;
    if (s_ok && j < m.H) {
        const float* gts = (exec_src ? st.g_pred : st.g_exec) + layer * K;
        const float* xb = ctl.ep.xbuf[ctl.ep.rank] + static_cast<long long>(layer & 1) * K * m.Hp;
        float out = 0.0f;
        for (int i = 0; i < K; ++i) {
            const float y = __ldcv(xb + static_cast<long long>(i) * m.Hp + j);
            st.y[static_cast<long long>(i) * m.Hp + j] = y;
            out += gts[i] * y;
        }
        st.m[static_cast<long long>(layer) * m.Hp + j] = out;
        xv = st.r[static_cast<long long>(layer) * m.Hp + j] + out;
        st.x[j] = xv;
    }
    warp_ssq_partial(xv, st.ssq_x + static_cast<long long>(layer + 1) * (m.Hp / 32) + rb);
    if (!last_cta(st.counters + 3, gridDim.x)) return;
    if (threadIdx.x == 0) ctl.ep.epoch[layer] += 1;
}

// ------------------------------------------------------------ final / argmax --
// h = rms_norm(x, final_gain); logits = unembed . h (model.cpp:388-389);
// greedy argmax, first maximum (model.cpp:391-396).
__global__ void __launch_bounds__(32 * kSplitWarps) k_final(DevModel m, DevState st, DevCtl ctl,
                                              int record_token) {
    KTRACE(12, 0);
    uint64_t* bar = reinterpret_cast<uint64_t*>(g_smem);
    double* red = reinterpret_cast<double*>(g_smem + 64);
    float* xs = reinterpret_cast<float*>(g_smem + 128);
    float* gs = xs + round_up(m.H, 32);
    unsigned char* pipe_mem = align128(reinterpret_cast<unsigned char*>(gs + round_up(m.H, 32)));
    const uint16_t* tile = m.unemb + static_cast<long long>(blockIdx.x) * m.H * 32;
    PipeBL pipe;
    SplitG sp;
    if (SMOE_FAST(m)) {
        sp.prime(tile, m.H);
    } else {
        pipe.init(pipe_mem);
        pipe.prime(tile, m.H);
    }
    Stager sg;
    sg.init(bar);
    sg.add(gs, m.final_gain, m.H * 4);  // static: before the PDL wait
    pdl_wait();
    KT_WAITED();
    pdl_trigger();  // after our own dependency: dependents launch at most one kernel ahead
    sg.add(xs, st.x, m.H * 4);
    const float scale = rms_scale_from_partials(st.ssq_x + static_cast<long long>(m.L) * (m.Hp / 32),
                                                m.Hp / 32, m.H, m.eps);
    sg.wait();
    block_apply_norm(xs, gs, m.H, scale, xs);
    const int rb = blockIdx.x;
    const float acc = SMOE_FAST(m) ? sp.run(tile, m.H, xs, reinterpret_cast<float*>(pipe_mem)) : pipe.run(tile, m.H, xs);
    const int v = rb * 32 + (threadIdx.x & 31);
    if (threadIdx.x < 32 && v < m.V) st.logits[v] = acc;
    if (!last_cta(st.counters + 2, gridDim.x)) return;
    if (threadIdx.x >= 32) return;
    // argmax_token (model.cpp:391-396): first maximum, warp-parallel
    int best = -1;
    float bv = -INFINITY;
    for (int i = threadIdx.x; i < m.V; i += 32) {
        const float v = __ldcg(st.logits + i);
        if (best < 0 || v > bv) {
            bv = v;
            best = i;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, best, o);
        if (oi >= 0 && (best < 0 || ov > bv || (ov == bv && oi < best))) {
            bv = ov;
            best = oi;
        }
    }
    if (threadIdx.x == 0) {
        *st.token = best;
        *st.pos = *st.pos + 1;
        if (record_token) {
            const int s = *ctl.step;
            ctl.tokens_out[s] = best;
            *ctl.step = s + 1;
        }
    }
}

// ----------------------------------------------------------- calibration ----

// Marks every layer's predicted decision as published for the current pass
// (profiling the prefetch form of the expert kernels outside a decode pass).
__global__ void k_mark_decided(DevState st, int L) {
    const int p = __ldcg(st.pass_id);
    for (int l = threadIdx.x; l < L; l += blockDim.x) st.dec_ready[l] = p;
}

__global__ void k_dv_accum(DevModel m, DevState st, double* sums, long long* counts, int layer) {
    pdl_wait();
    pdl_trigger();  // after our own dependency: dependents launch at most one kernel ahead
    const int K = m.K, H = m.H;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < K * H; t += gridDim.x * blockDim.x) {
        const int i = t / H, j = t % H;
        const int e = st.id_exec[layer * K + i];
        sums[(static_cast<long long>(layer) * m.E + e) * H + j] += st.y[static_cast<long long>(i) * m.Hp + j];
        if (j == 0) counts[static_cast<long long>(layer) * m.E + e] += 1;
    }
}

__global__ void k_dv_freeze(const double* sums, const long long* counts, float* dv, long long LE,
                            int H) {
    const long long n = LE * H;
    for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < n;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long c = counts[t / H];
        dv[t] = c == 0 ? 0.0f : static_cast<float>(sums[t] / static_cast<double>(c));
    }
}

// ------------------------------------------------------------ exp check --
// y = exp_glibc(x) for the parity test of the device exp (tests/test_gpu.py)
__global__ void k_exp_glibc(const double* x, double* y, long long n) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        y[i] = exp_glibc(x[i]);
}

// make_decision of `rows` logits rows (diagnostics / tests): one warp per row
// through warp_decision, the routine every router, predictor and estimator
// decision on the path uses.
__global__ void __launch_bounds__(32) k_decide(const float* logits, int E, int K, int gating, int* ids,
                                               float* gates) {
    extern __shared__ __align__(16) unsigned char dsm[];
    float* sp = reinterpret_cast<float*>(dsm);
    double* se = reinterpret_cast<double*>(dsm + 16 * ((E * 4 + 15) / 16));
    const long long r = blockIdx.x;
    warp_decision(logits + r * E, E, K, gating, sp, se, ids + r * K, gates + r * K);
}

cudaError_t launch_decide(const float* logits, int rows, int E, int K, int gating, int* ids, float* gates,
                          cudaStream_t s) {
    const size_t sm = 16 * ((E * 4 + 15) / 16) + 8ull * E;
    k_decide<<<rows, 32, sm, s>>>(logits, E, K, gating, ids, gates);
    return cudaGetLastError();
}

cudaError_t launch_exp_glibc(const double* x, double* y, long long n, cudaStream_t s) {
    k_exp_glibc<<<148, 256, 0, s>>>(x, y, n);
    return cudaGetLastError();
}

// ---------------------------------------------------------- distill data --
// DistillDatasetBuilder::add_token (speculation.cpp:455-471) over captured
// trace steps: one CTA per (token, predicting layer l).  Input: quasi-hidden
// q_l = rms_norm(r_l + layer_default(exec_l), gain_{l+1}) (mode 0), or s_{l+1}
// (mode 1); target: the true router logits of layer l+1.  The rms scale uses
// the decode path's partial order (warp_ssq_partial / rms_scale_from_partials).
__global__ void __launch_bounds__(256) k_distill(DevModel m, TraceDev tr, int first, int mode, float* inputs,
                                                 float* targets) {
    double* part = reinterpret_cast<double*>(g_smem);  // [ceil(H/32)]
    __shared__ float scale_s;
    const int L = m.L, H = m.H, E = m.E, K = m.K, lp = L - 1;
    const long long smp = blockIdx.x;
    const long long t = first + smp / lp;
    const int l = static_cast<int>(smp % lp);
    float* out = inputs + smp * H;
    if (mode == 1) {
        const float* s = tr.s + (t * L + l + 1) * H;
        for (int j = threadIdx.x; j < H; j += blockDim.x) out[j] = s[j];
    } else {
        const float* r = tr.r + (t * L + l) * H;
        const int* ids = tr.id_exec + (t * L + l) * K;
        const float* gts = tr.g_exec + (t * L + l) * K;
        const int nb = (H + 31) / 32;
        for (int rb = threadIdx.x >> 5; rb < nb; rb += blockDim.x >> 5) {
            const int j = rb * 32 + (threadIdx.x & 31);
            const float rd = j < H ? r[j] + layer_default_row(m, ids, gts, l, j) : 0.0f;
            if (j < H) out[j] = rd;
            warp_ssq_partial(rd, part + rb);
        }
        __syncthreads();
        if (threadIdx.x < 32) {  // rms_scale_from_partials' order over smem
            double v = 0.0;
            for (int i = threadIdx.x; i < nb; i += 32) v += part[i];
            for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
            if (threadIdx.x == 0)
                scale_s = static_cast<float>(1.0 / sqrt(v / static_cast<double>(H) + static_cast<double>(m.eps)));
        }
        __syncthreads();
        const float sc = scale_s;
        const float* gain = m.moe_gain + static_cast<long long>(l + 1) * H;
        for (int j = threadIdx.x; j < H; j += blockDim.x) out[j] = (out[j] * sc) * gain[j];
    }
    const float* lg = tr.lg_true + (t * L + l + 1) * E;
    for (int e = threadIdx.x; e < E; e += blockDim.x) targets[smp * E + e] = lg[e];
}

// Router-pf prediction `depth` layers ahead over captured steps (SURVEY §8f
// row 4): q = rms_norm(r_l + layer_default(exec_l), gain_{l+depth}), logits =
// gate_{l+depth} . q (sequential chains), top-k ids (value desc, index asc).
// depth 1 is the paper's router-pf (speculation.cpp:206-228).  One CTA per
// (token, l); writes ids of layer l+depth.
__global__ void __launch_bounds__(256) k_pred_ahead(DevModel m, TraceDev tr, int first, int depth, int* out) {
    const int L = m.L, H = m.H, E = m.E, K = m.K, nl = L - depth;
    const long long smp = blockIdx.x;
    const long long t = first + smp / nl;
    const int l = static_cast<int>(smp % nl), tl = l + depth;
    const int nb = (H + 31) / 32;
    double* part = reinterpret_cast<double*>(g_smem);
    float* q = reinterpret_cast<float*>(g_smem + round_up(nb, 2) * 8);
    float* lg = q + round_up(H, 4);
    __shared__ float scale_s;
    const float* r = tr.r + (t * L + l) * H;
    const int* ids = tr.id_exec + (t * L + l) * K;
    const float* gts = tr.g_exec + (t * L + l) * K;
    for (int rb = threadIdx.x >> 5; rb < nb; rb += blockDim.x >> 5) {
        const int j = rb * 32 + (threadIdx.x & 31);
        const float rd = j < H ? r[j] + layer_default_row(m, ids, gts, l, j) : 0.0f;
        if (j < H) q[j] = rd;
        warp_ssq_partial(rd, part + rb);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = 0.0;
        for (int i = threadIdx.x; i < nb; i += 32) v += part[i];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0)
            scale_s = static_cast<float>(1.0 / sqrt(v / static_cast<double>(H) + static_cast<double>(m.eps)));
    }
    __syncthreads();
    const float* gain = m.moe_gain + static_cast<long long>(tl) * H;
    for (int j = threadIdx.x; j < H; j += blockDim.x) q[j] = (q[j] * scale_s) * gain[j];
    __syncthreads();
    const uint16_t* g = m.gate + tl * m.gate_stride;
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        // row tile layout (k_gen_bf16): [E/32][H/8][32 rows][8 cols]
        const uint16_t* row = g + static_cast<long long>(e / 32) * H * 32 + (e % 32) * 8;
        float acc = 0.0f;
        for (int j = 0; j < H; ++j)
            acc = acc + __uint_as_float(static_cast<uint32_t>(row[(j >> 3) * 256 + (j & 7)]) << 16) * q[j];
        lg[e] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int* o = out + (t - first) * static_cast<long long>(L) * K + static_cast<long long>(tl) * K;
        for (int i = 0; i < K; ++i) {
            int best = -1;
            for (int e = 0; e < E; ++e) {
                bool taken = false;
                for (int p = 0; p < i; ++p) taken |= o[p] == e;
                if (taken) continue;
                if (best < 0 || lg[e] > lg[best]) best = e;
            }
            o[i] = best;
        }
    }
}

// ------------------------------------------------------ packed experts ----
// section offsets of a packed block (mirror of engine.h's xp_off_*)
__device__ __forceinline__ long long xp_off_sec_d(long long n) { return 32 + n / 4 + (4 * (n / 256) + 15) / 16 * 16; }
__device__ __forceinline__ long long xp_off_sm_d(long long n, long long nsec) {
    return xp_off_sec_d(n) + ((nsec + 1) / 2 + 15) / 16 * 16;
}

// Decoder of the xp11 expert block (engine.h, xpack.cpp): one warp per
// 256-weight group, lane l expands weights 8l..8l+7 — one 2-byte load of its
// primary codes, a warp scan of its secondary-code count (offset into the
// group's secondary stream, whose start the block's group table holds), its
// secondary nibbles, one 8-byte load of sign|mantissa bytes and one 16-byte
// store; an escaped weight takes its raw value from the ascending escape list
// (binary search; ~1e-4 of Gaussian weights).  HBM-bound: ~1.4 B read + 2 B
// written per weight, a few µs per 9.4 MB Q30 expert beside a ~120 µs H2D.
__global__ void __launch_bounds__(256) k_xp_unpack(const uint8_t* __restrict__ src, uint16_t* __restrict__ dst) {
    const uint32_t* hdr = reinterpret_cast<const uint32_t*>(src);
    const uint32_t ngroups = __ldg(hdr + 1), nsec = __ldg(hdr + 2), nesc = __ldg(hdr + 3);
    const uint32_t g = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (g >= ngroups) return;
    const uint32_t p0 = __ldg(hdr + 4), p1 = __ldg(hdr + 5), p2 = __ldg(hdr + 6), base = __ldg(hdr + 7);
    const long long n = static_cast<long long>(ngroups) * 256;
    const uint8_t* sc = src + xp_off_sec_d(n);
    const uint8_t* sm = src + xp_off_sm_d(n, nsec);
    const uint8_t* esc = sm + n;
    const uint32_t c16 = __ldg(reinterpret_cast<const unsigned short*>(src + 32 + static_cast<long long>(g) * 64) + lane);
    const int cnt = __popc(c16 & (c16 >> 1) & 0x5555u);  // codes == 3: secondary follows
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (static_cast<int>(lane) >= o) incl += t;
    }
    uint32_t k = __ldg(reinterpret_cast<const uint32_t*>(src + 32 + n / 4) + g) + (incl - cnt);
    const uint2 b = __ldcs(reinterpret_cast<const uint2*>(sm + static_cast<long long>(g) * 256) + lane);
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint32_t c = (c16 >> (2 * j)) & 3u;
        uint32_t e = c == 0 ? p0 : (c == 1 ? p1 : p2);
        bool escaped = false;
        if (c == 3u) {
            const uint32_t s2 = (__ldg(sc + (k >> 1)) >> (4 * (k & 1))) & 15u;
            ++k;
            e = base + s2;
            escaped = s2 == 15u;
        }
        const uint32_t byte = ((j < 4 ? b.x : b.y) >> (8 * (j & 3))) & 0xffu;
        uint32_t v = ((byte & 0x80u) << 8) | ((e & 0xffu) << 7) | (byte & 0x7fu);
        if (escaped) {  // raw value from the list (ascending indices)
            const uint32_t idx = static_cast<uint32_t>(g * 256 + lane * 8 + j);
            uint32_t lo = 0, hi = nesc;
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (__ldg(reinterpret_cast<const uint32_t*>(esc + 8ull * mid)) < idx) lo = mid + 1;
                else hi = mid;
            }
            v = __ldg(reinterpret_cast<const uint16_t*>(esc + 8ull * lo + 4));
        }
        if (j & 1) w[j >> 1] |= v << 16;
        else w[j >> 1] = v;
    }
    reinterpret_cast<uint4*>(dst + static_cast<long long>(g) * 256)[lane] = make_uint4(w[0], w[1], w[2], w[3]);
}

std::atomic<long long> g_xp_launches{0};  // copy-lane launches (outside the decode graphs)
long long xp_unpack_launches() { return g_xp_launches.load(); }

cudaError_t launch_xp_unpack(const uint8_t* src, uint16_t* dst, long long n, cudaStream_t s) {
    const long long groups = n / 256;
    k_xp_unpack<<<static_cast<unsigned>((groups + 7) / 8), 256, 0, s>>>(src, dst);
    ++g_xp_launches;
    return cudaGetLastError();
}

cudaError_t launch_pred_ahead(const DevModel& m, const TraceDev& tr, int first, int n, int depth, int* out,
                              cudaStream_t s) {
    const int nb = (m.H + 31) / 32;
    const size_t smem = round_up(nb, 2) * 8 + (round_up(m.H, 4) + m.E) * 4;
    k_pred_ahead<<<n * (m.L - depth), 256, smem, s>>>(m, tr, first, depth, out);
    return cudaGetLastError();
}

cudaError_t launch_distill(const DevModel& m, const TraceDev& tr, int first, int n, int mode, float* inputs,
                           float* targets, cudaStream_t s) {
    k_distill<<<n * (m.L - 1), 256, (m.H + 31) / 32 * 8, s>>>(m, tr, first, mode, inputs, targets);
    return cudaGetLastError();
}

// ----------------------------------------------------------------- trace ----

__global__ void k_trace(DevModel m, DevState st, TraceDev tr) {
    pdl_wait();
    pdl_trigger();  // after our own dependency: dependents launch at most one kernel ahead
    const int step = *tr.step;
    if (step >= tr.cap) return;
    const int L = m.L, H = m.H, E = m.E, K = m.K, V = m.V, Hp = m.Hp;
    const long long t0 = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (t0 == 0) tr.tok_in[step] = *st.tok_in;
    const long long gs = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long t = t0; t < static_cast<long long>(L) * K; t += gs) {
        const long long o = static_cast<long long>(step) * L * K + t;
        tr.id_true[o] = st.id_true[t];
        tr.id_exec[o] = st.id_exec[t];
        tr.id_pred[o] = st.id_pred[t];
        if (tr.full) {
            tr.g_true[o] = st.g_true[t];
            tr.g_exec[o] = st.g_exec[t];
            tr.g_pred[o] = st.g_pred[t];
        }
    }
    if (!tr.full) {
        __syncthreads();
        if (t0 == 0) *tr.step = step + 1;  // single CTA launch in ids-only mode
        return;
    }
    for (long long t = t0; t < static_cast<long long>(L) * H; t += gs) {
        const long long l = t / H, j = t % H;
        const long long o = static_cast<long long>(step) * L * H + t;
        tr.s[o] = st.s[l * Hp + j];
        tr.r[o] = st.r[l * Hp + j];
        tr.m[o] = st.m[l * Hp + j];
    }
    for (long long t = t0; t < static_cast<long long>(L) * E; t += gs) {
        const long long o = static_cast<long long>(step) * L * E + t;
        tr.lg_true[o] = st.lg_true[t];
        tr.lg_pred[o] = st.lg_pred[t];
    }
    for (long long t = t0; t < V; t += gs) tr.logits[static_cast<long long>(step) * V + t] = st.logits[t];
}

// Per-layer raw outputs are overwritten by the next layer, so the full trace
// grabs them right after each layer's down projection.
__global__ void k_trace_y(DevModel m, DevState st, TraceDev tr, int layer) {
    pdl_wait();
    pdl_trigger();  // after our own dependency: dependents launch at most one kernel ahead
    const int step = *tr.step;
    if (step >= tr.cap) return;
    const int K = m.K, H = m.H, L = m.L;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < K * H; t += gridDim.x * blockDim.x) {
        const int i = t / H, j = t % H;
        tr.y[((static_cast<long long>(step) * L + layer) * K + i) * H + j] = st.y[static_cast<long long>(i) * m.Hp + j];
    }
}

__global__ void k_trace_bump(TraceDev tr) {
    pdl_wait();
    if (*tr.step < tr.cap) *tr.step = *tr.step + 1;
}

// ============================================================== launchers ==

static long long g_launches = 0;

long long launch_counter() { return g_launches; }

static inline cudaError_t counted(int n = 1) {
    g_launches += n;
    return cudaGetLastError();
}

namespace {
inline int gen_blocks(long long n) {
    long long b = (n + 255) / 256;
    if (b > 148LL * 64) b = 148LL * 64;
    return static_cast<int>(b < 1 ? 1 : b);
}
size_t vec_bytes(int n) { return static_cast<size_t>(round_up(n, 32)) * 4; }
size_t qkv_smem(const DevModel& m) { return 128 + 2 * vec_bytes(m.H) + 128 + PipeBL::kBytes; }
size_t wo_smem(const DevModel&) { return 128 + kMaxD * 4 + 32 * 4 + 128 + PipeB::kBytes; }
// Router CTAs stay small enough (Q30: ~72 KB with q_l from k_wo) to co-reside
// with three k_ffn_gu CTAs, so the side-stream router never waits for SM space.
size_t router_smem(const DevModel& m, int needs_dv) {
    const size_t head = 256 + (3 + (needs_dv ? static_cast<size_t>(m.K) : 0)) * vec_bytes(m.H) + 128;
    // fast mode: no weight pipe (SplitLdg), only the warps' partial sums
    const size_t body = m.fast ? kRouterSplitWarps * 32 * 4 : PipeR::kBytes;
    return head + (body > kMaxE * 12 ? body : kMaxE * 12);
}
size_t est_smem(const DevModel& m) {
    int cols = m.est_d > m.est_mlp ? m.est_d : m.est_mlp;
    return vec_bytes(cols) + 64 + 128 + (PipeF::kBytes > kMaxE * 12 ? PipeF::kBytes : kMaxE * 12);
}
size_t gu_smem(const DevModel& m) { return 128 + vec_bytes(m.H) + 128 + PipeGU::kBytes; }
constexpr int kGuWarps = 1;
size_t gu_w_smem(const DevModel& m, int w) {
    return 128 + vec_bytes(m.H) + 128 + static_cast<size_t>(w) * round_up(PipeGU::kBytes, 128);
}
// warps per gate/up CTA (SMOE_GU_WARPS: 1 = k_ffn_gu, 2/3/4 = k_ffn_gu_w<W>)
int gu_warps() {
    static const int w = std::getenv("SMOE_GU_WARPS") ? std::atoi(std::getenv("SMOE_GU_WARPS")) : kGuWarps;
    return w >= 1 && w <= 4 ? w : 1;
}
size_t gu_cs_smem(const DevModel& m) {  // also k_ffn_cs: the staging holds s (H) or h (Hmp)
    return 128 + kCsWarps * 32 * 4 + vec_bytes(m.H > m.Hmp ? m.H : m.Hmp) + 128 +
           kCsWarps * round_up(PipeCs::kBytes, 128);
}
cudaError_t launch_gu(const DevModel& m, const DevState& st, const DevCtl& ctl, int layer, int exec_src,
                      int s_from_r, cudaStream_t s) {
    const int w = gu_warps(), nt = m.Hmp / 16;
    if (m.fast) {  // tolerance mode: column-split warps
        PDL(k_ffn_gu_cs, dim3(nt, m.K), 32 * kCsWarps, gu_cs_smem(m), s, m, st, ctl, layer, exec_src, s_from_r);
        return cudaSuccess;
    }
    switch (w) {
    case 2: PDL(k_ffn_gu_w<2>, dim3((nt + 1) / 2, m.K), 64, gu_w_smem(m, 2), s, m, st, ctl, layer, exec_src, s_from_r); break;
    case 3: PDL(k_ffn_gu_w<3>, dim3((nt + 2) / 3, m.K), 96, gu_w_smem(m, 3), s, m, st, ctl, layer, exec_src, s_from_r); break;
    case 4: PDL(k_ffn_gu_w<4>, dim3((nt + 3) / 4, m.K), 128, gu_w_smem(m, 4), s, m, st, ctl, layer, exec_src, s_from_r); break;
    default: PDL(k_ffn_gu, dim3(nt, m.K), 32, gu_smem(m), s, m, st, ctl, layer, exec_src, s_from_r);
    }
    return cudaSuccess;
}
size_t ffn_smem(const DevModel& m) { return 128 + 2 * vec_bytes(m.H) + 128 + PipeGU::kBytes; }
size_t down_smem(const DevModel& m) { return 128 + static_cast<size_t>(m.Hmp) * 4 + 128 + PipeD::kBytes; }
size_t down_rb_smem(const DevModel& m) {
    return static_cast<size_t>(m.K) * m.Hmp * 4 + 128 + static_cast<size_t>(m.K) * round_up(PipeDR::kBytes, 128);
}
size_t final_smem(const DevModel& m) { return 128 + 2 * vec_bytes(m.H) + 128 + PipeBL::kBytes; }
size_t attn_smem(const DevModel& m) {
    size_t b = 256 + kMaxD * 4 + 2ull * kAttnChunk * (2 * m.D + 4) * 4;
    if (m.cap <= kAttnSmemPositions) b += static_cast<size_t>(m.cap) * 12;
    return b;
}

cudaError_t set_smem(const void* fn, size_t bytes) {
    return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(bytes));
}
}  // namespace

// Per-kernel dynamic shared-memory needs against the limits preload_kernels
// sets; a config whose kernels cannot launch is rejected at session creation
// with the kernel named (instead of an opaque launch failure at first decode).
std::string kernel_limit_violation(const DevModel& m) {
    struct Need {
        const char* name;
        size_t bytes, limit;
    } v[] = {{"k_qkv", qkv_smem(m), 200 * 1024},     {"k_wo", wo_smem(m), 200 * 1024},
             {"k_router", router_smem(m, 0), 200 * 1024}, {"k_ffn_gu", gu_w_smem(m, gu_warps()), (gu_warps() > 1 ? 227u : 200u) * 1024},
             {"k_ffn_down", down_smem(m), 220 * 1024}, {"k_final", final_smem(m), 200 * 1024},
             {"k_ffn_gu_cs", gu_cs_smem(m), 200 * 1024},
             {"k_attn", attn_smem(m), 220 * 1024}};
    for (const Need& n : v)
        if (n.bytes > n.limit)
            return std::string(n.name) + " needs " + std::to_string(n.bytes / 1024) +
                   " KB of shared memory (limit " + std::to_string(n.limit / 1024) +
                   " KB): hidden / head_dim / top_k / max_positions too large for this path";
    return std::string();
}
std::string estimator_limit_violation(const DevModel& m) {
    if (est_smem(m) > 200 * 1024)
        return "k_est_stage needs " + std::to_string(est_smem(m) / 1024) +
               " KB of shared memory (limit 200 KB): estimator d / mlp too large";
    return std::string();
}

// CTAs of the split decode attention that can be co-resident on `device`:
// kAttnSplit when occupancy x SMs allows it, else 1 (single-CTA path).
int attn_grid_for(const DevModel& m, int device) {
    int nb = 0, sms = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_attn, kAttnThreads, attn_smem(m)) != cudaSuccess)
        return 1;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 1;
    return static_cast<long long>(nb) * sms >= kAttnSplit ? kAttnSplit : 1;
}

// The fused expert kernel needs every CTA of its grid co-resident (phase-2
// CTAs wait on phase-1 CTAs of the same grid), room for the side-stream
// predictor CTAs beside it, and h (Hmp floats) inside the input staging.
int ffn_fused_ok(const DevModel& m, int device) {
    int nb = 0, sms = 0;
    if (m.Hmp > 2 * round_up(m.H, 32)) return 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_ffn, 32, ffn_smem(m)) != cudaSuccess) return 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 0;
    const long long grid = static_cast<long long>(m.Hmp / 16) * m.K;
    return grid + 16 <= static_cast<long long>(nb) * sms ? 1 : 0;
}

// k_ffn_cs: every CTA co-resident (claimed down items wait on gate/up units
// of the same grid), with room left for the side-stream predictor CTAs.
// Opt-in (SMOE_FFN_CS_FUSED=1): measured slower than k_ffn_gu_cs + k_ffn_down
// on Q30 (22.2 vs 18.5 us per layer, tools/kbench.py): a claimed down item
// waits for the slowest gate/up tile of its expert, and one CTA streams a
// 48 KB down tile that 4 one-warp k_ffn_down CTAs on 4 SMs would share.
int ffn_cs_fused_ok(const DevModel& m, int device) {
    if (!std::getenv("SMOE_FFN_CS_FUSED")) return 0;
    int nb = 0, sms = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_ffn_cs, 32 * kCsWarps, gu_cs_smem(m)) != cudaSuccess)
        return 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 0;
    const long long grid = static_cast<long long>(m.Hmp / 16) * m.K;
    return grid + 16 <= static_cast<long long>(nb) * sms ? 1 : 0;
}

int down_rb_ok(const DevModel& m) { return m.K <= kMaxK && down_rb_smem(m) <= 224 * 1024 ? 1 : 0; }

int max_dynamic_smem_needed(const DevModel& m) {
    size_t v[] = {qkv_smem(m), wo_smem(m), router_smem(m, 0), est_smem(m), ffn_smem(m), down_smem(m),
                  final_smem(m), attn_smem(m)};
    size_t mx = 0;
    for (size_t x : v) mx = x > mx ? x : mx;
    return static_cast<int>(mx);
}

cudaError_t launch_gen_bf16(uint64_t seed, float stddev, int R, int C, int tile_cols, int layout,
                            int which, int row_off, uint16_t* out, cudaStream_t s) {
    // total destination elements covered by this call
    long long total;
    if (layout == kRowMajor) {
        total = static_cast<long long>(R) * C;
    } else if (layout == kRowTiled) {
        total = static_cast<long long>(round_up(R + row_off, 32)) * tile_cols;
    } else {
        total = static_cast<long long>(round_up(2 * R, 32)) * tile_cols;
    }
    k_gen_bf16<<<gen_blocks(total), 256, 0, s>>>(seed, static_cast<double>(stddev), R, C,
                                                  tile_cols, layout, which, row_off, total, out);
    return counted(1);
}

cudaError_t launch_embed(const DevModel& m, const DevState& st, const int* token_src,
                         cudaStream_t s, const int* stream, const int* step) {
    PDL(k_embed, m.Hp / 32, 32, 0, s, m, st, token_src, stream, step);
    return counted(1);
}

// Loads every kernel up front.  With CUDA lazy loading, the first launch of
// a not-yet-loaded kernel synchronises the context; if that happens while an
// expert kernel spins on a copy-ready flag the copy thread's API calls block
// behind it (observed deadlock).  Session construction calls this once.
cudaError_t preload_kernels() {
    {
        const int v = std::getenv("SMOE_DOWN_L2") ? 1 : 0;
        cudaError_t e = cudaMemcpyToSymbol(g_down_l2_dev, &v, sizeof v);
        if (e != cudaSuccess) return e;
        const int f = std::getenv("SMOE_FUSED_NO_L2PF") ? 0 : 1;
        e = cudaMemcpyToSymbol(g_fused_l2_dev, &f, sizeof f);
        if (e != cudaSuccess) return e;
    }
    const void* fns[] = {(const void*)k_gen_bf16, (const void*)k_embed, (const void*)k_qkv,
                         (const void*)k_attn, (const void*)k_wo, (const void*)k_router,
                         (const void*)k_est_stage, (const void*)k_ffn_gu, (const void*)k_ffn_down,
                         (const void*)k_final, (const void*)k_dv_accum, (const void*)k_dv_freeze,
                         (const void*)k_trace, (const void*)k_trace_y, (const void*)k_trace_bump,
                         (const void*)k_ep_mix, (const void*)k_quasi_rd, (const void*)k_l2_prefetch,
                         (const void*)k_ffn, (const void*)k_ffn_gu_w<2>, (const void*)k_ffn_gu_w<3>,
                         (const void*)k_ffn_gu_w<4>, (const void*)k_attn_fast, (const void*)k_ffn_gu_cs,
                         (const void*)k_ffn_gud, (const void*)k_down_reduce, (const void*)k_ffn_down_rb,
                         (const void*)k_xp_unpack, (const void*)k_ffn_cs};
    for (const void* f : fns) {
        cudaFuncAttributes a;
        cudaError_t e = cudaFuncGetAttributes(&a, f);
        if (e != cudaSuccess) return e;
        // Maximum shared-memory carveout for every kernel: the SM's L1/smem
        // split is chosen per kernel, and a kernel sized by its own needs
        // leaves no room for the CTAs of concurrent kernels (the side-stream
        // predictor, a PDL-launched dependent prefetching its weights).
        e = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return e;
    }
    cudaError_t e = cudaSuccess;
    const void* big[] = {(const void*)k_qkv, (const void*)k_wo, (const void*)k_router,
                         (const void*)k_est_stage, (const void*)k_ffn_gu, (const void*)k_final};
    for (const void* f : big)
        if ((e = set_smem(f, 200 * 1024)) != cudaSuccess) return e;
    const void* gu_w[] = {(const void*)k_ffn_gu_w<2>, (const void*)k_ffn_gu_w<3>, (const void*)k_ffn_gu_w<4>};
    for (const void* f : gu_w)
        if ((e = set_smem(f, 227 * 1024)) != cudaSuccess) return e;
    if ((e = set_smem((const void*)k_attn, 220 * 1024)) != cudaSuccess) return e;
    if ((e = set_smem((const void*)k_attn_fast, 200 * 1024)) != cudaSuccess) return e;
    if ((e = set_smem((const void*)k_ffn, 200 * 1024)) != cudaSuccess) return e;
    if ((e = set_smem((const void*)k_ffn_gu_cs, 200 * 1024)) != cudaSuccess) return e;
    if ((e = set_smem((const void*)k_ffn_gud, 200 * 1024)) != cudaSuccess) return e;
    if ((e = set_smem((const void*)k_ffn_down_rb, 224 * 1024)) != cudaSuccess) return e;
    if ((e = set_smem((const void*)k_ffn_cs, 200 * 1024)) != cudaSuccess) return e;
    return set_smem((const void*)k_ffn_down, 220 * 1024);
}

cudaError_t launch_qkv(const DevModel& m, const DevState& st, int layer, cudaStream_t s) {
    PDL(k_qkv, m.QKVp / 32, m.fast ? 32 * kSplitWarps : 32, qkv_smem(m), s, m, st, layer);
    return counted(1);
}

cudaError_t launch_attn(const DevModel& m, const DevState& st, double* scratch, int layer,
                        cudaStream_t s) {
    if (attn_fast_ok(m)) {  // tolerance mode: flash-decoding split over positions
        const int gcap = static_cast<int>(std::min<long long>(kAttnFastCtas, std::max(1, m.cap / kAttnFastChunk)));
        const int g = m.attn_fast_grid > 0 ? std::min(m.attn_fast_grid, gcap) : gcap;
        PDL(k_attn_fast, g, kAttnFastThreads, attn_fast_smem(m), s, m, st, scratch, layer);
        return counted(1);
    }
    static const int split = std::getenv("SMOE_ATTN_SPLIT") ? std::atoi(std::getenv("SMOE_ATTN_SPLIT")) : 1;
    PDL(k_attn, split && m.attn_grid > 1 ? m.attn_grid : 1, kAttnThreads, attn_smem(m), s, m, st, scratch, layer);
    return counted(1);
}

cudaError_t launch_l2_prefetch(const DevModel& m, const DevState& st, const DevCtl& ctl, int layer,
                               cudaStream_t s) {
    PDL(k_l2_prefetch, dim3(16, m.K), 32, 0, s, m, st, ctl, layer);
    return counted(1);
}

cudaError_t launch_quasi_rd(const DevModel& m, const DevState& st, int layer, cudaStream_t s) {
    PDL(k_quasi_rd, m.Hp / 32, 32, 0, s, m, st, layer);
    return counted(1);
}

cudaError_t launch_wo(const DevModel& m, const DevState& st, const DevCtl& ctl, int layer,
                      cudaStream_t s, int rd_from_pred) {
    PDL(k_wo, m.Hp / 32, 32, wo_smem(m), s, m, st, ctl, layer, rd_from_pred);
    return counted(1);
}

cudaError_t launch_router(const DevModel& m, const DevState& st, const DevCtl& ctl,
                          const RouterLaunch& rl, const DevState* shadow, cudaStream_t s) {
    const int nT = rl.do_true ? m.Ep / 32 : 0;
    const bool gemv_pred = rl.pred_kind == kBaselineS || rl.pred_kind == kRouterPF;
    const int nP = gemv_pred ? m.Ep / 32 : 0;
    const int nQ = rl.pred_kind == kEstPF ? 1 : 0;
    int grid = nT + nP + nQ;
    if (grid < 1) grid = 1;
    DevState sh = shadow ? *shadow : st;
    const int needs_dv = (rl.pred_kind == kRouterPF || rl.pred_kind == kEstPF) && !rl.quasi_ready;
    if (router_smem(m, needs_dv) > 200 * 1024) return cudaErrorInvalidConfiguration;
    PDL(k_router, grid, m.fast ? 32 * kRouterSplitWarps : 32, router_smem(m, needs_dv), s, m, st, ctl, rl, sh,
        shadow ? 1 : 0);
    return counted(1);
}

cudaError_t launch_log_routers(const DevModel& m, const DevState& st, const DevCtl& ctl, int l0,
                               int nl, int step_tag, cudaStream_t s) {
    RouterLaunch rl{l0, 1, kNone, -1, 0, 0, step_tag, 0};
    PDL(k_router, dim3(m.Ep / 32, nl), m.fast ? 32 * kRouterSplitWarps : 32, router_smem(m, 0), s, m, st, ctl, rl,
        st, 0);
    return counted(1);
}

cudaError_t launch_estimator(const DevModel& m, const DevState& st, const DevCtl& ctl, int layer,
                             int post_pred, int step_tag, cudaStream_t s) {
    const size_t sm = est_smem(m);
    PDL(k_est_stage, round_up(m.est_dm, 32) / 32, 32, sm, s, m, st, ctl, layer, 0, 0, step_tag);
    PDL(k_est_stage, round_up(m.est_mlp, 32) / 32, 32, sm, s, m, st, ctl, layer, 1, 0, step_tag);
    PDL(k_est_stage, round_up(m.est_dm, 32) / 32, 32, sm, s, m, st, ctl, layer, 2, 0, step_tag);
    PDL(k_est_stage, m.Ep / 32, 32, sm, s, m, st, ctl, layer, 3, post_pred, step_tag);
    return counted(4);
}

cudaError_t launch_ffn(const DevModel& m, const DevState& st, const DevCtl& ctl, int layer,
                       cudaStream_t s, int exec_src, int s_from_r) {
    if (ctl.ep.world == 1 && m.fast && m.ffn_gud) {  // tolerance mode, one GPU (k_ffn_gud)
        PDL(k_ffn_gud, dim3(m.Hmp / 16, m.K), 32 * kCsWarps, gu_cs_smem(m), s, m, st, ctl, layer, exec_src, s_from_r);
        PDL(k_down_reduce, m.Hp / 32, 32 * m.K, 0, s, m, st, ctl, layer, exec_src);
        return counted(2);
    }
    if (ctl.ep.world == 1 && m.fast && m.ffn_cs_fused) {  // tolerance mode: one launch per layer
        PDL(k_ffn_cs, (m.Hmp / 16) * m.K, 32 * kCsWarps, gu_cs_smem(m), s, m, st, ctl, layer, exec_src, s_from_r);
        return counted(1);
    }
    if (ctl.ep.world == 1 && m.ffn_fused) {
        PDL(k_ffn, (m.Hmp / 16) * m.K, 32, ffn_smem(m), s, m, st, ctl, layer, exec_src, s_from_r);
        return counted(1);
    }
    {
        const cudaError_t e = launch_gu(m, st, ctl, layer, exec_src, s_from_r, s);
        if (e != cudaSuccess) return e;
    }
    if (ctl.ep.world == 1 && m.fast && m.down_rb) {
        PDL(k_ffn_down_rb, m.Hp / 32, 32 * m.K, down_rb_smem(m), s, m, st, ctl, layer, exec_src);
        return counted(2);
    }
    PDL(k_ffn_down, dim3(m.Hp / 32, m.K), 32, down_smem(m), s, m, st, ctl, layer, exec_src);
    if (ctl.ep.world > 1) {
        PDL(k_ep_mix, m.Hp / 32, 32, 0, s, m, st, ctl, layer, exec_src);
        g_launches += 1;
    }
    return counted(2);
}

// Per-kernel timing (Session::profile_kernels): part 0 = k_ffn_gu as on-demand
// launches it (decision from this layer's router: PDL wait first), 2 = as the
// prefetch path launches it for layers >= 1 (decision published a layer ahead:
// slot lookup and weight stream start before the PDL wait; the flags are set
// by k_mark_decided), 1 = k_ffn_down.
cudaError_t launch_ffn_part(const DevModel& m, const DevState& st, const DevCtl& ctl, int layer,
                            int part, cudaStream_t s) {
    if (part == 0 || part == 2) {
        const cudaError_t e = launch_gu(m, st, ctl, layer, part == 2, part == 2, s);
        if (e != cudaSuccess) return e;
    } else if (ctl.ep.world == 1 && m.fast && m.down_rb) {
        PDL(k_ffn_down_rb, m.Hp / 32, 32 * m.K, down_rb_smem(m), s, m, st, ctl, layer, 0);
    } else {
        PDL(k_ffn_down, dim3(m.Hp / 32, m.K), 32, down_smem(m), s, m, st, ctl, layer, 0);
    }
    return counted(1);
}

cudaError_t launch_mark_decided(const DevState& st, int L, cudaStream_t s) {
    k_mark_decided<<<1, 64, 0, s>>>(st, L);
    return counted(1);
}

cudaError_t launch_final(const DevModel& m, const DevState& st, const DevCtl& ctl,
                         int record_token, cudaStream_t s) {
    PDL(k_final, m.Vp / 32, m.fast ? 32 * kSplitWarps : 32, final_smem(m), s, m, st, ctl, record_token);
    return counted(1);
}

cudaError_t launch_dv_accum(const DevModel& m, const DevState& st, double* sums,
                            long long* counts, int layer, cudaStream_t s) {
    PDL(k_dv_accum, (m.K * m.H + 255) / 256, 256, 0, s, m, st, sums, counts, layer);
    return counted(1);
}

cudaError_t launch_dv_freeze(const double* sums, const long long* counts, float* dv,
                             long long LE, int H, cudaStream_t s) {
    k_dv_freeze<<<gen_blocks(LE * H), 256, 0, s>>>(sums, counts, dv, LE, H);
    return counted(1);
}

cudaError_t launch_trace(const DevModel& m, const DevState& st, const TraceDev& tr,
                         cudaStream_t s) {
    if (!tr.full) {
        PDL(k_trace, 1, 256, 0, s, m, st, tr);
    } else {
        PDL(k_trace, 64, 256, 0, s, m, st, tr);
        PDL(k_trace_bump, 1, 1, 0, s, tr);
        g_launches += 1;
    }
    return counted(1);
}

cudaError_t launch_trace_y(const DevModel& m, const DevState& st, const TraceDev& tr, int layer,
                           cudaStream_t s) {
    PDL(k_trace_y, 16, 256, 0, s, m, st, tr, layer);
    return counted(1);
}

}  // namespace smoe
