// prefill_tc.cu — tensor-core expert GEMMs for the batched prefill
// (tolerance mode, SURVEY §8f row 2 / VERDICT r01 "tcgen05 grouped GEMM").
//
// At prefill every executed expert sees many tokens, so gate/up and down are
// dense contractions (M = tokens of the expert, N = expert rows, K = H or Hm)
// and belong on the 5th-generation tensor cores:
//
//   * A (activations, f32 in the reference) is split into two bf16 operands
//     a_hi = bf16(x), a_lo = bf16(x - a_hi), so x is carried to ~16 mantissa
//     bits; W is bf16 already (the stored weights).  D = W.a_hi + W.a_lo,
//     accumulated in f32 in TMEM.  The result differs from the reference's
//     sequential f32 chain only by the accumulation order and the ~2^-17
//     residue of x — a stated tolerance, not bit parity; the exact path
//     (prefill.cu, one lane per row walking the columns in order) stays the
//     default.
//   * Operands stream into shared memory with cp.async.bulk (the weight row
//     tiles need no re-layout: a 32-row tile's 8-column groups are exactly
//     UMMA's no-swizzle K-major core matrices, SBO = 128 B, LBO = 512 B); the
//     packed activations use the same canonical layout (SBO 128 B, LBO 2 KB).
//   * One thread issues tcgen05.mma (kind::f16, M = 128 tokens, N = 32 rows per
//     tile, K = 16) into a TMEM accumulator per tile; tcgen05.commit frees each
//     stage; the epilogue reads TMEM with tcgen05.ld (32x32b) — one warp per
//     32-token lane quarter — and applies SwiGLU (gate/up) or stores the raw
//     expert rows (down).
#include "kernels.h"
#include "smoe_chain.cuh"

namespace smoe {

namespace {

constexpr int kTcM = 128;          // tokens per tile (UMMA M)
constexpr int kTcTiles = 4;        // 32-row weight tiles per CTA (N = 128)
constexpr int kTcK = 64;           // K columns per stage
constexpr int kTcStages = 4;
constexpr int kTcAChunk = kTcM * kTcK * 2;          // bytes of one operand half (hi or lo) per stage
constexpr int kTcBTile = 32 * kTcK * 2;             // bytes of one tile's chunk per stage
constexpr int kTcStage = 2 * kTcAChunk + kTcTiles * kTcBTile;  // 48 KB
constexpr int kTcSmem = kTcStages * kTcStage + 1024;

__device__ __forceinline__ uint16_t bf16_rn(float x) {
    uint32_t u = __float_as_uint(x);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

// UMMA shared-memory descriptor (SM100 version 1): no swizzle, K-major.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
    d |= 1ull << 46;  // version
    return d;         // base offset 0, legacy LBO mode, layout SWIZZLE_NONE
}

// bf16 x bf16 -> f32, M = 128, N = 32, both K-major.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

// 32 consecutive TMEM columns of this warp's lane quarter.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Main loop: TMEM columns [32 t, 32 t + 32) += A(128 x K) . tile_t(32 x K)^T for
// t < nt.  a_hi / a_lo: the packed activations of this token block
// ([K/8][128][8] bf16 each); tiles: row-tile bases (layout [K/8][32][8]).
// Executed by thread 0 (copies and MMA issue); returns once the last MMA's
// completion is signalled on `done`.
__device__ void tc_mainloop(const uint16_t* a_hi, const uint16_t* a_lo, const uint16_t* const* tiles, int nt, int K,
                            unsigned char* smem, uint64_t* full, uint64_t* empty, uint64_t* done, uint32_t tmem) {
    const int nk = K / kTcK;
    const uint32_t bytes = 2 * kTcAChunk + nt * kTcBTile;
    auto issue = [&](int k) {
        const int st = k % kTcStages;
        unsigned char* s = smem + st * kTcStage;
        mbar_expect_tx(&full[st], bytes);
        bulk_g2s(s, a_hi + static_cast<long long>(k) * kTcM * kTcK, kTcAChunk, &full[st]);
        bulk_g2s(s + kTcAChunk, a_lo + static_cast<long long>(k) * kTcM * kTcK, kTcAChunk, &full[st]);
        for (int t = 0; t < nt; ++t)
            bulk_g2s(s + 2 * kTcAChunk + t * kTcBTile, tiles[t] + static_cast<long long>(k) * kTcK * 32, kTcBTile,
                     &full[st]);
    };
    for (int k = 0; k < kTcStages && k < nk; ++k) issue(k);
    for (int k = 0; k < nk; ++k) {
        const int st = k % kTcStages;
        mbar_wait(&full[st], static_cast<uint32_t>((k / kTcStages) & 1));
        tc_fence_after();
        const uint32_t s = smem_u32(smem + st * kTcStage);
#pragma unroll
        for (int kk = 0; kk < kTcK / 16; ++kk) {
            const uint64_t ah = umma_desc(s + kk * 4096, 2048, 128);
            const uint64_t al = umma_desc(s + kTcAChunk + kk * 4096, 2048, 128);
            for (int t = 0; t < nt; ++t) {
                const uint64_t b = umma_desc(s + 2 * kTcAChunk + t * kTcBTile + kk * 1024, 512, 128);
                tc_mma(tmem + 32 * t, ah, b, (k | kk) != 0);
                tc_mma(tmem + 32 * t, al, b, 1);
            }
        }
        tc_commit(&empty[st]);  // this stage's smem is free once these MMAs complete
        if (k + kTcStages < nk) {
            mbar_wait(&empty[st], static_cast<uint32_t>((k / kTcStages) & 1));
            issue(k + kTcStages);
        }
    }
    tc_commit(done);
}

// Shared prologue: barriers, TMEM allocation (128 columns), item decode.
struct TcCta {
    unsigned char* smem;
    uint64_t *full, *empty, *done;
    uint32_t* tptr;
    uint32_t tmem;
    __device__ void setup() {
        smem = align128(g_smem);
        unsigned char* tail = smem + kTcStages * kTcStage;
        full = reinterpret_cast<uint64_t*>(tail);
        empty = full + kTcStages;
        done = empty + kTcStages;
        tptr = reinterpret_cast<uint32_t*>(done + 1);
        if (threadIdx.x == 0) {
            for (int i = 0; i < kTcStages; ++i) {
                mbar_init(&full[i], 1);
                mbar_init(&empty[i], 1);
            }
            mbar_init(done, 1);
            fence_mbar_init();
        }
        if (threadIdx.x < 32) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(tptr))
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
        tmem = *tptr;
    }
    __device__ void teardown() {
        tc_fence_before();
        __syncthreads();
        if (threadIdx.x < 32)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem) : "memory");
    }
    __device__ void wait_done() {
        mbar_wait(done, 0);
        tc_fence_after();
    }
};

}  // namespace

// --------------------------------------------------------------- packing --
// Activations of one (wave expert, 128-token block) item into the canonical
// layout, hi and lo halves: dst + item * 2 * K * 128, [K/8][128][8] each.
// src rows: mode 0 — normalised s of the token of list entry (gate/up input:
// (R * scale) * gain, numerics.cpp:72-84, as pf_stage_norm); mode 1 — Hb row
// of the entry (down input).  grid (K/8 groups / 8, items), 256 threads.
__global__ void __launch_bounds__(256) k_tc_pack(DevModel m, PrefillDev pf, int layer, PfWave wv, int mode,
                                                 uint16_t* dst) {
    pdl_wait();
    pdl_trigger();
    const int K = mode == 0 ? m.H : m.Hm;
    const int it = blockIdx.y, u = __ldcg(pf.chunk_u + it), e = wv.e[u];
    const int b0 = pf.off[e], cnt = pf.off[e + 1] - b0, c0 = __ldcg(pf.chunk_c + it) * kTcM;
    uint16_t* hi = dst + static_cast<long long>(it) * 2 * K * kTcM;
    uint16_t* lo = hi + static_cast<long long>(K) * kTcM;
    const float* gain = m.moe_gain + static_cast<long long>(layer) * m.H;
    // thread -> (token row t, group g): 8 groups per block, 128 tokens
    const int t = threadIdx.x & 127, g = blockIdx.x * 16 + (threadIdx.x >> 7) * 8;
    const bool valid = c0 + t < cnt;
    const int ent = valid ? __ldcg(pf.list + b0 + c0 + t) : 0;
    float scale = 0.0f;
    const float* src;
    if (mode == 0) {
        const int tok = ent / m.K;
        scale = __ldcg(pf.scale + tok);
        src = pf.R + static_cast<long long>(tok) * m.Hp;
    } else {
        src = pf.Hb + static_cast<long long>(ent) * m.Hmp;
    }
    for (int q = 0; q < 8; ++q) {
        const int gg = g + q;
        if (gg * 8 >= K) break;
        uint32_t ph[4], pl[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            float x[2];
#pragma unroll
            for (int w = 0; w < 2; ++w) {
                const int c = gg * 8 + 2 * h + w;
                float v = valid ? __ldcg(src + c) : 0.0f;
                if (mode == 0 && valid) v = v * scale * __ldg(gain + c);
                x[w] = v;
            }
            const uint16_t h0 = bf16_rn(x[0]), h1 = bf16_rn(x[1]);
            const uint16_t l0 = bf16_rn(x[0] - __uint_as_float(static_cast<uint32_t>(h0) << 16));
            const uint16_t l1 = bf16_rn(x[1] - __uint_as_float(static_cast<uint32_t>(h1) << 16));
            ph[h] = static_cast<uint32_t>(h0) | (static_cast<uint32_t>(h1) << 16);
            pl[h] = static_cast<uint32_t>(l0) | (static_cast<uint32_t>(l1) << 16);
        }
        const long long o = (static_cast<long long>(gg) * kTcM + t) * 8;
        *reinterpret_cast<uint4*>(hi + o) = make_uint4(ph[0], ph[1], ph[2], ph[3]);
        *reinterpret_cast<uint4*>(lo + o) = make_uint4(pl[0], pl[1], pl[2], pl[3]);
    }
}

// gate/up: grid (ceil((Hmp/16) / 4), items), 128 threads.  CTA x covers the
// 16-row SwiGLU tiles 4x .. 4x+3 (virtual rows 2r = gate, 2r+1 = up); the
// epilogue forms h = silu(g) * u (silu in f64, numerics.cpp:86-89) per token.
__global__ void __launch_bounds__(128) k_tc_gu(DevModel m, PrefillDev pf, int layer, PfWave wv, const uint16_t* apk) {
    pdl_wait();
    pdl_trigger();
    TcCta c;
    c.setup();
    const int it = blockIdx.y, u = __ldcg(pf.chunk_u + it), e = wv.e[u];
    const int b0 = pf.off[e], cnt = pf.off[e + 1] - b0, c0 = __ldcg(pf.chunk_c + it) * kTcM;
    const int ntiles = m.Hmp / 16, t0 = blockIdx.x * kTcTiles, nt = min(kTcTiles, ntiles - t0);
    const uint16_t* blk = m.slots + (static_cast<long long>(layer) * m.C + wv.slot[u]) * m.expert_elems;
    if (threadIdx.x == 0) {
        const uint16_t* tiles[kTcTiles];
        for (int t = 0; t < kTcTiles; ++t) tiles[t] = blk + static_cast<long long>(t0 + min(t, nt - 1)) * m.H * 32;
        const uint16_t* hi = apk + static_cast<long long>(it) * 2 * m.H * kTcM;
        tc_mainloop(hi, hi + static_cast<long long>(m.H) * kTcM, tiles, nt, m.H, c.smem, c.full, c.empty, c.done,
                    c.tmem);
    }
    __syncwarp();
    c.wait_done();
    const int w = threadIdx.x >> 5, tok = w * 32 + (threadIdx.x & 31);
    const bool valid = c0 + tok < cnt;
    const int ent = valid ? __ldcg(pf.list + b0 + c0 + tok) : 0;
    for (int t = 0; t < nt; ++t) {
        float v[32];
        tmem_ld32(c.tmem + (static_cast<uint32_t>(w * 32) << 16) + 32 * t, v);
        if (valid)
#pragma unroll
            for (int r = 0; r < 16; ++r)
                pf.Hb[static_cast<long long>(ent) * m.Hmp + (t0 + t) * 16 + r] = silu_ref(v[2 * r]) * v[2 * r + 1];
    }
    c.teardown();
}

// down: grid (ceil((Hp/32) / 4), items), 128 threads: raw expert rows into Y.
__global__ void __launch_bounds__(128) k_tc_down(DevModel m, PrefillDev pf, int layer, PfWave wv,
                                                 const uint16_t* apk) {
    pdl_wait();
    pdl_trigger();
    TcCta c;
    c.setup();
    const int it = blockIdx.y, u = __ldcg(pf.chunk_u + it), e = wv.e[u];
    const int b0 = pf.off[e], cnt = pf.off[e + 1] - b0, c0 = __ldcg(pf.chunk_c + it) * kTcM;
    const int ntiles = m.Hp / 32, t0 = blockIdx.x * kTcTiles, nt = min(kTcTiles, ntiles - t0);
    const uint16_t* blk =
        m.slots + (static_cast<long long>(layer) * m.C + wv.slot[u]) * m.expert_elems + m.gu_elems;
    if (threadIdx.x == 0) {
        const uint16_t* tiles[kTcTiles];
        for (int t = 0; t < kTcTiles; ++t) tiles[t] = blk + static_cast<long long>(t0 + min(t, nt - 1)) * m.Hmp * 32;
        const uint16_t* hi = apk + static_cast<long long>(it) * 2 * m.Hm * kTcM;
        tc_mainloop(hi, hi + static_cast<long long>(m.Hm) * kTcM, tiles, nt, m.Hm, c.smem, c.full, c.empty, c.done,
                    c.tmem);
    }
    __syncwarp();
    c.wait_done();
    const int w = threadIdx.x >> 5, tok = w * 32 + (threadIdx.x & 31);
    const bool valid = c0 + tok < cnt;
    const int ent = valid ? __ldcg(pf.list + b0 + c0 + tok) : 0;
    for (int t = 0; t < nt; ++t) {
        float v[32];
        tmem_ld32(c.tmem + (static_cast<uint32_t>(w * 32) << 16) + 32 * t, v);
        if (valid) {
            float* y = pf.Y + static_cast<long long>(ent) * m.Hp + (t0 + t) * 32;
#pragma unroll
            for (int r = 0; r < 32; r += 4) *reinterpret_cast<float4*>(y + r) = make_float4(v[r], v[r + 1], v[r + 2], v[r + 3]);
        }
    }
    c.teardown();
}

bool tc_prefill_supported(const DevModel& m) {
    return m.H % kTcK == 0 && m.Hm % kTcK == 0 && m.Hmp == m.Hm && m.Hp == m.H;
}

size_t tc_pack_bytes(const DevModel& m, int items) {
    const size_t K = static_cast<size_t>(m.H > m.Hm ? m.H : m.Hm);
    return static_cast<size_t>(items) * 2 * K * kTcM * 2;
}

cudaError_t tc_preload() {
    cudaError_t e = cudaFuncSetAttribute(k_tc_gu, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_tc_down, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem);
    return e;
}

// items: (wave expert, 128-token block) pairs in pf.chunk_u / chunk_c.
cudaError_t launch_pf_experts_tc(const DevModel& m, const PrefillDev& pf, int layer, const PfWave& wv, int items,
                                 uint16_t* apk, cudaStream_t s) {
    if (items < 1) return cudaSuccess;
    PDL(k_tc_pack, dim3((m.H / 8 + 15) / 16, items), 256, 0, s, m, pf, layer, wv, 0, apk);
    PDL(k_tc_gu, dim3((m.Hmp / 16 + kTcTiles - 1) / kTcTiles, items), 128, kTcSmem, s, m, pf, layer, wv,
        static_cast<const uint16_t*>(apk));
    PDL(k_tc_pack, dim3((m.Hm / 8 + 15) / 16, items), 256, 0, s, m, pf, layer, wv, 1, apk);
    PDL(k_tc_down, dim3((m.Hp / 32 + kTcTiles - 1) / kTcTiles, items), 128, kTcSmem, s, m, pf, layer, wv,
        static_cast<const uint16_t*>(apk));
    return cudaGetLastError();
}

}  // namespace smoe
