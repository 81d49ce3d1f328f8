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
//   * Operands stream into shared memory with cp.async.bulk: the packed
//     activations in UMMA's no-swizzle K-major canonical layout (SBO 128 B,
//     LBO 2 KB), the weights of 8 consecutive 32-row tiles gathered per
//     8-column group into one K-major operand of N = 256 rows (SBO 128 B,
//     LBO 4 KB) — 512-byte pieces of the stored row tiles, no re-layout pass.
//   * A persistent, warp-specialised kernel per projection (k_tc_ffn): a TMA
//     producer lane, an MMA lane issuing tcgen05.mma (kind::f16, M = 128
//     tokens, N = 256 rows, K = 16) into one of two TMEM accumulators, and four
//     epilogue warps draining the other with tcgen05.ld (32x32b) — SwiGLU for
//     gate/up, raw expert rows for down.
#include "kernels.h"
#include "smoe_chain.cuh"

#include <cuda.h>

#include <algorithm>

namespace smoe {

namespace {

constexpr int kTcM = 128;          // tokens per tile (UMMA M)
constexpr int kTcTiles = 8;        // 32-row weight tiles per CTA (N = 256: half the activation re-reads of N = 128)
constexpr int kTcK = 64;           // K columns per stage
constexpr int kTcStages = 3;
constexpr int kTcAChunk = kTcM * kTcK * 2;          // bytes of one operand half (hi or lo) per stage
constexpr int kTcBTile = 32 * kTcK * 2;             // bytes of one tile's chunk per stage
constexpr int kTcStage = 2 * kTcAChunk + kTcTiles * kTcBTile;  // 64 KB
constexpr int kTcSmem = kTcStages * kTcStage + 1024;  // + barriers and the TMEM address
constexpr int kTcCols = 32 * kTcTiles;              // TMEM columns (one 32-column accumulator per tile)

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

// bf16 x bf16 -> f32, M = 128 tokens, N = 32 * kTcTiles weight rows, both K-major.
constexpr uint32_t kIdesc =
    (1u << 4) | (1u << 7) | (1u << 10) | (((32u * kTcTiles) >> 3) << 17) | ((128u >> 4) << 24);

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

// Persistent, warp-specialised expert GEMM (one CTA per SM, 6 warps):
//   warp 0 lane 0  TMA producer: for each work item of this CTA, the K/64
//                  stages of [a_hi | a_lo | nt weight-tile chunks] into a
//                  3-stage shared-memory ring (cp.async.bulk, mbarrier
//                  complete_tx), refilling a stage once its MMAs completed;
//   warp 1 lane 0  MMA issuer: per stage 2 x 4 tcgen05.mma (kind::f16,
//                  M = 128 tokens, N = 256 rows, K = 16) into one of two TMEM
//                  accumulators (2 x 256 columns: item i uses buffer i & 1),
//                  tcgen05.commit to free the stage, and to hand the finished
//                  accumulator to the epilogue;
//   warps 2-5      epilogue: tcgen05.ld (32x32b, warp w reads TMEM lanes
//                  32 (w % 4) ..) of tokens, SwiGLU (gate/up) or raw rows
//                  (down), then release the accumulator buffer.
// So the epilogue of item i overlaps the MMAs of item i + 1, and the ring
// keeps streaming across item boundaries.  A work item is (token block it,
// n-block nb of kTcTiles 32-row tiles).
constexpr int kTcThreads = 192;
constexpr int kTcBufCols = kTcCols;          // columns per accumulator buffer
constexpr int kTcTmemCols = 2 * kTcBufCols;  // TMEM allocation (power of two, <= 512)

struct TcItem {
    int it, e, b0, cnt, c0, t0, nt, slot;
};
__device__ __forceinline__ TcItem tc_item(const DevModel& m, const PrefillDev& pf, const PfWave& wv, int w,
                                          int nblk, int ntiles) {
    TcItem r;
    r.it = w / nblk;
    const int nb = w % nblk;
    const int u = __ldcg(pf.chunk_u + r.it);
    r.e = wv.e[u];
    r.slot = wv.slot[u];
    r.b0 = pf.off[r.e];
    r.cnt = pf.off[r.e + 1] - r.b0;
    r.c0 = __ldcg(pf.chunk_c + r.it) * kTcM;
    r.t0 = nb * kTcTiles;
    r.nt = min(kTcTiles, ntiles - r.t0);
    return r;
}

// MODE 0: gate/up (K = H, tiles of 16 SwiGLU rows, h = silu(g) * u into Hb);
// MODE 1: down (K = Hm, tiles of 32 rows, raw expert rows into Y).
// wmap (when use_map): 5-D TMA map of this projection's weight tiles in the
// slot pool — dims (8 cols, 32 rows, tile, 8-col group, layer * C + slot),
// strides (2 B, 16 B, tile, 512 B, expert block) — whose box (8, 32, 8, 8, 1)
// lands exactly the gathered [group][tile][row][col] operand; otherwise
// 512-byte bulk copies build the same layout.
template <int MODE>
__global__ void __launch_bounds__(kTcThreads, 1) k_tc_ffn(DevModel m, PrefillDev pf, int layer, PfWave wv,
                                                          const uint16_t* apk, int n_work,
                                                          const __grid_constant__ CUtensorMap wmap, int use_map) {
    pdl_wait();
    pdl_trigger();
    const int K = MODE == 0 ? m.H : m.Hm;
    const int ntiles = MODE == 0 ? m.Hmp / 16 : m.Hp / 32;
    const int nblk = (ntiles + kTcTiles - 1) / kTcTiles;
    const long long tile_elems = static_cast<long long>(K) * 32;
    const long long blk_off = MODE == 0 ? 0 : m.gu_elems;
    unsigned char* smem = align128(g_smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kTcStages * kTcStage);
    uint64_t* empty = full + kTcStages;
    uint64_t* acc_full = empty + kTcStages;  // [2]
    uint64_t* acc_empty = acc_full + 2;      // [2]
    uint32_t* tptr = reinterpret_cast<uint32_t*>(acc_empty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kTcStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 4);  // one arrival per epilogue warp
        }
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tptr)),
                     "n"(kTcTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tptr;
    const int nk = K / kTcK;
    if (warp == 0 && lane == 0) {  // ---- producer
        int g = 0;
        for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
            const TcItem r = tc_item(m, pf, wv, w, nblk, ntiles);
            const uint16_t* blk = m.slots + (static_cast<long long>(layer) * m.C + r.slot) * m.expert_elems + blk_off;
            const uint16_t* hi = apk + static_cast<long long>(r.it) * 2 * K * kTcM;
            const uint16_t* lo = hi + static_cast<long long>(K) * kTcM;
            // the tensor copy always lands its whole box (tiles past ntiles are zero-filled)
            const uint32_t bytes = 2 * kTcAChunk + (use_map ? kTcTiles : r.nt) * kTcBTile;
            for (int k = 0; k < nk; ++k, ++g) {
                const int st = g % kTcStages;
                if (g >= kTcStages) mbar_wait(&empty[st], static_cast<uint32_t>(((g / kTcStages) - 1) & 1));
                unsigned char* sp = smem + st * kTcStage;
                mbar_expect_tx(&full[st], bytes);
                bulk_g2s(sp, hi + static_cast<long long>(k) * kTcM * kTcK, kTcAChunk, &full[st]);
                bulk_g2s(sp + kTcAChunk, lo + static_cast<long long>(k) * kTcM * kTcK, kTcAChunk, &full[st]);
                // weights as ONE K-major operand of N = 32 * kTcTiles rows: the
                // 512-byte [32 rows][8 cols] block of tile t, column group j goes to
                // [j][t] (rows of consecutive tiles adjacent, SBO 128 B, LBO
                // kTcTiles * 512 B); rows of absent tiles (t >= nt) stay stale and
                // only feed accumulator columns the epilogue never reads
                if (use_map) {  // one 5-D tensor copy: box (8 cols, 32 rows, 8 tiles, 8 groups, 1 expert)
                    const int slot_idx = layer * m.C + r.slot;
                    asm volatile(
                        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
                        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(sp + 2 * kTcAChunk)),
                        "l"(reinterpret_cast<uint64_t>(&wmap)), "r"(0), "r"(0), "r"(r.t0), "r"(k * (kTcK / 8)),
                        "r"(slot_idx), "r"(smem_u32(&full[st]))
                        : "memory");
                } else {
                    for (int t = 0; t < r.nt; ++t) {
                        const uint16_t* src = blk + (r.t0 + t) * tile_elems + static_cast<long long>(k) * kTcK * 32;
                        for (int j = 0; j < kTcK / 8; ++j)
                            bulk_g2s(sp + 2 * kTcAChunk + (j * kTcTiles + t) * 512, src + j * 256, 512, &full[st]);
                    }
                }
            }
        }
    } else if (warp == 1 && lane == 0) {  // ---- MMA issuer
        int g = 0, i = 0;
        for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++i) {
            const int b = i & 1;
            if (i >= 2) mbar_wait(&acc_empty[b], static_cast<uint32_t>(((i >> 1) - 1) & 1));
            tc_fence_after();
            const uint32_t acc = tmem + b * kTcBufCols;
            for (int k = 0; k < nk; ++k, ++g) {
                const int st = g % kTcStages;
                mbar_wait(&full[st], static_cast<uint32_t>((g / kTcStages) & 1));
                tc_fence_after();
                const uint32_t sa = smem_u32(smem + st * kTcStage);
#pragma unroll
                for (int kk = 0; kk < kTcK / 16; ++kk) {
                    const uint64_t ah = umma_desc(sa + kk * 4096, 2048, 128);
                    const uint64_t al = umma_desc(sa + kTcAChunk + kk * 4096, 2048, 128);
                    const uint64_t bd = umma_desc(sa + 2 * kTcAChunk + kk * 2 * kTcTiles * 512, kTcTiles * 512, 128);
                    tc_mma(acc, ah, bd, (k | kk) != 0);  // M 128 x N 256 x K 16: all tiles at once
                    tc_mma(acc, al, bd, 1);
                }
                tc_commit(&empty[st]);
            }
            tc_commit(&acc_full[b]);
        }
    } else if (warp >= 2) {  // ---- epilogue
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        int i = 0;
        for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++i) {
            const TcItem r = tc_item(m, pf, wv, w, nblk, ntiles);
            const int b = i & 1;
            mbar_wait(&acc_full[b], static_cast<uint32_t>((i >> 1) & 1));
            tc_fence_after();
            const int tok = q * 32 + lane;
            const bool valid = r.c0 + tok < r.cnt;
            const int ent = valid ? __ldcg(pf.list + r.b0 + r.c0 + tok) : 0;
            for (int t = 0; t < r.nt; ++t) {
                float v[32];
                tmem_ld32(tmem + b * kTcBufCols + (static_cast<uint32_t>(q * 32) << 16) + 32 * t, v);
                if (!valid) continue;
                if (MODE == 0) {
                    float* h = pf.Hb + static_cast<long long>(ent) * m.Hmp + (r.t0 + t) * 16;
#pragma unroll
                    for (int rr = 0; rr < 16; rr += 4) {
                        float o[4];
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const float gv = v[2 * (rr + j)], uv = v[2 * (rr + j) + 1];
                            o[j] = gv / (1.0f + __expf(-gv)) * uv;  // f32 SiLU: tolerance mode
                        }
                        *reinterpret_cast<float4*>(h + rr) = make_float4(o[0], o[1], o[2], o[3]);
                    }
                } else {
                    float* y = pf.Y + static_cast<long long>(ent) * m.Hp + (r.t0 + t) * 32;
#pragma unroll
                    for (int rr = 0; rr < 32; rr += 4)
                        *reinterpret_cast<float4*>(y + rr) = make_float4(v[rr], v[rr + 1], v[rr + 2], v[rr + 3]);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[b]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTcTmemCols) : "memory");
}

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

bool tc_prefill_supported(const DevModel& m) {
    return m.H % kTcK == 0 && m.Hm % kTcK == 0 && m.Hmp == m.Hm && m.Hp == m.H;
}

size_t tc_pack_bytes(const DevModel& m, int items) {
    const size_t K = static_cast<size_t>(m.H > m.Hm ? m.H : m.Hm);
    return static_cast<size_t>(items) * 2 * K * kTcM * 2;
}

int g_tc_ctas = 148;  // persistent grid: one CTA per SM (set by tc_preload)

cudaError_t tc_preload() {
    cudaFuncAttributes fa;  // load every kernel now (lazy loading synchronises the context)
    cudaError_t e = cudaFuncGetAttributes(&fa, k_tc_pack);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_tc_ffn<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_tc_ffn<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem);
    int dev = 0, sms = 0;
    if (e == cudaSuccess) e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess && sms > 0) g_tc_ctas = sms;
    return e;
}

// The two weight gathers of the slot pool as 5-D TMA maps (built once per
// slot pool; SMOE_TC_NO_TMAP=1 or an encode failure selects the 512-byte
// bulk-copy path, same smem layout).
struct TcMaps {
    const uint16_t* slots = nullptr;
    long long key[5] = {0, 0, 0, 0, 0};  // H, Hmp, L, C, expert_elems of the pool the maps describe
    CUtensorMap gu{}, dn{};
    int ok = 0;
};
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
const TcMaps& tc_maps(const DevModel& m) {
    // per host thread (sessions driven from different threads never share an
    // entry; one thread alternating sessions re-encodes, two driver calls)
    thread_local TcMaps cache;
    const long long key[5] = {m.H, m.Hmp, m.L, m.C, m.expert_elems};
    if (cache.slots == m.slots && std::equal(key, key + 5, cache.key)) return cache;
    cache = TcMaps{};
    cache.slots = m.slots;
    std::copy(key, key + 5, cache.key);
    static EncodeTiledFn enc = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<EncodeTiledFn>(nullptr);
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    if (!enc) return cache;
    const cuuint64_t nslots = static_cast<cuuint64_t>(m.L) * m.C, eb = static_cast<cuuint64_t>(m.expert_elems) * 2;
    const cuuint32_t box[5] = {8, 32, kTcTiles, kTcK / 8, 1}, es[5] = {1, 1, 1, 1, 1};
    auto make = [&](CUtensorMap* out, const uint16_t* base, int K, int ntiles) {
        const cuuint64_t dims[5] = {8, 32, static_cast<cuuint64_t>(ntiles), static_cast<cuuint64_t>(K / 8), nslots};
        const cuuint64_t strides[4] = {16, static_cast<cuuint64_t>(K) * 64, 512, eb};
        return enc(out, CU_TENSOR_MAP_DATA_TYPE_UINT16, 5, const_cast<uint16_t*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    cache.ok = make(&cache.gu, m.slots, m.H, m.Hmp / 16) && make(&cache.dn, m.slots + m.gu_elems, m.Hmp, m.Hp / 32);
    return cache;
}

// items: (wave expert, 128-token block) pairs in pf.chunk_u / chunk_c.
cudaError_t launch_pf_experts_tc(const DevModel& m, const PrefillDev& pf, int layer, const PfWave& wv, int items,
                                 uint16_t* apk, cudaStream_t s) {
    if (items < 1) return cudaSuccess;
    PDL(k_tc_pack, dim3((m.H / 8 + 15) / 16, items), 256, 0, s, m, pf, layer, wv, 0, apk);
    const int gu_work = items * ((m.Hmp / 16 + kTcTiles - 1) / kTcTiles);
    const int dn_work = items * ((m.Hp / 32 + kTcTiles - 1) / kTcTiles);
    const TcMaps& tm = tc_maps(m);
    const int use_map = tm.ok && !std::getenv("SMOE_TC_NO_TMAP");
    PDL(k_tc_ffn<0>, std::min(g_tc_ctas, gu_work), kTcThreads, kTcSmem, s, m, pf, layer, wv,
        static_cast<const uint16_t*>(apk), gu_work, tm.gu, use_map);
    PDL(k_tc_pack, dim3((m.Hm / 8 + 15) / 16, items), 256, 0, s, m, pf, layer, wv, 1, apk);
    PDL(k_tc_ffn<1>, std::min(g_tc_ctas, dn_work), kTcThreads, kTcSmem, s, m, pf, layer, wv,
        static_cast<const uint16_t*>(apk), dn_work, tm.dn, use_map);
    return cudaGetLastError();
}

}  // namespace smoe
