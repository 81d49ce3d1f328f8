// smoe_chain.cuh — device primitives shared by kernels.cu and the tools'
// micro-benchmarks: mbarrier / cp.async.bulk helpers, programmatic dependent
// launch, the smem Stager, the bit-exact f64 block reductions and rms_norm,
// and WarpPipe, the per-warp TMA-fed sequential-chain GEMV.
#pragma once
#include "exp_glibc.cuh"
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "smoe_dev.h"

namespace smoe {

// ---------------------------------------------------------------- helpers --

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// L2 eviction-priority hints for weight streams (createpolicy): expert
// weights are read once per token and marked evict-first, so the dense
// per-layer weights (router gates, attention) keep their L2 residency.
enum L2Hint : int { kL2Normal = 0, kL2EvictFirst = 1, kL2EvictLast = 2 };
__device__ __forceinline__ uint64_t l2_policy(int hint) {
    uint64_t p = 0;
    if (hint == kL2EvictFirst)
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    else if (hint == kL2EvictLast)
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
// Non-blocking probe of a phase (mbarrier.test_wait): issued well before the
// data is needed so its latency (~90 cycles even when complete) overlaps the
// chain instead of stalling it.
__device__ __forceinline__ uint32_t mbar_test(uint64_t* b, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    return ok;
}
// One lane of a converged warp (elect.sync): lets ptxas issue the bulk copy
// without a per-lane uniformity loop.
__device__ __forceinline__ bool elect_one() {
    uint32_t p;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "elect.sync _|P, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}"
        : "=r"(p));
    return p != 0;
}
// Programmatic dependent launch: let the next kernel in the stream start its
// prologue (barrier init, static weight prefetch) while this one runs; every
// kernel calls pdl_wait() before touching activations written upstream.
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Optional phase timing (build with -DSMOE_PHASES; tools/phase_run.py): block
// (0,0)'s timeline between PHASE() marks, printed once per launch.
#ifdef SMOE_PHASES
__device__ __forceinline__ unsigned long long gtimer() {  // SM cycles
    return clock64();
}
// one printf per dump, so concurrent kernels do not interleave their lines
__device__ inline void phase_print(const char* name, const unsigned long long* ph, int n) {
    unsigned long long d[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int i = 1; i < n && i < 10; ++i) d[i - 1] = ph[i] - ph[i - 1];
    printf("%s (cycles): %llu %llu %llu %llu %llu %llu %llu %llu | %llu\n", name, d[0], d[1], d[2], d[3], d[4],
           d[5], d[6], d[7], ph[n - 1] - ph[0]);
}
#define PHASE_DECL \
    unsigned long long ph_[10];  \
    int nph_ = 0;
#define PHASE()                                  \
    do {                                         \
        if (nph_ < 10) ph_[nph_++] = gtimer();   \
    } while (0)
#define PHASE_DUMP(name)                                                                   \
    do {                                                                                   \
        if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) phase_print(name, ph_, nph_); \
    } while (0)
#else
#define PHASE_DECL
#define PHASE() \
    do {        \
    } while (0)
#define PHASE_DUMP(name) \
    do {                 \
    } while (0)
#endif

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ float bf2f(uint16_t b) {
    return __uint_as_float(static_cast<uint32_t>(b) << 16);
}
__device__ __forceinline__ float to_f(uint16_t b) { return bf2f(b); }
__device__ __forceinline__ float to_f(float f) { return f; }

// numerics.cpp:86-89 — silu in f64, rounded to f32.
__device__ __forceinline__ float silu_ref(float x) {
    const double xd = static_cast<double>(x);
    return static_cast<float>(xd / (1.0 + exp_glibc(-xd)));
}

// Deterministic block reduction of a per-thread double (tree order fixed by
// blockDim).  Returns the same value in every thread.
__device__ inline double block_sum_d(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    if ((threadIdx.x & 31) == 0) red[w] = v;
    __syncthreads();
    double t = 0.0;
    for (int i = 0; i < nw; ++i) t += red[i];
    __syncthreads();
    return t;
}

__device__ inline float block_max_f(float v, float* red) {
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_down_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    if ((threadIdx.x & 31) == 0) red[w] = v;
    __syncthreads();
    float t = red[0];
    for (int i = 1; i < nw; ++i) t = fmaxf(t, red[i]);
    __syncthreads();
    return t;
}

// rms_norm (numerics.cpp:72-84): out[i] = (v[i] * scale) * gain[i],
// scale = f32(1 / sqrt(sum_f64(v^2) / n + eps)).  Whole block participates;
// v, gain, out are 16-byte aligned shared arrays and n % 4 == 0 (H % 8 == 0 is
// validated).  The f64 sum runs as 4 independent partial sums per thread
// (fixed order: the reduction tree is deterministic).
__device__ inline void block_rms_norm(const float* v, const float* gain, int n, float eps, float* out,
                               double* red) {
    const float4* v4 = reinterpret_cast<const float4*>(v);
    const float4* g4 = reinterpret_cast<const float4*>(gain);
    float4* o4 = reinterpret_cast<float4*>(out);
    const int n4 = n >> 2;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    for (int i = threadIdx.x; i < n4; i += blockDim.x) {
        const float4 t = v4[i];
        a0 += static_cast<double>(t.x) * static_cast<double>(t.x);
        a1 += static_cast<double>(t.y) * static_cast<double>(t.y);
        a2 += static_cast<double>(t.z) * static_cast<double>(t.z);
        a3 += static_cast<double>(t.w) * static_cast<double>(t.w);
    }
    const double ss = block_sum_d((a0 + a1) + (a2 + a3), red);
    const float scale =
        static_cast<float>(1.0 / sqrt(ss / static_cast<double>(n) + static_cast<double>(eps)));
    for (int i = threadIdx.x; i < n4; i += blockDim.x) {
        const float4 t = v4[i], g = g4[i];
        o4[i] = make_float4(t.x * scale * g.x, t.y * scale * g.y, t.z * scale * g.z,
                            t.w * scale * g.w);
    }
    __syncthreads();
}

// Producer side of rms_norm (numerics.cpp:72-84) fused into the kernel that
// writes the vector: one warp's 32 rows -> one f64 partial sum of squares
// (fixed shuffle tree).  Every lane passes its value (0 for padding rows);
// lane 0 stores the partial.
__device__ __forceinline__ void warp_ssq_partial(float v, double* dst) {
    double d = static_cast<double>(v) * static_cast<double>(v);
    for (int o = 16; o > 0; o >>= 1) d += __shfl_down_sync(0xffffffffu, d, o);
    if ((threadIdx.x & 31) == 0) *dst = d;
}

// Consumer side: sum the nb partials in a fixed order (lane-strided, then a
// fixed shuffle tree) and form the reference's scale
// f32(1 / sqrt(sum / n + eps)).  Executed by a whole warp; every warp of a
// block computes the same value.  Like the in-block tree this replaces, the
// f64 order differs from the reference's sequential loop; the difference
// (~1e-16 relative) survives the f32 rounding of the scale only at
// measure-zero midpoints.
__device__ __forceinline__ float rms_scale_from_partials(const double* part, int nb, int n,
                                                         float eps) {
    double v = 0.0;
    for (int i = threadIdx.x & 31; i < nb; i += 32) v += __ldcg(part + i);
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    v = __shfl_sync(0xffffffffu, v, 0);
    return static_cast<float>(1.0 / sqrt(v / static_cast<double>(n) + static_cast<double>(eps)));
}

// out[i] = (v[i] * scale) * gain[i] over a block (16-byte aligned smem, n % 4 == 0).
__device__ __forceinline__ void block_apply_norm(const float* v, const float* gain, int n, float scale,
                                                 float* out) {
    const float4* v4 = reinterpret_cast<const float4*>(v);
    const float4* g4 = reinterpret_cast<const float4*>(gain);
    float4* o4 = reinterpret_cast<float4*>(out);
#pragma unroll 4
    for (int i = threadIdx.x; i < (n >> 2); i += blockDim.x) {
        const float4 t = v4[i], g = g4[i];
        o4[i] = make_float4(t.x * scale * g.x, t.y * scale * g.y, t.z * scale * g.z, t.w * scale * g.w);
    }
    __syncthreads();
}

// The first kGainRegs float4 of a block's share of a static norm gain, loaded
// into registers before the kernel's dependency wait so the normalisation
// after it costs no further global round trip (the rest, for n > 4 x 4 x
// blockDim, is read from global as block_apply_norm does).
struct GainRegs {
    static constexpr int kRegs = 4;
    float4 g[kRegs];
    __device__ __forceinline__ void load(const float* gain, int n) {
        const float4* g4 = reinterpret_cast<const float4*>(gain);
#pragma unroll
        for (int q = 0; q < kRegs; ++q) {
            const int i = threadIdx.x + q * blockDim.x;
            if (i < (n >> 2)) g[q] = __ldg(g4 + i);
        }
    }
};

// block_apply_norm with the gain's first part from registers (same arithmetic).
__device__ __forceinline__ void block_apply_norm_regs(const float* v, const GainRegs& gr, const float* gain, int n,
                                                      float scale, float* out) {
    const float4* v4 = reinterpret_cast<const float4*>(v);
    const float4* g4 = reinterpret_cast<const float4*>(gain);
    float4* o4 = reinterpret_cast<float4*>(out);
#pragma unroll
    for (int q = 0; q < GainRegs::kRegs; ++q) {
        const int i = threadIdx.x + q * blockDim.x;
        if (i < (n >> 2)) {
            const float4 t = v4[i], g = gr.g[q];
            o4[i] = make_float4(t.x * scale * g.x, t.y * scale * g.y, t.z * scale * g.z, t.w * scale * g.w);
        }
    }
    for (int i = threadIdx.x + GainRegs::kRegs * blockDim.x; i < (n >> 2); i += blockDim.x) {
        const float4 t = v4[i], g = g4[i];
        o4[i] = make_float4(t.x * scale * g.x, t.y * scale * g.y, t.z * scale * g.z, t.w * scale * g.w);
    }
    __syncthreads();
}

__device__ __forceinline__ unsigned char* align128(unsigned char* p) {
    return reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(p) + 127) & ~uintptr_t(127));
}

extern __shared__ __align__(128) unsigned char g_smem[];

// "Last CTA done" gate: returns true in every thread of the last CTA to arrive.
__device__ inline bool last_cta(int* counter, int total) {
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const int prev = atomicAdd(counter, 1);
        s_last = (prev == total - 1);
        if (s_last) *counter = 0;
    }
    __syncthreads();
    if (s_last) __threadfence();
    return s_last != 0;
}

// ------------------------------------------------------------ smem stager --
//
// Stages a kernel's input vectors (activations, gains, default-vector rows,
// expert hidden states) global -> shared with cp.async.bulk: thread 0 issues
// one bulk copy per vector on a single mbarrier, so every vector is in flight
// at once instead of one global-latency round trip per scalar load.  A
// vector whose address/size is not 16-byte aligned falls back to a
// block-strided copy.

__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}

struct Stager {
    uint64_t* bar;
    uint32_t phase;
    __device__ void init(uint64_t* b) {  // whole block
        bar = b;
        phase = 0;
        if (threadIdx.x == 0) {
            mbar_init(bar, 1);
            fence_mbar_init();
        }
        __syncthreads();
    }
    // whole block; `bytes` is rounded up to 16 (buffers are padded)
    __device__ void add(void* dst, const void* src, int bytes) {
        const uint32_t b = static_cast<uint32_t>((bytes + 15) & ~15);
        if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
            if (threadIdx.x == 0) {
                mbar_expect(bar, b);
                bulk_g2s(dst, src, b, bar);
            }
        } else {
            const float* s = static_cast<const float*>(src);
            float* d = static_cast<float*>(dst);
            for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) d[i] = s[i];
        }
    }
    __device__ void wait() {  // whole block
        if (threadIdx.x == 0) mbar_arrive(bar);
        mbar_wait(bar, phase);
        phase ^= 1;
        __syncthreads();
    }
};

// ------------------------------------------------------- warp tile stream --
//
// One warp computes 32 sequential dot products acc(lane) = sum_c W[c][lane]*x[c]
// over a row tile [cols][32] in global memory.  Lane 0 keeps S chunks of CC
// columns in flight with cp.async.bulk; every lane walks the columns in order.

__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(a));
    return v;
}
__device__ __forceinline__ float4 lds128f(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(a));
    return v;
}
// bf16 halves of a 32-bit word as f32, on the ALU pipe (PRMT / LOP3) so the
// FMA pipe is left to the FMUL/FADD chain (ptxas would use IMAD.SHL for <<).
__device__ __forceinline__ float lo_bf(uint32_t w) {
    uint32_t r;
    asm("prmt.b32 %0, %1, 0, 0x1044;" : "=r"(r) : "r"(w));
    return __uint_as_float(r);
}
__device__ __forceinline__ float hi_bf(uint32_t w) {
    uint32_t r;
    asm("lop3.b32 %0, %1, 0xffff0000, 0, 0xc0;" : "=r"(r) : "r"(w));
    return __uint_as_float(r);
}

// One 16-byte group of a lane's consecutive columns, in column order.
struct XG {  // the matching activations
    float4 a, b;
};
__device__ __forceinline__ XG load_x(uint32_t xa, uint16_t) { return {lds128f(xa), lds128f(xa + 16)}; }
__device__ __forceinline__ XG load_x(uint32_t xa, float) { return {lds128f(xa), make_float4(0, 0, 0, 0)}; }
// Products are formed two at a time with FMUL2 (__fmul2_rn: each lane of the
// pair rounds exactly like __fmul_rn) and summed by scalar FADDs in column
// order, so the FMA pipe carries 4 FMUL2 + 8 FADD per 8 columns (24 cycles at
// 2 cycles each) under the 32-cycle FADD latency chain.  The products must
// never feed a packed add: ptxas contracts FMUL2 -> FADD2 into FFMA2 even for
// _rn intrinsics (tests/test_sass.py checks the library has no FFMA2).
__device__ __forceinline__ float chain_group(float acc, uint4 w, const XG& x, uint16_t) {
    const float2 p0 = __fmul2_rn(make_float2(lo_bf(w.x), hi_bf(w.x)), make_float2(x.a.x, x.a.y));
    const float2 p1 = __fmul2_rn(make_float2(lo_bf(w.y), hi_bf(w.y)), make_float2(x.a.z, x.a.w));
    const float2 p2 = __fmul2_rn(make_float2(lo_bf(w.z), hi_bf(w.z)), make_float2(x.b.x, x.b.y));
    const float2 p3 = __fmul2_rn(make_float2(lo_bf(w.w), hi_bf(w.w)), make_float2(x.b.z, x.b.w));
    acc = acc + p0.x;
    acc = acc + p0.y;
    acc = acc + p1.x;
    acc = acc + p1.y;
    acc = acc + p2.x;
    acc = acc + p2.y;
    acc = acc + p3.x;
    acc = acc + p3.y;
    return acc;
}
__device__ __forceinline__ float chain_group(float acc, uint4 w, const XG& x, float) {
    const float4 x0 = x.a;
    acc = acc + __uint_as_float(w.x) * x0.x;
    acc = acc + __uint_as_float(w.y) * x0.y;
    acc = acc + __uint_as_float(w.z) * x0.z;
    acc = acc + __uint_as_float(w.w) * x0.w;
    return acc;
}
// The rounded products w[c] * x[c] of one group (acc + p is then the
// reference's `acc += w * x`: product rounded, then the add rounded).
__device__ __forceinline__ void products(uint4 w, const XG& x, float* p, uint16_t) {
    p[0] = lo_bf(w.x) * x.a.x;
    p[1] = hi_bf(w.x) * x.a.y;
    p[2] = lo_bf(w.y) * x.a.z;
    p[3] = hi_bf(w.y) * x.a.w;
    p[4] = lo_bf(w.z) * x.b.x;
    p[5] = hi_bf(w.z) * x.b.y;
    p[6] = lo_bf(w.w) * x.b.z;
    p[7] = hi_bf(w.w) * x.b.w;
}
__device__ __forceinline__ void products(uint4 w, const XG& x, float* p, float) {
    p[0] = __uint_as_float(w.x) * x.a.x;
    p[1] = __uint_as_float(w.y) * x.a.y;
    p[2] = __uint_as_float(w.z) * x.a.z;
    p[3] = __uint_as_float(w.w) * x.a.w;
}
__device__ __forceinline__ float group_elem(uint4 w, int i, uint16_t) {
    const uint32_t v = i < 2 ? w.x : i < 4 ? w.y : i < 6 ? w.z : w.w;
    return (i & 1) ? hi_bf(v) : lo_bf(v);
}
__device__ __forceinline__ float group_elem(uint4 w, int i, float) {
    return __uint_as_float(i == 0 ? w.x : i == 1 ? w.y : i == 2 ? w.z : w.w);
}

// Row tile layout (smoe_dev.h): 32 rows, columns in groups of G = 16 B / sizeof(WT);
// element (row lane, col c) at (c / G) * 32 * G + lane * G + c % G.  A chunk of
// CC columns (CC % G == 0) is CC * 32 contiguous elements = one bulk copy; each
// lane reads its G columns with one conflict-free ld.shared.v4.
#ifdef SMOE_PHASES
#define PIPE_WAIT(stmt)                 \
    do {                                \
        const long long t_ = clock64(); \
        stmt;                           \
        wait_cyc += clock64() - t_;     \
    } while (0)
#else
#define PIPE_WAIT(stmt) stmt
#endif

template <typename WT, int S, int CC>
struct WarpPipe {
#ifdef SMOE_PHASES
    long long wait_cyc = 0;  // cycles spent waiting for chunks (phase builds only)
#endif
    static constexpr int G = 16 / static_cast<int>(sizeof(WT));
    static constexpr int kS = S, kCC = CC;
    static constexpr int kChunkElems = CC * 32;
    static constexpr int kChunkBytes = kChunkElems * static_cast<int>(sizeof(WT));
    static constexpr int kBytes = S * kChunkBytes + S * 8;
    static_assert(CC % G == 0, "chunk must hold whole column groups");
    uint64_t* full;  // [S]
    WT* buf;         // [S][CC*32]
    uint32_t sbuf;   // shared-window address of buf
    int ctr;         // chunks consumed so far (phase tracking)
    int primed;      // chunks already issued for the next run()

    uint64_t policy;  // L2 hint for the weight stream (0 with hint kL2Normal)
    int hinted;
    __device__ void init(unsigned char* smem, int hint = kL2Normal) {  // owning warp; then syncwarp
        hinted = hint != kL2Normal;
        policy = hinted ? l2_policy(hint) : 0;
        buf = reinterpret_cast<WT*>(smem);
        sbuf = smem_u32(smem);
        full = reinterpret_cast<uint64_t*>(smem + S * kChunkBytes);
        ctr = 0;
        primed = 0;
        if ((threadIdx.x & 31) == 0) {
            for (int i = 0; i < S; ++i) mbar_init(&full[i], 1);
            fence_mbar_init();
        }
        __syncwarp();
    }

    __device__ void issue(const WT* tile, int cols, int n, int g) {
        const int st = g % S;
        const int c0 = n * CC;
        const int cn = min(CC, round_up(cols, G) - c0);
        const uint32_t bytes = static_cast<uint32_t>(cn) * 32u * sizeof(WT);
        mbar_expect_tx(&full[st], bytes);
        if (hinted)
            bulk_g2s_hint(buf + st * kChunkElems, tile + static_cast<long long>(c0) * 32, bytes, &full[st],
                          policy);
        else
            bulk_g2s(buf + st * kChunkElems, tile + static_cast<long long>(c0) * 32, bytes, &full[st]);
    }

    // Chunk g (absolute ring index, continuing ctr) as a gather of n pieces of
    // `piece` elements, piece p from src + p * stride, into consecutive places
    // of the chunk; one lane issues.
    __device__ void issue_gather(const WT* src, long long stride, int n, int piece, int g) {
        const int st = g % S;
        const uint32_t pb = static_cast<uint32_t>(piece) * sizeof(WT);
        mbar_expect_tx(&full[st], pb * static_cast<uint32_t>(n));
        for (int p = 0; p < n; ++p) {
            if (hinted)
                bulk_g2s_hint(buf + st * kChunkElems + p * piece, src + p * stride, pb, &full[st], policy);
            else
                bulk_g2s(buf + st * kChunkElems + p * piece, src + p * stride, pb, &full[st]);
        }
    }
    // Wait for chunk g; returns its shared-window address.
    __device__ uint32_t wait_chunk(int g) {
        mbar_wait(&full[g % S], static_cast<uint32_t>((g / S) & 1));
        return sbuf + (g % S) * kChunkBytes;
    }

    // Issue the first chunks of `tile` before the input vector exists (weights
    // are independent of the activations), so the first wait finds data.
    __device__ void prime(const WT* tile, int cols) {
        const int nch = (cols + CC - 1) / CC;
        if ((threadIdx.x & 31) == 0)
            for (int n = 0; n < S && n < nch; ++n) issue(tile, cols, n, ctr + n);
        primed = 1;
    }

    // Returns this lane's dot product over the first `cols` columns, in
    // column order.  xs: shared-memory f32 vector (16-byte aligned).
    //
    // Software pipeline: the shared loads of group j+2 are issued while group
    // j's FMUL/FADD chain runs (LDS latency ~30 cycles vs the 32-cycle FADD
    // chain of a group), also across chunk boundaries; the group loop of a
    // full chunk is unrolled so the only branches are one mbarrier wait and
    // one refill per chunk.  A partial last chunk takes the plain loop.
    __device__ float run(const WT* tile, int cols, const float* xs) {
        constexpr int GPC = CC / G;  // groups per chunk
        static_assert(GPC >= 2, "chunk must hold at least two groups");
        const int lane = threadIdx.x & 31;
        const int nch = (cols + CC - 1) / CC;
        if (lane == 0 && !primed)
            for (int n = 0; n < S && n < nch; ++n) issue(tile, cols, n, ctr + n);
        primed = 0;
        const uint32_t xbase = smem_u32(xs);
        const uint32_t lbase = sbuf + lane * 16;
        const int c0 = ctr;
        const int nfull = cols / CC;
        float acc = 0.0f;
        uint4 w0 = make_uint4(0, 0, 0, 0), w1 = w0;
        XG x0{}, x1{};
        if (nfull > 0) {
            PIPE_WAIT(mbar_wait(&full[c0 % S], static_cast<uint32_t>((c0 / S) & 1)));
            w0 = lds128(lbase + (c0 % S) * kChunkBytes);
            w1 = lds128(lbase + (c0 % S) * kChunkBytes + 512);
            x0 = load_x(xbase, WT{});
            x1 = load_x(xbase + G * 4, WT{});
        }
        for (int n = 0; n < nfull; ++n) {
            const int g = c0 + n;
            const uint32_t cb = lbase + (g % S) * kChunkBytes;
            const uint32_t nb = lbase + ((g + 1) % S) * kChunkBytes;
            const bool next_full = n + 1 < nfull;
            const uint32_t xc = xbase + n * CC * 4;
            uint32_t next_ready = 0;
#pragma unroll
            for (int j = 0; j < GPC; ++j) {
                const uint4 w = w0;
                const XG x = x0;
                w0 = w1;
                x0 = x1;
                if (j == GPC / 2 && next_full)  // early, non-blocking probe of the next chunk
                    next_ready = mbar_test(&full[(g + 1) % S], static_cast<uint32_t>(((g + 1) / S) & 1));
                if (j + 2 < GPC) {
                    w1 = lds128(cb + (j + 2) * 512);
                    x1 = load_x(xc + (j + 2) * G * 4, WT{});
                } else if (next_full) {
                    if (j + 2 == GPC && !next_ready)
                        PIPE_WAIT(mbar_wait(&full[(g + 1) % S], static_cast<uint32_t>(((g + 1) / S) & 1)));
                    w1 = lds128(nb + (j + 2 - GPC) * 512);
                    x1 = load_x(xc + (j + 2) * G * 4, WT{});
                }
                acc = chain_group(acc, w, x, WT{});
            }
            __syncwarp();  // every lane is done with this stage: refill it
            if (n + S < nch && elect_one()) issue(tile, cols, n + S, g + S);
        }
        if (nfull < nch) {  // partial last chunk
            const int n = nfull, g = c0 + n;
            mbar_wait(&full[g % S], static_cast<uint32_t>((g / S) & 1));
            const uint32_t wb = lbase + (g % S) * kChunkBytes;
            const uint32_t xb = xbase + n * CC * 4;
            const int cn = cols - n * CC;
            const int ng = cn / G;
            for (int q = 0; q < ng; ++q)
                acc = chain_group(acc, lds128(wb + q * 512), load_x(xb + q * G * 4, WT{}), WT{});
            const int tail = cn - ng * G;
            if (tail) {
                const uint4 w = lds128(wb + ng * 512);
                const float* xt = xs + n * CC + ng * G;
                for (int i = 0; i < tail; ++i) acc = acc + group_elem(w, i, WT{}) * xt[i];
            }
            __syncwarp();
        }
        ctr += nch;
        return acc;
    }

    // Tolerance ("fast") decode arithmetic: the same weight stream and the
    // same lane-per-row result, but the row's dot product is carried in four
    // independent packed f32 partial sums (column pairs 0-1, 2-3, 4-5, 6-7 of
    // every group) with fused multiply-adds (FFMA2), summed at the end.  No
    // dependent chain: the loop is issue-bound (~15 instructions per 8
    // columns) instead of FADD-latency bound, so the kernel is HBM-bound.
    // Differs from the reference's sequential sum by rounding only (DESIGN
    // "Decode arithmetic modes").  bf16 weights only.
    __device__ __forceinline__ float run_fast(const WT* tile, int cols, const float* xs) {
        static_assert(sizeof(WT) == 2, "fast chains take bf16 weights");
        constexpr int GPC = CC / G;
        const int lane = threadIdx.x & 31;
        const int nch = (cols + CC - 1) / CC;
        if (lane == 0 && !primed)
            for (int n = 0; n < S && n < nch; ++n) issue(tile, cols, n, ctr + n);
        primed = 0;
        const uint32_t xbase = smem_u32(xs);
        const uint32_t lbase = sbuf + lane * 16;
        const int c0 = ctr;
        float2 a0 = make_float2(0.f, 0.f), a1 = a0, a2 = a0, a3 = a0;
        for (int n = 0; n < nch; ++n) {
            const int g = c0 + n;
            mbar_wait(&full[g % S], static_cast<uint32_t>((g / S) & 1));
            const uint32_t cb = lbase + (g % S) * kChunkBytes;
            const uint32_t xc = xbase + n * CC * 4;
            const int cn = min(CC, cols - n * CC);
            if (cn == CC) {
#pragma unroll
                for (int j = 0; j < GPC; ++j) {
                    const uint4 w = lds128(cb + j * 512);
                    const float4 xa = lds128f(xc + j * 32), xb = lds128f(xc + j * 32 + 16);
                    a0 = __ffma2_rn(make_float2(lo_bf(w.x), hi_bf(w.x)), make_float2(xa.x, xa.y), a0);
                    a1 = __ffma2_rn(make_float2(lo_bf(w.y), hi_bf(w.y)), make_float2(xa.z, xa.w), a1);
                    a2 = __ffma2_rn(make_float2(lo_bf(w.z), hi_bf(w.z)), make_float2(xb.x, xb.y), a2);
                    a3 = __ffma2_rn(make_float2(lo_bf(w.w), hi_bf(w.w)), make_float2(xb.z, xb.w), a3);
                }
            } else {
                const int ng = cn / G;
                for (int j = 0; j < ng; ++j) {
                    const uint4 w = lds128(cb + j * 512);
                    const float4 xa = lds128f(xc + j * 32), xb = lds128f(xc + j * 32 + 16);
                    a0 = __ffma2_rn(make_float2(lo_bf(w.x), hi_bf(w.x)), make_float2(xa.x, xa.y), a0);
                    a1 = __ffma2_rn(make_float2(lo_bf(w.y), hi_bf(w.y)), make_float2(xa.z, xa.w), a1);
                    a2 = __ffma2_rn(make_float2(lo_bf(w.z), hi_bf(w.z)), make_float2(xb.x, xb.y), a2);
                    a3 = __ffma2_rn(make_float2(lo_bf(w.w), hi_bf(w.w)), make_float2(xb.z, xb.w), a3);
                }
                const int tail = cn - ng * G;
                if (tail) {
                    const uint4 w = lds128(cb + ng * 512);
                    const float* xt = xs + n * CC + ng * G;
                    for (int i = 0; i < tail; ++i) a0.x = fmaf(group_elem(w, i, WT{}), xt[i], a0.x);
                }
            }
            __syncwarp();  // every lane is done with this stage: refill it
            if (n + S < nch && elect_one()) issue(tile, cols, n + S, g + S);
        }
        ctr += nch;
        return ((a0.x + a0.y) + (a1.x + a1.y)) + ((a2.x + a2.y) + (a3.x + a3.y));
    }
};

// Tolerance-mode GEMV of one 32-row bf16 tile split over the columns across
// the CTA's warps (the exact chain cannot be split: it is one sequential
// sum).  Warp w takes a contiguous slice of 8-column groups; each lane loads
// its row's groups with 16-byte LDGs straight into registers (a warp-wide
// load is 512 contiguous bytes of the tile), NB groups in flight, the first
// batch issued before the kernel's PDL wait (weights never depend on the
// activations).  Packed FFMA partial sums per lane; the warps' sums meet in
// shared memory and warp 0 adds them in warp order (deterministic).  Used by
// the few-tile decode kernels (qkv, routers, unembed), whose single-warp
// chains are latency bound: 16 warps x 8 KB per tile go out in one round trip.
template <int NB>
struct SplitLdg {
    uint4 wv[NB];
    int g0, g1;  // this warp's groups [g0, g1)
    __device__ __forceinline__ void load(const uint16_t* tile, int gb) {
        const uint4* tp = reinterpret_cast<const uint4*>(tile) + (threadIdx.x & 31);
#pragma unroll
        for (int u = 0; u < NB; ++u)
            if (gb + u < g1) wv[u] = __ldg(tp + static_cast<long long>(gb + u) * 32);
    }
    __device__ __forceinline__ void prime(const uint16_t* tile, int cols) {
        const int nw = blockDim.x >> 5, w = threadIdx.x >> 5;
        const int ng = (cols + 7) / 8;
        const int per = (ng + nw - 1) / nw;
        g0 = min(ng, w * per);
        g1 = min(ng, g0 + per);
        load(tile, g0);
    }
    // red: [nwarps][32] floats of shared memory.  Returns the row sum in warp 0.
    __device__ __forceinline__ float run(const uint16_t* tile, int cols, const float* xs, float* red) {
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
        float2 a0 = make_float2(0.f, 0.f), a1 = a0, a2 = a0, a3 = a0;
        for (int gb = g0; gb < g1; gb += NB) {
            if (gb != g0) load(tile, gb);
#pragma unroll
            for (int u = 0; u < NB; ++u) {
                const int g = gb + u;
                if (g < g1) {
                    const uint4 wq = wv[u];
                    float4 xa = *reinterpret_cast<const float4*>(xs + g * 8);
                    float4 xb = *reinterpret_cast<const float4*>(xs + g * 8 + 4);
                    if (g * 8 + 8 > cols) {  // ragged last group: columns >= cols contribute 0
                        const int t = cols - g * 8;
                        if (t <= 0) xa.x = 0.f;
                        if (t <= 1) xa.y = 0.f;
                        if (t <= 2) xa.z = 0.f;
                        if (t <= 3) xa.w = 0.f;
                        if (t <= 4) xb.x = 0.f;
                        if (t <= 5) xb.y = 0.f;
                        if (t <= 6) xb.z = 0.f;
                        xb.w = 0.f;
                    }
                    a0 = __ffma2_rn(make_float2(lo_bf(wq.x), hi_bf(wq.x)), make_float2(xa.x, xa.y), a0);
                    a1 = __ffma2_rn(make_float2(lo_bf(wq.y), hi_bf(wq.y)), make_float2(xa.z, xa.w), a1);
                    a2 = __ffma2_rn(make_float2(lo_bf(wq.z), hi_bf(wq.z)), make_float2(xb.x, xb.y), a2);
                    a3 = __ffma2_rn(make_float2(lo_bf(wq.w), hi_bf(wq.w)), make_float2(xb.z, xb.w), a3);
                }
            }
        }
        red[w * 32 + lane] = ((a0.x + a0.y) + (a1.x + a1.y)) + ((a2.x + a2.y) + (a3.x + a3.y));
        __syncthreads();
        float s = 0.0f;
        if (w == 0)
            for (int q = 0; q < nw; ++q) s += red[q * 32 + lane];
        return s;
    }
};
constexpr int kSplitWarps = 16;       // warps per tile in the tolerance-mode split GEMVs (qkv, unembed)
constexpr int kRouterSplitWarps = 8;  // routers: 256 threads x <= 128 registers, so a side-stream
                                      // predictor CTA still fits beside three expert CTAs
using SplitG = SplitLdg<16>;

// Multi-token variant (batched prefill): the same bf16 row tile applied to nt
// <= T tokens at once — T independent sequential chains per lane, one weight
// stream.  xs: nt vectors of `xstride` floats in shared memory (16-byte
// aligned).  Every token's chain is the single-token chain bit for bit (same
// products, same column order); the T chains hide each other's FADD latency.
template <int T, typename Pipe>
__device__ inline void run_multi(Pipe& p, const uint16_t* tile, int cols, const float* xs, int xstride, int nt,
                          float (&acc)[T]) {
    constexpr int G = Pipe::G, CC = Pipe::kCC, S = Pipe::kS, GPC = CC / G;
    const int lane = threadIdx.x & 31;
    const int nch = (cols + CC - 1) / CC;
    if (lane == 0 && !p.primed)
        for (int n = 0; n < S && n < nch; ++n) p.issue(tile, cols, n, p.ctr + n);
    p.primed = 0;
    const uint32_t xbase = smem_u32(xs);
    const uint32_t lbase = p.sbuf + lane * 16;
    const int c0 = p.ctr;
#pragma unroll
    for (int t = 0; t < T; ++t) acc[t] = 0.0f;
    for (int n = 0; n < nch; ++n) {
        const int g = c0 + n;
        mbar_wait(&p.full[g % S], static_cast<uint32_t>((g / S) & 1));
        const uint32_t cb = lbase + (g % S) * Pipe::kChunkBytes;
        const int cn = min(CC, cols - n * CC);
        const int ng = cn / G;
        for (int q = 0; q < ng; ++q) {
            const uint4 w = lds128(cb + q * 512);
            const float w0 = lo_bf(w.x), w1 = hi_bf(w.x), w2 = lo_bf(w.y), w3 = hi_bf(w.y);
            const float w4 = lo_bf(w.z), w5 = hi_bf(w.z), w6 = lo_bf(w.w), w7 = hi_bf(w.w);
            const uint32_t xo = xbase + (n * CC + q * G) * 4;
            // all T chains run unconditionally (rows t >= nt compute on stale
            // staging and are discarded) so the compiler interleaves them
#pragma unroll
            for (int t = 0; t < T; ++t) {
                {
                    const float4 a = lds128f(xo + t * xstride * 4), b = lds128f(xo + t * xstride * 4 + 16);
                    const float2 p0 = __fmul2_rn(make_float2(w0, w1), make_float2(a.x, a.y));
                    const float2 p1 = __fmul2_rn(make_float2(w2, w3), make_float2(a.z, a.w));
                    const float2 p2 = __fmul2_rn(make_float2(w4, w5), make_float2(b.x, b.y));
                    const float2 p3 = __fmul2_rn(make_float2(w6, w7), make_float2(b.z, b.w));
                    float s = acc[t];
                    s = s + p0.x;
                    s = s + p0.y;
                    s = s + p1.x;
                    s = s + p1.y;
                    s = s + p2.x;
                    s = s + p2.y;
                    s = s + p3.x;
                    s = s + p3.y;
                    acc[t] = s;
                }
            }
        }
        const int tail = cn - ng * G;
        if (tail) {
            const uint4 w = lds128(cb + ng * 512);
#pragma unroll
            for (int t = 0; t < T; ++t)
                if (t < nt) {
                    const float* xt = xs + t * xstride + n * CC + ng * G;
                    for (int i = 0; i < tail; ++i) acc[t] = acc[t] + group_elem(w, i, uint16_t{}) * xt[i];
                }
        }
        __syncwarp();
        if (n + S < nch && elect_one()) p.issue(tile, cols, n + S, g + S);
    }
    __syncwarp();
    p.ctr += nch;
}

// Two row tiles of the same width against ONE input vector (fused expert
// kernel: two 32-row blocks of an expert's down projection per warp).  The
// tiles' chunks alternate through the pipe (virtual chunk 2n = tile A's chunk
// n, 2n+1 = tile B's); each lane keeps two independent chains (rows lane of A
// and of B), each in the reference's column order, so they hide each other's
// FADD latency.  Bit-identical to two run() calls.
// Issue the first chunks of a tile pair before the input vector exists.
template <typename Pipe>
__device__ inline void prime_pair(Pipe& p, const uint16_t* ta, const uint16_t* tb, int cols) {
    const int nv = 2 * ((cols + Pipe::kCC - 1) / Pipe::kCC);
    if ((threadIdx.x & 31) == 0)
        for (int v = 0; v < Pipe::kS && v < nv; ++v) p.issue((v & 1) ? tb : ta, cols, v >> 1, p.ctr + v);
    p.primed = 1;
}

template <typename Pipe>
__device__ inline void run_pair(Pipe& p, const uint16_t* ta, const uint16_t* tb, int cols, const float* xs,
                                float& acc_a, float& acc_b) {
    constexpr int G = Pipe::G, CC = Pipe::kCC, S = Pipe::kS;
    static_assert(S % 2 == 0, "pair pipe needs an even stage count");
    const int lane = threadIdx.x & 31;
    const int nch = (cols + CC - 1) / CC, nv = 2 * nch;
    const int c0 = p.ctr;
    if (lane == 0 && !p.primed)
        for (int v = 0; v < S && v < nv; ++v) p.issue((v & 1) ? tb : ta, cols, v >> 1, c0 + v);
    p.primed = 0;
    const uint32_t xbase = smem_u32(xs);
    const uint32_t lbase = p.sbuf + lane * 16;
    float a = 0.0f, b = 0.0f;
    for (int n = 0; n < nch; ++n) {
        const int ga = c0 + 2 * n, gb = ga + 1;
        mbar_wait(&p.full[ga % S], static_cast<uint32_t>((ga / S) & 1));
        mbar_wait(&p.full[gb % S], static_cast<uint32_t>((gb / S) & 1));
        const uint32_t ca = lbase + (ga % S) * Pipe::kChunkBytes, cbb = lbase + (gb % S) * Pipe::kChunkBytes;
        const int cn = min(CC, cols - n * CC);
        const int ng = cn / G;
        const uint32_t xo = xbase + n * CC * 4;
        int q = 0;
        for (; q + 1 < ng; q += 2) {  // two groups per step: four independent loads in flight
            const uint4 wa0 = lds128(ca + q * 512), wb0 = lds128(cbb + q * 512);
            const uint4 wa1 = lds128(ca + (q + 1) * 512), wb1 = lds128(cbb + (q + 1) * 512);
            const XG x0 = load_x(xo + q * G * 4, uint16_t{}), x1 = load_x(xo + (q + 1) * G * 4, uint16_t{});
            a = chain_group(a, wa0, x0, uint16_t{});
            b = chain_group(b, wb0, x0, uint16_t{});
            a = chain_group(a, wa1, x1, uint16_t{});
            b = chain_group(b, wb1, x1, uint16_t{});
        }
        for (; q < ng; ++q) {
            const XG x0 = load_x(xo + q * G * 4, uint16_t{});
            a = chain_group(a, lds128(ca + q * 512), x0, uint16_t{});
            b = chain_group(b, lds128(cbb + q * 512), x0, uint16_t{});
        }
        const int tail = cn - ng * G;
        if (tail) {
            const uint4 wa = lds128(ca + ng * 512), wb = lds128(cbb + ng * 512);
            const float* xt = xs + n * CC + ng * G;
            for (int i = 0; i < tail; ++i) {
                a = a + group_elem(wa, i, uint16_t{}) * xt[i];
                b = b + group_elem(wb, i, uint16_t{}) * xt[i];
            }
        }
        __syncwarp();  // both stages consumed by every lane: refill them
        if (elect_one()) {
            const int va = 2 * n + S, vb = va + 1;
            if (va < nv) p.issue(ta, cols, va >> 1, c0 + va);
            if (vb < nv) p.issue(tb, cols, vb >> 1, c0 + vb);
        }
    }
    __syncwarp();
    p.ctr += nv;
    acc_a = a;
    acc_b = b;
}

constexpr int kS = 4;       // stages per warp
constexpr int kCCb = 128;   // bf16 columns per chunk (8 KB)
constexpr int kCCf = 64;    // f32 columns per chunk (8 KB)
constexpr int kCCd = 192;   // down-projection columns per chunk (12 KB: a 768-column Q30 tile = 4 chunks, all in flight)
using PipeB = WarpPipe<uint16_t, kS, kCCb>;
#ifndef SMOE_GU_STAGES
#define SMOE_GU_STAGES 6
#endif
#ifndef SMOE_GU_CC
#define SMOE_GU_CC 128
#endif
using PipeGU = WarpPipe<uint16_t, SMOE_GU_STAGES, SMOE_GU_CC>;  // expert gate/up: deeper HBM stream per warp
using PipeBL = WarpPipe<uint16_t, kS, 256>;  // 16 KB chunks: few-CTA kernels (qkv, router, final)
using PipeF = WarpPipe<float, kS, kCCf>;
#ifndef SMOE_D_STAGES
#define SMOE_D_STAGES kS
#endif
#ifndef SMOE_D_CC
#define SMOE_D_CC kCCd
#endif
using PipeD = WarpPipe<uint16_t, SMOE_D_STAGES, SMOE_D_CC>;
using PipeR = WarpPipe<uint16_t, 3, 256>;  // router: 48 KB, fits beside three k_ffn_gu CTAs

// -------------------------------------------------------------- decision --
#ifdef DECISION_TIMING
__device__ long long g_dec_t[8];
#define DEC_T(i) do { __syncwarp(); if ((threadIdx.x & 31) == 0) g_dec_t[i] = clock64(); } while (0)
#else
#define DEC_T(i) do {} while (0)
#endif
//
// make_decision (model.cpp:258-274) for one logits row, executed by warp 0.
// softmax (numerics.cpp:37-54): f32 max, f64 exp, f64 partition summed in
// index order by lane 0 (exactly the reference's order), f32 probabilities;
// top_k (numerics.cpp:56-70): value desc, lower index first; gates renormalised
// by an f32 sum in rank order.  topk-softmax: top_k on logits, softmax of the k.
__device__ inline void warp_decision_rank(const float* logits, int E, int K, int gating, float* sp /*smem E*/,
                              double* se /*smem E*/, int* ids, float* gates) {
    const int lane = threadIdx.x & 31;
    DEC_T(0);
    // logits were written by other CTAs: L2 loads, all in flight, into smem
    for (int i0 = 0; i0 < E; i0 += 8 * 32) {
        float t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u * 32 + lane;
            t[u] = i < E ? __ldcg(logits + i) : 0.0f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u * 32 + lane;
            if (i < E) sp[i] = t[u];
        }
    }
    __syncwarp();
    DEC_T(1);
    if (gating == kSoftmaxTopK) {
        float mx = -INFINITY;
        for (int i = lane; i < E; i += 32) mx = fmaxf(mx, sp[i]);
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        // independent f64 exps per lane, 8 in flight (the routine is a long
        // dependent DFMA chain)
        for (int i0 = 0; i0 < E; i0 += 8 * 32) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = i0 + u * 32 + lane;
                if (i < E) se[i] = exp_glibc(static_cast<double>(sp[i]) - static_cast<double>(mx));
            }
        }
        __syncwarp();
        double z = 0.0;
        if (lane == 0)  // f64 partition in index order, as numerics.cpp:46-49
            for (int i = 0; i < E; ++i) z += se[i];
        z = __shfl_sync(0xffffffffu, z, 0);
        for (int i0 = 0; i0 < E; i0 += 8 * 32) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = i0 + u * 32 + lane;
                if (i < E) sp[i] = static_cast<float>(se[i] / z);
            }
        }
        __syncwarp();
    }
    DEC_T(2);
    // top_k (numerics.cpp:56-70): value descending, lower index first on ties.
    // Each element becomes a 64-bit key (order-preserving bits of the value,
    // then the inverted index), every lane keeps its elements' keys in
    // registers, and each of the K rounds takes the warp maximum with two
    // REDUX.MAX (high word, then low word among the lanes holding it).
    __shared__ int s_sel[kMaxK];
    __shared__ float s_val[kMaxK];
    if (E <= 8 * 32) {
        unsigned hi[8], lo[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = u * 32 + lane;
            if (i < E) {
                unsigned b = __float_as_uint(sp[i]);
                hi[u] = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
                lo[u] = 0xFFFFFFFFu - static_cast<unsigned>(i);
            } else {
                hi[u] = 0;
                lo[u] = 0;
            }
        }
        for (int t = 0; t < K; ++t) {
            unsigned mh = 0, ml = 0;
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (hi[u] > mh || (hi[u] == mh && lo[u] > ml)) {
                    mh = hi[u];
                    ml = lo[u];
                }
            const unsigned wh = __reduce_max_sync(0xffffffffu, mh);
            const unsigned wl = __reduce_max_sync(0xffffffffu, mh == wh ? ml : 0u);
            const int i = static_cast<int>(0xFFFFFFFFu - wl);
            if ((i & 31) == lane) {  // the owner drops the winner from its keys
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (u == (i >> 5)) {
                        hi[u] = 0;
                        lo[u] = 0;
                    }
            }
            if (lane == 0) {
                s_sel[t] = i;
                s_val[t] = sp[i];
            }
        }
    } else {  // large E: rank of i = #{j : v_j > v_i or (v_j == v_i and j < i)}
        for (int i0 = 0; i0 < E; i0 += 4 * 32) {
            float x[4];
            int rank[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * 32 + lane;
                x[u] = i < E ? sp[i] : 0.0f;
                rank[u] = 0;
            }
            for (int j = 0; j < E; ++j) {
                const float y = sp[j];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = i0 + u * 32 + lane;
                    rank[u] += (y > x[u]) | ((y == x[u]) & (j < i));
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * 32 + lane;
                if (i < E && rank[u] < K) {
                    s_sel[rank[u]] = i;
                    s_val[rank[u]] = x[u];
                }
            }
        }
    }
    __syncwarp();
    DEC_T(3);
    if (lane == 0) {
        if (gating == kSoftmaxTopK) {  // gates renormalised by an f32 sum in rank order
            float total = 0.0f;
            for (int t = 0; t < K; ++t) total += s_val[t];
            for (int t = 0; t < K; ++t) {
                ids[t] = s_sel[t];
                gates[t] = s_val[t] / total;
            }
        } else {  // topk-softmax: softmax of the k selected logits (f64 exp, f32 out)
            float mx = s_val[0];
            for (int t = 0; t < K; ++t) mx = fmaxf(mx, s_val[t]);
            double e[kMaxK], z = 0.0;
#pragma unroll
            for (int t = 0; t < kMaxK; ++t)
                if (t < K) e[t] = exp_glibc(static_cast<double>(s_val[t]) - static_cast<double>(mx));
#pragma unroll
            for (int t = 0; t < kMaxK; ++t)
                if (t < K) z += e[t];
#pragma unroll
            for (int t = 0; t < kMaxK; ++t)
                if (t < K) {
                    ids[t] = s_sel[t];
                    gates[t] = static_cast<float>(e[t] / z);
                }
        }
    }
    __syncwarp();
    DEC_T(4);
}

// f32(e / z) for e >= 0, z >= 1 without a division per element: q = e * (1/z)
// is within 3 double ulps of fl64(e / z) (two roundings), so the two round to
// the same f32 unless an f32 rounding midpoint (low 29 mantissa bits = 2^28)
// lies within a few ulps of q, or the result is f32-subnormal; those take the
// exact division.  Bit-identical to static_cast<float>(e / z) by construction.
__device__ __forceinline__ float div_to_f32(double e, double z, double rz) {
    if (e == 0.0) return 0.0f;  // 0 / z (underflowed exponentials, padding)
    const double q = e * rz;
    const long long b = __double_as_longlong(q);
    const int low = static_cast<int>(b & ((1ll << 29) - 1)) - (1 << 28);
    if (q < 2.3509887016445750e-38 || (low < 64 && low > -64)) return static_cast<float>(e / z);
    return static_cast<float>(q);
}

// Order-preserving u32 key of an f32 (larger value -> larger key).
__device__ __forceinline__ unsigned f32_key(float x) {
    const unsigned b = __float_as_uint(x);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float key_f32(unsigned k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// make_decision (model.cpp:258-274) for one logits row, executed by one warp,
// E <= 256 (larger E: warp_decision_rank).
// softmax (numerics.cpp:37-54): f32 max, f64 exp per element (glibc's
// algorithm), the f64 partition summed in index order by lane 0 (exactly the
// reference's order), f32 probabilities (div_to_f32).
// top_k (numerics.cpp:56-70): value descending, lower index first on ties.
// Each lane holds elements lane, lane+32, ... (ascending index), sorts its
// (key, index) list with a sorting network, and K rounds take the warp
// maximum of the list heads (REDUX on the key, then on the inverted index
// among equal keys); the winner's lane pops its head.  Lane t keeps round t.
// Gates: softmax-topk-renorm — p_t / (f32 sum of the K in rank order);
// topk-softmax — f64 softmax of the K selected logits (rank order), f32 out.
__device__ inline void warp_decision(const float* logits, int E, int K, int gating, float* sp /*smem E*/,
                                     double* se /*smem E*/, int* ids, float* gates) {
    if (E > 256) {
        warp_decision_rank(logits, E, K, gating, sp, se, ids, gates);
        return;
    }
    const int lane = threadIdx.x & 31;
    constexpr int U = 8;
    DEC_T(0);
    float v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int i = u * 32 + lane;
        v[u] = i < E ? __ldcg(logits + i) : 0.0f;
    }
    DEC_T(1);
    if (gating == kSoftmaxTopK) {
        float mx = -INFINITY;
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (u * 32 + lane < E) mx = fmaxf(mx, v[u]);
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        double e[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = u * 32 + lane;
            e[u] = i < E ? exp_glibc(static_cast<double>(v[u]) - static_cast<double>(mx)) : 0.0;
            if (i < E) se[i] = e[u];
        }
        __syncwarp();
        double z = 0.0;
        if (lane == 0) {  // f64 partition in index order, as numerics.cpp:46-49
            int i = 0;
            for (; i + 8 <= E; i += 8) {  // loads of a block in flight together, adds in order
                double t[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) t[q] = se[i + q];
#pragma unroll
                for (int q = 0; q < 8; ++q) z += t[q];
            }
            for (; i < E; ++i) z += se[i];
        }
        z = __shfl_sync(0xffffffffu, z, 0);
        const double rz = 1.0 / z;
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = div_to_f32(e[u], z, rz);
        __syncwarp();
    }
    DEC_T(2);
    // per-lane (key, index) lists, sorted by key desc then index asc
    unsigned kk[U];
    int ix[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int i = u * 32 + lane;
        kk[u] = i < E ? f32_key(v[u]) : 0u;
        ix[u] = i;
    }
    // Batcher odd-even merge sort of 8 (19 compare-exchanges); pairs (a, b)
    // with a < b hold lower indices at a, so "b first" only on a strictly
    // larger key keeps index order among equal keys
#define SMOE_CX(a, b)                                             \
    do {                                                          \
        if (kk[b] > kk[a]) {                                      \
            const unsigned tk = kk[a];                            \
            kk[a] = kk[b];                                        \
            kk[b] = tk;                                           \
            const int ti = ix[a];                                 \
            ix[a] = ix[b];                                        \
            ix[b] = ti;                                           \
        } else if (kk[b] == kk[a] && ix[b] < ix[a]) {             \
            const int ti = ix[a];                                 \
            ix[a] = ix[b];                                        \
            ix[b] = ti;                                           \
        }                                                         \
    } while (0)
    SMOE_CX(0, 1); SMOE_CX(2, 3); SMOE_CX(4, 5); SMOE_CX(6, 7);
    SMOE_CX(0, 2); SMOE_CX(1, 3); SMOE_CX(4, 6); SMOE_CX(5, 7);
    SMOE_CX(1, 2); SMOE_CX(5, 6);
    SMOE_CX(0, 4); SMOE_CX(1, 5); SMOE_CX(2, 6); SMOE_CX(3, 7);
    SMOE_CX(2, 4); SMOE_CX(3, 5);
    SMOE_CX(1, 2); SMOE_CX(3, 4); SMOE_CX(5, 6);
#undef SMOE_CX
    int my_idx = 0;
    float my_val = 0.0f;
    for (int t = 0; t < K; ++t) {
        const unsigned wk = __reduce_max_sync(0xffffffffu, kk[0]);
        const unsigned wi = __reduce_max_sync(0xffffffffu, kk[0] == wk ? 0xFFFFFFFFu - static_cast<unsigned>(ix[0]) : 0u);
        const int idx = static_cast<int>(0xFFFFFFFFu - wi);
        if ((idx & 31) == lane) {  // pop the head
#pragma unroll
            for (int u = 0; u + 1 < U; ++u) {
                kk[u] = kk[u + 1];
                ix[u] = ix[u + 1];
            }
            kk[U - 1] = 0u;
            ix[U - 1] = 0x7fffffff;
        }
        if (lane == t) {
            my_idx = idx;
            my_val = key_f32(wk);
        }
    }
    DEC_T(3);
    if (gating == kSoftmaxTopK) {  // gates renormalised by an f32 sum in rank order
        float total = 0.0f;
        for (int t = 0; t < K; ++t) total += __shfl_sync(0xffffffffu, my_val, t);
        if (lane < K) {
            ids[lane] = my_idx;
            gates[lane] = my_val / total;
        }
    } else {  // topk-softmax: softmax of the k selected logits (f64 exp, f32 out)
        float mx = lane < K ? my_val : -INFINITY;
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const double e = lane < K ? exp_glibc(static_cast<double>(my_val) - static_cast<double>(mx)) : 0.0;
        double z = 0.0;
        for (int t = 0; t < K; ++t) z += __shfl_sync(0xffffffffu, e, t);
        if (lane < K) {
            ids[lane] = my_idx;
            gates[lane] = static_cast<float>(e / z);
        }
    }
    __syncwarp();
    DEC_T(4);
}

// Tolerance-mode make_decision (model.cpp:258-274) for E <= 256: the top-k is
// taken on the logits themselves (exp is monotonic, so the order equals the
// order of the softmax probabilities except where two probabilities round to
// the same f32 — a near-tie the parity checker reports), and the gates of
// both gating orders are, in real arithmetic, the softmax of the K selected
// logits (softmax-topk-renorm: p_i / sum_top p_j = e_i / sum_top e_j, the
// partition cancels), computed in f32.  No f64 exponentials over all E and no
// sequential partition: ~1/4 of warp_decision's cycles.
__device__ inline void warp_decision_fast(const float* logits, int E, int K, int* ids, float* gates) {
    const int lane = threadIdx.x & 31;
    constexpr int U = 8;
    unsigned kk[U];
    int ix[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int i = u * 32 + lane;
        kk[u] = i < E ? f32_key(__ldcg(logits + i)) : 0u;
        ix[u] = i;
    }
#define SMOE_CX(a, b)                                             \
    do {                                                          \
        if (kk[b] > kk[a] || (kk[b] == kk[a] && ix[b] < ix[a])) { \
            const unsigned tk = kk[a];                            \
            kk[a] = kk[b];                                        \
            kk[b] = tk;                                           \
            const int ti = ix[a];                                 \
            ix[a] = ix[b];                                        \
            ix[b] = ti;                                           \
        }                                                         \
    } while (0)
    SMOE_CX(0, 1); SMOE_CX(2, 3); SMOE_CX(4, 5); SMOE_CX(6, 7);
    SMOE_CX(0, 2); SMOE_CX(1, 3); SMOE_CX(4, 6); SMOE_CX(5, 7);
    SMOE_CX(1, 2); SMOE_CX(5, 6);
    SMOE_CX(0, 4); SMOE_CX(1, 5); SMOE_CX(2, 6); SMOE_CX(3, 7);
    SMOE_CX(2, 4); SMOE_CX(3, 5);
    SMOE_CX(1, 2); SMOE_CX(3, 4); SMOE_CX(5, 6);
#undef SMOE_CX
    int my_idx = 0;
    float my_val = -INFINITY;
    for (int t = 0; t < K; ++t) {
        const unsigned wk = __reduce_max_sync(0xffffffffu, kk[0]);
        const unsigned wi = __reduce_max_sync(0xffffffffu, kk[0] == wk ? 0xFFFFFFFFu - static_cast<unsigned>(ix[0]) : 0u);
        const int idx = static_cast<int>(0xFFFFFFFFu - wi);
        if ((idx & 31) == lane) {
#pragma unroll
            for (int u = 0; u + 1 < U; ++u) {
                kk[u] = kk[u + 1];
                ix[u] = ix[u + 1];
            }
            kk[U - 1] = 0u;
            ix[U - 1] = 0x7fffffff;
        }
        if (lane == t) {
            my_idx = idx;
            my_val = key_f32(wk);
        }
    }
    const float mx = __shfl_sync(0xffffffffu, my_val, 0);  // rank 0 holds the maximum
    const float e = lane < K ? __expf(my_val - mx) : 0.0f;
    float z = e;
    for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
    if (lane < K) {
        ids[lane] = my_idx;
        gates[lane] = e / z;
    }
    __syncwarp();
}

// ------------------------------------------------------------- launching --
// Every decode-path kernel is launched with programmatic stream
// serialization (PDL); captured into the step graph as programmatic edges.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    // the stream's priority as a launch attribute, so it survives graph capture
    int prio = 0;
    cudaStreamGetPriority(s, &prio);
    attr[1].id = cudaLaunchAttributePriority;
    attr[1].val.priority = prio;
    static const bool no_pdl = std::getenv("SMOE_NO_PDL") != nullptr;  // diagnostics
    cfg.attrs = no_pdl ? attr + 1 : attr;
    cfg.numAttrs = no_pdl ? 1 : 2;
    return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}
#define PDL(k, grid, block, smem, s, ...)                                   \
    do {                                                                    \
        cudaError_t e_ = launch_pdl(k, dim3(grid), dim3(block), smem, s, __VA_ARGS__); \
        if (e_ != cudaSuccess) return e_;                                   \
    } while (0)

}  // namespace smoe
