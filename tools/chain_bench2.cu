// Microbenchmark (tools only): cycles per column of one 32-row sequential
// f32 chain tile (bf16 weights, grouped layout: lane's 8 consecutive columns =
// 16 bytes) with the tile already in shared memory.  Variants:
//   A  current single-warp loop (scalar FMUL + FADD, volatile LDS)
//   B  single warp, FMUL2 products (two columns per instruction) + scalar FADD chain
//   C  warp-specialised: producer warp (LDS, unpack, FMUL2, STS products) and
//      consumer warp (LDS.128 products + FADD chain), named-barrier ring
// Reports cycles/column for 1..4 tiles per SM (CTAs per SM).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ float4 lds128f(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts128f(uint32_t a, float4 v) {
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ float lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
// two rounded products {a0*b0, a1*b1} with one FMUL2
__device__ __forceinline__ float2 mul2(float a0, float a1, float b0, float b1) {
    unsigned long long a, b, p;
    asm("mov.b64 %0, {%1,%2};" : "=l"(a) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1,%2};" : "=l"(b) : "f"(b0), "f"(b1));
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(p) : "l"(a), "l"(b));
    float2 r;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(p));
    return r;
}

constexpr int COLS = 1024;  // columns per tile held in smem
extern __shared__ __align__(16) unsigned char sm[];

template <int V>
__global__ void kbench(float* out, long long* cyc, int reps) {
    uint16_t* w = reinterpret_cast<uint16_t*>(sm);                 // [COLS/8][32][8]
    float* x = reinterpret_cast<float*>(sm + COLS * 64);           // [COLS]
    float* pr = x + COLS;                                          // products ring [4][64 cols][32]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < COLS * 32; i += blockDim.x) w[i] = (uint16_t)(0x3f80 + (i % 7));
    for (int i = threadIdx.x; i < COLS; i += blockDim.x) x[i] = 1.0f / (1 + i % 5);
    __syncthreads();
    const uint32_t wb = (uint32_t)__cvta_generic_to_shared(w) + lane * 16;
    const uint32_t xb = (uint32_t)__cvta_generic_to_shared(x);
    const uint32_t pb = (uint32_t)__cvta_generic_to_shared(pr) + lane * 16;
    float acc = 0.f;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        if (V == 0) {
            uint4 wn = lds128(wb);
            float4 xa = lds128f(xb), xc = lds128f(xb + 16);
#pragma unroll 4
            for (int q = 0; q < COLS / 8; ++q) {
                uint4 ww = wn;
                float4 a = xa, c = xc;
                if (q + 1 < COLS / 8) {
                    wn = lds128(wb + (q + 1) * 512);
                    xa = lds128f(xb + (q + 1) * 32);
                    xc = lds128f(xb + (q + 1) * 32 + 16);
                }
                acc = acc + lo(ww.x) * a.x; acc = acc + hi(ww.x) * a.y; acc = acc + lo(ww.y) * a.z; acc = acc + hi(ww.y) * a.w;
                acc = acc + lo(ww.z) * c.x; acc = acc + hi(ww.z) * c.y; acc = acc + lo(ww.w) * c.z; acc = acc + hi(ww.w) * c.w;
            }
        } else if (V == 1) {
            uint4 wn = lds128(wb);
            float4 xa = lds128f(xb), xc = lds128f(xb + 16);
#pragma unroll 4
            for (int q = 0; q < COLS / 8; ++q) {
                uint4 ww = wn;
                float4 a = xa, c = xc;
                if (q + 1 < COLS / 8) {
                    wn = lds128(wb + (q + 1) * 512);
                    xa = lds128f(xb + (q + 1) * 32);
                    xc = lds128f(xb + (q + 1) * 32 + 16);
                }
                const float2 p0 = mul2(lo(ww.x), hi(ww.x), a.x, a.y);
                const float2 p1 = mul2(lo(ww.y), hi(ww.y), a.z, a.w);
                const float2 p2 = mul2(lo(ww.z), hi(ww.z), c.x, c.y);
                const float2 p3 = mul2(lo(ww.w), hi(ww.w), c.z, c.w);
                acc = acc + p0.x; acc = acc + p0.y; acc = acc + p1.x; acc = acc + p1.y;
                acc = acc + p2.x; acc = acc + p2.y; acc = acc + p3.x; acc = acc + p3.y;
            }
        } else {
            // producer (odd warp of the pair) / consumer (even warp); ring of 4 slots x 64 columns
            constexpr int SC = 64, NS = 4;
            const int pair = warp >> 1;  // only 1 pair per CTA in this bench
            (void)pair;
            if (warp & 1) {  // producer
                for (int n = 0; n < COLS / SC; ++n) {
                    const int s = n % NS;
                    if (n >= NS) asm volatile("bar.sync %0, 64;" ::"r"(1 + NS + s));  // slot free
#pragma unroll 4
                    for (int q = 0; q < SC / 8; ++q) {
                        const int g = n * SC / 8 + q;
                        const uint4 ww = lds128(wb + g * 512);
                        const float4 a = lds128f(xb + g * 32), c = lds128f(xb + g * 32 + 16);
                        const float2 p0 = mul2(lo(ww.x), hi(ww.x), a.x, a.y);
                        const float2 p1 = mul2(lo(ww.y), hi(ww.y), a.z, a.w);
                        const float2 p2 = mul2(lo(ww.z), hi(ww.z), c.x, c.y);
                        const float2 p3 = mul2(lo(ww.w), hi(ww.w), c.z, c.w);
                        const uint32_t d = pb + (s * SC / 4 + q * 2) * 512;
                        sts128f(d, make_float4(p0.x, p0.y, p1.x, p1.y));
                        sts128f(d + 512, make_float4(p2.x, p2.y, p3.x, p3.y));
                    }
                    asm volatile("bar.arrive %0, 64;" ::"r"(1 + s));  // slot full
                }
                for (int s = 0; s < NS; ++s) asm volatile("bar.sync %0, 64;" ::"r"(1 + NS + s));
            } else {  // consumer
                for (int n = 0; n < COLS / SC; ++n) {
                    const int s = n % NS;
                    asm volatile("bar.sync %0, 64;" ::"r"(1 + s));
                    const uint32_t src = pb + s * SC / 4 * 512;
                    float4 pn = lds128f(src);
#pragma unroll 4
                    for (int q = 0; q < SC / 4; ++q) {
                        const float4 p = pn;
                        if (q + 1 < SC / 4) pn = lds128f(src + (q + 1) * 512);
                        acc = acc + p.x; acc = acc + p.y; acc = acc + p.z; acc = acc + p.w;
                    }
                    asm volatile("bar.arrive %0, 64;" ::"r"(1 + NS + s));
                }
            }
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (lane == 0 && warp == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    float* out;
    long long* cyc;
    cudaMalloc(&out, 1 << 24);
    cudaMalloc(&cyc, 1 << 16);
    const int smem = COLS * 64 + COLS * 4 + 4 * 64 * 32 * 4;
    const char* names[] = {"A scalar FMUL+FADD (current)", "B FMUL2 + FADD chain", "C producer/consumer warps"};
    void (*ks[])(float*, long long*, int) = {kbench<0>, kbench<1>, kbench<2>};
    for (int v = 0; v < 3; ++v) {
        cudaFuncSetAttribute(ks[v], cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const int threads = v == 2 ? 64 : 32;
        for (int per_sm : {1, 2, 3}) {
            ks[v]<<<148 * per_sm, threads, smem>>>(out, cyc, 2);
            cudaDeviceSynchronize();
            ks[v]<<<148 * per_sm, threads, smem>>>(out, cyc, 8);
            cudaDeviceSynchronize();
            long long h[148 * 3];
            cudaMemcpy(h, cyc, sizeof(long long) * 148 * per_sm, cudaMemcpyDeviceToHost);
            double mx = 0, avg = 0;
            for (int i = 0; i < 148 * per_sm; ++i) { mx = h[i] > mx ? h[i] : mx; avg += h[i]; }
            avg /= 148 * per_sm;
            printf("%-32s tiles/SM %d: %.2f cycles/column (avg), %.2f (max)\n", names[v], per_sm,
                   avg / (8.0 * COLS), mx / (8.0 * COLS));
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
