// Microbenchmark of the sequential-chain GEMV inner loop (tools only).
// One CTA per SM, 1..4 warps, each warp owns a 32-row tile held in shared
// memory (grouped layout: lane's 8 consecutive bf16 columns = 16 bytes), x in
// shared memory; measures cycles per column per warp for loop variants.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 lds128(uint32_t a) { uint4 v; asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a)); return v; }
__device__ __forceinline__ float4 lds128f(uint32_t a) { float4 v; asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a)); return v; }
__device__ __forceinline__ uint4 lds128nv(uint32_t a) { uint4 v; asm("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a)); return v; }
__device__ __forceinline__ float4 lds128fnv(uint32_t a) { float4 v; asm("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a)); return v; }
__device__ __forceinline__ float lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

constexpr int COLS = 512;  // per tile in smem (16 KB bf16 + 4 KB x)
extern __shared__ __align__(16) unsigned char sm[];

template <int V>
__global__ void kbench(float* out, long long* cyc, int reps) {
    uint16_t* w = reinterpret_cast<uint16_t*>(sm);          // [COLS/8][32][8] per warp-tile
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* x = reinterpret_cast<float*>(sm + 4 * COLS * 64); // up to 4 tiles
    for (int i = threadIdx.x; i < 4 * COLS * 32; i += blockDim.x) w[i] = (uint16_t)(0x3f80 + (i % 7));
    for (int i = threadIdx.x; i < COLS; i += blockDim.x) x[i] = 1.0f / (1 + i % 5);
    __syncthreads();
    const uint32_t wb = (uint32_t)__cvta_generic_to_shared(w) + warp * COLS * 64 + lane * 16;
    const uint32_t xb = (uint32_t)__cvta_generic_to_shared(x);
    float acc = 0.f, acc2 = 0.f;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        if (V == 0) {  // current: loads one group ahead, chain per group
            uint4 wn = lds128(wb); float4 xa = lds128f(xb), xc = lds128f(xb + 16);
#pragma unroll 4
            for (int q = 0; q < COLS / 8; ++q) {
                uint4 ww = wn; float4 a = xa, c = xc;
                if (q + 1 < COLS / 8) { wn = lds128(wb + (q + 1) * 512); xa = lds128f(xb + (q + 1) * 32); xc = lds128f(xb + (q + 1) * 32 + 16); }
                acc = acc + lo(ww.x) * a.x; acc = acc + hi(ww.x) * a.y; acc = acc + lo(ww.y) * a.z; acc = acc + hi(ww.y) * a.w;
                acc = acc + lo(ww.z) * c.x; acc = acc + hi(ww.z) * c.y; acc = acc + lo(ww.w) * c.z; acc = acc + hi(ww.w) * c.w;
            }
        } else if (V == 1) {  // non-volatile loads, full unroll 8, compiler schedules freely
#pragma unroll 8
            for (int q = 0; q < COLS / 8; ++q) {
                uint4 ww = lds128nv(wb + q * 512); float4 a = lds128fnv(xb + q * 32), c = lds128fnv(xb + q * 32 + 16);
                acc = acc + lo(ww.x) * a.x; acc = acc + hi(ww.x) * a.y; acc = acc + lo(ww.y) * a.z; acc = acc + hi(ww.y) * a.w;
                acc = acc + lo(ww.z) * c.x; acc = acc + hi(ww.z) * c.y; acc = acc + lo(ww.w) * c.z; acc = acc + hi(ww.w) * c.w;
            }
        } else if (V == 2) {  // products one group ahead (registers), sum group behind
            float p[8], pn[8];
            { uint4 ww = lds128nv(wb); float4 a = lds128fnv(xb), c = lds128fnv(xb + 16);
              p[0]=lo(ww.x)*a.x; p[1]=hi(ww.x)*a.y; p[2]=lo(ww.y)*a.z; p[3]=hi(ww.y)*a.w; p[4]=lo(ww.z)*c.x; p[5]=hi(ww.z)*c.y; p[6]=lo(ww.w)*c.z; p[7]=hi(ww.w)*c.w; }
#pragma unroll 4
            for (int q = 0; q < COLS / 8; ++q) {
                if (q + 1 < COLS / 8) { uint4 ww = lds128nv(wb + (q + 1) * 512); float4 a = lds128fnv(xb + (q + 1) * 32), c = lds128fnv(xb + (q + 1) * 32 + 16);
                  pn[0]=lo(ww.x)*a.x; pn[1]=hi(ww.x)*a.y; pn[2]=lo(ww.y)*a.z; pn[3]=hi(ww.y)*a.w; pn[4]=lo(ww.z)*c.x; pn[5]=hi(ww.z)*c.y; pn[6]=lo(ww.w)*c.z; pn[7]=hi(ww.w)*c.w; }
#pragma unroll
                for (int i = 0; i < 8; ++i) acc = acc + p[i];
#pragma unroll
                for (int i = 0; i < 8; ++i) p[i] = pn[i];
            }
        } else if (V == 3) {  // two tiles per warp (2 independent chains per lane)
            const uint32_t wb2 = wb + COLS * 64;
#pragma unroll 4
            for (int q = 0; q < COLS / 8; ++q) {
                uint4 ww = lds128nv(wb + q * 512), w2 = lds128nv(wb2 + q * 512); float4 a = lds128fnv(xb + q * 32), c = lds128fnv(xb + q * 32 + 16);
                acc = acc + lo(ww.x) * a.x; acc2 = acc2 + lo(w2.x) * a.x; acc = acc + hi(ww.x) * a.y; acc2 = acc2 + hi(w2.x) * a.y;
                acc = acc + lo(ww.y) * a.z; acc2 = acc2 + lo(w2.y) * a.z; acc = acc + hi(ww.y) * a.w; acc2 = acc2 + hi(w2.y) * a.w;
                acc = acc + lo(ww.z) * c.x; acc2 = acc2 + lo(w2.z) * c.x; acc = acc + hi(ww.z) * c.y; acc2 = acc2 + hi(w2.z) * c.y;
                acc = acc + lo(ww.w) * c.z; acc2 = acc2 + lo(w2.w) * c.z; acc = acc + hi(ww.w) * c.w; acc2 = acc2 + hi(w2.w) * c.w;
            }
        } else if (V == 4) {  // x held as pre-duplicated? no: plain scalar LDS per column (baseline naive)
            const uint16_t* wl = w + warp * COLS * 32 + lane * 8;
            for (int c = 0; c < COLS; ++c) acc = acc + __uint_as_float(((uint32_t)wl[(c / 8) * 256 + c % 8]) << 16) * x[c];
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + acc2;
    if (lane == 0) cyc[blockIdx.x * 4 + warp] = t1 - t0;
}

int main() {
    float* out; long long* cyc; cudaMalloc(&out, 1 << 22); cudaMalloc(&cyc, 1 << 16);
    const int smem = 4 * COLS * 64 + COLS * 4;
    const char* names[] = {"V0 current (volatile lds, 1 group ahead)", "V1 nonvolatile unroll8", "V2 products 1 group ahead", "V3 two tiles/warp", "V4 naive scalar"};
    void (*ks[])(float*, long long*, int) = {kbench<0>, kbench<1>, kbench<2>, kbench<3>, kbench<4>};
    for (int v = 0; v < 5; ++v) {
        cudaFuncSetAttribute(ks[v], cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int nw : {1, 2, 4}) {
            ks[v]<<<148, 32 * nw, smem>>>(out, cyc, 2);
            cudaDeviceSynchronize();
            ks[v]<<<148, 32 * nw, smem>>>(out, cyc, 8);
            cudaDeviceSynchronize();
            long long h[4]; cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
            double cols = 8.0 * COLS * (v == 3 ? 1 : 1);
            printf("%-45s warps/CTA %d: %.2f cycles/column/warp (%s)\n", names[v], nw, h[0] / cols, v == 3 ? "64 rows/warp" : "32 rows/warp");
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
