// Microbenchmark (tools only): cycles per column of the sequential f32 chain
// over a 32-row bf16 tile in shared memory (grouped layout), single warp.
// Template knobs: ALU-pipe unpack (PRMT/LOP3 instead of IMAD.SHL), FMUL2
// products, register prefetch distance (groups of 8 columns).
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
template <bool P> __device__ __forceinline__ float lo(uint32_t w) {
    if (P) { uint32_t r; asm("prmt.b32 %0, %1, 0, 0x1044;" : "=r"(r) : "r"(w)); return __uint_as_float(r); }
    return __uint_as_float(w << 16);
}
template <bool P> __device__ __forceinline__ float hi(uint32_t w) {
    if (P) { uint32_t r; asm("lop3.b32 %0, %1, 0xffff0000, 0, 0xc0;" : "=r"(r) : "r"(w)); return __uint_as_float(r); }
    return __uint_as_float(w & 0xffff0000u);
}
__device__ __forceinline__ float2 mul2(float a0, float a1, float b0, float b1) {
    unsigned long long a, b, p;
    asm("mov.b64 %0, {%1,%2};" : "=l"(a) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1,%2};" : "=l"(b) : "f"(b0), "f"(b1));
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(p) : "l"(a), "l"(b));
    float2 r;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(p));
    return r;
}
template <bool P, bool M2>
__device__ __forceinline__ float group(float acc, uint4 w, float4 a, float4 c) {
    if (M2) {
        const float2 p0 = mul2(lo<P>(w.x), hi<P>(w.x), a.x, a.y);
        const float2 p1 = mul2(lo<P>(w.y), hi<P>(w.y), a.z, a.w);
        const float2 p2 = mul2(lo<P>(w.z), hi<P>(w.z), c.x, c.y);
        const float2 p3 = mul2(lo<P>(w.w), hi<P>(w.w), c.z, c.w);
        acc = acc + p0.x; acc = acc + p0.y; acc = acc + p1.x; acc = acc + p1.y;
        acc = acc + p2.x; acc = acc + p2.y; acc = acc + p3.x; acc = acc + p3.y;
    } else {
        acc = acc + lo<P>(w.x) * a.x; acc = acc + hi<P>(w.x) * a.y; acc = acc + lo<P>(w.y) * a.z; acc = acc + hi<P>(w.y) * a.w;
        acc = acc + lo<P>(w.z) * c.x; acc = acc + hi<P>(w.z) * c.y; acc = acc + lo<P>(w.w) * c.z; acc = acc + hi<P>(w.w) * c.w;
    }
    return acc;
}

constexpr int COLS = 1024;
extern __shared__ __align__(16) unsigned char sm[];

template <bool P, bool M2, int A>
__global__ void kbench(float* out, long long* cyc, int reps) {
    uint16_t* w = reinterpret_cast<uint16_t*>(sm);
    float* x = reinterpret_cast<float*>(sm + COLS * 64);
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < COLS * 32; i += blockDim.x) w[i] = (uint16_t)(0x3f80 + (i % 7));
    for (int i = threadIdx.x; i < COLS; i += blockDim.x) x[i] = 1.0f / (1 + i % 5);
    __syncthreads();
    const uint32_t wb = (uint32_t)__cvta_generic_to_shared(w) + lane * 16;
    const uint32_t xb = (uint32_t)__cvta_generic_to_shared(x);
    float acc = 0.f;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        uint4 wq[A];
        float4 xa[A], xc[A];
#pragma unroll
        for (int i = 0; i < A; ++i) {
            wq[i] = lds128(wb + i * 512);
            xa[i] = lds128f(xb + i * 32);
            xc[i] = lds128f(xb + i * 32 + 16);
        }
#pragma unroll 4
        for (int q = 0; q < COLS / 8; q += A) {
#pragma unroll
            for (int i = 0; i < A; ++i) {
                const uint4 ww = wq[i];
                const float4 a = xa[i], c = xc[i];
                if (q + i + A < COLS / 8) {
                    wq[i] = lds128(wb + (q + i + A) * 512);
                    xa[i] = lds128f(xb + (q + i + A) * 32);
                    xc[i] = lds128f(xb + (q + i + A) * 32 + 16);
                }
                acc = group<P, M2>(acc, ww, a, c);
            }
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (lane == 0) cyc[blockIdx.x] = t1 - t0;
}

template <bool P, bool M2, int A>
void run(const char* name) {
    float* out;
    long long* cyc;
    cudaMalloc(&out, 1 << 22);
    cudaMalloc(&cyc, 1 << 16);
    const int smem = COLS * 64 + COLS * 4;
    cudaFuncSetAttribute(kbench<P, M2, A>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kbench<P, M2, A><<<148, 32, smem>>>(out, cyc, 2);
    kbench<P, M2, A><<<148, 32, smem>>>(out, cyc, 8);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-44s %.2f cycles/column\n", name, h / (8.0 * COLS));
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    run<false, false, 1>("IMAD unpack, FMUL, ahead 1 (current)");
    run<false, false, 2>("IMAD unpack, FMUL, ahead 2");
    run<true, false, 1>("PRMT unpack, FMUL, ahead 1");
    run<true, false, 2>("PRMT unpack, FMUL, ahead 2");
    run<true, false, 4>("PRMT unpack, FMUL, ahead 4");
    run<false, true, 2>("IMAD unpack, FMUL2, ahead 2");
    run<true, true, 1>("PRMT unpack, FMUL2, ahead 1");
    run<true, true, 2>("PRMT unpack, FMUL2, ahead 2");
    run<true, true, 4>("PRMT unpack, FMUL2, ahead 4");
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
