// Microbenchmark (tools only): dependent-issue latency of FADD / FMUL / FFMA
// chains in registers, one warp per SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int V>
__global__ void k(float* out, long long* cyc, float a, float b) {
    float acc = a, p0 = b, p1 = b * 1.5f, p2 = b * 0.5f, p3 = b * 0.25f;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < 4096; ++i) {
        if (V == 0) { acc = acc + p0; acc = acc + p1; acc = acc + p2; acc = acc + p3; }
        if (V == 1) { acc = acc * p0; acc = acc * p1; acc = acc * p2; acc = acc * p3; }
        if (V == 2) { acc = __fmaf_rn(acc, p0, p1); acc = __fmaf_rn(acc, p2, p3); acc = __fmaf_rn(acc, p0, p1); acc = __fmaf_rn(acc, p2, p3); }
        if (V == 3) { acc = __fadd_rn(acc, p0); p0 = p0 * p1; acc = __fadd_rn(acc, p1); p1 = p1 * p2; acc = __fadd_rn(acc, p2); p2 = p2 * p3; acc = __fadd_rn(acc, p3); p3 = p3 * p0; }
    }
    long long t1 = clock64();
    out[threadIdx.x + blockIdx.x * 32] = acc + p0 + p1 + p2 + p3;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    float* o; long long* c; cudaMalloc(&o, 1 << 20); cudaMalloc(&c, 1 << 12);
    const char* n[] = {"FADD chain", "FMUL chain", "FFMA chain", "FADD chain + independent FMUL"};
    void (*ks[])(float*, long long*, float, float) = {k<0>, k<1>, k<2>, k<3>};
    for (int v = 0; v < 4; ++v) {
        ks[v]<<<148, 32>>>(o, c, 1.0f, 1e-7f); cudaDeviceSynchronize();
        ks[v]<<<148, 32>>>(o, c, 1.0f, 1e-7f); cudaDeviceSynchronize();
        long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("%-32s %.2f cycles per dependent op\n", n[v], h / (4096.0 * 4));
    }
}
