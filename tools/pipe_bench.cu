// Microbenchmark (tools only): the production WarpPipe (smoe_chain.cuh)
// streaming bf16 row tiles [cols][32] from HBM, one warp per CTA per tile,
// x resident in smem.  Reports µs per launch (CUDA events), achieved GB/s and
// the per-warp chain rate (cycles per column, clock64 around run()).
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>

#include "../paper_2603_19289_b200/csrc/smoe_chain.cuh"

using namespace smoe;
static bool g_random = false;
__device__ int g_norm_dev = 0;
extern __shared__ __align__(128) unsigned char g_smem[];

template <int S, int CC>
__global__ void __launch_bounds__(32) k_pipe(const uint16_t* w, int cols, const float* x, float* out,
                                             long long* cyc) {
    using P = WarpPipe<uint16_t, S, CC>;
    uint64_t* bar = reinterpret_cast<uint64_t*>(g_smem);
    double* red = reinterpret_cast<double*>(g_smem + 64);
    float* xs = reinterpret_cast<float*>(g_smem + 128);
    float* gs = xs + cols;
    unsigned char* pm = g_smem + 128 + ((2 * cols * 4 + 127) / 128) * 128;
    const uint16_t* tile = w + static_cast<long long>(blockIdx.x) * cols * 32;
    P pipe;
    pipe.init(pm);
    pipe.prime(tile, cols);
    Stager sg;
    sg.init(bar);
    if (g_norm_dev) {  // production prologue: bulk-stage x and gain, rms_norm in place
        sg.add(xs, x, cols * 4);
        sg.add(gs, x, cols * 4);
        sg.wait();
        block_rms_norm(xs, gs, cols, 1e-5f, xs, red);
    } else {
        for (int i = threadIdx.x; i < cols; i += 32) xs[i] = x[i];
        __syncwarp();
    }
    const long long t0 = clock64();
    const float acc = pipe.run(tile, cols, xs);
    const long long t1 = clock64();
    out[blockIdx.x * 32 + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int S, int CC>
void bench(int ntiles, int cols, const char* label) {
    using P = WarpPipe<uint16_t, S, CC>;
    uint16_t* w;
    float *x, *out;
    long long* cyc;
    const size_t bytes = static_cast<size_t>(ntiles) * cols * 32 * 2;
    cudaMalloc(&w, bytes);
    cudaMalloc(&x, cols * 4);
    if (g_random) {
        std::vector<uint16_t> hw(bytes / 2);
        uint32_t st = 12345;
        for (auto& v : hw) { st = st * 1664525u + 1013904223u; v = static_cast<uint16_t>(0x3c00 + (st >> 20) % 0x0400) ^ ((st >> 8) & 0x8000); }
        cudaMemcpy(w, hw.data(), bytes, cudaMemcpyHostToDevice);
        std::vector<float> hx(cols);
        for (auto& v : hx) { st = st * 1664525u + 1013904223u; v = ((st >> 8) & 0xffff) / 32768.0f - 1.0f; }
        cudaMemcpy(x, hx.data(), cols * 4, cudaMemcpyHostToDevice);
    } else {
        cudaMemset(w, 0x3c, bytes);
        cudaMemset(x, 0, cols * 4);
    }
    cudaMalloc(&out, ntiles * 32 * 4);
    cudaMalloc(&cyc, ntiles * 8);
    // flush buffer > L2 so every launch streams from HBM
    char* flush;
    cudaMalloc(&flush, 256 << 20);
    const int smem = 128 + ((2 * cols * 4 + 127) / 128) * 128 + P::kBytes + 128;
    cudaFuncSetAttribute(k_pipe<S, CC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float tot = 0;
    const int reps = 20;
    for (int r = 0; r < reps + 2; ++r) {
        cudaMemsetAsync(flush, r, 256 << 20);
        cudaEventRecord(a);
        k_pipe<S, CC><<<ntiles, 32, smem>>>(w, cols, x, out, cyc);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r >= 2) tot += ms;
    }
    std::vector<long long> h(ntiles);
    cudaMemcpy(h.data(), cyc, ntiles * 8, cudaMemcpyDeviceToHost);
    double avg = 0, mx = 0;
    for (auto v : h) { avg += v; mx = v > mx ? v : mx; }
    avg /= ntiles;
    const double us = 1000.0 * tot / reps;
    printf("%-10s tiles %4d cols %5d S=%d CC=%3d: %7.2f us  %7.0f GB/s  chain %.2f (max %.2f) cyc/col  err=%s\n",
           label, ntiles, cols, S, CC, us, bytes / us / 1e3, avg / cols, mx / cols,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(w); cudaFree(x); cudaFree(out); cudaFree(cyc); cudaFree(flush);
}

int main() {
    g_random = true;
    int nd = 1;
    cudaMemcpyToSymbol(g_norm_dev, &nd, 4);
    bench<4, 256>(12, 2048, "qkv");
    bench<3, 512>(12, 2048, "qkv");
    bench<2, 1024>(12, 2048, "qkv");
    bench<4, 128>(384, 2048, "ffn_gu");
    bench<3, 256>(384, 2048, "ffn_gu");
    bench<2, 256>(384, 2048, "ffn_gu");
    bench<2, 512>(384, 2048, "ffn_gu");
}
