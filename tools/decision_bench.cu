// Microbenchmark (tools only): warp_decision (smoe_chain.cuh) for E logits,
// top-k, both gating orders; cycles per call from one warp.
#define DECISION_TIMING
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2603_19289_b200/csrc/smoe_chain.cuh"

using namespace smoe;

__global__ void k_dec(const float* lg, int E, int K, int gating, int* ids, float* gates, long long* cyc) {
    __shared__ double se[kMaxE];
    __shared__ float sp[kMaxE];
    long long t0 = clock64();
    for (int r = 0; r < 10; ++r) warp_decision(lg + r * E, E, K, gating, sp, se, ids, gates);
    long long t1 = clock64();
    if (threadIdx.x == 0) *cyc = (t1 - t0) / 10;
}

__global__ void k_parts(const float* lg, int E, long long* cyc) {
    __shared__ double se[kMaxE];
    const int lane = threadIdx.x;
    long long t0 = clock64();
    for (int i = lane; i < E; i += 32) se[i] = exp(static_cast<double>(lg[i]));
    __syncwarp();
    long long t1 = clock64();
    double z = 0.0;
    if (lane == 0)
        for (int i = 0; i < E; ++i) z += se[i];
    z = __shfl_sync(0xffffffffu, z, 0);
    long long t2 = clock64();
    float s = 0;
    for (int i = lane; i < E; i += 32) s += static_cast<float>(se[i] / z);
    long long t3 = clock64();
    if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = (long long)s; }
}

int main() {
    const int E = 128, K = 8;
    float* lg; int* ids; float* g; long long* cyc;
    cudaMalloc(&lg, 4 * E * 16); cudaMalloc(&ids, 64); cudaMalloc(&g, 64); cudaMalloc(&cyc, 64);
    float h[E * 16];
    for (int i = 0; i < E * 16; ++i) h[i] = ((i * 7919) % 1000) / 500.0f - 1.0f;
    cudaMemcpy(lg, h, sizeof h, cudaMemcpyHostToDevice);
    for (int gating = 0; gating < 2; ++gating) {
        k_dec<<<1, 32>>>(lg, E, K, gating, ids, g, cyc);
        k_dec<<<1, 32>>>(lg, E, K, gating, ids, g, cyc);
        long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("warp_decision E=%d K=%d gating=%d: %lld cycles\n", E, K, gating, c);
        long long tt[8];
        cudaMemcpyFromSymbol(tt, g_dec_t, sizeof tt);
        printf("   stage %lld, softmax %lld, topk %lld, gates %lld\n", tt[1] - tt[0], tt[2] - tt[1], tt[3] - tt[2], tt[4] - tt[3]);
    }
    k_parts<<<1, 32>>>(lg, E, cyc);
    k_parts<<<1, 32>>>(lg, E, cyc);
    long long c[4]; cudaMemcpy(c, cyc, 32, cudaMemcpyDeviceToHost);
    printf("parts: f64 exp x%d/lane %lld, sequential f64 sum of %d %lld, f64 div %lld cycles\n", E / 32, c[0], E, c[1], c[2]);
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
