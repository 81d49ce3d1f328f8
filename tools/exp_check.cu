// Tools only: does CUDA's exp(double) return glibc's exp(double) bit for bit?
// The reference's softmax / silu / attention call std::exp on doubles
// (numerics.cpp:46, 104; model.cpp:343); the GPU path uses CUDA's exp.
// Inputs: N doubles per range, drawn like the decode's arguments (x - max <= 0
// for softmax, -x for silu), compared on the host against this box's libm.
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

#include "../paper_2603_19289_b200/csrc/exp_glibc.cuh"

__global__ void k_exp(const double* x, double* y, long long n, int glibc) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        y[i] = glibc ? smoe::exp_glibc(x[i]) : exp(x[i]);
}

int main(int argc, char** argv) {
    const long long n = argc > 1 ? atoll(argv[1]) : (1LL << 26);
    const double ranges[][2] = {{-40.0, 0.0}, {-1.0, 0.0}, {-745.0, 709.0}, {-0.001, 0.001}};
    std::vector<double> hx(n), hy(n);
    double *dx, *dy;
    cudaMalloc(&dx, n * 8);
    cudaMalloc(&dy, n * 8);
    uint64_t s = 0x9E3779B97F4A7C15ull;
    for (int glibc = 0; glibc < 2; ++glibc) {
    printf("%s\n", glibc ? "smoe::exp_glibc (device restatement of glibc exp)" : "CUDA exp(double)");
    long long total_bad = 0;
    for (auto& r : ranges) {
        for (long long i = 0; i < n; ++i) {
            s ^= s << 13; s ^= s >> 7; s ^= s << 17;
            const double u = (s >> 11) * 0x1.0p-53;
            hx[i] = r[0] + (r[1] - r[0]) * u;
            // also float-valued differences, as in softmax of f32 logits
            if (i & 1) hx[i] = (double)(float)hx[i] - (double)(float)(hx[i] * 0.25);
        }
        cudaMemcpy(dx, hx.data(), n * 8, cudaMemcpyHostToDevice);
        k_exp<<<1184, 256>>>(dx, dy, n, glibc);
        cudaMemcpy(hy.data(), dy, n * 8, cudaMemcpyDeviceToHost);
        long long bad = 0;
        for (long long i = 0; i < n; ++i) {
            const double ref = std::exp(hx[i]);
            if (std::memcmp(&ref, &hy[i], 8) != 0) {
                if (bad < 3) printf("  mismatch x=%a gpu=%a libm=%a\n", hx[i], hy[i], ref);
                ++bad;
            }
        }
        printf("range [%g, %g]: %lld inputs, %lld mismatches\n", r[0], r[1], n, bad);
        total_bad += bad;
    }
    printf("total mismatches %lld\n", total_bad);
    }
    return 0;
}
