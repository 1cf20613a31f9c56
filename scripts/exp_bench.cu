// exp_bench.cu -- B200 microbenchmark: cycles per 128-element softmax row (x = s*sc - m,
// 2^x, row sum, bf16 pack) per warp, with POLY of every 32 elements on the FMA pipe, and
// `warps` warps per SM running concurrently (148 CTAs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2602_22575_b200/csrc scripts/exp_bench.cu -o scripts/exp_bench
#include <cuda_runtime.h>
#include <cstdio>
#include "sm100.cuh"
using namespace s2o::sm100;
template <int POLY>
__global__ void bench(float* out, long long* cyc, int iters) {
    float sv[128];
    for (int i = 0; i < 128; ++i) sv[i] = (threadIdx.x * 7 + i * 13) % 97 * -0.01f;
    float acc = 0.f;
    uint32_t pk_acc = 0;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const float neg_ref = -0.001f * (it & 7);
        float rs[4] = {0, 0, 0, 0};
#pragma unroll
        for (int c0 = 0; c0 < 128; c0 += 32) {
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
                const float x0 = fmaf(sv[c0 + i], 0.127f, neg_ref);
                const float x1 = fmaf(sv[c0 + i + 1], 0.127f, neg_ref);
                const float e0 = (i >= 32 - POLY) ? ex2_poly(x0) : ex2(x0);
                const float e1 = (i >= 32 - POLY) ? ex2_poly(x1) : ex2(x1);
                rs[(i >> 1) & 3] += e0 + e1;
                pk_acc ^= pack_bf16(e0, e1);
            }
        }
        acc += rs[0] + rs[1] + rs[2] + rs[3];
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + (float)pk_acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int POLY>
void run(int warps) {
    float* o; long long* c;
    cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 148 * 8);
    const int iters = 2000;
    bench<POLY><<<148, 32 * warps>>>(o, c, iters);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
    double avg = 0; for (auto v : h) avg += v; avg /= 148;
    printf("poly=%2d/32 warps/SM=%2d: %7.1f clk per 128-elem row per warp (%s)\n", POLY, warps, avg / iters,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(o); cudaFree(c);
}
int main() {
    for (int w : {1, 4, 8, 16}) { run<0>(w); run<4>(w); run<8>(w); run<12>(w); run<16>(w); }
    return 0;
}
