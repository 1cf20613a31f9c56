// dfma_bench.cu -- B200 microbenchmark: fp64 FMA throughput per SM (32 independent chains per
// thread, `warps` warps per SM, 148 CTAs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/dfma_bench.cu -o scripts/dfma_bench
#include <cuda_runtime.h>
#include <cstdio>
__global__ void bench(double* out, long long* cyc, int iters) {
    double acc[32];
    const double a = 1.0000001 + threadIdx.x * 1e-9, b = 0.9999999;
    for (int i = 0; i < 32; ++i) acc[i] = i;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[i] = fma(acc[i], a, b);
    }
    const long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < 32; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    double* o; long long* c;
    cudaMalloc(&o, 148 * 1024 * 8); cudaMalloc(&c, 148 * 8);
    for (int w : {1, 2, 4, 8, 16, 32}) {
        const int iters = 4096;
        bench<<<148, 32 * w>>>(o, c, iters);
        cudaDeviceSynchronize();
        long long h[148];
        cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
        double avg = 0; for (auto v : h) avg += v; avg /= 148;
        printf("warps/SM=%2d: %.1f DFMA/clk/SM (%s)\n", w, 32.0 * w * 32 * iters / avg, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
