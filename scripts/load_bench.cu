// load_bench.cu -- B200 microbenchmark: cycles to land a 64 KB K+V block (2 x 128 rows x 256 B,
// random rows of an L2-resident table) in shared memory, `stages` blocks in flight per CTA,
// 148 CTAs, `warps` issuing warps. Row tokens are staged in shared memory (as in the kernel).
//   mode 1: TMA tile::gather4 for K and V (128 ops), ops spread over the warps
//   mode 3: cp.async 16 B for K and V (4096 pieces)
//   mode 5: gather4 for K, cp.async for V
//   mode 2: TMA 2-D tile, contiguous rows (reference point)
//   build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2602_22575_b200/csrc
//          scripts/load_bench.cu -o scripts/load_bench -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "sm100.cuh"
using namespace s2o::sm100;
constexpr int kBlock = 65536;
__device__ __forceinline__ void expect_tx_only(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
constexpr int kIters = 256;
__global__ void __launch_bounds__(512, 1) bench(int mode, int stages, int warps, const __grid_constant__ CUtensorMap gmap,
                                                const __grid_constant__ CUtensorMap tmap, const uint4* base,
                                                const int* rows, int nrows, long long* cycles) {
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + stages * kBlock);
    int* stok = reinterpret_cast<int*>(bars + 16);  // [2][256]
    const int warp = threadIdx.x / 32;
    const int nthr = 32 * warps;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) mbar_init(smem_u32(&bars[s]), nthr);
        fence_mbar_init();
    }
    __syncthreads();
    if (warp >= warps) return;
    const int t = threadIdx.x;
    const long long t0 = clock64();
    for (int it = 0; it < kIters; ++it) {
        const int s = it % stages;
        if (it >= stages) mbar_wait(smem_u32(&bars[s]), ((it / stages) - 1) & 1);
        const int* rr = rows + ((blockIdx.x * kIters + it) * 256) % (nrows * 64);
        int* tk = stok + (it & 1) * 256;
        for (int e = t; e < 256; e += nthr) tk[e] = rr[e];
        asm volatile("bar.sync 1, %0;" ::"r"(nthr));
        const uint32_t dst = smem_u32(sm + s * kBlock);
        const uint32_t bar = smem_u32(&bars[s]);
        if (mode == 2) {
            if (t == 0) {
                mbar_expect_tx(bar, kBlock);
                const int r0 = (tk[0] / 128) * 128;
                for (int u = 0; u < 2; ++u)
                    for (int h = 0; h < 2; ++h)
                        tma_load2d(dst + u * 32768 + h * 16384, &tmap, h * 64, (r0 + u * 128) % nrows, bar);
            } else {
                mbar_arrive(bar);
            }
            continue;
        }
        const int nops = (mode == 1) ? 128 : (mode == 5 ? 64 : 0);  // gather4 ops (K first)
        if (nops) {
            if (t == 0) expect_tx_only(bar, nops * 512);
            asm volatile("bar.sync 2, %0;" ::"r"(nthr));
            for (int op = t; op < nops; op += nthr) {
                const int grp = op / 2, h = op % 2;
                const int* r4 = tk + grp * 4;
                tma_gather4(dst + (grp / 32) * 32768 + h * 16384 + (grp % 32) * 512, &gmap, h * 64, r4[0], r4[1],
                            r4[2], r4[3], bar);
            }
        }
        const int p0 = (mode == 5) ? 2048 : (mode == 3 ? 0 : 4096);  // cp.async pieces [p0, 4096)
        for (int e = p0 + t; e < 4096; e += nthr) {
            const int row = e / 16, ch = e % 16;
            const uint32_t off = (row / 128) * 32768 + (ch / 8) * 16384 + sw128_offset(row % 128, (ch % 8) * 8);
            cp_async16(dst + off, base + (size_t)tk[row] * 16 + ch, 16);
        }
        if (mode == 1) mbar_arrive(bar);
        else cp_async_arrive_noinc(bar);
    }
    for (int it = kIters; it < kIters + stages; ++it) {
        const int s = it % stages;
        mbar_wait(smem_u32(&bars[s]), ((it / stages) - 1) & 1);
    }
    if (t == 0) cycles[blockIdx.x] = clock64() - t0;
}
int main() {
    const int nrows = 1 << 17;  // 128K rows x 256 B = 32 MB (L2-resident)
    uint4* dbase;
    int* drows;
    long long* dcyc;
    cudaMalloc(&dbase, (size_t)nrows * 256);
    cudaMemset(dbase, 1, (size_t)nrows * 256);
    std::vector<int> rows(nrows * 64);
    srand(3);
    for (auto& r : rows) r = rand() % nrows;
    cudaMalloc(&drows, rows.size() * 4);
    cudaMemcpy(drows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&dcyc, 148 * 8);
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    CUtensorMap gmap, tmap;
    cuuint64_t dims[2] = {128, (cuuint64_t)nrows};
    cuuint64_t str[1] = {256};
    cuuint32_t bg[2] = {64, 1}, bt[2] = {64, 128}, es[2] = {1, 1};
    enc(&gmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dbase, dims, str, bg, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dbase, dims, str, bt, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const char* names[6] = {"", "gather4 K+V", "tile2d contiguous", "cp.async K+V", "", "gather4 K + cp.async V"};
    for (int mode : {2, 1, 3, 5}) {
        for (int warps : {1, 2, 3, 4, 8}) {
            if (mode == 2 && warps > 1) continue;
            for (int stages : {2, 3}) {
                const int smem = stages * kBlock + 4096;
                cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                bench<<<148, 512, smem>>>(mode, stages, warps, gmap, tmap, dbase, drows, nrows, dcyc);
                cudaEvent_t a, b;
                cudaEventCreate(&a);
                cudaEventCreate(&b);
                cudaEventRecord(a);
                bench<<<148, 512, smem>>>(mode, stages, warps, gmap, tmap, dbase, drows, nrows, dcyc);
                cudaEventRecord(b);
                cudaError_t e = cudaDeviceSynchronize();
                float ms = 0;
                cudaEventElapsedTime(&ms, a, b);
                std::vector<long long> c(148);
                cudaMemcpy(c.data(), dcyc, 148 * 8, cudaMemcpyDeviceToHost);
                double avg = 0;
                for (auto x : c) avg += x;
                avg /= 148;
                printf("%-24s warps=%d stages=%d: %7.0f cycles/block %7.1f GB/s  %s\n", names[mode], warps, stages,
                       avg / kIters, 148.0 * kIters * kBlock / (ms * 1e-3) / 1e9, cudaGetErrorString(e));
            }
        }
    }
    return 0;
}
