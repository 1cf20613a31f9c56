// load_bench.cu -- B200 microbenchmark: cycles to land a 64 KB K+V block (2 x 128 rows x 256 B)
// in shared memory, per strategy, with `stages` blocks in flight per CTA, 148 CTAs.
//   0: TMA gather4 (box 64x1), 1 warp issues      1: gather4, 4 warps issue
//   2: TMA 2-D tile (box 64x128), contiguous rows  3: cp.async 16 B, 128 threads
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sm100.cuh"

using namespace s2o::sm100;

constexpr int kBlock = 65536;
constexpr int kIters = 256;

__global__ void __launch_bounds__(512, 1) bench(int mode, int stages, int issuers, const __grid_constant__ CUtensorMap gmap,
                                                const __grid_constant__ CUtensorMap tmap, const uint4* base,
                                                const int* rows, int nrows, long long* cycles) {
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + stages * kBlock);  // + rows after
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) mbar_init(smem_u32(&bars[s]), mode == 3 ? 32 * issuers : 1);
        fence_mbar_init();
    }
    __syncthreads();
    const long long t0 = clock64();
        for (int it = 0; it < kIters; ++it) {
        const int s = it % stages;
        if (it >= stages) mbar_wait(smem_u32(&bars[s]), ((it / stages) - 1) & 1);
        __syncthreads();
        const uint32_t dst = smem_u32(sm + s * kBlock);
        const int* rr = rows + ((blockIdx.x * kIters + it) * 256) % (nrows * 64);
        if (mode <= 1) {
            if (warp < issuers) {
                if (threadIdx.x == 0) mbar_expect_tx(smem_u32(&bars[s]), kBlock);
                __syncwarp();
                if (issuers > 1) asm volatile("bar.sync 1, %0;" :: "r"(32 * issuers));
                // 256 rows (K then V) x 2 halves = 128 gather4 ops
                for (int op = threadIdx.x; op < 128; op += 32 * issuers) {
                    const int grp = op / 2, h = op % 2;
                    const int* r4 = rr + grp * 4;
                    tma_gather4(dst + (grp / 32) * 32768 + h * 16384 + (grp % 32) * 512, &gmap, h * 64, r4[0], r4[1],
                                r4[2], r4[3], smem_u32(&bars[s]));
                }
            }
        } else if (mode == 4) {
            // one elected lane per issuing warp, warp-uniform operands from shared memory
            int* srows = reinterpret_cast<int*>(bars + 8);
            for (int e = threadIdx.x; e < 256; e += blockDim.x) srows[e] = rr[e];
            __syncthreads();
            if (warp == 0 && lane == 0) mbar_expect_tx(smem_u32(&bars[s]), kBlock);
            if (warp < issuers) {
                if (lane == 0) {
                    for (int op = warp; op < 128; op += issuers) {
                        const int grp = op / 2, h = op % 2;
                        const int4 r4 = *reinterpret_cast<const int4*>(srows + grp * 4);
                        tma_gather4(dst + (grp / 32) * 32768 + h * 16384 + (grp % 32) * 512, &gmap, h * 64, r4.x,
                                    r4.y, r4.z, r4.w, smem_u32(&bars[s]));
                    }
                }
            }
        } else if (mode == 2) {
            if (threadIdx.x == 0) {
                mbar_expect_tx(smem_u32(&bars[s]), kBlock);
                const int r0 = (rr[0] / 128) * 128;
                for (int t = 0; t < 2; ++t)
                    for (int h = 0; h < 2; ++h)
                        tma_load2d(dst + t * 32768 + h * 16384, &tmap, h * 64, (r0 + t * 128) % nrows, smem_u32(&bars[s]));
            }
        } else {
            if (threadIdx.x < 32 * issuers) {
                for (int e = threadIdx.x; e < 4096; e += 32 * issuers) {
                    const int row = e / 16, ch = e % 16;
                    const int r = rr[row];
                    const uint32_t off = (row / 128) * 32768 + (ch / 8) * 16384 + sw128_offset(row % 128, (ch % 8) * 8);
                    cp_async16(dst + off, base + (size_t)r * 16 + ch, 16);
                }
                cp_async_arrive_noinc(smem_u32(&bars[s]));
            }
        }
    }
    for (int it = kIters; it < kIters + stages; ++it) {
        const int s = it % stages;
        mbar_wait(smem_u32(&bars[s]), ((it / stages) - 1) & 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) cycles[blockIdx.x] = clock64() - t0;
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
    const char* names[5] = {"gather4", "gather4", "tile2d contiguous", "cp.async", "gather4 1lane/warp"};
    for (int mode : {4, 0}) {
      for (int issuers : {1, 2, 4, 8, 16}) {
        if (mode == 2 && issuers > 1) continue;
        for (int stages : {2}) {
            const int smem = stages * kBlock + 4096;
            cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            bench<<<148, 512, smem>>>(mode, stages, issuers, gmap, tmap, dbase, drows, nrows, dcyc);
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a);
            bench<<<148, 512, smem>>>(mode, stages, issuers, gmap, tmap, dbase, drows, nrows, dcyc);
            cudaEventRecord(b);
            cudaError_t e = cudaDeviceSynchronize();
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            std::vector<long long> c(148);
            cudaMemcpy(c.data(), dcyc, 148 * 8, cudaMemcpyDeviceToHost);
            double avg = 0;
            for (auto x : c) avg += x;
            avg /= 148;
            printf("%-20s warps=%2d stages=%d: %7.0f cycles/block  %7.1f GB/s total  %s\n", names[mode], issuers, stages,
                   avg / kIters, 148.0 * kIters * kBlock / (ms * 1e-3) / 1e9, cudaGetErrorString(e));
        }
      }
    }
    return 0;
}
