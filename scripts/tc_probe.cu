// tc_probe.cu -- standalone B200 probe of the primitives the tcgen05 attention kernel uses:
//   A) S = Q K^T  : tcgen05.mma kind::f16, A/B K-major SWIZZLE_128B from smem, fp32 in TMEM
//   B) O = P V    : B operand MN-major (V stored [keys][d] in SW128 64-column blocks)
//   C) TMA tile::gather4 of 4 arbitrary rows into an SW128 tile (box {64, 1})
//   D) TMA 2-D tile load (box {64, 128}) into an SW128 tile
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../paper_2602_22575_b200/csrc \
//            tc_probe.cu -o tc_probe
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "sm100.cuh"

using namespace s2o::sm100;

#define CK(x)                                                                      \
    do {                                                                           \
        cudaError_t e = (x);                                                       \
        if (e != cudaSuccess) {                                                    \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                               \
        }                                                                          \
    } while (0)

// smem: Q 32K | K 32K | P 32K | V 32K | gather 32K | tile 16K | bars
__global__ void __launch_bounds__(128) probe_kernel(const __nv_bfloat16* q, const __nv_bfloat16* k,
                                                    const __nv_bfloat16* p, const __nv_bfloat16* v,
                                                    float* s_out, float* o_out,
                                                    const __grid_constant__ CUtensorMap kmap_g,
                                                    const __grid_constant__ CUtensorMap kmap_t,
                                                    const int* gather_rows, __nv_bfloat16* gather_out,
                                                    __nv_bfloat16* tile_out, float* o2_out) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* sQ = smem;
    unsigned char* sK = smem + 32768;
    unsigned char* sP = smem + 65536;
    unsigned char* sV = smem + 98304;
    unsigned char* sG = smem + 131072;
    unsigned char* sT = smem + 163840;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 180224);
    uint32_t* tmem_base = reinterpret_cast<uint32_t*>(smem + 180224 + 64);
    const int tid = threadIdx.x;
    const int warp = tid / 32;

    // fill Q, K, P (K-major SW128) and V (same physical layout, used MN-major)
    for (int e = tid; e < 128 * 128; e += blockDim.x) {
        const int r = e / 128, c = e % 128;
        const uint32_t off = (c / 64) * 16384 + sw128_offset(r, c % 64);
        *reinterpret_cast<__nv_bfloat16*>(sQ + off) = q[e];
        *reinterpret_cast<__nv_bfloat16*>(sK + off) = k[e];
        *reinterpret_cast<__nv_bfloat16*>(sP + off) = p[e];
        *reinterpret_cast<__nv_bfloat16*>(sV + off) = v[e];
    }
    if (tid == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(smem_u32(&bars[i]), 1);
        fence_mbar_init();
    }
    fence_proxy_async_smem();
    if (warp == 0) {
        tmem_alloc(smem_u32(tmem_base), 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_base;

    if (tid == 0) {
        const uint32_t idesc_s = umma_idesc_bf16(128, 128, false, false);
        for (int kk = 0; kk < 8; ++kk) {
            const uint32_t koff = (kk / 4) * 16384 + (kk % 4) * 32;
            umma_bf16(tbase, umma_desc_sw128(smem_u32(sQ) + koff, 16, 1024),
                      umma_desc_sw128(smem_u32(sK) + koff, 16, 1024), idesc_s, kk > 0);
        }
        const uint32_t idesc_o = umma_idesc_bf16(128, 128, false, true);
        for (int kk = 0; kk < 8; ++kk) {
            const uint32_t aoff = (kk / 4) * 16384 + (kk % 4) * 32;
            const uint32_t boff = kk * 16 * 128;
            umma_bf16(tbase + 128, umma_desc_sw128(smem_u32(sP) + aoff, 16, 1024),
                      umma_desc_sw128(smem_u32(sV) + boff, 16384, 1024), idesc_o, kk > 0);
        }
        umma_commit(smem_u32(&bars[0]));
        // TMA probes
        mbar_expect_tx(smem_u32(&bars[1]), 4 * 128);
        tma_gather4(smem_u32(sG), &kmap_g, 0, gather_rows[0], gather_rows[1], gather_rows[2],
                    gather_rows[3], smem_u32(&bars[1]));
        mbar_expect_tx(smem_u32(&bars[2]), 128 * 128);
        tma_load2d(smem_u32(sT), &kmap_t, 0, 256, smem_u32(&bars[2]));
    }
    __syncwarp();
    mbar_wait(smem_u32(&bars[0]), 0);
    tc_fence_after();
    // each warp reads its 32 lanes
    for (int half = 0; half < 2; ++half) {
        for (int c0 = 0; c0 < 128; c0 += 32) {
            uint32_t r[32];
            tmem_ld32(tbase + ((uint32_t)(warp * 32) << 16) + half * 128 + c0, r);
            tmem_ld_wait();
            float* dst = (half == 0 ? s_out : o_out) + (warp * 32 + (tid % 32)) * 128 + c0;
            for (int i = 0; i < 32; ++i) dst[i] = __uint_as_float(r[i]);
        }
    }
    // E) P from TMEM (packed bf16x2, row = lane), V MN-major from smem: O2 = P V -> cols [384, 512)
    {
        const int row = warp * 32 + (tid % 32);
        for (int c0 = 0; c0 < 64; c0 += 16) {
            uint32_t pk[16];
            for (int i = 0; i < 16; ++i) {
                const __nv_bfloat16 lo = p[row * 128 + 2 * (c0 + i)], hi = p[row * 128 + 2 * (c0 + i) + 1];
                pk[i] = (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
            }
            tmem_st16(tbase + ((uint32_t)(warp * 32) << 16) + 256 + c0, pk);
        }
        tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
        const uint32_t idesc_o = umma_idesc_bf16(128, 128, false, true);
        for (int kk = 0; kk < 8; ++kk)
            umma_bf16_ts(tbase + 384, tbase + 256 + kk * 8, umma_desc_sw128(smem_u32(sV) + kk * 16 * 128, 16384, 1024),
                         idesc_o, kk > 0);
        umma_commit(smem_u32(&bars[3]));
    }
    __syncwarp();
    mbar_wait(smem_u32(&bars[3]), 0);
    tc_fence_after();
    for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tbase + ((uint32_t)(warp * 32) << 16) + 384 + c0, r);
        tmem_ld_wait();
        float* dst = o2_out + (warp * 32 + (tid % 32)) * 128 + c0;
        for (int i = 0; i < 32; ++i) dst[i] = __uint_as_float(r[i]);
    }
    mbar_wait(smem_u32(&bars[1]), 0);
    mbar_wait(smem_u32(&bars[2]), 0);
    for (int e = tid; e < 4 * 64; e += blockDim.x) {
        const int r = e / 64, c = e % 64;
        gather_out[e] = *reinterpret_cast<__nv_bfloat16*>(sG + sw128_offset(r, c));
    }
    for (int e = tid; e < 128 * 64; e += blockDim.x) {
        const int r = e / 64, c = e % 64;
        tile_out[e] = *reinterpret_cast<__nv_bfloat16*>(sT + sw128_offset(r, c));
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tbase, 512);
}

static float bf(const __nv_bfloat16& x) { return __bfloat162float(x); }

int main() {
    const int R = 1024;
    std::vector<__nv_bfloat16> hq(128 * 128), hk(128 * 128), hp(128 * 128), hv(128 * 128), hg(R * 128);
    srand(1);
    auto rnd = [] { return (float)(rand() % 2001 - 1000) / 500.0f; };
    for (auto& x : hq) x = __float2bfloat16(rnd());
    for (auto& x : hk) x = __float2bfloat16(rnd());
    for (auto& x : hp) x = __float2bfloat16(rnd());
    for (auto& x : hv) x = __float2bfloat16(rnd());
    for (auto& x : hg) x = __float2bfloat16(rnd());
    __nv_bfloat16 *dq, *dk, *dp, *dv, *dg, *dgo, *dto;
    float *ds, *dout, *do2;
    int* drows;
    CK(cudaMalloc(&dq, 32768)); CK(cudaMalloc(&dk, 32768)); CK(cudaMalloc(&dp, 32768)); CK(cudaMalloc(&dv, 32768));
    CK(cudaMalloc(&dg, R * 256)); CK(cudaMalloc(&dgo, 512)); CK(cudaMalloc(&dto, 128 * 128));
    CK(cudaMalloc(&ds, 65536)); CK(cudaMalloc(&dout, 65536)); CK(cudaMalloc(&do2, 65536)); CK(cudaMalloc(&drows, 16));
    CK(cudaMemcpy(dq, hq.data(), 32768, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dk, hk.data(), 32768, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dp, hp.data(), 32768, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dv, hv.data(), 32768, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dg, hg.data(), R * 256, cudaMemcpyHostToDevice));
    int rows[4] = {5, 900, 17, 333};
    CK(cudaMemcpy(drows, rows, 16, cudaMemcpyHostToDevice));

    PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    cudaDriverEntryPointQueryResult qres;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &qres));
    CUtensorMap map_g, map_t;
    cuuint64_t dims[2] = {128, (cuuint64_t)R};
    cuuint64_t strides[1] = {256};
    cuuint32_t box_g[2] = {64, 1};
    cuuint32_t box_t[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    CUresult r1 = encode(&map_g, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dg, dims, strides, box_g, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult r2 = encode(&map_t, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dg, dims, strides, box_t, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode gather(box 64x1)=%d tile(box 64x128)=%d\n", (int)r1, (int)r2);
    const int smem = 180224 + 1024 + 1024;
    CK(cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    probe_kernel<<<1, 128, smem>>>(dq, dk, dp, dv, ds, dout, map_g, map_t, drows, dgo, dto, do2);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<float> hs(128 * 128), ho(128 * 128), ho2(128 * 128);
    CK(cudaMemcpy(ho2.data(), do2, 65536, cudaMemcpyDeviceToHost));
    std::vector<__nv_bfloat16> hgo(256), hto(128 * 64);
    CK(cudaMemcpy(hs.data(), ds, 65536, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ho.data(), dout, 65536, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hgo.data(), dgo, 512, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hto.data(), dto, 128 * 128, cudaMemcpyDeviceToHost));
    double es_max = 0, eo_max = 0;
    for (int i = 0; i < 128; ++i)
        for (int j = 0; j < 128; ++j) {
            double s = 0, o = 0;
            for (int d = 0; d < 128; ++d) {
                s += (double)bf(hq[i * 128 + d]) * bf(hk[j * 128 + d]);
                o += (double)bf(hp[i * 128 + d]) * bf(hv[d * 128 + j]);
            }
            es_max = std::max(es_max, std::fabs(s - hs[i * 128 + j]));
            eo_max = std::max(eo_max, std::fabs(o - ho[i * 128 + j]));
        }
    double eo2 = 0;
    for (int i = 0; i < 128 * 128; ++i) eo2 = std::max(eo2, (double)std::fabs(ho2[i] - ho[i]));
    printf("E) PV with P from TMEM vs smem: max abs diff %.3e\n", eo2);
    int gbad = 0, tbad = 0;
    for (int i = 0; i < 4; ++i)
        for (int c = 0; c < 64; ++c)
            gbad += bf(hgo[i * 64 + c]) != bf(hg[rows[i] * 128 + c]);
    for (int i = 0; i < 128; ++i)
        for (int c = 0; c < 64; ++c) tbad += bf(hto[i * 64 + c]) != bf(hg[(256 + i) * 128 + c]);
    printf("A) QK^T max abs err %.3e  (S[0][0]=%f)\n", es_max, hs[0]);
    printf("B) PV   max abs err %.3e  (O[0][0]=%f)\n", eo_max, ho[0]);
    printf("C) gather4 mismatches %d / 256\n", gbad);
    printf("D) tile load mismatches %d / 8192\n", tbad);
    const bool ok = es_max < 1e-2 && eo_max < 1e-2 && gbad == 0 && tbad == 0 && eo2 < 1e-3;
    printf("%s\n", ok ? "PROBE OK" : "PROBE FAIL");
    return ok ? 0 : 1;
}
