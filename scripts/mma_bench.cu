// mma_bench.cu -- B200 microbenchmark: tcgen05.mma (kind::f16, bf16 -> fp32 TMEM, cta_group::1)
// cycles per 128-deep group (8 x K=16 instructions), one CTA per SM, 148 CTAs.
//   mode 0: SS  M128 N128, commit + wait after every group (issue-to-completion latency)
//   mode 1: SS  M128 N128, back to back (throughput)
//   mode 2: TS  M128 N128 (A = P from TMEM, B = V MN-major), back to back
//   mode 3: SS  M128 N256, back to back
//   mode 4: SS N128 + TS N128 alternating (the attention block pattern), back to back
//   mode 5: SS  M128 N64, back to back
//   mode 6: mode 4 while warps 1-3 stream tcgen05.ld/st over their TMEM lanes (softmax-like load)
//   mode 7: mode 4 while warps 1-3 stream ld.shared over the operand tiles
//   mode 8: TS (A = TMEM cols 0-63) -> SS writing cols 0-127 (the P-aliased-in-S hazard), back to back
//   mode 9: mode 8 for two slots interleaved (slot x at cols 256x): PV0 S0 PV1 S1
//   mode 10: mode 9 with a tcgen05.commit (no waiter) after every group
//   mode 11: the two-tile diagonal kernel's layout (S_x at 128x, O_x at 256 + 128x) and commits
//            (two after each S group, one after each P V group)
// probe (after the modes): clocks from issuing 16 MMAs to (a) the last issue returning, (b) a
// try_wait on an already-complete barrier returning, (c) the MMAs' commit completing
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2602_22575_b200/csrc
//        scripts/mma_bench.cu -o scripts/mma_bench
#include <cuda_runtime.h>
#include <cstdio>
#include "sm100.cuh"
using namespace s2o::sm100;

constexpr int kGroups = 512;

__device__ volatile int g_stop;
__global__ void __launch_bounds__(128, 1) bench(int mode, long long* out) {
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar, bar2c, bar3c;
    __shared__ uint32_t tbase_s;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 3 * 32768 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bar), 1);
        mbar_init(smem_u32(&bar2c), 1);
        mbar_init(smem_u32(&bar3c), 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(smem_u32(&tbase_s), 512);
        tmem_relinquish();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = tbase_s;
    __shared__ volatile int done;
    if (threadIdx.x == 0) done = 0;
    __syncthreads();
    if (warp > 0 && (mode == 6 || mode == 7)) {
        // interference: TMEM row traffic (mode 6) or shared-memory reads (mode 7) until warp 0 ends
        const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
        uint32_t acc = 0;
        while (!done) {
            if (mode == 6) {
                uint32_t v[32];
                tmem_ld32(tb + lane_off + 384, v);
                tmem_ld_wait();
                for (int i = 0; i < 32; ++i) acc += v[i];
                tmem_st32(tb + lane_off + 448, v);
                tmem_st_wait();
            } else {
                const uint4* p = reinterpret_cast<const uint4*>(sm);
                for (int i = 0; i < 64; ++i) { uint4 x = p[(threadIdx.x + i * 32) & 6143]; acc += x.x ^ x.w; }
            }
        }
        if (acc == 0x12345678u) out[0] = acc;
    }
    if (warp == 0) {
        const bool leader = elect_one();
        const uint32_t sA = smem_u32(sm), sB = sA + 32768, sV = sB + 32768;
        const uint64_t da = umma_desc_sw128(sA, 16, 1024), db = umma_desc_sw128(sB, 16, 1024);
        const uint64_t dv = umma_desc_sw128(sV, 16384, 1024);
        const uint32_t id128 = umma_idesc_bf16(128, 128, false, false);
        const uint32_t id256 = umma_idesc_bf16(128, 256, false, false);
        const uint32_t id64 = umma_idesc_bf16(128, 64, false, false);
        const uint32_t ido = umma_idesc_bf16(128, 128, false, true);
        uint32_t ph = 0;
        auto ss = [&](uint32_t d, uint32_t idesc) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint32_t off = ((kk / 4) * 16384 + (kk % 4) * 32) >> 4;
                if (leader) umma_bf16(d, da + off, db + off, idesc, kk > 0);
            }
        };
        auto ts = [&](uint32_t d, uint32_t a = 256) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
                if (leader) umma_bf16_ts(d, tb + a + kk * 8, dv + ((kk * 16 * 128) >> 4), ido, 1);
        };
        __syncwarp();
        const long long t0 = clock64();
        for (int g = 0; g < kGroups; ++g) {
            switch (mode) {
                case 0:
                    ss(tb, id128);
                    if (leader) umma_commit(smem_u32(&bar));
                    __syncwarp();
                    mbar_wait(smem_u32(&bar), ph & 1);
                    ++ph;
                    break;
                case 1: ss(tb + (g & 1) * 128, id128); break;
                case 2: ts(tb + 128); break;
                case 3: ss(tb, id256); break;
                case 4: if (g & 1) ts(tb + 128); else ss(tb, id128); break;
                case 5: ss(tb + (g & 3) * 64, id64); break;
                case 6: case 7: if (g & 1) ts(tb + 128); else ss(tb, id128); break;
                case 8: if (g & 1) ss(tb, id128); else ts(tb + 128, 0); break;
                case 9: {
                    const uint32_t x = (g >> 1) & 1;
                    if (g & 1) ss(tb + x * 256, id128); else ts(tb + x * 256 + 128, x * 256);
                } break;
                case 10: {
                    const uint32_t x = (g >> 1) & 1;
                    if (g & 1) ss(tb + x * 256, id128); else ts(tb + x * 256 + 128, x * 256);
                    if (leader) umma_commit(smem_u32(&bar2c));
                } break;
                case 11: {
                    const uint32_t x = (g >> 1) & 1;
                    if (g & 1) {
                        ss(tb + x * 128, id128);
                        if (leader) { umma_commit(smem_u32(&bar2c)); umma_commit(smem_u32(&bar3c)); }
                    } else {
                        ts(tb + 256 + x * 128, x * 128);
                        if (leader) umma_commit(smem_u32(&bar3c));
                    }
                } break;
            }
        }
        if (mode != 0) {
            if (leader) umma_commit(smem_u32(&bar));
            __syncwarp();
            mbar_wait(smem_u32(&bar), 0);
        }
        const long long t1 = clock64();
        if (leader) out[blockIdx.x] = t1 - t0;
        if (mode == 0 && blockIdx.x == 0) {
            // issue-blocking probe (one CTA): 16 MMAs, then a barrier check on a completed phase
            __shared__ uint64_t bar2;
            if (leader) { mbar_init(smem_u32(&bar2), 1); fence_mbar_init(); mbar_arrive(smem_u32(&bar2)); }
            __syncwarp();
            mbar_wait(smem_u32(&bar2), 0);
            const long long a0 = clock64();
            ss(tb, id128);
            ss(tb + 256, id128);
            const long long a1 = clock64();
            mbar_wait(smem_u32(&bar2), 0);
            const long long a2 = clock64();
            if (leader) umma_commit(smem_u32(&bar));
            __syncwarp();
            mbar_wait(smem_u32(&bar), ph & 1);
            const long long a3 = clock64();
            if (leader) printf("probe: 16 MMAs issued after %lld clk, completed-barrier check returns at %lld, MMAs done at %lld\n",
                               a1 - a0, a2 - a0, a3 - a0);
            // same, with a commit between the MMAs and the check; then an ld.shared poll instead
            ++ph;
            __shared__ volatile uint32_t flag;
            if (leader) flag = 7;
            __syncwarp();
            const long long b0 = clock64();
            ss(tb, id128);
            ss(tb + 256, id128);
            if (leader) umma_commit(smem_u32(&bar));
            const long long b1 = clock64();
            mbar_wait(smem_u32(&bar2), 0);
            const long long b2 = clock64();
            uint32_t f = flag;
            const long long b3 = clock64();
            mbar_wait(smem_u32(&bar), ph & 1);
            const long long b4 = clock64();
            if (leader) printf("probe: MMAs+commit issued at %lld, completed-barrier check after the commit returns at %lld, "
                               "ld.shared poll at %lld (f=%u), MMAs done at %lld\n", b1 - b0, b2 - b0, b3 - b0, f, b4 - b0);
            // ld.shared poll first, then the barrier check
            ++ph;
            const long long c0 = clock64();
            ss(tb, id128);
            ss(tb + 256, id128);
            if (leader) umma_commit(smem_u32(&bar));
            const long long c1 = clock64();
            f += flag;
            const long long c2 = clock64();
            mbar_wait(smem_u32(&bar), ph & 1);
            const long long c3 = clock64();
            if (leader) printf("probe: MMAs+commit issued at %lld, ld.shared right after at %lld (f=%u), MMAs done at %lld\n",
                               c1 - c0, c2 - c0, f, c3 - c0);
        }
        if (leader) done = 1;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 512);
}

int main() {
    long long* d;
    cudaMalloc(&d, 148 * sizeof(long long));
    const int smem = 3 * 32768 + 1024;
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const char* names[] = {"SS N128 latency/group", "SS N128 throughput", "TS N128 throughput", "SS N256 throughput",
                           "SS+TS N128 alternating", "SS N64 throughput", "SS+TS + TMEM ld/st traffic",
                           "SS+TS + ld.shared traffic", "TS(P@S)->SS(S) hazard", "hazard, 2 slots", "2 slots + commit/group",
                           "diag2 layout + commits"};
    for (int mode = 0; mode < 12; ++mode) {
        for (int rep = 0; rep < 2; ++rep) bench<<<148, 128, smem>>>(mode, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        long long h[148];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double s = 0;
        for (int i = 0; i < 148; ++i) s += h[i];
        const double per = s / 148 / kGroups;
        const int n = mode == 3 ? 256 : mode == 5 ? 64 : 128;
        printf("%-26s %8.1f clk/group  (%.0f flop/clk/SM)\n", names[mode], per, 2.0 * 128 * n * 128 / per);
    }
    return 0;
}
