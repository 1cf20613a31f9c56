// plan.cu -- Step 1 of S2O on the device: block scoring + permutation-index build.
//
// Reference: build_plan (proj/src/plan.cpp:140-162) = segment_representatives
// (plan.cpp:46-67, mean_pool_rows tensor.cpp:63-84) + guide = k_mean[segment 0]
// (plan.cpp:145-151) + rank_queries (plan.cpp:69-101) + rank_prefix_keys
// (plan.cpp:103-138), each ranking an argsort_desc_stable (tensor.cpp:43-61).
//
// Exactness: means are fp64 sums sequential over rows,
// then * (1.0/len) and a cast to fp32; dots are fp64 sequential over d (the
// fp32 x fp32 products are exact in fp64, so DFMA == mul+add); the sort is a
// total order on (order-preserving 64-bit key, index) == std::stable_sort.
//
// Kernels (all HBM/L2-bound integer-and-fp64 work, no tensor cores):
//   seg_mean_kernel    one thread per (slice, segment, column): coalesced across d
//   q_rank_kernel      one CTA per (z,h,segment): Q rows staged in smem, fused
//                      column sums (q_mean) + guide dots (q keys)
//   kv_score_kernel    one CTA per (z, kv head, 128-key block): K block staged
//                      transposed in smem, 8 (q head, segment) accumulators per
//                      thread share one converted K element (GQA reuse of K)
//   seg_table_kernel   per-segment run/tile prefix table
//   run_sort_kernel    bitonic sort of 2048-element runs in smem
//   merge_pass_kernel  merge-path merge of sorted run pairs, 2048 outputs per CTA
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "internal.h"
#include "sm100.cuh"
#include "sort.cuh"

#include <cub/block/block_radix_sort.cuh>

namespace s2o {

namespace {

constexpr int kRun = 2048;         // run length == merge tile
constexpr int kSortThreads = 256;  // kRun / 8
constexpr int kQRows = 64;         // Q rows staged per q_rank step

// ---------------------------------------------------------------- means
// out[(slice * nseg_out + n) * D + d] = mean of rows [nS, nS+len) of column d
__global__ void seg_mean_kernel(const void* __restrict__ x, int bf16, int64_t heads_per_z,
                                int64_t s0, int64_t s1, int64_t s2, int64_t d, int64_t S,
                                int64_t N, int64_t last_len, int64_t nseg_out,
                                float* __restrict__ out) {
    const int64_t slice = blockIdx.y;  // z * heads + h
    const int64_t n = blockIdx.z;
    const int64_t col = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (col >= d || n >= nseg_out) return;
    const int64_t base = (slice / heads_per_z) * s0 + (slice % heads_per_z) * s1 + col;
    const int64_t len = (n + 1 == N) ? last_len : S;
    const int64_t r0 = n * S;
    double acc = 0.0;
    int64_t r = 0;
    // unrolled loads, sequential fp64 adds in row order
    for (; r + 8 <= len; r += 8) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = ld_in(x, base + (r0 + r + u) * s2, bf16);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += (double)v[u];
    }
    for (; r < len; ++r) acc += (double)ld_in(x, base + (r0 + r) * s2, bf16);
    const double inv = 1.0 / (double)len;
    out[(slice * nseg_out + n) * d + col] = (float)(acc * inv);
}

// ---------------------------------------------------------------- q ranking
// One CTA (256 threads) per (zh, n). Streams the segment's rows through smem in chunks of
// kQRows; threads [0, 128) accumulate column sums in row order (q_mean, fp64 sequential),
// threads [128, 128 + kQRows) score one staged row each against the fp64 guide (sequential
// over d). When the segment fits one CTA sort (len <= kRun) the keys are sorted in smem and
// q_perm is written directly; otherwise keys go to `qkey` for the global sort.
constexpr int kQThreads = 256;

__global__ void __launch_bounds__(kQThreads)
q_rank_kernel(const void* __restrict__ q, Geo g, const float* __restrict__ guide,
              float* __restrict__ q_mean, uint64_t* __restrict__ qkey, int32_t* __restrict__ q_perm) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int64_t d = g.d;
    uint64_t* sk0 = reinterpret_cast<uint64_t*>(smem_raw);          // [kRun]
    uint64_t* sk1 = sk0 + kRun;                                      // [kRun]
    uint32_t* si0 = reinterpret_cast<uint32_t*>(sk1 + kRun);         // [kRun]
    uint32_t* si1 = si0 + kRun;                                      // [kRun]
    double* gd = reinterpret_cast<double*>(si1 + kRun);              // [d]
    float* rows = reinterpret_cast<float*>(gd + d);                  // [kQRows][d+1]
    const int64_t zh = blockIdx.x / g.N;
    const int64_t n = blockIdx.x % g.N;
    const int64_t len = g.seg_rows(n);
    const bool local_sort = len <= kRun;
    const int64_t z = zh / g.hq;
    const float* gsrc = guide + (z * g.hkv + g.kvh(zh)) * d;
    for (int64_t i = threadIdx.x; i < d; i += blockDim.x) gd[i] = (double)gsrc[i];
    const int64_t qb = g.q_base(zh);
    const int64_t rs = d + 1;
    double col_acc[4] = {0.0, 0.0, 0.0, 0.0};  // columns tid, tid+128, ... (d <= 512)
    for (int64_t c0 = 0; c0 < len; c0 += kQRows) {
        const int64_t cn = min((int64_t)kQRows, len - c0);
        __syncthreads();
        if (g.in_bf16 && (d % 8) == 0 && (g.qs[2] % 8) == 0) {
            const int64_t vec = d / 8;  // 16-byte vectors per row
            for (int64_t e = threadIdx.x; e < cn * vec; e += blockDim.x) {
                const int64_t r = e / vec, c = (e % vec) * 8;
                const uint4 w = *reinterpret_cast<const uint4*>(
                    reinterpret_cast<const __nv_bfloat16*>(q) + qb + (n * g.S + c0 + r) * g.qs[2] + c);
                const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&w);
                float* dst = rows + r * rs + c;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float2 f = __bfloat1622float2(h2[u]);
                    dst[2 * u] = f.x;
                    dst[2 * u + 1] = f.y;
                }
            }
        } else {
            for (int64_t e = threadIdx.x; e < cn * d; e += blockDim.x) {
                const int64_t r = e / d, c = e % d;
                rows[r * rs + c] = ld_in(q, qb + (n * g.S + c0 + r) * g.qs[2] + c, g.in_bf16);
            }
        }
        __syncthreads();
        if (threadIdx.x < 128) {
            for (int j = 0; j < 4; ++j) {
                const int64_t c = threadIdx.x + (int64_t)j * 128;
                if (c < d) {
                    double acc = col_acc[j];
                    for (int64_t r = 0; r < cn; ++r) acc += (double)rows[r * rs + c];
                    col_acc[j] = acc;
                }
            }
        } else if (threadIdx.x - 128 < cn) {
            const int rr = threadIdx.x - 128;
            const float* row = rows + rr * rs;
            double acc = 0.0;
            for (int64_t c = 0; c < d; ++c) acc = fma((double)row[c], gd[c], acc);
            const uint64_t key = desc_key(acc);
            const int64_t pos = c0 + rr;
            if (local_sort) {
                sk0[pos] = key;
                si0[pos] = (uint32_t)pos;
            } else {
                qkey[zh * g.N * g.S + n * g.S + pos] = key;
            }
        }
    }
    const double inv = 1.0 / (double)len;
    if (threadIdx.x < 128)
        for (int j = 0; j < 4; ++j) {
            const int64_t c = threadIdx.x + (int64_t)j * 128;
            if (c < d) q_mean[(zh * g.N + n) * d + c] = (float)(col_acc[j] * inv);
        }
    if (!local_sort) return;
    for (int64_t i = len + threadIdx.x; i < kRun; i += blockDim.x) {
        sk0[i] = ~0ull;
        si0[i] = 0xffffffffu;
    }
    __syncthreads();
    const int which = block_merge_sort<kQThreads, kRun / kQThreads>(sk0, si0, sk1, si1);
    const uint32_t* res = which ? si1 : si0;
    int32_t* out = q_perm + (zh * g.N + n) * g.S;
    for (int64_t i = threadIdx.x; i < len; i += blockDim.x) out[i] = (int32_t)res[i];
}

// Fast q ranking for the product shape (bf16, D = 128, 16-B aligned rows): 256 threads per
// (zh, n), 3 CTAs per SM. Rows stream through two shared buffers of 128 rows (odd 65-word row
// stride: the per-row dot and the per-column sum both read conflict-free). Every thread
// prefetches 1/256 of chunk c+1 into registers while warps 0-3 score the 128 rows of chunk c
// (one row per thread, fp64 sequential over d) and warps 4-7 extend the 128 column sums (fp64
// sequential over rows). The sort buffers reuse the staging memory. Same arithmetic, same
// order as q_rank_kernel / mean_pool_rows + dot_f.
constexpr int kQF_Threads = 256;
constexpr int kQF_Rows = 128;
constexpr int kQF_W = 65;  // 32-bit words per staged row (64 used)
constexpr int kQF_Per = kQF_Rows * 16 / kQF_Threads;  // 16-B pieces per thread per chunk (8)
constexpr size_t kQF_Stage = sizeof(uint32_t) * 2 * kQF_Rows * kQF_W;
constexpr size_t kQF_Sort = (2 * sizeof(uint64_t) + 2 * sizeof(uint32_t)) * kRun;
constexpr size_t kQF_Smem = sizeof(double) * 128 + (kQF_Stage > kQF_Sort ? kQF_Stage : kQF_Sort);

// Register-prefetched staging of 256 bf16 rows of 128 columns (row stride `rs` elements).
struct RowStager {
    uint4 reg[kQF_Per];
    __device__ void fetch(const __nv_bfloat16* base, int64_t rs, int r0, int len) {
#pragma unroll
        for (int i = 0; i < kQF_Per; ++i) {
            const int e = threadIdx.x + i * kQF_Threads;
            const int r = e >> 4, p = e & 15;
            reg[i] = (r0 + r < len) ? *reinterpret_cast<const uint4*>(base + (int64_t)(r0 + r) * rs + p * 8)
                                    : make_uint4(0, 0, 0, 0);
        }
    }
    __device__ void stash(uint32_t* dst) const {
#pragma unroll
        for (int i = 0; i < kQF_Per; ++i) {
            const int e = threadIdx.x + i * kQF_Threads;
            const int r = e >> 4, p = e & 15;
            uint32_t* d = dst + r * kQF_W + p * 4;
            d[0] = reg[i].x; d[1] = reg[i].y; d[2] = reg[i].z; d[3] = reg[i].w;
        }
    }
};

// fp64 running sum of column `col` over rows [0, cn) of a staged chunk, in row order.
__device__ __forceinline__ double column_sum(const uint32_t* buf, int col, int cn, double acc) {
    const uint32_t* cp = buf + (col >> 1);
    const int sh = (col & 1) ? 0 : 16;
    int r = 0;
    for (; r + 8 <= cn; r += 8) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __uint_as_float((cp[(r + u) * kQF_W] << sh) & 0xffff0000u);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += (double)v[u];
    }
    for (; r < cn; ++r) acc += (double)__uint_as_float((cp[r * kQF_W] << sh) & 0xffff0000u);
    return acc;
}

__global__ void __launch_bounds__(kQF_Threads, 3)
q_rank128_kernel(const __nv_bfloat16* __restrict__ q, Geo g, const float* __restrict__ guide,
                 float* __restrict__ q_mean, uint64_t* __restrict__ qkey, int32_t* __restrict__ q_perm) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* gd = reinterpret_cast<double*>(smem_raw);        // [128]
    uint32_t* stage = reinterpret_cast<uint32_t*>(gd + 128);  // [2][128][65]; after the row loop:
    uint64_t* sk0 = reinterpret_cast<uint64_t*>(gd + 128);    // sort buffers (keys round-trip
    uint64_t* sk1 = sk0 + kRun;                               // through qkey, L2-resident)
    uint32_t* si0 = reinterpret_cast<uint32_t*>(sk1 + kRun);
    uint32_t* si1 = si0 + kRun;
    const int tid = threadIdx.x;
    const int64_t zh = blockIdx.x / g.N;
    const int64_t n = blockIdx.x % g.N;
    const int len = (int)g.seg_rows(n);
    const bool local_sort = len <= kRun;
    const int64_t z = zh / g.hq;
    const float* gsrc = guide + (z * g.hkv + g.kvh(zh)) * 128;
    if (tid < 128) gd[tid] = (double)gsrc[tid];
    const __nv_bfloat16* qseg = q + g.q_base(zh) + n * g.S * g.qs[2];
    const int nchunks = (len + kQF_Rows - 1) / kQF_Rows;
    RowStager rows;
    rows.fetch(qseg, g.qs[2], 0, len);
    rows.stash(stage);
    __syncthreads();
    double col_acc = 0.0;
    for (int c = 0; c < nchunks; ++c) {
        const int r0 = c * kQF_Rows;
        const int cn = min(kQF_Rows, len - r0);
        const uint32_t* buf = stage + (c & 1) * kQF_Rows * kQF_W;
        if (c + 1 < nchunks) rows.fetch(qseg, g.qs[2], r0 + kQF_Rows, len);
        if (tid < 128) {
            if (tid < cn) {
                const uint32_t* row = buf + tid * kQF_W;
                double acc = 0.0;
#pragma unroll 8
                for (int w = 0; w < 64; ++w) {
                    const uint32_t x = row[w];
                    acc = fma((double)__uint_as_float(x << 16), gd[2 * w], acc);
                    acc = fma((double)__uint_as_float(x & 0xffff0000u), gd[2 * w + 1], acc);
                }
                qkey[zh * g.N * g.S + n * g.S + r0 + tid] = desc_key(acc);
            }
        } else {
            col_acc = column_sum(buf, tid - 128, cn, col_acc);
        }
        if (c + 1 < nchunks) rows.stash(stage + ((c + 1) & 1) * kQF_Rows * kQF_W);
        __syncthreads();
    }
    if (tid >= 128) q_mean[(zh * g.N + n) * 128 + (tid - 128)] = (float)(col_acc * (1.0 / (double)len));
    if (!local_sort) return;
    const uint64_t* kseg = qkey + zh * g.N * g.S + n * g.S;
    for (int i = tid; i < kRun; i += kQF_Threads) {
        sk0[i] = i < len ? kseg[i] : ~0ull;
        si0[i] = i < len ? (uint32_t)i : 0xffffffffu;
    }
    __syncthreads();
    const int which = block_merge_sort<kQF_Threads, kRun / kQF_Threads>(sk0, si0, sk1, si1);
    const uint32_t* res = which ? si1 : si0;
    int32_t* out = q_perm + (zh * g.N + n) * g.S;
    for (int i = tid; i < len; i += kQF_Threads) out[i] = (int32_t)res[i];
}

// Segment means for the product shape (bf16, D = 128): the same staged stream, column sums only.
// grid (z * heads, nseg_out).
__global__ void __launch_bounds__(kQF_Threads, 1)
seg_mean128_kernel(const __nv_bfloat16* __restrict__ x, int64_t heads_per_z, int64_t s0, int64_t s1, int64_t s2,
                   int64_t S, int64_t N, int64_t last_len, int64_t nseg_out, float* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t* stage = reinterpret_cast<uint32_t*>(smem_raw);
    const int tid = threadIdx.x;
    const int64_t slice = blockIdx.x, n = blockIdx.y;
    const int len = (int)((n + 1 == N) ? last_len : S);
    const __nv_bfloat16* seg = x + (slice / heads_per_z) * s0 + (slice % heads_per_z) * s1 + n * S * s2;
    const int nchunks = (len + kQF_Rows - 1) / kQF_Rows;
    RowStager rows;
    rows.fetch(seg, s2, 0, len);
    rows.stash(stage);
    __syncthreads();
    double acc = 0.0;
    for (int c = 0; c < nchunks; ++c) {
        const int r0 = c * kQF_Rows;
        const int cn = min(kQF_Rows, len - r0);
        if (c + 1 < nchunks) rows.fetch(seg, s2, r0 + kQF_Rows, len);
        if (tid < 128) acc = column_sum(stage + (c & 1) * kQF_Rows * kQF_W, tid, cn, acc);
        if (c + 1 < nchunks) rows.stash(stage + ((c + 1) & 1) * kQF_Rows * kQF_W);
        __syncthreads();
    }
    if (tid < 128) out[(slice * nseg_out + n) * 128 + tid] = (float)(acc * (1.0 / (double)len));
}

bool q_rank128_ok(const Geo& g, const void* q) {
    return g.in_bf16 && g.d == 128 && g.qs[0] % 8 == 0 && g.qs[1] % 8 == 0 && g.qs[2] % 8 == 0 &&
           (reinterpret_cast<uintptr_t>(q) & 15) == 0;
}

// q ranking dispatch: fast kernel for the product shape, generic kernel otherwise.
cudaError_t launch_q_rank(const Geo& g, const void* q, const float* guide, float* q_mean, uint64_t* qkey,
                          int32_t* q_perm, cudaStream_t st) {
    if (q_rank128_ok(g, q)) {
        cudaFuncSetAttribute(q_rank128_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kQF_Smem);
        q_rank128_kernel<<<(unsigned)(g.z * g.hq * g.N), kQF_Threads, kQF_Smem, st>>>(
            reinterpret_cast<const __nv_bfloat16*>(q), g, guide, q_mean, qkey, q_perm);
        return cudaGetLastError();
    }
    const size_t smem = (2 * sizeof(uint64_t) + 2 * sizeof(uint32_t)) * kRun + sizeof(double) * g.d +
                        sizeof(float) * kQRows * (g.d + 1);
    cudaFuncSetAttribute(q_rank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    q_rank_kernel<<<(unsigned)(g.z * g.hq * g.N), kQThreads, smem, st>>>(q, g, guide, q_mean, qkey, q_perm);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- kv scoring
// One CTA (128 threads) per (z, kv head, block of 128 keys). Register tile per thread:
// 4 keys x 8 (q head, segment) pairs = 32 fp64 accumulators; each K element is converted
// once and feeds 8 DFMAs, each q_mean element (fp64, broadcast from smem) feeds 4.
// s = sum_d q_mean[h,n,d] * K[t,d] in fp64, sequential in d (dot_f plan.cpp:14-20).
constexpr int kSK = 128;       // keys per CTA
constexpr int kSKThreads = 128;
constexpr int kSPairs = 32;    // pairs per batch (4 groups x 8)

__global__ void __launch_bounds__(kSKThreads)
kv_score_kernel(const void* __restrict__ k, Geo g, const float* __restrict__ q_mean,
                uint64_t* __restrict__ kvkey) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int d = (int)g.d;
    double* qm = reinterpret_cast<double*>(smem_raw);           // [d][kSPairs]
    float* kt = reinterpret_cast<float*>(qm + d * kSPairs);     // [d][kSK]
    const int64_t zg = blockIdx.y;  // z * hkv + kvh
    const int64_t z = zg / g.hkv, kvh = zg % g.hkv;
    const int64_t t0 = (int64_t)blockIdx.x * kSK;
    const int kg = threadIdx.x % 32, qg = threadIdx.x / 32;
    const int64_t kb = z * g.ks[0] + kvh * g.ks[1];
    for (int e = threadIdx.x; e < kSK * d; e += kSKThreads) {
        const int r = e / d, c = e % d;
        const int64_t row = t0 + r;
        kt[c * kSK + r] = (row < g.l) ? ld_in(k, kb + row * g.ks[2] + c, g.in_bf16) : 0.0f;
    }
    const int64_t n_lo = t0 / g.S + 1;  // first segment whose prefix reaches t0
    const int64_t nsegs = (n_lo < g.N) ? g.N - n_lo : 0;
    const int64_t pairs = g.group * nsegs;
    const int64_t kvp = g.kv_per_head();
    for (int64_t p0 = 0; p0 < pairs; p0 += kSPairs) {
        __syncthreads();
        for (int e = threadIdx.x; e < kSPairs * d; e += kSKThreads) {
            const int b = e / d, c = e % d;
            const int64_t p = p0 + b;
            double val = 0.0;
            if (p < pairs) {
                const int64_t h = kvh * g.group + p / nsegs;
                const int64_t n = n_lo + p % nsegs;
                val = (double)q_mean[((z * g.hq + h) * g.N + n) * d + c];
            }
            qm[c * kSPairs + b] = val;
        }
        __syncthreads();
        double acc[4][8];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int b = 0; b < 8; ++b) acc[i][b] = 0.0;
        const float4* kt4 = reinterpret_cast<const float4*>(kt) + kg;
        const double2* qm2 = reinterpret_cast<const double2*>(qm) + qg * 4;
#pragma unroll 2
        for (int c = 0; c < d; ++c) {
            const float4 kk = kt4[c * (kSK / 4)];
            const double kd[4] = {(double)kk.x, (double)kk.y, (double)kk.z, (double)kk.w};
            const double2* qrow = qm2 + c * (kSPairs / 2);
            double qv[8];
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const double2 x = qrow[b];
                qv[2 * b] = x.x;
                qv[2 * b + 1] = x.y;
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int b = 0; b < 8; ++b) acc[i][b] = fma(qv[b], kd[i], acc[i][b]);
        }
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const int64_t p = p0 + qg * 8 + b;
            if (p >= pairs) break;
            const int64_t h = kvh * g.group + p / nsegs;
            const int64_t n = n_lo + p % nsegs;
            const int64_t zh = z * g.hq + h;
            uint64_t* dst = kvkey + zh * kvp + g.kv_off(n);
            const int64_t t = t0 + kg * 4;
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (t + i < n * g.S) dst[t + i] = desc_key(acc[i][b]);
        }
    }
}

// Fast kv scoring for the product shape (bf16 K, D = 128): a register-tiled fp64 GEMM
// S[pairs x keys] = q_mean[pairs x 128] . K^T. CTA (128 threads, 2 per SM) = 64 (q head,
// segment) pairs x 128 keys, the whole d = 128 staged once: K as raw bf16 rows (272-B stride,
// conflict-free 16-B row reads), q_mean as fp64 [d][pair]. Warp tile 32 pairs x 64 keys; lane =
// 4 pair groups x 8 key groups holds pairs {8i + 2pg + e} x keys {kg + 8r}: 8 x 8 fp64
// accumulators. Per d a warp reads 5 x 16 B per lane (K once per 8 d) for 64 DFMAs per lane, so
// the FP64 pipe, not shared memory, is the bound. bf16 -> fp64 is exact. Each output
// accumulates d = 0..127 in order with DFMA from 0.0, exactly dot_f's sequence (plan.cpp:14-20).
// CTA = (key block kb, pair batch). A block's pair count (group x later segments) is rarely a
// multiple of 64: a remainder of <= 32 pairs is done by ONE "wide" CTA over the two key blocks
// kb, kb + 1 of the same segment (32 pairs x 256 keys, same shared memory), so padded work drops
// from 19 % to 10 %. CTAs without work exit.
constexpr int kKS_Pairs = 64, kKS_Threads = 128, kKS_KStride = 136;  // bf16 per staged K row
constexpr size_t kKS_SmemNarrow = sizeof(double) * 128 * kKS_Pairs + sizeof(__nv_bfloat16) * kSK * kKS_KStride;
constexpr size_t kKS_SmemWide = sizeof(double) * 128 * (kKS_Pairs / 2) + sizeof(__nv_bfloat16) * 2 * kSK * kKS_KStride;
constexpr size_t kKS_Smem = kKS_SmemNarrow > kKS_SmemWide ? kKS_SmemNarrow : kKS_SmemWide;  // 100 KB: 2 CTAs / SM

__device__ __forceinline__ double bf16_lo_to_f64(uint32_t w) { return (double)__uint_as_float(w << 16); }
__device__ __forceinline__ double bf16_hi_to_f64(uint32_t w) { return (double)__uint_as_float(w & 0xffff0000u); }

__global__ void __launch_bounds__(kKS_Threads, 2)
kv_score128_kernel(const __nv_bfloat16* __restrict__ k, Geo g, const float* __restrict__ q_mean,
                   uint64_t* __restrict__ kvkey, int max_batches, int64_t n_hi, const int32_t* __restrict__ skip) {
    if (skip && *skip) return;  // device-side gate (plan levels)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t kb = blockIdx.x / max_batches;
    const int batch = blockIdx.x % max_batches;
    const int64_t zg = blockIdx.y;  // z * hkv + kvh
    const int64_t z = zg / g.hkv, kvh = zg % g.hkv;
    const int64_t t0 = kb * kSK;
    const int64_t n_lo = t0 / g.S + 1;
    const int64_t n_end = n_hi < g.N ? n_hi : g.N;  // segments [n_lo, n_end) only
    const int64_t nsegs = (n_lo < n_end) ? n_end - n_lo : 0;
    const int64_t pairs = g.group * nsegs;
    auto pair_hn = [&](int64_t p, int64_t& h, int64_t& n) {  // pair p of this key block -> (q head, segment)
        h = kvh * g.group + p / nsegs;
        n = n_lo + p % nsegs;
    };
    const int64_t p0 = (int64_t)batch * kKS_Pairs;
    if (p0 >= pairs) return;
    const int64_t rem = pairs - p0;  // pairs from p0 on
    const bool can_wide = g.S % (2 * kSK) == 0;  // kb, kb + 1 always share a segment
    const bool wide = can_wide && rem <= kKS_Pairs / 2;
    if (wide && (kb & 1)) return;  // the even block's wide CTA covers this block
    const int np = wide ? kKS_Pairs / 2 : kKS_Pairs;  // pairs in the tile (Qd row length)
    const int nrows = wide ? 2 * kSK : kSK;           // staged K rows
    double* Qd = reinterpret_cast<double*>(smem_raw);                           // [128 d][np]
    __nv_bfloat16* Kn = reinterpret_cast<__nv_bfloat16*>(Qd + 128 * np);       // [nrows][136]
    {  // stage K rows (16-B chunks) and q_mean (fp32 -> fp64, transposed)
        const __nv_bfloat16* kbase = k + z * g.ks[0] + kvh * g.ks[1];
        for (int half = 0; half < nrows / kSK; ++half) {
            const int64_t tb = t0 + half * kSK;
            uint4 kr[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int c = tid + i * kKS_Threads, row = c >> 4, col = c & 15;
                kr[i] = (tb + row < g.l) ? *reinterpret_cast<const uint4*>(kbase + (tb + row) * g.ks[2] + col * 8)
                                         : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int c = tid + i * kKS_Threads, row = c >> 4, col = c & 15;
                *reinterpret_cast<uint4*>(Kn + (half * kSK + row) * kKS_KStride + col * 8) = kr[i];
            }
        }
        // q_mean: thread -> (pair qp, 64 / (128 / np) d values)
        const int parts = kKS_Threads / np;  // threads per pair: 2 (64 pairs) or 4 (32 pairs)
        const int qp = tid / parts, qh = tid % parts, dlen = 128 / parts;
        const int64_t pq = p0 + qp;
        const float* qsrc = nullptr;
        if (pq < pairs) {
            int64_t h, n;
            pair_hn(pq, h, n);
            qsrc = q_mean + ((z * g.hq + h) * g.N + n) * 128 + qh * dlen;
        }
#pragma unroll 4
        for (int c = 0; c < dlen / 4; ++c) {
            const float4 x = qsrc ? reinterpret_cast<const float4*>(qsrc)[c] : make_float4(0.f, 0.f, 0.f, 0.f);
            const int d = qh * dlen + 4 * c;
            Qd[(d + 0) * np + qp] = (double)x.x;
            Qd[(d + 1) * np + qp] = (double)x.y;
            Qd[(d + 2) * np + qp] = (double)x.z;
            Qd[(d + 3) * np + qp] = (double)x.w;
        }
    }
    __syncthreads();
    // warp -> (pair half, 64-key quarter) of a 64 x 128 tile, or (key block, 64-key half) of a
    // wide 32 x 256 tile: either way keys [64 wk_row, +64) of the staged rows and 32 pairs
    const int pg = lane >> 3, kg = lane & 7;
    const int wpair = wide ? 0 : (warp & 1);                      // 32-pair group
    const int wrow = wide ? warp : (warp >> 1);                   // 64-row group of the staged K
    double acc[8][8];  // [pair 2i+e][key r]
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int r = 0; r < 8; ++r) acc[i][r] = 0.0;
    const __nv_bfloat16* krow = Kn + (64 * wrow + kg) * kKS_KStride;
    const double* qcol = Qd + 32 * wpair + 2 * pg;
#pragma unroll 1
    for (int dg = 0; dg < 16; ++dg) {
        uint4 kr[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) kr[r] = *reinterpret_cast<const uint4*>(krow + 8 * r * kKS_KStride + 8 * dg);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int d = 8 * dg + j;
            double qv[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const double2 x = *reinterpret_cast<const double2*>(qcol + d * np + 8 * i);
                qv[2 * i] = x.x;
                qv[2 * i + 1] = x.y;
            }
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const uint32_t w = (j >> 1) == 0 ? kr[r].x : (j >> 1) == 1 ? kr[r].y : (j >> 1) == 2 ? kr[r].z : kr[r].w;
                const double kd = (j & 1) ? bf16_hi_to_f64(w) : bf16_lo_to_f64(w);
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[i][r] = fma(qv[i], kd, acc[i][r]);
            }
        }
    }
    const int64_t kvp = g.kv_per_head();
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t p = p0 + 32 * wpair + 8 * (i >> 1) + 2 * pg + (i & 1);
        if (p >= pairs) continue;
        int64_t h, n;
        pair_hn(p, h, n);
        uint64_t* dst = kvkey + (z * g.hq + h) * kvp + g.kv_off(n);
        const int64_t lim = n * g.S;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int64_t t = t0 + 64 * wrow + kg + 8 * r;
            if (t < lim) dst[t] = desc_key(acc[i][r]);
        }
    }
}

bool kv_score128_ok(const Geo& g, const void* k) {
    return g.in_bf16 && g.d == 128 && g.ks[0] % 8 == 0 && g.ks[1] % 8 == 0 && g.ks[2] % 8 == 0 &&
           (reinterpret_cast<uintptr_t>(k) & 15) == 0 && g.S % 2 == 0;
}

// Exact scores of segments [1, n_hi) (n_hi >= N: all); skip (device, optional): the launch exits
// at once when *skip != 0.
cudaError_t launch_kv_score(const Geo& g, const void* k, const float* q_mean, uint64_t* kvkey, cudaStream_t st,
                            int64_t n_hi = INT64_MAX, const int32_t* skip = nullptr) {
    const int64_t n_end = std::min<int64_t>(n_hi, g.N);
    if (n_end < 2) return cudaSuccess;
    const int64_t keys = (n_end - 1) * g.S;  // tokens that appear in some prefix
    const int64_t blocks = (keys + kSK - 1) / kSK;
    if (kv_score128_ok(g, k)) {
        const int max_batches = (int)((g.group * (n_end - 1) + kKS_Pairs - 1) / kKS_Pairs);
        dim3 grid((unsigned)(blocks * max_batches), (unsigned)(g.z * g.hkv));
        cudaFuncSetAttribute(kv_score128_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kKS_Smem);
        kv_score128_kernel<<<grid, kKS_Threads, kKS_Smem, st>>>(reinterpret_cast<const __nv_bfloat16*>(k), g, q_mean,
                                                         kvkey, max_batches, n_hi, skip);
        return cudaGetLastError();
    }
    if (n_end < g.N || skip) return cudaErrorInvalidValue;  // generic scoring: whole plans only
    const size_t smem = sizeof(double) * g.d * kSPairs + sizeof(float) * g.d * kSK;
    cudaFuncSetAttribute(kv_score_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid((unsigned)blocks, (unsigned)(g.z * g.hkv));
    kv_score_kernel<<<grid, kSKThreads, smem, st>>>(k, g, q_mean, kvkey);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- sort
// Segment geometry of a sort family. Segment n of head zh occupies
// [zh * head_stride + off(n), + len(n)) in both the key buffer and the output
// permutation. kind 0: q segments (off nS, len seg_rows); kind 1: kv prefixes
// (off S n(n-1)/2, len nS, n >= 1).
struct SortGeo {
    int kind;
    int64_t S, N, last_len, head_stride, heads;
    int64_t units_per_head;  // runs (== merge tiles) per head
    const int64_t* cum;      // [N+1] cumulative runs per head
    __device__ int64_t len(int64_t n) const {
        if (kind == 0) return (n + 1 == N) ? last_len : S;
        return n * S;
    }
    __device__ int64_t off(int64_t n) const { return kind == 0 ? n * S : S * n * (n - 1) / 2; }
};

__global__ void seg_table_kernel(int kind, int64_t S, int64_t N, int64_t last_len,
                                 int64_t* __restrict__ cum) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int64_t acc = 0;
    for (int64_t n = 0; n < N; ++n) {
        cum[n] = acc;
        const int64_t len = (kind == 0) ? ((n + 1 == N) ? last_len : S) : n * S;
        acc += (len + kRun - 1) / kRun;
    }
    cum[N] = acc;
}

__device__ __forceinline__ void locate(const SortGeo& sg, int64_t unit, int64_t& zh, int64_t& n,
                                       int64_t& j) {
    zh = unit / sg.units_per_head;
    const int64_t r = unit % sg.units_per_head;
    int64_t lo = 0, hi = sg.N - 1;  // largest n with cum[n] <= r
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (sg.cum[mid] <= r) lo = mid; else hi = mid - 1;
    }
    n = lo;
    j = r - sg.cum[n];
}

__device__ __forceinline__ bool elt_less(uint64_t ka, uint32_t ia, uint64_t kb, uint32_t ib) {
    return ka < kb || (ka == kb && ia < ib);
}

// Sorts run j of segment n (kRun elements) and writes either the sorted
// (key, idx) run or, if `final_out`, the int32 permutation directly.
__global__ void __launch_bounds__(kSortThreads)
run_sort_kernel(SortGeo sg, const uint64_t* __restrict__ keys, uint64_t* __restrict__ okeys,
                uint32_t* __restrict__ oidx, int32_t* __restrict__ final_out) {
    __shared__ uint64_t sk[2][kRun];
    __shared__ uint32_t si[2][kRun];
    int64_t zh, n, j;
    locate(sg, blockIdx.x, zh, n, j);
    const int64_t len = sg.len(n);
    const int64_t r0 = j * kRun;
    const int64_t cnt = min((int64_t)kRun, len - r0);
    const int64_t base = zh * sg.head_stride + sg.off(n);
    for (int i = threadIdx.x; i < kRun; i += kSortThreads) {
        if (i < cnt) {
            sk[0][i] = keys[base + r0 + i];
            si[0][i] = (uint32_t)(r0 + i);
        } else {
            sk[0][i] = ~0ull;
            si[0][i] = 0xffffffffu;
        }
    }
    __syncthreads();
    const int w = block_merge_sort<kSortThreads, kRun / kSortThreads>(sk[0], si[0], sk[1], si[1]);
    for (int i = threadIdx.x; i < cnt; i += kSortThreads) {
        if (final_out) {
            final_out[base + r0 + i] = (int32_t)si[w][i];
        } else {
            okeys[base + r0 + i] = sk[w][i];
            oidx[base + r0 + i] = si[w][i];
        }
    }
}

// Merges sorted runs of width w pairwise; CTA = one 2048-output tile, each thread merges
// 8 consecutive outputs after one merge-path search inside the CTA's smem slices.
__global__ void __launch_bounds__(kSortThreads)
merge_pass_kernel(SortGeo sg, int64_t w, const uint64_t* __restrict__ ikeys,
                  const uint32_t* __restrict__ iidx, uint64_t* __restrict__ okeys,
                  uint32_t* __restrict__ oidx, int32_t* __restrict__ final_out) {
    constexpr int E = kRun / kSortThreads;
    __shared__ uint64_t sk[kRun];
    __shared__ uint32_t si[kRun];
    __shared__ int64_t split[2];
    int64_t zh, n, j;
    locate(sg, blockIdx.x, zh, n, j);
    const int64_t len = sg.len(n);
    const int64_t base = zh * sg.head_stride + sg.off(n);
    const int64_t o0 = j * kRun;
    const int64_t p0 = (o0 / (2 * w)) * (2 * w);
    const int64_t a_beg = p0, a_len = min(w, len - p0);
    const int64_t b_beg = p0 + a_len, b_len = max((int64_t)0, min(w, len - b_beg));
    const int64_t d0 = o0 - p0;
    const int64_t d1 = min(d0 + (int64_t)kRun, a_len + b_len);
    const uint64_t* ak = ikeys + base + a_beg;
    const uint32_t* ai = iidx + base + a_beg;
    const uint64_t* bk = ikeys + base + b_beg;
    const uint32_t* bi = iidx + base + b_beg;
    if (threadIdx.x < 2) {
        const int64_t diag = threadIdx.x == 0 ? d0 : d1;
        int64_t lo = max((int64_t)0, diag - b_len), hi = min(diag, a_len);
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            const int64_t bj = diag - 1 - mid;
            if (elt_less(ak[mid], ai[mid], bk[bj], bi[bj])) lo = mid + 1; else hi = mid;
        }
        split[threadIdx.x] = lo;
    }
    __syncthreads();
    const int64_t a0 = split[0], a1 = split[1];
    const int64_t b0 = d0 - a0, b1 = d1 - a1;
    const int na = (int)(a1 - a0), nb = (int)(b1 - b0);
    for (int i = threadIdx.x; i < na; i += kSortThreads) {
        sk[i] = ak[a0 + i];
        si[i] = ai[a0 + i];
    }
    for (int i = threadIdx.x; i < nb; i += kSortThreads) {
        sk[na + i] = bk[b0 + i];
        si[na + i] = bi[b0 + i];
    }
    __syncthreads();
    const int tot = na + nb;
    const int o = threadIdx.x * E;
    if (o >= tot) return;
    const int a = merge_path(sk, si, na, sk + na, si + na, nb, o);
    uint64_t ok[E];
    uint32_t oi[E];
    merge_seq<E>(sk, si, na, sk + na, si + na, nb, a, o - a, ok, oi);
    const int64_t out0 = base + o0 + o;
    const int cnt = min(E, tot - o);
#pragma unroll
    for (int e = 0; e < E; ++e) {
        if (e >= cnt) break;
        if (final_out) {
            final_out[out0 + e] = (int32_t)oi[e];
        } else {
            okeys[out0 + e] = ok[e];
            oidx[out0 + e] = oi[e];
        }
    }
}

// ---------------------------------------------------------------- top-T selection
// For the fused operator only the leading chunks of each kv_perm segment are consumed (the walk
// stops early), so instead of fully sorting the prefix the plan materialises its exact top-T,
// per (zh, n >= 1), in two kernels:
//  * sel_scan_kernel (256 threads, several CTAs/SM, HBM-latency bound): radix-sort a 2048-key
//    sample, take a threshold key whose expected rank is ~1.15 T, compact every key <= threshold
//    in INDEX order (coalesced 8-key loads per thread + a block scan) into the segment's own slot
//    of the spare key1 / idx1 workspace. If the threshold catches fewer than T keys or more than
//    the capacity it retries with another sample rank; after the retries it keeps a
//    capacity-sized best-effort set and flags the segment (the host then builds the full plan).
//    Segments with at most kSelCap keys skip the scan: all their keys are candidates.
//  * sel_sort_kernel (512 threads, 1 CTA/SM, shared-memory bound): a stable block radix sort of
//    the candidates by key over only the bits where they differ (ties keep index order), then
//    the first T indices -- exactly the first T entries of argsort_desc_stable (a stable
//    sort's top T is a prefix of the full order).
// Split because the two phases want different occupancy: fused in one 512-thread CTA per SM
// the scan's load latency and the sort's shared-memory traffic never overlapped.
constexpr int kSelThreads = 512;
constexpr int kSelItems = 16;
constexpr int kSelCap = kSelThreads * kSelItems;  // 8192 candidates
constexpr int kSelSample = 2048;
constexpr int kSelRadixBits = 6;
constexpr int kScanThreads = 256;

using SelSort = cub::BlockRadixSort<uint64_t, kSelThreads, kSelItems, uint32_t, kSelRadixBits>;
using SampSort = cub::BlockRadixSort<uint64_t, kScanThreads, kSelSample / kScanThreads, cub::NullType, kSelRadixBits>;

struct SelSeg {
    int64_t zh, n, len, tt, off;  // off: the segment's first key in the [zh][kv_off] key layout
};
__device__ __forceinline__ SelSeg sel_seg(const Geo& g, const int32_t* seg_list, int64_t topt, int64_t lvl_base) {
    SelSeg s;
    if (seg_list) {
        s.zh = seg_list[blockIdx.x] / g.N;
        s.n = seg_list[blockIdx.x] % g.N;
    } else {
        s.zh = blockIdx.x / (g.N - 1);
        s.n = 1 + blockIdx.x % (g.N - 1);
    }
    s.len = s.n * g.S;
    s.tt = min(topt, s.len - lvl_base);
    s.off = s.zh * g.kv_per_head() + g.kv_off(s.n);
    return s;
}

// Level > 0 (seg_list / prev given): the same selection restricted to the keys that follow the
// previous level's last entry in the (key, index) order, i.e. entries [lvl_base, lvl_base + T).
__global__ void __launch_bounds__(kScanThreads, 3)
sel_scan_kernel(Geo g, const uint64_t* __restrict__ kvkey, int64_t topt, uint64_t* __restrict__ ckey,
                uint32_t* __restrict__ cidx, int32_t* __restrict__ ccount, int32_t* __restrict__ flags,
                const int32_t* __restrict__ seg_list, const int32_t* __restrict__ prev, int64_t lvl_base,
                const int32_t* __restrict__ nseg_dev, const int64_t* __restrict__ lvl_base_dev, int64_t n_max) {
    if (nseg_dev && (int64_t)blockIdx.x >= *nseg_dev) return;  // device-sized level: CTA not used
    if (lvl_base_dev) lvl_base = *lvl_base_dev;
    __shared__ typename SampSort::TempStorage samp;
    __shared__ int s_wsum[kScanThreads / 32];
    __shared__ int s_count;
    __shared__ uint64_t s_theta;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const SelSeg sg = sel_seg(g, seg_list, topt, lvl_base);
    const int64_t len = sg.len, tt = sg.tt;
    if (len <= kSelCap && !prev) return;  // every key is a candidate (sel_sort_kernel reads them)
    if (sg.n >= n_max) return;            // selected by the candidate path (plan_tc.cuh)
    const uint64_t* keys = kvkey + sg.off;
    uint64_t* ck = ckey + sg.off;  // candidates <= min(cap, len) fit the segment's own slot
    uint32_t* ci = cidx + sg.off;
    // keys at or before the bound (the previous level's last entry) are not candidates
    const int64_t bidx = prev ? prev[(sg.zh * g.N + sg.n) * topt + topt - 1] : -1;
    const uint64_t bkey = prev ? keys[bidx] : 0ull;
    auto after = [&](uint64_t k, int64_t i) { return !prev || k > bkey || (k == bkey && i > bidx); };
    // sample: 128 runs of 16 consecutive keys spread over the segment, radix-sorted (a short
    // segment of a later level takes every remaining key instead)
    const bool small = len <= kSelCap;
    constexpr int kPer = kSelSample / kScanThreads;
    uint64_t smp[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
        const int e = tid * kPer + u;
        smp[u] = small ? 0ull : keys[(int64_t)(e / 16) * (len / 128) + e % 16];
    }
    if (!small) SampSort(samp).Sort(smp);  // blocked: thread t holds ranks kPer t .. kPer t + kPer - 1
    // Threshold: first the sample key of the rank expected to hold ~1.15 T of the level's keys;
    // retries step the sample rank by the observed count's distance to the middle of the
    // [T, capacity] window until the window is bracketed, then bisect between the bracketing
    // keys (the count is monotone in the key, so this converges however dense the keys are).
    const double dens = (double)kSelSample / (double)len;  // sample ranks per key
    const double mid = (double)tt + 0.5 * (double)(kSelCap - tt);
    const double want = small ? (double)len : (double)lvl_base + 1.15 * (double)tt + 32.0;
    bool take_all = want >= (double)len;  // every remaining key fits the capacity
    int64_t rank = min((int64_t)ceil(want * dens) + 4, (int64_t)(kSelSample - 1));
    bool have_lo = false, have_hi = false;  // a threshold known to take too few / too many
    uint64_t t_lo = 0ull, t_hi = ~0ull;
    bool ok = false;
    int count = 0;
    for (int attempt = 0; attempt < 8 && !ok; ++attempt) {
        __syncthreads();  // previous attempt's s_count / s_theta reads are done
        const bool bisect = have_lo && have_hi;
        if (bisect) {
            if (tid == 0) s_theta = t_lo + (t_hi - t_lo) / 2;
        } else if (tid == (int)(rank / kPer)) {
            s_theta = take_all ? ~0ull : smp[rank % kPer];
        }
        if (tid == 0) s_count = 0;
        __syncthreads();
        const uint64_t theta = s_theta;
        const bool last_sample = theta == ~0ull;
        // order-preserving compaction of every key <= theta: 8 consecutive keys per thread, the
        // next iteration's keys loaded before this one's are used (the scan is latency-bound)
        constexpr int kU = 8;
        auto load8 = [&](int64_t i0, uint64_t (&kk)[kU]) {
            if (i0 + kU <= len) {
                const ulonglong2* src = reinterpret_cast<const ulonglong2*>(keys + i0);
#pragma unroll
                for (int u = 0; u < kU / 2; ++u) {
                    const ulonglong2 x = src[u];
                    kk[2 * u] = x.x;
                    kk[2 * u + 1] = x.y;
                }
            } else {
#pragma unroll
                for (int u = 0; u < kU; ++u) kk[u] = (i0 + u < len) ? keys[i0 + u] : ~0ull;
            }
        };
        constexpr int64_t kStep = (int64_t)kScanThreads * kU;
        uint64_t nk[kU];
        load8((int64_t)tid * kU, nk);
        for (int64_t b0 = 0; b0 < len; b0 += kStep) {
            const int64_t i0 = b0 + (int64_t)tid * kU;
            uint64_t kk[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) kk[u] = nk[u];
            if (b0 + kStep < len) load8(i0 + kStep, nk);
            uint32_t m = 0;  // taken keys of this thread, bit u
            if (!prev) {  // level 0: a plain threshold; the tail past len is masked
#pragma unroll
                for (int u = 0; u < kU; ++u) m |= (kk[u] <= theta ? 1u : 0u) << u;
                if (i0 + kU > len) m &= (i0 < len) ? (1u << (uint32_t)(len - i0)) - 1u : 0u;
            } else {
#pragma unroll
                for (int u = 0; u < kU; ++u)
                    m |= ((kk[u] <= theta && i0 + u < len && after(kk[u], i0 + u)) ? 1u : 0u) << u;
            }
            const int c = __popc(m);
            int x = c;  // warp inclusive scan
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) s_wsum[warp] = x;
            __syncthreads();
            int wbase = 0, total = 0;
#pragma unroll
            for (int w = 0; w < kScanThreads / 32; ++w) {
                const int v = s_wsum[w];
                wbase += (w < warp) ? v : 0;
                total += v;
            }
            int pos = s_count + wbase + x - c;
            if (m != 0u) {
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    if ((m >> u) & 1u) {
                        if (pos < kSelCap) {
                            ck[pos] = kk[u];
                            ci[pos] = (uint32_t)(i0 + u);
                        }
                        ++pos;
                    }
                }
            }
            __syncthreads();  // s_wsum reusable, s_count read by all
            if (tid == 0) s_count += total;
        }
        __syncthreads();
        const int cnt = s_count;
#ifdef S2O_SEL_DEBUG
        if (tid == 0 && (attempt > 0 || cnt < tt || cnt > kSelCap))
            printf("sel zh %lld n %lld len %lld tt %lld lvl %lld attempt %d rank %lld all %d cnt %d\n", (long long)sg.zh,
                   (long long)sg.n, (long long)len, (long long)tt, (long long)lvl_base, attempt, (long long)rank,
                   (int)take_all, cnt);
#endif
        if (cnt >= tt && cnt <= kSelCap) {
            ok = true;
            count = cnt;
        } else if (cnt < tt) {
            if (last_sample) {  // every remaining key is a candidate and still fewer than T
                count = min(cnt, kSelCap);
                ok = true;
                if (tid == 0) atomicExch(flags, 1);
            }
            have_lo = true;
            t_lo = theta;
            if (!have_hi) {
                rank += max((int64_t)1, (int64_t)ceil((mid - cnt) * dens));
                if (rank >= kSelSample - 1) {
                    rank = kSelSample - 1;
                    take_all = true;
                }
            }
        } else {
            have_hi = true;
            t_hi = theta;
            if (!have_lo) {
                if (rank == 0) {  // below the smallest sample key: bisect from key 0
                    have_lo = true;
                    t_lo = 0ull;
                }
                rank = take_all ? (int64_t)(kSelSample - 1)
                                : max((int64_t)0, rank - max((int64_t)1, (int64_t)ceil((cnt - mid) * dens)));
                take_all = false;
            }
        }
        if (!ok && have_lo && have_hi && t_hi - t_lo <= 1) break;  // equal keys straddle the window
    }
    if (!ok) {
        count = kSelCap;
        if (tid == 0) atomicExch(flags, 1);
    }
    if (tid == 0) ccount[sg.zh * g.N + sg.n] = count;
}

// Sort by a 32-bit coarse key -- the top 32 of the bits where candidates differ -- carrying the
// candidate's position: 6 radix passes over 8-byte pairs instead of 10 over 12-byte ones. The
// coarse sort is stable (index order within equal coarse keys); it is exact unless two coarse-
// equal candidates have different full keys in the wrong order, which is checked and then (rarely)
// settled by the full 64-bit sort.
using SelSortC = cub::BlockRadixSort<uint32_t, kSelThreads, kSelItems, uint32_t, kSelRadixBits>;
using SelXchg = cub::BlockExchange<uint32_t, kSelThreads, kSelItems>;
struct SelSortSmem {  // ~170 KB: 1 CTA / SM
    uint64_t key[kSelCap];  // candidates in index order (striped writes: conflict-free)
    uint32_t idx[kSelCap];
    uint32_t edge_c[kSelItems][kSelThreads / 32];  // each warp's last (coarse, pos) per rank row
    uint32_t edge_p[kSelItems][kSelThreads / 32];
    union {
        typename SelXchg::TempStorage xchg;
        typename SelSortC::TempStorage coarse;
        typename SelSort::TempStorage full;
    } t;
};

__global__ void __launch_bounds__(kSelThreads)
sel_sort_kernel(Geo g, const uint64_t* __restrict__ kvkey, const uint64_t* __restrict__ ckey,
                const uint32_t* __restrict__ cidx, const int32_t* __restrict__ ccount, int64_t topt,
                int32_t* __restrict__ kvtop, const int32_t* __restrict__ seg_list, int level0, int64_t lvl_base,
                const int32_t* __restrict__ nseg_dev, const int64_t* __restrict__ lvl_base_dev) {
    if (nseg_dev && (int64_t)blockIdx.x >= *nseg_dev) return;
    if (lvl_base_dev) lvl_base = *lvl_base_dev;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SelSortSmem& sm = *reinterpret_cast<SelSortSmem*>(smem_raw);
    __shared__ unsigned long long s_or;
    __shared__ uint64_t s_ref;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const SelSeg sg = sel_seg(g, seg_list, topt, lvl_base);
    const int64_t tt = sg.tt;
    int32_t* out = kvtop + (sg.zh * g.N + sg.n) * topt;
    const bool direct = sg.len <= kSelCap && level0;  // every key, in index order
    const int count = direct ? (int)sg.len : ccount[sg.zh * g.N + sg.n];
    const uint64_t* kk = direct ? kvkey + sg.off : ckey + sg.off;
    const uint32_t* ii = cidx + sg.off;
    if (tid == 0) {
        s_or = 0ull;
        s_ref = count > 0 ? kk[0] : 0ull;  // reference key: candidate 0
    }
    __syncthreads();
    const uint64_t ref = s_ref;
    // striped (coalesced) load; bits where candidates differ
    uint64_t ks[kSelItems];
    unsigned long long diff = 0ull;
#pragma unroll
    for (int e = 0; e < kSelItems; ++e) {
        const int i = e * kSelThreads + tid;
        ks[e] = i < count ? kk[i] : ~0ull;
        sm.key[i] = ks[e];
        sm.idx[i] = i < count ? (direct ? (uint32_t)i : ii[i]) : 0xffffffffu;
        if (i < count) diff |= ks[e] ^ ref;
    }
    for (int o = 16; o > 0; o >>= 1) diff |= __shfl_xor_sync(0xffffffffu, diff, o);
    if (lane == 0 && diff) atomicOr(&s_or, diff);
    __syncthreads();
    const unsigned long long all = s_or;
    const int end_bit = all ? 64 - __clzll((long long)all) : 1;
    // coarse key = the top 32 of the differing bits, relative to the common top bits (real
    // candidates share every bit above end_bit); pads (~0) get all ones and stay last: stable
    const int shift = end_bit > 32 ? end_bit - 32 : 0;
    const uint64_t base = ref & ~((end_bit >= 64) ? ~0ull : ((1ull << end_bit) - 1));
    uint32_t cc[kSelItems], pos[kSelItems];
#pragma unroll
    for (int e = 0; e < kSelItems; ++e) {
        const int i = e * kSelThreads + tid;
        cc[e] = i < count ? (uint32_t)((ks[e] - base) >> shift) : 0xffffffffu;
        pos[e] = (uint32_t)i;
    }
    SelXchg(sm.t.xchg).StripedToBlocked(cc, cc);  // index order == blocked order for the sort
    __syncthreads();
    SelXchg(sm.t.xchg).StripedToBlocked(pos, pos);
    __syncthreads();
    SelSortC(sm.t.coarse).SortBlockedToStriped(cc, pos, 0, end_bit - shift);  // rank e * 512 + tid
    // exact unless coarse-equal neighbours are out of full-key order (stable sort: equal full
    // keys keep index order)
    auto out_of_order = [&](uint32_t ca, uint32_t pa, uint32_t cb, uint32_t pb) {  // a before b
        return shift > 0 && ca == cb && sm.key[pb] < sm.key[pa];
    };
    bool bad = false;
    if (lane == 31) {
#pragma unroll
        for (int e = 0; e < kSelItems; ++e) {
            sm.edge_c[e][warp] = cc[e];
            sm.edge_p[e][warp] = pos[e];
        }
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < kSelItems; ++e) {
        const uint32_t pc = __shfl_up_sync(0xffffffffu, cc[e], 1), pp = __shfl_up_sync(0xffffffffu, pos[e], 1);
        if (lane > 0) {
            bad |= out_of_order(pc, pp, cc[e], pos[e]);
        } else if (warp > 0) {
            bad |= out_of_order(sm.edge_c[e][warp - 1], sm.edge_p[e][warp - 1], cc[e], pos[e]);
        } else if (e > 0) {  // rank e*512 follows rank (e-1)*512 + 511
            bad |= out_of_order(sm.edge_c[e - 1][kSelThreads / 32 - 1], sm.edge_p[e - 1][kSelThreads / 32 - 1], cc[e],
                                pos[e]);
        }
    }
    if (__syncthreads_or(bad)) {  // rare: full 64-bit sort
        uint64_t ck[kSelItems];
        uint32_t ci[kSelItems];
#pragma unroll
        for (int e = 0; e < kSelItems; ++e) {
            const int i = tid * kSelItems + e;
            ck[e] = sm.key[i];
            ci[e] = sm.idx[i];
        }
        __syncthreads();
        SelSort(sm.t.full).SortBlockedToStriped(ck, ci, 0, end_bit);
#pragma unroll
        for (int e = 0; e < kSelItems; ++e) {
            const int64_t r = (int64_t)e * kSelThreads + tid;
            if (r < tt) out[r] = (int32_t)ci[e];
        }
        return;
    }
#pragma unroll
    for (int e = 0; e < kSelItems; ++e) {
        const int64_t r = (int64_t)e * kSelThreads + tid;
        if (r < tt) out[r] = (int32_t)sm.idx[pos[e]];
    }
}

#include "plan_tc.cuh"

struct PlanWs {
    float* guide;      // [Z*Hkv*D]
    float* q_mean;     // [Z*Hq*N*D]
    int64_t* cum_q;    // [N+1]
    int64_t* cum_kv;   // [N+1]
    uint64_t* key0;    // [max_total]
    uint64_t* key1;
    uint32_t* idx0;
    uint32_t* idx1;
    int32_t* ccount;   // [Z*Hq*N] top-T candidate counts (candidates live in key1 / idx1)
    // candidate-pruned selection (plan_tc.cuh)
    float* thr;        // [Z*Hq*N]
    float* ec;         // [Z*Hq*N]
    uint64_t* kth;     // [Z*Hq*N]
    int32_t* ccnt;     // [Z*Hq*N][nch]
    int32_t* full;     // 1: key0 holds every exact prefix-key score (plan levels need them)
    uint8_t* scored;   // [Z*Hq*N] 1: key0 holds every exact prefix-key score of that segment
};

int64_t cand_chunks(const Geo& g) { return std::max<int64_t>(1, ((g.N - 1) * g.S + kCR - 1) / kCR); }

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

size_t plan_ws_layout(const Geo& g, char* base, PlanWs* out) {
    const int64_t zhq = g.z * g.hq;
    const int64_t total = std::max<int64_t>(zhq * g.N * g.S, zhq * g.kv_per_head());
    size_t off = 0;
    auto take = [&](size_t bytes) {
        char* p = base ? base + off : nullptr;
        off += align_up(bytes);
        return p;
    };
    PlanWs ws;
    ws.guide = reinterpret_cast<float*>(take(sizeof(float) * g.z * g.hkv * g.d));
    ws.q_mean = reinterpret_cast<float*>(take(sizeof(float) * zhq * g.N * g.d));
    ws.cum_q = reinterpret_cast<int64_t*>(take(sizeof(int64_t) * (g.N + 1)));
    ws.cum_kv = reinterpret_cast<int64_t*>(take(sizeof(int64_t) * (g.N + 1)));
    ws.key0 = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * total));
    ws.key1 = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * total));
    ws.idx0 = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * total));
    ws.idx1 = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * total));
    ws.ccount = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * zhq * g.N));
    ws.thr = reinterpret_cast<float*>(take(sizeof(float) * zhq * g.N));
    ws.ec = reinterpret_cast<float*>(take(sizeof(float) * zhq * g.N));
    ws.kth = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * zhq * g.N));
    ws.ccnt = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * zhq * g.N * cand_chunks(g)));
    ws.full = reinterpret_cast<int32_t*>(take(2 * sizeof(int32_t)));  // full, dense-gate scratch
    ws.scored = reinterpret_cast<uint8_t*>(take(zhq * g.N));
    if (out) *out = ws;
    return off;
}

int64_t units_per_head(int kind, const Geo& g) {
    int64_t acc = 0;
    for (int64_t n = 0; n < g.N; ++n) {
        const int64_t len = (kind == 0) ? g.seg_rows(n) : n * g.S;
        acc += (len + kRun - 1) / kRun;
    }
    return acc;
}

// Sorts every segment of a family; keys in ws key0; permutation to `perm`.
cudaError_t sort_family(int kind, const Geo& g, PlanWs& ws, int32_t* perm, cudaStream_t st) {
    SortGeo sg;
    sg.kind = kind;
    sg.S = g.S;
    sg.N = g.N;
    sg.last_len = g.last_len;
    sg.heads = g.z * g.hq;
    sg.head_stride = (kind == 0) ? g.N * g.S : g.kv_per_head();
    sg.units_per_head = units_per_head(kind, g);
    sg.cum = (kind == 0) ? ws.cum_q : ws.cum_kv;
    if (sg.units_per_head == 0) return cudaSuccess;
    seg_table_kernel<<<1, 1, 0, st>>>(kind, g.S, g.N, g.last_len, const_cast<int64_t*>(sg.cum));
    int64_t max_len = 0;
    for (int64_t n = 0; n < g.N; ++n)
        max_len = std::max<int64_t>(max_len, (kind == 0) ? g.seg_rows(n) : n * g.S);
    const int64_t units = sg.units_per_head * sg.heads;
    int passes = 0;
    for (int64_t w = kRun; w < max_len; w *= 2) ++passes;
    run_sort_kernel<<<(unsigned)units, kSortThreads, 0, st>>>(sg, ws.key0, ws.key1, ws.idx1,
                                                               passes == 0 ? perm : nullptr);
    uint64_t* ik = ws.key1;
    uint32_t* ii = ws.idx1;
    uint64_t* ok = ws.key0;
    uint32_t* oi = ws.idx0;
    int pass = 0;
    for (int64_t w = kRun; w < max_len; w *= 2, ++pass) {
        const bool last = pass == passes - 1;
        merge_pass_kernel<<<(unsigned)units, kSortThreads, 0, st>>>(sg, w, ik, ii, ok, oi,
                                                                     last ? perm : nullptr);
        std::swap(ik, ok);
        std::swap(ii, oi);
    }
    return cudaGetLastError();
}

}  // namespace

size_t plan_workspace_bytes(const Geo& g) { return plan_ws_layout(g, nullptr, nullptr) + 256; }

namespace {
// Top-T selection of `nseg` segments (all of them, or seg_list) over the keys in ws.key0.
cudaError_t launch_select(const Geo& g, const PlanWs& ws, int64_t nseg, const int32_t* seg_list,
                          const int32_t* prev, int64_t lvl_base, int32_t* kvtop, int64_t topt, int32_t* flags,
                          cudaStream_t st, const int32_t* nseg_dev = nullptr, const int64_t* lvl_base_dev = nullptr,
                          int64_t n_max = INT64_MAX) {
    sel_scan_kernel<<<(unsigned)nseg, kScanThreads, 0, st>>>(g, ws.key0, topt, ws.key1, ws.idx1, ws.ccount, flags,
                                                             seg_list, prev, lvl_base, nseg_dev, lvl_base_dev, n_max);
    const size_t ssm = sizeof(SelSortSmem);
    cudaFuncSetAttribute(sel_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
    sel_sort_kernel<<<(unsigned)nseg, kSelThreads, ssm, st>>>(g, ws.key0, ws.key1, ws.idx1, ws.ccount, topt, kvtop,
                                                              seg_list, prev == nullptr ? 1 : 0, lvl_base, nseg_dev,
                                                              lvl_base_dev);
    return cudaGetLastError();
}
}  // namespace



// Row tiles of kv_cand_kernel: replicate the rows of short prefixes (their candidates per key tile
// scale with 1 / n) so every lane carries a similar load: rep ~ (N - 1) / n, at most 4. False when
// the geometry needs more tiles than CandArgs holds (the caller then uses the dense selection).
bool cand_row_tiles(const Geo& g, int64_t n_cand, CandArgs* ca) {
    ca->ntiles = 0;
    if (g.group > 128) return false;
    // (A/B at C3, kv_cand ms: n * rep <= N - 1, rep <= 4: 1.12; <= 2 (N - 1): 1.44; rep <= 8 with
    // <= 2 (N - 1): 1.36; no replication: 1.21 -- more row tiles cost more K conversion and MMA)
    for (int64_t n = n_cand; n < g.N;) {
        int64_t rep = 4;
        while (rep > 1 && (n * rep > g.N - 1 || g.group * rep > 128)) rep /= 2;
        const int64_t nseg = std::min<int64_t>(std::max<int64_t>(1, 128 / rep / g.group), g.N - n);
        if (ca->ntiles == kCMaxRowTiles) return false;
        ca->tn0[ca->ntiles] = (int32_t)n;
        ca->tnc[ca->ntiles] = (int32_t)nseg;
        ca->trep[ca->ntiles] = (int32_t)rep;
        ++ca->ntiles;
        n += nseg;
    }
    return true;
}

int64_t cand_first_segment(const Geo& g, int64_t topt) {
    const int64_t n_direct = std::min<int64_t>(g.N, kSelCap / g.S + 1);
    return std::min<int64_t>(g.N, std::max<int64_t>(n_direct, (kCandDensity * topt + g.S - 1) / g.S));
}

// The candidate-pruned selection (plan_tc.cuh) serves bf16, D = 128 plans with 128-row-aligned,
// contiguous K rows and S % 128 == 0; S2O_PLAN_TC=0 forces the dense-scoring selection.
bool select_tc_ok(const Geo& g, const void* k, int64_t topt) {
    static const bool on = [] {
        const char* e = std::getenv("S2O_PLAN_TC");
        return !(e && std::strcmp(e, "0") == 0);
    }();
    CandArgs ca;
    return on && kv_score128_ok(g, k) && g.ks[2] == 128 && g.ks[1] % 128 == 0 && g.ks[0] % 128 == 0 &&
           g.S % 128 == 0 && g.N >= 2 && topt <= kSelCap && bf16_row_span(g.ks, g.z, g.hkv, g.l) < (int64_t(1) << 31) &&
           cand_row_tiles(g, cand_first_segment(g, topt), &ca);
}

cudaError_t launch_select_tc(const Geo& g, const void* k, const PlanWs& ws, int32_t* kvtop, int64_t topt,
                             int32_t* flags, cudaStream_t st) {
    cudaError_t err;
    const int64_t zhq = g.z * g.hq;
    // segments n < n_cand: dense exact scores (most of their keys would be candidates anyway);
    // n < n_direct of them (at most kSelCap keys) are sorted whole, the others selected by sel_scan
    const int64_t n_direct = std::min<int64_t>(g.N, kSelCap / g.S + 1);
    const int64_t n_cand = cand_first_segment(g, topt);
    if ((err = cudaMemsetAsync(ws.full, 0, sizeof(int32_t), st)) != cudaSuccess) return err;
    if ((err = cudaMemsetAsync(ws.scored, 0, zhq * g.N, st)) != cudaSuccess) return err;
    if (n_cand >= 2 && (err = launch_kv_score(g, k, ws.q_mean, ws.key0, st, n_cand)) != cudaSuccess) return err;
    if (n_cand < g.N) {
        // step 1: exact scores of every 16th key (a strided view of K), into key1
        Geo gv = g;
        gv.S = g.S / kSampStride;
        gv.l = (g.N - 1) * gv.S;
        gv.ks[2] = g.ks[2] * kSampStride;
        const void* kview = reinterpret_cast<const __nv_bfloat16*>(k) + kSampPhase * g.ks[2];
        if ((err = launch_kv_score(gv, kview, ws.q_mean, ws.key1, st)) != cudaSuccess) return err;
        const unsigned rows = (unsigned)(zhq * (g.N - 1));
        cand_thresh_kernel<<<rows, kThrThreads, 0, st>>>(g, ws.key1, gv.S, ws.q_mean, topt, n_cand, ws.thr, ws.ec, ws.kth);
        if ((err = cudaGetLastError()) != cudaSuccess) return err;
        // step 2: tensor-core candidates + exact rescoring, into the key0 / idx0 row regions
        CUtensorMap kmap;
        if (!make_bf16_row_map(&kmap, k, bf16_row_span(g.ks, g.z, g.hkv, g.l), 128)) return cudaErrorInvalidValue;
        CandArgs ca;
        ca.g = g;
        ca.q_mean = ws.q_mean;
        ca.thr = ws.thr;
        ca.ec = ws.ec;
        ca.ckey = ws.key0;
        ca.cidx = ws.idx0;
        ca.ccnt = ws.ccnt;
        ca.nch = cand_chunks(g);
        if (!cand_row_tiles(g, n_cand, &ca)) return cudaErrorInvalidValue;
        if ((err = set_max_dyn_smem((const void*)kv_cand_kernel, kCSmem)) != cudaSuccess) return err;
        dim3 grid((unsigned)ca.nch, (unsigned)ca.ntiles, (unsigned)(g.z * g.hkv));
        kv_cand_kernel<<<grid, kCThreads, kCSmem, st>>>(ca, kmap);
        if ((err = cudaGetLastError()) != cudaSuccess) return err;
        // step 3: certification + exact first-T compaction, into key1 / idx1 at the row offsets
        cand_pack_kernel<false><<<rows, kPackThreads, 0, st>>>(g, ws.key0, ws.idx0, ws.ccnt, ca.nch, ws.kth, topt,
                                                                n_cand, ws.key1, ws.idx1, ws.ccount, flags);
        if ((err = set_max_dyn_smem((const void*)cand_pack_kernel<true>, sizeof(PackSmem))) != cudaSuccess) return err;
        cand_pack_kernel<true><<<rows, kPackThreads, sizeof(PackSmem), st>>>(g, ws.key0, ws.idx0, ws.ccnt, ca.nch,
                                                                             ws.kth, topt, n_cand, ws.key1, ws.idx1,
                                                                             ws.ccount, flags);
        if ((err = cudaGetLastError()) != cudaSuccess) return err;
    }
    if (n_cand > n_direct)  // the densely scored segments too long to sort whole
        sel_scan_kernel<<<(unsigned)(zhq * (g.N - 1)), kScanThreads, 0, st>>>(
            g, ws.key0, topt, ws.key1, ws.idx1, ws.ccount, flags, nullptr, nullptr, 0, nullptr, nullptr, n_cand);
    // step 4: stable sort of each row's T candidates (or every key of a short segment)
    const size_t ssm = sizeof(SelSortSmem);
    if ((err = set_max_dyn_smem((const void*)sel_sort_kernel, (uint32_t)ssm)) != cudaSuccess) return err;
    sel_sort_kernel<<<(unsigned)(zhq * (g.N - 1)), kSelThreads, ssm, st>>>(g, ws.key0, ws.key1, ws.idx1, ws.ccount, topt,
                                                                          kvtop, nullptr, 1, 0, nullptr, nullptr);
    return cudaGetLastError();
}

// Plan levels read every exact prefix-key score of the segments they serve from key0. After a
// candidate-pruned level 0 those are scored here, stream-ordered (counts in device memory) and only
// when a level is needed:
//  * few listed segments (< kLevelDense): kv_score_rows_kernel, a persistent loop over (segment,
//    256-key block) items of the segments not scored before (~5 us per segment at C3);
//  * many (low tau): kv_score128_kernel over every key once (1.8 ms at C3), then `full` is set and
//    later levels skip both kernels.
constexpr int kLSKeys = 256, kLSThreads = 128, kLevelDense = 320;
__global__ void __launch_bounds__(kLSThreads)
kv_score_rows_kernel(Geo g, const __nv_bfloat16* __restrict__ k, const float* __restrict__ q_mean,
                     uint64_t* __restrict__ kvkey, const int32_t* __restrict__ seg_list,
                     const int32_t* __restrict__ nseg_dev, const uint8_t* __restrict__ scored,
                     const int32_t* __restrict__ full) {
    __shared__ double qs[128];
    if (*full || *nseg_dev >= kLevelDense) return;
    const int64_t nseg = *nseg_dev;
    const int64_t blocks = ((g.N - 1) * g.S + kLSKeys - 1) / kLSKeys;  // of the longest prefix
    for (int64_t w = blockIdx.x; w < nseg * blocks; w += gridDim.x) {
        const int64_t code = seg_list[w / blocks], kb = w % blocks;
        const int64_t zh = code / g.N, n = code % g.N;
        const int64_t t0 = kb * kLSKeys, len = n * g.S;
        if (scored[code] || t0 >= len) continue;  // uniform across the CTA
        __syncthreads();  // previous item's qs readers are done
        if (threadIdx.x < 128) qs[threadIdx.x] = (double)q_mean[code * 128 + threadIdx.x];
        __syncthreads();
        const __nv_bfloat16* kb0 = k + (zh / g.hq) * g.ks[0] + g.kvh(zh) * g.ks[1];
        uint64_t* dst = kvkey + zh * g.kv_per_head() + g.kv_off(n);
        for (int64_t t = t0 + threadIdx.x; t < min(len, t0 + kLSKeys); t += kLSThreads) {
            const uint4* kr = reinterpret_cast<const uint4*>(kb0 + t * g.ks[2]);
            double acc = 0.0;  // dot_f order: d = 0..127 from 0.0 (plan.cpp:14-20)
#pragma unroll 4
            for (int c = 0; c < 16; ++c) {
                const uint4 w4 = kr[c];
                const uint32_t wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    acc = fma(qs[8 * c + 2 * e], (double)__uint_as_float(wv[e] << 16), acc);
                    acc = fma(qs[8 * c + 2 * e + 1], (double)__uint_as_float(wv[e] & 0xffff0000u), acc);
                }
            }
            dst[t] = desc_key(acc);
        }
    }
}

__global__ void level_keys_done_kernel(const int32_t* __restrict__ seg_list, const int32_t* __restrict__ nseg_dev,
                                       uint8_t* __restrict__ scored, int32_t* __restrict__ full) {
    const int64_t nseg = *nseg_dev;
    if (nseg >= kLevelDense) {
        if (blockIdx.x == 0 && threadIdx.x == 0) *full = 1;
        return;
    }
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nseg; i += (int64_t)gridDim.x * blockDim.x)
        scored[seg_list[i]] = 1;
}

__global__ void dense_gate_kernel(const int32_t* __restrict__ nseg_dev, const int32_t* __restrict__ full,
                                  int32_t* __restrict__ skip) {
    *skip = (*full || *nseg_dev < kLevelDense) ? 1 : 0;
}

cudaError_t ensure_level_keys(const Geo& g, const void* k, const PlanWs& ws, const int32_t* seg_list,
                              const int32_t* nseg_dev, cudaStream_t st) {
    if (!kv_score128_ok(g, k)) return cudaSuccess;  // the generic selection always scores everything
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int32_t* skip = ws.full + 1;  // same 256-B slot
    dense_gate_kernel<<<1, 1, 0, st>>>(nseg_dev, ws.full, skip);
    cudaError_t err = launch_kv_score(g, k, ws.q_mean, ws.key0, st, INT64_MAX, skip);
    if (err != cudaSuccess) return err;
    kv_score_rows_kernel<<<sms * 8, kLSThreads, 0, st>>>(g, reinterpret_cast<const __nv_bfloat16*>(k), ws.q_mean,
                                                          ws.key0, seg_list, nseg_dev, ws.scored, ws.full);
    level_keys_done_kernel<<<8, 256, 0, st>>>(seg_list, nseg_dev, ws.scored, ws.full);
    return cudaGetLastError();
}

// Plan for the fused operator: q_perm in full, kv_perm truncated to its top `topt` entries
// per segment, laid out [Z*Hq][N][topt] (segment 0 unused). flags[0] is set if a selection
// could not certify its result (the caller then falls back to the full plan).
cudaError_t launch_plan_topk(const Geo& g, const void* q, const void* k, int32_t* q_perm, int32_t* kvtop,
                             int64_t topt, int32_t* flags, void* workspace, cudaStream_t st) {
    PlanWs ws;
    char* base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255));
    plan_ws_layout(g, base, &ws);
    cudaError_t err;
    if ((err = launch_segment_means(g, k, 1, 1, ws.guide, st)) != cudaSuccess) return err;
    {
        if ((err = launch_q_rank(g, q, ws.guide, ws.q_mean, ws.key0, q_perm, st)) != cudaSuccess) return err;
        if (g.S > kRun && (err = sort_family(0, g, ws, q_perm, st)) != cudaSuccess) return err;
    }
    if (g.N > 1) {
        if (select_tc_ok(g, k, topt)) return launch_select_tc(g, k, ws, kvtop, topt, flags, st);
        if ((err = launch_kv_score(g, k, ws.q_mean, ws.key0, st)) != cudaSuccess) return err;
        if (kv_score128_ok(g, k)) set_flag_kernel<<<1, 1, 0, st>>>(ws.full, 1);
        if ((err = launch_select(g, ws, g.z * g.hq * (g.N - 1), nullptr, nullptr, 0, kvtop, topt, flags, st)) !=
            cudaSuccess)
            return err;
    }
    return cudaSuccess;
}


cudaError_t launch_plan_level_dev(const Geo& g, const void* k, const int32_t* seg_list, const int32_t* nseg_dev,
                                  const int32_t* prev, const int64_t* lvl_base_dev, int32_t* kvtop, int64_t topt,
                                  int32_t* flags, void* workspace, cudaStream_t st) {
    const int64_t nmax = g.z * g.hq * (g.N - 1);
    if (nmax <= 0) return cudaSuccess;
    PlanWs ws;
    char* base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255));
    plan_ws_layout(g, base, &ws);
    cudaError_t err = ensure_level_keys(g, k, ws, seg_list, nseg_dev, st);
    if (err != cudaSuccess) return err;
    return launch_select(g, ws, nmax, seg_list, prev, 0, kvtop, topt, flags, st, nseg_dev, lvl_base_dev);
}

cudaError_t launch_segment_means(const Geo& g, const void* x, int which_kv, int64_t nseg_out,
                                 float* out, cudaStream_t st) {
    const int64_t heads = which_kv ? g.hkv : g.hq;
    const int64_t* s = which_kv ? g.ks : g.qs;
    if (g.in_bf16 && g.d == 128 && s[0] % 8 == 0 && s[1] % 8 == 0 && s[2] % 8 == 0 &&
        (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
        const size_t smem = sizeof(uint32_t) * 2 * kQF_Rows * kQF_W;
        cudaFuncSetAttribute(seg_mean128_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        dim3 grid((unsigned)(g.z * heads), (unsigned)nseg_out);
        seg_mean128_kernel<<<grid, kQF_Threads, smem, st>>>(reinterpret_cast<const __nv_bfloat16*>(x), heads, s[0],
                                                            s[1], s[2], g.S, g.N, g.last_len, nseg_out, out);
        return cudaGetLastError();
    }
    const int threads = (int)std::min<int64_t>(128, g.d);
    dim3 grid((unsigned)((g.d + threads - 1) / threads), (unsigned)(g.z * heads),
              (unsigned)nseg_out);
    seg_mean_kernel<<<grid, threads, 0, st>>>(x, g.in_bf16, heads, s[0], s[1], s[2], g.d, g.S, g.N,
                                              g.last_len, nseg_out, out);
    return cudaGetLastError();
}

// rank_queries (plan.cpp:69-101) with a caller-given guide per (z, q head) [Z, Hq, D] fp32: the q
// ranking kernels index the guide per kv head, so run them on a view with one kv head per q head.
cudaError_t launch_rank_queries(const Geo& g, const void* q, const float* guide, int32_t* q_perm, void* workspace,
                                cudaStream_t st) {
    PlanWs ws;
    char* base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255));
    plan_ws_layout(g, base, &ws);
    Geo gq = g;
    gq.hkv = g.hq;
    gq.group = 1;
    cudaError_t err;
    if ((err = launch_q_rank(gq, q, guide, ws.q_mean, ws.key0, q_perm, st)) != cudaSuccess) return err;
    if (g.S > kRun && (err = sort_family(0, gq, ws, q_perm, st)) != cudaSuccess) return err;
    return cudaSuccess;
}

// rank_prefix_keys (plan.cpp:103-138) with caller-given segment representatives q_mean [Z, Hq, N, D].
cudaError_t launch_rank_prefix_keys(const Geo& g, const void* k, const float* q_mean, int32_t* kv_perm,
                                    void* workspace, cudaStream_t st) {
    if (g.N < 2) return cudaSuccess;
    PlanWs ws;
    char* base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255));
    plan_ws_layout(g, base, &ws);
    cudaError_t err;
    if ((err = launch_kv_score(g, k, q_mean, ws.key0, st)) != cudaSuccess) return err;
    return sort_family(1, g, ws, kv_perm, st);
}

cudaError_t launch_plan_build(const Geo& g, const void* q, const void* k, int32_t* q_perm,
                              int32_t* kv_perm, void* workspace, cudaStream_t st) {
    PlanWs ws;
    char* base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255));
    plan_ws_layout(g, base, &ws);
    cudaError_t err;
    // guide = k_mean[segment 0] of each kv head
    if ((err = launch_segment_means(g, k, 1, 1, ws.guide, st)) != cudaSuccess) return err;
    // q_mean + q keys (+ in-CTA sort when a segment fits one run)
    {
        if ((err = launch_q_rank(g, q, ws.guide, ws.q_mean, ws.key0, q_perm, st)) != cudaSuccess) return err;
        if (g.S > kRun && (err = sort_family(0, g, ws, q_perm, st)) != cudaSuccess) return err;
    }
    if (g.N > 1) {
        if ((err = launch_kv_score(g, k, ws.q_mean, ws.key0, st)) != cudaSuccess) return err;
        if ((err = sort_family(1, g, ws, kv_perm, st)) != cudaSuccess) return err;
    }
    return cudaSuccess;
}

}  // namespace s2o
