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
#include "common.cuh"
#include "internal.h"

namespace s2o {

namespace {

constexpr int kRun = 2048;         // run length == merge tile
constexpr int kSortThreads = 256;  // kRun / 8
constexpr int kScoreKeys = 128;    // keys per kv_score CTA
constexpr int kBatch = 8;          // (q head, segment) accumulators per thread
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
// One CTA per (zh, n). Streams the segment's rows through smem; threads < D
// accumulate column sums in row order (q_mean), threads < kQRows score one
// staged row each against the fp64 guide (sequential over d).
__global__ void q_rank_kernel(const void* __restrict__ q, Geo g, const float* __restrict__ guide,
                              float* __restrict__ q_mean, uint64_t* __restrict__ qkey) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int64_t d = g.d;
    double* gd = reinterpret_cast<double*>(smem_raw);                 // [d]
    float* rows = reinterpret_cast<float*>(gd + d);                   // [kQRows][d+1]
    const int64_t zh = blockIdx.x / g.N;
    const int64_t n = blockIdx.x % g.N;
    const int64_t len = g.seg_rows(n);
    const int64_t z = zh / g.hq;
    const int64_t kvh = g.kvh(zh);
    const float* gsrc = guide + (z * g.hkv + kvh) * d;
    for (int64_t i = threadIdx.x; i < d; i += blockDim.x) gd[i] = (double)gsrc[i];
    const int64_t qb = g.q_base(zh);
    const int64_t rs = d + 1;
    double col_acc[4] = {0.0, 0.0, 0.0, 0.0};  // columns tid, tid+128, ... (d <= 512)
    for (int64_t c0 = 0; c0 < len; c0 += kQRows) {
        const int64_t cn = min((int64_t)kQRows, len - c0);
        __syncthreads();
        for (int64_t e = threadIdx.x; e < cn * d; e += blockDim.x) {
            const int64_t r = e / d, c = e % d;
            rows[r * rs + c] = ld_in(q, qb + (n * g.S + c0 + r) * g.qs[2] + c, g.in_bf16);
        }
        __syncthreads();
        for (int j = 0; j < 4; ++j) {
            const int64_t c = threadIdx.x + (int64_t)j * blockDim.x;
            if (c < d) {
                double a = col_acc[j];
                for (int64_t r = 0; r < cn; ++r) a += (double)rows[r * rs + c];
                col_acc[j] = a;
            }
        }
        if (threadIdx.x < cn) {
            const float* row = rows + threadIdx.x * rs;
            double acc = 0.0;
            for (int64_t c = 0; c < d; ++c) acc = fma((double)row[c], gd[c], acc);
            qkey[zh * g.l + n * g.S + c0 + threadIdx.x] = desc_key(acc);
        }
    }
    const double inv = 1.0 / (double)len;
    for (int j = 0; j < 4; ++j) {
        const int64_t c = threadIdx.x + (int64_t)j * blockDim.x;
        if (c < d) q_mean[(zh * g.N + n) * d + c] = (float)(col_acc[j] * inv);
    }
}

// ---------------------------------------------------------------- kv scoring
// One CTA per (z, kv head, block of 128 keys). Thread t owns key t0 + t.
// For every q head h of the kv group and every segment n whose prefix covers
// the key, s = sum_d q_mean[h,n,d] * K[t,d] in fp64, sequential in d.
__global__ void __launch_bounds__(kScoreKeys)
kv_score_kernel(const void* __restrict__ k, Geo g, const float* __restrict__ q_mean,
                uint64_t* __restrict__ kvkey) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int64_t d = g.d;
    double* qm = reinterpret_cast<double*>(smem_raw);  // [d][kBatch]
    float* kt = reinterpret_cast<float*>(qm + d * kBatch);  // [d][kScoreKeys]
    const int64_t zg = blockIdx.y;  // z * hkv + kvh
    const int64_t z = zg / g.hkv, kvh = zg % g.hkv;
    const int64_t t0 = (int64_t)blockIdx.x * kScoreKeys;
    const int64_t t = t0 + threadIdx.x;
    const int64_t kb = z * g.ks[0] + kvh * g.ks[1];
    // stage K block transposed: kt[c][key]
    for (int64_t e = threadIdx.x; e < (int64_t)kScoreKeys * d; e += blockDim.x) {
        const int64_t r = e / d, c = e % d;
        const int64_t row = t0 + r;
        kt[c * kScoreKeys + r] = (row < g.l) ? ld_in(k, kb + row * g.ks[2] + c, g.in_bf16) : 0.0f;
    }
    const int64_t n_lo = t0 / g.S + 1;  // first segment whose prefix reaches t0
    const int64_t nsegs = (n_lo < g.N) ? g.N - n_lo : 0;
    const int64_t pairs = g.group * nsegs;
    for (int64_t p0 = 0; p0 < pairs; p0 += kBatch) {
        __syncthreads();
        for (int64_t e = threadIdx.x; e < (int64_t)kBatch * d; e += blockDim.x) {
            const int64_t b = e / d, c = e % d;
            const int64_t p = p0 + b;
            double val = 0.0;
            if (p < pairs) {
                const int64_t h = kvh * g.group + p / nsegs;
                const int64_t n = n_lo + p % nsegs;
                val = (double)q_mean[((z * g.hq + h) * g.N + n) * d + c];
            }
            qm[c * kBatch + b] = val;
        }
        __syncthreads();
        double acc[kBatch];
#pragma unroll
        for (int b = 0; b < kBatch; ++b) acc[b] = 0.0;
        for (int64_t c = 0; c < d; ++c) {
            const double kd = (double)kt[c * kScoreKeys + threadIdx.x];
            const double2* q2 = reinterpret_cast<const double2*>(qm + c * kBatch);
#pragma unroll
            for (int b = 0; b < kBatch / 2; ++b) {
                const double2 qq = q2[b];
                acc[2 * b] = fma(qq.x, kd, acc[2 * b]);
                acc[2 * b + 1] = fma(qq.y, kd, acc[2 * b + 1]);
            }
        }
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
            const int64_t p = p0 + b;
            if (p >= pairs) break;
            const int64_t h = kvh * g.group + p / nsegs;
            const int64_t n = n_lo + p % nsegs;
            if (t < n * g.S) {
                const int64_t zh = z * g.hq + h;
                kvkey[zh * g.kv_per_head() + g.kv_off(n) + t] = desc_key(acc[b]);
            }
        }
    }
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
    __shared__ uint64_t sk[kRun];
    __shared__ uint32_t si[kRun];
    int64_t zh, n, j;
    locate(sg, blockIdx.x, zh, n, j);
    const int64_t len = sg.len(n);
    const int64_t r0 = j * kRun;
    const int64_t cnt = min((int64_t)kRun, len - r0);
    const int64_t base = zh * sg.head_stride + sg.off(n);
    for (int i = threadIdx.x; i < kRun; i += kSortThreads) {
        if (i < cnt) {
            sk[i] = keys[base + r0 + i];
            si[i] = (uint32_t)(r0 + i);
        } else {
            sk[i] = ~0ull;
            si[i] = 0xffffffffu;
        }
    }
    __syncthreads();
    for (int kk = 2; kk <= kRun; kk <<= 1) {
        for (int jj = kk >> 1; jj > 0; jj >>= 1) {
            for (int i = threadIdx.x; i < kRun; i += kSortThreads) {
                const int ixj = i ^ jj;
                if (ixj > i) {
                    const bool up = (i & kk) == 0;
                    const uint64_t a = sk[i], b = sk[ixj];
                    const uint32_t ia = si[i], ib = si[ixj];
                    const bool b_less = elt_less(b, ib, a, ia);
                    if (b_less == up) {
                        sk[i] = b; sk[ixj] = a;
                        si[i] = ib; si[ixj] = ia;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < cnt; i += kSortThreads) {
        if (final_out) {
            final_out[base + r0 + i] = (int32_t)si[i];
        } else {
            okeys[base + r0 + i] = sk[i];
            oidx[base + r0 + i] = si[i];
        }
    }
}

// Merges sorted runs of width w pairwise; CTA = one 2048-output tile.
__global__ void __launch_bounds__(kSortThreads)
merge_pass_kernel(SortGeo sg, int64_t w, const uint64_t* __restrict__ ikeys,
                  const uint32_t* __restrict__ iidx, uint64_t* __restrict__ okeys,
                  uint32_t* __restrict__ oidx, int32_t* __restrict__ final_out) {
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
        // merge path: number of A elements among the first `diag` outputs
        const int64_t diag = threadIdx.x == 0 ? d0 : d1;
        int64_t lo = max((int64_t)0, diag - b_len), hi = min(diag, a_len);
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            const int64_t bj = diag - 1 - mid;
            // A[mid] goes first iff A[mid] < B[bj]
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
    const int64_t out0 = base + o0;
    for (int i = threadIdx.x; i < na + nb; i += kSortThreads) {
        const uint64_t key = sk[i];
        const uint32_t id = si[i];
        int pos;
        if (i < na) {  // rank among B slice: count of B elements < this
            int lo = 0, hi = nb;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (elt_less(sk[na + mid], si[na + mid], key, id)) lo = mid + 1; else hi = mid;
            }
            pos = i + lo;
        } else {
            const int jb = i - na;
            int lo = 0, hi = na;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (elt_less(sk[mid], si[mid], key, id)) lo = mid + 1; else hi = mid;
            }
            pos = jb + lo;
        }
        if (final_out) {
            final_out[out0 + pos] = (int32_t)id;
        } else {
            okeys[out0 + pos] = key;
            oidx[out0 + pos] = id;
        }
    }
}

struct PlanWs {
    float* guide;      // [Z*Hkv*D]
    float* q_mean;     // [Z*Hq*N*D]
    int64_t* cum_q;    // [N+1]
    int64_t* cum_kv;   // [N+1]
    uint64_t* key0;    // [max_total]
    uint64_t* key1;
    uint32_t* idx0;
    uint32_t* idx1;
};

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

size_t plan_ws_layout(const Geo& g, char* base, PlanWs* out) {
    const int64_t zhq = g.z * g.hq;
    const int64_t total = std::max<int64_t>(zhq * g.l, zhq * g.kv_per_head());
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
    sg.head_stride = (kind == 0) ? g.l : g.kv_per_head();
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

cudaError_t launch_segment_means(const Geo& g, const void* x, int which_kv, int64_t nseg_out,
                                 float* out, cudaStream_t st) {
    const int64_t heads = which_kv ? g.hkv : g.hq;
    const int64_t* s = which_kv ? g.ks : g.qs;
    const int threads = (int)std::min<int64_t>(128, g.d);
    dim3 grid((unsigned)((g.d + threads - 1) / threads), (unsigned)(g.z * heads),
              (unsigned)nseg_out);
    seg_mean_kernel<<<grid, threads, 0, st>>>(x, g.in_bf16, heads, s[0], s[1], s[2], g.d, g.S, g.N,
                                              g.last_len, nseg_out, out);
    return cudaGetLastError();
}

cudaError_t launch_plan_build(const Geo& g, const void* q, const void* k, int32_t* q_perm,
                              int32_t* kv_perm, void* workspace, cudaStream_t st) {
    PlanWs ws;
    char* base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255));
    plan_ws_layout(g, base, &ws);
    cudaError_t err;
    // guide = k_mean[segment 0] of each kv head
    if ((err = launch_segment_means(g, k, 1, 1, ws.guide, st)) != cudaSuccess) return err;
    // q_mean + q keys
    {
        const size_t smem = sizeof(double) * g.d + sizeof(float) * kQRows * (g.d + 1);
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(q_rank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        q_rank_kernel<<<(unsigned)(g.z * g.hq * g.N), 128, smem, st>>>(q, g, ws.guide, ws.q_mean,
                                                                      ws.key0);
        if ((err = cudaGetLastError()) != cudaSuccess) return err;
        if ((err = sort_family(0, g, ws, q_perm, st)) != cudaSuccess) return err;
    }
    if (g.N > 1) {
        const size_t smem = sizeof(double) * g.d * kBatch + sizeof(float) * g.d * kScoreKeys;
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(kv_score_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const int64_t keys = (g.N - 1) * g.S;  // tokens that appear in some prefix
        dim3 grid((unsigned)((keys + kScoreKeys - 1) / kScoreKeys), (unsigned)(g.z * g.hkv));
        kv_score_kernel<<<grid, kScoreKeys, smem, st>>>(k, g, ws.q_mean, ws.key0);
        if ((err = cudaGetLastError()) != cudaSuccess) return err;
        if ((err = sort_family(1, g, ws, kv_perm, st)) != cudaSuccess) return err;
    }
    return cudaSuccess;
}

}  // namespace s2o
