// baseline.cu -- block top-k baseline: block_topk_attention
// (proj/src/baseline.cpp:106-185) on the device.
//
// Per query block, the self block plus the k prefix blocks of largest causal softmax MASS are
// kept, and a masked softmax runs over them. The selection here is exact (fp64, the reference's
// operation order), and the masked attention reuses the S2O passes: with segment = query block
// (S = block_rows = block_cols), pass-1 is exactly the self block, and pass-2 walks a kv list made
// of the selected blocks' tokens with tau = 0 (never stops) and no plan-level overflow.
//
//   bt_row_stats_kernel  per row i: m_i = max_{j<=i} s_ij and den_i = sum_j exp(s_ij - m_i),
//                        s_ij = dot_f(q_i, k_j) / sqrt(D) in fp64 (baseline.cpp:47-64)
//   bt_mass_kernel       mass[qb][kb] = sum_{i in qb} sum_{j in kb} exp(s_ij - m_i) / den_i for the
//                        full prefix blocks kb (k_end <= q_begin), rows then keys ascending, the
//                        reference's accumulation order (baseline.cpp:65-69)
//   bt_select_kernel     per query block: the k best prefix blocks by mass, descending, ties to the
//                        lower block, NaN last (baseline.cpp:74-92), written as token lists
//
// All three are fp64 SIMT (exact ranking parity with the reference): O(L^2 D) fp64 work, a
// tool for matched-sparsity comparisons, not a hot path.
#include <cmath>

#include "internal.h"

namespace s2o {
namespace {

__device__ __forceinline__ double dot_row(const void* q, int64_t qoff, const void* k, int64_t koff, int64_t d,
                                          int bf16) {
    double acc = 0.0;
    for (int64_t c = 0; c < d; ++c) acc = fma((double)ld_in(q, qoff + c, bf16), (double)ld_in(k, koff + c, bf16), acc);
    return acc;
}

__global__ void bt_row_stats_kernel(Geo g, const void* __restrict__ q, const void* __restrict__ k, double scale,
                                    double* __restrict__ rmax, double* __restrict__ rden) {
    const int64_t zh = blockIdx.y;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.l) return;
    const int64_t qo = g.q_base(zh) + i * g.qs[2];
    const int64_t kb = g.k_base(zh);
    double m = -INFINITY;
    for (int64_t j = 0; j <= i; ++j) m = fmax(m, dot_row(q, qo, k, kb + j * g.ks[2], g.d, g.in_bf16) * scale);
    double den = 0.0;
    for (int64_t j = 0; j <= i; ++j) den += exp(dot_row(q, qo, k, kb + j * g.ks[2], g.d, g.in_bf16) * scale - m);
    rmax[zh * g.l + i] = m;
    rden[zh * g.l + i] = den;
}

// CTA per (zh, query block); threads over the full prefix blocks.
__global__ void bt_mass_kernel(Geo g, const void* __restrict__ q, const void* __restrict__ k, double scale,
                               int64_t rows, int64_t cols, int64_t nkb, const double* __restrict__ rmax,
                               const double* __restrict__ rden, double* __restrict__ mass) {
    const int64_t zh = blockIdx.y, qb = blockIdx.x;
    const int64_t qs = qb * rows, qe = min(g.l, qs + rows);
    const int64_t npre = qs / cols;  // blocks with k_end <= q_begin
    const int64_t kbase = g.k_base(zh);
    for (int64_t kb = threadIdx.x; kb < npre; kb += blockDim.x) {
        double acc = 0.0;
        for (int64_t i = qs; i < qe; ++i) {
            const int64_t qo = g.q_base(zh) + i * g.qs[2];
            const double m = rmax[zh * g.l + i], den = rden[zh * g.l + i];
            for (int64_t j = kb * cols; j < (kb + 1) * cols; ++j)
                acc += exp(dot_row(q, qo, k, kbase + j * g.ks[2], g.d, g.in_bf16) * scale - m) / den;
        }
        mass[(zh * ((g.l + rows - 1) / rows) + qb) * nkb + kb] = acc;
    }
}

// Ranking key (baseline.cpp:82-90): mass descending, NaN as -inf, ties to the lower block.
__device__ __forceinline__ bool bt_before(double ma, int64_t a, double mb, int64_t b) {
    if (isnan(ma)) ma = -INFINITY;
    if (isnan(mb)) mb = -INFINITY;
    return ma > mb || (ma == mb && a < b);
}

// Thread per (zh, query block): the first min(k, npre) blocks of the ranking, as token lists in
// the truncated kv layout [zh][N][k * cols] (segment n = query block n).
__global__ void bt_select_kernel(Geo g, int64_t rows, int64_t cols, int64_t nkb, int64_t topk,
                                 const double* __restrict__ mass, int32_t* __restrict__ kvtop) {
    const int64_t nqb = (g.l + rows - 1) / rows;
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= g.z * g.hq * nqb) return;
    const int64_t zh = u / nqb, qb = u % nqb;
    const int64_t npre = (qb * rows) / cols;
    const double* mrow = mass + (zh * nqb + qb) * nkb;
    int32_t* out = kvtop + (zh * g.N + qb) * topk * cols;
    double last_m = INFINITY;
    int64_t last_b = -1;
    const int64_t take = min(topk, npre);
    for (int64_t t = 0; t < take; ++t) {
        double best_m = 0.0;
        int64_t best_b = -1;
        for (int64_t b = 0; b < npre; ++b) {
            const double mb = mrow[b];
            if (!(last_b < 0 || bt_before(last_m, last_b, mb, b))) continue;  // already taken
            if (best_b < 0 || bt_before(mb, b, best_m, best_b)) {
                best_m = mb;
                best_b = b;
            }
        }
        for (int64_t c = 0; c < cols; ++c) out[t * cols + c] = (int32_t)(best_b * cols + c);
        last_m = best_m;
        last_b = best_b;
    }
}

__global__ void add_pairs_kernel(int64_t* __restrict__ dst, const int64_t* __restrict__ src, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] += src[i];
}

}  // namespace

cudaError_t launch_add_pairs(int64_t* dst, const int64_t* src, int64_t n, cudaStream_t st) {
    add_pairs_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(dst, src, n);
    return cudaGetLastError();
}

cudaError_t launch_block_topk_select(const Geo& g, const void* q, const void* k, int64_t rows, int64_t cols,
                                     int64_t topk, double* rmax, double* rden, double* mass, int32_t* kvtop,
                                     cudaStream_t st) {
    const double scale = 1.0 / std::sqrt((double)g.d);
    const int64_t zh = g.z * g.hq;
    const int64_t nqb = (g.l + rows - 1) / rows, nkb = (g.l + cols - 1) / cols;
    bt_row_stats_kernel<<<dim3((unsigned)((g.l + 127) / 128), (unsigned)zh), 128, 0, st>>>(g, q, k, scale, rmax, rden);
    bt_mass_kernel<<<dim3((unsigned)nqb, (unsigned)zh), 128, 0, st>>>(g, q, k, scale, rows, cols, nkb, rmax, rden,
                                                                      mass);
    if (topk > 0) {
        const int64_t units = zh * nqb;
        bt_select_kernel<<<(unsigned)((units + 127) / 128), 128, 0, st>>>(g, rows, cols, nkb, topk, mass, kvtop);
    }
    return cudaGetLastError();
}

}  // namespace s2o
