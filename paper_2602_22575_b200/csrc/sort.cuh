// sort.cuh -- stable (key, index) sorting primitives in shared memory.
//
// Elements are (u64 order key, u32 index); the order is lexicographic, which equals the
// reference's std::stable_sort by key (argsort_desc_stable, tensor.cpp:43-61) because the
// index breaks every tie in ascending order. All routines are deterministic.
#pragma once

#include <stdint.h>

namespace s2o {

__device__ __forceinline__ bool kv_less(uint64_t ka, uint32_t ia, uint64_t kb, uint32_t ib) {
    return ka < kb || (ka == kb && ia < ib);
}

// Merge-path split: number of A elements among the first `diag` outputs of merge(A, B).
__device__ __forceinline__ int merge_path(const uint64_t* ak, const uint32_t* ai, int na,
                                          const uint64_t* bk, const uint32_t* bi, int nb, int diag) {
    int lo = max(0, diag - nb), hi = min(diag, na);
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const int bj = diag - 1 - mid;
        if (kv_less(ak[mid], ai[mid], bk[bj], bi[bj])) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Sequentially merge E outputs starting at (a, b) into registers.
template <int E>
__device__ __forceinline__ void merge_seq(const uint64_t* ak, const uint32_t* ai, int na, const uint64_t* bk,
                                          const uint32_t* bi, int nb, int a, int b, uint64_t (&ok)[E],
                                          uint32_t (&oi)[E]) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const bool take_a = (b >= nb) || (a < na && kv_less(ak[a], ai[a], bk[b], bi[b]));
        if (take_a) {
            ok[e] = ak[a];
            oi[e] = ai[a];
            ++a;
        } else {
            ok[e] = bk[b];
            oi[e] = bi[b];
            ++b;
        }
    }
}

// Block-wide merge sort of NT*E elements held in (k0, i0); (k1, i1) is scratch of the same
// size. Every thread of the block must call it. Returns 0 if the sorted result is in
// (k0, i0), 1 if in (k1, i1). Pad unused slots with (~0ull, 0xffffffff).
template <int NT, int E>
__device__ int block_merge_sort(uint64_t* k0, uint32_t* i0, uint64_t* k1, uint32_t* i1) {
    constexpr int N = NT * E;
    const int t = threadIdx.x;
    {
        uint64_t k[E];
        uint32_t id[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            k[e] = k0[t * E + e];
            id[e] = i0[t * E + e];
        }
        // odd-even transposition sort of E registers
#pragma unroll
        for (int round = 0; round < E; ++round) {
#pragma unroll
            for (int e = round & 1; e + 1 < E; e += 2) {
                if (kv_less(k[e + 1], id[e + 1], k[e], id[e])) {
                    const uint64_t tk = k[e];
                    k[e] = k[e + 1];
                    k[e + 1] = tk;
                    const uint32_t ti = id[e];
                    id[e] = id[e + 1];
                    id[e + 1] = ti;
                }
            }
        }
#pragma unroll
        for (int e = 0; e < E; ++e) {
            k0[t * E + e] = k[e];
            i0[t * E + e] = id[e];
        }
    }
    __syncthreads();
    int cur = 0;
    for (int w = E; w < N; w *= 2) {
        const uint64_t* sk = cur ? k1 : k0;
        const uint32_t* si = cur ? i1 : i0;
        uint64_t* dk = cur ? k0 : k1;
        uint32_t* di = cur ? i0 : i1;
        const int o = t * E;
        const int pb = (o / (2 * w)) * (2 * w);
        const int d = o - pb;
        const int a = merge_path(sk + pb, si + pb, w, sk + pb + w, si + pb + w, w, d);
        uint64_t ok[E];
        uint32_t oi[E];
        merge_seq<E>(sk + pb, si + pb, w, sk + pb + w, si + pb + w, w, a, d - a, ok, oi);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            dk[o + e] = ok[e];
            di[o + e] = oi[e];
        }
        __syncthreads();
        cur ^= 1;
    }
    return cur;
}

}  // namespace s2o
