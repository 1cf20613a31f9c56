// common.cuh -- shared device helpers for the S2O B200 kernels.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "s2o_cuda.h"

namespace s2o {

// Flattened problem passed to kernels by value.
struct Geo {
    int64_t z, hq, hkv, l, d;
    int64_t group;          // hq / hkv
    int64_t S, N, last_len; // segment layout (plan.hpp:16-29)
    int64_t qs[3], ks[3], vs[3], os[3];
    int32_t in_bf16, out_bf16;

    __host__ __device__ int64_t seg_rows(int64_t n) const { return (n + 1 == N) ? last_len : S; }
    __host__ __device__ int64_t kv_per_head() const { return S * N * (N - 1) / 2; }
    __host__ __device__ int64_t kv_off(int64_t n) const { return S * n * (n - 1) / 2; }
    // q head slice zh = z*hq + h -> element offset of row 0
    __host__ __device__ int64_t q_base(int64_t zh) const { return (zh / hq) * qs[0] + (zh % hq) * qs[1]; }
    __host__ __device__ int64_t o_base(int64_t zh) const { return (zh / hq) * os[0] + (zh % hq) * os[1]; }
    __host__ __device__ int64_t kvh(int64_t zh) const { return (zh % hq) / group; }
    __host__ __device__ int64_t k_base(int64_t zh) const { return (zh / hq) * ks[0] + kvh(zh) * ks[1]; }
    __host__ __device__ int64_t v_base(int64_t zh) const { return (zh / hq) * vs[0] + kvh(zh) * vs[1]; }
};

__device__ __forceinline__ float ld_in(const void* p, int64_t idx, int bf16) {
    if (bf16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[idx]);
    return reinterpret_cast<const float*>(p)[idx];
}

__device__ __forceinline__ void st_out(void* p, int64_t idx, float v, int bf16) {
    if (bf16) reinterpret_cast<__nv_bfloat16*>(p)[idx] = __float2bfloat16_rn(v);
    else reinterpret_cast<float*>(p)[idx] = v;
}

// Order key for argsort_desc_stable (tensor.cpp:43-61): NaN and values below
// lowest(float) map to the sentinel, -0.0 == +0.0; ascending order of the
// returned key == descending order of the score. Ties are broken by index.
__device__ __forceinline__ uint64_t desc_key(double s) {
    const double sentinel = -3.4028234663852886e+38;  // (double)lowest(float)
    if (s != s || s < sentinel) s = sentinel;
    if (s == 0.0) s = 0.0;  // fold -0.0
    uint64_t b = static_cast<uint64_t>(__double_as_longlong(s));
    uint64_t asc = (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
    return ~asc;
}

// std::max(a, b) semantics of the reference: (a < b) ? b : a (NaN b is dropped).
__device__ __forceinline__ double std_max(double a, double b) { return (a < b) ? b : a; }

}  // namespace s2o
