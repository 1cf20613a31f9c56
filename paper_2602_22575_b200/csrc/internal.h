// internal.h -- declarations shared between the translation units of libs2o_cuda.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"

namespace s2o {

// Pass modes (bit set).
enum PassMode : int {
    kDiag = 1,      // intra-segment causal scan (segment_causal_tile kernel.cpp:36-71)
    kPrefix = 2,    // ranked prefix traversal with stop (traverse_prefix kernel.cpp:86-122)
    kStateIn = 4,   // resume PassBuffers (kernel.cpp:275-286)
    kStateOut = 8,  // persist PassBuffers (kernel.cpp:206-213)
    kFinal = 16,    // finalize acc/ell and scatter (finalize_rows kernel.cpp:149-162)
};

struct PassArgs {
    Geo g;
    int64_t bm, bn;
    double tau;
    double scale;  // 1/sqrt(D) in fp64 (attention.cpp:47)
    int mode;
    int q_reorder;
    const void* q;
    const void* k;
    const void* v;
    void* o;
    const float* acc_in;
    const float* ell_in;
    const float* m_in;
    float* acc_out;
    float* ell_out;
    float* m_out;
    const int32_t* q_perm;
    const int32_t* kv_perm;
    int32_t* processed;     // [Z*Hq][N][T]
    int64_t* pass2_pairs;   // [Z*Hq]
    int64_t T;              // query tiles per full segment = ceil(S/bm)
    int64_t tiles_per_head; // sum over segments
    int32_t* err_flag;      // device: 1 uninitialized state, 2 uncovered row
    // truncated plan (fused operator): kv_perm laid out [Z*Hq][N][kv_top], 0 = packed full
    int64_t kv_top;
    int32_t* ovf_count;     // tiles that consumed their whole truncated list (next level needed)
    int32_t* ovf_tiles;
    int32_t* ovf_base;      // committed chunks so far of each overflow tile (parallel to ovf_tiles)
    const int32_t* tile_list;  // optional: process only these tiles
    const int32_t* tile_base;  // optional: committed chunks of earlier plan levels per tile-list entry
    int64_t tile_count;
    int64_t lvl_base;       // kv_perm entries of a segment consumed by earlier plan levels
    int no_overflow;        // a short kv list is the whole list (block top-k baseline), no next level
    int32_t* work_ctr;      // pass scratch: dynamic work counter of the tcgen05 pass kernel (zeroed per pass)
    // device-resident level state (stream-ordered plan levels, capi.cu): when set, the kernels
    // read the tile-list length and the level base from device memory instead of tile_count /
    // lvl_base (a launch whose list is empty exits at once)
    const int32_t* tile_count_dev;
    const int64_t* lvl_base_dev;
    // pass-1 on the diagonal tcgen05 kernel: tiles whose diagonal V block holds a non-finite value
    // (a masked future key would leak 0 * NaN through P V) are appended here and rerun exactly
    int32_t* poison_cnt;
    int32_t* poison_list;

    __host__ __device__ int64_t lvl() const {
#ifdef __CUDA_ARCH__
        return lvl_base_dev ? *lvl_base_dev : lvl_base;
#else
        return lvl_base;
#endif
    }
    // entries of segment n's (current level) kv list
    __host__ __device__ int64_t avail(int64_t n) const {
        const int64_t rem = n * g.S - lvl();
        return (kv_top > 0 && kv_top < rem) ? kv_top : rem;
    }
    // the level's list ran out before the segment's prefix did
    __host__ __device__ bool truncated(int64_t n) const { return !no_overflow && lvl() + avail(n) < n * g.S; }
    __host__ __device__ const int32_t* kv_seg(int64_t zh, int64_t n) const {
        return kv_top > 0 ? kv_perm + (zh * g.N + n) * kv_top : kv_perm + zh * g.kv_per_head() + g.kv_off(n);
    }
    __host__ __device__ int64_t num_tiles() const {
#ifdef __CUDA_ARCH__
        if (tile_list && tile_count_dev) return *tile_count_dev;
#endif
        return tile_list ? tile_count : g.z * g.hq * tiles_per_head;
    }
    // host: the largest tile count a launch can see (device-resident lists: every tile)
    int64_t max_tiles() const { return (tile_list && !tile_count_dev) ? tile_count : g.z * g.hq * tiles_per_head; }
    __device__ int64_t tile_at(int64_t i) const { return tile_list ? (int64_t)tile_list[i] : i; }
};

size_t plan_workspace_bytes(const Geo& g);
cudaError_t launch_plan_build(const Geo& g, const void* q, const void* k, int32_t* q_perm,
                              int32_t* kv_perm, void* workspace, cudaStream_t st);
cudaError_t launch_plan_topk(const Geo& g, const void* q, const void* k, int32_t* q_perm, int32_t* kvtop,
                             int64_t topt, int32_t* flags, void* workspace, cudaStream_t st);
// Next plan level: for the segments listed in seg_list (codes zh * N + n, count *nseg_dev), the
// topt entries of kv_perm that follow the last entry of `prev` (entries [lvl_base, lvl_base + topt)
// of the full order, *lvl_base_dev). The grid covers every segment and CTAs beyond *nseg_dev exit
// (stream-ordered plan levels). The first level after a candidate-pruned level 0 scores every
// prefix key once (K is needed for that).
cudaError_t launch_plan_level_dev(const Geo& g, const void* k, const int32_t* seg_list, const int32_t* nseg_dev,
                                  const int32_t* prev, const int64_t* lvl_base_dev, int32_t* kvtop, int64_t topt,
                                  int32_t* flags, void* workspace, cudaStream_t st);
cudaError_t launch_segment_means(const Geo& g, const void* x, int which_kv, int64_t nseg_out,
                                 float* out, cudaStream_t st);
cudaError_t launch_rank_queries(const Geo& g, const void* q, const float* guide, int32_t* q_perm, void* workspace,
                                cudaStream_t st);
cudaError_t launch_rank_prefix_keys(const Geo& g, const void* k, const float* q_mean, int32_t* kv_perm,
                                    void* workspace, cudaStream_t st);

// generic SIMT fp64 path
size_t generic_scratch_bytes(const PassArgs& a);
cudaError_t launch_generic_pass(const PassArgs& a, void* scratch, cudaStream_t st);

// 2-D TMA view of a [.., 128] bf16 tensor as rows of 128 elements (box: box_rows x 64 columns,
// SWIZZLE_128B); `map` is a CUtensorMap. Row span of a strided [z, h, l, 128] tensor in rows.
bool make_bf16_row_map(void* map, const void* base, int64_t rows, uint32_t box_rows);
int64_t bf16_row_span(const int64_t* st, int64_t z, int64_t h, int64_t l);
cudaError_t set_max_dyn_smem(const void* fn, uint32_t bytes);  // once per (kernel, device)

// tcgen05 path (bf16, D = 128, b_m = 128, b_n = 128)
bool tc_supported(const PassArgs& a);
bool tc_diag_used(const PassArgs& a);  // launch_tc_pass takes the diagonal (pass-1) kernel
cudaError_t launch_tc_pass(const PassArgs& a, cudaStream_t st);
cudaError_t launch_poison_scan(const PassArgs& a, cudaStream_t st);  // lists tiles with a non-finite diagonal V block

// block top-k baseline selection (baseline.cu): row stats, block masses, kv token lists
cudaError_t launch_block_topk_select(const Geo& g, const void* q, const void* k, int64_t rows, int64_t cols,
                                     int64_t topk, double* rmax, double* rden, double* mass, int32_t* kvtop,
                                     cudaStream_t st);
cudaError_t launch_add_pairs(int64_t* dst, const int64_t* src, int64_t n, cudaStream_t st);

// trace helpers
cudaError_t launch_trace_init(const PassArgs& a, int64_t* pass1_pairs, cudaStream_t st);

}  // namespace s2o
