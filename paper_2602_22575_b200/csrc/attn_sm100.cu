// attn_sm100.cu -- Step 2 of S2O on tcgen05 tensor cores (bf16 in, fp32 accumulate in TMEM).
//
// One persistent kernel serves pass-1 (intra-segment causal scan, segment_causal_tile
// kernel.cpp:36-71), pass-2 (ranked prefix traversal with the monotone-gain stop,
// traverse_prefix kernel.cpp:86-122 + early_stop_check kernel.cpp:220-234) and the fused
// single pass (kernel.cpp:300-349). A work unit is one 128-row query tile; its key stream is
// a list of 128-key blocks: first the causal blocks of its own segment (masked on original
// token positions), then the chunks of kv_perm in rank order (non-contiguous rows).
//
// Warp roles (256 threads, 1 CTA per SM):
//   warps 0-3  softmax/correction/epilogue: thread r owns query row r = TMEM lane r
//   warp 4     MMA issuer (one lane): S = Q K^T into TMEM (double-buffered), O += P V
//   warps 5-7  loaders: contiguous blocks (the causal blocks of pass-1, Q in token order) by
//              2-D tile TMA (4 ops per block); permuted rows (Q by q_perm, prefix chunks by
//              kv_perm) by TMA tile::gather4 spread over the three warps (the gather issue
//              rate, ~1 op per 22 cycles per SM, is the limit; see scripts/load_bench.cu)
//
// Early stop (reference semantics): for a prefix chunk the softmax warps
// compute each row's relative normaliser gain sum_j exp(s_j - m) / ell from the chunk's
// scores alone, reduce the max over the tile's rows, and compare with tau before P V is
// issued; a stopping chunk is discarded (no P V, no state change). QK^T of the next chunk
// is issued speculatively; it is simply dropped when the tile stops.
//
// Data layout in shared memory (all SWIZZLE_128B, 1024-B aligned):
//   sQ   [2][128 rows][128 B]        Q tile, K-major (two 64-column halves)
//   sK   [3 stages][2][128][128 B]   K block, K-major (B operand of Q K^T)
//   sV   [3 stages][2][128][128 B]   V block, used MN-major (B operand of P V)
//   P    = exp2(s - m) in bf16, K-major (A operand of P V), written into the K buffer of the
//          block's own stage: K(j) is dead once Q K^T(j) completed (the softmax only writes P
//          after reading S(j)), and the stage is released only after P V(j) completes.
// TMEM (512 columns): S buffers at columns [0,128) and [128,256), O at [256,384).
#include <cudaTypedefs.h>

#include <cmath>
#include <cstring>
#include <mutex>

#include "internal.h"
#include "sm100.cuh"

namespace s2o {

using namespace sm100;

namespace {

constexpr int kD = 128;
constexpr int kBM = 128;
constexpr int kBN = 128;
constexpr int kStages = 3;
constexpr int kThreads = 256;
constexpr int kLoaderWarps = 3;  // warps 5..7 issue TMA (gather4 issue rate scales with warps)
constexpr uint32_t kHalf = 128u * 128u;            // bytes of one 64-column half tile
constexpr uint32_t kTileBytes = 2 * kHalf;         // 32 KB
constexpr uint32_t kOffQ = 0;
constexpr uint32_t kOffK = kOffQ + kTileBytes;
constexpr uint32_t kOffV = kOffK + kStages * kTileBytes;
constexpr uint32_t kOffCtrl = kOffV + kStages * kTileBytes;
constexpr uint32_t kSmemBytes = kOffCtrl + 2048 + 1024;  // + control block + alignment slack
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColO = 256;
constexpr float kRescaleThresh = 8.0f;  // lazy max update, log2 units (factor 256)

struct Ctrl {
    uint64_t q_full, q_empty;
    uint64_t k_full[kStages], v_full[kStages], kv_empty[kStages];
    uint64_t s_full[2], s_empty[2];
    uint64_t p_full, o_done;
    uint32_t tmem_base;
    float red[4];
    uint8_t dec[4];  // decision ring (block j -> j & 3): 1 = commit, 2 = stop
};

struct TcParams {
    PassArgs a;
    float scale_log2;  // (1/sqrt(D)) * log2(e)
    int q_contig, kv_contig;  // token stride == one row (tile TMA usable)
};

struct TileInfo {
    int64_t zh, n, ti, t0, tn, seg_rows, sb, avail;
    int nd, np, nb;  // diag blocks, prefix blocks, total
};

__device__ __forceinline__ TileInfo tile_info(const PassArgs& a, int64_t tile) {
    const Geo& g = a.g;
    TileInfo t;
    t.zh = tile / a.tiles_per_head;
    const int64_t r_in = tile % a.tiles_per_head;
    const int64_t full = (g.N - 1) * a.T;
    if (r_in < full) { t.n = r_in / a.T; t.ti = r_in % a.T; }
    else { t.n = g.N - 1; t.ti = r_in - full; }
    t.sb = t.n * g.S;
    t.seg_rows = g.seg_rows(t.n);
    t.t0 = t.ti * kBM;
    t.tn = min((int64_t)kBM, t.seg_rows - t.t0);
    t.nd = (a.mode & kDiag) ? (int)((t.t0 + t.tn - 1) / kBN + 1) : 0;
    t.avail = a.avail(t.n);  // kv_perm entries available to walk
    t.np = ((a.mode & kPrefix) && t.n > 0) ? (int)((t.avail + kBN - 1) / kBN) : 0;
    t.nb = t.nd + t.np;
    return t;
}

// Absolute row (in D-element units) of q row `local` of the tile.
__device__ __forceinline__ int64_t q_local_row(const PassArgs& a, const TileInfo& t, int64_t r) {
    if (r >= t.tn) r = 0;  // ragged tail: duplicate a valid row, results discarded
    const int64_t local = ((a.mode & kStateIn) && a.q_reorder)
                              ? (int64_t)a.q_perm[(t.zh * a.g.N + t.n) * a.g.S + t.t0 + r]
                              : t.t0 + r;
    return t.sb + local;
}

// token index of key i of block j (clamped into the block's valid range)
__device__ __forceinline__ int64_t key_token(const PassArgs& a, const TileInfo& t, const int32_t* kv,
                                             int j, int i) {
    if (j < t.nd) {
        const int64_t k0 = (int64_t)j * kBN;
        const int64_t kn = min((int64_t)kBN, t.seg_rows - k0);
        return t.sb + k0 + (i < kn ? i : 0);
    }
    const int64_t c0 = (int64_t)(j - t.nd) * kBN;
    const int64_t cn = min((int64_t)kBN, t.avail - c0);
    return (int64_t)kv[c0 + (i < cn ? i : 0)];
}

__global__ void __launch_bounds__(kThreads, 1)
tc_pass_kernel(const TcParams p, const __grid_constant__ CUtensorMap qmap,
               const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
               const __grid_constant__ CUtensorMap qtile, const __grid_constant__ CUtensorMap ktile,
               const __grid_constant__ CUtensorMap vtile) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Ctrl& c = *reinterpret_cast<Ctrl*>(smem + kOffCtrl);
    const PassArgs& a = p.a;
    const Geo& g = a.g;
    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const uint32_t sQ = smem_u32(smem + kOffQ);
    const uint32_t sK = smem_u32(smem + kOffK);
    const uint32_t sV = smem_u32(smem + kOffV);

    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&c.q_full), 1);
        mbar_init(smem_u32(&c.q_empty), 1);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(smem_u32(&c.k_full[s]), 1);
            mbar_init(smem_u32(&c.v_full[s]), 1);
            mbar_init(smem_u32(&c.kv_empty[s]), 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(smem_u32(&c.s_full[s]), 1);
            mbar_init(smem_u32(&c.s_empty[s]), 4);
        }
        mbar_init(smem_u32(&c.p_full), 4);
        mbar_init(smem_u32(&c.o_done), 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(smem_u32(&c.tmem_base), kTmemCols);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = c.tmem_base;

    const int64_t total_tiles = a.num_tiles();
    const int64_t kv_div = g.d;  // row unit of the tensor maps = D elements

    if (warp >= 5) {
        // ============================== loaders ==============================
        const int lw = warp - 5;             // loader warp 0..2
        const int lt = lw * 32 + lane;       // loader thread 0..95
        const uint32_t lbar = 5 * 32;        // named barrier 2 over the 96 loader threads
        uint32_t gblk = 0, qcount = 0;
        for (int64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
            const TileInfo t = tile_info(a, a.tile_at(tile));
            if (t.nb == 0) continue;
            const int32_t* kv = (t.np > 0) ? a.kv_seg(t.zh, t.n) : nullptr;
            // Q rows; wait until the previous tile's Q K^T are done
            mbar_wait(smem_u32(&c.q_empty), (qcount & 1) ^ 1, 1001);
            const int64_t qb = g.q_base(t.zh) / kv_div;
            const bool q_tile = p.q_contig && !((a.mode & kStateIn) && a.q_reorder) && t.tn == kBM;
            if (lt == 0) mbar_expect_tx(smem_u32(&c.q_full), kTileBytes);
            named_bar_sync(2, 96);
            if (q_tile) {
                if (lt == 0)
                    for (int h = 0; h < 2; ++h)
                        tma_load2d(sQ + h * kHalf, &qtile, h * 64, (int32_t)(qb + t.sb + t.t0), smem_u32(&c.q_full));
            } else {
                for (int op = lt; op < 64; op += 96) {  // 32 row groups x 2 halves
                    const int grp = op >> 1, h = op & 1;
                    int32_t rows[4];
                    for (int i = 0; i < 4; ++i)
                        rows[i] = (int32_t)(qb + q_local_row(a, t, grp * 4 + i) * (g.qs[2] / kv_div));
                    tma_gather4(sQ + h * kHalf + grp * 512, &qmap, h * 64, rows[0], rows[1], rows[2], rows[3],
                                smem_u32(&c.q_full));
                }
            }
            ++qcount;
            const int64_t kb = g.k_base(t.zh) / kv_div, vb = g.v_base(t.zh) / kv_div;
            const int64_t ks = g.ks[2] / kv_div, vs = g.vs[2] / kv_div;
            int loaded = 0;
            // gather indices for block j live in registers; block j+1's are prefetched while
            // block j is issued (kv_perm reads are L2 round trips)
            auto fetch_rows = [&](int j, int32_t (&rk)[2][4], int32_t (&rv)[2][4]) {
                for (int u = 0; u < 2; ++u) {
                    const int op = lt + u * 96;
                    const int grp = (op >> 1) & 31;
                    for (int i = 0; i < 4; ++i) {
                        const int64_t tok = (j < t.nb) ? key_token(a, t, kv, j, grp * 4 + i) : 0;
                        rk[u][i] = (int32_t)(kb + tok * ks);
                        rv[u][i] = (int32_t)(vb + tok * vs);
                    }
                }
            };
            int32_t ck[2][4], cv[2][4], nk[2][4], nv[2][4];
            fetch_rows(0, ck, cv);
            for (int j = 0; j < t.nb; ++j) {
                const uint32_t gi = gblk + j;
                const int st = gi % kStages;
                if (j + 1 < t.nb && !(j + 1 < t.nd && p.kv_contig)) fetch_rows(j + 1, nk, nv);
                mbar_wait(smem_u32(&c.kv_empty[st]), ((gi / kStages) & 1) ^ 1, 1002);
                // acquiring stage j implies block j-kStages was decided; a stop there ends the tile
                if (j >= kStages && c.dec[(j - kStages) & 3] == 2) break;
                if (lt == 0) {
                    mbar_expect_tx(smem_u32(&c.k_full[st]), kTileBytes);
                    mbar_expect_tx(smem_u32(&c.v_full[st]), kTileBytes);
                }
                named_bar_sync(2, 96);
                const uint32_t kdst = sK + st * kTileBytes;
                const uint32_t vdst = sV + st * kTileBytes;
                if (j < t.nd && p.kv_contig) {
                    if (lt == 0) {
                        const int64_t tok = t.sb + (int64_t)j * kBN;
                        for (int h = 0; h < 2; ++h)
                            tma_load2d(kdst + h * kHalf, &ktile, h * 64, (int32_t)(kb + tok), smem_u32(&c.k_full[st]));
                        for (int h = 0; h < 2; ++h)
                            tma_load2d(vdst + h * kHalf, &vtile, h * 64, (int32_t)(vb + tok), smem_u32(&c.v_full[st]));
                    }
                } else {
                    // K first (Q K^T waits only for K), then V: 64 ops each, lt < 64 -> op 0/1
                    for (int u = 0; u < 2; ++u) {
                        const int op = lt + u * 96;  // ops [0,64): K, [64,128): V; op>>1 = group
                        if (op >= 128) break;
                        const int grp = (op >> 1) & 31, h = op & 1;
                        const bool isv = op >= 64;
                        tma_gather4((isv ? vdst : kdst) + h * kHalf + grp * 512, isv ? &vmap : &kmap, h * 64,
                                    isv ? cv[u][0] : ck[u][0], isv ? cv[u][1] : ck[u][1],
                                    isv ? cv[u][2] : ck[u][2], isv ? cv[u][3] : ck[u][3],
                                    smem_u32(isv ? &c.v_full[st] : &c.k_full[st]));
                    }
                }
                for (int u = 0; u < 2; ++u)
                    for (int i = 0; i < 4; ++i) {
                        ck[u][i] = nk[u][i];
                        cv[u][i] = nv[u][i];
                    }
                ++loaded;
            }
            gblk += loaded;
        }
    } else if (warp == 4) {
        // ============================== MMA issuer ==============================
        const uint32_t idesc_s = umma_idesc_bf16(kBM, kBN, false, false);
        const uint32_t idesc_o = umma_idesc_bf16(kBM, kD, false, true);
        uint32_t gblk = 0, gq = 0, qcount = 0, gp = 0;  // loads, Q K^T (S buffer uses), p_full
        for (int64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
            const TileInfo t = tile_info(a, a.tile_at(tile));
            if (t.nb == 0) continue;
            if (lane == 0) {
                mbar_wait(smem_u32(&c.q_full), qcount & 1, 2001);
                tc_fence_after();
            }
            ++qcount;
            int stop_at = -1;
            auto issue_qk = [&](int j) {
                const uint32_t gi = gblk + j;
                const uint32_t gs = gq + j;  // S buffer sequence (loads may run further ahead)
                const int st = gi % kStages;
                const int sb = gs & 1;
                mbar_wait(smem_u32(&c.k_full[st]), (gi / kStages) & 1, 2002);
                mbar_wait(smem_u32(&c.s_empty[sb]), ((gs >> 1) & 1) ^ 1, 2003);
                tc_fence_after();
                const uint32_t kbase = sK + st * kTileBytes;
                for (int kk = 0; kk < kD / 16; ++kk) {
                    const uint32_t off = (kk / 4) * kHalf + (kk % 4) * 32;
                    umma_bf16(tbase + sb * 128, umma_desc_sw128(sQ + off, 16, 1024),
                              umma_desc_sw128(kbase + off, 16, 1024), idesc_s, kk > 0);
                }
                umma_commit(smem_u32(&c.s_full[sb]));
            };
            if (lane == 0) {
                issue_qk(0);
                for (int j = 0; j < t.nb; ++j) {
                    if (j + 1 < t.nb) issue_qk(j + 1);
                    // decision for block j
                    mbar_wait(smem_u32(&c.p_full), gp & 1, 2004);
                    ++gp;
                    tc_fence_after();
                    const uint32_t gi = gblk + j;
                    const int st = gi % kStages;
                    if (c.dec[j & 3] == 1) {
                        mbar_wait(smem_u32(&c.v_full[st]), (gi / kStages) & 1, 2005);
                        tc_fence_after();
                        const uint32_t vbase = sV + st * kTileBytes;
                        const uint32_t pbase = sK + st * kTileBytes;  // P aliases K(j)
                        for (int kk = 0; kk < kBN / 16; ++kk) {
                            const uint32_t aoff = (kk / 4) * kHalf + (kk % 4) * 32;
                            umma_bf16(tbase + kColO, umma_desc_sw128(pbase + aoff, 16, 1024),
                                      umma_desc_sw128(vbase + kk * 16 * 128, kHalf, 1024), idesc_o, 1);
                        }
                        umma_commit(smem_u32(&c.kv_empty[st]));
                        umma_commit(smem_u32(&c.o_done));
                        if (j + 1 == t.nb) umma_commit(smem_u32(&c.q_empty));
                    } else {
                        // stop: no P V, no o_done completion (the softmax drained P V(j-1)
                        // before publishing this decision, so barrier phases never run
                        // two ahead of their waiters)
                        stop_at = j;
                        mbar_wait(smem_u32(&c.v_full[st]), (gi / kStages) & 1, 2006);
                        mbar_arrive(smem_u32(&c.kv_empty[st]));
                        if (j + 1 < t.nb) {
                            // Q K^T of block j+1 was issued speculatively: its V must land before
                            // the stage is freed (v_full phase accounting), then free it once done
                            const uint32_t g1 = gi + 1;
                            mbar_wait(smem_u32(&c.v_full[g1 % kStages]), (g1 / kStages) & 1, 2007);
                            umma_commit(smem_u32(&c.kv_empty[g1 % kStages]));
                        }
                        // blocks j+2 .. j+kStages-1 were loaded (the loader runs kStages ahead of
                        // the decisions) but never computed: consume and free them
                        for (int jj = j + 2; jj < min(t.nb, j + kStages); ++jj) {
                            const uint32_t g2 = gblk + jj;
                            mbar_wait(smem_u32(&c.k_full[g2 % kStages]), (g2 / kStages) & 1, 2008);
                            mbar_wait(smem_u32(&c.v_full[g2 % kStages]), (g2 / kStages) & 1, 2009);
                            mbar_arrive(smem_u32(&c.kv_empty[g2 % kStages]));
                        }
                        umma_commit(smem_u32(&c.q_empty));
                        break;
                    }
                }
            }
            __syncwarp();
            stop_at = __shfl_sync(0xffffffffu, stop_at, 0);
            gblk += (stop_at >= 0) ? min(t.nb, stop_at + kStages) : t.nb;
            gq += (stop_at >= 0) ? min(t.nb, stop_at + 2) : t.nb;
        }
    } else {
        // ============================== softmax / epilogue ==============================
        const int r = threadIdx.x;  // 0..127, TMEM lane
        const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
        uint32_t gblk = 0, gq = 0, gp = 0, od = 0;
        for (int64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
            const TileInfo t = tile_info(a, a.tile_at(tile));
            const bool valid = r < t.tn;
            const int64_t grow = q_local_row(a, t, r);  // segment row in [0, L)
            const int64_t slot = t.zh * g.l + grow;
            float m2, ell;
            // ---- state init: O in TMEM, (m, ell) in registers
            if (a.mode & kStateIn) {
                m2 = a.m_in[slot] * 1.4426950408889634f;
                ell = a.ell_in[slot];
                const float4* src = reinterpret_cast<const float4*>(a.acc_in + slot * kD);
                for (int c0 = 0; c0 < kD; c0 += 32) {
                    uint32_t v[32];
                    for (int i = 0; i < 8; ++i) {
                        const float4 x = src[c0 / 4 + i];
                        v[4 * i] = __float_as_uint(x.x);
                        v[4 * i + 1] = __float_as_uint(x.y);
                        v[4 * i + 2] = __float_as_uint(x.z);
                        v[4 * i + 3] = __float_as_uint(x.w);
                    }
                    tmem_st32(tbase + lane_off + kColO + c0, v);
                }
            } else {
                m2 = -INFINITY;
                ell = 0.0f;
                uint32_t z[32];
                for (int i = 0; i < 32; ++i) z[i] = 0u;
                for (int c0 = 0; c0 < kD; c0 += 32) tmem_st32(tbase + lane_off + kColO + c0, z);
            }
            tmem_st_wait();
            tc_fence_before();

            int committed = 0;
            int64_t pairs = 0;
            bool stopped = false;
            int stop_j = -1;
            for (int j = 0; j < t.nb; ++j) {
                const uint32_t gi = gblk + j;  // load sequence (K stage holding P)
                const uint32_t gs = gq + j;    // S buffer sequence
                const int sb = gs & 1;
                mbar_wait(smem_u32(&c.s_full[sb]), (gs >> 1) & 1, 3001);
                tc_fence_after();
                uint32_t sv[kBN];
                {
                    uint32_t (&v0)[32] = *reinterpret_cast<uint32_t(*)[32]>(&sv[0]);
                    uint32_t (&v1)[32] = *reinterpret_cast<uint32_t(*)[32]>(&sv[32]);
                    uint32_t (&v2)[32] = *reinterpret_cast<uint32_t(*)[32]>(&sv[64]);
                    uint32_t (&v3)[32] = *reinterpret_cast<uint32_t(*)[32]>(&sv[96]);
                    const uint32_t sa = tbase + lane_off + sb * 128;
                    tmem_ld32(sa, v0);
                    tmem_ld32(sa + 32, v1);
                    tmem_ld32(sa + 64, v2);
                    tmem_ld32(sa + 96, v3);
                    tmem_ld_wait();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&c.s_empty[sb]));
                float* s = reinterpret_cast<float*>(sv);
                // ---- masks: causal on original positions (diag) / clipped chunk (prefix)
                const bool is_diag = j < t.nd;
                int lim;  // keys [0, lim) of the block are visible to this row
                if (is_diag) {
                    const int64_t k0 = (int64_t)j * kBN;
                    const int64_t kn = min((int64_t)kBN, t.seg_rows - k0);
                    const int64_t vis = (k0 + kn - 1 <= t.t0) ? kn : min(kn, t.t0 + r - k0 + 1);
                    lim = (int)max((int64_t)0, vis);
                } else {
                    const int64_t c0 = (int64_t)(j - t.nd) * kBN;
                    lim = (int)min((int64_t)kBN, t.avail - c0);
                }
                if (lim < kBN) {
#pragma unroll
                    for (int i = 0; i < kBN; ++i)
                        if (i >= lim) s[i] = -INFINITY;
                }
                float mxa[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) mxa[u] = s[u];
#pragma unroll
                for (int i = 8; i < kBN; i += 8)
#pragma unroll
                    for (int u = 0; u < 8; ++u) mxa[u] = fmaxf(mxa[u], s[i + u]);
                const float mx = fmaxf(fmaxf(fmaxf(mxa[0], mxa[1]), fmaxf(mxa[2], mxa[3])),
                                       fmaxf(fmaxf(mxa[4], mxa[5]), fmaxf(mxa[6], mxa[7]))) * p.scale_log2;
                const float m_new = fmaxf(m2, mx);
                const bool rescale = (m_new > m2 + kRescaleThresh) || (m2 == -INFINITY);
                const float m_use = rescale ? m_new : m2;
                const float neg_ref = (m_use == -INFINITY) ? 0.0f : -m_use;
                float rs[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) rs[u] = 0.0f;
#pragma unroll
                for (int i = 0; i < kBN; i += 8)
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        s[i + u] = ex2(fmaf(s[i + u], p.scale_log2, neg_ref));
                        rs[u] += s[i + u];
                    }
                const float rowsum = ((rs[0] + rs[1]) + (rs[2] + rs[3])) + ((rs[4] + rs[5]) + (rs[6] + rs[7]));
                const float alpha = (m2 == -INFINITY) ? 0.0f : ex2(m2 + neg_ref);
                bool commit = true;
                if (!is_diag) {
                    // relative normaliser gain of this chunk (kernel.cpp:108-115)
                    const float prev = ell * alpha;
                    float gain = valid ? rowsum / prev : -INFINITY;
                    for (int o = 16; o > 0; o >>= 1) gain = fmaxf(gain, __shfl_xor_sync(0xffffffffu, gain, o));
                    if (lane == 0) c.red[warp] = gain;
                    named_bar_sync(1, 128);
                    const float mg = fmaxf(fmaxf(c.red[0], c.red[1]), fmaxf(c.red[2], c.red[3]));
                    commit = !(mg < (float)a.tau);
                    named_bar_sync(1, 128);  // red[] reusable
                }
                ++gp;
                // P V of block j-1 must be complete before this block's decision is published
                // (P buffer / O reuse, and one-phase-at-a-time on o_done and p_full)
                if (j > 0) {
                    mbar_wait(smem_u32(&c.o_done), od & 1, 3003);
                    ++od;
                    tc_fence_after();
                }
                if (!commit) {
                    if (r == 0) c.dec[j & 3] = 2;
                    __syncwarp();
                    if (lane == 0) mbar_arrive(smem_u32(&c.p_full));
                    stopped = true;
                    if (j + 1 < t.nb) {  // drain the speculative Q K^T of block j+1
                        const uint32_t gn = gs + 1;
                        mbar_wait(smem_u32(&c.s_full[gn & 1]), (gn >> 1) & 1, 3002);
                        __syncwarp();
                        if (lane == 0) mbar_arrive(smem_u32(&c.s_empty[gn & 1]));
                    }
                    stop_j = j;
                    break;
                }
                if (__any_sync(0xffffffffu, rescale && m2 != -INFINITY)) {
                    for (int c0 = 0; c0 < kD; c0 += 32) {
                        uint32_t v[32];
                        tmem_ld32(tbase + lane_off + kColO + c0, v);
                        tmem_ld_wait();
                        for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
                        tmem_st32(tbase + lane_off + kColO + c0, v);
                    }
                    tmem_st_wait();
                }
                // P (bf16) -> smem, K-major SW128
                unsigned char* prow = smem + kOffK + (gi % kStages) * kTileBytes + r * 128;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
#pragma unroll
                    for (int ch = 0; ch < 8; ++ch) {
                        const float* x = s + h * 64 + ch * 8;
                        uint4 w;
                        w.x = pack_bf16(x[0], x[1]);
                        w.y = pack_bf16(x[2], x[3]);
                        w.z = pack_bf16(x[4], x[5]);
                        w.w = pack_bf16(x[6], x[7]);
                        *reinterpret_cast<uint4*>(prow + h * kHalf + ((ch ^ (r & 7)) << 4)) = w;
                    }
                }
                ell = ell * alpha + rowsum;
                m2 = m_use;
                if (!is_diag) {
                    ++committed;
                    const int64_t c0 = (int64_t)(j - t.nd) * kBN;
                    pairs += min((int64_t)kBN, t.avail - c0);
                }
                fence_proxy_async_smem();
                tc_fence_before();
                if (r == 0) c.dec[j & 3] = 1;
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&c.p_full));
            }
            // ---- epilogue: the last P V (if the tile ran to completion) must be done
            if (t.nb > 0 && !stopped) {
                mbar_wait(smem_u32(&c.o_done), od & 1, 3004);
                ++od;
                tc_fence_after();
            }
            gblk += (t.nb == 0) ? 0 : (stopped ? min(t.nb, stop_j + kStages) : t.nb);
            gq += (t.nb == 0) ? 0 : (stopped ? min(t.nb, stop_j + 2) : t.nb);
            // ---- read O, finalize / persist
            const float inv = 1.0f / ell;
            for (int c0 = 0; c0 < kD; c0 += 32) {
                uint32_t v[32];
                tmem_ld32(tbase + lane_off + kColO + c0, v);
                tmem_ld_wait();
                if (!valid) continue;
                if (a.mode & kStateOut) {
                    float4* dst = reinterpret_cast<float4*>(a.acc_out + slot * kD + c0);
                    for (int i = 0; i < 8; ++i)
                        dst[i] = make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                             __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
                }
                if (a.mode & kFinal) {
                    const int64_t ooff = g.o_base(t.zh) + grow * g.os[2] + c0;
                    if (g.out_bf16) {
                        uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.o) + ooff);
                        for (int i = 0; i < 4; ++i) {
                            uint4 w;
                            w.x = pack_bf16(__uint_as_float(v[8 * i]) * inv, __uint_as_float(v[8 * i + 1]) * inv);
                            w.y = pack_bf16(__uint_as_float(v[8 * i + 2]) * inv, __uint_as_float(v[8 * i + 3]) * inv);
                            w.z = pack_bf16(__uint_as_float(v[8 * i + 4]) * inv, __uint_as_float(v[8 * i + 5]) * inv);
                            w.w = pack_bf16(__uint_as_float(v[8 * i + 6]) * inv, __uint_as_float(v[8 * i + 7]) * inv);
                            dst[i] = w;
                        }
                    } else {
                        float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(a.o) + ooff);
                        for (int i = 0; i < 8; ++i)
                            dst[i] = make_float4(__uint_as_float(v[4 * i]) * inv, __uint_as_float(v[4 * i + 1]) * inv,
                                                 __uint_as_float(v[4 * i + 2]) * inv, __uint_as_float(v[4 * i + 3]) * inv);
                    }
                }
            }
            if (valid && (a.mode & kStateOut)) {
                a.m_out[slot] = (m2 == -INFINITY) ? -INFINITY : m2 * 0.6931471805599453f;
                a.ell_out[slot] = ell;
            }
            if (valid && (a.mode & kFinal) && !(ell > 0.0f)) atomicExch(a.err_flag, 2);
            if ((a.mode & kPrefix) && r == 0) {
                const bool overflow = t.np > 0 && committed == t.np && t.avail < t.n * g.S;
                if (overflow) {
                    // walked the whole truncated list without stopping: rerun on the full plan
                    const int slot = atomicAdd(a.ovf_count, 1);
                    a.ovf_tiles[slot] = (int32_t)a.tile_at(tile);
                } else {
                    a.processed[(t.zh * g.N + t.n) * a.T + t.ti] = committed;
                    if (pairs) atomicAdd((unsigned long long*)&a.pass2_pairs[t.zh], (unsigned long long)(pairs * t.tn));
                }
            }
            tc_fence_before();
            named_bar_sync(1, 128);  // all rows done with this tile's O before the next init
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tbase, kTmemCols);
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    });
    return fn;
}

// 2-D view of a [.., D] bf16 tensor as rows of D elements; box = box_rows x 64 columns
// (1 row for tile::gather4, 128 rows for contiguous tile loads).
bool make_row_map(CUtensorMap* map, const void* base, int64_t rows, uint32_t box_rows = 1) {
    auto enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)kD, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)kD * 2};
    cuuint32_t box[2] = {64, box_rows};
    cuuint32_t es[2] = {1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int64_t span_rows(const int64_t* st, int64_t z, int64_t h, int64_t l) {
    // rows (of D elements) spanned by a strided [z, h, l, D] tensor
    return ((z - 1) * st[0] + (h - 1) * st[1] + (l - 1) * st[2]) / kD + 1;
}

bool strides_ok(const int64_t* st) {
    return st[0] % kD == 0 && st[1] % kD == 0 && st[2] % kD == 0;
}

}  // namespace

bool tc_supported(const PassArgs& a) {
    const Geo& g = a.g;
    if (!g.in_bf16 || g.d != kD || a.bm != kBM || a.bn != kBN) return false;
    if (!strides_ok(g.qs) || !strides_ok(g.ks) || !strides_ok(g.vs)) return false;
    if (g.os[2] % 8 != 0 || g.os[1] % 8 != 0 || g.os[0] % 8 != 0) return false;
    if (span_rows(g.qs, g.z, g.hq, g.l) >= (int64_t(1) << 31) ||
        span_rows(g.ks, g.z, g.hkv, g.l) >= (int64_t(1) << 31))
        return false;
    return get_encode() != nullptr;
}

cudaError_t launch_tc_pass(const PassArgs& a, cudaStream_t st) {
    const Geo& g = a.g;
    CUtensorMap qmap, kmap, vmap, qtile, ktile, vtile;
    const int64_t qrows = span_rows(g.qs, g.z, g.hq, g.l);
    const int64_t krows = span_rows(g.ks, g.z, g.hkv, g.l);
    const int64_t vrows = span_rows(g.vs, g.z, g.hkv, g.l);
    if (!make_row_map(&qmap, a.q, qrows) || !make_row_map(&kmap, a.k, krows) ||
        !make_row_map(&vmap, a.v, vrows) || !make_row_map(&qtile, a.q, qrows, kBM) ||
        !make_row_map(&ktile, a.k, krows, kBN) || !make_row_map(&vtile, a.v, vrows, kBN))
        return cudaErrorInvalidValue;
    TcParams p;
    std::memset(&p, 0, sizeof p);
    p.a = a;
    p.scale_log2 = (float)(a.scale * 1.4426950408889634);
    p.q_contig = g.qs[2] == kD;
    p.kv_contig = g.ks[2] == kD && g.vs[2] == kD;
    static bool attr_done = false;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(tc_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
        if (e != cudaSuccess) return e;
        attr_done = true;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t tiles = a.num_tiles();
    if (tiles == 0) return cudaSuccess;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, sms));
    tc_pass_kernel<<<grid, kThreads, kSmemBytes, st>>>(p, qmap, kmap, vmap, qtile, ktile, vtile);
    return cudaGetLastError();
}

}  // namespace s2o
