// attn_sm100.cu -- Step 2 of S2O on tcgen05 tensor cores (bf16 in, fp32 accumulate in TMEM).
//
// One persistent kernel serves pass-1 (intra-segment causal scan, segment_causal_tile
// kernel.cpp:36-71), pass-2 (ranked prefix traversal with the monotone-gain stop,
// traverse_prefix kernel.cpp:86-122 + early_stop_check kernel.cpp:220-234) and the fused
// single pass (kernel.cpp:300-349).
//
// Work unit: a PAIR of 128-row query tiles of the same (head, segment). Their key streams
// are the same list of 128-key blocks -- the segment's causal blocks (masked on original
// token positions; the second tile has one more) followed by the chunks of kv_perm in rank
// order -- so every K/V block is loaded once and feeds both tiles. TMA tile::gather4 is
// capped at ~22 cycles/op per SM (profiles/r01_summary.md), so sharing a gathered chunk
// between two tiles halves the dominant cost of pass-2.
//
// Warp roles (384 threads, 1 CTA per SM):
//   warps 0-3  softmax/correction/epilogue of slot 0 (thread r owns row r = TMEM lane r)
//   warps 4-7  softmax/correction/epilogue of slot 1
//   warp 8     MMA issuer (one lane): S_X = Q_X K^T (SS MMA), O_X += P_X V (TS MMA, P in TMEM)
//   warps 9-11 loaders: 2-D tile TMA for contiguous rows, TMA tile::gather4 for permuted rows
//
// Early stop (reference semantics): each row's relative normaliser gain of a prefix chunk,
// sum_j exp(s_j - m) / ell, is computed from the chunk's scores; the max over the tile's rows
// is compared with tau before P V is issued; a stopping chunk changes nothing (kernel.cpp:
// 114-117). The two tiles of a pair stop independently; the pair's stream ends when both did.
//
// Shared memory (SWIZZLE_128B, 1024-B aligned): Q slot 0/1 (2 x 32 KB), 2 stages x (K 32 KB +
// V 32 KB). TMEM (512 columns): slot X uses [256X, 256X+128) for S (P = exp2(s - m) in bf16 is
// written over the first 64 columns after S is read) and [256X+128, 256X+256) for O.
//
// Ordering facts the pipeline relies on:
//  * tcgen05.commit arrives when ALL earlier MMAs of the issuing thread completed, so
//    s_full[X](j) also certifies P_X V(j-1) done: the softmax may then overwrite P_X and
//    rescale O_X without another barrier.
//  * Every mbarrier completes at most one phase ahead of its waiter (parity waits).
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
constexpr int kStages = 2;
constexpr int kThreads = 384;
constexpr int kMmaWarp = 8;
constexpr int kLoadWarp0 = 9;
constexpr int kLoaderThreads = 96;
constexpr uint32_t kHalf = 128u * 128u;     // one 64-column half of a 128-row tile
constexpr uint32_t kTileBytes = 2 * kHalf;  // 32 KB
constexpr uint32_t kOffQ = 0;               // slot X at X * kTileBytes
constexpr uint32_t kOffK = 2 * kTileBytes;
constexpr uint32_t kOffV = kOffK + kStages * kTileBytes;
constexpr uint32_t kOffCtrl = kOffV + kStages * kTileBytes;
constexpr uint32_t kSmemBytes = kOffCtrl + 1024 + 1024;
constexpr uint32_t kTmemCols = 512;
constexpr float kRescaleThresh = 8.0f;  // lazy max update, log2 units (factor 256)

struct Ctrl {
    uint64_t q_full, q_empty;
    uint64_t k_full[kStages], v_full[kStages], kv_empty[kStages];
    uint64_t s_full[2], p_full[2], o_done[2];
    uint32_t tmem_base;
    float red[2][4];
    uint8_t dec[2][4];  // per slot decision ring (block j -> j & 3): 1 = commit, 2 = stop
};

struct TcParams {
    PassArgs a;
    float scale_log2;  // (1/sqrt(D)) * log2(e)
    int q_contig, kv_contig;
    int64_t pairs_per_head, pairs_full;  // pairs per head; pairs in a full segment
};

struct PairInfo {
    int64_t zh, n, sb, seg_rows, avail;
    int64_t ti[2], t0[2], tn[2];
    int has[2];
    int nd[2], ndmax, np, nb;
};

__device__ __forceinline__ PairInfo pair_info(const TcParams& p, int64_t idx) {
    const PassArgs& a = p.a;
    const Geo& g = a.g;
    PairInfo P;
    if (a.tile_list) {
        const int64_t tile = a.tile_list[idx];
        P.zh = tile / a.tiles_per_head;
        const int64_t r = tile % a.tiles_per_head;
        const int64_t full = (g.N - 1) * a.T;
        if (r < full) { P.n = r / a.T; P.ti[0] = r % a.T; }
        else { P.n = g.N - 1; P.ti[0] = r - full; }
        P.ti[1] = -1;
    } else {
        P.zh = idx / p.pairs_per_head;
        const int64_t r = idx % p.pairs_per_head;
        const int64_t full = (g.N - 1) * p.pairs_full;
        int64_t pi, tcount;
        if (r < full) { P.n = r / p.pairs_full; pi = r % p.pairs_full; tcount = a.T; }
        else { P.n = g.N - 1; pi = r - full; tcount = (g.last_len + kBM - 1) / kBM; }
        P.ti[0] = 2 * pi;
        P.ti[1] = (2 * pi + 1 < tcount) ? 2 * pi + 1 : -1;
    }
    P.sb = P.n * g.S;
    P.seg_rows = g.seg_rows(P.n);
    P.avail = a.avail(P.n);
    P.ndmax = 0;
    for (int x = 0; x < 2; ++x) {
        P.has[x] = P.ti[x] >= 0;
        P.t0[x] = P.has[x] ? P.ti[x] * kBM : 0;
        P.tn[x] = P.has[x] ? min((int64_t)kBM, P.seg_rows - P.t0[x]) : 0;
        P.nd[x] = (P.has[x] && (a.mode & kDiag)) ? (int)((P.t0[x] + P.tn[x] - 1) / kBN + 1) : 0;
        P.ndmax = max(P.ndmax, P.nd[x]);
    }
    P.np = ((a.mode & kPrefix) && P.n > 0) ? (int)((P.avail + kBN - 1) / kBN) : 0;
    P.nb = P.ndmax + P.np;
    return P;
}

__device__ __forceinline__ bool participates(const PairInfo& P, int x, int j) {
    return P.has[x] && (j < P.ndmax ? j < P.nd[x] : true);
}
__device__ __forceinline__ int last_block(const PairInfo& P, int x) {
    return P.np > 0 ? P.nb - 1 : P.nd[x] - 1;
}

// Segment row of query row r of slot x (ragged tails duplicate row 0; results discarded).
__device__ __forceinline__ int64_t q_row(const PassArgs& a, const PairInfo& P, int x, int64_t r) {
    if (r >= P.tn[x]) r = 0;
    const int64_t local = ((a.mode & kStateIn) && a.q_reorder)
                              ? (int64_t)a.q_perm[(P.zh * a.g.N + P.n) * a.g.S + P.t0[x] + r]
                              : P.t0[x] + r;
    return P.sb + local;
}

// Token index of key i of block j (clamped into the block's valid range).
__device__ __forceinline__ int64_t key_token(const PairInfo& P, const int32_t* kv, int j, int i) {
    if (j < P.ndmax) {
        const int64_t k0 = (int64_t)j * kBN;
        const int64_t kn = min((int64_t)kBN, P.seg_rows - k0);
        return P.sb + k0 + (i < kn ? i : 0);
    }
    const int64_t c0 = (int64_t)(j - P.ndmax) * kBN;
    const int64_t cn = min((int64_t)kBN, P.avail - c0);
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
        for (int x = 0; x < 2; ++x) {
            mbar_init(smem_u32(&c.s_full[x]), 1);
            mbar_init(smem_u32(&c.p_full[x]), 4);
            mbar_init(smem_u32(&c.o_done[x]), 1);
        }
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
    const int64_t total = a.tile_list ? a.tile_count : g.z * g.hq * p.pairs_per_head;
    const int64_t rowu = g.d;  // row unit of the tensor maps = D elements

    if (warp >= kLoadWarp0) {
        // ============================== loaders ==============================
        const int lt = (warp - kLoadWarp0) * 32 + lane;  // 0..95
        uint32_t gblk = 0, qcount = 0;
        for (int64_t it = blockIdx.x; it < total; it += gridDim.x) {
            const PairInfo P = pair_info(p, it);
            if (P.nb == 0) continue;
            const int32_t* kv = (P.np > 0) ? a.kv_seg(P.zh, P.n) : nullptr;
            mbar_wait(smem_u32(&c.q_empty), (qcount & 1) ^ 1, 1001);
            const int64_t qb = g.q_base(P.zh) / rowu, qs = g.qs[2] / rowu;
            const bool q_tile = p.q_contig && !((a.mode & kStateIn) && a.q_reorder);
            if (lt == 0) mbar_expect_tx(smem_u32(&c.q_full), (P.has[1] ? 2 : 1) * kTileBytes);
            named_bar_sync(3, kLoaderThreads);
            for (int x = 0; x < 2; ++x) {
                if (!P.has[x]) continue;
                const uint32_t qdst = sQ + x * kTileBytes;
                if (q_tile && P.tn[x] == kBM) {
                    if (lt == 0)
                        for (int h = 0; h < 2; ++h)
                            tma_load2d(qdst + h * kHalf, &qtile, h * 64, (int32_t)(qb + (P.sb + P.t0[x]) * qs),
                                       smem_u32(&c.q_full));
                } else if (lt < 64) {
                    const int grp = lt >> 1, h = lt & 1;
                    int32_t rows[4];
                    for (int i = 0; i < 4; ++i) rows[i] = (int32_t)(qb + q_row(a, P, x, grp * 4 + i) * qs);
                    tma_gather4(qdst + h * kHalf + grp * 512, &qmap, h * 64, rows[0], rows[1], rows[2], rows[3],
                                smem_u32(&c.q_full));
                }
            }
            ++qcount;
            const int64_t kb = g.k_base(P.zh) / rowu, vb = g.v_base(P.zh) / rowu;
            const int64_t ks = g.ks[2] / rowu, vs = g.vs[2] / rowu;
            // gather ops of one block: [0,64) K, [64,128) V; op -> (row group, half)
            auto fetch_rows = [&](int j, int32_t (&rr)[2][4]) {
                for (int u = 0; u < 2; ++u) {
                    const int op = lt + u * kLoaderThreads;
                    const int grp = (op >> 1) & 31;
                    const bool isv = op >= 64;
                    for (int i = 0; i < 4; ++i) {
                        const int64_t tok = (op < 128 && j < P.nb) ? key_token(P, kv, j, grp * 4 + i) : 0;
                        rr[u][i] = (int32_t)(isv ? vb + tok * vs : kb + tok * ks);
                    }
                }
            };
            const auto gathered = [&](int j) { return !(j < P.ndmax && p.kv_contig); };
            int32_t cur[2][4], nxt[2][4];
            if (gathered(0)) fetch_rows(0, cur);
            bool stop_known[2] = {false, false};
            int loaded = 0;
            for (int j = 0; j < P.nb; ++j) {
                const uint32_t gi = gblk + j;
                const int st = gi % kStages;
                if (j + 1 < P.nb && gathered(j + 1)) fetch_rows(j + 1, nxt);
                mbar_wait(smem_u32(&c.kv_empty[st]), ((gi / kStages) & 1) ^ 1, 1002);
                // acquiring stage j certifies that both slots' decisions on block j-2 are final
                if (j >= 2 && j - 2 >= P.ndmax)
                    for (int x = 0; x < 2; ++x)
                        if (participates(P, x, j - 2) && c.dec[x][(j - 2) & 3] == 2) stop_known[x] = true;
                bool need = false;
                for (int x = 0; x < 2; ++x) need |= participates(P, x, j) && !stop_known[x];
                if (!need) break;
                if (lt == 0) {
                    mbar_expect_tx(smem_u32(&c.k_full[st]), kTileBytes);
                    mbar_expect_tx(smem_u32(&c.v_full[st]), kTileBytes);
                }
                named_bar_sync(3, kLoaderThreads);
                const uint32_t kdst = sK + st * kTileBytes;
                const uint32_t vdst = sV + st * kTileBytes;
                if (!gathered(j)) {
                    if (lt == 0) {
                        const int64_t tok = P.sb + (int64_t)j * kBN;
                        for (int h = 0; h < 2; ++h)
                            tma_load2d(kdst + h * kHalf, &ktile, h * 64, (int32_t)(kb + tok * ks), smem_u32(&c.k_full[st]));
                        for (int h = 0; h < 2; ++h)
                            tma_load2d(vdst + h * kHalf, &vtile, h * 64, (int32_t)(vb + tok * vs), smem_u32(&c.v_full[st]));
                    }
                } else {
                    for (int u = 0; u < 2; ++u) {
                        const int op = lt + u * kLoaderThreads;
                        if (op >= 128) break;
                        const int grp = (op >> 1) & 31, h = op & 1;
                        const bool isv = op >= 64;
                        tma_gather4((isv ? vdst : kdst) + h * kHalf + grp * 512, isv ? &vmap : &kmap, h * 64,
                                    cur[u][0], cur[u][1], cur[u][2], cur[u][3],
                                    smem_u32(isv ? &c.v_full[st] : &c.k_full[st]));
                    }
                }
                for (int u = 0; u < 2; ++u)
                    for (int i = 0; i < 4; ++i) cur[u][i] = nxt[u][i];
                ++loaded;
            }
            gblk += loaded;
        }
    } else if (warp == kMmaWarp) {
        // ============================== MMA issuer ==============================
        if (lane == 0) {
            const uint32_t idesc_s = umma_idesc_bf16(kBM, kBN, false, false);
            const uint32_t idesc_o = umma_idesc_bf16(kBM, kD, false, true);
            uint32_t gblk = 0, qcount = 0;
            uint32_t ns[2] = {0, 0};  // s_full / p_full phases per slot
            for (int64_t it = blockIdx.x; it < total; it += gridDim.x) {
                const PairInfo P = pair_info(p, it);
                if (P.nb == 0) continue;
                mbar_wait(smem_u32(&c.q_full), qcount & 1, 2001);
                ++qcount;
                tc_fence_after();
                int stop_at[2] = {1 << 30, 1 << 30};
                int loaded = 0;
                for (int j = 0; j < P.nb; ++j) {
                    // same predicate as the loader: decisions on blocks <= j-2 are known there
                    bool need = false;
                    for (int x = 0; x < 2; ++x) need |= participates(P, x, j) && !(stop_at[x] <= j - 2);
                    if (!need) break;
                    ++loaded;
                    const uint32_t gi = gblk + j;
                    const int st = gi % kStages;
                    const uint32_t ph = (gi / kStages) & 1;
                    mbar_wait(smem_u32(&c.k_full[st]), ph, 2002);
                    tc_fence_after();
                    bool act[2];
                    for (int x = 0; x < 2; ++x) act[x] = participates(P, x, j) && stop_at[x] > j - 1;
                    const uint32_t kbase = sK + st * kTileBytes;
                    for (int x = 0; x < 2; ++x) {
                        if (!act[x]) continue;
                        const uint32_t qbase = sQ + x * kTileBytes;
                        for (int kk = 0; kk < kD / 16; ++kk) {
                            const uint32_t off = (kk / 4) * kHalf + (kk % 4) * 32;
                            umma_bf16(tbase + x * 256, umma_desc_sw128(qbase + off, 16, 1024),
                                      umma_desc_sw128(kbase + off, 16, 1024), idesc_s, kk > 0);
                        }
                        umma_commit(smem_u32(&c.s_full[x]));
                    }
                    bool v_ready = false;
                    for (int x = 0; x < 2; ++x) {
                        if (!act[x]) continue;
                        mbar_wait(smem_u32(&c.p_full[x]), ns[x] & 1, 2004);
                        ++ns[x];
                        tc_fence_after();
                        if (c.dec[x][j & 3] == 1) {
                            if (!v_ready) {
                                mbar_wait(smem_u32(&c.v_full[st]), ph, 2005);
                                tc_fence_after();
                                v_ready = true;
                            }
                            const uint32_t vbase = sV + st * kTileBytes;
                            for (int kk = 0; kk < kBN / 16; ++kk)
                                umma_bf16_ts(tbase + x * 256 + 128, tbase + x * 256 + kk * 8,
                                             umma_desc_sw128(vbase + kk * 16 * 128, kHalf, 1024), idesc_o, 1);
                            if (j == last_block(P, x)) umma_commit(smem_u32(&c.o_done[x]));
                        } else {
                            stop_at[x] = j;
                            umma_commit(smem_u32(&c.o_done[x]));  // slot finished
                        }
                    }
                    if (!v_ready) mbar_wait(smem_u32(&c.v_full[st]), ph, 2006);  // consume the phase
                    umma_commit(smem_u32(&c.kv_empty[st]));
                }
                umma_commit(smem_u32(&c.q_empty));
                gblk += loaded;
            }
        }
        __syncwarp();
    } else {
        // ============================== softmax / epilogue (slot x) ==============================
        const int x = warp / 4;
        const int r = threadIdx.x % 128;  // TMEM lane
        const uint32_t lane_off = (uint32_t)((warp % 4) * 32) << 16;
        const uint32_t tS = tbase + lane_off + x * 256;
        const uint32_t tO = tS + 128;
        const uint32_t bar_id = 1 + x;
        uint32_t ns = 0, no = 0;
        for (int64_t it = blockIdx.x; it < total; it += gridDim.x) {
            const PairInfo P = pair_info(p, it);
            if (!P.has[x]) continue;
            const bool valid = r < P.tn[x];
            const int64_t grow = q_row(a, P, x, r);
            const int64_t slot = P.zh * g.l + grow;
            float m2, ell;
            // ---- state init: O in TMEM, (m, ell) in registers
            if (a.mode & kStateIn) {
                m2 = a.m_in[slot] * 1.4426950408889634f;
                ell = a.ell_in[slot];
                const float4* src = reinterpret_cast<const float4*>(a.acc_in + slot * kD);
                for (int c0 = 0; c0 < kD; c0 += 32) {
                    uint32_t v[32];
                    for (int i = 0; i < 8; ++i) {
                        const float4 y = src[c0 / 4 + i];
                        v[4 * i] = __float_as_uint(y.x);
                        v[4 * i + 1] = __float_as_uint(y.y);
                        v[4 * i + 2] = __float_as_uint(y.z);
                        v[4 * i + 3] = __float_as_uint(y.w);
                    }
                    tmem_st32(tO + c0, v);
                }
            } else {
                m2 = -INFINITY;
                ell = 0.0f;
                uint32_t z[32];
                for (int i = 0; i < 32; ++i) z[i] = 0u;
                for (int c0 = 0; c0 < kD; c0 += 32) tmem_st32(tO + c0, z);
            }
            tmem_st_wait();
            tc_fence_before();

            int committed = 0;
            int64_t pairs = 0;
            bool any = false;
            for (int j = 0; j < P.nb; ++j) {
                if (!participates(P, x, j)) continue;
                any = true;
                mbar_wait(smem_u32(&c.s_full[x]), ns & 1, 3001);
                ++ns;
                tc_fence_after();
                // ---- visible keys of this block for this row
                const bool is_diag = j < P.ndmax;
                int lim;
                if (is_diag) {
                    const int64_t k0 = (int64_t)j * kBN;
                    const int64_t kn = min((int64_t)kBN, P.seg_rows - k0);
                    const int64_t vis = (k0 + kn - 1 <= P.t0[x]) ? kn : min(kn, P.t0[x] + r - k0 + 1);
                    lim = (int)max((int64_t)0, vis);
                } else {
                    const int64_t c0 = (int64_t)(j - P.ndmax) * kBN;
                    lim = (int)min((int64_t)kBN, P.avail - c0);
                }
                // ---- pass 1: row max (S read from TMEM in 32-column chunks)
                float mxa[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                for (int c0 = 0; c0 < kBN; c0 += 32) {
                    uint32_t v[32];
                    tmem_ld32(tS + c0, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const float sv = (c0 + i < lim) ? __uint_as_float(v[i]) : -INFINITY;
                        mxa[i & 3] = fmaxf(mxa[i & 3], sv);
                    }
                }
                const float mx = fmaxf(fmaxf(mxa[0], mxa[1]), fmaxf(mxa[2], mxa[3])) * p.scale_log2;
                const float m_new = fmaxf(m2, mx);
                const bool rescale = (m_new > m2 + kRescaleThresh) || (m2 == -INFINITY);
                const float m_use = rescale ? m_new : m2;
                const float neg_ref = (m_use == -INFINITY) ? 0.0f : -m_use;
                const float alpha = (m2 == -INFINITY) ? 0.0f : ex2(m2 + neg_ref);
                // O rescale (P V of the previous block is complete: s_full orders after it)
                if (__any_sync(0xffffffffu, rescale && m2 != -INFINITY)) {
                    for (int c0 = 0; c0 < kD; c0 += 32) {
                        uint32_t v[32];
                        tmem_ld32(tO + c0, v);
                        tmem_ld_wait();
                        for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
                        tmem_st32(tO + c0, v);
                    }
                }
                // ---- pass 2: P = exp2(s*scale - m) -> bf16 pairs over the first 64 S columns
                float rs[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
                for (int c0 = 0; c0 < kBN; c0 += 32) {
                    uint32_t v[32];
                    tmem_ld32(tS + c0, v);
                    tmem_ld_wait();
                    uint32_t pk[16];
#pragma unroll
                    for (int i = 0; i < 32; i += 2) {
                        const float e0 = (c0 + i < lim) ? ex2(fmaf(__uint_as_float(v[i]), p.scale_log2, neg_ref)) : 0.0f;
                        const float e1 = (c0 + i + 1 < lim) ? ex2(fmaf(__uint_as_float(v[i + 1]), p.scale_log2, neg_ref)) : 0.0f;
                        rs[(i >> 1) & 3] += e0 + e1;
                        pk[i >> 1] = pack_bf16(e0, e1);
                    }
                    tmem_st16(tS + c0 / 2, pk);
                }
                const float rowsum = (rs[0] + rs[1]) + (rs[2] + rs[3]);
                bool commit = true;
                if (!is_diag) {
                    // relative normaliser gain of this chunk (kernel.cpp:108-115)
                    const float prev = ell * alpha;
                    float gain = valid ? rowsum / prev : -INFINITY;
                    for (int o = 16; o > 0; o >>= 1) gain = fmaxf(gain, __shfl_xor_sync(0xffffffffu, gain, o));
                    if (lane == 0) c.red[x][warp % 4] = gain;
                    named_bar_sync(bar_id, 128);
                    const float mg = fmaxf(fmaxf(c.red[x][0], c.red[x][1]), fmaxf(c.red[x][2], c.red[x][3]));
                    commit = !(mg < (float)a.tau);
                    named_bar_sync(bar_id, 128);  // red[] reusable
                }
                // state update (on a stop the rescaled state is the same state: O/ell unchanged)
                ell = commit ? ell * alpha + rowsum : ell * alpha;
                m2 = m_use;
                if (commit && !is_diag) {
                    ++committed;
                    const int64_t c0 = (int64_t)(j - P.ndmax) * kBN;
                    pairs += min((int64_t)kBN, P.avail - c0);
                }
                tmem_st_wait();
                tc_fence_before();
                if (r == 0) c.dec[x][j & 3] = commit ? 1 : 2;
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&c.p_full[x]));
                if (!commit) break;
            }
            if (any) {
                mbar_wait(smem_u32(&c.o_done[x]), no & 1, 3004);
                ++no;
                tc_fence_after();
            }
            // ---- read O, finalize / persist
            const float inv = 1.0f / ell;
            for (int c0 = 0; c0 < kD; c0 += 32) {
                uint32_t v[32];
                tmem_ld32(tO + c0, v);
                tmem_ld_wait();
                if (!valid) continue;
                if (a.mode & kStateOut) {
                    float4* dst = reinterpret_cast<float4*>(a.acc_out + slot * kD + c0);
                    for (int i = 0; i < 8; ++i)
                        dst[i] = make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                             __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
                }
                if (a.mode & kFinal) {
                    const int64_t ooff = g.o_base(P.zh) + grow * g.os[2] + c0;
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
                const int64_t tile = P.zh * a.tiles_per_head + P.n * a.T + P.ti[x];
                const bool overflow = P.np > 0 && committed == P.np && P.avail < P.n * g.S;
                if (overflow) {
                    // walked the whole truncated list without stopping: rerun on the full plan
                    const int s2 = atomicAdd(a.ovf_count, 1);
                    a.ovf_tiles[s2] = (int32_t)tile;
                } else {
                    a.processed[(P.zh * g.N + P.n) * a.T + P.ti[x]] = committed;
                    if (pairs) atomicAdd((unsigned long long*)&a.pass2_pairs[P.zh], (unsigned long long)(pairs * P.tn[x]));
                }
            }
            tc_fence_before();
            named_bar_sync(bar_id, 128);  // all rows done with O before the next pair's init
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
    return ((z - 1) * st[0] + (h - 1) * st[1] + (l - 1) * st[2]) / kD + 1;
}

bool strides_ok(const int64_t* st) { return st[0] % kD == 0 && st[1] % kD == 0 && st[2] % kD == 0; }

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
    p.pairs_full = (a.T + 1) / 2;
    const int64_t t_last = (g.last_len + kBM - 1) / kBM;
    p.pairs_per_head = (g.N - 1) * p.pairs_full + (t_last + 1) / 2;
    static bool attr_done = false;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(tc_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
        if (e != cudaSuccess) return e;
        attr_done = true;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t work = a.tile_list ? a.tile_count : g.z * g.hq * p.pairs_per_head;
    if (work == 0) return cudaSuccess;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(work, sms));
    tc_pass_kernel<<<grid, kThreads, kSmemBytes, st>>>(p, qmap, kmap, vmap, qtile, ktile, vtile);
    return cudaGetLastError();
}

}  // namespace s2o
