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
#include <cstdlib>
#include <algorithm>
#include <climits>
#include <cstring>
#include <mutex>
#include <utility>
#include <vector>

#include "internal.h"
#include "sm100.cuh"

namespace s2o {

using namespace sm100;

namespace {

constexpr int kD = 128;
constexpr int kBM = 128;
constexpr int kBN = 128;
constexpr int kKStages = 3;  // K ring: block j may load once decisions <= j-3 are known (A/B: 2 stages +9 %)
constexpr int kVStages = 2;  // V ring: block j may load once decisions <= j-2 are known
constexpr int kThreads = 512;
constexpr int kMmaWarp = 8;
constexpr int kKWarp0 = 9;    // K loader group: warps 9-12 (also loads Q)
constexpr int kVWarp0 = 13;   // V loader group: warps 13-15
constexpr int kKThreads = 128;
constexpr int kVThreads = 96;
constexpr uint32_t kHalf = 128u * 128u;     // one 64-column half of a 128-row tile
constexpr uint32_t kTileBytes = 2 * kHalf;  // 32 KB
constexpr uint32_t kOffQ = 0;               // slot X at X * kTileBytes
constexpr uint32_t kOffK = 2 * kTileBytes;
constexpr uint32_t kOffV = kOffK + kKStages * kTileBytes;
constexpr uint32_t kOffCtrl = kOffV + kVStages * kTileBytes;
constexpr uint32_t kOffTok = kOffCtrl + 512;  // token rings: K group int32 [2][128], V group [2][128]
constexpr uint32_t kSmemBytes = kOffTok + 2304;  // 226.75 KB (base must be 1024-B aligned)
constexpr uint32_t kTmemCols = 512;
constexpr int kSoftmaxRegs = 176;   // setmaxnreg: softmax warpgroups (0, 1) (A/B: 192 5.69, 184 5.63, 176 5.59 ms)
constexpr int kOtherRegs = 80;      // MMA + loader warpgroups (2, 3)
constexpr int kLaunchRegs = 65536 / kThreads / 8 * 8;  // 128: what __launch_bounds__(512, 1) allots
// setmaxnreg.inc blocks until the pool has the registers: the decrements must cover it
static_assert(kSoftmaxRegs - kLaunchRegs <= kLaunchRegs - kOtherRegs, "register pool overcommitted");
static_assert(sizeof(uint64_t) * 33 + 4 + 64 + 8 <= 512, "Ctrl exceeds its 512 B");
constexpr float kRescaleThresh = 8.0f;
  // lazy max update, log2 units (factor 256)

struct Ctrl {
    uint64_t q_full[2], q_empty[2];  // per slot: a slot's Q tile is released when its stream ends
    uint64_t k_full[kKStages], k_empty[kKStages], v_full[kVStages], v_empty[kVStages];
    uint64_t s_full[2], p_full[2], o_done[2];
    uint32_t tmem_base;
    uint32_t red[2][2][4];  // continue votes [slot][block parity][warp]
    uint8_t dec[2][4];  // per slot decision ring (block j -> j & 3): 1 = commit, 2 = stop
    // dynamic work ring: the K loader group fetches pair indices from a global counter
    // (work_ctr) and every warp of the CTA takes them in order (item k in slot k & 3)
    uint64_t w_full[4], w_empty[4];
    int64_t wq[4];
};

constexpr int kWarps = kThreads / 32;

// Item k of the work ring (all lanes of the calling warp): the pair index, or -1 when done.
__device__ __forceinline__ int64_t ring_get(Ctrl& c, uint32_t k, int lane) {
    mbar_wait(smem_u32(&c.w_full[k & 3]), (k >> 2) & 1, 5001);
    const int64_t it = *reinterpret_cast<volatile int64_t*>(&c.wq[k & 3]);
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(&c.w_empty[k & 3]));
    return it;
}

// Division by a launch constant without the integer-division sequence (its MUFU.RCP would queue
// behind the softmax warps' exponentials on the same SMSP): q = (umulhi(n, mul) + n) >> shift,
// exact for n < 2^31 (Granlund-Montgomery; mul, shift from the host).
struct FastDiv {
    uint32_t d, mul, shift;
    FastDiv() = default;
    explicit FastDiv(uint32_t div) : d(div) {
        shift = 0;
        while ((1ull << shift) < div) ++shift;
        mul = (uint32_t)(((1ull << 32) * ((1ull << shift) - div)) / div + 1);
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const { return (__umulhi(n, mul) + n) >> shift; }
};

struct TcParams {
    PassArgs a;
    float scale_log2;  // (1/sqrt(D)) * log2(e)
    int q_contig, kv_contig;
    int vec_acc, vec_o;  // 256-bit epilogue accesses (32-B aligned state / output rows)
    int64_t pairs_per_head, pairs_full;  // pairs per head; pairs in a full segment
    unsigned long long* tl;              // optional timeline (CTA 0), see s2o_debug_timeline
    FastDiv fd_pg, fd_g, fd_pf, fd_tph, fd_t;  // pairs_per_head * group, group, pairs_full, tiles_per_head, T
    FastDiv fd_hq;                             // q heads per batch
};

// Geo's q_base / k_base / v_base / o_base with FastDiv (the tc kernels call these per item)
struct TcBase {
    int64_t z, h, kvh;
    __device__ __forceinline__ TcBase(const TcParams& p, int64_t zh) {
        z = p.fd_hq.div((uint32_t)zh);
        h = zh - z * (int64_t)p.fd_hq.d;
        kvh = p.fd_g.div((uint32_t)h);
    }
};
__device__ __forceinline__ int64_t tc_q_base(const TcParams& p, int64_t zh) {
    const TcBase b(p, zh);
    return b.z * p.a.g.qs[0] + b.h * p.a.g.qs[1];
}
__device__ __forceinline__ int64_t tc_o_base(const TcParams& p, int64_t zh) {
    const TcBase b(p, zh);
    return b.z * p.a.g.os[0] + b.h * p.a.g.os[1];
}
__device__ __forceinline__ int64_t tc_k_base(const TcParams& p, int64_t zh) {
    const TcBase b(p, zh);
    return b.z * p.a.g.ks[0] + b.kvh * p.a.g.ks[1];
}
__device__ __forceinline__ int64_t tc_v_base(const TcParams& p, int64_t zh) {
    const TcBase b(p, zh);
    return b.z * p.a.g.vs[0] + b.kvh * p.a.g.vs[1];
}

// Timeline events (profiling aid): tl[ev * kTlCap + seq] = clock64() in CTA 0.
[[maybe_unused]] constexpr int kTlCap = 1024;
// Compiled in only with -DS2O_TIMELINE (S2O_NVCC_FLAGS=-DS2O_TIMELINE python -m ...build).
__device__ __forceinline__ void tl_mark(const TcParams& p, int ev, uint32_t seq) {
#ifdef S2O_TIMELINE
    if (p.tl != nullptr && blockIdx.x == 0 && seq < (uint32_t)kTlCap)
        p.tl[ev * kTlCap + seq] = clock64();
#endif
}

// Per-CTA span in global-timer ns (timeline builds): tl[0][cta] = start, tl[3][cta] = end.
__device__ __forceinline__ void tl_cta(const TcParams& p, int ev) {
#ifdef S2O_TIMELINE
    if (p.tl != nullptr && blockIdx.x < (uint32_t)kTlCap) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.tl[ev * kTlCap + blockIdx.x] = t;
    }
#endif
}

// Early-stop decision from the four per-warp votes (early_stop_check kernel.cpp:220-234: stop iff
// max gain < tau, strictly, NaN gains dropped <=> continue iff some row has gain >= tau).
__device__ __forceinline__ bool chunk_commit(const uint32_t* red) {
    const volatile uint32_t* rv = red;
    return (rv[0] | rv[1] | rv[2] | rv[3]) != 0u;
}

// 32-bit fields (L < 2^31, checked by make_geo): the loader and MMA warps hold this for a whole
// pair at 64 registers.
struct PairInfo {
    int32_t zh, n, sb, seg_rows, avail;
    int32_t ti[2], t0[2], tn[2];
    int has[2];
    int nd[2], ndmax, np, nb;
};

__device__ __forceinline__ PairInfo pair_info(const TcParams& p, int64_t idx) {
    const PassArgs& a = p.a;
    const Geo& g = a.g;
    PairInfo P;
    int64_t ti0, ti1, n;
    // (32-bit FastDiv decode: item and tile indices < 2^31, checked by the launcher)
    if (a.tile_list) {
        const uint32_t tile = (uint32_t)a.tile_list[idx];
        const uint32_t zh = p.fd_tph.div(tile);
        P.zh = (int32_t)zh;
        const uint32_t r = tile - zh * p.fd_tph.d;
        const uint32_t full = (uint32_t)((g.N - 1) * a.T);
        if (r < full) { n = p.fd_t.div(r); ti0 = r - (uint32_t)n * p.fd_t.d; }
        else { n = g.N - 1; ti0 = r - full; }
        ti1 = -1;
    } else {
        // The q heads of a GQA group share K/V: interleave them (head fastest) so the group's
        // CTAs walk the same segment's K/V rows at the same time and hit L2 together.
        const uint32_t G = p.fd_g.d, i32 = (uint32_t)idx;
        const uint32_t zg = p.fd_pg.div(i32);
        const uint32_t rem = i32 - zg * p.fd_pg.d;
        const uint32_t r = p.fd_g.div(rem);
        P.zh = (int32_t)(zg * G + (rem - r * G));
        const uint32_t full = (uint32_t)((g.N - 1) * p.pairs_full);
        int64_t pi, tcount;
        if (r < full) {
            n = p.fd_pf.div(r);
            pi = r - (uint32_t)n * p.fd_pf.d;
            tcount = a.T;
        } else { n = g.N - 1; pi = r - full; tcount = (g.last_len + kBM - 1) / kBM; }
        ti0 = 2 * pi;
        ti1 = (2 * pi + 1 < tcount) ? 2 * pi + 1 : -1;
    }
    P.n = (int32_t)n;
    P.ti[0] = (int32_t)ti0;
    P.ti[1] = (int32_t)ti1;
    P.sb = (int32_t)(n * g.S);
    P.seg_rows = (int32_t)g.seg_rows(n);
    P.avail = (int32_t)a.avail(n);
    P.ndmax = 0;
    for (int x = 0; x < 2; ++x) {
        P.has[x] = P.ti[x] >= 0;
        P.t0[x] = P.has[x] ? P.ti[x] * kBM : 0;
        P.tn[x] = P.has[x] ? min(kBM, P.seg_rows - P.t0[x]) : 0;
        P.nd[x] = (P.has[x] && (a.mode & kDiag)) ? (P.t0[x] + P.tn[x] - 1) / kBN + 1 : 0;
        P.ndmax = max(P.ndmax, P.nd[x]);
    }
    P.np = ((a.mode & kPrefix) && P.n > 0) ? (P.avail + kBN - 1) / kBN : 0;
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

template <bool kPackedExp>
__global__ void __launch_bounds__(kThreads, 1)
tc_pass_kernel(const TcParams p, const __grid_constant__ CUtensorMap qmap,
               const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
               const __grid_constant__ CUtensorMap qtile, const __grid_constant__ CUtensorMap ktile,
               const __grid_constant__ CUtensorMap vtile) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw;
    if (p.a.tile_list && p.a.num_tiles() == 0) return;  // a stream-ordered level with nothing to redo
    if ((smem_u32(smem) & 1023u) != 0) __trap();  // SWIZZLE_128B tiles need a 1024-B aligned base
    Ctrl& c = *reinterpret_cast<Ctrl*>(smem + kOffCtrl);
    const PassArgs& a = p.a;
    const Geo& g = a.g;
    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const uint32_t sQ = smem_u32(smem + kOffQ);
    const uint32_t sK = smem_u32(smem + kOffK);
    const uint32_t sV = smem_u32(smem + kOffV);

    if (threadIdx.x == 0) {
        // full barriers: every loader thread arrives once per phase (TMA expect_tx by one
        // thread + plain arrives, or cp.async.mbarrier.arrive.noinc by all)
        for (int x = 0; x < 2; ++x) {
            mbar_init(smem_u32(&c.q_full[x]), kKThreads);
            mbar_init(smem_u32(&c.q_empty[x]), 1);
        }
        for (int s = 0; s < kKStages; ++s) {
            mbar_init(smem_u32(&c.k_full[s]), kKThreads);
            mbar_init(smem_u32(&c.k_empty[s]), 1);
        }
        for (int s = 0; s < kVStages; ++s) {
            mbar_init(smem_u32(&c.v_full[s]), kVThreads);
            mbar_init(smem_u32(&c.v_empty[s]), 1);
        }
        for (int x = 0; x < 2; ++x) {
            mbar_init(smem_u32(&c.s_full[x]), 1);
            mbar_init(smem_u32(&c.p_full[x]), 4);
            mbar_init(smem_u32(&c.o_done[x]), 1);
        }
        for (int w = 0; w < 4; ++w) {
            mbar_init(smem_u32(&c.w_full[w]), 1);
            mbar_init(smem_u32(&c.w_empty[w]), kWarps);
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
    if (threadIdx.x == 0) tl_cta(p, 0);
    const int64_t total = a.tile_list ? a.num_tiles() : g.z * g.hq * p.pairs_per_head;
    constexpr int64_t rowu = kD;  // row unit of the tensor maps = D elements (tc path: d == 128)

    if (warp >= kMmaWarp) setmaxnreg_dec<kOtherRegs>();  // warpgroups 2-3
    if (warp >= kKWarp0) {
        // ============================== loaders ==============================
        // Two independent groups: K (+ Q) and V, so K(j+1) never waits behind V(j)'s gating.
        // Gathered rows (permuted Q rows, ranked prefix keys) move with TMA tile::gather4 (4 rows
        // x one 64-column half per op) into the SWIZZLE_128B layout; contiguous 128-row blocks
        // with one 2-D TMA tile per 64-column half. Tokens of the next block wait in a shared
        // ring, one block ahead.
        const bool kgrp = warp < kVWarp0;
        const int nthr = kgrp ? kKThreads : kVThreads;
        const int lt = (warp - (kgrp ? kKWarp0 : kVWarp0)) * 32 + lane;
        const uint32_t gbar = kgrp ? 3 : 4;
        // token ring of the group: int32 [2 blocks][128 rows], row r of block j at ring0[(j & 1) * 128 + r]
        int32_t* ring0 = reinterpret_cast<int32_t*>(smem + kOffTok) + (kgrp ? 0 : 2 * kBN);
        const CUtensorMap* xtile = kgrp ? &ktile : &vtile;
        const uint32_t xbase = kgrp ? sK : sV;
        const int lag = kgrp ? kKStages : kVStages;  // decisions <= j-lag are final when stage j is acquired
        uint64_t* xfull = kgrp ? c.k_full : c.v_full;
        uint64_t* xempty = kgrp ? c.k_empty : c.v_empty;
        uint32_t gx = 0, qcount = 0, qslot[2] = {0u, 0u};
        for (uint32_t wk = 0;; ++wk) {
            if (kgrp && lt == 0) {  // producer: the next pair index (or -1) into ring slot wk & 3
                mbar_wait(smem_u32(&c.w_empty[wk & 3]), ((wk >> 2) & 1) ^ 1, 5002);
                const int64_t v = (int64_t)atomicAdd(a.work_ctr, 1);
                *reinterpret_cast<volatile int64_t*>(&c.wq[wk & 3]) = v < total ? v : -1;
                mbar_arrive(smem_u32(&c.w_full[wk & 3]));
            }
            const int64_t it = ring_get(c, wk, lane);
            if (it < 0) break;
            const PairInfo P = pair_info(p, it);
            if (P.nb == 0) continue;
            const int32_t* kv = (P.np > 0) ? a.kv_seg(P.zh, P.n) : nullptr;
            named_bar_sync(gbar, nthr);  // every thread of the group is done with its ring
            if (kgrp && lt == 0) tl_mark(p, 30, qcount);
            if (kgrp) {
                // ---- Q, per slot: slot x's tile loads as soon as slot x of the previous pair has
                // issued its last S (its stream can end blocks before the other slot's)
                const int64_t qb = tc_q_base(p, P.zh) / rowu, qs = g.qs[2] / rowu;
                const bool q_tile = p.q_contig && !((a.mode & kStateIn) && a.q_reorder) &&
                                    (!P.has[0] || P.tn[0] == kBM) && (!P.has[1] || P.tn[1] == kBM);
                for (int x = 0; x < 2; ++x) {
                    if (!P.has[x]) continue;
                    mbar_wait(smem_u32(&c.q_empty[x]), (qslot[x] & 1) ^ 1, 1001);
                    ++qslot[x];
                    if (lt == 0) mbar_expect_tx(smem_u32(&c.q_full[x]), kTileBytes);
                    else mbar_arrive(smem_u32(&c.q_full[x]));
                    if (q_tile) {
                        if (lt == 0)
                            for (int h = 0; h < 2; ++h)
                                tma_load2d(sQ + x * kTileBytes + h * kHalf, &qtile, h * 64,
                                           (int32_t)(qb + (P.sb + P.t0[x]) * qs), smem_u32(&c.q_full[x]));
                    } else if ((lt >> 6) == x) {
                        // permuted Q rows: one TMA gather4 op per lane (row group, column half)
                        // (A/B against 16-B cp.async: pass-2 6.03 -> 5.90 ms)
                        const int grp = (lt >> 1) & 31, h = lt & 1;
                        int32_t rr[4];
                        for (int i = 0; i < 4; ++i) rr[i] = (int32_t)(qb + q_row(a, P, x, grp * 4 + i) * qs);
                        tma_gather4(sQ + x * kTileBytes + h * kHalf + grp * 512, &qmap, h * 64, rr[0], rr[1], rr[2],
                                    rr[3], smem_u32(&c.q_full[x]));
                    }
                }
                if (lt == 0) tl_mark(p, 29, qcount);
                ++qcount;
            }
            const int64_t xb = (kgrp ? tc_k_base(p, P.zh) : tc_v_base(p, P.zh)) / rowu;
            const int64_t xs = (kgrp ? g.ks[2] : g.vs[2]) / rowu;
            const auto gathered = [&](int j) { return !(j < P.ndmax && p.kv_contig); };
            // tokens of block j: entries lt and lt + nthr (< 128) in registers, one block ahead
            // (stored as tensor-map row coordinates xb + token * xs, ready for the gather ops)
            auto fetch_tok = [&](int j, int32_t (&tk)[2]) {
                for (int u = 0; u < 2; ++u) {
                    const int i = lt + u * nthr;
                    tk[u] = (i < kBN && j < P.nb && gathered(j)) ? (int32_t)(xb + key_token(P, kv, j, i) * xs) : 0;
                }
            };
            int32_t tk[2];
            fetch_tok(0, tk);
            int stop_at[2] = {1 << 30, 1 << 30};
            int known = -1;  // decisions of blocks <= known have been read
            int nx = 0;
            for (int j = 0; j < P.nb; ++j) {
                const bool gat = gathered(j);
                int32_t* ring = ring0 + (j & 1) * kBN;
                if (gat)
                    for (int u = 0; u < 2; ++u)
                        if (lt + u * nthr < kBN) ring[lt + u * nthr] = tk[u];
                fetch_tok(j + 1, tk);  // prefetch (latency overlaps the stage wait)
                if (gat) named_bar_sync(gbar, nthr);
                const uint32_t gi = gx + j;
                // stage / phase with compile-time divisors (a runtime divisor needs MUFU.RCP, which
                // queues behind the softmax warps' exponentials)
                const int st = kgrp ? (int)(gi % kKStages) : (int)(gi % kVStages);
                const uint32_t sph = kgrp ? (gi / kKStages) & 1 : (gi / kVStages) & 1;
                mbar_wait(smem_u32(&xempty[st]), sph ^ 1, kgrp ? 1002 : 1003);
                if (lt == 0) tl_mark(p, kgrp ? 9 : 1, gi);
                // stage reuse certifies both slots' decisions on blocks <= j - lag
                for (; known < j - lag;) {
                    ++known;
                    if (known >= P.ndmax)
                        for (int x = 0; x < 2; ++x)
                            if (participates(P, x, known) && stop_at[x] > known && c.dec[x][known & 3] == 2)
                                stop_at[x] = known;
                }
                bool need = false;
                for (int x = 0; x < 2; ++x) need |= participates(P, x, j) && !(stop_at[x] <= j - lag);
                if (!need) break;
                const uint32_t dst = xbase + st * kTileBytes;
                if (lt == 0) mbar_expect_tx(smem_u32(&xfull[st]), kTileBytes);
                else mbar_arrive(smem_u32(&xfull[st]));
                if (!gat) {
                    if (lt == 0) {
                        const int64_t tok = P.sb + (int64_t)j * kBN;
                        for (int h = 0; h < 2; ++h)
                            tma_load2d(dst + h * kHalf, xtile, h * 64, (int32_t)(xb + tok * xs), smem_u32(&xfull[st]));
                    }
                } else {
                    // TMA tile::gather4 (A/B: 9 % faster pass-2 than 16-B cp.async, which competes with
                    // the tensor core for the LSU/shared-memory path): 64 ops (32 row groups x 2 column
                    // halves) on lanes 0-15 (K) / 0-21 (V) of the group's warps. Per-lane operands (the
                    // compiler issues them lane by lane); an elected-lane loop over warp-uniform operands
                    // measured slower (pass-2 6.05 -> 7.09 ms at C3: the serial per-op shuffle and load
                    // latencies outweigh the waterfall).
                    const int wl = lt & 31, wi = lt >> 5;
                    const int per = kgrp ? 16 : 22;
                    const int opi = wl < per ? wi * per + wl : 64;
                    if (opi < 64) {
                        const int grp = opi >> 1, h = opi & 1;
                        const int4 t4 = *reinterpret_cast<const int4*>(ring + 4 * grp);
                        tma_gather4(dst + h * kHalf + grp * 512, kgrp ? &kmap : &vmap, h * 64, t4.x, t4.y, t4.z, t4.w,
                                    smem_u32(&xfull[st]));
                    }
                }
                if (lt == 0) tl_mark(p, kgrp ? 10 : 2, gi);
                ++nx;
            }
            gx += nx;
        }
    } else if (warp == kMmaWarp) {
        // ============================== MMA issuer ==============================
        // Ping-pong order (per block j, per slot x): wait P_x(j) -> O_x += P_x V(j) -> S_x(j+1)
        // = Q_x K(j+1)^T. The tensor pipe runs slot 1's PV/S while slot 0's softmax works and
        // vice versa. S_x(j+1) overwrites P_x(j) only after the in-order pipe consumed it.
        // Blocks loaded (must match the loader): K(j) iff need(j, kKStages), V(j) iff need(j, kVStages).
        // The whole warp runs the control flow (warp-uniform values stay in uniform registers);
        // one elected lane issues each tcgen05 instruction.
        const bool leader = elect_one();
        {
            const uint32_t idesc_s = umma_idesc_bf16(kBM, kBN, false, false);
            const uint32_t idesc_o = umma_idesc_bf16(kBM, kD, false, true);
            uint32_t gk = 0, gv = 0, qcount = 0, qslot[2] = {0u, 0u};
            uint32_t ns[2] = {0, 0};  // p_full phases per slot
            // descriptor address field is addr >> 4 in the low bits: desc(a + off) = desc(a) + off/16
            const uint64_t dq0 = umma_desc_sw128(sQ, 16, 1024);
            const uint64_t dk0 = umma_desc_sw128(sK, 16, 1024);
            const uint64_t dv0 = umma_desc_sw128(sV, kHalf, 1024);
            auto issue_s = [&](int x, int st) {
                x = __shfl_sync(0xffffffffu, x, 0);  // warp-uniform: descriptors stay in uniform registers
                st = __shfl_sync(0xffffffffu, st, 0);
                const uint64_t dq = dq0 + ((x * kTileBytes) >> 4);
                const uint64_t dk = dk0 + ((st * kTileBytes) >> 4);
#pragma unroll
                for (int kk = 0; kk < kD / 16; ++kk) {
                    const uint32_t off = ((kk / 4) * kHalf + (kk % 4) * 32) >> 4;
                    if (leader) umma_bf16(tbase + x * 256, dq + off, dk + off, idesc_s, kk > 0);
                }
                if (leader) umma_commit(smem_u32(&c.s_full[x]));
            };
            auto wait_k = [&](uint32_t gki) {
                mbar_wait(smem_u32(&c.k_full[gki % kKStages]), (gki / kKStages) & 1, 2002);
                tl_mark(p, 5, gki);
                tc_fence_after();
            };
            for (uint32_t wk = 0;; ++wk) {
                const int64_t it = ring_get(c, wk, lane);
                if (it < 0) break;
                const PairInfo P = pair_info(p, it);
                if (P.nb == 0) continue;
                tl_mark(p, 26, qcount);
                ++qcount;
                int stop_at[2] = {1 << 30, 1 << 30};
                bool pv_any[2] = {false, false};  // first P V of a slot overwrites O (accumulate = 0)
                bool qrel[2] = {!P.has[0], !P.has[1]};  // slot's Q released (after its last S)
                auto release_q = [&](int x) {
                    if (!qrel[x] && leader) umma_commit(smem_u32(&c.q_empty[x]));
                    qrel[x] = true;
                };
                auto need = [&](int j, int lag) {
                    bool n = false;
                    for (int x = 0; x < 2; ++x) n |= participates(P, x, j) && !(stop_at[x] <= j - lag);
                    return n;
                };
                wait_k(gk);
                for (int x = 0; x < 2; ++x) {
                    if (!P.has[x]) continue;
                    mbar_wait(smem_u32(&c.q_full[x]), qslot[x] & 1, 2001);
                    ++qslot[x];
                    tc_fence_after();
                    if (participates(P, x, 0)) issue_s(x, gk % kKStages);
                    if (last_block(P, x) == 0) release_q(x);
                }
                tl_mark(p, 27, qcount - 1);
                int nk = 0, nv = 0;
                for (int j = 0;; ++j) {
                    const uint32_t gki = gk + j, gvi = gv + j;
                    const bool has_v = need(j, kVStages);
                    const bool has_kn = (j + 1 < P.nb) && need(j + 1, kKStages);
                    bool v_ready = false, kn_ready = false;
                    for (int x = 0; x < 2; ++x) {
                        if (participates(P, x, j) && stop_at[x] > j - 1) {
                            mbar_wait(smem_u32(&c.p_full[x]), ns[x] & 1, 2004);
                            tl_mark(p, 6 + x, gki);
                            ++ns[x];
                            tc_fence_after();
                            const bool commit = j < P.ndmax || chunk_commit(c.red[x][j & 1]);
                            __syncwarp();
                            if (leader) c.dec[x][j & 3] = commit ? 1 : 2;  // for the loaders' stop tracking
                            if (commit) {
                                if (!v_ready) {
                                    mbar_wait(smem_u32(&c.v_full[gvi % kVStages]), (gvi / kVStages) & 1, 2005);
                                    tl_mark(p, 28, gki);
                                    tc_fence_after();
                                    v_ready = true;
                                }
                                const int vst = __shfl_sync(0xffffffffu, (int)(gvi % kVStages), 0);
                                const int xu = __shfl_sync(0xffffffffu, x, 0);
                                const uint64_t dv = dv0 + ((vst * kTileBytes) >> 4);
#pragma unroll
                                for (int kk = 0; kk < kBN / 16; ++kk)
                                    if (leader)
                                        umma_bf16_ts(tbase + xu * 256 + 128, tbase + xu * 256 + kk * 8,
                                                     dv + ((kk * 16 * 128) >> 4), idesc_o, (kk > 0 || pv_any[x]) ? 1 : 0);
                                pv_any[x] = true;
                                if (leader && j == last_block(P, x)) umma_commit(smem_u32(&c.o_done[x]));
                            } else {
                                stop_at[x] = j;
                                release_q(x);  // no further S of this slot
                                if (leader) umma_commit(smem_u32(&c.o_done[x]));  // slot finished
                            }
                        }
                        if (has_kn && participates(P, x, j + 1) && stop_at[x] > j) {
                            if (!kn_ready) {
                                wait_k(gki + 1);
                                kn_ready = true;
                            }
                            issue_s(x, (gki + 1) % kKStages);
                            if (j + 1 == last_block(P, x)) release_q(x);
                            if (x == 0) tl_mark(p, 31, gki);
                        }
                    }
                    if (has_v && !v_ready) mbar_wait(smem_u32(&c.v_full[gvi % kVStages]), (gvi / kVStages) & 1, 2006);
                    // both slots' decisions on block j are read: the loader may reuse its stages
                    if (leader) {
                        umma_commit(smem_u32(&c.k_empty[gki % kKStages]));
                        if (has_v) umma_commit(smem_u32(&c.v_empty[gvi % kVStages]));
                    }
                    tl_mark(p, 8, gki);
                    ++nk;
                    nv += has_v ? 1 : 0;
                    if (!has_kn) break;
                    if (!kn_ready) wait_k(gki + 1);
                }
                release_q(0);  // (slots whose stream ended without reaching their last block)
                release_q(1);
                gk += nk;
                gv += nv;
            }
        }
        __syncwarp();
    } else {
        // ============================== softmax / epilogue (slot x) ==============================
        setmaxnreg_inc<kSoftmaxRegs>();
        const int x = warp / 4;
        const int r = threadIdx.x % 128;  // TMEM lane
        const uint32_t lane_off = (uint32_t)((warp % 4) * 32) << 16;
        const uint32_t tS = tbase + lane_off + x * 256;
        const uint32_t tO = tS + 128;
        const uint32_t bar_id = 1 + x;
        const float sc = p.scale_log2;
        uint32_t ns = 0, no = 0, npf = 0;
        for (uint32_t wk = 0;; ++wk) {
            const int64_t it = ring_get(c, wk, lane);
            if (it < 0) break;
            float m2, ell;
            float sacc = 1.0f;    // scale of the resumed accumulator (kStateIn)
            bool pv_any = false;  // a P V has been issued into O_x for this pair
            int committed = 0, pairs = 0;
            bool any = false;
            const bool tl_on = r == 0;
            {
            // 32-bit copies of what the block loop needs (keeps the 128 scores in registers)
            const PairInfo P = pair_info(p, it);
            if (!P.has[x]) continue;
            if (tl_on) tl_mark(p, 11 + 4 * x, no);
            const int nd_x = P.nd[x], ndmax = P.ndmax, nb = P.nb;
            const int t0x = (int)P.t0[x], segr = (int)P.seg_rows, avail = (int)P.avail;
            const bool valid = r < P.tn[x];
            const int64_t slot = P.zh * g.l + q_row(a, P, x, r);
            // ---- state init: (m, ell) in registers. O in TMEM starts from the first P V (issued
            // with accumulate = 0); a resumed pass-1 accumulator is added in the epilogue with the
            // product of the rescale factors applied since (sacc), so its HBM read is off the
            // critical path (L2 prefetch now, load at the end).
            if (a.mode & kStateIn) {
                m2 = a.m_in[slot] * 1.4426950408889634f;
                ell = a.ell_in[slot];
                const char* arow = reinterpret_cast<const char*>(a.acc_in + slot * kD);
#pragma unroll
                for (int i = 0; i < 4; ++i) asm volatile("prefetch.global.L2 [%0];" ::"l"(arow + 128 * i));
            } else {
                m2 = -INFINITY;
                ell = 0.0f;
            }
            if (tl_on) tl_mark(p, 12 + 4 * x, no);

            for (int j = 0; j < nb; ++j) {
                if (j < ndmax && j >= nd_x) continue;  // !participates
                any = true;
                mbar_wait(smem_u32(&c.s_full[x]), ns & 1, 3001);
                if (tl_on) tl_mark(p, 19 + 3 * x, ns);
                ++ns;
                tc_fence_after();
                // ---- all 128 scores of this row in registers (one TMEM round trip)
                uint32_t sv[kBN];
#pragma unroll
                for (int c0 = 0; c0 < kBN; c0 += 32) tmem_ld32(tS + c0, *reinterpret_cast<uint32_t(*)[32]>(&sv[c0]));
                tmem_ld_wait();
                if (tl_on && x == 0) tl_mark(p, 25, ns - 1);
                // ---- visible keys of this block for this row
                const bool is_diag = j < ndmax;
                int lim;
                if (is_diag) {
                    const int k0 = j * kBN;
                    const int kn = min(kBN, segr - k0);
                    const int vis = (k0 + kn - 1 <= t0x) ? kn : min(kn, t0x + r - k0 + 1);
                    lim = max(0, vis);
                } else {
                    lim = min(kBN, avail - (j - ndmax) * kBN);
                }
                const bool full = __all_sync(0xffffffffu, lim >= kBN);
                float m_use, alpha;
                bool rescale;
                float rs[4] = {0.0f, 0.0f, 0.0f, 0.0f};
                {
                    float mxa[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) mxa[i] = -INFINITY;
                    // three-input max (FMNMX3): 64 instructions for the 128 scores
                    if (full) {
#pragma unroll
                        for (int i = 0; i < kBN; i += 2)
                            mxa[(i >> 1) & 7] = fmax3(mxa[(i >> 1) & 7], __uint_as_float(sv[i]), __uint_as_float(sv[i + 1]));
                    } else {
#pragma unroll
                        for (int i = 0; i < kBN; i += 2)
                            mxa[(i >> 1) & 7] = fmax3(mxa[(i >> 1) & 7], i < lim ? __uint_as_float(sv[i]) : -INFINITY,
                                                      i + 1 < lim ? __uint_as_float(sv[i + 1]) : -INFINITY);
                    }
                    const float mx = fmax3(fmax3(mxa[0], mxa[1], mxa[2]), fmax3(mxa[3], mxa[4], mxa[5]),
                                           fmaxf(mxa[6], mxa[7])) * sc;
                    const float m_new = fmaxf(m2, mx);
                    // early_stop_check's "uninitialized state" (kernel.cpp:228): the reference's
                    // fp64 prev = ell * e^(m - m') is <= 0 iff ell <= 0 or e^(m - m') underflows
                    // fp64 (a max jump beyond 1075 log2 units) -- unless ell is NaN or infinite
                    // (a poisoned row: prev is NaN, which the reference does not reject)
                    if (!is_diag && valid && fabsf(ell) <= 3.402823466e38f && (ell <= 0.0f || m_new - m2 > 1075.0f))
                        atomicExch(a.err_flag, 1);
                    rescale = (m_new > m2 + kRescaleThresh) || (m2 == -INFINITY);
                    m_use = rescale ? m_new : m2;
                    const float neg_ref = (m_use == -INFINITY) ? 0.0f : -m_use;
                    alpha = (m2 == -INFINITY) ? 0.0f : ex2(m2 + neg_ref);
                    // P = exp2(s*scale - m) in bf16 over the first 64 S columns. (All on MUFU: an
                    // FMA-pipe polynomial for part of the row measured slower -- the softmax is
                    // latency- not MUFU-throughput-bound here, profiles/r01_summary.md.)
                    if (full) {
                        if constexpr (kPackedExp) {
                            // packed arguments and sums (FFMA2 / FADD2): A/B at C3 pass-2 -5.5 %, pass-1
                            // +5 % (so pass-1 launches the scalar instance)
                            const float2 sc2 = make_float2(sc, sc), nr2 = make_float2(neg_ref, neg_ref);
                            float2 rs2[2] = {make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f)};
#pragma unroll
                            for (int c0 = 0; c0 < kBN; c0 += 32) {
                                uint32_t pk[16];
#pragma unroll
                                for (int i = 0; i < 32; i += 2) {
                                    const float2 arg = ffma2(make_float2(__uint_as_float(sv[c0 + i]), __uint_as_float(sv[c0 + i + 1])),
                                                             sc2, nr2);
                                    const float2 e = make_float2(ex2(arg.x), ex2(arg.y));
                                    rs2[(i >> 1) & 1] = fadd2(rs2[(i >> 1) & 1], e);
                                    pk[i >> 1] = pack_bf16(e.x, e.y);
                                }
                                tmem_st16(tS + c0 / 2, pk);
                            }
                            rs[0] = rs2[0].x;
                            rs[1] = rs2[0].y;
                            rs[2] = rs2[1].x;
                            rs[3] = rs2[1].y;
                        } else {
#pragma unroll
                            for (int c0 = 0; c0 < kBN; c0 += 32) {
                                uint32_t pk[16];
#pragma unroll
                                for (int i = 0; i < 32; i += 2) {
                                    const float e0 = ex2(fmaf(__uint_as_float(sv[c0 + i]), sc, neg_ref));
                                    const float e1 = ex2(fmaf(__uint_as_float(sv[c0 + i + 1]), sc, neg_ref));
                                    rs[(i >> 1) & 3] += e0 + e1;
                                    pk[i >> 1] = pack_bf16(e0, e1);
                                }
                                tmem_st16(tS + c0 / 2, pk);
                            }
                        }
                    } else {
#pragma unroll
                        for (int c0 = 0; c0 < kBN; c0 += 32) {
                            uint32_t pk[16];
#pragma unroll
                            for (int i = 0; i < 32; i += 2) {
                                const float e0 = c0 + i < lim ? ex2(fmaf(__uint_as_float(sv[c0 + i]), sc, neg_ref)) : 0.0f;
                                const float e1 = c0 + i + 1 < lim ? ex2(fmaf(__uint_as_float(sv[c0 + i + 1]), sc, neg_ref)) : 0.0f;
                                rs[(i >> 1) & 3] += e0 + e1;
                                pk[i >> 1] = pack_bf16(e0, e1);
                            }
                            tmem_st16(tS + c0 / 2, pk);
                        }
                    }
                }
                const float rowsum = (rs[0] + rs[1]) + (rs[2] + rs[3]);
                // O rescale after the scores are dead (P V(j-1) is complete: s_full orders after it;
                // P V(j) is issued only after p_full)
                if (rescale) sacc *= alpha;
                if (__any_sync(0xffffffffu, pv_any && rescale && m2 != -INFINITY)) {
#pragma unroll
                    for (int c0 = 0; c0 < kD; c0 += 32) {
                        uint32_t v[32];
                        tmem_ld32(tO + c0, v);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
                        tmem_st32(tO + c0, v);
                    }
                }
                if (tl_on) tl_mark(p, 20 + 3 * x, ns - 1);
                // relative normaliser gain of this chunk (kernel.cpp:108-115): per-warp max into
                // red[] (double-buffered by block parity), then one arrive per warp on p_full; the
                // MMA issuer and these warps both take the decision from the four warp maxima
                // (gain >= tau  <=>  rowsum >= tau * prev; NaN rows never vote to continue)
                bool my_vote = false;
                if (!is_diag) {
                    const bool cont = valid && (rowsum >= (float)a.tau * (ell * alpha));
                    my_vote = __ballot_sync(0xffffffffu, cont) != 0u;
                    if (lane == 0) c.red[x][j & 1][warp % 4] = my_vote;
                }
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&c.p_full[x]));
                // a warp that voted to continue already knows the chunk commits (the decision is
                // an OR); only a warp that voted stop waits for the other three votes
                bool commit = true;
                if (!is_diag && !my_vote) {
                    mbar_wait(smem_u32(&c.p_full[x]), npf & 1, 3002);
                    commit = chunk_commit(c.red[x][j & 1]);
                }
                ++npf;
                // state update (on a stop the rescaled state is the same state: O/ell unchanged)
                ell = commit ? ell * alpha + rowsum : ell * alpha;
                pv_any |= commit;
                m2 = m_use;
                if (commit && !is_diag) {
                    ++committed;
                    pairs += min(kBN, avail - (j - ndmax) * kBN);
                }
                if (tl_on) tl_mark(p, 21 + 3 * x, ns - 1);
                if (!commit) break;
            }
            }  // block loop scope
            const PairInfo P = pair_info(p, it);
            const bool valid = r < P.tn[x];
            const int64_t grow = q_row(a, P, x, r);
            const int64_t slot = P.zh * g.l + grow;
            if (any) {
                mbar_wait(smem_u32(&c.o_done[x]), no & 1, 3004);
                ++no;
                tc_fence_after();
            }
            if (tl_on) tl_mark(p, 13 + 4 * x, no);
            // ---- read O, finalize / persist
            uint32_t ov[kD];
#pragma unroll
            for (int c0 = 0; c0 < kD; c0 += 32) tmem_ld32(tO + c0, *reinterpret_cast<uint32_t(*)[32]>(&ov[c0]));
            tmem_ld_wait();
            if (!pv_any) {
#pragma unroll
                for (int i = 0; i < kD; ++i) ov[i] = 0u;
            }
            if (a.mode & kStateIn) {
                if (p.vec_acc) {
                    const float* src = a.acc_in + slot * kD;
#pragma unroll
                    for (int i0 = 0; i0 < kD; i0 += 32) {  // 4 x 256-bit loads in flight per round
                        uint32_t y[4][8];
#pragma unroll
                        for (int u = 0; u < 4; ++u) ldg256(src + i0 + 8 * u, y[u]);
#pragma unroll
                        for (int u = 0; u < 4; ++u)
#pragma unroll
                            for (int e = 0; e < 8; ++e)
                                ov[i0 + 8 * u + e] = __float_as_uint(
                                    fmaf(__uint_as_float(y[u][e]), sacc, __uint_as_float(ov[i0 + 8 * u + e])));
                    }
                } else {
                    const float4* src = reinterpret_cast<const float4*>(a.acc_in + slot * kD);
#pragma unroll
                    for (int i = 0; i < kD / 4; ++i) {
                        const float4 y = src[i];
                        ov[4 * i] = __float_as_uint(fmaf(y.x, sacc, __uint_as_float(ov[4 * i])));
                        ov[4 * i + 1] = __float_as_uint(fmaf(y.y, sacc, __uint_as_float(ov[4 * i + 1])));
                        ov[4 * i + 2] = __float_as_uint(fmaf(y.z, sacc, __uint_as_float(ov[4 * i + 2])));
                        ov[4 * i + 3] = __float_as_uint(fmaf(y.w, sacc, __uint_as_float(ov[4 * i + 3])));
                    }
                }
            }
            const float inv = 1.0f / ell;
            // A tile that walked its whole (truncated) kv list without stopping continues at
            // the next plan level: its state is saved in place of the resumed one, no output yet.
            const bool overflow = (a.mode & kPrefix) && P.np > 0 && committed == P.np && a.truncated(P.n);
            const bool resume_later = overflow && a.acc_out != nullptr;
            const bool save_state = (a.mode & kStateOut) || resume_later;
            if (valid && save_state) {
                if (p.vec_acc) {
                    float* dst = a.acc_out + slot * kD;
#pragma unroll
                    for (int i = 0; i < kD; i += 8) stg256(dst + i, &ov[i]);
                } else {
                    float4* dst = reinterpret_cast<float4*>(a.acc_out + slot * kD);
#pragma unroll
                    for (int i = 0; i < kD / 4; ++i)
                        dst[i] = make_float4(__uint_as_float(ov[4 * i]), __uint_as_float(ov[4 * i + 1]),
                                             __uint_as_float(ov[4 * i + 2]), __uint_as_float(ov[4 * i + 3]));
                }
            }
            if (valid && (a.mode & kFinal) && !resume_later) {
                const int64_t ooff = tc_o_base(p, P.zh) + grow * g.os[2];
                if (g.out_bf16 && p.vec_o) {
                    __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(a.o) + ooff;
#pragma unroll
                    for (int i = 0; i < kD; i += 16) {
                        uint32_t w[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e)
                            w[e] = pack_bf16(__uint_as_float(ov[i + 2 * e]) * inv, __uint_as_float(ov[i + 2 * e + 1]) * inv);
                        stg256(dst + i, w);
                    }
                } else if (g.out_bf16) {
                    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.o) + ooff);
#pragma unroll
                    for (int i = 0; i < kD / 8; ++i) {
                        uint4 w;
                        w.x = pack_bf16(__uint_as_float(ov[8 * i]) * inv, __uint_as_float(ov[8 * i + 1]) * inv);
                        w.y = pack_bf16(__uint_as_float(ov[8 * i + 2]) * inv, __uint_as_float(ov[8 * i + 3]) * inv);
                        w.z = pack_bf16(__uint_as_float(ov[8 * i + 4]) * inv, __uint_as_float(ov[8 * i + 5]) * inv);
                        w.w = pack_bf16(__uint_as_float(ov[8 * i + 6]) * inv, __uint_as_float(ov[8 * i + 7]) * inv);
                        dst[i] = w;
                    }
                } else {
                    float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(a.o) + ooff);
#pragma unroll
                    for (int i = 0; i < kD / 4; ++i)
                        dst[i] = make_float4(__uint_as_float(ov[4 * i]) * inv, __uint_as_float(ov[4 * i + 1]) * inv,
                                             __uint_as_float(ov[4 * i + 2]) * inv, __uint_as_float(ov[4 * i + 3]) * inv);
                }
            }
            if (valid && save_state) {
                a.m_out[slot] = (m2 == -INFINITY) ? -INFINITY : m2 * 0.6931471805599453f;
                a.ell_out[slot] = ell;
            }
            if (valid && (a.mode & kFinal) && !resume_later && ell == 0.0f) atomicExch(a.err_flag, 2);
            if ((a.mode & kPrefix) && r == 0) {
                const int64_t tile = P.zh * a.tiles_per_head + P.n * a.T + P.ti[x];
                const int base = a.tile_base ? a.tile_base[it] : 0;
                if (overflow) {
                    const int s2 = atomicAdd(a.ovf_count, 1);
                    a.ovf_tiles[s2] = (int32_t)tile;
                    if (a.ovf_base) a.ovf_base[s2] = base + committed;
                } else {
                    a.processed[(P.zh * g.N + P.n) * a.T + P.ti[x]] = base + committed;
                }
                // (without a saved state the overflow tile is recomputed from scratch: no pairs)
                if (pairs && (!overflow || resume_later))
                    atomicAdd((unsigned long long*)&a.pass2_pairs[P.zh], (unsigned long long)pairs * P.tn[x]);
            }
            if (tl_on) tl_mark(p, 14 + 4 * x, no);
            tc_fence_before();
            named_bar_sync(bar_id, 128);  // all rows done with O before the next pair's init
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) tl_cta(p, 3);
    if (warp == 0) tmem_dealloc(tbase, kTmemCols);
}

// ============================================================== single-tile diagonal kernel
// Pass-1 (and any diagonal-only pass: the dense reference with S = L) on ONE 128-row query tile
// per work item, with the score buffer triple-buffered in TMEM: S(j+1), S(j+2) are computed while
// the softmax of block j runs, so the softmax warps run block after block without waiting on
// P V(j) + S(j+1) (the pair kernel's per-slot chain: softmax -> P V -> S -> softmax). The pair
// kernel shares a K/V block between two tiles, which matters for gathered prefix chunks; the
// diagonal blocks are contiguous 2-D TMA tiles served from L2, so one tile per item costs little.
//
//   warps 0-7   softmax: warp w < 4 takes key columns [0, 64) of rows 32w.. (TMEM lanes), warp
//               w + 4 columns [64, 128) of the same rows; the row max is exchanged in smem
//   warps 8-11  epilogue: read O of a finished tile from TMEM, persist state / write O, so the
//               softmax warps go straight on to the next tile
//   warp 12     MMA issuer (one elected lane)
//   warp 13     Q + K loader (lane 0, 2-D TMA tiles), warp 14 V loader (lane 0), warp 15 reads
//               (idle: the masked-key poison check is poison_scan_kernel)
//
// TMEM: S buffers at columns [0, 128), [128, 256), [256, 384) (P in bf16 over the first 64
// columns of its buffer), O at [384, 512) (kDSBuf = 2: two S buffers, O double-buffered by
// tile). Blocks are numbered globally per CTA (gb); block gb uses S buffer gb % kDSBuf. MMA
// order: S(0..kDSBuf-1), then per block j: P V(j), S(j+kDSBuf) (into the buffer P(j) held; the
// tensor pipe executes in order, so the new S overwrites P(j) only after P V(j) read it).
// A softmax that must rescale O at block gb (lazy max update, rare) first waits for P V(gb-1),
// i.e. all earlier P V of the tile, on the V stage barrier that P V commits (v_empty).
#ifndef S2O_DIAG_POLY
#define S2O_DIAG_POLY 8  // diagonal kernel: every n-th exponential pair on the FMA pipe (0 = all MUFU; A/B: 8 -3 %, 4 even)
#endif
#ifndef S2O_DIAG_SBUF
#define S2O_DIAG_SBUF 3  // S buffers in TMEM (3: single O buffer; 2: O double-buffered by tile)
#endif
constexpr int kDSBuf = S2O_DIAG_SBUF;
constexpr int kDOBuf = kDSBuf == 3 ? 1 : 2;
static_assert(kDSBuf * 128 + kDOBuf * 128 <= 512, "TMEM columns");
constexpr int kDThreads = 512;
constexpr int kDSoftWarps = 8, kDEpiWarp0 = 8, kDMmaWarp = 12, kDKWarp = 13, kDVWarp = 14;
constexpr int kDEpiRegs = 160, kDOtherRegs = 56;  // setmaxnreg (softmax warpgroups keep 128)
constexpr int kDKStages = 2, kDVStages = 2;
static_assert(kDKStages == kDVStages, "the diagonal loaders share one stage index");
constexpr int kDQBuf = 2;  // Q double-buffered by tile parity: the next tile's Q lands during this one
constexpr uint32_t kDOffQ = 0;
constexpr uint32_t kDOffK = kDQBuf * kTileBytes;
constexpr uint32_t kDOffV = kDOffK + kDKStages * kTileBytes;
constexpr uint32_t kDOffCtrl = kDOffV + kDVStages * kTileBytes;
constexpr uint32_t kDOffML = kDOffCtrl + 256;  // float [2 tile parity][m, ell half 0, ell half 1][128 rows]
constexpr uint32_t kDOffX = kDOffML + 2 * 3 * 128 * 4;  // float [2 block parity][2 halves][128 rows]: row max
constexpr uint32_t kDSmemBytes = kDOffX + 2 * 2 * 128 * 4;  // 197.25 KB

struct CtrlD {
    uint64_t q_full[kDQBuf], q_empty[kDQBuf];
    uint64_t k_full[kDKStages], k_empty[kDKStages], v_full[kDVStages], v_empty[kDVStages];
    uint64_t s_full[kDSBuf], p_full[kDSBuf];                    // per S buffer
    uint64_t o_done[kDOBuf], o_free[kDOBuf];                    // per O buffer
    uint64_t ml_full[2], ml_free[2];                            // (m, ell) hand-off slots (tile parity)
    uint32_t tmem_base;
};
static_assert(sizeof(CtrlD) <= 256, "CtrlD exceeds its 256 B");

struct TileInfo {
    int64_t zh, n, sb, t0;
    int tn, segr, nd;
};

// Work item idx -> (head, segment, tile). The q heads of a GQA group are interleaved (they read
// the same K/V rows, which then hit L2 together); within a head the longest tiles come first.
__device__ __forceinline__ TileInfo diag_tile(const TcParams& p, int64_t idx) {
    const Geo& g = p.a.g;
    const int64_t T = p.a.T, G = g.group;
    const int64_t tiles_head = p.pairs_per_head;  // tiles per head (launcher)
    const int64_t zg = idx / (tiles_head * G);
    const int64_t rem = idx % (tiles_head * G);
    TileInfo t;
    t.zh = zg * G + rem % G;
    int64_t r = rem / G;
    const int64_t t_last = (g.last_len + kBM - 1) / kBM;
    const int64_t full = (g.N - 1) * T;
    // longest first: reverse the tile order inside a segment
    if (r < full) { t.n = r / T; r = T - 1 - r % T; }
    else { t.n = g.N - 1; r = t_last - 1 - (r - full); }
    t.sb = t.n * g.S;
    t.segr = (int)g.seg_rows(t.n);
    t.t0 = r * kBM;
    t.tn = (int)min((int64_t)kBM, (int64_t)t.segr - t.t0);
    t.nd = (int)((t.t0 + t.tn - 1) / kBN + 1);
    return t;
}

__global__ void __launch_bounds__(kDThreads, 1)
tc_diag_kernel(const TcParams p, const __grid_constant__ CUtensorMap qtile,
               const __grid_constant__ CUtensorMap ktile, const __grid_constant__ CUtensorMap vtile) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw;
    if ((smem_u32(smem) & 1023u) != 0) __trap();
    CtrlD& c = *reinterpret_cast<CtrlD*>(smem + kDOffCtrl);
    const PassArgs& a = p.a;
    const Geo& g = a.g;
    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const uint32_t sQ = smem_u32(smem + kDOffQ);
    const uint32_t sK = smem_u32(smem + kDOffK);
    const uint32_t sV = smem_u32(smem + kDOffV);
    if (threadIdx.x == 0) {
        for (int b = 0; b < kDQBuf; ++b) {
            mbar_init(smem_u32(&c.q_full[b]), 1);
            mbar_init(smem_u32(&c.q_empty[b]), 1);
        }
        for (int s = 0; s < kDKStages; ++s) {
            mbar_init(smem_u32(&c.k_full[s]), 1);
            mbar_init(smem_u32(&c.k_empty[s]), 1);
        }
        for (int s = 0; s < kDVStages; ++s) {
            mbar_init(smem_u32(&c.v_full[s]), 1);
            mbar_init(smem_u32(&c.v_empty[s]), 1);
        }
        for (int b = 0; b < kDSBuf; ++b) {
            mbar_init(smem_u32(&c.s_full[b]), 1);
            mbar_init(smem_u32(&c.p_full[b]), kDSoftWarps);  // both row halves
        }
        for (int b = 0; b < kDOBuf; ++b) {
            mbar_init(smem_u32(&c.o_done[b]), 1);
            mbar_init(smem_u32(&c.o_free[b]), 4);   // epilogue warps
        }
        for (int b = 0; b < 2; ++b) {
            // per-thread arrivals: every writer / reader of the slot releases its own accesses
            mbar_init(smem_u32(&c.ml_full[b]), kDSoftWarps * 32);
            mbar_init(smem_u32(&c.ml_free[b]), 4 * 32);  // epilogue threads
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
    const int64_t total = g.z * g.hq * p.pairs_per_head;
    constexpr int64_t rowu = kD;  // (tc path: d == 128)
    float* ml = reinterpret_cast<float*>(smem + kDOffML);
    float* xch = reinterpret_cast<float*>(smem + kDOffX);
    // (setmaxnreg inside each role branch, so the softmax code is dominated by its increase)
    if (warp == kDKWarp || warp == kDVWarp || warp > kDVWarp) {
        setmaxnreg_dec<kDOtherRegs>();
        if (warp > kDVWarp) return;  // (the masked-key poison check is poison_scan_kernel)
        // ============================== loaders (one lane each) ==============================
        if (lane != 0) return;
        const bool kl = warp == kDKWarp;
        const CUtensorMap* xtile = kl ? &ktile : &vtile;
        const uint32_t xbase = kl ? sK : sV;
        uint64_t* xfull = kl ? c.k_full : c.v_full;
        uint64_t* xempty = kl ? c.k_empty : c.v_empty;
        uint32_t gi = 0, qc = 0;
        for (int64_t it = blockIdx.x; it < total; it += gridDim.x) {
            const TileInfo t = diag_tile(p, it);
            if (kl) {
                const uint32_t qb_i = qc % kDQBuf;
                mbar_wait(smem_u32(&c.q_empty[qb_i]), ((qc / kDQBuf) & 1) ^ 1, 4001);
                mbar_expect_tx(smem_u32(&c.q_full[qb_i]), kTileBytes);
                const int64_t qb = tc_q_base(p, t.zh) / rowu;
                for (int h = 0; h < 2; ++h)
                    tma_load2d(sQ + qb_i * kTileBytes + h * kHalf, &qtile, h * 64, (int32_t)(qb + t.sb + t.t0),
                               smem_u32(&c.q_full[qb_i]));
                ++qc;
            }
            const int64_t xb = (kl ? tc_k_base(p, t.zh) : tc_v_base(p, t.zh)) / rowu;
            for (int j = 0; j < t.nd; ++j, ++gi) {
                const int st = (int)(gi % kDKStages);  // (kDKStages == kDVStages)
                mbar_wait(smem_u32(&xempty[st]), ((gi / kDKStages) & 1) ^ 1, kl ? 4002 : 4003);
                mbar_expect_tx(smem_u32(&xfull[st]), kTileBytes);
                const uint32_t dst = xbase + st * kTileBytes;
                for (int h = 0; h < 2; ++h)
                    tma_load2d(dst + h * kHalf, xtile, h * 64, (int32_t)(xb + t.sb + (int64_t)j * kBN),
                               smem_u32(&xfull[st]));
            }
        }
        return;
    }
    if (warp == kDMmaWarp) {
        // ============================== MMA issuer ==============================
        setmaxnreg_dec<kDOtherRegs>();
        const bool leader = elect_one();
        const uint32_t idesc_s = umma_idesc_bf16(kBM, kBN, false, false);
        const uint32_t idesc_o = umma_idesc_bf16(kBM, kD, false, true);
        const uint64_t dq0 = umma_desc_sw128(sQ, 16, 1024);
        uint64_t dq = dq0;
        const uint64_t dk0 = umma_desc_sw128(sK, 16, 1024);
        const uint64_t dv0 = umma_desc_sw128(sV, kHalf, 1024);
        uint32_t gb = 0, qc = 0, tk = 0;
        auto issue_s = [&](uint32_t blk) {  // S(blk) into buffer blk & 1; K(blk) from stage blk % 3
            const uint32_t st = blk % kDKStages;
            mbar_wait(smem_u32(&c.k_full[st]), (blk / kDKStages) & 1, 4101);
            tc_fence_after();
            const uint64_t dk = dk0 + ((st * kTileBytes) >> 4);
#pragma unroll
            for (int kk = 0; kk < kD / 16; ++kk) {
                const uint32_t off = ((kk / 4) * kHalf + (kk % 4) * 32) >> 4;
                if (leader) umma_bf16(tbase + (blk % kDSBuf) * 128, dq + off, dk + off, idesc_s, kk > 0);
            }
            if (leader) {
                umma_commit(smem_u32(&c.s_full[blk % kDSBuf]));
                umma_commit(smem_u32(&c.k_empty[st]));
            }
            __syncwarp();
        };
        for (int64_t it = blockIdx.x; it < total; it += gridDim.x) {
            const TileInfo t = diag_tile(p, it);
            const uint32_t g0 = gb;
            const uint32_t qb_i = qc % kDQBuf;
            mbar_wait(smem_u32(&c.q_full[qb_i]), (qc / kDQBuf) & 1, 4102);
            dq = dq0 + ((qb_i * kTileBytes) >> 4);
            ++qc;
            for (int j = 0; j < t.nd && j < kDSBuf; ++j) issue_s(g0 + j);
            if (t.nd <= kDSBuf && leader) umma_commit(smem_u32(&c.q_empty[qb_i]));
            const uint32_t ob = tk % kDOBuf;
            for (int j = 0; j < t.nd; ++j) {
                const uint32_t blk = g0 + j;
                mbar_wait(smem_u32(&c.p_full[blk % kDSBuf]), (blk / kDSBuf) & 1, 4103);
                tl_mark(p, 6, blk);
                // the epilogue of the tile that used this O buffer last (tk - kDOBuf) read it
                if (j == 0) mbar_wait(smem_u32(&c.o_free[ob]), ((tk / kDOBuf) & 1) ^ 1, 4105);
                const uint32_t vst = blk % kDVStages;
                mbar_wait(smem_u32(&c.v_full[vst]), (blk / kDVStages) & 1, 4104);
                tc_fence_after();
                const uint64_t dv = dv0 + ((vst * kTileBytes) >> 4);
#pragma unroll
                for (int kk = 0; kk < kBN / 16; ++kk)
                    if (leader)
                        umma_bf16_ts(tbase + (kDSBuf + ob) * 128, tbase + (blk % kDSBuf) * 128 + kk * 8,
                                     dv + ((kk * 16 * 128) >> 4), idesc_o, (kk > 0 || j > 0) ? 1 : 0);
                if (leader) {
                    umma_commit(smem_u32(&c.v_empty[vst]));
                    if (j == t.nd - 1) umma_commit(smem_u32(&c.o_done[ob]));
                }
                __syncwarp();
                tl_mark(p, 7, blk);
                if (j + kDSBuf < t.nd) {
                    issue_s(blk + kDSBuf);  // into the buffer P(j) held: the pipe runs P V(j) first
                    tl_mark(p, 31, blk + kDSBuf);
                    if (j + kDSBuf == t.nd - 1 && leader) umma_commit(smem_u32(&c.q_empty[qb_i]));
                }
            }
            gb += t.nd;
            ++tk;
        }
        __syncwarp();
    } else if (warp < kDSoftWarps) {
        // ============================== softmax ==============================
        // Two warps per row quarter: warp w (w < 4) takes key columns [0, 64) of rows 32w.., warp
        // w + 4 columns [64, 128), so every SMSP runs two softmax warps. The row max is exchanged
        // through shared memory (named barrier per warp pair); both halves then use the same
        // reference, so each keeps a partial ell and the epilogue adds them.
        const int h = warp >> 2, q = warp & 3;
        const int r = q * 32 + lane;  // TMEM lane = row
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const uint32_t tS0 = tbase + lane_off;
        const float sc = p.scale_log2;
        uint32_t gb = 0, tk = 0;
        for (int64_t it = blockIdx.x; it < total; it += gridDim.x, ++tk) {
            const TileInfo t = diag_tile(p, it);
            const bool valid = r < t.tn;
            const int rr = valid ? r : 0;
            const uint32_t tO = tS0 + (kDSBuf + tk % kDOBuf) * 128 + h * 64;
            float m2 = -INFINITY, ell = 0.0f;
            const int t0x = (int)t.t0;
            for (int j = 0; j < t.nd; ++j, ++gb) {
                const uint32_t tS = tS0 + (gb % kDSBuf) * 128;
                mbar_wait(smem_u32(&c.s_full[gb % kDSBuf]), (gb / kDSBuf) & 1, 4201);
                if (threadIdx.x == 0) tl_mark(p, 19, gb);  // timeline (S2O_TIMELINE builds only)
                tc_fence_after();
                uint32_t sv[64];
                tmem_ld32(tS + h * 64, *reinterpret_cast<uint32_t(*)[32]>(&sv[0]));
                tmem_ld32(tS + h * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&sv[32]));
                tmem_ld_wait();
                // visible keys of this row in block j (causal on segment positions, kernel.cpp:58-69),
                // relative to this half's first key
                const int k0 = j * kBN;
                const int kn = min(kBN, t.segr - k0);
                const int vis = (k0 + kn - 1 <= t0x) ? kn : min(kn, t0x + rr - k0 + 1);
                const int lim = max(0, vis) - h * 64;
                const bool full = __all_sync(0xffffffffu, lim >= 64);
                float mxa[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) mxa[i] = -INFINITY;
                if (full) {
#pragma unroll
                    for (int i = 0; i < 64; i += 2)
                        mxa[(i >> 1) & 7] = fmax3(mxa[(i >> 1) & 7], __uint_as_float(sv[i]), __uint_as_float(sv[i + 1]));
                } else {
#pragma unroll
                    for (int i = 0; i < 64; i += 2)
                        mxa[(i >> 1) & 7] = fmax3(mxa[(i >> 1) & 7], i < lim ? __uint_as_float(sv[i]) : -INFINITY,
                                                  i + 1 < lim ? __uint_as_float(sv[i + 1]) : -INFINITY);
                }
                float mx = fmax3(fmax3(mxa[0], mxa[1], mxa[2]), fmax3(mxa[3], mxa[4], mxa[5]), fmaxf(mxa[6], mxa[7]));
                // exchange with the other half (double-buffered by block parity): after this barrier
                // both halves have also finished reading S, so P may overwrite it
                float* xb = xch + (gb & 1) * 256;
                xb[h * 128 + r] = mx;
                named_bar_sync(1 + q, 64);
                mx = fmaxf(mx, xb[(1 - h) * 128 + r]) * sc;
                if (threadIdx.x == 0) tl_mark(p, 25, gb);
                const float m_new = fmaxf(m2, mx);
                const bool rescale = (m_new > m2 + kRescaleThresh) || (m2 == -INFINITY);
                const float m_use = rescale ? m_new : m2;
                const float neg_ref = (m_use == -INFINITY) ? 0.0f : -m_use;
                const float alpha = (m2 == -INFINITY) ? 0.0f : ex2(m2 + neg_ref);
                float rs[4] = {0.0f, 0.0f, 0.0f, 0.0f};
                if (full) {
#pragma unroll
                    for (int c0 = 0; c0 < 64; c0 += 32) {
                        uint32_t pk[16];
#pragma unroll
                        for (int i = 0; i < 32; i += 2) {
                            float e0, e1;
#if S2O_DIAG_POLY > 0
                            if ((i >> 1) % S2O_DIAG_POLY == S2O_DIAG_POLY - 1) {  // FMA-pipe exp2 (MUFU offload)
                                const float2 e = ex2_poly4x2(make_float2(fmaf(__uint_as_float(sv[c0 + i]), sc, neg_ref),
                                                                         fmaf(__uint_as_float(sv[c0 + i + 1]), sc, neg_ref)));
                                e0 = e.x;
                                e1 = e.y;
                            } else
#endif
                            {
                                e0 = ex2(fmaf(__uint_as_float(sv[c0 + i]), sc, neg_ref));
                                e1 = ex2(fmaf(__uint_as_float(sv[c0 + i + 1]), sc, neg_ref));
                            }
                            rs[(i >> 1) & 3] += e0 + e1;
                            pk[i >> 1] = pack_bf16(e0, e1);
                        }
                        tmem_st16(tS + h * 32 + c0 / 2, pk);
                    }
                } else {
#pragma unroll
                    for (int c0 = 0; c0 < 64; c0 += 32) {
                        uint32_t pk[16];
#pragma unroll
                        for (int i = 0; i < 32; i += 2) {
                            const float e0 = c0 + i < lim ? ex2(fmaf(__uint_as_float(sv[c0 + i]), sc, neg_ref)) : 0.0f;
                            const float e1 =
                                c0 + i + 1 < lim ? ex2(fmaf(__uint_as_float(sv[c0 + i + 1]), sc, neg_ref)) : 0.0f;
                            rs[(i >> 1) & 3] += e0 + e1;
                            pk[i >> 1] = pack_bf16(e0, e1);
                        }
                        tmem_st16(tS + h * 32 + c0 / 2, pk);
                    }
                }
                const float rowsum = (rs[0] + rs[1]) + (rs[2] + rs[3]);
                // O rescale (lazy, rare; this half's 64 columns): all earlier P V of the tile done
                if (__any_sync(0xffffffffu, j > 0 && rescale && m2 != -INFINITY)) {
                    // P V(gb-1) done (then all earlier ones are): P V commits the V stage barrier
                    // v_empty[(gb-1) % kDVStages], whose next phase needs P V(gb+1), i.e. P(gb+1)
                    // from this very warp, so the parity wait is exact
                    mbar_wait(smem_u32(&c.v_empty[(gb - 1) % kDVStages]), ((gb - 1) / kDVStages) & 1, 4202);
                    tc_fence_after();
#pragma unroll
                    for (int c0 = 0; c0 < 64; c0 += 32) {
                        uint32_t v[32];
                        tmem_ld32(tO + c0, v);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
                        tmem_st32(tO + c0, v);
                    }
                }
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&c.p_full[gb % kDSBuf]));
                if (threadIdx.x == 0) tl_mark(p, 21, gb);
                ell = ell * alpha + rowsum;
                m2 = m_use;
            }
            // ---- hand the tile to the epilogue warps: (m, this half's ell) through smem
            {
                // the epilogue of tile tk-2 has read this slot (a tile short enough to need no
                // P V before its last S does not order this write otherwise)
                mbar_wait(smem_u32(&c.ml_free[tk & 1]), ((tk >> 1) & 1) ^ 1, 4206);
                float* mlb = ml + (tk & 1) * 384;
                if (h == 0) mlb[r] = m2;
                mlb[128 + h * 128 + r] = ell;
                mbar_arrive(smem_u32(&c.ml_full[tk & 1]));
            }
        }
    } else if (warp < kDEpiWarp0 + 4) {
        // ============================== epilogue ==============================
        setmaxnreg_inc<kDEpiRegs>();
        const int r = (warp - kDEpiWarp0) * 32 + lane;  // TMEM lane quarter = warp % 4
        const uint32_t lane_off = (uint32_t)((warp % 4) * 32) << 16;
        uint32_t tk = 0;
        for (int64_t it = blockIdx.x; it < total; it += gridDim.x, ++tk) {
            const TileInfo t = diag_tile(p, it);
            const bool valid = r < t.tn;
            const int rr = valid ? r : 0;
            const uint32_t ob = tk % kDOBuf, mb = tk & 1;
            mbar_wait(smem_u32(&c.ml_full[mb]), (tk >> 1) & 1, 4203);
            mbar_wait(smem_u32(&c.o_done[ob]), (tk / kDOBuf) & 1, 4204);
            tc_fence_after();
            uint32_t ov[kD];
#pragma unroll
            for (int c0 = 0; c0 < kD; c0 += 32)
                tmem_ld32(tbase + lane_off + (kDSBuf + ob) * 128 + c0, *reinterpret_cast<uint32_t(*)[32]>(&ov[c0]));
            tmem_ld_wait();
            const float m2 = ml[mb * 384 + r], ell = ml[mb * 384 + 128 + r] + ml[mb * 384 + 256 + r];
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&c.o_free[ob]));  // O buffer reusable
            mbar_arrive(smem_u32(&c.ml_free[mb]));                // (m, ell) slot reusable
            const int64_t grow = t.sb + t.t0 + rr;
            const int64_t slot = t.zh * g.l + grow;
            if (valid && (a.mode & kStateOut)) {
                if (p.vec_acc) {
                    float* dst = a.acc_out + slot * kD;
#pragma unroll
                    for (int i = 0; i < kD; i += 8) stg256(dst + i, &ov[i]);
                } else {
                    float4* dst = reinterpret_cast<float4*>(a.acc_out + slot * kD);
#pragma unroll
                    for (int i = 0; i < kD / 4; ++i)
                        dst[i] = make_float4(__uint_as_float(ov[4 * i]), __uint_as_float(ov[4 * i + 1]),
                                             __uint_as_float(ov[4 * i + 2]), __uint_as_float(ov[4 * i + 3]));
                }
                a.m_out[slot] = (m2 == -INFINITY) ? -INFINITY : m2 * 0.6931471805599453f;
                a.ell_out[slot] = ell;
            }
            if (valid && (a.mode & kFinal)) {
                const float inv = 1.0f / ell;
                const int64_t ooff = tc_o_base(p, t.zh) + grow * g.os[2];
                if (g.out_bf16 && p.vec_o) {
                    __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(a.o) + ooff;
#pragma unroll
                    for (int i = 0; i < kD; i += 16) {
                        uint32_t w[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e)
                            w[e] = pack_bf16(__uint_as_float(ov[i + 2 * e]) * inv, __uint_as_float(ov[i + 2 * e + 1]) * inv);
                        stg256(dst + i, w);
                    }
                } else if (g.out_bf16) {
                    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.o) + ooff);
#pragma unroll
                    for (int i = 0; i < kD / 8; ++i) {
                        uint4 w;
                        w.x = pack_bf16(__uint_as_float(ov[8 * i]) * inv, __uint_as_float(ov[8 * i + 1]) * inv);
                        w.y = pack_bf16(__uint_as_float(ov[8 * i + 2]) * inv, __uint_as_float(ov[8 * i + 3]) * inv);
                        w.z = pack_bf16(__uint_as_float(ov[8 * i + 4]) * inv, __uint_as_float(ov[8 * i + 5]) * inv);
                        w.w = pack_bf16(__uint_as_float(ov[8 * i + 6]) * inv, __uint_as_float(ov[8 * i + 7]) * inv);
                        dst[i] = w;
                    }
                } else {
                    float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(a.o) + ooff);
#pragma unroll
                    for (int i = 0; i < kD / 4; ++i)
                        dst[i] = make_float4(__uint_as_float(ov[4 * i]) * inv, __uint_as_float(ov[4 * i + 1]) * inv,
                                             __uint_as_float(ov[4 * i + 2]) * inv, __uint_as_float(ov[4 * i + 3]) * inv);
                }
                if (ell == 0.0f) atomicExch(a.err_flag, 2);
            }
        }
    }
    tc_fence_before();
    if (warp <= kDMmaWarp) named_bar_sync(5, 32 * (kDMmaWarp + 1));  // softmax, epilogue, MMA warps
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tbase, kTmemCols);
    }
}

// ============================================================== two-tile diagonal kernel
// Pass-1 with TWO 128-row query tiles in flight per CTA (the default; S2O_DIAG2=0 selects
// tc_diag_kernel). The tiles of a work item read the same K/V rows: the two q heads 2i, 2i+1 of
// a GQA group at the same (segment, tile) when the group is even, else two adjacent tiles of one
// head (the longer first). Every K/V block is loaded once for both.
//
//   warps 0-3   softmax of tile 0 (thread = row = TMEM lane, all 128 key columns)
//   warps 4-7   softmax of tile 1: the two warps an SMSP runs belong to different tiles, so one
//               tile's S load / row max / P store overlaps the other's exponentials
//   warps 8-11  epilogue (O of a finished tile -> state / output), warp 12 MMA issuer,
//               warp 13 K loader, warp 14 V loader, warp 15 Q loader
//
// TMEM: S_x (P_x in bf16 over its first 64 columns) at [128x, 128x + 128), O_x at
// [256 + 128x, ...). MMA order per block j: P V_0(j), S_0(j+1), P V_1(j), S_1(j+1); the tensor
// pipe is in order, so S_x(j+1) overwrites P_x(j) only after P V_x(j) read it, and s_full_x(j+1)
// (a commit after S_x(j+1)) also covers P V_x(j): a softmax that rescales O_x (lazy max) after
// waiting for s_full_x needs no other barrier. Q has three 32 KB slots, so the next item's first
// Q tile lands while this item runs.
constexpr int kEThreads = 512;
constexpr int kEEpiWarp0 = 8, kEMmaWarp = 12, kEKWarp = 13, kEQWarp = 15;  // warp 14: V loader
constexpr int kESoftRegs = 184, kEEpiRegs = 80, kEMmaRegs = 64, kELoadRegs = 64;
static_assert(8 * (kESoftRegs - 128) <= 4 * (128 - kEEpiRegs) + (128 - kEMmaRegs) + 3 * (128 - kELoadRegs),
              "register pool");
constexpr int kEQSlots = 3, kEKStages = 2, kEVStages = 2;
static_assert(kEKStages == kEVStages, "the K and V loaders share one stage index");
constexpr uint32_t kEOffQ = 0;
constexpr uint32_t kEOffK = kEQSlots * kTileBytes;
constexpr uint32_t kEOffV = kEOffK + kEKStages * kTileBytes;
constexpr uint32_t kEOffCtrl = kEOffV + kEVStages * kTileBytes;
constexpr uint32_t kEOffML = kEOffCtrl + 256;               // float [2 tiles][m, ell][128 rows]
constexpr uint32_t kESmemBytes = kEOffML + 2 * 2 * 128 * 4;  // 226.25 KB
static_assert(kESmemBytes <= 232448, "shared memory");

struct CtrlE {
    uint64_t q_full[kEQSlots], q_empty[kEQSlots];
    uint64_t k_full[kEKStages], k_empty[kEKStages], v_full[kEVStages], v_empty[kEVStages];
    uint64_t s_full[2], p_full[2], o_done[2], o_free[2], ml_full[2], ml_free[2];  // per tile slot
    uint32_t tmem_base;
};
static_assert(sizeof(CtrlE) <= 256, "CtrlE exceeds its 256 B");

// Work items of the two-tile kernel (launcher: pairs_per_head = tiles per head).
__device__ __forceinline__ int64_t diag2_items(const TcParams& p) {
    const Geo& g = p.a.g;
    if (g.group % 2 == 0) return g.z * g.hq / 2 * p.pairs_per_head;
    const int64_t T = p.a.T, t_last = (g.last_len + kBM - 1) / kBM;
    return g.z * g.hq * ((g.N - 1) * ((T + 1) / 2) + (t_last + 1) / 2);
}

// Tile x (0, 1) of work item idx; nd = 0 when the item has no second tile. Items are ordered
// as diag_tile's (GQA group interleaved innermost, longest tiles first within a head).
// Work-item cursor of the two-tile kernel. Every role walks items blockIdx.x, +gridDim.x, ...;
// the index is kept in mixed radix (a: head pair / head in the group, (n, u): segment and tile
// (pair) in longest-first order, zg: kv head) and advanced by carries, because integer division
// needs MUFU.RCP, which the softmax warps keep saturated (a division-based decode at every item
// boundary cost the MMA issuer ~2 k clk). Items are ordered as diag_tile's (GQA group innermost).
struct D2Cur {
    uint32_t a, n, u, zg;      // position
    uint32_t sa, sn, su, sz;   // the stride gridDim.x in the same radix
};
struct D2Rad {
    uint32_t A, U, Ul, N, T, tl, G;
    __device__ __forceinline__ explicit D2Rad(const TcParams& p) {
        const Geo& g = p.a.g;
        G = (uint32_t)g.group;
        T = (uint32_t)p.a.T;
        N = (uint32_t)g.N;
        tl = (uint32_t)((g.last_len + kBM - 1) / kBM);
        const bool hp = G % 2 == 0;  // q heads 2i, 2i+1 of the group (else adjacent tiles of one head)
        A = hp ? G / 2 : G;
        U = hp ? T : (T + 1) / 2;
        Ul = hp ? tl : (tl + 1) / 2;
    }
};

__device__ __forceinline__ void d2_decode(const D2Rad& R, uint32_t v, uint32_t& a, uint32_t& n, uint32_t& u, uint32_t& zg) {
    const uint32_t per = (R.N - 1) * R.U + R.Ul;  // units per kv head (or q head)
    a = v % R.A;
    const uint32_t q = v / R.A;
    const uint32_t r = q % per;
    zg = q / per;
    n = r / R.U;
    u = r % R.U;
}

__device__ __forceinline__ D2Cur d2_init(const D2Rad& R) {
    D2Cur c;
    d2_decode(R, blockIdx.x, c.a, c.n, c.u, c.zg);
    d2_decode(R, gridDim.x, c.sa, c.sn, c.su, c.sz);
    return c;
}

__device__ __forceinline__ void d2_next(const D2Rad& R, D2Cur& c) {
    c.a += c.sa;
    const uint32_t c1 = c.a >= R.A ? 1u : 0u;
    c.a -= c1 * R.A;
    c.u += c.su + c1;
    if (c.u >= R.U) {
        c.u -= R.U;
        ++c.n;
    }
    c.n += c.sn;
    if (c.n > R.N - 1 || (c.n == R.N - 1 && c.u >= R.Ul)) {  // past this kv head: subtract its units
        if (c.u >= R.Ul) c.u -= R.Ul;
        else {
            c.u += R.U - R.Ul;
            --c.n;
        }
        c.n -= R.N - 1;
        ++c.zg;
    }
    c.zg += c.sz;
}

// Tile x (0, 1) of the cursor's item; nd = 0 when the item has no second tile.
__device__ __forceinline__ TileInfo d2_tile(const TcParams& p, const D2Rad& R, const D2Cur& c, int x) {
    const Geo& g = p.a.g;
    const bool last = c.n == R.N - 1;
    // longest tile (pair) first in even segments, shortest first in odd ones: a CTA's items
    // (stride gridDim.x) then see every tile length, not a residue class of them
    const uint32_t u = (c.n & 1u) ? (last ? R.Ul : R.U) - 1 - c.u : c.u;
    int32_t ti;
    TileInfo t;
    if (R.G % 2 == 0) {
        t.zh = (int64_t)c.zg * R.G + 2 * c.a + x;
        ti = (int32_t)((last ? R.tl : R.T) - 1 - u);
    } else {
        t.zh = (int64_t)c.zg * R.G + c.a;
        ti = (int32_t)((last ? R.tl : R.T) - 1 - 2 * u) - x;
    }
    t.n = c.n;
    t.sb = (int64_t)c.n * g.S;
    t.segr = (int)g.seg_rows(c.n);
    if (ti < 0) {
        t.t0 = 0;
        t.tn = 0;
        t.nd = 0;
        return t;
    }
    t.t0 = (int64_t)ti * kBM;
    t.tn = min(kBM, t.segr - ti * kBM);
    t.nd = (ti * kBM + t.tn - 1) / kBN + 1;
    return t;
}

// P = exp2(s * scale - m) for a full row of 128 scores into the first 64 columns of S (bf16
// pairs), all on MUFU: with the row in 128 registers the FMA-pipe polynomial's temporaries do not
// fit, and every polynomial fraction measured slower (1/8 ... 1/2: +4 % ... +80 %).
__device__ __forceinline__ void d2_exps(const uint32_t (&sv)[128], float sc, float neg_ref, uint32_t tS, float (&rs)[4]) {
#pragma unroll
    for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
            const float e0 = ex2(fmaf(__uint_as_float(sv[c0 + i]), sc, neg_ref));
            const float e1 = ex2(fmaf(__uint_as_float(sv[c0 + i + 1]), sc, neg_ref));
            rs[(i >> 1) & 3] += e0 + e1;
            pk[i >> 1] = pack_bf16(e0, e1);
        }
        tmem_st16(tS + c0 / 2, pk);
    }
}

__global__ void __launch_bounds__(kEThreads, 1)
tc_diag2_kernel(const TcParams p, const __grid_constant__ CUtensorMap qtile,
                const __grid_constant__ CUtensorMap ktile, const __grid_constant__ CUtensorMap vtile) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw;
    if ((smem_u32(smem) & 1023u) != 0) __trap();
    CtrlE& c = *reinterpret_cast<CtrlE*>(smem + kEOffCtrl);
    if (threadIdx.x == 0) tl_cta(p, 0);
    const PassArgs& a = p.a;
    const Geo& g = a.g;
    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const uint32_t sQ = smem_u32(smem + kEOffQ);
    const uint32_t sK = smem_u32(smem + kEOffK);
    const uint32_t sV = smem_u32(smem + kEOffV);
    if (threadIdx.x == 0) {
        for (int b = 0; b < kEQSlots; ++b) {
            mbar_init(smem_u32(&c.q_full[b]), 1);
            mbar_init(smem_u32(&c.q_empty[b]), 1);
        }
        for (int s = 0; s < kEKStages; ++s) {
            mbar_init(smem_u32(&c.k_full[s]), 1);
            mbar_init(smem_u32(&c.k_empty[s]), 1);
        }
        for (int s = 0; s < kEVStages; ++s) {
            mbar_init(smem_u32(&c.v_full[s]), 1);
            mbar_init(smem_u32(&c.v_empty[s]), 1);
        }
        for (int x = 0; x < 2; ++x) {
            mbar_init(smem_u32(&c.s_full[x]), 1);
            mbar_init(smem_u32(&c.p_full[x]), 4);    // the tile's softmax warps
            mbar_init(smem_u32(&c.o_done[x]), 1);
            mbar_init(smem_u32(&c.o_free[x]), 4);    // epilogue warps
            mbar_init(smem_u32(&c.ml_full[x]), 128);  // per-thread: each releases its own write
            mbar_init(smem_u32(&c.ml_free[x]), 128);
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
    const int64_t total = diag2_items(p);
    const D2Rad R(p);
    constexpr int64_t rowu = kD;  // (tc path: d == 128)
    float* ml = reinterpret_cast<float*>(smem + kEOffML);
    if (warp >= kEKWarp) {
        // ============================== loaders (one lane each) ==============================
        // warp 13: K blocks, warp 14: V blocks, warp 15: Q tiles (its own lane, so a Q slot that
        // frees late never holds back the next item's first K block)
        setmaxnreg_dec<kELoadRegs>();
        if (lane != 0) return;
        if (warp == kEQWarp) {
            uint32_t qs = 0;
            D2Cur cu = d2_init(R);
            for (int64_t it = blockIdx.x; it < total; it += gridDim.x, d2_next(R, cu))
                for (int x = 0; x < 2; ++x) {
                    const TileInfo t = d2_tile(p, R, cu, x);
                    if (t.nd == 0) continue;
                    const uint32_t sl = qs % kEQSlots;
                    mbar_wait(smem_u32(&c.q_empty[sl]), ((qs / kEQSlots) & 1) ^ 1, 4011);
                    tl_mark(p, 24, qs);
                    mbar_expect_tx(smem_u32(&c.q_full[sl]), kTileBytes);
                    const int64_t qb = tc_q_base(p, t.zh) / rowu;
                    for (int h = 0; h < 2; ++h)
                        tma_load2d(sQ + sl * kTileBytes + h * kHalf, &qtile, h * 64, (int32_t)(qb + t.sb + t.t0),
                                   smem_u32(&c.q_full[sl]));
                    ++qs;
                    if (x == 0 && it + gridDim.x < total) {  // the next item's Q tiles into L2 (read from HBM once)
                        D2Cur cn = cu;
                        d2_next(R, cn);
                        for (int y = 0; y < 2; ++y) {
                            const TileInfo u = d2_tile(p, R, cn, y);
                            if (u.nd == 0) continue;
                            const int64_t ub = tc_q_base(p, u.zh) / rowu;
                            for (int h = 0; h < 2; ++h) tma_prefetch2d(&qtile, h * 64, (int32_t)(ub + u.sb + u.t0));
                        }
                    }
                }
            return;
        }
        const bool kl = warp == kEKWarp;
        const CUtensorMap* xtile = kl ? &ktile : &vtile;
        const uint32_t xbase = kl ? sK : sV;
        uint64_t* xfull = kl ? c.k_full : c.v_full;
        uint64_t* xempty = kl ? c.k_empty : c.v_empty;
        uint32_t gi = 0;
        D2Cur cu = d2_init(R);
        for (int64_t it = blockIdx.x; it < total; it += gridDim.x, d2_next(R, cu)) {
            const TileInfo t0 = d2_tile(p, R, cu, 0);
            const int64_t xb = (kl ? tc_k_base(p, t0.zh) : tc_v_base(p, t0.zh)) / rowu;
            for (int j = 0; j < t0.nd; ++j, ++gi) {  // tile 0 has the most blocks
                const int st = (int)(gi % kEKStages);  // (kEKStages == kEVStages)
                mbar_wait(smem_u32(&xempty[st]), ((gi / kEKStages) & 1) ^ 1, kl ? 4012 : 4013);
                tl_mark(p, kl ? 22 : 23, gi);
                mbar_expect_tx(smem_u32(&xfull[st]), kTileBytes);
                const uint32_t dst = xbase + st * kTileBytes;
                for (int h = 0; h < 2; ++h)
                    tma_load2d(dst + h * kHalf, xtile, h * 64, (int32_t)(xb + t0.sb + (int64_t)j * kBN),
                               smem_u32(&xfull[st]));
            }
        }
        return;
    }
    if (warp == kEMmaWarp) {
        // ============================== MMA issuer ==============================
        // Per tile slot the S / P V stream runs on across work items: the first S of the next
        // item's tile x is issued right after this item's last P V of slot x (and before the
        // other slot's), so the tensor pipe has work while the epilogue drains O.
        setmaxnreg_dec<kEMmaRegs>();
        const bool leader = elect_one();
        const uint32_t idesc_s = umma_idesc_bf16(kBM, kBN, false, false);
        const uint32_t idesc_o = umma_idesc_bf16(kBM, kD, false, true);
        const uint64_t dq0 = umma_desc_sw128(sQ, 16, 1024);
        const uint64_t dk0 = umma_desc_sw128(sK, 16, 1024);
        const uint64_t dv0 = umma_desc_sw128(sV, kHalf, 1024);
        uint32_t kc = 0, vc = 0, qs = 0;
        uint32_t bx[2] = {0u, 0u}, tx[2] = {0u, 0u};  // per tile slot: blocks, tiles so far
        auto issue_s = [&](int x, uint32_t qsl, uint32_t kst) {
            const uint64_t dq = dq0 + ((qsl * kTileBytes) >> 4);
            const uint64_t dk = dk0 + ((kst * kTileBytes) >> 4);
#pragma unroll
            for (int kk = 0; kk < kD / 16; ++kk) {
                const uint32_t off = ((kk / 4) * kHalf + (kk % 4) * 32) >> 4;
                if (leader) umma_bf16(tbase + x * 128, dq + off, dk + off, idesc_s, kk > 0);
            }
            if (leader) umma_commit(smem_u32(&c.s_full[x]));
        };
        // S_x(0) of an item's tile (Q slot assigned in load order); K(0) already waited for
        auto first_s = [&](int x, int nd, uint32_t kst) -> uint32_t {
            const uint32_t sl = qs % kEQSlots;
            mbar_wait(smem_u32(&c.q_full[sl]), (qs / kEQSlots) & 1, 4112);
            tl_mark(p, 25, qs);
            ++qs;
            tc_fence_after();
            issue_s(x, sl, kst);
            if (nd == 1 && leader) umma_commit(smem_u32(&c.q_empty[sl]));
            return sl;
        };
        int64_t it = blockIdx.x;
        int nd[2] = {0, 0};
        uint32_t qsl[2] = {0u, 0u};
        D2Cur cn = d2_init(R);  // the item after the current one (advanced at each item's start)
        if (it < total) {
            nd[0] = d2_tile(p, R, cn, 0).nd;
            nd[1] = d2_tile(p, R, cn, 1).nd;
        }
        for (bool first = true; it < total; it += gridDim.x, first = false) {
            if (first) {
                const uint32_t kst = kc % kEKStages;
                mbar_wait(smem_u32(&c.k_full[kst]), (kc / kEKStages) & 1, 4111);
                for (int x = 0; x < 2; ++x)
                    if (nd[x]) qsl[x] = first_s(x, nd[x], kst);
                if (leader) umma_commit(smem_u32(&c.k_empty[kst]));
                ++kc;
                __syncwarp();
            }
            const int64_t nit = it + gridDim.x;
            // the next item's shape, decoded inside the first block (off the item boundary: the
            // softmax warps sharing this SMSP leave the issuer few issue slots)
            int nn[2] = {0, 0};
            auto look = [&]() {
                d2_next(R, cn);
                if (nit < total) {
                    nn[0] = d2_tile(p, R, cn, 0).nd;
                    nn[1] = d2_tile(p, R, cn, 1).nd;
                }
            };
            if (nd[0] == 1) look();
            uint32_t nsl[2] = {0u, 0u};
            tl_mark(p, 28, vc);
            for (int j = 0; j < nd[0]; ++j) {
                const uint32_t vst = vc % kEVStages;
                const bool last = j + 1 == nd[0];
                const bool knext = !last || nn[0] > 0;  // a K block follows (this item's or the next's)
                const uint32_t kst = kc % kEKStages;
                bool kwait = false;
                tl_mark(p, 1, vc);
                mbar_wait(smem_u32(&c.v_full[vst]), (vc / kEVStages) & 1, 4113);
                const uint64_t dv = dv0 + ((vst * kTileBytes) >> 4);
                for (int x = 0; x < 2; ++x) {
                    if (j < nd[x]) {
                        mbar_wait(smem_u32(&c.p_full[x]), bx[x] & 1, 4114);
                        tl_mark(p, 2 + 3 * x, vc);
                        ++bx[x];
                        // the epilogue has read O_x of this slot's previous tile
                        if (j == 0) mbar_wait(smem_u32(&c.o_free[x]), (tx[x] & 1) ^ 1, 4115);
                        tc_fence_after();
#pragma unroll
                        for (int kk = 0; kk < kBN / 16; ++kk)
                            if (leader)
                                umma_bf16_ts(tbase + (2 + x) * 128, tbase + x * 128 + kk * 8,
                                             dv + ((kk * 16 * 128) >> 4), idesc_o, (kk > 0 || j > 0) ? 1 : 0);
                        tl_mark(p, 4 + 3 * x, vc);
                        if (j == nd[x] - 1) {
                            if (leader) umma_commit(smem_u32(&c.o_done[x]));
                            ++tx[x];
                        }
                    }
                    if (j + 1 < nd[x]) {  // S_x(j+1)
                        if (!kwait) {
                            mbar_wait(smem_u32(&c.k_full[kst]), (kc / kEKStages) & 1, 4116);
                            tc_fence_after();
                            kwait = true;
                        }
                        issue_s(x, qsl[x], kst);
                        tl_mark(p, 8 + x, vc);
                        if (j + 2 == nd[x] && leader) umma_commit(smem_u32(&c.q_empty[qsl[x]]));
                    } else if (last && nn[x] > 0) {  // S_x(0) of the next item
                        if (!kwait) {
                            mbar_wait(smem_u32(&c.k_full[kst]), (kc / kEKStages) & 1, 4117);
                            kwait = true;
                        }
                        nsl[x] = first_s(x, nn[x], kst);
                        tl_mark(p, 26 + x, vc);
                    }
                    __syncwarp();
                }
                if (j == 0 && nd[0] > 1) look();
                if (leader) umma_commit(smem_u32(&c.v_empty[vst]));
                ++vc;
                if (knext) {
                    if (leader) umma_commit(smem_u32(&c.k_empty[kst]));
                    ++kc;
                }
                __syncwarp();
            }
            tl_mark(p, 29, vc);
            nd[0] = nn[0];
            nd[1] = nn[1];
            qsl[0] = nsl[0];
            qsl[1] = nsl[1];
        }
        __syncwarp();
    } else if (warp < kEEpiWarp0) {
        // ============================== softmax ==============================
        setmaxnreg_inc<kESoftRegs>();
        const int x = warp >> 2, qd = warp & 3;
        const int r = qd * 32 + lane;  // TMEM lane = row
        const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
        const uint32_t tS = tbase + lane_off + x * 128;
        const uint32_t tO = tbase + lane_off + (2 + x) * 128;
        const float sc = p.scale_log2;
        uint32_t bx = 0, tx = 0;
        D2Cur cu = d2_init(R);
        for (int64_t it = blockIdx.x; it < total; it += gridDim.x, d2_next(R, cu)) {
            const TileInfo t = d2_tile(p, R, cu, x);
            if (t.nd == 0) continue;
            const bool valid = r < t.tn;
            const int rr = valid ? r : 0;
            const int t0x = (int)t.t0;
            float m2 = -INFINITY, ell = 0.0f;
            for (int j = 0; j < t.nd; ++j, ++bx) {
                mbar_wait(smem_u32(&c.s_full[x]), bx & 1, 4211);
                if (r == 0) tl_mark(p, 10 + 4 * x, bx);
                tc_fence_after();
                uint32_t sv[128];
#pragma unroll
                for (int c0 = 0; c0 < 128; c0 += 32) tmem_ld32(tS + c0, *reinterpret_cast<uint32_t(*)[32]>(&sv[c0]));
                tmem_ld_wait();
                if (r == 0) tl_mark(p, 11 + 4 * x, bx);
                // visible keys of this row in block j (causal on segment positions, kernel.cpp:58-69)
                const int k0 = j * kBN;
                const int kn = min(kBN, t.segr - k0);
                const int vis = (k0 + kn - 1 <= t0x) ? kn : min(kn, t0x + rr - k0 + 1);
                const int lim = max(0, vis);
                const bool full = __all_sync(0xffffffffu, lim >= 128);
                float mxa[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) mxa[i] = -INFINITY;
                if (full) {
#pragma unroll
                    for (int i = 0; i < 128; i += 2)
                        mxa[(i >> 1) & 7] = fmax3(mxa[(i >> 1) & 7], __uint_as_float(sv[i]), __uint_as_float(sv[i + 1]));
                } else {
#pragma unroll
                    for (int i = 0; i < 128; i += 2)
                        mxa[(i >> 1) & 7] = fmax3(mxa[(i >> 1) & 7], i < lim ? __uint_as_float(sv[i]) : -INFINITY,
                                                  i + 1 < lim ? __uint_as_float(sv[i + 1]) : -INFINITY);
                }
                const float mx =
                    fmax3(fmax3(mxa[0], mxa[1], mxa[2]), fmax3(mxa[3], mxa[4], mxa[5]), fmaxf(mxa[6], mxa[7])) * sc;
                const float m_new = fmaxf(m2, mx);
                const bool rescale = (m_new > m2 + kRescaleThresh) || (m2 == -INFINITY);
                const float m_use = rescale ? m_new : m2;
                const float neg_ref = (m_use == -INFINITY) ? 0.0f : -m_use;
                const float alpha = (m2 == -INFINITY) ? 0.0f : ex2(m2 + neg_ref);
                float rs[4] = {0.0f, 0.0f, 0.0f, 0.0f};
                if (full) {
                    d2_exps(sv, sc, neg_ref, tS, rs);
                } else {
#pragma unroll
                    for (int c0 = 0; c0 < 128; c0 += 32) {
                        uint32_t pk[16];
#pragma unroll
                        for (int i = 0; i < 32; i += 2) {
                            const float e0 = c0 + i < lim ? ex2(fmaf(__uint_as_float(sv[c0 + i]), sc, neg_ref)) : 0.0f;
                            const float e1 =
                                c0 + i + 1 < lim ? ex2(fmaf(__uint_as_float(sv[c0 + i + 1]), sc, neg_ref)) : 0.0f;
                            rs[(i >> 1) & 3] += e0 + e1;
                            pk[i >> 1] = pack_bf16(e0, e1);
                        }
                        tmem_st16(tS + c0 / 2, pk);
                    }
                }
                if (r == 0) tl_mark(p, 12 + 4 * x, bx);
                // O rescale (lazy, rare; after the exponentials, when S is no longer live): s_full_x(j)
                // was committed after P V_x(j-1)
                if (__any_sync(0xffffffffu, j > 0 && rescale && m2 != -INFINITY)) {
#pragma unroll
                    for (int c0 = 0; c0 < 128; c0 += 32) {
                        uint32_t v[32];
                        tmem_ld32(tO + c0, v);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
                        tmem_st32(tO + c0, v);
                    }
                }
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&c.p_full[x]));
                if (r == 0) tl_mark(p, 13 + 4 * x, bx);
                ell = ell * alpha + ((rs[0] + rs[1]) + (rs[2] + rs[3]));
                m2 = m_use;
            }
            // (m, ell) to the epilogue; the slot's previous tile has been read
            mbar_wait(smem_u32(&c.ml_free[x]), (tx & 1) ^ 1, 4212);
            ml[x * 256 + r] = m2;
            ml[x * 256 + 128 + r] = ell;
            mbar_arrive(smem_u32(&c.ml_full[x]));
            ++tx;
        }
    } else if (warp < kEEpiWarp0 + 4) {
        // ============================== epilogue ==============================
        setmaxnreg_dec<kEEpiRegs>();
        const int r = (warp - kEEpiWarp0) * 32 + lane;  // TMEM lane quarter = warp % 4
        const uint32_t lane_off = (uint32_t)((warp % 4) * 32) << 16;
        uint32_t tx[2] = {0u, 0u};
        D2Cur cu = d2_init(R);
        for (int64_t it = blockIdx.x; it < total; it += gridDim.x, d2_next(R, cu)) {
            for (int x = 0; x < 2; ++x) {
                const TileInfo t = d2_tile(p, R, cu, x);
                if (t.nd == 0) continue;
                const bool valid = r < t.tn;
                const int rr = valid ? r : 0;
                mbar_wait(smem_u32(&c.ml_full[x]), tx[x] & 1, 4213);
                const float m2 = ml[x * 256 + r], ell = ml[x * 256 + 128 + r];
                mbar_arrive(smem_u32(&c.ml_free[x]));
                mbar_wait(smem_u32(&c.o_done[x]), tx[x] & 1, 4214);
                if (r == 0) tl_mark(p, 18 + 2 * x, tx[x]);
                ++tx[x];
                tc_fence_after();
                const int64_t grow = t.sb + t.t0 + rr;
                const int64_t slot = t.zh * g.l + grow;
                const float inv = 1.0f / ell;
                const int64_t ooff = tc_o_base(p, t.zh) + grow * g.os[2];
#pragma unroll
                for (int c0 = 0; c0 < kD; c0 += 32) {
                    uint32_t ov[32];
                    tmem_ld32(tbase + lane_off + (2 + x) * 128 + c0, ov);
                    tmem_ld_wait();
                    if (c0 == kD - 32) {  // O_x fully read: the slot's next tile may accumulate
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(smem_u32(&c.o_free[x]));
                        if (r == 0) tl_mark(p, 19 + 2 * x, tx[x] - 1);
                    }
                    if (!valid) continue;
                    if (a.mode & kStateOut) {
                        if (p.vec_acc) {
                            float* dst = a.acc_out + slot * kD + c0;
#pragma unroll
                            for (int i = 0; i < 32; i += 8) stg256(dst + i, &ov[i]);
                        } else {
                            float4* dst = reinterpret_cast<float4*>(a.acc_out + slot * kD + c0);
#pragma unroll
                            for (int i = 0; i < 8; ++i)
                                dst[i] = make_float4(__uint_as_float(ov[4 * i]), __uint_as_float(ov[4 * i + 1]),
                                                     __uint_as_float(ov[4 * i + 2]), __uint_as_float(ov[4 * i + 3]));
                        }
                    }
                    if (a.mode & kFinal) {
                        if (g.out_bf16) {
                            uint32_t w[16];
#pragma unroll
                            for (int e = 0; e < 16; ++e)
                                w[e] = pack_bf16(__uint_as_float(ov[2 * e]) * inv, __uint_as_float(ov[2 * e + 1]) * inv);
                            __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(a.o) + ooff + c0;
                            if (p.vec_o) {
                                stg256(dst, w);
                                stg256(dst + 16, w + 8);
                            } else {
                                uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
                                for (int i = 0; i < 4; ++i) d4[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
                            }
                        } else {
                            float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(a.o) + ooff + c0);
#pragma unroll
                            for (int i = 0; i < 8; ++i)
                                dst[i] = make_float4(__uint_as_float(ov[4 * i]) * inv, __uint_as_float(ov[4 * i + 1]) * inv,
                                                     __uint_as_float(ov[4 * i + 2]) * inv, __uint_as_float(ov[4 * i + 3]) * inv);
                        }
                    }
                }
                if (valid && (a.mode & kStateOut)) {
                    a.m_out[slot] = (m2 == -INFINITY) ? -INFINITY : m2 * 0.6931471805599453f;
                    a.ell_out[slot] = ell;
                }
                if (valid && (a.mode & kFinal) && ell == 0.0f) atomicExch(a.err_flag, 2);
            }
        }
    }
    tc_fence_before();
    if (warp <= kEMmaWarp) named_bar_sync(5, 32 * (kEMmaWarp + 1));  // softmax, epilogue, MMA warps
    if (threadIdx.x == 0) tl_cta(p, 3);
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tbase, kTmemCols);
    }
}

// ============================================================== masked-key poison scan
// Masked keys are skipped by the reference (attention.cpp:55-57), but the tensor core multiplies
// them: 0 * NaN / 0 * Inf in P V would poison earlier rows of a diagonal tile. Only a tile's last
// (diagonal) block has masked keys, and on the diagonal passes V block b of a segment is the
// diagonal block of tile b. This kernel reads every V block once (one warp each; HBM-bound,
// ~40 us at C3) and lists, for a block holding a non-finite bf16 value, the tiles of all q heads
// of its group; run_pass recomputes the listed tiles on the exact path after the pass.
__global__ void __launch_bounds__(256) poison_scan_kernel(const PassArgs a) {
    const Geo& g = a.g;
    const int64_t per = a.tiles_per_head, hkv = g.hq / g.group;
    const int64_t total = g.z * hkv * per;
    const int lane = threadIdx.x % 32;
    const __nv_bfloat16* vbase = reinterpret_cast<const __nv_bfloat16*>(a.v);
    for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; w < total;
         w += (int64_t)gridDim.x * blockDim.x / 32) {
        const int64_t zk = w / per, r = w % per;
        const int64_t zh0 = (zk / hkv) * g.hq + (zk % hkv) * g.group;  // first q head of the group
        const int64_t full = (g.N - 1) * a.T;
        const int64_t n = r < full ? r / a.T : g.N - 1;
        const int64_t ti = r < full ? r % a.T : r - full;
        const int64_t k0 = n * g.S + ti * kBN;
        const int64_t kn = min((int64_t)kBN, g.seg_rows(n) - ti * kBN);
        const uint4* vb = reinterpret_cast<const uint4*>(vbase + g.v_base(zh0) + k0 * g.vs[2]);
        uint32_t bad = 0u;
        const int64_t row4 = g.vs[2] / 8;  // row stride in uint4 (strides_ok: a multiple of 128)
#pragma unroll 4
        for (int64_t i = lane; i < kn * (kD / 8); i += 32) {
            const uint4 x = vb[(i / (kD / 8)) * row4 + i % (kD / 8)];
            for (const uint32_t v : {x.x, x.y, x.z, x.w})
                bad |= (((v & 0x7f80u) == 0x7f80u) | ((v & 0x7f800000u) == 0x7f800000u)) ? 1u : 0u;
        }
        if (__any_sync(0xffffffffu, bad != 0u) && lane == 0) {
            const int pos = atomicAdd(a.poison_cnt, (int)g.group);
            for (int64_t u = 0; u < g.group; ++u) a.poison_list[pos + u] = (int32_t)((zh0 + u) * per + r);
        }
    }
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

unsigned long long* g_timeline = nullptr;

bool strides_ok(const int64_t* st) { return st[0] % kD == 0 && st[1] % kD == 0 && st[2] % kD == 0; }

// Max dynamic shared memory is a per-device function attribute: set it once per (kernel, device).
cudaError_t smem_attr(const void* fn, uint32_t bytes) {
    static std::mutex mu;
    static std::vector<std::pair<const void*, int>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    for (const auto& d : done)
        if (d.first == fn && d.second == dev) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) done.emplace_back(fn, dev);
    return e;
}

}  // namespace

bool make_bf16_row_map(void* map, const void* base, int64_t rows, uint32_t box_rows) {
    return make_row_map(reinterpret_cast<CUtensorMap*>(map), base, rows, box_rows);
}
int64_t bf16_row_span(const int64_t* st, int64_t z, int64_t h, int64_t l) { return span_rows(st, z, h, l); }
cudaError_t set_max_dyn_smem(const void* fn, uint32_t bytes) { return smem_attr(fn, bytes); }

// Diagonal-only passes (pass-1, the dense reference) on contiguous rows run on the single-tile
// kernel with double-buffered S (S2O_DIAG_KERNEL=0 selects the pair kernel instead).
bool tc_diag_used(const PassArgs& a) {
    static const bool diag_on = [] {
        const char* e = std::getenv("S2O_DIAG_KERNEL");
        return !(e && std::strcmp(e, "0") == 0);
    }();
    const Geo& g = a.g;
    return diag_on && (a.mode & kDiag) && !(a.mode & (kPrefix | kStateIn)) && !a.tile_list && g.qs[2] == kD &&
           g.ks[2] == kD && g.vs[2] == kD;
}

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

cudaError_t launch_poison_scan(const PassArgs& a, cudaStream_t st) {
    const int64_t warps = a.g.z * (a.g.hq / a.g.group) * a.tiles_per_head;
    if (warps == 0) return cudaSuccess;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((warps + 7) / 8, (int64_t)sms * 8));
    poison_scan_kernel<<<grid, 256, 0, st>>>(a);
    return cudaGetLastError();
}

// Grid of the two-tile kernel. CTA b takes items b, b + grid, ...; in plain longest-first order
// a CTA saw only every other tile length of a segment (148 / 2 = 74 = 10 mod 16 at C3: CTAs with
// even b / 2 got 9 blocks per item on average, the others 8, and the kernel ran as long as the
// busier half, measured CTA spans 2.16-2.60 ms). d2_tile alternates the order per segment; on
// top, among grids of [sms - 12, sms] this picks the one whose busiest CTA has the fewest blocks
// (host replica of the item order, computed once per shape).
int diag2_grid(const Geo& g, int64_t T, int64_t work, int sms) {
    if (work <= sms) return (int)std::max<int64_t>(1, work);
    struct Key { int64_t G, T, N, tl, kh; int sms; int grid; };
    static std::mutex mu;
    static std::vector<Key> cache;
    const int64_t G = g.group, N = g.N, tl = (g.last_len + kBM - 1) / kBM, kh = g.z * g.hq / g.group;
    {
        std::lock_guard<std::mutex> lock(mu);
        for (const Key& k : cache)
            if (k.G == G && k.T == T && k.N == N && k.tl == tl && k.kh == kh && k.sms == sms) return k.grid;
    }
    const bool hp = G % 2 == 0;
    const int64_t A = hp ? G / 2 : G, U = hp ? T : (T + 1) / 2, Ul = hp ? tl : (tl + 1) / 2;
    const int64_t R = (N - 1) * U + Ul;
    std::vector<int64_t> blocks(work);  // blocks of item i (both tiles)
    for (int64_t i = 0; i < work; ++i) {
        const int64_t r = (i / A) % R;
        const int64_t n = r < (N - 1) * U ? r / U : N - 1;
        const int64_t u0 = r - n * U;
        const int64_t u = (n & 1) ? (n == N - 1 ? Ul : U) - 1 - u0 : u0;  // d2_tile's snake order
        const int64_t top = (n == N - 1 ? tl : T) - 1;
        if (hp) blocks[i] = 2 * (top - u + 1);
        else {
            const int64_t t0 = top - 2 * u;
            blocks[i] = (t0 + 1) + (t0 >= 1 ? t0 : 0);
        }
    }
    int best = sms;
    int64_t best_load = INT64_MAX;
    std::vector<int64_t> load;
    for (int grid = sms; grid >= std::max(1, sms - 12); --grid) {
        load.assign(grid, 0);
        for (int64_t i = 0; i < work; ++i) load[i % grid] += blocks[i];
        const int64_t mx = *std::max_element(load.begin(), load.end());
        if (mx < best_load) {
            best_load = mx;
            best = grid;
        }
    }
    std::lock_guard<std::mutex> lock(mu);
    cache.push_back({G, T, N, tl, kh, sms, best});
    return best;
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
    // 256-bit epilogue accesses need 32-B aligned rows
    const auto al32 = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 31) == 0; };
    p.vec_acc = al32(a.acc_in) && al32(a.acc_out);
    p.vec_o = g.out_bf16 && al32(a.o) && g.os[0] % 16 == 0 && g.os[1] % 16 == 0 && g.os[2] % 16 == 0;
    p.pairs_full = (a.T + 1) / 2;
    p.tl = g_timeline;
    const int64_t t_last = (g.last_len + kBM - 1) / kBM;
    p.pairs_per_head = (g.N - 1) * p.pairs_full + (t_last + 1) / 2;
    if (g.z * g.hq * std::max<int64_t>(p.pairs_per_head, a.tiles_per_head) >= (int64_t(1) << 31))
        return cudaErrorInvalidValue;  // pair_info decodes 32-bit indices
    p.fd_pg = FastDiv((uint32_t)(p.pairs_per_head * g.group));
    p.fd_g = FastDiv((uint32_t)g.group);
    p.fd_pf = FastDiv((uint32_t)std::max<int64_t>(1, p.pairs_full));
    p.fd_tph = FastDiv((uint32_t)std::max<int64_t>(1, a.tiles_per_head));
    p.fd_t = FastDiv((uint32_t)std::max<int64_t>(1, a.T));
    p.fd_hq = FastDiv((uint32_t)g.hq);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // Diagonal-only passes (pass-1, the dense reference) on contiguous rows: the single-tile
    // kernel with double-buffered S (S2O_DIAG_KERNEL=0 selects the pair kernel instead).
    if (tc_diag_used(a)) {
        TcParams pd = p;
        pd.pairs_per_head = (g.N - 1) * a.T + t_last;  // tiles per head (diag_tile)
        static const bool two_tile = [] {  // S2O_DIAG2=0: the single-tile kernel (A/B aid)
            const char* e = std::getenv("S2O_DIAG2");
            return !(e && std::strcmp(e, "0") == 0);
        }();
        if (two_tile) {  // tc_diag2_kernel: two tiles sharing K/V per work item
            if (cudaError_t e = smem_attr((const void*)tc_diag2_kernel, kESmemBytes)) return e;
            const int64_t work = g.group % 2 == 0
                                     ? g.z * g.hq / 2 * pd.pairs_per_head
                                     : g.z * g.hq * ((g.N - 1) * ((a.T + 1) / 2) + (t_last + 1) / 2);
            if (work == 0) return cudaSuccess;
            if (work >= (int64_t(1) << 31)) return cudaErrorInvalidValue;  // D2Cur: 32-bit item index
            const int grid = diag2_grid(g, a.T, work, sms);
            tc_diag2_kernel<<<grid, kEThreads, kESmemBytes, st>>>(pd, qtile, ktile, vtile);
            return cudaGetLastError();
        }
        if (cudaError_t e = smem_attr((const void*)tc_diag_kernel, kDSmemBytes)) return e;
        const int64_t work = g.z * g.hq * pd.pairs_per_head;
        if (work == 0) return cudaSuccess;
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(work, sms));
        tc_diag_kernel<<<grid, kDThreads, kDSmemBytes, st>>>(pd, qtile, ktile, vtile);
        return cudaGetLastError();
    }
    for (const void* f : {(const void*)tc_pass_kernel<false>, (const void*)tc_pass_kernel<true>})
        if (cudaError_t e = smem_attr(f, kSmemBytes)) return e;
    const int64_t work = a.tile_list ? a.max_tiles() : g.z * g.hq * p.pairs_per_head;
    if (work == 0) return cudaSuccess;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(work, sms));
    if (a.mode & kPrefix)
        tc_pass_kernel<true><<<grid, kThreads, kSmemBytes, st>>>(p, qmap, kmap, vmap, qtile, ktile, vtile);
    else
        tc_pass_kernel<false><<<grid, kThreads, kSmemBytes, st>>>(p, qmap, kmap, vmap, qtile, ktile, vtile);
    return cudaGetLastError();
}

}  // namespace s2o

// Profiling aid (not part of the operator ABI): record clock64() pipeline events of CTA 0 of
// subsequent tcgen05 pass launches into a device buffer of 32 * 1024 uint64 (nullptr = off).
extern "C" void s2o_debug_timeline(void* dev_buf) {
    s2o::g_timeline = reinterpret_cast<unsigned long long*>(dev_buf);
}
