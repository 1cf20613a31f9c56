// plan_tc.cuh -- candidate-pruned exact top-T selection for the truncated plan. Included by
// plan.cu inside its anonymous namespace (uses Geo, desc_key, the sel_sort kernel).
//
// Reference: rank_prefix_keys (plan.cpp:103-138) scores every prefix key of segment n with
// dot_f(q_mean[n], K[t]) (fp64, sequential over d, plan.cpp:14-20) and argsort_desc_stable
// (tensor.cpp:43-61) orders them. The fused operator only consumes the first T entries of that
// order, so instead of scoring all S*N(N-1)/2 keys per head in fp64 (16.9 G DFMA at C3) the
// selection runs in four steps whose result is provably the same first T entries:
//
//  1. threshold (cand_thresh_kernel): exact fp64 scores of a 1/8 sample of each segment's prefix
//     keys (kv_score128_kernel on a strided view of K) -> theta = the sample key whose rank is
//     6 sigma above the expected sample rank of entry T (~1.24 T at T = 6144, so at most kSelCap = 8192
//     candidates but for ~1 % of the rows), and
//     e_q = kEpsC * ||q_mean[n]||_2.
//  2. candidates (kv_cand_kernel, tcgen05): s~ = q_mean . K^T on the tensor cores, q_mean split
//     into bf16 hi + lo terms (q - hi - lo <= 2^-18 |q|), fp32 accumulation, so
//     |s~ - s| <= 2^-14.5 ||q|| ||k|| (256 products, any accumulation order; kEpsC = 2^-12 keeps a
//     5.6x margin). Key t is a candidate iff NOT(s~ + e_q ||k_t|| < theta) (NaN -> candidate), so
//     every key with exact s >= theta is one. Each candidate is then rescored EXACTLY (fp64 DFMA
//     chain over d = 0..127 from 0.0, bit-identical to dot_f) in the same kernel, with the K tile
//     converted to fp64 in shared memory (exact) and q_mean in fp64 in TMEM, and appended in key
//     order to the (row, 2048-key chunk) region of the key workspace.
//  3. certification + compaction (cand_pack_kernel): if fewer than T candidates have an exact
//     score >= theta the row is flagged (the caller falls back to the full plan). Otherwise every
//     key with exact s >= s_T is a candidate; a radix select finds a key kv of rank in
//     [T, kSelCap] and the candidates below it (plus the first equal ones, by index) are compacted
//     in index order.
//  4. sel_sort_kernel (plan.cu) sorts them stably by key and keeps the first T: the first T entries
//     of argsort_desc_stable.
// Segments with fewer than kCandDensity * T prefix keys (n < n_cand: most of their keys would be
// candidates) are scored densely in fp64 (kv_score128) and selected as before (sel_scan, or sorted
// directly when at most kSelCap keys).
#pragma once

using namespace ::s2o::sm100;

constexpr int kCR = 2048;                // keys per candidate work unit (16 tiles of 128)
constexpr int kCTiles = kCR / 128;
constexpr int kCSub = 2;                 // row warps per TMEM lane quadrant (candidates split by rank parity)
constexpr int kCRowThreads = 128 * kCSub;
constexpr int kCConv = 2;                // converter warps per quadrant
constexpr int kCConvWarp0 = 4 * kCSub;   // 4 kCConv warps: K conversion (thread = key, d part) + masks (lane = row, key part)
constexpr int kCConvThreads = 128 * kCConv;
constexpr int kCTmaWarp = kCConvWarp0 + 4 * kCConv, kCMmaWarp = kCTmaWarp + 1;
constexpr int kCThreads = 32 * (kCMmaWarp + 1);
constexpr int kSampStride = 8;           // step-1 sample: token 8 i + kSampPhase
constexpr int kSampPhase = 3;
constexpr double kEpsC = 1.0 / 4096.0;   // error bound factor (see above)
constexpr int kPackCap = 12288;          // candidates a row may have (else: flagged); 2 CTAs / SM
constexpr int kPackThreads = 256;
constexpr int64_t kCandDensity = 4;      // segments with fewer than 4 T prefix keys are scored densely

constexpr uint32_t kCTile = 128 * 128 * 2;                   // bf16 [128 x 128] as two SW128 halves
constexpr uint32_t kCHalf = kCTile / 2;
constexpr uint32_t kKhStride = 129;                          // words per key row (odd: lanes on distinct banks)
constexpr uint32_t kKhBytes = 128 * kKhStride * 4;
constexpr uint32_t kCOffK = 0;                               // K stages 0, 1 (bf16, TMA)
constexpr uint32_t kCOffKh = 2 * kCTile;                     // 2 x K tile as fp64 high words [128][129]
constexpr uint32_t kCOffKn = kCOffKh + 2 * kKhBytes;         // key norms float[128] + partials [kCConv][128]
constexpr uint32_t kCOffMask = kCOffKn + 128 * 4 * (1 + kCConv);  // candidate masks uint32 [2][128 rows][4]
constexpr uint32_t kCOffCtrl = kCOffMask + 2 * 128 * 16;
constexpr uint32_t kCSmem = kCOffCtrl + 128;                 // 197.6 KB
// TMEM columns: s~ accumulator [0, 128), A = q_mean hi / lo in bf16 [128, 192) / [192, 256) (the MMA
// reads A from TMEM), q_mean in fp64 [256, 512)
constexpr uint32_t kCTmemAcc = 0, kCTmemAhi = 128, kCTmemAlo = 192, kCTmemQ = 256;

struct CandCtrl {
    uint64_t k_full[2], k_empty[2], a_full, a_empty, h_full[2], h_free[2];
    uint32_t tmem_base;
};
static_assert(sizeof(CandCtrl) <= 128, "CandCtrl");

struct CandArgs {
    Geo g;
    const float* q_mean;  // [Z*Hq*N][128]
    const float* thr;     // [Z*Hq*N] theta rounded down to fp32 (-inf: every key is a candidate)
    const float* ec;      // [Z*Hq*N] e_q rounded up
    uint64_t* ckey;       // candidate keys / indices: row (zh, n) chunk c at zh*kvp + kv_off(n) + c*kCR
    uint32_t* cidx;
    int32_t* ccnt;        // [Z*Hq*N][nch] candidates per (row, chunk)
    int64_t nch;          // chunks of the longest prefix
    // row tiles (the same for every kv head): tile y holds segments [tn0[y], tn0[y] + tnc[y]) of the
    // kv head's q heads, row u = (n - tn0) * group + h % group, U = tnc * group <= 128 / trep rows,
    // each replicated trep times over the 128 MMA rows / TMEM lanes (lane l holds row l % (128 /
    // trep)): a short prefix concentrates a row's candidates in few key tiles, so those rows get
    // more lanes (their candidates split by rank over the replicas)
    int32_t tn0[64], tnc[64], trep[64];
    int32_t ntiles;
};
constexpr int kCMaxRowTiles = 64;

// bf16 (as the high half of a fp32 word, low 16 bits zero) -> high 32 bits of the equal double;
// the low 32 bits are zero for every bf16 value. Zeros, infinities and NaN handled; a bf16
// subnormal goes through the (exact) F2F conversion.
__device__ __forceinline__ uint32_t f32hi_to_f64hi(uint32_t f) {
    const uint32_t e = f & 0x7f800000u;
    const uint32_t sign = f & 0x80000000u;
    if (e != 0u && e != 0x7f800000u) return sign | (((f & 0x7fffffffu) >> 3) + 0x38000000u);
    if ((f & 0x7fffffffu) == 0u) return sign;
    if (e == 0x7f800000u) return sign | 0x7ff00000u | ((f & 0x007fffffu) >> 3);
    return (uint32_t)__double2hiint((double)__uint_as_float(f));
}

// Work unit: (2048-key chunk, 128-row tile, (z, kv head)). Rows are (q head, segment) pairs of the
// kv head ordered by segment, so a warp's 32 lanes hold segments of similar prefix length (similar
// candidate counts). Per 128-key tile, pipelined one tile apart:
//   TMA warp        K(i) bf16 -> stage i % 2
//   MMA warp        s~(i) = [q_hi | q_lo] . K(i)^T into the TMEM accumulator (A from TMEM)
//   converter warps K(i) -> fp64 high words (buffer i % 2, thread = key) and key norms; then, lane
//                   = row, s~(i) -> candidate masks (smem) and the accumulator is released
//   row warps       exact fp64 rescoring of their candidates (q_mean fp64 from TMEM, K words from
//                   smem), appended to the row's region at the candidate's rank; buffer released
__global__ void __launch_bounds__(kCThreads, 1)
kv_cand_kernel(const CandArgs a, const __grid_constant__ CUtensorMap kmap) {
    extern __shared__ __align__(1024) unsigned char cand_smem[];
    unsigned char* smem = cand_smem;
    if ((smem_u32(smem) & 1023u) != 0) __trap();
    CandCtrl& c = *reinterpret_cast<CandCtrl*>(smem + kCOffCtrl);
    const Geo& g = a.g;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t chunk = blockIdx.x;
    const int64_t z = blockIdx.z / g.hkv, kvh = blockIdx.z % g.hkv;
    const int ty = blockIdx.y;
    const int64_t tn0 = a.tn0[ty], rep = a.trep[ty];
    const int64_t n_top = tn0 + a.tnc[ty] - 1;  // longest prefix of the tile
    const int64_t urows = (int64_t)a.tnc[ty] * g.group, uspan = 128 / rep;
    const int64_t key_end = n_top * g.S;
    const int64_t t_begin = chunk * kCR;
    if (t_begin >= key_end) return;  // nothing here
    const int ntiles = (int)min((int64_t)kCTiles, (key_end - t_begin + 127) / 128);
    const uint32_t sK = smem_u32(smem + kCOffK);
    float* kn = reinterpret_cast<float*>(smem + kCOffKn);
    uint32_t* masks = reinterpret_cast<uint32_t*>(smem + kCOffMask);
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(smem_u32(&c.k_full[s]), 1);
            mbar_init(smem_u32(&c.k_empty[s]), kCConvThreads + 1);  // converter threads + the MMA commit
            mbar_init(smem_u32(&c.h_full[s]), kCConvThreads);
            mbar_init(smem_u32(&c.h_free[s]), kCRowThreads);
        }
        mbar_init(smem_u32(&c.a_full), 1);
        mbar_init(smem_u32(&c.a_empty), kCConvThreads);
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(smem_u32(&c.tmem_base), 512);
        tmem_relinquish();
    }
    // ---- the row of TMEM lane r (quadrant warp % 4) for row and converter warps
    const int r = (warp % 4) * 32 + lane;
    const int64_t u = r % uspan;     // the lane's row (consecutive rows share a warp)
    const int replica = (int)(r / uspan);
    const bool in = warp < kCTmaWarp && u < urows;
    const int64_t n = in ? tn0 + u / g.group : 0;
    const int64_t zh = z * g.hq + kvh * g.group + (in ? u % g.group : 0);
    const int64_t rowcode = zh * g.N + n;
    const int64_t lim = in ? n * g.S : 0;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = c.tmem_base;
    if (warp < 4) {
        // A operand in TMEM: q_mean hi / lo in bf16 (two per column, even d in the low half), and
        // q_mean in fp64 (two words per d); lane r = MMA row r
        const uint32_t trow = tbase + ((uint32_t)(warp * 32) << 16);
        const float* qrow = a.q_mean + rowcode * 128;
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {  // d in [64 half, 64 half + 64)
            uint32_t hi[32], lo[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const float x0 = in ? qrow[64 * half + 2 * i] : 0.0f, x1 = in ? qrow[64 * half + 2 * i + 1] : 0.0f;
                const __nv_bfloat16 h0 = __float2bfloat16_rn(x0), h1 = __float2bfloat16_rn(x1);
                hi[i] = pack_bf16(__bfloat162float(h0), __bfloat162float(h1));
                lo[i] = pack_bf16(x0 - __bfloat162float(h0), x1 - __bfloat162float(h1));  // exact differences
            }
            tmem_st32(trow + kCTmemAhi + 32 * half, hi);
            tmem_st32(trow + kCTmemAlo + 32 * half, lo);
        }
#pragma unroll 1
        for (int i = 0; i < 8; ++i) {
            uint32_t w[32];
#pragma unroll
            for (int d = 0; d < 16; ++d) {
                const double x = in ? (double)qrow[16 * i + d] : 0.0;
                w[2 * d] = (uint32_t)__double2loint(x);
                w[2 * d + 1] = (uint32_t)__double2hiint(x);
            }
            tmem_st32(trow + kCTmemQ + 32 * i, w);
        }
        tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    if (warp == kCTmaWarp) {
        // ============================== K tiles (TMA) ==============================
        if (lane == 0) {
            const int64_t krow0 = (z * g.ks[0] + kvh * g.ks[1]) / 128;
            for (int i = 0; i < ntiles; ++i) {
                const int s = i & 1;
                mbar_wait(smem_u32(&c.k_empty[s]), ((i >> 1) & 1) ^ 1, 7001);
                mbar_expect_tx(smem_u32(&c.k_full[s]), kCTile);
                const int32_t row = (int32_t)(krow0 + t_begin + 128 * i);
                for (int h = 0; h < 2; ++h)
                    tma_load2d(sK + s * kCTile + h * kCHalf, &kmap, h * 64, row, smem_u32(&c.k_full[s]));
            }
        }
    } else if (warp == kCMmaWarp) {
        // ============================== MMA issuer ==============================
        const bool leader = elect_one();
        const uint32_t idesc = umma_idesc_bf16(128, 128, false, false);
        for (int i = 0; i < ntiles; ++i) {
            const int s = i & 1;
            mbar_wait(smem_u32(&c.k_full[s]), (i >> 1) & 1, 7002);
            mbar_wait(smem_u32(&c.a_empty), (i & 1) ^ 1, 7003);  // the converters have read s~(i-1)
            tc_fence_after();
            const uint64_t dk = umma_desc_sw128(sK + s * kCTile, 16, 1024);
            if (leader) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = ((kk / 4) * kCHalf + (kk % 4) * 32) >> 4;
                    umma_bf16_ts(tbase + kCTmemAcc, tbase + kCTmemAhi + kk * 8, dk + off, idesc, kk > 0);
                }
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = ((kk / 4) * kCHalf + (kk % 4) * 32) >> 4;
                    umma_bf16_ts(tbase + kCTmemAcc, tbase + kCTmemAlo + kk * 8, dk + off, idesc, 1);
                }
                umma_commit(smem_u32(&c.a_full));
                umma_commit(smem_u32(&c.k_empty[s]));
            }
            __syncwarp();
        }
    } else if (warp >= kCConvWarp0) {
        // ============================== converters ==============================
        const uint32_t lane_off = (uint32_t)((warp % 4) * 32) << 16;
        const float thr = in ? a.thr[rowcode] : INFINITY;
        const float ec = in ? a.ec[rowcode] : 0.0f;
        const int ct = threadIdx.x - kCConvWarp0 * 32;  // 0 .. kCConvThreads-1
        const int key = ct % 128, part = ct / 128;      // conversion: key row, d part
        const int mpart = (warp - kCConvWarp0) / 4;     // masks: lane = row, key part
        float* knp = kn + 128;
        for (int i = 0; i < ntiles; ++i) {
            const int s = i & 1;
            const int64_t t0 = t_begin + 128 * i;
            mbar_wait(smem_u32(&c.k_full[s]), (i >> 1) & 1, 7004);
            mbar_wait(smem_u32(&c.h_free[s]), ((i >> 1) & 1) ^ 1, 7006);  // the rows are done with tile i-2
            {
                const unsigned char* kt = smem + kCOffK + s * kCTile;
                uint32_t* dst = reinterpret_cast<uint32_t*>(smem + kCOffKh + s * kKhBytes) + key * kKhStride;
                float ss = 0.0f;
#pragma unroll 2
                for (int cc = part * (16 / kCConv); cc < (part + 1) * (16 / kCConv); ++cc) {
                    const uint4 w = *reinterpret_cast<const uint4*>(
                        kt + (cc >> 3) * kCHalf + key * 128 + ((((uint32_t)cc & 7u) ^ ((uint32_t)key & 7u)) << 4));
                    const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float f0 = __uint_as_float(wv[e] << 16), f1 = __uint_as_float(wv[e] & 0xffff0000u);
                        ss = fmaf(f0, f0, ss);
                        ss = fmaf(f1, f1, ss);
                        // exact widening (F2F); a bf16's double has a zero low word
                        dst[8 * cc + 2 * e] = (uint32_t)__double2hiint((double)f0);
                        dst[8 * cc + 2 * e + 1] = (uint32_t)__double2hiint((double)f1);
                    }
                }
                knp[part * 128 + key] = ss;
            }
            named_bar_sync(2, kCConvThreads);
            mbar_arrive(smem_u32(&c.k_empty[s]));
            if (ct < 128) {
                float ss = 0.0f;
#pragma unroll
                for (int p = 0; p < kCConv; ++p) ss += knp[p * 128 + ct];
                // ||k|| rounded up (fp32 sum of 128 squares: relative error < 2^-16); non-finite -> inf
                const float nrm = __fsqrt_ru(ss) * 1.0001f;
                kn[ct] = (nrm <= 3.0e38f) ? nrm : INFINITY;
            }
            named_bar_sync(2, kCConvThreads);  // every key norm of the tile
            // s~(i) -> candidate masks of row r, keys [128 mpart / kCConv, 128 (mpart + 1) / kCConv)
            mbar_wait(smem_u32(&c.a_full), (uint32_t)i & 1u, 7005);
            tc_fence_after();
            uint32_t* mrow = masks + (s * 128 + r) * 4;
#pragma unroll
            for (int qq = 0; qq < 4 / kCConv; ++qq) {
                const int q4 = mpart * (4 / kCConv) + qq;
                uint32_t v[32];
                tmem_ld32(tbase + lane_off + kCTmemAcc + 32 * q4, v);
                tmem_ld_wait();
                uint32_t bits = 0u;
#pragma unroll
                for (int jj = 0; jj < 32; ++jj) {
                    const float x = __uint_as_float(v[jj]) + ec * kn[32 * q4 + jj];
                    const bool cand = (t0 + 32 * q4 + jj < lim) && !(x < thr);
                    bits |= (cand ? 1u : 0u) << jj;
                }
                mrow[q4] = bits;
            }
            tc_fence_before();
            mbar_arrive(smem_u32(&c.a_empty));
            named_bar_sync(2, kCConvThreads);  // the key norms are rewritten by the next tile
            mbar_arrive(smem_u32(&c.h_full[s]));
        }
    } else {
        // ============================== rows ==============================
        const int sub = warp / 4;  // the row warps of a quadrant split the row's candidates
        const uint32_t tq = tbase + ((uint32_t)((warp % 4) * 32) << 16) + kCTmemQ;
        const int64_t region = zh * g.kv_per_head() + g.kv_off(n) + chunk * kCR;
        int run = 0;
        for (int i = 0; i < ntiles; ++i) {
            const int s = i & 1;
            const int64_t t0 = t_begin + 128 * i;
            mbar_wait(smem_u32(&c.h_full[s]), (i >> 1) & 1, 7007);
            const uint32_t* kh = reinterpret_cast<const uint32_t*>(smem + kCOffKh + s * kKhBytes);
            const uint4 mm = *reinterpret_cast<const uint4*>(masks + (s * 128 + r) * 4);
            const uint32_t m[4] = {mm.x, mm.y, mm.z, mm.w};
            const int pc0 = __popc(m[0]), pc1 = pc0 + __popc(m[1]), pc2 = pc1 + __popc(m[2]);
            const int total = pc2 + __popc(m[3]);
            // this thread's share of the row's candidates: ranks = replica * kCSub + sub (mod
            // trep * kCSub); for one replica, the parity of the rank (bit i of the prefix XOR x is
            // the parity of the candidates at or below i)
            static_assert(kCSub == 2, "rank split by parity");
            uint32_t mine[4];
            if (rep == 1) {
                uint32_t carry = 0u;  // parity of the candidates in earlier words
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                    uint32_t x = m[q4];
                    x ^= x << 1;
                    x ^= x << 2;
                    x ^= x << 4;
                    x ^= x << 8;
                    x ^= x << 16;
                    const uint32_t even = m[q4] & (carry ? ~x : x);  // global rank even
                    mine[q4] = sub == 0 ? even : (m[q4] & ~even);
                    carry ^= (uint32_t)__popc(m[q4]) & 1u;
                }
            } else {
                const int slots = (int)rep * kCSub, me = replica * kCSub + sub;  // slots: 2, 4 or 8
                int rk = 0;
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                    uint32_t w = m[q4], keep = 0u;
                    while (w) {
                        const uint32_t b = w & (0u - w);
                        if ((rk & (slots - 1)) == me) keep |= b;  // (power of two: no division)
                        ++rk;
                        w ^= b;
                    }
                    mine[q4] = keep;
                }
            }
            // ---- exact fp64 rescoring, kCG candidates at a time (dot_f order: d = 0..127 from 0.0)
            constexpr int kCG = 4;
            while (__any_sync(0xffffffffu, (mine[0] | mine[1] | mine[2] | mine[3]) != 0u)) {
                int jk[kCG];
#pragma unroll
                for (int u = 0; u < kCG; ++u) {
                    int j = -1;
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) {
                        if (j < 0 && mine[q4] != 0u) {
                            j = 32 * q4 + __ffs(mine[q4]) - 1;
                            mine[q4] &= mine[q4] - 1u;
                        }
                    }
                    jk[u] = j;
                }
                double acc[kCG];
                const uint32_t* krow[kCG];
#pragma unroll
                for (int u = 0; u < kCG; ++u) {
                    acc[u] = 0.0;
                    krow[u] = kh + (jk[u] < 0 ? 0 : jk[u]) * kKhStride;
                }
                // q_mean[row] in 16-d chunks from TMEM, software-pipelined: the load of chunk qc + 1
                // is in flight while chunk qc is used (the TMEM load latency is long)
                uint32_t qa[32], qb[32];
                tmem_ld32(tq, qa);
                tmem_ld_wait();
#pragma unroll
                for (int qc = 0; qc < 8; ++qc) {  // 16 d per round
                    uint32_t(&qv)[32] = (qc & 1) ? qb : qa;
                    uint32_t(&qn)[32] = (qc & 1) ? qa : qb;
                    if (qc + 1 < 8) tmem_ld32(tq + 32 * (qc + 1), qn);
#pragma unroll
                    for (int d = 0; d < 16; ++d) {
                        const double qd = __hiloint2double((int)qv[2 * d + 1], (int)qv[2 * d]);
#pragma unroll
                        for (int u = 0; u < kCG; ++u)  // one 32-bit load per DFMA: the low word is zero
                            acc[u] = fma(qd, __hiloint2double((int)krow[u][16 * qc + d], 0), acc[u]);
                    }
                    if (qc + 1 < 8) tmem_ld_wait();
                }
#pragma unroll
                for (int u = 0; u < kCG; ++u) {
                    const int j = jk[u];
                    if (j >= 0) {  // position: the candidate's rank among the row's candidates of this tile
                        const int q4 = j >> 5;
                        const int below = __popc(m[q4] & ((1u << (j & 31)) - 1u)) +
                                          (q4 == 0 ? 0 : q4 == 1 ? pc0 : q4 == 2 ? pc1 : pc2);
                        a.ckey[region + run + below] = desc_key(acc[u]);
                        a.cidx[region + run + below] = (uint32_t)(t0 + j);
                    }
                }
            }
            run += total;
            mbar_arrive(smem_u32(&c.h_free[s]));
        }
        if (sub == 0 && replica == 0 && lim > t_begin) a.ccnt[rowcode * a.nch + chunk] = run;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tbase, 512);
    }
}

// Block-wide approximate-rank radix select over 64-bit keys, 8-bit digits from the top: after each
// pass the bin holding rank r is known; once that bin has at most `slack` keys (or every bit is
// fixed) the result is the LARGEST key of the bin, so its rank lies in [r, r + slack]. Returns that
// key. visit(f) calls f(key, valid) for every key this thread owns (valid = false: padding; every
// lane of a warp makes the same calls). All threads of the block participate.
struct SelScratch {
    int hist[256];
    unsigned long long s_max;
    uint64_t s_prefix;
    int s_want, s_bin;
};
template <int kThreads, class Visit>
__device__ uint64_t block_select_max(Visit visit, int r, int slack, SelScratch& sc) {
    const int tid = threadIdx.x, lane = tid & 31;
    uint64_t prefix = 0ull, mask = 0ull;
    int want = r;
#pragma unroll 1
    for (int sh = 56; sh >= 0; sh -= 8) {
        for (int b = tid; b < 256; b += kThreads) sc.hist[b] = 0;
        __syncthreads();
        // warp-aggregated histogram (keys of similar scores share their leading digits)
        visit([&](uint64_t k, bool valid) {
            const bool in = valid && (k & mask) == prefix;
            const uint32_t dig = in ? (uint32_t)((k >> sh) & 255u) : 0xffffffffu;
            const uint32_t peers = __match_any_sync(0xffffffffu, dig);
            if (in && lane == __ffs(peers) - 1) atomicAdd(&sc.hist[dig], __popc(peers));
        });
        __syncthreads();
        if (tid < 32) {  // warp 0 locates the bin of rank `want` (8 bins per lane)
            int cnt[8], sum = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                cnt[i] = sc.hist[lane * 8 + i];
                sum += cnt[i];
            }
            int incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            int before = incl - sum;
            if (before < want && want <= incl) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    if (before < want && want <= before + cnt[i]) {
                        sc.s_bin = cnt[i];
                        sc.s_prefix = prefix | ((uint64_t)(lane * 8 + i) << sh);
                        sc.s_want = want - before;
                    }
                    before += cnt[i];
                }
            }
        }
        __syncthreads();
        prefix = sc.s_prefix;
        want = sc.s_want;
        mask |= 255ull << sh;
        const int bin = sc.s_bin;
        __syncthreads();
        if (bin <= slack + 1) break;
    }
    // the largest key of the bin
    if (tid == 0) sc.s_max = 0ull;
    __syncthreads();
    unsigned long long mx = 0ull;
    visit([&](uint64_t k, bool valid) {
        if (valid && (k & mask) == prefix && k > mx) mx = k;
    });
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = y > mx ? y : mx;
    }
    if (lane == 0 && mx) atomicMax(&sc.s_max, mx);
    __syncthreads();
    return (uint64_t)sc.s_max;
}

__device__ __forceinline__ double desc_key_value(uint64_t key) {  // inverse of desc_key
    const uint64_t asc = ~key;
    const uint64_t b = (asc & 0x8000000000000000ull) ? (asc & 0x7fffffffffffffffull) : ~asc;
    return __longlong_as_double((long long)b);
}

// Step 1: per row (zh, n >= n_cand): theta from the exact scores of the sampled keys, e_q.
constexpr int kThrThreads = 1024;
__global__ void __launch_bounds__(kThrThreads)
cand_thresh_kernel(Geo g, const uint64_t* __restrict__ samp, int64_t s2, const float* __restrict__ q_mean,
                   int64_t topt, int64_t n_cand, float* __restrict__ thr, float* __restrict__ ec,
                   uint64_t* __restrict__ kth) {
    __shared__ SelScratch sc;
    __shared__ double s_part[kThrThreads / 32];
    const int tid = threadIdx.x;
    const int64_t zh = blockIdx.x / (g.N - 1), n = 1 + blockIdx.x % (g.N - 1);
    if (n < n_cand) return;
    const int64_t row = zh * g.N + n;
    const int64_t len = n * g.S, tt = min(topt, len), m = n * s2;
    const uint64_t* keys = samp + zh * (s2 * g.N * (g.N - 1) / 2) + s2 * n * (n - 1) / 2;
    // x = expected sample keys among the first T; the rank keeps >= 6 sigma (binomial, ~sqrt(r))
    // between T and the count above theta, so certification fails ~1e-9 per row
    const double x = (double)tt * (double)m / (double)len;
    const int64_t rank = min(m, max((int64_t)1, (int64_t)ceil(x + 6.0 * sqrt(x) + 18.0)));
    constexpr int kPer = 16;  // keys per thread held in registers (m <= 16384), else re-read
    uint64_t kr[kPer];
    const bool in_regs = m <= kThrThreads * kPer;
    if (in_regs) {
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int64_t i = (int64_t)u * kThrThreads + tid;
            kr[u] = i < m ? keys[i] : ~0ull;
        }
    }
    auto visit = [&](auto f) {  // every lane of a warp makes the same calls (valid says if the key exists)
        if (in_regs) {
#pragma unroll
            for (int u = 0; u < kPer; ++u) f(kr[u], (int64_t)u * kThrThreads + tid < m);
        } else {
            for (int64_t i0 = 0; i0 < m; i0 += kThrThreads)
                f(i0 + tid < m ? keys[i0 + tid] : 0ull, i0 + tid < m);
        }
    };
    // theta need not be the exact rank-th sample key: any sample key of rank in [rank, rank + rank/64]
    const uint64_t key = block_select_max<kThrThreads>(visit, (int)rank, (int)(rank / 64), sc);
    // ||q_mean[n]||_2 in fp64
    double q2 = 0.0;
    if (tid < 128) {
        const double x = (double)q_mean[row * 128 + tid];
        q2 = x * x;
    }
    for (int o = 16; o > 0; o >>= 1) q2 += __shfl_xor_sync(0xffffffffu, q2, o);
    if ((tid & 31) == 0) s_part[tid >> 5] = q2;
    __syncthreads();
    if (tid == 0) {
        double qs = 0.0;
        for (int w = 0; w < 4; ++w) qs += s_part[w];  // warps 0-3 hold the 128 squares
        const double qn = sqrt(qs) * (1.0 + 1e-12);
        const double theta = desc_key_value(key);
        float t = __double2float_rd(theta);
        if (!(qn <= 1e300) || !(theta > -3.4028234663852886e+38)) t = -INFINITY;  // every key is a candidate
        thr[row] = t;
        ec[row] = __double2float_ru(kEpsC * qn);
        kth[row] = key;
    }
}

// Step 3: certify the row's candidates and compact exactly its first T (key, index) entries, in
// index order, into (ckey, cidx) at the row's offset; sel_sort_kernel sorts them.
struct PackSmem {  // the select variant's dynamic shared memory
    uint64_t key[kPackCap];
    SelScratch sc;
};

// kSelect = false: rows with at most kSelCap candidates (a plain copy; no dynamic shared memory, so
// many CTAs per SM overlap their loads); kSelect = true: the (rare) rows with more.
struct PackHdr {
    int pre[257];
    int s_total, s_cert;
};
template <bool kSelect>
__global__ void __launch_bounds__(kPackThreads)
cand_pack_kernel(Geo g, const uint64_t* __restrict__ ckey_in, const uint32_t* __restrict__ cidx_in,
                 const int32_t* __restrict__ ccnt, int64_t nch, const uint64_t* __restrict__ kth, int64_t topt,
                 int64_t n_cand, uint64_t* __restrict__ ckey, uint32_t* __restrict__ cidx,
                 int32_t* __restrict__ ccount, int32_t* __restrict__ flags) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PackSmem& sm = *reinterpret_cast<PackSmem*>(smem_raw);  // kSelect only
    __shared__ PackHdr hd;
    const int tid = threadIdx.x;
    const int64_t zh = blockIdx.x / (g.N - 1), n = 1 + blockIdx.x % (g.N - 1);
    if (n < n_cand) return;
    const int64_t row = zh * g.N + n;
    const int64_t len = n * g.S, tt = min(topt, len);
    const int64_t nc = (len + kCR - 1) / kCR;
    const int64_t base = zh * g.kv_per_head() + g.kv_off(n);
    // chunk prefix (one chunk per thread: nc <= 256, i.e. L <= 512K at kCR = 2048; more: flagged)
    {
        const int cnt = (tid < nc && nc <= 256) ? ccnt[row * nch + tid] : 0;
        int incl = cnt;
        const int lane = tid & 31, w = tid >> 5;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        __shared__ int wtot[kPackThreads / 32];
        if (lane == 31) wtot[w] = incl;
        if (tid == 0) hd.s_cert = 0;
        __syncthreads();
        int wb = 0, all = 0;
        for (int x = 0; x < kPackThreads / 32; ++x) {
            wb += x < w ? wtot[x] : 0;
            all += wtot[x];
        }
        if (tid <= nc && tid < 257) hd.pre[tid] = wb + incl - cnt;  // pre[nc] = total
        if (tid == 0) hd.s_total = nc <= 256 ? all : kPackCap + 1;
        __syncthreads();
    }
    const int total = hd.s_total;
    const uint64_t kthr = kth[row];
    bool fail = total > kPackCap || total < tt;
    // chunk of candidate i: the last chunk whose start is <= i (pre[] is ascending; empty chunks share
    // their start with the next one)
    auto chunk_of = [&](int i) {
        int lo = 0, hi = (int)nc - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (hd.pre[mid] <= i) lo = mid; else hi = mid - 1;
        }
        return lo;
    };
    const bool direct = !fail && total <= kSelCap;  // every candidate goes to the sort: a plain copy
    if (kSelect == direct) return;  // the other variant's row
    if (!fail) {
        int cert = 0;
        const int lane = tid & 31, w = tid >> 5;
        for (int cc = w; cc < nc; cc += kPackThreads / 32) {  // warp per chunk: coalesced
            const int c0 = hd.pre[cc], cn = hd.pre[cc + 1] - c0;
            for (int i = lane; i < cn; i += 32) {
                const uint64_t k = ckey_in[base + (int64_t)cc * kCR + i];
                cert += k <= kthr ? 1 : 0;
                if (!kSelect) {
                    ckey[base + c0 + i] = k;
                    cidx[base + c0 + i] = cidx_in[base + (int64_t)cc * kCR + i];
                } else {
                    sm.key[c0 + i] = k;
                }
            }
        }
        for (int o = 16; o > 0; o >>= 1) cert += __shfl_xor_sync(0xffffffffu, cert, o);
        if (lane == 0) atomicAdd(&hd.s_cert, cert);
        __syncthreads();
        fail = hd.s_cert < tt;  // some key outside the candidates could belong to the first T
    }
    int32_t* outc = ccount + row;
    uint64_t* ok = ckey + base;
    uint32_t* oi = cidx + base;
    if (fail) {  // flagged: any T valid indices keep the passes in bounds until the fallback
        for (int64_t i = tid; i < tt; i += kPackThreads) {
            ok[i] = (uint64_t)i;
            oi[i] = (uint32_t)i;
        }
        if (tid == 0) {
            *outc = (int32_t)tt;
            atomicExch(flags, 1);
        }
        return;
    }
    if constexpr (!kSelect) {
        if (tid == 0) *outc = total;
        return;
    }
    // a key kv of rank in [T, kSelCap]: every candidate below it, then the first (in index order)
    // candidates equal to it, up to kSelCap in all; sel_sort_kernel sorts them and keeps the first T
    auto visit = [&](auto f) {
        for (int i0 = 0; i0 < total; i0 += kPackThreads) f(i0 + tid < total ? sm.key[i0 + tid] : 0ull, i0 + tid < total);
    };
    const uint64_t kv = block_select_max<kPackThreads>(visit, (int)tt, kSelCap - (int)tt, sm.sc);
    // compaction in index order: per-thread contiguous ranges, block scans of (#less, #equal)
    const int per = (total + kPackThreads - 1) / kPackThreads;
    const int i0 = min(total, tid * per), i1 = min(total, i0 + per);
    int nl = 0, ne = 0;
    for (int i = i0; i < i1; ++i) {
        nl += sm.key[i] < kv;
        ne += sm.key[i] == kv;
    }
    long long v = ((long long)nl << 32) | (long long)ne, incl = v;
    const int lane = tid & 31, w = tid >> 5;
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    __shared__ long long wsum[kPackThreads / 32];
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    long long wb = 0, all = 0;
    for (int x = 0; x < kPackThreads / 32; ++x) {
        wb += x < w ? wsum[x] : 0;
        all += wsum[x];
    }
    const long long ex = wb + incl - v;
    int less_before = (int)(ex >> 32), eq_before = (int)(ex & 0xffffffff);
    const int n_less = (int)(all >> 32);
    const int need_eq = min((int)(all & 0xffffffff), kSelCap - n_less);
    int cc = i0 < total ? chunk_of(i0) : 0;
    for (int i = i0; i < i1; ++i) {
        while (cc + 1 < nc && hd.pre[cc + 1] <= i) ++cc;  // chunk of candidate i
        const uint64_t k = sm.key[i];
        bool take = false;
        int pos = 0;
        if (k < kv) {
            take = true;
            pos = less_before + min(eq_before, need_eq);
            ++less_before;
        } else if (k == kv) {
            take = eq_before < need_eq;
            pos = less_before + eq_before;
            ++eq_before;
        }
        if (take) {  // its index lives at the same region slot as its key
            ok[pos] = k;
            oi[pos] = cidx_in[base + (int64_t)cc * kCR + (i - hd.pre[cc])];
        }
    }
    if (tid == 0) *outc = n_less + need_eq;
}

__global__ void set_flag_kernel(int32_t* f, int32_t v) { *f = v; }
