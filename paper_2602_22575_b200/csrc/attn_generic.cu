// attn_generic.cu -- the exact SIMT path of Step 2 (any D, any tile shape, fp32/bf16 in).
//
// Mirrors the reference's per-row fp64 online softmax (os_update attention.cpp:31-88)
// operation by operation -- fp64 scores, the same max/rescale/accumulate order, no FMA
// contraction in the accumulators -- so outputs agree with the oracle to ~1 ulp of the
// exp() implementation and traces agree except exact threshold ties. Used for shapes the
// tcgen05 kernels do not cover (the reference's tiny fixtures, fp32 C1, odd tiles) and as
// the numerics cross-check of the tensor-core path.
//
// One CTA per query tile (grid-stride over all tiles), one thread per query row. The
// per-row fp64 state (acc[D], m, ell) lives in a per-CTA scratch slice in global memory.
// The stop decision of a prefix chunk is a CTA-wide max reduction of the rows' relative
// normaliser gains (early_stop_check kernel.cpp:220-234), taken before the chunk's V
// contribution is committed; a stopping chunk is discarded (kernel.cpp:114-117).
#include "internal.h"

namespace s2o {

namespace {

constexpr int kThreads = 128;

struct RowCtx {
    const void* q;
    int64_t qoff;  // element offset of the row's Q
};

__device__ __forceinline__ double dot_row(const void* q, int64_t qoff, const void* k, int64_t koff,
                                          int64_t d, int bf16) {
    double acc = 0.0;
    for (int64_t i = 0; i < d; ++i)
        acc = fma((double)ld_in(q, qoff + i, bf16), (double)ld_in(k, koff + i, bf16), acc);
    return acc;
}

__global__ void __launch_bounds__(kThreads) generic_pass_kernel(PassArgs a, double* scratch_all) {
    const Geo& g = a.g;
    const int64_t d = g.d;
    __shared__ double red[kThreads];
    __shared__ int stop_flag;
    // per-CTA scratch: acc[bm*d], m[bm], ell[bm], mn[bm], en[bm], rs[bm]; rows[bm] (int64)
    double* acc = scratch_all + (size_t)blockIdx.x * (size_t)(a.bm * d + 5 * a.bm + a.bm);
    double* m = acc + a.bm * d;
    double* ell = m + a.bm;
    double* mn = ell + a.bm;
    double* en = mn + a.bm;
    double* rsc = en + a.bm;
    int64_t* grow = reinterpret_cast<int64_t*>(rsc + a.bm);
    const int64_t total_tiles = a.num_tiles();
    const int64_t full_tiles = (g.N - 1) * a.T;

    for (int64_t it = blockIdx.x; it < total_tiles; it += gridDim.x) {
        const int64_t tile = a.tile_at(it);
        const int64_t zh = tile / a.tiles_per_head;
        const int64_t r_in = tile % a.tiles_per_head;
        int64_t n, ti;
        if (r_in < full_tiles) { n = r_in / a.T; ti = r_in % a.T; }
        else { n = g.N - 1; ti = r_in - full_tiles; }
        const int64_t sb = n * g.S;
        const int64_t seg_rows = g.seg_rows(n);
        const int64_t t0 = ti * a.bm;
        const int64_t tn = min(a.bm, seg_rows - t0);
        const int64_t qb = g.q_base(zh), kb = g.k_base(zh), vb = g.v_base(zh);
        const int64_t rowslot = zh * g.l;

        __syncthreads();  // previous tile's scratch readers are done
        for (int64_t r = threadIdx.x; r < tn; r += blockDim.x) {
            const int64_t local = (a.mode & kStateIn) && a.q_reorder
                                      ? (int64_t)a.q_perm[(zh * g.N + n) * g.S + t0 + r]
                                      : t0 + r;
            grow[r] = sb + local;
            if (a.mode & kStateIn) {
                const int64_t slot = rowslot + grow[r];
                m[r] = (double)a.m_in[slot];
                ell[r] = (double)a.ell_in[slot];
                for (int64_t i = 0; i < d; ++i) acc[r * d + i] = (double)a.acc_in[slot * d + i];
            } else {
                m[r] = -INFINITY;
                ell[r] = 0.0;
                for (int64_t i = 0; i < d; ++i) acc[r * d + i] = 0.0;
            }
        }

        // ---- intra-segment causal scan (segment_causal_tile kernel.cpp:36-71)
        if (a.mode & kDiag) {
            const int64_t last_row = t0 + tn - 1;
            for (int64_t r = threadIdx.x; r < tn; r += blockDim.x) {
                const int64_t qoff = qb + grow[r] * g.qs[2];
                double* ar = acc + r * d;
                for (int64_t k0 = 0; k0 <= last_row && k0 < seg_rows; k0 += a.bn) {
                    const int64_t kn = min(a.bn, seg_rows - k0);
                    const bool masked = !(k0 + kn - 1 <= t0);
                    int64_t vis = kn;
                    if (masked) vis = max((int64_t)0, min(kn, t0 + r - k0 + 1));
                    if (vis == 0) continue;  // fully masked tile: state unchanged
                    double tmax = -INFINITY;
                    for (int64_t j = 0; j < vis; ++j) {
                        const double s = dot_row(a.q, qoff, a.k, kb + (sb + k0 + j) * g.ks[2], d, g.in_bf16) * a.scale;
                        tmax = std_max(tmax, s);
                    }
                    const double m_new = std_max(m[r], tmax);
                    const double rescale = exp(m[r] - m_new);
                    double e = __dmul_rn(ell[r], rescale);
                    for (int64_t i = 0; i < d; ++i) ar[i] = __dmul_rn(ar[i], rescale);
                    for (int64_t j = 0; j < vis; ++j) {
                        const int64_t key = sb + k0 + j;
                        const double s = dot_row(a.q, qoff, a.k, kb + key * g.ks[2], d, g.in_bf16) * a.scale;
                        const double w = exp(s - m_new);
                        e = __dadd_rn(e, w);
                        const int64_t voff = vb + key * g.vs[2];
                        for (int64_t i = 0; i < d; ++i)
                            ar[i] = __dadd_rn(ar[i], __dmul_rn(w, (double)ld_in(a.v, voff + i, g.in_bf16)));
                    }
                    m[r] = m_new;
                    ell[r] = e;
                }
            }
        }

        // ---- ranked prefix traversal with the monotone-gain stop (kernel.cpp:86-122)
        int64_t committed = 0;
        bool overflow = false;
        if ((a.mode & kPrefix) && n > 0) {
            const int32_t* kv = a.kv_seg(zh, n);
            const int64_t kv_len = a.avail(n);
            int64_t pairs = 0;
            for (int64_t c0 = 0; c0 < kv_len; c0 += a.bn) {
                const int64_t cn = min(a.bn, kv_len - c0);
                double local_gain = -INFINITY;
                for (int64_t r = threadIdx.x; r < tn; r += blockDim.x) {
                    const int64_t qoff = qb + grow[r] * g.qs[2];
                    double tmax = -INFINITY;
                    for (int64_t j = 0; j < cn; ++j) {
                        const double s = dot_row(a.q, qoff, a.k, kb + (int64_t)kv[c0 + j] * g.ks[2], d, g.in_bf16) * a.scale;
                        tmax = std_max(tmax, s);
                    }
                    const double m_new = std_max(m[r], tmax);
                    const double rescale = exp(m[r] - m_new);
                    double e = __dmul_rn(ell[r], rescale);
                    for (int64_t j = 0; j < cn; ++j) {
                        const double s = dot_row(a.q, qoff, a.k, kb + (int64_t)kv[c0 + j] * g.ks[2], d, g.in_bf16) * a.scale;
                        e = __dadd_rn(e, exp(s - m_new));
                    }
                    const double prev = ell[r] * exp(m[r] - m_new);
                    if (!(prev > 0.0) && !(prev != prev)) atomicExch(a.err_flag, 1);
                    local_gain = std_max(local_gain, (e - prev) / prev);
                    mn[r] = m_new;
                    en[r] = e;
                    rsc[r] = rescale;
                }
                red[threadIdx.x] = local_gain;
                __syncthreads();
                if (threadIdx.x == 0) {
                    double mg = -INFINITY;
                    for (int i = 0; i < blockDim.x; ++i) mg = std_max(mg, red[i]);
                    stop_flag = (mg < a.tau) ? 1 : 0;
                }
                __syncthreads();
                if (stop_flag) break;
                for (int64_t r = threadIdx.x; r < tn; r += blockDim.x) {
                    const int64_t qoff = qb + grow[r] * g.qs[2];
                    double* ar = acc + r * d;
                    const double rescale = rsc[r];
                    for (int64_t i = 0; i < d; ++i) ar[i] = __dmul_rn(ar[i], rescale);
                    for (int64_t j = 0; j < cn; ++j) {
                        const int64_t key = kv[c0 + j];
                        const double s = dot_row(a.q, qoff, a.k, kb + key * g.ks[2], d, g.in_bf16) * a.scale;
                        const double w = exp(s - mn[r]);
                        const int64_t voff = vb + key * g.vs[2];
                        for (int64_t i = 0; i < d; ++i)
                            ar[i] = __dadd_rn(ar[i], __dmul_rn(w, (double)ld_in(a.v, voff + i, g.in_bf16)));
                    }
                    m[r] = mn[r];
                    ell[r] = en[r];
                }
                ++committed;
                pairs += tn * cn;
                __syncthreads();
            }
            overflow = a.truncated(n) && committed * a.bn >= kv_len;
            if (threadIdx.x == 0) {
                const int base = a.tile_base ? a.tile_base[it] : 0;
                if (overflow) {
                    const int slot = atomicAdd(a.ovf_count, 1);
                    a.ovf_tiles[slot] = (int32_t)tile;
                    if (a.ovf_base) a.ovf_base[slot] = base + (int32_t)committed;
                } else {
                    a.processed[(zh * g.N + n) * a.T + ti] = base + (int32_t)committed;
                }
                if (pairs && (!overflow || a.acc_out))
                    atomicAdd((unsigned long long*)&a.pass2_pairs[zh], (unsigned long long)pairs);
            }
        } else if ((a.mode & kPrefix) && threadIdx.x == 0) {
            a.processed[(zh * g.N + n) * a.T + ti] = 0;
        }

        // ---- outputs (an overflow tile with a state buffer resumes at the next plan level)
        const bool resume_later = overflow && a.acc_out != nullptr;
        for (int64_t r = threadIdx.x; r < tn; r += blockDim.x) {
            const int64_t slot = rowslot + grow[r];
            if ((a.mode & kStateOut) || resume_later) {
                a.m_out[slot] = (float)m[r];
                a.ell_out[slot] = (float)ell[r];
                for (int64_t i = 0; i < d; ++i) a.acc_out[slot * d + i] = (float)acc[r * d + i];
            }
            if ((a.mode & kFinal) && !resume_later) {
                if (ell[r] == 0.0) atomicExch(a.err_flag, 2);
                const int64_t ooff = g.o_base(zh) + grow[r] * g.os[2];
                for (int64_t i = 0; i < d; ++i)
                    st_out(a.o, ooff + i, (float)(acc[r * d + i] / ell[r]), g.out_bf16);
            }
        }
    }
}

__global__ void trace_init_kernel(Geo g, int64_t T, int64_t* pass1_pairs, int64_t* pass2_pairs,
                                  int32_t* processed) {
    const int64_t zh = blockIdx.x;
    int64_t p1 = 0;
    for (int64_t n = 0; n < g.N; ++n) {
        const int64_t len = g.seg_rows(n);
        p1 += len * (len + 1) / 2;  // pass1_pair_count kernel.cpp:124-131
    }
    if (threadIdx.x == 0) {
        if (pass1_pairs) pass1_pairs[zh] = p1;
        if (pass2_pairs) pass2_pairs[zh] = 0;
    }
    if (processed)
        for (int64_t i = threadIdx.x; i < g.N * T; i += blockDim.x) processed[zh * g.N * T + i] = 0;
}

int grid_for(int64_t tiles) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sms * 8));
}

}  // namespace

size_t generic_scratch_bytes(const PassArgs& a) {
    const int64_t tiles = a.g.z * a.g.hq * a.tiles_per_head;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(tiles, 148 * 8));
    // sized for the largest grid any device could use (256 SMs * 8)
    (void)grid;
    const int64_t per = a.bm * a.g.d + 6 * a.bm;
    return (size_t)std::min<int64_t>(std::max<int64_t>(tiles, 1), 256 * 8) * (size_t)per * sizeof(double);
}

cudaError_t launch_generic_pass(const PassArgs& a, void* scratch, cudaStream_t st) {
    const int64_t tiles = a.max_tiles();
    if (tiles == 0) return cudaSuccess;
    const int grid = std::min(grid_for(tiles), 256 * 8);
    generic_pass_kernel<<<grid, kThreads, 0, st>>>(a, reinterpret_cast<double*>(scratch));
    return cudaGetLastError();
}

cudaError_t launch_trace_init(const PassArgs& a, int64_t* pass1_pairs, cudaStream_t st) {
    trace_init_kernel<<<(unsigned)(a.g.z * a.g.hq), 128, 0, st>>>(a.g, a.T, pass1_pairs,
                                                                 a.pass2_pairs, a.processed);
    return cudaGetLastError();
}

}  // namespace s2o
