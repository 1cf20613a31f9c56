// oracle/ref_capi.cpp -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// A flat extern "C" wrapper around the UNMODIFIED reference implementation
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libs2o_ref.so). It lets the pytest parity suite and bench.py's
// cpu_baseline leg drive the reference's own code path with plain buffers:
//
//   build_plan          proj/src/plan.cpp:140-162
//   pass1_dense_init    proj/src/kernel.cpp:184-218
//   pass2_sparse        proj/src/kernel.cpp:236-298
//   fused_single_pass   proj/src/kernel.cpp:300-349
//   s2o_attention       proj/src/kernel.cpp:351-369
//   early_stop_check    proj/src/kernel.cpp:220-234
//   argsort_desc_stable proj/src/tensor.cpp:43-61
//   segment_representatives proj/src/plan.cpp:46-67
//   dense_causal_attention  proj/src/attention.cpp:90-125
//   generate_synthetic  proj/src/synthetic.cpp:276-328
//   save/load_tensor_file   proj/src/tensor_io.cpp:32-83 (S2OT)
//   block_topk_attention    proj/src/baseline.cpp (block top-k baseline)
//   run_sweep               proj/src/sweep.cpp:141-302 (report-format goldens)
//
// Flat layouts (shared with oracle/s2o_oracle.c and include/s2o_cuda.h):
//   tensors      fp32 [Z,H,L,D] row-major
//   q_perm       int64 [Z*H][N][S]  (segment-local offsets; last segment uses last_len slots)
//   kv_perm      int64 per (z,h): S*N*(N-1)/2 entries, segment n at S*n*(n-1)/2 (absolute ids)
//   trace        int64 [Z*H][N][ceil(S/b_m)]  committed chunk counts
//   pass bufs    fp64 acc [Z,H,L,D], ell/m [Z,H,L]
// Every entry point returns 0 on success, otherwise a nonzero code with the
// exception text available from ref_last_error().

#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <limits>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "s2o/attention.hpp"
#include "s2o/baseline.hpp"
#include "s2o/kernel.hpp"
#include "s2o/metrics.hpp"
#include "s2o/plan.hpp"
#include "s2o/sweep.hpp"
#include "s2o/synthetic.hpp"
#include "s2o/tensor.hpp"
#include "s2o/tensor_io.hpp"

using namespace s2o;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        g_err.clear();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 2;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 5;
    }
}

Tensor4 make_tensor(const float* p, int64_t z, int64_t h, int64_t l, int64_t d) {
    Tensor4 t(z, h, l, d);
    std::memcpy(t.data.data(), p, t.data.size() * sizeof(float));
    return t;
}

void store_tensor(const Tensor4& t, float* out) {
    std::memcpy(out, t.data.data(), t.data.size() * sizeof(float));
}

KernelConfig make_cfg(int64_t seg_len, double tau, int64_t b_m, int64_t b_n, int q_reorder,
                      int fused, int64_t local_window) {
    KernelConfig cfg;
    cfg.seg_len = seg_len;
    cfg.tau = tau;
    cfg.tiles = TileSpec{b_m, b_n};
    cfg.q_reorder = q_reorder != 0;
    cfg.fused = fused != 0;
    cfg.local_window = local_window;
    return cfg;
}

int64_t packed_kv_per_head(const SegmentConfig& seg) {
    return seg.seg_len * seg.seg_count * (seg.seg_count - 1) / 2;
}

void store_plan(const PermutationPlan& plan, int64_t* q_perm, int64_t* kv_perm) {
    const SegmentConfig& seg = plan.seg;
    const int64_t per_head = packed_kv_per_head(seg);
    for (int64_t zh = 0; zh < plan.z * plan.h; ++zh) {
        for (int64_t n = 0; n < seg.seg_count; ++n) {
            const IndexVec& qp = plan.q_perm[static_cast<size_t>(zh * seg.seg_count + n)];
            if (q_perm) {
                std::memcpy(q_perm + (zh * seg.seg_count + n) * seg.seg_len, qp.idx.data(),
                            qp.idx.size() * sizeof(int64_t));
            }
            const IndexVec& kv = plan.kv_perm[static_cast<size_t>(zh * seg.seg_count + n)];
            if (kv_perm && !kv.idx.empty()) {
                std::memcpy(kv_perm + zh * per_head + seg.seg_len * n * (n - 1) / 2,
                            kv.idx.data(), kv.idx.size() * sizeof(int64_t));
            }
        }
    }
}

PermutationPlan load_plan(int64_t z, int64_t h, int64_t l, int64_t seg_len,
                          const int64_t* q_perm, const int64_t* kv_perm) {
    PermutationPlan plan;
    plan.z = z;
    plan.h = h;
    plan.seg = SegmentConfig::for_sequence(l, seg_len);
    plan.guide_source = "k_mean[segment 0]";
    const SegmentConfig& seg = plan.seg;
    const int64_t per_head = packed_kv_per_head(seg);
    for (int64_t zh = 0; zh < z * h; ++zh) {
        for (int64_t n = 0; n < seg.seg_count; ++n) {
            const int64_t len = seg.len(n);
            const int64_t* qp = q_perm + (zh * seg.seg_count + n) * seg.seg_len;
            plan.q_perm.emplace_back(std::vector<int64_t>(qp, qp + len), len);
            const int64_t prefix = seg.prefix_len(n);
            const int64_t* kv = kv_perm + zh * per_head + seg.seg_len * n * (n - 1) / 2;
            plan.kv_perm.emplace_back(std::vector<int64_t>(kv, kv + prefix), prefix);
        }
    }
    return plan;
}

void store_trace(const KernelTrace& trace, int64_t tiles_per_seg, int64_t* processed,
                 int64_t* pass1_pairs, int64_t* pass2_pairs) {
    const int64_t zh_count = trace.z * trace.h;
    for (int64_t zh = 0; zh < zh_count; ++zh) {
        const auto& per_seg = trace.processed_tiles[static_cast<size_t>(zh)];
        for (size_t n = 0; n < per_seg.size(); ++n) {
            int64_t* dst = processed + (zh * static_cast<int64_t>(per_seg.size()) +
                                        static_cast<int64_t>(n)) * tiles_per_seg;
            for (int64_t t = 0; t < tiles_per_seg; ++t) {
                dst[t] = t < static_cast<int64_t>(per_seg[n].size()) ? per_seg[n][t] : 0;
            }
        }
        if (pass1_pairs) pass1_pairs[zh] = trace.pass1_pairs[static_cast<size_t>(zh)];
        if (pass2_pairs) pass2_pairs[zh] = trace.pass2_pairs[static_cast<size_t>(zh)];
    }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_argsort_desc_stable(const double* scores, int64_t n, int64_t* out) {
    return guarded([&] {
        const IndexVec idx = argsort_desc_stable(std::span<const double>(scores, static_cast<size_t>(n)));
        std::memcpy(out, idx.idx.data(), idx.idx.size() * sizeof(int64_t));
    });
}

int ref_early_stop_check(const double* prev_ell, const double* new_ell, int64_t n, double tau,
                         int* stop) {
    return guarded([&] {
        *stop = early_stop_check(std::span<const double>(prev_ell, static_cast<size_t>(n)),
                                 std::span<const double>(new_ell, static_cast<size_t>(n)), tau)
                    ? 1
                    : 0;
    });
}

int ref_segment_representatives(const float* q, const float* k, int64_t z, int64_t h, int64_t l,
                                int64_t d, int64_t seg_len, float* q_mean, float* k_mean) {
    return guarded([&] {
        const SegmentConfig seg = SegmentConfig::for_sequence(l, seg_len);
        const Representatives reps =
            segment_representatives(make_tensor(q, z, h, l, d), make_tensor(k, z, h, l, d), seg);
        std::memcpy(q_mean, reps.q_mean.data.data(), reps.q_mean.data.size() * sizeof(float));
        std::memcpy(k_mean, reps.k_mean.data.data(), reps.k_mean.data.size() * sizeof(float));
    });
}

int ref_build_plan(const float* q, const float* k, int64_t z, int64_t h, int64_t l, int64_t d,
                   int64_t seg_len, int64_t* q_perm, int64_t* kv_perm, int64_t* cost2) {
    return guarded([&] {
        auto [plan, cost] = build_plan(make_tensor(q, z, h, l, d), make_tensor(k, z, h, l, d), seg_len);
        store_plan(plan, q_perm, kv_perm);
        if (cost2) {
            cost2[0] = cost.dot_products;
            cost2[1] = cost.sort_items;
        }
    });
}

int ref_pass1(const float* q, const float* k, const float* v, int64_t z, int64_t h, int64_t l,
              int64_t d, int64_t seg_len, double tau, int64_t b_m, int64_t b_n, int q_reorder,
              int fused, int64_t local_window, double* acc, double* ell, double* m) {
    return guarded([&] {
        const KernelConfig cfg = make_cfg(seg_len, tau, b_m, b_n, q_reorder, fused, local_window);
        const PassBuffers bufs = pass1_dense_init(make_tensor(q, z, h, l, d), make_tensor(k, z, h, l, d),
                                                  make_tensor(v, z, h, l, d), cfg);
        std::memcpy(acc, bufs.acc.data(), bufs.acc.size() * sizeof(double));
        std::memcpy(ell, bufs.ell.data(), bufs.ell.size() * sizeof(double));
        std::memcpy(m, bufs.m.data(), bufs.m.size() * sizeof(double));
    });
}

int ref_pass2(const float* q, const float* k, const float* v, int64_t z, int64_t h, int64_t l,
              int64_t d, int64_t seg_len, double tau, int64_t b_m, int64_t b_n, int q_reorder,
              int fused, int64_t local_window, const double* acc, const double* ell,
              const double* m, const int64_t* q_perm, const int64_t* kv_perm, float* out,
              int64_t* processed, int64_t* pass1_pairs, int64_t* pass2_pairs) {
    return guarded([&] {
        const KernelConfig cfg = make_cfg(seg_len, tau, b_m, b_n, q_reorder, fused, local_window);
        PassBuffers bufs(z, h, l, d);
        std::memcpy(bufs.acc.data(), acc, bufs.acc.size() * sizeof(double));
        std::memcpy(bufs.ell.data(), ell, bufs.ell.size() * sizeof(double));
        std::memcpy(bufs.m.data(), m, bufs.m.size() * sizeof(double));
        const PermutationPlan plan = load_plan(z, h, l, seg_len, q_perm, kv_perm);
        auto [o, trace] = pass2_sparse(make_tensor(q, z, h, l, d), make_tensor(k, z, h, l, d),
                                       make_tensor(v, z, h, l, d), bufs, plan, cfg);
        store_tensor(o, out);
        store_trace(trace, (seg_len + b_m - 1) / b_m, processed, pass1_pairs, pass2_pairs);
    });
}

int ref_fused(const float* q, const float* k, const float* v, int64_t z, int64_t h, int64_t l,
              int64_t d, int64_t seg_len, double tau, int64_t b_m, int64_t b_n, int q_reorder,
              int fused, int64_t local_window, const int64_t* q_perm, const int64_t* kv_perm,
              float* out, int64_t* processed, int64_t* pass1_pairs, int64_t* pass2_pairs) {
    return guarded([&] {
        const KernelConfig cfg = make_cfg(seg_len, tau, b_m, b_n, q_reorder, fused, local_window);
        const PermutationPlan plan = load_plan(z, h, l, seg_len, q_perm, kv_perm);
        auto [o, trace] = fused_single_pass(make_tensor(q, z, h, l, d), make_tensor(k, z, h, l, d),
                                            make_tensor(v, z, h, l, d), plan, cfg);
        store_tensor(o, out);
        store_trace(trace, (seg_len + b_m - 1) / b_m, processed, pass1_pairs, pass2_pairs);
    });
}

int ref_attention(const float* q, const float* k, const float* v, int64_t z, int64_t h, int64_t l,
                  int64_t d, int64_t seg_len, double tau, int64_t b_m, int64_t b_n, int q_reorder,
                  int fused, int64_t local_window, float* out, int64_t* q_perm, int64_t* kv_perm,
                  int64_t* processed, int64_t* pass1_pairs, int64_t* pass2_pairs, int64_t* cost2) {
    return guarded([&] {
        const KernelConfig cfg = make_cfg(seg_len, tau, b_m, b_n, q_reorder, fused, local_window);
        const S2oResult res = s2o_attention(make_tensor(q, z, h, l, d), make_tensor(k, z, h, l, d),
                                            make_tensor(v, z, h, l, d), cfg);
        store_tensor(res.out, out);
        store_plan(res.plan, q_perm, kv_perm);
        store_trace(res.trace, (seg_len + b_m - 1) / b_m, processed, pass1_pairs, pass2_pairs);
        if (cost2) {
            cost2[0] = res.cost.dot_products;
            cost2[1] = res.cost.sort_items;
        }
    });
}

int ref_dense_causal(const float* q, const float* k, const float* v, int64_t z, int64_t h,
                     int64_t l, int64_t d, float* out) {
    return guarded([&] {
        store_tensor(dense_causal_attention(make_tensor(q, z, h, l, d), make_tensor(k, z, h, l, d),
                                            make_tensor(v, z, h, l, d)),
                     out);
    });
}

int ref_generate_synthetic(const char* pattern, int64_t stripe_count, double stripe_gain,
                           uint64_t seed, int64_t z, int64_t h, int64_t l, int64_t d, float* q,
                           float* k, float* v) {
    return guarded([&] {
        SyntheticSpec spec;
        spec.pattern = parse_stripe_pattern(pattern);
        spec.stripe_count = stripe_count;
        spec.stripe_gain = stripe_gain;
        spec.seed = seed;
        const SyntheticData data = generate_synthetic(spec, z, h, l, d);
        store_tensor(data.q, q);
        store_tensor(data.k, k);
        store_tensor(data.v, v);
    });
}

int ref_save_tensor(const char* path, const float* x, int64_t z, int64_t h, int64_t l, int64_t d) {
    return guarded([&] { save_tensor_file(make_tensor(x, z, h, l, d), path); });
}

// dims[4] = {z, h, l, d}; out (if non-null) receives the fp32 data
int ref_load_tensor(const char* path, int64_t* dims, float* out) {
    return guarded([&] {
        const Tensor4 t = load_tensor_file(path);
        dims[0] = t.z;
        dims[1] = t.h;
        dims[2] = t.l;
        dims[3] = t.d;
        if (out) store_tensor(t, out);
    });
}

int ref_block_topk(const float* q, const float* k, const float* v, int64_t z, int64_t h, int64_t l,
                   int64_t d, int64_t block_rows, int64_t block_cols, int64_t topk, float* out,
                   int64_t* pair_count) {
    return guarded([&] {
        BlockBudget b;
        b.block_rows = block_rows;
        b.block_cols = block_cols;
        b.k = topk;
        const BlockTopkResult r = block_topk_attention(make_tensor(q, z, h, l, d), make_tensor(k, z, h, l, d),
                                                       make_tensor(v, z, h, l, d), b);
        store_tensor(r.out, out);
        for (size_t i = 0; i < r.pair_count.size(); ++i) pair_count[i] = r.pair_count[i];
    });
}

// run_sweep on a synthetic input; variants comma-separated; writes <out_base>.{json,csv}.
// Returns 0, or 7 when the sweep itself recorded a failure (partial report).
int ref_run_sweep(const char* pattern, int64_t stripe_count, double stripe_gain, uint64_t seed, int64_t z,
                  int64_t h, int64_t l, int64_t d, const char* variants, const int64_t* seg_lens, int64_t n_seg,
                  const double* taus, int64_t n_tau, int64_t b_m, int64_t b_n, const int64_t* topk, int64_t n_topk,
                  int64_t block_rows, int64_t block_cols, int dump_plan, const char* out_base) {
    int partial = 0;
    std::string err;
    const int rc = guarded([&] {
        RunConfig cfg;
        SyntheticSpec spec;
        spec.pattern = parse_stripe_pattern(pattern);
        spec.stripe_count = stripe_count;
        spec.stripe_gain = stripe_gain;
        spec.seed = seed;
        cfg.synthetic = spec;
        cfg.z = z;
        cfg.h = h;
        cfg.l = l;
        cfg.d = d;
        cfg.variants.clear();
        std::string names(variants);
        for (size_t a = 0; a <= names.size();) {
            const size_t b = names.find(',', a);
            const std::string one = names.substr(a, b == std::string::npos ? std::string::npos : b - a);
            if (!one.empty()) cfg.variants.push_back(parse_variant(one));
            if (b == std::string::npos) break;
            a = b + 1;
        }
        cfg.seg_lens.assign(seg_lens, seg_lens + n_seg);
        cfg.taus.assign(taus, taus + n_tau);
        cfg.tiles = TileSpec{b_m, b_n};
        cfg.topk.assign(topk, topk + n_topk);
        cfg.block_shape = BlockBudget{block_rows, block_cols, 0};
        cfg.dump_plan = dump_plan != 0;
        cfg.out_base = out_base;
        const SweepResult r = run_sweep(cfg);
        if (r.partial) {
            err = r.error;
            partial = 1;
        }
    });
    if (rc == 0 && partial) g_err = err;
    return rc != 0 ? rc : (partial ? 7 : 0);
}

// Stop-decision evidence: the relative normaliser gain max_r (new-prev)/prev of
// each of the first `nchunks` kv_perm chunks of ONE query tile, with every chunk committed, built
// from the reference's own os_update (attention.cpp:31-88) exactly as traverse_prefix
// (kernel.cpp:86-122) would see it up to its stop chunk. rows: segment-local query rows of the tile
// (q_perm order for pass-2, t0.. for fused); each row's pass-1 state is the reference's per-row
// result of segment_causal_tile (kernel.cpp:36-71: b_n key chunks of the segment, masked by original
// position; rows are independent inside os_update). qh/kh/vh: one head [L, D] fp32; kv_seg: the nS
// absolute token ids of kv_perm[n]. gains[c] = NaN for a chunk past the list.
int ref_tile_gains(const float* qh, const float* kh, const float* vh, int64_t l, int64_t d, int64_t seg_len,
                   int64_t b_n, const int64_t* rows, int64_t tn, int64_t n, const int64_t* kv_seg,
                   int64_t nchunks, double* gains) {
    return guarded([&] {
        const int64_t sb = n * seg_len;
        const int64_t kv_len = n * seg_len;
        std::vector<OnlineSoftmaxState> st(static_cast<std::size_t>(tn), OnlineSoftmaxState(d));
        RowMatrix qt(tn, d), kt, vt;
        for (int64_t r = 0; r < tn; ++r) std::memcpy(qt.row(r), qh + (sb + rows[r]) * d, sizeof(float) * d);
        auto load = [&](RowMatrix& dst, const float* src, const int64_t* ids, int64_t cnt) {
            dst = RowMatrix(cnt, d);
            for (int64_t j = 0; j < cnt; ++j) std::memcpy(dst.row(j), src + ids[j] * d, sizeof(float) * d);
        };
        // pass-1 state, one row at a time (identical to the tile-wide scan: os_update is per row)
        std::vector<int64_t> ids;
        for (int64_t r = 0; r < tn; ++r) {
            RowMatrix q1(1, d);
            std::memcpy(q1.row(0), qt.row(r), sizeof(float) * d);
            std::span<OnlineSoftmaxState> one(&st[static_cast<std::size_t>(r)], 1);
            const int64_t rr = rows[r];
            const int64_t seg_rows = std::min(seg_len, l - sb);
            for (int64_t k0 = 0; k0 <= rr && k0 < seg_rows; k0 += b_n) {
                const int64_t kn = std::min(b_n, seg_rows - k0);
                ids.resize(static_cast<std::size_t>(kn));
                for (int64_t j = 0; j < kn; ++j) ids[static_cast<std::size_t>(j)] = sb + k0 + j;
                load(kt, kh, ids.data(), kn);
                load(vt, vh, ids.data(), kn);
                if (k0 + kn - 1 <= rr) {
                    os_update(one, q1, kt, vt);
                } else {
                    std::vector<std::uint8_t> mask(static_cast<std::size_t>(kn));
                    for (int64_t j = 0; j < kn; ++j) mask[static_cast<std::size_t>(j)] = (k0 + j <= rr) ? 1 : 0;
                    os_update(one, q1, kt, vt, mask);
                }
            }
        }
        std::vector<OnlineSoftmaxState> cand(st.size(), OnlineSoftmaxState(d));
        for (int64_t c = 0; c < nchunks; ++c) {
            const int64_t c0 = c * b_n;
            if (c0 >= kv_len) {
                gains[c] = std::numeric_limits<double>::quiet_NaN();
                continue;
            }
            const int64_t cn = std::min(b_n, kv_len - c0);
            load(kt, kh, kv_seg + c0, cn);
            load(vt, vh, kv_seg + c0, cn);
            for (std::size_t r = 0; r < st.size(); ++r) {
                cand[r].m = st[r].m;
                cand[r].ell = st[r].ell;
                cand[r].acc = st[r].acc;
            }
            os_update(std::span<OnlineSoftmaxState>(cand), qt, kt, vt);
            double max_gain = -std::numeric_limits<double>::infinity();
            for (std::size_t r = 0; r < st.size(); ++r) {
                const double prev = st[r].ell * std::exp(st[r].m - cand[r].m);
                max_gain = std::max(max_gain, (cand[r].ell - prev) / prev);  // kernel.cpp:226-232
            }
            gains[c] = max_gain;
            st.swap(cand);  // commit
        }
    });
}

int ref_rng_normals(uint64_t seed, int64_t n, double* out) {
    return guarded([&] {
        Rng rng(seed);
        for (int64_t i = 0; i < n; ++i) out[i] = rng.normal();
    });
}

uint64_t ref_mix_seed(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
    return mix_seed(seed, a, b, c);
}

}  // extern "C"
