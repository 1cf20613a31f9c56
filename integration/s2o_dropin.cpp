// integration/s2o_dropin.cpp -- the reference's hot-path API on the B200 kernels.
//
// Defines, with the reference's own declarations (/root/reference/proj/include/s2o/plan.hpp and
// kernel.hpp), every function of the two translation units it replaces -- src/plan.cpp and
// src/kernel.cpp -- on top of the C-ABI in include/s2o_cuda.h (libs2o_cuda.so):
//
//   SegmentConfig::for_sequence   plan.hpp:21      host (same checks and message)
//   segment_representatives       plan.hpp:100-102 s2o_segment_representatives
//   rank_queries                  plan.hpp:104-106 s2o_rank_queries
//   rank_prefix_keys              plan.hpp:108-111 s2o_rank_prefix_keys
//   build_plan                    plan.hpp:115-116 s2o_plan_build
//   KernelConfig::validate        kernel.hpp:27    s2o_kernel_config_validate
//   pass1_dense_init              kernel.hpp:70-71 s2o_pass1
//   early_stop_check              kernel.hpp:77-78 s2o_early_stop_check
//   pass2_sparse                  kernel.hpp:83-86 s2o_pass2 (+ s2o_pass_status)
//   fused_single_pass             kernel.hpp:92-95 s2o_fused (+ s2o_pass_status)
//   s2o_attention                 kernel.hpp:106-107 s2o_attention_fwd (+ s2o_attention_status)
//
// so a program built against the reference links this object in place of plan.o / kernel.o and
// runs unchanged (integration/Makefile links the reference's tests/acceptance_main.cpp this way).
// Tensor4 (host fp32) moves to the device and back per call; PermutationPlan, KernelTrace and
// PassBuffers are rebuilt from the device arrays. PassBuffers carry the device pass state, which is
// fp32 (acc, ell, m), widened to the reference's fp64 vectors. Status codes become the reference's
// exception types with the same messages.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "s2o/kernel.hpp"
#include "s2o/plan.hpp"
#include "s2o/tensor.hpp"
#include "s2o_cuda.h"

namespace s2o {
namespace {

// s2o_status -> the reference's exception (same text: s2o_last_error()).
void check(s2o_status st) {
    if (st == S2O_OK) return;
    const std::string msg = s2o_last_error()[0] ? s2o_last_error() : s2o_status_string(st);
    switch (st) {
        case S2O_ERR_UNCOVERED_ROW:
        case S2O_ERR_CUDA:
        case S2O_ERR_NO_DEVICE:
            throw std::runtime_error(msg);
        default:
            throw std::invalid_argument(msg);
    }
}

void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Device buffer owned for the duration of one call.
struct Dev {
    void* p = nullptr;
    explicit Dev(size_t bytes) {
        if (bytes) cuda(cudaMalloc(&p, bytes), "cudaMalloc");
    }
    ~Dev() {
        if (p) cudaFree(p);
    }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

template <typename T>
void h2d(const Dev& d, const T* src, size_t n) {
    if (n) cuda(cudaMemcpy(d.p, src, n * sizeof(T), cudaMemcpyHostToDevice), "h2d");
}
template <typename T>
void d2h(T* dst, const Dev& d, size_t n) {
    if (n) cuda(cudaMemcpy(dst, d.p, n * sizeof(T), cudaMemcpyDeviceToHost), "d2h");
}

size_t nelem(const Tensor4& t) { return t.data.size(); }

s2o_problem problem(const Tensor4& q, const Tensor4& k) {
    s2o_problem p;
    s2o_problem_init(&p, q.z, q.h, k.h, q.l, q.d, S2O_F32, S2O_F32);
    return p;
}

s2o_kernel_config kcfg(const KernelConfig& c) {
    s2o_kernel_config k;
    s2o_kernel_config_init(&k);
    k.seg_len = c.seg_len;
    k.tau = c.tau;
    k.b_m = c.tiles.b_m;
    k.b_n = c.tiles.b_n;
    k.q_reorder = c.q_reorder ? 1 : 0;
    k.fused = c.fused ? 1 : 0;
    k.local_window = c.local_window;
    return k;
}

void dims_match(const Tensor4& q, const Tensor4& k, const Tensor4& v) {
    if (!q.same_dims(k) || !q.same_dims(v)) throw std::invalid_argument("Q/K/V dims must match");
}

// check_plan_matches (kernel.cpp:26-33)
void plan_matches(const PermutationPlan& plan, const Tensor4& q, const KernelConfig& cfg) {
    const SegmentConfig want = SegmentConfig::for_sequence(q.l, cfg.seg_len);
    if (plan.z != q.z || plan.h != q.h || plan.seg.seg_len != want.seg_len ||
        plan.seg.seg_count != want.seg_count || plan.seg.last_len != want.last_len)
        throw std::invalid_argument("plan/config mismatch: segment layout differs");
}

int64_t kv_per_head(const SegmentConfig& s) { return s.seg_len * s.seg_count * (s.seg_count - 1) / 2; }

// PermutationPlan -> the device layouts (q_perm int32 [ZH][N][S], kv_perm int32 packed per head).
// Indices are validated like gather_rows_into (tensor.cpp:86-99: "gather index out of bounds").
void flatten_plan(const PermutationPlan& plan, int64_t l, std::vector<int32_t>& qp, std::vector<int32_t>& kv) {
    const SegmentConfig& s = plan.seg;
    const int64_t zh = plan.z * plan.h;
    qp.assign(static_cast<size_t>(zh * s.seg_count * s.seg_len), 0);
    kv.assign(static_cast<size_t>(std::max<int64_t>(1, zh * kv_per_head(s))), 0);
    for (int64_t i = 0; i < zh; ++i)
        for (int64_t n = 0; n < s.seg_count; ++n) {
            const size_t slot = static_cast<size_t>(i * s.seg_count + n);
            if (slot < plan.q_perm.size()) {
                const auto& v = plan.q_perm[slot].idx;
                for (size_t r = 0; r < v.size() && (int64_t)r < s.len(n); ++r) {
                    if (v[r] < 0 || v[r] >= s.len(n)) throw std::out_of_range("gather index out of bounds");
                    qp[static_cast<size_t>((i * s.seg_count + n) * s.seg_len) + r] = static_cast<int32_t>(v[r]);
                }
            }
            if (n > 0 && slot < plan.kv_perm.size()) {
                const auto& v = plan.kv_perm[slot].idx;
                const int64_t off = i * kv_per_head(s) + s.seg_len * n * (n - 1) / 2;
                for (size_t t = 0; t < v.size() && (int64_t)t < n * s.seg_len; ++t) {
                    if (v[t] < 0 || v[t] >= l) throw std::out_of_range("gather index out of bounds");
                    kv[static_cast<size_t>(off) + t] = static_cast<int32_t>(v[t]);
                }
            }
        }
}

PermutationPlan rebuild_plan(int64_t z, int64_t h, const SegmentConfig& s, const std::vector<int32_t>& qp,
                             const std::vector<int32_t>& kv) {
    PermutationPlan plan;
    plan.z = z;
    plan.h = h;
    plan.seg = s;
    plan.guide_source = "k_mean[segment 0]";
    plan.q_perm.resize(static_cast<size_t>(z * h * s.seg_count));
    plan.kv_perm.resize(plan.q_perm.size());
    for (int64_t i = 0; i < z * h; ++i)
        for (int64_t n = 0; n < s.seg_count; ++n) {
            const size_t slot = static_cast<size_t>(i * s.seg_count + n);
            const int32_t* q0 = qp.data() + (i * s.seg_count + n) * s.seg_len;
            plan.q_perm[slot] = IndexVec(std::vector<int64_t>(q0, q0 + s.len(n)), s.len(n));
            if (n == 0) {
                plan.kv_perm[slot] = IndexVec({}, 0);
            } else {
                const int32_t* k0 = kv.data() + i * kv_per_head(s) + s.seg_len * n * (n - 1) / 2;
                plan.kv_perm[slot] = IndexVec(std::vector<int64_t>(k0, k0 + n * s.seg_len), n * s.seg_len);
            }
        }
    return plan;
}

KernelTrace rebuild_trace(const Tensor4& q, const KernelConfig& cfg, const SegmentConfig& s,
                          const std::vector<int32_t>& proc, const std::vector<int64_t>& p1,
                          const std::vector<int64_t>& p2) {
    KernelTrace tr;
    tr.z = q.z;
    tr.h = q.h;
    tr.l = q.l;
    tr.seg_len = cfg.seg_len;
    tr.tiles = cfg.tiles;
    const int64_t T = (s.seg_len + cfg.tiles.b_m - 1) / cfg.tiles.b_m;
    tr.processed_tiles.resize(static_cast<size_t>(q.z * q.h));
    for (int64_t i = 0; i < q.z * q.h; ++i) {
        auto& per = tr.processed_tiles[static_cast<size_t>(i)];
        per.resize(static_cast<size_t>(s.seg_count));
        for (int64_t n = 0; n < s.seg_count; ++n) {
            const int64_t tiles = (s.len(n) + cfg.tiles.b_m - 1) / cfg.tiles.b_m;
            const int32_t* row = proc.data() + (i * s.seg_count + n) * T;
            per[static_cast<size_t>(n)].assign(row, row + tiles);
        }
    }
    tr.pass1_pairs = p1;
    tr.pass2_pairs = p2;
    return tr;
}

// Device copies of Q, K, V (fp32, dense [Z,H,L,D]).
struct Inputs {
    Dev q, k, v;
    Inputs(const Tensor4& tq, const Tensor4& tk, const Tensor4* tv)
        : q(nelem(tq) * sizeof(float)), k(nelem(tk) * sizeof(float)), v(tv ? nelem(*tv) * sizeof(float) : 0) {
        h2d(q, tq.data.data(), nelem(tq));
        h2d(k, tk.data.data(), nelem(tk));
        if (tv) h2d(v, tv->data.data(), nelem(*tv));
    }
};

size_t plan_ws(const s2o_problem& p, int64_t seg_len) {
    size_t b = 0;
    check(s2o_plan_workspace_size(&p, seg_len, &b));
    return b;
}
size_t pass_ws(const s2o_problem& p, const s2o_kernel_config& c) {
    size_t b = 0;
    check(s2o_pass_workspace_size(&p, &c, &b));
    return b;
}

std::pair<Tensor4, KernelTrace> run_prefix_pass(const Tensor4& q, const Tensor4& k, const Tensor4& v,
                                                const PassBuffers* bufs, const PermutationPlan& plan,
                                                const KernelConfig& cfg) {
    const s2o_problem p = problem(q, k);
    const s2o_kernel_config c = kcfg(cfg);
    const SegmentConfig& s = plan.seg;
    std::vector<int32_t> qp, kv;
    flatten_plan(plan, q.l, qp, kv);
    Inputs in(q, k, &v);
    Dev dqp(qp.size() * 4), dkv(kv.size() * 4), out(nelem(q) * 4);
    h2d(dqp, qp.data(), qp.size());
    h2d(dkv, kv.data(), kv.size());
    const int64_t zh = q.z * q.h;
    const int64_t T = (s.seg_len + cfg.tiles.b_m - 1) / cfg.tiles.b_m;
    Dev proc(static_cast<size_t>(zh * s.seg_count * T) * 4), p1(zh * 8), p2(zh * 8);
    const size_t wsb = pass_ws(p, c);
    Dev ws(wsb);
    if (bufs) {
        const size_t rows = static_cast<size_t>(zh * q.l);
        std::vector<float> acc(bufs->acc.begin(), bufs->acc.end()), ell(bufs->ell.begin(), bufs->ell.end()),
            m(bufs->m.begin(), bufs->m.end());
        Dev dacc(acc.size() * 4), dell(rows * 4), dm(rows * 4);
        h2d(dacc, acc.data(), acc.size());
        h2d(dell, ell.data(), rows);
        h2d(dm, m.data(), rows);
        check(s2o_pass2(&p, in.q.p, in.k.p, in.v.p, &c, dacc.as<float>(), dell.as<float>(), dm.as<float>(),
                        dqp.as<int32_t>(), dkv.as<int32_t>(), out.p, proc.as<int32_t>(), p1.as<int64_t>(),
                        p2.as<int64_t>(), ws.p, wsb, nullptr));
        check(s2o_pass_status(&p, &c, ws.p, wsb, nullptr));
    } else {
        check(s2o_fused(&p, in.q.p, in.k.p, in.v.p, &c, dkv.as<int32_t>(), out.p, proc.as<int32_t>(),
                        p1.as<int64_t>(), p2.as<int64_t>(), ws.p, wsb, nullptr));
        check(s2o_pass_status(&p, &c, ws.p, wsb, nullptr));
    }
    Tensor4 o(q.z, q.h, q.l, q.d);
    d2h(o.data.data(), out, nelem(o));
    std::vector<int32_t> hp(static_cast<size_t>(zh * s.seg_count * T));
    std::vector<int64_t> h1(static_cast<size_t>(zh)), h2(static_cast<size_t>(zh));
    d2h(hp.data(), proc, hp.size());
    d2h(h1.data(), p1, h1.size());
    d2h(h2.data(), p2, h2.size());
    return {std::move(o), rebuild_trace(q, cfg, s, hp, h1, h2)};
}

}  // namespace

SegmentConfig SegmentConfig::for_sequence(std::int64_t l, std::int64_t seg_len) {
    if (seg_len < 1 || seg_len > l) throw std::invalid_argument("segment length must satisfy 1 <= S <= L");
    SegmentConfig c;
    c.seg_len = seg_len;
    c.seg_count = (l + seg_len - 1) / seg_len;
    c.last_len = l - (c.seg_count - 1) * seg_len;
    return c;
}

Representatives segment_representatives(const Tensor4& q, const Tensor4& k, const SegmentConfig& seg) {
    if (!q.same_dims(k)) throw std::invalid_argument("Q/K/V dims must match");
    const s2o_problem p = problem(q, k);
    Inputs in(q, k, nullptr);
    Representatives reps;
    reps.q_mean = SegmentVectors(q.z, q.h, seg.seg_count, q.d);
    reps.k_mean = SegmentVectors(k.z, k.h, seg.seg_count, k.d);
    Dev qm(reps.q_mean.data.size() * 4), km(reps.k_mean.data.size() * 4);
    check(s2o_segment_representatives(&p, in.q.p, in.k.p, seg.seg_len, qm.as<float>(), km.as<float>(), nullptr));
    d2h(reps.q_mean.data.data(), qm, reps.q_mean.data.size());
    d2h(reps.k_mean.data.data(), km, reps.k_mean.data.size());
    return reps;
}

std::vector<IndexVec> rank_queries(const Tensor4& q, const HeadVectors& k_guide, const SegmentConfig& seg,
                                   RankingCost* cost) {
    if (k_guide.d != q.d || k_guide.z != q.z || k_guide.h != q.h)
        throw std::invalid_argument("guide vector dims must match Q");
    const s2o_problem p = problem(q, q);
    const size_t wsb = plan_ws(p, seg.seg_len);
    Dev dq(nelem(q) * 4), dg(k_guide.data.size() * 4), ws(wsb);
    Dev qp(static_cast<size_t>(q.z * q.h * seg.seg_count * seg.seg_len) * 4);
    h2d(dq, q.data.data(), nelem(q));
    h2d(dg, k_guide.data.data(), k_guide.data.size());
    check(s2o_rank_queries(&p, dq.p, dg.as<float>(), seg.seg_len, qp.as<int32_t>(), ws.p, wsb, nullptr));
    std::vector<int32_t> hq(static_cast<size_t>(q.z * q.h * seg.seg_count * seg.seg_len));
    d2h(hq.data(), qp, hq.size());
    std::vector<IndexVec> out(static_cast<size_t>(q.z * q.h * seg.seg_count));
    for (int64_t i = 0; i < q.z * q.h; ++i)
        for (int64_t n = 0; n < seg.seg_count; ++n) {
            const int32_t* r = hq.data() + (i * seg.seg_count + n) * seg.seg_len;
            out[static_cast<size_t>(i * seg.seg_count + n)] =
                IndexVec(std::vector<int64_t>(r, r + seg.len(n)), seg.len(n));
        }
    if (cost) {  // per-slice counters (plan.cpp:92-93)
        cost->dot_products += q.l;
        cost->sort_items += q.l;
    }
    return out;
}

std::vector<IndexVec> rank_prefix_keys(const SegmentVectors& q_mean, const Tensor4& k, const SegmentConfig& seg,
                                       RankingCost* cost) {
    if (q_mean.d != k.d || q_mean.z != k.z || q_mean.h != k.h || q_mean.n != seg.seg_count)
        throw std::invalid_argument("q_mean dims must match K and segment config");
    const s2o_problem p = problem(k, k);
    const size_t wsb = plan_ws(p, seg.seg_len);
    const int64_t kvn = std::max<int64_t>(1, k.z * k.h * kv_per_head(seg));
    Dev dk(nelem(k) * 4), dm(q_mean.data.size() * 4), ws(wsb), kv(static_cast<size_t>(kvn) * 4);
    h2d(dk, k.data.data(), nelem(k));
    h2d(dm, q_mean.data.data(), q_mean.data.size());
    check(s2o_rank_prefix_keys(&p, dk.p, dm.as<float>(), seg.seg_len, kv.as<int32_t>(), ws.p, wsb, nullptr));
    std::vector<int32_t> hk(static_cast<size_t>(kvn));
    d2h(hk.data(), kv, hk.size());
    std::vector<int32_t> none(static_cast<size_t>(k.z * k.h * seg.seg_count * seg.seg_len), 0);
    PermutationPlan tmp = rebuild_plan(k.z, k.h, seg, none, hk);
    if (cost) {  // plan.cpp:128-129
        cost->dot_products += kv_per_head(seg);
        cost->sort_items += kv_per_head(seg);
    }
    return std::move(tmp.kv_perm);
}

std::pair<PermutationPlan, RankingCost> build_plan(const Tensor4& q, const Tensor4& k, std::int64_t seg_len) {
    const SegmentConfig seg = SegmentConfig::for_sequence(q.l, seg_len);
    if (!q.same_dims(k)) throw std::invalid_argument("Q/K/V dims must match");
    const s2o_problem p = problem(q, k);
    s2o_kernel_config c;
    s2o_kernel_config_init(&c);
    c.seg_len = seg_len;
    const size_t wsb = plan_ws(p, seg_len);
    Inputs in(q, k, nullptr);
    const int64_t zh = q.z * q.h;
    const size_t nq = static_cast<size_t>(zh * seg.seg_count * seg.seg_len);
    const size_t nk = static_cast<size_t>(std::max<int64_t>(1, zh * kv_per_head(seg)));
    Dev qp(nq * 4), kv(nk * 4), ws(wsb);
    int64_t cost2[2] = {0, 0};
    check(s2o_plan_build(&p, in.q.p, in.k.p, &c, qp.as<int32_t>(), kv.as<int32_t>(), cost2, ws.p, wsb, nullptr));
    std::vector<int32_t> hq(nq), hk(nk);
    d2h(hq.data(), qp, nq);
    d2h(hk.data(), kv, nk);
    RankingCost cost;
    cost.dot_products = cost2[0];
    cost.sort_items = cost2[1];
    return {rebuild_plan(q.z, q.h, seg, hq, hk), cost};
}

void KernelConfig::validate(std::int64_t l) const {
    const s2o_kernel_config c = kcfg(*this);
    check(s2o_kernel_config_validate(&c, l));
}

PassBuffers pass1_dense_init(const Tensor4& q, const Tensor4& k, const Tensor4& v, const KernelConfig& cfg) {
    dims_match(q, k, v);
    cfg.validate(q.l);
    const s2o_problem p = problem(q, k);
    const s2o_kernel_config c = kcfg(cfg);
    Inputs in(q, k, &v);
    const size_t rows = static_cast<size_t>(q.z * q.h * q.l);
    Dev acc(rows * q.d * 4), ell(rows * 4), m(rows * 4);
    const size_t wsb = pass_ws(p, c);
    Dev ws(wsb);
    check(s2o_pass1(&p, in.q.p, in.k.p, in.v.p, &c, acc.as<float>(), ell.as<float>(), m.as<float>(), ws.p, wsb,
                    nullptr));
    std::vector<float> ha(rows * q.d), he(rows), hm(rows);
    d2h(ha.data(), acc, ha.size());
    d2h(he.data(), ell, rows);
    d2h(hm.data(), m, rows);
    PassBuffers bufs(q.z, q.h, q.l, q.d);
    std::copy(ha.begin(), ha.end(), bufs.acc.begin());
    std::copy(he.begin(), he.end(), bufs.ell.begin());
    std::copy(hm.begin(), hm.end(), bufs.m.begin());
    return bufs;
}

bool early_stop_check(std::span<const double> prev_ell, std::span<const double> new_ell, double tau) {
    if (prev_ell.size() != new_ell.size() || prev_ell.empty())
        throw std::invalid_argument("normalizer vectors must align");
    int32_t stop = 0;
    check(s2o_early_stop_check(prev_ell.data(), new_ell.data(), static_cast<int64_t>(prev_ell.size()), tau, &stop));
    return stop != 0;
}

std::pair<Tensor4, KernelTrace> pass2_sparse(const Tensor4& q, const Tensor4& k, const Tensor4& v,
                                             const PassBuffers& bufs, const PermutationPlan& plan,
                                             const KernelConfig& cfg) {
    dims_match(q, k, v);
    cfg.validate(q.l);
    plan_matches(plan, q, cfg);
    if (bufs.z != q.z || bufs.h != q.h || bufs.l != q.l || bufs.d != q.d)
        throw std::invalid_argument("pass buffers do not match tensor dims");
    return run_prefix_pass(q, k, v, &bufs, plan, cfg);
}

std::pair<Tensor4, KernelTrace> fused_single_pass(const Tensor4& q, const Tensor4& k, const Tensor4& v,
                                                  const PermutationPlan& plan, const KernelConfig& cfg) {
    dims_match(q, k, v);
    if (!cfg.fused || cfg.q_reorder) throw std::invalid_argument("fused variant requires fused = true, q_reorder = false");
    cfg.validate(q.l);
    plan_matches(plan, q, cfg);
    return run_prefix_pass(q, k, v, nullptr, plan, cfg);
}

S2oResult s2o_attention(const Tensor4& q, const Tensor4& k, const Tensor4& v, const KernelConfig& cfg) {
    cfg.validate(q.l);
    dims_match(q, k, v);
    const SegmentConfig seg = SegmentConfig::for_sequence(q.l, cfg.seg_len);
    const s2o_problem p = problem(q, k);
    const s2o_kernel_config c = kcfg(cfg);
    size_t wsb = 0;
    check(s2o_attention_workspace_size(&p, &c, &wsb));
    Inputs in(q, k, &v);
    const int64_t zh = q.z * q.h;
    const int64_t T = (seg.seg_len + cfg.tiles.b_m - 1) / cfg.tiles.b_m;
    const size_t nq = static_cast<size_t>(zh * seg.seg_count * seg.seg_len);
    const size_t nk = static_cast<size_t>(std::max<int64_t>(1, zh * kv_per_head(seg)));
    const size_t np = static_cast<size_t>(zh * seg.seg_count * T);
    Dev out(nelem(q) * 4), qp(nq * 4), kv(nk * 4), proc(np * 4), p1(zh * 8), p2(zh * 8), ws(wsb);
    check(s2o_attention_fwd(&p, in.q.p, in.k.p, in.v.p, &c, out.p, qp.as<int32_t>(), kv.as<int32_t>(),
                            proc.as<int32_t>(), p1.as<int64_t>(), p2.as<int64_t>(), ws.p, wsb, nullptr));
    check(s2o_attention_status(&p, &c, ws.p, wsb, nullptr));
    S2oResult res;
    res.out = Tensor4(q.z, q.h, q.l, q.d);
    d2h(res.out.data.data(), out, nelem(res.out));
    std::vector<int32_t> hq(nq), hk(nk), hp(np);
    std::vector<int64_t> h1(static_cast<size_t>(zh)), h2(static_cast<size_t>(zh));
    d2h(hq.data(), qp, nq);
    d2h(hk.data(), kv, nk);
    d2h(hp.data(), proc, np);
    d2h(h1.data(), p1, h1.size());
    d2h(h2.data(), p2, h2.size());
    res.trace = rebuild_trace(q, cfg, seg, hp, h1, h2);
    res.plan = rebuild_plan(q.z, q.h, seg, hq, hk);
    const int64_t dots = q.l + kv_per_head(seg);  // RankingCost per slice (plan.cpp:92-93, 128-129)
    res.cost.dot_products = dots;
    res.cost.sort_items = dots;
    return res;
}

}  // namespace s2o
