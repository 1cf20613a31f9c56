// capi.cu -- the extern "C" boundary (include/s2o_cuda.h): argument checks with the
// reference's exception messages, workspace layout, kernel dispatch, host-buffer entry.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <mutex>
#include <string>
#include <vector>

#include <cub/block/block_scan.cuh>

#include "internal.h"

namespace s2o {
namespace {

thread_local std::string g_err;

s2o_status fail(s2o_status st, const std::string& msg) {
    g_err = msg;
    return st;
}

s2o_status cuda_fail(cudaError_t e, const char* where) {
    return fail(S2O_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define S2O_CUDA_TRY(expr, where)                    \
    do {                                             \
        cudaError_t e_ = (expr);                     \
        if (e_ != cudaSuccess) return cuda_fail(e_, where); \
    } while (0)

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

constexpr int64_t kMaxPlanDepth = 6144;  // 3/4 of select_topk_kernel smem capacity (kSelCap = 8192)
// Level control words at the head of the overflow area: [0] overflow tiles, [1] selection flag,
// [2] segments of the next level, [3] tiles to rerun, [4..5] level base (int64).
constexpr int kCtlWords = 16;

// Geometry + generic argument checks shared by every entry point.
s2o_status make_geo(const s2o_problem* p, int64_t seg_len, Geo* g) {
    if (!p) return fail(S2O_ERR_INVALID_ARG, "null problem");
    if (p->z < 1 || p->hq < 1 || p->hkv < 1 || p->l < 1 || p->d < 1)
        return fail(S2O_ERR_INVALID_ARG, "tensor dims must all be >= 1");
    if (p->hq % p->hkv != 0) return fail(S2O_ERR_QKV_DIMS, "Q/K/V dims must match");
    if ((p->in_dtype != S2O_F32 && p->in_dtype != S2O_BF16) ||
        (p->out_dtype != S2O_F32 && p->out_dtype != S2O_BF16))
        return fail(S2O_ERR_INVALID_ARG, "unknown dtype");
    if (seg_len < 1 || seg_len > p->l)
        return fail(S2O_ERR_SEG_LEN, "segment length must satisfy 1 <= S <= L");
    if (p->d > 512) return fail(S2O_ERR_UNSUPPORTED, "head dim D > 512 is not supported");
    if (p->l > (int64_t(1) << 31) - 1) return fail(S2O_ERR_UNSUPPORTED, "L must fit int32");
    Geo& o = *g;
    o.z = p->z; o.hq = p->hq; o.hkv = p->hkv; o.l = p->l; o.d = p->d;
    o.group = p->hq / p->hkv;
    o.S = seg_len;
    o.N = (p->l + seg_len - 1) / seg_len;
    o.last_len = p->l - (o.N - 1) * seg_len;
    for (int i = 0; i < 3; ++i) {
        o.qs[i] = p->q_stride[i]; o.ks[i] = p->k_stride[i];
        o.vs[i] = p->v_stride[i]; o.os[i] = p->o_stride[i];
    }
    o.in_bf16 = p->in_dtype == S2O_BF16;
    o.out_bf16 = p->out_dtype == S2O_BF16;
    return S2O_OK;
}

s2o_status validate_cfg(const s2o_kernel_config* c, int64_t l) {
    if (!c) return fail(S2O_ERR_INVALID_ARG, "null config");
    if (c->seg_len < 1 || c->seg_len > l)
        return fail(S2O_ERR_SEG_LEN, "segment length must satisfy 1 <= S <= L");
    if (!(c->tau >= 0.0)) return fail(S2O_ERR_TAU, "tau must be >= 0");
    if (c->b_m < 1 || c->b_n < 1) return fail(S2O_ERR_TILES, "tile sizes must be >= 1");
    if (c->local_window > c->seg_len)
        return fail(S2O_ERR_LOCAL_WINDOW, "local window must satisfy W <= S");
    if (c->fused && c->q_reorder)
        return fail(S2O_ERR_FUSED_REORDER, "fused variant requires q_reorder = false");
    if (c->score_mode != S2O_SCORE_EXACT)
        return fail(S2O_ERR_UNSUPPORTED, "only exact (fp64 sequential) scoring is implemented");
    return S2O_OK;
}

PassArgs base_args(const Geo& g, const s2o_kernel_config* c) {
    PassArgs a;
    std::memset(&a, 0, sizeof a);
    a.g = g;
    a.bm = c->b_m;
    a.bn = c->b_n;
    a.tau = c->tau;
    a.scale = 1.0 / std::sqrt((double)g.d);
    a.q_reorder = c->q_reorder;
    a.T = (g.S + c->b_m - 1) / c->b_m;
    a.tiles_per_head = (g.N - 1) * a.T + (g.last_len + c->b_m - 1) / c->b_m;
    return a;
}

bool path_is_tc(const PassArgs& a, int32_t path) {
    if (path == S2O_PATH_GENERIC) return false;
    return tc_supported(a);
}

// Pass scratch: generic path scratch + error flag.
// pass scratch: generic SIMT scratch | flags (err_flag, work_ctr, poison count) | poison tile list
size_t pass_ws_bytes(const PassArgs& a) {
    return align256(generic_scratch_bytes(a)) + 256 + align256(sizeof(int32_t) * a.g.z * a.g.hq * a.tiles_per_head);
}

// The error flag lives in the (caller-owned, uninitialised) pass scratch; every pass clears it
// except a tile-list rerun, which must keep the flags of the tiles it does not revisit.
s2o_status run_pass(PassArgs a, int32_t path, void* ws, size_t ws_bytes, cudaStream_t st, bool clear_flag = true) {
    char* base = reinterpret_cast<char*>(ws);
    if (!ws || ws_bytes < pass_ws_bytes(a)) return fail(S2O_ERR_WORKSPACE, "workspace too small");
    a.err_flag = reinterpret_cast<int32_t*>(base + align256(generic_scratch_bytes(a)));
    a.work_ctr = a.err_flag + 4;  // same 256-B slot
    if (clear_flag) S2O_CUDA_TRY(cudaMemsetAsync(a.err_flag, 0, 8 * sizeof(int32_t), st), "memset");
    else S2O_CUDA_TRY(cudaMemsetAsync(a.work_ctr, 0, sizeof(int32_t), st), "memset");
    if (path == S2O_PATH_TCGEN05 && !tc_supported(a))
        return fail(S2O_ERR_UNSUPPORTED, "tcgen05 path needs bf16 inputs, D=128, b_m=128, b_n=128");
    if (path_is_tc(a, path)) {
        // diagonal passes (pass-1, dense): tiles whose diagonal V block holds a non-finite value
        // (masked keys the tensor core would multiply) are listed by poison_scan_kernel and
        // recomputed by the exact path, which skips masked keys
        static const bool poison_on = [] {  // S2O_POISON_CHECK=0: off (A/B aid)
            const char* e = std::getenv("S2O_POISON_CHECK");
            return !(e && std::strcmp(e, "0") == 0);
        }();
        const bool diag_only = poison_on && (a.mode & kDiag) && !(a.mode & (kPrefix | kStateIn)) && !a.tile_list;
        if (diag_only) {
            PassArgs s = a;
            s.poison_cnt = a.err_flag + 5;
            s.poison_list = reinterpret_cast<int32_t*>(base + align256(generic_scratch_bytes(a)) + 256);
            if (!clear_flag) S2O_CUDA_TRY(cudaMemsetAsync(s.poison_cnt, 0, sizeof(int32_t), st), "memset");
            S2O_CUDA_TRY(launch_poison_scan(s, st), "poison scan");
            S2O_CUDA_TRY(launch_tc_pass(a, st), "tcgen05 pass launch");
            PassArgs r = a;
            r.tile_list = s.poison_list;
            r.tile_count = 0;
            r.tile_count_dev = s.poison_cnt;
            S2O_CUDA_TRY(launch_generic_pass(r, base, st), "poison rerun");
        } else {
            S2O_CUDA_TRY(launch_tc_pass(a, st), "tcgen05 pass launch");
        }
    } else {
        S2O_CUDA_TRY(launch_generic_pass(a, base, st), "generic pass launch");
    }
    return S2O_OK;
}

// Stream/arena for the host-buffer entry point.
struct HostArena {
    std::mutex mu;
    cudaStream_t stream = nullptr;           // compute
    cudaStream_t s_in = nullptr, s_out = nullptr;  // host->device / device->host copies
    cudaEvent_t ev_h2d[2] = {}, ev_comp[2] = {}, ev_d2h[2] = {}, ev_kv[2] = {};
    void* dev = nullptr;
    size_t bytes = 0;
    int32_t* flags = nullptr;  // pinned, one per chunk
    int64_t nflags = 0;
} g_host;

// Block top-k baseline: workspace = fp64 row stats and block masses, the selected token lists,
// fp32 pass-1 state, trace and pass scratch.
struct BtLayout {
    size_t rmax, rden, mass, kvtop, acc, ell, m, proc, p2, pass, total;
};

s2o_status bt_setup(const s2o_problem* p, int64_t rows, int64_t cols, int64_t topk, Geo* g, PassArgs* a,
                           BtLayout* L) {
    if (rows < 1 || cols < 1 || topk < 0)
        return fail(S2O_ERR_BLOCK_BUDGET, "block budget must have positive shape and k >= 0");
    if (rows != cols) return fail(S2O_ERR_UNSUPPORTED, "block top-k baseline needs square blocks");
    s2o_status st = make_geo(p, p ? std::min<int64_t>(rows, p->l) : 0, g);
    if (st) return st;
    s2o_kernel_config c;
    s2o_kernel_config_init(&c);
    c.seg_len = g->S;
    c.tau = 0.0;  // never stops: every selected block is committed
    c.b_m = rows;
    c.b_n = cols;
    c.q_reorder = 0;
    *a = base_args(*g, &c);
    const int64_t zh = g->z * g->hq, nqb = g->N, nkb = (g->l + cols - 1) / cols;
    const int64_t topt = std::max<int64_t>(1, topk * cols);
    size_t off = 0;
    auto take = [&](size_t b) { size_t o = off; off += align256(b); return o; };
    L->rmax = take(sizeof(double) * zh * g->l);
    L->rden = take(sizeof(double) * zh * g->l);
    L->mass = take(sizeof(double) * zh * nqb * nkb);
    L->kvtop = take(sizeof(int32_t) * zh * g->N * topt);
    L->acc = take(sizeof(float) * zh * g->l * g->d);
    L->ell = take(sizeof(float) * zh * g->l);
    L->m = take(sizeof(float) * zh * g->l);
    L->proc = take(sizeof(int32_t) * zh * g->N * a->T);
    L->p2 = take(sizeof(int64_t) * zh);
    L->pass = take(pass_ws_bytes(*a));
    L->total = off + 256;
    return S2O_OK;
}

// ------------------------------------------------------------------ stream-ordered plan levels
// A tile that walks its whole truncated kv list without stopping resumes on the next plan level
// (the following topt entries of the same order). Whether that happens is known only on the
// device, so the level loop is a CUDA graph WHILE node: the body holds two levels (lists A -> B,
// then B -> A), each a prep kernel (reads the overflow count; builds the sorted segment list of
// the overflow tiles; sets the loop condition), the level selection (segment count from device
// memory) and the pass rerun (tile list length from device memory); kernels of an empty level
// exit at once. An IF node after the loop runs the full-plan fallback when a selection could not
// be certified. The nodes go into the caller's graph when `stream` is being captured, else into a
// cached executable graph launched on `stream`: either way nothing synchronises the host.
struct LevelLoop {
    Geo g;
    PassArgs a, a2;
    int32_t path, fused;
    int64_t topt;
    const void *q, *k;
    int32_t *qp, *kvp;
    int64_t* p1;
    int32_t* ctl;
    uint8_t* marks;
    int32_t* seglist;
    int32_t *lists[2], *tiles[2], *bases[2];
    float *acc, *ell, *m;
    char *plan_ws, *pass_ws;
    size_t pass_bytes;
};

__global__ void __launch_bounds__(1024)
level_prep_kernel(int32_t* __restrict__ ctl, const int32_t* __restrict__ tiles_in, int32_t* __restrict__ seglist,
                  uint8_t* __restrict__ marks, int64_t tiles_per_head, int64_t T, int64_t N, int64_t nsegs,
                  int64_t topt, cudaGraphConditionalHandle h_loop, cudaGraphConditionalHandle h_fallback) {
    using Scan = cub::BlockScan<int, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ int s_base;
    const int tid = threadIdx.x;
    const int cnt = ctl[0], flag = ctl[1];
    if (cnt == 0 || flag != 0) {  // no level needed, or a selection failed: leave the loop
        if (tid == 0) {
            ctl[2] = 0;
            ctl[3] = 0;
            cudaGraphSetConditional(h_loop, 0);
            cudaGraphSetConditional(h_fallback, flag != 0 ? 1u : 0u);
        }
        return;
    }
    const int64_t full = (N - 1) * T;
    for (int i = tid; i < cnt; i += blockDim.x) {
        const int64_t t = tiles_in[i], zh = t / tiles_per_head, r = t % tiles_per_head;
        marks[zh * N + (r < full ? r / T : N - 1)] = 1;
    }
    if (tid == 0) s_base = 0;
    __syncthreads();
    for (int64_t c0 = 0; c0 < nsegs; c0 += blockDim.x) {  // segment codes in increasing order
        const int64_t c = c0 + tid;
        const int mk = c < nsegs ? marks[c] : 0;
        int pos, tot;
        Scan(tmp).ExclusiveSum(mk, pos, tot);
        if (mk) {
            seglist[s_base + pos] = (int32_t)c;
            marks[c] = 0;
        }
        __syncthreads();
        if (tid == 0) s_base += tot;
        __syncthreads();
    }
    if (tid == 0) {
        ctl[2] = s_base;
        ctl[3] = cnt;
        ctl[0] = 0;
        *reinterpret_cast<int64_t*>(ctl + 4) += topt;
        cudaGraphSetConditional(h_loop, 1);
    }
}

// The loop body (two levels) and the fallback body, enqueued on `st` (being captured).
s2o_status level_body(const LevelLoop& L, cudaStream_t st, cudaGraphConditionalHandle hl,
                      cudaGraphConditionalHandle hf) {
    const Geo& g = L.g;
    const int64_t nsegs = g.z * g.hq * g.N;
    for (int cur = 0; cur < 2; ++cur) {
        level_prep_kernel<<<1, 1024, 0, st>>>(L.ctl, L.tiles[cur], L.seglist, L.marks, L.a.tiles_per_head, L.a.T,
                                              g.N, nsegs, L.topt, hl, hf);
        S2O_CUDA_TRY(cudaGetLastError(), "level prep");
        S2O_CUDA_TRY(launch_plan_level_dev(g, L.k, L.seglist, L.ctl + 2, L.lists[cur],
                                           reinterpret_cast<const int64_t*>(L.ctl + 4), L.lists[cur ^ 1], L.topt,
                                           L.ctl + 1, L.plan_ws, st), "plan level");
        PassArgs a3 = L.a2;
        if (L.fused) {  // the diagonal part is done: resume the saved state, prefix only
            a3.mode = kStateIn | kPrefix | kFinal;
            a3.acc_in = L.acc; a3.ell_in = L.ell; a3.m_in = L.m;
        }
        a3.kv_perm = L.lists[cur ^ 1];
        a3.lvl_base = 0;
        a3.lvl_base_dev = reinterpret_cast<const int64_t*>(L.ctl + 4);
        a3.tile_list = L.tiles[cur];
        a3.tile_base = L.bases[cur];
        a3.tile_count = 0;
        a3.tile_count_dev = L.ctl + 3;
        a3.ovf_tiles = L.tiles[cur ^ 1];
        a3.ovf_base = L.bases[cur ^ 1];
        if (s2o_status e = run_pass(a3, L.path, L.pass_ws, L.pass_bytes, st, false)) return e;
    }
    return S2O_OK;
}

s2o_status fallback_body(const LevelLoop& L, cudaStream_t st) {
    // a selection could not be certified: full plan, recompute everything
    S2O_CUDA_TRY(launch_plan_build(L.g, L.q, L.k, L.qp, L.kvp, L.plan_ws, st), "plan build");
    PassArgs a3 = L.a2;
    a3.kv_perm = L.kvp;
    a3.kv_top = 0;
    a3.lvl_base = 0;
    a3.acc_out = a3.ell_out = a3.m_out = nullptr;
    S2O_CUDA_TRY(launch_trace_init(L.a, L.p1, st), "trace init");
    if (!L.fused) {  // pass-1 state was overwritten by saved levels: redo pass-1
        PassArgs a1 = L.a;
        a1.mode = kDiag | kStateOut;
        a1.q_reorder = 0;
        a1.acc_out = L.acc; a1.ell_out = L.ell; a1.m_out = L.m;
        if (s2o_status e = run_pass(a1, L.path, L.pass_ws, L.pass_bytes, st)) return e;
    }
    return run_pass(a3, L.path, L.pass_ws, L.pass_bytes, st);
}

// Capture `fn` (enqueues work on a stream) into the body graph of a conditional node.
template <typename F>
s2o_status capture_into(cudaGraph_t body, cudaStream_t side, F&& fn) {
    S2O_CUDA_TRY(cudaStreamBeginCaptureToGraph(side, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed),
                 "begin capture");
    s2o_status e = fn(side);
    cudaGraph_t out = nullptr;
    cudaError_t ce = cudaStreamEndCapture(side, &out);
    if (e) return e;
    if (ce != cudaSuccess) return cuda_fail(ce, "end capture");
    return S2O_OK;
}

// Add WHILE(level loop) -> IF(fallback) to `graph` after `deps`; *last = the IF node.
s2o_status add_level_nodes(const LevelLoop& L, cudaGraph_t graph, const cudaGraphNode_t* deps, size_t ndeps,
                           cudaStream_t side, cudaGraphNode_t* last) {
    cudaGraphConditionalHandle hl, hf;
    S2O_CUDA_TRY(cudaGraphConditionalHandleCreate(&hl, graph, 1, cudaGraphCondAssignDefault), "cond handle");
    S2O_CUDA_TRY(cudaGraphConditionalHandleCreate(&hf, graph, 0, cudaGraphCondAssignDefault), "cond handle");
    cudaGraphNodeParams wp = {};
    wp.type = cudaGraphNodeTypeConditional;
    wp.conditional.handle = hl;
    wp.conditional.type = cudaGraphCondTypeWhile;
    wp.conditional.size = 1;
    cudaGraphNode_t wnode;
    S2O_CUDA_TRY(cudaGraphAddNode(&wnode, graph, deps, ndeps, &wp), "while node");
    if (s2o_status e = capture_into(wp.conditional.phGraph_out[0], side,
                                    [&](cudaStream_t t) { return level_body(L, t, hl, hf); }))
        return e;
    cudaGraphNodeParams fp = {};
    fp.type = cudaGraphNodeTypeConditional;
    fp.conditional.handle = hf;
    fp.conditional.type = cudaGraphCondTypeIf;
    fp.conditional.size = 1;
    S2O_CUDA_TRY(cudaGraphAddNode(last, graph, &wnode, 1, &fp), "if node");
    return capture_into(fp.conditional.phGraph_out[0], side, [&](cudaStream_t t) { return fallback_body(L, t); });
}

struct LoopCache {
    std::mutex mu;
    std::vector<std::pair<std::string, cudaGraphExec_t>> execs;  // (key bytes incl. device, exec)
    std::vector<std::pair<int, cudaStream_t>> side;               // per device capture stream
} g_loops;

s2o_status enqueue_level_loop(const LevelLoop& L, cudaStream_t s) {
    int dev = 0;
    S2O_CUDA_TRY(cudaGetDevice(&dev), "device");
    std::lock_guard<std::mutex> lock(g_loops.mu);
    cudaStream_t side = nullptr;
    for (auto& e : g_loops.side)
        if (e.first == dev) side = e.second;
    if (!side) {
        S2O_CUDA_TRY(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking), "stream");
        g_loops.side.emplace_back(dev, side);
    }
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    S2O_CUDA_TRY(cudaStreamIsCapturing(s, &cs), "capture status");
    if (cs == cudaStreamCaptureStatusActive) {  // into the caller's graph
        cudaGraph_t graph;
        const cudaGraphNode_t* deps = nullptr;
        size_t ndeps = 0;
        S2O_CUDA_TRY(cudaStreamGetCaptureInfo(s, &cs, nullptr, &graph, &deps, &ndeps), "capture info");
        cudaGraphNode_t last;
        if (s2o_status e = add_level_nodes(L, graph, deps, ndeps, side, &last)) return e;
        S2O_CUDA_TRY(cudaStreamUpdateCaptureDependencies(s, &last, 1, cudaStreamSetCaptureDependencies),
                     "capture dependencies");
        return S2O_OK;
    }
    std::string key(reinterpret_cast<const char*>(&L), sizeof L);
    key.append(reinterpret_cast<const char*>(&dev), sizeof dev);
    cudaGraphExec_t exec = nullptr;
    for (auto& e : g_loops.execs)
        if (e.first == key) exec = e.second;
    if (!exec) {
        cudaGraph_t graph;
        S2O_CUDA_TRY(cudaGraphCreate(&graph, 0), "graph");
        cudaGraphNode_t last;
        s2o_status e = add_level_nodes(L, graph, nullptr, 0, side, &last);
        if (!e) {
            cudaError_t ce = cudaGraphInstantiate(&exec, graph, 0);
            if (ce != cudaSuccess) e = cuda_fail(ce, "graph instantiate");
        }
        cudaGraphDestroy(graph);
        if (e) return e;
        if (g_loops.execs.size() >= 16) {  // bounded cache: drop the oldest
            cudaGraphExecDestroy(g_loops.execs.front().second);
            g_loops.execs.erase(g_loops.execs.begin());
        }
        g_loops.execs.emplace_back(std::move(key), exec);
    }
    S2O_CUDA_TRY(cudaGraphLaunch(exec, s), "graph launch");
    return S2O_OK;
}

}  // namespace
}  // namespace s2o

using namespace s2o;

extern "C" {

int s2o_abi_version(void) { return S2O_ABI_VERSION; }

const char* s2o_last_error(void) { return g_err.c_str(); }

const char* s2o_status_string(int status) {
    switch (status) {
        case S2O_OK: return "ok";
        case S2O_ERR_SEG_LEN: return "segment length must satisfy 1 <= S <= L";
        case S2O_ERR_TAU: return "tau must be >= 0";
        case S2O_ERR_TILES: return "tile sizes must be >= 1";
        case S2O_ERR_LOCAL_WINDOW: return "local window must satisfy W <= S";
        case S2O_ERR_FUSED_REORDER: return "fused variant requires q_reorder = false";
        case S2O_ERR_FUSED_FLAGS: return "fused variant requires fused = true, q_reorder = false";
        case S2O_ERR_PLAN_MISMATCH: return "plan/config mismatch: segment layout differs";
        case S2O_ERR_BUFS_MISMATCH: return "pass buffers do not match tensor dims";
        case S2O_ERR_QKV_DIMS: return "Q/K/V dims must match";
        case S2O_ERR_UNINIT_STATE: return "uninitialized state";
        case S2O_ERR_EMPTY_SCORES: return "empty score vector";
        case S2O_ERR_UNCOVERED_ROW: return "uncovered query row";
        case S2O_ERR_NORMALIZER_ALIGN: return "normalizer vectors must align";
        case S2O_ERR_INVALID_ARG: return "invalid argument";
        case S2O_ERR_UNSUPPORTED: return "unsupported shape";
        case S2O_ERR_WORKSPACE: return "workspace too small";
        case S2O_ERR_CUDA: return "CUDA error";
        case S2O_ERR_NO_DEVICE: return "no usable sm_100 device";
        default: return "unknown status";
    }
}

void s2o_problem_init(s2o_problem* p, int64_t z, int64_t hq, int64_t hkv, int64_t l, int64_t d,
                      int32_t in_dtype, int32_t out_dtype) {
    std::memset(p, 0, sizeof *p);
    p->z = z; p->hq = hq; p->hkv = hkv; p->l = l; p->d = d;
    p->in_dtype = in_dtype;
    p->out_dtype = out_dtype;
    const int64_t qs[3] = {hq * l * d, l * d, d};
    const int64_t ks[3] = {hkv * l * d, l * d, d};
    for (int i = 0; i < 3; ++i) {
        p->q_stride[i] = qs[i]; p->o_stride[i] = qs[i];
        p->k_stride[i] = ks[i]; p->v_stride[i] = ks[i];
    }
}

void s2o_kernel_config_init(s2o_kernel_config* c) {
    std::memset(c, 0, sizeof *c);
    c->seg_len = 128;
    c->tau = 0.005;
    c->b_m = 128;
    c->b_n = 128;
    c->q_reorder = 1;
    c->fused = 0;
    c->local_window = -1;
    c->path = S2O_PATH_AUTO;
    c->score_mode = S2O_SCORE_EXACT;
}

s2o_status s2o_kernel_config_validate(const s2o_kernel_config* c, int64_t l) {
    s2o_status st = validate_cfg(c, l);
    if (st == S2O_OK) g_err.clear();
    return st;
}

s2o_status s2o_early_stop_check(const double* prev, const double* nw, int64_t n, double tau,
                                int32_t* stop) {
    if (!prev || !nw || !stop || n <= 0)
        return fail(S2O_ERR_NORMALIZER_ALIGN, "normalizer vectors must align");
    double max_gain = -INFINITY;
    for (int64_t r = 0; r < n; ++r) {
        if (prev[r] <= 0.0) return fail(S2O_ERR_UNINIT_STATE, "uninitialized state");
        const double g = (nw[r] - prev[r]) / prev[r];
        max_gain = (max_gain < g) ? g : max_gain;
    }
    *stop = max_gain < tau;
    return S2O_OK;
}

s2o_status s2o_select_path(const s2o_problem* p, const s2o_kernel_config* c, int32_t* path) {
    Geo g;
    s2o_status st = make_geo(p, c ? c->seg_len : 0, &g);
    if (st) return st;
    if ((st = validate_cfg(c, p->l))) return st;
    PassArgs a = base_args(g, c);
    *path = path_is_tc(a, c->path) ? S2O_PATH_TCGEN05 : S2O_PATH_GENERIC;
    return S2O_OK;
}

s2o_status s2o_plan_workspace_size(const s2o_problem* p, int64_t seg_len, size_t* bytes) {
    Geo g;
    s2o_status st = make_geo(p, seg_len, &g);
    if (st) return st;
    *bytes = plan_workspace_bytes(g);
    return S2O_OK;
}

s2o_status s2o_segment_representatives(const s2o_problem* p, const void* q, const void* k,
                                       int64_t seg_len, float* q_mean, float* k_mean,
                                       void* stream) {
    Geo g;
    s2o_status st = make_geo(p, seg_len, &g);
    if (st) return st;
    if (!q || !k) return fail(S2O_ERR_INVALID_ARG, "null tensor");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (q_mean) S2O_CUDA_TRY(launch_segment_means(g, q, 0, g.N, q_mean, s), "segment means");
    if (k_mean) S2O_CUDA_TRY(launch_segment_means(g, k, 1, g.N, k_mean, s), "segment means");
    return S2O_OK;
}

s2o_status s2o_rank_queries(const s2o_problem* p, const void* q, const float* guide, int64_t seg_len,
                            int32_t* q_perm, void* workspace, size_t workspace_bytes, void* stream) {
    Geo g;
    s2o_status st = make_geo(p, seg_len, &g);
    if (st) return st;
    if (!q || !guide || !q_perm) return fail(S2O_ERR_INVALID_ARG, "null pointer");
    if (!workspace || workspace_bytes < plan_workspace_bytes(g)) return fail(S2O_ERR_WORKSPACE, "workspace too small");
    S2O_CUDA_TRY(launch_rank_queries(g, q, guide, q_perm, workspace, reinterpret_cast<cudaStream_t>(stream)),
                 "rank queries");
    g_err.clear();
    return S2O_OK;
}

s2o_status s2o_rank_prefix_keys(const s2o_problem* p, const void* k, const float* q_mean, int64_t seg_len,
                                int32_t* kv_perm, void* workspace, size_t workspace_bytes, void* stream) {
    Geo g;
    s2o_status st = make_geo(p, seg_len, &g);
    if (st) return st;
    if (!k || !q_mean || (g.N > 1 && !kv_perm)) return fail(S2O_ERR_INVALID_ARG, "null pointer");
    if (!workspace || workspace_bytes < plan_workspace_bytes(g)) return fail(S2O_ERR_WORKSPACE, "workspace too small");
    S2O_CUDA_TRY(launch_rank_prefix_keys(g, k, q_mean, kv_perm, workspace, reinterpret_cast<cudaStream_t>(stream)),
                 "rank prefix keys");
    g_err.clear();
    return S2O_OK;
}

s2o_status s2o_plan_build(const s2o_problem* p, const void* q, const void* k,
                          const s2o_kernel_config* cfg, int32_t* q_perm, int32_t* kv_perm,
                          int64_t* cost2, void* workspace, size_t workspace_bytes, void* stream) {
    if (!cfg) return fail(S2O_ERR_INVALID_ARG, "null config");
    Geo g;
    s2o_status st = make_geo(p, cfg->seg_len, &g);
    if (st) return st;
    if (!q || !k || !q_perm || (g.N > 1 && !kv_perm)) return fail(S2O_ERR_INVALID_ARG, "null pointer");
    if (!workspace || workspace_bytes < plan_workspace_bytes(g))
        return fail(S2O_ERR_WORKSPACE, "workspace too small");
    if (cfg->score_mode != S2O_SCORE_EXACT)
        return fail(S2O_ERR_UNSUPPORTED, "only exact (fp64 sequential) scoring is implemented");
    void* ws = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255));
    S2O_CUDA_TRY(launch_plan_build(g, q, k, q_perm, kv_perm, ws, reinterpret_cast<cudaStream_t>(stream)),
                 "plan build");
    if (cost2) {
        // RankingCost per slice: L query dots + sum of prefixes (plan.cpp:93-94, 130-131)
        const int64_t dots = g.l + g.S * g.N * (g.N - 1) / 2;
        cost2[0] = dots;
        cost2[1] = dots;
    }
    g_err.clear();
    return S2O_OK;
}

s2o_status s2o_plan_build_truncated(const s2o_problem* p, const void* q, const void* k,
                                    const s2o_kernel_config* cfg, int64_t depth, int32_t* q_perm,
                                    int32_t* kv_top, int32_t* flag, void* workspace,
                                    size_t workspace_bytes, void* stream) {
    if (!cfg) return fail(S2O_ERR_INVALID_ARG, "null config");
    Geo g;
    s2o_status st = make_geo(p, cfg->seg_len, &g);
    if (st) return st;
    if (!q || !k || !q_perm || !flag || (g.N > 1 && !kv_top) || depth < 1)
        return fail(S2O_ERR_INVALID_ARG, "null pointer or depth < 1");
    if (depth > kMaxPlanDepth) return fail(S2O_ERR_UNSUPPORTED, "truncated plan depth must be <= 6144");
    if (!workspace || workspace_bytes < plan_workspace_bytes(g))
        return fail(S2O_ERR_WORKSPACE, "workspace too small");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    void* ws = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255));
    S2O_CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(int32_t), s), "memset");
    S2O_CUDA_TRY(launch_plan_topk(g, q, k, q_perm, kv_top, depth, flag, ws, s), "plan top-k");
    g_err.clear();
    return S2O_OK;
}

s2o_status s2o_pass_workspace_size(const s2o_problem* p, const s2o_kernel_config* cfg,
                                   size_t* bytes) {
    Geo g;
    s2o_status st = make_geo(p, cfg ? cfg->seg_len : 0, &g);
    if (st) return st;
    if ((st = validate_cfg(cfg, p->l))) return st;
    *bytes = pass_ws_bytes(base_args(g, cfg));
    return S2O_OK;
}

// Device status word of the last pass on this workspace: 0 ok, 1 uninitialized state
// (kernel.cpp:228), 2 uncovered query row (kernel.cpp:155). One D2H read; synchronises `stream`.
static s2o_status read_status(const int32_t* dflag, cudaStream_t s) {
    int32_t flag = 0;
    S2O_CUDA_TRY(cudaMemcpyAsync(&flag, dflag, sizeof flag, cudaMemcpyDeviceToHost, s), "d2h status");
    S2O_CUDA_TRY(cudaStreamSynchronize(s), "sync");
    if (flag == 1) return fail(S2O_ERR_UNINIT_STATE, "uninitialized state");
    if (flag == 2) return fail(S2O_ERR_UNCOVERED_ROW, "uncovered query row");
    g_err.clear();
    return S2O_OK;
}

s2o_status s2o_pass_status(const s2o_problem* p, const s2o_kernel_config* cfg, const void* workspace,
                           size_t workspace_bytes, void* stream) {
    Geo g;
    s2o_status st = make_geo(p, cfg ? cfg->seg_len : 0, &g);
    if (st) return st;
    if ((st = validate_cfg(cfg, p->l))) return st;
    const PassArgs a = base_args(g, cfg);
    if (!workspace || workspace_bytes < pass_ws_bytes(a)) return fail(S2O_ERR_WORKSPACE, "workspace too small");
    const char* base = reinterpret_cast<const char*>(workspace);
    return read_status(reinterpret_cast<const int32_t*>(base + align256(generic_scratch_bytes(a))),
                       reinterpret_cast<cudaStream_t>(stream));
}

s2o_status s2o_pass1(const s2o_problem* p, const void* q, const void* k, const void* v,
                     const s2o_kernel_config* cfg, float* acc, float* ell, float* m,
                     void* workspace, size_t workspace_bytes, void* stream) {
    Geo g;
    s2o_status st = make_geo(p, cfg ? cfg->seg_len : 0, &g);
    if (st) return st;
    if ((st = validate_cfg(cfg, p->l))) return st;
    if (!q || !k || !v || !acc || !ell || !m) return fail(S2O_ERR_INVALID_ARG, "null pointer");
    PassArgs a = base_args(g, cfg);
    a.mode = kDiag | kStateOut;
    a.q = q; a.k = k; a.v = v;
    a.acc_out = acc; a.ell_out = ell; a.m_out = m;
    a.q_reorder = 0;
    st = run_pass(a, cfg->path, workspace, workspace_bytes, reinterpret_cast<cudaStream_t>(stream));
    if (st == S2O_OK) g_err.clear();
    return st;
}

s2o_status s2o_pass2(const s2o_problem* p, const void* q, const void* k, const void* v,
                     const s2o_kernel_config* cfg, const float* acc, const float* ell,
                     const float* m, const int32_t* q_perm, const int32_t* kv_perm, void* o,
                     int32_t* processed, int64_t* pass1_pairs, int64_t* pass2_pairs,
                     void* workspace, size_t workspace_bytes, void* stream) {
    Geo g;
    s2o_status st = make_geo(p, cfg ? cfg->seg_len : 0, &g);
    if (st) return st;
    if ((st = validate_cfg(cfg, p->l))) return st;
    if (!q || !k || !v || !acc || !ell || !m || !o || !processed || !pass2_pairs ||
        (cfg->q_reorder && !q_perm) || (g.N > 1 && !kv_perm))
        return fail(S2O_ERR_INVALID_ARG, "null pointer");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    PassArgs a = base_args(g, cfg);
    a.mode = kStateIn | kPrefix | kFinal;
    a.q = q; a.k = k; a.v = v; a.o = o;
    a.acc_in = acc; a.ell_in = ell; a.m_in = m;
    a.q_perm = q_perm; a.kv_perm = kv_perm;
    a.processed = processed; a.pass2_pairs = pass2_pairs;
    S2O_CUDA_TRY(launch_trace_init(a, pass1_pairs, s), "trace init");
    st = run_pass(a, cfg->path, workspace, workspace_bytes, s);
    if (st == S2O_OK) g_err.clear();
    return st;
}

s2o_status s2o_fused(const s2o_problem* p, const void* q, const void* k, const void* v,
                     const s2o_kernel_config* cfg, const int32_t* kv_perm, void* o,
                     int32_t* processed, int64_t* pass1_pairs, int64_t* pass2_pairs,
                     void* workspace, size_t workspace_bytes, void* stream) {
    if (cfg && (!cfg->fused || cfg->q_reorder))
        return fail(S2O_ERR_FUSED_FLAGS, "fused variant requires fused = true, q_reorder = false");
    Geo g;
    s2o_status st = make_geo(p, cfg ? cfg->seg_len : 0, &g);
    if (st) return st;
    if ((st = validate_cfg(cfg, p->l))) return st;
    if (!q || !k || !v || !o || !processed || !pass2_pairs || (g.N > 1 && !kv_perm))
        return fail(S2O_ERR_INVALID_ARG, "null pointer");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    PassArgs a = base_args(g, cfg);
    a.mode = kDiag | kPrefix | kFinal;
    a.q = q; a.k = k; a.v = v; a.o = o;
    a.kv_perm = kv_perm;
    a.processed = processed; a.pass2_pairs = pass2_pairs;
    a.q_reorder = 0;
    S2O_CUDA_TRY(launch_trace_init(a, pass1_pairs, s), "trace init");
    st = run_pass(a, cfg->path, workspace, workspace_bytes, s);
    if (st == S2O_OK) g_err.clear();
    return st;
}

// Workspace of the whole operator:
//   [plan ws][pass ws][q_perm][kv_perm][acc][ell][m][processed][pass1][pass2]
struct OpLayout {
    size_t plan, pass, qperm, kvperm, kvtop, ovf, acc, ell, m, proc, p1, p2, total;
    int64_t topt;
};

// Depth of the truncated kv plan (0 = full permutation).
static int64_t plan_topt(const Geo& g, const s2o_kernel_config* c) {
    if (c->plan_depth < 0) return 0;
    int64_t t = c->plan_depth == 0 ? 6144 : c->plan_depth;
    t = ((t + c->b_n - 1) / c->b_n) * c->b_n;
    if (t > kMaxPlanDepth) return 0;  // beyond the selection capacity: build the full plan
    if (t >= (g.N - 1) * g.S) return 0;  // no segment would be truncated
    return t;
}

static OpLayout op_layout(const Geo& g, const PassArgs& a, int fused, const s2o_kernel_config* c) {
    OpLayout L;
    size_t off = 0;
    auto take = [&](size_t b) { size_t o = off; off += align256(b); return o; };
    const int64_t zh = g.z * g.hq;
    L.topt = plan_topt(g, c);
    L.plan = take(plan_workspace_bytes(g));
    L.pass = take(pass_ws_bytes(a));
    L.qperm = take(sizeof(int32_t) * zh * g.N * g.S);
    L.kvperm = take(sizeof(int32_t) * std::max<int64_t>(1, zh * g.kv_per_head()));
    L.kvtop = take(2 * sizeof(int32_t) * std::max<int64_t>(1, zh * g.N * L.topt));  // level lists A, B
    // [0] overflow count, [1] selection flag, then tiles A/B, bases A/B, segment list
    // level control (kCtlWords int32: overflow count, selection flag, segment count, tile count,
    // level base (int64)), tiles A/B, bases A/B, segment list, then one mark byte per segment
    L.ovf = take(sizeof(int32_t) * (kCtlWords + 5 * zh * a.tiles_per_head) + zh * g.N);
    // pass state: pass-1 -> pass-2, and (also fused) the saved state of tiles that resume at the
    // next plan level of a truncated plan
    const bool state = !fused || L.topt > 0;
    L.acc = take(state ? sizeof(float) * zh * g.l * g.d : 0);
    L.ell = take(state ? sizeof(float) * zh * g.l : 0);
    L.m = take(state ? sizeof(float) * zh * g.l : 0);
    L.proc = take(sizeof(int32_t) * zh * g.N * a.T);
    L.p1 = take(sizeof(int64_t) * zh);
    L.p2 = take(sizeof(int64_t) * zh);
    L.total = off + 256;
    return L;
}

s2o_status s2o_attention_workspace_size(const s2o_problem* p, const s2o_kernel_config* cfg,
                                        size_t* bytes) {
    Geo g;
    s2o_status st = make_geo(p, cfg ? cfg->seg_len : 0, &g);
    if (st) return st;
    if ((st = validate_cfg(cfg, p->l))) return st;
    *bytes = op_layout(g, base_args(g, cfg), cfg->fused, cfg).total;
    return S2O_OK;
}

s2o_status s2o_attention_status(const s2o_problem* p, const s2o_kernel_config* cfg, const void* workspace,
                                size_t workspace_bytes, void* stream) {
    Geo g;
    s2o_status st = make_geo(p, cfg ? cfg->seg_len : 0, &g);
    if (st) return st;
    if ((st = validate_cfg(cfg, p->l))) return st;
    const PassArgs a = base_args(g, cfg);
    const OpLayout L = op_layout(g, a, cfg->fused, cfg);
    if (!workspace || workspace_bytes < L.total) return fail(S2O_ERR_WORKSPACE, "workspace too small");
    const char* base = reinterpret_cast<const char*>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255));
    return read_status(reinterpret_cast<const int32_t*>(base + L.pass + align256(generic_scratch_bytes(a))),
                       reinterpret_cast<cudaStream_t>(stream));
}

s2o_status s2o_attention_fwd(const s2o_problem* p, const void* q, const void* k, const void* v,
                             const s2o_kernel_config* cfg, void* o, int32_t* q_perm,
                             int32_t* kv_perm, int32_t* processed, int64_t* pass1_pairs,
                             int64_t* pass2_pairs, void* workspace, size_t workspace_bytes,
                             void* stream) {
    Geo g;
    s2o_status st = make_geo(p, cfg ? cfg->seg_len : 0, &g);
    if (st) return st;
    if ((st = validate_cfg(cfg, p->l))) return st;
    if (!q || !k || !v || !o) return fail(S2O_ERR_INVALID_ARG, "null pointer");
    PassArgs a = base_args(g, cfg);
    const OpLayout L = op_layout(g, a, cfg->fused, cfg);
    if (!workspace || workspace_bytes < L.total) return fail(S2O_ERR_WORKSPACE, "workspace too small");
    char* base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255));
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int32_t* qp = q_perm ? q_perm : reinterpret_cast<int32_t*>(base + L.qperm);
    int32_t* kvp = kv_perm ? kv_perm : reinterpret_cast<int32_t*>(base + L.kvperm);
    int32_t* proc = processed ? processed : reinterpret_cast<int32_t*>(base + L.proc);
    int64_t* p1 = pass1_pairs ? pass1_pairs : reinterpret_cast<int64_t*>(base + L.p1);
    int64_t* p2 = pass2_pairs ? pass2_pairs : reinterpret_cast<int64_t*>(base + L.p2);
    // Truncated plan unless the caller asked for the full kv_perm (or no segment is long enough)
    const int64_t topt = kv_perm ? 0 : L.topt;
    int32_t* ovf = reinterpret_cast<int32_t*>(base + L.ovf);  // level control words, see kCtlWords
    const int64_t ntiles = g.z * g.hq * a.tiles_per_head;
    if (topt > 0) {
        S2O_CUDA_TRY(cudaMemsetAsync(ovf, 0, kCtlWords * sizeof(int32_t), s), "memset");
        S2O_CUDA_TRY(cudaMemsetAsync(reinterpret_cast<char*>(ovf + kCtlWords + 5 * ntiles), 0, g.z * g.hq * g.N, s),
                     "memset");
        S2O_CUDA_TRY(launch_plan_topk(g, q, k, qp, reinterpret_cast<int32_t*>(base + L.kvtop), topt, ovf + 1,
                                      base + L.plan, s), "plan top-k");
    } else {
        S2O_CUDA_TRY(launch_plan_build(g, q, k, qp, kvp, base + L.plan, s), "plan build");
    }
    int32_t* lists[2] = {reinterpret_cast<int32_t*>(base + L.kvtop),
                         reinterpret_cast<int32_t*>(base + L.kvtop) + std::max<int64_t>(1, g.z * g.hq * g.N * L.topt)};
    int32_t* tiles[2] = {ovf + kCtlWords, ovf + kCtlWords + ntiles};
    int32_t* bases[2] = {ovf + kCtlWords + 2 * ntiles, ovf + kCtlWords + 3 * ntiles};
    a.q = q; a.k = k; a.v = v; a.o = o;
    a.kv_perm = topt > 0 ? lists[0] : kvp;
    a.kv_top = topt;
    a.ovf_count = ovf;
    a.ovf_tiles = tiles[0];
    a.ovf_base = bases[0];
    a.processed = proc;
    a.pass2_pairs = p2;
    S2O_CUDA_TRY(launch_trace_init(a, p1, s), "trace init");
    float* acc = reinterpret_cast<float*>(base + L.acc);
    float* ell = reinterpret_cast<float*>(base + L.ell);
    float* m = reinterpret_cast<float*>(base + L.m);
    PassArgs a2 = a;
    if (cfg->fused) {
        a2.mode = kDiag | kPrefix | kFinal;
        a2.q_reorder = 0;
        if (topt > 0) { a2.acc_out = acc; a2.ell_out = ell; a2.m_out = m; }  // resume state, as below
    } else {
        PassArgs a1 = a;
        a1.mode = kDiag | kStateOut;
        a1.q_reorder = 0;
        a1.acc_out = acc; a1.ell_out = ell; a1.m_out = m;
        if ((st = run_pass(a1, cfg->path, base + L.pass, pass_ws_bytes(a), s))) return st;
        a2.mode = kStateIn | kPrefix | kFinal;
        a2.q_perm = qp;
        a2.acc_in = acc; a2.ell_in = ell; a2.m_in = m;
        // a tile that exhausts a truncated list saves its state in place and resumes at the
        // next plan level (entries [T, 2T), [2T, 3T), ... of the same order)
        if (topt > 0) { a2.acc_out = acc; a2.ell_out = ell; a2.m_out = m; }
    }
    if ((st = run_pass(a2, cfg->path, base + L.pass, pass_ws_bytes(a), s))) return st;
    if (topt > 0) {
        LevelLoop lp;
        std::memset(&lp, 0, sizeof lp);  // the struct's bytes key the graph cache
        lp.g = g;
        lp.a = a;
        lp.a2 = a2;
        lp.path = cfg->path;
        lp.fused = cfg->fused;
        lp.topt = topt;
        lp.q = q; lp.k = k;
        lp.qp = qp; lp.kvp = kvp; lp.p1 = p1;
        lp.ctl = ovf;
        lp.marks = reinterpret_cast<uint8_t*>(ovf + kCtlWords + 5 * ntiles);
        lp.seglist = ovf + kCtlWords + 4 * ntiles;
        for (int i = 0; i < 2; ++i) { lp.lists[i] = lists[i]; lp.tiles[i] = tiles[i]; lp.bases[i] = bases[i]; }
        lp.acc = acc; lp.ell = ell; lp.m = m;
        lp.plan_ws = base + L.plan;
        lp.pass_ws = base + L.pass;
        lp.pass_bytes = pass_ws_bytes(a);
        if ((st = enqueue_level_loop(lp, s))) return st;
    }
    g_err.clear();
    return S2O_OK;
}

s2o_status s2o_block_topk_workspace_size(const s2o_problem* p, int64_t block_rows, int64_t block_cols,
                                         int64_t topk, size_t* bytes) {
    Geo g;
    PassArgs a;
    BtLayout L;
    if (!bytes) return fail(S2O_ERR_INVALID_ARG, "null pointer");
    s2o_status st = bt_setup(p, block_rows, block_cols, topk, &g, &a, &L);
    if (st) return st;
    *bytes = L.total;
    return S2O_OK;
}

s2o_status s2o_block_topk_fwd(const s2o_problem* p, const void* q, const void* k, const void* v,
                              int64_t block_rows, int64_t block_cols, int64_t topk, int32_t path, void* o,
                              int64_t* pair_count, void* workspace, size_t workspace_bytes, void* stream) {
    Geo g;
    PassArgs a;
    BtLayout L;
    s2o_status st = bt_setup(p, block_rows, block_cols, topk, &g, &a, &L);
    if (st) return st;
    if (!q || !k || !v || !o || !pair_count) return fail(S2O_ERR_INVALID_ARG, "null pointer");
    if (!workspace || workspace_bytes < L.total) return fail(S2O_ERR_WORKSPACE, "workspace too small");
    char* base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255));
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int32_t* kvtop = reinterpret_cast<int32_t*>(base + L.kvtop);
    S2O_CUDA_TRY(launch_block_topk_select(g, q, k, block_rows, block_cols, topk, reinterpret_cast<double*>(base + L.rmax),
                                          reinterpret_cast<double*>(base + L.rden),
                                          reinterpret_cast<double*>(base + L.mass), kvtop, s),
                 "block top-k selection");
    a.q = q; a.k = k; a.v = v; a.o = o;
    a.processed = reinterpret_cast<int32_t*>(base + L.proc);
    a.pass2_pairs = reinterpret_cast<int64_t*>(base + L.p2);
    a.kv_perm = kvtop;
    a.kv_top = std::max<int64_t>(1, topk * block_cols);
    a.no_overflow = 1;
    // pass1_pairs = the self blocks' exact triangles (self_pair_count, baseline.cpp:95-104)
    S2O_CUDA_TRY(launch_trace_init(a, pair_count, s), "trace init");
    PassArgs a1 = a;
    float* acc = reinterpret_cast<float*>(base + L.acc);
    float* ell = reinterpret_cast<float*>(base + L.ell);
    float* m = reinterpret_cast<float*>(base + L.m);
    a1.mode = topk > 0 ? (kDiag | kStateOut) : (kDiag | kFinal);
    a1.acc_out = acc; a1.ell_out = ell; a1.m_out = m;
    if ((st = run_pass(a1, path, base + L.pass, pass_ws_bytes(a), s))) return st;
    if (topk > 0) {
        PassArgs a2 = a;
        a2.mode = kStateIn | kPrefix | kFinal;
        a2.acc_in = acc; a2.ell_in = ell; a2.m_in = m;
        if ((st = run_pass(a2, path, base + L.pass, pass_ws_bytes(a), s))) return st;
        // pair_count = self triangles + rows x committed tokens of the kept prefix blocks
        S2O_CUDA_TRY(launch_add_pairs(pair_count, a.pass2_pairs, g.z * g.hq, s), "pair sum");
    }
    g_err.clear();
    return S2O_OK;
}

s2o_status s2o_dense_causal_fwd(const s2o_problem* p, const void* q, const void* k,
                                const void* v, int32_t path, void* o, void* workspace,
                                size_t workspace_bytes, void* stream) {
    Geo g;
    s2o_status st = make_geo(p, p ? p->l : 0, &g);  // one segment: S = L
    if (st) return st;
    if (!q || !k || !v || !o) return fail(S2O_ERR_INVALID_ARG, "null pointer");
    s2o_kernel_config c;
    s2o_kernel_config_init(&c);
    c.seg_len = p->l;
    c.q_reorder = 0;
    c.path = path;
    if (path == S2O_PATH_GENERIC) { c.b_m = 64; c.b_n = 64; }
    PassArgs a = base_args(g, &c);
    a.mode = kDiag | kFinal;
    a.q = q; a.k = k; a.v = v; a.o = o;
    st = run_pass(a, path, workspace, workspace_bytes, reinterpret_cast<cudaStream_t>(stream));
    if (st == S2O_OK) g_err.clear();
    return st;
}

// Host-buffer operator, pipelined over (batch, kv head) chunks -- heads are independent: chunk
// c+1 moves host->device while chunk c computes and chunk c-1 moves device->host, on three
// streams with double-buffered device chunk sets. Each chunk is the sub-problem
// {Z=1, Hq=group (or 1 for the split last group), Hkv=1} through s2o_attention_fwd, so results
// equal the one-shot call.
static s2o_status attention_host_pipelined(const s2o_problem* p, const Geo& g, const void* q, const void* k,
                                           const void* v, const s2o_kernel_config* cfg, void* o,
                                           int32_t* q_perm, int32_t* kv_perm, int32_t* processed,
                                           int64_t* pass1_pairs, int64_t* pass2_pairs) {
    const int64_t grp = p->hq / p->hkv;
    const int64_t nchunks = p->z * p->hkv;
    s2o_problem sp;
    s2o_problem_init(&sp, 1, grp, 1, p->l, p->d, p->in_dtype, p->out_dtype);
    Geo sg;
    s2o_status st = make_geo(&sp, cfg->seg_len, &sg);
    if (st) return st;
    PassArgs sa = base_args(sg, cfg);
    const OpLayout SL = op_layout(sg, sa, cfg->fused, cfg);
    const size_t esz_in = p->in_dtype == S2O_BF16 ? 2 : 4;
    const size_t esz_out = p->out_dtype == S2O_BF16 ? 2 : 4;
    const size_t row = (size_t)p->l * p->d;
    const size_t qb = esz_in * grp * row, kb = esz_in * row, ob = esz_out * grp * row;
    const size_t qpb = sizeof(int32_t) * grp * sg.N * sg.S;
    const size_t kvpb = kv_perm && sg.N > 1 ? sizeof(int32_t) * grp * sg.kv_per_head() : 0;
    const size_t prb = sizeof(int32_t) * grp * sg.N * sa.T;
    const size_t pairb = sizeof(int64_t) * grp;
    // chunk set: q k v o q_perm kv_perm processed pass1 pass2
    const size_t off_q = 0, off_k = align256(qb), off_v = off_k + align256(kb), off_o = off_v + align256(kb);
    const size_t off_qp = off_o + align256(ob), off_kvp = off_qp + align256(qpb);
    const size_t off_pr = off_kvp + align256(kvpb), off_p1 = off_pr + align256(prb), off_p2 = off_p1 + align256(pairb);
    const size_t set_bytes = off_p2 + align256(pairb);
    const size_t kvset = 2 * align256(kb);                         // K + V of one GQA group
    const size_t need = 2 * set_bytes + SL.total + 256 + 2 * kvset;  // + K/V of two groups in flight
    std::lock_guard<std::mutex> lock(g_host.mu);
    if (!g_host.stream) S2O_CUDA_TRY(cudaStreamCreateWithFlags(&g_host.stream, cudaStreamNonBlocking), "stream");
    if (!g_host.s_in) {
        S2O_CUDA_TRY(cudaStreamCreateWithFlags(&g_host.s_in, cudaStreamNonBlocking), "stream");
        S2O_CUDA_TRY(cudaStreamCreateWithFlags(&g_host.s_out, cudaStreamNonBlocking), "stream");
        for (int b = 0; b < 2; ++b) {
            S2O_CUDA_TRY(cudaEventCreateWithFlags(&g_host.ev_h2d[b], cudaEventDisableTiming), "event");
            S2O_CUDA_TRY(cudaEventCreateWithFlags(&g_host.ev_comp[b], cudaEventDisableTiming), "event");
            S2O_CUDA_TRY(cudaEventCreateWithFlags(&g_host.ev_d2h[b], cudaEventDisableTiming), "event");
            S2O_CUDA_TRY(cudaEventCreateWithFlags(&g_host.ev_kv[b], cudaEventDisableTiming), "event");
        }
    }
    if (g_host.bytes < need) {
        if (g_host.dev) cudaFree(g_host.dev);
        g_host.dev = nullptr;
        g_host.bytes = 0;
        S2O_CUDA_TRY(cudaMalloc(&g_host.dev, need), "arena alloc");
        g_host.bytes = need;
    }
    const int64_t max_chunks = nchunks * grp;  // at most one part per q head
    if (g_host.nflags < max_chunks) {
        if (g_host.flags) cudaFreeHost(g_host.flags);
        g_host.flags = nullptr;
        g_host.nflags = 0;
        S2O_CUDA_TRY(cudaMallocHost(&g_host.flags, sizeof(int32_t) * max_chunks), "pinned flags");
        g_host.nflags = max_chunks;
    }
    char* set[2] = {reinterpret_cast<char*>(g_host.dev), reinterpret_cast<char*>(g_host.dev) + set_bytes};
    char* ws = reinterpret_cast<char*>(g_host.dev) + 2 * set_bytes;
    char* kvbuf[2] = {ws + SL.total + 256, ws + SL.total + 256 + kvset};  // K/V of group zg in kvbuf[zg & 1]
    cudaStream_t sc = g_host.stream, si = g_host.s_in, so = g_host.s_out;
    // Chunks: a GQA group goes in parts of q heads with its K/V copied once, with the first part,
    // into a per-group-parity buffer. Whole groups, except the first, whose first part is one head
    // (the pipeline's fill: that H2D runs alone), and the last, which goes in halves (the drain: the
    // last compute + D2H run alone). Measured at C3 (e2e ms): this 35.3; whole groups + halved last
    // 36.0; S2O_HOST_PART_HEADS = parts for every group: 4 -> 36.8, 2 -> 37.3, 1 -> 44.6 (a 1-head
    // part computes slower than its copy; more parts add per-call overhead); a 1-head last part 35.5.
    static const int64_t split_env = [] {
        const char* e = std::getenv("S2O_HOST_PART_HEADS");
        return e ? std::atoll(e) : 0ll;
    }();
    struct Chunk { int64_t zg, q0, nq; bool first, last; };
    std::vector<Chunk> chunks;
    for (int64_t zg = 0; zg < nchunks; ++zg) {
        if (split_env <= 0 && zg == 0 && nchunks > 1 && grp >= 4) {
            // the fill: the first part's H2D runs alone, so it is one q head (+ the group's K/V)
            chunks.push_back({zg, 0, 1, true, false});
            chunks.push_back({zg, 1, grp - 1, false, true});
            continue;
        }
        const int64_t want = split_env > 0 ? split_env : (zg + 1 == nchunks ? grp / 2 : grp);
        const int64_t step = std::min<int64_t>(grp, std::max<int64_t>(1, want));
        for (int64_t h = 0; h < grp; h += step)
            chunks.push_back({zg, h, std::min(step, grp - h), h == 0, h + step >= grp});
    }
    const int64_t ncs = (int64_t)chunks.size();
    auto h0_of = [&](const Chunk& ch) { return (ch.zg / p->hkv) * p->hq + (ch.zg % p->hkv) * grp + ch.q0; };
    auto enqueue_in = [&](int64_t c) -> s2o_status {
        const Chunk& ch = chunks[c];
        const int b = (int)(c & 1);
        if (c >= 2) S2O_CUDA_TRY(cudaStreamWaitEvent(si, g_host.ev_comp[b], 0), "wait");
        const char* hq = reinterpret_cast<const char*>(q) + esz_in * row * h0_of(ch);
        const char* hk = reinterpret_cast<const char*>(k) + esz_in * row * ch.zg;
        const char* hv = reinterpret_cast<const char*>(v) + esz_in * row * ch.zg;
        S2O_CUDA_TRY(cudaMemcpyAsync(set[b] + off_q, hq, esz_in * row * ch.nq, cudaMemcpyHostToDevice, si), "h2d q");
        if (ch.first) {  // the group's K/V (its buffer was last read by group zg - 2's last part)
            char* kvd = kvbuf[ch.zg & 1];
            if (ch.zg >= 2) S2O_CUDA_TRY(cudaStreamWaitEvent(si, g_host.ev_kv[ch.zg & 1], 0), "wait");
            S2O_CUDA_TRY(cudaMemcpyAsync(kvd, hk, kb, cudaMemcpyHostToDevice, si), "h2d k");
            S2O_CUDA_TRY(cudaMemcpyAsync(kvd + align256(kb), hv, kb, cudaMemcpyHostToDevice, si), "h2d v");
        }
        S2O_CUDA_TRY(cudaEventRecord(g_host.ev_h2d[b], si), "record");
        return S2O_OK;
    };
    auto drain = [&]() {
        cudaStreamSynchronize(si);
        cudaStreamSynchronize(sc);
        cudaStreamSynchronize(so);
    };
    if ((st = enqueue_in(0))) return st;
    for (int64_t c = 0; c < ncs; ++c) {
        const Chunk& ch = chunks[c];
        const int b = (int)(c & 1);
        if (c + 1 < ncs && (st = enqueue_in(c + 1))) { drain(); return st; }
        S2O_CUDA_TRY(cudaStreamWaitEvent(sc, g_host.ev_h2d[b], 0), "wait");
        if (c >= 2) S2O_CUDA_TRY(cudaStreamWaitEvent(sc, g_host.ev_d2h[b], 0), "wait");
        char* cs = set[b];
        s2o_problem cp;
        s2o_problem_init(&cp, 1, ch.nq, 1, p->l, p->d, p->in_dtype, p->out_dtype);
        Geo cg;
        if ((st = make_geo(&cp, cfg->seg_len, &cg))) { drain(); return st; }
        const PassArgs ca = base_args(cg, cfg);
        const OpLayout CL = op_layout(cg, ca, cfg->fused, cfg);
        const char* dk = kvbuf[ch.zg & 1];
        const char* dv = kvbuf[ch.zg & 1] + align256(kb);
        st = s2o_attention_fwd(&cp, cs + off_q, dk, dv, cfg, cs + off_o,
                               reinterpret_cast<int32_t*>(cs + off_qp),
                               kvpb ? reinterpret_cast<int32_t*>(cs + off_kvp) : nullptr,
                               reinterpret_cast<int32_t*>(cs + off_pr), reinterpret_cast<int64_t*>(cs + off_p1),
                               reinterpret_cast<int64_t*>(cs + off_p2), ws, SL.total + 256, sc);
        if (st) { drain(); return st; }
        char* cwb = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
        const int32_t* dflag = reinterpret_cast<const int32_t*>(cwb + CL.pass + align256(generic_scratch_bytes(ca)));
        S2O_CUDA_TRY(cudaMemcpyAsync(&g_host.flags[c], dflag, sizeof(int32_t), cudaMemcpyDeviceToHost, sc), "d2h flag");
        S2O_CUDA_TRY(cudaEventRecord(g_host.ev_comp[b], sc), "record");
        if (ch.last) S2O_CUDA_TRY(cudaEventRecord(g_host.ev_kv[ch.zg & 1], sc), "record");  // K/V buffer free
        S2O_CUDA_TRY(cudaStreamWaitEvent(so, g_host.ev_comp[b], 0), "wait");
        const int64_t h0 = h0_of(ch), nq = ch.nq;
        S2O_CUDA_TRY(cudaMemcpyAsync(reinterpret_cast<char*>(o) + esz_out * row * h0, cs + off_o, esz_out * row * nq,
                                     cudaMemcpyDeviceToHost, so), "d2h o");
        if (q_perm)
            S2O_CUDA_TRY(cudaMemcpyAsync(q_perm + h0 * sg.N * sg.S, cs + off_qp, qpb / grp * nq, cudaMemcpyDeviceToHost,
                                         so), "d2h q_perm");
        if (kvpb)
            S2O_CUDA_TRY(cudaMemcpyAsync(kv_perm + h0 * sg.kv_per_head(), cs + off_kvp, kvpb / grp * nq,
                                         cudaMemcpyDeviceToHost, so), "d2h kv_perm");
        if (processed)
            S2O_CUDA_TRY(cudaMemcpyAsync(processed + h0 * sg.N * sa.T, cs + off_pr, prb / grp * nq,
                                         cudaMemcpyDeviceToHost, so), "d2h trace");
        if (pass1_pairs)
            S2O_CUDA_TRY(cudaMemcpyAsync(pass1_pairs + h0, cs + off_p1, pairb / grp * nq, cudaMemcpyDeviceToHost, so),
                         "d2h pairs");
        if (pass2_pairs)
            S2O_CUDA_TRY(cudaMemcpyAsync(pass2_pairs + h0, cs + off_p2, pairb / grp * nq, cudaMemcpyDeviceToHost, so),
                         "d2h pairs");
        S2O_CUDA_TRY(cudaEventRecord(g_host.ev_d2h[b], so), "record");
    }
    S2O_CUDA_TRY(cudaStreamSynchronize(so), "sync");
    S2O_CUDA_TRY(cudaStreamSynchronize(sc), "sync");
    for (int64_t c = 0; c < ncs; ++c) {
        if (g_host.flags[c] == 1) return fail(S2O_ERR_UNINIT_STATE, "uninitialized state");
        if (g_host.flags[c] == 2) return fail(S2O_ERR_UNCOVERED_ROW, "uncovered query row");
    }
    g_err.clear();
    return S2O_OK;
}

s2o_status s2o_attention_host(const s2o_problem* p, const void* q, const void* k, const void* v,
                              const s2o_kernel_config* cfg, void* o, int32_t* q_perm,
                              int32_t* kv_perm, int32_t* processed, int64_t* pass1_pairs,
                              int64_t* pass2_pairs) {
    Geo g;
    s2o_status st = make_geo(p, cfg ? cfg->seg_len : 0, &g);
    if (st) return st;
    if ((st = validate_cfg(cfg, p->l))) return st;
    if (!q || !k || !v || !o) return fail(S2O_ERR_INVALID_ARG, "null pointer");
    // host buffers are dense [Z,H,L,D]
    if (p->z * p->hkv >= 2)
        return attention_host_pipelined(p, g, q, k, v, cfg, o, q_perm, kv_perm, processed, pass1_pairs,
                                        pass2_pairs);
    s2o_problem dp;
    s2o_problem_init(&dp, p->z, p->hq, p->hkv, p->l, p->d, p->in_dtype, p->out_dtype);
    PassArgs a = base_args(g, cfg);
    const OpLayout L = op_layout(g, a, cfg->fused, cfg);
    const size_t esz_in = p->in_dtype == S2O_BF16 ? 2 : 4;
    const size_t esz_out = p->out_dtype == S2O_BF16 ? 2 : 4;
    const size_t qb = esz_in * p->z * p->hq * p->l * p->d;
    const size_t kb = esz_in * p->z * p->hkv * p->l * p->d;
    const size_t ob = esz_out * p->z * p->hq * p->l * p->d;
    const size_t need = align256(qb) + 2 * align256(kb) + align256(ob) + L.total;
    std::lock_guard<std::mutex> lock(g_host.mu);
    if (!g_host.stream) S2O_CUDA_TRY(cudaStreamCreateWithFlags(&g_host.stream, cudaStreamNonBlocking), "stream");
    if (g_host.bytes < need) {
        if (g_host.dev) cudaFree(g_host.dev);
        g_host.dev = nullptr;
        g_host.bytes = 0;
        S2O_CUDA_TRY(cudaMalloc(&g_host.dev, need), "arena alloc");
        g_host.bytes = need;
    }
    char* d = reinterpret_cast<char*>(g_host.dev);
    char* dq = d;
    char* dk = dq + align256(qb);
    char* dv = dk + align256(kb);
    char* dout = dv + align256(kb);
    char* ws = dout + align256(ob);
    cudaStream_t s = g_host.stream;
    S2O_CUDA_TRY(cudaMemcpyAsync(dq, q, qb, cudaMemcpyHostToDevice, s), "h2d q");
    S2O_CUDA_TRY(cudaMemcpyAsync(dk, k, kb, cudaMemcpyHostToDevice, s), "h2d k");
    S2O_CUDA_TRY(cudaMemcpyAsync(dv, v, kb, cudaMemcpyHostToDevice, s), "h2d v");
    char* wbase = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
    // the full kv_perm is only materialised when the caller asks for it
    int32_t* dkv = (kv_perm && g.N > 1) ? reinterpret_cast<int32_t*>(wbase + L.kvperm) : nullptr;
    st = s2o_attention_fwd(&dp, dq, dk, dv, cfg, dout, nullptr, dkv, nullptr, nullptr, nullptr,
                           ws, L.total, s);
    if (st) return st;
    S2O_CUDA_TRY(cudaMemcpyAsync(o, dout, ob, cudaMemcpyDeviceToHost, s), "d2h o");
    const int64_t zh = g.z * g.hq;
    if (q_perm)
        S2O_CUDA_TRY(cudaMemcpyAsync(q_perm, wbase + L.qperm, sizeof(int32_t) * zh * g.N * g.S,
                                     cudaMemcpyDeviceToHost, s), "d2h q_perm");
    if (kv_perm && g.N > 1)
        S2O_CUDA_TRY(cudaMemcpyAsync(kv_perm, wbase + L.kvperm, sizeof(int32_t) * zh * g.kv_per_head(),
                                     cudaMemcpyDeviceToHost, s), "d2h kv_perm");
    if (processed)
        S2O_CUDA_TRY(cudaMemcpyAsync(processed, wbase + L.proc, sizeof(int32_t) * zh * g.N * a.T,
                                     cudaMemcpyDeviceToHost, s), "d2h trace");
    if (pass1_pairs)
        S2O_CUDA_TRY(cudaMemcpyAsync(pass1_pairs, wbase + L.p1, sizeof(int64_t) * zh,
                                     cudaMemcpyDeviceToHost, s), "d2h pairs");
    if (pass2_pairs)
        S2O_CUDA_TRY(cudaMemcpyAsync(pass2_pairs, wbase + L.p2, sizeof(int64_t) * zh,
                                     cudaMemcpyDeviceToHost, s), "d2h pairs");
    int32_t flag = 0;
    S2O_CUDA_TRY(cudaMemcpyAsync(&flag, wbase + L.pass + align256(generic_scratch_bytes(a)),
                                 sizeof(int32_t), cudaMemcpyDeviceToHost, s), "d2h flag");
    S2O_CUDA_TRY(cudaStreamSynchronize(s), "sync");
    if (flag == 1) return fail(S2O_ERR_UNINIT_STATE, "uninitialized state");
    if (flag == 2) return fail(S2O_ERR_UNCOVERED_ROW, "uncovered query row");
    g_err.clear();
    return S2O_OK;
}

void s2o_host_release(void) {
    std::lock_guard<std::mutex> lock(g_host.mu);
    if (g_host.dev) cudaFree(g_host.dev);
    g_host.dev = nullptr;
    g_host.bytes = 0;
    if (g_host.flags) cudaFreeHost(g_host.flags);
    g_host.flags = nullptr;
    g_host.nflags = 0;
    for (cudaStream_t* s : {&g_host.stream, &g_host.s_in, &g_host.s_out}) {
        if (*s) cudaStreamDestroy(*s);
        *s = nullptr;
    }
    for (int b = 0; b < 2; ++b)
        for (cudaEvent_t* e : {&g_host.ev_h2d[b], &g_host.ev_comp[b], &g_host.ev_d2h[b], &g_host.ev_kv[b]}) {
            if (*e) cudaEventDestroy(*e);
            *e = nullptr;
        }
}

}  // extern "C"
