/*
 * include/s2o_cuda.h -- C-ABI of the B200-native S2O sparse prefill attention operator.
 *
 * This is the drop-in boundary for the reference's hot path. Each entry
 * point replaces one C++ function of the reference's public headers
 * (/root/reference/proj/include/s2o/{plan,kernel,tensor}.hpp); the citation is on each
 * declaration. Everything below is plain C: device pointers, sizes, a POD config mirroring
 * s2o::KernelConfig 1:1, and a CUDA stream passed as void*. No torch types.
 *
 * Conventions
 *  - Device entry points are stream-ordered and asynchronous; they never allocate device
 *    buffers, never synchronise, and are thread-safe for distinct streams/workspaces. They may be
 *    captured into a CUDA graph (s2o_attention_fwd's data-dependent plan levels are a graph
 *    WHILE node: added to the capturing graph, or launched as a cached graph otherwise).
 *  - Q is [Z, Hq, L, D]; K and V are [Z, Hkv, L, D] (GQA: q head h reads kv head
 *    h / (Hq/Hkv)). Element strides (batch, head, token) are given per tensor; the channel
 *    stride is 1. So both the reference [Z,H,L,D] layout and [Z,L,H,D] are accepted.
 *  - Segment layout (plan.hpp:16-29): N = ceil(L/S), last_len = L-(N-1)S, prefix(n) = nS.
 *  - q_perm   int32 [Z, Hq, N, S]    segment-local query offsets, best-first
 *                                     (segment n holds len(n) valid entries)
 *  - kv_perm  int32 [Z, Hq, P]       P = S*N*(N-1)/2; segment n at S*n*(n-1)/2, nS absolute
 *                                     token ids of the causal prefix, best-first
 *  - pass buffers: acc fp32 [Z,Hq,L,D] (unnormalised), ell fp32 [Z,Hq,L], m fp32 [Z,Hq,L]
 *    (running max of q.k/sqrt(D) in natural-log units, as PassBuffers kernel.hpp:31-47)
 *  - trace: processed int32 [Z, Hq, N, T], T = ceil(S/b_m) (committed prefix chunks per
 *    query tile; unused tail slots of a short last segment are 0), pass1_pairs/pass2_pairs
 *    int64 [Z, Hq] (KernelTrace kernel.hpp:52-66).
 *  - Status codes mirror the reference's exception messages one-to-one; the text of the last
 *    failure on the calling thread is returned by s2o_last_error().
 */
#ifndef S2O_CUDA_H_
#define S2O_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define S2O_ABI_VERSION 1

typedef enum s2o_status {
    S2O_OK = 0,
    S2O_ERR_SEG_LEN = 1,          /* "segment length must satisfy 1 <= S <= L" plan.cpp:37, kernel.cpp:168 */
    S2O_ERR_TAU = 2,              /* "tau must be >= 0" kernel.cpp:171 */
    S2O_ERR_TILES = 3,            /* "tile sizes must be >= 1" kernel.cpp:174 */
    S2O_ERR_LOCAL_WINDOW = 4,     /* "local window must satisfy W <= S" kernel.cpp:177 */
    S2O_ERR_FUSED_REORDER = 5,    /* "fused variant requires q_reorder = false" kernel.cpp:180 */
    S2O_ERR_FUSED_FLAGS = 6,      /* "fused variant requires fused = true, q_reorder = false" kernel.cpp:306 */
    S2O_ERR_PLAN_MISMATCH = 7,    /* "plan/config mismatch: segment layout differs" kernel.cpp:30 */
    S2O_ERR_BUFS_MISMATCH = 8,    /* "pass buffers do not match tensor dims" kernel.cpp:246 */
    S2O_ERR_QKV_DIMS = 9,         /* "Q/K/V dims must match" attention.cpp:24, kernel.cpp:189 */
    S2O_ERR_UNINIT_STATE = 10,    /* "uninitialized state" kernel.cpp:228 */
    S2O_ERR_EMPTY_SCORES = 11,    /* "empty score vector" tensor.cpp:45 */
    S2O_ERR_UNCOVERED_ROW = 12,   /* "uncovered query row" kernel.cpp:155 */
    S2O_ERR_NORMALIZER_ALIGN = 13,/* "normalizer vectors must align" kernel.cpp:223 */
    S2O_ERR_INVALID_ARG = 14,     /* null pointer, bad stride/dtype, Hq % Hkv != 0 */
    S2O_ERR_UNSUPPORTED = 15,     /* a shape no kernel of this build covers */
    S2O_ERR_WORKSPACE = 16,       /* workspace smaller than *_workspace_size() */
    S2O_ERR_CUDA = 17,            /* CUDA runtime error (text in s2o_last_error) */
    S2O_ERR_NO_DEVICE = 18,       /* no sm_100 device / kernels not loadable */
    S2O_ERR_BLOCK_BUDGET = 19     /* "block budget must have positive shape and k >= 0" baseline.cpp:23 */
} s2o_status;

typedef enum s2o_dtype { S2O_F32 = 0, S2O_BF16 = 1 } s2o_dtype;

/* Which kernels run the attention passes. AUTO picks the tcgen05 path when the shape is
 * covered (bf16, D=128, b_m=128, b_n=128, strides multiples of D), the generic SIMT fp64 path
 * otherwise. */
typedef enum s2o_path { S2O_PATH_AUTO = 0, S2O_PATH_GENERIC = 1, S2O_PATH_TCGEN05 = 2 } s2o_path;

/* How prefix keys / queries are scored for the permutation.
 * EXACT: fp64, sequential over d, identical to dot_f (plan.cpp:14-20) -> bit-identical plans.
 * FAST : reserved; every entry point rejects it with S2O_ERR_UNSUPPORTED. */
typedef enum s2o_score_mode { S2O_SCORE_EXACT = 0, S2O_SCORE_FAST = 1 } s2o_score_mode;

/* Problem geometry. Strides are in elements. */
typedef struct s2o_problem {
    int64_t z, hq, hkv, l, d;
    int32_t in_dtype;   /* s2o_dtype of Q, K, V */
    int32_t out_dtype;  /* s2o_dtype of O */
    int64_t q_stride[3], k_stride[3], v_stride[3], o_stride[3]; /* (batch, head, token) */
} s2o_problem;

/* s2o::KernelConfig (kernel.hpp:19-28) 1:1, plus execution knobs. */
typedef struct s2o_kernel_config {
    int64_t seg_len;      /* S */
    double tau;           /* early-stop threshold */
    int64_t b_m, b_n;     /* TileSpec (attention.hpp:15-18) */
    int32_t q_reorder;    /* bool */
    int32_t fused;        /* bool */
    int64_t local_window; /* -1 == S; only bounds-checked (kernel.hpp:16-18) */
    int32_t path;         /* s2o_path */
    int32_t score_mode;   /* s2o_score_mode */
    int32_t plan_depth;   /* kv_perm entries per segment s2o_attention_fwd materialises when the
                             caller does not ask for kv_perm: 0 = auto (6144), -1 = the full
                             permutation, > 0 = that many (rounded up to b_n). A tile that walks
                             its whole truncated list without stopping saves its state (fp32
                             acc, ell, m) and resumes on the next level (the following entries
                             of the same order). Traces and pair counts do not depend on this
                             knob; outputs agree to the fp32 state re-basing at level
                             boundaries (about one bf16 ulp). */
} s2o_kernel_config;

/* ------------------------------------------------------------------ utilities */
int s2o_abi_version(void);
const char* s2o_last_error(void);
const char* s2o_status_string(int status);
/* Fill a problem with dense [Z,H,L,D] strides. */
void s2o_problem_init(s2o_problem* p, int64_t z, int64_t hq, int64_t hkv, int64_t l, int64_t d,
                      int32_t in_dtype, int32_t out_dtype);
/* s2o::KernelConfig defaults (kernel.hpp:19-28): S=128, tau=0.005, 128x128, q_reorder. */
void s2o_kernel_config_init(s2o_kernel_config* c);
/* KernelConfig::validate (kernel.cpp:166-182). */
s2o_status s2o_kernel_config_validate(const s2o_kernel_config* c, int64_t l);
/* early_stop_check (kernel.cpp:220-234) on host arrays; *stop = 1 iff max gain < tau. */
s2o_status s2o_early_stop_check(const double* prev_ell, const double* new_ell, int64_t n,
                                double tau, int32_t* stop);
/* Which attention path AUTO resolves to for (problem, config): 1 generic, 2 tcgen05. */
s2o_status s2o_select_path(const s2o_problem* p, const s2o_kernel_config* c, int32_t* path);

/* ------------------------------------------------- Step 1: block scoring + permutation */
/* Bytes of device workspace s2o_plan_build needs for this problem and segment length. */
s2o_status s2o_plan_workspace_size(const s2o_problem* p, int64_t seg_len, size_t* bytes);

/* segment_representatives (plan.hpp:100-102, plan.cpp:46-67): fp64 sequential segment means
 * of Q -> q_mean fp32 [Z,Hq,N,D] and of K -> k_mean fp32 [Z,Hkv,N,D]. Either output may be
 * NULL. */
s2o_status s2o_segment_representatives(const s2o_problem* p, const void* q, const void* k,
                                       int64_t seg_len, float* q_mean, float* k_mean,
                                       void* stream);

/* rank_queries (plan.hpp:104-106, plan.cpp:69-101) with a caller-given guide, fp32 [Z, Hq, D] on the
 * device (one vector per q head): s_Q = fp64 sequential dot(Q row, guide), per-segment stable
 * descending argsort -> q_perm int32 [Z, Hq, N, S] (segment-local). Plan workspace. */
s2o_status s2o_rank_queries(const s2o_problem* p, const void* q, const float* guide, int64_t seg_len,
                            int32_t* q_perm, void* workspace, size_t workspace_bytes, void* stream);

/* rank_prefix_keys (plan.hpp:108-111, plan.cpp:103-138) with caller-given segment representatives
 * q_mean fp32 [Z, Hq, N, D] on the device: s_K[n, t] = fp64 sequential dot(q_mean[n], K[t]) for
 * t < nS, stable descending argsort -> kv_perm (packed as for s2o_plan_build). Plan workspace. */
s2o_status s2o_rank_prefix_keys(const s2o_problem* p, const void* k, const float* q_mean, int64_t seg_len,
                                int32_t* kv_perm, void* workspace, size_t workspace_bytes, void* stream);

/* build_plan (plan.hpp:115-116, plan.cpp:140-162): guide = k_mean[segment 0], q_perm
 * (rank_queries plan.cpp:69-101), kv_perm (rank_prefix_keys plan.cpp:103-138). Uses
 * cfg->seg_len and cfg->score_mode. cost2 (host, optional) receives RankingCost
 * {dot_products, sort_items} per (z,h) slice. */
s2o_status s2o_plan_build(const s2o_problem* p, const void* q, const void* k,
                          const s2o_kernel_config* cfg, int32_t* q_perm, int32_t* kv_perm,
                          int64_t* cost2, void* workspace, size_t workspace_bytes, void* stream);

/* Truncated plan for the fused operator: q_perm as above, and the exact top `depth` entries
 * of every kv_perm segment (== the first min(nS, depth) entries of argsort_desc_stable), laid
 * out int32 [Z, Hq, N, depth] (segment 0 unused), depth <= 6144. Selection, not a full sort. The
 * device int32 *flag is set to 1 if a segment's selection could not be certified (then use
 * s2o_plan_build). Same workspace as s2o_plan_build. */
s2o_status s2o_plan_build_truncated(const s2o_problem* p, const void* q, const void* k,
                                    const s2o_kernel_config* cfg, int64_t depth, int32_t* q_perm,
                                    int32_t* kv_top, int32_t* flag, void* workspace,
                                    size_t workspace_bytes, void* stream);

/* ------------------------------------------------------ Step 2: sparse attention passes */
/* pass1_dense_init (kernel.hpp:70-71, kernel.cpp:184-218). */
s2o_status s2o_pass1(const s2o_problem* p, const void* q, const void* k, const void* v,
                     const s2o_kernel_config* cfg, float* acc, float* ell, float* m,
                     void* workspace, size_t workspace_bytes, void* stream);

/* pass2_sparse (kernel.hpp:83-86, kernel.cpp:236-298): resumes pass buffers, walks kv_perm
 * chunks with the monotone-gain stop, writes O (scattered to original rows) and the trace. */
s2o_status s2o_pass2(const s2o_problem* p, const void* q, const void* k, const void* v,
                     const s2o_kernel_config* cfg, const float* acc, const float* ell,
                     const float* m, const int32_t* q_perm, const int32_t* kv_perm, void* o,
                     int32_t* processed, int64_t* pass1_pairs, int64_t* pass2_pairs,
                     void* workspace, size_t workspace_bytes, void* stream);

/* fused_single_pass (kernel.hpp:92-95, kernel.cpp:300-349): requires fused && !q_reorder. */
s2o_status s2o_fused(const s2o_problem* p, const void* q, const void* k, const void* v,
                     const s2o_kernel_config* cfg, const int32_t* kv_perm, void* o,
                     int32_t* processed, int64_t* pass1_pairs, int64_t* pass2_pairs,
                     void* workspace, size_t workspace_bytes, void* stream);

/* Bytes of workspace s2o_pass1/s2o_pass2/s2o_fused need (generic path scratch). */
s2o_status s2o_pass_workspace_size(const s2o_problem* p, const s2o_kernel_config* cfg,
                                   size_t* bytes);

/* Device-side errors of the last s2o_pass1/s2o_pass2/s2o_fused on `workspace`, which the
 * asynchronous entry points cannot return: reads the workspace's status word on `stream`
 * (synchronises it) and returns S2O_ERR_UNINIT_STATE ("uninitialized state", kernel.cpp:228),
 * S2O_ERR_UNCOVERED_ROW ("uncovered query row", kernel.cpp:155) or S2O_OK. */
s2o_status s2o_pass_status(const s2o_problem* p, const s2o_kernel_config* cfg, const void* workspace,
                           size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------- whole operator */
/* Workspace for s2o_attention_fwd: plan + pass buffers + scratch. */
s2o_status s2o_attention_workspace_size(const s2o_problem* p, const s2o_kernel_config* cfg,
                                        size_t* bytes);

/* Same as s2o_pass_status for the workspace of the last s2o_attention_fwd. */
s2o_status s2o_attention_status(const s2o_problem* p, const s2o_kernel_config* cfg, const void* workspace,
                                size_t workspace_bytes, void* stream);

/* s2o_attention (kernel.hpp:106-107, kernel.cpp:351-369): validate -> build_plan ->
 * (fused ? fused : pass1 + pass2). q_perm / kv_perm / processed / pair outputs are optional
 * (NULL -> kept in the workspace). When kv_perm is NULL the plan keeps only the exact top
 * plan_depth entries of each kv_perm segment (selection instead of a full sort); tiles that
 * exhaust them resume on the next plan level (see plan_depth). Device errors are reported by
 * s2o_attention_status. */
s2o_status s2o_attention_fwd(const s2o_problem* p, const void* q, const void* k, const void* v,
                             const s2o_kernel_config* cfg, void* o, int32_t* q_perm,
                             int32_t* kv_perm, int32_t* processed, int64_t* pass1_pairs,
                             int64_t* pass2_pairs, void* workspace, size_t workspace_bytes,
                             void* stream);

/* Same operator on HOST buffers (the reference's calling convention: Tensor4 in, result
 * out). Copies inputs host->device, runs s2o_attention_fwd on an internal stream with a
 * cached device arena, copies O (and the optional plan/trace outputs) back, synchronises.
 * Host pointers may be pageable or pinned. */
s2o_status s2o_attention_host(const s2o_problem* p, const void* q, const void* k, const void* v,
                              const s2o_kernel_config* cfg, void* o, int32_t* q_perm,
                              int32_t* kv_perm, int32_t* processed, int64_t* pass1_pairs,
                              int64_t* pass2_pairs);
/* Release the arena held by s2o_attention_host. */
void s2o_host_release(void);

/* Dense causal attention on the device through the same kernels with S = L (one segment,
 * pass-1 only): the MSE comparator path (attention.hpp:42). O in p->out_dtype. */
s2o_status s2o_dense_causal_fwd(const s2o_problem* p, const void* q, const void* k,
                                const void* v, int32_t path, void* o, void* workspace,
                                size_t workspace_bytes, void* stream);

/* --------------------------------------------------------------- block top-k baseline */
/* block_topk_attention (baseline.hpp:28-36, baseline.cpp:106-185): per query block of
 * block_rows rows, the self block plus the `topk` full prefix blocks of largest causal softmax
 * mass (exact fp64 ranking, ties to the lower block) are kept and a masked softmax runs over
 * them. Square blocks only (block_rows == block_cols). O in p->out_dtype; pair_count int64
 * [Z, Hq] = computed causal pairs (BlockTopkResult::pair_count). path as s2o_select_path
 * (tcgen05 for the masked attention when bf16, D = 128 and 128-token blocks). */
s2o_status s2o_block_topk_workspace_size(const s2o_problem* p, int64_t block_rows, int64_t block_cols,
                                         int64_t topk, size_t* bytes);
s2o_status s2o_block_topk_fwd(const s2o_problem* p, const void* q, const void* k, const void* v,
                              int64_t block_rows, int64_t block_cols, int64_t topk, int32_t path, void* o,
                              int64_t* pair_count, void* workspace, size_t workspace_bytes, void* stream);

/* --------------------------------------------------------------- synthetic inputs */
/* generate_synthetic (synthetic.hpp:45, synthetic.cpp:276-328) on the host, bit-identical
 * to the reference generator: pattern in {"gaussian","vertical","horizontal","slash",
 * "mixed"} (and the "-stripes" spellings); fp32 [Z,H,L,D] outputs; threads = 0 -> all
 * hardware threads. */
s2o_status s2o_synthetic_generate(const char* pattern, int64_t stripe_count, double stripe_gain,
                                  uint64_t seed, int64_t z, int64_t h, int64_t l, int64_t d,
                                  float* q, float* k, float* v, int32_t threads);

#ifdef __cplusplus
}
#endif
#endif /* S2O_CUDA_H_ */
