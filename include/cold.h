/* include/cold.h — C ABI of the B200-native COLD pre-ranking scorer.
 *
 * COLD (arXiv 2007.16122, "COLD: Towards the Next Generation of Pre-Ranking System").
 * Citations: "P:n" = PAPER.md line n, with the section or equation it falls in.
 *
 * One request is one user against N candidate ads (§2: the pre-ranking stage
 * scores ~10^4 candidates and passes the top N on). For every ad the library computes
 *   1. rows of every selected feature group: user / ad ids, and user x ad cross
 *      features (§3.3 "computes cross-features"; construction = DESIGN.md AMB-9);
 *   2. e_g = sum-pooled embedding of the rows ("sum-pooling");
 *   3. ê_g = linear_log(e_g) elementwise (P:278-287 Eq. eq:log; "in the first layer");
 *   4. s_g = sigmoid(w_g . ê_g + b_g), v_g = s_g ê_g (SE gate, P:11-14 Doc A / P:229-235
 *      §3.2; per-group reading AMB-1);
 *   5. x = concat of v_g over the selected groups in schema order ("D_in");
 *   6. the FC stack D_in x 1024 x 512 x 256 x 128 x 64 x 2 (§4.1) with ReLU
 *      (AMB-6) between layers;
 *   7. p = sigmoid(z1 - z0) for a 2-wide head, sigmoid(z) for a 1-wide head (AMB-7);
 * and cold_topk selects the K best ads per request by p (or eCPM = p * bid, P:155
 * footnote / P:332), ties by ascending position, NaN last (AMB-13).
 *
 * User-side groups are computed once per request and broadcast over its ads; their
 * contribution to FC1 (W1[:, user] x_u + b1) is computed once per request (exact:
 * FC1 is linear and, with the per-group SE, v_u does not depend on the ad).
 *
 * Conventions for every entry point:
 *  - Returns cold_status; never throws, never aborts. On an argument / shape error
 *    nothing is launched and outputs are untouched. cold_last_error() gives a
 *    thread-local detail message for the last failing call.
 *  - Launches are asynchronous on the given stream (cudaStream_t passed as void*;
 *    NULL = legacy default stream) unless stated otherwise. Asynchronous CUDA faults
 *    surface as COLD_ERR_CUDA on a later call.
 *  - A cold_ctx is externally synchronised (like a cuBLAS handle): one thread / stream
 *    at a time.
 *  - "device or host" pointers: the library inspects each pointer
 *    (cudaPointerGetAttributes). A batch whose id arrays are host memory (pinned
 *    recommended) is staged to the device by the library chunk by chunk on an internal
 *    copy stream, overlapped with compute; all arrays of one batch must then be host.
 */
#ifndef COLD_H
#define COLD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cold_ctx cold_ctx;   /* opaque: device parameters + workspace + streams */

typedef enum {
  COLD_OK = 0,
  COLD_ERR_INVALID_ARG = 1,   /* NULL pointer, bad enum, non-monotone offsets, empty request */
  COLD_ERR_SHAPE = 2,         /* widths chain / selection / group refs inconsistent */
  COLD_ERR_ID_RANGE = 3,      /* an id outside [0, cardinality) (only with COLD_VALIDATE_IDS) */
  COLD_ERR_K_RANGE = 4,       /* K < 1 or K > ads of some request */
  COLD_ERR_NOT_LOADED = 5,    /* scoring before cold_load_params */
  COLD_ERR_PARAMS = 6,        /* parameter arrays missing or wrong dtype */
  COLD_ERR_OOM = 7,           /* device allocation failed */
  COLD_ERR_CUDA = 8,          /* a CUDA runtime / driver call failed */
  COLD_ERR_UNSUPPORTED = 9,   /* a configuration this build has no kernel for */
  COLD_ERR_CAPACITY = 10      /* more requests / ads in one call than the ctx was created for */
} cold_status;

enum { COLD_USER = 0, COLD_AD = 1, COLD_CROSS = 2 };          /* feature-group side */
enum { COLD_FP32 = 0, COLD_FP16 = 1, COLD_BF16 = 2 };         /* compute / storage precision */
/* hidden activation: ReLU (AMB-6: the paper never names it), or PReLU with a learned slope per channel,
 * h = x for x > 0 and a_c x otherwise (the model-variant row SURVEY §8(f) F2; cold_params.act_slope) */
enum { COLD_RELU = 0, COLD_PRELU = 1 };

/* config.flags */
#define COLD_VALIDATE_IDS 1u   /* check every id against its cardinality (one D2H sync per call);
                                  without it out-of-range ids are clamped to card-1 */

/* config.kernel_flags: kernel-selection overrides. 0 selects the measured-fastest kernels;
 * the others exist so that the tests cover every kernel the library can fall back to (non-paper
 * widths, small calls) and for A/B measurement. Results are identical up to the stated tolerances. */
#define COLD_K_LAYERWISE    1u   /* FC1..FC3 as separate GEMM launches instead of the chain kernel */
#define COLD_K_NO_U1_MMA    2u   /* FC1 adds u1[request] in the epilogue instead of one extra K=16 MMA */
#define COLD_K_SINGLE_CTA   4u   /* single-CTA tcgen05 GEMMs instead of CTA pairs (cta_group::2) */
#define COLD_K_PAIR_STREAM  8u   /* CTA-pair GEMMs stream their weight half instead of keeping it resident */
#define COLD_K_STREAM_B    16u   /* single-CTA GEMMs stream the weight tile instead of keeping it resident */
#define COLD_K_TAIL_NONE   32u   /* no fused tail kernel: every hidden layer a GEMM (head fused into the last) */
#define COLD_K_TAIL3       64u   /* the FC(L-3)..head fused tail instead of FC(L-2)..head (tail45) */
#define COLD_K_CHAIN_TAIL 128u   /* FC4/FC5/head inside the chain kernel, in TMEM (H3/H4 as A operands; measured 1.5% slower; ReLU only) */
#define COLD_K_SERIAL_USER 256u  /* calls of <= 4 requests: user kernel before the gather, one stream */
#define COLD_K_NO_PDL     512u   /* no programmatic dependent launch between the kernels */
#define COLD_K_X_ROWS    1024u   /* X_ac row-major (512 B rows) instead of the half-slab layout */
#define COLD_K_LAT_TAIL45 2048u  /* small calls (below chain_min_ads): FC3 pair GEMM + tail45 instead of the FC3-FC5 tail kernel */
#define COLD_K_LAT_FC2_256 4096u /* small calls: FC2 as 256-wide pair tiles instead of 128-wide ones */

/* A feature group ("the embedding of the i-th feature group e_i"). */
typedef struct {
  int32_t side;          /* COLD_USER / COLD_AD / COLD_CROSS */
  int32_t pooled;        /* AD groups: 1 = multi-valued bag (CSR offsets), 0 = one id per ad.
                            USER groups are always CSR; pooled = 0 declares bags of exactly 1 (a
                            performance hint: crosses of two single groups are gathered in the merged
                            single-row pass; a request with another bag length still scores correctly
                            through the general path). CROSS: ignored (rows = user bag x ad bag, x-major). */
  int64_t cardinality;   /* table rows, >= 1 */
  int32_t user_ref;      /* CROSS: schema index of a USER group */
  int32_t ad_ref;        /* CROSS: schema index of an AD group */
} cold_group;

typedef struct {
  int32_t num_groups;            /* M, 1..64 */
  const cold_group* groups;      /* [M], schema order */
  int32_t emb_dim;               /* k, uniform over groups (16); one of 2, 4, 8, 16, 32 */
  int32_t num_selected;          /* groups fed to the network; 0 = all */
  const int32_t* selected;       /* [num_selected] schema indices, strictly ascending */
  int32_t num_layers;            /* L >= 1 */
  const int32_t* widths;         /* [L] FC output widths; input of layer 0 = D_in = k * #selected;
                                    last width in {1, 2}. Tensor-core path (FP16/BF16): L >= 2,
                                    hidden widths multiples of 64, last hidden width <= 256. */
  int32_t activation;            /* COLD_RELU or COLD_PRELU (slopes in cold_params.act_slope); every kernel
                                    path applies either (with PReLU, widths that would use the 3-layer
                                    fused tail run those layers as GEMMs instead) */
  int32_t linear_log;            /* 1 = apply linear_log to every pooled group embedding */
  int32_t precision;             /* COLD_FP32 (SIMT FFMA, no TF32), COLD_FP16, COLD_BF16 (tcgen05) */
  int32_t device;                /* CUDA device ordinal */
  int64_t max_ads_per_call;      /* capacity: ads summed over the requests of one call */
  int32_t max_requests_per_call; /* capacity: requests in one call */
  int32_t chunk_ads;             /* ads per pipeline chunk (0 = library default) */
  uint32_t flags;                /* COLD_VALIDATE_IDS */
  int32_t se_mode;               /* COLD_SE_GROUP (0, default): s_g = sigma(w_g . e_g + b_g), one k-vector
                                    per group (DESIGN.md AMB-1, Doc A). COLD_SE_DENSE (1): the
                                    other reading of P:229-234 (Doc B), s = sigma(W [e_1 .. e_M] + b) with
                                    W [n_sel x D_in] over the whole LL'd concat: s_g then depends on the ad,
                                    so the user block is no longer hoisted into u1 (FC1 runs over all D_in
                                    columns; cold_params.se_w_dense / se_b_dense are required, se_w / se_b
                                    are ignored). Not with cold_se_stats (COLD_ERR_UNSUPPORTED). */
  uint32_t kernel_flags;         /* COLD_K_* overrides; 0 = default kernel selection */
  int32_t gather_span_chunks;    /* chunks per column-wise gather pass; 0 = default (16) */
  int64_t chain_min_ads;         /* chunks of fewer ads run FC1..FC3 layer by layer (the chain needs >= 2
                                    256-row blocks per CTA pair to fill the GPU); 0 = default (256 x SMs),
                                    1 = the chain for every chunk */
  int32_t gather_ring;           /* cross-bag gather columns (user bag x single ad id): 0 = default, their own
                                    launch with register-held row bursts; -1 = one launch for every column;
                                    4, 5 or 8 = their own launch through a cp.async ring of that depth */
} cold_config;

enum { COLD_SE_GROUP = 0, COLD_SE_DENSE = 1 };

/* Model parameters. All pointers are HOST memory; cold_load_params copies them
 * synchronously, so the caller may free them on return. */
typedef struct {
  int32_t table_dtype;           /* dtype of `tables`: COLD_FP32 (the library rounds to the compute
                                    precision, RNE) or equal to config.precision (stored as-is; bf16 /
                                    fp16 as uint16 bit patterns) */
  const void* const* tables;     /* [M] each [cardinality x k], row-major */
  const float* se_w;             /* [M x k]  SE weight w_g (per-group reading AMB-1) */
  const float* se_b;             /* [M]      SE bias b_g */
  const float* const* fc_w;      /* [L] each [out_l x in_l], row-major (in_0 = D_in, schema order of
                                    the selected groups); rounded RNE to the compute precision for the
                                    tensor-core layers; the per-request user block of W1 stays fp32 */
  const float* const* fc_b;      /* [L] each [out_l], kept fp32 */
  /* Optional input normalisation ("one solution is to use normalization
   * layers like the batch-norm layer ... batch-norm layers use Float32"): inference-time batch norm
   * of the network input folded to an affine map per input column, x_j <- x_j * in_scale[j] +
   * in_shift[j] (in_scale = gamma / sqrt(var + eps), in_shift = beta - mean * in_scale), applied in
   * fp32 after the SE gate and before the 16-bit cast. [D_in] each, schema order of the selected
   * groups; both NULL = none. Usually paired with linear_log = 0 (the paper's other choice). */
  const float* in_scale;
  const float* in_shift;
  /* se_mode == COLD_SE_DENSE only (NULL otherwise): row j = output s_j of the j-th selected group
   * (schema order), columns = the D_in concat of the selected groups' linear_log'ed embeddings in
   * schema order; fp32, kept fp32 on the device (the gate is computed with fp32 FFMA). */
  const float* se_w_dense;       /* [n_sel x D_in] */
  const float* se_b_dense;       /* [n_sel] */
  /* activation == COLD_PRELU only (NULL otherwise): [L-1] each [out_l], the per-channel slopes of the
   * hidden layers, kept fp32 (COLD_ERR_PARAMS when missing). */
  const float* const* act_slope;
} cold_params;

/* One call's requests. Column-major per group ("column based computation"). */
typedef struct {
  int32_t num_requests;          /* R >= 1 */
  const int32_t* ad_offsets;     /* [R+1] ads of request r are [ad_offsets[r], ad_offsets[r+1]); device or host */
  const int32_t* ad_offsets_host;/* [R+1] host copy (sizing and validation without a sync); required */
  const int32_t* const* ids;     /* host array [M] of pointers: USER -> ids of the CSR bags; AD -> [N_tot]
                                    (single) or the bag ids; CROSS -> NULL (always computed) */
  const int32_t* const* offs;    /* host array [M] of pointers: USER -> [R+1]; AD pooled -> [N_tot+1];
                                    otherwise NULL */
  const int32_t* const* offs_host;/* host array [M] of host copies of `offs` (NULL entries allowed when
                                    ids are device memory; required for pooled groups of a host batch).
                                    Every non-NULL entry is validated on the host before any launch:
                                    offs[0] == 0 and non-decreasing over its R+1 (USER) or N_tot+1 (AD)
                                    entries, else COLD_ERR_INVALID_ARG. Bag offsets given only in device
                                    memory are NOT checked (a precondition: malformed device offsets read
                                    out of bounds). */
} cold_batch;

typedef struct {
  uint64_t version;              /* parameter version, +1 per cold_load_params */
  int32_t d_in, d_user, d_ad;    /* input widths: total, hoisted user part, ad + cross part */
  int32_t chunk_ads;             /* ads per pipeline chunk */
  int32_t kernels_per_chunk;     /* kernel launches per chunk */
  int32_t kernels_per_call;      /* launches per call outside the chunk loop */
  int32_t tensor_core;           /* 1 if the FC stack runs on tcgen05 */
  int64_t device_bytes;          /* device memory owned by the ctx */
  int32_t compressed_activations;/* 1 if the activation buffers got compressible memory (COLD_COMPRESS=1) */
  int32_t gather_span_chunks;    /* chunks per column-wise gather pass */
} cold_info;

/* Create a context on config->device: validates the schema (AMB-1..AMB-18 readings in
 * DESIGN.md), allocates the workspace for the stated capacities. */
cold_status cold_create(const cold_config* config, cold_ctx** out);
void cold_destroy(cold_ctx* ctx);

/* A context for another stream that shares src's device parameters (no second copy of the tables)
 * and owns its own workspace: the multi-stream serving form of the paper's MPS setup.
 * src must outlive the clone; cold_load_params on a clone, or on src while clones exist, returns
 * COLD_ERR_UNSUPPORTED. Clones of clones are refused (COLD_ERR_INVALID_ARG). */
cold_status cold_ctx_clone(cold_ctx* src, cold_ctx** out);

/* Upload parameters (synchronous). Replaces any previous version after all work already
 * queued on the ctx's streams (no call sees a mix of versions). */
cold_status cold_load_params(cold_ctx* ctx, const cold_params* params, uint64_t* version_out);

/* Score all ads of a batch: scores[N_tot] fp32 (device or host). */
cold_status cold_score_batch(cold_ctx* ctx, const cold_batch* batch, float* scores, void* stream);

/* Same as cold_score_batch for exactly one request (R == 1), the latency path. */
cold_status cold_score_request(cold_ctx* ctx, const cold_batch* one, float* scores, void* stream);

/* Per-request top-K: for request r, the K ads with the largest key, key = scores
 * (pCTR) or scores * bids (eCPM) when bids != NULL, ordered by (key desc, position asc),
 * NaN last. idx_out[r*K + i] = position of the ad within request r; key_out[r*K + i] = key.
 * scores / bids / ad_offsets / outputs: device or host. */
cold_status cold_topk(cold_ctx* ctx, const float* scores, const int32_t* ad_offsets,
                      const int32_t* ad_offsets_host, int32_t R, int32_t K, const float* bids,
                      int32_t* idx_out, float* key_out, void* stream);

/* ---- intra-request ad split across GPUs (P:248-250 / P:496-498: a query's
 * ads are split, scored in parallel, and the partial results merged) --------------------------
 * Split rule: rank g of G owns ads [floor(g * n_r / G), floor((g + 1) * n_r / G)) of request r
 * (n_r = ad_offsets[r+1] - ad_offsets[r]). Each rank scores its slices and runs cold_topk with
 * K = Kl on them; the G lists are all-gathered (e.g. NCCL all_gather_into_tensor) into
 * cand_key / cand_idx of layout [G][R][Kl] (rank-major), cand_idx = positions inside the rank's
 * slice as cold_topk returns them. cold_merge_topk then selects, per request, the K best of the
 * G * Kl candidates by (key desc, position asc) — identical to cold_topk over the unsplit request
 * whenever every slice has >= Kl ads and K <= Kl (ties: candidates are visited in rank order, and
 * within a rank in position order, which is request position order).
 * idx_out[r*K + i] = position within request r; key_out[r*K + i] = key. All buffers device memory
 * except ad_offsets_host. Errors: COLD_ERR_K_RANGE if K > Kl or a slice has < Kl ads. */
cold_status cold_merge_topk(cold_ctx* ctx, const float* cand_key, const int32_t* cand_idx, int32_t G, int32_t R,
                            int32_t Kl, const int32_t* ad_offsets, const int32_t* ad_offsets_host, int32_t K,
                            int32_t* idx_out, float* key_out, void* stream);

/* ---- the vector-product based pre-ranking model COLD is compared with (
 * PAPER.md L160-166 §2.2: p = sigma(v_u^T v_a), Table tab:sys) -------------------------------
 * Serving form: v_a precomputed per ad (ad tower), v_u per request (user tower). For every ad a of
 * request r: scores[a] = sigma(user_vecs[r] . ad_vecs[ad_ids[a]]), fp32 accumulation in index order.
 * ad_vecs: [num_vecs][d] of vec_dtype (COLD_FP32 / COLD_FP16 / COLD_BF16 bits), 32 B aligned;
 * user_vecs: [R][d] fp32; ad_ids: [N_tot]; ad_offsets: [R+1] (device) + its host copy; scores:
 * [N_tot] fp32. All device memory. d in {16, 32, 64, 128, 256}. Ids outside [0, num_vecs) are
 * clamped. Stateless: no ctx. Top-K of the result: cold_topk. */
cold_status cold_vps_score(const void* ad_vecs, int32_t vec_dtype, int64_t num_vecs, int32_t d, const float* user_vecs,
                           const int32_t* ad_ids, const int32_t* ad_offsets, const int32_t* ad_offsets_host,
                           int32_t R, float* scores, void* stream);

cold_status cold_get_info(const cold_ctx* ctx, cold_info* out);

/* ---- feature-group selection (§3.2 "Importance weight calculation" / "Feature group
 * selection") ------------------------------------------------------------ */

/* SE importance weights of EVERY schema group (selected or not) averaged over the ads of a
 * batch: mean_s_out[g] = (1 / N_tot) * sum over ads of s_g, s_g = sigma(w_g . LL(e_g) + b_g)
 * (per-group SE, AMB-1; a user group's s_g is shared by all ads of its request). The batch must
 * be device memory and carry the ids of every non-cross group. mean_s_out: HOST [M] fp64.
 * Runs on `stream` and synchronises it. Errors: as cold_score_batch; COLD_ERR_INVALID_ARG for a
 * host batch. The per-ad sums are accumulated with fp64 atomics, so the last bits may vary run
 * to run; the ranking below is insensitive to that except at exact ties. */
cold_status cold_se_stats(cold_ctx* ctx, const cold_batch* batch, double* mean_s_out, void* stream);

/* Host helper: the K groups with the largest mean_s (ties: lower schema index first), written
 * in ascending schema order to selected_out[K] — the `selected` list of a lighter COLD
 * ("select K groups of features with top weights"). Errors: COLD_ERR_K_RANGE unless
 * 1 <= K <= M; COLD_ERR_INVALID_ARG for NULL pointers. */
cold_status cold_select_groups(const double* mean_s, int32_t M, int32_t K, int32_t* selected_out);

/* ---- per-kernel timing (bench) -------------------------------------------------------- */

/* Kernel classes reported by cold_profile_read. Every launch is recorded under the class of the
 * kernel that ran, so a call that mixes the chain with the layer-by-layer GEMMs (e.g. a small last
 * chunk) never attributes one kernel's time to another's FLOPs. */
enum { COLD_PROF_USER = 0, COLD_PROF_GATHER = 1, COLD_PROF_TOPK = 2,
       COLD_PROF_FC = 3 /* + layer: one layer-by-layer tcgen05 GEMM (the last hidden one with the head fused) */,
       COLD_PROF_SE_DENSE = 3 + 16 /* the dense SE gate kernel */,
       COLD_PROF_CHAIN = 20 /* chain_kernel: FC1 -> FC2 -> FC3 in one launch */,
       COLD_PROF_TAIL = 21 /* fused tail: FC(L-2) -> FC(L-1) -> head (tail45) or FC(L-3) .. head */,
       COLD_PROF_MLP_F32 = 22 /* fp32 SIMT network (every layer) */,
       COLD_PROF_KINDS = 23 };

/* enable = 1: reset counters and record a CUDA event pair around every kernel the library
 * launches (on the launching stream); enable = 0: stop recording. */
cold_status cold_profile(cold_ctx* ctx, int32_t enable);

/* Synchronises the recorded events and returns, per kernel class, the summed device time
 * (ms), the launch count and the ALGORITHMIC FLOPs those launches computed since the last
 * cold_profile(ctx, 1): 2 * rows * sum(in_l * out_l) over the layers the launch covers (FC
 * classes; the hoisted user GEMV counts 2 * D_u * H per request under COLD_PROF_USER; 0 for the
 * other classes). Arrays of COLD_PROF_KINDS; `flop` may be NULL. */
cold_status cold_profile_read(cold_ctx* ctx, double* total_ms, int64_t* launches, double* flop);

/* ---- parity hooks (tests) ------------------------------------------------------------ */

/* Raw pooled sums e_g (before linear_log / SE), fp32, summed in bag order (cross: x-major):
 * out[N_tot][n_sel][k], device memory. */
cold_status cold_debug_pooled(cold_ctx* ctx, const cold_batch* batch, float* out, void* stream);

/* The network input x = [v_g] as the FC stack consumes it, widened to fp32:
 * out[N_tot][D_in], device memory (schema order of the selected groups; user groups are the
 * per-request fp32 values, ad/cross groups the stored fp16/bf16/fp32 values). */
cold_status cold_debug_features(cold_ctx* ctx, const cold_batch* batch, float* out, void* stream);

/* Rows of group g for every ad: rows_out[N_tot][max_rows] int64, -1 padded, device memory. */
cold_status cold_debug_rows(cold_ctx* ctx, const cold_batch* batch, int32_t group, int64_t* rows_out,
                            int32_t max_rows, void* stream);

/* ---- request-coalescing server (serving path; §3.3 and P:690-692: after Float16 each query was
 * too small to fill the GPU and the paper added MPS; here requests that arrive while the GPU is busy are
 * concatenated into one cold_score_batch + cold_topk call, with a dispatcher thread owning the ctx) ---- */

typedef struct cold_server cold_server;   /* opaque */

typedef struct {
  int32_t max_batch_requests;    /* requests coalesced into one call, 1 .. ctx max_requests_per_call */
  int64_t max_batch_ads;         /* ads in one call, 1 .. ctx max_ads_per_call (also the largest request) */
  int32_t top_k;                 /* K of every request (each request needs >= K ads) */
  int32_t max_wait_us;           /* an idle GPU waits up to this long for a fuller batch (0: dispatch at once) */
} cold_server_config;

/* Starts the dispatcher thread. The ctx must be loaded and must not be used by anyone else until
 * cold_server_destroy. Errors: COLD_ERR_CAPACITY (limits above the ctx's), COLD_ERR_K_RANGE, COLD_ERR_OOM. */
cold_status cold_server_create(cold_ctx* ctx, const cold_server_config* config, cold_server** out);
/* Completes queued requests, then stops the thread and frees the server (not the ctx). */
void cold_server_destroy(cold_server* server);
/* Enqueue the R requests of a HOST batch (cold_batch layout, offs_host required for bag groups). With
 * arrival_ns ([R], CLOCK_MONOTONIC nanoseconds) the call enqueues request r at arrival_ns[r] (spinning
 * until then: an open-loop replay); NULL enqueues all now. Request r's top-K (positions within the
 * request, keys; as cold_topk) is written to idx_out / key_out [r * K .. r * K + K) (host), after which
 * done_ns[r] receives the completion time (CLOCK_MONOTONIC ns; -1 if its call failed), stored with
 * release semantics; done_ns[r] is 0 until then. The batch arrays and the outputs must stay valid until
 * cold_server_drain returns. Errors (nothing enqueued): COLD_ERR_INVALID_ARG (also for device-memory arrays:
 * the dispatcher copies request slices on the CPU), COLD_ERR_K_RANGE (a request
 * with fewer than K ads), COLD_ERR_CAPACITY (a request larger than max_batch_ads). */
cold_status cold_server_submit(cold_server* server, const cold_batch* requests, const int64_t* arrival_ns,
                               int32_t* idx_out, float* key_out, int64_t* done_ns);
/* Waits until every submitted request is complete; returns the first error a coalesced call hit (its
 * requests got done_ns = -1; cold_last_error of the dispatcher thread is not visible here) or COLD_OK.
 * batches_out / requests_out (nullable): calls issued and requests they carried so far. */
cold_status cold_server_drain(cold_server* server, int64_t* batches_out, int64_t* requests_out);

const char* cold_status_string(cold_status s);
const char* cold_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* COLD_H */
