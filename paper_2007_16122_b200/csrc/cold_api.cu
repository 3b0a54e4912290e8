// cold_api.cu — host runtime behind include/cold.h: context, parameter upload, the chunked
// scoring pipeline, host-batch staging, top-K and the parity hooks.
//
// Per call:
//   user_kernel (once per request: x_u, u1 = b1 + W1_u x_u, ad -> request map)
//   for each chunk of `chunk_ads` ads (kept L2-sized so X_ac / H1 / H2 stay on chip):
//     gather_kernel  (ad + cross groups, column-wise)           -> X_ac   [chunk][D_ac_pad]
//     gemm FC1 (+u1[request], ReLU)                              -> H1     [chunk][1024]
//     gemm FC2 .. FC(L-2) (+bias, ReLU)                          -> H2 ...
//     gemm FC(L-1) (+bias, ReLU) with FC L + sigmoid fused       -> scores [chunk]
// fp32 precision replaces the GEMMs by the SIMT kernel mlp_f32 (no TF32).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/cold.h"
#include "internal.h"

using namespace cold;

static thread_local std::string g_last_error;
static unsigned long long* g_instr = nullptr;   // debug wait-cycle counters (COLD_INSTR)

static cold_status fail(cold_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

#define CK(call)                                                                                        \
  do {                                                                                                  \
    cudaError_t _e = (call);                                                                            \
    if (_e != cudaSuccess)                                                                              \
      return fail(COLD_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e));                   \
  } while (0)

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

struct cold_ctx {
  // ---- configuration ----
  int M = 0, k = 0, L = 0, precision = 0, device = 0, linear_log = 1;
  uint32_t flags = 0;
  std::vector<cold_group> groups;
  std::vector<int> sel, widths, sel_user, sel_ac, sel_pos;
  std::vector<int> gather_order;     // sel_ac positions, heaviest (cross over a user bag) first
  int d_u = 0, d_ac = 0, d_ac_pad = 0, d_in = 0;
  bool dense_se = false;             // COLD_SE_DENSE: X holds all D_in columns (schema order), u1 = b1
  int d_x = 0;                       // X width before padding: d_ac (per-group SE) or d_in (dense SE)
  int64_t max_ads = 0;
  int max_req = 0, chunk = 0, num_sms = 148;
  bool tensor = false;
  int bn[COLD_MAX_LAYERS] = {0};
  // ---- parameters (device) ----
  bool loaded = false;
  uint64_t version = 0;
  std::vector<void*> d_tables;
  DevGroup* d_groups = nullptr;
  std::vector<DevGroup> h_groups;    // host copy (gather kernel parameters)
  float* d_se_w = nullptr;
  std::vector<float> h_se_w, h_se_b;   // host copies (the gather passes its columns' SE weights as parameters)
  float* d_se_b = nullptr;
  float* d_w1u_t = nullptr;
  float* d_b1 = nullptr;
  void* d_w[COLD_MAX_LAYERS] = {nullptr};    // tensor path: compute-dtype weights of GEMM layers
  float* d_b[COLD_MAX_LAYERS] = {nullptr};
  float* d_wt[COLD_MAX_LAYERS] = {nullptr};  // fp32 path: transposed weights
  float* d_head_w = nullptr;
  float* d_head_b = nullptr;
  float* d_in_scale = nullptr;       // folded input batch norm [D_in] (nullable)
  float* d_in_shift = nullptr;
  float* d_sewd_t = nullptr;         // dense SE: Wd^T [D_in][n_sel] fp32
  float* d_sebd = nullptr;           // dense SE: bd [n_sel]
  bool prelu = false;                // COLD_PRELU hidden activation (F2)
  float* d_slope[COLD_MAX_LAYERS] = {nullptr};   // PReLU slopes of hidden layer l [out_l] fp32
  CUtensorMap tmB[COLD_MAX_LAYERS];
  // ---- workspace ----
  float* d_u1 = nullptr;
  float* d_xu = nullptr;
  float* d_E = nullptr;              // dense SE: [gspan * chunk][d_in] fp32 pre-SE ê of the span
  int32_t* d_req = nullptr;
  void* d_X = nullptr;
  void* d_H[COLD_MAX_LAYERS] = {nullptr};
  CUtensorMap tmA[COLD_MAX_LAYERS];
  std::vector<CUtensorMap> tmAX;     // layer-0 A maps, one per chunk slot of the gather span
  bool x_slab = false;               // X_ac in the half-slab layout [2 slot + h][span rows][8]
  bool u1mma = false;                // FC1 adds u1[request(row)] on the tensor core (kernels_gemm2.cu)
  bool chain = false;                // FC1 -> FC3 in one persistent kernel over 256-row blocks
  int64_t chain_min = 0;             // chunks smaller than this use the layer-by-layer kernels
  int u1_terms = 0, u1t_ld = 0;
  uint16_t* d_u1t = nullptr;         // [u1_terms * H][u1t_ld] 16-bit terms of u1 (written by user_kernel)
  uint16_t* d_ohot = nullptr;        // [gspan * chunk][16] one-hot u1 operand rows (written by gather)
  CUtensorMap tmU1T;
  bool chain_tail = false;           // FC4 -> FC5 -> head inside the chain kernel too
  CUtensorMap tmW4h, tmW5h;          // W4 / W5 with half-N boxes (CTA-pair tiles)
  // small calls (below chain_min: one request) run FC3 -> FC4 -> FC5 -> head in the one-CTA tail kernel
  // instead of the FC3 pair GEMM + tail45 (one launch fewer and 32 CTAs instead of 16 pairs for FC3)
  bool lat_tail3 = false;
  CUtensorMap tmW3full;              // W3 with whole-N boxes for that kernel
  // small calls also run FC2 as 128-wide pair tiles (twice the CTA pairs of the 256-wide tiles)
  bool lat_fc2_128 = false;
  CUtensorMap tmW2q;                 // W2 with 64-row boxes (half of a 128-wide pair tile)
  std::vector<CUtensorMap> tmOH;     // per chunk slot of the span
  int gspan = 1;                     // chunks per column-wise gather pass (X_ac holds gspan * chunk rows)
  int gather_ring = 0;               // > 0: cross-bag columns through a cp.async ring of this depth
  uint32_t kflags = 0;               // cold_config.kernel_flags
  int64_t cfg_chain_min = 0;         // cold_config.chain_min_ads / gather_span_chunks / gather_ring as given
  int cfg_span = 0, cfg_ring = 0;    //   (cold_ctx_clone recreates the same selection)
  CUtensorMap tmC[COLD_MAX_LAYERS];  // epilogue TMA-store maps (32 x 32 boxes)
  int cs[COLD_MAX_LAYERS] = {0};     // cluster size (weight-tile multicast) per GEMM layer
  bool resb[COLD_MAX_LAYERS] = {false};  // weight slice resident in shared memory (K x BN <= 128 KB)
  bool pair[COLD_MAX_LAYERS] = {false};  // CTA-pair (cta_group::2) GEMM
  bool pair_res[COLD_MAX_LAYERS] = {false};  // ... with the pair's weight half resident (one n-tile per pair)
  int tail_mode = 0;                 // 0: every layer a GEMM (head fused into the last); 1: FC(L-3..L-1) +
                                     // head fused (tail_kernel); 2: FC(L-2..L-1) + head fused (tail45_kernel)
  int n_tail = 0;                    // hidden layers inside the fused tail (0, 3 or 2)
  bool pdl = true;                   // programmatic dependent launch between the GEMM kernels
  int* d_err = nullptr;
  float* d_scores_stage = nullptr;  // [2][chunk] for host outputs
  int32_t* d_adoff = nullptr;       // [max_req+1] staged ad offsets
  const int32_t* cur_adoff = nullptr;  // device ad offsets of the call in flight
  // host-batch staging
  cudaStream_t copy_stream = nullptr;
  cudaStream_t side_stream = nullptr;   // few-request calls: the user kernel runs here, beside the gather
  cudaEvent_t ev_fork = nullptr, ev_user = nullptr;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_consumed[2] = {nullptr, nullptr};
  cudaEvent_t ev_scored[2] = {nullptr, nullptr}, ev_drained[2] = {nullptr, nullptr};
  void* d_stage[2] = {nullptr, nullptr};
  size_t stage_bytes = 0;
  void* d_user_stage = nullptr;
  size_t user_stage_bytes = 0;
  float* d_topk_in = nullptr;
  size_t topk_in_bytes = 0;
  void* d_topk_out = nullptr;
  size_t topk_out_bytes = 0;
  int64_t device_bytes = 0;
  std::vector<void*> allocs;
  // per-kernel event profiling
  bool prof = false;
  std::vector<cudaEvent_t> prof_events;       // pool
  size_t prof_used = 0;
  std::vector<int> prof_kind;                 // kind of each recorded pair
  std::vector<double> prof_fl;                // algorithmic FLOPs of each recorded pair
  double prof_ms[COLD_PROF_KINDS] = {0};
  int64_t prof_n[COLD_PROF_KINDS] = {0};
  double prof_flop[COLD_PROF_KINDS] = {0};

  bool owns_params = true;           // false for cold_ctx_clone contexts (parameters shared)
  cold_ctx* clone_of = nullptr;
  int clones = 0;                    // live clones sharing this context's parameters
  ~cold_ctx() {
    cudaSetDevice(device);
    cudaDeviceSynchronize();
    if (clone_of) clone_of->clones--;
    for (void* p : allocs) cudaFree(p);
    for (int i = 0; i < 2; i++) {
      if (d_stage[i]) cudaFree(d_stage[i]);
      if (ev_copied[i]) cudaEventDestroy(ev_copied[i]);
      if (ev_consumed[i]) cudaEventDestroy(ev_consumed[i]);
      if (ev_scored[i]) cudaEventDestroy(ev_scored[i]);
      if (ev_drained[i]) cudaEventDestroy(ev_drained[i]);
    }
    if (d_user_stage) cudaFree(d_user_stage);
    if (d_topk_in) cudaFree(d_topk_in);
    if (d_topk_out) cudaFree(d_topk_out);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (side_stream) cudaStreamDestroy(side_stream);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_user) cudaEventDestroy(ev_user);
    for (cudaEvent_t e : prof_events) cudaEventDestroy(e);
    freeParams();
    cudaGetLastError();
  }
  void freeParams() {
    if (!owns_params) {   // a clone only drops its references
      d_tables.clear();
      return;
    }
    for (void* p : d_tables) cudaFree(p);
    d_tables.clear();
    void** ps[] = {(void**)&d_groups, (void**)&d_se_w, (void**)&d_se_b, (void**)&d_w1u_t, (void**)&d_b1,
                   (void**)&d_head_w, (void**)&d_head_b, (void**)&d_in_scale, (void**)&d_in_shift,
                   (void**)&d_sewd_t, (void**)&d_sebd};
    for (void** p : ps) { if (*p) cudaFree(*p); *p = nullptr; }
    for (int l = 0; l < COLD_MAX_LAYERS; l++) {
      if (d_w[l]) cudaFree(d_w[l]);
      if (d_b[l]) cudaFree(d_b[l]);
      if (d_wt[l]) cudaFree(d_wt[l]);
      if (d_slope[l]) cudaFree(d_slope[l]);
      d_w[l] = nullptr; d_b[l] = nullptr; d_wt[l] = nullptr; d_slope[l] = nullptr;
    }
  }
  cudaError_t alloc(void** p, size_t bytes) {
    cudaError_t e = cudaMalloc(p, bytes < 16 ? 16 : bytes);
    if (e == cudaSuccess) { allocs.push_back(*p); device_bytes += (int64_t)bytes; }
    return e;
  }
  int elem() const { return precision == COLD_FP32 ? 4 : 2; }
  // input width of layer l as the kernels see it (layer 0: the ad + cross part, or all of D_in under
  // dense SE; the hoisted user block is counted with the user kernel)
  int layer_k(int l) const { return l == 0 ? d_x : widths[l - 1]; }
  // algorithmic FLOPs of layers [l0, l1) over n rows (l1 == L includes the head)
  double layer_flop(int l0, int l1, int64_t n) const {
    double f = 0.0;
    for (int l = l0; l < l1; l++) f += 2.0 * (double)layer_k(l) * (double)widths[l];
    return f * (double)n;
  }
  // bracket one kernel launch with an event pair (only while profiling)
  void mark_begin(cudaStream_t st) {
    if (!prof) return;
    while (prof_events.size() < prof_used + 2) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      prof_events.push_back(e);
    }
    cudaEventRecord(prof_events[prof_used], st);
  }
  void mark_end(int kind, cudaStream_t st, double flop = 0.0) {
    if (!prof) return;
    cudaEventRecord(prof_events[prof_used + 1], st);
    prof_kind.push_back(kind);
    prof_fl.push_back(flop);
    prof_used += 2;
    if (prof_used >= 8192) flush_profile();
  }
  void flush_profile() {
    if (prof_used == 0) return;
    cudaEventSynchronize(prof_events[prof_used - 1]);
    for (size_t i = 0; i < prof_kind.size(); i++) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, prof_events[2 * i], prof_events[2 * i + 1]);
      prof_ms[prof_kind[i]] += ms;
      prof_n[prof_kind[i]] += 1;
      prof_flop[prof_kind[i]] += prof_fl[i];
    }
    prof_kind.clear();
    prof_fl.clear();
    prof_used = 0;
  }
};

// ---------------------------------------------------------------------------------------------
extern "C" const char* cold_status_string(cold_status s) {
  switch (s) {
    case COLD_OK: return "ok";
    case COLD_ERR_INVALID_ARG: return "invalid argument";
    case COLD_ERR_SHAPE: return "shape mismatch";
    case COLD_ERR_ID_RANGE: return "id out of range";
    case COLD_ERR_K_RANGE: return "K out of range";
    case COLD_ERR_NOT_LOADED: return "parameters not loaded";
    case COLD_ERR_PARAMS: return "bad parameters";
    case COLD_ERR_OOM: return "out of device memory";
    case COLD_ERR_CUDA: return "CUDA error";
    case COLD_ERR_UNSUPPORTED: return "unsupported configuration";
    case COLD_ERR_CAPACITY: return "capacity exceeded";
  }
  return "unknown status";
}

extern "C" const char* cold_last_error(void) { return g_last_error.c_str(); }

static bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

static int pick_bn(int n) {
  if (n % 256 == 0) return 256;
  if (n % 128 == 0) return 128;
  return 64;
}

// 2-D row-major [rows][inner] 16-bit tensor; box {box_cols, box_rows}; operands use 64-col boxes with
// 128 B swizzle (tcgen05 SW128 K-major atoms), epilogue outputs 32-col boxes with 64 B swizzle.
static cold_status make_tmap(CUtensorMap* tm, void* ptr, int precision, uint64_t inner, uint64_t rows,
                             uint32_t box_rows, uint32_t box_cols = 64) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(COLD_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(tm, precision == COLD_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                   2, ptr, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   box_cols == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(COLD_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return COLD_OK;
}

// X_ac half-slab planes [planes][rows_total][8] 16-bit, viewed from chunk row offset `ptr`: a 3-D map
// {256 elements = 32 rows x 8 columns (contiguous in a plane), row group of 32, plane}, box {256, 4, 8} =
// one 64-column k-block of 128 rows in 512 B lines, landing as [8 planes][128 rows][8] = four no-swizzle
// K-major K = 16 operands (sdesc_k16_plain at +kk * BM * 32)
static cold_status make_tmap_slab(CUtensorMap* tm, void* ptr, int precision, uint64_t rows, uint64_t rows_total,
                                  uint64_t planes) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(COLD_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[3] = {256, rows / 32, planes};
  cuuint64_t strides[2] = {512, rows_total * 16};
  cuuint32_t box[3] = {256, 4, 8};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(tm, precision == COLD_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                   3, ptr, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(COLD_ERR_CUDA, "cuTensorMapEncodeTiled (slab) failed: " + std::to_string((int)r));
  return COLD_OK;
}

// 2-D 16-bit tensor, no swizzle: box rows of box_cols * 2 bytes land contiguously (the FC1 u1 operand)
static cold_status make_tmap_plain(CUtensorMap* tm, void* ptr, int precision, uint64_t inner, uint64_t rows,
                                   uint32_t box_rows, uint32_t box_cols) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(COLD_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(tm, precision == COLD_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                   2, ptr, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(COLD_ERR_CUDA, "cuTensorMapEncodeTiled (plain) failed: " + std::to_string((int)r));
  return COLD_OK;
}

// ---------------------------------------------------------------------------------------------
extern "C" cold_status cold_create(const cold_config* cfg, cold_ctx** out) {
  if (!cfg || !out) return fail(COLD_ERR_INVALID_ARG, "null config/out");
  *out = nullptr;
  if (cfg->num_groups < 1 || cfg->num_groups > COLD_MAX_GROUPS || !cfg->groups)
    return fail(COLD_ERR_INVALID_ARG, "num_groups must be in [1, 64]");
  if (cfg->emb_dim != 2 && cfg->emb_dim != 4 && cfg->emb_dim != 8 && cfg->emb_dim != 16 && cfg->emb_dim != 32)
    return fail(COLD_ERR_UNSUPPORTED, "emb_dim must be 2, 4, 8, 16 or 32");
  if (cfg->num_layers < 1 || cfg->num_layers > COLD_MAX_LAYERS || !cfg->widths)
    return fail(COLD_ERR_SHAPE, "num_layers must be in [1, 16]");
  if (cfg->precision < COLD_FP32 || cfg->precision > COLD_BF16) return fail(COLD_ERR_INVALID_ARG, "bad precision");
  if (cfg->activation != COLD_RELU && cfg->activation != COLD_PRELU)
    return fail(COLD_ERR_UNSUPPORTED, "activation must be COLD_RELU or COLD_PRELU");
  if (cfg->max_ads_per_call < 1 || cfg->max_requests_per_call < 1)
    return fail(COLD_ERR_INVALID_ARG, "capacities must be >= 1");
  for (int l = 0; l < cfg->num_layers; l++)
    if (cfg->widths[l] < 1) return fail(COLD_ERR_SHAPE, "widths must be >= 1");
  const int last = cfg->widths[cfg->num_layers - 1];
  if (last != 1 && last != 2) return fail(COLD_ERR_SHAPE, "last width must be 1 or 2");
  for (int g = 0; g < cfg->num_groups; g++) {
    const cold_group& G = cfg->groups[g];
    if (G.side < COLD_USER || G.side > COLD_CROSS) return fail(COLD_ERR_INVALID_ARG, "bad group side");
    if (G.cardinality < 1 || G.cardinality > (int64_t)1 << 40) return fail(COLD_ERR_INVALID_ARG, "bad cardinality");
    if (G.side == COLD_CROSS) {
      if (G.user_ref < 0 || G.user_ref >= cfg->num_groups || cfg->groups[G.user_ref].side != COLD_USER ||
          G.ad_ref < 0 || G.ad_ref >= cfg->num_groups || cfg->groups[G.ad_ref].side != COLD_AD)
        return fail(COLD_ERR_SHAPE, "cross group must reference a USER and an AD group");
    }
  }
  cold_ctx* c = new cold_ctx();
  c->M = cfg->num_groups;
  c->k = cfg->emb_dim;
  c->L = cfg->num_layers;
  c->precision = cfg->precision;
  c->device = cfg->device;
  c->linear_log = cfg->linear_log ? 1 : 0;
  c->prelu = cfg->activation == COLD_PRELU;
  c->flags = cfg->flags;
  c->groups.assign(cfg->groups, cfg->groups + cfg->num_groups);
  c->widths.assign(cfg->widths, cfg->widths + cfg->num_layers);
  if (cfg->num_selected > 0) {
    if (!cfg->selected) { delete c; return fail(COLD_ERR_INVALID_ARG, "selected is NULL"); }
    for (int j = 0; j < cfg->num_selected; j++) {
      int g = cfg->selected[j];
      if (g < 0 || g >= c->M || (j > 0 && g <= cfg->selected[j - 1])) {
        delete c;
        return fail(COLD_ERR_SHAPE, "selected must be strictly ascending schema indices");
      }
      c->sel.push_back(g);
    }
  } else {
    for (int g = 0; g < c->M; g++) c->sel.push_back(g);
  }
  if (c->sel.empty()) { delete c; return fail(COLD_ERR_SHAPE, "empty selection"); }
  c->sel_pos.assign(c->M, -1);
  for (size_t j = 0; j < c->sel.size(); j++) {
    int g = c->sel[j];
    c->sel_pos[g] = (int)j;
    if (c->groups[g].side == COLD_USER) c->sel_user.push_back(g);
    else c->sel_ac.push_back(g);
  }
  // heaviest-first dispatch order for the gather grid: cross groups over pooled bags first
  for (int pass = 0; pass < 3; pass++)
    for (size_t j = 0; j < c->sel_ac.size(); j++) {
      const cold_group& G = c->groups[c->sel_ac[j]];
      // class 0: cross groups (a user bag x ad id: L rows each); 1: ad bags; 2: single ad ids
      const int cls = G.side == COLD_CROSS ? 0 : (G.pooled ? 1 : 2);
      if (cls == pass) c->gather_order.push_back((int)j);
    }
  c->d_u = (int)c->sel_user.size() * c->k;
  c->d_ac = (int)c->sel_ac.size() * c->k;
  c->d_in = c->d_u + c->d_ac;
  if (cfg->se_mode != COLD_SE_GROUP && cfg->se_mode != COLD_SE_DENSE) { delete c; return fail(COLD_ERR_INVALID_ARG, "se_mode"); }
  c->dense_se = cfg->se_mode == COLD_SE_DENSE;
  c->d_x = c->dense_se ? c->d_in : c->d_ac;
  if (c->dense_se && se_dense_smem(c->d_in, (int)c->sel.size()) > 227 * 1024 - 1024) {
    delete c;
    return fail(COLD_ERR_UNSUPPORTED, "dense SE: Wd^T (D_in x n_sel fp32) must fit in shared memory");
  }
  c->max_ads = cfg->max_ads_per_call;
  c->max_req = cfg->max_requests_per_call;
  c->kflags = cfg->kernel_flags;
  c->cfg_chain_min = cfg->chain_min_ads;
  c->cfg_span = cfg->gather_span_chunks;
  c->cfg_ring = cfg->gather_ring;
  // 0 (default): cross-bag columns in their own register-burst launch; -1: one launch for all columns;
  // 4 / 5 / 8: cross-bag columns through a cp.async ring of that depth (measured slower: DESIGN.md §9)
  c->gather_ring = cfg->gather_ring;
  if (c->gather_ring != -1 && c->gather_ring != 4 && c->gather_ring != 5 && c->gather_ring != 8) c->gather_ring = 0;

  if (cudaSetDevice(c->device) != cudaSuccess) { delete c; return fail(COLD_ERR_CUDA, "cudaSetDevice failed"); }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, c->device) != cudaSuccess) {
    delete c;
    return fail(COLD_ERR_CUDA, "cudaGetDeviceProperties failed");
  }
  c->num_sms = prop.multiProcessorCount;
  c->tensor = (c->precision != COLD_FP32);
  if (c->tensor) {
    if (prop.major != 10) { delete c; return fail(COLD_ERR_UNSUPPORTED, "tcgen05 path needs an sm_100 device"); }
    if (c->L < 2) { delete c; return fail(COLD_ERR_UNSUPPORTED, "tensor-core path needs >= 2 layers"); }
    for (int l = 0; l < c->L - 1; l++)
      if (c->widths[l] % 64 != 0) { delete c; return fail(COLD_ERR_UNSUPPORTED, "hidden widths must be multiples of 64"); }
    const int pen = c->widths[c->L - 2];
    if (pen != 64 && pen != 128 && pen != 256) {
      delete c;
      return fail(COLD_ERR_UNSUPPORTED, "last hidden width must be 64, 128 or 256");
    }
    for (int l = 0; l < c->L - 1; l++) c->bn[l] = (l == c->L - 2) ? pen : pick_bn(c->widths[l]);
    c->d_ac_pad = std::max(64, (c->d_x + 63) / 64 * 64);
  } else {
    c->d_ac_pad = std::max(1, c->d_x);
  }
  int chunk = cfg->chunk_ads > 0 ? cfg->chunk_ads : c->num_sms * 128 * 8;
  if (c->tensor) chunk = (chunk + 127) / 128 * 128;
  c->chunk = (int)std::min<int64_t>(chunk, std::max<int64_t>(c->max_ads, 128));
  if (c->tensor) c->chunk = (c->chunk + 127) / 128 * 128;
  {
    // Column-wise gather over a span of several chunks ("column based computation"): one
    // group column is gathered for every ad of the span before the next group starts, so each
    // table's hot rows are fetched from HBM once per span and then served by L2.
    int span = cfg->gather_span_chunks > 0 ? cfg->gather_span_chunks : 16;   // measured: 4 -> 16 is +4% gather GB/s
    if (span < 1) span = 1;
    const int64_t need = (c->max_ads + c->chunk - 1) / c->chunk;
    c->gspan = (int)std::min<int64_t>(span, std::max<int64_t>(need, 1));
  }

  // ---- workspace ----
  const int W0 = c->widths[0];
  cudaError_t e = cudaSuccess;
  e = e ? e : c->alloc((void**)&c->d_u1, (size_t)c->max_req * W0 * 4);
  e = e ? e : c->alloc((void**)&c->d_xu, (size_t)c->max_req * std::max(1, c->d_u) * 4);
  e = e ? e : c->alloc((void**)&c->d_req, (size_t)c->max_ads * 4);
  const size_t x_rows = (size_t)c->gspan * c->chunk;
  e = e ? e : c->alloc((void**)&c->d_X, x_rows * c->d_ac_pad * c->elem());
  if (c->dense_se) e = e ? e : c->alloc((void**)&c->d_E, x_rows * c->d_in * 4);
  e = e ? e : c->alloc((void**)&c->d_err, 16);
  e = e ? e : c->alloc((void**)&c->d_scores_stage, (size_t)2 * c->chunk * 4);
  e = e ? e : c->alloc((void**)&c->d_adoff, (size_t)(c->max_req + 1) * 4);
  if (c->tensor)
    for (int l = 0; l < c->L - 2 && !e; l++) e = c->alloc(&c->d_H[l], (size_t)c->chunk * c->widths[l] * 2);
  if (e != cudaSuccess) {
    delete c;
    cudaGetLastError();
    return fail(COLD_ERR_OOM, std::string("workspace allocation failed: ") + cudaGetErrorString(e));
  }
  cudaMemset(c->d_X, 0, x_rows * c->d_ac_pad * c->elem());  // pad columns stay 0
  if (c->tensor) {
    const int cs_default = 1;   // weight-tile multicast over clusters measured slower at these sizes
    const uint32_t kf = c->kflags;
    c->pdl = !(kf & COLD_K_NO_PDL);
    const int Lg = c->L - 1;   // GEMM layers (the last layer is fused as the head)
    {
      const int want = (kf & COLD_K_TAIL_NONE) ? 0 : ((kf & COLD_K_TAIL3) ? 1 : 2);
      const int k4 = (Lg - 2 == 0) ? c->d_ac_pad : (Lg >= 3 ? c->widths[Lg - 3] : 0);
      const int k3 = (Lg - 3 == 0) ? c->d_ac_pad : (Lg >= 4 ? c->widths[Lg - 4] : 0);
      if (want == 2 && Lg >= 2 && tail45_supported(c->widths[Lg - 2], c->widths[Lg - 1], k4)) c->tail_mode = 2;
      else if (want >= 1 && Lg >= 3 && !c->prelu &&   // (the 3-layer tail kernel has no PReLU epilogue)
               tail_supported(c->widths[Lg - 3], c->widths[Lg - 2], c->widths[Lg - 1], k3))
        c->tail_mode = 1;
      c->n_tail = c->tail_mode == 1 ? 3 : (c->tail_mode == 2 ? 2 : 0);
    }
    for (int l = 0; l < c->L - 1; l++) {
      void* in = (l == 0) ? c->d_X : c->d_H[l - 1];
      int K = (l == 0) ? c->d_ac_pad : c->widths[l - 1];
      cold_status s = make_tmap(&c->tmA[l], in, c->precision, K, c->chunk, 128);
      if (s) { delete c; return s; }
      if (l == 0) {
        // X_ac half-slabs (coalesced gather stores) when FC1 runs as a GEMM / the chain with per-group SE
        // (not when layer 0 sits inside a fused tail kernel, nor for the dense-SE gate's row-major X)
        c->x_slab = !c->dense_se && c->k % 8 == 0 && (c->L - 1 - c->n_tail) >= 1 && !(c->kflags & COLD_K_X_ROWS);
        c->tmAX.resize(c->gspan);
        for (int j = 0; j < c->gspan; j++) {
          if (c->x_slab)
            s = make_tmap_slab(&c->tmAX[j], (uint8_t*)c->d_X + (size_t)j * c->chunk * 16, c->precision, c->chunk,
                               (uint64_t)c->gspan * c->chunk, (uint64_t)c->d_ac_pad / 8);
          else
            s = make_tmap(&c->tmAX[j], (uint8_t*)c->d_X + (size_t)j * c->chunk * c->d_ac_pad * 2, c->precision, K,
                          c->chunk, 128);
          if (s) { delete c; return s; }
        }
      }
      if (l < c->L - 2) {
        // epilogue store boxes: 32 rows x 64 columns (SW128) when each epilogue warp's column half is a
        // multiple of 64 (epi.cuh), else 32 x 32 (SW64)
        const bool wide = (c->bn[l] / 2) % 64 == 0;   // epi.cuh group boxes: 128 rows x 64 cols (SW128)
        s = make_tmap(&c->tmC[l], c->d_H[l], c->precision, c->widths[l], c->chunk, wide ? 128 : 32, wide ? 64 : 32);
        if (s) { delete c; return s; }
      } else {
        c->tmC[l] = c->tmA[l];   // unused by the head epilogue
      }
      int cs = cs_default;
      while (cs > 1 && (c->bn[l] / cs) % 8 != 0) cs >>= 1;   // B slices must be whole 8-row swizzle atoms
      c->cs[l] = (cs == 4 || cs == 2) ? cs : 1;
      if (c->n_tail && l >= Lg - c->n_tail) c->cs[l] = 1;   // the tail kernels load whole weight tiles
      c->resb[l] = c->cs[l] == 1 && gemm_resident_ok(c->bn[l], K) && !(kf & COLD_K_STREAM_B);
      // CTA pairs for the 256-wide layers that are not fused into the tail (FC1, FC2, FC3)
      const bool in_tail = c->n_tail && l >= Lg - c->n_tail;
      c->pair[l] = !in_tail && l < Lg - 1 && c->bn[l] == 256 && !(kf & COLD_K_SINGLE_CTA);
      if (c->pair[l]) { c->resb[l] = false; c->cs[l] = 1; }
      c->pair_res[l] = c->pair[l] && gemm_pair_resident_ok(c->bn[l], K) && !(kf & COLD_K_PAIR_STREAM);
    }
  }
  if (c->tensor && c->pair[0] && c->n_tail < c->L - 1) {
    c->u1mma = !(c->kflags & COLD_K_NO_U1_MMA);
  }
  if (c->u1mma) {
    c->u1_terms = c->precision == COLD_BF16 ? 3 : 2;
    c->u1t_ld = (c->max_req + 7) / 8 * 8;
    const size_t u1t_bytes = (size_t)c->u1_terms * W0 * c->u1t_ld * 2;
    const size_t oh_bytes = (size_t)c->gspan * c->chunk * 16 * 2;
    cudaError_t e2 = c->alloc((void**)&c->d_u1t, u1t_bytes);
    if (e2 == cudaSuccess) e2 = c->alloc((void**)&c->d_ohot, oh_bytes);
    if (e2 != cudaSuccess) { delete c; cudaGetLastError(); return fail(COLD_ERR_OOM, "u1 operand buffers"); }
    cudaMemset(c->d_u1t, 0, u1t_bytes);   // slots past the last request stay finite (0 x value = 0)
    cold_status s = make_tmap_plain(&c->tmU1T, c->d_u1t, c->precision, c->u1t_ld, (uint64_t)c->u1_terms * W0, 128, 8);
    if (s) { delete c; return s; }
    c->tmOH.resize(c->gspan);
    for (int j = 0; j < c->gspan; j++) {
      s = make_tmap_plain(&c->tmOH[j], c->d_ohot + (size_t)j * c->chunk * 16, c->precision, 16, c->chunk, 128, 8);
      if (s) { delete c; return s; }
    }
  }
  if (c->u1mma && c->tail_mode == 2 && c->L == 6 && c->pair[1] && c->pair[2] &&
      chain_supported(c->widths[0], c->widths[1], c->widths[2], c->d_ac_pad)) {
    c->chain = !(c->kflags & COLD_K_LAYERWISE);
    c->chain_min = cfg->chain_min_ads > 0 ? cfg->chain_min_ads : (int64_t)c->num_sms * 256;
    // COLD_K_CHAIN_TAIL also folds FC4 / FC5 / head into the chain, in TMEM (FC3's epilogue writes H3 back
    // into its accumulator buffer as FC4's A operand, H4 likewise for FC5): no H3 round trip and no tail
    // launch, but the in-place tail holds one of the two 256-column accumulator buffers from FC3 to the
    // head, so FC2's two n-tiles share the other one and wait for each other's drain: 304.9 us per chunk
    // vs 275.6 + 24.8 for chain + tail45 (profiles/r03/ab_tt_*.jsonl), off by default
    c->chain_tail = c->chain && chain_tail_supported(c->widths[3], c->widths[4], c->widths[2]) &&
                    c->widths[5] <= 2 && (c->kflags & COLD_K_CHAIN_TAIL) && !c->prelu;
    c->lat_tail3 = !c->chain_tail && !c->prelu && !(c->kflags & COLD_K_LAT_TAIL45) &&
                   tail_supported(c->widths[2], c->widths[3], c->widths[4], c->widths[1]);
    c->lat_fc2_128 = c->lat_tail3 && c->widths[1] % 128 == 0 && !(c->kflags & COLD_K_LAT_FC2_256);
  }
  if (cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
      [&] {   // the user kernel is on the latency path's critical chain: highest stream priority
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        return cudaStreamCreateWithPriority(&c->side_stream, cudaStreamNonBlocking, hi);
      }() != cudaSuccess) {
    delete c;
    return fail(COLD_ERR_CUDA, "stream create failed");
  }
  cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->ev_user, cudaEventDisableTiming);
  for (int i = 0; i < 2; i++) {
    cudaEventCreateWithFlags(&c->ev_copied[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->ev_consumed[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->ev_scored[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->ev_drained[i], cudaEventDisableTiming);
  }
  if (cudaDeviceSynchronize() != cudaSuccess) { delete c; return fail(COLD_ERR_CUDA, "init sync failed"); }
  *out = c;
  return COLD_OK;
}

extern "C" void cold_destroy(cold_ctx* c) { delete c; }

// A second context over the same device parameters with its own workspace (one per concurrent
// stream): the serving form of the paper's "MPS" multi-stream execution without duplicating
// the 4.8 GB of tables.
extern "C" cold_status cold_ctx_clone(cold_ctx* src, cold_ctx** out) {
  if (!src || !out) return fail(COLD_ERR_INVALID_ARG, "null ctx / out");
  *out = nullptr;
  if (src->clone_of) return fail(COLD_ERR_INVALID_ARG, "clone the source context, not a clone");
  cold_config cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.num_groups = src->M;
  cfg.groups = src->groups.data();
  cfg.emb_dim = src->k;
  cfg.num_selected = (int32_t)src->sel.size();
  cfg.selected = src->sel.data();
  cfg.num_layers = src->L;
  cfg.widths = src->widths.data();
  cfg.activation = src->prelu ? COLD_PRELU : COLD_RELU;
  cfg.linear_log = src->linear_log;
  cfg.precision = src->precision;
  cfg.device = src->device;
  cfg.max_ads_per_call = src->max_ads;
  cfg.max_requests_per_call = src->max_req;
  cfg.chunk_ads = src->chunk;
  cfg.flags = src->flags;
  cfg.se_mode = src->dense_se ? COLD_SE_DENSE : COLD_SE_GROUP;
  cfg.kernel_flags = src->kflags;
  cfg.chain_min_ads = src->cfg_chain_min;
  cfg.gather_span_chunks = src->cfg_span;
  cfg.gather_ring = src->cfg_ring;
  cold_ctx* c = nullptr;
  cold_status s = cold_create(&cfg, &c);
  if (s) return s;
  c->owns_params = false;
  c->clone_of = src;
  src->clones++;
  c->loaded = src->loaded;
  c->version = src->version;
  c->d_tables = src->d_tables;
  c->d_groups = src->d_groups;
  c->h_groups = src->h_groups;
  c->d_se_w = src->d_se_w;
  c->h_se_w = src->h_se_w;
  c->h_se_b = src->h_se_b;
  c->d_se_b = src->d_se_b;
  c->d_w1u_t = src->d_w1u_t;
  c->d_b1 = src->d_b1;
  c->d_head_w = src->d_head_w;
  c->d_head_b = src->d_head_b;
  c->d_in_scale = src->d_in_scale;
  c->d_in_shift = src->d_in_shift;
  c->d_sewd_t = src->d_sewd_t;
  c->d_sebd = src->d_sebd;
  for (int l = 0; l < COLD_MAX_LAYERS; l++) {
    c->d_w[l] = src->d_w[l];
    c->d_b[l] = src->d_b[l];
    c->d_wt[l] = src->d_wt[l];
    c->d_slope[l] = src->d_slope[l];
    c->tmB[l] = src->tmB[l];
  }
  c->tmW4h = src->tmW4h;
  c->tmW5h = src->tmW5h;
  c->tmW3full = src->tmW3full;
  c->tmW2q = src->tmW2q;
  *out = c;
  return COLD_OK;
}

// ---------------------------------------------------------------------------------------------
// RNE fp32 -> fp16 / bf16 on the host (parameter upload only)
static uint16_t f32_to_f16_bits(float f) {
  uint32_t x;
  memcpy(&x, &f, 4);
  uint32_t sign = (x >> 16) & 0x8000u;
  uint32_t ax = x & 0x7fffffffu;
  if (ax > 0x7f800000u) return (uint16_t)(sign | 0x7e00u);         // NaN
  if (ax >= 0x477ff000u) return (uint16_t)(sign | 0x7c00u);         // >= 65520 rounds to inf
  if (ax < 0x38800000u) {                                           // subnormal half
    const uint32_t e = ax >> 23;                                    // |x| = m * 2^(e-150)
    const uint32_t m = (ax & 0x7fffffu) | 0x800000u;                // in units of 2^-24: m >> (126-e)
    const uint32_t shift = 126u - e;                                // 14 .. 126
    if (shift > 24) return (uint16_t)sign;                          // < 2^-25, or the 2^-25 tie -> 0
    uint32_t val = m >> shift;
    const uint32_t rem = m & ((1u << shift) - 1u);
    const uint32_t half = 1u << (shift - 1);
    if (rem > half || (rem == half && (val & 1u))) val++;           // may carry into the smallest normal
    return (uint16_t)(sign | val);
  }
  uint32_t val = ((ax >> 13) - (112u << 10));
  uint32_t rem = ax & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (val & 1))) val++;
  return (uint16_t)(sign | val);
}
static uint16_t f32_to_bf16_bits(float f) {
  uint32_t x;
  memcpy(&x, &f, 4);
  if ((x & 0x7fffffffu) > 0x7f800000u) return 0x7fc0u;
  return (uint16_t)((x + 0x7fffu + ((x >> 16) & 1u)) >> 16);
}

template <typename F>
static cold_status upload(cold_ctx* c, void** dst, size_t bytes, F fill) {
  std::vector<uint8_t> h(bytes);
  fill(h.data());
  if (*dst) { cudaFree(*dst); *dst = nullptr; }
  if (cudaMalloc(dst, bytes < 16 ? 16 : bytes) != cudaSuccess) {
    cudaGetLastError();
    return fail(COLD_ERR_OOM, "parameter allocation failed");
  }
  CK(cudaMemcpy(*dst, h.data(), bytes, cudaMemcpyHostToDevice));
  return COLD_OK;
}

extern "C" cold_status cold_load_params(cold_ctx* c, const cold_params* p, uint64_t* version_out) {
  if (!c || !p) return fail(COLD_ERR_INVALID_ARG, "null ctx/params");
  if (!c->owns_params) return fail(COLD_ERR_UNSUPPORTED, "load parameters through the source context");
  if (c->clones > 0) return fail(COLD_ERR_UNSUPPORTED, "destroy the clones before reloading parameters");
  if (!p->tables || !p->se_w || !p->se_b || !p->fc_w || !p->fc_b) return fail(COLD_ERR_PARAMS, "missing arrays");
  if (p->table_dtype != COLD_FP32 && p->table_dtype != c->precision)
    return fail(COLD_ERR_PARAMS, "table_dtype must be FP32 or the compute precision");
  for (int g = 0; g < c->M; g++) if (!p->tables[g]) return fail(COLD_ERR_PARAMS, "missing table");
  for (int l = 0; l < c->L; l++) if (!p->fc_w[l] || !p->fc_b[l]) return fail(COLD_ERR_PARAMS, "missing fc layer");
  CK(cudaSetDevice(c->device));
  CK(cudaDeviceSynchronize());   // no in-flight call sees a mix of versions
  c->loaded = false;
  c->freeParams();
  const int k = c->k, es = c->elem();
  // tables
  c->d_tables.assign(c->M, nullptr);
  for (int g = 0; g < c->M; g++) {
    const size_t n = (size_t)c->groups[g].cardinality * k;
    void* d = nullptr;
    if (cudaMalloc(&d, n * es) != cudaSuccess) { cudaGetLastError(); return fail(COLD_ERR_OOM, "table allocation failed"); }
    c->d_tables[g] = d;
    if (p->table_dtype == c->precision) {
      CK(cudaMemcpy(d, p->tables[g], n * es, cudaMemcpyHostToDevice));
    } else {   // fp32 -> fp16 / bf16, RNE, in slabs
      const float* src = (const float*)p->tables[g];
      const size_t slab = (size_t)1 << 24;
      std::vector<uint16_t> h(std::min(n, slab));
      for (size_t o = 0; o < n; o += slab) {
        size_t m = std::min(slab, n - o);
        for (size_t i = 0; i < m; i++)
          h[i] = c->precision == COLD_FP16 ? f32_to_f16_bits(src[o + i]) : f32_to_bf16_bits(src[o + i]);
        CK(cudaMemcpy((uint16_t*)d + o, h.data(), m * 2, cudaMemcpyHostToDevice));
      }
    }
  }
  // group descriptors
  std::vector<DevGroup>& dg = c->h_groups;
  dg.assign(c->M, DevGroup());
  std::vector<int> slot(c->M, -1);
  for (size_t j = 0; j < c->sel_user.size(); j++) slot[c->sel_user[j]] = (int)j;
  for (size_t j = 0; j < c->sel_ac.size(); j++) slot[c->sel_ac[j]] = (int)j;
  for (int g = 0; g < c->M; g++) {
    dg[g].table = c->d_tables[g];
    dg[g].card = c->groups[g].cardinality;
    dg[g].side = c->groups[g].side;
    dg[g].pooled = c->groups[g].pooled;
    dg[g].user_ref = c->groups[g].user_ref;
    dg[g].ad_ref = c->groups[g].ad_ref;
    dg[g].sel_slot = slot[g];
    dg[g].sel_pos = c->sel_pos[g];
  }
  cold_status s;
  s = upload(c, (void**)&c->d_groups, sizeof(DevGroup) * c->M, [&](uint8_t* h) { memcpy(h, dg.data(), sizeof(DevGroup) * c->M); });
  if (s) return s;
  s = upload(c, (void**)&c->d_se_w, sizeof(float) * c->M * k, [&](uint8_t* h) { memcpy(h, p->se_w, sizeof(float) * c->M * k); });
  if (s) return s;
  s = upload(c, (void**)&c->d_se_b, sizeof(float) * c->M, [&](uint8_t* h) { memcpy(h, p->se_b, sizeof(float) * c->M); });
  if (s) return s;
  c->h_se_w.assign(p->se_w, p->se_w + (size_t)c->M * k);
  c->h_se_b.assign(p->se_b, p->se_b + c->M);
  if ((p->in_scale == nullptr) != (p->in_shift == nullptr))
    return fail(COLD_ERR_PARAMS, "in_scale and in_shift must both be set or both be NULL");
  if (p->in_scale) {
    s = upload(c, (void**)&c->d_in_scale, sizeof(float) * c->d_in, [&](uint8_t* h) { memcpy(h, p->in_scale, sizeof(float) * c->d_in); });
    if (s) return s;
    s = upload(c, (void**)&c->d_in_shift, sizeof(float) * c->d_in, [&](uint8_t* h) { memcpy(h, p->in_shift, sizeof(float) * c->d_in); });
    if (s) return s;
  }
  if (c->prelu) {   // PReLU slopes of the hidden layers, fp32 (F2)
    if (!p->act_slope) return fail(COLD_ERR_PARAMS, "activation PReLU needs act_slope");
    for (int l = 0; l < c->L - 1; l++) {
      if (!p->act_slope[l]) return fail(COLD_ERR_PARAMS, "act_slope[l] is NULL");
      s = upload(c, (void**)&c->d_slope[l], sizeof(float) * c->widths[l],
                 [&](uint8_t* h) { memcpy(h, p->act_slope[l], sizeof(float) * c->widths[l]); });
      if (s) return s;
    }
  }
  if (c->dense_se) {   // Wd^T [D_in][n_sel] and bd, fp32
    if (!p->se_w_dense || !p->se_b_dense) return fail(COLD_ERR_PARAMS, "se_mode dense needs se_w_dense and se_b_dense");
    const int ns = (int)c->sel.size();
    s = upload(c, (void**)&c->d_sewd_t, sizeof(float) * (size_t)c->d_in * ns, [&](uint8_t* h) {
      float* o = (float*)h;
      for (int j = 0; j < ns; j++)
        for (int i = 0; i < c->d_in; i++) o[(size_t)i * ns + j] = p->se_w_dense[(size_t)j * c->d_in + i];
    });
    if (s) return s;
    s = upload(c, (void**)&c->d_sebd, sizeof(float) * ns, [&](uint8_t* h) { memcpy(h, p->se_b_dense, sizeof(float) * ns); });
    if (s) return s;
  }
  // FC1 split into the per-request user block (fp32, transposed) and the ad+cross block
  // (dense SE: no split; the whole W1 multiplies the per-ad X, schema order)
  const int W0 = c->widths[0];
  const float* W1 = p->fc_w[0];   // [W0][d_in], columns = selected groups in schema order
  const int d_in = c->d_in;
  auto col_of = [&](int g, int d) { return c->sel_pos[g] * k + d; };
  s = upload(c, (void**)&c->d_w1u_t, sizeof(float) * (size_t)std::max(1, c->d_u) * W0, [&](uint8_t* h) {
    float* o = (float*)h;
    for (size_t j = 0; j < c->sel_user.size(); j++)
      for (int d = 0; d < k; d++)
        for (int n = 0; n < W0; n++) o[((size_t)j * k + d) * W0 + n] = W1[(size_t)n * d_in + col_of(c->sel_user[j], d)];
  });
  if (s) return s;
  s = upload(c, (void**)&c->d_b1, sizeof(float) * W0, [&](uint8_t* h) { memcpy(h, p->fc_b[0], sizeof(float) * W0); });
  if (s) return s;
  auto layer_in = [&](int l) { return l == 0 ? d_in : c->widths[l - 1]; };
  if (c->tensor) {
    for (int l = 0; l < c->L - 1; l++) {
      const int out = c->widths[l];
      const int Kp = (l == 0) ? c->d_ac_pad : c->widths[l - 1];
      const float* W = p->fc_w[l];
      s = upload(c, &c->d_w[l], (size_t)out * Kp * 2, [&](uint8_t* h) {
        uint16_t* o = (uint16_t*)h;
        for (int n = 0; n < out; n++)
          for (int kk = 0; kk < Kp; kk++) {
            float v = 0.0f;
            if (l == 0) {
              int j = kk / k, d = kk % k;
              if (c->dense_se) { if (kk < d_in) v = W[(size_t)n * d_in + kk]; }
              else if (j < (int)c->sel_ac.size()) v = W[(size_t)n * d_in + col_of(c->sel_ac[j], d)];
            } else {
              v = W[(size_t)n * Kp + kk];
            }
            o[(size_t)n * Kp + kk] = c->precision == COLD_FP16 ? f32_to_f16_bits(v) : f32_to_bf16_bits(v);
          }
      });
      if (s) return s;
      if (l > 0) {
        s = upload(c, (void**)&c->d_b[l], sizeof(float) * out, [&](uint8_t* h) { memcpy(h, p->fc_b[l], sizeof(float) * out); });
        if (s) return s;
      }
      s = make_tmap(&c->tmB[l], c->d_w[l], c->precision, Kp, out,
                    c->pair[l] ? c->bn[l] / 2 : c->bn[l] / c->cs[l]);
      if (s) return s;
      if (c->lat_tail3 && l == 2) {   // whole-N boxes for the small-call FC3-FC5 tail kernel
        s = make_tmap(&c->tmW3full, c->d_w[l], c->precision, Kp, out, c->bn[l]);
        if (s) return s;
      }
      if (c->lat_fc2_128 && l == 1) {   // 64-row boxes for the small-call 128-wide FC2 pair tiles
        s = make_tmap(&c->tmW2q, c->d_w[l], c->precision, Kp, out, 64);
        if (s) return s;
      }
      if (c->chain_tail && (l == 3 || l == 4)) {   // half-N boxes for the chain's pair tiles
        s = make_tmap(l == 3 ? &c->tmW4h : &c->tmW5h, c->d_w[l], c->precision, Kp, out, out / 2);
        if (s) return s;
      }
    }
    const int hl = c->L - 1, hin = c->widths[hl - 1], hout = c->widths[hl];
    s = upload(c, (void**)&c->d_head_w, sizeof(float) * hout * hin, [&](uint8_t* h) { memcpy(h, p->fc_w[hl], sizeof(float) * hout * hin); });
    if (s) return s;
    s = upload(c, (void**)&c->d_head_b, sizeof(float) * hout, [&](uint8_t* h) { memcpy(h, p->fc_b[hl], sizeof(float) * hout); });
    if (s) return s;
  } else {
    for (int l = 0; l < c->L; l++) {
      const int out = c->widths[l];
      const int in = (l == 0) ? c->d_x : layer_in(l);
      const float* W = p->fc_w[l];
      s = upload(c, (void**)&c->d_wt[l], sizeof(float) * (size_t)std::max(1, in) * out, [&](uint8_t* h) {
        float* o = (float*)h;
        for (int i = 0; i < in; i++)
          for (int n = 0; n < out; n++) {
            float v;
            if (l == 0) v = c->dense_se ? W[(size_t)n * d_in + i] : W[(size_t)n * d_in + col_of(c->sel_ac[i / k], i % k)];
            else v = W[(size_t)n * in + i];
            o[(size_t)i * out + n] = v;
          }
      });
      if (s) return s;
      if (l > 0) {
        s = upload(c, (void**)&c->d_b[l], sizeof(float) * out, [&](uint8_t* h) { memcpy(h, p->fc_b[l], sizeof(float) * out); });
        if (s) return s;
      }
    }
  }
  CK(cudaDeviceSynchronize());
  c->loaded = true;
  c->version++;
  if (version_out) *version_out = c->version;
  return COLD_OK;
}

// ---------------------------------------------------------------------------------------------
// batch validation and views

struct CallPlan {
  int R = 0;
  int64_t N = 0;
  bool host = false;
  std::vector<int> needed;      // non-cross groups whose ids the call reads
  BatchView bv;                 // device-mode view (host mode: per chunk)
};

static cold_status plan_batch(cold_ctx* c, const cold_batch* b, CallPlan& pl, bool all_groups = false) {
  if (!b || !b->ad_offsets || !b->ad_offsets_host || !b->ids || !b->offs)
    return fail(COLD_ERR_INVALID_ARG, "batch arrays missing");
  const int R = b->num_requests;
  if (R < 1) return fail(COLD_ERR_INVALID_ARG, "num_requests must be >= 1");
  if (R > c->max_req) return fail(COLD_ERR_CAPACITY, "more requests than max_requests_per_call");
  const int32_t* ao = b->ad_offsets_host;
  if (ao[0] != 0) return fail(COLD_ERR_INVALID_ARG, "ad_offsets[0] must be 0");
  for (int r = 0; r < R; r++)
    if (ao[r + 1] <= ao[r]) return fail(COLD_ERR_INVALID_ARG, "every request needs >= 1 ad (ad_offsets strictly increasing)");
  pl.R = R;
  pl.N = ao[R];
  if (pl.N > c->max_ads) return fail(COLD_ERR_CAPACITY, "more ads than max_ads_per_call");
  std::vector<char> need(c->M, 0);
  std::vector<int> groups_used = c->sel;
  if (all_groups) {
    groups_used.clear();
    for (int g = 0; g < c->M; g++) groups_used.push_back(g);
  }
  for (int g : groups_used) {
    if (c->groups[g].side == COLD_CROSS) { need[c->groups[g].user_ref] = 1; need[c->groups[g].ad_ref] = 1; }
    else need[g] = 1;
  }
  pl.host = !is_device_ptr(b->ad_offsets);
  for (int g = 0; g < c->M; g++) {
    if (!need[g]) continue;
    pl.needed.push_back(g);
    const cold_group& G = c->groups[g];
    if (!b->ids[g]) return fail(COLD_ERR_INVALID_ARG, "ids missing for a needed group");
    const bool has_offs = (G.side == COLD_USER) || G.pooled;
    if (has_offs && !b->offs[g]) return fail(COLD_ERR_INVALID_ARG, "offsets missing for a bag group");
    if (is_device_ptr(b->ids[g]) == pl.host) return fail(COLD_ERR_INVALID_ARG, "a batch must be all-host or all-device");
    if (pl.host && has_offs && (!b->offs_host || !b->offs_host[g]))
      return fail(COLD_ERR_INVALID_ARG, "host batch needs offs_host for bag groups");
    if (has_offs && b->offs_host && b->offs_host[g]) {   // CSR bag offsets: 0-based, non-decreasing
      const int32_t* o = b->offs_host[g];
      const int64_t len = (G.side == COLD_USER ? (int64_t)R : pl.N) + 1;
      if (o[0] != 0) return fail(COLD_ERR_INVALID_ARG, "bag offsets must start at 0 (group " + std::to_string(g) + ")");
      for (int64_t i = 1; i < len; i++)
        if (o[i] < o[i - 1])
          return fail(COLD_ERR_INVALID_ARG, "bag offsets must be non-decreasing (group " + std::to_string(g) + ")");
    }
  }
  memset(&pl.bv, 0, sizeof(pl.bv));
  if (!pl.host) {
    for (int g : pl.needed) {
      pl.bv.g[g].ids = b->ids[g];
      pl.bv.g[g].offs = b->offs[g];
    }
  }
  return COLD_OK;
}

static cold_status check_err(cold_ctx* c, cudaStream_t st) {
  if (!(c->flags & COLD_VALIDATE_IDS)) return COLD_OK;
  int h = 0;
  CK(cudaMemcpyAsync(&h, c->d_err, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (h) return fail(COLD_ERR_ID_RANGE, "an id is outside its group's cardinality");
  return COLD_OK;
}

// stage the user CSR arrays of a host batch (small) and the ad offsets
static cold_status stage_user(cold_ctx* c, const cold_batch* b, CallPlan& pl, cudaStream_t st) {
  size_t bytes = (size_t)(pl.R + 1) * 4;
  for (int g : pl.needed)
    if (c->groups[g].side == COLD_USER) bytes += (size_t)(pl.R + 1) * 4 + (size_t)b->offs_host[g][pl.R] * 4 + 64;
  if (bytes > c->user_stage_bytes) {
    CK(cudaStreamSynchronize(st));
    if (c->d_user_stage) cudaFree(c->d_user_stage);
    c->d_user_stage = nullptr;
    if (cudaMalloc(&c->d_user_stage, bytes * 2) != cudaSuccess) { cudaGetLastError(); return fail(COLD_ERR_OOM, "staging"); }
    c->user_stage_bytes = bytes * 2;
  }
  uint8_t* p = (uint8_t*)c->d_user_stage;
  CK(cudaMemcpyAsync(c->d_adoff, b->ad_offsets_host, (size_t)(pl.R + 1) * 4, cudaMemcpyHostToDevice, st));
  for (int g : pl.needed) {
    if (c->groups[g].side != COLD_USER) continue;
    int32_t* o = (int32_t*)p;
    p += ((size_t)(pl.R + 1) * 4 + 15) / 16 * 16;
    int32_t* ids = (int32_t*)p;
    const int64_t nids = b->offs_host[g][pl.R];
    p += ((size_t)nids * 4 + 15) / 16 * 16;
    CK(cudaMemcpyAsync(o, b->offs_host[g], (size_t)(pl.R + 1) * 4, cudaMemcpyHostToDevice, st));
    if (nids) CK(cudaMemcpyAsync(ids, b->ids[g], (size_t)nids * 4, cudaMemcpyHostToDevice, st));
    pl.bv.g[g].ids = ids;
    pl.bv.g[g].offs = o;
  }
  return COLD_OK;
}

// bytes of ad-side inputs for ads [a0, a1) of a host batch
static size_t chunk_stage_bytes(cold_ctx* c, const cold_batch* b, const CallPlan& pl, int64_t a0, int64_t a1) {
  size_t bytes = 0;
  for (int g : pl.needed) {
    const cold_group& G = c->groups[g];
    if (G.side != COLD_AD) continue;
    if (!G.pooled) bytes += (size_t)(a1 - a0) * 4 + 16;
    else bytes += (size_t)(a1 - a0 + 1) * 4 + 16 + (size_t)(b->offs_host[g][a1] - b->offs_host[g][a0]) * 4 + 16;
  }
  return bytes;
}

// copy ad-side inputs of [a0, a1) into stage slot `s` on the copy stream; fills bv
static cold_status stage_chunk(cold_ctx* c, const cold_batch* b, const CallPlan& pl, int64_t a0, int64_t a1, int s,
                               BatchView& bv) {
  uint8_t* p = (uint8_t*)c->d_stage[s];
  for (int g : pl.needed) {
    const cold_group& G = c->groups[g];
    if (G.side != COLD_AD) continue;
    if (!G.pooled) {
      CK(cudaMemcpyAsync(p, b->ids[g] + a0, (size_t)(a1 - a0) * 4, cudaMemcpyHostToDevice, c->copy_stream));
      bv.g[g].ids = (const int32_t*)p;
      bv.g[g].id_shift = a0;
      p += ((size_t)(a1 - a0) * 4 + 15) / 16 * 16;
    } else {
      const int32_t* oh = b->offs_host[g];
      CK(cudaMemcpyAsync(p, oh + a0, (size_t)(a1 - a0 + 1) * 4, cudaMemcpyHostToDevice, c->copy_stream));
      bv.g[g].offs = (const int32_t*)p;
      bv.g[g].offs_shift = a0;
      bv.g[g].val_shift = oh[a0];
      p += ((size_t)(a1 - a0 + 1) * 4 + 15) / 16 * 16;
      const int64_t nid = oh[a1] - oh[a0];
      if (nid) CK(cudaMemcpyAsync(p, b->ids[g] + oh[a0], (size_t)nid * 4, cudaMemcpyHostToDevice, c->copy_stream));
      bv.g[g].ids = (const int32_t*)p;
      p += ((size_t)nid * 4 + 15) / 16 * 16;
    }
  }
  return COLD_OK;
}

enum { RUN_SCORE = 0, RUN_DEBUG = 1 };

struct DebugOut {
  float* pooled = nullptr;
  float* feat = nullptr;
};

static UserArgs make_user_args(cold_ctx* c, const CallPlan& pl, const int32_t* d_adoff, const DebugOut& dbg) {
  UserArgs ua;
  memset(&ua, 0, sizeof(ua));
  ua.groups = c->d_groups;
  ua.bv = pl.bv;
  ua.n_user = (int)c->sel_user.size();
  for (int j = 0; j < ua.n_user; j++) ua.user_g[j] = c->sel_user[j];
  ua.k = c->k;
  ua.se_w = c->d_se_w;
  ua.se_b = c->d_se_b;
  ua.linear_log = c->linear_log;
  ua.w1u_t = c->d_w1u_t;
  ua.b1 = c->d_b1;
  ua.H = c->widths[0];
  ua.u1 = c->d_u1;
  ua.xu = c->d_xu;
  ua.ad_offsets = d_adoff;
  ua.req_of_ad = c->d_req;
  ua.validate = (c->flags & COLD_VALIDATE_IDS) ? 1 : 0;
  ua.err = c->d_err;
  ua.dbg_pooled = dbg.pooled;
  ua.dbg_feat = dbg.feat;
  ua.n_sel = (int)c->sel.size();
  ua.d_in = c->d_in;
  ua.in_scale = c->d_in_scale;
  ua.in_shift = c->d_in_shift;
  ua.u1t = c->u1mma ? c->d_u1t : nullptr;
  ua.u1t_ld = c->u1t_ld;
  ua.u1_terms = c->u1_terms;
  ua.bf16 = c->precision == COLD_BF16 ? 1 : 0;
  ua.dense = c->dense_se ? 1 : 0;
  return ua;
}

// the SE weights of the launch's columns into its parameters (read through the constant bank: the
// per-thread global loads of w_g were a quarter of the gather's LSU instructions)
static void fill_se_params(const cold_ctx* c, GatherArgs& ga) {
  ga.sew_in_params = 0;
  if ((size_t)ga.n_ac * c->k > sizeof(ga.sew_c) / sizeof(float) || c->h_se_w.empty()) return;
  for (int j = 0; j < ga.n_ac; j++) {
    const int g = ga.ac_g[j];
    memcpy(&ga.sew_c[(size_t)j * c->k], &c->h_se_w[(size_t)g * c->k], sizeof(float) * c->k);
    ga.seb_c[j] = c->h_se_b[g];
  }
  ga.sew_in_params = 1;
}

static GatherArgs make_gather_args(cold_ctx* c, const BatchView& bv, int64_t a0, int64_t n, const DebugOut& dbg) {
  GatherArgs ga;
  memset(&ga, 0, sizeof(ga));
  ga.groups = c->d_groups;
  for (int g = 0; g < c->M; g++) ga.gp[g] = c->h_groups[g];
  ga.bv = bv;
  ga.n_ac = 0;
  for (int j = 0; j < (int)c->sel_ac.size(); j++) {   // one grid.y column per group, heaviest first
    ga.ac_g[ga.n_ac] = c->sel_ac[c->gather_order[j]];
    ga.order[ga.n_ac] = ga.n_ac;
    ga.n_ac++;
  }
  ga.k = c->k;
  ga.se_w = c->d_se_w;
  ga.se_b = c->d_se_b;
  ga.linear_log = c->linear_log;
  ga.req_of_ad = c->d_req;
  ga.a0 = a0;
  ga.n = n;
  ga.X = c->d_X;
  ga.ldx = c->d_ac_pad;
  ga.x_slab = c->x_slab ? 1 : 0;
  ga.x_rows = (int64_t)c->gspan * c->chunk;
  ga.validate = (c->flags & COLD_VALIDATE_IDS) ? 1 : 0;
  ga.err = c->d_err;
  ga.dbg_pooled = dbg.pooled;
  ga.dbg_feat = dbg.feat;
  ga.n_sel = (int)c->sel.size();
  ga.d_in = c->d_in;
  ga.in_scale = c->d_in_scale;
  ga.in_shift = c->d_in_shift;
  ga.ohot = (c->u1mma && !dbg.pooled && !dbg.feat) ? c->d_ohot : nullptr;
  ga.chunk = c->chunk;
  ga.nslot = U1_NSLOT;
  ga.bf16 = c->precision == COLD_BF16 ? 1 : 0;
  if (c->dense_se) {
    ga.E = c->d_E;
    ga.lde = c->d_in;
  }
  fill_se_params(c, ga);
  return ga;
}

// the network on one chunk: X (rows a0 .. a0+n) -> scores_out[0 .. n)
static void run_network(cold_ctx* c, int64_t a0, int64_t n, int xslot, float* scores_out, cudaStream_t st) {
  auto tmA_of = [&](int l) -> const CUtensorMap* { return l == 0 ? &c->tmAX[xslot] : &c->tmA[l]; };
  if (!c->tensor) {
    MlpF32Args m;
    memset(&m, 0, sizeof(m));
    m.X = (const float*)c->d_X + (size_t)xslot * c->chunk * c->d_ac_pad;
    m.ldx = c->d_ac_pad;
    m.d_ac = c->d_x;
    m.u1 = c->d_u1;
    m.ld_u1 = c->widths[0];
    m.req_of_ad = c->d_req;
    m.a0 = a0;
    m.n = n;
    m.L = c->L;
    int mw = std::max(1, c->d_x);
    for (int l = 0; l < c->L; l++) {
      m.wt[l] = c->d_wt[l];
      m.b[l] = c->d_b[l];
      m.width[l] = c->widths[l];
      mw = std::max(mw, c->widths[l]);
    }
    m.max_w = (mw + 3) / 4 * 4;   // float4 activation reads
    for (int l = 0; l < c->L - 1; l++) m.slope[l] = c->d_slope[l];
    m.scores = scores_out;
    c->mark_begin(st);
    launch_mlp_f32(m, st);
    c->mark_end(COLD_PROF_MLP_F32, st, c->layer_flop(0, c->L, n));
    return;
  }
  int n_gemm = c->L - 1 - c->n_tail;
  // the chain walks 256-row blocks per CTA pair: below ~2 blocks per pair (e.g. one 4,000-ad request)
  // the layer-by-layer kernels expose more parallelism per layer and have lower latency
  if (c->chain && n >= c->chain_min) {   // FC1..FC3 in one launch (kernels_chain.cu), then the FC4/FC5/head tail below
    ChainParams cp;
    memset(&cp, 0, sizeof(cp));
    cp.b2 = c->d_b[1];
    cp.b3 = c->d_b[2];
    cp.x_slab = c->x_slab ? 1 : 0;
    cp.s1 = c->d_slope[0];
    cp.s2 = c->d_slope[1];
    cp.s3 = c->d_slope[2];
    cp.u1 = c->d_u1;
    cp.ld_u1 = c->widths[0];
    cp.req_of_ad = c->d_req;
    cp.a0 = a0;
    cp.n1 = c->widths[0];
    cp.n2 = c->widths[1];
    cp.n3 = c->widths[2];
    cp.k1 = c->d_ac_pad;
    cp.h1 = c->d_H[0];
    cp.h2 = c->d_H[1];
#ifdef COLD_INSTRUMENT   // wait-cycle instrumentation build (tools/probes/chain_instr.py)
    if (!g_instr) {
      cudaMalloc(&g_instr, 8 * 8 * COLD_MAX_LAYERS);
      cudaMemset(g_instr, 0, 8 * 8 * COLD_MAX_LAYERS);
    }
    cp.instr = g_instr + 8 * 4;   // slots 32..39
#endif
    if (c->chain_tail) {
      cp.tail = 1;
      cp.n4 = c->widths[3];
      cp.n5 = c->widths[4];
      cp.b4 = c->d_b[3];
      cp.b5 = c->d_b[4];
      cp.head_w = c->d_head_w;
      cp.head_b = c->d_head_b;
      cp.head_n = c->widths[5];
      cp.h3 = c->d_H[2];
      cp.h4 = c->d_H[3];
      cp.scores = scores_out;
    }
    const CUtensorMap* tm[12] = {&c->tmAX[xslot], &c->tmB[0], &c->tmB[1], &c->tmB[2], &c->tmC[0], &c->tmC[1],
                                 &c->tmC[2], &c->tmOH[xslot], &c->tmU1T,
                                 c->chain_tail ? &c->tmW4h : &c->tmB[0], c->chain_tail ? &c->tmW5h : &c->tmB[0],
                                 c->chain_tail ? &c->tmC[3] : &c->tmB[0]};
    c->mark_begin(st);
    launch_chain(tm, (int)n, c->precision == COLD_BF16 ? 1 : 0, cp, c->num_sms, c->pdl && !c->prof, st);
    c->mark_end(COLD_PROF_CHAIN, st, c->layer_flop(0, c->chain_tail ? c->L : 3, n));
    n_gemm = 0;
    if (c->chain_tail) return;   // FC4 / FC5 / head done inside the chain
  }
#ifdef COLD_INSTRUMENT
  const bool instr_on = true;
  if (!g_instr) {
    cudaMalloc(&g_instr, 8 * 8 * COLD_MAX_LAYERS);
    cudaMemset(g_instr, 0, 8 * 8 * COLD_MAX_LAYERS);
  }
#else
  const bool instr_on = false;
#endif
  // small calls: FC1, FC2 as pair GEMMs, then FC3 -> FC4 -> FC5 -> head in the one-CTA tail kernel
  const bool lat3 = c->lat_tail3 && n_gemm == c->L - 1 - c->n_tail && n < c->chain_min;
  if (lat3) n_gemm = c->L - 4;
  for (int l = 0; l < n_gemm; l++) {
    EpiParams ep;
    memset(&ep, 0, sizeof(ep));
    ep.relu = 1;
    ep.slope = c->d_slope[l];
    ep.a_slab = (l == 0 && c->x_slab) ? 1 : 0;
    if (l == 0) {
      ep.u1 = c->d_u1;
      ep.ld_u1 = c->widths[0];
      ep.req_of_ad = c->d_req;
      ep.a0 = a0;
      ep.ad_offsets = c->cur_adoff;
    } else {
      ep.bias = c->d_b[l];
    }
    const bool head = (l == c->L - 2);
    if (head) {
      ep.head_w = c->d_head_w;
      ep.head_b = c->d_head_b;
      ep.head_n = c->widths[c->L - 1];
      ep.scores = scores_out;
    } else {
      ep.out = c->d_H[l];
      ep.ldo = c->widths[l];
    }
    const int K = (l == 0) ? c->d_ac_pad : c->widths[l - 1];
    ep.instr = instr_on ? g_instr + 8 * l : nullptr;
    c->mark_begin(st);
    const bool q128 = lat3 && l == 1 && c->lat_fc2_128 && c->pair[l];
    if (c->pair[l])
      launch_gemm_pair(tmA_of(l), q128 ? &c->tmW2q : &c->tmB[l], &c->tmC[l], (int)n, c->widths[l], K, q128 ? 128 : c->bn[l],
                       c->precision == COLD_BF16 ? 1 : 0, ep, c->num_sms, c->pdl && !c->prof, st,
                       (l == 0 && c->u1mma) ? &c->tmOH[xslot] : nullptr, (l == 0 && c->u1mma) ? &c->tmU1T : nullptr,
                       c->pair_res[l]);
    else
      launch_gemm(tmA_of(l), &c->tmB[l], &c->tmC[l], (int)n, c->widths[l], K, c->bn[l],
                  c->precision == COLD_BF16 ? 1 : 0, c->cs[l], c->resb[l], ep, c->num_sms, c->pdl && !c->prof, st);
    c->mark_end(COLD_PROF_FC + l, st, c->layer_flop(l, head ? c->L : l + 1, n));
  }
  if (lat3) {
    const int l3 = c->L - 4;
    TailParams tp;
    memset(&tp, 0, sizeof(tp));
    tp.b3 = c->d_b[l3];
    tp.b4 = c->d_b[l3 + 1];
    tp.b5 = c->d_b[l3 + 2];
    tp.head_w = c->d_head_w;
    tp.head_b = c->d_head_b;
    tp.head_n = c->widths[c->L - 1];
    tp.scores = scores_out;
    c->mark_begin(st);
    launch_tail(tmA_of(l3), &c->tmW3full, &c->tmB[l3 + 1], &c->tmB[l3 + 2], (int)n, c->widths[l3 - 1],
                c->precision == COLD_BF16 ? 1 : 0, tp, c->num_sms, c->pdl && !c->prof, st);
    c->mark_end(COLD_PROF_TAIL, st, c->layer_flop(l3, c->L, n));
    return;
  }
  if (c->tail_mode == 2) {
    const int l4 = c->L - 3;
    TailParams tp;
    memset(&tp, 0, sizeof(tp));
    tp.b4 = c->d_b[l4];
    tp.b5 = c->d_b[l4 + 1];
    tp.head_w = c->d_head_w;
    tp.head_b = c->d_head_b;
    tp.head_n = c->widths[c->L - 1];
    tp.scores = scores_out;
    tp.s4 = c->d_slope[l4];
    tp.s5 = c->d_slope[l4 + 1];
    tp.reverse = 1;   // last tile first: the most recently written H3 rows are the ones still in L2
    c->mark_begin(st);
    launch_tail45(tmA_of(l4), &c->tmB[l4], &c->tmB[l4 + 1], (int)n, c->precision == COLD_BF16 ? 1 : 0, tp,
                  c->num_sms, c->pdl && !c->prof, st);
    c->mark_end(COLD_PROF_TAIL, st, c->layer_flop(l4, c->L, n));
  }
  if (c->tail_mode == 1) {
    const int l3 = c->L - 4;
    TailParams tp;
    memset(&tp, 0, sizeof(tp));
    tp.b3 = c->d_b[l3];
    tp.b4 = c->d_b[l3 + 1];
    tp.b5 = c->d_b[l3 + 2];
    tp.head_w = c->d_head_w;
    tp.head_b = c->d_head_b;
    tp.head_n = c->widths[c->L - 1];
    tp.scores = scores_out;
    const int K3 = (l3 == 0) ? c->d_ac_pad : c->widths[l3 - 1];
    c->mark_begin(st);
    launch_tail(tmA_of(l3), &c->tmB[l3], &c->tmB[l3 + 1], &c->tmB[l3 + 2], (int)n, K3,
                c->precision == COLD_BF16 ? 1 : 0, tp, c->num_sms, c->pdl && !c->prof, st);
    c->mark_end(COLD_PROF_TAIL, st, c->layer_flop(l3, c->L, n));
  }
}

static cold_status run(cold_ctx* c, const cold_batch* b, float* scores, cudaStream_t st, int mode, const DebugOut& dbg) {
  if (!c) return fail(COLD_ERR_INVALID_ARG, "null ctx");
  if (!c->loaded) return fail(COLD_ERR_NOT_LOADED, "cold_load_params has not been called");
  CallPlan pl;
  cold_status s = plan_batch(c, b, pl);
  if (s) return s;
  if (mode == RUN_SCORE && !scores) return fail(COLD_ERR_INVALID_ARG, "scores is NULL");
  CK(cudaSetDevice(c->device));
  cudaGetLastError();   // start clean: only report errors of this call's launches
  if (c->flags & COLD_VALIDATE_IDS) CK(cudaMemsetAsync(c->d_err, 0, 4, st));
  const int32_t* d_adoff = b->ad_offsets;
  if (pl.host) {
    s = stage_user(c, b, pl, st);
    if (s) return s;
    d_adoff = c->d_adoff;
  }
  const bool scores_dev = mode == RUN_SCORE && is_device_ptr(scores);
  c->cur_adoff = d_adoff;
  UserArgs ua = make_user_args(c, pl, d_adoff, dbg);
  const double user_flop = c->dense_se ? 0.0 : 2.0 * c->d_u * c->widths[0] * (double)pl.R;
  // Latency path (a few requests, scoring): the user side (pooling, u1 GEMV, ad -> request map) does not
  // feed the gather, which finds an ad's request by searching ad_offsets, so the two run concurrently
  // (fork onto the side stream, join before the FC stack). COLD_K_SERIAL_USER serialises them.
  const bool fork = !(c->kflags & COLD_K_SERIAL_USER) && mode == RUN_SCORE && pl.R <= 4;
  if (fork) {
    CK(cudaEventRecord(c->ev_fork, st));
    CK(cudaStreamWaitEvent(c->side_stream, c->ev_fork, 0));
    c->mark_begin(c->side_stream);
    launch_user(ua, pl.R, c->precision, c->side_stream);
    c->mark_end(COLD_PROF_USER, c->side_stream, user_flop);
    CK(cudaEventRecord(c->ev_user, c->side_stream));
  } else {
    c->mark_begin(st);
    launch_user(ua, pl.R, c->precision, st);
    c->mark_end(COLD_PROF_USER, st, user_flop);
  }
  CK(cudaGetLastError());
  bool joined = !fork;
  const int64_t chunk = c->chunk;
  const int64_t span = chunk * c->gspan;            // ads per column-wise gather pass
  const int64_t nspans = (pl.N + span - 1) / span;
  if (pl.host) {
    size_t need = 0;
    for (int64_t si = 0; si < nspans; si++)
      need = std::max(need, chunk_stage_bytes(c, b, pl, si * span, std::min(pl.N, (si + 1) * span)));
    if (need > c->stage_bytes) {
      CK(cudaStreamSynchronize(st));
      CK(cudaStreamSynchronize(c->copy_stream));
      for (int i = 0; i < 2; i++) {
        if (c->d_stage[i]) cudaFree(c->d_stage[i]);
        c->d_stage[i] = nullptr;
        if (cudaMalloc(&c->d_stage[i], need) != cudaSuccess) { cudaGetLastError(); return fail(COLD_ERR_OOM, "staging"); }
      }
      c->stage_bytes = need;
    }
    // the copy stream must not run ahead of earlier work on `st` that still reads the slots
    CK(cudaEventRecord(c->ev_consumed[0], st));
    CK(cudaStreamWaitEvent(c->copy_stream, c->ev_consumed[0], 0));
    CK(cudaEventRecord(c->ev_consumed[1], st));
  }
  int64_t ci = 0;   // running chunk counter (score staging slots)
  for (int64_t si = 0; si < nspans; si++) {
    const int64_t s0 = si * span, s1 = std::min(pl.N, s0 + span);
    const int slot = (int)(si & 1);
    BatchView bv = pl.bv;
    if (pl.host) {
      if (si >= 2) CK(cudaStreamWaitEvent(c->copy_stream, c->ev_consumed[slot], 0));
      s = stage_chunk(c, b, pl, s0, s1, slot, bv);
      if (s) return s;
      CK(cudaEventRecord(c->ev_copied[slot], c->copy_stream));
      CK(cudaStreamWaitEvent(st, c->ev_copied[slot], 0));
    }
    GatherArgs ga = make_gather_args(c, bv, s0, s1 - s0, dbg);
    if (fork) {
      ga.search_req = 1;
      ga.adoff = d_adoff;
      ga.R = pl.R;
    }
    if (c->gather_ring != -1 && c->tensor && c->k * c->elem() == 32 && !dbg.pooled && !dbg.feat &&
        s1 - s0 >= 148 * 128 * 4) {
      // cross-bag columns (user bag x single ad id) in the bag-only build, then the rest
      GatherArgs gb = ga, gr = ga;
      gb.n_ac = gr.n_ac = 0;
      gb.ohot = nullptr;
      gb.ring = c->gather_ring > 0 ? c->gather_ring : -1;
      for (int j = 0; j < ga.n_ac; j++) {
        const int g = ga.ac_g[ga.order[j]];
        const cold_group& G = c->groups[g];
        const bool bagx = G.side == COLD_CROSS && c->groups[G.user_ref].pooled && !c->groups[G.ad_ref].pooled;
        GatherArgs& d = bagx ? gb : gr;
        d.ac_g[d.n_ac] = g;
        d.order[d.n_ac] = d.n_ac;
        d.n_ac++;
      }
      fill_se_params(c, gb);
      fill_se_params(c, gr);
      c->mark_begin(st);
      if (gb.n_ac) launch_gather(gb, c->precision, st);
      launch_gather(gr, c->precision, st);
      c->mark_end(COLD_PROF_GATHER, st);
    } else {
      c->mark_begin(st);
      launch_gather(ga, c->precision, st);
      c->mark_end(COLD_PROF_GATHER, st);
    }
    if (!joined) {   // dense SE and the FC stack read x_u / u1 and req_of_ad (or the side-stream gather's X)
      CK(cudaStreamWaitEvent(st, c->ev_user, 0));
      joined = true;
    }
    if (c->dense_se) {   // dense SE gate over the span (the Doc B reading of P:229-234, AMB-1)
      SeDenseArgs sa;
      memset(&sa, 0, sizeof(sa));
      sa.E = c->d_E;
      sa.lde = c->d_in;
      sa.xu = c->d_xu;
      sa.ldu = c->d_u;
      sa.n_user = (int)c->sel_user.size();
      for (int j = 0; j < sa.n_user; j++) sa.user_pos[j] = c->sel_pos[c->sel_user[j]];
      sa.req_of_ad = c->d_req;
      sa.a0 = s0;
      sa.n = s1 - s0;
      sa.wdt = c->d_sewd_t;
      sa.bd = c->d_sebd;
      sa.n_sel = (int)c->sel.size();
      sa.k = c->k;
      sa.d_in = c->d_in;
      sa.in_scale = c->d_in_scale;
      sa.in_shift = c->d_in_shift;
      sa.X = c->d_X;
      sa.ldx = c->d_ac_pad;
      sa.dbg_feat = dbg.feat;
      c->mark_begin(st);
      launch_se_dense(sa, c->precision, st);
      c->mark_end(COLD_PROF_SE_DENSE, st);
    }
    if (pl.host) CK(cudaEventRecord(c->ev_consumed[slot], st));
    if (mode == RUN_SCORE) {
      const int64_t nch = (s1 - s0 + chunk - 1) / chunk;
      for (int64_t k = 0; k < nch; k++, ci++) {
        const int64_t a0 = s0 + k * chunk;
        const int64_t n = std::min(s1, a0 + chunk) - a0;
        const int oslot = (int)(ci & 1);
        float* out = scores_dev ? scores + a0 : c->d_scores_stage + (int64_t)oslot * chunk;
        if (!scores_dev && ci >= 2) CK(cudaStreamWaitEvent(st, c->ev_drained[oslot], 0));
        run_network(c, a0, n, (int)((a0 - s0) / chunk), out, st);
        if (!scores_dev) {
          CK(cudaEventRecord(c->ev_scored[oslot], st));
          CK(cudaStreamWaitEvent(c->copy_stream, c->ev_scored[oslot], 0));
          CK(cudaMemcpyAsync(scores + a0, out, (size_t)n * 4, cudaMemcpyDeviceToHost, c->copy_stream));
          CK(cudaEventRecord(c->ev_drained[oslot], c->copy_stream));
        }
      }
    }
    CK(cudaGetLastError());
  }
  if (pl.host || !scores_dev) {
    // join the copy stream back into the caller's stream
    CK(cudaEventRecord(c->ev_drained[0], c->copy_stream));
    CK(cudaStreamWaitEvent(st, c->ev_drained[0], 0));
  }
  return check_err(c, st);
}

extern "C" cold_status cold_score_batch(cold_ctx* c, const cold_batch* b, float* scores, void* stream) {
  return run(c, b, scores, (cudaStream_t)stream, RUN_SCORE, DebugOut());
}

extern "C" cold_status cold_score_request(cold_ctx* c, const cold_batch* one, float* scores, void* stream) {
  if (!one || one->num_requests != 1) return fail(COLD_ERR_INVALID_ARG, "cold_score_request takes exactly one request");
  return run(c, one, scores, (cudaStream_t)stream, RUN_SCORE, DebugOut());
}

extern "C" cold_status cold_debug_pooled(cold_ctx* c, const cold_batch* b, float* out, void* stream) {
  if (!out || !is_device_ptr(out)) return fail(COLD_ERR_INVALID_ARG, "out must be device memory");
  DebugOut d;
  d.pooled = out;
  return run(c, b, nullptr, (cudaStream_t)stream, RUN_DEBUG, d);
}

extern "C" cold_status cold_debug_features(cold_ctx* c, const cold_batch* b, float* out, void* stream) {
  if (!out || !is_device_ptr(out)) return fail(COLD_ERR_INVALID_ARG, "out must be device memory");
  DebugOut d;
  d.feat = out;
  return run(c, b, nullptr, (cudaStream_t)stream, RUN_DEBUG, d);
}

extern "C" cold_status cold_debug_rows(cold_ctx* c, const cold_batch* b, int32_t group, int64_t* rows_out,
                                       int32_t max_rows, void* stream) {
  if (!c) return fail(COLD_ERR_INVALID_ARG, "null ctx");
  if (!c->loaded) return fail(COLD_ERR_NOT_LOADED, "cold_load_params has not been called");
  if (group < 0 || group >= c->M || max_rows < 1 || !rows_out || !is_device_ptr(rows_out))
    return fail(COLD_ERR_INVALID_ARG, "bad group / max_rows / rows_out");
  CallPlan pl;
  cold_status s = plan_batch(c, b, pl);
  if (s) return s;
  if (pl.host) return fail(COLD_ERR_INVALID_ARG, "cold_debug_rows takes a device batch");
  const cold_group& G = c->groups[group];
  // the group's own ids (and for CROSS its refs) must be present
  std::vector<int> gs = {group};
  if (G.side == COLD_CROSS) gs = {G.user_ref, G.ad_ref};
  for (int g : gs) {
    if (!b->ids[g]) return fail(COLD_ERR_INVALID_ARG, "ids missing");
    pl.bv.g[g].ids = b->ids[g];
    pl.bv.g[g].offs = b->offs[g];
  }
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaSetDevice(c->device));
  cudaGetLastError();
  UserArgs ua = make_user_args(c, pl, b->ad_offsets, DebugOut());
  launch_user(ua, pl.R, c->precision, st);
  RowsArgs ra;
  ra.groups = c->d_groups;
  ra.bv = pl.bv;
  ra.g = group;
  ra.req_of_ad = c->d_req;
  ra.n = pl.N;
  ra.rows = rows_out;
  ra.max_rows = max_rows;
  launch_rows(ra, st);
  CK(cudaGetLastError());
  return COLD_OK;
}

// ---------------------------------------------------------------------------------------------
// feature-group selection statistics
extern "C" cold_status cold_se_stats(cold_ctx* c, const cold_batch* b, double* mean_s_out, void* stream) {
  if (c && c->dense_se) return fail(COLD_ERR_UNSUPPORTED, "cold_se_stats: per-group SE only (se_mode dense)");
  if (!c || !mean_s_out) return fail(COLD_ERR_INVALID_ARG, "null ctx / output");
  if (!c->loaded) return fail(COLD_ERR_NOT_LOADED, "cold_load_params has not been called");
  CallPlan pl;
  cold_status s = plan_batch(c, b, pl, true);
  if (s) return s;
  if (pl.host) return fail(COLD_ERR_INVALID_ARG, "cold_se_stats takes a device batch");
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaSetDevice(c->device));
  cudaGetLastError();
  double* d_stats = nullptr;
  if (cudaMallocAsync((void**)&d_stats, sizeof(double) * c->M, st) != cudaSuccess) {
    cudaGetLastError();
    return fail(COLD_ERR_OOM, "stats buffer");
  }
  CK(cudaMemsetAsync(d_stats, 0, sizeof(double) * c->M, st));
  if (c->flags & COLD_VALIDATE_IDS) CK(cudaMemsetAsync(c->d_err, 0, 4, st));
  // user side: every USER group of the schema, s_g weighted by the request's ad count
  UserArgs ua = make_user_args(c, pl, b->ad_offsets, DebugOut());
  ua.n_user = 0;
  for (int g = 0; g < c->M; g++)
    if (c->groups[g].side == COLD_USER) ua.user_g[ua.n_user++] = g;
  ua.stats = d_stats;
  launch_user(ua, pl.R, c->precision, st);   // also builds the ad -> request map
  // ad + cross side: every non-user group, column-wise over all ads of the batch
  GatherArgs ga = make_gather_args(c, pl.bv, 0, pl.N, DebugOut());
  ga.n_ac = 0;
  for (int pass = 0; pass < 3; pass++)
    for (int g = 0; g < c->M; g++) {
      const cold_group& G = c->groups[g];
      if (G.side == COLD_USER) continue;
      const int cls = G.side == COLD_CROSS ? 0 : (G.pooled ? 1 : 2);
      if (cls == pass) ga.ac_g[ga.n_ac++] = g;
    }
  for (int j = 0; j < ga.n_ac; j++) ga.order[j] = j;
  fill_se_params(c, ga);
  ga.X = nullptr;
  ga.ohot = nullptr;
  ga.stats = d_stats;
  launch_gather(ga, c->precision, st);
  CK(cudaGetLastError());
  std::vector<double> h(c->M);
  CK(cudaMemcpyAsync(h.data(), d_stats, sizeof(double) * c->M, cudaMemcpyDeviceToHost, st));
  CK(cudaFreeAsync(d_stats, st));
  CK(cudaStreamSynchronize(st));
  s = check_err(c, st);
  if (s) return s;
  for (int g = 0; g < c->M; g++) mean_s_out[g] = h[g] / (double)pl.N;
  return COLD_OK;
}

extern "C" cold_status cold_select_groups(const double* mean_s, int32_t M, int32_t K, int32_t* selected_out) {
  if (!mean_s || !selected_out) return fail(COLD_ERR_INVALID_ARG, "null pointer");
  if (M < 1 || K < 1 || K > M) return fail(COLD_ERR_K_RANGE, "K must be in [1, M]");
  std::vector<int> order(M);
  for (int g = 0; g < M; g++) order[g] = g;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return mean_s[x] > mean_s[y]; });
  std::vector<int> top(order.begin(), order.begin() + K);
  std::sort(top.begin(), top.end());
  for (int i = 0; i < K; i++) selected_out[i] = top[i];
  return COLD_OK;
}

// ---------------------------------------------------------------------------------------------
extern "C" cold_status cold_topk(cold_ctx* c, const float* scores, const int32_t* ad_offsets,
                                 const int32_t* ad_offsets_host, int32_t R, int32_t K, const float* bids,
                                 int32_t* idx_out, float* key_out, void* stream) {
  if (!c) return fail(COLD_ERR_INVALID_ARG, "null ctx");
  if (!scores || !ad_offsets || !ad_offsets_host || !idx_out || !key_out) return fail(COLD_ERR_INVALID_ARG, "null pointer");
  if (R < 1 || R > c->max_req) return fail(COLD_ERR_INVALID_ARG, "R out of range");
  if (ad_offsets_host[0] != 0) return fail(COLD_ERR_INVALID_ARG, "ad_offsets[0] must be 0");
  int32_t min_n = INT32_MAX;
  for (int r = 0; r < R; r++) {
    int32_t n = ad_offsets_host[r + 1] - ad_offsets_host[r];
    if (n < 1) return fail(COLD_ERR_INVALID_ARG, "every request needs >= 1 ad");
    min_n = std::min(min_n, n);
  }
  if (K < 1 || K > min_n) return fail(COLD_ERR_K_RANGE, "K must be in [1, min ads per request]");
  if (K > 4096) return fail(COLD_ERR_UNSUPPORTED, "K > 4096");
  const int64_t N = ad_offsets_host[R];
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaSetDevice(c->device));
  cudaGetLastError();
  const bool s_dev = is_device_ptr(scores), o_dev = is_device_ptr(ad_offsets);
  const bool b_dev = !bids || is_device_ptr(bids);
  const bool out_dev = is_device_ptr(idx_out) && is_device_ptr(key_out);
  size_t in_need = (s_dev ? 0 : (size_t)N * 4) + (b_dev ? 0 : (size_t)N * 4) + (o_dev ? 0 : (size_t)(R + 1) * 4) + 64;
  size_t out_need = out_dev ? 16 : (size_t)R * K * 8 + 64;
  if (in_need > c->topk_in_bytes) {
    CK(cudaStreamSynchronize(st));
    if (c->d_topk_in) cudaFree(c->d_topk_in);
    c->d_topk_in = nullptr;
    if (cudaMalloc((void**)&c->d_topk_in, in_need) != cudaSuccess) { cudaGetLastError(); return fail(COLD_ERR_OOM, "topk staging"); }
    c->topk_in_bytes = in_need;
  }
  if (out_need > c->topk_out_bytes) {
    CK(cudaStreamSynchronize(st));
    if (c->d_topk_out) cudaFree(c->d_topk_out);
    c->d_topk_out = nullptr;
    if (cudaMalloc(&c->d_topk_out, out_need) != cudaSuccess) { cudaGetLastError(); return fail(COLD_ERR_OOM, "topk staging"); }
    c->topk_out_bytes = out_need;
  }
  uint8_t* p = (uint8_t*)c->d_topk_in;
  TopkArgs ta;
  ta.scores = scores;
  ta.bids = bids;
  ta.ad_offsets = ad_offsets;
  if (!s_dev) {
    CK(cudaMemcpyAsync(p, scores, (size_t)N * 4, cudaMemcpyHostToDevice, st));
    ta.scores = (const float*)p;
    p += ((size_t)N * 4 + 15) / 16 * 16;
  }
  if (!b_dev) {
    CK(cudaMemcpyAsync(p, bids, (size_t)N * 4, cudaMemcpyHostToDevice, st));
    ta.bids = (const float*)p;
    p += ((size_t)N * 4 + 15) / 16 * 16;
  }
  if (!o_dev) {
    CK(cudaMemcpyAsync(p, ad_offsets_host, (size_t)(R + 1) * 4, cudaMemcpyHostToDevice, st));
    ta.ad_offsets = (const int32_t*)p;
  }
  ta.R = R;
  ta.K = K;
  ta.G = 0;
  ta.Kl = 0;
  ta.cand_idx = nullptr;
  ta.max_n = 0;
  for (int r = 0; r < R; r++) ta.max_n = std::max(ta.max_n, ad_offsets_host[r + 1] - ad_offsets_host[r]);
  ta.idx = out_dev ? idx_out : (int32_t*)c->d_topk_out;
  ta.key = out_dev ? key_out : (float*)((uint8_t*)c->d_topk_out + (size_t)R * K * 4);
  c->mark_begin(st);
  launch_topk(ta, st);
  c->mark_end(COLD_PROF_TOPK, st);
  CK(cudaGetLastError());
  if (!out_dev) {
    CK(cudaMemcpyAsync(idx_out, ta.idx, (size_t)R * K * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(key_out, ta.key, (size_t)R * K * 4, cudaMemcpyDeviceToHost, st));
  }
  return COLD_OK;
}

// F1: merge of per-rank top-K lists when one request's ads are split across G GPUs
extern "C" cold_status cold_merge_topk(cold_ctx* c, const float* cand_key, const int32_t* cand_idx, int32_t G,
                                       int32_t R, int32_t Kl, const int32_t* ad_offsets,
                                       const int32_t* ad_offsets_host, int32_t K, int32_t* idx_out, float* key_out,
                                       void* stream) {
  if (!c) return fail(COLD_ERR_INVALID_ARG, "null ctx");
  if (!cand_key || !cand_idx || !ad_offsets || !ad_offsets_host || !idx_out || !key_out)
    return fail(COLD_ERR_INVALID_ARG, "null pointer");
  if (G < 1 || R < 1 || Kl < 1) return fail(COLD_ERR_INVALID_ARG, "G, R, Kl must be >= 1");
  if ((int64_t)G * Kl > (1 << 30)) return fail(COLD_ERR_INVALID_ARG, "too many candidates");
  if (K < 1 || K > Kl) return fail(COLD_ERR_K_RANGE, "K must be in [1, Kl]");
  if (K > 4096) return fail(COLD_ERR_UNSUPPORTED, "K > 4096");
  if (ad_offsets_host[0] != 0) return fail(COLD_ERR_INVALID_ARG, "ad_offsets[0] must be 0");
  for (int r = 0; r < R; r++) {
    const int64_t n = (int64_t)ad_offsets_host[r + 1] - ad_offsets_host[r];
    for (int g = 0; g < G; g++) {   // every slice must have supplied Kl real candidates
      const int64_t sl = (int64_t)(g + 1) * n / G - (int64_t)g * n / G;
      if (sl < Kl) return fail(COLD_ERR_K_RANGE, "a rank's slice of a request has fewer than Kl ads");
    }
  }
  for (const void* p : {(const void*)cand_key, (const void*)cand_idx, (const void*)ad_offsets, (const void*)idx_out,
                        (const void*)key_out})
    if (!is_device_ptr(p)) return fail(COLD_ERR_INVALID_ARG, "cold_merge_topk takes device buffers");
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaSetDevice(c->device));
  cudaGetLastError();
  TopkArgs ta;
  memset(&ta, 0, sizeof(ta));
  ta.scores = cand_key;
  ta.ad_offsets = ad_offsets;
  ta.R = R;
  ta.K = K;
  ta.G = G;
  ta.max_n = G * Kl;
  ta.Kl = Kl;
  ta.cand_idx = cand_idx;
  ta.idx = idx_out;
  ta.key = key_out;
  c->mark_begin(st);
  launch_topk(ta, st);
  c->mark_end(COLD_PROF_TOPK, st);
  CK(cudaGetLastError());
  return COLD_OK;
}

// ---------------------------------------------------------------------------------------------
// F4: the vector-product based pre-ranking model, precomputed towers
extern "C" cold_status cold_vps_score(const void* ad_vecs, int32_t vec_dtype, int64_t num_vecs, int32_t d,
                                      const float* user_vecs, const int32_t* ad_ids, const int32_t* ad_offsets,
                                      const int32_t* ad_offsets_host, int32_t R, float* scores, void* stream) {
  if (!ad_vecs || !user_vecs || !ad_ids || !ad_offsets || !ad_offsets_host || !scores)
    return fail(COLD_ERR_INVALID_ARG, "null pointer");
  if (vec_dtype < COLD_FP32 || vec_dtype > COLD_BF16) return fail(COLD_ERR_INVALID_ARG, "bad vec_dtype");
  if (d != 16 && d != 32 && d != 64 && d != 128 && d != 256) return fail(COLD_ERR_UNSUPPORTED, "d must be 16..256, pow2");
  if (num_vecs < 1 || R < 1) return fail(COLD_ERR_INVALID_ARG, "num_vecs and R must be >= 1");
  if (ad_offsets_host[0] != 0) return fail(COLD_ERR_INVALID_ARG, "ad_offsets[0] must be 0");
  int max_n = 0;
  for (int r = 0; r < R; r++) {
    const int n = ad_offsets_host[r + 1] - ad_offsets_host[r];
    if (n < 1) return fail(COLD_ERR_INVALID_ARG, "every request needs >= 1 ad");
    max_n = std::max(max_n, n);
  }
  for (const void* p : {ad_vecs, (const void*)user_vecs, (const void*)ad_ids, (const void*)ad_offsets, (const void*)scores})
    if (!is_device_ptr(p)) return fail(COLD_ERR_INVALID_ARG, "cold_vps_score takes device buffers");
  if ((reinterpret_cast<uintptr_t>(ad_vecs) & 31) != 0) return fail(COLD_ERR_INVALID_ARG, "ad_vecs must be 32 B aligned");
  VpsArgs a;
  a.ad_vecs = ad_vecs;
  a.num_vecs = num_vecs;
  a.d = d;
  a.user_vecs = user_vecs;
  a.ad_ids = ad_ids;
  a.ad_offsets = ad_offsets;
  a.R = R;
  a.scores = scores;
  cudaGetLastError();
  CK(launch_vps(a, vec_dtype, max_n, (cudaStream_t)stream));
  return COLD_OK;
}

// debug: read (and reset) the GEMM wait-cycle counters recorded when COLD_INSTR is set.
// out[8 * layer + i]: 0 producer empty-wait, 1 MMA full-wait, 2 MMA tmem-empty-wait, 3 MMA resident-B
// wait, 4 epilogue tmem-full-wait (per warp), 5 epilogue u1 wait, 6 epilogue warps, 7 producer total.
extern "C" int cold_debug_instr(unsigned long long* out, int n) {
  if (!g_instr) return 0;
  cudaDeviceSynchronize();
  cudaMemcpy(out, g_instr, sizeof(unsigned long long) * (size_t)n, cudaMemcpyDeviceToHost);
  cudaMemset(g_instr, 0, sizeof(unsigned long long) * 8 * COLD_MAX_LAYERS);
  return 1;
}

extern "C" cold_status cold_profile(cold_ctx* c, int32_t enable) {
  if (!c) return fail(COLD_ERR_INVALID_ARG, "null ctx");
  CK(cudaSetDevice(c->device));
  if (enable) {
    c->flush_profile();
    for (int i = 0; i < COLD_PROF_KINDS; i++) { c->prof_ms[i] = 0; c->prof_n[i] = 0; c->prof_flop[i] = 0; }
  }
  c->prof = enable != 0;
  return COLD_OK;
}

extern "C" cold_status cold_profile_read(cold_ctx* c, double* total_ms, int64_t* launches, double* flop) {
  if (!c || !total_ms || !launches) return fail(COLD_ERR_INVALID_ARG, "null");
  CK(cudaSetDevice(c->device));
  c->flush_profile();
  for (int i = 0; i < COLD_PROF_KINDS; i++) {
    total_ms[i] = c->prof_ms[i];
    launches[i] = c->prof_n[i];
    if (flop) flop[i] = c->prof_flop[i];
  }
  return COLD_OK;
}

extern "C" void cold_ctx_describe(const cold_ctx* c, int* num_groups, const cold_group** groups, int* max_requests,
                                  int64_t* max_ads, int* device) {
  *num_groups = c->M;
  *groups = c->groups.data();
  *max_requests = c->max_req;
  *max_ads = c->max_ads;
  *device = c->device;
}

extern "C" cold_status cold_get_info(const cold_ctx* c, cold_info* out) {
  if (!c || !out) return fail(COLD_ERR_INVALID_ARG, "null");
  out->version = c->version;
  out->d_in = c->d_in;
  out->d_user = c->dense_se ? 0 : c->d_u;   // hoisted user part (none under dense SE)
  out->d_ad = c->d_x;
  out->chunk_ads = c->chunk;
  out->kernels_per_chunk = 1 + (c->tensor ? (c->L - 1 - c->n_tail + (c->n_tail ? 1 : 0)) : 1);
  out->kernels_per_call = 1;
  out->tensor_core = c->tensor ? 1 : 0;
  int64_t b = c->device_bytes;
  for (int g = 0; g < c->M && g < (int)c->d_tables.size(); g++) b += c->groups[g].cardinality * c->k * c->elem();
  out->device_bytes = b;
  out->compressed_activations = 0;   // (reserved: the compressible-memory variant measured neutral, removed)
  out->gather_span_chunks = c->gspan;
  return COLD_OK;
}
