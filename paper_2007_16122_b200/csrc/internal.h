// internal.h — launchers shared between the host runtime (cold_api.cu) and the kernel files.
#pragma once
#include <atomic>
#include <cuda.h>
#include "common.cuh"


namespace cold {

// cudaFuncSetAttribute (dynamic shared-memory opt-in, cluster sizes) applies per device context, and a
// process may hold contexts on several GPUs (cold_config.device): remember the opt-in per device ordinal.
struct DevOnce {
  std::atomic<unsigned long long> bits{0};
  // true the first time it is called on the current device
  bool first() {
    int d = 0;
    cudaGetDevice(&d);
    const unsigned long long bit = 1ull << (d & 63);
    return (bits.fetch_or(bit) & bit) == 0;
  }
};


struct UserArgs {
  const DevGroup* groups;
  BatchView bv;
  int n_user;                      // selected USER groups
  int user_g[COLD_MAX_GROUPS];     // their schema indices
  int k;
  const float* se_w;               // [M][k]
  const float* se_b;               // [M]
  int linear_log;
  const float* w1u_t;              // [D_u][H] fp32 (W1 user columns, transposed)
  const float* b1;                 // [H]
  int H;                           // FC1 width
  int part_off;                    // set by launch_user: shared-memory float offset of the [4][H] partial sums
  float* u1;                       // [R][H] out: b1 + W1_u x_u
  float* xu;                       // [R][D_u] out: x_u
  const int32_t* ad_offsets;       // [R+1] device
  int32_t* req_of_ad;              // [N] out
  int validate;
  int* err;
  // debug (nullable): user-group columns broadcast to every ad of the request
  float* dbg_pooled;               // [N][n_sel][k]
  float* dbg_feat;                 // [N][D_in]
  int n_sel, d_in;
  const float* in_scale;           // input normalisation [D_in] (nullable; cold_params.in_scale)
  const float* in_shift;
  double* stats;                   // SE statistics mode (cold_se_stats): [M] += s_g * ads of the request;
                                   // x_u / u1 are not written
  uint16_t* u1t;                   // FC1 u1 operand (nullable): [u1_terms * H][u1t_ld] f16/bf16 bits, the
                                   // 2 (f16) or 3 (bf16) RNE terms of u1[r][o] at [t * H + o][r]
  int u1t_ld, u1_terms, bf16;
  int dense;                       // dense SE (COLD_SE_DENSE): xu gets the pre-SE linear_log'ed ê_u, u1 = b1
};

struct GatherArgs {
  const DevGroup* groups;
  BatchView bv;
  int n_ac;                        // selected AD + CROSS groups
  int ac_g[COLD_MAX_GROUPS];
  int order[COLD_MAX_GROUPS];      // blockIdx.y -> index into ac_g, heaviest group first
  int k;
  const float* se_w;
  const float* se_b;
  int linear_log;
  const int32_t* req_of_ad;        // call-global
  int64_t a0;                      // first ad of the chunk (call-global index)
  int64_t n;                       // ads in the chunk
  void* X;                         // [n][ldx] storage dtype (chunk-local rows)
  int ldx;
  int validate;
  int* err;
  float* dbg_pooled;               // [N][n_sel][k] (call-global rows)
  float* dbg_feat;                 // [N][D_in]
  int n_sel, d_in;
  const float* in_scale;           // input normalisation [D_in] (nullable)
  const float* in_shift;
  double* stats;                   // SE statistics mode: [M] += s_g per ad; X is not written
  uint16_t* ohot;                  // FC1 u1 operand (nullable): [n][16] span-local rows, the one-hot slot of
                                   // the row's request in its 256-row CTA-pair tile, repeated in k 0-7 / 8-15
  int chunk;                       // rows per FC chunk (pair tiles are 256-row aligned inside a chunk)
  int nslot;                       // max requests per pair tile folded into the MMA (else all-zero rows)
  int bf16;
  float* E;                        // dense SE (nullable): [n][lde] fp32 pre-SE ê (after linear_log) at
  int lde;                         //   column sel_pos * k; the gate runs in se_dense_kernel
  DevGroup gp[COLD_MAX_GROUPS];    // copy of groups[0..M) in the parameters (read via the constant bank)
  // SE weights of the launch's columns in the parameters (constant bank): column j's w at
  // sew_c[j * k .. j * k + k), b at seb_c[j]; set when n_ac * k <= GATHER_SEW_MAX (else read from se_w / se_b)
  int sew_in_params;
  float sew_c[512];
  float seb_c[COLD_MAX_GROUPS];
  int x_slab;                      // X_ac in the half-slab layout: column block `slot` of ad a at
  int64_t x_rows;                  //   [(2 slot + h) * x_rows + a][8], h = 0 / 1 for columns 0-7 / 8-15
  int ring;                        // != 0: every column is a cross-bag column (user bag x single ad id), for
                                   // the bag-only build: -1 register bursts, > 0 a `ring`-deep cp.async ring
  int search_req;                  // 1: request of an ad by binary search of adoff (req_of_ad not yet written)
  const int32_t* adoff; int R;     // call-global ad offsets [R+1]
};

// dense SE gate (COLD_SE_DENSE, the Doc B reading of P:229-234): per ad, ê = [ê_g] over the selected
// groups in schema order (user columns from xu[request], the rest from E), s = sigma(Wd ê + bd),
// X[ad][sel_pos * k + d] = cast(s_g ê_g[d]) (input normalisation in fp32 before the cast).
struct SeDenseArgs {
  const float* E; int lde;         // span-local [n][lde] (ad + cross columns)
  const float* xu; int ldu;        // [R][ldu] per-request user ê, user group j at column j * k
  int n_user; int user_pos[COLD_MAX_GROUPS];   // selected position of user group j
  const int32_t* req_of_ad; int64_t a0; int64_t n;
  const float* wdt;                // [D_in][n_sel] (Wd transposed)
  const float* bd;                 // [n_sel]
  int n_sel, k, d_in;
  const float* in_scale; const float* in_shift;
  void* X; int ldx;                // span-local [n][ldx] storage dtype
  float* dbg_feat;                 // [N][D_in] (call-global rows, nullable)
};
void launch_se_dense(const SeDenseArgs& a, int precision, cudaStream_t s);
size_t se_dense_smem(int d_in, int n_sel);   // dynamic shared memory of the dense-SE kernel (<= 227 KB)

struct RowsArgs {
  const DevGroup* groups;
  BatchView bv;
  int g;
  const int32_t* req_of_ad;
  int64_t n;
  int64_t* rows;
  int max_rows;
};

// precision: 0 fp32, 1 fp16, 2 bf16 (storage dtype of tables and X)
void launch_user(const UserArgs& a, int R, int precision, cudaStream_t s);
void launch_gather(const GatherArgs& a, int precision, cudaStream_t s);
void launch_rows(const RowsArgs& a, cudaStream_t s);

// fp32 SIMT FC stack (no TF32): X -> scores
struct MlpF32Args {
  const float* X; int ldx; int d_ac;
  const float* u1; int ld_u1;      // [R][W0] (user part + b1)
  const int32_t* req_of_ad; int64_t a0; int64_t n;
  int L;
  const float* wt[COLD_MAX_LAYERS];  // layer 0: W1_ac^T [d_ac][W0]; l>0: W_l^T [in][out]
  const float* b[COLD_MAX_LAYERS];   // layer 0 unused (inside u1)
  int width[COLD_MAX_LAYERS];
  const float* slope[COLD_MAX_LAYERS];   // PReLU slopes of hidden layer l (F2; null: ReLU)
  int max_w;
  float* scores;                   // chunk-local [n]
};
void launch_mlp_f32(const MlpF32Args& a, cudaStream_t s);

// tcgen05 GEMM layer: out = act(A . B^T + bias [+ u1[req]]) or fused head -> scores
struct EpiParams {
  const float* bias;               // [N] or null
  const float* u1; int ld_u1;      // FC1: per-request pre-activation [R][ld_u1]
  const int32_t* req_of_ad; int64_t a0;
  const int32_t* ad_offsets;       // FC1: call-global [R+1] (request boundary inside a tile)
  void* out; int ldo;              // [M][ldo] storage dtype (null with a head); written through tmC
  const float* head_w;             // [head_n][N] fp32
  const float* head_b;             // [head_n]
  int head_n;                      // 0: no head; 1 or 2: fused last layer + sigmoid
  float* scores;                   // chunk-local [M]
  int relu;
  int a_slab;                      // A (layer 0: X_ac) in the half-slab layout via a 3-D map
  const float* slope;              // PReLU slopes [N] (F2; null: ReLU when relu)
  unsigned long long* instr;       // debug: per-role wait-cycle counters [8] (null = off)
  int dbg_mode;                    // timing experiments only (results invalid): 1 = epilogue only drains
                                   // TMEM (no math / stores), 2 = MMA issuer skips the MMAs, 3 = epilogue
                                   // math without smem / TMA stores, 4 = smem staging but no TMA store
};
cudaError_t launch_gemm(const CUtensorMap* tmA, const CUtensorMap* tmB, const CUtensorMap* tmC, int M, int N, int K,
                        int bn, int bf16, int cs, bool resb, const EpiParams& ep, int num_sms, bool pdl,
                        cudaStream_t s);
bool gemm_resident_ok(int bn, int K);
// CTA-pair (cta_group::2) variant: 256-row tiles, each CTA stages half of the weight tile
// FC1 (ep.u1 set): tmOH = one-hot rows of the chunk ([rows][16], box 8 x 128), tmU1T = u1 terms
// ([terms * H][R_pad], box 8 requests x 128 columns); the kernel adds u1[request(row)] with one (f16) or
// two (bf16) extra K = 16 MMAs per tile (kernels_gemm2.cu)
constexpr int U1_NSLOT = 8;
cudaError_t launch_gemm_pair(const CUtensorMap* tmA, const CUtensorMap* tmB, const CUtensorMap* tmC, int M, int N,
                             int K, int bn, int bf16, const EpiParams& ep, int num_sms, bool pdl, cudaStream_t s,
                             const CUtensorMap* tmOH = nullptr, const CUtensorMap* tmU1T = nullptr,
                             bool res = false);
// the pair's weight half fits resident (<= 64 KB): the RES variant keeps it in smem for the launch
bool gemm_pair_resident_ok(int bn, int K);

// fused FC(L-4) .. FC(L-2) + head (paper widths 256, 128, 64 -> 2)
struct TailParams {
  const float* b3; const float* b4; const float* b5;
  const float* head_w; const float* head_b; int head_n;
  float* scores;                   // chunk-local [M]
  int reverse;                     // tail45: walk tiles last-first (the most recently written H3 rows are
                                   // the ones still in L2)
  const float* s4; const float* s5;  // tail45 PReLU slopes of FC(L-3) / FC(L-2) (F2; null: ReLU)
};
bool tail_supported(int n3, int n4, int n5, int k3);
cudaError_t launch_tail(const CUtensorMap* tmA3, const CUtensorMap* tmB3, const CUtensorMap* tmB4,
                        const CUtensorMap* tmB5, int M, int K3, int bf16, const TailParams& tp, int num_sms, bool pdl,
                        cudaStream_t s);

// FC1 -> FC2 -> FC3 in one persistent CTA-pair kernel over 256-row blocks (kernels_chain.cu)
struct ChainParams {
  const float* b2; const float* b3;      // FC2 / FC3 biases (FC1's bias is inside u1)
  const float* s1; const float* s2; const float* s3;   // PReLU slopes of FC1..FC3 (F2; null: ReLU)
  int x_slab;                            // FC1's A (X_ac) in the half-slab layout (3-D map)
  const float* u1; int ld_u1;            // FC1 fallback for blocks spanning > U1_NSLOT requests
  const int32_t* req_of_ad; int64_t a0;
  int n1, n2, n3, k1;                    // widths of FC1..FC3 and FC1's K (D_ac_pad)
  const void* h1; const void* h2;        // H1 / H2 chunk buffers (for the L2 discards)
  // TAIL variant: FC4 (n4) -> FC5 (n5) -> head (head_n = 1 or 2) -> sigma -> scores, also in the chain
  int tail; int n4, n5;
  const float* b4; const float* b5; const float* head_w; const float* head_b; int head_n;
  const void* h3; const void* h4;
  float* scores;                         // chunk-local [M]
  unsigned long long* instr;             // debug (nullable): wait cycles [0] producer empty, [1] producer
                                         // hready, [2] MMA full, [3] MMA tempty, [4] MMA uxfull, [5] epi tfull
};
bool chain_supported(int n1, int n2, int n3, int k1);
bool chain_tail_supported(int n4, int n5, int n3);
// tm: X (slot), W1, W2, W3, H1, H2, H3, one-hot (slot), u1 terms, W4 half-box, W5 half-box, H4
cudaError_t launch_chain(const CUtensorMap* tm[12], int M, int bf16, const ChainParams& cp, int num_sms, bool pdl,
                         cudaStream_t s);

// fused FC(L-3) .. FC(L-2) + head after a GEMM FC(L-4) (paper widths 128, 64 -> 2), resident weights
bool tail45_supported(int n4, int n5, int k4);
cudaError_t launch_tail45(const CUtensorMap* tmA4, const CUtensorMap* tmB4, const CUtensorMap* tmB5, int M, int bf16,
                          const TailParams& tp, int num_sms, bool pdl, cudaStream_t s);

// vector-product baseline (F4): scores[ad] = sigma(user_vecs[request] . ad_vecs[ad_ids[ad]])
struct VpsArgs {
  const void* ad_vecs; int64_t num_vecs; int d;
  const float* user_vecs;          // [R][d] fp32
  const int32_t* ad_ids;           // [N]
  const int32_t* ad_offsets;       // [R+1]
  int R;
  float* scores;                   // [N]
};
cudaError_t launch_vps(const VpsArgs& a, int precision, int max_n, cudaStream_t s);

// top-K per request
struct TopkArgs {
  const float* scores; const float* bids; const int32_t* ad_offsets;
  int R; int K;
  int32_t* idx; float* key;
  // merge mode (G > 0, cold_merge_topk): `scores` holds the all-gathered per-rank top-Kl keys
  // [G][R][Kl], `cand_idx` their positions inside each rank's slice; request r's candidates are
  // (g, j) in rank order; the output position is cand_idx + the slice start floor(g * n_r / G)
  int G, Kl;
  const int32_t* cand_idx;
  int max_n;                       // longest segment (host-known): keys are staged in smem when small
  int stage;                       // set by launch_topk: smem key capacity (0 = read keys from global)
};
void launch_topk(const TopkArgs& a, cudaStream_t s);

}  // namespace cold
