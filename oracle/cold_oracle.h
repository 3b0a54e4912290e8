/* oracle/cold_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, fp64 CPU definition of COLD's online pre-ranking scoring pass
 * (arXiv 2007.16122). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. It shares no code,
 * header, table or constant with the CUDA path (paper_2007_16122_b200/).
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (section in brackets).
 * Readings of ambiguous passages (AMB-n) are listed in DESIGN.md §2.
 *
 * Parity pins (tests/test_oracle_*.py): every exported function is pinned to
 * something other than itself — closed forms, the paper's worked equation
 * values (tests/golden/), torch fp64 library routines, brute force and the
 * pure-Python twin oracle/mini.py. None is "parity unpinned".
 */
#ifndef COLD_ORACLE_H
#define COLD_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_ERR_ARG = 1, ORC_ERR_ID_RANGE = 2, ORC_ERR_K_RANGE = 3 };
enum { ORC_USER = 0, ORC_AD = 1, ORC_CROSS = 2 };
enum { ORC_F32 = 0, ORC_F16 = 1, ORC_BF16 = 2 };

typedef struct {
  int32_t side;          /* ORC_USER / ORC_AD / ORC_CROSS */
  int64_t card;          /* table rows */
  int32_t user_ref;      /* CROSS: schema index of the USER group crossed */
  int32_t ad_ref;        /* CROSS: schema index of the AD group crossed */
  int32_t table_dtype;   /* ORC_F32 / ORC_F16 / ORC_BF16: storage of `table` */
  const void* table;     /* [card * k], row-major, the values the scorer stores */
} orc_group;

typedef struct {
  int32_t M, k;                 /* groups, embedding dim ("set to be 16") */
  const orc_group* groups;      /* [M], schema order */
  int32_t n_sel;                /* selected groups, ascending schema order */
  const int32_t* sel;
  const double* se_w;           /* [M * k]: per-group SE weight w_g (AMB-1) */
  const double* se_b;           /* [M] */
  int32_t se_dense;             /* 1: Doc-B dense SE over the selected concat (AMB-1 alt.) */
  const double* se_W_dense;     /* [n_sel][n_sel * k] when se_dense */
  const double* se_b_dense;     /* [n_sel] when se_dense */
  int32_t linear_log;           /* 1: apply linear_log */
  int32_t ll_after_se;          /* 0: LL then SE (AMB-3 default); 1: SE on raw e, LL on v */
  int32_t L;                    /* FC layers */
  const int32_t* widths;        /* [L] outputs; input of layer 0 = n_sel * k */
  const double* const* W;       /* [L] each [out][in] */
  const double* const* b;       /* [L] each [out] */
  const double* in_scale;       /* [n_sel * k] or NULL: input batch norm folded to x_j * in_scale[j] +  */
  const double* in_shift;       /* in_shift[j] (P:276's alternative to linear_log)  */
  int32_t activation;           /* hidden activation: 0 ReLU (AMB-6), 1 PReLU */
  const double* const* slope;   /* PReLU: [L-1] each [out_l], h = x if x > 0 else slope * x */
} orc_model;

typedef struct {
  int32_t R;                    /* requests */
  const int32_t* ad_offsets;    /* [R+1] */
  const int32_t* const* ids;    /* [M]; NULL for CROSS */
  const int32_t* const* offs;   /* [M]; USER: [R+1]; AD: NULL (single) or [N+1]; CROSS: NULL */
} orc_batch;

/* linear_log, P:278-287 (Eq. eq:log), natural log (AMB-4). */
double orc_linear_log(double x);
/* sigma(z) = 1 / (1 + e^-z), P:163 (§2.1), evaluated in the stable branch form. */
double orc_sigmoid(double z);
/* MurmurHash3 64-bit finalizer (AMB-9). */
uint64_t orc_fmix64(uint64_t k);
/* Cross-feature row (AMB-9): floor(fmix64(fmix64(x ^ salt_g) ^ y) * C / 2^64). */
int64_t orc_cross_row(int32_t g, uint64_t x, uint64_t y, int64_t C);

/* Rows feeding group g for ad `a` (global ad index) — P:229; CROSS rows are
 * the x-major Cartesian product of the user bag and the ad bag, duplicates kept.
 * Writes up to max_rows rows, returns the total count (or -ORC_ERR_*). */
int64_t orc_rows(const orc_model* m, const orc_batch* bt, int32_t g, int64_t a,
                 int64_t* rows_out, int64_t max_rows);

/* Scores p (and the logit z, z1-z0 for a 2-wide head) for the listed global ads
 * (ad_list == NULL: all ads), steps 1-7 of DESIGN.md §2 in fp64, per (request, ad),
 * no user hoisting. nthreads <= 0: OpenMP default. */
int32_t orc_score(const orc_model* m, const orc_batch* bt, const int64_t* ad_list, int64_t n_list,
                  double* p_out, double* z_out, int32_t nthreads);

/* Concatenated SE-weighted features x = [v_g], g in sel (fp64), for the listed ads.
 * order 0 = row order (ads outermost), 1 = column order (groups outermost). */
int32_t orc_features(const orc_model* m, const orc_batch* bt, const int64_t* ad_list, int64_t n_list,
                     int32_t order, double* x_out);

/* fp32-ordered gather mode: raw pooled sums e_g (before LL/SE) accumulated in fp32,
 * sequentially in bag order (cross: x-major), for every selected group, listed ads.
 * out: [n_list][n_sel][k]. For the bit-exact gather parity (P-5). */
int32_t orc_pooled_f32(const orc_model* m, const orc_batch* bt, const int64_t* ad_list, int64_t n_list,
                       float* out);

/* SE importance weights s_g of every schema group (selected or not) for the listed ads,
 * pool -> linear_log -> sigma(w_g . e_g + b_g). out: [n_list][M]. Feature-group
 * selection ranks groups by the mean over a sample of ads (AMB-16). */
int32_t orc_se_gates(const orc_model* m, const orc_batch* bt, const int64_t* ad_list, int64_t n_list,
                     double* s_out);

/* Vector-product based model: p[a] = sigma(user_vecs[r] . table[ad_ids[a]]) for every ad a of
 * request r; table: [card][d] stored values of table_dtype (F4 baseline of SURVEY §8(f)). */
int32_t orc_vps_score(int32_t d, const void* ad_table, int32_t table_dtype, int64_t card, const double* user_vecs,
                      int32_t R, const int32_t* ad_offsets, const int32_t* ad_ids, double* p_out);

/* Top-K of one request: stable order by (key desc, position asc), NaN last. */
int32_t orc_topk(const double* key, int64_t n, int32_t K, int32_t* idx_out, double* key_out);

#ifdef __cplusplus
}
#endif
#endif
