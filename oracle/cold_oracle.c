/* oracle/cold_oracle.c — TEST INFRASTRUCTURE ONLY (see cold_oracle.h).
 *
 * The plain definition of COLD's scoring pass, in fp64, written in the paper's
 * order: rows -> sum-pool -> linear_log -> SE gate -> concat -> FC -> sigma -> top-K.
 * No hoisting, no blocking, no fusion. Build: gcc -O2 -fopenmp -ffp-contract=off.
 */
#include "cold_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---- scalar definitions ------------------------------------------------------ */

/* P:278-287, Eq. (eq:log):  -log(-x)-1 for x<-1;  x for -1<=x<=1;  log(x)+1 for x>1.
 * Natural log (AMB-4: only base e makes it C^1 at |x|=1, as P:289 claims).
 * Identity on the closed interval (AMB-5, as printed). */
double orc_linear_log(double x) {
  if (x < -1.0) return -log(-x) - 1.0;
  if (x > 1.0) return log(x) + 1.0;
  return x;
}

/* P:163 (§2.1): sigma(x) = 1/(1+e^-x). Two algebraically equal branches avoid
 * overflow of e^-x for very negative z. */
double orc_sigmoid(double z) {
  if (z >= 0.0) return 1.0 / (1.0 + exp(-z));
  double e = exp(z);
  return e / (1.0 + e);
}

/* MurmurHash3 fmix64 (AMB-9 reading of the undefined cross-feature construction,
 * P:245 "computes cross-features"). */
uint64_t orc_fmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33;
  return k;
}

/* AMB-9: cross_row(g,x,y,C) = floor(fmix64(fmix64(x ^ salt_g) ^ y) * C / 2^64),
 * salt_g = (g+1) * 0x9E3779B97F4A7C15 mod 2^64. */
int64_t orc_cross_row(int32_t g, uint64_t x, uint64_t y, int64_t C) {
  uint64_t salt = (uint64_t)(g + 1) * 0x9E3779B97F4A7C15ULL;
  uint64_t h = orc_fmix64(orc_fmix64(x ^ salt) ^ y);
  return (int64_t)(((unsigned __int128)h * (unsigned __int128)(uint64_t)C) >> 64);
}

/* IEEE binary16 -> double, exact (sign, 5-bit exponent, 10-bit fraction). */
static double half_to_double(uint16_t h) {
  int s = (h >> 15) & 1, e = (h >> 10) & 31, f = h & 1023;
  double v;
  if (e == 0) v = ldexp((double)f, -24);
  else if (e == 31) v = f ? NAN : INFINITY;
  else v = ldexp((double)(1024 + f), e - 25);
  return s ? -v : v;
}

/* bfloat16 bits are the top half of an IEEE binary32. */
static double bf16_to_double(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return (double)f;
}

static double table_value(const orc_group* G, int64_t row, int d, int k) {
  int64_t i = row * (int64_t)k + d;
  switch (G->table_dtype) {
    case ORC_F32: return (double)((const float*)G->table)[i];
    case ORC_F16: return half_to_double(((const uint16_t*)G->table)[i]);
    default: return bf16_to_double(((const uint16_t*)G->table)[i]);
  }
}

/* ---- rows of one (request, ad, group): P:229, P:245, P:276 ------------------- */

static int64_t request_of(const orc_batch* bt, int64_t a) {
  int64_t lo = 0, hi = bt->R - 1;           /* last r with ad_offsets[r] <= a */
  while (lo < hi) {
    int64_t mid = (lo + hi + 1) / 2;
    if (bt->ad_offsets[mid] <= a) lo = mid; else hi = mid - 1;
  }
  return lo;
}

/* the id list ("bag") of a USER group for request r or of an AD group for ad a */
static int64_t bag_of(const orc_model* m, const orc_batch* bt, int32_t g, int64_t r, int64_t a,
                      const int32_t** ids) {
  const orc_group* G = &m->groups[g];
  if (G->side == ORC_USER) {
    *ids = bt->ids[g] + bt->offs[g][r];
    return bt->offs[g][r + 1] - bt->offs[g][r];
  }
  if (bt->offs[g] == NULL) { *ids = bt->ids[g] + a; return 1; }
  *ids = bt->ids[g] + bt->offs[g][a];
  return bt->offs[g][a + 1] - bt->offs[g][a];
}

/* Enumerate rows in definition order; returns the count, -ORC_ERR_ID_RANGE on a bad id
 * (AMB-18: the oracle raises). rows may be NULL (count only). */
static int64_t rows_of(const orc_model* m, const orc_batch* bt, int32_t g, int64_t r, int64_t a,
                       int64_t* rows, int64_t max_rows) {
  const orc_group* G = &m->groups[g];
  int64_t n = 0;
  if (G->side != ORC_CROSS) {
    const int32_t* ids;
    int64_t L = bag_of(m, bt, g, r, a, &ids);
    for (int64_t i = 0; i < L; i++) {
      if (ids[i] < 0 || ids[i] >= G->card) return -ORC_ERR_ID_RANGE;
      if (rows && n < max_rows) rows[n] = ids[i];
      n++;
    }
    return n;
  }
  const int32_t *xs, *ys;
  int64_t Lx = bag_of(m, bt, G->user_ref, r, a, &xs);
  int64_t Ly = bag_of(m, bt, G->ad_ref, r, a, &ys);
  for (int64_t i = 0; i < Lx; i++) {               /* x-major Cartesian product */
    if (xs[i] < 0 || xs[i] >= m->groups[G->user_ref].card) return -ORC_ERR_ID_RANGE;
    for (int64_t j = 0; j < Ly; j++) {
      if (ys[j] < 0 || ys[j] >= m->groups[G->ad_ref].card) return -ORC_ERR_ID_RANGE;
      if (rows && n < max_rows) rows[n] = orc_cross_row(g, (uint64_t)xs[i], (uint64_t)ys[j], G->card);
      n++;
    }
  }
  return n;
}

int64_t orc_rows(const orc_model* m, const orc_batch* bt, int32_t g, int64_t a,
                 int64_t* rows_out, int64_t max_rows) {
  if (!m || !bt || g < 0 || g >= m->M || a < 0 || a >= bt->ad_offsets[bt->R]) return -ORC_ERR_ARG;
  return rows_of(m, bt, g, request_of(bt, a), a, rows_out, max_rows);
}

/* e_g = sum of the rows' embeddings, fp64 ("sum-pooling"; empty bag -> 0). */
static int pool(const orc_model* m, const orc_batch* bt, int32_t g, int64_t r, int64_t a, double* e) {
  const orc_group* G = &m->groups[g];
  int k = m->k;
  for (int d = 0; d < k; d++) e[d] = 0.0;
  int64_t n = rows_of(m, bt, g, r, a, NULL, 0);
  if (n < 0) return (int)-n;
  int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  rows_of(m, bt, g, r, a, rows, n);
  for (int64_t i = 0; i < n; i++)
    for (int d = 0; d < k; d++) e[d] += table_value(G, rows[i], d, k);
  free(rows);
  return ORC_OK;
}

/* x = [v_g] for one (request, ad): P:229-235 (SE), P:278-289 (linear_log), P:328 (concat). */
static int features(const orc_model* m, const orc_batch* bt, int64_t r, int64_t a, double* x,
                    double* eh_all) {
  int k = m->k;
  for (int j = 0; j < m->n_sel; j++) {
    int32_t g = m->sel[j];
    double* eh = eh_all + (size_t)j * k;
    int rc = pool(m, bt, g, r, a, eh);
    if (rc) return rc;
    if (m->linear_log && !m->ll_after_se)
      for (int d = 0; d < k; d++) eh[d] = orc_linear_log(eh[d]);
  }
  for (int j = 0; j < m->n_sel; j++) {
    int32_t g = m->sel[j];
    double* eh = eh_all + (size_t)j * k;
    double z = 0.0;
    if (!m->se_dense) {
      /* Doc A P:11-14: s_i = sigma(W e_i + b), W in R^{k x 1}, b in R^1 (per group). */
      for (int d = 0; d < k; d++) z += m->se_w[(size_t)g * k + d] * eh[d];
      z += m->se_b[g];
    } else {
      /* Doc B P:229-234: s = sigma(W [e_1..e_M] + b) over the whole selected concat. */
      const double* Wrow = m->se_W_dense + (size_t)j * m->n_sel * k;
      for (int i = 0; i < m->n_sel * k; i++) z += Wrow[i] * eh_all[i];
      z += m->se_b_dense[j];
    }
    double s = orc_sigmoid(z);
    /* v_i = s_i * e_i (field-wise multiplication). */
    for (int d = 0; d < k; d++) {
      double v = s * eh[d];
      if (m->linear_log && m->ll_after_se) v = orc_linear_log(v);
      /* batch norm of the network input, inference form (folded affine per column) */
      if (m->in_scale) v = v * m->in_scale[(size_t)j * k + d] + m->in_shift[(size_t)j * k + d];
      x[(size_t)j * k + d] = v;
    }
  }
  return ORC_OK;
}

static int max_width(const orc_model* m) {
  int w = m->n_sel * m->k;
  for (int l = 0; l < m->L; l++) if (m->widths[l] > w) w = m->widths[l];
  return w;
}

/* FC stack P:328: h_l = act(W_l h_{l-1} + b_l), last layer linear. act = ReLU (AMB-6: the paper never
 * names the activation), or PReLU with a per-channel slope a_j (act(x) = x for x > 0, a_j x otherwise;
 * the model variant of SURVEY §8(f) F2);
 * score P:163 / AMB-7: p = sigma(z1 - z0) for a 2-wide head, sigma(z) for 1-wide. */
static void fcn(const orc_model* m, const double* x, double* buf0, double* buf1, double* p, double* zo) {
  int in = m->n_sel * m->k;
  const double* h = x;
  double* out = buf0;
  for (int l = 0; l < m->L; l++) {
    int o = m->widths[l];
    const double* W = m->W[l];
    for (int j = 0; j < o; j++) {
      double acc = m->b[l][j];
      for (int i = 0; i < in; i++) acc += W[(size_t)j * in + i] * h[i];
      if (l == m->L - 1) out[j] = acc;
      else if (m->activation == 1) out[j] = acc > 0.0 ? acc : m->slope[l][j] * acc;
      else out[j] = acc > 0.0 ? acc : 0.0;
    }
    h = out;
    out = (out == buf0) ? buf1 : buf0;
    in = o;
  }
  double z = (m->widths[m->L - 1] == 2) ? h[1] - h[0] : h[0];
  *zo = z;
  *p = orc_sigmoid(z);
}

static int check_model(const orc_model* m) {
  if (!m || m->M <= 0 || m->k <= 0 || m->n_sel <= 0 || m->L <= 0) return ORC_ERR_ARG;
  int last = m->widths[m->L - 1];
  if (last != 1 && last != 2) return ORC_ERR_ARG;
  for (int j = 0; j < m->n_sel; j++) {
    if (m->sel[j] < 0 || m->sel[j] >= m->M) return ORC_ERR_ARG;
    if (j > 0 && m->sel[j] <= m->sel[j - 1]) return ORC_ERR_ARG;
  }
  for (int g = 0; g < m->M; g++) {
    const orc_group* G = &m->groups[g];
    if (G->card < 1) return ORC_ERR_ARG;
    if (G->side == ORC_CROSS) {
      if (G->user_ref < 0 || G->user_ref >= m->M || m->groups[G->user_ref].side != ORC_USER) return ORC_ERR_ARG;
      if (G->ad_ref < 0 || G->ad_ref >= m->M || m->groups[G->ad_ref].side != ORC_AD) return ORC_ERR_ARG;
    }
  }
  return ORC_OK;
}

int32_t orc_score(const orc_model* m, const orc_batch* bt, const int64_t* ad_list, int64_t n_list,
                  double* p_out, double* z_out, int32_t nthreads) {
  int rc = check_model(m);
  if (rc) return rc;
  if (!bt || bt->R < 1) return ORC_ERR_ARG;
  int64_t N = bt->ad_offsets[bt->R];
  if (!ad_list) n_list = N;
  int W = max_width(m);
  int err = ORC_OK;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
#pragma omp parallel
  {
    double* x = (double*)malloc(sizeof(double) * (size_t)m->n_sel * m->k);
    double* eh = (double*)malloc(sizeof(double) * (size_t)m->n_sel * m->k);
    double* b0 = (double*)malloc(sizeof(double) * (size_t)W);
    double* b1 = (double*)malloc(sizeof(double) * (size_t)W);
#pragma omp for schedule(dynamic, 64)
    for (int64_t i = 0; i < n_list; i++) {
      int64_t a = ad_list ? ad_list[i] : i;
      if (a < 0 || a >= N) { err = ORC_ERR_ARG; continue; }
      int64_t r = request_of(bt, a);
      int lrc = features(m, bt, r, a, x, eh);
      if (lrc) { err = lrc; continue; }
      double p, z;
      fcn(m, x, b0, b1, &p, &z);
      p_out[i] = p;
      if (z_out) z_out[i] = z;
    }
    free(x); free(eh); free(b0); free(b1);
  }
  return err;
}

int32_t orc_features(const orc_model* m, const orc_batch* bt, const int64_t* ad_list, int64_t n_list,
                     int32_t order, double* x_out) {
  int rc = check_model(m);
  if (rc) return rc;
  int64_t N = bt->ad_offsets[bt->R];
  if (!ad_list) n_list = N;
  int k = m->k, D = m->n_sel * k;
  double* eh = (double*)malloc(sizeof(double) * (size_t)D);
  double* x = (double*)malloc(sizeof(double) * (size_t)D);
  int err = ORC_OK;
  if (order == 0) {                       /* row order: ads one by one ("row based") */
    for (int64_t i = 0; i < n_list && !err; i++) {
      int64_t a = ad_list ? ad_list[i] : i;
      err = features(m, bt, request_of(bt, a), a, x, eh);
      memcpy(x_out + (size_t)i * D, x, sizeof(double) * (size_t)D);
    }
  } else if (!m->se_dense) {             /* column order: one group for all ads, then the next */
    for (int j = 0; j < m->n_sel && !err; j++) {
      int32_t g = m->sel[j];
      for (int64_t i = 0; i < n_list && !err; i++) {
        int64_t a = ad_list ? ad_list[i] : i;
        double e[64];
        if (k > 64) { err = ORC_ERR_ARG; break; }
        err = pool(m, bt, g, request_of(bt, a), a, e);
        if (m->linear_log && !m->ll_after_se) for (int d = 0; d < k; d++) e[d] = orc_linear_log(e[d]);
        double z = 0.0;
        for (int d = 0; d < k; d++) z += m->se_w[(size_t)g * k + d] * e[d];
        z += m->se_b[g];
        double s = orc_sigmoid(z);
        for (int d = 0; d < k; d++) {
          double v = s * e[d];
          if (m->linear_log && m->ll_after_se) v = orc_linear_log(v);
          if (m->in_scale) v = v * m->in_scale[(size_t)j * k + d] + m->in_shift[(size_t)j * k + d];
          x_out[(size_t)i * D + (size_t)j * k + d] = v;
        }
      }
    }
  } else {
    err = ORC_ERR_ARG;
  }
  free(eh); free(x);
  return err;
}

/* SE importance weights of EVERY schema group for the listed ads (§3.2 "Importance
 * weight calculation" / "Feature group selection"): pool -> linear_log (AMB-3 order) ->
 * s_g = sigma(w_g . e_g + b_g) (per-group reading AMB-1). s_out: [n_list][M]. The ranking of groups
 * by the mean of s_g over a sample of ads (AMB-16) selects the top-K groups. */
int32_t orc_se_gates(const orc_model* m, const orc_batch* bt, const int64_t* ad_list, int64_t n_list,
                     double* s_out) {
  if (!m || !bt || !s_out || m->M < 1 || m->k < 1 || m->k > 64 || m->se_dense) return ORC_ERR_ARG;
  int64_t N = bt->ad_offsets[bt->R];
  if (!ad_list) n_list = N;
  int k = m->k;
  for (int64_t i = 0; i < n_list; i++) {
    int64_t a = ad_list ? ad_list[i] : i;
    if (a < 0 || a >= N) return ORC_ERR_ARG;
    int64_t r = request_of(bt, a);
    for (int32_t g = 0; g < m->M; g++) {
      double e[64];
      int rc = pool(m, bt, g, r, a, e);
      if (rc) return rc;
      if (m->linear_log && !m->ll_after_se) for (int d = 0; d < k; d++) e[d] = orc_linear_log(e[d]);
      double z = 0.0;
      for (int d = 0; d < k; d++) z += m->se_w[(size_t)g * k + d] * e[d];
      z += m->se_b[g];
      s_out[(size_t)i * m->M + g] = orc_sigmoid(z);
    }
  }
  return ORC_OK;
}

int32_t orc_pooled_f32(const orc_model* m, const orc_batch* bt, const int64_t* ad_list, int64_t n_list,
                       float* out) {
  int rc = check_model(m);
  if (rc) return rc;
  int64_t N = bt->ad_offsets[bt->R];
  if (!ad_list) n_list = N;
  int k = m->k;
  for (int64_t i = 0; i < n_list; i++) {
    int64_t a = ad_list ? ad_list[i] : i;
    int64_t r = request_of(bt, a);
    for (int j = 0; j < m->n_sel; j++) {
      int32_t g = m->sel[j];
      const orc_group* G = &m->groups[g];
      int64_t n = rows_of(m, bt, g, r, a, NULL, 0);
      if (n < 0) return (int32_t)-n;
      int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
      rows_of(m, bt, g, r, a, rows, n);
      float* e = out + ((size_t)i * m->n_sel + j) * k;
      for (int d = 0; d < k; d++) e[d] = 0.0f;
      for (int64_t q = 0; q < n; q++)
        for (int d = 0; d < k; d++) e[d] = e[d] + (float)table_value(G, rows[q], d, k);
      free(rows);
    }
  }
  return ORC_OK;
}

/* ---- top-K ("selects top N candidates by certain metrics, e.g. eCPM") ---- */

typedef struct { double key; int64_t pos; } orc_kp;

static int kp_cmp(const void* pa, const void* pb) {
  const orc_kp* a = (const orc_kp*)pa;
  const orc_kp* b = (const orc_kp*)pb;
  int na = isnan(a->key), nb = isnan(b->key);
  if (na != nb) return na ? 1 : -1;              /* NaN ranks last (AMB-13) */
  if (!na && a->key != b->key) return a->key > b->key ? -1 : 1;
  return (a->pos > b->pos) - (a->pos < b->pos);  /* ties: ascending position */
}

/* Vector-product based pre-ranking model (§2.2): p = sigma(v_u^T v_a), v_u per request
 * (user tower output), v_a per ad looked up by id in the precomputed ad-tower table (stored values,
 * any storage dtype). fp64 dot product in index order. */
int32_t orc_vps_score(int32_t d, const void* ad_table, int32_t table_dtype, int64_t card, const double* user_vecs,
                      int32_t R, const int32_t* ad_offsets, const int32_t* ad_ids, double* p_out) {
  if (d < 1 || !ad_table || !user_vecs || !ad_offsets || !ad_ids || !p_out || R < 1 || card < 1) return ORC_ERR_ARG;
  orc_group G;
  G.side = ORC_AD;
  G.card = card;
  G.user_ref = -1;
  G.ad_ref = -1;
  G.table_dtype = table_dtype;
  G.table = ad_table;
  for (int32_t r = 0; r < R; r++)
    for (int64_t a = ad_offsets[r]; a < ad_offsets[r + 1]; a++) {
      int64_t id = ad_ids[a];
      if (id < 0 || id >= card) return ORC_ERR_ID_RANGE;
      double z = 0.0;
      for (int k = 0; k < d; k++) z += user_vecs[(size_t)r * d + k] * table_value(&G, id, k, d);
      p_out[a] = orc_sigmoid(z);
    }
  return ORC_OK;
}

int32_t orc_topk(const double* key, int64_t n, int32_t K, int32_t* idx_out, double* key_out) {
  if (n < 1) return ORC_ERR_ARG;
  if (K < 1 || K > n) return ORC_ERR_K_RANGE;
  orc_kp* v = (orc_kp*)malloc(sizeof(orc_kp) * (size_t)n);
  for (int64_t i = 0; i < n; i++) { v[i].key = key[i]; v[i].pos = i; }
  qsort(v, (size_t)n, sizeof(orc_kp), kp_cmp);
  for (int32_t i = 0; i < K; i++) {
    idx_out[i] = (int32_t)v[i].pos;
    if (key_out) key_out[i] = v[i].key;
  }
  free(v);
  return ORC_OK;
}
