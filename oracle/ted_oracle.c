/* ted_oracle.c -- TEST INFRASTRUCTURE ONLY (see ted_oracle.h).  A plain-C, fp64
 * restatement of the reference's MoE-layer hot path.  Every function cites the
 * reference file:line (paths relative to /root/reference/proj/core/) it restates. */
#include "ted_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- deterministic init: tensor.cpp:100-129 ---------------------------------- */

uint64_t o_mix_seed(uint64_t seed, const char* tag) {
  uint64_t h = 14695981039346656037ULL; /* FNV-1a offset basis */
  for (const unsigned char* p = (const unsigned char*)tag; *p; ++p) {
    h ^= *p;
    h *= 1099511628211ULL;
  }
  uint64_t z = seed + 0x9E3779B97F4A7C15ULL + h;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* std::mt19937_64 (parameters fixed by the C++ standard, [rand.predef]). */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t s) {
  g->mt[0] = s;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t y = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t v = g->mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = v;
    }
    g->idx = 0;
  }
  uint64_t x = g->mt[g->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

void o_seeded_init(double* out, int64_t n, uint64_t seed, double scale) {
  mt64 g;
  mt64_seed(&g, seed);
  for (int64_t i = 0; i < n; ++i) {
    const double u = (double)(mt64_next(&g) >> 11) * 0x1.0p-53; /* top 53 bits -> [0,1) */
    out[i] = (2.0 * u - 1.0) * scale;
  }
}

/* ---- top-1 gate: moe.cpp:158-208 --------------------------------------------- */

void o_gate_route_logits(const double* L, int64_t n, int E, int* expert, double* chosen,
                         double* probs) {
  for (int64_t k = 0; k < n; ++k) {
    const double* l = L + k * E;
    /* strict '>' scanning ascending from j=1 with top = l[0]: lowest index wins ties */
    double top = l[0];
    int best = 0;
    for (int j = 1; j < E; ++j)
      if (l[j] > top) {
        top = l[j];
        best = j;
      }
    double sum = 0.0;
    double* p = probs + k * E;
    for (int j = 0; j < E; ++j) {
      p[j] = exp(l[j] - top);
      sum += p[j];
    }
    for (int j = 0; j < E; ++j) p[j] /= sum;
    expert[k] = best;
    chosen[k] = p[best];
  }
}

void o_gate_forward(const double* a, const double* wg, int64_t n, int h, int E, double* logits,
                    int* expert, double* chosen, double* probs) {
  for (int64_t k = 0; k < n; ++k) {
    double* lk = logits + k * E;
    for (int j = 0; j < E; ++j) lk[j] = 0.0;
    for (int i = 0; i < h; ++i) {
      const double x = a[k * h + i];
      for (int j = 0; j < E; ++j) lk[j] += x * wg[(int64_t)i * E + j];
    }
  }
  o_gate_route_logits(logits, n, E, expert, chosen, probs);
}

void o_gate_backward(const double* a, const double* wg, const double* probs, const int* expert,
                     const double* dchosen, int64_t n, int h, int E, double* dwg,
                     double* dinput) {
  double* dl = (double*)malloc(sizeof(double) * (size_t)(n * E));
  for (int64_t k = 0; k < n; ++k) {
    const int e = expert[k];
    const double coef = dchosen[k] * probs[k * E + e];
    for (int j = 0; j < E; ++j) dl[k * E + j] = coef * ((j == e ? 1.0 : 0.0) - probs[k * E + j]);
  }
  if (dwg) { /* dWg = a^T dlogits  (matmul_tn, nn.cpp:35-46) */
    memset(dwg, 0, sizeof(double) * (size_t)h * E);
    for (int64_t k = 0; k < n; ++k)
      for (int i = 0; i < h; ++i) {
        const double x = a[k * h + i];
        for (int j = 0; j < E; ++j) dwg[(int64_t)i * E + j] += x * dl[k * E + j];
      }
  }
  if (dinput) /* dinput = dlogits Wg^T  (matmul_nt, nn.cpp:48-60) */
    for (int64_t k = 0; k < n; ++k)
      for (int i = 0; i < h; ++i) {
        double acc = 0.0;
        for (int j = 0; j < E; ++j) acc += dl[k * E + j] * wg[(int64_t)i * E + j];
        dinput[k * h + i] = acc;
      }
  free(dl);
}

/* ---- capacity (absent in the reference) -----------------------
 * C = ceil(cf * n / E) on the full pre-drop shard (every TP peer computes the same);
 * slot(k) = #{k' < k : e(k') = e(k)} -- the reference's append order (moe.cpp:456-462);
 * keep = slot < C.  cf <= 0 means "no capacity" = reference semantics. */
int64_t o_capacity(double cf, int64_t n, int E) {
  if (cf <= 0.0) return n;
  int64_t c = (int64_t)ceil(cf * (double)n / (double)E);
  return c > n ? n : c;
}

void o_route_capacity(const int* expert, int64_t n, int E, int64_t cap, int T, int* slot,
                      uint8_t* keep, int* kept_counts) {
  int64_t* seen = (int64_t*)calloc((size_t)E, sizeof(int64_t));
  if (kept_counts) memset(kept_counts, 0, sizeof(int) * (size_t)T * E);
  const int64_t chunk = n / T;
  for (int64_t k = 0; k < n; ++k) {
    const int e = expert[k];
    const int64_t s = seen[e]++;
    if (slot) slot[k] = (int)s;
    const int kp = s < cap;
    if (keep) keep[k] = (uint8_t)kp;
    if (kept_counts && kp) {
      int64_t c = chunk > 0 ? k / chunk : 0;
      if (c >= T) c = T - 1;
      kept_counts[c * E + e] += 1;
    }
  }
  free(seen);
}

/* ---- GELU (tanh form): nn.cpp:92-121 ----------------------------------------- */

double o_gelu(double x) {
  const double c = 0.7978845608028653558798921198687, k3 = 0.044715;
  return 0.5 * x * (1.0 + tanh(c * (x + k3 * x * x * x)));
}

double o_gelu_grad(double x) {
  const double c = 0.7978845608028653558798921198687, k3 = 0.044715;
  const double t = tanh(c * (x + k3 * x * x * x));
  return 0.5 * (1.0 + t) + 0.5 * x * (1.0 - t * t) * c * (1.0 + 3.0 * k3 * x * x);
}

/* ---- dense helpers (restating nn.cpp:22-90 with cache-friendly loop orders) --- */

/* y[m,n] = x[m,k] w[k,n] (+ b[n]) */
static void mm_nn(const double* x, const double* w, const double* b, int64_t m, int64_t k,
                  int64_t n, double* y) {
  for (int64_t i = 0; i < m; ++i) {
    double* yi = y + i * n;
    for (int64_t j = 0; j < n; ++j) yi[j] = b ? b[j] : 0.0;
    for (int64_t p = 0; p < k; ++p) {
      const double xv = x[i * k + p];
      const double* wp = w + p * n;
      for (int64_t j = 0; j < n; ++j) yi[j] += xv * wp[j];
    }
  }
}
/* y[m,k] = dy[m,n] w[k,n]^T */
static void mm_nt(const double* dy, const double* w, int64_t m, int64_t n, int64_t k, double* y) {
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < k; ++j) {
      double acc = 0.0;
      const double* d = dy + i * n;
      const double* wj = w + j * n;
      for (int64_t p = 0; p < n; ++p) acc += d[p] * wj[p];
      y[i * k + j] = acc;
    }
}
/* y[k,n] += x[m,k]^T dy[m,n] */
static void mm_tn_acc(const double* x, const double* dy, int64_t m, int64_t k, int64_t n,
                      double* y) {
  for (int64_t i = 0; i < m; ++i)
    for (int64_t p = 0; p < k; ++p) {
      const double xv = x[i * k + p];
      if (xv == 0.0) continue;
      double* yp = y + p * n;
      const double* d = dy + i * n;
      for (int64_t j = 0; j < n; ++j) yp[j] += xv * d[j];
    }
}

/* ---- MoE branch: SerialModel::forward_layer :989-1015, backward_layer :1034-1064 */

int o_moe_layer(int S, int64_t n, int h, int f, int E, double cf, const double* a,
                const double* wg, const double* w1, const double* b1, const double* w2,
                const double* b2, const double* dy_in, double* y, double* loss, double* da,
                double* dwg, double* dw1, double* db1, double* dw2, double* db2, int* expert_out,
                int* slot_out, uint8_t* keep_out, double* logits_out, double* probs_out) {
  const int64_t N = (int64_t)S * n;
  double* logits = (double*)malloc(sizeof(double) * (size_t)(N * E));
  double* probs = (double*)malloc(sizeof(double) * (size_t)(N * E));
  double* chosen = (double*)malloc(sizeof(double) * (size_t)N);
  int* expert = (int*)malloc(sizeof(int) * (size_t)N);
  int* slot = (int*)malloc(sizeof(int) * (size_t)N);
  uint8_t* keep = (uint8_t*)malloc((size_t)N);
  double* fhome = (double*)calloc((size_t)(N * h), sizeof(double));
  o_gate_forward(a, wg, N, h, E, logits, expert, chosen, probs);
  const int64_t cap = o_capacity(cf, n, E);
  for (int s = 0; s < S; ++s) /* capacity is per source shard */
    o_route_capacity(expert + s * n, n, E, cap, 1, slot + s * n, keep + s * n, NULL);

  /* per-expert row lists, ascending global token order (moe.cpp:995-999) */
  int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N > 0 ? N : 1));
  int64_t* start = (int64_t*)calloc((size_t)E + 1, sizeof(int64_t));
  for (int64_t k = 0; k < N; ++k)
    if (keep[k]) start[expert[k] + 1]++;
  for (int e = 0; e < E; ++e) start[e + 1] += start[e];
  {
    int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)E);
    for (int e = 0; e < E; ++e) cur[e] = start[e];
    for (int64_t k = 0; k < N; ++k)
      if (keep[k]) rows[cur[expert[k]]++] = k;
    free(cur);
  }
  int64_t maxr = 1;
  for (int e = 0; e < E; ++e)
    if (start[e + 1] - start[e] > maxr) maxr = start[e + 1] - start[e];
  double* xe = (double*)malloc(sizeof(double) * (size_t)(maxr * h));
  double* z = (double*)malloc(sizeof(double) * (size_t)(maxr * f));
  double* hh = (double*)malloc(sizeof(double) * (size_t)(maxr * f));
  double* fe = (double*)malloc(sizeof(double) * (size_t)(maxr * h));

  for (int e = 0; e < E; ++e) { /* forward per expert */
    const int64_t r = start[e + 1] - start[e];
    if (r == 0) continue;
    for (int64_t i = 0; i < r; ++i)
      memcpy(xe + i * h, a + rows[start[e] + i] * h, sizeof(double) * h);
    mm_nn(xe, w1 + (int64_t)e * h * f, b1 + (int64_t)e * f, r, h, f, z);
    for (int64_t i = 0; i < r * f; ++i) hh[i] = o_gelu(z[i]);
    mm_nn(hh, w2 + (int64_t)e * f * h, b2 + (int64_t)e * h, r, f, h, fe);
    for (int64_t i = 0; i < r; ++i)
      memcpy(fhome + rows[start[e] + i] * h, fe + i * h, sizeof(double) * h);
  }
  /* combine y = p * f_home (moe.cpp:1010-1015); dropped tokens have f_home = 0 */
  double acc = 0.0;
  double* yy = y ? y : (double*)malloc(sizeof(double) * (size_t)(N * h));
  for (int64_t k = 0; k < N; ++k)
    for (int j = 0; j < h; ++j) {
      const double v = chosen[k] * fhome[k * h + j];
      yy[k * h + j] = v;
      acc += v * v;
    }
  if (loss) *loss = acc / (2.0 * (double)N);

  if (da || dwg || dw1 || dw2 || db1 || db2) {
    double* dy = (double*)malloc(sizeof(double) * (size_t)(N * h));
    for (int64_t i = 0; i < N * h; ++i) dy[i] = dy_in ? dy_in[i] : yy[i] / (double)N;
    double* dchosen = (double*)malloc(sizeof(double) * (size_t)N);
    for (int64_t k = 0; k < N; ++k) { /* moe.cpp:1037-1047 */
      double d = 0.0;
      for (int j = 0; j < h; ++j) d += fhome[k * h + j] * dy[k * h + j];
      dchosen[k] = d;
    }
    double* dinput = (double*)malloc(sizeof(double) * (size_t)(N * h));
    o_gate_backward(a, wg, probs, expert, dchosen, N, h, E, dwg, dinput);
    double* dfe = (double*)malloc(sizeof(double) * (size_t)(maxr * h));
    double* dh = (double*)malloc(sizeof(double) * (size_t)(maxr * f));
    double* dx = (double*)malloc(sizeof(double) * (size_t)(maxr * h));
    if (da) memcpy(da, dinput, sizeof(double) * (size_t)(N * h));
    if (dw1) memset(dw1, 0, sizeof(double) * (size_t)E * h * f);
    if (dw2) memset(dw2, 0, sizeof(double) * (size_t)E * f * h);
    if (db1) memset(db1, 0, sizeof(double) * (size_t)E * f);
    if (db2) memset(db2, 0, sizeof(double) * (size_t)E * h);
    for (int e = 0; e < E; ++e) {
      const int64_t r = start[e + 1] - start[e];
      if (r == 0) continue;
      for (int64_t i = 0; i < r; ++i) {
        const int64_t k = rows[start[e] + i];
        memcpy(xe + i * h, a + k * h, sizeof(double) * h);
        for (int j = 0; j < h; ++j) dfe[i * h + j] = chosen[k] * dy[k * h + j];
      }
      mm_nn(xe, w1 + (int64_t)e * h * f, b1 + (int64_t)e * f, r, h, f, z); /* recompute acts */
      for (int64_t i = 0; i < r * f; ++i) hh[i] = o_gelu(z[i]);
      /* row_parallel/linear_backward of W2 (nn.cpp:84-90) */
      if (dw2) mm_tn_acc(hh, dfe, r, f, h, dw2 + (int64_t)e * f * h);
      if (db2)
        for (int64_t i = 0; i < r; ++i)
          for (int j = 0; j < h; ++j) db2[(int64_t)e * h + j] += dfe[i * h + j];
      mm_nt(dfe, w2 + (int64_t)e * f * h, r, h, f, dh);
      for (int64_t i = 0; i < r * f; ++i) dh[i] *= o_gelu_grad(z[i]); /* gelu_backward */
      if (dw1) mm_tn_acc(xe, dh, r, h, f, dw1 + (int64_t)e * h * f);
      if (db1)
        for (int64_t i = 0; i < r; ++i)
          for (int j = 0; j < f; ++j) db1[(int64_t)e * f + j] += dh[i * f + j];
      if (da) {
        mm_nt(dh, w1 + (int64_t)e * h * f, r, f, h, dx);
        for (int64_t i = 0; i < r; ++i) {
          const int64_t k = rows[start[e] + i];
          for (int j = 0; j < h; ++j) da[k * h + j] += dx[i * h + j];
        }
      }
    }
    free(dy);
    free(dchosen);
    free(dinput);
    free(dfe);
    free(dh);
    free(dx);
  }
  if (expert_out) memcpy(expert_out, expert, sizeof(int) * (size_t)N);
  if (slot_out) memcpy(slot_out, slot, sizeof(int) * (size_t)N);
  if (keep_out) memcpy(keep_out, keep, (size_t)N);
  if (logits_out) memcpy(logits_out, logits, sizeof(double) * (size_t)(N * E));
  if (probs_out) memcpy(probs_out, probs, sizeof(double) * (size_t)(N * E));
  if (!y) free(yy);
  free(logits);
  free(probs);
  free(chosen);
  free(expert);
  free(slot);
  free(keep);
  free(fhome);
  free(rows);
  free(start);
  free(xe);
  free(z);
  free(hh);
  free(fe);
  return 0;
}

/* ---- ZeRO-1 shard range + tiled AdamW: optimizer.cpp:12-28, :58-104 --------- */

void o_shard_range(int64_t total, int parts, int index, int64_t* begin, int64_t* end) {
  const int64_t base = total / parts, extra = total % parts;
  const int64_t b = index * base + (index < extra ? index : extra);
  *begin = b;
  *end = b + base + (index < extra ? 1 : 0);
}

uint64_t o_adam_step_owned(int64_t begin, int64_t end, int64_t step, double lr, double b1,
                           double b2, double eps, double wd, int tiles_enabled,
                           int64_t tile_size, const double* grad_full, double* master,
                           double* m1, double* m2, double* out_full) {
  const double c1 = 1.0 - pow(b1, (double)step); /* steps_done already incremented */
  const double c2 = 1.0 - pow(b2, (double)step);
  const int64_t owned = end - begin;
  const int64_t one = owned > 1 ? owned : 1;
  const int64_t tile = tiles_enabled ? (tile_size < one ? tile_size : one) : one;
  for (int64_t at = 0; at < owned; at += tile) { /* tile walk; math is per element */
    const int64_t len = tile < owned - at ? tile : owned - at;
    for (int64_t i = 0; i < len; ++i) {
      const int64_t j = at + i;
      const double g = grad_full[begin + j];
      m1[j] = b1 * m1[j] + (1.0 - b1) * g;
      m2[j] = b2 * m2[j] + (1.0 - b2) * g * g;
      const double mhat = m1[j] / c1, vhat = m2[j] / c2;
      double p = master[j];
      p -= lr * (mhat / (sqrt(vhat) + eps) + wd * p);
      master[j] = p;
      if (out_full) out_full[begin + j] = p;
    }
  }
  return owned == 0 ? 0 : (uint64_t)tile * 4u;
}
