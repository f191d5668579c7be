/*
 * rtec_cpu.c -- CPU oracle port (C + OpenMP, f64) -- TEST / BASELINE INFRASTRUCTURE ONLY.
 *
 * A multithreaded restatement of the same algorithms as oracle/graph.py and
 * oracle/engine.py (which are pinned to the reference's own outputs), for
 * gcn / graphsage / gin, so the CPU baseline can run the benchmark's
 * configs[1]-scale workload with every host core:
 *   - DynamicGraph.apply_batch semantics (graph.py:184-231): validation
 *     (first offender in batch order: range -> InvalidVertex, repeated edge ->
 *     ConfigError), reject duplicate inserts / absent deletes, DegreeDelta rows;
 *     adjacency kept as immutable CSR snapshots rebuilt by per-vertex merge;
 *   - Alg. 4 frontier with the SURVEY §8(a)-F1 every-layer degree rule;
 *   - Alg. 1 per destination (un-normalised aggregate S kept resident, which
 *     is strip(ctx, a); compose applied on read), zero in-degree rule
 *     (SPEC.md:277), update relu(W a) / W2 relu(W (h + a)) (models.py:107, :187).
 * Only tests/ and bench.py's CPU leg load it (via oracle/cport.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { M_GCN = 0, M_SAGE = 1, M_GIN = 2 };

typedef struct {
  int64_t n, m;
  int64_t *optr, *iptr; /* [n+1] */
  int32_t *oidx, *iidx; /* [m] */
  int64_t *ots;         /* [m] */
} csr_t;

typedef struct {
  csr_t g;
  int32_t *out_deg, *in_deg, *out_prev, *in_prev;
  int model, L;
  double off;
  int dims[8];
  double *W[8], *W2[8];
  double *H[9];      /* H[0] = X, H[l+1] output of layer l */
  double *S[8];      /* un-normalised aggregates */
  double *log_[8];   /* DeltaLog rows of H[l+1] for V_dst(l), indexed by slot */
  int32_t *slot[8];  /* vertex -> DeltaLog row, -1 if not in V_dst(l) */
  uint8_t *vdst[8];  /* V_dst(l) flags of the last batch */
  int64_t nvdst[8], necurr[8];
} eng_t;

static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}
static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return x < y ? -1 : x > y;
}

/* ---------------- CSR build (graph.py:81-121) ---------------- */
static void csr_from(int64_t n, int64_t m, const int32_t* own, const int32_t* nb, const int64_t* ts, int64_t** ptr,
                     int32_t** idx, int64_t** tso) {
  int64_t* p = calloc(n + 1, sizeof(int64_t));
  for (int64_t i = 0; i < m; ++i) p[own[i] + 1]++;
  for (int64_t v = 0; v < n; ++v) p[v + 1] += p[v];
  int64_t* fill = malloc(sizeof(int64_t) * (n + 1));
  memcpy(fill, p, sizeof(int64_t) * (n + 1));
  int32_t* x = malloc(sizeof(int32_t) * (m ? m : 1));
  int64_t* order = malloc(sizeof(int64_t) * (m ? m : 1));
  for (int64_t i = 0; i < m; ++i) order[fill[own[i]]++] = i;
  int64_t* t = tso ? malloc(sizeof(int64_t) * (m ? m : 1)) : NULL;
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t v = 0; v < n; ++v) {
    int64_t b = p[v], e = p[v + 1];
    if (e - b == 1) {
      x[b] = nb[order[b]];
      if (t) t[b] = ts ? ts[order[b]] : order[b];
      continue;
    }
    if (e == b) continue;
    /* sort the run by neighbour (carry the original index for ts) */
    uint64_t* tmp = malloc(sizeof(uint64_t) * (e - b + 1));
    for (int64_t k = b; k < e; ++k) tmp[k - b] = ((uint64_t)(uint32_t)nb[order[k]] << 32) | (uint64_t)(k - b);
    qsort(tmp, e - b, sizeof(uint64_t), cmp_u64);
    for (int64_t k = b; k < e; ++k) {
      int64_t src = order[b + (int64_t)(tmp[k - b] & 0xffffffffu)];
      x[k] = nb[src];
      if (t) t[k] = ts ? ts[src] : src;
    }
    free(tmp);
  }
  free(fill);
  free(order);
  *ptr = p;
  *idx = x;
  if (tso) *tso = t;
}

static void csr_free(csr_t* g) {
  free(g->optr); free(g->iptr); free(g->oidx); free(g->iidx); free(g->ots);
}

/* ---------------- engine ---------------- */
static double coeff(const eng_t* e, int32_t deg) {
  return e->model == M_GCN ? 1.0 / sqrt((double)deg + e->off) : 1.0;
}

static void layer_update_row(const eng_t* e, int l, int64_t v, const double* a, double* out) {
  int din = e->dims[l], dout = e->dims[l + 1];
  const double* W = e->W[l];
  if (e->model == M_GIN) {
    double* x = malloc(sizeof(double) * (din + dout));
    double* hid = x + din;
    const double* h = e->H[l] + v * din;
    for (int k = 0; k < din; ++k) x[k] = h[k] + a[k];
    for (int o = 0; o < dout; ++o) {
      double s = 0;
      const double* w = W + (int64_t)o * din;
      for (int k = 0; k < din; ++k) s += w[k] * x[k];
      hid[o] = s > 0 ? s : 0;
    }
    const double* W2 = e->W2[l];
    for (int o = 0; o < dout; ++o) {
      double s = 0;
      const double* w = W2 + (int64_t)o * dout;
      for (int k = 0; k < dout; ++k) s += w[k] * hid[k];
      out[o] = s;
    }
    free(x);
    return;
  }
  for (int o = 0; o < dout; ++o) {
    double s = 0;
    const double* w = W + (int64_t)o * din;
    for (int k = 0; k < din; ++k) s += w[k] * a[k];
    out[o] = s > 0 ? s : 0;
  }
}

/* composed aggregate of v from S (ms_cbn, operators.py:135) */
static void compose_row(const eng_t* e, int l, int64_t v, int32_t indeg, const double* s, double* a) {
  int d = e->dims[l];
  double sc = 1.0;
  if (indeg > 0) {
    if (e->model == M_GCN) sc = 1.0 / sqrt((double)indeg + e->off);
    else if (e->model == M_SAGE) sc = 1.0 / (double)indeg;
  }
  for (int k = 0; k < d; ++k) a[k] = indeg > 0 ? s[k] * sc : 0.0;
}

static void layer_full(eng_t* e, int l) {
  int64_t n = e->g.n;
  int din = e->dims[l], dout = e->dims[l + 1];
#pragma omp parallel
  {
    double* a = malloc(sizeof(double) * din);
#pragma omp for schedule(dynamic, 256)
    for (int64_t v = 0; v < n; ++v) {
      double* s = e->S[l] + v * din;
      for (int k = 0; k < din; ++k) s[k] = 0;
      for (int64_t j = e->g.iptr[v]; j < e->g.iptr[v + 1]; ++j) {
        int32_t u = e->g.iidx[j];
        double c = coeff(e, e->out_deg[u]);
        const double* h = e->H[l] + (int64_t)u * din;
        for (int k = 0; k < din; ++k) s[k] += c * h[k];
      }
      int32_t indeg = (int32_t)(e->g.iptr[v + 1] - e->g.iptr[v]);
      compose_row(e, l, v, indeg, s, a);
      layer_update_row(e, l, v, a, e->H[l + 1] + v * dout);
    }
    free(a);
  }
}

eng_t* rc_create(int64_t n, int64_t m, const int32_t* src, const int32_t* dst, const int64_t* ts, int model, int L,
                 const int32_t* dims, const double* const* W, const double* const* W2, double degree_offset,
                 const double* X) {
  eng_t* e = calloc(1, sizeof(eng_t));
  e->g.n = n;
  e->g.m = m;
  csr_from(n, m, src, dst, ts, &e->g.optr, &e->g.oidx, &e->g.ots);
  csr_from(n, m, dst, src, NULL, &e->g.iptr, &e->g.iidx, NULL);
  e->out_deg = malloc(sizeof(int32_t) * n);
  e->in_deg = malloc(sizeof(int32_t) * n);
  for (int64_t v = 0; v < n; ++v) {
    e->out_deg[v] = (int32_t)(e->g.optr[v + 1] - e->g.optr[v]);
    e->in_deg[v] = (int32_t)(e->g.iptr[v + 1] - e->g.iptr[v]);
  }
  e->out_prev = malloc(sizeof(int32_t) * n);
  e->in_prev = malloc(sizeof(int32_t) * n);
  e->model = model;
  e->L = L;
  e->off = degree_offset;
  for (int l = 0; l <= L; ++l) e->dims[l] = dims[l];
  e->H[0] = malloc(sizeof(double) * n * dims[0]);
  memcpy(e->H[0], X, sizeof(double) * n * dims[0]);
  for (int l = 0; l < L; ++l) {
    int64_t wsz = (int64_t)dims[l + 1] * dims[l];
    e->W[l] = malloc(sizeof(double) * wsz);
    memcpy(e->W[l], W[l], sizeof(double) * wsz);
    if (model == M_GIN) {
      e->W2[l] = malloc(sizeof(double) * dims[l + 1] * dims[l + 1]);
      memcpy(e->W2[l], W2[l], sizeof(double) * dims[l + 1] * dims[l + 1]);
    }
    e->H[l + 1] = calloc((size_t)n * dims[l + 1], sizeof(double));
    e->S[l] = calloc((size_t)n * dims[l], sizeof(double));
    e->log_[l] = malloc(sizeof(double) * n * dims[l + 1]);
    e->slot[l] = malloc(sizeof(int32_t) * n);
    e->vdst[l] = calloc(n, 1);
  }
  for (int l = 0; l < L; ++l) layer_full(e, l);
  return e;
}

void rc_free(eng_t* e) {
  csr_free(&e->g);
  free(e->out_deg); free(e->in_deg); free(e->out_prev); free(e->in_prev);
  for (int l = 0; l <= e->L; ++l) free(e->H[l]);
  for (int l = 0; l < e->L; ++l) {
    free(e->W[l]); free(e->W2[l]); free(e->S[l]); free(e->log_[l]); free(e->slot[l]); free(e->vdst[l]);
  }
  free(e);
}

/* merge applied updates (sorted by (own, nb)) into a CSR direction -> new arrays */
static void csr_merge(int64_t n, const int64_t* ptr, const int32_t* idx, const int64_t* ts, int64_t K,
                      const int32_t* own, const int32_t* nb, const uint8_t* op, const int64_t* uts, int64_t** nptr,
                      int32_t** nidx, int64_t** nts) {
  int64_t* np = calloc(n + 1, sizeof(int64_t));
  int64_t* first = malloc(sizeof(int64_t) * n);
  for (int64_t v = 0; v < n; ++v) first[v] = -1;
  for (int64_t v = 0; v < n; ++v) np[v + 1] = ptr[v + 1] - ptr[v];
  for (int64_t k = 0; k < K; ++k) {
    np[own[k] + 1] += op[k] == 0 ? 1 : -1;
    if (first[own[k]] < 0) first[own[k]] = k;
  }
  for (int64_t v = 0; v < n; ++v) np[v + 1] += np[v];
  int64_t M = np[n];
  int32_t* ni = malloc(sizeof(int32_t) * (M ? M : 1));
  int64_t* nt = ts ? malloc(sizeof(int64_t) * (M ? M : 1)) : NULL;
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t v = 0; v < n; ++v) {
    int64_t b = ptr[v], e = ptr[v + 1], o = np[v];
    if (first[v] < 0) {
      memcpy(ni + o, idx + b, sizeof(int32_t) * (e - b));
      if (nt) memcpy(nt + o, ts + b, sizeof(int64_t) * (e - b));
      continue;
    }
    int64_t k = first[v];
    int64_t j = b;
    while (j < e || (k < K && own[k] == v)) {
      int take_old;
      if (k < K && own[k] == v && (j >= e || nb[k] <= idx[j])) {
        if (op[k] == 1) { /* delete: skip the matching old entry */
          if (j < e && idx[j] == nb[k]) ++j;
          ++k;
          continue;
        }
        take_old = 0;
      } else {
        take_old = 1;
      }
      if (take_old) {
        ni[o] = idx[j];
        if (nt) nt[o] = ts[j];
        ++j;
      } else {
        ni[o] = nb[k];
        if (nt) nt[o] = uts ? uts[k] : 0;
        ++k;
      }
      ++o;
    }
  }
  free(first);
  *nptr = np;
  *nidx = ni;
  if (nts) *nts = nt;
}

typedef struct {
  uint64_t key;
  int64_t pos;
} kp_t;
static int cmp_kp(const void* a, const void* b) {
  const kp_t *x = a, *y = b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->pos < y->pos ? -1 : x->pos > y->pos;
}

/* returns 0 ok, 1 InvalidVertex, 2 ConfigError; status[B]; deltas[k,5] (k <= 2B) */
int rc_step(eng_t* e, int64_t B, const uint8_t* op, const int32_t* src, const int32_t* dst, const int64_t* ts,
            uint8_t* status, int64_t* deltas, int64_t* n_delta) {
  int64_t n = e->g.n;
  if (B < 0 || B > ((int64_t)1 << 40)) return 2;
  /* ---- validation (graph.py:192-198) */
  int64_t first_bad = B, first_dup = B;
  kp_t* kp = malloc(sizeof(kp_t) * (B ? B : 1));
  for (int64_t i = 0; i < B; ++i) {
    int ok = src[i] >= 0 && src[i] < n && dst[i] >= 0 && dst[i] < n;
    if (!ok && first_bad == B) first_bad = i;
    kp[i].key = ok ? (uint64_t)src[i] * (uint64_t)n + (uint64_t)dst[i] : (uint64_t)n * (uint64_t)n + (uint64_t)i;
    kp[i].pos = i;
  }
  qsort(kp, B, sizeof(kp_t), cmp_kp);
  for (int64_t i = 1; i < B; ++i)
    if (kp[i].key == kp[i - 1].key && kp[i].key < (uint64_t)n * (uint64_t)n && kp[i].pos < first_dup)
      first_dup = kp[i].pos;
  if (first_bad < B || first_dup < B) {
    free(kp);
    return first_bad <= first_dup ? 1 : 2;
  }
  /* ---- probe + applied list in (src,dst) order */
  int32_t *as = malloc(4 * (B + 1)), *ad = malloc(4 * (B + 1));
  uint8_t* ao = malloc(B + 1);
  int64_t* at = malloc(8 * (B + 1));
  int64_t K = 0;
  for (int64_t j = 0; j < B; ++j) {
    int64_t i = kp[j].pos;
    int32_t s = src[i], d = dst[i];
    const int32_t* run = e->g.oidx + e->g.optr[s];
    int64_t lo = 0, hi = e->g.optr[s + 1] - e->g.optr[s];
    while (lo < hi) {
      int64_t mid = (lo + hi) / 2;
      if (run[mid] < d) lo = mid + 1; else hi = mid;
    }
    int exists = lo < e->g.optr[s + 1] - e->g.optr[s] && run[lo] == d;
    int applied = op[i] == 0 ? !exists : exists;
    status[i] = (uint8_t)applied;
    if (applied) { as[K] = s; ad[K] = d; ao[K] = op[i]; at[K] = ts[i]; ++K; }
  }
  free(kp);
  /* ---- degrees, deltas (graph.py:201-230) */
  memcpy(e->out_prev, e->out_deg, sizeof(int32_t) * n);
  memcpy(e->in_prev, e->in_deg, sizeof(int32_t) * n);
  for (int64_t k = 0; k < K; ++k) {
    int dlt = ao[k] == 0 ? 1 : -1;
    e->out_deg[as[k]] += dlt;
    e->in_deg[ad[k]] += dlt;
  }
  int32_t* tv = malloc(sizeof(int32_t) * (2 * K + 1));
  for (int64_t k = 0; k < K; ++k) { tv[2 * k] = as[k]; tv[2 * k + 1] = ad[k]; }
  qsort(tv, 2 * K, sizeof(int32_t), cmp_i32);
  int64_t nd = 0;
  for (int64_t k = 0; k < 2 * K; ++k) {
    if (k && tv[k] == tv[k - 1]) continue;
    int32_t v = tv[k];
    if (e->in_prev[v] != e->in_deg[v] || e->out_prev[v] != e->out_deg[v]) {
      int64_t* r = deltas + 5 * nd++;
      r[0] = v; r[1] = e->in_prev[v]; r[2] = e->in_deg[v]; r[3] = e->out_prev[v]; r[4] = e->out_deg[v];
    }
  }
  *n_delta = nd;
  free(tv);
  /* ---- new CSR snapshots */
  {
    int64_t *np, *nt; int32_t* ni;
    csr_merge(n, e->g.optr, e->g.oidx, e->g.ots, K, as, ad, ao, at, &np, &ni, &nt);
    free(e->g.optr); free(e->g.oidx); free(e->g.ots);
    e->g.optr = np; e->g.oidx = ni; e->g.ots = nt;
    /* in direction: sort applied by (dst, src) */
    kp_t* ik = malloc(sizeof(kp_t) * (K + 1));
    for (int64_t k = 0; k < K; ++k) { ik[k].key = (uint64_t)ad[k] * (uint64_t)n + (uint64_t)as[k]; ik[k].pos = k; }
    qsort(ik, K, sizeof(kp_t), cmp_kp);
    int32_t *is_ = malloc(4 * (K + 1)), *id_ = malloc(4 * (K + 1));
    uint8_t* io = malloc(K + 1);
    for (int64_t k = 0; k < K; ++k) { is_[k] = as[ik[k].pos]; id_[k] = ad[ik[k].pos]; io[k] = ao[ik[k].pos]; }
    int64_t* ip; int32_t* ii;
    csr_merge(n, e->g.iptr, e->g.iidx, NULL, K, id_, is_, io, NULL, &ip, &ii, NULL);
    free(e->g.iptr); free(e->g.iidx);
    e->g.iptr = ip; e->g.iidx = ii;
    e->g.m = np[n];
    free(ik); free(is_); free(id_); free(io);
  }
  /* ---- frontier + layers (Alg. 4 F1, Alg. 1) */
  uint8_t* S = calloc(n, 1);
  uint8_t* isins_src = NULL; (void)isins_src;
  if (e->model == M_GCN)
    for (int64_t k = 0; k < nd; ++k)
      if (deltas[5 * k + 3] != deltas[5 * k + 4]) S[deltas[5 * k]] = 1;
  /* inserted-edge test: applied inserts sorted by (src,dst) */
  int64_t nI = 0;
  uint64_t* ins = malloc(sizeof(uint64_t) * (K + 1));
  for (int64_t k = 0; k < K; ++k)
    if (ao[k] == 0) ins[nI++] = (uint64_t)as[k] * (uint64_t)n + (uint64_t)ad[k];
  /* applied updates grouped by dst */
  int64_t* dfirst = malloc(sizeof(int64_t) * n);
  int64_t* dnext = malloc(sizeof(int64_t) * (K + 1));
  for (int64_t v = 0; v < n; ++v) dfirst[v] = -1;
  for (int64_t k = K - 1; k >= 0; --k) { dnext[k] = dfirst[ad[k]]; dfirst[ad[k]] = k; }
  uint8_t* chg = NULL;
  for (int l = 0; l < e->L; ++l) {
    int din = e->dims[l], dout = e->dims[l + 1];
    if (chg) for (int64_t v = 0; v < n; ++v) S[v] |= chg[v];
    uint8_t* vd = e->vdst[l];
    memset(vd, 0, n);
    for (int64_t k = 0; k < K; ++k) vd[ad[k]] = 1;
    int64_t necurr = 0;
#pragma omp parallel for schedule(dynamic, 1024) reduction(+ : necurr)
    for (int64_t u = 0; u < n; ++u) {
      if (!S[u]) continue;
      for (int64_t j = e->g.optr[u]; j < e->g.optr[u + 1]; ++j) {
        __atomic_store_n(&vd[e->g.oidx[j]], 1, __ATOMIC_RELAXED);
        ++necurr;
      }
    }
    for (int64_t k = 0; k < K; ++k) {
      if (ao[k] == 1) necurr++;
      else if (!S[as[k]]) necurr++;
    }
    e->necurr[l] = necurr;
    /* δ rows for S (computed on the fly per edge below from H[l] and the previous DeltaLog) */
    const double* hold_log = l > 0 ? e->log_[l - 1] : NULL;
    const int32_t* hold_slot = l > 0 ? e->slot[l - 1] : NULL;
    const uint8_t* hold_chg = chg;
    /* slots for this layer's DeltaLog */
    int64_t ns = 0;
    for (int64_t v = 0; v < n; ++v) e->slot[l][v] = vd[v] ? (int32_t)ns++ : -1;
    e->nvdst[l] = ns;
#pragma omp parallel
    {
      double* acc = malloc(sizeof(double) * din);
      double* a = malloc(sizeof(double) * din);
      double* hn = malloc(sizeof(double) * dout);
#pragma omp for schedule(dynamic, 256)
      for (int64_t v = 0; v < n; ++v) {
        if (!vd[v]) continue;
        for (int k = 0; k < din; ++k) acc[k] = 0;
        /* ValueChange edges: (u,v) in G_post, u in S, not inserted */
        for (int64_t j = e->g.iptr[v]; j < e->g.iptr[v + 1]; ++j) {
          int32_t u = e->g.iidx[j];
          if (!S[u]) continue;
          uint64_t key = (uint64_t)u * (uint64_t)n + (uint64_t)v;
          int64_t lo = 0, hi = nI;
          while (lo < hi) { int64_t mid = (lo + hi) / 2; if (ins[mid] < key) lo = mid + 1; else hi = mid; }
          if (lo < nI && ins[lo] == key) continue;
          int32_t dn = e->out_deg[u], dp = e->out_prev[u];
          if (dn <= 0 || dp <= 0) continue;
          double cn = coeff(e, dn), co = coeff(e, dp);
          const double* h = e->H[l] + (int64_t)u * din;
          const double* ho = (hold_chg && hold_chg[u]) ? hold_log + (int64_t)hold_slot[u] * din : h;
          for (int k = 0; k < din; ++k) acc[k] += cn * h[k] - co * ho[k];
        }
        /* structural edges */
        for (int64_t k = dfirst[v]; k >= 0; k = dnext[k]) {
          int32_t u = as[k];
          if (ao[k] == 0) {
            double c = coeff(e, e->out_deg[u]);
            const double* h = e->H[l] + (int64_t)u * din;
            for (int q = 0; q < din; ++q) acc[q] += c * h[q];
          } else {
            double c = coeff(e, e->out_prev[u]);
            const double* h = e->H[l] + (int64_t)u * din;
            const double* ho = (hold_chg && hold_chg[u]) ? hold_log + (int64_t)hold_slot[u] * din : h;
            for (int q = 0; q < din; ++q) acc[q] -= c * ho[q];
          }
        }
        double* s = e->S[l] + v * din;
        int32_t indeg = e->in_deg[v];
        if (indeg == 0) for (int k = 0; k < din; ++k) s[k] = 0;
        else if (e->in_prev[v] == 0) for (int k = 0; k < din; ++k) s[k] = acc[k];
        else for (int k = 0; k < din; ++k) s[k] += acc[k];
        compose_row(e, l, v, indeg, s, a);
        layer_update_row(e, l, v, a, hn);
        double* hrow = e->H[l + 1] + v * dout;
        memcpy(e->log_[l] + (int64_t)e->slot[l][v] * dout, hrow, sizeof(double) * dout);
        memcpy(hrow, hn, sizeof(double) * dout);
      }
      free(acc); free(a); free(hn);
    }
    chg = vd;
  }
  free(S); free(ins); free(dfirst); free(dnext);
  free(as); free(ad); free(ao); free(at);
  return 0;
}

void rc_get_h(const eng_t* e, int l, double* out) {
  memcpy(out, e->H[l], sizeof(double) * e->g.n * e->dims[l]);
}
/* rows ids[0..k) of H[l] (kind 0, width dims[l]) or of the un-normalised aggregate S[l]
 * (kind 1, width dims[l]) -- the bench's sampled parity check */
void rc_get_rows(const eng_t* e, int kind, int l, const int64_t* ids, int64_t k, double* out) {
  const int d = e->dims[l];
  const double* src = kind == 0 ? e->H[l] : e->S[l];
  for (int64_t i = 0; i < k; ++i) memcpy(out + i * d, src + ids[i] * d, sizeof(double) * d);
}
int64_t rc_num_edges(const eng_t* e) { return e->g.m; }
void rc_frontier(const eng_t* e, int l, int64_t* n_vdst, int64_t* n_ecurr) {
  *n_vdst = e->nvdst[l];
  *n_ecurr = e->necurr[l];
}
int rc_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
