/* oracle/qtn_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never shipped).
 *
 * Plain-C restatement of the reference's bucket-elimination hot path:
 *   NaiveBackend::contract   proj/src/engine.cpp:68-108
 *   contract_bucket          proj/src/engine.cpp:160-169
 *   contract_network         proj/src/engine.cpp:246-304
 *   state-vector oracle      proj/src/statevector.cpp:25-84
 *
 * Rounding follows the reference's x86-64 -O3 build exactly: complex products
 * are (ac - bd, ad + bc) with every product rounded (no FMA; this file is
 * compiled with -ffp-contract=off), accumulation in ascending assignment
 * order.  Parity of this restatement is pinned against the unmodified
 * reference by tests/test_oracle.py (golden vectors in tests/golden/).
 */
#include "qtn_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[512];

const char* qo_last_error(void) { return g_err; }

static int set_err(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

typedef struct {
  int rank;
  int* vars;
  double* data; /* 2 << rank doubles */
} qo_tensor;

static int cmp_int(const void* a, const void* b) {
  const int x = *(const int*)a, y = *(const int*)b;
  return (x > y) - (x < y);
}

/* sorted unique union of the tensors' vars (network.cpp:9-16). */
static int union_vars(int nt, const qo_tensor* ts, int** out) {
  int total = 0;
  for (int t = 0; t < nt; ++t) total += ts[t].rank;
  int* v = (int*)malloc(sizeof(int) * (size_t)(total > 0 ? total : 1));
  int k = 0;
  for (int t = 0; t < nt; ++t)
    for (int a = 0; a < ts[t].rank; ++a) v[k++] = ts[t].vars[a];
  qsort(v, (size_t)k, sizeof(int), cmp_int);
  int u = 0;
  for (int i = 0; i < k; ++i)
    if (u == 0 || v[u - 1] != v[i]) v[u++] = v[i];
  *out = v;
  return u;
}

static int pos_in(const int* sorted, int n, int v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) / 2;
    if (sorted[mid] < v) lo = mid + 1; else hi = mid;
  }
  return (lo < n && sorted[lo] == v) ? lo : -1;
}

/* NaiveBackend::contract restated. On success fills *res (caller frees). */
static int naive_contract(int nt, const qo_tensor* ts, int n_sum, const int* sum_vars,
                          qo_tensor* res) {
  int* uniq = NULL;
  const int r = union_vars(nt, ts, &uniq);
  /* present_sum_vars (engine.cpp:28-36) */
  int* sums = (int*)malloc(sizeof(int) * (size_t)(n_sum > 0 ? n_sum : 1));
  int ns = 0;
  for (int i = 0; i < n_sum; ++i)
    if (pos_in(uniq, r, sum_vars[i]) >= 0) sums[ns++] = sum_vars[i];
  if (ns != n_sum) {
    free(uniq);
    free(sums);
    return set_err(QO_SCHEDULE, "bucket sums a variable absent from its tensors");
  }
  qsort(sums, (size_t)ns, sizeof(int), cmp_int);
  int* kept = (int*)malloc(sizeof(int) * (size_t)(r > 0 ? r : 1));
  int nk = 0;
  for (int i = 0; i < r; ++i)
    if (pos_in(sums, ns, uniq[i]) < 0) kept[nk++] = uniq[i];

  /* bit maps: assignment bit of union position i lives at shift r-1-i */
  int total_axes = 0;
  for (int t = 0; t < nt; ++t) total_axes += ts[t].rank;
  int* src = (int*)malloc(sizeof(int) * (size_t)(total_axes + 1));
  int* dst = (int*)malloc(sizeof(int) * (size_t)(total_axes + 1));
  int* first = (int*)malloc(sizeof(int) * (size_t)(nt + 1));
  int k = 0;
  for (int t = 0; t < nt; ++t) {
    first[t] = k;
    for (int ax = 0; ax < ts[t].rank; ++ax) {
      src[k] = r - 1 - pos_in(uniq, r, ts[t].vars[ax]);
      dst[k] = ts[t].rank - 1 - ax;
      ++k;
    }
  }
  first[nt] = k;
  int* ksrc = (int*)malloc(sizeof(int) * (size_t)(nk > 0 ? nk : 1));
  for (int ax = 0; ax < nk; ++ax) ksrc[ax] = r - 1 - pos_in(uniq, r, kept[ax]);

  const uint64_t nout = (uint64_t)1 << nk;
  double* acc = (double*)calloc((size_t)(2 * nout), sizeof(double));
  const uint64_t total = (uint64_t)1 << r;
  for (uint64_t a = 0; a < total; ++a) {
    double pr = 1.0, pi = 0.0;
    for (int t = 0; t < nt; ++t) {
      uint64_t off = 0;
      for (int j = first[t]; j < first[t + 1]; ++j) off |= ((a >> src[j]) & 1u) << dst[j];
      const double xr = ts[t].data[2 * off], xi = ts[t].data[2 * off + 1];
      const double nr = pr * xr - pi * xi;
      const double ni = pr * xi + pi * xr;
      pr = nr;
      pi = ni;
    }
    uint64_t koff = 0;
    for (int ax = 0; ax < nk; ++ax) koff |= ((a >> ksrc[ax]) & 1u) << (nk - 1 - ax);
    acc[2 * koff] += pr;
    acc[2 * koff + 1] += pi;
  }
  res->rank = nk;
  res->vars = kept;
  res->data = acc;
  free(uniq);
  free(sums);
  free(src);
  free(dst);
  free(first);
  free(ksrc);
  return QO_OK;
}

static int parse_tensors(int n_tensors, const int* ranks, const int* vars, const double* data,
                         qo_tensor* ts) {
  long vo = 0, dof = 0;
  for (int t = 0; t < n_tensors; ++t) {
    if (ranks[t] < 0 || ranks[t] > 40) return set_err(QO_INVALID, "bad tensor rank");
    ts[t].rank = ranks[t];
    ts[t].vars = (int*)(vars + vo);
    ts[t].data = (double*)(data + 2 * dof);
    vo += ranks[t];
    dof += 1L << ranks[t];
  }
  return QO_OK;
}

int qo_contract_bucket(int n_tensors, const int* ranks, const int* vars, const double* data,
                       int n_sum, const int* sum_vars, int* out_vars, double* out_data,
                       int64_t out_cap) {
  qo_tensor* ts = (qo_tensor*)calloc((size_t)(n_tensors > 0 ? n_tensors : 1), sizeof(qo_tensor));
  int st = parse_tensors(n_tensors, ranks, vars, data, ts);
  if (st != QO_OK) { free(ts); return -st; }
  qo_tensor res;
  st = naive_contract(n_tensors, ts, n_sum, sum_vars, &res);
  free(ts);
  if (st != QO_OK) return -st;
  const int64_t n = (int64_t)1 << res.rank;
  if (n > out_cap) {
    free(res.vars);
    free(res.data);
    return -set_err(QO_INVALID, "output buffer too small");
  }
  memcpy(out_vars, res.vars, sizeof(int) * (size_t)res.rank);
  memcpy(out_data, res.data, sizeof(double) * (size_t)(2 * n));
  const int rank = res.rank;
  free(res.vars);
  free(res.data);
  return rank;
}

/* ------------------------------------------------------------ network */

typedef struct {
  int n_sum;
  const int* sum_vars;
  int n, cap;
  qo_tensor* items; /* owned copies (results) or borrowed (initial) */
  unsigned char* owned;
} qo_bucket;

static void bucket_push(qo_bucket* b, qo_tensor t, int owned) {
  if (b->n == b->cap) {
    b->cap = b->cap ? 2 * b->cap : 4;
    b->items = (qo_tensor*)realloc(b->items, sizeof(qo_tensor) * (size_t)b->cap);
    b->owned = (unsigned char*)realloc(b->owned, (size_t)b->cap);
  }
  b->items[b->n] = t;
  b->owned[b->n] = (unsigned char)owned;
  ++b->n;
}

static void bucket_clear(qo_bucket* b) {
  for (int i = 0; i < b->n; ++i)
    if (b->owned[i]) {
      free(b->items[i].vars);
      free(b->items[i].data);
    }
  b->n = 0;
}

int qo_contract_network(int n_buckets, const int* ints, const double* data,
                        int max_result_width, double* scalar_re_im, int* rec_seq,
                        int* rec_width, int rec_cap, int* n_records, uint64_t* peak_bytes) {
  qo_bucket* bs = (qo_bucket*)calloc((size_t)(n_buckets > 0 ? n_buckets : 1), sizeof(qo_bucket));
  long ip = 0, dof = 0;
  int max_var = -1;
  for (int i = 0; i < n_buckets; ++i) {
    bs[i].n_sum = ints[ip++];
    bs[i].sum_vars = ints + ip;
    for (int s = 0; s < bs[i].n_sum; ++s)
      if (bs[i].sum_vars[s] > max_var) max_var = bs[i].sum_vars[s];
    ip += bs[i].n_sum;
    const int nt = ints[ip++];
    for (int t = 0; t < nt; ++t) {
      qo_tensor x;
      x.rank = ints[ip++];
      x.vars = (int*)(ints + ip);
      for (int a = 0; a < x.rank; ++a)
        if (x.vars[a] > max_var) max_var = x.vars[a];
      ip += x.rank;
      x.data = (double*)(data + 2 * dof);
      dof += 1L << x.rank;
      bucket_push(&bs[i], x, 0);
    }
  }
  /* sum_var_positions (engine.cpp:190-195): later buckets overwrite. */
  int* pos = (int*)malloc(sizeof(int) * (size_t)(max_var + 2));
  for (int v = 0; v <= max_var; ++v) pos[v] = -1;
  for (int i = 0; i < n_buckets; ++i)
    for (int s = 0; s < bs[i].n_sum; ++s) pos[bs[i].sum_vars[s]] = i;

  double sr = 1.0, si = 0.0;
  int nrec = 0;
  uint64_t peak = 0;
  int status = QO_OK;
  char msg[256];
  for (int i = 0; i < n_buckets && status == QO_OK; ++i) {
    qo_bucket* b = &bs[i];
    if (b->n == 0) continue;
    /* liveness check (engine.cpp:261-266) */
    for (int s = 0; s < b->n_sum && status == QO_OK; ++s)
      for (int j = i + 1; j < n_buckets && status == QO_OK; ++j)
        for (int t = 0; t < bs[j].n && status == QO_OK; ++t)
          for (int a = 0; a < bs[j].items[t].rank; ++a)
            if (bs[j].items[t].vars[a] == b->sum_vars[s]) {
              snprintf(msg, sizeof msg, "sum variable %d still live outside its bucket",
                       b->sum_vars[s]);
              status = set_err(QO_SCHEDULE, msg);
              break;
            }
    if (status != QO_OK) break;
    int* uniq = NULL;
    const int width = union_vars(b->n, b->items, &uniq);
    free(uniq);
    const int result_width = width - b->n_sum;
    if (result_width > max_result_width) {
      snprintf(msg, sizeof msg, "contraction refused: result width %d exceeds cap %d",
               result_width, max_result_width);
      status = set_err(QO_RESOURCE, msg);
      break;
    }
    qo_tensor res;
    status = naive_contract(b->n, b->items, b->n_sum, b->sum_vars, &res);
    if (status != QO_OK) break;
    if (nrec < rec_cap) {
      rec_seq[nrec] = i;
      rec_width[nrec] = width;
    }
    ++nrec;
    const uint64_t bytes = (uint64_t)16 << res.rank;
    if (bytes > peak) peak = bytes;
    bucket_clear(b);
    if (res.rank == 0) {
      const double xr = res.data[0], xi = res.data[1];
      const double nr = sr * xr - si * xi;
      const double ni = sr * xi + si * xr;
      sr = nr;
      si = ni;
      free(res.vars);
      free(res.data);
      continue;
    }
    int target = 0x7fffffff;
    for (int a = 0; a < res.rank; ++a) {
      const int v = res.vars[a];
      const int p = (v >= 0 && v <= max_var) ? pos[v] : -1;
      if (p < 0) {
        status = set_err(QO_SCHEDULE, "result variable not covered by the schedule");
        break;
      }
      if (p < target) target = p;
    }
    if (status == QO_OK && target <= i)
      status = set_err(QO_SCHEDULE, "result tensor flows backwards in the schedule");
    if (status != QO_OK) {
      free(res.vars);
      free(res.data);
      break;
    }
    bucket_push(&bs[target], res, 1);
  }
  for (int i = 0; i < n_buckets; ++i) {
    bucket_clear(&bs[i]);
    free(bs[i].items);
    free(bs[i].owned);
  }
  free(bs);
  free(pos);
  scalar_re_im[0] = sr;
  scalar_re_im[1] = si;
  *n_records = nrec;
  *peak_bytes = peak;
  return status;
}

/* ------------------------------------------------------------ statevector */

int qo_statevector_energy(int n, int m, const int* edges, int p, const double* gammas,
                          const double* betas, double* energy) {
  if (n < 1 || n > 26) return set_err(QO_RESOURCE, "state vector size out of range");
  const size_t dim = (size_t)1 << n;
  double* re = (double*)malloc(sizeof(double) * dim);
  double* im = (double*)malloc(sizeof(double) * dim);
  const double amp = 1.0 / sqrt((double)dim);
  for (size_t z = 0; z < dim; ++z) { re[z] = amp; im[z] = 0.0; }
  for (int k = 0; k < p; ++k) {
    /* apply_phase_zz: anti-aligned assignments pick up e^{-i gamma} */
    const double wr = cos(-gammas[k]), wi = sin(-gammas[k]);
    for (int e = 0; e < m; ++e) {
      const size_t m1 = (size_t)1 << (n - 1 - edges[2 * e]);
      const size_t m2 = (size_t)1 << (n - 1 - edges[2 * e + 1]);
      for (size_t z = 0; z < dim; ++z)
        if (((z & m1) != 0) != ((z & m2) != 0)) {
          const double a = re[z], b = im[z];
          re[z] = a * wr - b * wi;
          im[z] = a * wi + b * wr;
        }
    }
    /* apply_mixer_x: [[c, -is], [-is, c]] on each qubit */
    const double c = cos(betas[k]), s = sin(betas[k]);
    for (int q = 0; q < n; ++q) {
      const size_t mask = (size_t)1 << (n - 1 - q);
      for (size_t z = 0; z < dim; ++z) {
        if (z & mask) continue;
        const double ar = re[z], ai = im[z], br = re[z | mask], bi = im[z | mask];
        re[z] = c * ar + s * bi;
        im[z] = c * ai - s * br;
        re[z | mask] = s * ai + c * br;
        im[z | mask] = -s * ar + c * bi;
      }
    }
  }
  double sum = 0.0;
  for (int e = 0; e < m; ++e) {
    const size_t m1 = (size_t)1 << (n - 1 - edges[2 * e]);
    const size_t m2 = (size_t)1 << (n - 1 - edges[2 * e + 1]);
    double acc = 0.0;
    for (size_t z = 0; z < dim; ++z) {
      const double sign = (((z & m1) != 0) != ((z & m2) != 0)) ? -1.0 : 1.0;
      acc += sign * (re[z] * re[z] + im[z] * im[z]);
    }
    sum += acc;
  }
  *energy = 0.5 * (double)m - 0.5 * sum;
  free(re);
  free(im);
  return QO_OK;
}
