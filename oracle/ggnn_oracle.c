/*
 * ggnn_oracle.c -- CPU restatement of the GGNN hot path, used ONLY as a test
 * checker (tests/, __graft_entry__.smoke(), bench.py's cpu_baseline leg).
 * It is never linked into, or called by, the product library.
 *
 * Every function restates the reference implementation `graphann`
 * (/root/reference/pkg/src/graphann/_core.pyx) in plain C with the same
 * arithmetic: float32 inputs promoted to double, sequential double
 * accumulation, ties broken by ascending id.  The restatement is pinned
 * against the reference's own outputs by tests/golden/ (generated from the
 * compiled reference, see tests/golden/make_golden.py) in
 * tests/test_oracle.py.
 *
 * Differences from the reference are deliberate and semantic-free:
 *   - the per-call refcount / ever arrays are allocated here with calloc
 *     (the reference allocates numpy arrays, _core.pyx:326-327);
 *   - the `distinct` counter is computed from the same ever[] array.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define TERM_STOP 0
#define TERM_EMPTY 1
#define TERM_CAP 2

/* _core.pyx:30-37 : sequential double sum of (double)a - (double)b squared */
double ggo_sqdist(const float *a, const float *b, int64_t d) {
    double acc = 0.0;
    for (int64_t i = 0; i < d; ++i) {
        double diff = (double)a[i] - (double)b[i];
        acc += diff * diff;
    }
    return acc;
}

/* _core.pyx:58-67 : index of the first entry sorting strictly after (d, id) */
static int upper_pos(const double *dist, const int32_t *ids, int len, double d, int32_t id) {
    int lo = 0, hi = len;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (dist[mid] < d || (dist[mid] == d && ids[mid] <= id))
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

/* _core.pyx:70-83 : bounded sorted insert, returns the new length */
static int bounded_insert(double *dist, int32_t *ids, int len, int cap, double d, int32_t id) {
    int pos = upper_pos(dist, ids, len, d, id);
    if (len == cap) {
        if (pos == cap) return len;
        len -= 1;
    }
    memmove(dist + pos + 1, dist + pos, (size_t)(len - pos) * sizeof(double));
    memmove(ids + pos + 1, ids + pos, (size_t)(len - pos) * sizeof(int32_t));
    dist[pos] = d;
    ids[pos] = id;
    return len + 1;
}

/* _core.pyx:86-104 : exact top-k of q against all n rows of X, ties by row */
int ggo_exhaustive_topk(const float *X, int64_t n, int64_t d, const float *q, int k,
                        int32_t *out_ids, double *out_dists) {
    if (k > n) k = (int)n;
    int len = 0;
    for (int64_t i = 0; i < n; ++i) {
        double dv = ggo_sqdist(q, X + i * d, d);
        if (len < k || dv < out_dists[len - 1] ||
            (dv == out_dists[len - 1] && (int32_t)i < out_ids[len - 1]))
            len = bounded_insert(out_dists, out_ids, len, k, dv, (int32_t)i);
    }
    return len;
}

/* _core.pyx:107-130 : within-batch kNN, self excluded, ties by member position;
 * pos/dist are (m, k_nn), pre-filled here with -1 / +inf. */
void ggo_batch_bruteforce(const float *X, int64_t d, const int32_t *member_rows, int m,
                          int k_nn, int32_t *pos, double *dist) {
    for (int64_t i = 0; i < (int64_t)m * k_nn; ++i) {
        pos[i] = -1;
        dist[i] = INFINITY;
    }
    int k_eff = k_nn < m - 1 ? k_nn : m - 1;
    if (k_eff <= 0) return;
    for (int i = 0; i < m; ++i) {
        double *di = dist + (int64_t)i * k_nn;
        int32_t *pi = pos + (int64_t)i * k_nn;
        int len = 0;
        const float *xi = X + (int64_t)member_rows[i] * d;
        for (int j = 0; j < m; ++j) {
            if (j == i) continue;
            double dv = ggo_sqdist(xi, X + (int64_t)member_rows[j] * d, d);
            if (len < k_eff || dv < di[len - 1] || (dv == di[len - 1] && j < pi[len - 1]))
                len = bounded_insert(di, pi, len, k_eff, dv, j);
        }
    }
}

/* ---- the search cache (ring + visited ring + refcounts), _core.pyx:135-176 ---- */
typedef struct {
    int cap, len;
    double *rd;
    int32_t *rid;
    uint8_t *rvis;
    int vsize, vlen, vpos;
    int32_t *vring;
    uint8_t *cnt;  /* refcount over ring u visited ring, per node */
    uint8_t *ever; /* touched at least once during the call */
    long forgotten;
} cache_t;

static void vring_push(cache_t *c, int32_t node) {
    if (c->vlen == c->vsize) {
        int32_t old = c->vring[c->vpos];
        if (--c->cnt[old] == 0) c->forgotten++;
        c->vring[c->vpos] = node;
        c->vpos = (c->vpos + 1) % c->vsize;
    } else {
        c->vring[c->vlen++] = node;
    }
    c->cnt[node]++;
}

static void ring_insert(cache_t *c, double d, int32_t node) {
    int pos = upper_pos(c->rd, c->rid, c->len, d, node);
    if (c->len == c->cap) {
        if (pos == c->cap) { /* worse than the tail of a full ring */
            c->forgotten++;
            return;
        }
        int32_t tail = c->rid[c->cap - 1];
        if (c->rvis[c->cap - 1]) vring_push(c, tail);
        if (--c->cnt[tail] == 0) c->forgotten++;
    } else {
        c->len++;
    }
    for (int i = c->len - 1; i > pos; --i) {
        c->rd[i] = c->rd[i - 1];
        c->rid[i] = c->rid[i - 1];
        c->rvis[i] = c->rvis[i - 1];
    }
    c->rd[pos] = d;
    c->rid[pos] = node;
    c->rvis[pos] = 0;
    c->cnt[node]++;
}

/* counters layout: [visited_count, steps, term, distinct, forgotten] */
typedef struct {
    long visited, steps, distinct;
    int term;
} run_t;

/* _core.pyx:190-311 : the shared greedy loop.  target >= 0 selects found-target
 * mode (stop as soon as the target is admitted, expansion budget `budget`). */
static void greedy_core(const float *X, int64_t d, const int32_t *to_row, const int32_t *adj,
                        int k, int k_nn, const int32_t *sym_count, const float *q,
                        const int32_t *seed_ids, const double *seed_dists, int nseeds, int k_out,
                        double tau, double dmax, long max_iter, int32_t target, long budget,
                        cache_t *c, double *cand_d, int32_t *cand_id, run_t *st) {
    c->len = c->vlen = c->vpos = 0;
    c->forgotten = 0;
    st->visited = st->steps = st->distinct = 0;
    st->term = TERM_EMPTY;
    for (int i = 0; i < nseeds; ++i) {
        int32_t node = seed_ids[i];
        if (c->cnt[node] > 0) continue;
        ring_insert(c, seed_dists[i], node);
        if (!c->ever[node]) {
            c->ever[node] = 1;
            st->distinct++;
        }
    }
    for (;;) {
        int pos = -1;
        for (int i = 0; i < c->len; ++i)
            if (!c->rvis[i]) {
                pos = i;
                break;
            }
        if (pos < 0) {
            st->term = TERM_EMPTY;
            break;
        }
        double thr = INFINITY;
        if (c->len >= k_out) thr = c->rd[k_out - 1] + tau * fmin(dmax, c->rd[0]);
        if (c->rd[pos] > thr) {
            st->term = TERM_STOP;
            break;
        }
        if (target >= 0) {
            if (st->steps >= budget) {
                st->term = TERM_CAP;
                break;
            }
        } else if (st->steps >= max_iter) {
            st->term = TERM_CAP;
            break;
        }
        int32_t node = c->rid[pos];
        c->rvis[pos] = 1;
        vring_push(c, node);

        int m = 0;
        const int32_t *row = adj + (int64_t)node * k;
        int nslots = k_nn + sym_count[node];
        for (int j = 0; j < nslots; ++j) {
            int32_t nb = row[j];
            if (j < k_nn && nb < 0) continue; /* sym slots are trusted */
            if (c->cnt[nb] > 0) continue;
            int dup = 0;
            for (int i = 0; i < m; ++i)
                if (cand_id[i] == nb) {
                    dup = 1;
                    break;
                }
            if (dup) continue;
            cand_d[m] = ggo_sqdist(q, X + (int64_t)to_row[nb] * d, d);
            cand_id[m] = nb;
            m++;
            st->visited++;
            if (!c->ever[nb]) {
                c->ever[nb] = 1;
                st->distinct++;
            }
        }
        /* insertion sort by (dist, id), _core.pyx:286-296 */
        for (int i = 1; i < m; ++i) {
            double dv = cand_d[i];
            int32_t nb = cand_id[i];
            int j = i - 1;
            while (j >= 0 && (cand_d[j] > dv || (cand_d[j] == dv && cand_id[j] > nb))) {
                cand_d[j + 1] = cand_d[j];
                cand_id[j + 1] = cand_id[j];
                --j;
            }
            cand_d[j + 1] = dv;
            cand_id[j + 1] = nb;
        }
        int found = 0;
        for (int i = 0; i < m; ++i) {
            if (cand_d[i] <= thr) { /* frozen threshold, non-strict */
                ring_insert(c, cand_d[i], cand_id[i]);
                if (cand_id[i] == target) found = 1;
            } else {
                c->forgotten++;
            }
        }
        st->steps++;
        if (found) {
            st->term = 1;
            return;
        }
    }
    if (target >= 0) st->term = 0;
}

static int cache_alloc(cache_t *c, int cap, int vsize, int64_t node_count) {
    memset(c, 0, sizeof(*c));
    c->cap = cap;
    c->vsize = vsize;
    c->rd = (double *)malloc(sizeof(double) * (size_t)cap);
    c->rid = (int32_t *)malloc(sizeof(int32_t) * (size_t)cap);
    c->rvis = (uint8_t *)calloc((size_t)cap, 1);
    c->vring = (int32_t *)malloc(sizeof(int32_t) * (size_t)vsize);
    c->cnt = (uint8_t *)calloc((size_t)node_count, 1);
    c->ever = (uint8_t *)calloc((size_t)node_count, 1);
    return c->rd && c->rid && c->rvis && c->vring && c->cnt && c->ever ? 0 : -1;
}

static void cache_free(cache_t *c) {
    free(c->rd);
    free(c->rid);
    free(c->rvis);
    free(c->vring);
    free(c->cnt);
    free(c->ever);
}

/* _core.pyx:314-353 : returns the hit count; counters[5] as documented above. */
int ggo_greedy_search(const float *X, int64_t d, const int32_t *to_row, const int32_t *adj,
                      int64_t node_count, int k, int k_nn, const int32_t *sym_count,
                      const float *q, const int32_t *seed_ids, const double *seed_dists,
                      int nseeds, int k_out, double tau, double dmax, long max_iter,
                      int prioq_size, int visited_size, int32_t *out_ids, double *out_dists,
                      long *counters) {
    cache_t c;
    int cap = k_out + prioq_size;
    if (cache_alloc(&c, cap, visited_size, node_count)) {
        cache_free(&c);
        return -1;
    }
    double *cand_d = (double *)malloc(sizeof(double) * (size_t)k);
    int32_t *cand_id = (int32_t *)malloc(sizeof(int32_t) * (size_t)k);
    run_t st;
    greedy_core(X, d, to_row, adj, k, k_nn, sym_count, q, seed_ids, seed_dists, nseeds, k_out,
                tau, dmax, max_iter, -1, 0, &c, cand_d, cand_id, &st);
    int nh = c.len < k_out ? c.len : k_out;
    for (int i = 0; i < nh; ++i) {
        out_ids[i] = c.rid[i];
        out_dists[i] = c.rd[i];
    }
    counters[0] = st.visited;
    counters[1] = st.steps;
    counters[2] = st.term;
    counters[3] = st.distinct;
    counters[4] = c.forgotten;
    free(cand_d);
    free(cand_id);
    cache_free(&c);
    return nh;
}

/* _core.pyx:375-435 : reachability check of x from z.  Returns the verdict
 * (0 already linked, 1 reached, 2 link needed); fb[n_fallback] is filled with
 * the closest explored ids (excluding x and z), -1 padded. */
int ggo_sym_check_pair(const float *X, int64_t d, const int32_t *to_row, const int32_t *adj,
                       int64_t node_count, int k, int k_nn, const int32_t *sym_count, int32_t x,
                       int32_t z, double d_xz, double tau, double dmax, long budget, int k_out,
                       int prioq_size, int visited_size, int n_fallback, int32_t *fb) {
    for (int j = 0; j < n_fallback; ++j) fb[j] = -1;
    const int32_t *zr = adj + (int64_t)z * k;
    for (int j = 0; j < k_nn + sym_count[z]; ++j)
        if (zr[j] == x) return 0;
    cache_t c;
    if (cache_alloc(&c, k_out + prioq_size, visited_size, node_count)) {
        cache_free(&c);
        return -1;
    }
    double *cand_d = (double *)malloc(sizeof(double) * (size_t)k);
    int32_t *cand_id = (int32_t *)malloc(sizeof(int32_t) * (size_t)k);
    run_t st;
    double seed_d = d_xz;
    greedy_core(X, d, to_row, adj, k, k_nn, sym_count, X + (int64_t)to_row[x] * d, &z, &seed_d,
                1, k_out, tau, dmax, 0, x, budget, &c, cand_d, cand_id, &st);
    int verdict = st.term ? 1 : 2;
    if (verdict == 2) {
        int m = c.len < k_out ? c.len : k_out, w = 0;
        for (int j = 0; j < m && w < n_fallback; ++j) {
            int32_t node = c.rid[j];
            if (node != x && node != z) fb[w++] = node;
        }
    }
    free(cand_d);
    free(cand_id);
    cache_free(&c);
    return verdict;
}
