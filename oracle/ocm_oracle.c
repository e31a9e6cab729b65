/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle. Only tests/, the smoke check in
 * __graft_entry__.py and bench.py's cpu_baseline / reference legs may load
 * this library, and only as the checker. The product (paper_1111_0627_b200)
 * never links or calls it.
 *
 * Plain-C restatement of the reference's sequential policy iteration and its
 * supporting pieces, each function citing the reference file:line it
 * follows (paths relative to the reference's proj/ directory):
 *
 *   oc_build_csr         src/graph.cpp:23      build_graph (stable counting sort)
 *   oc_tarjan            src/scc.cpp:37        tarjan_scc (iterative low-link)
 *   improve_policy       include/ocm/howard.hpp:63
 *   find_policy_cycles   include/ocm/howard.hpp:105
 *   select_min_cycle     include/ocm/howard.hpp:145
 *   rebuild_policy       include/ocm/howard.hpp:163
 *   propagate_values     include/ocm/howard.hpp:232
 *   howard_region        include/ocm/howard.hpp:268  howard_solve
 *   oc_solve_howard      src/solve.cpp:43/117   run_howard_seq / solve()
 *   oc_dp_min_cycle_mean include/ocm/oracle.hpp:137 dp_min_cycle_mean
 *   oc_generate_model    src/model_gen.cpp:88  generate_model (state bound as a parameter)
 *   oc_generate_*        (no reference counterpart) the seeded synthetic
 *                        generators shared bit-for-bit with the CUDA library
 *
 * Parity pinning: tests/test_oracle_golden.py checks this file against golden
 * vectors produced by the reference library itself (oracle/_ref, built from
 * the reference sources by oracle/Makefile; generator tests/golden/make_golden.py).
 *
 * Arithmetic follows the reference's two modes (include/ocm/policy.hpp):
 * ExactMode keeps values as (wsum, steps) pairs compared by 128-bit cross
 * multiplication against lambda = num/den; FloatMode uses doubles with the
 * relative 1e-9 replacement band.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NONE32 0xffffffffu
#define NONE64 0xffffffffffffffffull

typedef struct {
    uint32_t n;
    uint64_t m;
    uint64_t *fidx;  /* n+1 */
    uint32_t *ftgt;  /* m */
    uint32_t *fsrc;  /* m */
    double *w;       /* m */
    uint64_t *bidx;  /* n+1 */
    uint32_t *bsrc;  /* m */
    uint64_t *bfe;   /* m: forward edge of each backward slot */
    int exact;
} oc_graph;

typedef struct {
    int32_t has_cycle;
    int32_t exact;
    int64_t mu_num;
    int64_t mu_den;
    double mu;
    uint32_t cycle_len;
    uint32_t outer_iters_seq;   /* run_howard_seq: sum over regions */
    uint32_t spf_passes_seq;
    uint32_t outer_iters_par;   /* howard-par lane: max over regions */
    uint32_t spf_passes_par;
    uint32_t regions;
    uint32_t trivial_regions;
} oc_result;

static int64_t gcd64(int64_t a, int64_t b) {
    if (a < 0) a = -a;
    while (b) { int64_t t = a % b; a = b; b = t; }
    return a;
}

/* Rational normalisation, include/ocm/rational.hpp:20. */
static void rat_norm(int64_t *num, int64_t *den) {
    if (*den < 0) { *num = -*num; *den = -*den; }
    int64_t g = gcd64(*num, *den);
    if (g > 1) { *num /= g; *den /= g; }
}

/* src/graph.cpp:23 build_graph: stable counting sort by source for the
 * forward CSR, then a stable pass over forward ids for the backward CSR. */
int oc_build_csr(oc_graph *g, uint32_t n, uint64_t m, const uint32_t *src, const uint32_t *dst,
                 const double *w) {
    memset(g, 0, sizeof *g);
    g->n = n;
    g->m = m;
    int exact = 1;
    for (uint64_t i = 0; i < m; ++i) {
        if (src[i] >= n || dst[i] >= n) return 1;
        if (!isfinite(w[i])) return 2;
        exact = exact && floor(w[i]) == w[i] && fabs(w[i]) < 9007199254740992.0;
    }
    g->exact = exact;
    g->fidx = calloc((size_t)n + 1, sizeof(uint64_t));
    g->bidx = calloc((size_t)n + 1, sizeof(uint64_t));
    g->ftgt = malloc((m ? m : 1) * sizeof(uint32_t));
    g->fsrc = malloc((m ? m : 1) * sizeof(uint32_t));
    g->w = malloc((m ? m : 1) * sizeof(double));
    g->bsrc = malloc((m ? m : 1) * sizeof(uint32_t));
    g->bfe = malloc((m ? m : 1) * sizeof(uint64_t));
    uint64_t *cur = malloc(((size_t)n + 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i < m; ++i) g->fidx[src[i] + 1]++;
    for (uint32_t v = 0; v < n; ++v) g->fidx[v + 1] += g->fidx[v];
    memcpy(cur, g->fidx, ((size_t)n + 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i < m; ++i) {
        uint64_t id = cur[src[i]]++;
        g->fsrc[id] = src[i];
        g->ftgt[id] = dst[i];
        g->w[id] = w[i];
    }
    for (uint64_t e = 0; e < m; ++e) g->bidx[g->ftgt[e] + 1]++;
    for (uint32_t v = 0; v < n; ++v) g->bidx[v + 1] += g->bidx[v];
    memcpy(cur, g->bidx, ((size_t)n + 1) * sizeof(uint64_t));
    for (uint64_t e = 0; e < m; ++e) {
        uint64_t s = cur[g->ftgt[e]]++;
        g->bsrc[s] = g->fsrc[e];
        g->bfe[s] = e;
    }
    free(cur);
    return 0;
}

void oc_free_csr(oc_graph *g) {
    free(g->fidx); free(g->ftgt); free(g->fsrc); free(g->w);
    free(g->bidx); free(g->bsrc); free(g->bfe);
    memset(g, 0, sizeof *g);
}

/* src/scc.cpp:37 tarjan_scc, iterative; region ids in completion order.
 * Returns region count; fills region_of. */
static uint32_t oc_tarjan(const oc_graph *g, uint32_t *region_of) {
    uint32_t n = g->n, count = 0, next_index = 1;
    uint32_t *index = calloc(n ? n : 1, sizeof(uint32_t));
    uint32_t *low = calloc(n ? n : 1, sizeof(uint32_t));
    char *on = calloc(n ? n : 1, 1);
    uint32_t *stack = malloc((n ? n : 1) * sizeof(uint32_t));
    uint32_t *cv = malloc((n ? n : 1) * sizeof(uint32_t));
    uint64_t *ce = malloc((n ? n : 1) * sizeof(uint64_t));
    size_t sp = 0, cp = 0;
    for (uint32_t v = 0; v < n; ++v) region_of[v] = NONE32;
    for (uint32_t root = 0; root < n; ++root) {
        if (index[root]) continue;
        cv[cp] = root; ce[cp] = g->fidx[root]; cp++;
        index[root] = low[root] = next_index++;
        stack[sp++] = root; on[root] = 1;
        while (cp) {
            uint32_t fv = cv[cp - 1];
            if (ce[cp - 1] != g->fidx[fv + 1]) {
                uint32_t t = g->ftgt[ce[cp - 1]++];
                if (!index[t]) {
                    cv[cp] = t; ce[cp] = g->fidx[t]; cp++;
                    index[t] = low[t] = next_index++;
                    stack[sp++] = t; on[t] = 1;
                } else if (on[t] && index[t] < low[fv]) {
                    low[fv] = index[t];
                }
                continue;
            }
            if (low[fv] == index[fv]) {
                uint32_t r = count++, x;
                do { x = stack[--sp]; on[x] = 0; region_of[x] = r; } while (x != fv);
            }
            cp--;
            if (cp) {
                uint32_t p = cv[cp - 1];
                if (low[fv] < low[p]) low[p] = low[fv];
            }
        }
    }
    free(index); free(low); free(on); free(stack); free(cv); free(ce);
    return count;
}

/* ---------------- policy iteration over one region ---------------- */

typedef struct {
    const oc_graph *g;
    const uint32_t *region_of;
    uint32_t region;
    const uint32_t *members; /* ascending */
    uint32_t cnt;
    int exact;
    /* state (global-sized arrays, only members touched) */
    uint64_t *succ;
    int64_t *ws[2], *st[2]; /* exact planes */
    double *fv[2];          /* float planes */
    int64_t lnum, lden;     /* exact lambda */
    double lf;              /* float lambda */
    int parity;
    char *conn;
    uint32_t *queue;
} region_ctx;

#define INR(c, v) ((c)->region_of[v] == (c)->region)

static int64_t wint(const oc_graph *g, uint64_t e) { return (int64_t)g->w[e]; }

/* ExactMode::compare, include/ocm/policy.hpp:73 */
static int cmp_exact(int64_t aw, int64_t as, int64_t bw, int64_t bs, int64_t num, int64_t den) {
    __int128 lhs = (__int128)(aw - bw) * den;
    __int128 rhs = (__int128)(as - bs) * num;
    return lhs < rhs ? -1 : (lhs > rhs ? 1 : 0);
}

/* FloatMode::strictly_better, include/ocm/policy.hpp:116 */
static int better_float(double cand, double inc) {
    double m = 1.0, a = fabs(cand), b = fabs(inc);
    if (a > m) m = a;
    if (b > m) m = b;
    return cand < inc - 1e-9 * m;
}

/* include/ocm/howard.hpp:63 improve_policy; returns whether any edge changed. */
static int improve_policy(region_ctx *c) {
    const oc_graph *g = c->g;
    int improved = 0, rd = c->parity, wr = c->parity ^ 1;
    for (uint32_t i = 0; i < c->cnt; ++i) {
        uint32_t v = c->members[i];
        uint64_t best_e = NONE64;
        int64_t bw = 0, bs = 0;
        double bf = 0;
        for (uint64_t e = g->fidx[v]; e < g->fidx[v + 1]; ++e) {
            uint32_t t = g->ftgt[e];
            if (!INR(c, t)) continue;
            if (c->exact) {
                int64_t cw = c->ws[rd][t] + wint(g, e), cs = c->st[rd][t] + 1;
                if (best_e == NONE64 || cmp_exact(cw, cs, bw, bs, c->lnum, c->lden) < 0) {
                    bw = cw; bs = cs; best_e = e;
                }
            } else {
                double cf = c->fv[rd][t] + g->w[e] - c->lf;
                if (best_e == NONE64 || cf < bf) { bf = cf; best_e = e; }
            }
        }
        if (best_e == NONE64) return -1; /* structural error */
        uint64_t cur = c->succ[v];
        if (c->exact) {
            c->ws[wr][v] = bw; c->st[wr][v] = bs;
        } else {
            c->fv[wr][v] = bf;
        }
        if (cur == NONE64) {
            c->succ[v] = best_e; improved = 1;
        } else if (c->exact) {
            uint32_t t = g->ftgt[cur];
            int64_t cw = c->ws[rd][t] + wint(g, cur), cs = c->st[rd][t] + 1;
            if (cmp_exact(bw, bs, cw, cs, c->lnum, c->lden) < 0) { c->succ[v] = best_e; improved = 1; }
        } else {
            double cf = c->fv[rd][g->ftgt[cur]] + g->w[cur] - c->lf;
            if (better_float(bf, cf)) { c->succ[v] = best_e; improved = 1; }
        }
    }
    return improved;
}

typedef struct {
    uint32_t anchor, length;
    int64_t wi;   /* exact weight sum */
    double wf;    /* float weight sum */
    int64_t num, den; /* exact mean (normalised) */
    double mean;
} cyc_rec;

static int rec_less(const cyc_rec *a, const cyc_rec *b, int exact) {
    if (exact) {
        __int128 l = (__int128)a->num * b->den, r = (__int128)b->num * a->den;
        if (l < r) return 1;
        if (l > r) return 0;
    } else {
        if (a->mean < b->mean) return 1;
        if (b->mean < a->mean) return 0;
    }
    return a->anchor < b->anchor;
}

#define SUCCV(c, v) ((c)->g->ftgt[(c)->succ[v]])

/* include/ocm/howard.hpp:105 find_policy_cycles + :145 select_min_cycle. */
static cyc_rec find_min_cycle(region_ctx *c, uint32_t *color) {
    cyc_rec best;
    int have = 0;
    memset(&best, 0, sizeof best);
    for (uint32_t i = 0; i < c->cnt; ++i) color[c->members[i]] = 0;
    for (uint32_t i = 0; i < c->cnt; ++i) {
        uint32_t s = c->members[i];
        if (color[s]) continue;
        uint32_t mark = s + 2, u = s;
        while (color[u] == 0) { color[u] = mark; u = SUCCV(c, u); }
        if (color[u] == mark) {
            cyc_rec r;
            memset(&r, 0, sizeof r);
            r.anchor = u;
            for (uint32_t w = SUCCV(c, u); w != u; w = SUCCV(c, w))
                if (w < r.anchor) r.anchor = w;
            uint32_t w = r.anchor;
            do {
                uint64_t e = c->succ[w];
                r.wi += c->exact ? wint(c->g, e) : 0;
                r.wf += c->g->w[e];
                r.length++;
                w = c->g->ftgt[e];
            } while (w != r.anchor);
            if (c->exact) {
                r.num = r.wi; r.den = r.length; rat_norm(&r.num, &r.den);
                r.mean = (double)r.num / (double)r.den;
            } else {
                r.mean = r.wf / r.length;
            }
            if (!have || rec_less(&r, &best, c->exact)) { best = r; have = 1; }
        }
        for (uint32_t w = s; color[w] == mark; w = SUCCV(c, w)) color[w] = 1;
    }
    return best;
}

/* include/ocm/howard.hpp:163 rebuild_policy. */
static int rebuild_policy(region_ctx *c, uint32_t anchor) {
    const oc_graph *g = c->g;
    for (uint32_t i = 0; i < c->cnt; ++i) c->conn[c->members[i]] = 0;
    size_t qn = 0;
    uint32_t u = anchor;
    do { c->conn[u] = 1; c->queue[qn++] = u; u = SUCCV(c, u); } while (u != anchor);
    for (size_t qi = 0; qi < qn; ++qi) {
        uint32_t v = c->queue[qi];
        for (uint64_t s = g->bidx[v]; s < g->bidx[v + 1]; ++s) {
            uint32_t x = g->bsrc[s];
            if (!INR(c, x) || c->conn[x]) continue;
            if (c->succ[x] == g->bfe[s]) { c->conn[x] = 1; c->queue[qn++] = x; }
        }
    }
    size_t remaining = c->cnt - qn;
    uint32_t *lv = malloc((c->cnt ? c->cnt : 1) * sizeof(uint32_t));
    uint64_t *le = malloc((c->cnt ? c->cnt : 1) * sizeof(uint64_t));
    while (remaining) {
        size_t ln = 0;
        for (uint32_t i = 0; i < c->cnt; ++i) {
            uint32_t v = c->members[i];
            if (c->conn[v]) continue;
            for (uint64_t e = g->fidx[v]; e < g->fidx[v + 1]; ++e) {
                uint32_t t = g->ftgt[e];
                if (INR(c, t) && c->conn[t]) { lv[ln] = v; le[ln] = e; ln++; break; }
            }
        }
        if (!ln) { free(lv); free(le); return -1; }
        for (size_t k = 0; k < ln; ++k) { c->succ[lv[k]] = le[k]; c->conn[lv[k]] = 1; }
        remaining -= ln;
    }
    free(lv); free(le);
    return 0;
}

/* include/ocm/howard.hpp:232 propagate_values (backward BFS from the anchor). */
static void propagate_values(region_ctx *c, uint32_t anchor) {
    const oc_graph *g = c->g;
    int p = c->parity;
    if (c->exact) { c->ws[p][anchor] = 0; c->st[p][anchor] = 0; }
    else c->fv[p][anchor] = 0.0;
    size_t qn = 0;
    c->queue[qn++] = anchor;
    for (size_t qi = 0; qi < qn; ++qi) {
        uint32_t v = c->queue[qi];
        for (uint64_t s = g->bidx[v]; s < g->bidx[v + 1]; ++s) {
            uint32_t u = g->bsrc[s];
            if (!INR(c, u) || u == anchor) continue;
            uint64_t e = g->bfe[s];
            if (c->succ[u] != e) continue;
            if (c->exact) { c->ws[p][u] = c->ws[p][v] + wint(g, e); c->st[p][u] = c->st[p][v] + 1; }
            else c->fv[p][u] = c->fv[p][v] + g->w[e] - c->lf;
            c->queue[qn++] = u;
        }
    }
}

/* include/ocm/howard.hpp:268 howard_solve restricted to one region.
 * Returns improvement passes (>0) or -1 on structural error. */
static int howard_region(region_ctx *c, cyc_rec *out_rec, uint32_t *color, uint32_t *outer) {
    int passes = 0;
    *outer = 0;
    c->parity = 0;
    c->lnum = 0; c->lden = 1; c->lf = 0.0;
    for (;;) {
        int imp = improve_policy(c);
        if (imp < 0) return -1;
        passes++;
        if (!imp) break;
        (*outer)++;
        c->parity ^= 1;
        cyc_rec r = find_min_cycle(c, color);
        if (c->exact) { c->lnum = r.num; c->lden = r.den; }
        else c->lf = r.mean;
        if (rebuild_policy(c, r.anchor) < 0) return -1;
        propagate_values(c, r.anchor);
        *out_rec = r;
    }
    return passes;
}

/* src/graph.cpp:105 augment_hamiltonian (big_w = 2n(max|w|+1)+1). */
static void hamiltonian_edges(uint32_t n, uint64_t m, const uint32_t *src, const uint32_t *dst,
                              const double *w, uint32_t **s2, uint32_t **d2, double **w2,
                              double *no_cycle_above) {
    double max_abs = 0.0;
    for (uint64_t i = 0; i < m; ++i) if (fabs(w[i]) > max_abs) max_abs = fabs(w[i]);
    double big = 2.0 * (double)n * (max_abs + 1.0) + 1.0;
    *s2 = malloc((m + n) * sizeof(uint32_t));
    *d2 = malloc((m + n) * sizeof(uint32_t));
    *w2 = malloc((m + n) * sizeof(double));
    memcpy(*s2, src, m * sizeof(uint32_t));
    memcpy(*d2, dst, m * sizeof(uint32_t));
    memcpy(*w2, w, m * sizeof(double));
    for (uint32_t v = 0; v < n; ++v) {
        (*s2)[m + v] = v; (*d2)[m + v] = (v + 1) % n; (*w2)[m + v] = big;
    }
    *no_cycle_above = max_abs;
}

/*
 * src/solve.cpp:198 solve() -> run_howard_seq (src/solve.cpp:43).
 * objective: 0 min, 1 max (weights negated, answer negated back).
 * scc_off: 1 = Hamiltonian augmentation instead of Tarjan regions.
 * Optional outputs (may be NULL): cycle_buf (cap entries), final value plane
 * (exact: wsum/steps, float: fval), per-vertex region lambda, succ_vertex.
 * Returns 0, or 1 bad input, 3 structural error.
 */
int oc_solve_howard(uint32_t n, uint64_t m, const uint32_t *src, const uint32_t *dst,
                    const double *w_in, int objective, int scc_off, oc_result *res,
                    uint32_t *cycle_buf, uint32_t cap, int64_t *out_wsum, int64_t *out_steps,
                    double *out_fval, int64_t *out_lnum, int64_t *out_lden, double *out_lf,
                    uint32_t *out_succv) {
    memset(res, 0, sizeof *res);
    if (n == 0) return 0;
    double *w = malloc((m ? m : 1) * sizeof(double));
    for (uint64_t i = 0; i < m; ++i) w[i] = objective ? -w_in[i] : w_in[i];
    uint32_t *s2 = (uint32_t *)src, *d2 = (uint32_t *)dst;
    double *w2 = w;
    uint64_t m2 = m;
    double nca = 0.0;
    if (scc_off) {
        hamiltonian_edges(n, m, src, dst, w, &s2, &d2, &w2, &nca);
        m2 = m + n;
    }
    oc_graph g;
    int rc = oc_build_csr(&g, n, m2, s2, d2, w2);
    if (rc) { if (scc_off) { free(s2); free(d2); free(w2); } free(w); oc_free_csr(&g); return 1; }
    uint32_t *region_of = malloc(n * sizeof(uint32_t));
    uint32_t rcount;
    if (scc_off) { for (uint32_t v = 0; v < n; ++v) region_of[v] = 0; rcount = 1; }
    else rcount = oc_tarjan(&g, region_of);
    /* members grouped by region, ascending within (RegionMap::finalize). */
    uint64_t *roff = calloc((size_t)rcount + 1, sizeof(uint64_t));
    uint32_t *mem = malloc(n * sizeof(uint32_t));
    for (uint32_t v = 0; v < n; ++v) roff[region_of[v] + 1]++;
    for (uint32_t r = 0; r < rcount; ++r) roff[r + 1] += roff[r];
    uint64_t *cur = malloc(((size_t)rcount + 1) * sizeof(uint64_t));
    memcpy(cur, roff, ((size_t)rcount + 1) * sizeof(uint64_t));
    for (uint32_t v = 0; v < n; ++v) mem[cur[region_of[v]]++] = v;
    free(cur);

    region_ctx c;
    memset(&c, 0, sizeof c);
    c.g = &g;
    c.region_of = region_of;
    c.exact = g.exact;
    c.succ = malloc(n * sizeof(uint64_t));
    for (int p = 0; p < 2; ++p) {
        c.ws[p] = calloc(n, sizeof(int64_t));
        c.st[p] = calloc(n, sizeof(int64_t));
        c.fv[p] = calloc(n, sizeof(double));
    }
    c.conn = calloc(n, 1);
    c.queue = malloc(n * sizeof(uint32_t));
    uint32_t *color = calloc(n, sizeof(uint32_t));
    for (uint32_t v = 0; v < n; ++v) c.succ[v] = NONE64;
    /* final plane per vertex is plane[parity_of_its_region] */
    int *final_parity = calloc(rcount ? rcount : 1, sizeof(int));
    int64_t *rl_num = calloc(rcount ? rcount : 1, sizeof(int64_t));
    int64_t *rl_den = calloc(rcount ? rcount : 1, sizeof(int64_t));
    double *rl_f = calloc(rcount ? rcount : 1, sizeof(double));

    res->exact = g.exact;
    res->regions = rcount;
    cyc_rec best;
    int found = 0, err = 0;
    memset(&best, 0, sizeof best);
    for (uint32_t r = 0; r < rcount; ++r) {
        rl_den[r] = 1;
        uint32_t cnt = (uint32_t)(roff[r + 1] - roff[r]);
        const uint32_t *members = mem + roff[r];
        int trivial = 0;
        if (!scc_off && cnt == 1) {
            uint32_t v = members[0];
            trivial = 1;
            for (uint64_t e = g.fidx[v]; e < g.fidx[v + 1]; ++e) if (g.ftgt[e] == v) trivial = 0;
        }
        if (trivial) { res->trivial_regions++; continue; }
        c.region = r;
        c.members = members;
        c.cnt = cnt;
        cyc_rec rec;
        uint32_t outer = 0;
        int passes = howard_region(&c, &rec, color, &outer);
        if (passes < 0 || outer == 0) { err = 1; break; }
        res->outer_iters_seq += outer;
        res->spf_passes_seq += (uint32_t)passes;
        if ((uint32_t)passes > res->spf_passes_par) res->spf_passes_par = (uint32_t)passes;
        final_parity[r] = c.parity;
        rl_num[r] = c.lnum; rl_den[r] = c.lden; rl_f[r] = c.lf;
        if (!found || rec_less(&rec, &best, g.exact)) { best = rec; found = 1; }
    }
    res->outer_iters_par = res->spf_passes_par ? res->spf_passes_par - 1 : 0;
    if (!err && found) {
        int acyclic = 0;
        if (scc_off) {
            if (g.exact) acyclic = (__int128)(int64_t)nca * best.den < (__int128)best.num;
            else acyclic = nca < best.mean;
        }
        if (!acyclic) {
            res->has_cycle = 1;
            res->mu_num = objective ? -best.num : best.num;
            res->mu_den = best.den;
            res->mu = objective ? -best.mean : best.mean;
            if (!g.exact) { res->mu_num = 0; res->mu_den = 1; }
            /* cycle vertices from the anchor along the final policy
             * (howard.hpp:251 cycle_vertices_of) */
            uint32_t u = best.anchor, len = 0;
            do {
                if (cycle_buf && len < cap) cycle_buf[len] = u;
                len++;
                u = g.ftgt[c.succ[u]];
            } while (u != best.anchor);
            res->cycle_len = len;
        }
    }
    if (!err) {
        for (uint32_t v = 0; v < n; ++v) {
            uint32_t r = region_of[v];
            int p = final_parity[r];
            if (out_wsum) out_wsum[v] = c.ws[p][v];
            if (out_steps) out_steps[v] = c.st[p][v];
            if (out_fval) out_fval[v] = c.fv[p][v];
            if (out_lnum) out_lnum[v] = rl_num[r];
            if (out_lden) out_lden[v] = rl_den[r];
            if (out_lf) out_lf[v] = rl_f[r];
            if (out_succv) out_succv[v] = c.succ[v] == NONE64 ? NONE32 : g.ftgt[c.succ[v]];
        }
    }
    free(final_parity); free(rl_num); free(rl_den); free(rl_f);
    free(color); free(c.queue); free(c.conn); free(c.succ);
    for (int p = 0; p < 2; ++p) { free(c.ws[p]); free(c.st[p]); free(c.fv[p]); }
    free(mem); free(roff); free(region_of);
    oc_free_csr(&g);
    if (scc_off) { free(s2); free(d2); free(w2); }
    free(w);
    return err ? 3 : 0;
}

/* include/ocm/oracle.hpp:137 dp_min_cycle_mean (walk-length DP, exact on
 * integer weights). Returns 0 ok (has_cycle set), 1 refused (n > 2000). */
int oc_dp_min_cycle_mean(uint32_t n, uint64_t m, const uint32_t *src, const uint32_t *dst,
                         const double *w, int32_t *has_cycle, int32_t *exact, int64_t *num,
                         int64_t *den, double *mean) {
    *has_cycle = 0;
    if (n > 2000) return 1;
    oc_graph g;
    if (oc_build_csr(&g, n, m, src, dst, w)) { oc_free_csr(&g); return 2; }
    *exact = g.exact;
    if (n == 0) { oc_free_csr(&g); return 0; }
    size_t N = n;
    if (g.exact) {
        const int64_t INF = INT64_MAX;
        int64_t *t = malloc((N + 1) * N * sizeof(int64_t));
        for (size_t i = 0; i < (N + 1) * N; ++i) t[i] = INF;
        for (size_t v = 0; v < N; ++v) t[v] = 0;
        for (size_t k = 1; k <= N; ++k) {
            const int64_t *pr = t + (k - 1) * N;
            int64_t *row = t + k * N;
            for (uint32_t v = 0; v < n; ++v) {
                int64_t b = INF;
                for (uint64_t s = g.bidx[v]; s < g.bidx[v + 1]; ++s) {
                    int64_t pw = pr[g.bsrc[s]];
                    if (pw == INF) continue;
                    int64_t cnd = pw + (int64_t)g.w[g.bfe[s]];
                    if (cnd < b) b = cnd;
                }
                row[v] = b;
            }
        }
        const int64_t *last = t + N * N;
        int found = 0;
        int64_t bn = 0, bd = 1;
        for (uint32_t v = 0; v < n; ++v) {
            if (last[v] == INF) continue;
            int any = 0;
            int64_t vn = 0, vd = 1;
            for (size_t j = 0; j < N; ++j) {
                int64_t ej = t[j * N + v];
                if (ej == INF) continue;
                int64_t cn = last[v] - ej, cd = (int64_t)(N - j);
                rat_norm(&cn, &cd);
                if (!any || (__int128)vn * cd < (__int128)cn * vd) { vn = cn; vd = cd; any = 1; }
            }
            if (any && (!found || (__int128)vn * bd < (__int128)bn * vd)) { bn = vn; bd = vd; found = 1; }
        }
        free(t);
        *has_cycle = found;
        if (found) { *num = bn; *den = bd; *mean = (double)bn / (double)bd; }
    } else {
        double *t = malloc((N + 1) * N * sizeof(double));
        for (size_t i = 0; i < (N + 1) * N; ++i) t[i] = INFINITY;
        for (size_t v = 0; v < N; ++v) t[v] = 0;
        for (size_t k = 1; k <= N; ++k) {
            const double *pr = t + (k - 1) * N;
            double *row = t + k * N;
            for (uint32_t v = 0; v < n; ++v) {
                double b = INFINITY;
                for (uint64_t s = g.bidx[v]; s < g.bidx[v + 1]; ++s) {
                    double pw = pr[g.bsrc[s]];
                    if (pw == INFINITY) continue;
                    double cnd = pw + g.w[g.bfe[s]];
                    if (cnd < b) b = cnd;
                }
                row[v] = b;
            }
        }
        const double *last = t + N * N;
        int found = 0;
        double best = INFINITY;
        for (uint32_t v = 0; v < n; ++v) {
            if (last[v] == INFINITY) continue;
            double vmax = -INFINITY;
            int any = 0;
            for (size_t j = 0; j < N; ++j) {
                double ej = t[j * N + v];
                if (ej == INFINITY) continue;
                double cnd = (last[v] - ej) / (double)(N - j);
                if (!any || cnd > vmax) { vmax = cnd; any = 1; }
            }
            if (any && (!found || vmax < best)) { best = vmax; found = 1; }
        }
        free(t);
        *has_cycle = found;
        if (found) { *mean = best; *num = 0; *den = 1; }
    }
    oc_free_csr(&g);
    return 0;
}

/* ---------------- seeded synthetic generators ----------------
 * Shared bit-for-bit with paper_1111_0627_b200/csrc/gen.cu (same splitmix64
 * counter hash), so the CPU oracle and the GPU library see the same graph.
 */
static inline uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

static inline uint64_t hash2(uint64_t seed, uint64_t stream, uint64_t i) {
    return splitmix64(splitmix64(seed ^ (stream * 0xd1342543de82ef95ull)) + i);
}

/* Uniform random digraph, every vertex exactly `deg` out-edges (edge i of
 * vertex v has id v*deg+i), targets uniform, integer weights in [wlo, whi]. */
void oc_generate_uniform(uint32_t n, uint32_t deg, int32_t wlo, int32_t whi, uint64_t seed,
                         uint32_t *src, uint32_t *dst, double *w) {
    uint64_t span = (uint64_t)((int64_t)whi - wlo + 1);
    for (uint64_t e = 0; e < (uint64_t)n * deg; ++e) {
        src[e] = (uint32_t)(e / deg);
        dst[e] = (uint32_t)(hash2(seed, 1, e) % n);
        w[e] = (double)(wlo + (int64_t)(hash2(seed, 2, e) % span));
    }
}

/* Power-law out-degree generator (paper_1111_0627_b200/csrc/gen.hpp
 * generate_powerlaw / generate_powerlaw_hubs, restated): deg(v) =
 * min(dmax, floor(dmin / sqrt(u_v))); hubs = q > 0 draws targets as
 * floor(n * u^(2^q)) scattered by x -> (x * A + B) mod n (q = 1 "powerlaw-hubs",
 * q = 3 "powerlaw-web"). Two calls: with
 * src == NULL only the edge count is returned. */
uint64_t oc_generate_powerlaw(uint32_t n, uint32_t dmin, uint32_t dmax, int32_t wlo, int32_t whi,
                              uint64_t seed, int hubs, uint32_t *src, uint32_t *dst, double *w) {
    const uint64_t prime = 2654435761ull;
    uint64_t mul = (n % prime == 0) ? 1 : prime % n;
    uint64_t add = hash2(seed, 4, 0) % n;
    uint64_t span = (uint64_t)((int64_t)whi - wlo + 1);
    uint64_t e = 0;
    for (uint32_t v = 0; v < n; ++v) {
        double u = (double)((hash2(seed, 3, v) >> 11) + 1) * (1.0 / 9007199254740992.0);
        double d = (double)dmin / sqrt(u);
        uint32_t deg = d >= (double)dmax ? dmax : (uint32_t)d;
        if (src) {
            for (uint32_t i = 0; i < deg; ++i, ++e) {
                uint64_t h = hash2(seed, 1, e);
                uint32_t t;
                if (hubs) {
                    double uu = (double)((h >> 11) + 1) * (1.0 / 9007199254740992.0);
                    for (int q = 0; q < hubs; ++q) /* 1: u^2 (hubs), 3: u^8 (web) */
                        uu = uu * uu;
                    double x = (double)n * uu;
                    uint64_t r = (uint64_t)x;
                    if (r >= n)
                        r = n - 1;
                    t = (uint32_t)((r * mul + add) % n);
                } else {
                    t = (uint32_t)(h % n);
                }
                src[e] = v;
                dst[e] = t;
                w[e] = (double)(wlo + (int64_t)(hash2(seed, 2, e) % span));
            }
        } else {
            e += deg;
        }
    }
    return e;
}

/* Composite state space of `clients` interleaved copies of a scenario
 * (restates proj/src/model_gen.cpp:88-148 generate_model, with the state
 * bound max_states instead of kMaxModelStates = 5'000'000 of
 * model_gen.hpp:65): states are packed client_bits per client plus the
 * server owner, numbered in breadth-first discovery order; for every state
 * (in that order), every client (ascending) and every scenario transition
 * (declaration order) enabled for it, one edge of that transition's cost.
 * Returns 0, 1 on a malformed scenario, 2 past max_states, 3 out of memory.
 * The edge arrays are malloc'ed (release with oc_free). */
typedef struct {
    uint64_t *keys;
    uint32_t *ids;
    uint64_t cap, size;
} oc_state_map;

static uint64_t oc_mix(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    return x;
}

static int oc_map_grow(oc_state_map *m, uint64_t cap) {
    uint64_t *ok = m->keys;
    uint32_t *oi = m->ids;
    uint64_t ocap = m->cap;
    m->keys = (uint64_t *)calloc(cap, sizeof(uint64_t));
    m->ids = (uint32_t *)malloc(cap * sizeof(uint32_t));
    if (!m->keys || !m->ids)
        return 3;
    memset(m->ids, 0xff, cap * sizeof(uint32_t));
    m->cap = cap;
    for (uint64_t i = 0; i < ocap; ++i)
        if (oi[i] != 0xffffffffu) {
            uint64_t h = oc_mix(ok[i]) & (cap - 1);
            while (m->ids[h] != 0xffffffffu)
                h = (h + 1) & (cap - 1);
            m->keys[h] = ok[i];
            m->ids[h] = oi[i];
        }
    free(ok);
    free(oi);
    return 0;
}

/* id of `key`, inserting it as `fresh` when absent (*inserted = 1) */
static uint32_t oc_map_intern(oc_state_map *m, uint64_t key, uint32_t fresh, int *inserted) {
    uint64_t h = oc_mix(key) & (m->cap - 1);
    while (m->ids[h] != 0xffffffffu) {
        if (m->keys[h] == key) {
            *inserted = 0;
            return m->ids[h];
        }
        h = (h + 1) & (m->cap - 1);
    }
    m->keys[h] = key;
    m->ids[h] = fresh;
    m->size++;
    *inserted = 1;
    return fresh;
}

static uint32_t oc_bits_for(uint64_t values) {
    uint32_t b = 0;
    while (b < 64 && ((uint64_t)1 << b) < values)
        ++b;
    return b;
}

void oc_free(void *p) { free(p); }

int oc_generate_model(uint32_t states, uint32_t ntr, const uint32_t *from, const uint32_t *to,
                      const int64_t *cost, const int32_t *acquires, const int32_t *releases,
                      int uses_server, uint32_t clients, uint64_t max_states, uint32_t *n_out,
                      uint64_t *m_out, uint32_t **src_out, uint32_t **dst_out, double **w_out) {
    if (states == 0 || clients == 0)
        return 1;
    for (uint32_t k = 0; k < ntr; ++k) {
        if (from[k] >= states || to[k] >= states)
            return 1;
        if ((acquires[k] || releases[k]) && !uses_server)
            return 1;
    }
    uint32_t cb = oc_bits_for(states);
    if (cb < 1)
        cb = 1;
    uint32_t ob = uses_server ? oc_bits_for((uint64_t)clients + 1) : 0;
    if ((uint64_t)cb * clients + ob > 64)
        return 1;
    uint64_t cmask = ((uint64_t)1 << cb) - 1;
    uint64_t oshift = (uint64_t)clients * cb;
    uint64_t omask = ob ? ((((uint64_t)1 << ob) - 1) << oshift) : 0;

    oc_state_map map = {0};
    uint64_t *queue = NULL, qcap = 0, nq = 0;
    uint32_t *src = NULL, *dst = NULL;
    double *w = NULL;
    uint64_t ecap = 0, m = 0;
    int rc = 0;
    if (oc_map_grow(&map, 1 << 16))
        return 3;
    int ins;
    oc_map_intern(&map, 0, 0, &ins); /* all clients in state 0, server free */
    qcap = 1 << 16;
    queue = (uint64_t *)malloc(qcap * sizeof(uint64_t));
    if (!queue)
        return 3;
    queue[nq++] = 0;
    for (uint64_t head = 0; head < nq && rc == 0; ++head) {
        uint64_t s = queue[head];
        uint64_t owner = ob ? (s & omask) >> oshift : 0;
        for (uint32_t i = 0; i < clients && rc == 0; ++i) {
            uint64_t shift = (uint64_t)i * cb;
            uint32_t loc = (uint32_t)((s >> shift) & cmask);
            for (uint32_t k = 0; k < ntr; ++k) {
                if (from[k] != loc)
                    continue;
                if (acquires[k] && owner != 0)
                    continue;
                if (releases[k] && owner != (uint64_t)i + 1)
                    continue;
                uint64_t ns = (s & ~(cmask << shift)) | ((uint64_t)to[k] << shift);
                if (acquires[k])
                    ns = (ns & ~omask) | ((uint64_t)(i + 1) << oshift);
                if (releases[k])
                    ns &= ~omask;
                if ((map.size + 1) * 2 > map.cap && oc_map_grow(&map, map.cap * 2)) {
                    rc = 3;
                    break;
                }
                uint32_t id = oc_map_intern(&map, ns, (uint32_t)nq, &ins);
                if (ins) {
                    if (nq + 1 > max_states) {
                        rc = 2;
                        break;
                    }
                    if (nq == qcap) {
                        qcap *= 2;
                        uint64_t *q2 = (uint64_t *)realloc(queue, qcap * sizeof(uint64_t));
                        if (!q2) {
                            rc = 3;
                            break;
                        }
                        queue = q2;
                    }
                    queue[nq++] = ns;
                }
                if (m == ecap) {
                    ecap = ecap ? ecap * 2 : (1 << 16);
                    uint32_t *s2 = (uint32_t *)realloc(src, ecap * sizeof(uint32_t));
                    if (s2) src = s2;
                    uint32_t *d2 = (uint32_t *)realloc(dst, ecap * sizeof(uint32_t));
                    if (d2) dst = d2;
                    double *w2 = (double *)realloc(w, ecap * sizeof(double));
                    if (w2) w = w2;
                    if (!s2 || !d2 || !w2) {
                        rc = 3;
                        break;
                    }
                }
                src[m] = (uint32_t)head;
                dst[m] = id;
                w[m] = (double)cost[k];
                ++m;
            }
        }
    }
    free(map.keys);
    free(map.ids);
    free(queue);
    if (rc) {
        free(src);
        free(dst);
        free(w);
        return rc;
    }
    *n_out = (uint32_t)nq;
    *m_out = m;
    *src_out = src;
    *dst_out = dst;
    *w_out = w;
    return 0;
}
