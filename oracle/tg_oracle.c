/*
 * oracle/tg_oracle.c -- TEST INFRASTRUCTURE ONLY (parity checker for tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg; the product never
 * links it).  Plain-C restatement of the reference 2D-PT hot path; every
 * function cites the reference lines it follows (paths under
 * /root/reference/proj).  The only departures from the reference are the ones
 * the parity contract names: the mt19937_64 engine is replaced by the Philox
 * stream of philox_ref.h, a heat-bath update rule is offered next to
 * Metropolis, and two alternative RNG associations (bit-plane draws and packed
 * draws keyed by the physical state) are offered next to the reference's
 * per-slot streams.
 * Floating-point expressions are written in the reference's evaluation order
 * so that the port is bit-identical to the reference objects (checked against
 * oracle/_ref in tests/test_oracle_ref.py).
 */
#include "tg_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "philox_ref.h"

#define REFRESH_INTERVAL 256 /* engine.cpp:79 kRefreshInterval */

static void set_err(char* err, int errlen, const char* fmt, ...) {
    if (!err || errlen <= 0) return;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(err, (size_t)errlen, fmt, ap);
    va_end(ap);
}

/* ------------------------------------------------------------------ model */

typedef struct {
    int i, j;
    double w;
} coupling_t;

typedef struct {
    int n;
    int m;
    coupling_t* c; /* sorted canonical (i<j) */
    double* h;
    int* off;      /* CSR, neighbour order of ising.cpp:55-61 */
    int* nbr;
    double* nbw;
} model_t;

static int cmp_coupling(const void* a, const void* b) {
    const coupling_t* x = (const coupling_t*)a;
    const coupling_t* y = (const coupling_t*)b;
    if (x->i != y->i) return x->i < y->i ? -1 : 1;
    if (x->j != y->j) return x->j < y->j ? -1 : 1;
    return 0;
}

static void model_free(model_t* m) {
    free(m->c); free(m->h); free(m->off); free(m->nbr); free(m->nbw);
    memset(m, 0, sizeof(*m));
}

/* IsingModel::IsingModel, ising.cpp:21-62 (validation, canonical sort, CSR). */
static int model_build(model_t* m, int n, int nc, const int* ci, const int* cj,
                       const double* cw, const double* h, char* err, int errlen) {
    memset(m, 0, sizeof(*m));
    if (n <= 0) { set_err(err, errlen, "model: n_spins must be positive"); return TGO_CONFIG_ERROR; }
    m->n = n;
    m->m = nc;
    m->c = (coupling_t*)malloc(sizeof(coupling_t) * (size_t)(nc > 0 ? nc : 1));
    m->h = (double*)malloc(sizeof(double) * (size_t)n);
    for (int i = 0; i < n; ++i) m->h[i] = h ? h[i] : 0.0;
    for (int k = 0; k < nc; ++k) {
        int a = ci[k], b = cj[k];
        if (a == b) { set_err(err, errlen, "model: self-loop on spin %d", a); model_free(m); return TGO_CONFIG_ERROR; }
        if (a > b) { int t = a; a = b; b = t; }
        if (a < 0 || b >= n) {
            set_err(err, errlen, "model: coupling index out of range: (%d, %d)", a, b);
            model_free(m);
            return TGO_CONFIG_ERROR;
        }
        m->c[k].i = a; m->c[k].j = b; m->c[k].w = cw[k];
    }
    /* std::sort is not stable, but keys are unique after the duplicate check. */
    qsort(m->c, (size_t)nc, sizeof(coupling_t), cmp_coupling);
    for (int k = 1; k < nc; ++k)
        if (m->c[k - 1].i == m->c[k].i && m->c[k - 1].j == m->c[k].j) {
            set_err(err, errlen, "model: duplicate coupling (%d, %d)", m->c[k].i, m->c[k].j);
            model_free(m);
            return TGO_CONFIG_ERROR;
        }
    int* deg = (int*)calloc((size_t)n, sizeof(int));
    for (int k = 0; k < nc; ++k) { deg[m->c[k].i]++; deg[m->c[k].j]++; }
    m->off = (int*)malloc(sizeof(int) * (size_t)(n + 1));
    m->off[0] = 0;
    for (int i = 0; i < n; ++i) m->off[i + 1] = m->off[i] + deg[i];
    m->nbr = (int*)malloc(sizeof(int) * (size_t)(m->off[n] > 0 ? m->off[n] : 1));
    m->nbw = (double*)malloc(sizeof(double) * (size_t)(m->off[n] > 0 ? m->off[n] : 1));
    int* cur = deg; /* reuse as cursor */
    for (int i = 0; i < n; ++i) cur[i] = m->off[i];
    for (int k = 0; k < nc; ++k) {
        const coupling_t c = m->c[k];
        m->nbr[cur[c.i]] = c.j; m->nbw[cur[c.i]++] = c.w;
        m->nbr[cur[c.j]] = c.i; m->nbw[cur[c.j]++] = c.w;
    }
    free(deg);
    return TGO_OK;
}

/* energy, ising.cpp:70-77 */
static double model_energy(const model_t* m, const int8_t* s) {
    double e = 0.0;
    for (int k = 0; k < m->m; ++k) {
        const coupling_t c = m->c[k];
        e -= c.w * (double)s[c.i] * (double)s[c.j];
    }
    for (int i = 0; i < m->n; ++i) e -= m->h[i] * (double)s[i];
    return e;
}

/* local_fields, ising.cpp:79-88 */
static void model_local_fields(const model_t* m, const int8_t* s, double* local) {
    for (int i = 0; i < m->n; ++i) {
        double sum = m->h[i];
        for (int k = m->off[i]; k < m->off[i + 1]; ++k) sum += m->nbw[k] * (double)s[m->nbr[k]];
        local[i] = sum;
    }
}

/* apply_flip, ising.cpp:90-96 */
static void model_apply_flip(const model_t* m, int8_t* s, int i, double* local) {
    s[i] = (int8_t)-s[i];
    const double two_si = 2.0 * (double)s[i];
    for (int k = m->off[i]; k < m->off[i + 1]; ++k) local[m->nbr[k]] += two_si * m->nbw[k];
}

/* ------------------------------------------------------------ constraints */

typedef struct {
    int n;
    int m;
    int* pa; /* normalised a<b, input order */
    int* pb;
    int* off;
    int* partners;
} cset_t;

static void cset_free(cset_t* c) {
    free(c->pa); free(c->pb); free(c->off); free(c->partners);
    memset(c, 0, sizeof(*c));
}

/* ConstraintSet::ConstraintSet, constraints.cpp:16-39 */
static int cset_build(cset_t* c, int n, int np, const int* pa, const int* pb, char* err, int errlen) {
    memset(c, 0, sizeof(*c));
    c->n = n;
    c->m = np;
    c->pa = (int*)malloc(sizeof(int) * (size_t)(np > 0 ? np : 1));
    c->pb = (int*)malloc(sizeof(int) * (size_t)(np > 0 ? np : 1));
    for (int k = 0; k < np; ++k) {
        int a = pa[k], b = pb[k];
        if (a == b) { set_err(err, errlen, "constraint: pair on a single spin %d", a); cset_free(c); return TGO_CONFIG_ERROR; }
        if (a > b) { int t = a; a = b; b = t; }
        if (a < 0 || b >= n) {
            set_err(err, errlen, "constraint: index out of range: (%d, %d)", a, b);
            cset_free(c);
            return TGO_CONFIG_ERROR;
        }
        c->pa[k] = a; c->pb[k] = b;
    }
    int* deg = (int*)calloc((size_t)n, sizeof(int));
    for (int k = 0; k < np; ++k) { deg[c->pa[k]]++; deg[c->pb[k]]++; }
    c->off = (int*)malloc(sizeof(int) * (size_t)(n + 1));
    c->off[0] = 0;
    for (int i = 0; i < n; ++i) c->off[i + 1] = c->off[i] + deg[i];
    c->partners = (int*)malloc(sizeof(int) * (size_t)(c->off[n] > 0 ? c->off[n] : 1));
    for (int i = 0; i < n; ++i) deg[i] = c->off[i];
    for (int k = 0; k < np; ++k) {
        c->partners[deg[c->pa[k]]++] = c->pb[k];
        c->partners[deg[c->pb[k]]++] = c->pa[k];
    }
    free(deg);
    return TGO_OK;
}

/* ConstraintSet::evaluate, constraints.cpp:41-48 */
static double cset_evaluate(const cset_t* c, const int8_t* s) {
    double g = 0.0;
    for (int k = 0; k < c->m; ++k) {
        const double d = (double)s[c->pa[k]] - (double)s[c->pb[k]];
        g += d * d;
    }
    return g;
}

/* ConstraintSet::delta_flip, constraints.hpp:32-37 */
static double cset_delta_flip(const cset_t* c, const int8_t* s, int i) {
    double d = 0.0;
    for (int k = c->off[i]; k < c->off[i + 1]; ++k) d += 4.0 * (double)s[i] * (double)s[c->partners[k]];
    return d;
}

/* ------------------------------------------------------- effective model */

typedef struct {
    model_t merged;
    const cset_t* cs;
    double penalty;
    double offset;
} view_t;

typedef struct {
    int a, b, ord;
    double w;
} wentry_t;

static int cmp_wentry(const void* x, const void* y) {
    const wentry_t* p = (const wentry_t*)x;
    const wentry_t* q = (const wentry_t*)y;
    if (p->a != q->a) return p->a < q->a ? -1 : 1;
    if (p->b != q->b) return p->b < q->b ? -1 : 1;
    return p->ord < q->ord ? -1 : (p->ord > q->ord);
}

/* build_effective, constraints.cpp:122-140: every pair merged as a +2P
 * coupling (std::map accumulation order: cost weight first, then pairs in
 * input order), offset 2P*m. */
static int view_build(view_t* v, const model_t* cost, const cset_t* cs, double penalty,
                      char* err, int errlen) {
    memset(v, 0, sizeof(*v));
    if (penalty < 0.0) { set_err(err, errlen, "build_effective: penalty must be >= 0"); return TGO_CONFIG_ERROR; }
    const int tot = cost->m + cs->m;
    wentry_t* e = (wentry_t*)malloc(sizeof(wentry_t) * (size_t)(tot > 0 ? tot : 1));
    int k = 0;
    for (int q = 0; q < cost->m; ++q, ++k) { e[k].a = cost->c[q].i; e[k].b = cost->c[q].j; e[k].w = cost->c[q].w; e[k].ord = k; }
    for (int q = 0; q < cs->m; ++q, ++k) { e[k].a = cs->pa[q]; e[k].b = cs->pb[q]; e[k].w = 2.0 * penalty; e[k].ord = k; }
    qsort(e, (size_t)tot, sizeof(wentry_t), cmp_wentry);
    int* mi = (int*)malloc(sizeof(int) * (size_t)(tot > 0 ? tot : 1));
    int* mj = (int*)malloc(sizeof(int) * (size_t)(tot > 0 ? tot : 1));
    double* mw = (double*)malloc(sizeof(double) * (size_t)(tot > 0 ? tot : 1));
    int nm = 0;
    for (int q = 0; q < tot;) {
        double w = 0.0;
        int r = q;
        while (r < tot && e[r].a == e[q].a && e[r].b == e[q].b) { w += e[r].w; ++r; }
        mi[nm] = e[q].a; mj[nm] = e[q].b; mw[nm] = w; ++nm;
        q = r;
    }
    int rc = model_build(&v->merged, cost->n, nm, mi, mj, mw, cost->h, err, errlen);
    free(e); free(mi); free(mj); free(mw);
    if (rc) return rc;
    v->cs = cs;
    v->penalty = penalty;
    v->offset = 2.0 * penalty * (double)cs->m;
    return TGO_OK;
}

/* energy_breakdown, constraints.cpp:142-147 */
static void view_breakdown(const view_t* v, const int8_t* s, double* f, double* g) {
    const double gg = cset_evaluate(v->cs, s);
    const double eff = model_energy(&v->merged, s) + v->offset;
    *g = gg;
    *f = eff - v->penalty * gg;
}

/* ------------------------------------------------------------- replicas */

typedef struct {
    int8_t* spins;
    double* local;
    double f, g;
    int id; /* physical state id = initial slot; travels with the state */
} rstate_t;

/* refresh_sweep_state, mc.cpp:14-19 */
static void refresh(const view_t* v, rstate_t* st) {
    model_local_fields(&v->merged, st->spins, st->local);
    view_breakdown(v, st->spins, &st->f, &st->g);
}

typedef struct {
    int mode;
    uint64_t slot_seed;  /* SLOT: derive_seed(seed, replica, slot) */
    uint64_t* slot_ctr;  /* SLOT: 64-bit outputs consumed so far */
    uint64_t pkey;       /* PLANE: run key derive_seed(seed, PLANE, 0) */
    uint64_t t;          /* PLANE: global sweep index */
} draw_ctx_t;

static inline uint64_t next_u53(draw_ctx_t* d, const rstate_t* st, int site) {
    if (d->mode == TGO_RNG_SLOT) {
        const uint64_t b = tgo_stream_bits(d->slot_seed, (*d->slot_ctr)++);
        return b >> 11; /* rng.hpp:53-55 */
    }
    if (d->mode == TGO_RNG_PACK) return tgo_pack_u53(d->pkey, (uint32_t)st->id, d->t, (uint32_t)site);
    return tgo_plane_u53(d->pkey, (uint32_t)(st->id >> 5), d->t, (uint32_t)site, st->id & 31);
}

/* u < T for the bit-plane uniform u = U53 * 2^-53 of (state, site, sweep),
 * decided exactly with the bits of U53 drawn MSB first (philox_ref.h
 * tgo_plane_u53 word layout: plane b = bit `lane` of word b & 3 of block
 * b >> 2), stopping as soon as the comparison is decided.  Same result as
 * tgo_u53_to_unit(tgo_plane_u53(...)) < T (tests/test_oracle_lazy.py). */
static int plane_less(const draw_ctx_t* d, const rstate_t* st, int site, double T) {
    if (!(T > 0.0)) return 0;
    if (T >= 1.0) return 1; /* U53 <= 2^53 - 1 */
    /* U53 < T * 2^53  <=>  U53 < K = ceil(T * 2^53) (exact: power-of-two scaling) */
    const uint64_t K = (uint64_t)ceil(ldexp(T, 53));
    const uint32_t grp = (uint32_t)(st->id >> 5);
    const int lane = st->id & 31;
    const uint32_t key[2] = {(uint32_t)d->pkey, (uint32_t)(d->pkey >> 32)};
    for (int blk = 0; blk < 14; ++blk) {
        const uint32_t ctr[4] = {(uint32_t)site, (uint32_t)d->t, (uint32_t)(d->t >> 32),
                                 (uint32_t)blk | (grp << 4)};
        uint32_t o[4];
        tgo_philox4x32_10(ctr, key, o);
        for (int w = 0; w < 4; ++w) {
            const int b = blk * 4 + w;
            if (b >= 53) return 0; /* U53 == K */
            const uint32_t ub = (o[w] >> lane) & 1u;
            const uint32_t kb = (uint32_t)(K >> (52 - b)) & 1u;
            if (ub != kb) return ub < kb;
        }
    }
    return 0;
}

/* metropolis_sweep, mc.cpp:21-35 (rule 0); heat-bath variant (rule 1) with
 * the same one-draw-per-spin contract and the same f/g bookkeeping. */
static void sweep(const view_t* v, double beta, rstate_t* st, draw_ctx_t* d, int rule) {
    const int n = v->merged.n;
    const int lazy = d->mode == TGO_RNG_PLANE;
    for (int i = 0; i < n; ++i) {
        const double local_i = st->local[i];
        const double de = 2.0 * (double)st->spins[i] * local_i;
        int flip;
        if (lazy) { /* bit-plane draws: the same u < T decided bit by bit */
            if (rule == TGO_RULE_METROPOLIS) {
                flip = (de <= 0.0 || plane_less(d, st, i, exp(-beta * de)));
            } else {
                const double p = 1.0 / (1.0 + exp(-2.0 * beta * local_i));
                const int8_t nv = plane_less(d, st, i, p) ? (int8_t)1 : (int8_t)-1;
                flip = nv != st->spins[i];
            }
        } else if (rule == TGO_RULE_METROPOLIS) {
            const double u = tgo_u53_to_unit(next_u53(d, st, i));
            flip = (de <= 0.0 || u < exp(-beta * de));
        } else {
            const double u = tgo_u53_to_unit(next_u53(d, st, i));
            const double p = 1.0 / (1.0 + exp(-2.0 * beta * local_i));
            const int8_t nv = (u < p) ? (int8_t)1 : (int8_t)-1;
            flip = nv != st->spins[i];
        }
        if (flip) {
            const double dg = cset_delta_flip(v->cs, st->spins, i);
            model_apply_flip(&v->merged, st->spins, i, st->local);
            st->f += de - v->penalty * dg;
            st->g += dg;
        }
    }
}

/* ------------------------------------------------------------ public API */

double tgo_p_swap_probability(double beta, double d_penalty, double dg) {
    const double x = beta * d_penalty * dg; /* engine.cpp:18-21 */
    return x >= 0.0 ? 1.0 : exp(x);
}
double tgo_beta_swap_probability(double d_beta, double d_energy) {
    const double x = d_beta * d_energy; /* engine.cpp:23-26 */
    return x >= 0.0 ? 1.0 : exp(x);
}
double tgo_general_swap_probability(double beta_a, double beta_b, double de_a, double de_b) {
    const double x = beta_a * de_a + beta_b * de_b; /* engine.cpp:28-32 */
    return x >= 0.0 ? 1.0 : exp(x);
}

uint64_t tgo_digest(const int8_t* s, int n) {
    uint64_t d = 0;
    for (int i = 0; i < n; ++i)
        if (s[i] > 0) d += tgo_digest_term((uint64_t)i);
    return d;
}

uint64_t tgo_encode_state(const int8_t* s, int n) { /* oracle.cpp:17-22 */
    uint64_t e = 0;
    for (int i = 0; i < n && i < 64; ++i)
        if (s[i] > 0) e |= (uint64_t)1 << i;
    return e;
}

void tgo_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    tgo_philox4x32_10(ctr, key, out);
}
uint64_t tgo_derive(uint64_t master, uint64_t purpose, uint64_t index) {
    return tgo_derive_seed(master, purpose, index);
}
uint64_t tgo_bits(uint64_t seed, uint64_t n) { return tgo_stream_bits(seed, n); }
uint64_t tgo_plane(uint64_t pkey, uint32_t grp, uint64_t t, uint32_t site, int lane) {
    return tgo_plane_u53(pkey, grp, t, site, lane);
}
uint64_t tgo_pack(uint64_t pkey, uint32_t m, uint64_t t, uint32_t site) {
    return tgo_pack_u53(pkey, m, t, site);
}
int tgo_plane_less(uint64_t pkey, uint32_t grp, uint64_t t, uint32_t site, int lane, double T) {
    draw_ctx_t d;
    memset(&d, 0, sizeof d);
    d.mode = TGO_RNG_PLANE;
    d.pkey = pkey;
    d.t = t;
    rstate_t st;
    memset(&st, 0, sizeof st);
    st.id = (int)(grp << 5) | lane;
    return plane_less(&d, &st, (int)site, T);
}

int tgo_energy_breakdown(const tgo_problem* p, double penalty, const int8_t* s, double* f,
                         double* g) {
    model_t cost;
    cset_t cs;
    view_t v;
    char err[256];
    int rc = model_build(&cost, p->n, p->n_couplings, p->ci, p->cj, p->cw, p->fields, err, 256);
    if (rc) return rc;
    rc = cset_build(&cs, p->n, p->n_pairs, p->pa, p->pb, err, 256);
    if (rc) { model_free(&cost); return rc; }
    rc = view_build(&v, &cost, &cs, penalty, err, 256);
    if (!rc) { view_breakdown(&v, s, f, g); model_free(&v.merged); }
    cset_free(&cs);
    model_free(&cost);
    return rc;
}

/* Greedy colouring in index order over cost couplings and chain pairs, then
 * the canonical order: stable sort by (colour, chain degree, cost degree).
 * This is the relabel under which a sequential index-order sweep equals a
 * chromatic sweep (no two same-colour spins are adjacent). */
int tgo_canonical_order(const tgo_problem* p, int32_t* color, int32_t* order, int32_t* n_colors) {
    const int n = p->n;
    int* dc = (int*)calloc((size_t)n, sizeof(int));
    int* dq = (int*)calloc((size_t)n, sizeof(int));
    int* deg = (int*)calloc((size_t)n, sizeof(int));
    for (int k = 0; k < p->n_couplings; ++k) { dc[p->ci[k]]++; dc[p->cj[k]]++; }
    for (int k = 0; k < p->n_pairs; ++k) { dq[p->pa[k]]++; dq[p->pb[k]]++; }
    for (int i = 0; i < n; ++i) deg[i] = dc[i] + dq[i];
    int* off = (int*)malloc(sizeof(int) * (size_t)(n + 1));
    off[0] = 0;
    for (int i = 0; i < n; ++i) off[i + 1] = off[i] + deg[i];
    int* adj = (int*)malloc(sizeof(int) * (size_t)(off[n] > 0 ? off[n] : 1));
    int* cur = (int*)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
    for (int i = 0; i < n; ++i) cur[i] = off[i];
    for (int k = 0; k < p->n_couplings; ++k) { adj[cur[p->ci[k]]++] = p->cj[k]; adj[cur[p->cj[k]]++] = p->ci[k]; }
    for (int k = 0; k < p->n_pairs; ++k) { adj[cur[p->pa[k]]++] = p->pb[k]; adj[cur[p->pb[k]]++] = p->pa[k]; }
    int maxc = 0;
    unsigned char* used = (unsigned char*)calloc((size_t)n + 2, 1);
    for (int i = 0; i < n; ++i) {
        for (int k = off[i]; k < off[i + 1]; ++k)
            if (adj[k] < i) used[color[adj[k]]] = 1;
        int c = 0;
        while (used[c]) ++c;
        color[i] = c;
        if (c + 1 > maxc) maxc = c + 1;
        for (int k = off[i]; k < off[i + 1]; ++k)
            if (adj[k] < i) used[color[adj[k]]] = 0;
    }
    /* stable counting sort by key (color, dq, dc) */
    int nq = 0, ncd = 0;
    for (int i = 0; i < n; ++i) { if (dq[i] + 1 > nq) nq = dq[i] + 1; if (dc[i] + 1 > ncd) ncd = dc[i] + 1; }
    int pos = 0;
    for (int c = 0; c < maxc; ++c)
        for (int q = 0; q < nq; ++q)
            for (int d = 0; d < ncd; ++d)
                for (int i = 0; i < n; ++i)
                    if (color[i] == c && dq[i] == q && dc[i] == d) order[pos++] = i;
    *n_colors = maxc;
    free(dc); free(dq); free(deg); free(off); free(adj); free(cur); free(used);
    return TGO_OK;
}

static int check_monotone(const double* v, int len, const char* what, char* err, int errlen) {
    /* engine.cpp:41-52 */
    if (len <= 0) { set_err(err, errlen, "%s vector must be non-empty", what); return TGO_CONFIG_ERROR; }
    for (int k = 0; k < len; ++k)
        if (!isfinite(v[k])) { set_err(err, errlen, "%s entries must be finite", what); return TGO_CONFIG_ERROR; }
    for (int k = 1; k < len; ++k)
        if (v[k] <= v[k - 1]) { set_err(err, errlen, "%s vector must be strictly increasing", what); return TGO_CONFIG_ERROR; }
    return TGO_OK;
}

/* One round's sweeps of every replica (engine.cpp:125-132, for_each_replica
 * :61-77): replicas are independent between swap phases, so a strided
 * partition over threads (r = w mod T, as the reference) gives the same
 * result for any thread count. */
typedef struct {
    const view_t* views;
    const tgo_run_cfg* cfg;
    rstate_t* rep;
    const uint64_t* slot_seed;
    uint64_t* slot_ctr;
    uint64_t pkey;
    int64_t rn;
    int R, J;
    int64_t sps;
    int w, T;
} sweep_job_t;

static void* sweep_worker(void* arg) {
    const sweep_job_t* jb = (const sweep_job_t*)arg;
    for (int r = jb->w; r < jb->R; r += jb->T) {
        const view_t* v = &jb->views[r % jb->J];
        const double beta = jb->cfg->betas[r / jb->J];
        for (int64_t s = 0; s < jb->sps; ++s) {
            draw_ctx_t d;
            d.mode = jb->cfg->rng_mode;
            d.slot_seed = jb->slot_seed[r];
            d.slot_ctr = &jb->slot_ctr[r];
            d.pkey = jb->pkey;
            d.t = (uint64_t)((jb->rn - 1) * jb->sps + s);
            sweep(v, beta, &jb->rep[r], &d, jb->cfg->rule);
        }
        if (jb->rn % REFRESH_INTERVAL == 0) refresh(v, &jb->rep[r]);
    }
    return NULL;
}

static void run_sweeps(const sweep_job_t* job, int T) {
    if (T <= 1) {
        sweep_worker((void*)job);
        return;
    }
    pthread_t th[256];
    sweep_job_t jobs[256];
    int started = 0;
    for (int w = 0; w < T; ++w) {
        jobs[w] = *job;
        jobs[w].w = w;
        jobs[w].T = T;
    }
    for (int w = 1; w < T; ++w) {
        if (pthread_create(&th[w], NULL, sweep_worker, &jobs[w]) != 0) break;
        started = w;
    }
    /* threads that could not start: their share runs here */
    for (int w = started + 1; w < T; ++w) sweep_worker(&jobs[w]);
    sweep_worker(&jobs[0]);
    for (int w = 1; w <= started; ++w) pthread_join(th[w], NULL);
}

/* TGO_THREADS (environment, default 1): sweep threads of tgo_run_2dpt; the
 * result does not depend on it. */
static int oracle_threads(int R, int n) {
    const char* e = getenv("TGO_THREADS");
    int t = e ? atoi(e) : 1;
    if (t > 256) t = 256;
    if (t > R) t = R;
    if ((int64_t)R * n < 65536) t = 1;
    return t < 1 ? 1 : t;
}

int tgo_run_2dpt(const tgo_problem* prob, const tgo_run_cfg* cfg, tgo_outputs* out, char* err,
                 int errlen) {
    model_t cost;
    cset_t cs;
    int rc = model_build(&cost, prob->n, prob->n_couplings, prob->ci, prob->cj, prob->cw,
                         prob->fields, err, errlen);
    if (rc) return rc;
    rc = cset_build(&cs, prob->n, prob->n_pairs, prob->pa, prob->pb, err, errlen);
    if (rc) { model_free(&cost); return rc; }

    /* engine.cpp:85-87, 53-59 */
    if ((rc = check_monotone(cfg->betas, cfg->n_betas, "beta", err, errlen)) ||
        (rc = check_monotone(cfg->penalties, cfg->n_penalties, "penalty", err, errlen))) {
        cset_free(&cs); model_free(&cost); return rc;
    }
    if (cfg->sweeps_per_swap < 1) { set_err(err, errlen, "run: sweeps_per_swap must be >= 1"); rc = TGO_CONFIG_ERROR; }
    else if (cfg->total_sweeps < cfg->sweeps_per_swap) { set_err(err, errlen, "run: total_sweeps must be >= sweeps_per_swap"); rc = TGO_CONFIG_ERROR; }
    if (rc) { cset_free(&cs); model_free(&cost); return rc; }

    const int I = cfg->n_betas, J = cfg->n_penalties, R = I * J, n = prob->n;
    view_t* views = (view_t*)calloc((size_t)J, sizeof(view_t));
    for (int j = 0; j < J; ++j) {
        rc = view_build(&views[j], &cost, &cs, cfg->penalties[j], err, errlen);
        if (rc) {
            for (int q = 0; q < j; ++q) model_free(&views[q].merged);
            free(views); cset_free(&cs); model_free(&cost); return rc;
        }
    }

    rstate_t* rep = (rstate_t*)calloc((size_t)R, sizeof(rstate_t));
    uint64_t* slot_seed = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)R);
    uint64_t* slot_ctr = (uint64_t*)calloc((size_t)R, sizeof(uint64_t));
    const uint64_t pkey = tgo_derive_seed(cfg->seed,
                                          cfg->rng_mode == TGO_RNG_PACK ? TGO_PURPOSE_PACK : TGO_PURPOSE_PLANE, 0);
    for (int r = 0; r < R; ++r) { /* engine.cpp:98-106 */
        rep[r].spins = (int8_t*)malloc((size_t)n);
        rep[r].local = (double*)malloc(sizeof(double) * (size_t)n);
        rep[r].id = r;
        const uint64_t iseed = tgo_derive_seed(cfg->seed, TGO_PURPOSE_INIT, (uint64_t)r);
        for (int i = 0; i < n; ++i) /* random_state, ising.cpp:15-19 */
            rep[r].spins[i] = (tgo_stream_bits(iseed, (uint64_t)i) >> 63) ? (int8_t)1 : (int8_t)-1;
        refresh(&views[r % J], &rep[r]);
        slot_seed[r] = tgo_derive_seed(cfg->seed, TGO_PURPOSE_REPLICA, (uint64_t)r);
    }
    const uint64_t swap_seed = tgo_derive_seed(cfg->seed, TGO_PURPOSE_SWAP, 0);
    uint64_t swap_ctr = 0;

    const int np = I * (J > 1 ? J - 1 : 0);
    const int nb = (I > 1 ? I - 1 : 0) * J;
    int64_t* att_p = (int64_t*)calloc((size_t)(np + 1), sizeof(int64_t));
    int64_t* acc_p = (int64_t*)calloc((size_t)(np + 1), sizeof(int64_t));
    int64_t* att_b = (int64_t*)calloc((size_t)(nb + 1), sizeof(int64_t));
    int64_t* acc_b = (int64_t*)calloc((size_t)(nb + 1), sizeof(int64_t));

    const int64_t sps = cfg->sweeps_per_swap;
    const int64_t n_swap = cfg->total_sweeps / sps;
    const int n_threads = oracle_threads(R, n);
    int direction = 1;
    for (int64_t rn = 1; rn <= n_swap; ++rn) { /* engine.cpp:121-217 */
        const int even_swap = (rn % 2 == 0) ? 1 : 0;
        sweep_job_t job = {views, cfg, rep, slot_seed, slot_ctr, pkey, rn, R, J, sps, 0, 1};
        run_sweeps(&job, n_threads);
        int do_p, do_b;
        if (I == 1 && J == 1) { do_p = do_b = 0; }
        else if (I == 1) { do_p = 1; do_b = 0; }
        else if (J == 1) { do_p = 0; do_b = 1; }
        else { do_p = direction == 1; do_b = !do_p; }

        if (do_p) { /* engine.cpp:148-167 */
            for (int i = 0; i < I; ++i)
                for (int p = even_swap; p + 1 < J; p += 2) {
                    rstate_t* a = &rep[i * J + p];
                    rstate_t* b = &rep[i * J + p + 1];
                    const double x = cfg->betas[i] * (cfg->penalties[p + 1] - cfg->penalties[p]) * (b->g - a->g);
                    const double u = tgo_u53_to_unit(tgo_stream_bits(swap_seed, swap_ctr++) >> 11);
                    ++att_p[i * (J - 1) + p];
                    if (x >= 0.0 || u < exp(x)) {
                        rstate_t t = *a; *a = *b; *b = t;
                        refresh(&views[p], a);
                        refresh(&views[p + 1], b);
                        ++acc_p[i * (J - 1) + p];
                    }
                }
        }
        if (do_b) { /* engine.cpp:168-187 */
            for (int j = 0; j < J; ++j)
                for (int b = even_swap; b + 1 < I; b += 2) {
                    rstate_t* lo = &rep[b * J + j];
                    rstate_t* hi = &rep[(b + 1) * J + j];
                    const double pj = cfg->penalties[j];
                    const double e_lo = lo->f + pj * lo->g;
                    const double e_hi = hi->f + pj * hi->g;
                    const double x = (cfg->betas[b + 1] - cfg->betas[b]) * (e_hi - e_lo);
                    const double u = tgo_u53_to_unit(tgo_stream_bits(swap_seed, swap_ctr++) >> 11);
                    ++att_b[b * J + j];
                    if (x >= 0.0 || u < exp(x)) {
                        rstate_t t = *lo; *lo = *hi; *hi = t;
                        ++acc_b[b * J + j];
                    }
                }
        }
        /* record, engine.cpp:189-214 */
        const rstate_t* tg = &rep[R - 1];
        const int64_t k = rn - 1;
        if (out->f) out->f[k] = tg->f;
        if (out->g) out->g[k] = tg->g;
        if (out->feasible) out->feasible[k] = (uint8_t)(tg->g == 0.0);
        if (out->digest) out->digest[k] = tgo_digest(tg->spins, n);
        if (out->states) memcpy(out->states + k * n, tg->spins, (size_t)n);
        if (out->grid_states)
            for (int r = 0; r < R; ++r) memcpy(out->grid_states + (k * R + r) * n, rep[r].spins, (size_t)n);
        if (out->round_acc_p && np) memcpy(out->round_acc_p + k * np, acc_p, sizeof(int64_t) * (size_t)np);
        if (out->round_acc_b && nb) memcpy(out->round_acc_b + k * nb, acc_b, sizeof(int64_t) * (size_t)nb);
        if (even_swap) direction = -direction;
    }
    if (out->attempts_p) memcpy(out->attempts_p, att_p, sizeof(int64_t) * (size_t)np);
    if (out->accepts_p) memcpy(out->accepts_p, acc_p, sizeof(int64_t) * (size_t)np);
    if (out->attempts_b) memcpy(out->attempts_b, att_b, sizeof(int64_t) * (size_t)nb);
    if (out->accepts_b) memcpy(out->accepts_b, acc_b, sizeof(int64_t) * (size_t)nb);
    for (int r = 0; r < R; ++r) {
        if (out->final_grid) memcpy(out->final_grid + (size_t)r * n, rep[r].spins, (size_t)n);
        if (out->final_f) out->final_f[r] = rep[r].f;
        if (out->final_g) out->final_g[r] = rep[r].g;
        if (out->final_state_id) out->final_state_id[r] = rep[r].id;
    }

    for (int r = 0; r < R; ++r) { free(rep[r].spins); free(rep[r].local); }
    free(rep); free(slot_seed); free(slot_ctr);
    free(att_p); free(acc_p); free(att_b); free(acc_b);
    for (int j = 0; j < J; ++j) model_free(&views[j].merged);
    free(views);
    cset_free(&cs);
    model_free(&cost);
    return TGO_OK;
}

/* run_jcolumn_pt, engine.cpp:221-270: standard PT (beta swaps only) at a fixed
 * penalty, repeated with independent seeds (StreamPurpose::repeat = 5,
 * rng.hpp:28) and merged per round. */
int tgo_run_jcolumn(const tgo_problem* prob, const tgo_run_cfg* cfg, double p_fixed,
                    int j_repeats, tgo_baseline_out* out, char* err, int errlen) {
    if (p_fixed <= 0.0) { set_err(err, errlen, "baseline: P must be positive"); return TGO_CONFIG_ERROR; }
    if (j_repeats < 1) { set_err(err, errlen, "baseline: repeats must be >= 1"); return TGO_CONFIG_ERROR; }
    const int64_t rounds = cfg->sweeps_per_swap >= 1 ? cfg->total_sweeps / cfg->sweeps_per_swap : 0;
    double* f = (double*)calloc((size_t)(rounds > 0 ? rounds : 1), sizeof(double));
    double* g = (double*)calloc((size_t)(rounds > 0 ? rounds : 1), sizeof(double));
    uint8_t* fe = (uint8_t*)calloc((size_t)(rounds > 0 ? rounds : 1), 1);
    int64_t feasible_total = 0, sample_total = 0;
    int rc = TGO_OK;
    for (int rep = 0; rep < j_repeats; ++rep) {
        tgo_run_cfg c = *cfg;
        c.n_penalties = 1;
        c.penalties = &p_fixed;
        c.seed = tgo_derive(cfg->seed, 5, (uint64_t)rep);
        tgo_outputs o;
        memset(&o, 0, sizeof o);
        o.f = f;
        o.g = g;
        o.feasible = fe;
        rc = tgo_run_2dpt(prob, &c, &o, err, errlen);
        if (rc != TGO_OK) break;
        for (int64_t k = 0; k < rounds; ++k) {
            if (rep == 0) {
                if (out->round) out->round[k] = k + 1;
                if (out->sweep_count) out->sweep_count[k] = (k + 1) * cfg->sweeps_per_swap;
                if (out->best_f) out->best_f[k] = NAN;
                if (out->any_feasible) out->any_feasible[k] = 0;
                if (out->n_feasible) out->n_feasible[k] = 0;
                if (out->n_total) out->n_total[k] = 0;
            }
            if (out->n_total) ++out->n_total[k];
            ++sample_total;
            if (fe[k]) {
                if (out->n_feasible) ++out->n_feasible[k];
                ++feasible_total;
                if (out->best_f && (!out->any_feasible[k] || f[k] < out->best_f[k])) out->best_f[k] = f[k];
                if (out->any_feasible) out->any_feasible[k] = 1;
            }
        }
    }
    if (rc == TGO_OK && out->feasible_fraction)
        *out->feasible_fraction = sample_total == 0 ? 0.0 : (double)feasible_total / (double)sample_total;
    free(f);
    free(g);
    free(fe);
    return rc;
}

/* probe_population, schedule.cpp:18-52: n_chains independent chains at
 * (beta, P), each on ONE stream derive_seed(seed, probe = 4, c) that first
 * draws the random initial state (ising.cpp:15-19) and then one uniform per
 * spin per sweep; the second half of every chain's per-sweep (E = f + P g, g)
 * is pooled in chain-major order. */
int tgo_probe_population(const tgo_problem* prob, double beta, double penalty, int n_chains,
                         int sweeps, uint64_t seed, int rule, tgo_probe_stats* out, char* err,
                         int errlen) {
    if (n_chains < 2) { set_err(err, errlen, "probe: need at least 2 chains"); return TGO_CONFIG_ERROR; }
    if (sweeps < 2) { set_err(err, errlen, "probe: need at least 2 sweeps"); return TGO_CONFIG_ERROR; }
    model_t cost;
    cset_t cs;
    view_t v;
    int rc = model_build(&cost, prob->n, prob->n_couplings, prob->ci, prob->cj, prob->cw,
                         prob->fields, err, errlen);
    if (rc) return rc;
    rc = cset_build(&cs, prob->n, prob->n_pairs, prob->pa, prob->pb, err, errlen);
    if (rc) { model_free(&cost); return rc; }
    rc = view_build(&v, &cost, &cs, penalty, err, errlen);
    if (rc) { cset_free(&cs); model_free(&cost); return rc; }
    const int n = prob->n, burn_in = sweeps / 2;
    double sum_e = 0.0, sum_e2 = 0.0, sum_g = 0.0, sum_g2 = 0.0;
    int64_t kept = 0;
    rstate_t st;
    st.spins = (int8_t*)malloc((size_t)n);
    st.local = (double*)malloc(sizeof(double) * (size_t)n);
    st.id = 0;
    for (int c = 0; c < n_chains; ++c) {
        const uint64_t key = tgo_derive_seed(seed, 4, (uint64_t)c);
        uint64_t ctr = 0;
        for (int i = 0; i < n; ++i) st.spins[i] = (tgo_stream_bits(key, ctr++) >> 63) ? (int8_t)1 : (int8_t)-1;
        refresh(&v, &st);
        for (int s = 0; s < sweeps; ++s) {
            draw_ctx_t d;
            d.mode = TGO_RNG_SLOT;
            d.slot_seed = key;
            d.slot_ctr = &ctr;
            d.pkey = 0;
            d.t = 0;
            sweep(&v, beta, &st, &d, rule);
            if (s < burn_in) continue;
            const double e = st.f + penalty * st.g;
            sum_e += e;
            sum_e2 += e * e;
            sum_g += st.g;
            sum_g2 += st.g * st.g;
            ++kept;
        }
    }
    const double inv = 1.0 / (double)kept;
    out->row = out->column = 0;
    out->beta = beta;
    out->penalty = penalty;
    out->mean_g = sum_g * inv;
    const double mean_e = sum_e * inv;
    const double ve = sum_e2 * inv - mean_e * mean_e;
    out->sigma_e = sqrt(ve > 0.0 ? ve : 0.0);
    const double vg = sum_g2 * inv - out->mean_g * out->mean_g;
    out->sigma_g = sqrt(vg > 0.0 ? vg : 0.0);
    free(st.spins);
    free(st.local);
    model_free(&v.merged);
    cset_free(&cs);
    model_free(&cost);
    return TGO_OK;
}

static int cmp_double(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return x < y ? -1 : (x > y);
}

/* std::min / std::max semantics (NaN-order identical to <algorithm>) */
static inline double std_min(double a, double b) { return (b < a) ? b : a; }
static inline double std_max(double a, double b) { return (a < b) ? b : a; }

/* lower median, schedule.cpp:57-60 */
static double median_of(double* v, int n) {
    qsort(v, (size_t)n, sizeof(double), cmp_double);
    return v[(n - 1) / 2];
}

/* build_schedule, schedule.cpp:77-163.  The reference's std::map of
 * proposals keyed (row, column) is a dense [i_max][j_max + 2] table here;
 * collecting column j in row order equals the map's ordered iteration. */
int tgo_build_schedule(const tgo_problem* prob, const tgo_schedule_cfg* cfg, int rule,
                       double* betas, int* n_betas, double* penalties, int* n_penalties,
                       tgo_probe_stats* stats, int stats_cap, int* n_stats, int* budget_exhausted,
                       char* err, int errlen) {
    /* check_config, schedule.cpp:62-73 */
    if (cfg->beta0 <= 0.0) { set_err(err, errlen, "schedule: beta0 must be > 0"); return TGO_CONFIG_ERROR; }
    if (cfg->p0 < 0.0) { set_err(err, errlen, "schedule: P0 must be >= 0"); return TGO_CONFIG_ERROR; }
    if (cfg->i_max < 1 || cfg->j_max < 1) { set_err(err, errlen, "schedule: I_max and J_max must be >= 1"); return TGO_CONFIG_ERROR; }
    if (cfg->alpha_beta <= 0.0 || cfg->alpha_p <= 0.0) { set_err(err, errlen, "schedule: learning rates must be > 0"); return TGO_CONFIG_ERROR; }
    if (cfg->replica_budget < 1) { set_err(err, errlen, "schedule: replica budget must be >= 1"); return TGO_CONFIG_ERROR; }
    if ((long long)cfg->i_max * cfg->j_max > cfg->replica_budget) { set_err(err, errlen, "schedule: I_max * J_max exceeds replica budget"); return TGO_CONFIG_ERROR; }
    const double sigma_min = cfg->sigma_min > 0.0 ? cfg->sigma_min : 0.5 * sqrt((double)prob->n);
    const double p_cap = 2.0 * cfg->p0 + 1.0;
    const int IM = cfg->i_max, JC = cfg->j_max + 2;
    double* prop = (double*)calloc((size_t)IM * JC, sizeof(double));
    uint8_t* has = (uint8_t*)calloc((size_t)IM * JC, 1);
    double* cols = (double*)malloc(sizeof(double) * (size_t)IM * (cfg->j_max + 1));
    double* column = (double*)malloc(sizeof(double) * (size_t)IM);
    double* tmp = (double*)malloc(sizeof(double) * (size_t)(IM > cfg->j_max + 1 ? IM : cfg->j_max + 1));
    uint64_t probe_counter = 0;
    int ns = 0, np = 0, ncols = 0, rc = TGO_OK;
    *budget_exhausted = 0;
    penalties[np++] = cfg->p0;
#define PINC(beta, sg) std_min(cfg->alpha_p / ((beta) * std_max((sg), 1e-300)), p_cap)
#define PROBE(BETA_, PEN_, ROW_, COL_)                                                               \
    do {                                                                                        \
        rc = tgo_probe_population(prob, (BETA_), (PEN_), cfg->n_chains, cfg->sweeps_per_probe,    \
                                  tgo_derive_seed(cfg->seed, 4, probe_counter++), rule, &last,  \
                                  err, errlen);                                                 \
        if (rc) goto done;                                                                      \
        last.row = (ROW_);                                                                      \
        last.column = (COL_);                                                                   \
        if (ns < stats_cap) stats[ns] = last;                                                   \
        ++ns;                                                                                   \
    } while (0)
    tgo_probe_stats last;
    memset(&last, 0, sizeof last);
    int clen = 0;
    column[clen++] = cfg->beta0;
    for (int i = 0;; ++i) {
        PROBE(column[i], cfg->p0, i, 0);
        if (last.sigma_e <= sigma_min) break;
        prop[i * JC + 1] = cfg->p0 + PINC(column[i], last.sigma_g);
        has[i * JC + 1] = 1;
        if (i + 1 >= cfg->i_max) break;
        column[clen++] = column[i] + cfg->alpha_beta / last.sigma_e;
    }
    for (int i = 0; i < clen; ++i) cols[(size_t)ncols * IM + i] = column[i];
    ++ncols;
    const int n_rows = clen;
    if (last.mean_g >= 0.5) {
        int any = 0;
        for (int q = 0; q < IM * JC; ++q) any |= has[q];
        if (!any) { prop[0 * JC + 1] = cfg->p0 + PINC(cfg->beta0, last.sigma_g); has[1] = 1; }
        for (int j = 1;; ++j) {
            int nn = 0;
            for (int i = 0; i < IM; ++i)
                if (j < JC && has[i * JC + j]) tmp[nn++] = prop[i * JC + j];
            if ((long long)(j + 1) * n_rows > cfg->replica_budget || j >= cfg->j_max) {
                *budget_exhausted = 1;
                break;
            }
            const double prev = penalties[np - 1];
            const double med = median_of(tmp, nn);
            const double floor_ = prev + 1e-9 * (1.0 + fabs(prev));
            penalties[np++] = std_max(med, floor_);
            clen = 0;
            column[clen++] = cfg->beta0;
            for (int i = 0; i < n_rows; ++i) {
                PROBE(column[i], penalties[j], i, j);
                const double base = has[i * JC + j] ? prop[i * JC + j] : penalties[j];
                prop[i * JC + j + 1] = base + PINC(column[i], last.sigma_g);
                has[i * JC + j + 1] = 1;
                if (i + 1 < n_rows)
                    column[clen++] = column[i] + cfg->alpha_beta / std_max(last.sigma_e, sigma_min);
            }
            for (int i = 0; i < clen; ++i) cols[(size_t)ncols * IM + i] = column[i];
            ++ncols;
            if (last.mean_g < 0.5) break;
        }
    }
    for (int i = 0; i < n_rows; ++i) {
        for (int q = 0; q < ncols; ++q) tmp[q] = cols[(size_t)q * IM + i];
        betas[i] = median_of(tmp, ncols);
    }
    *n_betas = n_rows;
    *n_penalties = np;
    *n_stats = ns;
#undef PROBE
#undef PINC
done:
    free(prop);
    free(has);
    free(cols);
    free(column);
    free(tmp);
    return rc;
}

/* enumerate_boltzmann (oracle.cpp:86-165): energies by encoding (bit i of the
 * encoding = spin i is +1, oracle.cpp:17-29), max-shifted exponentials summed
 * in encoding order, then normalised. */
int tgo_enumerate_boltzmann(const tgo_problem* lp, double beta, double* probs,
                            double* log_partition, char* err, int errlen) {
    if (lp->n > 24) {
        set_err(err, errlen, "exact enumeration refused for %d spins (limit 24)", lp->n);
        return TGO_RESOURCE_ERROR;
    }
    model_t m;
    int rc = model_build(&m, lp->n, lp->n_couplings, lp->ci, lp->cj, lp->cw, lp->fields, err, errlen);
    if (rc) return rc;
    const uint64_t K = (uint64_t)1 << lp->n;
    int8_t* st = (int8_t*)malloc((size_t)lp->n);
    double max_log = -INFINITY;
    for (uint64_t enc = 0; enc < K; ++enc) {
        for (int i = 0; i < lp->n; ++i) st[i] = ((enc >> i) & 1) ? (int8_t)1 : (int8_t)-1;
        probs[enc] = model_energy(&m, st);
        const double x = -beta * probs[enc];
        if (max_log < x) max_log = x;
    }
    double sum = 0.0;
    for (uint64_t enc = 0; enc < K; ++enc) {
        probs[enc] = exp(-beta * probs[enc] - max_log);
        sum += probs[enc];
    }
    if (log_partition) *log_partition = max_log + log(sum);
    for (uint64_t enc = 0; enc < K; ++enc) probs[enc] /= sum;
    free(st);
    model_free(&m);
    return TGO_OK;
}

int tgo_kl_curve(const tgo_problem* prob, const tgo_run_cfg* cfg, const tgo_decoder* dec,
                 double beta, int discard_infeasible, int64_t* t, int64_t* samples, double* kl,
                 char* err, int errlen) {
    const int nl = dec->logical->n, n = prob->n;
    const uint64_t K = (uint64_t)1 << (nl > 24 ? 0 : nl);
    double* probs = (double*)malloc(sizeof(double) * (size_t)K);
    int rc = tgo_enumerate_boltzmann(dec->logical, beta, probs, NULL, err, errlen);
    if (rc) { free(probs); return rc; }
    const int64_t rounds = cfg->sweeps_per_swap >= 1 ? cfg->total_sweeps / cfg->sweeps_per_swap : 0;
    int8_t* states = (int8_t*)malloc((size_t)(rounds > 0 ? rounds : 1) * (size_t)n);
    tgo_outputs o;
    memset(&o, 0, sizeof o);
    o.states = states;
    rc = tgo_run_2dpt(prob, cfg, &o, err, errlen);
    uint64_t* cnt = (uint64_t*)calloc((size_t)K, sizeof(uint64_t));
    uint64_t total = 0;
    for (int64_t k = 0; rc == TGO_OK && k < rounds; ++k) {
        const int8_t* ph = states + (size_t)k * n;
        uint64_t enc = 0;
        int feasible = 1;
        for (int u = 0; u < nl; ++u) { /* decode, constraints.cpp:149-160 */
            int sum = 0;
            for (int q = dec->copy_off[u]; q < dec->copy_off[u + 1]; ++q) sum += ph[dec->copies[q]];
            const int8_t v = sum != 0 ? (sum > 0 ? 1 : -1) : ph[dec->copies[dec->copy_off[u]]];
            if (v > 0) enc |= (uint64_t)1 << u;
            for (int q = dec->copy_off[u]; q + 1 < dec->copy_off[u + 1]; ++q)
                if (ph[dec->copies[q]] != ph[dec->copies[q + 1]]) feasible = 0;
        }
        if (feasible || !discard_infeasible) { ++cnt[enc]; ++total; }
        t[k] = (k + 1) * cfg->sweeps_per_swap;
        samples[k] = (int64_t)total;
        if (total == 0) { kl[k] = NAN; continue; }
        double acc = 0.0; /* kl_divergence, oracle.cpp:178-195 (std::map order = ascending) */
        for (uint64_t e = 0; e < K; ++e) {
            if (!cnt[e]) continue;
            const double ph_ = (double)cnt[e] / (double)total;
            if (probs[e] <= 0.0) {
                set_err(err, errlen, "kl: target has zero mass on an observed state");
                rc = TGO_CONFIG_ERROR;
                break;
            }
            acc += ph_ * log(ph_ / probs[e]);
        }
        kl[k] = acc;
    }
    free(cnt);
    free(states);
    free(probs);
    return rc;
}
