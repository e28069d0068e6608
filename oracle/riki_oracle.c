/*
 * riki_oracle.c -- CPU ORACLE FOR TESTS ONLY.
 *
 * This file is test infrastructure.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * path (paper_2001_06770_b200/ + libriki.so) never links, imports or calls it,
 * and it shares no code, header, table or helper with csrc/.
 *
 * It is a plain, slow, single-threaded transcription of the paper
 * "Efficient Radial Pattern Keyword Search on Knowledge Graphs in Parallel"
 * (Yang & Tung, arXiv 2001.06770).  Citations "P:n" are lines of PAPER.md;
 * "R<n>" are the readings of SURVEY.md §8(c), restated in DESIGN.md §3.
 *
 *   orc_fine_weights  P:193-194      label-frequency weights, min-max rescale
 *   orc_coarsen       P:202-217      Eq. 1-3 reward/penalty coarsening (R1,R4,R5)
 *   orc_bound         P:242-251      Theorem boundEdgeWeight (diagnostic only)
 *   orc_path_score    P:229-236      Def. pathScoring
 *   orc_phase         P:343-464      initialisation, enqueue, identification,
 *                                    Alg. 1 expansion (literal, with re-scans)
 *   orc_search        P:301-381,503-561  two runs + Alg. 2 recovery + PTC + rank
 *                     P:293              optional weight-sum tie-break (tie_break 1, R29)
 *
 * Every floating-point expression is evaluated in IEEE fp64 in exactly the
 * order written here; the file must be compiled with -ffp-contract=off.
 * Parity status: every function is pinned by tests/test_oracle_*.py (worked
 * examples, closed forms, brute force); see DESIGN.md §4 for the pin list.
 */
#define _POSIX_C_SOURCE 199309L
#include <math.h>
#include <quadmath.h>
#include <stdint.h>
#include <time.h>
#include <stdlib.h>
#include <string.h>

#define ORC_INF 0xFFu /* h = infinity (unreached); all finite levels are <= 254 (R8) */

/* ------------------------------------------------------------------ */
/* small growable vectors                                              */
/* ------------------------------------------------------------------ */
typedef struct { uint32_t *a; uint64_t n, cap; } vu32;
typedef struct { uint64_t *a; uint64_t n, cap; } vu64;

static void vu32_push(vu32 *v, uint32_t x) {
    if (v->n == v->cap) { v->cap = v->cap ? v->cap * 2 : 16; v->a = realloc(v->a, v->cap * sizeof(uint32_t)); }
    v->a[v->n++] = x;
}
static void vu64_push(vu64 *v, uint64_t x) {
    if (v->n == v->cap) { v->cap = v->cap ? v->cap * 2 : 16; v->a = realloc(v->a, v->cap * sizeof(uint64_t)); }
    v->a[v->n++] = x;
}
static int cmp_u32(const void *x, const void *y) {
    uint32_t a = *(const uint32_t *)x, b = *(const uint32_t *)y; return a < b ? -1 : a > b;
}
static int cmp_u64(const void *x, const void *y) {
    uint64_t a = *(const uint64_t *)x, b = *(const uint64_t *)y; return a < b ? -1 : a > b;
}
static void sort_unique_u32(vu32 *v) {
    if (!v->n) return;
    qsort(v->a, v->n, sizeof(uint32_t), cmp_u32);
    uint64_t m = 1;
    for (uint64_t i = 1; i < v->n; i++) if (v->a[i] != v->a[m - 1]) v->a[m++] = v->a[i];
    v->n = m;
}
static void sort_unique_u64(vu64 *v) {
    if (!v->n) return;
    qsort(v->a, v->n, sizeof(uint64_t), cmp_u64);
    uint64_t m = 1;
    for (uint64_t i = 1; i < v->n; i++) if (v->a[i] != v->a[m - 1]) v->a[m++] = v->a[i];
    v->n = m;
}

/* ------------------------------------------------------------------ */
/* Weighting                                               */
/* ------------------------------------------------------------------ */

/* w_ij = log(|{e_ix : l(e_ix) = l(e_ij)}| + |{e_xj : l(e_xj) = l(e_ij)}|)
 * over out-edges of v_i and in-edges of v_j; both counts include e_ij (R3); log is the
 * natural log (R2), its fp64 value correctly rounded (R31, orc_ln_count);
 * the label class is (label, inverse flag) as the caller encodes it in cls[].
 * rescale to [0,1] by min-max; all zero when max = min (R2). */
typedef struct { uint64_t key, e; } keyed_edge;
static int cmp_keyed(const void *x, const void *y) {
    const keyed_edge *a = x, *b = y;
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    return a->e < b->e ? -1 : a->e > b->e;
}

/* cnt[e] = number of edges e' with node[e'] == node[e] and cls[e'] == cls[e]: bucket the
 * edges by node (counting sort), sort each bucket's (class, e) pairs, and give every run of
 * equal classes its length. */
static int count_node_class(uint32_t V, uint64_t E, const uint32_t *node, const uint32_t *cls, uint64_t *cnt) {
    uint64_t *ptr = calloc((uint64_t)V + 2, sizeof(uint64_t));
    keyed_edge *b = malloc((E ? E : 1) * sizeof(keyed_edge));
    if (!ptr || !b) { free(ptr); free(b); return -2; }
    for (uint64_t e = 0; e < E; e++) ptr[node[e] + 2]++;
    for (uint64_t v = 0; v < V; v++) ptr[v + 2] += ptr[v + 1];
    for (uint64_t e = 0; e < E; e++) { keyed_edge *x = &b[ptr[node[e] + 1]++]; x->key = cls[e]; x->e = e; }
    for (uint64_t v = 0; v < V; v++) {
        uint64_t lo = ptr[v], hi = ptr[v + 1];
        qsort(b + lo, hi - lo, sizeof(keyed_edge), cmp_keyed);
        for (uint64_t r = lo; r < hi;) {
            uint64_t x = r;
            while (x < hi && b[x].key == b[r].key) x++;
            for (uint64_t t = r; t < x; t++) cnt[b[t].e] = x - r;
            r = x;
        }
    }
    free(ptr); free(b);
    return 0;
}

/* R31: the fp64 value of ln n for an integer n >= 1, correctly rounded: binary128 logq is
 * accurate to ~2^-112, so one rounding to 53 bits gives the nearest double (ln n is never
 * exactly a rounding midpoint for n > 1).  glibc's log is within ~0.52 ulp and is not. */
double orc_ln_count(uint64_t n) { return (double)logq((__float128)n); }

int orc_fine_weights(uint32_t V, uint64_t E, const uint32_t *src, const uint32_t *dst,
                     const uint32_t *cls, double *w01) {
    double *raw = w01;
    uint64_t *co = malloc((E ? E : 1) * sizeof(uint64_t)), *ci = malloc((E ? E : 1) * sizeof(uint64_t));
    if (!co || !ci) { free(co); free(ci); return -2; }
    /* |{e_ix : l(e_ix) = l(e_ij)}|: out-edges of the source with the edge's class;
     * |{e_xj : l(e_xj) = l(e_ij)}|: in-edges of the target with the edge's class */
    if (count_node_class(V, E, src, cls, co) || count_node_class(V, E, dst, cls, ci)) { free(co); free(ci); return -2; }
    /* R31: ln of the integer count, correctly rounded to fp64 -- evaluated in binary128
     * (113-bit) arithmetic and rounded once; memoised per distinct count */
    uint64_t cmax = 0;
    for (uint64_t e = 0; e < E; e++) if (co[e] + ci[e] > cmax) cmax = co[e] + ci[e];
    double *lnc = malloc((cmax + 1) * sizeof(double));
    uint8_t *have = calloc(cmax + 1, 1);
    if (!lnc || !have) { free(co); free(ci); free(lnc); free(have); return -2; }
    for (uint64_t e = 0; e < E; e++) {
        uint64_t n = co[e] + ci[e];
        if (!have[n]) { lnc[n] = orc_ln_count(n); have[n] = 1; }
        raw[e] = lnc[n];
    }
    free(co); free(ci); free(lnc); free(have);
    if (E == 0) return 0;
    double mn = raw[0], mx = raw[0];
    for (uint64_t e = 1; e < E; e++) { if (raw[e] < mn) mn = raw[e]; if (raw[e] > mx) mx = raw[e]; }
    for (uint64_t e = 0; e < E; e++) w01[e] = (mx == mn) ? 0.0 : (raw[e] - mn) / (mx - mn);
    return 0;
}

/* Eq. 1-3.  Reward = A*(alpha-w)/alpha, Penalty = A*(w-alpha)/(1-alpha);
 * a = Rounding(A - Reward) or Rounding(A + Penalty).  Rounding is half-up (R1),
 * A is the raw real average (R4), operation order fixed (R5). */
int orc_coarsen(double w, double alpha, double avg) {
    double x;
    if (w <= alpha) x = avg - (avg * (alpha - w)) / alpha;
    else            x = avg + (avg * (w - alpha)) / (1.0 - alpha);
    return (int)floor(x + 0.5);
}

void orc_coarsen_all(uint64_t n, const double *w, double alpha, double avg, uint8_t *a) {
    for (uint64_t i = 0; i < n; i++) a[i] = (uint8_t)orc_coarsen(w[i], alpha, avg);
}

/* Theorem boundEdgeWeight: half-open [lo, hi) containing w given a. */
void orc_bound(int a, double alpha, double avg, double *lo, double *hi) {
    int r = (int)floor(avg + 0.5); /* Rounding(A) */
    if (a < r) {
        *lo = alpha * (a - 0.5) / avg;
        *hi = alpha * (a + 0.5) / avg;
    } else if (a == r) {
        *lo = alpha * (a - 0.5) / avg;
        *hi = 1.0 + (a + 0.5 - 2.0 * avg) * (1.0 - alpha) / avg;
    } else {
        *lo = 1.0 + (a - 0.5 - 2.0 * avg) * (1.0 - alpha) / avg;
        *hi = 1.0 + (a + 0.5 - 2.0 * avg) * (1.0 - alpha) / avg;
    }
}

/* Def. pathScoring: F(single node) = 0; F(p) = max(F(prefix), a_last) + 1. */
int orc_path_score(const int *seq, int n) {
    if (n == 0) return 0;
    int prefix = orc_path_score(seq, n - 1);
    return (prefix > seq[n - 1] ? prefix : seq[n - 1]) + 1;
}

/* Eq. 6, additive combination, fixed evaluation order (R5, R22). */
double orc_rpg_score(double gamma, uint32_t sc, uint32_t sm) {
    return gamma * (double)sc + (1.0 - gamma) * (double)sm;
}

/* ------------------------------------------------------------------ */
/* Graph: plain adjacency in input edge order (P:339 CSR)              */
/* ------------------------------------------------------------------ */
typedef struct orc_graph {
    uint32_t V; uint64_t E;
    uint32_t *src, *dst; uint8_t *act;
    uint64_t *out_ptr, *out_e; /* out-edges of v: out_e[out_ptr[v] .. out_ptr[v+1]) */
    uint64_t *in_ptr, *in_e;   /* in-edges of v (N_i, Alg. 2 line 5) */
} orc_graph;

orc_graph *orc_graph_new(uint32_t V, uint64_t E, const uint32_t *src, const uint32_t *dst, const uint8_t *act) {
    orc_graph *g = calloc(1, sizeof(orc_graph));
    g->V = V; g->E = E;
    g->src = malloc((E + 1) * 4); g->dst = malloc((E + 1) * 4); g->act = malloc(E + 1);
    memcpy(g->src, src, E * 4); memcpy(g->dst, dst, E * 4); memcpy(g->act, act, E);
    g->out_ptr = calloc(V + 1, 8); g->in_ptr = calloc(V + 1, 8);
    g->out_e = malloc((E + 1) * 8); g->in_e = malloc((E + 1) * 8);
    for (uint64_t e = 0; e < E; e++) { g->out_ptr[src[e] + 1]++; g->in_ptr[dst[e] + 1]++; }
    for (uint32_t v = 0; v < V; v++) { g->out_ptr[v + 1] += g->out_ptr[v]; g->in_ptr[v + 1] += g->in_ptr[v]; }
    uint64_t *fo = malloc((V + 1) * 8), *fi = malloc((V + 1) * 8);
    memcpy(fo, g->out_ptr, (V + 1) * 8); memcpy(fi, g->in_ptr, (V + 1) * 8);
    for (uint64_t e = 0; e < E; e++) { g->out_e[fo[src[e]]++] = e; g->in_e[fi[dst[e]]++] = e; }
    free(fo); free(fi);
    return g;
}

void orc_graph_free(orc_graph *g) {
    if (!g) return;
    free(g->src); free(g->dst); free(g->act); free(g->out_ptr); free(g->in_ptr); free(g->out_e); free(g->in_e);
    free(g);
}

/* ------------------------------------------------------------------ */
/* Exploration phase, one run over T keyword columns       */
/* ------------------------------------------------------------------ */
enum { BLOCK_NONE = 0, BLOCK_ALL_TERMS = 1 /* central: CF when row complete */,
       BLOCK_MARGINAL = 2 /* stop rule P:373, only when T >= 2 (R11) */ };

typedef struct {
    uint32_t T;
    uint8_t *H;      /* V x T, node-major */
    uint8_t *block;  /* CF as the level it was set at, ORC_INF if never (R10) */
    uint8_t *F;      /* Frontier Flag Array shared by all keywords */
    uint32_t *phi;   /* extracted frontier queue Phi_l, ascending id */
    uint32_t nphi;
    int blocking;    /* 1 if identification sets CF in this run */
} phase_t;

static void phase_init(phase_t *p, const orc_graph *g, uint32_t T, const uint64_t *tptr, const uint32_t *tnodes,
                       int block_mode) {
    uint32_t V = g->V;
    p->T = T;
    p->H = malloc((uint64_t)V * T + 1);
    p->block = malloc(V + 1);
    p->F = calloc(V + 1, 1);
    p->phi = malloc((V + 1) * 4);
    p->nphi = 0;
    memset(p->H, ORC_INF, (uint64_t)V * T);
    memset(p->block, ORC_INF, V);
    /* "In the beginning, we set F_i of all keyword nodes to 1"; h = 0 at
     * keyword nodes (Def. pathScoring, single node scores 0; R6). */
    for (uint32_t j = 0; j < T; j++)
        for (uint64_t i = tptr[j]; i < tptr[j + 1]; i++) {
            uint32_t v = tnodes[i];
            p->H[(uint64_t)v * T + j] = 0;
            p->F[v] = 1;
        }
    p->blocking = (block_mode == BLOCK_ALL_TERMS) || (block_mode == BLOCK_MARGINAL && T >= 2);
}

static void phase_free(phase_t *p) { free(p->H); free(p->block); free(p->F); free(p->phi); }

/* Frontier enqueue: extract F = 1 in ascending id, then clear F. */
static void phase_enqueue(phase_t *p, uint32_t V) {
    p->nphi = 0;
    for (uint32_t v = 0; v < V; v++)
        if (p->F[v]) { p->phi[p->nphi++] = v; p->F[v] = 0; }
}

static int row_complete(const phase_t *p, uint32_t v) {
    for (uint32_t j = 0; j < p->T; j++) if (p->H[(uint64_t)v * p->T + j] == ORC_INF) return 0;
    return 1;
}
static uint32_t row_max(const phase_t *p, uint32_t v) {
    uint32_t m = 0;
    for (uint32_t j = 0; j < p->T; j++) { uint32_t h = p->H[(uint64_t)v * p->T + j]; if (h > m) m = h; }
    return m;
}

/* Result identification (Theorem identifyCG): over the extracted
 * frontiers in ascending id; a node with every column finite is identified,
 * gets CF (block) = l and score max_j h.  Appends (score, v) to *ids. */
static void phase_identify(phase_t *p, uint32_t l, vu64 *ids) {
    if (!p->blocking) return;
    for (uint32_t i = 0; i < p->nphi; i++) {
        uint32_t v = p->phi[i];
        if (p->block[v] != ORC_INF) continue;
        if (!row_complete(p, v)) continue;
        p->block[v] = (uint8_t)l;
        if (ids) vu64_push(ids, ((uint64_t)row_max(p, v) << 32) | v);
    }
}

/* Alg. 1, literal: for each frontier v_f with CF = 0, each keyword
 * t_i with h_fi <= l, each out-neighbour v_n: if a_fn > l then F_f = 1 (stays a
 * frontier) else if h_ni = inf then h_ni = l+1, F_n = 1. */
static void phase_expand(phase_t *p, const orc_graph *g, uint32_t l) {
    uint32_t T = p->T;
    for (uint32_t i = 0; i < p->nphi; i++) {
        uint32_t f = p->phi[i];
        if (p->block[f] != ORC_INF) continue;                       /* line 2: CF_f = 1 */
        for (uint32_t j = 0; j < T; j++) {                          /* line 4 */
            uint32_t sf = p->H[(uint64_t)f * T + j];                /* line 5 */
            if (sf > l) continue;                                   /* line 6 */
            for (uint64_t k = g->out_ptr[f]; k < g->out_ptr[f + 1]; k++) { /* line 8 */
                uint64_t e = g->out_e[k];
                uint32_t n = g->dst[e];
                if (g->act[e] > l) { p->F[f] = 1; continue; }       /* lines 9-11 */
                if (p->H[(uint64_t)n * T + j] != ORC_INF) continue; /* lines 12-14 */
                p->H[(uint64_t)n * T + j] = (uint8_t)(l + 1);       /* line 16 */
                p->F[n] = 1;                                        /* line 17 */
            }
        }
    }
}

/* relaxations R = sum_j #{e=(f->n): h_fj finite, L = max(h_fj, a_e),
 * L < L_end, L < block[f]} -- the (edge, keyword) pairs the method relaxes.  */
static uint64_t phase_relaxations(const phase_t *p, const orc_graph *g, uint32_t L_end) {
    uint64_t R = 0;
    for (uint32_t f = 0; f < g->V; f++)
        for (uint32_t j = 0; j < p->T; j++) {
            uint32_t h = p->H[(uint64_t)f * p->T + j];
            if (h == ORC_INF) continue;
            for (uint64_t k = g->out_ptr[f]; k < g->out_ptr[f + 1]; k++) {
                uint32_t a = g->act[g->out_e[k]];
                uint32_t L = h > a ? h : a;
                if (L < L_end && L < p->block[f]) R++;
            }
        }
    return R;
}

/* Raw exploration to depth D with no termination other than l = D or an empty
 * frontier (debug boundary riki_hitting_levels).  Returns L_end. */
int orc_phase(const orc_graph *g, uint32_t T, const uint64_t *tptr, const uint32_t *tnodes, uint32_t depth,
              int block_mode, uint8_t *H_out, uint8_t *block_out, uint64_t *relax_out) {
    phase_t p;
    phase_init(&p, g, T, tptr, tnodes, block_mode);
    uint32_t l = 0;
    for (;; l++) {
        phase_enqueue(&p, g->V);
        phase_identify(&p, l, NULL);
        if (l == depth || p.nphi == 0) break;
        phase_expand(&p, g, l);
    }
    if (H_out) memcpy(H_out, p.H, (uint64_t)g->V * T);
    if (block_out) memcpy(block_out, p.block, g->V);
    if (relax_out) *relax_out = phase_relaxations(&p, g, l);
    phase_free(&p);
    return (int)l;
}

/* ------------------------------------------------------------------ */
/* Recovery (Alg. 2) with R16 (block-aware) and R17 (seen)   */
/* ------------------------------------------------------------------ */
typedef struct {
    uint32_t *seen; uint32_t stamp; /* V-sized visit stamps for the per-keyword BFS */
} scratch_t;

/* One keyword column j: reverse BFS from the sources.  Edge e = (n -> q) is
 * recovered iff h_nj finite, h_qj = max(h_nj, a_e) + 1 (Lemma recover)
 * and max(h_nj, a_e) < block[n] (n really expanded over e; R16).  n is
 * continued from iff h_nj != 0 (Alg. 2 line 10) and not yet seen (R17). */
static void recover_col(const orc_graph *g, const phase_t *p, uint32_t j, const uint32_t *srcs, uint32_t nsrc,
                        scratch_t *s, vu64 *edges, vu32 *nodes) {
    uint32_t T = p->T;
    vu32 q = {0};
    s->stamp++;
    for (uint32_t i = 0; i < nsrc; i++) {
        if (s->seen[srcs[i]] == s->stamp) continue;
        s->seen[srcs[i]] = s->stamp;
        vu32_push(&q, srcs[i]);
    }
    for (uint64_t qi = 0; qi < q.n; qi++) {
        uint32_t v_q = q.a[qi];
        uint32_t hq = p->H[(uint64_t)v_q * T + j];
        for (uint64_t k = g->in_ptr[v_q]; k < g->in_ptr[v_q + 1]; k++) {
            uint64_t e = g->in_e[k];
            uint32_t v_n = g->src[e];
            uint32_t hn = p->H[(uint64_t)v_n * T + j];
            if (hn == ORC_INF) continue;
            uint32_t L = hn > g->act[e] ? hn : g->act[e];
            if (hq != L + 1 || L >= p->block[v_n]) continue;
            vu64_push(edges, e);
            vu32_push(nodes, v_n);
            if (hn != 0 && s->seen[v_n] != s->stamp) { s->seen[v_n] = s->stamp; vu32_push(&q, v_n); }
        }
    }
    free(q.a);
}

/* ------------------------------------------------------------------ */
/* PTC (Def. RPG) -- reading R19                            */
/* ------------------------------------------------------------------ */
static uint32_t uf_find(uint32_t *par, uint32_t x) { while (par[x] != x) { par[x] = par[par[x]]; x = par[x]; } return x; }

/* nodes: sorted unique node set of G^r; edges: sorted unique edge ids of G^r;
 * vc: sorted V_C; Hm: marginal matrix (T = nm).  mode 0/1: RPG-wide inclusive
 * (R19); mode 2: G^m-only; mode 3: SPEC exclusive. */
static int ptc_check(const orc_graph *g, const vu32 *nodes, const vu64 *edges, const vu32 *vc,
                     const uint8_t *Hm, uint32_t nm, int mode, const vu64 *medges, const vu32 *mnodes) {
    if (nm == 1) return 1; /* P:146 trivial case: connected to V_C by construction */
    const vu32 *N = nodes; const vu64 *Ed = edges;
    if (mode == 2) { N = mnodes; Ed = medges; }
    uint64_t n = N->n;
    uint8_t *isx = calloc(n + 1, 1), *invc = calloc(n + 1, 1);
    int any_x_in_vc = 0;
    uint64_t nx = 0;
    for (uint64_t i = 0; i < n; i++) {
        uint32_t v = N->a[i];
        for (uint32_t t = 0; t < nm; t++) if (Hm[(uint64_t)v * nm + t] == 0) isx[i] = 1;
        invc[i] = bsearch(&v, vc->a, vc->n, 4, cmp_u32) != NULL;
        if (isx[i] && invc[i]) any_x_in_vc = 1;
        nx += isx[i];
    }
    int pass;
    /* P:145 "at least two different marginal keyword nodes" (R19'): a pair with an
     * endpoint on V_C qualifies; otherwise the pair must be separated by V_C. */
    if (nx < 2) pass = 0;
    else if (mode != 3 && any_x_in_vc) pass = 1;
    else {
        uint32_t *par = malloc((n + 1) * 4);
        for (uint64_t i = 0; i < n; i++) par[i] = (uint32_t)i;
        for (uint64_t i = 0; i < Ed->n; i++) {
            uint64_t e = Ed->a[i];
            uint32_t a = g->src[e], b = g->dst[e];
            uint32_t *pa = bsearch(&a, N->a, n, 4, cmp_u32), *pb = bsearch(&b, N->a, n, 4, cmp_u32);
            if (!pa || !pb) continue;
            uint64_t ia = pa - N->a, ib = pb - N->a;
            if (invc[ia] || invc[ib]) continue;  /* G^r minus V_C (undirected) */
            uint32_t ra = uf_find(par, (uint32_t)ia), rb = uf_find(par, (uint32_t)ib);
            if (ra != rb) par[ra] = rb;
        }
        /* X meets >= 2 components of G^r - V_C (X restricted to nodes outside V_C) */
        int64_t first = -1; pass = 0;
        for (uint64_t i = 0; i < n; i++) {
            if (!isx[i] || invc[i]) continue;
            uint32_t r = uf_find(par, (uint32_t)i);
            if (first < 0) first = r; else if ((uint32_t)first != r) { pass = 1; break; }
        }
        free(par);
    }
    free(isx); free(invc);
    return pass;
}

/* ------------------------------------------------------------------ */
/* Full search (Def. RPKSP; framework run twice) */
/* ------------------------------------------------------------------ */
typedef struct {
    double gamma;      /* Eq. 6 (R22 default 0.5) */
    uint32_t beam_w;   /* 0 -> k */
    int beam_mode;     /* 0 keep ties at the terminating level (R13 default), 1 truncate to w */
    int ptc_mode;      /* 0 filter (R19/R20), 1 flag only, 2 filter G^m-only, 3 filter SPEC-exclusive */
    int early_term;    /* 0 exact bound (R21), 1 paper-literal inequality, 2 none (exhaustive) */
    int tie_break;     /* 0 (S^r, S^c, v) (R23); 1 (S^r, S^c, W, v), W = edge-weight sum (R29) */
    const double *wfine; /* tie_break 1: fine edge weights w01[e] by caller edge id */
} orc_params;

typedef struct {
    uint32_t v, sc, sm;
    double sr;
    int attached, ptc;
    vu32 nodes; vu64 edges; vu32 vc;   /* CG then RPG node/edge sets */
    vu32 cnodes; vu64 cedges;          /* CG part */
    vu32 mnodes; vu64 medges;          /* G^m part */
    uint8_t *cdist, *mdist;
    uint64_t wsum;                     /* tie_break 1: W of the CG (beam) or of the RPG (ranking) */
} cand_t;

typedef struct orc_result {
    uint32_t nc, nm, k;
    uint32_t ncand; cand_t *cand;      /* candidate CGs in (S^c, v) order */
    uint32_t nres; uint32_t *res;      /* indices into cand, ranked */
    uint8_t *Hc, *Hm, *bc, *bm;        /* final matrices and block arrays */
    uint32_t V;
    int Lc, Lm;                        /* terminating levels (-1 if the run did not happen) */
    uint64_t relax_c, relax_m;
    uint32_t n_attached, n_ptc_fail;
    double t_central, t_marginal;      /* seconds (steady clock): run 1 + CG recovery, then run 2 */
} orc_result;

/* steady clock for the phase split of the timing protocol (Fig. 5 analogue) */
static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static int key_less(const cand_t *a, const cand_t *b, int tie) {
    /* (S^r, S^c, v) ascending (R23); tie_break 1: (S^r, S^c, W, v) -- P:293 "break the ties
       by a re-ranking operation, e.g. using the sum of edge weights" (R29: smaller W first) */
    if (a->sr != b->sr) return a->sr < b->sr;
    if (a->sc != b->sc) return a->sc < b->sc;
    if (tie && a->wsum != b->wsum) return a->wsum < b->wsum;
    return a->v < b->v;
}

/* R29: a fine weight w in [0,1] as the integer round(w * 2^32) (w * 2^32 is exact in fp64,
   so the sum below is exact and independent of the summation order). */
static uint64_t weight_fixed(double w) { return (uint64_t)floor(w * 4294967296.0 + 0.5); }

/* W(G) = sum of the fine weights of the DISTINCT edges of G (edges sorted, unique). */
static uint64_t edge_weight_sum(const vu64 *edges, const double *wfine) {
    uint64_t W = 0;
    for (uint64_t i = 0; i < edges->n; i++) W += weight_fixed(wfine[edges->a[i]]);
    return W;
}

/* Insertion into the running k-best list (indices into cand), ascending keys. */
static void kbest_insert(uint32_t *kb, uint32_t *nkb, uint32_t k, cand_t *cand, uint32_t c, int tie) {
    uint32_t pos = *nkb;
    while (pos > 0 && key_less(&cand[c], &cand[kb[pos - 1]], tie)) pos--;
    if (pos >= k) return;
    uint32_t end = *nkb < k ? *nkb : k - 1;
    for (uint32_t i = end; i > pos; i--) kb[i] = kb[i - 1];
    kb[pos] = c;
    if (*nkb < k) (*nkb)++;
}

static void merge_sets(cand_t *c) {
    c->nodes.n = 0; c->edges.n = 0;
    for (uint64_t i = 0; i < c->cnodes.n; i++) vu32_push(&c->nodes, c->cnodes.a[i]);
    for (uint64_t i = 0; i < c->mnodes.n; i++) vu32_push(&c->nodes, c->mnodes.a[i]);
    for (uint64_t i = 0; i < c->cedges.n; i++) vu64_push(&c->edges, c->cedges.a[i]);
    for (uint64_t i = 0; i < c->medges.n; i++) vu64_push(&c->edges, c->medges.a[i]);
    sort_unique_u32(&c->nodes); sort_unique_u64(&c->edges);
}

orc_result *orc_search(const orc_graph *g,
                       uint32_t nc, const uint64_t *cptr, const uint32_t *cnodes,
                       uint32_t nm, const uint64_t *mptr, const uint32_t *mnodes,
                       uint32_t k, uint32_t depth, const orc_params *prm) {
    orc_params P = {0.5, 0, 0, 0, 0, 0, NULL};
    if (prm) P = *prm;
    const int tie = P.tie_break == 1 && P.wfine != NULL;
    uint32_t w = P.beam_w ? P.beam_w : k;
    orc_result *r = calloc(1, sizeof(orc_result));
    r->nc = nc; r->nm = nm; r->k = k; r->V = g->V; r->Lc = -1; r->Lm = -1;
    scratch_t s; s.seen = calloc(g->V + 1, 4); s.stamp = 0;
    const double t0 = now_s();

    /* ---- first run: central keywords -> candidate CGs ---- */
    phase_t pc;
    phase_init(&pc, g, nc, cptr, cnodes, BLOCK_ALL_TERMS);
    vu64 ids = {0};
    uint32_t l = 0;
    for (;; l++) {
        phase_enqueue(&pc, g->V);
        phase_identify(&pc, l, &ids);
        /* P:362 "terminates once we collect at least w CGs"; R8 depth; empty frontier */
        if (ids.n >= w || l == depth || pc.nphi == 0) break;
        phase_expand(&pc, g, l);
    }
    r->Lc = (int)l;
    r->relax_c = phase_relaxations(&pc, g, l);
    /* candidates: all CGs identified by the terminating level, ordered by (S^c, v) (R13) */
    sort_unique_u64(&ids);
    uint32_t ncand = (uint32_t)ids.n;
    if (P.beam_mode == 1 && ncand > w && !tie) ncand = w;  /* (tie-break: truncated after recovery) */
    r->ncand = ncand;
    r->cand = calloc(ncand + 1, sizeof(cand_t));
    for (uint32_t i = 0; i < ncand; i++) {
        cand_t *c = &r->cand[i];
        c->v = (uint32_t)ids.a[i]; c->sc = (uint32_t)(ids.a[i] >> 32);
        c->cdist = malloc(nc + 1); c->mdist = malloc(nm + 1);
        for (uint32_t j = 0; j < nc; j++) c->cdist[j] = pc.H[(uint64_t)c->v * nc + j];
        /* Alg. 2: recover SP(c_j, v) for every central keyword */
        vu32_push(&c->cnodes, c->v);
        for (uint32_t j = 0; j < nc; j++) recover_col(g, &pc, j, &c->v, 1, &s, &c->cedges, &c->cnodes);
        sort_unique_u32(&c->cnodes); sort_unique_u64(&c->cedges);
        /* V_C: CG nodes holding >= 1 central keyword (R15) */
        for (uint64_t t = 0; t < c->cnodes.n; t++) {
            uint32_t v = c->cnodes.a[t];
            for (uint32_t j = 0; j < nc; j++) if (pc.H[(uint64_t)v * nc + j] == 0) { vu32_push(&c->vc, v); break; }
        }
        if (tie) c->wsum = edge_weight_sum(&c->cedges, P.wfine);
    }
    free(ids.a);
    if (tie && P.beam_mode == 1 && ncand > w) {
        /* beam of width w with the tie-break (R29): the w smallest (S^c, W(CG), v), then back
           to (S^c, v) order; the dropped candidates are released */
        for (uint32_t i = 1; i < ncand; i++)        /* insertion sort by (S^c, W, v) */
            for (uint32_t j = i; j > 0; j--) {
                cand_t *a = &r->cand[j - 1], *b = &r->cand[j];
                int less = b->sc != a->sc ? b->sc < a->sc : b->wsum != a->wsum ? b->wsum < a->wsum : b->v < a->v;
                if (!less) break;
                cand_t t = *a; *a = *b; *b = t;
            }
        for (uint32_t i = w; i < ncand; i++) {
            cand_t *c = &r->cand[i];
            free(c->cnodes.a); free(c->cedges.a); free(c->vc.a); free(c->cdist); free(c->mdist);
            memset(c, 0, sizeof(*c));
        }
        ncand = w;
        r->ncand = w;
        for (uint32_t i = 1; i < ncand; i++)        /* (S^c, v) order */
            for (uint32_t j = i; j > 0; j--) {
                cand_t *a = &r->cand[j - 1], *b = &r->cand[j];
                int less = b->sc != a->sc ? b->sc < a->sc : b->v < a->v;
                if (!less) break;
                cand_t t = *a; *a = *b; *b = t;
            }
    }

    uint32_t *kb = calloc(k + 1, 4), nkb = 0;
    const double t1 = now_s();
    r->t_central = t1 - t0;
    if (nm == 0) {
        /* M = empty is a classic keyword search: top-k CGs by (S^c, v) */
        for (uint32_t i = 0; i < ncand; i++) {
            cand_t *c = &r->cand[i];
            c->attached = 1; c->ptc = 1; c->sm = 0; c->sr = (double)c->sc;
            merge_sets(c);
            if (tie) c->wsum = edge_weight_sum(&c->edges, P.wfine);
            kbest_insert(kb, &nkb, k, r->cand, i, tie);
        }
    } else {
        /* ---- second run: marginal keywords with a fresh H (R12) ---- */
        phase_t pm;
        phase_init(&pm, g, nm, mptr, mnodes, BLOCK_MARGINAL);
        uint32_t unattached = ncand;
        for (l = 0;; l++) {
            phase_enqueue(&pm, g->V);
            phase_identify(&pm, l, NULL);
            /* attach (R14): D_gi = min over V_C of h_m[v][i], all finite -> RPG */
            for (uint32_t ci = 0; ci < ncand; ci++) {
                cand_t *c = &r->cand[ci];
                if (c->attached) continue;
                int ok = 1; uint32_t sm = 0;
                for (uint32_t i = 0; i < nm; i++) {
                    uint32_t d = ORC_INF;
                    for (uint64_t t = 0; t < c->vc.n; t++) {
                        uint32_t h = pm.H[(uint64_t)c->vc.a[t] * nm + i];
                        if (h < d) d = h;
                    }
                    c->mdist[i] = (uint8_t)d;
                    if (d == ORC_INF) ok = 0; else if (d > sm) sm = d;
                }
                if (!ok) continue;
                c->attached = 1; unattached--; r->n_attached++;
                c->sm = sm;                                       /* Eq. 5 */
                c->sr = orc_rpg_score(P.gamma, c->sc, c->sm);     /* Eq. 6 */
                /* RPG recovery (R18): per marginal, from V_C nodes at the min distance */
                for (uint32_t i = 0; i < nm; i++) {
                    vu32 starts = {0};
                    for (uint64_t t = 0; t < c->vc.n; t++)
                        if (pm.H[(uint64_t)c->vc.a[t] * nm + i] == c->mdist[i]) vu32_push(&starts, c->vc.a[t]);
                    for (uint64_t t = 0; t < starts.n; t++) vu32_push(&c->mnodes, starts.a[t]);
                    recover_col(g, &pm, i, starts.a, (uint32_t)starts.n, &s, &c->medges, &c->mnodes);
                    free(starts.a);
                }
                sort_unique_u32(&c->mnodes); sort_unique_u64(&c->medges);
                merge_sets(c);
                if (tie) c->wsum = edge_weight_sum(&c->edges, P.wfine);  /* W(G^r), G^r = CG u G^m */
                c->ptc = ptc_check(g, &c->nodes, &c->edges, &c->vc, pm.H, nm, P.ptc_mode, &c->medges, &c->mnodes);
                if (!c->ptc) r->n_ptc_fail++;
                if (c->ptc || P.ptc_mode == 1) kbest_insert(kb, &nkb, k, r->cand, ci, tie);
            }
            /* termination (P:375-381 with R21) */
            int stop = (l == depth) || (pm.nphi == 0) || (unattached == 0);
            if (!stop && nkb >= k && P.early_term != 2) {
                const cand_t *kth = &r->cand[kb[k - 1]];
                if (P.early_term == 0) {
                    int all_worse = 1;
                    for (uint32_t ci = 0; ci < ncand && all_worse; ci++) {
                        const cand_t *c = &r->cand[ci];
                        if (c->attached) continue;
                        cand_t best = *c;
                        best.sr = orc_rpg_score(P.gamma, c->sc, l + 1);
                        /* best <= kth: could still enter.  With the tie-break its W is unknown
                           until it attaches, so only a strictly larger (S^r, S^c) excludes it */
                        if (tie ? !(kth->sr < best.sr || (kth->sr == best.sr && kth->sc < best.sc))
                                : !key_less(kth, &best, 0))
                            all_worse = 0;
                    }
                    stop = all_worse;
                } else {
                    uint32_t mins = ORC_INF;
                    for (uint32_t ci = 0; ci < ncand; ci++)
                        if (!r->cand[ci].attached && r->cand[ci].sc < mins) mins = r->cand[ci].sc;
                    double rhs = P.gamma * (double)mins + (1.0 - P.gamma) * (double)kth->sm;
                    stop = (mins == ORC_INF) || kth->sr <= rhs;
                }
            }
            if (stop) break;
            phase_expand(&pm, g, l);
        }
        r->Lm = (int)l;
        r->relax_m = phase_relaxations(&pm, g, l);
        r->Hm = pm.H; r->bm = pm.block; pm.H = NULL; pm.block = NULL;
        free(pm.F); free(pm.phi);
    }
    r->nres = nkb; r->res = kb;
    r->t_marginal = now_s() - t1;
    r->Hc = pc.H; r->bc = pc.block; pc.H = NULL; pc.block = NULL;
    free(pc.F); free(pc.phi);
    free(s.seen);
    return r;
}

void orc_result_free(orc_result *r) {
    if (!r) return;
    for (uint32_t i = 0; i < r->ncand; i++) {
        cand_t *c = &r->cand[i];
        free(c->nodes.a); free(c->edges.a); free(c->vc.a); free(c->cnodes.a); free(c->cedges.a);
        free(c->mnodes.a); free(c->medges.a); free(c->cdist); free(c->mdist);
    }
    free(r->cand); free(r->res); free(r->Hc); free(r->Hm); free(r->bc); free(r->bm);
    free(r);
}

/* ---- accessors (plain C types for ctypes) ---- */
uint32_t orc_res_count(const orc_result *r) { return r->nres; }
void orc_res_times(const orc_result *r, double *t_central, double *t_marginal) {
    *t_central = r->t_central; *t_marginal = r->t_marginal;
}
uint32_t orc_res_ncand(const orc_result *r) { return r->ncand; }
void orc_res_levels(const orc_result *r, int *Lc, int *Lm, uint64_t *relax_c, uint64_t *relax_m,
                    uint32_t *n_attached, uint32_t *n_ptc_fail) {
    *Lc = r->Lc; *Lm = r->Lm; *relax_c = r->relax_c; *relax_m = r->relax_m;
    *n_attached = r->n_attached; *n_ptc_fail = r->n_ptc_fail;
}
/* candidate i (in (S^c, v) order): v, sc, attached, ptc, sm, sr */
void orc_res_cand(const orc_result *r, uint32_t i, uint32_t *v, uint32_t *sc, int *attached, int *ptc,
                  uint32_t *sm, double *sr, uint64_t *n_cnodes, uint64_t *n_cedges, uint64_t *n_vc) {
    const cand_t *c = &r->cand[i];
    *v = c->v; *sc = c->sc; *attached = c->attached; *ptc = c->ptc; *sm = c->sm; *sr = c->sr;
    *n_cnodes = c->cnodes.n; *n_cedges = c->cedges.n; *n_vc = c->vc.n;
}
void orc_res_cand_lists(const orc_result *r, uint32_t i, uint32_t *cnodes, uint64_t *cedges, uint32_t *vc) {
    const cand_t *c = &r->cand[i];
    if (cnodes) memcpy(cnodes, c->cnodes.a, c->cnodes.n * 4);
    if (cedges) memcpy(cedges, c->cedges.a, c->cedges.n * 8);
    if (vc) memcpy(vc, c->vc.a, c->vc.n * 4);
}
/* ranked result i: candidate index, sizes */
uint64_t orc_res_wsum(const orc_result *r, uint32_t i) { return r->cand[r->res[i]].wsum; }
void orc_res_get(const orc_result *r, uint32_t i, uint32_t *cand_index, uint32_t *v, uint32_t *sc, uint32_t *sm,
                 double *sr, int *ptc, uint64_t *n_nodes, uint64_t *n_edges, uint64_t *n_vc) {
    const cand_t *c = &r->cand[r->res[i]];
    *cand_index = r->res[i]; *v = c->v; *sc = c->sc; *sm = c->sm; *sr = c->sr; *ptc = c->ptc;
    *n_nodes = c->nodes.n; *n_edges = c->edges.n; *n_vc = c->vc.n;
}
void orc_res_lists(const orc_result *r, uint32_t i, uint32_t *nodes, uint64_t *edges, uint32_t *vc,
                   uint8_t *cdist, uint8_t *mdist) {
    const cand_t *c = &r->cand[r->res[i]];
    if (nodes) memcpy(nodes, c->nodes.a, c->nodes.n * 4);
    if (edges) memcpy(edges, c->edges.a, c->edges.n * 8);
    if (vc) memcpy(vc, c->vc.a, c->vc.n * 4);
    if (cdist) memcpy(cdist, c->cdist, r->nc);
    if (mdist && r->nm) memcpy(mdist, c->mdist, r->nm);
}
/* phase 0 = central, 1 = marginal; copies V*T bytes of H and V bytes of block */
int orc_res_matrix(const orc_result *r, int phase, uint8_t *H, uint8_t *block) {
    const uint8_t *h = phase ? r->Hm : r->Hc, *b = phase ? r->bm : r->bc;
    uint32_t T = phase ? r->nm : r->nc;
    if (!h) return -1;
    if (H) memcpy(H, h, (uint64_t)r->V * T);
    if (block) memcpy(block, b, r->V);
    return 0;
}
