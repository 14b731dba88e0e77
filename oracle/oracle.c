/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct CPU
 * max-flow / min-cut for Wu-Chen proper-ordered multi-column graphs.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_2601_17026_b200/, libcolgraph.so) never includes, links or calls it,
 * and this file includes nothing from the product tree.
 *
 * What it computes (§1.2-1.3):
 *   - the s-t graph of a VCE-weight net-surface problem with vertex weights
 *     only ("The weights on the nodes w(v) are correspondingly
 *     converted to the costs associated with the edges connecting the node v
 *     to the source or the sink"), built EXPLICITLY (CSR adjacency lists) with
 *     the literal Wu-Chen arcs:
 *         s -> v  capacity -w(v)   if w(v) < 0
 *         v -> t  capacity  w(v)   if w(v) > 0
 *         (x,y,z) -> (x,y,z-1)                 capacity INF, z >= 1
 *         (x,y,z) -> (x',y',max(0, z-Delta))    capacity INF, every z, every
 *                                              in-range 4-neighbour (x',y')
 *     with w(x,y,0) = c(x,y,0) - (sum_z c(x,y,z) + 1) and
 *          w(x,y,z) = c(x,y,z) - c(x,y,z-1), z >= 1     (reading R1)
 *   - the maximum flow value |f| = sum_v f(v,t) (Eq. 5) by
 *     Dinitz blocking flows over BFS level graphs (§2) or by
 *     Edmonds-Karp shortest augmenting paths (§2);
 *   - the minimal min-cut source set S = vertices reachable from s in the
 *     residual graph r_f(u,v) = c(u,v) - f(u,v) > 0 (§2.1;
 *     cut definition Eq. 6-7; Theorem 1);
 *   - the surface S(x,y) = max { z : (x,y,z) in S }, or -1 and
 *     status 6 (EMPTY_COLUMN) for a column with no source-side
 *     vertex;
 *   - self-checks: capacity (Eq. 2), antisymmetry of each arc pair (Eq. 3),
 *     conservation at non-terminals (Eq. 4), |f| = net flow out of s,
 *     t not in S, cut capacity c(S, V-S) = |f| with no INF arc crossing
 *     (Theorem 1 / Eq. 6).
 *
 * All arithmetic is int64; INF = 2^62.  Single-threaded.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_INF ((int64_t)1 << 62)

enum { OR_OK = 0, OR_E_INVAL = 1, OR_E_NOMEM = 3, OR_E_EMPTY_COLUMN = 6 };

/* check bits returned in *checks (all set = every invariant holds) */
enum {
    CHK_CAPACITY = 1 << 0,     /* 0 <= f <= c on every arc (Eq. 2) */
    CHK_ANTISYM = 1 << 1,      /* res[a] + res[rev a] == cap[a] + cap[rev a] (Eq. 3) */
    CHK_CONSERVE = 1 << 2,     /* inflow == outflow at every non-terminal (Eq. 4) */
    CHK_VALUE = 1 << 3,        /* flow into t == flow out of s (Eq. 5) */
    CHK_T_NOT_IN_S = 1 << 4,   /* no augmenting path */
    CHK_CUT_EQ_FLOW = 1 << 5,  /* c(S, V-S) == |f|, no INF arc crosses (Theorem 1) */
};

typedef struct {
    int64_t nn;      /* nodes including s, t */
    int64_t m;       /* half-arcs */
    int64_t *first;  /* CSR offsets, nn + 1 */
    int32_t *head;
    int64_t *rev;
    int64_t *cap;    /* original capacity */
    int64_t *res;    /* residual capacity */
    int64_t *fill;   /* scratch insertion cursor */
} graph_t;

static void g_free(graph_t *g) {
    free(g->first); free(g->head); free(g->rev); free(g->cap); free(g->res); free(g->fill);
    memset(g, 0, sizeof(*g));
}

/* ---- explicit graph construction: two passes (count, then insert) ---- */

static void add_arc(graph_t *g, int pass, int64_t u, int64_t v, int64_t c) {
    if (pass == 0) {
        g->first[u + 1]++;
        g->first[v + 1]++;
        return;
    }
    int64_t a = g->fill[u]++;
    int64_t b = g->fill[v]++;
    g->head[a] = (int32_t)v; g->cap[a] = c; g->res[a] = c; g->rev[a] = b;
    g->head[b] = (int32_t)u; g->cap[b] = 0; g->res[b] = 0; g->rev[b] = a;
}

static int g_alloc(graph_t *g, int64_t nn) {
    memset(g, 0, sizeof(*g));
    g->nn = nn;
    g->first = (int64_t *)calloc((size_t)nn + 1, sizeof(int64_t));
    return g->first ? 0 : -1;
}

static int g_finish_count(graph_t *g) {
    for (int64_t i = 0; i < g->nn; i++) g->first[i + 1] += g->first[i];
    g->m = g->first[g->nn];
    size_t m = (size_t)(g->m ? g->m : 1);
    g->head = (int32_t *)malloc(m * sizeof(int32_t));
    g->rev = (int64_t *)malloc(m * sizeof(int64_t));
    g->cap = (int64_t *)malloc(m * sizeof(int64_t));
    g->res = (int64_t *)malloc(m * sizeof(int64_t));
    g->fill = (int64_t *)malloc((size_t)g->nn * sizeof(int64_t));
    if (!g->head || !g->rev || !g->cap || !g->res || !g->fill) return -1;
    memcpy(g->fill, g->first, (size_t)g->nn * sizeof(int64_t));
    return 0;
}

/* Vertex weights of the net-surface construction (reading R1). */
static void column_weights(const int32_t *c, int64_t Z, int64_t col, int64_t *w) {
    const int32_t *cc = c + col * Z;
    int64_t sum = 0;
    for (int64_t z = 0; z < Z; z++) sum += cc[z];
    w[0] = (int64_t)cc[0] - (sum + 1);
    for (int64_t z = 1; z < Z; z++) w[z] = (int64_t)cc[z] - (int64_t)cc[z - 1];
}

/* Narrow band (the graphs are narrow bands around
 * landmarks): the surface of column col is confined to [lo, hi).  The base rule R1 applies to the
 * band: w(lo) = c(lo) - (sum_{lo <= z < hi} c(z) + 1), w(z) = c(z) - c(z-1) for lo < z < hi, and
 * every vertex outside the band has no terminal arc (w = 0).  The infinite down arcs put the
 * vertices below the band into every source set that contains (col, lo), i.e. every one, and no
 * arc of the original graph leads into the vertices above the band from below, so the minimal
 * source set never contains them: S(col) = max{z in S} lies in [lo, hi). */
static void column_weights_band(const int32_t *c, int64_t Z, int64_t col, int32_t lo, int32_t hi, int64_t *w) {
    const int32_t *cc = c + col * Z;
    int64_t sum = 0;
    for (int64_t z = lo; z < hi; z++) sum += cc[z];
    for (int64_t z = 0; z < Z; z++) w[z] = 0;
    w[lo] = (int64_t)cc[lo] - (sum + 1);
    for (int64_t z = lo + 1; z < hi; z++) w[z] = (int64_t)cc[z] - (int64_t)cc[z - 1];
}

/* Inter-column arcs (x,y,z) -> (x',y',max(0,z-Delta_d)): the edge interval toward the
 * adjacent column in direction d.  dl[d] for d = +x, -x, +y, -y: the arc of p
 * toward its neighbour q in direction d encodes S(p) - S(q) <= dl[d], so the pair (p, q = p + x)
 * has S(q) - S(p) in [-dl[+x], dl[-x]] -- a general (possibly asymmetric) proper-ordered edge
 * interval; dl = {D, D, D, D} is the paper's isotropic case and
 * {Dx, Dx, Dy, Dy} the anisotropic one. */
/* Soft smoothness (VCE-weight net surface): a convex
 * penalty f(d) for |S(p) - S(q)| = d adds finite arcs (x,y,z) -> (x',y',z-k), k = 0..Delta_d-1,
 * z-k >= 0, with capacity c_0 = f(1), c_k = f(k+1) - 2f(k) + f(k-1): the arc is cut for
 * (d - k)_+ values of z, so the cut cost of the pair telescopes to f(d).
 * penalty[i] = f(i+1), npenalty >= max(Delta_x, Delta_y); NULL = hard constraint only. */
static const int32_t *g_penalty = NULL;
static int g_npenalty = 0;

static int64_t soft_cap(int k) {
    const int64_t f1 = g_penalty[k];                         /* f(k+1) */
    const int64_t f0 = k >= 1 ? g_penalty[k - 1] : 0;        /* f(k) */
    const int64_t fm = k >= 2 ? g_penalty[k - 2] : 0;        /* f(k-1) */
    return k == 0 ? f1 : f1 - 2 * f0 + fm;
}

static void colgraph_arcs(graph_t *g, int pass, const int32_t *in, int X, int Y, int Z, const int32_t *dl4,
                          const int32_t *band, int input_is_weight, int64_t *wbuf) {
    const int64_t n = (int64_t)X * Y * Z, s = n, t = n + 1;
    const int dx[4] = {+1, -1, 0, 0}, dy[4] = {0, 0, +1, -1};
    for (int64_t x = 0; x < X; x++)
        for (int64_t y = 0; y < Y; y++) {
            int64_t col = x * Y + y;
            if (input_is_weight) {
                for (int64_t z = 0; z < Z; z++) wbuf[z] = in[col * Z + z];
            } else if (band) {
                column_weights_band(in, Z, col, band[2 * col], band[2 * col + 1], wbuf);
            } else {
                column_weights(in, Z, col, wbuf);
            }
            for (int64_t z = 0; z < Z; z++) {
                int64_t v = col * Z + z;
                if (wbuf[z] < 0) add_arc(g, pass, s, v, -wbuf[z]);
                if (wbuf[z] > 0) add_arc(g, pass, v, t, wbuf[z]);
                if (z >= 1) add_arc(g, pass, v, v - 1, OR_INF);
                for (int d = 0; d < 4; d++) {
                    int64_t x2 = x + dx[d], y2 = y + dy[d];
                    if (x2 < 0 || x2 >= X || y2 < 0 || y2 >= Y) continue;
                    const int64_t dl = dl4[d];
                    const int64_t zt = z - dl > 0 ? z - dl : 0;
                    add_arc(g, pass, v, (x2 * Y + y2) * Z + zt, OR_INF);
                    for (int64_t k = 0; g_penalty && k < dl && z - k >= 0; k++) {
                        const int64_t cap = soft_cap((int)k);
                        if (cap > 0) add_arc(g, pass, v, (x2 * Y + y2) * Z + z - k, cap);
                    }
                }
            }
        }
}

/* ---- max-flow algorithms ---- */

static int bfs_levels(const graph_t *g, int64_t s, int64_t t, int32_t *level, int32_t *queue) {
    for (int64_t i = 0; i < g->nn; i++) level[i] = -1;
    int64_t qh = 0, qt = 0;
    level[s] = 0;
    queue[qt++] = (int32_t)s;
    while (qh < qt) {
        int64_t u = queue[qh++];
        for (int64_t a = g->first[u]; a < g->first[u + 1]; a++) {
            int64_t v = g->head[a];
            if (g->res[a] > 0 && level[v] < 0) {
                level[v] = level[u] + 1;
                queue[qt++] = (int32_t)v;
            }
        }
    }
    return level[t] >= 0;
}

/* Dinitz: blocking flow on the BFS level graph, iterative DFS with current-arc pointers. */
static int64_t dinic(graph_t *g, int64_t s, int64_t t, int *err) {
    int32_t *level = (int32_t *)malloc((size_t)g->nn * sizeof(int32_t));
    int32_t *queue = (int32_t *)malloc((size_t)g->nn * sizeof(int32_t));
    int64_t *it = (int64_t *)malloc((size_t)g->nn * sizeof(int64_t));
    int64_t *path = (int64_t *)malloc((size_t)g->nn * sizeof(int64_t));
    int64_t total = 0;
    if (!level || !queue || !it || !path) { *err = OR_E_NOMEM; goto done; }
    while (bfs_levels(g, s, t, level, queue)) {
        memcpy(it, g->first, (size_t)g->nn * sizeof(int64_t));
        int64_t depth = 0, v = s;
        for (;;) {
            if (v == t) {
                int64_t f = OR_INF;
                for (int64_t i = 0; i < depth; i++)
                    if (g->res[path[i]] < f) f = g->res[path[i]];
                for (int64_t i = 0; i < depth; i++) {
                    g->res[path[i]] -= f;
                    g->res[g->rev[path[i]]] += f;
                }
                total += f;
                int64_t k = 0;
                while (g->res[path[k]] > 0) k++;
                depth = k;
                v = g->head[g->rev[path[k]]]; /* tail of the first saturated arc */
                continue;
            }
            int64_t a = it[v], end = g->first[v + 1];
            while (a < end && !(g->res[a] > 0 && level[g->head[a]] == level[v] + 1)) a++;
            it[v] = a;
            if (a < end) {
                path[depth++] = a;
                v = g->head[a];
            } else {
                level[v] = -1; /* dead end in this phase */
                if (v == s) break;
                depth--;
                v = g->head[g->rev[path[depth]]];
                it[v]++;
            }
        }
    }
done:
    free(level); free(queue); free(it); free(path);
    return total;
}

/* Edmonds-Karp: repeated BFS shortest augmenting path. */
static int64_t edmonds_karp(graph_t *g, int64_t s, int64_t t, int *err) {
    int64_t *parent = (int64_t *)malloc((size_t)g->nn * sizeof(int64_t));
    int32_t *queue = (int32_t *)malloc((size_t)g->nn * sizeof(int32_t));
    int64_t total = 0;
    if (!parent || !queue) { *err = OR_E_NOMEM; goto done; }
    for (;;) {
        for (int64_t i = 0; i < g->nn; i++) parent[i] = -1;
        int64_t qh = 0, qt = 0;
        queue[qt++] = (int32_t)s;
        parent[s] = -2;
        while (qh < qt && parent[t] == -1) {
            int64_t u = queue[qh++];
            for (int64_t a = g->first[u]; a < g->first[u + 1]; a++) {
                int64_t v = g->head[a];
                if (g->res[a] > 0 && parent[v] == -1) {
                    parent[v] = a;
                    queue[qt++] = (int32_t)v;
                }
            }
        }
        if (parent[t] == -1) break;
        int64_t f = OR_INF;
        for (int64_t v = t; v != s; v = g->head[g->rev[parent[v]]])
            if (g->res[parent[v]] < f) f = g->res[parent[v]];
        for (int64_t v = t; v != s; v = g->head[g->rev[parent[v]]]) {
            g->res[parent[v]] -= f;
            g->res[g->rev[parent[v]]] += f;
        }
        total += f;
    }
done:
    free(parent); free(queue);
    return total;
}

/* Residual BFS from s: the minimal min-cut source set (mark[v] = 1). */
static int source_set(const graph_t *g, int64_t s, uint8_t *mark) {
    int32_t *queue = (int32_t *)malloc((size_t)g->nn * sizeof(int32_t));
    if (!queue) return -1;
    memset(mark, 0, (size_t)g->nn);
    int64_t qh = 0, qt = 0;
    mark[s] = 1;
    queue[qt++] = (int32_t)s;
    while (qh < qt) {
        int64_t u = queue[qh++];
        for (int64_t a = g->first[u]; a < g->first[u + 1]; a++) {
            int64_t v = g->head[a];
            if (g->res[a] > 0 && !mark[v]) { mark[v] = 1; queue[qt++] = (int32_t)v; }
        }
    }
    free(queue);
    return 0;
}

static int check_invariants(const graph_t *g, int64_t s, int64_t t, const uint8_t *mark, int64_t flow) {
    int ok = CHK_CAPACITY | CHK_ANTISYM | CHK_CONSERVE | CHK_VALUE | CHK_T_NOT_IN_S | CHK_CUT_EQ_FLOW;
    int64_t into_t = 0, out_s = 0, cut = 0;
    for (int64_t u = 0; u < g->nn; u++) {
        int64_t net = 0; /* inflow - outflow */
        for (int64_t a = g->first[u]; a < g->first[u + 1]; a++) {
            int64_t b = g->rev[a];
            if (g->res[a] < 0) ok &= ~CHK_CAPACITY;
            if (g->res[a] + g->res[b] != g->cap[a] + g->cap[b]) ok &= ~CHK_ANTISYM;
            if (g->cap[a] > 0) { /* forward (original) arc u -> head */
                int64_t f = g->cap[a] - g->res[a];
                if (f < 0 || f > g->cap[a]) ok &= ~CHK_CAPACITY;
                net -= f;
                if (g->head[a] == t) into_t += f;
                if (u == s) out_s += f;
                if (mark[u] && !mark[g->head[a]]) {
                    if (g->cap[a] >= OR_INF) ok &= ~CHK_CUT_EQ_FLOW;
                    else cut += g->cap[a];
                }
            } else if (g->cap[b] > 0) { /* reverse slot of an arc head -> u */
                net += g->cap[b] - g->res[b];
            }
        }
        if (u != s && u != t && net != 0) ok &= ~CHK_CONSERVE;
    }
    if (into_t != flow || out_s != flow) ok &= ~CHK_VALUE;
    if (mark[t]) ok &= ~CHK_T_NOT_IN_S;
    if (cut != flow) ok &= ~CHK_CUT_EQ_FLOW;
    return ok;
}

/*
 * Push-relabel (Goldberg-Tarjan; §2.1: labels, push, relabel, global
 * relabeling), textbook FIFO form in two phases so that it ends with a maximum FLOW:
 *   phase 1: labels d(v) = residual distance to t (exact by a global relabel -- BFS from t over
 *            reverse residual arcs -- at the start and after every n relabels); a vertex with
 *            excess and d(v) < n pushes on admissible arcs (residual > 0, d(v) = d(w) + 1), else
 *            relabels to 1 + min d(w) over residual arcs; ends when no vertex below n is active,
 *            i.e. with a maximum preflow;
 *   phase 2: the same with s as the terminal (labels = residual distance to s, by BFS from s over
 *            reverse residual arcs): every remaining excess returns to s, giving a maximum flow.
 * Slower to state than Dinitz but its work on column graphs does not grow with the number of
 * distinct augmenting-path lengths (C5's Dinitz run needs thousands of phases).  The result is
 * certified like the others (check_invariants: Eq. 2-5, Theorem 1) and pinned by the same tests.
 */
/* Exact labels: residual distance to `root` (t in phase 1, s in phase 2); the other terminal
 * gets n (never a push target: nothing flows into s in phase 1, or into t in phase 2).  In phase 2
 * excess reaches s only by cancelling flow on an arc s -> u (the reverse slot u -> s, capacity 0),
 * never over an original arc into s, so no flow enters s (as with augmenting paths). */
static void pr_global(const graph_t *g, int64_t root, int64_t other, int phase2, int64_t n, int64_t *d,
                      int32_t *queue) {
    for (int64_t i = 0; i < g->nn; i++) d[i] = n;  /* n: cannot reach root */
    int64_t qh = 0, qt = 0;
    d[root] = 0;
    queue[qt++] = (int32_t)root;
    while (qh < qt) {
        const int64_t v = queue[qh++];
        for (int64_t a = g->first[v]; a < g->first[v + 1]; a++) {
            const int64_t u = g->head[a], ua = g->rev[a]; /* arc ua: u -> v */
            if (u == other || d[u] != n || g->res[ua] <= 0) continue;
            if (phase2 && v == root && g->cap[ua] > 0) continue;
            d[u] = d[v] + 1;
            queue[qt++] = (int32_t)u;
        }
    }
    d[other] = n;
}

static int pr_phase(graph_t *g, int64_t s, int64_t t, int phase2, int64_t *ex, int64_t *d, int64_t *cur,
                    int32_t *fifo, uint8_t *inq, int32_t *bfsq) {
    const int64_t n = g->nn, term = phase2 ? s : t, other = phase2 ? t : s;
    int64_t qh = 0, qt = 0, work = 0;
    pr_global(g, term, other, phase2, n, d, bfsq);
    for (int64_t v = 0; v < n; v++) {
        cur[v] = g->first[v];
        inq[v] = 0;
        if (v != s && v != t && ex[v] > 0 && d[v] < n) { fifo[qt++ % n] = (int32_t)v; inq[v] = 1; }
    }
    while (qh != qt) {
        const int64_t v = fifo[qh++ % n];
        inq[v] = 0;
        while (ex[v] > 0 && d[v] < n) {
            if (cur[v] == g->first[v + 1]) {        /* relabel */
                int64_t m = 2 * n;
                for (int64_t a = g->first[v]; a < g->first[v + 1]; a++)
                    if (g->res[a] > 0 && d[g->head[a]] + 1 < m && !(phase2 && g->head[a] == s && g->cap[a] > 0))
                        m = d[g->head[a]] + 1;
                d[v] = m < n ? m : n;
                cur[v] = g->first[v];
                if (++work >= n) {                  /* periodic global relabel */
                    work = 0;
                    pr_global(g, term, other, phase2, n, d, bfsq);
                    for (int64_t u = 0; u < n; u++) cur[u] = g->first[u];
                }
                continue;
            }
            const int64_t a = cur[v], w = g->head[a];
            if (g->res[a] > 0 && d[v] == d[w] + 1 && !(phase2 && w == s && g->cap[a] > 0)) { /* push */
                const int64_t f = ex[v] < g->res[a] ? ex[v] : g->res[a];
                g->res[a] -= f;
                g->res[g->rev[a]] += f;
                ex[v] -= f;
                ex[w] += f;
                if (w != s && w != t && !inq[w] && d[w] < n) { fifo[qt++ % n] = (int32_t)w; inq[w] = 1; }
            } else {
                cur[v]++;
            }
        }
    }
    return 0;
}

static int64_t push_relabel(graph_t *g, int64_t s, int64_t t, int *err) {
    const int64_t n = g->nn;
    int64_t *ex = (int64_t *)calloc((size_t)n, sizeof(int64_t));
    int64_t *d = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *cur = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int32_t *fifo = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    int32_t *bfsq = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    uint8_t *inq = (uint8_t *)malloc((size_t)n);
    int64_t flow = 0;
    if (!ex || !d || !cur || !fifo || !bfsq || !inq) { *err = OR_E_NOMEM; goto done; }
    for (int64_t a = g->first[s]; a < g->first[s + 1]; a++) { /* saturate the source arcs */
        const int64_t f = g->res[a];
        if (f <= 0) continue;
        g->res[a] -= f;
        g->res[g->rev[a]] += f;
        ex[g->head[a]] += f;
        ex[s] -= f;
    }
    pr_phase(g, s, t, 0, ex, d, cur, fifo, inq, bfsq); /* phase 1: maximum preflow */
    pr_phase(g, s, t, 1, ex, d, cur, fifo, inq, bfsq); /* phase 2: excess back to s */
    flow = ex[t];
done:
    free(ex); free(d); free(cur); free(fifo); free(bfsq); free(inq);
    return flow;
}

static int64_t run_maxflow(graph_t *g, int64_t s, int64_t t, int algo, int *err) {
    return algo == 1 ? edmonds_karp(g, s, t, err) : algo == 2 ? push_relabel(g, s, t, err) : dinic(g, s, t, err);
}

/*
 * Column-graph oracle.
 *   in[X*Y*Z]       int32 costs c[x][y][z] (z fastest), or vertex weights if input_is_weight
 *   delta, delta_y  smoothness toward x- / y-neighbours (delta_y = -1: same as delta)
 *   algo            0 = Dinitz, 1 = Edmonds-Karp, 2 = two-phase FIFO push-relabel
 *   flow_out        |f| (int64)
 *   surface_out     int32[X*Y], max z in S per column, -1 if none (nullable)
 *   mask_out        uint8[X*Y*Z], 1 if the vertex is in the minimal source set (nullable)
 *   checks_out      invariant bits (nullable)
 *   n_arcs_out      number of explicit arcs built (nullable)
 * Returns 0, 1 (invalid dims), 3 (out of memory) or 6 (a column has no source-side vertex).
 */
int oracle_colgraph_solve_soft(const int32_t *in, int X, int Y, int Z, int delta, int delta_y, const int32_t *penalty,
                               int npenalty, int input_is_weight, int algo, int64_t *flow_out, int32_t *surface_out,
                               uint8_t *mask_out, int32_t *checks_out, int64_t *n_arcs_out);

int oracle_colgraph_solve(const int32_t *in, int X, int Y, int Z, int delta, int delta_y, int input_is_weight,
                          int algo, int64_t *flow_out, int32_t *surface_out, uint8_t *mask_out, int32_t *checks_out,
                          int64_t *n_arcs_out) {
    return oracle_colgraph_solve_soft(in, X, Y, Z, delta, delta_y, NULL, 0, input_is_weight, algo, flow_out,
                                      surface_out, mask_out, checks_out, n_arcs_out);
}

int oracle_colgraph_solve_general(const int32_t *in, int X, int Y, int Z, const int32_t *dl4, const int32_t *band,
                                  const int32_t *penalty, int npenalty, int input_is_weight, int algo,
                                  int64_t *flow_out, int32_t *surface_out, uint8_t *mask_out, int32_t *checks_out,
                                  int64_t *n_arcs_out);

int oracle_colgraph_solve_soft(const int32_t *in, int X, int Y, int Z, int delta, int delta_y, const int32_t *penalty,
                               int npenalty, int input_is_weight, int algo, int64_t *flow_out, int32_t *surface_out,
                               uint8_t *mask_out, int32_t *checks_out, int64_t *n_arcs_out) {
    if (delta_y == -1) delta_y = delta; /* isotropic */
    const int32_t dl4[4] = {delta, delta, delta_y, delta_y};
    return oracle_colgraph_solve_general(in, X, Y, Z, dl4, NULL, penalty, npenalty, input_is_weight, algo, flow_out,
                                         surface_out, mask_out, checks_out, n_arcs_out);
}

/*
 * General entry (NEXT-3): dl4[4] = Delta toward +x, -x, +y, -y (see colgraph_arcs); band nullable
 * int32[2*X*Y] = (lo, hi) per column, 0 <= lo < hi <= Z, costs only (see column_weights_band).
 */
int oracle_colgraph_solve_general(const int32_t *in, int X, int Y, int Z, const int32_t *dl4, const int32_t *band,
                                  const int32_t *penalty, int npenalty, int input_is_weight, int algo,
                                  int64_t *flow_out, int32_t *surface_out, uint8_t *mask_out, int32_t *checks_out,
                                  int64_t *n_arcs_out) {
    if (!in || !dl4 || X < 1 || Y < 1 || Z < 1) return OR_E_INVAL;
    int dmax = 0;
    for (int d = 0; d < 4; d++) {
        if (dl4[d] < 0) return OR_E_INVAL;
        if (dl4[d] > dmax) dmax = dl4[d];
    }
    if (band) {
        if (input_is_weight) return OR_E_INVAL;
        for (int64_t col = 0; col < (int64_t)X * Y; col++)
            if (band[2 * col] < 0 || band[2 * col] >= band[2 * col + 1] || band[2 * col + 1] > Z) return OR_E_INVAL;
    }
    if (penalty && npenalty < dmax) return OR_E_INVAL;
    g_penalty = penalty;
    g_npenalty = npenalty;
    if (penalty) /* convex, non-negative capacities */
        for (int k = 0; k < npenalty; k++)
            if (soft_cap(k) < 0) return OR_E_INVAL;
    if ((int64_t)X * Y * Z + 2 > INT32_MAX) return OR_E_INVAL;
    const int64_t n = (int64_t)X * Y * Z, s = n, t = n + 1;
    graph_t g;
    int err = OR_OK;
    int64_t *wbuf = (int64_t *)malloc((size_t)Z * sizeof(int64_t));
    uint8_t *mark = (uint8_t *)malloc((size_t)n + 2);
    if (!wbuf || !mark || g_alloc(&g, n + 2)) { free(wbuf); free(mark); return OR_E_NOMEM; }
    colgraph_arcs(&g, 0, in, X, Y, Z, dl4, band, input_is_weight, wbuf);
    if (g_finish_count(&g)) { g_free(&g); free(wbuf); free(mark); return OR_E_NOMEM; }
    colgraph_arcs(&g, 1, in, X, Y, Z, dl4, band, input_is_weight, wbuf);
    if (n_arcs_out) *n_arcs_out = g.m / 2;
    int64_t flow = run_maxflow(&g, s, t, algo, &err);
    if (err) { g_free(&g); free(wbuf); free(mark); return err; }
    if (source_set(&g, s, mark)) { g_free(&g); free(wbuf); free(mark); return OR_E_NOMEM; }
    if (checks_out) *checks_out = check_invariants(&g, s, t, mark, flow);
    *flow_out = flow;
    int status = OR_OK;
    for (int64_t col = 0; col < (int64_t)X * Y; col++) {
        int32_t top = -1;
        for (int64_t z = 0; z < Z; z++)
            if (mark[col * Z + z]) top = (int32_t)z;
        if (top < 0) status = OR_E_EMPTY_COLUMN;
        if (surface_out) surface_out[col] = top;
    }
    if (mask_out) memcpy(mask_out, mark, (size_t)n);
    g_free(&g); free(wbuf); free(mark);
    return status;
}

/*
 * Generic max-flow on an explicit arc list (for pinning the max-flow core
 * against brute-force minimum cuts on small general graphs).
 *   tails/heads/caps [m]; nodes 0..nn-1; s, t.
 *   source_side_out uint8[nn] (nullable): minimal source set.
 */
int oracle_graph_maxflow(int nn, int m, const int32_t *tails, const int32_t *heads, const int64_t *caps,
                         int s, int t, int algo, int64_t *flow_out, uint8_t *source_side_out,
                         int32_t *checks_out) {
    if (nn < 2 || m < 0 || s < 0 || t < 0 || s >= nn || t >= nn || s == t) return OR_E_INVAL;
    graph_t g;
    int err = OR_OK;
    if (g_alloc(&g, nn)) return OR_E_NOMEM;
    for (int i = 0; i < m; i++) {
        if (tails[i] < 0 || tails[i] >= nn || heads[i] < 0 || heads[i] >= nn || caps[i] < 0) {
            g_free(&g);
            return OR_E_INVAL;
        }
        add_arc(&g, 0, tails[i], heads[i], caps[i]);
    }
    if (g_finish_count(&g)) { g_free(&g); return OR_E_NOMEM; }
    for (int i = 0; i < m; i++) add_arc(&g, 1, tails[i], heads[i], caps[i]);
    int64_t flow = run_maxflow(&g, s, t, algo, &err);
    uint8_t *mark = (uint8_t *)malloc((size_t)nn);
    if (err || !mark || source_set(&g, s, mark)) { g_free(&g); free(mark); return err ? err : OR_E_NOMEM; }
    if (checks_out) *checks_out = check_invariants(&g, s, t, mark, flow);
    *flow_out = flow;
    if (source_side_out) memcpy(source_side_out, mark, (size_t)nn);
    g_free(&g); free(mark);
    return OR_OK;
}

/*
 * Invariant checker on a GIVEN residual state (test entry point; pins check_invariants itself).
 * The explicit graph is built from the arc list exactly as oracle_graph_maxflow builds it, then
 * the residuals are overwritten with the caller's: res_fwd[i] on arc i (tail -> head, original
 * capacity caps[i]) and res_rev[i] on its paired reverse slot (capacity 0).  The claimed flow value
 * and source-side marks are checked as they are, so a corrupted state must clear the bit of the
 * invariant it breaks: capacity (Eq. 2), antisymmetry (Eq. 3), conservation
 * (Eq. 4), value (Eq. 5), t not in S, cut == flow (Theorem 1; Eq. 6).
 */
int oracle_graph_check(int nn, int m, const int32_t *tails, const int32_t *heads, const int64_t *caps,
                       const int64_t *res_fwd, const int64_t *res_rev, int s, int t, const uint8_t *source_side,
                       int64_t flow, int32_t *checks_out) {
    if (nn < 2 || m < 0 || s < 0 || t < 0 || s >= nn || t >= nn || s == t || !checks_out) return OR_E_INVAL;
    graph_t g;
    if (g_alloc(&g, nn)) return OR_E_NOMEM;
    for (int i = 0; i < m; i++) {
        if (tails[i] < 0 || tails[i] >= nn || heads[i] < 0 || heads[i] >= nn || caps[i] < 0) {
            g_free(&g);
            return OR_E_INVAL;
        }
        add_arc(&g, 0, tails[i], heads[i], caps[i]);
    }
    if (g_finish_count(&g)) { g_free(&g); return OR_E_NOMEM; }
    for (int i = 0; i < m; i++) {
        const int64_t a = g.fill[tails[i]]; /* the slot add_arc is about to use for arc i */
        add_arc(&g, 1, tails[i], heads[i], caps[i]);
        g.res[a] = res_fwd[i];
        g.res[g.rev[a]] = res_rev[i];
    }
    *checks_out = check_invariants(&g, s, t, source_side, flow);
    g_free(&g);
    return OR_OK;
}
