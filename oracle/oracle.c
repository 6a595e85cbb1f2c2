/*
 * oracle.c — plain, slow, single-threaded CPU oracle for MPDP
 * (arXiv 2202.13511, "Efficient Massively Parallel Join Optimization for
 * Large Queries").  TEST INFRASTRUCTURE ONLY — see oracle.h.
 *
 * What it computes (DESIGN.md §"Oracle"): for a connected query graph,
 *
 *   best(S) = argmin over unordered CCP splits {A, B} of S of
 *             key = ( fl(fl(cost(A) + cost(B)) + card(S)), min(A, B) )
 *   cost(S) = key.first, left(S) = key.second, cost({v}) = leaf_cost[v]
 *
 * i.e. the optimum of Alg. generic_dpsub / Alg.
 * mpdp_generalization (same optimum by the Theorem at)
 * under the C_out cost with DESIGN.md readings R1-R8.
 *
 * Parity pins (tests/test_oracle.py, all `-m "not gpu"`):
 *   primitives ........ paper worked examples P:195
 *                       (tests/golden/ fixtures), brute force on tiny graphs
 *   counters .......... closed forms (chain/star/clique/cycle), "2805",
 *                       "12024x", Lemma 8, Lemma 5
 *   optimisers ........ O3 brute force over all trees (n <= 7, exact cost),
 *                       O0 == O1 == O2 on random graphs (n <= 14), tree counts
 *   oracle_card ....... closed-form products on power-of-two inputs
 *   oracle_unrank_colex SPEC examples S:37-39 + exhaustive bijection
 * The chosen plan tree under the tie-break R7 has no paper value to pin
 * ("parity unpinned" beyond O0==O1==O2 agreement and cost recomputation);
 * see DESIGN.md.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* Internal graph: adjacency bitmasks, full selectivity matrix.              */
/* ------------------------------------------------------------------------ */
typedef struct {
    int n;
    uint64_t adj[64];
    double card[64];
    double leaf[64];
    double sel[64][64];       /* sel[u][v] = sel[v][u]; 0 = no edge */
} G;

static uint64_t bit(int v) { return (uint64_t)1 << v; }
static int lowest(uint64_t S) { return __builtin_ctzll(S); }
static int popc(uint64_t S) { return __builtin_popcountll(S); }

static int load_graph(const oracle_graph* in, G* g) {
    if (!in || in->n == 0 || in->n > 64 || !in->card) return ORACLE_ERR_ARG;
    if (in->n_edges && (!in->edges || !in->sel)) return ORACLE_ERR_ARG;
    memset(g, 0, sizeof(*g));
    g->n = (int)in->n;
    for (int v = 0; v < g->n; v++) {
        double c = in->card[v];
        if (!(c >= 0.0) || !isfinite(c)) return ORACLE_ERR_ARG;   /* reading R18: 0 allowed */
        g->card[v] = c;
        g->leaf[v] = in->leaf_cost ? in->leaf_cost[v] : 0.0;
        if (!isfinite(g->leaf[v]) || g->leaf[v] < 0.0) return ORACLE_ERR_ARG;
    }
    for (uint32_t e = 0; e < in->n_edges; e++) {
        uint32_t u = in->edges[2 * e], v = in->edges[2 * e + 1];
        double s = in->sel[e];
        if (u >= v || v >= in->n) return ORACLE_ERR_ARG;
        if (g->adj[u] & bit((int)v)) return ORACLE_ERR_ARG;          /* duplicate */
        if (!(s > 0.0) || !(s <= 1.0)) return ORACLE_ERR_ARG;
        g->adj[u] |= bit((int)v);
        g->adj[v] |= bit((int)u);
        g->sel[u][v] = g->sel[v][u] = s;
    }
    return ORACLE_OK;
}

/* Neighbourhood N(S) = { v not in S | exists u in S, (u, v) in E }. */
static uint64_t neigh(const G* g, uint64_t S) {
    uint64_t N = 0;
    for (uint64_t T = S; T; T &= T - 1) N |= g->adj[lowest(T)];   /* v in S */
    return N & ~S;
}

/* Alg. grow, literally: one vertex x = first(N) per iteration,
 * N <- (N u (Neighbours(x) n Restriction)) \ V. */
static uint64_t grow(const G* g, uint64_t source, uint64_t restriction) {
    uint64_t V = 0, N = source;
    while (N) {
        int x = lowest(N);
        V |= bit(x);
        N = (N | (g->adj[x] & restriction)) & ~V;
    }
    return V;
}

/* Alg. connected: false for the empty set, else
 * grow(min(S), S) == S (seed = lowest vertex, reading R9). */
static int connected(const G* g, uint64_t S) {
    if (S == 0) return 0;
    return grow(g, bit(lowest(S)), S) == S;
}

/* The four CCP-Pair conditions of §2.1. */
static int is_ccp(const G* g, uint64_t S1, uint64_t S2) {
    if (S1 == 0 || S2 == 0) return 0;                 /* 1: non-empty   */
    if (!connected(g, S1) || !connected(g, S2)) return 0; /* 2: connected */
    if (S1 & S2) return 0;                            /* 3: disjoint    */
    for (uint64_t T = S1; T; T &= T - 1)              /* 4: an edge     */
        if (g->adj[lowest(T)] & S2) return 1;
    return 0;
}

/* card(S): product of base cardinalities and of the selectivities of the
 * edges induced by S, in the canonical order of reading R5:
 *   x = 1; for v in S ascending { x *= card[v]; for u in S n adj(v), u < v
 *   ascending: x *= sel(u, v) }. */
static double card_of(const G* g, uint64_t S) {
    double x = 1.0;
    for (uint64_t T = S; T; T &= T - 1) {             /* v in S ascending */
        int v = lowest(T);
        x = x * g->card[v];
        for (uint64_t U = S & g->adj[v] & (bit(v) - 1); U; U &= U - 1)  /* u < v ascending */
            x = x * g->sel[lowest(U)][v];
    }
    return x;
}

/* Blocks (biconnected components) of G[S] by the DFS of Hopcroft and
 * Tarjan (cited at P:587), textbook recursive form with a vertex stack.
 * A block is emitted when low[u] >= disc[v] for the tree edge (v, u). */
typedef struct {
    const G* g;
    uint64_t S;
    int disc[64], low[64], stack[64], sp, time;
    uint64_t* out;
    int nout, max_out;
} Bcc;

static void bcc_dfs(Bcc* b, int v, int parent) {
    b->disc[v] = b->low[v] = ++b->time;
    b->stack[b->sp++] = v;
    for (uint64_t U = b->S & b->g->adj[v]; U; U &= U - 1) {   /* u ascending */
        int u = lowest(U);
        if (!b->disc[u]) {
            bcc_dfs(b, u, v);
            if (b->low[u] < b->low[v]) b->low[v] = b->low[u];
            if (b->low[u] >= b->disc[v]) {        /* v separates u's subtree */
                uint64_t B = bit(v);
                int w;
                do {
                    w = b->stack[--b->sp];
                    B |= bit(w);
                } while (w != u);
                if (b->nout < b->max_out) b->out[b->nout] = B;
                b->nout++;
            }
        } else if (u != parent) {
            if (b->disc[u] < b->low[v]) b->low[v] = b->disc[u];
        }
    }
}

static int blocks_of(const G* g, uint64_t S, uint64_t* out, int max_out) {
    Bcc b;
    memset(&b, 0, sizeof(b));
    b.g = g;
    b.S = S;
    b.out = out;
    b.max_out = max_out;
    if (popc(S) < 2) return 0;              /* a single vertex has no edge */
    bcc_dfs(&b, lowest(S), -1);
    return b.nout;
}

/* Join pairs MPDP evaluates for one connected set (reading R3): per block B,
 * the subsets lb of B that contain B's lowest vertex and differ from B, i.e.
 * 2^(|B|-1) - 1 unordered block splits (P:547 enumerates all lb of the block;
 * the mirror (rb, lb) is the same unordered split). */
static uint64_t mpdp_pairs(const G* g, uint64_t S) {
    uint64_t blocks[64];
    int nb = blocks_of(g, S, blocks, 64);
    uint64_t total = 0;
    for (int i = 0; i < nb; i++) total += (((uint64_t)1) << (popc(blocks[i]) - 1)) - 1;
    return total;
}

/* ------------------------------------------------------------------------ */
/* Public primitives                                                         */
/* ------------------------------------------------------------------------ */
uint64_t oracle_neighbours(const oracle_graph* in, uint64_t S) {
    G g;
    if (load_graph(in, &g)) return 0;
    return neigh(&g, S);
}
uint64_t oracle_grow(const oracle_graph* in, uint64_t source, uint64_t restriction) {
    G g;
    if (load_graph(in, &g)) return 0;
    return grow(&g, source, restriction);
}
int oracle_connected(const oracle_graph* in, uint64_t S) {
    G g;
    if (load_graph(in, &g)) return -1;
    return connected(&g, S);
}
int oracle_is_ccp(const oracle_graph* in, uint64_t S1, uint64_t S2) {
    G g;
    if (load_graph(in, &g)) return -1;
    return is_ccp(&g, S1, S2);
}
double oracle_card(const oracle_graph* in, uint64_t S) {
    G g;
    if (load_graph(in, &g)) return NAN;
    return card_of(&g, S);
}
int oracle_blocks(const oracle_graph* in, uint64_t S, uint64_t* blocks, int max_blocks) {
    G g;
    if (load_graph(in, &g)) return -1;
    return blocks_of(&g, S, blocks, max_blocks);
}
uint64_t oracle_mpdp_pairs(const oracle_graph* in, uint64_t S) {
    G g;
    if (load_graph(in, &g)) return 0;
    return mpdp_pairs(&g, S);
}

/* Binomial coefficient by the multiplicative formula (exact for n <= 64). */
static uint64_t binom(uint32_t n, uint32_t k) {
    if (k > n) return 0;
    if (k > n - k) k = n - k;
    uint64_t r = 1;
    for (uint32_t i = 1; i <= k; i++) r = r / i * (n - k + i) + r % i * (n - k + i) / i;
    return r;
}

/* Colex combinadic (reading R10): the r-th k-subset has
 * elements c_k > ... > c_1 with r = sum_i C(c_i, i); greedy from the top. */
uint64_t oracle_unrank_colex(uint32_t n, uint32_t k, uint64_t r) {
    uint64_t S = 0;
    int c = (int)n - 1;
    for (uint32_t i = k; i >= 1; i--) {
        while (c >= 0 && binom((uint32_t)c, i) > r) c--;
        S |= bit(c);
        r -= binom((uint32_t)c, i);
        c--;
    }
    return S;
}

/* ------------------------------------------------------------------------ */
/* Memo shared by the optimisers: direct arrays indexed by the subset mask.  */
/* ------------------------------------------------------------------------ */
typedef struct {
    const G* g;
    uint64_t size;
    double* cost;        /* +inf = no plan yet                          */
    uint64_t* left;      /* min(S_left, S_right) of the best split      */
    double* card;        /* card cache, NaN = not computed              */
    uint8_t* used;       /* DPccp order check: set consumed as a child  */
    uint64_t lvl_ccp[65];
    int order_violation;
} Memo;

static int memo_init(Memo* m, const G* g) {
    memset(m, 0, sizeof(*m));
    m->g = g;
    m->size = (uint64_t)1 << g->n;
    m->cost = (double*)malloc(m->size * sizeof(double));
    m->left = (uint64_t*)malloc(m->size * sizeof(uint64_t));
    m->card = (double*)malloc(m->size * sizeof(double));
    m->used = (uint8_t*)calloc(m->size, 1);
    if (!m->cost || !m->left || !m->card || !m->used) return ORACLE_ERR_OOM;
    for (uint64_t S = 0; S < m->size; S++) {
        m->cost[S] = INFINITY;
        m->left[S] = UINT64_MAX;
        m->card[S] = NAN;
    }
    for (int v = 0; v < g->n; v++) m->cost[bit(v)] = g->leaf[v]; /* Alg.1 line 2 */
    return ORACLE_OK;
}

static void memo_free(Memo* m) {
    free(m->cost);
    free(m->left);
    free(m->card);
    free(m->used);
}

static double memo_card(Memo* m, uint64_t S) {
    if (isnan(m->card[S])) m->card[S] = card_of(m->g, S);
    return m->card[S];
}

/* CreatePlan + "if CurrPlan < BestPlan(S)" with C_out (P:977,
 * S:197): cost = (cost(A) + cost(B)) + card(S), compared lexicographically
 * with left = min(A, B) on exact ties (reading R7). */
static void consider(Memo* m, uint64_t A, uint64_t B) {
    uint64_t S = A | B;
    double c = (m->cost[A] + m->cost[B]) + memo_card(m, S);
    uint64_t l = A < B ? A : B;
    if (m->used[S]) m->order_violation = 1;   /* S already consumed as a child */
    m->used[A] = m->used[B] = 1;
    if (c < m->cost[S] || (c == m->cost[S] && l < m->left[S])) {
        m->cost[S] = c;
        m->left[S] = l;
    }
    m->lvl_ccp[popc(S)]++;
}

static int graph_connected(const G* g) {
    uint64_t all = (g->n == 64) ? UINT64_MAX : (bit(g->n) - 1);
    return connected(g, all);
}

/* Plan extraction: node(S) = join(node(left(S)), node(S\left(S))),
 * post-order, root last. */
static int32_t extract(Memo* m, uint64_t S, oracle_result* out) {
    int32_t idx;
    if (popc(S) == 1) {
        idx = (int32_t)out->n_nodes++;
        if ((uint32_t)idx >= out->capacity) return -1;
        oracle_node* nd = &out->nodes[idx];
        nd->left = nd->right = -1;
        nd->relation = lowest(S);
        nd->set = S;
        nd->card = m->g->card[lowest(S)];
        nd->cost = m->cost[S];
        return idx;
    }
    uint64_t L = m->left[S];
    int32_t a = extract(m, L, out);
    if (a < 0) return -1;
    int32_t b = extract(m, S & ~L, out);
    if (b < 0) return -1;
    idx = (int32_t)out->n_nodes++;
    if ((uint32_t)idx >= out->capacity) return -1;
    oracle_node* nd = &out->nodes[idx];
    nd->left = a;
    nd->right = b;
    nd->relation = -1;
    nd->set = S;
    nd->card = memo_card(m, S);
    nd->cost = m->cost[S];
    return idx;
}

static int finish(Memo* m, oracle_result* out, const uint64_t* lvl_csg, const uint64_t* lvl_pairs) {
    const G* g = m->g;
    uint64_t all = (g->n == 64) ? UINT64_MAX : (bit(g->n) - 1);
    out->n_nodes = 0;
    if (out->nodes && out->capacity >= (uint32_t)(2 * g->n - 1)) {
        if (extract(m, all, out) < 0) return ORACLE_ERR_ARG;
    }
    out->cost = m->cost[all];
    out->csg_count = out->ccp_pairs = out->pairs_evaluated = 0;
    for (int k = 0; k <= g->n; k++) {
        out->csg_count += lvl_csg[k];
        out->ccp_pairs += m->lvl_ccp[k];
        out->pairs_evaluated += lvl_pairs[k];
        if (out->level_csg) out->level_csg[k] = lvl_csg[k];
        if (out->level_ccp) out->level_ccp[k] = m->lvl_ccp[k];
        if (out->level_pairs) out->level_pairs[k] = lvl_pairs[k];
    }
    return ORACLE_OK;
}

/* Next k-subset in increasing numeric (= colex) order (Gosper's hack, cited
 * by the paper's improved unrank P:922-926). */
static uint64_t next_same_popcount(uint64_t v) {
    uint64_t t = v | (v - 1);
    return (t + 1) | (((~t & -~t) - 1) >> (__builtin_ctzll(v) + 1));
}

/* ------------------------------------------------------------------------ */
/* O0 — the plain definition: Alg. generic_dpsub with the       */
/* unordered split (left side holds min(S), reading R2), size by size.       */
/* ------------------------------------------------------------------------ */
int oracle_optimize_definition(const oracle_graph* in, oracle_result* out) {
    G g;
    int st = load_graph(in, &g);
    if (st) return st;
    if (g.n > 20) return ORACLE_ERR_CAPACITY;
    if (!graph_connected(&g)) return ORACLE_ERR_DISCONNECTED;
    Memo m;
    if (memo_init(&m, &g)) { memo_free(&m); return ORACLE_ERR_OOM; }
    uint64_t lvl_csg[65] = {0}, lvl_pairs[65] = {0};
    lvl_csg[1] = (uint64_t)g.n;
    for (int i = 2; i <= g.n; i++) {                       /* line 3 */
        uint64_t last = ((bit(i) - 1) << (g.n - i));
        for (uint64_t S = bit(i) - 1;; S = next_same_popcount(S)) {
            if (connected(&g, S)) {                        /* line 4 */
                lvl_csg[i]++;
                lvl_pairs[i] += mpdp_pairs(&g, S);
                uint64_t lo = bit(lowest(S)), R = S & ~lo;
                /* every subset A of S holding min(S), A != S: the unordered
                 * Join-Pairs of line 6 */
                uint64_t sub = 0;
                do {
                    uint64_t A = lo | sub, B = S & ~A;
                    if (B && is_ccp(&g, A, B)) consider(&m, A, B); /* CCP block */
                    sub = (sub - R) & R;
                } while (sub != 0);
            }
            if (S == last) break;
        }
    }
    m.order_violation = 0;   /* size order is valid by construction */
    st = finish(&m, out, lvl_csg, lvl_pairs);
    memo_free(&m);
    return st;
}

/* ------------------------------------------------------------------------ */
/* O1 — DPccp (Moerkotte & Neumann, cited as [dpccp] at P:189/P:993):       */
/* EnumerateCsg / EnumerateCsgRec / EmitCsg / EnumerateCmpRec.               */
/* ------------------------------------------------------------------------ */
typedef struct {
    Memo* m;
    uint64_t lvl_csg[65], lvl_pairs[65];
    int with_pairs;
} Ccp;

static uint64_t Bset(int i) { return (i >= 63) ? UINT64_MAX : (bit(i + 1) - 1); } /* {v_j : j <= i} */

static void enum_cmp_rec(Ccp* c, uint64_t S1, uint64_t S2, uint64_t X) {
    uint64_t N = neigh(c->m->g, S2) & ~X;
    if (!N) return;
    for (uint64_t s = (0 - N) & N; s; s = (s - N) & N) consider(c->m, S1, S2 | s);
    for (uint64_t s = (0 - N) & N; s; s = (s - N) & N) enum_cmp_rec(c, S1, S2 | s, X | N);
}

static void emit_csg(Ccp* c, uint64_t S1) {
    const G* g = c->m->g;
    int k = popc(S1);
    c->lvl_csg[k]++;
    if (c->with_pairs && k >= 2) c->lvl_pairs[k] += mpdp_pairs(g, S1);
    uint64_t X = S1 | Bset(lowest(S1));
    uint64_t N = neigh(g, S1) & ~X;
    for (int i = g->n - 1; i >= 0; i--) {           /* v_i in N, descending */
        if (!(N & bit(i))) continue;
        uint64_t S2 = bit(i);
        consider(c->m, S1, S2);
        enum_cmp_rec(c, S1, S2, X | (Bset(i) & N));
    }
}

static void enum_csg_rec(Ccp* c, uint64_t S, uint64_t X) {
    uint64_t N = neigh(c->m->g, S) & ~X;
    if (!N) return;
    for (uint64_t s = (0 - N) & N; s; s = (s - N) & N) emit_csg(c, S | s);
    for (uint64_t s = (0 - N) & N; s; s = (s - N) & N) enum_csg_rec(c, S | s, X | N);
}

int oracle_optimize_dpccp(const oracle_graph* in, oracle_result* out) {
    G g;
    int st = load_graph(in, &g);
    if (st) return st;
    if (g.n > 28) return ORACLE_ERR_CAPACITY;
    if (!graph_connected(&g)) return ORACLE_ERR_DISCONNECTED;
    Memo m;
    if (memo_init(&m, &g)) { memo_free(&m); return ORACLE_ERR_OOM; }
    Ccp c;
    memset(&c, 0, sizeof(c));
    c.m = &m;
    c.with_pairs = 1;
    for (int i = g.n - 1; i >= 0; i--) {              /* EnumerateCsg */
        emit_csg(&c, bit(i));
        enum_csg_rec(&c, bit(i), Bset(i));
    }
    if (m.order_violation) { memo_free(&m); return 8; }
    st = finish(&m, out, c.lvl_csg, c.lvl_pairs);
    memo_free(&m);
    return st;
}

/* ------------------------------------------------------------------------ */
/* O2 — DPsize over connected sets: level s joins   */
/* every ordered pair of memo entries of sizes (l, s-l); counts every check. */
/* ------------------------------------------------------------------------ */
int oracle_optimize_dpsize(const oracle_graph* in, oracle_result* out) {
    G g;
    int st = load_graph(in, &g);
    if (st) return st;
    if (g.n > 16) return ORACLE_ERR_CAPACITY;
    if (!graph_connected(&g)) return ORACLE_ERR_DISCONNECTED;
    Memo m;
    if (memo_init(&m, &g)) { memo_free(&m); return ORACLE_ERR_OOM; }
    uint64_t* lists[65] = {0};
    uint64_t cnt[65] = {0};
    uint64_t lvl_csg[65] = {0}, lvl_pairs[65] = {0}, checks = 0;
    lists[1] = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)g.n);
    for (int v = 0; v < g.n; v++) lists[1][cnt[1]++] = bit(v);
    lvl_csg[1] = (uint64_t)g.n;
    for (int s = 2; s <= g.n; s++) {
        uint64_t before[65];
        memcpy(before, m.lvl_ccp, sizeof(before));
        for (int l = 1; l < s; l++)
            for (uint64_t a = 0; a < cnt[l]; a++)
                for (uint64_t b = 0; b < cnt[s - l]; b++) {
                    uint64_t A = lists[l][a], B = lists[s - l][b];
                    checks++;
                    if (A & B) continue;
                    if (!(neigh(&g, A) & B)) continue;
                    consider(&m, A, B);
                }
        /* each unordered pair was seen twice (as (A,B) and (B,A)) */
        m.lvl_ccp[s] = before[s] + (m.lvl_ccp[s] - before[s]) / 2;
        lists[s] = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)binom((uint32_t)g.n, (uint32_t)s));
        uint64_t last = ((bit(s) - 1) << (g.n - s));
        for (uint64_t S = bit(s) - 1;; S = next_same_popcount(S)) {
            if (isfinite(m.cost[S])) {
                lists[s][cnt[s]++] = S;
                lvl_csg[s]++;
                lvl_pairs[s] += mpdp_pairs(&g, S);
            }
            if (S == last) break;
        }
    }
    m.order_violation = 0;
    st = finish(&m, out, lvl_csg, lvl_pairs);
    out->dpsize_checks = checks;
    for (int s = 0; s <= 64; s++) free(lists[s]);
    memo_free(&m);
    return st;
}

/* ------------------------------------------------------------------------ */
/* O3 — brute force: the cost of EVERY cross-product-free bushy tree with    */
/* ordered children (built from CCP-Pairs), listed explicitly.    */
/* ------------------------------------------------------------------------ */
int oracle_bruteforce(const oracle_graph* in, double* min_cost, uint64_t* n_trees) {
    G g;
    int st = load_graph(in, &g);
    if (st) return st;
    if (g.n > 7) return ORACLE_ERR_CAPACITY;
    if (!graph_connected(&g)) return ORACLE_ERR_DISCONNECTED;
    uint64_t size = (uint64_t)1 << g.n;
    double** costs = (double**)calloc(size, sizeof(double*));
    uint64_t* count = (uint64_t*)calloc(size, sizeof(uint64_t));
    for (int v = 0; v < g.n; v++) {
        costs[bit(v)] = (double*)malloc(sizeof(double));
        costs[bit(v)][0] = g.leaf[v];
        count[bit(v)] = 1;
    }
    for (uint64_t S = 1; S < size; S++) {            /* subsets before supersets */
        if (popc(S) < 2 || !connected(&g, S)) continue;
        uint64_t total = 0;
        for (uint64_t A = (S - 1) & S; A; A = (A - 1) & S)
            if (is_ccp(&g, A, S & ~A)) total += count[A] * count[S & ~A];
        costs[S] = (double*)malloc(sizeof(double) * (total ? total : 1));
        double cs = card_of(&g, S);
        uint64_t t = 0;
        for (uint64_t A = (S - 1) & S; A; A = (A - 1) & S) {
            uint64_t B = S & ~A;
            if (!is_ccp(&g, A, B)) continue;
            for (uint64_t i = 0; i < count[A]; i++)
                for (uint64_t j = 0; j < count[B]; j++) costs[S][t++] = (costs[A][i] + costs[B][j]) + cs;
        }
        count[S] = total;
    }
    uint64_t all = size - 1;
    double best = INFINITY;
    for (uint64_t i = 0; i < count[all]; i++)
        if (costs[all][i] < best) best = costs[all][i];
    *min_cost = best;
    *n_trees = count[all];
    for (uint64_t S = 0; S < size; S++) free(costs[S]);
    free(costs);
    free(count);
    return ORACLE_OK;
}

/* ------------------------------------------------------------------------ */
/* O4 — counters by definition: scan all 2^n subsets with connected().      */
/* ------------------------------------------------------------------------ */
int oracle_counters(const oracle_graph* in, uint64_t* level_csg, uint64_t* level_pairs) {
    G g;
    int st = load_graph(in, &g);
    if (st) return st;
    if (g.n > 28) return ORACLE_ERR_CAPACITY;
    for (int k = 0; k <= g.n; k++) level_csg[k] = level_pairs[k] = 0;
    uint64_t size = (uint64_t)1 << g.n;
    for (uint64_t S = 1; S < size; S++) {
        if (!connected(&g, S)) continue;
        level_csg[popc(S)]++;
        if (popc(S) >= 2) level_pairs[popc(S)] += mpdp_pairs(&g, S);
    }
    return ORACLE_OK;
}
