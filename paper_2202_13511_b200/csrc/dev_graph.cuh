// dev_graph.cuh — the query graph as the level kernels see it (shared memory)
// and the per-set graph primitives: canonical card(S), grow, connectivity,
// blocks (biconnected components) and MPDP's join-pair enumeration.
#pragma once
#include "dev_common.cuh"

namespace mpdp {

template <typename M> struct MaxN;
template <> struct MaxN<uint32_t> { static constexpr int value = 32; };
template <> struct MaxN<uint64_t> { static constexpr int value = kMaxN; };

// Query as staged in global memory (written by the host once per query).
template <typename M> struct QueryDev {
    static constexpr int N = MaxN<M>::value;
    int n, cls, max_depth, has_leaf_costs;
    unsigned long long epoch;   // look-back epoch base of this query (query counter << 6)
    unsigned int gen;           // HASH memo tag of this query
    int dpsub;                  // MPDP_FLAG_DPSUB_ENUM ablation: every set is one CCP-checked block
    M adj[N];            // adjacency bitmaps ("adjacency lists ... as bitmap sets")
    M desc[N];           // CLS_TREE: vertices of the subtree rooted at v (root = 0)
    M depth_mask[N];     // CLS_TREE: vertices at depth d
    double card[N];      // base cardinalities
    double leaf[N];      // leaf costs (0 for base relations, subplan cost for composites)
    double sel[N * N];   // sel[u * n + v] for edges, 0 otherwise
    unsigned long long binom[(N + 1) * (N + 1)];   // C(i, j) at i * (N + 1) + j
};

// Neighbourhood of a vertex set by byte lookups (32-bit masks): nb[c][b] = OR
// of adj[8c + i] over the bits i of b, so N(F) = OR_c nb[c][byte_c(F)] -- four
// shared-memory loads per BFS frontier step instead of a data-dependent loop
// over the frontier's vertices (the CCP connectivity checks of general graphs
// were 43% of k_dp_fused<GENERAL>'s instructions on random-20).  Built only by
// the general-graph kernels (SQ::nbtab); 64-bit masks keep the loop.
template <typename M> struct NbTab {};
template <> struct NbTab<uint32_t> {
    uint32_t t[4][256];
};

// The part every kernel keeps in shared memory (sel compacted to n x n).
template <typename M> struct SQ {
    static constexpr int N = MaxN<M>::value;
    int n, cls, max_depth, pad;            // pad = has_leaf_costs (any leaf cost != 0)
    int dpsub, nbtab;                      // DPSUB-enumeration ablation (QueryDev::dpsub); nb is built
    // general graphs on the bitmask-indexed memo (MEMO_MASK): the cost array,
    // pre-filled with kMemoAbsent by the host, so that the connectivity of any
    // proper subset of the set under evaluation is one probe (reading R20);
    // null = connectivity by BFS
    const double* mc;
    NbTab<M> nb;
    M adj[N];
    M desc[N];
    M depth_mask[N];
    double card[N];
    double leaf[N];
    double sel[N * N];
};

template <typename M>
__device__ __forceinline__ void load_query(SQ<M>& s, const QueryDev<M>* q) {
    const int n = q->n;
    if (threadIdx.x == 0) {
        s.n = n;
        s.cls = q->cls;
        s.max_depth = q->max_depth;
        s.pad = q->has_leaf_costs;
        s.dpsub = q->dpsub;
        s.nbtab = 0;
        s.mc = nullptr;
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        s.adj[i] = q->adj[i];
        s.desc[i] = q->desc[i];
        s.depth_mask[i] = q->depth_mask[i];
        s.card[i] = q->card[i];
        s.leaf[i] = q->leaf[i];
    }
    for (int i = threadIdx.x; i < n * n; i += blockDim.x) s.sel[i] = q->sel[i];
}

// card(S) in the canonical order of reading R5 (no FMA: only multiplies,
// and __dmul_rn pins round-to-nearest):
//   x = 1; for v in S ascending { x *= card[v]; for u in S n adj(v), u < v ascending: x *= sel(u,v) }
template <typename M>
__device__ __forceinline__ double card_of(const SQ<M>& q, M S) {
    double x = 1.0;
    for (M T = S; T; T &= T - 1) {
        const int v = ctz(T);
        x = __dmul_rn(x, q.card[v]);
        for (M U = S & q.adj[v] & (bitm<M>(v) - 1); U; U &= U - 1)
            x = __dmul_rn(x, q.sel[ctz(U) * q.n + v]);
    }
    return x;
}

// OR of adj[v] over the vertices v of F
template <typename M>
__device__ __forceinline__ M nbrs(const SQ<M>& q, M F) {
    M N = 0;
    for (M T = F; T; T &= T - 1) N |= q.adj[ctz(T)];
    return N;
}
template <>
__device__ __forceinline__ uint32_t nbrs(const SQ<uint32_t>& q, uint32_t F) {
    if (q.nbtab) return q.nb.t[0][F & 255u] | q.nb.t[1][(F >> 8) & 255u] | q.nb.t[2][(F >> 16) & 255u] | q.nb.t[3][F >> 24];
    uint32_t N = 0;
    for (uint32_t T = F; T; T &= T - 1) N |= q.adj[ctz(T)];
    return N;
}

// Build SQ::nb from the device query (call after load_query, before the
// __syncthreads that publishes the shared query)
__device__ __forceinline__ void build_nbtab(SQ<uint32_t>& s, const QueryDev<uint32_t>* q) {
    const int n = q->n;
    for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) {
        const int c = i >> 8, b = i & 255;
        uint32_t x = 0;
        for (int j = 0; j < 8; j++)
            if (((b >> j) & 1) && 8 * c + j < n) x |= q->adj[8 * c + j];
        s.nb.t[c][b] = x;
    }
    if (threadIdx.x == 0) s.nbtab = 1;
}

// grow(source, restriction) (Alg. grow): all vertices of the
// restriction reachable from the source.  Frontier-at-a-time BFS in registers:
// N = (OR adj[v] over the frontier) & restriction & ~V.
template <typename M>
__device__ __forceinline__ M grow(const SQ<M>& q, M source, M restriction) {
    M V = source, F = source;
    while (F) {
        M N = nbrs(q, F);
        N &= restriction & ~V;
        V |= N;
        F = N;
    }
    return V;
}

// connected(S) (Alg. connected): grow from the lowest vertex
// (reading R9), stopping as soon as every vertex is reached.
template <typename M>
__device__ __forceinline__ bool connected(const SQ<M>& q, M S) {
    if (!S) return false;
    M V = lowbit(S), F = V;
    while (F) {
        if (V == S) return true;
        M N = nbrs(q, F);
        N &= S & ~V;
        V |= N;
        F = N;
    }
    return V == S;
}

// Reading R20 (memo connectivity).  Level by level, every connected set of
// j < k relations is in the memo before level k starts, and with
// the bitmask-indexed memo a set's slot is its mask.  The host fills the cost
// array with kMemoAbsent (an all-ones NaN that no sum of non-negative costs
// produces), so a proper subset X of a level-k set is connected iff its slot
// holds anything else: the CCP-block tests of Alg. mpdp_generalization
// ("lb is connected", "rb is connected") become one probe each
// instead of a BFS (Alg. connected).  Singletons are connected.
constexpr unsigned long long kMemoAbsent = ~0ull;
__device__ __forceinline__ bool memo_present(double c) {
    // (the high word decides: a cost, >= 0 or +inf, never has an all-ones one)
    return __double2hiint(c) != -1;
}
template <typename M>
__device__ __forceinline__ bool conn_sub(const SQ<M>& q, M X) {
    if (q.mc) return (X & (X - 1)) == 0 ? X != 0 : memo_present(q.mc[X]);
    return connected(q, X);
}

// 2|E(G[S])|
template <typename M>
__device__ __forceinline__ int induced_degree_sum(const SQ<M>& q, M S) {
    int e2 = 0;
    for (M T = S; T; T &= T - 1) e2 += popc(q.adj[ctz(T)] & S);
    return e2;
}

// Connectivity filter specialised by graph class (same predicate as Alg.
// connected):
//   clique : every non-empty subset is connected;
//   others : grow from the lowest vertex (register BFS; on stars and
//            snowflakes it stops after a few frontier steps, which measured
//            faster than counting induced edges).
template <typename M, int CLS>
__device__ __forceinline__ bool connected_cls(const SQ<M>& q, M S, int k) {
    if (CLS == CLS_CLIQUE) return S != 0;
    return connected(q, S);
}

// Cut vertices of a connected G[S], |S| >= 3, with memo connectivity (reading
// R20): v is a cut vertex iff S \ {v} is disconnected, i.e. absent from the
// memo.  Eight probes in flight.
template <typename M>
__device__ __forceinline__ M cut_vertices_memo(const SQ<M>& q, M S) {
    M cut = 0;
    for (M T = S; T;) {
        double c[8];
        M b[8];
#pragma unroll
        for (int i = 0; i < 8; i++) {
            b[i] = lowbit(T);
            c[i] = 0.0;
            if (T) {
                c[i] = q.mc[S & ~b[i]];
                T &= T - 1;
            }
        }
#pragma unroll
        for (int i = 0; i < 8; i++)
            if (!memo_present(c[i])) cut |= b[i];
    }
    return cut;
}

// Find-Blocks from the cut vertices (reading R21), registers and frontier BFS
// only.  For a vertex x that is not a cut vertex, its block is
//     B(x) = intersection over cut vertices c of (comp(S \ {c}, x) + c)
// where comp(X, x) = grow({x}, X): each term contains B(x) (a block minus one
// vertex stays connected), and a vertex y outside B(x) is cut off from x by the
// cut vertex of B(x) on the way to y in the block-cut tree.  The same holds for
// an edge (u, v) in place of x (comp taken from the endpoint that is not c),
// which finds the blocks made only of cut vertices.  A pendant x (one
// neighbour u in S) is the block {x, u} directly.
template <typename M>
__device__ __forceinline__ M block_of_edge(const SQ<M>& q, M S, M cut, int u, int v) {
    M B = S;
    for (M T = cut; T; T &= T - 1) {
        const int c = ctz(T);
        B &= grow(q, bitm<M>(c == u ? v : u), S & ~bitm<M>(c)) | bitm<M>(c);
    }
    return B;
}
template <typename M>
__device__ int blocks_from_cut(const SQ<M>& q, M S, M cut, M* blk) {
    int nb = 0;
    M done = 0;
    for (M rest = S & ~cut; rest; rest = S & ~cut & ~done) {
        const int x = ctz(rest);
        const M nx = q.adj[x] & S;
        const M B = (nx & (nx - 1)) == 0 ? (bitm<M>(x) | nx) : block_of_edge(q, S, cut, x, ctz(nx));
        blk[nb++] = B;
        done |= B;
    }
    for (M U = cut; U; U &= U - 1) {       // blocks of cut vertices only
        const int u = ctz(U);
        for (M V = q.adj[u] & cut & ~(bitm<M>(u + 1) - 1); V; V &= V - 1) {
            const int v = ctz(V);
            const M uv = bitm<M>(u) | bitm<M>(v);
            bool found = false;
            for (int i = 0; i < nb && !found; i++) found = (blk[i] & uv) == uv;
            if (!found) blk[nb++] = block_of_edge(q, S, cut, u, v);
        }
    }
    return nb;
}

// Find-Blocks: biconnected components of G[S] by an iterative
// Hopcroft-Tarjan DFS with a vertex stack; bitmask adjacency, small local arrays.
// With memo connectivity (q.mc) the blocks come from the cut vertices instead
// (reading R21: no DFS stacks in local memory).
template <typename M>
__device__ int find_blocks(const SQ<M>& q, M S, M* blk) {
    if (q.mc) return blocks_from_cut(q, S, cut_vertices_memo(q, S), blk);
    constexpr int N = MaxN<M>::value;
    unsigned char disc[N], low[N], par[N], vst[N], dst[N];
    M rem[N];
    int vsp = 0, dsp = 0, t = 0, nb = 0;
    const int r = ctz(S);
    M visited = bitm<M>(r);
    disc[r] = low[r] = (unsigned char)t++;
    par[r] = 0xff;
    rem[r] = q.adj[r] & S;
    vst[vsp++] = (unsigned char)r;
    dst[dsp++] = (unsigned char)r;
    while (dsp) {
        const int v = dst[dsp - 1];
        if (rem[v]) {
            const int u = ctz(rem[v]);
            rem[v] &= rem[v] - 1;
            if (!((visited >> u) & 1)) {
                visited |= bitm<M>(u);
                par[u] = (unsigned char)v;
                disc[u] = low[u] = (unsigned char)t++;
                rem[u] = q.adj[u] & S;
                vst[vsp++] = (unsigned char)u;
                dst[dsp++] = (unsigned char)u;
            } else if (u != par[v]) {
                if (disc[u] < low[v]) low[v] = disc[u];
            }
        } else {
            --dsp;
            if (dsp) {
                const int p = par[v];
                if (low[v] < low[p]) low[p] = low[v];
                if (low[v] >= disc[p]) {          // p separates v's subtree: a block
                    M B = bitm<M>(p);
                    int w;
                    do {
                        w = vst[--vsp];
                        B |= bitm<M>(w);
                    } while (w != v);
                    blk[nb++] = B;
                }
            }
        }
    }
    return nb;
}

enum SetKind : int { KIND_TREE = 0, KIND_COMPLETE = 1, KIND_BLOCKS = 2, KIND_ONEBLOCK = 3 };

// G[S] (connected, |S| >= 3) is biconnected -- Find-Blocks would return the one
// block S -- iff no vertex has induced degree < 2 and no S \ {v} is
// disconnected (register BFS per vertex; cheaper than the Hopcroft-Tarjan DFS
// with its local-memory stacks, and the common case on dense random graphs)
template <typename M>
__device__ __forceinline__ bool biconnected(const SQ<M>& q, M S) {
    for (M T = S; T; T &= T - 1)
        if (popc(q.adj[ctz(T)] & S) < 2) return false;
    if (q.mc) {                            // reading R20: |S| - 1 >= 2, four probes in flight
        for (M T = S; T;) {
            double c[4];
#pragma unroll
            for (int i = 0; i < 4; i++) {
                c[i] = 0.0;
                if (T) {
                    c[i] = q.mc[S & ~lowbit(T)];
                    T &= T - 1;
                }
            }
#pragma unroll
            for (int i = 0; i < 4; i++)
                if (!memo_present(c[i])) return false;
        }
        return true;
    }
    for (M T = S; T; T &= T - 1)
        if (!connected(q, S & ~lowbit(T))) return false;
    return true;
}

// Kind and MPDP join-pair count (reading R3) of one connected set of size k:
// tree-induced sets have one pair per edge (Alg. mpdp_trees);
// complete sets are one block with 2^(k-1)-1 splits (Lemma generic:opt);
// otherwise sum over blocks of 2^(b-1)-1 (Alg. mpdp_generalization).
// (blk_out: the first kHeavyBlk blocks of a KIND_BLOCKS set and their count in
// *nb_out, cached with the heavy list so that work items skip Find-Blocks)
constexpr int kHeavyBlk = 8;
template <typename M, int CLS>
__device__ __forceinline__ int set_kind(const SQ<M>& q, M S, int k, unsigned long long& w, M* blk_out = nullptr,
                                        int* nb_out = nullptr, M* cut_out = nullptr) {
    if (CLS == CLS_TREE) {
        w = (unsigned long long)(k - 1);
        return KIND_TREE;
    }
    if (CLS == CLS_CLIQUE) {
        w = (1ull << (k - 1)) - 1;
        return KIND_COMPLETE;
    }
    if (q.dpsub) {                         // ablation: Alg. generic_dpsub's enumeration
        w = (1ull << (k - 1)) - 1;
        return KIND_BLOCKS;
    }
    const int e2 = induced_degree_sum(q, S);
    if (e2 == 2 * (k - 1)) {
        w = (unsigned long long)(k - 1);
        return KIND_TREE;
    }
    if (e2 == k * (k - 1)) {
        w = (1ull << (k - 1)) - 1;
        return KIND_COMPLETE;
    }
    M blk[MaxN<M>::value];
    int nb;
    if (q.mc) {                            // reading R21: cut vertices by probes, blocks from them
        const M cut = cut_vertices_memo(q, S);
        if (cut_out) *cut_out = cut;
        if (!cut) {                        // one (non-complete) block: S
            w = (1ull << (k - 1)) - 1;
            return KIND_ONEBLOCK;
        }
        nb = blocks_from_cut(q, S, cut, blk);
    } else {
        if (biconnected(q, S)) {           // one (non-complete) block: S
            w = (1ull << (k - 1)) - 1;
            return KIND_ONEBLOCK;
        }
        nb = find_blocks(q, S, blk);
    }
    unsigned long long s = 0;
    for (int i = 0; i < nb; i++) s += (1ull << (popc(blk[i]) - 1)) - 1;
    w = s;
    if (blk_out) {
        for (int i = 0; i < nb && i < kHeavyBlk; i++) blk_out[i] = blk[i];
        *nb_out = nb;
    }
    return KIND_BLOCKS;
}

// Pair count of a set whose kind is already known (set_kind's w without its
// tests): closed forms, or Find-Blocks for KIND_BLOCKS (blocks cached as in
// set_kind).
// (cut: the cut vertices of a KIND_BLOCKS set when set_kind found them by
// probes, reading R21; 0 = not known)
template <typename M, int CLS>
__device__ __forceinline__ unsigned long long kind_pairs(const SQ<M>& q, M S, int k, int kind, M* blk_out = nullptr,
                                                         int* nb_out = nullptr, M cut = 0) {
    if (kind == KIND_TREE) return (unsigned long long)(k - 1);
    if (kind != KIND_BLOCKS || q.dpsub) return (1ull << (k - 1)) - 1;
    M blk[MaxN<M>::value];
    const int nb = (q.mc && cut) ? blocks_from_cut(q, S, cut, blk) : find_blocks(q, S, blk);
    unsigned long long s = 0;
    for (int i = 0; i < nb; i++) s += (1ull << (popc(blk[i]) - 1)) - 1;
    if (blk_out) {
        for (int i = 0; i < nb && i < kHeavyBlk; i++) blk_out[i] = blk[i];
        *nb_out = nb;
    }
    return s;
}

// colex combinadic unrank (reading R10): the r-th k-subset of {0..n-1} has
// elements c_k > ... > c_1 with r = sum_i C(c_i, i)
template <typename M>
__device__ __forceinline__ M unrank_colex(const unsigned long long* binom, int stride, int n, int k,
                                          unsigned long long r) {
    M S = 0;
    int c = n - 1;
    for (int i = k; i >= 1; i--) {
        while (binom[c * stride + i] > r) c--;
        S |= bitm<M>(c);
        r -= binom[c * stride + i];
        c--;
    }
    return S;
}

}  // namespace mpdp
