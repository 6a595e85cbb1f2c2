// heuristics.cpp — IDP2 and UnionDP drivers for large
// queries, generic over an exact inner DP.  The product calls them with the GPU
// MPDP as the inner solver (mpdp_optimize, algo IDP2_MPDP / UNIONDP_MPDP); the
// exported mpdp_heuristic_optimize lets a caller plug any inner solver (the
// CPU tests use it to check the driver logic on machines without a GPU).
//
// Plans of the drivers live in a host node pool.  A composite node (a
// temporary table of IDP2, a partition of UnionDP) is a pool subtree; inner
// sub-problems see it as one relation with card = card of its subplan and
// leaf_cost = cost of its subplan (reading R17).  Edges between
// composites are the original edges between their relation sets, merged by
// multiplying their selectivities in edge-id order.
//
// Cardinality of a join node: card(L) * card(R) * prod of the selectivities
// of the original edges crossing (L, R) in edge-id order; cost = (cost(L) +
// cost(R)) + card (C_out).  The reported cost of a heuristic plan is
// recomputed bottom-up over the final tree with this recurrence.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <numeric>
#include <queue>
#include <tuple>
#include <string>
#include <unordered_map>
#include <vector>

#include "mpdp.h"
#include "heuristics.h"

namespace mpdp_heur {

struct HNode {
    int left = -1, right = -1;   // pool indices
    int relation = -1;           // base relation for leaves
    double card = 0, cost = 0;
    int nleaves = 1;             // leaves of the CURRENT tree (a temp table counts 1)
    int temp = -1;               // IDP2: this leaf is a temp table whose subplan is pool[temp]
    int parent = -1;
    int minrel = -1;             // lowest base relation under this node (IDP2's last tie-break)
};

struct Query {
    int n = 0;
    std::vector<double> card, leaf;
    std::vector<std::pair<int, int>> edges;
    std::vector<double> sel;
    std::vector<std::vector<std::pair<int, int>>> adj;   // (neighbour, edge id)
};

struct Driver {
    const Query& Q;
    InnerSolver solve;
    void* user;
    std::vector<HNode> pool;
    unsigned long long pairs = 0, ccp = 0, csg = 0, calls = 0;
    std::string err;

    InnerBatchSolver solve_batch = nullptr;   // optional: independent sub-problems in one call
    double solve_ms = 0;                      // host wall time inside the inner solver calls
    unsigned long long batch_calls = 0, batched = 0;

    Driver(const Query& q, InnerSolver s, void* u) : Q(q), solve(s), user(u) {}

    // relation set of every pool node as a bitset of W words (a leaf: its bit;
    // a join: the OR of its children), and its relation count, so a join's
    // cross edges are found from the smaller side alone (join_card_cost)
    int W = 0;
    std::vector<uint64_t> bits;
    std::vector<int> nrel;
    int add_node(const HNode& h) {
        if (!W) W = (Q.n + 63) / 64;
        pool.push_back(h);
        const int id = (int)pool.size() - 1;
        bits.resize((size_t)(id + 1) * W, 0);
        nrel.resize(id + 1, 0);
        uint64_t* b = &bits[(size_t)id * W];
        if (h.relation >= 0) {
            b[h.relation >> 6] |= 1ull << (h.relation & 63);
            nrel[id] = 1;
        } else {
            const uint64_t* l = &bits[(size_t)h.left * W];
            const uint64_t* r = &bits[(size_t)h.right * W];
            for (int w = 0; w < W; w++) b[w] = l[w] | r[w];
            nrel[id] = nrel[h.left] + nrel[h.right];
        }
        return id;
    }
    int leaf(int r) {
        HNode h;
        h.relation = r;
        h.minrel = r;
        h.card = Q.card[r];
        h.cost = Q.leaf[r];
        return add_node(h);
    }

    // A sub-problem over the composites `nodes` (pool roots covering disjoint
    // relation sets): its query graph (merged edges: product of selectivities
    // in edge-id order) and the buffers of its result.
    struct SubGraph {
        std::vector<int> nodes;
        std::vector<double> card, lc, es;
        std::vector<uint32_t> ed;
        std::vector<mpdp_plan_node> out;
        mpdp_query_graph g;
        mpdp_result r;
    };
    void prepare_sub(const std::vector<int>& nodes, const std::vector<int>& owner_of_rel_local, SubGraph& sg) {
        const int m = (int)nodes.size();
        sg.nodes = nodes;
        std::map<std::pair<int, int>, double> merged;
        for (size_t e = 0; e < Q.edges.size(); e++) {
            const int a = owner_of_rel_local[Q.edges[e].first], b = owner_of_rel_local[Q.edges[e].second];
            if (a < 0 || b < 0 || a == b) continue;
            auto key = std::make_pair(std::min(a, b), std::max(a, b));
            auto it = merged.find(key);
            if (it == merged.end()) merged.emplace(key, Q.sel[e]);
            else it->second = it->second * Q.sel[e];
        }
        sg.card.resize(m);
        sg.lc.resize(m);
        for (int i = 0; i < m; i++) {
            sg.card[i] = pool[nodes[i]].card;
            sg.lc[i] = pool[nodes[i]].cost;
        }
        for (auto& kv : merged) {
            sg.ed.push_back((uint32_t)kv.first.first);
            sg.ed.push_back((uint32_t)kv.first.second);
            sg.es.push_back(kv.second);
        }
        sg.g.n = (uint32_t)m;
        sg.g.cardinalities = sg.card.data();
        sg.g.n_edges = (uint32_t)sg.es.size();
        sg.g.edges = sg.ed.data();
        sg.g.selectivities = sg.es.data();
        sg.g.leaf_costs = sg.lc.data();
        sg.out.assign(2 * m - 1, mpdp_plan_node{});
        memset(&sg.r, 0, sizeof(sg.r));
        sg.r.nodes = sg.out.data();
        sg.r.capacity = (uint32_t)sg.out.size();
    }
    // counters + translation of a solved sub-problem: local leaf i -> composite
    // nodes[i]; returns the pool root of the subplan
    int finish_sub(const SubGraph& sg) {
        const mpdp_result& r = sg.r;
        pairs += r.pairs_evaluated;
        ccp += r.ccp_pairs;
        csg += r.csg_count;
        std::vector<int> map(r.n_nodes, -1);
        for (uint32_t i = 0; i < r.n_nodes; i++) {
            const mpdp_plan_node& nd = sg.out[i];
            if (nd.relation >= 0) {
                map[i] = sg.nodes[nd.relation];
                continue;
            }
            HNode h;
            h.left = map[nd.left];
            h.right = map[nd.right];
            h.nleaves = pool[h.left].nleaves + pool[h.right].nleaves;
            h.minrel = std::min(pool[h.left].minrel, pool[h.right].minrel);
            const int id = add_node(h);
            join_card_cost(id);
            map[i] = id;
        }
        return map[r.n_nodes - 1];
    }
    // Solve the sub-problem whose relations are the composites `nodes`;
    // returns the pool root of the optimal subplan (composites expanded), or -1.
    int solve_sub(const std::vector<int>& nodes, const std::vector<std::vector<int>>& rels,
                  const std::vector<int>& owner_of_rel_local) {
        (void)rels;
        if (nodes.size() == 1) return nodes[0];
        SubGraph sg;
        prepare_sub(nodes, owner_of_rel_local, sg);
        const auto t0 = std::chrono::steady_clock::now();
        const mpdp_status st = solve(user, &sg.g, &sg.r);
        solve_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        calls++;
        if (st != MPDP_OK) {
            err = "inner DP failed (status " + std::to_string((int)st) + ")";
            return -1;
        }
        return finish_sub(sg);
    }

    // card/cost of a join node from its children (recurrence of the header)
    void collect(int x, std::vector<int>& rels) const {
        if (pool[x].relation >= 0) {
            rels.push_back(pool[x].relation);
            return;
        }
        collect(pool[x].left, rels);
        collect(pool[x].right, rels);
    }
    // the edges between the two sides: the smaller side's relations are
    // walked, the larger side is a bitset lookup
    std::vector<int> scratch_s, cross;
    void join_card_cost(int id) {
        HNode& h = pool[id];
        const bool lsmall = nrel[h.left] <= nrel[h.right];
        scratch_s.clear();
        collect(lsmall ? h.left : h.right, scratch_s);
        const uint64_t* big = &bits[(size_t)(lsmall ? h.right : h.left) * W];
        cross.clear();
        for (int r : scratch_s)
            for (auto [u, e] : Q.adj[r])
                if ((big[u >> 6] >> (u & 63)) & 1ull) cross.push_back(e);
        std::sort(cross.begin(), cross.end());   // the product in edge-id order (reading R17)
        double c = pool[h.left].card * pool[h.right].card;
        for (int e : cross) c = c * Q.sel[e];
        h.card = c;
        h.cost = (pool[h.left].cost + pool[h.right].cost) + c;
    }
};

// ---------------------------------------------------------------- GOO
// Greedy Operator Ordering (initial plan of IDP2):
// repeatedly join the two connected components whose join has the smallest
// cardinality (ties: smaller cost, then smaller lowest relation id).
static int goo(Driver& D) {
    const Query& Q = D.Q;
    const int n = Q.n;
    std::vector<int> root(n), comp_of(n);
    std::vector<int> minrel(n);
    std::vector<std::map<int, double>> nb(n);   // component -> neighbour component -> sel product
    for (int v = 0; v < n; v++) {
        root[v] = D.leaf(v);
        comp_of[v] = v;
        minrel[v] = v;
    }
    for (size_t e = 0; e < Q.edges.size(); e++) {
        const int a = Q.edges[e].first, b = Q.edges[e].second;
        auto it = nb[a].find(b);
        if (it == nb[a].end()) {
            nb[a][b] = Q.sel[e];
            nb[b][a] = Q.sel[e];
        } else {
            it->second = it->second * Q.sel[e];
            nb[b][a] = it->second;
        }
    }
    std::vector<char> alive(n, 1);
    // Candidate joins ordered as a full scan of the component pairs would
    // order them: (card, cost, lowest relation, a, b) with a < b.  Each
    // component caches its best pair; a merge recomputes the merged
    // component's pairs and the cache of a neighbour only when its cached pair
    // touched the merged components or the new pair beats it.  The step's join
    // is the minimum over the caches (O(n) per step instead of O(E) map walks).
    struct Cand {
        double c = 0, cost = 0;
        int key = 0, a = -1, b = -1;
        bool less(const Cand& o) const {
            if (o.a < 0) return a >= 0;
            if (a < 0) return false;
            if (c != o.c) return c < o.c;
            if (cost != o.cost) return cost < o.cost;
            if (key != o.key) return key < o.key;
            if (a != o.a) return a < o.a;
            return b < o.b;
        }
    };
    auto pair_cand = [&](int x, int y, double s) {
        Cand t;
        t.a = std::min(x, y);
        t.b = std::max(x, y);
        t.c = D.pool[root[t.a]].card * D.pool[root[t.b]].card * s;
        t.cost = (D.pool[root[t.a]].cost + D.pool[root[t.b]].cost) + t.c;
        t.key = std::min(minrel[t.a], minrel[t.b]);
        return t;
    };
    std::vector<Cand> best(n);
    auto recompute = [&](int x) {
        Cand m;
        for (auto& [y, s] : nb[x]) {
            const Cand t = pair_cand(x, y, s);
            if (t.less(m)) m = t;
        }
        best[x] = m;
    };
    for (int a = 0; a < n; a++) recompute(a);
    for (int step = 0; step < n - 1; step++) {
        int ba = -1, bb = -1;
        {
            Cand m;
            for (int a = 0; a < n; a++)
                if (alive[a] && best[a].less(m)) m = best[a];
            ba = m.a;
            bb = m.b;
        }
        if (ba < 0) return -1;   // disconnected (validated before)
        HNode h;
        const bool swap = minrel[bb] < minrel[ba];
        h.left = root[swap ? bb : ba];
        h.right = root[swap ? ba : bb];
        h.nleaves = D.pool[h.left].nleaves + D.pool[h.right].nleaves;
        h.minrel = std::min(D.pool[h.left].minrel, D.pool[h.right].minrel);
        const int id = D.add_node(h);
        D.join_card_cost(id);
        // merge component bb into ba
        root[ba] = id;
        minrel[ba] = std::min(minrel[ba], minrel[bb]);
        alive[bb] = 0;
        for (auto& [c, s] : nb[bb]) {
            if (c == ba) continue;
            auto it = nb[ba].find(c);
            if (it == nb[ba].end()) nb[ba][c] = s;
            else it->second = it->second * s;
            nb[c].erase(bb);
            nb[c][ba] = nb[ba][c];
        }
        nb[ba].erase(bb);
        nb[bb].clear();
        recompute(ba);
        for (auto& [c, sv] : nb[ba]) {         // neighbours: their pair with ba changed
            const Cand t = pair_cand(c, ba, sv);
            if (best[c].a == ba || best[c].b == ba || best[c].a == bb || best[c].b == bb) recompute(c);
            else if (t.less(best[c])) best[c] = t;
        }
    }
    for (int a = 0; a < n; a++)
        if (alive[a]) return root[a];
    return -1;
}

// ---------------------------------------------------------------- IDP2
// Alg. idp2_goo: T <- GOO; while T has more than one leaf: pick
// the subtree T' with 1 < leaves(T') <= k and maximal cost C(T') (ties: more
// leaves, then lower lowest relation id), optimise its leaves with the inner
// DP and replace T' by a temporary table; finally expand the temporaries.
static int idp2(Driver& D, int k) {
    int root = goo(D);
    if (root < 0) return -1;
    while (true) {
        // current tree: leaves are base relations or temp tables
        std::vector<int> order;                 // post-order of internal nodes
        std::vector<int> st{root};
        std::vector<int> post;
        while (!st.empty()) {
            const int x = st.back();
            st.pop_back();
            post.push_back(x);
            const HNode& h = D.pool[x];
            if (h.relation < 0 && h.temp < 0) {
                st.push_back(h.left);
                st.push_back(h.right);
            }
        }
        std::reverse(post.begin(), post.end());
        std::vector<int> minrel(D.pool.size(), 0);   // per pool node (was a hash map: ~8 ms at n = 1000)
        int best = -1;
        for (int x : post) {
            HNode& h = D.pool[x];
            if (h.relation >= 0 || h.temp >= 0) {
                h.nleaves = 1;
                minrel[x] = h.minrel;          // cached when the node / temp table was made
                continue;
            }
            h.nleaves = D.pool[h.left].nleaves + D.pool[h.right].nleaves;
            h.cost = (D.pool[h.left].cost + D.pool[h.right].cost) + h.card;
            minrel[x] = std::min(minrel[h.left], minrel[h.right]);
            if (h.nleaves > 1 && h.nleaves <= k) {
                if (best < 0) {
                    best = x;
                } else {
                    const HNode& b = D.pool[best];
                    if (h.cost > b.cost || (h.cost == b.cost && h.nleaves > b.nleaves) ||
                        (h.cost == b.cost && h.nleaves == b.nleaves && minrel[x] < minrel[best]))
                        best = x;
                }
            }
        }
        if (best < 0) break;                    // the root is a single temp table / leaf
        // leaves of the chosen subtree
        std::vector<int> leaves;
        st.assign(1, best);
        while (!st.empty()) {
            const int x = st.back();
            st.pop_back();
            const HNode& h = D.pool[x];
            if (h.relation >= 0 || h.temp >= 0) leaves.push_back(x);
            else {
                st.push_back(h.right);
                st.push_back(h.left);
            }
        }
        // inner DP over the leaves (temp tables as composites)
        std::vector<int> comps;
        std::vector<std::vector<int>> rels;
        std::vector<int> owner(D.Q.n, -1);
        for (size_t i = 0; i < leaves.size(); i++) {
            const int body = D.pool[leaves[i]].temp >= 0 ? D.pool[leaves[i]].temp : leaves[i];
            comps.push_back(body);
            std::vector<int> r;
            D.collect(body, r);
            for (int x : r) owner[x] = (int)i;
            rels.push_back(r);
        }
        const int sub = D.solve_sub(comps, rels, owner);
        if (sub < 0) return -1;
        // replace the subtree `best` by a temp table leaf
        HNode t;
        t.temp = sub;
        t.minrel = D.pool[sub].minrel;
        t.card = D.pool[sub].card;
        t.cost = D.pool[sub].cost;
        D.pool[best] = t;
        if (D.pool[root].temp >= 0) {          // the whole query is one temp table: done
            root = D.pool[root].temp;
            break;
        }
    }
    // expand temp tables
    std::vector<int> st{root};
    while (!st.empty()) {
        const int x = st.back();
        st.pop_back();
        HNode& h = D.pool[x];
        if (h.relation >= 0) continue;
        if (h.temp >= 0) {
            D.pool[x] = D.pool[h.temp];
            st.push_back(x);
            continue;
        }
        st.push_back(h.left);
        st.push_back(h.right);
    }
    return root;
}

// ---------------------------------------------------------------- UnionDP
// Alg. uniondp: while the (composite)
// graph has more than k nodes: weight every edge by the C_out cost of joining
// its two endpoints; union-find over nodes, repeatedly uniting the two sets of
// the edge with minimal (combined size, weight, edge id) among edges whose sets
// differ and whose combined size is <= t; optimise each partition with the
// inner DP; contract partitions into composite nodes; recurse.  k bounds the
// final exact DP (the recursion ends once <= k composites remain), t <= k the
// partitions (the paper's upper threshold, "t in [1, k]"; its GPU
// runs use k = 25, t = 15).  t = k is Alg. uniondp as listed.
static int uniondp(Driver& D, int k, int t) {
    const Query& Q = D.Q;
    std::vector<int> node_of(Q.n);          // relation -> current composite index
    std::vector<int> comp;                  // composite -> pool root
    for (int r = 0; r < Q.n; r++) {
        comp.push_back(D.leaf(r));
        node_of[r] = r;
    }
    while ((int)comp.size() > k) {
        const int m = (int)comp.size();
        // composite edges (merged original edges, edge-id order), weight = join cost
        std::map<std::pair<int, int>, double> msel;
        std::map<std::pair<int, int>, int> mid;
        for (size_t e = 0; e < Q.edges.size(); e++) {
            const int a = node_of[Q.edges[e].first], b = node_of[Q.edges[e].second];
            if (a == b) continue;
            auto key = std::make_pair(std::min(a, b), std::max(a, b));
            auto it = msel.find(key);
            if (it == msel.end()) {
                msel.emplace(key, Q.sel[e]);
                mid.emplace(key, (int)e);
            } else {
                it->second = it->second * Q.sel[e];
            }
        }
        struct CE {
            int a, b, id;
            double w;
        };
        std::vector<CE> ce;
        for (auto& kv : msel) {
            const int a = kv.first.first, b = kv.first.second;
            const double c = D.pool[comp[a]].card * D.pool[comp[b]].card * kv.second;
            ce.push_back({a, b, mid[kv.first], (D.pool[comp[a]].cost + D.pool[comp[b]].cost) + c});
        }
        std::vector<int> uf(m), sz(m, 1);
        std::iota(uf.begin(), uf.end(), 0);
        auto find = [&](int x) {
            while (uf[x] != x) x = uf[x] = uf[uf[x]];
            return x;
        };
        // repeatedly the edge of minimal (combined size, weight, edge id) among
        // edges joining different sets with combined size <= k: a min-heap with
        // lazy re-keying -- set sizes only grow, so a stored key never exceeds
        // the edge's current key, and an entry whose key is still current is
        // the minimum (O(E log E) per level instead of a scan per union)
        using UKey = std::tuple<int, double, int, int>;   // (combined size, weight, edge id, ce index)
        std::priority_queue<UKey, std::vector<UKey>, std::greater<UKey>> pq;
        for (size_t i = 0; i < ce.size(); i++) pq.emplace(2, ce[i].w, ce[i].id, (int)i);
        int unions = 0;
        while (!pq.empty()) {
            const auto [s0, w0, id0, i] = pq.top();
            pq.pop();
            const int ra = find(ce[i].a), rb = find(ce[i].b);
            if (ra == rb) continue;                    // joined already
            const int s = sz[ra] + sz[rb];
            if (s > t) continue;                       // can only grow: never valid again
            if (s != s0) {                             // stale size: re-key
                pq.emplace(s, w0, id0, i);
                continue;
            }
            uf[rb] = ra;
            sz[ra] += sz[rb];
            unions++;
        }
        if (!unions) {
            D.err = "UnionDP made no progress";
            return -1;
        }
        // optimise every partition; contract
        std::map<int, std::vector<int>> parts;  // uf root -> composites (ascending)
        for (int i = 0; i < m; i++) parts[find(i)].push_back(i);
        std::vector<int> newcomp;
        std::vector<int> new_of_old(m);
        // the partitions of this level are independent sub-problems: with a
        // batch solver they are solved in one call (one CTA per small one on
        // the GPU), then translated in partition order as before
        std::vector<Driver::SubGraph> subs;
        subs.reserve(parts.size());
        std::vector<int> sub_of_part;
        for (auto& [r, members] : parts) {
            if (members.size() == 1) {
                sub_of_part.push_back(-1);
                continue;
            }
            std::vector<int> nodes;
            std::vector<int> owner(Q.n, -1);
            for (size_t i = 0; i < members.size(); i++) {
                nodes.push_back(comp[members[i]]);
                std::vector<int> rr;
                D.collect(comp[members[i]], rr);
                for (int x : rr) owner[x] = (int)i;
            }
            subs.emplace_back();
            D.prepare_sub(nodes, owner, subs.back());
            sub_of_part.push_back((int)subs.size() - 1);
        }
        if (D.solve_batch && subs.size() > 1) {
            std::vector<mpdp_query_graph> gs;
            std::vector<mpdp_result> rs;
            for (auto& sg : subs) {
                gs.push_back(sg.g);
                rs.push_back(sg.r);
            }
            const auto t0 = std::chrono::steady_clock::now();
            const mpdp_status st = D.solve_batch(D.user, gs.data(), (uint32_t)gs.size(), rs.data());
            D.solve_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            D.calls += subs.size();
            D.batch_calls++;
            D.batched += subs.size();
            if (st != MPDP_OK) {
                D.err = "inner DP batch failed (status " + std::to_string((int)st) + ")";
                return -1;
            }
            for (size_t i = 0; i < subs.size(); i++) subs[i].r = rs[i];
        } else {
            for (auto& sg : subs) {
                const auto t0 = std::chrono::steady_clock::now();
                const mpdp_status st = D.solve(D.user, &sg.g, &sg.r);
                D.solve_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
                D.calls++;
                if (st != MPDP_OK) {
                    D.err = "inner DP failed (status " + std::to_string((int)st) + ")";
                    return -1;
                }
            }
        }
        size_t pi = 0;
        for (auto& [r, members] : parts) {
            const int si = sub_of_part[pi++];
            const int sub = si < 0 ? comp[members[0]] : D.finish_sub(subs[si]);
            for (int x : members) new_of_old[x] = (int)newcomp.size();
            newcomp.push_back(sub);
        }
        for (int r = 0; r < Q.n; r++) node_of[r] = new_of_old[node_of[r]];
        comp.swap(newcomp);
    }
    // final exact DP over the remaining composites
    std::vector<int> nodes = comp;
    std::vector<std::vector<int>> rels;
    std::vector<int> owner(Q.n, -1);
    for (size_t i = 0; i < nodes.size(); i++) {
        std::vector<int> rr;
        D.collect(nodes[i], rr);
        for (int x : rr) owner[x] = (int)i;
        rels.push_back(rr);
    }
    return D.solve_sub(nodes, rels, owner);
}

// ---------------------------------------------------------------- validation
static mpdp_status load(const mpdp_query_graph* g, Query& Q, std::string& err) {
    if (!g || g->n == 0 || !g->cardinalities || (g->n_edges && (!g->edges || !g->selectivities))) {
        err = "bad graph";
        return MPDP_ERR_INVALID_ARGUMENT;
    }
    Q.n = (int)g->n;
    Q.card.assign(g->cardinalities, g->cardinalities + Q.n);
    Q.leaf.assign(Q.n, 0.0);
    if (g->leaf_costs) Q.leaf.assign(g->leaf_costs, g->leaf_costs + Q.n);
    Q.adj.assign(Q.n, {});
    for (int v = 0; v < Q.n; v++) {
        if (!(Q.card[v] >= 0) || !std::isfinite(Q.card[v]) || !(Q.leaf[v] >= 0) || !std::isfinite(Q.leaf[v])) {
            err = "bad cardinality/leaf cost " + std::to_string(v);
            return MPDP_ERR_INVALID_ARGUMENT;
        }
    }
    std::vector<std::pair<int, int>> seen;
    for (uint32_t e = 0; e < g->n_edges; e++) {
        const uint32_t u = g->edges[2 * e], v = g->edges[2 * e + 1];
        const double s = g->selectivities[e];
        if (!(u < v) || v >= g->n || !(s > 0.0) || !(s <= 1.0)) {
            err = "bad edge " + std::to_string(e);
            return MPDP_ERR_INVALID_ARGUMENT;
        }
        Q.edges.emplace_back((int)u, (int)v);
        Q.sel.push_back(s);
        Q.adj[u].emplace_back((int)v, (int)e);
        Q.adj[v].emplace_back((int)u, (int)e);
    }
    std::vector<std::pair<int, int>> sorted = Q.edges;
    std::sort(sorted.begin(), sorted.end());
    if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end()) {
        err = "duplicate edge";
        return MPDP_ERR_INVALID_ARGUMENT;
    }
    std::vector<char> vis(Q.n, 0);
    std::vector<int> st{0};
    vis[0] = 1;
    int cnt = 1;
    while (!st.empty()) {
        const int x = st.back();
        st.pop_back();
        for (auto [u, e] : Q.adj[x])
            if (!vis[u]) {
                vis[u] = 1;
                cnt++;
                st.push_back(u);
            }
    }
    if (cnt != Q.n) {
        err = "query graph is not connected (cross products excluded)";
        return MPDP_ERR_DISCONNECTED;
    }
    return MPDP_OK;
}

mpdp_status run(const mpdp_query_graph* g, mpdp_algo algo, uint32_t k, InnerSolver solve, void* user,
                mpdp_result* out, std::string& err, InnerBatchSolver solve_batch, uint32_t t) {
    const auto t0 = std::chrono::steady_clock::now();
    if (!out) {
        err = "out is NULL";
        return MPDP_ERR_INVALID_ARGUMENT;
    }
    if (k < 2 || k > 32) {
        err = "k must be in [2, 32] for IDP2/UnionDP";
        return MPDP_ERR_INVALID_ARGUMENT;
    }
    if (t == 0) t = k;
    if (t < 2 || t > k) {
        err = "t must be in [2, k] for UnionDP";
        return MPDP_ERR_INVALID_ARGUMENT;
    }
    // the drivers do O(n) host work per GOO merge / IDP2 iteration (scans of the
    // components and temp tables), O(n^2) per query: bounded where that is
    // still milliseconds
    if (g && g->n > (uint32_t)kMaxHeuristicN) {
        err = "IDP2/UnionDP drivers support n <= " + std::to_string(kMaxHeuristicN);
        return MPDP_ERR_CAPACITY;
    }
    Query Q;
    mpdp_status st = load(g, Q, err);
    if (st != MPDP_OK) return st;
    const int n = Q.n;
    if (out->nodes && out->capacity < (uint32_t)(2 * n - 1)) {
        err = "result capacity < 2n-1";
        return MPDP_ERR_INVALID_ARGUMENT;
    }
    Driver D(Q, solve, user);
    D.solve_batch = solve_batch;
    D.pool.reserve(8 * (size_t)n);
    int root;
    if (n == 1) root = D.leaf(0);
    else root = (algo == MPDP_ALGO_IDP2_MPDP) ? idp2(D, (int)k) : uniondp(D, (int)k, (int)t);
    if (root < 0) {
        err = D.err.empty() ? "heuristic failed" : D.err;
        return MPDP_ERR_INTERNAL;
    }
    if (getenv("MPDP_DEBUG_HEUR_TIME"))
        fprintf(stderr, "[heuristic] %s n=%d k=%u t=%u: %.2f ms total, %.2f ms in %llu inner calls (%llu batched in %llu "
                        "batch calls)\n",
                algo == MPDP_ALGO_IDP2_MPDP ? "IDP2" : "UnionDP", n, k, t,
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(), D.solve_ms,
                D.calls, D.batched, D.batch_calls);
    // recompute card/cost bottom-up over the final tree and emit post-order
    std::vector<int> post;
    std::vector<std::pair<int, int>> st2{{root, 0}};
    while (!st2.empty()) {
        auto& [x, s] = st2.back();
        const HNode& h = D.pool[x];
        if (h.relation >= 0 || s == 2) {
            post.push_back(x);
            st2.pop_back();
            continue;
        }
        const int child = s == 0 ? h.left : h.right;
        s++;
        st2.push_back({child, 0});
    }
    std::unordered_map<int, int> idx;
    std::vector<uint64_t> mask(D.pool.size(), 0);
    uint32_t nn = 0;
    for (int x : post) {
        HNode& h = D.pool[x];
        if (h.relation >= 0) {
            h.card = Q.card[h.relation];
            h.cost = Q.leaf[h.relation];
            if (n <= 64) mask[x] = 1ull << h.relation;
        } else {
            D.join_card_cost(x);
            mask[x] = mask[h.left] | mask[h.right];
        }
        if (out->nodes) {
            mpdp_plan_node& nd = out->nodes[nn];
            nd.relation = h.relation;
            nd.left = h.relation >= 0 ? -1 : idx[h.left];
            nd.right = h.relation >= 0 ? -1 : idx[h.right];
            // internal nodes: left.set < right.set (R7 orientation) when masks exist
            if (h.relation < 0 && n <= 64 && mask[h.left] > mask[h.right]) std::swap(nd.left, nd.right);
            nd.reserved = 0;
            nd.set = n <= 64 ? mask[x] : 0ull;
            nd.cardinality = h.card;
            nd.cost = h.cost;
        }
        idx[x] = (int)nn++;
    }
    out->n_nodes = nn;
    out->root = nn ? nn - 1 : 0;
    out->cost = D.pool[root].cost;
    out->pairs_evaluated = D.pairs;
    out->ccp_pairs = D.ccp;
    out->csg_count = D.csg;
    out->gpu_launches = 0;
    out->time_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    out->inner_calls = (uint32_t)D.calls;
    return MPDP_OK;
}

}  // namespace mpdp_heur
