// star_kernel.cuh — the level loop of Alg. mpdp_gpu for STAR
// queries (a hub adjacent to every other relation), one cooperative kernel.
//
// In a star every connected set of size k >= 2 is {hub} u L with L any
// (k-1)-subset of the n-1 leaves, and G[S] is a star whose k-1 edges are its
// join pairs (Alg. mpdp_trees): ({v}, S \ {v}) for v in L.  So, as
// for cliques, the level needs no enumeration, connectivity filter or
// compaction: set h of level k IS the colex rank h of L
// among the (k-1)-subsets of the leaves, and
//   * the memo of level k is an array of C(n-1, k-1) entries indexed by that
//     rank (half of the C(n, k) rank space, which the general tree kernel
//     scans and filters: 50% of it is disconnected);
//   * rank(L \ {l_m}) = h - C(l_m, m+1) - sum_{i>m} (C(l_i, i+1) - C(l_i, i))
//     (the incremental colex rank of the tree fast path, reading R10);
//   * card(S) = card(S \ {max}) * card[max] * sel(hub, max) bit for bit
//     (reading R19) when max(S) is a leaf.
// Sets are spread lane-consecutively over the grid (each one unranked); small
// levels give G = 2 or 4 lanes to a set.  One grid barrier per level.
#pragma once
#include "fused.cuh"

#include <type_traits>

namespace mpdp {

constexpr int kStarMinBlocks = 3;
constexpr unsigned int kStarSolo = 300;     // levels of at most this many sets run on CTA 0 alone

// leaf space: the vertices other than the hub, vertex v -> v - (v > hub)
__device__ __forceinline__ uint32_t star_compress(uint32_t S, int hub) {
    const unsigned long long s = S;
    return (uint32_t)((s & ((1ull << hub) - 1ull)) | ((s >> (hub + 1)) << hub));
}
__device__ __forceinline__ uint32_t star_expand(uint32_t L, int hub) {
    const unsigned long long l = L;
    return (uint32_t)((l & ((1ull << hub) - 1ull)) | ((l >> hub) << (hub + 1)) | (1ull << hub));
}
__device__ __forceinline__ int star_vertex(int li, int hub) { return li < hub ? li : li + 1; }

__host__ __device__ constexpr size_t star_smem_bytes() {
    return sizeof(SQ<uint32_t>) + sizeof(unsigned int) * 33 * 33 + 8 + sizeof(uint2) * 33 * 33;
}

// (cost, left, card) of a star set of the memo (extraction)
__device__ __forceinline__ unsigned long long star_slot(const Params<uint32_t>& p, const unsigned int* bin, uint32_t S) {
    const uint32_t L = star_compress(S, p.star_hub);
    unsigned int r = 0;
    int i = 1;
    for (uint32_t T = L; T; T &= T - 1, i++) r += bin[(__ffs(T) - 1) * 33 + i];
    return p.star_off[__popc(S)] + r;
}

__global__ void __launch_bounds__(kBlock, kStarMinBlocks) k_dp_star(const __grid_constant__ Params<uint32_t> p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SQ<uint32_t>& q = *reinterpret_cast<SQ<uint32_t>*>(smem_raw);
    unsigned int* bin = reinterpret_cast<unsigned int*>(smem_raw + sizeof(SQ<uint32_t>));   // 33 x 33
    load_query(q, p.q);
    constexpr int NB = MaxN<uint32_t>::value + 1;
    for (int i = threadIdx.x; i < 33 * 33; i += blockDim.x) {
        const int a = i / 33, b = i % 33;
        bin[i] = (a < NB && b < NB) ? (unsigned int)p.q->binom[a * NB + b] : 0u;
    }
    // (C(v, m+1), C(v, m+1) - C(v, m)) pairs of the descending walk, 8-byte aligned
    uint2* binp = reinterpret_cast<uint2*>(smem_raw + ((sizeof(SQ<uint32_t>) + sizeof(unsigned int) * 33 * 33 + 7) & ~size_t(7)));
    __syncthreads();
    for (int i = threadIdx.x; i < 33 * 32; i += blockDim.x) {
        const int a = i / 32, b = i % 32;
        binp[a * 33 + b] = make_uint2(bin[a * 33 + b + 1], bin[a * 33 + b + 1] - bin[a * 33 + b]);
    }
    unsigned int nbar = 0;
    __syncthreads();
    const int n = p.n, hub = p.star_hub, nl = n - 1;
    const bool leaf_costs = q.pad != 0;
    // Levels with at most kStarSolo sets (the first and last few) run on CTA 0
    // alone with __syncthreads as the level barrier; the grid barrier is taken
    // only where a full-grid level follows (a grid barrier costs ~1.5 us plus a
    // global round trip of every set's data).
    auto solo = [&](int k) { return k >= p.k_begin && k <= p.k_end && p.share_hi[k] - p.share_lo[k] <= kStarSolo; };
    for (int k = p.k_begin; k <= p.k_end; k++) {
        const bool one = solo(k);
        if (one && blockIdx.x != 0) {                         // CTA 0's level: join at the next grid barrier
            if (!solo(k + 1) && k < p.k_end) grid_sync(p.gbar, nbar, &p.result->error);
            continue;
        }
        const unsigned long long T = one ? blockDim.x : (unsigned long long)gridDim.x * blockDim.x;
        const unsigned long long gtid = one ? threadIdx.x : (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
        if (blockIdx.x == 0 && threadIdx.x == 0) p.result->t_level[k] = globaltimer_ns();
        const int kl = k - 1;                                 // leaves per set
        // this launch's share [lo, lo + C) of the level's C(n-1, k-1) sets
        // (all of them on one GPU; a rank's segment when sharded)
        const unsigned int lo = p.share_lo[k], C = p.share_hi[k] - lo;
        const double* lvl = p.memo.dcost + p.star_off[k - 1];
        const double* lcard = p.memo.dcard + p.star_off[k - 1];
        const unsigned long long out = p.star_off[k];
        unsigned int G = 1;                                   // lanes per set (small levels)
        while (G < 4 && 2ull * G * C <= T) G <<= 1;
        const unsigned long long ng = T / G, grp = gtid / G;
        const unsigned int sub = threadIdx.x & (G - 1);
        // lane-consecutive sets, each (run) unranked: colex neighbours share
        // their high elements, so a warp's probes of those coalesce (per-thread
        // Gosper runs over a whole share put lanes ~24 sets apart: 27 sectors
        // per request instead of 8.4, star-25 1.19 vs 1.01 ms)
        // runs of RUN consecutive sets per group (one unrank, then Gosper) on
        // levels with several sets per thread: fewer unranks for slightly less
        // coalescing (star-25: RUN 1 -> 2 1.006 -> 0.945 ms; 4 on the largest
        // levels 0.83 -> 0.81 ms; RUN > 1 on small levels costs parallelism)
        const unsigned int RUN = C >= 8ull * T ? 4u : (C >= 4ull * T ? 2u : 1u);
        const unsigned long long rounds = (C + ng * RUN - 1) / (ng * RUN) * RUN;
        uint32_t L = 0;
        unsigned long long nsets = 0;
        for (unsigned long long it = 0; it < rounds; it++) {
            const unsigned long long h = lo + (it / RUN * ng + grp) * RUN + it % RUN;
            const bool act = h < lo + (unsigned long long)C;
            if (act) L = (it % RUN == 0) ? unrank_colex32(bin, nl, kl, (unsigned int)h) : gosper(L);
            Key best = key_inf();
            double cS = 0.0;
            uint32_t S = 0;
            if (act) {
                S = star_expand(L, hub);
                if (k == 2) {                                 // ({hub}, {v}): both leaves of the plan
                    cS = card_of(q, S);
                    const int v = star_vertex(__ffs(L) - 1, hub);
                    const double c = __dadd_rn(__dadd_rn(q.leaf[hub], q.leaf[v]), cS);
                    const uint32_t a = 1u << hub, b = 1u << v;
                    best = Key{(unsigned long long)__double_as_longlong(c), (unsigned long long)(a < b ? a : b)};
                } else {
                    const int pl = 31 - __clz(L);             // max leaf (leaf space)
                    const int pv = star_vertex(pl, hub);
                    if (pv > hub) {                           // max(S) is a leaf: card(S) from card(S \ max)
                        double x = __dmul_rn(__ldcs(lcard + ((unsigned int)h - bin[pl * 33 + kl])), q.card[pv]);
                        cS = __dmul_rn(x, q.sel[hub * q.n + pv]);
                    } else {
                        cS = card_of(q, S);
                    }
                    // descending walk over L, 4 probes in flight
                    double bc = __longlong_as_double(0x7ff0000000000000ll);   // +inf
                    uint32_t bl = 0xffffffffu;
                    unsigned int SD = 0;
                    uint32_t W = L;
                    int m = kl - 1;
                    // batches of 4 elements: kl / 4 full ones without guards, then
                    // the remainder
                    auto batch = [&](auto guard) {
                        constexpr bool GUARD = decltype(guard)::value;
                        unsigned int rk[4];
                        int vv[4];
                        bool ok[4];
#pragma unroll
                        for (int u = 0; u < 4; u++) {
                            const bool has = !GUARD || W != 0;
                            const int l = has ? 31 - __clz(W) : 0;
                            W ^= has ? 1u << l : 0u;
                            const uint2 cc = binp[l * 33 + (has ? m : 0)];
                            rk[u] = (unsigned int)h - cc.x - SD;
                            SD += has ? cc.y : 0u;
                            ok[u] = has && ((unsigned int)m & (G - 1)) == sub;
                            vv[u] = star_vertex(l, hub);
                            m -= has ? 1 : 0;
                        }
                        double dv[4];
#pragma unroll
                        for (int u = 0; u < 4; u++) dv[u] = ok[u] ? lvl[rk[u]] : 0.0;
#pragma unroll
                        for (int u = 0; u < 4; u++) {
                            // min of (cost, left) in f64 / u32 (costs are >= 0: the
                            // f64 order is the bit order of the Key)
                            const double a = leaf_costs ? __dadd_rn(q.leaf[vv[u]], dv[u]) : dv[u];
                            const double c = __dadd_rn(a, cS);
                            const uint32_t lb = 1u << vv[u], rb = S ^ lb, l = lb < rb ? lb : rb;
                            const bool better = ok[u] && (c < bc || (c == bc && l < bl));
                            bc = better ? c : bc;
                            bl = better ? l : bl;
                        }
                    };
                    for (int bt = kl >> 2; bt > 0; bt--) batch(std::false_type{});
                    if (kl & 3) batch(std::true_type{});
                    best = Key{(unsigned long long)__double_as_longlong(bc), (unsigned long long)bl};
                }
            }
            best = group_min(best, G);
            if (act && sub == 0) {
                const unsigned long long idx = out + h;
                p.memo.dcost[idx] = __longlong_as_double((long long)best.c);
                __stcs(p.memo.dleft + idx, (unsigned int)best.l);
                p.memo.dcard[idx] = cS;
                nsets++;
            }
        }
        if ((p.count_levels >> k) & 1ull) {
            // every written set evaluated its kl join pairs (kl non-singleton
            // probes when k >= 3)
            const unsigned long long pairs = nsets * (unsigned long long)kl, nprobe = k >= 3 ? pairs : 0ull;
            flush_counters(&p.desc[k], pairs, pairs, nprobe, nsets);
        }
        if (one && (solo(k + 1) || k == p.k_end)) __syncthreads();   // CTA 0 continues alone
        else grid_sync(p.gbar, nbar, &p.result->error);
    }
    if (!(p.do_extract && blockIdx.x == 0 && threadIdx.x < 32)) return;
    // ---- counters and plan extraction, warp 0 of CTA 0
    ResultDev* r = p.result;
    const unsigned int lane = threadIdx.x;
    if (lane == 0) r->t_level[n + 1] = globaltimer_ns();
    level_counters_warp(p, r);
    if (ld_relaxed_u32(&r->error)) {
        if (lane == 0) r->n_nodes = 0;
        return;
    }
    // The optimal plan of a star set is a caterpillar: every join splits one
    // leaf v off, ({v}, S \ {v}).  Walk the chain from V (one memo read per
    // step; the colex rank of each set's leaf set is a warp sum of one binomial
    // per element), then emit the post-order nodes from the recorded chain.
    __shared__ uint32_t c_set[32], c_left[32];
    __shared__ double c_cost[32], c_card[32];
    uint32_t S = n == 32 ? ~0u : (1u << n) - 1u;
    int len = 0;
    while (__popc(S) >= 2) {
        const uint32_t L = star_compress(S, hub);
        const int kl = __popc(L);
        unsigned int term = 0;
        if ((int)lane < kl) term = bin[(__fns(L, 0, lane + 1)) * 33 + lane + 1];
        for (int o = 16; o > 0; o >>= 1) term += __shfl_xor_sync(0xffffffffu, term, o);
        const unsigned long long idx = p.star_off[kl + 1] + term;
        uint32_t left = 0;
        if (lane == 0) {
            left = __ldcg(p.memo.dleft + idx);
            c_set[len] = S;
            c_left[len] = left;
            c_cost[len] = __ldcg(p.memo.dcost + idx);
            c_card[len] = __ldcg(p.memo.dcard + idx);
        }
        left = __shfl_sync(0xffffffffu, left, 0);
        const uint32_t right = S ^ left;
        S = (left & (left - 1)) ? left : right;           // the multi-relation side (a singleton at the end)
        len++;
        if ((S & (S - 1)) == 0) break;
    }
    if (lane != 0) return;
    // post-order (left subtree, right subtree, node): with prefix_i = [v_i] when
    // the leaf is the left child and suffix_i = [v_i if it is the right child,
    // S_i], the sequence is prefix_0 .. prefix_{len-2}, the bottom pair (two
    // leaves, then S_{len-1}), suffix_{len-2} .. suffix_0
    auto leaf_node = [&](uint32_t X, int at) {
        const int vtx = __ffs(X) - 1;
        mpdp_plan_node& nd = r->nodes[at];
        nd.left = nd.right = -1;
        nd.relation = vtx;
        nd.reserved = 0;
        nd.set = X;
        nd.cardinality = q.card[vtx];
        nd.cost = q.leaf[vtx];
    };
    auto join_node = [&](int i, int a, int b, int at) {
        mpdp_plan_node& nd = r->nodes[at];
        nd.left = a;
        nd.right = b;
        nd.relation = -1;
        nd.reserved = 0;
        nd.set = c_set[i];
        nd.cardinality = c_card[i];
        nd.cost = c_cost[i];
    };
    int pos_leaf[32];
    int nn = 0;
    for (int i = 0; i + 1 < len; i++)
        if ((c_left[i] & (c_left[i] - 1)) == 0) {     // leaf is the left child
            leaf_node(c_left[i], nn);
            pos_leaf[i] = nn++;
        }
    {
        const int b = len - 1;
        const uint32_t A = c_left[b], B = c_set[b] ^ A;
        leaf_node(A, nn);
        leaf_node(B, nn + 1);
        join_node(b, nn, nn + 1, nn + 2);
        nn += 3;
    }
    int inner = nn - 1;
    for (int i = len - 2; i >= 0; i--) {
        const uint32_t A = c_left[i];
        if ((A & (A - 1)) == 0) {
            join_node(i, pos_leaf[i], inner, nn);
        } else {                                          // leaf is the right child
            leaf_node(c_set[i] ^ A, nn);
            join_node(i, inner, nn, nn + 1);
            nn++;
        }
        inner = nn++;
    }
    r->n_nodes = (unsigned int)nn;
    r->cost = r->nodes[nn - 1].cost;
}

}  // namespace mpdp
