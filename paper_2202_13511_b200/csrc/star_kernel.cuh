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
    const unsigned long long T = (unsigned long long)gridDim.x * blockDim.x;
    const unsigned long long gtid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    for (int k = p.k_begin; k <= p.k_end; k++) {
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
        grid_sync(p.gbar, nbar, &p.result->error);
    }
    if (!(p.do_extract && blockIdx.x == 0 && threadIdx.x == 0)) return;
    // ---- counters and plan extraction
    ResultDev* r = p.result;
    r->t_level[n + 1] = globaltimer_ns();
    // bit 1 of count_levels: this rank counts the n singletons (level 1)
    const unsigned long long n1 = ((p.count_levels >> 1) & 1ull) ? (unsigned long long)n : 0ull;
    unsigned long long csg = n1, ccp = 0, pr = 0, probes = 0;
    r->lvl_csg[0] = r->lvl_ccp[0] = r->lvl_pairs[0] = 0;
    r->lvl_csg[1] = n1;
    r->lvl_ccp[1] = r->lvl_pairs[1] = 0;
    for (int j = 2; j <= n; j++) {
        const LevelDesc& d = p.desc[j];                       // (zero for levels another rank counts)
        r->lvl_csg[j] = d.n_light;
        r->lvl_ccp[j] = d.ccp;
        r->lvl_pairs[j] = d.pairs;
        csg += d.n_light;
        ccp += d.ccp;
        pr += d.pairs;
        probes += d.probes;
    }
    r->csg = csg;
    r->ccp = ccp;
    r->pairs = pr;
    r->probes = probes;
    if (r->error) {
        r->n_nodes = 0;
        return;
    }
    uint32_t st_set[2 * 32], st_L[2 * 32];
    double st_c[2 * 32], st_card[2 * 32];
    int st_state[2 * 32], st_left[2 * 32];
    int sp = 1, nn = 0, last = -1;
    st_set[0] = n == 32 ? ~0u : (1u << n) - 1u;
    st_state[0] = 0;
    while (sp) {
        const int top = sp - 1;
        const uint32_t S = st_set[top];
        if ((S & (S - 1)) == 0) {
            const int vtx = __ffs(S) - 1;
            mpdp_plan_node& nd = r->nodes[nn];
            nd.left = nd.right = -1;
            nd.relation = vtx;
            nd.reserved = 0;
            nd.set = S;
            nd.cardinality = q.card[vtx];
            nd.cost = q.leaf[vtx];
            last = nn++;
            --sp;
            continue;
        }
        if (st_state[top] == 0) {
            const unsigned long long idx = star_slot(p, bin, S);
            st_L[top] = p.memo.dleft[idx];
            st_c[top] = p.memo.dcost[idx];
            st_card[top] = p.memo.dcard[idx];
            st_state[top] = 1;
            st_set[sp] = st_L[top];
            st_state[sp++] = 0;
        } else if (st_state[top] == 1) {
            st_left[top] = last;
            st_state[top] = 2;
            st_set[sp] = S & ~st_L[top];
            st_state[sp++] = 0;
        } else {
            mpdp_plan_node& nd = r->nodes[nn];
            nd.left = st_left[top];
            nd.right = last;
            nd.relation = -1;
            nd.reserved = 0;
            nd.set = S;
            nd.cardinality = st_card[top];
            nd.cost = st_c[top];
            last = nn++;
            --sp;
        }
    }
    r->n_nodes = (unsigned int)nn;
    r->cost = r->nodes[nn - 1].cost;
}

}  // namespace mpdp
