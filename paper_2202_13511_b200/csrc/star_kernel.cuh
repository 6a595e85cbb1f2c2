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
#include "dataflow.cuh"

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

// Sets [lo, hi) of star level k on the CTA's compute threads, G lanes per
// set, runs of RUN consecutive sets per group (one unrank, then Gosper):
// lane-consecutive groups, so a warp's probes of the shared high elements
// coalesce and the CTA's warps share L1 lines.  Counts the join pairs this
// thread evaluated and the sets it wrote.
template <int G, bool XR>
__device__ __forceinline__ void star_chunk(const Params<uint32_t>& p, const SQ<uint32_t>& q, const unsigned int* bin,
                                           const uint2* binp, int k, unsigned int lo, unsigned int hi,
                                           unsigned int RUN, unsigned long long& npairs, unsigned long long& nsets,
                                           const DfRank& x) {
    const int hub = p.star_hub, nl = p.n - 1, kl = k - 1;   // kl leaves per set
    const bool leaf_costs = q.pad != 0;
    const double* lvl = (XR ? x.dcost : p.memo.dcost) + p.star_off[k - 1];   // this rank's replica
    const double* lcard = (XR ? x.dcard : p.memo.dcard) + p.star_off[k - 1];
    const unsigned long long out = p.star_off[k];
    constexpr unsigned int NG = kDfCompute / G;              // groups per CTA
    const unsigned int grp = threadIdx.x / G, sub = threadIdx.x & (G - 1);
    uint32_t L = 0;
    for (unsigned int r0 = lo; r0 < hi; r0 += NG * RUN) {     // uniform trip count
        const unsigned int h0 = r0 + grp * RUN;
        for (unsigned int it = 0; it < RUN; it++) {
            const unsigned int h = h0 + it;
            const bool act = h < hi;
            if (act) L = (it == 0) ? unrank_colex32(bin, nl, kl, h) : gosper(L);
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
                    npairs += sub == 0;
                } else {
                    const int pl = 31 - __clz(L);             // max leaf (leaf space)
                    const int pv = star_vertex(pl, hub);
                    // max(S) is a leaf: card(S) from card(S \ max) (reading
                    // R19); the load is issued here, the product formed after
                    // the first batch of probes is in flight
                    const bool fold = pv > hub && !p.shard_local;
                    const double craw = fold ? __ldcs(lcard + (h - bin[pl * 33 + kl])) : 0.0;
                    bool need_cs = true;
                    // Pair ({v}, S \ {v}) per leaf v, walked from the largest
                    // leaf down.  Tie-break key (reading R7, min(left, right)
                    // as a mask) in leaf space: {v} for every leaf but the
                    // largest vertex of S, whose pair's smaller side is
                    // S \ {v} (key 32, above every singleton); so along the
                    // descending walk a later candidate of equal cost always
                    // has the smaller key, and "<=" is the exact R7 min.
                    double bc = __longlong_as_double(0x7ff0000000000000ll);   // +inf
                    int bl = 64;
                    unsigned int SD = 0;
                    uint32_t W = L;
                    int m = kl - 1;
                    const bool top_rb = pv > hub;             // the largest leaf is max(S)
                    auto batch = [&](auto guard) {
                        constexpr bool GUARD = decltype(guard)::value;
                        unsigned int rk[4];
                        int ll[4];
                        bool ok[4];
#pragma unroll
                        for (int u = 0; u < 4; u++) {
                            const bool has = !GUARD || W != 0;
                            const int l = has ? 31 - __clz(W) : 0;
                            W ^= has ? 1u << l : 0u;
                            const uint2 cc = binp[l * 33 + (has ? m : 0)];
                            rk[u] = h - cc.x - SD;
                            SD += has ? cc.y : 0u;
                            ok[u] = has && (G == 1 || ((unsigned int)m & (G - 1)) == sub);
                            ll[u] = (m == kl - 1 && top_rb) ? 32 : l;
                            m -= has ? 1 : 0;
                        }
                        double dv[4];
#pragma unroll
                        for (int u = 0; u < 4; u++) dv[u] = ok[u] ? lvl[rk[u]] : 0.0;
                        if (need_cs) {
                            cS = fold ? __dmul_rn(__dmul_rn(craw, q.card[pv]), q.sel[hub * q.n + pv]) : card_of(q, S);
                            need_cs = false;
                        }
#pragma unroll
                        for (int u = 0; u < 4; u++) {
                            const double a =
                                leaf_costs ? __dadd_rn(q.leaf[star_vertex(ll[u] == 32 ? pl : ll[u], hub)], dv[u]) : dv[u];
                            const double c = __dadd_rn(a, cS);
                            const bool better = ok[u] && c <= bc;
                            bc = better ? c : bc;
                            bl = better ? ll[u] : bl;
                            npairs += ok[u];
                        }
                    };
                    for (int bt = kl >> 2; bt > 0; bt--) batch(std::false_type{});
                    if (kl & 3) batch(std::true_type{});
                    // the real left mask of the best key (group_min compares
                    // masks across lanes)
                    uint32_t lm = 0xffffffffu;
                    if (bl == 32) lm = S ^ (1u << pv);
                    else if (bl < 32) lm = 1u << star_vertex(bl, hub);
                    best = Key{(unsigned long long)__double_as_longlong(bc), (unsigned long long)lm};
                }
            }
            if (G > 1) best = group_min(best, G);
            if (act && sub == 0) {
                const unsigned long long idx = out + h;
                // the cost into every replica (fused exchange: peer stores;
                // one rank: the local array); left and card stay local
                const double bcost = __longlong_as_double((long long)best.c);
                if constexpr (XR) {
                    for (int s = 0; s < x.W; s++) x.xr->cost[s][idx] = bcost;
                    __stcs(x.dleft + idx, (unsigned int)best.l);
                    x.dcard[idx] = cS;
                } else {
                    p.memo.dcost[idx] = bcost;
                    __stcs(p.memo.dleft + idx, (unsigned int)best.l);
                    p.memo.dcard[idx] = cS;
                }
                nsets++;
            }
        }
    }
}

__device__ __noinline__ void star_extract(const Params<uint32_t>& p, const SQ<uint32_t>& q, const unsigned int* bin,
                                          int hub, const DfRank& x);
__device__ void star_emit_chain(const Params<uint32_t>& p, const SQ<uint32_t>& q, const uint32_t* c_set,
                                const uint32_t* c_left, const double* c_cost, const double* c_card, int len,
                                const DfRank& x);

// Sharded extraction (p.shard_local): the ranks exchanged only the memo costs,
// so every rank re-derives the chain's splits from its complete cost replica:
// at S the warp evaluates the pairs ({v}, S \ {v}) exactly as the level did
// (same C_out order of additions, reading R7's key on the real masks) and
// takes their minimum; card(S) by reading R5's fold.  Lane 0 of warp 0.
__device__ __noinline__ void star_extract_sharded(const Params<uint32_t>& p, const SQ<uint32_t>& q, int hub,
                                                  const DfRank& x) {
    const unsigned int lane = threadIdx.x & 31;
    __shared__ uint32_t x_set[32], x_left[32];
    __shared__ double x_cost[32], x_card[32];
    const int n = p.n;
    const bool leaf_costs = q.pad != 0;
    uint32_t S = n == 32 ? ~0u : (1u << n) - 1u;
    int len = 0;
    while (__popc(S) >= 2) {
        const uint32_t L = star_compress(S, hub);
        const int kl = __popc(L);
        const double cS = card_of(q, S);
        Key best = key_inf();
        for (int j = (int)lane; j < kl; j += 32) {
            const int li = (int)__fns(L, 0, j + 1), v = star_vertex(li, hub);
            const uint32_t lb = 1u << v, rb = S ^ lb;
            double c;
            if (kl == 1) {                                   // ({hub}, {v})
                c = __dadd_rn(__dadd_rn(q.leaf[hub], q.leaf[v]), cS);
            } else {
                // rank of the leaf set L \ {li} among the (kl-1)-subsets
                const uint32_t Lr = L & ~(1u << li);
                unsigned int r = 0;
                int i = 1;
                for (uint32_t T = Lr; T; T &= T - 1, i++) {
                    const int e = __ffs(T) - 1;
                    unsigned long long b = 1;                // C(e, i)
                    for (int t = 0; t < i; t++) b = b * (unsigned long long)(e - t) / (unsigned long long)(t + 1);
                    r += e >= i ? (unsigned int)b : 0u;
                }
                const double dv = __ldcg(x.dcost + p.star_off[kl] + r);
                const double a = leaf_costs ? __dadd_rn(q.leaf[v], dv) : dv;
                c = __dadd_rn(a, cS);
            }
            const uint32_t l = lb < rb ? lb : rb;
            const Key cand{(unsigned long long)__double_as_longlong(c), (unsigned long long)l};
            if (key_less(cand, best)) best = cand;
        }
        best = warp_min(best);
        if (lane == 0) {
            x_set[len] = S;
            x_left[len] = (uint32_t)best.l;
            x_cost[len] = __longlong_as_double((long long)best.c);
            x_card[len] = cS;
        }
        len++;
        const uint32_t left = (uint32_t)best.l, right = S ^ left;
        S = (left & (left - 1)) ? left : right;
        if ((S & (S - 1)) == 0) break;
    }
    __syncwarp();
    if (lane == 0) star_emit_chain(p, q, x_set, x_left, x_cost, x_card, len, x);
}

// Star levels as dataflow chunks (dataflow.cuh): level k's sets are the
// colex ranks of its (k-1)-leaf sets; a chunk needs level k-1 up to the
// largest leaf of its last set.
template <bool XR>
struct StarSched {
    const Params<uint32_t>& p;
    const unsigned int* bin;
    const DfRank& x;
    __device__ unsigned int total() const { return p.dfl[p.k_end + 1].base; }
    __device__ void locate(unsigned int t, DfSlot& d) const {
        int k = p.k_begin;
        while (t >= p.dfl[k + 1].base) k++;
        const DfLevel& L = p.dfl[k];
        d.t = t;
        d.k = k;
        d.k2 = L.solo > k ? L.solo : k;
        d.lo = p.share_lo[k] + (t - L.base) * L.chunk;
        d.hi = min(d.lo + L.chunk, p.share_hi[k]);
    }
    __device__ int need(const DfSlot& d) const {
        return (d.k >= 3 && d.k - 1 >= p.k_begin) ? colex_top(bin, d.k - 1, d.hi - 1) : -1;
    }
    // sets of level k1 (k1 - 1 leaves) whose largest leaf is j
    __device__ unsigned int need_count(int k1, int j) const { return bin[j * 33 + k1 - 2]; }
    __device__ void publish(const DfSlot& d) const {
        DataflowDev* const ldf = XR ? x.df : p.df;
        df_publish_colex<XR>(x, ldf, bin, d.k, d.k - 1, d.lo, d.hi);
        for (int k = d.k + 1; k <= d.k2; k++) df_publish_colex<XR>(x, ldf, bin, k, k - 1, p.share_lo[k], p.share_hi[k]);
    }
};

template <bool XR>
__global__ void __launch_bounds__(kDfThreads, kStarMinBlocks) k_dp_star(const __grid_constant__ Params<uint32_t> p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SQ<uint32_t>& q = *reinterpret_cast<SQ<uint32_t>*>(smem_raw);
    unsigned int* bin = reinterpret_cast<unsigned int*>(smem_raw + sizeof(SQ<uint32_t>));   // 33 x 33
    __shared__ DfCounters sc;
    __shared__ DfShared sh;
    __shared__ DfRank xr;                  // this CTA's rank and replica (fused exchange)
    if (blockIdx.x == 0 && threadIdx.x == 0) p.result->t_level[0] = globaltimer_ns();   // kernel start
    if (threadIdx.x == 0) {
        df_rank_init(xr, p);
        if (XR) df_start_barrier(p, xr);
    }
    load_query(q, p.q);
    constexpr int NB = MaxN<uint32_t>::value + 1;
    for (int i = threadIdx.x; i < 33 * 33; i += blockDim.x) {
        const int a = i / 33, b = i % 33;
        bin[i] = (a < NB && b < NB) ? (unsigned int)p.q->binom[a * NB + b] : 0u;
    }
    for (int i = threadIdx.x; i < (kMaxN + 1) * 3; i += blockDim.x) (&sc.v[0][0])[i] = 0;
    for (int i = threadIdx.x; i <= kMaxN; i += blockDim.x) sh.ready[i] = i < p.k_begin ? 64 : -1;
    if (threadIdx.x < kDfSlots) sh.done[threadIdx.x] = 0;
    // (C(v, m+1), C(v, m+1) - C(v, m)) pairs of the descending walk, 8-byte aligned
    uint2* binp = reinterpret_cast<uint2*>(smem_raw + ((sizeof(SQ<uint32_t>) + sizeof(unsigned int) * 33 * 33 + 7) & ~size_t(7)));
    __syncthreads();
    for (int i = threadIdx.x; i < 33 * 32; i += blockDim.x) {
        const int a = i / 32, b = i % 32;
        binp[a * 33 + b] = make_uint2(bin[a * 33 + b + 1], bin[a * 33 + b + 1] - bin[a * 33 + b]);
    }
    __syncthreads();
    const int hub = p.star_hub;
    if (threadIdx.x >= kDfCompute) {
        df_control<XR>(p, StarSched<XR>{p, bin, xr}, sh, xr);
    } else {
        int kc = p.k_begin;
        unsigned long long npairs = 0, nsets = 0;      // this thread, level kc
        DfSlot d;
        unsigned long long st_take = 0;
        const unsigned long long st0 = p.df_stats ? globaltimer_ns() : 0ull;
        unsigned long long* stp = (p.df_stats && threadIdx.x == 0) ? &st_take : nullptr;
        for (unsigned int i = 0; df_take(sh, i, d, stp); i++) {
            // (a solo chunk runs whole small levels d.k..d.k2 back to back,
            // the compute warps' named barrier 3 between them)
            for (int k = d.k; k <= d.k2; k++) {
                if (k != kc) {
                    df_count(sc, kc, npairs, kc >= 3 ? npairs : 0ull, nsets);
                    npairs = nsets = 0;
                    kc = k;
                }
                if (k > d.k) {
                    asm volatile("bar.sync 3, %0;" ::"r"(kDfCompute) : "memory");
                    if (threadIdx.x == 0) xr.result->t_level[k] = globaltimer_ns();
                }
                const DfLevel& L = p.dfl[k];
                const unsigned int lo = k == d.k ? d.lo : p.share_lo[k], hi = k == d.k ? d.hi : p.share_hi[k];
                switch (L.G) {
                    case 1: star_chunk<1, XR>(p, q, bin, binp, k, lo, hi, L.run, npairs, nsets, xr); break;
                    case 2: star_chunk<2, XR>(p, q, bin, binp, k, lo, hi, L.run, npairs, nsets, xr); break;
                    default: star_chunk<4, XR>(p, q, bin, binp, k, lo, hi, L.run, npairs, nsets, xr); break;
                }
            }
            df_finish(sh, i);
        }
        if (stp) {
            p.df_stats[8ull * blockIdx.x + 4] = st_take;
            p.df_stats[8ull * blockIdx.x + 5] = globaltimer_ns() - st0;
        }
        // every pair of a set of level >= 3 probes one memo entry (S \ {v}, >= 2 relations)
        df_count(sc, kc, npairs, kc >= 3 ? npairs : 0ull, nsets);
    }
    if (!df_exit<XR>(p, sc, xr)) return;
    if (p.do_extract && threadIdx.x < 32) star_extract(p, q, bin, hub, xr);
    df_reset(p, xr);
}

// Counters and plan extraction, warp 0 of the last CTA out.
__device__ __noinline__ void star_extract(const Params<uint32_t>& p, const SQ<uint32_t>& q, const unsigned int* bin,
                                          int hub, const DfRank& x) {
    const int n = p.n;
    ResultDev* r = x.result;
    const unsigned int lane = threadIdx.x;             // warp 0
    if (lane == 0) r->t_level[n + 1] = globaltimer_ns();
    level_counters_warp(p, r, x.desc);
    if (ld_relaxed_u32(&x.df->error)) {
        if (lane == 0) r->n_nodes = 0;
        return;
    }
    if (p.shard_local) {
        star_extract_sharded(p, q, hub, x);
        return;
    }
    // The optimal plan of a star set is a caterpillar: every join splits one
    // leaf v off, ({v}, S \ {v}).  Walk the chain from V two steps per memo
    // round trip: while lane 31 reads the entry of S, lane j reads the entry of
    // S \ {leaf j} (the colex rank of its leaf set from two warp scans of the
    // binomial terms), so once left(S) names v the entry of the next set is
    // already in the registers of v's lane.  The recorded chain is then
    // emitted as post-order nodes.
    __shared__ uint32_t c_set[32], c_left[32];
    __shared__ double c_cost[32], c_card[32];
    uint32_t S = n == 32 ? ~0u : (1u << n) - 1u;
    int len = 0;
    while (__popc(S) >= 2) {
        const uint32_t L = star_compress(S, hub);
        const int kl = __popc(L);
        const bool mine = (int)lane < kl;
        const int lj = mine ? (int)__fns(L, 0, lane + 1) : 0;            // leaf j (leaf space)
        const unsigned int a = mine ? bin[lj * 33 + lane + 1] : 0u;      // C(l_j, j+1): term of rank(L)
        const unsigned int b = mine ? bin[lj * 33 + lane] : 0u;          // C(l_j, j): term once l_j moves down
        unsigned int ia = a, ib = b;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned int x = __shfl_up_sync(0xffffffffu, ia, o), y = __shfl_up_sync(0xffffffffu, ib, o);
            if ((int)lane >= o) {
                ia += x;
                ib += y;
            }
        }
        const unsigned int ra = __shfl_sync(0xffffffffu, ia, 31), rb = __shfl_sync(0xffffffffu, ib, 31);
        // S itself (lane 31), S \ {leaf j} (lane j < kl, when it keeps >= 2 relations)
        unsigned long long idx = 0;
        bool load = false;
        if (lane == 31) {
            idx = p.star_off[kl + 1] + ra;
            load = true;
        } else if (mine && kl >= 2) {
            idx = p.star_off[kl] + (ia - a) + (rb - ib);
            load = true;
        }
        uint32_t e_left = 0;
        double e_cost = 0.0, e_card = 0.0;
        if (load) {
            e_left = __ldcg(x.dleft + idx);
            e_cost = __ldcg(x.dcost + idx);
            e_card = __ldcg(x.dcard + idx);
        }
        const uint32_t left = __shfl_sync(0xffffffffu, e_left, 31);
        const double cS = __shfl_sync(0xffffffffu, e_cost, 31), kS = __shfl_sync(0xffffffffu, e_card, 31);
        if (lane == 0) {
            c_set[len] = S;
            c_left[len] = left;
            c_cost[len] = cS;
            c_card[len] = kS;
        }
        len++;
        const uint32_t right = S ^ left;
        const uint32_t S1 = (left & (left - 1)) ? left : right;     // the multi-relation side
        if ((S1 & (S1 - 1)) == 0) break;                            // S was a pair: chain complete
        // S1 = S \ {v}: its entry sits in the lane of leaf v
        const uint32_t vm = star_compress(S ^ S1, hub);              // {v} in leaf space
        const int src = __popc(L & (vm - 1u));
        const uint32_t l1 = __shfl_sync(0xffffffffu, e_left, src);
        const double c1 = __shfl_sync(0xffffffffu, e_cost, src), k1 = __shfl_sync(0xffffffffu, e_card, src);
        if (lane == 0) {
            c_set[len] = S1;
            c_left[len] = l1;
            c_cost[len] = c1;
            c_card[len] = k1;
        }
        len++;
        const uint32_t r1 = S1 ^ l1;
        S = (l1 & (l1 - 1)) ? l1 : r1;
        if ((S & (S - 1)) == 0) break;
    }
    __syncwarp();
    if (lane == 0) star_emit_chain(p, q, c_set, c_left, c_cost, c_card, len, x);
}


// Post-order plan nodes of a recorded caterpillar chain (one thread).
__device__ void star_emit_chain(const Params<uint32_t>& p, const SQ<uint32_t>& q, const uint32_t* c_set,
                                const uint32_t* c_left, const double* c_cost, const double* c_card, int len,
                                const DfRank& x) {
    ResultDev* r = x.result;
    const int n = p.n;
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
    atomicMax(&x.df->t_done[n + 1], globaltimer_ns());     // extraction end
    r->cost = r->nodes[nn - 1].cost;
}

}  // namespace mpdp
