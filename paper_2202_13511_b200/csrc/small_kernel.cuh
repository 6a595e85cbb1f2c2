// small_kernel.cuh — the whole level loop of Alg. mpdp_gpu for a
// SMALL query on ONE CTA, with the memo in shared memory.
//
// For n <= kSmallMaxN the memo indexed by relation bitmask fits in shared
// memory: cost[2^n] (f64), card[2^n] (f64), left[2^n] (u16) = 18 B x 8192 =
// 144 KB at n = 13.  Every step of the path then stays on one SM:
//   * connectivity filter + stream compaction of EVERY level up front
//     (the enumeration reads no memo): the 2^n masks are
//     filtered in bitmask order, counted per size, and written into per-size
//     segments of a shared-memory list (two passes, 32-bit shared atomics);
//   * per level, evaluate: G lanes per set (about 8 pairs per
//     lane, more lanes when the level is small), each lane a contiguous range of the set's csg-cmp
//     pairs through the same enumeration as the multi-CTA kernels
//     (eval_range: trees, complete blocks, Find-Blocks), C_out cost from the
//     shared-memory memo, group shuffle min of (cost, left), one memo write;
//   * __syncthreads() is the level barrier; the plan is extracted from shared
//     memory by one thread.
// The multi-CTA kernels pay a grid barrier and global-memory round trips per
// level (~5-10 us); here a level of star-10 costs about a microsecond.  Used for
// the configs' small queries (star-10) and for IDP2 / UnionDP inner DPs.
#pragma once
#include "fused.cuh"

namespace mpdp {

constexpr int kSmallMaxN = 13;
constexpr int kSmallBlock = 512;

__host__ __device__ constexpr size_t small_smem_bytes(int n) {
    return sizeof(SQ<uint32_t>) + (size_t(1) << n) * (8 + 8 + 2 + 2) + 64;   // cost, card, left, list
}

struct SmallSink {
    static constexpr bool kChk = false;    // CCP tests by BFS (reading R20 is MEMO_MASK only)
    const double* cost;
    double cS;
    Key best;
    unsigned long long nprobe;
    __device__ __forceinline__ void add(uint32_t a, uint32_t b) {
        const double c = __dadd_rn(__dadd_rn(cost[a], cost[b]), cS);
        nprobe += (unsigned long long)((a & (a - 1)) != 0) + (unsigned long long)((b & (b - 1)) != 0);
        const Key key{(unsigned long long)__double_as_longlong(c), (unsigned long long)(a < b ? a : b)};
        if (key_less(key, best)) best = key;
    }
};

// Per-warp partial sums of three counters (64-bit shared-memory atomics are
// CAS spin loops on sm_100 -- ATOMS.CAST.SPIN.64 -- and 16-32 warps hitting one
// address cost microseconds per level); block_sum3_final reduces them in warp 0
// after a barrier, lane 0 gets the totals.
__device__ __forceinline__ void block_sum3_part(unsigned long long a, unsigned long long b, unsigned long long c,
                                                unsigned long long (*part)[32]) {
    a = warp_sum(a);
    b = warp_sum(b);
    c = warp_sum(c);
    if ((threadIdx.x & 31) == 0) {
        part[0][threadIdx.x >> 5] = a;
        part[1][threadIdx.x >> 5] = b;
        part[2][threadIdx.x >> 5] = c;
    }
}
__device__ __forceinline__ void block_sum3_final(unsigned long long (*part)[32], unsigned long long* out) {
    const unsigned int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
#pragma unroll
    for (int i = 0; i < 3; i++) {
        const unsigned long long x = warp_sum(lane < nw ? part[i][lane] : 0ull);
        if (lane == 0) out[i] = x;
    }
}

// card(S) as card_fast (reading R5 / R19), from the shared-memory card array
template <int CLS>
__device__ __forceinline__ double small_card(const SQ<uint32_t>& q, const double* card, uint32_t S, int k) {
    const int p = 31 - __clz(S);
    const uint32_t b = 1u << p;
    const bool in_memo = k >= 3 && ((CLS == CLS_TREE && (S & q.desc[p]) == b) || CLS == CLS_CLIQUE);
    if (!in_memo) return card_of(q, S);
    double x = __dmul_rn(card[S ^ b], q.card[p]);
    for (uint32_t W = S & q.adj[p] & (b - 1u); W; W &= W - 1) x = __dmul_rn(x, q.sel[(__ffs(W) - 1) * q.n + p]);
    return x;
}

// inclusive block scan of one u32 per thread; also returns the block total and
// a block max of `mx`
__device__ __forceinline__ unsigned int block_scan_max(unsigned int x, unsigned long long mx, unsigned int& total,
                                                       unsigned long long& bmax, unsigned int* s_sum,
                                                       unsigned long long* s_max) {
    const unsigned int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    unsigned int inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= (unsigned int)o) inc += t;
        const unsigned long long m = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = m > mx ? m : mx;
    }
    if (lane == 31) s_sum[wid] = inc;
    if (lane == 0) s_max[wid] = mx;
    __syncthreads();
    if (wid == 0) {
        unsigned int y = lane < nw ? s_sum[lane] : 0u, z = y;
        unsigned long long m = lane < nw ? s_max[lane] : 0ull;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned int t = __shfl_up_sync(0xffffffffu, z, o);
            if (lane >= (unsigned int)o) z += t;
            const unsigned long long mm = __shfl_xor_sync(0xffffffffu, m, o);
            m = mm > m ? mm : m;
        }
        if (lane < nw) s_sum[lane] = z - y;          // exclusive warp offsets
        if (lane == 31) {
            s_sum[32] = z;
            s_max[32] = m;
        }
    }
    __syncthreads();
    total = s_sum[32];
    bmax = s_max[32];
    const unsigned int r = s_sum[wid] + inc;
    __syncthreads();                                 // s_sum / s_max reused by the next call
    return r;
}

template <int CLS>
__device__ __forceinline__ void small_body(const QueryDev<uint32_t>* qd, ResultDev* r) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SQ<uint32_t>& q = *reinterpret_cast<SQ<uint32_t>*>(smem_raw);
    load_query(q, qd);
    const int n = qd->n;
    const unsigned int NS = 1u << n;
    double* cost = reinterpret_cast<double*>(smem_raw + sizeof(SQ<uint32_t>));
    double* card = cost + NS;
    unsigned short* left = reinterpret_cast<unsigned short*>(card + NS);
    unsigned short* list = left + NS;                        // connected sets (<= 2^n), grouped by size
    __shared__ unsigned int s_len[kSmallMaxN + 2];           // sets per level, then level offsets
    __shared__ unsigned int s_fill[kSmallMaxN + 2];
    __shared__ unsigned int s_lvl[kSmallMaxN + 1][3];        // ccp, pairs, probes per level (u32: n <= 13)
    if (threadIdx.x <= kSmallMaxN + 1) s_len[threadIdx.x] = s_fill[threadIdx.x] = 0;
    if (threadIdx.x < (kSmallMaxN + 1) * 3) (&s_lvl[0][0])[threadIdx.x] = 0;
    if (threadIdx.x == 0) {
        r->error = 0;
        r->t_level[2] = globaltimer_ns();
    }
    __syncthreads();
    if (CLS == CLS_GENERAL) {              // reading R20 on the shared-memory memo: every slot
        for (unsigned int S = threadIdx.x; S < NS; S += blockDim.x)   // starts absent
            cost[S] = __longlong_as_double((long long)kMemoAbsent);
        if (threadIdx.x == 0) q.mc = cost;
        __syncthreads();
    }
    for (int v = threadIdx.x; v < n; v += blockDim.x) {      // level 1
        cost[1u << v] = q.leaf[v];
        card[1u << v] = q.card[v];
    }
    // ---- unrank + connectivity filter + compaction of EVERY level at once
    // (enumeration reads no memo): the masks are walked in
    // bitmask order, counted per size, then written into per-size segments
    // (list order inside a level is irrelevant: the memo is indexed by mask)
    const unsigned int per = (NS + blockDim.x - 1) / blockDim.x;
    const unsigned int m0 = threadIdx.x * per, m1 = m0 + per < NS ? m0 + per : NS;
    for (unsigned int S = m0 > 3u ? m0 : 3u; S < m1; S++)
        if ((S & (S - 1)) && connected_cls<uint32_t, CLS>(q, S, __popc(S))) atomicAdd(&s_len[__popc(S)], 1u);
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int acc = 0;
        for (int k = 2; k <= n; k++) {
            const unsigned int c = s_len[k];
            s_len[k] = acc;                                  // exclusive offsets
            acc += c;
        }
        s_len[n + 1] = acc;
    }
    __syncthreads();
    for (unsigned int S = m0 > 3u ? m0 : 3u; S < m1; S++)
        if ((S & (S - 1)) && connected_cls<uint32_t, CLS>(q, S, __popc(S))) {
            const int k = __popc(S);
            list[s_len[k] + atomicAdd(&s_fill[k], 1u)] = (unsigned short)S;
        }
    __syncthreads();
    // ---- levels: evaluate (G lanes per set, about 8 pairs per lane), barrier
    for (int k = 2; k <= n; k++) {
        const unsigned int L0 = s_len[k], N = s_len[k + 1] - L0;
        const unsigned long long maxw = CLS == CLS_TREE ? (unsigned long long)(k - 1) : (1ull << (k - 1)) - 1;
        unsigned int G = 1;
        while (G < 32 && (8ull * G < maxw || G * N * 2 <= blockDim.x)) G <<= 1;
        const unsigned int ngroups = blockDim.x / G, grp = threadIdx.x / G, sub = threadIdx.x & (G - 1);
        const unsigned int rounds = (N + ngroups - 1) / ngroups;
        unsigned long long pairs = 0, nccp = 0, nprobe = 0;
        for (unsigned int it = 0; it < rounds; it++) {
            const unsigned int e = it * ngroups + grp;
            const bool act = e < N;
            SmallSink sink{cost, 0.0, key_inf(), 0};
            uint32_t S = 0;
            unsigned long long w = 0;
            if (act) {
                S = list[L0 + e];
                const int kind = set_kind<uint32_t, CLS>(q, S, k, w);
                sink.cS = small_card<CLS>(q, card, S, k);
                const unsigned long long pl = (w + G - 1) / G;
                unsigned long long j0 = pl * sub, j1 = j0 + pl;
                if (j0 > w) j0 = w;
                if (j1 > w) j1 = w;
                eval_range<uint32_t, CLS>(q, S, k, kind, j0, j1, sink, nccp);
                nprobe += sink.nprobe;
            }
            const Key best = group_min(sink.best, G);
            if (act && sub == 0) {
                cost[S] = __longlong_as_double((long long)best.c);
                left[S] = (unsigned short)best.l;
                card[S] = sink.cS;
                pairs += w;
            }
        }
        nccp = warp_sum(nccp);
        pairs = warp_sum(pairs);
        nprobe = warp_sum(nprobe);
        if ((threadIdx.x & 31) == 0) {                       // 32-bit shared atomics are native
            if (nccp) atomicAdd(&s_lvl[k][0], (unsigned int)nccp);
            if (pairs) atomicAdd(&s_lvl[k][1], (unsigned int)pairs);
            if (nprobe) atomicAdd(&s_lvl[k][2], (unsigned int)nprobe);
        }
        __syncthreads();                                     // level barrier: level k is final
        if (threadIdx.x == 0) r->t_level[k + 1] = globaltimer_ns();
    }
    if (threadIdx.x != 0) return;
    unsigned long long tot[4] = {(unsigned long long)n, 0, 0, 0};
    r->lvl_csg[0] = r->lvl_ccp[0] = r->lvl_pairs[0] = 0;
    r->lvl_csg[1] = (unsigned long long)n;
    r->lvl_ccp[1] = r->lvl_pairs[1] = 0;
    for (int k = 2; k <= n; k++) {
        r->lvl_csg[k] = s_len[k + 1] - s_len[k];
        r->lvl_ccp[k] = s_lvl[k][0];
        r->lvl_pairs[k] = s_lvl[k][1];
        tot[0] += s_len[k + 1] - s_len[k];
        tot[1] += s_lvl[k][0];
        tot[2] += s_lvl[k][1];
        tot[3] += s_lvl[k][2];
    }
    r->csg = tot[0];
    r->ccp = tot[1];
    r->pairs = tot[2];
    r->probes = tot[3];
    // ---- plan extraction (post-order, root last) from shared memory
    uint32_t st_set[2 * kSmallMaxN];
    int st_state[2 * kSmallMaxN], st_left[2 * kSmallMaxN];
    int sp = 1, nn = 0, last = -1;
    st_set[0] = NS - 1u;
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
            st_state[top] = 1;
            st_set[sp] = left[S];
            st_state[sp++] = 0;
        } else if (st_state[top] == 1) {
            st_left[top] = last;
            st_state[top] = 2;
            st_set[sp] = S & ~(uint32_t)left[S];
            st_state[sp++] = 0;
        } else {
            mpdp_plan_node& nd = r->nodes[nn];
            nd.left = st_left[top];
            nd.right = last;
            nd.relation = -1;
            nd.reserved = 0;
            nd.set = S;
            nd.cardinality = card[S];
            nd.cost = cost[S];
            last = nn++;
            --sp;
        }
    }
    r->n_nodes = (unsigned int)nn;
    r->cost = r->nodes[nn - 1].cost;
}

template <int CLS>
__global__ void __launch_bounds__(kSmallBlock, 1) k_dp_small(const __grid_constant__ Params<uint32_t> p) {
    small_body<CLS>(p.q, p.result);
}

// Batched small queries (mpdp_optimize_batch): CTA b solves query b -- the
// independent sub-problems of a heuristic level (UnionDP partitions) or any
// set of small tree queries run side by side, one SM each.
template <int CLS>
__global__ void __launch_bounds__(kSmallBlock, 1) k_dp_small_batch(const QueryDev<uint32_t>* __restrict__ qs,
                                                                   ResultDev* __restrict__ rs) {
    small_body<CLS>(qs + blockIdx.x, rs + blockIdx.x);
}

// ------------------------------------------------------------ k_dp_tree1
// Sparse tree queries (snowflakes, chains) whose levels hold a few thousand
// connected sets: ONE CTA, level lists in shared memory, the colex-rank memo in
// global memory (L2-resident).  Level 2 is the edge list; level k+1 is
// generated from level k's sets during their evaluation (fused generation of
// the list kernel: S' = S u {v} is emitted once, from S' minus
// its largest leaf), so no C(n,k) rank space is ever scanned.  The level barrier
// is __syncthreads instead of a grid barrier over ~300 CTAs, which is what the
// multi-CTA list kernel pays per level on these queries (9-13 us of which the
// set evaluations are ~1 us).  The host picks this kernel from the exact
// per-level csg counts of the tree (a subtree-counting DP) for queries whose
// levels hold at most kTree1MaxLevel sets (chains, thin snowflakes); with a few
// thousand sets per level one SM becomes instruction-bound and the multi-CTA
// list kernel is faster.
constexpr int kTree1Block = 1024;
constexpr int kTree1ListCap = 6144;
constexpr int kTree1MaxLevel = 512;        // eligibility: largest level (sets) routed to this kernel

__host__ __device__ constexpr size_t tree1_smem_bytes(unsigned int rank_entries) {
    return sizeof(SQ<uint32_t>) + sizeof(unsigned int) * (rank_entries + 33 * 33 + 1) +
           2ull * kTree1ListCap * sizeof(unsigned long long) + 16;
}

__global__ void __launch_bounds__(kTree1Block, 1) k_dp_tree1(const __grid_constant__ Params<uint32_t> p) {
    constexpr int MEMO = MEMO_DENSE;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SQ<uint32_t>& q = *reinterpret_cast<SQ<uint32_t>*>(smem_raw);
    unsigned int* rtab = reinterpret_cast<unsigned int*>(smem_raw + sizeof(SQ<uint32_t>));
    unsigned int* bin = rtab + p.memo.rg.entries;
    unsigned long long* lists =
        reinterpret_cast<unsigned long long*>(smem_raw + ((sizeof(SQ<uint32_t>) + sizeof(unsigned int) *
                                                           (p.memo.rg.entries + 33 * 33) + 15) & ~size_t(15)));
    __shared__ MemoView v;
    __shared__ unsigned int s_cnt[2];
    __shared__ unsigned long long s_part[3][32];         // per-warp ccp, pairs, probes of the level
    __shared__ unsigned long long s_lvl[3];
    memo_prologue<uint32_t, MEMO>(p, p.n, q, v, rtab);
    const int n = p.n;
    const unsigned int gen = p.q->gen;
    ResultDev* r = p.result;
    if (threadIdx.x == 0) {
        s_cnt[0] = 0;
        s_cnt[1] = 0;
        r->error = 0;
        r->t_level[2] = globaltimer_ns();
    }
    __syncthreads();
    // level 2: the edges {u, v}, u < v, colex rank u + C(v, 2)
    for (int a = threadIdx.x; a < n; a += blockDim.x)
        for (uint32_t U = q.adj[a] & ((1u << a) - 1u); U; U &= U - 1) {
            const int u = __ffs(U) - 1;
            const unsigned int d = atomicAdd(&s_cnt[0], 1u);
            const unsigned int R = (unsigned int)u + bin[a * 33 + 2];
            if (d < kTree1ListCap) lists[d] = ((unsigned long long)R << 32) | ((1u << u) | (1u << a));
        }
    __syncthreads();
    for (int k = 2; k <= n; k++) {
        const unsigned long long* cur = lists + (size_t)(k & 1) * kTree1ListCap;
        unsigned long long* nxt = lists + (size_t)((k + 1) & 1) * kTree1ListCap;
        const unsigned int N = s_cnt[k & 1] < kTree1ListCap ? s_cnt[k & 1] : kTree1ListCap;
        if (s_cnt[k & 1] > kTree1ListCap && threadIdx.x == 0) atomicOr(&r->error, ERR_CAPACITY);
        unsigned long long pairs = 0, nccp = 0, nprobe = 0;
        // G lanes per set when the level has fewer sets than threads: each
        // lane takes ceil((k-1)/G) of the set's join pairs, so a set costs one
        // round of probes instead of k/4 dependent rounds
        unsigned int G = 1;
        while (G < 32 && 2u * G * N <= blockDim.x) G <<= 1;
        const unsigned int sub = threadIdx.x & (G - 1), ngrp = blockDim.x / G;
        const unsigned int rounds = (N + ngrp - 1) / ngrp;
        for (unsigned int it = 0; it < rounds; it++) {
            const unsigned int e = it * ngrp + threadIdx.x / G;
            const bool act = e < N;
            const unsigned long long ent = act ? cur[e] : 0ull;
            const uint32_t S = (uint32_t)ent;
            const unsigned int R = (unsigned int)(ent >> 32);
            TreeSetInfo info;
            bool lead = act;
            if (G == 1) {
                if (act && k > 2) {
                    eval_tree_dense<MEMO, false, true>(p.memo, gen, v, rtab, bin, q, S, k, R, nprobe, nullptr, &info);
                } else if (act) {                        // both sides are leaves
                    PairSink<uint32_t, MEMO> sink;
                    sink.init(&p.memo, gen, &v, rtab, &q, card_of(q, S));
                    const uint32_t lo = S & (0u - S);
                    sink.add(lo, S ^ lo);
                    sink.flush();
                    const unsigned long long idx = v.off[2] + R;
                    p.memo.dcost[idx] = __longlong_as_double((long long)sink.best.c);
                    __stcs(p.memo.dleft + idx, (unsigned int)sink.best.l);
                    p.memo.dcard[idx] = sink.cS;
                }
            } else {
                Key best = key_inf();
                double cS = 0.0;
                if (act) {
                    unsigned long long w;
                    const int kind = set_kind<uint32_t, CLS_TREE>(q, S, k, w);
                    cS = card_fast<CLS_TREE, MEMO>(p.memo, v, bin, q, S, k, R);
                    PairSink<uint32_t, MEMO> sink;
                    sink.init(&p.memo, gen, &v, rtab, &q, cS);
                    const unsigned long long per = (w + G - 1) / G;
                    unsigned long long j0 = per * sub, j1 = j0 + per;
                    if (j0 > w) j0 = w;
                    if (j1 > w) j1 = w;
                    unsigned long long dummy = 0;
                    eval_range<uint32_t, CLS_TREE>(q, S, k, kind, j0, j1, sink, dummy);
                    sink.flush();
                    nprobe += sink.nprobe;
                    best = sink.best;
                }
                best = group_min(best, G);
                lead = act && sub == 0;
                if (lead) {
                    const unsigned long long idx = v.off[k] + R;
                    p.memo.dcost[idx] = __longlong_as_double((long long)best.c);
                    __stcs(p.memo.dleft + idx, (unsigned int)best.l);
                    p.memo.dcard[idx] = cS;
                }
            }
            if (lead && (G > 1 || k == 2)) {             // leaves and neighbourhood of S
                uint32_t L = 0, nb = 0;
                for (uint32_t T = S; T; T &= T - 1) {
                    const uint32_t a = q.adj[__ffs(T) - 1];
                    nb |= a;
                    if (__popc(a & S) == 1) L |= T & (0u - T);
                }
                info.leaves = L;
                info.nb = nb;
            }
            if (lead) {
                pairs += (unsigned long long)(k - 1);
                nccp += (unsigned long long)(k - 1);
            }
            if (lead && k < n) {                         // children S u {v}, each generated once
                const uint32_t acc = children_of(q, S, info);
                if (acc) {
                    unsigned int d = atomicAdd(&s_cnt[(k + 1) & 1], (unsigned int)__popc(acc));
                    const int mx = 31 - __clz(S);
                    for (uint32_t V = acc; V; V &= V - 1, d++) {
                        const int w = __ffs(V) - 1;
                        const uint32_t Sp = S | (1u << w);
                        unsigned int Rp;
                        if (w > mx) {
                            Rp = R + bin[w * 33 + k + 1];
                        } else {
                            Rp = 0;
                            int i = 1;
                            for (uint32_t T = Sp; T; T &= T - 1, i++) Rp += bin[(__ffs(T) - 1) * 33 + i];
                        }
                        if (d < kTree1ListCap) nxt[d] = ((unsigned long long)Rp << 32) | Sp;
                    }
                }
            }
        }
        block_sum3_part(nccp, pairs, nprobe, s_part);
        __syncthreads();                                 // level k is final in the memo
        if (threadIdx.x < 32) block_sum3_final(s_part, s_lvl);
        if (threadIdx.x == 0) {
            LevelDesc& d = p.desc[k];
            d.n_light = N;
            d.n_heavy = 0;
            d.ccp = s_lvl[0];
            d.pairs = s_lvl[1];
            d.probes = s_lvl[2];
            s_cnt[k & 1] = 0;                            // becomes level k+2's counter
            r->t_level[k + 1] = globaltimer_ns();
        }
        __syncthreads();
    }
    if (p.do_extract && threadIdx.x < 32) {
        level_counters_warp(p, p.result);
        if (threadIdx.x == 0) extract_phase<uint32_t, MEMO>(p, q, v, rtab, gen);
    }
}

}  // namespace mpdp
