// batch128.cuh — independent tree sub-problems (UnionDP's partitions of one
// recursion level) solved together by ONE launch: CTA b runs the
// whole level loop of Alg. mpdp_gpu for sub-problem b, and all
// sub-problems share ONE open-addressing memo in HBM keyed by the 128-bit
// composite key {sub-problem, relation bitmask} (north_star: "128-bit for
// composite IDP/UnionDP subproblems"; "batched into one table
// with 128-bit keys (sub-problem id u64, local mask u64)").
//
// Per CTA (1024 threads):
//   * level lists in shared memory: level 2 = the edges of the tree, level k+1
//     generated from level k's sets while they are evaluated (S' = S u {v}
//     emitted once, from S' minus its largest leaf: children_of),
//     so no C(n, k) rank space is scanned and the list sizes are the tree's
//     csg counts (checked against the host's subtree count);
//   * a tree set S of k relations has the k-1 join pairs (S n desc(v), rest)
//     over the non-top vertices v of S (Alg. mpdp_trees; Lemma 8:
//     all of them are CCP pairs); G lanes per set split them on small levels;
//   * C_out: (cost(A) + cost(B)) + card(S), card by reading R5's fold,
//     singletons from the query (leaf cost / cardinality), the rest from the
//     shared memo; the lexicographic min over (cost, min(A, B)) (reading R7);
//   * plan extraction by thread 0 from the memo.
// The memo is never cleared: the high key word carries a per-batch epoch, and
// a slot of another epoch counts as free when inserting and ends a probe when
// looking up (every key of a batch is inserted once, by its own CTA, before
// any lookup of it, so probe chains of the current batch hold no stale slot).
#pragma once
#include "small_kernel.cuh"

namespace mpdp {

constexpr int kBatchBlock = 1024;
constexpr int kBatchListCap = 6144;       // sets per level list (shared memory)
constexpr int kBatchMaxN = 32;

struct __align__(16) Key128 {
    unsigned long long hi;                 // epoch << 32 | (sub-problem + 1); 0 = never used
    unsigned long long lo;                 // relation bitmask of the set
};
struct Val128 {
    double cost, card;
    unsigned long long left;
};
struct Memo128 {
    Key128* keys;
    Val128* vals;
    unsigned long long mask;               // capacity - 1 (power of two)
    unsigned int epoch;
};

__device__ __forceinline__ unsigned long long memo128_hash(unsigned long long hi, unsigned long long lo) {
    return fmix((uint64_t)(lo * 0x9e3779b97f4a7c15ull ^ fmix((uint64_t)hi)));
}

__device__ __forceinline__ Key128 ld_key128(const Key128* k) {
    Key128 r;
    asm volatile("ld.global.cg.v2.u64 {%0, %1}, [%2];" : "=l"(r.hi), "=l"(r.lo) : "l"(k));
    return r;
}

// insert a key of this batch (never present yet); claims the first slot that
// is empty or of an older epoch with one 128-bit CAS
__device__ bool memo128_insert(const Memo128& m, unsigned long long hi, unsigned long long lo, const Val128& val) {
    unsigned long long h = memo128_hash(hi, lo) & m.mask;
    for (unsigned long long probe = 0; probe <= m.mask; probe++, h = (h + 1) & m.mask) {
        Key128 cur = ld_key128(&m.keys[h]);
        while ((cur.hi >> 32) != m.epoch || cur.hi == 0) {   // free for this batch
            unsigned long long olo, ohi;
            cas128(reinterpret_cast<unsigned long long*>(&m.keys[h]), cur.hi, cur.lo, hi, lo, ohi, olo);
            if (ohi == cur.hi && olo == cur.lo) {
                m.vals[h] = val;
                return true;
            }
            cur.hi = ohi;
            cur.lo = olo;
        }
    }
    return false;                          // table full (the host sizes it at load factor <= 0.5)
}

// look a key of this batch up (inserted earlier by this CTA, before a
// __syncthreads): slot index, or -1 if absent
__device__ __forceinline__ long long memo128_find(const Memo128& m, unsigned long long hi, unsigned long long lo) {
    unsigned long long h = memo128_hash(hi, lo) & m.mask;
    for (unsigned long long probe = 0; probe <= m.mask; probe++, h = (h + 1) & m.mask) {
        const Key128 cur = ld_key128(&m.keys[h]);
        if (cur.hi == hi && cur.lo == lo) return (long long)h;
        if (cur.hi == 0 || (cur.hi >> 32) != m.epoch) return -1;
    }
    return -1;
}

__host__ __device__ constexpr size_t batch128_smem_bytes() {
    return sizeof(SQ<uint32_t>) + sizeof(unsigned int) * 33 * 33 + 2ull * kBatchListCap * sizeof(uint32_t) + 16;
}

__global__ void __launch_bounds__(kBatchBlock, 1) k_dp_tree_batch(const QueryDev<uint32_t>* __restrict__ qs,
                                                                  ResultDev* __restrict__ rs, Memo128 m,
                                                                  const unsigned int* __restrict__ sub_ids) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SQ<uint32_t>& q = *reinterpret_cast<SQ<uint32_t>*>(smem_raw);
    unsigned int* bin = reinterpret_cast<unsigned int*>(smem_raw + sizeof(SQ<uint32_t>));
    uint32_t* lists = reinterpret_cast<uint32_t*>(smem_raw + ((sizeof(SQ<uint32_t>) + sizeof(unsigned int) * 33 * 33 +
                                                               15) & ~size_t(15)));
    __shared__ unsigned int s_cnt[2];
    __shared__ unsigned long long s_part[3][32];
    __shared__ unsigned long long s_lvl[3];
    const QueryDev<uint32_t>* qd = qs + blockIdx.x;
    ResultDev* r = rs + blockIdx.x;
    load_query(q, qd);
    constexpr int NB = MaxN<uint32_t>::value + 1;
    for (int i = threadIdx.x; i < 33 * 33; i += blockDim.x) {
        const int a = i / 33, b = i % 33;
        bin[i] = (a < NB && b < NB) ? (unsigned int)qd->binom[a * NB + b] : 0u;
    }
    const unsigned long long hi = ((unsigned long long)m.epoch << 32) | (unsigned long long)(sub_ids[blockIdx.x] + 1);
    if (threadIdx.x == 0) {
        s_cnt[0] = 0;
        s_cnt[1] = 0;
        r->error = 0;
        r->probes = 0;
        r->t_level[2] = globaltimer_ns();
    }
    __syncthreads();
    const int n = q.n;
    // level 2: the edges {u, a}, u < a
    for (int a = threadIdx.x; a < n; a += blockDim.x)
        for (uint32_t U = q.adj[a] & ((1u << a) - 1u); U; U &= U - 1) {
            const unsigned int d = atomicAdd(&s_cnt[0], 1u);
            if (d < kBatchListCap) lists[d] = (1u << (__ffs(U) - 1)) | (1u << a);
        }
    __syncthreads();
    // cost of a side of a split: a leaf from the query, else the memo
    auto side_cost = [&](uint32_t X) -> double {
        if ((X & (X - 1)) == 0) return q.leaf[__ffs(X) - 1];
        const long long at = memo128_find(m, hi, X);
        if (at < 0) {
            atomicOr(&r->error, ERR_PROBE);
            return 0.0;
        }
        return __ldcg(&m.vals[at].cost);
    };
    for (int k = 2; k <= n; k++) {
        const uint32_t* cur = lists + (size_t)(k & 1) * kBatchListCap;
        uint32_t* nxt = lists + (size_t)((k + 1) & 1) * kBatchListCap;
        const unsigned int N = s_cnt[k & 1] < kBatchListCap ? s_cnt[k & 1] : kBatchListCap;
        if (s_cnt[k & 1] > kBatchListCap && threadIdx.x == 0) atomicOr(&r->error, ERR_CAPACITY);
        unsigned long long pairs = 0, nprobe = 0;
        unsigned int G = 1;                              // lanes per set (small levels)
        while (G < 32 && 2u * G * N <= blockDim.x) G <<= 1;
        const unsigned int sub = threadIdx.x & (G - 1), ngrp = blockDim.x / G;
        const unsigned int rounds = (N + ngrp - 1) / ngrp;
        for (unsigned int it = 0; it < rounds; it++) {
            const unsigned int e = it * ngrp + threadIdx.x / G;
            const bool act = e < N;
            const uint32_t S = act ? cur[e] : 0u;
            Key best = key_inf();
            double cS = 0.0;
            if (act) {
                cS = card_of(q, S);
                // the top vertex of S (minimal depth in the tree rooted at 0):
                // the one whose subtree holds all of S
                uint32_t top = 0;
                for (uint32_t T = S; T; T &= T - 1) {
                    const int v = __ffs(T) - 1;
                    if ((q.desc[v] & S) == S) top = 1u << v;
                }
                double bc = __longlong_as_double(0x7ff0000000000000ll);
                uint32_t bl = 0xffffffffu;
                unsigned int j = 0;
                for (uint32_t T = S ^ top; T; T &= T - 1, j++) {   // the k-1 pairs, j-th to lane j mod G
                    if ((j & (G - 1)) != sub) continue;
                    const int v = __ffs(T) - 1;
                    const uint32_t A = S & q.desc[v], B = S ^ A;
                    const double ca = side_cost(A), cb = side_cost(B);
                    nprobe += ((A & (A - 1)) != 0) + ((B & (B - 1)) != 0);
                    const double c = __dadd_rn(__dadd_rn(ca, cb), cS);
                    const uint32_t l = A < B ? A : B;
                    if (c < bc || (c == bc && l < bl)) {
                        bc = c;
                        bl = l;
                    }
                    pairs++;
                }
                if (bl != 0xffffffffu) best = Key{(unsigned long long)__double_as_longlong(bc), (unsigned long long)bl};
            }
            best = group_min(best, G);
            const bool lead = act && sub == 0;
            if (lead) {
                Val128 val;
                val.cost = __longlong_as_double((long long)best.c);
                val.card = cS;
                val.left = best.l;
                if (!memo128_insert(m, hi, S, val)) atomicOr(&r->error, ERR_TABLE_FULL);
            }
            if (lead && k < n) {                         // children S u {v}, each generated once
                TreeSetInfo info;
                uint32_t L = 0, nb = 0;
                for (uint32_t T = S; T; T &= T - 1) {
                    const uint32_t a = q.adj[__ffs(T) - 1];
                    nb |= a;
                    if (__popc(a & S) == 1) L |= T & (0u - T);
                }
                info.leaves = L;
                info.nb = nb;
                const uint32_t acc = children_of(q, S, info);
                if (acc) {
                    unsigned int d = atomicAdd(&s_cnt[(k + 1) & 1], (unsigned int)__popc(acc));
                    for (uint32_t V = acc; V; V &= V - 1, d++)
                        if (d < kBatchListCap) nxt[d] = S | (V & (0u - V));
                }
            }
        }
        block_sum3_part(pairs, pairs, nprobe, s_part);
        __syncthreads();                                 // level k is final in the memo
        if (threadIdx.x < 32) block_sum3_final(s_part, s_lvl);
        if (threadIdx.x == 0) {
            r->lvl_csg[k] = N;
            r->lvl_ccp[k] = s_lvl[0];                    // trees: every pair is a ccp pair (Lemma 8)
            r->lvl_pairs[k] = s_lvl[1];
            r->probes += s_lvl[2];
            s_cnt[k & 1] = 0;                            // becomes level k+2's counter
            r->t_level[k + 1] = globaltimer_ns();
        }
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    // counters and plan extraction (post-order, root last)
    unsigned long long csg = n, ccp = 0, prs = 0;
    r->lvl_csg[1] = n;
    r->lvl_ccp[1] = r->lvl_pairs[1] = 0;
    for (int k = 2; k <= n; k++) {
        csg += r->lvl_csg[k];
        ccp += r->lvl_ccp[k];
        prs += r->lvl_pairs[k];
    }
    r->csg = csg;
    r->ccp = ccp;
    r->pairs = prs;
    if (r->error) {
        r->n_nodes = 0;
        return;
    }
    uint32_t st_set[2 * kBatchMaxN], st_L[2 * kBatchMaxN];
    double st_c[2 * kBatchMaxN], st_card[2 * kBatchMaxN];
    int st_state[2 * kBatchMaxN], st_left[2 * kBatchMaxN];
    int sp = 1, nn = 0, last = -1;
    st_set[0] = n == 32 ? ~0u : (1u << n) - 1u;
    st_state[0] = 0;
    while (sp) {
        const int t = sp - 1;
        const uint32_t S = st_set[t];
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
        if (st_state[t] == 0) {
            const long long at = memo128_find(m, hi, S);
            if (at < 0) {
                r->error |= ERR_PROBE;
                r->n_nodes = 0;
                return;
            }
            const Val128 val = m.vals[at];
            st_c[t] = val.cost;
            st_card[t] = val.card;
            st_L[t] = (uint32_t)val.left;
            st_state[t] = 1;
            st_set[sp] = st_L[t];
            st_state[sp] = 0;
            sp++;
        } else if (st_state[t] == 1) {
            st_left[t] = last;
            st_state[t] = 2;
            st_set[sp] = S & ~st_L[t];
            st_state[sp] = 0;
            sp++;
        } else {
            mpdp_plan_node& nd = r->nodes[nn];
            nd.left = st_left[t];
            nd.right = last;
            nd.relation = -1;
            nd.reserved = 0;
            nd.set = S;
            nd.cardinality = st_card[t];
            nd.cost = st_c[t];
            last = nn++;
            --sp;
        }
    }
    r->n_nodes = (unsigned int)nn;
    r->cost = r->nodes[nn - 1].cost;
    r->t_level[n + 1] = globaltimer_ns();
}

}  // namespace mpdp
