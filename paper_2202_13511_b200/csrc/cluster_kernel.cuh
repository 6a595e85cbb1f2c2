// cluster_kernel.cuh — sparse tree queries (snowflakes) on ONE thread-block
// cluster of up to 16 CTAs (Blackwell thread-block clusters): the whole level
// loop of Alg. mpdp_gpu with the hardware cluster barrier between
// levels instead of a software grid barrier over ~300 CTAs.
//
// Why: a snowflake-20 level holds at most a few thousand connected sets of <= 19
// join pairs, far too little work to fill 148 SMs, and on the multi-CTA list
// kernel each level costs ~10-14 us of fixed latency -- the grid barrier, the
// per-CTA count prefix, and the dependent chain list load -> probes -> memo
// write -> next list.  One CTA (k_dp_tree1) has no grid barrier but is
// instruction-bound with thousands of sets per level.  A cluster keeps the
// cheap barrier (UCGABAR + one L1 invalidation) and spreads a level over 16
// SMs (snowflake-20: 0.266 -> 0.235 ms; a variant keeping the level lists in
// the CTAs' shared memory, read over DSMEM, measured 0.247 ms).
//
// Per level k (tree rooted at 0; the sets are connected subtrees):
//   * the level list (rank << 32 | mask, global, double-buffered) is cut into
//     one contiguous slice per CTA; a set is evaluated by G lanes (tree1's
//     rule), with the colex-rank memo in global memory (eval_tree_dense /
//     eval_range: the k-1 edge splits of Alg. mpdp_trees);
//   * the children S u {v} of the set are generated into a shared-memory
//     staging list (emitted once, from S' minus its largest leaf: children_of,
//     SURVEY NEXT-4), reserved in the global next list with ONE atomic per CTA
//     and copied out; the next list's counter rotates over three slots;
//   * cluster.sync() (release / acquire at cluster scope) ends the level.
// CTA 0 extracts the plan after the last level.
#pragma once
#include <cooperative_groups.h>

#include "small_kernel.cuh"

namespace mpdp {

constexpr int kClusterBlock = 1024;
constexpr int kClusterStage = 6144;       // staged children per CTA and level (shared memory)
constexpr int kClusterMaxLevel = 6144;    // eligibility: largest level (sets)

__host__ __device__ constexpr size_t cluster_smem_bytes(unsigned int rank_entries) {
    return sizeof(SQ<uint32_t>) + sizeof(unsigned int) * (rank_entries + 33 * 33 + 1) +
           kClusterStage * sizeof(unsigned long long) + 16;
}

__global__ void __launch_bounds__(kClusterBlock, 1) k_dp_tree_cluster(const __grid_constant__ Params<uint32_t> p) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    constexpr int MEMO = MEMO_DENSE;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SQ<uint32_t>& q = *reinterpret_cast<SQ<uint32_t>*>(smem_raw);
    unsigned int* rtab = reinterpret_cast<unsigned int*>(smem_raw + sizeof(SQ<uint32_t>));
    unsigned int* bin = rtab + p.memo.rg.entries;
    unsigned long long* stage =
        reinterpret_cast<unsigned long long*>(smem_raw + ((sizeof(SQ<uint32_t>) + sizeof(unsigned int) *
                                                           (p.memo.rg.entries + 33 * 33) + 15) & ~size_t(15)));
    __shared__ MemoView v;
    __shared__ unsigned int s_stage, s_base;
    __shared__ unsigned long long s_part[3][32];
    __shared__ unsigned long long s_lvl[3];
    memo_prologue<uint32_t, MEMO>(p, p.n, q, v, rtab);
    const int n = p.n;
    const unsigned int gen = p.q->gen;
    ResultDev* r = p.result;
    const unsigned int cs = cluster.num_blocks(), cr = cluster.block_rank();
    unsigned long long* lists = reinterpret_cast<unsigned long long*>(p.light);
    const unsigned long long cap = p.list_cap;            // entries per list buffer (two buffers)
    unsigned int* cnt = p.seg_cnt;                        // [3]: level k's set count at cnt[k % 3]
    if (cr == 0) {
        for (int j = threadIdx.x; j <= n; j += blockDim.x) p.desc[j] = LevelDesc{};
        if (threadIdx.x == 0) {
            cnt[0] = cnt[1] = cnt[2] = 0;
            r->error = 0;
            r->t_level[2] = globaltimer_ns();
        }
    }
    if (threadIdx.x == 0) s_stage = 0;
    __syncthreads();
    // level 2: the edges {u, a}, u < a, colex rank u + C(a, 2) (CTA 0)
    if (cr == 0) {
        for (int a = threadIdx.x; a < n; a += blockDim.x)
            for (uint32_t U = q.adj[a] & ((1u << a) - 1u); U; U &= U - 1) {
                const int u = __ffs(U) - 1;
                const unsigned int d = atomicAdd(&cnt[2], 1u);
                const unsigned int R = (unsigned int)u + bin[a * 33 + 2];
                if (d < cap) lists[d] = ((unsigned long long)R << 32) | ((1u << u) | (1u << a));
            }
    }
    cluster.sync();
    for (int k = 2; k <= n; k++) {
        const unsigned long long* cur = lists + (size_t)(k & 1) * cap;
        unsigned long long* nxt = lists + (size_t)((k + 1) & 1) * cap;
        const unsigned int Nall = __ldcg(&cnt[k % 3]);
        const unsigned int N = Nall < cap ? Nall : (unsigned int)cap;
        if (Nall > cap && cr == 0 && threadIdx.x == 0) atomicOr(&r->error, ERR_CAPACITY);
        if (cr == 0 && threadIdx.x == 0) cnt[(k + 2) % 3] = 0;   // level k+2's counter (read two barriers on)
        // this CTA's slice of the level
        const unsigned int e0 = (unsigned int)((unsigned long long)N * cr / cs);
        const unsigned int e1 = (unsigned int)((unsigned long long)N * (cr + 1) / cs);
        const unsigned int M = e1 - e0;
        unsigned long long pairs = 0, nccp = 0, nprobe = 0;
        unsigned int G = 1;                              // lanes per set (tree1's rule)
        while (G < 32 && 2u * G * M <= blockDim.x) G <<= 1;
        const unsigned int sub = threadIdx.x & (G - 1), ngrp = blockDim.x / G;
        const unsigned int rounds = (M + ngrp - 1) / ngrp;
        for (unsigned int it = 0; it < rounds; it++) {
            const unsigned int e = e0 + it * ngrp + threadIdx.x / G;
            const bool act = e < e1;
            const unsigned long long ent = act ? __ldcg(cur + e) : 0ull;
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
                    unsigned int d = atomicAdd(&s_stage, (unsigned int)__popc(acc));
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
                        if (d < kClusterStage) stage[d] = ((unsigned long long)Rp << 32) | Sp;
                    }
                }
            }
        }
        block_sum3_part(nccp, pairs, nprobe, s_part);
        __syncthreads();
        if (threadIdx.x < 32) block_sum3_final(s_part, s_lvl);
        if (threadIdx.x == 0) {
            const unsigned int ns = s_stage < kClusterStage ? s_stage : kClusterStage;
            if (s_stage > kClusterStage) atomicOr(&r->error, ERR_CAPACITY);
            s_base = ns ? atomicAdd(&cnt[(k + 1) % 3], ns) : 0u;   // ONE reservation per CTA
            LevelDesc& d = p.desc[k];
            if (M) atomicAdd(&d.n_light, (unsigned long long)M);
            if (s_lvl[0]) atomicAdd(&d.ccp, s_lvl[0]);
            if (s_lvl[1]) atomicAdd(&d.pairs, s_lvl[1]);
            if (s_lvl[2]) atomicAdd(&d.probes, s_lvl[2]);
        }
        __syncthreads();
        const unsigned int ns = s_stage < kClusterStage ? s_stage : kClusterStage;
        for (unsigned int i = threadIdx.x; i < ns; i += blockDim.x) {
            const unsigned long long dst = (unsigned long long)s_base + i;
            if (dst < cap) nxt[dst] = stage[i];
            else atomicOr(&r->error, ERR_CAPACITY);
        }
        __syncthreads();
        if (threadIdx.x == 0) s_stage = 0;
        if (cr == 0 && threadIdx.x == 0) r->t_level[k + 1] = globaltimer_ns();
        cluster.sync();                                  // level k is final in the memo and the next list
    }
    if (cr == 0 && p.do_extract && threadIdx.x < 32) {
        level_counters_warp(p, p.result);
        if (threadIdx.x == 0) extract_phase<uint32_t, MEMO>(p, q, v, rtab, gen);
    }
}

}  // namespace mpdp
