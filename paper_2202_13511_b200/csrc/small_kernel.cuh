// small_kernel.cuh — the whole level loop of Alg. mpdp_gpu for a
// SMALL query on ONE CTA, with the memo in shared memory.
//
// For n <= kSmallMaxN the memo indexed by relation bitmask fits in shared
// memory: cost[2^n] (f64), card[2^n] (f64), left[2^n] (u16) = 18 B x 8192 =
// 144 KB at n = 13.  Every step of the path then stays on one SM:
//   * unrank + connectivity filter of level k: every thread
//     walks a contiguous run of colex ranks (one unrank, then Gosper);
//   * stream compaction: a block scan of the survivor counts writes the
//     level list to shared memory; the same scan yields max w (pairs per set);
//   * evaluate: G lanes per set (G = the power of two nearest
//     max_w / 8, 1..32), each lane a contiguous range of the set's csg-cmp
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
constexpr int kSmallListCap = 1716;        // max_k C(13, k)

__host__ __device__ constexpr size_t small_smem_bytes(int n) {
    return sizeof(SQ<uint32_t>) + (size_t(1) << n) * (8 + 8 + 2) + 4 * kSmallListCap + 33 * 33 * 4 + 64;
}

struct SmallSink {
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
__global__ void __launch_bounds__(kSmallBlock, 1) k_dp_small(const __grid_constant__ Params<uint32_t> p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SQ<uint32_t>& q = *reinterpret_cast<SQ<uint32_t>*>(smem_raw);
    load_query(q, p.q);
    const int n = p.n;
    const unsigned int NS = 1u << n;
    double* cost = reinterpret_cast<double*>(smem_raw + sizeof(SQ<uint32_t>));
    double* card = cost + NS;
    unsigned short* left = reinterpret_cast<unsigned short*>(card + NS);
    uint32_t* list = reinterpret_cast<uint32_t*>(left + NS + (NS & 1u));
    unsigned int* bin = list + kSmallListCap;                 // 33 x 33 u32 binomials
    __shared__ unsigned int s_sum[33];
    __shared__ unsigned long long s_max[33];
    __shared__ unsigned long long s_cnt[3];                   // ccp, pairs, probes of the level
    __shared__ unsigned long long s_tot[4];                   // csg, ccp, pairs, probes
    ResultDev* r = p.result;
    for (int i = threadIdx.x; i < 33 * 33; i += blockDim.x) {
        const int a = i / 33, b = i % 33;
        constexpr int NB = MaxN<uint32_t>::value + 1;
        bin[i] = (a < NB && b < NB) ? (unsigned int)p.q->binom[a * NB + b] : 0u;
    }
    if (threadIdx.x < 4) s_tot[threadIdx.x] = 0;
    if (threadIdx.x < 3) s_cnt[threadIdx.x] = 0;
    if (threadIdx.x == 0) r->error = 0;
    __syncthreads();
    for (int v = threadIdx.x; v < n; v += blockDim.x) {      // level 1
        cost[1u << v] = q.leaf[v];
        card[1u << v] = q.card[v];
    }
    if (threadIdx.x == 0) {
        r->t_level[2] = globaltimer_ns();
        s_tot[0] = (unsigned long long)n;
        r->lvl_csg[0] = r->lvl_ccp[0] = r->lvl_pairs[0] = 0;
        r->lvl_csg[1] = (unsigned long long)n;
        r->lvl_ccp[1] = r->lvl_pairs[1] = 0;
    }
    const unsigned int T = blockDim.x, lane = threadIdx.x & 31;
    for (int k = 2; k <= n; k++) {
        // ---- unrank + filter + compaction into list[]
        const unsigned int C = bin[n * 33 + k];
        const unsigned int r0 = (unsigned int)((unsigned long long)C * threadIdx.x / T);
        const unsigned int r1 = (unsigned int)((unsigned long long)C * (threadIdx.x + 1) / T);
        unsigned int flags = 0;
        unsigned long long wmax = 0;
        uint32_t S0 = r0 < r1 ? unrank_colex32(bin, n, k, r0) : 0u;
        {
            uint32_t S = S0;
            for (unsigned int i = 0; r0 + i < r1; i++) {
                if (connected_cls<uint32_t, CLS>(q, S, k)) {
                    flags |= 1u << i;
                    unsigned long long w;
                    set_kind<uint32_t, CLS>(q, S, k, w);
                    wmax = w > wmax ? w : wmax;
                }
                if (r0 + i + 1 < r1) S = gosper(S);
            }
        }
        unsigned int N;
        unsigned long long maxw;
        const unsigned int incl = block_scan_max((unsigned int)__popc(flags), wmax, N, maxw, s_sum, s_max);
        {
            unsigned int d = incl - (unsigned int)__popc(flags);
            uint32_t S = S0;
            for (unsigned int i = 0; r0 + i < r1; i++) {
                if ((flags >> i) & 1u) list[d++] = S;
                if (r0 + i + 1 < r1) S = gosper(S);
            }
        }
        __syncthreads();
        // ---- evaluate: G lanes per set, about 8 pairs per lane
        unsigned int G = 1;
        while (G < 32 && 8ull * G < maxw) G <<= 1;
        const unsigned int ngroups = T / G, grp = threadIdx.x / G, sub = threadIdx.x & (G - 1);
        const unsigned int rounds = (N + ngroups - 1) / ngroups;
        unsigned long long pairs = 0, nccp = 0, nprobe = 0;
        for (unsigned int it = 0; it < rounds; it++) {
            const unsigned int e = it * ngroups + grp;
            const bool act = e < N;
            SmallSink sink{cost, 0.0, key_inf(), 0};
            uint32_t S = 0;
            unsigned long long w = 0;
            if (act) {
                S = list[e];
                const int kind = set_kind<uint32_t, CLS>(q, S, k, w);
                sink.cS = small_card<CLS>(q, card, S, k);
                const unsigned long long per = (w + G - 1) / G;
                unsigned long long j0 = per * sub, j1 = j0 + per;
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
        if (lane == 0) {
            if (nccp) atomicAdd(&s_cnt[0], nccp);
            if (pairs) atomicAdd(&s_cnt[1], pairs);
            if (nprobe) atomicAdd(&s_cnt[2], nprobe);
        }
        __syncthreads();                                    // level barrier: level k is final
        if (threadIdx.x == 0) {
            r->lvl_csg[k] = N;
            r->lvl_ccp[k] = s_cnt[0];
            r->lvl_pairs[k] = s_cnt[1];
            s_tot[0] += N;
            s_tot[1] += s_cnt[0];
            s_tot[2] += s_cnt[1];
            s_tot[3] += s_cnt[2];
            s_cnt[0] = s_cnt[1] = s_cnt[2] = 0;       // (the next level adds after its scan's barriers)
            r->t_level[k + 1] = globaltimer_ns();
        }
    }
    if (threadIdx.x != 0) return;
    r->csg = s_tot[0];
    r->ccp = s_tot[1];
    r->pairs = s_tot[2];
    r->probes = s_tot[3];
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

}  // namespace mpdp
