// list_kernel.cuh — the level loop of Alg. mpdp_gpu for tree
// queries (CLS_TREE: every set is light, k-1 join pairs) as ONE persistent
// cooperative kernel with level lists and enumerate-ahead.
//
// Phase k (between two grid barriers) does two independent things:
//   * unrank + connectivity filter of level k+1 into the
//     other level list -- enumeration does not read the memo, so it runs one
//     level ahead;
//   * evaluation of level k's list (csg-cmp pairs, C_out, per-set min, memo
//     scatter), G lanes per set (small_phase).
// The stream compaction of P:889 is a warp-aggregated reservation: a warp's
// survivors are written contiguously at an offset from one atomicAdd on the
// level counter (list order is irrelevant: every entry carries its colex rank,
// which is its memo slot).  Compared with the tile kernel (fused.cuh) the work
// of both halves is split evenly over all threads of the grid, so the CTAs
// reach the barrier within one set evaluation of each other, and there is one
// grid barrier per level.
#pragma once
#include "fused.cuh"

namespace mpdp {

constexpr int kListChunk = 32;             // ranks per thread per reservation pass

// Level k's share [share_lo, share_hi) -> segmented list `out` (entries
// rank << 32 | mask): CTA b owns the segment [b * seg, (b + 1) * seg) with
// seg = blockDim * rpt (its ranks); *cnt (this CTA's counter, zeroed
// beforehand; shared memory inside the level loop) counts its survivors.  Every thread walks a contiguous run of rpt ranks (one unrank,
// then Gosper); per pass of kListChunk ranks a warp reserves its survivors with
// one atomic on its CTA's counter.  No CTA-wide synchronisation, so warps can
// interleave enumeration and evaluation.  (One grid-wide counter serialised
// thousands of same-address atomics at one L2 slice: the last warps waited
// ~200 us.)
__device__ __forceinline__ unsigned long long list_rpt(unsigned long long nranks) {
    const unsigned long long T = (unsigned long long)gridDim.x * blockDim.x;
    return (nranks + T - 1) / T;
}

template <int CLS>
__device__ void enum_to_list(const Params<uint32_t>& p, int k, const SQ<uint32_t>& q, const unsigned int* bin,
                             unsigned long long* out, unsigned int* cnt) {
    const unsigned int lo = p.share_lo[k], hi = p.share_hi[k];
    const unsigned long long rpt = list_rpt(hi - lo);
    const unsigned long long gtid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned long long b0 = lo + gtid * rpt;
    const unsigned long long b1 = b0 + rpt < hi ? b0 + rpt : hi;
    unsigned long long* seg = out + (unsigned long long)blockIdx.x * blockDim.x * rpt;
    const unsigned int lane = threadIdx.x & 31;
    uint32_t S = b0 < b1 ? unrank_colex32(bin, p.n, k, (unsigned int)b0) : 0u;
    for (unsigned long long pass = 0; pass < rpt; pass += kListChunk) {   // same trip count on every lane
        const unsigned long long r0 = b0 + pass;
        const uint32_t S0 = S;
        unsigned int flags = 0;
#pragma unroll 4
        for (int i = 0; i < kListChunk; i++) {
            if (r0 + i < b1) {
                if (connected_cls<uint32_t, CLS>(q, S, k)) flags |= 1u << i;
                if (r0 + i + 1 < b1) S = gosper(S);
            }
        }
        const unsigned int c = __popc(flags);
        unsigned int inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned int t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= (unsigned int)o) inc += t;
        }
        const unsigned int total = __shfl_sync(0xffffffffu, inc, 31);
        unsigned int base = 0;
        if (lane == 31 && total) base = atomicAdd(cnt, total);   // this CTA's counter: only its warps contend
        base = __shfl_sync(0xffffffffu, base, 31);
        if (c) {
            unsigned long long d = base + inc - c;
            // the segment end must stay inside the list (plan_layout may clamp
            // list_cap to the scratch space): overflow is an error, never a
            // write past the list
            const unsigned long long seg0 = (unsigned long long)blockIdx.x * blockDim.x * rpt;
            if (seg0 + d + c > p.list_cap) {
                atomicOr(&p.result->error, ERR_CAPACITY);
            } else {
                uint32_t X = S0;
                for (int i = 0; i < kListChunk && r0 + i < b1; i++) {
                    if ((flags >> i) & 1u) seg[d++] = ((r0 + i) << 32) | X;
                    if (r0 + i + 1 < b1) X = gosper(X);
                }
            }
        }
    }
}

// Sparse generation of level k+1 from level k's list (trees; SURVEY §8(f)
// NEXT-4), used when a thread's share of the candidates (n - k per set) is
// well below its share of the C(n, k+1) ranks: every connected
// S' of size k+1 is S u {v} for a connected S and a neighbour v of S, and is
// emitted exactly once -- from S = S' \ {u*}, u* the largest leaf of G[S'] (a
// new vertex v is always a leaf of the tree G[S u {v}]; the leaves are the
// vertices whose removal keeps the set connected).  Replaces the scan of all
// C(n, k+1) ranks, whose survivors are a vanishing fraction on sparse graphs
// (chain: n - k of C(n, k+1)).  CTA b expands the inputs [N*b/grid,
// N*(b+1)/grid) into its output segment of `seg` entries.
template <typename Locate>
__device__ void expand_to_list(const Params<uint32_t>& p, int k, const SQ<uint32_t>& q, const unsigned int* bin,
                               const unsigned long long* src, const Locate& loc, unsigned long long N,
                               unsigned long long* out, unsigned int* cnt, unsigned long long seg,
                               Team tm = whole_cta()) {
    // G lanes per input set (largest power of two <= 32 that keeps every set a
    // group); lane `sub` tests the candidates v with index = sub (mod G)
    const unsigned long long nthreads = (unsigned long long)gridDim.x * tm.size;
    unsigned int G = 1;
    while (G < 32 && 2ull * G * N <= nthreads) G <<= 1;
    const unsigned int sub = tm.tid & (G - 1), gpc = tm.size / G;
    const unsigned long long c_lo = N * blockIdx.x / gridDim.x, c_hi = N * (blockIdx.x + 1) / gridDim.x;
    unsigned long long* segp = out + (unsigned long long)blockIdx.x * seg;
    const unsigned int lane = threadIdx.x & 31;
    for (unsigned long long base = c_lo; base < c_hi; base += gpc) {   // same trip count on every lane
        const unsigned long long e = base + tm.tid / G;
        uint32_t S = 0, em = 0;
        if (e < c_hi) {
            S = (uint32_t)src[loc(e)];
            uint32_t Nb = 0;
            for (uint32_t T = S; T; T &= T - 1) Nb |= q.adj[__ffs(T) - 1];
            unsigned int j = 0;
            for (uint32_t V = Nb & ~S; V; V &= V - 1, j++) {
                if ((j & (G - 1)) != sub) continue;
                const int v = __ffs(V) - 1;
                const uint32_t Sp = S | (1u << v);
                bool ok = true;                     // no leaf of G[S'] above v
                for (uint32_t U = S & ~((2u << v) - 1u); U; U &= U - 1)
                    if (__popc(q.adj[__ffs(U) - 1] & Sp) == 1) {
                        ok = false;
                        break;
                    }
                if (ok) em |= 1u << v;
            }
        }
        const unsigned int c = __popc(em);
        unsigned int inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned int t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= (unsigned int)o) inc += t;
        }
        const unsigned int total = __shfl_sync(0xffffffffu, inc, 31);
        unsigned int wbase = 0;
        if (lane == 31 && total) wbase = atomicAdd(cnt, total);
        wbase = __shfl_sync(0xffffffffu, wbase, 31);
        unsigned long long d = wbase + inc - c;
        for (uint32_t E = em; E; E &= E - 1) {
            const uint32_t Sp = S | (E & (0u - E));
            unsigned int R = 0;                     // colex rank of S'
            int i = 1;
            for (uint32_t T = Sp; T; T &= T - 1, i++) R += bin[(__ffs(T) - 1) * 33 + i];
            if (d < seg)
                segp[d] = ((unsigned long long)R << 32) | Sp;
            else
                atomicOr(&p.result->error, ERR_CAPACITY);
            d++;
        }
    }
}

// Locate entry e of a segmented level list: s_pre holds the exclusive prefix of
// the per-CTA counts (grid + 1 entries, in shared memory).
struct SegLocate {
    const unsigned int* pre;
    unsigned int nseg;
    unsigned long long seg;
    __device__ __forceinline__ unsigned int seek(unsigned long long e) const {
        unsigned int lo = 0, hi = nseg;            // largest b with pre[b] <= e
        while (hi - lo > 1) {
            const unsigned int mid = (lo + hi) >> 1;
            if (pre[mid] <= e) lo = mid; else hi = mid;
        }
        return lo;
    }
    // sequential access with a cursor (e never decreases)
    __device__ __forceinline__ unsigned long long at(unsigned long long e, unsigned int& b) const {
        while (b + 1 < nseg && pre[b + 1] <= e) b++;
        return (unsigned long long)b * seg + (e - pre[b]);
    }
    __device__ __forceinline__ unsigned long long operator()(unsigned long long e) const {
        unsigned int b = seek(e);
        return at(e, b);
    }
};

// Exclusive prefix of cnt[0..g) into pre[0..g] (shared memory), block-wide:
// per-thread partial sums, warp shuffle scans, one scan of the warp totals.
__device__ __forceinline__ void seg_prefix(const unsigned int* cnt, unsigned int g, unsigned int* pre) {
    __shared__ unsigned int s_warp[kBlock / 32];
    const unsigned int per = (g + blockDim.x - 1) / blockDim.x;
    const unsigned int i0 = threadIdx.x * per;
    const unsigned int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned int sum = 0;
    for (unsigned int i = i0; i < i0 + per && i < g; i++) sum += ld_relaxed_u32(cnt + i);
    unsigned int inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= (unsigned int)o) inc += t;
    }
    if (lane == 31) s_warp[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        const unsigned int nw = blockDim.x >> 5;
        unsigned int x = lane < nw ? s_warp[lane] : 0u, y = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned int t = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= (unsigned int)o) y += t;
        }
        if (lane < nw) s_warp[lane] = y - x;      // exclusive
        if (lane == nw - 1) pre[g] = y;
    }
    __syncthreads();
    unsigned int acc = s_warp[wid] + inc - sum;
    for (unsigned int i = i0; i < i0 + per && i < g; i++) {
        pre[i] = acc;
        acc += ld_relaxed_u32(cnt + i);
    }
    __syncthreads();
}

template <int CLS>
__global__ void __launch_bounds__(kBlock, 2) k_dp_list(const __grid_constant__ Params<uint32_t> p) {
    constexpr int MEMO = MEMO_DENSE;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SQ<uint32_t>& q = *reinterpret_cast<SQ<uint32_t>*>(smem_raw);
    unsigned int* rtab = reinterpret_cast<unsigned int*>(smem_raw + sizeof(SQ<uint32_t>));
    unsigned int* bin = rtab + p.memo.rg.entries;                  // 33 x 33 binomials
    // (C(v, m+1), C(v, m+1) - C(v, m)) pairs of the tree walk, 8-byte aligned
    uint2* binp = reinterpret_cast<uint2*>(bin + 33 * 33 + ((p.memo.rg.entries + 33 * 33) & 1u));
    __shared__ MemoView v;

    memo_prologue<uint32_t, MEMO>(p, p.n, q, v, rtab);
    unsigned int nbar = 0;                 // grid barriers passed (thread 0)
    __syncthreads();
    for (int i = threadIdx.x; i < 33 * 32; i += blockDim.x) {
        const int a = i / 32, b = i % 32;
        binp[a * 33 + b] = make_uint2(bin[a * 33 + b + 1], bin[a * 33 + b + 1] - bin[a * 33 + b]);
    }
    const unsigned int gen = p.q->gen;
    __syncthreads();
    unsigned long long* lists[2] = {reinterpret_cast<unsigned long long*>(p.light),
                                    reinterpret_cast<unsigned long long*>(p.light) + p.list_cap};
    unsigned int* cnts[2] = {p.seg_cnt, p.seg_cnt + kMaxGrid};
    __shared__ unsigned int s_pre[kMaxGrid + 1];

    if (blockIdx.x == 0 && threadIdx.x == 0) p.result->t_level[p.k_begin] = globaltimer_ns();
    if (threadIdx.x == 0) cnts[p.k_begin & 1][blockIdx.x] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0)
        p.desc[p.k_begin].seg = (unsigned int)(blockDim.x * list_rpt(p.share_hi[p.k_begin] - p.share_lo[p.k_begin]));
    __syncthreads();
    enum_to_list<CLS>(p, p.k_begin, q, bin, lists[p.k_begin & 1], cnts[p.k_begin & 1] + blockIdx.x);
    grid_sync(p.gbar, nbar, &p.result->error);
    for (int k = p.k_begin; k <= p.k_end; k++) {
        if (blockIdx.x == 0 && threadIdx.x == 0 && k > p.k_begin) p.result->t_level[k] = globaltimer_ns();
        if (threadIdx.x == 0 && k < p.k_end) cnts[(k + 1) & 1][blockIdx.x] = 0;   // read by every CTA in phase k-1 only
        seg_prefix(cnts[k & 1], gridDim.x, s_pre);                                 // (its syncs publish the zero)
        const unsigned long long N = s_pre[gridDim.x];
        const SegLocate loc{s_pre, gridDim.x, ld_relaxed_u32(&p.desc[k].seg)};
        const bool counting = (p.count_levels >> k) & 1ull;
        // level k+1: sparse expansion of this list when its candidates are far
        // fewer than the ranks (whole levels only: a rank share of a sharded
        // level is not closed under expansion)
        bool expand = false, fused_grow = false;
        unsigned long long seg_next = 0;
        if (k < p.k_end) {
            const unsigned long long C1 = p.share_hi[k + 1] - p.share_lo[k + 1];
            const bool whole = p.share_lo[k] == 0 && p.share_lo[k + 1] == 0 && p.share_hi[k] == bin[p.n * 33 + k] &&
                               p.share_hi[k + 1] == bin[p.n * 33 + k + 1];
            // fewer candidates than ranks, and per-thread work ((sets per
            // thread) * (n - k) candidates over up to 32 lanes per set) below
            // the per-thread share of the ranks
            const unsigned long long T = (unsigned long long)gridDim.x * blockDim.x;
            const double cand = p.expand_fac * (double)N * (double)(p.n - k);   // weighted candidates
            const unsigned long long seg_grow = ((N + gridDim.x - 1) / gridDim.x + 1) * (unsigned long long)(p.n - k);
            expand = CLS == CLS_TREE && whole && cand <= (double)C1 && seg_grow * gridDim.x <= p.list_cap &&
                     2ull * ((32ull * N + T - 1) / T) * (unsigned long long)(p.n - k) <= 32ull * ((C1 + T - 1) / T);
            // dense tree levels (one thread per set): the evaluation walk itself
            // generates level k+1 (emit_children), no rank scan
            // (only where the candidates are few next to the ranks: the rank scan
            // writes the next list in colex order, which the star levels' probes
            // need for locality -- measured 1.42 vs 1.59 ms on star-25)
            fused_grow = CLS == CLS_TREE && whole && k >= 3 && 2ull * N > T && seg_grow * gridDim.x <= p.list_cap &&
                         cand <= (double)C1;
            if (fused_grow) expand = false;
            seg_next = (expand || fused_grow) ? seg_grow : (unsigned long long)blockDim.x * list_rpt(C1);
            if (blockIdx.x == 0 && threadIdx.x == 0) p.desc[k + 1].seg = (unsigned int)seg_next;
        }
#ifdef MPDP_TRACE
        __shared__ unsigned long long s_me, s_mv;
        if (threadIdx.x == 0) s_me = s_mv = 0;
        __syncthreads();
        const unsigned long long ct_a = globaltimer_ns();
#endif
        // even warps enumerate level k+1 first, odd warps evaluate level k
        // first: ALU-bound enumeration overlaps latency-bound evaluation.  On
        // sparse levels (few sets per thread, next level by expansion) the
        // two halves of the CTA split the work instead: warps 0..3 expand,
        // warps 4..7 evaluate, so the level costs max(expand, evaluate) of
        // latency instead of their sum.
        const bool split = expand && 8ull * N <= (unsigned long long)gridDim.x * blockDim.x && blockDim.x >= 64;
        const unsigned int half = blockDim.x / 2;
        const bool enum_first = split ? threadIdx.x < half : ((threadIdx.x >> 5) & 1) == 0;
        const Team tm_enum = split ? Team{threadIdx.x, half} : whole_cta();
        const Team tm_eval = split ? Team{threadIdx.x - half, half} : whole_cta();
        unsigned long long pairs = 0, nccp = 0, nprobe = 0;
        __shared__ unsigned int s_emit;
        if (threadIdx.x == 0) s_emit = 0;
        __syncthreads();
        const EmitCtx ectx{lists[(k + 1) & 1] + (unsigned long long)blockIdx.x * seg_next, seg_next, &s_emit};
        auto next_level = [&]() {
            if (k >= p.k_end || fused_grow) return;
            if (expand)
                expand_to_list(p, k, q, bin, lists[k & 1], loc, N, lists[(k + 1) & 1], &s_emit, seg_next, tm_enum);
            else
                enum_to_list<CLS>(p, k + 1, q, bin, lists[(k + 1) & 1], &s_emit);
        };
        if (enum_first) next_level();
#ifdef MPDP_TRACE
        const unsigned long long ct_b = globaltimer_ns();
#endif
        if (N && (!split || !enum_first))
            small_phase<CLS, MEMO>(p, k, q, v, rtab, bin, gen, lists[k & 1], loc, N, pairs, nccp, nprobe, binp,
                                   fused_grow ? &ectx : nullptr, tm_eval);
        if (!enum_first && !split) next_level();
        if (k < p.k_end) {                     // this CTA's count of level k+1 (reserved in shared memory)
            __syncthreads();
            if (threadIdx.x == 0) cnts[(k + 1) & 1][blockIdx.x] = s_emit;
        }
#ifdef MPDP_TRACE
        const unsigned long long ct_c = globaltimer_ns();
        if ((threadIdx.x & 31) == 0) {
            atomicMax(&s_me, ct_b - ct_a);
            atomicMax(&s_mv, ct_c - ct_b);
        }
#endif
        if (counting) {
            if (blockIdx.x == 0 && threadIdx.x == 0) p.desc[k].n_light = N;
            flush_counters(&p.desc[k], pairs, nccp, nprobe);
        }
#ifdef MPDP_TRACE
        __syncthreads();
        if (threadIdx.x == 0 && blockIdx.x < kCtaTraceMax) {
            unsigned long long* o = g_cta_arrive + ((unsigned long long)k * kCtaTraceMax + blockIdx.x) * kCtaTraceSlots;
            o[0] = ct_a;
            o[1] = ct_b - ct_a;                // enumerate ahead (thread 0's warp)
            o[2] = s_me;                       // slowest warp: enumerate
            o[3] = ct_c - ct_b;                // evaluate (thread 0's warp)
            o[4] = 1;
            o[5] = globaltimer_ns();           // whole CTA done
            o[6] = s_mv;                       // slowest warp: evaluate
            o[7] = N;
        }
#endif
        grid_sync(p.gbar, nbar, &p.result->error);
    }
    if (p.do_extract && blockIdx.x == 0 && threadIdx.x < 32) {
        if (threadIdx.x == 0) p.result->t_level[p.n + 1] = globaltimer_ns();
        level_counters_warp(p, p.result);
        if (threadIdx.x == 0) extract_phase<uint32_t, MEMO>(p, q, v, rtab, gen);
    }
}

}  // namespace mpdp
