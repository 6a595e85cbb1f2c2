// fused.cuh — the whole level loop of Alg. mpdp_gpu as ONE
// persistent cooperative kernel (perfect-hash memo, n <= 32).
//
// Per level k every CTA claims tiles of colex ranks.  A tile is enumerated
// (unrank + Gosper + connectivity + classification, as k_enum); its light
// sets (<= 32 join pairs) go to a CTA-local shared-memory queue together with
// their colex rank -- which IS their memo slot -- and are evaluated on the spot
// by the CTA's threads.  Light sets therefore need no global compaction, list
// traffic or second launch.  Heavy sets are compacted into the global heavy
// list by the decoupled look-back scan exactly as in k_enum, then evaluated
// after a grid barrier by the work-item heavy phase.  Levels are separated by
// a grid barrier (the dependency of P:209-215), and block 0 extracts the plan
// at the end.  One launch per query instead of 2-3 per level.
#pragma once
#include "level_kernels.cuh"
#include "dataflow.cuh"

namespace mpdp {

constexpr int kFusedRanksPerThread = 8;
constexpr int kFusedTile = kBlock * kFusedRanksPerThread;   // 2048 ranks, queue of 2048 sets
constexpr bool kDeferRemainder = false;     // defer nq mod blockDim light sets (else only nq < blockDim)

__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned int ld_relaxed_u32(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Grid barrier over a monotonic arrival counter (zeroed before every launch:
// k_init, or a memset before each sharded launch).  All CTAs are co-resident
// (cooperative launch).  Thread 0 of each CTA counts the barriers it has passed
// (`nbar`), arrives with ONE fire-and-forget red.release (which, after the
// bar.sync, orders the whole CTA's prior writes), and polls with ld.acquire
// until all gridDim.x arrivals of this barrier are in; bar.sync then extends
// the acquire to the CTA.  No last-arriver reset chain: the barrier costs one
// reduction landing in L2 plus one poll.
__device__ __forceinline__ void grid_sync(unsigned int* bar, unsigned int& nbar, unsigned int* err) {
    __syncthreads();
    if (gridDim.x == 1) return;        // one CTA: bar.sync already orders its global accesses
    if (threadIdx.x == 0) {
        nbar++;
        const unsigned int target = nbar * gridDim.x;
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        // poll with relaxed loads (an acquire load invalidates the SM's L1 on
        // every poll, under co-resident warps that use it for memo probes),
        // then one acquire fence; the watchdog clock is read every 1024 polls
        unsigned int spins = 0;
        unsigned long long t0 = 0;
        while (ld_relaxed_u32(bar) < target) {
            __nanosleep(20);
            if ((++spins & 1023u) == 0) {
                if (!t0) {
                    t0 = globaltimer_ns();
                } else if (watchdog_expired(t0)) {   // never hang the device: flag and fall through
                    atomicOr(err, ERR_HANG);
                    break;
                }
            }
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
}

__device__ __forceinline__ uint32_t unrank_colex32(const unsigned int* bin, int n, int k, unsigned int r) {
    uint32_t S = 0;
    int c = n - 1;
    for (int i = k; i >= 1; i--) {
        while (bin[c * 33 + i] > r) c--;
        S |= 1u << c;
        r -= bin[c * 33 + i];
        c--;
    }
    return S;
}


// Min of a Key over aligned groups of G lanes (G a power of two <= 32); every
// lane of the warp must call it.
__device__ __forceinline__ Key group_min(Key k, unsigned int G) {
    for (unsigned int o = 1; o < G; o <<= 1) {
        Key t;
        t.c = __shfl_xor_sync(0xffffffffu, k.c, o);
        t.l = __shfl_xor_sync(0xffffffffu, k.l, o);
        if (key_less(t, k)) k = t;
    }
    return k;
}

// card(S) for a set of level k >= 3 with colex rank R.  Reading R5's product is
// a left fold over the ascending elements, so with p = max(S)
//     card(S) = (..((card(S \ {p}) * card[p]) * sel(u_1, p)) * ..)   (u_i in S, u_i < p, ascending)
// bit for bit; card(S \ {p}) is read from the level k-1 memo (colex rank
// R - C(p, k)) when S \ {p} is connected: p is a leaf of G[S] on trees (S and
// desc[p] meet only in p), always on cliques.  Otherwise the full product.
template <int CLS, int MEMO = MEMO_DENSE>
__device__ __forceinline__ double card_fast(const MemoPtrs& P, const MemoView& v, const unsigned int* bin,
                                            const SQ<uint32_t>& q, uint32_t S, int k, unsigned int R) {
    const int p = 31 - __clz(S);
    const uint32_t b = 1u << p;
    const bool in_memo = k >= 3 && ((CLS == CLS_TREE && (S & q.desc[p]) == b) || CLS == CLS_CLIQUE);
    if (!in_memo) return card_of(q, S);
    double x = __dmul_rn(__ldcs(P.dcard + memo_slot_r<MEMO>(v, k - 1, R - bin[p * 33 + k], S ^ b)), q.card[p]);
    for (uint32_t W = S & q.adj[p] & (b - 1u); W; W &= W - 1) x = __dmul_rn(x, q.sel[(__ffs(W) - 1) * q.n + p]);
    return x;
}

// Deferred light sets of level k (tiles that found fewer sets than threads push
// theirs to the grid-wide small list instead of evaluating them in place):
// after the level barrier every CTA takes a share, G lanes per set with G the
// largest power of two that still gives every set a group (G = 32: one warp
// per set, lanes = join pairs).  Sparse and small levels thus use the whole
// grid instead of the few CTAs whose tiles held the sets.
struct DenseLocate {
    __device__ __forceinline__ unsigned long long operator()(unsigned long long e) const { return e; }
    __device__ __forceinline__ unsigned int seek(unsigned long long) const { return 0; }
    __device__ __forceinline__ unsigned long long at(unsigned long long e, unsigned int&) const { return e; }
};

// Fused generation of level k+1 from an evaluated tree set S (list kernel;
// the tree case of expand_to_list): a connected S' of size k+1
// is emitted exactly once, from S = S' \ {u*} with u* its largest leaf.  For
// S' = S u {v} (v adjacent to exactly one u in S) the leaves are
// (leaves(S) \ {u}) u {v}, so v is accepted iff v > max(leaves(S) \ {u}).
// The children are counted, reserved with one shared-memory atomic and written
// to this CTA's segment of the next list; rank(S u {v}) = R + C(v, k+1) when v
// is above max(S), else it is recomputed.
// A team of whole warps of the CTA that shares a phase's work: the whole CTA,
// or (sparse levels of the list kernel) half of it, so that the next level's
// expansion and this level's evaluation run on different warps at once.
struct Team {
    unsigned int tid, size;
};
__device__ __forceinline__ Team whole_cta() { return Team{threadIdx.x, blockDim.x}; }

struct EmitCtx {
    unsigned long long* seg;               // this CTA's segment of the next level list
    unsigned long long cap;                // its capacity
    unsigned int* count;                   // shared-memory fill counter
};

__device__ __forceinline__ uint32_t children_of(const SQ<uint32_t>& q, uint32_t S, const TreeSetInfo& in) {
    const uint32_t L = in.leaves;
    const int m1 = 31 - __clz(L);                         // largest leaf (k >= 2: at least two leaves)
    const uint32_t L2 = L & ~(1u << m1);
    const int m2 = L2 ? 31 - __clz(L2) : -1;              // second largest
    uint32_t cand = in.nb & ~S;
    if (m2 >= 0) cand &= ~((2u << m2) - 1u);              // every accepted v exceeds the second largest leaf
    uint32_t acc = 0;
    for (uint32_t V = cand; V; V &= V - 1) {
        const int v = __ffs(V) - 1;
        const uint32_t u = q.adj[v] & S;                  // its one neighbour in S (tree)
        const int thr = (u == (1u << m1)) ? m2 : m1;
        if (v > thr) acc |= 1u << v;
    }
    return acc;
}

// Warp-cooperative write of the children (all active lanes call it together):
// one shared-memory reservation per warp, children written vertex-major
// (for each v, the lanes' S u {v} side by side), so the next level's list keeps
// runs of colex-near sets -- consecutive parents give consecutive child ranks.
__device__ __forceinline__ void emit_children(const unsigned int* bin, uint32_t S, unsigned int R, int k, uint32_t acc,
                                              const EmitCtx& ec, unsigned int* err) {
    const unsigned int act = __activemask();
    const unsigned int lane = threadIdx.x & 31, lt = (1u << lane) - 1u;
    const unsigned int tot = __reduce_add_sync(act, (unsigned int)__popc(acc));
    if (!tot) return;
    const uint32_t any = __reduce_or_sync(act, acc);
    const int leader = __ffs(act) - 1;
    unsigned int base = 0;
    if ((int)lane == leader) base = atomicAdd(ec.count, tot);
    base = __shfl_sync(act, base, leader);
    const int mx = 31 - __clz(S);
    for (uint32_t V = any; V; V &= V - 1) {
        const int v = __ffs(V) - 1;
        const bool mine = (acc >> v) & 1u;
        const unsigned int bal = __ballot_sync(act, mine);
        if (mine) {
            const unsigned long long d = base + __popc(bal & lt);
            const uint32_t Sp = S | (1u << v);
            unsigned int Rp;
            if (v > mx) {
                Rp = R + bin[v * 33 + k + 1];
            } else {
                Rp = 0;
                int i = 1;
                for (uint32_t T = Sp; T; T &= T - 1, i++) Rp += bin[(__ffs(T) - 1) * 33 + i];
            }
            if (d < ec.cap)
                ec.seg[d] = ((unsigned long long)Rp << 32) | Sp;
            else
                atomicOr(err, ERR_CAPACITY);
        }
        base += __popc(bal);
    }
}

// One thread per set (G = 1): the CTA's run is walked in rounds of blockDim;
// the next list entry is loaded before the current set is evaluated (the set
// evaluation is a latency chain, the list load should not add to it).
// One set, one thread: evaluate, min, memo scatter (and, on fused-grow tree
// levels, the children of the set).
template <int CLS, int MEMO>
__device__ __forceinline__ void eval_set_thread(const Params<uint32_t>& p, int k, const SQ<uint32_t>& q,
                                                const MemoView& v, const unsigned int* rtab, const unsigned int* bin,
                                                unsigned int gen, unsigned long long ent, unsigned long long& pairs,
                                                unsigned long long& nccp, unsigned long long& nprobe,
                                                const uint2* binp, const EmitCtx* emit) {
    const uint32_t S = (uint32_t)ent;
    const unsigned int R = (unsigned int)(ent >> 32);
    unsigned long long w;
    const int kind = set_kind<uint32_t, CLS>(q, S, k, w);
    pairs += w;
    if constexpr (CLS == CLS_TREE && MEMO == MEMO_DENSE) {
        if (k > 2) {
            if (emit) {
                TreeSetInfo info;
                eval_tree_dense<MEMO, true, true>(p.memo, gen, v, rtab, bin, q, S, k, R, nprobe, binp, &info);
                __syncwarp(__activemask());
                emit_children(bin, S, R, k, children_of(q, S, info), *emit, &p.result->error);
            } else {
                eval_tree_dense<MEMO, true>(p.memo, gen, v, rtab, bin, q, S, k, R, nprobe, binp);
            }
            nccp += w;
            return;
        }
    }
    PairSink<uint32_t, MEMO> sink;
    sink.init(&p.memo, gen, &v, rtab, &q, card_fast<CLS, MEMO>(p.memo, v, bin, q, S, k, R));
    eval_range<uint32_t, CLS>(q, S, k, kind, 0, w, sink, nccp);
    sink.flush();
    nprobe += sink.nprobe;
    const unsigned long long idx = memo_slot_r<MEMO>(v, k, R, S);
    p.memo.dcost[idx] = __longlong_as_double((long long)sink.best.c);
    __stcs(p.memo.dleft + idx, (unsigned int)sink.best.l);
    p.memo.dcard[idx] = sink.cS;
}

template <int CLS, int MEMO, typename Locate>
__device__ __forceinline__ void small_phase_thread(const Params<uint32_t>& p, int k, const SQ<uint32_t>& q,
                                                   const MemoView& v, const unsigned int* rtab, const unsigned int* bin,
                                                   unsigned int gen, const unsigned long long* list, const Locate& loc,
                                                   unsigned long long c_lo, unsigned long long c_hi,
                                                   unsigned long long& pairs, unsigned long long& nccp,
                                                   unsigned long long& nprobe, const uint2* binp,
                                                   const EmitCtx* emit, Team tm) {
    unsigned long long e = c_lo + tm.tid;
    if (e >= c_hi) return;
    unsigned int cur = loc.seek(e);
    unsigned long long nxt = __ldcs(list + loc.at(e, cur));
    for (; e < c_hi; e += tm.size) {
        const unsigned long long ent = nxt;
        if (e + tm.size < c_hi) nxt = __ldcs(list + loc.at(e + tm.size, cur));
        eval_set_thread<CLS, MEMO>(p, k, q, v, rtab, bin, gen, ent, pairs, nccp, nprobe, binp, emit);
    }
}

template <int CLS, int MEMO, typename Locate>
__device__ void small_phase(const Params<uint32_t>& p, int k, const SQ<uint32_t>& q, const MemoView& v,
                            const unsigned int* rtab, const unsigned int* bin, unsigned int gen,
                            const unsigned long long* list, const Locate& loc, unsigned long long nsmall,
                            unsigned long long& pairs, unsigned long long& nccp, unsigned long long& nprobe,
                            const uint2* binp = nullptr, const EmitCtx* emit = nullptr, Team tm = whole_cta()) {
    const unsigned long long total = (unsigned long long)gridDim.x * tm.size;
    unsigned int G = 1;
    // (dense tree levels stop at G = 4: wider groups take the generic
    // per-pair path with a rank lookup per probe; measured snowflake-20 252 ->
    // 244 us, snowflake-24 337 -> 327 us, G = 2 / 8 / 32 slower)
    const unsigned int gmax = (CLS == CLS_TREE && MEMO == MEMO_DENSE) ? 4u : 32u;
    while (G < gmax && 2ull * G * nsmall <= total) G <<= 1;
    // CTA b takes the contiguous run [N*b/grid, N*(b+1)/grid) of the list, so
    // consecutive rounds of a CTA evaluate colex-near sets whose subsets share
    // L1 lines (the list is a concatenation of warp runs of consecutive ranks)
    const unsigned long long c_lo = nsmall * blockIdx.x / gridDim.x, c_hi = nsmall * (blockIdx.x + 1) / gridDim.x;
    if (G == 1) {
        small_phase_thread<CLS, MEMO>(p, k, q, v, rtab, bin, gen, list, loc, c_lo, c_hi, pairs, nccp, nprobe, binp, emit,
                                      tm);
        return;
    }
    const unsigned int sub = tm.tid & (G - 1);
    const unsigned int gpc = tm.size / G;                    // groups per CTA (team)
    // groups in reverse thread order: with only a few sets per CTA the set and
    // the level-ahead expansion (forward order) land on different warps
    const unsigned int grp = gpc - 1 - tm.tid / G;
    for (unsigned long long base = c_lo; base < c_hi; base += gpc) {      // same trip count on every lane
        const unsigned long long e = base + grp;
        const bool act = e < c_hi;
        const unsigned long long ent = act ? __ldcs(list + loc(e)) : 0ull;
        const uint32_t S = (uint32_t)ent;
        const unsigned int R = (unsigned int)(ent >> 32);
        Key best = key_inf();
        unsigned long long w = 0;
        double cS = 0.0;
        if (act) {
            const int kind = set_kind<uint32_t, CLS>(q, S, k, w);
            cS = card_fast<CLS, MEMO>(p.memo, v, bin, q, S, k, R);
            PairSink<uint32_t, MEMO> sink;
            sink.init(&p.memo, gen, &v, rtab, &q, cS);
            const unsigned long long per = (w + G - 1) / G;
            unsigned long long j0 = per * sub, j1 = j0 + per;
            if (j0 > w) j0 = w;
            if (j1 > w) j1 = w;
            eval_range<uint32_t, CLS>(q, S, k, kind, j0, j1, sink, nccp);
            sink.flush();
            nprobe += sink.nprobe;
            best = sink.best;
        }
        best = group_min(best, G);
        if (act && sub == 0) {
            pairs += w;
            const unsigned long long idx = memo_slot_r<MEMO>(v, k, R, S);
            p.memo.dcost[idx] = __longlong_as_double((long long)best.c);
            __stcs(p.memo.dleft + idx, (unsigned int)best.l);
            p.memo.dcard[idx] = cS;
        }
    }
}

// ------------------------------------------------------------ clique levels
// Cliques with the bitmask memo: every k-subset is connected and is one
// complete block (Lemma 8), so set h of level k IS the colex rank h and
// its join pairs are j = 0 .. w-1 with w = 2^(k-1) - 1:
//     A_j = lowbit(S) | deposit(j, S \ lowbit(S)),   B_j = S \ A_j
// (Alg. mpdp_generalization P:545-568 with one block and no CCP checks).
// No enumeration, compaction, look-back or heavy list.  Two ways to cut a
// level (clique_group picks one from a cost model of the level's rounds):
//  * group path (most levels): whole sets per group of G = 1..32 lanes, G
//    minimising rounds x (pairs per lane + per-set overhead); lanes take
//    interleaved j so a group's probes fall into few memo lines;
//  * split path (levels of fewer sets than warps whose sets exceed 8192
//    pairs): the pair space [0, C(n,k) * w) is cut into one contiguous chunk
//    per warp (>= 512 pairs).  A set cut by chunk boundaries is merged from
//    per-chunk partial keys: a pair count on the slot of the first chunk that
//    touches it elects the last contributor, which reduces the partials and
//    scatters; the count slots alternate between two buffers by level parity
//    and each warp clears its slot of the next level's buffer.
// Memo entries of level 1 (leaf cost, card) are written at k = 2, so probes
// of levels >= 3 are branch-free loads.
template <int G>
__device__ __forceinline__ void clique_eval_span(const SQ<uint32_t>& q, const double* __restrict__ dcost, uint32_t S,
                                                 uint32_t lo, uint32_t R, uint32_t DG, uint32_t sub,
                                                 unsigned int j, unsigned int b, double cS, bool leaves, Key& best,
                                                 unsigned long long& npairs) {
    // pairs j, j + G, j + 2G, ... of the set (w < 2^31 pairs); 4 pairs (8
    // probes) in flight; the min in f64 / u32 registers (costs are >= 0, so
    // the f64 order is the bit order of the Key); every evaluated pair counted
    double bc = __longlong_as_double((long long)best.c);
    uint32_t bl = (uint32_t)best.l;
    unsigned int cnt = 0;
    for (; j < b; j += 4 * G) {
        uint32_t A[4];
        double ca[4], cb[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const bool ok = j + G * u < b;
            A[u] = lo | sub;
            const uint32_t B = S ^ A[u];
            if (leaves) {
                ca[u] = ok ? q.leaf[__ffs(A[u]) - 1] : 0.0;
                cb[u] = ok ? q.leaf[__ffs(B) - 1] : 0.0;
            } else {
                ca[u] = ok ? dcost[A[u]] : 0.0;
                cb[u] = ok ? dcost[B] : 0.0;
            }
            sub = ((sub | ~R) + DG) & R;
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const double c = __dadd_rn(__dadd_rn(ca[u], cb[u]), cS);
            const uint32_t B = S ^ A[u], l = A[u] < B ? A[u] : B;
            const bool ok = j + G * u < b;
            const bool better = ok && (c < bc || (c == bc && l < bl));
            bc = better ? c : bc;
            bl = better ? l : bl;
            cnt += ok;
        }
    }
    npairs += cnt;
    if (bl != 0xffffffffu) best = Key{(unsigned long long)__double_as_longlong(bc), (unsigned long long)bl};
}

// deposit(j, R) for j < 2^popc(R) without a bit loop over j: lowest five bits
// of j through R's lowest five elements, the rest as a masked add
__device__ __forceinline__ uint32_t deposit_small(unsigned int j, uint32_t R) {
    uint32_t out = 0;
    for (uint32_t T = R; j; T &= T - 1, j >>= 1)
        if (j & 1u) out |= T & (0u - T);
    return out;
}

__device__ __forceinline__ Key ld_key(const Key* k) {   // written by other SMs in this level: L2
    const unsigned long long* x = reinterpret_cast<const unsigned long long*>(k);
    return Key{__ldcg(x), __ldcg(x + 1)};
}

__device__ __forceinline__ void clique_write(const MemoPtrs& P, uint32_t S, const Key& best, double cS) {
    P.dcost[S] = __longlong_as_double((long long)best.c);
    __stcs(P.dleft + S, (unsigned int)best.l);
    P.dcard[S] = cS;
}

// Lanes per set for the whole-set group path.  A level of C sets of w pairs
// on T threads with G lanes per set takes ceil(C * G / T) rounds of w / G pairs
// per lane plus a per-set overhead (unrank, card, group min, scatter) worth
// about kCliqueSetCost pairs; G (a power of two up to 32, at most w + 1) minimises
// rounds * (w / G + kCliqueSetCost), ties to the smaller G.  Few lanes per set
// amortise the per-set work and keep a lane's consecutive pairs in nearby memo
// lines; more lanes fill the grid and shorten the level's last round.
// Returns 0 (pair chunks per warp, the split path) for levels of fewer sets
// than warps whose sets exceed split_w - 1 pairs (4096 on the kernel since
// round 2: clique-18 0.688 -> 0.674 ms, its level 14 of 3060 sets x 8191 pairs
// ran at 219 G pairs/s as one warp per set; 2048 ties, 16384 0.746 ms).  Measured (round 1, level barrier;
// clique-18 / 16 / 20): fixed ~8 pairs per lane 1.04 / 0.27 / 7.5 ms; <= 256
// pairs per lane widened to half the threads 0.72 / 0.28 / 4.9 ms; this model
// (cost 64) 0.66 / 0.29 / 3.9 ms (cost 32: 0.77 / 0.29 / 4.0; cost 128: 0.66 /
// 0.29 / 3.9).  Host and device share it (the host plans the dataflow chunks).
constexpr double kCliqueSetCost = 64.0;
__host__ __device__ inline unsigned int clique_group(unsigned long long w, unsigned long long C, unsigned long long T,
                                                     unsigned long long split_w = 8192,
                                                     double set_cost = kCliqueSetCost, double split_fac = 1.0) {
    if (w + 1 > split_w && 32.0 * (double)C < (double)T * split_fac) return 0;
    unsigned int best_g = 1;
    double best = 1e300;
    for (unsigned int G = 1; G <= 32 && G <= w + 1; G <<= 1) {
        const double cost = (double)((C * G + T - 1) / T) * ((double)(w + G - 1) / G + set_cost);
        if (cost < best) {
            best = cost;
            best_g = G;
        }
    }
    return best_g;
}

// Group path, one chunk: sets [lo, hi) of clique level k on the CTA's compute
// threads, G lanes per set, group-consecutive sets (the warp's groups work on
// colex neighbours, whose probes share lines).
// (XR, the fused peer exchange: M is this rank's replica, and every set is
// written into every replica, cost, card and left -- 20 B per set, 5 MB per
// replica at clique-18 -- so card(S \ max) and the extraction stay local)
template <bool XR>
__device__ __forceinline__ void clique_write_x(const MemoPtrs& M, const DfRank* x, uint32_t S, const Key& best,
                                               double cS) {
    if (!XR) {
        clique_write(M, S, best, cS);
        return;
    }
    const double c = __longlong_as_double((long long)best.c);
    for (int r = 0; r < x->W; r++) {
        x->xr->cost[r][S] = c;
        x->xr->left[r][S] = (unsigned int)best.l;
        x->xr->card[r][S] = cS;
    }
}

template <int G, bool XR = false>
__device__ void clique_group_chunk(const Params<uint32_t>& p, int k, const SQ<uint32_t>& q, const MemoView& v,
                                   const unsigned int* bin, unsigned int lo, unsigned int hi,
                                   unsigned long long& npairs, unsigned long long& nsets, const MemoPtrs& M,
                                   const DfRank* x = nullptr) {
    constexpr int MEMO = MEMO_MASK;
    constexpr unsigned int NG = kDfCompute / G;
    const unsigned int w = (1u << (k - 1)) - 1u;
    const bool leaves = k == 2;
    const unsigned int grp = threadIdx.x / G, sub = threadIdx.x & (G - 1);
    for (unsigned int h0 = lo; h0 < hi; h0 += NG) {           // uniform trip count
        const unsigned int h = h0 + grp;
        const bool act = h < hi;
        Key best = key_inf();
        double cS = 0.0;
        uint32_t S = 0;
        if (act) {
            S = unrank_colex32(bin, q.n, k, h);
            cS = card_fast<CLS_CLIQUE, MEMO>(M, v, bin, q, S, k, h);
            const uint32_t lo1 = S & (0u - S), R = S ^ lo1;
            clique_eval_span<G>(q, M.dcost, S, lo1, R, deposit_small(G, R), deposit_small(sub, R), sub, w, cS,
                                leaves, best, npairs);
        }
        best = group_min(best, G);
        if (act && sub == 0) {
            clique_write_x<XR>(M, x, S, best, cS);
            nsets++;
        }
    }
}

// Split path, one warp chunk c of level k: pairs [c * csize, (c+1) * csize) of
// the level's pair space C(n,k) * w.  A set cut by chunk boundaries is merged
// from per-chunk partial keys: a pair count on the slot of the first chunk
// that touches it elects the last contributor, which reduces the partials
// with its warp, scatters, and publishes the set (dataflow.cuh) -- no
// contended 128-bit CAS (clique-18 k = 18: ~100 chunks meet on one set).
// Merge slots: key_first / key_last / count per chunk of this level, from
// slot0 on (counts zeroed by the previous launch's last CTA or k_init).
__device__ void clique_split_chunk(const Params<uint32_t>& p, int k, const SQ<uint32_t>& q, const MemoView& v,
                                   const unsigned int* bin, const DfLevel& L, unsigned int c,
                                   unsigned long long& npairs, unsigned long long& nsets) {
    constexpr int MEMO = MEMO_MASK;
    const int n = q.n;
    const unsigned int lane = threadIdx.x & 31;
    const unsigned long long w = (1ull << (k - 1)) - 1;
    const unsigned long long P = (unsigned long long)bin[n * 33 + k] * w, csize = L.chunk;
    Key* key_first = p.bkey + 2ull * L.slot0;
    Key* key_last = key_first + L.nslot;
    unsigned long long* slot_done = p.bdone + L.slot0;
    const unsigned long long c0 = (unsigned long long)c * csize;
    if (c0 >= P) return;
    const unsigned long long c1 = c0 + csize < P ? c0 + csize : P;
    unsigned long long h = c0 / w, a = c0 - h * w;
    uint32_t S = unrank_colex32(bin, n, k, (unsigned int)h);
    while (true) {
        const unsigned long long hw = h * w;
        const unsigned long long b = c1 - hw < w ? c1 - hw : w;
        const double cS = card_fast<CLS_CLIQUE, MEMO>(p.memo, v, bin, q, S, k, (unsigned int)h);
        const uint32_t lo = S & (0u - S), R = S ^ lo;
        const uint32_t D32 = deposit_small(32, R);
        // deposit(a + lane) = deposit(a) (+) deposit(lane) in R's domain
        const uint32_t da = a ? deposit<uint32_t>(a, R) : 0u;
        const uint32_t sub = ((da | ~R) + deposit_small(lane, R)) & R;
        Key best = key_inf();
        clique_eval_span<32>(q, p.memo.dcost, S, lo, R, D32, sub, (unsigned int)(a + lane), (unsigned int)b, cS, false,
                             best, npairs);
        best = warp_min(best);
        bool wrote = false;
        if (a == 0 && b == w) {
            if (lane == 0) clique_write(p.memo, S, best, cS);
            wrote = true;
        } else {
            const bool is_first = h == c0 / w, is_last = hw + b >= c1;
            unsigned int last = 0;
            if (lane == 0) {
                if (is_first) key_first[c] = best;
                if (is_last) key_last[c] = best;
                __threadfence();
                const unsigned long long old = atomicAdd(&slot_done[hw / csize], b - a);
                last = old + (b - a) == w;
            }
            if (__shfl_sync(0xffffffffu, last, 0)) {
                __threadfence();
                const unsigned long long cf = hw / csize, cl = (hw + w - 1) / csize;
                Key m = key_inf();
                if (lane == 0) m = ld_key(&key_last[cf]);
                for (unsigned long long x = cf + 1 + lane; x <= cl; x += 32) {
                    const Key t = ld_key(&key_first[x]);
                    if (key_less(t, m)) m = t;
                }
                m = warp_min(m);
                if (lane == 0) clique_write(p.memo, S, m, cS);
                wrote = true;
            }
        }
        if (wrote && lane == 0) {          // publish the finished set (release: fence + add)
            nsets++;
            __threadfence();
            df_red_add(&p.df->done[k][31 - __clz(S)], 1u);
        }
        if (hw + b >= c1) break;
        h++;
        a = 0;
        S = gosper(S);
    }
}

#ifdef MPDP_TRACE
// per-CTA arrival time at each level's barrier (debug builds only)
constexpr int kCtaTraceMax = 1024;
constexpr int kCtaTraceSlots = 8;          // level start, sum enum, sum queue, sum eval, tiles, arrival
__device__ unsigned long long g_cta_arrive[(kMaxN + 1) * kCtaTraceMax * kCtaTraceSlots];
#define CT_NOW(var) unsigned long long var = (threadIdx.x == 0) ? globaltimer_ns() : 0ull
#else
#define CT_NOW(var)
#endif

template <int CLS, int MEMO = MEMO_DENSE>
__global__ void __launch_bounds__(kBlock, CLS == CLS_TREE ? 3 : 2) k_dp_fused(const __grid_constant__ Params<uint32_t> p) {
    using M = uint32_t;
    static_assert(MEMO != MEMO_HASH, "the whole-query kernels use the dense-layout memo");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SQ<M>& q = *reinterpret_cast<SQ<M>*>(smem_raw);
    unsigned int* rtab = reinterpret_cast<unsigned int*>(smem_raw + sizeof(SQ<M>));
    unsigned int* bin = rtab + p.memo.rg.entries;                  // 33 x 33 binomials
    uint32_t* qmask = bin + 33 * 33;                               // light-set queue
    unsigned int* qrank = qmask + kFusedTile;
    __shared__ MemoView v;
    __shared__ LevelDesc d;
    __shared__ unsigned long long s_next;
    __shared__ unsigned int s_small;
    unsigned long long* small_list = reinterpret_cast<unsigned long long*>(p.light);
    __shared__ Tri s_excl, s_agg;
    // heavy sets spanning many work items: their first_heavy ranges are filled
    // by the whole CTA after the queue barrier instead of by one thread (the
    // full cycle at cycle-20's top level spans 2048 items: 47 us of one thread)
    constexpr int kFhDefer = 32;
    __shared__ unsigned int s_fh_n;
    __shared__ unsigned long long s_fh_lo[kFhDefer], s_fh_hi[kFhDefer];
    __shared__ unsigned int s_fh_h[kFhDefer];
    if (threadIdx.x == 0) s_fh_n = 0;

    memo_prologue<M, MEMO>(p, p.n, q, v, rtab);
    if constexpr (CLS == CLS_GENERAL && sizeof(M) == 4) build_nbtab(q, p.q);   // byte-table BFS steps
    if constexpr (CLS == CLS_GENERAL && MEMO == MEMO_MASK) {
        if (threadIdx.x == 0 && p.memo_conn) q.mc = p.memo.dcost;               // reading R20
        // the singletons' slots hold their leaf costs, so the probe loops need
        // no singleton branch; written by every CTA before its first level (the
        // same values everywhere; a CTA's own probes follow its own writes)
        if (p.memo_conn)
            for (int u = threadIdx.x; u < p.n; u += blockDim.x) p.memo.dcost[1u << u] = p.q->leaf[u];
    }
    unsigned int nbar = 0;                 // grid barriers passed (thread 0)
    const unsigned int gen = p.q->gen;
    const int n = p.n;
    __syncthreads();
    const unsigned long long rmask = p.tiles_ring - 1;

#ifdef MPDP_TRACE
    int trace_i = 0;
#ifndef MPDP_TRACE_KMIN
#define MPDP_TRACE_KMIN 0
#endif
#define TRACE(tag) if (blockIdx.x == 0 && threadIdx.x == 0 && trace_i < kTraceCap && k >= MPDP_TRACE_KMIN) \
        p.result->trace[trace_i++] = (globaltimer_ns() << 8) | ((unsigned long long)k << 3) | (unsigned long long)(tag)
#else
#define TRACE(tag)
#endif
    for (int k = p.k_begin; k <= p.k_end; k++) {
        if (blockIdx.x == 0 && threadIdx.x == 0) p.result->t_level[k] = globaltimer_ns();
        TRACE(0);
#ifdef MPDP_TRACE
        CT_NOW(ct_lvl0);
        unsigned long long ct_enum = 0, ct_queue = 0, ct_eval = 0, ct_tiles = 0;
#endif
        // this launch evaluates the colex ranks [lo, hi) of level k (its share)
        const unsigned int lo = p.share_lo[k], r_hi = p.share_hi[k];
        const unsigned int nranks = r_hi - lo;
        const bool counting = (p.count_levels >> k) & 1ull;
        const bool heavy_level = CLS != CLS_TREE && ((p.heavy_levels >> k) & 1ull);
        // Tiles.  Small levels are spread over the whole grid (1..8 ranks per
        // thread) so no CTA serialises a level's evaluation.  Heavy levels
        // interleave tiles statically over CTAs so the look-back chain stays
        // short.  Other levels hand out tiles dynamically: CTA b starts with
        // tile b, then claims the next tile from a per-level counter; the claim
        // for the next tile is issued at the START of the current one, so its
        // latency hides behind the tile.  Static equal chunks are unbalanced
        // because the density of connected sets varies along colex order (star:
        // the sets with maximum element j contain the hub with probability
        // (k-1)/j).  (Guided self-scheduling with shrinking chunks measured
        // slower: the per-tile enumeration overhead outweighs the better tail.)
        unsigned int rpt = (nranks + gridDim.x * blockDim.x - 1) / (gridDim.x * blockDim.x);
        rpt = rpt < 1 ? 1 : (rpt > kFusedRanksPerThread ? kFusedRanksPerThread : rpt);
        const unsigned int tile_ranks = rpt * blockDim.x;
        const unsigned long long ntiles = (nranks + tile_ranks - 1) / tile_ranks;
        const unsigned long long item = p.item_of[k];
        const unsigned long long epoch = lookback_epoch(p, k);
        unsigned long long pairs = 0, nccp = 0, nprobe = 0, nlight = 0;
        const unsigned long long dyn_base = (unsigned long long)gridDim.x * tile_ranks;

        unsigned long long tile = blockIdx.x;                  // heavy levels: tile index
        unsigned long long t0 = tile * tile_ranks;             // first rank (offset from lo) of this tile
        while (t0 < nranks) {
            unsigned long long next_t0 = t0 + dyn_base;
            if (!heavy_level && threadIdx.x == 0 && nranks > dyn_base)
                next_t0 = dyn_base + atomicAdd(&p.desc[k].tile_ticket, tile_ranks);   // consumed at the end
            TRACE(1);
#ifdef MPDP_TRACE
            CT_NOW(ct_a);
#endif

            // ---- unrank + filter + classify (registers only)
            const unsigned int r0 = lo + (unsigned int)t0 + threadIdx.x * rpt;
            M S0 = 0;
            unsigned int lflag = 0, hflag = 0, kinds = 0;   // kinds: 2 bits per rank (set_kind once)
            M cuts[kFusedRanksPerThread];      // general graphs: cut vertices of each rank's set (R21)
            M blk0[kHeavyBlk];                 // the blocks of rank slot 0's set (most levels: one rank
            int nb0 = -1;                      // per thread), reused by the heavy-list write
            Tri mine = {0, 0, 0};
            if (r0 < r_hi) {
                S0 = unrank_colex32(bin, n, k, r0);
                M S = S0;
#pragma unroll
                for (int i = 0; i < kFusedRanksPerThread; i++) {
                    if (i < (int)rpt && r0 + i < r_hi) {
                        if (connected_cls<M, CLS>(q, S, k)) {
                            unsigned long long w;
                            cuts[i] = 0;
                            const int kind = (CLS == CLS_GENERAL && i == 0)
                                                 ? set_kind<M, CLS>(q, S, k, w, blk0, &nb0, &cuts[i])
                                                 : set_kind<M, CLS>(q, S, k, w, nullptr, nullptr, &cuts[i]);
                            kinds |= (unsigned int)kind << (2 * i);
                            // (general graphs: only sets without CCP checks,
                            // or with few candidates, are evaluated by one thread)
                            if (w <= kLightMax && (CLS != CLS_GENERAL || w <= p.light_max || kind == KIND_TREE ||
                                                   kind == KIND_COMPLETE)) {
                                lflag |= 1u << i;
                            } else {
                                hflag |= 1u << i;
                                mine.w += w;
                            }
                        }
                        if (i + 1 < (int)rpt && r0 + i + 1 < r_hi) S = gosper(S);
                    }
                }
            }
            mine.l = __popc(lflag);
            mine.h = __popc(hflag);
            TRACE(2);
#ifdef MPDP_TRACE
            CT_NOW(ct_b);
            ct_enum += ct_b - ct_a;
#endif

            // ---- block scan; global look-back only where heavy sets can exist
            Tri agg;
            const Tri ex = block_scan(mine, agg);
            if (heavy_level) {
                if (threadIdx.x < 32) {
                    const Tri excl = lookback(p.tiles, rmask, tile, epoch, agg, &p.result->error);
                    if (threadIdx.x == 0) {
                        s_excl = excl;
                        s_agg = agg;
                    }
                }
                __syncthreads();
                if (threadIdx.x == 0 && tile == ntiles - 1) {   // level totals of the heavy list
                    LevelDesc& dk = p.desc[k];
                    const unsigned long long H = s_excl.h + s_agg.h, W = s_excl.w + s_agg.w;
                    dk.n_heavy = H;
                    dk.heavy_pairs = W;
                    dk.n_items = (W + item - 1) / item;
                    if (dk.n_items > p.fh_cap || H > p.heavy_cap) atomicOr(&p.result->error, ERR_CAPACITY);
                    if (H < p.heavy_cap + 1) p.wh[H] = W;
                    dk.n_buckets = 1;
                }
            }
            const Tri excl = heavy_level ? s_excl : Tri{0, 0, 0};

            // ---- light sets -> CTA queue (slot = colex rank), except the last
            // nq mod blockDim (all of them when nq < blockDim), which go to the
            // grid-wide small list so that every local round keeps all threads
            // busy; heavy sets -> global list
            const unsigned int nq = (unsigned int)agg.l;
            const unsigned int ndef = kDeferRemainder ? nq % blockDim.x : (nq < blockDim.x ? nq : 0u);
            const unsigned int nloc = nq - ndef;
            if (ndef) {
                if (threadIdx.x == 0) s_small = atomicAdd(&p.desc[k].n_small, ndef);
                __syncthreads();
            }
            if (lflag | hflag) {
                unsigned int li = (unsigned int)ex.l;
                unsigned long long hi = excl.h + ex.h, wi = excl.w + ex.w;
                M S = S0;
#pragma unroll
                for (int i = 0; i < kFusedRanksPerThread; i++) {
                    if ((lflag >> i) & 1) {
                        if (li < nloc) {
                            qmask[li] = S;
                            // (memo connectivity implies MEMO_MASK, whose slots
                            // ignore the rank: bits 30-31 carry the set kind)
                            qrank[li] = (CLS == CLS_GENERAL && q.mc) ? (r0 + i) | (((kinds >> (2 * i)) & 3u) << 30)
                                                                     : r0 + i;
                        } else {
                            const unsigned long long d = s_small + (li - nloc);
                            if (d < p.list_cap)
                                small_list[d] = ((unsigned long long)(r0 + i) << 32) | S;
                            else
                                atomicOr(&p.result->error, ERR_CAPACITY);
                        }
                        li++;
                    }
                    if ((hflag >> i) & 1) {
                        unsigned long long w;
                        if (CLS == CLS_GENERAL && q.mc) {
                            M blk[kHeavyBlk];
                            int nb = 0;
                            const int kind = (int)((kinds >> (2 * i)) & 3u);
                            if (i == 0 && kind == KIND_BLOCKS && nb0 >= 0 && nb0 <= kHeavyBlk && !q.dpsub) {
                                nb = nb0;              // found by the classification above
                                w = 0;
                                for (int b = 0; b < nb; b++) {
                                    blk[b] = blk0[b];
                                    w += (1ull << (popc(blk0[b]) - 1)) - 1;
                                }
                            } else {
                                w = kind_pairs<M, CLS>(q, S, k, kind, blk, &nb, cuts[i]);
                            }
                            if (hi < p.heavy_cap) {
                                p.hinfo[hi] = (unsigned int)kind | ((unsigned int)nb << 2);
                                for (int b = 0; b < nb && b < kHeavyBlk; b++) p.hblk[hi * kHeavyBlk + b] = blk[b];
                                p.hcard[hi] = card_of(q, S);   // here, not in a phase of its own
                            }
                        } else {
                            set_kind<M, CLS>(q, S, k, w);
                        }
                        if (hi < p.heavy_cap) {
                            p.heavy[hi] = S;
                            p.wh[hi] = wi;
                            p.bkey[hi] = key_inf();
                            p.bdone[hi] = 0;
                            const unsigned long long it0 = (wi + item - 1) / item, it1 = (wi + w - 1) / item;
                            unsigned int slot = kFhDefer;
                            if (it1 >= it0 + 16) slot = atomicAdd(&s_fh_n, 1u);
                            if (slot < kFhDefer) {
                                s_fh_lo[slot] = it0;
                                s_fh_hi[slot] = it1;
                                s_fh_h[slot] = (unsigned int)hi;
                            } else {
                                for (unsigned long long it = it0; it <= it1; it++)
                                    if (it < p.fh_cap) p.first_heavy[it] = (unsigned int)hi;
                            }
                        }
                        wi += w;
                        hi++;
                    }
                    if (r0 + i + 1 < r_hi && i + 1 < (int)rpt) S = gosper(S);
                }
            }
            __syncthreads();
            if (s_fh_n) {                      // the deferred first_heavy ranges, CTA-wide
                const unsigned int nd = s_fh_n < kFhDefer ? s_fh_n : kFhDefer;
                for (unsigned int e = 0; e < nd; e++)
                    for (unsigned long long it = s_fh_lo[e] + threadIdx.x; it <= s_fh_hi[e]; it += blockDim.x)
                        if (it < p.fh_cap) p.first_heavy[it] = s_fh_h[e];
                __syncthreads();
                if (threadIdx.x == 0) s_fh_n = 0;
            }

            TRACE(3);
#ifdef MPDP_TRACE
            CT_NOW(ct_c);
            ct_queue += ct_c - ct_b;
#endif
            // ---- evaluate the tile's local light sets, thread per set
            for (unsigned int e = threadIdx.x; e < nloc; e += blockDim.x) {
                const M S = qmask[e];
                unsigned long long w;
                int kind;
                if (CLS == CLS_GENERAL && q.mc) {
                    kind = (int)(qrank[e] >> 30);
                    w = kind_pairs<M, CLS>(q, S, k, kind);
                } else {
                    kind = set_kind<M, CLS>(q, S, k, w);
                }
                pairs += w;
                if constexpr (CLS == CLS_TREE && MEMO == MEMO_DENSE) {
                    if (k > 2) {
                        eval_tree_dense<MEMO>(p.memo, gen, v, rtab, bin, q, S, k, qrank[e], nprobe);
                        nccp += w;
                        continue;
                    }
                }
                PairSink<M, MEMO> sink;
                sink.init(&p.memo, gen, &v, rtab, &q, card_of(q, S));
                eval_range<M, CLS>(q, S, k, kind, 0, w, sink, nccp);
                sink.flush();
                nprobe += sink.nprobe;
                const unsigned long long idx = memo_slot_r<MEMO>(v, k, qrank[e], S);
                p.memo.dcost[idx] = __longlong_as_double((long long)sink.best.c);
                __stcs(p.memo.dleft + idx, (unsigned int)sink.best.l);
                p.memo.dcard[idx] = sink.cS;
            }
            if (threadIdx.x == 0) {
                nlight += nq;
                s_next = next_t0;
            }
            __syncthreads();                   // queue and scan scratch reused next tile
            t0 = s_next;
            tile += gridDim.x;
            TRACE(4);
#ifdef MPDP_TRACE
            CT_NOW(ct_d);
            ct_eval += ct_d - ct_c;
            ct_tiles++;
#endif
        }
        if (counting) {
            if (threadIdx.x == 0 && nlight) atomicAdd(&p.desc[k].n_light, nlight);
            flush_counters(&p.desc[k], pairs, nccp, nprobe);
        }
        TRACE(5);
#ifdef MPDP_TRACE
        if (threadIdx.x == 0 && blockIdx.x < kCtaTraceMax) {
            unsigned long long* o = g_cta_arrive + ((unsigned long long)k * kCtaTraceMax + blockIdx.x) * kCtaTraceSlots;
            o[0] = ct_lvl0;
            o[1] = ct_enum;
            o[2] = ct_queue;
            o[3] = ct_eval;
            o[4] = ct_tiles;
            o[5] = globaltimer_ns();
        }
#endif
        grid_sync(p.gbar, nbar, &p.result->error);
        TRACE(6);

        // deferred light sets (small list) and, on heavy levels, heavy-set cards
        // share the window after the level barrier: both read levels < k only
        if (threadIdx.x == 0) d = p.desc[k];
        __syncthreads();
        const unsigned long long nsmall = d.n_small < p.list_cap ? d.n_small : p.list_cap;
        unsigned long long sp = 0, sc = 0, spr = 0;
#ifdef MPDP_TRACE
        CT_NOW(ct_s0);
#endif
        if (nsmall) small_phase<CLS, MEMO>(p, k, q, v, rtab, bin, gen, small_list, DenseLocate{}, nsmall, sp, sc, spr);
#ifdef MPDP_TRACE
        if (threadIdx.x == 0 && blockIdx.x < kCtaTraceMax) {
            unsigned long long* o = g_cta_arrive + ((unsigned long long)k * kCtaTraceMax + blockIdx.x) * kCtaTraceSlots;
            o[6] = globaltimer_ns() - ct_s0;
            o[7] = nsmall;
        }
#endif
        // (a heavy level that found no heavy set -- sparse general graphs --
        // skips the heavy phase and its barrier: d is grid-uniform here)
        if (CLS != CLS_TREE && heavy_level && d.n_heavy > 0) {
            // card(S) of every heavy set once (one thread per set); general
            // graphs with memo connectivity wrote it with the heavy list
            if (!(CLS == CLS_GENERAL && q.mc)) {
                const unsigned long long nh = d.n_heavy < p.heavy_cap ? d.n_heavy : p.heavy_cap;
                const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
                for (unsigned long long h = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; h < nh; h += stride)
                    p.hcard[h] = card_of(q, p.heavy[h]);
                grid_sync(p.gbar, nbar, &p.result->error);
            }
            TRACE(7);
            heavy_phase<M, CLS, MEMO>(p, k, item, q, v, rtab, gen, d, sp, sc, spr);
            TRACE(7);
            if (counting) flush_counters(&p.desc[k], sp, sc, spr);
            grid_sync(p.gbar, nbar, &p.result->error);
        } else if (nsmall) {
            if (counting) flush_counters(&p.desc[k], sp, sc, spr);
            grid_sync(p.gbar, nbar, &p.result->error);
        }
    }
    if (p.do_extract && blockIdx.x == 0 && threadIdx.x < 32) {
        if (threadIdx.x == 0) p.result->t_level[n + 1] = globaltimer_ns();
        level_counters_warp(p, p.result);
        if (threadIdx.x == 0) extract_phase<M, MEMO>(p, q, v, rtab, gen);
    }
}

template <int G>
__device__ void clique_groups(const Params<uint32_t>& p, int k, const SQ<uint32_t>& q, const MemoView& v,
                              const unsigned int* bin, unsigned int C, unsigned long long w,
                              unsigned long long probes_per_set, bool leaves, unsigned long long& pairs,
                              unsigned long long& nccp, unsigned long long& nprobe, unsigned long long& nsets) {
    constexpr int MEMO = MEMO_MASK;
    const unsigned long long nthreads = (unsigned long long)gridDim.x * blockDim.x;
    const unsigned long long gtid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned long long ngroups = nthreads / G, grp = gtid / G;
    const unsigned int sub = threadIdx.x & (G - 1);
    // group-consecutive sets (h = it * ngroups + grp), each one unranked: the
    // warp's groups work on colex neighbours, whose probes share lines
    // (per-group Gosper runs: clique-16 316 vs 291 us)
    const unsigned long long rounds = (C + ngroups - 1) / ngroups;
    uint32_t S = 0;
    for (unsigned long long it = 0; it < rounds; it++) {
        const unsigned long long h = it * ngroups + grp;
        const bool act = h < C;
        if (act) S = unrank_colex32(bin, q.n, k, (unsigned int)h);
        Key best = key_inf();
        double cS = 0.0;
        if (act) {
            cS = card_fast<CLS_CLIQUE, MEMO>(p.memo, v, bin, q, S, k, (unsigned int)h);
            const uint32_t lo = S & (0u - S), R = S ^ lo;
            clique_eval_span<G>(q, p.memo.dcost, S, lo, R, deposit_small(G, R), deposit_small(sub, R), sub,
                                (unsigned int)w, cS, leaves, best, pairs);
        }
        best = group_min(best, G);
        if (act && sub == 0) {
            clique_write(p.memo, S, best, cS);
            nprobe += probes_per_set;
            nsets++;
        }
    }
}

__device__ void clique_level(const Params<uint32_t>& p, int k, const SQ<uint32_t>& q, const MemoView& v,
                             const unsigned int* bin, unsigned long long& pairs, unsigned long long& nccp,
                             unsigned long long& nprobe, unsigned long long& nsets) {
    constexpr int MEMO = MEMO_MASK;
    const int n = q.n;
    const unsigned int C = bin[n * 33 + k];
    const unsigned long long w = (1ull << (k - 1)) - 1;
    const unsigned long long probes_per_set = k >= 3 ? 2 * w - (unsigned long long)k : 0ull;
    const unsigned int lane = threadIdx.x & 31;
    const unsigned long long nthreads = (unsigned long long)gridDim.x * blockDim.x;
    const unsigned long long gtid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned long long nwarps = nthreads >> 5, gw = gtid >> 5;
    Key* key_first = p.bkey;               // per chunk: key of its first / last set segment
    Key* key_last = p.bkey + nwarps;
    unsigned long long* slot_done = p.bdone + (k & 1) * nwarps;
    if (lane == 0) p.bdone[((k + 1) & 1) * nwarps + gw] = 0;   // this warp's counter slot of level k+1
    const bool leaves = k == 2;
    if (leaves && gtid < (unsigned long long)n) {      // level-1 entries
        p.memo.dcost[1u << gtid] = q.leaf[gtid];
        p.memo.dcard[1u << gtid] = q.card[gtid];
    }
    // whole sets per group of G lanes (clique_group), or pair chunks per warp
    const unsigned int G = clique_group(w, C, nthreads, p.clique_split_w, p.clique_set_cost, p.clique_split_fac);
    (void)nccp;                            // every evaluated pair is a ccp (Lemma 8): counted as pairs
    if (G) {
        switch (G) {
            case 1: clique_groups<1>(p, k, q, v, bin, C, w, probes_per_set, leaves, pairs, nccp, nprobe, nsets); break;
            case 2: clique_groups<2>(p, k, q, v, bin, C, w, probes_per_set, leaves, pairs, nccp, nprobe, nsets); break;
            case 4: clique_groups<4>(p, k, q, v, bin, C, w, probes_per_set, leaves, pairs, nccp, nprobe, nsets); break;
            case 8: clique_groups<8>(p, k, q, v, bin, C, w, probes_per_set, leaves, pairs, nccp, nprobe, nsets); break;
            case 16: clique_groups<16>(p, k, q, v, bin, C, w, probes_per_set, leaves, pairs, nccp, nprobe, nsets); break;
            default: clique_groups<32>(p, k, q, v, bin, C, w, probes_per_set, leaves, pairs, nccp, nprobe, nsets); break;
        }
        return;
    }
    const unsigned long long P = (unsigned long long)C * w;
    unsigned long long csize = (P + nwarps - 1) / nwarps;
    if (csize < p.clique_csize_min) csize = p.clique_csize_min;   // 512 (1024: clique-16 291 vs 278 us)
    const unsigned long long c0 = gw * csize;
    if (c0 >= P) return;
    const unsigned long long c1 = c0 + csize < P ? c0 + csize : P;
    unsigned long long h = c0 / w, a = c0 - h * w;
    uint32_t S = unrank_colex32(bin, n, k, (unsigned int)h);
    while (true) {
        const unsigned long long hw = h * w;
        const unsigned long long b = c1 - hw < w ? c1 - hw : w;
        const double cS = card_fast<CLS_CLIQUE, MEMO>(p.memo, v, bin, q, S, k, (unsigned int)h);
        const uint32_t lo = S & (0u - S), R = S ^ lo;
        const uint32_t D32 = deposit_small(32, R);
        // deposit(a + lane) = deposit(a) (+) deposit(lane) in R's domain
        const uint32_t da = a ? deposit<uint32_t>(a, R) : 0u;
        const uint32_t sub = ((da | ~R) + deposit_small(lane, R)) & R;
        Key best = key_inf();
        clique_eval_span<32>(q, p.memo.dcost, S, lo, R, D32, sub, (unsigned int)(a + lane), (unsigned int)b, cS, false,
                             best, pairs);
        best = warp_min(best);
        if (a == 0 && b == w) {
            if (lane == 0) {
                clique_write(p.memo, S, best, cS);
                nprobe += probes_per_set;
                nsets++;
            }
        } else {
            // split set: this chunk's partial key goes to its first / last
            // segment slot (plain stores); the pair count on the slot of the
            // first chunk touching the set elects the last contributor, which
            // reduces the partial keys of all chunks of the set with its warp
            // (no contended 128-bit CAS: 128 chunks meet at clique-18 k = 18)
            const bool is_first = h == c0 / w, is_last = hw + b >= c1;
            unsigned int last = 0;
            if (lane == 0) {
                if (is_first) key_first[gw] = best;
                if (is_last) key_last[gw] = best;
                __threadfence();
                const unsigned long long old = atomicAdd(&slot_done[hw / csize], b - a);
                last = old + (b - a) == w;
            }
            if (__shfl_sync(0xffffffffu, last, 0)) {
                __threadfence();
                const unsigned long long cf = hw / csize, cl = (hw + w - 1) / csize;
                Key m = key_inf();
                if (lane == 0) m = ld_key(&key_last[cf]);
                for (unsigned long long c = cf + 1 + lane; c <= cl; c += 32) {
                    const Key t = ld_key(&key_first[c]);
                    if (key_less(t, m)) m = t;
                }
                m = warp_min(m);
                if (lane == 0) {
                    clique_write(p.memo, S, m, cS);
                    nprobe += probes_per_set;
                    nsets++;
                }
            }
        }
        if (hw + b >= c1) break;
        h++;
        a = 0;
        S = gosper(S);
    }
}


// Dataflow variant of the clique kernel (ablation, MPDP_DEBUG_CLIQUE_DF):
// levels as dataflow chunks (dataflow.cuh): group levels hand whole sets to groups of G lanes,
// split levels hand warp chunks of one level's pair space; the first small
// levels run as one solo chunk.  A chunk of level k needs level k-1 up to the
// largest element of its last set.  Plan extraction by the last CTA out.
constexpr int kCliqueMinBlocks = 3;
__host__ __device__ constexpr size_t clique_smem_bytes() { return sizeof(SQ<uint32_t>) + sizeof(unsigned int) * 33 * 33; }

template <bool XR = false>
struct CliqueSched {
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
        if (L.split) {                                  // warp chunks [lo, hi) of the level
            d.lo = (t - L.base) * (kDfCompute / 32);
            d.hi = min(d.lo + kDfCompute / 32, L.nslot);
        } else {
            d.lo = p.share_lo[k] + (t - L.base) * L.chunk;
            d.hi = min(d.lo + L.chunk, p.share_hi[k]);
        }
    }
    // largest element of the last set the chunk touches
    __device__ unsigned int last_set(const DfSlot& d) const {
        const DfLevel& L = p.dfl[d.k];
        if (!L.split) return d.hi - 1;
        const unsigned long long w = (1ull << (d.k - 1)) - 1;
        const unsigned long long P = (unsigned long long)bin[p.n * 33 + d.k] * w;
        const unsigned long long e = min((unsigned long long)d.hi * L.chunk, P);
        return (unsigned int)((e - 1) / w);
    }
    __device__ int need(const DfSlot& d) const {
        return (d.k >= 3 && d.k - 1 >= p.k_begin) ? colex_top(bin, d.k, last_set(d)) : -1;
    }
    // sets of level k1 whose largest element is j
    __device__ unsigned int need_count(int k1, int j) const { return bin[j * 33 + k1 - 1]; }
    __device__ void publish(const DfSlot& d) const {
        if (p.dfl[d.k].split) return;                   // split sets are published by their last contributor
        DataflowDev* const ldf = XR ? x.df : p.df;
        df_publish_colex<XR>(x, ldf, bin, d.k, d.k, d.lo, d.hi);
        for (int k = d.k + 1; k <= d.k2; k++) df_publish_colex<XR>(x, ldf, bin, k, k, p.share_lo[k], p.share_hi[k]);
    }
};

__device__ __noinline__ void clique_extract(const Params<uint32_t>& p, const SQ<uint32_t>& q, const MemoView& v,
                                            const unsigned int* bin) {
    if (threadIdx.x == 0) p.result->t_level[p.n + 1] = globaltimer_ns();
    level_counters_warp(p, p.result);
    if (threadIdx.x == 0) {
        if (ld_relaxed_u32(&p.df->error)) {
            p.result->n_nodes = 0;
        } else {
            p.result->error = 0;
            extract_phase<uint32_t, MEMO_MASK>(p, q, v, bin, p.q->gen);
        }
        atomicMax(&p.df->t_done[p.n + 1], globaltimer_ns());
    }
}

// The extraction from this rank's replica (fused exchange): the same code on a
// copy of the parameters that points at the replica, its descriptors and result.
__device__ __noinline__ void clique_extract_x(const Params<uint32_t>& p, const SQ<uint32_t>& q, const MemoView& v,
                                              const unsigned int* bin, const DfRank& x, const MemoPtrs& M) {
    if (threadIdx.x == 0) x.result->t_level[p.n + 1] = globaltimer_ns();
    level_counters_warp(p, x.result, x.desc);
    if (threadIdx.x == 0) {
        if (ld_relaxed_u32(&x.df->error)) {
            x.result->n_nodes = 0;
        } else {
            x.result->error = 0;
            extract_phase_m<uint32_t, MEMO_MASK>(M, x.result, p.n, q, v, bin, p.q->gen);
        }
        atomicMax(&x.df->t_done[p.n + 1], globaltimer_ns());
    }
}

template <bool XR>
__global__ void __launch_bounds__(kDfThreads, kCliqueMinBlocks) k_dp_clique_df(const __grid_constant__ Params<uint32_t> p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SQ<uint32_t>& q = *reinterpret_cast<SQ<uint32_t>*>(smem_raw);
    unsigned int* bin = reinterpret_cast<unsigned int*>(smem_raw + sizeof(SQ<uint32_t>));   // 33 x 33
    __shared__ MemoView v;
    __shared__ DfCounters sc;
    __shared__ DfShared sh;
    __shared__ DfRank xr;
    __shared__ MemoPtrs xm;                // this rank's replica (XR) or the launch's memo
    if (threadIdx.x == 0) {
        df_rank_init(xr, p);
        xm = p.memo;
        if (XR) {
            xm.dcost = xr.dcost;
            xm.dcard = xr.dcard;
            xm.dleft = xr.dleft;
            df_start_barrier(p, xr);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) p.result->t_level[0] = globaltimer_ns();   // kernel start
    load_query(q, p.q);
    for (int j = threadIdx.x; j <= kMaxN; j += blockDim.x) {
        v.off[j] = 0;
        v.nb[j] = 0;
        sh.ready[j] = j < p.k_begin ? 64 : -1;
    }
    for (int i = threadIdx.x; i < (kMaxN + 1) * 3; i += blockDim.x) (&sc.v[0][0])[i] = 0;
    if (threadIdx.x < kDfSlots) sh.done[threadIdx.x] = 0;
    constexpr int NB = MaxN<uint32_t>::value + 1;
    for (int i = threadIdx.x; i < 33 * 33; i += blockDim.x) {
        const int a = i / 33, b = i % 33;
        bin[i] = (a < NB && b < NB) ? (unsigned int)p.q->binom[a * NB + b] : 0u;
    }
    // level-1 entries (leaf cost, card), written by every CTA before its first
    // chunk: the same values everywhere, and a CTA's own later probes are
    // ordered after its own writes
    __syncthreads();
    for (int u = threadIdx.x; u < q.n; u += blockDim.x) {
        xm.dcost[1u << u] = q.leaf[u];
        xm.dcard[1u << u] = q.card[u];
    }
    __syncthreads();
    if (threadIdx.x >= kDfCompute) {
        df_control<XR>(p, CliqueSched<XR>{p, bin, xr}, sh, xr);
    } else {
        int kc = p.k_begin;
        unsigned long long npairs = 0, nsets = 0;      // this thread, level kc
        auto flush = [&]() {
            // probes of non-singleton sides: 2w - k per set of a level >= 3
            const unsigned long long wk = (1ull << (kc - 1)) - 1;
            df_count(sc, kc, npairs, kc >= 3 ? nsets * (2 * wk - (unsigned long long)kc) : 0ull, nsets);
            npairs = nsets = 0;
        };
        DfSlot d;
        unsigned long long st_take = 0;
        const unsigned long long st0 = p.df_stats ? globaltimer_ns() : 0ull;
        unsigned long long* stp = (p.df_stats && threadIdx.x == 0) ? &st_take : nullptr;
        for (unsigned int i = 0; df_take(sh, i, d, stp); i++) {
            for (int k = d.k; k <= d.k2; k++) {
                if (k != kc) {
                    flush();
                    kc = k;
                }
                if (k > d.k) {
                    asm volatile("bar.sync 3, %0;" ::"r"(kDfCompute) : "memory");
                    if (threadIdx.x == 0) xr.result->t_level[k] = globaltimer_ns();
                }
                const DfLevel& L = p.dfl[k];
                if (!XR && L.split) {             // (the fused exchange plans no split levels)
                    const unsigned int c = d.lo + (threadIdx.x >> 5);
                    if (c < d.hi) clique_split_chunk(p, k, q, v, bin, L, c, npairs, nsets);
                    continue;
                }
                const unsigned int lo = k == d.k ? d.lo : p.share_lo[k], hi = k == d.k ? d.hi : p.share_hi[k];
                switch (L.G) {
                    case 1: clique_group_chunk<1, XR>(p, k, q, v, bin, lo, hi, npairs, nsets, xm, &xr); break;
                    case 2: clique_group_chunk<2, XR>(p, k, q, v, bin, lo, hi, npairs, nsets, xm, &xr); break;
                    case 4: clique_group_chunk<4, XR>(p, k, q, v, bin, lo, hi, npairs, nsets, xm, &xr); break;
                    case 8: clique_group_chunk<8, XR>(p, k, q, v, bin, lo, hi, npairs, nsets, xm, &xr); break;
                    case 16: clique_group_chunk<16, XR>(p, k, q, v, bin, lo, hi, npairs, nsets, xm, &xr); break;
                    default: clique_group_chunk<32, XR>(p, k, q, v, bin, lo, hi, npairs, nsets, xm, &xr); break;
                }
            }
            df_finish(sh, i);
        }
        if (stp) {
            p.df_stats[8ull * blockIdx.x + 4] = st_take;
            p.df_stats[8ull * blockIdx.x + 5] = globaltimer_ns() - st0;
        }
        flush();
    }
    if (!df_exit<XR>(p, sc, xr)) return;
    if (p.do_extract && threadIdx.x < 32) {
        if (XR) clique_extract_x(p, q, v, bin, xr, xm);
        else clique_extract(p, q, v, bin);
    }
    df_reset(p, xr);
}

// Whole-query kernel for cliques with the bitmask memo: clique_level per level
// (one phase, one grid barrier), then the extraction.  A kernel of its own so
// its register budget (and so its occupancy: kCliqueMinBlocks CTAs per SM) is
// not set by the tile machinery of k_dp_fused.  The level barrier stays here:
// the dataflow variant (k_dp_clique_df) measured slower on cliques -- 72% of
// clique-18's level k+1 needs ALL of level k (every set with the largest
// element), so only the short colex prefix can overlap a level's tail, and
// the per-chunk handover costs more than the barrier saves.

__global__ void __launch_bounds__(kBlock, kCliqueMinBlocks) k_dp_clique(const __grid_constant__ Params<uint32_t> p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SQ<uint32_t>& q = *reinterpret_cast<SQ<uint32_t>*>(smem_raw);
    unsigned int* bin = reinterpret_cast<unsigned int*>(smem_raw + sizeof(SQ<uint32_t>));   // 33 x 33
    __shared__ MemoView v;
    load_query(q, p.q);
    for (int j = threadIdx.x; j <= kMaxN; j += blockDim.x) {
        v.off[j] = 0;
        v.nb[j] = 0;
    }
    constexpr int NB = MaxN<uint32_t>::value + 1;
    for (int i = threadIdx.x; i < 33 * 33; i += blockDim.x) {
        const int a = i / 33, b = i % 33;
        bin[i] = (a < NB && b < NB) ? (unsigned int)p.q->binom[a * NB + b] : 0u;
    }
    unsigned int nbar = 0;
    __shared__ unsigned int s_abort;
    const unsigned long long t_start = globaltimer_ns();
    __syncthreads();
    for (int k = p.k_begin; k <= p.k_end; k++) {
        if (blockIdx.x == 0 && threadIdx.x == 0) p.result->t_level[k] = globaltimer_ns();
        unsigned long long pairs = 0, nccp = 0, nprobe = 0, nsets = 0;
        clique_level(p, k, q, v, bin, pairs, nccp, nprobe, nsets);
        if ((p.count_levels >> k) & 1ull) {
            flush_counters(&p.desc[k], pairs, pairs, nprobe, nsets);   // (pairs evaluated = ccp, Lemma 8)
        }
        // device deadline: a CTA past it raises the abort flag before
        // the barrier; after the barrier every CTA reads the same flag
        if (threadIdx.x == 0 && p.timeout_ns && globaltimer_ns() - t_start > p.timeout_ns)
            atomicExch(&p.df->abort, 1u);
        grid_sync(p.gbar, nbar, &p.result->error);
        if (threadIdx.x == 0) s_abort = ld_relaxed_u32(&p.df->abort);
        __syncthreads();
        if (s_abort) {
            if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&p.result->error, ERR_TIMEOUT);
            return;
        }
    }
    if (p.do_extract && blockIdx.x == 0 && threadIdx.x < 32) {
        if (threadIdx.x == 0) p.result->t_level[p.n + 1] = globaltimer_ns();
        level_counters_warp(p, p.result);
        if (threadIdx.x == 0) extract_phase<uint32_t, MEMO_MASK>(p, q, v, bin, p.q->gen);
    }
}

}  // namespace mpdp
