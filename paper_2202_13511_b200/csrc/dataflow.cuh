// dataflow.cuh — barrier-free level scheduling for the closed-form
// whole-query kernels (k_dp_star, k_dp_clique).
//
// Alg. mpdp_gpu runs the levels k = 2..n in order because a set of
// size k reads only the memo entries of its subsets, i.e. of levels < k
// (the sets of one level are independent).  It needs
// no more order than that: in colex order the k-subsets whose largest element
// is <= m are a PREFIX of level k (ranks < C(m+1, k)), and every subset of
// such a set lies in the same prefix of its own level.  So instead of a grid
// barrier per level, the launch is one queue of chunks (level-major, colex
// order inside a level) claimed from an atomic ticket, and a chunk of level k
// waits only until level k-1 is finished up to the largest element m of its
// last set:
//     done[k-1][j] == (number of sets of level k-1 with largest element j)
// for j <= m.  Levels below k-1 are finished up to m as well (transitively: a
// level-(k-1) set with largest element j waited for level k-2 up to j before
// it was evaluated).  The tail of level k overlaps the start of level k+1, and
// the small levels at both ends cost one chunk each instead of a grid barrier.
//
// Deadlock freedom: a chunk depends only on chunks with smaller tickets;
// tickets are claimed in order by co-resident CTAs (cooperative launch), each
// CTA holds at most one unfinished chunk, so the smallest unfinished ticket
// always runs.
//
// CTA shape: 8 compute warps and one control warp (df_control).  The control
// warp claims tickets, waits for dependencies, hands chunks over through two
// shared slots and publishes finished chunks; the compute warps only compute.
//
// Memory order: a chunk's memo entries are written by the compute warps, each
// releases at cta scope (done counter in shared memory); the control lane
// acquires them, fences at gpu scope and adds to done[k][m] (release
// pattern).  A waiting control lane polls done[k-1][.] with relaxed loads and
// then issues ONE fence.acq_rel.gpu (acquire pattern; it also invalidates the
// SM's L1, whose lines may hold entries of the level that were unwritten when
// the line was loaded); the chunk is then handed over through a named
// barrier (bar.arrive / bar.sync order the compute warps after it).
#pragma once
#include "level_kernels.cuh"

namespace mpdp {

__device__ __forceinline__ unsigned int df_ld_relaxed(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void df_red_add(unsigned int* p, unsigned int v) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void df_fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// The rank view of a CTA (shared memory, written by thread 0 before the first
// __syncthreads): which rank it works for and that rank's replica.  Without an
// XrTable there is one rank and the replica is the launch's own state.
struct DfRank {
    int W, r;                              // ranks, this CTA's rank
    unsigned int nctas, cta;               // CTAs of this rank, this CTA's index among them
    DataflowDev* df;                       // the rank's replica: dataflow state, descriptors, result,
    ResultDev* result;                     // memo arrays
    LevelDesc* desc;
    double* dcost;
    double* dcard;
    unsigned int* dleft;
    const XrTable* xr;
    // every replica (XR: the fused exchange is compiled in; otherwise W == 1)
    template <bool XR> __device__ int ranks() const { return XR ? W : 1; }
    template <bool XR> __device__ DataflowDev* dfs(int s) const { return XR ? xr->df[s] : df; }
    template <bool XR> __device__ LevelDesc* descs(int s) const { return XR ? xr->desc[s] : desc; }
    template <bool XR> __device__ double* costs(int s) const { return XR ? xr->cost[s] : dcost; }
};
__device__ __forceinline__ void df_rank_init(DfRank& x, const Params<uint32_t>& p) {
    if (p.xr) {
        const XrTable& t = *p.xr;
        x.W = t.W;
        x.r = t.emulate ? (int)(blockIdx.x % (unsigned int)t.W) : t.rank;
        x.nctas = t.emulate ? (gridDim.x - (unsigned int)x.r + (unsigned int)t.W - 1) / (unsigned int)t.W : gridDim.x;
        x.cta = t.emulate ? blockIdx.x / (unsigned int)t.W : blockIdx.x;
        x.df = t.df[x.r];
        x.result = t.result[x.r];
        x.desc = t.desc[x.r];
        x.dcost = t.cost[x.r];
        x.dcard = t.card[x.r];
        x.dleft = t.left[x.r];
        x.xr = p.xr;
    } else {
        x.W = 1;
        x.r = 0;
        x.nctas = gridDim.x;
        x.cta = blockIdx.x;
        x.df = p.df;
        x.result = p.result;
        x.desc = p.desc;
        x.dcost = p.memo.dcost;
        x.dcard = p.memo.dcard;
        x.dleft = p.memo.dleft;
        x.xr = nullptr;
    }
}
// Across ranks (peer memory) the synchronisation is at system scope.
template <bool XR>
__device__ __forceinline__ void df_red_add_x(unsigned int* p, unsigned int v) {
    if (XR) asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
    else asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
template <bool XR>
__device__ __forceinline__ unsigned int df_ld_relaxed_x(const unsigned int* p) {
    unsigned int v;
    if (XR) asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    else asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
template <bool XR>
__device__ __forceinline__ void df_fence_rel_x() {
    if (XR) __threadfence_system();
    else __threadfence();
}
template <bool XR>
__device__ __forceinline__ void df_fence_acq_x() {
    if (XR) asm volatile("fence.acq_rel.sys;" ::: "memory");
    else asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
// an abort pushes a rank's ticket counter here: local ticket u maps to the
// global ticket u * W + r, which then lies past every chunk
constexpr unsigned int kDfAbortTicket = 0x08000000u;

// largest element of the colex-rank-r j-subset (j >= 1): the largest c with
// C(c, j) <= r.  bin: 33 x 33 binomials (u32) in shared memory.
__device__ __forceinline__ int colex_top(const unsigned int* bin, int j, unsigned int r) {
    int c = j - 1;                                         // C(j-1, j) = 0 <= r
    while (c < 31 && bin[(c + 1) * 33 + j] <= r) c++;
    return c;
}

// One lane (the control warp's, after acquiring the chunk's memo writes and
// a gpu-scope fence): publish sets [lo, hi) of level k -- colex ranks of
// j-subsets, j = elements per set in the rank space -- per largest element.
// Every replica's counters (fused exchange: the other ranks' through peer memory).
// (ldf: the local dataflow state, p.df for one rank -- the constant bank, not
// the shared-memory view)
template <bool XR>
__device__ __forceinline__ void df_publish_colex(const DfRank& x, DataflowDev* ldf, const unsigned int* bin, int k,
                                                 int j, unsigned int lo, unsigned int hi) {
    const int ma = colex_top(bin, j, lo), mb = colex_top(bin, j, hi - 1);
    for (int m = ma; m <= mb; m++) {
        const unsigned int a = lo > bin[m * 33 + j] ? lo : bin[m * 33 + j];
        const unsigned int e = bin[(m + 1) * 33 + j];
        const unsigned int b = hi < e ? hi : e;
        if (XR)
            for (int s = 0; s < x.W; s++) df_red_add_x<XR>(&x.xr->df[s]->done[k][m], b - a);
        else
            df_red_add_x<XR>(&ldf->done[k][m], b - a);
    }
}

__device__ __forceinline__ unsigned int df_ld_acquire_cta(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"((unsigned int)__cvta_generic_to_shared(p)) : "memory");
    return v;
}
__device__ __forceinline__ void df_add_release_cta(unsigned int* p, unsigned int v) {
    asm volatile("red.release.cta.shared.add.u32 [%0], %1;" ::"r"((unsigned int)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}
// Stop the launch: flag the error, and push the ticket counter past every
// ticket so that no CTA claims another chunk.
template <bool XR>
__device__ __forceinline__ void df_abort(const DfRank& x, unsigned int err) {
    atomicOr(&x.df->error, err);
    for (int s = 0; s < x.ranks<XR>(); s++) atomicExch_system(&x.dfs<XR>(s)->abort, 1u);
    atomicMax(&x.df->ticket, kDfAbortTicket);
}

// ---------------------------------------------------------------------------
// Warp-specialised CTA: kDfCompute threads (8 warps) evaluate chunks, one
// control warp claims tickets, waits for each chunk's dependency, hands the
// chunk over in one of two shared slots (named barrier 1 + slot: the control
// warp arrives, the compute warps sync) and publishes finished chunks (fence
// + relaxed adds).  The compute warps never wait for a ticket claim, a
// dependency poll or a fence while the next chunk is ready.  All 8 compute
// warps take part in each chunk together (the handover barrier), so a chunk
// finishes -- and its dependants can start -- as early as possible and the
// CTA's warps share L1 lines.  (Measured alternatives, star-25 / clique-18:
// CTA-wide barriers around every chunk 0.797 / -- ms; warps decoupled through
// a ring of 2-4 posted slots 0.79-1.07 / 0.84 ms -- chunks complete later, so
// more of the claimed chunks wait on dependencies; this scheme 0.73 / 0.79.)
constexpr int kDfCompute = kBlock;
constexpr int kDfThreads = kBlock + 32;
constexpr int kDfSlots = 2;

struct DfSlot {
    unsigned int t;                        // ticket; ~0u: no more chunks
    int k, k2;                             // levels k..k2 (k2 > k: a solo chunk of whole small levels)
    unsigned int lo, hi;                   // sets [lo, hi) of level k (split levels: warp chunks)
};

struct DfShared {
    DfSlot slot[kDfSlots];
    unsigned int done[kDfSlots];           // compute warps finished with the slot's chunk
    int ready[kMaxN + 1];                  // control: level j known finished up to largest element ready[j]
};

// named barriers 1 / 2 (slot 0 / 1) with compile-time ids (a run-time id makes
// ptxas reserve all 16 barriers of the CTA)
__device__ __forceinline__ void df_bar_sync(int s) {
    if (s == 0) asm volatile("bar.sync 1, %0;" ::"r"(kDfThreads) : "memory");
    else asm volatile("bar.sync 2, %0;" ::"r"(kDfThreads) : "memory");
}
__device__ __forceinline__ void df_bar_arrive(int s) {
    if (s == 0) asm volatile("bar.arrive 1, %0;" ::"r"(kDfThreads) : "memory");
    else asm volatile("bar.arrive 2, %0;" ::"r"(kDfThreads) : "memory");
}

// Compute warps: the next chunk (blocks until the control warp hands it over);
// false when the launch has no more chunks for this CTA.
__device__ __forceinline__ bool df_take(DfShared& sh, unsigned int i, DfSlot& d, unsigned long long* stats = nullptr) {
    const unsigned long long w = stats ? globaltimer_ns() : 0ull;
    df_bar_sync(i & 1);
    if (stats) *stats += globaltimer_ns() - w;
    d = sh.slot[i & 1];
    return d.t != ~0u;
}
// Compute warps, every lane: chunk i finished by this warp (its memo writes
// are ordered before the cta-scope release by __syncwarp).
__device__ __forceinline__ void df_finish(DfShared& sh, unsigned int i) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) df_add_release_cta(&sh.done[i & 1], 1u);
}

// The control warp.  Sched: total(), locate(t, DfSlot&), need(const DfSlot&)
// = largest element of level k-1 the chunk needs (-1: none), need_count(k1, j)
// = sets of level k1 with largest element j, publish(const DfSlot&) (after the
// chunk's writes are acquired and fenced).  Lane 0 works; the whole warp
// arrives at the handover barriers.
template <bool XR, typename P, typename Sched>
__device__ void df_control(const P& p, const Sched& S, DfShared& sh, const DfRank& x) {
    const unsigned int lane = threadIdx.x & 31;
    const unsigned long long t0 = globaltimer_ns();   // timeout origin: this CTA's start
    const unsigned int total = S.total();
    constexpr unsigned int kWarps = kDfCompute / 32;
    DfSlot fly0, fly1;                     // lane 0: chunk in flight per slot (t == ~0u: none)
    fly0.t = fly1.t = ~0u;
    unsigned long long w0 = 0;             // watchdog origin of the current wait
    unsigned int t = 0;
    DataflowDev* const ldf = XR ? x.df : p.df;   // registers, not the shared view
    ResultDev* const lres = XR ? x.result : p.result;
    // this rank's chunks: local ticket u is global ticket u * W + r
    auto claim = [&]() -> unsigned int {
        const unsigned int u = atomicAdd(&ldf->ticket, 1u);
        if (!XR) return u;
        return u >= kDfAbortTicket ? ~0u : u * (unsigned int)x.W + (unsigned int)x.r;
    };
    if (lane == 0) t = claim();
    unsigned long long st_slot = 0, st_dep = 0, st_n = 0;   // MPDP_DEBUG_DF_STATS
    // publish a finished chunk in flight (lane 0); true if slot s is free
    auto retire = [&](int s) -> bool {
        DfSlot& f = s ? fly1 : fly0;
        if (f.t == ~0u) return true;
        if (df_ld_acquire_cta(&sh.done[s]) < kWarps) return false;
        df_fence_rel_x<XR>();              // release the CTA's memo writes (every replica)
        S.publish(f);
        const unsigned long long now = globaltimer_ns();
        for (int k = f.k; k <= f.k2; k++) atomicMax(&ldf->t_done[k], now);
        sh.done[s] = 0;
        f.t = ~0u;
        return true;
    };
    // watchdog / timeout while polling (lane 0)
    unsigned int spins = 0;
    auto stalled = [&]() -> bool {
        if (++spins > 64) __nanosleep(32);         // spin hot first: most waits are short
        if ((spins & 63u) != 0) return false;
        if (df_ld_relaxed_x<XR>(&ldf->abort)) return true;
        if (p.timeout_ns && globaltimer_ns() - t0 > p.timeout_ns) {
            df_abort<XR>(x, ERR_TIMEOUT);
            return true;
        }
        const unsigned long long now = globaltimer_ns();
        if (!w0) w0 = now;
        if (now - w0 > 2000000000ull) {    // never hang the device
            df_abort<XR>(x, ERR_HANG);
            return true;
        }
        return false;
    };
    for (unsigned int i = 0;; i++) {
        const int s = i & 1;
        DfSlot d;
        d.t = ~0u;
        if (lane == 0) {
            w0 = 0;
            spins = 0;
            const unsigned long long ts0 = p.df_stats ? globaltimer_ns() : 0ull;
            while (!retire(s)) {           // slot s: chunk i-2 must be finished
                retire(s ^ 1);
                if (stalled()) break;
            }
            const unsigned long long ts1 = p.df_stats ? globaltimer_ns() : 0ull;
            st_slot += ts1 - ts0;
            bool go = t < total;
            unsigned int nxt = 0;
            if (go) {
                S.locate(t, d);
                const int m = S.need(d);
                const int k1 = d.k - 1;
                if (m > sh.ready[k1]) {    // level k-1 up to largest element m
                    w0 = 0;
                    spins = 0;
                    for (int j = sh.ready[k1] + 1; j <= m && go; j++) {
                        const unsigned int want = S.need_count(k1, j);
                        while (df_ld_relaxed_x<XR>(&ldf->done[k1][j]) < want) {
                            retire(s ^ 1);     // our own previous chunk may be what we wait for
                            if (stalled()) {
                                go = false;
                                break;
                            }
                        }
                    }
                    if (go) {
                        df_fence_acq_x<XR>();  // acquire (+ L1 invalidation) once per advance
                        sh.ready[k1] = m;
                    }
                    if (p.df_stats) st_dep += globaltimer_ns() - ts1;
                }
                if (go && p.timeout_ns && globaltimer_ns() - t0 > p.timeout_ns) {
                    df_abort<XR>(x, ERR_TIMEOUT);
                    go = false;
                }
                // claim ahead, after the acquire fence (which would wait for
                // the claim); its latency hides behind this chunk.  An abort
                // pushes the counter past every ticket, so the claim sees it.
                if (go) nxt = claim();
            }
            if (!go) d.t = ~0u;
            else if (t == p.dfl[d.k].base) lres->t_level[d.k] = globaltimer_ns();
            sh.slot[s] = d;
            (s ? fly1 : fly0) = d;
            t = nxt;
            st_n++;
        }
        __syncwarp();
        df_bar_arrive(s);
        if (__shfl_sync(0xffffffffu, d.t, 0) == ~0u) break;
    }
    if (lane == 0) {                       // drain: the chunk still in flight
        w0 = 0;
        spins = 0;
        while (!(retire(0) & retire(1)))
            if (stalled()) break;
        if (p.df_stats) {
            unsigned long long* o = p.df_stats + 8ull * blockIdx.x;
            o[0] = st_slot;
            o[1] = st_dep;
            o[2] = globaltimer_ns() - t0;
            o[3] = st_n;
        }
    }
    __syncwarp();
}

// Per-CTA level counters (shared memory), flushed once when the CTA exits.
struct DfCounters {
    unsigned long long v[kMaxN + 1][3];    // pairs (= ccp on stars / cliques), probes, sets
};

__device__ __forceinline__ void df_count(DfCounters& sc, int k, unsigned long long pairs, unsigned long long probes,
                                         unsigned long long sets) {
    pairs = warp_sum(pairs);
    probes = warp_sum(probes);
    sets = warp_sum(sets);
    if ((threadIdx.x & 31) == 0) {
        if (pairs) atomicAdd(&sc.v[k][0], pairs);
        if (probes) atomicAdd(&sc.v[k][1], probes);
        if (sets) atomicAdd(&sc.v[k][2], sets);
    }
}

// Every CTA at exit: flush its counters into the level descriptors (they
// accumulate over the launches of a sharded query); returns true in the last
// CTA out (after an acquire fence: every chunk of the launch is finished and
// visible).
// With several ranks every CTA adds its counters to every replica's
// descriptors and then counts itself in every replica's `flushed`; the last
// CTA of a rank waits until all CTAs of all ranks have flushed into its
// replica -- each flushed after its last chunk was published to every
// replica, so the replica is then complete -- before it extracts.
template <bool XR, typename P>
__device__ bool df_exit(const P& p, DfCounters& sc, const DfRank& x) {
    __syncthreads();
    for (int j = threadIdx.x; j <= p.n; j += blockDim.x) {
        if (!((p.count_levels >> j) & 1ull)) continue;
        for (int s = 0; s < x.ranks<XR>(); s++) {
            LevelDesc& d = x.descs<XR>(s)[j];
            if (sc.v[j][0]) {
                atomicAdd_system(&d.pairs, sc.v[j][0]);
                atomicAdd_system(&d.ccp, sc.v[j][0]);
            }
            if (sc.v[j][1]) atomicAdd_system(&d.probes, sc.v[j][1]);
            if (sc.v[j][2]) atomicAdd_system(&d.n_light, sc.v[j][2]);
        }
    }
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        df_fence_rel_x<XR>();
        if (XR)
            for (int s = 0; s < x.W; s++) df_red_add_x<XR>(&x.dfs<XR>(s)->flushed, 1u);
        s_last = atomicAdd(&x.df->exited, 1u) == x.nctas - 1;
        if (XR && s_last) {
            const unsigned long long w0 = globaltimer_ns();
            while (df_ld_relaxed_x<XR>(&x.df->flushed) < x.xr->ctas_total) {
                if (globaltimer_ns() - w0 > 4000000000ull) {   // never hang the device
                    atomicOr(&x.df->error, ERR_HANG);
                    break;
                }
                __nanosleep(64);
            }
        }
        if (s_last) df_fence_acq_x<XR>();
    }
    __syncthreads();
    return s_last;
}

// The last CTA out, all threads, after the extraction (which read the level
// descriptors): hand the error bits and level finish times to the result and
// return the launch state to zero for the next launch.  Descriptors, errors and
// finish times are kept across the level launches of a sharded query and
// cleared by the launch that extracts.
template <typename P>
__device__ void df_reset(const P& p, const DfRank& x) {
    __syncthreads();
    DataflowDev& df = *x.df;
    if (p.do_extract) {
        if (threadIdx.x == 0) x.result->error = df.error;
        for (int j = threadIdx.x; j < kMaxN + 2; j += blockDim.x) {
            x.result->t_done[j] = df.t_done[j];
            df.t_done[j] = 0;
        }
        for (int j = threadIdx.x; j <= p.n; j += blockDim.x) x.desc[j] = LevelDesc{};
        __syncthreads();
        if (threadIdx.x == 0) df.error = 0;
    }
    for (int i = threadIdx.x; i < (kMaxN + 1) * kDfMaxElem; i += blockDim.x) (&df.done[0][0])[i] = 0;
    if (!p.xr)
        for (unsigned long long i = threadIdx.x; i < p.zero_words; i += blockDim.x) p.bdone[i] = 0;   // merge counts
    if (threadIdx.x == 0) {
        df.ticket = 0;
        df.exited = 0;
        df.abort = 0;
        df.flushed = 0;
    }
}

// Start of a query with several ranks: no rank may store into a peer's
// replica before that peer has finished the previous query (its extraction
// reads the replica, its reset clears the counters).  The first CTA of each
// rank counts the rank in every replica's `epoch`; every CTA then waits for
// W * query arrivals in its own replica.  Thread 0.
template <typename P>
__device__ void df_start_barrier(const P& p, const DfRank& x) {
    if (x.cta == 0)
        for (int s = 0; s < x.W; s++) df_red_add_x<true>(&x.dfs<true>(s)->epoch, 1u);
    const unsigned int want = (unsigned int)x.W * p.xr_epoch;
    const unsigned long long w0 = globaltimer_ns();
    while ((int)(df_ld_relaxed_x<true>(&x.df->epoch) - want) < 0) {
        if (globaltimer_ns() - w0 > 4000000000ull) {
            df_abort<true>(x, ERR_HANG);
            break;
        }
        __nanosleep(64);
    }
    df_fence_acq_x<true>();
}

}  // namespace mpdp
