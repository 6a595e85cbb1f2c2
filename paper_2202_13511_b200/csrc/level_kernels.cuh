// level_kernels.cuh — the per-level kernels of the MPDP dynamic program
// (Alg. mpdp_gpu) for sm_100a.
//
//   k_enum<M,CLS>          unrank (colex + Gosper) -> connectivity
//                          filter (grow from the lowest vertex) ->
//                          set kind + join-pair count -> stream compaction into a
//                          light list (<= 32 pairs: thread per set) and a heavy
//                          list, single-pass decoupled look-back scan.
//   k_eval_light/heavy     evaluate MPDP's join pairs (Alg.
//                          mpdp_generalization P:531-579), C_out cost
//                          from memo probes, per-set min (prune fused into
//                          evaluate), scatter into the memo.
//   k_extract<M,MEMO>      plan extraction from the memo + counters.
#pragma once
#include "memo.cuh"
#include "../../include/mpdp.h"

namespace mpdp {

struct __align__(16) LevelDesc {
    unsigned long long n_light, n_heavy;   // compacted connected sets
    unsigned long long heavy_pairs;        // sum of heavy-set pair counts
    unsigned long long n_items;            // heavy work items of `item` pairs
    unsigned long long pairs, ccp;         // counters (R3, R2)
    unsigned long long probes;             // memo probes of non-singleton sets
    unsigned long long bucket_off, n_buckets;   // HASH: this level's table
    unsigned int tile_ticket, work_ticket;
    unsigned int n_small;                  // fused: light sets deferred to the grid-wide small list
    unsigned int seg;                      // list kernel: per-CTA segment size of this level's list
};

struct __align__(64) TileRec {            // decoupled look-back record (ring slot)
    unsigned long long flag;               // tile << 28 | epoch26 << 2 | state (1 aggregate, 2 inclusive)
    unsigned long long agg_l, agg_h, agg_w;
    unsigned long long inc_l, inc_h, inc_w, pad;
};

constexpr int kTraceCap = 512;
constexpr int kMaxGrid = 2048;            // CTAs of a persistent whole-query kernel

// Barrier-free level scheduling of the closed-form whole-query kernels
// (k_dp_star, k_dp_clique; dataflow.cuh).  The sets of one level are
// independent and level k reads only levels < k; in
// colex order the sets whose largest element is <= m are a prefix of every
// level, and all subsets of such a set lie in those prefixes.  So a chunk of
// level k can start as soon as level k-1 is finished up to the largest
// element of the chunk's last set -- no grid barrier between levels.
constexpr int kDfMaxElem = 32;
// Self-resetting: all zero between launches (the workspace is zeroed at
// context creation and by k_init; the last CTA out of a dataflow launch
// zeroes it again), so the dataflow kernels need no init launch.
struct DataflowDev {
    unsigned int ticket;                   // next chunk of the launch (level-major, colex order)
    unsigned int exited;                   // CTAs that ran out of chunks (the last one extracts)
    unsigned int abort;                    // timeout / watchdog: stop claiming and waiting
    unsigned int error;                    // ERR_* bits, kept until the extracting launch copies them
    unsigned long long t_done[kMaxN + 2];  // per level: when its last chunk finished (idem)
    unsigned int done[kMaxN + 1][kDfMaxElem];   // finished sets per (level, largest element)
    // fused peer exchange (XrTable): CTAs of every rank that flushed their
    // counters into this replica, and the start-of-query arrivals (monotonic,
    // never reset: W per query)
    unsigned int flushed;
    unsigned int epoch;
};

struct ResultDev;
// Fused exchange over peer memory: W ranks, each with a full
// replica of the star memo.  A rank's chunks store their costs into EVERY
// replica (NVLink peer stores) and add their completion counts to every
// replica's done counters, so no level ends in a collective: a chunk of level
// k waits, in its own replica, for exactly the sets of level k-1 it reads,
// whichever rank wrote them.  In emulation (one GPU) the ranks are the CTA
// groups blockIdx % W of one cooperative launch and the replicas are shards
// of one workspace; across GPUs the pointers of the other ranks are peer
// mappings (cudaIpcOpenMemHandle) and every rank launches its own kernel.
constexpr int kMaxXr = 8;
struct XrTable {
    int W;                                 // ranks
    int emulate;                           // 1: rank of a CTA = blockIdx.x % W (one launch)
    int rank;                              // (emulate = 0) this process's rank
    unsigned int ctas_total;               // CTAs over all ranks (counter flushes per replica)
    double* cost[kMaxXr];                  // every replica's arrays (peer pointers but [rank])
    double* card[kMaxXr];
    unsigned int* left[kMaxXr];
    DataflowDev* df[kMaxXr];
    LevelDesc* desc[kMaxXr];
    ResultDev* result[kMaxXr];
};
struct DfLevel {
    unsigned int base;                     // first ticket of the level (dfl[k_end + 1].base = total)
    unsigned int chunk;                    // sets per ticket, or (split) pairs per warp chunk
    unsigned int slot0;                    // split levels: first merge slot of the level
    unsigned int nslot;                    // split levels: warp chunks (merge slots) of the level
    unsigned char G, run, split;           // lanes per set, consecutive sets per group, split mode
    unsigned char solo;                    // > k: levels k..solo are ONE chunk (small levels, one CTA)
};

struct ResultDev {
    double cost;
    unsigned long long csg, ccp, pairs, probes;
    unsigned int n_nodes, error;
    unsigned long long lvl_csg[kMaxN + 1], lvl_ccp[kMaxN + 1], lvl_pairs[kMaxN + 1];
    unsigned long long t_level[kMaxN + 2];  // fused kernel: globaltimer at each level start (+ end)
    unsigned long long t_done[kMaxN + 2];   // dataflow kernels: globaltimer when the level's last chunk finished
    unsigned long long trace[kTraceCap];    // MPDP_TRACE builds: (ns << 8 | level << 3 | phase) of block 0
    mpdp_plan_node nodes[2 * kMaxN - 1];
};

template <typename M> struct Params {
    const QueryDev<M>* q;
    LevelDesc* desc;                       // [kMaxN + 1], indexed by subset size
    MemoPtrs memo;
    unsigned long long dense_off[kMaxN + 1];   // DENSE: first entry of level j
    M* light;                              // compacted level lists (reused per level)
    M* heavy;
    unsigned long long* wh;                // [heavy_cap + 1] exclusive heavy pair prefix
    Key* bkey;                             // [heavy_cap] cross-warp (cost, left) min
    double* hcard;                         // [heavy_cap] card(S) of heavy sets (computed once)
    // general graphs with memo connectivity (q.mc): per heavy set its kind |
    // (number of blocks << 2), and its first kHeavyBlk blocks (KIND_BLOCKS),
    // written with the heavy list so work items skip set_kind / Find-Blocks
    unsigned int* hinfo;                   // [heavy_cap]
    M* hblk;                               // [heavy_cap * kHeavyBlk]
    unsigned long long* bdone;             // [heavy_cap] pairs merged so far
    unsigned int* first_heavy;             // [fh_cap] heavy set holding item i's first pair
    unsigned long long fh_cap;
    TileRec* tiles;                        // ring of look-back records
    unsigned long long tiles_ring;         // power of two
    unsigned long long list_cap;           // light list capacity
    unsigned long long heavy_cap;          // heavy list capacity
    ResultDev* result;
    unsigned int* gbar;                    // whole-query kernels: grid barrier arrival counter
    unsigned int* seg_cnt;                 // list kernel: [2][kMaxGrid] per-CTA level-list counts
    unsigned long long heavy_levels;       // bit k: level k can have heavy sets
    unsigned long long item_of[kMaxN + 1]; // heavy work-item size per level
    // fused kernel, multi-GPU sharding: levels [k_begin, k_end]
    // of this launch, the colex-rank share [share_lo, share_hi) of each level
    // this rank evaluates, which levels it counts, and whether it extracts
    int k_begin, k_end, do_extract, epoch_salt;   // salt: shard index (look-back epochs)
    unsigned long long count_levels;
    unsigned int share_lo[kMaxN + 1], share_hi[kMaxN + 1];
    int n;
    int memo_kind;                         // MEMO_HASH / MEMO_DENSE / MEMO_MASK
    double inv_load;                       // HASH: buckets = ceil(count * inv_load / 2)
    int no_ccc;                            // MPDP_FLAG_NO_CCC: lane-contiguous candidates (ablation)
    int star_hub;                          // k_dp_star: the hub relation
    unsigned long long star_off[kMaxN + 1];   // k_dp_star: first memo entry of level k (C(n-1, k-1) per level)
    // dataflow scheduling (k_dp_star, k_dp_clique): per level its tickets and
    // chunk geometry, the shared state, and the timeout (0 = none)
    DataflowDev* df;
    const XrTable* xr;                     // k_dp_star: fused peer exchange (null: one rank)
    unsigned int xr_epoch;                 // this query's index (start-of-query barrier of the ranks)
    DfLevel dfl[kMaxN + 2];
    unsigned long long timeout_ns;
    unsigned long long zero_words;         // k_init: bdone[0 .. zero_words) cleared (clique merge counts)
    int mask_leaves;                       // k_init: level-1 entries of the bitmask memo (cliques)
    unsigned long long* df_stats;          // debug (MPDP_DEBUG_DF_STATS): per CTA 8 timing words, else null
    // sharded runs (multi-GPU, §8): only the memo COSTS are exchanged; card(S)
    // is recomputed locally (reading R5's fold) and the chosen split of a
    // plan node is re-derived at extraction from the replicated costs
    int shard_local;
    // general graphs: sets with more join-pair candidates than this go to the
    // warp-parallel heavy phase (CCC) instead of one thread (light)
    unsigned int light_max;
    // heavy phase: sets of at most this many pairs are evaluated whole by the
    // warp whose claim holds their first pair (no cross-warp merge); larger
    // sets are cut at the claim boundaries and merged
    unsigned long long heavy_whole;
    // tree list kernel: the next level is generated from this one (sparse
    // expansion) when expand_fac x sets x (n - k) candidates <= C(n, k+1) ranks
    double expand_fac;
    // general graphs on the bitmask memo: the cost array was filled with
    // kMemoAbsent at staging, so connectivity checks may probe it (reading R20)
    int memo_conn;
    unsigned long long clique_split_w;     // k_dp_clique: split levels whose sets exceed this many pairs + 1
    double clique_set_cost;                // k_dp_clique: per-set overhead of the group cost model, in pairs
    double clique_split_fac;               // k_dp_clique: split levels of fewer than fac x (warps) sets
    unsigned long long clique_csize_min;   // k_dp_clique: smallest warp chunk of the split path, in pairs
};

// ------------------------------------------------------------- mem helpers
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ------------------------------------------------------------ pair sink
// Collects the join pairs (A, B) of one set and evaluates them NP at a time:
// cost = (cost(A) + cost(B)) + card(S) (C_out; no FMA, reading R6),
// keeping the lexicographic (cost, min(A, B)) minimum (reading R7).
template <typename M, int MEMO>
struct PairSink {
    static constexpr int NP = (MEMO != MEMO_HASH) ? 4 : 2;
    static constexpr bool kChk = true;     // supports chk (reading R20)
    const MemoPtrs* P;                     // kernel parameter space
    const MemoView* v;
    const unsigned int* rtab;
    const SQ<M>* q;
    unsigned int gen;
    M A[NP], B[NP];
    int cnt;
    double cS;
    Key best;
    unsigned long long nprobe;
    // reading R20: with chk set, a pair (A, B) counts (nvalid) and competes only
    // when both probes found their set, i.e. both sides are connected
    bool chk;
    unsigned long long nvalid;

    __device__ __forceinline__ void init(const MemoPtrs* P_, unsigned int gen_, const MemoView* v_,
                                         const unsigned int* rt, const SQ<M>* q_, double card) {
        P = P_;
        gen = gen_;
        v = v_;
        rtab = rt;
        q = q_;
        cnt = 0;
        cS = card;
        best = key_inf();
        nprobe = 0;
        chk = false;
        nvalid = 0;
    }
    __device__ __forceinline__ void flush() {
        if (!cnt) return;
        M X[2 * NP];
        unsigned valid = 0;
#pragma unroll
        for (int u = 0; u < NP; u++) {
            X[2 * u] = A[u];
            X[2 * u + 1] = B[u];
            if (u < cnt) valid |= 3u << (2 * u);
        }
        double c[2 * NP];
        memo_lookup<M, MEMO, 2 * NP>(*P, gen, *v, rtab, *q, X, valid, c, nprobe);
#pragma unroll
        for (int u = 0; u < NP; u++) {
            if (u < cnt) {
                if (chk) {
                    if (!memo_present(c[2 * u]) || !memo_present(c[2 * u + 1])) continue;
                    nvalid++;
                }
                const double x = __dadd_rn(__dadd_rn(c[2 * u], c[2 * u + 1]), cS);
                const Key key{(unsigned long long)__double_as_longlong(x),
                              (unsigned long long)(A[u] < B[u] ? A[u] : B[u])};
                if (key_less(key, best)) best = key;
            }
        }
        cnt = 0;
    }
    __device__ __forceinline__ void add(M a, M b) {
#pragma unroll
        for (int u = NP - 1; u > 0; u--) {
            A[u] = A[u - 1];
            B[u] = B[u - 1];
        }
        A[0] = a;
        B[0] = b;
        if (++cnt == NP) flush();
    }
};

// ------------------------------------------------------------ k_init
template <typename M>
__global__ void k_init(const __grid_constant__ Params<M> p) {
    for (int i = threadIdx.x; i <= kMaxN; i += blockDim.x) {
        LevelDesc d = {};
        p.desc[i] = d;
    }
    if (threadIdx.x == 0) {
        p.result->error = 0;
        if (p.gbar) p.gbar[0] = 0;         // grid barrier arrival counter of the next launch
    }
    for (int i = threadIdx.x; i < kMaxN + 2; i += blockDim.x) p.result->t_level[i] = p.result->t_done[i] = 0;
    for (int i = threadIdx.x; i < kTraceCap; i += blockDim.x) p.result->trace[i] = 0;
    if (p.df) {                            // dataflow state of the next launch (not the
        unsigned int* w = reinterpret_cast<unsigned int*>(p.df);   // monotonic start-barrier epoch)
        for (unsigned int i = threadIdx.x; i < offsetof(DataflowDev, epoch) / 4; i += blockDim.x) w[i] = 0;
        __syncthreads();
        if (threadIdx.x == 0) p.result->t_done[0] = globaltimer_ns();   // (t_done[0]: k_init ran)
    }
    for (unsigned long long i = threadIdx.x; i < p.zero_words; i += blockDim.x) p.bdone[i] = 0;
    if (p.mask_leaves)                     // bitmask memo: level-1 entries (leaf cost, card)
        for (int v = threadIdx.x; v < p.q->n; v += blockDim.x) {
            p.memo.dcost[1ull << v] = p.q->leaf[v];
            p.memo.dcard[1ull << v] = p.q->card[v];
        }
}

// ------------------------------------------------------------ k_enum
// Block-wide exclusive scan of three counters (light sets, heavy sets, heavy pairs).
struct Tri {
    unsigned long long l, h, w;
};

__device__ __forceinline__ Tri block_scan(Tri v, Tri& total) {
    __shared__ Tri s_warp[kBlock / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    Tri inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long l = __shfl_up_sync(0xffffffffu, inc.l, o);
        const unsigned long long h = __shfl_up_sync(0xffffffffu, inc.h, o);
        const unsigned long long w = __shfl_up_sync(0xffffffffu, inc.w, o);
        if (lane >= o) {
            inc.l += l;
            inc.h += h;
            inc.w += w;
        }
    }
    if (lane == 31) s_warp[wid] = inc;
    __syncthreads();
    Tri base = {0, 0, 0}, tot = {0, 0, 0};
#pragma unroll
    for (int i = 0; i < kBlock / 32; i++) {
        if (i < wid) {
            base.l += s_warp[i].l;
            base.h += s_warp[i].h;
            base.w += s_warp[i].w;
        }
        tot.l += s_warp[i].l;
        tot.h += s_warp[i].h;
        tot.w += s_warp[i].w;
    }
    total = tot;
    return Tri{base.l + inc.l - v.l, base.h + inc.h - v.h, base.w + inc.w - v.w};
}

// Look-back records are tagged with (tile, epoch); the epoch is unique per
// (query, level, local shard) over a window of 2^15 queries (the host clears
// the ring before it wraps), so a reader never takes a stale record.
template <typename M>
__device__ __forceinline__ unsigned long long lookback_epoch(const Params<M>& p, int k) {
    return (((p.q->epoch + (unsigned long long)k) * kMaxShards + (unsigned long long)p.epoch_salt) &
            ((1ull << 26) - 1)) << 2;
}

// Warp-parallel decoupled look-back (warp 0 of the CTA): lanes read the flags of
// the 32 preceding tiles at once; the exclusive prefix is the sum of aggregates
// back to the nearest tile that already published its inclusive prefix.
__device__ __forceinline__ Tri lookback(TileRec* tiles, unsigned long long rmask, unsigned long long tile,
                                        unsigned long long epoch, Tri agg, unsigned int* err) {
    const int lane = threadIdx.x & 31;
    TileRec* tr = tiles + (tile & rmask);
    const unsigned long long me = (tile << 28) | epoch;
    if (lane == 0) {
        if (tile == 0) {
            tr->inc_l = agg.l;
            tr->inc_h = agg.h;
            tr->inc_w = agg.w;
            st_release(&tr->flag, me | 2ull);
        } else {
            tr->agg_l = agg.l;
            tr->agg_h = agg.h;
            tr->agg_w = agg.w;
            st_release(&tr->flag, me | 1ull);
        }
    }
    Tri excl = {0, 0, 0};
    if (tile == 0) return excl;
    long long top = (long long)tile - 1;
    const unsigned long long t0 = globaltimer_ns();
    while (true) {
        const long long jj = top - lane;
        const TileRec* pr = tiles + ((unsigned long long)jj & rmask);
        bool ready = true, inc = true;
        if (jj >= 0) {
            const unsigned long long f = ld_acquire(&pr->flag);
            const bool mine = (f & ~3ull) == (((unsigned long long)jj << 28) | epoch);
            ready = mine && (f & 3ull) != 0;
            inc = mine && (f & 3ull) == 2;
        }
        const unsigned inc_mask = __ballot_sync(0xffffffffu, inc);
        const unsigned ready_mask = __ballot_sync(0xffffffffu, ready);
        const int first_inc = inc_mask ? __ffs(inc_mask) - 1 : 32;
        const unsigned need = (first_inc >= 31) ? 0xffffffffu : ((2u << first_inc) - 1u);
        if ((ready_mask & need) != need) {                   // a predecessor has not published yet
            if (watchdog_expired(t0)) {
                if (lane == 0) atomicOr(err, ERR_HANG);
                break;
            }
            continue;
        }
        Tri v = {0, 0, 0};
        if (jj >= 0 && lane <= first_inc) {
            if (lane == first_inc) {
                v.l = ld_relaxed(&pr->inc_l);
                v.h = ld_relaxed(&pr->inc_h);
                v.w = ld_relaxed(&pr->inc_w);
            } else {
                v.l = ld_relaxed(&pr->agg_l);
                v.h = ld_relaxed(&pr->agg_h);
                v.w = ld_relaxed(&pr->agg_w);
            }
        }
        excl.l += warp_sum(v.l);
        excl.h += warp_sum(v.h);
        excl.w += warp_sum(v.w);
        if (first_inc < 32) break;
        top -= 32;
    }
    if (lane == 0) {
        tr->inc_l = excl.l + agg.l;
        tr->inc_h = excl.h + agg.h;
        tr->inc_w = excl.w + agg.w;
        st_release(&tr->flag, me | 2ull);
    }
    return excl;
}

// Persistent CTAs claim tiles of kTile consecutive colex ranks in ticket order.
template <typename M, int CLS>
__global__ void __launch_bounds__(kBlock) k_enum(const __grid_constant__ Params<M> p, int k, unsigned long long nranks,
                                                 unsigned long long ntiles, unsigned long long item) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SQ<M>& q = *reinterpret_cast<SQ<M>*>(smem_raw);    // only n, dpsub and adj[] are used here
    constexpr int NB = MaxN<M>::value + 1;
    unsigned long long* binom = reinterpret_cast<unsigned long long*>(smem_raw + sizeof(SQ<M>));
    __shared__ unsigned long long s_tile;
    __shared__ Tri s_excl, s_agg;

    const int n = p.q->n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) q.adj[i] = p.q->adj[i];
    for (int i = threadIdx.x; i < n * NB; i += blockDim.x) binom[i] = p.q->binom[i];
    if (threadIdx.x == 0) {
        q.n = n;
        q.dpsub = p.q->dpsub;              // set_kind reads it
        q.nbtab = 0;                       // connected() takes the loop (no byte tables here)
        q.mc = nullptr;                    // and BFS connectivity (reading R20 is MEMO_MASK only)
    }
    const unsigned long long rmask = p.tiles_ring - 1;
    const unsigned long long epoch = lookback_epoch(p, k);

    while (true) {
        if (threadIdx.x == 0) s_tile = atomicAdd(&p.desc[k].tile_ticket, 1u);
        __syncthreads();
        const unsigned long long tile = s_tile;
        if (tile >= ntiles) break;

        // ---- unrank + filter + classify (registers only)
        const unsigned long long r0 = tile * kTile + (unsigned long long)threadIdx.x * kRanksPerThread;
        M S0 = 0;
        unsigned int lflag = 0, hflag = 0;
        Tri mine = {0, 0, 0};
        if (r0 < nranks) {
            S0 = unrank_colex<M>(binom, NB, n, k, r0);
            M S = S0;
#pragma unroll
            for (int i = 0; i < kRanksPerThread; i++) {
                if (r0 + i < nranks) {
                    if (connected_cls<M, CLS>(q, S, k)) {
                        unsigned long long w;
                        const int kind = set_kind<M, CLS>(q, S, k, w);
                        if (w <= kLightMax && (CLS != CLS_GENERAL || w <= p.light_max || kind == KIND_TREE ||
                                               kind == KIND_COMPLETE)) {
                            lflag |= 1u << i;
                        } else {
                            hflag |= 1u << i;
                            mine.w += w;
                        }
                    }
                    if (r0 + i + 1 < nranks) S = gosper(S);
                }
            }
        }
        mine.l = __popc(lflag);
        mine.h = __popc(hflag);

        // ---- block scan + warp-parallel decoupled look-back
        Tri agg;
        const Tri ex = block_scan(mine, agg);
        if (threadIdx.x < 32) {
            const Tri excl = lookback(p.tiles, rmask, tile, epoch, agg, &p.result->error);
            if (threadIdx.x == 0) {
                s_excl = excl;
                s_agg = agg;
            }
        }
        __syncthreads();
        const Tri excl = s_excl;
        if (threadIdx.x == 0 && tile == ntiles - 1) {   // the last tile knows the level totals
            LevelDesc& d = p.desc[k];
            const Tri a = s_agg;
            const unsigned long long L = excl.l + a.l, H = excl.h + a.h, W = excl.w + a.w;
            d.n_light = L;
            d.n_heavy = H;
            d.heavy_pairs = W;
            d.n_items = (W + item - 1) / item;
            if (d.n_items > p.fh_cap) atomicOr(&p.result->error, ERR_ITEMS);
            if (H < p.heavy_cap + 1) p.wh[H] = W;
            const unsigned long long cnt = L + H;
            bool over = L > p.list_cap || H > p.heavy_cap;
            unsigned long long nbk = 1, off = 0;
            if (p.memo_kind == MEMO_HASH) {     // size this level's table from the exact count
                nbk = (unsigned long long)ceil((double)cnt * p.inv_load * 0.5);
                if (nbk < 1) nbk = 1;
                off = (k <= 2) ? 0ull : p.desc[k - 1].bucket_off + p.desc[k - 1].n_buckets;
                over = over || off + nbk > p.memo.arena_buckets;
            }
            if (over) {
                atomicOr(&p.result->error, ERR_CAPACITY);
                nbk = 0;
            }
            d.bucket_off = off;
            d.n_buckets = nbk;
            d.work_ticket = 0;
        }

        // ---- scatter this thread's survivors (colex order is preserved)
        if (lflag | hflag) {
            unsigned long long li = excl.l + ex.l, hi = excl.h + ex.h, wi = excl.w + ex.w;
            M S = S0;
#pragma unroll
            for (int i = 0; i < kRanksPerThread; i++) {
                if ((lflag >> i) & 1) {
                    if (li < p.list_cap) p.light[li] = S;
                    li++;
                }
                if ((hflag >> i) & 1) {
                    unsigned long long w;
                    set_kind<M, CLS>(q, S, k, w);
                    if (hi < p.heavy_cap) {
                        p.heavy[hi] = S;
                        p.wh[hi] = wi;
                        p.bkey[hi] = key_inf();
                        p.bdone[hi] = 0;
                        // items whose first pair lies in [wi, wi + w)
                        const unsigned long long it0 = (wi + item - 1) / item, it1 = (wi + w - 1) / item;
                        for (unsigned long long it = it0; it <= it1; it++)
                            if (it < p.fh_cap) p.first_heavy[it] = (unsigned int)hi;
                    }
                    wi += w;
                    hi++;
                }
                if (r0 + i + 1 < nranks && i + 1 < kRanksPerThread) S = gosper(S);
            }
        }
        __syncthreads();                   // s_tile / s_excl / scan scratch reused next tile
    }
}

// The candidates j, j + step, j + 2 step, ... < b of one block of S with memo
// connectivity (reading R20): lb = lo | deposit(j, R) advanced by a masked add
// of D = deposit(step, R); S_left = lb, or with HANG lb plus the hanging parts
// of its cut vertices C (eval_blocks_hang).  Four pairs (eight probes) in
// flight per lane; a pair competes iff both probes found their set (the CCP
// test of the block); the min is kept in f64 / mask registers (costs >= 0, so
// the f64 order is the bit order of the Key, reading R7).  Singletons read the
// leaf cost.  Counts valid pairs and non-singleton probes.
//
// The singletons' slots hold their leaf costs (written by every CTA of the
// kernel before its first level), so every probe is one branch-free load.
// COUNT: count the non-singleton probes pair by pair (else the caller uses
// mc_probes_closed).
template <bool HANG, typename M, bool COUNT = true>
__device__ __forceinline__ void mc_span(const SQ<M>& q, M S, M lo, M R, M D, M sub, unsigned long long j,
                                        unsigned long long b, unsigned int step, double cS, M C, const M* hang,
                                        Key& best, unsigned long long& nvalid, unsigned long long& nprobe) {
    const double* __restrict__ mc = q.mc;
    double bc = __longlong_as_double((long long)best.c);
    M bl = (M)best.l;
    unsigned int nv = 0, np = 0;
    // (32-bit counters: the bitmask memo has n <= 24, so a set has < 2^23 pairs)
    const unsigned int b32 = (unsigned int)b;
    for (unsigned int j32 = (unsigned int)j; j32 < b32; j32 += 4u * step) {
        M A[4];
        double ca[4], cb[4];
        bool ok[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            ok[u] = j32 + step * u < b32;
            M X = lo | sub;
            if (HANG)
                for (M T = X & C; T; T &= T - 1) X |= hang[ctz(T)];
            A[u] = X;
            const M Y = S ^ X;
            ca[u] = ok[u] ? mc[X] : 0.0;
            cb[u] = ok[u] ? mc[Y] : 0.0;
            if (COUNT) np += ok[u] ? (unsigned int)((X & (X - 1)) != 0) + (unsigned int)((Y & (Y - 1)) != 0) : 0u;
            sub = ((sub | ~R) + D) & R;
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const bool valid = ok[u] && memo_present(ca[u]) && memo_present(cb[u]);
            const double c = __dadd_rn(__dadd_rn(ca[u], cb[u]), cS);
            const M Y = S ^ A[u], l = A[u] < Y ? A[u] : Y;
            const bool better = valid && (c < bc || (c == bc && l < bl));
            bc = better ? c : bc;
            bl = better ? l : bl;
            nv += valid;
        }
    }
    nvalid += nv;
    nprobe += np;
    best = Key{(unsigned long long)__double_as_longlong(bc), (unsigned long long)bl};
}

// Non-singleton probes of the one-block candidates j in [a, b) of a set whose
// lowest vertex is lo and R = S \ {lo}, r = |R|: two per pair, less the
// singleton sides -- lb = {lo} at j = 0, and rb = {v} at j = 2^r - 1 - 2^t.
__device__ __forceinline__ unsigned long long mc_probes_closed(unsigned long long a, unsigned long long b, int r) {
    if (b <= a) return 0;
    unsigned long long singles = a == 0 ? 1 : 0;
    const unsigned long long full = (1ull << r) - 1;
    for (int t = 0; t < r; t++) {
        const unsigned long long j = full - (1ull << t);
        singles += (j >= a && j < b) ? 1 : 0;
    }
    return 2 * (b - a) - singles;
}

// ------------------------------------------------------------ k_eval
template <typename M, int CLS, typename Sink>
__device__ void eval_range(const SQ<M>& q, M S, int k, int kind, unsigned long long j0, unsigned long long j1,
                           Sink& sink, unsigned long long& nccp) {
    if (j0 >= j1) return;
    if (kind == KIND_TREE) {
        if (CLS == CLS_TREE) {
            M top = 0;
            for (int d = 0; d <= q.max_depth; d++) {
                const M T = S & q.depth_mask[d];
                if (T) {
                    top = lowbit(T);
                    break;
                }
            }
            M Mv = S & ~top;                       // one pair per edge (v, parent v)
            for (unsigned long long j = 0; j < j0; j++) Mv &= Mv - 1;
            for (unsigned long long j = j0; j < j1; j++) {
                const int v = ctz(Mv);
                Mv &= Mv - 1;
                const M A = S & q.desc[v];
                sink.add(A, S ^ A);
            }
        } else if (CLS == CLS_GENERAL) {
            unsigned long long j = 0;
            for (M T = S; T && j < j1; T &= T - 1) {
                const int v = ctz(T);
                const M up = q.adj[v] & S & ~(bitm<M>(v + 1) - 1);   // neighbours u > v in S
                const unsigned long long c = (unsigned long long)popc(up);
                if (j + c <= j0) {
                    j += c;
                    continue;
                }
                for (M U = up; U && j < j1; U &= U - 1, j++) {
                    if (j < j0) continue;
                    const int u = ctz(U);
                    const M A = grow(q, bitm<M>(v), S & ~bitm<M>(u));
                    sink.add(A, S ^ A);
                }
            }
        }
        nccp += j1 - j0;
        return;
    }
    if (CLS == CLS_TREE) return;           // trees have no other kind
    if (kind == KIND_COMPLETE) {
        const M lo = lowbit(S), R = S ^ lo;
        M sub = deposit<M>(j0, R);
        for (unsigned long long j = j0; j < j1; j++) {
            const M A = lo | sub;
            sink.add(A, S ^ A);
            sub = (sub - R) & R;
        }
        nccp += j1 - j0;
        return;
    }
    if (CLS != CLS_GENERAL) return;        // cliques are one complete block
    // KIND_BLOCKS / KIND_ONEBLOCK
    M blk[MaxN<M>::value];
    int nb;
    if (q.dpsub || kind == KIND_ONEBLOCK) {   // the whole set is the only block (dpsub: ablation)
        blk[0] = S;
        nb = 1;
    } else {
        nb = find_blocks(q, S, blk);
    }
    if constexpr (Sink::kChk) if (nb == 1 && q.mc) {   // one block S: S_left = lb (grow(lb, lb) = lb);
        const M lo = lowbit(S), R = S ^ lo;    // the probes of lb and rb are the CCP test (R20)
        sink.flush();
        unsigned long long nv = 0;
        unsigned long long np0 = 0;
        mc_span<false, M, false>(q, S, lo, R, lowbit(R), deposit<M>(j0, R), j0, j1, 1u, sink.cS, (M)0, nullptr,
                                 sink.best, nv, np0);
        sink.nprobe += mc_probes_closed(j0, j1, popc(R));
        nccp += nv;
        return;
    }
    if constexpr (Sink::kChk) if (q.mc) {  // reading R20: S_left = grow(lb, S \ rb) is connected
        sink.flush();                          // iff lb is, so the pair's probes are the CCP test;
        unsigned long long nv = 0;             // S_left from the hanging parts (eval_blocks_hang)
        M hv[MaxN<M>::value];
        unsigned long long base = 0;
        for (int bi = 0; bi < nb && base < j1; bi++) {
            const M Bm = blk[bi];
            const unsigned long long wb = (1ull << (popc(Bm) - 1)) - 1;
            if (base + wb > j0) {
                const unsigned long long a0 = (j0 > base ? j0 - base : 0), a1 = (j1 - base < wb ? j1 - base : wb);
                const M ext = S & ~Bm;
                M C = 0;                       // vertices of B with neighbours outside B
                for (M T = Bm; T; T &= T - 1) {
                    const int u = ctz(T);
                    if (q.adj[u] & ext) {
                        C |= lowbit(T);
                        hv[u] = grow(q, bitm<M>(u), ext | bitm<M>(u));
                    }
                }
                const M lo = lowbit(Bm), R = Bm ^ lo;
                mc_span<true, M>(q, S, lo, R, lowbit(R), deposit<M>(a0, R), a0, a1, 1u, sink.cS, C, hv, sink.best,
                                 nv, sink.nprobe);
            }
            base += wb;
        }
        nccp += nv;
        return;
    }
    unsigned long long base = 0;
    for (int bi = 0; bi < nb && base < j1; bi++) {
        const M Bm = blk[bi];
        const int b = popc(Bm);
        const unsigned long long wb = (1ull << (b - 1)) - 1;
        if (base + wb <= j0) {
            base += wb;
            continue;
        }
        const bool complete = !q.dpsub && induced_degree_sum(q, Bm) == b * (b - 1);
        const unsigned long long a0 = (j0 > base ? j0 - base : 0), a1 = (j1 - base < wb ? j1 - base : wb);
        const M lo = lowbit(Bm), R = Bm ^ lo;
        M sub = deposit<M>(a0, R);
        for (unsigned long long j = a0; j < a1; j++) {
            const M lb = lo | sub, rb = Bm ^ lb;
            sub = (sub - R) & R;
            if (!complete && !(conn_sub(q, lb) && conn_sub(q, rb))) continue;   // CCP block
            nccp++;
            const M A = grow(q, lb, S & ~rb);
            sink.add(A, S ^ A);                                        // S_right = S \ S_left
        }
        base += wb;
    }
}

// Tree fast path (CLS_TREE, DENSE memo; 32-bit masks).  For a set S with
// elements p_0 < ... < p_{k-1} and colex rank R = sum_i C(p_i, i+1) (passed in:
// the fused kernel knows it from the enumeration), removing a single element
// p_m gives
//     rank(S \ {p_m}) = R - C(p_m, m+1) - sum_{i>m} (C(p_i, i+1) - C(p_i, i)),
// so every split of S along an edge (v, parent v) whose lower side is the single
// vertex v (all splits of a star) costs two binomial lookups instead of a rank
// computation.  Other splits go through the generic sink.
//
// card(S) comes from the memo: reading R5's product is a left fold over the
// ascending elements in which the factors of p_0..p_{k-2} only involve edges
// among them, so for p = p_{k-1} = max(S)
//     card(S) = (..((card(S \ {p}) * card[p]) * sel(u_1, p)) * ..)   (u_i in S, u_i < p, ascending)
// bit for bit.  S \ {p} is connected (and therefore in the level k-1 memo)
// exactly when p is a leaf split of G[S], which is the first element of the
// descending walk; its card load travels with the first batch of probes.
// Otherwise the product is evaluated in full.
// Binomial pair of element position m of vertex v for the descending walk:
// x = C(v, m+1), y = C(v, m+1) - C(v, m).  Either from a precomputed uint2
// table (one 8-byte shared load) or from the plain 33 x 33 table.
template <bool PAIRS>
__device__ __forceinline__ uint2 tree_bin(const unsigned int* bin, const uint2* binp, int v, int m) {
    if constexpr (PAIRS) {
        return binp[v * 33 + m];
    } else {
        const unsigned int c1 = bin[v * 33 + m + 1], c0 = bin[v * 33 + m];
        return make_uint2(c1, c1 - c0);
    }
}

// Leaves and neighbourhood of a tree set, reported by the evaluation walk for
// the fused generation of the next level (list kernel).
struct TreeSetInfo {
    uint32_t leaves;                       // degree-1 vertices of G[S]
    uint32_t nb;                           // OR of the adjacency of S's vertices
};

template <int MEMO, bool PAIRS = false, bool INFO = false>
__device__ __forceinline__ void eval_tree_dense(const MemoPtrs& P, unsigned int gen, const MemoView& v,
                                                const unsigned int* rtab, const unsigned int* bin, const SQ<uint32_t>& q,
                                                uint32_t S, int k, unsigned int R, unsigned long long& nprobe,
                                                const uint2* binp = nullptr, TreeSetInfo* info = nullptr) {
    constexpr int U = 4;                   // elements per step = probes in flight
    uint32_t top = 0;
    for (int d = 0; d <= q.max_depth; d++) {
        const uint32_t T = S & q.depth_mask[d];
        if (T) {
            top = T & (0u - T);
            break;
        }
    }
    const bool leaf_costs = q.pad != 0;    // any non-zero leaf cost in this query
    const double* lvl = P.dcost + v.off[k - 1];
    // ---- descending walk, U elements per step, branch-free: leaf splits get
    // their incremental rank, splits at internal vertices are only recorded
    unsigned int SD = 0;
    uint32_t internal = 0, leaves = 0, nbm = 0;
    int m = k - 1;
    uint32_t T = S;
    double best_c = __longlong_as_double(0x7ff0000000000000ll);
    uint32_t best_l = 0xffffffffu;
    double cS = 0.0;
    auto step = [&](bool guard, unsigned int* rk, uint32_t* lb) {
#pragma unroll
        for (int u = 0; u < U; u++) {
            const bool ok = !guard || T != 0;
            const int vtx = ok ? 31 - __clz(T) : 0;
            const uint32_t b = ok ? 1u << vtx : 0u;
            T ^= b;
            const uint2 cc = tree_bin<PAIRS>(bin, binp, vtx, ok ? m : 0);
            const bool leaf = ok && b != top && (S & q.desc[vtx]) == b;   // v is a leaf of G[S]: B = S \ {v}
            if constexpr (INFO) nbm |= ok ? q.adj[vtx] : 0u;
            lb[u] = leaf ? b : 0u;
            internal |= (ok && b != top && !leaf) ? b : 0u;
            rk[u] = R - cc.x - SD;
            SD += ok ? cc.y : 0u;
            m -= ok ? 1 : 0;
        }
    };
    auto consume = [&](const uint32_t* lb, const double* dv) {
#pragma unroll
        for (int u = 0; u < U; u++) {
            const double a = leaf_costs && lb[u] ? __dadd_rn(q.leaf[__ffs(lb[u]) - 1], dv[u]) : dv[u];
            const double c = __dadd_rn(a, cS);
            const uint32_t Bm = S ^ lb[u];
            const uint32_t l = lb[u] < Bm ? lb[u] : Bm;
            const bool better = lb[u] != 0u && (c < best_c || (c == best_c && l < best_l));
            best_c = better ? c : best_c;
            best_l = better ? l : best_l;
            leaves |= lb[u];
        }
    };
    {   // first step: its element 0 is max(S); card(S) from card(S \ max) (R19)
        unsigned int rk[U];
        uint32_t lb[U];
        double dv[U];
        step(k < U, rk, lb);
#pragma unroll
        for (int u = 0; u < U; u++) dv[u] = lb[u] ? lvl[rk[u]] : 0.0;
        const int p = 31 - __clz(S);
        double x;
        if (lb[0]) {
            x = __dmul_rn(__ldcs(P.dcard + v.off[k - 1] + rk[0]), q.card[p]);
        } else {
            x = 1.0;
            for (uint32_t A = S ^ (1u << p); A; A &= A - 1) {
                const int a = __ffs(A) - 1;
                x = __dmul_rn(x, q.card[a]);
                for (uint32_t W = S & q.adj[a] & ((1u << a) - 1u); W; W &= W - 1)
                    x = __dmul_rn(x, q.sel[(__ffs(W) - 1) * q.n + a]);
            }
            x = __dmul_rn(x, q.card[p]);
        }
        for (uint32_t W = S & q.adj[p] & ((1u << p) - 1u); W; W &= W - 1)
            x = __dmul_rn(x, q.sel[(__ffs(W) - 1) * q.n + p]);
        cS = x;
        consume(lb, dv);
    }
    for (int rem = k - U; rem > 0; rem -= U) {
        unsigned int rk[U];
        uint32_t lb[U];
        double dv[U];
        step(rem < U, rk, lb);
#pragma unroll
        for (int u = 0; u < U; u++) dv[u] = lb[u] ? lvl[rk[u]] : 0.0;
        consume(lb, dv);
    }
    nprobe += __popc(leaves);
    if constexpr (INFO) {                  // the top vertex is a leaf too when it has one neighbour in S
        info->leaves = leaves | (__popc(q.adj[__ffs(top) - 1] & S) == 1 ? top : 0u);
        info->nb = nbm;
    }
    Key best{(unsigned long long)__double_as_longlong(best_c), (unsigned long long)best_l};
    if (internal) {                        // generic splits: both sides are multi-vertex
        PairSink<uint32_t, MEMO> sink;
        sink.init(&P, gen, &v, rtab, &q, cS);
        for (uint32_t I = internal; I; I &= I - 1) {
            const uint32_t A = S & q.desc[__ffs(I) - 1];
            sink.add(A, S ^ A);
        }
        sink.flush();
        nprobe += sink.nprobe;
        if (key_less(sink.best, best)) best = sink.best;
    }
    // ---- scatter with the rank already known
    const unsigned long long idx = v.off[k] + R;
    P.dcost[idx] = __longlong_as_double((long long)best.c);
    __stcs(P.dleft + idx, (unsigned int)best.l);
    P.dcard[idx] = cS;
}

// Shared prologue of the evaluate / extract kernels: the query, the memo view
// (per-level table geometry) and, for DENSE, the rank tables go to shared memory.
template <typename M, int MEMO>
__device__ __forceinline__ void memo_prologue(const Params<M>& p, int kmax, SQ<M>& q, MemoView& v,
                                              unsigned int* rtab) {
    load_query(q, p.q);
    for (int j = threadIdx.x; j <= kmax; j += blockDim.x) {
        if (MEMO != MEMO_HASH) {
            v.off[j] = p.dense_off[j];         // (unused by MEMO_MASK)
            v.nb[j] = 0;
        } else {
            v.off[j] = (j >= 2) ? p.desc[j].bucket_off : 0;
            v.nb[j] = (j >= 2) ? p.desc[j].n_buckets : 0;
        }
    }
    if (MEMO != MEMO_HASH) {
        for (unsigned int i = threadIdx.x; i < p.memo.rg.entries; i += blockDim.x) rtab[i] = p.memo.rank_tab[i];
        // 32-bit binomials C(i, j), i < 33, j < 33, after the rank tables (tree fast path)
        unsigned int* bin = rtab + p.memo.rg.entries;
        constexpr int NB = MaxN<M>::value + 1;
        for (int i = threadIdx.x; i < 33 * 33; i += blockDim.x) {
            const int a = i / 33, b = i % 33;
            bin[i] = (a < NB && b < NB) ? (unsigned int)p.q->binom[a * NB + b] : 0u;
        }
    }
}

// Level counters of a CTA into the level descriptor: warp sums, then one
// reduction per counter per CTA (every warp reducing into the same four
// addresses serialised ~10k same-address atomics per level at one L2 slice,
// and the level barrier's release waits for them: 25 us of star-25).  Every
// thread of the CTA must call it (it contains a __syncthreads).
__device__ __forceinline__ void flush_counters(LevelDesc* dk, unsigned long long pairs, unsigned long long nccp,
                                               unsigned long long nprobe, unsigned long long nsets = 0) {
    __shared__ unsigned long long s_fc[32][4];
    pairs = warp_sum(pairs);
    nccp = warp_sum(nccp);
    nprobe = warp_sum(nprobe);
    nsets = warp_sum(nsets);
    const unsigned int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_fc[w][0] = pairs;
        s_fc[w][1] = nccp;
        s_fc[w][2] = nprobe;
        s_fc[w][3] = nsets;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        unsigned long long x = 0;
        for (unsigned int i = 0; i < (blockDim.x >> 5); i++) x += s_fc[i][threadIdx.x];
        unsigned long long* dst[4] = {&dk->pairs, &dk->ccp, &dk->probes, &dk->n_light};
        if (x) atomicAdd(dst[threadIdx.x], x);
    }
}

// Light sets (<= kLightMax join pairs): one thread evaluates a whole set, keeps
// its min in registers and scatters it (prune fused into evaluate).
template <typename M, int CLS, int MEMO>
__global__ void __launch_bounds__(kLightBlock, kLightMinBlocks) k_eval_light(const __grid_constant__ Params<M> p, int k) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SQ<M>& q = *reinterpret_cast<SQ<M>*>(smem_raw);
    unsigned int* rtab = reinterpret_cast<unsigned int*>(smem_raw + sizeof(SQ<M>));
    __shared__ MemoView v;
    __shared__ LevelDesc d;
    memo_prologue<M, MEMO>(p, k, q, v, rtab);
    const unsigned int gen = p.q->gen;     // the per-query tag lives with the staged query
    if (threadIdx.x == 0) d = p.desc[k];
    __syncthreads();
    if (d.n_buckets == 0) return;          // capacity error already flagged
    unsigned long long pairs = 0, nccp = 0, nprobe = 0;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    const unsigned long long n_light = d.n_light;
    const unsigned long long units = (n_light + stride - 1) / stride;
    for (unsigned long long u = 0; u < units; u++) {     // warp-uniform trip count
        const unsigned long long i = u * stride + (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
        if (i < n_light) {
            const M S = p.light[i];
            unsigned long long w;
            const int kind = set_kind<M, CLS>(q, S, k, w);
            if constexpr (CLS == CLS_TREE && MEMO == MEMO_DENSE && sizeof(M) == 4) {
                if (k > 2) {                   // k = 2: both sides are leaves (no level-1 table)
                    eval_tree_dense<MEMO>(p.memo, gen, v, rtab, rtab + p.memo.rg.entries, q, S, k,
                                           rank_of(p.memo.rg, rtab, S), nprobe);
                    nccp += w;
                    pairs += w;
                    continue;
                }
            }
            PairSink<M, MEMO> sink;
            sink.init(&p.memo, gen, &v, rtab, &q, card_of(q, S));
            eval_range<M, CLS>(q, S, k, kind, 0, w, sink, nccp);
            sink.flush();
            nprobe += sink.nprobe;
            pairs += w;
            memo_insert<M, MEMO>(p.memo, gen, v, rtab, k, S, sink.best, sink.cS);
        }
    }
    // card(S) of the heavy sets, one thread per set, for k_eval_heavy (next in
    // stream order) so its work-item warps never recompute the product chain
    const unsigned long long n_heavy = d.n_heavy < p.heavy_cap ? d.n_heavy : p.heavy_cap;
    for (unsigned long long h = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; h < n_heavy; h += stride)
        p.hcard[h] = card_of(q, p.heavy[h]);
    flush_counters(&p.desc[k], pairs, nccp, nprobe);
}

// Heavy sets: the heavy pair space is cut into `item`-pair work items; warps
// claim groups of items dynamically, evaluate lane-contiguous chunks, reduce
// with shuffles, and merge split sets through a 128-bit CAS min + a pair
// counter (the last contributor scatters the set).
// Heavy phase of level k (shared by k_eval_heavy and the fused kernel): the
// heavy pair space is cut into `item`-pair work items; warps claim groups of
// items dynamically, evaluate lane-contiguous chunks, reduce with shuffles and
// merge split sets through a 128-bit CAS min + a pair counter (the last
// contributor scatters the set).
// Collaborative Context Collection for the candidates [a, b) of a
// block-decomposed set, one warp: per step the 32 lanes test 32 consecutive
// candidates (block subset lb, CCP check of lb and rb inside the block, then
// S_left = grow(lb, S \ rb)); the valid ones are stashed in shared
// memory, and whenever 32 are stashed every lane takes one and evaluates it
// (memo probes, C_out, min).  The probe/compare work then always runs with a
// full warp instead of with the lanes whose candidate passed (35% on random-20).
constexpr int kCccStash = 64;
template <typename M, typename Sink>
__device__ __forceinline__ void eval_blocks_ccc(const SQ<M>& q, M S, int kind, unsigned long long a,
                                                unsigned long long b, Sink& sink, unsigned long long& nccp, M* stash) {
    const unsigned int lane = threadIdx.x & 31, lt = (1u << lane) - 1u;
    M blk[MaxN<M>::value];
    int nb;
    if (q.dpsub || kind == KIND_ONEBLOCK) {
        blk[0] = S;
        nb = 1;
    } else {
        nb = find_blocks(q, S, blk);
    }
    unsigned int cnt = 0;                  // stashed pairs (warp-uniform)
    unsigned long long base = 0;
    for (int bi = 0; bi < nb && base < b; bi++) {
        const M Bm = blk[bi];
        const int bsz = popc(Bm);
        const unsigned long long wb = (1ull << (bsz - 1)) - 1;
        if (base + wb <= a) {
            base += wb;
            continue;
        }
        const bool complete = !q.dpsub && induced_degree_sum(q, Bm) == bsz * (bsz - 1);
        const unsigned long long a0 = (a > base ? a - base : 0), a1 = (b - base < wb ? b - base : wb);
        const M lo = lowbit(Bm), R = Bm ^ lo;
        const M D32 = popc(R) > 5 ? deposit_lo<M>(32u, R) : (M)0;
        M sub = a0 + lane < a1 ? deposit<M>(a0 + lane, R) : (M)0;
        for (unsigned long long j0 = a0; j0 < a1; j0 += 32) {
            const unsigned long long j = j0 + lane;
            bool valid = false;
            M A = 0;
            if (j < a1) {
                const M lb = lo | sub, rb = Bm ^ lb;
                valid = complete || (conn_sub(q, lb) && conn_sub(q, rb));     // CCP block
                if (valid) A = grow(q, lb, S & ~rb);
            }
            sub = ((sub | ~R) + D32) & R;
            const unsigned int bal = __ballot_sync(0xffffffffu, valid);
            if (valid) {
                stash[cnt + __popc(bal & lt)] = A;
                nccp++;
            }
            cnt += __popc(bal);
            __syncwarp();
            if (cnt >= 32) {                   // a full warp of valid pairs
                const M X = stash[cnt - 32 + lane];
                sink.add(X, S ^ X);            // S_right = S \ S_left
                cnt -= 32;
                __syncwarp();
            }
        }
        base += wb;
    }
    if (lane < cnt) {
        const M X = stash[lane];
        sink.add(X, S ^ X);
    }
    __syncwarp();
}

// Block-decomposed set S (reading R20, one warp, candidates [a, b) in block
// order).  For a block B of S and v in B let H_v = grow({v}, (S \ B) + v), the
// part of S that hangs off B at v (H_v = {v} unless v is a cut vertex with
// neighbours outside B).  The H_v of B partition S and meet only at B's
// vertices, so for a split (lb, rb) of B
//     S_left = grow(lb, S \ rb) = OR of H_v over v in lb
//     S_right = S \ S_left      = OR of H_v over v in rb
// and S_left is connected iff lb is (a hanging part touches B at one vertex
// only).  So no per-candidate BFS: lanes take interleaved candidates, OR in
// the hanging parts of the cut vertices in lb (usually none or one), and the
// sink's probes of S_left and S_right are the CCP test of (lb, rb)
// (P:553-560).  hang[] is the warp's scratch (>= MaxN entries).
// The blocks come from the heavy list's cache (gblk, nb <= kHeavyBlk) or are
// found again.
//
// A set evaluated whole (whole: [a, b) = [0, w)) first takes the candidates of
// all its small blocks (at most kSmallBlockPairs each: bridges, triangles)
// together, one lane per candidate with S_left = grow(lb, S \ rb) --
// otherwise every bridge would cost the warp a memory round trip for one pair.
constexpr unsigned long long kSmallBlockPairs = 7;
template <typename M, typename Sink>
__device__ __forceinline__ void eval_blocks_hang(const SQ<M>& q, M S, unsigned long long a, unsigned long long b,
                                                 bool whole, Sink& sink, M* hang, M lblk, int nb) {
    const unsigned int lane = threadIdx.x & 31;
    M blk[MaxN<M>::value];
    const bool cached = nb <= kHeavyBlk;   // lane i holds cached block i & 7
    if (!cached) nb = find_blocks(q, S, blk);
    sink.chk = true;
    if (whole) {
        unsigned int nsmall = 0;           // candidates of the small blocks
        for (int bi = 0; bi < nb; bi++) {
            const M Bm = cached ? __shfl_sync(0xffffffffu, lblk, bi) : blk[bi];
            const unsigned long long wb = (1ull << (popc(Bm) - 1)) - 1;
            if (wb <= kSmallBlockPairs) nsmall += (unsigned int)wb;
        }
        for (unsigned int r = 0; r < nsmall; r += 32) {
            const unsigned int idx = r + lane;
            M Bm = 0;
            unsigned int j = idx;
            for (int bi = 0; bi < nb; bi++) {      // (uniform trip count: shuffles inside)
                const M X = cached ? __shfl_sync(0xffffffffu, lblk, bi) : blk[bi];
                const unsigned int wb = (1u << (popc(X) - 1)) - 1u;
                if (wb <= kSmallBlockPairs && !Bm) {
                    if (j < wb) Bm = X;
                    else j -= wb;
                }
            }
            if (idx < nsmall) {
                const M lo = lowbit(Bm), lb = lo | deposit<M>(j, Bm ^ lo), rb = Bm ^ lb;
                const M A = grow(q, lb, S & ~rb);
                mc_span<false, M>(q, S, A, (M)0, (M)0, (M)0, 0, 1, 1u, sink.cS, (M)0, nullptr, sink.best,
                                  sink.nvalid, sink.nprobe);
            }
        }
    }
    unsigned long long base = 0;
    for (int bi = 0; bi < nb && base < b; bi++) {
        const M Bm = cached ? __shfl_sync(0xffffffffu, lblk, bi) : blk[bi];
        const int bsz = popc(Bm);
        const unsigned long long wb = (1ull << (bsz - 1)) - 1;
        if (base + wb <= a || (whole && wb <= kSmallBlockPairs)) {
            base += wb;
            continue;
        }
        const unsigned long long a0 = (a > base ? a - base : 0), a1 = (b - base < wb ? b - base : wb);
        const M ext = S & ~Bm;
        M C = 0;                               // vertices of B with neighbours outside B
        for (M T = Bm; T; T &= T - 1)
            if (q.adj[ctz(T)] & ext) C |= lowbit(T);
        __syncwarp();
        if ((int)lane < popc(C)) {
            const int v = nth_bit(C, (int)lane);
            hang[v] = grow(q, bitm<M>(v), ext | bitm<M>(v));
        }
        __syncwarp();
        const M lo = lowbit(Bm), R = Bm ^ lo, D = popc(R) > 5 ? deposit_lo<M>(32u, R) : (M)0;
        const unsigned long long j = a0 + lane;
        if (j < a1) {
            // deposit(a0 + lane) = deposit(a0) (+) deposit(lane) in R's domain
            const M da = a0 ? deposit<M>(a0, R) : (M)0;
            const M sub = ((da | ~R) + deposit_lo<M>(lane, R)) & R;
            mc_span<true, M>(q, S, lo, R, D, sub, j, a1, 32u, sink.cS, C, hang, sink.best, sink.nvalid, sink.nprobe);
        }
        base += wb;
    }
    __syncwarp();
}

template <typename M, int CLS, int MEMO>
__device__ void heavy_phase(const Params<M>& p, int k, unsigned long long item, const SQ<M>& q, const MemoView& v,
                            const unsigned int* rtab, unsigned int gen, const LevelDesc& d,
                            unsigned long long& pairs, unsigned long long& nccp, unsigned long long& nprobe) {
    __shared__ M s_ccc[kBlock / 32][kCccStash];    // per-warp CCC stash (general graphs)
    if (d.n_buckets == 0 || d.n_items == 0) return;
    const int lane = threadIdx.x & 31;
    const unsigned long long nwarps = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
    unsigned long long G = d.n_items / (nwarps * 4);
    if (G < 1) G = 1;
    const unsigned long long ngroups = (d.n_items + G - 1) / G;
    while (true) {
        unsigned long long g = 0;
        if (lane == 0) g = atomicAdd(&p.desc[k].work_ticket, 1u);
        g = __shfl_sync(0xffffffffu, g, 0);
        if (g >= ngroups) break;
        const unsigned long long c0 = g * G * item;
        unsigned long long c1 = (g + 1) * G * item;
        if (c1 > d.heavy_pairs) c1 = d.heavy_pairs;
        unsigned long long h = p.first_heavy[g * G];
        for (; h < d.n_heavy; h++) {
            // the set's record in one memory round trip: every load is issued
            // before the first use (general graphs: lane l also fetches cached
            // block l & 7)
            const unsigned long long W0 = p.wh[h], W1 = p.wh[h + 1];
            const M S = p.heavy[h];
            const double hc = p.hcard[h];
            unsigned int inf = 0;
            M lblk = 0;
            if (CLS == CLS_GENERAL && q.mc) {
                inf = p.hinfo[h];
                lblk = p.hblk[h * kHeavyBlk + (lane & (kHeavyBlk - 1))];
            }
            const unsigned long long w = W1 - W0;
            if (W0 >= c1) break;
            const bool whole = w <= p.heavy_whole;
            if (whole && W0 < c0) continue;    // owned by the claim holding its first pair
            const unsigned long long a = whole ? 0 : (c0 > W0 ? c0 - W0 : 0),
                                     b = whole ? w : (c1 - W0 < w ? c1 - W0 : w);
            unsigned long long wk;
            int kind, hnb = 0;
            if (CLS == CLS_GENERAL && q.mc) {
                kind = (int)(inf & 3u);
                hnb = (int)(inf >> 2);
            } else {
                kind = set_kind<M, CLS>(q, S, k, wk);
            }
            PairSink<M, MEMO> sink;
            sink.init(&p.memo, gen, &v, rtab, &q, hc);
            const unsigned long long cnt = b - a;
            if (kind == KIND_COMPLETE) {
                // lane-interleaved pairs j = a + lane + 32 i: the lanes' left
                // sides differ in the lowest elements of S, so one warp's probes
                // fall into few memo lines; +32 in the deposited domain is a
                // masked add (carries skip the bits outside R)
                const M lo = lowbit(S), R = S ^ lo, D = popc(R) > 5 ? deposit_lo<M>(32u, R) : (M)0;   // (<= 32 pairs: one round)
                unsigned long long j = a + lane;
                M sub = j < b ? deposit<M>(j, R) : 0;
                for (; j < b; j += 32) {
                    const M A = lo | sub;
                    sink.add(A, S ^ A);
                    sub = ((sub | ~R) + D) & R;
                    nccp++;
                }
            } else if (CLS == CLS_GENERAL && q.mc && (kind == KIND_ONEBLOCK || (q.dpsub && kind == KIND_BLOCKS))) {
                // one block S (or every set, DPSUB ablation): S_left = lb, and
                // the probes of lb and rb are the CCP test (reading R20); lanes
                // interleaved as for complete sets
                const M lo = lowbit(S), R = S ^ lo, D = popc(R) > 5 ? deposit_lo<M>(32u, R) : (M)0;
                const unsigned long long j = a + lane;
                if (j < b) {
                    const M da = a ? deposit<M>(a, R) : (M)0;      // deposit(a + lane), as a masked add
                    const M sub = ((da | ~R) + deposit_lo<M>(lane, R)) & R;
                    unsigned long long np0 = 0;
                    mc_span<false, M, false>(q, S, lo, R, D, sub, j, b, 32u, sink.cS, (M)0, nullptr, sink.best,
                                             sink.nvalid, np0);
                }
                if (lane == 0) sink.nprobe += mc_probes_closed(a, b, popc(R));
                nccp += sink.nvalid;
            } else if (CLS == CLS_GENERAL && q.mc && kind == KIND_BLOCKS) {
                eval_blocks_hang<M>(q, S, a, b, a == 0 && b == w, sink, s_ccc[threadIdx.x >> 5], lblk, hnb);
                nccp += sink.nvalid;
            } else if (CLS == CLS_GENERAL && kind >= KIND_BLOCKS && !p.no_ccc) {
                eval_blocks_ccc<M>(q, S, kind, a, b, sink, nccp, s_ccc[threadIdx.x >> 5]);
            } else {                               // lane-contiguous chunks of [a, b)
                const unsigned long long per = (cnt + 31) >> 5;
                unsigned long long j0 = a + per * lane, j1 = j0 + per;
                if (j0 > b) j0 = b;
                if (j1 > b) j1 = b;
                eval_range<M, CLS>(q, S, k, kind, j0, j1, sink, nccp);
            }
            sink.flush();
            nprobe += sink.nprobe;
            const Key best = warp_min(sink.best);
            if (lane == 0) {
                pairs += cnt;
                if (a == 0 && b == w) {
                    memo_insert<M, MEMO>(p.memo, gen, v, rtab, k, S, best, p.hcard[h]);
                } else {
                    atomic_key_min(&p.bkey[h], best);
                    __threadfence();
                    const unsigned long long old = atomicAdd(&p.bdone[h], cnt);
                    if (old + cnt == w) {      // last contributor finalises the set
                        __threadfence();
                        const unsigned long long* kp = reinterpret_cast<const unsigned long long*>(&p.bkey[h]);
                        const Key fin{ld_relaxed(kp), ld_relaxed(kp + 1)};
                        memo_insert<M, MEMO>(p.memo, gen, v, rtab, k, S, fin, p.hcard[h]);
                    }
                }
            }
        }
    }
}

template <typename M, int CLS, int MEMO>
__global__ void __launch_bounds__(kBlock, 2) k_eval_heavy(const __grid_constant__ Params<M> p, int k, unsigned long long item) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SQ<M>& q = *reinterpret_cast<SQ<M>*>(smem_raw);
    unsigned int* rtab = reinterpret_cast<unsigned int*>(smem_raw + sizeof(SQ<M>));
    __shared__ MemoView v;
    __shared__ LevelDesc d;
    memo_prologue<M, MEMO>(p, k, q, v, rtab);
    const unsigned int gen = p.q->gen;
    if (threadIdx.x == 0) d = p.desc[k];
    __syncthreads();
    unsigned long long pairs = 0, nccp = 0, nprobe = 0;
    heavy_phase<M, CLS, MEMO>(p, k, item, q, v, rtab, gen, d, pairs, nccp, nprobe);
    flush_counters(&p.desc[k], pairs, nccp, nprobe);
}

// ------------------------------------------------------------ k_extract
// One thread walks the memo from the full set: left(S) from the
// memo, right = S \ left; nodes in post-order, root last.  Also sums counters.
// Level counters into the result, one warp: lane j reads the descriptor of
// level j (a single thread walking the levels waited one load round trip per
// level, ~15 us at n = 25).  Bit 1 of count_levels: this rank counts the n
// singletons (level 1).
template <typename M>
__device__ void level_counters_warp(const Params<M>& p, ResultDev* r, const LevelDesc* desc = nullptr) {
    const int n = p.n;
    if (!desc) desc = p.desc;
    const unsigned int lane = threadIdx.x & 31;
    unsigned long long csg = 0, ccp = 0, pairs = 0, probes = 0;
    for (int j = (int)lane; j <= n; j += 32) {
        unsigned long long a = 0, b = 0, c = 0, d = 0;
        if (j == 1) {
            a = ((p.count_levels >> 1) & 1ull) ? (unsigned long long)n : 0ull;
        } else if (j >= 2 && ((p.count_levels >> j) & 1ull)) {
            const LevelDesc& ds = desc[j];
            a = ds.n_light + ds.n_heavy;
            b = ds.ccp;
            c = ds.pairs;
            d = ds.probes;
        }
        r->lvl_csg[j] = a;
        r->lvl_ccp[j] = b;
        r->lvl_pairs[j] = c;
        csg += a;
        ccp += b;
        pairs += c;
        probes += d;
    }
    csg = warp_sum(csg);
    ccp = warp_sum(ccp);
    pairs = warp_sum(pairs);
    probes = warp_sum(probes);
    if (lane == 0) {
        r->csg = csg;
        r->ccp = ccp;
        r->pairs = pairs;
        r->probes = probes;
    }
    __syncwarp();
}

template <typename M, int MEMO>
__device__ void extract_phase_m(const MemoPtrs& PM, ResultDev* r, int n, const SQ<M>& q, const MemoView& v,
                                const unsigned int* rtab, unsigned int gen);
template <typename M, int MEMO>
__device__ void extract_phase(const Params<M>& p, const SQ<M>& q, const MemoView& v, const unsigned int* rtab,
                              unsigned int gen) {
    extract_phase_m<M, MEMO>(p.memo, p.result, p.n, q, v, rtab, gen);
}
// (the memo, result and n explicitly: the fused exchange extracts from a
// rank's replica)
template <typename M, int MEMO>
__device__ void extract_phase_m(const MemoPtrs& PM, ResultDev* r, int n, const SQ<M>& q, const MemoView& v,
                                const unsigned int* rtab, unsigned int gen) {
    // (the level counters are written by level_counters_warp before)
    if (r->error) {
        r->n_nodes = 0;
        return;
    }
    // explicit-stack post-order walk; one memo read per internal node (its
    // left, cost and, in the dense layouts, card are kept on the stack)
    M st_set[2 * kMaxN], st_L[2 * kMaxN];
    double st_c[2 * kMaxN], st_card[2 * kMaxN];
    int st_state[2 * kMaxN], st_left[2 * kMaxN];
    int sp = 0, nn = 0;
    const M all = (n == (int)(8 * sizeof(M))) ? ~(M)0 : (bitm<M>(n) - 1);
    st_set[0] = all;
    st_state[0] = 0;
    sp = 1;
    int last = -1;
    while (sp) {
        const int top = sp - 1;
        const M S = st_set[top];
        if (popc(S) == 1) {
            const int vtx = ctz(S);
            mpdp_plan_node& nd = r->nodes[nn];
            nd.left = nd.right = -1;
            nd.relation = vtx;
            nd.reserved = 0;
            nd.set = (unsigned long long)S;
            nd.cardinality = q.card[vtx];
            nd.cost = q.leaf[vtx];
            last = nn++;
            --sp;
            continue;
        }
        if (st_state[top] == 0) {
            M L;
            st_c[top] = memo_get<M, MEMO>(PM, gen, v, rtab, S, L, &st_card[top]);
            st_L[top] = L;
            st_state[top] = 1;
            st_set[sp] = L;
            st_state[sp] = 0;
            sp++;
        } else if (st_state[top] == 1) {
            st_left[top] = last;
            st_state[top] = 2;
            st_set[sp] = S & ~st_L[top];
            st_state[sp] = 0;
            sp++;
        } else {
            mpdp_plan_node& nd = r->nodes[nn];
            nd.left = st_left[top];
            nd.right = last;
            nd.relation = -1;
            nd.reserved = 0;
            nd.set = (unsigned long long)S;
            nd.cardinality = MEMO != MEMO_HASH ? st_card[top] : card_of(q, S);   // (reading R5: bit-equal)
            nd.cost = st_c[top];
            last = nn++;
            --sp;
        }
    }
    r->n_nodes = (unsigned int)nn;
    r->cost = r->nodes[nn - 1].cost;
}

template <typename M, int MEMO>
__global__ void k_extract(const __grid_constant__ Params<M> p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SQ<M>& q = *reinterpret_cast<SQ<M>*>(smem_raw);
    unsigned int* rtab = reinterpret_cast<unsigned int*>(smem_raw + sizeof(SQ<M>));
    __shared__ MemoView v;
    memo_prologue<M, MEMO>(p, p.n, q, v, rtab);
    const unsigned int gen = p.q->gen;
    __syncthreads();
    if (threadIdx.x < 32) {
        level_counters_warp(p, p.result);
        if (threadIdx.x == 0) extract_phase<M, MEMO>(p, q, v, rtab, gen);
    }
}

}  // namespace mpdp
