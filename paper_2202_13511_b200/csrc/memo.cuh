// memo.cuh — the GPU memo of Alg. mpdp_gpu: one table per
// subset size (the per-size tables of), keyed by the relation bitmask.
//
// Two implementations behind one interface (template parameter MEMO):
//
//  MEMO_DENSE  (default, n <= 32): the table of level j is addressed by a
//      MINIMAL PERFECT HASH of the key: its colex rank among the C(n, j)
//      j-subsets.  Probe length is always 1, no key is stored, a probe is one
//      8-byte load and an insert one store.  The rank is computed from four
//      8-bit chunks with tables in shared memory:
//         rank(T) = sum_c R_c[popc(T below chunk c)][byte_c(T)],
//         R_c[o][b] = sum_{bit i of b} C(8c + i, o + #(bits of b below i) + 1).
//  MEMO_MASK   (clique / general queries, n <= kMaskMaxN, one GPU): the same
//      three arrays indexed by the relation bitmask itself (2^n entries, all
//      levels in one array).  A probe is one load with no rank arithmetic;
//      the whole cost array (2 MB at n = 18) is L2-resident.  Trees keep the
//      colex layout: their level-k-1 arrays are contiguous, bitmask slots of
//      one level are scattered over all 2^n.
//  MEMO_HASH   (n > 32, and as an ablation): Murmur3-finalised open addressing
//      with linear probing over 32-byte buckets of two 16-byte slots
//      {tagged key, cost}; a per-query tag in the key word makes stale slots of
//      earlier queries read as empty, so tables are never cleared.
#pragma once
#include "dev_graph.cuh"

namespace mpdp {

enum MemoKind : int { MEMO_HASH = 0, MEMO_DENSE = 1, MEMO_MASK = 2 };

enum ErrBits : unsigned int { ERR_CAPACITY = 1u, ERR_PROBE = 2u, ERR_ITEMS = 4u, ERR_TABLE_FULL = 8u, ERR_HANG = 16u,
                             ERR_TIMEOUT = 32u };

// Watchdog for device spin-waits: a bug must surface as an error, never as a
// hung GPU.  Returns true once `t0` (from globaltimer_ns) is more than 2 s old.
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ bool watchdog_expired(unsigned long long t0) {
    return globaltimer_ns() - t0 > 2000000000ull;
}

constexpr int kRankChunks = 4;             // 4 x 8 bits cover n <= 32
constexpr int kMaskMaxN = 24;              // MEMO_MASK: 2^24 x 20 B = 336 MB of arrays at most

// Host/device-shared geometry of the chunked rank tables for n relations.
struct RankGeom {
    unsigned int base[kRankChunks], len[kRankChunks], entries;
    int nch;
};
__host__ __device__ inline RankGeom rank_geom(int n) {
    RankGeom g{};
    unsigned int at = 0;
    g.nch = (n + 7) / 8;
    for (int c = 0; c < kRankChunks; c++) {
        const int bits = (n - 8 * c) < 8 ? ((n - 8 * c) > 0 ? n - 8 * c : 0) : 8;
        g.base[c] = at;
        g.len[c] = c < g.nch ? (1u << bits) : 0u;
        at += c < g.nch ? (unsigned int)(8 * c + 1) * g.len[c] : 0u;
    }
    g.entries = at;
    return g;
}

// The memo as seen by one CTA (filled in the kernel prologue, lives in smem).
struct MemoView {
    unsigned long long off[kMaxN + 1];     // per level: DENSE entry offset / HASH bucket offset
    unsigned long long nb[kMaxN + 1];      // HASH: buckets per level
};

struct MemoPtrs {
    // DENSE
    double* dcost;                         // [sum_j C(n,j)] cost by (level offset + rank)
    double* dcard;                         // [sum_j C(n,j)] card(S) (reading R5), same index
    unsigned int* dleft;                   // [sum_j C(n,j)] left(S) (32-bit masks)
    const unsigned int* rank_tab;          // [RankGeom::entries]
    // HASH
    RankGeom rg;                           // chunk geometry of the rank tables (depends on n)
    Bucket* arena;
    void* cold;                            // left(S) per slot (2 per bucket), mask width
    unsigned long long arena_buckets;
    unsigned int* error;
};

// -------------------------------------------------------------- dense memo
// The geometry comes from the kernel parameter block (constant bank, warp
// uniform); only the table itself is in shared memory.
__device__ __forceinline__ unsigned int rank_of(const RankGeom& g, const unsigned int* tab, uint32_t T) {
    unsigned int r = tab[T & 255u];                          // chunk 0: offset 0
#pragma unroll
    for (int c = 1; c < kRankChunks; c++) {
        if (c < g.nch) {
            const unsigned int b = (T >> (8 * c)) & 255u;
            const unsigned int o = (unsigned int)__popc(T & ((1u << (8 * c)) - 1u));
            r += tab[g.base[c] + o * g.len[c] + b];
        }
    }
    return r;
}

// Slot of set T of size j in the dense-layout arrays (DENSE: level offset +
// colex rank; MASK: the bitmask), and the same when the rank R is known.
template <int MEMO>
__device__ __forceinline__ unsigned long long memo_slot(const MemoView& v, const RankGeom& g, const unsigned int* tab,
                                                         int j, uint32_t T) {
    return MEMO == MEMO_MASK ? (unsigned long long)T : v.off[j] + rank_of(g, tab, T);
}
template <int MEMO>
__device__ __forceinline__ unsigned long long memo_slot_r(const MemoView& v, int j, unsigned int R, uint32_t T) {
    return MEMO == MEMO_MASK ? (unsigned long long)T : v.off[j] + R;
}

// -------------------------------------------------------------- hash memo
struct B4 {
    unsigned long long k0, c0, k1, c1;
};
// One bucket = one 32-byte L2 sector, fetched with a single 256-bit read-only
// load (LDG.E.ENL2.256): tables of earlier levels are immutable during level k.
__device__ __forceinline__ B4 ld_bucket(const Bucket* b) {
    B4 r;
    asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(r.k0), "=l"(r.c0), "=l"(r.k1), "=l"(r.c1)
                 : "l"(b));
    return r;
}

template <typename M>
__device__ __forceinline__ unsigned long long hash_home(const MemoView& v, M T, int j) {
    return fastrange(fmix(T), v.nb[j]);
}

// Walk the probe sequence from bucket b until T or an empty slot is found.
template <typename M>
__device__ double hash_walk(const MemoPtrs& P, unsigned int gen, const MemoView& v, M T, int j,
                            unsigned long long b, unsigned long long* slot_out) {
    const unsigned long long want = Tag<M>::make(T, gen);
    const unsigned int g = Tag<M>::gen_of(want);
    const unsigned long long nb = v.nb[j];
    for (unsigned long long guard = 0; guard < nb; guard++) {
        const B4 x = ld_bucket(P.arena + v.off[j] + b);
        if (x.k0 == want) {
            if (slot_out) *slot_out = (v.off[j] + b) * 2;
            return __longlong_as_double((long long)x.c0);
        }
        if (x.k1 == want) {
            if (slot_out) *slot_out = (v.off[j] + b) * 2 + 1;
            return __longlong_as_double((long long)x.c1);
        }
        if (Tag<M>::gen_of(x.k0) != g || Tag<M>::gen_of(x.k1) != g) break;   // empty slot: absent
        b = (b + 1 == nb) ? 0 : b + 1;
    }
    atomicOr(P.error, ERR_PROBE);
    return __longlong_as_double(0x7ff8000000000000ll);
}

template <typename M>
__device__ __forceinline__ void hash_insert(const MemoPtrs& P, unsigned int gen, unsigned long long off,
                                            unsigned long long nb, M S, const Key& best) {
    const unsigned long long want = Tag<M>::make(S, gen);
    const unsigned int g = Tag<M>::gen_of(want);
    Bucket* base = P.arena + off;
    unsigned long long b = fastrange(fmix(S), nb);
    for (unsigned long long guard = 0; guard < nb; guard++) {
#pragma unroll
        for (int s = 0; s < 2; s++) {
            unsigned long long* kp = &base[b].s[s].key;
            unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(kp);
            while (Tag<M>::gen_of(cur) != g) {
                const unsigned long long old = atomicCAS(kp, cur, want);
                if (old == cur) {
                    base[b].s[s].cost = __longlong_as_double((long long)best.c);
                    reinterpret_cast<M*>(P.cold)[(off + b) * 2 + s] = (M)best.l;
                    return;
                }
                cur = old;
            }
        }
        b = (b + 1 == nb) ? 0 : b + 1;
    }
    atomicOr(P.error, ERR_TABLE_FULL);
}

// ----------------------------------------------------------- interface
// Batched cost lookup: every load of the batch is issued before any is used,
// so a thread keeps NP probes in flight.  Singletons read the leaf cost.
template <typename M, int MEMO, int NP>
__device__ __forceinline__ void memo_lookup(const MemoPtrs& P, unsigned int gen, const MemoView& v,
                                            const unsigned int* rtab,
                                            const SQ<M>& q, const M (&X)[NP], unsigned valid, double (&c)[NP],
                                            unsigned long long& nprobe) {
    if (MEMO != MEMO_HASH) {
        double d[NP];
#pragma unroll
        for (int i = 0; i < NP; i++) {
            const int j = popc(X[i]);
            d[i] = 0.0;
            if (((valid >> i) & 1) && j > 1)
                d[i] = P.dcost[memo_slot<MEMO>(v, P.rg, rtab, j, (uint32_t)X[i])];   // coherent load
        }
#pragma unroll
        for (int i = 0; i < NP; i++) {
            const int j = popc(X[i]);
            c[i] = (j == 1) ? q.leaf[ctz(X[i])] : d[i];
            if (((valid >> i) & 1) && j > 1) nprobe++;
        }
    } else {
        B4 bk[NP];
        unsigned long long bi[NP];
#pragma unroll
        for (int i = 0; i < NP; i++) {
            const int j = popc(X[i]);
            bi[i] = 0;
            if (((valid >> i) & 1) && j > 1) {
                bi[i] = hash_home(v, X[i], j);
                bk[i] = ld_bucket(P.arena + v.off[j] + bi[i]);
            }
        }
        // resolve; keys displaced past their home bucket are walked in a
        // warp-converged loop (no per-lane divergent call)
        unsigned pending = 0;
#pragma unroll
        for (int i = 0; i < NP; i++) {
            const int j = popc(X[i]);
            c[i] = 0.0;
            if (!((valid >> i) & 1)) continue;
            if (j == 1) {
                c[i] = q.leaf[ctz(X[i])];
                continue;
            }
            nprobe++;
            const unsigned long long want = Tag<M>::make(X[i], gen);
            if (bk[i].k0 == want) c[i] = __longlong_as_double((long long)bk[i].c0);
            else if (bk[i].k1 == want) c[i] = __longlong_as_double((long long)bk[i].c1);
            else pending |= 1u << i;
        }
        while (__any_sync(__activemask(), pending != 0)) {
#pragma unroll
            for (int i = 0; i < NP; i++) {
                if ((pending >> i) & 1) {
                    const int j = popc(X[i]);
                    const unsigned long long nbj = v.nb[j];
                    bi[i] = (bi[i] + 1 == nbj) ? 0 : bi[i] + 1;
                    bk[i] = ld_bucket(P.arena + v.off[j] + bi[i]);
                }
            }
#pragma unroll
            for (int i = 0; i < NP; i++) {
                if ((pending >> i) & 1) {
                    const unsigned long long want = Tag<M>::make(X[i], gen);
                    if (bk[i].k0 == want) {
                        c[i] = __longlong_as_double((long long)bk[i].c0);
                        pending &= ~(1u << i);
                    } else if (bk[i].k1 == want) {
                        c[i] = __longlong_as_double((long long)bk[i].c1);
                        pending &= ~(1u << i);
                    } else if (Tag<M>::gen_of(bk[i].k0) != Tag<M>::gen_of(want) ||
                               Tag<M>::gen_of(bk[i].k1) != Tag<M>::gen_of(want)) {
                        atomicOr(P.error, ERR_PROBE);       // empty slot: not in the memo
                        c[i] = __longlong_as_double(0x7ff8000000000000ll);
                        pending &= ~(1u << i);
                    }
                }
            }
        }
    }
}

// scatter (S, best(S)) into the level-k table
template <typename M, int MEMO>
__device__ __forceinline__ void memo_insert(const MemoPtrs& P, unsigned int gen, const MemoView& v,
                                            const unsigned int* rtab, int k, M S, const Key& best, double card) {
    if (MEMO != MEMO_HASH) {
        const unsigned long long idx = memo_slot<MEMO>(v, P.rg, rtab, k, (uint32_t)S);
        P.dcost[idx] = __longlong_as_double((long long)best.c);
        __stcs(P.dleft + idx, (unsigned int)best.l);
        P.dcard[idx] = card;
    } else {
        hash_insert(P, gen, v.off[k], v.nb[k], S, best);
    }
}

// (cost, left) of a finished set (extraction)
template <typename M, int MEMO>
__device__ __forceinline__ double memo_get(const MemoPtrs& P, unsigned int gen, const MemoView& v,
                                           const unsigned int* rtab, M S, M& left, double* card = nullptr) {
    const int j = popc(S);
    if (MEMO != MEMO_HASH) {
        const unsigned long long idx = memo_slot<MEMO>(v, P.rg, rtab, j, (uint32_t)S);
        left = (M)P.dleft[idx];
        if (card) *card = P.dcard[idx];
        return P.dcost[idx];
    } else {
        unsigned long long slot = 0;
        const double c = hash_walk(P, gen, v, S, j, hash_home(v, S, j), &slot);
        left = reinterpret_cast<const M*>(P.cold)[slot];
        return c;
    }
}

}  // namespace mpdp
