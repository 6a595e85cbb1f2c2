// dev_common.cuh — bitset, hash, slot and atomic primitives for the MPDP
// level kernels (sm_100a).  Sets are fixed-width bitmaps:
// uint32_t for n <= 32 (every benchmark configuration), uint64_t above.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mpdp {

// ---------------------------------------------------------------- constants
constexpr int kBlock = 256;          // threads per CTA for every level kernel
constexpr int kRanksPerThread = 16;  // unrank one, Gosper-step 15 more
constexpr int kTile = kBlock * kRanksPerThread;
constexpr uint64_t kLightMax = 32;   // sets with <= 32 join pairs: thread per set
constexpr unsigned int kLightGeneral = 32;   // general graphs: CCP-checked sets above this go to CCC
constexpr int kSinkPairs = 2;        // join pairs whose memo probes are issued together
constexpr int kLightBlock = 128;     // k_eval_light CTA size
constexpr int kLightMinBlocks = 5;   // k_eval_light occupancy target -> <= 102 registers
constexpr int kMaxN = 56;            // exact path bound (masks <= 2^56 ranks)
constexpr int kMaxShards = 16;       // simulated multi-GPU world (one device)

enum GraphClass : int { CLS_TREE = 0, CLS_CLIQUE = 1, CLS_GENERAL = 2 };

// ------------------------------------------------------------ bit utilities
__device__ __forceinline__ int popc(uint32_t x) { return __popc(x); }
__device__ __forceinline__ int popc(uint64_t x) { return __popcll(x); }
__device__ __forceinline__ int ctz(uint32_t x) { return __ffs(x) - 1; }
__device__ __forceinline__ int ctz(uint64_t x) { return __ffsll((long long)x) - 1; }
template <typename M> __device__ __forceinline__ M lowbit(M x) { return x & (M)(0 - x); }
template <typename M> __device__ __forceinline__ M bitm(int v) { return (M)1 << v; }

// next larger integer with the same popcount == next k-subset in colex order
// (the "next lexicographical bit permutation" of P:924-926)
template <typename M> __device__ __forceinline__ M gosper(M v) {
    M t = v | (v - 1);
    return (t + 1) | (((~t & (M)(0 - ~t)) - 1) >> (ctz(v) + 1));
}

// position of the (t+1)-th lowest set bit of x (t = 0 -> lowest)
__device__ __forceinline__ int nth_bit(uint32_t x, int t) { return (int)__fns(x, 0, t + 1); }
__device__ __forceinline__ int nth_bit(uint64_t x, int t) {
    uint32_t lo = (uint32_t)x;
    int c = __popc(lo);
    if (t < c) return (int)__fns(lo, 0, t + 1);
    return 32 + (int)__fns((uint32_t)(x >> 32), 0, t - c + 1);
}

// parallel bit deposit (no PDEP on the GPU): bit i of j -> i-th set bit of R
template <typename M> __device__ __forceinline__ M deposit(uint64_t j, M R) {
    M out = 0;
    while (j) {
        int t = __ffsll((long long)j) - 1;
        out |= bitm<M>(nth_bit(R, t));
        j &= j - 1;
    }
    return out;
}

// deposit(j, R) for a small j (lane offsets, strides): walks R's elements
// while j has bits left -- at most log2(j) + 1 steps and no bit search
template <typename M> __device__ __forceinline__ M deposit_lo(unsigned int j, M R) {
    M out = 0;
    for (M T = R; j && T; T &= T - 1, j >>= 1)
        if (j & 1u) out |= T & (M)(0 - T);
    return out;
}

// ---------------------------------------------------------------- hashing
// Murmur3 finalisers ("fast Murmur3 hashing")
__device__ __forceinline__ uint32_t fmix(uint32_t h) {
    h ^= h >> 16; h *= 0x85ebca6bu; h ^= h >> 13; h *= 0xc2b2ae35u; h ^= h >> 16;
    return h;
}
__device__ __forceinline__ uint64_t fmix(uint64_t k) {
    k ^= k >> 33; k *= 0xff51afd7ed558ccdull; k ^= k >> 33; k *= 0xc4ceb9fe1a85ec53ull; k ^= k >> 33;
    return k;
}
// map a hash onto [0, n) without division (Lemire's multiply-high)
__device__ __forceinline__ uint64_t fastrange(uint32_t h, uint64_t n) {
    return (uint64_t)__umulhi(h, (uint32_t)n);   // n < 2^32 whenever masks are 32-bit
}
__device__ __forceinline__ uint64_t fastrange(uint64_t h, uint64_t n) {
    return (uint64_t)(((unsigned __int128)h * n) >> 64);
}

// ------------------------------------------------------------- memo slots
// One 16-byte slot = {tagged key, cost}; two slots form a 32-byte bucket = one
// L2 sector, so a probe that misses its first slot usually hits the second in
// the same sector.  The tag makes stale slots of earlier queries read as empty
// without clearing the table: tagged = mask | gen << 32 (n <= 32) or
// mask | gen8 << 56 (n <= 56).
struct __align__(16) Slot {
    unsigned long long key;
    double cost;
};
struct __align__(32) Bucket {
    Slot s[2];
};

template <typename M> struct Tag;
template <> struct Tag<uint32_t> {
    static __device__ __forceinline__ unsigned long long make(uint32_t S, uint32_t gen) {
        return (unsigned long long)S | ((unsigned long long)gen << 32);
    }
    static __device__ __forceinline__ uint32_t gen_of(unsigned long long w) { return (uint32_t)(w >> 32); }
};
template <> struct Tag<uint64_t> {
    static __device__ __forceinline__ unsigned long long make(uint64_t S, uint32_t gen) {
        return (unsigned long long)S | ((unsigned long long)(gen & 0xffu) << 56);
    }
    static __device__ __forceinline__ uint32_t gen_of(unsigned long long w) { return (uint32_t)(w >> 56); }
};

// ------------------------------------------------- (cost, left) min keys
// cost >= 0, so its IEEE bits order like unsigned integers; the lexicographic
// min over (cost_bits, left) is the tie-break of reading R7.
struct __align__(16) Key {
    unsigned long long c;   // __double_as_longlong(cost)
    unsigned long long l;   // left mask
};
__device__ __forceinline__ bool key_less(const Key& a, const Key& b) {
    return a.c < b.c || (a.c == b.c && a.l < b.l);
}
__device__ __forceinline__ Key key_inf() { return Key{0x7ff0000000000000ull, ~0ull}; }

__device__ __forceinline__ Key warp_min(Key k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        Key t;
        t.c = __shfl_xor_sync(0xffffffffu, k.c, o);
        t.l = __shfl_xor_sync(0xffffffffu, k.l, o);
        if (key_less(t, k)) k = t;
    }
    return k;
}

__device__ __forceinline__ void cas128(unsigned long long* p, unsigned long long elo, unsigned long long ehi,
                                       unsigned long long nlo, unsigned long long nhi,
                                       unsigned long long& olo, unsigned long long& ohi) {
    asm volatile(
        "{\n\t.reg .b128 d, e, n;\n\t"
        "mov.b128 e, {%2, %3};\n\t"
        "mov.b128 n, {%4, %5};\n\t"
        "atom.global.cas.b128 d, [%6], e, n;\n\t"
        "mov.b128 {%0, %1}, d;\n\t}"
        : "=l"(olo), "=l"(ohi)
        : "l"(elo), "l"(ehi), "l"(nlo), "l"(nhi), "l"(p)
        : "memory");
}

// merge a candidate into a 16-byte (cost, left) accumulator with a CAS loop
__device__ __forceinline__ void atomic_key_min(Key* dst, Key k) {
    unsigned long long* p = reinterpret_cast<unsigned long long*>(dst);
    unsigned long long clo = ((volatile unsigned long long*)p)[0];
    unsigned long long chi = ((volatile unsigned long long*)p)[1];
    while (key_less(k, Key{clo, chi})) {
        unsigned long long olo, ohi;
        cas128(p, clo, chi, k.c, k.l, olo, ohi);
        if (olo == clo && ohi == chi) return;
        clo = olo;
        chi = ohi;
    }
}

__device__ __forceinline__ uint64_t warp_sum(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace mpdp
