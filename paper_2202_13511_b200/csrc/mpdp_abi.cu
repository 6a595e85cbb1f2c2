// mpdp_abi.cu — host engine + C ABI (include/mpdp.h) of the B200 MPDP library.
//
// The host validates and stages the query graph (a0 of SURVEY §8(a)), carves
// the workspace, and enqueues the level loop of Alg. mpdp_gpu:
//   k_init -> for k = 2..n { k_enum<k> ; k_eval<k> } -> k_extract
// All on one CUDA stream with no host synchronisation between levels (the
// per-level table size and heavy-work counts live in device memory), so a
// query costs one H2D copy, 2n kernels and one D2H copy.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <dlfcn.h>
#include <string>
#include <vector>

#include "list_kernel.cuh"
#include "small_kernel.cuh"
#include "star_kernel.cuh"
#include "batch128.cuh"
#include "cluster_kernel.cuh"
#include "heuristics.h"

using namespace mpdp;

namespace {

thread_local std::string g_tls_error;

struct DevLayout {
    size_t query = 0, desc = 0, result = 0, gbar = 0, df = 0, segcnt = 0, rank = 0, tiles = 0, light = 0, heavy = 0, wh = 0, bkey = 0, bdone = 0,
           hcard = 0, hinfo = 0, hblk = 0,
           fh = 0, arena = 0, cold = 0, dcost = 0, dleft = 0, memo_end = 0, end = 0;
    int memo_kind = MEMO_HASH;
    bool mask_memo = false;               // dense arrays indexed by bitmask (MEMO_MASK)
    // multi-GPU sharding: per local shard its own level descriptors, result and
    // perfect-hash memo replica (shard 0 = the fields above)
    int nshards = 1;
    size_t sh_desc[kMaxShards] = {}, sh_result[kMaxShards] = {}, sh_dcost[kMaxShards] = {}, sh_dleft[kMaxShards] = {},
           sh_dcard[kMaxShards] = {}, sh_df[kMaxShards] = {};
    size_t xr = 0;                        // XrTable of the fused peer exchange
    unsigned long long list_cap = 0, heavy_cap = 0, tiles_cap = 0, fh_cap = 0, arena_buckets = 0;
};

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// ---- NCCL, loaded at run time (only multi-GPU contexts need it).  The few
// declarations below mirror nccl.h of NCCL 2.x; the library torch ships
// (nvidia-nccl, 2.28) is the one already mapped into the process.
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;
enum { kNcclUint32 = 3, kNcclUint64 = 5, kNcclFloat64 = 8 };
enum { kNcclSum = 0, kNcclMax = 2 };
struct NcclApi {
    void* lib = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi* nccl_api(std::string& err) {
    static NcclApi api;
    static bool tried = false;
    if (tried) {
        if (!api.lib) err = "libnccl.so.2 could not be loaded";
        return api.lib ? &api : nullptr;
    }
    tried = true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
        api.lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
        if (api.lib) break;
    }
    if (!api.lib) {
        err = "libnccl.so.2 could not be loaded";
        return nullptr;
    }
#define NCCL_SYM(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(api.lib, "nccl" #f))
    NCCL_SYM(GetUniqueId);
    NCCL_SYM(CommInitRank);
    NCCL_SYM(CommDestroy);
    NCCL_SYM(AllGather);
    NCCL_SYM(AllReduce);
    NCCL_SYM(GroupStart);
    NCCL_SYM(GroupEnd);
    NCCL_SYM(GetErrorString);
#undef NCCL_SYM
    if (!api.GetUniqueId || !api.CommInitRank || !api.AllGather || !api.AllReduce || !api.GroupStart || !api.GroupEnd) {
        err = "libnccl.so.2 lacks required symbols";
        api.lib = nullptr;
        return nullptr;
    }
    return &api;
}

}  // namespace

struct mpdp_ctx {
    int device = 0, rank = 0, world = 1;
    bool simulate = false;                // world ranks simulated as shards on this device
    // MPDP_FLAG_NCCL_SELF (testing): world == 1 with a real 1-rank NCCL
    // communicator, every query on the sharded path with every level sharded
    bool nccl_self = false;
    bool multi = false;                   // the sharded path: world > 1 || nccl_self
    // fused peer exchange (MPDP_FLAG_FUSED_EXCHANGE, star queries): every
    // rank's workspace (IPC-mapped peers, [rank] = ws), the staging of the
    // XrTable, and the number of fused-exchange queries run (start barrier)
    unsigned char* peer_ws[kMaxXr] = {};
    bool peers_open = false;
    void* h_xr = nullptr;
    unsigned int xr_epoch = 0;
    bool xr_run = false;                  // the last run used the fused exchange
    NcclApi* nccl = nullptr;
    ncclComm_t comm = nullptr;
    ResultDev* h_results = nullptr;       // pinned, one per local shard
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    unsigned char* ws = nullptr;
    size_t ws_bytes = 0;
    bool own_ws = false;
    int num_sms = 0;
    double timeout_ms = 0;
    std::string err;

    // staged query
    int n = 0, cls = CLS_TREE;
    unsigned long long m = 0;             // edges of the staged query
    bool wide = false;                    // 64-bit masks
    bool staged = false;
    std::vector<unsigned long long> binom;
    void* h_query = nullptr;              // pinned QueryDev<uint64_t>-sized buffer
    ResultDev* h_result = nullptr;        // pinned
    DevLayout lay;
    unsigned int gen32 = 0, gen8 = 0;
    int last_width = 0;
    unsigned long long query_counter = 0;
    unsigned int launches = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    bool ran = false;
    int occ[2][3][2][3] = {};            // [wide][class][memo][enum, light, heavy]
    int fused_occ[6] = {}, fused_n[6] = {};   // [CLS + 3 * mask_memo]
    // occupancy of the whole-query kernels per (slot, n) -- the dynamic shared
    // memory (rank tables) depends on n; the heuristics' inner DPs change n on
    // almost every call, and re-querying cost ~0.1 ms of host time per call
    int occ_by_n[6][kMaxN + 1] = {};
    bool attr_set[6] = {};
    bool small_attr[3] = {};              // k_dp_small<CLS>: dynamic smem attribute set
    bool small = false;                   // last query ran a single-CTA kernel
    bool tree1_attr = false;
    bool tree1 = false;                   // last query ran k_dp_tree1 (memo_kind 1, global memo)
    // mpdp_optimize_batch: per-query device / pinned staging of the batched
    // single-CTA launch
    QueryDev<uint32_t>* d_bq = nullptr;
    ResultDev* d_br = nullptr;
    QueryDev<uint32_t>* h_bq = nullptr;
    ResultDev* h_br = nullptr;
    uint32_t batch_cap = 0;
    bool batch_attr = false;
    int star_hub = -1;                    // star queries: the relation adjacent to all others
    bool memo_conn = false;               // general graph, bitmask memo pre-filled absent (R20)
    int star_occ = 0;                     // k_dp_star CTAs per SM
    int star_occ_xr = 0;                  // k_dp_star<true> (fused peer exchange)
    int clique_xr_occ = 0;                // k_dp_clique_df<true> (fused peer exchange)
    int cluster_size = 0;                 // k_dp_tree_cluster: CTAs per cluster (0 = not probed yet)
    int clique_df_occ = 0;                // k_dp_clique_df (ablation) CTAs per SM
    bool clique_df_attr = false;
    bool star = false;                    // last query ran k_dp_star (memo_kind 4)
    unsigned long long tree_max_level = 0;  // tree queries: largest level (connected sets of one size)
    unsigned long long tree_csg = 0;        // tree queries: connected sets (subtree count)
    // mpdp_optimize_batch, mid-size tree sub-problems: one CTA each, a shared
    // memo with 128-bit {sub-problem, mask} keys (batch128.cuh)
    Key128* b_keys = nullptr;
    Val128* b_vals = nullptr;
    unsigned long long b_cap = 0;
    unsigned int b_epoch = 0;
    unsigned int* d_sub_ids = nullptr;
    unsigned int* h_sub_ids = nullptr;
    bool batch128_attr = false;
    bool fused = false;                  // last run used the fused kernel
    // the level descriptors are zero (the dataflow kernels leave them zeroed;
    // every k_init-based path leaves them dirty): the star / clique dataflow
    // launch needs no k_init when this holds
    bool desc_clean = true;
    bool sharded = false;                // last run used the sharded (multi-GPU) path
    struct SubProblem {                  // MPDP_FLAG_RECORD_SUBPROBLEMS
        std::vector<double> card, sel, leaf;
        std::vector<uint32_t> edges;
        std::vector<mpdp_plan_node> nodes;
        mpdp_result res;
    };
    std::vector<SubProblem> subs;
    int occ_n[2][3][2] = {};
    unsigned int flags = 0;
    double load_factor = 0.5;
    int last_memo = -1;
    struct GraphEntry {
        cudaGraphExec_t exec;
        unsigned int launches, enum_launches, eval_launches;
        int nkev;
    };
    std::map<unsigned long long, GraphEntry> graphs;   // level loop per (n, class, memo, width, flags)
    int rank_n = -1;                      // n the uploaded rank tables were built for
    std::vector<unsigned int> rank_cache[33];   // host rank tables per n
    unsigned int* h_rank_pinned = nullptr;  // staging of the async rank-table upload
    cudaEvent_t kev[2 * kMaxN + 2] = {};  // MPDP_FLAG_PROFILE_KERNELS: around every level kernel
    int nkev = 0;
    unsigned int enum_launches = 0, eval_launches = 0;
    size_t h2d_bytes = 0, d2h_bytes = 0;
};

static mpdp_status fail(mpdp_ctx* c, mpdp_status s, const std::string& msg) {
    g_tls_error = msg;
    if (c) c->err = msg;
    return s;
}

#define CUDA_TRY(ctx, x)                                                                      \
    do {                                                                                      \
        cudaError_t e_ = (x);                                                                 \
        if (e_ != cudaSuccess)                                                                \
            return fail(ctx, e_ == cudaErrorMemoryAllocation ? MPDP_ERR_OOM : MPDP_ERR_CUDA, \
                        std::string(#x) + ": " + cudaGetErrorString(e_));                     \
    } while (0)

static unsigned long long binom_u64(int n, int k) {
    if (k < 0 || k > n) return 0;
    if (k > n - k) k = n - k;
    unsigned long long r = 1;
    for (int i = 1; i <= k; i++) r = r / i * (n - k + i) + r % i * (n - k + i) / i;
    return r;
}

static unsigned long long sat_mul(unsigned long long a, unsigned long long b) {
    if (a && b > ~0ull / a) return ~0ull;
    return a * b;
}

// ------------------------------------------------------------ validation
static mpdp_status validate(mpdp_ctx* c, const mpdp_query_graph* g, std::vector<unsigned long long>& adj) {
    if (!g) return fail(c, MPDP_ERR_INVALID_ARGUMENT, "graph is NULL");
    if (g->n == 0) return fail(c, MPDP_ERR_INVALID_ARGUMENT, "n == 0");
    if (g->n > (uint32_t)kMaxN)
        return fail(c, MPDP_ERR_CAPACITY, "exact MPDP supports n <= 56 relations (unranking bound)");
    if (!g->cardinalities) return fail(c, MPDP_ERR_INVALID_ARGUMENT, "cardinalities is NULL");
    if (g->n_edges && (!g->edges || !g->selectivities))
        return fail(c, MPDP_ERR_INVALID_ARGUMENT, "edges/selectivities is NULL");
    const int n = (int)g->n;
    adj.assign(n, 0);
    double lsum = 0;
    for (int v = 0; v < n; v++) {
        const double x = g->cardinalities[v];
        if (!(x >= 0.0) || !std::isfinite(x))
            return fail(c, MPDP_ERR_INVALID_ARGUMENT, "cardinality[" + std::to_string(v) + "] not finite >= 0");
        lsum += std::log10(std::max(x, 1.0));
        if (g->leaf_costs && (!(g->leaf_costs[v] >= 0.0) || !std::isfinite(g->leaf_costs[v])))
            return fail(c, MPDP_ERR_INVALID_ARGUMENT, "leaf_costs[" + std::to_string(v) + "] not finite >= 0");
    }
    if (lsum > 300.0) return fail(c, MPDP_ERR_INVALID_ARGUMENT, "sum of log10 cardinalities > 300");
    for (uint32_t e = 0; e < g->n_edges; e++) {
        const uint32_t u = g->edges[2 * e], v = g->edges[2 * e + 1];
        const double s = g->selectivities[e];
        if (!(u < v) || v >= g->n)
            return fail(c, MPDP_ERR_INVALID_ARGUMENT, "edge " + std::to_string(e) + " not u < v < n");
        if (adj[u] >> v & 1ull) return fail(c, MPDP_ERR_INVALID_ARGUMENT, "duplicate edge " + std::to_string(e));
        if (!(s > 0.0) || !(s <= 1.0))
            return fail(c, MPDP_ERR_INVALID_ARGUMENT, "selectivity " + std::to_string(e) + " outside (0,1]");
        adj[u] |= 1ull << v;
        adj[v] |= 1ull << u;
    }
    // connectivity (no cross products): host BFS over the adjacency
    unsigned long long seen = 1ull, frontier = 1ull;
    while (frontier) {
        unsigned long long nx = 0;
        for (unsigned long long f = frontier; f; f &= f - 1) nx |= adj[__builtin_ctzll(f)];
        nx &= ~seen;
        seen |= nx;
        frontier = nx;
    }
    const unsigned long long all = (n == 64) ? ~0ull : ((1ull << n) - 1);
    if (seen != all) return fail(c, MPDP_ERR_DISCONNECTED, "query graph is not connected (cross products excluded)");
    return MPDP_OK;
}

// ------------------------------------------------------------ staging
template <typename M>
static void fill_query(mpdp_ctx* c, const mpdp_query_graph* g, const std::vector<unsigned long long>& adj,
                       QueryDev<M>* q) {
    const int n = (int)g->n;
    memset(q, 0, sizeof(QueryDev<M>));
    q->n = n;
    q->cls = c->cls;
    q->dpsub = (c->flags & MPDP_FLAG_DPSUB_ENUM) ? 1 : 0;
    q->epoch = c->query_counter << 6;     // + level k (k <= 56 < 64)
    q->gen = c->wide ? c->gen8 : c->gen32;
    q->has_leaf_costs = 0;
    for (int v = 0; v < n; v++) {
        q->adj[v] = (M)adj[v];
        q->card[v] = g->cardinalities[v];
        q->leaf[v] = g->leaf_costs ? g->leaf_costs[v] : 0.0;
        if (q->leaf[v] != 0.0) q->has_leaf_costs = 1;
    }
    for (uint32_t e = 0; e < g->n_edges; e++) {
        const uint32_t u = g->edges[2 * e], v = g->edges[2 * e + 1];
        q->sel[u * n + v] = q->sel[v * n + u] = g->selectivities[e];
    }
    if (c->cls == CLS_TREE) {             // root the tree at 0: subtree masks + depth masks
        std::vector<int> order, parent(n, -1), depth(n, 0);
        order.push_back(0);
        parent[0] = 0;
        for (size_t i = 0; i < order.size(); i++) {
            const int v = order[i];
            for (unsigned long long a = adj[v]; a; a &= a - 1) {
                const int u = __builtin_ctzll(a);
                if (parent[u] < 0) {
                    parent[u] = v;
                    depth[u] = depth[v] + 1;
                    order.push_back(u);
                }
            }
        }
        std::vector<unsigned long long> desc(n, 0);
        for (int i = (int)order.size() - 1; i >= 0; i--) {
            const int v = order[i];
            desc[v] |= 1ull << v;
            if (v != 0) desc[parent[v]] |= desc[v];
        }
        int maxd = 0;
        for (int v = 0; v < n; v++) {
            q->desc[v] = (M)desc[v];
            q->depth_mask[depth[v]] |= (M)1 << v;
            maxd = std::max(maxd, depth[v]);
        }
        q->max_depth = maxd;
        // connected sets per size (subtrees of the tree): with f_v(x) the
        // generating polynomial of the subtrees whose top vertex is v,
        // f_v = x * prod over children u of (1 + f_u); level s holds sum_v [x^s] f_v
        std::vector<std::vector<unsigned long long>> f(n);
        std::vector<unsigned long long> cnt(n + 1, 0);
        for (int i = (int)order.size() - 1; i >= 0; i--) {
            const int v = order[i];
            std::vector<unsigned long long> a(2, 0);
            a[1] = 1;
            for (int u = 0; u < n; u++) {
                if (u == v || parent[u] != v) continue;
                std::vector<unsigned long long> b(a.size() + f[u].size() - 1, 0);
                for (size_t x = 0; x < a.size(); x++) {
                    if (!a[x]) continue;
                    b[x] += a[x];                                // the child's subtree left out
                    for (size_t y = 1; y < f[u].size(); y++) b[x + y] += a[x] * f[u][y];
                }
                a.swap(b);
            }
            for (size_t x = 0; x < a.size() && x <= (size_t)n; x++) cnt[x] += a[x];
            f[v].swap(a);
        }
        c->tree_max_level = 0;
        c->tree_csg = (unsigned long long)n;
        for (int x = 2; x <= n; x++) {
            c->tree_max_level = std::max(c->tree_max_level, cnt[x]);
            c->tree_csg += cnt[x];
        }
        c->star_hub = -1;
        for (int v = 0; v < n && n >= 3; v++)
            if (__builtin_popcountll(adj[v]) == n - 1) c->star_hub = v;
    }
    // the binomial table is the same for every query: built once per width
    // (1089 / 4225 binom_u64 calls with divisions were ~0.1 ms of host time
    // per query)
    constexpr int NB = MaxN<M>::value + 1;
    static const std::vector<unsigned long long> table = [] {
        std::vector<unsigned long long> t(NB * NB);
        for (int i = 0; i < NB; i++)
            for (int j = 0; j < NB; j++) t[i * NB + j] = binom_u64(i, j);
        return t;
    }();
    memcpy(q->binom, table.data(), sizeof(unsigned long long) * NB * NB);
}

// general graphs: sets with more CCP-checked candidates than this are heavy
static unsigned int light_max_general() {
    const char* e = getenv("MPDP_DEBUG_LIGHT_GENERAL");         // experiments only
    return e ? (unsigned int)std::max(1, std::min(32, atoi(e))) : kLightGeneral;
}

static unsigned long long heavy_pair_bound(int n, int k, int cls) {
    const unsigned long long C = binom_u64(n, k);
    if (cls == CLS_TREE) return (k - 1 > (int)kLightMax) ? sat_mul(C, (unsigned long long)(k - 1)) : 0ull;
    if (k - 1 >= 63) return ~0ull;
    const unsigned long long w = (1ull << (k - 1)) - 1;
    if (w <= (cls == CLS_GENERAL ? (unsigned long long)light_max_general() : kLightMax)) return 0;
    return sat_mul(C, w);
}

static unsigned long long level_item(int n, int k, int cls, unsigned long long fh_cap) {
    const unsigned long long ub = heavy_pair_bound(n, k, cls);
    unsigned long long item = 256;
    if (cls == CLS_GENERAL) {
        const char* e = getenv("MPDP_DEBUG_ITEM_GENERAL");     // experiments only
        item = e ? std::max(32ull, strtoull(e, nullptr, 10)) : 256ull;
    }
    if (fh_cap && ub / fh_cap + 1 > item) item = ub / fh_cap + 1;
    return (item + 31) / 32 * 32;
}

// Workspace layout: [header | memo arena (buckets) | cold left[] | scratch].
// The arena has a fixed position and size for a given (workspace, mask width),
// so stale bytes inside it are always memo slots of earlier queries (their tag
// differs) and never need clearing; the per-query scratch (look-back ring, level
// lists, heavy bookkeeping) lives after it.
static mpdp_status plan_layout(mpdp_ctx* c) {
    DevLayout L;
    const int n = c->n;
    const size_t msz = c->wide ? 8 : 4;
    unsigned long long list_cap = 1, tiles_cap = 1, heavy_cap = 1, fh_need = 1;
    for (int k = 2; k <= n; k++) {
        const unsigned long long C = binom_u64(n, k);
        list_cap = std::max(list_cap, C);
        tiles_cap = std::max(tiles_cap, (C + kTile - 1) / kTile);
        const unsigned long long ub = heavy_pair_bound(n, k, c->cls);
        if (ub) {
            heavy_cap = std::max(heavy_cap, C);
            fh_need = std::max(fh_need, std::min<unsigned long long>(ub / 256 + 2, 1ull << 24));
        }
    }
    size_t off = 0;
    auto take = [&](size_t bytes) {
        off = align_up(off, 256);
        const size_t at = off;
        off += bytes;
        return at;
    };
    const int W = c->world, nsh = c->simulate ? c->world : 1;
    L.nshards = nsh;
    L.query = take(sizeof(QueryDev<uint64_t>));
    for (int sh = 0; sh < nsh; sh++) {
        L.sh_desc[sh] = take(sizeof(LevelDesc) * (kMaxN + 1));
        L.sh_result[sh] = take(sizeof(ResultDev));
    }
    L.desc = L.sh_desc[0];
    L.result = L.sh_result[0];
    L.gbar = take(64);
    for (int sh = 0; sh < nsh; sh++) L.sh_df[sh] = take(sizeof(DataflowDev));
    L.df = L.sh_df[0];
    L.xr = take(sizeof(XrTable));
    L.segcnt = take(4 * 2 * kMaxGrid);
    L.rank = take(sizeof(unsigned int) * 256 * (1 + 9 + 17 + 25));
    off = align_up(off, 256);
    if (off + (64u << 20) > c->ws_bytes) return fail(c, MPDP_ERR_CAPACITY, "workspace smaller than 64 MiB");
    const size_t body = c->ws_bytes - off - 1024;
    const size_t memo_bytes = body * 3 / 4;
    const size_t memo0 = off;
    // memo region (fixed position): DENSE = cost[] + card[] + left[] over all C(n,k);
    // HASH = buckets + cold left[] (geometry fixed per mask width)
    // dense levels are padded by W entries so that W equal rank segments of
    // ceil(C(n,k)/W) fit (in-place allgather of the sharded levels)
    unsigned long long dense_entries = 0;
    for (int k = 2; k <= n; k++) dense_entries += binom_u64(n, k) + (unsigned long long)W;
    // MEMO_MASK: clique / general queries on one GPU through the whole-query
    // kernel index the same arrays by bitmask (2^n entries)
    // (multi-GPU cliques with the fused peer exchange keep the bitmask memo:
    // every rank holds a full replica of it)
    const bool xr_clique = c->multi && !c->nccl_self && c->cls == CLS_CLIQUE && (c->flags & MPDP_FLAG_FUSED_EXCHANGE);
    const bool mask = c->cls != CLS_TREE && (!c->multi || xr_clique) && !c->wide && n >= 2 && n <= kMaskMaxN &&
                      !(c->flags & (MPDP_FLAG_HASH_MEMO | MPDP_FLAG_RANK_MEMO | MPDP_FLAG_NO_FUSED |
                                    MPDP_FLAG_PROFILE_KERNELS)) &&
                      (c->timeout_ms <= 0 || c->cls == CLS_CLIQUE);   // (k_dp_clique checks the deadline)
    if (mask) dense_entries = std::max(dense_entries, 1ull << n);
    const size_t dense_bytes = 2 * align_up(8 * dense_entries, 256) + align_up(4 * dense_entries, 256);
    const bool dense_ok = !c->wide && !(c->flags & MPDP_FLAG_HASH_MEMO) &&
                          (size_t)nsh * dense_bytes + 1024 <= memo_bytes;
    L.memo_kind = dense_ok ? MEMO_DENSE : MEMO_HASH;
    L.mask_memo = dense_ok && mask;
    if (c->multi && !dense_ok)
        return fail(c, MPDP_ERR_CAPACITY, "multi-GPU sharding needs the perfect-hash memo (n <= 32) and " +
                                              std::to_string(nsh * dense_bytes >> 20) + " MiB of memo space");
    const unsigned long long buckets = (unsigned long long)(memo_bytes / (sizeof(Bucket) + 2 * msz));
    L.arena = take(sizeof(Bucket) * buckets);
    L.cold = take(2 * msz * buckets);
    for (int sh = 0; sh < nsh; sh++) {
        L.sh_dcost[sh] = memo0 + sh * dense_bytes;
        L.sh_dcard[sh] = align_up(L.sh_dcost[sh] + 8 * dense_entries, 256);
        L.sh_dleft[sh] = align_up(L.sh_dcard[sh] + 8 * dense_entries, 256);
    }
    L.dcost = L.sh_dcost[0];
    L.dleft = L.sh_dleft[0];
    L.memo_end = off;
    const size_t scratch0 = align_up(off, 256);
    const size_t scratch = c->ws_bytes - scratch0 - 1024;
    // level lists are bounded by C(n,k) and by the scratch space (sparse graphs with
    // large n keep few of their C(n,k) subsets); overflow is detected on the device
    // ring >= 4096 records: more than the tiles that can be in flight at once
    // (resident CTAs), and never smaller than the tile count of the smallest tile
    // size (the fused kernel uses 2048-rank tiles)
    tiles_cap = tiles_cap * (kTile / kFusedTile) + 1;
    unsigned long long ring = 4096;
    while (ring < tiles_cap && ring < (1ull << 20)) ring <<= 1;
    tiles_cap = ring;
    const size_t fixed = sizeof(TileRec) * tiles_cap + 4 * fh_need + 4096;
    if (fixed >= scratch) return fail(c, MPDP_ERR_CAPACITY, "workspace too small for n = " + std::to_string(n));
    const size_t avail = scratch - fixed;
    // the list kernel's level lists are segmented per CTA (segments of blockDim *
    // ranks-per-thread entries), which can exceed C(n,k) by one rank per thread
    list_cap += (unsigned long long)kMaxGrid * kBlock;
    // tree queries: the list kernel generates level k+1 from level k's sets in
    // per-CTA segments of (sets per CTA + 1) * (n - k) entries (emit_children /
    // expand_to_list); when this does not fit, it falls back to the rank scan
    if (c->cls == CLS_TREE)
        for (int k = 2; k < n; k++)
            list_cap = std::max(list_cap, sat_mul(binom_u64(n, k) + 2ull * kMaxGrid, (unsigned long long)(n - k)));
    // cliques with the bitmask memo merge split sets through (key, key, count)
    // slots per warp chunk of each split level (about one per warp of the grid
    // per split level: k_dp_clique)
    if (L.mask_memo && c->cls == CLS_CLIQUE)
        heavy_cap = std::max<unsigned long long>(heavy_cap, 8ull * kMaxGrid * (kBlock / 32));
    list_cap = std::min<unsigned long long>(list_cap, (avail / 2) / 16);   // fused: two lists of (rank << 32 | mask)
    heavy_cap = std::min<unsigned long long>(heavy_cap, (avail / 2) / (msz + 44 + msz * kHeavyBlk));
    if (L.mask_memo && c->cls == CLS_CLIQUE && heavy_cap < 8ull * kMaxGrid * (kBlock / 32))
        return fail(c, MPDP_ERR_CAPACITY, "workspace too small for the clique merge slots");
    L.tiles = take(sizeof(TileRec) * tiles_cap);
    L.light = take(16 * list_cap);
    L.heavy = take(msz * heavy_cap);
    L.wh = take(8 * (heavy_cap + 1));
    L.bkey = take(16 * heavy_cap);
    L.bdone = take(8 * heavy_cap);
    L.hcard = take(8 * heavy_cap);
    L.hinfo = take(4 * heavy_cap);
    L.hblk = take(msz * kHeavyBlk * heavy_cap);
    L.fh = take(4 * fh_need);
    L.end = off;
    if (L.end > c->ws_bytes) return fail(c, MPDP_ERR_INTERNAL, "layout overflow");
    L.list_cap = list_cap;
    L.heavy_cap = heavy_cap;
    L.tiles_cap = tiles_cap;
    L.fh_cap = fh_need;
    L.arena_buckets = buckets;
    c->lay = L;
    return MPDP_OK;
}

template <typename M>
static Params<M> make_params(mpdp_ctx* c, int shard = 0) {
    Params<M> p;
    memset(&p, 0, sizeof(p));
    unsigned char* b = c->ws;
    const DevLayout& L = c->lay;
    p.q = reinterpret_cast<const QueryDev<M>*>(b + L.query);
    p.desc = reinterpret_cast<LevelDesc*>(b + L.sh_desc[shard]);
    p.memo.arena = reinterpret_cast<Bucket*>(b + L.arena);
    p.memo.cold = b + L.cold;
    p.memo.arena_buckets = L.arena_buckets;
    p.memo.dcost = reinterpret_cast<double*>(b + L.sh_dcost[shard]);
    p.memo.dleft = reinterpret_cast<unsigned int*>(b + L.sh_dleft[shard]);
    p.memo.dcard = reinterpret_cast<double*>(b + L.sh_dcard[shard]);
    p.memo.rank_tab = reinterpret_cast<const unsigned int*>(b + L.rank);
    p.memo.rg = rank_geom(c->n <= 32 ? c->n : 32);
    p.memo.error = &reinterpret_cast<ResultDev*>(b + L.sh_result[shard])->error;
    p.memo_kind = L.memo_kind;
    p.gbar = reinterpret_cast<unsigned int*>(b + L.gbar);
    p.df = reinterpret_cast<DataflowDev*>(b + L.sh_df[shard]);
    // debug: per-CTA timing words of the dataflow kernels in the (unused by
    // them) level-list scratch
    p.df_stats = getenv("MPDP_DEBUG_DF_STATS") ? reinterpret_cast<unsigned long long*>(b + L.light) : nullptr;
    p.timeout_ns = c->timeout_ms > 0 ? (unsigned long long)(c->timeout_ms * 1e6) : 0ull;
    p.seg_cnt = reinterpret_cast<unsigned int*>(b + L.segcnt);
    p.heavy_levels = 0;
    for (int k = 2; k <= c->n; k++) {
        if (heavy_pair_bound(c->n, k, c->cls)) p.heavy_levels |= 1ull << k;
        p.item_of[k] = level_item(c->n, k, c->cls, L.fh_cap);
    }
    unsigned long long acc = 0;
    for (int k = 0; k <= kMaxN; k++) {
        p.dense_off[k] = acc;
        if (k >= 2 && k <= c->n) acc += binom_u64(c->n, k) + (unsigned long long)c->world;   // + padding
    }
    // single-launch defaults: every level, whole rank space, counted, extracted
    p.k_begin = 2;
    p.k_end = c->n;
    p.do_extract = 1;
    p.count_levels = ~0ull;
    for (int k = 0; k <= kMaxN; k++) {
        p.share_lo[k] = 0;
        p.share_hi[k] = (k >= 2 && k <= c->n) ? (unsigned int)binom_u64(c->n, k) : 0u;
    }
    p.light = reinterpret_cast<M*>(b + L.light);
    p.heavy = reinterpret_cast<M*>(b + L.heavy);
    p.wh = reinterpret_cast<unsigned long long*>(b + L.wh);
    p.bkey = reinterpret_cast<Key*>(b + L.bkey);
    p.bdone = reinterpret_cast<unsigned long long*>(b + L.bdone);
    p.hcard = reinterpret_cast<double*>(b + L.hcard);
    p.hinfo = reinterpret_cast<unsigned int*>(b + L.hinfo);
    p.hblk = reinterpret_cast<M*>(b + L.hblk);
    p.first_heavy = reinterpret_cast<unsigned int*>(b + L.fh);
    p.fh_cap = L.fh_cap;
    p.tiles = reinterpret_cast<TileRec*>(b + L.tiles);
    p.tiles_ring = L.tiles_cap;
    p.list_cap = L.list_cap;
    p.heavy_cap = L.heavy_cap;
    p.result = reinterpret_cast<ResultDev*>(b + L.sh_result[shard]);
    p.epoch_salt = shard;
    p.n = c->n;
    p.inv_load = 1.0 / c->load_factor;
    p.no_ccc = (c->flags & MPDP_FLAG_NO_CCC) ? 1 : 0;
    p.light_max = light_max_general();
    p.memo_conn = c->memo_conn ? 1 : 0;
    p.heavy_whole = getenv("MPDP_DEBUG_HEAVY_WHOLE") ? strtoull(getenv("MPDP_DEBUG_HEAVY_WHOLE"), nullptr, 10) : 2048;
    p.expand_fac = getenv("MPDP_DEBUG_EXPAND_FAC") ? atof(getenv("MPDP_DEBUG_EXPAND_FAC")) : 0.1;
    p.clique_split_w = getenv("MPDP_DEBUG_CLIQUE_SPLIT") ? strtoull(getenv("MPDP_DEBUG_CLIQUE_SPLIT"), nullptr, 10) : 4096;
    p.clique_set_cost = getenv("MPDP_DEBUG_CLIQUE_SETCOST") ? atof(getenv("MPDP_DEBUG_CLIQUE_SETCOST")) : kCliqueSetCost;
    p.clique_split_fac = getenv("MPDP_DEBUG_CLIQUE_SPLITFAC") ? atof(getenv("MPDP_DEBUG_CLIQUE_SPLITFAC")) : 1.0;
    p.clique_csize_min = getenv("MPDP_DEBUG_CLIQUE_CSIZE") ? strtoull(getenv("MPDP_DEBUG_CLIQUE_CSIZE"), nullptr, 10) : 512;
    p.star_hub = c->star_hub;
    {   // star levels: C(n-1, k-1) entries + `world` padding (equal rank segments, as dense_off)
        unsigned long long so = 0;
        for (int k = 0; k <= kMaxN; k++) {
            p.star_off[k] = so;
            if (k >= 2 && k <= c->n) so += binom_u64(c->n - 1, k - 1) + (unsigned long long)c->world;
        }
    }
    return p;
}

template <typename M, int CLS, int MEMO>
static mpdp_status prepare_kernels(mpdp_ctx* c) {
    const size_t smem_enum = sizeof(SQ<M>) + sizeof(unsigned long long) * (MaxN<M>::value + 1) * (MaxN<M>::value + 1);
    const size_t smem_eval = sizeof(SQ<M>) + (MEMO == MEMO_DENSE ? sizeof(unsigned int) * (rank_geom(c->n).entries + 33 * 33) : 0);
    const size_t smem_max = sizeof(SQ<M>) + sizeof(unsigned int) * (256 * (1 + 9 + 17 + 25) + 33 * 33);
    int* occ = c->occ[c->wide][CLS][MEMO];   // {enum, light, heavy} CTAs per SM
    if (!occ[0] || c->occ_n[c->wide][CLS][MEMO] != c->n) {
        CUDA_TRY(c, cudaFuncSetAttribute(k_enum<M, CLS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_enum));
        CUDA_TRY(c, cudaFuncSetAttribute(k_eval_light<M, CLS, MEMO>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max));
        CUDA_TRY(c, cudaFuncSetAttribute(k_eval_heavy<M, CLS, MEMO>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max));
        CUDA_TRY(c, cudaFuncSetAttribute(k_extract<M, MEMO>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max));
        CUDA_TRY(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[0], k_enum<M, CLS>, kBlock, smem_enum));
        CUDA_TRY(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[1], k_eval_light<M, CLS, MEMO>, kLightBlock, smem_eval));
        CUDA_TRY(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[2], k_eval_heavy<M, CLS, MEMO>, kBlock, smem_eval));
        for (int i = 0; i < 3; i++) occ[i] = std::max(occ[i], 1);
        c->occ_n[c->wide][CLS][MEMO] = c->n;
    }
    return MPDP_OK;
}

// Enqueue the whole query on c->stream: k_init, per level k_enum + evaluate,
// k_extract, and the D2H copy of the result.  Used directly (timeout mode) or
// under stream capture to build the cached CUDA graph.
template <typename M, int CLS, int MEMO>
static mpdp_status enqueue_query(mpdp_ctx* c, const Params<M>& p, bool sync_levels) {
    const size_t smem_enum = sizeof(SQ<M>) + sizeof(unsigned long long) * (MaxN<M>::value + 1) * (MaxN<M>::value + 1);
    const size_t smem_eval = sizeof(SQ<M>) + (MEMO == MEMO_DENSE ? sizeof(unsigned int) * (rank_geom(c->n).entries + 33 * 33) : 0);
    const int* occ = c->occ[c->wide][CLS][MEMO];
    const bool prof = c->flags & MPDP_FLAG_PROFILE_KERNELS;
    const auto t0 = std::chrono::steady_clock::now();
    c->nkev = 0;
    c->enum_launches = c->eval_launches = 0;
    k_init<M><<<1, 64, 0, c->stream>>>(p);
    c->launches = 1;
    if (prof && c->n >= 2) CUDA_TRY(c, cudaEventRecord(c->kev[c->nkev++], c->stream));
    for (int k = 2; k <= c->n; k++) {
        const unsigned long long nranks = binom_u64(c->n, k);
        const unsigned long long ntiles = (nranks + kTile - 1) / kTile;
        const unsigned long long item = level_item(c->n, k, CLS, c->lay.fh_cap);
        const unsigned int grid_enum = (unsigned int)std::min<unsigned long long>(ntiles, (unsigned long long)c->num_sms * occ[0]);
        // a level has at most C(n,k) light sets: no more light CTAs than that
        const unsigned long long light_ctas = (nranks + kLightBlock - 1) / kLightBlock;
        const unsigned int grid_light = (unsigned int)std::min<unsigned long long>(light_ctas, (unsigned long long)c->num_sms * occ[1]);
        k_enum<M, CLS><<<grid_enum, kBlock, smem_enum, c->stream>>>(p, k, nranks, ntiles, item);
        if (prof) CUDA_TRY(c, cudaEventRecord(c->kev[c->nkev++], c->stream));
        k_eval_light<M, CLS, MEMO><<<grid_light, kLightBlock, smem_eval, c->stream>>>(p, k);
        c->launches += 2;
        if (heavy_pair_bound(c->n, k, CLS)) {
            k_eval_heavy<M, CLS, MEMO><<<c->num_sms * occ[2], kBlock, smem_eval, c->stream>>>(p, k, item);
            c->launches++;
        }
        if (prof) CUDA_TRY(c, cudaEventRecord(c->kev[c->nkev++], c->stream));
        c->enum_launches++;
        c->eval_launches++;
        CUDA_TRY(c, cudaGetLastError());
        if (sync_levels && c->timeout_ms > 0) {
            CUDA_TRY(c, cudaStreamSynchronize(c->stream));
            const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            if (ms > c->timeout_ms) return fail(c, MPDP_ERR_TIMEOUT, "timeout after level " + std::to_string(k));
        }
    }
    k_extract<M, MEMO><<<1, 64, smem_eval, c->stream>>>(p);
    c->launches++;
    CUDA_TRY(c, cudaGetLastError());
    CUDA_TRY(c, cudaMemcpyAsync(c->h_result, c->ws + c->lay.result, sizeof(ResultDev), cudaMemcpyDeviceToHost, c->stream));
    c->d2h_bytes = sizeof(ResultDev);
    return MPDP_OK;
}

// The whole-query kernel of a class: trees (no heavy sets) use the level-list
// kernel with enumerate-ahead, the other classes the tile kernel.
template <int CLS>
static const void* level_loop_kernel(bool mask_memo = false) {
    if constexpr (CLS == CLS_TREE)
        return (const void*)k_dp_list<CLS>;
    else if constexpr (CLS == CLS_CLIQUE)
        return mask_memo ? (const void*)k_dp_clique : (const void*)k_dp_fused<CLS, MEMO_DENSE>;
    else
        return mask_memo ? (const void*)k_dp_fused<CLS, MEMO_MASK> : (const void*)k_dp_fused<CLS, MEMO_DENSE>;
}
template <int CLS>
static size_t level_loop_smem(int n) {
    return sizeof(SQ<uint32_t>) +
           sizeof(unsigned int) * (rank_geom(n).entries + 33 * 33 + (CLS == CLS_TREE ? 1 + 2 * 33 * 33 : 2 * kFusedTile));
}

// Dataflow chunks of the clique levels (k_dp_clique on `grid` CTAs): per
// level the cost model's lanes per set (clique_group), or the split path's
// warp chunks of >= 512 pairs with their merge slots; the first levels of at
// most kCliqueSoloPairs pairs run as one solo chunk.  Returns false when the
// merge slots exceed the workspace's.
constexpr unsigned long long kCliqueSoloPairs = 512;
static bool plan_clique_df(Params<uint32_t>& p, unsigned int grid, unsigned long long slot_cap,
                           bool allow_split = true) {
    const unsigned long long T = (unsigned long long)grid * kDfCompute, nwarps = T / 32;
    const int n = p.n;
    unsigned int base = 0;
    unsigned long long slot = 0;
    unsigned long long target = 32768;
    if (const char* e = getenv("MPDP_DEBUG_CLIQUE_PAIRS")) target = strtoull(e, nullptr, 10);   // experiments only
    for (int k = p.k_begin; k <= p.k_end; k++) {
        const unsigned long long C = binom_u64(n, k), w = (1ull << (k - 1)) - 1;
        DfLevel& L = p.dfl[k];
        L = DfLevel{};
        L.base = base;
        const unsigned int G = allow_split ? clique_group(w, C, T) : clique_group(w, C, T, ~0ull);
        if (!G) {                                          // split path
            const unsigned long long P = C * w;
            const unsigned long long csize = std::max<unsigned long long>(512, (P + nwarps - 1) / nwarps);
            L.split = 1;
            L.chunk = (unsigned int)csize;
            L.nslot = (unsigned int)((P + csize - 1) / csize);
            L.slot0 = (unsigned int)slot;
            slot += L.nslot;
            base += (L.nslot + kDfCompute / 32 - 1) / (kDfCompute / 32);
            continue;
        }
        if (C * w <= kCliqueSoloPairs && k < p.k_end) {    // a run of small levels: one chunk
            int kb = k;
            while (kb + 1 <= p.k_end && binom_u64(n, kb + 1) * ((1ull << kb) - 1) <= kCliqueSoloPairs) kb++;
            if (kb > k) {
                for (int j = k; j <= kb; j++) {
                    const unsigned long long Cj = binom_u64(n, j), wj = (1ull << (j - 1)) - 1;
                    DfLevel& Lj = p.dfl[j];
                    Lj = DfLevel{};
                    Lj.base = j == k ? base : base + 1;
                    Lj.G = (unsigned char)std::max(1u, clique_group(wj, Cj, kDfCompute));
                    Lj.chunk = (unsigned int)Cj;
                }
                L.solo = (unsigned char)kb;
                base += 1;
                k = kb;
                continue;
            }
        }
        // R rounds of the CTA per ticket: about `target` pairs per chunk (the
        // control warp's per-chunk work -- fence, publish, claim -- must hide
        // behind a chunk), but at least one ticket per CTA on the level
        const unsigned long long round = kDfCompute / G;
        unsigned long long R = std::max<unsigned long long>(1, (target + round * w - 1) / (round * w));
        R = std::min(R, std::max<unsigned long long>(1, C / (round * grid)));
        L.G = (unsigned char)G;
        L.chunk = (unsigned int)(round * R);
        base += (unsigned int)((C + L.chunk - 1) / L.chunk);
    }
    p.dfl[p.k_end + 1] = DfLevel{};
    p.dfl[p.k_end + 1].base = base;
    p.zero_words = slot;
    return 2 * slot <= slot_cap;
}

static mpdp_status run_clique_df(mpdp_ctx* c, Params<uint32_t> p) {
    const size_t smem = clique_smem_bytes();
    int& occ = c->clique_df_occ;
    if (!c->clique_df_attr) {
        CUDA_TRY(c, cudaFuncSetAttribute(k_dp_clique_df<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        c->clique_df_attr = true;
    }
    if (!occ) {
        CUDA_TRY(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dp_clique_df<false>, kDfThreads, smem));
        if (occ < 1) return fail(c, MPDP_ERR_CUDA, "clique kernel does not fit on an SM");
    }
    unsigned long long want = 1;
    for (int k = 2; k <= c->n; k++) {
        want = std::max(want, (binom_u64(c->n, k) + 511) / 512);
        want = std::max(want, heavy_pair_bound(c->n, k, CLS_CLIQUE) / 2048);
    }
    const unsigned int grid = (unsigned int)std::min<unsigned long long>(
        std::min<unsigned long long>(want, (unsigned long long)c->num_sms * occ), (unsigned long long)kMaxGrid);
    if (!plan_clique_df(p, grid, c->lay.heavy_cap)) return fail(c, MPDP_ERR_CAPACITY, "clique merge slots exceed the workspace");
    CUDA_TRY(c, cudaEventRecord(c->ev0, c->stream));
    unsigned int nl = 1;
    if (!c->desc_clean) {                  // (the dataflow kernels leave their state zeroed)
        k_init<uint32_t><<<1, 256, 0, c->stream>>>(p);
        nl++;
    }
    c->desc_clean = true;
    void* args[] = {&p};
    CUDA_TRY(c, cudaEventRecord(c->kev[0], c->stream));
    CUDA_TRY(c, cudaLaunchCooperativeKernel((const void*)k_dp_clique_df<false>, dim3(grid), dim3(kDfThreads), args, smem, c->stream));
    CUDA_TRY(c, cudaEventRecord(c->kev[1], c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(c->h_result, c->ws + c->lay.result, sizeof(ResultDev), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaEventRecord(c->ev1, c->stream));
    c->launches = nl;
    c->enum_launches = 0;
    c->eval_launches = 1;
    c->nkev = 2;
    c->fused = true;
    c->d2h_bytes = sizeof(ResultDev);
    return MPDP_OK;
}

// The fused path: k_init, ONE cooperative persistent kernel for every level
// and the extraction, then the D2H copy of the result.
template <int CLS>
static mpdp_status run_fused(mpdp_ctx* c, const Params<uint32_t>& p) {
    const bool mask = c->lay.mask_memo;
    const size_t smem = (CLS == CLS_CLIQUE && mask) ? clique_smem_bytes() : level_loop_smem<CLS>(c->n);
    const void* kern = level_loop_kernel<CLS>(mask);
    const int slot = CLS + (mask ? 3 : 0);
    int& occ = c->occ_by_n[slot][c->n];
    if (!c->attr_set[slot]) {              // once, for the largest n (32) this kernel can see
        const size_t smax = (CLS == CLS_CLIQUE && mask) ? clique_smem_bytes() : level_loop_smem<CLS>(32);
        CUDA_TRY(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax));
        c->attr_set[slot] = true;
    }
    if (!occ) {
        CUDA_TRY(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kBlock, smem));
        if (occ < 1) return fail(c, MPDP_ERR_CUDA, "fused kernel does not fit on an SM");
    }
    CUDA_TRY(c, cudaEventRecord(c->ev0, c->stream));
    k_init<uint32_t><<<1, 64, 0, c->stream>>>(p);
    // grid: enough CTAs for the widest level (tiles) and the heavy work, never
    // more than can be co-resident; small queries get a small grid so the grid
    // barriers between levels stay cheap
    unsigned long long want = 1;
    for (int k = 2; k <= c->n; k++) {
        want = std::max(want, (binom_u64(c->n, k) + 511) / 512);
        want = std::max(want, heavy_pair_bound(c->n, k, CLS) / 2048);
    }
    if (CLS == CLS_GENERAL && c->n > 12) want = ~0ull;     // heavy work unknown up front
    unsigned int grid = (unsigned int)std::min<unsigned long long>(
        std::min<unsigned long long>(want, (unsigned long long)c->num_sms * occ), (unsigned long long)kMaxGrid);
    if (const char* e = getenv("MPDP_DEBUG_GRID")) {      // experiments only: cap the whole-query grid
        const unsigned int g = (unsigned int)atoi(e);
        if (g >= 1 && g < grid) grid = g;
    }
    void* args[] = {const_cast<Params<uint32_t>*>(&p)};
    CUDA_TRY(c, cudaEventRecord(c->kev[0], c->stream));    // device time of the fused kernel itself
    CUDA_TRY(c, cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(kBlock), args, smem, c->stream));
    CUDA_TRY(c, cudaEventRecord(c->kev[1], c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(c->h_result, c->ws + c->lay.result, sizeof(ResultDev), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaEventRecord(c->ev1, c->stream));
    c->launches = 2;
    c->enum_launches = 0;
    c->eval_launches = 1;
    c->nkev = 2;
    c->fused = true;
    c->d2h_bytes = sizeof(ResultDev);
    return MPDP_OK;
}

// ------------------------------------------------------------ small queries
// One CTA with the memo in shared memory (small_kernel.cuh) when the query is
// small enough that the multi-CTA kernels' per-level grid barriers and global
// round trips dominate: tree queries with n <= 13.
static bool small_eligible(const mpdp_ctx* c) {
    const int n = c->n;
    if (c->wide || c->multi || n < 2 || n > kSmallMaxN || c->timeout_ms > 0) return false;
    if (c->flags & (MPDP_FLAG_NO_SMALL | MPDP_FLAG_NO_FUSED | MPDP_FLAG_PROFILE_KERNELS | MPDP_FLAG_HASH_MEMO))
        return false;
    // measured (B200): star-10 115 -> 54 us, snowflake-12 -> 74 us; cliques and
    // general graphs gain nothing or lose (clique-9 59 vs 62 us, cycle-12 and
    // random-12 several times slower: Find-Blocks and the pair counts need the
    // whole GPU), so only tree queries take this path
    // With memo-probe connectivity in shared memory (reading R20) general
    // graphs with few independent cycles or n <= 10 now gain too (B200:
    // cycle-12 0.244 -> 0.145 ms, cycle-13 0.270 -> 0.188, random-10 0.338 ->
    // 0.246) while denser ones still lose (random-12 0.46 -> 0.72, random-13
    // 0.46 -> 2.48 ms: their pairs need the whole GPU).
    if (c->cls == CLS_GENERAL) {
        if (const char* e = getenv("MPDP_DEBUG_SMALL_GENERAL")) return atoi(e) != 0;   // experiments only
        return n <= 10 || c->m + 1 <= (unsigned long long)n + 4;     // cyclomatic number <= 4
    }
    return c->cls == CLS_TREE;
}

// Sparse tree queries whose every level fits the single-CTA kernel's shared
// memory lists (k_dp_tree1; global colex-rank memo).
static bool tree1_eligible(const mpdp_ctx* c) {
    if (c->cls != CLS_TREE || c->wide || c->multi || c->n < 3 || c->n > 32 || c->timeout_ms > 0) return false;
    if (c->flags & (MPDP_FLAG_NO_SMALL | MPDP_FLAG_NO_FUSED | MPDP_FLAG_PROFILE_KERNELS | MPDP_FLAG_HASH_MEMO))
        return false;
    // measured (B200): chain-25 (<= 24 sets per level) 290 -> 222 us; snowflake-20
    // (up to ~2k sets per level) 253 -> 345 us: one SM is then instruction-bound,
    // so only levels of at most kTree1MaxLevel sets take this kernel
    return c->lay.memo_kind == MEMO_DENSE && c->tree_max_level <= (unsigned long long)kTree1MaxLevel;
}

// Sparse tree queries with up to kClusterMaxLevel sets per level (snowflakes):
// one thread-block cluster runs the level loop (cluster_kernel.cuh).
static bool cluster_eligible(const mpdp_ctx* c) {
    if (c->cls != CLS_TREE || c->wide || c->multi || c->n < 3 || c->n > 32 || c->timeout_ms > 0) return false;
    if (c->flags & (MPDP_FLAG_NO_SMALL | MPDP_FLAG_NO_FUSED | MPDP_FLAG_PROFILE_KERNELS | MPDP_FLAG_HASH_MEMO))
        return false;
    if (getenv("MPDP_DEBUG_NO_CLUSTER")) return false;      // experiments only
    return c->lay.memo_kind == MEMO_DENSE && c->tree_max_level <= (unsigned long long)kClusterMaxLevel &&
           c->lay.list_cap >= c->tree_max_level;
}

static mpdp_status run_tree_cluster(mpdp_ctx* c, const Params<uint32_t>& p) {
    const size_t smem = cluster_smem_bytes(p.memo.rg.entries);
    if (!c->cluster_size) {                // largest cluster the device schedules: 16 (non-portable), else 8
        CUDA_TRY(c, cudaFuncSetAttribute(k_dp_tree_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)cluster_smem_bytes(rank_geom(32).entries)));
        cudaFuncSetAttribute(k_dp_tree_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        for (int cs : {16, 8, 4}) {
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = cs;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.gridDim = dim3(cs);
            cfg.blockDim = dim3(kClusterBlock);
            cfg.dynamicSmemBytes = cluster_smem_bytes(rank_geom(32).entries);
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            int nclusters = 0;
            if (cudaOccupancyMaxActiveClusters(&nclusters, (void*)k_dp_tree_cluster, &cfg) == cudaSuccess && nclusters > 0) {
                c->cluster_size = cs;
                break;
            }
            cudaGetLastError();
        }
        if (!c->cluster_size) return fail(c, MPDP_ERR_CUDA, "no thread-block cluster fits the tree kernel");
    }
    int cs = c->cluster_size;
    if (const char* e = getenv("MPDP_DEBUG_CLUSTER")) cs = std::max(1, std::min(cs, atoi(e)));   // experiments only
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(kClusterBlock);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CUDA_TRY(c, cudaEventRecord(c->ev0, c->stream));
    CUDA_TRY(c, cudaEventRecord(c->kev[0], c->stream));
    CUDA_TRY(c, cudaLaunchKernelEx(&cfg, k_dp_tree_cluster, p));
    CUDA_TRY(c, cudaEventRecord(c->kev[1], c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(c->h_result, c->ws + c->lay.result, sizeof(ResultDev), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaEventRecord(c->ev1, c->stream));
    c->launches = 1;
    c->enum_launches = 0;
    c->eval_launches = 1;
    c->nkev = 2;
    c->fused = true;
    c->d2h_bytes = sizeof(ResultDev);
    return MPDP_OK;
}

static mpdp_status run_tree1(mpdp_ctx* c, const Params<uint32_t>& p) {
    const size_t smem = tree1_smem_bytes(p.memo.rg.entries);
    if (!c->tree1_attr) {
        CUDA_TRY(c, cudaFuncSetAttribute(k_dp_tree1, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)tree1_smem_bytes(rank_geom(32).entries)));
        c->tree1_attr = true;
    }
    CUDA_TRY(c, cudaEventRecord(c->ev0, c->stream));
    CUDA_TRY(c, cudaEventRecord(c->kev[0], c->stream));
    k_dp_tree1<<<1, kTree1Block, smem, c->stream>>>(p);
    CUDA_TRY(c, cudaGetLastError());
    CUDA_TRY(c, cudaEventRecord(c->kev[1], c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(c->h_result, c->ws + c->lay.result, sizeof(ResultDev), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaEventRecord(c->ev1, c->stream));
    c->launches = 1;
    c->enum_launches = 0;
    c->eval_launches = 1;
    c->nkev = 2;
    c->fused = true;
    c->small = true;
    c->tree1 = true;
    c->d2h_bytes = sizeof(ResultDev);
    return MPDP_OK;
}

// Star queries on one GPU (k_dp_star): closed-form set indexing, memo of
// C(n-1, k-1) entries per level inside the dense region.
static bool star_eligible(const mpdp_ctx* c) {
    // (honours timeout_ms on the device: the deadline is checked at every
    // chunk claim and in every dependency wait, dataflow.cuh)
    if (c->cls != CLS_TREE || c->star_hub < 0 || c->wide || c->multi || c->n < 3 || c->n > 32) return false;
    if (c->flags & (MPDP_FLAG_NO_STAR | MPDP_FLAG_NO_FUSED | MPDP_FLAG_PROFILE_KERNELS | MPDP_FLAG_HASH_MEMO))
        return false;
    return c->lay.memo_kind == MEMO_DENSE;
}

// Chunk geometry of the star levels [k_begin, k_end] of one launch on `grid`
// CTAs (dataflow tickets, one CTA's compute warps per ticket): G lanes per set
// on levels with fewer sets than half the threads (G <= 4), runs of RUN
// consecutive sets per group on levels with several sets per thread (one
// unrank per run); one ticket = R rounds of the CTA (kDfCompute / G groups x
// RUN sets) with R = 2 on the largest levels (star-25: 0.758 -> 0.749 ms).
static void plan_star_df(Params<uint32_t>& p, unsigned int grid) {
    const unsigned long long T = (unsigned long long)grid * kBlock;
    int run_max = 4, rounds = 2;
    if (const char* e = getenv("MPDP_DEBUG_STAR_RUN")) run_max = std::max(1, atoi(e));   // experiments only
    if (const char* e = getenv("MPDP_DEBUG_STAR_ROUNDS")) rounds = std::max(1, atoi(e));
    // runs of consecutive levels of at most `solo` sets are ONE chunk (one
    // CTA, the compute warps' barrier between the levels): a level handoff
    // through the dataflow counters costs a few us of fence / poll latency
    unsigned long long solo = 300;
    if (const char* e = getenv("MPDP_DEBUG_STAR_SOLO")) solo = strtoull(e, nullptr, 10);
    unsigned int base = 0;
    for (int k = p.k_begin; k <= p.k_end; k++) {
        const unsigned long long C = p.share_hi[k] - p.share_lo[k];
        const bool small = C <= solo && p.k_end > p.k_begin;
        const unsigned long long TT = small ? (unsigned long long)kDfCompute : T;
        unsigned int G = 1;
        while (G < 4 && 2ull * G * C <= TT) G <<= 1;
        unsigned int run = 1;
        while ((int)run < run_max && C >= 4ull * run * TT) run <<= 1;
        DfLevel& L = p.dfl[k];
        L = DfLevel{};
        L.base = base;
        L.G = (unsigned char)G;
        L.run = (unsigned char)run;
        L.solo = 0;
        if (small) {
            int kb = k;                                    // the run of small levels k..kb
            while (kb + 1 <= p.k_end && p.share_hi[kb + 1] - p.share_lo[kb + 1] <= solo) kb++;
            if (kb > k) {
                L.chunk = (unsigned int)C;
                L.solo = (unsigned char)kb;
                base += 1;
                for (int j = k + 1; j <= kb; j++) {
                    const unsigned long long Cj = p.share_hi[j] - p.share_lo[j];
                    DfLevel& Lj = p.dfl[j];
                    Lj = DfLevel{};
                    Lj.base = base;                        // no tickets of their own
                    Lj.G = 1;
                    while (Lj.G < 4 && 2ull * Lj.G * Cj <= (unsigned long long)kDfCompute) Lj.G <<= 1;
                    Lj.run = 1;
                    Lj.chunk = (unsigned int)Cj;
                }
                k = kb;
                continue;
            }
        }
        L.chunk = (kDfCompute / G) * run * (C >= 8ull * T ? rounds : 1);
        base += (unsigned int)((C + L.chunk - 1) / L.chunk);
    }
    p.dfl[p.k_end + 1] = DfLevel{};
    p.dfl[p.k_end + 1].base = base;
}

static mpdp_status run_star(mpdp_ctx* c, Params<uint32_t> p) {
    for (int k = 2; k <= c->n; k++) {                      // every level: all C(n-1, k-1) sets
        p.share_lo[k] = 0;
        p.share_hi[k] = (unsigned int)binom_u64(c->n - 1, k - 1);
    }
    const size_t smem = star_smem_bytes();
    if (!c->star_occ) {
        CUDA_TRY(c, cudaFuncSetAttribute(k_dp_star<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CUDA_TRY(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->star_occ, k_dp_star<false>, kDfThreads, smem));
        if (c->star_occ < 1) return fail(c, MPDP_ERR_CUDA, "star kernel does not fit on an SM");
    }
    unsigned long long want = 1;
    for (int k = 2; k <= c->n; k++) want = std::max(want, (binom_u64(c->n - 1, k - 1) + 255) / 256);
    const unsigned int grid = (unsigned int)std::min<unsigned long long>(
        std::min<unsigned long long>(want, (unsigned long long)c->num_sms * c->star_occ), (unsigned long long)kMaxGrid);
    plan_star_df(p, grid);
    CUDA_TRY(c, cudaEventRecord(c->ev0, c->stream));
    // no k_init when the previous launch was a dataflow kernel: the dataflow
    // state, the level descriptors and the error bits were returned to zero by
    // its last CTA
    unsigned int nl = 1;
    if (!c->desc_clean) {
        k_init<uint32_t><<<1, 256, 0, c->stream>>>(p);
        nl++;
    }
    c->desc_clean = true;
    void* args[] = {const_cast<Params<uint32_t>*>(&p)};
    CUDA_TRY(c, cudaEventRecord(c->kev[0], c->stream));
    CUDA_TRY(c, cudaLaunchCooperativeKernel((const void*)k_dp_star<false>, dim3(grid), dim3(kDfThreads), args, smem, c->stream));
    CUDA_TRY(c, cudaEventRecord(c->kev[1], c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(c->h_result, c->ws + c->lay.result, sizeof(ResultDev), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaEventRecord(c->ev1, c->stream));
    c->launches = nl;
    c->enum_launches = 0;
    c->eval_launches = 1;
    c->nkev = 2;
    c->fused = true;
    c->star = true;
    c->d2h_bytes = sizeof(ResultDev);
    return MPDP_OK;
}

template <int CLS>
static mpdp_status run_small(mpdp_ctx* c, const Params<uint32_t>& p) {
    const size_t smem = small_smem_bytes(c->n);
    if (!c->small_attr[CLS]) {
        CUDA_TRY(c, cudaFuncSetAttribute(k_dp_small<CLS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)small_smem_bytes(kSmallMaxN)));
        c->small_attr[CLS] = true;
    }
    CUDA_TRY(c, cudaEventRecord(c->ev0, c->stream));
    CUDA_TRY(c, cudaEventRecord(c->kev[0], c->stream));
    k_dp_small<CLS><<<1, kSmallBlock, smem, c->stream>>>(p);
    CUDA_TRY(c, cudaGetLastError());
    CUDA_TRY(c, cudaEventRecord(c->kev[1], c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(c->h_result, c->ws + c->lay.result, sizeof(ResultDev), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaEventRecord(c->ev1, c->stream));
    c->launches = 1;
    c->enum_launches = 0;
    c->eval_launches = 1;
    c->nkev = 2;
    c->fused = true;
    c->small = true;
    c->d2h_bytes = sizeof(ResultDev);
    return MPDP_OK;
}

// ------------------------------------------------------------ sharded run
// Multi-GPU: per level k, rank r evaluates the colex ranks
// [r*seg, (r+1)*seg) of the level (seg = ceil(C(n,k)/W)) with the fused kernel
// restricted to that share; its memo entries are then one contiguous segment
// of the level's perfect-hash array, so the exchange is an in-place
// ncclAllGather of `seg` costs, `seg` left masks and `seg` cards per rank (the
// cards feed card(S) = card(S \ max) x ... and the plan extraction) -- no
// packing and no replica insert.  Levels below kShardMinRanks are computed redundantly by
// every rank (counted by rank 0 only).  Counters are summed with one
// ncclAllReduce at the end; every rank extracts the identical plan from its
// complete replica.  In simulated mode the ranks are shards of this context
// and the transport is device-to-device copies.
constexpr unsigned long long kShardMinRanks = 1ull << 14;

static mpdp_status exchange_level(mpdp_ctx* c, const Params<uint32_t>* P, int k, unsigned long long C,
                                  unsigned long long seg, bool with_card, unsigned long long off, bool with_left) {
    const int W = c->world;
    if (c->simulate) {
        for (int s = 0; s < W; s++) {
            const unsigned long long lo = std::min(C, s * seg), hi = std::min(C, (s + 1) * seg);
            if (hi <= lo) continue;
            for (int t = 0; t < W; t++) {
                if (t == s) continue;
                CUDA_TRY(c, cudaMemcpyAsync(P[t].memo.dcost + off + lo, P[s].memo.dcost + off + lo, (hi - lo) * 8,
                                            cudaMemcpyDeviceToDevice, c->stream));
                if (with_left)
                    CUDA_TRY(c, cudaMemcpyAsync(P[t].memo.dleft + off + lo, P[s].memo.dleft + off + lo, (hi - lo) * 4,
                                                cudaMemcpyDeviceToDevice, c->stream));
                if (with_card)
                    CUDA_TRY(c, cudaMemcpyAsync(P[t].memo.dcard + off + lo, P[s].memo.dcard + off + lo, (hi - lo) * 8,
                                                cudaMemcpyDeviceToDevice, c->stream));
            }
        }
        return MPDP_OK;
    }
    double* dc = P[0].memo.dcost + off;
    unsigned int* dl = P[0].memo.dleft + off;
    ncclResult_t r = c->nccl->GroupStart();
    if (!r) r = c->nccl->AllGather(dc + c->rank * seg, dc, seg, kNcclFloat64, c->comm, c->stream);
    if (!r && with_left) r = c->nccl->AllGather(dl + c->rank * seg, dl, seg, kNcclUint32, c->comm, c->stream);
    double* dk = P[0].memo.dcard + off;    // card(S \ max) feeds card_fast (trees, cliques)
    if (!r && with_card) r = c->nccl->AllGather(dk + c->rank * seg, dk, seg, kNcclFloat64, c->comm, c->stream);
    const ncclResult_t r2 = c->nccl->GroupEnd();
    if (r || r2) return fail(c, MPDP_ERR_NCCL, "ncclAllGather of level " + std::to_string(k) + " failed");
    return MPDP_OK;
}

// Fused peer exchange (MPDP_FLAG_FUSED_EXCHANGE): one launch of
// k_dp_star per rank whose chunks store their costs into every rank's replica
// and count themselves in every replica's dataflow counters (XrTable,
// level_kernels.cuh) -- the exchange overlaps the computation chunk by chunk
// and no level ends in a launch or a collective.  Simulated world: the W ranks
// are the CTA groups blockIdx % W of ONE cooperative launch over the W shards
// of this workspace (ranks that wait on one another must be co-resident);
// across GPUs the replicas are the IPC-mapped workspaces of
// mpdp_ctx_open_peers, every rank extracts the plan from its own replica.
static mpdp_status run_star_xr(mpdp_ctx* c) {
    const int n = c->n, W = c->world;
    if (W > kMaxXr) return fail(c, MPDP_ERR_INVALID_ARGUMENT, "fused exchange: world > 8");
    if (!c->simulate && !c->peers_open)
        return fail(c, MPDP_ERR_INVALID_ARGUMENT, "fused exchange across GPUs needs mpdp_ctx_open_peers first");
    const DevLayout& L = c->lay;
    Params<uint32_t> p = make_params<uint32_t>(c, 0);
    for (int k = 2; k <= n; k++) {                      // every level: all C(n-1, k-1) sets
        p.share_lo[k] = 0;
        p.share_hi[k] = (unsigned int)binom_u64(n - 1, k - 1);
    }
    const size_t smem = star_smem_bytes();
    if (!c->star_occ_xr) {
        CUDA_TRY(c, cudaFuncSetAttribute(k_dp_star<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CUDA_TRY(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->star_occ_xr, k_dp_star<true>, kDfThreads, smem));
        if (c->star_occ_xr < 1) return fail(c, MPDP_ERR_CUDA, "star kernel does not fit on an SM");
    }
    const unsigned int full = (unsigned int)std::min<unsigned long long>((unsigned long long)c->num_sms * c->star_occ_xr,
                                                                         (unsigned long long)kMaxGrid);
    const unsigned int grid = c->simulate ? full / (unsigned int)W * (unsigned int)W : full;
    const unsigned int ctas_total = c->simulate ? grid : grid * (unsigned int)W;
    plan_star_df(p, ctas_total);           // chunks sized for every CTA of every rank
    p.shard_local = 1;                     // costs only cross ranks: card(S) local, splits re-derived
    p.do_extract = 1;
    XrTable t;
    memset(&t, 0, sizeof(t));
    t.W = W;
    t.emulate = c->simulate ? 1 : 0;
    t.rank = c->simulate ? 0 : c->rank;
    t.ctas_total = ctas_total;
    for (int s = 0; s < W; s++) {
        unsigned char* base = c->simulate ? c->ws : c->peer_ws[s];
        const int sh = c->simulate ? s : 0;
        t.cost[s] = reinterpret_cast<double*>(base + L.sh_dcost[sh]);
        t.card[s] = reinterpret_cast<double*>(base + L.sh_dcard[sh]);
        t.left[s] = reinterpret_cast<unsigned int*>(base + L.sh_dleft[sh]);
        t.df[s] = reinterpret_cast<DataflowDev*>(base + L.sh_df[sh]);
        t.desc[s] = reinterpret_cast<LevelDesc*>(base + L.sh_desc[sh]);
        t.result[s] = reinterpret_cast<ResultDev*>(base + L.sh_result[sh]);
    }
    if (!c->h_xr && cudaMallocHost(&c->h_xr, sizeof(XrTable)) != cudaSuccess)
        return fail(c, MPDP_ERR_OOM, "pinned host allocation failed");
    memcpy(c->h_xr, &t, sizeof(t));
    CUDA_TRY(c, cudaMemcpyAsync(c->ws + L.xr, c->h_xr, sizeof(XrTable), cudaMemcpyHostToDevice, c->stream));
    p.xr = reinterpret_cast<const XrTable*>(c->ws + L.xr);
    p.xr_epoch = ++c->xr_epoch;
    CUDA_TRY(c, cudaEventRecord(c->ev0, c->stream));
    unsigned int nl = 1;
    if (!c->desc_clean) {                  // the local replicas' dataflow state and descriptors
        for (int sh = 0; sh < L.nshards; sh++) {
            k_init<uint32_t><<<1, 256, 0, c->stream>>>(make_params<uint32_t>(c, sh));
            nl++;
        }
    }
    c->desc_clean = true;
    void* args[] = {&p};
    CUDA_TRY(c, cudaEventRecord(c->kev[0], c->stream));
    CUDA_TRY(c, cudaLaunchCooperativeKernel((const void*)k_dp_star<true>, dim3(grid), dim3(kDfThreads), args, smem, c->stream));
    CUDA_TRY(c, cudaEventRecord(c->kev[1], c->stream));
    for (int sh = 0; sh < L.nshards; sh++)
        CUDA_TRY(c, cudaMemcpyAsync(c->h_results + sh, c->ws + L.sh_result[sh], sizeof(ResultDev),
                                    cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaEventRecord(c->ev1, c->stream));
    c->launches = nl;
    c->enum_launches = 0;
    c->eval_launches = 1;
    c->nkev = 2;
    c->fused = true;
    c->star = true;
    c->sharded = false;
    c->xr_run = true;
    c->d2h_bytes = sizeof(ResultDev) * L.nshards;
    return MPDP_OK;
}

// Fused peer exchange for cliques (MPDP_FLAG_FUSED_EXCHANGE): k_dp_clique_df
// with every set written into every rank's bitmask-memo replica (cost, card
// and left) and counted in every replica's dataflow counters; no split levels
// (a set is evaluated by one group of one rank, so no cross-rank merges).
// Simulated world: the ranks are the CTA groups blockIdx % W of one launch.
static mpdp_status run_clique_xr(mpdp_ctx* c) {
    const int W = c->world;
    if (W > kMaxXr) return fail(c, MPDP_ERR_INVALID_ARGUMENT, "fused exchange: world > 8");
    if (!c->simulate && !c->peers_open)
        return fail(c, MPDP_ERR_INVALID_ARGUMENT, "fused exchange across GPUs needs mpdp_ctx_open_peers first");
    const DevLayout& L = c->lay;
    Params<uint32_t> p = make_params<uint32_t>(c, 0);
    const size_t smem = clique_smem_bytes();
    if (!c->clique_xr_occ) {
        CUDA_TRY(c, cudaFuncSetAttribute(k_dp_clique_df<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CUDA_TRY(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->clique_xr_occ, k_dp_clique_df<true>, kDfThreads, smem));
        if (c->clique_xr_occ < 1) return fail(c, MPDP_ERR_CUDA, "clique kernel does not fit on an SM");
    }
    const unsigned int full = (unsigned int)std::min<unsigned long long>((unsigned long long)c->num_sms * c->clique_xr_occ,
                                                                         (unsigned long long)kMaxGrid);
    const unsigned int grid = c->simulate ? full / (unsigned int)W * (unsigned int)W : full;
    const unsigned int ctas_total = c->simulate ? grid : grid * (unsigned int)W;
    plan_clique_df(p, ctas_total, ~0ull, false);
    p.do_extract = 1;
    XrTable t;
    memset(&t, 0, sizeof(t));
    t.W = W;
    t.emulate = c->simulate ? 1 : 0;
    t.rank = c->simulate ? 0 : c->rank;
    t.ctas_total = ctas_total;
    for (int s = 0; s < W; s++) {
        unsigned char* base = c->simulate ? c->ws : c->peer_ws[s];
        const int sh = c->simulate ? s : 0;
        t.cost[s] = reinterpret_cast<double*>(base + L.sh_dcost[sh]);
        t.card[s] = reinterpret_cast<double*>(base + L.sh_dcard[sh]);
        t.left[s] = reinterpret_cast<unsigned int*>(base + L.sh_dleft[sh]);
        t.df[s] = reinterpret_cast<DataflowDev*>(base + L.sh_df[sh]);
        t.desc[s] = reinterpret_cast<LevelDesc*>(base + L.sh_desc[sh]);
        t.result[s] = reinterpret_cast<ResultDev*>(base + L.sh_result[sh]);
    }
    if (!c->h_xr && cudaMallocHost(&c->h_xr, sizeof(XrTable)) != cudaSuccess)
        return fail(c, MPDP_ERR_OOM, "pinned host allocation failed");
    memcpy(c->h_xr, &t, sizeof(t));
    CUDA_TRY(c, cudaMemcpyAsync(c->ws + L.xr, c->h_xr, sizeof(XrTable), cudaMemcpyHostToDevice, c->stream));
    p.xr = reinterpret_cast<const XrTable*>(c->ws + L.xr);
    p.xr_epoch = ++c->xr_epoch;
    CUDA_TRY(c, cudaEventRecord(c->ev0, c->stream));
    unsigned int nl = 1;
    if (!c->desc_clean) {
        for (int sh = 0; sh < L.nshards; sh++) {
            k_init<uint32_t><<<1, 256, 0, c->stream>>>(make_params<uint32_t>(c, sh));
            nl++;
        }
    }
    c->desc_clean = true;
    void* args[] = {&p};
    CUDA_TRY(c, cudaEventRecord(c->kev[0], c->stream));
    CUDA_TRY(c, cudaLaunchCooperativeKernel((const void*)k_dp_clique_df<true>, dim3(grid), dim3(kDfThreads), args, smem,
                                            c->stream));
    CUDA_TRY(c, cudaEventRecord(c->kev[1], c->stream));
    for (int sh = 0; sh < L.nshards; sh++)
        CUDA_TRY(c, cudaMemcpyAsync(c->h_results + sh, c->ws + L.sh_result[sh], sizeof(ResultDev),
                                    cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaEventRecord(c->ev1, c->stream));
    c->launches = nl;
    c->enum_launches = 0;
    c->eval_launches = 1;
    c->nkev = 2;
    c->fused = true;
    c->sharded = false;
    c->xr_run = true;
    c->d2h_bytes = sizeof(ResultDev) * L.nshards;
    return MPDP_OK;
}

template <int CLS>
static mpdp_status run_sharded(mpdp_ctx* c) {
    if (c->wide || c->lay.memo_kind != MEMO_DENSE)
        return fail(c, MPDP_ERR_CAPACITY, "multi-GPU sharding needs n <= 32 and the perfect-hash memo");
    const int n = c->n, W = c->world, nsh = c->lay.nshards;
    // star queries shard k_dp_star's leaf-set ranks; everything else the
    // whole-query kernel's colex ranks
    const bool star = CLS == CLS_TREE && c->star_hub >= 0 && n >= 3 &&
                      !(c->flags & (MPDP_FLAG_NO_STAR | MPDP_FLAG_NO_FUSED | MPDP_FLAG_PROFILE_KERNELS));
    if (star && (c->flags & MPDP_FLAG_FUSED_EXCHANGE) && !c->nccl_self) return run_star_xr(c);
    if (CLS == CLS_CLIQUE && c->lay.mask_memo && (c->flags & MPDP_FLAG_FUSED_EXCHANGE) && !c->nccl_self)
        return run_clique_xr(c);
    const void* kern = star ? (const void*)k_dp_star<false> : level_loop_kernel<CLS>();
    const size_t smem = star ? star_smem_bytes() : level_loop_smem<CLS>(n);
    int occ_star = 0;
    int& occ = star ? occ_star : c->fused_occ[CLS];
    const int block = star ? kDfThreads : kBlock;
    if (star) {
        CUDA_TRY(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CUDA_TRY(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, block, smem));
        if (occ < 1) return fail(c, MPDP_ERR_CUDA, "star kernel does not fit on an SM");
    } else if (!occ || c->fused_n[CLS] != n) {
        // function attributes are process-wide (shared by every context): always
        // raise the limit to the largest n, never lower it below another
        // context's launch
        CUDA_TRY(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)level_loop_smem<CLS>(32)));
        CUDA_TRY(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kBlock, smem));
        if (occ < 1) return fail(c, MPDP_ERR_CUDA, "fused kernel does not fit on an SM");
        c->fused_n[CLS] = n;
    }
    const unsigned long long full = std::min<unsigned long long>((unsigned long long)c->num_sms * occ, kMaxGrid);
    std::vector<Params<uint32_t>> P(nsh);
    std::vector<unsigned long long> counted(nsh, 0);
    CUDA_TRY(c, cudaEventRecord(c->ev0, c->stream));
    c->launches = 0;
    for (int sh = 0; sh < nsh; sh++) {
        P[sh] = make_params<uint32_t>(c, sh);
        P[sh].timeout_ns = 0;              // (the sharded host loop has no device deadline)
        P[sh].shard_local = star ? 1 : 0;
        k_init<uint32_t><<<1, 256, 0, c->stream>>>(P[sh]);
        c->launches++;
    }
    auto launch = [&](Params<uint32_t>& p, unsigned long long grid) -> mpdp_status {
        void* args[] = {&p};
        CUDA_TRY(c, cudaMemsetAsync(p.gbar, 0, sizeof(unsigned int), c->stream));   // barrier counter per launch
        if (star) plan_star_df(p, (unsigned int)grid);   // dataflow tickets of this launch's levels
        CUDA_TRY(c, cudaLaunchCooperativeKernel(kern, dim3((unsigned int)grid), dim3(block), args, smem, c->stream));
        c->launches++;
        return MPDP_OK;
    };
    const unsigned long long min_shard = (c->flags & MPDP_FLAG_SHARD_ALL_LEVELS) ? 0ull : kShardMinRanks;
    for (int k = 2; k <= n; k++) {
        const unsigned long long C = star ? binom_u64(n - 1, k - 1) : binom_u64(n, k);
        const bool sharded = (W > 1 && C >= min_shard) || c->nccl_self;
        const unsigned long long seg = (C + W - 1) / W;
        for (int sh = 0; sh < nsh; sh++) {
            const int rank = c->simulate ? sh : c->rank;
            Params<uint32_t>& p = P[sh];
            p.k_begin = p.k_end = k;
            p.do_extract = 0;
            uint64_t lo = 0, hi = C;
            if (sharded) mpdp_share(C, rank, W, &lo, &hi);
            p.share_lo[k] = (unsigned int)lo;
            p.share_hi[k] = (unsigned int)hi;
            const bool counts = sharded || rank == 0;
            p.count_levels = counts ? (1ull << k) : 0ull;
            if (counts) counted[sh] |= 1ull << k;
            if (hi <= lo) continue;
            unsigned long long grid = std::max<unsigned long long>(1, (hi - lo + (star ? 255 : 511)) / (star ? 256 : 512));
            grid = std::max(grid, heavy_pair_bound(n, k, CLS) / ((unsigned long long)W * 16384));
            if (CLS == CLS_GENERAL) grid = full;
            const mpdp_status st = launch(p, std::min(grid, full));
            if (st != MPDP_OK) return st;
        }
        if (sharded) {
            // star: costs only (8 B per set; card(S) is recomputed locally and
            // the extraction re-derives the chosen splits from the costs);
            // others: costs, left masks and cards (card(S \ max) of the next
            // level and the extraction read them)
            const mpdp_status st = exchange_level(c, P.data(), k, C, seg, !star, star ? P[0].star_off[k] : P[0].dense_off[k],
                                                  !star);
            if (st != MPDP_OK) return st;
        }
        CUDA_TRY(c, cudaGetLastError());
    }
    for (int sh = 0; sh < nsh; sh++) {                  // extraction from each complete replica
        const int rank = c->simulate ? sh : c->rank;
        Params<uint32_t>& p = P[sh];
        p.k_begin = n + 1;
        p.k_end = n;
        p.do_extract = 1;
        p.count_levels = counted[sh] | (rank == 0 ? 2ull : 0ull);
        const mpdp_status st = launch(p, 1);
        if (st != MPDP_OK) return st;
    }
    if (!c->simulate) {                                 // sum the per-rank counters
        ResultDev* r = reinterpret_cast<ResultDev*>(c->ws + c->lay.sh_result[0]);
        ncclResult_t e = c->nccl->GroupStart();
        if (!e) e = c->nccl->AllReduce(&r->csg, &r->csg, 4, kNcclUint64, kNcclSum, c->comm, c->stream);
        if (!e) e = c->nccl->AllReduce(r->lvl_csg, r->lvl_csg, 3 * (kMaxN + 1), kNcclUint64, kNcclSum, c->comm, c->stream);
        if (!e) e = c->nccl->AllReduce(&r->n_nodes, &r->n_nodes, 2, kNcclUint32, kNcclMax, c->comm, c->stream);
        const ncclResult_t e2 = c->nccl->GroupEnd();
        if (e || e2) return fail(c, MPDP_ERR_NCCL, "ncclAllReduce of the counters failed");
    }
    for (int sh = 0; sh < nsh; sh++)
        CUDA_TRY(c, cudaMemcpyAsync(c->h_results + sh, c->ws + c->lay.sh_result[sh], sizeof(ResultDev),
                                    cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaEventRecord(c->ev1, c->stream));
    c->enum_launches = 0;
    c->eval_launches = (unsigned int)(nsh * (n - 1));
    c->nkev = 0;
    c->d2h_bytes = sizeof(ResultDev) * nsh;
    c->sharded = true;
    c->star = star;
    return MPDP_OK;
}

template <typename M, int CLS, int MEMO>
static mpdp_status run_query(mpdp_ctx* c) {
    const bool was_clean = c->desc_clean;
    c->desc_clean = false;                 // every path but the dataflow kernels leaves them dirty
    (void)was_clean;
    c->sharded = false;
    c->small = false;
    c->tree1 = false;
    c->star = false;
    c->xr_run = false;
    if constexpr (MEMO == MEMO_DENSE && sizeof(M) == 4) {
        if (c->multi) {
            c->desc_clean = was_clean;     // (the fused exchange keeps the dataflow state clean)
            const mpdp_status st = run_sharded<CLS>(c);
            if (!c->xr_run) c->desc_clean = false;
            return st;
        }
    }
    if (c->multi) return fail(c, MPDP_ERR_CAPACITY, "multi-GPU sharding needs n <= 32 and the perfect-hash memo");
    c->fused = false;
    c->small = false;
    if constexpr (MEMO == MEMO_DENSE && sizeof(M) == 4) {
        if (small_eligible(c)) return run_small<CLS>(c, make_params<M>(c));
        if (tree1_eligible(c)) return run_tree1(c, make_params<M>(c));
        if (!(c->star_hub >= 0 && star_eligible(c)) && cluster_eligible(c)) return run_tree_cluster(c, make_params<M>(c));
        if (star_eligible(c)) {
            c->desc_clean = was_clean;
            return run_star(c, make_params<M>(c));
        }
        const bool clique_mask = CLS == CLS_CLIQUE && c->lay.mask_memo && c->n >= 2 &&
                                 !(c->flags & (MPDP_FLAG_NO_FUSED | MPDP_FLAG_PROFILE_KERNELS));
        if (clique_mask && getenv("MPDP_DEBUG_CLIQUE_DF")) {   // ablation: the dataflow variant
            c->desc_clean = was_clean;
            return run_clique_df(c, make_params<M>(c));
        }
        // (k_dp_clique checks timeout_ms on the device at every level barrier)
        if ((c->timeout_ms <= 0 || clique_mask) && !(c->flags & (MPDP_FLAG_NO_FUSED | MPDP_FLAG_PROFILE_KERNELS)) &&
            c->n >= 2)
            return run_fused<CLS>(c, make_params<M>(c));
    }
    mpdp_status st = prepare_kernels<M, CLS, MEMO>(c);
    if (st != MPDP_OK) return st;
    const Params<M> p = make_params<M>(c);   // query-invariant: epoch/tag live in QueryDev
    // per-kernel profiling events are recorded on the direct-launch path
    const bool graph = c->timeout_ms <= 0 && !(c->flags & (MPDP_FLAG_NO_GRAPH | MPDP_FLAG_PROFILE_KERNELS));
    if (!graph) {
        CUDA_TRY(c, cudaEventRecord(c->ev0, c->stream));
        st = enqueue_query<M, CLS, MEMO>(c, p, true);
        if (st != MPDP_OK) return st;
        CUDA_TRY(c, cudaEventRecord(c->ev1, c->stream));
        return MPDP_OK;
    }
    const unsigned long long key = (unsigned long long)c->n | (unsigned long long)CLS << 8 |
                                   (unsigned long long)MEMO << 10 | (unsigned long long)c->wide << 11 |
                                   (unsigned long long)(c->flags & MPDP_FLAG_PROFILE_KERNELS) << 12;
    auto it = c->graphs.find(key);
    if (it == c->graphs.end()) {
        cudaGraph_t g = nullptr;
        CUDA_TRY(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        st = enqueue_query<M, CLS, MEMO>(c, p, false);
        const cudaError_t ec = cudaStreamEndCapture(c->stream, &g);
        if (st != MPDP_OK) {
            if (g) cudaGraphDestroy(g);
            return st;
        }
        if (ec != cudaSuccess) return fail(c, MPDP_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(ec));
        mpdp_ctx::GraphEntry e{};
        const cudaError_t ei = cudaGraphInstantiate(&e.exec, g, 0);
        cudaGraphDestroy(g);
        if (ei != cudaSuccess) return fail(c, MPDP_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ei));
        e.launches = c->launches;
        e.enum_launches = c->enum_launches;
        e.eval_launches = c->eval_launches;
        e.nkev = c->nkev;
        it = c->graphs.emplace(key, e).first;
    }
    c->launches = it->second.launches;
    c->enum_launches = it->second.enum_launches;
    c->eval_launches = it->second.eval_launches;
    c->nkev = it->second.nkev;
    c->d2h_bytes = sizeof(ResultDev);
    CUDA_TRY(c, cudaEventRecord(c->ev0, c->stream));
    CUDA_TRY(c, cudaGraphLaunch(it->second.exec, c->stream));
    CUDA_TRY(c, cudaEventRecord(c->ev1, c->stream));
    return MPDP_OK;
}

template <typename M, int MEMO>
static mpdp_status run_memo(mpdp_ctx* c) {
    switch (c->cls) {
        case CLS_TREE: return run_query<M, CLS_TREE, MEMO>(c);
        case CLS_CLIQUE: return run_query<M, CLS_CLIQUE, MEMO>(c);
        default: return run_query<M, CLS_GENERAL, MEMO>(c);
    }
}

template <typename M>
static mpdp_status run_typed(mpdp_ctx* c) {
    if (!c->wide && c->lay.memo_kind == MEMO_DENSE) return run_memo<M, MEMO_DENSE>(c);
    return run_memo<M, MEMO_HASH>(c);
}

// ------------------------------------------------------------ heuristics
extern "C" mpdp_status mpdp_optimize(mpdp_ctx* c, const mpdp_query_graph* g, mpdp_algo algo, uint32_t k,
                                     mpdp_result* out);

// inner exact DP of IDP2/UnionDP: the GPU MPDP on the same context
static mpdp_status gpu_inner_solver(void* user, const mpdp_query_graph* sub, mpdp_result* out) {
    mpdp_ctx* c = static_cast<mpdp_ctx*>(user);
    // multi-GPU contexts: a sequential inner DP (IDP2's iterations depend on
    // each other) of <= 32 relations runs redundantly on every rank
    // with the single-GPU kernels -- per-level sharding of such small DPs
    // would pay a collective per level for microseconds of work; independent
    // sub-problems go through the distributed batch instead
    const bool sm = c->multi, sn = c->nccl_self;
    const int sw = c->world;
    if (c->multi && !c->simulate) {
        c->multi = false;
        c->nccl_self = false;
        c->world = 1;
    }
    const mpdp_status st = mpdp_optimize(c, sub, MPDP_ALGO_MPDP, 0, out);
    c->multi = sm;
    c->nccl_self = sn;
    c->world = sw;
    if (st == MPDP_OK && (c->flags & MPDP_FLAG_RECORD_SUBPROBLEMS)) {
        mpdp_ctx::SubProblem sp;
        sp.card.assign(sub->cardinalities, sub->cardinalities + sub->n);
        sp.sel.assign(sub->selectivities, sub->selectivities + sub->n_edges);
        sp.edges.assign(sub->edges, sub->edges + 2 * sub->n_edges);
        if (sub->leaf_costs) sp.leaf.assign(sub->leaf_costs, sub->leaf_costs + sub->n);
        sp.nodes.assign(out->nodes, out->nodes + out->n_nodes);
        sp.res = *out;
        sp.res.nodes = nullptr;
        sp.res.level_csg = sp.res.level_ccp = sp.res.level_pairs = nullptr;
        sp.res.level_ms = nullptr;
        c->subs.push_back(std::move(sp));
    }
    return st;
}

extern "C" mpdp_status mpdp_optimize_batch(mpdp_ctx* c, const mpdp_query_graph* graphs, uint32_t count,
                                           mpdp_result* results);
// independent sub-problems of a UnionDP level in one call (recorded like the
// single ones)
static mpdp_status gpu_inner_batch(void* user, const mpdp_query_graph* subs, uint32_t count, mpdp_result* outs) {
    mpdp_ctx* c = static_cast<mpdp_ctx*>(user);
    const mpdp_status st = mpdp_optimize_batch(c, subs, count, outs);
    if (st == MPDP_OK && (c->flags & MPDP_FLAG_RECORD_SUBPROBLEMS)) {
        for (uint32_t i = 0; i < count; i++) {
            const mpdp_query_graph* sub = subs + i;
            const mpdp_result* out = outs + i;
            mpdp_ctx::SubProblem sp;
            sp.card.assign(sub->cardinalities, sub->cardinalities + sub->n);
            sp.sel.assign(sub->selectivities, sub->selectivities + sub->n_edges);
            sp.edges.assign(sub->edges, sub->edges + 2 * sub->n_edges);
            if (sub->leaf_costs) sp.leaf.assign(sub->leaf_costs, sub->leaf_costs + sub->n);
            sp.nodes.assign(out->nodes, out->nodes + out->n_nodes);
            sp.res = *out;
            sp.res.nodes = nullptr;
            sp.res.level_csg = sp.res.level_ccp = sp.res.level_pairs = nullptr;
            sp.res.level_ms = nullptr;
            c->subs.push_back(std::move(sp));
        }
    }
    return st;
}

// ------------------------------------------------------------ C ABI
extern "C" {

int mpdp_subproblem_count(const mpdp_ctx* c) { return c ? (int)c->subs.size() : 0; }

mpdp_status mpdp_subproblem_get(const mpdp_ctx* c, uint32_t i, mpdp_query_graph* g, mpdp_result* r) {
    if (!c || i >= c->subs.size()) return fail(nullptr, MPDP_ERR_INVALID_ARGUMENT, "no such sub-problem");
    const mpdp_ctx::SubProblem& sp = c->subs[i];
    if (g) {
        g->n = (uint32_t)sp.card.size();
        g->cardinalities = sp.card.data();
        g->n_edges = (uint32_t)sp.sel.size();
        g->edges = sp.edges.data();
        g->selectivities = sp.sel.data();
        g->leaf_costs = sp.leaf.empty() ? nullptr : sp.leaf.data();
    }
    if (r) {
        mpdp_plan_node* nodes = r->nodes;
        const uint32_t cap = r->capacity;
        *r = sp.res;
        r->nodes = nodes;
        r->capacity = cap;
        if (nodes && cap >= sp.nodes.size()) memcpy(nodes, sp.nodes.data(), sizeof(mpdp_plan_node) * sp.nodes.size());
    }
    return MPDP_OK;
}

mpdp_status mpdp_heuristic_optimize_t(const mpdp_query_graph* g, mpdp_algo algo, uint32_t k, uint32_t t,
                                      mpdp_inner_solver solver, void* user, mpdp_result* out) {
    if (!solver) return fail(nullptr, MPDP_ERR_INVALID_ARGUMENT, "solver is NULL");
    if (algo != MPDP_ALGO_IDP2_MPDP && algo != MPDP_ALGO_UNIONDP_MPDP)
        return fail(nullptr, MPDP_ERR_INVALID_ARGUMENT, "algo must be IDP2_MPDP or UNIONDP_MPDP");
    if (algo == MPDP_ALGO_IDP2_MPDP && t != 0 && t != k)
        return fail(nullptr, MPDP_ERR_INVALID_ARGUMENT, "t applies to UNIONDP_MPDP only");
    std::string err;
    const mpdp_status st = mpdp_heur::run(g, algo, k, solver, user, out, err, nullptr, t);
    if (st != MPDP_OK) return fail(nullptr, st, err);
    return MPDP_OK;
}

mpdp_status mpdp_heuristic_optimize(const mpdp_query_graph* g, mpdp_algo algo, uint32_t k,
                                    mpdp_inner_solver solver, void* user, mpdp_result* out) {
    return mpdp_heuristic_optimize_t(g, algo, k, 0, solver, user, out);
}

mpdp_status mpdp_optimize_uniondp(mpdp_ctx* c, const mpdp_query_graph* g, uint32_t k, uint32_t t, mpdp_result* out) {
    if (!c) return fail(nullptr, MPDP_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (!out) return fail(c, MPDP_ERR_INVALID_ARGUMENT, "out is NULL");
    c->subs.clear();
    std::string err;
    const mpdp_status st = mpdp_heur::run(g, MPDP_ALGO_UNIONDP_MPDP, k, gpu_inner_solver, c, out, err, gpu_inner_batch, t);
    if (st != MPDP_OK) return fail(c, st, err.empty() ? c->err : err);
    return MPDP_OK;
}


int mpdp_abi_version(void) { return MPDP_ABI_VERSION; }

const char* mpdp_status_string(mpdp_status s) {
    switch (s) {
        case MPDP_OK: return "MPDP_OK";
        case MPDP_ERR_INVALID_ARGUMENT: return "MPDP_ERR_INVALID_ARGUMENT";
        case MPDP_ERR_DISCONNECTED: return "MPDP_ERR_DISCONNECTED";
        case MPDP_ERR_CAPACITY: return "MPDP_ERR_CAPACITY";
        case MPDP_ERR_TIMEOUT: return "MPDP_ERR_TIMEOUT";
        case MPDP_ERR_OOM: return "MPDP_ERR_OOM";
        case MPDP_ERR_CUDA: return "MPDP_ERR_CUDA";
        case MPDP_ERR_NCCL: return "MPDP_ERR_NCCL";
        case MPDP_ERR_INTERNAL: return "MPDP_ERR_INTERNAL";
        case MPDP_ERR_UNSUPPORTED: return "MPDP_ERR_UNSUPPORTED";
    }
    return "unknown";
}

const char* mpdp_last_error(const mpdp_ctx* ctx) {
    if (ctx) return ctx->err.c_str();
    return g_tls_error.c_str();
}

void mpdp_share(uint64_t total, int rank, int world, uint64_t* lo, uint64_t* hi) {
    if (world < 1) world = 1;
    const uint64_t seg = (total + (uint64_t)world - 1) / (uint64_t)world;   // equal segments (in-place allgather)
    *lo = std::min<uint64_t>(total, (uint64_t)rank * seg);
    *hi = std::min<uint64_t>(total, (uint64_t)(rank + 1) * seg);
}

mpdp_status mpdp_ctx_create(const mpdp_ctx_config* cfg, mpdp_ctx** out) {
    if (!cfg || !out) return fail(nullptr, MPDP_ERR_INVALID_ARGUMENT, "cfg/out is NULL");
    *out = nullptr;
    if (cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world)
        return fail(nullptr, MPDP_ERR_INVALID_ARGUMENT, "bad rank/world");
    const bool simulate = cfg->world > 1 && (cfg->flags & MPDP_FLAG_SIMULATE_WORLD);
    if (simulate && (cfg->rank != 0 || cfg->world > kMaxShards))
        return fail(nullptr, MPDP_ERR_INVALID_ARGUMENT, "simulated world: rank must be 0 and world <= 16");
    if (cfg->world > 1 && !simulate && !cfg->nccl_unique_id)
        return fail(nullptr, MPDP_ERR_INVALID_ARGUMENT, "world > 1 needs an NCCL unique id");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(nullptr, MPDP_ERR_CUDA, "no CUDA device (this library has no CPU path)");
    if (cfg->device < 0 || cfg->device >= ndev) return fail(nullptr, MPDP_ERR_INVALID_ARGUMENT, "bad device");
    if (cfg->load_factor < 0.0 || cfg->load_factor > 0.9)
        return fail(nullptr, MPDP_ERR_INVALID_ARGUMENT, "load_factor outside (0, 0.9]");
    mpdp_ctx* c = new mpdp_ctx();
    c->device = cfg->device;
    c->rank = cfg->rank;
    c->world = cfg->world;
    c->simulate = simulate;
    c->nccl_self = cfg->world == 1 && (cfg->flags & MPDP_FLAG_NCCL_SELF);
    c->multi = cfg->world > 1 || c->nccl_self;
    c->timeout_ms = cfg->timeout_ms;
    c->flags = cfg->flags;
    if (cfg->load_factor > 0.0) c->load_factor = cfg->load_factor;
    auto bail = [&](mpdp_status s) {
        mpdp_ctx_destroy(c);
        return s;
    };
    if (cudaSetDevice(c->device) != cudaSuccess) return bail(fail(nullptr, MPDP_ERR_CUDA, "cudaSetDevice failed"));
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, c->device);
    c->num_sms = prop.multiProcessorCount;
    if (prop.major < 10) return bail(fail(nullptr, MPDP_ERR_CUDA, "needs an sm_100 (Blackwell B200) device"));
    if (cfg->cuda_stream) {
        c->stream = (cudaStream_t)cfg->cuda_stream;
    } else {
        if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
            return bail(fail(nullptr, MPDP_ERR_CUDA, "stream create failed"));
        c->own_stream = true;
    }
    if (cfg->workspace) {
        c->ws = (unsigned char*)cfg->workspace;
        c->ws_bytes = cfg->workspace_bytes;
    } else {
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        size_t want = cfg->mem_budget_bytes ? cfg->mem_budget_bytes : (size_t)(fr * 0.25);
        if (cudaMalloc(&c->ws, want) != cudaSuccess) return bail(fail(nullptr, MPDP_ERR_OOM, "workspace allocation failed"));
        c->ws_bytes = want;
        c->own_ws = true;
    }
    if (cudaMemsetAsync(c->ws, 0, c->ws_bytes, c->stream) != cudaSuccess)
        return bail(fail(nullptr, MPDP_ERR_CUDA, "workspace clear failed"));
    const int nsh = simulate ? cfg->world : 1;
    if (cudaMallocHost(&c->h_query, sizeof(QueryDev<uint64_t>)) != cudaSuccess ||
        cudaMallocHost(&c->h_results, sizeof(ResultDev) * nsh) != cudaSuccess ||
        cudaMallocHost(&c->h_rank_pinned, sizeof(unsigned int) * rank_geom(32).entries) != cudaSuccess)
        return bail(fail(nullptr, MPDP_ERR_OOM, "pinned host allocation failed"));
    c->h_result = c->h_results;
    if ((cfg->world > 1 && !simulate) || c->nccl_self) {     // one NCCL communicator per context
        std::string err;
        c->nccl = nccl_api(err);
        if (!c->nccl) return bail(fail(nullptr, MPDP_ERR_NCCL, err));
        ncclUniqueId id;
        if (c->nccl_self) {                // a 1-rank communicator of our own
            if (c->nccl->GetUniqueId(&id) != 0) return bail(fail(nullptr, MPDP_ERR_NCCL, "ncclGetUniqueId failed"));
        } else {
            memcpy(&id, cfg->nccl_unique_id, sizeof(id));
        }
        const ncclResult_t r = c->nccl->CommInitRank(&c->comm, cfg->world, id, cfg->rank);
        if (r != 0)
            return bail(fail(nullptr, MPDP_ERR_NCCL, std::string("ncclCommInitRank: ") +
                                                         (c->nccl->GetErrorString ? c->nccl->GetErrorString(r) : "")));
    }
    cudaEventCreate(&c->ev0);
    cudaEventCreate(&c->ev1);
    for (auto& e : c->kev) cudaEventCreate(&e);
    if (cudaStreamSynchronize(c->stream) != cudaSuccess) return bail(fail(nullptr, MPDP_ERR_CUDA, "init sync failed"));
    *out = c;
    return MPDP_OK;
}

mpdp_status mpdp_ctx_peer_record(mpdp_ctx* c, void* out) {
    if (!c || !out) return fail(c, MPDP_ERR_INVALID_ARGUMENT, "ctx/out is NULL");
    if (c->world < 2 || c->simulate)
        return fail(c, MPDP_ERR_INVALID_ARGUMENT, "peer records are for multi-GPU contexts (world > 1, not simulated)");
    if (!c->own_ws) return fail(c, MPDP_ERR_INVALID_ARGUMENT, "peer records need a library-allocated workspace");
    CUDA_TRY(c, cudaSetDevice(c->device));
    cudaIpcMemHandle_t h;
    CUDA_TRY(c, cudaIpcGetMemHandle(&h, c->ws));
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    memcpy(out, &h, 64);
    const unsigned long long sz = c->ws_bytes;
    memcpy(static_cast<unsigned char*>(out) + 64, &sz, 8);
    return MPDP_OK;
}

mpdp_status mpdp_ctx_open_peers(mpdp_ctx* c, const void* records) {
    if (!c || !records) return fail(c, MPDP_ERR_INVALID_ARGUMENT, "ctx/records is NULL");
    if (c->world < 2 || c->simulate || c->world > kMaxXr)
        return fail(c, MPDP_ERR_INVALID_ARGUMENT, "peers: multi-GPU contexts of 2..8 ranks only");
    if (c->peers_open) return fail(c, MPDP_ERR_INVALID_ARGUMENT, "peers already open");
    const unsigned char* rec = static_cast<const unsigned char*>(records);
    for (int s = 0; s < c->world; s++) {
        unsigned long long sz;
        memcpy(&sz, rec + s * MPDP_PEER_RECORD_BYTES + 64, 8);
        if (sz != c->ws_bytes) return fail(c, MPDP_ERR_INVALID_ARGUMENT, "peers: unequal workspace sizes");
    }
    CUDA_TRY(c, cudaSetDevice(c->device));
    for (int s = 0; s < c->world; s++) {
        if (s == c->rank) {
            c->peer_ws[s] = c->ws;
            continue;
        }
        cudaIpcMemHandle_t h;
        memcpy(&h, rec + s * MPDP_PEER_RECORD_BYTES, 64);
        void* ptr = nullptr;
        if (cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            cudaGetLastError();
            for (int t = 0; t < s; t++)
                if (t != c->rank && c->peer_ws[t]) cudaIpcCloseMemHandle(c->peer_ws[t]);
            for (int t = 0; t < kMaxXr; t++) c->peer_ws[t] = nullptr;
            return fail(c, MPDP_ERR_CUDA, "cudaIpcOpenMemHandle of rank " + std::to_string(s) + " failed");
        }
        c->peer_ws[s] = static_cast<unsigned char*>(ptr);
    }
    c->peers_open = true;
    return MPDP_OK;
}

mpdp_status mpdp_ctx_destroy(mpdp_ctx* c) {
    if (!c) return MPDP_OK;
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->own_ws && c->ws) cudaFree(c->ws);
    if (c->h_query) cudaFreeHost(c->h_query);
    if (c->h_rank_pinned) cudaFreeHost(c->h_rank_pinned);
    if (c->comm && c->nccl && c->nccl->CommDestroy) c->nccl->CommDestroy(c->comm);
    if (c->h_results) cudaFreeHost(c->h_results);
    if (c->h_xr) cudaFreeHost(c->h_xr);
    for (int s = 0; s < kMaxXr; s++)
        if (c->peers_open && s != c->rank && c->peer_ws[s]) cudaIpcCloseMemHandle(c->peer_ws[s]);
    if (c->h_bq) cudaFreeHost(c->h_bq);
    if (c->h_br) cudaFreeHost(c->h_br);
    if (c->d_bq) cudaFree(c->d_bq);
    if (c->d_br) cudaFree(c->d_br);
    if (c->b_keys) cudaFree(c->b_keys);
    if (c->b_vals) cudaFree(c->b_vals);
    if (c->d_sub_ids) cudaFree(c->d_sub_ids);
    if (c->h_sub_ids) cudaFreeHost(c->h_sub_ids);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    for (auto& e : c->kev)
        if (e) cudaEventDestroy(e);
    for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second.exec);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
    return MPDP_OK;
}

mpdp_status mpdp_stage(mpdp_ctx* c, const mpdp_query_graph* g) {
    if (!c) return fail(nullptr, MPDP_ERR_INVALID_ARGUMENT, "ctx is NULL");
    c->staged = false;
    c->ran = false;
    std::vector<unsigned long long> adj;
    mpdp_status st = validate(c, g, adj);
    if (st != MPDP_OK) return st;
    CUDA_TRY(c, cudaSetDevice(c->device));
    // the previous query's D2H must be done before the pinned buffers are reused
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    const int n = (int)g->n;
    c->n = n;
    c->wide = n > 32 || (c->flags & MPDP_FLAG_FORCE_WIDE_MASKS);
    const unsigned long long m = g->n_edges;
    c->m = m;
    if (n >= 3 && m == (unsigned long long)n * (n - 1) / 2) c->cls = CLS_CLIQUE;
    else if (m == (unsigned long long)(n - 1)) c->cls = CLS_TREE;
    else c->cls = CLS_GENERAL;
    if (c->flags & MPDP_FLAG_DPSUB_ENUM) c->cls = CLS_GENERAL;   // ablation: the generic kernels
    const DevLayout prev = c->lay;
    st = plan_layout(c);
    if (st != MPDP_OK) return st;
    // memo tags: a fresh tag per query makes every slot of an earlier query read as empty
    const int width = c->wide ? 64 : 32;
    bool clear = (c->last_width != 0 && c->last_width != width);   // arena geometry changed
    // dense memo entries are plain doubles: they must not be read as hash tags later
    if (c->lay.memo_kind == MEMO_HASH && c->last_memo == MEMO_DENSE) clear = true;
    if (prev.tiles != c->lay.tiles || prev.tiles_cap != c->lay.tiles_cap)   // ring moved/grew over scratch
        CUDA_TRY(c, cudaMemsetAsync(c->ws + c->lay.tiles, 0, sizeof(TileRec) * c->lay.tiles_cap, c->stream));
    if (c->wide) {
        if (++c->gen8 > 255) { c->gen8 = 1; clear = true; }
    } else {
        if (++c->gen32 == 0) { c->gen32 = 1; clear = true; }
    }
    if (clear) CUDA_TRY(c, cudaMemsetAsync(c->ws + c->lay.arena, 0, c->lay.cold - c->lay.arena, c->stream));
    c->last_width = width;
    c->last_memo = c->lay.memo_kind;
    // reading R20: general graphs on the bitmask memo test connectivity of
    // subsets by probing the cost array, so every slot starts absent
    c->memo_conn = c->lay.mask_memo && c->cls == CLS_GENERAL && !getenv("MPDP_DEBUG_BFS_CONN");
    if (c->memo_conn)
        CUDA_TRY(c, cudaMemsetAsync(c->ws + c->lay.dcost, 0xff, sizeof(double) << n, c->stream));
    if (c->lay.memo_kind == MEMO_DENSE && c->rank_n != n) {       // chunked colex-rank tables
        const RankGeom rg = rank_geom(n);
        std::vector<unsigned int>& tab = c->rank_cache[n];       // built once per n
        if (tab.empty()) {
            tab.assign(rg.entries, 0);
            for (int ch = 0; ch < rg.nch; ch++) {
                const int bits = std::min(8, n - 8 * ch);
                for (int o = 0; o <= 8 * ch; o++)
                    for (unsigned int bv = 0; bv < (1u << bits); bv++) {
                        unsigned long long val = 0;
                        int seen = 0;
                        for (int i = 0; i < bits; i++)
                            if (bv >> i & 1) val += binom_u64(8 * ch + i, o + (seen++) + 1);
                        tab[rg.base[ch] + o * rg.len[ch] + bv] = (unsigned int)val;
                    }
            }
        }
        // async from pinned memory: the stream is idle here (synchronised above),
        // so the staging buffer is free, and the kernels follow in stream order
        memcpy(c->h_rank_pinned, tab.data(), sizeof(unsigned int) * rg.entries);
        CUDA_TRY(c, cudaMemcpyAsync(c->ws + c->lay.rank, c->h_rank_pinned, sizeof(unsigned int) * rg.entries,
                                    cudaMemcpyHostToDevice, c->stream));
        c->rank_n = n;
    }
    c->query_counter++;
    // look-back epochs are 26 bits wide ((query * 64 + level) * 16 + shard):
    // recycle the ring records before an epoch value can repeat
    if ((c->query_counter & ((1ull << 15) - 1)) == 0)
        CUDA_TRY(c, cudaMemsetAsync(c->ws + c->lay.tiles, 0, sizeof(TileRec) * c->lay.tiles_cap, c->stream));
    if (c->wide) {
        fill_query<uint64_t>(c, g, adj, (QueryDev<uint64_t>*)c->h_query);
        CUDA_TRY(c, cudaMemcpyAsync(c->ws + c->lay.query, c->h_query, sizeof(QueryDev<uint64_t>), cudaMemcpyHostToDevice, c->stream));
        c->h2d_bytes = sizeof(QueryDev<uint64_t>);
    } else {
        fill_query<uint32_t>(c, g, adj, (QueryDev<uint32_t>*)c->h_query);
        CUDA_TRY(c, cudaMemcpyAsync(c->ws + c->lay.query, c->h_query, sizeof(QueryDev<uint32_t>), cudaMemcpyHostToDevice, c->stream));
        c->h2d_bytes = sizeof(QueryDev<uint32_t>);
    }
    c->staged = true;
    return MPDP_OK;
}

mpdp_status mpdp_run(mpdp_ctx* c) {
    if (!c) return fail(nullptr, MPDP_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (!c->staged) return fail(c, MPDP_ERR_INVALID_ARGUMENT, "no staged query");
    CUDA_TRY(c, cudaSetDevice(c->device));
    const mpdp_status st = c->wide ? run_typed<uint64_t>(c) : run_typed<uint32_t>(c);
    if (st == MPDP_OK) c->ran = true;
    return st;
}

mpdp_status mpdp_fetch(mpdp_ctx* c, mpdp_result* out) {
    if (!c || !out) return fail(c, MPDP_ERR_INVALID_ARGUMENT, "ctx/out is NULL");
    if (!c->ran) return fail(c, MPDP_ERR_INVALID_ARGUMENT, "nothing was run");
    const int n = c->n;
    if (out->nodes && out->capacity < (uint32_t)(2 * n - 1))
        return fail(c, MPDP_ERR_INVALID_ARGUMENT, "result capacity < 2n-1");
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    CUDA_TRY(c, cudaGetLastError());
    if (c->xr_run && c->simulate) {       // fused exchange: every replica holds the totals and the plan
        ResultDev* r0 = c->h_results;
        for (int sh = 1; sh < c->lay.nshards; sh++) {
            const ResultDev* rs = c->h_results + sh;
            r0->error |= rs->error;
            if (!r0->error && (rs->n_nodes != r0->n_nodes || rs->csg != r0->csg || rs->pairs != r0->pairs ||
                               rs->ccp != r0->ccp ||
                               memcmp(rs->nodes, r0->nodes, sizeof(mpdp_plan_node) * r0->n_nodes) != 0 ||
                               memcmp(&rs->cost, &r0->cost, sizeof(double)) != 0))
                return fail(c, MPDP_ERR_INTERNAL, "fused-exchange replicas extracted different plans or counters");
        }
    }
    if (c->sharded && c->simulate) {      // sum the shards' counters; all shards must agree on the plan
        ResultDev* r0 = c->h_results;
        for (int sh = 1; sh < c->lay.nshards; sh++) {
            const ResultDev* rs = c->h_results + sh;
            r0->error |= rs->error;
            r0->csg += rs->csg;
            r0->ccp += rs->ccp;
            r0->pairs += rs->pairs;
            r0->probes += rs->probes;
            for (int k = 0; k <= n; k++) {
                r0->lvl_csg[k] += rs->lvl_csg[k];
                r0->lvl_ccp[k] += rs->lvl_ccp[k];
                r0->lvl_pairs[k] += rs->lvl_pairs[k];
            }
            if (!r0->error && (rs->n_nodes != r0->n_nodes ||
                               memcmp(rs->nodes, r0->nodes, sizeof(mpdp_plan_node) * r0->n_nodes) != 0 ||
                               memcmp(&rs->cost, &r0->cost, sizeof(double)) != 0))
                return fail(c, MPDP_ERR_INTERNAL, "simulated ranks extracted different plans");
        }
    }
    const ResultDev* r = c->h_result;
    if (r->error) {
        if (r->error & ERR_TIMEOUT)
            return fail(c, MPDP_ERR_TIMEOUT, "timeout_ms exceeded on the device (checked at every chunk of the level loop)");
        if (r->error & ERR_HANG)
            return fail(c, MPDP_ERR_INTERNAL, "device watchdog fired (a spin-wait exceeded 2 s); results discarded");
        if (r->error & (ERR_CAPACITY | ERR_ITEMS))
            return fail(c, MPDP_ERR_CAPACITY, "memo does not fit the workspace (device error bits " + std::to_string(r->error) + ")");
        return fail(c, MPDP_ERR_INTERNAL, "device consistency check failed (bits " + std::to_string(r->error) + ")");
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, c->ev0, c->ev1);
    out->time_ms = ms;
    out->n_nodes = r->n_nodes;
    out->root = r->n_nodes ? r->n_nodes - 1 : 0;
    out->cost = r->cost;
    out->csg_count = r->csg;
    out->ccp_pairs = r->ccp;
    out->pairs_evaluated = r->pairs;
    out->gpu_launches = c->launches;
    out->probes = r->probes;
    out->h2d_bytes = c->h2d_bytes;
    out->d2h_bytes = c->d2h_bytes;
    out->enum_launches = c->enum_launches;
    out->eval_launches = c->eval_launches;
    out->memo_kind = c->star ? 4u : c->tree1 ? 1u : c->small ? 3u : c->lay.mask_memo && c->fused ? 2u : (uint32_t)c->lay.memo_kind;
    out->enum_ms = out->eval_ms = 0;
    if (c->fused && c->nkev == 2) {      // the fused kernel: enumeration and evaluation together
        float t = 0;
        cudaEventElapsedTime(&t, c->kev[0], c->kev[1]);
        out->eval_ms = t;
    }
    for (int i = 0; !c->fused && i + 1 < c->nkev; i++) {
        float t = 0;
        cudaEventElapsedTime(&t, c->kev[i], c->kev[i + 1]);
        if (i % 2 == 0) out->enum_ms += t;
        else out->eval_ms += t;
    }
    if (out->nodes) memcpy(out->nodes, r->nodes, sizeof(mpdp_plan_node) * r->n_nodes);
    for (int k = 0; k <= n; k++) {
        if (out->level_ms)
            out->level_ms[k] = (k >= 2 && r->t_level[k] && r->t_level[k + 1]) ? 1e-6 * (double)(r->t_level[k + 1] - r->t_level[k]) : 0.0;
        if (out->level_csg) out->level_csg[k] = r->lvl_csg[k];
        if (out->level_ccp) out->level_ccp[k] = r->lvl_ccp[k];
        if (out->level_pairs) out->level_pairs[k] = r->lvl_pairs[k];
    }
    return MPDP_OK;
}

mpdp_status mpdp_optimize(mpdp_ctx* c, const mpdp_query_graph* g, mpdp_algo algo, uint32_t k, mpdp_result* out) {
    if (!c) return fail(nullptr, MPDP_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (!out) return fail(c, MPDP_ERR_INVALID_ARGUMENT, "out is NULL");
    switch (algo) {
        case MPDP_ALGO_MPDP:
            if (k != 0) return fail(c, MPDP_ERR_INVALID_ARGUMENT, "k must be 0 for MPDP");
            break;
        case MPDP_ALGO_DPSIZE_REF:
            return fail(c, MPDP_ERR_UNSUPPORTED,
                        "DPSIZE_REF is the CPU reference; it lives in the test oracle (oracle/liboracle.so), "
                        "not in this GPU library");
        case MPDP_ALGO_IDP2_MPDP:
        case MPDP_ALGO_UNIONDP_MPDP: {
            c->subs.clear();
            std::string err;
            const mpdp_status st = mpdp_heur::run(g, algo, k, gpu_inner_solver, c, out, err, gpu_inner_batch);
            if (st != MPDP_OK) return fail(c, st, err.empty() ? c->err : err);
            return MPDP_OK;
        }
        default:
            return fail(c, MPDP_ERR_INVALID_ARGUMENT, "unknown algorithm");
    }
    mpdp_status st = mpdp_stage(c, g);
    if (st != MPDP_OK) return st;
    st = mpdp_run(c);
    if (st != MPDP_OK) return st;
    return mpdp_fetch(c, out);
}

// Multi-GPU batch (independent sub-problems, e.g. one UnionDP level's
// partitions): rank r solves the queries i = r (mod W) with the
// single-GPU kernels and the ranks allgather the results (plan, cost,
// counters) over NCCL, so every rank returns every result.
struct BatchRec {
    double cost, time_ms;
    unsigned long long csg, ccp, pairs, probes;
    unsigned int n_nodes, memo_kind, gpu_launches, status;
    mpdp_plan_node nodes[2 * kMaxN - 1];
};

static mpdp_status batch_distributed(mpdp_ctx* c, const mpdp_query_graph* graphs, uint32_t count,
                                     mpdp_result* results) {
    const int W = c->nccl_self ? 1 : c->world, rank = c->nccl_self ? 0 : c->rank;
    std::vector<mpdp_query_graph> lg;
    std::vector<mpdp_result> lr;
    std::vector<uint32_t> li;
    for (uint32_t i = (uint32_t)rank; i < count; i += (uint32_t)W) {
        li.push_back(i);
        lg.push_back(graphs[i]);
        lr.push_back(results[i]);
    }
    const bool sm = c->multi, sn = c->nccl_self;
    const int sw = c->world;
    c->multi = false;                      // this rank's share on the single-GPU kernels
    c->nccl_self = false;
    c->world = 1;
    const mpdp_status st = li.empty() ? MPDP_OK : mpdp_optimize_batch(c, lg.data(), (uint32_t)lg.size(), lr.data());
    c->multi = sm;
    c->nccl_self = sn;
    c->world = sw;
    const unsigned long long seg = (count + (uint32_t)W - 1) / (uint32_t)W;
    std::vector<BatchRec> mine(seg);
    memset(mine.data(), 0, sizeof(BatchRec) * seg);
    for (size_t j = 0; j < li.size(); j++) {
        BatchRec& b = mine[j];
        const mpdp_result& r = lr[j];
        b.status = (unsigned int)st;
        if (st != MPDP_OK) continue;
        b.cost = r.cost;
        b.time_ms = r.time_ms;
        b.csg = r.csg_count;
        b.ccp = r.ccp_pairs;
        b.pairs = r.pairs_evaluated;
        b.probes = r.probes;
        b.n_nodes = r.n_nodes;
        b.memo_kind = r.memo_kind;
        b.gpu_launches = r.gpu_launches;
        if (r.nodes) memcpy(b.nodes, r.nodes, sizeof(mpdp_plan_node) * std::min<uint32_t>(r.n_nodes, 2 * kMaxN - 1));
        else b.n_nodes = 0;
    }
    if (st != MPDP_OK && W == 1) return st;
    // allgather of the fixed-size records (device staging)
    const size_t bytes = sizeof(BatchRec) * seg;
    unsigned char* d = nullptr;
    CUDA_TRY(c, cudaMalloc(&d, bytes * W));
    std::vector<BatchRec> all(seg * W);
    mpdp_status out = MPDP_OK;
    if (cudaMemcpyAsync(d + bytes * rank, mine.data(), bytes, cudaMemcpyHostToDevice, c->stream) != cudaSuccess) {
        out = fail(c, MPDP_ERR_CUDA, "batch record upload failed");
    } else {
        ncclResult_t e = c->nccl->AllGather(d + bytes * rank, d, bytes, /*ncclInt8*/ 0, c->comm, c->stream);
        if (e) out = fail(c, MPDP_ERR_NCCL, "ncclAllGather of the batch results failed");
        else if (cudaMemcpyAsync(all.data(), d, bytes * W, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
                 cudaStreamSynchronize(c->stream) != cudaSuccess)
            out = fail(c, MPDP_ERR_CUDA, "batch record download failed");
    }
    cudaFree(d);
    if (out != MPDP_OK) return out;
    for (uint32_t i = 0; i < count; i++) {
        const BatchRec& b = all[(i % (uint32_t)W) * seg + i / (uint32_t)W];
        if (b.status != MPDP_OK) return fail(c, (mpdp_status)b.status, "a batched query failed on rank " + std::to_string(i % W));
        mpdp_result& r = results[i];
        r.cost = b.cost;
        r.time_ms = b.time_ms;
        r.csg_count = b.csg;
        r.ccp_pairs = b.ccp;
        r.pairs_evaluated = b.pairs;
        r.probes = b.probes;
        r.n_nodes = b.n_nodes;
        r.root = b.n_nodes ? b.n_nodes - 1 : 0;
        r.memo_kind = b.memo_kind;
        r.gpu_launches = b.gpu_launches;
        r.inner_calls = 0;
        if (r.nodes) memcpy(r.nodes, b.nodes, sizeof(mpdp_plan_node) * b.n_nodes);
    }
    c->staged = false;
    c->ran = false;
    return MPDP_OK;
}

mpdp_status mpdp_optimize_batch(mpdp_ctx* c, const mpdp_query_graph* graphs, uint32_t count, mpdp_result* results) {
    if (!c) return fail(nullptr, MPDP_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (count && (!graphs || !results)) return fail(c, MPDP_ERR_INVALID_ARGUMENT, "graphs/results is NULL");
    CUDA_TRY(c, cudaSetDevice(c->device));
    if (c->multi && c->nccl && !c->simulate && count) return batch_distributed(c, graphs, count, results);
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));     // pinned staging is reused
    const bool batchable = !c->multi && c->timeout_ms <= 0 &&
                           !(c->flags & (MPDP_FLAG_NO_SMALL | MPDP_FLAG_NO_FUSED | MPDP_FLAG_PROFILE_KERNELS |
                                         MPDP_FLAG_HASH_MEMO | MPDP_FLAG_FORCE_WIDE_MASKS | MPDP_FLAG_DPSUB_ENUM));
    // three kinds: small trees (n <= 13: one CTA each, memo in shared memory),
    // mid-size trees (n <= 32, every level <= kBatchListCap sets: one CTA each,
    // the shared 128-bit-key memo), everything else one by one
    std::vector<uint32_t> small, mid;
    std::vector<std::vector<unsigned long long>> adj_small, adj_mid;
    for (uint32_t i = 0; i < count; i++) {
        std::vector<unsigned long long> adj;
        const mpdp_status st = validate(c, &graphs[i], adj);
        if (st != MPDP_OK) return st;
        const int n = (int)graphs[i].n;
        if (results[i].nodes && results[i].capacity < (uint32_t)(2 * n - 1))
            return fail(c, MPDP_ERR_INVALID_ARGUMENT, "result capacity < 2n-1");
        const bool tree = n >= 2 && graphs[i].n_edges == (uint32_t)(n - 1);
        if (!batchable || !tree) continue;
        if (n <= kSmallMaxN) {
            small.push_back(i);
            adj_small.push_back(std::move(adj));
        } else if (n <= kBatchMaxN) {
            mid.push_back(i);
            adj_mid.push_back(std::move(adj));
        }
    }
    const uint32_t ns = (uint32_t)small.size();
    // fill_query writes per-query context fields (n, class, width, star hub,
    // largest tree level, csg): the batch restores them afterwards
    const int saved_n = c->n, saved_cls = c->cls, saved_hub = c->star_hub;
    const bool saved_wide = c->wide;
    const unsigned long long saved_tml = c->tree_max_level, saved_csg = c->tree_csg;
    std::vector<uint32_t> mid_ok;                        // mid trees whose levels fit the lists
    std::vector<unsigned long long> mid_csg;
    if (ns + mid.size() > c->batch_cap) {                // grow the staging
        if (c->h_bq) cudaFreeHost(c->h_bq);
        if (c->h_br) cudaFreeHost(c->h_br);
        if (c->d_bq) cudaFree(c->d_bq);
        if (c->d_br) cudaFree(c->d_br);
        if (c->h_sub_ids) cudaFreeHost(c->h_sub_ids);
        if (c->d_sub_ids) cudaFree(c->d_sub_ids);
        c->h_bq = nullptr;
        c->h_br = nullptr;
        c->d_bq = nullptr;
        c->d_br = nullptr;
        c->h_sub_ids = nullptr;
        c->d_sub_ids = nullptr;
        c->batch_cap = 0;
        const uint32_t cap = std::max<uint32_t>(ns + (uint32_t)mid.size(), 64);
        if (cudaMallocHost(&c->h_bq, sizeof(QueryDev<uint32_t>) * cap) != cudaSuccess ||
            cudaMallocHost(&c->h_br, sizeof(ResultDev) * cap) != cudaSuccess ||
            cudaMallocHost(&c->h_sub_ids, sizeof(unsigned int) * cap) != cudaSuccess ||
            cudaMalloc(&c->d_bq, sizeof(QueryDev<uint32_t>) * cap) != cudaSuccess ||
            cudaMalloc(&c->d_br, sizeof(ResultDev) * cap) != cudaSuccess ||
            cudaMalloc(&c->d_sub_ids, sizeof(unsigned int) * cap) != cudaSuccess)
            return fail(c, MPDP_ERR_OOM, "batch staging allocation failed");
        c->batch_cap = cap;
    }
    int maxn = 2;
    for (uint32_t b = 0; b < ns; b++) {
        const mpdp_query_graph& g = graphs[small[b]];
        c->n = (int)g.n;
        c->cls = CLS_TREE;
        c->wide = false;
        fill_query<uint32_t>(c, &g, adj_small[b], c->h_bq + b);
        maxn = std::max(maxn, (int)g.n);
    }
    unsigned long long csg_total = 0;
    for (size_t b = 0; b < mid.size(); b++) {
        const mpdp_query_graph& g = graphs[mid[b]];
        c->n = (int)g.n;
        c->cls = CLS_TREE;
        c->wide = false;
        const uint32_t at = ns + (uint32_t)mid_ok.size();
        fill_query<uint32_t>(c, &g, adj_mid[b], c->h_bq + at);
        if (c->tree_max_level > (unsigned long long)kBatchListCap) continue;   // one by one
        c->h_sub_ids[at] = (uint32_t)mid_ok.size();
        mid_ok.push_back(mid[b]);
        mid_csg.push_back(c->tree_csg);
        csg_total += c->tree_csg;
    }
    c->n = saved_n;
    c->cls = saved_cls;
    c->wide = saved_wide;
    c->star_hub = saved_hub;
    c->tree_max_level = saved_tml;
    c->tree_csg = saved_csg;
    const uint32_t nm = (uint32_t)mid_ok.size();
    if (nm) {                                            // the shared memo: load factor <= 0.5
        unsigned long long cap = 1024;
        while (cap < 2 * csg_total) cap <<= 1;
        if (cap > c->b_cap) {
            if (c->b_keys) cudaFree(c->b_keys);
            if (c->b_vals) cudaFree(c->b_vals);
            c->b_keys = nullptr;
            c->b_vals = nullptr;
            c->b_cap = 0;
            if (cudaMalloc(&c->b_keys, sizeof(Key128) * cap) != cudaSuccess ||
                cudaMalloc(&c->b_vals, sizeof(Val128) * cap) != cudaSuccess)
                return fail(c, MPDP_ERR_OOM, "batch memo allocation failed");
            CUDA_TRY(c, cudaMemsetAsync(c->b_keys, 0, sizeof(Key128) * cap, c->stream));
            c->b_cap = cap;
            c->b_epoch = 0;
        }
        if (++c->b_epoch >= (1u << 31)) {                // epochs wrapped: clear once
            CUDA_TRY(c, cudaMemsetAsync(c->b_keys, 0, sizeof(Key128) * c->b_cap, c->stream));
            c->b_epoch = 1;
        }
    }
    const uint32_t nb = ns + nm;
    if (nb) {
        CUDA_TRY(c, cudaEventRecord(c->ev0, c->stream));
        CUDA_TRY(c, cudaMemcpyAsync(c->d_bq, c->h_bq, sizeof(QueryDev<uint32_t>) * nb, cudaMemcpyHostToDevice, c->stream));
        if (ns) {
            if (!c->batch_attr) {
                CUDA_TRY(c, cudaFuncSetAttribute(k_dp_small_batch<CLS_TREE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)small_smem_bytes(kSmallMaxN)));
                c->batch_attr = true;
            }
            k_dp_small_batch<CLS_TREE><<<ns, kSmallBlock, small_smem_bytes(maxn), c->stream>>>(c->d_bq, c->d_br);
            CUDA_TRY(c, cudaGetLastError());
        }
        if (nm) {
            if (!c->batch128_attr) {
                CUDA_TRY(c, cudaFuncSetAttribute(k_dp_tree_batch, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)batch128_smem_bytes()));
                c->batch128_attr = true;
            }
            CUDA_TRY(c, cudaMemcpyAsync(c->d_sub_ids + ns, c->h_sub_ids + ns, sizeof(unsigned int) * nm,
                                        cudaMemcpyHostToDevice, c->stream));
            Memo128 m{c->b_keys, c->b_vals, c->b_cap - 1, c->b_epoch};
            k_dp_tree_batch<<<nm, kBatchBlock, batch128_smem_bytes(), c->stream>>>(c->d_bq + ns, c->d_br + ns, m,
                                                                                c->d_sub_ids + ns);
            CUDA_TRY(c, cudaGetLastError());
        }
        CUDA_TRY(c, cudaMemcpyAsync(c->h_br, c->d_br, sizeof(ResultDev) * nb, cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(c, cudaEventRecord(c->ev1, c->stream));
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
        float ms = 0;
        cudaEventElapsedTime(&ms, c->ev0, c->ev1);
        for (uint32_t b = 0; b < nb; b++) {
            const ResultDev* r = c->h_br + b;
            const uint32_t qi = b < ns ? small[b] : mid_ok[b - ns];
            mpdp_result* out = &results[qi];
            const int n = (int)graphs[qi].n;
            if (r->error) return fail(c, MPDP_ERR_INTERNAL, "device consistency check failed in a batched query (bits " +
                                             std::to_string(r->error) + ")");
            if (b >= ns && r->csg != mid_csg[b - ns])
                return fail(c, MPDP_ERR_INTERNAL, "batched tree query: connected sets differ from the subtree count");
            out->time_ms = ms;                  // the whole batched launch
            out->n_nodes = r->n_nodes;
            out->root = r->n_nodes ? r->n_nodes - 1 : 0;
            out->cost = r->cost;
            out->csg_count = r->csg;
            out->ccp_pairs = r->ccp;
            out->pairs_evaluated = r->pairs;
            out->gpu_launches = 1;
            out->probes = r->probes;
            out->h2d_bytes = sizeof(QueryDev<uint32_t>);
            out->d2h_bytes = sizeof(ResultDev);
            out->enum_launches = 0;
            out->eval_launches = 1;
            out->memo_kind = b < ns ? 3u : 5u;
            out->inner_calls = 0;
            out->enum_ms = 0;
            out->eval_ms = ms;
            if (out->nodes) memcpy(out->nodes, r->nodes, sizeof(mpdp_plan_node) * r->n_nodes);
            for (int k = 0; k <= n; k++) {
                if (out->level_ms) out->level_ms[k] = (k >= 2 && r->t_level[k] && r->t_level[k + 1]) ? 1e-6 * (double)(r->t_level[k + 1] - r->t_level[k]) : 0.0;
                if (out->level_csg) out->level_csg[k] = r->lvl_csg[k];
                if (out->level_ccp) out->level_ccp[k] = r->lvl_ccp[k];
                if (out->level_pairs) out->level_pairs[k] = r->lvl_pairs[k];
            }
        }
    }
    // the rest one by one
    std::vector<char> done(count, 0);
    for (uint32_t i : small) done[i] = 1;
    for (uint32_t i : mid_ok) done[i] = 1;
    const auto t1 = std::chrono::steady_clock::now();
    unsigned int singles = 0, max_single_n = 0;
    for (uint32_t i = 0; i < count; i++) {
        if (done[i]) continue;
        const mpdp_status st = mpdp_optimize(c, &graphs[i], MPDP_ALGO_MPDP, 0, &results[i]);
        if (st != MPDP_OK) return st;
        singles++;
        max_single_n = std::max(max_single_n, graphs[i].n);
    }
    if (getenv("MPDP_DEBUG_HEUR_TIME"))
        fprintf(stderr, "[batch] %u queries: %u small + %u mid in %.3f ms device time, %u one by one (max n %u) in %.3f ms\n",
                count, ns, nm, nb ? results[ns ? small[0] : mid_ok[0]].time_ms : 0.0, singles, max_single_n,
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count());
    // a batch replaces whatever mpdp_stage had staged (the one-by-one queries
    // restage the context): a later mpdp_run / mpdp_fetch must restage first
    c->staged = false;
    c->ran = false;
    return MPDP_OK;
}

#ifdef MPDP_TRACE
// Debug: per-CTA barrier arrival times of the last fused run, [level][cta].
int mpdp_debug_cta_trace(unsigned long long* out, int cap) {
    const int n = (kMaxN + 1) * kCtaTraceMax * kCtaTraceSlots;
    if (cap < n) return 0;
    if (cudaMemcpyFromSymbol(out, g_cta_arrive, sizeof(unsigned long long) * n) != cudaSuccess) return 0;
    return kCtaTraceMax;
}
void mpdp_debug_cta_trace_clear() {
    void* a = nullptr;
    if (cudaGetSymbolAddress(&a, g_cta_arrive) == cudaSuccess) cudaMemset(a, 0, sizeof(g_cta_arrive));
    cudaDeviceSynchronize();
}
#endif

// Debug: copy the block-0 phase trace of the last fused run (MPDP_TRACE builds).
int mpdp_debug_trace(const mpdp_ctx* c, unsigned long long* out, int cap) {
    if (!c || !c->h_result || !out) return 0;
    int nn = 0;
    for (int i = 0; i < kTraceCap && i < cap; i++) {
        if (!c->h_result->trace[i]) break;
        out[nn++] = c->h_result->trace[i];
    }
    return nn;
}

// Debug: per level k of the last whole-query run, the start (first chunk /
// level start) and, for the dataflow kernels, the finish of its last chunk, in
// us after the start of level 2 (0 = not recorded).  Returns n.
int mpdp_debug_level_span(const mpdp_ctx* c, double* start_us, double* done_us, int cap) {
    if (!c || !c->h_result || !start_us || !done_us) return 0;
    const ResultDev* r = c->h_result;
    unsigned long long t0 = ~0ull;
    for (int k = 2; k <= c->n + 1 && k < kMaxN + 2; k++)
        if (r->t_level[k]) t0 = std::min(t0, r->t_level[k]);
    int nn = 0;
    auto us = [&](unsigned long long t) { return t && t0 != ~0ull ? 1e-3 * ((double)t - (double)t0) : 0.0; };
    for (int k = 0; k <= c->n + 1 && k < cap && k < kMaxN + 2; k++, nn++) {
        start_us[k] = us(r->t_level[k]);
        done_us[k] = us(r->t_done[k]);
    }
    return nn;
}

// Debug (MPDP_DEBUG_DF_STATS set when the query ran): per CTA of the last
// dataflow launch 8 words {control: ns waiting for a free slot, ns waiting for
// dependencies, ns in the loop, chunks; compute warp 0: ns waiting for chunks,
// ns in the loop, -, -}.  Returns the words copied.
int mpdp_debug_df_stats(const mpdp_ctx* c, unsigned long long* out, int cap) {
    if (!c || !out || !getenv("MPDP_DEBUG_DF_STATS")) return 0;
    const int words = std::min(cap, 8 * kMaxGrid);
    if (cudaMemcpy(out, c->ws + c->lay.light, sizeof(unsigned long long) * words, cudaMemcpyDeviceToHost) != cudaSuccess)
        return 0;
    return words;
}

mpdp_status mpdp_nccl_get_unique_id(void* out128) {
    if (!out128) return fail(nullptr, MPDP_ERR_INVALID_ARGUMENT, "out is NULL");
    std::string err;
    NcclApi* api = nccl_api(err);
    if (!api) return fail(nullptr, MPDP_ERR_NCCL, err);
    ncclUniqueId id;
    const ncclResult_t r = api->GetUniqueId(&id);
    if (r != 0) return fail(nullptr, MPDP_ERR_NCCL, "ncclGetUniqueId failed");
    memcpy(out128, &id, sizeof(id));
    return MPDP_OK;
}

}  // extern "C"
