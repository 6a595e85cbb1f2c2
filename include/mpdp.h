/*
 * mpdp.h — C ABI of the B200-native MPDP exact join-order optimiser.
 *
 * What it computes: the minimum-C_out bushy join tree without cross products
 * for a connected query graph G(R, E) (§2.1), by the
 * level-by-level dynamic program of Alg. mpdp_gpu: for subset size
 * i = 2..n, unrank all i-subsets, filter the connected ones, evaluate MPDP's
 * block-based join pairs (Alg. mpdp_generalization), keep the best
 * pair per set and scatter it into a GPU memo hash table.
 * Every step runs in CUDA kernels on one B200 (sm_100a); the host only
 * validates the input, stages it and launches.  There is NO CPU fallback:
 * without a usable CUDA device every call returns MPDP_ERR_CUDA.
 *
 * Conventions (readings R1-R10):
 *   cost(leaf v) = leaf_costs[v] (0 when leaf_costs == NULL)
 *   cost(S)      = (cost(L) + cost(R)) + card(S)          (C_out)
 *   card(S)      = product of cardinalities of S and selectivities of the
 *                  edges induced by S, multiplied in the canonical order R5
 *   tie-break    = among equal costs the split with the numerically smaller
 *                  min(L, R) bitmask wins (R7); costs compare exactly
 *   counters     = csg_count incl. singletons (R1), unordered ccp_pairs (R2),
 *                  pairs_evaluated = sum over blocks (2^(b-1) - 1) (R3).
 *                  Counter convention: UNORDERED join pairs ({A,B} counted
 *                  once); the ordered convention of SPEC ("including the
 *                  symmetric ones") is exactly 2x ccp_pairs and 2x
 *                  pairs_evaluated.  Every pairs/s figure uses the unordered
 *                  count.
 *
 * Threading: a context is used by one host thread at a time.  All pointers
 * passed in are borrowed for the duration of the call and never retained.
 */
#ifndef MPDP_H
#define MPDP_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPDP_ABI_VERSION 1
/* exact algorithms: n <= 56.  SURVEY §8(b) asks for 64; the bound is the
 * 57 x 57 u64 binomial table staged per query (colex unranking of 64-bit masks)
 * and it is not binding in practice: a connected query with n > 40 only fits
 * the memo when it is sparse (the open-addressing memo holds its csg).        */
#define MPDP_MAX_RELATIONS_EXACT 56
#define MPDP_MAX_RELATIONS_HEURISTIC 16384  /* IDP2 / UnionDP drivers (O(n^2) host work) */

typedef enum {
    MPDP_OK = 0,
    MPDP_ERR_INVALID_ARGUMENT = 1,  /* bad pointer/size/value (see mpdp_optimize) */
    MPDP_ERR_DISCONNECTED = 2,      /* G is not connected: no CP-free plan */
    MPDP_ERR_CAPACITY = 3,          /* n too large or memo exceeds mem budget      */
    MPDP_ERR_TIMEOUT = 4,           /* timeout_ms exceeded (checked per level)     */
    MPDP_ERR_OOM = 5,               /* device allocation failed                    */
    MPDP_ERR_CUDA = 6,              /* CUDA runtime / no device / kernel fault     */
    MPDP_ERR_NCCL = 7,              /* NCCL failure (multi-GPU)                    */
    MPDP_ERR_INTERNAL = 8,          /* device-side consistency check failed        */
    MPDP_ERR_UNSUPPORTED = 9        /* algorithm not provided by this library      */
} mpdp_status;

typedef enum {
    MPDP_ALGO_DPSIZE_REF = 0,      /* the CPU reference: NOT in this library, by
                                      design and final.  The reference DP is the
                                      test oracle (oracle/liboracle.so), which the
                                      product may never link or call, so this value
                                      is reserved and always returns
                                      MPDP_ERR_UNSUPPORTED                          */
    MPDP_ALGO_MPDP = 1,            /* exact MPDP on the GPU                        */
    MPDP_ALGO_IDP2_MPDP = 2,       /* IDP2 with MPDP inner DP, bound k */
    MPDP_ALGO_UNIONDP_MPDP = 3     /* UnionDP with MPDP inner DP, k    */
} mpdp_algo;

/* The query graph (host memory).  Relations are 0..n-1, bit v of a set mask
 * is relation v. */
typedef struct {
    uint32_t n;                    /* relations, 1..56 for exact algorithms          */
    const double* cardinalities;   /* [n], finite, >= 0 (0 = empty input; composite
                                      cards of huge sub-plans can underflow to 0)     */
    uint32_t n_edges;
    const uint32_t* edges;         /* [2*n_edges] pairs {u, v}: u < v < n, no dups    */
    const double* selectivities;   /* [n_edges], in (0, 1]                            */
    const double* leaf_costs;      /* [n] finite >= 0, or NULL (= 0 for every leaf)   */
} mpdp_query_graph;

/* One plan node.  Internal nodes satisfy nodes[left].set < nodes[right].set
 * numerically (tie-break R7). */
typedef struct {
    int32_t left, right;           /* child node indices, -1 for leaves              */
    int32_t relation;              /* leaf: relation index; internal: -1             */
    uint32_t reserved;
    uint64_t set;                  /* relation bitmask of the subtree                */
    double cardinality;            /* card(set)                                      */
    double cost;                   /* C_out cost of the subtree                      */
} mpdp_plan_node;

typedef struct {
    mpdp_plan_node* nodes;         /* caller-owned, capacity >= 2n-1, post-order,
                                      root last; may be NULL (no plan copied)        */
    uint32_t capacity;
    uint32_t n_nodes;              /* out: 2n-1                                       */
    uint32_t root;                 /* out: n_nodes-1                                  */
    uint32_t gpu_launches;         /* out: kernels launched by this call              */
    double cost;                   /* out: optimal cost                               */
    uint64_t pairs_evaluated;      /* out: R3 units                                   */
    uint64_t ccp_pairs;            /* out: R2 units                                   */
    uint64_t csg_count;            /* out: R1 units                                   */
    uint64_t* level_csg;           /* optional [n+1] per-subset-size breakdowns       */
    uint64_t* level_ccp;           /* optional [n+1]                                  */
    uint64_t* level_pairs;         /* optional [n+1]                                  */
    double time_ms;                /* out: device time of the DP (CUDA events)        */
    uint64_t probes;               /* out: memo probes of non-singleton sets          */
    uint64_t h2d_bytes;            /* out: host->device bytes copied by this call     */
    uint64_t d2h_bytes;            /* out: device->host bytes copied by this call     */
    double enum_ms;                /* out, MPDP_FLAG_PROFILE_KERNELS: sum of k_enum   */
    double eval_ms;                /* out, MPDP_FLAG_PROFILE_KERNELS: sum of k_eval   */
    uint32_t enum_launches;        /* out: k_enum launches                            */
    uint32_t eval_launches;        /* out: k_eval launches                            */
    uint32_t memo_kind;            /* out: 1 = perfect-hash (colex rank) memo,
                                           0 = Murmur3 open-addressing memo,
                                           2 = bitmask-indexed memo (MEMO_MASK),
                                           3 = shared-memory bitmask memo of the
                                               single-CTA small-query kernel,
                                           4 = star memo (k_dp_star: C(n-1,k-1)
                                               entries per level, leaf-set rank),
                                           5 = the shared open-addressing memo of
                                               a batch, 128-bit {sub-problem,
                                               mask} keys (mpdp_optimize_batch) */
    uint32_t inner_calls;          /* out, IDP2/UnionDP: inner exact DP calls          */
    double* level_ms;              /* optional [n+1]: device time of each level (fused
                                      kernel: %globaltimer at the level barriers; 0 on
                                      the per-level-kernel path)                       */
} mpdp_result;

typedef struct {
    int device;                    /* CUDA device ordinal                              */
    int rank, world;               /* multi-GPU SPMD rank / size (1 process per GPU).
                                      world > 1: every level with >= 16384 k-subsets is
                                      split into `world` contiguous colex-rank shares;
                                      after the level each rank's memo segment is
                                      allgathered (ncclAllGather, in place); smaller
                                      levels are computed redundantly by every rank   */
    const void* nccl_unique_id;    /* 128 bytes (mpdp_nccl_get_unique_id on rank 0,
                                      broadcast by the caller); NULL when world == 1  */
    void* cuda_stream;             /* cudaStream_t to run on, or NULL (own stream)     */
    uint64_t mem_budget_bytes;     /* device memory the context may use; 0 = 75% of free */
    double timeout_ms;             /* 0 = none; checked between levels                 */
    void* workspace;               /* optional caller-owned device buffer (e.g. a torch
                                      tensor) the context sub-allocates from; NULL = the
                                      library allocates mem_budget_bytes itself        */
    uint64_t workspace_bytes;
    uint32_t flags;                /* MPDP_FLAG_* (0 for normal use)                   */
    double load_factor;            /* memo load factor in (0, 0.9]; 0 = default 0.5    */
} mpdp_ctx_config;

/* flags: use 64-bit set masks even when n <= 32 (exercises the wide kernels) */
#define MPDP_FLAG_FORCE_WIDE_MASKS 1u
/* flags: record CUDA events around every level kernel (enum_ms / eval_ms);
 * implies the direct-launch path (no graph replay)                             */
#define MPDP_FLAG_PROFILE_KERNELS 2u
/* flags: use the Murmur3 open-addressing memo even where the perfect-hash
 * (colex-rank) memo applies (n <= 32); for ablations                           */
#define MPDP_FLAG_HASH_MEMO 4u
/* flags: launch kernels one by one instead of replaying the cached CUDA graph
 * of the level loop (always the case when timeout_ms > 0)                      */
#define MPDP_FLAG_NO_GRAPH 8u
/* flags: do not use the single persistent cooperative kernel for the level
 * loop (perfect-hash memo); launch per-level kernels instead (ablation)        */
#define MPDP_FLAG_NO_FUSED 16u
/* flags: world > 1 WITHOUT NCCL: the context runs all `world` ranks as shards
 * (memo replicas) on its own device and exchanges the sharded levels by
 * device copies -- the sharded code path minus the NCCL transport (testing)   */
#define MPDP_FLAG_SIMULATE_WORLD 32u
/* flags: shard every level across ranks, even small ones (testing)             */
#define MPDP_FLAG_SHARD_ALL_LEVELS 64u
/* Ablation: enumerate every set as Alg. generic_dpsub does
 * (P:233-272): all 2^(|S|-1)-1 unordered splits with the CCP check on both
 * sides, no Find-Blocks and no tree/complete fast paths.  The plan and cost are
 * those of MPDP; pairs_evaluated becomes sum over connected S of
 * (2^(|S|-1) - 1) (reading R3's unordered convention; "2805x" of P:319 is the
 * ordered ratio).  The query runs through the general-graph kernels.           */
#define MPDP_FLAG_DPSUB_ENUM 256u
/* flags: keep the colex-rank memo layout on clique / general queries instead of
 * the bitmask-indexed one (MEMO_MASK, used for n <= 24 on one GPU by the
 * whole-query kernel); for ablations                                           */
#define MPDP_FLAG_RANK_MEMO 512u
/* flags: do not use the single-CTA shared-memory kernel for small queries
 * (n <= 13); run them through the multi-CTA whole-query kernels (ablation)    */
#define MPDP_FLAG_NO_SMALL 1024u
/* flags: no Collaborative Context Collection in the heavy phase of
 * block-decomposed sets (general graphs): lanes walk contiguous candidate
 * chunks and evaluate their valid pairs in place (ablation)                   */
#define MPDP_FLAG_NO_CCC 2048u
/* flags: run star queries (one relation adjacent to all others, n >= 14)
 * through the general tree kernel instead of k_dp_star (ablation)              */
#define MPDP_FLAG_NO_STAR 4096u
/* flags (testing, world == 1): create a real 1-rank NCCL communicator and run
 * every query on the multi-GPU sharded path with EVERY level sharded, so the
 * per-level ncclAllGather exchange and the counter ncclAllReduce execute on a
 * single GPU (bit-identical results to the single-GPU kernels)            */
#define MPDP_FLAG_NCCL_SELF 8192u
/* flags (multi-GPU contexts, star and clique queries): the FUSED PEER EXCHANGE instead of
 * per-level ncclAllGather (sets of one size are independent,
 * P:214, and a set reads only its subsets).  One
 * k_dp_star launch per rank; each chunk of sets stores its costs into every
 * rank's memo replica (NVLink peer stores) and adds its completion count to
 * every replica's per-(level, largest element) counters, so a chunk of level k
 * waits in its own replica for exactly the level-(k-1) sets it reads and no
 * level ends in a launch or a collective (cliques: k_dp_clique_df, every set's
 * cost, card and left into every rank's bitmask-memo replica).  With MPDP_FLAG_SIMULATE_WORLD the W
 * ranks are the CTA groups (blockIdx mod W) of ONE cooperative launch over the
 * W shards of the workspace; across GPUs call mpdp_ctx_open_peers first.
 * Results are bit-identical to the single-GPU kernel; every rank extracts the
 * plan from its own replica.  Other query shapes keep the NCCL path.        */
#define MPDP_FLAG_FUSED_EXCHANGE 16384u

/* Bytes of one rank's peer record for mpdp_ctx_open_peers: the CUDA IPC
 * handle of the context's workspace (64 B) and its size (8 B). */
#define MPDP_PEER_RECORD_BYTES 72

typedef struct mpdp_ctx mpdp_ctx;

/* Create a context on cfg->device.  Allocates (or adopts) the workspace and, for
 * world > 1, initialises the NCCL communicator.  Errors: INVALID_ARGUMENT (NULL
 * pointers, world < 1, rank out of range, world > 1 without a unique id),
 * CUDA (no device), OOM, NCCL. */
mpdp_status mpdp_ctx_create(const mpdp_ctx_config* cfg, mpdp_ctx** out);
mpdp_status mpdp_ctx_destroy(mpdp_ctx* ctx);

/* Fused peer exchange across GPUs (MPDP_FLAG_FUSED_EXCHANGE, world > 1 over
 * NCCL).  mpdp_ctx_peer_record writes this rank's MPDP_PEER_RECORD_BYTES-byte
 * record into out (host memory, caller-owned): the IPC handle of the
 * workspace, which must have been allocated by the library (cfg->workspace ==
 * NULL), and its size.  The caller gathers the records of all ranks (any host
 * collective) and passes them, rank-ordered and contiguous (world x
 * MPDP_PEER_RECORD_BYTES bytes, host memory, read only during the call), to
 * mpdp_ctx_open_peers, which maps every other rank's workspace into this
 * process (cudaIpcOpenMemHandle; the mappings are released by
 * mpdp_ctx_destroy).  All ranks must use equal workspace sizes (identical
 * layouts).  Errors: INVALID_ARGUMENT (NULL pointers, world == 1, simulated
 * world, adopted workspace, unequal sizes), CUDA (IPC not available). */
mpdp_status mpdp_ctx_peer_record(mpdp_ctx* ctx, void* out);
mpdp_status mpdp_ctx_open_peers(mpdp_ctx* ctx, const void* records);

/* Optimise one query end to end: validate, copy the graph host->device, run
 * every level, extract the plan on the device and copy the result back.
 * Blocks until the result is in *out.
 *   algo MPDP: k must be 0.  IDP2_MPDP / UNIONDP_MPDP: 2 <= k <= 32 (the
 *   paper uses 15 and 25).
 * Errors: INVALID_ARGUMENT (NULL pointers, n == 0, u >= v, v >= n, duplicate
 * edge, selectivity outside (0,1], cardinality < 0 or non-finite, negative or
 * non-finite leaf cost, out->capacity < 2n-1 with out->nodes != NULL, sum of
 * log10 cardinalities > 300), DISCONNECTED, CAPACITY (n > 56, memo larger than
 * the budget), TIMEOUT, CUDA, UNSUPPORTED (DPSIZE_REF).  On error *out is left
 * unspecified and mpdp_last_error() describes it. */
mpdp_status mpdp_optimize(mpdp_ctx* ctx, const mpdp_query_graph* graph, mpdp_algo algo,
                          uint32_t k, mpdp_result* out);

/* mpdp_optimize(MPDP) of `count` independent queries (e.g. the partitions of
 * one UnionDP level).  Small tree queries (n <= 13) are solved
 * together by ONE launch with one CTA per query (memo in shared memory);
 * tree queries with 14 <= n <= 32 whose levels hold at most 6144 connected
 * sets by a second launch, one CTA per query, all sharing ONE open-addressing
 * memo in HBM keyed by 128-bit {sub-problem, relation mask} (memo_kind 5);
 * the others run one by one as mpdp_optimize.  graphs[i] / results[i] have the
 * meaning, layout and ownership of mpdp_optimize's graph / out (results[i].nodes
 * caller-owned, capacity >= 2n-1); batched results report the launch's device
 * time.  Errors: as mpdp_optimize (the first one is returned; results of the
 * queries before it are valid).  Multi-GPU contexts (world > 1 over NCCL):
 * rank r solves the queries i = r (mod world) with the single-GPU kernels and
 * the ranks allgather the results (plan, cost, counters; the optional level
 * arrays are not exchanged), so every rank returns every result -- UnionDP's
 * independent partitions run on different GPUs.  A batch replaces
 * any query staged by mpdp_stage:
 * mpdp_run / mpdp_fetch after it fail with INVALID_ARGUMENT until the next
 * mpdp_stage.                                                                   */
mpdp_status mpdp_optimize_batch(mpdp_ctx* ctx, const mpdp_query_graph* graphs, uint32_t count,
                                mpdp_result* results);

/* Split form of mpdp_optimize(MPDP) for device-resident timing:
 *   mpdp_stage : validate + stage the graph (async H2D on the context stream)
 *   mpdp_run   : enqueue every level + plan extraction; returns without a host
 *                sync (single GPU), the memo and the plan stay in device memory
 *   mpdp_fetch : copy the result back (blocks) and check device status      */
mpdp_status mpdp_stage(mpdp_ctx* ctx, const mpdp_query_graph* graph);
mpdp_status mpdp_run(mpdp_ctx* ctx);
mpdp_status mpdp_fetch(mpdp_ctx* ctx, mpdp_result* out);

/* ---- IDP2 / UnionDP (algo IDP2_MPDP / UNIONDP_MPDP) ------------
 * Heuristic plans for large queries (n <= MPDP_MAX_RELATIONS_HEURISTIC, else
 * CAPACITY; plan node `set` masks are only filled when n <= 64).  The driver repeatedly solves sub-problems of at
 * most k relations exactly with the GPU MPDP (composite nodes carry
 * card = card of their subplan and leaf_cost = its cost).  result: the final
 * plan, its C_out cost recomputed over the whole tree, the counters summed over
 * the inner DP calls, inner_calls, and host wall time in time_ms.
 *
 * With MPDP_FLAG_RECORD_SUBPROBLEMS the context keeps every inner sub-problem
 * of the last call; mpdp_subproblem_get returns its graph (pointers into the
 * context, valid until the next call) and its result (nodes copied when
 * result->nodes != NULL and capacity suffices).                               */
#define MPDP_FLAG_RECORD_SUBPROBLEMS 128u
int mpdp_subproblem_count(const mpdp_ctx* ctx);
mpdp_status mpdp_subproblem_get(const mpdp_ctx* ctx, uint32_t i, mpdp_query_graph* graph,
                                mpdp_result* result);

/* The IDP2/UnionDP driver with a caller-supplied inner exact solver (host
 * logic only, no device needed; the product path is mpdp_optimize).  Used by
 * the tests to check the driver on machines without a GPU. */
typedef mpdp_status (*mpdp_inner_solver)(void* user, const mpdp_query_graph* sub, mpdp_result* out);
mpdp_status mpdp_heuristic_optimize(const mpdp_query_graph* graph, mpdp_algo algo, uint32_t k,
                                    mpdp_inner_solver solver, void* user, mpdp_result* out);
/* As mpdp_heuristic_optimize, with UnionDP's partition threshold t (0 = k;
 * IDP2 accepts only 0 or k). */
mpdp_status mpdp_heuristic_optimize_t(const mpdp_query_graph* graph, mpdp_algo algo, uint32_t k, uint32_t t,
                                      mpdp_inner_solver solver, void* user, mpdp_result* out);

/* UnionDP with the GPU MPDP inner DP and a partition threshold t
 * separate from k: partitions grow while their union has at most t relations
 * ("upper threshold t in [1, k]"), the recursion stops once at most
 * k composites remain (their exact plan is the root).  The paper's GPU runs
 * use k = 25, t = 15.  t = 0 means t = k (mpdp_optimize's
 * UNIONDP_MPDP).  Meaning, ownership and errors as mpdp_optimize; also
 * INVALID_ARGUMENT unless 2 <= t <= k <= 32. */
mpdp_status mpdp_optimize_uniondp(mpdp_ctx* ctx, const mpdp_query_graph* graph, uint32_t k, uint32_t t,
                                  mpdp_result* out);

/* Thread-local description of the last error on this context (never NULL). */
const char* mpdp_last_error(const mpdp_ctx* ctx);
const char* mpdp_status_string(mpdp_status s);
int mpdp_abi_version(void);

/* Debug: phase timestamps of CTA 0 of the last fused run (builds with
 * -DMPDP_TRACE; otherwise returns 0).  Entry = ns << 8 | level << 3 | phase. */
int mpdp_debug_trace(const mpdp_ctx* ctx, unsigned long long* out, int cap);

/* Debug: per subset size k (index k of caller-owned arrays of `cap` doubles)
 * of the last single-GPU whole-query run: when level k started and (dataflow
 * kernels k_dp_star / k_dp_clique) when its last chunk finished, in
 * microseconds after the first level start; 0 = not recorded.  Returns the
 * number of entries written (n + 2, at most cap). */
int mpdp_debug_level_span(const mpdp_ctx* ctx, double* start_us, double* done_us, int cap);

/* Debug: with the environment variable MPDP_DEBUG_DF_STATS set while the last
 * query ran on a dataflow kernel (k_dp_star / k_dp_clique), copies up to cap
 * words: per CTA 8 words {control warp: ns waiting for a free slot, ns waiting
 * for dependencies, ns in its loop, chunks; compute warp 0: ns waiting for a
 * chunk, ns in its loop, 0, 0}.  Returns the number of words (0 otherwise). */
int mpdp_debug_df_stats(const mpdp_ctx* ctx, unsigned long long* out, int cap);

/* Multi-GPU bootstrap: 128-byte NCCL unique id (call on rank 0 only). */
mpdp_status mpdp_nccl_get_unique_id(void* out128);

/* Contiguous share [lo, hi) of the `total` colex ranks of a level for `rank`
 * of `world`: equal segments of ceil(total/world) (the last ones may be short
 * or empty), so the sharded memo segments can be allgathered in place
 * (SURVEY §8(e)).  Pure host arithmetic, used by the sharded level loop and
 * exported so the multi-process host logic is testable on CPU. */
void mpdp_share(uint64_t total, int rank, int world, uint64_t* lo, uint64_t* hi);

#ifdef __cplusplus
}
#endif
#endif /* MPDP_H */
