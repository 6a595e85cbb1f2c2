/*
 * oracle.h — CPU oracle for the MPDP exact join-order DP (arXiv 2202.13511).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load liboracle.so.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2202_13511_b200/csrc, include/mpdp.h) and never includes them.
 *
 * Everything is plain, single-threaded C99 in IEEE-754 double precision,
 * compiled with -ffp-contract=off (reading R6: no FMA contraction).
 * Sets are uint64_t bitmasks, bit v = relation v, n <= 28 for the optimisers
 * (direct 2^n memo arrays), n <= 64 for the primitives.
 *
 * Parity status per function is listed in oracle.c's header and DESIGN.md.
 */
#ifndef MPDP_ORACLE_H
#define MPDP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    uint32_t n;                 /* relations, 1..64 (optimisers: 1..28)        */
    const double* card;         /* [n] base cardinalities, >= 0 (R18)          */
    uint32_t n_edges;
    const uint32_t* edges;      /* [2*n_edges] pairs {u, v}, u < v             */
    const double* sel;          /* [n_edges] selectivities in (0, 1]           */
    const double* leaf_cost;    /* [n] or NULL (= 0 for base relations)        */
} oracle_graph;

typedef struct {
    int32_t left, right;        /* child node indices, -1 for leaves           */
    int32_t relation;           /* leaf: relation index, else -1               */
    uint64_t set;               /* relation bitmask                            */
    double card, cost;
} oracle_node;

typedef struct {
    oracle_node* nodes;         /* caller-owned, capacity >= 2n-1              */
    uint32_t capacity;
    uint32_t n_nodes;           /* 2n-1, post-order, root last                 */
    double cost;                /* cost of the root                            */
    uint64_t csg_count;         /* connected subsets incl. singletons (R1)     */
    uint64_t ccp_pairs;         /* unordered csg-cmp pairs (R2)                */
    uint64_t pairs_evaluated;   /* MPDP unordered block splits (R3)            */
    uint64_t* level_csg;        /* optional [n+1]: per subset size             */
    uint64_t* level_ccp;        /* optional [n+1]                              */
    uint64_t* level_pairs;      /* optional [n+1]                              */
    uint64_t dpsize_checks;     /* DPsize only: ordered memo-pair checks (R4)  */
} oracle_result;

/* status codes */
#define ORACLE_OK 0
#define ORACLE_ERR_ARG 1
#define ORACLE_ERR_DISCONNECTED 2
#define ORACLE_ERR_CAPACITY 3
#define ORACLE_ERR_OOM 5

/* ---- primitives (n <= 64) ------------------------------------------------ */
uint64_t oracle_neighbours(const oracle_graph* g, uint64_t S);
uint64_t oracle_grow(const oracle_graph* g, uint64_t source, uint64_t restriction);
int      oracle_connected(const oracle_graph* g, uint64_t S);
int      oracle_is_ccp(const oracle_graph* g, uint64_t S1, uint64_t S2);
double   oracle_card(const oracle_graph* g, uint64_t S);
/* blocks of G[S]; writes up to max_blocks masks, returns the block count */
int      oracle_blocks(const oracle_graph* g, uint64_t S, uint64_t* blocks, int max_blocks);
/* MPDP evaluated join pairs for one connected set: sum over blocks (2^(b-1)-1) */
uint64_t oracle_mpdp_pairs(const oracle_graph* g, uint64_t S);
/* colex unrank of the r-th k-subset of {0..n-1} */
uint64_t oracle_unrank_colex(uint32_t n, uint32_t k, uint64_t r);

/* ---- optimisers (n <= 28) ------------------------------------------------ */
/* O0: the plain definition (DPsub over unordered CCP splits), n <= 20         */
int oracle_optimize_definition(const oracle_graph* g, oracle_result* out);
/* O1: DPccp (Moerkotte-Neumann enumeration), n <= 28                          */
int oracle_optimize_dpccp(const oracle_graph* g, oracle_result* out);
/* O2: DPsize over connected sets, n <= 16                                     */
int oracle_optimize_dpsize(const oracle_graph* g, oracle_result* out);
/* O3: brute force over every ordered-children CP-free bushy tree, n <= 7     */
int oracle_bruteforce(const oracle_graph* g, double* min_cost, uint64_t* n_trees);
/* O4: counters by definition (csg by scanning all 2^n subsets; MPDP pairs)   */
int oracle_counters(const oracle_graph* g, uint64_t* level_csg, uint64_t* level_pairs);

#ifdef __cplusplus
}
#endif
#endif
