// heuristics.h — internal interface of the IDP2 / UnionDP drivers.
#pragma once
#include <string>

#include "mpdp.h"

namespace mpdp_heur {
constexpr int kMaxHeuristicN = MPDP_MAX_RELATIONS_HEURISTIC;
typedef mpdp_status (*InnerSolver)(void* user, const mpdp_query_graph* sub, mpdp_result* out);
// optional: `count` independent sub-problems in one call (UnionDP levels)
typedef mpdp_status (*InnerBatchSolver)(void* user, const mpdp_query_graph* subs, uint32_t count, mpdp_result* outs);
// t: UnionDP's partition threshold (0 = k)
mpdp_status run(const mpdp_query_graph* g, mpdp_algo algo, uint32_t k, InnerSolver solve, void* user,
                mpdp_result* out, std::string& err, InnerBatchSolver solve_batch = nullptr, uint32_t t = 0);
}  // namespace mpdp_heur
