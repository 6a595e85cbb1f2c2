import sys, os
sys.path.insert(0, 'os.path.dirname(os.path.dirname(os.path.abspath(__file__)))'); sys.path.insert(0, 'os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests")')
import workload as W
from oracle import pyoracle as O
from test_heuristics_cpu import run, recompute
for seed in range(4):
    g = W.snowflake(22, seed)
    ex = O.optimize_dpccp(g).cost
    goo,_ = run(g, "IDP2_MPDP", 2)
    idp,_ = run(g, "IDP2_MPDP", 8)
    uni,subs = run(g, "UNIONDP_MPDP", 8)
    print(f"seed {seed}: exact {ex:.4g}  GOO {goo.cost/ex:.3f}  IDP2(8) {idp.cost/ex:.3f}  UnionDP(8) {uni.cost/ex:.3f}  parts {[q.n for q in subs]}")
