"""Optimise one query and compare with the oracle: python tools/one_query.py star-11 [seed] [flags]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workload as W  # noqa: E402
from oracle import pyoracle as O  # noqa: E402
from paper_2202_13511_b200 import mpdp  # noqa: E402

name = sys.argv[1]
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
flags = int(sys.argv[3]) if len(sys.argv) > 3 else 0
topo, n = name.rsplit("-", 1)
g = W.generate(topo, int(n), seed)
with mpdp.Context(device=0, workspace_bytes=1 << 30, flags=flags) as ctx:
    r = ctx.mpdp_optimize(g)
o = O.optimize(g)
print(name, "gpu", r.cost, "oracle", o.cost, "tree_equal", r.tree() == O.tree_of(o.nodes))
