#!/bin/bash
# Round evidence on one B200 (run under gpurun from the repo root):
#   launch lists, DRAM traffic per config, ncu --set full of the whole-query
#   kernels, bench_all, and one default bench.py line.  Usage: tools/round_profiles.sh r01
set -u
TAG=${1:-r01}
O=gpurun_out/rp                      # merged back by gpurun; copy into profiles/ afterwards
mkdir -p $O
for cfg in star-10 snowflake-20 star-25 clique-18; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/${TAG}_launches_${cfg}.csv python tools/profile_one.py $cfg 1 > /dev/null 2>&1
done
TRAFFIC_DIR=$O timeout 900 python tools/traffic.py $TAG star-10 snowflake-20 star-25 clique-18 chain-25 > $O/traffic.log 2>&1
timeout 400 ncu --set full --import-source on --clock-control none -k regex:k_dp_ -s 1 -c 1 \
  -o gpurun_out/prof_${TAG}_star-25 -f python tools/profile_one.py star-25 1 > gpurun_out/ncu_star.log 2>&1
timeout 400 ncu --set full --import-source on --clock-control none -k regex:k_dp_ -s 1 -c 1 \
  -o gpurun_out/prof_${TAG}_clique-18 -f python tools/profile_one.py clique-18 1 > gpurun_out/ncu_clique.log 2>&1
timeout 300 python tools/bench_all.py 10 > $O/${TAG}_bench_all.txt 2>&1
timeout 300 python bench.py > $O/${TAG}_bench_star25.json 2> gpurun_out/bench.err
tail -1 $O/${TAG}_bench_star25.json
cat $O/${TAG}_bench_all.txt
