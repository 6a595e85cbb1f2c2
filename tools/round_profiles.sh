#!/bin/bash
# Round evidence on one B200 (run under gpurun from the repo root):
#   launch lists, DRAM traffic + warp instructions per config, ncu --set full
#   of the whole-query kernels, bench_all, ablations, config-5 heuristics, one
#   default bench.py line.  Usage: tools/round_profiles.sh r02
set -u
TAG=${1:-r02}
O=gpurun_out/rp                      # merged back by gpurun; copy into profiles/ afterwards
mkdir -p $O
for cfg in star-10 snowflake-20 star-25 clique-18; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/${TAG}_launches_${cfg}.csv python tools/profile_one.py $cfg 1 > /dev/null 2>&1
done
TRAFFIC_DIR=$O timeout 900 python tools/traffic.py $TAG star-25 clique-18 star-10 snowflake-20 chain-20 cycle-20 chain-25 random-20 > $O/traffic.log 2>&1
cp $O/traffic.json profiles/traffic.json
timeout 400 ncu --set full --import-source on --clock-control none -k regex:k_dp_ -s 1 -c 1 \
  -o /tmp/prof_${TAG}_star-25 -f python tools/profile_one.py star-25 1 > gpurun_out/ncu_star.log 2>&1
timeout 400 ncu --set full --import-source on --clock-control none -k regex:k_dp_ -s 1 -c 1 \
  -o /tmp/prof_${TAG}_clique-18 -f python tools/profile_one.py clique-18 1 > gpurun_out/ncu_clique.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dp_fused -s 1 -c 1 \
  -o /tmp/prof_${TAG}_random-20 -f python tools/profile_one.py random-20 1 > gpurun_out/ncu_random.log 2>&1
# summaries on the box (the .ncu-rep files stay in /tmp: gpurun_out is capped at 64 MiB)
for c in star-25 clique-18 random-20; do
  (python tools/ncu_summary.py /tmp/prof_${TAG}_$c.ncu-rep 30; python tools/ncu_lines.py /tmp/prof_${TAG}_$c.ncu-rep 40) \
    > $O/${TAG}_ncu_$c.txt 2>&1
done
timeout 300 python tools/bench_all.py 10 > $O/${TAG}_bench_all.txt 2>&1
timeout 600 python tools/ablation.py 5 star-20 star-25 snowflake-20 clique-16 clique-18 cycle-16 random-18 > $O/${TAG}_ablation.txt 2>&1
MPDP_DEBUG_HEUR_TIME=1 timeout 300 python tools/heuristic_run.py 1000 25 2 > $O/${TAG}_config5_heuristics.txt 2>&1
MPDP_DEBUG_DF_STATS=1 timeout 120 python tools/df_stats.py star-25 > $O/${TAG}_df_stats_star-25.txt 2>&1
timeout 300 python tools/time_cfg.py star-25 star-20 --seeds 3 --reps 10 > $O/${TAG}_level_spans.txt 2>&1
timeout 300 python tools/general_compare.py random-16 random-18 random-20 cycle-20 > $O/${TAG}_general_compare.txt 2>&1
timeout 300 python tools/xr_time.py star-20 star-25 > $O/${TAG}_xr_emulated.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > $O/${TAG}_bench_star25.json 2> gpurun_out/bench.err
tail -1 $O/${TAG}_bench_star25.json
cat $O/${TAG}_bench_all.txt
