#!/bin/bash
# Profile capture for the judged numbers (run on the GPU box through gpurun):
#   bash profiles/capture.sh
# 1. the plain command (must exit 0 before ncu touches it),
# 2. the launch list: every kernel of that command with its device time
#    (cold-cache, serialised: compare shares, not absolutes),
# 3. one `ncu --set full` capture of the two dominant kernels (K3 score and
#    K4 segment pass 1) in the steady state.
# Outputs land in gpurun_out/; profiles/summarize.py turns them into the
# committed JSON summaries.
set -u
OUT=gpurun_out
mkdir -p $OUT
CFG=${CFG:-tw}
B="python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 $B > $OUT/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches.csv $B > $OUT/ncu_launch.log 2>&1 || echo "launch list failed"
timeout 900 $B > $OUT/plain2.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"score_kernel|segment_pass1" -s 40 -c 4 -o $OUT/prof_full $B > $OUT/ncu_full.log 2>&1 \
  || echo "full capture failed"
