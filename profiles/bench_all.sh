#!/bin/bash
# Every config's bench line for a profile snapshot (run on the GPU box through
# gpurun): bash profiles/bench_all.sh; outputs gpurun_out/bench_<name>.json.
set -u
OUT=gpurun_out
mkdir -p $OUT
run() {  # name, args...
  local n=$1; shift
  timeout 900 python bench.py "$@" > $OUT/bench_$n.json 2> $OUT/bench_$n.err
  echo "$n rc=$? $(head -c 160 $OUT/bench_$n.json)"
}
run tw
run ref --impl reference
run lj --config lj --steps 5
run fm --config fm --steps 5
run friendster --config friendster --steps 5
run fb15k --config fb15k --steps 5
run shared --negatives 1000 --shared-chunk 1000 --steps 10
run rounds --schedule rounds --steps 3
