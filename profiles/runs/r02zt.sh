# full epochs of the round schedule for every BASELINE config (steps = rounds per epoch)
set -x
OUT=gpurun_out/r02zt
mkdir -p $OUT
run() { local n=$1; shift; timeout 1500 python bench.py "$@" --no-cpu-baseline --no-e2e > $OUT/epoch_$n.json 2> $OUT/epoch_$n.err; echo "$n rc=$?"; python -c "import json;d=json.loads(open('$OUT/epoch_$n.json').read().strip().splitlines()[-1]);print('$n', d['value']/1e6, d['steps'], d['ms_per_step'], d['config'].get('edges_per_rank'), d['roofline']['frac'], d['clocks'])"; }
run tw --steps 15 --warmup 3
run lj --config lj --steps 7 --warmup 3
run fm --config fm --steps 31 --warmup 3
run friendster --config friendster --steps 31 --warmup 3
