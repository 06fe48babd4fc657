# final evidence of the committed code (after the gather-kernel TMA change)
set -x
OUT=gpurun_out/r02zzf
mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -3 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke.log
run() { local n=$1; shift; timeout 900 python bench.py "$@" > $OUT/bench_$n.json 2> $OUT/bench_$n.err; echo "$n rc=$?"; python -c "import json;d=json.loads(open('$OUT/bench_$n.json').read().strip().splitlines()[-1]);print('$n', d['value'], (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('frac'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('tensor_roofline') or {}).get('frac'))"; }
run tw --steps 20 --warmup 5
run tw_plan --schedule plan --steps 20 --warmup 5
run ref --impl reference --steps 5 --warmup 1
run lj --config lj --steps 5
run fm --config fm --steps 5
run friendster --config friendster --steps 5
run fb15k --config fb15k --steps 5 --warmup 3
run shared --negatives 1000 --shared-chunk 1000 --steps 10
run eval --eval 1000000
