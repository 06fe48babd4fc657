# TransE K4 with TMA bulk-copy staging (default now): parity and Friendster / TW lines
set -x
OUT=gpurun_out/r02zz2
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py tests/test_gpu_checked.py tests/test_gpu_rounds.py -q -m gpu -x > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/tests.log
for cfg in friendster tw; do
timeout 600 python bench.py --config $cfg --steps 5 > $OUT/bench_$cfg.json 2>/dev/null; echo "bench rc=$?"
python -c "import json;d=json.loads(open('$OUT/bench_$cfg.json').read().strip().splitlines()[-1]);print('$cfg', d['value']/1e6, d['e2e']['value']/1e6, d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
done
