# TransE K3 in 4-warp blocks
set -x
OUT=gpurun_out/r02zm
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py tests/test_gpu_checked.py -q -m gpu -x -k "transe or friendster or checked" > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/tests.log
for i in 1 2; do
timeout 600 python bench.py --config friendster --steps 5 > $OUT/bench_friendster_$i.json 2>/dev/null; echo "bench rc=$?"
python -c "import json;d=json.loads(open('$OUT/bench_friendster_$i.json').read().strip().splitlines()[-1]);print('friendster', d['value']/1e6, d['e2e']['value']/1e6, d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
done
