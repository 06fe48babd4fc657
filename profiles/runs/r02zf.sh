# TransE K3: 16-byte shared loads in the score dots; the online-softmax rescale test
set -x
OUT=gpurun_out/r02zf
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py tests/test_gpu_shared.py tests/test_gpu_checked.py -q -m gpu -x -k "transe or friendster or rescale or checked" > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
for i in 1 2; do
timeout 600 python bench.py --config friendster --steps 5 --no-cpu-baseline --no-e2e > $OUT/bench_friendster_$i.json 2>/dev/null; echo "bench rc=$?"
python -c "import json;d=json.loads(open('$OUT/bench_friendster_$i.json').read().strip().splitlines()[-1]);print('friendster', d['value']/1e6, d['roofline']['frac'], d['roofline']['phase_ms'], d['clocks']['sm_mhz'])"
done
