set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -q -m gpu -x > gpurun_out/r02o_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02o_tests.log
for i in 1 2; do
timeout 300 python bench.py --schedule plan --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02o_plan$i.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/r02o_plan$i.json').read().strip().splitlines()[-1]);print('plan', d['value']/1e6, d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
