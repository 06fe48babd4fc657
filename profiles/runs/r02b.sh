set -x
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/r02b_pytest.log 2>&1; echo "gpu tests rc=$?"
tail -15 gpurun_out/r02b_pytest.log
for k4 in 2 1 2 1; do
  LGD_K4=$k4 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02b_bench_k4_$k4.json 2> gpurun_out/r02b_bench_k4_$k4.err; echo "bench K4=$k4 rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/r02b_bench_k4_$k4.json').read().strip().splitlines()[-1]);print('K4=$k4', d['value']/1e6, d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['roofline']['phase_ms'], d['clocks'])"
done
