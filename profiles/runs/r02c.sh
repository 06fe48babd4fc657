set -x
timeout 1200 python -m pytest tests -q -m gpu -x -k "k4 or shared or golden or fb15k or presort or transe" > gpurun_out/r02c_pytest.log 2>&1; echo "gpu tests rc=$?"
tail -15 gpurun_out/r02c_pytest.log
for k4 in 2 1; do
  LGD_K4=$k4 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02c_bench_k4_$k4.json 2> gpurun_out/r02c_bench_k4_$k4.err; echo "bench K4=$k4 rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/r02c_bench_k4_$k4.json').read().strip().splitlines()[-1]);print('K4=$k4', d['value']/1e6, d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['roofline']['phase_ms'], d['clocks'])"
done
LGD_K4=2 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02c_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02c_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
