set -x
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/r02d_pytest.log 2>&1; echo "gpu tests rc=$?"
tail -15 gpurun_out/r02d_pytest.log
for k4 in 2 1; do
  LGD_K4=$k4 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02d_bench_k4_$k4.json 2> gpurun_out/r02d_bench_k4_$k4.err; echo "bench K4=$k4 rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/r02d_bench_k4_$k4.json').read().strip().splitlines()[-1]);print('K4=$k4', d['value']/1e6, d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['roofline']['phase_ms'], d['clocks'])"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02d_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02d_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"segment_heads|score_kernel" -s 20 -c 2 -o gpurun_out/r02d_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02d_ncu_full.log 2>&1; echo "ncu full rc=$?"
