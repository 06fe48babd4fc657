set -x
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r02f_pytest.log 2>&1; echo "gpu tests rc=$?"
tail -30 gpurun_out/r02f_pytest.log
timeout 900 python bench.py --schedule plan --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02f_bench_plan.json 2> gpurun_out/r02f_bench_plan.err; echo "bench plan rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r02f_bench_plan.json').read().strip().splitlines()[-1]);print('plan', d['value']/1e6, d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['roofline']['phase_ms'], d['clocks'])"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"segment_heads" -s 10 -c 1 -o gpurun_out/r02f_full python bench.py --schedule plan --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02f_ncu_full.log 2>&1; echo "ncu full rc=$?"
