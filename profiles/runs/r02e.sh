set -x
timeout 1200 python -m pytest tests/test_gpu_rounds.py tests/test_gpu_checked.py -q -m gpu > gpurun_out/r02e_pytest.log 2>&1; echo "gpu tests rc=$?"
tail -30 gpurun_out/r02e_pytest.log
timeout 900 python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/r02e_bench_rounds.json 2> gpurun_out/r02e_bench_rounds.err; echo "bench rounds rc=$?"
tail -c 2500 gpurun_out/r02e_bench_rounds.json; tail -5 gpurun_out/r02e_bench_rounds.err
timeout 900 python bench.py --schedule plan --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02e_bench_plan.json 2> gpurun_out/r02e_bench_plan.err; echo "bench plan rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r02e_bench_plan.json').read().strip().splitlines()[-1]);print('plan', d['value']/1e6, d['e2e'], d['roofline']['frac'])"
