set -x
timeout 300 python bench.py --schedule plan --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02n_plan.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/r02n_plan.json').read().strip().splitlines()[-1]);print('plan', d['value']/1e6, d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
timeout 300 python bench.py --eval 200000 > gpurun_out/r02n_eval.json 2>/dev/null; tail -c 300 gpurun_out/r02n_eval.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"eval_" -c 2 -o gpurun_out/r02n_eval python bench.py --eval 200000 > gpurun_out/r02n_ncu_eval.log 2>&1; echo "ncu eval rc=$?"
