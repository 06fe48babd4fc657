set -x
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/r02q_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02q_tests.log
for ovl in 1 0 1 0; do
  LGD_OVERLAP_PREP=$ovl timeout 300 python bench.py --schedule plan --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02q_plan_$ovl.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r02q_plan_$ovl.json').read().strip().splitlines()[-1]);print('plan ovl=$ovl', d['value']/1e6, d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
for ovl in 1 0; do
  LGD_OVERLAP_PREP=$ovl timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02q_rounds_$ovl.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r02q_rounds_$ovl.json').read().strip().splitlines()[-1]);print('rounds ovl=$ovl', d['value']/1e6, d['e2e']['value']/1e6, d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
timeout 300 python bench.py --eval 1000000 > gpurun_out/r02q_eval.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/r02q_eval.json').read().strip().splitlines()[-1]);print('eval', d['value']/1e6, d['roofline']['frac'])"
