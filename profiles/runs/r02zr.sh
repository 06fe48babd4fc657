# sanity after reverting the relation-rows-in-shared-memory experiment: TW plan and rounds
set -x
OUT=gpurun_out/r02zr
mkdir -p $OUT
timeout 600 python bench.py --schedule plan --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/tw_plan.json 2>/dev/null
python -c "import json;d=json.loads(open('$OUT/tw_plan.json').read().strip().splitlines()[-1]);print('tw plan', d['value']/1e6, d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/tw.json 2>/dev/null
python -c "import json;d=json.loads(open('$OUT/tw.json').read().strip().splitlines()[-1]);print('tw rounds', d['value']/1e6, d['e2e']['value']/1e6, d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
