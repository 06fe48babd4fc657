# K4 ring indexing by slot number + phase (32-bit mbarrier addresses): parity and plan lines
set -x
OUT=gpurun_out/r02zz3
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py tests/test_gpu_checked.py -q -m gpu -x > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/tests.log
for cfg in tw lj fm friendster tw; do
  timeout 600 python bench.py --config $cfg --schedule plan --steps 5 --no-cpu-baseline --no-e2e > $OUT/b_$cfg.json 2>/dev/null
  python -c "import json;d=json.loads(open('$OUT/b_$cfg.json').read().strip().splitlines()[-1]);print('$cfg', d['value']/1e6, d['roofline']['avg_launch_ms'], d['roofline']['phase_ms']['update'], d['clocks']['sm_mhz'])"
done
