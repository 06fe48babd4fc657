# K4: FP64 relation rows in shared memory at a fixed address (template variant) vs through L1
set -x
OUT=gpurun_out/r02zu
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py tests/test_gpu_checked.py -q -m gpu -x > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/tests.log
for cfg in tw friendster; do
for v in 1 0 1 0; do
  LGD_K4_RELSMEM=$v timeout 600 python bench.py --config $cfg --schedule plan --steps 5 --no-cpu-baseline --no-e2e > $OUT/b_${cfg}_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('$OUT/b_${cfg}_$v.json').read().strip().splitlines()[-1]);print('$cfg relsmem=$v', d['value']/1e6, d['roofline']['avg_launch_ms'], d['roofline']['phase_ms']['update'], d['clocks']['sm_mhz'])"
done
done
