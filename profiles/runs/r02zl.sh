# per-model K4 ring depth (3 for Dot / ComplEx): parity and LJ / FM bench lines
set -x
OUT=gpurun_out/r02zl
mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/pytest_gpu.log
for cfg in lj fm tw; do
timeout 600 python bench.py --config $cfg --steps 5 > $OUT/bench_$cfg.json 2>/dev/null; echo "bench rc=$?"
python -c "import json;d=json.loads(open('$OUT/bench_$cfg.json').read().strip().splitlines()[-1]);print('$cfg', d['value']/1e6, d['e2e']['value']/1e6, d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
done
