# persistent SG3 vs one CTA per item (LGD_SG3_CLASSIC=1)
set -x
OUT=gpurun_out/r02zo
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_shared.py tests/test_gpu_checked.py -q -m gpu -x > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
B="python bench.py --schedule plan --negatives 1000 --shared-chunk 1000 --no-cpu-baseline --no-e2e"
for v in 0 1 0 1; do
LGD_SG3_CLASSIC=$v timeout 300 $B --steps 10 --warmup 3 > $OUT/bench_$v.json 2>&1; echo "bench rc=$?"
python -c "import json;d=json.loads(open('$OUT/bench_$v.json').read().strip().splitlines()[-1]);print('shared classic=$v', d['value']/1e6, d['tensor_roofline']['frac'], d['roofline']['phase_ms']['score'], d['clocks']['sm_mhz'])"
done
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"sg3" -s 4 -c 2 --csv $B --steps 2 --warmup 3 > $OUT/ncu.csv 2> $OUT/ncu.err; echo "ncu rc=$?"
grep -E "sg3" $OUT/ncu.csv | cut -c1-250
