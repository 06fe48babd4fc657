# shared-negative kernels after: -dst folded into prep, weights from one offset, unmasked full blocks
set -x
OUT=gpurun_out/r02s
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_shared.py tests/test_gpu_checked.py -q -m gpu -x > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
B="python bench.py --schedule plan --negatives 1000 --shared-chunk 1000 --no-cpu-baseline --no-e2e"
timeout 300 $B --steps 10 --warmup 3 > $OUT/bench.json 2>&1; echo "bench rc=$?"
python -c "import json;d=json.loads(open('$OUT/bench.json').read().strip().splitlines()[-1]);print('shared', d['value']/1e6, d['tensor_roofline']['frac'], d['roofline']['phase_ms'], d['clocks']['sm_mhz'])"
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"sg1_stats|sg2_mix|sg3_grad|shared_prep|shared_gather" -s 40 -c 5 --csv $B --steps 2 --warmup 3 > $OUT/ncu.csv 2> $OUT/ncu.err; echo "ncu rc=$?"
grep -E "sg1|sg2|sg3|prep|gather" $OUT/ncu.csv | cut -c1-300 | awk -F'","' '{print $5, $(NF-2), $NF}'
