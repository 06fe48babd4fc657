# full GPU tests + shared-negative bench after the SG1 fold / SG2 / SG3 tail work
set -x
OUT=gpurun_out/r02zd
mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/pytest_gpu.log
B="python bench.py --schedule plan --negatives 1000 --shared-chunk 1000"
timeout 600 $B --steps 10 --warmup 3 > $OUT/bench_shared.json 2> $OUT/bench_shared.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('$OUT/bench_shared.json').read().strip().splitlines()[-1]);print('shared', d['value']/1e6, d['e2e']['value']/1e6, d['tensor_roofline']['frac'], d['clocks'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sg2_mix|sg3_grad" -s 20 -c 2 -o $OUT/shared_full $B --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_full.log 2>&1; echo "ncu rc=$?"
ncu -i $OUT/shared_full.ncu-rep --page raw --csv > $OUT/raw.csv 2>/dev/null
rm -f $OUT/shared_full.ncu-rep
