# shared-negative kernels: two MMA-issuing warps per CTA
set -x
OUT=gpurun_out/r02w
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_shared.py tests/test_gpu_checked.py -q -m gpu -x > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
LGD_LIBRARY=paper_2505_09258_b200/trace/liblegend_b200.so timeout 300 python profiles/micro/trace_sg.py > $OUT/trace.txt 2>&1; echo "trace rc=$?"
B="python bench.py --schedule plan --negatives 1000 --shared-chunk 1000 --no-cpu-baseline --no-e2e"
timeout 300 $B --steps 10 --warmup 3 > $OUT/bench.json 2>&1; echo "bench rc=$?"
python -c "import json;d=json.loads(open('$OUT/bench.json').read().strip().splitlines()[-1]);print('shared', d['value']/1e6, d['tensor_roofline']['frac'], d['roofline']['phase_ms'], d['clocks']['sm_mhz'])"
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"sg2_mix|sg3_grad|shared_prep|shared_gather" -s 40 -c 5 --csv $B --steps 2 --warmup 3 > $OUT/ncu.csv 2> $OUT/ncu.err; echo "ncu rc=$?"
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/r02w/ncu.csv')))
hdr=None
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); print(d['Kernel Name'][:30], d['Metric Name'], d['Metric Value'])
PY
