# shared-negative prep kernel with TMA bulk row copies
set -x
OUT=gpurun_out/r02zza
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_shared.py tests/test_gpu_checked.py -q -m gpu -x > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/tests.log
B="python bench.py --schedule plan --negatives 1000 --shared-chunk 1000 --no-cpu-baseline --no-e2e"
timeout 300 $B --steps 10 --warmup 3 > $OUT/bench.json 2>&1; echo "bench rc=$?"
python -c "import json;d=json.loads(open('$OUT/bench.json').read().strip().splitlines()[-1]);print('shared', d['value']/1e6, d['tensor_roofline']['frac'], d['roofline']['phase_ms']['score'], d['clocks']['sm_mhz'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"shared_prep|shared_gather|sg2|sg3" -s 20 -c 4 --csv $B --steps 2 --warmup 3 > $OUT/ncu.csv 2> $OUT/ncu.err; echo "ncu rc=$?"
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/r02zza/ncu.csv')))
hdr=None
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); print(d['Kernel Name'][:30], d['Metric Name'], d['Metric Value'])
PY
