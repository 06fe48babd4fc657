# K3 with 4-warp blocks (finer occupancy granularity at d = 128) vs 8-warp blocks
set -x
OUT=gpurun_out/r02zg
mkdir -p $OUT
for cfg in friendster tw lj; do
for v in base var4 base var4; do
  if [ $v = var4 ]; then export LGD_LIBRARY=paper_2505_09258_b200/var4/liblegend_b200.so; else unset LGD_LIBRARY; fi
  timeout 600 python bench.py --config $cfg --schedule plan --steps 5 --no-cpu-baseline --no-e2e > $OUT/b_${cfg}_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('$OUT/b_${cfg}_$v.json').read().strip().splitlines()[-1]);print('$cfg $v', d['value']/1e6, d['roofline']['phase_ms']['score'], d['clocks']['sm_mhz'])"
done
done
