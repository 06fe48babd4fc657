# K4 theta / state rows by bulk copies, operand by cp.async (hybrid, default build) vs all cp.async (rows0)
set -x
OUT=gpurun_out/r02zz5
mkdir -p $OUT
for cfg in tw lj fm; do
for v in base rows0 base rows0; do
  if [ $v = base ]; then unset LGD_LIBRARY; else export LGD_LIBRARY=paper_2505_09258_b200/var_$v/liblegend_b200.so; fi
  timeout 600 python bench.py --config $cfg --schedule plan --steps 5 --no-cpu-baseline --no-e2e > $OUT/b_${cfg}_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('$OUT/b_${cfg}_$v.json').read().strip().splitlines()[-1]);print('$cfg $v', d['value']/1e6, d['roofline']['avg_launch_ms'], d['roofline']['phase_ms']['update'], d['clocks']['sm_mhz'])"
done
done
