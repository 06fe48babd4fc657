# K4 register budget between the block-count steps: 128-thread blocks at 64 / 72 / 80 registers (__maxnreg__)
set -x
OUT=gpurun_out/r02zzg
mkdir -p $OUT
for cfg in tw lj fm; do
for v in base r64 r72 r80 base r72; do
  if [ $v = base ]; then unset LGD_LIBRARY; else export LGD_LIBRARY=paper_2505_09258_b200/var_$v/liblegend_b200.so; fi
  timeout 600 python bench.py --config $cfg --schedule plan --steps 5 --no-cpu-baseline --no-e2e > $OUT/b_${cfg}_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('$OUT/b_${cfg}_$v.json').read().strip().splitlines()[-1]);print('$cfg $v', d['value']/1e6, d['roofline']['avg_launch_ms'], d['roofline']['phase_ms']['update'], d['clocks']['sm_mhz'])"
done
done
