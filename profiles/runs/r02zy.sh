# K4 staging: cp.async pieces per lane (default) vs TMA bulk copies per row issued by one lane (K4_BULK)
set -x
OUT=gpurun_out/r02zy
mkdir -p $OUT
LGD_LIBRARY=paper_2505_09258_b200/var_bulk/liblegend_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "wide or golden or epoch or hubs" > $OUT/tests_bulk.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/tests_bulk.log
for cfg in tw lj fm friendster; do
for v in base bulk base bulk; do
  if [ $v = base ]; then unset LGD_LIBRARY; else export LGD_LIBRARY=paper_2505_09258_b200/var_$v/liblegend_b200.so; fi
  timeout 600 python bench.py --config $cfg --schedule plan --steps 5 --no-cpu-baseline --no-e2e > $OUT/b_${cfg}_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('$OUT/b_${cfg}_$v.json').read().strip().splitlines()[-1]);print('$cfg $v', d['value']/1e6, d['roofline']['avg_launch_ms'], d['roofline']['phase_ms']['update'], d['clocks']['sm_mhz'])"
done
done
