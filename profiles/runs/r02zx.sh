# K3 row loads: per-lane TMA bulk copies (default) vs warp-wide 16-byte cp.async (SCORE_CPA)
set -x
OUT=gpurun_out/r02zx
mkdir -p $OUT
LGD_LIBRARY=paper_2505_09258_b200/var_cpa/liblegend_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "wide or golden or epoch" > $OUT/tests_cpa.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/tests_cpa.log
for cfg in tw lj friendster; do
for v in base cpa base cpa; do
  if [ $v = base ]; then unset LGD_LIBRARY; else export LGD_LIBRARY=paper_2505_09258_b200/var_$v/liblegend_b200.so; fi
  timeout 600 python bench.py --config $cfg --schedule plan --steps 5 --no-cpu-baseline --no-e2e > $OUT/b_${cfg}_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('$OUT/b_${cfg}_$v.json').read().strip().splitlines()[-1]);print('$cfg $v', d['value']/1e6, d['roofline']['phase_ms']['score'], d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
done
done
