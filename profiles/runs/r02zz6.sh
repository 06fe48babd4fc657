# warp-specialised K4 with TMA-bulk producers (LGD_K4=3; 4 / 2 / 1 producer warps per 8 consumers) vs segment_heads
set -x
OUT=gpurun_out/r02zz6
mkdir -p $OUT
LGD_K4=3 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "wide or golden or epoch or hubs" > $OUT/tests_ws.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/tests_ws.log
LGD_K4=3 LGD_LIBRARY=paper_2505_09258_b200/var_ws1/liblegend_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "wide or hubs" > $OUT/tests_ws1.log 2>&1; echo "tests ws1 rc=$?"; tail -2 $OUT/tests_ws1.log
for cfg in tw lj; do
for v in heads ws4 ws2 ws1 heads ws4 ws2 ws1; do
  unset LGD_LIBRARY; unset LGD_K4
  case $v in
    ws4) export LGD_K4=3 ;;
    ws2) export LGD_K4=3 LGD_LIBRARY=paper_2505_09258_b200/var_ws2/liblegend_b200.so ;;
    ws1) export LGD_K4=3 LGD_LIBRARY=paper_2505_09258_b200/var_ws1/liblegend_b200.so ;;
  esac
  timeout 600 python bench.py --config $cfg --schedule plan --steps 5 --no-cpu-baseline --no-e2e > $OUT/b_${cfg}_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('$OUT/b_${cfg}_$v.json').read().strip().splitlines()[-1]);print('$cfg $v', d['value']/1e6, d['roofline']['avg_launch_ms'], d['roofline']['phase_ms']['update'], d['clocks']['sm_mhz'])"
done
done
