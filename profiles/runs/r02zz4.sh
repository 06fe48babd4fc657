# K6 evaluate: candidate rows by TMA bulk copies (default now) vs 16-byte cp.async pieces
set -x
OUT=gpurun_out/r02zz4
mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -x -k "evaluate or eval or adapter or checked" > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/tests.log
for v in base evc base evc; do
  if [ $v = base ]; then unset LGD_LIBRARY; else export LGD_LIBRARY=paper_2505_09258_b200/var_$v/liblegend_b200.so; fi
  timeout 300 python bench.py --eval 1000000 > $OUT/eval_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('$OUT/eval_$v.json').read().strip().splitlines()[-1]);print('eval $v', d['value']/1e6, d['roofline']['frac'], d['mrr'], d['device_s'])"
done
unset LGD_LIBRARY
timeout 300 python bench.py --eval 1000000 --config friendster > $OUT/eval_friendster.json 2>/dev/null
python -c "import json;d=json.loads(open('$OUT/eval_friendster.json').read().strip().splitlines()[-1]);print('eval friendster', d['value']/1e6, d['roofline']['frac'], d['mrr'])"
