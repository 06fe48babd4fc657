set -x
timeout 300 gpurun_out/adagrad_probe 4294967296 0; echo "probe mode0 rc=$?"
timeout 300 gpurun_out/adagrad_probe 4294967296 1; echo "probe mode1 rc=$?"
LGD_K4=4 timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "golden or k4_segment" > gpurun_out/r02j_flat.log 2>&1; echo "flat tests rc=$?"; tail -12 gpurun_out/r02j_flat.log
LGD_K4=4 LGD_LIBRARY=paper_2505_09258_b200/liblegend_b200_checked.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "k4_segment" > gpurun_out/r02j_flat_checked.log 2>&1; echo "flat checked rc=$?"; tail -12 gpurun_out/r02j_flat_checked.log
LGD_LIBRARY=paper_2505_09258_b200/variants/liblegend_b200_a1.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "golden or k4_segment or fb15k" > gpurun_out/r02j_a1.log 2>&1; echo "a1 tests rc=$?"; tail -5 gpurun_out/r02j_a1.log
for v in base a1 base a1; do
  if [ $v = a1 ]; then export LGD_LIBRARY=paper_2505_09258_b200/variants/liblegend_b200_a1.so; else unset LGD_LIBRARY; fi
  timeout 300 python bench.py --schedule plan --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02j_bench_$v.json 2> gpurun_out/r02j_bench_$v.err; echo "bench $v rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/r02j_bench_$v.json').read().strip().splitlines()[-1]);print('$v', d['value']/1e6, d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['clocks'])"
done
unset LGD_LIBRARY
LGD_K4=4 timeout 200 python bench.py --schedule plan --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02j_bench_flat.json 2> gpurun_out/r02j_bench_flat.err; echo "bench flat rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r02j_bench_flat.json').read().strip().splitlines()[-1]);print('flat', d['value']/1e6, d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['clocks'])"
