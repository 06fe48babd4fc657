# K4 variants A/B on one box: segment_heads (default) vs staging-ring depth 2 / 4 and the
# flattened kernel with next-step prefetch; then an ncu capture of the flattened kernel
set -x
LGD_K4=4 timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "golden or k4_segment" > gpurun_out/r02m_flat.log 2>&1; echo "flat tests rc=$?"; tail -3 gpurun_out/r02m_flat.log
b() { timeout 300 python bench.py --schedule plan --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02m_$1.json 2> gpurun_out/r02m_$1.err; python -c "import json;d=json.loads(open('gpurun_out/r02m_$1.json').read().strip().splitlines()[-1]);print('$1', d['value']/1e6, d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'])"; }
for rep in 1 2; do
  unset LGD_LIBRARY LGD_K4; b heads$rep
  LGD_K4=4 b flat$rep
  LGD_LIBRARY=paper_2505_09258_b200/variants/liblegend_b200_d2.so b d2_$rep
  LGD_LIBRARY=paper_2505_09258_b200/variants/liblegend_b200_d4.so b d4_$rep
done
unset LGD_LIBRARY
LGD_K4=4 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"segment_flat" -s 10 -c 1 -o gpurun_out/r02m_flat python bench.py --schedule plan --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02m_ncu_flat.log 2>&1; echo "ncu flat rc=$?"
