set -x
LGD_K4=4 timeout 1500 python -m pytest tests -q -m gpu -x -k "k4 or golden or fb15k or presort or transe or headline or rounds" > gpurun_out/r02i_pytest.log 2>&1; echo "gpu tests (K4=4) rc=$?"
tail -15 gpurun_out/r02i_pytest.log
for k4 in 4 2 4; do
LGD_K4=$k4 timeout 900 python bench.py --schedule plan --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02i_bench_$k4.json 2> gpurun_out/r02i_bench_$k4.err; echo "bench $k4 rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r02i_bench_$k4.json').read().strip().splitlines()[-1]);print('K4=$k4', d['value']/1e6, d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['roofline']['phase_ms'], d['clocks'])"
done
LGD_K4=4 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"segment_flat" -s 10 -c 1 -o gpurun_out/r02i_full python bench.py --schedule plan --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02i_ncu_full.log 2>&1; echo "ncu full rc=$?"
