set -x
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r02h_pytest.log 2>&1; echo "gpu tests rc=$?"
tail -15 gpurun_out/r02h_pytest.log
for k4 in 3 2; do
LGD_K4=$k4 timeout 900 python bench.py --schedule plan --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02h_bench_$k4.json 2> gpurun_out/r02h_bench_$k4.err; echo "bench $k4 rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r02h_bench_$k4.json').read().strip().splitlines()[-1]);print('K4=$k4', d['value']/1e6, d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['roofline']['phase_ms'], d['clocks'])"
done
timeout 900 python bench.py --eval 1000000 > gpurun_out/r02h_eval.json 2> gpurun_out/r02h_eval.err; echo "eval rc=$?"; tail -c 1500 gpurun_out/r02h_eval.json
timeout 1200 python bench.py --schedule plan --steps 256 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02h_epoch_plan.json 2> gpurun_out/r02h_epoch_plan.err; echo "epoch plan rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r02h_epoch_plan.json').read().strip().splitlines()[-1]);print('epoch plan', d['value']/1e6, d['ms_per_step'], d['roofline']['frac'], d['clocks'])"
timeout 1200 python bench.py --steps 15 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02h_epoch_rounds.json 2> gpurun_out/r02h_epoch_rounds.err; echo "epoch rounds rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r02h_epoch_rounds.json').read().strip().splitlines()[-1]);print('epoch rounds', d['value']/1e6, d['ms_per_step'], d['roofline']['frac'], d['clocks'])"
