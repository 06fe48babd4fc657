set -x
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_headline.py -x -q -m gpu > gpurun_out/r02a_pytest_new.log 2>&1; echo "new tests rc=$?"
tail -5 gpurun_out/r02a_pytest_new.log
timeout 600 python -m pytest tests -q -m gpu -k "evaluate or epoch_matches_golden or fb15k" > gpurun_out/r02a_pytest_eval.log 2>&1; echo "eval tests rc=$?"
tail -5 gpurun_out/r02a_pytest_eval.log
timeout 120 python profiles/sanitize_workload.py exact > gpurun_out/san_plain.txt 2>&1; echo "plain rc=$?"
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python profiles/sanitize_workload.py exact > gpurun_out/san_${tool}_exact.txt 2>&1; echo "$tool exact rc=$?"
  tail -3 gpurun_out/san_${tool}_exact.txt
done
for tool in memcheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python profiles/sanitize_workload.py shared > gpurun_out/san_${tool}_shared.txt 2>&1; echo "$tool shared rc=$?"
  tail -3 gpurun_out/san_${tool}_shared.txt
done
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r02a_bench.json
