set -x
timeout 600 python -m pytest tests -q -m gpu -x -k "evaluate or eval or adapter or checked" > gpurun_out/r02p_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02p_tests.log
timeout 300 python bench.py --eval 1000000 > gpurun_out/r02p_eval.json 2>/dev/null; tail -c 400 gpurun_out/r02p_eval.json
timeout 300 python bench.py --eval 1000000 --config friendster > gpurun_out/r02p_eval_friendster.json 2>/dev/null; tail -c 300 gpurun_out/r02p_eval_friendster.json
