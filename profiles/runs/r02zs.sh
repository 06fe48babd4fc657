# one-rank NCCL communicators (run-time libnccl, init / split / allgather, IPC handles) vs the local runner
set -x
OUT=gpurun_out/r02zs
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_rounds.py -q -m gpu -x -rA > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -12 $OUT/tests.log
