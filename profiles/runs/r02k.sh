set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o gpurun_out/adagrad_probe profiles/micro/adagrad_probe.cu
timeout 300 gpurun_out/adagrad_probe 4294967296 0; echo "probe mode0 rc=$?"
timeout 300 gpurun_out/adagrad_probe 4294967296 1; echo "probe mode1 rc=$?"
