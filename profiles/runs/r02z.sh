# one full ncu capture of SG2 (source-level stalls of the tail)
set -x
OUT=gpurun_out/r02z
mkdir -p $OUT
B="python bench.py --schedule plan --negatives 1000 --shared-chunk 1000 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sg2_mix" -s 10 -c 1 -o $OUT/sg2 $B > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
