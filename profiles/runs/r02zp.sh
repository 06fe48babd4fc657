# K4 segment_heads (TW DistMult): per-instruction executed counts and stalls (SASS source page)
set -x
OUT=gpurun_out/r02zp
mkdir -p $OUT
B="python bench.py --schedule plan --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"segment_heads" -s 8 -c 1 -o /tmp/k4 $B > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/k4.ncu-rep --page source --csv --print-source sass > $OUT/k4_source.csv 2>/dev/null
ncu -i /tmp/k4.ncu-rep --page source --csv --print-source cuda,sass > $OUT/k4_source_cuda.csv 2>/dev/null
ls -la $OUT
