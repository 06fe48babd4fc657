# shared-negative tcgen05 kernels: one full ncu capture of SG1 / SG2 / SG3 (TW, C = k = 1000)
set -x
OUT=gpurun_out/r02r
mkdir -p $OUT
B="python bench.py --schedule plan --negatives 1000 --shared-chunk 1000 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $B > $OUT/plain.json 2>&1; echo "plain rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"sg1_stats|sg2_mix|sg3_grad|shared_prep|shared_gather" -s 40 -c 5 -o $OUT/shared $B > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i $OUT/shared.ncu-rep --page raw --csv > $OUT/raw.csv 2>/dev/null
python - <<'PY'
import csv, json, re
rows = list(csv.reader(open("gpurun_out/r02r/raw.csv")))
hdr = rows[0]
want = re.compile(r"gpu__time_duration.sum|sm__pipe_tensor.*pct_of_peak_sustained_active|lts__throughput.avg.pct|l1tex__throughput.avg.pct|dram__throughput.avg.pct|smsp__issue_active.avg.pct|sm__warps_active.avg.pct|smsp__average_warp_latency_issue_stalled_.*ratio|smsp__average_warps_issue_stalled_.*per_issue_active.ratio|lts__t_bytes.sum$|l1tex__m_xbar2l1tex_read_bytes.sum$|sm__pipe_shared_cycles_active|smsp__inst_executed.sum$|sm__inst_executed_pipe_xu|Kernel Name")
out = []
for r in rows[2:]:
    d = {h: v for h, v in zip(hdr, r) if want.search(h)}
    out.append(d)
json.dump(out, open("gpurun_out/r02r/summary.json", "w"), indent=1)
for d in out:
    print(d.get("Kernel Name", "")[:40], d.get("gpu__time_duration.sum"))
PY
