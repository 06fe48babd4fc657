# final round-2 evidence: GPU tests, smoke, every config's bench line, the
# reference arm, launch list and full ncu captures per config.  ncu reports are
# reduced to CSV pages / JSON summaries on the box (gpurun copies back <= 64 MiB).
set -x
OUT=gpurun_out/r02final
mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -4 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke.log
run() { local n=$1; shift; timeout 900 python bench.py "$@" > $OUT/bench_$n.json 2> $OUT/bench_$n.err; echo "$n rc=$?"; python -c "import json;d=json.loads(open('$OUT/bench_$n.json').read().strip().splitlines()[-1]);print('$n', d['value'], (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('frac'), (d.get('clocks') or {}).get('sm_mhz'))"; }
run tw --steps 20 --warmup 5
run tw_plan --schedule plan --steps 20 --warmup 5
run ref --impl reference --steps 20 --warmup 5
run lj --config lj --steps 5
run fm --config fm --steps 5
run friendster --config friendster --steps 5
run fb15k --config fb15k --steps 5 --warmup 3
run shared --negatives 1000 --shared-chunk 1000 --steps 10
run eval --eval 1000000
B="python bench.py --schedule plan --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $B > $OUT/ncu_launch.log 2>&1; echo "launches rc=$?"
for c in tw fm friendster lj; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"segment_heads|score_kernel" -s 12 -c 2 -o /tmp/full_$c $B --config $c > $OUT/ncu_full_$c.log 2>&1; echo "full $c rc=$?"
  python profiles/summarize.py $OUT/launches.csv /tmp/full_$c.ncu-rep $OUT $c > /dev/null 2>&1; echo "summary $c rc=$?"
  ncu -i /tmp/full_$c.ncu-rep --page source --csv --print-source sass > /tmp/src_$c.csv 2>/dev/null
  python - "$c" <<'PY'
import csv, json, sys, collections
c = sys.argv[1]
rows = list(csv.reader(open(f"/tmp/src_{c}.csv")))
out = {}
kernel = None
for r in rows:
    if len(r) >= 2 and r[0] == "Kernel Name":
        kernel = r[1]; out[kernel] = collections.Counter(); continue
    if kernel is None or len(r) < 6 or r[0] == "Address":
        continue
    try:
        n = int(r[5])
    except ValueError:
        continue
    src = r[1].strip()
    op = (src.split()[1] if src.startswith("@") else src.split()[0]).split(".")[0] if src else "?"
    out[kernel][op] += n
res = {k: {"warp_instructions": sum(v.values()), "mix_top": v.most_common(25)} for k, v in out.items()}
json.dump(res, open(f"gpurun_out/r02final/sass_mix_{c}.json", "w"), indent=1)
PY
  rm -f /tmp/full_$c.ncu-rep
done
cp profiles/ncu_traffic.json $OUT/ncu_traffic.json
du -sh gpurun_out
