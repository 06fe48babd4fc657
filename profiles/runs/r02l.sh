# final round-2 evidence: GPU tests, smoke, every config's bench line, the
# reference arm, launch list and full ncu captures per config
set -x
OUT=gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > $OUT/r02l_pytest.log 2>&1; echo "gpu tests rc=$?"; tail -4 $OUT/r02l_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/r02l_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/r02l_smoke.log
run() { local n=$1; shift; timeout 900 python bench.py "$@" > $OUT/r02l_bench_$n.json 2> $OUT/r02l_bench_$n.err; echo "$n rc=$? $(tail -c 400 $OUT/r02l_bench_$n.json | head -c 400)"; }
run tw --steps 20 --warmup 5
run tw_plan --schedule plan --steps 20 --warmup 5
run ref --impl reference --steps 20 --warmup 5
run lj --config lj --steps 5
run fm --config fm --steps 5
run friendster --config friendster --steps 5
run fb15k --config fb15k --steps 5 --warmup 3
run shared --negatives 1000 --shared-chunk 1000 --steps 10
run eval --eval 1000000
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/r02l_launches.csv $B > $OUT/r02l_ncu_launch.log 2>&1; echo "launches rc=$?"
for c in tw fm friendster lj; do
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"segment_heads|score_kernel" -s 12 -c 2 -o $OUT/r02l_full_$c $B --config $c > $OUT/r02l_ncu_full_$c.log 2>&1; echo "full $c rc=$?"
done
