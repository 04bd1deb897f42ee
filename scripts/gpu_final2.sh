# Round evidence: GPU tests, smoke, every bench line, reference arm, launch lists, ncu captures.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/bench gpurun_out/prof
timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/bench/pytest_gpu.log 2>&1; echo "PYTEST $?"; tail -1 gpurun_out/bench/pytest_gpu.log
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/bench/smoke.log 2>&1; echo "SMOKE $?"; tail -1 gpurun_out/bench/smoke.log
run() { timeout -s KILL 900 python bench.py --config $1 --steps $2 --warmup $3 --cpu-seconds 10 > gpurun_out/bench/ours_$1.json 2> gpurun_out/bench/ours_$1.err; echo "BENCH $1 $?"; }
run c2 20000 200
run c1 20000 200
run c3 100 5
run c3bf16 40 3
run c4 2000 20
run c5 30 3
run c1st 5000 50
run c2st 5000 50
run c2st4 5000 50
run c4st 300 10
timeout -s KILL 600 python bench.py --impl reference --config c2 --steps 50 --warmup 3 > gpurun_out/bench/ref_c2.json 2> gpurun_out/bench/ref_c2.err; echo "REF c2 $?"
timeout -s KILL 600 python bench.py --impl reference --config c5 --steps 5 --warmup 1 > gpurun_out/bench/ref_c5.json 2> gpurun_out/bench/ref_c5.err; echo "REF c5 $?"
for cfg in c2 c4; do
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof/launches_$cfg.csv python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "LAUNCH $cfg $?"
done
cap() { timeout -s KILL 200 python scripts/prof_layer.py --config $2 --iters 2 --nograph $4 > /dev/null 2>&1 && timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:$5 -s $3 -c 1 -o gpurun_out/prof/$1 python scripts/prof_layer.py --config $2 --iters 2 --nograph $4 > /dev/null 2>&1; echo "CAP $1 $?"; }
cap c2_l0 c2 1 "" kan_gather
cap c3_l0 c3 3 "" kan_gather
cap c4_conv c4 1 "" kan_conv3
cap c5_l2 c5 0 "--batch 8192" "kan_conv3"
for f in gpurun_out/bench/ours_*.json; do python -c "
import json,sys;d=json.load(open('$f'));r=d['roofline'];c=d.get('cpu_baseline') or {}
print('$f'.split('/')[-1], '%.4g'%d['value'], round(d['ms_per_step']*1e3,1),'us', r['bound'], round(r['frac'],3), 'e2e %.3g'%d['e2e']['value'], 'cpu', round(c.get('value') or 0,1), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"; done
