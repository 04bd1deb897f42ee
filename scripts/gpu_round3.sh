cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/bench gpurun_out/prof
timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/bench/pytest_gpu.log 2>&1; echo "PYTEST $?"; tail -1 gpurun_out/bench/pytest_gpu.log
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/bench/smoke.log 2>&1; echo "SMOKE $?"; tail -1 gpurun_out/bench/smoke.log
run() { timeout -s KILL 900 python bench.py --config $1 --steps $2 --warmup $3 --cpu-seconds 10 > gpurun_out/bench/ours_$1.json 2> gpurun_out/bench/ours_$1.err; echo "BENCH $1 $?"; }
run c2 20000 200
run c1 20000 200
run c1st 5000 50
run c2st 5000 50
timeout -s KILL 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline > gpurun_out/bench/default.json 2>/dev/null; echo "DEFAULT $?"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof/launches_c2.csv python bench.py --config c2 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "LAUNCH c2 $?"
for f in gpurun_out/bench/ours_*.json gpurun_out/bench/default.json; do python -c "
import json,sys;d=json.load(open('$f'));r=d['roofline'];c=d.get('cpu_baseline') or {}
print('$f'.split('/')[-1], '%.4g'%d['value'], round(d['ms_per_step']*1e3,1),'us', r['bound'], round(r['frac'],3), 'e2e %.3g'%d['e2e']['value'], 'cpu', round(c.get('value') or 0,1), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'), d['config'].get('streams'))"; done
