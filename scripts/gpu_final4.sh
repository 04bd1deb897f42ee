# Round evidence after the epilogue instantiations: GPU tests, smoke, bench lines, launch lists, C2 ncu.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/f4
timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/f4/pytest_gpu.log 2>&1; echo "PYTEST $?"; tail -1 gpurun_out/f4/pytest_gpu.log
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f4/smoke.log 2>&1; echo "SMOKE $?"; tail -1 gpurun_out/f4/smoke.log
run() { timeout -s KILL 900 python bench.py --config $1 --steps $2 --warmup $3 --cpu-seconds 10 > gpurun_out/f4/ours_$1.json 2> gpurun_out/f4/ours_$1.err; echo "BENCH $1 $?"; }
run c2 20000 200
run c1 20000 200
run c3 100 5
run c3bf16 40 3
run c4 2000 20
run c5 30 3
for cfg in c2 c1; do
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f4/launches_$cfg.csv python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "LAUNCH $cfg $?"
done
timeout -s KILL 200 python scripts/prof_layer.py --config c2 --iters 2 --nograph > /dev/null 2>&1 && timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:kan_gather -s 1 -c 1 -o gpurun_out/f4/c2_l0 python scripts/prof_layer.py --config c2 --iters 2 --nograph > /dev/null 2>&1; echo "CAP $?"
for f in gpurun_out/f4/ours_*.json; do python -c "
import json,sys;d=json.load(open('$f'));r=d['roofline'];c=d.get('cpu_baseline') or {}
print('$f'.split('/')[-1], '%.4g'%d['value'], round(d['ms_per_step']*1e3,1),'us', r['bound'], round(r['frac'],3), 'e2e %.3g'%d['e2e']['value'], 'cpu', round(c.get('value') or 0,1), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"; done
