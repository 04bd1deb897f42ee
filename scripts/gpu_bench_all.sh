cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/bench
run() { # config steps warmup
  timeout -s KILL 900 python bench.py --config $1 --steps $2 --warmup $3 --cpu-seconds 10 > gpurun_out/bench/ours_$1.json 2> gpurun_out/bench/ours_$1.err
  echo "BENCH $1 $?"
}
run c2 20000 200
run c1 20000 200
run c3 100 5
run c3bf16 40 3
run c4 2000 20
run c5 30 3
timeout -s KILL 600 python bench.py --impl reference --config c2 --steps 50 --warmup 3 > gpurun_out/bench/ref_c2.json 2> gpurun_out/bench/ref_c2.err; echo "REF c2 $?"
timeout -s KILL 600 python bench.py --impl reference --config c5 --steps 5 --warmup 1 > gpurun_out/bench/ref_c5.json 2> gpurun_out/bench/ref_c5.err; echo "REF c5 $?"
for f in gpurun_out/bench/ours_*.json; do python -c "
import json,sys;d=json.load(open('$f'));r=d['roofline'];c=d.get('cpu_baseline') or {}
print('$f'.split('/')[-1], round(d['value']), round(d['ms_per_step']*1e3,1),'us', r['bound'], round(r['frac'],3), 'e2e', round(d['e2e']['value']), 'cpu', round(c.get('value') or 0,1), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"; done
