cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/bench
run() { timeout -s KILL 900 python bench.py --config $1 --steps $2 --warmup $3 --cpu-seconds 10 > gpurun_out/bench/ours_$1.json 2> gpurun_out/bench/ours_$1.err; echo "BENCH $1 $?"; }
run c2 20000 200
run c1 20000 200
for f in gpurun_out/bench/ours_c1.json gpurun_out/bench/ours_c2.json; do python -c "
import json,sys;d=json.load(open('$f'));r=d['roofline']
print('$f'.split('/')[-1], '%.4g'%d['value'], round(d['ms_per_step']*1e3,1),'us', r['bound'], round(r['frac'],3), r['kernel'], d['clocks'])"; done
