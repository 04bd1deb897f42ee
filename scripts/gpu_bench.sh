cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() { # config steps warmup
  timeout -s KILL 600 python bench.py --config $1 --steps $2 --warmup $3 --cpu-seconds 10 > gpurun_out/bench_$1.json 2> gpurun_out/bench_$1.err
  echo "BENCH $1 $?"
  python -c "import json;d=json.load(open('gpurun_out/bench_$1.json'));r=d['roofline'];print(d['value'],d['ms_per_step'],r['bound'],round(r['frac'],3),[round(v*1e3,1) for v in r['layer_avg_ms']], d['e2e']['value'], (d['cpu_baseline'] or {}).get('value'))" 2>&1 | tail -1
}
run c4 2000 20
run c5 40 3
run c2 20000 200
run c3 100 5
