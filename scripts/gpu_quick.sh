cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/t3.log 2>&1; echo PYTEST $?
tail -3 gpurun_out/t3.log
for cfg in c2 c1 c3; do echo "== $cfg"; timeout -s KILL 200 python scripts/prof_layer.py --config $cfg --iters 20; done
timeout -s KILL 300 python bench.py --steps 20000 --warmup 200 --no-cpu-baseline > gpurun_out/bench_c2b.json 2> gpurun_out/bench_c2b.err; echo BENCH $?
python -c "import json;d=json.load(open('gpurun_out/bench_c2b.json'));print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['roofline']['layer_avg_ms'])"
