cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python -m pytest tests/test_gpu_spline_table.py tests/test_gpu_fakequant.py -q -p no:cacheprovider 2>&1 | tail -2
for v in 1 0; do for c in c1st c2st; do KAN_ST_PREPASS=$v timeout -s KILL 300 python bench.py --config $c --steps 3000 --warmup 30 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('prepass $v $c', round(d['ms_per_step']*1e3,2), 'us', d['gpu_launches']//d['steps'])"; done; done
