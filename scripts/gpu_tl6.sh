cd $GRAFT_REPO_ROOT
timeout -s KILL 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_conv.py -q -p no:cacheprovider 2>&1 | tail -2
echo "== c2"; KAN_TIMELINE=1 timeout -s KILL 120 python scripts/timeline.py --config c2 2>&1 | grep -E "lastA|tmemfull|partials|reduced|done|span"
for c in c2 c1; do timeout -s KILL 200 python bench.py --config $c --steps 5000 --warmup 50 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('bench $c', round(d['ms_per_step']*1e3,2), 'us')"; done
