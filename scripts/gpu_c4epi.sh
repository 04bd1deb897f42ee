cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python -m pytest tests/test_gpu_conv.py tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 300 --timeout-method=thread 2>&1 | tail -1
timeout -s KILL 300 python scripts/prof_layer.py --config c4 --iters 20 2>&1 | grep "layer 0"
timeout -s KILL 300 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('c5', round(d['ms_per_step'],2), 'ms')"
