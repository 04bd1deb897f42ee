cd $GRAFT_REPO_ROOT
KAN_CONV3_MC=4 timeout -s KILL 600 python -m pytest tests/test_gpu_conv.py -q -p no:cacheprovider --timeout 120 --timeout-method=thread 2>&1 | tail -1
for mc in 2 4 8; do KAN_CONV3_MC=$mc timeout -s KILL 120 python scripts/prof_layer.py --config c4 --iters 20 2>&1 | grep "layer 0" | sed "s/^/c4 mc $mc: /"; done
for mc in 2 4; do KAN_CONV3_MC=$mc timeout -s KILL 300 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('c5 mc $mc', round(d['ms_per_step'],2), 'ms')"; done
